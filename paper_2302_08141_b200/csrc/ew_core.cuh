// ew_core.cuh — device code of the elementwise chain programs (ew_defs.h), shared by the
// nvcc-built interpreter kernels (k_elementwise.cu) and the per-program kernels ew_jit.cpp
// compiles with NVRTC at program load.  One instruction's semantics live in EwStep only: the
// interpreter calls it with the (warp-uniform) instruction read from the program, a specialized
// kernel with literal constants, so the compiler folds every switch away and the two paths
// execute the same arithmetic in the same order (bit-identical results by construction).
//
// One 16-byte vector per input per thread-iteration (8 bf16 / 4 fp32 elements); bf16 stays
// packed (bf16x2 add/mul round exactly like the fp32 op + bf16 rounding: a bf16 sum or product
// is exact in fp32).
#pragma once

#ifndef __CUDACC_RTC__  // (NVRTC: ew_jit.cpp's prelude provides these)
#include <cuda_bf16.h>

#include "ew_defs.h"
#include "pdl.cuh"
#include "unary.cuh"
#endif

namespace rh {

template <bool kBf16>
__device__ __forceinline__ float LoadScalar(const void* p, int64_t i) {
  if (kBf16) return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
  return reinterpret_cast<const float*>(p)[i];
}
template <bool kBf16>
__device__ __forceinline__ void StoreScalar(void* p, int64_t i, float x) {
  if (kBf16) {
    reinterpret_cast<__nv_bfloat16*>(p)[i] = __float2bfloat16_rn(x);
  } else {
    reinterpret_cast<float*>(p)[i] = x;
  }
}

__device__ __forceinline__ uint4 EwPick(const uint4 (&r)[kMaxEwIn], int k) {
  switch (k) {  // warp-uniform: static register indices, no local memory
    case 0: return r[0];
    case 1: return r[1];
    case 2: return r[2];
    case 3: return r[3];
    case 4: return r[4];
    case 5: return r[5];
    case 6: return r[6];
    default: return r[7];
  }
}

// Programs with at most N inputs: only N input vectors live (the rematerializing backward
// chains: 4, which buys a third / fourth resident block per SM).
template <int N>
__device__ __forceinline__ uint4 EwPickN(const uint4 (&r)[kMaxEwIn], int k) {
  if constexpr (N <= 1) return r[0];
  if constexpr (N == 2) return k == 0 ? r[0] : r[1];
  if constexpr (N <= 4) {
    switch (k) {
      case 0: return r[0];
      case 1: return r[1];
      case 2: return r[2];
      default: return r[3];
    }
  }
  return EwPick(r, k);
}

__device__ __forceinline__ uint32_t AddBf16x2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("add.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}
__device__ __forceinline__ uint32_t MulBf16x2(uint32_t a, uint32_t b) {
  uint32_t d;
  asm("mul.rn.bf16x2 %0, %1, %2;" : "=r"(d) : "r"(a), "r"(b));
  return d;
}

// TanhRunLookup on both halves of a bf16x2 register.
__device__ __forceinline__ uint32_t TanhRunLookup2(uint32_t p, const uint16_t* tab) {
  constexpr uint32_t kLo = 122u << 7, kSpan = 0x7f80u - (122u << 7), kLast = kTanhRunEntries - 1;
  const uint32_t lo = p & 0x7fffu, hi = (p >> 16) & 0x7fffu;
  const uint32_t ulo = lo - kLo, uhi = hi - kLo;
  const uint32_t tlo = tab[min(ulo, kLast)], thi = tab[min(uhi, kLast)];
  const uint32_t rlo = ulo > kSpan ? lo : tlo;
  const uint32_t rhi = uhi > kSpan ? hi : thi;
  return (p & 0x80008000u) | rlo | (rhi << 16);
}

// Ladder rows of 8 packed bf16 values (2 x 16-byte shared loads each; |x| < 2^-5 and NaN pass
// through every T^c unchanged, as in the ladder kernel).
// kHalf: a table of half rows (columns 0..7 only, 16 bytes per row): programs whose
// rematerialized operands use at most 8 powers fetch one 16-byte row per element, not two.
template <bool kHalf = false>
__device__ __forceinline__ void LadderRows(const uint4 v, const uint4* lad_s, uint4 (&r)[8][2]) {
  constexpr uint32_t kLo = 122u << 7, kSpan = 0x7f80u - (122u << 7), kLast = kTanhRunEntries - 1;
  const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    const uint32_t ab = ((e & 1) ? (w[e >> 1] >> 16) : w[e >> 1]) & 0x7fffu;
    const uint32_t u = ab - kLo;
    const uint32_t row = min(u, kLast);
    if constexpr (kHalf) {
      r[e][0] = lad_s[row];
      if (u > kSpan) {
        const uint32_t rep = ab | (ab << 16);
        r[e][0] = make_uint4(rep, rep, rep, rep);
      }
    } else {
      r[e][0] = lad_s[2 * row];
      r[e][1] = lad_s[2 * row + 1];
      if (u > kSpan) {
        const uint32_t rep = ab | (ab << 16);
        r[e][0] = r[e][1] = make_uint4(rep, rep, rep, rep);
      }
    }
  }
}

__device__ __forceinline__ uint32_t U32OfRow(const uint4 (&r)[2], int w) {
  const uint4 q = r[w >> 2];
  return (w & 3) == 0 ? q.x : (w & 3) == 1 ? q.y : (w & 3) == 2 ? q.z : q.w;
}

// S must fold to a constant (template argument, or an unrolled loop index): static registers.
__device__ __forceinline__ uint4 LadderColI(const uint4 (&r)[8][2], uint4 base, const int S) {
  const uint32_t sel = (S & 1) ? 0x7632u : 0x5410u;
  const uint32_t b[4] = {base.x, base.y, base.z, base.w};
  uint32_t p[4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
    p[q] = __byte_perm(U32OfRow(r[2 * q], S >> 1), U32OfRow(r[2 * q + 1], S >> 1), sel) | (b[q] & 0x80008000u);
  return make_uint4(p[0], p[1], p[2], p[3]);
}

template <int S>
__device__ __forceinline__ uint4 LadderCol(const uint4 (&r)[8][2], uint4 base) {
  return LadderColI(r, base, S);
}

// Operand k of the program: an input vector, or (k >= kEwSrcVirt) a ladder column of the
// rematerialization base (warp-uniform switch: static register indices).
template <bool kHalf, int kIn>
__device__ __forceinline__ uint4 EwOperand(const uint4 (&raw)[kMaxEwIn], const uint4 (&r)[8][2], uint4 base,
                                           int k) {
  if (k < kEwSrcVirt) return EwPickN<kIn>(raw, k);
  if constexpr (kHalf) {
    switch (k - kEwSrcVirt) {
      case 0: return LadderCol<0>(r, base);
      case 1: return LadderCol<1>(r, base);
      case 2: return LadderCol<2>(r, base);
      case 3: return LadderCol<3>(r, base);
      case 4: return LadderCol<4>(r, base);
      case 5: return LadderCol<5>(r, base);
      case 6: return LadderCol<6>(r, base);
      default: return LadderCol<7>(r, base);
    }
  }
  switch (k - kEwSrcVirt) {
    case 0: return LadderCol<0>(r, base);
    case 1: return LadderCol<1>(r, base);
    case 2: return LadderCol<2>(r, base);
    case 3: return LadderCol<3>(r, base);
    case 4: return LadderCol<4>(r, base);
    case 5: return LadderCol<5>(r, base);
    case 6: return LadderCol<6>(r, base);
    case 7: return LadderCol<7>(r, base);
    case 8: return LadderCol<8>(r, base);
    case 9: return LadderCol<9>(r, base);
    case 10: return LadderCol<10>(r, base);
    case 11: return LadderCol<11>(r, base);
    case 12: return LadderCol<12>(r, base);
    case 13: return LadderCol<13>(r, base);
    case 14: return LadderCol<14>(r, base);
    default: return LadderCol<15>(r, base);
  }
}

// Scalar form of a ladder column (tail elements; the table in global memory).
__device__ __forceinline__ float LadderScalar(float x, const uint4* lad, int s) {
  constexpr uint32_t kLo = 122u << 7, kSpan = 0x7f80u - (122u << 7), kLast = kTanhRunEntries - 1;
  const uint32_t bits = __float_as_uint(x) >> 16;
  const uint32_t ab = bits & 0x7fffu, u = ab - kLo;
  const uint16_t* t = reinterpret_cast<const uint16_t*>(lad);
  const uint32_t v = u > kSpan ? ab : t[min(u, kLast) * kLadderWidth + s];
  return __uint_as_float(((bits & 0x8000u) | v) << 16);
}

// Per-thread state of one vector of the program.
template <int kIn>
struct EwVec {
  uint4 raw[kMaxEwIn];
  uint4 vr[8][2];  // rematerialization ladder rows (kRemat)
  uint4 vbase;
  uint32_t acc[4], keep[4];
};

// One instruction (op, arg) of the program on vector i.  kIn: inputs live in registers.
template <bool kBf16, bool kRemat, bool kHalf, int kIn>
__device__ __forceinline__ void EwStep(const EwArgs& a, int64_t i, const uint16_t* tabs, EwVec<kIn>& v,
                                       const int op, const int arg) {
  uint32_t (&acc)[4] = v.acc;
  uint32_t (&keep)[4] = v.keep;
  switch (op) {
    case kEwLoad: {
      const uint4 x = kRemat ? EwOperand<kHalf, kIn>(v.raw, v.vr, v.vbase, arg) : EwPickN<kIn>(v.raw, arg);
      acc[0] = x.x; acc[1] = x.y; acc[2] = x.z; acc[3] = x.w;
      break;
    }
    case kEwKeep:
#pragma unroll
      for (int e = 0; e < 4; ++e) keep[e] = acc[e];
      break;
    case kEwStore:
      reinterpret_cast<uint4*>(a.out[arg])[i] = make_uint4(acc[0], acc[1], acc[2], acc[3]);
      break;
    case kEwTanhBwdLad: {
      if constexpr (kBf16 && kRemat) {
        const int hi = arg & 15, cnt = arg >> 4;
#pragma unroll
        for (int S = kHalf ? 7 : 15; S >= 0; --S) {
          if (S > hi || S <= hi - cnt) continue;
          const uint4 x = LadderColI(v.vr, v.vbase, S);
          const uint32_t y[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            keep[e] = acc[e];
            const uint32_t t = MulBf16x2(MulBf16x2(acc[e], y[e]), y[e]);
            acc[e] = AddBf16x2(keep[e], t ^ 0x80008000u);
          }
        }
      } else {
        __trap();  // emitted only for bf16 rematerializing programs (EmitEwChain): misrouted
      }
      break;
    }
    case kEwTanhBwd: {
      const uint4 x = kRemat ? EwOperand<kHalf, kIn>(v.raw, v.vr, v.vbase, arg) : EwPickN<kIn>(v.raw, arg);
      const uint32_t y[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        keep[e] = acc[e];
        if constexpr (kBf16) {
          const uint32_t t = MulBf16x2(MulBf16x2(acc[e], y[e]), y[e]);
          acc[e] = AddBf16x2(keep[e], t ^ 0x80008000u);
        } else {
          const float yy = __uint_as_float(y[e]);
          const float t = __fmul_rn(__fmul_rn(__uint_as_float(acc[e]), yy), yy);
          acc[e] = __float_as_uint(__fadd_rn(__uint_as_float(keep[e]), -t));
        }
      }
      break;
    }
    case kEwAdd:
    case kEwMul: {
      uint32_t w[4];
      if (arg == kEwSrcKeep) {
#pragma unroll
        for (int e = 0; e < 4; ++e) w[e] = keep[e];
      } else if (arg == kEwSrcAcc) {
#pragma unroll
        for (int e = 0; e < 4; ++e) w[e] = acc[e];
      } else {
        const uint4 x = kRemat ? EwOperand<kHalf, kIn>(v.raw, v.vr, v.vbase, arg) : EwPickN<kIn>(v.raw, arg);
        w[0] = x.x; w[1] = x.y; w[2] = x.z; w[3] = x.w;
      }
      if constexpr (kBf16) {
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[e] = op == kEwAdd ? AddBf16x2(acc[e], w[e]) : MulBf16x2(acc[e], w[e]);
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float x = __uint_as_float(acc[e]), y = __uint_as_float(w[e]);
          acc[e] = __float_as_uint(op == kEwAdd ? __fadd_rn(x, y) : __fmul_rn(x, y));
        }
      }
      break;
    }
    default:  // kEwUnary
      if constexpr (kBf16) {
        if (arg >= kFnTanhRun) {
          const uint16_t* tab = tabs + (arg - kFnTanhRun) * kTanhRunEntries;
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[e] = TanhRunLookup2(acc[e], tab);
        } else {
          const int32_t fn = arg;
          ApplyChainPackedBf16<4>(&fn, 1, acc, tabs);
        }
      } else {
        float x[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) x[e] = __uint_as_float(acc[e]);
        const int32_t fn = arg;
        ApplyChainVecF32<4>(&fn, 1, x);
#pragma unroll
        for (int e = 0; e < 4; ++e) acc[e] = __float_as_uint(x[e]);
      }
  }
}

// Loads vector i's inputs (kExact: exactly kIn inputs, else the first a.n_in <= kIn) and, for
// rematerializing programs, the base's ladder rows; clears acc / keep.  kPre: the inputs are
// already in v.raw (loaded one iteration ahead).
template <bool kBf16, bool kRemat, bool kHalf, int kIn, bool kExact, bool kPre = false>
__device__ __forceinline__ void EwVecBegin(const EwArgs& a, int64_t i, const uint4* vlad_s, EwVec<kIn>& v) {
  if constexpr (!kPre) {
#pragma unroll
    for (int k = 0; k < kIn; ++k)
      if (kExact || k < a.n_in) v.raw[k] = reinterpret_cast<const uint4*>(a.in[k])[i];
  }
  v.vbase = make_uint4(0, 0, 0, 0);
  if constexpr (kBf16 && kRemat) {
    v.vbase = EwPickN<kIn>(v.raw, a.vlad_in);
    LadderRows<kHalf>(v.vbase, vlad_s, v.vr);
  }
#pragma unroll
  for (int e = 0; e < 4; ++e) v.acc[e] = v.keep[e] = 0;
}

// The interpreter: instructions [0, pc_end) of the program, read per vector.
template <bool kBf16, bool kRemat, bool kHalf, int kIn>
struct EwInterp {
  int pc_end;
  __device__ __forceinline__ void operator()(const EwArgs& a, int64_t i, const uint16_t* tabs, EwVec<kIn>& v) const {
    for (int pc = 0; pc < pc_end; ++pc) {
      const int ins = a.code[pc];
      EwStep<kBf16, kRemat, kHalf, kIn>(a, i, tabs, v, ins & 0xff, ins >> 8);
    }
  }
};

// Scalar tail (n not a multiple of the vector): same semantics on unpacked values.
template <bool kBf16>
__device__ __forceinline__ float EwScalarOperand(const EwArgs& a, int64_t i, int k) {
  if (k < kEwSrcVirt) return LoadScalar<kBf16>(a.in[k], i);
  return LadderScalar(LoadScalar<kBf16>(a.in[a.vlad_in], i), a.vlad, k - kEwSrcVirt);
}

template <bool kBf16>
__device__ __noinline__ void EwRunScalar(const EwArgs& a, int64_t i, const uint16_t* tabs) {
  float acc = 0.0f, keep = 0.0f;
  for (int pc = 0; pc < a.n_code; ++pc) {
    const int ins = a.code[pc], op = ins & 0xff, arg = ins >> 8;
    switch (op) {
      case kEwLoad: acc = EwScalarOperand<kBf16>(a, i, arg); break;
      case kEwKeep: keep = acc; break;
      case kEwStore: StoreScalar<kBf16>(a.out[arg], i, acc); break;
      case kEwTanhBwdLad: {
        const int hi = arg & 15, cnt = arg >> 4;
        const float b = LoadScalar<kBf16>(a.in[a.vlad_in], i);
        for (int c = 0; c < cnt; ++c) {
          const float y = LadderScalar(b, a.vlad, hi - c);
          keep = acc;
          float t = __fmul_rn(acc, y);
          if (kBf16) t = RoundBf16(t);
          t = __fmul_rn(t, y);
          if (kBf16) t = RoundBf16(t);
          acc = __fadd_rn(keep, -t);
          if (kBf16) acc = RoundBf16(acc);
        }
        break;
      }
      case kEwTanhBwd: {
        const float y = EwScalarOperand<kBf16>(a, i, arg);
        keep = acc;
        float t = __fmul_rn(acc, y);
        if (kBf16) t = RoundBf16(t);
        t = __fmul_rn(t, y);
        if (kBf16) t = RoundBf16(t);
        acc = __fadd_rn(keep, -t);
        if (kBf16) acc = RoundBf16(acc);
        break;
      }
      case kEwAdd:
      case kEwMul: {
        const float w = arg == kEwSrcKeep ? keep : arg == kEwSrcAcc ? acc : EwScalarOperand<kBf16>(a, i, arg);
        acc = op == kEwAdd ? __fadd_rn(acc, w) : __fmul_rn(acc, w);
        if (kBf16) acc = RoundBf16(acc);
        break;
      }
      default:
        if (kBf16 && arg >= kFnTanhRun) {
          acc = __uint_as_float(TanhRunLookup(__float_as_uint(acc) >> 16, tabs + (arg - kFnTanhRun) * kTanhRunEntries) << 16);
        } else {
          const int32_t fn = arg;
          acc = ApplyChainFns<kBf16>(&fn, 1, acc);
        }
    }
  }
}

// Block-wide copy of n table entries global -> shared with every thread's loads issued before
// its stores (the tables are L2-resident: one round trip instead of n / blockDim dependent ones).
// Assumes blockDim.x == 256 and n <= 8 * 256.
template <typename T>
__device__ __forceinline__ void StageTable(T* __restrict__ dst, const T* __restrict__ src, int n, int src_stride = 1) {
  T v[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int i = threadIdx.x + j * 256;
    if (i < n) v[j] = src[static_cast<int64_t>(i) * src_stride];
  }
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    const int i = threadIdx.x + j * 256;
    if (i < n) dst[i] = v[j];
  }
}

// Kernel body of a chain program: stage the tanh-run tables (and the rematerialization ladder)
// in shared memory, then one vector per thread-iteration through `prog` (EwInterp, or a
// specialized instruction sequence), then the scalar tail.
template <bool kBf16, bool kRemat, bool kHalf, int kIn, bool kExact, class Prog>
__device__ __forceinline__ void EwProgBody(const EwArgs& a, const Prog& prog) {
  PdlTrigger();
  __shared__ uint16_t tab_s[kBf16 ? kMaxTanhRuns * kTanhRunEntries : 1];
  extern __shared__ uint4 vlad_s[];  // rematerialization ladder (vlad_n > 0); kHalf: half rows
  if constexpr (kBf16) {
    for (int t = 0; t < a.n_tab; ++t)
      StageTable(tab_s + t * kTanhRunEntries, a.tab[t], kTanhRunEntries);
    if (kRemat) {
      if (kHalf) StageTable(vlad_s, a.vlad, kTanhRunEntries, 2);
      else StageTable(vlad_s, a.vlad, kTanhRunEntries * 2);
    }
    __syncthreads();
  }
  PdlWait();
  constexpr int E = kBf16 ? 8 : 4;
  const int64_t nv = a.n / E;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
#ifndef RH_EW_PAIR_VECTORS
#define RH_EW_PAIR_VECTORS 1
#endif
  if constexpr (kExact && !kRemat && kIn <= 4 && RH_EW_PAIR_VECTORS) {
    // specialized programs with few inputs: two vectors per iteration, the second one's inputs
    // loaded before the first one's program runs (two loads per input in flight per thread;
    // measured -5..10% on the C5 forward chains, neutral on the rematerializing ones, whose
    // ladder rows double the live registers: profiles/r2/ew_jit_c5.txt)
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nv; i += 2 * stride) {
      const int64_t i2 = i + stride;
      uint4 nxt[kIn];
      if (i2 < nv) {
#pragma unroll
        for (int k = 0; k < kIn; ++k) nxt[k] = reinterpret_cast<const uint4*>(a.in[k])[i2];
      }
      if constexpr (kRemat) {
        const int64_t nx = i + 2 * stride;
        if (nx < nv)
#pragma unroll
          for (int k = 0; k < kIn; ++k)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const uint4*>(a.in[k]) + nx));
      }
      {
        EwVec<kIn> v;
        EwVecBegin<kBf16, kRemat, kHalf, kIn, kExact>(a, i, vlad_s, v);
        prog(a, i, tab_s, v);
      }
      if (i2 < nv) {
        EwVec<kIn> v;
#pragma unroll
        for (int k = 0; k < kIn; ++k) v.raw[k] = nxt[k];
        EwVecBegin<kBf16, kRemat, kHalf, kIn, kExact, true>(a, i2, vlad_s, v);
        prog(a, i2, tab_s, v);
      }
    }
  } else {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nv; i += stride) {
    if constexpr (kRemat) {
      // few warps per SM: L2-prefetch the next iteration's vectors so their loads do not wait
      // on HBM latency (no registers held)
      const int64_t nx = i + stride;
      if (nx < nv)
        for (int k = 0; k < (kExact ? kIn : a.n_in); ++k)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const uint4*>(a.in[k]) + nx));
    }
    EwVec<kIn> v;
    EwVecBegin<kBf16, kRemat, kHalf, kIn, kExact>(a, i, vlad_s, v);
    prog(a, i, tab_s, v);
  }
  }
  for (int64_t i = nv * E + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < a.n; i += stride)
    EwRunScalar<kBf16>(a, i, tab_s);
}

// bf16 chain program with a tanh ladder suffix (EwArgs::lad_*): `prog` runs the prefix
// [0, lad_pc), then every element's lad_n outputs come from its ladder row (2 x 16-byte shared
// loads) and are re-packed per output with byte permutes: ~30 instructions per element for a
// 12-store chain instead of ~20 per op and element.  |x| < 2^-5 and NaN pass through every
// T^c unchanged; T is odd, so the sign is OR-ed back.
template <bool kRemat, int kIn, bool kExact, class Prog>
__device__ __forceinline__ void EwLadderBody(const EwArgs& a, const Prog& prog) {
  PdlTrigger();
  extern __shared__ uint4 lad_s[];  // kTanhRunEntries rows x 2 uint4
  __shared__ uint16_t tab_s[kMaxTanhRuns * kTanhRunEntries];
  for (int t = 0; t < a.n_tab; ++t)
    StageTable(tab_s + t * kTanhRunEntries, a.tab[t], kTanhRunEntries);
  StageTable(lad_s, a.lad, kTanhRunEntries * 2);
  uint4* vlad_s = lad_s + kTanhRunEntries * 2;  // rematerialization ladder (vlad_n > 0)
  if (kRemat)
    StageTable(vlad_s, a.vlad, kTanhRunEntries * 2);
  __syncthreads();
  PdlWait();
  constexpr uint32_t kLo = 122u << 7, kSpan = 0x7f80u - (122u << 7), kLast = kTanhRunEntries - 1;
  const int64_t nv = a.n / 8;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nv; i += stride) {
    EwVec<kIn> v;
    EwVecBegin<true, kRemat, false, kIn, kExact>(a, i, vlad_s, v);
    prog(a, i, tab_s, v);
    uint4 r[8][2];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t pr = v.acc[e >> 1];
      const uint32_t ab = ((e & 1) ? (pr >> 16) : pr) & 0x7fffu;
      const uint32_t u = ab - kLo;
      const uint32_t row = min(u, kLast);
      r[e][0] = lad_s[2 * row];
      r[e][1] = lad_s[2 * row + 1];
      if (u > kSpan) {
        const uint32_t rep = ab | (ab << 16);
        r[e][0] = r[e][1] = make_uint4(rep, rep, rep, rep);
      }
    }
    uint32_t sg[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) sg[q] = v.acc[q] & 0x80008000u;
#pragma unroll
    for (int s = 0; s < kLadderWidth; ++s) {
      if (s >= a.lad_n) break;
      const uint32_t sel = (s & 1) ? 0x7632u : 0x5410u;
      uint32_t p[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        p[q] = __byte_perm(U32OfRow(r[2 * q], s >> 1), U32OfRow(r[2 * q + 1], s >> 1), sel) | sg[q];
      reinterpret_cast<uint4*>(a.out[a.lad_out[s]])[i] = make_uint4(p[0], p[1], p[2], p[3]);
    }
  }
  for (int64_t i = nv * 8 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < a.n; i += stride)
    EwRunScalar<true>(a, i, tab_s);
}

}  // namespace rh
