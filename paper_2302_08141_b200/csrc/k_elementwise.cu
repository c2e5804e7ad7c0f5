// k_elementwise.cu — local (per-rank) non-GEMM operators: K2 add/mul, K3 fused unary chains,
// softmax rows, K4 reduce_sum, K5 transpose, K6 broadcast, K7 concat.  All HBM-bound: 16-byte
// vector loads/stores, grid-stride loops sized to the 148 SMs.
//
// Unary semantics (the reference leaves them undefined, include/parashard/ir.h:87; DESIGN.md
// §Semantics): evaluated in fp32 with the expression order below (explicit _rn intrinsics so
// no FMA contraction changes the rounding); bf16 outputs are rounded after every op.
#include <cuda_bf16.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "kernels.h"
#include "launch.cuh"
#include "unary.cuh"

namespace rh {
namespace {

template <bool kBf16>
__device__ __forceinline__ float ApplyChain(const ChainArgs& c, float x) {
  return ApplyChainFns<kBf16>(c.fns, c.n_fn, x);
}

// The chain's T^k tables (kernel arguments, arena-resident) staged into shared memory once per
// block: n_tab x 897 x 2 bytes.
__device__ __forceinline__ void LoadRunTables(const ChainArgs& c, uint16_t* smem) {
  for (int t = 0; t < c.n_tab; ++t)
    for (int i = threadIdx.x; i < kTanhRunEntries; i += blockDim.x)
      smem[t * kTanhRunEntries + i] = c.tab[t][i];
  __syncthreads();
}

// ------------------------------------------ host -------------------------------------------

float Bf16BitsToFloat(uint32_t h) {
  uint32_t u = h << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

// Round a positive finite double to the nearest bf16 (ties to even), directly (no fp32 step).
uint16_t RneBf16(double t) {
  float f = static_cast<float>(t);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  const uint32_t lo = u & 0xffff0000u;
  uint32_t best = lo;
  double bd = 1e300;
  for (int k = -1; k <= 1; ++k) {
    const uint32_t c = lo + static_cast<uint32_t>(k) * 0x10000u;
    const double dv = std::fabs(static_cast<double>(Bf16BitsToFloat(c >> 16)) - t);
    if (dv < bd || (dv == bd && ((c >> 16) & 1u) == 0)) {
      bd = dv;
      best = c;
    }
  }
  return static_cast<uint16_t>(best >> 16);
}

// The correctly rounded bf16 tanh (the semantics of one unlabeled/tanh op on a bf16 value).
uint16_t TanhBf16(uint16_t h) {
  const uint32_t a = h & 0x7fffu, s = h & 0x8000u;
  if (a < (122u << 7) || a > 0x7f80u) return h;  // tanh(x) rounds to x below 2^-5; NaN
  if (a >= (129u << 7)) return static_cast<uint16_t>(s | 0x3f80u);  // |x| >= 4 -> +-1
  return static_cast<uint16_t>(s | RneBf16(std::tanh(static_cast<double>(Bf16BitsToFloat(a)))));
}

}  // namespace

void TanhRunTable(int k, uint16_t* out) {
  for (int i = 0; i < kTanhRunEntries; ++i) {
    uint16_t h = i < 896 ? static_cast<uint16_t>((122u << 7) + i) : static_cast<uint16_t>(129u << 7);
    for (int j = 0; j < k; ++j) h = TanhBf16(h);
    out[i] = h;
  }
}

void TanhLadderTable(const int* powers, int n, uint16_t* out) {
  for (int i = 0; i < kTanhRunEntries; ++i) {
    uint16_t h = i < 896 ? static_cast<uint16_t>((122u << 7) + i) : static_cast<uint16_t>(129u << 7);
    int done = 0;
    for (int s = 0; s < kLadderWidth; ++s) {
      if (s < n) {
        for (; done < powers[s]; ++done) h = TanhBf16(h);
        out[i * kLadderWidth + s] = h;
      } else {
        out[i * kLadderWidth + s] = 0;
      }
    }
  }
}

namespace {

// 16-byte packets: 4 fp32 or 8 bf16.
template <bool kBf16>
struct Pack {
  static constexpr int E = kBf16 ? 8 : 4;
  float v[E];
  __device__ __forceinline__ void Load(const void* p, int64_t i) {
    uint4 u = reinterpret_cast<const uint4*>(p)[i];
    if (kBf16) {
      const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&u);
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = __bfloat162float(b[e]);
    } else {
      const float* f = reinterpret_cast<const float*>(&u);
#pragma unroll
      for (int e = 0; e < E; ++e) v[e] = f[e];
    }
  }
  __device__ __forceinline__ void Store(void* p, int64_t i) const {
    uint4 u;
    if (kBf16) {
      __nv_bfloat16* b = reinterpret_cast<__nv_bfloat16*>(&u);
#pragma unroll
      for (int e = 0; e < E; ++e) b[e] = __float2bfloat16_rn(v[e]);
    } else {
      float* f = reinterpret_cast<float*>(&u);
#pragma unroll
      for (int e = 0; e < E; ++e) f[e] = v[e];
    }
    reinterpret_cast<uint4*>(p)[i] = u;
  }
};

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

// Each thread owns two 16-byte packets per iteration (16 bf16 / 8 fp32 elements) so the chain's
// dependent ops of independent elements interleave.
template <bool kBf16>
__global__ void __launch_bounds__(256) UnaryChainKernel(void* out, const void* in, int64_t n,
                                                        ChainArgs c) {
  PdlTrigger();
  constexpr int E = Pack<kBf16>::E;
  __shared__ uint16_t tab_s[kBf16 ? kMaxTanhRuns * kTanhRunEntries : 1];
  const uint16_t* tab = nullptr;
  if constexpr (kBf16) {
    LoadRunTables(c, tab_s);
    tab = tab_s;
  }
  PdlWait();  // the tables are program constants; inputs come from the previous kernel
  const int64_t nv = n / E;
  const int64_t npair = nv / 2;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npair; i += stride) {
    const uint4 u0 = reinterpret_cast<const uint4*>(in)[2 * i];
    const uint4 u1 = reinterpret_cast<const uint4*>(in)[2 * i + 1];
    if constexpr (kBf16) {
      uint32_t p[8] = {u0.x, u0.y, u0.z, u0.w, u1.x, u1.y, u1.z, u1.w};
      ApplyChainPackedBf16<8>(c.fns, c.n_fn, p, tab);
      reinterpret_cast<uint4*>(out)[2 * i] = make_uint4(p[0], p[1], p[2], p[3]);
      reinterpret_cast<uint4*>(out)[2 * i + 1] = make_uint4(p[4], p[5], p[6], p[7]);
    } else {
      float v[8] = {__uint_as_float(u0.x), __uint_as_float(u0.y), __uint_as_float(u0.z),
                    __uint_as_float(u0.w), __uint_as_float(u1.x), __uint_as_float(u1.y),
                    __uint_as_float(u1.z), __uint_as_float(u1.w)};
      ApplyChainVecF32<8>(c.fns, c.n_fn, v);
      reinterpret_cast<float4*>(out)[2 * i] = make_float4(v[0], v[1], v[2], v[3]);
      reinterpret_cast<float4*>(out)[2 * i + 1] = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
  for (int64_t i = npair * 2 * E + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
    if constexpr (kBf16) {
      uint32_t p[1] = {static_cast<uint32_t>(reinterpret_cast<const uint16_t*>(in)[i])};
      ApplyChainPackedBf16<1>(c.fns, c.n_fn, p, tab);
      reinterpret_cast<uint16_t*>(out)[i] = static_cast<uint16_t>(p[0] & 0xffffu);
    } else {
      float v[1] = {reinterpret_cast<const float*>(in)[i]};
      ApplyChainVecF32<1>(c.fns, c.n_fn, v);
      reinterpret_cast<float*>(out)[i] = v[0];
    }
  }
}

template <bool kBf16>
__global__ void __launch_bounds__(256) BinaryKernel(void* out, const void* a, const void* b,
                                                    int64_t n, bool mul, ChainArgs c) {
  PdlTrigger();
  constexpr int E = Pack<kBf16>::E;
  __shared__ uint16_t tab_s[kBf16 ? kMaxTanhRuns * kTanhRunEntries : 1];
  const uint16_t* tab = nullptr;
  if constexpr (kBf16) {
    LoadRunTables(c, tab_s);
    tab = tab_s;
  }
  PdlWait();  // the tables are program constants; inputs come from the previous kernel
  const int64_t nv = n / E;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nv; i += stride) {
    Pack<kBf16> x, y;
    x.Load(a, i);
    y.Load(b, i);
#pragma unroll
    for (int e = 0; e < E; ++e) x.v[e] = mul ? __fmul_rn(x.v[e], y.v[e]) : __fadd_rn(x.v[e], y.v[e]);
    if constexpr (kBf16) {
      uint32_t p[E / 2];
#pragma unroll
      for (int e = 0; e < E / 2; ++e) p[e] = PackBf16x2(x.v[2 * e], x.v[2 * e + 1]);
      ApplyChainPackedBf16<E / 2>(c.fns, c.n_fn, p, tab);
      reinterpret_cast<uint4*>(out)[i] = make_uint4(p[0], p[1], p[2], p[3]);
    } else {
      ApplyChainVecF32<E>(c.fns, c.n_fn, x.v);
      x.Store(out, i);
    }
  }
  for (int64_t i = nv * E + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
    float xa = LoadScalar<kBf16>(a, i), xb = LoadScalar<kBf16>(b, i);
    float r = mul ? __fmul_rn(xa, xb) : __fadd_rn(xa, xb);
    if (kBf16) r = RoundBf16(r);
    StoreScalar<kBf16>(out, i, ApplyChain<kBf16>(c, r));
  }
}

// ------------------------------- elementwise chain programs --------------------------------
// One 16-byte vector per input per thread-iteration (8 bf16 / 4 fp32 elements).  All inputs
// are loaded up front (up to kMaxEwIn x 16 B in flight per thread), then the warp-uniform
// program runs on registers; bf16 stays packed (bf16x2 add/mul round exactly like the fp32
// op + bf16 rounding: a bf16 sum or product is exact in fp32).

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

// Programs with at most 4 inputs (the rematerializing backward chains): 4 input vectors live,
// not 8 — the registers buy a third / fourth resident block per SM.
template <int N>
__device__ __forceinline__ uint4 EwPickN(const uint4 (&r)[kMaxEwIn], int k) {
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
// through every T^c unchanged, as in EwLadderKernel).
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
  constexpr uint32_t sel = (S & 1) ? 0x7632u : 0x5410u;
  const uint32_t b[4] = {base.x, base.y, base.z, base.w};
  uint32_t p[4];
#pragma unroll
  for (int q = 0; q < 4; ++q)
    p[q] = __byte_perm(U32OfRow(r[2 * q], S >> 1), U32OfRow(r[2 * q + 1], S >> 1), sel) | (b[q] & 0x80008000u);
  return make_uint4(p[0], p[1], p[2], p[3]);
}

// Operand k of the program: an input vector, or (k >= kEwSrcVirt) a ladder column of the
// rematerialization base (warp-uniform switch: static register indices).
template <bool kHalf = false>
__device__ __forceinline__ uint4 EwOperand(const uint4 (&raw)[kMaxEwIn], const uint4 (&r)[8][2], uint4 base,
                                           int k) {
  if (k < kEwSrcVirt) return EwPickN<kHalf ? 4 : kMaxEwIn>(raw, k);
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

template <bool kBf16, bool kRemat = false, bool kHalf = false>
__device__ __forceinline__ void EwRunVec(const EwArgs& a, int64_t i, const uint16_t* tabs, int pc_end,
                                         uint32_t (&acc)[4], const uint4* vlad_s = nullptr) {
  constexpr int kIn = kHalf ? 4 : kMaxEwIn;  // kHalf programs have at most 4 inputs (launcher)
  uint4 raw[kMaxEwIn];
#pragma unroll
  for (int k = 0; k < kIn; ++k)
    if (k < a.n_in) raw[k] = reinterpret_cast<const uint4*>(a.in[k])[i];
  uint4 vr[8][2];
  uint4 vbase = make_uint4(0, 0, 0, 0);
  if constexpr (kBf16 && kRemat) {
    vbase = EwPickN<kIn>(raw, a.vlad_in);
    LadderRows<kHalf>(vbase, vlad_s, vr);
  }
  uint32_t keep[4] = {0, 0, 0, 0};
#pragma unroll
  for (int e = 0; e < 4; ++e) acc[e] = 0;
  for (int pc = 0; pc < pc_end; ++pc) {
    const int ins = a.code[pc], op = ins & 0xff, arg = ins >> 8;
    switch (op) {
      case kEwLoad: {
        const uint4 v = (kRemat ? EwOperand<kHalf>(raw, vr, vbase, arg) : EwPickN<kIn>(raw, arg));
        acc[0] = v.x; acc[1] = v.y; acc[2] = v.z; acc[3] = v.w;
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
            const uint4 v = LadderColI(vr, vbase, S);
            const uint32_t y[4] = {v.x, v.y, v.z, v.w};
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
        const uint4 v = (kRemat ? EwOperand<kHalf>(raw, vr, vbase, arg) : EwPickN<kIn>(raw, arg));
        const uint32_t y[4] = {v.x, v.y, v.z, v.w};
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
          const uint4 v = (kRemat ? EwOperand<kHalf>(raw, vr, vbase, arg) : EwPickN<kIn>(raw, arg));
          w[0] = v.x; w[1] = v.y; w[2] = v.z; w[3] = v.w;
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
          float v[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) v[e] = __uint_as_float(acc[e]);
          const int32_t fn = arg;
          ApplyChainVecF32<4>(&fn, 1, v);
#pragma unroll
          for (int e = 0; e < 4; ++e) acc[e] = __float_as_uint(v[e]);
        }
    }
  }
}

// Scalar tail (n not a multiple of the vector): same semantics on unpacked values.
template <bool kBf16>
__device__ __forceinline__ float EwScalarOperand(const EwArgs& a, int64_t i, int k) {
  if (k < kEwSrcVirt) return LoadScalar<kBf16>(a.in[k], i);
  return LadderScalar(LoadScalar<kBf16>(a.in[a.vlad_in], i), a.vlad, k - kEwSrcVirt);
}

template <bool kBf16>
__device__ __forceinline__ void EwRunScalar(const EwArgs& a, int64_t i, const uint16_t* tabs) {
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

template <bool kBf16, bool kRemat, bool kHalf = false>
__global__ void __launch_bounds__(256, kHalf ? 4 : 1) EwProgKernel(const __grid_constant__ EwArgs a) {
  PdlTrigger();
  __shared__ uint16_t tab_s[kBf16 ? kMaxTanhRuns * kTanhRunEntries : 1];
  extern __shared__ uint4 vlad_s[];  // rematerialization ladder (vlad_n > 0); kHalf: half rows
  if constexpr (kBf16) {
    for (int t = 0; t < a.n_tab; ++t)
      for (int i = threadIdx.x; i < kTanhRunEntries; i += blockDim.x) tab_s[t * kTanhRunEntries + i] = a.tab[t][i];
    if (kRemat) {
      if (kHalf)
        for (int i = threadIdx.x; i < kTanhRunEntries; i += blockDim.x) vlad_s[i] = a.vlad[2 * i];
      else
        for (int i = threadIdx.x; i < kTanhRunEntries * 2; i += blockDim.x) vlad_s[i] = a.vlad[i];
    }
    __syncthreads();
  }
  PdlWait();
  constexpr int E = kBf16 ? 8 : 4;
  const int64_t nv = a.n / E;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nv; i += stride) {
    if constexpr (kRemat) {
      // few warps per SM (128 registers): L2-prefetch the next iteration's vectors so their
      // loads do not wait on HBM latency (no registers held)
      const int64_t nx = i + stride;
      if (nx < nv)
        for (int k = 0; k < a.n_in; ++k)
          asm volatile("prefetch.global.L2 [%0];" ::"l"(reinterpret_cast<const uint4*>(a.in[k]) + nx));
    }
    uint32_t acc[4];
    EwRunVec<kBf16, kRemat, kHalf>(a, i, tab_s, a.n_code, acc, vlad_s);
  }
  for (int64_t i = nv * E + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < a.n; i += stride)
    EwRunScalar<kBf16>(a, i, tab_s);
}

// bf16 chain program with a tanh ladder suffix (EwArgs::lad_*): the interpreter runs the
// prefix, then every element's lad_n outputs come from its ladder row (2 x 16-byte shared
// loads) and are re-packed per output with byte permutes: ~30 instructions per element for a
// 12-store chain instead of ~20 per op and element.  |x| < 2^-5 and NaN pass through every
// T^c unchanged; T is odd, so the sign is OR-ed back.
__device__ __forceinline__ uint32_t U32Of(const uint4 (&r)[2], int w) {
  const uint4 q = r[w >> 2];
  return (w & 3) == 0 ? q.x : (w & 3) == 1 ? q.y : (w & 3) == 2 ? q.z : q.w;
}

template <bool kRemat>
__global__ void __launch_bounds__(256, kRemat ? 1 : 2) EwLadderKernel(const __grid_constant__ EwArgs a) {
  PdlTrigger();
  extern __shared__ uint4 lad_s[];  // kTanhRunEntries rows x 2 uint4
  __shared__ uint16_t tab_s[kMaxTanhRuns * kTanhRunEntries];
  for (int t = 0; t < a.n_tab; ++t)
    for (int i = threadIdx.x; i < kTanhRunEntries; i += blockDim.x) tab_s[t * kTanhRunEntries + i] = a.tab[t][i];
  for (int i = threadIdx.x; i < kTanhRunEntries * 2; i += blockDim.x) lad_s[i] = a.lad[i];
  uint4* vlad_s = lad_s + kTanhRunEntries * 2;  // rematerialization ladder (vlad_n > 0)
  if (kRemat)
    for (int i = threadIdx.x; i < kTanhRunEntries * 2; i += blockDim.x) vlad_s[i] = a.vlad[i];
  __syncthreads();
  PdlWait();
  constexpr uint32_t kLo = 122u << 7, kSpan = 0x7f80u - (122u << 7), kLast = kTanhRunEntries - 1;
  const int64_t nv = a.n / 8;
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < nv; i += stride) {
    uint32_t acc[4];
    EwRunVec<true, kRemat>(a, i, tab_s, a.lad_pc, acc, vlad_s);
    uint4 r[8][2];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t pr = acc[e >> 1];
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
    for (int q = 0; q < 4; ++q) sg[q] = acc[q] & 0x80008000u;
#pragma unroll
    for (int s = 0; s < kLadderWidth; ++s) {
      if (s >= a.lad_n) break;
      const uint32_t sel = (s & 1) ? 0x7632u : 0x5410u;
      uint32_t p[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        p[q] = __byte_perm(U32Of(r[2 * q], s >> 1), U32Of(r[2 * q + 1], s >> 1), sel) | sg[q];
      reinterpret_cast<uint4*>(a.out[a.lad_out[s]])[i] = make_uint4(p[0], p[1], p[2], p[3]);
    }
  }
  for (int64_t i = nv * 8 + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < a.n; i += stride)
    EwRunScalar<true>(a, i, tab_s);
}

template <bool kBf16>
__global__ void __launch_bounds__(256) SoftmaxRowsKernel(void* out, const void* in, int64_t cols) {
  PdlTrigger();
  PdlWait();
  const int64_t row = blockIdx.x;
  const int64_t base = row * cols;
  __shared__ float red[32];
  float mx = -INFINITY;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x) mx = fmaxf(mx, LoadScalar<kBf16>(in, base + j));
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : -INFINITY;
    for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  mx = red[0];
  __syncthreads();
  float s = 0.0f;
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x)
    s += expf(__fsub_rn(LoadScalar<kBf16>(in, base + j), mx));
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    float v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0f;
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (threadIdx.x == 0) red[0] = v;
  }
  __syncthreads();
  s = red[0];
  for (int64_t j = threadIdx.x; j < cols; j += blockDim.x)
    StoreScalar<kBf16>(out, base + j, __fdiv_rn(expf(__fsub_rn(LoadScalar<kBf16>(in, base + j), mx)), s));
}

// Column sums: one thread per (outer, inner) column, coalesced across `inner`.
template <bool kBf16>
__global__ void __launch_bounds__(256) ReduceColsKernel(void* out, const void* in, int64_t outer,
                                                        int64_t e, int64_t inner) {
  PdlTrigger();
  PdlWait();
  const int64_t n = outer * inner;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t o = t / inner, i = t - o * inner;
    const int64_t base = o * e * inner + i;
    float s = 0.0f;
    for (int64_t c = 0; c < e; ++c) s = __fadd_rn(s, LoadScalar<kBf16>(in, base + c * inner));
    StoreScalar<kBf16>(out, t, s);
  }
}

// Row sums (inner == 1): one warp per row, shuffle tree.
template <bool kBf16>
__global__ void __launch_bounds__(256) ReduceRowsKernel(void* out, const void* in, int64_t rows,
                                                        int64_t e) {
  PdlTrigger();
  PdlWait();
  const int64_t warp = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  float s = 0.0f;
  for (int64_t c = lane; c < e; c += 32) s += LoadScalar<kBf16>(in, warp * e + c);
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) StoreScalar<kBf16>(out, warp, s);
}

// 2-D transpose [R,C] -> [C,R] through a padded shared-memory tile (coalesced both sides).
template <typename T>
__global__ void __launch_bounds__(256) Transpose2DKernel(T* out, const T* in, int64_t R, int64_t C) {
  PdlTrigger();
  PdlWait();
  __shared__ T tile[32][33];
  const int64_t r0 = blockIdx.y * 32, c0 = blockIdx.x * 32;
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int64_t r = r0 + j, c = c0 + threadIdx.x;
    if (r < R && c < C) tile[j][threadIdx.x] = in[r * C + c];
  }
  __syncthreads();
  for (int j = threadIdx.y; j < 32; j += 8) {
    const int64_t c = c0 + j, r = r0 + threadIdx.x;
    if (r < R && c < C) out[c * R + r] = tile[threadIdx.x][j];
  }
}

struct PermDev {
  int nd;
  int64_t odims[RH_MAX_RANK];
  int64_t istride_of_out[RH_MAX_RANK];
};

template <typename T>
__global__ void TransposeNDKernel(T* out, const T* in, PermDev p, int64_t n) {
  PdlTrigger();
  PdlWait();
  for (int64_t f = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; f < n;
       f += int64_t(gridDim.x) * blockDim.x) {
    int64_t t = f, src = 0;
    for (int i = p.nd - 1; i >= 0; --i) {
      const int64_t c = t % p.odims[i];
      t /= p.odims[i];
      src += c * p.istride_of_out[i];
    }
    out[f] = in[src];
  }
}

template <typename T>
__global__ void BroadcastKernel(T* out, const T* in, int64_t n_out, int64_t n_in) {
  PdlTrigger();
  PdlWait();
  for (int64_t f = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; f < n_out;
       f += int64_t(gridDim.x) * blockDim.x)
    out[f] = in[f % n_in];
}

template <typename T>
__global__ void ConcatPieceKernel(T* out, const T* in, int64_t outer, int64_t row, int64_t orow,
                                  int64_t off) {
  PdlTrigger();
  PdlWait();
  const int64_t n = outer * row;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n;
       t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t o = t / row, j = t - o * row;
    out[o * orow + off + j] = in[t];
  }
}

// All pieces of a concat in one launch: blockIdx.y = piece, 16-byte units (every piece row,
// output row and column offset a multiple of 16 bytes).
__global__ void __launch_bounds__(256) ConcatKernel(ConcatArgs a) {
  PdlTrigger();
  PdlWait();
  const int p = blockIdx.y;
  const uint32_t row = static_cast<uint32_t>(a.row16[p]);
  const uint32_t n = static_cast<uint32_t>(a.outer) * row;
  const uint4* in = static_cast<const uint4*>(a.in[p]);
  uint4* out = static_cast<uint4*>(a.out) + a.off16[p];
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
    const uint32_t o = t / row;
    out[static_cast<int64_t>(o) * a.orow16 + (t - o * row)] = in[t];
  }
}

int Blocks(int64_t n, int per_thread = 1) {
  static const int per_sm = [] {  // A/B knob (profiles/): grid cap in blocks per SM
    const char* v = getenv("RH_EW_BLOCKS_PER_SM");
    return v && *v ? atoi(v) : 16;
  }();
  return static_cast<int>(
      std::max<int64_t>(1, std::min<int64_t>((n / per_thread + 255) / 256, SmCount() * per_sm)));
}

}  // namespace

void LaunchUnaryChain(void* out, const void* in, int64_t n, const ChainArgs& c, int dtype,
                      cudaStream_t s) {
  if (n == 0) return;
  if (dtype == RH_BF16) {
    LaunchPdl(UnaryChainKernel<true>, Blocks(n, 8), 256, 0, s, out, in, n, c);
  } else {
    LaunchPdl(UnaryChainKernel<false>, Blocks(n, 4), 256, 0, s, out, in, n, c);
  }
  RH_CUDA(cudaGetLastError());
}

void LaunchSoftmaxRows(void* out, const void* in, int64_t rows, int64_t cols, int dtype,
                       cudaStream_t s) {
  if (rows == 0) return;
  if (rows > 0x7fffffff) Fail("softmax: too many rows");
  if (dtype == RH_BF16) {
    LaunchPdl(SoftmaxRowsKernel<true>, static_cast<unsigned>(rows), 256, 0, s, out, in, cols);
  } else {
    LaunchPdl(SoftmaxRowsKernel<false>, static_cast<unsigned>(rows), 256, 0, s, out, in, cols);
  }
  RH_CUDA(cudaGetLastError());
}

void LaunchEwProg(const EwArgs& a, int dtype, cudaStream_t s) {
  if (a.n == 0) return;
  constexpr int kLadSmem = kTanhRunEntries * kLadderWidth * 2;
  const int vsmem = dtype == RH_BF16 && a.vlad_n > 0 ? kLadSmem : 0;
  int dev = 0;
  RH_CUDA(cudaGetDevice(&dev));
  if (dtype == RH_BF16 && a.lad_n > 0) {
    static bool attr[64] = {};
    if (dev < 64 && !attr[dev]) {
      RH_CUDA(cudaFuncSetAttribute(EwLadderKernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kLadSmem));
      RH_CUDA(cudaFuncSetAttribute(EwLadderKernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kLadSmem));
      attr[dev] = true;
    }
    // persistent-ish grid: each block stages the 28 KB ladder table once
    const int blocks = std::min(Blocks(a.n, 8), SmCount() * 4);
    if (vsmem) LaunchPdl(EwLadderKernel<true>, blocks, 256, kLadSmem + vsmem, s, a);
    else LaunchPdl(EwLadderKernel<false>, blocks, 256, kLadSmem, s, a);
  } else if (dtype == RH_BF16 && vsmem && a.vlad_n <= 8 && a.n_in <= 4 && !getenv("RH_REMAT_FULL_ROWS")) {
    // at most 8 rematerialized powers and 4 inputs: half rows (14 KB table, one 16-byte row per
    // element) and 3 resident blocks per SM
    LaunchPdl(EwProgKernel<true, true, true>, std::min(Blocks(a.n, 8), SmCount() * 4), 256, vsmem / 2, s, a);
  } else if (dtype == RH_BF16 && vsmem) {
    static bool attr[64] = {};
    if (dev < 64 && !attr[dev]) {
      RH_CUDA(cudaFuncSetAttribute(EwProgKernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, vsmem));
      attr[dev] = true;
    }
    // the 28 KB rematerialization table is staged per block: persistent-ish grid
    LaunchPdl(EwProgKernel<true, true>, std::min(Blocks(a.n, 8), SmCount() * 2), 256, vsmem, s, a);
  } else if (dtype == RH_BF16) {
    LaunchPdl(EwProgKernel<true, false>, Blocks(a.n, 8), 256, 0, s, a);
  } else {
    LaunchPdl(EwProgKernel<false, false>, Blocks(a.n, 4), 256, 0, s, a);
  }
  RH_CUDA(cudaGetLastError());
}

void LaunchBinary(void* out, const void* a, const void* b, int64_t n, bool mul, const ChainArgs& c,
                  int dtype, cudaStream_t s) {
  if (n == 0) return;
  if (dtype == RH_BF16) {
    LaunchPdl(BinaryKernel<true>, Blocks(n, 8), 256, 0, s, out, a, b, n, mul, c);
  } else {
    LaunchPdl(BinaryKernel<false>, Blocks(n, 4), 256, 0, s, out, a, b, n, mul, c);
  }
  RH_CUDA(cudaGetLastError());
}

void LaunchReduceSum(void* out, const void* in, int64_t outer, int64_t e, int64_t inner, int dtype,
                     cudaStream_t s) {
  if (outer * inner == 0) return;
  const bool bf = dtype == RH_BF16;
  if (inner == 1) {
    const int64_t threads = outer * 32;
    const int blocks = static_cast<int>((threads + 255) / 256);
    if (bf) LaunchPdl(ReduceRowsKernel<true>, blocks, 256, 0, s, out, in, outer, e);
    else LaunchPdl(ReduceRowsKernel<false>, blocks, 256, 0, s, out, in, outer, e);
  } else {
    if (bf) LaunchPdl(ReduceColsKernel<true>, Blocks(outer * inner), 256, 0, s, out, in, outer, e, inner);
    else LaunchPdl(ReduceColsKernel<false>, Blocks(outer * inner), 256, 0, s, out, in, outer, e, inner);
  }
  RH_CUDA(cudaGetLastError());
}

void LaunchTranspose(void* out, const void* in, int nd, const int64_t* in_dims, const int* perm,
                     int dtype, cudaStream_t s) {
  int64_t n = 1;
  for (int i = 0; i < nd; ++i) n *= in_dims[i];
  if (n == 0) return;
  const bool bf = dtype == RH_BF16;
  if (nd == 2 && perm[0] == 1 && perm[1] == 0) {
    const int64_t R = in_dims[0], C = in_dims[1];
    dim3 grid(static_cast<unsigned>((C + 31) / 32), static_cast<unsigned>((R + 31) / 32));
    dim3 block(32, 8);
    if (bf) LaunchPdl(Transpose2DKernel<uint16_t>, grid, block, 0, s, static_cast<uint16_t*>(out), static_cast<const uint16_t*>(in), R, C);
    else LaunchPdl(Transpose2DKernel<uint32_t>, grid, block, 0, s, static_cast<uint32_t*>(out), static_cast<const uint32_t*>(in), R, C);
  } else {
    PermDev p{};
    p.nd = nd;
    int64_t istride[RH_MAX_RANK];
    int64_t st = 1;
    for (int i = nd - 1; i >= 0; --i) {
      istride[i] = st;
      st *= in_dims[i];
    }
    for (int i = 0; i < nd; ++i) {
      p.odims[i] = in_dims[perm[i]];
      p.istride_of_out[i] = istride[perm[i]];
    }
    if (bf) LaunchPdl(TransposeNDKernel<uint16_t>, Blocks(n), 256, 0, s, static_cast<uint16_t*>(out), static_cast<const uint16_t*>(in), p, n);
    else LaunchPdl(TransposeNDKernel<uint32_t>, Blocks(n), 256, 0, s, static_cast<uint32_t*>(out), static_cast<const uint32_t*>(in), p, n);
  }
  RH_CUDA(cudaGetLastError());
}

void LaunchBroadcast(void* out, const void* in, int64_t n_out, int64_t n_in, int dtype,
                     cudaStream_t s) {
  if (n_out == 0) return;
  if (dtype == RH_BF16) LaunchPdl(BroadcastKernel<uint16_t>, Blocks(n_out), 256, 0, s, static_cast<uint16_t*>(out), static_cast<const uint16_t*>(in), n_out, n_in);
  else LaunchPdl(BroadcastKernel<uint32_t>, Blocks(n_out), 256, 0, s, static_cast<uint32_t*>(out), static_cast<const uint32_t*>(in), n_out, n_in);
  RH_CUDA(cudaGetLastError());
}

namespace {
template <bool kBf16>
__global__ void __launch_bounds__(256) SgdKernel(void* w, const void* g, int64_t n, float lr) {
  PdlTrigger();
  PdlWait();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    if constexpr (kBf16) {
      __nv_bfloat16* wp = static_cast<__nv_bfloat16*>(w);
      const float v = __fsub_rn(__bfloat162float(wp[i]),
                                __fmul_rn(lr, __bfloat162float(static_cast<const __nv_bfloat16*>(g)[i])));
      wp[i] = __float2bfloat16_rn(v);
    } else {
      float* wp = static_cast<float*>(w);
      wp[i] = __fsub_rn(wp[i], __fmul_rn(lr, static_cast<const float*>(g)[i]));
    }
  }
}
}  // namespace

// 16-byte vectors (8 bf16 / 4 fp32 per thread and iteration): a write-back pass of the whole
// parameter set is HBM-bound.
template <bool kBf16>
__global__ void __launch_bounds__(256) SgdVecKernel(uint4* w, const uint4* g, int64_t n16, float lr) {
  PdlTrigger();
  PdlWait();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n16; i += int64_t(gridDim.x) * blockDim.x) {
    uint4 a = w[i];
    const uint4 b = g[i];
    uint32_t* x = reinterpret_cast<uint32_t*>(&a);
    const uint32_t* y = reinterpret_cast<const uint32_t*>(&b);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if constexpr (kBf16) {
        const float lo = __fsub_rn(__uint_as_float(x[k] << 16), __fmul_rn(lr, __uint_as_float(y[k] << 16)));
        const float hi = __fsub_rn(__uint_as_float(x[k] & 0xffff0000u), __fmul_rn(lr, __uint_as_float(y[k] & 0xffff0000u)));
        x[k] = PackBf16x2(lo, hi);
      } else {
        x[k] = __float_as_uint(__fsub_rn(__uint_as_float(x[k]), __fmul_rn(lr, __uint_as_float(y[k]))));
      }
    }
    w[i] = a;
  }
}

void LaunchSgd(void* w, const void* g, int64_t n, float lr, int dtype, cudaStream_t s) {
  if (n == 0) return;
  const int eb = ElemBytes(dtype);
  if ((n * eb) % 16 == 0 && (reinterpret_cast<uintptr_t>(w) | reinterpret_cast<uintptr_t>(g)) % 16 == 0) {
    const int64_t n16 = n * eb / 16;
    if (dtype == RH_BF16) LaunchPdl(SgdVecKernel<true>, Blocks(n16), 256, 0, s, static_cast<uint4*>(w), static_cast<const uint4*>(g), n16, lr);
    else LaunchPdl(SgdVecKernel<false>, Blocks(n16), 256, 0, s, static_cast<uint4*>(w), static_cast<const uint4*>(g), n16, lr);
  } else if (dtype == RH_BF16) {
    LaunchPdl(SgdKernel<true>, Blocks(n), 256, 0, s, w, g, n, lr);
  } else {
    LaunchPdl(SgdKernel<false>, Blocks(n), 256, 0, s, w, g, n, lr);
  }
  RH_CUDA(cudaGetLastError());
}

bool LaunchConcat(const ConcatArgs& a, cudaStream_t s) {
  if (a.n < 1 || a.n > kMaxConcat || a.outer == 0) return false;
  int64_t most = 0;
  for (int p = 0; p < a.n; ++p) {
    if (reinterpret_cast<uintptr_t>(a.in[p]) % 16) return false;
    most = std::max(most, a.outer * a.row16[p]);
  }
  if (reinterpret_cast<uintptr_t>(a.out) % 16 || most >= (int64_t{1} << 32)) return false;
  const int bx = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((most + 1023) / 1024, SmCount() * 8 / a.n + 1)));
  LaunchPdl(ConcatKernel, dim3(bx, a.n), 256, 0, s, a);
  RH_CUDA(cudaGetLastError());
  return true;
}

void LaunchConcatPiece(void* out, const void* in, int64_t outer, int64_t row, int64_t orow,
                       int64_t off, int dtype, cudaStream_t s) {
  if (outer * row == 0) return;
  if (dtype == RH_BF16) LaunchPdl(ConcatPieceKernel<uint16_t>, Blocks(outer * row), 256, 0, s, static_cast<uint16_t*>(out), static_cast<const uint16_t*>(in), outer, row, orow, off);
  else LaunchPdl(ConcatPieceKernel<uint32_t>, Blocks(outer * row), 256, 0, s, static_cast<uint32_t*>(out), static_cast<const uint32_t*>(in), outer, row, orow, off);
  RH_CUDA(cudaGetLastError());
}

}  // namespace rh
