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

#include "ew_core.cuh"
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
  for (int t = 0; t < c.n_tab; ++t) StageTable(smem + t * kTanhRunEntries, c.tab[t], kTanhRunEntries);
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
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  if constexpr (kBf16) {
    // four 16-byte vectors per thread in flight (vectors i + q * stride: every load instruction
    // coalesced); the persistent-ish grid otherwise keeps too few bytes in flight to cover HBM
    // latency (one C3 step's 1-lookup chain ran at 2.2 TB/s)
    int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x;
    for (; i + 3 * stride < nv; i += 4 * stride) {
      uint4 u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) u[q] = reinterpret_cast<const uint4*>(in)[i + q * stride];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t p[4] = {u[q].x, u[q].y, u[q].z, u[q].w};
        ApplyChainPackedBf16<4>(c.fns, c.n_fn, p, tab);
        reinterpret_cast<uint4*>(out)[i + q * stride] = make_uint4(p[0], p[1], p[2], p[3]);
      }
    }
    for (; i < nv; i += stride) {
      const uint4 u0 = reinterpret_cast<const uint4*>(in)[i];
      uint32_t p[4] = {u0.x, u0.y, u0.z, u0.w};
      ApplyChainPackedBf16<4>(c.fns, c.n_fn, p, tab);
      reinterpret_cast<uint4*>(out)[i] = make_uint4(p[0], p[1], p[2], p[3]);
    }
  }
  const int64_t npair = nv / 2;
  if constexpr (!kBf16) {  // fp32: two 16-byte packets per thread-iteration
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < npair; i += stride) {
      const uint4 u0 = reinterpret_cast<const uint4*>(in)[2 * i];
      const uint4 u1 = reinterpret_cast<const uint4*>(in)[2 * i + 1];
      float v[8] = {__uint_as_float(u0.x), __uint_as_float(u0.y), __uint_as_float(u0.z),
                    __uint_as_float(u0.w), __uint_as_float(u1.x), __uint_as_float(u1.y),
                    __uint_as_float(u1.z), __uint_as_float(u1.w)};
      ApplyChainVecF32<8>(c.fns, c.n_fn, v);
      reinterpret_cast<float4*>(out)[2 * i] = make_float4(v[0], v[1], v[2], v[3]);
      reinterpret_cast<float4*>(out)[2 * i + 1] = make_float4(v[4], v[5], v[6], v[7]);
    }
  }
  const int64_t done = kBf16 ? nv * E : npair * 2 * E;  // elements the vector loops covered
  for (int64_t i = done + blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += stride) {
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
// Interpreter kernels (ew_core.cuh): the program is read per vector from the kernel argument.
// Programs compiled by ew_jit.cpp run the same bodies with the instruction sequence inlined.
template <bool kBf16, bool kRemat, bool kHalf = false>
__global__ void __launch_bounds__(256, kHalf ? 4 : 1) EwProgKernel(const __grid_constant__ EwArgs a) {
  constexpr int kIn = kHalf ? 4 : kMaxEwIn;  // kHalf programs have at most 4 inputs (launcher)
  EwProgBody<kBf16, kRemat, kHalf, kIn, false>(a, EwInterp<kBf16, kRemat, kHalf, kIn>{a.n_code});
}

template <bool kRemat>
__global__ void __launch_bounds__(256, kRemat ? 1 : 2) EwLadderKernel(const __grid_constant__ EwArgs a) {
  EwLadderBody<kRemat, kMaxEwIn, false>(a, EwInterp<true, kRemat, false, kMaxEwIn>{a.lad_pc});
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
    // blocks that stage T^k tables: a persistent-ish grid, so each block's staging is amortized
    // over several iterations (16 blocks per SM did ~1 vector pair per thread after staging)
    const int blocks = c.n_tab ? std::min(Blocks(n, 16), SmCount() * 4) : Blocks(n, 8);
    LaunchPdl(UnaryChainKernel<true>, blocks, 256, 0, s, out, in, n, c);
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

int EwKindOf(const EwArgs& a, int dtype) {
  if (dtype != RH_BF16) return kEwKindF32;
  if (a.lad_n > 0) return a.vlad_n > 0 ? kEwKindLadderRemat : kEwKindLadder;
  if (a.vlad_n > 0) {
    // at most 8 rematerialized powers and 4 inputs: half rows (14 KB table, one 16-byte row per
    // element) and 4 resident blocks per SM
    static const bool full_rows = getenv("RH_REMAT_FULL_ROWS") != nullptr;
    return a.vlad_n <= 8 && a.n_in <= 4 && !full_rows ? kEwKindRematHalf : kEwKindRematFull;
  }
  return kEwKindBf16;
}

void LaunchEwProg(const EwArgs& a, int dtype, cudaStream_t s) {
  if (a.n == 0) return;
  constexpr int kLadSmem = kTanhRunEntries * kLadderWidth * 2;
  const int kind = EwKindOf(a, dtype);
  int blocks = 0;
  size_t smem = 0;
  switch (kind) {
    case kEwKindLadder:
    case kEwKindLadderRemat:  // persistent-ish grid: each block stages the 28 KB ladder table once
      blocks = std::min(Blocks(a.n, 8), SmCount() * 4);
      smem = kind == kEwKindLadderRemat ? 2 * kLadSmem : kLadSmem;
      break;
    case kEwKindRematHalf:
      blocks = std::min(Blocks(a.n, 8), SmCount() * 4);
      smem = kLadSmem / 2;
      break;
    case kEwKindRematFull:  // the 28 KB rematerialization table is staged per block
      blocks = std::min(Blocks(a.n, 8), SmCount() * 2);
      smem = kLadSmem;
      break;
    case kEwKindBf16: blocks = a.n_tab ? std::min(Blocks(a.n, 8), SmCount() * 4) : Blocks(a.n, 8); break;
    default: blocks = Blocks(a.n, 4);
  }
  if (a.jit && EwJitLaunch(a, blocks, smem, s)) return;
  int dev = 0;
  RH_CUDA(cudaGetDevice(&dev));
  static bool attr[64] = {};
  if (dev < 64 && !attr[dev]) {
    RH_CUDA(cudaFuncSetAttribute(EwLadderKernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kLadSmem));
    RH_CUDA(cudaFuncSetAttribute(EwLadderKernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * kLadSmem));
    RH_CUDA(cudaFuncSetAttribute(EwProgKernel<true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kLadSmem));
    attr[dev] = true;
  }
  switch (kind) {
    case kEwKindLadder: LaunchPdl(EwLadderKernel<false>, blocks, 256, smem, s, a); break;
    case kEwKindLadderRemat: LaunchPdl(EwLadderKernel<true>, blocks, 256, smem, s, a); break;
    case kEwKindRematHalf: LaunchPdl(EwProgKernel<true, true, true>, blocks, 256, smem, s, a); break;
    case kEwKindRematFull: LaunchPdl(EwProgKernel<true, true>, blocks, 256, smem, s, a); break;
    case kEwKindBf16: LaunchPdl(EwProgKernel<true, false>, blocks, 256, 0, s, a); break;
    default: LaunchPdl(EwProgKernel<false, false>, blocks, 256, 0, s, a);
  }
  RH_CUDA(cudaGetLastError());
}

void LaunchBinary(void* out, const void* a, const void* b, int64_t n, bool mul, const ChainArgs& c,
                  int dtype, cudaStream_t s) {
  if (n == 0) return;
  if (dtype == RH_BF16) {
    const int blocks = c.n_tab ? std::min(Blocks(n, 8), SmCount() * 4) : Blocks(n, 8);
    LaunchPdl(BinaryKernel<true>, blocks, 256, 0, s, out, a, b, n, mul, c);
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
