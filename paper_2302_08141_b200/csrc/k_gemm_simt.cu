// k_gemm_simt.cu — CUDA-core GEMM (FFMA, fp32 accumulation) for any shape and any of the four
// transpose layouts of a rank-2 MatMul (proj/src/ir.cpp:121-137).  It is the reference kernel the
// tcgen05 path is tested against and the path for shapes the tensor-core kernel does not tile.
#include <cuda_bf16.h>

#include <algorithm>

#include "kernels.h"
#include "launch.cuh"
#include "unary.cuh"

namespace rh {
namespace {

constexpr int BM = 128, BN = 128, BK = 8;

template <typename T>
__device__ __forceinline__ float Ld(const T* p, int64_t i);
template <>
__device__ __forceinline__ float Ld<float>(const float* p, int64_t i) {
  return p[i];
}
template <>
__device__ __forceinline__ float Ld<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}

// Split-K (blockIdx.z = split): small-M GEMMs (the MLP configs' [64,1024] activations) have too
// few 128x128 tiles to fill 148 SMs; each split writes its fp32 partial tile to `ws` and a reduce
// kernel sums the splits in order, then rounds and applies the epilogue chain.
// Epilogue chain on one value; bf16 tanh runs are T^k table lookups (global tables, the
// executor's run compression, kernels.h kFnTanhRun), every other op as in ApplyChainFns.
template <typename T>
__device__ __forceinline__ float EpiChain(const ChainArgs& epi, float v) {
  if constexpr (sizeof(T) == 2) {
    for (int i = 0; i < epi.n_fn; ++i) {
      const int fn = epi.fns[i];
      if (fn >= kFnTanhRun) {
        const uint32_t h = TanhRunLookup(__float_as_uint(v) >> 16, epi.tab[fn - kFnTanhRun]);
        v = __uint_as_float(h << 16);
      } else {
        v = RoundBf16(ApplyFn<true>(fn, v));
      }
    }
    return v;
  } else {
    return ApplyChainFns<false>(epi.fns, epi.n_fn, v);
  }
}

template <typename T, bool TA, bool TB>
__global__ void __launch_bounds__(256) GemmSimtKernel(T* __restrict__ C, const T* __restrict__ A,
                                                      const T* __restrict__ B, int64_t M,
                                                      int64_t N, int64_t K, ChainArgs epi,
                                                      int64_t kchunk, float* __restrict__ ws,
                                                      const T* __restrict__ resid) {
  PdlTrigger();
  PdlWait();
  __shared__ __align__(16) float As[BK][BM];
  __shared__ __align__(16) float Bs[BK][BN];
  const int tid = threadIdx.x;
  const int tx = tid % 16, ty = tid / 16;
  const int64_t m0 = int64_t(blockIdx.y) * BM, n0 = int64_t(blockIdx.x) * BN;
  const int64_t kbeg = int64_t(blockIdx.z) * kchunk;
  const int64_t kend = min(K, kbeg + kchunk);
  float acc[8][8];
#pragma unroll
  for (int i = 0; i < 8; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[i][j] = 0.0f;

  for (int64_t k0 = kbeg; k0 < kend; k0 += BK) {
    // A tile -> As[k][m]
    if (!TA) {  // A [M,K]: 4 consecutive k per thread
      const int r = tid / 2, kc = (tid % 2) * 4;
      const int64_t gm = m0 + r;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t gk = k0 + kc + j;
        As[kc + j][r] = (gm < M && gk < kend) ? Ld<T>(A, gm * K + gk) : 0.0f;
      }
    } else {  // A stored [K,M]: 4 consecutive m per thread
      const int kr = tid / 32, mc = (tid % 32) * 4;
      const int64_t gk = k0 + kr;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t gm = m0 + mc + j;
        As[kr][mc + j] = (gm < M && gk < kend) ? Ld<T>(A, gk * M + gm) : 0.0f;
      }
    }
    if (!TB) {  // B [K,N]: 4 consecutive n per thread
      const int kr = tid / 32, nc = (tid % 32) * 4;
      const int64_t gk = k0 + kr;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t gn = n0 + nc + j;
        Bs[kr][nc + j] = (gn < N && gk < kend) ? Ld<T>(B, gk * N + gn) : 0.0f;
      }
    } else {  // B stored [N,K]: 4 consecutive k per thread
      const int r = tid / 2, kc = (tid % 2) * 4;
      const int64_t gn = n0 + r;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int64_t gk = k0 + kc + j;
        Bs[kc + j][r] = (gn < N && gk < kend) ? Ld<T>(B, gn * K + gk) : 0.0f;
      }
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float a[8], b[8];
      const float4 a0 = *reinterpret_cast<const float4*>(&As[kk][ty * 4]);
      const float4 a1 = *reinterpret_cast<const float4*>(&As[kk][64 + ty * 4]);
      const float4 b0 = *reinterpret_cast<const float4*>(&Bs[kk][tx * 4]);
      const float4 b1 = *reinterpret_cast<const float4*>(&Bs[kk][64 + tx * 4]);
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      b[0] = b0.x; b[1] = b0.y; b[2] = b0.z; b[3] = b0.w;
      b[4] = b1.x; b[5] = b1.y; b[6] = b1.z; b[7] = b1.w;
#pragma unroll
      for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int64_t gm = m0 + (i < 4 ? ty * 4 + i : 64 + ty * 4 + (i - 4));
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const int64_t gn = n0 + (j < 4 ? tx * 4 + j : 64 + tx * 4 + (j - 4));
      if (gn >= N) continue;
      float v = acc[i][j];
      if (ws) {  // split-K partial
        ws[(int64_t(blockIdx.z) * M + gm) * N + gn] = v;
        continue;
      }
      if constexpr (sizeof(T) == 2) v = RoundBf16(v);
      v = EpiChain<T>(epi, v);
      if (resid) v = __fadd_rn(v, Ld<T>(resid, gm * N + gn));  // fused add (rounded below)
      if constexpr (sizeof(T) == 2) {
        C[gm * N + gn] = __float2bfloat16_rn(v);
      } else {
        C[gm * N + gn] = v;
      }
    }
  }
}

template <typename T>
__global__ void __launch_bounds__(256) SplitReduceKernel(T* __restrict__ C, const float* __restrict__ ws,
                                                         int64_t n, int splits, ChainArgs epi,
                                                         const T* __restrict__ resid) {
  PdlTrigger();
  PdlWait();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    float v = ws[i];
    for (int z = 1; z < splits; ++z) v = __fadd_rn(v, ws[int64_t(z) * n + i]);
    if constexpr (sizeof(T) == 2) v = RoundBf16(v);
    v = EpiChain<T>(epi, v);
    if (resid) v = __fadd_rn(v, Ld<T>(resid, i));  // fused add (rounded below)
    if constexpr (sizeof(T) == 2) {
      C[i] = __float2bfloat16_rn(v);
    } else {
      C[i] = v;
    }
  }
}

int SplitsFor(const GemmArgs& g) {
  const int64_t tiles = ((g.m + BM - 1) / BM) * ((g.n + BN - 1) / BN);
  if (tiles >= SmCount() || g.k < 128) return 1;
  int64_t splits = (296 + tiles - 1) / tiles;
  splits = std::min<int64_t>(splits, std::min<int64_t>(g.k / 64, 32));
  return static_cast<int>(std::max<int64_t>(splits, 1));
}

template <typename T>
int Dispatch(const GemmArgs& g, cudaStream_t s) {
  const int splits = g.scratch ? SplitsFor(g) : 1;
  const int64_t kchunk = ((g.k + splits - 1) / splits + BK - 1) / BK * BK;
  const int z = static_cast<int>((g.k + kchunk - 1) / kchunk);
  float* ws = z > 1 ? static_cast<float*>(g.scratch) : nullptr;
  dim3 grid(static_cast<unsigned>((g.n + BN - 1) / BN), static_cast<unsigned>((g.m + BM - 1) / BM),
            static_cast<unsigned>(z));
  T* c = static_cast<T*>(g.c);
  const T* a = static_cast<const T*>(g.a);
  const T* b = static_cast<const T*>(g.b);
  const T* rs = static_cast<const T*>(g.resid);
  if (!g.ta && !g.tb) LaunchPdl(GemmSimtKernel<T, false, false>, grid, 256, 0, s, c, a, b, g.m, g.n, g.k, g.epi, kchunk, ws, rs);
  else if (!g.ta && g.tb) LaunchPdl(GemmSimtKernel<T, false, true>, grid, 256, 0, s, c, a, b, g.m, g.n, g.k, g.epi, kchunk, ws, rs);
  else if (g.ta && !g.tb) LaunchPdl(GemmSimtKernel<T, true, false>, grid, 256, 0, s, c, a, b, g.m, g.n, g.k, g.epi, kchunk, ws, rs);
  else LaunchPdl(GemmSimtKernel<T, true, true>, grid, 256, 0, s, c, a, b, g.m, g.n, g.k, g.epi, kchunk, ws, rs);
  if (!ws) return 1;
  const int64_t n = g.m * g.n;
  const int blocks = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, SmCount() * 8)));
  LaunchPdl(SplitReduceKernel<T>, blocks, 256, 0, s, c, ws, n, z, g.epi, rs);
  return 2;
}

__global__ void __launch_bounds__(256) ZeroWordsKernel(uint32_t* p, int64_t n) {
  PdlTrigger();
  PdlWait();
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
    p[i] = 0;
}

}  // namespace

size_t GemmSimtScratchBytes(const GemmArgs& g) {
  const int splits = SplitsFor(g);
  return splits > 1 ? static_cast<size_t>(splits) * g.m * g.n * 4 : 0;
}

int LaunchGemmSimt(const GemmArgs& g, cudaStream_t s) {
  if (g.m == 0 || g.n == 0) return 0;
  if (g.k == 0) {  // empty contraction: C = 0 (a kernel, not a memset node: PDL edges link kernels)
    const int64_t words = g.m * g.n * ElemBytes(g.dtype) / 4;
    LaunchPdl(ZeroWordsKernel, static_cast<int>(std::max<int64_t>(1, std::min<int64_t>((words + 255) / 256, SmCount() * 8))),
              256, 0, s, static_cast<uint32_t*>(g.c), words);
    return 1;
  }
  if (g.m / BM >= 65535) Fail("gemm: M too large for the SIMT grid");
  const int launches = g.dtype == RH_BF16 ? Dispatch<__nv_bfloat16>(g, s) : Dispatch<float>(g, s);
  RH_CUDA(cudaGetLastError());
  return launches;
}

}  // namespace rh
