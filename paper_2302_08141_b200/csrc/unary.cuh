// unary.cuh — the UnaryElementwise semantics (the reference leaves `fn`
// undefined, include/parashard/ir.h:87), shared by the chain kernel and the GEMM epilogues.
//
// fp32 programs: IEEE-rounded fp32 arithmetic in the order below (explicit _rn intrinsics, no
// FMA contraction) and CUDA's accurate tanhf/expf (<= 2 ulp from glibc's).
// bf16 programs: the same formulas evaluated to ~2^-20 relative error with SFU-based code
// (FastTanh below, ex2-based __expf, rsqrtf) and the result of every op rounded to bf16 — the
// per-op rounding the oracle applies; the bf16 results then equal the oracle's correctly rounded
// ones except in rare boundary cases.
#pragma once

#ifndef __CUDACC_RTC__  // (NVRTC: ew_jit.cpp's prelude provides these)
#include <cuda_bf16.h>

#include "ew_defs.h"
#include "rhino_exec.h"
#endif

namespace rh {

// tanh for the bf16 path: relative error < 2^-20 (an odd Taylor polynomial below |x| = 1/4,
// 1 - 2 / (1 + 2^(2|x| log2 e)) with the SFU ex2 / rcp above), so rounding the result to bf16
// reproduces the correctly rounded value except within 2^-20 of a rounding boundary.  The raw
// tanh.approx.f32 (2^-11) is NOT used: its 1-ulp bf16 misroundings compound through the
// fixture's 12-36-op tanh chains and the attention GEMMs (measured: 0.3 normwise on the block).
__device__ __forceinline__ float FastTanh(float x) {
  const float ax = fabsf(x);
  if (ax < 0.25f) {
    const float x2 = x * x;
    return x * fmaf(x2, fmaf(x2, fmaf(x2, fmaf(x2, 0.021869488f, -0.053968254f), 0.13333334f),
                             -0.33333334f), 1.0f);
  }
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(ax * 2.8853900817779268f));  // 2 log2(e)
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
  return copysignf(fmaf(-2.0f, r, 1.0f), x);
}

template <bool kFast>
__device__ __forceinline__ float ApplyFn(int fn, float x) {
  switch (fn) {
    case RH_FN_RELU: return x > 0.0f ? x : 0.0f;
    case RH_FN_GELU: {
      const float x3 = __fmul_rn(__fmul_rn(x, x), x);
      const float inner = __fmul_rn(0.7978845608028654f, __fadd_rn(x, __fmul_rn(0.044715f, x3)));
      const float t = kFast ? FastTanh(inner) : tanhf(inner);
      return __fmul_rn(__fmul_rn(0.5f, x), __fadd_rn(1.0f, t));
    }
    case RH_FN_TANH: return kFast ? FastTanh(x) : tanhf(x);
    case RH_FN_EXP: return kFast ? __expf(x) : expf(x);
    case RH_FN_SIGMOID:
      return kFast ? __fdividef(1.0f, 1.0f + __expf(-x)) : __fdiv_rn(1.0f, __fadd_rn(1.0f, expf(-x)));
    case RH_FN_NEG: return -x;
    case RH_FN_RSQRT:
      return kFast ? rsqrtf(fabsf(x) + 1e-6f) : __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(fabsf(x), 1e-6f)));
    default: return x;  // identity (and unlabeled resolved to identity by the lowering)
  }
}

__device__ __forceinline__ float RoundBf16(float x) { return __bfloat162float(__float2bfloat16_rn(x)); }

// One op's stored value: bf16 programs round after every op.
template <bool kBf16>
__device__ __forceinline__ float ApplyChainFns(const int32_t* fns, int n, float x) {
  for (int i = 0; i < n; ++i) {
    x = ApplyFn<kBf16>(fns[i], x);
    if (kBf16) x = RoundBf16(x);
  }
  return x;
}

// fp32 chain over E independent elements: the (warp-uniform) fn switch sits outside the
// element loop so the E elements' dependency chains interleave (ILP E).
template <int E>
__device__ __forceinline__ void ApplyChainVecF32(const int32_t* fns, int n, float (&v)[E]) {
  for (int i = 0; i < n; ++i) {
    const int fn = fns[i];
    switch (fn) {
      case RH_FN_TANH:
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = tanhf(v[e]);
        break;
      case RH_FN_IDENTITY:
        break;
      default:
#pragma unroll
        for (int e = 0; e < E; ++e) v[e] = ApplyFn<false>(fn, v[e]);
    }
  }
}

__device__ __forceinline__ uint32_t ReluBf16x2(uint32_t x) {
  uint32_t y;
  asm("max.bf16x2 %0, %1, %2;" : "=r"(y) : "r"(x), "r"(0u));
  return y;
}
__device__ __forceinline__ uint32_t PackBf16x2(float lo, float hi) {
  uint32_t y;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(y) : "f"(hi), "f"(lo));
  return y;
}

// A run of k tanh ops on a bf16 value = one lookup in the table of T^k (T = correctly rounded
// bf16 tanh): |x| < 2^-5 is a fixed point of T (tanh(x)/x > 1 - 2^-11.6 never crosses half an
// ulp), |x| >= 4 maps like 4 (T(x) = +-1), NaN stays NaN, and the 7 binades [2^-5, 4) (896
// entries) are tabulated; T is odd.  Branch-free: the clamped slot is always read.
// One unsigned compare covers both pass-through cases: u = a - 2^-5's pattern wraps around for
// a < 2^-5 and exceeds 0x7f80 - (122 << 7) only for NaN.
__device__ __forceinline__ uint32_t TanhRunLookup(uint32_t h, const uint16_t* tab) {
  const uint32_t a = h & 0x7fffu;
  const uint32_t u = a - (122u << 7);
  const uint32_t t = tab[min(u, static_cast<uint32_t>(kTanhRunEntries - 1))];
  return (h & 0x8000u) | (u > 0x7f80u - (122u << 7) ? a : t);
}

// bf16 chain over P packed bf16x2 registers (2P elements).  tanh runs (tables in shared memory,
// `tabs` = kTanhRunEntries-strided), relu, neg, identity stay in packed bf16; other fns unpack to
// fp32, apply, and round back — every op's result is a bf16 value.
template <int P>
__device__ __forceinline__ void ApplyChainPackedBf16(const int32_t* fns, int n, uint32_t (&p)[P],
                                                     const uint16_t* tabs = nullptr) {
  for (int i = 0; i < n; ++i) {
    const int fn = fns[i];
    if (fn >= kFnTanhRun) {
      const uint16_t* tab = tabs + (fn - kFnTanhRun) * kTanhRunEntries;
#pragma unroll
      for (int e = 0; e < P; ++e)
        p[e] = TanhRunLookup(p[e] & 0xffffu, tab) | (TanhRunLookup(p[e] >> 16, tab) << 16);
      continue;
    }
    switch (fn) {
      case RH_FN_TANH:  // (runs are table-compressed by the lowering; kept for completeness)
#pragma unroll
        for (int e = 0; e < P; ++e) {
          const float lo = __uint_as_float(p[e] << 16), hi = __uint_as_float(p[e] & 0xffff0000u);
          p[e] = PackBf16x2(FastTanh(lo), FastTanh(hi));
        }
        break;
      case RH_FN_RELU:
#pragma unroll
        for (int e = 0; e < P; ++e) p[e] = ReluBf16x2(p[e]);
        break;
      case RH_FN_NEG:
#pragma unroll
        for (int e = 0; e < P; ++e) p[e] ^= 0x80008000u;
        break;
      case RH_FN_IDENTITY:
        break;
      default:
#pragma unroll
        for (int e = 0; e < P; ++e) {
          const float lo = __uint_as_float(p[e] << 16), hi = __uint_as_float(p[e] & 0xffff0000u);
          p[e] = PackBf16x2(ApplyFn<true>(fn, lo), ApplyFn<true>(fn, hi));
        }
    }
  }
}

}  // namespace rh
