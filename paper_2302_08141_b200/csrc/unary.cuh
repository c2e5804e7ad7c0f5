// unary.cuh — the UnaryElementwise semantics (the reference leaves `fn`
// undefined, include/parashard/ir.h:87), shared by the chain kernel and the GEMM epilogues.
//
// fp32 programs: IEEE-rounded fp32 arithmetic in the order below (explicit _rn intrinsics, no
// FMA contraction) and CUDA's accurate tanhf/expf (<= 2 ulp from glibc's).
// bf16 programs: the same formulas with the SFU approximations (tanh.approx.f32, ex2-based
// __expf, rsqrtf; relative error <= 2^-10.7, below half a bf16 ulp) and the result of every op
// rounded to bf16 — the per-op rounding the oracle applies.
#pragma once

#include <cuda_bf16.h>

#include "rhino_exec.h"

namespace rh {

__device__ __forceinline__ float FastTanh(float x) {
  float y;
  asm("tanh.approx.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
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

}  // namespace rh
