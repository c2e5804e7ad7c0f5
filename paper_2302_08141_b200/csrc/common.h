// common.h — errors, dtype helpers and the block-cyclic layout math shared by host and device.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "rhino_exec.h"

namespace rh {

struct Error : std::runtime_error {
  int status;
  Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

[[noreturn]] inline void Fail(const std::string& m, int status = RH_ERR_INVALID) {
  throw Error(status, m);
}

#define RH_CUDA(x)                                                                         \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess)                                                                 \
      ::rh::Fail(std::string("CUDA: ") + cudaGetErrorString(e_) + " at " + __FILE__ + ":" + \
                     std::to_string(__LINE__) + " (" #x ")",                               \
                 RH_ERR_CUDA);                                                             \
  } while (0)

inline int ElemBytes(int dtype) { return dtype == RH_BF16 ? 2 : 4; }

// SMs of the current device (148 on B200; queried once per device, so persistent grids and wave
// heuristics follow the part they run on: another SKU, a MIG slice or a green context).
inline int SmCount() {
  static int cache[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

// ---------------------------------------------------------------------------------------------
// Single-axis block-cyclic view (sharding.cpp:61-72).  Shard(dim, s) on an axis of size d over
// a tensor of `dims`: write the flat index as f = ((p * d + r) * Qs + u) with
//   P  = outer(dim) * extent/(d*s),   Qs = s * inner(dim),   u in [0, Qs),
// so rank r owns p in [0,P), u in [0,Qs) and its local buffer is l = p * Qs + u (its runs in
// ascending global order).  Replicated / Partial: l = f.
struct AxisView {
  int32_t kind;   // rh_spec_kind
  int32_t d;
  int64_t P, Qs;  // shard only
};

inline AxisView MakeAxisView(const rh_spec& s, int ndim, const int64_t* dims, int d) {
  AxisView v{s.kind, d, 0, 0};
  if (s.kind == RH_SHARD) {
    int64_t outer = 1, inner = 1;
    for (int i = 0; i < s.dim; ++i) outer *= dims[i];
    for (int i = s.dim + 1; i < ndim; ++i) inner *= dims[i];
    v.P = outer * (dims[s.dim] / (d * s.stride));
    v.Qs = s.stride * inner;
  }
  return v;
}

// ---------------------------------------------------------------------------------------------
// Composed multi-axis map (axis k acts on the shape left by axes < k, sharding.cpp:390-403):
// local flat index of one rank -> global flat index.
struct ComposedMap {
  int32_t nd;
  int32_t nshard;
  int64_t gdims[RH_MAX_RANK];
  int64_t ldims[RH_MAX_RANK];
  struct Ax {
    int32_t dim;
    int32_t d;
    int64_t stride;
    int64_t coord;
  } ax[RH_MAX_AXES];  // shard axes only, in mesh-axis order
};

__host__ __device__ inline int64_t ComposedLocalToGlobal(const ComposedMap& m, int64_t l) {
  int64_t c[RH_MAX_RANK];
  for (int k = m.nd - 1; k >= 0; --k) {
    c[k] = l % m.ldims[k];
    l /= m.ldims[k];
  }
  for (int a = m.nshard - 1; a >= 0; --a) {
    const auto& x = m.ax[a];
    int64_t lc = c[x.dim];
    c[x.dim] = (lc / x.stride) * x.stride * x.d + x.coord * x.stride + lc % x.stride;
  }
  int64_t f = 0;
  for (int k = 0; k < m.nd; ++k) f = f * m.gdims[k] + c[k];
  return f;
}

}  // namespace rh
