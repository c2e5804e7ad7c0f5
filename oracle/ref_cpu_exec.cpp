// ref_cpu_exec.cpp — CPU oracle (TEST INFRASTRUCTURE ONLY; see ref_cpu_exec.h for the rules
// on who may load it and for the reference files each part restates).
//
// Storage: every tensor value is kept as fp32 on the host; for bf16 programs every op output is
// rounded to bf16 (round-to-nearest-even) so the fp32 copy holds exactly the bf16 value.
#include "ref_cpu_exec.h"

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace {

thread_local std::string g_err;

struct OxError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
[[noreturn]] void Fail(const std::string& m) { throw OxError(m); }

using Dims = std::vector<int64_t>;
using Specs = std::vector<rh_spec>;  // one per mesh axis

int64_t Prod(const Dims& d) {
  int64_t n = 1;
  for (int64_t x : d) n *= x;
  return n;
}
int64_t Inner(const Dims& d, int dim) {  // TensorShape::inner_size (ir.h:51-55)
  int64_t n = 1;
  for (size_t i = dim + 1; i < d.size(); ++i) n *= d[i];
  return n;
}
bool SpecEq(const rh_spec& a, const rh_spec& b) {
  if (a.kind != b.kind) return false;
  if (a.kind != RH_SHARD) return true;
  return a.dim == b.dim && a.stride == b.stride;
}
bool SpecsEq(const Specs& a, const Specs& b) {
  for (size_t i = 0; i < a.size(); ++i)
    if (!SpecEq(a[i], b[i])) return false;
  return true;
}
std::string SpecStr(const rh_spec& s) {
  if (s.kind == RH_REPLICATED) return "replicated";
  if (s.kind == RH_PARTIAL) return "partial";
  return "shard(" + std::to_string(s.dim) + "," + std::to_string(s.stride) + ")";
}
rh_spec Rep() { return rh_spec{RH_REPLICATED, -1, 0}; }
rh_spec Par() { return rh_spec{RH_PARTIAL, -1, 0}; }
rh_spec Sh(int dim, int64_t s) { return rh_spec{RH_SHARD, dim, s}; }

// SpecValidForShape (sharding.cpp:47-53)
bool Valid(const rh_spec& s, const Dims& d, int n) {
  if (s.kind != RH_SHARD) return true;
  if (s.dim < 0 || s.dim >= static_cast<int>(d.size()) || s.stride < 1) return false;
  return d[s.dim] % (n * s.stride) == 0;
}

float Bf16Round(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x7fffffu)) {
    u = (u | 0x00400000u) & 0xffff0000u;  // quiet NaN
  } else {
    u += 0x7fffu + ((u >> 16) & 1u);
    u &= 0xffff0000u;
  }
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

// ---------------------------------------------------------------------------------------------
// Layout: Shard(dim, s) on an axis of size d deals runs of s coordinates round-robin
// (owner r = (c/s) % d, OwnerOfFlatIndex sharding.cpp:67-72); the rank's local buffer holds its
// runs in ascending global order: l = (c/(s*d))*s + c%s, inverse c = (l/s)*s*d + r*s + l%s.
// Axis k acts on the local shape left by axes < k (EffectiveShapes, sharding.cpp:390-403).

struct Mesh {
  std::vector<int> dims;
  int world() const {
    int w = 1;
    for (int x : dims) w *= x;
    return w;
  }
  std::vector<int> Coords(int rank) const {
    std::vector<int> c(dims.size());
    for (int a = static_cast<int>(dims.size()) - 1; a >= 0; --a) {
      c[a] = rank % dims[a];
      rank /= dims[a];
    }
    return c;
  }
};

Dims LocalDims(const Dims& g, const Specs& specs, const Mesh& m) {
  Dims l = g;
  for (size_t a = 0; a < specs.size(); ++a) {
    if (specs[a].kind == RH_SHARD) l[specs[a].dim] /= m.dims[a];
  }
  return l;
}

// Precomputed local->global flat map for one rank (int64 per local element).
std::vector<int64_t> LocalToGlobal(const Dims& g, const Specs& specs, const Mesh& m, int rank) {
  const Dims l = LocalDims(g, specs, m);
  const int nd = static_cast<int>(g.size());
  const int64_t n = Prod(l);
  std::vector<int> rc = m.Coords(rank);
  std::vector<int64_t> out(n);
  // Shapes after each axis, to unshard in reverse axis order.
  std::vector<Dims> after(specs.size() + 1);
  after[0] = g;
  for (size_t a = 0; a < specs.size(); ++a) {
    after[a + 1] = after[a];
    if (specs[a].kind == RH_SHARD) after[a + 1][specs[a].dim] /= m.dims[a];
  }
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    int64_t c[RH_MAX_RANK];
    int64_t t = i;
    for (int k = nd - 1; k >= 0; --k) {
      c[k] = t % l[k];
      t /= l[k];
    }
    for (int a = static_cast<int>(specs.size()) - 1; a >= 0; --a) {
      const rh_spec& s = specs[a];
      if (s.kind != RH_SHARD) continue;
      int64_t lc = c[s.dim];
      c[s.dim] = (lc / s.stride) * s.stride * m.dims[a] + rc[a] * s.stride + lc % s.stride;
    }
    int64_t f = 0;
    for (int k = 0; k < nd; ++k) f = f * g[k] + c[k];
    out[i] = f;
  }
  return out;
}

// Global value of a tensor held per rank under `specs`.  Replicated axes read coordinate 0;
// Partial axes are summed in ascending rank order in fp32.
std::vector<float> Assemble(const Dims& g, const Specs& specs, const Mesh& m,
                            const std::vector<std::vector<float>>& locals, bool bf16) {
  std::vector<float> full(Prod(g), 0.0f);
  bool any_partial = false;
  for (auto& s : specs) any_partial |= s.kind == RH_PARTIAL;
  for (int rank = 0; rank < m.world(); ++rank) {
    std::vector<int> rc = m.Coords(rank);
    bool skip = false, first = true;
    for (size_t a = 0; a < specs.size(); ++a) {
      if (specs[a].kind == RH_REPLICATED && rc[a] != 0) skip = true;
      if (specs[a].kind == RH_PARTIAL && rc[a] != 0) first = false;
    }
    if (skip) continue;
    auto map = LocalToGlobal(g, specs, m, rank);
    const auto& loc = locals[rank];
    const int64_t n = static_cast<int64_t>(map.size());
    if (first) {
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) full[map[i]] = loc[i];
    } else {
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) full[map[i]] += loc[i];
    }
  }
  if (any_partial && bf16) {
    for (auto& v : full) v = Bf16Round(v);
  }
  return full;
}

// Per-rank buffers of a global value under `specs`; Partial axes keep the value on
// coordinate 0 and zero-fill the others (sharding.cpp:132-135).
std::vector<std::vector<float>> Distribute(const Dims& g, const Specs& specs, const Mesh& m,
                                           const std::vector<float>& full) {
  std::vector<std::vector<float>> out(m.world());
  for (int rank = 0; rank < m.world(); ++rank) {
    std::vector<int> rc = m.Coords(rank);
    bool zero = false;
    for (size_t a = 0; a < specs.size(); ++a)
      if (specs[a].kind == RH_PARTIAL && rc[a] != 0) zero = true;
    auto map = LocalToGlobal(g, specs, m, rank);
    auto& loc = out[rank];
    loc.resize(map.size());
    const int64_t n = static_cast<int64_t>(map.size());
    if (zero) {
      std::fill(loc.begin(), loc.end(), 0.0f);
    } else {
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < n; ++i) loc[i] = full[map[i]];
    }
  }
  return out;
}

// ---------------------------------------------------------------------------------------------
// Philox4x32-10 and the synthetic-value contract.

void Philox(const uint32_t ctr_in[4], const uint32_t key_in[2], uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0;
    uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
    uint32_t hi0 = static_cast<uint32_t>(p0 >> 32), lo0 = static_cast<uint32_t>(p0);
    uint32_t hi1 = static_cast<uint32_t>(p1 >> 32), lo1 = static_cast<uint32_t>(p1);
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0;
  out[1] = c1;
  out[2] = c2;
  out[3] = c3;
}

float SynthValue(uint64_t seed, uint32_t op_index, uint64_t flat, float scale) {
  uint32_t key[2] = {static_cast<uint32_t>(seed), op_index};
  uint64_t blk = flat >> 2;
  uint32_t ctr[4] = {static_cast<uint32_t>(blk), static_cast<uint32_t>(blk >> 32),
                     static_cast<uint32_t>(seed >> 32), 0u};
  uint32_t o[4];
  Philox(ctr, key, o);
  uint32_t w = o[flat & 3];
  float v = static_cast<float>(static_cast<int32_t>(w >> 8) - 8388608) * (1.0f / 8388608.0f);
  return v * scale;
}

float ParamScale(int64_t fan_in) {
  return static_cast<float>(std::sqrt(3.0 / static_cast<double>(fan_in)));
}

// ---------------------------------------------------------------------------------------------
// Program.

struct Op {
  rh_op raw{};
  std::vector<int> inputs;
  std::vector<Specs> in_specs;  // [slot][axis]
  Specs out_spec;               // [axis]
  Dims dims;
  bool bf16 = false;
};

}  // namespace

struct ox_program {
  std::vector<Op> ops;
  std::vector<int> outputs;
  Mesh mesh;
  uint32_t flags = 0;
  std::vector<int> order;
  std::vector<std::vector<float>> source;  // full values of sources
  std::vector<std::vector<float>> unpart;  // [op] full result
  std::vector<std::vector<std::vector<float>>> part;  // [op][rank]
  double flops = 0;
};

namespace {

// -------------------------------- local kernels (on local shapes) -----------------------------

void Round(std::vector<float>& v, bool bf16) {
  if (!bf16) return;
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < static_cast<int64_t>(v.size()); ++i) v[i] = Bf16Round(v[i]);
}

// GEMM accumulation type: fp32 (default; what a CPU executor would run) or fp64 (flag 0x200,
// the high-accuracy reference used to state the GPU path's forward error).
thread_local bool g_gemm_f64 = false;

template <typename Acc>
void GemmBlocked(const float* pa, const float* pb, float* C, int64_t m, int64_t n, int64_t k) {
  const int64_t NB = 512;
#pragma omp parallel for schedule(dynamic, 1) collapse(2)
  for (int64_t i0 = 0; i0 < m; i0 += 4) {
    for (int64_t j0 = 0; j0 < n; j0 += NB) {
      const int64_t i1 = std::min(i0 + 4, m), j1 = std::min(j0 + NB, n);
      Acc acc[4][512];
      for (int64_t i = i0; i < i1; ++i)
        for (int64_t j = j0; j < j1; ++j) acc[i - i0][j - j0] = 0;
      for (int64_t kk = 0; kk < k; ++kk) {
        const float* brow = pb + kk * n + j0;
        for (int64_t i = i0; i < i1; ++i) {
          const Acc a = pa[i * k + kk];
          Acc* ar = acc[i - i0];
#pragma omp simd
          for (int64_t j = 0; j < j1 - j0; ++j) ar[j] += a * static_cast<Acc>(brow[j]);
        }
      }
      for (int64_t i = i0; i < i1; ++i)
        for (int64_t j = j0; j < j1; ++j) C[i * n + j] = static_cast<float>(acc[i - i0][j - j0]);
    }
  }
}

// C[m,n] = op(A)[m,k] . op(B)[k,n], accumulation in ascending k.
std::vector<float> MatMul(const std::vector<float>& A, const Dims& ad, bool ta,
                          const std::vector<float>& B, const Dims& bd, bool tb, Dims* cd) {
  const int64_t m = ta ? ad[1] : ad[0], k = ta ? ad[0] : ad[1];
  const int64_t n = tb ? bd[0] : bd[1];
  if ((tb ? bd[1] : bd[0]) != k) Fail("matmul: local contracted extents disagree");
  std::vector<float> a2, b2;
  const float* pa = A.data();
  const float* pb = B.data();
  if (ta) {  // materialize op(A) as [m,k]
    a2.resize(m * k);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; ++i)
      for (int64_t j = 0; j < k; ++j) a2[i * k + j] = A[j * m + i];
    pa = a2.data();
  }
  if (tb) {  // materialize op(B) as [k,n]
    b2.resize(k * n);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < k; ++i)
      for (int64_t j = 0; j < n; ++j) b2[i * n + j] = B[j * k + i];
    pb = b2.data();
  }
  std::vector<float> C(m * n, 0.0f);
  if (g_gemm_f64) {
    GemmBlocked<double>(pa, pb, C.data(), m, n, k);
  } else {
    GemmBlocked<float>(pa, pb, C.data(), m, n, k);
  }
  *cd = {m, n};
  return C;
}

float Unary(int fn, float x) {
  switch (fn) {
    case RH_FN_RELU: return x > 0.0f ? x : 0.0f;
    case RH_FN_GELU: {
      // 0.5 x (1 + tanh(sqrt(2/pi) (x + 0.044715 x^3))), evaluated in this exact order.
      float x3 = (x * x) * x;
      float inner = 0.7978845608028654f * (x + 0.044715f * x3);
      return (0.5f * x) * (1.0f + std::tanh(inner));
    }
    case RH_FN_TANH: return std::tanh(x);
    case RH_FN_EXP: return std::exp(x);
    case RH_FN_SIGMOID: return 1.0f / (1.0f + std::exp(-x));
    case RH_FN_NEG: return -x;
    case RH_FN_RSQRT: return 1.0f / std::sqrt(std::fabs(x) + 1e-6f);
    case RH_FN_IDENTITY: return x;
  }
  Fail("unary: bad fn " + std::to_string(fn));
}

// bf16 programs: each unary op is the correctly rounded bf16 result of the exact function
// (evaluated in fp64, rounded once from fp64 to bf16 with ties to even).
double UnaryD(int fn, double x) {
  switch (fn) {
    case RH_FN_RELU: return x > 0.0 ? x : 0.0;
    case RH_FN_GELU: return 0.5 * x * (1.0 + std::tanh(0.7978845608028654 * (x + 0.044715 * x * x * x)));
    case RH_FN_TANH: return std::tanh(x);
    case RH_FN_EXP: return std::exp(x);
    case RH_FN_SIGMOID: return 1.0 / (1.0 + std::exp(-x));
    case RH_FN_NEG: return -x;
    case RH_FN_RSQRT: return 1.0 / std::sqrt(std::fabs(x) + 1e-6);
    case RH_FN_IDENTITY: return x;
  }
  Fail("unary: bad fn " + std::to_string(fn));
}

float Bf16FromDouble(double t) {
  if (!std::isfinite(t) || t == 0.0) return Bf16Round(static_cast<float>(t));
  const bool neg = t < 0;
  const double a = neg ? -t : t;
  const float f = static_cast<float>(a);
  uint32_t u;
  std::memcpy(&u, &f, 4);
  const uint32_t lo = u & 0xffff0000u;
  uint32_t best = lo;
  double bd = 1e300;
  for (int k = -1; k <= 1; ++k) {
    const uint32_t c = lo + static_cast<uint32_t>(k) * 0x10000u;
    float cf;
    std::memcpy(&cf, &c, 4);
    const double dv = std::fabs(static_cast<double>(cf) - a);
    if (dv < bd || (dv == bd && ((c >> 16) & 1u) == 0)) {
      bd = dv;
      best = c;
    }
  }
  float r;
  std::memcpy(&r, &best, 4);
  return neg ? -r : r;
}

std::vector<float> UnaryOp(int fn, const std::vector<float>& in, const Dims& ld, bool bf16) {
  std::vector<float> out(in.size());
  if (bf16 && fn != RH_FN_SOFTMAX) {
    const int64_t n = static_cast<int64_t>(in.size());
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = Bf16FromDouble(UnaryD(fn, static_cast<double>(in[i])));
    return out;
  }
  const int64_t n = static_cast<int64_t>(in.size());
  if (fn == RH_FN_SOFTMAX) {
    const int64_t cols = ld.back(), rows = n / cols;
#pragma omp parallel for schedule(static)
    for (int64_t r = 0; r < rows; ++r) {
      const float* x = in.data() + r * cols;
      float* y = out.data() + r * cols;
      float mx = -INFINITY;
      for (int64_t j = 0; j < cols; ++j) mx = std::max(mx, x[j]);
      float s = 0.0f;
      for (int64_t j = 0; j < cols; ++j) {
        y[j] = std::exp(x[j] - mx);
        s += y[j];
      }
      for (int64_t j = 0; j < cols; ++j) y[j] = y[j] / s;
    }
  } else {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = Unary(fn, in[i]);
  }
  Round(out, bf16);
  return out;
}

std::vector<float> Transpose(const std::vector<float>& in, const Dims& id, const std::vector<int>& perm,
                             Dims* od) {
  const int nd = static_cast<int>(id.size());
  Dims o(nd);
  for (int i = 0; i < nd; ++i) o[i] = id[perm[i]];
  std::vector<int64_t> istride(nd);
  int64_t s = 1;
  for (int i = nd - 1; i >= 0; --i) {
    istride[i] = s;
    s *= id[i];
  }
  std::vector<float> out(in.size());
  const int64_t n = static_cast<int64_t>(in.size());
#pragma omp parallel for schedule(static)
  for (int64_t f = 0; f < n; ++f) {
    int64_t t = f, src = 0;
    for (int i = nd - 1; i >= 0; --i) {
      int64_t c = t % o[i];
      t /= o[i];
      src += c * istride[perm[i]];
    }
    out[f] = in[src];
  }
  *od = o;
  return out;
}

std::vector<float> ReduceSum(const std::vector<float>& in, const Dims& id, int axis, bool bf16,
                             Dims* od) {
  const int64_t outer = Prod(Dims(id.begin(), id.begin() + axis));
  const int64_t e = id[axis], inner = Inner(id, axis);
  std::vector<float> out(outer * inner);
#pragma omp parallel for schedule(static)
  for (int64_t o = 0; o < outer; ++o)
    for (int64_t i = 0; i < inner; ++i) {
      float s = 0.0f;
      for (int64_t c = 0; c < e; ++c) s += in[(o * e + c) * inner + i];
      out[o * inner + i] = s;
    }
  Dims o = id;
  o.erase(o.begin() + axis);
  *od = o;
  Round(out, bf16);
  return out;
}

// ---------------------------------- per-op natural specs (A.3) -------------------------------

std::vector<int> EffPerm(const Op& op, int rank) {
  std::vector<int> p(rank);
  for (int i = 0; i < rank; ++i) p[i] = op.raw.has_perm ? op.raw.perm[i] : rank - 1 - i;
  return p;
}

// ReshapePassthrough (sharding.cpp:144-160).
bool Passthrough(const Dims& in, const Dims& out, const rh_spec& s, int d, rh_spec* res) {
  if (s.kind == RH_REPLICATED) {
    *res = s;
    return true;
  }
  if (s.kind == RH_PARTIAL || !Valid(s, in, d)) return false;
  const int64_t run = Inner(in, s.dim) * s.stride;
  for (int dim = 0; dim < static_cast<int>(out.size()); ++dim) {
    int64_t inner = Inner(out, dim);
    if (run % inner != 0) continue;
    rh_spec c = Sh(dim, run / inner);
    if (Valid(c, out, d)) {
      *res = c;
      return true;
    }
  }
  return false;
}

// Output spec on one axis that the local computation of `op` produces when its inputs arrive
// in `in` (one spec per slot) — the local-op table of FollowInput/ProduceOutput
// (sharding.cpp:225-388).  `in_dims` are the per-slot shapes on this axis, `out_dims` the
// output's.
rh_spec Natural(const Op& op, const std::vector<rh_spec>& in, const std::vector<Dims>& in_dims,
                const Dims& out_dims, int d, const rh_spec& planned) {
  auto bad = [&]() -> rh_spec {
    std::string m = "op kind " + std::to_string(op.raw.kind) + ": no local rule for inputs";
    for (auto& s : in) m += " " + SpecStr(s);
    Fail(m);
  };
  bool all_rep = true;
  for (auto& s : in) all_rep &= s.kind == RH_REPLICATED;
  // ProduceOutput, Broadcast with want.dim < off (sharding.cpp:360-367): a replicated input and
  // an output sharded on a broadcast (leading) dim — each rank holds its rows of the broadcast
  if (all_rep && op.raw.kind == RH_OP_BROADCAST && planned.kind == RH_SHARD && !in_dims.empty() &&
      planned.dim < static_cast<int>(out_dims.size() - in_dims[0].size()) &&
      out_dims[planned.dim] % (static_cast<int64_t>(d) * planned.stride) == 0)
    return planned;
  if (all_rep) return Rep();
  // P + P -> P (local accumulation of partial sums; the executor's LocalAccumulate extension)
  if (op.raw.kind == RH_OP_ADD && in.size() == 2 && in[0].kind == RH_PARTIAL && in[1].kind == RH_PARTIAL) return Par();
  for (auto& s : in)
    if (s.kind == RH_PARTIAL) bad();
  switch (op.raw.kind) {
    case RH_OP_MATMUL: {
      const int a_m = op.raw.transpose_a ? 1 : 0, a_k = 1 - a_m;
      const int b_k = op.raw.transpose_b ? 1 : 0, b_n = 1 - b_k;
      const rh_spec &A = in[0], &B = in[1];
      if (A.kind == RH_SHARD && A.dim == a_m && B.kind == RH_REPLICATED) return Sh(0, A.stride);
      if (A.kind == RH_REPLICATED && B.kind == RH_SHARD && B.dim == b_n) return Sh(1, B.stride);
      if (A.kind == RH_SHARD && B.kind == RH_SHARD && A.dim == a_k && B.dim == b_k &&
          A.stride == B.stride)
        return Par();
      return bad();
    }
    case RH_OP_ADD:
    case RH_OP_MUL:
      if (SpecEq(in[0], in[1])) return in[0];
      return bad();
    case RH_OP_UNARY:
      if (op.raw.fn == RH_FN_SOFTMAX && in[0].dim == static_cast<int>(out_dims.size()) - 1) {
        Fail("softmax over a sharded last dim is not a local op");
      }
      return in[0];
    case RH_OP_RESHAPE: {
      rh_spec r;
      if (!Passthrough(in_dims[0], out_dims, in[0], d, &r)) Fail("reshape: no pass-through");
      return r;
    }
    case RH_OP_TRANSPOSE: {
      auto perm = EffPerm(op, static_cast<int>(in_dims[0].size()));
      for (size_t p = 0; p < perm.size(); ++p)
        if (perm[p] == in[0].dim) return Sh(static_cast<int>(p), in[0].stride);
      return bad();
    }
    case RH_OP_REDUCE_SUM:
      if (in[0].dim == op.raw.axis) return Par();
      return Sh(in[0].dim - (in[0].dim > op.raw.axis ? 1 : 0), in[0].stride);
    case RH_OP_BROADCAST:
      return Sh(in[0].dim + static_cast<int>(out_dims.size() - in_dims[0].size()), in[0].stride);
    case RH_OP_CONCAT:
      for (auto& s : in)
        if (!SpecEq(s, in[0]) || s.dim == op.raw.axis) bad();
      return in[0];
  }
  return bad();
}

// ------------------------------------------ execution ----------------------------------------

struct Exec {
  ox_program* p;
  Mesh mesh;   // mesh used for this run (unpartitioned: no axes)
  bool partitioned;
  // tensors: per op, per spec-vector key: per-rank locals
  std::vector<std::map<std::string, std::vector<std::vector<float>>>> cache;

  std::string Key(const Specs& s) {
    std::string k;
    for (auto& x : s) k += SpecStr(x) + ";";
    return k;
  }

  Specs OutSpecs(int i) { return partitioned ? p->ops[i].out_spec : Specs(); }
  Specs InSpecs(int i, int slot) { return partitioned ? p->ops[i].in_specs[slot] : Specs(); }

  // Producer `src` in spec vector `want`: assemble the global value, re-slice.
  const std::vector<std::vector<float>>& Get(int src, const Specs& want) {
    auto& c = cache[src];
    std::string k = Key(want);
    auto it = c.find(k);
    if (it != c.end()) return it->second;
    const Op& op = p->ops[src];
    const Specs have = OutSpecs(src);
    auto hit = c.find(Key(have));
    if (hit == c.end()) Fail("oracle: producer not computed");
    for (size_t a = 0; a < want.size(); ++a)
      if (!Valid(want[a], LocalDims(op.dims, Specs(want.begin(), want.begin() + a), mesh),
                 mesh.dims[a]))
        Fail("oracle: invalid demanded spec " + SpecStr(want[a]));
    auto full = Assemble(op.dims, have, mesh, hit->second, op.bf16);
    c[k] = Distribute(op.dims, want, mesh, full);
    return c[k];
  }

  void RunOp(int i) {
    const Op& op = p->ops[i];
    const int world = mesh.world();
    const Specs out = OutSpecs(i);
    if (op.raw.kind == RH_OP_PARAMETER || op.raw.kind == RH_OP_INPUT) {
      cache[i][Key(out)] = Distribute(op.dims, out, mesh, p->source[i]);
      return;
    }
    const int nin = static_cast<int>(op.inputs.size());
    std::vector<const std::vector<std::vector<float>>*> ins(nin);
    std::vector<Specs> ispecs(nin);
    for (int s = 0; s < nin; ++s) {
      ispecs[s] = InSpecs(i, s);
      ins[s] = &Get(op.inputs[s], ispecs[s]);
    }
    // Natural output spec per axis, composed over axes.
    Specs nat(out.size());
    for (size_t a = 0; a < out.size(); ++a) {
      std::vector<rh_spec> in_a(nin);
      std::vector<Dims> in_d(nin);
      for (int s = 0; s < nin; ++s) {
        in_a[s] = ispecs[s][a];
        in_d[s] = LocalDims(p->ops[op.inputs[s]].dims,
                            Specs(ispecs[s].begin(), ispecs[s].begin() + a), mesh);
      }
      Dims od = LocalDims(op.dims, Specs(nat.begin(), nat.begin() + a), mesh);
      nat[a] = Natural(op, in_a, in_d, od, mesh.dims[a], out[a]);
    }
    std::vector<std::vector<float>> res(world);
    for (int r = 0; r < world; ++r) {
      std::vector<Dims> ld(nin);
      for (int s = 0; s < nin; ++s) ld[s] = LocalDims(p->ops[op.inputs[s]].dims, ispecs[s], mesh);
      const Dims want = LocalDims(op.dims, nat, mesh);
      Dims got;
      std::vector<float> y;
      const auto& x0 = (*ins[0])[r];
      switch (op.raw.kind) {
        case RH_OP_MATMUL:
          y = MatMul(x0, ld[0], op.raw.transpose_a, (*ins[1])[r], ld[1], op.raw.transpose_b, &got);
          Round(y, op.bf16);
          if (r == 0) p->flops += 2.0 * got[0] * got[1] * (op.raw.transpose_a ? ld[0][0] : ld[0][1]);
          break;
        case RH_OP_ADD:
        case RH_OP_MUL: {
          const auto& x1 = (*ins[1])[r];
          y.resize(x0.size());
          const bool mul = op.raw.kind == RH_OP_MUL;
#pragma omp parallel for schedule(static)
          for (int64_t e = 0; e < static_cast<int64_t>(y.size()); ++e)
            y[e] = mul ? x0[e] * x1[e] : x0[e] + x1[e];
          Round(y, op.bf16);
          got = ld[0];
          break;
        }
        case RH_OP_UNARY: {
          int fn = op.raw.fn;
          if (fn == RH_FN_UNLABELED)
            fn = (p->flags & RH_FLAG_UNLABELED_IDENTITY) ? RH_FN_IDENTITY : RH_FN_TANH;
          y = UnaryOp(fn, x0, ld[0], op.bf16);
          got = ld[0];
          break;
        }
        case RH_OP_RESHAPE:
          y = x0;
          got = want;
          break;
        case RH_OP_TRANSPOSE:
          y = Transpose(x0, ld[0], EffPerm(op, static_cast<int>(ld[0].size())), &got);
          break;
        case RH_OP_REDUCE_SUM:
          y = ReduceSum(x0, ld[0], op.raw.axis, op.bf16, &got);
          break;
        case RH_OP_BROADCAST: {
          const int64_t inner = static_cast<int64_t>(x0.size());
          y.resize(Prod(want));
          for (int64_t e = 0; e < static_cast<int64_t>(y.size()); ++e) y[e] = x0[e % inner];
          got = want;
          break;
        }
        case RH_OP_CONCAT: {
          const int ax = op.raw.axis;
          const int64_t outer = Prod(Dims(want.begin(), want.begin() + ax));
          y.resize(Prod(want));
          int64_t off = 0;
          const int64_t orow = want[ax] * Inner(want, ax);
          for (int s = 0; s < nin; ++s) {
            const int64_t row = ld[s][ax] * Inner(ld[s], ax);
            const auto& xs = (*ins[s])[r];
            for (int64_t o = 0; o < outer; ++o)
              std::memcpy(&y[o * orow + off], &xs[o * row], row * sizeof(float));
            off += row;
          }
          got = want;
          break;
        }
        default:
          Fail("oracle: unknown op kind");
      }
      if (got != want) Fail("oracle: local shape mismatch for op kind " + std::to_string(op.raw.kind));
      res[r] = std::move(y);
    }
    if (SpecsEq(nat, out)) {
      cache[i][Key(out)] = std::move(res);
    } else {  // pinned op with no rule: computed replicated, realise the pin by slicing
      cache[i][Key(nat)] = std::move(res);
      auto full = Assemble(op.dims, nat, mesh, cache[i][Key(nat)], op.bf16);
      cache[i][Key(out)] = Distribute(op.dims, out, mesh, full);
    }
  }

  void Run() {
    g_gemm_f64 = (p->flags & 0x200u) != 0;
    cache.assign(p->ops.size(), {});
    p->flops = 0;
    const bool keep = (p->flags & 0x100u) != 0;
    std::vector<int> remaining(p->ops.size(), 0);
    for (auto& op : p->ops)
      for (int s : op.inputs) ++remaining[s];
    std::vector<bool> is_out(p->ops.size(), false);
    for (int o : p->outputs) is_out[o] = true;
    for (int i : p->order) {
      RunOp(i);
      if (keep) continue;
      for (int s : p->ops[i].inputs) {
        if (--remaining[s] == 0 && !is_out[s]) cache[s].clear();
      }
    }
    if (partitioned) {
      p->part.assign(p->ops.size(), {});
      for (size_t i = 0; i < p->ops.size(); ++i) {
        auto it = cache[i].find(Key(p->ops[i].out_spec));
        if (it != cache[i].end()) p->part[i] = std::move(it->second);
      }
    } else {
      p->unpart.assign(p->ops.size(), {});
      for (size_t i = 0; i < p->ops.size(); ++i) {
        auto it = cache[i].find(Key(Specs()));
        if (it != cache[i].end()) p->unpart[i] = std::move(it->second[0]);
      }
    }
  }
};

template <typename F>
int Guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return -1;
  }
}

void ToDtype(const std::vector<float>& v, bool bf16, void* dst) {
  if (!bf16) {
    std::memcpy(dst, v.data(), v.size() * 4);
    return;
  }
  auto* o = static_cast<uint16_t*>(dst);
  for (size_t i = 0; i < v.size(); ++i) o[i] = ox_f32_to_bf16(v[i]);
}
std::vector<float> FromDtype(const void* src, size_t n, bool bf16) {
  std::vector<float> v(n);
  if (!bf16) {
    std::memcpy(v.data(), src, n * 4);
  } else {
    auto* s = static_cast<const uint16_t*>(src);
    for (size_t i = 0; i < n; ++i) v[i] = ox_bf16_to_f32(s[i]);
  }
  return v;
}

}  // namespace

extern "C" {

const char* ox_last_error(void) { return g_err.c_str(); }

void ox_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]) {
  Philox(ctr, key, out);
}

float ox_synthetic_value(uint64_t seed, uint32_t op_index, uint64_t flat, int is_param,
                         int64_t fan_in) {
  return SynthValue(seed, op_index, flat, is_param ? ParamScale(fan_in) : 1.0f);
}

uint16_t ox_f32_to_bf16(float x) {
  float r = Bf16Round(x);
  uint32_t u;
  std::memcpy(&u, &r, 4);
  return static_cast<uint16_t>(u >> 16);
}
float ox_bf16_to_f32(uint16_t x) {
  uint32_t u = static_cast<uint32_t>(x) << 16;
  float f;
  std::memcpy(&f, &u, 4);
  return f;
}

int64_t ox_owner_of_flat(int ndim, const int64_t* dims, rh_spec spec, int d, int64_t flat) {
  if (spec.kind != RH_SHARD) return -1;
  Dims g(dims, dims + ndim);
  int64_t c = (flat / Inner(g, spec.dim)) % g[spec.dim];
  return (c / spec.stride) % d;
}

int64_t ox_local_of_flat(int ndim, const int64_t* dims, rh_spec spec, int d, int64_t flat) {
  Dims g(dims, dims + ndim);
  if (spec.kind != RH_SHARD) return flat;
  const int64_t inner = Inner(g, spec.dim), e = g[spec.dim];
  const int64_t o = flat / (inner * e), c = (flat / inner) % e, i = flat % inner;
  const int64_t l = (c / (spec.stride * d)) * spec.stride + c % spec.stride;
  return (o * (e / d) + l) * inner + i;
}

int ox_reshard(int d, int ndim, const int64_t* dims, rh_spec from, rh_spec to, int dtype,
               const void* const* src, void* const* dst) {
  return Guard([&] {
    Dims g(dims, dims + ndim);
    Mesh m;
    m.dims = {d};
    if (!Valid(from, g, d) || !Valid(to, g, d)) Fail("ox_reshard: spec invalid for shape");
    const bool bf16 = dtype == RH_BF16;
    const size_t nloc = static_cast<size_t>(Prod(LocalDims(g, {from}, m)));
    std::vector<std::vector<float>> locals(d);
    for (int r = 0; r < d; ++r) locals[r] = FromDtype(src[r], nloc, bf16);
    auto full = Assemble(g, {from}, m, locals, bf16);
    auto out = Distribute(g, {to}, m, full);
    for (int r = 0; r < d; ++r) ToDtype(out[r], bf16, dst[r]);
  });
}

int ox_load(const rh_op* ops, int n_ops, const int* outputs, int n_out, int n_axes,
            const int* mesh, uint32_t flags, ox_program** out) {
  return Guard([&] {
    auto p = std::make_unique<ox_program>();
    p->mesh.dims.assign(mesh, mesh + n_axes);
    p->flags = flags;
    p->outputs.assign(outputs, outputs + n_out);
    p->ops.resize(n_ops);
    for (int i = 0; i < n_ops; ++i) {
      Op& op = p->ops[i];
      op.raw = ops[i];
      op.dims.assign(ops[i].dims, ops[i].dims + ops[i].rank);
      op.bf16 = ops[i].dtype == RH_BF16;
      op.inputs.assign(ops[i].inputs, ops[i].inputs + ops[i].n_in);
      op.out_spec.assign(ops[i].out_spec, ops[i].out_spec + n_axes);
      op.in_specs.assign(ops[i].n_in, Specs(n_axes));
      for (int a = 0; a < n_axes; ++a)
        for (int s = 0; s < ops[i].n_in; ++s) op.in_specs[s][a] = ops[i].in_specs[a * ops[i].n_in + s];
      op.raw.inputs = nullptr;
      op.raw.in_specs = nullptr;
      for (int s : op.inputs)
        if (s < 0 || s >= n_ops) Fail("ox_load: bad input index");
    }
    // Kahn order (any topological order computes the same values; ops are pure).
    std::vector<int> indeg(n_ops, 0);
    std::vector<std::vector<int>> cons(n_ops);
    for (int i = 0; i < n_ops; ++i)
      for (int s : p->ops[i].inputs) {
        ++indeg[i];
        cons[s].push_back(i);
      }
    std::vector<int> q;
    for (int i = 0; i < n_ops; ++i)
      if (!indeg[i]) q.push_back(i);
    for (size_t h = 0; h < q.size(); ++h)
      for (int c : cons[q[h]])
        if (--indeg[c] == 0) q.push_back(c);
    if (static_cast<int>(q.size()) != n_ops) Fail("ox_load: program has a cycle");
    p->order = q;
    p->source.resize(n_ops);
    *out = p.release();
  });
}

void ox_destroy(ox_program* p) { delete p; }

int ox_init_synthetic(ox_program* p, uint64_t seed) {
  return Guard([&] {
    for (size_t i = 0; i < p->ops.size(); ++i) {
      const Op& op = p->ops[i];
      if (op.raw.kind != RH_OP_PARAMETER && op.raw.kind != RH_OP_INPUT) continue;
      const float scale = op.raw.kind == RH_OP_PARAMETER ? ParamScale(op.dims[0]) : 1.0f;
      auto& v = p->source[i];
      v.resize(Prod(op.dims));
      const int64_t n = static_cast<int64_t>(v.size());
#pragma omp parallel for schedule(static)
      for (int64_t f = 0; f < n; ++f)
        v[f] = SynthValue(seed, static_cast<uint32_t>(i), static_cast<uint64_t>(f), scale);
      Round(v, op.bf16);
    }
  });
}

int ox_set_full(ox_program* p, int op, const void* src, size_t bytes) {
  return Guard([&] {
    const Op& o = p->ops.at(op);
    const size_t n = static_cast<size_t>(Prod(o.dims));
    if (bytes != n * (o.bf16 ? 2 : 4)) Fail("ox_set_full: size mismatch");
    p->source[op] = FromDtype(src, n, o.bf16);
  });
}

int ox_run_unpartitioned(ox_program* p, int threads) {
  return Guard([&] {
    if (threads > 0) omp_set_num_threads(threads);
    Exec e{p, Mesh{}, false, {}};
    e.Run();
  });
}

int ox_run_partitioned(ox_program* p, int threads) {
  return Guard([&] {
    if (threads > 0) omp_set_num_threads(threads);
    Exec e{p, p->mesh, true, {}};
    e.Run();
  });
}

int ox_read_full(ox_program* p, int op, int which, void* dst, size_t bytes) {
  return Guard([&] {
    const Op& o = p->ops.at(op);
    const size_t n = static_cast<size_t>(Prod(o.dims));
    if (bytes != n * (o.bf16 ? 2 : 4)) Fail("ox_read_full: size mismatch");
    if (which == 0) {
      if (p->unpart.empty() || p->unpart[op].empty()) Fail("ox_read_full: op not retained");
      ToDtype(p->unpart[op], o.bf16, dst);
    } else {
      if (p->part.empty() || p->part[op].empty()) Fail("ox_read_full: op not retained");
      ToDtype(Assemble(o.dims, o.out_spec, p->mesh, p->part[op], o.bf16), o.bf16, dst);
    }
  });
}

int ox_read_local(ox_program* p, int op, int rank, void* dst, size_t bytes) {
  return Guard([&] {
    const Op& o = p->ops.at(op);
    if (p->part.empty() || p->part[op].empty()) Fail("ox_read_local: op not retained");
    const auto& v = p->part[op].at(rank);
    if (bytes != v.size() * (o.bf16 ? 2 : 4)) Fail("ox_read_local: size mismatch");
    ToDtype(v, o.bf16, dst);
  });
}

int ox_local_bytes(ox_program* p, int op, size_t* bytes) {
  return Guard([&] {
    const Op& o = p->ops.at(op);
    *bytes = static_cast<size_t>(Prod(LocalDims(o.dims, o.out_spec, p->mesh))) * (o.bf16 ? 2 : 4);
  });
}

double ox_last_flops(ox_program* p) { return p->flops; }

}  // extern "C"
