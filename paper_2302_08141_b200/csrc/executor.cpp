// executor.cpp — lowering a partitioned program (rh_op records) into a static schedule of
// sm_100a kernels and resharding transitions, and running it.
//
// Semantics followed (reference files):
//   local-op rules          proj/src/sharding.cpp:225-388 (FollowInput / ProduceOutput)
//   pin fallback            proj/src/sharding.cpp:477-487 (compute replicated, then slice)
//   transitions             proj/src/sharding.cpp:104-142 (reshard_cost's collective table)
//   axis composition        proj/src/sharding.cpp:390-403 (EffectiveShapes)
//   reshape pass-through    proj/src/sharding.cpp:144-160 (metadata only: buffers alias)
//   per-edge transitions    proj/src/spmd.cpp:1033-1045 (CollectStrategyStats' edge loop)
#include "executor.h"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <sstream>

using rh::Fail;
using rh::Step;
using rh::Tensor;

std::vector<int> rh_mesh::Coords(int rank) const {
  std::vector<int> c(dims.size());
  for (int a = static_cast<int>(dims.size()) - 1; a >= 0; --a) {
    c[a] = rank % dims[a];
    rank /= dims[a];
  }
  return c;
}

std::vector<int> rh_mesh::Group(int axis, int rank) const {
  std::vector<int> c = Coords(rank);
  std::vector<int> out;
  for (int k = 0; k < dims[axis]; ++k) {
    c[axis] = k;
    int r = 0;
    for (size_t a = 0; a < dims.size(); ++a) r = r * dims[a] + c[a];
    out.push_back(r);
  }
  return out;
}

int rh_program::LocalIndex(int global_rank) const {
  int li = global_rank - mesh->rt->first_rank;
  if (li < 0 || li >= mesh->rt->n_local()) Fail("rank " + std::to_string(global_rank) + " is not local");
  return li;
}

namespace rh {
namespace {

int64_t Prod(const Dims& d) {
  int64_t n = 1;
  for (auto x : d) n *= x;
  return n;
}
int64_t Inner(const Dims& d, int dim) {
  int64_t n = 1;
  for (size_t i = dim + 1; i < d.size(); ++i) n *= d[i];
  return n;
}
bool SpecEq(const rh_spec& a, const rh_spec& b) {
  if (a.kind != b.kind) return false;
  return a.kind != RH_SHARD || (a.dim == b.dim && a.stride == b.stride);
}
bool SpecsEq(const Specs& a, const Specs& b) {
  for (size_t i = 0; i < a.size(); ++i)
    if (!SpecEq(a[i], b[i])) return false;
  return true;
}
std::string SpecStr(const rh_spec& s) {
  if (s.kind == RH_REPLICATED) return "R";
  if (s.kind == RH_PARTIAL) return "P";
  return "S(" + std::to_string(s.dim) + "," + std::to_string(s.stride) + ")";
}
std::string SpecsStr(const Specs& s) {
  std::string k;
  for (size_t i = 0; i < s.size(); ++i) k += (i ? "," : "") + SpecStr(s[i]);
  return k;
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

Dims LocalDims(const Dims& g, const Specs& specs, const std::vector<int>& mesh, size_t upto) {
  Dims l = g;
  for (size_t a = 0; a < upto && a < specs.size(); ++a)
    if (specs[a].kind == RH_SHARD) l[specs[a].dim] /= mesh[a];
  return l;
}

bool Passthrough(const Dims& in, const Dims& out, const rh_spec& s, int d, rh_spec* res) {
  if (s.kind == RH_REPLICATED) {
    *res = s;
    return true;
  }
  if (s.kind == RH_PARTIAL || !Valid(s, in, d)) return false;
  const int64_t run = Inner(in, s.dim) * s.stride;
  for (int dim = 0; dim < static_cast<int>(out.size()); ++dim) {
    const int64_t inner = Inner(out, dim);
    if (run % inner != 0) continue;
    rh_spec c = Sh(dim, run / inner);
    if (Valid(c, out, d)) {
      *res = c;
      return true;
    }
  }
  return false;
}

std::vector<int> EffPerm(const rh_op& op, int rank) {
  std::vector<int> p(rank);
  for (int i = 0; i < rank; ++i) p[i] = op.has_perm ? op.perm[i] : rank - 1 - i;
  return p;
}

const char* KindName(int k) {
  static const char* names[] = {"param", "input", "matmul", "add", "mul", "unary",
                                "reshape", "transpose", "reduce_sum", "broadcast", "concat"};
  return (k >= 0 && k <= 10) ? names[k] : "?";
}

// The output spec (one mesh axis) the local computation produces from the given input specs.
// `planned`: the op's planned output spec on this axis — it decides the one rule whose output is
// not a function of the inputs: ProduceOutput's Broadcast R -> Shard(y < off) (sharding.cpp:
// 360-367), where every rank writes only its own rows of the broadcast.
rh_spec Natural(const rh_op& op, const std::vector<rh_spec>& in, const std::vector<Dims>& in_dims,
                const Dims& out_dims, int d, const rh_spec& planned) {
  auto bad = [&]() -> rh_spec {
    std::string m = std::string("no local rule for ") + KindName(op.kind) + " with inputs";
    for (auto& s : in) m += " " + SpecStr(s);
    Fail(m);
  };
  bool all_rep = true;
  for (auto& s : in) all_rep = all_rep && s.kind == RH_REPLICATED;
  if (all_rep && op.kind == RH_OP_BROADCAST && planned.kind == RH_SHARD && !in_dims.empty() &&
      planned.dim < static_cast<int>(out_dims.size() - in_dims[0].size()) && Valid(planned, out_dims, d))
    return planned;
  if (all_rep) return Rep();
  // Accumulating partial sums (P + P -> P: the sum of per-rank addends is linear): the local
  // gradient accumulation of a microbatched step (LocalAccumulate, taskgraph.cpp:149-160) adds
  // unreduced data-parallel gradients and reduces once.  Not in the reference's rule table
  // (ProduceOutput never yields Partial from an add, sharding.cpp:313-329): executor extension.
  if (op.kind == RH_OP_ADD && in.size() == 2 && in[0].kind == RH_PARTIAL && in[1].kind == RH_PARTIAL) return Par();
  for (auto& s : in)
    if (s.kind == RH_PARTIAL) bad();
  switch (op.kind) {
    case RH_OP_MATMUL: {  // MatMulLayout (sharding.cpp:202-212) + rules :277-292, :376-384
      const int a_m = op.transpose_a ? 1 : 0, a_k = 1 - a_m;
      const int b_k = op.transpose_b ? 1 : 0, b_n = 1 - b_k;
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
      if (op.fn == RH_FN_SOFTMAX && in[0].dim == static_cast<int>(out_dims.size()) - 1)
        Fail("softmax over a sharded last dim is not executable as a local op");
      return in[0];
    case RH_OP_RESHAPE: {
      rh_spec r;
      if (!Passthrough(in_dims[0], out_dims, in[0], d, &r)) Fail("reshape without a pass-through spec");
      return r;
    }
    case RH_OP_TRANSPOSE: {
      auto perm = EffPerm(op, static_cast<int>(in_dims[0].size()));
      for (size_t p = 0; p < perm.size(); ++p)
        if (perm[p] == in[0].dim) return Sh(static_cast<int>(p), in[0].stride);
      return bad();
    }
    case RH_OP_REDUCE_SUM:
      if (in[0].dim == op.axis) return Par();
      return Sh(in[0].dim - (in[0].dim > op.axis ? 1 : 0), in[0].stride);
    case RH_OP_BROADCAST:
      return Sh(in[0].dim + static_cast<int>(out_dims.size() - in_dims[0].size()), in[0].stride);
    case RH_OP_CONCAT:
      for (auto& s : in)
        if (!SpecEq(s, in[0]) || s.dim == op.axis) bad();
      return in[0];
    default:
      return bad();
  }
}

// Grid cap of side-stream (overlapped) pull kernels; RH_SIDE_BLOCKS overrides (tuning).
int SideBlocks() {
  static const int n = [] {
    const char* e = std::getenv("RH_SIDE_BLOCKS");
    return e ? std::max(1, std::atoi(e)) : SmCount() * 2;
  }();
  return n;
}

// Reshard wire bytes of one single-axis transition (sharding.cpp:113-135).
double WireBytes(const rh_spec& from, const rh_spec& to, double S, int d) {
  const double frac = static_cast<double>(d - 1) / d;
  if (from.kind == RH_PARTIAL) return to.kind == RH_REPLICATED ? 2.0 * frac * S : frac * S;
  if (from.kind == RH_SHARD) {
    if (to.kind == RH_SHARD) return S / d * frac;
    return frac * S;
  }
  return 0.0;
}

const char* CollectiveName(const rh_spec& from, const rh_spec& to) {
  if (from.kind == RH_PARTIAL) return to.kind == RH_REPLICATED ? "all_reduce" : "reduce_scatter";
  if (from.kind == RH_SHARD) return to.kind == RH_SHARD ? "all_to_all" : "all_gather";
  return to.kind == RH_PARTIAL ? "zero_fill" : "slice";
}

ncclDataType_t NcclType(int dtype) { return dtype == RH_BF16 ? ncclBfloat16 : ncclFloat32; }

#define RH_NCCL(x)                                                                        \
  do {                                                                                    \
    ncclResult_t r_ = (x);                                                                \
    if (r_ != ncclSuccess)                                                                \
      ::rh::Fail(std::string("NCCL: ") + ncclGetErrorString(r_) + " (" #x ")", RH_ERR_NCCL); \
  } while (0)

struct EwPlan {
  std::vector<int> members;                   // chain ops in order (members[0] = head)
  std::vector<std::vector<int>> src;          // per member, per operand: -1 acc, kEwSrcKeep,
                                              // kEwSrcAcc (second use of acc), k = inputs[k]
  std::vector<std::pair<int, Specs>> inputs;  // external operands (producer, demanded specs)
  std::vector<bool> keep_after, stored;
};

// Fine-grained single-axis transitions (runs under 64 bytes on a side, LaunchFine): which
// kernel(s) move the data with 16-byte vectors on every global access.  a / b: source / target
// run lengths Qs (elements; the whole tensor for Replicated / Partial).  For a transition
// between block-cyclic layouts the pieces are:
//   a % (d*b) == 0: rank k's elements for rank r are runs of b in k's buffer (k side) and runs
//                   of a/d in r's buffer (r side);
//   b % (d*a) == 0: runs of b/d on the k side, runs of a on the r side.
// Coarse k side -> pull (plain, or interleave if the r side is fine); fine k side, coarse r side
// -> push (de-interleave straight into the peers' destinations); both fine -> two phases:
// de-interleave into the peers' staging streams, then interleave locally.
struct FinePlan {
  int mode = 0;  // 0 plain pull, 1 push, 2 pull-interleave, 3 two-phase, 4 partial two-phase,
                 // 5 local slice (Replicated source)
  int64_t u1 = 0, u2 = 0;  // unit elements: de-interleave (phase 1), interleave (phase 2)
  int64_t run = 0;         // strided-side run for push / pull-interleave (0: linear offsets)
};

FinePlan ClassifyFine(const AxisView& f, const AxisView& t, int eb, int d, int64_t n) {
  FinePlan p;
  if (d < 2) return p;
  const int64_t tel = 64 / eb, E = 16 / eb;
  auto pow2 = [](int64_t x) { return x > 0 && (x & (x - 1)) == 0; };
  auto ok = [&](int64_t u, int64_t n_contig) {
    return pow2(u) && u * eb <= 32 && FineSupported(d, static_cast<int>(u * eb), eb, n_contig);
  };
  const int64_t ns = f.kind == RH_SHARD ? n / d : n, nt = t.kind == RH_SHARD ? n / d : n;
  if (f.kind == RH_SHARD && t.kind == RH_SHARD) {
    const int64_t a = f.Qs, b = t.Qs;
    if (a >= tel && b >= tel) return p;
    if (a % (d * b) == 0) {
      if (b >= tel) return p;  // coarse k side: plain pull
      if (a / d >= tel) {
        if (ok(b, ns) && a % (d * std::max(E, b)) == 0) p = {1, b, 0, a};
      } else if (ok(b, ns) && ok(a / d, nt)) {
        p = {3, b, a / d, 0};
      }
      return p;
    }
    if (b % (d * a) == 0) {
      if (b / d >= tel) {
        if (a < tel && ok(a, nt) && b % (d * std::max(E, a)) == 0) p = {2, 0, a, b};
      } else if (ok(b / d, ns) && ok(a, nt)) {
        p = {3, b / d, a, 0};
      }
    }
    return p;
  }
  if (f.kind == RH_PARTIAL && t.kind == RH_SHARD && t.Qs < tel && ok(t.Qs, n)) return {4, t.Qs, 0, 0};
  if (f.kind == RH_REPLICATED && t.kind == RH_SHARD && t.Qs < tel && ok(t.Qs, n)) return {5, t.Qs, 0, 0};
  if (f.kind == RH_SHARD && t.kind == RH_REPLICATED && f.Qs < tel && ok(f.Qs, n)) return {2, 0, f.Qs, 0};
  return p;
}

// The fused-barrier arguments of flag row `slot` for local rank li's group on `axis` (the pull
// kernels' PeerSync, also used by the GEMM output push and its post-barrier).
PeerSync SyncOf(const rh_program* P, int axis, int slot, int li) {
  PeerSync y{};
  if (slot < 0) return y;
  const int g = P->mesh->rt->first_rank + li;
  const std::vector<int> members = P->mesh->Group(axis, g);
  const size_t row = P->sync_off + static_cast<size_t>(slot) * P->mesh->rt->world * 4;
  y.d = static_cast<int>(members.size());
  y.me = g;
  for (size_t k = 0; k < members.size(); ++k) {
    y.members[k] = members[k];
    y.peer_slot[k] = reinterpret_cast<uint32_t*>(P->peer_base[members[k]] + row);
  }
  y.my_slot = reinterpret_cast<uint32_t*>(P->peer_base[g] + row);
  y.epoch = reinterpret_cast<const uint32_t*>(P->peer_base[g] + P->epoch_off);
  y.err = reinterpret_cast<uint32_t*>(P->peer_base[g] + P->err_off);
  y.timeout_ns = SyncTimeoutNs();
  return y;
}

// A GEMM step's output push (GemmPush), filled in when the output's materialization is fused
// into it (TryPushMaterialize), after the step was emitted.
struct PushPlan {
  int dst_t = -1;  // the replicated copy every member's kernel writes into
  int axis = 0, slot = -1;
  int64_t rows_local = 0;
  // reduce-scatter form (TryPushReduceScatter): partial tiles go to their owner's staging
  int scatter_dim = -1;
  int64_t part = 0;
  size_t stage_off = 0, slot_bytes = 0;
};

class Lowerer {
 public:
  explicit Lowerer(rh_program* p) : p_(p), mesh_(p->mesh->dims), rt_(p->mesh->rt) {}

  void Lower() {
    const int n = static_cast<int>(p_->ops.size());
    p_->out_tensor.assign(n, -1);
    p_->mat_tensor.assign(n, -1);
    p_->in_tensor.assign(n, {});
    // flags + barrier counter live at the front of the arena
    p_->flags_off = Alloc(static_cast<size_t>(rt_->world) * 4);
    p_->counter_off = Alloc(4);
    p_->err_off = Alloc(4);
    if (rt_->dist && rt_->world > 1) {  // rh_program_run_host's overlapped input gather
      p_->e2e_sync_off = Alloc(static_cast<size_t>(rt_->world) * 4);
      p_->e2e_epoch_off = Alloc(4);
    }
    ValidateSpecs();
    const bool pipeline = p_->pipeline_axis >= 0;
    const bool eager = rt_->dist && rt_->world > 1 && !(p_->flags & RH_FLAG_NO_OVERLAP) &&
                       !getenv("RH_NO_EAGER_TRANSITIONS") && !pipeline;
    if (eager) TransitionFirstOrder();
    PlanGemmGroups();
    if (pipeline) PipelineOrder();
    SortGroupMembers();
    PlanFusion();
    RefineGemmGroups();
    PlanAttnChains();
    for (int i : p_->order) {
      const rh_op& op = p_->ops[i];
      cur_stage_ = StageOfOp(i);
      if (op.kind == RH_OP_PARAMETER || op.kind == RH_OP_INPUT) {
        p_->out_tensor[i] = NewTensor(i, p_->out_specs[i]);
        continue;
      }
      if (absorbed_[i]) continue;  // computed by its chain head's kernel
      if (!ew_of_.empty() && ew_of_[i] >= 0) {  // elementwise chain: one kernel at its tail
        const auto& c = ew_[ew_of_[i]];
        if (c.members.back() == i) {
          EmitEwChain(c);
          if (eager)
            for (size_t j = 0; j < c.members.size(); ++j)
              if (c.stored[j]) EagerTransitions(c.members[j]);
        }
        continue;
      }
      if (!group_of_.empty() && group_of_[i] >= 0) {  // grouped GEMM: one launch at its first member
        const int gi = group_of_[i];
        const std::vector<int>& g = groups_[gi];
        if (g.front() == i && !attn_done_[gi]) {
          const int g2 = attn_pair_[gi];
          if (g2 >= 0 && EmitAttnChain(gi, g2)) {  // score + chain + context in one kernel
            attn_done_[g2] = true;
            if (eager)
              for (int m : groups_[g2]) EagerTransitions(m);
          } else {
            EmitGemmGroup(g);
            if (eager)
              for (int m : g) EagerTransitions(chain_[m].empty() ? m : chain_[m].back());
          }
        }
        continue;
      }
      EmitOp(i);
      if (eager) EagerTransitions(Tail(i));
    }
    if ((p_->flags & RH_FLAG_REDUCE_OUTPUTS) && !(p_->flags & RH_FLAG_NO_MATERIALIZE)) {
      // training-step outputs: reduce Partial axes (the gradient all-reduce / reduce of a
      // data-parallel step), keep sharded axes sharded (the optimizer updates shards in place)
      for (int o : p_->outputs) {
        cur_stage_ = StageOfOp(o);
        Specs fin = p_->tensors[p_->out_tensor[o]].specs;
        bool rep = true;
        for (auto& x : fin) {
          if (x.kind == RH_PARTIAL) x = Rep();
          rep = rep && x.kind == RH_REPLICATED;
        }
        p_->out_tensor[o] = GetTensor(o, fin, "reduce");
        if (rep) p_->mat_tensor[o] = p_->out_tensor[o];
      }
    } else if (!(p_->flags & RH_FLAG_NO_MATERIALIZE)) {
      for (int o : p_->outputs) {
        cur_stage_ = StageOfOp(o);
        if (TryPushMaterialize(o)) continue;
        Specs rep(p_->n_axes, Rep());
        p_->mat_tensor[o] = GetTensor(o, rep, "materialize");
      }
    }
    for (const auto& rq : p_->requests) {
      cur_stage_ = StageOfOp(rq.first);
      p_->request_tensors.push_back(GetTensor(rq.first, rq.second, "request"));
    }
    EmitApply();
    if (p_->gemm_scratch_bytes) p_->gemm_scratch_off = Alloc(p_->gemm_scratch_bytes);
    p_->gemm_flags_off = Alloc(kGemmSkFlagBytes);
    if (p_->n_sync_slots) {
      p_->sync_off = Alloc(static_cast<size_t>(p_->n_sync_slots) * rt_->world * 4);
      p_->epoch_off = Alloc(4);
    }
    MergeTransitions();
    PlanAsync();
    FinalizePulls();
    EwJitBuild();
    PlanArena();
    p_->arena_bytes = arena_;
    // Barrier elision: transition sources are persistent (never recycled by the arena planner)
    // and written once per run, so a peer can only overwrite what a transition reads in the
    // NEXT run.  Every main-stream p2p transition but the last one on its axis can drop its
    // post-barrier: the next p2p transition on that axis begins with a barrier of the same
    // group, which peers cannot pass before we finished.  Async (side-stream) transitions keep
    // their post-barrier (on the side stream's own barrier state).
    // (keyed by axis and pipeline stage: the ranks of one stage run only that stage's steps;
    // cross-stage transfers (stage -2) carry their own pairwise rendezvous)
    const int n_st = std::max(1, p_->n_stages) + 1;
    auto slot_of = [&](const Step& st) { return st.axis * n_st + (st.stage < 0 ? 0 : st.stage + 1); };
    std::vector<int> last(static_cast<size_t>(p_->n_axes) * n_st, -1);
    for (size_t i = 0; i < p_->steps.size(); ++i)
      if (p_->steps[i].p2p && !p_->steps[i].async && p_->steps[i].stage != -2)
        last[slot_of(p_->steps[i])] = static_cast<int>(i);
    for (size_t i = 0; i < p_->steps.size(); ++i)
      if (p_->steps[i].p2p && p_->steps[i].stage != -2)
        p_->steps[i].post_sync = p_->steps[i].async || static_cast<int>(i) == last[slot_of(p_->steps[i])];
    // The last one on an axis: the NEXT run's first main-stream p2p transition on that axis
    // begins with the same group's barrier.  If it comes before the step that (re)writes every
    // tensor the last transition reads (kernel-written, own storage: not a source op, which the
    // host may overwrite between runs, nor an alias), peers cannot overwrite what we read before
    // we passed that barrier, and the post-barrier kernel can go too.
    std::vector<int> first(last.size(), -1);
    for (size_t i = 0; i < p_->steps.size(); ++i) {
      const Step& st = p_->steps[i];
      if (st.p2p && !st.async && st.stage != -2 && first[slot_of(st)] < 0) first[slot_of(st)] = static_cast<int>(i);
    }
    for (size_t a = 0; a < last.size(); ++a) {
      const int l = last[a];
      if (l < 0 || getenv("RH_KEEP_LAST_POST_SYNC")) continue;
      bool ok = true;
      for (int t : p_->steps[l].reads) {
        const Tensor& T = p_->tensors[t];
        const int kind = p_->ops[T.op].kind;
        if (T.alias >= 0 || !T.storage || kind == RH_OP_INPUT || kind == RH_OP_PARAMETER) {
          ok = false;
          break;
        }
        int writer = -1;
        for (size_t i = 0; i < p_->steps.size() && writer < 0; ++i)
          for (int w : p_->steps[i].writes)
            if (w == t) writer = static_cast<int>(i);
        ok = ok && writer > first[a];
      }
      if (ok) p_->steps[l].post_sync = false;
    }
    for (auto& st : p_->steps) {
      if (st.post_mode == 1) st.post_sync = true;
      if (st.post_mode == 2) st.post_sync = false;
    }
  }

 private:
  size_t Alloc(size_t bytes) {
    const size_t off = arena_;
    arena_ += Align(bytes);
    return off;
  }
  static size_t Align(size_t bytes) { return (bytes + 255) / 256 * 256; }

  // Overlap (dist mode): a p2p transition whose result is first needed well after it can start
  // runs on a side stream, concurrently with the main stream's kernels — the gradient
  // reductions of a backward pass, activations resharded for a much later consumer.  The main
  // stream waits for it right before its first reader (or at the end of the run).  Estimated
  // times: kernels max(flops / 1.2 PF/s, bytes / 5 TB/s) + 2 us, transitions wire / 500 GB/s +
  // 15 us; a transition goes async when the main-stream work it can hide behind is at least
  // half its own estimate.
  void PlanAsync() {
    auto& S = p_->steps;
    const int ns = static_cast<int>(S.size());
    p_->joins_at.assign(ns, {});
    if (!rt_->dist || rt_->world < 2 || (p_->flags & RH_FLAG_NO_OVERLAP) || p_->pipeline_axis >= 0) return;
    auto est = [&](const Step& s) {
      if (s.kind == Step::kTransition) return s.wire_bytes / 5e11 + 15e-6;
      return std::max(s.alg_flops / 1.2e15, s.alg_bytes / 5e12) + 2e-6;
    };
    for (int i = 0; i < ns; ++i) {
      Step& st = S[i];
      if (st.kind != Step::kTransition || !st.p2p || st.sync_slot < 0 || st.writes.size() != 1 || st.no_async) continue;
      const int y = Root(st.writes[0]);
      int j = -1;
      for (int k = i + 1; k < ns && j < 0; ++k)
        for (int r : S[k].reads)
          if (Root(r) == y) {
            j = k;
            break;
          }
      double hide = 0;
      for (int k = i + 1; k < (j < 0 ? ns : j); ++k)
        if (!S[k].async) hide += est(S[k]);
      if (hide < 0.5 * est(st)) continue;
      st.async = true;
      st.name += " [overlap]";
      st.join = j;
      st.async_id = p_->n_async++;
      if (j >= 0) p_->joins_at[j].push_back(st.async_id);
    }
    if (p_->n_async) {
      p_->side_flags_off = Alloc(static_cast<size_t>(rt_->world) * 4);
      p_->side_counter_off = Alloc(4);
    }
  }

  int Root(int t) const {
    while (p_->tensors[t].alias >= 0) t = p_->tensors[t].alias;
    return t;
  }

  // Grouped transitions: a run of consecutive peer-memory transitions on one mesh axis, none
  // reading another's result (the per-head K / V all-gathers feeding one grouped GEMM), becomes
  // one step: one fused barrier and one launch (PullMultiKernel) instead of one ~15-20 us
  // latency-bound transition each.  RH_NO_GROUP_TRANSITIONS=1 disables (A/B).
  void MergeTransitions() {
    static const bool off = getenv("RH_NO_GROUP_TRANSITIONS") != nullptr;
    if (off || (p_->flags & RH_FLAG_NO_FUSION)) return;
    std::vector<Step> out;
    std::vector<int> count;
    for (auto& st : p_->steps) {
      if (!out.empty() && st.kind == Step::kTransition && !st.pulls.empty()) {
        Step& pv = out.back();
        bool ok = pv.kind == Step::kTransition && !pv.pulls.empty() && pv.axis == st.axis &&
                  (pv.sync_slot >= 0) == (st.sync_slot >= 0) && pv.stage == st.stage;
        for (int r : st.reads)
          for (int w : pv.writes) ok = ok && Root(r) != Root(w);
        if (ok) {
          for (auto& f : st.pulls) pv.pulls.push_back(std::move(f));
          pv.reads.insert(pv.reads.end(), st.reads.begin(), st.reads.end());
          pv.writes.insert(pv.writes.end(), st.writes.begin(), st.writes.end());
          pv.wire_bytes += st.wire_bytes;
          pv.alg_bytes += st.alg_bytes;
          ++count.back();
          continue;
        }
      }
      out.push_back(std::move(st));
      count.push_back(1);
    }
    for (size_t i = 0; i < out.size(); ++i)
      if (count[i] > 1) out[i].name = "grouped[" + std::to_string(count[i]) + "] " + out[i].name;
    p_->steps = std::move(out);
  }

  // Launch closures of the peer-memory transitions (after merging and overlap planning): the
  // fused pre-barrier unless the step is overlapped (side stream: a 1-CTA barrier kernel instead
  // of a grid spinning next to the main stream's kernels), a capped grid on the side stream,
  // and for merged steps the grouped launch (its segment table written at load).
  void FinalizePulls() {
    rh_program* P = p_;
    for (size_t i = 0; i < p_->steps.size(); ++i) {
      Step& st = p_->steps[i];
      if (st.pulls.empty() && !st.fine) continue;
      const bool async = st.async;
      const int slot = async ? -1 : st.sync_slot;
      const int axis = st.axis;
      const int n = static_cast<int>(st.pulls.size());
      st.launches = 1;
      auto sync_of = [P, axis, slot](int li) {
        PeerSync y{};
        if (slot < 0) return y;
        const int g = P->mesh->rt->first_rank + li;
        const std::vector<int> members = P->mesh->Group(axis, g);
        const size_t row = P->sync_off + static_cast<size_t>(slot) * P->mesh->rt->world * 4;
        y.d = static_cast<int>(members.size());
        y.me = g;
        for (size_t k = 0; k < members.size(); ++k) {
          y.members[k] = members[k];
          y.peer_slot[k] = reinterpret_cast<uint32_t*>(P->peer_base[members[k]] + row);
        }
        y.my_slot = reinterpret_cast<uint32_t*>(P->peer_base[g] + row);
        y.epoch = reinterpret_cast<const uint32_t*>(P->peer_base[g] + P->epoch_off);
        y.err = reinterpret_cast<uint32_t*>(P->peer_base[g] + P->err_off);
        y.timeout_ns = SyncTimeoutNs();
        return y;
      };
      const std::vector<std::function<PullArgs(int)>> pulls = st.pulls;
      const int cap = async ? SideBlocks() : 0;
      if (st.fine) {
        const auto fine = st.fine;
        st.run = [fine, sync_of, cap](int li, cudaStream_t s) { return fine(li, s, sync_of(li), cap); };
        continue;
      }
      if (n == 1) {
        st.run = [pulls, sync_of, cap](int li, cudaStream_t s) {
          PullArgs a = pulls[0](li);
          a.max_blocks = cap;
          a.sync = sync_of(li);
          return LaunchPull(a, s);
        };
        continue;
      }
      const size_t off = Alloc(PullMultiTableBytes(n));
      auto ok = std::make_shared<std::vector<char>>(rt_->n_local(), 0);
      st.init = [P, pulls, cap, off, ok](int li) {
        std::vector<PullArgs> v;
        for (const auto& f : pulls) v.push_back(f(li));
        (*ok)[li] = PreparePullMulti(v.data(), static_cast<int>(v.size()), cap,
                                     P->peer_base[P->mesh->rt->first_rank + li] + off);
      };
      st.fini = [P, off](int li) { ReleasePullMulti(P->peer_base[P->mesh->rt->first_rank + li] + off); };
      st.run = [P, pulls, sync_of, cap, off, ok](int li, cudaStream_t s) {
        if ((*ok)[li]) return LaunchPullMulti(P->peer_base[P->mesh->rt->first_rank + li] + off, sync_of(li), s);
        // not groupable (zero-fill / staged / mixed kinds): one pull each, the first one's
        // barrier orders all of them (every source was produced before the step)
        int launches = 0;
        for (size_t k = 0; k < pulls.size(); ++k) {
          PullArgs a = pulls[k](li);
          a.max_blocks = cap;
          if (k == 0) a.sync = sync_of(li);
          launches += LaunchPull(a, s);
        }
        return launches;
      };
    }
  }

  // Arena planner: tensor storage is placed after lowering, from the schedule's liveness.
  // Persistent (own storage for the program's lifetime): parameters and inputs, outputs and
  // their materialized copies, request targets, and every tensor a transition reads from a
  // PEER (a peer may still be reading it while this rank runs ahead; the transition barriers
  // only order the next write of that same buffer).  Every other buffer lives from the step
  // that writes it to the last step that reads it, and buffers with disjoint lifetimes share
  // storage (best-fit over a coalescing free list).  The schedule is one stream per rank, so
  // stream order is the only ordering reuse needs.  RH_FLAG_KEEP_ALL disables reuse.
  void PlanArena() {
    auto& T = p_->tensors;
    const int nt = static_cast<int>(T.size());
    const int ns = static_cast<int>(p_->steps.size());
    std::vector<bool> persist(nt, (p_->flags & RH_FLAG_KEEP_ALL) != 0);
    for (size_t i = 0; i < p_->ops.size(); ++i)
      if ((p_->ops[i].kind == RH_OP_PARAMETER || p_->ops[i].kind == RH_OP_INPUT) && p_->out_tensor[i] >= 0)
        persist[Root(p_->out_tensor[i])] = true;
    for (int o : p_->outputs) {
      if (p_->out_tensor[o] >= 0) persist[Root(p_->out_tensor[o])] = true;
      if (p_->mat_tensor[o] >= 0) persist[Root(p_->mat_tensor[o])] = true;
    }
    for (int t : p_->request_tensors) persist[Root(t)] = true;
    for (int t : remote_read_) persist[Root(t)] = true;
    std::vector<int> def(nt, -1), last(nt, -1);
    for (int s = 0; s < ns; ++s) {
      for (int w : p_->steps[s].writes) {
        const int r = Root(w);
        if (def[r] < 0) def[r] = s;
        last[r] = std::max(last[r], s);
      }
      for (int x : p_->steps[s].reads) {
        const int r = Root(x);
        if (def[r] < 0) persist[r] = true;  // read before any step writes it: host-written
        last[r] = std::max(last[r], s);
      }
    }
    std::vector<std::vector<int>> born(ns), dies(ns);
    for (int t = 0; t < nt; ++t) {
      if (!T[t].storage || T[t].alias >= 0) continue;
      if (persist[t] || def[t] < 0) {
        persist[t] = true;
        T[t].offset = Alloc(T[t].bytes);
        continue;
      }
      born[def[t]].push_back(t);
      dies[last[t]].push_back(t);
    }
    const size_t base = arena_;
    size_t top = 0;
    std::map<size_t, size_t> free_blocks;  // offset -> size (coalesced)
    for (int s = 0; s < ns; ++s) {
      for (int t : born[s]) {  // outputs of step s never overlap its inputs (freed after)
        const size_t need = Align(T[t].bytes);
        auto best = free_blocks.end();
        for (auto it = free_blocks.begin(); it != free_blocks.end(); ++it)
          if (it->second >= need && (best == free_blocks.end() || it->second < best->second)) best = it;
        if (best != free_blocks.end()) {
          T[t].offset = base + best->first;
          if (best->second > need) free_blocks[best->first + need] = best->second - need;
          free_blocks.erase(best);
        } else if (!free_blocks.empty() && std::prev(free_blocks.end())->first + std::prev(free_blocks.end())->second == top) {
          auto tail = std::prev(free_blocks.end());  // grow the block at the top
          T[t].offset = base + tail->first;
          top = tail->first + need;
          free_blocks.erase(tail);
        } else {
          T[t].offset = base + top;
          top += need;
        }
        T[t].recycled = true;
      }
      for (int t : dies[s]) {
        size_t off = T[t].offset - base, len = Align(T[t].bytes);
        auto next = free_blocks.lower_bound(off);
        if (next != free_blocks.end() && off + len == next->first) {
          len += next->second;
          next = free_blocks.erase(next);
        }
        if (next != free_blocks.begin()) {
          auto prev = std::prev(next);
          if (prev->first + prev->second == off) {
            off = prev->first;
            len += prev->second;
            free_blocks.erase(prev);
          }
        }
        free_blocks[off] = len;
      }
    }
    arena_ = base + top;
    p_->pool_bytes = top;
    for (int t = 0; t < nt; ++t) {
      if (T[t].alias < 0) continue;
      const int r = Root(t);
      T[t].offset = T[r].offset;
      T[t].recycled = T[r].recycled;
    }
  }

  Dims GDims(int i) const { return Dims(p_->ops[i].dims, p_->ops[i].dims + p_->ops[i].rank); }

  static constexpr int kOpStage = -3;  // NewTensor: the stage that computes the op
  int NewTensor(int op, const Specs& specs, bool alloc = true, int stage = kOpStage) {
    Tensor t;
    t.op = op;
    t.stage = stage == kOpStage ? StageOfOp(op) : stage;
    t.specs = specs;
    t.gdims = GDims(op);
    t.ldims = LocalDims(t.gdims, specs, mesh_, specs.size());
    t.dtype = p_->ops[op].dtype;
    t.bytes = static_cast<size_t>(t.elems()) * ElemBytes(t.dtype);
    t.storage = alloc;  // placed by PlanArena
    p_->tensors.push_back(t);
    const int idx = static_cast<int>(p_->tensors.size()) - 1;
    cache_[Key(op, specs, p_->tensors[idx].stage)] = idx;
    return idx;
  }

  static std::string Key(int op, const Specs& s, int stage) {
    return std::to_string(op) + "|" + SpecsStr(s) + "@" + std::to_string(stage);
  }
  int StageOfOp(int i) const { return p_->pipeline_axis >= 0 ? p_->ops[i].stage : -1; }
  // pipeline programs: one kernel never spans two tasks (stage, microbatch, phase) of the 1F1B
  // order — fusion would move an op out of its task
  bool SameTask(int a, int b) const {
    if (p_->pipeline_axis < 0) return true;
    const rh_op &x = p_->ops[a], &y = p_->ops[b];
    return x.stage == y.stage && x.microbatch == y.microbatch && x.phase == y.phase;
  }

  void ValidateSpecs() {
    for (size_t i = 0; i < p_->ops.size(); ++i) {
      const Dims g = GDims(static_cast<int>(i));
      auto check = [&](const Specs& s, const Dims& dims, const std::string& what) {
        for (int a = 0; a < p_->n_axes; ++a) {
          if (!Valid(s[a], LocalDims(dims, s, mesh_, a), mesh_[a]))
            Fail("op " + std::to_string(i) + ": " + what + " spec " + SpecStr(s[a]) +
                 " invalid on axis " + std::to_string(a));
        }
      };
      check(p_->out_specs[i], g, "output");
      for (size_t s = 0; s < p_->inputs[i].size(); ++s)
        check(p_->in_specs[i][s], GDims(p_->inputs[i][s]), "input");
      if (p_->pipeline_axis >= 0) {  // the pipeline axis places stages, it shards nothing
        const int pa = p_->pipeline_axis;
        bool rep = p_->out_specs[i][pa].kind == RH_REPLICATED;
        for (const auto& sp : p_->in_specs[i]) rep = rep && sp[pa].kind == RH_REPLICATED;
        if (!rep) Fail("op " + std::to_string(i) + ": spec on the pipeline axis must be replicated");
        const rh_op& op = p_->ops[i];
        if (op.stage < 0 || op.stage >= p_->n_stages) Fail("op " + std::to_string(i) + ": stage out of range");
      }
    }
  }

  // 1F1B (taskgraph.cpp:173-211): stage s runs min(m, S - s) forward microbatches, then
  // alternates backward(b) [+ LocalAccumulate(b)] and the next forward.  The op order is a
  // topological order in which every stage's ops come task by task in that sequence (an op is
  // eligible when its inputs are done and every earlier task of its stage is); ops of tasks the
  // sequence does not list (no backward, accumulations of microbatch 1) follow their stage's
  // last listed task.  Cross-stage transfers are emitted at their consumer, so each Send/Recv
  // rendezvous sits at one point of this global order.
  void PipelineOrder() {
    const int n = static_cast<int>(p_->ops.size()), S = p_->n_stages;
    int m = 1;
    for (const auto& op : p_->ops) m = std::max(m, static_cast<int>(op.microbatch));
    std::vector<std::map<std::pair<int, int>, int>> seq(S);  // (phase, microbatch) -> index
    for (int s = 0; s < S; ++s) {
      int k = 0;
      auto put = [&](int ph, int mb) { seq[s].emplace(std::make_pair(ph, mb), k++); };
      const int warm = std::min(m, S - s);
      int next = 1;
      for (; next <= warm; ++next) put(RH_PHASE_FWD, next);
      for (int b = 1; b <= m; ++b) {
        put(RH_PHASE_BWD, b);
        if (b >= 2) put(RH_PHASE_ACC, b);
        if (next <= m) put(RH_PHASE_FWD, next++);
      }
    }
    std::vector<int> task(n);
    for (int i = 0; i < n; ++i) {
      const rh_op& op = p_->ops[i];
      if (op.kind == RH_OP_PARAMETER || op.kind == RH_OP_INPUT) {
        task[i] = -1;  // sources: before everything
        continue;
      }
      auto it = seq[op.stage].find({op.phase, op.microbatch});
      task[i] = it != seq[op.stage].end() ? it->second : static_cast<int>(seq[op.stage].size());
    }
    // nodes: single ops, or a grouped-GEMM group (same stage and task) as one node
    auto node = [&](int i) { return group_of_.empty() || group_of_[i] < 0 ? i : n + group_of_[i]; };
    const int nn = n + static_cast<int>(groups_.size());
    std::vector<std::vector<int>> members(nn);
    std::vector<int> pos(n);
    for (int k = 0; k < n; ++k) pos[p_->order[k]] = k;
    for (int k = 0; k < n; ++k) members[node(p_->order[k])].push_back(p_->order[k]);
    std::vector<int> prio(nn, n), indeg(nn, 0), ntask(nn, -1), nstage(nn, 0);
    std::vector<std::vector<int>> succ(nn);
    for (int i = 0; i < n; ++i) {
      const int v = node(i);
      prio[v] = std::min(prio[v], pos[i]);
      ntask[v] = task[i];
      nstage[v] = p_->ops[i].stage;
      for (int x : p_->inputs[i]) {
        succ[node(x)].push_back(v);
        ++indeg[v];
      }
    }
    std::vector<std::vector<int>> left(S);  // ops left per (stage, task)
    for (int s = 0; s < S; ++s) left[s].assign(seq[s].size() + 1, 0);
    for (int i = 0; i < n; ++i)
      if (task[i] >= 0) ++left[p_->ops[i].stage][task[i]];
    std::vector<int> cur(S, 0);
    auto advance = [&](int s) {
      while (cur[s] < static_cast<int>(left[s].size()) && left[s][cur[s]] == 0) ++cur[s];
    };
    for (int s = 0; s < S; ++s) advance(s);
    std::set<std::pair<int, int>> ready, parked;  // (priority, node)
    auto offer = [&](int v) {
      if (ntask[v] < 0 || ntask[v] == cur[nstage[v]]) ready.insert({prio[v], v});
      else parked.insert({prio[v], v});
    };
    for (int v = 0; v < nn; ++v)
      if (!members[v].empty() && !indeg[v]) offer(v);
    std::vector<int> order;
    while (!ready.empty()) {
      const int v = ready.begin()->second;
      ready.erase(ready.begin());
      for (int i : members[v]) order.push_back(i);
      if (ntask[v] >= 0) {
        const int s = nstage[v];
        left[s][ntask[v]] -= static_cast<int>(members[v].size());
        const int before = cur[s];
        advance(s);
        if (cur[s] != before) {  // the stage's next task opened: release its parked nodes
          for (auto it = parked.begin(); it != parked.end();) {
            if (nstage[it->second] == s && ntask[it->second] == cur[s]) {
              ready.insert(*it);
              it = parked.erase(it);
            } else {
              ++it;
            }
          }
        }
      }
      for (int w : succ[v])
        if (--indeg[w] == 0) offer(w);
    }
    if (static_cast<int>(order.size()) != n)
      Fail("pipeline program: the 1F1B task order contradicts the data dependencies");
    p_->order = order;
  }

  // ApplyGradients (taskgraph.cpp:161-165): each parameter is updated in place by its stage,
  // p -= lr * g, with the gradient brought to the parameter's own layout first (Partial axes
  // reduced, shards matched).
  void EmitApply() {
    rh_program* P = p_;
    for (const auto& ap : p_->apply) {
      const int g = ap.first, w = ap.second;
      if (p_->ops[w].kind != RH_OP_PARAMETER) Fail("apply: op " + std::to_string(w) + " is not a parameter");
      if (GDims(g) != GDims(w) || p_->ops[g].dtype != p_->ops[w].dtype) Fail("apply: gradient / parameter mismatch");
      cur_stage_ = StageOfOp(w);
      const int wt = p_->out_tensor[w];
      const int gt = GetTensor(g, p_->tensors[wt].specs, "apply");
      Step st;
      st.kind = Step::kKernel;
      st.name = "apply_sgd op" + std::to_string(w);
      st.launches = 1;
      st.alg_bytes = 3.0 * p_->tensors[wt].bytes;
      st.alg_flops = 2.0 * p_->tensors[wt].elems();
      const float lr = p_->lr;
      const int first = rt_->first_rank;
      st.run = [P, wt, gt, lr, first](int li, cudaStream_t s) {
        const int r = first + li;
        LaunchSgd(P->Ptr(P->tensors[wt], r), P->Ptr(P->tensors[gt], r), P->tensors[wt].elems(), lr,
                  P->tensors[wt].dtype, s);
        return 1;
      };
      st.reads = {gt, wt};
      st.writes = {wt};
      AddStep(std::move(st));
    }
  }

  Specs NaturalSpecs(int i, const std::vector<Specs>& ins) {
    const rh_op& op = p_->ops[i];
    Specs nat(p_->n_axes);
    for (int a = 0; a < p_->n_axes; ++a) {
      std::vector<rh_spec> in_a;
      std::vector<Dims> in_d;
      for (size_t s = 0; s < ins.size(); ++s) {
        in_a.push_back(ins[s][a]);
        in_d.push_back(LocalDims(GDims(p_->inputs[i][s]), ins[s], mesh_, a));
      }
      nat[a] = Natural(op, in_a, in_d, LocalDims(GDims(i), nat, mesh_, a), mesh_[a], p_->out_specs[i][a]);
    }
    return nat;
  }

  bool IsElementwiseUnary(int i) const {
    return p_->ops[i].kind == RH_OP_UNARY && p_->ops[i].fn != RH_FN_SOFTMAX;
  }

  // Fusion of comm-free unary chains into one kernel, and into the epilogue of the GEMM /
  // add / mul that produces them.  Op u is absorbed into its producer's kernel when u is an
  // elementwise unary whose single input edge needs no resharding and whose producer has no
  // other consumer and is not a program output.
  void PlanFusion() {
    const int n = static_cast<int>(p_->ops.size());
    absorbed_.assign(n, false);
    chain_.assign(n, {});
    resid_.assign(n, Resid{});
    if (p_->flags & RH_FLAG_NO_FUSION) return;
    std::vector<int> uses(n, 0);
    std::vector<int> consumer(n, -1);
    for (int i = 0; i < n; ++i)
      for (int s : p_->inputs[i]) {
        ++uses[s];
        consumer[s] = i;
      }
    std::vector<bool> is_out(n, false);
    for (int o : p_->outputs) is_out[o] = true;
    auto natural_ok = [&](int i) {
      try {
        return SpecsEq(NaturalSpecs(i, p_->in_specs[i]), p_->out_specs[i]);
      } catch (const Error&) {
        return false;
      }
    };
    auto no_partial = [&](const Specs& s) {
      for (auto& x : s)
        if (x.kind == RH_PARTIAL) return false;
      return true;
    };
    std::vector<int> pos(n, 0);
    for (size_t k = 0; k < p_->order.size(); ++k) pos[p_->order[k]] = static_cast<int>(k);
    for (int h : p_->order) {
      const rh_op& op = p_->ops[h];
      if (op.kind != RH_OP_MATMUL || absorbed_[h]) continue;  // elementwise heads: PlanEwChains
      int cur = h;
      while (true) {
        if (uses[cur] != 1 || is_out[cur]) break;
        const int v = consumer[cur];
        if (!IsElementwiseUnary(v) || p_->ops[v].dtype != op.dtype || !SameTask(v, h)) break;
        if (!SpecsEq(p_->in_specs[v][0], p_->out_specs[cur])) break;
        if (!no_partial(p_->out_specs[cur]) || !natural_ok(cur) || !natural_ok(v)) break;
        if (static_cast<int>(chain_[h].size()) + 1 >= kMaxChain) break;
        chain_[h].push_back(v);
        absorbed_[v] = true;
        cur = v;
      }
      // The GEMM epilogue runs on 4 warps per SM: only short chains ride in it; a longer chain
      // runs as one full-occupancy elementwise kernel instead (same HBM traffic, 10x the issue
      // rate for its transcendental work).
      // bf16 GEMM epilogues take only the exact packed ops (relu / neg / identity); tanh runs
      // use the T^k tables of the elementwise kernels.
      bool epi_ok = chain_[h].size() <= kMaxGemmEpilogue;
      if (op.dtype == RH_BF16) {
        // bf16: exact packed ops and tanh runs (a run of k tanh = one lookup in the T^k table,
        // staged in the GEMM's shared memory), at most kMaxGemmEpilogue of them after run
        // compression (ChainOf)
        int n_fn = 0;
        bool ok = true, in_run = false, has_tanh = false;
        for (int v : chain_[h]) {
          const int fn = UnaryFn(v);
          if (fn == RH_FN_TANH) {
            has_tanh = true;
            if (!in_run) ++n_fn;
            in_run = true;
            continue;
          }
          in_run = false;
          ++n_fn;
          ok = ok && (fn == RH_FN_RELU || fn == RH_FN_NEG || fn == RH_FN_IDENTITY);
        }
        static const bool no_tanh = getenv("RH_NO_EPI_TANH") != nullptr;  // A/B knob (profiles/)
        epi_ok = ok && n_fn <= static_cast<int>(kMaxGemmEpilogue) && !(no_tanh && has_tanh);
      }
      if (op.kind == RH_OP_MATMUL && !epi_ok) {
        for (int v : chain_[h]) absorbed_[v] = false;
        chain_[h].clear();
      }
      // Residual add after the GEMM (and its epilogue chain): bf16, the add's other operand in
      // the same layout, no other reader of the pre-add value -> the GEMM's epilogue adds it
      // (GemmArgs::resid; the separate add kernel re-read the GEMM output from HBM).
      static const bool no_resid = getenv("RH_NO_RESID_FUSION") != nullptr;  // A/B knob
      const int t = chain_[h].empty() ? h : chain_[h].back();
      if (!no_resid && op.dtype == RH_BF16 && uses[t] == 1 && !is_out[t] &&
          (group_of_.empty() || group_of_[h] < 0)) {
        const int v = consumer[t];
        const rh_op& a = p_->ops[v];
        if (a.kind == RH_OP_ADD && a.dtype == op.dtype && SameTask(v, h) && p_->inputs[v].size() == 2) {
          const int slot = p_->inputs[v][0] == t ? 1 : 0;
          const int x = p_->inputs[v][slot];
          // x must be read in the layout it is produced in: a residual that needs a transition
          // would move that transition's join up to the GEMM's start (C5 at N=2: +0.5 ms
          // exposed transition time when it did)
          if (x != t && pos[x] < pos[h] && SpecsEq(p_->in_specs[v][slot], p_->out_specs[x]) &&
              SpecsEq(p_->in_specs[v][0], p_->out_specs[t]) && SpecsEq(p_->in_specs[v][1], p_->out_specs[t]) &&
              SpecsEq(p_->out_specs[v], p_->out_specs[t]) && no_partial(p_->out_specs[t]) && natural_ok(t) &&
              natural_ok(v) && GDims(x) == GDims(v) && GDims(v) == GDims(t)) {
            resid_[h] = Resid{v, x, slot};
            absorbed_[v] = true;
          }
        }
      }
    }
    PlanTransposeFold(uses, consumer, is_out);
    PlanEwChains(is_out, natural_ok, no_partial);
    PlanRemat(is_out, no_partial);
  }

  // Horizontal fusion of independent MatMuls (the per-head q/k/v, score and context GEMMs of
  // the 32-head block: 96 + 32 + 32 rank-2 matmuls, each far below a wave): MatMuls with the
  // same local shapes, transposes, specs and DAG depth (no path can join two ops of equal depth)
  // run as one grouped tcgen05 launch (GemmTcGroup).  The schedule order is re-derived on the
  // DAG with every group contracted to one node, so each group's members are contiguous and
  // all their inputs precede the first of them.  Membership is refined after fusion planning
  // (equal epilogue chains and folded-transpose flags).  RH_NO_GEMM_GROUP=1 disables (A/B).
  void PlanGemmGroups() {
    const int n = static_cast<int>(p_->ops.size());
    group_of_.assign(n, -1);
    groups_.clear();
    if ((p_->flags & (RH_FLAG_NO_FUSION | RH_FLAG_SIMT_GEMM)) || getenv("RH_NO_GEMM_GROUP")) return;
    std::vector<int> depth(n, 0);
    for (int i : p_->order)
      for (int s : p_->inputs[i]) depth[i] = std::max(depth[i], depth[s] + 1);
    std::map<std::string, std::vector<int>> cand;
    for (int i : p_->order) {
      const rh_op& op = p_->ops[i];
      if (op.kind != RH_OP_MATMUL || op.dtype != RH_BF16 || p_->inputs[i].size() != 2) continue;
      try {
        if (!SpecsEq(NaturalSpecs(i, p_->in_specs[i]), p_->out_specs[i])) continue;
      } catch (const Error&) {
        continue;
      }
      std::ostringstream key;
      key << depth[i] << '|' << op.transpose_a << op.transpose_b << '|' << SpecsStr(p_->out_specs[i]);
      if (p_->pipeline_axis >= 0) key << "|s" << op.stage << '.' << op.microbatch << '.' << op.phase;
      for (int sl = 0; sl < 2; ++sl) {
        key << '|' << SpecsStr(p_->in_specs[i][sl]);
        for (auto x : LocalDims(GDims(p_->inputs[i][sl]), p_->in_specs[i][sl], mesh_, p_->n_axes)) key << ',' << x;
      }
      cand[key.str()].push_back(i);
    }
    for (auto& kv : cand) {
      if (kv.second.size() < 2) continue;
      for (int m : kv.second) group_of_[m] = static_cast<int>(groups_.size());
      groups_.push_back(kv.second);
    }
    if (groups_.empty() || p_->pipeline_axis >= 0) return;  // pipeline: PipelineOrder contracts them
    // contracted topological order (ties: the earliest member's position in the current order)
    std::vector<int> pos(n);
    for (int k = 0; k < n; ++k) pos[p_->order[k]] = k;
    auto node = [&](int i) { return group_of_[i] >= 0 ? n + group_of_[i] : i; };
    const int nn = n + static_cast<int>(groups_.size());
    std::vector<std::vector<int>> members(nn);
    for (int k = 0; k < n; ++k) members[node(p_->order[k])].push_back(p_->order[k]);
    std::vector<int> prio(nn, n), indeg(nn, 0);
    std::vector<std::vector<int>> succ(nn);
    for (int i = 0; i < n; ++i) {
      prio[node(i)] = std::min(prio[node(i)], pos[i]);
      for (int s : p_->inputs[i]) {
        succ[node(s)].push_back(node(i));
        ++indeg[node(i)];
      }
    }
    std::set<std::pair<int, int>> ready;
    for (int v = 0; v < nn; ++v)
      if (!members[v].empty() && indeg[v] == 0) ready.insert({prio[v], v});
    std::vector<int> order;
    while (!ready.empty()) {
      const int v = ready.begin()->second;
      ready.erase(ready.begin());
      for (int m : members[v]) order.push_back(m);
      for (int w : succ[v])
        if (--indeg[w] == 0) ready.insert({prio[w], w});
    }
    if (static_cast<int>(order.size()) != n) Fail("internal: grouped schedule is not a topological order");
    p_->order = order;
  }

  void SortGroupMembers() {
    std::vector<int> pos(p_->ops.size());
    for (size_t k = 0; k < p_->order.size(); ++k) pos[p_->order[k]] = static_cast<int>(k);
    for (auto& g : groups_) std::sort(g.begin(), g.end(), [&](int a, int b) { return pos[a] < pos[b]; });
  }

  // After fusion planning: members of one launch must share the epilogue chain (unary fns of
  // the fused tail) and the folded-transpose flags.  Singletons fall back to a plain GEMM.
  void RefineGemmGroups() {
    if (groups_.empty()) return;
    std::vector<std::vector<int>> out;
    std::fill(group_of_.begin(), group_of_.end(), -1);
    for (const auto& g : groups_) {
      std::map<std::string, std::vector<int>> parts;
      std::vector<std::string> keys;
      for (int m : g) {
        std::ostringstream k;
        for (int v : chain_[m]) k << UnaryFn(v) << ',';
        if (!fold_t_.empty()) k << '|' << fold_t_[m][0] << fold_t_[m][1];
        if (!parts.count(k.str())) keys.push_back(k.str());
        parts[k.str()].push_back(m);
      }
      for (const auto& k : keys) {
        if (parts[k].size() < 2) continue;
        for (int m : parts[k]) group_of_[m] = static_cast<int>(out.size());
        out.push_back(parts[k]);
      }
    }
    groups_ = std::move(out);
  }

  // One grouped tcgen05 launch for the members (all inputs already computed: they precede the
  // group in the schedule).  Falls back to one GEMM per member when the grouped kernel cannot
  // take the shape.
  void EmitGemmGroup(const std::vector<int>& mem) {
    rh_program* P = p_;
    const int n = static_cast<int>(mem.size());
    std::vector<std::array<int, 2>> in_t(n);
    std::vector<int> out_t(n);
    for (int k = 0; k < n; ++k) {
      const int i = mem[k];
      for (int sl = 0; sl < 2; ++sl) {
        if (!fold_t_.empty() && fold_t_[i][sl]) {
          const int t = p_->inputs[i][sl];
          in_t[k][sl] = GetTensor(p_->inputs[t][0], Transposed(p_->in_specs[i][sl]), "edge");
        } else {
          in_t[k][sl] = GetTensor(p_->inputs[i][sl], p_->in_specs[i][sl], "edge");
        }
      }
      p_->in_tensor[i] = {in_t[k][0], in_t[k][1]};
      for (int sl = 0; sl < 2; ++sl)
        if (!fold_t_.empty() && fold_t_[i][sl]) p_->in_tensor[i][sl] = -1;
    }
    for (int k = 0; k < n; ++k) {
      const int i = mem[k];
      const int tail = chain_[i].empty() ? i : chain_[i].back();
      out_t[k] = NewTensor(tail, p_->out_specs[i]);
      if (tail != i) p_->tensors[out_t[k]].gdims = GDims(i);
      p_->out_tensor[tail] = out_t[k];
    }
    const int i0 = mem[0];
    const rh_op& op = P->ops[i0];
    const Dims ad = P->tensors[in_t[0][0]].ldims, bd = P->tensors[in_t[0][1]].ldims;
    const bool fa = !fold_t_.empty() && fold_t_[i0][0], fb = !fold_t_.empty() && fold_t_[i0][1];
    GemmArgs g{};
    g.ta = op.transpose_a != fa;
    g.tb = op.transpose_b != fb;
    g.m = g.ta ? ad[1] : ad[0];
    g.k = g.ta ? ad[0] : ad[1];
    g.n = g.tb ? bd[0] : bd[1];
    g.dtype = op.dtype;
    g.epi = ChainOf(i0, false);
    bool shared_a = true;
    for (int k = 1; k < n; ++k) shared_a = shared_a && in_t[k][0] == in_t[0][0];
    if (!GemmTcGroupSupported(g, n, shared_a)) {
      for (int k = 0; k < n; ++k) EmitKernel(mem[k], {in_t[k][0], in_t[k][1]}, out_t[k]);
      return;
    }
    const size_t off = Alloc(GemmTcGroupTableBytes(n));
    Step st;
    st.kind = Step::kKernel;
    st.launches = 1;
    st.name = "gemm_tc_group[" + std::to_string(n) + "] " + OpName(mem.front()) + ".." + OpName(mem.back()) +
              (fa || fb ? " [T-folded]" : "") + GemmTcGroupSchedule(g, n, shared_a);
    st.alg_flops = 2.0 * g.m * g.n * g.k * n;
    std::set<int> rd;
    for (int k = 0; k < n; ++k) {
      rd.insert(in_t[k][0]);
      rd.insert(in_t[k][1]);
    }
    for (int t : rd) st.alg_bytes += static_cast<double>(P->tensors[t].bytes);
    for (int t : out_t) st.alg_bytes += static_cast<double>(P->tensors[t].bytes);
    const int first = rt_->first_rank;
    st.init = [P, g, in_t, out_t, off, first, n](int li) {
      const int r = first + li;
      std::vector<const void*> a(n), b(n);
      std::vector<void*> c(n);
      for (int k = 0; k < n; ++k) {
        a[k] = P->Ptr(P->tensors[in_t[k][0]], r);
        b[k] = P->Ptr(P->tensors[in_t[k][1]], r);
        c[k] = P->Ptr(P->tensors[out_t[k]], r);
      }
      GemmArgs x = g;
      x.epi = Patch(P, g.epi, r);
      PrepareGemmTcGroup(x, n, a.data(), b.data(), c.data(), P->peer_base[r] + off);
    };
    st.fini = [P, off, first](int li) { ReleaseGemmTcGroup(P->peer_base[first + li] + off); };
    st.run = [P, g, off, first](int li, cudaStream_t s) {
      const int r = first + li;
      GemmArgs x = g;
      x.epi = Patch(P, g.epi, r);
      LaunchGemmTcGroup(x, P->peer_base[r] + off, s);
      return 1;
    };
    st.reads.assign(rd.begin(), rd.end());
    st.writes = out_t;
    AddStep(std::move(st));
  }
  // Fused attention-head chains: a grouped score GEMM (Q_h K_h^T, epilogue chain) whose every
  // member's value is read only by the matching member of one grouped context GEMM
  // (chain(S_h) V_h) runs with it as one kernel (LaunchAttnChain): the scores never reach HBM.
  // attn_pair_[score group] = context group; local shapes are checked at emission
  // (EmitAttnChain falls back to the two grouped launches).  RH_NO_ATTN_FUSION disables.
  void PlanAttnChains() {
    const int n = static_cast<int>(p_->ops.size());
    attn_pair_.assign(groups_.size(), -1);
    attn_done_.assign(groups_.size(), false);
    static const bool off = getenv("RH_NO_ATTN_FUSION") != nullptr;
    if (off || groups_.empty() || (p_->flags & (RH_FLAG_NO_FUSION | RH_FLAG_SIMT_GEMM | RH_FLAG_KEEP_ALL))) return;
    std::vector<int> uses(n, 0), consumer(n, -1), slot(n, -1), pos(n, 0);
    for (int i = 0; i < n; ++i)
      for (size_t k = 0; k < p_->inputs[i].size(); ++k) {
        const int src = p_->inputs[i][k];
        ++uses[src];
        consumer[src] = i;
        slot[src] = static_cast<int>(k);
      }
    std::vector<bool> is_out(n, false);
    for (int o : p_->outputs) is_out[o] = true;
    for (size_t k = 0; k < p_->order.size(); ++k) pos[p_->order[k]] = static_cast<int>(k);
    auto folded = [&](int m) { return !fold_t_.empty() && (fold_t_[m][0] || fold_t_[m][1]); };
    for (size_t g1 = 0; g1 < groups_.size(); ++g1) {
      const std::vector<int>& G = groups_[g1];
      int g2 = -1;
      bool ok = G.size() >= 1;
      std::vector<int> ctx;
      for (int m : G) {
        const rh_op& op = p_->ops[m];
        const int t = Tail(m);
        ok = ok && op.kind == RH_OP_MATMUL && op.dtype == RH_BF16 && !op.transpose_a && op.transpose_b && !folded(m) &&
             resid_[m].v < 0 && uses[t] == 1 && !is_out[t];
        if (!ok) break;
        const int c = consumer[t];
        const rh_op& co = p_->ops[c];
        ok = co.kind == RH_OP_MATMUL && slot[t] == 0 && !co.transpose_a && !co.transpose_b && !folded(c) &&
             chain_[c].empty() && resid_[c].v < 0 && group_of_[c] >= 0 && SameTask(c, m) &&
             SpecsEq(p_->in_specs[c][0], p_->out_specs[t]) && pos[p_->inputs[c][1]] < pos[G.front()];
        if (!ok) break;
        if (g2 < 0) g2 = group_of_[c];
        ok = group_of_[c] == g2 && ChainSig(m) == ChainSig(G.front());
        ctx.push_back(c);
      }
      if (!ok || g2 < 0 || groups_[g2].size() != G.size()) continue;
      // the context group's members in the score group's order
      std::vector<int> sorted_ctx = ctx;
      std::sort(sorted_ctx.begin(), sorted_ctx.end());
      std::vector<int> g2m = groups_[g2];
      std::sort(g2m.begin(), g2m.end());
      if (sorted_ctx != g2m) continue;
      attn_pair_[g1] = g2;
      attn_ctx_[g1] = ctx;
    }
  }

  std::string ChainSig(int m) {
    std::ostringstream k;
    for (int v : chain_[m]) k << UnaryFn(v) << ',';
    return k.str();
  }

  bool EmitAttnChain(int g1, int g2) {
    rh_program* P = p_;
    const std::vector<int>& S = groups_[g1];
    const std::vector<int>& C = attn_ctx_[g1];
    const int n = static_cast<int>(S.size());
    std::vector<int> qt(n), kt(n), vt(n), ot(n);
    for (int h = 0; h < n; ++h) {
      qt[h] = GetTensor(p_->inputs[S[h]][0], p_->in_specs[S[h]][0], "edge");
      kt[h] = GetTensor(p_->inputs[S[h]][1], p_->in_specs[S[h]][1], "edge");
      vt[h] = GetTensor(p_->inputs[C[h]][1], p_->in_specs[C[h]][1], "edge");
    }
    const Dims qd = P->tensors[qt[0]].ldims, kd = P->tensors[kt[0]].ldims, vd = P->tensors[vt[0]].ldims;
    bool ok = qd.size() == 2 && kd.size() == 2 && vd.size() == 2 && qd[1] == kd[1] && kd == vd &&
              AttnChainSupported(n, qd[0], kd[0], qd[1]) && SpecsEq(NaturalSpecs(S[0], p_->in_specs[S[0]]), p_->out_specs[S[0]]);
    for (int h = 0; h < n && ok; ++h)
      ok = P->tensors[qt[h]].ldims == qd && P->tensors[kt[h]].ldims == kd && P->tensors[vt[h]].ldims == vd &&
           SpecsEq(NaturalSpecs(C[h], p_->in_specs[C[h]]), p_->out_specs[C[h]]);
    if (!ok) return false;  // (transitions fetched above are cached; the groups reuse them)
    for (int h = 0; h < n; ++h) {
      ot[h] = NewTensor(C[h], p_->out_specs[C[h]]);
      p_->out_tensor[C[h]] = ot[h];
      p_->in_tensor[S[h]] = {qt[h], kt[h]};
      p_->in_tensor[C[h]] = {-1, vt[h]};  // the chained scores are never materialized
    }
    const int64_t sq = qd[0], sk = kd[0];
    const ChainArgs epi = ChainOf(S[0], false);
    const size_t off = Alloc(AttnChainTableBytes(n));
    Step st;
    st.kind = Step::kKernel;
    st.launches = 1;
    st.name = "attn_chain[" + std::to_string(n) + "] " + OpName(S.front()) + ".." + OpName(C.back()) +
              " (score + chain + context)";
    st.alg_flops = 2.0 * 2.0 * static_cast<double>(sq) * sk * qd[1] * n;
    std::set<int> rd;
    for (int h = 0; h < n; ++h) {
      rd.insert(qt[h]);
      rd.insert(kt[h]);
      rd.insert(vt[h]);
    }
    for (int t : rd) st.alg_bytes += static_cast<double>(P->tensors[t].bytes);
    for (int t : ot) st.alg_bytes += static_cast<double>(P->tensors[t].bytes);
    const int first = rt_->first_rank;
    st.init = [P, qt, kt, vt, ot, off, first, n, sq, sk](int li) {
      const int r = first + li;
      std::vector<const void*> q(n), k(n), v(n);
      std::vector<void*> o(n);
      for (int h = 0; h < n; ++h) {
        q[h] = P->Ptr(P->tensors[qt[h]], r);
        k[h] = P->Ptr(P->tensors[kt[h]], r);
        v[h] = P->Ptr(P->tensors[vt[h]], r);
        o[h] = P->Ptr(P->tensors[ot[h]], r);
      }
      PrepareAttnChain(n, sq, sk, q.data(), k.data(), v.data(), o.data(), P->peer_base[r] + off);
    };
    st.run = [P, epi, off, first, n, sq, sk](int li, cudaStream_t s) {
      const int r = first + li;
      LaunchAttnChain(n, sq, sk, Patch(P, epi, r), P->peer_base[r] + off, s);
      return 1;
    };
    st.reads.assign(rd.begin(), rd.end());
    st.writes = ot;
    AddStep(std::move(st));
    (void)g2;
    return true;
  }
  // Output materialization fused into the producing GEMM (dist runs): a bf16 tcgen05 GEMM (no
  // split-K) whose output is sharded by contiguous row blocks on one mesh axis and replicated on
  // the others pushes every output tile, from its epilogue, into the replicated copy of every
  // member of that axis (GemmPush; the GEMM's own barrier, fused into it, orders the pushes
  // after every member's copy is free).  The pull all-gather after the GEMM becomes a barrier
  // step (every push landed).  RH_NO_PUSH_MATERIALIZE disables.
  bool TryPushMaterialize(int o) {
    static const bool off = getenv("RH_NO_PUSH_MATERIALIZE") != nullptr;
    if (off || !rt_->dist || rt_->world <= 1 || p_->pipeline_axis >= 0) return false;
    auto it = gemm_push_.find(o);
    if (it == gemm_push_.end() || p_->out_tensor[o] < 0) return false;
    const Tensor T = p_->tensors[p_->out_tensor[o]];
    if (T.alias >= 0 || T.gdims.size() != 2) return false;
    int axis = -1;
    for (int a = 0; a < p_->n_axes; ++a) {
      const rh_spec& sp = T.specs[a];
      if (sp.kind == RH_REPLICATED) continue;
      if (sp.kind != RH_SHARD || sp.dim != 0 || axis >= 0) return false;
      if (sp.stride * mesh_[a] != T.gdims[0]) return false;  // one contiguous row block per rank
      axis = a;
    }
    if (axis < 0 || mesh_[axis] > kMaxGroup) return false;
    GemmArgs g = it->second.g;
    if (!GemmTcPushSupported(g) || g.m != T.ldims[0] || g.n != T.gdims[1]) return false;
    Specs rep(p_->n_axes, Rep());
    const int dst = NewTensor(o, rep);
    p_->mat_tensor[o] = dst;
    PushPlan& pp = *it->second.plan;
    pp.dst_t = dst;
    pp.axis = axis;
    pp.slot = p_->n_sync_slots++;
    pp.rows_local = T.ldims[0];
    p_->steps[it->second.step].name += " [+all_gather push]";
    p_->steps[it->second.step].writes.push_back(dst);
    Step st;
    st.kind = Step::kTransition;
    st.axis = axis;
    st.p2p = true;
    st.no_async = true;
    st.post_mode = 2;  // itself the barrier after the pushes
    st.sync_slot = p_->n_sync_slots++;
    st.name = "all_gather op" + std::to_string(o) + " " + SpecStr(T.specs[axis]) + "->R@" + std::to_string(axis) +
              " (materialize) [pushed by the GEMM; barrier]";
    st.launches = 1;
    rh_program* P = p_;
    const int slot = st.sync_slot;
    st.run = [P, axis, slot](int li, cudaStream_t s) {
      LaunchPeerSync(SyncOf(P, axis, slot, li), s);
      return 1;
    };
    st.writes = {dst};
    AddStep(std::move(st));
    return true;
  }
  // Reduce-scatter of a GEMM's Partial output fused into the GEMM (dist runs): a bf16 tcgen05
  // GEMM without split-K whose output goes Partial -> Shard(t, s) with one contiguous block per
  // rank (t = 0 or 1) on one axis (the others replicated) stores each partial output box, from
  // its epilogue, into the box owner's staging slot for this rank (TMA bulk stores over NVLink,
  // behind a barrier fused into the GEMM).  The transition becomes a local rank-order sum of
  // the d slots behind the usual fused barrier (every member's pushes landed): the same fp32
  // rank-order reduction and single bf16 rounding as the pull-sum, so bit-identical.
  // Opt-in (RH_PUSH_REDUCE_SCATTER=1): the fused form runs on the main stream, so in programs
  // whose reduce-scatters PlanAsync overlaps with compute (C5's backward at N=2/4) it lost more
  // than it saved (16.45 -> 18.87 ms); on C3 it saved 2 us at N=4.
  bool TryPushReduceScatter(int src, int dst, int axis, const Specs& to_specs, const char* why) {
    static const bool off = [] {
      const char* e = getenv("RH_PUSH_REDUCE_SCATTER");
      return !(e && e[0] == '1');
    }();
    if (off || !rt_->dist || rt_->world <= 1 || p_->pipeline_axis >= 0 || (p_->flags & RH_FLAG_TRANSPORT_NCCL))
      return false;
    const Tensor X = p_->tensors[src];
    const Tensor Y = p_->tensors[dst];
    const int d = mesh_[axis];
    if (X.dtype != RH_BF16 || X.ldims.size() != 2 || d > kMaxGroup) return false;
    if (X.specs[axis].kind != RH_PARTIAL || to_specs[axis].kind != RH_SHARD) return false;
    for (int a = 0; a < p_->n_axes; ++a)
      if (a != axis && (X.specs[a].kind != RH_REPLICATED || to_specs[a].kind != RH_REPLICATED)) return false;
    const int t = to_specs[axis].dim;
    if (t < 0 || t > 1 || to_specs[axis].stride * d != X.ldims[t]) return false;
    const int64_t part = X.ldims[t] / d;
    if (part % 32 || X.ldims[1 - t] % 32) return false;
    auto it = gemm_push_.find(X.op);
    if (it == gemm_push_.end() || p_->out_tensor[X.op] != src) return false;
    PushPlan& pp = *it->second.plan;
    if (pp.dst_t >= 0 || pp.scatter_dim >= 0) return false;
    const GemmArgs& g = it->second.g;
    if (!GemmTcPushSupported(g, /*single_pass=*/true) || g.m != X.ldims[0] || g.n != X.ldims[1]) return false;
    pp.scatter_dim = t;
    pp.part = part;
    pp.axis = axis;
    pp.slot = p_->n_sync_slots++;
    pp.slot_bytes = static_cast<size_t>(Prod(X.ldims)) / d * ElemBytes(X.dtype);
    pp.stage_off = Alloc(pp.slot_bytes * d);
    p_->steps[it->second.step].name += " [+reduce_scatter push]";
    // the transition: sum of the d staged slots (local memory) in rank order into Y
    Step st;
    st.kind = Step::kTransition;
    st.axis = axis;
    st.p2p = true;
    st.no_async = true;
    st.post_mode = 2;  // peers rewrite this rank's staging only after its next GEMM's barrier
    if (rt_->dist && rt_->world > 1) st.sync_slot = p_->n_sync_slots++;
    st.name = std::string("reduce_scatter op") + std::to_string(X.op) + " P->" + SpecStr(to_specs[axis]) + "@" +
              std::to_string(axis) + " (" + why + ") [pushed by the GEMM; local sum]";
    st.alg_bytes = static_cast<double>(Y.elems()) * ElemBytes(X.dtype) * (d + 1);
    st.launches = 1;
    rh_program* P = p_;
    const Dims YD = Y.ldims;
    const rh_spec rp{RH_PARTIAL, -1, 0}, rr = Rep();
    const AxisView pv = MakeAxisView(rp, static_cast<int>(YD.size()), YD.data(), d);
    const AxisView rv = MakeAxisView(rr, static_cast<int>(YD.size()), YD.data(), d);
    const size_t soff = pp.stage_off, sb = pp.slot_bytes;
    const int dtype = X.dtype;
    st.pulls.push_back([P, dst, axis, soff, sb, pv, rv, dtype, d](int li) {
      const int g2 = P->mesh->rt->first_rank + li;
      PullArgs a{};
      a.dst = P->Ptr(P->tensors[dst], g2);
      for (int k = 0; k < d; ++k) a.src[k] = P->peer_base[g2] + soff + static_cast<size_t>(k) * sb;  // local slots
      a.from = pv;
      a.to = rv;
      a.coord = P->mesh->Coords(g2)[axis];
      a.n_dst = P->tensors[dst].elems();
      a.dtype = dtype;
      return a;
    });
    st.reads = {};
    st.writes = {dst};
    AddStep(std::move(st));
    return true;
  }
  struct GemmPushRef {
    std::shared_ptr<PushPlan> plan;
    GemmArgs g;
    int step;
  };
  std::map<int, GemmPushRef> gemm_push_;  // op whose value a tcgen05 GEMM step writes -> its push plan

  std::vector<int> attn_pair_;                 // score group -> context group (-1: none)
  std::vector<bool> attn_done_;                // context group emitted inside its score group's kernel
  std::map<int, std::vector<int>> attn_ctx_;   // score group -> context members, score order

  std::vector<int> group_of_;             // op -> grouped GEMM id (-1: none)
  std::vector<std::vector<int>> groups_;  // members in schedule order

  // Rematerialization of forward tanh values (bf16 chain programs).  y = T^p(b), a run of p
  // tanh ops from a base b whose value is stored, is one ladder-table column away from b (the
  // table composes the per-op rounding: bit-identical).  A chain program that reads such y's
  // reads b instead (EwArgs::vlad_*), and a forward chain member y whose every outside consumer
  // does so is no longer stored.  RH_REMAT=0 disables (A/B), RH_REMAT=1 forces it on.
  struct Remat {
    int base = -1;
    Specs spec;
    std::vector<int> col;     // per chain input: ladder column, -1 = read as is
    std::vector<int> powers;  // per column
  };
  template <typename NoPartial>
  void PlanRemat(const std::vector<bool>& is_out, NoPartial no_partial) {
    const int n = static_cast<int>(p_->ops.size());
    remat_.assign(ew_.size(), Remat{});
    // Default on.  The round-1 C5 N=2 hang seen with it did not reproduce after this round's
    // barrier / transition changes (N=2 and N=4 benches and the dist parity suite run with it,
    // DESIGN §8); every cross-GPU wait is bounded, so a recurrence fails as RH_ERR_TIMEOUT
    // instead of hanging.  RH_REMAT=0 disables it (A/B).
    const char* env = getenv("RH_REMAT");
    const bool on = env ? env[0] != '0' : true;
    if (!on || ew_.empty() || (p_->flags & RH_FLAG_KEEP_ALL)) return;
    if (p_->ops[0].dtype != RH_BF16) return;
    // GEMM-epilogue tails: their value is the fused kernel's stored output (a base, not a
    // rematerialized value: the pre-epilogue value does not exist)
    std::vector<bool> epi_tail(n, false);
    for (int h = 0; h < n; ++h)
      if (Tail(h) != h) epi_tail[Tail(h)] = true;
    std::vector<int> base_of(n, -1), pow_of(n, 0);
    for (int m : p_->order) {
      if (!IsElementwiseUnary(m) || UnaryFn(m) != RH_FN_TANH || p_->ops[m].dtype != RH_BF16) continue;
      const int in = p_->inputs[m][0];
      if (!SpecsEq(p_->in_specs[m][0], p_->out_specs[in]) || !SpecsEq(p_->out_specs[m], p_->out_specs[in]) ||
          !no_partial(p_->out_specs[m]) || GDims(m) != GDims(in))
        continue;
      if (pow_of[in] > 0 && !epi_tail[in]) {
        base_of[m] = base_of[in];
        pow_of[m] = pow_of[in] + 1;
      } else {
        base_of[m] = in;
        pow_of[m] = 1;
      }
    }
    auto member_pos = [&](int op) {
      const auto& c = ew_[ew_of_[op]];
      for (size_t j = 0; j < c.members.size(); ++j)
        if (c.members[j] == op) return static_cast<int>(j);
      return -1;
    };
    // the base's value must exist as a tensor: a source, an unfused kernel output (no epilogue
    // chain), or a stored chain-program member
    auto base_ok = [&](int b) {
      if (b < 0 || !chain_[b].empty()) return false;
      if (absorbed_[b]) return static_cast<bool>(epi_tail[b]);
      if (ew_of_[b] >= 0) return static_cast<bool>(ew_[ew_of_[b]].stored[member_pos(b)]);
      return true;
    };
    std::vector<bool> requested(n, false);
    for (const auto& rq : p_->requests) requested[rq.first] = true;
    for (size_t ci = 0; ci < ew_.size(); ++ci) {
      const EwPlan& c = ew_[ci];
      std::map<int, int> votes;
      for (const auto& in : c.inputs)
        if (pow_of[in.first] > 0 && SpecsEq(in.second, p_->out_specs[in.first]) && base_ok(base_of[in.first]))
          ++votes[base_of[in.first]];
      int b = -1, best = 0;
      for (auto& kv : votes)
        if (kv.second > best) {
          best = kv.second;
          b = kv.first;
        }
      if (b < 0 || StageOfOp(b) != StageOfOp(c.members.front())) continue;
      Remat r;
      r.base = b;
      r.spec = p_->out_specs[b];
      r.col.assign(c.inputs.size(), -1);
      // ladder columns in ascending power (TanhLadderTable composes column to column)
      std::set<int> pw;
      for (size_t k = 0; k < c.inputs.size(); ++k) {
        const int y = c.inputs[k].first;
        if (base_of[y] == b && pow_of[y] > 0 && SpecsEq(c.inputs[k].second, p_->out_specs[y]) &&
            (static_cast<int>(pw.size()) < kLadderWidth || pw.count(pow_of[y])))
          pw.insert(pow_of[y]);
      }
      r.powers.assign(pw.begin(), pw.end());
      for (size_t k = 0; k < c.inputs.size(); ++k) {
        const int y = c.inputs[k].first;
        if (base_of[y] != b || pow_of[y] <= 0 || !SpecsEq(c.inputs[k].second, p_->out_specs[y])) continue;
        const auto it = std::find(r.powers.begin(), r.powers.end(), pow_of[y]);
        if (it != r.powers.end()) r.col[k] = static_cast<int>(it - r.powers.begin());
      }
      remat_[ci] = std::move(r);
    }
    // forward members no longer stored: every consumer outside their own chain rematerializes
    std::vector<std::vector<int>> cons(n);
    for (int i = 0; i < n; ++i)
      for (int sidx : p_->inputs[i]) cons[sidx].push_back(i);
    for (size_t fi = 0; fi < ew_.size(); ++fi) {
      EwPlan& f = ew_[fi];
      for (size_t j = 0; j + 1 < f.members.size(); ++j) {
        const int y = f.members[j];
        if (!f.stored[j] || pow_of[y] <= 0 || is_out[y] || requested[y]) continue;
        bool all = true;
        for (int cn : cons[y]) {
          if (ew_of_[cn] == static_cast<int>(fi)) continue;
          if (ew_of_[cn] < 0) {
            if (getenv("RH_REMAT_DEBUG"))
              fprintf(stderr, "remat: %s kept: consumer %s not in a chain program\n", OpName(y).c_str(), OpName(cn).c_str());
            all = false;
            break;
          }
          const Remat& r = remat_[ew_of_[cn]];
          const auto& ci = ew_[ew_of_[cn]].inputs;
          bool covered = false;
          for (size_t k = 0; k < ci.size(); ++k)
            if (ci[k].first == y && r.col.size() > k && r.col[k] >= 0) covered = true;
          if (!covered && getenv("RH_REMAT_DEBUG"))
            fprintf(stderr, "remat: %s kept: chain of %s (base %s) does not cover it\n", OpName(y).c_str(),
                    OpName(cn).c_str(), r.base >= 0 ? OpName(r.base).c_str() : "-");
          all = all && covered;
        }
        if (all) f.stored[j] = false;
        if (all && getenv("RH_REMAT_DEBUG")) fprintf(stderr, "remat: %s not stored\n", OpName(y).c_str());
      }
    }
  }

  // Dist runs: a topological order that computes the producers of resharded values as soon as
  // they are ready (ties: the load order), and emits their transitions right after them
  // (EagerTransitions), so that independent compute lands between a transition and its first
  // consumer — PlanAsync then moves the transition to the side stream (at N=2 the all-gather of
  // v runs under the q / k / score GEMMs).  Any topological order computes the same values.
  void TransitionFirstOrder() {
    const int n = static_cast<int>(p_->ops.size());
    std::vector<int> pos(n), indeg(n, 0);
    for (int k = 0; k < n; ++k) pos[p_->order[k]] = k;
    std::vector<std::vector<int>> cons(n);
    std::vector<char> tprod(n, 0);
    for (int c = 0; c < n; ++c)
      for (size_t sl = 0; sl < p_->inputs[c].size(); ++sl) {
        const int i = p_->inputs[c][sl];
        ++indeg[c];
        cons[i].push_back(c);
        if (!SpecsEq(p_->in_specs[c][sl], p_->out_specs[i])) tprod[i] = 1;
      }
    // lead: load position of the earliest resharded value an op leads to (itself included): the
    // producers of resharded values first, then the ops feeding the next transition, so that
    // independent ones fill its wait
    std::vector<int> lead(n, n);
    for (int k = n - 1; k >= 0; --k) {
      const int i = p_->order[k];
      if (tprod[i]) lead[i] = pos[i];
      for (int c : cons[i]) lead[i] = std::min(lead[i], lead[c]);
    }
    // ready set ordered by (not a resharded producer, lead, load position)
    auto key = [&](int i) { return std::make_pair((tprod[i] ? 0 : n + 1) + lead[i], pos[i]); };
    std::set<std::pair<int, int>> ready;
    for (int i = 0; i < n; ++i)
      if (!indeg[i]) ready.insert(key(i));
    std::vector<int> order;
    order.reserve(n);
    while (!ready.empty()) {
      const int i = p_->order[ready.begin()->second];
      ready.erase(ready.begin());
      order.push_back(i);
      for (int c : cons[i])
        if (--indeg[c] == 0) ready.insert(key(c));
    }
    if (static_cast<int>(order.size()) == n) p_->order = order;
  }

  // Emit now every transition a consumer of `prod` will fetch (GetTensor caches it for the
  // consumer).  Folded transposes fetch their input in the permuted spec and are left alone.
  void EagerTransitions(int prod) {
    if (p_->out_tensor[prod] < 0) return;
    if (users_.empty()) {
      users_.resize(p_->ops.size());
      for (size_t c = 0; c < p_->ops.size(); ++c)
        for (int i : p_->inputs[c]) users_[i].push_back(static_cast<int>(c));
    }
    for (int c : users_[prod]) {
      if (absorbed_[c]) continue;  // fused consumers read inside their kernel; folded transposes
      for (size_t sl = 0; sl < p_->inputs[c].size(); ++sl)
        if (p_->inputs[c][sl] == prod && !SpecsEq(p_->in_specs[c][sl], p_->out_specs[prod]) &&
            !(sl < 2 && !fold_t_.empty() && fold_t_[c][sl]))
          GetTensor(prod, p_->in_specs[c][sl], "edge");
    }
  }
  std::vector<std::vector<int>> users_;

  // A 2-D transpose whose only consumer is a MatMul folds into the GEMM's operand layout (the
  // tcgen05 / SIMT kernels read K-major and MN-major operands straight from the buffer): the
  // MatMul fetches the transpose's input in the permuted spec — the local buffer of a
  // block-cyclic layout transposes with the tensor, Shard(p, s) of the output <-> Shard(perm[p],
  // s) of the input — and flips its transpose flag.  No transpose kernel, no extra buffer.
  void PlanTransposeFold(const std::vector<int>& uses, const std::vector<int>& consumer,
                         const std::vector<bool>& is_out) {
    const int n = static_cast<int>(p_->ops.size());
    fold_t_.assign(n, {false, false});
    static const bool off = getenv("RH_NO_TRANSPOSE_FOLD") != nullptr;  // A/B knob (profiles/)
    if (off) return;
    (void)uses;
    (void)consumer;
    std::vector<std::vector<int>> users(n);
    for (int i = 0; i < n; ++i)
      for (int s : p_->inputs[i]) users[s].push_back(i);
    for (int t = 0; t < n; ++t) {
      const rh_op& op = p_->ops[t];
      if (op.kind != RH_OP_TRANSPOSE || op.rank != 2 || users[t].empty() || is_out[t] || absorbed_[t]) continue;
      if (EffPerm(op, 2) != std::vector<int>{1, 0}) continue;
      // every consumer must be a MatMul reading it in exactly one slot (the forward score GEMM
      // and the backward's gradient GEMMs all read k^T)
      bool ok = true;
      for (int c : users[t]) {
        const auto& ins = p_->inputs[c];
        ok = ok && p_->ops[c].kind == RH_OP_MATMUL && !absorbed_[c] && p_->ops[c].dtype == op.dtype &&
             ins.size() == 2 && ins[0] != ins[1] && StageOfOp(c) == StageOfOp(t);
      }
      if (!ok) continue;
      for (int c : users[t]) fold_t_[c][p_->inputs[c][0] == t ? 0 : 1] = true;
      absorbed_[t] = true;
    }
  }

  // Spec of the transpose's input that matches spec `s` of its (2-D, perm [1,0]) output.
  static Specs Transposed(const Specs& s) {
    Specs o = s;
    for (auto& x : o)
      if (x.kind == RH_SHARD) x.dim = 1 - x.dim;
    return o;
  }

  bool IsEw(int i) const {
    const int k = p_->ops[i].kind;
    return IsElementwiseUnary(i) || k == RH_OP_ADD || k == RH_OP_MUL;
  }

  // Elementwise chains (kernels.h EwArgs).  Greedy over the schedule order: a chain starts at an
  // elementwise op and follows the accumulator to the EARLIEST elementwise consumer whose edge
  // needs no resharding; the consumer's other operand is an external input, the kept register
  // (an earlier chain value) or the accumulator itself.  Chain values with consumers outside the
  // chain are stored.  The kernel runs at the tail's position, so a chain may only grow while
  // every outside consumer of its values comes after the new tail (which also guarantees that
  // no external input depends on a chain value).  A chain that is a plain single-use unary run
  // behind one op is handed to the classic head + chain kernels (chain_).
  template <typename NatOk, typename NoPartial>
  void PlanEwChains(const std::vector<bool>& is_out, NatOk natural_ok, NoPartial no_partial) {
    const int n = static_cast<int>(p_->ops.size());
    std::vector<std::vector<int>> cons(n);
    for (int i = 0; i < n; ++i)
      for (int s : p_->inputs[i])
        if (cons[s].empty() || cons[s].back() != i) cons[s].push_back(i);
    std::vector<int> pos(n, 0);
    for (size_t k = 0; k < p_->order.size(); ++k) pos[p_->order[k]] = static_cast<int>(k);
    ew_of_.assign(n, -1);
    const bool bf16_prog = !p_->ops.empty() && p_->ops[0].dtype == RH_BF16;
    (void)bf16_prog;
    for (int h : p_->order) {
      if (!IsEw(h) || absorbed_[h] || ew_of_[h] >= 0 || !natural_ok(h)) continue;
      EwPlan c;
      c.members = {h};
      auto add_input = [&](int prod, const Specs& sp) {
        for (size_t k = 0; k < c.inputs.size(); ++k)
          if (c.inputs[k].first == prod && SpecsEq(c.inputs[k].second, sp)) return static_cast<int>(k);
        c.inputs.emplace_back(prod, sp);
        return static_cast<int>(c.inputs.size()) - 1;
      };
      {
        std::vector<int> src;
        for (size_t sl = 0; sl < p_->inputs[h].size(); ++sl) src.push_back(add_input(p_->inputs[h][sl], p_->in_specs[h][sl]));
        if (src.size() == 2 && src[1] == src[0]) src[1] = kEwSrcAcc;
        c.src.push_back(src);
      }
      c.keep_after.push_back(false);
      int cur = h, kept = -1, last_keep_use = -1;
      auto member_index = [&](int op) {
        for (size_t j = 0; j < c.members.size(); ++j)
          if (c.members[j] == op) return static_cast<int>(j);
        return -1;
      };
      while (static_cast<int>(c.members.size()) < kMaxChain) {
        if (!no_partial(p_->out_specs[cur])) break;
        // successor: the earliest qualifying elementwise consumer of the accumulator
        int v = -1;
        for (int cand : cons[cur]) {
          if (!IsEw(cand) || absorbed_[cand] || ew_of_[cand] >= 0 || member_index(cand) >= 0) continue;
          if (p_->ops[cand].dtype != p_->ops[h].dtype || GDims(cand) != GDims(cur) || !natural_ok(cand)) continue;
          if (!SameTask(cand, h)) continue;
          bool edge_ok = false;
          for (size_t sl = 0; sl < p_->inputs[cand].size(); ++sl)
            if (p_->inputs[cand][sl] == cur && SpecsEq(p_->in_specs[cand][sl], p_->out_specs[cur])) edge_ok = true;
          if (!edge_ok) continue;
          if (v < 0 || pos[cand] < pos[v]) v = cand;
        }
        if (v < 0) break;
        // operands of v
        EwPlan t = c;
        int t_kept = kept, t_last = last_keep_use;
        const int vi = static_cast<int>(t.members.size());
        std::vector<int> src;
        bool acc_used = false, ok = true;
        for (size_t sl = 0; sl < p_->inputs[v].size() && ok; ++sl) {
          const int pr = p_->inputs[v][sl];
          const int j = member_index(pr);
          if (pr == cur && SpecsEq(p_->in_specs[v][sl], p_->out_specs[cur])) {
            src.push_back(acc_used ? kEwSrcAcc : -1);
            acc_used = true;
          } else if (j >= 0) {
            if (!SpecsEq(p_->in_specs[v][sl], p_->out_specs[pr])) { ok = false; break; }
            if (t_kept != j) {
              if (t_last > j) { ok = false; break; }
              t.keep_after[j] = true;
              t_kept = j;
            }
            t_last = vi;
            src.push_back(kEwSrcKeep);
          } else {
            EwPlan* tp = &t;
            int k = -1;
            for (size_t q = 0; q < tp->inputs.size(); ++q)
              if (tp->inputs[q].first == pr && SpecsEq(tp->inputs[q].second, p_->in_specs[v][sl])) k = static_cast<int>(q);
            if (k < 0) {
              tp->inputs.emplace_back(pr, p_->in_specs[v][sl]);
              k = static_cast<int>(tp->inputs.size()) - 1;
            }
            src.push_back(k);
          }
        }
        if (!ok || !acc_used || static_cast<int>(t.inputs.size()) > kMaxEwIn) break;
        // the accumulator operand goes first (ops are commutative; bf16/fp32 results identical)
        if (src.size() == 2 && src[0] != -1) std::swap(src[0], src[1]);
        t.members.push_back(v);
        t.src.push_back(src);
        t.keep_after.push_back(false);
        // schedule check + output / code budget
        std::vector<bool> in_chain(n, false);
        for (int m : t.members) in_chain[m] = true;
        int stores = 0, code = 1;
        bool order_ok = true;
        for (size_t j = 0; j < t.members.size(); ++j) {
          const int m = t.members[j];
          bool outside = is_out[m] || j + 1 == t.members.size();
          for (int cns : cons[m])
            if (!in_chain[cns]) {
              outside = true;
              if (pos[cns] < pos[v]) order_ok = false;
            }
          stores += outside;
          code += 2 + (outside ? 1 : 0) + (t.keep_after[j] ? 1 : 0);
        }
        if (!order_ok || stores > kMaxEwOut || code > kMaxEwCode) break;
        c = std::move(t);
        kept = t_kept;
        last_keep_use = t_last;
        cur = v;
      }
      if (c.members.size() < 2) continue;
      // stored values
      std::vector<bool> in_chain(n, false);
      for (int m : c.members) in_chain[m] = true;
      c.stored.assign(c.members.size(), false);
      for (size_t j = 0; j < c.members.size(); ++j) {
        const int m = c.members[j];
        bool st = is_out[m] || j + 1 == c.members.size();
        for (int cns : cons[m]) st = st || !in_chain[cns];
        c.stored[j] = st;
      }
      // classic form: one op then single-use unary ops, only the tail stored
      bool classic = true;
      for (size_t j = 1; j < c.members.size(); ++j)
        classic = classic && IsElementwiseUnary(c.members[j]) && !c.stored[j - 1] && !c.keep_after[j - 1];
      if (classic) {
        for (size_t j = 1; j < c.members.size(); ++j) {
          chain_[h].push_back(c.members[j]);
          absorbed_[c.members[j]] = true;
        }
        continue;
      }
      const int id = static_cast<int>(ew_.size());
      for (int m : c.members) ew_of_[m] = id;
      ew_.push_back(std::move(c));
    }
  }
  static constexpr size_t kMaxGemmEpilogue = 2;

  int UnaryFn(int i) const {
    int fn = p_->ops[i].fn;
    if (fn == RH_FN_UNLABELED)
      fn = (p_->flags & RH_FLAG_UNLABELED_IDENTITY) ? RH_FN_IDENTITY : RH_FN_TANH;
    return fn;
  }

  ChainArgs ChainOf(int h, bool include_head) {
    std::vector<int> fns;
    if (include_head) fns.push_back(UnaryFn(h));
    for (int v : chain_[h]) fns.push_back(UnaryFn(v));
    ChainArgs c{};
    const bool bf16 = p_->ops[h].dtype == RH_BF16;
    for (size_t i = 0; i < fns.size();) {
      size_t j = i;
      while (j < fns.size() && fns[j] == RH_FN_TANH) ++j;
      if (bf16 && j > i && c.n_tab < kMaxTanhRuns) {  // run of tanh -> one T^k lookup
        c.tab_off[c.n_tab] = TanhTable(static_cast<int>(j - i));
        c.fns[c.n_fn++] = kFnTanhRun + c.n_tab;
        ++c.n_tab;
        i = j;
      } else {
        c.fns[c.n_fn++] = fns[i++];
      }
    }
    return c;
  }

  // Arena offset of the tanh ladder table for these cumulative powers (TanhLadderTable).
  size_t LadderTable(const std::vector<int>& powers) {
    auto it = ladder_tables_.find(powers);
    if (it != ladder_tables_.end()) return it->second;
    std::vector<uint16_t> tab(static_cast<size_t>(kTanhRunEntries) * kLadderWidth);
    TanhLadderTable(powers.data(), static_cast<int>(powers.size()), tab.data());
    const size_t off = Alloc(tab.size() * 2);
    p_->uploads.emplace_back(off, std::vector<char>(reinterpret_cast<char*>(tab.data()),
                                                    reinterpret_cast<char*>(tab.data()) + tab.size() * 2));
    ladder_tables_[powers] = off;
    return off;
  }

  // Arena offset of the T^k table (uploaded to every rank's arena after allocation).
  size_t TanhTable(int k) {
    auto it = tanh_tables_.find(k);
    if (it != tanh_tables_.end()) return it->second;
    std::vector<uint16_t> tab(kTanhRunEntries);
    TanhRunTable(k, tab.data());
    const size_t off = Alloc(tab.size() * 2);
    p_->uploads.emplace_back(off, std::vector<char>(reinterpret_cast<char*>(tab.data()),
                                                    reinterpret_cast<char*>(tab.data()) + tab.size() * 2));
    tanh_tables_[k] = off;
    return off;
  }

 public:
  // The chain with its tables' device pointers for global rank r.
  static ChainArgs Patch(const rh_program* P, const ChainArgs& c, int r) {
    ChainArgs o = c;
    for (int t = 0; t < c.n_tab; ++t)
      o.tab[t] = reinterpret_cast<const uint16_t*>(P->peer_base[r] + c.tab_off[t]);
    return o;
  }

 private:

  std::string OpName(int i) const { return "op" + std::to_string(i); }

  void AddStep(Step s) {
    if (s.stage == -1) s.stage = cur_stage_;  // pipeline programs: run by the current op's stage
    p_->steps.push_back(std::move(s));
  }

  void EmitOp(int i) {
    const rh_op& op = p_->ops[i];
    const int nin = static_cast<int>(p_->inputs[i].size());
    std::vector<int> in_t(nin);
    for (int s = 0; s < nin; ++s) {
      if (s < 2 && !fold_t_.empty() && fold_t_[i][s]) {  // folded transpose: its input, permuted spec
        const int t = p_->inputs[i][s];
        in_t[s] = GetTensor(p_->inputs[t][0], Transposed(p_->in_specs[i][s]), "edge");
      } else {
        in_t[s] = GetTensor(p_->inputs[i][s], p_->in_specs[i][s], "edge");
      }
    }
    p_->in_tensor[i] = in_t;
    for (int s = 0; s < nin && s < 2; ++s)
      if (!fold_t_.empty() && fold_t_[i][s]) p_->in_tensor[i][s] = -1;  // not materialized
    const Specs nat = NaturalSpecs(i, p_->in_specs[i]);
    const int tail = Tail(i);
    const bool direct = SpecsEq(nat, p_->out_specs[i]);
    if (tail != i && !direct) Fail("internal: fused head without a natural spec");
    // Reshape: pass-through layouts keep the local buffer byte-identical -> alias, no kernel.
    if (op.kind == RH_OP_RESHAPE) {
      int t = NewTensor(i, nat, /*alloc=*/false);
      p_->tensors[t].alias = in_t[0];
      p_->out_tensor[i] = t;
      if (!direct) p_->out_tensor[i] = GetTensor(i, p_->out_specs[i], "pin");
      return;
    }
    const int out_t = NewTensor(tail, nat);
    if (tail != i) {  // intermediate members of the chain have no buffer
      p_->tensors[out_t].gdims = GDims(i);
    }
    EmitKernel(i, in_t, out_t);
    p_->out_tensor[tail] = out_t;
    if (!direct) {  // pinned op without a rule: computed replicated, then sliced (sharding.cpp:477-487)
      p_->out_tensor[i] = out_t;
      p_->out_tensor[i] = GetTensor(i, p_->out_specs[i], "pin");
    }
  }

  void EmitEwChain(const EwPlan& c) {
    rh_program* P = p_;
    const int h = c.members.front();
    const int dtype = P->ops[h].dtype;
    const bool bf16 = dtype == RH_BF16;
    // operand code of each chain input: its in_t index, or kEwSrcVirt + ladder column
    const int ci = ew_of_[h];
    const Remat* rm = ci >= 0 && ci < static_cast<int>(remat_.size()) && remat_[ci].base >= 0 ? &remat_[ci] : nullptr;
    std::vector<int> in_t, opnd(c.inputs.size(), -1);
    int vbase = -1;
    for (size_t k = 0; k < c.inputs.size(); ++k) {
      if (rm && rm->col[k] >= 0) {
        opnd[k] = kEwSrcVirt + rm->col[k];
        continue;
      }
      opnd[k] = static_cast<int>(in_t.size());
      in_t.push_back(GetTensor(c.inputs[k].first, c.inputs[k].second, "edge"));
      if (rm && c.inputs[k].first == rm->base && SpecsEq(c.inputs[k].second, rm->spec)) vbase = opnd[k];
    }
    if (rm && vbase < 0) {
      vbase = static_cast<int>(in_t.size());
      in_t.push_back(GetTensor(rm->base, rm->spec, "edge"));
    }
    if (static_cast<int>(in_t.size()) > kMaxEwIn) Fail("internal: rematerialized chain has too many inputs");
    auto opx = [&](int v) { return v >= 0 && v < kEwSrcKeep ? opnd[v] : v; };
    // tensors of the stored values
    std::vector<int> out_t;
    std::vector<int> out_slot(c.members.size(), -1);
    for (size_t j = 0; j < c.members.size(); ++j) {
      if (!c.stored[j]) continue;
      const int m = c.members[j];
      const int t = NewTensor(m, p_->out_specs[m]);
      p_->out_tensor[m] = t;
      out_slot[j] = static_cast<int>(out_t.size());
      out_t.push_back(t);
    }
    for (int m : c.members) {
      std::vector<int> ins;
      for (size_t sl = 0; sl < p_->inputs[m].size(); ++sl) {
        auto it = cache_.find(Key(p_->inputs[m][sl], p_->in_specs[m][sl], cur_stage_));
        ins.push_back(it != cache_.end() ? it->second : -1);
      }
      p_->in_tensor[m] = ins;
    }
    // tanh runs (bf16): maximal runs of tanh members whose intermediate values are neither
    // stored nor kept become one T^k lookup; at most kMaxTanhRuns distinct k per kernel (other
    // lengths decompose into T^1 lookups)
    std::vector<int> run_len(c.members.size(), 0);  // at a run's first member
    std::vector<bool> in_run(c.members.size(), false);
    std::map<int, int> len_count;
    if (bf16) {
      for (size_t j = 0; j < c.members.size();) {
        if (!(IsElementwiseUnary(c.members[j]) && UnaryFn(c.members[j]) == RH_FN_TANH)) {
          ++j;
          continue;
        }
        size_t k = j;
        while (k + 1 < c.members.size() && !c.stored[k] && !c.keep_after[k] &&
               IsElementwiseUnary(c.members[k + 1]) && UnaryFn(c.members[k + 1]) == RH_FN_TANH)
          ++k;
        run_len[j] = static_cast<int>(k - j + 1);
        for (size_t q = j; q <= k; ++q) in_run[q] = true;
        ++len_count[run_len[j]];
        j = k + 1;
      }
    }
    EwArgs a{};
    std::map<int, int> table_of;  // run length -> table slot
    auto table = [&](int k) {
      auto it = table_of.find(k);
      if (it != table_of.end()) return it->second;
      const int slot = a.n_tab++;
      a.tab_off[slot] = TanhTable(k);
      table_of[k] = slot;
      return slot;
    };
    if (bf16 && !len_count.empty()) {
      std::vector<std::pair<int, int>> by_count;
      for (auto& kv : len_count) by_count.emplace_back(-kv.second, kv.first);
      std::sort(by_count.begin(), by_count.end());
      if (static_cast<int>(by_count.size()) > kMaxTanhRuns) table(1);
      for (auto& bc : by_count)
        if (a.n_tab < kMaxTanhRuns) table(bc.second);
    }
    std::vector<int32_t> code;
    auto emit_after = [&](size_t j) {
      if (out_slot[j] >= 0) code.push_back(EwIns(kEwStore, out_slot[j]));
      if (c.keep_after[j]) code.push_back(EwIns(kEwKeep, 0));
    };
    for (size_t j = 0; j < c.members.size(); ++j) {
      const int m = c.members[j];
      const auto& src = c.src[j];
      if (j == 0) code.push_back(EwIns(kEwLoad, opx(src[0])));
      if (IsElementwiseUnary(m)) {
        if (bf16 && in_run[j]) {
          if (run_len[j] == 0) continue;  // inside a run: covered by its first member
          const int k = run_len[j];
          if (table_of.count(k)) {
            code.push_back(EwIns(kEwUnary, kFnTanhRun + table_of[k]));
          } else {
            for (int q = 0; q < k; ++q) code.push_back(EwIns(kEwUnary, kFnTanhRun + table_of.at(1)));
          }
          emit_after(j + k - 1);
          continue;
        }
        code.push_back(EwIns(kEwUnary, UnaryFn(m)));
      } else {
        const int other = j == 0 ? src[1] : (src[0] == -1 ? src[1] : src[0]);
        code.push_back(EwIns(p_->ops[m].kind == RH_OP_MUL ? kEwMul : kEwAdd, opx(other)));
      }
      emit_after(j);
    }
    // peephole for the tanh backward (dy - (dy*y)*y), same roundings in one instruction:
    //   KEEP, MUL k, MUL k, UNARY neg, ADD keep      ->  TBWD k
    //   LOAD b, MUL k, MUL k, UNARY neg, ADD b       ->  LOAD b, TBWD k   (TBWD also sets keep:
    //                                                    only when no later instruction reads the
    //                                                    old keep before the next KEEP)
    auto keep_read_later = [&](size_t from) {
      for (size_t q = from; q < code.size(); ++q) {
        if (code[q] == EwIns(kEwKeep, 0)) return false;
        const int op = code[q] & 0xff;
        if ((op == kEwAdd || op == kEwMul) && (code[q] >> 8) == kEwSrcKeep) return true;
      }
      return false;
    };
    for (size_t q = 0; q + 4 < code.size(); ++q) {
      const int32_t m = code[q + 1];
      const bool mm = (m & 0xff) == kEwMul && ((m >> 8) < kMaxEwIn || (m >> 8) >= kEwSrcVirt) && code[q + 2] == m &&
                      code[q + 3] == EwIns(kEwUnary, RH_FN_NEG);
      if (!mm) continue;
      if (code[q] == EwIns(kEwKeep, 0) && code[q + 4] == EwIns(kEwAdd, kEwSrcKeep)) {
        code[q] = EwIns(kEwTanhBwd, m >> 8);
        code.erase(code.begin() + q + 1, code.begin() + q + 5);
      } else if ((code[q] & 0xff) == kEwLoad && code[q + 4] == EwIns(kEwAdd, code[q] >> 8) &&
                 !keep_read_later(q + 5)) {
        code[q + 1] = EwIns(kEwTanhBwd, m >> 8);
        code.erase(code.begin() + q + 2, code.begin() + q + 5);
      }
    }
    // runs of TBWD on descending consecutive ladder columns -> one unrolled instruction
    if (rm && !getenv("RH_REMAT_NO_RUNS")) {
      std::vector<int32_t> fused;
      for (size_t q = 0; q < code.size();) {
        const int op = code[q] & 0xff, arg = code[q] >> 8;
        size_t e = q + 1;
        if (op == kEwTanhBwd && arg >= kEwSrcVirt) {
          while (e < code.size() && (code[e] & 0xff) == kEwTanhBwd &&
                 (code[e] >> 8) == arg - static_cast<int>(e - q))
            ++e;
        }
        if (e - q >= 2) {
          fused.push_back(EwIns(kEwTanhBwdLad, (arg - kEwSrcVirt) | (static_cast<int>(e - q) << 4)));
        } else {
          fused.push_back(code[q]);
          e = q + 1;
        }
        q = e;
      }
      code.swap(fused);
    }
    if (static_cast<int>(code.size()) > kMaxEwCode) Fail("internal: elementwise chain code too long");
    // tanh ladder (bf16): the maximal suffix of tanh runs and stores, from its first tanh run
    // on (stores before it belong to the prefix), with >= 3 stores -> one ladder-table row per
    // element (EwArgs::lad_*).  The full code stays for the scalar tail.
    a.lad_pc = static_cast<int32_t>(code.size());
    static const bool no_ladder = getenv("RH_NO_LADDER") != nullptr;  // A/B knob (profiles/)
    if (bf16 && !no_ladder) {
      std::map<int, int> k_of_slot;
      for (auto& kv : table_of) k_of_slot[kv.second] = kv.first;
      size_t q = code.size();
      while (q > 0) {
        const int op = code[q - 1] & 0xff, arg = code[q - 1] >> 8;
        if (op == kEwStore || op == kEwKeep || (op == kEwUnary && arg >= kFnTanhRun)) --q;
        else break;
      }
      while (q < code.size() && (code[q] & 0xff) != kEwUnary) ++q;
      std::vector<int> powers, outs;
      int cum = 0;
      for (size_t z = q; z < code.size(); ++z) {
        const int op = code[z] & 0xff, arg = code[z] >> 8;
        if (op == kEwUnary) cum += k_of_slot.at(arg - kFnTanhRun);
        else if (op == kEwStore) {
          powers.push_back(cum);
          outs.push_back(arg);
        }
      }
      if (q > 0 && powers.size() >= 3 && powers.size() <= static_cast<size_t>(kLadderWidth)) {
        a.lad_pc = static_cast<int32_t>(q);
        a.lad_n = static_cast<int32_t>(powers.size());
        std::copy(outs.begin(), outs.end(), a.lad_out);
        a.lad_off = LadderTable(powers);
      }
    }
    if (rm) {
      a.vlad_in = vbase;
      a.vlad_n = static_cast<int32_t>(rm->powers.size());
      a.vlad_off = LadderTable(rm->powers);
    }
    a.n_code = static_cast<int32_t>(code.size());
    a.n_in = static_cast<int32_t>(in_t.size());
    std::copy(code.begin(), code.end(), a.code);
    a.n = P->tensors[out_t[0]].elems();
    a.jit = EwJitRegister(a, dtype);  // compiled with the program's other chains (EwJitBuild)
    Step st;
    st.kind = Step::kKernel;
    st.launches = 1;
    st.name = "ew_chain " + OpName(h) + ".." + OpName(c.members.back()) + " (" +
              std::to_string(c.members.size()) + " ops, " + std::to_string(in_t.size()) + " in, " +
              std::to_string(out_t.size()) + " out)" + (a.lad_n ? " [ladder]" : "") +
              (a.vlad_n ? " [remat " + std::to_string(a.vlad_n) + "]" : "");
    for (int t : in_t) st.alg_bytes += static_cast<double>(P->tensors[t].bytes);
    for (int t : out_t) st.alg_bytes += static_cast<double>(P->tensors[t].bytes);
    const int first = rt_->first_rank;
    st.run = [P, a, in_t, out_t, first, dtype](int li, cudaStream_t s) {
      const int r = first + li;
      EwArgs x = a;
      for (size_t k = 0; k < in_t.size(); ++k) x.in[k] = P->Ptr(P->tensors[in_t[k]], r);
      for (size_t k = 0; k < out_t.size(); ++k) x.out[k] = P->Ptr(P->tensors[out_t[k]], r);
      for (int t = 0; t < x.n_tab; ++t)
        x.tab[t] = reinterpret_cast<const uint16_t*>(P->peer_base[r] + x.tab_off[t]);
      if (x.lad_n) x.lad = reinterpret_cast<const uint4*>(P->peer_base[r] + x.lad_off);
      if (x.vlad_n) x.vlad = reinterpret_cast<const uint4*>(P->peer_base[r] + x.vlad_off);
      LaunchEwProg(x, dtype, s);
      return 1;
    };
    st.reads = in_t;
    st.writes = out_t;
    AddStep(std::move(st));
  }

  void EmitKernel(int i, const std::vector<int>& in_t, int out_t) {
    rh_program* P = p_;
    const rh_op& op = P->ops[i];
    const int first = rt_->first_rank;
    // fused residual add operand (matmul, PlanFusion): fetched before T is referenced (GetTensor
    // may emit transitions and grow the tensor table)
    int resid_t = -1;
    if (op.kind == RH_OP_MATMUL && !resid_.empty() && resid_[i].v >= 0)
      resid_t = GetTensor(resid_[i].x, p_->in_specs[resid_[i].v][resid_[i].slot], "edge");
    const Tensor& T = P->tensors[out_t];
    const int dtype = op.dtype;
    const int eb = ElemBytes(dtype);
    Step st;
    st.kind = Step::kKernel;
    st.launches = 1;
    const int64_t n_out = T.elems();
    double in_bytes = 0;
    for (int t : in_t) in_bytes += static_cast<double>(P->tensors[t].bytes);
    st.alg_bytes = in_bytes + static_cast<double>(T.bytes);
    const std::string id = OpName(i);
    switch (op.kind) {
      case RH_OP_MATMUL: {
        const Dims ad = P->tensors[in_t[0]].ldims, bd = P->tensors[in_t[1]].ldims;
        const bool fa = !fold_t_.empty() && fold_t_[i][0], fb = !fold_t_.empty() && fold_t_[i][1];
        const bool eta = op.transpose_a != fa, etb = op.transpose_b != fb;
        GemmArgs g{};
        g.m = eta ? ad[1] : ad[0];
        g.k = eta ? ad[0] : ad[1];
        g.n = etb ? bd[0] : bd[1];
        if ((etb ? bd[1] : bd[0]) != g.k) Fail("matmul " + id + ": local k mismatch");
        if (T.ldims[0] != g.m || T.ldims[1] != g.n) Fail("matmul " + id + ": local output shape mismatch");
        if (resid_t >= 0) {  // fused residual add (PlanFusion)
          const Resid& R = resid_[i];
          if (P->tensors[resid_t].ldims != T.ldims) Fail("matmul " + id + ": residual shape mismatch");
          p_->in_tensor[R.v].assign(2, -1);  // the pre-add operand is not materialized
          p_->in_tensor[R.v][R.slot] = resid_t;
          st.alg_bytes += static_cast<double>(P->tensors[resid_t].bytes);
        }
        g.ta = eta;
        g.tb = etb;
        g.dtype = dtype;
        g.epi = ChainOf(i, false);
        // fp32 GEMMs run as 3xTF32 and need split scratch: one region shared by all GEMMs of the
        // program (stream-ordered), sized to the largest and placed at the end of lowering.
        if (dtype == RH_F32) g.scratch = reinterpret_cast<void*>(uintptr_t{256});  // support probe
        g.sk_flags = reinterpret_cast<uint32_t*>(uintptr_t{256});  // stream-K allowed (flags at run)
        const bool tc = !(P->flags & RH_FLAG_SIMT_GEMM) && GemmTcSupported(g);
        if (tc) P->gemm_scratch_bytes = std::max(P->gemm_scratch_bytes, GemmTcScratchBytes(g));
        if (!tc) P->gemm_scratch_bytes = std::max(P->gemm_scratch_bytes, GemmSimtScratchBytes(g));
        g.scratch = nullptr;
        st.name = std::string(tc ? (dtype == RH_F32 ? "gemm_tc_3xtf32 " : "gemm_tc ") : "gemm_simt ") + id +
                  (fa || fb ? " [T-folded]" : "");
        st.alg_flops = 2.0 * g.m * g.n * g.k;
        const int ta = in_t[0], tb = in_t[1];
        const int rs = resid_t;
        if (rs >= 0) st.name += " +add " + OpName(resid_[i].v);
        auto pp = std::make_shared<PushPlan>();
        if (tc && dtype == RH_BF16) gemm_push_[Tail(i)] = {pp, g, static_cast<int>(p_->steps.size())};
        st.run = [P, g, ta, tb, out_t, first, tc, rs, pp](int li, cudaStream_t s) {
          GemmArgs a = g;
          const int r = first + li;
          a.a = P->Ptr(P->tensors[ta], r);
          a.b = P->Ptr(P->tensors[tb], r);
          a.c = P->Ptr(P->tensors[out_t], r);
          if (rs >= 0) a.resid = P->Ptr(P->tensors[rs], r);
          if (pp->dst_t >= 0) {  // the output all-gather, fused (TryPushMaterialize)
            a.push.sync = SyncOf(P, pp->axis, pp->slot, li);
            a.push.n = a.push.sync.d;
            for (int k = 0; k < a.push.n; ++k) a.push.dst[k] = P->Ptr(P->tensors[pp->dst_t], a.push.sync.members[k]);
            a.push.row_off = P->mesh->Coords(r)[pp->axis] * pp->rows_local;
            a.push.rows_full = P->tensors[pp->dst_t].gdims[0];
          } else if (pp->scatter_dim >= 0) {  // the reduce-scatter, fused (TryPushReduceScatter)
            a.push.sync = SyncOf(P, pp->axis, pp->slot, li);
            a.push.n = a.push.sync.d;
            const int64_t me = P->mesh->Coords(r)[pp->axis];
            for (int k = 0; k < a.push.n; ++k)
              a.push.dst[k] = P->peer_base[a.push.sync.members[k]] + pp->stage_off + me * pp->slot_bytes;
            a.push.scatter_dim = pp->scatter_dim;
            a.push.part = pp->part;
          }
          a.epi = Patch(P, g.epi, r);
          if (P->gemm_scratch_bytes) a.scratch = P->peer_base[r] + P->gemm_scratch_off;
          a.sk_flags = reinterpret_cast<uint32_t*>(P->peer_base[r] + P->gemm_flags_off);
          if (!tc) return LaunchGemmSimt(a, s);  // (+ split-K reduce for small M)
          LaunchGemmTc(a, s);
          return GemmTcLaunches(a);
        };
        if (tc) {
          st.launches = GemmTcLaunches(g);
          st.name += GemmTcSchedule(g);
        }
        if (!tc && GemmSimtScratchBytes(g) > 0) st.launches = 2;
        if (tc && dtype == RH_F32) {
          st.launches = 3;
          st.alg_bytes += 3.0 * 4 * (g.m * g.k + g.k * g.n);  // split pass: read x, write hi + lo
        }
        break;
      }
      case RH_OP_ADD:
      case RH_OP_MUL: {
        const bool mul = op.kind == RH_OP_MUL;
        const ChainArgs c = ChainOf(i, false);
        st.name = std::string(mul ? "mul " : "add ") + id + (c.n_fn ? "+chain" : "");
        st.alg_flops = static_cast<double>(n_out) * (1 + c.n_fn);
        const int ta = in_t[0], tb = in_t[1];
        st.run = [P, ta, tb, out_t, first, n_out, mul, c, dtype](int li, cudaStream_t s) {
          const int r = first + li;
          LaunchBinary(P->Ptr(P->tensors[out_t], r), P->Ptr(P->tensors[ta], r),
                       P->Ptr(P->tensors[tb], r), n_out, mul, Patch(P, c, r), dtype, s);
          return 1;
        };
        break;
      }
      case RH_OP_UNARY: {
        const int ti = in_t[0];
        if (op.fn == RH_FN_SOFTMAX) {
          const int64_t cols = T.ldims.back();
          const int64_t rows = n_out / cols;
          st.name = "softmax " + id;
          st.alg_flops = 4.0 * n_out;
          st.run = [P, ti, out_t, first, rows, cols, dtype](int li, cudaStream_t s) {
            const int r = first + li;
            LaunchSoftmaxRows(P->Ptr(P->tensors[out_t], r), P->Ptr(P->tensors[ti], r), rows, cols,
                              dtype, s);
            return 1;
          };
        } else {
          const ChainArgs c = ChainOf(i, true);
          st.name = "unary_chain[" + std::to_string(c.n_fn) + "] " + id;
          st.alg_flops = static_cast<double>(n_out) * c.n_fn;
          st.run = [P, ti, out_t, first, n_out, c, dtype](int li, cudaStream_t s) {
            const int r = first + li;
            LaunchUnaryChain(P->Ptr(P->tensors[out_t], r), P->Ptr(P->tensors[ti], r), n_out,
                             Patch(P, c, r), dtype, s);
            return 1;
          };
        }
        break;
      }
      case RH_OP_TRANSPOSE: {
        const int ti = in_t[0];
        const Dims id_ = P->tensors[ti].ldims;
        const std::vector<int> perm = EffPerm(op, static_cast<int>(id_.size()));
        st.name = "transpose " + id;
        st.run = [P, ti, out_t, first, id_, perm, dtype](int li, cudaStream_t s) {
          const int r = first + li;
          LaunchTranspose(P->Ptr(P->tensors[out_t], r), P->Ptr(P->tensors[ti], r),
                          static_cast<int>(id_.size()), id_.data(), perm.data(), dtype, s);
          return 1;
        };
        break;
      }
      case RH_OP_REDUCE_SUM: {
        const int ti = in_t[0];
        const Dims id_ = P->tensors[ti].ldims;
        int64_t outer = 1;
        for (int k = 0; k < op.axis; ++k) outer *= id_[k];
        const int64_t e = id_[op.axis], inner = Inner(id_, op.axis);
        st.name = "reduce_sum " + id;
        st.alg_flops = static_cast<double>(outer * e * inner);
        st.run = [P, ti, out_t, first, outer, e, inner, dtype](int li, cudaStream_t s) {
          const int r = first + li;
          LaunchReduceSum(P->Ptr(P->tensors[out_t], r), P->Ptr(P->tensors[ti], r), outer, e, inner,
                          dtype, s);
          return 1;
        };
        break;
      }
      case RH_OP_BROADCAST: {
        const int ti = in_t[0];
        const int64_t n_in = P->tensors[ti].elems();
        st.name = "broadcast " + id;
        st.run = [P, ti, out_t, first, n_out, n_in, dtype](int li, cudaStream_t s) {
          const int r = first + li;
          LaunchBroadcast(P->Ptr(P->tensors[out_t], r), P->Ptr(P->tensors[ti], r), n_out, n_in,
                          dtype, s);
          return 1;
        };
        break;
      }
      case RH_OP_CONCAT: {
        const int ax = op.axis;
        const Dims od = T.ldims;
        int64_t outer = 1;
        for (int k = 0; k < ax; ++k) outer *= od[k];
        const int64_t orow = od[ax] * Inner(od, ax);
        std::vector<int64_t> rows, offs;
        int64_t off = 0;
        for (int t : in_t) {
          const Dims ld = P->tensors[t].ldims;
          rows.push_back(ld[ax] * Inner(ld, ax));
          offs.push_back(off);
          off += rows.back();
        }
        if (off != orow) Fail("concat " + id + ": local shapes do not add up");
        st.name = "concat " + id;
        st.launches = static_cast<int>(in_t.size());
        const std::vector<int> ins = in_t;
        bool vec = static_cast<int>(ins.size()) <= kMaxConcat && (orow * eb) % 16 == 0;
        for (size_t k = 0; k < ins.size(); ++k) vec = vec && (rows[k] * eb) % 16 == 0 && (offs[k] * eb) % 16 == 0;
        if (vec) st.launches = 1;
        st.run = [P, ins, out_t, first, outer, orow, rows, offs, dtype, vec, eb](int li, cudaStream_t s) {
          const int r = first + li;
          if (vec) {  // one launch for every piece
            ConcatArgs a{};
            a.out = P->Ptr(P->tensors[out_t], r);
            a.n = static_cast<int>(ins.size());
            a.outer = outer;
            a.orow16 = orow * eb / 16;
            for (size_t k = 0; k < ins.size(); ++k) {
              a.in[k] = P->Ptr(P->tensors[ins[k]], r);
              a.row16[k] = rows[k] * eb / 16;
              a.off16[k] = offs[k] * eb / 16;
            }
            if (LaunchConcat(a, s)) return 1;
          }
          for (size_t k = 0; k < ins.size(); ++k)
            LaunchConcatPiece(P->Ptr(P->tensors[out_t], r), P->Ptr(P->tensors[ins[k]], r), outer,
                              rows[k], orow, offs[k], dtype, s);
          return static_cast<int>(ins.size());
        };
        break;
      }
      default:
        Fail(std::string("cannot execute op kind ") + KindName(op.kind));
    }
    (void)eb;
    st.reads = in_t;
    if (resid_t >= 0) st.reads.push_back(resid_t);
    st.writes = {out_t};
    AddStep(std::move(st));
  }

  // Fine-grained transition (ClassifyFine): one or two steps of LaunchFine kernels.
  int EmitFine(const FinePlan& fp, int src, int dst, int axis, const AxisView& fv, const AxisView& tv,
               double S, const char* why) {
    rh_program* P = p_;
    const Tensor X = p_->tensors[src];
    const int d = mesh_[axis];
    const int eb = ElemBytes(X.dtype);
    const int64_t n_src = X.elems(), n_dst = p_->tensors[dst].elems();
    const rh_spec from = X.specs[axis], to = p_->tensors[dst].specs[axis];
    const bool multi = rt_->dist && rt_->world > 1;
    auto base_step = [&](const std::string& tag) {
      Step st;
      st.kind = Step::kTransition;
      st.axis = axis;
      st.name = std::string(CollectiveName(from, to)) + " op" + std::to_string(X.op) + " " + SpecStr(from) + "->" +
                SpecStr(to) + "@" + std::to_string(axis) + " (" + why + ") [" + tag + "]";
      st.launches = 1;
      return st;
    };
    static const char* kMode[] = {"", "push", "pull-interleave", "two-phase", "two-phase", "slice"};
    if (fp.mode == 5) {  // Replicated -> fine Shard: local de-interleave keeping this rank's units
      Step st = base_step("slice");
      st.alg_bytes = static_cast<double>(n_dst) * eb * 2;
      const int64_t u = fp.u1;
      st.fine = [P, src, dst, axis, d, eb, u, n_src](int li, cudaStream_t s, const PeerSync&, int cap) {
        const int g = P->mesh->rt->first_rank + li;
        FineArgs a{};
        a.kind = 0;
        a.d = d;
        a.unit_bytes = static_cast<int>(u * eb);
        a.eb = eb;
        a.in[0] = P->Ptr(P->tensors[src], g);
        a.only = P->mesh->Coords(g)[axis];
        a.out[a.only] = P->Ptr(P->tensors[dst], g);
        a.n = n_src;
        a.lin = 1;
        a.max_blocks = cap;
        return LaunchFine(a, s);
      };
      st.reads = {src};
      st.writes = {dst};
      AddStep(std::move(st));
      return dst;
    }
    if (fp.mode == 1 || fp.mode == 2) {  // one step: push into the peers / pull-interleave from them
      const bool push = fp.mode == 1;
      Step st = base_step(kMode[fp.mode]);
      st.p2p = true;
      st.wire_bytes = WireBytes(from, to, S, d);
      st.alg_bytes = static_cast<double>(push ? n_src : n_dst) * eb * 2;
      if (multi) st.sync_slot = p_->n_sync_slots++;
      if (push) st.post_mode = 1;  // peers wrote this rank's destination: barrier before any read
      const int64_t u = push ? fp.u1 : fp.u2, run = fp.run, n = push ? n_src : n_dst;
      st.fine = [P, src, dst, axis, d, eb, u, run, n, push](int li, cudaStream_t s, const PeerSync& sync, int cap) {
        const int g = P->mesh->rt->first_rank + li;
        const std::vector<int> members = P->mesh->Group(axis, g);
        FineArgs a{};
        a.kind = push ? 0 : 1;
        a.d = d;
        a.unit_bytes = static_cast<int>(u * eb);
        a.eb = eb;
        for (int k = 0; k < d; ++k) {
          if (push) a.out[k] = P->Ptr(P->tensors[dst], members[k]);
          else a.in[k] = P->Ptr(P->tensors[src], members[k]);
        }
        if (push) a.in[0] = P->Ptr(P->tensors[src], g);
        else a.out[0] = P->Ptr(P->tensors[dst], g);
        a.n = n;
        a.lin = run == 0;
        a.run = run;
        a.c = P->mesh->Coords(g)[axis];
        a.sync = sync;
        a.max_blocks = cap;
        return LaunchFine(a, s);
      };
      if (!push) remote_read_.push_back(src);
      st.reads = {src};
      st.writes = {dst};
      AddStep(std::move(st));
      return dst;
    }
    // two phases: (A) de-interleave this rank's buffer into every member's staging stream for
    // it, (B) after a group barrier, interleave (or sum, Partial) the d local streams
    const bool partial = fp.mode == 4;
    const int64_t seg = partial ? n_dst : n_dst / d;  // elements of one member's stream
    const size_t stage_off = Alloc(static_cast<size_t>(seg) * d * eb);  // persistent, symmetric
    Step a_st = base_step("two-phase push");
    a_st.p2p = true;
    a_st.wire_bytes = WireBytes(from, to, S, d);
    a_st.alg_bytes = static_cast<double>(n_src) * eb * 2;
    a_st.post_mode = 2;
    a_st.no_async = true;
    if (multi) a_st.sync_slot = p_->n_sync_slots++;
    const int64_t u1 = fp.u1, u2 = fp.u2;
    a_st.fine = [P, src, axis, d, eb, u1, n_src, seg, stage_off](int li, cudaStream_t s, const PeerSync& sync, int cap) {
      const int g = P->mesh->rt->first_rank + li;
      const std::vector<int> members = P->mesh->Group(axis, g);
      const int c = P->mesh->Coords(g)[axis];
      FineArgs a{};
      a.kind = 0;
      a.d = d;
      a.unit_bytes = static_cast<int>(u1 * eb);
      a.eb = eb;
      a.in[0] = P->Ptr(P->tensors[src], g);
      for (int k = 0; k < d; ++k)
        a.out[k] = P->peer_base[members[k]] + stage_off + static_cast<size_t>(c) * seg * eb;  // stream c of member k
      a.n = n_src;
      a.lin = 1;
      a.sync = sync;
      a.max_blocks = cap;
      return LaunchFine(a, s);
    };
    a_st.reads = {src};
    AddStep(std::move(a_st));
    Step b_st = base_step(partial ? "two-phase sum" : "two-phase unpack");
    b_st.p2p = true;  // group-ordered after the pushes (fused barrier / stream joins)
    b_st.alg_bytes = static_cast<double>(n_dst) * eb * (partial ? d + 1 : 2);
    b_st.post_mode = 2;
    b_st.no_async = true;
    if (multi) b_st.sync_slot = p_->n_sync_slots++;
    const int dtype = X.dtype;
    b_st.fine = [P, dst, d, eb, u2, n_dst, seg, stage_off, partial, dtype](int li, cudaStream_t s, const PeerSync& sync,
                                                                          int cap) {
      const int g = P->mesh->rt->first_rank + li;
      char* stage = P->peer_base[g] + stage_off;
      if (partial) {  // sum of the d streams in member order (the rank-order sum of DESIGN §3)
        PullArgs pa{};
        pa.dst = P->Ptr(P->tensors[dst], g);
        for (int k = 0; k < d; ++k) pa.src[k] = stage + static_cast<size_t>(k) * seg * eb;
        pa.from = AxisView{RH_PARTIAL, d, 0, 0};
        pa.to = AxisView{RH_REPLICATED, d, 0, 0};
        pa.n_dst = n_dst;
        pa.dtype = dtype;
        pa.sync = sync;
        pa.max_blocks = cap;
        return LaunchPull(pa, s);
      }
      FineArgs a{};
      a.kind = 1;
      a.d = d;
      a.unit_bytes = static_cast<int>(u2 * eb);
      a.eb = eb;
      for (int k = 0; k < d; ++k) a.in[k] = stage + static_cast<size_t>(k) * seg * eb;
      a.out[0] = P->Ptr(P->tensors[dst], g);
      a.n = n_dst;
      a.lin = 1;
      a.sync = sync;
      a.max_blocks = cap;
      return LaunchFine(a, s);
    };
    b_st.writes = {dst};
    AddStep(std::move(b_st));
    return dst;
  }

  // Producer `p` in the per-axis layout `want`, inserting single-axis transitions as needed.
  int GetTensor(int p, const Specs& want, const char* why) {
    auto it = cache_.find(Key(p, want, cur_stage_));
    if (it != cache_.end()) return it->second;
    int cur = p_->out_tensor[p];
    if (cur < 0) Fail("internal: producer " + std::to_string(p) + " has no buffer");
    if (p_->tensors[cur].stage != cur_stage_) {  // produced by another pipeline stage
      auto jt = cache_.find(Key(p, p_->tensors[cur].specs, cur_stage_));
      cur = jt != cache_.end() ? jt->second : Transfer(cur, cur_stage_);
    }
    Specs cs = p_->tensors[cur].specs;
    if (SpecsEq(cs, want)) return cur;
    int m = 0;
    while (SpecEq(cs[m], want[m])) ++m;
    // Gather later sharded axes first so every single-axis move sees Replicated/Partial beyond
    // its own axis (its buffers are then exactly the axis-local tensor).
    for (int j = p_->n_axes - 1; j > m; --j) {
      if (cs[j].kind == RH_SHARD) {
        cs[j] = Rep();
        cur = Move(cur, j, cs, why);
      }
    }
    cs[m] = want[m];
    cur = Move(cur, m, cs, why);
    for (int j = m + 1; j < p_->n_axes; ++j) {
      if (!SpecEq(cs[j], want[j])) {
        cs[j] = want[j];
        cur = Move(cur, j, cs, why);
      }
    }
    return cur;
  }

  // Cross-stage Send/Recv (taskgraph.cpp:115-130): the receiving stage's rank pulls the tensor,
  // in its producer's layout, from the rank of the producing stage with the same non-pipeline
  // coordinates (same local layout: a plain copy), between two pairwise rendezvous — before:
  // the sender has produced it; after: the receiver has read it (the sender may overwrite it in
  // its next run).  Both sides run the step at the consumer's position in the schedule, so every
  // rendezvous is one point of the global order (deadlock-free).  Within the receiving stage
  // the usual transitions take it to the consumer's demanded layout (the cut placeholder's
  // reshard, planner.cpp:84-91).
  int Transfer(int src, int to_stage) {
    rh_program* P = p_;
    const Tensor X = p_->tensors[src];
    const int dst = NewTensor(X.op, X.specs, true, to_stage);
    const int from_stage = X.stage, paxis = p_->pipeline_axis;
    Step st;
    st.kind = Step::kTransition;
    st.stage = -2;
    st.axis = paxis;
    st.p2p = true;
    st.post_mode = 2;  // the closure's own pairwise rendezvous
    st.no_async = true;
    st.name = "send_recv op" + std::to_string(X.op) + " stage " + std::to_string(from_stage) + "->" +
              std::to_string(to_stage);
    st.wire_bytes = static_cast<double>(X.bytes);
    st.alg_bytes = 2.0 * X.bytes;
    const bool multi = rt_->dist && rt_->world > 1;
    const int slot_a = multi ? p_->n_sync_slots++ : -1, slot_b = multi ? p_->n_sync_slots++ : -1;
    st.sync_slot = -1;  // no group barrier / fused group sync: the pair rendezvous below
    st.run = [P, src, dst, from_stage, to_stage, paxis, slot_a, slot_b](int li, cudaStream_t s) {
      const int g = P->mesh->rt->first_rank + li;
      std::vector<int> c = P->mesh->Coords(g);
      const int me = c[paxis];
      if (me != from_stage && me != to_stage) return 0;
      c[paxis] = me == to_stage ? from_stage : to_stage;
      int peer = 0;
      for (size_t a = 0; a < c.size(); ++a) peer = peer * P->mesh->dims[a] + c[a];
      auto pair = [&](int slot) {
        PeerSync y{};
        if (slot < 0) return y;
        const size_t row = P->sync_off + static_cast<size_t>(slot) * P->mesh->rt->world * 4;
        const int mem[2] = {std::min(g, peer), std::max(g, peer)};
        y.d = 2;
        y.me = g;
        for (int k = 0; k < 2; ++k) {
          y.members[k] = mem[k];
          y.peer_slot[k] = reinterpret_cast<uint32_t*>(P->peer_base[mem[k]] + row);
        }
        y.my_slot = reinterpret_cast<uint32_t*>(P->peer_base[g] + row);
        y.epoch = reinterpret_cast<const uint32_t*>(P->peer_base[g] + P->epoch_off);
        y.err = reinterpret_cast<uint32_t*>(P->peer_base[g] + P->err_off);
        y.timeout_ns = SyncTimeoutNs();
        return y;
      };
      if (me == from_stage) {  // sender: rendezvous before and after the receiver's read
        LaunchPeerSync(pair(slot_a), s);
        LaunchPeerSync(pair(slot_b), s);
        return slot_a >= 0 ? 2 : 0;
      }
      PullArgs a{};
      a.dst = P->Ptr(P->tensors[dst], g);
      for (int k = 0; k < kMaxGroup; ++k) a.src[k] = P->Ptr(P->tensors[src], peer);
      a.from = AxisView{RH_REPLICATED, 1, 0, 0};
      a.to = AxisView{RH_REPLICATED, 1, 0, 0};
      a.coord = 0;
      a.n_dst = P->tensors[dst].elems();
      a.dtype = P->tensors[dst].dtype;
      a.sync = pair(slot_a);
      int n = LaunchPull(a, s);
      LaunchPeerSync(pair(slot_b), s);
      return n + (slot_b >= 0 ? 1 : 0);
    };
    remote_read_.push_back(src);
    st.reads = {src};
    st.writes = {dst};
    AddStep(std::move(st));
    return dst;
  }

  int Move(int src, int axis, const Specs& to_specs, const char* why) {
    auto it = cache_.find(Key(p_->tensors[src].op, to_specs, p_->tensors[src].stage));
    if (it != cache_.end()) return it->second;
    const Tensor X = p_->tensors[src];
    {
      // All-reduce over d > 2 peers as reduce-scatter + all-gather: each rank then moves
      // 2(d-1)/d of the tensor over NVLink (reshard_cost's bytes) instead of the (d-1)x of a
      // one-shot pull of every peer's full partial.
      const int d = mesh_[axis];
      const bool nccl = (p_->flags & RH_FLAG_TRANSPORT_NCCL) && rt_->dist;
      if (X.specs[axis].kind == RH_PARTIAL && to_specs[axis].kind == RH_REPLICATED && d > 2 && !nccl) {
        const Dims D = LocalDims(X.gdims, X.specs, mesh_, axis);
        for (int dim = 0; dim < static_cast<int>(D.size()); ++dim) {
          if (D[dim] % d != 0) continue;
          Specs mid = to_specs;
          mid[axis] = Sh(dim, D[dim] / d);
          const int m = Move(src, axis, mid, why);
          return Move(m, axis, to_specs, why);
        }
      }
    }
    const int dst = NewTensor(X.op, to_specs, true, X.stage);
    const Tensor Y = p_->tensors[dst];
    const int d = mesh_[axis];
    const Dims D = LocalDims(X.gdims, X.specs, mesh_, axis);  // axis-local tensor
    const rh_spec from = X.specs[axis], to = to_specs[axis];
    if (!Valid(to, D, d)) Fail("reshard: target spec " + SpecStr(to) + " invalid on axis " + std::to_string(axis));
    const AxisView fv = MakeAxisView(from, static_cast<int>(D.size()), D.data(), d);
    const AxisView tv = MakeAxisView(to, static_cast<int>(D.size()), D.data(), d);
    const int eb = ElemBytes(X.dtype);
    const double S = static_cast<double>(Prod(D)) * eb;
    if (TryPushReduceScatter(src, dst, axis, to_specs, why)) return dst;
    {
      static const bool no_fine = getenv("RH_NO_FINE") != nullptr;  // A/B knob (profiles/)
      const bool nccl_t = (p_->flags & RH_FLAG_TRANSPORT_NCCL) && rt_->dist;
      const FinePlan fp = ClassifyFine(fv, tv, eb, d, Prod(D));
      if (fp.mode && !no_fine && !nccl_t) return EmitFine(fp, src, dst, axis, fv, tv, S, why);
    }
    Step st;
    st.kind = Step::kTransition;
    st.axis = axis;
    st.name = std::string(CollectiveName(from, to)) + " op" + std::to_string(X.op) + " " +
              SpecStr(from) + "->" + SpecStr(to) + "@" + std::to_string(axis) + " (" + why + ")";
    st.wire_bytes = WireBytes(from, to, S, d);
    const double n_dst = static_cast<double>(Y.elems());
    st.alg_bytes = n_dst * eb * (from.kind == RH_PARTIAL ? d + 1 : 2);
    if (to.kind == RH_PARTIAL) st.alg_bytes = n_dst * eb * 2;
    st.launches = 1;
    rh_program* P = p_;
    const int first = rt_->first_rank;
    const int dtype = X.dtype;
    const bool remote = from.kind != RH_REPLICATED && d > 1;
    const bool nccl = (P->flags & RH_FLAG_TRANSPORT_NCCL) && rt_->dist && remote;
    st.p2p = remote && !nccl;
    // One process per GPU: the pre-transition group barrier rides inside the pull kernel
    // (not for zero-fill targets, whose non-zero-coordinate ranks launch no kernel).
    if (st.p2p && rt_->dist && rt_->world > 1 && to.kind != RH_PARTIAL) st.sync_slot = p_->n_sync_slots++;
    // Push all-gather of the output materialization: opt-in (RH_PUSH_AG=1).  Measured no faster
    // than the pull (C3 N=4: 40.2 vs 39.0 us, N=2: 32.3 vs 30.7 us, profiles/r2/push_ag_ab.log):
    // the posted writes gain nothing over the pull's reads and it needs a post-barrier.
    static const bool push_ag = getenv("RH_PUSH_AG") && getenv("RH_PUSH_AG")[0] == '1';
    if (!nccl && push_ag && st.p2p && from.kind == RH_SHARD && to.kind == RH_REPLICATED &&
        std::string(why) == "materialize" && (fv.Qs * eb) % 16 == 0) {
      // Output materialization into its persistent replicated buffer: push (every rank writes
      // its shard into every member's copy: posted NVLink writes), fused pre-barrier (the
      // members' copies are free: they reached this step), post-barrier (every push landed).
      st.name += " [push]";
      st.post_mode = 1;
      st.fine = [P, src, dst, axis, fv, tv, dtype](int li, cudaStream_t s, const PeerSync& sync, int cap) {
        const int g = P->mesh->rt->first_rank + li;
        const std::vector<int> members = P->mesh->Group(axis, g);
        PullArgs a{};
        a.dst = P->Ptr(P->tensors[src], g);  // roles reversed (LaunchPushGather)
        for (size_t k = 0; k < members.size(); ++k) a.src[k] = P->Ptr(P->tensors[dst], members[k]);
        a.from = fv;
        a.to = tv;
        a.coord = P->mesh->Coords(g)[axis];
        a.n_dst = P->tensors[dst].elems();
        a.dtype = dtype;
        a.sync = sync;
        a.max_blocks = cap;
        return LaunchPushGather(a, s);
      };
    } else if (!nccl) {
      // the launch (and the fused barrier) is set up by FinalizePulls once transitions are
      // merged and the overlap plan is known
      st.pulls.push_back([P, src, dst, axis, fv, tv, dtype](int li) {
        const int g = P->mesh->rt->first_rank + li;
        const std::vector<int> members = P->mesh->Group(axis, g);
        PullArgs a{};
        a.dst = P->Ptr(P->tensors[dst], g);
        for (size_t k = 0; k < members.size(); ++k) a.src[k] = P->Ptr(P->tensors[src], members[k]);
        a.from = fv;
        a.to = tv;
        a.coord = P->mesh->Coords(g)[axis];
        a.n_dst = P->tensors[dst].elems();
        a.dtype = dtype;
        return a;
      });
    } else {
      // Baseline: NCCL collective on this axis's communicator (+ pack/unpack pull kernels).
      const size_t chunk = static_cast<size_t>(Prod(LocalDims(D, {from.kind == RH_SHARD ? from : to}, {d}, 1)));
      const size_t stage_off = Alloc(static_cast<size_t>(Prod(D)) * eb);
      st.name += " [nccl]";
      st.run = [P, src, dst, axis, fv, tv, dtype, from, to, d, chunk, stage_off, eb, first](int li, cudaStream_t s) {
        const int g = first + li;
        ncclComm_t comm = P->mesh->axis_comm[axis];
        const int coord = P->mesh->Coords(g)[axis];
        char* x = P->Ptr(P->tensors[src], g);
        char* y = P->Ptr(P->tensors[dst], g);
        char* stage = P->peer_base[g] + stage_off;
        const int64_t ny = P->tensors[dst].elems();
        int launches = 0;
        if (from.kind == RH_PARTIAL && to.kind == RH_REPLICATED) {
          RH_NCCL(ncclAllReduce(x, y, ny, NcclType(dtype), ncclSum, comm, s));
          return 1;
        }
        if (from.kind == RH_PARTIAL) {  // pack each member's chunk, reduce-scatter
          AxisView rep = fv;
          rep.kind = RH_REPLICATED;
          for (int k = 0; k < d; ++k) {
            PullArgs a{};
            a.dst = stage + static_cast<size_t>(k) * chunk * eb;
            for (int j = 0; j < d; ++j) a.src[j] = x;  // Replicated view: any coordinate reads x
            a.from = rep;
            a.to = tv;
            a.coord = k;
            a.n_dst = static_cast<int64_t>(chunk);
            a.dtype = dtype;
            launches += LaunchPull(a, s);
          }
          RH_NCCL(ncclReduceScatter(stage, y, chunk, NcclType(dtype), ncclSum, comm, s));
          return launches + 1;
        }
        // Shard source: all-gather the shards, then one pull from the staging chunks.
        RH_NCCL(ncclAllGather(x, stage, chunk, NcclType(dtype), comm, s));
        PullArgs a{};
        a.dst = y;
        for (int k = 0; k < d; ++k) a.src[k] = stage + static_cast<size_t>(k) * chunk * eb;
        a.from = fv;
        a.to = tv;
        a.coord = coord;
        a.n_dst = ny;
        a.dtype = dtype;
        return 1 + LaunchPull(a, s);
      };
    }
    if (remote) remote_read_.push_back(src);
    st.reads = {src};
    st.writes = {dst};
    AddStep(std::move(st));
    return dst;
  }

  rh_program* p_;
  std::vector<int> mesh_;
  rh_runtime* rt_;
  size_t arena_ = 0;
  std::map<std::string, int> cache_;
  std::vector<bool> absorbed_;
  // GEMM head -> the add fused into its epilogue (v), the add's other operand (x, input slot)
  struct Resid {
    int v = -1, x = -1, slot = -1;
  };
  std::vector<Resid> resid_;
  // The op whose value a GEMM head's kernel writes: the fused add, else its chain's tail.
  int Tail(int i) const {
    if (!resid_.empty() && resid_[i].v >= 0) return resid_[i].v;
    return chain_[i].empty() ? i : chain_[i].back();
  }
  std::vector<std::array<bool, 2>> fold_t_;  // matmul slot reads a folded 2-D transpose
  std::vector<std::vector<int>> chain_;
  std::map<int, size_t> tanh_tables_;
  std::map<std::vector<int>, size_t> ladder_tables_;
  std::vector<int> remote_read_;  // tensors read by peers (transition sources)
  std::vector<EwPlan> ew_;
  std::vector<Remat> remat_;  // per chain program (PlanRemat)
  std::vector<int> ew_of_;  // op -> elementwise chain id (-1: none)
  int cur_stage_ = -1;      // pipeline programs: stage of the op being emitted
};

}  // namespace

void LowerProgram(rh_program* p) { Lowerer(p).Lower(); }

// The local-op rule table on its own (rh_op_natural_specs): composed over the mesh axes exactly
// as the lowering does (axis a sees the shapes left by axes < a, sharding.cpp:390-403).
Specs NaturalSpecsOf(const rh_op* ops, int n_ops, int i, const std::vector<int>& mesh) {
  if (i < 0 || i >= n_ops) Fail("bad op index");
  const rh_op& op = ops[i];
  const int n_axes = static_cast<int>(mesh.size());
  auto gdims = [&](int k) { return Dims(ops[k].dims, ops[k].dims + ops[k].rank); };
  Specs nat(n_axes), out(op.out_spec, op.out_spec + n_axes);
  for (int a = 0; a < n_axes; ++a) {
    std::vector<rh_spec> in_a;
    std::vector<Dims> in_d;
    for (int sl = 0; sl < op.n_in; ++sl) {
      Specs ins(n_axes);
      for (int b = 0; b < n_axes; ++b) ins[b] = op.in_specs[b * op.n_in + sl];
      in_a.push_back(ins[a]);
      in_d.push_back(LocalDims(gdims(op.inputs[sl]), ins, mesh, a));
    }
    nat[a] = Natural(op, in_a, in_d, LocalDims(gdims(i), nat, mesh, a), mesh[a], out[a]);
  }
  return nat;
}

}  // namespace rh
