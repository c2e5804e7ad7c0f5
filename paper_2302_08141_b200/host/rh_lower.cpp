// rh_lower.cpp — see rh_lower.h.  Every call below is a public reference API; nothing of the
// reference is re-implemented here except the ~40 lines of search glue that sit in the
// anonymous namespace of proj/src/planner.cpp:122-167 (SpmdSearchAllAxes).
#include "rh_lower.h"

#include <cmath>
#include <set>
#include <limits>
#include <stdexcept>

#include "nlohmann/json.hpp"
#include "parashard/ir.h"
#include "parashard/spmd.h"

namespace rhino {

using parashard::AxisSpec;
using parashard::OpStrategy;
using parashard::TensorProgram;
using json = nlohmann::ordered_json;

namespace {

const char* IlpStatusName(parashard::IlpStatus s) {
  switch (s) {
    case parashard::IlpStatus::kOptimal: return "optimal";
    case parashard::IlpStatus::kFeasible: return "feasible";
    case parashard::IlpStatus::kInfeasible: return "infeasible";
  }
  return "?";
}

OpStrategy AllReplicated(const TensorProgram& g, int i) {
  OpStrategy s;
  s.input_specs.assign(g.input_indices(i).size(), AxisSpec::Replicated());
  s.output_spec = AxisSpec::Replicated();
  s.comp_flops = g.op(i).flops;
  return s;
}

// ExtractStage (proj/src/planner.cpp:75-110, file-local there): the ops of stage s, with a
// "__cut_<id>" Input placeholder for every producer outside the stage; outputs are the global
// outputs of the stage and every op consumed by another stage.  Same public calls, same order.
struct StageSub {
  TensorProgram prog;
  std::vector<int> global_op;  // sub index -> global index, -1 for cut placeholders
  std::vector<int> cut_of;     // sub index -> global producer of the placeholder (-1: not a cut)
};

StageSub ExtractStageSub(const TensorProgram& g, const std::vector<int>& stage_of, int s) {
  StageSub sub;
  std::set<int> external;
  for (int i = 0; i < g.size(); ++i) {
    if (stage_of[i] != s) continue;
    for (int p : g.input_indices(i))
      if (stage_of[p] != s) external.insert(p);
  }
  for (int p : external) {
    parashard::Operator ph;
    ph.id = "__cut_" + g.op(p).id;
    ph.kind = parashard::OpKind::kInput;
    ph.output_shape = g.op(p).output_shape;
    sub.prog.Add(std::move(ph));
    sub.global_op.push_back(-1);
    sub.cut_of.push_back(p);
  }
  std::set<int> global_outputs(g.output_indices().begin(), g.output_indices().end());
  std::vector<parashard::OpId> outputs;
  for (int i = 0; i < g.size(); ++i) {
    if (stage_of[i] != s) continue;
    parashard::Operator op = g.op(i);
    for (parashard::OpId& in : op.inputs)
      if (stage_of[g.IndexOf(in)] != s) in = "__cut_" + in;
    sub.prog.Add(std::move(op));
    sub.global_op.push_back(i);
    sub.cut_of.push_back(-1);
    bool is_out = global_outputs.count(i) > 0;
    for (int c : g.consumer_indices(i)) is_out = is_out || stage_of[c] != s;
    if (is_out) outputs.push_back(g.op(i).id);
  }
  if (!outputs.empty()) sub.prog.SetOutputs(std::move(outputs));
  sub.prog.Validate();
  return sub;
}

// The per-axis search replay on one (sub)program: axes in order, `skip_axis` (the pipeline axis)
// and size-1 axes all Replicated; `planned(axis, i)` = the plan's spec of sub op i, or nullptr
// when the plan does not record it (cut placeholders).
template <typename Planned>
void ReplayAxes(const TensorProgram& g, const parashard::ExecutionPlan& plan, const parashard::PlanOptions& opts,
                int skip_axis, Planned planned, std::vector<std::vector<OpStrategy>>* strat,
                std::vector<AxisRecovery>* recovery) {
  const int n = g.size();
  const int naxes = plan.mesh.num_axes();
  strat->assign(naxes, std::vector<OpStrategy>(n));
  std::vector<std::vector<AxisSpec>> chosen;
  std::vector<int> chosen_d;
  for (int axis = 0; axis < naxes; ++axis) {
    AxisRecovery rec;
    rec.axis = axis;
    rec.d = plan.mesh.dims[axis];
    if (rec.d < 2 || axis == skip_axis) {  // planner.cpp:133 (size-1 axes), :131 (pipeline axis)
      for (int i = 0; i < n; ++i) (*strat)[axis][i] = AllReplicated(g, i);
      rec.ilp_status = axis == skip_axis ? "pipeline" : "skipped";
      recovery->push_back(rec);
      continue;
    }
    parashard::SpmdAxisContext ctx;
    ctx.g = &g;
    ctx.shapes = parashard::EffectiveShapes(g, chosen, chosen_d);
    ctx.mesh = plan.mesh;
    ctx.axis = axis;
    ctx.device_flops = plan.cluster.device_flops;
    ctx.ilp_time_limit = opts.ilp_time_limit;
    ctx.flops_threshold = opts.flops_threshold;
    parashard::CandidateMap cand = parashard::generate_candidates(g, ctx.shapes, rec.d, opts.flops_threshold, axis);
    std::optional<parashard::MemoryBudget> budget;
    if (plan.memory_limit_bytes > 0) budget = parashard::MemoryBudget{plan.memory_limit_bytes, plan.optimizer_multiplier};
    parashard::SpmdResult r = plan.opt_level >= 3 ? parashard::search_o3(ctx, cand, budget ? &*budget : nullptr)
                                                  : parashard::search_o2(ctx, cand, budget ? &*budget : nullptr);
    if (budget) {
      // SpmdResult.choice indexes the memory-pruned map (proj/src/spmd.cpp:675-678).
      cand = parashard::apply_memory_constraint(g, ctx.shapes, cand, *budget, rec.d, r.forced_k).candidates;
    }
    rec.ilp_status = IlpStatusName(r.status);
    std::vector<AxisSpec> specs(n);
    for (int i = 0; i < n; ++i) {
      const OpStrategy& s = cand[i][r.choice[i]];
      const AxisSpec* want = planned(axis, i);
      if (!want || s.output_spec == *want) {
        (*strat)[axis][i] = s;
        specs[i] = s.output_spec;
        continue;
      }
      // Fallback: the candidate emitting the planned spec with the least
      // resharding against the producers' planned specs; ties -> lowest index.
      rec.replay_matched = false;
      rec.fallback_ops.push_back(g.op(i).id);
      int best = -1;
      double best_cost = std::numeric_limits<double>::infinity();
      for (size_t c = 0; c < cand[i].size(); ++c) {
        if (!(cand[i][c].output_spec == *want)) continue;
        double cost = 0;
        const auto& in_idx = g.input_indices(i);
        for (size_t slot = 0; slot < in_idx.size(); ++slot) {
          const int p = in_idx[slot];
          const AxisSpec* pw = planned(axis, p);
          cost += parashard::reshard_cost(pw ? *pw : cand[p][r.choice[p]].output_spec, cand[i][c].input_specs[slot],
                                          ctx.shapes[p], plan.mesh, axis)
                      .seconds;
        }
        if (cost < best_cost) {
          best_cost = cost;
          best = static_cast<int>(c);
        }
      }
      if (best < 0)
        throw std::runtime_error("strategy recovery: no candidate of op '" + g.op(i).id + "' emits planned spec " +
                                 want->ToString());
      (*strat)[axis][i] = cand[i][best];
      specs[i] = *want;
    }
    recovery->push_back(rec);
    chosen.push_back(specs);
    chosen_d.push_back(rec.d);
  }
}

LoweredProgram RecoverPipeline(const TensorProgram& g, const parashard::ExecutionPlan& plan,
                               const parashard::PlanOptions& opts) {
  const int n = g.size(), naxes = plan.mesh.num_axes();
  const int S = plan.mesh.dims[plan.pipeline_axis];
  LoweredProgram lp;
  lp.mesh = plan.mesh.dims;
  lp.descriptor = plan.descriptor;
  lp.pipeline_axis = plan.pipeline_axis;
  lp.microbatches = plan.microbatches;
  lp.stage_of = plan.stages.stage_of;
  lp.strat.assign(naxes, std::vector<OpStrategy>(n));
  for (int s = 0; s < S; ++s) {
    const StageSub sub = ExtractStageSub(g, plan.stages.stage_of, s);
    std::vector<std::vector<OpStrategy>> st;
    std::vector<AxisRecovery> rec;
    ReplayAxes(sub.prog, plan, opts, plan.pipeline_axis,
               [&](int axis, int i) -> const AxisSpec* {
                 return sub.global_op[i] >= 0 ? &plan.sharding[axis][sub.global_op[i]] : nullptr;
               },
               &st, &rec);
    for (int i = 0; i < sub.prog.size(); ++i) {
      if (sub.global_op[i] >= 0) {
        for (int a = 0; a < naxes; ++a) lp.strat[a][sub.global_op[i]] = st[a][i];
      } else {
        CutSpec c;
        c.stage = s;
        c.producer = sub.cut_of[i];
        for (int a = 0; a < naxes; ++a) c.specs.push_back(st[a][i].output_spec);
        lp.cuts.push_back(c);
      }
    }
    for (auto& r : rec) {
      r.axis += 100 * s;  // stage-tagged (axis + 100 * stage) in the diagnostics
      lp.recovery.push_back(r);
    }
  }
  return lp;
}

}  // namespace

LoweredProgram RecoverStrategies(const TensorProgram& g, const parashard::ExecutionPlan& plan,
                                 const parashard::PlanOptions& opts) {
  if (plan.pipeline_axis >= 0) return RecoverPipeline(g, plan, opts);
  const int n = g.size();
  const int naxes = plan.mesh.num_axes();
  LoweredProgram lp;
  lp.mesh = plan.mesh.dims;
  lp.descriptor = plan.descriptor;
  lp.strat.assign(naxes, std::vector<OpStrategy>(n));
  std::vector<std::vector<AxisSpec>> chosen;
  std::vector<int> chosen_d;
  for (int axis = 0; axis < naxes; ++axis) {
    AxisRecovery rec;
    rec.axis = axis;
    rec.d = plan.mesh.dims[axis];
    if (rec.d < 2) {  // the planner skips size-1 axes (planner.cpp:133): all Replicated
      for (int i = 0; i < n; ++i) lp.strat[axis][i] = AllReplicated(g, i);
      rec.ilp_status = "skipped";
      lp.recovery.push_back(rec);
      continue;
    }
    parashard::SpmdAxisContext ctx;
    ctx.g = &g;
    ctx.shapes = parashard::EffectiveShapes(g, chosen, chosen_d);
    ctx.mesh = plan.mesh;
    ctx.axis = axis;
    ctx.device_flops = plan.cluster.device_flops;
    ctx.ilp_time_limit = opts.ilp_time_limit;
    ctx.flops_threshold = opts.flops_threshold;
    parashard::CandidateMap cand =
        parashard::generate_candidates(g, ctx.shapes, rec.d, opts.flops_threshold, axis);
    std::optional<parashard::MemoryBudget> budget;
    if (plan.memory_limit_bytes > 0) {
      budget = parashard::MemoryBudget{plan.memory_limit_bytes, plan.optimizer_multiplier};
    }
    parashard::SpmdResult r = plan.opt_level >= 3
                                  ? parashard::search_o3(ctx, cand, budget ? &*budget : nullptr)
                                  : parashard::search_o2(ctx, cand, budget ? &*budget : nullptr);
    if (budget) {
      // SpmdResult.choice indexes the memory-pruned map (proj/src/spmd.cpp:675-678).
      cand = parashard::apply_memory_constraint(g, ctx.shapes, cand, *budget, rec.d, r.forced_k)
                 .candidates;
    }
    rec.ilp_status = IlpStatusName(r.status);
    const auto& planned = plan.sharding[axis];
    for (int i = 0; i < n; ++i) {
      const OpStrategy& s = cand[i][r.choice[i]];
      if (s.output_spec == planned[i]) {
        lp.strat[axis][i] = s;
        continue;
      }
      // Fallback: the candidate emitting the planned spec with the least
      // resharding against the producers' planned specs; ties -> lowest index.
      rec.replay_matched = false;
      rec.fallback_ops.push_back(g.op(i).id);
      int best = -1;
      double best_cost = std::numeric_limits<double>::infinity();
      for (size_t c = 0; c < cand[i].size(); ++c) {
        if (!(cand[i][c].output_spec == planned[i])) continue;
        double cost = 0;
        const auto& in_idx = g.input_indices(i);
        for (size_t slot = 0; slot < in_idx.size(); ++slot) {
          int p = in_idx[slot];
          cost += parashard::reshard_cost(planned[p], cand[i][c].input_specs[slot], ctx.shapes[p],
                                          plan.mesh, axis)
                      .seconds;
        }
        if (cost < best_cost) {
          best_cost = cost;
          best = static_cast<int>(c);
        }
      }
      if (best < 0) {
        throw std::runtime_error("strategy recovery: no candidate of op '" + g.op(i).id +
                                 "' emits planned spec " + planned[i].ToString());
      }
      lp.strat[axis][i] = cand[i][best];
    }
    lp.recovery.push_back(rec);
    chosen.push_back(planned);
    chosen_d.push_back(rec.d);
  }
  return lp;
}

LoweredProgram StrategiesFromChoice(const TensorProgram& g, const std::vector<int>& mesh,
                                    const std::vector<std::vector<AxisSpec>>& out_specs,
                                    const std::vector<std::vector<OpStrategy>>& strat) {
  LoweredProgram lp;
  lp.mesh = mesh;
  lp.strat = strat;
  (void)out_specs;
  (void)g;
  for (size_t a = 0; a < mesh.size(); ++a) {
    AxisRecovery rec;
    rec.axis = static_cast<int>(a);
    rec.d = mesh[a];
    rec.ilp_status = "explicit";
    lp.recovery.push_back(rec);
  }
  lp.descriptor = "explicit";
  return lp;
}

rh_spec ToRhSpec(const AxisSpec& s) {
  rh_spec r{};
  if (s.is_shard()) {
    r.kind = RH_SHARD;
    r.dim = s.dim;
    r.stride = s.stride;
  } else if (s.is_partial()) {
    r.kind = RH_PARTIAL;
    r.dim = -1;
  } else {
    r.kind = RH_REPLICATED;
    r.dim = -1;
  }
  return r;
}

int ToRhFn(const std::string& fn) {
  if (fn.empty()) return RH_FN_UNLABELED;
  if (fn == "relu") return RH_FN_RELU;
  if (fn == "gelu") return RH_FN_GELU;
  if (fn == "tanh") return RH_FN_TANH;
  if (fn == "exp") return RH_FN_EXP;
  if (fn == "sigmoid") return RH_FN_SIGMOID;
  if (fn == "softmax") return RH_FN_SOFTMAX;
  if (fn == "neg") return RH_FN_NEG;
  if (fn == "rsqrt") return RH_FN_RSQRT;
  if (fn == "identity") return RH_FN_IDENTITY;
  throw std::runtime_error("unknown unary fn '" + fn + "'");
}

std::string LoweredToJson(const TensorProgram& g, const LoweredProgram& lp, const std::string& name,
                          const std::string& dtype) {
  json j;
  j["schema"] = lp.pipeline_axis >= 0 ? "rhino-lowered/2" : "rhino-lowered/1";
  j["name"] = name;
  j["descriptor"] = lp.descriptor;
  j["mesh"] = lp.mesh;
  j["dtype"] = dtype;
  json ops = json::array();
  for (int i = 0; i < g.size(); ++i) {
    const parashard::Operator& op = g.op(i);
    json o;
    o["id"] = op.id;
    o["kind"] = parashard::OpKindName(op.kind);
    o["inputs"] = g.input_indices(i);
    o["shape"] = op.output_shape.dims;
    o["elem_bytes"] = op.output_shape.elem_bytes;
    o["flops"] = op.flops;
    if (op.kind == parashard::OpKind::kUnaryElementwise) o["fn"] = op.fn;
    if (op.kind == parashard::OpKind::kMatMul) {
      o["transpose_a"] = op.transpose_a;
      o["transpose_b"] = op.transpose_b;
    }
    if (op.kind == parashard::OpKind::kReduceSum || op.kind == parashard::OpKind::kConcat) {
      o["axis"] = op.axis;
    }
    if (op.kind == parashard::OpKind::kTranspose) o["perm"] = op.perm;
    json out_spec = json::array(), in_specs = json::array(), comp = json::array();
    for (size_t a = 0; a < lp.strat.size(); ++a) {
      const OpStrategy& s = lp.strat[a][i];
      out_spec.push_back(s.output_spec.ToString());
      json slots = json::array();
      for (const auto& sp : s.input_specs) slots.push_back(sp.ToString());
      in_specs.push_back(slots);
      comp.push_back(s.comp_flops);
    }
    o["out_spec"] = out_spec;
    o["in_specs"] = in_specs;
    o["comp_flops"] = comp;
    if (lp.pipeline_axis >= 0) o["stage"] = i < static_cast<int>(lp.stage_of.size()) ? lp.stage_of[i] : -1;
    ops.push_back(o);
  }
  j["ops"] = ops;
  if (lp.pipeline_axis >= 0) {  // wire format v2: stages, microbatches, cut placeholder specs
    j["pipeline_axis"] = lp.pipeline_axis;
    j["microbatches"] = lp.microbatches;
    json cuts = json::array();
    for (const auto& c : lp.cuts) {
      json sp = json::array();
      for (const auto& x : c.specs) sp.push_back(x.ToString());
      cuts.push_back({{"stage", c.stage}, {"producer", c.producer}, {"id", "__cut_" + g.op(c.producer).id},
                      {"spec", sp}});
    }
    j["cuts"] = cuts;
  }
  j["outputs"] = g.output_indices();
  j["topo"] = parashard::TopoOrderIndices(g);
  json rec = json::array();
  for (const auto& r : lp.recovery) {
    rec.push_back({{"axis", r.axis},
                   {"d", r.d},
                   {"ilp_status", r.ilp_status},
                   {"replay_matched", r.replay_matched},
                   {"fallback_ops", r.fallback_ops}});
  }
  j["recovery"] = rec;
  return j.dump(1) + "\n";
}

}  // namespace rhino
