// rh_lower.cpp — see rh_lower.h.  Every call below is a public reference API; nothing of the
// reference is re-implemented here except the ~40 lines of search glue that sit in the
// anonymous namespace of proj/src/planner.cpp:122-167 (SpmdSearchAllAxes).
#include "rh_lower.h"

#include <cmath>
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

}  // namespace

LoweredProgram RecoverStrategies(const TensorProgram& g, const parashard::ExecutionPlan& plan,
                                 const parashard::PlanOptions& opts) {
  if (plan.pipeline_axis >= 0) {
    throw std::runtime_error("pipeline plans are not executable in this tier (SURVEY §8f-1)");
  }
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
  j["schema"] = "rhino-lowered/1";
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
    ops.push_back(o);
  }
  j["ops"] = ops;
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
