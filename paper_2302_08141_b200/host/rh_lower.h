// rh_lower.h — reference-side lowering: parashard::ExecutionPlan -> rh_op records.
//
// This is the glue a maintainer adds to the reference (it includes the reference's own public
// headers and links libparashard unchanged).  The plan keeps only each op's OUTPUT spec per
// mesh axis (ExecutionPlan.sharding, proj/include/parashard/planner.h:77; only r.specs is kept
// at proj/src/planner.cpp:150), so the input specs each op demands (OpStrategy.input_specs,
// proj/include/parashard/sharding.h:99-111) are recovered by replaying the per-axis search the
// planner ran in its file-local SpmdSearchAllAxes (proj/src/planner.cpp:122-167) with the same
// public calls: EffectiveShapes -> generate_candidates -> [apply_memory_constraint] ->
// search_o3 / search_o2, then OpStrategy = cand[i][choice[i]].
#ifndef RH_LOWER_H_
#define RH_LOWER_H_

#include <string>
#include <vector>

#include "parashard/planner.h"
#include "parashard/sharding.h"
#include "rhino_exec.h"

namespace rhino {

struct AxisRecovery {
  int axis = 0;
  int d = 1;
  std::string ilp_status;      // optimal | feasible | infeasible | skipped
  bool replay_matched = true;  // replayed specs == plan.sharding[axis]
  std::vector<std::string> fallback_ops;  // ops recovered by the output-spec fallback
};

// A pipeline plan's cut placeholder (proj/src/planner.cpp:84-91): producer `producer` (of an
// earlier stage), read by stage `stage` as input "__cut_<id>", in the per-axis specs the stage's
// own search chose for the placeholder (the plan does not record them, planner.cpp:219-221).
struct CutSpec {
  int stage = 0;
  int producer = 0;
  std::vector<parashard::AxisSpec> specs;  // [axis]
};

struct LoweredProgram {
  std::vector<int> mesh;                                    // DeviceMesh::dims
  std::vector<std::vector<parashard::OpStrategy>> strat;   // [axis][op]
  std::vector<AxisRecovery> recovery;
  std::string descriptor;
  // pipeline plans (ExecutionPlan.pipeline_axis >= 0): stage of every op, microbatches, cuts
  int pipeline_axis = -1;
  int microbatches = 1;
  std::vector<int> stage_of;
  std::vector<CutSpec> cuts;
};

// Recovers every op's OpStrategy on every mesh axis of `plan`.  Pipeline plans: per stage, the
// stage subprogram (ExtractStage, planner.cpp:75-110) is searched again on the non-pipeline axes
// (SpmdSearchAllAxes with skip_axis, planner.cpp:122-167); ops get their stage and the cut
// placeholders their specs; every op is Replicated on the pipeline axis.  `opts` must be the
// PlanOptions the plan was made with.
LoweredProgram RecoverStrategies(const parashard::TensorProgram& g,
                                 const parashard::ExecutionPlan& plan,
                                 const parashard::PlanOptions& opts);

// Strategies from an explicit per-axis candidate choice (used to generate random but valid
// partitioned programs: any candidate combination is a legal SPMD program).
LoweredProgram StrategiesFromChoice(const parashard::TensorProgram& g, const std::vector<int>& mesh,
                                    const std::vector<std::vector<parashard::AxisSpec>>& out_specs,
                                    const std::vector<std::vector<parashard::OpStrategy>>& strat);

rh_spec ToRhSpec(const parashard::AxisSpec& s);
int ToRhFn(const std::string& fn);

// Lowered program as a self-contained JSON document (schema "rhino-lowered/1").
std::string LoweredToJson(const parashard::TensorProgram& g, const LoweredProgram& lp,
                          const std::string& name, const std::string& dtype);

}  // namespace rhino

#endif  // RH_LOWER_H_
