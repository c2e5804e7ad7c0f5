// rh_plan — plan a program with the UNCHANGED reference planner and emit the lowered program.
//
// This is the `parashard plan` path (proj/tools/parashard_main.cpp:56-125: LoadGraph -> plan)
// with RunPlan's tail replaced by strategy recovery + lowering (rh_lower.h).  The output JSON
// ("rhino-lowered/1") is what the executor consumes through the C-ABI (include/rhino_exec.h).
//
//   rh_plan (--text F | --json F | --fixture family:layers:hidden:batch)
//           [--devices N | --machines M --gpus G] [--equal-bw] [--ilp-time-limit S]
//           [--random-choice SEED --mesh d0[,d1]] [--dtype f32|bf16] [--name NAME]
//           [--pipeline-stages S --microbatches M] [--plan-out PLAN.json] -o OUT.json
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <limits>
#include <random>
#include <sstream>
#include <string>

#include "nlohmann/json.hpp"
#include "parashard/fixtures.h"
#include "parashard/parser.h"
#include "parashard/planner.h"
#include "rh_lower.h"

using namespace parashard;
using json = nlohmann::ordered_json;

namespace {

std::string ReadFile(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot read " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

std::vector<int> ParseInts(const std::string& s, char sep) {
  std::vector<int> out;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, sep)) out.push_back(std::stoi(tok));
  return out;
}

// Random but legal partitioned program: per axis, a uniformly random candidate per op from
// generate_candidates (proj/src/sharding.cpp:405-491); later axes see the composed shapes
// (EffectiveShapes, :390-403) exactly as the planner's searches do.
rhino::LoweredProgram RandomChoice(const TensorProgram& g, const std::vector<int>& mesh,
                                   uint64_t seed) {
  std::mt19937_64 rng(seed);
  std::vector<std::vector<AxisSpec>> chosen;
  std::vector<int> chosen_d;
  std::vector<std::vector<OpStrategy>> strat(mesh.size(), std::vector<OpStrategy>(g.size()));
  for (size_t axis = 0; axis < mesh.size(); ++axis) {
    int d = mesh[axis];
    auto shapes = EffectiveShapes(g, chosen, chosen_d);
    CandidateMap cand = generate_candidates(g, shapes, d, 0.0, static_cast<int>(axis));
    std::vector<AxisSpec> specs(g.size());
    for (int i = 0; i < g.size(); ++i) {
      // Keep only candidates whose demanded input specs are valid on the composed shape the
      // consumer actually receives (its own input specs on earlier axes).  The planner prices
      // each axis on the producer's effective shape (EffectiveShapes), so a random mix can
      // demand a layout that does not exist on the consumer's side of a multi-axis edge.
      std::vector<const OpStrategy*> ok;
      for (const auto& c : cand[i]) {
        bool valid = true;
        const auto& in_idx = g.input_indices(i);
        for (size_t slot = 0; slot < in_idx.size() && valid; ++slot) {
          TensorShape s = g.op(in_idx[slot]).output_shape;
          for (size_t a = 0; a < axis; ++a) s = LocalShape(s, strat[a][i].input_specs[slot], mesh[a]);
          valid = SpecValidForShape(c.input_specs[slot], s, d);
        }
        if (valid) ok.push_back(&c);
      }
      if (ok.empty()) throw std::runtime_error("no consistent candidate for op " + g.op(i).id);
      strat[axis][i] = *ok[rng() % ok.size()];
      specs[i] = strat[axis][i].output_spec;
    }
    chosen.push_back(specs);
    chosen_d.push_back(d);
  }
  return rhino::StrategiesFromChoice(g, mesh, chosen, strat);
}

// Forward + backward programs: the reference search (cone tables + ILP) does not
// scale to the backward graph (every backward op is multi-input; measured >17 GB and minutes on
// a 298-op block), so the first `k_fwd` ops (the forward program) are planned by the UNCHANGED
// planner, and every later op takes, in order, the candidate of the reference's own
// generate_candidates that minimises the reference's objective terms (comp_flops/device_flops +
// reshard_cost from its producers' chosen specs) — a greedy solver over the planner's candidates
// and cost model.
rhino::LoweredProgram PlanFwdGreedyBwd(const TensorProgram& g, int k_fwd, const ClusterConfig& cluster,
                                       const PlanOptions& opts, json* extra) {
  TensorProgram gf;
  for (int i = 0; i < k_fwd; ++i) gf.Add(g.op(i));
  gf.SetOutputs({g.op(k_fwd - 1).id});
  gf.Validate();
  ExecutionPlan pf = plan(gf, cluster, opts);
  rhino::LoweredProgram lf = rhino::RecoverStrategies(gf, pf, opts);
  const std::vector<int>& mesh = pf.mesh.dims;
  std::vector<std::vector<AxisSpec>> chosen;
  std::vector<int> chosen_d;
  std::vector<std::vector<OpStrategy>> strat(mesh.size(), std::vector<OpStrategy>(g.size()));
  for (size_t axis = 0; axis < mesh.size(); ++axis) {
    const int d = mesh[axis];
    std::vector<AxisSpec> specs(g.size(), AxisSpec::Replicated());
    if (d < 2 || static_cast<int>(axis) == pf.pipeline_axis) {  // pipeline axis: all Replicated
      for (int i = 0; i < g.size(); ++i) {
        strat[axis][i].input_specs.assign(g.input_indices(i).size(), AxisSpec::Replicated());
        strat[axis][i].output_spec = AxisSpec::Replicated();
      }
      chosen.push_back(specs);
      chosen_d.push_back(d);
      continue;
    }
    auto shapes = EffectiveShapes(g, chosen, chosen_d);
    CandidateMap cand = generate_candidates(g, shapes, d, opts.flops_threshold, static_cast<int>(axis));
    for (int i = 0; i < g.size(); ++i) {
      if (i < k_fwd) {
        strat[axis][i] = lf.strat[axis][i];
        specs[i] = strat[axis][i].output_spec;
        continue;
      }
      const auto& in_idx = g.input_indices(i);
      double best_cost = std::numeric_limits<double>::infinity();
      int best = -1;
      for (size_t c = 0; c < cand[i].size(); ++c) {
        bool valid = true;
        double cost = cand[i][c].comp_flops / cluster.device_flops;
        for (size_t slot = 0; slot < in_idx.size() && valid; ++slot) {
          TensorShape s = g.op(in_idx[slot]).output_shape;
          for (size_t a = 0; a < axis; ++a) s = LocalShape(s, strat[a][i].input_specs[slot], mesh[a]);
          valid = SpecValidForShape(cand[i][c].input_specs[slot], s, d);
          if (valid)
            cost += reshard_cost(specs[in_idx[slot]], cand[i][c].input_specs[slot], shapes[in_idx[slot]],
                                 pf.mesh, static_cast<int>(axis)).seconds;
        }
        if (valid && cost < best_cost) {
          best_cost = cost;
          best = static_cast<int>(c);
        }
      }
      if (best < 0) throw std::runtime_error("no consistent candidate for op " + g.op(i).id);
      strat[axis][i] = cand[i][best];
      specs[i] = strat[axis][i].output_spec;
    }
    chosen.push_back(specs);
    chosen_d.push_back(d);
  }
  (*extra)["forward_plan"] = {{"descriptor", pf.descriptor}, {"ops", k_fwd},
                              {"recovery_matched", lf.recovery.empty() || lf.recovery[0].replay_matched}};
  rhino::LoweredProgram lp = rhino::StrategiesFromChoice(g, mesh, chosen, strat);
  lp.descriptor = pf.descriptor + "+greedy-bwd";
  if (pf.pipeline_axis >= 0) {  // forward stages from the plan; backward ops staged by the caller
    lp.pipeline_axis = lf.pipeline_axis;
    lp.microbatches = lf.microbatches;
    lp.stage_of.assign(g.size(), -1);
    for (int i = 0; i < k_fwd; ++i) lp.stage_of[i] = lf.stage_of[i];
    lp.cuts = lf.cuts;
  }
  return lp;
}

}  // namespace

int main(int argc, char** argv) {
  std::string text_path, json_path, fixture, out_path, plan_out, name, dtype = "f32", mesh_s;
  int devices = 0, machines = 0, gpus = 0;
  bool equal_bw = false;
  long long random_seed = -1;
  double ilp_limit = 60.0;
  int opt_level = 0;  // PlanOptions.opt_level: 0 auto (O3 below 5000 ops), 2 = O2, 3 = O3
  int greedy_after = 0;  // > 0: plan the first N ops (forward) with the planner, rest greedy
  int pipeline_stages = -1, microbatches = 0;  // SPMD plans unless --pipeline-stages
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) throw std::runtime_error("missing value for " + a);
      return argv[++i];
    };
    if (a == "--text") text_path = next();
    else if (a == "--json") json_path = next();
    else if (a == "--fixture") fixture = next();
    else if (a == "--devices") devices = std::stoi(next());
    else if (a == "--machines") machines = std::stoi(next());
    else if (a == "--gpus") gpus = std::stoi(next());
    else if (a == "--equal-bw") equal_bw = true;
    else if (a == "--ilp-time-limit") ilp_limit = std::stod(next());
    else if (a == "--opt-level") opt_level = std::stoi(next());
    else if (a == "--greedy-after") greedy_after = std::stoi(next());
    else if (a == "--random-choice") random_seed = std::stoll(next());
    else if (a == "--pipeline-stages") pipeline_stages = std::stoi(next());
    else if (a == "--microbatches") microbatches = std::stoi(next());
    else if (a == "--mesh") mesh_s = next();
    else if (a == "--dtype") dtype = next();
    else if (a == "--name") name = next();
    else if (a == "--plan-out") plan_out = next();
    else if (a == "-o") out_path = next();
    else {
      std::cerr << "unknown argument " << a << "\n";
      return 2;
    }
  }
  try {
    TensorProgram g;
    if (!text_path.empty()) {
      g = parse_program(ReadFile(text_path));
    } else if (!json_path.empty()) {
      g = ParseProgramJson(ReadFile(json_path));
    } else if (!fixture.empty()) {
      std::stringstream ss(fixture);
      FixtureSpec fs;
      std::string tok;
      std::getline(ss, fs.family, ':');
      std::getline(ss, tok, ':');
      fs.layers = std::stoi(tok);
      std::getline(ss, tok, ':');
      fs.hidden = std::stoi(tok);
      std::getline(ss, tok, ':');
      fs.batch = std::stoi(tok);
      g = generate(fs);
    } else {
      throw std::runtime_error("one of --text/--json/--fixture is required");
    }
    if (name.empty()) name = fixture.empty() ? (text_path.empty() ? json_path : text_path) : fixture;

    rhino::LoweredProgram lp;
    json extra;
    auto t0 = std::chrono::steady_clock::now();
    if (random_seed >= 0) {
      lp = RandomChoice(g, ParseInts(mesh_s, ','), static_cast<uint64_t>(random_seed));
    } else {
      ClusterConfig cluster;
      if (devices > 0) {
        cluster.machines = 1;
        cluster.gpus_per_machine = devices;
      } else {
        cluster.machines = machines > 0 ? machines : 1;
        cluster.gpus_per_machine = gpus > 0 ? gpus : 1;
      }
      if (equal_bw) {
        cluster.inter_bandwidth = cluster.intra_bandwidth;
        cluster.inter_alpha = cluster.intra_alpha;
      }
      PlanOptions opts;
      opts.pipeline_stages = pipeline_stages;  // -1: SPMD plans; S > 0: S pipeline stages
      opts.microbatches = microbatches;
      opts.ilp_time_limit = ilp_limit;
      opts.opt_level = opt_level;
      if (greedy_after > 0) {
        lp = PlanFwdGreedyBwd(g, greedy_after, cluster, opts, &extra);
        extra["plan_seconds"] =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        json jj = json::parse(rhino::LoweredToJson(g, lp, name, dtype));
        for (auto it = extra.begin(); it != extra.end(); ++it) jj[it.key()] = it.value();
        std::ofstream(out_path) << jj.dump(1) << "\n";
        std::cerr << "rh_plan: " << name << " fwd+greedy-bwd mesh=" << json(lp.mesh).dump()
                  << " ops=" << g.size() << "\n";
        return 0;
      }
      ExecutionPlan p = plan(g, cluster, opts);
      auto t1 = std::chrono::steady_clock::now();
      lp = rhino::RecoverStrategies(g, p, opts);
      extra["plan_seconds"] = std::chrono::duration<double>(t1 - t0).count();
      extra["cost_report"] = {{"communication_bytes", p.cost.communication_bytes},
                              {"communication_seconds", p.cost.communication_seconds},
                              {"computation_seconds", p.cost.computation_seconds},
                              {"collective_counts", p.cost.collective_counts}};
      json sh = json::array();
      for (const auto& axis : p.sharding) {
        json a = json::array();
        for (const auto& s : axis) a.push_back(s.ToString());
        sh.push_back(a);
      }
      extra["plan_sharding"] = sh;
      if (!plan_out.empty()) {
        std::ofstream(plan_out) << PlanToJsonText(p, g);
      }
    }
    json j = json::parse(rhino::LoweredToJson(g, lp, name, dtype));
    for (auto it = extra.begin(); it != extra.end(); ++it) j[it.key()] = it.value();
    std::string text = j.dump(1) + "\n";
    if (out_path.empty()) {
      std::cout << text;
    } else {
      std::ofstream(out_path) << text;
    }
    std::cerr << "rh_plan: " << name << " mesh=" << json(lp.mesh).dump() << " ops=" << g.size()
              << " descriptor=" << lp.descriptor << "\n";
  } catch (const std::exception& e) {
    std::cerr << "rh_plan: error: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
