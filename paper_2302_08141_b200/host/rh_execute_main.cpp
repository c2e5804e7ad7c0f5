// rh_execute — the `execute` path a maintainer adds to the reference CLI,
// compiled: the reference's own LoadGraph / plan() calls (proj/tools/parashard_main.cpp:56-76),
// then, instead of RunPlan's JSON tail (:77-81), strategy recovery (rh_lower.h) and execution
// through the C-ABI of librhino_exec.so (include/rhino_exec.h).  Links libparashard (the
// UNCHANGED reference sources) statically and the executor dynamically.
//
//   rh_execute (--text F | --json F | --fixture family:layers:hidden:batch) --devices N
//              [--gpus G] [--dtype f32|bf16] [--iters K] [--seed S] [--out FILE]
//
// Ranks 0..N-1 of mesh (N) run on CUDA devices rank % G (G = 1: every rank emulated on cuda:0).
// --out writes the first program output, materialized replicated, as raw bytes (the GPU parity
// test compares it with the CPU oracle).  Prints one JSON line: plan descriptor, ms per step.
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#include "parashard/fixtures.h"
#include "parashard/parser.h"
#include "parashard/planner.h"
#include "rh_lower.h"
#include "rhino_exec.h"

using namespace parashard;

namespace {

std::string ReadFile(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot read " + path);
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

// LoadGraph (parashard_main.cpp:56-63): text IR, JSON program or a named fixture.
TensorProgram LoadGraph(const std::string& text, const std::string& json_path, const std::string& fixture) {
  if (!text.empty()) return parse_program(ReadFile(text));
  if (!json_path.empty()) return ParseProgramJson(ReadFile(json_path));
  if (fixture.empty()) throw std::runtime_error("one of --text/--json/--fixture is required");
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
  return generate(fs);
}

#define RH_TRY(x)                                                                  \
  do {                                                                             \
    if ((x) != RH_OK) throw std::runtime_error(std::string(#x) + ": " + rh_last_error()); \
  } while (0)

}  // namespace

int main(int argc, char** argv) {
  std::string text, json_path, fixture, out_path, dtype = "f32";
  int devices = 1, gpus = 1, iters = 10;
  uint64_t seed = 0;
  for (int i = 1; i < argc; ++i) {
    std::string a = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) throw std::runtime_error("missing value for " + a);
      return argv[++i];
    };
    if (a == "--text") text = next();
    else if (a == "--json") json_path = next();
    else if (a == "--fixture") fixture = next();
    else if (a == "--devices") devices = std::stoi(next());
    else if (a == "--gpus") gpus = std::stoi(next());
    else if (a == "--dtype") dtype = next();
    else if (a == "--iters") iters = std::stoi(next());
    else if (a == "--seed") seed = std::stoull(next());
    else if (a == "--out") out_path = next();
    else {
      std::cerr << "unknown argument " << a << "\n";
      return 2;
    }
  }
  rh_runtime* rt = nullptr;
  rh_mesh* mesh = nullptr;
  rh_program* prog = nullptr;
  int rc = 0;
  try {
    // -------- the reference, unchanged: graph -> plan (parashard_main.cpp:56-76) --------
    TensorProgram g = LoadGraph(text, json_path, fixture);
    ClusterConfig cluster;
    cluster.machines = 1;
    cluster.gpus_per_machine = devices;
    PlanOptions opts;
    opts.pipeline_stages = -1;  // SPMD plans (pipeline stages: SURVEY §8f-1)
    ExecutionPlan p = plan(g, cluster, opts);
    // -------- the execute tail: strategies -> rh_op records -> librhino_exec --------
    rhino::LoweredProgram lp = rhino::RecoverStrategies(g, p, opts);
    const int n = g.size(), naxes = static_cast<int>(lp.mesh.size());
    std::vector<rh_op> ops(n);
    std::vector<std::vector<int32_t>> ins(n);
    std::vector<std::vector<rh_spec>> in_specs(n);
    for (int i = 0; i < n; ++i) {
      const Operator& op = g.op(i);
      rh_op& r = ops[i];
      r = rh_op{};
      r.kind = static_cast<int32_t>(op.kind);  // same enum order as ir.h:58-70
      r.fn = rhino::ToRhFn(op.fn);
      r.dtype = dtype == "bf16" ? RH_BF16 : RH_F32;
      r.rank = op.output_shape.rank();
      for (int k = 0; k < r.rank; ++k) r.dims[k] = op.output_shape.dims[k];
      ins[i].assign(g.input_indices(i).begin(), g.input_indices(i).end());
      r.n_in = static_cast<int32_t>(ins[i].size());
      r.inputs = ins[i].data();
      r.transpose_a = op.transpose_a;
      r.transpose_b = op.transpose_b;
      r.axis = op.axis;
      r.has_perm = !op.perm.empty();
      for (size_t k = 0; k < op.perm.size(); ++k) r.perm[k] = op.perm[k];
      for (int a = 0; a < naxes; ++a) {
        r.out_spec[a] = rhino::ToRhSpec(lp.strat[a][i].output_spec);
        for (const auto& s : lp.strat[a][i].input_specs) in_specs[i].push_back(rhino::ToRhSpec(s));
      }
      r.in_specs = in_specs[i].data();  // [axis][slot]
    }
    std::vector<int> outs(g.output_indices().begin(), g.output_indices().end());
    std::vector<int> devs(static_cast<size_t>(p.mesh.devices()));
    for (size_t k = 0; k < devs.size(); ++k) devs[k] = static_cast<int>(k) % std::max(1, gpus);
    RH_TRY(rh_runtime_create(static_cast<int>(devs.size()), devs.data(), &rt));
    RH_TRY(rh_mesh_create(rt, naxes, lp.mesh.data(), &mesh));
    RH_TRY(rh_program_load(mesh, ops.data(), n, outs.data(), static_cast<int>(outs.size()), 0, &prog));
    RH_TRY(rh_program_init_synthetic(prog, seed));
    double ms = 0;
    RH_TRY(rh_program_run(prog, iters, &ms));
    if (!out_path.empty()) {
      const TensorShape& s = g.op(outs[0]).output_shape;
      std::vector<char> buf(static_cast<size_t>(s.elems()) * (dtype == "bf16" ? 2 : 4));
      RH_TRY(rh_program_read_full(prog, outs[0], buf.data(), buf.size()));
      std::ofstream(out_path, std::ios::binary).write(buf.data(), static_cast<std::streamsize>(buf.size()));
    }
    int nsteps = 0;
    RH_TRY(rh_program_num_steps(prog, &nsteps));
    std::printf("{\"descriptor\": \"%s\", \"mesh\": %d, \"ops\": %d, \"steps\": %d, \"ms_per_step\": %.6f}\n",
                p.descriptor.c_str(), static_cast<int>(p.mesh.devices()), n, nsteps, ms);
  } catch (const std::exception& e) {
    std::cerr << "rh_execute: error: " << e.what() << "\n";
    rc = 1;
  }
  if (prog) rh_program_destroy(prog);
  if (mesh) rh_mesh_destroy(mesh);
  if (rt) rh_runtime_destroy(rt);
  return rc;
}
