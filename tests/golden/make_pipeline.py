#!/usr/bin/env python3
"""pipeline-parallel training steps, planned by the UNCHANGED reference planner.

  1. The forward fixture at the microbatch size (gpt_like:L:H:B/m) is planned with
     PlanOptions.pipeline_stages = S and microbatches = m on a machines x gpus mesh: the planner
     chooses the pipeline axis, the stage of every op (assign_stages) and every stage's SPMD specs
     on the other axes; rh_plan recovers the strategies per stage and the cut placeholders' specs
     (wire format v2, paper_2302_08141_b200/host/rh_lower.cpp RecoverPipeline).
  2. The backward of that microbatch program (make_fwd_bwd.fwd_bwd_ir) is planned greedily over
     the planner's own candidates on the non-pipeline axes (rh_plan --greedy-after); every backward
     op runs on the stage of the forward op it differentiates.
  3. The step program holds m copies of the microbatch program (one per microbatch, sharing the
     parameters), each op tagged with (stage, microbatch, fwd|bwd); the gradients of each
     parameter are summed over microbatches by add ops tagged LocalAccumulate (taskgraph.cpp:
     149-160) and applied in place by the executor (ApplyGradients, :161-165: p -= lr * g).
  The executor runs every stage's tasks in 1F1B order (taskgraph.cpp:173-211).

    python tests/golden/make_pipeline.py gpt_like:2:64:32 --machines 2 --gpus 2 --stages 2 --microbatches 2
"""
import argparse
import gzip
import json
import os
import subprocess
import sys
import tempfile
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
from make_fwd_bwd import RH_PLAN, forward_graph, fwd_bwd_ir  # noqa: E402

LR = 0.0078125  # 2^-7: exact in bf16


def plan_microbatch(fixture, machines, gpus, stages, m, ilp_limit):
    g = forward_graph(fixture)
    origin = {}
    ir = fwd_bwd_ir(g, origin)
    with tempfile.TemporaryDirectory() as td:
        prog = os.path.join(td, "mb.ir")
        with open(prog, "w") as f:
            f.write(ir)
        out = os.path.join(td, "mb.json")
        r = subprocess.run([RH_PLAN, "--text", prog, "--machines", str(machines), "--gpus", str(gpus), "--equal-bw",
                            "--pipeline-stages", str(stages), "--microbatches", str(m), "--greedy-after",
                            str(len(g["ops"])), "--ilp-time-limit", str(ilp_limit), "-o", out],
                           capture_output=True, text=True)
        if r.returncode:
            raise SystemExit(r.stderr)
        return json.load(open(out)), origin, len(g["ops"])


def step_program(mb, origin, k_fwd, m, name):
    ops = mb["ops"]
    idx = {o["id"]: i for i, o in enumerate(ops)}
    stage = [o["stage"] for o in ops]
    for i, o in enumerate(ops):  # backward ops: the stage of the forward op they differentiate
        if i >= k_fwd and o["id"] in origin:
            stage[i] = stage[idx[origin[o["id"]]]]
    cons = [[] for _ in ops]
    for i, o in enumerate(ops):
        for x in o["inputs"]:
            cons[x].append(i)
    for i, o in enumerate(ops):  # remaining inputs (dy): the stage of their first consumer
        if stage[i] < 0:
            stage[i] = min(stage[c] for c in cons[i] if stage[c] >= 0)
    assert all(s >= 0 for s in stage)
    out_ids = {ops[j]["id"] for j in mb["outputs"]}
    grads = [i for i, o in enumerate(ops) if o["id"].startswith("d_") and o["id"] in out_ids]
    loss_side = [j for j in mb["outputs"] if j not in grads]
    new, where = [], {}

    def add(o, st, mbi, phase):
        o = dict(o)
        o["stage"], o["microbatch"], o["phase"] = st, mbi, phase
        new.append(o)
        return len(new) - 1

    for i, o in enumerate(ops):  # shared parameters
        if o["kind"] == "param":
            where[(i, 0)] = add(dict(o, inputs=[]), stage[i], 1, "fwd")
    for mbi in range(1, m + 1):
        for i, o in enumerate(ops):
            if o["kind"] == "param":
                continue
            ins = [where[(x, 0)] if ops[x]["kind"] == "param" else where[(x, mbi)] for x in o["inputs"]]
            where[(i, mbi)] = add(dict(o, id=f"{o['id']}@{mbi}", inputs=ins), stage[i], mbi,
                                  "fwd" if i < k_fwd else "bwd")
    outputs = [where[(j, mbi)] for mbi in range(1, m + 1) for j in loss_side]
    apply = []
    for gi in grads:
        acc = where[(gi, 1)]
        g = ops[gi]
        for mbi in range(2, m + 1):  # LocalAccumulate: the running sum, in the gradient's layout
            spec = g["out_spec"]
            acc = add({"id": f"{g['id']}@acc{mbi}", "kind": "add", "inputs": [acc, where[(gi, mbi)]],
                       "shape": g["shape"], "elem_bytes": g.get("elem_bytes", 4), "flops": 0.0,
                       "out_spec": spec, "in_specs": [[s, s] for s in spec]}, stage[gi], mbi, "acc")
        outputs.append(acc)
        param = idx[g["id"][2:]]
        apply.append([acc, where[(param, 0)]])
    doc = {"schema": "rhino-lowered/2", "name": name, "descriptor": mb["descriptor"], "mesh": mb["mesh"],
           "dtype": mb.get("dtype", "f32"), "pipeline_axis": mb["pipeline_axis"], "microbatches": m,
           "ops": new, "outputs": outputs, "apply": apply, "lr": LR, "cuts": mb.get("cuts", []),
           "recovery": mb.get("recovery", []), "microbatch_program": {"ops": len(ops), "forward_ops": k_fwd}}
    return doc


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("fixture", help="family:layers:hidden:batch (the whole step's batch)")
    ap.add_argument("--machines", type=int, default=2)
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--stages", type=int, default=2)
    ap.add_argument("--microbatches", type=int, default=2)
    ap.add_argument("--ilp-time-limit", default="60")
    ap.add_argument("--name", default=None)
    a = ap.parse_args()
    fam, layers, hidden, batch = a.fixture.split(":")
    m = a.microbatches
    mb_fixture = f"{fam}:{layers}:{hidden}:{int(batch) // m}"
    t = time.time()
    mb, origin, k_fwd = plan_microbatch(mb_fixture, a.machines, a.gpus, a.stages, m, a.ilp_time_limit)
    name = a.name or f"pp_{fam}_{layers}_{hidden}_{batch}_{a.machines}x{a.gpus}_s{a.stages}_m{m}"
    doc = step_program(mb, origin, k_fwd, m, name)
    out = os.path.join(HERE, "plans", name + ".json")
    text = json.dumps(doc, indent=1)
    if len(text) > (1 << 20):
        with gzip.open(out + ".gz", "wt", compresslevel=9) as f:
            f.write(text)
    else:
        with open(out, "w") as f:
            f.write(text)
    print(f"{name}: {mb['descriptor']} ops={len(doc['ops'])} stages={a.stages} m={m} "
          f"apply={len(doc['apply'])} {time.time() - t:.1f}s")


if __name__ == "__main__":
    main()
