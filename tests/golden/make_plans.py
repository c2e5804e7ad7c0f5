#!/usr/bin/env python3
"""Generate the lowered-program fixtures under tests/golden/plans/ with the UNCHANGED reference
planner (oracle/_ref/rh_plan links /root/reference/proj/src/*.cpp, built by `make -C oracle ref`).

Run in the dev container (the reference is not present on the GPU box):
    python tests/golden/make_plans.py [--only NAME]

Each fixture is "rhino-lowered/1" JSON: the program graph, the planner's output specs
(`plan_sharding`, ExecutionPlan.sharding, proj/include/parashard/planner.h:77) and, per op and
mesh axis, the OpStrategy recovered by replaying the search (paper_2302_08141_b200/host/rh_lower.cpp).
"""
import argparse
import gzip
import json
import os
import subprocess
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.abspath(os.path.join(HERE, "..", ".."))
RH_PLAN = os.path.join(REPO, "oracle", "_ref", "rh_plan")
PROG = os.path.join(HERE, "programs")
OUT = os.path.join(HERE, "plans")


def gpt_heads_ir(heads=32, hidden=4096, seq=2048, head_dim=128, score_chain=14):
    """C3 per-head variant: the gpt_like block (proj/src/fixtures.cpp:101-137)
    with attention split into `heads` rank-2 heads joined by Concat (ir.cpp:205-220).  Chain
    lengths are the fixture's own (kGptLn1/kGptScore/kGptMix/kGptGate/kGptLn2/kGptGelu =
    12/14/4/36/12/12, fixtures.cpp:90-99); every head carries the full 14-op score chain."""
    H, B, F, D = hidden, seq, 4 * hidden, head_dim
    L = [f"x = input f32[{B},{H}]"]
    for n in ("wo",):
        L.append(f"{n} = param f32[{H},{H}]")
    L.append(f"w1 = param f32[{H},{F}]")
    L.append(f"w2 = param f32[{F},{H}]")

    def chain(prefix, src, n, shape):
        cur = src
        for i in range(n):
            nid = f"{prefix}_{i:02d}"
            L.append(f"{nid} = unary({cur}) : f32[{shape}]")
            cur = nid
        return cur

    n1 = chain("ln1", "x", 12, f"{B},{H}")
    ctxs = []
    for h in range(heads):
        p = f"h{h:02d}"
        for w in ("wq", "wk", "wv"):
            L.append(f"{p}_{w} = param f32[{H},{D}]")
        L.append(f"{p}_q = matmul({n1}, {p}_wq)")
        L.append(f"{p}_k = matmul({n1}, {p}_wk)")
        L.append(f"{p}_v = matmul({n1}, {p}_wv)")
        L.append(f"{p}_score = matmul({p}_q, {p}_k^T)")
        sm = chain(f"{p}_smax", f"{p}_score", score_chain, f"{B},{B}")
        L.append(f"{p}_ctx = matmul({sm}, {p}_v)")
        ctxs.append(f"{p}_ctx")
    L.append(f"attn = concat({', '.join(ctxs)}) : f32[{B},{H}] {{axis=1}}")
    L.append("proj = matmul(attn, wo)")
    mix = chain("mix", "proj", 4, f"{B},{H}")
    gate = chain("gate", "x", 36, f"{B},{H}")
    L.append(f"res1 = add({gate}, {mix})")
    n2 = chain("ln2", "res1", 12, f"{B},{H}")
    L.append(f"ffn1 = matmul({n2}, w1)")
    gl = chain("gelu", "ffn1", 12, f"{B},{F}")
    L.append(f"ffn2 = matmul({gl}, w2)")
    L.append("res2 = add(res1, ffn2)")
    L.append("@outputs res2")
    return "\n".join(L) + "\n"


def jobs():
    J = []
    c1 = os.path.join(PROG, "c1_mlp.ir")
    for d in (1, 2, 4, 8):
        J.append((f"c1_mlp_d{d}", ["--text", c1, "--devices", str(d)]))
    J.append(("c1_fixture_mlp_d4", ["--fixture", "mlp:2:1024:64", "--devices", "4"]))
    for d in (2, 4, 8):
        J.append((f"c2_mlp_reshape_d{d}",
                  ["--text", os.path.join(PROG, "c2_mlp_reshape.ir"), "--devices", str(d)]))
        J.append((f"c2_mlp_pinned_d{d}",
                  ["--json", os.path.join(PROG, "c2_mlp_pinned.json"), "--devices", str(d)]))
    g = "gpt_like:1:4096:2048"
    for d in (1, 2, 4, 8):
        J.append((f"c3_gpt_block_d{d}", ["--fixture", g, "--devices", str(d)]))
    J.append(("c3_gpt_block_2x2", ["--fixture", g, "--machines", "2", "--gpus", "2", "--equal-bw"]))
    J.append(("c3_gpt_block_2x4", ["--fixture", g, "--machines", "2", "--gpus", "4", "--equal-bw"]))
    # small programs exercising every op kind / rule (reduce_sum, broadcast, transpose, mul)
    for d in (2, 4):
        J.append((f"moe_small_d{d}", ["--fixture", "moe_like:1:64:32", "--devices", str(d)]))
        J.append((f"gpt_small_d{d}", ["--fixture", "gpt_like:1:64:32", "--devices", str(d)]))
        J.append((f"skipnet_small_d{d}", ["--fixture", "skipnet:4:64:32", "--devices", str(d)]))
    J.append(("gpt_small_2x2", ["--fixture", "gpt_like:1:64:32", "--machines", "2", "--gpus", "2",
                                "--equal-bw"]))
    # random legal strategy choices: every candidate combination is a valid partitioned program
    for seed in range(6):
        for fam, mesh in (("moe_like:1:64:32", "4"), ("gpt_like:1:64:32", "2,2"),
                          ("mlp:2:64:32", "8")):
            short = fam.split(":")[0]
            J.append((f"rand_{short}_{mesh.replace(',', 'x')}_s{seed}",
                      ["--fixture", fam, "--random-choice", str(seed), "--mesh", mesh]))
    # C5's forward pass alone (24 layers, H 2048, 2048 tokens): the oracle-checked forward
    J.append(("c5_big_gpt24_fwd_d1", ["--fixture", "gpt_like:24:2048:2048", "--devices", "1"]))
    heads = os.path.join(PROG, "c3_gpt_heads32.ir")
    for d in (1, 2, 4, 8):
        J.append((f"c3_gpt_heads32_d{d}", ["--text", heads, "--devices", str(d)]))
    return J


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default=None)
    args = ap.parse_args()
    os.makedirs(OUT, exist_ok=True)
    with open(os.path.join(PROG, "c3_gpt_heads32.ir"), "w") as f:
        f.write(gpt_heads_ir())
    for name, argv in jobs():
        if args.only and args.only not in name:
            continue
        t = time.time()
        out = os.path.join(OUT, name + ".json")
        r = subprocess.run([RH_PLAN, *argv, "--name", name, "-o", out], capture_output=True, text=True)
        if r.returncode != 0:
            print(f"FAILED {name}: {r.stderr}", file=sys.stderr)
            sys.exit(1)
        j = json.load(open(out))
        rec = ",".join(f"{x['ilp_status']}/{'ok' if x['replay_matched'] else 'fallback'}"
                       for x in j["recovery"])
        print(f"{name:32s} mesh={j['mesh']} ops={len(j['ops'])} {rec} {time.time() - t:.1f}s")
        if os.path.getsize(out) > (1 << 20):  # large plans are committed gzipped
            with open(out, "rb") as f, gzip.open(out + ".gz", "wb", compresslevel=9) as g:
                g.write(f.read())
            os.remove(out)


if __name__ == "__main__":
    main()
