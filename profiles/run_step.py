#!/usr/bin/env python3
"""Small driver for ncu captures (profiles/README.md): load a plan, init, run W warm-up steps
and K steps of the partitioned program on cuda:0 (emulated ranks when the plan has several)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2302_08141_b200 import runtime as rx  # noqa: E402
from paper_2302_08141_b200.abi import RH_BF16, RH_F32  # noqa: E402
from paper_2302_08141_b200.program import LoweredProgram  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--plan", default="c3_gpt_block_d1")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--flags", type=int, default=0)
    a = ap.parse_args()
    prog = LoweredProgram.load(a.plan).with_dtype(RH_BF16 if a.dtype == "bf16" else RH_F32)
    rt = rx.Runtime(devices=[0] * prog.world)
    mesh = rx.Mesh(rt, prog.mesh)
    gp = rx.Program(mesh, prog, a.flags)
    gp.init_synthetic(0)
    gp.run(a.warmup)
    ms = gp.run(a.steps)
    print(f"{a.plan} {a.dtype}: {ms:.3f} ms/step, steps: {len(gp.steps())}")
    gp.close()
    mesh.close()
    rt.close()


if __name__ == "__main__":
    main()
