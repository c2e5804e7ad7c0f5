"""Every step of a plan's schedule with its profiled time (one GPU, emulated ranks)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_08141_b200 import runtime as rx  # noqa: E402
from paper_2302_08141_b200.abi import RH_BF16  # noqa: E402
from paper_2302_08141_b200.program import LoweredProgram  # noqa: E402

plan = sys.argv[1] if len(sys.argv) > 1 else "c3_gpt_block_d1"
prog = LoweredProgram.load(plan).with_dtype(RH_BF16)
rt = rx.Runtime(devices=[0] * prog.world)
mesh = rx.Mesh(rt, prog.mesh)
gp = rx.Program(mesh, prog, 0)
gp.init_synthetic(0)
gp.run(3)
print(f"{plan}: {gp.run(10) * 1e3:.1f} us/step (graph), profiled {gp.profile(5) * 1e3:.1f} us/step")
for s in gp.steps():
    gbs = s["alg_bytes"] / (s["ms"] * 1e-3) / 1e9 if s["ms"] else 0
    tf = s["alg_flops"] / (s["ms"] * 1e-3) / 1e12 if s["ms"] else 0
    print(f"  {s['ms'] * 1e3:8.1f} us  {s['alg_bytes'] / 1e6:8.1f} MB {gbs:6.0f} GB/s {tf:6.0f} TF/s  {s['name']}")
gp.close()
mesh.close()
rt.close()
