"""Per-GEMM step times of a plan (profiled pass), for A/B runs of GEMM schedules."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_08141_b200 import runtime as rx
from paper_2302_08141_b200.abi import RH_BF16
from paper_2302_08141_b200.program import LoweredProgram
plan = sys.argv[1] if len(sys.argv) > 1 else "c3_gpt_block_d1"
prog = LoweredProgram.load(plan).with_dtype(RH_BF16)
rt = rx.Runtime(devices=[0] * prog.world); mesh = rx.Mesh(rt, prog.mesh); gp = rx.Program(mesh, prog, 0)
gp.init_synthetic(0); gp.run(3)
ms = gp.run(10)
gp.profile(5)
tot = 0
rows = {}
for s in gp.steps():
    if s["name"].startswith("gemm"):
        tot += s["ms"]
        ops = prog.ops[int(s["name"].split("op")[1].split(" ")[0])]
        key = (tuple(ops.shape), s["alg_flops"])
        rows.setdefault(key, []).append(s["ms"])
print(f"{plan}: run {ms*1e3:.1f} us/step, gemm total {tot*1e3:.1f} us (profiled)")
for (shape, fl), v in sorted(rows.items(), key=lambda kv: -sum(kv[1])):
    m = sum(v) / len(v)
    print(f"  out {shape} {fl/1e9:7.1f} GFLOP x{len(v):3d}: {m*1e3:7.1f} us  {fl/(m*1e-3)/1e12:6.0f} TFLOP/s")
print("  schedules:", sorted({s["name"].split(" ", 2)[-1] if "[" in s["name"] else "plain" for s in gp.steps() if s["name"].startswith("gemm")}))
