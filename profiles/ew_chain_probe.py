"""Elementwise-chain breakdown of the C5 fwd+bwd step: time and achieved GB/s grouped by chain
signature (ops, inputs, outputs, elements)."""
import collections
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2302_08141_b200 import runtime as rx  # noqa: E402
from paper_2302_08141_b200.abi import RH_BF16  # noqa: E402
from paper_2302_08141_b200.program import LoweredProgram  # noqa: E402

plan = sys.argv[1] if len(sys.argv) > 1 else "c5_big_gpt24_d1"
prog = LoweredProgram.load(plan).with_dtype(RH_BF16)
rt = rx.Runtime(devices=[0] * prog.world)
mesh = rx.Mesh(rt, prog.mesh)
gp = rx.Program(mesh, prog, 0)
gp.init_synthetic(0)
gp.run(2)
gp.profile(3)
st = gp.steps()
print("arena/pool GB", [x / 1e9 for x in gp.memory()])
g = collections.defaultdict(lambda: [0, 0.0, 0.0])
for s in st:
    if s["kind"] != 0:
        continue
    name = s["name"]
    if name.startswith("ew_chain"):
        sig = "ew " + name[name.index("("):]
    else:
        sig = name.split(" ")[0]
    k = (sig, round(s["alg_bytes"] / 1e6, 1))
    g[k][0] += 1
    g[k][1] += s["ms"]
    g[k][2] += s["alg_bytes"]
tot = sum(v[1] for v in g.values())
print(f"kernel steps total {tot:.2f} ms (profiled)")
for (sig, mb), (n, ms, b) in sorted(g.items(), key=lambda kv: -kv[1][1])[:40]:
    print(f"{ms:8.3f} ms  x{n:4d}  {mb:8.1f} MB/launch  {b / (ms * 1e-3) / 1e9:6.0f} GB/s  {sig}")
