import sys, os
sys.path.insert(0, "/root/repo")
from paper_2302_08141_b200 import runtime as rx
from paper_2302_08141_b200.abi import RH_BF16
from paper_2302_08141_b200.program import LoweredProgram
prog = LoweredProgram.load("c5_big_gpt24_d1").with_dtype(RH_BF16)
rt = rx.Runtime(devices=[0]); mesh = rx.Mesh(rt, [1]); gp = rx.Program(mesh, prog, 0)
gp.init_synthetic(0); gp.run(2); gp.profile(2)
st = gp.steps()
ew = [s for s in st if s["name"].startswith("ew_chain")]
print("arena/pool GB", [x / 1e9 for x in gp.memory()])
print("n ew", len(ew), "total ms", sum(s["ms"] for s in ew))
for s in sorted(ew, key=lambda s: -s["ms"])[:25]:
    print(f'{s["ms"]*1e3:8.1f} us {s["alg_bytes"]/1e6:8.1f} MB {s["alg_bytes"]/(s["ms"]*1e-3)/1e9:7.0f} GB/s  {s["name"]}')
# one layer's worth in order
for s in st[:80]:
    print(f'{s["ms"]*1e3:8.1f} us {s["alg_bytes"]/1e6:8.1f} MB  {s["name"]}')
