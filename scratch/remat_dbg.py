import os, sys
sys.path.insert(0, os.getcwd())
os.environ["RH_REMAT"] = "1"; os.environ["RH_REMAT_DEBUG"] = "1"
from paper_2302_08141_b200 import runtime as rx
from paper_2302_08141_b200.program import LoweredProgram
from paper_2302_08141_b200.abi import RH_BF16
prog = LoweredProgram.load("c5_big_gpt1_d1").with_dtype(RH_BF16)
rt = rx.Runtime(devices=[0]); mesh = rx.Mesh(rt, prog.mesh); gp = rx.Program(mesh, prog, 0)
for s in gp.steps():
    if s["name"].startswith("ew_chain"): print(s["name"], s["alg_bytes"] / 2**20, "MiB")
