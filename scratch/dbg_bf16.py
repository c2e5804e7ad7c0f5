import sys, numpy as np
sys.path.insert(0, "/root/repo")
from oracle import pyoracle as O
from paper_2302_08141_b200 import runtime as rx
from paper_2302_08141_b200.abi import *
from paper_2302_08141_b200.program import LoweredProgram
def nw(a,b): a=a.astype(np.float64); b=b.astype(np.float64); return np.abs(a-b).max()/max(np.abs(b).max(),1e-30)
for name in sys.argv[1:]:
    prog = LoweredProgram.load(name).with_dtype(RH_BF16)
    o = O.OracleProgram(prog, keep_all=True); o.init_synthetic(13); o.run_partitioned()
    flags = RH_FLAG_NO_FUSION
    rt = rx.Runtime(devices=[0]*prog.world); mesh = rx.Mesh(rt, prog.mesh); gp = rx.Program(mesh, prog, flags)
    gp.init_synthetic(13); gp.run(1)
    print(name, [s["name"] for s in gp.steps() if s["kind"]==1])
    for op in prog.ops:
        g = O.bf16_to_f32(gp.read_local(op.index, 0)); w = O.bf16_to_f32(o.read_local(op.index, 0))
        e = nw(g, w)
        if e > 1e-3 and ("_08" in op.id or not "_" in op.id[4:] or op.kind not in (5,)): print(f"  {op.index:3d} {op.id:14s} kind={op.kind} err={e:.3e} spec={[str(s) for s in op.out_spec]} maxabs={np.abs(w).max():.3f}")
    gp.close(); mesh.close(); rt.close()
