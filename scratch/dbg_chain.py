import sys, numpy as np
sys.path.insert(0, "/root/repo")
from oracle import pyoracle as O
from paper_2302_08141_b200 import runtime as rx
from paper_2302_08141_b200.abi import *
from paper_2302_08141_b200.program import LoweredProgram
R=["replicated"]
def doc(n, fns, dtype):
    ops=[{"id":"x","kind":"input","inputs":[],"shape":[n],"out_spec":R,"in_specs":[[]]}]
    for i,f in enumerate(fns):
        ops.append({"id":f"u{i}","kind":"unary","fn":f,"inputs":[i],"shape":[n],"out_spec":R,"in_specs":[R]})
    return {"schema":"rhino-lowered/1","name":"chain","mesh":[1],"dtype":dtype,"ops":ops,"outputs":[len(ops)-1]}
for dtype in ["bf16","f32"]:
  for fns in [[""]*4, ["tanh"]*3, ["relu","neg","gelu","sigmoid","exp","rsqrt"]]:
    for flags in [0, RH_FLAG_NO_FUSION]:
        prog = LoweredProgram(doc(4096, fns, dtype))
        o = O.OracleProgram(prog, keep_all=True); o.init_synthetic(1); o.run_partitioned()
        rt = rx.Runtime(devices=[0]); mesh = rx.Mesh(rt, [1]); gp = rx.Program(mesh, prog, flags)
        gp.init_synthetic(1); gp.run(1)
        res=[]
        for op in prog.ops:
            if flags==0 and op.index not in (0, len(prog.ops)-1): continue
            g=gp.read_local(op.index,0); w=o.read_local(op.index,0)
            if dtype=="bf16":
                nd = int((g!=w).sum()); gi=g.astype(np.int32); wi=w.astype(np.int32)
                res.append((op.id, nd, int(np.abs(gi-wi).max())))
            else:
                res.append((op.id, int((g!=w).sum()), float(np.abs(g-w).max())))
        print(dtype, fns, flags, res, flush=True)
        gp.close(); mesh.close(); rt.close()
