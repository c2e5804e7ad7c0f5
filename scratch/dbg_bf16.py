import sys, numpy as np
sys.path.insert(0, "/root/repo")
from oracle import pyoracle as O
from paper_2302_08141_b200 import runtime as rx
from paper_2302_08141_b200.abi import *
from paper_2302_08141_b200.program import LoweredProgram
def nw(a,b): a=a.astype(np.float64); b=b.astype(np.float64); return np.abs(a-b).max()/np.abs(b).max()
name = sys.argv[1]
prog = LoweredProgram.load(name).with_dtype(RH_BF16)
o = O.OracleProgram(prog, keep_all=True); o.init_synthetic(13); o.run_partitioned()
for flags in [0, RH_FLAG_SIMT_GEMM, RH_FLAG_NO_FUSION, RH_FLAG_NO_FUSION|RH_FLAG_SIMT_GEMM]:
    rt = rx.Runtime(devices=[0]*prog.world); mesh = rx.Mesh(rt, prog.mesh); gp = rx.Program(mesh, prog, flags)
    gp.init_synthetic(13); gp.run(1)
    out = prog.outputs[0]
    print(flags, "out err", nw(O.bf16_to_f32(gp.read_full(out)), O.bf16_to_f32(o.read_full(out, True))), flush=True)
    if flags & RH_FLAG_NO_FUSION:
        for op in prog.ops:
            g = O.bf16_to_f32(gp.read_local(op.index, 0)); w = O.bf16_to_f32(o.read_local(op.index, 0))
            e = nw(g, w) if np.abs(w).max() > 0 else np.abs(g).max()
            if e > 2e-2: print("   first bad op", op.index, op.id, prog.ops[op.index].kind, e, [s for s in gp.steps() if f"op{op.index} " in s["name"] or s["name"].endswith(f"op{op.index}")][:3]); break
    gp.close(); mesh.close(); rt.close()
