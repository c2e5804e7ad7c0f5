#!/usr/bin/env python3
"""Evidence run (not in the test suite: ~4 min of CPU oracle): the 24-layer GPT training step
under the planner's pipeline plan (pp_gpt24_2x2_m4: 2 stages x 2-way SPMD, 4 microbatches of 512
tokens, 1F1B, LocalAccumulate + ApplyGradients), 4 ranks emulated on cuda:0, fp32 against the
oracle with the suite's rule (max(1e-5, 2 x the oracle's own fp32-vs-fp64 spread)).  In bf16 this
depth is chaotic (the oracle's own spread is O(1)): bf16 pipelines are gated op by op
(tests/test_gpu_oplevel.py)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import pyoracle  # noqa: E402
from paper_2302_08141_b200 import runtime as rx  # noqa: E402
from paper_2302_08141_b200.abi import RH_BF16, RH_F32, RH_FLAG_NO_GRAPH, RH_FLAG_UNLABELED_IDENTITY  # noqa: E402
from paper_2302_08141_b200.program import LoweredProgram  # noqa: E402


def nw(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


args = [a for a in sys.argv[1:] if not a.startswith("--")]
# --identity: unlabeled unary ops as identity (RH_FLAG_UNLABELED_IDENTITY): without the 90 tanh
# ops per layer the 24-layer fwd+bwd is not chaotic, so the end-to-end comparison discriminates
FLAGS = RH_FLAG_UNLABELED_IDENTITY if "--identity" in sys.argv else 0
DTYPE = RH_BF16 if "--bf16" in sys.argv else RH_F32
prog = LoweredProgram.load(args[0] if args else "pp_gpt24_2x2_m4").with_dtype(DTYPE)
conv = pyoracle.bf16_to_f32 if DTYPE == RH_BF16 else (lambda a: a)
rt = rx.Runtime(devices=[0] * prog.world)
mesh = rx.Mesh(rt, prog.mesh)
t = time.time()
gp = rx.Program(mesh, prog, RH_FLAG_NO_GRAPH | FLAGS)
print(f"{prog.name}: {len(prog.ops)} ops, load {time.time() - t:.1f} s, {len(gp.steps())} steps", flush=True)
gp.init_synthetic(7)
gp.run(1)
outs = {o: conv(gp.read_full(o)) for o in prog.outputs}
gp.close()
mesh.close()
rt.close()
ref = {}
for key, fl in (("f64", pyoracle.OracleProgram.GEMM_F64), ("f32", 0)):
    t = time.time()
    o = pyoracle.OracleProgram(prog, flags=fl | FLAGS)
    o.init_synthetic(7)
    o.run_unpartitioned()
    ref[key] = {k: conv(o.read_full(k, partitioned=False)) for k in prog.outputs}
    print(f"oracle ({key} GEMM accumulation) {time.time() - t:.0f} s", flush=True)
spread = max(nw(ref["f32"][k], ref["f64"][k]) for k in prog.outputs)
worst = max((nw(outs[k], ref["f64"][k]), prog.ops[k].id) for k in prog.outputs)
tol = max(2e-2 if DTYPE == RH_BF16 else 1e-5, 2 * spread)
print(f"{'bf16' if DTYPE == RH_BF16 else 'f32'}{' identity' if FLAGS else ''} "
      f"outputs {len(prog.outputs)}: worst normwise {worst[0]:.3e} ({worst[1]}), oracle spread {spread:.3e}, "
      f"tol {tol:.3e} -> {'PASS' if worst[0] <= tol else 'FAIL'}", flush=True)
