"""One GEMM shape as a one-op program (for ncu): python profiles/gemm_one.py M K N [ta tb] [iters]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from paper_2302_08141_b200 import runtime as rx  # noqa: E402
from paper_2302_08141_b200.program import LoweredProgram  # noqa: E402
from test_gpu_gemm import matmul_doc  # noqa: E402

m, k, n = (int(v) for v in sys.argv[1:4])
ta, tb = (int(sys.argv[4]), int(sys.argv[5])) if len(sys.argv) > 5 else (0, 0)
iters = int(sys.argv[6]) if len(sys.argv) > 6 else 3
prog = LoweredProgram(matmul_doc(m, k, n, bool(tb), ta=bool(ta)))
rt = rx.Runtime(devices=[0])
mesh = rx.Mesh(rt, [1])
gp = rx.Program(mesh, prog, 0)
gp.init_synthetic(1)
ms = gp.run(iters)
print(f"{m}x{k}x{n} ta={ta} tb={tb}: {ms * 1e3:.1f} us/iter, {2.0 * m * k * n / ms / 1e9:.0f} TFLOP/s, "
      f"launches/iter {gp.launch_count()}, steps {[s['name'] for s in gp.steps()]}")
gp.close()
mesh.close()
rt.close()
