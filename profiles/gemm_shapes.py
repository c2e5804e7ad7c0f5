"""Single-GEMM microbenchmark: the tcgen05 kernel (one-op programs through the C-ABI, graph
replays) against cuBLAS (torch.matmul, the library yardstick) on the shapes the C3/C5 plans run.

  python profiles/gemm_shapes.py [--iters 50] [--flags 0] > gpurun_out/gemm_shapes.txt
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_08141_b200 import runtime as rx  # noqa: E402
from paper_2302_08141_b200.program import LoweredProgram  # noqa: E402
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_gemm import matmul_doc  # noqa: E402

# (m, k, n, transpose_a, transpose_b): C3 at N=1/2/4/8 and the C5 layer (H=2048, 2048 tokens)
# forward (NN) and backward (NT: dx = dy w^T, TN: dw = x^T dy) GEMMs
SHAPES = [
    (2048, 4096, 16384, 0, 0), (2048, 16384, 4096, 0, 0), (2048, 4096, 4096, 0, 0),
    (2048, 4096, 2048, 0, 0), (2048, 2048, 2048, 0, 0), (2048, 4096, 1024, 0, 0),
    (2048, 1024, 4096, 0, 0), (2048, 2048, 8192, 0, 0), (2048, 8192, 2048, 0, 0),
    (2048, 2048, 2048, 0, 1), (2048, 2048, 2048, 1, 0), (2048, 8192, 2048, 0, 1),
    (8192, 2048, 2048, 1, 0), (2048, 2048, 8192, 1, 0), (1024, 4096, 4096, 0, 0),
    (512, 4096, 4096, 0, 0),
    # fixed overhead vs mainloop rate: 128 tiles (2048 x 4096 output), K swept
    (2048, 8192, 4096, 0, 0), (2048, 16384, 4096, 0, 0),
    # 148-SM-friendly tile counts
    (2048, 4096, 9472, 0, 0), (4736, 4096, 2048, 0, 0),
    # C3 at N=4 (row-split FFN: 512-row shards) and N=2
    (512, 16384, 4096, 0, 0), (512, 4096, 16384, 0, 0), (1024, 16384, 4096, 0, 0), (1024, 4096, 16384, 0, 0),
]


os.environ.setdefault("RH_NO_GEMM_GROUP", "1")  # the reps below would otherwise be one grouped launch


def ours(m, k, n, ta, tb, iters, flags, reps=16):
    # reps independent matmuls of the same operands in one program (one graph): per-GEMM time
    # includes the inter-kernel gap, as inside a real program, not a graph launch per GEMM
    doc = matmul_doc(m, k, n, bool(tb), ta=bool(ta))
    for r in range(1, reps):
        op = dict(doc["ops"][2], id=f"c{r}")
        doc["ops"].append(op)
    doc["outputs"] = list(range(2, 2 + reps))
    prog = LoweredProgram(doc)
    rt = rx.Runtime(devices=[0])
    mesh = rx.Mesh(rt, [1])
    gp = rx.Program(mesh, prog, flags)
    try:
        gp.init_synthetic(1)
        gp.run(5)
        ms = min(gp.run(max(1, iters // reps)) for _ in range(3)) / reps
        name = [s["name"] for s in gp.steps() if s["name"].startswith("gemm")][0]
    finally:
        gp.close()
        mesh.close()
        rt.close()
    return ms, name


def cublas(m, k, n, ta, tb, iters):
    a = torch.randn((k, m) if ta else (m, k), device="cuda", dtype=torch.bfloat16)
    b = torch.randn((n, k) if tb else (k, n), device="cuda", dtype=torch.bfloat16)
    A = a.t() if ta else a
    B = b.t() if tb else b
    c = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
    for _ in range(5):
        torch.matmul(A, B, out=c)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(iters):
            torch.matmul(A, B, out=c)
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / iters)
    return best


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=50)
    ap.add_argument("--flags", type=int, default=0)
    ap.add_argument("--no-cublas", action="store_true")
    ap.add_argument("--shapes", default=None, help="m,k,n,ta,tb;... (default: the plan shapes)")
    args = ap.parse_args()
    shapes = SHAPES if not args.shapes else [tuple(int(v) for v in s.split(",")) for s in args.shapes.split(";")]
    print(f"{'m':>5} {'k':>6} {'n':>6} ta tb | {'ours us':>8} {'TF/s':>6} | {'cuBLAS us':>9} {'TF/s':>6} | schedule")
    for m, k, n, ta, tb in shapes:
        fl = 2.0 * m * k * n
        ms, name = ours(m, k, n, ta, tb, args.iters, args.flags)
        cb = float("nan") if args.no_cublas else cublas(m, k, n, ta, tb, args.iters)
        print(f"{m:5d} {k:6d} {n:6d} {ta:2d} {tb:2d} | {ms*1e3:8.1f} {fl/ms/1e9:6.0f} | {cb*1e3:9.1f} "
              f"{fl/cb/1e9:6.0f} | {name}", flush=True)


if __name__ == "__main__":
    main()
