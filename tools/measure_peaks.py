#!/usr/bin/env python3
"""Measured compute peaks that MEASURED_PEAKS.json (driver-written: HBM copy GB/s and cuBLAS bf16)
does not carry: the fp32 programs' roofline denominators.

  tf32_tflops  cuBLAS fp32 GEMM with TF32 tensor cores (torch allow_tf32), 8192^3, best of 10
  fp32_tflops  cuBLAS fp32 GEMM on CUDA cores (allow_tf32 off), 8192^3, best of 5
  bf16_tflops  cuBLAS bf16, 8192^3, best of 10 (cross-check against MEASURED_PEAKS.json)

The 3xTF32 GEMM (k_gemm_tc.cu GemmTf32x3Kernel: three kind::tf32 MMAs per product) is bounded by
tf32_tflops / 3.  Output: profiles/peaks_extra.json (committed; bench.py reads it).

    python tools/measure_peaks.py
"""
import json
import os
import time

import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def best(fn, n, iters):
    ts = []
    for _ in range(iters):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return 2.0 * n ** 3 / (min(ts) * 1e-3) / 1e12


def main():
    n = 8192
    out = {"gpu_name": torch.cuda.get_device_name(0), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "torch": torch.__version__, "n": n}
    x = torch.randn(n, n, device="cuda", dtype=torch.float32)
    y = torch.randn(n, n, device="cuda", dtype=torch.float32)
    torch.backends.cuda.matmul.allow_tf32 = True
    for _ in range(3):
        x @ y
    out["tf32_tflops"] = best(lambda: x @ y, n, 10)
    torch.backends.cuda.matmul.allow_tf32 = False
    x @ y
    out["fp32_tflops"] = best(lambda: x @ y, n, 5)
    xb, yb = x.bfloat16(), y.bfloat16()
    for _ in range(3):
        xb @ yb
    out["bf16_tflops"] = best(lambda: xb @ yb, n, 10)
    out["how"] = "torch.matmul 8192^3 (2*N^3 flops), CUDA events, best of K after warm-up"
    path = os.path.join(REPO, "profiles", "peaks_extra.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
