"""HBM read-only / write-only / copy bandwidth on this B200 (torch kernels, CUDA events): the
ceiling for write-heavy elementwise chains (a forward tanh chain writes 12 outputs per input)."""
import torch

n = 1 << 29  # 1 GiB of bf16
a = torch.empty(n, dtype=torch.bfloat16, device="cuda").uniform_()
b = torch.empty_like(a)
outs = [torch.empty(n // 12, dtype=torch.bfloat16, device="cuda") for _ in range(12)]


def t(fn, it=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it * 1e-3


s = t(lambda: b.fill_(1.0))
print(f"write-only fill: {2 * n / s / 1e9:.0f} GB/s")
s = t(lambda: a.sum())
print(f"read-only sum: {2 * n / s / 1e9:.0f} GB/s")
s = t(lambda: b.copy_(a))
print(f"copy: {4 * n / s / 1e9:.0f} GB/s (read+write)")
s = t(lambda: [o.fill_(1.0) for o in outs])
print(f"12 x fill (sequential kernels): {2 * n / s / 1e9:.0f} GB/s")
