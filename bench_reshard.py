#!/usr/bin/env python3
"""C4 (BASELINE.json configs[3]): the resharding microbenchmark sweep.

All spec-to-spec transitions of one mesh axis on [N, 4096] tensors (fp32 / bf16), tensor sizes
1 MiB .. 4 GiB, through rh_reshard (the executor's transition path: peer-memory pull kernels with
group barriers, or --transport nccl for the NCCL baseline).  Specs: R, S0, S1, strided S0~s /
S1~s for s in {1, 8, 64}, and P as a source.  One JSON line per case:
  busbw_gbs  = reshard_cost wire bytes (proj/src/sharding.cpp:104-142) / time, vs NVLink 770 GB/s
  hbm_gbs    = algorithmic HBM bytes of the rank's kernel (reads + writes) / time, vs 6552 GB/s

  torchrun --nproc-per-node N bench_reshard.py            # one process per GPU (dist mode)
  python bench_reshard.py --emulate 8                      # 8 ranks on cuda:0 (local copies only)
"""
import argparse
import json
import os
import re
import sys

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

HBM_PEAK, NVLINK_PEAK = 6552.3, 770.0


def specs_for(d):
    out = ["replicated", "shard(0,max)", "shard(1,max)"]
    for s in (1, 8, 64):
        out += [f"shard(0,{s})", f"shard(1,{s})"]
    return out


def resolve(s, dims, d):
    from paper_2302_08141_b200.abi import AxisSpec
    if "max" in s:
        dim = int(s[6])
        return AxisSpec.shard(dim, dims[dim] // d)
    return AxisSpec.from_string(s)


def wire_bytes(fs, ts, S, d):
    frac = (d - 1) / d
    if fs.kind == 2:
        return 2 * frac * S if ts.kind == 1 else frac * S
    if fs.kind == 0:
        return S / d * frac if ts.kind == 0 else frac * S
    return 0.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--sizes", default="1M,16M,256M,1G,4G")
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--emulate", type=int, default=0)
    ap.add_argument("--transport", default="p2p", choices=["p2p", "nccl"])
    ap.add_argument("--pairs", default="all", help="all | quick | FROM:TO[,FROM:TO]")
    ap.add_argument("--flags", type=lambda x: int(x, 0), default=0, help="extra rh_program flags")
    a = ap.parse_args()

    import torch

    from paper_2302_08141_b200 import dist as D
    from paper_2302_08141_b200 import runtime as rx
    from paper_2302_08141_b200.abi import RH_BF16, RH_F32, RH_FLAG_TRANSPORT_NCCL

    world, rank, local = D.env()
    if a.emulate:
        d = a.emulate
        rt = rx.Runtime(devices=[0] * d)
    else:
        d = world
        torch.cuda.set_device(local)
        rt = D.make_runtime()
    mesh = rx.Mesh(rt, [d])
    dtype = RH_BF16 if a.dtype == "bf16" else RH_F32
    eb = 2 if dtype == RH_BF16 else 4
    flags = (RH_FLAG_TRANSPORT_NCCL if a.transport == "nccl" else 0) | a.flags
    mult = {"K": 1 << 10, "M": 1 << 20, "G": 1 << 30}
    sizes = [int(x[:-1]) * mult[x[-1]] for x in a.sizes.split(",")]
    names = specs_for(d)
    if a.pairs == "all":
        pairs = [(f, t) for f in names + ["partial"] for t in names if f != t]
    elif a.pairs == "quick":
        pairs = [("partial", "replicated"), ("partial", "shard(0,max)"), ("shard(0,max)", "replicated"),
                 ("shard(1,max)", "shard(0,max)"), ("replicated", "shard(0,max)"), ("shard(1,1)", "shard(0,max)")]
    else:
        spec = r"(?:[a-z]+\([^)]*\)|[a-z]+)"  # commas inside shard(dim,stride) are not separators
        pairs = re.findall(rf"({spec}):({spec})", a.pairs)
    n_local = rt.n_local
    results = []
    for S in sizes:
        rows = S // (4096 * eb)
        dims = [rows, 4096]
        for fname, tname in pairs:
            fs, ts = resolve(fname, dims, d), resolve(tname, dims, d)
            if fs == ts or rows % (d * 64) != 0:
                continue
            n_src = S // eb // (d if fs.kind == 0 else 1)
            n_dst = S // eb // (d if ts.kind == 0 else 1)
            tdt = torch.bfloat16 if dtype == RH_BF16 else torch.float32
            src = [torch.randn(n_src, device="cuda", dtype=tdt) for _ in range(n_local)]
            dst = [torch.empty(n_dst, device="cuda", dtype=tdt) for _ in range(n_local)]
            torch.cuda.synchronize()
            ms = mesh.reshard(0, fs, ts, dims, dtype, [x.data_ptr() for x in src],
                              [x.data_ptr() for x in dst], flags, a.iters)
            ms = D.max_over_ranks(ms) if not a.emulate else ms
            wb = wire_bytes(fs, ts, S, d)
            reads = n_dst * eb * (d if fs.kind == 2 else 1)
            hbm = (reads + n_dst * eb) * (n_local if a.emulate else 1)
            r = {"from": fname, "to": tname, "bytes": S, "d": d, "dtype": a.dtype, "ms": ms,
                 "wire_bytes": wb, "busbw_gbs": wb / (ms * 1e-3) / 1e9 if wb else None,
                 "hbm_gbs": hbm / (ms * 1e-3) / 1e9, "transport": a.transport,
                 "mode": "emulated" if a.emulate else "dist"}
            r["busbw_frac"] = r["busbw_gbs"] / NVLINK_PEAK if r["busbw_gbs"] else None
            r["hbm_frac"] = r["hbm_gbs"] / HBM_PEAK
            results.append(r)
            if rank == 0:
                print(json.dumps(r), flush=True)
            del src, dst
            torch.cuda.empty_cache()
    mesh.close()
    rt.close()


if __name__ == "__main__":
    main()
