"""torchrun worker for the multi-GPU parity tests (tests/test_gpu_dist.py): one process per GPU,
executor in dist mode (CUDA-IPC peer buffers + NCCL per mesh axis).  Every rank checks its own
local buffers against the CPU oracle's partitioned execution (bit-exact for data movement) and
the materialized outputs against the oracle's single-device result; rank 0 prints one JSON line.
"""
import json
import os
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

from oracle import pyoracle  # noqa: E402
from paper_2302_08141_b200 import dist as D  # noqa: E402
from paper_2302_08141_b200 import runtime as rx  # noqa: E402
from paper_2302_08141_b200.abi import (RH_BF16, RH_FLAG_KEEP_ALL, RH_FLAG_NO_FUSION, RH_FLAG_SIMT_GEMM,  # noqa: E402
                                       RH_FLAG_TRANSPORT_NCCL)
from paper_2302_08141_b200.program import LoweredProgram  # noqa: E402

DATA_MOVEMENT = {0, 1, 6, 7, 9, 10}
_ORACLES = {}


def normwise(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def check(rt, name, flags, dtype=None):
    print(f"[dist r{rt.first_rank}] {name} flags={flags} dtype={dtype}", file=sys.stderr, flush=True)
    prog = LoweredProgram.load(name)
    if dtype is not None:
        prog = prog.with_dtype(dtype)
    mesh = rx.Mesh(rt, prog.mesh)
    # NO_FUSION runs read every op's local buffer afterwards: keep all intermediates
    gp = rx.Program(mesh, prog, flags | (RH_FLAG_KEEP_ALL if flags & RH_FLAG_NO_FUSION else 0))
    res = {"name": name, "flags": flags, "ok": True, "err": 0.0}
    try:
        gp.init_synthetic(21)
        gp.run(3)
        key = (name, prog.dtype)
        if key not in _ORACLES and not (prog.dtype == RH_BF16 and name.startswith("c3_")):
            o = pyoracle.OracleProgram(prog, keep_all=True)
            o.init_synthetic(21)
            threads = max(1, (os.cpu_count() or 2) // max(1, rt.world))  # torchrun sets OMP=1
            o.run_unpartitioned(threads)
            if not name.startswith("c3_"):
                o.run_partitioned(threads)
            _ORACLES[key] = o
        o = _ORACLES.get(key)
        bf = prog.dtype == RH_BF16
        # fp32 GPT block: fp32-accumulation forward error of the 108-op block (~6e-5, see
        # test_gpu_parity.test_gpt_block_fp32 for the rule); everything else 1e-5.
        tol = 2e-2 if bf else (2e-4 if name.startswith("c3_") else 1e-5)
        conv = pyoracle.bf16_to_f32 if bf else (lambda a: a)
        if bf and name.startswith("c3_"):
            # bf16 full block: compare with the SAME partitioned program run as emulated ranks on
            # this GPU (test_gpu_parity checks that one against the oracle).  The peer-memory
            # transport must reproduce it bit for bit (same kernels, same rank-order sums).
            rt_e = rx.Runtime(devices=[rt.first_rank] * prog.world)
            mesh_e = rx.Mesh(rt_e, prog.mesh)
            ge = rx.Program(mesh_e, prog, flags & ~RH_FLAG_TRANSPORT_NCCL)
            ge.init_synthetic(21)
            ge.run(1)
            for out in prog.outputs:
                got, want = gp.read_full(out), ge.read_full(out)
                if flags & RH_FLAG_TRANSPORT_NCCL:  # NCCL sums in its own order
                    e = normwise(conv(got), conv(want))
                    res["ok"] &= e <= tol
                else:
                    e = float(np.count_nonzero(got != want))
                    res["ok"] &= e == 0
                res["err"] = max(res["err"], e)
            ge.close()
            mesh_e.close()
            rt_e.close()
            if rt.first_rank == 0 and not (flags & RH_FLAG_TRANSPORT_NCCL):
                # ... and that result against the bf16 oracle of the same partitioned program
                # (rule of test_gpu_parity.test_gpt_block_bf16), on rank 0 with every host core
                ref = {}
                for key_, fl in (("f64", pyoracle.OracleProgram.GEMM_F64), ("f32", 0)):
                    oo = pyoracle.OracleProgram(prog, flags=fl)
                    oo.init_synthetic(21)
                    oo.run_partitioned(os.cpu_count() or 1)
                    ref[key_] = conv(oo.read_full(prog.outputs[0], partitioned=True))
                tol_o = max(2e-2, 2.0 * normwise(ref["f32"], ref["f64"]))
                e = normwise(conv(gp.read_full(prog.outputs[0])), ref["f64"])
                res["oracle_err"] = e
                res["ok"] &= e <= tol_o
            D.barrier()  # the other ranks wait here (host), not in a device barrier of the next run
        else:
            for out in prog.outputs:
                e = normwise(conv(gp.read_full(out)), conv(o.read_full(out, partitioned=False)))
                res["err"] = max(res["err"], e)
                res["ok"] &= e <= tol
        if flags == 0 and any(op.id == "x" for op in prog.ops):
            # pipelined host path vs the serial one on the same host x: outputs[0] read back as
            # this process's 1/world slice of the materialized tensor, bit-identical
            x = prog.op_index("x")
            out0 = prog.outputs[0]
            xf = np.random.default_rng(5).uniform(-1, 1, prog.full_bytes(x) // prog.elem_bytes()).astype(np.float32)
            xin = (xf.view(np.uint32) >> 16).astype(np.uint16) if bf else xf
            want = np.zeros(prog.full_bytes(out0), np.uint8)
            got = np.zeros(prog.full_bytes(out0), np.uint8)
            gp.step_host([x], [xin.ctypes.data], [want.ctypes.data])
            gp.run_host(5, [x], [xin.ctypes.data], [got.ctypes.data])  # stage buffers reused
            part = want.size // rt.world
            sl = slice(part * rt.first_rank, part * (rt.first_rank + 1))
            res["ok"] &= bool(np.array_equal(got[sl], want[sl])) and bool(want[sl].any())
        if flags & RH_FLAG_NO_FUSION:
            exact = set()
            for op in prog.ops:
                if op.kind in DATA_MOVEMENT and all(i in exact for i in op.inputs):
                    exact.add(op.index)
            for op in prog.ops:
                got = gp.read_local(op.index, rt.first_rank)
                want = o.read_local(op.index, rt.first_rank)
                if op.index in exact:
                    res["ok"] &= bool(np.array_equal(got, want))
                elif np.abs(want).max() > 0:
                    res["ok"] &= normwise(conv(got), conv(want)) <= tol
    except Exception as e:  # report, do not hang the other ranks
        res["ok"] = False
        res["exc"] = repr(e)
    finally:
        gp.close()
        mesh.close()
    ok = D.max_over_ranks(0.0 if res["ok"] else 1.0) == 0.0
    res["ok"] = ok
    return res


def check_reshard(rt):
    """rh_reshard in dist mode (peer memory, fused barriers) for every ordered spec pair —
    including the fine-grained layouts that push into the peers' buffers or run in two phases —
    against the oracle's reshard, bit-exact on this rank's destination."""
    import torch
    from paper_2302_08141_b200.abi import RH_F32, AxisSpec
    d = rt.world
    dims = [64, 1024]
    specs = ["replicated", "partial", "shard(0,1)", "shard(0,max)", "shard(1,1)", "shard(1,2)", "shard(1,8)",
             "shard(1,64)", "shard(1,max)"]

    def spec(x):
        if "max" in x:
            dim = int(x[6])
            return AxisSpec.shard(dim, dims[dim] // d)
        return AxisSpec.from_string(x)
    mesh = rx.Mesh(rt, [d])
    res = {"name": f"reshard_d{d}", "flags": 0, "ok": True, "err": 0.0, "bad": []}
    try:
        for a in specs:
            for b in specs:
                fs, ts = spec(a), spec(b)
                if a == b or fs == ts or b == "partial":
                    continue
                n = dims[0] * dims[1]
                n_src, n_dst = (n // d if fs.kind == 0 else n), (n // d if ts.kind == 0 else n)
                srcs = [np.random.default_rng(100 + r).standard_normal(n_src).astype(np.float32) for r in range(d)]
                if fs.kind == 1:
                    srcs = [srcs[0].copy() for _ in range(d)]
                want = pyoracle.reshard(d, dims, fs, ts, RH_F32, srcs, n_dst)[rt.first_rank]
                ts_ = torch.from_numpy(srcs[rt.first_rank]).cuda()
                td = torch.empty(n_dst, device="cuda")
                mesh.reshard(0, fs, ts, dims, RH_F32, [ts_.data_ptr()], [td.data_ptr()], 0, 2)
                torch.cuda.synchronize()
                if not np.array_equal(td.cpu().numpy(), want):
                    res["ok"] = False
                    res["bad"].append(f"{a}->{b}")
    except Exception as e:
        res["ok"] = False
        res["exc"] = repr(e)
    finally:
        mesh.close()
    res["ok"] = D.max_over_ranks(0.0 if res["ok"] else 1.0) == 0.0
    return res


def check_pipeline(rt, name, dtype):
    """A pipeline step program (2 stages on the pipeline axis, 1F1B, Send/Recv over NVLink,
    LocalAccumulate + in-place ApplyGradients): one eager step, then every output this process's
    stage holds against the oracle's unpartitioned run of the same step program."""
    from paper_2302_08141_b200.abi import RH_FLAG_NO_GRAPH
    prog = LoweredProgram.load(name)
    prog = prog.with_dtype(dtype) if dtype is not None else prog
    mesh = rx.Mesh(rt, prog.mesh)
    res = {"name": name + (" bf16" if dtype == RH_BF16 else ""), "flags": RH_FLAG_NO_GRAPH, "ok": True, "err": 0.0}
    gp = rx.Program(mesh, prog, RH_FLAG_NO_GRAPH)
    try:
        gp.init_synthetic(7)
        gp.run(1)
        coords, r = [], rt.first_rank
        for dim in reversed(prog.mesh):
            coords.insert(0, r % dim)
            r //= dim
        stage = coords[prog.pipeline_axis]
        conv = pyoracle.bf16_to_f32 if dtype == RH_BF16 else (lambda a: a)
        mine = [o for o in prog.outputs if prog.ops[o].stage == stage]
        got = {o: conv(gp.read_full(o)) for o in mine}
        key = (name, dtype)
        if key not in _ORACLES:
            o = pyoracle.OracleProgram(prog)
            o.init_synthetic(7)
            o.run_unpartitioned(max(1, (os.cpu_count() or 2) // max(1, rt.world)))
            _ORACLES[key] = o
        tol = 2e-2 if dtype == RH_BF16 else 1e-5
        for o in mine:
            e = normwise(got[o], conv(_ORACLES[key].read_full(o, partitioned=False)))
            res["err"] = max(res["err"], e)
            res["ok"] &= e <= tol
        res["outputs_checked"] = len(mine)
    except Exception as e:
        res["ok"] = False
        res["exc"] = repr(e)
    finally:
        gp.close()
        mesh.close()
    res["ok"] = D.max_over_ranks(0.0 if res["ok"] else 1.0) == 0.0
    return res


def main():
    names = sys.argv[1].split(",")
    rt = D.make_runtime()
    out = [check_reshard(rt)]
    for name in [n for n in names if n.startswith("pp_")]:
        out.append(check_pipeline(rt, name, None))
        out.append(check_pipeline(rt, name, RH_BF16))
    names = [n for n in names if not n.startswith("pp_")]
    for name in names:
        full = not name.startswith("c3_")  # full-size block: outputs only (oracle cost)
        for flags in ((0, RH_FLAG_NO_FUSION | RH_FLAG_SIMT_GEMM, RH_FLAG_TRANSPORT_NCCL) if full
                      else (0, RH_FLAG_TRANSPORT_NCCL)):
            out.append(check(rt, name, flags))
        if name.startswith(("c3_", "c1_", "c5_")):
            out.append(check(rt, name, 0, RH_BF16))
        if name.startswith("c5_"):  # rematerialized tanh values over real peers (bounded waits)
            os.environ["RH_REMAT"] = "1"
            try:
                r = check(rt, name, 0, RH_BF16)
                r["name"] += " [RH_REMAT=1]"
                out.append(r)
            finally:
                del os.environ["RH_REMAT"]
    rt.close()
    if rt.first_rank == 0:
        print("DIST_RESULT " + json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
