"""Resharding transitions (K9-K14, sharding.cpp:104-142) through rh_reshard vs the oracle's
ox_reshard: bit-exact, including Partial sums (both sum in rank order 0..d-1 in fp32) and the
strided (block-cyclic) layouts, for fp32 and bf16, on emulated meshes of 2/4/8 ranks."""
import itertools

import numpy as np
import pytest

from paper_2302_08141_b200.abi import RH_BF16, RH_F32, AxisSpec

pytestmark = pytest.mark.gpu

SPECS = ["replicated", "partial", "shard(0,1)", "shard(0,8)", "shard(0,max)", "shard(1,1)", "shard(1,2)",
         "shard(1,8)", "shard(1,64)", "shard(1,max)"]


def spec_of(s, dims, d):
    if "max" in s:
        dim = int(s[6])
        return AxisSpec.shard(dim, dims[dim] // d)
    return AxisSpec.from_string(s)


def local_elems(spec, dims, d):
    n = int(np.prod(dims))
    return n // d if spec.is_shard else n


@pytest.mark.parametrize("d", [2, 4, 8])
@pytest.mark.parametrize("dtype", [RH_F32, RH_BF16])
@pytest.mark.parametrize("dims", [[64, 512], [256, 2048]])
def test_all_transitions_bit_exact(oracle_lib, d, dtype, dims):
    """Every ordered spec pair, including the fine-grained layouts (runs of 1-8 elements) that take
    the push / pull-interleave / two-phase kernels (executor.cpp ClassifyFine)."""
    import torch
    from paper_2302_08141_b200 import runtime as rx
    rt = rx.Runtime(devices=[0] * d)
    mesh = rx.Mesh(rt, [d])
    rng = np.random.default_rng(d)
    npd = np.uint16 if dtype == RH_BF16 else np.float32
    try:
        for a, b in itertools.product(SPECS, SPECS):
            if a == b or (a == "partial" and b == "partial"):
                continue
            fs, ts = spec_of(a, dims, d), spec_of(b, dims, d)
            if fs == ts:  # e.g. shard(0,8) == shard(0,max) on 64 rows at d=8
                continue
            n_src, n_dst = local_elems(fs, dims, d), local_elems(ts, dims, d)
            srcs = []
            for r in range(d):
                v = rng.standard_normal(n_src).astype(np.float32)
                srcs.append(oracle_lib.f32_to_bf16(v) if dtype == RH_BF16 else v)
            if fs.kind == 1:  # replicated: identical copies
                srcs = [srcs[0].copy() for _ in range(d)]
            want = oracle_lib.reshard(d, dims, fs, ts, dtype, srcs, n_dst)
            tsrc = [torch.from_numpy(s.view(np.int16) if dtype == RH_BF16 else s).cuda() for s in srcs]
            tdst = [torch.empty(n_dst, dtype=tsrc[0].dtype, device="cuda") for _ in range(d)]
            mesh.reshard(0, fs, ts, dims, dtype, [t.data_ptr() for t in tsrc],
                         [t.data_ptr() for t in tdst])
            torch.cuda.synchronize()
            for r in range(d):
                got = tdst[r].cpu().numpy().view(npd)
                np.testing.assert_array_equal(got, want[r], err_msg=f"{a}->{b} d={d} rank {r}")
    finally:
        mesh.close()
        rt.close()


def test_two_axis_mesh_transitions(oracle_lib):
    """Axis-1 transitions on a 2x2 mesh act inside axis-1 groups on the axis-0-local tensor."""
    import torch
    from paper_2302_08141_b200 import runtime as rx
    rt = rx.Runtime(devices=[0] * 4)
    mesh = rx.Mesh(rt, [2, 2])
    dims = [32, 64]
    try:
        for axis in (0, 1):
            fs, ts = AxisSpec.shard(0, 4), AxisSpec.shard(1, 2)
            srcs = [np.random.default_rng(r).standard_normal(int(np.prod(dims)) // 2).astype(np.float32)
                    for r in range(4)]
            tsrc = [torch.from_numpy(s).cuda() for s in srcs]
            tdst = [torch.empty(int(np.prod(dims)) // 2, device="cuda") for _ in range(4)]
            mesh.reshard(axis, fs, ts, dims, RH_F32, [t.data_ptr() for t in tsrc],
                         [t.data_ptr() for t in tdst])
            torch.cuda.synchronize()
            for r in range(4):
                coords = (r // 2, r % 2)
                group = [r2 for r2 in range(4) if (r2 // 2, r2 % 2)[1 - axis] == coords[1 - axis]]
                want = oracle_lib.reshard(2, dims, fs, ts, RH_F32, [srcs[g] for g in group],
                                          int(np.prod(dims)) // 2)
                np.testing.assert_array_equal(tdst[r].cpu().numpy(), want[coords[axis]])
    finally:
        mesh.close()
        rt.close()
