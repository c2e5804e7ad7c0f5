"""K1: the tcgen05/TMEM/TMA GEMM (bf16 in, fp32 accumulate) and the CUDA-core GEMM against an
fp64 reference on the same bf16 inputs, through the C-ABI (single-op programs), including the
fused unary-chain epilogue and all four operand layouts (transpose_a x transpose_b)."""
import numpy as np
import pytest

from paper_2302_08141_b200.abi import RH_BF16, RH_F32, RH_FLAG_SIMT_GEMM
from paper_2302_08141_b200.program import LoweredProgram

pytestmark = pytest.mark.gpu


def matmul_doc(m, k, n, tb=False, chain=(), dtype="bf16", ta=False):
    R = ["replicated"]
    ops = [
        {"id": "a", "kind": "input", "inputs": [], "shape": [k, m] if ta else [m, k], "out_spec": R,
         "in_specs": [[]]},
        {"id": "b", "kind": "param", "inputs": [], "shape": [n, k] if tb else [k, n], "out_spec": R,
         "in_specs": [[]]},
        {"id": "c", "kind": "matmul", "inputs": [0, 1], "shape": [m, n], "transpose_a": ta,
         "transpose_b": tb, "out_spec": R, "in_specs": [R * 2]},
    ]
    for i, fn in enumerate(chain):
        ops.append({"id": f"u{i}", "kind": "unary", "fn": fn, "inputs": [len(ops) - 1], "shape": [m, n],
                    "out_spec": R, "in_specs": [R]})
    return {"schema": "rhino-lowered/1", "name": "gemm", "mesh": [1], "dtype": dtype, "ops": ops,
            "outputs": [len(ops) - 1]}


def bf16_to_f64(a):
    return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


def run(doc, flags=0):
    from paper_2302_08141_b200 import runtime as rx
    prog = LoweredProgram(doc)
    rt = rx.Runtime(devices=[0])
    mesh = rx.Mesh(rt, [1])
    gp = rx.Program(mesh, prog, flags)
    try:
        gp.init_synthetic(9)
        gp.run(1)
        a = gp.read_full(0)
        b = gp.read_full(1)
        c = gp.read_full(prog.outputs[0])
        names = [s["name"] for s in gp.steps()]
    finally:
        gp.close()
        mesh.close()
        rt.close()
    return a, b, c, names


# (512, 1024, 1024) and (2048, 16384, 512): split-K; 128 / 256 / 384-tile shapes: one and a half
# to three waves on 148 SMs
@pytest.mark.parametrize("m,k,n", [(128, 64, 128), (128, 128, 256), (256, 512, 384), (512, 1024, 1024),
                                   (2048, 4096, 4096), (2048, 16384, 512), (2048, 2048, 2048),
                                   (4096, 3072, 1024)])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("ta", [False, True])
def test_tc_gemm_vs_fp64(m, k, n, tb, ta):
    a, b, c, names = run(matmul_doc(m, k, n, tb, ta=ta))
    assert any(s.startswith("gemm_tc") for s in names), names
    A, B = bf16_to_f64(a), bf16_to_f64(b)
    ref = (A.T if ta else A) @ (B.T if tb else B)
    got = bf16_to_f64(c)
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err <= 1e-2, err  # bf16 output rounding (2^-9) + fp32 accumulation


@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("ta", [False, True])
def test_tc_matches_simt(tb, ta):
    _, _, c_tc, n1 = run(matmul_doc(256, 1024, 512, tb, ta=ta))
    _, _, c_simt, n2 = run(matmul_doc(256, 1024, 512, tb, ta=ta), RH_FLAG_SIMT_GEMM)
    assert any("gemm_tc" in s for s in n1) and any("gemm_simt" in s for s in n2)
    x, y = bf16_to_f64(c_tc), bf16_to_f64(c_simt)
    # same inputs, both fp32-accumulated (different orders), both rounded to bf16: the results
    # differ by at most one bf16 rounding step relative to the output scale
    assert np.abs(x - y).max() <= 2.0 ** -8 * np.abs(y).max()
    assert (x == y).mean() > 0.9


def test_tc_fused_epilogue_chain():
    _, _, c, names = run(matmul_doc(256, 256, 256, False, ("relu", "neg")))
    assert len(names) == 1 and "gemm_tc" in names[0]  # short exact chains ride in the epilogue
    _, _, c2, names2 = run(matmul_doc(256, 256, 256, False, ("relu", "neg")), RH_FLAG_SIMT_GEMM)
    x, y = bf16_to_f64(c), bf16_to_f64(c2)
    assert np.abs(x - y).max() <= 2.0 ** -6
    # chains of more than two ops after run compression get their own kernel
    _, _, _, names3 = run(matmul_doc(256, 256, 256, False, ("relu", "tanh", "neg", "relu")))
    assert len(names3) == 2 and "unary_chain" in names3[1]


@pytest.mark.parametrize("m,k,n", [(256, 256, 256), (2048, 4096, 4096), (256, 16384, 512), (64, 128, 64)])
def test_tc_epilogue_tanh_runs_bit_exact(m, k, n):
    """A tanh run (one T^k table lookup staged in shared memory) and an exact op in the GEMM
    epilogue — single-CTA, CTA-pair, split-K reduce and CUDA-core GEMMs — are bit-identical to
    the unfused one-op-per-kernel schedule."""
    from paper_2302_08141_b200.abi import RH_FLAG_NO_FUSION
    chain = ("tanh", "", "tanh", "relu")
    _, _, c, names = run(matmul_doc(m, k, n, False, chain))
    _, _, c0, names0 = run(matmul_doc(m, k, n, False, chain), RH_FLAG_NO_FUSION)
    assert len(names) == 1, names
    assert len(names0) == 1 + len(chain), names0
    np.testing.assert_array_equal(c, c0)


@pytest.mark.parametrize("m,k,n", [(128, 32, 128), (256, 512, 384), (1024, 4096, 1024),
                                   (2048, 16384, 512)])
@pytest.mark.parametrize("tb", [False, True])
@pytest.mark.parametrize("ta", [False, True])
def test_tc_3xtf32_vs_fp64(m, k, n, tb, ta):
    """fp32 programs: 3xTF32 on tcgen05 (kind::tf32), fp32-level accuracy (parity 1e-5)."""
    a, b, c, names = run(matmul_doc(m, k, n, tb, dtype="f32", ta=ta))
    assert any(s.startswith("gemm_tc_3xtf32") for s in names), names
    A = a.astype(np.float64)
    ref = (A.T if ta else A) @ (b.astype(np.float64).T if tb else b.astype(np.float64))
    err = np.abs(c - ref).max() / np.abs(ref).max()
    assert err <= 1e-5, err


def test_simt_fp32_gemm_vs_fp64():
    a, b, c, names = run(matmul_doc(300, 200, 100, True, dtype="f32"))
    assert any("gemm_simt" in s for s in names)
    ref = a.astype(np.float64) @ b.astype(np.float64).T
    assert np.abs(c - ref).max() / np.abs(ref).max() <= 1e-5


def group_doc(P, m, k, n, shared_a, ta=False, tb=False, chain=()):
    """P independent MatMuls of one shape (the per-head GEMMs of an attention block): with
    shared_a every problem reads the same A (q/k/v projections), else each its own (score, ctx)."""
    R = ["replicated"]
    ops = []
    ash = [k, m] if ta else [m, k]
    bsh = [n, k] if tb else [k, n]
    if shared_a:
        ops.append({"id": "a", "kind": "input", "inputs": [], "shape": ash, "out_spec": R, "in_specs": [[]]})
    outs = []
    for p in range(P):
        if not shared_a:
            ops.append({"id": f"a{p}", "kind": "input", "inputs": [], "shape": ash, "out_spec": R, "in_specs": [[]]})
        ai = 0 if shared_a else len(ops) - 1
        ops.append({"id": f"b{p}", "kind": "param", "inputs": [], "shape": bsh, "out_spec": R, "in_specs": [[]]})
        ops.append({"id": f"c{p}", "kind": "matmul", "inputs": [ai, len(ops) - 1], "shape": [m, n],
                    "transpose_a": ta, "transpose_b": tb, "out_spec": R, "in_specs": [R * 2]})
        for i, fn in enumerate(chain):
            ops.append({"id": f"u{p}_{i}", "kind": "unary", "fn": fn, "inputs": [len(ops) - 1], "shape": [m, n],
                        "out_spec": R, "in_specs": [R]})
        outs.append(len(ops) - 1)
    return {"schema": "rhino-lowered/1", "name": "group", "mesh": [1], "dtype": "bf16", "ops": ops,
            "outputs": outs}


def run_group(doc, env_off=False, monkeypatch=None):
    from paper_2302_08141_b200 import runtime as rx
    if monkeypatch is not None:
        if env_off:
            monkeypatch.setenv("RH_NO_GEMM_GROUP", "1")
        else:
            monkeypatch.delenv("RH_NO_GEMM_GROUP", raising=False)
    prog = LoweredProgram(doc)
    rt = rx.Runtime(devices=[0])
    mesh = rx.Mesh(rt, [1])
    gp = rx.Program(mesh, prog)
    try:
        gp.init_synthetic(21)
        gp.run(2)
        vals = {op.index: gp.read_full(op.index) for op in prog.ops if op.kind in (0, 1)}
        outs = [gp.read_full(o) for o in prog.outputs]
        names = [s["name"] for s in gp.steps()]
    finally:
        gp.close()
        mesh.close()
        rt.close()
    return prog, vals, outs, names


# q/k/v-like (shared A, N = head_dim 128: tiles span two problems), score-like (own A, tb),
# ctx-like (own A, N = 128), and MN-major / transposed-A variants
@pytest.mark.parametrize("P,m,k,n,shared_a,ta,tb", [
    (24, 2048, 512, 128, True, False, False),   # CTA-pair 256-wide tiles: one problem per CTA
    (24, 2048, 256, 128, True, False, True),
    (64, 384, 256, 128, True, False, False),    # single-CTA 256-wide tiles spanning two problems
    (12, 512, 1024, 128, True, False, False),
    (6, 256, 512, 256, True, False, True),
    (4, 512, 128, 512, False, False, True),
    (5, 256, 512, 128, False, False, False),
    (3, 256, 256, 256, False, True, False),
    (8, 2048, 256, 128, True, True, True),
])
def test_tc_grouped_gemm(monkeypatch, P, m, k, n, shared_a, ta, tb):
    """One grouped tcgen05 launch for P independent MatMuls (per-problem TMA maps and output
    pointers from a device table) against fp64, and against the one-launch-per-GEMM schedule."""
    doc = group_doc(P, m, k, n, shared_a, ta, tb)
    prog, vals, outs, names = run_group(doc, monkeypatch=monkeypatch)
    assert any(s.startswith("gemm_tc_group[%d]" % P) for s in names), names
    _, _, outs0, names0 = run_group(doc, env_off=True, monkeypatch=monkeypatch)
    assert not any("group" in s for s in names0)
    for p, o in enumerate(prog.outputs):
        mm = prog.ops[o]
        A, B = bf16_to_f64(vals[mm.inputs[0]]), bf16_to_f64(vals[mm.inputs[1]])
        ref = (A.T if ta else A) @ (B.T if tb else B)
        got = bf16_to_f64(outs[p])
        assert np.abs(got - ref).max() / np.abs(ref).max() <= 1e-2, p
        y = bf16_to_f64(outs0[p])
        assert np.abs(got - y).max() <= 2.0 ** -8 * np.abs(y).max(), p


def test_tc_grouped_gemm_epilogue_bit_exact(monkeypatch):
    """Grouped launches keep the fused tanh-run epilogue: bit-identical to NO_FUSION."""
    from paper_2302_08141_b200.abi import RH_FLAG_NO_FUSION
    from paper_2302_08141_b200 import runtime as rx
    doc = group_doc(6, 256, 512, 256, False, False, True, chain=("", "", "tanh"))
    prog, _, outs, names = run_group(doc, monkeypatch=monkeypatch)
    assert names[0].startswith("gemm_tc_group[6]") and len(names) == 1, names
    rt = rx.Runtime(devices=[0])
    mesh = rx.Mesh(rt, [1])
    gp = rx.Program(mesh, LoweredProgram(doc), RH_FLAG_NO_FUSION)
    try:
        gp.init_synthetic(21)
        gp.run(1)
        ref = [gp.read_full(o) for o in prog.outputs]
    finally:
        gp.close()
        mesh.close()
        rt.close()
    for a, b in zip(outs, ref):
        np.testing.assert_array_equal(a, b)
