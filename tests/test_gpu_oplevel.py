"""Op-level parity ("teacher forcing") on the full-size GPT block: every op the executor ran is
re-executed by the CPU oracle on the executor's OWN input values, and the two outputs compared.

Why: the fixture block chains 90 tanh ops around 8 GEMMs with K up to 16384, so end-to-end
comparisons of two correct fp32/bf16 executions drift apart (GEMM accumulation order; see
test_gpu_parity.test_gpt_block_fp32).  Per op the comparison is tight and non-chaotic:
  * data movement (transpose / reshape / broadcast / concat): bit-exact;
  * elementwise ops: bit-exact for bf16 (per-op rounding matches), <= 2 fp32 ulp-ish for fp32
    (CUDA vs glibc tanhf/expf);
  * matmul / reduce_sum (accumulation order differs): normwise <= 1e-5 (fp32), <= 2^-7 (bf16).
Partitioned plans run with RH_FLAG_NO_FUSION so every op is materialized; each op's global value
is assembled from the ranks' local buffers (Partial outputs summed), i.e. this also checks the
placement of every intermediate.
"""
import numpy as np
import pytest

from paper_2302_08141_b200.abi import OP_KINDS, RH_BF16, RH_F32, RH_FLAG_KEEP_ALL, RH_FLAG_NO_FUSION
from paper_2302_08141_b200.program import LoweredProgram

pytestmark = pytest.mark.gpu

MOVE = {"reshape", "transpose", "broadcast", "concat"}


def one_op_doc(prog, i, dtype):
    R = ["replicated"]
    op = prog.ops[i]
    ops = [{"id": f"in{k}", "kind": "input", "inputs": [], "shape": prog.ops[p].shape, "out_spec": R,
            "in_specs": [[]]} for k, p in enumerate(op.inputs)]
    o = {"id": op.id, "kind": OP_KINDS[op.kind], "inputs": list(range(len(op.inputs))), "shape": op.shape,
         "out_spec": R, "in_specs": [R * len(op.inputs)], "fn": op.fn, "transpose_a": op.transpose_a,
         "transpose_b": op.transpose_b, "axis": op.axis}
    if op.perm:
        o["perm"] = op.perm
    ops.append(o)
    return LoweredProgram({"schema": "rhino-lowered/1", "name": f"op_{op.id}", "mesh": [1],
                           "dtype": "bf16" if dtype == RH_BF16 else "f32", "ops": ops,
                           "outputs": [len(ops) - 1]})


def as_f64(a):
    if a.dtype == np.uint16:
        return (a.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    return a.astype(np.float64)


@pytest.mark.parametrize("name,dtype", [(n, d) for n in ("c3_gpt_block_d1", "c3_gpt_block_d8", "c3_gpt_block_2x4",
                                                        "c5_gpt_small_d2", "c5_gpt_small_d4")
                                         for d in (RH_BF16, RH_F32)] + [("c3_gpt_heads32_d4", RH_BF16),
                                                                        ("pp_gpt_small_2x2_m2", RH_BF16),
                                                                        ("pp_gpt6_2x2_m4", RH_BF16)])
def test_gpt_block_op_level(oracle_lib, name, dtype):
    from paper_2302_08141_b200 import runtime as rx
    prog = LoweredProgram.load(name).with_dtype(dtype)
    if prog.pipeline_axis >= 0:
        prog.apply = []  # no in-place ApplyGradients: every run reads the same parameters
    rt = rx.Runtime(devices=[0] * prog.world)
    mesh = rx.Mesh(rt, prog.mesh)
    gp = rx.Program(mesh, prog, RH_FLAG_NO_FUSION | RH_FLAG_KEEP_ALL)
    try:
        gp.init_synthetic(17)
        gp.run(1)
        vals = {op.index: gp.read_full(op.index) for op in prog.ops}
        # what each op actually consumed (after its input transitions: e.g. a multi-axis
        # Partial -> Shard sums per axis, which rounds differently from a one-shot sum)
        ins = {op.index: [gp.read_input_full(op.index, k) for k in range(len(op.inputs))]
               for op in prog.ops if op.kind not in (0, 1)}
    finally:
        gp.close()
        mesh.close()
        rt.close()
    worst = {}
    for op in prog.ops:
        if op.kind in (0, 1):
            continue
        small = one_op_doc(prog, op.index, dtype)
        o = oracle_lib.OracleProgram(small)
        for k in range(len(op.inputs)):
            o.set_full(k, ins[op.index][k])
        o.run_unpartitioned()
        want = o.read_full(len(op.inputs), partitioned=False)
        got = vals[op.index]
        kind = OP_KINDS[op.kind]
        if kind in MOVE:
            np.testing.assert_array_equal(got, want, err_msg=op.id)
            continue
        g, w = as_f64(got), as_f64(want)
        err = np.abs(g - w).max() / max(np.abs(w).max(), 1e-30)
        worst[kind] = max(worst.get(kind, 0.0), err)
        partial_out = any(sp.kind == 2 for sp in op.out_spec)  # local P + P adds (LocalAccumulate)
        if kind in ("matmul", "reduce_sum") or partial_out:
            assert err <= (2.0 ** -7 if dtype == RH_BF16 else 1e-5), (op.id, err)
        elif dtype == RH_BF16:
            mism = np.count_nonzero(got != want)
            assert mism <= max(2, got.size // 10000), (op.id, mism)  # rare 2^-20 boundary cases
            assert err <= 2.0 ** -7, (op.id, err)
        else:
            assert np.all(np.abs(g - w) <= 4 * np.spacing(np.abs(w).astype(np.float32)) + 1e-30), op.id
    print(name, dtype, {k: f"{v:.2e}" for k, v in worst.items()})
