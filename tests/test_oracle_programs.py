"""Oracle self-consistency on every lowered fixture small enough for the CPU suite: the
partitioned execution (all ranks simulated, block-cyclic local buffers) equals the
unpartitioned single-device execution — bit-exact when the program only moves data, within
the fp32 tolerance otherwise (SURVEY §8c parity contract)."""
import glob
import os

import numpy as np
import pytest

from paper_2302_08141_b200.abi import RH_BF16
from paper_2302_08141_b200.program import PLANS_DIR, LoweredProgram

SMALL = sorted(os.path.basename(p)[:-5] for p in glob.glob(os.path.join(PLANS_DIR, "*.json"))
               if not os.path.basename(p).startswith(("c3_", "c5_big", "pp_")))
TOL_F32, TOL_BF16 = 1e-5, 2e-2


def normwise(a, b):
    a = a.astype(np.float64)
    b = b.astype(np.float64)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)


@pytest.mark.parametrize("name", SMALL)
def test_partitioned_equals_unpartitioned(oracle_lib, name):
    p = LoweredProgram.load(name)
    o = oracle_lib.OracleProgram(p)
    o.init_synthetic(1)
    o.run_unpartitioned()
    o.run_partitioned()
    for out in p.outputs:
        a = o.read_full(out, partitioned=True)
        b = o.read_full(out, partitioned=False)
        assert normwise(a, b) <= TOL_F32, name


@pytest.mark.parametrize("name", ["c1_mlp_d4", "c2_mlp_reshape_d8", "rand_gpt_like_2x2_s1"])
def test_bf16_partitioned(oracle_lib, name):
    p = LoweredProgram.load(name).with_dtype(RH_BF16)
    o = oracle_lib.OracleProgram(p)
    o.init_synthetic(2)
    o.run_unpartitioned()
    o.run_partitioned()
    for out in p.outputs:
        a = oracle_lib.bf16_to_f32(o.read_full(out, True))
        b = oracle_lib.bf16_to_f32(o.read_full(out, False))
        assert normwise(a, b) <= TOL_BF16


def test_sources_bit_exact_across_layouts(oracle_lib):
    """Sharded synthetic init = slice of the replicated init (K17: keyed by global index)."""
    p = LoweredProgram.load("c1_mlp_d4")
    o = oracle_lib.OracleProgram(p, keep_all=True)
    o.init_synthetic(0)
    o.run_partitioned()
    o.run_unpartitioned()
    w1 = p.op_index("w1")
    full = o.read_full(w1, partitioned=False)
    for r in range(4):
        np.testing.assert_array_equal(o.read_local(w1, r), full[:, r * 256:(r + 1) * 256].ravel())
