"""The compiled reference-side binding: oracle/_ref/rh_execute runs the
reference's own parse -> plan() path (libparashard, unchanged sources) and executes the plan
through the C-ABI of librhino_exec.so.  Its output must match the CPU oracle on the committed
lowered fixture of the same program (same planner, same Philox inputs)."""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2302_08141_b200.program import LoweredProgram

pytestmark = pytest.mark.gpu

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(REPO, "oracle", "_ref", "rh_execute")


def normwise(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)


@pytest.mark.parametrize("program,devices,fixture", [("c1_mlp.ir", 4, "c1_mlp_d4"),
                                                     ("c2_mlp_reshape.ir", 8, "c2_mlp_reshape_d8")])
def test_rh_execute_matches_oracle(oracle_lib, tmp_path, program, devices, fixture):
    assert os.path.exists(EXE), "oracle/_ref/rh_execute is built by __graft_entry__.build()"
    out = tmp_path / "y.bin"
    r = subprocess.run([EXE, "--text", os.path.join(REPO, "tests", "golden", "programs", program),
                        "--devices", str(devices), "--seed", "3", "--iters", "2", "--out", str(out)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    info = json.loads(r.stdout.strip().splitlines()[-1])
    assert info["mesh"] == devices and info["ms_per_step"] > 0
    prog = LoweredProgram.load(fixture)
    y = np.fromfile(out, dtype=np.float32).reshape(prog.ops[prog.outputs[0]].shape)
    o = oracle_lib.OracleProgram(prog)
    o.init_synthetic(3)
    o.run_unpartitioned()
    assert normwise(y, o.read_full(prog.outputs[0], partitioned=False)) <= 1e-5
