"""Multi-GPU parity (one process per GPU via torchrun, executor in dist mode): needs >= 2 GPUs;
skipped on a 1-GPU box (the emulated-rank tests in test_gpu_parity.py cover the same programs)."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def n_gpus():
    import torch
    return torch.cuda.device_count()


PLANS = {
    2: ["c1_mlp_d2", "c2_mlp_reshape_d2", "c2_mlp_pinned_d2", "moe_small_d2", "gpt_small_d2",
        "skipnet_small_d2", "c3_gpt_block_d2", "c3_gpt_heads32_d2", "c5_gpt_small_d2"],
    4: ["c1_mlp_d4", "c2_mlp_reshape_d4", "c2_mlp_pinned_d4", "moe_small_d4", "gpt_small_2x2",
        "rand_gpt_like_2x2_s0", "rand_moe_like_4_s2", "c3_gpt_block_d4", "c3_gpt_heads32_d4", "c3_gpt_block_2x2",
        "c5_gpt_small_d4", "pp_gpt_small_2x2_m2", "pp_gpt_small_2x2_m4"],
}


@pytest.mark.parametrize("world", [2, 4])
def test_dist_parity(world):
    if n_gpus() < world:
        pytest.skip(f"needs {world} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + world),
           os.path.join(HERE, "_dist_worker.py"), ",".join(PLANS[world])]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=1800)
    lines = [l for l in r.stdout.splitlines() if l.startswith("DIST_RESULT ")]
    assert r.returncode == 0 and lines, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(lines[0][len("DIST_RESULT "):])
    out_dir = os.path.join(os.path.dirname(HERE), "gpurun_out")
    if os.path.isdir(out_dir):
        with open(os.path.join(out_dir, f"dist_parity_{world}.json"), "w") as f:
            json.dump(res, f, indent=1)
    bad = [x for x in res if not x["ok"]]
    assert not bad, bad
