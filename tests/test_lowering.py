"""Lowered-program fixtures (tests/golden/plans, written by the reference planner through
oracle/_ref/rh_plan) are self-consistent: strategy recovery reproduced the plan, every spec is
valid on the composed shapes, and the rh_op conversion round-trips."""
import glob
import os

import pytest

from paper_2302_08141_b200.abi import AxisSpec, composed_local_shape, spec_valid
from paper_2302_08141_b200.program import PLANS_DIR, LoweredProgram

PLANS = sorted({os.path.basename(p).split(".json")[0]
                for p in glob.glob(os.path.join(PLANS_DIR, "*.json")) + glob.glob(os.path.join(PLANS_DIR, "*.json.gz"))})


def test_fixtures_present():
    for need in ["c1_mlp_d4", "c2_mlp_reshape_d4", "c2_mlp_pinned_d8", "c3_gpt_block_d8",
                 "c3_gpt_block_2x4", "c3_gpt_heads32_d1", "c3_gpt_heads32_d2", "c3_gpt_heads32_d4",
                 "c3_gpt_heads32_d8", "c5_big_gpt24_d4"]:
        assert need in PLANS


@pytest.mark.parametrize("name", PLANS)
def test_plan_fixture_consistent(name):
    p = LoweredProgram.load(name)
    assert p.doc["schema"] == ("rhino-lowered/2" if name.startswith("pp_") else "rhino-lowered/1")
    for rec in p.doc["recovery"]:
        assert rec["replay_matched"], rec
    if "plan_sharding" in p.doc:  # recovered strategies emit exactly the planner's specs
        for a, axis in enumerate(p.doc["plan_sharding"]):
            for i, s in enumerate(axis):
                assert AxisSpec.from_string(s) == p.ops[i].out_spec[a]
    for op in p.ops:
        specs = op.out_spec
        for a, d in enumerate(p.mesh):
            shape = composed_local_shape(op.shape, specs[:a], p.mesh[:a])
            assert spec_valid(specs[a], shape, d), (op.id, a, str(specs[a]))
        for a in range(len(p.mesh)):
            assert len(op.in_specs[a]) == len(op.inputs)
    arr, outs = p.to_c()
    assert len(arr) == len(p.ops)
    for i, op in enumerate(p.ops):
        assert arr[i].rank == len(op.shape) and arr[i].n_in == len(op.inputs)


def test_axis_spec_strings():
    for s in ["shard(0,8)", "shard(1,1)", "replicated", "partial"]:
        assert str(AxisSpec.from_string(s)) == s
    assert AxisSpec.from_string("R") == AxisSpec.replicated()
    assert AxisSpec.from_string("P") == AxisSpec.partial()
    with pytest.raises(ValueError):
        AxisSpec.from_string("shard(x)")


PIPELINE = [p for p in PLANS if p.startswith("pp_")]


@pytest.mark.parametrize("name", PIPELINE)
def test_pipeline_plan_fixture(name):
    """Wire format v2: stages, microbatches, cut placeholder specs and the
    ApplyGradients pairs; every op Replicated on the pipeline axis (it places stages)."""
    p = LoweredProgram.load(name)
    assert p.doc["schema"] == "rhino-lowered/2" and p.pipeline_axis >= 0
    S = p.mesh[p.pipeline_axis]
    assert all(0 <= op.stage < S for op in p.ops)
    assert all(str(op.out_spec[p.pipeline_axis]) == "replicated" for op in p.ops)
    assert {op.microbatch for op in p.ops} == set(range(1, p.microbatches + 1))
    assert p.doc["cuts"] and all(c["id"].startswith("__cut_") for c in p.doc["cuts"])
    for g, w in p.apply:
        assert p.ops[w].kind == 0 and p.ops[g].shape == p.ops[w].shape
        assert p.ops[g].stage == p.ops[w].stage
    # each stage's ops read only values of their own stage or of cut producers (Send/Recv)
    cut_producers = {c["producer"] for c in p.doc["cuts"]}
    assert cut_producers
