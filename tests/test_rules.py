"""The executor's local-op rule table against the reference planner, on every lowered fixture
(CPU only: rh_op_natural_specs is host code in librhino_exec.so).

The executor computes each op's output in the spec its local rule yields from the demanded input
specs (the local side of FollowInput / ProduceOutput, proj/src/sharding.cpp:225-388); a planned
spec that differs is executed by the pin fallback (compute, then slice, :477-487).  The oracle
shares that rule table, so a wrong rule would surface only as a silent pin.  Here the reference
planner is the judge: for every op of every fixture the rule must reproduce the planner's own
output spec (ExecutionPlan.sharding, written into the fixture by the unchanged planner), except
for ops the program explicitly pins (JSON "pin", proj/src/parser.cpp:280-284)."""
import glob
import json
import os

import pytest

from paper_2302_08141_b200 import runtime as rx
from paper_2302_08141_b200.program import PLANS_DIR, LoweredProgram

HERE = os.path.dirname(os.path.abspath(__file__))
# the 24-layer plans have 11k ops each: the 1-layer plan of the same generator covers their rules
FIXTURES = sorted(os.path.basename(p)[:-5] for p in glob.glob(os.path.join(PLANS_DIR, "*.json"))
                  if "gpt24" not in p)


def pinned_ids(prog):
    """Ops pinned by the program source (an op's "pin": {axis: spec} in c2_mlp_pinned.json)."""
    if "pinned" not in prog.name:
        return set()
    src = json.load(open(os.path.join(HERE, "golden", "programs", "c2_mlp_pinned.json")))
    return {o["id"] for o in src["ops"] if o.get("pin")}


@pytest.mark.parametrize("name", FIXTURES)
def test_local_rules_reproduce_planned_specs(name):
    prog = LoweredProgram.load(name)
    pins = pinned_ids(prog)
    mism = []
    for op in prog.ops:
        if not op.inputs:
            continue
        nat = rx.natural_specs(prog, op.index)
        if [str(x) for x in nat] != [str(x) for x in op.out_spec]:
            mism.append((op.id, [str(x) for x in nat], [str(x) for x in op.out_spec]))
    unexpected = [m for m in mism if m[0] not in pins]
    assert not unexpected, unexpected[:5]
    if pins:
        assert mism, "the pinned op should be executed by the pin fallback"


def test_broadcast_replicated_to_leading_shard_is_a_local_rule():
    """ProduceOutput's Broadcast R -> Shard(y < off) (sharding.cpp:360-367): every rank writes its
    own rows of the broadcast — not a replicated broadcast plus a slice."""
    R = ["replicated"]
    doc = {"schema": "rhino-lowered/1", "name": "bcast", "mesh": [4], "dtype": "f32",
           "ops": [{"id": "b", "kind": "param", "inputs": [], "shape": [64], "out_spec": R, "in_specs": [[]]},
                   {"id": "y", "kind": "broadcast", "inputs": [0], "shape": [32, 64],
                    "out_spec": ["shard(0,2)"], "in_specs": [R]}],
           "outputs": [1]}
    prog = LoweredProgram(doc)
    assert [str(x) for x in rx.natural_specs(prog, 1)] == ["shard(0,2)"]
