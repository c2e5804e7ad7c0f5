"""Lowered programs ("rhino-lowered/1" JSON written by the reference-side tool rh_plan) and their
conversion to rh_op records for the C-ABI.

A lowered program is the reference TensorProgram (proj/include/parashard/ir.h:97-158) plus, per
op and mesh axis, the OpStrategy the planner chose (proj/include/parashard/sharding.h:99-111).
"""
import ctypes
import gzip
import json
import math
import os

from .abi import (OP_KINDS, RH_BF16, RH_F32, RH_MAX_AXES, RH_MAX_RANK, UNARY_FNS, AxisSpec, RhOp,
                  RhSpec, composed_local_shape)

# Lowered-program library searched by LoweredProgram.load(name): RH_PLANS_DIR, else the fixtures
# the reference-side tool wrote for the BASELINE configs (tests/golden/plans).  A caller with its
# own plan passes a path instead of a name.
PLANS_DIR = os.environ.get("RH_PLANS_DIR") or os.path.join(
    os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden", "plans")


class LoweredOp:
    __slots__ = ("index", "id", "kind", "inputs", "shape", "fn", "transpose_a", "transpose_b",
                 "axis", "perm", "out_spec", "in_specs", "flops", "stage", "microbatch", "phase")

    def local_shape(self, mesh):
        return composed_local_shape(self.shape, self.out_spec, mesh)


class LoweredProgram:
    def __init__(self, doc):
        if doc.get("schema") not in ("rhino-lowered/1", "rhino-lowered/2"):
            raise ValueError("not a rhino-lowered/1|2 document")
        self.doc = doc
        self.name = doc.get("name", "")
        self.mesh = list(doc["mesh"])
        self.dtype = RH_BF16 if doc.get("dtype") == "bf16" else RH_F32
        self.outputs = list(doc["outputs"])
        self.ops = []
        for i, o in enumerate(doc["ops"]):
            op = LoweredOp()
            op.index = i
            op.id = o["id"]
            op.kind = OP_KINDS.index(o["kind"])
            op.inputs = list(o["inputs"])
            op.shape = list(o["shape"])
            op.fn = o.get("fn", "")
            op.transpose_a = bool(o.get("transpose_a", False))
            op.transpose_b = bool(o.get("transpose_b", False))
            op.axis = int(o.get("axis", 0))
            op.perm = list(o.get("perm", []))
            op.out_spec = [AxisSpec.from_string(s) for s in o["out_spec"]]
            op.in_specs = [[AxisSpec.from_string(s) for s in axis] for axis in o["in_specs"]]
            op.flops = float(o.get("flops", 0.0))
            op.stage = int(o.get("stage", 0))
            op.microbatch = int(o.get("microbatch", 1))
            op.phase = {"fwd": 0, "bwd": 1, "acc": 2}.get(o.get("phase", "fwd"), 0)
            self.ops.append(op)
        # wire format v2 (pipeline plans): pipeline axis, microbatches, cut placeholder specs,
        # and the ApplyGradients pairs {gradient op, parameter op} with the learning rate
        self.pipeline_axis = int(doc.get("pipeline_axis", -1))
        self.microbatches = int(doc.get("microbatches", 1))
        self.apply = [tuple(x) for x in doc.get("apply", [])]
        self.lr = float(doc.get("lr", 0.0))
        self._keep = None

    @staticmethod
    def load(path_or_name):
        """A plan file (.json or .json.gz) or the name of one in PLANS_DIR."""
        path = path_or_name
        if not os.path.exists(path):
            path = os.path.join(PLANS_DIR, path_or_name + ".json")
            if not os.path.exists(path) and os.path.exists(path + ".gz"):
                path += ".gz"
        opener = gzip.open if path.endswith(".gz") else open
        with opener(path, "rt") as f:
            return LoweredProgram(json.load(f))

    @property
    def world(self):
        return math.prod(self.mesh)

    def op_index(self, op_id):
        for op in self.ops:
            if op.id == op_id:
                return op.index
        raise KeyError(op_id)

    def with_dtype(self, dtype):
        """Same program re-typed (the IR carries elem_bytes only, ir.h:37-56)."""
        p = LoweredProgram(self.doc)
        p.dtype = dtype
        return p

    def elem_bytes(self):
        return 2 if self.dtype == RH_BF16 else 4

    def full_bytes(self, op):
        return math.prod(self.ops[op].shape) * self.elem_bytes()

    def local_bytes(self, op):
        return math.prod(self.ops[op].local_shape(self.mesh)) * self.elem_bytes()

    def flops(self):
        return sum(op.flops for op in self.ops)

    def to_c(self):
        """rh_op array (+ the arrays it points into, kept alive on self)."""
        n = len(self.ops)
        naxes = len(self.mesh)
        if naxes > RH_MAX_AXES:
            raise ValueError("mesh has too many axes")
        arr = (RhOp * n)()
        keep = []
        for i, op in enumerate(self.ops):
            r = arr[i]
            r.kind = op.kind
            r.fn = UNARY_FNS[op.fn]
            r.dtype = self.dtype
            if len(op.shape) > RH_MAX_RANK:
                raise ValueError("rank too large")
            r.rank = len(op.shape)
            for k, d in enumerate(op.shape):
                r.dims[k] = d
            r.n_in = len(op.inputs)
            ins = (ctypes.c_int32 * max(1, len(op.inputs)))(*op.inputs)
            keep.append(ins)
            r.inputs = ins
            r.transpose_a = int(op.transpose_a)
            r.transpose_b = int(op.transpose_b)
            r.axis = op.axis
            r.has_perm = 1 if op.perm else 0
            for k, p in enumerate(op.perm):
                r.perm[k] = p
            for a in range(naxes):
                r.out_spec[a] = op.out_spec[a].to_c()
            specs = (RhSpec * max(1, naxes * len(op.inputs)))()
            for a in range(naxes):
                for s in range(len(op.inputs)):
                    specs[a * len(op.inputs) + s] = op.in_specs[a][s].to_c()
            keep.append(specs)
            r.in_specs = specs
            r.stage = op.stage
            r.microbatch = op.microbatch
            r.phase = op.phase
        outs = (ctypes.c_int * max(1, len(self.outputs)))(*self.outputs)
        keep.append(outs)
        self._keep = keep
        return arr, outs
