"""ctypes mirror of include/rhino_exec.h (the C-ABI) and of the reference's AxisSpec.

`AxisSpec` follows parashard::AxisSpec (proj/include/parashard/sharding.h:32-53): wire strings
"shard(d,s)", "replicated", "partial" (also "R", "P"), parsed like AxisSpec::FromString
(proj/src/sharding.cpp:36-45).
"""
import ctypes
import re
from dataclasses import dataclass

RH_MAX_RANK = 8
RH_MAX_AXES = 4
RH_UID_BYTES = 128

RH_SHARD, RH_REPLICATED, RH_PARTIAL = 0, 1, 2
RH_F32, RH_BF16 = 0, 1

# parashard::OpKind order (proj/include/parashard/ir.h:58-70) and OpKindName (proj/src/ir.cpp:41-53).
OP_KINDS = ["param", "input", "matmul", "add", "mul", "unary", "reshape", "transpose",
            "reduce_sum", "broadcast", "concat"]
UNARY_FNS = {"": 0, "relu": 1, "gelu": 2, "tanh": 3, "exp": 4, "sigmoid": 5, "softmax": 6,
             "neg": 7, "rsqrt": 8, "identity": 9}

RH_FLAG_UNLABELED_IDENTITY = 0x1
RH_FLAG_NO_FUSION = 0x2
RH_FLAG_TRANSPORT_NCCL = 0x4
RH_FLAG_NO_MATERIALIZE = 0x8
RH_FLAG_SIMT_GEMM = 0x10
RH_FLAG_NO_GRAPH = 0x20
RH_FLAG_KEEP_ALL = 0x40
RH_FLAG_REDUCE_OUTPUTS = 0x80
RH_FLAG_NO_OVERLAP = 0x100
RH_FLAG_NO_PDL = 0x200


class RhSpec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("dim", ctypes.c_int32), ("stride", ctypes.c_int64)]


class RhOp(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("fn", ctypes.c_int32),
        ("dtype", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("dims", ctypes.c_int64 * RH_MAX_RANK),
        ("n_in", ctypes.c_int32),
        ("inputs", ctypes.POINTER(ctypes.c_int32)),
        ("transpose_a", ctypes.c_int32),
        ("transpose_b", ctypes.c_int32),
        ("axis", ctypes.c_int32),
        ("has_perm", ctypes.c_int32),
        ("perm", ctypes.c_int32 * RH_MAX_RANK),
        ("out_spec", RhSpec * RH_MAX_AXES),
        ("in_specs", ctypes.POINTER(RhSpec)),
        ("stage", ctypes.c_int32),
        ("microbatch", ctypes.c_int32),
        ("phase", ctypes.c_int32),
    ]


class RhStepInfo(ctypes.Structure):
    _fields_ = [
        ("name", ctypes.c_char * 64),
        ("kind", ctypes.c_int32),
        ("launches", ctypes.c_int32),
        ("alg_bytes", ctypes.c_double),
        ("alg_flops", ctypes.c_double),
        ("wire_bytes", ctypes.c_double),
        ("ms", ctypes.c_double),
    ]


_SHARD_RE = re.compile(r"^shard\((-?\d+),(-?\d+)\)$")


@dataclass(frozen=True)
class AxisSpec:
    kind: int
    dim: int = -1
    stride: int = 0

    @staticmethod
    def shard(dim, stride):
        return AxisSpec(RH_SHARD, dim, stride)

    @staticmethod
    def replicated():
        return AxisSpec(RH_REPLICATED)

    @staticmethod
    def partial():
        return AxisSpec(RH_PARTIAL)

    @staticmethod
    def from_string(s):
        if s in ("replicated", "R"):
            return AxisSpec.replicated()
        if s in ("partial", "P"):
            return AxisSpec.partial()
        m = _SHARD_RE.match(s.replace(" ", ""))
        if not m:
            raise ValueError(f"bad spec string {s!r}")
        return AxisSpec.shard(int(m.group(1)), int(m.group(2)))

    def __str__(self):
        if self.kind == RH_REPLICATED:
            return "replicated"
        if self.kind == RH_PARTIAL:
            return "partial"
        return f"shard({self.dim},{self.stride})"

    def to_c(self):
        return RhSpec(self.kind, self.dim, self.stride)

    @staticmethod
    def from_c(c):
        if c.kind == RH_SHARD:
            return AxisSpec.shard(c.dim, c.stride)
        return AxisSpec(c.kind)

    @property
    def is_shard(self):
        return self.kind == RH_SHARD


def spec_valid(spec, dims, d):
    """SpecValidForShape (proj/src/sharding.cpp:47-53)."""
    if spec.kind != RH_SHARD:
        return True
    if spec.dim < 0 or spec.dim >= len(dims) or spec.stride < 1:
        return False
    return dims[spec.dim] % (d * spec.stride) == 0


def local_shape(dims, spec, d):
    """LocalShape (proj/src/sharding.cpp:61-65)."""
    out = list(dims)
    if spec.kind == RH_SHARD:
        out[spec.dim] //= d
    return out


def composed_local_shape(dims, specs, mesh):
    """Axis k acts on the shape left by axes < k (EffectiveShapes, sharding.cpp:390-403)."""
    out = list(dims)
    for spec, d in zip(specs, mesh):
        out = local_shape(out, spec, d)
    return out


def rank_coords(rank, mesh):
    """Row-major, axis 0 slowest (grid.dims = {machines, gpus}, proj/src/planner.cpp:58-63)."""
    c = []
    for d in reversed(mesh):
        c.append(rank % d)
        rank //= d
    return list(reversed(c))
