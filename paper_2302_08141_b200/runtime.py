"""Python host mirror of the executor's C-ABI (include/rhino_exec.h) over ctypes.

The product path is the in-tree shared library paper_2302_08141_b200/lib/librhino_exec.so;
there is no CPU fallback: if the library is missing or a CUDA device is absent, calls fail.
"""
import ctypes
import os

import numpy as np

from .abi import RH_BF16, RH_UID_BYTES, RhOp, RhSpec, RhStepInfo
from .program import LoweredProgram

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "librhino_exec.so")

EXPORTS = [
    "rh_last_error", "rh_version", "rh_get_unique_id", "rh_runtime_create",
    "rh_runtime_create_dist", "rh_runtime_world", "rh_runtime_destroy", "rh_mesh_create",
    "rh_mesh_destroy", "rh_program_load", "rh_program_destroy", "rh_program_init_synthetic",
    "rh_program_write_full", "rh_program_run", "rh_program_step_host", "rh_program_run_host", "rh_program_read_local",
    "rh_program_read_full", "rh_program_read_input_full", "rh_program_local_bytes", "rh_program_memory", "rh_program_num_steps",
    "rh_program_step_info", "rh_program_profile", "rh_program_launch_count", "rh_reshard",
    "rh_op_natural_specs", "rh_program_load_pipeline",
]

_lib = None


class RhinoError(RuntimeError):
    pass


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RhinoError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i, u32, u64, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint64, ctypes.c_size_t
    P = ctypes.POINTER
    L.rh_last_error.restype = ctypes.c_char_p
    L.rh_version.restype = ctypes.c_char_p
    L.rh_get_unique_id.argtypes = [P(ctypes.c_uint8)]
    L.rh_runtime_create.argtypes = [i, P(i), P(vp)]
    L.rh_runtime_create_dist.argtypes = [i, i, i, P(ctypes.c_uint8), P(vp)]
    L.rh_runtime_world.argtypes = [vp, P(i), P(i), P(i)]
    L.rh_runtime_destroy.argtypes = [vp]
    L.rh_runtime_destroy.restype = None
    L.rh_mesh_create.argtypes = [vp, i, P(i), P(vp)]
    L.rh_mesh_destroy.argtypes = [vp]
    L.rh_mesh_destroy.restype = None
    L.rh_program_load.argtypes = [vp, P(RhOp), i, P(i), i, u32, P(vp)]
    L.rh_op_natural_specs.argtypes = [P(RhOp), i, i, i, P(i), P(RhSpec)]
    L.rh_program_load_pipeline.argtypes = [vp, i, P(RhOp), i, P(i), i, P(i), i, ctypes.c_float, u32, P(vp)]
    L.rh_program_destroy.argtypes = [vp]
    L.rh_program_destroy.restype = None
    L.rh_program_init_synthetic.argtypes = [vp, u64]
    L.rh_program_write_full.argtypes = [vp, i, vp, sz]
    L.rh_program_run.argtypes = [vp, i, P(ctypes.c_double)]
    L.rh_program_step_host.argtypes = [vp, i, P(i), P(vp), i, P(vp), P(ctypes.c_double)]
    L.rh_program_run_host.argtypes = [vp, i, i, P(i), P(vp), i, P(vp), P(ctypes.c_double)]
    L.rh_program_read_local.argtypes = [vp, i, i, vp, sz]
    L.rh_program_read_full.argtypes = [vp, i, vp, sz]
    L.rh_program_read_input_full.argtypes = [vp, i, i, vp, sz]
    L.rh_program_local_bytes.argtypes = [vp, i, i, P(sz)]
    L.rh_program_memory.argtypes = [vp, P(sz), P(sz)]
    L.rh_program_num_steps.argtypes = [vp, P(i)]
    L.rh_program_step_info.argtypes = [vp, i, P(RhStepInfo)]
    L.rh_program_profile.argtypes = [vp, i, P(ctypes.c_double)]
    L.rh_program_launch_count.argtypes = [vp, P(ctypes.c_int64)]
    L.rh_reshard.argtypes = [vp, i, RhSpec, RhSpec, i, P(ctypes.c_int64), i, P(vp), P(vp), u32, i,
                             P(ctypes.c_double)]
    _lib = L
    return L


def check(rc):
    if rc != 0:
        raise RhinoError(f"rhino_exec error {rc}: {lib().rh_last_error().decode()}")


def unique_id():
    buf = (ctypes.c_uint8 * RH_UID_BYTES)()
    check(lib().rh_get_unique_id(buf))
    return bytes(buf)


def natural_specs(prog: LoweredProgram, op: int):
    """rh_op_natural_specs: the executor's own local-op rule (host only): the per-axis output spec
    op `op` computes locally from the input specs its strategy demands."""
    ops, _ = prog.to_c()
    n = len(prog.mesh)
    dims = (ctypes.c_int * n)(*prog.mesh)
    out = (RhSpec * n)()
    check(lib().rh_op_natural_specs(ops, len(prog.ops), op, n, dims, out))
    from .abi import AxisSpec
    return [AxisSpec.from_c(out[a]) for a in range(n)]


class Runtime:
    """rh_runtime: all ranks in this process (`devices`, may repeat = emulated mesh), or one
    rank of a torchrun world (`dist=(world, rank, device, uid)`)."""

    def __init__(self, devices=None, dist=None):
        h = ctypes.c_void_p()
        if dist is not None:
            world, rank, dev, uid = dist
            u = (ctypes.c_uint8 * RH_UID_BYTES)(*uid)
            check(lib().rh_runtime_create_dist(world, rank, dev, u, ctypes.byref(h)))
        else:
            ids = (ctypes.c_int * len(devices))(*devices)
            check(lib().rh_runtime_create(len(devices), ids, ctypes.byref(h)))
        self.h = h
        w, f, n = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        check(lib().rh_runtime_world(h, ctypes.byref(w), ctypes.byref(f), ctypes.byref(n)))
        self.world, self.first_rank, self.n_local = w.value, f.value, n.value

    def close(self):
        if self.h:
            lib().rh_runtime_destroy(self.h)
            self.h = None


class Mesh:
    def __init__(self, runtime, dims):
        h = ctypes.c_void_p()
        arr = (ctypes.c_int * len(dims))(*dims)
        check(lib().rh_mesh_create(runtime.h, len(dims), arr, ctypes.byref(h)))
        self.h, self.rt, self.dims = h, runtime, list(dims)

    def close(self):
        if self.h:
            lib().rh_mesh_destroy(self.h)
            self.h = None

    def reshard(self, axis, from_spec, to_spec, dims, dtype, srcs, dsts, flags=0, iters=1):
        """rh_reshard: srcs/dsts = device pointers of this process's ranks."""
        n = len(srcs)
        d = (ctypes.c_int64 * len(dims))(*dims)
        sp = (ctypes.c_void_p * n)(*srcs)
        dp = (ctypes.c_void_p * n)(*dsts)
        ms = ctypes.c_double()
        check(lib().rh_reshard(self.h, axis, from_spec.to_c(), to_spec.to_c(), len(dims), d, dtype,
                               sp, dp, flags, iters, ctypes.byref(ms)))
        return ms.value


def _np_dtype(dtype):
    return np.uint16 if dtype == RH_BF16 else np.float32


class Program:
    """A loaded partitioned program (rh_program)."""

    def __init__(self, mesh, prog: LoweredProgram, flags=0):
        if list(mesh.dims) != list(prog.mesh):
            raise RhinoError(f"mesh {mesh.dims} does not match the plan's mesh {prog.mesh}")
        arr, outs = prog.to_c()
        h = ctypes.c_void_p()
        if getattr(prog, "pipeline_axis", -1) >= 0:  # rh_program_load_pipeline (wire format v2)
            ap = [x for pair in prog.apply for x in pair]
            apc = (ctypes.c_int * max(1, len(ap)))(*ap)
            check(lib().rh_program_load_pipeline(mesh.h, prog.pipeline_axis, arr, len(prog.ops), outs,
                                                 len(prog.outputs), apc, len(prog.apply), prog.lr, flags,
                                                 ctypes.byref(h)))
        else:
            check(lib().rh_program_load(mesh.h, arr, len(prog.ops), outs, len(prog.outputs), flags,
                                        ctypes.byref(h)))
        self.h, self.mesh, self.prog = h, mesh, prog

    def close(self):
        if self.h:
            lib().rh_program_destroy(self.h)
            self.h = None

    def init_synthetic(self, seed):
        check(lib().rh_program_init_synthetic(self.h, seed))

    def write_full(self, op, arr):
        arr = np.ascontiguousarray(arr)
        check(lib().rh_program_write_full(self.h, op, arr.ctypes.data, arr.nbytes))

    def run(self, iters=1):
        ms = ctypes.c_double()
        check(lib().rh_program_run(self.h, iters, ctypes.byref(ms)))
        return ms.value

    def profile(self, iters=1):
        ms = ctypes.c_double()
        check(lib().rh_program_profile(self.h, iters, ctypes.byref(ms)))
        return ms.value

    def step_host(self, in_ops, in_ptrs, out_ptrs):
        n = len(in_ops)
        ops = (ctypes.c_int * max(n, 1))(*in_ops)
        ip = (ctypes.c_void_p * max(n, 1))(*in_ptrs)
        op_ = (ctypes.c_void_p * max(len(out_ptrs), 1))(*out_ptrs)
        ms = ctypes.c_double()
        check(lib().rh_program_step_host(self.h, n, ops, ip, len(out_ptrs), op_, ctypes.byref(ms)))
        return ms.value

    def run_host(self, iters, in_ops, in_ptrs, out_ptrs):
        """Pipelined end-to-end steps (rh_program_run_host): ms per step."""
        n = len(in_ops)
        ops = (ctypes.c_int * max(n, 1))(*in_ops)
        ip = (ctypes.c_void_p * max(n, 1))(*in_ptrs)
        op_ = (ctypes.c_void_p * max(len(out_ptrs), 1))(*out_ptrs)
        ms = ctypes.c_double()
        check(lib().rh_program_run_host(self.h, iters, n, ops, ip, len(out_ptrs), op_, ctypes.byref(ms)))
        return ms.value

    def local_bytes(self, op, rank=0):
        n = ctypes.c_size_t()
        check(lib().rh_program_local_bytes(self.h, op, rank, ctypes.byref(n)))
        return n.value

    def read_local(self, op, rank):
        nb = self.local_bytes(op, rank)
        out = np.empty(nb // self.prog.elem_bytes(), dtype=_np_dtype(self.prog.dtype))
        check(lib().rh_program_read_local(self.h, op, rank, out.ctypes.data, out.nbytes))
        return out

    def read_full(self, op):
        out = np.empty(self.prog.ops[op].shape, dtype=_np_dtype(self.prog.dtype))
        check(lib().rh_program_read_full(self.h, op, out.ctypes.data, out.nbytes))
        return out

    def read_input_full(self, op, slot):
        """The value op `op` consumed at input `slot` (after resharding), assembled."""
        src = self.prog.ops[self.prog.ops[op].inputs[slot]]
        out = np.empty(src.shape, dtype=_np_dtype(self.prog.dtype))
        check(lib().rh_program_read_input_full(self.h, op, slot, out.ctypes.data, out.nbytes))
        return out

    def steps(self):
        n = ctypes.c_int()
        check(lib().rh_program_num_steps(self.h, ctypes.byref(n)))
        out = []
        for k in range(n.value):
            s = RhStepInfo()
            check(lib().rh_program_step_info(self.h, k, ctypes.byref(s)))
            out.append({"name": s.name.decode(), "kind": s.kind, "launches": s.launches,
                        "alg_bytes": s.alg_bytes, "alg_flops": s.alg_flops,
                        "wire_bytes": s.wire_bytes, "ms": s.ms})
        return out

    def memory(self):
        """(arena bytes, liveness-planned pool bytes) per rank."""
        a, p = ctypes.c_size_t(), ctypes.c_size_t()
        check(lib().rh_program_memory(self.h, ctypes.byref(a), ctypes.byref(p)))
        return a.value, p.value

    def launch_count(self):
        n = ctypes.c_int64()
        check(lib().rh_program_launch_count(self.h, ctypes.byref(n)))
        return n.value
