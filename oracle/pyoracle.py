"""ctypes binding of the CPU oracle (oracle/_build/libref_cpu_exec.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports this module.
"""
import ctypes
import os
import subprocess

import numpy as np

from paper_2302_08141_b200.abi import RH_BF16, RhOp, RhSpec

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libref_cpu_exec.so")
_lib = None


def build():
    subprocess.run(["make", "-s", "-C", HERE, "oracle"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.ox_last_error.restype = ctypes.c_char_p
        L.ox_synthetic_value.restype = ctypes.c_float
        L.ox_synthetic_value.argtypes = [ctypes.c_uint64, ctypes.c_uint32, ctypes.c_uint64,
                                         ctypes.c_int, ctypes.c_int64]
        L.ox_philox4x32_10.argtypes = [ctypes.POINTER(ctypes.c_uint32)] * 3
        L.ox_owner_of_flat.restype = ctypes.c_int64
        L.ox_owner_of_flat.argtypes = [ctypes.c_int, ctypes.POINTER(ctypes.c_int64), RhSpec,
                                       ctypes.c_int, ctypes.c_int64]
        L.ox_local_of_flat.restype = ctypes.c_int64
        L.ox_local_of_flat.argtypes = L.ox_owner_of_flat.argtypes
        L.ox_reshard.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int64), RhSpec,
                                 RhSpec, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p),
                                 ctypes.POINTER(ctypes.c_void_p)]
        L.ox_load.argtypes = [ctypes.POINTER(RhOp), ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                              ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                              ctypes.c_uint32, ctypes.POINTER(ctypes.c_void_p)]
        L.ox_destroy.argtypes = [ctypes.c_void_p]
        L.ox_init_synthetic.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
        L.ox_set_full.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t]
        L.ox_run_unpartitioned.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.ox_run_partitioned.argtypes = [ctypes.c_void_p, ctypes.c_int]
        L.ox_read_full.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                   ctypes.c_size_t]
        L.ox_read_local.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                    ctypes.c_size_t]
        L.ox_local_bytes.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_size_t)]
        L.ox_last_flops.restype = ctypes.c_double
        L.ox_last_flops.argtypes = [ctypes.c_void_p]
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise RuntimeError("oracle: " + lib().ox_last_error().decode())


def np_dtype(dtype):
    return np.uint16 if dtype == RH_BF16 else np.float32


def bf16_to_f32(a):
    return (a.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(a):
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32).astype(np.uint64)
    nan = (u & 0x7F800000) == 0x7F800000
    nan &= (u & 0x7FFFFF) != 0
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    r[nan] = ((u[nan] | 0x400000) >> 16).astype(np.uint16)
    return r


def philox(ctr, key):
    c = (ctypes.c_uint32 * 4)(*ctr)
    k = (ctypes.c_uint32 * 2)(*key)
    o = (ctypes.c_uint32 * 4)()
    lib().ox_philox4x32_10(c, k, o)
    return list(o)


def synthetic_value(seed, op_index, flat, is_param=False, fan_in=1):
    return lib().ox_synthetic_value(seed, op_index, flat, int(is_param), fan_in)


def owner_of_flat(dims, spec, d, flat):
    a = (ctypes.c_int64 * len(dims))(*dims)
    return lib().ox_owner_of_flat(len(dims), a, spec.to_c(), d, flat)


def local_of_flat(dims, spec, d, flat):
    a = (ctypes.c_int64 * len(dims))(*dims)
    return lib().ox_local_of_flat(len(dims), a, spec.to_c(), d, flat)


def reshard(d, dims, from_spec, to_spec, dtype, srcs, local_elems_to):
    """Single-axis transition over d ranks; srcs = list of numpy arrays (rank order)."""
    a = (ctypes.c_int64 * len(dims))(*dims)
    srcs = [np.ascontiguousarray(s) for s in srcs]
    dsts = [np.empty(local_elems_to, dtype=np_dtype(dtype)) for _ in range(d)]
    sp = (ctypes.c_void_p * d)(*[s.ctypes.data for s in srcs])
    dp = (ctypes.c_void_p * d)(*[x.ctypes.data for x in dsts])
    _check(lib().ox_reshard(d, len(dims), a, from_spec.to_c(), to_spec.to_c(), dtype, sp, dp))
    return dsts


class OracleProgram:
    """CPU execution of a LoweredProgram (unpartitioned and partitioned)."""

    KEEP_ALL = 0x100
    GEMM_F64 = 0x200

    def __init__(self, prog, flags=0, keep_all=False):
        self.prog = prog
        arr, outs = prog.to_c()
        mesh = (ctypes.c_int * len(prog.mesh))(*prog.mesh)
        h = ctypes.c_void_p()
        f = flags | (self.KEEP_ALL if keep_all else 0)
        _check(lib().ox_load(arr, len(prog.ops), outs, len(prog.outputs), len(prog.mesh), mesh, f,
                             ctypes.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ox_destroy(self.h)
            self.h = None

    def init_synthetic(self, seed):
        _check(lib().ox_init_synthetic(self.h, seed))

    def set_full(self, op, arr):
        arr = np.ascontiguousarray(arr)
        _check(lib().ox_set_full(self.h, op, arr.ctypes.data, arr.nbytes))

    def run_unpartitioned(self, threads=0):
        _check(lib().ox_run_unpartitioned(self.h, threads))

    def run_partitioned(self, threads=0):
        _check(lib().ox_run_partitioned(self.h, threads))

    def read_full(self, op, partitioned=False):
        o = self.prog.ops[op]
        out = np.empty(o.shape, dtype=np_dtype(self.prog.dtype))
        _check(lib().ox_read_full(self.h, op, int(partitioned), out.ctypes.data, out.nbytes))
        return out

    def read_local(self, op, rank):
        n = ctypes.c_size_t()
        _check(lib().ox_local_bytes(self.h, op, ctypes.byref(n)))
        out = np.empty(n.value // self.prog.elem_bytes(), dtype=np_dtype(self.prog.dtype))
        _check(lib().ox_read_local(self.h, op, rank, out.ctypes.data, out.nbytes))
        return out

    def last_flops(self):
        return lib().ox_last_flops(self.h)
