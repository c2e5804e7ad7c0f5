"""The per-program elementwise kernels (csrc/ew_jit.cpp) are compiled at program load by NVRTC
from device headers embedded in the library.  This CPU test compiles one program of every kernel
family through that path (no GPU needed), so a header change the run-time compiler rejects fails
here and not first on the B200.  The GPU tests check the compiled kernels' results
(test_gpu_parity.test_ew_jit_matches_interpreter and the parity suite, which runs on them)."""
import ctypes

from paper_2302_08141_b200 import runtime


def test_jit_headers_compile_with_nvrtc():
    L = runtime.lib()
    f = L.rh_test_ew_jit_compile
    f.restype = ctypes.c_longlong
    size = f()
    assert size > 10000, "NVRTC could not compile the embedded chain-program headers (see stderr)"
