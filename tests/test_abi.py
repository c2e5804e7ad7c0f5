"""The C-ABI library loads without a GPU and exports every entry point include/rhino_exec.h
declares (no compute calls here)."""
import os
import re

from paper_2302_08141_b200 import runtime

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    text = open(os.path.join(REPO, "include", "rhino_exec.h")).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rh_[a-z_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared()
    assert "rh_program_load" in names and "rh_reshard" in names
    assert set(names) == set(runtime.EXPORTS)


def test_library_exports_every_symbol():
    L = runtime.lib()
    for name in declared():
        assert hasattr(L, name), name
    assert L.rh_version().decode().startswith("rhino-b200")
    assert L.rh_last_error() is not None


def test_runtime_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        return
    try:
        runtime.Runtime(devices=[0])
    except runtime.RhinoError as e:
        assert "CUDA" in str(e) or "rhino" in str(e)
    else:
        raise AssertionError("runtime creation must fail without a CUDA device (no CPU fallback)")
