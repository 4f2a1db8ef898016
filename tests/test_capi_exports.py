"""The C-ABI library loads and exports every symbol include/poslo_gpu.h
declares; without a GPU every call fails loudly (no CPU fallback). CPU only."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "poslo_gpu.h")).read()
    return sorted(set(re.findall(r"\b(poslo_(?:gpu|log)_[a-z_0-9]+)\s*\(", src)))


def test_header_matches_binding():
    from paper_2506_08781_b200 import _native as N
    assert set(declared_symbols()) == set(N.EXPORTS)


def test_library_exports_every_declared_symbol():
    from paper_2506_08781_b200 import _native as N
    lib = N.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.poslo_gpu_version()


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2506_08781_b200 import DeviceError, Verifier
    with pytest.raises(DeviceError):
        Verifier(0)


def test_sass_is_sm100a():
    import subprocess
    lib = os.path.join(ROOT, "paper_2506_08781_b200", "libposlo_gpu.so")
    out = subprocess.run(["cuobjdump", "--list-elf", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out
