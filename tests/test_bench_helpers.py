"""bench.py helpers that must agree with the C generator (include/poslo_synth.h):
the numpy port of the variable-length generator. CPU only."""
import ctypes
import os
import subprocess
import tempfile

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_synth_varlen_numpy_port_matches_c():
    from paper_2506_08781_b200 import synth as bench
    src = ('#include "poslo_synth.h"\n'
           'uint32_t vl(uint64_t s, uint64_t k) { return poslo_synth_varlen(s, k); }\n'
           'uint8_t ab(uint64_t s, uint64_t k, uint32_t b) { return poslo_synth_ascii(s, k, b); }\n')
    d = tempfile.mkdtemp()
    c = os.path.join(d, "s.c")
    so = os.path.join(d, "s.so")
    open(c, "w").write(src)
    subprocess.check_call(["gcc", "-O2", "-shared", "-fPIC", "-I", os.path.join(ROOT, "include"), c, "-o", so])
    lib = ctypes.CDLL(so)
    lib.vl.restype = ctypes.c_uint32
    lib.vl.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
    for seed, first in ((0x5EED, 0), (7, 123456789), (2**63 + 5, 2**40)):
        got = bench.synth_varlen(seed, first, 1000)
        ref = np.array([lib.vl(seed, first + t) for t in range(1000)], dtype=np.uint64)
        assert (got == ref).all()
        assert got.min() >= 64 and got.max() <= 1024
