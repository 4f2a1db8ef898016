"""Python face of the CPU oracle — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may import
this module. It loads oracle/build/libposlo_oracle.so (the C restatement in
oracle/poslo_oracle.c) and re-exports oracle/ristretto.py, plus parsers for
the reference wire formats the tests need:
  - SeedStack wire        proj/src/seed_manager.cpp:32-53
  - EpochSignature "PSC1" proj/src/poslo_c.cpp:38-61
  - PoslocPublicKey "PPKC" proj/src/poslo_c.cpp:63-89
  - CCD "PCCD"            proj/src/distiller.cpp:235-302
"""
from __future__ import annotations

import ctypes
import os
import struct
import subprocess
from dataclasses import dataclass, field

from . import ristretto  # noqa: F401  (re-export)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "build", "libposlo_oracle.so")
REF_TOOL = os.path.join(HERE, "_ref", "ref_tool")
L = ristretto.L

OK, FORMAT_ERROR, STATE_ERROR, SEED_NOT_DISCLOSED = 0, 1, 2, 3


def build() -> str:
    os.makedirs(os.path.dirname(LIB_PATH), exist_ok=True)
    src = os.path.join(HERE, "poslo_oracle.c")
    if not os.path.exists(LIB_PATH) or os.path.getmtime(LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-fPIC", "-shared", "-o", LIB_PATH, src, "-lpthread"])
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
        c = ctypes
        _lib.orc_agg_ekeys.argtypes = [c.c_int, c.c_void_p, c.c_void_p, c.c_uint32, c.c_void_p,
                                       c.c_void_p, c.c_uint32, c.c_char_p, c.c_size_t, c.c_uint32,
                                       c.c_void_p, c.POINTER(c.c_uint32), c.c_int]
        _lib.orc_sr.argtypes = [c.c_int, c.c_char_p, c.c_size_t, c.c_uint32, c.c_uint32, c.c_char_p]
        _lib.orc_hash_to_scalar.argtypes = [c.c_int, c.c_char_p, c.c_size_t, c.c_char_p, c.c_char_p]
        _lib.orc_onetime_seed.argtypes = [c.c_int, c.c_char_p, c.c_uint32, c.c_char_p]
        _lib.orc_prf.argtypes = [c.c_int, c.c_int, c.c_char_p, c.c_char_p]
        _lib.orc_sha256.argtypes = [c.c_char_p, c.c_size_t, c.c_char_p]
        _lib.orc_aes128.argtypes = [c.c_char_p, c.c_char_p, c.c_char_p]
        _lib.orc_mmo.argtypes = [c.c_char_p, c.c_size_t, c.c_char_p]
        _lib.orc_mdc2.argtypes = [c.c_char_p, c.c_size_t, c.c_char_p]
        _lib.orc_reduce_wide_be.argtypes = [c.c_char_p, c.c_char_p]
        _lib.orc_sc_add.argtypes = [c.c_char_p, c.c_char_p, c.c_char_p]
    return _lib


def _out(n):
    return ctypes.create_string_buffer(n)


def sha256(m: bytes) -> bytes:
    o = _out(32); lib().orc_sha256(m, len(m), o); return o.raw


def aes128(key: bytes, block: bytes) -> bytes:
    o = _out(16); lib().orc_aes128(key, block, o); return o.raw


def mmo(m: bytes) -> bytes:
    o = _out(16)
    if lib().orc_mmo(m, len(m), o):
        raise ValueError("mmo_hash: empty message")
    return o.raw


def mdc2(m: bytes) -> bytes:
    o = _out(32)
    if lib().orc_mdc2(m, len(m), o):
        raise ValueError("mdc2_hash: empty message")
    return o.raw


def prf(suite: int, j: int, x: bytes) -> bytes:
    o = _out(16); lib().orc_prf(suite, j, x, o); return o.raw


def onetime_seed(suite: int, x0: bytes, j: int) -> bytes:
    o = _out(16); lib().orc_onetime_seed(suite, x0, j, o); return o.raw


def hash_to_scalar(suite: int, m: bytes, x: bytes) -> bytes:
    o = _out(32)
    if lib().orc_hash_to_scalar(suite, m, len(m), x, o):
        raise ValueError("FormatError")
    return o.raw


def reduce_wide_be(w: bytes) -> bytes:
    o = _out(32); lib().orc_reduce_wide_be(w, o); return o.raw


def sc_add(a: bytes, b: bytes) -> bytes:
    o = _out(32); lib().orc_sc_add(a, b, o); return o.raw


def sr(suite: int, ds: bytes, cap: int, i: int):
    o = _out(16)
    st = lib().orc_sr(suite, ds, len(ds), cap, i, o)
    return st, o.raw


def agg_ekeys_packed(suite, payload: bytes, offsets, entry_len, epochs, epoch_starts, ds: bytes,
                     cap: int, threads: int = os.cpu_count() or 1):
    """Returns (status, err_epoch, [e_tilde LE bytes per epoch])."""
    import numpy as np
    pay = np.frombuffer(payload, dtype=np.uint8) if len(payload) else np.zeros(1, np.uint8)
    offs = None if offsets is None else np.ascontiguousarray(offsets, dtype=np.uint64)
    eps = np.ascontiguousarray(epochs, dtype=np.uint32)
    starts = np.ascontiguousarray(epoch_starts, dtype=np.uint64)
    out = np.zeros(max(len(eps), 1) * 32, dtype=np.uint8)
    err = ctypes.c_uint32(0)
    st = lib().orc_agg_ekeys(suite, pay.ctypes.data, None if offs is None else offs.ctypes.data,
                             entry_len, eps.ctypes.data, starts.ctypes.data, len(eps), ds, len(ds),
                             cap, out.ctypes.data, ctypes.byref(err), threads)
    return st, err.value, [out[32 * k:32 * k + 32].tobytes() for k in range(len(eps))]


def sum_scalars(parts) -> bytes:
    acc = bytes(32)
    for p in parts:
        acc = sc_add(acc, p)
    return acc


# ---------------------------------------------------------------- wire formats
class _R:
    def __init__(self, b: bytes):
        self.b, self.o = b, 0

    def take(self, n):
        if len(self.b) - self.o < n:
            raise ValueError("truncated input")
        v = self.b[self.o:self.o + n]
        self.o += n
        return v

    def u8(self):
        return self.take(1)[0]

    def be32(self):
        return struct.unpack(">I", self.take(4))[0]


@dataclass
class PublicKey:
    suite: int
    n1: int
    n2: int
    n_u: int
    y: bytes
    r_hats: dict = field(default_factory=dict)

    @property
    def depth(self):
        return self.n1.bit_length() - 1


def parse_pk(b: bytes) -> PublicKey:
    r = _R(b)
    assert r.take(4) == b"PPKC"
    suite, n1, n2, nu = r.u8(), r.be32(), r.be32(), r.be32()
    y = r.take(32)
    pk = PublicKey(suite, n1, n2, nu, y)
    for _ in range(r.be32()):
        i = r.be32()
        pk.r_hats[i] = r.take(32)
    return pk


def parse_ds(r: _R) -> bytes:
    start = r.o
    c = r.u8()
    r.take(21 * c)
    return r.b[start:r.o]


@dataclass
class EpochSig:
    s_hat_le: bytes
    r_hat: bytes | None
    ds: bytes


def parse_sig(b: bytes) -> EpochSig:
    r = _R(b)
    assert r.take(4) == b"PSC1"
    s = r.take(32)[::-1]
    flag = r.u8()
    rh = r.take(32) if flag == 1 else None
    return EpochSig(s, rh, parse_ds(r))
