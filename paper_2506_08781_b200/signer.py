"""Signer side on the GPU: fixtures with the reference's own
key derivation at sizes the CPU signer cannot reach.

PoslocSecretKey::kg (poslo_c.cpp:91-113): R-hat_i = alpha^(sum_j
nonce_to_scalar(r, i, j)); sig_epoch (:115-134): s-hat_i = sum_j (r_ij -
e_ij y) = r-hat_i - y e~_i. Both run on the device (poslo_gpu_kg_commitments,
poslo_gpu_sig_epochs). The disclosed-seed stacks a live signer emits epoch by
epoch (`so`, seed_manager.cpp:55-69) are not reproduced: the fixtures carry
the root node, which discloses every epoch (the stack a finished stream ends
with).
"""
import ctypes
import struct
from dataclasses import dataclass
from typing import Dict, Optional, Sequence

import numpy as np

from . import api
from .api import FormatError, PackedBatch, SeedNode, SeedStack, SuiteConfig, _buf


@dataclass
class PoslocSecretKey:
    """poslo_c.hpp:33-70; wire "PSKC" (poslo_c.cpp:136-164)."""
    suite: SuiteConfig
    y: bytes          # secret scalar, 32 B little-endian
    r: bytes          # nonce seed, 16 B
    root: bytes       # seed-tree root value, 16 B
    next_epoch: int = 0
    ds: Optional[SeedStack] = None

    @staticmethod
    def deserialize(b: bytes) -> "PoslocSecretKey":
        if len(b) < 4 or b[:4] != b"PSKC":
            raise FormatError("bad magic, expected PSKC")
        if len(b) < 4 + 13 + 32 + 32 + 4:
            raise FormatError("truncated input")
        suite = SuiteConfig(b[4], *struct.unpack(">III", b[5:17]))
        suite.validate()
        y = api.scalar_from_be(b[17:49])
        r, root = bytes(b[49:65]), bytes(b[65:81])
        (nxt,) = struct.unpack(">I", b[81:85])
        ds, used = SeedStack.deserialize(b, suite.depth(), 85)
        if 85 + used != len(b):
            raise FormatError("trailing bytes")
        if nxt > suite.n1:
            raise FormatError("epoch out of range")
        return PoslocSecretKey(suite, y, r, root, nxt, ds)

    def root_stack(self) -> SeedStack:
        d = self.suite.depth()
        return SeedStack(d, [SeedNode(d, 0, self.root)])


def kg_public_key(sk: PoslocSecretKey, verifier: Optional[api.Verifier] = None,
                  epochs: Optional[Sequence[int]] = None) -> api.PoslocPublicKey:
    """The public key kg derives from sk (Y = alpha^y, R-hat_i for every epoch)."""
    v = verifier or api.default_verifier()
    ep = np.array(range(sk.suite.n1) if epochs is None else list(epochs), dtype=np.uint32)
    out = ctypes.create_string_buffer(max(len(ep), 1) * 32)
    v._call(v._lib.poslo_gpu_kg_commitments, sk.suite.suite, _buf(sk.r), ep.ctypes.data if len(ep) else None,
            len(ep), sk.suite.n2, out, None)
    raw = out.raw
    y_pub = v.exp_base(sk.y)
    return api.PoslocPublicKey(sk.suite, y_pub, {int(e): raw[32 * k:32 * k + 32] for k, e in enumerate(ep)})


def sign_epochs(sk: PoslocSecretKey, batches: Dict[int, Sequence[bytes]],
                verifier: Optional[api.Verifier] = None) -> Dict[int, bytes]:
    """s-hat (32 B LE) of every epoch of `batches`, as sig_epoch computes it."""
    v = verifier or api.default_verifier()
    pb = PackedBatch(sk.suite.suite, sk.suite.n2, batches, sk.root_stack())
    n = len(pb.epochs)
    out = ctypes.create_string_buffer(max(n, 1) * 32)
    cb = pb.cstruct()
    v._call(v._lib.poslo_gpu_sig_epochs, ctypes.byref(cb), _buf(sk.r), _buf(sk.y), out)
    raw = out.raw  # ctypes .raw copies the whole buffer per access
    return {int(e): raw[32 * k:32 * k + 32] for k, e in enumerate(pb.epochs)}
