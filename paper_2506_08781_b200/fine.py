"""POSLO-F (fine-grained scheme) on the GPU: wire types and verifiers.

Mirrors include/poslo/poslo_f.hpp / src/poslo_f.cpp:
  PoslofPublicKey ("PPKF", poslo_f.cpp:88-104), FineSignature ("PSF1",
  :59-86), aver_f_single (:223-231), aver_f_batch (:233-246). Every scalar
  and group check runs on the device (poslo_gpu_fine_verify /
  poslo_gpu_aver_f_batch); entry seeds are either the signature's seed tail
  or derived on the device from a disclosed-seed stack.
"""
import ctypes
import struct
from dataclasses import dataclass
from typing import Dict, List, Optional, Sequence, Union

import numpy as np

from . import _native as N
from . import api
from .api import FormatError, SeedStack, SuiteConfig, _buf

NO_SLOT = 0xFFFFFFFF


@dataclass
class PoslofPublicKey:
    suite: SuiteConfig
    y: bytes

    def serialize(self) -> bytes:
        s = self.suite
        return b"PPKF" + bytes([s.suite]) + struct.pack(">III", s.n1, s.n2, s.n_u) + self.y

    @staticmethod
    def deserialize(b: bytes, verifier: Optional[api.Verifier] = None) -> "PoslofPublicKey":
        if len(b) < 4 or b[:4] != b"PPKF":
            raise FormatError("bad magic, expected PPKF")
        if len(b) < 4 + 13 + 32:
            raise FormatError("truncated input")
        suite = SuiteConfig(b[4], *struct.unpack(">III", b[5:17]))
        suite.validate()
        y = bytes(b[17:49])
        if not (verifier or api.default_verifier()).is_valid_point_batch([y])[0]:
            raise FormatError("invalid group element encoding")
        if len(b) != 49:
            raise FormatError("trailing bytes")
        return PoslofPublicKey(suite, y)


@dataclass
class FineSignature:
    s: bytes                          # 32 B little-endian
    r: bytes                          # 32 B ristretto255
    tail: Union[bytes, SeedStack]     # 16-byte seed, or the disclosed-seed stack (last entry of an epoch)

    def carries_ds(self) -> bool:
        return isinstance(self.tail, SeedStack)

    def serialize(self) -> bytes:
        out = b"PSF1" + self.s[::-1] + self.r
        if self.carries_ds():
            return out + b"\x01" + self.tail.serialize()
        return out + b"\x00" + self.tail

    @staticmethod
    def deserialize(b: bytes, depth: int, offset: int = 0, verifier: Optional[api.Verifier] = None,
                    validate: bool = True):
        """Returns (signature, bytes consumed). GroupElement::from_bytes
        validation of r runs on the device unless validate=False (the caller
        then validates a whole batch at once)."""
        o = offset
        if b[o:o + 4] != b"PSF1":
            raise FormatError("bad magic, expected PSF1")
        if len(b) - o < 4 + 64 + 1:
            raise FormatError("truncated input")
        s = api.scalar_from_be(b[o + 4:o + 36])
        r = bytes(b[o + 36:o + 68])
        if validate and not (verifier or api.default_verifier()).is_valid_point_batch([r])[0]:
            raise FormatError("invalid group element encoding")
        tag = b[o + 68]
        o += 69
        if tag == 0:
            if len(b) - o < 16:
                raise FormatError("truncated input")
            return FineSignature(s, r, bytes(b[o:o + 16])), o + 16 - offset
        if tag == 1:
            ds, used = SeedStack.deserialize(b, depth, o)
            return FineSignature(s, r, ds), o + used - offset
        raise FormatError("bad tail tag")


class FineBatch:
    """Packs scheme-F entries for poslo_fine_batch (include/poslo_gpu.h)."""

    def __init__(self, suite: int, msgs: Sequence[bytes], seeds: Sequence[Optional[bytes]],
                 derive: Optional[Sequence[Optional[tuple]]] = None,
                 slot_epochs: Sequence[int] = (), slot_ds: Optional[Sequence[SeedStack]] = None,
                 ds: Optional[SeedStack] = None, capacity: int = 0):
        """derive[t] = (slot, j) for entries whose seed comes from a stack, else None.
        Stacks: slot_ds (one per slot) or ds (shared)."""
        self.suite = suite
        n = len(msgs)
        self.n = n
        lens = [len(m) for m in msgs]
        self.payload = np.frombuffer(b"".join(msgs), dtype=np.uint8) if n and sum(lens) else np.zeros(1, np.uint8)
        self.payload_bytes = sum(lens)
        if n and all(x == lens[0] for x in lens):
            self.entry_len, self.offsets = lens[0], None
        else:
            self.entry_len = 0
            self.offsets = np.zeros(n + 1, dtype=np.uint64)
            if n:
                np.cumsum(lens, out=self.offsets[1:])
        self.seeds = np.frombuffer(b"".join(x if x is not None else bytes(16) for x in seeds), dtype=np.uint8) \
            if n else None
        self.slot = self.j = None
        if derive is not None:
            self.slot = np.array([d[0] if d else NO_SLOT for d in derive], dtype=np.uint32)
            self.j = np.array([d[1] if d else 0 for d in derive], dtype=np.uint32)
        self.slot_epochs = np.array(list(slot_epochs), dtype=np.uint32)
        self.ds_offsets = None
        if slot_ds is not None:
            blobs = [d.serialize() for d in slot_ds]
            self.ds_offsets = np.zeros(len(blobs) + 1, dtype=np.uint64)
            np.cumsum([len(x) for x in blobs], out=self.ds_offsets[1:])
            self.ds_bytes = b"".join(blobs) or b"\x00"
        else:
            self.ds_bytes = (ds or SeedStack(capacity)).serialize()
        self.capacity = capacity

    def cstruct(self) -> N.PosloFineBatch:
        f = N.PosloFineBatch()
        f.suite = self.suite
        f.payload = self.payload.ctypes.data
        f.payload_bytes = self.payload_bytes
        f.offsets = self.offsets.ctypes.data if self.offsets is not None else None
        f.entry_len = self.entry_len
        f.n_entries = self.n
        f.device_resident = 0
        f.seeds = self.seeds.ctypes.data if self.seeds is not None and len(self.seeds) else None
        f.derive_slot = self.slot.ctypes.data if self.slot is not None and len(self.slot) else None
        f.j = self.j.ctypes.data if self.j is not None and len(self.j) else None
        f.slot_epochs = self.slot_epochs.ctypes.data if len(self.slot_epochs) else None
        f.n_slots = len(self.slot_epochs)
        self._dsbuf = ctypes.create_string_buffer(self.ds_bytes, len(self.ds_bytes))
        f.ds = ctypes.addressof(self._dsbuf)
        f.ds_len = len(self.ds_bytes)
        f.ds_capacity = self.capacity
        f.ds_offsets = self.ds_offsets.ctypes.data if self.ds_offsets is not None else None
        return f


def fine_scalars(v: api.Verifier, fb: FineBatch, want_each=True, want_sum=False):
    out = ctypes.create_string_buffer(max(fb.n, 1) * 32) if want_each else None
    tot = ctypes.create_string_buffer(32) if want_sum else None
    cs = fb.cstruct()
    v._call(v._lib.poslo_gpu_fine_scalars, ctypes.byref(cs), out, tot)
    raw = out.raw  # ctypes .raw copies the whole buffer per access
    each = [raw[32 * k:32 * k + 32] for k in range(fb.n)] if want_each else None
    return each, (tot.raw if want_sum else None)


def fine_verify(v: api.Verifier, fb: FineBatch, y: bytes, s: Sequence[bytes], r: Sequence[bytes]) -> List[bool]:
    verd = ctypes.create_string_buffer(max(fb.n, 1))
    cs = fb.cstruct()
    v._call(v._lib.poslo_gpu_fine_verify, ctypes.byref(cs), _buf(y), _buf(b"".join(s)) if s else None,
            _buf(b"".join(r)) if r else None, verd)
    vr = verd.raw
    return [bool(vr[k]) for k in range(fb.n)]


def aver_f_single_batch(pk: PoslofPublicKey, msgs: Sequence[bytes], sigs: Sequence[FineSignature],
                        verifier: Optional[api.Verifier] = None) -> List[bool]:
    """aver_f_single (poslo_f.cpp:223-231) for many entries in one device call."""
    for sg in sigs:
        if sg.carries_ds():
            raise FormatError("single-entry verification needs the seed tail, not ds")
    v = verifier or api.default_verifier()
    fb = FineBatch(pk.suite.suite, msgs, [sg.tail for sg in sigs])
    return fine_verify(v, fb, pk.y, [sg.s for sg in sigs], [sg.r for sg in sigs])


def aver_f_single(pk: PoslofPublicKey, msg: bytes, sig: FineSignature,
                  verifier: Optional[api.Verifier] = None) -> bool:
    return aver_f_single_batch(pk, [msg], [sig], verifier)[0]


def aver_f_batch(pk: PoslofPublicKey, entries: Dict[int, bytes], s: bytes, r: bytes, ds: SeedStack,
                 verifier: Optional[api.Verifier] = None) -> bool:
    """aver_f_batch (poslo_f.cpp:233-246): entries = global index -> message."""
    v = verifier or api.default_verifier()
    n2 = pk.suite.n2
    ts = sorted(entries)
    epochs = sorted({t // n2 for t in ts})
    slot = {e: k for k, e in enumerate(epochs)}
    fb = FineBatch(pk.suite.suite, [entries[t] for t in ts], [None] * len(ts),
                   [(slot[t // n2], t % n2) for t in ts], epochs, None, ds, ds.capacity)
    verdict = ctypes.c_uint8(0)
    cs = fb.cstruct()
    v._call(v._lib.poslo_gpu_aver_f_batch, ctypes.byref(cs), _buf(pk.y), _buf(s), _buf(r), ctypes.byref(verdict))
    return bool(verdict.value)
