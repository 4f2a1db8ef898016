"""Host-side mirror of the reference's batch-verification interface.

Same names, argument meaning and error behaviour as the reference C++ API
(/root/reference/proj/include/poslo/batch_verify.hpp:11-30, poslo_c.hpp,
seed_manager.hpp, common.hpp:22-40), over the C-ABI in include/poslo_gpu.h.
Every compute call goes to the CUDA library; nothing here computes a hash,
a scalar or a group element on the CPU.

Scalars are 32-byte little-endian `bytes` (the reference's in-memory
Scalar form); wire formats use big-endian as the reference does.
"""
from __future__ import annotations

import ctypes
import struct
import threading
from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from . import _native as N

L = 2**252 + 27742317777372353535851937790883648493


# ---------------------------------------------------------------- errors (common.hpp:22-40)
class FormatError(RuntimeError):
    """Malformed input: wrong lengths, bad encodings, broken files."""


class StateError(RuntimeError):
    """An operation asked for something its state cannot provide."""


class SeedNotDisclosed(RuntimeError):
    """Seed retrieval for an epoch the disclosed-seed stack does not cover."""

    def __init__(self, epoch: int):
        super().__init__(f"seed for epoch {epoch} not yet disclosed")
        self.epoch = epoch


class DeviceError(RuntimeError):
    """CUDA failure or missing sm_100 device (there is no CPU fallback)."""


def _raise(rc: int, err: N.PosloError):
    msg = err.message.decode(errors="replace")
    if rc == N.FORMAT_ERROR:
        e = FormatError(msg)
        e.epoch = err.epoch
        raise e
    if rc == N.STATE_ERROR:
        e = StateError(msg)
        e.epoch = err.epoch
        raise e
    if rc == N.SEED_NOT_DISCLOSED:
        raise SeedNotDisclosed(err.epoch)
    if rc == N.INVALID_ARGUMENT:
        raise ValueError(msg)
    raise DeviceError(msg)


# ---------------------------------------------------------------- types
SHA256, MMO_MDC2, MMO_ADDQ = 1, 2, 3


@dataclass
class SuiteConfig:
    """primitives.hpp:19-28"""
    suite: int = SHA256
    n1: int = 0
    n2: int = 0
    n_u: int = 1

    def depth(self) -> int:
        d, v = 0, self.n1
        while v > 1:
            v >>= 1
            d += 1
        return d

    def validate(self):
        if self.suite not in (1, 2, 3):
            raise FormatError("unknown suite id")
        if self.n1 < 2 or self.n1 & (self.n1 - 1):
            raise FormatError("n1 must be a power of two >= 2")
        if self.n2 < 1:
            raise FormatError("n2 must be positive")
        if self.n_u < 1 or self.n1 % self.n_u:
            raise FormatError("n_u must be positive and divide n1")


@dataclass
class SeedNode:
    depth: int
    index: int
    value: bytes


@dataclass
class SeedStack:
    """Disclosed-seed stack; wire format seed_manager.cpp:32-53."""
    capacity: int = 0
    nodes: List[SeedNode] = field(default_factory=list)

    def serialize(self) -> bytes:
        out = bytearray([len(self.nodes)])
        for n in self.nodes:
            out += bytes([n.depth]) + struct.pack(">I", n.index) + n.value
        return bytes(out)

    @staticmethod
    def deserialize(b: bytes, capacity: int, offset: int = 0):
        """Returns (stack, bytes consumed)."""
        if len(b) - offset < 1:
            raise FormatError("truncated input")
        cnt = b[offset]
        o = offset + 1
        st = SeedStack(capacity)
        for _ in range(cnt):
            if len(b) - o < 21:
                raise FormatError("truncated input")
            n = SeedNode(b[o], struct.unpack(">I", b[o + 1:o + 5])[0], bytes(b[o + 5:o + 21]))
            if len(st.nodes) >= capacity:
                raise StateError("seed stack overflow")
            if st.nodes and st.nodes[-1].depth <= n.depth:
                raise StateError("seed stack depth order violated")
            st.nodes.append(n)
            o += 21
        return st, o - offset


def scalar_from_be(b: bytes) -> bytes:
    """Scalar::from_be_bytes (group.cpp:46-49): rejects values >= l."""
    if len(b) != 32 or int.from_bytes(b, "big") >= L:
        raise FormatError("non-canonical scalar")
    return bytes(b[::-1])


@dataclass
class PoslocPublicKey:
    """poslo_c.hpp:22-31; wire "PPKC" poslo_c.cpp:63-89."""
    suite: SuiteConfig
    y: bytes
    r_hats: Dict[int, bytes] = field(default_factory=dict)

    def serialize(self) -> bytes:
        s = self.suite
        out = bytearray(b"PPKC") + bytes([s.suite]) + struct.pack(">III", s.n1, s.n2, s.n_u)
        out += self.y + struct.pack(">I", len(self.r_hats))
        for i in sorted(self.r_hats):
            out += struct.pack(">I", i) + self.r_hats[i]
        return bytes(out)

    @staticmethod
    def deserialize(b: bytes, verifier: "Verifier" = None) -> "PoslocPublicKey":
        if len(b) < 4 or b[:4] != b"PPKC":
            raise FormatError("bad magic, expected PPKC")
        if len(b) < 4 + 13 + 32 + 4:
            raise FormatError("truncated input")
        suite = SuiteConfig(b[4], *struct.unpack(">III", b[5:17]))
        suite.validate()
        y = bytes(b[17:49])
        (cnt,) = struct.unpack(">I", b[49:53])
        o = 53
        r = {}
        pts = [y]
        for _ in range(cnt):
            if len(b) - o < 36:
                raise FormatError("truncated input")
            i = struct.unpack(">I", b[o:o + 4])[0]
            r.setdefault(i, bytes(b[o + 4:o + 36]))
            pts.append(bytes(b[o + 4:o + 36]))
            o += 36
        if o != len(b):
            raise FormatError("trailing bytes")
        # GroupElement::from_bytes membership validation, on the device
        v = verifier or default_verifier()
        if not all(v.is_valid_point_batch(pts)):
            raise FormatError("invalid group element encoding")
        return PoslocPublicKey(suite, y, r)


@dataclass
class EpochSignature:
    """poslo_c.hpp:14-20; wire "PSC1" poslo_c.cpp:38-61."""
    s_hat: bytes                     # 32 B little-endian
    r_hat: Optional[bytes]
    ds: SeedStack

    def serialize(self) -> bytes:
        out = bytearray(b"PSC1") + self.s_hat[::-1]
        out += b"\x01" + self.r_hat if self.r_hat is not None else b"\x00"
        return bytes(out + self.ds.serialize())

    @staticmethod
    def deserialize(b: bytes, depth: int, offset: int = 0):
        o = offset
        if b[o:o + 4] != b"PSC1":
            raise FormatError("bad magic, expected PSC1")
        if len(b) - o < 37:
            raise FormatError("truncated input")
        s = scalar_from_be(b[o + 4:o + 36])
        flag = b[o + 36]
        o += 37
        r = None
        if flag == 1:
            if len(b) - o < 32:
                raise FormatError("truncated input")
            r = bytes(b[o:o + 32])
            o += 32
        elif flag != 0:
            raise FormatError("bad commitment presence flag")
        ds, used = SeedStack.deserialize(b, depth, o)
        return EpochSignature(s, r, ds), o + used - offset


# ---------------------------------------------------------------- packing
class PackedBatch:
    """The map<u32, vector<Bytes>> of the reference packed into one payload
    buffer + offsets (or a fixed stride) + epoch ranges (include/poslo_gpu.h)."""

    def __init__(self, suite: int, n2: int, batches: Dict[int, Sequence[bytes]], ds: SeedStack,
                 epoch_ds: Optional[Dict[int, SeedStack]] = None):
        """epoch_ds: optional per-epoch seed stacks (EpochSignature::ds): epoch i is
        then derived from epoch_ds[i] instead of ds (poslo_batch.ds_offsets)."""
        self.suite = suite
        self.n2 = n2
        self.epochs = np.array(sorted(batches), dtype=np.uint32)
        counts = [len(batches[int(e)]) for e in self.epochs]
        flat = [m for e in self.epochs for m in batches[int(e)]]
        lens = [len(m) for m in flat]
        self.payload = np.frombuffer(b"".join(flat), dtype=np.uint8) if flat else np.zeros(0, np.uint8)
        self.n_entries = len(flat)
        if lens and all(x == lens[0] for x in lens):
            self.entry_len, self.offsets = lens[0], None
        elif not lens:
            self.entry_len, self.offsets = 0, None
        else:
            self.entry_len = 0
            self.offsets = np.zeros(len(lens) + 1, dtype=np.uint64)
            np.cumsum(lens, out=self.offsets[1:])
        if all(c == n2 for c in counts):
            self.starts = None
        else:
            self.starts = np.zeros(len(counts) + 1, dtype=np.uint64)
            np.cumsum(counts, out=self.starts[1:])
        self.ds_bytes = ds.serialize()
        self.ds_capacity = ds.capacity
        self.ds_offsets = None
        if epoch_ds is not None:
            blobs = [epoch_ds[int(e)].serialize() for e in self.epochs]
            self.ds_offsets = np.zeros(len(blobs) + 1, dtype=np.uint64)
            np.cumsum([len(x) for x in blobs], out=self.ds_offsets[1:])
            self.ds_bytes = b"".join(blobs) or b"\x00"
        self._keep = []

    def cstruct(self) -> N.PosloBatch:
        b = N.PosloBatch()
        b.suite = self.suite
        b.n2 = self.n2
        pay = self.payload if len(self.payload) else np.zeros(1, np.uint8)
        self._keep = [pay]
        b.payload = pay.ctypes.data
        b.payload_bytes = len(self.payload)
        b.offsets = self.offsets.ctypes.data if self.offsets is not None else None
        b.entry_len = self.entry_len
        b.n_entries = self.n_entries
        b.epochs = self.epochs.ctypes.data if len(self.epochs) else None
        b.epoch_starts = self.starts.ctypes.data if self.starts is not None else None
        b.n_epochs = len(self.epochs)
        self._dsbuf = ctypes.create_string_buffer(self.ds_bytes, len(self.ds_bytes))
        b.ds = ctypes.addressof(self._dsbuf)
        b.ds_len = len(self.ds_bytes)
        b.ds_capacity = self.ds_capacity
        b.device_resident = 0
        b.ds_offsets = self.ds_offsets.ctypes.data if self.ds_offsets is not None else None
        return b


def _buf(b: Optional[bytes]):
    return None if b is None else ctypes.create_string_buffer(bytes(b), len(b))


# ---------------------------------------------------------------- verifier
class Verifier:
    """One device context (re-entrant; calls on one context serialise).

    devices: several device indices -> a multi-device context
    (poslo_gpu_create_multi): agg_ekeys / paver / epoch_verify / distillation
    shard their epochs over the members and combine on the first; a device may
    repeat (members sharing one GPU)."""

    def __init__(self, device: int = 0, devices: Optional[Sequence[int]] = None):
        self._lib = N.load()
        self._ctx = ctypes.c_void_p()
        err = N.PosloError()
        if devices is not None and len(devices) > 1:
            arr = (ctypes.c_int * len(devices))(*devices)
            rc = self._lib.poslo_gpu_create_multi(arr, len(devices), ctypes.byref(self._ctx), ctypes.byref(err))
            device = devices[0]
        else:
            if devices:
                device = devices[0]
            rc = self._lib.poslo_gpu_create(device, ctypes.byref(self._ctx), ctypes.byref(err))
        if rc:
            _raise(rc, err)
        self.device = device

    def members(self) -> int:
        return int(self._lib.poslo_gpu_member_count(self._ctx))

    def close(self):
        if self._ctx:
            self._lib.poslo_gpu_destroy(self._ctx)
            self._ctx = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _call(self, fn, *args):
        err = N.PosloError()
        rc = fn(self._ctx, *args, ctypes.byref(err))
        if rc:
            _raise(rc, err)

    def set_stream(self, stream_ptr: int):
        self._lib.poslo_gpu_set_stream(self._ctx, stream_ptr or None)

    def enable_timing(self, on: bool = True):
        self._lib.poslo_gpu_enable_timing(self._ctx, 1 if on else 0)

    def last_timings(self):
        arr = (ctypes.c_float * 6)()
        self._lib.poslo_gpu_last_timings(self._ctx, arr)
        return dict(zip(["seed", "hash", "finalize", "sum", "group", "total"], list(arr)))

    def last_launches(self) -> int:
        return int(self._lib.poslo_gpu_last_launches(self._ctx))

    # -- group operation counters (group.hpp:86-97), process-wide
    def group_op_counts(self) -> Dict[str, int]:
        arr = (ctypes.c_uint64 * 4)()
        self._lib.poslo_gpu_group_op_counts(arr)
        return dict(zip(["exp_base", "exp_var", "double_exp", "combine"], [int(x) for x in arr]))

    def reset_group_op_counts(self):
        self._lib.poslo_gpu_reset_group_op_counts()

    # -- multi-rank coarse PAVer: partial e-hat into device memory, rank-ordered fold + check
    def agg_ekeys_partial(self, cb: "N.PosloBatch", d_out: int):
        """e-hat of this shard's batch (a filled N.PosloBatch) into 32 bytes of device memory."""
        self._call(self._lib.poslo_gpu_agg_ekeys_partial, ctypes.byref(cb), ctypes.c_void_p(d_out))

    def combine_check_prepare(self, y: bytes, s_hat: bytes, r_hat: bytes):
        """Queues the e-hat-independent half of the next combine_check with these
        inputs (overlaps the caller's hashing and all-gather)."""
        self._call(self._lib.poslo_gpu_combine_check_prepare, _buf(y), _buf(s_hat), _buf(r_hat))

    def combine_check(self, parts, y: bytes, s_hat: bytes, r_hat: bytes, n_parts: Optional[int] = None) -> bool:
        """parts: bytes (host, n x 32) or an int device pointer (then n_parts is required)."""
        v = ctypes.c_uint8(0)
        if isinstance(parts, int):
            self._call(self._lib.poslo_gpu_combine_check, n_parts, ctypes.c_void_p(parts), 1, _buf(y), _buf(s_hat),
                       _buf(r_hat), ctypes.byref(v))
        else:
            self._call(self._lib.poslo_gpu_combine_check, len(parts) // 32, _buf(parts), 0, _buf(y), _buf(s_hat),
                       _buf(r_hat), ctypes.byref(v))
        return bool(v.value)

    # -- agg_ekeys / aggregate_ekey (batch_verify.cpp:11-62, poslo_c.cpp:177-190)
    def agg_ekeys(self, suite: SuiteConfig, batches: Dict[int, Sequence[bytes]], ds: SeedStack,
                  workers: int = 1):
        if workers == 0:
            raise StateError("worker count must be at least 1")
        pb = PackedBatch(suite.suite, suite.n2, batches, ds)
        return self.agg_ekeys_packed(pb)

    def agg_ekeys_log(self, rb):
        """agg_ekeys over a RecordBatch (logfile.py): the raw log image is hashed in place."""
        return self.agg_ekeys_packed(rb)

    def paver_log(self, pk: PoslocPublicKey, rb, s_hat: bytes, r_hat_agg: Optional[bytes] = None) -> bool:
        """paver over a RecordBatch (every epoch holds n2 records by construction)."""
        r_hats = None
        if r_hat_agg is None:
            rows = []
            for i in rb.epochs:
                if int(i) not in pk.r_hats:
                    raise StateError(f"commitment for epoch {int(i)} no longer in public key")
                rows.append(pk.r_hats[int(i)])
            r_hats = b"".join(rows)
        cb = rb.cstruct()
        v = ctypes.c_uint8(0)
        self._call(self._lib.poslo_gpu_paver, ctypes.byref(cb), _buf(pk.y), _buf(s_hat),
                   _buf(r_hat_agg), _buf(r_hats), ctypes.byref(v))
        return bool(v.value)

    def agg_ekeys_packed(self, pb: PackedBatch):
        n = len(pb.epochs)
        out = ctypes.create_string_buffer(max(n, 1) * 32)
        tot = ctypes.create_string_buffer(32)
        cb = pb.cstruct()
        self._call(self._lib.poslo_gpu_agg_ekeys, ctypes.byref(cb), out, tot)
        raw = out.raw
        return [(int(pb.epochs[k]), raw[32 * k:32 * k + 32]) for k in range(n)], tot.raw

    def aggregate_ekey(self, suite: SuiteConfig, batches, ds: SeedStack) -> bytes:
        return self.agg_ekeys(suite, batches, ds)[1]

    # -- paver (batch_verify.cpp:64-87)
    def paver(self, pk: PoslocPublicKey, batches: Dict[int, Sequence[bytes]], s_hat: bytes,
              r_hat_agg: Optional[bytes], ds: SeedStack, workers: int = 1) -> bool:
        for i, msgs in batches.items():
            if len(msgs) != pk.suite.n2:
                raise StateError("every batch must hold exactly n2 entries")
        r_hats = None
        if r_hat_agg is None:
            rows = []
            for i in sorted(batches):
                if i not in pk.r_hats:
                    raise StateError(f"commitment for epoch {i} no longer in public key")
                rows.append(pk.r_hats[i])
            r_hats = b"".join(rows)
        if workers == 0:
            raise StateError("worker count must be at least 1")
        pb = PackedBatch(pk.suite.suite, pk.suite.n2, batches, ds)
        cb = pb.cstruct()
        v = ctypes.c_uint8(0)
        self._call(self._lib.poslo_gpu_paver, ctypes.byref(cb), _buf(pk.y), _buf(s_hat),
                   _buf(r_hat_agg), _buf(r_hats), ctypes.byref(v))
        return bool(v.value)

    def aver(self, pk, batches, s_hat, r_hat_agg, ds) -> bool:
        """aver (poslo_c.cpp:192-213) has the same decision as paver."""
        return self.paver(pk, batches, s_hat, r_hat_agg, ds, 1)

    # -- per-epoch verdicts (distill_epoch's aver per epoch, distiller.cpp:60-89)
    def epoch_verify(self, pk: PoslocPublicKey, batches, s_hats: Dict[int, bytes], ds: SeedStack):
        pb = PackedBatch(pk.suite.suite, pk.suite.n2, batches, ds)
        eps = [int(e) for e in pb.epochs]
        s = b"".join(s_hats[e] for e in eps)
        r = b"".join(pk.r_hats[e] for e in eps)
        out = ctypes.create_string_buffer(max(len(eps), 1))
        et = ctypes.create_string_buffer(max(len(eps), 1) * 32)
        cb = pb.cstruct()
        self._call(self._lib.poslo_gpu_epoch_verify, ctypes.byref(cb), _buf(pk.y), _buf(s), _buf(r),
                   out, et)
        raw = out.raw
        return [bool(raw[k]) for k in range(len(eps))]

    def epoch_verify_packed(self, pk: PoslocPublicKey, pb, s_hats: Dict[int, bytes]):
        """epoch_verify over a packed / record / image batch (logfile.py). A
        device-resident batch takes device-resident signature arrays too (the
        C-ABI contract), so s-hat / R-hat are staged into HBM for it."""
        eps = [int(e) for e in pb.epochs]
        s = b"".join(s_hats[e] for e in eps)
        r = b"".join(pk.r_hats[e] for e in eps)
        out = ctypes.create_string_buffer(max(len(eps), 1))
        cb = pb.cstruct()
        if cb.device_resident:
            import torch
            keep = [torch.frombuffer(bytearray(x or b"\0"), dtype=torch.uint8).cuda() for x in (s, r)]
            torch.cuda.synchronize()
            sp, rp = (ctypes.c_void_p(t.data_ptr()) for t in keep)
        else:
            sp, rp = _buf(s), _buf(r)
        self._call(self._lib.poslo_gpu_epoch_verify, ctypes.byref(cb), _buf(pk.y), sp, rp, out, None)
        raw = out.raw
        return [bool(raw[k]) for k in range(len(eps))]

    # -- batched coarse distillation (distiller.cpp:60-89): verdicts + masked umbrella folds
    def distill_coarse(self, pk: PoslocPublicKey, batches, sigs: Dict[int, "EpochSignature"],
                       seg: Sequence[int], want_e: bool = False):
        """Epochs of `batches` (consecutive, n2 entries each) verified against
        their own signatures (s_hat, pk.r_hats[i], sig.ds). seg: batch-position
        boundaries (len n_seg + 1). Returns (verdicts, [(s_le, r)] per segment),
        with want_e (verdicts, [(s_le, r, e_le)]): e = sum of the segment's valid e~."""
        ds_any = next(iter(sigs.values())).ds if sigs else SeedStack(pk.suite.depth())
        pb = PackedBatch(pk.suite.suite, pk.suite.n2, batches, ds_any,
                         epoch_ds={i: sigs[i].ds for i in batches})
        eps = [int(e) for e in pb.epochs]
        s = b"".join(sigs[e].s_hat for e in eps)
        r = b"".join(pk.r_hats[e] for e in eps)
        segs = np.array(seg, dtype=np.uint32)
        ng = max(len(segs) - 1, 0)
        verd = ctypes.create_string_buffer(max(len(eps), 1))
        out_s = ctypes.create_string_buffer(max(ng, 1) * 32)
        out_r = ctypes.create_string_buffer(max(ng, 1) * 32)
        out_e = ctypes.create_string_buffer(max(ng, 1) * 32)
        cb = pb.cstruct()
        self._call(self._lib.poslo_gpu_distill_coarse_ex, ctypes.byref(cb), _buf(pk.y), _buf(s) if s else None,
                   _buf(r) if r else None, segs.ctypes.data if ng else None, ng, verd, out_s, out_r,
                   out_e if want_e else None)
        vr, sr_, rr, er = verd.raw, out_s.raw, out_r.raw, out_e.raw
        if want_e:
            return ([bool(vr[k]) for k in range(len(eps))],
                    [(sr_[32 * g:32 * g + 32], rr[32 * g:32 * g + 32], er[32 * g:32 * g + 32]) for g in range(ng)])
        return ([bool(vr[k]) for k in range(len(eps))],
                [(sr_[32 * g:32 * g + 32], rr[32 * g:32 * g + 32]) for g in range(ng)])

    def distill_step(self, pk: PoslocPublicKey, epoch: int, msgs: Sequence[bytes], sig: "EpochSignature",
                     acc: Sequence[Tuple[bytes, bytes]]):
        """ONE distill_epoch (distiller.cpp:60-89) in one device round trip
        (poslo_gpu_distill_step): returns (verdict, [valid (s, r), umbrella (s, r)])
        with (sig.s_hat, pk.r_hats[epoch]) folded into both aggregates when valid."""
        pb = PackedBatch(pk.suite.suite, pk.suite.n2, {epoch: list(msgs)}, sig.ds)
        cb = pb.cstruct()
        acc_s = acc[0][0] + acc[1][0]
        acc_r = acc[0][1] + acc[1][1]
        v = ctypes.c_uint8(0)
        out_s = ctypes.create_string_buffer(64)
        out_r = ctypes.create_string_buffer(64)
        self._call(self._lib.poslo_gpu_distill_step, ctypes.byref(cb), _buf(pk.y), _buf(sig.s_hat),
                   _buf(pk.r_hats[epoch]), _buf(acc_s), _buf(acc_r), ctypes.byref(v), out_s, out_r)
        rs, rr = out_s.raw, out_r.raw
        return bool(v.value), [(rs[:32], rr[:32]), (rs[32:], rr[32:])]

    def segfold(self, scalars: Sequence[bytes], points: Sequence[bytes], mask: Optional[Sequence[bool]],
                seg: Sequence[int]):
        """Masked segmented (sum mod l, group_combine fold) on the device."""
        n = max(len(scalars), len(points))
        segs = np.array(seg, dtype=np.uint32)
        ng = max(len(segs) - 1, 0)
        m = bytes(int(bool(x)) for x in mask) if mask is not None else None
        out_s = ctypes.create_string_buffer(max(ng, 1) * 32)
        out_r = ctypes.create_string_buffer(max(ng, 1) * 32)
        self._call(self._lib.poslo_gpu_segfold, n, _buf(b"".join(scalars)) if scalars else None,
                   _buf(b"".join(points)) if points else None, _buf(m) if m else None,
                   segs.ctypes.data if ng else None, ng, out_s if scalars else None,
                   out_r if points else None)
        rs, rr = out_s.raw, out_r.raw  # ctypes .raw copies the whole buffer per access
        return [(rs[32 * g:32 * g + 32], rr[32 * g:32 * g + 32]) for g in range(ng)]

    # -- SeBVer over a coarse CCD (distiller.cpp:181-233)
    def sebver(self, y: bytes, suite: SuiteConfig, all_msgs, ds: SeedStack, epochs_distilled: int,
               invalid: Sequence, umbrellas: Sequence, valid=None, hashed: Optional[Sequence[int]] = None,
               want: str = "VUI"):
        """invalid: [(epoch, s_le, r)], umbrellas: [(u, s_le, r)], valid: (s_le, r) or None.
        hashed: the epochs to hash (default: every distilled epoch); the C-ABI derives
        seeds and hashes only those. want: the modes to evaluate. Returns dict with
        keys V (list, only when valid given), U, I."""
        eps = range(epochs_distilled) if hashed is None else hashed
        for i in eps:  # a missing epoch is the reference's FormatError, not a KeyError
            if i not in all_msgs:
                raise FormatError(f"messages for epoch {i} missing")
        batches = {i: all_msgs[i] for i in eps}
        pb = PackedBatch(suite.suite, suite.n2, batches, ds)
        cb = pb.cstruct()
        inv = np.array([x[0] for x in invalid], dtype=np.uint32)
        inv_s = b"".join(x[1] for x in invalid)
        inv_r = b"".join(x[2] for x in invalid)
        ui = np.array([x[0] for x in umbrellas], dtype=np.uint32)
        us = b"".join(x[1] for x in umbrellas)
        ur = b"".join(x[2] for x in umbrellas)
        vbit = ctypes.c_uint8(0)
        ubits = ctypes.create_string_buffer(max(len(umbrellas), 1))
        ibits = ctypes.create_string_buffer(max(len(invalid), 1))
        self._call(self._lib.poslo_gpu_sebver, ctypes.byref(cb), _buf(y), suite.n1, suite.n_u,
                   inv.ctypes.data if len(inv) else None, _buf(inv_s) if inv_s else None,
                   _buf(inv_r) if inv_r else None, len(invalid),
                   _buf(valid[0]) if valid else None, _buf(valid[1]) if valid else None,
                   ctypes.byref(vbit) if (valid and "V" in want) else None, ui.ctypes.data if len(ui) else None,
                   _buf(us) if us else None, _buf(ur) if ur else None, len(umbrellas),
                   ubits if "U" in want else None, ibits if "I" in want else None)
        ub, ib = ubits.raw, ibits.raw
        res = {"U": [bool(ub[k]) for k in range(len(umbrellas))],
               "I": [bool(ib[k]) for k in range(len(invalid))]}
        if valid:
            res["V"] = [bool(vbit.value)]
        return res

    # -- group layer (group.cpp), batched on the device
    def commit_check_batch(self, y: bytes, es: Sequence[bytes], ss: Sequence[bytes]) -> List[bytes]:
        n = len(es)
        out = ctypes.create_string_buffer(max(n, 1) * 32)
        self._call(self._lib.poslo_gpu_commit_check, n, _buf(y), _buf(b"".join(es)),
                   _buf(b"".join(ss)), out)
        raw = out.raw
        return [raw[32 * k:32 * k + 32] for k in range(n)]

    def commit_check(self, y: bytes, e: bytes, s: bytes) -> bytes:
        return self.commit_check_batch(y, [e], [s])[0]

    def exp_base(self, s: bytes) -> bytes:
        return self.commit_check(bytes(32), bytes(32), s)

    def scalar_sum(self, scalars: Sequence[bytes]) -> bytes:
        """Sum mod l on the device (rank-ordered fold of shard partials)."""
        out = ctypes.create_string_buffer(32)
        self._call(self._lib.poslo_gpu_scalar_sum, len(scalars),
                   _buf(b"".join(scalars)) if scalars else None, out)
        return out.raw

    def group_check(self, y: bytes, es: Sequence[bytes], ss: Sequence[bytes], rs: Sequence[bytes]):
        """verdict[i] = (commit_check(Y, e_i, s_i) == R_i) (batch_verify.cpp:86)."""
        n = len(es)
        out = ctypes.create_string_buffer(max(n, 1))
        self._call(self._lib.poslo_gpu_group_check, n, _buf(y), _buf(b"".join(es)), _buf(b"".join(ss)),
                   _buf(b"".join(rs)), out)
        raw = out.raw
        return [bool(raw[k]) for k in range(n)]

    def group_fold(self, pts: Sequence[bytes]) -> bytes:
        out = ctypes.create_string_buffer(32)
        self._call(self._lib.poslo_gpu_group_fold, len(pts), _buf(b"".join(pts)) if pts else None,
                   out)
        return out.raw

    def group_combine(self, a: bytes, b: bytes) -> bytes:
        return self.group_fold([a, b])

    def is_valid_point_batch(self, pts: Sequence[bytes]) -> List[bool]:
        n = len(pts)
        out = ctypes.create_string_buffer(max(n, 1))
        self._call(self._lib.poslo_gpu_point_valid, n, _buf(b"".join(pts)) if pts else None, out)
        raw = out.raw
        return [bool(raw[k]) for k in range(n)]

    # -- stage-level parity hooks
    def seed_retrieve(self, suite: int, ds: SeedStack, epochs: Sequence[int]) -> List[bytes]:
        ep = np.array(epochs, dtype=np.uint32)
        out = ctypes.create_string_buffer(max(len(ep), 1) * 16)
        w = ds.serialize()
        self._call(self._lib.poslo_gpu_seed_retrieve, suite, _buf(w), len(w), ds.capacity,
                   ep.ctypes.data if len(ep) else None, len(ep), out)
        raw = out.raw
        return [raw[16 * k:16 * k + 16] for k in range(len(ep))]

    def entry_scalars(self, suite: SuiteConfig, batches, ds: SeedStack) -> List[bytes]:
        pb = PackedBatch(suite.suite, suite.n2, batches, ds)
        out = ctypes.create_string_buffer(max(pb.n_entries, 1) * 32)
        cb = pb.cstruct()
        self._call(self._lib.poslo_gpu_entry_scalars, ctypes.byref(cb), out)
        raw = out.raw
        return [raw[32 * k:32 * k + 32] for k in range(pb.n_entries)]


_default = None
_default_lock = threading.Lock()


def default_verifier() -> Verifier:
    global _default
    with _default_lock:
        if _default is None:
            _default = Verifier(0)
        return _default


def agg_ekeys(suite: SuiteConfig, batches, ds: SeedStack, workers: int):
    """batch_verify.hpp:20-23 — list of (epoch, e~ LE bytes), ascending."""
    return default_verifier().agg_ekeys(suite, batches, ds, workers)[0]


def paver(pk: PoslocPublicKey, batches, s_hat: bytes, r_hat_agg: Optional[bytes], ds: SeedStack,
          workers: int) -> bool:
    """batch_verify.hpp:27-30."""
    return default_verifier().paver(pk, batches, s_hat, r_hat_agg, ds, workers)
