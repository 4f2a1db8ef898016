"""Verify-then-compress pipeline on the GPU: ColdCryptoData (CCD), coarse scheme.

Mirrors the reference's distiller (include/poslo/distiller.hpp:31-98,
src/distiller.cpp). `distill_epochs` is `distill_epoch` (distiller.cpp:60-89)
applied to a run of consecutive epochs in ONE device call
(poslo_gpu_distill_coarse): per-epoch verdicts, each epoch verified with its
own signature's seed stack, and the valid epochs' (s-hat, R-hat) folded per
umbrella piece on the device; the host only keeps the running CCD state.
Results, state and raised errors are those of calling distill_epoch once per
epoch: on an error at epoch e the epochs before e are committed first, as the
reference (which distils epoch by epoch) leaves them.

The CCD wire format (serialize / deserialize, CRC-32 trailer) follows
distiller.cpp:235-304 byte for byte. SeBVer (distiller.cpp:181-233) runs on
the device via Verifier.sebver.
"""
import struct
import zlib
from typing import Dict, List, Optional, Sequence, Tuple

from . import api
from .api import FormatError, SeedStack, StateError, SuiteConfig

IDENTITY = bytes(32)
ZERO = bytes(32)  # scalar 0 (LE)
COARSE, FINE = ord("C"), ord("F")


class ColdCryptoData:
    def __init__(self, scheme: int = COARSE, suite: Optional[SuiteConfig] = None,
                 verifier: Optional[api.Verifier] = None):
        self.scheme = scheme
        self.suite = suite or SuiteConfig()
        if suite is not None:
            suite.validate()
        self.v = verifier or api.default_verifier()
        self.next_epoch = 0
        self.has_valid = False
        self.valid_ = (ZERO, IDENTITY)      # (s LE, r)
        self.umb_acc = (ZERO, IDENTITY)
        self.umb_nonempty = False
        self.umbrellas: List[Tuple[int, bytes, bytes]] = []   # (index, s LE, r)
        self.invalid: List[Tuple[int, bytes, bytes]] = []     # (epoch, s LE, r)
        self.ds = SeedStack(self.suite.depth() if suite is not None else 0)

    # -- accessors (distiller.hpp:37-47)
    def epochs_distilled(self) -> int:
        return self.next_epoch

    def valid(self):
        if not self.has_valid:
            raise StateError("no valid aggregate distilled yet")
        return self.valid_

    def umbrella_width(self) -> int:
        return self.suite.n1 // self.suite.n_u

    # -- distillation
    def distill_epoch(self, pk: api.PoslocPublicKey, msgs: Sequence[bytes], sig: api.EpochSignature):
        self.distill_epochs(pk, [msgs], [sig])

    def distill_epochs(self, pk: api.PoslocPublicKey, msgs_list: Sequence[Sequence[bytes]],
                       sigs: Sequence[api.EpochSignature]):
        """distill_epoch for epochs next_epoch, next_epoch + 1, ... in one batch."""
        if self.scheme != COARSE:
            raise StateError("coarse distillation on a fine-grained stream")
        # host-side checks of distill_epoch/aver, in stream order (distiller.cpp:63-71,
        # poslo_c.cpp:195-197); the first failing epoch ends the run
        stop, exc = len(msgs_list), None
        for k, msgs in enumerate(msgs_list):
            i = self.next_epoch + k
            if i >= self.suite.n1:
                stop, exc = k, StateError("stream already complete")
                break
            if i not in pk.r_hats:
                stop, exc = k, StateError(f"epoch {i} already distilled (commitment gone)")
                break
            if len(msgs) != self.suite.n2:
                stop, exc = k, StateError("every batch must hold exactly n2 entries")
                break
        if stop:
            try:
                self._run(pk, msgs_list[:stop], sigs[:stop])
            except (api.SeedNotDisclosed, FormatError) as e:
                bad = getattr(e, "epoch", None)
                done = (bad - self.next_epoch) if bad is not None else 0
                if 0 < done < stop:  # commit the epochs before the failing one, then raise
                    self._run(pk, msgs_list[:done], sigs[:done])
                raise
        if exc is not None:
            raise exc

    def _run(self, pk, msgs_list, sigs):
        n, i0, w = len(msgs_list), self.next_epoch, self.umbrella_width()
        batches = {i0 + k: list(m) for k, m in enumerate(msgs_list)}
        sig_of = {i0 + k: s for k, s in enumerate(sigs)}
        # umbrella pieces: cut where an epoch index is a multiple of w
        seg = [0] + [k for k in range(1, n) if (i0 + k) % w == 0] + [n]
        verdicts, parts = self.v.distill_coarse(pk, batches, sig_of, seg)
        nseg = len(seg) - 1
        has = [any(verdicts[seg[g]:seg[g + 1]]) for g in range(nseg)]
        # one device fold for the running aggregates: group 0 = valid, group 1 + g = umbrella
        # accumulator after piece g (piece 0 continues the incoming accumulator)
        sc, pt, bounds = [], [], [0]
        sc.append(self.valid_[0]); pt.append(self.valid_[1])
        for g in range(nseg):
            if has[g]:
                sc.append(parts[g][0]); pt.append(parts[g][1])
        bounds.append(len(sc))
        for g in range(nseg):
            if g == 0:
                sc.append(self.umb_acc[0]); pt.append(self.umb_acc[1])
            if has[g]:
                sc.append(parts[g][0]); pt.append(parts[g][1])
            bounds.append(len(sc))
        folded = self.v.segfold(sc, pt, None, bounds)
        if any(has):
            self.valid_ = folded[0]
            self.has_valid = True
        for k in range(n):
            i = i0 + k
            if not verdicts[k]:
                self.invalid.append((i, sig_of[i].s_hat, pk.r_hats[i]))
        for g in range(nseg):
            acc = folded[1 + g]
            nonempty = has[g] or (g == 0 and self.umb_nonempty)
            end = i0 + seg[g + 1]  # epochs distilled after this piece
            if end % w == 0:
                self.umbrellas.append(((end - 1) // w, acc[0], acc[1]))
                self.umb_acc, self.umb_nonempty = (ZERO, IDENTITY), False
            else:
                self.umb_acc, self.umb_nonempty = acc, nonempty
        for k in range(n):
            del pk.r_hats[i0 + k]
        if n:
            self.ds = sigs[-1].ds
        self.next_epoch += n

    def finalize(self):
        """distiller.cpp:131-138"""
        if self.umb_nonempty:
            self.umbrellas.append(((self.next_epoch - 1) // self.umbrella_width(), *self.umb_acc))
            self.umb_acc, self.umb_nonempty = (ZERO, IDENTITY), False

    # -- SeBVer (distiller.cpp:181-233), on the device
    def sebver(self, y: bytes, all_msgs: Dict[int, Sequence[bytes]], mode: str) -> List[bool]:
        if self.scheme != COARSE:
            raise StateError("fine-grained SeBVer is not part of the GPU path")
        if mode == "V" and not self.has_valid:
            raise StateError("mode V needs a valid aggregate")
        for i in range(self.next_epoch):
            if i not in all_msgs:
                raise FormatError(f"messages for epoch {i} missing")
            if len(all_msgs[i]) != self.suite.n2:
                raise FormatError("epoch batch size mismatch")
        res = self.v.sebver(y, self.suite, all_msgs, self.ds, self.next_epoch, self.invalid,
                            self.umbrellas if mode == "U" else [],
                            self.valid_ if mode == "V" else None)
        return res[mode]

    # -- wire format (distiller.cpp:235-304)
    def serialize(self) -> bytes:
        s = self.suite
        out = bytearray(b"PCCD") + bytes([self.scheme, s.suite])
        out += struct.pack(">IIII", s.n1, s.n2, s.n_u, self.next_epoch)
        out += b"\x01" if self.has_valid else b"\x00"
        out += self.valid_[0][::-1] + self.valid_[1]
        out += struct.pack(">I", len(self.umbrellas))
        for u, sv, rv in self.umbrellas:
            out += struct.pack(">I", u) + sv[::-1] + rv
        out += struct.pack(">I", len(self.invalid))
        for i, sv, rv in self.invalid:
            out += struct.pack(">I", i) + sv[::-1] + rv
        out += self.ds.serialize()
        out += struct.pack(">I", zlib.crc32(bytes(out)) & 0xFFFFFFFF)
        return bytes(out)

    @staticmethod
    def deserialize(b: bytes, verifier: Optional[api.Verifier] = None) -> "ColdCryptoData":
        if len(b) < 4:
            raise FormatError("truncated CCD")
        if struct.unpack(">I", b[-4:])[0] != zlib.crc32(b[:-4]) & 0xFFFFFFFF:
            raise FormatError("CCD checksum mismatch")
        body, o = b[:-4], 0

        def take(k):
            nonlocal o
            if len(body) - o < k:
                raise FormatError("truncated input")
            o += k
            return body[o - k:o]

        if take(4) != b"PCCD":
            raise FormatError("bad magic, expected PCCD")
        ccd = ColdCryptoData.__new__(ColdCryptoData)
        ccd.v = verifier or api.default_verifier()
        ccd.scheme = take(1)[0]
        if ccd.scheme not in (COARSE, FINE):
            raise FormatError("bad CCD scheme byte")
        suite_id = take(1)[0]
        n1, n2, n_u, nxt = struct.unpack(">IIII", take(16))
        ccd.suite = SuiteConfig(suite_id, n1, n2, n_u)
        ccd.suite.validate()
        ccd.next_epoch = nxt
        flag = take(1)[0]
        if flag > 1:
            raise FormatError("bad valid-aggregate flag")
        ccd.has_valid = flag == 1
        pts = []

        def pair():
            s = api.scalar_from_be(take(32))
            r = bytes(take(32))
            pts.append(r)
            return s, r

        ccd.valid_ = pair()
        ccd.umbrellas = []
        for _ in range(struct.unpack(">I", take(4))[0]):
            u = struct.unpack(">I", take(4))[0]
            ccd.umbrellas.append((u, *pair()))
        ccd.invalid = []
        for _ in range(struct.unpack(">I", take(4))[0]):
            i = struct.unpack(">I", take(4))[0]
            ccd.invalid.append((i, *pair()))
        if not all(ccd.v.is_valid_point_batch(pts)):  # GroupElement::from_bytes, before the ds
            raise FormatError("invalid group element encoding")
        ccd.ds, used = SeedStack.deserialize(body, ccd.suite.depth(), o)
        o += used
        if o != len(body):
            raise FormatError("trailing bytes")
        ccd.umb_acc, ccd.umb_nonempty = (ZERO, IDENTITY), False
        return ccd
