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
        cuts = [0] + list(range((-i0) % w or w, n, w)) + [n]  # k >= 1 with (i0 + k) % w == 0
        verdicts, parts = self.v.distill_coarse(pk, batches, sig_of, cuts)
        has = [any(verdicts[cuts[g]:cuts[g + 1]]) for g in range(len(cuts) - 1)]
        for k in range(n):
            i = i0 + k
            if not verdicts[k]:
                self.invalid.append((i, sig_of[i].s_hat, pk.r_hats[i]))
        self._accumulate(parts, has, [i0 + c for c in cuts[1:]])
        for k in range(n):
            del pk.r_hats[i0 + k]
        if n:
            self.ds = sigs[-1].ds
        self.next_epoch += n

    def _accumulate(self, parts, has, piece_end_epoch):
        """Folds per-piece sums of valid (s, r) into the running aggregates
        (fold_valid, distiller.cpp:45-53) and emits the umbrella records that
        complete (:82-88). One device segfold for every running aggregate:
        group 0 = valid, group 1 + g = the umbrella accumulator after piece g
        (piece 0 continues the incoming accumulator)."""
        w = self.umbrella_width()
        nseg = len(parts)
        sc, pt, bounds = [self.valid_[0]], [self.valid_[1]], [0]
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
        for g in range(nseg):
            acc = folded[1 + g]
            nonempty = has[g] or (g == 0 and self.umb_nonempty)
            end = piece_end_epoch[g]  # epochs distilled after this piece
            if end % w == 0:
                self.umbrellas.append(((end - 1) // w, acc[0], acc[1]))
                self.umb_acc, self.umb_nonempty = (ZERO, IDENTITY), False
            else:
                self.umb_acc, self.umb_nonempty = acc, nonempty

    def distill_epoch_step(self, pk: api.PoslocPublicKey, msgs: Sequence[bytes], sig: api.EpochSignature):
        """distill_epoch (distiller.cpp:60-89) through the single-epoch device
        step (poslo_gpu_distill_step), the route of the C++ drop-in
        (host/distiller_gpu.cpp): same state and errors as distill_epoch."""
        if self.scheme != COARSE:
            raise StateError("coarse distillation on a fine-grained stream")
        if self.next_epoch >= self.suite.n1:
            raise StateError("stream already complete")
        i = self.next_epoch
        if i not in pk.r_hats:
            raise StateError(f"epoch {i} already distilled (commitment gone)")
        if len(msgs) != self.suite.n2:
            raise StateError("every batch must hold exactly n2 entries")
        ok, (valid, umb) = self.v.distill_step(pk, i, msgs, sig, [self.valid_, self.umb_acc])
        if ok:
            self.valid_, self.umb_acc = valid, umb
            self.has_valid = True
            self.umb_nonempty = True
        else:
            self.invalid.append((i, sig.s_hat, pk.r_hats[i]))
        del pk.r_hats[i]
        self.ds = sig.ds
        self.next_epoch += 1
        w = self.umbrella_width()
        if self.next_epoch % w == 0:
            self.umbrellas.append(((self.next_epoch - 1) // w, *self.umb_acc))
            self.umb_acc, self.umb_nonempty = (ZERO, IDENTITY), False

    # -- fine-grained distillation (distiller.cpp:91-129)
    def distill_epoch_fine(self, pk, msgs: Sequence[bytes], sigs):
        self.distill_epochs_fine(pk, [msgs], [sigs])

    def distill_epochs_fine(self, pk, msgs_list, sigs_list):
        """distill_epoch_fine for epochs next_epoch, next_epoch + 1, ... in one batch.
        pk: fine.PoslofPublicKey; sigs_list[k]: the epoch's n2 FineSignatures."""
        if self.scheme != FINE:
            raise StateError("fine distillation on a coarse stream")
        stop, exc = len(msgs_list), None
        for k, (msgs, sigs) in enumerate(zip(msgs_list, sigs_list)):
            if self.next_epoch + k >= self.suite.n1:
                stop, exc = k, StateError("stream already complete")
                break
            if len(msgs) != self.suite.n2 or len(sigs) != self.suite.n2:
                stop, exc = k, StateError("epoch must hold exactly n2 entries and signatures")
                break
            if not sigs[-1].carries_ds():
                stop, exc = k, FormatError("last entry of the epoch must carry ds")
                break
        if stop:
            try:
                self._run_fine(pk, msgs_list[:stop], sigs_list[:stop])
            except (api.SeedNotDisclosed, FormatError) as e:
                bad = getattr(e, "epoch", None)
                if isinstance(e, FormatError) and bad is not None:
                    bad = self.next_epoch + bad // self.suite.n2  # entry position -> epoch
                done = (bad - self.next_epoch) if bad is not None else 0
                if 0 < done < stop:
                    self._run_fine(pk, msgs_list[:done], sigs_list[:done])
                raise
        if exc is not None:
            raise exc

    def _run_fine(self, pk, msgs_list, sigs_list):
        from . import fine as F
        n, i0, n2, w = len(msgs_list), self.next_epoch, self.suite.n2, self.umbrella_width()
        msgs = [m for ms in msgs_list for m in ms]
        sigs = [sg for ss in sigs_list for sg in ss]
        # entries carrying ds derive x from the epoch's NEW stack (its last signature's ds)
        derive = [(t // n2, t % n2) if sg.carries_ds() else None for t, sg in enumerate(sigs)]
        fb = F.FineBatch(self.suite.suite, msgs, [None if sg.carries_ds() else sg.tail for sg in sigs], derive,
                         [i0 + k for k in range(n)], [ss[-1].tail for ss in sigs_list], None, self.suite.depth())
        verdicts = F.fine_verify(self.v, fb, pk.y, [sg.s for sg in sigs], [sg.r for sg in sigs])
        cuts = [0] + [k * n2 for k in range((-i0) % w or w, n, w)] + [n * n2]
        parts = self.v.segfold([sg.s for sg in sigs], [sg.r for sg in sigs], verdicts, cuts)
        has = [any(verdicts[cuts[g]:cuts[g + 1]]) for g in range(len(cuts) - 1)]
        for t, ok in enumerate(verdicts):
            if not ok:
                self.invalid.append((i0 * n2 + t, sigs[t].s, sigs[t].r))
        self._accumulate(parts, has, [i0 + c // n2 for c in cuts[1:]])
        if n:
            self.ds = sigs_list[-1][-1].tail
        self.next_epoch += n

    def finalize(self):
        """distiller.cpp:131-138"""
        if self.umb_nonempty:
            self.umbrellas.append(((self.next_epoch - 1) // self.umbrella_width(), *self.umb_acc))
            self.umb_acc, self.umb_nonempty = (ZERO, IDENTITY), False

    # -- SeBVer (distiller.cpp:156-233), on the device
    def sebver(self, y: bytes, all_msgs: Dict[int, Sequence[bytes]], mode: str) -> List[bool]:
        if mode not in ("V", "U", "I"):
            raise StateError("unknown mode")
        if mode == "V" and not self.has_valid:
            raise StateError("mode V needs a valid aggregate")
        if self.scheme == FINE:
            return self._sebver_fine(y, all_msgs, mode)
        w = self.umbrella_width()
        bad = {i for i, _, _ in self.invalid}
        # the groups SeBVer checks, in its order, with the epochs each one reads
        # (collect_epochs, :140-154, or the mode-I lookup, :208-210) and hashes
        # (verify_range skips invalid epochs, :161-162)
        if mode == "I":
            groups = [([i], [i]) for i, _, _ in self.invalid]
        elif mode == "V":
            rng = list(range(self.next_epoch))
            groups = [(rng, [i for i in rng if i not in bad])]
        else:
            groups = []
            for u, _, _ in self.umbrellas:
                rng = list(range(u * w, min((u + 1) * w, self.next_epoch)))
                groups.append((rng, [i for i in rng if i not in bad]))
        # the reference raises at the first group whose messages are missing, after
        # hashing (and raising the hashing errors of) every group before it
        hashed, missing, live = set(), None, len(groups)
        for k, (read, hash_) in enumerate(groups):
            for i in read:
                if i not in all_msgs:
                    missing = FormatError("messages for invalid epoch missing" if mode == "I"
                                          else f"messages for epoch {i} missing")
                    break
                if mode != "I" and len(all_msgs[i]) != self.suite.n2:
                    missing = FormatError("epoch batch size mismatch")
                    break
            if missing is not None:
                live = k
                break
            hashed.update(hash_)
        if missing is not None and live == 0:
            raise missing
        res = self.v.sebver(y, self.suite, all_msgs, self.ds, self.next_epoch,
                            self.invalid[:live] if mode == "I" else self.invalid,
                            self.umbrellas[:live] if mode == "U" else [],
                            self.valid_ if mode == "V" else None, hashed=sorted(hashed), want=mode)
        if missing is not None:
            raise missing
        return res[mode]

    def _sebver_fine(self, y, all_msgs, mode):
        from . import fine as F
        n2, w = self.suite.n2, self.umbrella_width()
        bad = {t for t, _, _ in self.invalid}
        if mode == "I":
            msgs, derive, eps = [], [], []
            for t, _, _ in self.invalid:
                i, j = t // n2, t % n2
                if i not in all_msgs or len(all_msgs[i]) <= j:
                    raise FormatError("message for invalid entry missing")
                msgs.append(all_msgs[i][j])
                eps.append(i)
            slots = sorted(set(eps))
            derive = [(slots.index(t // n2), t % n2) for t, _, _ in self.invalid]
            if not msgs:
                return []
            fb = F.FineBatch(self.suite.suite, msgs, [None] * len(msgs), derive, slots, None, self.ds,
                             self.suite.depth())
            return F.fine_verify(self.v, fb, y, [s for _, s, _ in self.invalid], [r for _, _, r in self.invalid])
        ranges = [(0, self.next_epoch, self.valid_)] if mode == "V" else \
            [(u * w, (u + 1) * w, (sv, rv)) for u, sv, rv in self.umbrellas]
        ranges = [(lo, min(hi, self.next_epoch), sig) for lo, hi, sig in ranges]
        epochs = sorted({i for lo, hi, _ in ranges for i in range(lo, hi)})
        for i in epochs:  # collect_epochs (:140-154)
            if i not in all_msgs:
                raise FormatError(f"messages for epoch {i} missing")
            if len(all_msgs[i]) != n2:
                raise FormatError("epoch batch size mismatch")
        pos = {i: k for k, i in enumerate(epochs)}
        msgs = [m for i in epochs for m in all_msgs[i]]
        derive = [(k, j) for k in range(len(epochs)) for j in range(n2)]
        es = []
        if msgs:
            fb = F.FineBatch(self.suite.suite, msgs, [None] * len(msgs), derive, epochs, None, self.ds,
                             self.suite.depth())
            es, _ = F.fine_scalars(self.v, fb)
        # e-sum per range over its non-invalid entries: one masked segfold over concatenated items
        items, mask, bounds = [], [], [0]
        for lo, hi, _ in ranges:
            for i in range(lo, hi):
                for j in range(n2):
                    items.append(es[pos[i] * n2 + j])
                    mask.append((i * n2 + j) not in bad)
            bounds.append(len(items))
        sums = self.v.segfold(items, [], mask, bounds) if ranges else []
        return self.v.group_check(y, [s for s, _ in sums], [sig[0] for _, _, sig in ranges],
                                  [sig[1] for _, _, sig in ranges]) if ranges else []

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
