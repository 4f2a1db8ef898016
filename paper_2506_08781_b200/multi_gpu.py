"""Multi-rank sharding of the batch verifier: one process per
GPU, torch.distributed for the plumbing (NCCL over NVLink on the box; gloo
works too, e.g. several ranks sharing one device in tests).

The log is sharded by contiguous, epoch-aligned entry ranges (rank r owns
epochs shard_range(n1, world, r)); each rank hashes and checks its own epochs
on its GPU. The only data exchanges are the ones SURVEY §8e names:
  coarse PAVer   the 32-byte partial e-hat of every rank, all-gathered straight
                 from device memory, folded mod l in rank order and checked
                 once on rank 0 (batch_verify.cpp:83-86);
  per-epoch      verdict bytes gathered to every rank in epoch order;
  distillation   verdicts -> the ascending invalid-epoch list; umbrella pieces
                 (sum of valid s-hat, e~ and the R-hat fold) of umbrellas a
                 shard cut splits, folded in rank order on rank 0
                 (distiller.cpp:45-53, 82-88), then one check per umbrella
                 (SeBVer mode U, :156-179).
NCCL all-reduce is never used: there is no mod-l operator and limb-wise sums
drop carries. Before every exchange of results the ranks exchange a status
record, so an error on one rank (SeedNotDisclosed, FormatError, ...) is
raised on every rank — the lowest failing rank's error, i.e. the lowest
epoch's — instead of leaving the others blocked in a collective.
"""
from __future__ import annotations

import ctypes
import struct
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np
import torch
import torch.distributed as dist

from . import api


def shard_range(n_epochs: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous epoch range [lo, hi) of `rank`; sizes differ by at most 1."""
    base, extra = divmod(n_epochs, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def shard_by_bytes(epoch_bytes: Sequence[int], world: int, rank: int) -> Tuple[int, int]:
    """Epoch-aligned cut by a byte prefix sum (variable-length logs, config 4):
    each rank gets ~1/world of the bytes (hash work scales with bytes)."""
    total = sum(epoch_bytes)
    acc, cuts = 0, [0]
    target = [total * (r + 1) / world for r in range(world)]
    t = 0
    for i, b in enumerate(epoch_bytes):
        acc += b
        while t < world - 1 and acc >= target[t]:
            cuts.append(i + 1)
            t += 1
    while len(cuts) < world:
        cuts.append(len(epoch_bytes))
    cuts.append(len(epoch_bytes))
    return cuts[rank], cuts[rank + 1]


def _device_for(group):
    backend = dist.get_backend(group)
    return torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")


def all_gather_bytes(blob: bytes, group=None) -> List[bytes]:
    """All-gather one fixed-size byte string per rank, returned in rank order."""
    world = dist.get_world_size(group)
    dev = _device_for(group)
    t = torch.frombuffer(bytearray(blob), dtype=torch.uint8).to(dev) if blob else torch.zeros(0, dtype=torch.uint8,
                                                                                              device=dev)
    out = torch.empty(world * len(blob), dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(out, t, group=group)
    raw = out.cpu().numpy().tobytes()
    n = len(blob)
    return [raw[r * n:(r + 1) * n] for r in range(world)]


def all_gather_var(blob: bytes, group=None) -> List[bytes]:
    """All-gather byte strings of differing lengths (padded to the longest)."""
    sizes = [struct.unpack("<Q", x)[0] for x in all_gather_bytes(struct.pack("<Q", len(blob)), group)]
    width = max(sizes) if sizes else 0
    parts = all_gather_bytes(blob + bytes(width - len(blob)), group) if width else [b""] * len(sizes)
    return [p[:s] for p, s in zip(parts, sizes)]


# ---------------------------------------------------------------- error agreement
_KIND = {api.FormatError: 1, api.StateError: 2, api.SeedNotDisclosed: 3, ValueError: 5}


def _status(exc: Optional[BaseException]) -> bytes:
    if exc is None:
        return bytes(128)
    kind = next((k for cls, k in _KIND.items() if isinstance(exc, cls)), 4)
    epoch = int(getattr(exc, "epoch", 0) or 0)
    msg = str(exc).encode(errors="replace")[:119]
    return struct.pack("<BI", kind, epoch & 0xFFFFFFFF) + bytes([len(msg)]) + msg + bytes(122 - len(msg))


def agree(exc: Optional[BaseException], group=None):
    """Every rank contributes its status; if any rank failed, every rank raises
    the lowest failing rank's error (ranks hold ascending epochs)."""
    recs = all_gather_bytes(_status(exc), group)
    for r, rec in enumerate(recs):
        kind = rec[0]
        if not kind:
            continue
        if r == dist.get_rank(group) and exc is not None:
            raise exc
        epoch = struct.unpack("<I", rec[1:5])[0]
        msg = rec[6:6 + rec[5]].decode(errors="replace")
        if kind == 3:
            raise api.SeedNotDisclosed(epoch)
        cls = {1: api.FormatError, 2: api.StateError, 5: ValueError}.get(kind, api.DeviceError)
        e = cls(f"rank {r}: {msg}")
        e.epoch = epoch
        raise e


def _guard(fn):
    try:
        return fn(), None
    except (api.FormatError, api.StateError, api.SeedNotDisclosed, api.DeviceError, ValueError) as e:
        return None, e


def _root(group) -> int:
    return dist.get_global_rank(group, 0) if group is not None else 0


# ---------------------------------------------------------------- coarse PAVer
class ShardedPaver:
    """Coarse PAVer over a sharded log: partial e-hat into device memory, ONE
    all-gather of (partial, status) per rank (NCCL: device to device, no host
    hop), the rank-ordered fold mod l and ONE check on rank 0, whose verdict
    every rank receives. Rank 0 queues the e-hat-independent half of the check
    (alpha^s-hat, the R-hat operand) on a side stream before hashing, so after
    the all-gather only the fold and the Y^e-hat half remain. Buffers are
    allocated once and reused across steps."""

    REC = 64  # bytes per rank in the gather: partial e-hat (32) | status (1) | pad

    def __init__(self, v: api.Verifier, group=None):
        self.v, self.group = v, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.nccl = dist.get_backend(group) == "nccl"
        dev = torch.device("cuda", torch.cuda.current_device())
        self.rec = torch.zeros(self.REC, dtype=torch.uint8, device=dev)
        self.recs = torch.zeros(self.REC * self.world, dtype=torch.uint8, device=dev if self.nccl else "cpu")
        self.flag = torch.zeros(1, dtype=torch.uint8, device=dev if self.nccl else "cpu")

    def __call__(self, cb, y: bytes, s_hat: bytes, r_hat: bytes) -> bool:
        prep_exc = None
        if self.rank == 0:  # overlaps this rank's hashing
            _, prep_exc = _guard(lambda: self.v.combine_check_prepare(y, s_hat, r_hat))
        _, exc = _guard(lambda: self.v.agg_ekeys_partial(cb, self.rec.data_ptr()))
        if exc is not None:
            self.rec[32] = 1
        else:
            self.rec[32] = 0
        if self.nccl:
            dist.all_gather_into_tensor(self.recs, self.rec, group=self.group)
        else:
            dist.all_gather_into_tensor(self.recs, self.rec.cpu(), group=self.group)
        ok, exc0 = None, None
        if self.rank == 0:
            host = self.recs.cpu().numpy().reshape(self.world, self.REC)  # one small D2H: statuses + partials
            if host[:, 32].any():
                res = 2
            else:
                parts = host[:, :32].tobytes()
                ok, exc0 = _guard(lambda: self.v.combine_check(parts, y, s_hat, r_hat))
                if exc0 is None and prep_exc is not None:
                    exc0 = prep_exc
                res = 2 if exc0 is not None else (1 if ok else 0)
            self.flag[0] = res
        dist.broadcast(self.flag, src=_root(self.group), group=self.group)
        res = int(self.flag.item())
        if res == 2:  # a rank failed while hashing, or rank 0's check raised: every rank raises the same
            agree(exc if exc is not None else (exc0 if self.rank == 0 else None), self.group)
        return res == 1


def sharded_paver(v: api.Verifier, cb, y: bytes, s_hat: bytes, r_hat: bytes, group=None) -> bool:
    """One-shot form of ShardedPaver: every rank passes ITS shard's batch."""
    return ShardedPaver(v, group)(cb, y, s_hat, r_hat)


def sharded_e_tilde(v: api.Verifier, cb, group=None) -> List[bytes]:
    """agg_ekeys over a sharded log: every rank gets every e~ in epoch order."""
    n = cb.n_epochs
    out = ctypes.create_string_buffer(max(n, 1) * 32)
    _, exc = _guard(lambda: v._call(v._lib.poslo_gpu_agg_ekeys, ctypes.byref(cb), out, None))
    agree(exc, group)
    raw = b"".join(all_gather_var(out.raw[:32 * n], group))
    return [raw[32 * k:32 * k + 32] for k in range(len(raw) // 32)]


# ---------------------------------------------------------------- per-epoch verdicts
def sharded_epoch_verdicts(v: api.Verifier, cb, y: bytes, s_hats, r_hats, group=None) -> bytes:
    """Per-epoch verdicts: each rank checks its own epochs (no exchange) and the
    verdict bytes are gathered to every rank in epoch order. s_hats / r_hats:
    host bytes, or device pointers for a device-resident batch."""
    n = cb.n_epochs
    verd = ctypes.create_string_buffer(max(n, 1))
    args = [ctypes.c_void_p(x) if isinstance(x, int) else api._buf(x) for x in (s_hats, r_hats)]
    _, exc = _guard(lambda: v._call(v._lib.poslo_gpu_epoch_verify, ctypes.byref(cb), api._buf(y), *args, verd,
                                    None))
    agree(exc, group)
    return b"".join(all_gather_var(verd.raw[:n], group))


# ---------------------------------------------------------------- distillation
def umbrella_cuts(first_epoch: int, n_epochs: int, w: int) -> List[int]:
    """Batch positions where this shard's epochs cross an umbrella boundary."""
    first = (-first_epoch) % w or w  # smallest k >= 1 with (first_epoch + k) % w == 0
    return [0] + list(range(first, n_epochs, w)) + [n_epochs]


def sharded_distill(v: api.Verifier, cb, first_epoch: int, y: bytes, s_hats, r_hats, w: int, group=None,
                    check_umbrellas: bool = True) -> Optional[Dict]:
    """Coarse distillation of a sharded log (distill_epoch over every epoch,
    distiller.cpp:60-89): on rank 0 returns {"verdicts": bytes (epoch order),
    "invalid": ascending invalid epochs, "umbrellas": [(u, s, R, e)] with the
    valid epochs of umbrella u folded across shards, "u_bits": SeBVer mode U
    (one commit_check per umbrella)}; None on other ranks."""
    n = cb.n_epochs
    cuts = umbrella_cuts(first_epoch, n, w)
    seg = np.array(cuts, dtype=np.uint32)
    ng = len(cuts) - 1
    verd = ctypes.create_string_buffer(max(n, 1))
    out_s, out_r, out_e = (ctypes.create_string_buffer(max(ng, 1) * 32) for _ in range(3))
    args = [ctypes.c_void_p(x) if isinstance(x, int) else api._buf(x) for x in (s_hats, r_hats)]
    _, exc = _guard(lambda: v._call(v._lib.poslo_gpu_distill_coarse_ex, ctypes.byref(cb), api._buf(y), *args,
                                    ctypes.c_void_p(seg.ctypes.data), ng, verd, out_s, out_r, out_e))
    agree(exc, group)
    # pieces: (umbrella index, s, R, e) of this shard, in epoch order
    rs, rr, re_ = out_s.raw, out_r.raw, out_e.raw  # one copy each (.raw copies per access)
    pieces = b"".join(struct.pack("<I", (first_epoch + cuts[g]) // w) + rs[32 * g:32 * g + 32] +
                      rr[32 * g:32 * g + 32] + re_[32 * g:32 * g + 32] for g in range(ng))
    verd_all = all_gather_var(verd.raw[:n], group)
    piece_all = all_gather_var(pieces, group)
    if dist.get_rank(group) != 0:
        return None
    verdicts = b"".join(verd_all)
    # rank 0 holds the first shard
    invalid = (np.flatnonzero(np.frombuffer(verdicts, dtype=np.uint8) == 0) + first_epoch).tolist()
    # fold the pieces of each umbrella in rank order (one segmented fold on the device)
    recs = [(struct.unpack("<I", p[k:k + 4])[0], p[k + 4:k + 36], p[k + 36:k + 68], p[k + 68:k + 100])
            for p in piece_all for k in range(0, len(p), 100)]
    us = sorted({u for u, _, _, _ in recs})
    bounds, sc, pt, es = [0], [], [], []
    for u in us:
        for uu, s_, r_, e_ in recs:
            if uu == u:
                sc.append(s_)
                pt.append(r_)
                es.append(e_)
        bounds.append(len(sc))
    folded = v.segfold(sc, pt, None, bounds)
    efold = v.segfold(es, [], None, bounds)
    umbrellas = [(u, folded[k][0], folded[k][1], efold[k][0]) for k, u in enumerate(us)]
    u_bits = v.group_check(y, [e for _, _, _, e in umbrellas], [s for _, s, _, _ in umbrellas],
                           [r for _, _, r, _ in umbrellas]) if (check_umbrellas and umbrellas) else []
    return {"verdicts": verdicts, "invalid": invalid, "umbrellas": umbrellas, "u_bits": u_bits}
