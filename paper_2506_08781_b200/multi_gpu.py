"""Multi-GPU sharding of the batch verifier.

One process per GPU. The log is sharded by contiguous, epoch-aligned entry
ranges; each rank runs stages 0-2 on its own epochs and produces a partial
e-hat (32 bytes). Coarse mode needs ONE exchange: an all-gather of the
partials (NCCL over NVLink on the box; any torch.distributed backend works),
then a rank-ordered fold mod l and a single group check. NCCL all-reduce is
never used: there is no mod-l reduction operator and limb-wise sums drop
carries. Per-epoch verdicts need no exchange except gathering the verdict
bits to rank 0.

`backend` is anything with agg_ekeys_packed / scalar_sum / group_check: the
Verifier (device) in production; tests/test_multi_gloo.py drives the same
host logic on CPU with world_size 2 over gloo.
"""
from __future__ import annotations

from typing import Sequence, Tuple

import torch
import torch.distributed as dist


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


def all_gather_bytes(blob: bytes, group=None) -> list:
    """All-gather one fixed-size byte string per rank, returned in rank order."""
    world = dist.get_world_size(group)
    dev = _device_for(group)
    t = torch.frombuffer(bytearray(blob), dtype=torch.uint8).to(dev)
    out = torch.empty(world * len(blob), dtype=torch.uint8, device=dev)
    dist.all_gather_into_tensor(out, t, group=group)
    raw = out.cpu().numpy().tobytes()
    n = len(blob)
    return [raw[r * n:(r + 1) * n] for r in range(world)]


def sharded_paver(backend, packed_shard, y: bytes, s_hat: bytes, r_hat: bytes, group=None) -> bool:
    """Coarse PAVer over a sharded log: every rank passes ITS shard; all ranks
    return the same verdict (broadcast from rank 0)."""
    _, e_part = backend.agg_ekeys_packed(packed_shard)
    parts = all_gather_bytes(e_part, group)
    verdict = torch.zeros(1, dtype=torch.uint8, device=_device_for(group))
    if dist.get_rank(group) == 0:
        e_hat = backend.scalar_sum(parts)          # rank-ordered fold mod l on the device
        verdict[0] = int(backend.group_check(y, [e_hat], [s_hat], [r_hat])[0])
    dist.broadcast(verdict, src=0, group=group)
    return bool(verdict.item())


def sharded_epoch_verdicts(backend, pk, shard_batches, s_hats, ds, group=None) -> list:
    """Per-epoch verdicts: each rank checks its own epochs; verdict bits are
    gathered to every rank in epoch order (ranks hold ascending shards)."""
    local = backend.epoch_verify(pk, shard_batches, s_hats, ds)
    world = dist.get_world_size(group)
    n = torch.tensor([len(local)], dtype=torch.int64, device=_device_for(group))
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    width = int(max(s.item() for s in sizes))
    blob = bytes(int(x) for x in local) + bytes(width - len(local))
    parts = all_gather_bytes(blob, group)
    out = []
    for r, p in enumerate(parts):
        out += [bool(b) for b in p[:int(sizes[r].item())]]
    return out
