"""World-size-2 gloo tests (CPU) of the multi-rank host logic in
paper_2506_08781_b200/multi_gpu.py: the error agreement that keeps a failing
rank from leaving the others blocked in a collective (every rank raises the
lowest failing rank's error), variable-size gathers, and the epoch / byte /
umbrella cuts. The device paths (partial e-hat all-gather, rank-ordered fold
and check, verdict and umbrella gathers) run in tests/test_gpu_multirank.py."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    from paper_2506_08781_b200 import api
    from paper_2506_08781_b200 import multi_gpu as M
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        # variable-size gather, rank order
        out["var"] = M.all_gather_var(bytes([rank]) * (3 + 5 * rank))
        # no error anywhere: agree returns
        M.agree(None)
        out["ok"] = True
        # rank 1 fails with SeedNotDisclosed(77): every rank raises it
        exc = api.SeedNotDisclosed(77) if rank == 1 else None
        try:
            M.agree(exc)
            out["raised"] = None
        except api.SeedNotDisclosed as e:
            out["raised"] = ("seed", e.epoch)
        # both fail: the lowest rank's error wins on both
        exc = api.FormatError("bad entry") if rank == 0 else api.StateError("later")
        exc.epoch = 5 + rank
        try:
            M.agree(exc)
        except (api.FormatError, api.StateError) as e:
            out["both"] = (type(e).__name__, e.epoch)
        q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_error_agreement_and_gathers_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank in (0, 1):
        r = res[rank]
        assert r["var"] == [b"\x00" * 3, b"\x01" * 8]
        assert r["ok"]
        assert r["raised"] == ("seed", 77)
        assert r["both"] == ("FormatError", 5)


def test_shard_ranges_cover_and_balance():
    from paper_2506_08781_b200 import multi_gpu as M
    for n in (1, 7, 64, 1000):
        for w in (1, 2, 4, 8):
            rs = [M.shard_range(n, w, r) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            assert max(b - a for a, b in rs) - min(b - a for a, b in rs) <= 1
    sizes = list(np.random.default_rng(1).integers(64 * 1024, 1024 * 1024, size=256))
    cuts = [M.shard_by_bytes(sizes, 8, r) for r in range(8)]
    assert cuts[0][0] == 0 and cuts[-1][1] == 256
    loads = [sum(sizes[a:b]) for a, b in cuts]
    assert max(loads) / (sum(sizes) / 8) < 1.1


@pytest.mark.parametrize("first,n,w", [(0, 10, 4), (6, 10, 4), (8, 8, 4), (3, 1, 4), (0, 4096, 1024)])
def test_umbrella_cuts_split_at_multiples_of_w(first, n, w):
    from paper_2506_08781_b200 import multi_gpu as M
    c = M.umbrella_cuts(first, n, w)
    assert c[0] == 0 and c[-1] == n and c == sorted(set(c))
    for a, b in zip(c, c[1:]):  # every piece lies in one umbrella
        assert (first + a) // w == (first + b - 1) // w
