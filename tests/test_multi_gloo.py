"""World-size-2 gloo test of the multi-GPU host logic (paper_2506_08781_b200/
multi_gpu.py): epoch sharding, the all-gather of partial e-hat, the
rank-ordered fold and the single check, and per-epoch verdict gathering.
The compute backend here is the CPU oracle (test infrastructure) standing in
for the device Verifier, so the plumbing is exercised without a GPU. CPU only."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from conftest import load_golden
from golden_util import Stream


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


class OracleBackend:
    """Oracle stand-in with the Verifier's multi-GPU surface."""

    def __init__(self, suite, ds, cap, n2):
        from oracle import oracle as O
        self.O, self.suite, self.ds, self.cap, self.n2 = O, suite, ds, cap, n2

    def agg_ekeys_packed(self, shard):
        epochs, batches = shard
        flat = [m for i in epochs for m in batches[i]]
        offs = np.zeros(len(flat) + 1, dtype=np.uint64)
        np.cumsum([len(m) for m in flat], out=offs[1:])
        starts = np.arange(len(epochs) + 1, dtype=np.uint64) * self.n2
        rc, _, et = self.O.agg_ekeys_packed(self.suite, b"".join(flat), offs, 0, epochs, starts, self.ds,
                                            self.cap)
        assert rc == 0
        return list(zip(epochs, et)), self.O.sum_scalars(et)

    def scalar_sum(self, parts):
        return self.O.sum_scalars(parts)

    def group_check(self, y, es, ss, rs):
        R = self.O.ristretto
        return [R.commit_check(y, e, s) == r for e, s, r in zip(es, ss, rs)]

    def epoch_verify(self, pk, batches, s_hats, ds):
        R = self.O.ristretto
        parts, _ = self.agg_ekeys_packed((sorted(batches), batches))
        return [R.commit_check(pk.y, e, s_hats[i]) == pk.r_hats[i] for i, e in parts]


def _worker(rank, world, port, name, q):
    import torch.distributed as dist
    from paper_2506_08781_b200 import multi_gpu as M
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        st = Stream(load_golden(name))
        be = OracleBackend(st.suite, st.ds, st.depth, st.n2)
        lo, hi = M.shard_range(st.n1, world, rank)
        shard = (list(range(lo, hi)), {i: st.batches[i] for i in range(lo, hi)})
        ok = M.sharded_paver(be, shard, st.pk.y, st.s_hat, st.r_hat_agg)
        s_hats = {i: st.sigs[i].s_hat_le for i in range(lo, hi)}
        verdicts = M.sharded_epoch_verdicts(be, st.pk, shard[1], s_hats, None)
        q.put((rank, ok, verdicts))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["stream_s1_tamper.json", "stream_s1_clean_big.json"])
def test_sharded_paver_gloo_world2(name):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    g = load_golden(name)
    for rank, ok, verdicts in res:
        assert ok == bool(g["paver"])
        assert [int(v) for v in verdicts] == g["epoch_verdicts"]


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
