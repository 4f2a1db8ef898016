"""Multi-rank determinism gate on the DEVICE ("outputs must be
byte-identical at G = 1, 2, 4, 8"): the same multi_gpu.py code runs at world
size 1, 2 and 4 (gloo, all ranks on cuda:0 — the box has one GPU; NCCL needs
one GPU per rank), each rank verifying its epoch shard with the device Verifier,
and every gathered output must equal the world-1 output byte for byte:

  config 2 shape (coarse PAVer, n2 = 256): every e~, the folded e-hat, the verdict;
  config 3 shape (per-epoch, n2 = 1024, 16 tampered entries): the verdict bitmap;
  config 5 shape (distillation, n2 = 1024, 16 tampered entries, w = 64): the
      ascending invalid-epoch list, every umbrella's folded (s-hat, R-hat, e-sum)
      across the shard cut, and the SeBVer mode-U bits.

Each at 2^22 entries. The world-1 run is also checked against direct
single-context C-ABI calls, and the invalid list against the tampered epochs."""
import ctypes
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu

LOG2N = 22
D = 14  # 2^14 epochs of 256 (coarse) / 2^12 of 1024 fit under 2^14


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    from paper_2506_08781_b200 import api
    from paper_2506_08781_b200 import multi_gpu as M
    from paper_2506_08781_b200.synth import SignedLog
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = {}
    try:
        v = api.Verifier(0)
        n = 1 << LOG2N
        # ---- config 2 shape: coarse
        n2 = 256
        lo, hi = M.shard_range(n // n2, world, rank)
        sl = SignedLog(v, lo, hi - lo, n2, D, seed=101)
        S = v.scalar_sum([x for x in M.all_gather_bytes(sl.S_part)])
        R = v.group_fold([x for x in M.all_gather_bytes(sl.R_part)])
        sp = M.ShardedPaver(v)
        out["c2_verdict"] = sp(sl.batch(), sl.Y, S, R)
        if rank == 0:
            p = sp.recs.cpu().numpy().tobytes()  # per rank: partial e-hat (32 B) | status | pad
            out["c2_e_hat"] = v.scalar_sum([p[sp.REC * r:sp.REC * r + 32] for r in range(world)])
        out["c2_e_tilde"] = b"".join(M.sharded_e_tilde(v, sl.batch()))
        if world == 1:  # the direct single-context calls agree
            et, eh = ctypes.create_string_buffer(32 * sl.n1), ctypes.create_string_buffer(32)
            b = sl.batch()
            v._call(v._lib.poslo_gpu_agg_ekeys, ctypes.byref(b), et, eh)
            out["direct_c2"] = (et.raw, eh.raw)
            vd = ctypes.c_uint8(0)
            v._call(v._lib.poslo_gpu_paver, ctypes.byref(b), sl.Y, S, R, None, ctypes.byref(vd))
            out["direct_c2_verdict"] = bool(vd.value)
        del sl
        # ---- config 3 / 5 shape: per-epoch verdicts and distillation with tampers
        n2 = 1024
        lo, hi = M.shard_range(n // n2, world, rank)
        sl = SignedLog(v, lo, hi - lo, n2, D, seed=202)
        # the same 16 global positions in both splits: tamper by global index
        import random
        rng = random.Random(9)
        bad_global = sorted(rng.sample(range(n), 16))
        for t in bad_global:
            if lo * n2 <= t < hi * n2:
                sl.log[(t - lo * n2) * 32] ^= 1
        torch.cuda.synchronize()
        out["bad_epochs"] = sorted({t // n2 for t in bad_global})
        Y = sl.Y
        out["c3_verdicts"] = M.sharded_epoch_verdicts(v, sl.batch(), Y, sl.s_dev.data_ptr(), sl.r_dev.data_ptr())
        res = M.sharded_distill(v, sl.batch(), lo, Y, sl.s_dev.data_ptr(), sl.r_dev.data_ptr(), 64)
        if rank == 0:
            out["c5"] = res
        if world == 1:
            vb = ctypes.create_string_buffer(sl.n1)
            b = sl.batch()
            v._call(v._lib.poslo_gpu_epoch_verify, ctypes.byref(b), Y, ctypes.c_void_p(sl.s_dev.data_ptr()),
                    ctypes.c_void_p(sl.r_dev.data_ptr()), vb, None)
            out["direct_c3"] = vb.raw
        q.put((rank, out))
        v.close()
    finally:
        dist.destroy_process_group()


def _run(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=900) for _ in procs)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 4])
def test_world1_vs_world_n_byte_identical_on_device(world):
    g1 = _run(1)[0]
    g2s = _run(world)
    g2 = g2s[0]
    # world 1 equals the direct single-context calls
    assert g1["c2_e_tilde"] == g1["direct_c2"][0] and g1["c2_e_hat"] == g1["direct_c2"][1]
    assert g1["c2_verdict"] is True and g1["direct_c2_verdict"] is True
    assert g1["c3_verdicts"] == g1["direct_c3"]
    # the determinism gate: G = world gathered outputs == G = 1, on every rank
    for r, g in g2s.items():
        assert g["c2_verdict"] == g1["c2_verdict"]
        assert g["c2_e_tilde"] == g1["c2_e_tilde"]
        assert g["c3_verdicts"] == g1["c3_verdicts"]
    assert g2["c2_e_hat"] == g1["c2_e_hat"]
    c5_1, c5_2 = g1["c5"], g2["c5"]
    assert c5_2["verdicts"] == c5_1["verdicts"] == g1["c3_verdicts"]
    assert c5_2["invalid"] == c5_1["invalid"] == g1["bad_epochs"]
    assert c5_2["umbrellas"] == c5_1["umbrellas"]
    assert len(c5_1["umbrellas"]) == (1 << LOG2N) // 1024 // 64
    assert c5_2["u_bits"] == c5_1["u_bits"] and all(c5_1["u_bits"])
