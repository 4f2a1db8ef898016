"""Scheme-F per-entry verification throughput (poslo_gpu_fine_verify: one
hash_to_scalar + one commit_check per ENTRY, the EC-bound row f3) on cuda:0,
inputs in PINNED host memory: 2^k 32-byte entries with seed tails, random s
and a valid-encoding R per entry (verdicts are mostly false; the work is the
same). POSLO_COMB16_MIN picks the check path (radix-2^16 split checks for
large batches by default)."""
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2506_08781_b200 import _native as N
from paper_2506_08781_b200 import api

v = api.Verifier(0)
lib = v._lib
rng = np.random.default_rng(1)


def pinned(a):
    t = torch.empty(a.size, dtype=torch.uint8, pin_memory=True)
    t.numpy()[:] = a.reshape(-1)
    return t


for log2n in (16, 18, 20):
    n = 1 << log2n
    pay = rng.integers(0, 256, n * 32, dtype=np.uint8)
    seeds = rng.integers(0, 256, n * 16, dtype=np.uint8)
    s = np.zeros((n, 32), dtype=np.uint8)
    s[:, :31] = rng.integers(0, 256, (n, 31), dtype=np.uint8)
    r1 = v.exp_base((12345).to_bytes(32, "little"))
    r = np.frombuffer(r1 * n, dtype=np.uint8).copy()
    y = v.exp_base((777).to_bytes(32, "little"))
    keep = [pinned(x) for x in (pay, seeds, s, r)]
    pay_p, seeds_p, s_p, r_p = (t.data_ptr() for t in keep)
    fb = N.PosloFineBatch()
    fb.suite, fb.payload, fb.payload_bytes = 1, pay_p, pay.size
    fb.offsets, fb.entry_len, fb.n_entries, fb.device_resident = None, 32, n, 0
    fb.seeds = seeds_p
    verd = np.zeros(n, dtype=np.uint8)
    err = N.PosloError()
    ts = []
    for it in range(4):
        t0 = time.perf_counter()
        rc = lib.poslo_gpu_fine_verify(v._ctx, ctypes.byref(fb), y, s_p, r_p,
                                       verd.ctypes.data, ctypes.byref(err))
        ts.append(time.perf_counter() - t0)
        assert rc == 0, err.message
    t = min(ts[1:])
    print(f"2^{log2n} entries: {t * 1e3:.2f} ms, {n / t:.3e} entries/s (pinned host inputs, incl. H2D)", flush=True)
