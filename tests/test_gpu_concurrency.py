"""Re-entrancy of the boundary (SURVEY.md §8b "Threading": agg_ekeys "may be
called concurrently from many host threads"; "externally a
pure, thread-safe function"). Host threads call the C-ABI at once — on one
shared context (calls serialise on its mutex) and on one context each — and
every per-epoch result must equal the pinned CPU oracle on the same inputs.
ctypes drops the GIL for the foreign call, so the calls really overlap. The
C++ drop-in gets the same treatment against the reference's own sequential
aggregate_ekey (paper_2506_08781_b200/host/test_concurrency.cpp)."""
import os
import subprocess
import threading

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _job(api, seed):
    rng = np.random.default_rng(seed)
    suite = 1 + seed % 2
    n1, n2 = 32, 16 + seed % 7
    batches = {}
    for i in range(n1):
        if rng.integers(0, 3) == 0:
            continue
        lens = rng.integers(0, 150, size=n2)
        batches[i] = [bytes(rng.integers(0, 256, int(L), dtype=np.uint8)) for L in lens]
    D = (n1 - 1).bit_length()
    ds = api.SeedStack(D, [api.SeedNode(D, 0, bytes(rng.integers(0, 256, 16, dtype=np.uint8)))])
    cfg = api.SuiteConfig(suite, n1, n2, 1)
    epochs = sorted(batches)
    flat = [m for i in epochs for m in batches[i]]
    offs = np.zeros(len(flat) + 1, dtype=np.uint64)
    np.cumsum([len(m) for m in flat], out=offs[1:])
    starts = np.zeros(len(epochs) + 1, dtype=np.uint64)
    np.cumsum([len(batches[i]) for i in epochs], out=starts[1:])
    rc, _, ref = O.agg_ekeys_packed(suite, b"".join(flat), offs, 0, epochs, starts, ds.serialize(), ds.capacity)
    assert rc == 0
    return cfg, batches, ds, list(zip(epochs, ref))


def _hammer(make_verifier, n_threads=6, iters=4):
    from paper_2506_08781_b200 import api
    jobs = [_job(api, s) for s in range(n_threads * iters)]
    errors = []

    def run(t):
        try:
            v = make_verifier(t)
            for k in range(iters):
                cfg, batches, ds, want = jobs[t * iters + k]
                parts, _ = v.agg_ekeys(cfg, batches, ds, 1)
                if parts != want:
                    errors.append((t, k))
        except Exception as e:  # surfaced below, never swallowed
            errors.append((t, repr(e)))

    threads = [threading.Thread(target=run, args=(t,)) for t in range(n_threads)]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors


def test_threads_share_one_context(verifier):
    _hammer(lambda t: verifier)


def test_threads_with_own_contexts():
    from paper_2506_08781_b200 import api
    own = {}

    def make(t):
        own[t] = api.Verifier(0)
        return own[t]

    _hammer(make)
    for v in own.values():
        v.close()


def test_cpp_drop_in_concurrent_callers():
    exe = os.path.join(ROOT, "oracle", "_ref", "test_concurrency_gpu")
    if not os.path.exists(exe):
        pytest.fail(f"{exe} missing: build with __graft_entry__.build() where /root/reference exists")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "mismatches 0" in out.stdout
