"""Parity at BASELINE sizes (SURVEY §8d "sampled"): the device verifies the
full synthetic log of config 2 (2^26 x 32 B, n2 = 256), a per-epoch config-3
slice (2^24 x 32 B, n2 = 1024) and a config-4 slice (2^20 syslog entries);
e~ of 256 randomly chosen epochs (64 for config 4) must equal the pinned CPU
oracle on the same bytes, and e-hat must equal the sum of all e~ (a
size-independent checksum of checksums)."""
import ctypes
import random

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _run(verifier, log2n, n2, varlen, samples, seed):
    import torch
    from paper_2506_08781_b200 import _native as N
    from paper_2506_08781_b200 import api
    lib = verifier._lib
    n, n1 = 1 << log2n, (1 << log2n) // n2
    D = max(1, (n1 - 1).bit_length())
    rng = random.Random(seed)
    root = bytes(rng.getrandbits(8) for _ in range(16))
    ds = api.SeedStack(D, [api.SeedNode(D, 0, root)])
    dsb = ds.serialize()
    dsbuf = ctypes.create_string_buffer(dsb, len(dsb))
    err = N.PosloError()
    offs_dev = None
    if varlen:
        import bench
        lens = bench.synth_varlen(seed, 0, n)
        offs = np.zeros(n + 1, dtype=np.uint64)
        np.cumsum(lens, out=offs[1:])
        offs_dev = torch.from_numpy(offs.view(np.int64)).cuda()
        log = torch.empty(int(offs[-1]), dtype=torch.uint8, device="cuda")
        assert lib.poslo_gpu_synth_varlog(verifier._ctx, seed, 0, n, ctypes.c_void_p(offs_dev.data_ptr()),
                                          ctypes.c_void_p(log.data_ptr()), ctypes.byref(err)) == 0
    else:
        log = torch.empty(n * 32, dtype=torch.uint8, device="cuda")
        assert lib.poslo_gpu_synth_log(verifier._ctx, seed, 0, n, 32, ctypes.c_void_p(log.data_ptr()),
                                       ctypes.byref(err)) == 0
    epochs = np.arange(n1, dtype=np.uint32)
    b = N.PosloBatch()
    b.suite, b.n2, b.payload, b.payload_bytes = 1, n2, log.data_ptr(), log.numel()
    b.offsets = offs_dev.data_ptr() if varlen else None
    b.entry_len, b.n_entries = 0 if varlen else 32, n
    b.epochs, b.epoch_starts, b.n_epochs = epochs.ctypes.data, None, n1
    b.ds, b.ds_len, b.ds_capacity, b.device_resident = ctypes.addressof(dsbuf), len(dsb), D, 1
    et = ctypes.create_string_buffer(n1 * 32)
    eh = ctypes.create_string_buffer(32)
    verifier._call(lib.poslo_gpu_agg_ekeys, ctypes.byref(b), et, eh)
    raw = et.raw
    # checksum of checksums: e-hat = sum of every e~ (device fold of the device outputs)
    assert verifier.scalar_sum([raw[32 * k:32 * k + 32] for k in range(n1)]) == eh.raw
    # sampled epochs against the oracle on the same bytes
    host = log.cpu().numpy()
    pick = sorted(rng.sample(range(n1), samples))
    flat, lens_s = [], []
    for i in pick:
        for t in range(i * n2, (i + 1) * n2):
            if varlen:
                m = host[int(offs[t]):int(offs[t + 1])].tobytes()
            else:
                m = host[32 * t:32 * t + 32].tobytes()
            flat.append(m)
            lens_s.append(len(m))
    o = np.zeros(len(flat) + 1, dtype=np.uint64)
    np.cumsum(lens_s, out=o[1:])
    starts = np.arange(len(pick) + 1, dtype=np.uint64) * n2
    rc, _, ref = O.agg_ekeys_packed(1, b"".join(flat), o, 0, pick, starts, dsb, D)
    assert rc == 0
    assert [raw[32 * i:32 * i + 32] for i in pick] == ref


def test_config2_full_size_sampled_parity(verifier):
    _run(verifier, 26, 256, False, 256, 21)


def test_config3_slice_sampled_parity(verifier):
    _run(verifier, 24, 1024, False, 256, 23)


def test_config4_slice_sampled_parity(verifier):
    _run(verifier, 20, 1024, True, 64, 24)
