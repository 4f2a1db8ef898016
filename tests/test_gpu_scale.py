"""Parity at BASELINE sizes: config 1 in full (2^20 x 32 B,
every epoch against the oracle); "sampled" above it: the device verifies the
full synthetic log of config 2 (2^26 x 32 B, n2 = 256), a per-epoch config-3
slice (2^24 x 32 B, n2 = 1024), a config-4 slice (2^20 syslog entries) and a
config-5 slice (tamper localisation over 2^22 signed entries);
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
        from paper_2506_08781_b200 import synth as bench
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


def test_config1_full_parity(verifier):
    """Config 1 (2^20 x 32 B, n2 = 256, the reference's CPU-runnable case):
    EVERY epoch's e~ (all 4096) against the oracle, not a sample."""
    _run(verifier, 20, 256, False, 4096, 11)


def test_config2_full_size_sampled_parity(verifier):
    _run(verifier, 26, 256, False, 256, 21)


def test_config3_slice_sampled_parity(verifier):
    _run(verifier, 24, 1024, False, 256, 23)


def test_config4_slice_sampled_parity(verifier):
    _run(verifier, 20, 1024, True, 64, 24)


def test_config5_slice_tamper_localisation(verifier):
    """Config 5 at 2^22 x 32 B (4096 epochs of 1024): keys and epoch signatures
    by the reference's derivation (kg / sig_epoch on the device), 16 entries
    tampered after signing (one bit each), then device distillation of every
    epoch: the invalid-epoch list is exactly the tampered epochs, each umbrella
    piece's folded (s, R) equals the fold of its valid epochs, and sampled
    verdicts (tampered and clean) equal the CPU oracle's commit_check on the
    same bytes."""
    import torch
    from oracle import ristretto as RR
    from paper_2506_08781_b200 import _native as N
    from paper_2506_08781_b200 import api
    lib = verifier._lib
    n2, n = 1024, 1 << 22
    n1 = n // n2
    D = (n1 - 1).bit_length()
    rng = random.Random(55)
    ds = api.SeedStack(D, [api.SeedNode(D, 0, bytes(rng.getrandbits(8) for _ in range(16)))])
    dsb = ds.serialize()
    dsbuf = ctypes.create_string_buffer(dsb, len(dsb))
    err = N.PosloError()
    log = torch.empty(n * 32, dtype=torch.uint8, device="cuda")
    assert lib.poslo_gpu_synth_log(verifier._ctx, 9, 0, n, 32, ctypes.c_void_p(log.data_ptr()),
                                   ctypes.byref(err)) == 0
    epochs = np.arange(n1, dtype=np.uint32)
    b = N.PosloBatch()
    b.suite, b.n2, b.payload, b.payload_bytes = 1, n2, log.data_ptr(), n * 32
    b.offsets, b.entry_len, b.n_entries = None, 32, n
    b.epochs, b.epoch_starts, b.n_epochs = epochs.ctypes.data, None, n1
    b.ds, b.ds_len, b.ds_capacity, b.device_resident = ctypes.addressof(dsbuf), len(dsb), D, 1
    y = rng.randrange(1, O.L).to_bytes(32, "little")
    r_seed = bytes(rng.getrandbits(8) for _ in range(16))
    r_hats = ctypes.create_string_buffer(n1 * 32)
    verifier._call(lib.poslo_gpu_kg_commitments, 1, r_seed, ctypes.c_void_p(epochs.ctypes.data), n1, n2, r_hats,
                   None)
    s_hats = ctypes.create_string_buffer(n1 * 32)
    verifier._call(lib.poslo_gpu_sig_epochs, ctypes.byref(b), r_seed, y, s_hats)
    tampered = sorted(rng.sample(range(n), 16))
    for t in tampered:
        log[t * 32] ^= 1
    torch.cuda.synchronize()
    bad = sorted({t // n2 for t in tampered})
    w = 64  # n_u = 64 umbrellas
    cuts = np.array(list(range(0, n1 + 1, w)), dtype=np.uint32)
    n_seg = len(cuts) - 1
    Y = verifier.exp_base(y)
    s_dev = torch.frombuffer(bytearray(s_hats.raw), dtype=torch.uint8).cuda()
    r_dev = torch.frombuffer(bytearray(r_hats.raw), dtype=torch.uint8).cuda()
    torch.cuda.synchronize()
    verd = ctypes.create_string_buffer(n1)
    seg_s = ctypes.create_string_buffer(32 * n_seg)
    seg_r = ctypes.create_string_buffer(32 * n_seg)
    verifier._call(lib.poslo_gpu_distill_coarse, ctypes.byref(b), Y, ctypes.c_void_p(s_dev.data_ptr()),
                   ctypes.c_void_p(r_dev.data_ptr()), ctypes.c_void_p(cuts.ctypes.data), n_seg, verd, seg_s, seg_r)
    v = verd.raw
    assert [i for i in range(n1) if not v[i]] == bad
    S, Rh = s_hats.raw, r_hats.raw
    for g in range(n_seg):
        ok = [i for i in range(cuts[g], cuts[g + 1]) if v[i]]
        assert seg_s.raw[32 * g:32 * g + 32] == verifier.scalar_sum([S[32 * i:32 * i + 32] for i in ok])
        assert seg_r.raw[32 * g:32 * g + 32] == verifier.group_fold([Rh[32 * i:32 * i + 32] for i in ok])
    # sampled verdicts against the oracle (hashing + commit_check on the CPU)
    host = log.cpu().numpy()
    for i in bad[:3] + rng.sample([i for i in range(n1) if v[i]], 3):
        flat = host[32 * n2 * i:32 * n2 * (i + 1)].tobytes()
        offs = np.arange(n2 + 1, dtype=np.uint64) * 32
        rc, _, et = O.agg_ekeys_packed(1, flat, offs, 0, [i], np.array([0, n2], dtype=np.uint64), dsb, D)
        assert rc == 0
        want = RR.commit_check(Y, et[0], S[32 * i:32 * i + 32]) == Rh[32 * i:32 * i + 32]
        assert bool(v[i]) == want
