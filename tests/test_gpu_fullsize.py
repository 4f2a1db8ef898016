"""Parity at the FULL BASELINE sizes, beyond the slices of
test_gpu_scale.py:

* config 1 (2^20 x 32 B, n2 = 256): the PAVer DECISION of the device path
  equals the unmodified reference `poslo::paver` (oracle/_ref/ref_tool paver,
  the reference compiled from /root/reference/proj/src) on the same keys,
  log and signature -- accepted, with and without the R-hat aggregate, and
  rejected after a one-bit tamper and after a wrong s-hat -- and the two
  e-hats are equal;
* config 3 (2^30 x 32 B, n2 = 2^10 -> 2^20 per-epoch groups): every per-epoch
  verdict accepts the honestly signed log, 256 sampled e~ equal the pinned CPU
  oracle, e-hat equals the device fold of all 2^20 e~;
* config 5 (the same 2^30 log, n_u = 2^10 umbrellas of w = 2^10 epochs, k in
  {1, 16, 1024} tampered entries): the distillation's ascending invalid-epoch
  list is exactly the tampered epochs; every umbrella's (s, R, e) fold equals
  the fold of its valid epochs; sampled tampered/clean verdicts and the
  umbrella e-sums of the tampered umbrellas equal the CPU oracle on the same
  bytes; SeBVer V/U/I (distiller.cpp:181-233) over the resulting CCD: V and
  every U bit accept, every I bit rejects, and U of the tampered umbrellas
  equals the oracle's commit_check.

Keys and signatures use the reference's own derivation (kg / sig_epoch on the
device, tests/test_gpu_signer.py pins them against the reference signer)."""
import ctypes
import json
import os
import random
import struct
import subprocess
import tempfile

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_TOOL = os.path.join(ROOT, "oracle", "_ref", "ref_tool")


def _batch(N, log, n, n2, dsbuf, dsb, D, epochs=None, first_epoch=0):
    n1 = n // n2
    eps = np.arange(first_epoch, first_epoch + n1, dtype=np.uint32) if epochs is None else epochs
    b = N.PosloBatch()
    b.suite, b.n2, b.payload, b.payload_bytes = 1, n2, log.data_ptr(), n * 32
    b.offsets, b.entry_len, b.n_entries = None, 32, n
    b.epochs, b.epoch_starts, b.n_epochs = eps.ctypes.data, None, len(eps)
    b.ds, b.ds_len, b.ds_capacity, b.device_resident = ctypes.addressof(dsbuf), len(dsb), D, 1
    return b, eps


def _signed_log(verifier, log2n, n2, seed):
    """Synthetic log on the device, keys and per-epoch signatures by the
    reference derivation; returns a dict of everything the tests need."""
    import torch
    from paper_2506_08781_b200 import _native as N
    from paper_2506_08781_b200 import api
    lib = verifier._lib
    n = 1 << log2n
    n1 = n // n2
    D = max(1, (n1 - 1).bit_length())
    rng = random.Random(seed)
    ds = api.SeedStack(D, [api.SeedNode(D, 0, bytes(rng.getrandbits(8) for _ in range(16)))])
    dsb = ds.serialize()
    dsbuf = ctypes.create_string_buffer(dsb, len(dsb))
    err = N.PosloError()
    log = torch.empty(n * 32, dtype=torch.uint8, device="cuda")
    assert lib.poslo_gpu_synth_log(verifier._ctx, seed, 0, n, 32, ctypes.c_void_p(log.data_ptr()),
                                   ctypes.byref(err)) == 0
    b, eps = _batch(N, log, n, n2, dsbuf, dsb, D)
    y = rng.randrange(1, O.L).to_bytes(32, "little")
    r_seed = bytes(rng.getrandbits(8) for _ in range(16))
    r_hats = ctypes.create_string_buffer(n1 * 32)
    verifier._call(lib.poslo_gpu_kg_commitments, 1, r_seed, ctypes.c_void_p(eps.ctypes.data), n1, n2, r_hats, None)
    s_hats = ctypes.create_string_buffer(n1 * 32)
    verifier._call(lib.poslo_gpu_sig_epochs, ctypes.byref(b), r_seed, y, s_hats)
    torch.cuda.synchronize()
    return dict(N=N, api=api, lib=lib, torch=torch, n=n, n1=n1, n2=n2, D=D, ds=ds, dsb=dsb, dsbuf=dsbuf,
                log=log, b=b, eps=eps, y=y, Y=verifier.exp_base(y), r_hats=r_hats.raw, s_hats=s_hats.raw,
                rng=rng)


def _oracle_etilde(F, epochs):
    """CPU oracle e~ of the given epochs, reading only their bytes back."""
    n2 = F["n2"]
    parts = [F["log"][32 * n2 * i:32 * n2 * (i + 1)].cpu().numpy().tobytes() for i in epochs]
    starts = np.arange(len(epochs) + 1, dtype=np.uint64) * n2
    rc, _, et = O.agg_ekeys_packed(1, b"".join(parts), None, 32, list(epochs), starts, F["dsb"], F["D"])
    assert rc == 0
    return et


# ------------------------------------------------------------------ config 1
def _ref_paver(F, pk_bytes, s_hat, r_hat_agg, payload):
    n1, n2 = F["n1"], F["n2"]
    hdr = b"PVIO" + struct.pack("<8I", 1, n1, n2, 4, 32, n1, 8, F["D"])
    body = (struct.pack("<I", len(pk_bytes)) + pk_bytes + struct.pack("<I", len(F["dsb"])) + F["dsb"] + s_hat
            + (b"\x01" + r_hat_agg if r_hat_agg else b"\x00" + bytes(32)) + F["eps"].tobytes() + payload)
    with tempfile.NamedTemporaryFile(suffix=".pvio", delete=False) as f:
        f.write(hdr + body)
        path = f.name
    try:
        out = subprocess.run([REF_TOOL, "paver", path], capture_output=True, text=True, timeout=600)
    finally:
        os.unlink(path)
    assert out.returncode == 0, out.stderr
    return json.loads(out.stdout)


@pytest.mark.skipif(not os.path.exists(REF_TOOL), reason="oracle/_ref/ref_tool not built (build())")
def test_config1_paver_decision_equals_reference(verifier):
    F = _signed_log(verifier, 20, 256, 101)
    api, lib, n1 = F["api"], F["lib"], F["n1"]
    suite = api.SuiteConfig(1, n1, F["n2"], 4)
    S, Rh = F["s_hats"], F["r_hats"]
    pk = api.PoslocPublicKey(suite, F["Y"], {i: Rh[32 * i:32 * i + 32] for i in range(n1)})
    pkb = pk.serialize()
    s_hat = verifier.scalar_sum([S[32 * i:32 * i + 32] for i in range(n1)])
    r_agg = verifier.group_fold([Rh[32 * i:32 * i + 32] for i in range(n1)])

    def gpu(s, agg):
        v = ctypes.c_uint8(0)
        verifier._call(lib.poslo_gpu_paver, ctypes.byref(F["b"]), F["Y"], s, agg, None if agg else Rh,
                       ctypes.byref(v))
        return int(v.value)

    log = F["log"]
    cases = []
    for name, s, agg in (("accept, R-hat folded from pk", s_hat, None), ("accept, R-hat aggregate", s_hat, r_agg),
                         ("reject, wrong s-hat", O.sc_add(s_hat, (1).to_bytes(32, "little")), r_agg)):
        cases.append((name, s, agg))
    results = []
    for name, s, agg in cases:
        ref = _ref_paver(F, pkb, s, agg, log.cpu().numpy().tobytes())
        assert ref["error"] == "", ref
        results.append((name, gpu(s, agg), ref["paver"], ref["e_hat"]))
    # one bit flipped in entry 777 after signing
    log[777 * 32 + 5] ^= 0x10
    F["torch"].cuda.synchronize()
    ref = _ref_paver(F, pkb, s_hat, None, log.cpu().numpy().tobytes())
    results.append(("reject, tampered entry", gpu(s_hat, None), ref["paver"], ref["e_hat"]))
    e_dev = ctypes.create_string_buffer(32)
    verifier._call(lib.poslo_gpu_agg_ekeys, ctypes.byref(F["b"]), None, e_dev)
    assert e_dev.raw.hex() == ref["e_hat"], "e-hat of the tampered log differs from the reference"
    for name, g, r, _ in results:
        assert g == r, f"{name}: device {g} vs reference {r}"
    assert [r for _, _, r, _ in results] == [1, 1, 0, 0]


# ------------------------------------------------------------- configs 3 / 5
@pytest.fixture(scope="module")
def big(verifier):
    F = _signed_log(verifier, 30, 1024, 303)
    yield F
    del F["log"]
    F["torch"].cuda.empty_cache()


def test_config3_full_size_epoch_verdicts(verifier, big):
    F = big
    lib, n1 = F["lib"], F["n1"]
    verd = ctypes.create_string_buffer(n1)
    et = ctypes.create_string_buffer(n1 * 32)
    torch = F["torch"]
    s_dev = torch.frombuffer(bytearray(F["s_hats"]), dtype=torch.uint8).cuda()  # device-resident batch:
    r_dev = torch.frombuffer(bytearray(F["r_hats"]), dtype=torch.uint8).cuda()  # signatures on the device too
    torch.cuda.synchronize()
    verifier._call(lib.poslo_gpu_epoch_verify, ctypes.byref(F["b"]), F["Y"], ctypes.c_void_p(s_dev.data_ptr()),
                   ctypes.c_void_p(r_dev.data_ptr()), verd, et)
    assert verd.raw == b"\x01" * n1, "an honestly signed epoch was rejected"
    raw = et.raw
    e_hat = ctypes.create_string_buffer(32)
    verifier._call(lib.poslo_gpu_agg_ekeys, ctypes.byref(F["b"]), None, e_hat)
    assert verifier.scalar_sum([raw[32 * k:32 * k + 32] for k in range(n1)]) == e_hat.raw
    pick = sorted(F["rng"].sample(range(n1), 256))
    assert [raw[32 * i:32 * i + 32] for i in pick] == _oracle_etilde(F, pick)
    F["e_tilde"] = raw


@pytest.mark.parametrize("k", [1, 16, 1024])
def test_config5_full_size_tamper_localisation(verifier, big, k):
    from oracle import ristretto as RR
    F = big
    lib, torch, n, n1, n2 = F["lib"], F["torch"], F["n"], F["n1"], F["n2"]
    rng = random.Random(5000 + k)
    tampered = sorted(rng.sample(range(n), k))
    flips = [(t, rng.randrange(32), 1 << rng.randrange(8)) for t in tampered]
    log = F["log"]
    idx = torch.tensor([32 * t + o for t, o, _ in flips], dtype=torch.int64, device="cuda")
    msk = torch.tensor([m for _, _, m in flips], dtype=torch.uint8, device="cuda")
    log[idx] ^= msk
    torch.cuda.synchronize()
    try:
        bad = sorted({t // n2 for t in tampered})
        w = 1024
        cuts = np.arange(0, n1 + 1, w, dtype=np.uint32)
        n_seg = len(cuts) - 1
        s_dev = torch.frombuffer(bytearray(F["s_hats"]), dtype=torch.uint8).cuda()
        r_dev = torch.frombuffer(bytearray(F["r_hats"]), dtype=torch.uint8).cuda()
        verd = ctypes.create_string_buffer(n1)
        seg_s, seg_r, seg_e = (ctypes.create_string_buffer(32 * n_seg) for _ in range(3))
        verifier._call(lib.poslo_gpu_distill_coarse_ex, ctypes.byref(F["b"]), F["Y"], ctypes.c_void_p(s_dev.data_ptr()),
                       ctypes.c_void_p(r_dev.data_ptr()), ctypes.c_void_p(cuts.ctypes.data), n_seg, verd, seg_s,
                       seg_r, seg_e)
        v = verd.raw
        invalid = [i for i in range(n1) if not v[i]]
        assert invalid == bad, "invalid-epoch list differs from the tampered epochs"
        S, Rh = F["s_hats"], F["r_hats"]
        et = F.get("e_tilde")
        # every umbrella's folds over its valid epochs (device folds of the inputs)
        badset = set(bad)
        for g in range(n_seg):
            ok = [i for i in range(cuts[g], cuts[g + 1]) if i not in badset]
            assert seg_s.raw[32 * g:32 * g + 32] == verifier.scalar_sum([S[32 * i:32 * i + 32] for i in ok])
            assert seg_r.raw[32 * g:32 * g + 32] == verifier.group_fold([Rh[32 * i:32 * i + 32] for i in ok])
            if et is not None:  # clean e~ of the same epochs (the tamper touched only invalid ones)
                assert seg_e.raw[32 * g:32 * g + 32] == verifier.scalar_sum([et[32 * i:32 * i + 32] for i in ok])
        # sampled verdicts against the CPU oracle on the same (tampered) bytes
        clean = [i for i in rng.sample(range(n1), 64) if i not in badset][:16]
        probe = bad[:16] + clean
        for i, e in zip(probe, _oracle_etilde(F, probe)):
            want = RR.commit_check(F["Y"], e, S[32 * i:32 * i + 32]) == Rh[32 * i:32 * i + 32]
            assert bool(v[i]) == want, f"epoch {i}"
        # umbrella e-sums of (up to 4) tampered umbrellas and 1 clean one against the oracle
        umbs = sorted({i // w for i in bad})[:4] + [u for u in range(n_seg) if all(i // w != u for i in bad)][:1]
        for u in umbs:
            ok = [i for i in range(u * w, (u + 1) * w) if i not in badset]
            e_or = O.sum_scalars(_oracle_etilde(F, ok))
            assert seg_e.raw[32 * u:32 * u + 32] == e_or
            s_or = O.sum_scalars([S[32 * i:32 * i + 32] for i in ok])
            assert seg_s.raw[32 * u:32 * u + 32] == s_or
            # the oracle's U verdict for this umbrella record (the device's is checked below)
            assert RR.commit_check(F["Y"], e_or, s_or) == seg_r.raw[32 * u:32 * u + 32]
        # SeBVer over the CCD the distillation produced: V and U accept, I rejects
        vs = verifier.scalar_sum([seg_s.raw[32 * g:32 * g + 32] for g in range(n_seg)])
        vr = verifier.group_fold([seg_r.raw[32 * g:32 * g + 32] for g in range(n_seg)])
        inv = np.array(bad, dtype=np.uint32)
        inv_s = b"".join(S[32 * i:32 * i + 32] for i in bad)
        inv_r = b"".join(Rh[32 * i:32 * i + 32] for i in bad)
        ui = np.arange(n_seg, dtype=np.uint32)
        vbit = ctypes.c_uint8(0)
        ubits = ctypes.create_string_buffer(n_seg)
        ibits = ctypes.create_string_buffer(len(bad))
        verifier._call(lib.poslo_gpu_sebver, ctypes.byref(F["b"]), F["Y"], n1, n_seg,
                       ctypes.c_void_p(inv.ctypes.data), inv_s, inv_r, len(bad), vs, vr, ctypes.byref(vbit),
                       ctypes.c_void_p(ui.ctypes.data), seg_s.raw, seg_r.raw, n_seg, ubits, ibits)
        assert vbit.value == 1
        assert ubits.raw == b"\x01" * n_seg
        assert ibits.raw == b"\x00" * len(bad)
    finally:
        log[idx] ^= msk
        torch.cuda.synchronize()
