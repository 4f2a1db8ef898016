"""Device parity: every stage of the CUDA path against the reference's own
golden outputs (tests/golden, from the UNMODIFIED reference) and the pinned
CPU oracle on the same seeded inputs. Bit-exact throughout (integer work)."""
import random

import numpy as np
import pytest

from conftest import STREAMS, load_golden
from golden_util import Stream
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def A():
    from paper_2506_08781_b200 import api
    return api


# ------------------------------------------------------------------ golden streams
@pytest.mark.parametrize("name", STREAMS)
def test_agg_ekeys_matches_reference(verifier, name):
    st = Stream(load_golden(name + ".json"))
    suite, pk, ds = st.api_objects()
    parts, e_hat = verifier.agg_ekeys(suite, st.batches, ds, 4)
    assert [p[0] for p in parts] == sorted(st.batches)
    assert [p[1] for p in parts] == st.e_tilde
    assert e_hat == st.e_hat


def test_warp_decode_and_table_chain_on_kat_points(verifier, kat):
    """The warp-cooperative paths (ristretto.cuh fw_*) on every KAT encoding,
    14 valid and 34 invalid (RFC 9496 negative vectors among them):
    commit_check with the point as Y builds Y's comb tables (decode by a whole
    warp, then the 252-doubling chain three products per round) and must
    equal the oracle, or raise FormatError for an invalid Y; as the paver's
    R-hat aggregate (decoded by a warp in k_check_pre) only the correct
    aggregate verifies, and an invalid encoding is a plain reject."""
    import random
    api = A()
    from oracle import ristretto as R
    rng = random.Random(255)
    e = rng.randrange(R.L).to_bytes(32, "little")
    s = rng.randrange(R.L).to_bytes(32, "little")
    pts = [(bytes.fromhex(h), bool(v)) for h, v in kat["point_valid"]]
    assert sum(v for _, v in pts) == 14 and len(pts) == 48
    for y, valid in pts:
        if valid:
            assert verifier.commit_check(y, e, s) == R.commit_check(y, e, s)
        else:
            with pytest.raises(api.FormatError):
                verifier.commit_check(y, e, s)
    st = Stream(load_golden("stream_s1_clean_big.json"))
    suite, pk, ds = st.api_objects()
    assert verifier.paver(pk, st.batches, st.s_hat, st.r_hat_agg, ds, 1) is True
    for r, _ in pts:
        assert verifier.paver(pk, st.batches, st.s_hat, r, ds, 1) == (r == st.r_hat_agg)


@pytest.mark.parametrize("name", STREAMS)
def test_paver_matches_reference(verifier, name):
    st = Stream(load_golden(name + ".json"))
    suite, pk, ds = st.api_objects()
    assert verifier.paver(pk, st.batches, st.s_hat, None, ds, 8) == bool(st.d["paver"])
    assert verifier.paver(pk, st.batches, st.s_hat, st.r_hat_agg, ds, 2) == bool(st.d["paver_agg"])


@pytest.mark.parametrize("name", STREAMS)
def test_epoch_verdicts_match_reference(verifier, name):
    """Per-epoch accept/reject (the distiller's per-epoch aver, tamper localisation)."""
    st = Stream(load_golden(name + ".json"))
    suite, pk, ds = st.api_objects()
    s_hats = {i: st.sigs[i].s_hat_le for i in range(st.n1)}
    # each epoch signature carries its own ds; the final ds covers every epoch
    verdicts = verifier.epoch_verify(pk, st.batches, s_hats, ds)
    assert [int(v) for v in verdicts] == st.d["epoch_verdicts"]
    assert [i for i, v in enumerate(verdicts) if not v] == st.d["invalid_epochs"]


@pytest.mark.parametrize("name", STREAMS)
def test_sebver_matches_reference(verifier, name):
    st = Stream(load_golden(name + ".json"))
    api = A()
    c = st.ccd
    suite = api.SuiteConfig(c["suite"], c["n1"], c["n2"], c["n_u"])
    ds, _ = api.SeedStack.deserialize(c["ds"], c["depth"])
    res = verifier.sebver(st.pk.y, suite, st.batches, ds, c["next"], c["invalid"], c["umbrellas"],
                          c["valid"] if c["has_valid"] else None)
    assert [int(b) for b in res["U"]] == st.d["sebver_U"]
    assert [int(b) for b in res["I"]] == st.d["sebver_I"]
    if "sebver_V" in st.d:
        assert [int(b) for b in res["V"]] == st.d["sebver_V"]


# ------------------------------------------------------------------ stage parity
@pytest.mark.parametrize("suite", [1, 2, 3])
def test_seed_retrieve_matches_reference(verifier, kat, suite):
    api = A()
    d = kat[f"suite{suite}"]
    ds, _ = api.SeedStack.deserialize(bytes.fromhex(d["ds_after_11"]), 4)
    got = verifier.seed_retrieve(suite, ds, list(range(12)))
    assert [g.hex() for g in got] == d["sr"]
    with pytest.raises(api.SeedNotDisclosed) as ei:
        verifier.seed_retrieve(suite, ds, [3, 12, 13])
    assert ei.value.epoch == 12


@pytest.mark.parametrize("suite", [1, 2, 3])
def test_entry_scalars_match_oracle(verifier, suite):
    api = A()
    rng = random.Random(100 + suite)
    n1, n2 = 8, 16
    maxlen = 31 if suite == 3 else 300
    batches = {i: [bytes(rng.getrandbits(8) for _ in range(rng.randint(1, maxlen))) for _ in range(n2)]
               for i in range(n1)}
    root = bytes(rng.getrandbits(8) for _ in range(16))
    ds = api.SeedStack(3, [api.SeedNode(3, 0, root)])
    got = verifier.entry_scalars(api.SuiteConfig(suite, n1, n2, 1), batches, ds)
    k = 0
    for i in range(n1):
        _, x0 = O.sr(suite, ds.serialize(), 3, i)
        for j, m in enumerate(batches[i]):
            assert got[k] == O.hash_to_scalar(suite, m, O.onetime_seed(suite, x0, j)), (i, j)
            k += 1


def test_group_primitives_match_reference(verifier, kat):
    rows = kat["commit_check"]
    for Y, e, s, P in rows:
        assert verifier.commit_check(bytes.fromhex(Y), bytes.fromhex(e), bytes.fromhex(s)).hex() == P
    for s, p in kat["exp_base"]:
        assert verifier.exp_base(bytes.fromhex(s)).hex() == p
    for a, b, c in kat["group_combine"]:
        assert verifier.group_combine(bytes.fromhex(a), bytes.fromhex(b)).hex() == c
    pts = [bytes.fromhex(p) for p, _ in kat["point_valid"]]
    assert verifier.is_valid_point_batch(pts) == [bool(v) for _, v in kat["point_valid"]]


def test_commit_check_batched(verifier, kat):
    rows = kat["commit_check"][5:]
    Y = bytes.fromhex(rows[0][0])
    es = [bytes.fromhex(r[1]) for r in rows]
    ss = [bytes.fromhex(r[2]) for r in rows]
    got = verifier.commit_check_batch(Y, es, ss)
    from oracle import ristretto as R
    for e, s, g in zip(es, ss, got):
        assert g == R.commit_check(Y, e, s)


@pytest.mark.parametrize("comb16", [False, True])
def test_commit_check_radix256_path(verifier, kat, comb16, monkeypatch):
    """n > 1024 checks run thread-per-check on the radix-256 combs (or, with
    POSLO_COMB16_MIN = 1, on the radix-2^16 combs large batches take by
    default); they must agree with the CTA path (radix-16 combs, n <= 1024)
    and the oracle, including edge scalars (0, 1, l - 1, digits that carry,
    2^16-digit boundaries)."""
    import random
    monkeypatch.setenv("POSLO_COMB16_MIN", "1" if comb16 else "4294967295")
    from oracle import ristretto as R
    rng = random.Random(256)
    Y = bytes.fromhex(kat["commit_check"][5][0])
    L = R.L if hasattr(R, "L") else 2**252 + 27742317777372353535851937790883648493
    edge = [0, 1, 2, 127, 128, 255, 256, 0x80 * 0x0101010101, L - 1, L - 128, 2**252,
            32767, 32768, 32769, 65535, 65536, 0x8000 * (1 + 2**16 + 2**32 + 2**48), 2**240 - 1]
    vals = edge + [rng.randrange(L) for _ in range(1100 - len(edge))]
    es = [v.to_bytes(32, "little") for v in vals]
    ss = [rng.randrange(L).to_bytes(32, "little") for _ in vals]
    ss[0] = bytes(32)
    wide = verifier.commit_check_batch(Y, es, ss)          # 1100 > 1024: radix-256 path
    narrow = []
    for k in range(0, len(es), 1000):                        # <= 1024: radix-16 CTA path
        narrow += verifier.commit_check_batch(Y, es[k:k + 1000], ss[k:k + 1000])
    assert wide == narrow
    for k in list(range(len(edge))) + [500, 1099]:
        assert wide[k] == R.commit_check(Y, es[k], ss[k])


# ------------------------------------------------------------------ synthetic scale parity
def _synthetic(suite, n1, n2, L, seed, ragged=False):
    api = A()
    rng = np.random.default_rng(seed)
    if ragged:
        lens = rng.integers(0 if suite != 3 else 1, (31 if suite == 3 else 700) + 1, size=n1 * n2)
        pay = rng.integers(0, 256, size=int(lens.sum()), dtype=np.uint8).tobytes()
        offs = np.zeros(len(lens) + 1, dtype=np.uint64)
        np.cumsum(lens, out=offs[1:])
        ents = [pay[offs[t]:offs[t + 1]] for t in range(n1 * n2)]
    else:
        pay = rng.integers(0, 256, size=n1 * n2 * L, dtype=np.uint8).tobytes()
        ents = [pay[t * L:(t + 1) * L] for t in range(n1 * n2)]
    batches = {i: ents[i * n2:(i + 1) * n2] for i in range(n1)}
    D = max(1, (n1 - 1).bit_length())
    root = bytes(rng.integers(0, 256, 16, dtype=np.uint8))
    ds = api.SeedStack(D, [api.SeedNode(D, 0, root)])
    return api.SuiteConfig(suite, 1 << D, n2, 1), batches, ds


def _oracle_etilde(suite, batches, ds):
    epochs = sorted(batches)
    flat = [m for i in epochs for m in batches[i]]
    offs = np.zeros(len(flat) + 1, dtype=np.uint64)
    np.cumsum([len(m) for m in flat], out=offs[1:])
    starts = np.zeros(len(epochs) + 1, dtype=np.uint64)
    np.cumsum([len(batches[i]) for i in epochs], out=starts[1:])
    rc, _, et = O.agg_ekeys_packed(suite, b"".join(flat), offs, 0, epochs, starts, ds.serialize(),
                                   ds.capacity)
    assert rc == 0
    return et


@pytest.mark.parametrize("suite,n1,n2,L", [
    (1, 64, 256, 32), (1, 16, 1024, 32), (1, 4, 3000, 32), (1, 300, 5, 32),
    (2, 32, 256, 32), (2, 4, 1100, 32), (1, 32, 64, 48), (2, 16, 64, 17), (3, 32, 64, 31),
])
def test_uniform_batches_match_oracle(verifier, suite, n1, n2, L):
    cfg, batches, ds = _synthetic(suite, n1, n2, L, seed=n1 * 7 + n2 + L + suite)
    parts, e_hat = verifier.agg_ekeys(cfg, batches, ds, 1)
    ref = _oracle_etilde(suite, batches, ds)
    assert [p[1] for p in parts] == ref
    assert e_hat == O.sum_scalars(ref)


@pytest.mark.parametrize("suite", [1, 2])
def test_every_entry_length_and_alignment(verifier, suite):
    """Every entry length 0..320 (each residue mod 64 five times: the block
    boundaries of both hash streams, incl. L + 25 = 0 mod 64 where stream 0
    ends one block before stream 1) at every start alignment mod 16."""
    api = A()
    rng = np.random.default_rng(4242 + suite)
    n1, n2 = 16, 321
    batches = {}
    for i in range(n1):
        lens = rng.permutation(n2)
        batches[i] = [bytes(rng.integers(0, 256, int(L), dtype=np.uint8)) for L in lens]
    cfg = api.SuiteConfig(suite, n1, n2, 1)
    D = (n1 - 1).bit_length()
    ds = api.SeedStack(D, [api.SeedNode(D, 0, bytes(range(16)))])
    parts, e_hat = verifier.agg_ekeys(cfg, batches, ds, 1)
    ref = _oracle_etilde(suite, batches, ds)
    assert [p[1] for p in parts] == ref
    assert e_hat == O.sum_scalars(ref)


@pytest.mark.parametrize("suite", [1, 2, 3])
def test_ragged_batches_match_oracle(verifier, suite):
    """Variable-length entries (incl. empty ones) and uneven epoch sizes."""
    cfg, batches, ds = _synthetic(suite, 24, 40, 0, seed=77 + suite, ragged=True)
    rng = random.Random(suite)
    for i in list(batches)[::3]:
        batches[i] = batches[i][:rng.randint(0, len(batches[i]))]  # uneven / empty epochs
    parts, e_hat = verifier.agg_ekeys(cfg, batches, ds, 1)
    ref = _oracle_etilde(suite, batches, ds)
    assert [p[1] for p in parts] == ref
    assert e_hat == O.sum_scalars(ref)


def test_sparse_epoch_query(verifier):
    """Queried epochs need not be contiguous (map keys)."""
    cfg, batches, ds = _synthetic(1, 64, 32, 32, seed=5)
    sub = {i: batches[i] for i in (0, 3, 17, 40, 63)}
    parts, e_hat = verifier.agg_ekeys(cfg, sub, ds, 1)
    assert [p[1] for p in parts] == _oracle_etilde(1, sub, ds)


def test_empty_batch(verifier):
    cfg, batches, ds = _synthetic(1, 4, 4, 32, seed=1)
    parts, e_hat = verifier.agg_ekeys(cfg, {}, ds, 1)
    assert parts == [] and e_hat == bytes(32)


# ------------------------------------------------------------------ error taxonomy and order
def test_errors_follow_reference_order(verifier):
    api = A()
    st = Stream(load_golden("stream_s1_tamper.json"))
    suite, pk, ds = st.api_objects()
    # workers == 0 -> StateError (batch_verify.cpp:15, test_batch_verify.cpp:66-73)
    with pytest.raises(api.StateError):
        verifier.agg_ekeys(suite, st.batches, ds, 0)
    with pytest.raises(api.StateError):
        verifier.paver(pk, st.batches, st.s_hat, None, ds, 0)
    # undisclosed epoch -> SeedNotDisclosed naming it (test_batch_verify.cpp:75-80)
    b2 = dict(st.batches)
    b2[40] = b2[0]
    b2[35] = b2[1]
    with pytest.raises(api.SeedNotDisclosed) as ei:
        verifier.agg_ekeys(suite, b2, ds, 4)
    assert ei.value.epoch == 35  # lowest, as with workers == 1
    # batch size != n2 -> StateError before anything else (batch_verify.cpp:68-70)
    b3 = dict(b2)
    b3[2] = b3[2][:-1]
    with pytest.raises(api.StateError):
        verifier.paver(pk, b3, st.s_hat, None, ds, 1)
    # missing commitment -> StateError (batch_verify.cpp:76-79)
    pk2 = api.PoslocPublicKey(pk.suite, pk.y, {k: v for k, v in pk.r_hats.items() if k != 7})
    with pytest.raises(api.StateError):
        verifier.paver(pk2, st.batches, st.s_hat, None, ds, 1)
    # ... but not with an aggregate commitment
    assert verifier.paver(pk2, st.batches, st.s_hat, st.r_hat_agg, ds, 1) is False


def test_suite3_format_error_vs_seed_error_order(verifier):
    api = A()
    cfg, batches, ds = _synthetic(3, 4, 4, 16, seed=3)
    ds = api.SeedStack(ds.capacity, [api.SeedNode(1, 0, ds.nodes[0].value)])  # covers epochs 0,1
    bad = dict(batches)
    bad[1] = [bad[1][0] + bytes(20)] + bad[1][1:]  # 36-byte entry in epoch 1
    with pytest.raises(api.FormatError):
        verifier.agg_ekeys(cfg, bad, ds, 1)  # epoch 1 hashing error before epoch 2's seed error
    ok = dict(batches)
    ok[3] = [ok[3][0] + bytes(20)] + ok[3][1:]
    with pytest.raises(api.SeedNotDisclosed) as ei:
        verifier.agg_ekeys(cfg, ok, ds, 1)  # epoch 2 undisclosed wins over epoch 3
    assert ei.value.epoch == 2


def test_device_reports_launches(verifier):
    st = Stream(load_golden("stream_s1_n256.json"))
    suite, pk, ds = st.api_objects()
    verifier.paver(pk, st.batches, st.s_hat, None, ds, 1)
    assert verifier.last_launches() >= 4


# ------------------------------------------------------------------ K0 dense/sparse seed paths
@pytest.mark.parametrize("suite", [1, 2])
def test_seed_derivation_dense_and_sparse_stacks(verifier, suite):
    """Grouped (8 aligned consecutive epochs under one node) and per-epoch
    paths of K0 against the oracle's sr, over a multi-node stack."""
    api = A()
    rng = random.Random(suite)
    vals = [bytes(rng.getrandbits(8) for _ in range(16)) for _ in range(4)]
    # D = 6: nodes cover [0,32) depth 5, [32,48) depth 4, [48,50) depth 1, [50,51) depth 0
    ds = api.SeedStack(6, [api.SeedNode(5, 0, vals[0]), api.SeedNode(4, 2, vals[1]),
                           api.SeedNode(1, 24, vals[2]), api.SeedNode(0, 50, vals[3])])
    w = ds.serialize()
    for epochs in (list(range(51)), list(range(8, 48)), [0, 2, 3, 9, 16, 17, 18, 19, 20, 21, 22, 23, 49, 50],
                   list(range(40, 51))):
        got = verifier.seed_retrieve(suite, ds, epochs)
        for q, g in zip(epochs, got):
            st, ref = O.sr(suite, w, 6, q)
            assert st == 0 and g == ref, (epochs, q)
    with pytest.raises(api.SeedNotDisclosed) as ei:
        verifier.seed_retrieve(suite, ds, list(range(40, 56)))
    assert ei.value.epoch == 51


def test_chunked_host_path_matches_device_resident(verifier):
    """A host-resident log > 128 MiB streams in 64 MiB chunks on a copy
    stream (from pinned memory directly, from pageable memory through the
    pinned staging ring); results must equal the device-resident call bit for
    bit."""
    import ctypes

    import torch
    from paper_2506_08781_b200 import _native as N
    api = A()
    n2, L, n1 = 256, 32, 1 << 14  # 2^22 entries, 128 MiB
    n = n1 * n2
    rng = np.random.default_rng(9)
    host = torch.from_numpy(rng.integers(0, 256, size=n * L, dtype=np.uint8)).pin_memory()
    dev = host.cuda()
    root = bytes(range(16))
    ds = api.SeedStack(14, [api.SeedNode(14, 0, root)])
    dsb = ds.serialize()
    dsbuf = ctypes.create_string_buffer(dsb, len(dsb))
    epochs = np.arange(n1, dtype=np.uint32)

    def run(ptr, resident):
        b = N.PosloBatch()
        b.suite, b.n2, b.payload, b.payload_bytes = 1, n2, ptr, n * L
        b.offsets, b.entry_len, b.n_entries = None, L, n
        b.epochs, b.epoch_starts, b.n_epochs = epochs.ctypes.data, None, n1
        b.ds, b.ds_len, b.ds_capacity, b.device_resident = ctypes.addressof(dsbuf), len(dsb), 14, resident
        et = ctypes.create_string_buffer(n1 * 32)
        eh = ctypes.create_string_buffer(32)
        err = N.PosloError()
        assert verifier._lib.poslo_gpu_agg_ekeys(verifier._ctx, ctypes.byref(b), et, eh, ctypes.byref(err)) == 0
        return et.raw, eh.raw

    et_h, eh_h = run(host.data_ptr(), 0)
    et_d, eh_d = run(dev.data_ptr(), 1)
    assert et_h == et_d and eh_h == eh_d
    # the same log in PAGEABLE host memory: staged through the pinned ring by host copies
    pageable = host.numpy().copy()
    et_p, eh_p = run(pageable.ctypes.data, 0)
    assert et_p == et_d and eh_p == eh_d
    # sampled epochs against the oracle
    for k in (0, 1, 4097, n1 - 1):
        ents = [bytes(host[(k * n2 + j) * L:(k * n2 + j + 1) * L].numpy()) for j in range(n2)]
        ref = _oracle_etilde(1, {k: ents}, ds)
        assert et_h[32 * k:32 * k + 32] == ref[0]


@pytest.mark.parametrize("n2", [65, 100, 128, 129, 200, 256])
def test_multi_epoch_tiles_match_oracle(verifier, n2):
    """Small epochs (n2 <= 256) run several epochs per CTA (k_hash_s1_l32m),
    including a partial last CTA."""
    cfg, batches, ds = _synthetic(1, 37, n2, 32, seed=n2)
    parts, e_hat = verifier.agg_ekeys(cfg, batches, ds, 1)
    ref = _oracle_etilde(1, batches, ds)
    assert [p[1] for p in parts] == ref
    assert e_hat == O.sum_scalars(ref)


def test_device_resident_signatures_match_host(verifier):
    """epoch_verify / distill_coarse with a device-resident batch take the
    per-epoch signature arrays from HBM too; verdicts equal the host path."""
    import ctypes

    import torch
    from paper_2506_08781_b200 import _native as N
    from conftest import load_golden
    from golden_util import Stream
    api = A()
    st = Stream(load_golden("stream_s1_tamper.json"))
    suite, pk, ds = st.api_objects()
    s_hats = {i: st.sigs[i].s_hat_le for i in range(st.n1)}
    host_verdicts = verifier.epoch_verify(pk, st.batches, s_hats, ds)
    flat = b"".join(m for i in range(st.n1) for m in st.batches[i])
    pay = torch.frombuffer(bytearray(flat), dtype=torch.uint8).cuda()
    s_dev = torch.frombuffer(bytearray(b"".join(s_hats[i] for i in range(st.n1))), dtype=torch.uint8).cuda()
    r_dev = torch.frombuffer(bytearray(b"".join(pk.r_hats[i] for i in range(st.n1))), dtype=torch.uint8).cuda()
    dsb = ds.serialize()
    dsbuf = ctypes.create_string_buffer(dsb, len(dsb))
    epochs = np.arange(st.n1, dtype=np.uint32)
    b = N.PosloBatch()
    b.suite, b.n2, b.payload, b.payload_bytes = 1, st.n2, pay.data_ptr(), len(flat)
    b.offsets, b.entry_len, b.n_entries = None, 32, st.n1 * st.n2
    b.epochs, b.epoch_starts, b.n_epochs = epochs.ctypes.data, None, st.n1
    b.ds, b.ds_len, b.ds_capacity, b.device_resident = ctypes.addressof(dsbuf), len(dsb), ds.capacity, 1
    verd = ctypes.create_string_buffer(st.n1)
    verifier._call(verifier._lib.poslo_gpu_epoch_verify, ctypes.byref(b), pk.y, ctypes.c_void_p(s_dev.data_ptr()),
                   ctypes.c_void_p(r_dev.data_ptr()), verd, None)
    assert [bool(x) for x in verd.raw] == host_verdicts
    seg = np.array([0, 5, st.n1], dtype=np.uint32)
    so, ro = ctypes.create_string_buffer(64), ctypes.create_string_buffer(64)
    verifier._call(verifier._lib.poslo_gpu_distill_coarse, ctypes.byref(b), pk.y, ctypes.c_void_p(s_dev.data_ptr()),
                   ctypes.c_void_p(r_dev.data_ptr()), ctypes.c_void_p(seg.ctypes.data), 2, verd, so, ro)
    assert [bool(x) for x in verd.raw] == host_verdicts


def test_epochs_must_ascend(verifier):
    """A C-ABI misuse (epochs not strictly ascending) is rejected even though
    the check runs after the kernels are queued."""
    api = A()
    cfg, batches, ds = _synthetic(1, 8, 4, 32, seed=3)
    pb = api.PackedBatch(1, 4, batches, ds)
    pb.epochs = pb.epochs[[0, 2, 1, 3, 4, 5, 6, 7]].copy()
    cb = pb.cstruct()
    out = __import__("ctypes").create_string_buffer(32 * 8)
    with pytest.raises(ValueError, match="ascending"):
        verifier._call(verifier._lib.poslo_gpu_agg_ekeys, __import__("ctypes").byref(cb), out, None)
    pb.epochs = pb.epochs[[0, 1, 2, 3, 4, 5, 7, 7]].copy()  # last - first == n - 1 but a repeat
    cb = pb.cstruct()
    with pytest.raises(ValueError, match="ascending"):
        verifier._call(verifier._lib.poslo_gpu_agg_ekeys, __import__("ctypes").byref(cb), out, None)


def test_chunked_varlen_host_path_matches_device_resident(verifier):
    """Variable-length host-resident logs stream in epoch-aligned chunks cut
    by byte offsets; e~ must equal the device-resident call bit for bit."""
    import ctypes

    import torch
    from paper_2506_08781_b200 import synth as bench
    from paper_2506_08781_b200 import _native as N
    api = A()
    n2, n = 1024, 1 << 18  # ~143 MB of syslog-style entries: > 2 chunks
    n1 = n // n2
    lens = bench.synth_varlen(5, 0, n)
    offs = np.zeros(n + 1, dtype=np.uint64)
    np.cumsum(lens, out=offs[1:])
    offs_dev = torch.from_numpy(offs.view(np.int64)).cuda()
    dev = torch.empty(int(offs[-1]), dtype=torch.uint8, device="cuda")
    err = N.PosloError()
    assert verifier._lib.poslo_gpu_synth_varlog(verifier._ctx, 5, 0, n, ctypes.c_void_p(offs_dev.data_ptr()),
                                                ctypes.c_void_p(dev.data_ptr()), ctypes.byref(err)) == 0
    host = dev.cpu().pin_memory()
    ds = api.SeedStack(8, [api.SeedNode(8, 0, bytes(range(16)))])
    dsb = ds.serialize()
    dsbuf = ctypes.create_string_buffer(dsb, len(dsb))
    epochs = np.arange(n1, dtype=np.uint32)

    def run(ptr, off_ptr, resident):
        b = N.PosloBatch()
        b.suite, b.n2, b.payload, b.payload_bytes = 1, n2, ptr, int(offs[-1])
        b.offsets, b.entry_len, b.n_entries = off_ptr, 0, n
        b.epochs, b.epoch_starts, b.n_epochs = epochs.ctypes.data, None, n1
        b.ds, b.ds_len, b.ds_capacity, b.device_resident = ctypes.addressof(dsbuf), len(dsb), 8, resident
        et = ctypes.create_string_buffer(n1 * 32)
        eh = ctypes.create_string_buffer(32)
        verifier._call(verifier._lib.poslo_gpu_agg_ekeys, ctypes.byref(b), et, eh)
        return et.raw, eh.raw

    a = run(dev.data_ptr(), offs_dev.data_ptr(), 1)
    h = run(host.data_ptr(), offs.ctypes.data, 0)
    assert a == h


@pytest.mark.parametrize("comb16", [False, "sqrt", "decode", "encode", "split"])
@pytest.mark.parametrize("resident", [0, 1])
def test_batched_epoch_checks_large(verifier, resident, comb16, monkeypatch):
    """> 1024 per-epoch checks take the split path (R-hat decoded on a side
    stream; device-resident batches also pipeline the checks behind the
    hashing): signatures from the reference derivation (signer.py) verify, and
    exactly the tampered epochs fail — on the radix-256 combs (8 lanes per
    check) and (POSLO_COMB16_MIN = 1) on the radix-2^16 combs large batches
    take by default, in each check form (POSLO_CHECK16): no square root per
    check (sqrt, the default), a thread per check against decoded R-hat
    (decode), encoding compare (encode), 8 lanes per check (split). Device-resident batches also run
    distill_coarse (whose checks always use the decoded R-hat)."""
    monkeypatch.setenv("POSLO_COMB16_MIN", "1" if comb16 else "4294967295")
    if comb16:
        monkeypatch.setenv("POSLO_CHECK16", comb16)
    import ctypes

    import torch
    from paper_2506_08781_b200 import _native as N
    from paper_2506_08781_b200 import signer
    api = A()
    n1, n2 = 4096, 4  # 4096 one-epoch tiles: two pipelined pieces of kPipeMinTiles (capi.cu)
    suite = api.SuiteConfig(1, n1, n2, 8)
    rng = random.Random(41)
    sk = signer.PoslocSecretKey(suite, rng.randrange(1, O.L).to_bytes(32, "little"),
                                bytes(rng.getrandbits(8) for _ in range(16)),
                                bytes(rng.getrandbits(8) for _ in range(16)))
    batches = {i: [bytes(rng.getrandbits(8) for _ in range(32)) for _ in range(n2)] for i in range(n1)}
    pk = signer.kg_public_key(sk, verifier)
    s_hats = signer.sign_epochs(sk, batches, verifier)
    bad = {5, 1024, 2047, 4095}
    for i in bad:
        m = bytearray(batches[i][1])
        m[0] ^= 1
        batches[i][1] = bytes(m)
    ds = sk.root_stack()
    if not resident:
        got = verifier.epoch_verify(pk, batches, s_hats, ds)
    else:
        flat = b"".join(m for i in range(n1) for m in batches[i])
        pay = torch.frombuffer(bytearray(flat), dtype=torch.uint8).cuda()
        s_dev = torch.frombuffer(bytearray(b"".join(s_hats[i] for i in range(n1))), dtype=torch.uint8).cuda()
        r_dev = torch.frombuffer(bytearray(b"".join(pk.r_hats[i] for i in range(n1))), dtype=torch.uint8).cuda()
        dsb = ds.serialize()
        dsbuf = ctypes.create_string_buffer(dsb, len(dsb))
        epochs = np.arange(n1, dtype=np.uint32)
        b = N.PosloBatch()
        b.suite, b.n2, b.payload, b.payload_bytes = 1, n2, pay.data_ptr(), len(flat)
        b.offsets, b.entry_len, b.n_entries = None, 32, n1 * n2
        b.epochs, b.epoch_starts, b.n_epochs = epochs.ctypes.data, None, n1
        b.ds, b.ds_len, b.ds_capacity, b.device_resident = ctypes.addressof(dsbuf), len(dsb), ds.capacity, 1
        verd = ctypes.create_string_buffer(n1)
        verifier._call(verifier._lib.poslo_gpu_epoch_verify, ctypes.byref(b), pk.y, ctypes.c_void_p(s_dev.data_ptr()),
                       ctypes.c_void_p(r_dev.data_ptr()), verd, None)
        got = [bool(x) for x in verd.raw]
        seg = np.array([0, 1000, n1], dtype=np.uint32)
        dverd = ctypes.create_string_buffer(n1)
        so, ro = ctypes.create_string_buffer(64), ctypes.create_string_buffer(64)
        verifier._call(verifier._lib.poslo_gpu_distill_coarse, ctypes.byref(b), pk.y,
                       ctypes.c_void_p(s_dev.data_ptr()), ctypes.c_void_p(r_dev.data_ptr()),
                       ctypes.c_void_p(seg.ctypes.data), 2, dverd, so, ro)
        assert dverd.raw == verd.raw
        # umbrella folds of the valid epochs (the sqrt form folds its computed
        # points e Y + s B instead of decoding R-hat: the same group elements)
        for g in range(2):
            ok = [i for i in range(seg[g], seg[g + 1]) if verd.raw[i]]
            assert so.raw[32 * g:32 * g + 32] == verifier.scalar_sum([s_hats[i] for i in ok])
            assert ro.raw[32 * g:32 * g + 32] == verifier.group_fold([pk.r_hats[i] for i in ok])
    assert [i for i, ok in enumerate(got) if not ok] == sorted(bad)


@pytest.mark.parametrize("mode", ["sqrt", "decode", "encode", "split"])
def test_epoch_checks_on_adversarial_r_hats(verifier, mode, monkeypatch):
    """Per-epoch verdicts when R-hat_i is not the signer's commitment: the
    identity encoding, s = p (non-canonical), an odd (negative) s, bit 255
    set, and valid encodings of other points (including -R and R + one
    generator). Every form of the radix-2^16 check must reject exactly those
    epochs, as the reference's byte compare encode(e Y + s B) == R does."""
    monkeypatch.setenv("POSLO_COMB16_MIN", "1")
    monkeypatch.setenv("POSLO_CHECK16", mode)
    from paper_2506_08781_b200 import signer
    from oracle import ristretto as R
    api = A()
    n1, n2 = 2048, 2
    suite = api.SuiteConfig(1, n1, n2, 8)
    rng = random.Random(43)
    sk = signer.PoslocSecretKey(suite, rng.randrange(1, O.L).to_bytes(32, "little"),
                                bytes(rng.getrandbits(8) for _ in range(16)),
                                bytes(rng.getrandbits(8) for _ in range(16)))
    batches = {i: [bytes(rng.getrandbits(8) for _ in range(32)) for _ in range(n2)] for i in range(n1)}
    pk = signer.kg_public_key(sk, verifier)
    s_hats = signer.sign_epochs(sk, batches, verifier)
    gen = R.encode(R.BASE)
    def neg(enc):
        x, y, z, t = R.decode(enc)
        return R.encode(((-x) % R.P, y, z, (-t) % R.P))
    bad = {
        3: bytes(32),                                              # identity
        100: R.P.to_bytes(32, "little"),                           # s = p: non-canonical
        101: (R.P + 2).to_bytes(32, "little"),                     # s = p + 2: non-canonical
        777: (int.from_bytes(pk.r_hats[777], "little") | 1).to_bytes(32, "little"),  # odd s
        900: (int.from_bytes(pk.r_hats[900], "little") | (1 << 255)).to_bytes(32, "little"),  # bit 255
        1500: neg(pk.r_hats[1500]),                                # -R
        2047: R.group_combine(pk.r_hats[2047], gen),               # R + B
    }
    r_hats = dict(pk.r_hats)
    for i, r in bad.items():
        assert r != pk.r_hats[i]
        r_hats[i] = r
    pk2 = api.PoslocPublicKey(pk.suite, pk.y, r_hats)
    got = verifier.epoch_verify(pk2, batches, s_hats, sk.root_stack())
    assert [i for i, ok in enumerate(got) if not ok] == sorted(bad)


def test_device_resident_host_pointers_rejected(verifier):
    """A batch flagged device_resident that points at pageable host memory
    (payload, or the per-epoch signature arrays) is refused with
    INVALID_ARGUMENT instead of faulting in a kernel; the context keeps
    working afterwards."""
    import ctypes

    import torch
    from paper_2506_08781_b200 import _native as N
    api = A()
    cfg, batches, ds = _synthetic(1, 8, 64, 32, seed=3)
    flat = b"".join(m for i in range(8) for m in batches[i])
    host = np.frombuffer(flat, dtype=np.uint8).copy()
    dsb = ds.serialize()
    dsbuf = ctypes.create_string_buffer(dsb, len(dsb))
    epochs = np.arange(8, dtype=np.uint32)

    def batch(ptr):
        b = N.PosloBatch()
        b.suite, b.n2, b.payload, b.payload_bytes = 1, 64, ptr, len(flat)
        b.offsets, b.entry_len, b.n_entries = None, 32, 8 * 64
        b.epochs, b.epoch_starts, b.n_epochs = epochs.ctypes.data, None, 8
        b.ds, b.ds_len, b.ds_capacity, b.device_resident = ctypes.addressof(dsbuf), len(dsb), ds.capacity, 1
        return b

    et, eh = ctypes.create_string_buffer(8 * 32), ctypes.create_string_buffer(32)
    with pytest.raises(ValueError, match="host pointer"):
        verifier._call(verifier._lib.poslo_gpu_agg_ekeys, ctypes.byref(batch(host.ctypes.data)), et, eh)
    dev = torch.frombuffer(bytearray(flat), dtype=torch.uint8).cuda()
    bd = batch(dev.data_ptr())
    Y = verifier.exp_base((5).to_bytes(32, "little"))
    s = ctypes.create_string_buffer(8 * 32)
    r = ctypes.create_string_buffer(b"".join([Y] * 8), 8 * 32)
    verd = ctypes.create_string_buffer(8)
    with pytest.raises(ValueError, match="host signature arrays"):
        verifier._call(verifier._lib.poslo_gpu_epoch_verify, ctypes.byref(bd), Y, s, r, verd, None)
    verifier._call(verifier._lib.poslo_gpu_agg_ekeys, ctypes.byref(bd), et, eh)  # still healthy
    parts, _ = verifier.agg_ekeys(cfg, batches, ds, 1)
    assert [p[1] for p in parts] == [et.raw[32 * k:32 * k + 32] for k in range(8)]
