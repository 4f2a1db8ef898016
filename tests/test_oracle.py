"""Pins the CPU oracle (oracle/poslo_oracle.c + oracle/ristretto.py) against
the golden vectors produced by the UNMODIFIED reference (tests/golden) and
against external FIPS examples. CPU only."""
import hashlib

import numpy as np
import pytest

from conftest import STREAMS, load_golden
from golden_util import Stream
from oracle import oracle as O
from oracle import ristretto as R


def test_sha256_fips_examples():
    # FIPS 180-4 / NIST CSRC examples, and hashlib across block boundaries
    assert O.sha256(b"abc").hex() == "ba7816bf8f01cfea414140de5dae2223b00361a396177a9cb410ff61f20015ad"
    assert O.sha256(b"").hex() == "e3b0c44298fc1c149afbf4c8996fb92427ae41e4649b934ca495991b7852b855"
    for n in list(range(0, 140)) + [1000, 4095]:
        m = bytes((i * 7 + n) & 0xFF for i in range(n))
        assert O.sha256(m) == hashlib.sha256(m).digest()


def test_aes128_fips197_example():
    key = bytes.fromhex("000102030405060708090a0b0c0d0e0f")
    pt = bytes.fromhex("00112233445566778899aabbccddeeff")
    assert O.aes128(key, pt).hex() == "69c4e0d86a7b0430d8cdb78070b4c55a"
    key = bytes.fromhex("2b7e151628aed2a6abf7158809cf4f3c")
    pt = bytes.fromhex("3243f6a8885a308d313198a2e0370734")
    assert O.aes128(key, pt).hex() == "3925841d02dc09fbdc118597196a0b32"


@pytest.mark.parametrize("suite", [1, 2, 3])
def test_primitives_vs_reference(kat, suite):
    d = kat[f"suite{suite}"]
    x0 = bytes(range(16))
    assert O.prf(suite, 0, x0).hex() == d["prf0"]
    assert O.prf(suite, 1, x0).hex() == d["prf1"]
    assert O.onetime_seed(suite, x0, 0).hex() == d["ots0"]
    assert O.onetime_seed(suite, x0, 5).hex() == d["ots5"]
    for m, x, e in d["h2s"]:
        assert O.hash_to_scalar(suite, bytes.fromhex(m), bytes.fromhex(x)).hex() == e
    for x, j, o in d["ots"]:
        assert O.onetime_seed(suite, bytes.fromhex(x), j).hex() == o
    ds = bytes.fromhex(d["ds_after_11"])
    for i, v in enumerate(d["sr"]):
        assert O.sr(suite, ds, 4, i) == (0, bytes.fromhex(v))
    assert O.sr(suite, ds, 4, 12)[0] == O.SEED_NOT_DISCLOSED
    for m, h, h2 in d.get("mmo", []):
        assert O.mmo(bytes.fromhex(m)).hex() == h
        assert O.mdc2(bytes.fromhex(m)).hex() == h2


def test_appendix_c_anchors():
    # SURVEY.md Appendix C values (computed against the reference in the survey)
    x0 = bytes(range(16))
    assert O.prf(1, 0, x0).hex() == "23bb842412745468d897d75ec47aae60"
    assert O.onetime_seed(2, x0, 5).hex() == "6d14513dc062a1634206fe74ca63f8e8"
    assert O.reduce_wide_be(b"\xff" * 64).hex() == \
        "000f9c44e31106a447938568a71b0ed065bef517d273ecce3d9a307c1b419903"


def test_suite3_rejects_long_entries():
    with pytest.raises(ValueError):
        O.hash_to_scalar(3, bytes(32), bytes(16))


def test_scalars_vs_reference(kat):
    for w, r in kat["reduce_wide_be"]:
        assert O.reduce_wide_be(bytes.fromhex(w)).hex() == r
        assert int.from_bytes(bytes.fromhex(r), "little") == int.from_bytes(bytes.fromhex(w), "big") % O.L
    for a, b, c, _ in kat["scalar_add"]:
        assert O.sc_add(bytes.fromhex(a), bytes.fromhex(b)).hex() == c


def test_ristretto_vs_reference(kat):
    assert R.encode(R.BASE).hex() == kat["generator"]
    for s, p in kat["exp_base"]:
        assert R.exp_base(bytes.fromhex(s)).hex() == p
    for Y, e, s, P in kat["commit_check"][:12]:
        assert R.commit_check(bytes.fromhex(Y), bytes.fromhex(e), bytes.fromhex(s)).hex() == P
    for a, b, c in kat["group_combine"][:8]:
        assert R.group_combine(bytes.fromhex(a), bytes.fromhex(b)).hex() == c
    for p, v in kat["point_valid"]:
        assert R.is_valid_point(bytes.fromhex(p)) == bool(v)


@pytest.mark.parametrize("name", STREAMS)
def test_agg_ekeys_oracle_vs_reference(name):
    st = Stream(load_golden(name + ".json"))
    epochs = sorted(st.batches)
    flat = [m for i in epochs for m in st.batches[i]]
    lens = [len(m) for m in flat]
    offs = np.zeros(len(flat) + 1, dtype=np.uint64)
    np.cumsum(lens, out=offs[1:])
    starts = np.arange(len(epochs) + 1, dtype=np.uint64) * st.n2
    rc, _, et = O.agg_ekeys_packed(st.suite, b"".join(flat), offs, 0, epochs, starts, st.ds, st.depth)
    assert rc == 0
    assert et == st.e_tilde
    assert O.sum_scalars(et) == st.e_hat


@pytest.mark.parametrize("name", ["stream_s1_mixed", "stream_s2_mixed", "stream_s1_tamper"])
def test_group_check_oracle_vs_reference(name):
    """paver decision = (commit_check(Y, e^, s^) == fold of R_i) (batch_verify.cpp:64-87)."""
    st = Stream(load_golden(name + ".json"))
    r_fold = bytes(32)
    for i in sorted(st.pk.r_hats):
        r_fold = R.group_combine(r_fold, st.pk.r_hats[i])
    assert r_fold == st.r_hat_agg
    ok = R.commit_check(st.pk.y, st.e_hat, st.s_hat) == r_fold
    assert ok == bool(st.d["paver"]) == bool(st.d["aver"])


def _encoding_matches_by_squares(pt, r: bytes) -> bool:
    """The device's square-root-free check (ristretto.cuh rist_encoding_matches):
    every branch of RFC 9496 §4.3.2 depends only on z_inv = T / u2, and
    s = |invsqrt K| with invsqrt^2 = 1 / (u1 u2^2), so for a canonical
    non-negative s: encode(P) == r  <=>  s^2 u1 u2^2 == K^2."""
    P = R.P
    s = int.from_bytes(r, "little")
    if s >= P or s & 1:
        return False
    x0, y0, z0, t0 = pt
    u1 = (z0 + y0) * (z0 - y0) % P
    u2 = x0 * y0 % P
    if u2 == 0:
        return s == 0
    z_inv = t0 * pow(u2, P - 2, P) % P
    rotate = R._is_neg(t0 * z_inv)
    x, y = (y0 * R.SQRT_M1 % P, x0 * R.SQRT_M1 % P) if rotate else (x0, y0)
    k = u1 * R.INVSQRT_A_MINUS_D % P if rotate else u2
    if R._is_neg(x * z_inv):
        y = (-y) % P
    K = k * (z0 - y) % P
    return s * s % P * (u1 * u2 % P * u2) % P == K * K % P


def test_square_root_free_encoding_check_matches_encode():
    """The identity behind the square-root-free checks, on the oracle: for
    random multiples of the generator, their 4-torsion representatives and
    projective rescalings, the check accepts the point's encoding and rejects
    neighbours, other points, non-canonical and negative encodings."""
    import random
    rng = random.Random(2025)
    P = R.P
    torsion = [(0, 1, 1, 0), (0, P - 1, 1, 0), (R.SQRT_M1, 0, 1, 0), (P - R.SQRT_M1, 0, 1, 0)]
    for t in torsion:  # the identity class encodes to 0
        assert R.encode(t) == bytes(32) and _encoding_matches_by_squares(t, bytes(32))
    for it in range(150):
        pt = R.scalarmult(rng.randrange(1, R.L), R.BASE)
        if it % 3 == 1:
            pt = R.add(pt, torsion[rng.randrange(4)])
        if it % 4 == 2:
            z = rng.randrange(1, P)
            pt = tuple(c * z % P for c in pt)
        e = R.encode(pt)
        assert _encoding_matches_by_squares(pt, e)
        s = int.from_bytes(e, "little")
        for wrong in (bytes(32), (s ^ 2).to_bytes(32, "little"), ((P - s) % P).to_bytes(32, "little"),
                      (s + P).to_bytes(32, "little") if s + P < 2**256 else bytes(32),
                      R.encode(R.add(pt, R.BASE))):
            if wrong != e:
                assert not _encoding_matches_by_squares(pt, wrong)
