"""The device math headers (paper_2506_08781_b200/csrc/*.cuh) compiled for the
host by tests/native/devmath_host.cpp, checked against the pinned oracle and
the reference's golden vectors. Catches arithmetic bugs before GPU time; the
GPU parity tests re-check the same on the device. CPU only."""
import ctypes
import os
import random
import subprocess

import pytest

from oracle import oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "tests", "native", "devmath_host.cpp")
LIB = os.path.join(ROOT, "tests", "native", "build", "libdevmath_host.so")


@pytest.fixture(scope="module")
def dm():
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    subprocess.check_call(["g++", "-std=c++17", "-O2", "-fPIC", "-shared", "-Wno-unknown-pragmas",
                           "-o", LIB, SRC])
    return ctypes.CDLL(LIB)


def out(n):
    return ctypes.create_string_buffer(n)


@pytest.mark.parametrize("suite", [1, 2, 3])
def test_prf(dm, kat, suite):
    x0 = bytes(range(16))
    for bit, key in ((0, "prf0"), (1, "prf1")):
        o = out(16)
        dm.dm_prf(suite, bit, x0, o)
        assert o.raw.hex() == kat[f"suite{suite}"][key]


@pytest.mark.parametrize("suite", [1, 2, 3])
def test_entry_generic(dm, suite):
    rng = random.Random(suite)
    for t in range(200):
        L = rng.randint(1, 31) if suite == 3 else rng.choice([0, 1, 15, 16, 17, 31, 32, 33, 47, 48, 55, 56,
                                                              63, 64, 100, 200, rng.randint(0, 300)])
        m = bytes(rng.getrandbits(8) for _ in range(L))
        x0 = bytes(rng.getrandbits(8) for _ in range(16))
        j = t if t < 8 else rng.getrandbits(32)
        o = out(32)
        assert dm.dm_entry_generic(suite, m, L, x0, j, o, None) == 0
        assert o.raw == O.hash_to_scalar(suite, m, O.onetime_seed(suite, x0, j))
    if suite == 3:
        assert dm.dm_entry_generic(3, bytes(32), 32, bytes(16), 0, out(32), None) == 1


@pytest.mark.parametrize("suite", [1, 2])
def test_entry_fast32_and_deferred_sum(dm, suite):
    rng = random.Random(10 + suite)
    n = 64
    limbs = (ctypes.c_uint32 * (16 * n))()
    ref = bytes(32)
    for t in range(n):
        m = bytes(rng.getrandbits(8) for _ in range(32))
        x0 = bytes(rng.getrandbits(8) for _ in range(16))
        j = rng.getrandbits(32)
        one = (ctypes.c_uint32 * 16)()
        dm.dm_entry_fast32(suite, m, x0, j, one)
        for k in range(16):
            limbs[16 * t + k] = one[k]
        ref = O.sc_add(ref, O.hash_to_scalar(suite, m, O.onetime_seed(suite, x0, j)))
    o = out(32)
    dm.dm_sum_reduce(limbs, n, o)
    assert o.raw == ref  # sum of raw digests reduced once == sum of reductions


@pytest.mark.parametrize("mode", [0, 1, 2, 3, 4, 5, 6, 7])
def test_sha_pipe_balance_modes(dm, mode):
    rng = random.Random(20 + mode)
    for t in range(64):
        m = bytes(rng.getrandbits(8) for _ in range(32))
        x0 = bytes(rng.getrandbits(8) for _ in range(16))
        j = rng.getrandbits(32) if t else 0
        limbs = (ctypes.c_uint32 * 16)()
        dm.dm_entry_s1_mode(mode, m, x0, j, limbs)
        o = out(32)
        dm.dm_sum_reduce(limbs, 1, o)
        assert o.raw == O.hash_to_scalar(1, m, O.onetime_seed(1, x0, j))


def test_ots_specialised_schedule(dm):
    # the lean kernel's onetime_seed: per-epoch constants + reduced schedule W16..W31
    rng = random.Random(77)
    for t in range(200):
        x0 = bytes(rng.getrandbits(8) for _ in range(16))
        j = [0, 1, 255, 1023, 0xFFFFFFFF][t] if t < 5 else rng.getrandbits(32)
        o = out(16)
        dm.dm_ots_spec(x0, j, o)
        assert o.raw == O.onetime_seed(1, x0, j)


def test_deferred_sum_worst_case(dm):
    # all-ones digests maximise carries through the 17-limb accumulator
    n = 4096
    limbs = (ctypes.c_uint32 * (16 * n))(*([0xFFFFFFFF] * (16 * n)))
    o = out(32)
    dm.dm_sum_reduce(limbs, n, o)
    assert int.from_bytes(o.raw, "little") == (n * (2**512 - 1)) % O.L


def test_scalar_ops(dm, kat):
    for w, r in kat["reduce_wide_be"]:
        o = out(32)
        dm.dm_reduce_wide_be(bytes.fromhex(w), o)
        assert o.raw.hex() == r
    for a, b, c, _ in kat["scalar_add"]:
        o = out(32)
        dm.dm_sc_add(bytes.fromhex(a), bytes.fromhex(b), o)
        assert o.raw.hex() == c


def test_group_ops(dm, kat):
    for Y, e, s, P in kat["commit_check"]:
        o = out(32)
        assert dm.dm_commit_check(bytes.fromhex(Y), bytes.fromhex(e), bytes.fromhex(s), o) == 0
        assert o.raw.hex() == P
    for Y, e, s, P in kat["commit_check"][:16]:
        o = out(32)
        assert dm.dm_commit_check_comb(bytes.fromhex(Y), bytes.fromhex(e), bytes.fromhex(s), o) == 0
        assert o.raw.hex() == P
    for p, v in kat["point_valid"]:
        assert dm.dm_point_valid(bytes.fromhex(p)) == v
    # split check (paver): e*Y == R - s*B  <=>  encode(e*Y + s*B) == R
    rows = kat["commit_check"][:12]
    for i, (Y, e, s, P) in enumerate(rows):
        Yb, eb, sb, Pb = (bytes.fromhex(x) for x in (Y, e, s, P))
        assert dm.dm_check_split(Yb, eb, sb, Pb) == 1
        other = bytes.fromhex(rows[(i + 1) % len(rows)][3])
        assert dm.dm_check_split(Yb, eb, sb, other) == int(other == Pb)
        assert dm.dm_check_split(Yb, eb, sb, b"\xff" * 32) == 0  # invalid R never verifies
    for a, b, c in kat["group_combine"]:
        o = out(32)
        assert dm.dm_fold(2, bytes.fromhex(a) + bytes.fromhex(b), o) == 0
        assert o.raw.hex() == c


def test_square_root_free_check_host(dm, kat):
    """ristretto.cuh rist_encoding_matches (the device's per-epoch verdict with
    no square root) compiled for the CPU: accepts exactly the reference's
    commit_check encoding, incl. e = s = 0 (the identity), and rejects other
    points' encodings, negated / non-canonical / bit-255 variants."""
    rows = kat["commit_check"]
    P = 2**255 - 19
    for i, (Y, e, s, Pk) in enumerate(rows):
        Yb, eb, sb, Pb = (bytes.fromhex(x) for x in (Y, e, s, Pk))
        assert dm.dm_check_sqrtfree(Yb, eb, sb, Pb) == 1
        v = int.from_bytes(Pb, "little")
        wrongs = [bytes.fromhex(rows[(i + 1) % len(rows)][3]), ((P - v) % P).to_bytes(32, "little"),
                  (v | (1 << 255)).to_bytes(32, "little"), (v ^ 4).to_bytes(32, "little")]
        if v + P < 2**256:
            wrongs.append((v + P).to_bytes(32, "little"))
        for w in wrongs:
            if w != Pb:
                assert dm.dm_check_sqrtfree(Yb, eb, sb, w) == 0
    Y0 = bytes.fromhex(rows[0][0])
    assert dm.dm_check_sqrtfree(Y0, bytes(32), bytes(32), bytes(32)) == 1  # identity encodes to 0
    assert dm.dm_check_sqrtfree(Y0, bytes(32), bytes(32), bytes.fromhex(rows[0][3])) == int(
        bytes.fromhex(rows[0][3]) == bytes(32))


def test_signer_math_matches_reference_keys(dm):
    """kg / sig_epoch on the device math: R-hat_i =
    alpha^(sum_j nonce_to_scalar(r, i, j)) equals the reference's public key,
    and s-hat_i = r-hat_i - y e~_i its epoch signatures (untampered epochs)."""
    import json
    import os
    import struct
    from conftest import GOLDEN
    from golden_util import Stream
    for name in ("stream_s1_tamper", "stream_s2_mixed", "stream_s3_mixed"):
        g = json.load(open(os.path.join(GOLDEN, name + ".json")))
        st = Stream(g)
        sk = bytes.fromhex(g["sk"])
        assert sk[:4] == b"PSKC"
        y_le = sk[17:49][::-1]
        r = sk[49:65]
        for i in range(st.n1):
            o = out(32)
            dm.dm_nonce_sum(st.suite, r, i, st.n2, o)
            assert O.ristretto.exp_base(o.raw) == st.pk.r_hats[i], (name, i)
            if g["epoch_verdicts"][i]:
                s = out(32)
                dm.dm_sc_mul_sub(o.raw, y_le, st.e_tilde[i], s)
                assert s.raw == st.sigs[i].s_hat_le, (name, i)


def test_scalar_mul_sub(dm):
    rng = random.Random(99)
    for t in range(200):
        r, y, e = (rng.randrange(O.L) for _ in range(3))
        if t == 0:
            r, y, e = 0, O.L - 1, O.L - 1
        o = out(32)
        dm.dm_sc_mul_sub(r.to_bytes(32, "little"), y.to_bytes(32, "little"), e.to_bytes(32, "little"), o)
        assert int.from_bytes(o.raw, "little") == (r - y * e) % O.L


def test_field_arithmetic_radix_25_5(dm):
    """GF(2^255-19) in radix 2^25.5 (ristretto.cuh) against Python integers:
    canonical inputs, the top of the range (p - 1, 2^255 - 1 reduced), and
    long mixed chains that keep every intermediate in lazy (carried) form."""
    P = 2**255 - 19
    rng = random.Random(2551)
    edge = [0, 1, 2, 19, P - 1, P - 2, P - 19, 2**255 - 20, 2**254, 2**26 - 1, 2**51, (2**255 - 1) % P]
    vals = edge + [rng.randrange(P) for _ in range(300)]
    fb = lambda v: v.to_bytes(32, "little")
    for t_ in range(400):
        a = vals[t_ % len(vals)]
        b = vals[(t_ * 7 + 3) % len(vals)]
        for op, ref in ((0, a * b % P), (1, a * a % P), (2, (a + b) % P), (3, (a - b) % P), (4, (-a) % P), (5, a)):
            o = out(32)
            dm.dm_fe_op(op, fb(a), fb(b), o)
            assert int.from_bytes(o.raw, "little") == ref, (op, a, b)
    # non-canonical 32-byte inputs (>= p, bit 255 ignored) reduce like the reference's field
    for v in (P, P + 1, 2**255 - 1):
        o = out(32)
        dm.dm_fe_op(5, fb(v), fb(0), o)
        assert int.from_bytes(o.raw, "little") == (v % 2**255) % P
    for t_ in range(20):
        a, b = rng.randrange(P), rng.randrange(P)
        x, y = a, b
        for _ in range(50):
            s, d = (x + y) % P, (x - y) % P
            x = s * d % P
            y = pow((y - 2 * s) % P, 2, P)
        o = out(32)
        dm.dm_fe_chain(fb(a), fb(b), 50, o)
        assert int.from_bytes(o.raw, "little") == (x + y) % P
