"""ristretto255 restated in pure Python big integers — test infrastructure only.

Restates the group the reference uses through libsodium 1.0.20 (third-party,
absent from /root/reference): proj/src/group.cpp:107-178 calls
`crypto_core_ristretto255_is_valid_point`, `crypto_scalarmult_ristretto255`,
`crypto_scalarmult_ristretto255_base` and `crypto_core_ristretto255_add`.
The algorithms follow the published ristretto255 definition (RFC 9496 §4.3:
decode, encode, SQRT_RATIO_M1, equality) over edwards25519 in extended
twisted-Edwards coordinates. Constants are derived from their definitions,
not typed in. Pinned by tests/test_oracle.py against golden vectors produced
by the reference (tests/golden/kat.json: generator, exp_base, commit_check,
group_combine, point validity).

Semantics reproduced from group.cpp: scalars are canonical little-endian;
libsodium reports an identity result as failure and the reference maps that
to the identity encoding (32 zero bytes), so commit_check(Y, e, s) is exactly
encode(e*Y + s*B) (group.cpp:144-167).
"""
from __future__ import annotations

P = 2**255 - 19
L = 2**252 + 27742317777372353535851937790883648493
D = (-121665 * pow(121666, P - 2, P)) % P
SQRT_M1 = pow(2, (P - 1) // 4, P)


def _is_neg(x: int) -> bool:
    return (x % P) & 1 == 1


def _abs(x: int) -> int:
    x %= P
    return (P - x) % P if _is_neg(x) else x


def sqrt_ratio_m1(u: int, v: int):
    """RFC 9496 §4.2 SQRT_RATIO_M1: (was_square, non-negative root)."""
    u %= P
    v %= P
    v3 = v * v % P * v % P
    v7 = v3 * v3 % P * v % P
    r = u * v3 % P * pow(u * v7 % P, (P - 5) // 8, P) % P
    check = v * r % P * r % P
    correct = check == u
    flipped = check == (-u) % P
    flipped_i = check == (-u * SQRT_M1) % P
    if flipped or flipped_i:
        r = r * SQRT_M1 % P
    return (correct or flipped), _abs(r)


# 1/sqrt(a - d) with a = -1, chosen non-negative (RFC 9496 §4.1 constants)
INVSQRT_A_MINUS_D = sqrt_ratio_m1(1, (-1 - D) % P)[1]

IDENTITY = (0, 1, 1, 0)


def decode(b: bytes):
    """RFC 9496 §4.3.1; returns extended point or None (invalid encoding)."""
    if len(b) != 32:
        return None
    s = int.from_bytes(b, "little")
    if s >= P or _is_neg(s):
        return None
    ss = s * s % P
    u1 = (1 - ss) % P
    u2 = (1 + ss) % P
    u2_sqr = u2 * u2 % P
    v = (-(D * u1 % P * u1) - u2_sqr) % P
    was_square, invsqrt = sqrt_ratio_m1(1, v * u2_sqr % P)
    den_x = invsqrt * u2 % P
    den_y = invsqrt * den_x % P * v % P
    x = _abs(2 * s * den_x)
    y = u1 * den_y % P
    t = x * y % P
    if not was_square or _is_neg(t) or y == 0:
        return None
    return (x, y, 1, t)


def encode(pt) -> bytes:
    """RFC 9496 §4.3.2."""
    x0, y0, z0, t0 = pt
    u1 = (z0 + y0) * (z0 - y0) % P
    u2 = x0 * y0 % P
    _, invsqrt = sqrt_ratio_m1(1, u1 * u2 % P * u2 % P)
    den1 = invsqrt * u1 % P
    den2 = invsqrt * u2 % P
    z_inv = den1 * den2 % P * t0 % P
    ix0 = x0 * SQRT_M1 % P
    iy0 = y0 * SQRT_M1 % P
    enchanted = den1 * INVSQRT_A_MINUS_D % P
    rotate = _is_neg(t0 * z_inv)
    if rotate:
        x, y, den_inv = iy0, ix0, enchanted
    else:
        x, y, den_inv = x0, y0, den2
    if _is_neg(x * z_inv):
        y = (-y) % P
    s = _abs(den_inv * (z0 - y))
    return s.to_bytes(32, "little")


def add(p1, p2):
    """Extended-coordinate addition on -x^2 + y^2 = 1 + d x^2 y^2 (a = -1)."""
    x1, y1, z1, t1 = p1
    x2, y2, z2, t2 = p2
    a = (y1 - x1) * (y2 - x2) % P
    b = (y1 + x1) * (y2 + x2) % P
    c = t1 * 2 * D % P * t2 % P
    d = z1 * 2 * z2 % P
    e, f, g, h = (b - a) % P, (d - c) % P, (d + c) % P, (b + a) % P
    return (e * f % P, g * h % P, f * g % P, e * h % P)


def scalarmult(k: int, pt):
    acc = IDENTITY
    for bit in bin(k)[2:] if k else "":
        acc = add(acc, acc)
        if bit == "1":
            acc = add(acc, pt)
    return acc


def _base():
    y = 4 * pow(5, P - 2, P) % P
    # x^2 = (y^2 - 1) / (d y^2 + 1), pick the even root
    num = (y * y - 1) % P
    den = (D * y * y + 1) % P
    ok, x = sqrt_ratio_m1(num, den)
    assert ok
    return (x, y, 1, x * y % P)


BASE = _base()


def equal(p1, p2) -> bool:
    x1, y1, _, _ = p1
    x2, y2, _, _ = p2
    return (x1 * y2 - y1 * x2) % P == 0 or (y1 * y2 - x1 * x2) % P == 0


# ---- the reference's group API (group.cpp) over 32-byte encodings ---------

def is_valid_point(b: bytes) -> bool:
    return decode(b) is not None


def exp_base(s_le: bytes) -> bytes:
    return encode(scalarmult(int.from_bytes(s_le, "little"), BASE))


def exp(base: bytes, s_le: bytes) -> bytes:
    pt = decode(base)
    assert pt is not None
    return encode(scalarmult(int.from_bytes(s_le, "little"), pt))


def commit_check(y: bytes, e_le: bytes, s_le: bytes) -> bytes:
    """Y^e * alpha^s (group.cpp:144-167)."""
    yp = decode(y)
    assert yp is not None
    acc = add(scalarmult(int.from_bytes(e_le, "little"), yp),
              scalarmult(int.from_bytes(s_le, "little"), BASE))
    return encode(acc)


def group_combine(a: bytes, b: bytes) -> bytes:
    """group.cpp:169-178."""
    pa, pb = decode(a), decode(b)
    assert pa is not None and pb is not None
    return encode(add(pa, pb))
