// AES-128 encryption with per-block key expansion, and the MMO / MDC-2
// constructions of suites 2/3 (primitives.cpp:13-19 aes128_block, :28-48
// 10* padding, :76-87 mmo_hash, :89-111 mdc2_hash).
//
// Layout: the 16-byte AES state / key / block is four little-endian packed
// "memory words" (byte 4c+r of the block = bits 8r..8r+7 of word c), which is
// exactly what a 32-bit load of the block from memory yields. Round function
// is the T-table formulation over ONE table T0 (bytes 2S,S,S,3S), the other
// three being byte rotations of it (or stored, see SmemT4). The table lives in shared memory
// replicated once per bank ([x][lane] layout, 32 KiB) so the 16 data-dependent
// lookups of a round never bank-conflict; S[x] is byte 1 of T0[x].
//
// The table is passed as a "lookup" functor so the same code runs from shared
// memory on the device and from a plain array in the host-side unit tests:
// lk(w, k) = T0[byte k of w], lkr(w, k, r) = rotl(T0[byte k of w], 8r).
#pragma once
#include "poslo_common.cuh"

PHD uint8_t aes_xtime(uint8_t a) { return (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1b : 0)); }

PHD uint8_t aes_gmul(uint8_t a, uint8_t b) {
    uint8_t p = 0;
    while (b) {
        if (b & 1) p ^= a;
        a = aes_xtime(a);
        b >>= 1;
    }
    return p;
}

// S-box from its definition (GF(2^8) inverse + affine map, FIPS-197 §5.1.1).
PHD uint8_t aes_sbox_compute(int x) {
    uint8_t inv = 0;
    if (x)
        for (int y = 1; y < 256; y++)
            if (aes_gmul((uint8_t)x, (uint8_t)y) == 1) {
                inv = (uint8_t)y;
                break;
            }
    uint8_t s = inv;
    for (int r = 1; r <= 4; r++) s ^= (uint8_t)((inv << r) | (inv >> (8 - r)));
    return (uint8_t)(s ^ 0x63);
}

// T0[x] = 2S | S << 8 | S << 16 | 3S << 24 (little-endian packed column)
PHD uint32_t aes_t0_entry(uint8_t s) {
    uint8_t s2 = aes_xtime(s), s3 = (uint8_t)(s2 ^ s);
    return (uint32_t)s2 | (uint32_t)s << 8 | (uint32_t)s << 16 | (uint32_t)s3 << 24;
}

PHD uint32_t rotl32(uint32_t x, int n) { return rotr32(x, (32 - n) & 31); }

PHD uint32_t byte_of(uint32_t x, int k) { return (x >> (8 * k)) & 0xffu; }

// Encrypts `in` under `key` (both 4 memory words); round keys are expanded
// on the fly alongside the rounds (MMO rekeys on every block).
// Byte assembly of the last round / SubWord: S[x] = byte 1 of T0[x]; picks
// byte 1 of each of four T0 values into bytes 0..3 (two PRMTs + one).
PHD uint32_t sbox4(uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
#ifdef __CUDA_ARCH__
    const uint32_t ab = __byte_perm(a, b, 0x0051u);  // bytes: a.1, b.1
    const uint32_t cd = __byte_perm(c, d, 0x0051u);  // bytes: c.1, d.1
    return __byte_perm(ab, cd, 0x5410u);
#else
    return ((a >> 8) & 0xffu) | (b & 0xff00u) | ((c << 8) & 0xff0000u) | ((d << 16) & 0xff000000u);
#endif
}

// Encrypts `in` under `key` (both 4 memory words); round keys are expanded
// on the fly alongside the rounds (MMO rekeys on every block). The T-table
// functor supplies lk(w, k) = T0[byte k of w].
template <class T0>
PHD void aes128_encrypt(const T0& t0, const uint32_t key[4], const uint32_t in[4], uint32_t out[4]) {
    uint32_t k0 = key[0], k1 = key[1], k2 = key[2], k3 = key[3];
    uint32_t s0 = in[0] ^ k0, s1 = in[1] ^ k1, s2 = in[2] ^ k2, s3 = in[3] ^ k3;
    uint32_t rcon = 1;
    // rounds 1..9 as a rolled loop: one copy of the round code per call site
    // (17 AES per 32-byte suite-2 entry; unrolled they overflow the
    // instruction cache), then the final round without MixColumns
#pragma unroll 1
    for (int r = 1; r < 10; r++) {
        // next round key: w = SubWord(RotWord(k3)) ^ rcon; RotWord folds into the byte picks
        const uint32_t sw = sbox4(t0.lk(k3, 1), t0.lk(k3, 2), t0.lk(k3, 3), t0.lk(k3, 0));
        k0 ^= sw ^ rcon;
        k1 ^= k0;
        k2 ^= k1;
        k3 ^= k2;
        rcon = (rcon << 1) ^ ((rcon & 0x80u) ? 0x11bu : 0u);
        // T_r[x] = rotl(T0[x], 8r): lkr(w, k, r) = T_r[byte k of w] (a rotation
        // of a T0 lookup, or a lookup in a stored T_r, per table functor)
        const uint32_t n0 = t0.lk(s0, 0) ^ t0.lkr(s1, 1, 1) ^ t0.lkr(s2, 2, 2) ^ t0.lkr(s3, 3, 3);
        const uint32_t n1 = t0.lk(s1, 0) ^ t0.lkr(s2, 1, 1) ^ t0.lkr(s3, 2, 2) ^ t0.lkr(s0, 3, 3);
        const uint32_t n2 = t0.lk(s2, 0) ^ t0.lkr(s3, 1, 1) ^ t0.lkr(s0, 2, 2) ^ t0.lkr(s1, 3, 3);
        const uint32_t n3 = t0.lk(s3, 0) ^ t0.lkr(s0, 1, 1) ^ t0.lkr(s1, 2, 2) ^ t0.lkr(s2, 3, 3);
        s0 = n0 ^ k0;
        s1 = n1 ^ k1;
        s2 = n2 ^ k2;
        s3 = n3 ^ k3;
    }
    {  // round 10: SubBytes + ShiftRows + AddRoundKey (rcon = 0x36 here)
        const uint32_t sw = sbox4(t0.lk(k3, 1), t0.lk(k3, 2), t0.lk(k3, 3), t0.lk(k3, 0));
        k0 ^= sw ^ rcon;
        k1 ^= k0;
        k2 ^= k1;
        k3 ^= k2;
        const uint32_t n0 = sbox4(t0.lk(s0, 0), t0.lk(s1, 1), t0.lk(s2, 2), t0.lk(s3, 3));
        const uint32_t n1 = sbox4(t0.lk(s1, 0), t0.lk(s2, 1), t0.lk(s3, 2), t0.lk(s0, 3));
        const uint32_t n2 = sbox4(t0.lk(s2, 0), t0.lk(s3, 1), t0.lk(s0, 2), t0.lk(s1, 3));
        const uint32_t n3 = sbox4(t0.lk(s3, 0), t0.lk(s0, 1), t0.lk(s1, 2), t0.lk(s2, 3));
        s0 = n0 ^ k0;
        s1 = n1 ^ k1;
        s2 = n2 ^ k2;
        s3 = n3 ^ k3;
    }
    out[0] = s0; out[1] = s1; out[2] = s2; out[3] = s3;
}

#define MMO_IV_WORD 0x52525252u
#define MDC2_IV2_WORD 0x25252525u

// One MMO step: h <- E_h(m) ^ m (primitives.cpp:83-84)
template <class T0>
PHD void mmo_step(const T0& t0, uint32_t h[4], const uint32_t m[4]) {
    uint32_t e[4];
    aes128_encrypt(t0, h, m, e);
#pragma unroll
    for (int k = 0; k < 4; k++) h[k] = e[k] ^ m[k];
}

// One MDC-2 step with the cross-swap of second halves (primitives.cpp:97-105)
template <class T0>
PHD void mdc2_step(const T0& t0, uint32_t h[4], uint32_t h2[4], const uint32_t m[4]) {
    uint32_t a[4], b[4];
    aes128_encrypt(t0, h, m, a);
    aes128_encrypt(t0, h2, m, b);
#pragma unroll
    for (int k = 0; k < 4; k++) {
        a[k] ^= m[k];
        b[k] ^= m[k];
    }
    h[0] = a[0]; h[1] = a[1]; h[2] = b[2]; h[3] = b[3];
    h2[0] = b[0]; h2[1] = b[1]; h2[2] = a[2]; h2[3] = a[3];
}

// Byte source over the logical (unpadded) message; 10* padding to 16-byte
// blocks with a full pad block when n % 16 == 0 (primitives.cpp:28-48).
template <class Src>
PHD void pad16_block(const Src& src, uint64_t n, uint64_t off, uint32_t m[4]) {
#pragma unroll
    for (int k = 0; k < 4; k++) {
        uint32_t w = 0;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            uint64_t p = off + 4 * k + i;
            uint32_t b = p < n ? src(p) : (p == n ? 0x80u : 0u);
            w |= b << (8 * i);
        }
        m[k] = w;
    }
}

template <class T0, class Src>
PHD void mmo_hash_dev(const T0& t0, const Src& src, uint64_t n, uint32_t h[4]) {
    h[0] = h[1] = h[2] = h[3] = MMO_IV_WORD;
    uint64_t nb = n / 16 + 1;
    for (uint64_t b = 0; b < nb; b++) {
        uint32_t m[4];
        pad16_block(src, n, 16 * b, m);
        mmo_step(t0, h, m);
    }
}

template <class T0, class Src>
PHD void mdc2_hash_dev(const T0& t0, const Src& src, uint64_t n, uint32_t h[4], uint32_t h2[4]) {
    h[0] = h[1] = h[2] = h[3] = MMO_IV_WORD;
    h2[0] = h2[1] = h2[2] = h2[3] = MDC2_IV2_WORD;
    uint64_t nb = n / 16 + 1;
    for (uint64_t b = 0; b < nb; b++) {
        uint32_t m[4];
        pad16_block(src, n, 16 * b, m);
        mdc2_step(t0, h, h2, m);
    }
}
