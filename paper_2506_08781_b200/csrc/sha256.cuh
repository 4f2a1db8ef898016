// SHA-256 compression for the device (FIPS 180-4 §6.2), used by suite 1
// (SuiteId::Sha256): prf (primitives.cpp:113-127), onetime_seed (:209-223)
// and hash_to_scalar (:149-193), all of which call OpenSSL SHA256 (:21-23).
//
// Fully unrolled over register arrays: with W5..W15 literal constants the
// compiler folds the zero/padding schedule words, and round constants become
// immediates. Rotations lower to SHF.R.W (funnel shift), Ch/Maj/XOR3 to LOP3.
#pragma once
#include "poslo_common.cuh"

#define SHA_IV0 0x6a09e667u
#define SHA_IV1 0xbb67ae85u
#define SHA_IV2 0x3c6ef372u
#define SHA_IV3 0xa54ff53au
#define SHA_IV4 0x510e527fu
#define SHA_IV5 0x9b05688cu
#define SHA_IV6 0x1f83d9abu
#define SHA_IV7 0x5be0cd19u

PHD uint32_t sha_k(int t) {
    const uint32_t K[64] = {
        0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u,
        0xab1c5ed5u, 0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu,
        0x9bdc06a7u, 0xc19bf174u, 0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu,
        0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau, 0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u,
        0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u, 0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu,
        0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u, 0xa2bfe8a1u, 0xa81a664bu,
        0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u, 0x19a4c116u,
        0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
        0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u,
        0xc67178f2u};
    return K[t];
}

PHD uint32_t sha_S0(uint32_t a) { return rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22); }
PHD uint32_t sha_S1(uint32_t e) { return rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25); }
PHD uint32_t sha_s0(uint32_t w) { return rotr32(w, 7) ^ rotr32(w, 18) ^ (w >> 3); }
PHD uint32_t sha_s1(uint32_t w) { return rotr32(w, 17) ^ rotr32(w, 19) ^ (w >> 10); }
PHD uint32_t sha_ch(uint32_t e, uint32_t f, uint32_t g) { return (e & f) ^ (~e & g); }
PHD uint32_t sha_maj(uint32_t a, uint32_t b, uint32_t c) { return (a & b) | (c & (a | b)); }

PHD void sha256_init(uint32_t st[8]) {
    st[0] = SHA_IV0; st[1] = SHA_IV1; st[2] = SHA_IV2; st[3] = SHA_IV3;
    st[4] = SHA_IV4; st[5] = SHA_IV5; st[6] = SHA_IV6; st[7] = SHA_IV7;
}

// Rounds [R0, R1) of one compression over the message words W (rolling
// 16-word schedule, updated in place). The working variables live in st[]
// (a..h); the caller adds the chaining value at the end (sha256_feed_forward)
// so a hoisted mid-state can resume at round R0 > 0.
template <int R0, int R1>
PHD void sha256_rounds(uint32_t st[8], uint32_t W[16]) {
    uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
#pragma unroll
    for (int t = R0; t < R1; t++) {
        uint32_t w;
        if (t < 16) {
            w = W[t];
        } else {
            w = W[t & 15] + sha_s0(W[(t - 15) & 15]) + W[(t - 7) & 15] + sha_s1(W[(t - 2) & 15]);
            W[t & 15] = w;
        }
        uint32_t t1 = h + sha_S1(e) + sha_ch(e, f, g) + sha_k(t) + w;
        uint32_t t2 = sha_S0(a) + sha_maj(a, b, c);
        h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    st[0] = a; st[1] = b; st[2] = c; st[3] = d; st[4] = e; st[5] = f; st[6] = g; st[7] = h;
}

// Full compression of one block into chaining value H.
PHD void sha256_compress(uint32_t H[8], uint32_t W[16]) {
    uint32_t st[8];
#pragma unroll
    for (int i = 0; i < 8; i++) st[i] = H[i];
    sha256_rounds<0, 64>(st, W);
#pragma unroll
    for (int i = 0; i < 8; i++) H[i] += st[i];
}

// ---- suite-1 onetime_seed: F(x0 || be32(j))[0:16], one block (20 B) ------
// W0..W3 = x0 (constant per epoch), W4 = j, W5 = 0x80000000 (pad),
// W6..W14 = 0, W15 = 160 (bit length). Rounds 0..3 only touch W0..W3, so
// their state is hoisted per epoch (ots_pre) and each entry resumes at 4.
PHD void ots_pre(const uint32_t x0w[4], uint32_t pre[8]) {
    uint32_t W[16] = {x0w[0], x0w[1], x0w[2], x0w[3], 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
    sha256_init(pre);
    sha256_rounds<0, 4>(pre, W);
}

PHD void ots_finish(const uint32_t x0w[4], const uint32_t pre[8], uint32_t j, uint32_t out[4]) {
    uint32_t W[16] = {x0w[0], x0w[1], x0w[2], x0w[3], j, 0x80000000u, 0, 0, 0, 0, 0, 0, 0, 0, 0, 160u};
    uint32_t st[8];
#pragma unroll
    for (int i = 0; i < 8; i++) st[i] = pre[i];
    sha256_rounds<4, 64>(st, W);
    out[0] = st[0] + SHA_IV0;
    out[1] = st[1] + SHA_IV1;
    out[2] = st[2] + SHA_IV2;
    out[3] = st[3] + SHA_IV3;
}

// ---- suite-1 prf: F(x || u8(j))[0:16], one block (17 B) ------------------
PHD void prf_sha256(const uint32_t xw[4], int j, uint32_t out[4]) {
    uint32_t W[16] = {xw[0], xw[1], xw[2], xw[3], (uint32_t)(j & 1) << 24 | 0x00800000u,
                      0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 136u};
    uint32_t H[8];
    sha256_init(H);
    sha256_compress(H, W);
    out[0] = H[0]; out[1] = H[1]; out[2] = H[2]; out[3] = H[3];
}

// ---- suite-1 hash_to_scalar digests for a 32-byte entry ------------------
// m: 8 big-endian words, x: the 4 one-time-seed words (already big-endian as
// produced by ots_finish). H0 = SHA256(m || x) (48 B, one block) and
// H1 = SHA256(0x01 || m || x) (49 B, one block; every word is the byte-shifted
// funnel of two neighbours). Returns the 512-bit integer H0 || H1 as 16
// little-endian 32-bit limbs (H0 is the high half, primitives.cpp:166-176).
PHD void h2s_sha256_len32(const uint32_t m[8], const uint32_t x[4], uint32_t limbs[16]) {
    uint32_t W[16] = {m[0], m[1], m[2], m[3], m[4], m[5], m[6], m[7],
                      x[0], x[1], x[2], x[3], 0x80000000u, 0, 0, 384u};
    uint32_t H[8];
    sha256_init(H);
    sha256_compress(H, W);
#pragma unroll
    for (int k = 0; k < 8; k++) limbs[15 - k] = H[k];
    uint32_t V[16];
    V[0] = 0x01000000u | (m[0] >> 8);
#pragma unroll
    for (int k = 1; k < 8; k++) V[k] = fshr32(m[k], m[k - 1], 8);
    V[8] = fshr32(x[0], m[7], 8);
    V[9] = fshr32(x[1], x[0], 8);
    V[10] = fshr32(x[2], x[1], 8);
    V[11] = fshr32(x[3], x[2], 8);
    V[12] = (x[3] << 24) | 0x00800000u;
    V[13] = 0;
    V[14] = 0;
    V[15] = 392u;
    sha256_init(H);
    sha256_compress(H, V);
#pragma unroll
    for (int k = 0; k < 8; k++) limbs[7 - k] = H[k];
}

// ---- generic streaming SHA-256 over a byte source (any length) ------------
// src(p) returns byte p (< n) of the logical message; FIPS 180-4 padding.
template <class Src>
PHD void sha256_stream(const Src& src, uint64_t n, uint32_t H[8]) {
    sha256_init(H);
    uint64_t nb = (n + 9 + 63) / 64;
    for (uint64_t b = 0; b < nb; b++) {
        uint32_t W[16];
#pragma unroll
        for (int k = 0; k < 16; k++) {
            uint32_t w = 0;
#pragma unroll
            for (int i = 0; i < 4; i++) {
                uint64_t p = 64 * b + 4 * k + i;
                uint32_t byte = p < n ? src(p) : (p == n ? 0x80u : 0u);
                w = (w << 8) | byte;
            }
            W[k] = w;
        }
        if (b == nb - 1) {
            W[14] = (uint32_t)((n * 8) >> 32);
            W[15] = (uint32_t)(n * 8);
        }
        sha256_compress(H, W);
    }
}
