// Per-entry challenge computation e_i^j = hash_to_scalar(m, onetime_seed(x0_i, j))
// as a raw 512-bit integer (before the deferred mod-l reduction), for every
// suite, plus the seed-tree PRF step. Host+device (PHD) so the kernels and
// the CPU unit tests in tests/native run the same code.
//   prf            primitives.cpp:113-127
//   onetime_seed   primitives.cpp:209-223
//   hash_to_scalar primitives.cpp:149-193 (digest pair H(m||x) || H(0x01||m||x))
#pragma once
#include "aes128.cuh"
#include "sha256.cuh"
#include "scalar.cuh"

namespace poslo_gpu {

// PRF_b(x) = F(x || b)[0:16] on little-endian memory words.
template <class T0>
PHD void prf_dev(int suite, const T0& t0, uint32_t x[4], int bit) {
    if (suite == 1) {
        uint32_t xw[4] = {bswap32(x[0]), bswap32(x[1]), bswap32(x[2]), bswap32(x[3])}, o[4];
        prf_sha256(xw, bit, o);
#pragma unroll
        for (int k = 0; k < 4; k++) x[k] = bswap32(o[k]);
    } else {
        // MMO over 17 bytes: block0 = x, block1 = bit || 0x80 || 0^14
        uint32_t h[4] = {MMO_IV_WORD, MMO_IV_WORD, MMO_IV_WORD, MMO_IV_WORD};
        uint32_t b1[4] = {(uint32_t)(bit & 1) | 0x8000u, 0, 0, 0};
        mmo_step(t0, h, x);
        mmo_step(t0, h, b1);
#pragma unroll
        for (int k = 0; k < 4; k++) x[k] = h[k];
    }
}


struct PlainMsg {  // the untagged stream m || x
    const uint8_t* m;
    uint32_t L;
    uint32_t x[4];  // memory words
    PHDM uint32_t operator()(uint64_t p) const {
        if (p < L) return m[p];
        uint32_t q = (uint32_t)(p - L);
        return (x[q >> 2] >> (8 * (q & 3))) & 0xffu;
    }
};
struct TaggedMsg {  // 0x01 || m || x
    PlainMsg inner;
    PHDM uint32_t operator()(uint64_t p) const { return p == 0 ? 1u : inner(p - 1); }
};
struct OtsMsg {  // x0 || be32(j) (AES suites)
    uint32_t x0[4];
    uint32_t j;
    PHDM uint32_t operator()(uint64_t p) const {
        if (p < 16) return (x0[p >> 2] >> (8 * (p & 3))) & 0xffu;
        return (j >> (8 * (19 - p))) & 0xffu;
    }
};

// x = onetime_seed(x0, j) (primitives.cpp:209-223) as little-endian memory words.
template <class T0>
PHD void entry_seed(int suite, const T0& t0, const uint32_t x0m[4], uint32_t j, uint32_t x[4]) {
    if (suite == 1) {
        const uint32_t x0w[4] = {bswap32(x0m[0]), bswap32(x0m[1]), bswap32(x0m[2]), bswap32(x0m[3])};
        uint32_t pre[8], xw[4];
        ots_pre(x0w, pre);
        ots_finish(x0w, pre, j, xw);
#pragma unroll
        for (int k = 0; k < 4; k++) x[k] = bswap32(xw[k]);
    } else {
        OtsMsg om{{x0m[0], x0m[1], x0m[2], x0m[3]}, j};
        mmo_hash_dev(t0, om, 20, x);
    }
}

// hash_to_scalar(m, x) (primitives.cpp:149-193) for a given one-time seed x
// (memory words) as a raw 512-bit integer (16 limbs); false on a suite-3
// over-length entry (:179-181). Scheme F's aver_f_single supplies x directly.
template <class T0>
PHD bool entry_limbs_x(int suite, const T0& t0, const uint8_t* m, uint32_t L, const uint32_t x[4],
                       uint32_t limbs[16]) {
    if (suite == 3) {
        if (L > 31) return false;
        // (int_be(m) + int_be(x)) < 2^248 + 2^128 < l: no reduction needed
#pragma unroll
        for (int k = 0; k < 16; k++) limbs[k] = 0;
        for (uint32_t p = 0; p < L; p++) {
            uint32_t bitpos = 8 * (L - 1 - p);
            limbs[bitpos >> 5] |= (uint32_t)m[p] << (bitpos & 31);
        }
        uint32_t xv[4];
#pragma unroll
        for (int k = 0; k < 4; k++) xv[k] = bswap32(x[3 - k]);  // int_be(x) as LE limbs
        uint64_t c = 0;
#pragma unroll
        for (int k = 0; k < 8; k++) {
            c += (uint64_t)limbs[k] + (k < 4 ? xv[k] : 0u);
            limbs[k] = (uint32_t)c;
            c >>= 32;
        }
        return true;
    }
    PlainMsg pm{m, L, {x[0], x[1], x[2], x[3]}};
    TaggedMsg tm{pm};
    if (suite == 1) {
        uint32_t H[8];
        sha256_stream(pm, (uint64_t)L + 16, H);
#pragma unroll
        for (int k = 0; k < 8; k++) limbs[15 - k] = H[k];
        sha256_stream(tm, (uint64_t)L + 17, H);
#pragma unroll
        for (int k = 0; k < 8; k++) limbs[7 - k] = H[k];
    } else {
        uint32_t h[4], h2[4];
        mdc2_hash_dev(t0, pm, (uint64_t)L + 16, h, h2);
#pragma unroll
        for (int k = 0; k < 4; k++) {
            limbs[15 - k] = bswap32(h[k]);
            limbs[11 - k] = bswap32(h2[k]);
        }
        mdc2_hash_dev(t0, tm, (uint64_t)L + 17, h, h2);
#pragma unroll
        for (int k = 0; k < 4; k++) {
            limbs[7 - k] = bswap32(h[k]);
            limbs[3 - k] = bswap32(h2[k]);
        }
    }
    return true;
}

// Per-entry contribution e(m, onetime_seed(x0, j)) as 16 limbs (agg_ekeys).
template <class T0>
PHD bool entry_limbs(int suite, const T0& t0, const uint8_t* m, uint32_t L, const uint32_t x0m[4], uint32_t j,
                     uint32_t limbs[16]) {
    uint32_t x[4];
    entry_seed(suite, t0, x0m, j, x);
    return entry_limbs_x(suite, t0, m, L, x, limbs);
}

// ---- signer side: nonce_to_scalar (primitives.cpp:195-207)
// r-seed || be32(i) || be32(j) || counter, expanded by expand_wide (:128-146):
// F(msg || 0x00) || F(msg || 0x01), F = SHA-256 or MDC-2, reduced mod l and
// retried with the next counter while zero.
struct NonceMsg {  // the 26-byte expand_wide input
    uint32_t r[4];  // seed memory words
    uint32_t i, j, counter, tag;
    PHDM uint32_t operator()(uint64_t p) const {
        if (p < 16) return (r[p >> 2] >> (8 * (p & 3))) & 0xffu;
        if (p < 20) return (i >> (8 * (19 - p))) & 0xffu;
        if (p < 24) return (j >> (8 * (23 - p))) & 0xffu;
        return p == 24 ? (counter & 0xffu) : tag;
    }
};

template <class T0>
PHD void nonce_scalar(int suite, const T0& t0, const uint32_t r[4], uint32_t i, uint32_t j, uint32_t out[8]) {
    for (uint32_t counter = 0;; counter++) {
        uint32_t limbs[16];
        for (uint32_t tag = 0; tag < 2; tag++) {
            NonceMsg nm{{r[0], r[1], r[2], r[3]}, i, j, counter, tag};
            const int hi = tag ? 7 : 15;  // d0 is the high half of the wide value
            if (suite == 1) {
                uint32_t W[16] = {bswap32(r[0]), bswap32(r[1]), bswap32(r[2]), bswap32(r[3]), i, j,
                                  (counter & 0xffu) << 24 | tag << 16 | 0x8000u, 0, 0, 0, 0, 0, 0, 0, 0, 208u};
                uint32_t H[8];
                sha256_init(H);
                sha256_compress(H, W);
                for (int k = 0; k < 8; k++) limbs[hi - k] = H[k];
            } else {
                uint32_t h[4], h2[4];
                mdc2_hash_dev(t0, nm, 26, h, h2);
                for (int k = 0; k < 4; k++) {
                    limbs[hi - k] = bswap32(h[k]);
                    limbs[hi - 4 - k] = bswap32(h2[k]);
                }
            }
        }
        sc_reduce_limbs(limbs, 16, out);
        if (!sc_is_zero(out)) return;
    }
}

// ---- fast path, suite 1, 32-byte entry: m as 8 big-endian words, x0w the
// epoch seed as big-endian words with its hoisted onetime_seed mid-state.
template <int MODE = 0>
PHD void entry_limbs_s1_l32(const uint32_t x0w[4], const uint32_t pre[8], uint32_t j,
                            const uint32_t m[8], uint32_t limbs[16], uint32_t one = 1) {
    uint32_t x[4];
    ots_finish<MODE>(x0w, pre, j, x, one);
    h2s_sha256_len32<MODE>(m, x, limbs, one);
}

// ---- fast path, suite 2 (MMO/MDC-2), 32-byte entry -----------------------
// onetime_seed = MMO(x0 || be32 j) over 2 blocks; the first block (x0 under
// the constant IV key) is hoisted per epoch into hpre. hash_to_scalar =
// MDC-2(m || x) (48 B -> 4 blocks incl. a full pad block) and
// MDC-2(0x01 || m || x) (49 B -> 4 blocks), 2 AES per block.
template <class T0>
PHD void mdc2_digest_limbs(const T0& t0, const uint32_t blk[16],
                                                  uint32_t limbs_hi_index, uint32_t limbs[16]) {
    uint32_t h[4] = {MMO_IV_WORD, MMO_IV_WORD, MMO_IV_WORD, MMO_IV_WORD};
    uint32_t h2[4] = {MDC2_IV2_WORD, MDC2_IV2_WORD, MDC2_IV2_WORD, MDC2_IV2_WORD};
#pragma unroll 1
    for (int b = 0; b < 4; b++) {  // rolled: one copy of the two AES per call site
        const uint32_t m[4] = {blk[4 * b], blk[4 * b + 1], blk[4 * b + 2], blk[4 * b + 3]};
        mdc2_step(t0, h, h2, m);
    }
    // digest bytes h || h2 read as big-endian words 0..7
#pragma unroll
    for (int k = 0; k < 4; k++) {
        limbs[limbs_hi_index - k] = bswap32(h[k]);
        limbs[limbs_hi_index - 4 - k] = bswap32(h2[k]);
    }
}


template <class T0>
PHD void entry_limbs_s2_l32(const T0& t0, const uint32_t hpre[4], uint32_t j, const uint32_t m[8],
                            uint32_t limbs[16]) {
    // x = MMO(x0 || be32 j): second block = be32(j) || 0x80 || 0^11
    uint32_t x[4] = {hpre[0], hpre[1], hpre[2], hpre[3]};
    const uint32_t b1[4] = {bswap32(j), 0x80u, 0, 0};
    mmo_step(t0, x, b1);
    // untagged stream m || x || pad (48 B + full pad block)
    uint32_t blk[16] = {m[0], m[1], m[2], m[3], m[4], m[5], m[6], m[7],
                        x[0], x[1], x[2], x[3], 0x80u, 0, 0, 0};
    mdc2_digest_limbs(t0, blk, 15, limbs);
    // tagged stream 0x01 || m || x || 0x80 || 0^14 (49 B -> 64 B):
    // memory word k = bytes 4k-1 .. 4k+2 of the untagged stream
    uint32_t tb[16];
    const uint32_t u[13] = {m[0], m[1], m[2], m[3], m[4], m[5], m[6], m[7], x[0], x[1], x[2], x[3], 0x80u};
    tb[0] = 0x01u | (u[0] << 8);
#pragma unroll
    for (int k = 1; k < 13; k++) tb[k] = fshr32(u[k - 1], u[k], 24);
    tb[13] = 0;  // (u[12] >> 24) | (u[13] << 8) with u[13] = 0
    tb[14] = 0;
    tb[15] = 0;
    mdc2_digest_limbs(t0, tb, 7, limbs);
}

}  // namespace poslo_gpu
