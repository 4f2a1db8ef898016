// SHA-256 compression for the device (FIPS 180-4 §6.2), used by suite 1
// (SuiteId::Sha256): prf (primitives.cpp:113-127), onetime_seed (:209-223)
// and hash_to_scalar (:149-193), all of which call OpenSSL SHA256 (:21-23).
//
// Fully unrolled over register arrays: with W5..W15 literal constants the
// compiler folds the zero/padding schedule words, and round constants become
// immediates. Rotations lower to SHF.R.W (funnel shift), Ch/Maj/XOR3 to LOP3.
#pragma once
#include "poslo_common.cuh"

#ifndef POSLO_KADD
#define POSLO_KADD 0  // + K of the FMA == 5 round: 0 VIADD, 1 onev * K IMAD, 2 K from shared memory
#endif

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

// Pipe balancing (B200): the SM issues one warp-instruction per cycle per
// sub-partition, but LOP3/SHF/IADD3 all run on the ALU pipe (16 lanes/clk)
// while the FMA pipe (IMAD) idles. SHA-256 is rotation/XOR heavy, so in
// MODE >= 1 every addition whose operands are not compile-time constants is
// emitted as IMAD (a * one + b, `one` = 1 from an opaque kernel parameter)
// to move it to the FMA pipe; MODE 2 also moves the logical shifts of
// sigma0/1 to IMAD.HI. MODE 0 is plain C (host tests, cold paths). CM / ZM
// are bit masks of the message words W0..W15 that are compile-time
// constants / zero (ZM documents which constants are zero), so constant
// terms fold and zero terms vanish.
// Inline PTX so LLVM cannot reassociate chains of a*one+b back into IADD3s.
#ifndef POSLO_FADD
#define POSLO_FADD 0  // 0: mad.lo a * one + b; 1: add.u32 (ptxas picks IADD3 / IMAD.IADD); 2: mad.lo a * 1 + b
                      // 3: a * c_fadd_one + b with the multiplier read from the constant bank
#endif
#if defined(__CUDACC__) && POSLO_FADD == 3
__constant__ uint32_t c_fadd_one = 1u;
#endif
PHD uint32_t fadd(uint32_t a, uint32_t b, uint32_t one) {
#ifdef __CUDA_ARCH__
    uint32_t r;
#if POSLO_FADD == 3
    (void)one;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(c_fadd_one), "r"(b));
#elif POSLO_FADD == 1
    (void)one;
    asm("add.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(b));
#elif POSLO_FADD == 2
    (void)one;
    asm("mad.lo.u32 %0, %1, 1, %2;" : "=r"(r) : "r"(a), "r"(b));
#else
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(a), "r"(one), "r"(b));
#endif
    return r;
#else
    return a * one + b;
#endif
}

template <int MODE>
PHD uint32_t shr_via(uint32_t w, int n, uint32_t one) {
#ifdef __CUDA_ARCH__
    if (MODE >= 2) return __umulhi(w, one << (32 - n));
#endif
    return w >> n;
}

// Opaque multipliers for moving rotations and shifts to the FMA pipe.
// rotr(x, n) = lo(x * 2^(32-n)) + hi(x * 2^(32-n)) (the two halves have
// disjoint bits), i.e. one IMAD.HI + one IMAD, no ALU instruction; x >> n =
// hi(x * 2^(32-n)) is one IMAD.HI. The multipliers arrive as kernel
// parameters so ptxas cannot strength-reduce them back into SHF/LEA (ALU).
struct PipeK {
    uint32_t one;       // 1
    uint32_t r22, r25;  // 2^(32-22), 2^(32-25): rotr 22 (Sigma0), rotr 25 (Sigma1)
    uint32_t s3, s10;   // 2^29, 2^22: >> 3 (sigma0), >> 10 (sigma1)
    uint32_t onev;      // 1 in a VECTOR register (pipek_vec), for IMAD onev * K + x (FMA == 5)
};

PHD PipeK pipek_make() {
    PipeK k;
    k.one = 1u;
    k.r22 = 1u << 10;
    k.r25 = 1u << 7;
    k.s3 = 1u << 29;
    k.s10 = 1u << 22;
    k.onev = 1u;
    return k;
}

// An opaque 1 that lives in a vector register: `one` is a kernel parameter
// (uniform register), and an IMAD has room for only one uniform operand, so
// h + W + K with K itself uniform (constant bank / loop-indexed) cannot be
// one * K + x on `one`. onev * K + x can: IMAD Rd, R_onev, UR_K|imm, Rx.
// Loaded once per thread through a volatile global read so ptxas cannot fold
// it back into an IADD3 on the ALU pipe.
#ifdef __CUDACC__
static __device__ uint32_t g_sha_onev = 1u;
#endif
PHD PipeK pipek_vec(PipeK k) {
#ifdef __CUDA_ARCH__
    k.onev = *reinterpret_cast<volatile const uint32_t*>(&g_sha_onev);
#endif
    return k;
}

// x + k on the FMA pipe with k as the multiplicand of the vector 1
PHD uint32_t kmad(uint32_t x, uint32_t k, const PipeK& pk) {
#ifdef __CUDA_ARCH__
    uint32_t r;
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(pk.onev), "r"(k), "r"(x));
    return r;
#else
    (void)pk;
    return x + k;
#endif
}

// rotr(x, n) with p = 2^(32-n), on the FMA pipe
PHD uint32_t rotr_fma(uint32_t x, uint32_t p) {
#ifdef __CUDA_ARCH__
    uint32_t hi, r;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(x), "r"(p));
    asm("mad.lo.u32 %0, %1, %2, %3;" : "=r"(r) : "r"(x), "r"(p), "r"(hi));
    return r;
#else
    return (uint32_t)(((uint64_t)x * p) >> 32) + x * p;
#endif
}

// x >> n with p = 2^(32-n), on the FMA pipe
PHD uint32_t shr_fma(uint32_t x, uint32_t p) {
#ifdef __CUDA_ARCH__
    uint32_t hi;
    asm("mul.hi.u32 %0, %1, %2;" : "=r"(hi) : "r"(x), "r"(p));
    return hi;
#else
    return (uint32_t)(((uint64_t)x * p) >> 32);
#endif
}

// Constness of all 64 schedule words, evaluated at compile time: W[t] is a
// constant iff all four words it is derived from are.
template <uint32_t CM>
struct WConst {
    static constexpr uint64_t compute() {
        uint64_t m = CM;
        for (int t = 16; t < 64; t++) {
            bool c = ((m >> (t - 16)) & 1) && ((m >> (t - 15)) & 1) && ((m >> (t - 7)) & 1) && ((m >> (t - 2)) & 1);
            if (c) m |= 1ull << t;
        }
        return m;
    }
    static constexpr uint64_t value = compute();
};

// Rounds [R0, R1) of one compression over the message words W (rolling
// 16-word schedule, updated in place). The working variables live in st[]
// (a..h); the caller adds the chaining value, so a hoisted mid-state can
// resume at round R0 > 0.
template <int R0, int R1, uint32_t CM = 0, uint32_t ZM = 0, int MODE = 0>
PHD void sha256_rounds(uint32_t st[8], uint32_t W[16], uint32_t one = 1) {
    constexpr uint64_t CMASK = WConst<CM>::value;
    uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
#pragma unroll
    for (int t = R0; t < R1; t++) {
        uint32_t w;
        const bool wc = (CMASK >> t) & 1;
        if (t < 16) {
            w = W[t];
        } else {
            const int i16 = t - 16, i15 = t - 15, i7 = t - 7, i2 = t - 2;
            const uint32_t x16 = W[i16 & 15], x15 = W[i15 & 15], x7 = W[i7 & 15], x2 = W[i2 & 15];
            if (MODE == 0 || wc) {
                w = x16 + sha_s0(x15) + x7 + sha_s1(x2);
            } else {
                // constant terms first (folded), variable terms chained on IMAD
                uint32_t acc = 0;
                const bool c16 = (CMASK >> i16) & 1, c15 = (CMASK >> i15) & 1;
                const bool c7 = (CMASK >> i7) & 1, c2 = (CMASK >> i2) & 1;
                if (c16) acc += x16;  // zero words (ZM) are constants and fold away here
                if (c15) acc += sha_s0(x15);
                if (c7) acc += x7;
                if (c2) acc += sha_s1(x2);
                if (!c2) acc = fadd(rotr32(x2, 17) ^ rotr32(x2, 19) ^ shr_via<MODE>(x2, 10, one), acc, one);
                if (!c15) acc = fadd(rotr32(x15, 7) ^ rotr32(x15, 18) ^ shr_via<MODE>(x15, 3, one), acc, one);
                if (!c7) acc = fadd(x7, acc, one);
                if (!c16) acc = fadd(x16, acc, one);
                w = acc;
            }
            W[t & 15] = w;
        }
        uint32_t na, ne;
        if (MODE == 0 || (R0 == 0 && t < 4)) {  // plain (or partially-constant IV start: fold)
            const uint32_t t1 = h + sha_S1(e) + sha_ch(e, f, g) + sha_k(t) + w;
            na = t1 + sha_S0(a) + sha_maj(a, b, c);
            ne = d + t1;
        } else {
            const uint32_t kw = wc ? sha_k(t) + w : fadd(w, sha_k(t), one);
            const uint32_t t1 = fadd(sha_ch(e, f, g), fadd(sha_S1(e), fadd(h, kw, one), one), one);
            na = fadd(sha_maj(a, b, c), fadd(sha_S0(a), t1, one), one);
            ne = fadd(d, t1, one);
        }
        h = g; g = f; f = e; e = ne;
        d = c; c = b; b = a; a = na;
    }
    st[0] = a; st[1] = b; st[2] = c; st[3] = d; st[4] = e; st[5] = f; st[6] = g; st[7] = h;
}

// Full compression of one block into chaining value H.
template <uint32_t CM = 0, uint32_t ZM = 0, int MODE = 0>
PHD void sha256_compress(uint32_t H[8], uint32_t W[16], uint32_t one = 1) {
    uint32_t st[8];
#pragma unroll
    for (int i = 0; i < 8; i++) st[i] = H[i];
    sha256_rounds<0, 64, CM, ZM, MODE>(st, W, one);
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

template <int MODE = 0>
PHD void ots_finish(const uint32_t x0w[4], const uint32_t pre[8], uint32_t j, uint32_t out[4],
                    uint32_t one = 1) {
    uint32_t W[16] = {x0w[0], x0w[1], x0w[2], x0w[3], j, 0x80000000u, 0, 0, 0, 0, 0, 0, 0, 0, 0, 160u};
    uint32_t st[8];
#pragma unroll
    for (int i = 0; i < 8; i++) st[i] = pre[i];
    // W5..W15 constant, W6..W14 zero
    sha256_rounds<4, 64, 0xFFE0u, 0x7FC0u, MODE>(st, W, one);
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
template <int MODE = 0>
PHD void h2s_sha256_len32(const uint32_t m[8], const uint32_t x[4], uint32_t limbs[16],
                          uint32_t one = 1) {
    uint32_t W[16] = {m[0], m[1], m[2], m[3], m[4], m[5], m[6], m[7],
                      x[0], x[1], x[2], x[3], 0x80000000u, 0, 0, 384u};
    uint32_t H[8];
    sha256_init(H);
    sha256_compress<0xF000u, 0x6000u, MODE>(H, W, one);  // W12..15 constant, W13/W14 zero
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
    sha256_compress<0xE000u, 0x6000u, MODE>(H, V, one);  // W13..15 constant, W13/W14 zero
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

// ---- compact form (instruction-cache friendly) ----------------------------
// The fully unrolled compressions above are ~1.4k SASS instructions each;
// three of them per entry (x E entries per thread) overflow the SM's
// instruction caches and ncu shows warps stalled on "no instruction" most
// of the time. The compact form keeps rounds 0..15 unrolled and runs rounds
// 16..63 as a 3-trip loop over a 16-round unrolled body (K from constant
// memory, indexed by the uniform trip counter); the three compressions of an
// entry share one copy of this code.
#ifdef __CUDACC__
__constant__ uint32_t c_sha_k[64] = {
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
#endif

#if defined(__CUDACC__) && POSLO_KADD == 2
// K in shared memory (a vector register after the LDS), so + K can be an IMAD
// on the uniform `one` (sha_k_smem_init() fills it at kernel start)
static __shared__ uint32_t s_sha_k[64];
#endif
PHD void sha_k_smem_init() {
#if defined(__CUDA_ARCH__) && POSLO_KADD == 2
    if (threadIdx.x < 64) s_sha_k[threadIdx.x] = c_sha_k[threadIdx.x];
    __syncthreads();
#endif
}

PHD uint32_t sha_kc(int t) {
#if defined(__CUDA_ARCH__) && POSLO_KADD == 2
    return s_sha_k[t];
#elif defined(__CUDA_ARCH__)
    return c_sha_k[t];
#else
    return sha_k(t);
#endif
}

#define SHA_RND(a, b, c, d, e, f, g, h, w, k)                                         \
    do {                                                                              \
        uint32_t t1_ = (h) + sha_S1(e) + sha_ch((e), (f), (g)) + (k) + (w);            \
        (d) += t1_;                                                                   \
        (h) = t1_ + sha_S0(a) + sha_maj((a), (b), (c));                               \
    } while (0)

// Pipe-balanced round (FMA >= 1): h + w + K stays one IADD3 on the ALU
// pipe, the remaining additions go to the FMA pipe as IMADs with the opaque
// `one` (fadd), so the ALU pipe only carries rotations, LOP3s and one add.
#define SHA_RND_F(a, b, c, d, e, f, g, h, w, k)                                       \
    do {                                                                              \
        uint32_t t1_ = fadd(sha_ch((e), (f), (g)), fadd(sha_S1(e), (h) + (w) + (k), one), one); \
        (d) = fadd((d), t1_, one);                                                    \
        (h) = fadd(sha_maj((a), (b), (c)), fadd(sha_S0(a), t1_, one), one);           \
    } while (0)

// FMA >= 3: also h + (K + w) on the FMA pipe (K as the IMAD multiplicand, so
// it can stay an immediate / constant-bank operand): the ALU pipe carries
// only the six rotations and four LOP3s of a round.
#define SHA_RND_F3(a, b, c, d, e, f, g, h, w, k)                                      \
    do {                                                                              \
        uint32_t t1_ = fadd(sha_ch((e), (f), (g)),                                    \
                            fadd(sha_S1(e), fadd((h), fadd((k), (w), one), one), one), one); \
        (d) = fadd((d), t1_, one);                                                    \
        (h) = fadd(sha_maj((a), (b), (c)), fadd(sha_S0(a), t1_, one), one);           \
    } while (0)

// FMA == 4, balanced: one rotation of each Sigma on the FMA pipe
// (rotr_fma) plus the additions of SHA_RND_F. Per round 4 SHF + 4 LOP3 +
// 1 IADD3 on the ALU pipe and 9 IMAD-class on the FMA pipe; per schedule word
// 4 SHF + 2 LOP3 (ALU) and 2 IMAD.HI + 3 IMAD (FMA). Per compression
// ALU 864 / FMA 816 instructions, against ALU 1088 / FMA 464 for FMA == 2:
// the two pipes (16 lanes/clk each per SMSP) are then nearly equally loaded
// and the bound moves to the issue slot (1 instruction/clk/SMSP).
#define SHA_RND_B(a, b, c, d, e, f, g, h, w, k)                                       \
    do {                                                                              \
        const uint32_t s1_ = rotr32((e), 6) ^ rotr32((e), 11) ^ rotr_fma((e), pk.r25); \
        const uint32_t s0_ = rotr32((a), 2) ^ rotr32((a), 13) ^ rotr_fma((a), pk.r22); \
        uint32_t t1_ = fadd(sha_ch((e), (f), (g)), fadd(s1_, (h) + (w) + (k), one), one); \
        (d) = fadd((d), t1_, one);                                                    \
        (h) = fadd(sha_maj((a), (b), (c)), fadd(s0_, t1_, one), one);                 \
    } while (0)
// + K of SHA_RND_K: 0 = a two-input add (ptxas emits VIADD R, R, UR|imm, an
// FMA-pipe instruction on sm_100), 1 = onev * K + x (IMAD).
#if POSLO_KADD == 2
#define SHA_KADD(x, k) fadd((x), (k), one)
#elif POSLO_KADD
#define SHA_KADD(x, k) kmad((x), (k), pk)
#else
#define SHA_KADD(x, k) ((x) + (k))
#endif
// FMA == 5: every addition on the FMA pipe. As SHA_RND_F, plus h + W + K as
// an IMAD (h + W on `one`) and a VIADD / IMAD for + K (SHA_KADD).
// Per round 6 SHF + 4 LOP3 on the ALU pipe and 7 FMA-pipe adds, so the
// ALU pipe carries exactly the 1024 ALU-only operations of a compression.
#define SHA_RND_K(a, b, c, d, e, f, g, h, w, k)                                       \
    do {                                                                              \
        const uint32_t hwk_ = SHA_KADD(fadd((h), (w), one), (k));                     \
        uint32_t t1_ = fadd(sha_ch((e), (f), (g)), fadd(sha_S1(e), hwk_, one), one);  \
        (d) = fadd((d), t1_, one);                                                    \
        (h) = fadd(sha_maj((a), (b), (c)), fadd(sha_S0(a), t1_, one), one);           \
    } while (0)
#define SHA_SCHED_B(i)                                                                 \
    do {                                                                              \
        const uint32_t x15_ = W[((i) + 1) & 15], x2_ = W[((i) + 14) & 15];            \
        const uint32_t s0_ = rotr32(x15_, 7) ^ rotr32(x15_, 18) ^ shr_fma(x15_, pk.s3); \
        const uint32_t s1_ = rotr32(x2_, 17) ^ rotr32(x2_, 19) ^ shr_fma(x2_, pk.s10); \
        W[i] = fadd(s0_, fadd(s1_, fadd(W[((i) + 9) & 15], W[i], one), one), one);    \
    } while (0)

// Pipe-assignment sweep (FMA >= 16: P = FMA - 16 is a bit set). Each bit moves
// one class of work of a round / schedule word between the ALU pipe (IADD3,
// LOP3, SHF) and the FMA pipe (IMAD; IMAD.HI is half rate, measured):
//   P&1  sigma shifts on IMAD.HI          P&2  h + w + K on IMADs
//   P&4  Sigma1 rotr 25 on IMAD.HI+IMAD   P&8  Sigma0 rotr 22 on IMAD.HI+IMAD
//   P&16 T1 = IADD3(hwk, S1, Ch)          P&32 schedule sum as 2 IADD3
//   P&64 e' = d + T1 on the ALU           P&128 a' = IADD3(T1, S0, Maj)
template <int P>
PHD void sha_rnd_p(uint32_t a, uint32_t b, uint32_t c, uint32_t& d, uint32_t e, uint32_t f, uint32_t g,
                   uint32_t& h, uint32_t w, uint32_t k, const PipeK& pk) {
    const uint32_t one = pk.one;
    const uint32_t r25 = (P & 4) ? rotr_fma(e, pk.r25) : rotr32(e, 25);
    const uint32_t r22 = (P & 8) ? rotr_fma(a, pk.r22) : rotr32(a, 22);
    const uint32_t s1 = rotr32(e, 6) ^ rotr32(e, 11) ^ r25;
    const uint32_t s0 = rotr32(a, 2) ^ rotr32(a, 13) ^ r22;
    const uint32_t hwk = (P & 2) ? fadd(h, fadd(k, w, one), one) : h + w + k;
    const uint32_t t1 = (P & 16) ? hwk + s1 + sha_ch(e, f, g) : fadd(sha_ch(e, f, g), fadd(s1, hwk, one), one);
    d = (P & 64) ? d + t1 : fadd(d, t1, one);
    h = (P & 128) ? t1 + s0 + sha_maj(a, b, c) : fadd(sha_maj(a, b, c), fadd(s0, t1, one), one);
}

template <int P>
PHD uint32_t sha_sched_p(uint32_t w16, uint32_t w15, uint32_t w7, uint32_t w2, const PipeK& pk) {
    const uint32_t one = pk.one;
    const uint32_t sh3 = (P & 1) ? shr_fma(w15, pk.s3) : w15 >> 3;
    const uint32_t sh10 = (P & 1) ? shr_fma(w2, pk.s10) : w2 >> 10;
    const uint32_t s0 = rotr32(w15, 7) ^ rotr32(w15, 18) ^ sh3;
    const uint32_t s1 = rotr32(w2, 17) ^ rotr32(w2, 19) ^ sh10;
    return (P & 32) ? w16 + s0 + w7 + s1 : fadd(s0, fadd(s1, fadd(w7, w16, one), one), one);
}

#define SHA_SCHED(i)                                                                   \
    W[i] += sha_s0(W[((i) + 1) & 15]) + W[((i) + 9) & 15] + sha_s1(W[((i) + 14) & 15])
#define SHA_SCHED_F(i)                                                                 \
    W[i] = fadd(sha_s0(W[((i) + 1) & 15]), fadd(sha_s1(W[((i) + 14) & 15]),            \
                fadd(W[((i) + 9) & 15], W[i], one), one), one)

#define SHA_RND_SEL(...)                                        \
    do {                                                        \
        if (FMA >= 16) sha_rnd_p<FMA - 16>(__VA_ARGS__, pk);    \
        else if (FMA == 5) SHA_RND_K(__VA_ARGS__);              \
        else if (FMA >= 4) SHA_RND_B(__VA_ARGS__);              \
        else if (FMA >= 3) SHA_RND_F3(__VA_ARGS__);             \
        else if (FMA) SHA_RND_F(__VA_ARGS__);                   \
        else SHA_RND(__VA_ARGS__);                              \
    } while (0)

// 16 rounds starting at round t0 + 0 whose message words are W[0..15]
// (after the schedule update): the body shared by all compressions.
#define SHA_16_ROUNDS(KF, t0)                                                  \
    do {                                                                       \
        SHA_RND_SEL(a, b, c, d, e, f, g, h, W[0], KF((t0) + 0));               \
        SHA_RND_SEL(h, a, b, c, d, e, f, g, W[1], KF((t0) + 1));               \
        SHA_RND_SEL(g, h, a, b, c, d, e, f, W[2], KF((t0) + 2));               \
        SHA_RND_SEL(f, g, h, a, b, c, d, e, W[3], KF((t0) + 3));               \
        SHA_RND_SEL(e, f, g, h, a, b, c, d, W[4], KF((t0) + 4));               \
        SHA_RND_SEL(d, e, f, g, h, a, b, c, W[5], KF((t0) + 5));               \
        SHA_RND_SEL(c, d, e, f, g, h, a, b, W[6], KF((t0) + 6));               \
        SHA_RND_SEL(b, c, d, e, f, g, h, a, W[7], KF((t0) + 7));               \
        SHA_RND_SEL(a, b, c, d, e, f, g, h, W[8], KF((t0) + 8));               \
        SHA_RND_SEL(h, a, b, c, d, e, f, g, W[9], KF((t0) + 9));               \
        SHA_RND_SEL(g, h, a, b, c, d, e, f, W[10], KF((t0) + 10));             \
        SHA_RND_SEL(f, g, h, a, b, c, d, e, W[11], KF((t0) + 11));             \
        SHA_RND_SEL(e, f, g, h, a, b, c, d, W[12], KF((t0) + 12));             \
        SHA_RND_SEL(d, e, f, g, h, a, b, c, W[13], KF((t0) + 13));             \
        SHA_RND_SEL(c, d, e, f, g, h, a, b, W[14], KF((t0) + 14));             \
        SHA_RND_SEL(b, c, d, e, f, g, h, a, W[15], KF((t0) + 15));             \
    } while (0)

// Rounds r0..15 (r0 = 0, or 4 resuming after a hoisted round 3) over W[0..15].
// st is a..h in the usual order on entry and exit. CM: rounds whose W is a
// compile-time constant; with FMA == 5 they keep the SHA_RND_F form, where
// h + (W + K) folds to one VIADD with an immediate (the FMA == 5 form would
// be an IMAD with an immediate addend, whose multiplier `one` ptxas must
// then hold in a vector register for the whole kernel: R-R-R IMADs).
template <int FMA = 0, uint32_t CM = 0>
PHD void sha256_rounds_head(uint32_t st[8], const uint32_t W[16], int r0, const PipeK& pk) {
    const uint32_t one = pk.one;
    (void)one;
#define RNDC(i, ...)                                                    \
    do {                                                                \
        if (FMA == 5 && ((CM >> (i)) & 1u)) SHA_RND_F(__VA_ARGS__);     \
        else SHA_RND_SEL(__VA_ARGS__);                                  \
    } while (0)
    uint32_t a, b, c, d, e, f, g, h;
    if (r0 == 0) {
        a = st[0]; b = st[1]; c = st[2]; d = st[3]; e = st[4]; f = st[5]; g = st[6]; h = st[7];
        RNDC(0, a, b, c, d, e, f, g, h, W[0], sha_k(0));
        RNDC(1, h, a, b, c, d, e, f, g, W[1], sha_k(1));
        RNDC(2, g, h, a, b, c, d, e, f, W[2], sha_k(2));
        RNDC(3, f, g, h, a, b, c, d, e, W[3], sha_k(3));
    } else {  // resume after round 3: the names are rotated by four
        e = st[0]; f = st[1]; g = st[2]; h = st[3]; a = st[4]; b = st[5]; c = st[6]; d = st[7];
    }
    RNDC(4, e, f, g, h, a, b, c, d, W[4], sha_k(4));
    RNDC(5, d, e, f, g, h, a, b, c, W[5], sha_k(5));
    RNDC(6, c, d, e, f, g, h, a, b, W[6], sha_k(6));
    RNDC(7, b, c, d, e, f, g, h, a, W[7], sha_k(7));
    RNDC(8, a, b, c, d, e, f, g, h, W[8], sha_k(8));
    RNDC(9, h, a, b, c, d, e, f, g, W[9], sha_k(9));
    RNDC(10, g, h, a, b, c, d, e, f, W[10], sha_k(10));
    RNDC(11, f, g, h, a, b, c, d, e, W[11], sha_k(11));
    RNDC(12, e, f, g, h, a, b, c, d, W[12], sha_k(12));
    RNDC(13, d, e, f, g, h, a, b, c, W[13], sha_k(13));
    RNDC(14, c, d, e, f, g, h, a, b, W[14], sha_k(14));
    RNDC(15, b, c, d, e, f, g, h, a, W[15], sha_k(15));
#undef RNDC
    st[0] = a; st[1] = b; st[2] = c; st[3] = d; st[4] = e; st[5] = f; st[6] = g; st[7] = h;
}

// Rounds blk0..63 (blk0 = 16 or 32) as a rolled loop over one 16-round body:
// schedule update of the rolling window W (W[i] = W_{blk-16+i} on entry),
// then 16 rounds with K from constant memory.
template <int FMA = 0>
PHD void sha256_rounds_loop(uint32_t st[8], uint32_t W[16], int blk0, const PipeK& pk) {
    const uint32_t one = pk.one;
    (void)one;
    uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
#pragma unroll 1
    for (int blk = blk0; blk < 64; blk += 16) {
#pragma unroll
        for (int i = 0; i < 16; i++) {
            if (FMA >= 16) W[i] = sha_sched_p<FMA - 16>(W[i], W[(i + 1) & 15], W[(i + 9) & 15], W[(i + 14) & 15], pk);
            else if (FMA == 5) SHA_SCHED_F(i);
            else if (FMA >= 4) SHA_SCHED_B(i);
            else if (FMA >= 2) SHA_SCHED_F(i);
            else SHA_SCHED(i);
        }
        SHA_16_ROUNDS(sha_kc, blk);
    }
    st[0] = a; st[1] = b; st[2] = c; st[3] = d; st[4] = e; st[5] = f; st[6] = g; st[7] = h;
}

// Working state st (a..h) from round r0 (0 or 4; rounds < r0 already applied)
// through round 63 over message words W (destroyed).
template <int FMA = 0>
PHD void sha256_rounds_compact(uint32_t st[8], uint32_t W[16], int r0, const PipeK& pk) {
    sha256_rounds_head<FMA>(st, W, r0, pk);
    sha256_rounds_loop<FMA>(st, W, 16, pk);
}

// ---- entry-hash specialisation: one-block messages with W13 = W14 = 0 --------
// Both entry hashes of a 32-byte entry (m || x: W12 = 0x80000000, W15 = 384;
// 0x01 || m || x: W12 varies, W15 = 392) have W13 = W14 = 0 and a constant
// W15, so sigma1(W14), sigma0(W13), sigma0(W14) vanish and sigma1(W15),
// sigma0(W15) are constants (s1w15, s0w15) in W16..W31. Runs rounds 0..31
// and leaves W = W16..W31 for sha256_rounds_loop(.., 32, ..).
template <int FMA_H = 2, int FMA_B = FMA_H>  // FMA_B: pipe assignment of rounds 16..31
PHD void entry_head_rounds(uint32_t st[8], uint32_t W[16], uint32_t s1w15, uint32_t s0w15, const PipeK& pk) {
    constexpr int FMA = FMA_H;
    const uint32_t one = pk.one;
    (void)one;
    sha256_rounds_head<FMA, (1u << 13) | (1u << 14) | (1u << 15)>(st, W, 0, pk);  // W13 = W14 = 0, W15 uniform
    const uint32_t w0 = W[0], w1 = W[1], w2 = W[2], w3 = W[3], w4 = W[4], w5 = W[5], w6 = W[6], w7 = W[7];
    const uint32_t w8 = W[8], w9 = W[9], w10 = W[10], w11 = W[11], w12 = W[12], w15 = W[15];
    W[0] = fadd(sha_s0(w1), fadd(w9, w0, one), one);                                   // W16
    W[1] = fadd(sha_s0(w2), fadd(w10, fadd(w1, s1w15, one), one), one);              // W17
    W[2] = fadd(sha_s1(W[0]), fadd(sha_s0(w3), fadd(w11, w2, one), one), one);       // W18
    W[3] = fadd(sha_s1(W[1]), fadd(sha_s0(w4), fadd(w12, w3, one), one), one);       // W19
    W[4] = fadd(sha_s1(W[2]), fadd(sha_s0(w5), w4, one), one);                       // W20 (W13 = 0)
    W[5] = fadd(sha_s1(W[3]), fadd(sha_s0(w6), w5, one), one);                       // W21 (W14 = 0)
    W[6] = fadd(sha_s1(W[4]), fadd(sha_s0(w7), fadd(w15, w6, one), one), one);       // W22
    W[7] = fadd(sha_s1(W[5]), fadd(sha_s0(w8), fadd(W[0], w7, one), one), one);      // W23
    W[8] = fadd(sha_s1(W[6]), fadd(sha_s0(w9), fadd(W[1], w8, one), one), one);      // W24
    W[9] = fadd(sha_s1(W[7]), fadd(sha_s0(w10), fadd(W[2], w9, one), one), one);     // W25
    W[10] = fadd(sha_s1(W[8]), fadd(sha_s0(w11), fadd(W[3], w10, one), one), one);   // W26
    W[11] = fadd(sha_s1(W[9]), fadd(sha_s0(w12), fadd(W[4], w11, one), one), one);   // W27
    W[12] = fadd(sha_s1(W[10]), fadd(W[5], w12, one), one);                          // W28 (sigma0(W13) = 0)
    W[13] = fadd(sha_s1(W[11]), W[6], one);                                          // W29 (W13 = W14 = 0)
    W[14] = fadd(sha_s1(W[12]), fadd(W[7], s0w15, one), one);                        // W30 (W14 = 0)
    W[15] = fadd(sha_s1(W[13]), fadd(sha_s0(W[0]), fadd(W[8], w15, one), one), one); // W31
    uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
    {
        constexpr int FMA = FMA_B;  // rounds 16..31
        SHA_16_ROUNDS(sha_k, 16);
    }
    st[0] = a; st[1] = b; st[2] = c; st[3] = d; st[4] = e; st[5] = f; st[6] = g; st[7] = h;
}

// ---- onetime_seed specialisation: F(x0 || be32 j) for all j of an epoch ----
// The message is x0 (4 words, per epoch), W4 = j and the constants
// W5 = 0x80000000, W6..W14 = 0, W15 = 160. Hence W16..W18 are per-epoch
// constants, and in W19..W31 every sigma0 term and the W_{t-16} / W_{t-7}
// terms drawn from W5..W15 are compile-time or per-epoch constants. OtsEpoch
// holds the per-epoch values; ots_head_rounds runs rounds 4..31 with the
// reduced schedule (13 sigma1 evaluations and one sigma0 instead of 16 of
// each) and leaves W = W16..W31 for sha256_rounds_loop(.., 32, ..).
struct OtsEpoch {
    uint32_t w16, w17, w18;
    uint32_t c19;  // sigma1(W17) + W3
    uint32_t c20;  // sigma1(W18) + sigma0(0x80000000)
    uint32_t c31;  // sigma0(W16) + 160
};

PHD OtsEpoch ots_epoch_consts(const uint32_t x0w[4]) {
    OtsEpoch E;
    E.w16 = sha_s0(x0w[1]) + x0w[0];
    E.w17 = sha_s1(160u) + sha_s0(x0w[2]) + x0w[1];
    E.w18 = sha_s1(E.w16) + sha_s0(x0w[3]) + x0w[2];
    E.c19 = sha_s1(E.w17) + x0w[3];
    E.c20 = sha_s1(E.w18) + sha_s0(0x80000000u);
    E.c31 = sha_s0(E.w16) + 160u;
    return E;
}

template <int FMA_H = 2, int FMA_B = FMA_H>  // FMA_B: pipe assignment of rounds 16..31
PHD void ots_head_rounds(uint32_t st[8], uint32_t W[16], uint32_t j, const OtsEpoch& E, const PipeK& pk) {
    constexpr int FMA = FMA_H;
    const uint32_t one = pk.one;
    (void)one;
    // rounds 4..15: W4 = j, the rest compile-time constants
    const uint32_t Wm[16] = {0, 0, 0, 0, j, 0x80000000u, 0, 0, 0, 0, 0, 0, 0, 0, 0, 160u};
    sha256_rounds_head<FMA, 0xffe0u>(st, Wm, 4, pk);  // W5..W15 constant
    // schedule words 16..31
    W[0] = E.w16;
    W[1] = E.w17;
    W[2] = E.w18;
    W[3] = fadd(sha_s0(j), E.c19, one);
    W[4] = fadd(j, E.c20, one);
    W[5] = sha_s1(W[3]) + 0x80000000u;
    W[6] = sha_s1(W[4]) + 160u;
    W[7] = fadd(sha_s1(W[5]), W[0], one);
    W[8] = fadd(sha_s1(W[6]), W[1], one);
    W[9] = fadd(sha_s1(W[7]), W[2], one);
    W[10] = fadd(sha_s1(W[8]), W[3], one);
    W[11] = fadd(sha_s1(W[9]), W[4], one);
    W[12] = fadd(sha_s1(W[10]), W[5], one);
    W[13] = fadd(sha_s1(W[11]), W[6], one);
    W[14] = fadd(sha_s1(W[12]), W[7] + sha_s0(160u), one);
    W[15] = fadd(sha_s1(W[13]), fadd(W[8], E.c31, one), one);
    uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6], h = st[7];
    {
        constexpr int FMA = FMA_B;  // rounds 16..31
        SHA_16_ROUNDS(sha_k, 16);
    }
    st[0] = a; st[1] = b; st[2] = c; st[3] = d; st[4] = e; st[5] = f; st[6] = g; st[7] = h;
}

// Suite-1 per-entry digest pair for a 32-byte entry in compact form: one
// loop over the three compressions (onetime_seed resumed at round 4 from
// the hoisted mid-state, then H(m||x) and H(0x01||m||x)) sharing one copy of
// the round code. Output as in h2s_sha256_len32.
template <int FMA = 0>
PHD void entry_limbs_s1_l32_compact(const uint32_t x0w[4], const uint32_t pre[8], uint32_t j,
                                    const uint32_t m[8], uint32_t limbs[16], const PipeK& pk) {
    uint32_t x[4] = {0, 0, 0, 0};
#pragma unroll 1
    for (int c = 0; c < 3; c++) {
        uint32_t W[16], st[8];
        int r0 = 0;
        if (c == 0) {
            W[0] = x0w[0]; W[1] = x0w[1]; W[2] = x0w[2]; W[3] = x0w[3];
            W[4] = j; W[5] = 0x80000000u;
#pragma unroll
            for (int k = 6; k < 15; k++) W[k] = 0;
            W[15] = 160u;
#pragma unroll
            for (int k = 0; k < 8; k++) st[k] = pre[k];
            r0 = 4;
        } else if (c == 1) {
#pragma unroll
            for (int k = 0; k < 8; k++) W[k] = m[k];
            W[8] = x[0]; W[9] = x[1]; W[10] = x[2]; W[11] = x[3];
            W[12] = 0x80000000u; W[13] = 0; W[14] = 0; W[15] = 384u;
            sha256_init(st);
        } else {
            W[0] = 0x01000000u | (m[0] >> 8);
#pragma unroll
            for (int k = 1; k < 8; k++) W[k] = fshr32(m[k], m[k - 1], 8);
            W[8] = fshr32(x[0], m[7], 8);
            W[9] = fshr32(x[1], x[0], 8);
            W[10] = fshr32(x[2], x[1], 8);
            W[11] = fshr32(x[3], x[2], 8);
            W[12] = (x[3] << 24) | 0x00800000u;
            W[13] = 0; W[14] = 0; W[15] = 392u;
            sha256_init(st);
        }
        sha256_rounds_compact<FMA>(st, W, r0, pk);
        const uint32_t iv[8] = {SHA_IV0, SHA_IV1, SHA_IV2, SHA_IV3, SHA_IV4, SHA_IV5, SHA_IV6, SHA_IV7};
        if (c == 0) {
#pragma unroll
            for (int k = 0; k < 4; k++) x[k] = st[k] + iv[k];
        } else if (c == 1) {
#pragma unroll
            for (int k = 0; k < 8; k++) limbs[15 - k] = st[k] + iv[k];
        } else {
#pragma unroll
            for (int k = 0; k < 8; k++) limbs[7 - k] = st[k] + iv[k];
        }
    }
}
