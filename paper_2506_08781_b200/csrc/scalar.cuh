// Z_l arithmetic for the segmented modular sum.
//
// Replaces Scalar::reduce_wide_be (group.cpp:51-59) + Scalar::add
// (group.cpp:68-73), i.e. libsodium's crypto_core_ristretto255_scalar_reduce
// and _scalar_add, with DEFERRED reduction: the raw 512-bit digests
// H(m||x) || H(0x01||m||x) are summed exactly in a 17-limb (544-bit)
// accumulator and reduced mod l once per segment. This is exact because
// sum(D_i mod l) == (sum D_i) mod l; 2^32 digests of < 2^512 fit in 544 bits.
//
// l = 2^252 + c, c = 27742317777372353535851937790883648493 (125 bits).
#pragma once
#include "poslo_common.cuh"

#define SC_L0 0x5cf5d3edu
#define SC_L1 0x5812631au
#define SC_L2 0xa2f79cd6u
#define SC_L3 0x14def9deu
#define SC_L7 0x10000000u

// acc[0..16] += v[0..15] (little-endian 32-bit limbs), full carry chain.
PHD void acc17_add16(uint32_t acc[17], const uint32_t v[16]) {
#ifdef __CUDA_ARCH__
    asm("add.cc.u32 %0, %0, %17;\n\t"
        "addc.cc.u32 %1, %1, %18;\n\t"
        "addc.cc.u32 %2, %2, %19;\n\t"
        "addc.cc.u32 %3, %3, %20;\n\t"
        "addc.cc.u32 %4, %4, %21;\n\t"
        "addc.cc.u32 %5, %5, %22;\n\t"
        "addc.cc.u32 %6, %6, %23;\n\t"
        "addc.cc.u32 %7, %7, %24;\n\t"
        "addc.cc.u32 %8, %8, %25;\n\t"
        "addc.cc.u32 %9, %9, %26;\n\t"
        "addc.cc.u32 %10, %10, %27;\n\t"
        "addc.cc.u32 %11, %11, %28;\n\t"
        "addc.cc.u32 %12, %12, %29;\n\t"
        "addc.cc.u32 %13, %13, %30;\n\t"
        "addc.cc.u32 %14, %14, %31;\n\t"
        "addc.cc.u32 %15, %15, %32;\n\t"
        "addc.u32 %16, %16, 0;\n\t"
        : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2]), "+r"(acc[3]), "+r"(acc[4]), "+r"(acc[5]),
          "+r"(acc[6]), "+r"(acc[7]), "+r"(acc[8]), "+r"(acc[9]), "+r"(acc[10]), "+r"(acc[11]),
          "+r"(acc[12]), "+r"(acc[13]), "+r"(acc[14]), "+r"(acc[15]), "+r"(acc[16])
        : "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
          "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
          "r"(v[15]));
#else
    uint64_t c = 0;
    for (int i = 0; i < 16; i++) {
        c += (uint64_t)acc[i] + v[i];
        acc[i] = (uint32_t)c;
        c >>= 32;
    }
    acc[16] += (uint32_t)c;
#endif
}

// acc[0..16] += v[0..16].
PHD void acc17_add17(uint32_t acc[17], const uint32_t v[17]) {
#ifdef __CUDA_ARCH__
    asm("add.cc.u32 %0, %0, %17;\n\t"
        "addc.cc.u32 %1, %1, %18;\n\t"
        "addc.cc.u32 %2, %2, %19;\n\t"
        "addc.cc.u32 %3, %3, %20;\n\t"
        "addc.cc.u32 %4, %4, %21;\n\t"
        "addc.cc.u32 %5, %5, %22;\n\t"
        "addc.cc.u32 %6, %6, %23;\n\t"
        "addc.cc.u32 %7, %7, %24;\n\t"
        "addc.cc.u32 %8, %8, %25;\n\t"
        "addc.cc.u32 %9, %9, %26;\n\t"
        "addc.cc.u32 %10, %10, %27;\n\t"
        "addc.cc.u32 %11, %11, %28;\n\t"
        "addc.cc.u32 %12, %12, %29;\n\t"
        "addc.cc.u32 %13, %13, %30;\n\t"
        "addc.cc.u32 %14, %14, %31;\n\t"
        "addc.cc.u32 %15, %15, %32;\n\t"
        "addc.u32 %16, %16, %33;\n\t"
        : "+r"(acc[0]), "+r"(acc[1]), "+r"(acc[2]), "+r"(acc[3]), "+r"(acc[4]), "+r"(acc[5]),
          "+r"(acc[6]), "+r"(acc[7]), "+r"(acc[8]), "+r"(acc[9]), "+r"(acc[10]), "+r"(acc[11]),
          "+r"(acc[12]), "+r"(acc[13]), "+r"(acc[14]), "+r"(acc[15]), "+r"(acc[16])
        : "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
          "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
          "r"(v[15]), "r"(v[16]));
#else
    uint64_t c = 0;
    for (int i = 0; i < 17; i++) {
        c += (uint64_t)acc[i] + v[i];
        acc[i] = (uint32_t)c;
        c >>= 32;
    }
#endif
}

PHD void acc17_zero(uint32_t acc[17]) {
#pragma unroll
    for (int i = 0; i < 17; i++) acc[i] = 0;
}

// One Horner step in radix 2^32: r <- (r * 2^32 + limb) mod l, r canonical.
// v = r*2^32 + limb < 2^285; q = v >> 252 < 2^33; v == q*2^252 + lo with
// 2^252 == -c (mod l), so v == lo - q*c where lo < 2^252 < l and
// q*c < 2^158 < l: one conditional +l lands in [0, l).
PHD void sc_horner_step(uint32_t r[8], uint32_t limb) {
    uint32_t v[9];
    v[0] = limb;
#pragma unroll
    for (int i = 0; i < 8; i++) v[i + 1] = r[i];
    uint64_t q = ((uint64_t)v[8] << 4) | (v[7] >> 28);
    v[7] &= 0x0fffffffu;
    // p = q * c (q < 2^33, c < 2^125) as 6 limbs
    const uint32_t c[4] = {SC_L0, SC_L1, SC_L2, SC_L3};
    uint32_t qlo = (uint32_t)q, qhi = (uint32_t)(q >> 32);
    uint32_t p[6];
    uint64_t carry = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        uint64_t t = (uint64_t)qlo * c[i] + carry;
        p[i] = (uint32_t)t;
        carry = t >> 32;
    }
    p[4] = (uint32_t)carry;
    p[5] = 0;
    // qhi in {0,1}: p += (qhi * c) << 32
    uint64_t cc = 0;
#pragma unroll
    for (int i = 0; i < 4; i++) {
        cc += (uint64_t)p[i + 1] + (qhi ? c[i] : 0u);
        p[i + 1] = (uint32_t)cc;
        cc >>= 32;
    }
    p[5] += (uint32_t)cc;
    // r = lo - p (mod 2^256), then + l on borrow
    int64_t bw = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        int64_t t = (int64_t)v[i] - (i < 6 ? (int64_t)p[i] : 0) + bw;
        r[i] = (uint32_t)t;
        bw = t >> 32;  // 0 or -1
    }
    if (bw) {
        const uint32_t L[8] = {SC_L0, SC_L1, SC_L2, SC_L3, 0, 0, 0, SC_L7};
        uint64_t s = 0;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            s += (uint64_t)r[i] + L[i];
            r[i] = (uint32_t)s;
            s >>= 32;
        }
    }
}

// out = (v[0..n-1] little-endian limbs) mod l, canonical.
PHD void sc_reduce_limbs(const uint32_t* v, int n, uint32_t out[8]) {
#pragma unroll
    for (int i = 0; i < 8; i++) out[i] = 0;
    for (int k = n - 1; k >= 0; k--) sc_horner_step(out, v[k]);
}

// (a + b) mod l for canonical a, b.
PHD void sc_add(const uint32_t a[8], const uint32_t b[8], uint32_t out[8]) {
    const uint32_t L[8] = {SC_L0, SC_L1, SC_L2, SC_L3, 0, 0, 0, SC_L7};
    uint32_t s[8], d[8];
    uint64_t c = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        c += (uint64_t)a[i] + b[i];
        s[i] = (uint32_t)c;
        c >>= 32;
    }
    // a + b < 2l < 2^254: no carry out of limb 7
    int64_t bw = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        int64_t t = (int64_t)s[i] - L[i] + bw;
        d[i] = (uint32_t)t;
        bw = t >> 32;
    }
#pragma unroll
    for (int i = 0; i < 8; i++) out[i] = bw ? s[i] : d[i];
}

PHD bool sc_is_zero(const uint32_t a[8]) {
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) x |= a[i];
    return x == 0;
}

// (a * b) mod l for canonical a, b (Scalar::mul, group.cpp:82-87): the
// 512-bit product by column sums, then one Horner reduction.
PHD void sc_mul(const uint32_t a[8], const uint32_t b[8], uint32_t out[8]) {
    uint32_t t[16];
    uint64_t carry = 0;
    for (int k = 0; k < 15; k++) {
        uint64_t lo = carry & 0xffffffffu, hi = carry >> 32;
        for (int i = 0; i < 8; i++) {
            const int j = k - i;
            if (j < 0 || j > 7) continue;
            const uint64_t p = (uint64_t)a[i] * b[j];
            lo += p & 0xffffffffu;
            hi += p >> 32;
        }
        hi += lo >> 32;
        t[k] = (uint32_t)lo;
        carry = hi;
    }
    t[15] = (uint32_t)carry;
    sc_reduce_limbs(t, 16, out);
}

// (a - b) mod l for canonical a, b (Scalar::sub): a + (l - b), reduced.
PHD void sc_sub(const uint32_t a[8], const uint32_t b[8], uint32_t out[8]) {
    const uint32_t L[8] = {SC_L0, SC_L1, SC_L2, SC_L3, 0, 0, 0, SC_L7};
    uint32_t nb[8];
    int64_t bw = 0;
    for (int i = 0; i < 8; i++) {  // l - b >= 1 for b < l (and = l for b = 0, reduced below)
        const int64_t t = (int64_t)L[i] - b[i] + bw;
        nb[i] = (uint32_t)t;
        bw = t >> 32;
    }
    uint32_t sum[9];
    uint64_t c = 0;
    for (int i = 0; i < 8; i++) {
        c += (uint64_t)a[i] + nb[i];
        sum[i] = (uint32_t)c;
        c >>= 32;
    }
    sum[8] = (uint32_t)c;
    sc_reduce_limbs(sum, 9, out);
}

