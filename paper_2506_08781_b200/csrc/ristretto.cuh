// ristretto255 over edwards25519 for the device group check (stage 3).
//
// Replaces the libsodium calls behind the reference's group layer
// (proj/src/group.cpp): crypto_core_ristretto255_is_valid_point (:107-114),
// crypto_scalarmult_ristretto255 / _base and _add inside commit_check
// (:144-167) and group_combine (:169-178), plus the byte-equality of
// GroupElement::operator== (include/poslo/group.hpp:59).
//
// Field GF(2^255-19): 8 x 32-bit limbs, values kept loosely in [0, 2^256)
// and canonicalised only for encode/compare (2^256 == 38 mod p). Points are
// extended twisted-Edwards (X:Y:Z:T), a = -1. Ristretto decode/encode and
// SQRT_RATIO_M1 follow the published ristretto255 definition (RFC 9496 §4);
// constants were derived from their definitions (oracle/ristretto.py) and the
// whole layer is pinned against the reference's own outputs
// (tests/golden/kat.json) on CPU (tests/native) and GPU (tests/test_gpu_*).
//
// Verification handles public data only, so everything is variable-time.
#pragma once
#include "poslo_common.cuh"

#define FE_D_LIMBS 0x135978a3u, 0x75eb4dcau, 0x4141d8abu, 0x00700a4du, 0x7779e898u, 0x8cc74079u, 0x2b6ffe73u, 0x52036ceeu
#define FE_D2_LIMBS 0x26b2f159u, 0xebd69b94u, 0x8283b156u, 0x00e0149au, 0xeef3d130u, 0x198e80f2u, 0x56dffce7u, 0x2406d9dcu
#define FE_SQRTM1_LIMBS 0x4a0ea0b0u, 0xc4ee1b27u, 0xad2fe478u, 0x2f431806u, 0x3dfbd7a7u, 0x2b4d0099u, 0x4fc1df0bu, 0x2b832480u
#define FE_INVSQRT_A_MINUS_D_LIMBS 0x805d40eau, 0x99c8fdaau, 0x5a4172beu, 0x9d2f1617u, 0xfe01d840u, 0x16c27b91u, 0xcfaffca2u, 0x786c8905u
#define FE_BASE_X_LIMBS 0x8f25d51au, 0xc9562d60u, 0x9525a7b2u, 0x692cc760u, 0xfdd6dc5cu, 0xc0a4e231u, 0xcd6e53feu, 0x216936d3u
#define FE_BASE_Y_LIMBS 0x66666658u, 0x66666666u, 0x66666666u, 0x66666666u, 0x66666666u, 0x66666666u, 0x66666666u, 0x66666666u
#define FE_BASE_T_LIMBS 0xa5b7dda3u, 0x6dde8ab3u, 0x775152f5u, 0x20f09f80u, 0x64abe37du, 0x66ea4e8eu, 0xd78b7665u, 0x67875f0fu

struct fe {
    uint32_t v[8];
};

struct gpt {  // extended coordinates, x = X/Z, y = Y/Z, xy = T/Z
    fe X, Y, Z, T;
};

PHD fe fe_from(const uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t a4, uint32_t a5,
               uint32_t a6, uint32_t a7) {
    fe r;
    r.v[0] = a0; r.v[1] = a1; r.v[2] = a2; r.v[3] = a3;
    r.v[4] = a4; r.v[5] = a5; r.v[6] = a6; r.v[7] = a7;
    return r;
}
#define FE_CONST(LIMBS) fe_from(LIMBS)

PHD fe fe_zero() { return fe_from(0, 0, 0, 0, 0, 0, 0, 0); }
PHD fe fe_one() { return fe_from(1, 0, 0, 0, 0, 0, 0, 0); }

// r = a + 38 * c folded until no carry remains (c is the overflow count).
PHD void fe_fold(uint32_t r[8], uint64_t c) {
    for (int pass = 0; pass < 2; pass++) {
        uint64_t t = c * 38;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            t += r[i];
            r[i] = (uint32_t)t;
            t >>= 32;
        }
        c = t;
    }
}

PHD fe fe_add(const fe& a, const fe& b) {
    fe r;
    uint64_t c = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        c += (uint64_t)a.v[i] + b.v[i];
        r.v[i] = (uint32_t)c;
        c >>= 32;
    }
    fe_fold(r.v, c);
    return r;
}

PHD fe fe_sub(const fe& a, const fe& b) {
    fe r;
    int64_t bw = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        int64_t t = (int64_t)a.v[i] - b.v[i] + bw;
        r.v[i] = (uint32_t)t;
        bw = t >> 32;
    }
    // a wrapped: true value = r - 2^256 == r - 38 (mod p); at most twice
    for (int pass = 0; pass < 2 && bw; pass++) {
        int64_t t2 = -38;
        bw = 0;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            int64_t t = (int64_t)r.v[i] + (i == 0 ? t2 : 0) + bw;
            r.v[i] = (uint32_t)t;
            bw = t >> 32;
        }
    }
    return r;
}

#ifdef __CUDA_ARCH__
// 8x8-limb product with carry-flag chains (two per row: low and high
// halves), then the 2^256 == 38 fold: ~170 instructions, about half of the
// portable C version. Identical results (tests/native + GPU parity tests).
__device__ __forceinline__ fe fe_mul_ptx(const fe& a, const fe& b) {
    fe r;
    asm("{\n\t.reg .u32 r<16>;\n\tmov.u32 r0, 0;\n\tmov.u32 r1, 0;\n\tmov.u32 r2, 0;\n\tmov.u32 r3, 0;\n\tmov.u32 r4, 0;\n\tmov.u32 r5, 0;\n\tmov.u32 r6, 0;\n\tmov.u32 r7, 0;\n\tmov.u32 r8, 0;\n\tmov.u32 r9, 0;\n\tmov.u32 r10, 0;\n\tmov.u32 r11, 0;\n\tmov.u32 r12, 0;\n\tmov.u32 r13, 0;\n\tmov.u32 r14, 0;\n\tmov.u32 r15, 0;\n\tmad.lo.cc.u32 r0, %8, %16, r0;\n\tmadc.lo.cc.u32 r1, %9, %16, r1;\n\tmadc.lo.cc.u32 r2, %10, %16, r2;\n\tmadc.lo.cc.u32 r3, %11, %16, r3;\n\tmadc.lo.cc.u32 r4, %12, %16, r4;\n\tmadc.lo.cc.u32 r5, %13, %16, r5;\n\tmadc.lo.cc.u32 r6, %14, %16, r6;\n\tmadc.lo.cc.u32 r7, %15, %16, r7;\n\taddc.u32 r8, 0, 0;\n\tmad.hi.cc.u32 r1, %8, %16, r1;\n\tmadc.hi.cc.u32 r2, %9, %16, r2;\n\tmadc.hi.cc.u32 r3, %10, %16, r3;\n\tmadc.hi.cc.u32 r4, %11, %16, r4;\n\tmadc.hi.cc.u32 r5, %12, %16, r5;\n\tmadc.hi.cc.u32 r6, %13, %16, r6;\n\tmadc.hi.cc.u32 r7, %14, %16, r7;\n\tmadc.hi.u32 r8, %15, %16, r8;\n\tmad.lo.cc.u32 r1, %8, %17, r1;\n\tmadc.lo.cc.u32 r2, %9, %17, r2;\n\tmadc.lo.cc.u32 r3, %10, %17, r3;\n\tmadc.lo.cc.u32 r4, %11, %17, r4;\n\tmadc.lo.cc.u32 r5, %12, %17, r5;\n\tmadc.lo.cc.u32 r6, %13, %17, r6;\n\tmadc.lo.cc.u32 r7, %14, %17, r7;\n\tmadc.lo.cc.u32 r8, %15, %17, r8;\n\taddc.u32 r9, 0, 0;\n\tmad.hi.cc.u32 r2, %8, %17, r2;\n\tmadc.hi.cc.u32 r3, %9, %17, r3;\n\tmadc.hi.cc.u32 r4, %10, %17, r4;\n\tmadc.hi.cc.u32 r5, %11, %17, r5;\n\tmadc.hi.cc.u32 r6, %12, %17, r6;\n\tmadc.hi.cc.u32 r7, %13, %17, r7;\n\tmadc.hi.cc.u32 r8, %14, %17, r8;\n\tmadc.hi.u32 r9, %15, %17, r9;\n\tmad.lo.cc.u32 r2, %8, %18, r2;\n\tmadc.lo.cc.u32 r3, %9, %18, r3;\n\tmadc.lo.cc.u32 r4, %10, %18, r4;\n\tmadc.lo.cc.u32 r5, %11, %18, r5;\n\tmadc.lo.cc.u32 r6, %12, %18, r6;\n\tmadc.lo.cc.u32 r7, %13, %18, r7;\n\tmadc.lo.cc.u32 r8, %14, %18, r8;\n\tmadc.lo.cc.u32 r9, %15, %18, r9;\n\taddc.u32 r10, 0, 0;\n\tmad.hi.cc.u32 r3, %8, %18, r3;\n\tmadc.hi.cc.u32 r4, %9, %18, r4;\n\tmadc.hi.cc.u32 r5, %10, %18, r5;\n\tmadc.hi.cc.u32 r6, %11, %18, r6;\n\tmadc.hi.cc.u32 r7, %12, %18, r7;\n\tmadc.hi.cc.u32 r8, %13, %18, r8;\n\tmadc.hi.cc.u32 r9, %14, %18, r9;\n\tmadc.hi.u32 r10, %15, %18, r10;\n\tmad.lo.cc.u32 r3, %8, %19, r3;\n\tmadc.lo.cc.u32 r4, %9, %19, r4;\n\tmadc.lo.cc.u32 r5, %10, %19, r5;\n\tmadc.lo.cc.u32 r6, %11, %19, r6;\n\tmadc.lo.cc.u32 r7, %12, %19, r7;\n\tmadc.lo.cc.u32 r8, %13, %19, r8;\n\tmadc.lo.cc.u32 r9, %14, %19, r9;\n\tmadc.lo.cc.u32 r10, %15, %19, r10;\n\taddc.u32 r11, 0, 0;\n\tmad.hi.cc.u32 r4, %8, %19, r4;\n\tmadc.hi.cc.u32 r5, %9, %19, r5;\n\tmadc.hi.cc.u32 r6, %10, %19, r6;\n\tmadc.hi.cc.u32 r7, %11, %19, r7;\n\tmadc.hi.cc.u32 r8, %12, %19, r8;\n\tmadc.hi.cc.u32 r9, %13, %19, r9;\n\tmadc.hi.cc.u32 r10, %14, %19, r10;\n\tmadc.hi.u32 r11, %15, %19, r11;\n\tmad.lo.cc.u32 r4, %8, %20, r4;\n\tmadc.lo.cc.u32 r5, %9, %20, r5;\n\tmadc.lo.cc.u32 r6, %10, %20, r6;\n\tmadc.lo.cc.u32 r7, %11, %20, r7;\n\tmadc.lo.cc.u32 r8, %12, %20, r8;\n\tmadc.lo.cc.u32 r9, %13, %20, r9;\n\tmadc.lo.cc.u32 r10, %14, %20, r10;\n\tmadc.lo.cc.u32 r11, %15, %20, r11;\n\taddc.u32 r12, 0, 0;\n\tmad.hi.cc.u32 r5, %8, %20, r5;\n\tmadc.hi.cc.u32 r6, %9, %20, r6;\n\tmadc.hi.cc.u32 r7, %10, %20, r7;\n\tmadc.hi.cc.u32 r8, %11, %20, r8;\n\tmadc.hi.cc.u32 r9, %12, %20, r9;\n\tmadc.hi.cc.u32 r10, %13, %20, r10;\n\tmadc.hi.cc.u32 r11, %14, %20, r11;\n\tmadc.hi.u32 r12, %15, %20, r12;\n\tmad.lo.cc.u32 r5, %8, %21, r5;\n\tmadc.lo.cc.u32 r6, %9, %21, r6;\n\tmadc.lo.cc.u32 r7, %10, %21, r7;\n\tmadc.lo.cc.u32 r8, %11, %21, r8;\n\tmadc.lo.cc.u32 r9, %12, %21, r9;\n\tmadc.lo.cc.u32 r10, %13, %21, r10;\n\tmadc.lo.cc.u32 r11, %14, %21, r11;\n\tmadc.lo.cc.u32 r12, %15, %21, r12;\n\taddc.u32 r13, 0, 0;\n\tmad.hi.cc.u32 r6, %8, %21, r6;\n\tmadc.hi.cc.u32 r7, %9, %21, r7;\n\tmadc.hi.cc.u32 r8, %10, %21, r8;\n\tmadc.hi.cc.u32 r9, %11, %21, r9;\n\tmadc.hi.cc.u32 r10, %12, %21, r10;\n\tmadc.hi.cc.u32 r11, %13, %21, r11;\n\tmadc.hi.cc.u32 r12, %14, %21, r12;\n\tmadc.hi.u32 r13, %15, %21, r13;\n\tmad.lo.cc.u32 r6, %8, %22, r6;\n\tmadc.lo.cc.u32 r7, %9, %22, r7;\n\tmadc.lo.cc.u32 r8, %10, %22, r8;\n\tmadc.lo.cc.u32 r9, %11, %22, r9;\n\tmadc.lo.cc.u32 r10, %12, %22, r10;\n\tmadc.lo.cc.u32 r11, %13, %22, r11;\n\tmadc.lo.cc.u32 r12, %14, %22, r12;\n\tmadc.lo.cc.u32 r13, %15, %22, r13;\n\taddc.u32 r14, 0, 0;\n\tmad.hi.cc.u32 r7, %8, %22, r7;\n\tmadc.hi.cc.u32 r8, %9, %22, r8;\n\tmadc.hi.cc.u32 r9, %10, %22, r9;\n\tmadc.hi.cc.u32 r10, %11, %22, r10;\n\tmadc.hi.cc.u32 r11, %12, %22, r11;\n\tmadc.hi.cc.u32 r12, %13, %22, r12;\n\tmadc.hi.cc.u32 r13, %14, %22, r13;\n\tmadc.hi.u32 r14, %15, %22, r14;\n\tmad.lo.cc.u32 r7, %8, %23, r7;\n\tmadc.lo.cc.u32 r8, %9, %23, r8;\n\tmadc.lo.cc.u32 r9, %10, %23, r9;\n\tmadc.lo.cc.u32 r10, %11, %23, r10;\n\tmadc.lo.cc.u32 r11, %12, %23, r11;\n\tmadc.lo.cc.u32 r12, %13, %23, r12;\n\tmadc.lo.cc.u32 r13, %14, %23, r13;\n\tmadc.lo.cc.u32 r14, %15, %23, r14;\n\taddc.u32 r15, 0, 0;\n\tmad.hi.cc.u32 r8, %8, %23, r8;\n\tmadc.hi.cc.u32 r9, %9, %23, r9;\n\tmadc.hi.cc.u32 r10, %10, %23, r10;\n\tmadc.hi.cc.u32 r11, %11, %23, r11;\n\tmadc.hi.cc.u32 r12, %12, %23, r12;\n\tmadc.hi.cc.u32 r13, %13, %23, r13;\n\tmadc.hi.cc.u32 r14, %14, %23, r14;\n\tmadc.hi.u32 r15, %15, %23, r15;\n\t.reg .u32 t8, c38;\n\tmov.u32 c38, 38;\n\tmad.lo.cc.u32 r0, r8, c38, r0;\n\tmadc.lo.cc.u32 r1, r9, c38, r1;\n\tmadc.lo.cc.u32 r2, r10, c38, r2;\n\tmadc.lo.cc.u32 r3, r11, c38, r3;\n\tmadc.lo.cc.u32 r4, r12, c38, r4;\n\tmadc.lo.cc.u32 r5, r13, c38, r5;\n\tmadc.lo.cc.u32 r6, r14, c38, r6;\n\tmadc.lo.cc.u32 r7, r15, c38, r7;\n\taddc.u32 t8, 0, 0;\n\tmad.hi.cc.u32 r1, r8, c38, r1;\n\tmadc.hi.cc.u32 r2, r9, c38, r2;\n\tmadc.hi.cc.u32 r3, r10, c38, r3;\n\tmadc.hi.cc.u32 r4, r11, c38, r4;\n\tmadc.hi.cc.u32 r5, r12, c38, r5;\n\tmadc.hi.cc.u32 r6, r13, c38, r6;\n\tmadc.hi.cc.u32 r7, r14, c38, r7;\n\tmadc.hi.u32 t8, r15, c38, t8;\n\tmul.lo.u32 t8, t8, c38;\n\tadd.cc.u32 r0, r0, t8;\n\taddc.cc.u32 r1, r1, 0;\n\taddc.cc.u32 r2, r2, 0;\n\taddc.cc.u32 r3, r3, 0;\n\taddc.cc.u32 r4, r4, 0;\n\taddc.cc.u32 r5, r5, 0;\n\taddc.cc.u32 r6, r6, 0;\n\taddc.cc.u32 r7, r7, 0;\n\taddc.u32 t8, 0, 0;\n\tmul.lo.u32 t8, t8, c38;\n\tadd.cc.u32 r0, r0, t8;\n\taddc.cc.u32 r1, r1, 0;\n\taddc.cc.u32 r2, r2, 0;\n\taddc.cc.u32 r3, r3, 0;\n\taddc.cc.u32 r4, r4, 0;\n\taddc.cc.u32 r5, r5, 0;\n\taddc.cc.u32 r6, r6, 0;\n\taddc.cc.u32 r7, r7, 0;\n\taddc.u32 t8, 0, 0;\n\tmov.u32 %0, r0;\n\tmov.u32 %1, r1;\n\tmov.u32 %2, r2;\n\tmov.u32 %3, r3;\n\tmov.u32 %4, r4;\n\tmov.u32 %5, r5;\n\tmov.u32 %6, r6;\n\tmov.u32 %7, r7;\n\t}"
        : "=r"(r.v[0]), "=r"(r.v[1]), "=r"(r.v[2]), "=r"(r.v[3]), "=r"(r.v[4]), "=r"(r.v[5]),
          "=r"(r.v[6]), "=r"(r.v[7])
        : "r"(a.v[0]), "r"(a.v[1]), "r"(a.v[2]), "r"(a.v[3]), "r"(a.v[4]), "r"(a.v[5]), "r"(a.v[6]),
          "r"(a.v[7]), "r"(b.v[0]), "r"(b.v[1]), "r"(b.v[2]), "r"(b.v[3]), "r"(b.v[4]), "r"(b.v[5]),
          "r"(b.v[6]), "r"(b.v[7]));
    return r;
}
#endif

// Product scanning: the 64 32x32 products are independent and every column
// is summed on its own (96-bit column accumulators), so only the final carry
// sweep is serial — short dependency chains for the latency-bound single-
// check path, where the old row-by-row carry chain dominated.
#if defined(__CUDA_ARCH__) && defined(POSLO_FE_CALL)
// Out-of-line field multiplication (~170 SASS instructions): the group
// kernels call it instead of inlining it at every use, which keeps a point
// addition at a few hundred instructions and the kernels inside the
// instruction cache (inlined, k_check_split stalled on no_instruction).
__device__ __noinline__ fe fe_mul_call(fe a, fe b) { return fe_mul_ptx(a, b); }
#endif

PHD fe fe_mul(const fe& a, const fe& b) {
#ifdef __CUDA_ARCH__
#ifdef POSLO_FE_CALL
    return fe_mul_call(a, b);
#else
    return fe_mul_ptx(a, b);
#endif
#endif
    uint32_t t[16];
    uint64_t carry = 0;  // < 2^36
#pragma unroll
    for (int k = 0; k < 15; k++) {
        uint64_t lo = 0;
        uint32_t hi = 0;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int j = k - i;
            if (j < 0 || j > 7) continue;
            const uint64_t p = (uint64_t)a.v[i] * b.v[j];
            lo += p;
            hi += lo < p;
        }
        lo += carry;
        hi += lo < carry;
        t[k] = (uint32_t)lo;
        carry = (lo >> 32) | ((uint64_t)hi << 32);
    }
    t[15] = (uint32_t)carry;
    // 2^256 == 38 (mod p): r = t_lo + 38 * t_hi, folded twice
    fe r;
    uint64_t c = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        c += (uint64_t)t[i] + (uint64_t)t[i + 8] * 38;
        r.v[i] = (uint32_t)c;
        c >>= 32;
    }
    fe_fold(r.v, c);
    return r;
}

PHD fe fe_sq(const fe& a) { return fe_mul(a, a); }

PHD fe fe_sqn(fe a, int n) {
    for (int i = 0; i < n; i++) a = fe_sq(a);
    return a;
}

// Canonical representative in [0, p).
PHD fe fe_canon(const fe& a) {
    fe r = a;
    // fold bit 255: r = (r mod 2^255) + 19 * (r >> 255)  (< 2^255 + 19)
    uint32_t top = r.v[7] >> 31;
    r.v[7] &= 0x7fffffffu;
    uint64_t c = (uint64_t)top * 19;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        c += r.v[i];
        r.v[i] = (uint32_t)c;
        c >>= 32;
    }
    // r >= p  <=>  r + 19 >= 2^255
    fe s;
    c = 19;
#pragma unroll
    for (int i = 0; i < 8; i++) {
        c += r.v[i];
        s.v[i] = (uint32_t)c;
        c >>= 32;
    }
    if (s.v[7] >> 31) {
        s.v[7] &= 0x7fffffffu;
        return s;
    }
    return r;
}

PHD bool fe_is_neg(const fe& a) { return fe_canon(a).v[0] & 1; }

PHD bool fe_is_zero(const fe& a) {
    fe c = fe_canon(a);
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 8; i++) x |= c.v[i];
    return x == 0;
}

PHD bool fe_eq(const fe& a, const fe& b) { return fe_is_zero(fe_sub(a, b)); }

PHD fe fe_neg(const fe& a) { return fe_sub(fe_zero(), a); }

PHD fe fe_abs(const fe& a) { return fe_is_neg(a) ? fe_neg(a) : a; }

// z^((p-5)/8) = z^(2^252 - 3)
PHD fe fe_pow22523(const fe& z) {
    fe z2 = fe_sq(z);
    fe z3 = fe_mul(z2, z);                       // 2^2 - 1
    fe z15 = fe_mul(fe_sqn(z3, 2), z3);          // 2^4 - 1
    fe z31 = fe_mul(fe_sq(z15), z);              // 2^5 - 1
    fe z10 = fe_mul(fe_sqn(z31, 5), z31);        // 2^10 - 1
    fe z20 = fe_mul(fe_sqn(z10, 10), z10);       // 2^20 - 1
    fe z40 = fe_mul(fe_sqn(z20, 20), z20);       // 2^40 - 1
    fe z50 = fe_mul(fe_sqn(z40, 10), z10);       // 2^50 - 1
    fe z100 = fe_mul(fe_sqn(z50, 50), z50);      // 2^100 - 1
    fe z200 = fe_mul(fe_sqn(z100, 100), z100);   // 2^200 - 1
    fe z250 = fe_mul(fe_sqn(z200, 50), z50);     // 2^250 - 1
    return fe_mul(fe_sqn(z250, 2), z);           // 2^252 - 3
}

// SQRT_RATIO_M1(u, v): returns was_square, r = non-negative root.
PHD bool fe_sqrt_ratio_m1(const fe& u, const fe& v, fe& r) {
    const fe sqrtm1 = FE_CONST(FE_SQRTM1_LIMBS);
    fe v3 = fe_mul(fe_sq(v), v);
    fe v7 = fe_mul(fe_sq(v3), v);
    r = fe_mul(fe_mul(u, v3), fe_pow22523(fe_mul(u, v7)));
    fe check = fe_mul(v, fe_sq(r));
    fe nu = fe_neg(u);
    bool correct = fe_eq(check, u);
    bool flipped = fe_eq(check, nu);
    bool flipped_i = fe_eq(check, fe_mul(nu, sqrtm1));
    if (flipped || flipped_i) r = fe_mul(r, sqrtm1);
    r = fe_abs(r);
    return correct || flipped;
}

PHD fe fe_from_bytes_le(const uint8_t b[32]) {
    fe r;
#pragma unroll
    for (int i = 0; i < 8; i++)
        r.v[i] = (uint32_t)b[4 * i] | (uint32_t)b[4 * i + 1] << 8 | (uint32_t)b[4 * i + 2] << 16 |
                 (uint32_t)b[4 * i + 3] << 24;
    return r;
}

PHD void fe_to_bytes_le(const fe& a, uint8_t b[32]) {
    fe c = fe_canon(a);
#pragma unroll
    for (int i = 0; i < 8; i++) {
        b[4 * i] = (uint8_t)c.v[i];
        b[4 * i + 1] = (uint8_t)(c.v[i] >> 8);
        b[4 * i + 2] = (uint8_t)(c.v[i] >> 16);
        b[4 * i + 3] = (uint8_t)(c.v[i] >> 24);
    }
}

PHD gpt pt_identity() {
    gpt p;
    p.X = fe_zero(); p.Y = fe_one(); p.Z = fe_one(); p.T = fe_zero();
    return p;
}

PHD gpt pt_base() {
    gpt p;
    p.X = FE_CONST(FE_BASE_X_LIMBS);
    p.Y = FE_CONST(FE_BASE_Y_LIMBS);
    p.Z = fe_one();
    p.T = FE_CONST(FE_BASE_T_LIMBS);
    return p;
}

// add-2008-hwcd-3 (a = -1, k = 2d)
PHD gpt pt_add(const gpt& p, const gpt& q) {
    const fe d2 = FE_CONST(FE_D2_LIMBS);
    fe A = fe_mul(fe_sub(p.Y, p.X), fe_sub(q.Y, q.X));
    fe B = fe_mul(fe_add(p.Y, p.X), fe_add(q.Y, q.X));
    fe C = fe_mul(fe_mul(p.T, d2), q.T);
    fe D = fe_mul(fe_add(p.Z, p.Z), q.Z);
    fe E = fe_sub(B, A), F = fe_sub(D, C), G = fe_add(D, C), H = fe_add(B, A);
    gpt r;
    r.X = fe_mul(E, F);
    r.Y = fe_mul(G, H);
    r.T = fe_mul(E, H);
    r.Z = fe_mul(F, G);
    return r;
}

// dbl-2008-hwcd (a = -1): D = -A, G = B - A, F = G - C, H = -A - B
PHD gpt pt_dbl(const gpt& p) {
    fe A = fe_sq(p.X);
    fe B = fe_sq(p.Y);
    fe C = fe_sq(p.Z);
    C = fe_add(C, C);
    fe E = fe_sub(fe_sub(fe_sq(fe_add(p.X, p.Y)), A), B);
    fe G = fe_sub(B, A);
    fe F = fe_sub(G, C);
    fe H = fe_neg(fe_add(A, B));
    gpt r;
    r.X = fe_mul(E, F);
    r.Y = fe_mul(G, H);
    r.T = fe_mul(E, H);
    r.Z = fe_mul(F, G);
    return r;
}

PHD gpt pt_neg(const gpt& p) {
    gpt r = p;
    r.X = fe_neg(p.X);
    r.T = fe_neg(p.T);
    return r;
}

// Ristretto decode with full validation (RFC 9496 §4.3.1); false = invalid
// encoding, exactly the set crypto_core_ristretto255_is_valid_point rejects.
PHD bool rist_decode(const uint8_t b[32], gpt& out) {
    fe s = fe_from_bytes_le(b);
    // canonical: s < p (so bit 255 clear) and non-negative
    fe sc = fe_canon(s);
    bool canonical = true;
#pragma unroll
    for (int i = 0; i < 8; i++) canonical = canonical && (sc.v[i] == s.v[i]);
    if (!canonical || (s.v[0] & 1)) return false;
    const fe d = FE_CONST(FE_D_LIMBS);
    fe ss = fe_sq(s);
    fe u1 = fe_sub(fe_one(), ss);
    fe u2 = fe_add(fe_one(), ss);
    fe u2sq = fe_sq(u2);
    fe v = fe_sub(fe_neg(fe_mul(d, fe_sq(u1))), u2sq);
    fe inv;
    bool was_square = fe_sqrt_ratio_m1(fe_one(), fe_mul(v, u2sq), inv);
    fe den_x = fe_mul(inv, u2);
    fe den_y = fe_mul(fe_mul(inv, den_x), v);
    fe x = fe_abs(fe_mul(fe_add(s, s), den_x));
    fe y = fe_mul(u1, den_y);
    fe t = fe_mul(x, y);
    if (!was_square || fe_is_neg(t) || fe_is_zero(y)) return false;
    out.X = x;
    out.Y = y;
    out.Z = fe_one();
    out.T = t;
    return true;
}

// Ristretto encode (RFC 9496 §4.3.2) -> 32 canonical bytes.
PHD void rist_encode(const gpt& p, uint8_t out[32]) {
    const fe sqrtm1 = FE_CONST(FE_SQRTM1_LIMBS);
    const fe isqrt_amd = FE_CONST(FE_INVSQRT_A_MINUS_D_LIMBS);
    fe u1 = fe_mul(fe_add(p.Z, p.Y), fe_sub(p.Z, p.Y));
    fe u2 = fe_mul(p.X, p.Y);
    fe inv;
    fe_sqrt_ratio_m1(fe_one(), fe_mul(u1, fe_sq(u2)), inv);
    fe den1 = fe_mul(inv, u1);
    fe den2 = fe_mul(inv, u2);
    fe z_inv = fe_mul(fe_mul(den1, den2), p.T);
    fe ix0 = fe_mul(p.X, sqrtm1);
    fe iy0 = fe_mul(p.Y, sqrtm1);
    fe enchanted = fe_mul(den1, isqrt_amd);
    bool rotate = fe_is_neg(fe_mul(p.T, z_inv));
    fe x = rotate ? iy0 : p.X;
    fe y = rotate ? ix0 : p.Y;
    fe den_inv = rotate ? enchanted : den2;
    if (fe_is_neg(fe_mul(x, z_inv))) y = fe_neg(y);
    fe s = fe_abs(fe_mul(den_inv, fe_sub(p.Z, y)));
    fe_to_bytes_le(s, out);
}

// Scalar bit i of a canonical 32-byte little-endian scalar held as 8 limbs.
PHD int sc_bit(const uint32_t s[8], int i) { return (s[i >> 5] >> (i & 31)) & 1; }

// Y^e * alpha^s as a point: joint (Shamir) double-and-add over 253 bits.
PHD gpt double_scalarmult(const gpt& Y, const uint32_t e[8], const uint32_t s[8]) {
    gpt B = pt_base();
    gpt YB = pt_add(Y, B);
    gpt acc = pt_identity();
    bool started = false;
    for (int i = 252; i >= 0; i--) {
        if (started) acc = pt_dbl(acc);
        int be = sc_bit(e, i), bs = sc_bit(s, i);
        if (be | bs) {
            const gpt& q = (be && bs) ? YB : (be ? Y : B);
            acc = started ? pt_add(acc, q) : q;
            started = true;
        }
    }
    return acc;
}

// commit_check(Y, e, s) (group.cpp:144-167) -> encoding of Y^e * alpha^s.
PHD void commit_check_enc(const gpt& Y, const uint32_t e[8], const uint32_t s[8], uint8_t out[32]) {
    gpt P = double_scalarmult(Y, e, s);
    rist_encode(P, out);
}

// ---- fixed-base comb tables (stage 3 v2) ---------------------------------
// For a base P: tab[8k + i] = (i+1) * 16^k * P, k = 0..63, i = 0..7, in
// affine Niels form (y+x, y-x, 2dxy) with Z = 1, so one table addition (a
// mixed addition) costs 7 multiplications. With signed radix-16 digits
// s = sum d_k 16^k, d_k in [-8, 8), a scalar multiplication is 64 table
// additions and NO doublings. Y is fixed per public key and alpha forever,
// so both exponentiations of commit_check are fixed-base (SURVEY.md §7.5).
struct gcached {
    fe YpX, YmX, T2d;
};

// z^(p-2) = z^(2^255 - 21)
PHD fe fe_invert(const fe& z) {
    fe z2 = fe_sq(z);
    fe z9 = fe_mul(fe_sqn(z2, 2), z);            // z^9
    fe z11 = fe_mul(z9, z2);                     // z^11
    fe z5 = fe_mul(fe_sq(z11), z9);              // 2^5 - 1
    fe z10 = fe_mul(fe_sqn(z5, 5), z5);          // 2^10 - 1
    fe z20 = fe_mul(fe_sqn(z10, 10), z10);       // 2^20 - 1
    fe z40 = fe_mul(fe_sqn(z20, 20), z20);       // 2^40 - 1
    fe z50 = fe_mul(fe_sqn(z40, 10), z10);       // 2^50 - 1
    fe z100 = fe_mul(fe_sqn(z50, 50), z50);      // 2^100 - 1
    fe z200 = fe_mul(fe_sqn(z100, 100), z100);   // 2^200 - 1
    fe z250 = fe_mul(fe_sqn(z200, 50), z50);     // 2^250 - 1
    return fe_mul(fe_sqn(z250, 5), z11);         // 2^255 - 21
}

PHD gcached pt_to_cached(const gpt& p) {
    const fe d2 = FE_CONST(FE_D2_LIMBS);
    fe zi = fe_invert(p.Z);
    fe x = fe_mul(p.X, zi), y = fe_mul(p.Y, zi);
    gcached c;
    c.YpX = fe_add(y, x);
    c.YmX = fe_sub(y, x);
    c.T2d = fe_mul(fe_mul(x, y), d2);
    return c;
}

PHD gcached cached_neg(const gcached& c) {
    gcached r;
    r.YpX = c.YmX;
    r.YmX = c.YpX;
    r.T2d = fe_neg(c.T2d);
    return r;
}

// mixed addition p + q (q affine Niels): add-2008-hwcd-3 with Z2 = 1
PHD gpt pt_add_cached(const gpt& p, const gcached& q) {
    fe A = fe_mul(fe_sub(p.Y, p.X), q.YmX);
    fe B = fe_mul(fe_add(p.Y, p.X), q.YpX);
    fe C = fe_mul(p.T, q.T2d);
    fe D = fe_add(p.Z, p.Z);
    fe E = fe_sub(B, A), F = fe_sub(D, C), G = fe_add(D, C), H = fe_add(B, A);
    gpt r;
    r.X = fe_mul(E, F);
    r.Y = fe_mul(G, H);
    r.T = fe_mul(E, H);
    r.Z = fe_mul(F, G);
    return r;
}

// Signed radix-16 recoding of a canonical scalar (< 2^253): d[k] in [-8, 8),
// sum d[k] 16^k = s.
PHD void sc_signed_radix16(const uint32_t s[8], int8_t d[64]) {
    int carry = 0;
    for (int k = 0; k < 64; k++) {
        int v = (int)((s[k >> 3] >> (4 * (k & 7))) & 15u) + carry;
        carry = (v + 8) >> 4;
        d[k] = (int8_t)(v - (carry << 4));
    }
}

PHD gcached table_pick(const gcached* tab, int k, int digit) {
    int a = digit < 0 ? -digit : digit;
    gcached c = tab[8 * k + a - 1];
    return digit < 0 ? cached_neg(c) : c;
}

// acc + s * P via the comb table of P (64 additions, skipping zero digits).
PHD gpt comb_mul_add(gpt acc, const gcached* tab, const int8_t d[64]) {
    for (int k = 0; k < 64; k++)
        if (d[k]) acc = pt_add_cached(acc, table_pick(tab, k, d[k]));
    return acc;
}

// Signed radix-256 recoding (throughput-mode combs): d[k] in [-128, 128),
// sum d[k] 256^k = s; s < 2^253 so the top digit never carries out.
PHD void sc_signed_radix256(const uint32_t s[8], int16_t d[32]) {
    int carry = 0;
    for (int k = 0; k < 32; k++) {
        int v = (int)((s[k >> 2] >> (8 * (k & 3))) & 255u) + carry;
        carry = (v + 128) >> 8;
        d[k] = (int16_t)(v - (carry << 8));
    }
}

// acc + s * P via the radix-256 comb table of P (tab[128 k + |d| - 1] =
// |d| 256^k P): 32 mixed additions instead of the radix-16 table's 64.
PHD gpt comb256_mul_add(gpt acc, const gcached* tab, const uint32_t s[8]) {
    int16_t d[32];
    sc_signed_radix256(s, d);
    for (int k = 0; k < 32; k++) {
        const int dig = d[k];
        if (!dig) continue;
        const int a = dig < 0 ? -dig : dig;
        const gcached c = tab[128 * k + a - 1];
        acc = pt_add_cached(acc, dig < 0 ? cached_neg(c) : c);
    }
    return acc;
}

// Ristretto equality of classes (RFC 9496 §4.3.3): X1*Y2 == Y1*X2 or
// Y1*Y2 == X1*X2. Equal classes <=> equal canonical encodings, so comparing
// against a decoded R replaces encoding P (the reference's byte compare).
PHD bool rist_equal(const gpt& p, const gpt& q) {
    return fe_eq(fe_mul(p.X, q.Y), fe_mul(p.Y, q.X)) || fe_eq(fe_mul(p.Y, q.Y), fe_mul(p.X, q.X));
}
