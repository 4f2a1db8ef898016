// ristretto255 over edwards25519 for the device group check (stage 3).
//
// Replaces the libsodium calls behind the reference's group layer
// (proj/src/group.cpp): crypto_core_ristretto255_is_valid_point (:107-114),
// crypto_scalarmult_ristretto255 / _base and _add inside commit_check
// (:144-167) and group_combine (:169-178), plus the byte-equality of
// GroupElement::operator== (include/poslo/group.hpp:59).
//
// Field GF(2^255-19): radix 2^25.5, see the field section below. Points are
// extended twisted-Edwards (X:Y:Z:T), a = -1. Ristretto decode/encode and
// SQRT_RATIO_M1 follow the published ristretto255 definition (RFC 9496 §4);
// constants were derived from their definitions (oracle/ristretto.py) and the
// whole layer is pinned against the reference's own outputs
// (tests/golden/kat.json) on CPU (tests/native) and GPU (tests/test_gpu_*).
//
// Verification handles public data only, so everything is variable-time.
#pragma once
#include "poslo_common.cuh"

// Field GF(2^255-19) in radix 2^25.5 (10 limbs alternating 26 / 25 bits,
// bit offsets 0, 26, 51, ..., 230): a product of two field elements is 100
// 32x32->64 multiply-adds (IMAD.WIDE with a 64-bit addend, full rate on the
// FMA pipe) into 10 column sums that cannot overflow 64 bits, and ONE carry
// chain — where 32-bit limbs need a carry per product on the ALU pipe.
// Elements are kept "carried" (limb i < 2^w_i, slack of a few bits on limb 1)
// after every operation; canonical form only for encode / compare.
#define FE_D_LIMBS 0x35978a3u, 0x0d37284u, 0x3156ebdu, 0x06a0a0eu, 0x001c029u, 0x179e898u, 0x3a03cbbu, 0x1ce7198u, 0x2e2b6ffu, 0x1480db3u
#define FE_D2_LIMBS 0x2b2f159u, 0x1a6e509u, 0x22add7au, 0x0d4141du, 0x0038052u, 0x0f3d130u, 0x3407977u, 0x19ce331u, 0x1c56dffu, 0x0901b67u
#define FE_SQRTM1_LIMBS 0x20ea0b0u, 0x186c9d2u, 0x08f189du, 0x035697fu, 0x0bd0c60u, 0x1fbd7a7u, 0x2804c9eu, 0x1e16569u, 0x004fc1du, 0x0ae0c92u
#define FE_INVSQRT_A_MINUS_D_LIMBS 0x05d40eau, 0x03f6aa0u, 0x257d339u, 0x0bad20bu, 0x274bc58u, 0x001d840u, 0x13dc8ffu, 0x19442d8u, 0x05cfaffu, 0x1e1b224u
#define FE_BASE_X_LIMBS 0x325d51au, 0x18b5823u, 0x0f6592au, 0x104a92du, 0x1a4b31du, 0x1d6dc5cu, 0x27118feu, 0x07fd814u, 0x13cd6e5u, 0x085a4dbu
#define FE_BASE_Y_LIMBS 0x2666658u, 0x1999999u, 0x0ccccccu, 0x1333333u, 0x1999999u, 0x0666666u, 0x3333333u, 0x0ccccccu, 0x2666666u, 0x1999999u
#define FE_BASE_T_LIMBS 0x1b7dda3u, 0x1a2ace9u, 0x25eadbbu, 0x003ba8au, 0x083c27eu, 0x0abe37du, 0x1274732u, 0x0ccacddu, 0x0fd78b7u, 0x19e1d7cu

struct fe {
    uint32_t v[10];
};

struct gpt {  // extended coordinates, x = X/Z, y = Y/Z, xy = T/Z
    fe X, Y, Z, T;
};

#define FE_M26 0x3ffffffu
#define FE_M25 0x1ffffffu

PHD constexpr int fe_width(int i) { return (i & 1) ? 25 : 26; }
PHD constexpr int fe_offset(int i) { return 26 * ((i + 1) / 2) + 25 * (i / 2); }

PHD fe fe_from(uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3, uint32_t a4, uint32_t a5, uint32_t a6,
               uint32_t a7, uint32_t a8, uint32_t a9) {
    fe r;
    r.v[0] = a0; r.v[1] = a1; r.v[2] = a2; r.v[3] = a3; r.v[4] = a4;
    r.v[5] = a5; r.v[6] = a6; r.v[7] = a7; r.v[8] = a8; r.v[9] = a9;
    return r;
}
#define FE_CONST(LIMBS) fe_from(LIMBS)

PHD fe fe_zero() { return fe_from(0, 0, 0, 0, 0, 0, 0, 0, 0, 0); }
PHD fe fe_one() { return fe_from(1, 0, 0, 0, 0, 0, 0, 0, 0, 0); }

// One carry pass over 64-bit column values into carried 32-bit limbs:
// 2^255 == 19 folds the top carry into limb 0.
PHD fe fe_carry64(uint64_t h[10]) {
#pragma unroll
    for (int i = 0; i < 9; i++) {
        h[i + 1] += h[i] >> fe_width(i);
        h[i] &= (i & 1) ? FE_M25 : FE_M26;
    }
    h[0] += 19 * (h[9] >> 25);
    h[9] &= FE_M25;
    h[1] += h[0] >> 26;
    h[0] &= FE_M26;
    fe r;
#pragma unroll
    for (int i = 0; i < 10; i++) r.v[i] = (uint32_t)h[i];
    return r;
}

PHD fe fe_carry32(const uint32_t t[10]) {
    uint64_t h[10];
#pragma unroll
    for (int i = 0; i < 10; i++) h[i] = t[i];
    return fe_carry64(h);
}

PHD fe fe_add(const fe& a, const fe& b) {
    uint32_t t[10];
#pragma unroll
    for (int i = 0; i < 10; i++) t[i] = a.v[i] + b.v[i];
    return fe_carry32(t);
}

// a + 2p - b: 2p's limbs dominate every carried b, so no limb underflows.
PHD fe fe_sub(const fe& a, const fe& b) {
    uint32_t t[10];
#pragma unroll
    for (int i = 0; i < 10; i++) {
        const uint32_t bias = i == 0 ? 0x7ffffdau : ((i & 1) ? 0x3fffffeu : 0x7fffffeu);
        t[i] = a.v[i] + bias - b.v[i];
    }
    return fe_carry32(t);
}

// Column sums h_k = sum over i + j == k (mod 10) of f_i g_j, with x19 for the
// wrapped terms (2^255 == 19) and x2 when both limb offsets round down
// (i and j odd): every term < 2^58, every column < 2^62.
PHD fe fe_mul_impl(const fe& f, const fe& g) {
    uint32_t g19[10], f2[10];
#pragma unroll
    for (int i = 0; i < 10; i++) {
        g19[i] = 19u * g.v[i];
        f2[i] = (i & 1) ? 2u * f.v[i] : f.v[i];
    }
    uint64_t h[10];
#pragma unroll
    for (int k = 0; k < 10; k++) h[k] = 0;
#pragma unroll
    for (int i = 0; i < 10; i++)
#pragma unroll
        for (int j = 0; j < 10; j++) {
            const uint32_t fi = (j & 1) ? f2[i] : f.v[i];
            const uint32_t gj = (i + j >= 10) ? g19[j] : g.v[j];
            h[(i + j) % 10] += (uint64_t)fi * gj;
        }
    return fe_carry64(h);
}

// Squaring: the symmetric products once, doubled (55 multiply-adds).
PHD fe fe_sq_impl(const fe& f) {
    uint32_t f19[10];
#pragma unroll
    for (int i = 0; i < 10; i++) f19[i] = 19u * f.v[i];
    uint64_t h[10];
#pragma unroll
    for (int k = 0; k < 10; k++) h[k] = 0;
#pragma unroll
    for (int i = 0; i < 10; i++)
#pragma unroll
        for (int j = i; j < 10; j++) {
            const uint32_t c = (i != j ? 2u : 1u) * ((i & 1) && (j & 1) ? 2u : 1u);
            const uint32_t fi = c * f.v[i];
            const uint32_t fj = (i + j >= 10) ? f19[j] : f.v[j];
            h[(i + j) % 10] += (uint64_t)fi * fj;
        }
    return fe_carry64(h);
}

#if defined(__CUDA_ARCH__) && defined(POSLO_FE_CALL)
// Out of line in the group kernels: a point addition then stays a few hundred
// instructions and the kernels fit the instruction cache (inlined,
// k_check_split stalled on no_instruction).
__device__ __noinline__ fe fe_mul_call(fe a, fe b) { return fe_mul_impl(a, b); }
__device__ __noinline__ fe fe_sq_call(fe a) { return fe_sq_impl(a); }
PHD fe fe_mul(const fe& a, const fe& b) { return fe_mul_call(a, b); }
PHD fe fe_sq(const fe& a) { return fe_sq_call(a); }
#else
PHD fe fe_mul(const fe& a, const fe& b) { return fe_mul_impl(a, b); }
PHD fe fe_sq(const fe& a) { return fe_sq_impl(a); }
#endif

PHD fe fe_sqn(fe a, int n) {
    for (int i = 0; i < n; i++) a = fe_sq(a);
    return a;
}

// Canonical representative in [0, p): exact limb widths (two carry passes),
// then v >= p  <=>  v + 19 >= 2^255.
PHD fe fe_canon(const fe& a) {
    uint32_t h[10];
#pragma unroll
    for (int i = 0; i < 10; i++) h[i] = a.v[i];
    for (int pass = 0; pass < 2; pass++) {
#pragma unroll
        for (int i = 0; i < 9; i++) {
            h[i + 1] += h[i] >> fe_width(i);
            h[i] &= (i & 1) ? FE_M25 : FE_M26;
        }
        h[0] += 19 * (h[9] >> 25);
        h[9] &= FE_M25;
    }
#pragma unroll
    for (int i = 0; i < 9; i++) {  // h0 may still hold a carry from the fold
        h[i + 1] += h[i] >> fe_width(i);
        h[i] &= (i & 1) ? FE_M25 : FE_M26;
    }
    uint32_t t[10];
    uint32_t c = 19;
#pragma unroll
    for (int i = 0; i < 10; i++) {
        t[i] = h[i] + c;
        c = t[i] >> fe_width(i);
        t[i] &= (i & 1) ? FE_M25 : FE_M26;
    }
    fe r;
#pragma unroll
    for (int i = 0; i < 10; i++) r.v[i] = c ? t[i] : h[i];
    return r;
}

PHD bool fe_is_neg(const fe& a) { return fe_canon(a).v[0] & 1; }

PHD bool fe_is_zero(const fe& a) {
    fe c = fe_canon(a);
    uint32_t x = 0;
#pragma unroll
    for (int i = 0; i < 10; i++) x |= c.v[i];
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

#ifdef __CUDACC__
// ---- warp-cooperative exponentiation (latency paths) ----------------------
// One product on one thread is a serial 10-limb carry chain (~900 cycles);
// the inverse square root behind every encode / decode is 252 squarings and
// 11 products of them. Where ONE encode or decode sits on a critical path
// (a single check, a distill step, a fold's result) the whole warp runs it:
// the element is spread over lanes 0..9 (lane k holds limb k), lane k forms
// column k of a product from 10 broadcast limbs of a and 10 rotated limbs of
// b (20 shuffles, 10 IMAD.WIDE), and the carries run as parallel passes
// (shuffle up; lane 0 takes 19 x lane 9's carry). Lanes 10..31 mirror lane 0.
// Results leaving the warp form are carried (limb < 2^w + 38), as fe_carry64's.

// One parallel carry pass over 32-bit limbs (limb k keeps its low w bits and
// takes lane k-1's carry; lane 0 takes 19 x lane 9's).
__device__ __forceinline__ uint32_t fw_carry32(uint32_t h, int k, int base = 0) {
    const int w = (k & 1) ? 25 : 26;
    const uint32_t c = h >> w;
    const uint32_t cin = __shfl_sync(0xffffffffu, c, base + (k == 0 ? 9 : k - 1));
    return (h & ((1u << w) - 1)) + (k == 0 ? 19u * cin : cin);
}

// Column sums (< 2^61) -> limbs < 2^w + 2^20 in two parallel passes: enough
// for the next product's bounds (and for fe_sub's bias); a result leaving the
// warp form takes a third (fw_carry32).
__device__ __forceinline__ uint32_t fw_carry(uint64_t h, int k, int base = 0) {
    const int w = (k & 1) ? 25 : 26;
    const int src = base + (k == 0 ? 9 : k - 1);
    const uint64_t c = h >> w;  // < 2^36
    const uint64_t cin = __shfl_sync(0xffffffffu, c, src);
    h = (h & ((1ull << w) - 1)) + (k == 0 ? 19 * cin : cin);  // < 2^41
    const uint32_t c2 = (uint32_t)(h >> w);                      // < 2^16
    const uint32_t cin2 = __shfl_sync(0xffffffffu, c2, src);
    return (uint32_t)(h & ((1ull << w) - 1)) + (k == 0 ? 19u * cin2 : cin2);
}

// base: the group's first lane (0, or 10 / 20 when a warp holds three
// elements, fw3_*), k: this lane's limb index within its group.
__device__ __forceinline__ uint32_t fw_mul(uint32_t a, uint32_t b, int k, int base = 0) {
    uint64_t h0 = 0, h1 = 0;  // two accumulation chains (even / odd i): half the dependent IMAD.WIDEs
#pragma unroll
    for (int i = 0; i < 10; i++) {
        const uint32_t ai = __shfl_sync(0xffffffffu, a, base + i);
        const int j = k >= i ? k - i : k - i + 10;  // column k = i + j (mod 10)
        const uint32_t bj = __shfl_sync(0xffffffffu, b, base + j);
        // x19 for the wrapped terms (2^255 == 19), x2 when both limb offsets round down
        const uint32_t f = (k >= i ? 1u : 19u) << (i & j & 1);
        if (i & 1) h1 += (uint64_t)ai * (bj * f);
        else h0 += (uint64_t)ai * (bj * f);
    }
    return fw_carry(h0 + h1, k, base);
}

__device__ __noinline__ uint32_t fw_sqn(uint32_t a, int n, int k) {
#pragma unroll 1
    for (int i = 0; i < n; i++) a = fw_mul(a, a, k);
    return a;
}

// fe_pow22523 by the whole (converged) warp; z and the result are the same
// value in every lane.
__device__ __noinline__ fe fe_pow22523_w(const fe& zf) {
    const int lane = threadIdx.x & 31, k = lane < 10 ? lane : 0;
    uint32_t z = zf.v[0];
#pragma unroll
    for (int i = 1; i < 10; i++)
        if (k == i) z = zf.v[i];
    const uint32_t z2 = fw_mul(z, z, k);
    const uint32_t z3 = fw_mul(z2, z, k);                         // 2^2 - 1
    const uint32_t z15 = fw_mul(fw_sqn(z3, 2, k), z3, k);         // 2^4 - 1
    const uint32_t z31 = fw_mul(fw_sqn(z15, 1, k), z, k);         // 2^5 - 1
    const uint32_t z10 = fw_mul(fw_sqn(z31, 5, k), z31, k);       // 2^10 - 1
    const uint32_t z20 = fw_mul(fw_sqn(z10, 10, k), z10, k);      // 2^20 - 1
    const uint32_t z40 = fw_mul(fw_sqn(z20, 20, k), z20, k);      // 2^40 - 1
    const uint32_t z50 = fw_mul(fw_sqn(z40, 10, k), z10, k);      // 2^50 - 1
    const uint32_t z100 = fw_mul(fw_sqn(z50, 50, k), z50, k);     // 2^100 - 1
    const uint32_t z200 = fw_mul(fw_sqn(z100, 100, k), z100, k);  // 2^200 - 1
    const uint32_t z250 = fw_mul(fw_sqn(z200, 50, k), z50, k);    // 2^250 - 1
    const uint32_t r = fw_carry32(fw_mul(fw_sqn(z250, 2, k), z, k), k);  // 2^252 - 3, limbs < 2^w + 38
    fe out;
#pragma unroll
    for (int i = 0; i < 10; i++) out.v[i] = __shfl_sync(0xffffffffu, r, i);
    return out;
}

// ---- warp-cooperative doubling chain (comb-table builds) -------------------
// Three elements per warp: group g = lane / 10 (lanes 30, 31 mirror group
// 2's limb 0) holds limb k = lane % 10 of its element, so one round of
// fw_mul multiplies three independent pairs. A doubling (dbl-2008-hwcd with
// 2XY for (X + Y)^2 - X^2 - Y^2) is three rounds: {X^2, Y^2, XY}, {Z^2},
// {EF, GH, FG} (+ {EH} for T when the point is stored), the coordinates
// replicated in every group between rounds by one shuffle each.
struct Fw3Lane {
    int g, k, base;
};
__device__ __forceinline__ Fw3Lane fw3_lane() {
    const int lane = threadIdx.x & 31;
    Fw3Lane L;
    L.g = lane < 30 ? lane / 10 : 2;
    L.k = lane < 30 ? lane % 10 : 0;
    L.base = 10 * L.g;
    return L;
}
// limb k of a replicated fe
__device__ __forceinline__ uint32_t fw_pick(const fe& a, int k) {
    uint32_t x = a.v[0];
#pragma unroll
    for (int i = 1; i < 10; i++)
        if (k == i) x = a.v[i];
    return x;
}
// 2p - b + a per limb (b carried: limb < 2^w + 2^20), then one carry pass
__device__ __forceinline__ uint32_t fw_sub(uint32_t a, uint32_t b, const Fw3Lane& L) {
    const uint32_t bias = L.k == 0 ? 0x7ffffdau : ((L.k & 1) ? 0x3fffffeu : 0x7fffffeu);
    return fw_carry32(a + bias - b, L.k, L.base);
}
__device__ __forceinline__ uint32_t fw_add(uint32_t a, uint32_t b, const Fw3Lane& L) {
    return fw_carry32(a + b, L.k, L.base);
}
// the value group `from` holds, in every group (limb for limb)
__device__ __forceinline__ uint32_t fw_bcast(uint32_t x, int from, const Fw3Lane& L) {
    return __shfl_sync(0xffffffffu, x, 10 * from + L.k);
}

// Store pk[k] = 16^k P for k < n (n = 256 / 4 = 64 here): the power chain of
// the comb tables, P given replicated in every lane; T is formed only for
// the stored points. Every lane of the warp calls.
__device__ __noinline__ void fw3_pow16_chain(const gpt& P, gpt* out, int n) {
    const Fw3Lane L = fw3_lane();
    uint32_t X = fw_pick(P.X, L.k), Y = fw_pick(P.Y, L.k), Z = fw_pick(P.Z, L.k), T = fw_pick(P.T, L.k);
#pragma unroll 1
    for (int q = 0; q < n; q++) {
        {  // group 0 stores the point, a limb per lane (T: from the last doubling)
            const uint32_t xs = fw_carry32(X, L.k, L.base), ys = fw_carry32(Y, L.k, L.base);
            const uint32_t zs = fw_carry32(Z, L.k, L.base), ts = fw_carry32(T, L.k, L.base);
            if ((threadIdx.x & 31) < 10) {
                out[q].X.v[L.k] = xs;
                out[q].Y.v[L.k] = ys;
                out[q].Z.v[L.k] = zs;
                out[q].T.v[L.k] = ts;
            }
        }
        if (q + 1 == n) break;
#pragma unroll 1
        for (int d = 0; d < 4; d++) {
            // round 1: A = X^2 (group 0), B = Y^2 (1), XY (2)
            const uint32_t u = L.g == 1 ? Y : X, v = L.g == 0 ? X : Y;
            const uint32_t r1 = fw_mul(u, v, L.k, L.base);
            const uint32_t A = fw_bcast(r1, 0, L), B = fw_bcast(r1, 1, L), XY = fw_bcast(r1, 2, L);
            // round 2: Z^2 (every group)
            const uint32_t Z2 = fw_mul(Z, Z, L.k, L.base);
            const uint32_t E = fw_add(XY, XY, L);
            const uint32_t G = fw_sub(B, A, L);
            const uint32_t F = fw_sub(G, fw_add(Z2, Z2, L), L);
            const uint32_t H = fw_sub(0u, fw_add(A, B, L), L);
            // round 3: X3 = EF (0), Y3 = GH (1), Z3 = FG (2); T3 = EH on the last doubling
            const uint32_t p = L.g == 1 ? G : (L.g == 0 ? E : F), r = L.g == 1 ? H : (L.g == 0 ? F : G);
            const uint32_t r3 = fw_mul(p, r, L.k, L.base);
            X = fw_bcast(r3, 0, L);
            Y = fw_bcast(r3, 1, L);
            Z = fw_bcast(r3, 2, L);
            if (d == 3) T = fw_mul(E, H, L.k, L.base);
        }
    }
}
#endif

// W = true: the exponentiation by the whole warp (every lane of a converged
// warp calls with the same operands; device code only).
template <bool W>
PHD fe fe_pow22523_sel(const fe& z) {
#ifdef __CUDA_ARCH__
    if constexpr (W) return fe_pow22523_w(z);
#endif
    return fe_pow22523(z);
}

// SQRT_RATIO_M1(u, v): returns was_square, r = non-negative root.
template <bool W = false>
PHD bool fe_sqrt_ratio_m1(const fe& u, const fe& v, fe& r) {
    const fe sqrtm1 = FE_CONST(FE_SQRTM1_LIMBS);
    fe v3 = fe_mul(fe_sq(v), v);
    fe v7 = fe_mul(fe_sq(v3), v);
    r = fe_mul(fe_mul(u, v3), fe_pow22523_sel<W>(fe_mul(u, v7)));
    fe check = fe_mul(v, fe_sq(r));
    fe nu = fe_neg(u);
    bool correct = fe_eq(check, u);
    bool flipped = fe_eq(check, nu);
    bool flipped_i = fe_eq(check, fe_mul(nu, sqrtm1));
    if (flipped || flipped_i) r = fe_mul(r, sqrtm1);
    r = fe_abs(r);
    return correct || flipped;
}

// 32 little-endian bytes -> limbs; bit 255 is ignored (decode compares the
// re-encoded bytes to reject it).
PHD fe fe_from_bytes_le(const uint8_t b[32]) {
    uint64_t w[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        uint64_t x = 0;
#pragma unroll
        for (int i = 7; i >= 0; i--) x = (x << 8) | b[8 * k + i];
        w[k] = x;
    }
    fe r;
#pragma unroll
    for (int i = 0; i < 10; i++) {
        const int off = fe_offset(i), q = off >> 6, sh = off & 63;
        uint64_t x = w[q] >> sh;
        if (sh && q < 3) x |= w[q + 1] << (64 - sh);
        r.v[i] = (uint32_t)x & ((i & 1) ? FE_M25 : FE_M26);
    }
    return r;
}

PHD void fe_to_bytes_le(const fe& a, uint8_t b[32]) {
    const fe c = fe_canon(a);
    uint64_t w[4] = {0, 0, 0, 0};
#pragma unroll
    for (int i = 0; i < 10; i++) {
        const int off = fe_offset(i), q = off >> 6, sh = off & 63;
        w[q] |= (uint64_t)c.v[i] << sh;
        if (sh + fe_width(i) > 64 && q < 3) w[q + 1] |= (uint64_t)c.v[i] >> (64 - sh);
    }
#pragma unroll
    for (int k = 0; k < 4; k++)
#pragma unroll
        for (int i = 0; i < 8; i++) b[8 * k + i] = (uint8_t)(w[k] >> (8 * i));
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
// W = true: the inverse square root by the whole warp (every lane calls with
// the same bytes; rist_decode_w).
template <bool W>
PHD bool rist_decode_t(const uint8_t b[32], gpt& out) {
    fe s = fe_from_bytes_le(b);
    // canonical: s < p and bit 255 clear (re-encoding reproduces b), non-negative
    uint8_t rb[32];
    fe_to_bytes_le(s, rb);
    uint32_t diff = 0;
#pragma unroll
    for (int i = 0; i < 32; i++) diff |= rb[i] ^ b[i];
    if (diff || (b[0] & 1)) return false;
    const fe d = FE_CONST(FE_D_LIMBS);
    fe ss = fe_sq(s);
    fe u1 = fe_sub(fe_one(), ss);
    fe u2 = fe_add(fe_one(), ss);
    fe u2sq = fe_sq(u2);
    fe v = fe_sub(fe_neg(fe_mul(d, fe_sq(u1))), u2sq);
    fe inv;
    bool was_square = fe_sqrt_ratio_m1<W>(fe_one(), fe_mul(v, u2sq), inv);
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

PHD bool rist_decode(const uint8_t b[32], gpt& out) { return rist_decode_t<false>(b, out); }

// Ristretto encode (RFC 9496 §4.3.2) -> 32 canonical bytes.
template <bool W>
PHD void rist_encode_t(const gpt& p, uint8_t out[32]) {
    const fe sqrtm1 = FE_CONST(FE_SQRTM1_LIMBS);
    const fe isqrt_amd = FE_CONST(FE_INVSQRT_A_MINUS_D_LIMBS);
    fe u1 = fe_mul(fe_add(p.Z, p.Y), fe_sub(p.Z, p.Y));
    fe u2 = fe_mul(p.X, p.Y);
    fe inv;
    fe_sqrt_ratio_m1<W>(fe_one(), fe_mul(u1, fe_sq(u2)), inv);
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

PHD void rist_encode(const gpt& p, uint8_t out[32]) { rist_encode_t<false>(p, out); }
#ifdef __CUDACC__
// by the whole converged warp, same operands in every lane
__device__ __forceinline__ bool rist_decode_w(const uint8_t b[32], gpt& out) { return rist_decode_t<true>(b, out); }
__device__ __forceinline__ void rist_encode_w(const gpt& p, uint8_t out[32]) { rist_encode_t<true>(p, out); }
#endif

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
// so both exponentiations of commit_check are fixed-base.
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

// acc + s * P on a radix-2^16 comb of P (16 windows x 32768 affine Niels
// points): signed 16-bit digits, 16 mixed additions. s < 2^253, so the top
// digit never carries out.
PHD gpt comb65536_mul_add(gpt acc, const gcached* tab, const uint32_t s[8]) {
    int carry = 0;
    for (int k = 0; k < 16; k++) {
        const int a = (int)((s[k >> 1] >> (16 * (k & 1))) & 0xffffu) + carry;
        carry = (a + 32768) >> 16;
        const int dig = a - (carry << 16);
        if (!dig) continue;
        const int m = dig < 0 ? -dig : dig;
        const gcached c = tab[32768 * k + m - 1];
        acc = pt_add_cached(acc, dig < 0 ? cached_neg(c) : c);
    }
    return acc;
}

// encode(P) == r without a square root. In RFC 9496 §4.3.2 every branch of
// the encoding depends on z_inv = den1 den2 T = T / u2 (u1 = Z^2 - Y^2,
// u2 = XY, invsqrt^2 = 1 / (u1 u2^2): the sign of invsqrt cancels), and the
// output is s = |invsqrt K| with K = (rotate ? u1 INVSQRT_A_MINUS_D : u2)(Z - y).
// For a valid point W = u1 u2^2 is a square, so with r's s canonical and
// non-negative: encode(P) == r  <=>  s^2 W == K^2 (the square map is
// injective on non-negative elements). u2 == 0 is the identity class, which
// encodes to 0. inv_u2 = 1 / u2 comes from a batched inversion
// (k_batch_invert); checked against the encoding on random points, torsion
// representatives and rescaled coordinates (tests/test_gpu_parity.py).
PHD bool rist_encoding_matches(const gpt& p, const fe& inv_u2, const uint8_t r[32]) {
    const fe s = fe_from_bytes_le(r);
    uint8_t rb[32];
    fe_to_bytes_le(s, rb);
    uint32_t diff = 0;
#pragma unroll
    for (int i = 0; i < 32; i++) diff |= rb[i] ^ r[i];
    if (diff || (r[0] & 1)) return false;  // encodings are canonical and non-negative
    const fe u2 = fe_mul(p.X, p.Y);
    if (fe_is_zero(u2)) return fe_is_zero(s);
    const fe u1 = fe_mul(fe_add(p.Z, p.Y), fe_sub(p.Z, p.Y));
    const fe z_inv = fe_mul(p.T, inv_u2);
    const bool rotate = fe_is_neg(fe_mul(p.T, z_inv));
    const fe sqrtm1 = FE_CONST(FE_SQRTM1_LIMBS);
    const fe x = rotate ? fe_mul(p.Y, sqrtm1) : p.X;
    fe y = rotate ? fe_mul(p.X, sqrtm1) : p.Y;
    if (fe_is_neg(fe_mul(x, z_inv))) y = fe_neg(y);
    const fe k = rotate ? fe_mul(u1, FE_CONST(FE_INVSQRT_A_MINUS_D_LIMBS)) : u2;
    const fe K = fe_mul(k, fe_sub(p.Z, y));
    const fe W = fe_mul(u1, fe_sq(u2));
    return fe_eq(fe_mul(fe_sq(s), W), fe_sq(K));
}

// Ristretto equality of classes (RFC 9496 §4.3.3): X1*Y2 == Y1*X2 or
// Y1*Y2 == X1*X2. Equal classes <=> equal canonical encodings, so comparing
// against a decoded R replaces encoding P (the reference's byte compare).
PHD bool rist_equal(const gpt& p, const gpt& q) {
    return fe_eq(fe_mul(p.X, q.Y), fe_mul(p.Y, q.X)) || fe_eq(fe_mul(p.Y, q.Y), fe_mul(p.X, q.X));
}
