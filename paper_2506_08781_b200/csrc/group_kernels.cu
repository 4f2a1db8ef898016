// Stage 3 of the batch verifier on sm_100a: batched ristretto255 group
// checks (commit_check(Y, e, s) == R, group.cpp:144-167 + group.hpp:59),
// the R-hat fold of paver (batch_verify.cpp:75-81, group_combine
// group.cpp:169-178) and point validation (GroupElement::from_bytes,
// group.cpp:107-114). One thread per check; folds are block trees.
#ifndef POSLO_FE_INLINE
#define POSLO_FE_CALL 1  // out-of-line field multiplication in the group kernels (i-cache)
#endif
#include "poslo_internal.h"
#include "ristretto.cuh"
#include "scalar.cuh"

namespace poslo_gpu {

static_assert(sizeof(fe) == kFeBytes && sizeof(gpt) == kGptBytes && sizeof(gcached) == kCachedBytes,
              "buffer sizes in poslo_internal.h follow the field representation");

namespace {

__device__ __forceinline__ void load32(const uint8_t* p, uint8_t b[32]) {
#pragma unroll
    for (int k = 0; k < 32; k++) b[k] = p[k];
}

__global__ void __launch_bounds__(128) k_group_check(const uint8_t* __restrict__ y, uint32_t n,
                                                     const uint32_t* __restrict__ e,
                                                     const uint32_t* __restrict__ s,
                                                     const uint8_t* __restrict__ r,
                                                     uint8_t* __restrict__ enc,
                                                     uint8_t* __restrict__ verdict, int* ybad) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t yb[32];
    load32(y, yb);
    gpt Y;
    if (!rist_decode(yb, Y)) {
        if (ybad) atomicOr(ybad, 1);
        if (verdict) verdict[i] = 0;
        return;
    }
    uint32_t ee[8], ss[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        ee[k] = e[(size_t)i * 8 + k];
        ss[k] = s[(size_t)i * 8 + k];
    }
    uint8_t out[32];
    commit_check_enc(Y, ee, ss, out);
    if (enc)
#pragma unroll
        for (int k = 0; k < 32; k++) enc[(size_t)i * 32 + k] = out[k];
    if (r && verdict) {
        uint32_t diff = 0;
#pragma unroll
        for (int k = 0; k < 32; k++) diff |= out[k] ^ r[(size_t)i * 32 + k];
        verdict[i] = diff == 0;
    }
}

__device__ __forceinline__ void block_reduce_pt(gpt& acc, gpt* sh) {
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w >= 1; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] = pt_add(sh[threadIdx.x], sh[threadIdx.x + w]);
        __syncthreads();
    }
    acc = sh[0];
}

__global__ void __launch_bounds__(128) k_fold_stage1(const uint8_t* __restrict__ pts, uint64_t n,
                                                     gpt* __restrict__ partial, int* bad) {
    __shared__ gpt sh[128];
    gpt acc = pt_identity();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint8_t b[32];
        load32(pts + i * 32, b);
        gpt P;
        if (!rist_decode(b, P)) {
            atomicAdd(bad, 1);
            continue;
        }
        acc = pt_add(acc, P);
    }
    block_reduce_pt(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(128) k_fold_stage2(const gpt* __restrict__ partial, uint32_t n,
                                                     uint8_t* __restrict__ out) {
    __shared__ gpt sh[128];
    gpt acc = pt_identity();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) acc = pt_add(acc, partial[i]);
    block_reduce_pt(acc, sh);
    if (threadIdx.x < 32) {  // the encode by the whole warp 0
        uint8_t b[32];
        rist_encode_w(acc, b);
        if (threadIdx.x == 0)
#pragma unroll
            for (int k = 0; k < 32; k++) out[k] = b[k];
    }
}

__global__ void k_validate(const uint8_t* __restrict__ pts, uint32_t n, uint8_t* __restrict__ ok) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t b[32];
    load32(pts + (size_t)i * 32, b);
    gpt P;
    ok[i] = rist_decode(b, P) ? 1 : 0;
}

// ---- comb tables ------------------------------------------------------------
// Builds the fixed-base table of P (decoded from `enc`, or the ristretto255
// generator when enc == nullptr). Stage A (one warp, warp-cooperative field
// products): the 64 powers P_k = 16^k P. Stage B (one thread per entry): the
// multiples of P_k (radix 16 / 256 / 2^16 fills) in cached form.
template <int W>
__global__ void k_table_pow(const uint8_t* __restrict__ enc, gpt* __restrict__ pk, int* bad) {
    // one warp: the decode and the 252-doubling chain warp-cooperatively
    // (rist_decode_w, fw3_pow16_chain: three field products per round)
    static_assert(W == 4, "the warp chain stores 16^k P");
    if (blockIdx.x != 0 || threadIdx.x >= 32) return;
    gpt P;
    if (enc) {
        uint8_t b[32];
        load32(enc, b);
        if (!rist_decode_w(b, P)) {
            if (threadIdx.x == 0) atomicOr(bad, 1);
            P = pt_identity();
        }
    } else {
        P = pt_base();
    }
    fw3_pow16_chain(P, pk, 256 / W);
}

// Radix-256 fill: thread t = 128 k + i writes (i + 1) 256^k P, by
// double-and-add on the bits of i + 1 (<= 8 doublings + 8 additions).
__global__ void k_table_fill256(const gpt* __restrict__ pk, gcached* __restrict__ tab) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 32 * 128) return;
    const int k = t >> 7, m = (t & 127) + 1;
    const gpt base = pk[2 * k];  // pk[i] = 16^i P: 256^k P = pk[2k]
    gpt q = pt_identity();
    for (int b = 7; b >= 0; b--) {
        q = pt_dbl(q);
        if ((m >> b) & 1) q = pt_add(q, base);
    }
    tab[t] = pt_to_cached(q);
}

// Radix-2^16 fill: m 2^(16k) P for m = 1 .. 32768 (signed digits |d| <=
// 2^15), 16 bases 2^(16k) P = pk[4k]. Thread t owns a run of kRun consecutive
// multiples m0 .. m0 + kRun - 1 of one base: m0 B by double-and-add, then one
// mixed addition of B per multiple, the run's Z coordinates inverted together
// (Montgomery's trick: one inversion and 3 multiplications per point instead
// of an inversion per point). The table slots hold (X, Y, Z) until the
// backward pass overwrites them with the affine Niels form.
constexpr uint32_t kRun = 32;
__global__ void __launch_bounds__(128) k_table_fill65536(const gpt* __restrict__ pk, gcached* __restrict__ tab) {
    const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 16u * (32768u / kRun)) return;
    const uint32_t k = t / (32768u / kRun), m0 = (t % (32768u / kRun)) * kRun + 1;
    const gpt base = pk[4 * k];  // pk[i] = 16^i P: 2^(16k) P = pk[4k]
    const gcached bc = pt_to_cached(base);
    gpt q = pt_identity();
#pragma unroll 1
    for (int b = 15; b >= 0; b--) {
        q = pt_dbl(q);
        if ((m0 >> b) & 1) q = pt_add(q, base);
    }
    gcached* out = tab + (size_t)k * 32768u + (m0 - 1);
    fe pre[kRun];  // prefix products of Z (local memory)
#pragma unroll 1
    for (uint32_t r = 0; r < kRun; r++) {
        out[r].YpX = q.X;
        out[r].YmX = q.Y;
        out[r].T2d = q.Z;
        pre[r] = r ? fe_mul(pre[r - 1], q.Z) : q.Z;
        if (r + 1 < kRun) q = pt_add_cached(q, bc);
    }
    const fe d2 = FE_CONST(FE_D2_LIMBS);
    fe inv = fe_invert(pre[kRun - 1]);
#pragma unroll 1
    for (int r = (int)kRun - 1; r >= 0; r--) {
        const fe X = out[r].YpX, Y = out[r].YmX, Z = out[r].T2d;
        const fe zi = r ? fe_mul(inv, pre[r - 1]) : inv;
        if (r) inv = fe_mul(inv, Z);
        const fe x = fe_mul(X, zi), y = fe_mul(Y, zi);
        gcached c;
        c.YpX = fe_add(y, x);
        c.YmX = fe_sub(y, x);
        c.T2d = fe_mul(fe_mul(x, y), d2);
        out[r] = c;
    }
}

__global__ void k_table_fill(const gpt* __restrict__ pk, gcached* __restrict__ tab) {
    int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= 512) return;
    int k = t >> 3, i = t & 7;
    gpt base = pk[k];
    gpt q = base;
    for (int m = 0; m < i; m++) q = pt_add(q, base);
    tab[t] = pt_to_cached(q);
}

// One CTA of 128 threads per check (latency mode, few checks): thread t < 64
// takes window t of e from Y's table, thread 64 + t window t of s from the
// generator's table; a 7-level shared-memory tree adds the 128 points.
__global__ void __launch_bounds__(128) k_check_cta(const gcached* __restrict__ tabY,
                                                   const gcached* __restrict__ tabB,
                                                   const uint32_t* __restrict__ e,
                                                   const uint32_t* __restrict__ s,
                                                   const uint8_t* __restrict__ r,
                                                   uint8_t* __restrict__ enc,
                                                   uint8_t* __restrict__ verdict) {
    __shared__ int8_t dig[128];
    __shared__ gpt sh[128];
    const uint32_t i = blockIdx.x;
    if (threadIdx.x < 2) {
        uint32_t v[8];
        const uint32_t* src = threadIdx.x == 0 ? e : s;
#pragma unroll
        for (int k = 0; k < 8; k++) v[k] = src[(size_t)i * 8 + k];
        int8_t d[64];
        sc_signed_radix16(v, d);
        for (int k = 0; k < 64; k++) dig[64 * threadIdx.x + k] = d[k];
    }
    __syncthreads();
    const int t = threadIdx.x;
    const int dgt = dig[t];
    gpt acc = pt_identity();
    if (dgt) acc = pt_add_cached(acc, table_pick(t < 64 ? tabY : tabB, t & 63, dgt));
    sh[t] = acc;
    __syncthreads();
    for (int w = 64; w >= 1; w >>= 1) {
        if (t < w) sh[t] = pt_add(sh[t], sh[t + w]);
        __syncthreads();
    }
    if (t < 32) {  // the encode by the whole warp 0, lane 0 writes
        uint8_t out[32];
        rist_encode_w(sh[0], out);
        if (t != 0) return;
        if (enc)
#pragma unroll
            for (int k = 0; k < 32; k++) enc[(size_t)i * 32 + k] = out[k];
        if (r && verdict) {
            uint32_t diff = 0;
#pragma unroll
            for (int k = 0; k < 32; k++) diff |= out[k] ^ r[(size_t)i * 32 + k];
            verdict[i] = diff == 0;
        }
    }
}

// One thread per check (throughput mode, e.g. 2^20 per-epoch checks), on
// the radix-256 combs: 64 mixed additions + one encode per check.
// Thread per check on the radix-2^16 combs: 32 mixed additions + the encode
// compare (for batches of >= POSLO_COMB16_MIN checks).
__global__ void __launch_bounds__(128) k_check_thread16(const gcached* __restrict__ tabY,
                                                        const gcached* __restrict__ tabB, uint32_t n,
                                                        const uint32_t* __restrict__ e,
                                                        const uint32_t* __restrict__ s,
                                                        const uint8_t* __restrict__ r,
                                                        uint8_t* __restrict__ enc,
                                                        uint8_t* __restrict__ verdict) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t v[8];
    gpt acc = pt_identity();
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = e[(size_t)i * 8 + k];
    acc = comb65536_mul_add(acc, tabY, v);
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = s[(size_t)i * 8 + k];
    acc = comb65536_mul_add(acc, tabB, v);
    uint8_t out[32];
    rist_encode(acc, out);
    if (enc)
#pragma unroll
        for (int k = 0; k < 32; k++) enc[(size_t)i * 32 + k] = out[k];
    if (r && verdict) {
        uint32_t diff = 0;
#pragma unroll
        for (int k = 0; k < 32; k++) diff |= out[k] ^ r[(size_t)i * 32 + k];
        verdict[i] = diff == 0;
    }
}

// k_check_thread16 against R-hat decoded ahead (k_decode_pts, side stream):
// the ristretto class compare (RFC 9496 4.3.3, 4 multiplications) replaces
// the encoding's inverse square root, about half of a thread-per-check
// check. A failed decode can never equal a canonical encoding: verdict 0.
#ifndef POSLO_CHECK16D_MINB
#define POSLO_CHECK16D_MINB 1
#endif
__global__ void __launch_bounds__(128, POSLO_CHECK16D_MINB) k_check_thread16d(const gcached* __restrict__ tabY,
                                                         const gcached* __restrict__ tabB, uint32_t n,
                                                         const uint32_t* __restrict__ e,
                                                         const uint32_t* __restrict__ s,
                                                         const gpt* __restrict__ R,
                                                         const uint8_t* __restrict__ rok,
                                                         uint8_t* __restrict__ verdict) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t v[8];
    gpt acc = pt_identity();
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = e[(size_t)i * 8 + k];
    acc = comb65536_mul_add(acc, tabY, v);
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = s[(size_t)i * 8 + k];
    acc = comb65536_mul_add(acc, tabB, v);
    verdict[i] = (rok[i] && rist_equal(acc, R[i])) ? 1 : 0;
}

// ---- radix-2^16 checks with no square root per check ----------------------
// (rist_encoding_matches): stage 1 the combs -> P and u2 = XY, stage 2 one
// batched inversion of u2 per chunk of kInvChunk checks (Montgomery's trick:
// 3 products per element + one inversion per chunk), stage 3 the verdict
// encode(P) == R-hat from P, 1 / u2 and R-hat's bytes (~15 products). Against
// decoding R-hat (an inverse square root, ~265 products) + the class compare.
constexpr uint32_t kInvChunk = 32;

__global__ void __launch_bounds__(128) k_check16e_comb(const gcached* __restrict__ tabY,
                                                       const gcached* __restrict__ tabB, uint32_t n,
                                                       const uint32_t* __restrict__ e,
                                                       const uint32_t* __restrict__ s, gpt* __restrict__ P,
                                                       fe* __restrict__ u2) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t v[8];
    gpt acc = pt_identity();
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = e[(size_t)i * 8 + k];
    acc = comb65536_mul_add(acc, tabY, v);
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = s[(size_t)i * 8 + k];
    acc = comb65536_mul_add(acc, tabB, v);
    P[i] = acc;
    const fe t = fe_mul(acc.X, acc.Y);
    u2[i] = fe_is_zero(t) ? fe_one() : t;  // the identity class (u2 = 0) is decided without 1 / u2
}

// a[lo, hi) <- 1 / a[lo, hi) for the chunk of thread t; pre[] holds the prefix products
__global__ void __launch_bounds__(64) k_batch_invert(fe* __restrict__ a, fe* __restrict__ pre, uint32_t n) {
    const uint32_t lo = (blockIdx.x * blockDim.x + threadIdx.x) * kInvChunk;
    if (lo >= n) return;
    const uint32_t hi = min(n, lo + kInvChunk);
    fe acc = a[lo];
    pre[lo] = acc;
#pragma unroll 1
    for (uint32_t i = lo + 1; i < hi; i++) {
        acc = fe_mul(acc, a[i]);
        pre[i] = acc;
    }
    fe inv = fe_invert(acc);
#pragma unroll 1
    for (uint32_t i = hi - 1; i > lo; i--) {
        const fe ai = a[i];
        a[i] = fe_mul(inv, pre[i - 1]);
        inv = fe_mul(inv, ai);
    }
    a[lo] = inv;
}

__global__ void __launch_bounds__(128) k_check16e_verify(const gpt* __restrict__ P, const fe* __restrict__ inv_u2,
                                                         uint32_t n, const uint8_t* __restrict__ r,
                                                         uint8_t* __restrict__ verdict) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t b[32];
    load32(r + (size_t)i * 32, b);
    verdict[i] = rist_encoding_matches(P[i], inv_u2[i], b) ? 1 : 0;
}

__global__ void __launch_bounds__(128) k_check_thread(const gcached* __restrict__ tabY,
                                                      const gcached* __restrict__ tabB, uint32_t n,
                                                      const uint32_t* __restrict__ e,
                                                      const uint32_t* __restrict__ s,
                                                      const uint8_t* __restrict__ r,
                                                      uint8_t* __restrict__ enc,
                                                      uint8_t* __restrict__ verdict) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint32_t v[8];
    gpt acc = pt_identity();
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = e[(size_t)i * 8 + k];
    acc = comb256_mul_add(acc, tabY, v);
#pragma unroll
    for (int k = 0; k < 8; k++) v[k] = s[(size_t)i * 8 + k];
    acc = comb256_mul_add(acc, tabB, v);
    uint8_t out[32];
    rist_encode(acc, out);
    if (enc)
#pragma unroll
        for (int k = 0; k < 32; k++) enc[(size_t)i * 32 + k] = out[k];
    if (r && verdict) {
        uint32_t diff = 0;
#pragma unroll
        for (int k = 0; k < 32; k++) diff |= out[k] ^ r[(size_t)i * 32 + k];
        verdict[i] = diff == 0;
    }
}

// ---- batched checks with R decoded ahead ----------------------------------
// commit_check(Y, e, s) == R (byte equality of canonical encodings) <=> R is
// a valid encoding and eY + sB == R as ristretto classes (RFC 9496 §4.3.3).
// Decoding R does not depend on the hashes, so it runs on a side stream
// while the log is hashed; the check itself is then 64 mixed additions spread
// over 8 lanes (8 radix-256 windows each, 4 of e and 4 of s) and a 3-level
// shuffle tree, plus a 4-multiplication compare: no inverse square root on
// the critical path and 8x the threads of the thread-per-check kernel.
#ifndef POSLO_DECODE_MINB
#define POSLO_DECODE_MINB 1
#endif
__global__ void __launch_bounds__(128, POSLO_DECODE_MINB) k_decode_pts(const uint8_t* __restrict__ enc, uint32_t n,
                                                    gpt* __restrict__ out, uint8_t* __restrict__ ok) {
    const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t b[32];
    load32(enc + (size_t)i * 32, b);
    gpt P;
    const bool v = rist_decode(b, P);
    out[i] = v ? P : pt_identity();
    ok[i] = v ? 1 : 0;
}

__device__ __forceinline__ gpt shfl_pt(const gpt& p, int off) {
    gpt r;
    const fe* src[4] = {&p.X, &p.Y, &p.Z, &p.T};
    fe* dst[4] = {&r.X, &r.Y, &r.Z, &r.T};
#pragma unroll
    for (int c = 0; c < 4; c++)
#pragma unroll
        for (int k = 0; k < (int)(sizeof(fe) / 4); k++) dst[c]->v[k] = __shfl_down_sync(0xffffffffu, src[c]->v[k], off, 8);
    return r;
}

#ifndef POSLO_CHECK_MINB
#define POSLO_CHECK_MINB 1
#endif
__global__ void __launch_bounds__(128, POSLO_CHECK_MINB) k_check_split(const gcached* __restrict__ tabY,
                                                     const gcached* __restrict__ tabB, uint32_t n,
                                                     const uint32_t* __restrict__ e,
                                                     const uint32_t* __restrict__ s,
                                                     const gpt* __restrict__ R,
                                                     const uint8_t* __restrict__ rok,
                                                     uint8_t* __restrict__ verdict) {
    const uint32_t gid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t i = gid >> 3, sub = gid & 7;
    const bool live = i < n;
    const uint32_t ic = live ? i : 0;
    // this lane's windows: signed radix-256 digits 4 sub .. 4 sub + 3 of e (Y
    // table) and of s (alpha table); the recoding carry runs through all 32
    uint32_t ve[8], vs[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        ve[k] = e[(size_t)ic * 8 + k];
        vs[k] = s[(size_t)ic * 8 + k];
    }
    int de[4] = {0, 0, 0, 0}, dsg[4] = {0, 0, 0, 0};
    int ce = 0, cs = 0;
#pragma unroll
    for (int k = 0; k < 32; k++) {
        const int a = (int)((ve[k >> 2] >> (8 * (k & 3))) & 255u) + ce;
        ce = (a + 128) >> 8;
        const int b = (int)((vs[k >> 2] >> (8 * (k & 3))) & 255u) + cs;
        cs = (b + 128) >> 8;
        if ((uint32_t)(k >> 2) == sub) {
            de[k & 3] = a - (ce << 8);
            dsg[k & 3] = b - (cs << 8);
        }
    }
    // one addition site for the 8 windows (e then s per window): a rolled loop
    // keeps the kernel small enough for the instruction cache
    uint32_t pe = 0, ps = 0;  // the four signed digits, one per byte
#pragma unroll
    for (int q = 0; q < 4; q++) {
        pe |= ((uint32_t)de[q] & 0xffu) << (8 * q);
        ps |= ((uint32_t)dsg[q] & 0xffu) << (8 * q);
    }
    gpt acc = pt_identity();
#pragma unroll 1
    for (int t = 0; t < 8; t++) {
        const int q = t >> 1;
        const int dig = (int)(int8_t)(((t & 1) ? ps : pe) >> (8 * q));
        if (!dig) continue;
        const int a = dig < 0 ? -dig : dig;
        const gcached c = ((t & 1) ? tabB : tabY)[128 * (4 * (int)sub + q) + a - 1];
        acc = pt_add_cached(acc, dig < 0 ? cached_neg(c) : c);
    }
#pragma unroll 1
    for (int off = 4; off >= 1; off >>= 1) {
        const gpt o = shfl_pt(acc, off);
        if (sub < (uint32_t)off) acc = pt_add(acc, o);
    }
    if (live && sub == 0) verdict[i] = (rok[i] && rist_equal(acc, R[i])) ? 1 : 0;
}

// k_check_split on radix-2^16 combs (16 windows per scalar, 32768 affine
// Niels points per window: 60 MiB per base in HBM): each lane adds 2 windows
// of e and 2 of s, half the additions of the radix-256 form, for batches
// large enough to amortise the table builds (and Y's, cached per Y).
__global__ void __launch_bounds__(128) k_check_split16(const gcached* __restrict__ tabY,
                                                       const gcached* __restrict__ tabB, uint32_t n,
                                                       const uint32_t* __restrict__ e,
                                                       const uint32_t* __restrict__ s,
                                                       const gpt* __restrict__ R,
                                                       const uint8_t* __restrict__ rok,
                                                       uint8_t* __restrict__ verdict) {
    const uint32_t gid = blockIdx.x * blockDim.x + threadIdx.x;
    const uint32_t i = gid >> 3, sub = gid & 7;
    const bool live = i < n;
    const uint32_t ic = live ? i : 0;
    uint32_t ve[8], vs[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        ve[k] = e[(size_t)ic * 8 + k];
        vs[k] = s[(size_t)ic * 8 + k];
    }
    // signed radix-2^16 digits (scalars < 2^253: the top digit never carries out);
    // this lane keeps digits 2 sub and 2 sub + 1 of each
    int de[2] = {0, 0}, dsg[2] = {0, 0};
    int ce = 0, cs = 0;
#pragma unroll
    for (int k = 0; k < 16; k++) {
        const int a = (int)((ve[k >> 1] >> (16 * (k & 1))) & 0xffffu) + ce;
        ce = (a + 32768) >> 16;
        const int b = (int)((vs[k >> 1] >> (16 * (k & 1))) & 0xffffu) + cs;
        cs = (b + 32768) >> 16;
        if ((uint32_t)(k >> 1) == sub) {
            de[k & 1] = a - (ce << 16);
            dsg[k & 1] = b - (cs << 16);
        }
    }
    gpt acc = pt_identity();
#pragma unroll 1
    for (int t = 0; t < 4; t++) {
        const int q = t >> 1;
        const int dig = (t & 1) ? dsg[q] : de[q];
        if (!dig) continue;
        const int a = dig < 0 ? -dig : dig;
        const gcached c = ((t & 1) ? tabB : tabY)[32768 * (2 * (int)sub + q) + a - 1];
        acc = pt_add_cached(acc, dig < 0 ? cached_neg(c) : c);
    }
#pragma unroll 1
    for (int off = 4; off >= 1; off >>= 1) {
        const gpt o = shfl_pt(acc, off);
        if (sub < (uint32_t)off) acc = pt_add(acc, o);
    }
    if (live && sub == 0) verdict[i] = (rok[i] && rist_equal(acc, R[i])) ? 1 : 0;
}

// Masked segmented fold over already-decoded points (distillation after the
// split checks: R-hat is decoded once for both).
__global__ void __launch_bounds__(128) k_segfold_gpt(const gpt* __restrict__ pts,
                                                     const uint32_t* __restrict__ seg,
                                                     const uint8_t* __restrict__ mask,
                                                     uint8_t* __restrict__ out) {
    __shared__ gpt sh[128];
    const uint32_t g = blockIdx.x, lo = seg[g], hi = seg[g + 1];
    gpt acc = pt_identity();
    for (uint32_t k = lo + threadIdx.x; k < hi; k += blockDim.x)
        if (!mask || mask[k]) acc = pt_add(acc, pts[k]);
    block_reduce_pt(acc, sh);
    if (threadIdx.x < 32) {  // the encode by the whole warp 0
        uint8_t o[32];
        rist_encode_w(acc, o);
        if (threadIdx.x == 0)
#pragma unroll
            for (int k = 0; k < 32; k++) out[(size_t)g * 32 + k] = o[k];
    }
}

// ---- split single check: commit_check(Y, e, s) == R <=> e*Y == R - s*B ----
// The pre part (R decode + s*B) does not depend on e-hat, so paver runs it on
// a side stream concurrently with hashing; after hashing only e*Y (64 table
// lookups + a 6-level tree) and a 4-multiplication equality remain.
struct CheckPre {
    gpt T;   // R - s*B
    int ok;  // R decoded
};
static_assert(sizeof(CheckPre) <= 256, "b_pre holds one CheckPre");

__device__ __forceinline__ void named_sync64() { asm volatile("bar.sync 1, 64;" ::: "memory"); }
__device__ __forceinline__ void named_sync128() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// 64 threads each take one signed radix-16 window of the scalar from the
// table, then a 6-level shared-memory tree (named barrier over warps 0-1).
__device__ __forceinline__ gpt comb_tree64(const gcached* tab, const uint32_t* scal, int8_t* dig, gpt* sh) {
    const int t = threadIdx.x;
    if (t == 0) {
        uint32_t v[8];
#pragma unroll
        for (int k = 0; k < 8; k++) v[k] = scal[k];
        int8_t d[64];
        sc_signed_radix16(v, d);
        for (int k = 0; k < 64; k++) dig[k] = d[k];
    }
    named_sync64();
    gpt acc = pt_identity();
    if (dig[t]) acc = pt_add_cached(acc, table_pick(tab, t, dig[t]));
    sh[t] = acc;
    named_sync64();
    for (int w = 32; w >= 1; w >>= 1) {
        if (t < w) sh[t] = pt_add(sh[t], sh[t + w]);
        named_sync64();
    }
    return sh[0];
}

__global__ void __launch_bounds__(96) k_check_pre(const gcached* __restrict__ tabB,
                                                  const uint32_t* __restrict__ s,
                                                  const uint8_t* __restrict__ r_enc,
                                                  CheckPre* __restrict__ out) {
    __shared__ int8_t dig[64];
    __shared__ gpt sh[64];
    __shared__ gpt R;
    __shared__ int rok;
    if (threadIdx.x < 64) {
        gpt S = comb_tree64(tabB, s, dig, sh);
        (void)S;
    } else {  // warp 2 decodes R concurrently (the whole warp: rist_decode_w)
        uint8_t b[32];
        load32(r_enc, b);
        gpt P;
        const bool ok = rist_decode_w(b, P);
        if (threadIdx.x == 64) {
            rok = ok ? 1 : 0;
            R = P;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        out->ok = rok;
        out->T = rok ? pt_add(R, pt_neg(sh[0])) : pt_identity();
    }
}

__global__ void __launch_bounds__(64) k_check_post(const gcached* __restrict__ tabY,
                                                   const uint32_t* __restrict__ e,
                                                   const CheckPre* __restrict__ pre,
                                                   uint8_t* __restrict__ verdict) {
    __shared__ int8_t dig[64];
    __shared__ gpt sh[64];
    gpt E = comb_tree64(tabY, e, dig, sh);
    if (threadIdx.x == 0) verdict[0] = (pre->ok && rist_equal(E, pre->T)) ? 1 : 0;
}

// Masked segmented fold: CTA g folds the valid points of [seg[g], seg[g+1]).
__global__ void __launch_bounds__(128) k_segfold_points(const uint8_t* __restrict__ pts,
                                                        const uint32_t* __restrict__ seg,
                                                        const uint8_t* __restrict__ mask,
                                                        uint8_t* __restrict__ out, int* bad) {
    __shared__ gpt sh[128];
    const uint32_t g = blockIdx.x, lo = seg[g], hi = seg[g + 1];
    gpt acc = pt_identity();
    for (uint32_t k = lo + threadIdx.x; k < hi; k += blockDim.x) {
        if (mask && !mask[k]) continue;
        uint8_t b[32];
        load32(pts + (size_t)k * 32, b);
        gpt P;
        if (!rist_decode(b, P)) {
            atomicOr(bad, 1);
            continue;
        }
        acc = pt_add(acc, P);
    }
    block_reduce_pt(acc, sh);
    if (threadIdx.x < 32) {  // the encode by the whole warp 0
        uint8_t o[32];
        rist_encode_w(acc, o);
        if (threadIdx.x == 0)
#pragma unroll
            for (int k = 0; k < 32; k++) out[(size_t)g * 32 + k] = o[k];
    }
}

// One distill_epoch step (poslo_gpu_distill_step) in one CTA of 224 threads:
// warps 0-3 evaluate e Y + s B on the radix-16 combs (thread t < 64 window t
// of e on Y's table, 64 + t window t of s on alpha's) while warps 4-6 decode
// R-hat and the two running aggregates' points (a warp-cooperative inverse
// square root each); the verdict is the
// projective ristretto equality of e Y + s B and R-hat (no encode on the
// check's path), and on a valid verdict R-hat is added to both aggregates and
// the two sums encoded by two warps at once (Scalar::add / group_combine,
// distiller.cpp:45-53). in: s_items = [acc_s0, s_hat, acc_s1] (8 limbs each),
// pts = [acc_r0, r_hat, acc_r1] encodings. out: verdict, out_s (2 x 8 limbs),
// out_r (2 x 32 B); *bad on an undecodable point.
__global__ void __launch_bounds__(224) k_distill_step(const gcached* __restrict__ tabY,
                                                      const gcached* __restrict__ tabB,
                                                      const uint32_t* __restrict__ e, const uint32_t* __restrict__ s_items,
                                                      const uint8_t* __restrict__ pts, uint8_t* __restrict__ verdict,
                                                      uint32_t* __restrict__ out_s, uint8_t* __restrict__ out_r,
                                                      int* __restrict__ bad) {
    __shared__ int8_t dig[128];
    __shared__ gpt sh[128];
    __shared__ gpt dec[3];
    __shared__ int dec_ok[3];
    __shared__ int s_verdict;
    const int t = threadIdx.x;
    if (t >= 128) {  // warps 4-6: the three decodes (a warp each), concurrently with the comb
        const int q = (t - 128) >> 5;
        uint8_t b[32];
        load32(pts + 32 * q, b);
        gpt P;
        const bool ok = rist_decode_w(b, P);
        if ((t & 31) == 0) {
            dec[q] = ok ? P : pt_identity();
            dec_ok[q] = ok;
        }
    } else {  // warps 0-3: comb and tree, synchronised among themselves only (barrier 1)
        if (t < 2) {
            uint32_t v[8];
            const uint32_t* src = t == 0 ? e : s_items + 8;
#pragma unroll
            for (int k = 0; k < 8; k++) v[k] = src[k];
            int8_t d[64];
            sc_signed_radix16(v, d);
            for (int k = 0; k < 64; k++) dig[64 * t + k] = d[k];
        }
        named_sync128();
        const int dgt = dig[t];
        gpt acc = pt_identity();
        if (dgt) acc = pt_add_cached(acc, table_pick(t < 64 ? tabY : tabB, t & 63, dgt));
        sh[t] = acc;
        named_sync128();
        for (int w = 64; w >= 1; w >>= 1) {
            if (t < w) sh[t] = pt_add(sh[t], sh[t + w]);
            named_sync128();
        }
    }
    __syncthreads();  // the decodes
    if (t == 0) {
        // an R-hat that does not decode never equals a canonical encoding (false,
        // as the encoding comparison); undecodable aggregates are a format error
        if (!dec_ok[0] || !dec_ok[2]) atomicOr(bad, 1);
        s_verdict = dec_ok[0] && dec_ok[1] && dec_ok[2] && rist_equal(sh[0], dec[1]);
        *verdict = (uint8_t)s_verdict;
    }
    __syncthreads();
    const bool v = s_verdict != 0;
    if (t < 64) {  // the two aggregates: point add + encode, a warp each
        const int w = t >> 5;
        const int a = 2 * w;  // item 0 = valid aggregate, item 2 = umbrella aggregate
        uint8_t o[32];
        if (v) {
            rist_encode_w(pt_add(dec[a], dec[1]), o);
        } else {
            load32(pts + 32 * a, o);
        }
        if ((t & 31) == 0)
#pragma unroll
            for (int k = 0; k < 32; k++) out_r[32 * w + k] = o[k];
    } else if (t == 64 || t == 65) {  // scalars
        const int i = t - 64;
        uint32_t a[8], b[8], r[8];
#pragma unroll
        for (int k = 0; k < 8; k++) {
            a[k] = s_items[16 * i + k];
            b[k] = v ? s_items[8 + k] : 0u;
        }
        sc_add(a, b, r);
#pragma unroll
        for (int k = 0; k < 8; k++) out_s[8 * i + k] = r[k];
    }
}

}  // namespace

void launch_distill_step(const void* d_tabY, const void* d_tabB, const uint32_t* d_e, const uint32_t* d_s_items,
                         const uint8_t* d_pts, uint8_t* d_verdict, uint32_t* d_out_s, uint8_t* d_out_r, int* d_bad,
                         cudaStream_t s) {
    k_distill_step<<<1, 224, 0, s>>>(static_cast<const gcached*>(d_tabY), static_cast<const gcached*>(d_tabB), d_e,
                                     d_s_items, d_pts, d_verdict, d_out_s, d_out_r, d_bad);
}

void launch_decode_points(const uint8_t* d_enc, uint32_t n, void* d_pts, uint8_t* d_ok, cudaStream_t s) {
    if (!n) return;
    k_decode_pts<<<(n + 127) / 128, 128, 0, s>>>(d_enc, n, static_cast<gpt*>(d_pts), d_ok);
}

void launch_check_split(const void* d_tabY256, const void* d_tabB256, uint32_t n, const uint32_t* d_e,
                        const uint32_t* d_s, const void* d_pts, const uint8_t* d_ok, uint8_t* d_verdict,
                        cudaStream_t s) {
    if (!n) return;
    const uint64_t threads = (uint64_t)n * 8;
    k_check_split<<<(unsigned)((threads + 127) / 128), 128, 0, s>>>(
        static_cast<const gcached*>(d_tabY256), static_cast<const gcached*>(d_tabB256), n, d_e, d_s,
        static_cast<const gpt*>(d_pts), d_ok, d_verdict);
}

void launch_check_thread16(const void* d_tabY16, const void* d_tabB16, uint32_t n, const uint32_t* d_e,
                           const uint32_t* d_s, const uint8_t* d_r, uint8_t* d_enc, uint8_t* d_verdict,
                           cudaStream_t s) {
    if (!n) return;
    k_check_thread16<<<(n + 127) / 128, 128, 0, s>>>(static_cast<const gcached*>(d_tabY16),
                                                     static_cast<const gcached*>(d_tabB16), n, d_e, d_s, d_r, d_enc,
                                                     d_verdict);
}

void launch_check_thread16d(const void* d_tabY16, const void* d_tabB16, uint32_t n, const uint32_t* d_e,
                            const uint32_t* d_s, const void* d_pts, const uint8_t* d_ok, uint8_t* d_verdict,
                            cudaStream_t s) {
    if (!n) return;
    k_check_thread16d<<<(n + 127) / 128, 128, 0, s>>>(static_cast<const gcached*>(d_tabY16),
                                                      static_cast<const gcached*>(d_tabB16), n, d_e, d_s,
                                                      static_cast<const gpt*>(d_pts), d_ok, d_verdict);
}

void launch_check16e(const void* d_tabY16, const void* d_tabB16, uint32_t n, const uint32_t* d_e, const uint32_t* d_s,
                     const uint8_t* d_r, void* d_P, void* d_u2, void* d_pre, uint8_t* d_verdict, cudaStream_t s) {
    if (!n) return;
    gpt* P = static_cast<gpt*>(d_P);
    fe* u2 = static_cast<fe*>(d_u2);
    fe* pre = static_cast<fe*>(d_pre);
    k_check16e_comb<<<(n + 127) / 128, 128, 0, s>>>(static_cast<const gcached*>(d_tabY16),
                                                    static_cast<const gcached*>(d_tabB16), n, d_e, d_s, P, u2);
    const uint32_t chunks = (n + kInvChunk - 1) / kInvChunk;
    k_batch_invert<<<(chunks + 63) / 64, 64, 0, s>>>(u2, pre, n);
    k_check16e_verify<<<(n + 127) / 128, 128, 0, s>>>(P, u2, n, d_r, d_verdict);
}

void launch_check_split16(const void* d_tabY16, const void* d_tabB16, uint32_t n, const uint32_t* d_e,
                          const uint32_t* d_s, const void* d_pts, const uint8_t* d_ok, uint8_t* d_verdict,
                          cudaStream_t s) {
    if (!n) return;
    const uint64_t threads = (uint64_t)n * 8;
    k_check_split16<<<(unsigned)((threads + 127) / 128), 128, 0, s>>>(
        static_cast<const gcached*>(d_tabY16), static_cast<const gcached*>(d_tabB16), n, d_e, d_s,
        static_cast<const gpt*>(d_pts), d_ok, d_verdict);
}

void launch_segfold_decoded(const void* d_pts, const uint32_t* d_seg, uint32_t n_seg, const uint8_t* d_mask,
                            uint8_t* d_out, cudaStream_t s) {
    if (!n_seg) return;
    k_segfold_gpt<<<n_seg, 128, 0, s>>>(static_cast<const gpt*>(d_pts), d_seg, d_mask, d_out);
}

void launch_segfold_points(const uint8_t* d_pts, const uint32_t* d_seg, uint32_t n_seg, const uint8_t* d_mask,
                           uint8_t* d_out, int* d_bad, cudaStream_t s) {
    if (!n_seg) return;
    k_segfold_points<<<n_seg, 128, 0, s>>>(d_pts, d_seg, d_mask, d_out, d_bad);
}

void launch_group_check(const uint8_t* d_y, uint32_t n, const uint32_t* d_e, const uint32_t* d_s,
                        const uint8_t* d_r, uint8_t* d_enc, uint8_t* d_verdict, int* d_ybad,
                        cudaStream_t s) {
    if (!n) return;
    k_group_check<<<(n + 127) / 128, 128, 0, s>>>(d_y, n, d_e, d_s, d_r, d_enc, d_verdict, d_ybad);
}

void launch_point_fold(const uint8_t* d_pts, uint64_t n, uint8_t* d_out, int* d_bad, void* d_scratch,
                       cudaStream_t s) {
    uint64_t want = (n + 127) / 128;
    uint32_t blocks = (uint32_t)(want < 1 ? 1 : (want > 1024 ? 1024 : want));
    gpt* part = static_cast<gpt*>(d_scratch);
    k_fold_stage1<<<blocks, 128, 0, s>>>(d_pts, n, part, d_bad);
    k_fold_stage2<<<1, 128, 0, s>>>(part, blocks, d_out);
}

void launch_point_validate(const uint8_t* d_pts, uint32_t n, uint8_t* d_ok, cudaStream_t s) {
    if (!n) return;
    k_validate<<<(n + 127) / 128, 128, 0, s>>>(d_pts, n, d_ok);
}

// One chain of powers pk[i] = 16^i P (i < 64) serves every comb radix
// (256^k P = pk[2k], 2^(16k) P = pk[4k]): computed once per point.
void launch_table_powers(const uint8_t* d_enc, void* d_pk, int* d_bad, cudaStream_t s) {
    k_table_pow<4><<<1, 32, 0, s>>>(d_enc, static_cast<gpt*>(d_pk), d_bad);
}

void launch_table_fill(int kind, const void* d_pk, void* d_table, cudaStream_t s) {
    const gpt* pk = static_cast<const gpt*>(d_pk);
    gcached* tab = static_cast<gcached*>(d_table);
    if (kind == 0)
        k_table_fill<<<4, 128, 0, s>>>(pk, tab);
    else if (kind == 1)
        k_table_fill256<<<32, 128, 0, s>>>(pk, tab);
    else
        k_table_fill65536<<<16 * (32768 / kRun) / 128, 128, 0, s>>>(pk, tab);
}

void launch_build_table(const uint8_t* d_enc, void* d_pk_scratch, void* d_table, int* d_bad,
                        cudaStream_t s) {
    launch_table_powers(d_enc, d_pk_scratch, d_bad, s);
    launch_table_fill(0, d_pk_scratch, d_table, s);
}

void launch_build_table65536(const uint8_t* d_enc, void* d_pk_scratch, void* d_table, int* d_bad, cudaStream_t s) {
    launch_table_powers(d_enc, d_pk_scratch, d_bad, s);
    launch_table_fill(2, d_pk_scratch, d_table, s);
}

void launch_build_table256(const uint8_t* d_enc, void* d_pk_scratch, void* d_table, int* d_bad, cudaStream_t s) {
    launch_table_powers(d_enc, d_pk_scratch, d_bad, s);
    launch_table_fill(1, d_pk_scratch, d_table, s);
}

void launch_group_check_comb(const void* d_tabY, const void* d_tabB, const void* d_tabY256,
                             const void* d_tabB256, uint32_t n, const uint32_t* d_e, const uint32_t* d_s,
                             const uint8_t* d_r, uint8_t* d_enc, uint8_t* d_verdict, cudaStream_t s) {
    if (!n) return;
    if (n <= kCtaCheckMax)
        k_check_cta<<<n, 128, 0, s>>>(static_cast<const gcached*>(d_tabY), static_cast<const gcached*>(d_tabB),
                                      d_e, d_s, d_r, d_enc, d_verdict);
    else
        k_check_thread<<<(n + 127) / 128, 128, 0, s>>>(static_cast<const gcached*>(d_tabY256),
                                                       static_cast<const gcached*>(d_tabB256), n, d_e, d_s,
                                                       d_r, d_enc, d_verdict);
}

void launch_check_pre(const void* d_tabB, const uint32_t* d_s, const uint8_t* d_r, void* d_pre,
                      cudaStream_t s) {
    k_check_pre<<<1, 96, 0, s>>>(static_cast<const gcached*>(d_tabB), d_s, d_r, static_cast<CheckPre*>(d_pre));
}

void launch_check_post(const void* d_tabY, const uint32_t* d_e, const void* d_pre, uint8_t* d_verdict,
                       cudaStream_t s) {
    k_check_post<<<1, 64, 0, s>>>(static_cast<const gcached*>(d_tabY), d_e, static_cast<const CheckPre*>(d_pre),
                                  d_verdict);
}

}  // namespace poslo_gpu
