// K1+K2 fast path for suite 1 (SHA-256) with 32-byte entries, uniform epochs.
#include <cstdlib>

#include "entry_hash.cuh"
#include "tile_common.cuh"

// Pipe assignment of the lean kernel's SHA rounds (sha256.cuh SHA_RND_SEL).
// 5: every addition on the FMA pipe, h + W + K included, so the ALU pipe
// carries only the rotations and LOP3s (12.05 -> 11.52 ms per 2^26 entries
// vs 2, which keeps h + W + K as one IADD3 on the ALU pipe). This needs the
// multiplier `one` in a uniform register (IMAD R, R, UR, R): no FMA-pipe add
// may take an immediate or uniform addend (sha256_rounds_head's CM masks),
// or ptxas holds `one` in a vector register for the whole kernel and every
// IMAD reads three vector registers (slower than 2, profiles/r02_ab_var.txt).
#ifndef POSLO_S1_FMA
#define POSLO_S1_FMA 5
#endif
#ifndef POSLO_S1_LOOP_FMA
#define POSLO_S1_LOOP_FMA POSLO_S1_FMA  // ... of the rolled rounds 32-63
#endif
#ifndef POSLO_S1_OTSB_FMA
#define POSLO_S1_OTSB_FMA POSLO_S1_FMA  // ... of onetime_seed rounds 16-31
#endif
#ifndef POSLO_S1_ENTB_FMA
#define POSLO_S1_ENTB_FMA POSLO_S1_FMA  // ... of the entry hashes' rounds 16-31
#endif
#ifndef POSLO_ENTRY_SPEC
#define POSLO_ENTRY_SPEC 1  // entry-hash head specialisation (W13 = W14 = 0): 12.13 vs 12.16 ms
#endif
#ifndef POSLO_OTS_SPEC
#define POSLO_OTS_SPEC 1  // onetime_seed-specialised schedule in the lean kernel (12.15 vs 12.34 ms)
#endif

namespace poslo_gpu {

namespace {

using namespace tilec;

constexpr int kLeanStride = 256;  // threads per CTA of the register-lean kernel

// ---------------------------------------------------------------- K1+K2, suite 1, L = 32
// Compact variant (default): E entries per thread in a rolled loop, the
// three compressions of an entry in one rolled loop over shared round code.
template <int T, int E, int FMA>
__global__ void __launch_bounds__(T) k_hash_s1_l32c(const uint4* __restrict__ pay, uint32_t n2,
                                                    uint32_t tpe, const uint4* __restrict__ x0,
                                                    uint32_t* __restrict__ partial,
                                                    uint32_t* __restrict__ etilde, uint32_t tile0,
                                                    const PipeK pk) {
    __shared__ uint32_t red[(T / 32) * 17];
    const uint32_t tile = tile0 + blockIdx.x;
    const uint32_t ep = tile / tpe, sub = tile - ep * tpe;
    const uint4 xr = __ldg(x0 + ep);
    const uint32_t x0w[4] = {bswap32(xr.x), bswap32(xr.y), bswap32(xr.z), bswap32(xr.w)};
    uint32_t pre[8];
    ots_pre(x0w, pre);
    uint32_t acc[17];
    acc17_zero(acc);
    const uint32_t jbase = sub * (T * E) + threadIdx.x;
#pragma unroll 1
    for (int i = 0; i < E; i++) {
        const uint32_t j = jbase + i * T;
        if (j < n2) {
            const uint64_t ent = (uint64_t)ep * n2 + j;
            const uint4 a = __ldg(pay + 2 * ent), b = __ldg(pay + 2 * ent + 1);
            const uint32_t m[8] = {bswap32(a.x), bswap32(a.y), bswap32(a.z), bswap32(a.w),
                                   bswap32(b.x), bswap32(b.y), bswap32(b.z), bswap32(b.w)};
            uint32_t limbs[16];
            entry_limbs_s1_l32_compact<FMA>(x0w, pre, j, m, limbs, pk);
            acc17_add16(acc, limbs);
        }
    }
    block_reduce_acc17(acc, red);
    if (threadIdx.x == 0) store_tile(acc, tpe == 1, ep, tile, partial, etilde);
}

// Register-lean multi-epoch kernel. The three compressions of an entry are
// a dependency chain with little instruction-level parallelism, so the
// hash rate is set by how many warps each scheduler can choose from. Here
// only the compression state (16 schedule words + 8 working words), the
// one-time seed x and loop indices stay in registers: the per-epoch seed
// words and hoisted onetime_seed mid-state live in shared memory, the entry
// is re-read from L1 for each of its two hashes, and the running sums live
// in shared memory as two 9-limb accumulators (H0 and H1 halves, one column
// per thread: conflict-free). That allows MINB CTAs of T threads per SM.
PD void smem_acc9_add8(uint32_t* s, const uint32_t v[8]) {
    uint32_t a[9];
#pragma unroll
    for (int k = 0; k < 9; k++) a[k] = s[k * kLeanStride];
    asm("add.cc.u32 %0, %0, %9;\n\t"
        "addc.cc.u32 %1, %1, %10;\n\t"
        "addc.cc.u32 %2, %2, %11;\n\t"
        "addc.cc.u32 %3, %3, %12;\n\t"
        "addc.cc.u32 %4, %4, %13;\n\t"
        "addc.cc.u32 %5, %5, %14;\n\t"
        "addc.cc.u32 %6, %6, %15;\n\t"
        "addc.cc.u32 %7, %7, %16;\n\t"
        "addc.u32 %8, %8, 0;\n\t"
        : "+r"(a[0]), "+r"(a[1]), "+r"(a[2]), "+r"(a[3]), "+r"(a[4]), "+r"(a[5]), "+r"(a[6]), "+r"(a[7]),
          "+r"(a[8])
        : "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
#pragma unroll
    for (int k = 0; k < 9; k++) s[k * kLeanStride] = a[k];
}

template <int T, int EPC, int FMA, int MINB>
__global__ void __launch_bounds__(T, MINB) k_hash_s1_l32r(const uint4* __restrict__ pay, uint32_t n2,
                                                          uint32_t n_epochs, uint32_t epoch0,
                                                          const uint4* __restrict__ x0,
                                                          uint32_t* __restrict__ epoch_sum, const PipeK pk_in) {
    static_assert(T == kLeanStride, "accumulator column stride");
    const PipeK pk = pk_in;
    if (FMA == 5) sha_k_smem_init();
    constexpr int TPE = T / EPC;  // threads per epoch (multiple of 32)
    __shared__ uint32_t s_pre[EPC][8], s_x0w[EPC][4];
#if POSLO_OTS_SPEC
    __shared__ OtsEpoch s_ots[EPC];
#endif
    __shared__ uint32_t s_acc[18 * T];  // rows 0..8: sum of H1 words, rows 9..17: sum of H0 words
    __shared__ uint32_t red[(T / 32) * 17];
    const uint32_t le = threadIdx.x / TPE, lt = threadIdx.x % TPE;
    const uint32_t ep = epoch0 + blockIdx.x * EPC + le;
    const bool live = ep < n_epochs;
    if (lt == 0 && live) {
        const uint4 xr = __ldg(x0 + ep);
        const uint32_t x0w[4] = {bswap32(xr.x), bswap32(xr.y), bswap32(xr.z), bswap32(xr.w)};
        uint32_t pre[8];
        ots_pre(x0w, pre);
#pragma unroll
        for (int k = 0; k < 8; k++) s_pre[le][k] = pre[k];
#pragma unroll
        for (int k = 0; k < 4; k++) s_x0w[le][k] = x0w[k];
#if POSLO_OTS_SPEC
        s_ots[le] = ots_epoch_consts(x0w);
#endif
    }
    uint32_t* acc = s_acc + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 18; k++) acc[k * T] = 0;
    __syncthreads();
    if (live) {
#pragma unroll 1
        for (uint32_t j = lt; j < n2; j += TPE) {
            const uint4* pe = pay + 2 * ((uint64_t)ep * n2 + j);
            uint32_t x[4] = {0, 0, 0, 0};
#pragma unroll 1
            for (int c = 0; c < 3; c++) {
                uint32_t W[16], st[8];
                int r0 = 0;
                if (c == 0) {  // x = onetime_seed(x0, j), resumed at round 4
#pragma unroll
                    for (int k = 0; k < 4; k++) W[k] = s_x0w[le][k];
                    W[4] = j;
                    W[5] = 0x80000000u;
#pragma unroll
                    for (int k = 6; k < 15; k++) W[k] = 0;
                    W[15] = 160u;
#pragma unroll
                    for (int k = 0; k < 8; k++) st[k] = s_pre[le][k];
                    r0 = 4;
                } else {
                    const uint4 a = __ldg(pe), b = __ldg(pe + 1);
                    const uint32_t r[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};  // little-endian words
                    if (c == 1) {  // m || x
#pragma unroll
                        for (int k = 0; k < 8; k++) W[k] = bswap32(r[k]);
                        W[8] = x[0]; W[9] = x[1]; W[10] = x[2]; W[11] = x[3];
                        W[12] = 0x80000000u; W[13] = 0; W[14] = 0; W[15] = 384u;
                    } else {  // 0x01 || m || x: each big-endian word is one PRMT of two raw words
                        W[0] = __byte_perm(r[0], 1u, 0x4012u);
#pragma unroll
                        for (int k = 1; k < 8; k++) W[k] = __byte_perm(r[k - 1], r[k], 0x3456u);
                        W[8] = __byte_perm(x[0], r[7], 0x7321u);
                        W[9] = fshr32(x[1], x[0], 8);
                        W[10] = fshr32(x[2], x[1], 8);
                        W[11] = fshr32(x[3], x[2], 8);
                        W[12] = __byte_perm(x[3], 0x80u, 0x0455u);
                        W[13] = 0; W[14] = 0; W[15] = 392u;
                    }
                    sha256_init(st);
                }
#if POSLO_OTS_SPEC
                // onetime_seed: rounds 4-31 on the per-epoch-constant schedule, the
                // 16-round loop (rounds 32-63, or 16-63 for the entry hashes) shared
                int blk0 = 16;
                if (c == 0) {
                    ots_head_rounds<FMA, POSLO_S1_OTSB_FMA>(st, W, j, s_ots[le], pk);
                    blk0 = 32;
                } else {
#if POSLO_ENTRY_SPEC
                    // W13 = W14 = 0, W15 = 384 / 392: sigma terms of W13..W15 fold
                    entry_head_rounds<FMA, POSLO_S1_ENTB_FMA>(st, W, c == 1 ? sha_s1(384u) : sha_s1(392u),
                                           c == 1 ? sha_s0(384u) : sha_s0(392u), pk);
                    blk0 = 32;
#else
                    sha256_rounds_head<FMA>(st, W, 0, pk);
#endif
                }
                sha256_rounds_loop<POSLO_S1_LOOP_FMA>(st, W, blk0, pk);
                (void)r0;
#else
                sha256_rounds_compact<FMA>(st, W, r0, pk);
#endif
                const uint32_t iv[8] = {SHA_IV0, SHA_IV1, SHA_IV2, SHA_IV3, SHA_IV4, SHA_IV5, SHA_IV6, SHA_IV7};
                if (c == 0) {
#pragma unroll
                    for (int k = 0; k < 4; k++) x[k] = st[k] + iv[k];
                } else {
                    // digest word k is limb 7 - k of its half (H0 = high half, H1 = low half)
                    uint32_t v[8];
#pragma unroll
                    for (int k = 0; k < 8; k++) v[7 - k] = st[k] + iv[k];
                    smem_acc9_add8(acc + (c == 1 ? 9 * T : 0), v);
                }
            }
        }
    }
    // acc17 = lo9 + hi9 * 2^256
    uint32_t a17[17];
#pragma unroll
    for (int k = 0; k < 8; k++) a17[k] = acc[k * T];
    {
        uint32_t lo8 = acc[8 * T], hi[9];
#pragma unroll
        for (int k = 0; k < 9; k++) hi[k] = acc[(9 + k) * T];
        asm("add.cc.u32 %0, %9, %10;\n\t"
            "addc.cc.u32 %1, %11, 0;\n\t"
            "addc.cc.u32 %2, %12, 0;\n\t"
            "addc.cc.u32 %3, %13, 0;\n\t"
            "addc.cc.u32 %4, %14, 0;\n\t"
            "addc.cc.u32 %5, %15, 0;\n\t"
            "addc.cc.u32 %6, %16, 0;\n\t"
            "addc.cc.u32 %7, %17, 0;\n\t"
            "addc.u32 %8, %18, 0;\n\t"
            : "=r"(a17[8]), "=r"(a17[9]), "=r"(a17[10]), "=r"(a17[11]), "=r"(a17[12]), "=r"(a17[13]),
              "=r"(a17[14]), "=r"(a17[15]), "=r"(a17[16])
            : "r"(lo8), "r"(hi[0]), "r"(hi[1]), "r"(hi[2]), "r"(hi[3]), "r"(hi[4]), "r"(hi[5]), "r"(hi[6]),
              "r"(hi[7]), "r"(hi[8]));
    }
    const unsigned full = 0xffffffffu;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        uint32_t v[17];
#pragma unroll
        for (int k = 0; k < 17; k++) v[k] = __shfl_down_sync(full, a17[k], off);
        acc17_add17(a17, v);
    }
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int k = 0; k < 17; k++) red[warp * 17 + k] = a17[k];
    __syncthreads();
    if (lt == 0 && live) {
#pragma unroll 1
        for (int w = 1; w < TPE / 32; w++) {
            uint32_t v[17];
#pragma unroll
            for (int k = 0; k < 17; k++) v[k] = red[(warp + w) * 17 + k];
            acc17_add17(a17, v);
        }
        // raw 544-bit epoch sum; the mod-l reduction runs in a full-warp kernel
        // (k_epoch_finalize) or not at all when only e-hat is needed
#pragma unroll
        for (int k = 0; k < 17; k++) epoch_sum[(size_t)ep * 17 + k] = a17[k];
    }
}

}  // namespace

static PipeK pipek_host() { return pipek_make(); }

// Large epochs (n2 > kLeanMaxN2): tiles of T * E entries, partial sums
// finalised per epoch by launch_epoch_finalize.
template <int T, int E>
static void launch_tiled(uint32_t n_tiles, const uint4* pay, const TileMap& tm, const uint4* d_x0,
                         uint32_t* d_partial, uint32_t* d_etilde, cudaStream_t s) {
    k_hash_s1_l32c<T, E, 2><<<n_tiles, T, 0, s>>>(pay, tm.n2, tm.tiles_per_epoch, d_x0, d_partial, d_etilde,
                                                  tm.tile_begin, pipek_host());
}

#ifndef POSLO_LEAN_EPC8_MAX
#define POSLO_LEAN_EPC8_MAX 256  // largest n2 run 8 epochs per 256-thread CTA (else 4)
#endif
#ifndef POSLO_S1_MINB
#define POSLO_S1_MINB 4  // __launch_bounds__ min CTAs/SM of the lean kernel (48 regs: 5 fit anyway)
#endif

void launch_hash_s1_l32(const EntryLayout& lay, const TileMap& tm, const uint4* d_x0,
                        uint32_t* d_partial, uint32_t* d_etilde, cudaStream_t s) {
    uint32_t n_tiles = tm.tile_count ? tm.tile_count : tm.n_epochs * tm.tiles_per_epoch;
    if (!n_tiles) return;
    const uint4* pay = reinterpret_cast<const uint4*>(lay.payload);
    if (tm.tiles_per_epoch == 1 && tm.n2 <= kLeanMaxN2) {
        // whole epochs per CTA (tile == epoch): register-lean kernel, raw epoch sums
        const uint32_t e0 = tm.tile_begin, ne = e0 + n_tiles;
        const PipeK pk = pipek_host();
        // 8 epochs per CTA (a warp per epoch) up to n2 = POSLO_LEAN_EPC8_MAX: the
        // per-epoch prologue amortised over more entries per thread (config 2,
        // n2 = 256: 12.04 vs 12.10 ms); 4 epochs per CTA above (config 3,
        // n2 = 1024: equal within noise)
        if (tm.n2 <= POSLO_LEAN_EPC8_MAX)
            k_hash_s1_l32r<256, 8, POSLO_S1_FMA, POSLO_S1_MINB><<<(n_tiles + 7) / 8, 256, 0, s>>>(pay, tm.n2, ne, e0, d_x0, d_partial, pk);
        else
            k_hash_s1_l32r<256, 4, POSLO_S1_FMA, POSLO_S1_MINB><<<(n_tiles + 3) / 4, 256, 0, s>>>(pay, tm.n2, ne, e0, d_x0, d_partial, pk);
        return;
    }
    if (tm.tile_entries == 256 * 4)
        launch_tiled<256, 4>(n_tiles, pay, tm, d_x0, d_partial, d_etilde, s);
    else if (tm.tile_entries == 128 * 2)
        launch_tiled<128, 2>(n_tiles, pay, tm, d_x0, d_partial, d_etilde, s);
    else
        launch_tiled<128, 1>(n_tiles, pay, tm, d_x0, d_partial, d_etilde, s);
}

}  // namespace poslo_gpu
