// K1+K2 fast path for suite 1 (SHA-256) with 32-byte entries, uniform epochs.
#include <cstdlib>

#include "entry_hash.cuh"
#include "tile_common.cuh"

namespace poslo_gpu {

namespace {

using namespace tilec;

// ---------------------------------------------------------------- K1+K2, suite 1, L = 32
// MODE selects the ALU/FMA pipe balance of the SHA-256 rounds (sha256.cuh);
// `one` is 1 at run time but opaque to the compiler so additions stay IMADs.
template <int T, int E, int MODE>
__global__ void __launch_bounds__(T) k_hash_s1_l32(const uint4* __restrict__ pay, uint32_t n2,
                                                   uint32_t tpe, const uint4* __restrict__ x0,
                                                   uint32_t* __restrict__ partial,
                                                   uint32_t* __restrict__ etilde, uint32_t one,
                                                   uint32_t tile0) {
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
#pragma unroll
    for (int i = 0; i < E; i++) {
        const uint32_t j = jbase + i * T;
        if (j < n2) {
            const uint64_t ent = (uint64_t)ep * n2 + j;
            const uint4 a = __ldg(pay + 2 * ent), b = __ldg(pay + 2 * ent + 1);
            const uint32_t m[8] = {bswap32(a.x), bswap32(a.y), bswap32(a.z), bswap32(a.w),
                                   bswap32(b.x), bswap32(b.y), bswap32(b.z), bswap32(b.w)};
            uint32_t limbs[16];
            entry_limbs_s1_l32<MODE>(x0w, pre, j, m, limbs, one);
            acc17_add16(acc, limbs);
        }
    }
    block_reduce_acc17(acc, red);
    if (threadIdx.x == 0) store_tile(acc, tpe == 1, ep, tile, partial, etilde);
}

// Compact variant (default): E entries per thread in a rolled loop, the
// three compressions of an entry in one rolled loop over shared round code.
template <int T, int E, int FMA>
__global__ void __launch_bounds__(T) k_hash_s1_l32c(const uint4* __restrict__ pay, uint32_t n2,
                                                    uint32_t tpe, const uint4* __restrict__ x0,
                                                    uint32_t* __restrict__ partial,
                                                    uint32_t* __restrict__ etilde, uint32_t tile0,
                                                    uint32_t one) {
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
            entry_limbs_s1_l32_compact<FMA>(x0w, pre, j, m, limbs, one);
            acc17_add16(acc, limbs);
        }
    }
    block_reduce_acc17(acc, red);
    if (threadIdx.x == 0) store_tile(acc, tpe == 1, ep, tile, partial, etilde);
}

// Multi-epoch tiles for small epochs (n2 <= T/EPC * E, e.g. the n2 = 256 of
// the coarse configs): EPC epochs per CTA, T/EPC threads per epoch, so the
// CTA-wide fixed costs (hoisted OTS rounds, the 17-limb reduction) are paid
// once per 4 entries per thread instead of once per 2. Reduction: warp
// shuffles, then the first thread of each epoch folds its warps' partials.
template <int T, int E, int FMA, int EPC, int MINB>
__global__ void __launch_bounds__(T, MINB) k_hash_s1_l32m(const uint4* __restrict__ pay, uint32_t n2,
                                                    uint32_t n_epochs, uint32_t epoch0,
                                                    const uint4* __restrict__ x0,
                                                    uint32_t* __restrict__ etilde, uint32_t one) {
    constexpr int TPE = T / EPC;  // threads per epoch (multiple of 32)
    __shared__ uint32_t red[(T / 32) * 17];
    const uint32_t ep = epoch0 + blockIdx.x * EPC + threadIdx.x / TPE;
    const uint32_t lt = threadIdx.x % TPE;
    const bool live = ep < n_epochs;
    uint32_t acc[17];
    acc17_zero(acc);
    if (live) {
        const uint4 xr = __ldg(x0 + ep);
        const uint32_t x0w[4] = {bswap32(xr.x), bswap32(xr.y), bswap32(xr.z), bswap32(xr.w)};
        uint32_t pre[8];
        ots_pre(x0w, pre);
#pragma unroll 1
        for (int i = 0; i < E; i++) {
            const uint32_t j = lt + i * TPE;
            if (j < n2) {
                const uint64_t ent = (uint64_t)ep * n2 + j;
                const uint4 a = __ldg(pay + 2 * ent), b = __ldg(pay + 2 * ent + 1);
                const uint32_t m[8] = {bswap32(a.x), bswap32(a.y), bswap32(a.z), bswap32(a.w),
                                       bswap32(b.x), bswap32(b.y), bswap32(b.z), bswap32(b.w)};
                uint32_t limbs[16];
                entry_limbs_s1_l32_compact<FMA>(x0w, pre, j, m, limbs, one);
                acc17_add16(acc, limbs);
            }
        }
    }
    const unsigned full = 0xffffffffu;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        uint32_t v[17];
#pragma unroll
        for (int k = 0; k < 17; k++) v[k] = __shfl_down_sync(full, acc[k], off);
        acc17_add17(acc, v);
    }
    const int warp = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int k = 0; k < 17; k++) red[warp * 17 + k] = acc[k];
    __syncthreads();
    if (lt == 0 && live) {
#pragma unroll 1
        for (int w = 1; w < TPE / 32; w++) {
            uint32_t v[17];
#pragma unroll
            for (int k = 0; k < 17; k++) v[k] = red[(warp + w) * 17 + k];
            acc17_add17(acc, v);
        }
        uint32_t e[8];
        sc_reduce_limbs(acc, 17, e);
#pragma unroll
        for (int k = 0; k < 8; k++) etilde[(size_t)ep * 8 + k] = e[k];
    }
}

}  // namespace

static int sha_mode() {
    static int mode = [] {
        const char* e = std::getenv("POSLO_SHA_MODE");
        // 3-6 = compact (3 plain, 4 IMAD rounds, 5 + IMAD schedule, 6 + IMAD K+w),
        // 0-2 = fully unrolled variants (instruction-cache bound; kept for comparison)
        int m = e ? std::atoi(e) : 5;  // measured best on B200: 13.0 ms / 2^26 entries
        return (m < 0 || m > 6) ? 5 : m;
    }();
    return mode;
}

template <int T, int E>
static void launch_cfg(int mode, uint32_t n_tiles, const uint4* pay, const TileMap& tm, const uint4* d_x0,
                uint32_t* d_partial, uint32_t* d_etilde, cudaStream_t s) {
    if (mode == 3)
        k_hash_s1_l32c<T, E, 0><<<n_tiles, T, 0, s>>>(pay, tm.n2, tm.tiles_per_epoch, d_x0, d_partial, d_etilde, tm.tile_begin, 1u);
    else if (mode == 4)
        k_hash_s1_l32c<T, E, 1><<<n_tiles, T, 0, s>>>(pay, tm.n2, tm.tiles_per_epoch, d_x0, d_partial, d_etilde, tm.tile_begin, 1u);
    else if (mode == 5)
        k_hash_s1_l32c<T, E, 2><<<n_tiles, T, 0, s>>>(pay, tm.n2, tm.tiles_per_epoch, d_x0, d_partial, d_etilde, tm.tile_begin, 1u);
    else if (mode == 6)
        k_hash_s1_l32c<T, E, 3><<<n_tiles, T, 0, s>>>(pay, tm.n2, tm.tiles_per_epoch, d_x0, d_partial, d_etilde, tm.tile_begin, 1u);
    else if (mode == 0)
        k_hash_s1_l32<T, E, 0><<<n_tiles, T, 0, s>>>(pay, tm.n2, tm.tiles_per_epoch, d_x0, d_partial, d_etilde, 1u, tm.tile_begin);
    else if (mode == 1)
        k_hash_s1_l32<T, E, 1><<<n_tiles, T, 0, s>>>(pay, tm.n2, tm.tiles_per_epoch, d_x0, d_partial, d_etilde, 1u, tm.tile_begin);
    else
        k_hash_s1_l32<T, E, 2><<<n_tiles, T, 0, s>>>(pay, tm.n2, tm.tiles_per_epoch, d_x0, d_partial, d_etilde, 1u, tm.tile_begin);
}

void launch_hash_s1_l32(const EntryLayout& lay, const TileMap& tm, const uint4* d_x0,
                        uint32_t* d_partial, uint32_t* d_etilde, cudaStream_t s) {
    uint32_t n_tiles = tm.tile_count ? tm.tile_count : tm.n_epochs * tm.tiles_per_epoch;
    if (!n_tiles) return;
    const uint4* pay = reinterpret_cast<const uint4*>(lay.payload);
    const int mode = sha_mode();
    // small epochs (one tile each): multi-epoch CTAs, 4 entries per thread
    if (mode == 5 && tm.tiles_per_epoch == 1 && tm.n2 > 64 && tm.n2 <= 256) {
        const uint32_t e0 = tm.tile_begin, ne = e0 + n_tiles;  // tile == epoch here
        const uint32_t epc = tm.n2 <= 128 ? 8 : 4;
        const uint32_t grid = (n_tiles + epc - 1) / epc;
        static const int minb = [] {
            const char* e = std::getenv("POSLO_S1M_MINB");
            return e ? std::atoi(e) : 3;
        }();
        if (epc == 4 && minb == 2)
            k_hash_s1_l32m<256, 4, 2, 4, 2><<<grid, 256, 0, s>>>(pay, tm.n2, ne, e0, d_x0, d_etilde, 1u);
        else if (epc == 4)
            k_hash_s1_l32m<256, 4, 2, 4, 3><<<grid, 256, 0, s>>>(pay, tm.n2, ne, e0, d_x0, d_etilde, 1u);
        else
            k_hash_s1_l32m<256, 4, 2, 8, 3><<<grid, 256, 0, s>>>(pay, tm.n2, ne, e0, d_x0, d_etilde, 1u);
        return;
    }
    if (tm.tile_entries == 256 * 4)
        launch_cfg<256, 4>(mode, n_tiles, pay, tm, d_x0, d_partial, d_etilde, s);
    else if (tm.tile_entries == 128 * 2)
        launch_cfg<128, 2>(mode, n_tiles, pay, tm, d_x0, d_partial, d_etilde, s);
    else
        launch_cfg<128, 1>(mode, n_tiles, pay, tm, d_x0, d_partial, d_etilde, s);
}

}  // namespace poslo_gpu
