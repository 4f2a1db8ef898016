// K1+K2 fast path for suite 1 (SHA-256) with 32-byte entries, uniform epochs.
#include "entry_hash.cuh"
#include "tile_common.cuh"

namespace poslo_gpu {

namespace {

using namespace tilec;

// ---------------------------------------------------------------- K1+K2, suite 1, L = 32
template <int T, int E>
__global__ void __launch_bounds__(T) k_hash_s1_l32(const uint4* __restrict__ pay, uint32_t n2,
                                                   uint32_t tpe, const uint4* __restrict__ x0,
                                                   uint32_t* __restrict__ partial,
                                                   uint32_t* __restrict__ etilde) {
    __shared__ uint32_t red[(T / 32) * 17];
    const uint32_t tile = blockIdx.x;
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
            entry_limbs_s1_l32(x0w, pre, j, m, limbs);
            acc17_add16(acc, limbs);
        }
    }
    block_reduce_acc17(acc, red);
    if (threadIdx.x == 0) store_tile(acc, tpe == 1, ep, tile, partial, etilde);
}

}  // namespace

void launch_hash_s1_l32(const EntryLayout& lay, const TileMap& tm, const uint4* d_x0,
                        uint32_t* d_partial, uint32_t* d_etilde, cudaStream_t s) {
    uint32_t n_tiles = tm.n_epochs * tm.tiles_per_epoch;
    if (!n_tiles) return;
    const uint4* pay = reinterpret_cast<const uint4*>(lay.payload);
    if (tm.tile_entries == 256 * 4)
        k_hash_s1_l32<256, 4><<<n_tiles, 256, 0, s>>>(pay, tm.n2, tm.tiles_per_epoch, d_x0, d_partial, d_etilde);
    else if (tm.tile_entries == 128 * 2)
        k_hash_s1_l32<128, 2><<<n_tiles, 128, 0, s>>>(pay, tm.n2, tm.tiles_per_epoch, d_x0, d_partial, d_etilde);
    else
        k_hash_s1_l32<128, 1><<<n_tiles, 128, 0, s>>>(pay, tm.n2, tm.tiles_per_epoch, d_x0, d_partial, d_etilde);
}

}  // namespace poslo_gpu
