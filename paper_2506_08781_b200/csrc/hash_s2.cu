// K1+K2 fast path for suite 2 (MMO/MDC-2 over AES-128) with 32-byte entries, uniform epochs.
#include "entry_hash.cuh"
#include "tile_common.cuh"

namespace poslo_gpu {

namespace {

using namespace tilec;

// ---------------------------------------------------------------- K1+K2, suite 2, L = 32
// onetime_seed = MMO(x0 || be32 j) over 2 blocks (first key = IV 0x52^16);
// hash_to_scalar = MDC-2(m || x) (48 B -> 4 blocks incl. a full pad block)
// and MDC-2(0x01 || m || x) (49 B -> 4 blocks), 2 AES per block.
template <int T, int E>
__global__ void __launch_bounds__(T) k_hash_s2_l32(const uint4* __restrict__ pay, uint32_t n2,
                                                   uint32_t tpe, const uint4* __restrict__ x0,
                                                   uint32_t* __restrict__ partial,
                                                   uint32_t* __restrict__ etilde,
                                                   const uint32_t* __restrict__ t0g, uint32_t tile0) {
    extern __shared__ uint32_t sT0[];
    __shared__ uint32_t red[(T / 32) * 17];
    load_t0(sT0, t0g);
    SmemT0 t0{sT0, threadIdx.x & 31u};
    const uint32_t tile = tile0 + blockIdx.x;
    const uint32_t ep = tile / tpe, sub = tile - ep * tpe;
    const uint4 xr = __ldg(x0 + ep);
    const uint32_t x0m[4] = {xr.x, xr.y, xr.z, xr.w};
    // MMO first block is x0 under the constant IV key: hoisted per epoch
    uint32_t hpre[4] = {MMO_IV_WORD, MMO_IV_WORD, MMO_IV_WORD, MMO_IV_WORD};
    mmo_step(t0, hpre, x0m);
    uint32_t acc[17];
    acc17_zero(acc);
    const uint32_t jbase = sub * (T * E) + threadIdx.x;
#pragma unroll 1
    for (int i = 0; i < E; i++) {
        const uint32_t j = jbase + i * T;
        if (j < n2) {
            const uint64_t ent = (uint64_t)ep * n2 + j;
            const uint4 a = __ldg(pay + 2 * ent), b = __ldg(pay + 2 * ent + 1);
            const uint32_t m[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            uint32_t limbs[16];
            entry_limbs_s2_l32(t0, hpre, j, m, limbs);
            acc17_add16(acc, limbs);
        }
    }
    block_reduce_acc17(acc, red);
    if (threadIdx.x == 0) store_tile(acc, tpe == 1, ep, tile, partial, etilde);
}

}  // namespace

void launch_hash_s2_l32(const EntryLayout& lay, const TileMap& tm, const uint4* d_x0,
                        uint32_t* d_partial, uint32_t* d_etilde, const uint32_t* d_t0, cudaStream_t s) {
    uint32_t n_tiles = tm.tile_count ? tm.tile_count : tm.n_epochs * tm.tiles_per_epoch;
    if (!n_tiles) return;
    const uint4* pay = reinterpret_cast<const uint4*>(lay.payload);
    size_t smem = kAesSmemWords * sizeof(uint32_t);
    if (tm.tile_entries == 256 * 4) {
        cudaFuncSetAttribute(k_hash_s2_l32<256, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_hash_s2_l32<256, 4><<<n_tiles, 256, smem, s>>>(pay, tm.n2, tm.tiles_per_epoch, d_x0, d_partial, d_etilde, d_t0, tm.tile_begin);
    } else if (tm.tile_entries == 128 * 2) {
        cudaFuncSetAttribute(k_hash_s2_l32<128, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_hash_s2_l32<128, 2><<<n_tiles, 128, smem, s>>>(pay, tm.n2, tm.tiles_per_epoch, d_x0, d_partial, d_etilde, d_t0, tm.tile_begin);
    } else {
        cudaFuncSetAttribute(k_hash_s2_l32<128, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_hash_s2_l32<128, 1><<<n_tiles, 128, smem, s>>>(pay, tm.n2, tm.tiles_per_epoch, d_x0, d_partial, d_etilde, d_t0, tm.tile_begin);
    }
}

}  // namespace poslo_gpu
