// K1+K2 fast path for suite 2 (MMO/MDC-2 over AES-128) with 32-byte entries, uniform epochs.
#include <algorithm>
#include <cstdlib>

#include "entry_hash.cuh"
#include "tile_common.cuh"

namespace poslo_gpu {

namespace {

using namespace tilec;

// ---------------------------------------------------------------- K1+K2, suite 2, L = 32
// onetime_seed = MMO(x0 || be32 j) over 2 blocks (first key = IV 0x52^16);
// hash_to_scalar = MDC-2(m || x) (48 B -> 4 blocks incl. a full pad block)
// and MDC-2(0x01 || m || x) (49 B -> 4 blocks), 2 AES per block: 17 AES-128
// with a fresh key schedule each, i.e. 3400 data-dependent T-table lookups
// per entry (16 per round + 4 for the key schedule, x 10 rounds).
//
// The lookups are the bound (one 32-bit LDS lane each), so the kernel is
// shaped around the table: persistent, one 1024-thread CTA per SM holding
// all four T-tables (T_r = rotl(T0, 8r), each replicated per bank: 128 KiB,
// filled ONCE per SM rather than once per tile), and each warp works through
// whole tiles on its own (lane-private entries, warp-shuffle reduction, no
// CTA barrier after the fill). Storing T1..T3 turns the 12 rotations of a
// round into table selects, taking them off the ALU pipe (the co-bound).
template <int kS2Threads>
__global__ void __launch_bounds__(kS2Threads, 1) k_hash_s2_p(const uint4* __restrict__ pay, uint32_t n2,
                                                             uint32_t tpe, uint32_t tile_entries,
                                                             const uint4* __restrict__ x0,
                                                             uint32_t* __restrict__ partial,
                                                             uint32_t* __restrict__ etilde,
                                                             const uint32_t* __restrict__ t0g, uint32_t tile0,
                                                             uint32_t n_tiles) {
    extern __shared__ __align__(16) uint8_t dyn[];
    const SmemT4 t4 = load_t4(dyn, t0g);
    const uint32_t lane = threadIdx.x & 31u;
    const uint32_t warps = gridDim.x * (kS2Threads / 32);
#pragma unroll 1
    for (uint32_t t = blockIdx.x * (kS2Threads / 32) + (threadIdx.x >> 5); t < n_tiles; t += warps) {
        const uint32_t tile = tile0 + t;
        const uint32_t ep = tile / tpe, sub = tile - ep * tpe;
        const uint4 xr = __ldg(x0 + ep);
        const uint32_t x0m[4] = {xr.x, xr.y, xr.z, xr.w};
        // MMO first block is x0 under the constant IV key: once per lane per tile
        uint32_t hpre[4] = {MMO_IV_WORD, MMO_IV_WORD, MMO_IV_WORD, MMO_IV_WORD};
        mmo_step(t4, hpre, x0m);
        uint32_t acc[17];
        acc17_zero(acc);
        const uint32_t j_end = min(n2, (sub + 1) * tile_entries);
#pragma unroll 1
        for (uint32_t j = sub * tile_entries + lane; j < j_end; j += 32) {
            const uint64_t ent = (uint64_t)ep * n2 + j;
            const uint4 a = __ldg(pay + 2 * ent), b = __ldg(pay + 2 * ent + 1);
            const uint32_t m[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
            uint32_t limbs[16];
            entry_limbs_s2_l32(t4, hpre, j, m, limbs);
            acc17_add16(acc, limbs);
        }
        const unsigned full = 0xffffffffu;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            uint32_t v[17];
#pragma unroll
            for (int k = 0; k < 17; k++) v[k] = __shfl_down_sync(full, acc[k], off);
            acc17_add17(acc, v);
        }
        if (lane == 0) store_tile(acc, tpe == 1, ep, tile, partial, etilde);
    }
}

}  // namespace

void launch_hash_s2_l32(const EntryLayout& lay, const TileMap& tm, const uint4* d_x0,
                        uint32_t* d_partial, uint32_t* d_etilde, const uint32_t* d_t0, cudaStream_t s) {
    uint32_t n_tiles = tm.tile_count ? tm.tile_count : tm.n_epochs * tm.tiles_per_epoch;
    if (!n_tiles) return;
    struct Cfg {
        int sms, threads;
    };
    static const Cfg cfg = [] {  // once per process (thread-safe static init)
        int dev = 0, sms = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const char* e = std::getenv("POSLO_S2_THREADS");  // tuning knob: 256 / 384 / 512 / 768 / 1024
        const size_t smem = kAes4DynBytes;
        cudaFuncSetAttribute(k_hash_s2_p<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_hash_s2_p<384>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_hash_s2_p<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_hash_s2_p<768>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        cudaFuncSetAttribute(k_hash_s2_p<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        return Cfg{sms, e ? std::atoi(e) : 512};
    }();
    const int sms = cfg.sms, threads = cfg.threads;
    const size_t smem = kAes4DynBytes;
    // one CTA per SM (128 KiB of tables), fewer when there are fewer tiles than warps
    const uint32_t warps_per_cta = (uint32_t)threads / 32;
    const uint32_t grid = std::min<uint32_t>((uint32_t)sms, (n_tiles + warps_per_cta - 1) / warps_per_cta);
    const uint4* pay = reinterpret_cast<const uint4*>(lay.payload);
#define S2_LAUNCH(T)                                                                                        \
    k_hash_s2_p<T><<<grid, T, smem, s>>>(pay, tm.n2, tm.tiles_per_epoch, tm.tile_entries, d_x0, d_partial, \
                                         d_etilde, d_t0, tm.tile_begin, n_tiles)
    if (threads == 256)
        S2_LAUNCH(256);
    else if (threads == 384)
        S2_LAUNCH(384);
    else if (threads == 512)
        S2_LAUNCH(512);
    else if (threads == 768)
        S2_LAUNCH(768);
    else
        S2_LAUNCH(1024);
#undef S2_LAUNCH
}

}  // namespace poslo_gpu
