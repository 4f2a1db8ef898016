// Helpers shared by the hashing kernels (verify_kernels.cu, hash_s1.cu,
// hash_s2.cu): AES table staging, CTA-wide 17-limb reduction, tile stores.
#pragma once
#include "aes128.cuh"
#include "poslo_internal.h"
#include "scalar.cuh"
#include "sha256.cuh"

namespace poslo_gpu {
namespace tilec {

constexpr int kAesSmemWords = 256 * 32;  // T0 replicated per bank

struct SmemT0 {
    const uint32_t* s;
    uint32_t lane;
    PD uint32_t operator()(uint32_t x) const { return s[(x << 5) | lane]; }
    // T0[byte k of w]: one PRMT (byte extract, ALU) + one IMAD (row address,
    // FMA pipe) + the LDS, instead of shift/mask/or on the ALU pipe
    PD uint32_t lk(uint32_t w, int k) const {
        const uint32_t x = __byte_perm(w, 0u, 0x4440u + (uint32_t)k);
        return s[x * 32u + lane];
    }
};

static __device__ __forceinline__ void load_t0(uint32_t* sT0, const uint32_t* t0g) {
    for (int i = threadIdx.x; i < kAesSmemWords; i += blockDim.x) sT0[i] = __ldg(t0g + (i >> 5));
    __syncthreads();
}

static __device__ __forceinline__ void err_min(unsigned long long* err, unsigned long long key) {
    if (err) atomicMin(err, key);
}

// Sum of the 17-limb accumulators of all threads of the CTA; result valid
// in thread 0. red: (blockDim.x / 32) * 17 words of shared memory.
static __device__ __forceinline__ void block_reduce_acc17(uint32_t acc[17], uint32_t* red) {
    const unsigned full = 0xffffffffu;
#pragma unroll
    for (int off = 16; off >= 1; off >>= 1) {
        uint32_t v[17];
#pragma unroll
        for (int k = 0; k < 17; k++) v[k] = __shfl_down_sync(full, acc[k], off);
        acc17_add17(acc, v);
    }
    int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    if (lane == 0)
#pragma unroll
        for (int k = 0; k < 17; k++) red[warp * 17 + k] = acc[k];
    __syncthreads();
    if (warp == 0) {
#pragma unroll
        for (int k = 0; k < 17; k++) acc[k] = lane < nw ? red[lane * 17 + k] : 0u;
#pragma unroll
        for (int off = 16; off >= 1; off >>= 1) {
            uint32_t v[17];
#pragma unroll
            for (int k = 0; k < 17; k++) v[k] = __shfl_down_sync(full, acc[k], off);
            acc17_add17(acc, v);
        }
    }
}

// Writes a finished tile: the epoch's e~ (mod l) when the tile is the whole
// epoch, else the raw 17-limb partial.
static __device__ __forceinline__ void store_tile(const uint32_t acc[17], bool whole_epoch, uint32_t ep,
                                           uint32_t tile, uint32_t* partial, uint32_t* etilde) {
    if (whole_epoch) {
        uint32_t e[8];
        sc_reduce_limbs(acc, 17, e);
#pragma unroll
        for (int k = 0; k < 8; k++) etilde[(size_t)ep * 8 + k] = e[k];
    } else {
#pragma unroll
        for (int k = 0; k < 17; k++) partial[(size_t)tile * 17 + k] = acc[k];
    }
}

}  // namespace tilec
}  // namespace poslo_gpu
