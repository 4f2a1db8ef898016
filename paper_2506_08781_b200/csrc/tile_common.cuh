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
    PD uint32_t lkr(uint32_t w, int k, int r) const { return rotl32(lk(w, k), 8 * r); }
};

// T0..T3 all stored, each replicated per bank (4 x 32 KiB): the rotations of
// the round function become table selects (no ALU work), for kernels that
// can spend 128 KiB of shared memory on them (hash_s2.cu). Layout: row x of
// 256 bytes holds [T_a lane 0..31 | T_b lane 0..31], (T_a, T_b) = (T0, T1) in
// the first 64 KiB and (T2, T3) in the second. The tables start at a 64 KiB
// aligned shared-window address T, so the shared address of T_r[x] for this
// lane is T | x << 8 | lane << 2 (+ 128 for odd r, + 64 KiB for r >= 2):
// ONE PRMT builds it (byte k of the state word into byte 1, lane << 2 and T's
// byte 2 from a per-thread constant) and the table select is the LDS
// immediate. A lookup is PRMT + LDS, nothing else.
constexpr int kAes4SmemWords = 4 * kAesSmemWords;
constexpr uint32_t kAes4Align = 65536;
constexpr size_t kAes4DynBytes = kAes4Align + kAes4SmemWords * sizeof(uint32_t);  // + alignment slack

struct SmemT4 {
    uint32_t key;  // T | lane << 2 (bytes 4..7 of the PRMT)
    template <int R>
    PD uint32_t at(uint32_t w, int k) const {
        const uint32_t a = __byte_perm(w, key, 0x7604u | ((uint32_t)k << 4));
        uint32_t v;
        asm("ld.shared.u32 %0, [%1+%2];" : "=r"(v) : "r"(a), "n"((R >> 1) * 65536 + (R & 1) * 128));
        return v;
    }
    PD uint32_t operator()(uint32_t x) const { return at<0>(x, 0); }
    PD uint32_t lk(uint32_t w, int k) const { return at<0>(w, k); }
    PD uint32_t lkr(uint32_t w, int k, int r) const {
        return r == 1 ? at<1>(w, k) : r == 2 ? at<2>(w, k) : r == 3 ? at<3>(w, k) : at<0>(w, k);
    }
};

// Fills the four tables in the dynamic shared memory `dyn` (kAes4DynBytes)
// and returns this thread's SmemT4.
static __device__ __forceinline__ SmemT4 load_t4(uint8_t* dyn, const uint32_t* t0g) {
    const uint32_t base = (uint32_t)__cvta_generic_to_shared(dyn);
    const uint32_t T = (base + kAes4Align - 1) & ~(kAes4Align - 1);
    uint32_t* sT = reinterpret_cast<uint32_t*>(dyn + (T - base));
    for (int i = threadIdx.x; i < kAesSmemWords; i += blockDim.x) {
        const uint32_t x = (uint32_t)i >> 5, lane = (uint32_t)i & 31u;
        const uint32_t v = __ldg(t0g + x);
#pragma unroll
        for (int r = 0; r < 4; r++) sT[(r >> 1) * 16384 + x * 64 + (r & 1) * 32 + lane] = rotl32(v, 8 * r);
    }
    __syncthreads();
    return SmemT4{T | (threadIdx.x & 31u) << 2};
}

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
