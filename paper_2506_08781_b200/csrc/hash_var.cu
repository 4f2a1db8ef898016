// K1+K2 for suite 1 (SHA-256) over VARIABLE-length entries (BASELINE config 4:
// syslog-style 64..1024-byte records), uniform or ragged epochs.
//
// onetime_seed (primitives.cpp:209-223) then H(m||x) and H(0x01||m||x)
// (primitives.cpp:162-176) streamed block by block straight from the packed
// payload: each message word is one funnel-shifted pair of aligned 32-bit
// loads (the entry can start at any byte), so no staging copy is needed;
// only the last one or two blocks (x, 0x80 padding, bit length) take a
// byte-assembled slow path. Work per entry grows with L
// (ceil((L+25)/64) + ceil((L+26)/64) + 1 compressions), so each CTA first
// counting-sorts its tile by block count in shared memory: threads of a warp
// then hash entries of similar length and the warp does not idle on the
// longest one.
#include "entry_hash.cuh"
#include "tile_common.cuh"

namespace poslo_gpu {

namespace {

using namespace tilec;

constexpr int kVarT = 256;        // threads per CTA
constexpr int kVarTile = 1024;    // entries per tile
constexpr int kVarBuckets = 32;   // block-count buckets (clamped)

// Big-endian word at byte offset p of the logical stream
//   [0x01 if tagged] || m (L bytes) || x (16 bytes) || 0x80 || 0.. || bitlen
// where total = message length (L + 16 [+1]) and nb = number of 64-byte blocks.
struct VarStream {
    const uint8_t* m;
    uint32_t L;
    uint32_t tag;       // 0 or 1 (bytes of prefix)
    uint32_t x[4];      // x as big-endian words
    uint64_t total;     // L + 16 + tag
    uint64_t nb;        // blocks

    __device__ __forceinline__ uint32_t m_word_fast(uint32_t q) const {  // bytes m[q..q+3], q+3 < L
        const uintptr_t a = (uintptr_t)(m + q);
        const uint32_t* base = reinterpret_cast<const uint32_t*>(a & ~(uintptr_t)3);
        const uint32_t sh = (uint32_t)(a & 3) * 8;
        uint32_t lo = __ldg(base);
        uint32_t v = sh ? __funnelshift_r(lo, __ldg(base + 1), sh) : lo;
        return bswap32(v);
    }
    __device__ __forceinline__ uint32_t byte_at(uint64_t p) const {
        if (p < tag) return 0x01u;
        uint64_t q = p - tag;
        if (q < L) return m[q];
        q -= L;
        if (q < 16) return (x[q >> 2] >> (24 - 8 * (q & 3))) & 0xffu;
        if (p == total) return 0x80u;
        return 0u;
    }
    __device__ __forceinline__ uint32_t word(uint64_t p) const {
        if (p >= tag && p - tag + 3 < L) return m_word_fast((uint32_t)(p - tag));
        uint32_t w = 0;
#pragma unroll
        for (int i = 0; i < 4; i++) w = (w << 8) | byte_at(p + i);
        return w;
    }
};

__device__ __forceinline__ void sha256_var(const VarStream& s, uint32_t H[8]) {
    sha256_init(H);
    for (uint64_t b = 0; b < s.nb; b++) {
        uint32_t W[16];
        const uint64_t p0 = 64 * b;
        const bool fast = p0 + 64 <= s.tag + s.L && p0 >= s.tag;
        if (fast) {
#pragma unroll
            for (int k = 0; k < 16; k++) W[k] = s.m_word_fast((uint32_t)(p0 - s.tag + 4 * k));
        } else {
#pragma unroll
            for (int k = 0; k < 16; k++) W[k] = s.word(p0 + 4 * k);
        }
        if (b == s.nb - 1) {
            W[14] = (uint32_t)((s.total * 8) >> 32);
            W[15] = (uint32_t)(s.total * 8);
        }
        uint32_t st[8];
#pragma unroll
        for (int i = 0; i < 8; i++) st[i] = H[i];
        sha256_rounds_compact<2>(st, W, 0, pipek_make());
#pragma unroll
        for (int i = 0; i < 8; i++) H[i] += st[i];
    }
}

__device__ __forceinline__ uint32_t nblocks(uint64_t msg_len) { return (uint32_t)((msg_len + 9 + 63) / 64); }

__global__ void __launch_bounds__(kVarT) k_hash_s1_var(EntryLayout lay, TileMap tm,
                                                       const uint4* __restrict__ x0,
                                                       uint32_t* __restrict__ partial) {
    __shared__ uint32_t red[(kVarT / 32) * 17];
    __shared__ uint16_t order[kVarTile];
    __shared__ uint32_t bucket_count[kVarBuckets];
    __shared__ uint32_t bucket_base[kVarBuckets];
    const uint32_t tile = tm.tile_begin + blockIdx.x;
    uint32_t ep, j0, count;
    uint64_t ebase;
    if (tm.tiles) {
        uint4 t = tm.tiles[tile];
        ep = t.x; j0 = t.y; count = t.z;
        ebase = tm.epoch_starts[ep];
    } else {
        ep = tile / tm.tiles_per_epoch;
        const uint32_t sub = tile - ep * tm.tiles_per_epoch;
        j0 = sub * tm.tile_entries;
        count = min(tm.tile_entries, tm.n2 - j0);
        ebase = (uint64_t)ep * tm.n2;
    }
    // counting sort of the tile by block count (longest first)
    if (threadIdx.x < kVarBuckets) bucket_count[threadIdx.x] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < count; i += kVarT) {
        const uint64_t ent = ebase + j0 + i;
        const uint64_t L = lay.offsets ? lay.offsets[ent + 1] - lay.offsets[ent] : lay.entry_len;
        atomicAdd(&bucket_count[min(nblocks(L + 17), (uint32_t)kVarBuckets - 1)], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t acc = 0;
        for (int k = kVarBuckets - 1; k >= 0; k--) {
            bucket_base[k] = acc;
            acc += bucket_count[k];
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < count; i += kVarT) {
        const uint64_t ent = ebase + j0 + i;
        const uint64_t L = lay.offsets ? lay.offsets[ent + 1] - lay.offsets[ent] : lay.entry_len;
        const uint32_t slot = atomicAdd(&bucket_base[min(nblocks(L + 17), (uint32_t)kVarBuckets - 1)], 1u);
        order[slot] = (uint16_t)i;
    }
    __syncthreads();

    const uint4 xr = __ldg(x0 + ep);
    const uint32_t x0w[4] = {bswap32(xr.x), bswap32(xr.y), bswap32(xr.z), bswap32(xr.w)};
    uint32_t pre[8];
    ots_pre(x0w, pre);
    uint32_t acc[17];
    acc17_zero(acc);
    for (uint32_t i = threadIdx.x; i < count; i += kVarT) {
        const uint32_t idx = order[i];
        const uint32_t j = j0 + idx;
        const uint64_t ent = ebase + j;
        const uint8_t* m;
        uint64_t L;
        if (lay.offsets) {
            const uint64_t o0 = lay.offsets[ent];
            m = lay.payload + o0;
            L = lay.offsets[ent + 1] - o0;
        } else {
            m = lay.payload + ent * lay.entry_len;
            L = lay.entry_len;
        }
        uint32_t xw[4];
        ots_finish(x0w, pre, j, xw);
        uint32_t limbs[16], H[8];
        VarStream s1{m, (uint32_t)L, 0u, {xw[0], xw[1], xw[2], xw[3]}, L + 16, nblocks(L + 16)};
        sha256_var(s1, H);
#pragma unroll
        for (int k = 0; k < 8; k++) limbs[15 - k] = H[k];
        VarStream s2{m, (uint32_t)L, 1u, {xw[0], xw[1], xw[2], xw[3]}, L + 17, nblocks(L + 17)};
        sha256_var(s2, H);
#pragma unroll
        for (int k = 0; k < 8; k++) limbs[7 - k] = H[k];
        acc17_add16(acc, limbs);
    }
    block_reduce_acc17(acc, red);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < 17; k++) partial[(size_t)tile * 17 + k] = acc[k];
}

}  // namespace

void launch_hash_s1_var(const EntryLayout& lay, const TileMap& tm, const uint4* d_x0, uint32_t* d_partial,
                        cudaStream_t s) {
    uint32_t n_tiles = tm.tile_count ? tm.tile_count : (tm.tiles ? tm.n_tiles : tm.n_epochs * tm.tiles_per_epoch);
    if (!n_tiles) return;
    k_hash_s1_var<<<n_tiles, kVarT, 0, s>>>(lay, tm, d_x0, d_partial);
}

}  // namespace poslo_gpu
