// K1+K2 for suite 1 (SHA-256) over VARIABLE-length entries (BASELINE config 4:
// syslog-style 64..1024-byte records), uniform or ragged epochs.
//
// onetime_seed (primitives.cpp:209-223) then H(m||x) and H(0x01||m||x)
// (primitives.cpp:162-176), the two hash streams advanced block by block in
// lockstep from one staged 72-byte window per block step (see stage_window):
// 16-byte vector loads instead of per-word gathers, so the L1 sees 6 wide
// requests per block pair rather than 64 narrow ones. Work per entry grows with L
// (ceil((L+25)/64) + ceil((L+26)/64) + 1 compressions), so each CTA first
// counting-sorts its tile by block count in shared memory: threads of a warp
// then hash entries of similar length and the warp does not idle on the
// longest one.
#include "entry_hash.cuh"
#include "tile_common.cuh"

#ifndef POSLO_VAR_MINB
#define POSLO_VAR_MINB 6  // min CTAs/SM of k_hash_s1_var (register cap 65536 / (128 x MINB))
#endif
#ifndef POSLO_VAR_FMA
#define POSLO_VAR_FMA 2  // pipe assignment of the SHA rounds (sha256.cuh SHA_RND_SEL)
#endif

namespace poslo_gpu {

namespace {

using namespace tilec;

constexpr int kVarT = 128;        // threads per CTA
constexpr int kVarTile = 1024;    // entries per tile
constexpr int kVarBuckets = 32;   // block-count buckets (clamped)

// per-thread staging slot: 24-word window + E = [0, x (4 words), 0x80, 0];
// 36 words keeps the 16-byte alignment of the vector stores and spreads the
// same-index LDS of a warp over 8 banks (a stride of 32 would put all 32
// lanes on one bank)
constexpr int kSlotWords = 36;
constexpr uint32_t kNoEntry = 0xffffffffu;

__device__ __forceinline__ uint32_t nblocks(uint64_t msg_len) { return (uint32_t)((msg_len + 9 + 63) / 64); }

// Staging of one 64-byte block step. Both hash streams of an entry read the
// same bytes: H(m || x) at stream offset p reads m[p], H(0x01 || m || x)
// reads m[p - 1], and x || 0x80 || 0.. follows m in both. For block b a
// thread stages the window of m positions [64b - 4, 64b + 68) in its private
// shared-memory slot: six 16-byte aligned vector loads (only chunks that hold
// bytes of this entry are read), then the bytes at positions >= L are
// overwritten with x || 0x80 || 0.. and, for b = 0, position -1 with the
// 0x01 tag. Message words are then one LDS + one PRMT each (the PRMT does
// both the byte-misaligned funnel and the big-endian swap).
struct VarEntry {
    const uint8_t* m;  // entry bytes
    uint32_t L;
    uint32_t* slot;    // kSlotWords words of shared memory
    uintptr_t base;    // 16-byte aligned global address of slot word 0 (window start)
};

__device__ __forceinline__ void stage_window(VarEntry& v, uint32_t b) {
    const uintptr_t a = (uintptr_t)v.m;
    const uintptr_t lo = a + 64ull * b - 4;
    v.base = lo & ~(uintptr_t)15;
    uint4* s4 = reinterpret_cast<uint4*>(v.slot);
#pragma unroll
    for (int c = 0; c < 6; c++) {
        const uintptr_t cs = v.base + 16 * c;
        uint4 q = make_uint4(0, 0, 0, 0);
        if (cs < a + v.L && cs + 16 > a) q = __ldg(reinterpret_cast<const uint4*>(cs));
        s4[c] = q;
    }
    const int64_t off = (int64_t)(a - v.base);  // slot byte of m position 0 (negative for b > 0)
    if (b == 0) reinterpret_cast<uint8_t*>(v.slot)[off - 1] = 0x01;  // tag byte of the second stream
    // Suffix x || 0x80 at m positions L .. L+16. Only those bytes need writing:
    // a chunk holding position >= L+16 starts past L and was not loaded
    // (zero), so the neighbour bytes a loaded chunk carries past the entry
    // all lie in L .. L+14. Five word writes at the suffix start's word
    // alignment, funnel-shifted out of the slot tail E = [0, x0..x3, 0x80, 0].
    const int64_t sp = off + (int64_t)v.L;  // slot byte of position L
    if (sp < 4 * 24 && sp + 17 > 0) {
        const uint32_t c0 = (uint32_t)sp & 3;
        const int w0 = (int)(sp >> 2);
        const uint32_t* E = v.slot + 24 + (c0 == 0);
        const uint32_t sh = ((4 - c0) & 3) * 8;
        const uint32_t keep = c0 ? (1u << (8 * c0)) - 1 : 0u;  // bytes of word w0 before position L
#pragma unroll
        for (int i = 0; i < 5; i++) {
            const int wi = w0 + i;
            if (wi >= 0 && wi < 24) {
                const uint32_t sw = __funnelshift_r(E[i], E[i + 1], sh);
                v.slot[wi] = i == 0 ? (v.slot[wi] & keep) | sw : sw;
            }
        }
    }
}

// Message words of block b of one stream (tag = 0 or 1 prefix bytes).
__device__ __forceinline__ void load_block(const VarEntry& v, uint32_t b, uint32_t tag, uint32_t W[16]) {
    const uint32_t d = (uint32_t)((uintptr_t)v.m + 64ull * b - tag - v.base);  // slot byte of word 0
    const uint32_t r = d & 3;
    const uint32_t sel = (r + 3) | (r + 2) << 4 | (r + 1) << 8 | r << 12;
    const uint32_t* s = v.slot + (d >> 2);
    uint32_t lo = s[0];
#pragma unroll
    for (int k = 0; k < 16; k++) {
        const uint32_t hi = s[k + 1];
        W[k] = __byte_perm(lo, hi, sel);
        lo = hi;
    }
}

__device__ __forceinline__ void compress_into(uint32_t H[8], uint32_t W[16], const PipeK& pk) {
    uint32_t st[8];
#pragma unroll
    for (int i = 0; i < 8; i++) st[i] = H[i];
    sha256_rounds_compact<POSLO_VAR_FMA>(st, W, 0, pk);
#pragma unroll
    for (int i = 0; i < 8; i++) H[i] += st[i];
}

PD void smem_acc9_add8v(uint32_t* s, int stride, const uint32_t v[8]) {
    uint32_t a[9];
#pragma unroll
    for (int k = 0; k < 9; k++) a[k] = s[k * stride];
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
    for (int k = 0; k < 9; k++) s[k * stride] = a[k];
}

__global__ void __launch_bounds__(kVarT, POSLO_VAR_MINB) k_hash_s1_var(EntryLayout lay, TileMap tm,
                                                          const uint4* __restrict__ x0,
                                                          uint32_t* __restrict__ partial, const PipeK pk) {
    __shared__ uint32_t red[(kVarT / 32) * 17];
    __shared__ uint16_t order[kVarTile];
    __shared__ uint32_t bucket_count[kVarBuckets];
    __shared__ uint32_t bucket_base[kVarBuckets];
    __shared__ __align__(16) uint32_t slots[kVarT * kSlotWords];
    __shared__ uint32_t s_acc[18 * kVarT];  // rows 0..8: sum of H1 digests, 9..17: sum of H0 digests
    __shared__ uint32_t s_pre[8], s_x0w[4];
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
    // counting sort of the tile by block count (longest first): the lanes of
    // a warp then run the same number of block steps
    if (threadIdx.x < kVarBuckets) bucket_count[threadIdx.x] = 0;
    if (threadIdx.x == 0) {
        const uint4 xr = __ldg(x0 + ep);
        const uint32_t x0w[4] = {bswap32(xr.x), bswap32(xr.y), bswap32(xr.z), bswap32(xr.w)};
        uint32_t pre[8];
        ots_pre(x0w, pre);
#pragma unroll
        for (int k = 0; k < 8; k++) s_pre[k] = pre[k];
#pragma unroll
        for (int k = 0; k < 4; k++) s_x0w[k] = x0w[k];
    }
    uint32_t* acc = s_acc + threadIdx.x;
#pragma unroll
    for (int k = 0; k < 18; k++) acc[k * kVarT] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < count; i += kVarT) {
        const uint64_t ent = ebase + j0 + i;
        const uint64_t L = lay.offsets ? lay.offsets[ent + 1] - lay.offsets[ent] - lay.header : lay.entry_len;
        atomicAdd(&bucket_count[min(nblocks(L + 17), (uint32_t)kVarBuckets - 1)], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t a = 0;
        for (int k = kVarBuckets - 1; k >= 0; k--) {
            bucket_base[k] = a;
            a += bucket_count[k];
        }
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < count; i += kVarT) {
        const uint64_t ent = ebase + j0 + i;
        const uint64_t L = lay.offsets ? lay.offsets[ent + 1] - lay.offsets[ent] - lay.header : lay.entry_len;
        const uint32_t slot = atomicAdd(&bucket_base[min(nblocks(L + 17), (uint32_t)kVarBuckets - 1)], 1u);
        order[slot] = (uint16_t)i;
    }
    __syncthreads();

    VarEntry v;
    v.slot = slots + threadIdx.x * kSlotWords;
    v.slot[24] = 0;
    v.slot[29] = 0x80u;
    v.slot[30] = 0;
#pragma unroll 1
    for (uint32_t i = threadIdx.x; i < count; i += kVarT) {
        const uint32_t j = j0 + order[i];
        const uint64_t ent = ebase + j;
        uint64_t L;
        if (lay.offsets) {
            const uint64_t o0 = lay.offsets[ent] + lay.header;
            v.m = lay.payload + o0;
            L = lay.offsets[ent + 1] - o0;
        } else {
            v.m = lay.payload + ent * lay.entry_len;
            L = lay.entry_len;
        }
        v.L = (uint32_t)L;
        // One job loop shares ONE copy of the compression code (the kernel
        // stays inside the instruction cache): job 0 is x = onetime_seed(x0, j)
        // (resumed at round 4), then block b of stream 0 and of stream 1
        // alternate; Hc/Ho are the current/other stream's chaining values,
        // swapped after every job so both stay in registers.
        const uint32_t nb0 = nblocks(L + 16), nb1 = nblocks(L + 17);
        uint32_t Hc[8], Ho[8];
        sha256_init(Hc);
        sha256_init(Ho);
#pragma unroll 1
        for (uint32_t job = 0; job <= 2 * nb1; job++) {
            uint32_t W[16], st[8];
            int r0 = 0;
            bool active = true;
            if (job == 0) {
#pragma unroll
                for (int k = 0; k < 4; k++) W[k] = s_x0w[k];
                W[4] = j;
                W[5] = 0x80000000u;
#pragma unroll
                for (int k = 6; k < 15; k++) W[k] = 0;
                W[15] = 160u;
#pragma unroll
                for (int k = 0; k < 8; k++) st[k] = s_pre[k];
                r0 = 4;
            } else {
                const uint32_t b = (job - 1) >> 1, stream = (job - 1) & 1;
                if (!stream) stage_window(v, b);
                active = stream || b < nb0;
                if (active) {
                    load_block(v, b, stream, W);
                    const uint32_t nb = stream ? nb1 : nb0;
                    if (b == nb - 1) {
                        const uint64_t bits = (L + 16 + stream) * 8;
                        W[14] = (uint32_t)(bits >> 32);
                        W[15] = (uint32_t)bits;
                    }
#pragma unroll
                    for (int k = 0; k < 8; k++) st[k] = Hc[k];
                } else {  // stream 0 ended one block earlier (L + 25 = 0 mod 64): add nothing
#pragma unroll
                    for (int k = 0; k < 8; k++) st[k] = 0;
                }
            }
            if (active) sha256_rounds_compact<POSLO_VAR_FMA>(st, W, r0, pk);
            if (job == 0) {  // x kept in the slot tail (bytes in stream order) for the suffix writes
                const uint32_t iv[4] = {SHA_IV0, SHA_IV1, SHA_IV2, SHA_IV3};
#pragma unroll
                for (int k = 0; k < 4; k++) v.slot[25 + k] = bswap32(st[k] + iv[k]);
                continue;
            }
#pragma unroll
            for (int k = 0; k < 8; k++) {
                const uint32_t c = Hc[k] + st[k];
                Hc[k] = Ho[k];
                Ho[k] = c;
            }
        }
        // an even number of swaps: Hc is stream 0 (H0), Ho stream 1 (H1)
        uint32_t* H0 = Hc;
        uint32_t* H1 = Ho;
        // H0 is the high half of the 512-bit wide value: digest word k is limb 7 - k of its half
        uint32_t d[8];
#pragma unroll
        for (int k = 0; k < 8; k++) d[7 - k] = H0[k];
        smem_acc9_add8v(acc + 9 * kVarT, kVarT, d);
#pragma unroll
        for (int k = 0; k < 8; k++) d[7 - k] = H1[k];
        smem_acc9_add8v(acc, kVarT, d);
    }
    uint32_t a17[17];
#pragma unroll
    for (int k = 0; k < 8; k++) a17[k] = acc[k * kVarT];
    {
        uint32_t lo8 = acc[8 * kVarT], hi[9];
#pragma unroll
        for (int k = 0; k < 9; k++) hi[k] = acc[(9 + k) * kVarT];
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
    block_reduce_acc17(a17, red);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < 17; k++) partial[(size_t)tile * 17 + k] = a17[k];
}

}  // namespace

void launch_hash_s1_var(const EntryLayout& lay, const TileMap& tm, const uint4* d_x0, uint32_t* d_partial,
                        cudaStream_t s) {
    uint32_t n_tiles = tm.tile_count ? tm.tile_count : (tm.tiles ? tm.n_tiles : tm.n_epochs * tm.tiles_per_epoch);
    if (!n_tiles) return;
    k_hash_s1_var<<<n_tiles, kVarT, 0, s>>>(lay, tm, d_x0, d_partial, pipek_make());
}

}  // namespace poslo_gpu
