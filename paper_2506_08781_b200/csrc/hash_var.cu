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
#define POSLO_VAR_FMA 5  // pipe assignment of the SHA rounds (sha256.cuh SHA_RND_SEL)
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
};

// Per-entry, per-stream constants kept in shared memory (one LDS.128 per
// block instead of re-deriving them on the ALU pipe every job): the shared
// address of the stream's word 0 in the slot, the PRMT selector, the index of
// its last block, and its message length in bits (low word; < 2^32 here).
struct StreamDesc {
    uint32_t word_addr, sel, last_b, bits;
};

// Edge block step (b = 0, or a window reaching past the entry): relative
// 32-bit arithmetic on m positions. The window of block b covers m positions
// [64b - d0, 64b - d0 + 96) (d0 = slot byte of m[0] in block 0, 4..19);
// chunk c is loaded only if it holds a byte of the entry.
__device__ __forceinline__ void stage_window(const VarEntry& v, uintptr_t base0, uint32_t d0, uint32_t b) {
    const int r0 = (int)(64 * b) - (int)d0;  // m position of slot byte 0
    const uint4* src = reinterpret_cast<const uint4*>(base0 + 64ull * b);
    uint4* s4 = reinterpret_cast<uint4*>(v.slot);
#pragma unroll
    for (int c = 0; c < 6; c++) {
        const int rc = r0 + 16 * c;
        uint4 q = make_uint4(0, 0, 0, 0);
        // rc > -16 can only fail for chunk 0 of block 0 (d0 >= 16)
        if (rc < (int)v.L && (c > 0 || rc > -16)) q = __ldg(src + c);
        s4[c] = q;
    }
    const int off = -r0;  // slot byte of m position 0 (negative for b > 0)
    if (b == 0) reinterpret_cast<uint8_t*>(v.slot)[off - 1] = 0x01;  // tag byte of the second stream
    // Suffix x || 0x80 at m positions L .. L+16. Only those bytes need writing:
    // a chunk holding position >= L+16 starts past L and was not loaded
    // (zero), so the neighbour bytes a loaded chunk carries past the entry
    // all lie in L .. L+14. Five word writes at the suffix start's word
    // alignment, funnel-shifted out of the slot tail E = [0, x0..x3, 0x80, 0].
    const int sp = off + (int)v.L;  // slot byte of position L
    if (sp < 4 * 24 && sp + 17 > 0) {
        const uint32_t c0 = (uint32_t)sp & 3;
        const int w0 = sp >> 2;
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

// Interior block step: the whole window lies inside the entry (b >= 1 and
// 64b + 96 - d0 <= L), so it is six unconditional 16-byte loads at
// base0 + 64b with nothing to patch (no tag, no suffix).
__device__ __forceinline__ void stage_interior(const VarEntry& v, uintptr_t base0, uint32_t b) {
    const uint4* src = reinterpret_cast<const uint4*>(base0 + 64ull * b);
    uint4* s4 = reinterpret_cast<uint4*>(v.slot);
#pragma unroll
    for (int c = 0; c < 6; c++) s4[c] = __ldg(src + c);
}

// PRMT selector that funnels bytes r..r+3 of (lo, hi) into one big-endian word
__device__ __forceinline__ uint32_t prmt_sel(uint32_t r) { return (r + 3) | (r + 2) << 4 | (r + 1) << 8 | r << 12; }

// Message words of one stream's block: slot words from word_addr funnelled
// by sel. The window of block b starts at base0 + 64b, so a stream's word 0
// sits at the same slot byte d0 - tag in every block: per-entry constants.
__device__ __forceinline__ void load_block(uint32_t word_addr, uint32_t sel, uint32_t W[16]) {
    uint32_t w[17];
#define POSLO_LDS_W(k) asm volatile("ld.shared.u32 %0, [%1+" #k "];" : "=r"(w[(k) / 4]) : "r"(word_addr))
    POSLO_LDS_W(0); POSLO_LDS_W(4); POSLO_LDS_W(8); POSLO_LDS_W(12); POSLO_LDS_W(16); POSLO_LDS_W(20);
    POSLO_LDS_W(24); POSLO_LDS_W(28); POSLO_LDS_W(32); POSLO_LDS_W(36); POSLO_LDS_W(40); POSLO_LDS_W(44);
    POSLO_LDS_W(48); POSLO_LDS_W(52); POSLO_LDS_W(56); POSLO_LDS_W(60); POSLO_LDS_W(64);
#undef POSLO_LDS_W
#pragma unroll
    for (int k = 0; k < 16; k++) W[k] = __byte_perm(w[k], w[k + 1], sel);
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
                                                          uint32_t* __restrict__ partial, const PipeK pk_in) {
    const PipeK pk = POSLO_VAR_FMA == 5 ? pipek_vec(pk_in) : pk_in;
    __shared__ uint32_t red[(kVarT / 32) * 17];
    __shared__ uint16_t order[kVarTile];
    __shared__ uint32_t bucket_count[kVarBuckets];
    __shared__ uint32_t bucket_base[kVarBuckets];
    __shared__ __align__(16) uint32_t slots[kVarT * kSlotWords];
    __shared__ uint32_t s_acc[18 * kVarT];  // rows 0..8: sum of H1 digests, 9..17: sum of H0 digests
    __shared__ uint32_t s_pre[8], s_x0w[4];
    __shared__ uint4 s_desc[2 * kVarT];  // StreamDesc of this thread's entry, streams 0 and 1
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
    // Sorted position of this thread's entry in iteration it: the tile's 128
    // positions of an iteration go to the 4 warps in a rotating order, so every
    // warp takes each rank (longest .. shortest quarter) equally often and the
    // warps of a CTA finish together at the reduction barrier (a fixed order
    // gave warp 0 the longest quarter every time).
    const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#pragma unroll 1
    for (uint32_t base = 0, it = 0; base < count; base += kVarT, it++) {
        const uint32_t i = base + (((warp + it) & (kVarT / 32 - 1)) << 5) + lane;
        if (i >= count) continue;
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
        const uintptr_t base0 = ((uintptr_t)v.m - 4) & ~(uintptr_t)15;  // window of block 0
        const uint32_t d0 = (uint32_t)((uintptr_t)v.m - base0);          // slot byte of m[0]: 4..19
        const uint32_t fast_hi = v.L + d0 >= 96 ? (v.L + d0 - 96) >> 6 : 0u;  // interior blocks 1..fast_hi
        // One job loop shares ONE copy of the compression code (the kernel
        // stays inside the instruction cache): job 0 is x = onetime_seed(x0, j)
        // (resumed at round 4), then block b of stream 0 and of stream 1
        // alternate; Hc/Ho are the current/other stream's chaining values,
        // swapped after every job so both stay in registers.
        const uint32_t nb0 = nblocks(L + 16), nb1 = nblocks(L + 17);
        {
            const uint32_t slot_addr = (uint32_t)__cvta_generic_to_shared(v.slot);
            s_desc[2 * threadIdx.x] = make_uint4(slot_addr + (d0 & ~3u), prmt_sel(d0 & 3), nb0 - 1,
                                                 (uint32_t)((L + 16) * 8));
            s_desc[2 * threadIdx.x + 1] = make_uint4(slot_addr + ((d0 - 1) & ~3u), prmt_sel((d0 - 1) & 3),
                                                     nb1 - 1, (uint32_t)((L + 17) * 8));
        }
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
                if (!stream) {
                    if (b - 1u < fast_hi) stage_interior(v, base0, b);
                    else stage_window(v, base0, d0, b);
                }
                const uint4 sd = s_desc[2 * threadIdx.x + stream];
                active = b <= sd.z;  // stream 0 may end one block before stream 1
                if (active) {
                    load_block(sd.x, sd.y, W);
                    if (b == sd.z) {  // entries < 512 MiB: the bit length fits one word
                        W[14] = 0;
                        W[15] = sd.w;
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
