// Stages 0-2 of the batch verifier on sm_100a:
//   K0 seed_derive   sr -> sc -> prf      (seed_manager.cpp:71-85, :5-16; primitives.cpp:113-127)
//   K1 hash          onetime_seed + hash_to_scalar (primitives.cpp:149-223)
//   K2 segmented sum Scalar::add folds    (batch_verify.cpp:37-42, :84-85; distiller.cpp:160-176)
// K1 and the entry->epoch level of K2 are one fused kernel: each CTA hashes a
// tile of one epoch, keeps the raw 512-bit digests in a 17-limb per-thread
// accumulator (deferred reduction, see scalar.cuh), reduces across the CTA
// with warp shuffles + shared memory, and reduces mod l once per epoch.
#include "../../include/poslo_synth.h"
#include "entry_hash.cuh"
#include "tile_common.cuh"

namespace poslo_gpu {

namespace {

using namespace tilec;

// ---------------------------------------------------------------- K0
// sr for one queried epoch q: scan from the top of the stack
// (seed_manager.cpp:74-84); returns the covering node index or -1.
__device__ __forceinline__ int ds_cover(const DsParam& ds, uint32_t q) {
    for (int c = ds.count - 1; c >= 0; c--) {
        const DsNode& nd = ds.nodes[c];
        uint64_t lo = (uint64_t)nd.index << nd.depth;
        uint64_t hi = (uint64_t)(uint32_t)(nd.index + 1u) << nd.depth;
        if (q >= hi && c == ds.count - 1) return -1;
        if (q >= lo && q < hi) return c;
    }
    return -1;
}

// Walks `steps` levels down from x along the bits of rel (sc, :5-16).
template <class T0>
__device__ __forceinline__ void ds_walk(int suite, const T0& t0, uint32_t x[4], uint32_t rel, int steps) {
    for (int j = steps - 1; j >= 0; j--) prf_dev(suite, t0, x, (rel >> j) & 1);
}

// K0: one thread per group of G = 8 queried epochs. When the group is 8
// consecutive, 8-aligned epochs under one ds node of depth >= 3 (the dense
// case: every full verification), the thread walks to their common
// depth-3 ancestor once and expands its 8 leaves in a depth-first order:
// (D - 3) + 14 PRFs per 8 epochs instead of 8 * D. Otherwise each epoch of
// the group is walked on its own, exactly as sr does.
constexpr int kSeedGroup = 8;

__global__ void k_seed_derive(int suite, DsParam ds, const uint32_t* __restrict__ epochs_in, uint32_t epoch0,
                              uint32_t n, uint4* __restrict__ x0, unsigned long long* err,
                              const uint32_t* __restrict__ t0g) {
    // epochs_in == nullptr: the queried epochs are epoch0, epoch0 + 1, ... (no list upload)
    auto epochs = [&](uint32_t k) { return epochs_in ? epochs_in[k] : epoch0 + k; };
    extern __shared__ uint32_t sT0[];
    if (suite != 1) load_t0(sT0, t0g);
    SmemT0 t0{sT0, threadIdx.x & 31u};
    const uint32_t k0 = (blockIdx.x * blockDim.x + threadIdx.x) * kSeedGroup;
    if (k0 >= n) return;
    const uint32_t q0 = epochs(k0);
    bool dense = (q0 % kSeedGroup) == 0 && k0 + kSeedGroup <= n;
    int c0 = ds_cover(ds, q0);
    if (dense && c0 >= 0 && ds.nodes[c0].depth >= 3) {
#pragma unroll
        for (int i = 1; i < kSeedGroup; i++) dense = dense && epochs(k0 + i) == q0 + i;
    } else {
        dense = false;
    }
    if (dense) {
        const DsNode& nd = ds.nodes[c0];
        uint32_t x[4] = {nd.value[0], nd.value[1], nd.value[2], nd.value[3]};
        const uint32_t rel = q0 - (uint32_t)((uint64_t)nd.index << nd.depth);
        ds_walk(suite, t0, x, rel >> 3, (int)nd.depth - 3);
        for (int a = 0; a < 2; a++) {
            uint32_t x1[4] = {x[0], x[1], x[2], x[3]};
            prf_dev(suite, t0, x1, a);
            for (int b = 0; b < 2; b++) {
                uint32_t x2[4] = {x1[0], x1[1], x1[2], x1[3]};
                prf_dev(suite, t0, x2, b);
                for (int c = 0; c < 2; c++) {
                    uint32_t x3[4] = {x2[0], x2[1], x2[2], x2[3]};
                    prf_dev(suite, t0, x3, c);
                    x0[k0 + 4 * a + 2 * b + c] = make_uint4(x3[0], x3[1], x3[2], x3[3]);
                }
            }
        }
        return;
    }
    const uint32_t kend = min(n, k0 + kSeedGroup);
    for (uint32_t k = k0; k < kend; k++) {
        const uint32_t q = epochs(k);
        const int c = ds_cover(ds, q);
        if (c < 0) {
            x0[k] = make_uint4(0, 0, 0, 0);
            err_min(err, (unsigned long long)k << 1);  // SeedNotDisclosed, before hashing errors
            continue;
        }
        const DsNode& nd = ds.nodes[c];
        uint32_t x[4] = {nd.value[0], nd.value[1], nd.value[2], nd.value[3]};
        ds_walk(suite, t0, x, q - (uint32_t)((uint64_t)nd.index << nd.depth), (int)nd.depth);
        x0[k] = make_uint4(x[0], x[1], x[2], x[3]);
    }
}

// K0 with per-epoch seed stacks: the host resolved each epoch's covering
// node (value, offset below it, depth); one thread walks one epoch.
__global__ void k_seed_walk(int suite, const SeedStart* __restrict__ starts, uint32_t n, uint4* __restrict__ x0,
                            const uint32_t* __restrict__ t0g) {
    extern __shared__ uint32_t sT0[];
    if (suite != 1) load_t0(sT0, t0g);
    SmemT0 t0{sT0, threadIdx.x & 31u};
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const SeedStart st = starts[k];
    uint32_t x[4] = {st.value[0], st.value[1], st.value[2], st.value[3]};
    ds_walk(suite, t0, x, st.rel, (int)st.depth);
    x0[k] = make_uint4(x[0], x[1], x[2], x[3]);
}

// Scheme F per-entry scalars (poslo_f.cpp:223-246, distiller.cpp:103-115):
// e_t = hash_to_scalar(m_t, x_t) mod l, x_t the signature's seed tail or
// onetime_seed(x0[slot_t], j_t) when the entry's seed is derived from a stack.
__global__ void __launch_bounds__(128) k_fine_scalars(int suite, EntryLayout lay, uint64_t n,
                                                      const uint4* __restrict__ seeds,
                                                      const uint32_t* __restrict__ dslot,
                                                      const uint32_t* __restrict__ jj,
                                                      const uint4* __restrict__ x0,
                                                      uint32_t* __restrict__ e_out,
                                                      unsigned long long* err,
                                                      const uint32_t* __restrict__ t0g) {
    extern __shared__ uint32_t sT0[];
    if (suite != 1) load_t0(sT0, t0g);
    SmemT0 t0{sT0, threadIdx.x & 31u};
    const uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint8_t* m;
    uint32_t L;
    if (lay.offsets) {
        const uint64_t o0 = lay.offsets[t] + lay.header;
        m = lay.payload + o0;
        L = (uint32_t)(lay.offsets[t + 1] - o0);
    } else {
        m = lay.payload + t * lay.entry_len;
        L = lay.entry_len;
    }
    uint32_t x[4];
    if (dslot && dslot[t] != 0xFFFFFFFFu) {
        const uint4 xr = __ldg(x0 + dslot[t]);
        const uint32_t x0m[4] = {xr.x, xr.y, xr.z, xr.w};
        entry_seed(suite, t0, x0m, jj[t], x);
    } else {
        const uint4 xr = __ldg(seeds + t);
        x[0] = xr.x; x[1] = xr.y; x[2] = xr.z; x[3] = xr.w;
    }
    uint32_t limbs[16], e[8];
    if (!entry_limbs_x(suite, t0, m, L, x, limbs)) {
        err_min(err, (t << 1) | 1ull);  // FormatError (suite 3, L > 31)
#pragma unroll
        for (int k = 0; k < 16; k++) limbs[k] = 0;
    }
    sc_reduce_limbs(limbs, 16, e);
#pragma unroll
    for (int k = 0; k < 8; k++) e_out[t * 8 + k] = e[k];
}

// ---------------------------------------------------------------- signer side
// kg's commitment scalars r-hat_i = sum_j nonce_to_scalar(r, i, j) mod l
// (poslo_c.cpp:104-110): one CTA per epoch, entries strided over the threads.
struct Seed4 {
    uint32_t w[4];
};

__global__ void __launch_bounds__(256) k_nonce_sums(int suite, Seed4 r, const uint32_t* __restrict__ epochs,
                                                    uint32_t n2, uint32_t* __restrict__ out,
                                                    const uint32_t* __restrict__ t0g) {
    extern __shared__ uint32_t sT0[];
    __shared__ uint32_t red[8 * 17];
    if (suite != 1) load_t0(sT0, t0g);
    SmemT0 t0{sT0, threadIdx.x & 31u};
    const uint32_t i = epochs[blockIdx.x];
    uint32_t acc[17];
    acc17_zero(acc);
    for (uint32_t j = threadIdx.x; j < n2; j += blockDim.x) {
        uint32_t s[8], v[17];
        nonce_scalar(suite, t0, r.w, i, j, s);
#pragma unroll
        for (int k = 0; k < 17; k++) v[k] = k < 8 ? s[k] : 0u;
        acc17_add17(acc, v);
    }
    block_reduce_acc17(acc, red);
    if (threadIdx.x == 0) {
        uint32_t e[8];
        sc_reduce_limbs(acc, 17, e);
#pragma unroll
        for (int k = 0; k < 8; k++) out[(size_t)blockIdx.x * 8 + k] = e[k];
    }
}

// sig_epoch's s-hat_i = sum_j (r_ij - e_ij y) = r-hat_i - y e~_i mod l (poslo_c.cpp:115-134)
struct Scalar8 {
    uint32_t w[8];
};

__global__ void k_sign_combine(uint32_t n, const uint32_t* __restrict__ r_hat, const uint32_t* __restrict__ e,
                               Scalar8 y, uint32_t* __restrict__ out) {
    const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    uint32_t rr[8], ee[8], p[8], o[8];
#pragma unroll
    for (int q = 0; q < 8; q++) {
        rr[q] = r_hat[(size_t)k * 8 + q];
        ee[q] = e[(size_t)k * 8 + q];
    }
    sc_mul(y.w, ee, p);
    sc_sub(rr, p, o);
#pragma unroll
    for (int q = 0; q < 8; q++) out[(size_t)k * 8 + q] = o[q];
}

// ---------------------------------------------------------------- generic K1+K2
__global__ void __launch_bounds__(256) k_hash_generic(int suite, EntryLayout lay, TileMap tm,
                                                      const uint4* __restrict__ x0,
                                                      uint32_t* __restrict__ partial,
                                                      uint32_t* __restrict__ entry_e,
                                                      unsigned long long* err,
                                                      const uint32_t* __restrict__ t0g) {
    extern __shared__ uint32_t sT0[];
    __shared__ uint32_t red[8 * 17];
    if (suite != 1) load_t0(sT0, t0g);
    SmemT0 t0{sT0, threadIdx.x & 31u};
    const uint32_t tile = tm.tile_begin + blockIdx.x;
    uint32_t ep, j0, count;
    uint64_t ebase;
    if (tm.tiles) {
        uint4 t = tm.tiles[tile];
        ep = t.x; j0 = t.y; count = t.z;
        ebase = tm.epoch_starts[ep];
    } else {
        ep = tile / tm.tiles_per_epoch;
        uint32_t sub = tile - ep * tm.tiles_per_epoch;
        j0 = sub * tm.tile_entries;
        count = min(tm.tile_entries, tm.n2 - j0);
        ebase = (uint64_t)ep * tm.n2;
    }
    const uint4 xr = __ldg(x0 + ep);
    const uint32_t x0m[4] = {xr.x, xr.y, xr.z, xr.w};
    uint32_t acc[17];
    acc17_zero(acc);
    for (uint32_t idx = threadIdx.x; idx < count; idx += blockDim.x) {
        const uint32_t j = j0 + idx;
        const uint64_t ent = ebase + j;
        const uint8_t* m;
        uint32_t L;
        if (lay.offsets) {
            uint64_t o0 = lay.offsets[ent] + lay.header, o1 = lay.offsets[ent + 1];
            m = lay.payload + o0;
            L = (uint32_t)(o1 - o0);
        } else {
            m = lay.payload + ent * lay.entry_len;
            L = lay.entry_len;
        }
        uint32_t limbs[16];
        if (!entry_limbs(suite, t0, m, L, x0m, j, limbs)) {
            err_min(err, ((unsigned long long)ep << 1) | 1ull);  // FormatError
            continue;
        }
        acc17_add16(acc, limbs);
        if (entry_e) {
            uint32_t e[8];
            sc_reduce_limbs(limbs, 16, e);
#pragma unroll
            for (int k = 0; k < 8; k++) entry_e[ent * 8 + k] = e[k];
        }
    }
    block_reduce_acc17(acc, red);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < 17; k++) partial[(size_t)tile * 17 + k] = acc[k];
}

// ---------------------------------------------------------------- epoch finalize
__global__ void k_epoch_finalize(TileMap tm, uint32_t ep0, uint32_t ep1, const uint32_t* __restrict__ partial,
                                 uint32_t* __restrict__ etilde) {
    uint32_t ep = ep0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (ep >= ep1) return;
    uint32_t b, e;
    if (tm.tiles) {
        b = tm.epoch_tile_begin[ep];
        e = tm.epoch_tile_begin[ep + 1];
    } else {
        b = ep * tm.tiles_per_epoch;
        e = b + tm.tiles_per_epoch;
    }
    uint32_t acc[17];
    acc17_zero(acc);
    for (uint32_t t = b; t < e; t++) {
        uint32_t v[17];
#pragma unroll
        for (int k = 0; k < 17; k++) v[k] = partial[(size_t)t * 17 + k];
        acc17_add17(acc, v);
    }
    uint32_t r[8];
    sc_reduce_limbs(acc, 17, r);
#pragma unroll
    for (int k = 0; k < 8; k++) etilde[(size_t)ep * 8 + k] = r[k];
}

// ---------------------------------------------------------------- sums mod l
__device__ __forceinline__ void load_item(const uint32_t* items, int limbs, uint64_t i, uint32_t v[17]) {
#pragma unroll
    for (int k = 0; k < 17; k++) v[k] = k < limbs ? items[i * limbs + k] : 0u;
}

__global__ void __launch_bounds__(256) k_sum_stage1(const uint32_t* __restrict__ items, int limbs,
                                                    uint64_t n, const uint8_t* __restrict__ mask,
                                                    uint32_t* __restrict__ out) {
    __shared__ uint32_t red[8 * 17];
    uint32_t acc[17];
    acc17_zero(acc);
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        if (mask && mask[i]) continue;
        uint32_t v[17];
        load_item(items, limbs, i, v);
        acc17_add17(acc, v);
    }
    block_reduce_acc17(acc, red);
    if (threadIdx.x == 0)
#pragma unroll
        for (int k = 0; k < 17; k++) out[blockIdx.x * 17 + k] = acc[k];
}

__global__ void __launch_bounds__(256) k_sum_stage2(const uint32_t* __restrict__ parts, uint32_t n,
                                                    uint32_t* __restrict__ out) {
    __shared__ uint32_t red[8 * 17];
    uint32_t acc[17];
    acc17_zero(acc);
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
        uint32_t v[17];
        load_item(parts, 17, i, v);
        acc17_add17(acc, v);
    }
    block_reduce_acc17(acc, red);
    if (threadIdx.x == 0) {
        uint32_t r[8];
        sc_reduce_limbs(acc, 17, r);
#pragma unroll
        for (int k = 0; k < 8; k++) out[k] = r[k];
    }
}

__global__ void __launch_bounds__(256) k_segsum(const uint32_t* __restrict__ items,
                                                const uint64_t* __restrict__ seg,
                                                const uint8_t* __restrict__ mask, uint8_t skip_val,
                                                uint32_t* __restrict__ out) {
    __shared__ uint32_t red[8 * 17];
    const uint32_t g = blockIdx.x;
    uint32_t acc[17];
    acc17_zero(acc);
    for (uint64_t i = seg[g] + threadIdx.x; i < seg[g + 1]; i += blockDim.x) {
        if (mask && mask[i] == skip_val) continue;
        uint32_t v[17];
        load_item(items, 8, i, v);
        acc17_add17(acc, v);
    }
    block_reduce_acc17(acc, red);
    if (threadIdx.x == 0) {
        uint32_t r[8];
        sc_reduce_limbs(acc, 17, r);
#pragma unroll
        for (int k = 0; k < 8; k++) out[(size_t)g * 8 + k] = r[k];
    }
}

// ---------------------------------------------------------------- synthetic logs
// Counter-based synthetic entries (include/poslo_synth.h), byte-identical to
// what the CPU reference harness regenerates (oracle/ref_tools/ref_tool.cpp).
__global__ void k_synth_fixed(uint64_t seed, uint64_t first, uint64_t n, uint32_t L,
                              uint8_t* __restrict__ out) {
    uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    uint64_t k = first + t;
    if ((L & 7) == 0 && ((uintptr_t)out & 7) == 0) {
        uint64_t* o = reinterpret_cast<uint64_t*>(out + t * L);
        for (uint32_t w = 0; w < L / 8; w++) o[w] = poslo_synth_word(seed, k, w);
    } else {
        for (uint32_t b = 0; b < L; b++) out[t * L + b] = poslo_synth_byte(seed, k, b);
    }
}

// Variable-length printable entries at caller-provided offsets (lengths from
// poslo_synth_varlen), byte-identical to the CPU generator.
__global__ void k_synth_var(uint64_t seed, uint64_t first, uint64_t n, const uint64_t* __restrict__ offsets,
                            uint8_t* __restrict__ out) {
    uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (t >= n) return;
    const uint64_t o0 = offsets[t], o1 = offsets[t + 1];
    for (uint64_t b = 0; b < o1 - o0; b++) out[o0 + b] = poslo_synth_ascii(seed, first + t, (uint32_t)b);
}

}  // namespace

// ---------------------------------------------------------------- launchers
// One thread per gap, grid-strided: a read of 8 bytes per entry (~10 us per
// 2^22 offsets), run once per call before any hashing kernel.
__global__ void __launch_bounds__(256) k_check_offsets(const uint64_t* __restrict__ off, uint64_t n, uint32_t header,
                                                       uint64_t lo, uint64_t hi, int* bad) {
    bool ok = true;
    for (uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; t < n; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t a = off[t], z = off[t + 1];
        ok &= z >= a && z - a >= header;
        if (t == 0) ok &= a >= lo;
        if (t == n - 1) ok &= z <= hi;
    }
    if (__syncthreads_or(!ok) && threadIdx.x == 0) atomicOr(bad, 1);
}

void launch_check_offsets(const uint64_t* d_off, uint64_t n, uint32_t header, uint64_t lo, uint64_t hi, int* d_bad,
                          cudaStream_t s) {
    const uint64_t blocks = std::min<uint64_t>((n + 255) / 256, 148 * 8);
    k_check_offsets<<<(unsigned)std::max<uint64_t>(blocks, 1), 256, 0, s>>>(d_off, n, header, lo, hi, d_bad);
}

void launch_seed_derive(int suite, const DsParam& ds, const uint32_t* d_epochs, uint32_t epoch0, uint32_t n_epochs,
                        uint4* d_x0, unsigned long long* d_err, const uint32_t* d_t0, cudaStream_t s) {
    if (n_epochs == 0) return;
    int T = 64;
    size_t smem = suite == 1 ? 0 : kAesSmemWords * sizeof(uint32_t);
    if (smem) cudaFuncSetAttribute(k_seed_derive, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    uint32_t groups = (n_epochs + kSeedGroup - 1) / kSeedGroup;
    k_seed_derive<<<(groups + T - 1) / T, T, smem, s>>>(suite, ds, d_epochs, epoch0, n_epochs, d_x0, d_err, d_t0);
}

void launch_seed_walk(int suite, const SeedStart* d_starts, uint32_t n, uint4* d_x0, const uint32_t* d_t0,
                      cudaStream_t s) {
    if (!n) return;
    int T = 64;
    size_t smem = suite == 1 ? 0 : kAesSmemWords * sizeof(uint32_t);
    if (smem) cudaFuncSetAttribute(k_seed_walk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_seed_walk<<<(n + T - 1) / T, T, smem, s>>>(suite, d_starts, n, d_x0, d_t0);
}

void launch_fine_scalars(int suite, const EntryLayout& lay, uint64_t n, const uint4* d_seeds, const uint32_t* d_dslot,
                         const uint32_t* d_j, const uint4* d_x0, uint32_t* d_e, unsigned long long* d_err,
                         const uint32_t* d_t0, cudaStream_t s) {
    if (!n) return;
    size_t smem = suite == 1 ? 0 : kAesSmemWords * sizeof(uint32_t);
    if (smem) cudaFuncSetAttribute(k_fine_scalars, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_fine_scalars<<<(unsigned)((n + 127) / 128), 128, smem, s>>>(suite, lay, n, d_seeds, d_dslot, d_j, d_x0, d_e,
                                                                 d_err, d_t0);
}

void launch_nonce_sums(int suite, const uint32_t r_words[4], const uint32_t* d_epochs, uint32_t n, uint32_t n2,
                       uint32_t* d_out, const uint32_t* d_t0, cudaStream_t s) {
    if (!n) return;
    Seed4 r;
    for (int k = 0; k < 4; k++) r.w[k] = r_words[k];
    size_t smem = suite == 1 ? 0 : kAesSmemWords * sizeof(uint32_t);
    if (smem) cudaFuncSetAttribute(k_nonce_sums, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_nonce_sums<<<n, 256, smem, s>>>(suite, r, d_epochs, n2, d_out, d_t0);
}

void launch_sign_combine(uint32_t n, const uint32_t* d_rhat, const uint32_t* d_e, const uint32_t y_words[8],
                         uint32_t* d_out, cudaStream_t s) {
    if (!n) return;
    Scalar8 y;
    for (int k = 0; k < 8; k++) y.w[k] = y_words[k];
    k_sign_combine<<<(n + 127) / 128, 128, 0, s>>>(n, d_rhat, d_e, y, d_out);
}

void launch_hash_generic(int suite, const EntryLayout& lay, const TileMap& tm, const uint4* d_x0,
                         uint32_t* d_partial, uint32_t* d_entry_e, unsigned long long* d_err,
                         const uint32_t* d_t0, cudaStream_t s) {
    uint32_t n_tiles = tm.tile_count ? tm.tile_count : (tm.tiles ? tm.n_tiles : tm.n_epochs * tm.tiles_per_epoch);
    if (!n_tiles) return;
    size_t smem = suite == 1 ? 0 : kAesSmemWords * sizeof(uint32_t);
    if (smem) cudaFuncSetAttribute(k_hash_generic, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_hash_generic<<<n_tiles, 256, smem, s>>>(suite, lay, tm, d_x0, d_partial, d_entry_e, d_err, d_t0);
}

void launch_epoch_finalize(const TileMap& tm, const uint32_t* d_partial, uint32_t* d_etilde,
                           cudaStream_t s) {
    if (!tm.n_epochs) return;
    k_epoch_finalize<<<(tm.n_epochs + 127) / 128, 128, 0, s>>>(tm, 0, tm.n_epochs, d_partial, d_etilde);
}

void launch_epoch_finalize_range(const TileMap& tm, uint32_t e0, uint32_t e1, const uint32_t* d_partial,
                                 uint32_t* d_etilde, cudaStream_t s) {
    if (e1 <= e0) return;
    k_epoch_finalize<<<(e1 - e0 + 127) / 128, 128, 0, s>>>(tm, e0, e1, d_partial, d_etilde);
}

void launch_sum_mod_l(const uint32_t* d_items, int limbs, uint64_t n, const uint8_t* d_mask,
                      uint32_t* d_out, uint32_t* d_scratch, cudaStream_t s) {
    uint64_t want = (n + 255) / 256;
    uint32_t blocks = (uint32_t)(want < 1 ? 1 : (want > 1024 ? 1024 : want));
    k_sum_stage1<<<blocks, 256, 0, s>>>(d_items, limbs, n, d_mask, d_scratch);
    k_sum_stage2<<<1, 256, 0, s>>>(d_scratch, blocks, d_out);
}

void launch_segsum_mod_l(const uint32_t* d_items, const uint64_t* d_seg, uint32_t n_groups,
                         const uint8_t* d_mask, uint32_t* d_out, cudaStream_t s, uint8_t skip_val) {
    if (!n_groups) return;
    k_segsum<<<n_groups, 256, 0, s>>>(d_items, d_seg, d_mask, skip_val, d_out);
}

void launch_synth_fixed(uint64_t seed, uint64_t first, uint64_t n, uint32_t L, uint8_t* d_out,
                        cudaStream_t s) {
    if (!n) return;
    k_synth_fixed<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(seed, first, n, L, d_out);
}

void launch_synth_var(uint64_t seed, uint64_t first, uint64_t n, const uint64_t* d_offsets, uint8_t* d_out,
                      cudaStream_t s) {
    if (!n) return;
    k_synth_var<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(seed, first, n, d_offsets, d_out);
}

}  // namespace poslo_gpu
