// Internal launcher interface between the C-ABI layer (capi.cu) and the
// kernels (verify_kernels.cu, group_kernels.cu). Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace poslo_gpu {

// One disclosed-seed-stack node, parsed from the SeedStack wire format
// (proj/src/seed_manager.cpp:32-53).
struct DsNode {
    uint32_t depth;
    uint32_t index;
    uint32_t value[4];  // 16 seed bytes as little-endian memory words
};
struct DsParam {
    int count;
    DsNode nodes[32];
};

// How the entries of the queried epochs are laid out in device memory.
struct EntryLayout {
    const uint8_t* payload;   // entry bytes
    const uint64_t* offsets;  // n_entries + 1 byte offsets, or nullptr (fixed stride)
    uint32_t entry_len;       // stride / length when offsets == nullptr
    uint32_t header;          // bytes before each entry at offsets[t] (4: LE32 log records), else 0
};

// Tiles: a tile is a contiguous run of entries of ONE epoch that one CTA
// hashes and sums. Uniform batches (every epoch n2 entries, the k-th queried
// epoch's entries at [k*n2, (k+1)*n2)) use implicit tiles; ragged batches
// pass an explicit tile table built on the host from epoch_starts.
struct TileMap {
    uint32_t n_epochs;
    uint32_t n2;                    // uniform only
    uint32_t tile_entries;          // entries per tile (uniform only)
    uint32_t tiles_per_epoch;       // uniform only
    const uint4* tiles;             // explicit: {epoch_idx, j0, count, 0}; nullptr = uniform
    const uint64_t* epoch_starts;   // explicit: n_epochs + 1 entry indices
    const uint32_t* epoch_tile_begin;  // explicit: n_epochs + 1 tile indices
    uint32_t n_tiles;
    uint32_t tile_begin;  // launch only tiles [tile_begin, tile_begin + tile_count) (chunked H2D)
    uint32_t tile_count;  // 0 = all tiles
};

// Per-epoch seed stacks (poslo_batch.ds_offsets): walk `depth` levels from
// the covering node's value along the low bits of rel.
struct SeedStart {
    uint32_t value[4];
    uint32_t rel;
    uint32_t depth;
};
void launch_seed_walk(int suite, const SeedStart* d_starts, uint32_t n, uint4* d_x0, const uint32_t* d_t0,
                      cudaStream_t s);
// Scheme F per-entry scalars mod l (8 limbs each): x from seeds[t], or
// onetime_seed(x0[dslot[t]], j[t]) where dslot[t] != UINT32_MAX.
void launch_fine_scalars(int suite, const EntryLayout& lay, uint64_t n, const uint4* d_seeds, const uint32_t* d_dslot,
                         const uint32_t* d_j, const uint4* d_x0, uint32_t* d_e, unsigned long long* d_err,
                         const uint32_t* d_t0, cudaStream_t s);
// Signer side (kg / sig_epoch): per-epoch nonce sums r-hat (8 limbs) and
// s-hat = r-hat - y e~ mod l.
void launch_nonce_sums(int suite, const uint32_t r_words[4], const uint32_t* d_epochs, uint32_t n, uint32_t n2,
                       uint32_t* d_out, const uint32_t* d_t0, cudaStream_t s);
void launch_sign_combine(uint32_t n, const uint32_t* d_rhat, const uint32_t* d_e, const uint32_t y_words[8],
                         uint32_t* d_out, cudaStream_t s);
// d_epochs == nullptr: epochs epoch0, epoch0 + 1, ..., epoch0 + n_epochs - 1.
void launch_seed_derive(int suite, const DsParam& ds, const uint32_t* d_epochs, uint32_t epoch0, uint32_t n_epochs,
                        uint4* d_x0, unsigned long long* d_err, const uint32_t* d_t0, cudaStream_t s);

// Fast path: suite 1, 32-byte entries, uniform epochs. Writes per-tile
// 17-limb partial sums, or e_tilde directly when one tile covers an epoch.
// Suite-1, 32-byte uniform epochs of at most kLeanMaxN2 entries are hashed one
// epoch per CTA slice (tile == epoch); larger epochs are tiled.
constexpr uint32_t kLeanMaxN2 = 4096;
void launch_hash_s1_l32(const EntryLayout& lay, const TileMap& tm, const uint4* d_x0,
                        uint32_t* d_partial, uint32_t* d_etilde, cudaStream_t s);

// Fast path: suite 2 (MMO/MDC-2 over AES-128), 32-byte entries, uniform.
void launch_hash_s2_l32(const EntryLayout& lay, const TileMap& tm, const uint4* d_x0,
                        uint32_t* d_partial, uint32_t* d_etilde, const uint32_t* d_t0, cudaStream_t s);

// Generic path: any suite, any entry length, uniform or ragged epochs.
// Optional per-entry scalars (debug/parity: e_i^j mod l, 8 limbs each).
void launch_hash_generic(int suite, const EntryLayout& lay, const TileMap& tm, const uint4* d_x0,
                         uint32_t* d_partial, uint32_t* d_entry_e, unsigned long long* d_err,
                         const uint32_t* d_t0, cudaStream_t s);

// Suite 1 over variable-length (or any non-32-byte) entries: streamed SHA-256
// straight from the payload, tiles length-sorted in shared memory. Writes
// per-tile partials (tile_entries must be <= 1024).
void launch_hash_s1_var(const EntryLayout& lay, const TileMap& tm, const uint4* d_x0, uint32_t* d_partial,
                        cudaStream_t s);

// Layout check of caller-supplied entry offsets (n entries, n + 1 offsets):
// *d_bad = 1 unless lo <= off[0], off[t] + header <= off[t+1] and off[n] <= hi.
void launch_check_offsets(const uint64_t* d_off, uint64_t n, uint32_t header, uint64_t lo, uint64_t hi, int* d_bad,
                          cudaStream_t s);

// Per-epoch e~ from tile partials (skipped when tiles_per_epoch == 1 on the
// fast paths, which finalise in the hashing kernel).
void launch_epoch_finalize(const TileMap& tm, const uint32_t* d_partial, uint32_t* d_etilde,
                           cudaStream_t s);
// Epochs [e0, e1) only (pipelined per-chunk finalize).
void launch_epoch_finalize_range(const TileMap& tm, uint32_t e0, uint32_t e1, const uint32_t* d_partial,
                                 uint32_t* d_etilde, cudaStream_t s);

// out (8 limbs) = sum of n items mod l; items are `limbs`-limb little-endian
// integers (8 for scalars, 17 for partial accumulators). Optional mask: skip
// item i when mask[i] != 0. d_scratch >= 17 * 1024 u32.
void launch_sum_mod_l(const uint32_t* d_items, int limbs, uint64_t n, const uint8_t* d_mask,
                      uint32_t* d_out, uint32_t* d_scratch, cudaStream_t s);

// Segmented variant: out[g] = sum of items [seg[g], seg[g+1]) (mask honoured).
void launch_segsum_mod_l(const uint32_t* d_items, const uint64_t* d_seg, uint32_t n_groups,
                         const uint8_t* d_mask, uint32_t* d_out, cudaStream_t s,
                         uint8_t skip_val = 1);

// Batched commit_check: enc[i] = encode(Y^e_i * alpha^s_i); verdict[i] =
// (enc[i] == r[i]) when r != nullptr. Y is decoded once (d_ybad set when Y
// is not a valid encoding). e/s are 8-limb canonical scalars.
void launch_group_check(const uint8_t* d_y, uint32_t n, const uint32_t* d_e, const uint32_t* d_s,
                        const uint8_t* d_r, uint8_t* d_enc, uint8_t* d_verdict, int* d_ybad,
                        cudaStream_t s);

// Fixed-base comb table (512 affine Niels points, 48 KiB) of the point encoded at
// d_enc, or of the generator when d_enc == nullptr. d_pk_scratch >= 64 * kGptBytes.
constexpr size_t kFeBytes = 40;                    // field element: 10 x 32-bit limbs (radix 2^25.5)
constexpr size_t kCachedBytes = 3 * kFeBytes;       // affine Niels point (y+x, y-x, 2dxy)
constexpr size_t kGptBytes = 4 * kFeBytes;          // extended point (X, Y, Z, T)
constexpr size_t kCombTableBytes = 512 * kCachedBytes;      // radix 16: 64 x 8 affine Niels points
constexpr size_t kComb256TableBytes = 4096 * kCachedBytes;  // radix 256: 32 x 128 points
constexpr size_t kComb16TableBytes = (size_t)16 * 32768 * kCachedBytes;  // radix 2^16: 16 x 32768 points (60 MiB)
constexpr uint32_t kCtaCheckMax = 1024;          // larger batches use one thread per check (radix-256 combs)
// One coarse distill step on the radix-16 combs (k_distill_step): s_items =
// [acc_s0, s_hat, acc_s1], pts = [acc_r0, r_hat, acc_r1] (encodings).
void launch_distill_step(const void* d_tabY, const void* d_tabB, const uint32_t* d_e, const uint32_t* d_s_items,
                         const uint8_t* d_pts, uint8_t* d_verdict, uint32_t* d_out_s, uint8_t* d_out_r, int* d_bad,
                         cudaStream_t s);
// pk[i] = 16^i P, i < 64 (P decoded from d_enc, or the generator); then the
// comb table of radix kind 0 = 16, 1 = 256, 2 = 2^16 from those powers.
void launch_table_powers(const uint8_t* d_enc, void* d_pk, int* d_bad, cudaStream_t s);
void launch_table_fill(int kind, const void* d_pk, void* d_table, cudaStream_t s);
void launch_build_table(const uint8_t* d_enc, void* d_pk_scratch, void* d_table, int* d_bad,
                        cudaStream_t s);
// commit_check via comb tables of Y and alpha (CTA-per-check for n <= 1024,
// thread-per-check above).
// Raw log image scan (log_scan.cu): chunk / window geometry and the three phases.
constexpr uint64_t kScanChunk = 1ull << 20;
constexpr uint32_t kScanWindow = 2048;
// Pipelined ingestion: scan + incremental stitch + offsets for chunks
// [c_first, c_last); d_state = {next record position, records so far}.
// chunk_bytes: kScanChunk, or kRawScanChunk in the pipelined path (short
// chunks: each emitting thread walks ~100 records, not ~2000). d_exit /
// d_count hold the (c_last - c_first) x kScanWindow candidate exits of this range.
constexpr uint64_t kRawScanChunk = 1ull << 16;
void launch_log_scan_range(const uint8_t* d_raw, uint64_t n, uint32_t c_first, uint32_t c_last, uint64_t chunk_bytes,
                           uint64_t* d_exit, uint32_t* d_count, uint64_t* d_start, uint64_t* d_base,
                           unsigned long long* d_state, uint64_t* d_offsets, uint64_t cap, cudaStream_t s);
void launch_log_scan_a(const uint8_t* d_raw, uint64_t n, uint32_t n_chunks, uint64_t* d_exit, uint32_t* d_count,
                       cudaStream_t s);
void launch_log_scan_b(const uint8_t* d_raw, uint64_t n, uint32_t n_chunks, const uint64_t* d_exit,
                       const uint32_t* d_count, uint64_t* d_start, uint64_t* d_base, unsigned long long* d_state,
                       cudaStream_t s);
void launch_log_scan_c(const uint8_t* d_raw, uint64_t n, uint32_t n_chunks, const uint64_t* d_start,
                       const uint64_t* d_base, uint64_t* d_offsets, cudaStream_t s);
// Masked segmented group_combine fold: one CTA per segment; out = encodings
// (identity = zeros). *d_bad set when a point fails to decode.
void launch_segfold_points(const uint8_t* d_pts, const uint32_t* d_seg, uint32_t n_seg, const uint8_t* d_mask,
                           uint8_t* d_out, int* d_bad, cudaStream_t s);
// Batched checks with R decoded ahead (side stream, overlapping the hashing):
// d_pts n x 128 B (extended coordinates), d_ok n bytes; check_split runs 8
// lanes per check on the radix-256 combs; segfold_decoded folds decoded points.
constexpr size_t kPointBytes = kGptBytes;
void launch_decode_points(const uint8_t* d_enc, uint32_t n, void* d_pts, uint8_t* d_ok, cudaStream_t s);
// Radix-2^16 tables (kComb16TableBytes) and the 8-lane check on them.
void launch_build_table65536(const uint8_t* d_enc, void* d_pk_scratch, void* d_table, int* d_bad, cudaStream_t s);
void launch_check_thread16(const void* d_tabY16, const void* d_tabB16, uint32_t n, const uint32_t* d_e,
                           const uint32_t* d_s, const uint8_t* d_r, uint8_t* d_enc, uint8_t* d_verdict,
                           cudaStream_t s);
void launch_check_thread16d(const void* d_tabY16, const void* d_tabB16, uint32_t n, const uint32_t* d_e,
                            const uint32_t* d_s, const void* d_pts, const uint8_t* d_ok, uint8_t* d_verdict,
                            cudaStream_t s);
// radix-2^16 checks without a square root per check (encode(P) == R-hat by
// squares, one batched inversion per 32 checks): d_P n x kGptBytes (the points
// e Y + s B, kept: distillation folds them in place of the decoded R-hat),
// d_u2 and d_pre n x kFeBytes scratch
constexpr size_t kCheck16eScratch = kGptBytes + 2 * kFeBytes;
void launch_check16e(const void* d_tabY16, const void* d_tabB16, uint32_t n, const uint32_t* d_e, const uint32_t* d_s,
                     const uint8_t* d_r, void* d_P, void* d_u2, void* d_pre, uint8_t* d_verdict, cudaStream_t s);
void launch_check_split16(const void* d_tabY16, const void* d_tabB16, uint32_t n, const uint32_t* d_e,
                          const uint32_t* d_s, const void* d_pts, const uint8_t* d_ok, uint8_t* d_verdict,
                          cudaStream_t s);
void launch_check_split(const void* d_tabY256, const void* d_tabB256, uint32_t n, const uint32_t* d_e,
                        const uint32_t* d_s, const void* d_pts, const uint8_t* d_ok, uint8_t* d_verdict,
                        cudaStream_t s);
void launch_segfold_decoded(const void* d_pts, const uint32_t* d_seg, uint32_t n_seg, const uint8_t* d_mask,
                            uint8_t* d_out, cudaStream_t s);
// Radix-256 tables (kComb256TableBytes) for the thread-per-check path.
void launch_build_table256(const uint8_t* d_enc, void* d_pk_scratch, void* d_table, int* d_bad, cudaStream_t s);
void launch_group_check_comb(const void* d_tabY, const void* d_tabB, const void* d_tabY256,
                             const void* d_tabB256, uint32_t n, const uint32_t* d_e, const uint32_t* d_s,
                             const uint8_t* d_r, uint8_t* d_enc, uint8_t* d_verdict, cudaStream_t s);

// Split single check for paver: pre (R decode, T = R - s*alpha; independent
// of e-hat, overlappable with hashing) and post (e*Y == T). d_pre >= 256 B.
void launch_check_pre(const void* d_tabB, const uint32_t* d_s, const uint8_t* d_r, void* d_pre,
                      cudaStream_t s);
void launch_check_post(const void* d_tabY, const uint32_t* d_e, const void* d_pre, uint8_t* d_verdict,
                       cudaStream_t s);

// Fold of n encoded points with the group law (group_combine); d_bad counts
// invalid encodings. d_scratch >= 1024 * 128 bytes.
void launch_point_fold(const uint8_t* d_pts, uint64_t n, uint8_t* d_out, int* d_bad,
                       void* d_scratch, cudaStream_t s);

// Point validation (GroupElement::from_bytes): ok[i] = 1 if valid.
void launch_point_validate(const uint8_t* d_pts, uint32_t n, uint8_t* d_ok, cudaStream_t s);

// Synthetic fixed-length log entries [first, first+n) (include/poslo_synth.h).
void launch_synth_fixed(uint64_t seed, uint64_t first, uint64_t n, uint32_t L, uint8_t* d_out,
                        cudaStream_t s);

// Synthetic variable-length printable entries at device offsets (n + 1).
void launch_synth_var(uint64_t seed, uint64_t first, uint64_t n, const uint64_t* d_offsets, uint8_t* d_out,
                      cudaStream_t s);

}  // namespace poslo_gpu
