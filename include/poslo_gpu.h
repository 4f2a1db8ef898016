/* poslo_gpu.h — C-ABI of the B200 batch verifier for POSLO (arXiv 2506.08781).
 *
 * Drop-in boundary for the reference's batch-verification path
 * (/root/reference/proj/include/poslo/batch_verify.hpp:11-30). Plain pointers
 * and sizes only; no C++ or torch types. The C++ drop-in
 * (paper_2506_08781_b200/host/batch_verify_gpu.cpp) implements the reference
 * signatures `poslo::agg_ekeys` / `poslo::paver` on top of these calls, and
 * INTEGRATION.md shows the binding a reference maintainer would add.
 *
 * Conventions
 *   - Scalars are 32-byte LITTLE-endian canonical values (< l), the reference's
 *     in-memory Scalar form (group.hpp:38,43); the big-endian wire form is the
 *     host's business.
 *   - Group elements are 32-byte canonical ristretto255 encodings; identity is
 *     32 zero bytes (group.hpp:47-59).
 *   - `ds` is the SeedStack wire format exactly as SeedStack::serialize
 *     writes it (seed_manager.cpp:32-39), with capacity D = log2(n1).
 *   - Entry layout: the queried epochs' entries are packed back to back in
 *     epoch order; epoch k (k-th entry of `epochs`) owns entries
 *     [epoch_starts[k], epoch_starts[k+1]) — or [k*n2, (k+1)*n2) when
 *     epoch_starts is NULL. Entry t's bytes are payload[offsets[t] ..
 *     offsets[t+1]) — or payload[t*entry_len .. (t+1)*entry_len) when offsets
 *     is NULL.
 *   - `device_resident`: payload/offsets are device pointers (already in HBM);
 *     everything else is always host memory.
 *   - Every call is synchronous with respect to its outputs and re-entrant
 *     per context (a context serialises its own calls; use one context per
 *     host thread for concurrency).
 *
 * Errors (same taxonomy and order as the reference): return
 * value and err->code are one of POSLO_OK, POSLO_FORMAT_ERROR (FormatError),
 * POSLO_STATE_ERROR (StateError), POSLO_SEED_NOT_DISCLOSED (SeedNotDisclosed,
 * err->epoch = the epoch, the lowest one as with workers == 1),
 * POSLO_CUDA_ERROR, POSLO_INVALID_ARGUMENT. No call ever falls back to a CPU
 * implementation; without a usable sm_100 device every call returns
 * POSLO_CUDA_ERROR. */
#ifndef POSLO_GPU_H
#define POSLO_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define POSLO_OK 0
#define POSLO_FORMAT_ERROR 1
#define POSLO_STATE_ERROR 2
#define POSLO_SEED_NOT_DISCLOSED 3
#define POSLO_CUDA_ERROR 4
#define POSLO_INVALID_ARGUMENT 5

typedef struct poslo_gpu_ctx poslo_gpu_ctx;

typedef struct poslo_error {
    int32_t code;
    uint32_t epoch; /* offending epoch for POSLO_SEED_NOT_DISCLOSED / StateError */
    char message[240];
} poslo_error;

/* A packed batch: the `std::map<uint32_t, std::vector<Bytes>> batches`
 * argument of agg_ekeys/paver (batch_verify.hpp:20-30) plus the
 * SuiteConfig and SeedStack it is verified against. */
typedef struct poslo_batch {
    uint8_t suite;                 /* SuiteId: 1 SHA-256, 2 MMO/MDC-2, 3 MMO/ADD_Q */
    uint32_t n2;                   /* entries per epoch (SuiteConfig::n2) */
    const uint8_t* payload;        /* entry bytes */
    uint64_t payload_bytes;
    const uint64_t* offsets;       /* n_entries + 1 byte offsets, or NULL */
    uint32_t entry_len;            /* fixed entry length when offsets == NULL */
    uint64_t n_entries;
    const uint32_t* epochs;        /* n_epochs queried epoch indices, strictly ascending (host) */
    const uint64_t* epoch_starts;  /* n_epochs + 1 entry indices (host), or NULL = uniform n2 */
    uint32_t n_epochs;
    const uint8_t* ds;             /* SeedStack wire bytes (host) */
    uint32_t ds_len;
    uint32_t ds_capacity;          /* D = log2(n1) */
    int32_t device_resident;       /* payload/offsets live in device memory */
    const uint64_t* ds_offsets;    /* optional (host): n_epochs + 1 byte offsets into `ds`; epoch k
                                      is then derived from its OWN stack ds[ds_offsets[k] ..
                                      ds_offsets[k+1]) (EpochSignature::ds, the distill_epoch
                                      semantics). NULL: one stack `ds` for every epoch. */
    uint32_t record_header;        /* 0, or 4 for a raw log file (log_file.hpp:34-51): `payload` is
                                      the file's bytes, offsets[t] the position of record t's LE32
                                      length and the entry is payload[offsets[t] + 4 .. offsets[t+1])
                                      (offsets from poslo_log_scan; zero-copy ingestion).
                                      With offsets == NULL the payload is a WHOLE raw image whose
                                      records the device finds itself (read_log + epochs_of): the
                                      record count must be n_epochs x n2 (uniform epochs). A host
                                      image is then copied in 64 MiB chunks with the record scan and
                                      the hashing of every completed epoch behind the copy. Errors:
                                      FormatError "truncated log record" (read_log), "record count
                                      must be a nonzero multiple of n2" (epochs_of), then
                                      INVALID_ARGUMENT when the count names other epochs. */
    /* Optional host producer of the entry bytes, for callers whose entries are not
     * contiguous in memory (the reference's std::map<u32, vector<Bytes>>): with
     * payload == NULL and device_resident == 0, the library calls
     * fill(fill_user, first, count, dst) to write entries [first, first + count)
     * back to back into dst (pinned staging of up to 64 MiB for fixed-length
     * entries: whole epochs per call, ascending, from the calling thread), and copies
     * and hashes each chunk while the next one is being produced. payload_bytes
     * (and offsets, for variable lengths) still describe the packed layout. A
     * nonzero return aborts the call with POSLO_INVALID_ARGUMENT. */
    int (*fill)(void* fill_user, uint64_t first, uint64_t count, uint8_t* dst);
    void* fill_user;
} poslo_batch;

/* Scheme F (POSLO-F, include/poslo/poslo_f.hpp) entries: each entry t has a
 * one-time seed x_t, either the FineSignature seed tail (seeds[t], 16 B) or,
 * where derive_slot[t] != UINT32_MAX, onetime_seed(sr(stack, slot_epochs[s]),
 * j[t]) with s = derive_slot[t] and the slot's stack ds (ds_offsets: one
 * stack per slot, else the one stack for all slots). Entry bytes as in
 * poslo_batch (payload/offsets/entry_len). */
typedef struct poslo_fine_batch {
    uint8_t suite;
    const uint8_t* payload;
    uint64_t payload_bytes;
    const uint64_t* offsets;       /* n_entries + 1, or NULL (fixed entry_len) */
    uint32_t entry_len;
    uint64_t n_entries;
    int32_t device_resident;       /* payload/offsets in device memory */
    const uint8_t* seeds;          /* n_entries x 16 B (host); may be NULL when every entry is derived */
    const uint32_t* derive_slot;   /* n_entries (host) or NULL (all from seeds) */
    const uint32_t* j;             /* n_entries (host): position in the epoch, for derived entries */
    const uint32_t* slot_epochs;   /* n_slots epoch indices (host) */
    uint32_t n_slots;
    const uint8_t* ds;             /* SeedStack wire bytes (host) */
    uint32_t ds_len;
    uint32_t ds_capacity;
    const uint64_t* ds_offsets;    /* n_slots + 1 (host) or NULL */
} poslo_fine_batch;

/* ---- log ingestion (read_log, include/poslo/log_file.hpp:34-51) -------------
 * Host-side scan of a raw log file image (records: LE32 length + payload).
 * Writes the record header positions to offsets[0..n] (offsets[n] = len)
 * and n to *n_records. FormatError "truncated log record" exactly where
 * read_log throws it. cap = capacity of `offsets` in records (it needs n + 1
 * slots); when too small, returns POSLO_INVALID_ARGUMENT with *n_records =
 * the count needed. Pure host code; no device is touched. */
int poslo_log_scan(const uint8_t* raw, uint64_t len, uint64_t* offsets, uint64_t cap, uint64_t* n_records,
                   poslo_error* err);
/* The same on the device (speculative chunk walks + stitch, log_scan.cu):
 * identical offsets and errors, ~100x the host scan's rate on large images.
 * device_resident: raw and offsets are device pointers (the image stays in
 * HBM for a zero-copy record batch), else host memory. */
int poslo_gpu_log_scan(poslo_gpu_ctx* ctx, const uint8_t* raw, uint64_t len, int32_t device_resident,
                       uint64_t* offsets, uint64_t cap, uint64_t* n_records, poslo_error* err);

/* ---- context -------------------------------------------------------------- */
int poslo_gpu_create(int device, poslo_gpu_ctx** out, poslo_error* err);
/* Multi-device context (SURVEY §8b "select GPU count", §8e): one member
 * context per entry of `devices` (a device may repeat: members then share
 * it, which exercises the sharded path on one GPU). agg_ekeys, paver,
 * epoch_verify and distill_coarse shard the queried epochs into contiguous
 * ranges balanced by entry bytes, one range per member, run the members
 * concurrently (one host thread and stream per member) and combine on member
 * 0: e-hat partials folded mod l in member order, R-hat partials with the
 * group law, per-epoch outputs concatenated, umbrella pieces that a shard cut
 * splits folded back together — byte-identical to the single-device result.
 * Device-resident batches run on the member owning the memory; raw images
 * without offsets and every other call run on member 0. */
int poslo_gpu_create_multi(const int* devices, int n_devices, poslo_gpu_ctx** out, poslo_error* err);
/* Members of a context (1 for a single-device context). */
int poslo_gpu_member_count(const poslo_gpu_ctx* ctx);
/* Visible CUDA devices (0 without a driver / device). */
int poslo_gpu_device_count(void);
void poslo_gpu_destroy(poslo_gpu_ctx* ctx);
/* Run subsequent work on this cudaStream_t (NULL = the context's own stream,
 * a blocking stream: ordered after work on the legacy default stream). */
int poslo_gpu_set_stream(poslo_gpu_ctx* ctx, void* cuda_stream);
/* Device stage timings (ms) of the last call when enabled: [seed, hash,
 * epoch_finalize, sum, group, total]. */
int poslo_gpu_enable_timing(poslo_gpu_ctx* ctx, int on);
int poslo_gpu_last_timings(poslo_gpu_ctx* ctx, float out_ms[6]);
/* Number of kernels the last call launched. */
uint32_t poslo_gpu_last_launches(poslo_gpu_ctx* ctx);
const char* poslo_gpu_version(void);

/* ---- agg_ekeys (batch_verify.cpp:11-62) -------------------------------------
 * e_tilde_out: n_epochs x 32 B (LE), per queried epoch in the given
 * (ascending) order — EpochKeyAggregate::e; may be NULL.
 * e_hat_out: 32 B, sum of all e~ mod l (aggregate_ekey, poslo_c.cpp:177-190);
 * may be NULL. Errors: SeedNotDisclosed / FormatError (suite 3, L > 31) for
 * the lowest offending epoch, seed retrieval first. */
int poslo_gpu_agg_ekeys(poslo_gpu_ctx* ctx, const poslo_batch* batch, uint8_t* e_tilde_out,
                        uint8_t* e_hat_out, poslo_error* err);

/* ---- paver (batch_verify.cpp:64-87) -----------------------------------------
 * Checks every epoch holds n2 entries (StateError), folds R-hat from
 * r_hats (n_epochs x 32 B, pk.r_hats[epoch] in batch order) unless
 * r_hat_agg (32 B) is given, computes e-hat and returns
 * *verdict = (commit_check(Y, e-hat, s-hat) == R-hat). */
int poslo_gpu_paver(poslo_gpu_ctx* ctx, const poslo_batch* batch, const uint8_t y[32],
                    const uint8_t s_hat[32], const uint8_t* r_hat_agg, const uint8_t* r_hats,
                    uint8_t* verdict, poslo_error* err);

/* ---- multi-rank coarse PAVer (one process per GPU) ---------------
 * agg_ekeys_partial: e-hat of this shard (sum of its e~ mod l) written to
 * d_e_part, a 32-byte DEVICE pointer on the context's device, in stream order
 * on the context's stream (so a collective queued on the same stream after
 * the call gathers it without a host round trip). Errors as agg_ekeys.
 * combine_check: e-hat = sum of the n_parts partials mod l (in the given =
 * rank order), *verdict = (commit_check(Y, e-hat, s-hat) == r_hat) — the
 * fold and final check of paver (batch_verify.cpp:83-86). parts_on_device:
 * e_parts is a device pointer (e.g. the output of an all-gather). */
int poslo_gpu_agg_ekeys_partial(poslo_gpu_ctx* ctx, const poslo_batch* batch, uint8_t* d_e_part, poslo_error* err);
/* The e-hat-independent half of a later combine_check with the same (y, s_hat,
 * r_hat) -- alpha^s-hat and the R-hat operand -- queued now on an internal
 * stream, so it overlaps the caller's agg_ekeys_partial and the all-gather
 * and combine_check is left with the fold and the Y^e-hat half. Optional: a
 * combine_check with other inputs (or without a prepare) computes it inline. */
int poslo_gpu_combine_check_prepare(poslo_gpu_ctx* ctx, const uint8_t y[32], const uint8_t s_hat[32],
                                    const uint8_t r_hat[32], poslo_error* err);
int poslo_gpu_combine_check(poslo_gpu_ctx* ctx, uint32_t n_parts, const uint8_t* e_parts, int32_t parts_on_device,
                            const uint8_t y[32], const uint8_t s_hat[32], const uint8_t r_hat[32], uint8_t* verdict,
                            poslo_error* err);

/* ---- group operation counters (group.hpp:86-97 GroupOpCounts) ------------------
 * Process-wide counts of the group operations the device performed, in the
 * reference's units: double_exp = commit_check evaluations (one per checked
 * group: 1 per coarse paver, n per per-epoch batch), exp_base = fixed-base
 * exponentiations (kg commitments), exp_var = 0 (never used on the path),
 * combine = group_combine folds of caller-supplied points (one per folded
 * element, as the reference's fold from the identity counts them). Relaxed
 * atomics; out = {exp_base, exp_var, double_exp, combine}. */
void poslo_gpu_group_op_counts(uint64_t out[4]);
void poslo_gpu_reset_group_op_counts(void);

/* ---- per-epoch verification (distill_epoch verdicts, distiller.cpp:60-89) ---
 * verdicts[k] = (commit_check(Y, e~_k, s_hats[k]) == r_hats[k]) for every
 * queried epoch; e_tilde_out optional (n_epochs x 32 B). When the batch is
 * device_resident, s_hats / r_hats are device pointers too (scalars already
 * canonical: they were validated when the signatures were parsed). */
int poslo_gpu_epoch_verify(poslo_gpu_ctx* ctx, const poslo_batch* batch, const uint8_t y[32],
                           const uint8_t* s_hats, const uint8_t* r_hats, uint8_t* verdicts,
                           uint8_t* e_tilde_out, poslo_error* err);

/* ---- SeBVer (distiller.cpp:156-233) over a coarse CCD --------------------------
 * The batch holds the epochs SeBVer hashes (verify_range / the mode-I lookup
 * read no others), any ascending subset of the distilled epochs, n2 each;
 * seeds are derived only for them. A group's e-sum runs over the batch
 * epochs in its range that are not in the invalid list; an I record's epoch
 * must be in the batch (else FormatError "messages for invalid epoch missing").
 * invalid: n_invalid ascending epoch indices (CCD invalid list).
 * Mode V: v_s/v_r = CCD valid aggregate -> *v_bit.
 * Mode U: n_umb umbrella records (index u, s, r; width w = n1/n_u) -> u_bits.
 * Mode I: one bit per invalid record (s, r) -> i_bits.
 * Any output pointer may be NULL to skip that mode. */
int poslo_gpu_sebver(poslo_gpu_ctx* ctx, const poslo_batch* batch, const uint8_t y[32],
                     uint32_t n1, uint32_t n_u, const uint32_t* invalid, const uint8_t* invalid_s,
                     const uint8_t* invalid_r, uint32_t n_invalid, const uint8_t* v_s,
                     const uint8_t* v_r, uint8_t* v_bit, const uint32_t* umb_index,
                     const uint8_t* umb_s, const uint8_t* umb_r, uint32_t n_umb, uint8_t* u_bits,
                     uint8_t* i_bits, poslo_error* err);

/* ---- coarse distillation (ColdCryptoData::distill_epoch, distiller.cpp:60-89) ---
 * Batched: the batch holds consecutive epochs in stream order (n2 entries
 * each), usually with per-epoch seed stacks (batch->ds_offsets: each epoch
 * verified with its own signature's ds, as aver(pk, {i: msgs}, sig.s_hat,
 * nullopt, sig.ds) does). verdicts[k] = epoch k valid. The batch is cut
 * into n_seg segments [seg[g], seg[g+1]) of batch positions (the pieces of
 * umbrellas, distiller.cpp:82-88); per segment, over its VALID epochs only:
 * seg_s[g] = sum of s_hats mod l (Scalar::add fold, :48) and seg_r[g] = the
 * group_combine fold of r_hats (:49, identity = 32 zero bytes when none).
 * The running CCD state (valid/umbrella accumulators, invalid list, ds) is
 * the caller's; see paper_2506_08781_b200/distill.py. s_hats / r_hats are
 * device pointers when the batch is device_resident (as epoch_verify). */
int poslo_gpu_distill_coarse(poslo_gpu_ctx* ctx, const poslo_batch* batch, const uint8_t y[32],
                             const uint8_t* s_hats, const uint8_t* r_hats, const uint32_t* seg,
                             uint32_t n_seg, uint8_t* verdicts, uint8_t* seg_s, uint8_t* seg_r,
                             poslo_error* err);
/* The same with one more per-segment output (NULL to skip): seg_e[g] = sum of
 * e~ mod l over the segment's VALID epochs — the e-sum SeBVer mode U checks
 * against the umbrella record (distiller.cpp:156-179), so a sharded caller can
 * fold umbrella pieces of e, s and R-hat across shards without rehashing. */
int poslo_gpu_distill_coarse_ex(poslo_gpu_ctx* ctx, const poslo_batch* batch, const uint8_t y[32],
                                const uint8_t* s_hats, const uint8_t* r_hats, const uint32_t* seg,
                                uint32_t n_seg, uint8_t* verdicts, uint8_t* seg_s, uint8_t* seg_r,
                                uint8_t* seg_e, poslo_error* err);

/* One distill_epoch (distiller.cpp:60-89) in a single device round trip, for
 * callers that distil a stream epoch by epoch (the C++ ColdCryptoData
 * drop-in): the host-resident batch holds ONE epoch (n2 entries, verified
 * with the batch's ds = the epoch signature's stack); s_hat / r_hat its
 * signature scalar and commitment; acc_s / acc_r the running valid and
 * umbrella aggregates (2 x 32 B each: [valid, umbrella]). *verdict = aver's
 * result; out_s / out_r = the aggregates with (s_hat, r_hat) folded into
 * both when valid (Scalar::add, group_combine), unchanged otherwise. Errors
 * as agg_ekeys (SeedNotDisclosed, FormatError), StateError for a batch size
 * other than n2. */
int poslo_gpu_distill_step(poslo_gpu_ctx* ctx, const poslo_batch* batch, const uint8_t y[32],
                           const uint8_t s_hat[32], const uint8_t r_hat[32], const uint8_t acc_s[64],
                           const uint8_t acc_r[64], uint8_t* verdict, uint8_t out_s[64], uint8_t out_r[64],
                           poslo_error* err);

/* Masked segmented folds on the device: for g < n_seg, over items k in
 * [seg[g], seg[g+1]) with mask[k] != 0 (mask NULL = all): out_s[g] = sum of
 * scalars mod l and out_r[g] = group_combine fold of points. Either of
 * scalars/out_s or points/out_r may be NULL. */
int poslo_gpu_segfold(poslo_gpu_ctx* ctx, uint32_t n, const uint8_t* scalars, const uint8_t* points,
                      const uint8_t* mask, const uint32_t* seg, uint32_t n_seg, uint8_t* out_s,
                      uint8_t* out_r, poslo_error* err);

/* ---- scheme F (poslo_f.cpp:223-246, distiller.cpp:91-129) --------------------
 * Errors in entry order (the reference loops entries ascending): for entry t,
 * SeedNotDisclosed (err->epoch = its epoch) when its derived seed's stack
 * does not cover the epoch, then FormatError (suite 3, L > 31; err->epoch =
 * t). fine_scalars: e_out n x 32 B LE (hash_to_scalar(m_t, x_t)), e_sum the
 * sum mod l; either may be NULL. fine_verify: verdicts[t] =
 * (commit_check(Y, e_t, s[t]) == r[t]) — aver_f_single per entry / the
 * per-entry checks of distill_epoch_fine. aver_f_batch: *verdict =
 * (commit_check(Y, sum e_t, s) == r) with every seed derived (x_t =
 * onetime_seed(sr(ds, t / n2), t % n2)). */
int poslo_gpu_fine_scalars(poslo_gpu_ctx* ctx, const poslo_fine_batch* fb, uint8_t* e_out, uint8_t* e_sum,
                           poslo_error* err);
int poslo_gpu_fine_verify(poslo_gpu_ctx* ctx, const poslo_fine_batch* fb, const uint8_t y[32],
                          const uint8_t* s, const uint8_t* r, uint8_t* verdicts, poslo_error* err);
int poslo_gpu_aver_f_batch(poslo_gpu_ctx* ctx, const poslo_fine_batch* fb, const uint8_t y[32],
                           const uint8_t s[32], const uint8_t r[32], uint8_t* verdict, poslo_error* err);

/* ---- signer side: fixtures with the reference's own key derivation ----------
 * (PoslocSecretKey::kg / sig_epoch, poslo_c.cpp:91-134)
 * kg_commitments: for each of the n epochs, r-hat_i = sum over j < n2 of
 * nonce_to_scalar(suite, r_seed, i, j) (primitives.cpp:195-207) and the
 * public commitment R-hat_i = alpha^r-hat_i; r_hats_out n x 32 B
 * (ristretto255), r_scalars_out n x 32 B LE or NULL.
 * sig_epochs: s-hat for every epoch of the batch, = sum_j (r_ij - e_ij y)
 * = r-hat_i - y e~_i mod l (e~ through the verifier's own hashing of the
 * batch; the batch's ds must disclose every epoch — the signer's root node
 * does). y: the secret scalar, 32 B LE. */
int poslo_gpu_kg_commitments(poslo_gpu_ctx* ctx, uint8_t suite, const uint8_t r_seed[16], const uint32_t* epochs,
                             uint32_t n, uint32_t n2, uint8_t* r_hats_out, uint8_t* r_scalars_out,
                             poslo_error* err);
int poslo_gpu_sig_epochs(poslo_gpu_ctx* ctx, const poslo_batch* batch, const uint8_t r_seed[16],
                         const uint8_t y[32], uint8_t* s_hats_out, poslo_error* err);

/* ---- group primitives (group.cpp), batched on the device ----------------------
 * commit_check: out[i] = encode(Y^e[i] * alpha^s[i]) (group.cpp:144-167).
 * Y = identity gives exp_base. */
int poslo_gpu_commit_check(poslo_gpu_ctx* ctx, uint32_t n, const uint8_t y[32], const uint8_t* e,
                           const uint8_t* s, uint8_t* out, poslo_error* err);
/* group_combine fold of n points (agg_elements, poslo_c.cpp:170-174). */
int poslo_gpu_group_fold(poslo_gpu_ctx* ctx, uint64_t n, const uint8_t* pts, uint8_t out[32],
                         poslo_error* err);
/* GroupElement::from_bytes validity (group.cpp:107-114): ok[i] in {0,1}. */
int poslo_gpu_point_valid(poslo_gpu_ctx* ctx, uint32_t n, const uint8_t* pts, uint8_t* ok,
                          poslo_error* err);

/* Batched check: verdicts[i] = (commit_check(Y, e[i], s[i]) == r[i]) — the
 * final step of paver (batch_verify.cpp:86), used for multi-GPU combines. */
int poslo_gpu_group_check(poslo_gpu_ctx* ctx, uint32_t n, const uint8_t y[32], const uint8_t* e,
                          const uint8_t* s, const uint8_t* r, uint8_t* verdicts, poslo_error* err);
/* out = sum of n scalars mod l (Scalar::add fold, batch_verify.cpp:84-85);
 * used to fold per-shard partial e-hat in rank order. */
int poslo_gpu_scalar_sum(poslo_gpu_ctx* ctx, uint64_t n, const uint8_t* scalars, uint8_t out[32],
                         poslo_error* err);

/* ---- stage-level entry points (parity/debug) ----------------------------------
 * sr (seed_manager.cpp:71-85) for each epoch: x0_out n x 16 B. */
int poslo_gpu_seed_retrieve(poslo_gpu_ctx* ctx, uint8_t suite, const uint8_t* ds, uint32_t ds_len,
                            uint32_t ds_capacity, const uint32_t* epochs, uint32_t n,
                            uint8_t* x0_out, poslo_error* err);
/* Per-entry e = hash_to_scalar(m, onetime_seed(x0, j)) mod l for every entry
 * of the batch (n_entries x 32 B LE), through the generic device path. */
int poslo_gpu_entry_scalars(poslo_gpu_ctx* ctx, const poslo_batch* batch, uint8_t* e_out,
                            poslo_error* err);

/* Counter-based synthetic log (include/poslo_synth.h) written to device
 * memory d_out: entries [first, first + n) of entry_len bytes each. Bench and
 * fixture tooling; byte-identical to the CPU harness's generator. */
int poslo_gpu_synth_log(poslo_gpu_ctx* ctx, uint64_t seed, uint64_t first, uint64_t n,
                        uint32_t entry_len, void* d_out, poslo_error* err);

/* Variable-length printable synthetic log ("syslog-style", BASELINE config 4):
 * entry first + t gets bytes poslo_synth_ascii(seed, first + t, b) at
 * d_out[d_offsets[t] .. d_offsets[t+1]) (lengths from poslo_synth_varlen). */
int poslo_gpu_synth_varlog(poslo_gpu_ctx* ctx, uint64_t seed, uint64_t first, uint64_t n,
                           const uint64_t* d_offsets, void* d_out, poslo_error* err);

#ifdef __cplusplus
}
#endif
#endif /* POSLO_GPU_H */
