// Internal: the device context behind the C-ABI handle (include/poslo_gpu.h).
// Shared by capi.cu (single-device calls) and multi.cu (multi-device
// contexts: one member context per device, epoch shards per member).
#pragma once
#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <vector>

#include "../../include/poslo_gpu.h"

namespace poslo_gpu_detail {

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
};

}  // namespace poslo_gpu_detail
using poslo_gpu_detail::DevBuf;

struct PinnedStage {  // pinned host landing zone for the per-call small D2H copies
    unsigned long long err_key;
    unsigned long long err_init;  // H2D: error word seeded with host-detected seed failures
    int flags[4];
    uint8_t verdict;
    unsigned long long scan[3];  // raw-image scan state {next record, records so far} + sentinel
    uint8_t step_out[128];       // poslo_gpu_distill_step: the two updated (s, R) pairs
};

struct poslo_gpu_ctx {
    int device = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    cudaStream_t copy = nullptr;  // H2D of host-resident logs, overlapped with hashing
    cudaStream_t side = nullptr;  // e-hat-independent part of the group check, overlapped with hashing
    cudaEvent_t ev_side[2] = {};
    // combine_check_prepare: the e-hat-independent half of the next
    // combine_check (alpha^s-hat, R-hat decode) queued on `side`, keyed by its inputs
    bool pre_valid = false;
    uint8_t pre_key[96] = {};
    cudaEvent_t ev_pre = nullptr;
    cudaStream_t hash2 = nullptr;  // second hash stream: epoch pieces alternate so one piece's tail
    cudaEvent_t ev_hash[2] = {};   // overlaps the next piece instead of idling at a kernel boundary
    std::vector<cudaEvent_t> chunk_ev;
    std::mutex mtx;
    uint32_t* d_t0 = nullptr;
    DevBuf b_epochs, b_x0, b_partial, b_etilde, b_sum, b_scratch, b_tiles, b_starts, b_tbegin,
        b_err, b_flags, b_payload, b_offsets, b_e, b_s, b_r, b_enc, b_verdict, b_mask, b_seg,
        b_y, b_pts, b_foldscratch, b_rhat, b_pre, b_starts_ds, b_seg32, b_out_s, b_out_r, b_dpts, b_dok, b_scan_exit, b_scan_cnt, b_scan_start, b_scan_base, b_scan_off, b_scan_state, b_seg_e, b_out_e, b_ppre_s, b_ppre_r, b_ppre, b_scr16e;
    // fixed-base comb tables: generator (built once) and the last Y seen
    void* d_tabB = nullptr;
    void* d_tabY = nullptr;
    void* d_tabB256 = nullptr;  // radix-256 combs for batched checks (built on first use)
    void* d_tabY256 = nullptr;
    void* d_pk = nullptr;          // 64 powers 16^i P of the last point P tables were built for
    int pk_owner = 0;              // whose powers d_pk holds: 0 none, 1 the generator, 2 Y = pk_key
    uint8_t pk_key[32] = {};
    uint8_t tabY_key[32] = {};
    bool tabY_valid = false;
    uint8_t tabY256_key[32] = {};
    bool tabY256_valid = false;
    void* d_tabB16 = nullptr;  // radix-2^16 combs (60 MiB each) for large check batches
    void* d_tabY16 = nullptr;
    uint8_t tabY16_key[32] = {};
    bool tabY16_valid = false;
    PinnedStage* stage = nullptr;
    bool timing = false;
    cudaEvent_t ev[7] = {};
    float last_ms[6] = {};
    uint32_t launches = 0;
    // pinned staging ring for poslo_batch.fill producers (allocated on first use)
    static constexpr int kFillSlots = 3;
    uint8_t* fill_slot[kFillSlots] = {};
    size_t fill_cap = 0;
    cudaEvent_t fill_ev[kFillSlots] = {};
    // group-operation counting (poslo_gpu_group_op_counts); off while a
    // multi-device context folds its members' partial results
    bool count_ops = true;
    // multi-device context: one member per device; empty for a single device
    std::vector<poslo_gpu_ctx*> members;
};

// Process-wide group-operation counters (group.hpp:86-97 units).
namespace poslo_gpu_detail {
enum { kOpExpBase = 0, kOpExpVar = 1, kOpDoubleExp = 2, kOpCombine = 3 };
void count_op(const poslo_gpu_ctx* ctx, int which, uint64_t n);

// Multi-device contexts (multi.cu): shard the batch over the members and
// combine on member 0; called by the public entry points when ctx->members
// is not empty.
int multi_agg_ekeys(poslo_gpu_ctx* ctx, const poslo_batch* b, uint8_t* e_tilde_out, uint8_t* e_hat_out,
                    poslo_error* err);
int multi_paver(poslo_gpu_ctx* ctx, const poslo_batch* b, const uint8_t y[32], const uint8_t s_hat[32],
                const uint8_t* r_hat_agg, const uint8_t* r_hats, uint8_t* verdict, poslo_error* err);
int multi_epoch_verify(poslo_gpu_ctx* ctx, const poslo_batch* b, const uint8_t y[32], const uint8_t* s_hats,
                       const uint8_t* r_hats, uint8_t* verdicts, uint8_t* e_tilde_out, poslo_error* err);
int multi_distill_coarse(poslo_gpu_ctx* ctx, const poslo_batch* b, const uint8_t y[32], const uint8_t* s_hats,
                         const uint8_t* r_hats, const uint32_t* seg, uint32_t n_seg, uint8_t* verdicts,
                         uint8_t* seg_s, uint8_t* seg_r, uint8_t* seg_e, poslo_error* err);
}  // namespace poslo_gpu_detail
using poslo_gpu_detail::multi_agg_ekeys;
using poslo_gpu_detail::multi_distill_coarse;
using poslo_gpu_detail::multi_epoch_verify;
using poslo_gpu_detail::multi_paver;

