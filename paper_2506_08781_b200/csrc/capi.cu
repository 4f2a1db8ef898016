// C-ABI of the B200 batch verifier (include/poslo_gpu.h).
//
// Host orchestration of one verification call on the context's stream:
//   validate + parse ds (SeedStack wire, seed_manager.cpp:41-53)
//   -> [H2D of the packed log when it is host-resident]
//   -> K0 seed_derive -> K1+K2 hash/segmented sum -> epoch finalize
//   -> sum mod l (e-hat) / R-hat fold -> K3 group check -> D2H of verdicts.
// Errors follow the reference's taxonomy and order; the
// lowest offending epoch wins, seed retrieval before hashing.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <atomic>
#include <condition_variable>
#include <functional>
#include <mutex>
#include <thread>
#include <type_traits>
#include <vector>

#include "../../include/poslo_gpu.h"
#include "aes128.cuh"
#include "poslo_internal.h"

using namespace poslo_gpu;

#include "capi_ctx.h"

extern "C" {  // defined with the batched-check entry points below
static int start_decode(poslo_gpu_ctx* ctx, uint32_t n, const uint8_t* d_r, void** d_pts, uint8_t** d_ok,
                        poslo_error* err);
// Scratch of the square-root-free radix-2^16 checks (launch_check16e): the
// points P = e Y + s B of every check, 1 / u2 and the inversion's prefixes.
struct Scr16e {
    uint8_t* P = nullptr;
    uint8_t* u2 = nullptr;
    uint8_t* pre = nullptr;
    explicit operator bool() const { return P != nullptr; }
    Scr16e at(uint32_t e0) const {  // the checks of epochs e0 ..
        if (!P) return Scr16e{};
        return Scr16e{P + kGptBytes * (size_t)e0, u2 + kFeBytes * (size_t)e0, pre + kFeBytes * (size_t)e0};
    }
};
static int split_checks(poslo_gpu_ctx* ctx, uint32_t n, const uint32_t* d_e, const uint32_t* d_s, const uint8_t* d_r,
                        const void* d_pts, const uint8_t* d_ok, uint8_t* d_verdict, poslo_error* err,
                        const Scr16e& scr = Scr16e{});
static int ensure_scr16e(poslo_gpu_ctx* ctx, uint32_t n, Scr16e& out, poslo_error* err);
}

namespace {

constexpr uint64_t kChunkBytes = 64ull << 20;
constexpr uint32_t kPipePieces = 8;  // epoch pieces when per-epoch checks overlap hashing
// POSLO_PIPE_PIECES overrides it (tuning; 1 = hash everything, then check)
uint32_t pipe_pieces() {
    static const uint32_t v = [] {
        const char* e = std::getenv("POSLO_PIPE_PIECES");
        return e ? (uint32_t)std::max(1, std::atoi(e)) : kPipePieces;
    }();
    return v;
}
constexpr uint32_t kPipeMinTiles = 2048;  // hash CTAs per piece: > 2 waves of 148 SMs x 5-6 CTAs
constexpr int kEvSeed = 0, kEvHash = 1, kEvFin = 2, kEvSum = 3, kEvGroup = 4, kEvEnd = 5;

int set_err(poslo_error* err, int code, uint32_t epoch, const char* fmt, ...) {
    if (err) {
        err->code = code;
        err->epoch = epoch;
        va_list ap;
        va_start(ap, fmt);
        vsnprintf(err->message, sizeof err->message, fmt, ap);
        va_end(ap);
    }
    return code;
}

std::atomic<uint64_t> g_ops[4];  // poslo_gpu_group_op_counts

int ok(poslo_error* err) {
    if (err) {
        err->code = POSLO_OK;
        err->epoch = 0;
        err->message[0] = 0;
    }
    return POSLO_OK;
}

#define CU(call)                                                                            \
    do {                                                                                    \
        cudaError_t e_ = (call);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return set_err(err, POSLO_CUDA_ERROR, 0, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

template <class T>
constexpr size_t elem_bytes() {  // void buffers are counted in bytes
    if constexpr (std::is_void<T>::value) return 1;
    else return sizeof(T);
}

template <class T>
int ensure(DevBuf& b, size_t count, T** out, poslo_error* err) {
    size_t bytes = std::max<size_t>(count * elem_bytes<T>(), 16);
    if (b.cap < bytes) {
        size_t want = std::max(bytes, b.cap * 3 / 2);
        if (b.p) cudaFree(b.p);
        b.p = nullptr;
        b.cap = 0;
        CU(cudaMalloc(&b.p, want));
        b.cap = want;
    }
    *out = static_cast<T*>(b.p);
    return POSLO_OK;
}

#define ENSURE(buf, n, ptr)                                  \
    do {                                                     \
        int rc_ = ensure(ctx->buf, (n), &(ptr), err);        \
        if (rc_) return rc_;                                 \
    } while (0)

void mark(poslo_gpu_ctx* ctx, int i) {
    if (ctx->timing) cudaEventRecord(ctx->ev[i], ctx->stream);
}

// SeedStack::deserialize + push invariants (seed_manager.cpp:18-23, 41-53).
int parse_ds(const uint8_t* w, uint32_t n, uint32_t cap, DsParam& ds, poslo_error* err) {
    if (!w || n < 1) return set_err(err, POSLO_FORMAT_ERROR, 0, "truncated input");
    uint32_t count = w[0];
    size_t off = 1;
    ds.count = 0;
    for (uint32_t k = 0; k < count; k++) {
        if (n - off < 21) return set_err(err, POSLO_FORMAT_ERROR, 0, "truncated input");
        if (k >= cap) return set_err(err, POSLO_STATE_ERROR, 0, "seed stack overflow");
        if (k >= 32) return set_err(err, POSLO_FORMAT_ERROR, 0, "seed stack deeper than 32");
        DsNode& nd = ds.nodes[k];
        nd.depth = w[off];
        nd.index = (uint32_t)w[off + 1] << 24 | (uint32_t)w[off + 2] << 16 | (uint32_t)w[off + 3] << 8 | w[off + 4];
        std::memcpy(nd.value, w + off + 5, 16);
        if (k > 0 && ds.nodes[k - 1].depth <= nd.depth)
            return set_err(err, POSLO_STATE_ERROR, 0, "seed stack depth order violated");
        if (nd.depth > 32) return set_err(err, POSLO_FORMAT_ERROR, 0, "seed node depth out of range");
        ds.count = (int)k + 1;
        off += 21;
    }
    return POSLO_OK;
}

// sr (seed_manager.cpp:71-85) resolved on the host for per-epoch stacks:
// for every queried epoch, its covering node in its own stack (ds_offsets,
// or the one stack `ds` when ds_offsets == NULL). Undisclosed epochs get a
// zero start and lower *host_err to (k << 1) (or (first_entry[k] << 1)).
int resolve_seed_starts(const uint8_t* ds_w, uint32_t ds_len, const uint64_t* ds_offsets, uint32_t cap,
                        const uint32_t* epochs, uint32_t n, std::vector<SeedStart>& starts,
                        const uint64_t* first_entry, unsigned long long* host_err, poslo_error* err) {
    starts.resize(n);
    DsParam ds;
    if (!ds_offsets) {
        int rc = parse_ds(ds_w, ds_len, cap, ds, err);
        if (rc) return rc;
    }
    for (uint32_t k = 0; k < n; k++) {
        if (ds_offsets) {
            const uint64_t o0 = ds_offsets[k], o1 = ds_offsets[k + 1];
            if (o1 < o0 || o1 > ds_len) return set_err(err, POSLO_INVALID_ARGUMENT, epochs[k], "bad ds_offsets");
            int rc = parse_ds(ds_w + o0, (uint32_t)(o1 - o0), cap, ds, err);
            if (rc) {
                if (err) err->epoch = epochs[k];
                return rc;
            }
        }
        const uint32_t q = epochs[k];
        int c = -1;
        for (int i = ds.count - 1; i >= 0; i--) {
            const uint64_t lo = (uint64_t)ds.nodes[i].index << ds.nodes[i].depth;
            const uint64_t hi = (uint64_t)(uint32_t)(ds.nodes[i].index + 1u) << ds.nodes[i].depth;
            if (q >= hi && i == ds.count - 1) break;
            if (q >= lo && q < hi) {
                c = i;
                break;
            }
        }
        SeedStart& st = starts[k];
        if (c < 0) {  // SeedNotDisclosed, ordered before the hashing errors of the same position
            std::memset(&st, 0, sizeof st);
            const unsigned long long pos = first_entry ? first_entry[k] : k;
            *host_err = std::min<unsigned long long>(*host_err, pos << 1);
            continue;
        }
        std::memcpy(st.value, ds.nodes[c].value, 16);
        st.rel = q - (uint32_t)((uint64_t)ds.nodes[c].index << ds.nodes[c].depth);
        st.depth = ds.nodes[c].depth;
    }
    return POSLO_OK;
}

struct Prepared {
    EntryLayout lay{};
    TileMap tm{};
    bool fast = false;
    bool uniform = false;
    bool want_etilde = true;        // false: only e-hat is needed (paver, agg_ekeys without e~ out)
    uint32_t* d_etilde = nullptr;   // per-epoch e~ (8 limbs), valid when want_etilde
    const uint32_t* sum_src = nullptr;  // what e-hat sums: e~ (8 limbs) or raw epoch sums (17 limbs)
    int sum_limbs = 8;
    // Pipelining hook: when set (and the log is device-resident), the hash is
    // launched in epoch pieces and on_piece(e0, e1, st) runs after each piece's
    // e~ are final on stream st, so the caller can start its per-epoch
    // checks for that piece while the next one hashes.
    std::function<int(uint32_t, uint32_t, cudaStream_t)> on_piece;
    // Runs right after the seed kernel is queued, before any hashing: a side-
    // stream job queued here (the R-hat decode) starts behind the seeds and
    // runs beside the hashing instead of delaying the seeds and the first
    // hash CTAs.
    std::function<int()> on_seeded;
};

// Entries per tile of the generic / variable-length kernels (<= 1024, the
// kernels' sort buffer). POSLO_VAR_TILE overrides for experiments.
uint32_t var_tile_entries() {
    static const uint32_t te = [] {
        const char* e = std::getenv("POSLO_VAR_TILE");
        uint32_t v = e ? (uint32_t)std::atoi(e) : 1024u;
        return (v >= 128 && v <= 1024) ? v : 1024u;
    }();
    return te;
}

bool is_uniform(const poslo_batch* b) {
    if (!b->epoch_starts) return true;
    for (uint32_t k = 0; k <= b->n_epochs; k++)
        if (b->epoch_starts[k] != (uint64_t)k * b->n2) return false;
    return true;
}

// A device_resident batch must hand the kernels memory they can read:
// device or managed memory, or registered (pinned, mapped) host memory.
// Plain pageable host memory would fault inside a kernel and leave the
// context unusable, so it is rejected up front.
bool device_readable(const void* p) {
    if (!p) return true;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();  // clear the sticky-free error of the query
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged ||
           (a.type == cudaMemoryTypeHost && a.devicePointer != nullptr);
}

// Plain pageable host memory (not registered with CUDA): a DMA from it is
// staged by the driver synchronously, chunk by chunk, at a fraction of the
// link rate, so run_hash stages such logs itself (parallel host copies into
// the pinned ring, the DMA of chunk c overlapping the copy of chunk c + 1).
bool host_pageable(const void* p) {
    if (!p) return false;
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return true;
    }
    return a.type == cudaMemoryTypeUnregistered;
}

// Persistent host workers for copy_parallel (one copy at a time per process;
// concurrent callers serialise on the pool, each copy still runs on every core).
class HostCopyPool {
public:
    static HostCopyPool& get() {
        // never destroyed: the detached workers may still wait on cv_ at exit
        static HostCopyPool* p = new HostCopyPool();
        return *p;
    }
    void copy(uint8_t* dst, const uint8_t* src, size_t bytes) {
        const size_t T = th_.size() + 1;
        if (bytes < (4u << 20) || T == 1) {
            std::memcpy(dst, src, bytes);
            return;
        }
        std::lock_guard<std::mutex> one(call_);
        {
            std::lock_guard<std::mutex> lk(m_);
            dst_ = dst;
            src_ = src;
            bytes_ = bytes;
            parts_ = T;
            next_.store(0);
            busy_ = (int)th_.size();
            gen_++;
        }
        cv_.notify_all();
        run();
        std::unique_lock<std::mutex> lk(m_);
        done_.wait(lk, [this] { return busy_ == 0; });
    }

private:
    HostCopyPool() {
        const unsigned n = std::min(std::max(1u, std::thread::hardware_concurrency()), 64u) - 1;
        for (unsigned i = 0; i < n; i++) th_.emplace_back([this] { work(); });
        for (auto& t : th_) t.detach();  // process lifetime: never joined at exit
    }
    void run() {
        for (size_t k = next_.fetch_add(1); k < parts_; k = next_.fetch_add(1)) {
            const size_t a = bytes_ * k / parts_, z = bytes_ * (k + 1) / parts_;
            std::memcpy(dst_ + a, src_ + a, z - a);
        }
    }
    void work() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return gen_ != seen; });
                seen = gen_;
            }
            run();
            std::lock_guard<std::mutex> lk(m_);
            if (--busy_ == 0) done_.notify_one();
        }
    }
    std::vector<std::thread> th_;
    std::mutex m_, call_;
    std::condition_variable cv_, done_;
    uint8_t* dst_ = nullptr;
    const uint8_t* src_ = nullptr;
    size_t bytes_ = 0, parts_ = 0;
    std::atomic<size_t> next_{0};
    int busy_ = 0;
    uint64_t gen_ = 0;
};

// After the whole raw image is scanned: read_log's FormatError on a
// truncated record, epochs_of's on a count that is not a nonzero multiple of
// n2 (tools/poslo.cpp:32-40), and the batch must name exactly that many
// epochs; then offsets[n] = image length (the record-end sentinel).
int raw_scan_result(poslo_gpu_ctx* ctx, const poslo_batch* b, uint64_t n_entries,
                    const unsigned long long* d_state, uint64_t* d_off, cudaStream_t s, poslo_error* err) {
    CU(cudaMemcpyAsync(ctx->stage->scan, d_state, 16, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    const unsigned long long q = ctx->stage->scan[0], total = ctx->stage->scan[1];
    if (q == ~0ull) return set_err(err, POSLO_FORMAT_ERROR, 0, "truncated log record");
    if (total == 0 || total % b->n2) return set_err(err, POSLO_FORMAT_ERROR, 0, "record count must be a nonzero multiple of n2");
    if (total != n_entries)
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "log holds %llu epochs, the batch names %u",
                       (unsigned long long)(total / b->n2), b->n_epochs);
    ctx->stage->scan[2] = b->payload_bytes;
    CU(cudaMemcpyAsync(d_off + total, &ctx->stage->scan[2], 8, cudaMemcpyHostToDevice, s));
    return POSLO_OK;
}

// Stages 0-2 for a batch: leaves per-epoch e~ (8 limbs each) in
// ctx->b_etilde and returns the status after reading the error word.
int run_hash(poslo_gpu_ctx* ctx, const poslo_batch* b, Prepared& P, poslo_error* err) {
    if (!b) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null batch");
    if (b->suite < 1 || b->suite > 3) return set_err(err, POSLO_FORMAT_ERROR, 0, "unknown suite id");
    if (b->n_epochs && !b->epochs) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null epochs");
    // (the strictly-ascending check of `epochs` runs on the host after the
    // kernels are queued, overlapping them; see the end of this function)
    DsParam ds;
    int rc = POSLO_OK;
    std::vector<SeedStart> starts;  // per-epoch stacks: resolved covering nodes
    unsigned long long host_err = ~0ull;
    if (b->ds_offsets) {
        rc = resolve_seed_starts(b->ds, b->ds_len, b->ds_offsets, b->ds_capacity, b->epochs, b->n_epochs, starts,
                                 nullptr, &host_err, err);
        if (rc) return rc;
    } else {
        rc = parse_ds(b->ds, b->ds_len, b->ds_capacity, ds, err);
        if (rc) return rc;
    }
    P.uniform = is_uniform(b);
    // Raw record image (record_header = 4, no offsets): the records are found
    // on the device (log_scan.cu) and, for a host image, the record scan and
    // the hashing run chunk by chunk behind the H2D copy.
    const bool raw_image = b->record_header == 4 && !b->offsets;
    if (raw_image && !P.uniform)
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "a raw record image needs uniform epochs of n2 records");
    uint64_t n_entries = P.uniform ? (uint64_t)b->n_epochs * b->n2 : b->epoch_starts[b->n_epochs];
    if (b->epoch_starts && b->epoch_starts[0] != 0)
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "epoch_starts[0] must be 0");
    if (n_entries > b->n_entries && !raw_image)
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "batch describes more entries than given");
    // a producer callback stands in for a host payload (poslo_batch.fill)
    const bool has_fill = b->fill && !b->payload && !b->device_resident;
    if (has_fill && raw_image)
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "a fill producer needs entry offsets or a fixed length");
    if (n_entries && !b->payload && !has_fill && !(b->offsets == nullptr && b->entry_len == 0))
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null payload");
    // layout bounds: the kernels read payload[offsets[t] + header .. offsets[t+1]) or
    // payload[t L .. (t+1) L); a batch whose layout leaves the payload is refused
    // before any copy or kernel touches it (host offsets: the ends here and the
    // monotonicity on the device below; device offsets: all on the device)
    if (!raw_image && !b->offsets && n_entries && (uint64_t)b->entry_len * n_entries > b->payload_bytes)
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "n_entries x entry_len exceeds payload_bytes");
    uint64_t off_lo = 0, off_hi = b->payload_bytes;  // byte span of the described entries
    if (!b->offsets && !raw_image) off_hi = (uint64_t)b->entry_len * n_entries;
    if (b->offsets && !b->device_resident) {
        off_lo = b->offsets[0];
        off_hi = b->offsets[n_entries];
        if (off_lo > off_hi || off_hi > b->payload_bytes)
            return set_err(err, POSLO_INVALID_ARGUMENT, 0, "entry offsets outside the payload");
    }

    cudaStream_t s = ctx->stream;
    uint32_t n_ep = b->n_epochs;
    uint32_t* d_epochs;
    uint4* d_x0;
    unsigned long long* d_err;
    ENSURE(b_epochs, n_ep, d_epochs);
    ENSURE(b_x0, n_ep, d_x0);
    ENSURE(b_err, 1, d_err);
    ENSURE(b_etilde, (size_t)n_ep * 8, P.d_etilde);

    // entry layout (H2D when host-resident). Large uniform fixed-length logs
    // stream in epoch-aligned 64 MiB chunks on the copy stream, each chunk's
    // hashing waiting only for its own bytes (SPEC.md:496 chunked streaming).
    P.lay.entry_len = b->entry_len;
    if (b->record_header != 0 && b->record_header != 4)
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "record_header must be 0 or 4");
    P.lay.header = b->record_header;
    const uint64_t epoch_bytes = (uint64_t)b->n2 * b->entry_len;
    // Host-resident uniform logs (fixed length, or byte offsets / raw record
    // images) stream in epoch-aligned chunks of <= 64 MiB on the copy stream.
    const bool chunked = !raw_image && !b->device_resident && P.uniform && (b->offsets || epoch_bytes > 0) &&
                         ((b->payload_bytes >= 2 * kChunkBytes && n_ep > 1) || (has_fill && n_ep > 0));
    const bool raw_chunked = raw_image && !b->device_resident && b->payload_bytes >= 2 * kChunkBytes && n_ep > 1;
    // a pageable host log goes through the pinned ring like a producer's chunks
    const bool stage_pageable = chunked && !has_fill && host_pageable(b->payload);
    const bool use_ring = has_fill || stage_pageable;
    auto epoch_byte = [&](uint32_t e) -> uint64_t {  // first payload byte of the e-th queried epoch
        return b->offsets ? b->offsets[(uint64_t)e * b->n2] : (uint64_t)e * epoch_bytes;
    };
    if (b->device_resident) {
        if ((b->payload_bytes && !device_readable(b->payload)) || !device_readable(b->offsets))
            return set_err(err, POSLO_INVALID_ARGUMENT, 0, "device_resident batch with a host pointer");
        P.lay.payload = b->payload;
        P.lay.offsets = b->offsets;
    } else {
        // only the described entries' bytes travel: [off_lo, off_hi) lands at
        // d_pay, and the kernels index it through the shifted base d_pay - off_lo
        // with the caller's absolute offsets (a sub-range of a larger log, e.g.
        // one shard of a multi-device call, copies only its own bytes)
        uint8_t* d_pay;
        const uint64_t span = off_hi - off_lo;
        ENSURE(b_payload, span, d_pay);
        if (span && !chunked && !raw_chunked) {
            if (has_fill) {
                const size_t need = (size_t)span;
                if (!ctx->fill_slot[0] || ctx->fill_cap < need) {
                    CU(cudaStreamSynchronize(s));
                    CU(cudaStreamSynchronize(ctx->copy));
                    for (auto& p : ctx->fill_slot)
                        if (p) {
                            cudaFreeHost(p);
                            p = nullptr;
                        }
                    ctx->fill_cap = 0;
                    for (auto& p : ctx->fill_slot) CU(cudaMallocHost(&p, need));
                    ctx->fill_cap = need;
                }
                CU(cudaEventSynchronize(ctx->fill_ev[0]));
                if (b->fill(b->fill_user, 0, n_entries, ctx->fill_slot[0]) != 0)
                    return set_err(err, POSLO_INVALID_ARGUMENT, 0, "fill producer failed");
                CU(cudaMemcpyAsync(d_pay, ctx->fill_slot[0], span, cudaMemcpyHostToDevice, s));
                CU(cudaEventRecord(ctx->fill_ev[0], s));
            } else {
                CU(cudaMemcpyAsync(d_pay, b->payload + off_lo, span, cudaMemcpyHostToDevice, s));
            }
        }
        P.lay.payload = d_pay - off_lo;
        P.lay.offsets = nullptr;
        if (b->offsets) {
            uint64_t* d_off;
            ENSURE(b_offsets, n_entries + 1, d_off);
            CU(cudaMemcpyAsync(d_off, b->offsets, (n_entries + 1) * 8, cudaMemcpyHostToDevice, s));
            P.lay.offsets = d_off;
        }
    }
    // offsets must be non-decreasing with room for each record header and stay
    // inside [off_lo, off_hi] (device-resident: inside the payload), checked on
    // the device before the first hashing kernel reads through them
    if (P.lay.offsets && !raw_image && n_entries) {
        int* d_bad;
        ENSURE(b_flags, 4, d_bad);
        CU(cudaMemsetAsync(d_bad, 0, 16, s));
        launch_check_offsets(P.lay.offsets, n_entries, b->record_header, off_lo, off_hi, d_bad, s);
        ctx->launches += 1;
        CU(cudaMemcpyAsync(ctx->stage->flags, d_bad, 4, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        if (ctx->stage->flags[0])
            return set_err(err, POSLO_INVALID_ARGUMENT, 0, "entry offsets not ascending or outside the payload");
    }

    // raw image: record offsets found on the device
    // record chunks: 1 MiB for a one-shot scan, kRawScanChunk when pipelined
    // (exits then only for one copy chunk's worth of record chunks at a time)
    const uint64_t scan_chunk = raw_chunked ? kRawScanChunk : kScanChunk;
    const uint32_t n_scan = (uint32_t)((b->payload_bytes + scan_chunk - 1) / scan_chunk);
    const uint32_t exit_chunks = raw_chunked ? (uint32_t)(kChunkBytes / kRawScanChunk) : n_scan;
    uint64_t *d_sc_exit = nullptr, *d_sc_start = nullptr, *d_sc_base = nullptr;
    uint32_t* d_sc_cnt = nullptr;
    unsigned long long* d_sc_state = nullptr;
    if (raw_image) {
        uint64_t* d_off;
        ENSURE(b_scan_off, n_entries + 1, d_off);
        ENSURE(b_scan_exit, (size_t)std::max<uint32_t>(exit_chunks, 1) * kScanWindow, d_sc_exit);
        ENSURE(b_scan_cnt, (size_t)std::max<uint32_t>(exit_chunks, 1) * kScanWindow, d_sc_cnt);
        ENSURE(b_scan_start, std::max<uint32_t>(n_scan, 1), d_sc_start);
        ENSURE(b_scan_base, std::max<uint32_t>(n_scan, 1), d_sc_base);
        ENSURE(b_scan_state, 2, d_sc_state);
        CU(cudaMemsetAsync(d_sc_state, 0, 16, s));
        P.lay.offsets = d_off;
        if (!raw_chunked) {
            launch_log_scan_range(P.lay.payload, b->payload_bytes, 0, n_scan, scan_chunk, d_sc_exit, d_sc_cnt,
                                  d_sc_start, d_sc_base, d_sc_state, d_off, n_entries + 1, s);
            ctx->launches += 3;
            int rc2 = raw_scan_result(ctx, b, n_entries, d_sc_state, d_off, s, err);
            if (rc2) return rc2;
        }
    }

    mark(ctx, kEvSeed);
    ctx->stage->err_init = host_err;
    CU(cudaMemcpyAsync(d_err, &ctx->stage->err_init, 8, cudaMemcpyHostToDevice, s));
    // a contiguous epoch range (every full verification) needs no list upload;
    // with the ascending check below, last - first == n - 1 proves contiguity
    const bool contiguous = n_ep > 0 && b->epochs[n_ep - 1] - b->epochs[0] == n_ep - 1;
    if (n_ep && !contiguous) CU(cudaMemcpyAsync(d_epochs, b->epochs, (size_t)n_ep * 4, cudaMemcpyHostToDevice, s));
    if (b->ds_offsets) {
        SeedStart* d_starts;
        ENSURE(b_starts_ds, std::max<size_t>(starts.size(), 1), d_starts);
        if (n_ep) CU(cudaMemcpyAsync(d_starts, starts.data(), starts.size() * sizeof(SeedStart),
                                     cudaMemcpyHostToDevice, s));
        CU(cudaStreamSynchronize(s));  // `starts` is a host vector
        launch_seed_walk(b->suite, d_starts, n_ep, d_x0, ctx->d_t0, s);
    } else {
        launch_seed_derive(b->suite, ds, contiguous ? nullptr : d_epochs, n_ep ? b->epochs[0] : 0, n_ep, d_x0, d_err,
                           ctx->d_t0, s);
    }
    ctx->launches += n_ep ? 1 : 0;
    if (P.on_seeded) {
        rc = P.on_seeded();
        if (rc) return rc;
    }
    mark(ctx, kEvHash);

    // tiles
    TileMap& tm = P.tm;
    tm.n_epochs = n_ep;
    tm.n2 = b->n2;
    bool aligned = ((uintptr_t)P.lay.payload & 15) == 0;
    P.fast = !raw_image && P.uniform && !b->offsets && b->entry_len == 32 && (b->suite == 1 || b->suite == 2) &&
             aligned;
    uint32_t* d_partial = nullptr;
    if (P.uniform) {
        if (P.fast && b->suite == 1 && b->n2 <= kLeanMaxN2)
            tm.tile_entries = std::max<uint32_t>(b->n2, 1);  // one tile per epoch (lean kernel)
        else if (P.fast)
            tm.tile_entries = b->n2 <= 128 ? 128 : (b->n2 <= 256 ? 256 : 1024);
        else
            tm.tile_entries = var_tile_entries();
        tm.tiles_per_epoch = b->n2 ? (b->n2 + tm.tile_entries - 1) / tm.tile_entries : 0;
        tm.n_tiles = n_ep * tm.tiles_per_epoch;
    } else {
        std::vector<uint4> tiles;
        std::vector<uint32_t> tbegin(n_ep + 1);
        const uint32_t te = var_tile_entries();
        for (uint32_t k = 0; k < n_ep; k++) {
            tbegin[k] = (uint32_t)tiles.size();
            uint64_t cnt = b->epoch_starts[k + 1] - b->epoch_starts[k];
            if (b->epoch_starts[k + 1] < b->epoch_starts[k])
                return set_err(err, POSLO_INVALID_ARGUMENT, 0, "epoch_starts must be non-decreasing");
            for (uint64_t j0 = 0; j0 < cnt; j0 += te)
                tiles.push_back(make_uint4(k, (uint32_t)j0, (uint32_t)std::min<uint64_t>(te, cnt - j0), 0));
        }
        tbegin[n_ep] = (uint32_t)tiles.size();
        uint4* d_tiles;
        uint64_t* d_starts;
        uint32_t* d_tb;
        ENSURE(b_tiles, tiles.size(), d_tiles);
        ENSURE(b_starts, n_ep + 1, d_starts);
        ENSURE(b_tbegin, n_ep + 1, d_tb);
        if (!tiles.empty()) CU(cudaMemcpyAsync(d_tiles, tiles.data(), tiles.size() * sizeof(uint4), cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(d_starts, b->epoch_starts, (n_ep + 1) * 8, cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(d_tb, tbegin.data(), (n_ep + 1) * 4, cudaMemcpyHostToDevice, s));
        CU(cudaStreamSynchronize(s));  // host vectors go out of scope
        tm.tiles = d_tiles;
        tm.epoch_starts = d_starts;
        tm.epoch_tile_begin = d_tb;
        tm.n_tiles = (uint32_t)tiles.size();
    }
    ENSURE(b_partial, (size_t)std::max<uint32_t>(tm.n_tiles, 1) * 17, d_partial);
    // The lean suite-1 kernel leaves each epoch's raw 544-bit digest sum in
    // d_partial; the mod-l reduction to e~ is a separate full-warp kernel, and
    // is skipped when only e-hat is wanted (sum of raw sums, reduced once;
    // exact while the batch has < 2^32 entries, so 17 limbs cannot overflow).
    const bool lean = P.fast && b->suite == 1 && tm.tiles_per_epoch == 1 && b->n2 <= kLeanMaxN2;
    bool need_finalize = P.fast ? (tm.tiles_per_epoch != 1 || lean) : true;
    P.sum_src = P.d_etilde;
    P.sum_limbs = 8;
    if (lean && !P.want_etilde && n_entries < (1ull << 32)) {
        need_finalize = false;
        P.sum_src = d_partial;
        P.sum_limbs = 17;
    }
    auto launch_hash = [&](const TileMap& t, cudaStream_t hs) {
        if (P.fast) {
            if (b->suite == 1)
                launch_hash_s1_l32(P.lay, t, d_x0, d_partial, P.d_etilde, hs);
            else
                launch_hash_s2_l32(P.lay, t, d_x0, d_partial, P.d_etilde, ctx->d_t0, hs);
        } else if (b->suite == 1) {
            launch_hash_s1_var(P.lay, t, d_x0, d_partial, hs);
        } else {
            launch_hash_generic(b->suite, P.lay, t, d_x0, d_partial, nullptr, d_err, ctx->d_t0, hs);
        }
        ctx->launches += 1;
    };
    if (raw_chunked) {
        // all copies queued first (kChunkBytes each, on the copy stream); then per
        // copy chunk c: scan its record chunks once chunk c + 1 has landed (a
        // record header may straddle into it), extend the true record chain,
        // and hash every epoch whose records are now all known and present
        const uint64_t len = b->payload_bytes;
        const uint32_t n_cc = (uint32_t)((len + kChunkBytes - 1) / kChunkBytes);
        const uint32_t per_cc = (uint32_t)(kChunkBytes / kRawScanChunk);
        while (ctx->chunk_ev.size() < n_cc + 1) {
            cudaEvent_t ev;
            CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            ctx->chunk_ev.push_back(ev);
        }
        CU(cudaEventRecord(ctx->chunk_ev[n_cc], s));
        CU(cudaStreamWaitEvent(ctx->copy, ctx->chunk_ev[n_cc], 0));
        uint8_t* d_pay = const_cast<uint8_t*>(P.lay.payload);
        for (uint32_t c = 0; c < n_cc; c++) {
            const uint64_t off = (uint64_t)c * kChunkBytes, bytes = std::min<uint64_t>(kChunkBytes, len - off);
            CU(cudaMemcpyAsync(d_pay + off, b->payload + off, bytes, cudaMemcpyHostToDevice, ctx->copy));
            CU(cudaEventRecord(ctx->chunk_ev[c], ctx->copy));
        }
        uint64_t* d_off = const_cast<uint64_t*>(P.lay.offsets);
        uint32_t e_done = 0;
        for (uint32_t c = 0; c < n_cc; c++) {
            const bool last = c + 1 == n_cc;
            CU(cudaStreamWaitEvent(s, ctx->chunk_ev[last ? c : c + 1], 0));
            launch_log_scan_range(P.lay.payload, len, c * per_cc, std::min<uint32_t>((c + 1) * per_cc, n_scan),
                                  kRawScanChunk, d_sc_exit, d_sc_cnt, d_sc_start, d_sc_base, d_sc_state, d_off,
                                  n_entries + 1, s);
            ctx->launches += 3;
            uint32_t e_ready;
            if (last) {
                int rc2 = raw_scan_result(ctx, b, n_entries, d_sc_state, d_off, s, err);
                if (rc2) return rc2;
                e_ready = n_ep;
            } else {
                CU(cudaMemcpyAsync(ctx->stage->scan, d_sc_state, 16, cudaMemcpyDeviceToHost, s));
                CU(cudaStreamSynchronize(s));
                if (ctx->stage->scan[0] == ~0ull) continue;  // truncated: reported after the last chunk
                // epoch e is complete once record (e + 1) n2 has been seen (its start bounds e's last record)
                const uint64_t seen = ctx->stage->scan[1];
                e_ready = seen ? (uint32_t)std::min<uint64_t>(n_ep, (seen - 1) / b->n2) : 0;
            }
            if (e_ready > e_done) {
                TileMap t = tm;
                t.tile_begin = e_done * tm.tiles_per_epoch;
                t.tile_count = (e_ready - e_done) * tm.tiles_per_epoch;
                launch_hash(t, s);
                e_done = e_ready;
            }
        }
    } else if (chunked) {
        // chunk c covers epochs [cut[c], cut[c+1]): as many whole epochs as fit in kChunkBytes (>= 1)
        std::vector<uint32_t> cut{0};
        while (cut.back() < n_ep) {
            const uint32_t e0 = cut.back();
            uint32_t e1 = e0 + 1;
            if (!b->offsets) {
                e1 = std::min<uint32_t>(n_ep, e0 + (uint32_t)std::max<uint64_t>(1, kChunkBytes / epoch_bytes));
            } else {
                while (e1 < n_ep && epoch_byte(e1 + 1) - epoch_byte(e0) <= kChunkBytes) e1++;
            }
            cut.push_back(e1);
        }
        // the hashing of the last chunk is the exposed tail behind the copy:
        // land it as four quarter chunks (fixed-length logs; a variable-length
        // tail is bounded by the latency of one 1024-entry tile instead)
        if (!b->offsets && cut.size() >= 3 && cut.back() - cut[cut.size() - 2] >= 8) {
            const uint32_t a = cut[cut.size() - 2], z = cut.back();
            cut.pop_back();
            for (uint32_t q = 1; q <= 4; q++) cut.push_back(a + (uint32_t)((uint64_t)(z - a) * q / 4));
        }
        const uint32_t n_chunks = (uint32_t)cut.size() - 1;
        while (ctx->chunk_ev.size() < n_chunks + 1) {
            cudaEvent_t ev;
            CU(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            ctx->chunk_ev.push_back(ev);
        }
        if (use_ring) {  // pinned ring for the producer / pageable source: kFillSlots chunks in flight
            size_t need = 0;
            for (uint32_t c = 0; c < n_chunks; c++)
                need = std::max<size_t>(need, epoch_byte(cut[c + 1]) - epoch_byte(cut[c]));
            if (!ctx->fill_slot[0] || ctx->fill_cap < need) {
                CU(cudaStreamSynchronize(s));
                CU(cudaStreamSynchronize(ctx->copy));
                for (auto& p : ctx->fill_slot)
                    if (p) {
                        cudaFreeHost(p);
                        p = nullptr;
                    }
                ctx->fill_cap = 0;
                for (auto& p : ctx->fill_slot) CU(cudaMallocHost(&p, std::max<size_t>(need, 1)));
                ctx->fill_cap = std::max<size_t>(need, 1);
            }
        }
        // the copy stream must not overwrite the buffer before earlier work on s is done
        CU(cudaEventRecord(ctx->chunk_ev[n_chunks], s));
        CU(cudaStreamWaitEvent(ctx->copy, ctx->chunk_ev[n_chunks], 0));
        uint8_t* d_pay = const_cast<uint8_t*>(P.lay.payload);
        for (uint32_t c = 0; c < n_chunks; c++) {
            const uint32_t e0 = cut[c], e1 = cut[c + 1];
            const uint64_t off = epoch_byte(e0), bytes = epoch_byte(e1) - off;
            if (use_ring) {
                // produce chunk c into a free slot while chunks c-1, c-2 copy and hash
                const int sl = (int)(c % poslo_gpu_ctx::kFillSlots);
                CU(cudaEventSynchronize(ctx->fill_ev[sl]));
                if (stage_pageable)
                    HostCopyPool::get().copy(ctx->fill_slot[sl], b->payload + off, bytes);
                else if (b->fill(b->fill_user, (uint64_t)e0 * b->n2, (uint64_t)(e1 - e0) * b->n2, ctx->fill_slot[sl]) != 0) {
                    cudaStreamSynchronize(ctx->copy);
                    cudaStreamSynchronize(s);
                    return set_err(err, POSLO_INVALID_ARGUMENT, 0, "fill producer failed");
                }
                CU(cudaMemcpyAsync(d_pay + off, ctx->fill_slot[sl], bytes, cudaMemcpyHostToDevice, ctx->copy));
                CU(cudaEventRecord(ctx->fill_ev[sl], ctx->copy));
            } else {
                CU(cudaMemcpyAsync(d_pay + off, b->payload + off, bytes, cudaMemcpyHostToDevice, ctx->copy));
            }
            CU(cudaEventRecord(ctx->chunk_ev[c], ctx->copy));
            CU(cudaStreamWaitEvent(s, ctx->chunk_ev[c], 0));
            TileMap t = tm;
            t.tile_begin = e0 * tm.tiles_per_epoch;
            t.tile_count = (e1 - e0) * tm.tiles_per_epoch;
            if (t.tile_count) launch_hash(t, s);
        }
    } else if (tm.n_tiles && P.on_piece && need_finalize && tm.tiles == nullptr && pipe_pieces() > 1 &&
               n_ep >= 2 * pipe_pieces() && tm.n_tiles >= 2 * kPipeMinTiles) {
        // device-resident, uniform: epoch pieces, each finalised and handed to the caller;
        // every piece keeps >= kPipeMinTiles CTAs so no piece runs the GPU part-full
        // Pieces alternate between the context stream and hash2, so piece q+1's
        // CTAs fill the SMs while piece q drains (a single stream would idle the
        // tail wave of every piece at the kernel boundary).
        const uint32_t pieces = std::min<uint32_t>(pipe_pieces(), tm.n_tiles / kPipeMinTiles);
        cudaStream_t hs[2] = {s, ctx->hash2};
        CU(cudaEventRecord(ctx->ev_hash[0], s));
        CU(cudaStreamWaitEvent(ctx->hash2, ctx->ev_hash[0], 0));
        for (uint32_t q = 0; q < pieces; q++) {
            const uint32_t e0 = (uint32_t)((uint64_t)n_ep * q / pieces);
            const uint32_t e1 = (uint32_t)((uint64_t)n_ep * (q + 1) / pieces);
            TileMap t = tm;
            t.tile_begin = e0 * tm.tiles_per_epoch;
            t.tile_count = (e1 - e0) * tm.tiles_per_epoch;
            if (t.tile_count) launch_hash(t, hs[q & 1]);
            launch_epoch_finalize_range(tm, e0, e1, d_partial, P.d_etilde, hs[q & 1]);
            ctx->launches += 1;
            int rc2 = P.on_piece(e0, e1, hs[q & 1]);
            if (rc2) {
                cudaStreamSynchronize(ctx->hash2);
                return rc2;
            }
        }
        CU(cudaEventRecord(ctx->ev_hash[1], ctx->hash2));
        CU(cudaStreamWaitEvent(s, ctx->ev_hash[1], 0));
        need_finalize = false;
    } else if (tm.n_tiles) {
        launch_hash(tm, s);
    }
    mark(ctx, kEvFin);
    if (need_finalize && n_ep) {
        launch_epoch_finalize(tm, d_partial, P.d_etilde, s);
        ctx->launches += 1;
    }
    CU(cudaGetLastError());
    // host-side argument check, overlapping the queued device work
    for (uint32_t k = 1; k < n_ep; k++)
        if (b->epochs[k] <= b->epochs[k - 1]) {
            cudaStreamSynchronize(s);
            return set_err(err, POSLO_INVALID_ARGUMENT, 0, "epochs must be strictly ascending");
        }
    return POSLO_OK;
}

int map_hash_error(unsigned long long key, const poslo_batch* b, poslo_error* err) {
    if (key == ~0ull) return POSLO_OK;
    uint32_t k = (uint32_t)(key >> 1);
    uint32_t epoch = k < b->n_epochs ? b->epochs[k] : 0;
    if ((key & 1) == 0)
        return set_err(err, POSLO_SEED_NOT_DISCLOSED, epoch, "seed for epoch %u not yet disclosed", epoch);
    return set_err(err, POSLO_FORMAT_ERROR, epoch, "modular-addition hash: entry too long for this suite");
}

// Reads the error word (synchronises) and maps it to the reference error.
int check_hash_errors(poslo_gpu_ctx* ctx, const poslo_batch* b, poslo_error* err) {
    CU(cudaMemcpyAsync(&ctx->stage->err_key, ctx->b_err.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return map_hash_error(ctx->stage->err_key, b, err);
}

void finish_timing(poslo_gpu_ctx* ctx) {
    if (!ctx->timing) return;
    cudaEventRecord(ctx->ev[kEvEnd], ctx->stream);
    cudaEventSynchronize(ctx->ev[kEvEnd]);
    cudaEventElapsedTime(&ctx->last_ms[0], ctx->ev[kEvSeed], ctx->ev[kEvHash]);
    cudaEventElapsedTime(&ctx->last_ms[1], ctx->ev[kEvHash], ctx->ev[kEvFin]);
    cudaEventElapsedTime(&ctx->last_ms[2], ctx->ev[kEvFin], ctx->ev[kEvSum]);
    cudaEventElapsedTime(&ctx->last_ms[3], ctx->ev[kEvSum], ctx->ev[kEvGroup]);
    cudaEventElapsedTime(&ctx->last_ms[4], ctx->ev[kEvGroup], ctx->ev[kEvEnd]);
    cudaEventElapsedTime(&ctx->last_ms[5], ctx->ev[kEvSeed], ctx->ev[kEvEnd]);
}

// Serialises the calls on one context and makes its device current for the
// call; the caller's current device is restored on exit (a torch thread on
// cuda:0 calling a context on device 1 keeps allocating on cuda:0).
struct Guard {
    poslo_gpu_ctx* ctx;
    std::lock_guard<std::mutex> lk;
    int prev = -1;
    explicit Guard(poslo_gpu_ctx* c) : ctx(c), lk(c->mtx) {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            cudaGetLastError();
            prev = -1;
        }
        if (prev != c->device) cudaSetDevice(c->device);
        c->launches = 0;
    }
    ~Guard() {
        if (prev >= 0 && prev != ctx->device) cudaSetDevice(prev);
    }
    Guard(const Guard&) = delete;
    Guard& operator=(const Guard&) = delete;
};

int upload(poslo_gpu_ctx* ctx, DevBuf& buf, const void* src, size_t bytes, void** out, poslo_error* err) {
    uint8_t* d;
    int rc = ensure(buf, bytes, &d, err);
    if (rc) return rc;
    if (bytes) CU(cudaMemcpyAsync(d, src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    *out = d;
    return POSLO_OK;
}

#define UPLOAD(buf, src, bytes, ptr)                                              \
    do {                                                                          \
        void* p_;                                                                 \
        int rc_ = upload(ctx, ctx->buf, (src), (bytes), &p_, err);                \
        if (rc_) return rc_;                                                      \
        ptr = static_cast<decltype(ptr)>(p_);                                     \
    } while (0)

// Comb tables of alpha (once per context) and of Y (cached per Y value).
// Y validation (GroupElement::from_bytes) happens in the table build.
// Batches of at least POSLO_COMB16_MIN checks (default 2^17) use the
// radix-2^16 combs: half the additions per check for a one-time build of
// alpha's table per context and Y's per Y value (~10 ms each).
uint32_t comb16_min() {
    const char* e = std::getenv("POSLO_COMB16_MIN");
    return e ? (uint32_t)std::strtoul(e, nullptr, 10) : (1u << 17);
}

// The generator's tables depend on nothing but the device: built once per
// process and device (on the first context's stream, then synchronised so
// every later context and stream can read them) and shared by all contexts.
struct GenTables {
    void* tab[3] = {};  // radix 16, radix 256, radix 2^16
};
std::mutex g_gen_mtx;
GenTables g_gen[64];

int gen_table(poslo_gpu_ctx* ctx, int kind, int* d_flags, void** out, poslo_error* err) {
    std::lock_guard<std::mutex> lk(g_gen_mtx);
    if (ctx->device < 0 || ctx->device >= 64) return set_err(err, POSLO_CUDA_ERROR, 0, "device index out of range");
    void*& t = g_gen[ctx->device].tab[kind];
    if (!t) {
        const size_t bytes = kind == 0 ? kCombTableBytes : kind == 1 ? kComb256TableBytes : kComb16TableBytes;
        void* p = nullptr;
        CU(cudaMalloc(&p, bytes));
        if (ctx->pk_owner != 1) {  // the generator's powers, once per context for all radices
            launch_table_powers(nullptr, ctx->d_pk, d_flags, ctx->stream);
            ctx->pk_owner = 1;
            ctx->launches += 1;
        }
        launch_table_fill(kind, ctx->d_pk, p, ctx->stream);
        ctx->launches += 1;
        cudaError_t e = cudaStreamSynchronize(ctx->stream);
        if (e != cudaSuccess) {
            cudaFree(p);
            return set_err(err, POSLO_CUDA_ERROR, 0, "generator table: %s", cudaGetErrorString(e));
        }
        t = p;
    }
    *out = t;
    return POSLO_OK;
}

// d_pk <- the powers 16^i Y, unless it already holds them (one chain per Y
// serves the radix-16, 256 and 2^16 tables).
int y_powers(poslo_gpu_ctx* ctx, const uint8_t y[32], int* d_flags, poslo_error* err) {
    if (ctx->pk_owner == 2 && std::memcmp(ctx->pk_key, y, 32) == 0) return POSLO_OK;
    uint8_t* d_y;
    UPLOAD(b_y, y, 32, d_y);
    launch_table_powers(d_y, ctx->d_pk, d_flags, ctx->stream);
    ctx->pk_owner = 2;
    std::memcpy(ctx->pk_key, y, 32);
    ctx->launches += 1;
    return POSLO_OK;
}

int ensure_tables(poslo_gpu_ctx* ctx, const uint8_t y[32], int* d_flags, poslo_error* err, bool wide = false,
                  bool xwide = false) {
    if (!ctx->d_pk) CU(cudaMalloc(&ctx->d_pk, 64 * kGptBytes));
    // the generator's tables first (one power chain for all of them), then Y's
    if (!ctx->d_tabB) {
        int rc = gen_table(ctx, 0, d_flags, &ctx->d_tabB, err);
        if (rc) return rc;
    }
    if (wide && !ctx->d_tabB256) {
        int rc = gen_table(ctx, 1, d_flags, &ctx->d_tabB256, err);
        if (rc) return rc;
    }
    if (xwide && !ctx->d_tabB16) {
        int rc = gen_table(ctx, 2, d_flags, &ctx->d_tabB16, err);
        if (rc) return rc;
    }
    if (!ctx->d_tabY) CU(cudaMalloc(&ctx->d_tabY, kCombTableBytes));
    if (!ctx->tabY_valid || std::memcmp(ctx->tabY_key, y, 32) != 0) {
        uint8_t* d_y;
        UPLOAD(b_y, y, 32, d_y);
        launch_table_powers(d_y, ctx->d_pk, d_flags, ctx->stream);
        ctx->pk_owner = 2;
        std::memcpy(ctx->pk_key, y, 32);
        launch_table_fill(0, ctx->d_pk, ctx->d_tabY, ctx->stream);
        ctx->launches += 2;
        int bad = 0;
        CU(cudaMemcpyAsync(&bad, d_flags, 4, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
        if (bad) {
            ctx->tabY_valid = false;
            return set_err(err, POSLO_FORMAT_ERROR, 0, "invalid group element encoding");
        }
        std::memcpy(ctx->tabY_key, y, 32);
        ctx->tabY_valid = true;
    }
    if (wide) {
        if (!ctx->d_tabB256) {
            int rc = gen_table(ctx, 1, d_flags, &ctx->d_tabB256, err);
            if (rc) return rc;
        }
        if (!ctx->d_tabY256) CU(cudaMalloc(&ctx->d_tabY256, kComb256TableBytes));
        if (!ctx->tabY256_valid || std::memcmp(ctx->tabY256_key, y, 32) != 0) {
            const int rc = y_powers(ctx, y, d_flags, err);  // Y already validated by the radix-16 build above
            if (rc) return rc;
            launch_table_fill(1, ctx->d_pk, ctx->d_tabY256, ctx->stream);
            ctx->launches += 1;
            std::memcpy(ctx->tabY256_key, y, 32);
            ctx->tabY256_valid = true;
        }
    }
    if (xwide) {
        if (!ctx->d_tabB16) {
            int rc = gen_table(ctx, 2, d_flags, &ctx->d_tabB16, err);
            if (rc) return rc;
        }
        if (!ctx->d_tabY16) CU(cudaMalloc(&ctx->d_tabY16, kComb16TableBytes));
        if (!ctx->tabY16_valid || std::memcmp(ctx->tabY16_key, y, 32) != 0) {
            const int rc = y_powers(ctx, y, d_flags, err);  // Y already validated by the radix-16 build above
            if (rc) return rc;
            launch_table_fill(2, ctx->d_pk, ctx->d_tabY16, ctx->stream);
            ctx->launches += 1;
            std::memcpy(ctx->tabY16_key, y, 32);
            ctx->tabY16_valid = true;
        }
    }
    return POSLO_OK;
}

// Form of the radix-2^16 batched checks (POSLO_CHECK16, A/B knob):
//   sqrt    no square root per check: combs -> one batched inversion per 32
//           checks -> encode(P) == R-hat by squares (launch_check16e); the
//           default for per-epoch verdicts
//   decode  a thread per check against R-hat decoded on a side stream while the
//           log is hashed (k_check_thread16d); distillation always decodes R-hat
//           (it folds the decoded points) and checks this way
//   split   8 lanes per check against decoded R-hat (k_check_split16)
//   encode  a thread per check comparing encodings (k_check_thread16)
enum class Check16 { Sqrt, Decode, Split, Encode };
static Check16 check16_mode() {
    const char* e = std::getenv("POSLO_CHECK16");
    if (!e) return Check16::Sqrt;
    if (!std::strcmp(e, "decode")) return Check16::Decode;
    if (!std::strcmp(e, "split")) return Check16::Split;
    if (!std::strcmp(e, "encode")) return Check16::Encode;
    return Check16::Sqrt;
}

// POSLO_DECODE_EARLY=1: queue the R-hat decode before the seeds (A/B knob;
// default: behind the seed kernel, beside the hashing)
static bool decode_early() {
    const char* e = std::getenv("POSLO_DECODE_EARLY");
    return e && std::strcmp(e, "1") == 0;
}

// The batched checks on the widest tables ensure_tables built. Radix 2^16, a
// thread per check: with scratch (scr) and no decoded R-hat, no square root
// per check (launch_check16e, the points kept in scr.P); with R-hat decoded
// ahead (d_pts, d_ok), the class compare (or 8 lanes per check, POSLO_CHECK16=
// split); with neither, encodings compared (d_r). Radix 256: 8 lanes per check
// against decoded R-hat.
void launch_checks(poslo_gpu_ctx* ctx, bool xwide, uint32_t n, const uint32_t* d_e, const uint32_t* d_s,
                   const uint8_t* d_r, const void* d_pts, const uint8_t* d_ok, uint8_t* d_verdict, cudaStream_t st,
                   const Scr16e& scr = Scr16e{}) {
    if (xwide && !d_pts && scr)  // no square root per check (launch_check16e)
        launch_check16e(ctx->d_tabY16, ctx->d_tabB16, n, d_e, d_s, d_r, scr.P, scr.u2, scr.pre, d_verdict, st);
    else if (xwide && !d_pts)
        launch_check_thread16(ctx->d_tabY16, ctx->d_tabB16, n, d_e, d_s, d_r, nullptr, d_verdict, st);
    else if (xwide && check16_mode() == Check16::Split)
        launch_check_split16(ctx->d_tabY16, ctx->d_tabB16, n, d_e, d_s, d_pts, d_ok, d_verdict, st);
    else if (xwide)
        launch_check_thread16d(ctx->d_tabY16, ctx->d_tabB16, n, d_e, d_s, d_pts, d_ok, d_verdict, st);
    else
        launch_check_split(ctx->d_tabY256, ctx->d_tabB256, n, d_e, d_s, d_pts, d_ok, d_verdict, st);
}

// Batched group check on device arrays; verdicts/encodings to host.
int group_check_dev(poslo_gpu_ctx* ctx, const uint8_t y[32], uint32_t n, const uint32_t* d_e,
                    const uint32_t* d_s, const uint8_t* d_r, uint8_t* h_verdict, uint8_t* h_enc,
                    poslo_error* err) {
    int* d_flags;
    uint8_t* d_verdict = nullptr;
    uint8_t* d_enc = nullptr;
    ENSURE(b_flags, 4, d_flags);
    CU(cudaMemsetAsync(d_flags, 0, 16, ctx->stream));
    const bool xwide = n > kCtaCheckMax && n >= comb16_min();  // radix-2^16 combs, thread per check
    int rc = ensure_tables(ctx, y, d_flags, err, n > kCtaCheckMax, xwide);
    if (rc) return rc;
    if (h_verdict) ENSURE(b_verdict, n, d_verdict);
    if (h_enc) ENSURE(b_enc, (size_t)n * 32, d_enc);
    if (xwide && !d_enc && d_r && d_verdict && check16_mode() == Check16::Sqrt) {
        // verdicts only: no square root per check (launch_check16e)
        Scr16e scr;
        rc = ensure_scr16e(ctx, n, scr, err);
        if (rc) return rc;
        launch_check16e(ctx->d_tabY16, ctx->d_tabB16, n, d_e, d_s, d_r, scr.P, scr.u2, scr.pre, d_verdict,
                        ctx->stream);
    } else if (xwide) {
        launch_check_thread16(ctx->d_tabY16, ctx->d_tabB16, n, d_e, d_s, d_r, d_enc, d_verdict, ctx->stream);
    } else
        launch_group_check_comb(ctx->d_tabY, ctx->d_tabB, ctx->d_tabY256, ctx->d_tabB256, n, d_e, d_s, d_r, d_enc,
                                d_verdict, ctx->stream);
    ctx->launches += n ? 1 : 0;
    CU(cudaGetLastError());
    int ybad = 0;
    CU(cudaMemcpyAsync(&ybad, d_flags, 4, cudaMemcpyDeviceToHost, ctx->stream));
    if (h_verdict && n) CU(cudaMemcpyAsync(h_verdict, d_verdict, n, cudaMemcpyDeviceToHost, ctx->stream));
    if (h_enc && n) CU(cudaMemcpyAsync(h_enc, d_enc, (size_t)n * 32, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (ybad) return set_err(err, POSLO_FORMAT_ERROR, 0, "invalid group element encoding");
    return POSLO_OK;
}


// LE 32-byte scalar -> 8 limbs (identical memory image on little-endian hosts).
bool scalar_canonical(const uint8_t* s) {
    static const uint8_t L[32] = {0xed, 0xd3, 0xf5, 0x5c, 0x1a, 0x63, 0x12, 0x58, 0xd6, 0x9c, 0xf7,
                                  0xa2, 0xde, 0xf9, 0xde, 0x14, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0,
                                  0, 0, 0, 0x10};
    for (int i = 31; i >= 0; i--) {
        if (s[i] < L[i]) return true;
        if (s[i] > L[i]) return false;
    }
    return false;
}

}  // namespace

void poslo_gpu_detail::count_op(const poslo_gpu_ctx* ctx, int which, uint64_t n) {
    if (ctx->count_ops && n) g_ops[which].fetch_add(n, std::memory_order_relaxed);
}
using poslo_gpu_detail::count_op;
using poslo_gpu_detail::kOpCombine;
using poslo_gpu_detail::kOpDoubleExp;
using poslo_gpu_detail::kOpExpBase;

extern "C" {

void poslo_gpu_group_op_counts(uint64_t out[4]) {
    if (!out) return;
    for (int i = 0; i < 4; i++) out[i] = g_ops[i].load(std::memory_order_relaxed);
}

void poslo_gpu_reset_group_op_counts(void) {
    for (auto& c : g_ops) c.store(0, std::memory_order_relaxed);
}

const char* poslo_gpu_version(void) { return "poslo-b200 0.1 (sm_100a)"; }

int poslo_gpu_create(int device, poslo_gpu_ctx** out, poslo_error* err) {
    if (!out) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null out");
    *out = nullptr;
    int ndev = 0;
    CU(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return set_err(err, POSLO_CUDA_ERROR, 0, "no CUDA device %d (have %d)", device, ndev);
    cudaDeviceProp prop;
    CU(cudaGetDeviceProperties(&prop, device));
    if (prop.major < 10)
        return set_err(err, POSLO_CUDA_ERROR, 0, "device %d is sm_%d%d; this build targets sm_100a",
                       device, prop.major, prop.minor);
    CU(cudaSetDevice(device));
    poslo_gpu_ctx* ctx = new poslo_gpu_ctx();
    ctx->device = device;
    // The context's own stream is a BLOCKING stream: work a caller queued on
    // the legacy default stream (e.g. torch's default stream filling a
    // device-resident batch) is ordered before ours without an explicit
    // sync. Internal copy / side streams stay non-blocking.
    cudaError_t e = cudaStreamCreateWithFlags(&ctx->own, cudaStreamDefault);
    if (e != cudaSuccess) {
        delete ctx;
        return set_err(err, POSLO_CUDA_ERROR, 0, "stream: %s", cudaGetErrorString(e));
    }
    ctx->stream = ctx->own;
    e = cudaStreamCreateWithFlags(&ctx->copy, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&ctx->hash2, cudaStreamNonBlocking);
    for (int i = 0; i < 2 && e == cudaSuccess; i++)
        e = cudaEventCreateWithFlags(&ctx->ev_side[i], cudaEventDisableTiming);
    for (int i = 0; i < 2 && e == cudaSuccess; i++)
        e = cudaEventCreateWithFlags(&ctx->ev_hash[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ctx->ev_pre, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        poslo_gpu_destroy(ctx);
        return set_err(err, POSLO_CUDA_ERROR, 0, "stream: %s", cudaGetErrorString(e));
    }
    uint32_t t0[256];
    for (int x = 0; x < 256; x++) t0[x] = aes_t0_entry(aes_sbox_compute(x));
    e = cudaMalloc(&ctx->d_t0, sizeof t0);
    if (e == cudaSuccess) e = cudaMemcpy(ctx->d_t0, t0, sizeof t0, cudaMemcpyHostToDevice);
    for (int i = 0; i < 7 && e == cudaSuccess; i++) e = cudaEventCreate(&ctx->ev[i]);
    for (int i = 0; i < poslo_gpu_ctx::kFillSlots && e == cudaSuccess; i++)
        e = cudaEventCreateWithFlags(&ctx->fill_ev[i], cudaEventDisableTiming);
    if (e == cudaSuccess) e = cudaMallocHost(&ctx->stage, sizeof(PinnedStage));
    if (e != cudaSuccess) {
        poslo_gpu_destroy(ctx);
        return set_err(err, POSLO_CUDA_ERROR, 0, "init: %s", cudaGetErrorString(e));
    }
    *out = ctx;
    return ok(err);
}

int poslo_gpu_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int poslo_gpu_create_multi(const int* devices, int n_devices, poslo_gpu_ctx** out, poslo_error* err) {
    if (!out || !devices || n_devices < 1) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "bad argument");
    *out = nullptr;
    if (n_devices == 1) return poslo_gpu_create(devices[0], out, err);
    poslo_gpu_ctx* ctx = new poslo_gpu_ctx();
    ctx->device = devices[0];
    for (int k = 0; k < n_devices; k++) {
        poslo_gpu_ctx* m = nullptr;
        int rc = poslo_gpu_create(devices[k], &m, err);
        if (rc) {
            poslo_gpu_destroy(ctx);
            return rc;
        }
        ctx->members.push_back(m);
    }
    *out = ctx;
    return ok(err);
}

int poslo_gpu_member_count(const poslo_gpu_ctx* ctx) {
    if (!ctx) return 0;
    return ctx->members.empty() ? 1 : (int)ctx->members.size();
}

void poslo_gpu_destroy(poslo_gpu_ctx* ctx) {
    if (!ctx) return;
    if (!ctx->members.empty()) {  // a multi-device context owns only its members
        for (poslo_gpu_ctx* m : ctx->members) poslo_gpu_destroy(m);
        delete ctx;
        return;
    }
    int prev = -1;
    if (cudaGetDevice(&prev) != cudaSuccess) {
        cudaGetLastError();
        prev = -1;
    }
    cudaSetDevice(ctx->device);
    DevBuf* bufs[] = {&ctx->b_epochs, &ctx->b_x0, &ctx->b_partial, &ctx->b_etilde, &ctx->b_sum,
                      &ctx->b_scratch, &ctx->b_tiles, &ctx->b_starts, &ctx->b_tbegin, &ctx->b_err,
                      &ctx->b_flags, &ctx->b_payload, &ctx->b_offsets, &ctx->b_e, &ctx->b_s,
                      &ctx->b_r, &ctx->b_enc, &ctx->b_verdict, &ctx->b_mask, &ctx->b_seg, &ctx->b_y,
                      &ctx->b_pts, &ctx->b_foldscratch, &ctx->b_rhat, &ctx->b_pre, &ctx->b_starts_ds,
                      &ctx->b_seg32, &ctx->b_out_s, &ctx->b_out_r, &ctx->b_dpts, &ctx->b_dok,
                      &ctx->b_scan_exit, &ctx->b_scan_cnt, &ctx->b_scan_start, &ctx->b_scan_base,
                      &ctx->b_scan_off, &ctx->b_scan_state, &ctx->b_seg_e, &ctx->b_out_e, &ctx->b_ppre_s, &ctx->b_ppre_r,
                      &ctx->b_ppre, &ctx->b_scr16e};
    for (DevBuf* b : bufs)
        if (b->p) cudaFree(b->p);
    if (ctx->d_t0) cudaFree(ctx->d_t0);
    if (ctx->stage) cudaFreeHost(ctx->stage);
    // (the generator tables d_tabB* are the process's, shared: not freed here)
    for (void* p : {ctx->d_tabY, ctx->d_tabY256, ctx->d_tabY16, ctx->d_pk})
        if (p) cudaFree(p);
    for (auto* p : ctx->fill_slot)
        if (p) cudaFreeHost(p);
    for (auto& ev : ctx->fill_ev)
        if (ev) cudaEventDestroy(ev);
    for (auto& ev : ctx->ev)
        if (ev) cudaEventDestroy(ev);
    for (auto& ev : ctx->chunk_ev) cudaEventDestroy(ev);
    if (ctx->copy) cudaStreamDestroy(ctx->copy);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->hash2) cudaStreamDestroy(ctx->hash2);
    for (auto& ev : ctx->ev_side)
        if (ev) cudaEventDestroy(ev);
    for (auto& ev : ctx->ev_hash)
        if (ev) cudaEventDestroy(ev);
    if (ctx->ev_pre) cudaEventDestroy(ctx->ev_pre);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    delete ctx;
    if (prev >= 0) cudaSetDevice(prev);
}

int poslo_gpu_set_stream(poslo_gpu_ctx* ctx, void* stream) {
    if (!ctx) return POSLO_INVALID_ARGUMENT;
    if (!ctx->members.empty()) ctx = ctx->members[0];  // a stream belongs to one device: member 0's
    std::lock_guard<std::mutex> lk(ctx->mtx);
    ctx->stream = stream ? static_cast<cudaStream_t>(stream) : ctx->own;
    return POSLO_OK;
}

int poslo_gpu_enable_timing(poslo_gpu_ctx* ctx, int on) {
    if (!ctx) return POSLO_INVALID_ARGUMENT;
    for (poslo_gpu_ctx* m : ctx->members) m->timing = on != 0;
    ctx->timing = on != 0;
    return POSLO_OK;
}

int poslo_gpu_last_timings(poslo_gpu_ctx* ctx, float out_ms[6]) {
    if (!ctx || !out_ms) return POSLO_INVALID_ARGUMENT;
    if (!ctx->members.empty()) {  // the slowest member's stages
        std::memset(out_ms, 0, 6 * sizeof(float));
        for (poslo_gpu_ctx* m : ctx->members)
            for (int i = 0; i < 6; i++) out_ms[i] = std::max(out_ms[i], m->last_ms[i]);
        return POSLO_OK;
    }
    std::memcpy(out_ms, ctx->last_ms, sizeof ctx->last_ms);
    return POSLO_OK;
}

int poslo_log_scan(const uint8_t* raw, uint64_t len, uint64_t* offsets, uint64_t cap, uint64_t* n_records,
                   poslo_error* err) {
    // read_log (log_file.hpp:34-51): LE32 length, then that many bytes; the
    // walk is inherently sequential (each record's position depends on every
    // earlier length), so it is one tight host loop over the file image.
    if (!n_records || (len && !raw)) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    uint64_t off = 0, n = 0;
    while (off < len) {
        if (len - off < 4) return set_err(err, POSLO_FORMAT_ERROR, 0, "truncated log record");
        uint32_t l;
        std::memcpy(&l, raw + off, 4);  // little-endian host (x86-64 / aarch64)
        if (len - off - 4 < l) return set_err(err, POSLO_FORMAT_ERROR, 0, "truncated log record");
        if (offsets && n < cap) offsets[n] = off;
        off += 4 + (uint64_t)l;
        n++;
    }
    *n_records = n;
    if (!offsets || n + 1 > cap) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "offsets capacity %llu < %llu",
                                                (unsigned long long)cap, (unsigned long long)(n + 1));
    offsets[n] = len;
    return ok(err);
}

int poslo_gpu_log_scan(poslo_gpu_ctx* ctx, const uint8_t* raw, uint64_t len, int32_t device_resident,
                       uint64_t* offsets, uint64_t cap, uint64_t* n_records, poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!n_records || (len && !raw)) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    Guard g(ctx);
    cudaStream_t s = ctx->stream;
    const uint8_t* d_raw = raw;
    if (device_resident && ((len && !device_readable(raw)) || !device_readable(offsets)))
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "device_resident image with a host pointer");
    if (!device_resident && len) {
        uint8_t* d;
        ENSURE(b_payload, len, d);
        CU(cudaMemcpyAsync(d, raw, len, cudaMemcpyHostToDevice, s));
        d_raw = d;
    }
    const uint32_t n_chunks = (uint32_t)((len + kScanChunk - 1) / kScanChunk);
    uint64_t *d_exit, *d_start, *d_base;
    uint32_t* d_cnt;
    unsigned long long* d_state;
    ENSURE(b_scan_exit, (size_t)std::max<uint32_t>(n_chunks, 1) * kScanWindow, d_exit);
    ENSURE(b_scan_cnt, (size_t)std::max<uint32_t>(n_chunks, 1) * kScanWindow, d_cnt);
    ENSURE(b_scan_start, std::max<uint32_t>(n_chunks, 1), d_start);
    ENSURE(b_scan_base, std::max<uint32_t>(n_chunks, 1), d_base);
    ENSURE(b_err, 1, d_state);
    launch_log_scan_a(d_raw, len, n_chunks, d_exit, d_cnt, s);
    launch_log_scan_b(d_raw, len, n_chunks, d_exit, d_cnt, d_start, d_base, d_state, s);
    ctx->launches += 2;
    CU(cudaGetLastError());
    unsigned long long total = 0;
    if (len) {
        CU(cudaMemcpyAsync(&ctx->stage->err_key, d_state, 8, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        total = ctx->stage->err_key;
    }
    if (total == ~0ull) return set_err(err, POSLO_FORMAT_ERROR, 0, "truncated log record");
    *n_records = total;
    if (!offsets || total + 1 > cap)
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "offsets capacity %llu < %llu", (unsigned long long)cap,
                       (unsigned long long)(total + 1));
    uint64_t* d_off = offsets;
    if (!device_resident) ENSURE(b_scan_off, total + 1, d_off);
    launch_log_scan_c(d_raw, len, n_chunks, d_start, d_base, d_off, s);
    ctx->launches += n_chunks ? 1 : 0;
    ctx->stage->err_init = len;
    CU(cudaMemcpyAsync(d_off + total, &ctx->stage->err_init, 8, cudaMemcpyHostToDevice, s));
    if (!device_resident) CU(cudaMemcpyAsync(offsets, d_off, (total + 1) * 8, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    return ok(err);
}

uint32_t poslo_gpu_last_launches(poslo_gpu_ctx* ctx) {
    if (!ctx) return 0;
    uint32_t n = ctx->launches;
    for (poslo_gpu_ctx* m : ctx->members) n += m->launches;
    return n;
}

int poslo_gpu_agg_ekeys(poslo_gpu_ctx* ctx, const poslo_batch* b, uint8_t* e_tilde_out,
                        uint8_t* e_hat_out, poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!ctx->members.empty()) return multi_agg_ekeys(ctx, b, e_tilde_out, e_hat_out, err);
    Guard g(ctx);
    Prepared P;
    P.want_etilde = e_tilde_out != nullptr;
    int rc = run_hash(ctx, b, P, err);
    if (rc) return rc;
    mark(ctx, kEvSum);
    uint32_t* d_sum = nullptr;
    if (e_hat_out) {
        uint32_t* d_scr;
        ENSURE(b_sum, 8, d_sum);
        ENSURE(b_scratch, 17 * 1024, d_scr);
        launch_sum_mod_l(P.sum_src, P.sum_limbs, b->n_epochs, nullptr, d_sum, d_scr, ctx->stream);
        ctx->launches += 2;
    }
    mark(ctx, kEvGroup);
    rc = check_hash_errors(ctx, b, err);
    if (rc) return rc;
    if (e_tilde_out && b->n_epochs)
        CU(cudaMemcpyAsync(e_tilde_out, P.d_etilde, (size_t)b->n_epochs * 32, cudaMemcpyDeviceToHost, ctx->stream));
    if (e_hat_out) CU(cudaMemcpyAsync(e_hat_out, d_sum, 32, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    finish_timing(ctx);
    return ok(err);
}

int poslo_gpu_agg_ekeys_partial(poslo_gpu_ctx* ctx, const poslo_batch* b, uint8_t* d_e_part, poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!d_e_part) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (!ctx->members.empty()) {  // fold of the members' shards, left on member 0's device
        uint8_t part[32];
        int rc = multi_agg_ekeys(ctx, b, nullptr, part, err);
        if (rc) return rc;
        poslo_gpu_ctx* m0 = ctx->members[0];
        Guard g(m0);
        CU(cudaMemcpyAsync(d_e_part, part, 32, cudaMemcpyHostToDevice, m0->stream));
        CU(cudaStreamSynchronize(m0->stream));
        return ok(err);
    }
    if (!device_readable(d_e_part)) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "d_e_part is not device memory");
    Guard g(ctx);
    Prepared P;
    P.want_etilde = false;
    int rc = run_hash(ctx, b, P, err);
    if (rc) return rc;
    mark(ctx, kEvSum);
    uint32_t* d_scr;
    ENSURE(b_scratch, 17 * 1024, d_scr);
    launch_sum_mod_l(P.sum_src, P.sum_limbs, b->n_epochs, nullptr, reinterpret_cast<uint32_t*>(d_e_part), d_scr,
                     ctx->stream);
    ctx->launches += 2;
    mark(ctx, kEvGroup);
    rc = check_hash_errors(ctx, b, err);
    if (rc) return rc;
    finish_timing(ctx);
    return ok(err);
}

// The e-hat-independent half of the next combine_check with these inputs,
// queued on the side stream now (before the caller's hashing), so that only
// the fold and the Y^e-hat half remain after the all-gather.
int poslo_gpu_combine_check_prepare(poslo_gpu_ctx* ctx, const uint8_t y[32], const uint8_t s_hat[32],
                                    const uint8_t r_hat[32], poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!y || !s_hat || !r_hat) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    if (!scalar_canonical(s_hat)) return set_err(err, POSLO_FORMAT_ERROR, 0, "non-canonical scalar");
    Guard g(ctx);
    int* d_flags;
    ENSURE(b_flags, 4, d_flags);
    CU(cudaMemsetAsync(d_flags, 0, 16, ctx->stream));
    int rc = ensure_tables(ctx, y, d_flags, err);
    if (rc) return rc;
    // own buffers: the side-stream kernel may run after later calls reuse the shared ones
    uint32_t* d_s;
    uint8_t* d_rhat;
    uint8_t* d_pre;  // a CheckPre record (group_kernels.cu), 256 bytes reserved
    UPLOAD(b_ppre_s, s_hat, 32, d_s);
    UPLOAD(b_ppre_r, r_hat, 32, d_rhat);
    ENSURE(b_ppre, 256, d_pre);
    CU(cudaEventRecord(ctx->ev_side[0], ctx->stream));
    CU(cudaStreamWaitEvent(ctx->side, ctx->ev_side[0], 0));
    launch_check_pre(ctx->d_tabB, d_s, d_rhat, d_pre, ctx->side);
    ctx->launches += 1;
    CU(cudaEventRecord(ctx->ev_pre, ctx->side));
    std::memcpy(ctx->pre_key, y, 32);
    std::memcpy(ctx->pre_key + 32, s_hat, 32);
    std::memcpy(ctx->pre_key + 64, r_hat, 32);
    ctx->pre_valid = true;
    return ok(err);
}

int poslo_gpu_combine_check(poslo_gpu_ctx* ctx, uint32_t n_parts, const uint8_t* e_parts, int32_t parts_on_device,
                            const uint8_t y[32], const uint8_t s_hat[32], const uint8_t r_hat[32], uint8_t* verdict,
                            poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!y || !s_hat || !r_hat || !verdict || (n_parts && !e_parts))
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    if (!scalar_canonical(s_hat)) return set_err(err, POSLO_FORMAT_ERROR, 0, "non-canonical scalar");
    if (parts_on_device) {
        if (n_parts && !device_readable(e_parts))
            return set_err(err, POSLO_INVALID_ARGUMENT, 0, "parts_on_device with a host pointer");
    } else {
        for (uint32_t k = 0; k < n_parts; k++)
            if (!scalar_canonical(e_parts + 32 * (size_t)k))
                return set_err(err, POSLO_FORMAT_ERROR, 0, "non-canonical scalar");
    }
    Guard g(ctx);
    int* d_flags;
    ENSURE(b_flags, 4, d_flags);
    CU(cudaMemsetAsync(d_flags, 0, 16, ctx->stream));
    int rc = ensure_tables(ctx, y, d_flags, err);  // validates Y (syncs only when Y changed)
    if (rc) return rc;
    const uint32_t* d_parts;
    if (parts_on_device) {
        d_parts = reinterpret_cast<const uint32_t*>(e_parts);
    } else {
        uint32_t* d_up;
        UPLOAD(b_e, e_parts, (size_t)n_parts * 32, d_up);
        d_parts = d_up;
    }
    uint32_t *d_sum, *d_scr;
    uint8_t* d_verdict;
    uint8_t* d_pre;
    ENSURE(b_sum, 8, d_sum);
    ENSURE(b_scratch, 17 * 1024, d_scr);
    ENSURE(b_pre, 256, d_pre);
    ENSURE(b_verdict, 1, d_verdict);
    // the rank-ordered fold mod l (batch_verify.cpp:83-85), then the one check (:86)
    launch_sum_mod_l(d_parts, 8, n_parts, nullptr, d_sum, d_scr, ctx->stream);
    const bool prepared = ctx->pre_valid && std::memcmp(ctx->pre_key, y, 32) == 0 &&
                          std::memcmp(ctx->pre_key + 32, s_hat, 32) == 0 &&
                          std::memcmp(ctx->pre_key + 64, r_hat, 32) == 0;
    ctx->pre_valid = false;
    if (prepared) {  // queued by combine_check_prepare on the side stream
        CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_pre, 0));
        d_pre = static_cast<uint8_t*>(ctx->b_ppre.p);
    } else {
        uint32_t* d_s;
        uint8_t* d_rhat;
        UPLOAD(b_s, s_hat, 32, d_s);
        UPLOAD(b_rhat, r_hat, 32, d_rhat);
        launch_check_pre(ctx->d_tabB, d_s, d_rhat, d_pre, ctx->stream);
        ctx->launches += 1;
    }
    launch_check_post(ctx->d_tabY, d_sum, d_pre, d_verdict, ctx->stream);
    ctx->launches += 3;
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(&ctx->stage->verdict, d_verdict, 1, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    *verdict = ctx->stage->verdict;
    count_op(ctx, kOpDoubleExp, 1);
    return ok(err);
}

int poslo_gpu_paver(poslo_gpu_ctx* ctx, const poslo_batch* b, const uint8_t y[32],
                    const uint8_t s_hat[32], const uint8_t* r_hat_agg, const uint8_t* r_hats,
                    uint8_t* verdict, poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!b || !y || !s_hat || !verdict) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (!ctx->members.empty()) return multi_paver(ctx, b, y, s_hat, r_hat_agg, r_hats, verdict, err);
    Guard g(ctx);
    // 1. every batch holds exactly n2 entries (batch_verify.cpp:68-70)
    if (b->epoch_starts)
        for (uint32_t k = 0; k < b->n_epochs; k++)
            if (b->epoch_starts[k + 1] - b->epoch_starts[k] != b->n2)
                return set_err(err, POSLO_STATE_ERROR, b->epochs[k], "every batch must hold exactly n2 entries");
    // 2. R-hat: given aggregate or fold of the per-epoch commitments (:71-82)
    if (!r_hat_agg && !r_hats && b->n_epochs)
        return set_err(err, POSLO_STATE_ERROR, b->epochs[0], "commitment for epoch %u no longer in public key",
                       b->epochs[0]);
    if (!scalar_canonical(s_hat)) return set_err(err, POSLO_FORMAT_ERROR, 0, "non-canonical scalar");
    uint8_t* d_rhat;
    ENSURE(b_rhat, 32, d_rhat);
    int* d_flags;
    ENSURE(b_flags, 4, d_flags);
    CU(cudaMemsetAsync(d_flags, 0, 16, ctx->stream));
    if (r_hat_agg) {
        CU(cudaMemcpyAsync(d_rhat, r_hat_agg, 32, cudaMemcpyHostToDevice, ctx->stream));
    } else {
        uint8_t* d_pts;
        void* d_fs;
        UPLOAD(b_pts, r_hats, (size_t)b->n_epochs * 32, d_pts);
        ENSURE(b_foldscratch, 1024 * kGptBytes, d_fs);
        launch_point_fold(d_pts, b->n_epochs, d_rhat, d_flags + 1, d_fs, ctx->stream);
        ctx->launches += 2;
    }
    // 3. the e-hat-independent half of the check (R decode, R - s*alpha) on
    // the side stream, overlapped with hashing
    int rc = ensure_tables(ctx, y, d_flags, err);  // syncs only when Y changed
    if (rc) return rc;
    uint32_t *d_sum, *d_scr, *d_s;
    uint8_t* d_pre;
    uint8_t* d_verdict;
    UPLOAD(b_s, s_hat, 32, d_s);
    ENSURE(b_pre, 256, d_pre);
    ENSURE(b_verdict, 1, d_verdict);
    CU(cudaEventRecord(ctx->ev_side[0], ctx->stream));
    CU(cudaStreamWaitEvent(ctx->side, ctx->ev_side[0], 0));
    launch_check_pre(ctx->d_tabB, d_s, d_rhat, d_pre, ctx->side);
    ctx->launches += 1;
    CU(cudaEventRecord(ctx->ev_side[1], ctx->side));
    // 4. e-hat = sum of agg_ekeys (:83-85)
    Prepared P;
    P.want_etilde = false;
    rc = run_hash(ctx, b, P, err);
    if (rc) {
        cudaStreamSynchronize(ctx->side);
        return rc;
    }
    mark(ctx, kEvSum);
    ENSURE(b_sum, 8, d_sum);
    ENSURE(b_scratch, 17 * 1024, d_scr);
    launch_sum_mod_l(P.sum_src, P.sum_limbs, b->n_epochs, nullptr, d_sum, d_scr, ctx->stream);
    ctx->launches += 2;
    mark(ctx, kEvGroup);
    // 5. one commitment check (:86): e-hat * Y == R - s*alpha, then ONE
    // synchronisation for the error word, the fold's counter and the verdict
    CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_side[1], 0));
    launch_check_post(ctx->d_tabY, d_sum, d_pre, d_verdict, ctx->stream);
    ctx->launches += 1;
    CU(cudaGetLastError());
    PinnedStage* hs = ctx->stage;
    CU(cudaMemcpyAsync(&hs->err_key, ctx->b_err.p, 8, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(hs->flags, d_flags, 16, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(&hs->verdict, d_verdict, 1, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    rc = map_hash_error(hs->err_key, b, err);
    if (rc) return rc;
    if (!r_hat_agg && hs->flags[1]) return set_err(err, POSLO_FORMAT_ERROR, 0, "invalid group element encoding");
    *verdict = hs->verdict;
    // batch_verify.cpp:80 (one group_combine per folded epoch) and :86 (one commit_check)
    if (!r_hat_agg) count_op(ctx, kOpCombine, b->n_epochs);
    count_op(ctx, kOpDoubleExp, 1);
    finish_timing(ctx);
    return ok(err);
}

// R-hat decoding for batched checks: queued on the side stream behind
// everything already on the main stream (their upload), so it overlaps the
// hashing that follows; split_checks waits for it.
static int ensure_scr16e(poslo_gpu_ctx* ctx, uint32_t n, Scr16e& out, poslo_error* err) {
    uint8_t* base;
    ENSURE(b_scr16e, (size_t)std::max<uint32_t>(n, 1) * kCheck16eScratch, base);
    out.P = base;
    out.u2 = base + kGptBytes * (size_t)n;
    out.pre = out.u2 + kFeBytes * (size_t)n;
    return POSLO_OK;
}

static int start_decode(poslo_gpu_ctx* ctx, uint32_t n, const uint8_t* d_r, void** d_pts, uint8_t** d_ok,
                        poslo_error* err) {
    ENSURE(b_dpts, (size_t)std::max<uint32_t>(n, 1) * kPointBytes, *d_pts);
    ENSURE(b_dok, std::max<uint32_t>(n, 1), *d_ok);
    CU(cudaEventRecord(ctx->ev_side[0], ctx->stream));
    CU(cudaStreamWaitEvent(ctx->side, ctx->ev_side[0], 0));
    launch_decode_points(d_r, n, *d_pts, *d_ok, ctx->side);
    ctx->launches += n ? 1 : 0;
    CU(cudaEventRecord(ctx->ev_side[1], ctx->side));
    return POSLO_OK;
}

static int split_checks(poslo_gpu_ctx* ctx, uint32_t n, const uint32_t* d_e, const uint32_t* d_s, const uint8_t* d_r,
                        const void* d_pts, const uint8_t* d_ok, uint8_t* d_verdict, poslo_error* err,
                        const Scr16e& scr) {
    if (d_pts) CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_side[1], 0));  // the R-hat decode
    launch_checks(ctx, n >= comb16_min(), n, d_e, d_s, d_r, d_pts, d_ok, d_verdict, ctx->stream, scr);
    ctx->launches += n ? 1 : 0;
    CU(cudaGetLastError());
    return POSLO_OK;
}

// Per-epoch signature arrays (s-hat LE, R-hat): device pointers as given when
// the batch is device-resident, else uploaded.
static int sig_arrays(poslo_gpu_ctx* ctx, const poslo_batch* b, const uint8_t* s_hats, const uint8_t* r_hats,
                      const uint32_t** d_s_out, const uint8_t** d_r_out, poslo_error* err) {
    if (b->device_resident) {
        if (b->n_epochs && (!device_readable(s_hats) || !device_readable(r_hats)))
            return set_err(err, POSLO_INVALID_ARGUMENT, 0, "device_resident batch with host signature arrays");
        *d_s_out = reinterpret_cast<const uint32_t*>(s_hats);
        *d_r_out = r_hats;
        return POSLO_OK;
    }
    uint32_t* d_s;
    uint8_t* d_r;
    UPLOAD(b_s, s_hats, (size_t)b->n_epochs * 32, d_s);
    UPLOAD(b_r, r_hats, (size_t)b->n_epochs * 32, d_r);
    *d_s_out = d_s;
    *d_r_out = d_r;
    return POSLO_OK;
}

int poslo_gpu_epoch_verify(poslo_gpu_ctx* ctx, const poslo_batch* b, const uint8_t y[32],
                           const uint8_t* s_hats, const uint8_t* r_hats, uint8_t* verdicts,
                           uint8_t* e_tilde_out, poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!b || !y || (b->n_epochs && (!s_hats || !r_hats || !verdicts)))
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (!ctx->members.empty()) return multi_epoch_verify(ctx, b, y, s_hats, r_hats, verdicts, e_tilde_out, err);
    Guard g(ctx);
    if (!b->device_resident)  // device-resident signature arrays were validated when parsed
        for (uint32_t k = 0; k < b->n_epochs; k++)
            if (!scalar_canonical(s_hats + 32 * (size_t)k))
                return set_err(err, POSLO_FORMAT_ERROR, 0, "non-canonical scalar");
    const uint32_t n = b->n_epochs;
    const bool split = n > kCtaCheckMax;
    const uint32_t* d_s = nullptr;
    const uint8_t* d_r = nullptr;
    void* d_pts = nullptr;
    uint8_t* d_ok = nullptr;
    int rc;
    bool want_decode = false;
    Scr16e scr;  // the square-root-free checks (Check16::Sqrt)
    if (split) {  // tables and R-hat decoding ahead of (and overlapping) the hashing
        int* d_flags;
        ENSURE(b_flags, 4, d_flags);
        CU(cudaMemsetAsync(d_flags, 0, 16, ctx->stream));
        rc = ensure_tables(ctx, y, d_flags, err, true, n >= comb16_min());
        if (rc) return rc;
        rc = sig_arrays(ctx, b, s_hats, r_hats, &d_s, &d_r, err);
        if (rc) return rc;
        // radix 256 (n < comb16_min) and the decode / split forms check against
        // R-hat decoded while the log is hashed; the default radix-2^16 form
        // needs no decode (launch_check16e)
        const Check16 mode = check16_mode();
        want_decode = n < comb16_min() || mode == Check16::Decode || mode == Check16::Split;
        if (n >= comb16_min() && mode == Check16::Sqrt) {
            rc = ensure_scr16e(ctx, n, scr, err);
            if (rc) return rc;
        }
        if (want_decode && decode_early()) {
            rc = start_decode(ctx, n, d_r, &d_pts, &d_ok, err);
            if (rc) return rc;
            want_decode = false;
        }
    }
    Prepared P;
    if (want_decode) P.on_seeded = [&]() { return start_decode(ctx, n, d_r, &d_pts, &d_ok, err); };
    uint8_t* d_vpipe = nullptr;
    bool piped = false;
    if (split && b->device_resident) {  // checks of piece q overlap the hashing of piece q + 1
        ENSURE(b_verdict, n, d_vpipe);
        P.on_piece = [&](uint32_t e0, uint32_t e1, cudaStream_t hs) -> int {
            CU(cudaEventRecord(ctx->ev_side[0], hs));
            CU(cudaStreamWaitEvent(ctx->side, ctx->ev_side[0], 0));  // side: after the decode, then this piece
            launch_checks(ctx, n >= comb16_min(), e1 - e0, P.d_etilde + 8 * (size_t)e0, d_s + 8 * (size_t)e0,
                          d_r + 32 * (size_t)e0,
                          d_pts ? static_cast<const uint8_t*>(d_pts) + kPointBytes * (size_t)e0 : nullptr,
                          d_ok ? d_ok + e0 : nullptr, d_vpipe + e0, ctx->side, scr.at(e0));
            ctx->launches += 1;
            piped = true;
            return POSLO_OK;
        };
    }
    rc = run_hash(ctx, b, P, err);
    if (rc) {
        cudaStreamSynchronize(ctx->side);
        return rc;
    }
    mark(ctx, kEvSum);
    if (!split) {
        rc = sig_arrays(ctx, b, s_hats, r_hats, &d_s, &d_r, err);
        if (rc) return rc;
    }
    mark(ctx, kEvGroup);
    rc = check_hash_errors(ctx, b, err);
    if (rc) {
        cudaStreamSynchronize(ctx->side);
        return rc;
    }
    if (split && piped) {
        CU(cudaEventRecord(ctx->ev_side[1], ctx->side));
        CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_side[1], 0));
        CU(cudaMemcpyAsync(verdicts, d_vpipe, n, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
    } else if (split) {
        uint8_t* d_verdict;
        ENSURE(b_verdict, n, d_verdict);
        rc = split_checks(ctx, n, P.d_etilde, d_s, d_r, d_pts, d_ok, d_verdict, err, scr);
        if (rc) return rc;
        CU(cudaMemcpyAsync(verdicts, d_verdict, n, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
    } else {
        rc = group_check_dev(ctx, y, n, P.d_etilde, d_s, d_r, verdicts, nullptr, err);
        if (rc) return rc;
    }
    if (e_tilde_out && b->n_epochs)
        CU(cudaMemcpy(e_tilde_out, P.d_etilde, (size_t)b->n_epochs * 32, cudaMemcpyDeviceToHost));
    count_op(ctx, kOpDoubleExp, n);  // one commit_check per epoch
    finish_timing(ctx);
    return ok(err);
}

// Masked segmented folds on device buffers (scalars: n x 8 limbs; points:
// n x 32 B encodings); results to host. mask: keep item k iff mask[k] != 0.
static int segfold_dev(poslo_gpu_ctx* ctx, uint32_t n, const uint32_t* d_s, const uint8_t* d_r, const uint8_t* d_mask,
                const uint32_t* seg, uint32_t n_seg, uint8_t* out_s, uint8_t* out_r, poslo_error* err) {
    if (!n_seg) return POSLO_OK;
    for (uint32_t g = 0; g < n_seg; g++)
        if (seg[g] > seg[g + 1] || seg[g + 1] > n)
            return set_err(err, POSLO_INVALID_ARGUMENT, 0, "segments must be non-decreasing within [0, n]");
    cudaStream_t s = ctx->stream;
    if (d_s && out_s) {
        std::vector<uint64_t> seg64(seg, seg + n_seg + 1);
        uint64_t* d_seg;
        uint32_t* d_out;
        UPLOAD(b_seg, seg64.data(), seg64.size() * 8, d_seg);
        ENSURE(b_out_s, (size_t)n_seg * 8, d_out);
        launch_segsum_mod_l(d_s, d_seg, n_seg, d_mask, d_out, s, /*skip_val=*/0);
        ctx->launches += 1;
        CU(cudaMemcpyAsync(out_s, d_out, (size_t)n_seg * 32, cudaMemcpyDeviceToHost, s));
    }
    if (d_r && out_r) {
        uint32_t* d_seg;
        uint8_t* d_out;
        int* d_bad;
        UPLOAD(b_seg32, seg, (size_t)(n_seg + 1) * 4, d_seg);
        ENSURE(b_out_r, (size_t)n_seg * 32, d_out);
        ENSURE(b_flags, 4, d_bad);
        CU(cudaMemsetAsync(d_bad, 0, 4, s));
        launch_segfold_points(d_r, d_seg, n_seg, d_mask, d_out, d_bad, s);
        ctx->launches += 1;
        CU(cudaMemcpyAsync(out_r, d_out, (size_t)n_seg * 32, cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(ctx->stage->flags, d_bad, 4, cudaMemcpyDeviceToHost, s));
        CU(cudaStreamSynchronize(s));
        if (ctx->stage->flags[0]) return set_err(err, POSLO_FORMAT_ERROR, 0, "invalid group element encoding");
    }
    CU(cudaStreamSynchronize(s));
    return POSLO_OK;
}

int poslo_gpu_segfold(poslo_gpu_ctx* ctx, uint32_t n, const uint8_t* scalars, const uint8_t* points,
                      const uint8_t* mask, const uint32_t* seg, uint32_t n_seg, uint8_t* out_s, uint8_t* out_r,
                      poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (n_seg && !seg) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null segments");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    Guard g(ctx);
    uint32_t* d_s = nullptr;
    uint8_t* d_r = nullptr;
    uint8_t* d_mask = nullptr;
    if (scalars && out_s) UPLOAD(b_s, scalars, (size_t)std::max<uint32_t>(n, 1) * 32, d_s);
    if (points && out_r) UPLOAD(b_r, points, (size_t)std::max<uint32_t>(n, 1) * 32, d_r);
    if (mask) UPLOAD(b_mask, mask, std::max<uint32_t>(n, 1), d_mask);
    int rc = segfold_dev(ctx, n, d_s, d_r, d_mask, seg, n_seg, out_s, out_r, err);
    if (rc) return rc;
    if (points && out_r) {  // group_combine per folded point
        uint64_t kept = 0;
        for (uint32_t g2 = 0; g2 < n_seg; g2++)
            for (uint32_t k = seg[g2]; k < seg[g2 + 1]; k++) kept += !mask || mask[k];
        count_op(ctx, kOpCombine, kept);
    }
    return ok(err);
}

int poslo_gpu_distill_coarse(poslo_gpu_ctx* ctx, const poslo_batch* b, const uint8_t y[32],
                             const uint8_t* s_hats, const uint8_t* r_hats, const uint32_t* seg, uint32_t n_seg,
                             uint8_t* verdicts, uint8_t* seg_s, uint8_t* seg_r, poslo_error* err) {
    return poslo_gpu_distill_coarse_ex(ctx, b, y, s_hats, r_hats, seg, n_seg, verdicts, seg_s, seg_r, nullptr, err);
}

int poslo_gpu_distill_coarse_ex(poslo_gpu_ctx* ctx, const poslo_batch* b, const uint8_t y[32],
                                const uint8_t* s_hats, const uint8_t* r_hats, const uint32_t* seg, uint32_t n_seg,
                                uint8_t* verdicts, uint8_t* seg_s, uint8_t* seg_r, uint8_t* seg_e, poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!ctx->members.empty())
        return multi_distill_coarse(ctx, b, y, s_hats, r_hats, seg, n_seg, verdicts, seg_s, seg_r, seg_e, err);
    if (!b || !y || (b->n_epochs && (!s_hats || !r_hats || !verdicts)) || (n_seg && !seg))
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "bad argument");
    Guard g(ctx);
    // aver (poslo_c.cpp:195-197): every epoch must hold exactly n2 entries
    if (b->epoch_starts)
        for (uint32_t k = 0; k < b->n_epochs; k++)
            if (b->epoch_starts[k + 1] - b->epoch_starts[k] != b->n2)
                return set_err(err, POSLO_STATE_ERROR, b->epochs[k], "every batch must hold exactly n2 entries");
    const uint32_t n = b->n_epochs;
    const bool split = n > kCtaCheckMax;
    const uint32_t* d_s = nullptr;
    const uint8_t* d_r = nullptr;
    void* d_pts = nullptr;
    uint8_t* d_ok = nullptr;
    int* d_flags;
    ENSURE(b_flags, 4, d_flags);
    CU(cudaMemsetAsync(d_flags, 0, 16, ctx->stream));
    int rc = ensure_tables(ctx, y, d_flags, err, split, split && n >= comb16_min());
    if (rc) return rc;
    if (n) {
        rc = sig_arrays(ctx, b, s_hats, r_hats, &d_s, &d_r, err);
        if (rc) return rc;
    }
    // Radix-2^16 checks with no square root per check keep the points
    // P_i = e_i Y + s_i B, and for a valid epoch P_i IS R-hat_i as a ristretto
    // element (encode(P_i) == R-hat_i), so the umbrella folds add the P_i of
    // the valid epochs: R-hat is never decoded. The other forms decode R-hat
    // once, on the side stream during hashing, for the fold and the checks.
    const bool sqrt16 = split && n >= comb16_min() && check16_mode() == Check16::Sqrt;
    Scr16e scr;
    if (sqrt16) {
        rc = ensure_scr16e(ctx, n, scr, err);
        if (rc) return rc;
    }
    if (split && !sqrt16 && decode_early()) {
        rc = start_decode(ctx, n, d_r, &d_pts, &d_ok, err);
        if (rc) return rc;
    }
    Prepared P;
    if (split && !sqrt16 && !decode_early())
        P.on_seeded = [&]() { return start_decode(ctx, n, d_r, &d_pts, &d_ok, err); };
    // per-epoch verdicts stay on the device as the fold mask
    uint8_t* d_verdict;
    ENSURE(b_verdict, std::max<uint32_t>(n, 1), d_verdict);
    bool piped = false;
    if (split && b->device_resident) {  // checks of piece q overlap the hashing of piece q + 1
        P.on_piece = [&](uint32_t e0, uint32_t e1, cudaStream_t hs) -> int {
            CU(cudaEventRecord(ctx->ev_side[0], hs));
            CU(cudaStreamWaitEvent(ctx->side, ctx->ev_side[0], 0));
            launch_checks(ctx, n >= comb16_min(), e1 - e0, P.d_etilde + 8 * (size_t)e0, d_s + 8 * (size_t)e0,
                          d_r + 32 * (size_t)e0,
                          d_pts ? static_cast<const uint8_t*>(d_pts) + kPointBytes * (size_t)e0 : nullptr,
                          d_ok ? d_ok + e0 : nullptr, d_verdict + e0, ctx->side, scr.at(e0));
            ctx->launches += 1;
            piped = true;
            return POSLO_OK;
        };
    }
    rc = run_hash(ctx, b, P, err);
    if (!rc) rc = check_hash_errors(ctx, b, err);
    if (rc) {
        cudaStreamSynchronize(ctx->side);
        return rc;
    }
    if (!n) return ok(err);
    mark(ctx, kEvSum);
    mark(ctx, kEvGroup);
    if (split && piped) {
        CU(cudaEventRecord(ctx->ev_side[1], ctx->side));
        CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_side[1], 0));
    } else if (split) {
        rc = split_checks(ctx, n, P.d_etilde, d_s, d_r, d_pts, d_ok, d_verdict, err, scr);
        if (rc) return rc;
    } else {
        launch_group_check_comb(ctx->d_tabY, ctx->d_tabB, ctx->d_tabY256, ctx->d_tabB256, n, P.d_etilde, d_s,
                                d_r, nullptr, d_verdict, ctx->stream);
        ctx->launches += 1;
    }
    CU(cudaMemcpyAsync(verdicts, d_verdict, n, cudaMemcpyDeviceToHost, ctx->stream));
    if (seg_e && n_seg) {  // e-sums of the valid epochs per segment (SeBVer mode U's operand)
        for (uint32_t g2 = 0; g2 < n_seg; g2++)
            if (seg[g2] > seg[g2 + 1] || seg[g2 + 1] > n)
                return set_err(err, POSLO_INVALID_ARGUMENT, 0, "segments must be non-decreasing within [0, n]");
        std::vector<uint64_t> seg64(seg, seg + n_seg + 1);
        uint64_t* d_seg;
        uint32_t* d_out;
        UPLOAD(b_seg_e, seg64.data(), seg64.size() * 8, d_seg);
        ENSURE(b_out_e, (size_t)n_seg * 8, d_out);
        launch_segsum_mod_l(P.d_etilde, d_seg, n_seg, d_verdict, d_out, ctx->stream, /*skip_val=*/0);
        ctx->launches += 1;
        CU(cudaMemcpyAsync(seg_e, d_out, (size_t)n_seg * 32, cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (split) {  // scalars as before; points from the checks' P_i or the decoded R-hats (no second decode)
        rc = segfold_dev(ctx, n, d_s, nullptr, d_verdict, seg, n_seg, seg_s, nullptr, err);
        if (rc) return rc;
        if (n_seg) {
            for (uint32_t g2 = 0; g2 < n_seg; g2++)
                if (seg[g2] > seg[g2 + 1] || seg[g2 + 1] > n)
                    return set_err(err, POSLO_INVALID_ARGUMENT, 0, "segments must be non-decreasing within [0, n]");
            uint32_t* d_seg;
            uint8_t* d_out;
            UPLOAD(b_seg32, seg, (size_t)(n_seg + 1) * 4, d_seg);
            ENSURE(b_out_r, (size_t)n_seg * 32, d_out);
            CU(cudaStreamWaitEvent(ctx->stream, ctx->ev_side[1], 0));  // the R-hat decode / piped checks
            launch_segfold_decoded(sqrt16 ? static_cast<const void*>(scr.P) : d_pts, d_seg, n_seg, d_verdict, d_out,
                                   ctx->stream);
            ctx->launches += 1;
            CU(cudaMemcpyAsync(seg_r, d_out, (size_t)n_seg * 32, cudaMemcpyDeviceToHost, ctx->stream));
        }
        CU(cudaStreamSynchronize(ctx->stream));
    } else {
        rc = segfold_dev(ctx, n, d_s, d_r, d_verdict, seg, n_seg, seg_s, seg_r, err);
        if (rc) return rc;
    }
    CU(cudaStreamSynchronize(ctx->stream));
    // per epoch, aver (poslo_c.cpp:199-212: one R-hat combine, one commit_check),
    // then fold_valid (distiller.cpp:45-53: two combines per valid epoch)
    uint64_t n_valid = 0;
    for (uint32_t k = 0; k < n; k++) n_valid += verdicts[k] != 0;
    count_op(ctx, kOpDoubleExp, n);
    count_op(ctx, kOpCombine, n + 2 * n_valid);
    finish_timing(ctx);
    return ok(err);
}

// One distill_epoch (distiller.cpp:60-89) in ONE device round trip: hash,
// check, and on a valid verdict the fold of (s-hat, R-hat) into both running
// aggregates (fold_valid, :45-53), all queued on the stream; the hash error
// word, the verdict and the two updated pairs come back in one pinned copy.
int poslo_gpu_distill_step(poslo_gpu_ctx* ctx, const poslo_batch* b, const uint8_t y[32], const uint8_t s_hat[32],
                           const uint8_t r_hat[32], const uint8_t acc_s[64], const uint8_t acc_r[64],
                           uint8_t* verdict, uint8_t out_s[64], uint8_t out_r[64], poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!b || !y || !s_hat || !r_hat || !acc_s || !acc_r || !verdict || !out_s || !out_r)
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (b->n_epochs != 1 || b->device_resident)
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "distill_step takes one host-resident epoch");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    Guard g(ctx);
    if (b->epoch_starts && b->epoch_starts[1] - b->epoch_starts[0] != b->n2)
        return set_err(err, POSLO_STATE_ERROR, b->epochs[0], "every batch must hold exactly n2 entries");
    if (!scalar_canonical(s_hat) || !scalar_canonical(acc_s) || !scalar_canonical(acc_s + 32))
        return set_err(err, POSLO_FORMAT_ERROR, 0, "non-canonical scalar");
    cudaStream_t s = ctx->stream;
    int* d_flags;
    ENSURE(b_flags, 4, d_flags);
    CU(cudaMemsetAsync(d_flags, 0, 16, s));
    int rc = ensure_tables(ctx, y, d_flags, err);
    if (rc) return rc;
    // scalars [valid acc, s_hat, umbrella acc], points [valid acc, R-hat, umbrella acc]
    uint8_t items[192];
    std::memcpy(items, acc_s, 32);
    std::memcpy(items + 32, s_hat, 32);
    std::memcpy(items + 64, acc_s + 32, 32);
    std::memcpy(items + 96, acc_r, 32);
    std::memcpy(items + 128, r_hat, 32);
    std::memcpy(items + 160, acc_r + 32, 32);
    uint8_t* d_items;
    UPLOAD(b_s, items, sizeof items, d_items);
    Prepared P;
    rc = run_hash(ctx, b, P, err);
    if (rc) return rc;
    uint8_t *d_verdict, *d_out_r;
    uint32_t* d_out_s;
    ENSURE(b_verdict, 1, d_verdict);
    ENSURE(b_out_s, 16, d_out_s);
    ENSURE(b_out_r, 64, d_out_r);
    // check + both folds in one CTA: the decodes run beside the comb, the
    // verdict is a projective comparison, the two new aggregates encode at once
    launch_distill_step(ctx->d_tabY, ctx->d_tabB, P.d_etilde, reinterpret_cast<const uint32_t*>(d_items),
                        d_items + 96, d_verdict, d_out_s, d_out_r, d_flags + 1, s);
    ctx->launches += 1;
    PinnedStage* st = ctx->stage;
    CU(cudaMemcpyAsync(&st->err_key, ctx->b_err.p, 8, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(&st->verdict, d_verdict, 1, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(st->flags, d_flags, 8, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(st->step_out, d_out_s, 64, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(st->step_out + 64, d_out_r, 64, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    rc = map_hash_error(st->err_key, b, err);
    if (rc) return rc;
    if (st->flags[0]) return set_err(err, POSLO_FORMAT_ERROR, 0, "invalid group element encoding (Y)");
    if (st->flags[1]) return set_err(err, POSLO_FORMAT_ERROR, 0, "invalid group element encoding");
    *verdict = st->verdict;
    std::memcpy(out_s, st->step_out, 64);
    std::memcpy(out_r, st->step_out + 64, 64);
    count_op(ctx, kOpDoubleExp, 1);
    count_op(ctx, kOpCombine, 1 + (st->verdict ? 2 : 0));
    finish_timing(ctx);
    return ok(err);
}

// ---- scheme F ----------------------------------------------------------------
// Per-entry scalars of a fine batch into device memory (d_e: n x 8 limbs).
static int fine_scalars_dev(poslo_gpu_ctx* ctx, const poslo_fine_batch* fb, uint32_t** d_e_out, poslo_error* err) {
    if (!fb) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null batch");
    if (fb->suite < 1 || fb->suite > 3) return set_err(err, POSLO_FORMAT_ERROR, 0, "unknown suite id");
    const uint64_t n = fb->n_entries;
    if (n >= (1ull << 62)) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "too many entries");
    if (n && !fb->derive_slot && !fb->seeds) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null seeds");
    if (fb->derive_slot && (!fb->j || (fb->n_slots && !fb->slot_epochs)))
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "derived seeds need j and slot_epochs");
    cudaStream_t s = ctx->stream;
    // seeds of derived entries: host-resolved covers, one walk per slot
    std::vector<uint64_t> first(fb->n_slots, ~0ull);
    if (fb->derive_slot)
        for (uint64_t t = 0; t < n; t++) {
            const uint32_t sl = fb->derive_slot[t];
            if (sl == 0xFFFFFFFFu) continue;
            if (sl >= fb->n_slots) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "derive_slot out of range");
            first[sl] = std::min<uint64_t>(first[sl], t);
        }
    unsigned long long host_err = ~0ull;
    std::vector<SeedStart> starts;
    uint4* d_x0 = nullptr;
    if (fb->derive_slot && fb->n_slots) {
        int rc = resolve_seed_starts(fb->ds, fb->ds_len, fb->ds_offsets, fb->ds_capacity, fb->slot_epochs, fb->n_slots,
                                     starts, first.data(), &host_err, err);
        if (rc) return rc;
        for (uint32_t k = 0; k < fb->n_slots; k++)  // slots no entry uses cannot fail
            if (first[k] == ~0ull && host_err == (~0ull << 1)) host_err = ~0ull;
        SeedStart* d_starts;
        ENSURE(b_starts_ds, fb->n_slots, d_starts);
        ENSURE(b_x0, fb->n_slots, d_x0);
        CU(cudaMemcpyAsync(d_starts, starts.data(), starts.size() * sizeof(SeedStart), cudaMemcpyHostToDevice, s));
        launch_seed_walk(fb->suite, d_starts, fb->n_slots, d_x0, ctx->d_t0, s);
        ctx->launches += 1;
    }
    // entries
    EntryLayout lay{};
    lay.entry_len = fb->entry_len;
    if (fb->device_resident) {
        if ((fb->payload_bytes && !device_readable(fb->payload)) || !device_readable(fb->offsets))
            return set_err(err, POSLO_INVALID_ARGUMENT, 0, "device_resident batch with a host pointer");
        lay.payload = fb->payload;
        lay.offsets = fb->offsets;
    } else {
        uint8_t* d_pay;
        ENSURE(b_payload, fb->payload_bytes, d_pay);
        if (fb->payload_bytes) CU(cudaMemcpyAsync(d_pay, fb->payload, fb->payload_bytes, cudaMemcpyHostToDevice, s));
        lay.payload = d_pay;
        if (fb->offsets) {
            uint64_t* d_off;
            ENSURE(b_offsets, n + 1, d_off);
            CU(cudaMemcpyAsync(d_off, fb->offsets, (n + 1) * 8, cudaMemcpyHostToDevice, s));
            lay.offsets = d_off;
        }
    }
    uint4* d_seeds = nullptr;
    uint32_t *d_slot = nullptr, *d_j = nullptr, *d_e;
    unsigned long long* d_err;
    if (fb->seeds) UPLOAD(b_pts, fb->seeds, (size_t)std::max<uint64_t>(n, 1) * 16, d_seeds);
    if (fb->derive_slot) {
        UPLOAD(b_epochs, fb->derive_slot, (size_t)std::max<uint64_t>(n, 1) * 4, d_slot);
        UPLOAD(b_tbegin, fb->j, (size_t)std::max<uint64_t>(n, 1) * 4, d_j);
    }
    ENSURE(b_e, (size_t)std::max<uint64_t>(n, 1) * 8, d_e);
    ENSURE(b_err, 1, d_err);
    ctx->stage->err_init = host_err;
    CU(cudaMemcpyAsync(d_err, &ctx->stage->err_init, 8, cudaMemcpyHostToDevice, s));
    launch_fine_scalars(fb->suite, lay, n, d_seeds, d_slot, d_j, d_x0, d_e, d_err, ctx->d_t0, s);
    ctx->launches += n ? 1 : 0;
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(&ctx->stage->err_key, d_err, 8, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    const unsigned long long key = ctx->stage->err_key;
    if (key != ~0ull) {
        const uint64_t t = key >> 1;
        if ((key & 1) == 0) {
            const uint32_t ep = fb->derive_slot && t < n && fb->derive_slot[t] < fb->n_slots
                                    ? fb->slot_epochs[fb->derive_slot[t]] : 0;
            return set_err(err, POSLO_SEED_NOT_DISCLOSED, ep, "seed for epoch %u not yet disclosed", ep);
        }
        return set_err(err, POSLO_FORMAT_ERROR, (uint32_t)t, "modular-addition hash: entry too long for this suite");
    }
    *d_e_out = d_e;
    return POSLO_OK;
}

int poslo_gpu_fine_scalars(poslo_gpu_ctx* ctx, const poslo_fine_batch* fb, uint8_t* e_out, uint8_t* e_sum,
                           poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    Guard g(ctx);
    uint32_t* d_e;
    int rc = fine_scalars_dev(ctx, fb, &d_e, err);
    if (rc) return rc;
    if (e_sum) {
        uint32_t *d_sum, *d_scr;
        ENSURE(b_sum, 8, d_sum);
        ENSURE(b_scratch, 17 * 1024, d_scr);
        launch_sum_mod_l(d_e, 8, fb->n_entries, nullptr, d_sum, d_scr, ctx->stream);
        ctx->launches += 2;
        CU(cudaMemcpyAsync(e_sum, d_sum, 32, cudaMemcpyDeviceToHost, ctx->stream));
    }
    if (e_out && fb->n_entries)
        CU(cudaMemcpyAsync(e_out, d_e, fb->n_entries * 32, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return ok(err);
}

int poslo_gpu_fine_verify(poslo_gpu_ctx* ctx, const poslo_fine_batch* fb, const uint8_t y[32], const uint8_t* s,
                          const uint8_t* r, uint8_t* verdicts, poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!fb || !y || (fb->n_entries && (!s || !r || !verdicts)))
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "bad argument");
    if (fb->n_entries > 0xFFFFFFFFull) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "too many entries");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    // FineSignature::s was parsed with Scalar::from_be_bytes (< l): refuse others
    for (uint64_t t = 0; t < fb->n_entries; t++)
        if (!scalar_canonical(s + 32 * t)) return set_err(err, POSLO_FORMAT_ERROR, 0, "non-canonical scalar");
    Guard g(ctx);
    uint32_t* d_e;
    int rc = fine_scalars_dev(ctx, fb, &d_e, err);
    if (rc) return rc;
    const uint32_t n = (uint32_t)fb->n_entries;
    if (!n) return ok(err);
    count_op(ctx, kOpDoubleExp, n);
    uint32_t* d_s;
    uint8_t* d_r;
    UPLOAD(b_s, s, (size_t)n * 32, d_s);
    UPLOAD(b_r, r, (size_t)n * 32, d_r);
    rc = group_check_dev(ctx, y, n, d_e, d_s, d_r, verdicts, nullptr, err);
    if (rc) return rc;
    return ok(err);
}

int poslo_gpu_aver_f_batch(poslo_gpu_ctx* ctx, const poslo_fine_batch* fb, const uint8_t y[32], const uint8_t s[32],
                           const uint8_t r[32], uint8_t* verdict, poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!fb || !y || !s || !r || !verdict) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "bad argument");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    if (!scalar_canonical(s)) return set_err(err, POSLO_FORMAT_ERROR, 0, "non-canonical scalar");
    Guard g(ctx);
    uint32_t* d_e;
    int rc = fine_scalars_dev(ctx, fb, &d_e, err);
    if (rc) return rc;
    count_op(ctx, kOpDoubleExp, 1);
    uint32_t *d_sum, *d_scr, *d_s;
    uint8_t* d_r;
    ENSURE(b_sum, 8, d_sum);
    ENSURE(b_scratch, 17 * 1024, d_scr);
    launch_sum_mod_l(d_e, 8, fb->n_entries, nullptr, d_sum, d_scr, ctx->stream);  // empty: e_sum = 0
    ctx->launches += 2;
    UPLOAD(b_s, s, 32, d_s);
    UPLOAD(b_r, r, 32, d_r);
    rc = group_check_dev(ctx, y, 1, d_sum, d_s, d_r, verdict, nullptr, err);
    if (rc) return rc;
    return ok(err);
}

int poslo_gpu_sebver(poslo_gpu_ctx* ctx, const poslo_batch* b, const uint8_t y[32], uint32_t n1,
                     uint32_t n_u, const uint32_t* invalid, const uint8_t* invalid_s,
                     const uint8_t* invalid_r, uint32_t n_invalid, const uint8_t* v_s,
                     const uint8_t* v_r, uint8_t* v_bit, const uint32_t* umb_index,
                     const uint8_t* umb_s, const uint8_t* umb_r, uint32_t n_umb, uint8_t* u_bits,
                     uint8_t* i_bits, poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    if (!b || !y || n_u == 0 || n1 % n_u) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "bad argument");
    if ((n_invalid && (!invalid || (i_bits && (!invalid_s || !invalid_r)))) || (v_bit && (!v_s || !v_r)) ||
        (u_bits && n_umb && (!umb_index || !umb_s || !umb_r)))
        return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    // CCD scalars were parsed with Scalar::from_be_bytes (< l); the comb digit
    // recoding relies on it, so a C-ABI caller's non-canonical scalar is refused
    auto canon = [](const uint8_t* p, uint32_t cnt) {
        for (uint32_t k = 0; k < cnt; k++)
            if (!scalar_canonical(p + 32 * (size_t)k)) return false;
        return true;
    };
    if ((i_bits && !canon(invalid_s, n_invalid)) || (v_bit && !canon(v_s, 1)) || (u_bits && !canon(umb_s, n_umb)))
        return set_err(err, POSLO_FORMAT_ERROR, 0, "non-canonical scalar");
    Guard g(ctx);
    Prepared P;
    int rc = run_hash(ctx, b, P, err);  // only the epochs SeBVer reads are in the batch
    if (rc) return rc;
    rc = check_hash_errors(ctx, b, err);
    if (rc) return rc;
    cudaStream_t s = ctx->stream;
    const uint32_t n_ep = b->n_epochs;
    const uint32_t* ep = b->epochs;
    // batch position of the first epoch >= e (the batch is ascending)
    auto pos = [&](uint64_t e) -> uint64_t {
        if (e > 0xFFFFFFFFull) return n_ep;
        return (uint64_t)(std::lower_bound(ep, ep + n_ep, (uint32_t)e) - ep);
    };
    std::vector<uint8_t> mask(std::max<uint32_t>(n_ep, 1), 0);  // 1 = invalid epoch: left out of every e-sum
    for (uint32_t k = 0; k < n_invalid; k++) {
        const uint64_t q = pos(invalid[k]);
        if (q < n_ep && ep[q] == invalid[k]) mask[q] = 1;
    }
    uint8_t* d_mask;
    UPLOAD(b_mask, mask.data(), mask.size(), d_mask);
    const uint32_t w = n1 / n_u;
    // groups: [V] + U umbrellas + I records, e per group on device
    const uint32_t nV = v_bit ? 1 : 0, nU = u_bits ? n_umb : 0, nI = i_bits ? n_invalid : 0;
    const uint32_t ng = nV + nU + nI;
    if (!ng) return ok(err);
    std::vector<uint64_t> seg;
    std::vector<uint8_t> hs((size_t)ng * 32), hr((size_t)ng * 32);
    uint32_t gi = 0;
    if (nV) {  // every batch epoch (the distilled ones that SeBVer hashes)
        seg.push_back(0);
        seg.push_back(n_ep);
        std::memcpy(&hs[0], v_s, 32);
        std::memcpy(&hr[0], v_r, 32);
        gi++;
    }
    for (uint32_t u = 0; u < nU; u++, gi++) {  // batch epochs in [u w, (u + 1) w)
        seg.push_back(pos((uint64_t)umb_index[u] * w));
        seg.push_back(pos((uint64_t)(umb_index[u] + 1) * w));
        std::memcpy(&hs[32 * gi], umb_s + 32 * (size_t)u, 32);
        std::memcpy(&hr[32 * gi], umb_r + 32 * (size_t)u, 32);
    }
    uint32_t* d_e;
    ENSURE(b_e, (size_t)ng * 8, d_e);
    const uint32_t n_seg_groups = nV + nU;
    if (n_seg_groups) {  // one masked sum per [lo, hi) pair
        uint64_t* d_seg;
        UPLOAD(b_seg, seg.data(), seg.size() * 8, d_seg);
        for (uint32_t g2 = 0; g2 < n_seg_groups; g2++) {
            launch_segsum_mod_l(P.d_etilde, d_seg + 2 * g2, 1, d_mask, d_e + 8 * g2, s);
            ctx->launches += 1;
        }
    }
    for (uint32_t k = 0; k < nI; k++, gi++) {
        const uint32_t e = invalid[k];
        const uint64_t q = pos(e);
        if (q >= n_ep || ep[q] != e) return set_err(err, POSLO_FORMAT_ERROR, e, "messages for invalid epoch missing");
        CU(cudaMemcpyAsync(d_e + 8 * (size_t)gi, P.d_etilde + 8 * q, 32, cudaMemcpyDeviceToDevice, s));
        std::memcpy(&hs[32 * gi], invalid_s + 32 * (size_t)k, 32);
        std::memcpy(&hr[32 * gi], invalid_r + 32 * (size_t)k, 32);
    }
    uint32_t* d_s;
    uint8_t* d_r;
    UPLOAD(b_s, hs.data(), hs.size(), d_s);
    UPLOAD(b_r, hr.data(), hr.size(), d_r);
    std::vector<uint8_t> bits(ng);
    rc = group_check_dev(ctx, y, ng, d_e, d_s, d_r, bits.data(), nullptr, err);
    if (rc) return rc;
    count_op(ctx, kOpDoubleExp, ng);  // verify_range / the mode-I check: one commit_check each
    gi = 0;
    if (nV) *v_bit = bits[gi++];
    for (uint32_t u = 0; u < nU; u++) u_bits[u] = bits[gi++];
    for (uint32_t k = 0; k < nI; k++) i_bits[k] = bits[gi++];
    return ok(err);
}

int poslo_gpu_kg_commitments(poslo_gpu_ctx* ctx, uint8_t suite, const uint8_t r_seed[16], const uint32_t* epochs,
                             uint32_t n, uint32_t n2, uint8_t* r_hats_out, uint8_t* r_scalars_out,
                             poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (suite < 1 || suite > 3) return set_err(err, POSLO_FORMAT_ERROR, 0, "unknown suite id");
    if (!r_seed || (n && (!epochs || !r_hats_out))) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    Guard g(ctx);
    if (!n) return ok(err);
    uint32_t rw[4];
    std::memcpy(rw, r_seed, 16);
    uint32_t *d_ep, *d_r, *d_zero;
    UPLOAD(b_epochs, epochs, (size_t)n * 4, d_ep);
    ENSURE(b_s, (size_t)n * 8, d_r);
    ENSURE(b_e, (size_t)n * 8, d_zero);
    CU(cudaMemsetAsync(d_zero, 0, (size_t)n * 32, ctx->stream));
    launch_nonce_sums(suite, rw, d_ep, n, n2, d_r, ctx->d_t0, ctx->stream);
    ctx->launches += 1;
    // R-hat_i = exp_base(r-hat_i) = commit_check(identity, 0, r-hat_i)
    static const uint8_t identity[32] = {0};
    int rc = group_check_dev(ctx, identity, n, d_zero, d_r, nullptr, nullptr, r_hats_out, err);
    if (rc) return rc;
    count_op(ctx, kOpExpBase, n);  // kg: one exp_base per epoch (poslo_c.cpp:91-113)
    if (r_scalars_out) {
        CU(cudaMemcpyAsync(r_scalars_out, d_r, (size_t)n * 32, cudaMemcpyDeviceToHost, ctx->stream));
        CU(cudaStreamSynchronize(ctx->stream));
    }
    return ok(err);
}

int poslo_gpu_sig_epochs(poslo_gpu_ctx* ctx, const poslo_batch* b, const uint8_t r_seed[16], const uint8_t y[32],
                         uint8_t* s_hats_out, poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!b || !r_seed || !y || (b->n_epochs && !s_hats_out)) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (!scalar_canonical(y)) return set_err(err, POSLO_FORMAT_ERROR, 0, "non-canonical scalar");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    Guard g(ctx);
    // sig_epoch (poslo_c.cpp:117-118): every epoch batch holds exactly n2 entries
    if (b->epoch_starts)
        for (uint32_t k = 0; k < b->n_epochs; k++)
            if (b->epoch_starts[k + 1] - b->epoch_starts[k] != b->n2)
                return set_err(err, POSLO_STATE_ERROR, b->epochs[k], "epoch batch must hold exactly n2 entries");
    Prepared P;
    int rc = run_hash(ctx, b, P, err);  // e~ per epoch
    if (!rc) rc = check_hash_errors(ctx, b, err);
    if (rc) return rc;
    const uint32_t n = b->n_epochs;
    if (!n) return ok(err);
    uint32_t rw[4], yw[8];
    std::memcpy(rw, r_seed, 16);
    std::memcpy(yw, y, 32);
    uint32_t *d_ep, *d_r, *d_out;
    UPLOAD(b_seg32, b->epochs, (size_t)n * 4, d_ep);
    ENSURE(b_s, (size_t)n * 8, d_r);
    ENSURE(b_out_s, (size_t)n * 8, d_out);
    launch_nonce_sums(b->suite, rw, d_ep, n, b->n2, d_r, ctx->d_t0, ctx->stream);
    launch_sign_combine(n, d_r, P.d_etilde, yw, d_out, ctx->stream);
    ctx->launches += 2;
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(s_hats_out, d_out, (size_t)n * 32, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return ok(err);
}

int poslo_gpu_commit_check(poslo_gpu_ctx* ctx, uint32_t n, const uint8_t y[32], const uint8_t* e,
                           const uint8_t* s, uint8_t* out, poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!y || (n && (!e || !s || !out))) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    Guard g(ctx);
    for (uint32_t i = 0; i < n; i++)
        if (!scalar_canonical(e + 32 * (size_t)i) || !scalar_canonical(s + 32 * (size_t)i))
            return set_err(err, POSLO_FORMAT_ERROR, 0, "non-canonical scalar");
    uint32_t *d_e, *d_s;
    UPLOAD(b_e, e, (size_t)n * 32, d_e);
    UPLOAD(b_s, s, (size_t)n * 32, d_s);
    int rc = group_check_dev(ctx, y, n, d_e, d_s, nullptr, nullptr, out, err);
    if (rc) return rc;
    bool y_id = true;
    for (int k = 0; k < 32; k++) y_id &= y[k] == 0;
    count_op(ctx, y_id ? kOpExpBase : kOpDoubleExp, n);
    return ok(err);
}

int poslo_gpu_group_fold(poslo_gpu_ctx* ctx, uint64_t n, const uint8_t* pts, uint8_t out[32],
                         poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!out || (n && !pts)) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    Guard g(ctx);
    uint8_t *d_pts, *d_out;
    void* d_fs;
    int* d_flags;
    UPLOAD(b_pts, pts, n * 32, d_pts);
    ENSURE(b_foldscratch, 1024 * kGptBytes, d_fs);
    ENSURE(b_rhat, 32, d_out);
    ENSURE(b_flags, 4, d_flags);
    CU(cudaMemsetAsync(d_flags, 0, 16, ctx->stream));
    launch_point_fold(d_pts, n, d_out, d_flags, d_fs, ctx->stream);
    ctx->launches += 2;
    CU(cudaGetLastError());
    int bad = 0;
    CU(cudaMemcpyAsync(&bad, d_flags, 4, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaMemcpyAsync(out, d_out, 32, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (bad) return set_err(err, POSLO_FORMAT_ERROR, 0, "invalid group element encoding");
    count_op(ctx, kOpCombine, n);  // agg_elements: one group_combine per element (poslo_c.cpp:170-174)
    return ok(err);
}

int poslo_gpu_point_valid(poslo_gpu_ctx* ctx, uint32_t n, const uint8_t* pts, uint8_t* okv,
                          poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (n && (!pts || !okv)) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    Guard g(ctx);
    uint8_t *d_pts, *d_ok;
    UPLOAD(b_pts, pts, (size_t)n * 32, d_pts);
    ENSURE(b_verdict, n, d_ok);
    launch_point_validate(d_pts, n, d_ok, ctx->stream);
    ctx->launches += n ? 1 : 0;
    CU(cudaGetLastError());
    if (n) CU(cudaMemcpyAsync(okv, d_ok, n, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return ok(err);
}

int poslo_gpu_seed_retrieve(poslo_gpu_ctx* ctx, uint8_t suite, const uint8_t* ds, uint32_t ds_len,
                            uint32_t ds_capacity, const uint32_t* epochs, uint32_t n,
                            uint8_t* x0_out, poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (n && (!epochs || !x0_out)) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (suite < 1 || suite > 3) return set_err(err, POSLO_FORMAT_ERROR, 0, "unknown suite id");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    Guard g(ctx);
    DsParam dsp;
    int rc = parse_ds(ds, ds_len, ds_capacity, dsp, err);
    if (rc) return rc;
    uint32_t* d_ep;
    uint4* d_x0;
    unsigned long long* d_err;
    UPLOAD(b_epochs, epochs, (size_t)n * 4, d_ep);
    ENSURE(b_x0, n, d_x0);
    ENSURE(b_err, 1, d_err);
    unsigned long long init = ~0ull;
    CU(cudaMemcpyAsync(d_err, &init, 8, cudaMemcpyHostToDevice, ctx->stream));
    launch_seed_derive(suite, dsp, d_ep, 0, n, d_x0, d_err, ctx->d_t0, ctx->stream);
    ctx->launches += n ? 1 : 0;
    CU(cudaGetLastError());
    unsigned long long key;
    CU(cudaMemcpyAsync(&key, d_err, 8, cudaMemcpyDeviceToHost, ctx->stream));
    if (n) CU(cudaMemcpyAsync(x0_out, d_x0, (size_t)n * 16, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    if (key != ~0ull) {
        uint32_t ep = epochs[key >> 1];
        return set_err(err, POSLO_SEED_NOT_DISCLOSED, ep, "seed for epoch %u not yet disclosed", ep);
    }
    return ok(err);
}

int poslo_gpu_entry_scalars(poslo_gpu_ctx* ctx, const poslo_batch* b, uint8_t* e_out, poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!b || !e_out) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    Guard g(ctx);
    // Force the generic path with per-entry output.
    Prepared P;
    poslo_batch nb = *b;
    int rc = run_hash(ctx, &nb, P, err);  // also validates + derives seeds
    if (rc) return rc;
    uint64_t n_entries = P.uniform ? (uint64_t)b->n_epochs * b->n2 : b->epoch_starts[b->n_epochs];
    uint32_t *d_ent, *d_partial;
    ENSURE(b_e, std::max<uint64_t>(n_entries, 1) * 8, d_ent);
    TileMap tm = P.tm;
    if (P.fast) {  // the fast path used its own tile size; re-tile for generic
        tm.tile_entries = 1024;
        tm.tiles_per_epoch = b->n2 ? (b->n2 + 1023) / 1024 : 0;
        tm.n_tiles = tm.n_epochs * tm.tiles_per_epoch;
    }
    ENSURE(b_scratch, (size_t)std::max<uint32_t>(tm.n_tiles, 1024) * 17, d_partial);
    launch_hash_generic(b->suite, P.lay, tm, static_cast<const uint4*>(ctx->b_x0.p), d_partial, d_ent,
                        static_cast<unsigned long long*>(ctx->b_err.p), ctx->d_t0, ctx->stream);
    ctx->launches += 1;
    CU(cudaGetLastError());
    rc = check_hash_errors(ctx, b, err);
    if (rc) return rc;
    if (n_entries) CU(cudaMemcpy(e_out, d_ent, n_entries * 32, cudaMemcpyDeviceToHost));
    return ok(err);
}

int poslo_gpu_scalar_sum(poslo_gpu_ctx* ctx, uint64_t n, const uint8_t* scalars, uint8_t out[32],
                         poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!out || (n && !scalars)) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    Guard g(ctx);
    for (uint64_t i = 0; i < n; i++)
        if (!scalar_canonical(scalars + 32 * i)) return set_err(err, POSLO_FORMAT_ERROR, 0, "non-canonical scalar");
    uint32_t *d_in, *d_sum, *d_scr;
    UPLOAD(b_e, scalars, n * 32, d_in);
    ENSURE(b_sum, 8, d_sum);
    ENSURE(b_scratch, 17 * 1024, d_scr);
    launch_sum_mod_l(d_in, 8, n, nullptr, d_sum, d_scr, ctx->stream);
    ctx->launches += 2;
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(out, d_sum, 32, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    return ok(err);
}

int poslo_gpu_group_check(poslo_gpu_ctx* ctx, uint32_t n, const uint8_t y[32], const uint8_t* e,
                          const uint8_t* s, const uint8_t* r, uint8_t* verdicts, poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (!y || (n && (!e || !s || !r || !verdicts))) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    Guard g(ctx);
    for (uint32_t i = 0; i < n; i++)
        if (!scalar_canonical(e + 32 * (size_t)i) || !scalar_canonical(s + 32 * (size_t)i))
            return set_err(err, POSLO_FORMAT_ERROR, 0, "non-canonical scalar");
    uint32_t *d_e, *d_s;
    uint8_t* d_r;
    UPLOAD(b_e, e, (size_t)n * 32, d_e);
    UPLOAD(b_s, s, (size_t)n * 32, d_s);
    UPLOAD(b_r, r, (size_t)n * 32, d_r);
    int rc = group_check_dev(ctx, y, n, d_e, d_s, d_r, verdicts, nullptr, err);
    if (rc) return rc;
    count_op(ctx, kOpDoubleExp, n);
    return ok(err);
}

int poslo_gpu_synth_log(poslo_gpu_ctx* ctx, uint64_t seed, uint64_t first, uint64_t n,
                        uint32_t entry_len, void* d_out, poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (n && !d_out) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    Guard g(ctx);
    launch_synth_fixed(seed, first, n, entry_len, static_cast<uint8_t*>(d_out), ctx->stream);
    ctx->launches += n ? 1 : 0;
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(ctx->stream));
    return ok(err);
}

int poslo_gpu_synth_varlog(poslo_gpu_ctx* ctx, uint64_t seed, uint64_t first, uint64_t n,
                           const uint64_t* d_offsets, void* d_out, poslo_error* err) {
    if (!ctx) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null context");
    if (n && (!d_out || !d_offsets)) return set_err(err, POSLO_INVALID_ARGUMENT, 0, "null argument");
    if (!ctx->members.empty()) ctx = ctx->members[0];
    Guard g(ctx);
    launch_synth_var(seed, first, n, d_offsets, static_cast<uint8_t*>(d_out), ctx->stream);
    ctx->launches += n ? 1 : 0;
    CU(cudaGetLastError());
    CU(cudaStreamSynchronize(ctx->stream));
    return ok(err);
}

}  // extern "C"
