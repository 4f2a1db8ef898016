// Multi-device contexts (poslo_gpu_create_multi, include/poslo_gpu.h): the
// batch verifier over several GPUs from one process (SURVEY.md §8b "select
// GPU count", §8e).
//
// The queried epochs are cut into contiguous ranges balanced by hashing work
// (entries and entry bytes), one range per member context. Every member runs
// the single-device call on its range on its own device, stream and host
// thread; the partial results are combined on member 0 exactly as the
// reference combines them on one machine:
//   agg_ekeys   e~ concatenated in epoch order; e-hat = the members' partial
//               sums folded mod l in member order (batch_verify.cpp:83-85).
//   paver       the same e-hat, R-hat = group_combine fold of the members'
//               partial folds (:75-81), then ONE commit_check (:86).
//   epoch_verify / distill_coarse
//               per-epoch verdicts concatenated; an umbrella piece that a
//               shard cut splits is folded back together (sum mod l of s and
//               e, group law on R-hat: distiller.cpp:45-53, 82-88).
// Sums mod l and the group law are associative and commutative and every
// output is a canonical encoding, so results are byte-identical to one
// device. Errors: the lowest failing member wins — members hold ascending
// epoch ranges, so that is the reference's lowest-epoch error (workers = 1).
#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <thread>
#include <vector>

#include "capi_ctx.h"

namespace poslo_gpu_detail {

namespace {

int fail(poslo_error* err, int code, uint32_t epoch, const char* fmt, ...) {
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

int succeed(poslo_error* err) {
    if (err) {
        err->code = POSLO_OK;
        err->epoch = 0;
        err->message[0] = 0;
    }
    return POSLO_OK;
}

uint64_t entry_of(const poslo_batch* b, uint32_t k) {
    return b->epoch_starts ? b->epoch_starts[k] : (uint64_t)k * b->n2;
}

uint64_t byte_of(const poslo_batch* b, uint64_t t) { return b->offsets ? b->offsets[t] : t * (uint64_t)b->entry_len; }

// Hashing work of the first k queried epochs, in SHA-256 compressions: about
// three per entry plus one per 64 bytes of entry (suite 1; proportional for
// the AES suites).
double work_upto(const poslo_batch* b, uint32_t k) {
    const uint64_t t = entry_of(b, k);
    return 3.0 * (double)t + (double)(byte_of(b, t) - byte_of(b, 0)) / 64.0;
}

// cut[g] .. cut[g + 1]: the epoch range of member g (contiguous, ascending).
std::vector<uint32_t> shard_cuts(const poslo_batch* b, int G) {
    const uint32_t n = b->n_epochs;
    std::vector<uint32_t> cut(G + 1, 0);
    const double total = work_upto(b, n);
    for (int g = 1; g < G; g++) {
        const double target = total * g / G;
        uint32_t lo = cut[g - 1], hi = n;
        while (lo < hi) {  // smallest k with work_upto(k) >= target
            const uint32_t mid = lo + (hi - lo) / 2;
            if (work_upto(b, mid) >= target)
                hi = mid;
            else
                lo = mid + 1;
        }
        cut[g] = std::max(cut[g - 1], lo);
    }
    cut[G] = n;
    return cut;
}

// poslo_batch.fill of a shard: entries are numbered from the shard's first
struct FillShift {
    int (*fill)(void*, uint64_t, uint64_t, uint8_t*);
    void* user;
    uint64_t base;
};

int shifted_fill(void* user, uint64_t first, uint64_t count, uint8_t* dst) {
    const FillShift* f = static_cast<const FillShift*>(user);
    return f->fill(f->user, f->base + first, count, dst);
}

struct Shard {
    uint32_t k0 = 0, k1 = 0;  // batch positions
    poslo_batch b{};
    std::vector<uint64_t> starts;
    FillShift fs{};
};

// Member g's view of the batch: epochs [k0, k1) with their entries. Fixed-length
// payloads are re-based; variable-length ones keep the caller's absolute
// offsets (the single-device call copies only the shard's byte span).
void make_shard(const poslo_batch* b, uint32_t k0, uint32_t k1, Shard& sh) {
    sh.k0 = k0;
    sh.k1 = k1;
    sh.b = *b;
    const uint64_t e0 = entry_of(b, k0), e1 = entry_of(b, k1);
    sh.b.epochs = b->epochs ? b->epochs + k0 : nullptr;
    sh.b.n_epochs = k1 - k0;
    if (b->epoch_starts) {
        sh.starts.resize(k1 - k0 + 1);
        for (uint32_t k = k0; k <= k1; k++) sh.starts[k - k0] = b->epoch_starts[k] - e0;
        sh.b.epoch_starts = sh.starts.data();
    }
    sh.b.n_entries = e1 - e0;
    if (b->ds_offsets) sh.b.ds_offsets = b->ds_offsets + k0;
    if (b->offsets) {
        sh.b.offsets = b->offsets + e0;
    } else {
        if (b->payload) sh.b.payload = b->payload + e0 * b->entry_len;
        sh.b.payload_bytes = (e1 - e0) * b->entry_len;
    }
    if (b->fill) {
        sh.fs = FillShift{b->fill, b->fill_user, e0};
        sh.b.fill = shifted_fill;
        sh.b.fill_user = &sh.fs;
    }
}

// Runs f(g) for every member g concurrently (member 0 on the calling thread).
template <class F>
void run_members(int G, F&& f) {
    std::vector<std::thread> th;
    th.reserve(G > 0 ? G - 1 : 0);
    for (int g = 1; g < G; g++) th.emplace_back([&f, g] { f(g); });
    f(0);
    for (auto& t : th) t.join();
}

// The member that runs a batch whole: the owner of device-resident memory,
// else member 0 (raw images without offsets, empty batches, ...). Returns
// nullptr when the batch must be sharded.
poslo_gpu_ctx* whole_batch_member(poslo_gpu_ctx* ctx, const poslo_batch* b, int* rc, poslo_error* err) {
    *rc = POSLO_OK;
    if (b->device_resident) {
        cudaPointerAttributes a{};
        const void* p = b->payload ? (const void*)b->payload : (const void*)b->offsets;
        if (p && cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type != cudaMemoryTypeUnregistered) {
            for (poslo_gpu_ctx* m : ctx->members)
                if (m->device == a.device) return m;
        }
        cudaGetLastError();
        *rc = fail(err, POSLO_INVALID_ARGUMENT, 0, "device_resident batch on no member's device");
        return nullptr;
    }
    if ((b->record_header == 4 && !b->offsets) || b->n_epochs < 2) return ctx->members[0];
    return nullptr;
}

bool ascending(const poslo_batch* b) {
    for (uint32_t k = 1; k < b->n_epochs; k++)
        if (b->epochs[k] <= b->epochs[k - 1]) return false;
    return true;
}

int first_error(const std::vector<int>& rcs, const std::vector<poslo_error>& errs, poslo_error* err) {
    for (size_t g = 0; g < rcs.size(); g++)
        if (rcs[g] != POSLO_OK) {
            if (err) *err = errs[g];
            return rcs[g];
        }
    return POSLO_OK;
}

// Member 0 folds without counting: the members already counted the group
// operations of their shards, which together are the single-device count.
struct Uncounted {
    poslo_gpu_ctx* m;
    explicit Uncounted(poslo_gpu_ctx* c) : m(c) { m->count_ops = false; }
    ~Uncounted() { m->count_ops = true; }
};

// Scalar::from_be_bytes's range check (group.cpp:46-49) on a 32-byte LE scalar.
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

int shard_count(poslo_gpu_ctx* ctx, const poslo_batch* b) {
    return (int)std::min<size_t>(ctx->members.size(), b->n_epochs);
}

}  // namespace

int multi_agg_ekeys(poslo_gpu_ctx* ctx, const poslo_batch* b, uint8_t* e_tilde_out, uint8_t* e_hat_out,
                    poslo_error* err) {
    if (!b) return fail(err, POSLO_INVALID_ARGUMENT, 0, "null batch");
    std::lock_guard<std::mutex> lk(ctx->mtx);
    int rc;
    if (poslo_gpu_ctx* m = whole_batch_member(ctx, b, &rc, err)) return poslo_gpu_agg_ekeys(m, b, e_tilde_out, e_hat_out, err);
    if (rc) return rc;
    if (b->n_epochs && !b->epochs) return fail(err, POSLO_INVALID_ARGUMENT, 0, "null epochs");
    if (!ascending(b)) return fail(err, POSLO_INVALID_ARGUMENT, 0, "epochs must be strictly ascending");
    const int G = shard_count(ctx, b);
    const std::vector<uint32_t> cut = shard_cuts(b, G);
    std::vector<Shard> sh(G);
    for (int g = 0; g < G; g++) make_shard(b, cut[g], cut[g + 1], sh[g]);
    std::vector<uint8_t> parts(32 * (size_t)G);
    std::vector<int> rcs(G, POSLO_OK);
    std::vector<poslo_error> errs(G);
    run_members(G, [&](int g) {
        rcs[g] = poslo_gpu_agg_ekeys(ctx->members[g], &sh[g].b, e_tilde_out ? e_tilde_out + 32 * (size_t)sh[g].k0 : nullptr,
                                     e_hat_out ? &parts[32 * (size_t)g] : nullptr, &errs[g]);
    });
    rc = first_error(rcs, errs, err);
    if (rc) return rc;
    if (e_hat_out) {  // rank-ordered fold mod l on member 0
        Uncounted u(ctx->members[0]);
        rc = poslo_gpu_scalar_sum(ctx->members[0], G, parts.data(), e_hat_out, err);
        if (rc) return rc;
    }
    return succeed(err);
}

int multi_paver(poslo_gpu_ctx* ctx, const poslo_batch* b, const uint8_t y[32], const uint8_t s_hat[32],
                const uint8_t* r_hat_agg, const uint8_t* r_hats, uint8_t* verdict, poslo_error* err) {
    std::lock_guard<std::mutex> lk(ctx->mtx);
    int rc;
    if (poslo_gpu_ctx* m = whole_batch_member(ctx, b, &rc, err))
        return poslo_gpu_paver(m, b, y, s_hat, r_hat_agg, r_hats, verdict, err);
    if (rc) return rc;
    // the single-device validation order (batch_verify.cpp:68-82, then s-hat, then Y)
    if (b->epoch_starts)
        for (uint32_t k = 0; k < b->n_epochs; k++)
            if (b->epoch_starts[k + 1] - b->epoch_starts[k] != b->n2)
                return fail(err, POSLO_STATE_ERROR, b->epochs[k], "every batch must hold exactly n2 entries");
    if (!r_hat_agg && !r_hats && b->n_epochs)
        return fail(err, POSLO_STATE_ERROR, b->epochs[0], "commitment for epoch %u no longer in public key",
                    b->epochs[0]);
    if (!b->epochs) return fail(err, POSLO_INVALID_ARGUMENT, 0, "null epochs");
    if (!ascending(b)) return fail(err, POSLO_INVALID_ARGUMENT, 0, "epochs must be strictly ascending");
    if (!scalar_canonical(s_hat)) return fail(err, POSLO_FORMAT_ERROR, 0, "non-canonical scalar");
    poslo_gpu_ctx* m0 = ctx->members[0];
    uint8_t y_ok = 0;  // GroupElement::from_bytes on Y, before any hashing (as one device)
    rc = poslo_gpu_point_valid(m0, 1, y, &y_ok, err);
    if (rc) return rc;
    if (!y_ok) return fail(err, POSLO_FORMAT_ERROR, 0, "invalid group element encoding");
    const int G = shard_count(ctx, b);
    const std::vector<uint32_t> cut = shard_cuts(b, G);
    std::vector<Shard> sh(G);
    for (int g = 0; g < G; g++) make_shard(b, cut[g], cut[g + 1], sh[g]);
    std::vector<uint8_t> eparts(32 * (size_t)G), rparts(32 * (size_t)G);
    std::vector<int> rcs(G, POSLO_OK), rcs_r(G, POSLO_OK);
    std::vector<poslo_error> errs(G), errs_r(G);
    run_members(G, [&](int g) {
        poslo_gpu_ctx* m = ctx->members[g];
        rcs[g] = poslo_gpu_agg_ekeys(m, &sh[g].b, nullptr, &eparts[32 * (size_t)g], &errs[g]);
        if (!r_hat_agg && rcs[g] == POSLO_OK)  // this shard's part of the R-hat fold (one combine per epoch)
            rcs_r[g] = poslo_gpu_group_fold(m, sh[g].k1 - sh[g].k0, r_hats + 32 * (size_t)sh[g].k0,
                                            &rparts[32 * (size_t)g], &errs_r[g]);
    });
    rc = first_error(rcs, errs, err);  // hashing errors first, as one device reports them
    if (rc) return rc;
    rc = first_error(rcs_r, errs_r, err);
    if (rc) return rc;
    uint8_t r_hat[32];
    if (r_hat_agg) {
        std::memcpy(r_hat, r_hat_agg, 32);
    } else {
        Uncounted u(m0);
        rc = poslo_gpu_group_fold(m0, G, rparts.data(), r_hat, err);
        if (rc) return rc;
    }
    // e-hat folded in member order and the single check on member 0 (counted once)
    return poslo_gpu_combine_check(m0, G, eparts.data(), 0, y, s_hat, r_hat, verdict, err);
}

int multi_epoch_verify(poslo_gpu_ctx* ctx, const poslo_batch* b, const uint8_t y[32], const uint8_t* s_hats,
                       const uint8_t* r_hats, uint8_t* verdicts, uint8_t* e_tilde_out, poslo_error* err) {
    std::lock_guard<std::mutex> lk(ctx->mtx);
    int rc;
    if (poslo_gpu_ctx* m = whole_batch_member(ctx, b, &rc, err))
        return poslo_gpu_epoch_verify(m, b, y, s_hats, r_hats, verdicts, e_tilde_out, err);
    if (rc) return rc;
    if (!b->epochs) return fail(err, POSLO_INVALID_ARGUMENT, 0, "null epochs");
    if (!ascending(b)) return fail(err, POSLO_INVALID_ARGUMENT, 0, "epochs must be strictly ascending");
    const int G = shard_count(ctx, b);
    const std::vector<uint32_t> cut = shard_cuts(b, G);
    std::vector<Shard> sh(G);
    for (int g = 0; g < G; g++) make_shard(b, cut[g], cut[g + 1], sh[g]);
    std::vector<int> rcs(G, POSLO_OK);
    std::vector<poslo_error> errs(G);
    run_members(G, [&](int g) {
        const size_t k0 = sh[g].k0;
        rcs[g] = poslo_gpu_epoch_verify(ctx->members[g], &sh[g].b, y, s_hats + 32 * k0, r_hats + 32 * k0,
                                        verdicts + k0, e_tilde_out ? e_tilde_out + 32 * k0 : nullptr, &errs[g]);
    });
    rc = first_error(rcs, errs, err);
    if (rc) return rc;
    return succeed(err);
}

int multi_distill_coarse(poslo_gpu_ctx* ctx, const poslo_batch* b, const uint8_t y[32], const uint8_t* s_hats,
                         const uint8_t* r_hats, const uint32_t* seg, uint32_t n_seg, uint8_t* verdicts,
                         uint8_t* seg_s, uint8_t* seg_r, uint8_t* seg_e, poslo_error* err) {
    if (!b || !y || (b->n_epochs && (!s_hats || !r_hats || !verdicts)) || (n_seg && !seg))
        return fail(err, POSLO_INVALID_ARGUMENT, 0, "bad argument");
    std::lock_guard<std::mutex> lk(ctx->mtx);
    int rc;
    if (poslo_gpu_ctx* m = whole_batch_member(ctx, b, &rc, err))
        return poslo_gpu_distill_coarse_ex(m, b, y, s_hats, r_hats, seg, n_seg, verdicts, seg_s, seg_r, seg_e, err);
    if (rc) return rc;
    if (b->epoch_starts)  // aver (poslo_c.cpp:195-197)
        for (uint32_t k = 0; k < b->n_epochs; k++)
            if (b->epoch_starts[k + 1] - b->epoch_starts[k] != b->n2)
                return fail(err, POSLO_STATE_ERROR, b->epochs[k], "every batch must hold exactly n2 entries");
    if (!b->epochs) return fail(err, POSLO_INVALID_ARGUMENT, 0, "null epochs");
    if (!ascending(b)) return fail(err, POSLO_INVALID_ARGUMENT, 0, "epochs must be strictly ascending");
    const uint32_t n = b->n_epochs;
    for (uint32_t g = 0; g < n_seg; g++)
        if (seg[g] > seg[g + 1] || seg[g + 1] > n)
            return fail(err, POSLO_INVALID_ARGUMENT, 0, "segments must be non-decreasing within [0, n]");
    const int G = shard_count(ctx, b);
    const std::vector<uint32_t> cut = shard_cuts(b, G);
    std::vector<Shard> sh(G);
    // member g's segments: the global segments cut at its range ends; piece i of
    // member g belongs to global segment owner[g][i] (-1: outside every segment)
    std::vector<std::vector<uint32_t>> lseg(G);
    std::vector<std::vector<int64_t>> owner(G);
    for (int g = 0; g < G; g++) {
        make_shard(b, cut[g], cut[g + 1], sh[g]);
        const uint32_t k0 = cut[g], k1 = cut[g + 1];
        std::vector<uint32_t> bnd{k0};
        for (uint32_t j = 0; j <= n_seg && n_seg; j++)
            if (seg[j] > k0 && seg[j] < k1 && seg[j] != bnd.back()) bnd.push_back(seg[j]);
        bnd.push_back(k1);
        for (size_t i = 0; i + 1 < bnd.size(); i++) {
            const uint32_t a = bnd[i];
            int64_t j = -1;
            if (n_seg && a >= seg[0] && a < seg[n_seg])
                j = (int64_t)(std::upper_bound(seg, seg + n_seg + 1, a) - seg) - 1;
            owner[g].push_back(j);
        }
        for (uint32_t& x : bnd) x -= k0;
        lseg[g] = std::move(bnd);
    }
    std::vector<std::vector<uint8_t>> ls(G), lr(G), le(G);
    std::vector<int> rcs(G, POSLO_OK);
    std::vector<poslo_error> errs(G);
    run_members(G, [&](int g) {
        const size_t k0 = sh[g].k0, np = lseg[g].size() - 1;
        ls[g].resize(32 * np);
        lr[g].resize(32 * np);
        le[g].resize(32 * np);
        rcs[g] = poslo_gpu_distill_coarse_ex(ctx->members[g], &sh[g].b, y, s_hats + 32 * k0, r_hats + 32 * k0,
                                             lseg[g].data(), (uint32_t)np, verdicts + k0, seg_s ? ls[g].data() : nullptr,
                                             seg_r ? lr[g].data() : nullptr, seg_e ? le[g].data() : nullptr, &errs[g]);
    });
    rc = first_error(rcs, errs, err);
    if (rc) return rc;
    if (!n_seg || (!seg_s && !seg_r && !seg_e)) return succeed(err);
    // the pieces of every global segment, in member order -> one segmented fold on member 0
    std::vector<uint8_t> is, ir, ie;
    std::vector<uint32_t> bounds{0};
    for (uint32_t j = 0; j < n_seg; j++) {
        for (int g = 0; g < G; g++)
            for (size_t i = 0; i < owner[g].size(); i++)
                if (owner[g][i] == (int64_t)j) {
                    is.insert(is.end(), &ls[g][32 * i], &ls[g][32 * i] + 32);
                    ir.insert(ir.end(), &lr[g][32 * i], &lr[g][32 * i] + 32);
                    ie.insert(ie.end(), &le[g][32 * i], &le[g][32 * i] + 32);
                }
        bounds.push_back((uint32_t)(is.size() / 32));
    }
    poslo_gpu_ctx* m0 = ctx->members[0];
    Uncounted u(m0);
    const uint32_t n_items = bounds.back();
    if (!n_items) {  // every segment empty: sum 0, identity fold
        for (uint8_t* o : {seg_s, seg_r, seg_e})
            if (o) std::memset(o, 0, 32 * (size_t)n_seg);
        return succeed(err);
    }
    if (seg_s || seg_r) {
        rc = poslo_gpu_segfold(m0, n_items, seg_s ? is.data() : nullptr, seg_r ? ir.data() : nullptr, nullptr,
                               bounds.data(), n_seg, seg_s, seg_r, err);
        if (rc) return rc;
    }
    if (seg_e) {
        rc = poslo_gpu_segfold(m0, n_items, ie.data(), nullptr, nullptr, bounds.data(), n_seg, seg_e, nullptr, err);
        if (rc) return rc;
    }
    return succeed(err);
}

}  // namespace poslo_gpu_detail
