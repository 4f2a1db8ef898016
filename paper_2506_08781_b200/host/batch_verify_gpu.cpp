// B200 drop-in for the reference's batch verifier: defines poslo::agg_ekeys
// and poslo::paver with the exact signatures and error behaviour of
// /root/reference/proj/include/poslo/batch_verify.hpp:11-30 (implementation
// it replaces: proj/src/batch_verify.cpp:11-87), on top of the C-ABI in
// include/poslo_gpu.h. Compiled against the reference's own headers in place
// of src/batch_verify.cpp; see INTEGRATION.md.
//
// `workers` keeps its reference meaning as the degree of parallelism: the
// call runs on min(workers, #GPUs) devices (batch_verify.cpp:51-59 spawns
// min(workers, #epochs) threads), sharded by contiguous epoch ranges inside
// one C-ABI call (poslo_gpu_create_multi); workers == 0 -> StateError.
// POSLO_GPU_DEVICES=0,1,... lists the devices (a device may repeat: members
// then share it), default every visible device; POSLO_GPU_DEVICE=k pins one.
//
// The std::map<uint32_t, std::vector<Bytes>> is not copied up front: the C-ABI
// pulls the entries chunk by chunk through poslo_batch.fill, and each chunk is
// gathered into pinned staging by all host cores (a persistent worker pool)
// while the previous chunks are copied to the device and hashed.
#if defined(__SSE2__)
#include <immintrin.h>
#endif

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <condition_variable>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <thread>

#include "poslo/batch_verify.hpp"
#include "poslo_gpu.h"

namespace poslo {

namespace {

// Persistent host workers for the gather/sizing loops: parallel_for(n, f)
// runs f(0..n-1) on every core (the caller included); one loop at a time.
class Pool {
public:
    Pool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const unsigned n = std::min(hw, 64u) - 1;
        for (unsigned i = 0; i < n; i++) th_.emplace_back([this] { work(); });
    }
    ~Pool() {
        {
            std::lock_guard<std::mutex> lk(m_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : th_) t.join();
    }
    void parallel_for(int64_t n, const std::function<void(int64_t)>& f) {
        if (n <= 0) return;
        std::lock_guard<std::mutex> one(call_);
        if (th_.empty() || n == 1) {
            for (int64_t i = 0; i < n; i++) f(i);
            return;
        }
        {
            std::lock_guard<std::mutex> lk(m_);
            job_ = &f;
            n_ = n;
            next_.store(0);
            busy_ = (int)th_.size();
            gen_++;
        }
        cv_.notify_all();
        run();
        std::unique_lock<std::mutex> lk(m_);
        done_.wait(lk, [this] { return busy_ == 0; });
        job_ = nullptr;
    }

private:
    void run() {
        for (int64_t i = next_.fetch_add(1); i < n_; i = next_.fetch_add(1)) (*job_)(i);
    }
    void work() {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(m_);
                cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
                if (stop_) return;
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
    const std::function<void(int64_t)>* job_ = nullptr;
    int64_t n_ = 0;
    std::atomic<int64_t> next_{0};
    int busy_ = 0;
    uint64_t gen_ = 0;
    bool stop_ = false;
};

Pool& pool() {
    static Pool p;
    return p;
}

// f over [0, n) in blocks of `grain` on the pool
void parallel_blocks(int64_t n, int64_t grain, const std::function<void(int64_t, int64_t)>& f) {
    const int64_t nb = (n + grain - 1) / grain;
    pool().parallel_for(nb, [&](int64_t blk) { f(blk * grain, std::min(n, (blk + 1) * grain)); });
}

std::vector<int> parse_devices() {
    std::vector<int> out;
    if (const char* e = std::getenv("POSLO_GPU_DEVICES")) {
        const std::string s(e);
        size_t p = 0;
        while (p < s.size()) {
            size_t q = s.find(',', p);
            if (q == std::string::npos) q = s.size();
            if (q > p) out.push_back(std::atoi(s.substr(p, q - p).c_str()));
            p = q + 1;
        }
    } else if (const char* e1 = std::getenv("POSLO_GPU_DEVICE")) {
        out.push_back(std::atoi(e1));
    } else {
        const int n = poslo_gpu_device_count();
        for (int d = 0; d < n; d++) out.push_back(d);
    }
    if (out.empty()) out.push_back(0);
    return out;
}

const std::vector<int>& device_list() {
    static const std::vector<int> list = parse_devices();
    return list;
}

// Device contexts of one host thread, one per GPU count: the C-ABI serialises
// calls per context, so thread-local contexts keep concurrent callers
// independent ("externally a pure, thread-safe function").
struct DeviceContexts {
    std::map<size_t, poslo_gpu_ctx*> by_count;
    ~DeviceContexts() {
        for (auto& [g, c] : by_count) poslo_gpu_destroy(c);
    }
    poslo_gpu_ctx* get(size_t g) {
        auto it = by_count.find(g);
        if (it != by_count.end()) return it->second;
        poslo_gpu_ctx* c = nullptr;
        poslo_error err{};
        const std::vector<int>& L = device_list();
        const int rc = g > 1 ? poslo_gpu_create_multi(L.data(), static_cast<int>(g), &c, &err)
                             : poslo_gpu_create(L[0], &c, &err);
        if (rc != POSLO_OK) throw std::runtime_error(std::string("poslo_gpu: ") + err.message);
        by_count[g] = c;
        return c;
    }
};

poslo_gpu_ctx* device(unsigned workers) {
    thread_local DeviceContexts dc;
    const size_t g = std::min<size_t>(std::max(1u, workers), device_list().size());
    return dc.get(g);
}

[[noreturn]] void rethrow(const poslo_error& e) {
    switch (e.code) {
        case POSLO_FORMAT_ERROR: throw FormatError(e.message);
        case POSLO_STATE_ERROR: throw StateError(e.message);
        case POSLO_SEED_NOT_DISCLOSED: throw SeedNotDisclosed(e.epoch);
        default: throw std::runtime_error(std::string("poslo_gpu: ") + e.message);
    }
}

// The batches as the C-ABI sees them: epoch list, entry ranges, byte
// offsets for variable-length entries, and a producer that gathers any entry
// range into a packed buffer.
struct Packed {
    std::vector<const std::vector<Bytes>*> msgs;  // per queried epoch, map order
    std::vector<uint32_t> epochs;
    std::vector<uint64_t> starts;   // n_epochs + 1 entry indices
    std::vector<uint64_t> offsets;  // n_entries + 1 byte offsets (variable lengths only)
    bool fixed = true, uniform = true;
    uint32_t len0 = 0;
    std::atomic<bool> mismatch{false};  // gather met an entry of another length (fixed layout assumed)
    Bytes ds;
    poslo_batch b{};
    double fill_ms = 0;  // time inside gather() (the host side of the pipelined copy)
};

// Host-side breakdown of the last paver / agg_ekeys call of this process
// (poslo_dropin_last_stats): pack = sizing the map, fill = gathering it into
// the pinned staging ring (overlapped with the copies and hashing), call =
// the whole drop-in call.
std::mutex g_stats_m;
double g_stats[4] = {0, 0, 0, 0};  // pack_ms, fill_ms, call_ms, entries
using sclock = std::chrono::steady_clock;
double ms_between(sclock::time_point a, sclock::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
}
void record_stats(double pack_ms, double fill_ms, double call_ms, double entries) {
    std::lock_guard<std::mutex> lk(g_stats_m);
    g_stats[0] = pack_ms;
    g_stats[1] = fill_ms;
    g_stats[2] = call_ms;
    g_stats[3] = entries;
}

uint64_t byte_at(const Packed& p, uint64_t t) { return p.fixed ? t * p.len0 : p.offsets[t]; }

// Fixed-length copy of entries [t0, t1) of one epoch; L a compile-time
// constant for the common sizes (inlined moves), the data of later entries
// prefetched (their heap blocks are scattered); false on a length mismatch.
// The staging writes are non-temporal: the chunk goes to the device by DMA,
// never back through this core's caches (no read-for-ownership of dst).
template <uint32_t L>
bool copy_fixed(const std::vector<Bytes>& ms, uint64_t s0, uint64_t t0, uint64_t t1, uint8_t* d, uint32_t len) {
    const uint32_t n = L ? L : len;
    constexpr uint64_t kAhead = 8;
    for (uint64_t t = t0; t < t1; t++, d += n) {
        if (t + kAhead < t1) __builtin_prefetch(ms[t + kAhead - s0].data());
        const Bytes& m = ms[t - s0];
        if (m.size() != n) return false;
#if defined(__SSE2__)
        if constexpr (L != 0 && L % 16 == 0) {
            if ((reinterpret_cast<uintptr_t>(d) & 15) == 0) {
                const __m128i* src = reinterpret_cast<const __m128i*>(m.data());
                __m128i* dd = reinterpret_cast<__m128i*>(d);
                for (uint32_t q = 0; q < L / 16; q++) _mm_stream_si128(dd + q, _mm_loadu_si128(src + q));
                continue;
            }
        }
#endif
        std::memcpy(d, m.data(), L ? L : len);
    }
    return true;
}

// poslo_batch.fill: entries [first, first + count) back to back into dst,
// epochs spread over the host cores.
int gather(void* user, uint64_t first, uint64_t count, uint8_t* dst) {
    Packed& p = *static_cast<Packed*>(user);
    const auto t_fill = sclock::now();
    const uint64_t last = first + count;
    const int64_t k0 = std::upper_bound(p.starts.begin(), p.starts.end(), first) - p.starts.begin() - 1;
    const int64_t k1 = std::lower_bound(p.starts.begin(), p.starts.end(), last) - p.starts.begin();
    const uint64_t base = byte_at(p, first);
    const int64_t kb = std::max<int64_t>(k0, 0);
    parallel_blocks(k1 - kb, 16, [&](int64_t a, int64_t z) {
        for (int64_t k = kb + a; k < kb + z; k++) {
            const std::vector<Bytes>& ms = *p.msgs[k];
            const uint64_t s0 = p.starts[k];
            const uint64_t t0 = std::max(s0, first), t1 = std::min(p.starts[k + 1], last);
            if (p.fixed) {
                uint8_t* d = dst + (t0 * p.len0 - base);
                const bool ok = p.len0 == 32   ? copy_fixed<32>(ms, s0, t0, t1, d, 32)
                                : p.len0 == 64 ? copy_fixed<64>(ms, s0, t0, t1, d, 64)
                                               : copy_fixed<0>(ms, s0, t0, t1, d, p.len0);
                if (!ok) p.mismatch.store(true, std::memory_order_relaxed);
#if defined(__SSE2__)
                _mm_sfence();  // the streaming stores are visible before the DMA reads the slot
#endif
            } else {
                for (uint64_t t = t0; t < t1; t++) {
                    const Bytes& m = ms[t - s0];
                    if (!m.empty()) std::memcpy(dst + (p.offsets[t] - base), m.data(), m.size());
                }
            }
        }
    });
    p.fill_ms += ms_between(t_fill, sclock::now());
    return p.mismatch.load() ? 1 : 0;  // a mismatch aborts the call; the caller re-packs with offsets
}

// One in-order walk of the map into p.epochs / p.msgs / p.starts (the batch
// sizes, turned into entry offsets by the caller). The map's nodes are
// scattered between the entries' heap blocks, so a serial walk is one cache
// and TLB miss per epoch (~25 ms at 2^18 epochs); the key range is cut into
// pieces at lower_bound() of evenly spaced keys and the pieces are walked on
// every host core, each writing its own slice (its offset in the map is its
// count of earlier nodes, from a first parallel counting pass over the same
// pieces, which also warms the nodes for the second).
void walk_map(const std::map<uint32_t, std::vector<Bytes>>& batches, Packed& p) {
    const size_t ne = batches.size();
    if (ne == 0) return;
    const int64_t pieces = ne >= 4096 ? 256 : 1;
    const uint64_t k_lo = batches.begin()->first, k_hi = batches.rbegin()->first;
    std::vector<std::map<uint32_t, std::vector<Bytes>>::const_iterator> cut(pieces + 1);
    cut[0] = batches.begin();
    cut[pieces] = batches.end();
    for (int64_t q = 1; q < pieces; q++)
        cut[q] = batches.lower_bound((uint32_t)(k_lo + (k_hi - k_lo + 1) * (uint64_t)q / (uint64_t)pieces));
    std::vector<size_t> first(pieces + 1, 0);
    pool().parallel_for(pieces, [&](int64_t q) {
        size_t c = 0;
        for (auto it = cut[q]; it != cut[q + 1]; ++it) c++;
        first[q + 1] = c;
    });
    for (int64_t q = 0; q < pieces; q++) first[q + 1] += first[q];
    pool().parallel_for(pieces, [&](int64_t q) {
        size_t k = first[q];
        for (auto it = cut[q]; it != cut[q + 1]; ++it, ++k) {
            p.epochs[k] = it->first;
            p.msgs[k] = &it->second;
            p.starts[k] = it->second.size();
        }
    });
}

// fixed_guess: assume one entry length (checked entry by entry while the
// chunks are gathered, so the common case reads each entry header once);
// false: the sizing pass computes byte offsets for mixed lengths.
void pack(const SuiteConfig& suite, const std::map<uint32_t, std::vector<Bytes>>& batches,
          const SeedStack& ds, Packed& p, bool fixed_guess) {
    const size_t ne = batches.size();
    p.msgs.resize(ne);
    p.epochs.resize(ne);
    p.starts.resize(ne + 1);
    walk_map(batches, p);
    uint64_t t = 0;
    for (size_t k = 0; k < ne; k++) {  // entry index of each epoch (the walk stored sizes in starts)
        const uint64_t sz = p.starts[k];
        p.starts[k] = t;
        t += sz;
        if (sz != suite.n2) p.uniform = false;
    }
    p.starts[ne] = t;
    const uint64_t n = t;
    // sizing pass over the entry headers, in parallel: one length, or offsets
    for (size_t k = 0; k < ne && p.len0 == 0 && n; k++)
        if (!p.msgs[k]->empty()) p.len0 = static_cast<uint32_t>((*p.msgs[k])[0].size());
    p.fixed = fixed_guess;
    uint64_t total = n * p.len0;
    if (!p.fixed) {
        std::vector<uint64_t> ep_bytes(ne + 1, 0);
        parallel_blocks((int64_t)ne, 256, [&](int64_t a, int64_t z) {
            for (int64_t k = a; k < z; k++) {
                uint64_t s = 0;
                for (const Bytes& m : *p.msgs[k]) s += m.size();
                ep_bytes[k + 1] = s;
            }
        });
        for (size_t k = 0; k < ne; k++) ep_bytes[k + 1] += ep_bytes[k];
        p.offsets.resize(n + 1);
        parallel_blocks((int64_t)ne, 256, [&](int64_t a, int64_t z) {
            for (int64_t k = a; k < z; k++) {
                uint64_t o = ep_bytes[k], tt = p.starts[k];
                for (const Bytes& m : *p.msgs[k]) {
                    p.offsets[tt++] = o;
                    o += m.size();
                }
            }
        });
        p.offsets[n] = ep_bytes[ne];
        total = ep_bytes[ne];
    }
    ds.serialize(p.ds);
    poslo_batch& b = p.b;
    b.suite = static_cast<uint8_t>(suite.suite);
    b.n2 = suite.n2;
    b.payload = nullptr;  // produced on demand by gather()
    b.payload_bytes = total;
    b.offsets = p.fixed ? nullptr : p.offsets.data();
    b.entry_len = p.fixed ? p.len0 : 0;
    b.n_entries = n;
    b.epochs = p.epochs.data();
    b.epoch_starts = p.uniform ? nullptr : p.starts.data();
    b.n_epochs = static_cast<uint32_t>(p.epochs.size());
    b.ds = p.ds.data();
    b.ds_len = static_cast<uint32_t>(p.ds.size());
    b.ds_capacity = ds.capacity();
    b.device_resident = 0;
    b.fill = n ? gather : nullptr;
    b.fill_user = &p;
}

}  // namespace

std::vector<EpochKeyAggregate> agg_ekeys(const SuiteConfig& suite,
                                         const std::map<uint32_t, std::vector<Bytes>>& batches,
                                         const SeedStack& ds, unsigned workers) {
    if (workers == 0) throw StateError("worker count must be at least 1");
    Packed p;
    pack(suite, batches, ds, p, true);
    std::vector<uint8_t> et(32 * std::max<size_t>(p.epochs.size(), 1));
    poslo_error err{};
    int rc = poslo_gpu_agg_ekeys(device(workers), &p.b, et.data(), nullptr, &err);
    if (rc != POSLO_OK && p.mismatch.load()) {  // mixed entry lengths: again with byte offsets
        Packed q;
        pack(suite, batches, ds, q, false);
        rc = poslo_gpu_agg_ekeys(device(workers), &q.b, et.data(), nullptr, &err);
    }
    if (rc != POSLO_OK) rethrow(err);
    std::vector<EpochKeyAggregate> out(p.epochs.size());
    for (size_t k = 0; k < p.epochs.size(); k++)
        out[k] = EpochKeyAggregate{p.epochs[k], Scalar::from_canonical_le(et.data() + 32 * k)};
    return out;  // ascending epoch order, as the ordered map
}

bool paver(const PoslocPublicKey& pk, const std::map<uint32_t, std::vector<Bytes>>& batches,
           const Scalar& s_hat, const std::optional<GroupElement>& r_hat_agg, const SeedStack& ds,
           unsigned workers) {
    // same validation order as batch_verify.cpp:68-83: batch sizes (the
    // pack's map walk), the commitments, then workers (agg_ekeys, :15)
    const auto t_call = sclock::now();
    double pack_ms = 0;
    Packed p;
    pack(pk.suite, batches, ds, p, true);
    pack_ms += ms_between(t_call, sclock::now());
    for (const std::vector<Bytes>* m : p.msgs)
        if (m->size() != pk.suite.n2) throw StateError("every batch must hold exactly n2 entries");
    std::vector<uint8_t> r_hats;
    if (!r_hat_agg) {  // both key lists are ordered: one merge walk finds every commitment
        r_hats.resize(32 * p.epochs.size());
        auto it = pk.r_hats.begin();
        size_t k = 0;
        for (const uint32_t i : p.epochs) {
            while (it != pk.r_hats.end() && it->first < i) ++it;
            if (it == pk.r_hats.end() || it->first != i)
                throw StateError("commitment for epoch " + std::to_string(i) + " no longer in public key");
            std::memcpy(&r_hats[32 * k++], it->second.bytes().data(), 32);
        }
    }
    if (workers == 0) throw StateError("worker count must be at least 1");
    uint8_t verdict = 0;
    poslo_error err{};
    auto run = [&](bool fixed_guess, Packed& q) {
        if (&q != &p) {
            const auto t_pack = sclock::now();
            pack(pk.suite, batches, ds, q, fixed_guess);
            pack_ms += ms_between(t_pack, sclock::now());
        }
        return poslo_gpu_paver(device(workers), &q.b, pk.y.bytes().data(), s_hat.le_bytes().data(),
                               r_hat_agg ? r_hat_agg->bytes().data() : nullptr, r_hat_agg ? nullptr : r_hats.data(),
                               &verdict, &err);
    };
    int rc = run(true, p);
    double fill_ms = p.fill_ms, entries = (double)p.b.n_entries;
    if (rc != POSLO_OK && p.mismatch.load()) {  // mixed entry lengths: again with byte offsets
        Packed q;
        rc = run(false, q);
        fill_ms += q.fill_ms;
    }
    record_stats(pack_ms, fill_ms, ms_between(t_call, sclock::now()), entries);
    if (rc != POSLO_OK) rethrow(err);
    return verdict != 0;
}

}  // namespace poslo

// Host-side breakdown of the last drop-in paver call: {pack_ms, fill_ms,
// call_ms, entries} (bench.py's e2e_dropin line reports it).
extern "C" void poslo_dropin_last_stats(double out[4]) {
    std::lock_guard<std::mutex> lk(poslo::g_stats_m);
    for (int k = 0; k < 4; k++) out[k] = poslo::g_stats[k];
}
