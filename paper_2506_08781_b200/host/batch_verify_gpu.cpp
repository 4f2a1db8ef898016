// B200 drop-in for the reference's batch verifier: defines poslo::agg_ekeys
// and poslo::paver with the exact signatures and error behaviour of
// /root/reference/proj/include/poslo/batch_verify.hpp:11-30 (implementation
// it replaces: proj/src/batch_verify.cpp:11-87), on top of the C-ABI in
// include/poslo_gpu.h. Compiled against the reference's own headers in place
// of src/batch_verify.cpp; see INTEGRATION.md.
//
// The std::map<uint32_t, std::vector<Bytes>> batches are packed into one
// payload (+ byte offsets when lengths differ) and epoch ranges; all hashing,
// modular sums and the group check run on the device. `workers` keeps its
// reference meaning only as a parameter check (0 -> StateError).
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "poslo/batch_verify.hpp"
#include "poslo_gpu.h"

namespace poslo {

namespace {

// One device context per host thread: the C-ABI serialises calls per
// context, so thread-local contexts keep concurrent callers independent
// ("externally a pure, thread-safe function").
struct DeviceContext {
    poslo_gpu_ctx* ctx = nullptr;
    DeviceContext() {
        poslo_error err{};
        int dev = 0;
        if (const char* e = std::getenv("POSLO_GPU_DEVICE")) dev = std::atoi(e);
        if (poslo_gpu_create(dev, &ctx, &err) != POSLO_OK)
            throw std::runtime_error(std::string("poslo_gpu: ") + err.message);
    }
    ~DeviceContext() { poslo_gpu_destroy(ctx); }
};

poslo_gpu_ctx* device() {
    thread_local std::unique_ptr<DeviceContext> dc;
    if (!dc) dc = std::make_unique<DeviceContext>();
    return dc->ctx;
}

[[noreturn]] void rethrow(const poslo_error& e) {
    switch (e.code) {
        case POSLO_FORMAT_ERROR: throw FormatError(e.message);
        case POSLO_STATE_ERROR: throw StateError(e.message);
        case POSLO_SEED_NOT_DISCLOSED: throw SeedNotDisclosed(e.epoch);
        default: throw std::runtime_error(std::string("poslo_gpu: ") + e.message);
    }
}

struct Packed {
    std::vector<uint8_t> payload;
    std::vector<uint64_t> offsets;
    std::vector<uint32_t> epochs;
    std::vector<uint64_t> starts;
    Bytes ds;
    poslo_batch b{};
};

void pack(const SuiteConfig& suite, const std::map<uint32_t, std::vector<Bytes>>& batches,
          const SeedStack& ds, Packed& p) {
    size_t total = 0, n = 0;
    bool fixed = true, uniform = true;
    size_t len0 = SIZE_MAX;
    for (const auto& [i, msgs] : batches) {
        p.epochs.push_back(i);
        if (msgs.size() != suite.n2) uniform = false;
        for (const auto& m : msgs) {
            if (len0 == SIZE_MAX) len0 = m.size();
            if (m.size() != len0) fixed = false;
            total += m.size();
            n++;
        }
    }
    p.payload.reserve(total);
    if (!fixed) p.offsets.reserve(n + 1);
    if (!uniform) p.starts.reserve(batches.size() + 1);
    uint64_t t = 0;
    for (const auto& [i, msgs] : batches) {
        if (!uniform) p.starts.push_back(t);
        for (const auto& m : msgs) {
            if (!fixed) p.offsets.push_back(p.payload.size());
            p.payload.insert(p.payload.end(), m.begin(), m.end());
            t++;
        }
    }
    if (!fixed) p.offsets.push_back(p.payload.size());
    if (!uniform) p.starts.push_back(t);
    ds.serialize(p.ds);
    poslo_batch& b = p.b;
    b.suite = static_cast<uint8_t>(suite.suite);
    b.n2 = suite.n2;
    b.payload = p.payload.data();
    b.payload_bytes = p.payload.size();
    b.offsets = fixed ? nullptr : p.offsets.data();
    b.entry_len = fixed && len0 != SIZE_MAX ? static_cast<uint32_t>(len0) : 0;
    b.n_entries = n;
    b.epochs = p.epochs.data();
    b.epoch_starts = uniform ? nullptr : p.starts.data();
    b.n_epochs = static_cast<uint32_t>(p.epochs.size());
    b.ds = p.ds.data();
    b.ds_len = static_cast<uint32_t>(p.ds.size());
    b.ds_capacity = ds.capacity();
    b.device_resident = 0;
}

}  // namespace

std::vector<EpochKeyAggregate> agg_ekeys(const SuiteConfig& suite,
                                         const std::map<uint32_t, std::vector<Bytes>>& batches,
                                         const SeedStack& ds, unsigned workers) {
    if (workers == 0) throw StateError("worker count must be at least 1");
    Packed p;
    pack(suite, batches, ds, p);
    std::vector<uint8_t> et(32 * std::max<size_t>(p.epochs.size(), 1));
    poslo_error err{};
    if (poslo_gpu_agg_ekeys(device(), &p.b, et.data(), nullptr, &err) != POSLO_OK) rethrow(err);
    std::vector<EpochKeyAggregate> out(p.epochs.size());
    for (size_t k = 0; k < p.epochs.size(); k++)
        out[k] = EpochKeyAggregate{p.epochs[k], Scalar::from_canonical_le(et.data() + 32 * k)};
    return out;  // ascending epoch order, as the ordered map
}

bool paver(const PoslocPublicKey& pk, const std::map<uint32_t, std::vector<Bytes>>& batches,
           const Scalar& s_hat, const std::optional<GroupElement>& r_hat_agg, const SeedStack& ds,
           unsigned workers) {
    // same validation order as batch_verify.cpp:68-83
    for (const auto& [i, msgs] : batches)
        if (msgs.size() != pk.suite.n2) throw StateError("every batch must hold exactly n2 entries");
    std::vector<uint8_t> r_hats;
    if (!r_hat_agg) {
        r_hats.reserve(32 * batches.size());
        for (const auto& [i, msgs] : batches) {
            auto it = pk.r_hats.find(i);
            if (it == pk.r_hats.end())
                throw StateError("commitment for epoch " + std::to_string(i) + " no longer in public key");
            r_hats.insert(r_hats.end(), it->second.bytes().begin(), it->second.bytes().end());
        }
    }
    if (workers == 0) throw StateError("worker count must be at least 1");
    Packed p;
    pack(pk.suite, batches, ds, p);
    uint8_t verdict = 0;
    poslo_error err{};
    int rc = poslo_gpu_paver(device(), &p.b, pk.y.bytes().data(), s_hat.le_bytes().data(),
                             r_hat_agg ? r_hat_agg->bytes().data() : nullptr,
                             r_hat_agg ? nullptr : r_hats.data(), &verdict, &err);
    if (rc != POSLO_OK) rethrow(err);
    return verdict != 0;
}

}  // namespace poslo
