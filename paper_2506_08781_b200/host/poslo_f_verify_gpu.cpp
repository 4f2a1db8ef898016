// B200 drop-in for the scheme-F verifiers: defines poslo::aver_f_single and
// poslo::aver_f_batch with the signatures and error behaviour of
// /root/reference/proj/include/poslo/poslo_f.hpp:83-91 (implementation it
// replaces: proj/src/poslo_f.cpp:223-246), on top of the C-ABI in
// include/poslo_gpu.h:
//   aver_f_single -> poslo_gpu_fine_verify, one entry with its seed tail
//   aver_f_batch  -> poslo_gpu_aver_f_batch, every seed derived from ds
//                    (one slot per epoch t / n2, ascending like the map)
// The signer side of poslo_f.cpp stays the reference's. A build takes these two
// definitions instead of the reference's by moving them out of poslo_f.cpp, or
// (as host/Makefile does for the reference's own test_poslo_f.cpp) by linking
// a copy of poslo_f.o whose two symbols are weakened with objcopy.
#include <cstring>
#include <memory>
#include <string>

#include "poslo/poslo_f.hpp"
#include "poslo_gpu.h"

namespace poslo {

namespace {

struct FCtx {
    poslo_gpu_ctx* ctx = nullptr;
    FCtx() {
        poslo_error err{};
        int dev = 0;
        if (const char* e = std::getenv("POSLO_GPU_DEVICE")) dev = std::atoi(e);
        if (poslo_gpu_create(dev, &ctx, &err) != POSLO_OK)
            throw std::runtime_error(std::string("poslo_gpu: ") + err.message);
    }
    ~FCtx() { poslo_gpu_destroy(ctx); }
};

poslo_gpu_ctx* fdev() {
    thread_local std::unique_ptr<FCtx> c;
    if (!c) c = std::make_unique<FCtx>();
    return c->ctx;
}

void fcheck(int rc, const poslo_error& e) {
    if (rc == POSLO_OK) return;
    switch (e.code) {
        case POSLO_FORMAT_ERROR: throw FormatError(e.message);
        case POSLO_STATE_ERROR: throw StateError(e.message);
        case POSLO_SEED_NOT_DISCLOSED: throw SeedNotDisclosed(e.epoch);
        default: throw std::runtime_error(std::string("poslo_gpu: ") + e.message);
    }
}

const uint8_t* nonnull(const Bytes& b) {
    static const uint8_t none = 0;
    return b.empty() ? &none : b.data();
}

}  // namespace

bool aver_f_single(const PoslofPublicKey& pk, const Bytes& msg, const FineSignature& sig) {
    const Seed* x = std::get_if<Seed>(&sig.tail);
    if (!x) throw FormatError("single-entry verification needs the seed tail, not ds");
    const uint64_t offs[2] = {0, msg.size()};
    poslo_fine_batch fb{};
    fb.suite = static_cast<uint8_t>(pk.suite.suite);
    fb.payload = nonnull(msg);
    fb.payload_bytes = msg.size();
    fb.offsets = offs;
    fb.n_entries = 1;
    fb.seeds = x->data();
    const auto s = sig.s.le_bytes();
    uint8_t verdict = 0;
    poslo_error err{};
    fcheck(poslo_gpu_fine_verify(fdev(), &fb, pk.y.bytes().data(), s.data(), sig.r.bytes().data(),
                                 &verdict, &err),
           err);
    return verdict != 0;
}

bool aver_f_batch(const PoslofPublicKey& pk, const std::map<uint32_t, Bytes>& entries, const Scalar& s,
                  const GroupElement& r, const SeedStack& ds) {
    const uint32_t n2 = pk.suite.n2;
    std::vector<uint8_t> payload;
    std::vector<uint64_t> offs{0};
    std::vector<uint32_t> slot, jj, slot_epochs;
    slot.reserve(entries.size());
    jj.reserve(entries.size());
    for (const auto& [t, msg] : entries) {
        const uint32_t i = t / n2;
        if (slot_epochs.empty() || slot_epochs.back() != i) slot_epochs.push_back(i);
        slot.push_back(static_cast<uint32_t>(slot_epochs.size() - 1));
        jj.push_back(t % n2);
        payload.insert(payload.end(), msg.begin(), msg.end());
        offs.push_back(payload.size());
    }
    Bytes dsw;
    ds.serialize(dsw);
    poslo_fine_batch fb{};
    fb.suite = static_cast<uint8_t>(pk.suite.suite);
    fb.payload = nonnull(payload);
    fb.payload_bytes = payload.size();
    fb.offsets = offs.data();
    fb.n_entries = entries.size();
    fb.derive_slot = slot.data();
    fb.j = jj.data();
    fb.slot_epochs = slot_epochs.data();
    fb.n_slots = static_cast<uint32_t>(slot_epochs.size());
    fb.ds = dsw.data();
    fb.ds_len = static_cast<uint32_t>(dsw.size());
    fb.ds_capacity = pk.suite.depth();
    const auto sb = s.le_bytes();
    uint8_t verdict = 0;
    poslo_error err{};
    fcheck(poslo_gpu_aver_f_batch(fdev(), &fb, pk.y.bytes().data(), sb.data(), r.bytes().data(), &verdict,
                                  &err),
           err);
    return verdict != 0;
}

}  // namespace poslo
