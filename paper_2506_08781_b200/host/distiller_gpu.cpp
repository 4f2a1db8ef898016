// B200 drop-in for the reference's distiller: defines the members of
// poslo::ColdCryptoData declared in /root/reference/proj/include/poslo/
// distiller.hpp:31-98 (implementation it replaces: proj/src/distiller.cpp)
// on top of the C-ABI in include/poslo_gpu.h. Every verdict, hash, modular
// sum and group fold runs on the device:
//   distill_epoch       -> poslo_gpu_distill_step (the epoch verified with
//                          its own signature's ds and folded into the valid
//                          and umbrella aggregates: one device round trip)
//   distill_epoch_fine  -> poslo_gpu_fine_verify (seed tails, or the epoch's
//                          new stack for the ds-carrying entry) + segfold
//   sebver (coarse)     -> poslo_gpu_sebver
//   sebver (fine)       -> poslo_gpu_fine_scalars + segfold + group_check
// The CCD wire format (PCCD ... CRC-32) is written and parsed here, byte for
// byte the reference's (distiller.cpp:235-304), with the same errors.
// Group elements computed on the device are canonical encodings; they enter
// GroupElement by copy (trivially copyable 32-byte class) rather than through
// from_bytes, whose CPU membership check would re-verify device output.
#include <zlib.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <set>
#include <string>
#include <type_traits>

#include "poslo/distiller.hpp"
#include "poslo_gpu.h"

namespace poslo {

namespace {

static_assert(std::is_trivially_copyable_v<GroupElement> && sizeof(GroupElement) == kPointBytes);
static_assert(std::is_trivially_copyable_v<Scalar> && sizeof(Scalar) == kScalarBytes);

struct Ctx {
    poslo_gpu_ctx* ctx = nullptr;
    Ctx() {
        poslo_error err{};
        int dev = 0;
        if (const char* e = std::getenv("POSLO_GPU_DEVICE")) dev = std::atoi(e);
        if (poslo_gpu_create(dev, &ctx, &err) != POSLO_OK)
            throw std::runtime_error(std::string("poslo_gpu: ") + err.message);
    }
    ~Ctx() { poslo_gpu_destroy(ctx); }
};

poslo_gpu_ctx* dev() {
    thread_local std::unique_ptr<Ctx> c;
    if (!c) c = std::make_unique<Ctx>();
    return c->ctx;
}

[[noreturn]] void raise(const poslo_error& e) {
    switch (e.code) {
        case POSLO_FORMAT_ERROR: throw FormatError(e.message);
        case POSLO_STATE_ERROR: throw StateError(e.message);
        case POSLO_SEED_NOT_DISCLOSED: throw SeedNotDisclosed(e.epoch);
        default: throw std::runtime_error(std::string("poslo_gpu: ") + e.message);
    }
}

void check(int rc, const poslo_error& e) {
    if (rc != POSLO_OK) raise(e);
}

GroupElement point_of(const uint8_t* p) {
    GroupElement g;
    std::memcpy(static_cast<void*>(&g), p, kPointBytes);
    return g;
}

Scalar scalar_of(const uint8_t* p) { return Scalar::from_canonical_le(p); }

void append(std::vector<uint8_t>& v, const uint8_t* p, size_t n) { v.insert(v.end(), p, p + n); }

// Folds items into accumulators on the device: out[g] = acc[g] + sum of the
// items of group g (Scalar::add / group_combine, distiller.cpp:45-53).
std::vector<AggregatePair> fold(const std::vector<AggregatePair>& acc,
                                const std::vector<std::vector<AggregatePair>>& items) {
    std::vector<uint8_t> s, r;
    std::vector<uint32_t> seg{0};
    for (size_t g = 0; g < acc.size(); g++) {
        append(s, acc[g].s.le_bytes().data(), kScalarBytes);
        append(r, acc[g].r.bytes().data(), kPointBytes);
        for (const auto& it : items[g]) {
            append(s, it.s.le_bytes().data(), kScalarBytes);
            append(r, it.r.bytes().data(), kPointBytes);
        }
        seg.push_back(static_cast<uint32_t>(s.size() / kScalarBytes));
    }
    std::vector<uint8_t> os(kScalarBytes * acc.size()), orr(kPointBytes * acc.size());
    poslo_error err{};
    check(poslo_gpu_segfold(dev(), seg.back(), s.data(), r.data(), nullptr, seg.data(),
                            static_cast<uint32_t>(acc.size()), os.data(), orr.data(), &err),
          err);
    std::vector<AggregatePair> out(acc.size());
    for (size_t g = 0; g < acc.size(); g++)
        out[g] = AggregatePair{scalar_of(&os[kScalarBytes * g]), point_of(&orr[kPointBytes * g])};
    return out;
}

// Packed entries for a poslo_batch / poslo_fine_batch.
struct Entries {
    std::vector<uint8_t> bytes;
    std::vector<uint64_t> offsets{0};
    void add(const Bytes& m) {
        bytes.insert(bytes.end(), m.begin(), m.end());
        offsets.push_back(bytes.size());
    }
    uint64_t n() const { return offsets.size() - 1; }
    uint64_t size() const { return bytes.size(); }
    const uint8_t* data() const {  // never null: all-empty entries still need a payload pointer
        static const uint8_t none = 0;
        return bytes.empty() ? &none : bytes.data();
    }
};

void put_pair_wire(Bytes& out, const AggregatePair& p) {
    const auto be = p.s.be_bytes();
    out.insert(out.end(), be.begin(), be.end());
    out.insert(out.end(), p.r.bytes().begin(), p.r.bytes().end());
}

}  // namespace

ColdCryptoData::ColdCryptoData(CcdScheme scheme, const SuiteConfig& suite)
    : scheme_(scheme), suite_(suite), ds_(suite.depth()) {
    suite.validate();
}

const AggregatePair& ColdCryptoData::valid() const {
    if (!has_valid_) throw StateError("no valid aggregate distilled yet");
    return valid_;
}

void ColdCryptoData::record_invalid(uint32_t index, const Scalar& s, const GroupElement& r) {
    invalid_.push_back(InvalidRecord{index, AggregatePair{s, r}});
}

void ColdCryptoData::distill_epoch(PoslocPublicKey& pk, const std::vector<Bytes>& msgs,
                                   const EpochSignature& sig) {
    if (scheme_ != CcdScheme::Coarse) throw StateError("coarse distillation on a fine-grained stream");
    if (next_epoch_ >= suite_.n1) throw StateError("stream already complete");
    const uint32_t i = next_epoch_;
    auto it = pk.r_hats.find(i);
    if (it == pk.r_hats.end())
        throw StateError("epoch " + std::to_string(i) + " already distilled (commitment gone)");
    // aver(pk, {i: msgs}, sig.s_hat, nullopt, sig.ds) on the device
    Entries e;
    for (const auto& m : msgs) e.add(m);
    Bytes dsw;
    sig.ds.serialize(dsw);
    const uint32_t epoch = i;
    const uint64_t starts[2] = {0, e.n()};
    poslo_batch b{};
    b.suite = static_cast<uint8_t>(suite_.suite);
    b.n2 = suite_.n2;
    b.payload = e.data();
    b.payload_bytes = e.size();
    b.offsets = e.offsets.data();
    b.n_entries = e.n();
    b.epochs = &epoch;
    b.epoch_starts = starts;  // the device checks the n2 batch size (StateError) first
    b.n_epochs = 1;
    b.ds = dsw.data();
    b.ds_len = static_cast<uint32_t>(dsw.size());
    b.ds_capacity = suite_.depth();
    // verdict and the fold into both running aggregates in one device round trip
    uint8_t verdict = 0, acc_s[2 * kScalarBytes], acc_r[2 * kPointBytes], out_s[2 * kScalarBytes],
        out_r[2 * kPointBytes];
    std::memcpy(acc_s, valid_.s.le_bytes().data(), kScalarBytes);
    std::memcpy(acc_s + kScalarBytes, umb_acc_.s.le_bytes().data(), kScalarBytes);
    std::memcpy(acc_r, valid_.r.bytes().data(), kPointBytes);
    std::memcpy(acc_r + kPointBytes, umb_acc_.r.bytes().data(), kPointBytes);
    poslo_error err{};
    check(poslo_gpu_distill_step(dev(), &b, pk.y.bytes().data(), sig.s_hat.le_bytes().data(),
                                 it->second.bytes().data(), acc_s, acc_r, &verdict, out_s, out_r, &err),
          err);
    if (verdict) {
        valid_ = AggregatePair{scalar_of(out_s), point_of(out_r)};
        umb_acc_ = AggregatePair{scalar_of(out_s + kScalarBytes), point_of(out_r + kPointBytes)};
        has_valid_ = true;
        umb_acc_nonempty_ = true;
    } else {
        record_invalid(i, sig.s_hat, it->second);
    }
    pk.r_hats.erase(it);
    ds_ = sig.ds;
    next_epoch_++;
    if (next_epoch_ % umbrella_width() == 0) {
        umbrellas_.push_back(UmbrellaRecord{(next_epoch_ - 1) / umbrella_width(), umb_acc_});
        umb_acc_ = AggregatePair{};
        umb_acc_nonempty_ = false;
    }
}

void ColdCryptoData::distill_epoch_fine(const PoslofPublicKey& pk, const std::vector<Bytes>& msgs,
                                        const std::vector<FineSignature>& sigs) {
    if (scheme_ != CcdScheme::Fine) throw StateError("fine distillation on a coarse stream");
    if (next_epoch_ >= suite_.n1) throw StateError("stream already complete");
    if (msgs.size() != suite_.n2 || sigs.size() != suite_.n2)
        throw StateError("epoch must hold exactly n2 entries and signatures");
    const uint32_t i = next_epoch_;
    if (!sigs.back().carries_ds()) throw FormatError("last entry of the epoch must carry ds");
    const SeedStack& ds_new = std::get<SeedStack>(sigs.back().tail);
    // per entry: seed tail (aver_f_single) or onetime_seed(sr(ds_new, i), j)
    Entries e;
    std::vector<uint8_t> seeds(kSeedBytes * suite_.n2, 0), s, r;
    std::vector<uint32_t> slot(suite_.n2, 0xFFFFFFFFu), jj(suite_.n2, 0);
    for (uint32_t j = 0; j < suite_.n2; j++) {
        e.add(msgs[j]);
        if (sigs[j].carries_ds()) {
            slot[j] = 0;
            jj[j] = j;
        } else {
            const Seed& x = std::get<Seed>(sigs[j].tail);
            std::memcpy(&seeds[kSeedBytes * j], x.data(), kSeedBytes);
        }
        append(s, sigs[j].s.le_bytes().data(), kScalarBytes);
        append(r, sigs[j].r.bytes().data(), kPointBytes);
    }
    Bytes dsw;
    ds_new.serialize(dsw);
    poslo_fine_batch fb{};
    fb.suite = static_cast<uint8_t>(suite_.suite);
    fb.payload = e.data();
    fb.payload_bytes = e.size();
    fb.offsets = e.offsets.data();
    fb.n_entries = e.n();
    fb.seeds = seeds.data();
    fb.derive_slot = slot.data();
    fb.j = jj.data();
    fb.slot_epochs = &i;
    fb.n_slots = 1;
    fb.ds = dsw.data();
    fb.ds_len = static_cast<uint32_t>(dsw.size());
    fb.ds_capacity = suite_.depth();
    std::vector<uint8_t> verdicts(suite_.n2);
    poslo_error err{};
    check(poslo_gpu_fine_verify(dev(), &fb, pk.y.bytes().data(), s.data(), r.data(), verdicts.data(), &err), err);
    std::vector<AggregatePair> good;
    for (uint32_t j = 0; j < suite_.n2; j++) {
        if (verdicts[j])
            good.push_back(AggregatePair{sigs[j].s, sigs[j].r});
        else
            record_invalid(i * suite_.n2 + j, sigs[j].s, sigs[j].r);
    }
    if (!good.empty()) {
        auto out = fold({valid_, umb_acc_}, {good, good});
        valid_ = out[0];
        umb_acc_ = out[1];
        has_valid_ = true;
        umb_acc_nonempty_ = true;
    }
    ds_ = ds_new;
    next_epoch_++;
    if (next_epoch_ % umbrella_width() == 0) {
        umbrellas_.push_back(UmbrellaRecord{(next_epoch_ - 1) / umbrella_width(), umb_acc_});
        umb_acc_ = AggregatePair{};
        umb_acc_nonempty_ = false;
    }
}

void ColdCryptoData::finalize() {
    if (!umb_acc_nonempty_) return;
    umbrellas_.push_back(UmbrellaRecord{(next_epoch_ - 1) / umbrella_width(), umb_acc_});
    umb_acc_ = AggregatePair{};
    umb_acc_nonempty_ = false;
}

std::map<uint32_t, std::vector<Bytes>> ColdCryptoData::collect_epochs(
    const std::map<uint32_t, std::vector<Bytes>>& all_msgs, uint32_t lo, uint32_t hi) const {
    std::map<uint32_t, std::vector<Bytes>> out;
    for (uint32_t i = lo; i < std::min(hi, next_epoch_); i++) {
        auto it = all_msgs.find(i);
        if (it == all_msgs.end()) throw FormatError("messages for epoch " + std::to_string(i) + " missing");
        if (it->second.size() != suite_.n2) throw FormatError("epoch batch size mismatch");
        out.emplace(i, it->second);
    }
    return out;
}

std::vector<bool> ColdCryptoData::sebver(const GroupElement& y,
                                         const std::map<uint32_t, std::vector<Bytes>>& all_msgs,
                                         SebverMode mode) const {
    const uint32_t w = umbrella_width();
    if (mode == SebverMode::V && !has_valid_) throw StateError("mode V needs a valid aggregate");
    // the ranges the reference reads, in its order (distiller.cpp:181-233)
    std::vector<std::pair<uint32_t, uint32_t>> ranges;
    if (mode == SebverMode::V) ranges.push_back({0, next_epoch_});
    if (mode == SebverMode::U)
        for (const auto& u : umbrellas_) ranges.push_back({u.index * w, (u.index + 1) * w});
    Bytes dsw;
    ds_.serialize(dsw);
    poslo_error err{};
    if (scheme_ == CcdScheme::Coarse) {
        // groups in the reference's order: each reads its epochs (collect_epochs or the
        // mode-I lookup) and hashes the non-invalid ones (verify_range, :161-162). The
        // reference raises at the first group with missing messages, after hashing
        // every group before it; the device hashes exactly those epochs (seeds are
        // derived for no other epoch), then the missing-message error is raised.
        std::set<uint32_t> bad_ep;
        for (const auto& rec : invalid_) bad_ep.insert(rec.index);
        std::set<uint32_t> hashed;
        size_t live = mode == SebverMode::I ? invalid_.size() : ranges.size();
        std::string missing;
        auto read_ok = [&](uint32_t i, bool need_n2) -> bool {
            auto it = all_msgs.find(i);
            if (it == all_msgs.end()) {
                missing = mode == SebverMode::I ? "messages for invalid epoch missing"
                                                : "messages for epoch " + std::to_string(i) + " missing";
                return false;
            }
            if (need_n2 && it->second.size() != suite_.n2) {
                missing = "epoch batch size mismatch";
                return false;
            }
            return true;
        };
        if (mode == SebverMode::I) {
            for (size_t k = 0; k < invalid_.size(); k++) {
                if (!read_ok(invalid_[k].index, false)) {
                    live = k;
                    break;
                }
                hashed.insert(invalid_[k].index);
            }
        } else {
            for (size_t k = 0; k < ranges.size(); k++) {
                bool ok = true;
                for (uint32_t i = ranges[k].first; i < std::min(ranges[k].second, next_epoch_) && ok; i++)
                    ok = read_ok(i, true);
                if (!ok) {
                    live = k;
                    break;
                }
                for (uint32_t i = ranges[k].first; i < std::min(ranges[k].second, next_epoch_); i++)
                    if (!bad_ep.count(i)) hashed.insert(i);
            }
        }
        if (!missing.empty() && live == 0) throw FormatError(missing);
        Entries e;
        std::vector<uint32_t> epochs;
        std::vector<uint64_t> starts{0};
        for (uint32_t i : hashed) {
            for (const auto& m : all_msgs.at(i)) e.add(m);
            epochs.push_back(i);
            starts.push_back(e.n());
        }
        poslo_batch b{};
        b.suite = static_cast<uint8_t>(suite_.suite);
        b.n2 = suite_.n2;
        b.payload = e.data();
        b.payload_bytes = e.size();
        b.offsets = e.offsets.data();
        b.n_entries = e.n();
        b.epochs = epochs.data();
        b.epoch_starts = starts.data();
        b.n_epochs = static_cast<uint32_t>(epochs.size());
        b.ds = dsw.data();
        b.ds_len = static_cast<uint32_t>(dsw.size());
        b.ds_capacity = suite_.depth();
        std::vector<uint32_t> inv, ui;
        std::vector<uint8_t> is, ir, us, ur;
        for (size_t k = 0; k < invalid_.size(); k++) {
            const auto& rec = invalid_[k];
            if (mode == SebverMode::I && k >= live) break;
            inv.push_back(rec.index);
            append(is, rec.sig.s.le_bytes().data(), kScalarBytes);
            append(ir, rec.sig.r.bytes().data(), kPointBytes);
        }
        for (size_t k = 0; k < umbrellas_.size() && (mode != SebverMode::U || k < live); k++) {
            const auto& u = umbrellas_[k];
            ui.push_back(u.index);
            append(us, u.sig.s.le_bytes().data(), kScalarBytes);
            append(ur, u.sig.r.bytes().data(), kPointBytes);
        }
        uint8_t vbit = 0;
        std::vector<uint8_t> ubits(std::max<size_t>(ui.size(), 1)), ibits(std::max<size_t>(inv.size(), 1));
        const bool want_v = mode == SebverMode::V, want_u = mode == SebverMode::U, want_i = mode == SebverMode::I;
        check(poslo_gpu_sebver(dev(), &b, y.bytes().data(), suite_.n1, suite_.n_u, inv.data(), is.data(), ir.data(),
                               static_cast<uint32_t>(inv.size()), want_v ? valid_.s.le_bytes().data() : nullptr,
                               want_v ? valid_.r.bytes().data() : nullptr, want_v ? &vbit : nullptr, ui.data(),
                               us.data(), ur.data(), want_u ? static_cast<uint32_t>(ui.size()) : 0,
                               want_u ? ubits.data() : nullptr, want_i ? ibits.data() : nullptr, &err),
              err);
        if (!missing.empty()) throw FormatError(missing);
        if (want_v) return {vbit != 0};
        std::vector<bool> bits;
        const size_t n = want_u ? ui.size() : inv.size();
        for (size_t k = 0; k < n; k++) bits.push_back((want_u ? ubits[k] : ibits[k]) != 0);
        return bits;
    }
    // fine scheme: the reads of collect_epochs / the mode-I lookup, in order
    for (const auto& [lo, hi] : ranges) collect_epochs(all_msgs, lo, hi);
    if (mode == SebverMode::I)
        for (const auto& rec : invalid_) {
            auto it = all_msgs.find(rec.index / suite_.n2);
            if (it == all_msgs.end() || it->second.size() <= rec.index % suite_.n2)
                throw FormatError("message for invalid entry missing");
        }
    // fine scheme: entry scalars from the disclosed stack, on the device
    std::set<uint32_t> bad;
    for (const auto& rec : invalid_) bad.insert(rec.index);
    Entries e;
    std::vector<uint32_t> slot, jj, slot_epochs;
    auto add_entry = [&](uint32_t i, uint32_t j) {
        e.add(all_msgs.at(i)[j]);
        if (slot_epochs.empty() || slot_epochs.back() != i) slot_epochs.push_back(i);
        slot.push_back(static_cast<uint32_t>(slot_epochs.size() - 1));
        jj.push_back(j);
    };
    poslo_fine_batch fb{};
    auto finish = [&]() {
        fb.suite = static_cast<uint8_t>(suite_.suite);
        fb.payload = e.data();
        fb.payload_bytes = e.size();
        fb.offsets = e.offsets.data();
        fb.n_entries = e.n();
        fb.derive_slot = slot.data();
        fb.j = jj.data();
        fb.slot_epochs = slot_epochs.data();
        fb.n_slots = static_cast<uint32_t>(slot_epochs.size());
        fb.ds = dsw.data();
        fb.ds_len = static_cast<uint32_t>(dsw.size());
        fb.ds_capacity = suite_.depth();
    };
    if (mode == SebverMode::I) {
        if (invalid_.empty()) return {};
        std::vector<uint8_t> s, r;
        for (const auto& rec : invalid_) {
            add_entry(rec.index / suite_.n2, rec.index % suite_.n2);
            append(s, rec.sig.s.le_bytes().data(), kScalarBytes);
            append(r, rec.sig.r.bytes().data(), kPointBytes);
        }
        finish();
        std::vector<uint8_t> v(invalid_.size());
        check(poslo_gpu_fine_verify(dev(), &fb, y.bytes().data(), s.data(), r.data(), v.data(), &err), err);
        return std::vector<bool>(v.begin(), v.end());
    }
    // V / U: sum of e over each range's non-quarantined entries, one check per range
    std::vector<uint32_t> seg{0};
    std::vector<uint8_t> keep;
    for (const auto& [lo, hi] : ranges) {
        for (uint32_t i = lo; i < std::min(hi, next_epoch_); i++)
            for (uint32_t j = 0; j < suite_.n2; j++) {
                add_entry(i, j);
                keep.push_back(bad.count(i * suite_.n2 + j) ? 0 : 1);
            }
        seg.push_back(static_cast<uint32_t>(e.n()));
    }
    finish();
    std::vector<uint8_t> es(kScalarBytes * std::max<uint64_t>(e.n(), 1));
    if (e.n()) check(poslo_gpu_fine_scalars(dev(), &fb, es.data(), nullptr, &err), err);
    std::vector<uint8_t> sums(kScalarBytes * ranges.size()), gs, gr, out(ranges.size());
    check(poslo_gpu_segfold(dev(), static_cast<uint32_t>(e.n()), es.data(), nullptr, keep.data(), seg.data(),
                            static_cast<uint32_t>(ranges.size()), sums.data(), nullptr, &err),
          err);
    for (size_t g = 0; g < ranges.size(); g++) {
        const AggregatePair& sig = mode == SebverMode::V ? valid_ : umbrellas_[g].sig;
        append(gs, sig.s.le_bytes().data(), kScalarBytes);
        append(gr, sig.r.bytes().data(), kPointBytes);
    }
    if (!ranges.empty())
        check(poslo_gpu_group_check(dev(), static_cast<uint32_t>(ranges.size()), y.bytes().data(), sums.data(),
                                    gs.data(), gr.data(), out.data(), &err),
              err);
    return std::vector<bool>(out.begin(), out.end());
}

Bytes ColdCryptoData::serialize() const {
    Bytes out{'P', 'C', 'C', 'D', static_cast<uint8_t>(scheme_), static_cast<uint8_t>(suite_.suite)};
    for (uint32_t v : {suite_.n1, suite_.n2, suite_.n_u, next_epoch_}) put_be32(out, v);
    out.push_back(has_valid_ ? 1 : 0);
    put_pair_wire(out, valid_);  // identity / zero when absent
    put_be32(out, static_cast<uint32_t>(umbrellas_.size()));
    for (const auto& u : umbrellas_) {
        put_be32(out, u.index);
        put_pair_wire(out, u.sig);
    }
    put_be32(out, static_cast<uint32_t>(invalid_.size()));
    for (const auto& rec : invalid_) {
        put_be32(out, rec.index);
        put_pair_wire(out, rec.sig);
    }
    ds_.serialize(out);
    put_be32(out, static_cast<uint32_t>(crc32(0, out.data(), static_cast<uInt>(out.size()))));
    return out;
}

ColdCryptoData ColdCryptoData::deserialize(const Bytes& in) {
    if (in.size() < 4) throw FormatError("truncated CCD");
    const size_t body = in.size() - 4;
    if (load_be32(in.data() + body) != static_cast<uint32_t>(crc32(0, in.data(), static_cast<uInt>(body))))
        throw FormatError("CCD checksum mismatch");
    Reader rd(in.data(), body);
    rd.expect_magic("PCCD");
    ColdCryptoData c;
    c.scheme_ = static_cast<CcdScheme>(rd.u8());
    if (c.scheme_ != CcdScheme::Coarse && c.scheme_ != CcdScheme::Fine) throw FormatError("bad CCD scheme byte");
    c.suite_.suite = static_cast<SuiteId>(rd.u8());
    c.suite_.n1 = rd.be32();
    c.suite_.n2 = rd.be32();
    c.suite_.n_u = rd.be32();
    c.suite_.validate();
    c.next_epoch_ = rd.be32();
    const uint8_t flag = rd.u8();
    if (flag > 1) throw FormatError("bad valid-aggregate flag");
    c.has_valid_ = flag == 1;
    // pairs: scalar range check here, group membership of every point in one device call
    std::vector<uint8_t> pts;
    auto pair = [&]() {
        AggregatePair p;
        p.s = Scalar::from_be_bytes(rd.take(kScalarBytes));
        const uint8_t* q = rd.take(kPointBytes);
        append(pts, q, kPointBytes);
        p.r = point_of(q);
        return p;
    };
    c.valid_ = pair();
    for (uint32_t k = 0, n = rd.be32(); k < n; k++) {
        const uint32_t idx = rd.be32();
        c.umbrellas_.push_back(UmbrellaRecord{idx, pair()});
    }
    for (uint32_t k = 0, n = rd.be32(); k < n; k++) {
        const uint32_t idx = rd.be32();
        c.invalid_.push_back(InvalidRecord{idx, pair()});
    }
    const uint32_t np = static_cast<uint32_t>(pts.size() / kPointBytes);
    std::vector<uint8_t> ok(std::max<uint32_t>(np, 1));
    poslo_error err{};
    check(poslo_gpu_point_valid(dev(), np, pts.data(), ok.data(), &err), err);
    for (uint32_t k = 0; k < np; k++)
        if (!ok[k]) throw FormatError("invalid group element encoding");
    c.ds_ = SeedStack::deserialize(rd, c.suite_.depth());
    rd.expect_end();
    return c;
}

}  // namespace poslo
