// Reference-side harness: links the UNMODIFIED reference library built from
// /root/reference/proj/src (oracle/Makefile.ref) and drives it through its
// public API only. Test infrastructure — never on the product path.
//
//   ref_tool kat                       known-answer values (SURVEY App. C inputs
//                                      + random scalar/group anchors), JSON
//   ref_tool golden S N1 N2 NU LEN SEED [TAMPER...]
//                                      one signed coarse stream from the real
//                                      signer (kg/sig_epoch) with deterministic
//                                      randombytes, plus every verifier output
//                                      the GPU path must reproduce, JSON
//   ref_tool golden_f S N1 N2 NU LEN SEED BPV_V BPV_K [TAMPER...]
//                                      one signed fine-grained (POSLO-F) stream from
//                                      the real signer (kg/sig_one) with every
//                                      scheme-F verifier output: aver_f_single per
//                                      entry, aver_f_batch (all / a subset), fine
//                                      distillation CCD + SeBVer V/U/I, JSON
//   ref_tool paver FILE                the reference paver (and agg_ekeys' e-hat)
//                                      on a fixture written by the GPU tests
//                                      (tests/test_gpu_fullsize.py, "PVIO"
//                                      layout below), JSON
//   ref_tool bench S LOG2N N2 LEN WORKERS SEED REPS [MODE]
//                                      times reference paver (MODE=coarse) or
//                                      the per-epoch aver loop sharded over
//                                      WORKERS threads (MODE=epoch) on the
//                                      synthetic log of include/poslo_synth.h,
//                                      cmd_bench-style (proj/tools/poslo.cpp:248-254)
#include <sodium.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <string>
#include <thread>

#include "../../include/poslo_synth.h"
#include "poslo/batch_verify.hpp"
#include "poslo/distiller.hpp"
#include "poslo/poslo_f.hpp"

using namespace poslo;

namespace {

// ---- deterministic randombytes (so kg/sig fixtures reproduce) -------------
uint64_t g_rb_state = 0x0123456789abcdefULL;
uint64_t rb_next() {
    uint64_t z = (g_rb_state += 0x9E3779B97F4A7C15ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
const char* rb_name() { return "splitmix64-fixture"; }
uint32_t rb_random() { return static_cast<uint32_t>(rb_next()); }
void rb_stir() {}
uint32_t rb_uniform(const uint32_t ub) {
    if (ub < 2) return 0;
    uint32_t min = (1U + ~ub) % ub, r;
    do r = rb_random(); while (r < min);
    return r % ub;
}
void rb_buf(void* const buf, const size_t size) {
    auto* p = static_cast<uint8_t*>(buf);
    for (size_t i = 0; i < size; i++) p[i] = static_cast<uint8_t>(rb_next() >> 24);
}
int rb_close() { return 0; }
randombytes_implementation g_rb_impl = {rb_name, rb_random, rb_stir, rb_uniform, rb_buf, rb_close};

std::string hex(const uint8_t* p, size_t n) {
    static const char* d = "0123456789abcdef";
    std::string s;
    for (size_t i = 0; i < n; i++) { s += d[p[i] >> 4]; s += d[p[i] & 15]; }
    return s;
}
template <class C> std::string hexv(const C& c) { return hex(c.data(), c.size()); }

Bytes synth_entry(uint64_t seed, uint64_t k, size_t len) {
    Bytes b(len);
    for (size_t i = 0; i < len; i++) b[i] = poslo_synth_byte(seed, k, static_cast<uint32_t>(i));
    return b;
}

// ---- kat -----------------------------------------------------------------
int cmd_kat() {
    std::mt19937_64 rng(0x5eed0fca7ULL);
    auto rbytes = [&](size_t n) { Bytes b(n); for (auto& x : b) x = uint8_t(rng()); return b; };
    Seed x0;
    for (int i = 0; i < 16; i++) x0[i] = uint8_t(i);
    Bytes m(32);
    for (int i = 0; i < 32; i++) m[i] = uint8_t(0x20 + i);
    std::printf("{\n");
    for (SuiteId s : {SuiteId::Sha256, SuiteId::MmoMdc2, SuiteId::MmoAddQ}) {
        int sn = int(s);
        std::printf("\"suite%d\": {\n", sn);
        std::printf("  \"prf0\": \"%s\", \"prf1\": \"%s\",\n", hexv(prf(s, 0, x0)).c_str(),
                    hexv(prf(s, 1, x0)).c_str());
        std::printf("  \"ots0\": \"%s\", \"ots5\": \"%s\",\n", hexv(onetime_seed(s, x0, 0)).c_str(),
                    hexv(onetime_seed(s, x0, 5)).c_str());
        // hash_to_scalar over lengths 1..200 with random m, x (suite 3: <=31)
        std::printf("  \"h2s\": [");
        size_t maxlen = s == SuiteId::MmoAddQ ? 31 : 200;
        for (size_t len = 1; len <= maxlen; len++) {
            Bytes mm = rbytes(len);
            Seed xx;
            for (auto& b : xx) b = uint8_t(rng());
            Scalar e = hash_to_scalar(s, mm.data(), mm.size(), xx);
            std::printf("%s[\"%s\",\"%s\",\"%s\"]", len > 1 ? "," : "", hexv(mm).c_str(),
                        hexv(xx).c_str(), hexv(e.le_bytes()).c_str());
        }
        std::printf("],\n");
        // onetime_seed over random x0/j
        std::printf("  \"ots\": [");
        for (int t = 0; t < 64; t++) {
            Seed xx;
            for (auto& b : xx) b = uint8_t(rng());
            uint32_t j = t < 8 ? uint32_t(t) : uint32_t(rng());
            std::printf("%s[\"%s\",%u,\"%s\"]", t ? "," : "", hexv(xx).c_str(), j,
                        hexv(onetime_seed(s, xx, j)).c_str());
        }
        std::printf("],\n");
        // seed retrieval: a full D=4 tree disclosed up to epoch 11
        SeedNode root{4, 0, x0};
        SeedStack ds(4);
        std::printf("  \"so_x0\": [");
        for (uint32_t i = 0; i < 12; i++)
            std::printf("%s\"%s\"", i ? "," : "", hexv(so(s, ds, root, i)).c_str());
        Bytes dsw;
        ds.serialize(dsw);
        std::printf("], \"ds_after_11\": \"%s\",\n  \"sr\": [", hexv(dsw).c_str());
        for (uint32_t i = 0; i < 12; i++)
            std::printf("%s\"%s\"", i ? "," : "", hexv(sr(s, ds, i)).c_str());
        std::printf("]");
        if (s != SuiteId::MmoAddQ) {
            // mmo / mdc2 over boundary lengths (AES suites only)
            std::printf(",\n  \"mmo\": [");
            int first = 1;
            for (size_t len : {1, 15, 16, 17, 31, 32, 48, 49, 64, 160, 200}) {
                Bytes mm = rbytes(len);
                auto h = mmo_hash(mm.data(), mm.size());
                auto h2 = mdc2_hash(mm.data(), mm.size());
                std::printf("%s[\"%s\",\"%s\",\"%s\"]", first ? "" : ",", hexv(mm).c_str(),
                            hexv(h).c_str(), hexv(h2).c_str());
                first = 0;
            }
            std::printf("]");
        }
        std::printf("\n},\n");
    }
    // scalar anchors
    std::printf("\"reduce_wide_be\": [");
    for (int t = 0; t < 64; t++) {
        Bytes w = rbytes(64);
        if (t == 0) std::memset(w.data(), 0xff, 64);
        if (t == 1) std::memset(w.data(), 0x00, 64);
        Scalar s = Scalar::reduce_wide_be(w.data(), 64);
        std::printf("%s[\"%s\",\"%s\"]", t ? "," : "", hexv(w).c_str(), hexv(s.le_bytes()).c_str());
    }
    std::printf("],\n\"scalar_add\": [");
    for (int t = 0; t < 32; t++) {
        Bytes w1 = rbytes(64), w2 = rbytes(64);
        Scalar a = Scalar::reduce_wide_be(w1.data(), 64), b = Scalar::reduce_wide_be(w2.data(), 64);
        std::printf("%s[\"%s\",\"%s\",\"%s\",\"%s\"]", t ? "," : "", hexv(a.le_bytes()).c_str(),
                    hexv(b.le_bytes()).c_str(), hexv(a.add(b).le_bytes()).c_str(),
                    hexv(a.mul(b).le_bytes()).c_str());
    }
    // group anchors
    std::printf("],\n\"generator\": \"%s\",\n", hexv(GroupElement::generator().bytes()).c_str());
    std::printf("\"exp_base\": [");
    for (int t = 0; t < 24; t++) {
        Bytes w = rbytes(64);
        Scalar s = Scalar::reduce_wide_be(w.data(), 64);
        if (t < 4) {
            uint8_t small[32] = {uint8_t(t)};
            s = Scalar::from_canonical_le(small);
        }
        std::printf("%s[\"%s\",\"%s\"]", t ? "," : "", hexv(s.le_bytes()).c_str(),
                    hexv(exp_base(s).bytes()).c_str());
    }
    std::printf("],\n\"commit_check\": [");
    for (int t = 0; t < 40; t++) {
        Bytes w1 = rbytes(64), w2 = rbytes(64), w3 = rbytes(64);
        Scalar y = Scalar::reduce_wide_be(w1.data(), 64);
        Scalar e = Scalar::reduce_wide_be(w2.data(), 64);
        Scalar s = Scalar::reduce_wide_be(w3.data(), 64);
        GroupElement Y = exp_base(y);
        if (t == 0) e = Scalar();
        if (t == 1) s = Scalar();
        if (t == 2) { e = Scalar(); s = Scalar(); }
        if (t == 3) Y = GroupElement::identity();
        if (t == 4) { s = Scalar().sub(e.mul(y)); }  // Y^e * a^s == identity
        GroupElement P = commit_check(Y, e, s);
        std::printf("%s[\"%s\",\"%s\",\"%s\",\"%s\"]", t ? "," : "", hexv(Y.bytes()).c_str(),
                    hexv(e.le_bytes()).c_str(), hexv(s.le_bytes()).c_str(), hexv(P.bytes()).c_str());
    }
    std::printf("],\n\"group_combine\": [");
    for (int t = 0; t < 24; t++) {
        Bytes w1 = rbytes(64), w2 = rbytes(64);
        GroupElement A = exp_base(Scalar::reduce_wide_be(w1.data(), 64));
        GroupElement B = exp_base(Scalar::reduce_wide_be(w2.data(), 64));
        if (t == 0) B = GroupElement::identity();
        if (t == 1) B = A;
        if (t == 2) B = exp_base(Scalar().sub(Scalar::reduce_wide_be(w1.data(), 64)));
        std::printf("%s[\"%s\",\"%s\",\"%s\"]", t ? "," : "", hexv(A.bytes()).c_str(),
                    hexv(B.bytes()).c_str(), hexv(group_combine(A, B).bytes()).c_str());
    }
    std::printf("],\n\"point_valid\": [");
    for (int t = 0; t < 48; t++) {
        Bytes p = rbytes(32);
        if (t % 3 == 0) {
            Bytes w = rbytes(64);
            auto e = exp_base(Scalar::reduce_wide_be(w.data(), 64)).bytes();
            p.assign(e.begin(), e.end());
            if (t % 6 == 3) p[0] ^= 1;  // odd/negative encodings are rejected
        }
        if (t == 1) p.assign(32, 0);
        if (t == 2) { p.assign(32, 0xff); p[31] = 0x7f; }
        bool ok = crypto_core_ristretto255_is_valid_point(p.data()) == 1;
        std::printf("%s[\"%s\",%d]", t ? "," : "", hexv(p).c_str(), ok ? 1 : 0);
    }
    std::printf("]\n}\n");
    return 0;
}

// ---- golden --------------------------------------------------------------
struct Stream {
    SuiteConfig suite;
    PoslocPublicKey pk;
    std::map<uint32_t, std::vector<Bytes>> msgs;
    std::vector<EpochSignature> sigs;
    Scalar s_hat;
    SeedStack ds;
};

void print_bits(const char* key, const std::vector<bool>& bits) {
    std::printf("\"%s\": [", key);
    for (size_t i = 0; i < bits.size(); i++) std::printf("%s%d", i ? "," : "", bits[i] ? 1 : 0);
    std::printf("]");
}

int cmd_golden(int argc, char** argv) {
    if (argc < 8) return 2;
    SuiteConfig suite{static_cast<SuiteId>(std::atoi(argv[2])), uint32_t(std::atoi(argv[3])),
                      uint32_t(std::atoi(argv[4])), uint32_t(std::atoi(argv[5]))};
    int len = std::atoi(argv[6]);
    uint64_t seed = std::strtoull(argv[7], nullptr, 0);
    std::vector<uint64_t> tampers;  // global entry indices to flip bit 0 of byte 0
    for (int a = 8; a < argc; a++) tampers.push_back(std::strtoull(argv[a], nullptr, 0));
    g_rb_state = seed;
    std::mt19937_64 rng(seed ^ 0xfeedULL);

    auto [sk, pk] = PoslocSecretKey::kg(suite);
    const Bytes sk_fresh = sk.serialize();  // before signing advances it
    Stream st{suite, pk, {}, {}, {}, SeedStack(suite.depth())};
    for (uint32_t i = 0; i < suite.n1; i++) {
        std::vector<Bytes> epoch;
        for (uint32_t j = 0; j < suite.n2; j++) {
            size_t l = len > 0 ? size_t(len) : 1 + rng() % (suite.suite == SuiteId::MmoAddQ ? 31 : 64);
            Bytes b(l);
            for (auto& x : b) x = uint8_t(rng());
            epoch.push_back(std::move(b));
        }
        st.sigs.push_back(sk.sig_epoch(epoch));
        st.s_hat = st.s_hat.add(st.sigs.back().s_hat);
        st.ds = st.sigs.back().ds;
        st.msgs.emplace(i, std::move(epoch));
    }
    for (uint64_t t : tampers) st.msgs.at(uint32_t(t / suite.n2))[t % suite.n2][0] ^= 0x01;

    std::printf("{\n\"suite\": %d, \"n1\": %u, \"n2\": %u, \"n_u\": %u, \"seed\": %llu,\n",
                int(suite.suite), suite.n1, suite.n2, suite.n_u, (unsigned long long)seed);
    std::printf("\"tampered_entries\": [");
    for (size_t k = 0; k < tampers.size(); k++)
        std::printf("%s%llu", k ? "," : "", (unsigned long long)tampers[k]);
    std::printf("],\n\"pk\": \"%s\",\n", hexv(st.pk.serialize()).c_str());
    std::printf("\"sk\": \"%s\",\n", hexv(sk_fresh).c_str());
    std::printf("\"sigs\": [");
    for (size_t i = 0; i < st.sigs.size(); i++)
        std::printf("%s\"%s\"", i ? "," : "", hexv(st.sigs[i].serialize()).c_str());
    std::printf("],\n\"entries\": [");
    bool first = true;
    for (auto& [i, v] : st.msgs)
        for (auto& m : v) { std::printf("%s\"%s\"", first ? "" : ",", hexv(m).c_str()); first = false; }
    Bytes dsw;
    st.ds.serialize(dsw);
    std::printf("],\n\"s_hat\": \"%s\", \"ds\": \"%s\",\n", hexv(st.s_hat.le_bytes()).c_str(),
                hexv(dsw).c_str());
    // agg_ekeys / aggregate_ekey / paver / aver (hot path)
    auto parts = agg_ekeys(st.suite, st.msgs, st.ds, 4);
    std::printf("\"e_tilde\": [");
    for (size_t k = 0; k < parts.size(); k++)
        std::printf("%s\"%s\"", k ? "," : "", hexv(parts[k].e.le_bytes()).c_str());
    Scalar e_hat = aggregate_ekey(st.suite, st.msgs, st.ds);
    std::printf("],\n\"e_hat\": \"%s\",\n", hexv(e_hat.le_bytes()).c_str());
    bool pv = paver(st.pk, st.msgs, st.s_hat, std::nullopt, st.ds, 4);
    bool av = aver(st.pk, st.msgs, st.s_hat, std::nullopt, st.ds);
    GroupElement r_agg;
    for (auto& [i, r] : st.pk.r_hats) r_agg = group_combine(r_agg, r);
    bool pv_agg = paver(st.pk, st.msgs, st.s_hat, r_agg, st.ds, 2);
    std::printf("\"r_hat_agg\": \"%s\", \"paver\": %d, \"aver\": %d, \"paver_agg\": %d,\n",
                hexv(r_agg.bytes()).c_str(), pv, av, pv_agg);
    // per-epoch verdicts (aver on each epoch with its own signature)
    std::vector<bool> per_epoch;
    for (uint32_t i = 0; i < suite.n1; i++)
        per_epoch.push_back(aver(st.pk, {{i, st.msgs.at(i)}}, st.sigs[i]));
    print_bits("epoch_verdicts", per_epoch);
    // distillation + SeBVer V/U/I (tamper localisation)
    ColdCryptoData ccd(CcdScheme::Coarse, suite);
    PoslocPublicKey pk2 = st.pk;
    for (uint32_t i = 0; i < suite.n1; i++) ccd.distill_epoch(pk2, st.msgs.at(i), st.sigs[i]);
    ccd.finalize();
    std::printf(",\n\"invalid_epochs\": [");
    for (size_t k = 0; k < ccd.invalid().size(); k++)
        std::printf("%s%u", k ? "," : "", ccd.invalid()[k].index);
    std::printf("],\n\"ccd\": \"%s\",\n", hexv(ccd.serialize()).c_str());
    if (ccd.has_valid()) {
        print_bits("sebver_V", ccd.sebver(st.pk.y, st.msgs, SebverMode::V));
        std::printf(",\n");
    }
    print_bits("sebver_U", ccd.sebver(st.pk.y, st.msgs, SebverMode::U));
    std::printf(",\n");
    print_bits("sebver_I", ccd.sebver(st.pk.y, st.msgs, SebverMode::I));
    std::printf("\n}\n");
    return 0;
}

// ---- golden_f (scheme F) ---------------------------------------------------
int cmd_golden_f(int argc, char** argv) {
    if (argc < 10) return 2;
    SuiteConfig suite{static_cast<SuiteId>(std::atoi(argv[2])), uint32_t(std::atoi(argv[3])),
                      uint32_t(std::atoi(argv[4])), uint32_t(std::atoi(argv[5]))};
    int len = std::atoi(argv[6]);
    uint64_t seed = std::strtoull(argv[7], nullptr, 0);
    uint32_t bv = uint32_t(std::atoi(argv[8])), bk = uint32_t(std::atoi(argv[9]));
    std::vector<uint64_t> tampers;
    for (int a = 10; a < argc; a++) tampers.push_back(std::strtoull(argv[a], nullptr, 0));
    g_rb_state = seed;
    std::mt19937_64 rng(seed ^ 0xf1f1ULL);
    auto [sk, pk] = PoslofSecretKey::kg(suite, bv, bk);
    std::map<uint32_t, std::vector<Bytes>> msgs;
    std::vector<FineSignature> sigs;
    for (uint32_t i = 0; i < suite.n1; i++) {
        std::vector<Bytes> epoch;
        for (uint32_t j = 0; j < suite.n2; j++) {
            size_t l = len > 0 ? size_t(len) : 1 + rng() % (suite.suite == SuiteId::MmoAddQ ? 31 : 64);
            Bytes b(l);
            for (auto& x : b) x = uint8_t(rng());
            sigs.push_back(sk.sig_one(b));
            epoch.push_back(std::move(b));
        }
        msgs.emplace(i, std::move(epoch));
    }
    for (uint64_t t : tampers) msgs.at(uint32_t(t / suite.n2))[t % suite.n2][0] ^= 0x01;
    std::printf("{\n\"scheme\": \"F\", \"suite\": %d, \"n1\": %u, \"n2\": %u, \"n_u\": %u, \"seed\": %llu,\n",
                int(suite.suite), suite.n1, suite.n2, suite.n_u, (unsigned long long)seed);
    std::printf("\"bpv\": [%u, %u], \"tampered_entries\": [", bv, bk);
    for (size_t k = 0; k < tampers.size(); k++)
        std::printf("%s%llu", k ? "," : "", (unsigned long long)tampers[k]);
    std::printf("],\n\"pk\": \"%s\",\n\"sigs\": [", hexv(pk.serialize()).c_str());
    for (size_t t = 0; t < sigs.size(); t++) std::printf("%s\"%s\"", t ? "," : "", hexv(sigs[t].serialize()).c_str());
    std::printf("],\n\"entries\": [");
    bool first = true;
    for (auto& [i, v] : msgs)
        for (auto& m : v) { std::printf("%s\"%s\"", first ? "" : ",", hexv(m).c_str()); first = false; }
    std::printf("],\n");
    // aver_f_single per entry (entries carrying ds raise FormatError: -1)
    std::printf("\"single\": [");
    for (size_t t = 0; t < sigs.size(); t++) {
        int v;
        try {
            v = aver_f_single(pk, msgs.at(uint32_t(t / suite.n2))[t % suite.n2], sigs[t]) ? 1 : 0;
        } catch (const FormatError&) {
            v = -1;
        }
        std::printf("%s%d", t ? "," : "", v);
    }
    // aver_f_batch over every entry and over every third entry, final ds
    const SeedStack& ds = std::get<SeedStack>(sigs.back().tail);
    Bytes dsw;
    ds.serialize(dsw);
    auto batch = [&](uint32_t stride, uint32_t off) {
        std::map<uint32_t, Bytes> ents;
        Scalar s;
        GroupElement r;
        for (uint32_t t = off; t < sigs.size(); t += stride) {
            ents.emplace(t, msgs.at(t / suite.n2)[t % suite.n2]);
            s = s.add(sigs[t].s);
            r = group_combine(r, sigs[t].r);
        }
        bool ok = aver_f_batch(pk, ents, s, r, ds);
        std::printf("{\"stride\": %u, \"offset\": %u, \"s\": \"%s\", \"r\": \"%s\", \"ok\": %d}", stride, off,
                    hexv(s.le_bytes()).c_str(), hexv(r.bytes()).c_str(), ok ? 1 : 0);
    };
    std::printf("],\n\"ds\": \"%s\",\n\"batch\": [", hexv(dsw).c_str());
    batch(1, 0);
    std::printf(", ");
    batch(3, 1);
    std::printf("],\n");
    // fine distillation + SeBVer
    ColdCryptoData ccd(CcdScheme::Fine, suite);
    for (uint32_t i = 0; i < suite.n1; i++) {
        std::vector<FineSignature> es(sigs.begin() + i * suite.n2, sigs.begin() + (i + 1) * suite.n2);
        ccd.distill_epoch_fine(pk, msgs.at(i), es);
    }
    ccd.finalize();
    std::printf("\"invalid_entries\": [");
    for (size_t k = 0; k < ccd.invalid().size(); k++) std::printf("%s%u", k ? "," : "", ccd.invalid()[k].index);
    std::printf("],\n\"ccd\": \"%s\",\n", hexv(ccd.serialize()).c_str());
    if (ccd.has_valid()) {
        print_bits("sebver_V", ccd.sebver(pk.y, msgs, SebverMode::V));
        std::printf(",\n");
    }
    print_bits("sebver_U", ccd.sebver(pk.y, msgs, SebverMode::U));
    std::printf(",\n");
    print_bits("sebver_I", ccd.sebver(pk.y, msgs, SebverMode::I));
    std::printf("\n}\n");
    return 0;
}

// ---- paver on a fixture file -----------------------------------------------
// "PVIO" u32 suite, n1, n2, n_u, entry_len, n_epochs, workers, ds_capacity (LE)
// u32 pk_len, pk (PoslocPublicKey wire), u32 ds_len, ds (SeedStack wire),
// s_hat (32 B LE), u8 has_agg, r_hat_agg (32 B), epochs (u32 LE x n_epochs),
// payload (n_epochs x n2 x entry_len bytes, epoch-major).
int cmd_paver(int argc, char** argv) {
    if (argc < 3) return 2;
    FILE* f = std::fopen(argv[2], "rb");
    if (!f) return 3;
    Bytes buf;
    uint8_t tmp[1 << 16];
    size_t got;
    while ((got = std::fread(tmp, 1, sizeof tmp, f)) > 0) buf.insert(buf.end(), tmp, tmp + got);
    std::fclose(f);
    size_t pos = 0;
    auto u32 = [&]() {
        uint32_t v;
        std::memcpy(&v, buf.data() + pos, 4);
        pos += 4;
        return v;
    };
    if (buf.size() < 4 || std::memcmp(buf.data(), "PVIO", 4) != 0) return 4;
    pos = 4;
    SuiteConfig suite{static_cast<SuiteId>(u32()), 0, 0, 0};
    suite.n1 = u32();
    suite.n2 = u32();
    suite.n_u = u32();
    const uint32_t len = u32(), n_ep = u32(), workers = u32(), cap = u32();
    const uint32_t pk_len = u32();
    PoslocPublicKey pk = PoslocPublicKey::deserialize(Bytes(buf.begin() + pos, buf.begin() + pos + pk_len));
    pos += pk_len;
    const uint32_t ds_len = u32();
    Reader rd(buf.data() + pos, ds_len);
    SeedStack ds = SeedStack::deserialize(rd, cap);
    pos += ds_len;
    Scalar s_hat = Scalar::from_canonical_le(buf.data() + pos);
    pos += 32;
    const bool has_agg = buf[pos++] != 0;
    std::optional<GroupElement> agg;
    if (has_agg) agg = GroupElement::from_bytes(buf.data() + pos);
    pos += 32;
    std::vector<uint32_t> eps(n_ep);
    for (auto& e : eps) e = u32();
    std::map<uint32_t, std::vector<Bytes>> batches;
    for (uint32_t k = 0; k < n_ep; k++) {
        std::vector<Bytes> ep;
        ep.reserve(suite.n2);
        for (uint32_t j = 0; j < suite.n2; j++, pos += len) ep.emplace_back(buf.begin() + pos, buf.begin() + pos + len);
        batches.emplace(eps[k], std::move(ep));
    }
    std::string error;
    int verdict = -1;
    Scalar e_hat;
    try {
        for (auto& p : agg_ekeys(suite, batches, ds, workers)) e_hat = e_hat.add(p.e);
        verdict = paver(pk, batches, s_hat, agg, ds, workers) ? 1 : 0;
    } catch (const std::exception& ex) {
        error = ex.what();
    }
    std::printf("{\"paver\": %d, \"error\": \"%s\", \"e_hat\": \"", verdict, error.c_str());
    for (uint8_t c : e_hat.le_bytes()) std::printf("%02x", c);
    std::printf("\"}\n");
    return 0;
}

// ---- bench ---------------------------------------------------------------
int cmd_bench(int argc, char** argv) {
    if (argc < 9) return 2;
    SuiteId sid = static_cast<SuiteId>(std::atoi(argv[2]));
    int log2n = std::atoi(argv[3]);
    uint32_t n2 = uint32_t(std::atoi(argv[4]));
    size_t len = size_t(std::atoi(argv[5]));
    unsigned workers = unsigned(std::atoi(argv[6]));
    uint64_t seed = std::strtoull(argv[7], nullptr, 0);
    int reps = std::atoi(argv[8]);
    std::string mode = argc > 9 ? argv[9] : "coarse";
    if (workers == 0) workers = std::max(1u, std::thread::hardware_concurrency());
    uint64_t n = uint64_t(1) << log2n;
    uint32_t n1 = uint32_t(n / n2);
    uint32_t n1p2 = 2;
    while (n1p2 < n1) n1p2 <<= 1;
    SuiteConfig suite{sid, n1p2, n2, std::min<uint32_t>(n1p2, 4)};
    g_rb_state = seed;

    using clock = std::chrono::steady_clock;
    auto t0 = clock::now();
    // Fixture (untimed): ds from the real `so` over a deterministic root, y and
    // per-epoch r random; R_i = a^{r_i}; s_i = r_i - e_i*y with e_i from the
    // reference agg_ekeys itself (SURVEY.md §8d "Fixtures at scale").
    SeedNode root{uint8_t(suite.depth()), 0, {}};
    rb_buf(root.value.data(), 16);
    SeedStack ds(suite.depth());
    for (uint32_t i = 0; i < n1; i++) so(sid, ds, root, i);
    std::map<uint32_t, std::vector<Bytes>> batches;
    for (uint32_t i = 0; i < n1; i++) {
        std::vector<Bytes> ep;
        ep.reserve(n2);
        for (uint32_t j = 0; j < n2; j++) {
            const uint64_t k = uint64_t(i) * n2 + j;
            if (len) {
                ep.push_back(synth_entry(seed, k, len));
            } else {  // LEN 0: the syslog-style log of BASELINE config 4 (bench.py --varlen)
                Bytes b(poslo_synth_varlen(seed, k));
                for (size_t t = 0; t < b.size(); t++) b[t] = poslo_synth_ascii(seed, k, uint32_t(t));
                ep.push_back(std::move(b));
            }
        }
        batches.emplace(i, std::move(ep));
    }
    Scalar y = Scalar::random();
    PoslocPublicKey pk;
    pk.suite = suite;
    pk.y = exp_base(y);
    auto parts = agg_ekeys(suite, batches, ds, workers);
    std::vector<EpochSignature> sigs(n1);
    Scalar s_hat;
    GroupElement r_hat;
    bool per_epoch = mode == "epoch";
    for (uint32_t i = 0; i < n1; i++) {
        Scalar r = Scalar::random();
        Scalar s = r.sub(parts[i].e.mul(y));
        s_hat = s_hat.add(s);
        if (per_epoch || i < 1) {
            GroupElement R = exp_base(r);
            pk.r_hats.emplace(i, R);
            r_hat = group_combine(r_hat, R);
        }
        sigs[i].s_hat = s;
        sigs[i].ds = ds;
    }
    if (!per_epoch) {  // one aggregate commitment for the whole sample
        s_hat = Scalar();
        for (uint32_t i = 0; i < n1; i++) s_hat = s_hat.add(sigs[i].s_hat);
        // rebuild: R = a^{sum r}: recover sum r = s_hat + e_hat*y
        Scalar e_hat;
        for (auto& p : parts) e_hat = e_hat.add(p.e);
        r_hat = exp_base(s_hat.add(e_hat.mul(y)));
    }
    double setup_s = std::chrono::duration<double>(clock::now() - t0).count();

    double best = 1e30, total = 0;
    int ok_all = 1;
    std::vector<double> times;
    for (int r = 0; r < reps; r++) {
        t0 = clock::now();
        bool ok;
        if (!per_epoch) {
            ok = paver(pk, batches, s_hat, r_hat, ds, workers);
        } else {
            // shipped per-epoch aver loop (acceptance.cpp:477-481 pattern),
            // sharded over `workers` threads (aver is pure)
            std::atomic<uint32_t> cur{0};
            std::atomic<int> bad{0};
            auto run = [&] {
                for (uint32_t i = cur.fetch_add(1); i < n1; i = cur.fetch_add(1))
                    if (!aver(pk, {{i, batches.at(i)}}, sigs[i].s_hat, std::nullopt, ds)) bad++;
            };
            std::vector<std::thread> pool;
            for (unsigned w = 0; w < workers; w++) pool.emplace_back(run);
            for (auto& t : pool) t.join();
            ok = bad.load() == 0;
        }
        double dt = std::chrono::duration<double>(clock::now() - t0).count();
        best = std::min(best, dt);
        total += dt;
        times.push_back(dt);
        ok_all &= ok ? 1 : 0;
    }
    std::printf("{\"entries\": %llu, \"n1\": %u, \"n2\": %u, \"entry_len\": %zu, \"suite\": %d, "
                "\"workers\": %u, \"mode\": \"%s\", \"reps\": %d, \"setup_s\": %.3f, "
                "\"best_s\": %.6f, \"mean_s\": %.6f, \"eps_best\": %.1f, \"eps_mean\": %.1f, "
                "\"verdict\": %d, \"times\": [",
                (unsigned long long)n, n1, n2, len, int(sid), workers, mode.c_str(), reps, setup_s,
                best, total / reps, double(n) / best, double(n) * reps / total, ok_all);
    for (size_t i = 0; i < times.size(); i++) std::printf("%s%.6f", i ? "," : "", times[i]);
    std::printf("]}\n");
    return 0;
}

}  // namespace

int main(int argc, char** argv) {
    randombytes_set_implementation(&g_rb_impl);
    if (sodium_init() < 0) return 3;
    if (argc < 2) {
        std::fprintf(stderr, "usage: ref_tool kat|golden|golden_f|paver|bench ...\n");
        return 2;
    }
    std::string cmd = argv[1];
    try {
        if (cmd == "kat") return cmd_kat();
        if (cmd == "golden") return cmd_golden(argc, argv);
        if (cmd == "golden_f") return cmd_golden_f(argc, argv);
        if (cmd == "bench") return cmd_bench(argc, argv);
        if (cmd == "paver") return cmd_paver(argc, argv);
    } catch (std::exception& e) {
        std::fprintf(stderr, "ref_tool: %s\n", e.what());
        return 1;
    }
    return 2;
}
