// Times the C++ drop-in poslo::paver / poslo::agg_ekeys (batch_verify_gpu.cpp,
// linked through libposlo_dropin.so) on the reference's own input type, a
// std::map<uint32_t, std::vector<Bytes>> of per-entry heap vectors — the path
// the reference CLI takes (proj/tools/poslo.cpp:193-205, 252-254). bench.py
// reports it as `e2e_dropin`.
//
//   dropin_bench <suite> <log2 entries> <n2> <entry_len> <reps> <workers> [seed]
//
// Fixture: the synthetic log of include/poslo_synth.h; keys and signatures by
// the reference's kg / sig_epoch derivation on the device (C-ABI signer):
// R-hat_i = alpha^(sum_j nonce_to_scalar(r, i, j)), s-hat_i = r-hat_i - y e~_i,
// the coarse aggregate (sum s-hat, group_combine fold of R-hat). A second key
// y' over the same commitments gives the fresh-Y call (its comb tables are not
// yet built). Prints one JSON line.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <random>
#include <thread>
#include <vector>

#include "../../include/poslo_synth.h"
#include "poslo/batch_verify.hpp"
#include "poslo/poslo_c.hpp"
#include "poslo_gpu.h"

using namespace poslo;
using clk = std::chrono::steady_clock;

extern "C" void poslo_dropin_last_stats(double out[4]);

// f(t, T) on T host threads
template <class F>
static void on_threads(unsigned T, F f) {
    std::vector<std::thread> th;
    for (unsigned t = 0; t < T; t++) th.emplace_back([&, t] { f(t, T); });
    for (auto& x : th) x.join();
}

static double ms_since(clk::time_point t0) { return std::chrono::duration<double, std::milli>(clk::now() - t0).count(); }

static void die(const char* what, const poslo_error& e) {
    std::fprintf(stderr, "%s: %s\n", what, e.message);
    std::exit(2);
}

int main(int argc, char** argv) {
    if (argc < 7) {
        std::fprintf(stderr, "usage: %s suite log2n n2 entry_len reps workers [seed]\n", argv[0]);
        return 1;
    }
    const int suite_no = std::atoi(argv[1]);
    const uint64_t n = 1ull << std::atoi(argv[2]);
    const uint32_t n2 = (uint32_t)std::atoi(argv[3]);
    const uint32_t L = (uint32_t)std::atoi(argv[4]);
    const int reps = std::atoi(argv[5]);
    const unsigned workers = (unsigned)std::atoi(argv[6]);
    const uint64_t seed = argc > 7 ? std::strtoull(argv[7], nullptr, 0) : 0x5EED;
    const uint32_t n1 = (uint32_t)(n / n2);
    uint32_t D = 0;
    while ((1u << D) < n1) D++;

    auto t_build = clk::now();
    // the reference's input: one heap vector per entry
    std::map<uint32_t, std::vector<Bytes>> batches;
    for (uint32_t i = 0; i < n1; i++) {
        std::vector<Bytes> v(n2, Bytes(L));
        for (uint32_t j = 0; j < n2; j++) {
            const uint64_t k = (uint64_t)i * n2 + j;
            for (uint32_t b = 0; b < L; b += 8) {
                const uint64_t w = poslo_synth_word(seed, k, b >> 3);
                std::memcpy(v[j].data() + b, &w, std::min<uint32_t>(8, L - b));
            }
        }
        batches.emplace(i, std::move(v));
    }
    const double build_ms = ms_since(t_build);

    // keys and signatures on the device (C-ABI signer), contiguous copy of the log
    std::mt19937_64 rng(seed);
    auto rand_scalar = [&] {
        uint8_t b[32];
        for (auto& x : b) x = (uint8_t)rng();
        b[31] &= 0x0f;  // < 2^252 < l
        return Scalar::from_canonical_le(b);
    };
    const Scalar y = rand_scalar(), y2 = rand_scalar();
    uint8_t r_seed[16], root[16];
    for (auto& x : r_seed) x = (uint8_t)rng();
    for (auto& x : root) x = (uint8_t)rng();
    SeedStack ds(D);
    SeedNode node;
    node.depth = (uint8_t)D;
    node.index = 0;
    std::memcpy(node.value.data(), root, 16);
    ds.push(node);
    Bytes dsw;
    ds.serialize(dsw);

    poslo_gpu_ctx* ctx = nullptr;
    poslo_error err{};
    if (poslo_gpu_create(0, &ctx, &err)) die("create", err);
    std::vector<uint8_t> flat((size_t)n * L);
    for (const auto& [i, v] : batches)
        for (uint32_t j = 0; j < n2; j++) std::memcpy(&flat[((size_t)i * n2 + j) * L], v[j].data(), L);
    std::vector<uint32_t> epochs(n1);
    for (uint32_t i = 0; i < n1; i++) epochs[i] = i;
    poslo_batch b{};
    b.suite = (uint8_t)suite_no;
    b.n2 = n2;
    b.payload = flat.data();
    b.payload_bytes = flat.size();
    b.entry_len = L;
    b.n_entries = n;
    b.epochs = epochs.data();
    b.n_epochs = n1;
    b.ds = dsw.data();
    b.ds_len = (uint32_t)dsw.size();
    b.ds_capacity = D;
    std::vector<uint8_t> r_hats((size_t)n1 * 32), s1((size_t)n1 * 32), s2((size_t)n1 * 32);
    if (poslo_gpu_kg_commitments(ctx, (uint8_t)suite_no, r_seed, epochs.data(), n1, n2, r_hats.data(), nullptr, &err))
        die("kg", err);
    if (poslo_gpu_sig_epochs(ctx, &b, r_seed, y.le_bytes().data(), s1.data(), &err)) die("sig", err);
    if (poslo_gpu_sig_epochs(ctx, &b, r_seed, y2.le_bytes().data(), s2.data(), &err)) die("sig2", err);
    uint8_t S1[32], S2[32], R[32];
    if (poslo_gpu_scalar_sum(ctx, n1, s1.data(), S1, &err) || poslo_gpu_scalar_sum(ctx, n1, s2.data(), S2, &err) ||
        poslo_gpu_group_fold(ctx, n1, r_hats.data(), R, &err))
        die("fold", err);
    poslo_gpu_destroy(ctx);
    flat.clear();
    flat.shrink_to_fit();

    PoslocPublicKey pk, pk2;
    pk.suite = SuiteConfig{(SuiteId)suite_no, n1, n2, 1};
    pk.y = exp_base(y);
    pk2.suite = pk.suite;
    pk2.y = exp_base(y2);
    for (uint32_t i = 0; i < n1; i++) {
        pk.r_hats.emplace(i, GroupElement::from_bytes(&r_hats[32 * (size_t)i]));
    }
    pk2.r_hats = pk.r_hats;
    const Scalar s_hat = Scalar::from_canonical_le(S1), s_hat2 = Scalar::from_canonical_le(S2);
    const GroupElement r_agg = GroupElement::from_bytes(R);

    // first call of the process: CUDA context, module load, generator and Y tables
    auto t0 = clk::now();
    const bool ok_first = paver(pk, batches, s_hat, r_agg, ds, workers);
    const double first_ms = ms_since(t0);
    // warm calls, aggregate R-hat given (the CLI's verify V, tools/poslo.cpp:204-205)
    std::vector<double> warm;
    bool ok_warm = true;
    for (int r = 0; r < reps; r++) {
        t0 = clk::now();
        ok_warm = ok_warm && paver(pk, batches, s_hat, r_agg, ds, workers);
        warm.push_back(ms_since(t0));
    }
    // a fresh Y on the warm process (its comb tables are built in this call)
    t0 = clk::now();
    const bool ok_fresh = paver(pk2, batches, s_hat2, r_agg, ds, workers);
    const double fresh_ms = ms_since(t0);
    // R-hat folded from pk.r_hats (the CLI's bench path, :252-254)
    t0 = clk::now();
    const bool ok_fold = paver(pk, batches, s_hat, std::nullopt, ds, workers);
    const double fold_ms = ms_since(t0);
    // agg_ekeys (per-epoch e~ back to the host)
    t0 = clk::now();
    auto parts = agg_ekeys(pk.suite, batches, ds, workers);
    const double agg_ms = ms_since(t0);
    // a tampered entry must be rejected
    batches[n1 / 2][n2 / 3][0] ^= 1;
    const bool ok_tamper = paver(pk, batches, s_hat, r_agg, ds, workers);
    batches[n1 / 2][n2 / 3][0] ^= 1;

    double st[4];
    poslo_dropin_last_stats(st);  // the tamper call: same shape as a warm call

    // Host roofline of the drop-in: (a) a plain parallel memcpy of the same
    // bytes between two contiguous buffers, (b) a parallel gather of the
    // std::map into one contiguous buffer with no device work; best of 3,
    // every host thread.
    const unsigned T = std::max(1u, std::thread::hardware_concurrency());
    const size_t bytes = (size_t)n * L;
    std::vector<uint8_t> src(bytes, 1), dst(bytes, 0);
    double copy_ms = 1e30, gather_ms = 1e30;
    for (int r = 0; r < 3; r++) {
        auto t1 = clk::now();
        on_threads(T, [&](unsigned t, unsigned TT) {
            const size_t a = bytes * t / TT, z = bytes * (t + 1) / TT;
            std::memcpy(dst.data() + a, src.data() + a, z - a);
        });
        copy_ms = std::min(copy_ms, ms_since(t1));
    }
    std::vector<const std::vector<Bytes>*> eps;
    for (const auto& [i, v] : batches) eps.push_back(&v);
    for (int r = 0; r < 3; r++) {
        auto t1 = clk::now();
        on_threads(T, [&](unsigned t, unsigned TT) {
            const size_t a = eps.size() * t / TT, z = eps.size() * (t + 1) / TT;
            for (size_t k = a; k < z; k++) {
                uint8_t* d = dst.data() + k * (size_t)n2 * L;
                for (const Bytes& m : *eps[k]) {
                    std::memcpy(d, m.data(), L);
                    d += L;
                }
            }
        });
        gather_ms = std::min(gather_ms, ms_since(t1));
    }

    double best = 1e30, sum = 0;
    for (double w : warm) {
        best = std::min(best, w);
        sum += w;
    }
    const double mean = warm.empty() ? 0 : sum / warm.size();
    std::printf(
        "{\"entries\": %llu, \"n2\": %u, \"entry_len\": %u, \"suite\": %d, \"workers\": %u, \"gpus\": %d, "
        "\"build_map_ms\": %.1f, \"first_call_ms\": %.3f, \"warm_ms\": [%s], \"warm_best_ms\": %.3f, "
        "\"warm_mean_ms\": %.3f, \"fresh_y_ms\": %.3f, \"fold_rhat_ms\": %.3f, \"agg_ekeys_ms\": %.3f, "
        "\"eps_warm_best\": %.1f, \"eps_warm_mean\": %.1f, \"ok\": %s, \"tamper_rejected\": %s, "
        "\"n_parts\": %zu, \"host_threads\": %u, \"host_copy_ms\": %.3f, \"host_copy_gbs\": %.2f, "
        "\"host_gather_ms\": %.3f, \"last_call\": {\"pack_ms\": %.3f, \"fill_ms\": %.3f, \"call_ms\": %.3f}}\n",
        (unsigned long long)n, n2, L, suite_no, workers, poslo_gpu_device_count(), build_ms, first_ms,
        [&] {
            static char buf[4096];
            buf[0] = 0;
            for (size_t k = 0; k < warm.size(); k++)
                std::snprintf(buf + std::strlen(buf), sizeof buf - std::strlen(buf), "%s%.3f", k ? ", " : "", warm[k]);
            return buf;
        }(),
        best, mean, fresh_ms, fold_ms, agg_ms, n / (best * 1e-3), n / (mean * 1e-3),
        (ok_first && ok_warm && ok_fresh && ok_fold) ? "true" : "false", ok_tamper ? "false" : "true", parts.size(),
        T, copy_ms, bytes / (copy_ms * 1e6), gather_ms, st[0], st[1], st[2]);
    return 0;
}
