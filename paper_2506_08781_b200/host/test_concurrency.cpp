// Re-entrancy check for the C++ drop-in (SURVEY.md §8b "Threading": agg_ekeys
// "may be called concurrently from many host threads"). Several host threads
// call poslo::agg_ekeys (batch_verify_gpu.cpp, one device context per
// thread) at once on different suites, shapes and ragged entries, and every
// per-epoch aggregate is compared with the reference's own sequential
// poslo::aggregate_ekey (src/poslo_c.cpp:177-190, CPU) on the same epoch.
// Links libposlo_dropin.so (reference objects + the drop-ins).
#include <atomic>
#include <cstdio>
#include <random>
#include <thread>
#include <vector>

#include "poslo/batch_verify.hpp"
#include "poslo/poslo_c.hpp"

using namespace poslo;

int main() {
    const int kThreads = 6, kIters = 3;
    std::atomic<int> bad{0}, epochs{0};
    auto worker = [&](int t) {
        std::mt19937_64 rng(1000 + t);
        for (int it = 0; it < kIters; it++) {
            const SuiteId sid = (t + it) % 2 ? SuiteId::MmoMdc2 : SuiteId::Sha256;
            SuiteConfig suite{sid, 64, uint32_t(24 + 8 * t + it), 4};
            SeedStack ds(suite.depth());
            SeedNode root{uint8_t(suite.depth()), 0, {}};
            for (auto& b : root.value) b = uint8_t(rng());
            ds.push(root);
            std::map<uint32_t, std::vector<Bytes>> batches;
            for (uint32_t i = 0; i < suite.n1; i++) {
                if (rng() % 3 == 0) continue;  // sparse epoch query
                std::vector<Bytes> ep(suite.n2);
                for (auto& m : ep) {
                    m.resize(rng() % 200);
                    for (auto& b : m) b = uint8_t(rng());
                }
                batches.emplace(i, std::move(ep));
            }
            const auto parts = agg_ekeys(suite, batches, ds, unsigned(1 + t));
            if (parts.size() != batches.size()) {
                bad++;
                continue;
            }
            size_t k = 0;
            for (const auto& [i, msgs] : batches) {
                const Scalar ref = aggregate_ekey(suite, {{i, msgs}}, ds);
                if (parts[k].epoch != i || !(parts[k].e == ref)) bad++;
                k++;
                epochs++;
            }
        }
    };
    std::vector<std::thread> pool;
    for (int t = 0; t < kThreads; t++) pool.emplace_back(worker, t);
    for (auto& th : pool) th.join();
    std::printf("threads %d, calls %d, epochs compared %d, mismatches %d\n", kThreads, kThreads * kIters,
                epochs.load(), bad.load());
    return bad.load() == 0 && epochs.load() > 0 ? 0 : 1;
}
