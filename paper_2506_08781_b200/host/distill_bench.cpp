// Times the C++ distiller drop-in (distiller_gpu.cpp, linked through
// libposlo_dropin.so) the way the reference's callers drive it: one
// ColdCryptoData::distill_epoch per epoch of a signed stream
// (proj/src/distiller.cpp:60-89), then SeBVer V / U / I over the finished CCD
// (:181-233). The stream comes from the reference's own signer (kg /
// sig_epoch, CPU), with `tamper` epochs corrupted after signing.
//
//   distill_bench <n1> <n2> <n_u> <entry_len> <tamper epochs> [reps]
//
// Prints one JSON line: per-epoch distill latency (mean / best over the
// stream), SeBVer times, and the CCD outcome (invalid list size, V/U/I bits).
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>

#include "poslo/distiller.hpp"
#include "poslo/poslo_c.hpp"

using namespace poslo;
using clk = std::chrono::steady_clock;

static double ms_since(clk::time_point t0) { return std::chrono::duration<double, std::milli>(clk::now() - t0).count(); }

int main(int argc, char** argv) {
    if (argc < 6) {
        std::fprintf(stderr, "usage: %s n1 n2 n_u entry_len tamper_epochs [reps]\n", argv[0]);
        return 1;
    }
    const uint32_t n1 = (uint32_t)std::atoi(argv[1]), n2 = (uint32_t)std::atoi(argv[2]);
    const uint32_t n_u = (uint32_t)std::atoi(argv[3]), L = (uint32_t)std::atoi(argv[4]);
    const uint32_t n_bad = (uint32_t)std::atoi(argv[5]);
    const int reps = argc > 6 ? std::atoi(argv[6]) : 2;
    SuiteConfig suite{SuiteId::Sha256, n1, n2, n_u};
    auto t0 = clk::now();
    auto [sk, pk0] = PoslocSecretKey::kg(suite);
    std::map<uint32_t, std::vector<Bytes>> msgs;
    std::vector<EpochSignature> sigs;
    for (uint32_t i = 0; i < n1; i++) {
        std::vector<Bytes> ep(n2, Bytes(L));
        for (uint32_t j = 0; j < n2; j++)
            for (uint32_t b = 0; b < L; b++) ep[j][b] = (uint8_t)(i * 131 + j * 7 + b);
        sigs.push_back(sk.sig_epoch(ep));
        msgs.emplace(i, std::move(ep));
    }
    for (uint32_t k = 0; k < n_bad; k++) msgs[(k * 2654435761u) % n1][k % n2][0] ^= 1;  // after signing
    const double sign_ms = ms_since(t0);

    double best = 1e30, mean_sum = 0, first_ms = 0;
    size_t n_invalid = 0;
    double v_ms = 0, u_ms = 0, i_ms = 0;
    bool v_ok = false;
    size_t u_true = 0, i_true = 0;
    for (int r = 0; r < reps; r++) {
        PoslocPublicKey pk = pk0;
        ColdCryptoData ccd(CcdScheme::Coarse, suite);
        auto t1 = clk::now();
        for (uint32_t i = 0; i < n1; i++) {
            auto te = clk::now();
            ccd.distill_epoch(pk, msgs.at(i), sigs[i]);
            if (r == 0 && i == 0) first_ms = ms_since(te);
        }
        const double per = ms_since(t1) / n1;
        best = std::min(best, per);
        if (r > 0 || reps == 1) mean_sum += per;  // rep 0 carries context creation and table builds
        n_invalid = ccd.invalid().size();
        auto ts = clk::now();
        auto V = ccd.sebver(pk0.y, msgs, SebverMode::V);
        v_ms = ms_since(ts);
        ts = clk::now();
        auto U = ccd.sebver(pk0.y, msgs, SebverMode::U);
        u_ms = ms_since(ts);
        ts = clk::now();
        auto I = ccd.sebver(pk0.y, msgs, SebverMode::I);
        i_ms = ms_since(ts);
        v_ok = !V.empty() && V[0];
        u_true = std::count(U.begin(), U.end(), true);
        i_true = std::count(I.begin(), I.end(), true);
    }
    std::printf(
        "{\"n1\": %u, \"n2\": %u, \"n_u\": %u, \"entry_len\": %u, \"tampered_epochs\": %u, \"reps\": %d, "
        "\"sign_ms\": %.1f, \"first_epoch_ms\": %.3f, \"distill_ms_per_epoch_best\": %.4f, "
        "\"distill_ms_per_epoch_warm_mean\": %.4f, \"invalid\": %zu, \"sebver_v_ms\": %.3f, \"sebver_u_ms\": %.3f, "
        "\"sebver_i_ms\": %.3f, \"V\": %s, \"U_true\": %zu, \"I_true\": %zu}\n",
        n1, n2, n_u, L, n_bad, reps, sign_ms, first_ms, best, mean_sum / (reps > 1 ? reps - 1 : 1), n_invalid, v_ms, u_ms, i_ms,
        v_ok ? "true" : "false", u_true, i_true);
    return 0;
}
