// CPU harness over the device math headers (paper_2506_08781_b200/csrc/*.cuh)
// compiled as plain C++: lets tests/test_devmath_host.py pin the kernels'
// arithmetic (SHA-256/AES/MMO/MDC-2 per-entry paths, deferred mod-l
// reduction, ristretto255) against the reference's golden vectors without a
// GPU. Test infrastructure only — the product never runs this code on a CPU.
#include <cstring>
#include <vector>

#include "../../paper_2506_08781_b200/csrc/entry_hash.cuh"
#include "../../paper_2506_08781_b200/csrc/ristretto.cuh"
#include "../../paper_2506_08781_b200/csrc/scalar.cuh"

using namespace poslo_gpu;

namespace {
struct HostT0 {
    uint32_t t[256];
    HostT0() {
        for (int x = 0; x < 256; x++) t[x] = aes_t0_entry(aes_sbox_compute(x));
    }
    uint32_t operator()(uint32_t x) const { return t[x]; }
    uint32_t lk(uint32_t w, int k) const { return t[(w >> (8 * k)) & 0xffu]; }
    uint32_t lkr(uint32_t w, int k, int r) const { return rotl32(lk(w, k), 8 * r); }
};
const HostT0& T0() {
    static HostT0 t;
    return t;
}
void words_le(const uint8_t* b, uint32_t* w, int n) {
    for (int i = 0; i < n; i++) w[i] = b[4 * i] | b[4 * i + 1] << 8 | b[4 * i + 2] << 16 | (uint32_t)b[4 * i + 3] << 24;
}
void le_words_out(const uint32_t* w, uint8_t* b, int n) {
    for (int i = 0; i < n; i++)
        for (int k = 0; k < 4; k++) b[4 * i + k] = (uint8_t)(w[i] >> (8 * k));
}
}  // namespace

extern "C" {

// prf (seed tree step)
void dm_prf(int suite, int bit, const uint8_t x[16], uint8_t out[16]) {
    uint32_t w[4];
    words_le(x, w, 4);
    prf_dev(suite, T0(), w, bit);
    le_words_out(w, out, 4);
}

// e = hash_to_scalar(m, onetime_seed(x0, j)) mod l via the generic path;
// returns 0, or 1 for FormatError
int dm_entry_generic(int suite, const uint8_t* m, uint32_t L, const uint8_t x0[16], uint32_t j,
                     uint8_t e_out[32], uint32_t limbs_out[16]) {
    uint32_t x0m[4], limbs[16], e[8];
    words_le(x0, x0m, 4);
    if (!entry_limbs(suite, T0(), m, L, x0m, j, limbs)) return 1;
    sc_reduce_limbs(limbs, 16, e);
    le_words_out(e, e_out, 8);
    if (limbs_out) std::memcpy(limbs_out, limbs, 64);
    return 0;
}

// the 32-byte fast paths (suite 1 / suite 2)
void dm_entry_fast32(int suite, const uint8_t m[32], const uint8_t x0[16], uint32_t j,
                     uint32_t limbs_out[16]) {
    uint32_t x0m[4], mm[8];
    words_le(x0, x0m, 4);
    words_le(m, mm, 8);
    if (suite == 1) {
        uint32_t x0w[4], mw[8], pre[8];
        for (int k = 0; k < 4; k++) x0w[k] = bswap32(x0m[k]);
        for (int k = 0; k < 8; k++) mw[k] = bswap32(mm[k]);
        ots_pre(x0w, pre);
        entry_limbs_s1_l32(x0w, pre, j, mw, limbs_out);
    } else {
        uint32_t hpre[4] = {MMO_IV_WORD, MMO_IV_WORD, MMO_IV_WORD, MMO_IV_WORD};
        mmo_step(T0(), hpre, x0m);
        entry_limbs_s2_l32(T0(), hpre, j, mm, limbs_out);
    }
}

// the pipe-balanced SHA variants (MODE 1/2) with one = 1: exercises the
// constant/zero word masks of sha256_rounds on the CPU
void dm_entry_s1_mode(int mode, const uint8_t m[32], const uint8_t x0[16], uint32_t j,
                      uint32_t limbs_out[16]) {
    uint32_t x0m[4], mm[8], x0w[4], mw[8], pre[8];
    words_le(x0, x0m, 4);
    words_le(m, mm, 8);
    for (int k = 0; k < 4; k++) x0w[k] = bswap32(x0m[k]);
    for (int k = 0; k < 8; k++) mw[k] = bswap32(mm[k]);
    ots_pre(x0w, pre);
    if (mode >= 3)
        (mode == 3 ? entry_limbs_s1_l32_compact<0>
         : mode == 4 ? entry_limbs_s1_l32_compact<1>
         : mode == 5 ? entry_limbs_s1_l32_compact<2>
         : mode == 6 ? entry_limbs_s1_l32_compact<3>
                     : entry_limbs_s1_l32_compact<4>)(
            x0w, pre, j, mw, limbs_out, pipek_make());
    else if (mode == 1)
        entry_limbs_s1_l32<1>(x0w, pre, j, mw, limbs_out, 1u);
    else if (mode == 2)
        entry_limbs_s1_l32<2>(x0w, pre, j, mw, limbs_out, 1u);
    else
        entry_limbs_s1_l32<0>(x0w, pre, j, mw, limbs_out, 1u);
}

// onetime_seed through the specialised schedule of the lean kernel
// (ots_epoch_consts + ots_head_rounds + sha256_rounds_loop from round 32)
void dm_ots_spec(const uint8_t x0[16], uint32_t j, uint8_t out[16]) {
    uint32_t x0m[4], x0w[4], st[8], W[16];
    words_le(x0, x0m, 4);
    for (int k = 0; k < 4; k++) x0w[k] = bswap32(x0m[k]);
    ots_pre(x0w, st);
    const OtsEpoch E = ots_epoch_consts(x0w);
    const PipeK pk = pipek_make();
    ots_head_rounds<2>(st, W, j, E, pk);
    sha256_rounds_loop<2>(st, W, 32, pk);
    const uint32_t iv[4] = {SHA_IV0, SHA_IV1, SHA_IV2, SHA_IV3};
    for (int k = 0; k < 4; k++) {
        uint32_t v = st[k] + iv[k];
        out[4 * k] = v >> 24; out[4 * k + 1] = v >> 16; out[4 * k + 2] = v >> 8; out[4 * k + 3] = v;
    }
}

// signer side: r-hat_i = sum_j nonce_to_scalar(r, i, j) mod l (kg, poslo_c.cpp:104-110)
void dm_nonce_sum(int suite, const uint8_t r[16], uint32_t i, uint32_t n2, uint8_t out[32]) {
    uint32_t rm[4], acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    words_le(r, rm, 4);
    for (uint32_t j = 0; j < n2; j++) {
        uint32_t s[8];
        nonce_scalar(suite, T0(), rm, i, j, s);
        sc_add(acc, s, acc);
    }
    le_words_out(acc, out, 8);
}

void dm_sc_mul_sub(const uint8_t r[32], const uint8_t y[32], const uint8_t e[32], uint8_t out[32]) {
    uint32_t rr[8], yy[8], ee[8], p[8], o[8];
    words_le(r, rr, 8);
    words_le(y, yy, 8);
    words_le(e, ee, 8);
    sc_mul(yy, ee, p);
    sc_sub(rr, p, o);
    le_words_out(o, out, 8);
}

// field ops through the byte interface: op 0 mul, 1 sq, 2 add, 3 sub, 4 neg, 5 canon (a only)
void dm_fe_op(int op, const uint8_t a[32], const uint8_t b[32], uint8_t out[32]) {
    const fe x = fe_from_bytes_le(a), y = fe_from_bytes_le(b);
    fe r;
    switch (op) {
        case 0: r = fe_mul(x, y); break;
        case 1: r = fe_sq(x); break;
        case 2: r = fe_add(x, y); break;
        case 3: r = fe_sub(x, y); break;
        case 4: r = fe_neg(x); break;
        default: r = x; break;
    }
    fe_to_bytes_le(r, out);
}

// a long chain of mixed operations (limb bounds under repeated lazy use)
void dm_fe_chain(const uint8_t a[32], const uint8_t b[32], int n, uint8_t out[32]) {
    fe x = fe_from_bytes_le(a), y = fe_from_bytes_le(b);
    for (int i = 0; i < n; i++) {
        fe s = fe_add(x, y), d = fe_sub(x, y);
        x = fe_mul(s, d);
        y = fe_sq(fe_sub(y, fe_add(s, s)));
    }
    fe_to_bytes_le(fe_add(x, y), out);
}

// sum of n 16-limb values via the 17-limb accumulator, reduced mod l
void dm_sum_reduce(const uint32_t* limbs16, uint32_t n, uint8_t e_out[32]) {
    uint32_t acc[17];
    acc17_zero(acc);
    for (uint32_t i = 0; i < n; i++) acc17_add16(acc, limbs16 + 16 * i);
    uint32_t e[8];
    sc_reduce_limbs(acc, 17, e);
    le_words_out(e, e_out, 8);
}

void dm_reduce_wide_be(const uint8_t in[64], uint8_t out[32]) {
    uint32_t limbs[16];
    for (int k = 0; k < 16; k++) limbs[15 - k] = load_be32p(in + 4 * k);
    uint32_t e[8];
    sc_reduce_limbs(limbs, 16, e);
    le_words_out(e, out, 8);
}

void dm_sc_add(const uint8_t a[32], const uint8_t b[32], uint8_t out[32]) {
    uint32_t x[8], y[8], r[8];
    words_le(a, x, 8);
    words_le(b, y, 8);
    sc_add(x, y, r);
    le_words_out(r, out, 8);
}

int dm_point_valid(const uint8_t p[32]) {
    gpt P;
    return rist_decode(p, P) ? 1 : 0;
}

int dm_commit_check(const uint8_t y[32], const uint8_t e[32], const uint8_t s[32], uint8_t out[32]) {
    gpt Y;
    if (!rist_decode(y, Y)) return 1;
    uint32_t ee[8], ss[8];
    words_le(e, ee, 8);
    words_le(s, ss, 8);
    commit_check_enc(Y, ee, ss, out);
    return 0;
}

// the comb-table path of stage 3 v2 (tables built exactly as the device does)
static void host_table(const gpt& P0, std::vector<gcached>& tab) {
    gpt P = P0;
    tab.resize(512);
    for (int k = 0; k < 64; k++) {
        gpt q = P;
        for (int i = 0; i < 8; i++) {
            tab[8 * k + i] = pt_to_cached(q);
            q = pt_add(q, P);
        }
        P = pt_dbl(pt_dbl(pt_dbl(pt_dbl(P))));
    }
}

int dm_commit_check_comb(const uint8_t y[32], const uint8_t e[32], const uint8_t s[32], uint8_t out[32]) {
    gpt Y;
    if (!rist_decode(y, Y)) return 1;
    std::vector<gcached> ty, tb;
    host_table(Y, ty);
    host_table(pt_base(), tb);
    uint32_t ee[8], ss[8];
    words_le(e, ee, 8);
    words_le(s, ss, 8);
    int8_t d[64];
    gpt acc = pt_identity();
    sc_signed_radix16(ee, d);
    acc = comb_mul_add(acc, ty.data(), d);
    sc_signed_radix16(ss, d);
    acc = comb_mul_add(acc, tb.data(), d);
    rist_encode(acc, out);
    return 0;
}

// split check used by paver: e*Y == R - s*B, compared with rist_equal
int dm_check_split(const uint8_t y[32], const uint8_t e[32], const uint8_t s[32], const uint8_t r[32]) {
    gpt Y, R;
    if (!rist_decode(y, Y)) return -1;
    if (!rist_decode(r, R)) return 0;
    std::vector<gcached> ty, tb;
    host_table(Y, ty);
    host_table(pt_base(), tb);
    uint32_t ee[8], ss[8];
    words_le(e, ee, 8);
    words_le(s, ss, 8);
    int8_t d[64];
    sc_signed_radix16(ss, d);
    gpt S = comb_mul_add(pt_identity(), tb.data(), d);
    gpt T = pt_add(R, pt_neg(S));
    sc_signed_radix16(ee, d);
    gpt E = comb_mul_add(pt_identity(), ty.data(), d);
    return rist_equal(E, T) ? 1 : 0;
}

// the square-root-free verdict of the per-epoch checks (rist_encoding_matches)
// on P = e Y + s B, with 1 / u2 from fe_invert (the device batches it)
int dm_check_sqrtfree(const uint8_t y[32], const uint8_t e[32], const uint8_t s[32], const uint8_t r[32]) {
    gpt Y;
    if (!rist_decode(y, Y)) return -1;
    uint32_t ee[8], ss[8];
    words_le(e, ee, 8);
    words_le(s, ss, 8);
    const gpt P = double_scalarmult(Y, ee, ss);
    const fe u2 = fe_mul(P.X, P.Y);
    const fe inv = fe_is_zero(u2) ? fe_one() : fe_invert(u2);
    return rist_encoding_matches(P, inv, r) ? 1 : 0;
}

int dm_fold(uint32_t n, const uint8_t* pts, uint8_t out[32]) {
    gpt acc = pt_identity();
    for (uint32_t i = 0; i < n; i++) {
        gpt P;
        if (!rist_decode(pts + 32 * i, P)) return 1;
        acc = pt_add(acc, P);
    }
    rist_encode(acc, out);
    return 0;
}

}  // extern "C"
