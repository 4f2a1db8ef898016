/* poslo_oracle.c — CPU restatement of the reference's batch-verification
 * hot path (POSLO, /root/reference/proj), used ONLY as the parity checker by
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg. It is never
 * linked into, loaded by or called from the product path
 * (paper_2506_08781_b200/), which fails loudly without its CUDA library.
 *
 * Pinned: tests/test_oracle.py checks every function here against the golden
 * vectors in tests/golden/ that were produced by the UNMODIFIED reference
 * compiled in oracle/_ref (tests/golden/make_golden.py) and against external
 * FIPS 180-4 / FIPS-197 examples.
 *
 * Third-party algorithms restated here (absent from /root/reference):
 *   - SHA-256 (OpenSSL 3.0.13 `SHA256`, FIPS 180-4), used by primitives.cpp:21-23
 *   - AES-128 encryption (OpenSSL `AES_set_encrypt_key`/`AES_encrypt`,
 *     FIPS-197), used by primitives.cpp:13-19
 *   - Z_l arithmetic (libsodium 1.0.20 `crypto_core_ristretto255_scalar_reduce`
 *     and `_scalar_add`), used by group.cpp:51-59, 68-73; restated as plain
 *     bit-serial big-integer reduction mod l.
 * The ristretto255 group operations are restated in oracle/ristretto.py.
 *
 * Deliberately literal: per-entry reduction then modular add, exactly the
 * reference's operation order (batch_verify.cpp:37-42) — the device path's
 * deferred reduction is proven equal against this. */
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_FORMAT_ERROR 1
#define ORC_STATE_ERROR 2
#define ORC_SEED_NOT_DISCLOSED 3

/* ---------------- SHA-256 (FIPS 180-4 §6.2) ---------------- */
static const uint32_t K256[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4, 0xab1c5ed5,
    0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174,
    0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967,
    0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85,
    0xa2bfe8a1, 0xa81a664b, 0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

static uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

static void sha256_block(uint32_t h[8], const uint8_t blk[64]) {
    uint32_t w[64];
    for (int t = 0; t < 16; t++)
        w[t] = (uint32_t)blk[4 * t] << 24 | (uint32_t)blk[4 * t + 1] << 16 |
               (uint32_t)blk[4 * t + 2] << 8 | blk[4 * t + 3];
    for (int t = 16; t < 64; t++) {
        uint32_t s0 = rotr(w[t - 15], 7) ^ rotr(w[t - 15], 18) ^ (w[t - 15] >> 3);
        uint32_t s1 = rotr(w[t - 2], 17) ^ rotr(w[t - 2], 19) ^ (w[t - 2] >> 10);
        w[t] = w[t - 16] + s0 + w[t - 7] + s1;
    }
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], hh = h[7];
    for (int t = 0; t < 64; t++) {
        uint32_t S1 = rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25);
        uint32_t ch = (e & f) ^ (~e & g);
        uint32_t t1 = hh + S1 + ch + K256[t] + w[t];
        uint32_t S0 = rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22);
        uint32_t maj = (a & b) ^ (a & c) ^ (b & c);
        uint32_t t2 = S0 + maj;
        hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

void orc_sha256(const uint8_t *m, size_t len, uint8_t out[32]) {
    uint32_t h[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                     0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
    size_t off = 0;
    for (; off + 64 <= len; off += 64) sha256_block(h, m + off);
    uint8_t tail[128];
    size_t rem = len - off;
    memset(tail, 0, sizeof tail);
    memcpy(tail, m + off, rem);
    tail[rem] = 0x80;
    size_t tl = rem + 9 <= 64 ? 64 : 128;
    uint64_t bits = (uint64_t)len * 8;
    for (int i = 0; i < 8; i++) tail[tl - 1 - i] = (uint8_t)(bits >> (8 * i));
    sha256_block(h, tail);
    if (tl == 128) sha256_block(h, tail + 64);
    for (int i = 0; i < 8; i++) {
        out[4 * i] = (uint8_t)(h[i] >> 24); out[4 * i + 1] = (uint8_t)(h[i] >> 16);
        out[4 * i + 2] = (uint8_t)(h[i] >> 8); out[4 * i + 3] = (uint8_t)h[i];
    }
}

/* ---------------- AES-128 (FIPS-197) ---------------- */
static uint8_t SBOX[256];
static pthread_once_t sbox_once = PTHREAD_ONCE_INIT;

static uint8_t gmul(uint8_t a, uint8_t b) {
    uint8_t p = 0;
    while (b) {
        if (b & 1) p ^= a;
        a = (uint8_t)((a << 1) ^ ((a & 0x80) ? 0x1b : 0));
        b >>= 1;
    }
    return p;
}

/* S-box derived from its definition (multiplicative inverse in GF(2^8)
 * followed by the affine map, FIPS-197 §5.1.1) rather than typed in. */
static void sbox_init(void) {
    for (int x = 0; x < 256; x++) {
        uint8_t inv = 0;
        if (x) for (int y = 1; y < 256; y++) if (gmul((uint8_t)x, (uint8_t)y) == 1) { inv = (uint8_t)y; break; }
        uint8_t s = inv;
        for (int r = 1; r <= 4; r++) s ^= (uint8_t)((inv << r) | (inv >> (8 - r)));
        SBOX[x] = s ^ 0x63;
    }
}

void orc_aes128(const uint8_t key[16], const uint8_t in[16], uint8_t out[16]) {
    pthread_once(&sbox_once, sbox_init);
    uint8_t rk[176];
    memcpy(rk, key, 16);
    uint8_t rcon = 1;
    for (int i = 16; i < 176; i += 4) {
        uint8_t t[4] = {rk[i - 4], rk[i - 3], rk[i - 2], rk[i - 1]};
        if (i % 16 == 0) {
            uint8_t t0 = t[0];
            t[0] = SBOX[t[1]] ^ rcon; t[1] = SBOX[t[2]]; t[2] = SBOX[t[3]]; t[3] = SBOX[t0];
            rcon = gmul(rcon, 2);
        }
        for (int k = 0; k < 4; k++) rk[i + k] = rk[i - 16 + k] ^ t[k];
    }
    uint8_t s[16];
    for (int k = 0; k < 16; k++) s[k] = in[k] ^ rk[k];
    for (int r = 1; r <= 10; r++) {
        uint8_t u[16];
        for (int k = 0; k < 16; k++) u[k] = SBOX[s[k]];
        /* ShiftRows: byte (row, col) at index 4*col+row moves left by row */
        for (int c = 0; c < 4; c++)
            for (int row = 0; row < 4; row++) s[4 * c + row] = u[4 * ((c + row) % 4) + row];
        if (r != 10) {
            for (int c = 0; c < 4; c++) {
                uint8_t *col = s + 4 * c, a0 = col[0], a1 = col[1], a2 = col[2], a3 = col[3];
                col[0] = gmul(a0, 2) ^ gmul(a1, 3) ^ a2 ^ a3;
                col[1] = a0 ^ gmul(a1, 2) ^ gmul(a2, 3) ^ a3;
                col[2] = a0 ^ a1 ^ gmul(a2, 2) ^ gmul(a3, 3);
                col[3] = gmul(a0, 3) ^ a1 ^ a2 ^ gmul(a3, 2);
            }
        }
        for (int k = 0; k < 16; k++) s[k] ^= rk[16 * r + k];
    }
    memcpy(out, s, 16);
}

/* ---------------- MMO / MDC-2 (primitives.cpp:28-111) ---------------- */
/* 10* padding to 16-byte blocks, a full pad block when len % 16 == 0
 * (primitives.cpp:28-48). Returns padded length; caller frees. */
static uint8_t *pad10(const uint8_t *m, size_t len, size_t *plen) {
    size_t n = (len / 16 + 1) * 16;
    uint8_t *buf = (uint8_t *)calloc(n, 1);
    memcpy(buf, m, len);
    buf[len] = 0x80;
    *plen = n;
    return buf;
}

int orc_mmo(const uint8_t *m, size_t len, uint8_t out[16]) {
    if (len == 0) return ORC_FORMAT_ERROR; /* primitives.cpp:77 */
    size_t n;
    uint8_t *buf = pad10(m, len, &n), h[16], e[16];
    memset(h, 0x52, 16);
    for (size_t off = 0; off < n; off += 16) {
        orc_aes128(h, buf + off, e);
        for (int k = 0; k < 16; k++) h[k] = e[k] ^ buf[off + k];
    }
    memcpy(out, h, 16);
    free(buf);
    return ORC_OK;
}

int orc_mdc2(const uint8_t *m, size_t len, uint8_t out[32]) {
    if (len == 0) return ORC_FORMAT_ERROR; /* primitives.cpp:90 */
    size_t n;
    uint8_t *buf = pad10(m, len, &n), h[16], h2[16], e[16], a[16], b[16];
    memset(h, 0x52, 16);
    memset(h2, 0x25, 16);
    for (size_t off = 0; off < n; off += 16) {
        orc_aes128(h, buf + off, e);
        for (int k = 0; k < 16; k++) a[k] = e[k] ^ buf[off + k];
        orc_aes128(h2, buf + off, e);
        for (int k = 0; k < 16; k++) b[k] = e[k] ^ buf[off + k];
        memcpy(h, a, 8); memcpy(h + 8, b + 8, 8);   /* swap of second halves */
        memcpy(h2, b, 8); memcpy(h2 + 8, a + 8, 8); /* primitives.cpp:102-105 */
    }
    memcpy(out, h, 16);
    memcpy(out + 16, h2, 16);
    free(buf);
    return ORC_OK;
}

/* ---------------- Z_l (group.cpp:51-73 via libsodium) ---------------- */
/* l = 2^252 + 27742317777372353535851937790883648493, little-endian 64-bit limbs */
static const uint64_t L64[4] = {0x5812631a5cf5d3edULL, 0x14def9dea2f79cd6ULL, 0, 0x1000000000000000ULL};

static int geq_l(const uint64_t r[4]) {
    for (int i = 3; i >= 0; i--) {
        if (r[i] > L64[i]) return 1;
        if (r[i] < L64[i]) return 0;
    }
    return 1;
}
static void sub_l(uint64_t r[4]) {
    unsigned __int128 borrow = 0;
    for (int i = 0; i < 4; i++) {
        unsigned __int128 d = (unsigned __int128)r[i] - L64[i] - borrow;
        r[i] = (uint64_t)d;
        borrow = (d >> 64) ? 1 : 0;
    }
}

/* x (big-endian, n bytes) mod l, bit-serial: r = 2r + bit, subtract l when
 * r >= l. r < 2l < 2^254 always fits in 256 bits. */
static void mod_l_be(const uint8_t *be, size_t n, uint64_t r[4]) {
    r[0] = r[1] = r[2] = r[3] = 0;
    for (size_t byte = 0; byte < n; byte++)
        for (int bit = 7; bit >= 0; bit--) {
            r[3] = r[3] << 1 | r[2] >> 63;
            r[2] = r[2] << 1 | r[1] >> 63;
            r[1] = r[1] << 1 | r[0] >> 63;
            r[0] = r[0] << 1 | ((be[byte] >> bit) & 1);
            if (geq_l(r)) sub_l(r);
        }
}

static void limbs_to_le(const uint64_t r[4], uint8_t out[32]) {
    for (int i = 0; i < 32; i++) out[i] = (uint8_t)(r[i / 8] >> (8 * (i % 8)));
}
static void le_to_limbs(const uint8_t in[32], uint64_t r[4]) {
    for (int i = 0; i < 4; i++) {
        r[i] = 0;
        for (int k = 7; k >= 0; k--) r[i] = r[i] << 8 | in[8 * i + k];
    }
}

/* Scalar::reduce_wide_be (group.cpp:51-59) */
void orc_reduce_wide_be(const uint8_t in[64], uint8_t out_le[32]) {
    uint64_t r[4];
    mod_l_be(in, 64, r);
    limbs_to_le(r, out_le);
}

/* Scalar::add (group.cpp:68-73); inputs canonical (< l) */
void orc_sc_add(const uint8_t a[32], const uint8_t b[32], uint8_t out[32]) {
    uint64_t x[4], y[4];
    le_to_limbs(a, x);
    le_to_limbs(b, y);
    unsigned __int128 c = 0;
    for (int i = 0; i < 4; i++) {
        c += (unsigned __int128)x[i] + y[i];
        x[i] = (uint64_t)c;
        c >>= 64;
    }
    if (geq_l(x)) sub_l(x);
    limbs_to_le(x, out);
}

/* ---------------- primitives (primitives.cpp:113-223) ---------------- */
static int aes_suite(int s) { return s == 2 || s == 3; }

/* prf: F(x || j)[0:16] (primitives.cpp:113-127) */
void orc_prf(int suite, int j, const uint8_t x[16], uint8_t out[16]) {
    uint8_t in[17], d[32];
    memcpy(in, x, 16);
    in[16] = (uint8_t)(j & 1);
    if (aes_suite(suite)) orc_mmo(in, 17, d);
    else orc_sha256(in, 17, d);
    memcpy(out, d, 16);
}

/* onetime_seed: F(x0 || be32(j))[0:16] (primitives.cpp:209-223) */
void orc_onetime_seed(int suite, const uint8_t x0[16], uint32_t j, uint8_t out[16]) {
    uint8_t in[20], d[32];
    memcpy(in, x0, 16);
    in[16] = (uint8_t)(j >> 24); in[17] = (uint8_t)(j >> 16);
    in[18] = (uint8_t)(j >> 8); in[19] = (uint8_t)j;
    if (aes_suite(suite)) orc_mmo(in, 20, d);
    else orc_sha256(in, 20, d);
    memcpy(out, d, 16);
}

/* hash_to_scalar (primitives.cpp:149-193). Returns ORC_FORMAT_ERROR for a
 * suite-3 entry longer than 31 bytes or an unknown suite. */
int orc_hash_to_scalar(int suite, const uint8_t *m, size_t mlen, const uint8_t x[16], uint8_t e_le[32]) {
    if (suite == 1 || suite == 2) {
        uint8_t *buf = (uint8_t *)malloc(1 + mlen + 16), wide[64];
        buf[0] = 0x01;
        memcpy(buf + 1, m, mlen);
        memcpy(buf + 1 + mlen, x, 16);
        size_t n = mlen + 16;
        if (suite == 1) {
            orc_sha256(buf + 1, n, wide);     /* H(m || x): high half */
            orc_sha256(buf, n + 1, wide + 32); /* H(0x01 || m || x): low half */
        } else {
            orc_mdc2(buf + 1, n, wide);
            orc_mdc2(buf, n + 1, wide + 32);
        }
        free(buf);
        orc_reduce_wide_be(wide, e_le);
        return ORC_OK;
    }
    if (suite == 3) {
        if (mlen > 31) return ORC_FORMAT_ERROR;
        uint64_t a[4], b[4];
        uint8_t ea[32], eb[32];
        mod_l_be(m, mlen, a);
        mod_l_be(x, 16, b);
        limbs_to_le(a, ea);
        limbs_to_le(b, eb);
        orc_sc_add(ea, eb, e_le);
        return ORC_OK;
    }
    return ORC_FORMAT_ERROR;
}

/* ---------------- seed tree (seed_manager.cpp) ---------------- */
typedef struct { uint8_t depth; uint32_t index; uint8_t value[16]; } orc_node;

/* SeedStack::deserialize (seed_manager.cpp:41-53) + push checks (:18-23) */
static int parse_ds(const uint8_t *w, size_t n, uint32_t cap, orc_node *nodes, int *count) {
    if (n < 1) return ORC_FORMAT_ERROR;
    int c = w[0];
    size_t off = 1;
    for (int k = 0; k < c; k++) {
        if (n - off < 21) return ORC_FORMAT_ERROR;
        if ((uint32_t)k >= cap) return ORC_STATE_ERROR;
        nodes[k].depth = w[off];
        nodes[k].index = (uint32_t)w[off + 1] << 24 | (uint32_t)w[off + 2] << 16 |
                         (uint32_t)w[off + 3] << 8 | w[off + 4];
        memcpy(nodes[k].value, w + off + 5, 16);
        if (k > 0 && nodes[k - 1].depth <= nodes[k].depth) return ORC_STATE_ERROR;
        off += 21;
    }
    *count = c;
    return ORC_OK;
}

/* sr (seed_manager.cpp:71-85) walking down with sc (:5-16) */
static int sr_nodes(int suite, const orc_node *nodes, int count, uint32_t q, uint8_t out[16]) {
    if (count == 0) return ORC_SEED_NOT_DISCLOSED;
    for (int k = count - 1; k >= 0; k--) {
        const orc_node *nd = &nodes[k];
        uint64_t lo = (uint64_t)nd->index << nd->depth;
        uint64_t hi = (uint64_t)(uint32_t)(nd->index + 1) << nd->depth; /* u32 add as in :76 */
        if (q >= hi && k + 1 == count) return ORC_SEED_NOT_DISCLOSED;
        if (q >= lo && q < hi) {
            uint8_t x[16], y[16];
            memcpy(x, nd->value, 16);
            uint32_t rel = q - (uint32_t)lo;
            for (int j = nd->depth - 1; j >= 0; j--) {
                orc_prf(suite, (rel >> j) & 1, x, y);
                memcpy(x, y, 16);
            }
            memcpy(out, x, 16);
            return ORC_OK;
        }
    }
    return ORC_SEED_NOT_DISCLOSED;
}

int orc_sr(int suite, const uint8_t *ds, size_t ds_len, uint32_t cap, uint32_t q, uint8_t out[16]) {
    orc_node nodes[256];
    int count = 0;
    int st = parse_ds(ds, ds_len, cap, nodes, &count);
    if (st) return st;
    return sr_nodes(suite, nodes, count, q, out);
}

/* ---------------- agg_ekeys (batch_verify.cpp:11-62) ---------------- */
typedef struct {
    int suite;
    const uint8_t *payload;
    const uint64_t *offsets; /* n_entries + 1, or NULL for a fixed stride */
    uint32_t entry_len;
    const uint32_t *epochs;
    const uint64_t *epoch_starts; /* n_epochs + 1 */
    uint32_t n_epochs;
    const orc_node *nodes;
    int count;
    uint8_t *e_out;
    int *status; /* per epoch */
    volatile uint32_t cursor;
    pthread_mutex_t mtx;
} agg_job;

static void *agg_worker(void *arg) {
    agg_job *J = (agg_job *)arg;
    for (;;) {
        pthread_mutex_lock(&J->mtx);
        uint32_t k = J->cursor++;
        pthread_mutex_unlock(&J->mtx);
        if (k >= J->n_epochs) break;
        uint8_t x0[16], x[16], e[32], acc[32] = {0};
        int st = sr_nodes(J->suite, J->nodes, J->count, J->epochs[k], x0);
        if (st == ORC_OK) {
            for (uint64_t t = J->epoch_starts[k]; t < J->epoch_starts[k + 1]; t++) {
                uint32_t j = (uint32_t)(t - J->epoch_starts[k]);
                const uint8_t *m;
                size_t mlen;
                if (J->offsets) { m = J->payload + J->offsets[t]; mlen = J->offsets[t + 1] - J->offsets[t]; }
                else { m = J->payload + t * J->entry_len; mlen = J->entry_len; }
                orc_onetime_seed(J->suite, x0, j, x);
                st = orc_hash_to_scalar(J->suite, m, mlen, x, e);
                if (st) break;
                orc_sc_add(acc, e, acc);
            }
        }
        J->status[k] = st;
        memcpy(J->e_out + 32 * (size_t)k, acc, 32);
    }
    return NULL;
}

/* Returns ORC_OK or the first error in epoch order (the workers == 1
 * behaviour); *err_epoch receives the offending epoch index. */
int orc_agg_ekeys(int suite, const uint8_t *payload, const uint64_t *offsets, uint32_t entry_len,
                  const uint32_t *epochs, const uint64_t *epoch_starts, uint32_t n_epochs,
                  const uint8_t *ds, size_t ds_len, uint32_t cap, uint8_t *e_out,
                  uint32_t *err_epoch, int threads) {
    orc_node nodes[256];
    int count = 0;
    int st = parse_ds(ds, ds_len, cap, nodes, &count);
    if (st) return st;
    agg_job J;
    J.suite = suite; J.payload = payload; J.offsets = offsets; J.entry_len = entry_len;
    J.epochs = epochs; J.epoch_starts = epoch_starts; J.n_epochs = n_epochs;
    J.nodes = nodes; J.count = count; J.e_out = e_out; J.cursor = 0;
    J.status = (int *)calloc(n_epochs ? n_epochs : 1, sizeof(int));
    pthread_mutex_init(&J.mtx, NULL);
    if (threads < 1) threads = 1;
    if ((uint32_t)threads > n_epochs) threads = n_epochs ? (int)n_epochs : 1;
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * threads);
    for (int i = 0; i < threads; i++) pthread_create(&th[i], NULL, agg_worker, &J);
    for (int i = 0; i < threads; i++) pthread_join(th[i], NULL);
    free(th);
    pthread_mutex_destroy(&J.mtx);
    int rc = ORC_OK;
    for (uint32_t k = 0; k < n_epochs; k++)
        if (J.status[k]) { rc = J.status[k]; if (err_epoch) *err_epoch = epochs[k]; break; }
    free(J.status);
    return rc;
}
