/* Declaration-only shim for libsodium 1.0.20 (the pyzmq-bundled build at
 * site-packages/pyzmq.libs/libsodium-19479d6d.so.26.2.0). The image ships the
 * library but not its headers; these prototypes follow libsodium's public API
 * exactly as the reference calls it (proj/src/group.cpp, poslo_c.cpp,
 * poslo_f.cpp). Test infrastructure only: used to build oracle/_ref. */
#ifndef ORACLE_SHIM_SODIUM_H
#define ORACLE_SHIM_SODIUM_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
int sodium_init(void);
void randombytes_buf(void *const buf, const size_t size);
uint32_t randombytes_uniform(const uint32_t upper_bound);
typedef struct randombytes_implementation {
    const char *(*implementation_name)(void);
    uint32_t (*random)(void);
    void (*stir)(void);
    uint32_t (*uniform)(const uint32_t upper_bound);
    void (*buf)(void *const buf, const size_t size);
    int (*close)(void);
} randombytes_implementation;
int randombytes_set_implementation(const randombytes_implementation *impl);
void crypto_core_ristretto255_scalar_reduce(unsigned char *r, const unsigned char *s);
void crypto_core_ristretto255_scalar_random(unsigned char *r);
void crypto_core_ristretto255_scalar_add(unsigned char *z, const unsigned char *x, const unsigned char *y);
void crypto_core_ristretto255_scalar_sub(unsigned char *z, const unsigned char *x, const unsigned char *y);
void crypto_core_ristretto255_scalar_mul(unsigned char *z, const unsigned char *x, const unsigned char *y);
int crypto_core_ristretto255_is_valid_point(const unsigned char *p);
int crypto_core_ristretto255_add(unsigned char *r, const unsigned char *p, const unsigned char *q);
int crypto_core_ristretto255_sub(unsigned char *r, const unsigned char *p, const unsigned char *q);
int crypto_core_ristretto255_from_hash(unsigned char *p, const unsigned char *r);
int crypto_scalarmult_ristretto255(unsigned char *q, const unsigned char *n, const unsigned char *p);
int crypto_scalarmult_ristretto255_base(unsigned char *q, const unsigned char *n);
int crypto_hash_sha256(unsigned char *out, const unsigned char *in, unsigned long long inlen);
#ifdef __cplusplus
}
#endif
#endif
