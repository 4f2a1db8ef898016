/* Declaration-only shim for GMP 6.x (runtime libgmp.so.10 is in the image, the
 * header is not). Only the mpz calls the reference tests use. Test
 * infrastructure only: used to build oracle/_ref. */
#ifndef ORACLE_SHIM_GMP_H
#define ORACLE_SHIM_GMP_H
#include <stddef.h>
#ifdef __cplusplus
extern "C" {
#endif
typedef struct { int _mp_alloc; int _mp_size; void *_mp_d; } __mpz_struct;
typedef __mpz_struct mpz_t[1];
typedef __mpz_struct *mpz_ptr;
typedef const __mpz_struct *mpz_srcptr;
#define mpz_init __gmpz_init
#define mpz_inits __gmpz_inits
#define mpz_clear __gmpz_clear
#define mpz_clears __gmpz_clears
#define mpz_set_str __gmpz_set_str
#define mpz_set_ui __gmpz_set_ui
#define mpz_import __gmpz_import
#define mpz_export __gmpz_export
#define mpz_add __gmpz_add
#define mpz_sub __gmpz_sub
#define mpz_mul __gmpz_mul
#define mpz_mod __gmpz_mod
#define mpz_submul __gmpz_submul
#define mpz_cmp __gmpz_cmp
void mpz_init(mpz_ptr);
void mpz_inits(mpz_ptr, ...);
void mpz_clear(mpz_ptr);
void mpz_clears(mpz_ptr, ...);
int mpz_set_str(mpz_ptr, const char *, int);
void mpz_set_ui(mpz_ptr, unsigned long);
void mpz_import(mpz_ptr, size_t, int, size_t, int, size_t, const void *);
void *mpz_export(void *, size_t *, int, size_t, int, size_t, mpz_srcptr);
void mpz_add(mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_sub(mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_mul(mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_mod(mpz_ptr, mpz_srcptr, mpz_srcptr);
void mpz_submul(mpz_ptr, mpz_srcptr, mpz_srcptr);
int mpz_cmp(mpz_srcptr, mpz_srcptr);
#ifdef __cplusplus
}
#endif
#endif
