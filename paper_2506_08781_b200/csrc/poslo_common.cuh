// Shared device/host helpers for the POSLO batch verifier (sm_100a).
//
// All arithmetic on this path is integer: byte/word hashing, 32-bit limbs,
// mod l and mod 2^255-19. Math headers are written as plain
// __host__ __device__ C so tests/native can exercise the same code on the CPU;
// PTX fast paths are confined to `#ifdef __CUDA_ARCH__` branches.
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define PHD __host__ __device__ __forceinline__
#define PHDM __host__ __device__ __forceinline__
#define PD __device__ __forceinline__
#else
#define PHD static inline
#define PHDM inline
#define PD static inline
#endif

PHD uint32_t rotr32(uint32_t x, int n) {
#ifdef __CUDA_ARCH__
    return __funnelshift_r(x, x, n);
#else
    return (x >> n) | (x << ((32 - n) & 31));
#endif
}

// (hi:lo) >> n, low 32 bits: the byte-misaligned word of a shifted stream.
PHD uint32_t fshr32(uint32_t lo, uint32_t hi, int n) {
#ifdef __CUDA_ARCH__
    return __funnelshift_r(lo, hi, n);
#else
    return n == 0 ? lo : (lo >> n) | (hi << (32 - n));
#endif
}

PHD uint32_t bswap32(uint32_t x) {
#ifdef __CUDA_ARCH__
    return __byte_perm(x, 0, 0x0123);
#else
    return (x >> 24) | ((x >> 8) & 0xff00u) | ((x << 8) & 0xff0000u) | (x << 24);
#endif
}

PHD uint32_t load_be32p(const uint8_t* p) {
    return (uint32_t)p[0] << 24 | (uint32_t)p[1] << 16 | (uint32_t)p[2] << 8 | p[3];
}

// Status codes shared with include/poslo_gpu.h.
#define POSLO_ST_OK 0
#define POSLO_ST_FORMAT 1
#define POSLO_ST_STATE 2
#define POSLO_ST_SEED 3
