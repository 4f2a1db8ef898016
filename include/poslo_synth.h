/* Counter-based synthetic log generator shared by the device bench, the
 * oracle and the reference-side harness (oracle/ref_tools/ref_tool.cpp), so
 * every party regenerates byte-identical logs from (seed, entry index) and
 * any sub-range can be rebuilt for sampled parity.
 *
 * Entry k (global index, 0-based) of a fixed-length log has L bytes; byte b
 * is byte (b % 8) (little-endian) of poslo_synth_word(seed, k, b / 8).
 * Variable-length ("syslog-style", BASELINE config 4) entries have length
 * 64 + word(seed ^ LEN_TWEAK, k, 0) % 961 in [64, 1024] and printable ASCII
 * bytes 0x20 + (raw % 95). */
#ifndef POSLO_SYNTH_H
#define POSLO_SYNTH_H
#include <stdint.h>

#if defined(__CUDACC__)
#define POSLO_SYNTH_FN static __host__ __device__ __forceinline__
#else
#define POSLO_SYNTH_FN static inline
#endif

#define POSLO_SYNTH_LEN_TWEAK 0x6c656e677468ULL

POSLO_SYNTH_FN uint64_t poslo_synth_word(uint64_t seed, uint64_t k, uint32_t w) {
    uint64_t z = seed + 0x9E3779B97F4A7C15ULL * ((k << 8) + (uint64_t)w + 1ULL);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

POSLO_SYNTH_FN uint8_t poslo_synth_byte(uint64_t seed, uint64_t k, uint32_t b) {
    return (uint8_t)(poslo_synth_word(seed, k, b >> 3) >> (8 * (b & 7)));
}

POSLO_SYNTH_FN uint32_t poslo_synth_varlen(uint64_t seed, uint64_t k) {
    return 64u + (uint32_t)(poslo_synth_word(seed ^ POSLO_SYNTH_LEN_TWEAK, k, 0) % 961ULL);
}

POSLO_SYNTH_FN uint8_t poslo_synth_ascii(uint64_t seed, uint64_t k, uint32_t b) {
    return (uint8_t)(0x20 + poslo_synth_byte(seed, k, b) % 95);
}

#endif
