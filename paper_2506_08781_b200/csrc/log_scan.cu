// Record-boundary discovery of a raw log image on the device (read_log,
// include/poslo/log_file.hpp:34-51: records are LE32 length + payload).
//
// Each record's position depends on every earlier length, so the walk is
// sequential per record; the device makes it parallel by speculation:
//   A  k_scan_chunk — the image is cut into kScanChunk-byte chunks; for every
//      candidate start q in the first kScanWindow bytes of a chunk, a thread
//      walks records from q until it leaves the chunk, hits a truncated record,
//      or lands on a later candidate of the same window (then the two are
//      linked and resolved by pointer jumping in shared memory). Wrong
//      candidates read garbage lengths and die or jump out in one step.
//   B  k_scan_stitch — one thread follows the TRUE chain from offset 0 chunk by
//      chunk through those exits (O(#chunks) steps), walking record by record
//      only where a record ends deeper in a chunk than the window.
//   C  k_scan_emit — one thread per chunk on the true chain rewalks its records
//      and writes their offsets at the stitched prefix positions.
// Exact for any input; FormatError exactly where read_log would throw it.
#include "poslo_internal.h"

namespace poslo_gpu {

namespace {

constexpr uint64_t kTrunc = ~0ull;

__device__ __forceinline__ uint32_t le32_at(const uint8_t* raw, uint64_t p) {
    return (uint32_t)raw[p] | (uint32_t)raw[p + 1] << 8 | (uint32_t)raw[p + 2] << 16 | (uint32_t)raw[p + 3] << 24;
}

// One record step from p (read_log's checks): returns the next position, or kTrunc.
__device__ __forceinline__ uint64_t step(const uint8_t* raw, uint64_t n, uint64_t p) {
    if (n - p < 4) return kTrunc;
    const uint32_t len = le32_at(raw, p);
    if (n - p - 4 < len) return kTrunc;
    return p + 4 + len;
}

constexpr int kScanThreads = 256;

__global__ void __launch_bounds__(kScanThreads) k_scan_chunk(const uint8_t* __restrict__ raw, uint64_t n,
                                                             uint32_t first, uint64_t chunk_bytes,
                                                             uint64_t* __restrict__ exit_out,
                                                             uint32_t* __restrict__ count_out) {
    __shared__ uint64_t s_exit[kScanWindow];
    __shared__ uint32_t s_cnt[kScanWindow];
    __shared__ int16_t s_link[kScanWindow];
    const uint32_t chunk = first + blockIdx.x;
    const uint64_t c0 = (uint64_t)chunk * chunk_bytes;
    const uint64_t cend = min(c0 + chunk_bytes, n);
    const uint64_t wend = min(c0 + kScanWindow, cend);
    for (uint32_t k = threadIdx.x; k < kScanWindow; k += kScanThreads) {
        const uint64_t q = c0 + k;
        uint64_t p = q;
        uint32_t cnt = 0;
        int link = -1;
        if (q < wend) {
            while (p < cend) {
                if (p > q && p < wend) {
                    link = (int)(p - c0);
                    break;
                }
                p = step(raw, n, p);
                if (p == kTrunc) break;
                cnt++;
            }
        }
        s_exit[k] = p;
        s_cnt[k] = cnt;
        s_link[k] = (int16_t)link;
    }
    __syncthreads();
    // pointer jumping: follow links (always forward) until every candidate has its chunk exit
    for (int round = 0; round < 12; round++) {
        uint64_t ex[kScanWindow / kScanThreads];
        uint32_t ct[kScanWindow / kScanThreads];
        int16_t lk[kScanWindow / kScanThreads];
#pragma unroll
        for (int i = 0; i < kScanWindow / kScanThreads; i++) {
            const int k = threadIdx.x + i * kScanThreads;
            const int l = s_link[k];
            ex[i] = s_exit[k];
            ct[i] = s_cnt[k];
            lk[i] = (int16_t)l;
            if (l >= 0) {
                ex[i] = s_exit[l];
                ct[i] = s_cnt[k] + s_cnt[l];
                lk[i] = s_link[l];
            }
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < kScanWindow / kScanThreads; i++) {
            const int k = threadIdx.x + i * kScanThreads;
            s_exit[k] = ex[i];
            s_cnt[k] = ct[i];
            s_link[k] = lk[i];
        }
        __syncthreads();
    }
    for (uint32_t k = threadIdx.x; k < kScanWindow; k += kScanThreads) {
        exit_out[(uint64_t)blockIdx.x * kScanWindow + k] = s_exit[k];  // relative to `first`
        count_out[(uint64_t)blockIdx.x * kScanWindow + k] = s_cnt[k];
    }
}

// state[0] = record count or ~0 on a truncated record; start/base per chunk
__global__ void k_scan_stitch(const uint8_t* __restrict__ raw, uint64_t n, uint32_t n_chunks,
                              const uint64_t* __restrict__ exits, const uint32_t* __restrict__ counts,
                              uint64_t* __restrict__ start, uint64_t* __restrict__ base,
                              unsigned long long* __restrict__ state) {
    if (threadIdx.x || blockIdx.x) return;
    for (uint32_t c = 0; c < n_chunks; c++) start[c] = kTrunc;
    uint64_t q = 0, total = 0;
    while (q < n) {
        const uint64_t c = q / kScanChunk, off = q - c * kScanChunk;
        start[c] = q;
        base[c] = total;
        uint64_t p;
        if (off < kScanWindow) {
            p = exits[c * kScanWindow + off];
            total += counts[c * kScanWindow + off];
        } else {  // the previous record ended deep in this chunk: walk it here
            const uint64_t cend = min((c + 1) * kScanChunk, n);
            p = q;
            while (p < cend && p != kTrunc) {
                p = step(raw, n, p);
                total++;
            }
        }
        if (p == kTrunc) {
            state[0] = ~0ull;
            return;
        }
        q = p;
    }
    state[0] = total;
}

__global__ void k_scan_emit(const uint8_t* __restrict__ raw, uint64_t n, uint32_t n_chunks,
                            const uint64_t* __restrict__ start, const uint64_t* __restrict__ base,
                            uint64_t* __restrict__ offsets) {
    const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n_chunks || start[c] == kTrunc) return;
    const uint64_t cend = min((uint64_t)(c + 1) * kScanChunk, n);
    uint64_t p = start[c], k = base[c];
    while (p < cend) {
        offsets[k++] = p;
        p = step(raw, n, p);  // valid on the true chain (checked by the stitch)
    }
}

// Incremental form of the stitch for a pipelined ingestion (chunks arrive
// one after another): continues the true chain from state = {next record
// position q (kTrunc after a truncated record), records so far} through the
// chunks [c_first, c_last), which must all have been scanned by k_scan_chunk.
__global__ void k_scan_stitch_inc(const uint8_t* __restrict__ raw, uint64_t n, uint32_t c_first, uint32_t c_last,
                                  uint64_t chunk_bytes, const uint64_t* __restrict__ exits,
                                  const uint32_t* __restrict__ counts, uint64_t* __restrict__ start,
                                  uint64_t* __restrict__ base, unsigned long long* __restrict__ state) {
    if (threadIdx.x || blockIdx.x) return;
    for (uint32_t c = c_first; c < c_last; c++) start[c] = kTrunc;
    uint64_t q = state[0], total = state[1];
    const uint64_t lim = min((uint64_t)c_last * chunk_bytes, n);
    while (q != kTrunc && q < lim) {
        const uint64_t c = q / chunk_bytes, off = q - c * chunk_bytes;
        start[c] = q;
        base[c] = total;
        uint64_t p;
        if (off < kScanWindow) {
            const uint64_t w = (c - c_first) * kScanWindow + off;  // exits of this range only
            p = exits[w];
            total += counts[w];
        } else {
            const uint64_t cend = min((c + 1) * chunk_bytes, n);
            p = q;
            while (p < cend && p != kTrunc) {
                p = step(raw, n, p);
                total++;
            }
        }
        q = p;
    }
    state[0] = q;
    state[1] = total;
}

// Offsets of the records starting in chunks [c_first, c_last); writes only
// below cap (a log with more records than expected is reported by the caller).
__global__ void k_scan_emit_range(const uint8_t* __restrict__ raw, uint64_t n, uint32_t c_first, uint32_t c_last,
                                  uint64_t chunk_bytes, const uint64_t* __restrict__ start,
                                  const uint64_t* __restrict__ base, uint64_t* __restrict__ offsets, uint64_t cap) {
    const uint32_t c = c_first + blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= c_last || start[c] == kTrunc) return;
    const uint64_t cend = min((uint64_t)(c + 1) * chunk_bytes, n);
    uint64_t p = start[c], k = base[c];
    while (p < cend && k < cap) {
        offsets[k++] = p;
        p = step(raw, n, p);
    }
}

}  // namespace

void launch_log_scan_range(const uint8_t* d_raw, uint64_t n, uint32_t c_first, uint32_t c_last, uint64_t chunk_bytes,
                           uint64_t* d_exit, uint32_t* d_count, uint64_t* d_start, uint64_t* d_base,
                           unsigned long long* d_state, uint64_t* d_offsets, uint64_t cap, cudaStream_t s) {
    if (c_last <= c_first) return;
    k_scan_chunk<<<c_last - c_first, kScanThreads, 0, s>>>(d_raw, n, c_first, chunk_bytes, d_exit, d_count);
    k_scan_stitch_inc<<<1, 1, 0, s>>>(d_raw, n, c_first, c_last, chunk_bytes, d_exit, d_count, d_start, d_base,
                                      d_state);
    k_scan_emit_range<<<(c_last - c_first + 127) / 128, 128, 0, s>>>(d_raw, n, c_first, c_last, chunk_bytes, d_start,
                                                                     d_base, d_offsets, cap);
}

void launch_log_scan_a(const uint8_t* d_raw, uint64_t n, uint32_t n_chunks, uint64_t* d_exit, uint32_t* d_count,
                       cudaStream_t s) {
    if (n_chunks) k_scan_chunk<<<n_chunks, kScanThreads, 0, s>>>(d_raw, n, 0, kScanChunk, d_exit, d_count);
}

void launch_log_scan_b(const uint8_t* d_raw, uint64_t n, uint32_t n_chunks, const uint64_t* d_exit,
                       const uint32_t* d_count, uint64_t* d_start, uint64_t* d_base, unsigned long long* d_state,
                       cudaStream_t s) {
    k_scan_stitch<<<1, 1, 0, s>>>(d_raw, n, n_chunks, d_exit, d_count, d_start, d_base, d_state);
}

void launch_log_scan_c(const uint8_t* d_raw, uint64_t n, uint32_t n_chunks, const uint64_t* d_start,
                       const uint64_t* d_base, uint64_t* d_offsets, cudaStream_t s) {
    if (n_chunks) k_scan_emit<<<(n_chunks + 127) / 128, 128, 0, s>>>(d_raw, n, n_chunks, d_start, d_base, d_offsets);
}

}  // namespace poslo_gpu
