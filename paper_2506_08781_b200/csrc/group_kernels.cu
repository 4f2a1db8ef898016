// Stage 3 of the batch verifier on sm_100a: batched ristretto255 group
// checks (commit_check(Y, e, s) == R, group.cpp:144-167 + group.hpp:59),
// the R-hat fold of paver (batch_verify.cpp:75-81, group_combine
// group.cpp:169-178) and point validation (GroupElement::from_bytes,
// group.cpp:107-114). One thread per check; folds are block trees.
#include "poslo_internal.h"
#include "ristretto.cuh"

namespace poslo_gpu {

namespace {

__device__ __forceinline__ void load32(const uint8_t* p, uint8_t b[32]) {
#pragma unroll
    for (int k = 0; k < 32; k++) b[k] = p[k];
}

__global__ void __launch_bounds__(128) k_group_check(const uint8_t* __restrict__ y, uint32_t n,
                                                     const uint32_t* __restrict__ e,
                                                     const uint32_t* __restrict__ s,
                                                     const uint8_t* __restrict__ r,
                                                     uint8_t* __restrict__ enc,
                                                     uint8_t* __restrict__ verdict, int* ybad) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t yb[32];
    load32(y, yb);
    gpt Y;
    if (!rist_decode(yb, Y)) {
        if (ybad) atomicOr(ybad, 1);
        if (verdict) verdict[i] = 0;
        return;
    }
    uint32_t ee[8], ss[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        ee[k] = e[(size_t)i * 8 + k];
        ss[k] = s[(size_t)i * 8 + k];
    }
    uint8_t out[32];
    commit_check_enc(Y, ee, ss, out);
    if (enc)
#pragma unroll
        for (int k = 0; k < 32; k++) enc[(size_t)i * 32 + k] = out[k];
    if (r && verdict) {
        uint32_t diff = 0;
#pragma unroll
        for (int k = 0; k < 32; k++) diff |= out[k] ^ r[(size_t)i * 32 + k];
        verdict[i] = diff == 0;
    }
}

__device__ __forceinline__ void block_reduce_pt(gpt& acc, gpt* sh) {
    sh[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w >= 1; w >>= 1) {
        if ((int)threadIdx.x < w) sh[threadIdx.x] = pt_add(sh[threadIdx.x], sh[threadIdx.x + w]);
        __syncthreads();
    }
    acc = sh[0];
}

__global__ void __launch_bounds__(128) k_fold_stage1(const uint8_t* __restrict__ pts, uint64_t n,
                                                     gpt* __restrict__ partial, int* bad) {
    __shared__ gpt sh[128];
    gpt acc = pt_identity();
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
         i += (uint64_t)gridDim.x * blockDim.x) {
        uint8_t b[32];
        load32(pts + i * 32, b);
        gpt P;
        if (!rist_decode(b, P)) {
            atomicAdd(bad, 1);
            continue;
        }
        acc = pt_add(acc, P);
    }
    block_reduce_pt(acc, sh);
    if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

__global__ void __launch_bounds__(128) k_fold_stage2(const gpt* __restrict__ partial, uint32_t n,
                                                     uint8_t* __restrict__ out) {
    __shared__ gpt sh[128];
    gpt acc = pt_identity();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) acc = pt_add(acc, partial[i]);
    block_reduce_pt(acc, sh);
    if (threadIdx.x == 0) {
        uint8_t b[32];
        rist_encode(acc, b);
#pragma unroll
        for (int k = 0; k < 32; k++) out[k] = b[k];
    }
}

__global__ void k_validate(const uint8_t* __restrict__ pts, uint32_t n, uint8_t* __restrict__ ok) {
    uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    uint8_t b[32];
    load32(pts + (size_t)i * 32, b);
    gpt P;
    ok[i] = rist_decode(b, P) ? 1 : 0;
}

}  // namespace

void launch_group_check(const uint8_t* d_y, uint32_t n, const uint32_t* d_e, const uint32_t* d_s,
                        const uint8_t* d_r, uint8_t* d_enc, uint8_t* d_verdict, int* d_ybad,
                        cudaStream_t s) {
    if (!n) return;
    k_group_check<<<(n + 127) / 128, 128, 0, s>>>(d_y, n, d_e, d_s, d_r, d_enc, d_verdict, d_ybad);
}

void launch_point_fold(const uint8_t* d_pts, uint64_t n, uint8_t* d_out, int* d_bad, void* d_scratch,
                       cudaStream_t s) {
    uint64_t want = (n + 127) / 128;
    uint32_t blocks = (uint32_t)(want < 1 ? 1 : (want > 1024 ? 1024 : want));
    gpt* part = static_cast<gpt*>(d_scratch);
    k_fold_stage1<<<blocks, 128, 0, s>>>(d_pts, n, part, d_bad);
    k_fold_stage2<<<1, 128, 0, s>>>(part, blocks, d_out);
}

void launch_point_validate(const uint8_t* d_pts, uint32_t n, uint8_t* d_ok, cudaStream_t s) {
    if (!n) return;
    k_validate<<<(n + 127) / 128, 128, 0, s>>>(d_pts, n, d_ok);
}

}  // namespace poslo_gpu
