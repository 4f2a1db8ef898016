// Integer-pipe peak microbenchmark (SURVEY.md §8d "P_int"): the roofline
// denominator for the integer-bound hashing kernel. MEASURED_PEAKS.json has
// HBM and bf16 peaks only, so bench.py measures this live, under the same
// clocks as the timed region. Modes:
//   0  ALU pipe only  (LOP3 chains)
//   1  FMA pipe only  (IMAD chains, multiplier opaque to the compiler)
//   2  both pipes     (interleaved LOP3 + IMAD, the dual-issue ceiling)
//   3  IMAD with an immediate multiplier      4  LOP3 + immediate IMAD
//   5  SHF.R.W funnel rotate (ALU pipe)       6  IMAD.HI immediate
//   7  LOP3 + IMAD.HI immediate
//   8  IMAD.WIDE.U32, 64-bit addend          9  LOP3 + IMAD.WIDE.U32
//  11  LOP3 + IMAD with a per-thread REGISTER multiplier (R-R-R operands)
//  12  LOP3 + two-input add, register addend (ptxas: VIADD R, R, R?)
//  13  LOP3 + two-input add, uniform addend (VIADD R, R, UR)
//  14  LOP3 on three vector registers + IMAD R-R-R (register-read pressure)
//  15  LOP3 on three vector registers + IMAD R-UR-R
//  10  shared-memory table lookups: data-dependent 32-bit LDS from a
//      bank-replicated 256-entry table ([x][lane], the AES T-table layout of
//      tile_common.cuh SmemT0), i.e. the suite-2 kernel's bound
// Every thread runs 8 independent chains; lane-ops = threads * iters * 8 (16 for mode 2).
// Not part of the verifier ABI (separate library libposlo_microbench.so).
#include <cuda_runtime.h>
#include <stdint.h>

static __device__ uint32_t g_mb_mult = 0x9e3779b9u;  // the `a` multiplier, read opaquely

template <int MODE>
__global__ void __launch_bounds__(256) k_int_peak(uint32_t* out, uint32_t a, uint32_t b, int iters) {
    uint32_t x[8], y[8];
#pragma unroll
    for (int k = 0; k < 8; k++) {
        x[k] = threadIdx.x * (k + 1) ^ a;
        y[k] = blockIdx.x + k * b + threadIdx.x * 0x10001u;  // per-lane: keeps IMADs off the uniform datapath
    }
    const uint32_t mreg = *reinterpret_cast<volatile const uint32_t*>(&g_mb_mult);  // == a, in a vector register
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 8; k++) {
            if (MODE == 0 || MODE == 2 || MODE == 4 || MODE == 7)
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[k]) : "r"(b), "r"(x[(k + 1) & 7]));
            if (MODE == 1 || MODE == 2)
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(y[k]) : "r"(a), "r"(y[(k + 3) & 7]));
            if (MODE == 3 || MODE == 4)  // IMAD, immediate multiplier
                asm volatile("mad.lo.u32 %0, %0, 0x9e3779b9, %1;" : "+r"(y[k]) : "r"(y[(k + 3) & 7]));
            if (MODE == 5)  // SHF funnel rotate
                asm volatile("shf.r.wrap.b32 %0, %0, %0, 13;" : "+r"(x[k]));
            if (MODE == 6 || MODE == 7)  // IMAD.HI, immediate multiplier
                asm volatile("mad.hi.u32 %0, %0, 0x9e3779b9, %1;" : "+r"(y[k]) : "r"(y[(k + 3) & 7]));
            if (MODE == 8 || MODE == 9) {  // IMAD.WIDE.U32 with a 64-bit addend (radix-2^26 field products)
                uint64_t acc = ((uint64_t)x[k] << 32) | y[k];
                asm volatile("mad.wide.u32 %0, %1, %2, %0;" : "+l"(acc) : "r"(y[(k + 3) & 7]), "r"(a));
                y[k] = (uint32_t)acc;
                if (MODE == 8) x[k] = (uint32_t)(acc >> 32);
            }
            if (MODE >= 11 && MODE <= 13)
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[k]) : "r"(b), "r"(x[(k + 1) & 7]));
            if (MODE == 11)
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(y[k]) : "r"(mreg), "r"(y[(k + 3) & 7]));
            if (MODE == 12)
                asm volatile("add.u32 %0, %0, %1;" : "+r"(y[k]) : "r"(y[(k + 3) & 7]));
            if (MODE == 13)
                asm volatile("add.u32 %0, %0, %1;" : "+r"(y[k]) : "r"(a));
            if (MODE == 14 || MODE == 15)
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[k]) : "r"(x[(k + 5) & 7]), "r"(x[(k + 1) & 7]));
            if (MODE == 14)
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(y[k]) : "r"(mreg), "r"(y[(k + 3) & 7]));
            if (MODE == 15)
                asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(y[k]) : "r"(a), "r"(y[(k + 3) & 7]));
            if (MODE == 9)
                asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(x[k]) : "r"(b), "r"(x[(k + 1) & 7]));
        }
    }
    uint32_t r = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) r ^= x[k] + y[k];
    if (r == 0x12345678u) out[0] = r;
}

__global__ void __launch_bounds__(256) k_lds_peak(uint32_t* out, uint32_t a, int iters) {
    extern __shared__ uint32_t tab[];  // 256 x 32 words
    const uint32_t lane = threadIdx.x & 31u;
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) tab[i] = (uint32_t)i * 0x9e3779b9u ^ a;
    __syncthreads();
    uint32_t x[8];
#pragma unroll
    for (int k = 0; k < 8; k++) x[k] = threadIdx.x * (k + 7) ^ a;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < 8; k++) x[k] = tab[__byte_perm(x[k], 0u, 0x4441u) * 32u + lane];
    }
    uint32_t r = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) r ^= x[k];
    if (r == 0x12345678u) out[0] = r;
}

extern "C" int poslo_microbench_int_peak(int device, int mode, double* ops_per_s, double* ms_out) {
    if (cudaSetDevice(device) != cudaSuccess) return 1;
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, device);
    uint32_t* out;
    cudaMalloc(&out, 4);
    int blocks = p.multiProcessorCount * 8;  // 2048 threads per SM
    int iters = mode == 10 ? 1 << 14 : 1 << 16;
    if (mode == 10) cudaFuncSetAttribute(k_lds_peak, cudaFuncAttributeMaxDynamicSharedMemorySize, 32768);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto launch = [&]() {
        const uint32_t a = 0x9e3779b9u, b = 0x7f4a7c15u;
        switch (mode) {
            case 0: k_int_peak<0><<<blocks, 256>>>(out, a, b, iters); break;
            case 1: k_int_peak<1><<<blocks, 256>>>(out, a, b, iters); break;
            case 2: k_int_peak<2><<<blocks, 256>>>(out, a, b, iters); break;
            case 3: k_int_peak<3><<<blocks, 256>>>(out, a, b, iters); break;
            case 4: k_int_peak<4><<<blocks, 256>>>(out, a, b, iters); break;
            case 5: k_int_peak<5><<<blocks, 256>>>(out, a, b, iters); break;
            case 6: k_int_peak<6><<<blocks, 256>>>(out, a, b, iters); break;
            case 7: k_int_peak<7><<<blocks, 256>>>(out, a, b, iters); break;
            case 8: k_int_peak<8><<<blocks, 256>>>(out, a, b, iters); break;
            case 11: k_int_peak<11><<<blocks, 256>>>(out, a, b, iters); break;
            case 12: k_int_peak<12><<<blocks, 256>>>(out, a, b, iters); break;
            case 13: k_int_peak<13><<<blocks, 256>>>(out, a, b, iters); break;
            case 14: k_int_peak<14><<<blocks, 256>>>(out, a, b, iters); break;
            case 15: k_int_peak<15><<<blocks, 256>>>(out, a, b, iters); break;
            case 10: k_lds_peak<<<blocks / 2, 256, 32768>>>(out, a, iters); break;
            default: k_int_peak<9><<<blocks, 256>>>(out, a, b, iters); break;
        }
    };
    launch();  // warm-up (clock ramp)
    launch();
    cudaEventRecord(e0);
    const int reps = 5;
    for (int r = 0; r < reps; r++) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    double per_iter = (mode == 2 || mode == 4 || mode == 7 || mode == 9 || mode >= 11) ? 16.0 : 8.0;
    double ops = (double)(mode == 10 ? blocks / 2 : blocks) * 256 * iters * per_iter * reps;
    *ops_per_s = ops / (ms * 1e-3);
    if (ms_out) *ms_out = ms / reps;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    return cudaGetLastError() == cudaSuccess ? 0 : 2;
}
