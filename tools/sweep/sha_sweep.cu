// Pipe-assignment sweep for the suite-1 hash kernel (not part of the product).
// Times k_hash_s1_l32m<256, 4, 16 + P, 4, 2> for a list of P bit sets (see
// sha_rnd_p in csrc/sha256.cuh) on 2^26 x 32-byte entries, n2 = 256, and
// checks every variant's per-epoch e~ against P = 0 (bit-exact).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../../paper_2506_08781_b200/csrc \
//        -o sha_sweep sha_sweep.cu
#include "hash_s1.cu"

#include <cstdio>
#include <cstring>
#include <vector>

using namespace poslo_gpu;

template <int FMA, int MINB>
static float run_r(const uint4* pay, const uint4* x0, uint32_t* et, uint32_t n_ep, int reps) {
    const uint32_t grid = (n_ep + 3) / 4;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_hash_s1_l32r<256, 4, FMA, MINB><<<grid, 256>>>(pay, 256, n_ep, 0, x0, et, pipek_make());
    cudaEventRecord(a);
    for (int r = 0; r < reps; r++)
        k_hash_s1_l32r<256, 4, FMA, MINB><<<grid, 256>>>(pay, 256, n_ep, 0, x0, et, pipek_make());
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    return ms / reps;
}

__global__ void fill(uint32_t* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint64_t z = i * 0x9e3779b97f4a7c15ull;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        p[i] = (uint32_t)(z ^ (z >> 31));
    }
}

int main() {
    const uint32_t n = 1u << 26, n_ep = n / 256;
    uint4 *pay, *x0;
    uint32_t *et, *et0;
    cudaMalloc(&pay, (size_t)n * 32);
    cudaMalloc(&x0, (size_t)n_ep * 16);
    cudaMalloc(&et, (size_t)n_ep * 68);
    fill<<<1184, 256>>>((uint32_t*)pay, (size_t)n * 8);
    fill<<<1184, 256>>>((uint32_t*)x0, (size_t)n_ep * 4);
    std::vector<uint32_t> ref(n_ep * 17), got(n_ep * 17);
    const int reps = 5;
    auto check = [&](int P, float ms) {
        cudaMemcpy(got.data(), et, got.size() * 4, cudaMemcpyDeviceToHost);
        bool ok = P == 1000 ? (ref = got, true) : memcmp(ref.data(), got.data(), ref.size() * 4) == 0;
        printf("P=%3d  %8.3f ms  %.3e entries/s  %s\n", P, ms, n / (ms * 1e-3), ok ? "ok" : "MISMATCH");
        fflush(stdout);
    };
#define R(P, MINB) printf("lean MINB=%d ", MINB), check(1000 + P, run_r<16 + P, MINB>(pay, x0, et, n_ep, reps));
    R(0, 3) R(0, 4) R(0, 5) R(1, 4) R(2, 4) R(3, 4) R(4, 4) R(5, 4) R(7, 4) R(13, 4) R(16, 4) R(18, 4) R(19, 4)
    R(33, 4) R(35, 4) R(65, 4) R(3, 5) R(2, 5) R(1, 5) R(5, 5) R(0, 6) R(3, 6)
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
