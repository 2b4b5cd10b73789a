// ubench_scatter.cu -- microbenchmark (not product code): throughput of scattered 8-byte
// stores grouped in runs of L consecutive items (L = 1 .. 32), the access pattern of the
// split / S5 / S9 scatters.  Each warp writes 32/L runs per instruction; run r of the whole
// grid goes to a pseudo-random run slot (bijective multiply mod 2^m).
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CKE(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__global__ void k_scatter(const unsigned long long* __restrict__ src, unsigned long long* __restrict__ dst, int lg_items,
                          int lg_run) {
    const uint64_t n = 1ull << lg_items;
    const uint64_t nruns_mask = (1ull << (lg_items - lg_run)) - 1;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t run = i >> lg_run, j = i & ((1ull << lg_run) - 1);
        const uint64_t slot = (run * 0x9E3779B97F4A7C15ull) & nruns_mask;
        dst[(slot << lg_run) | j] = __ldcs(src + i);
    }
}

int main() {
    const int lg = 28;
    unsigned long long *s, *d;
    CKE(cudaMalloc(&s, 8ull << lg));
    CKE(cudaMalloc(&d, 8ull << lg));
    CKE(cudaMemset(s, 1, 8ull << lg));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int lr = 0; lr <= 5; ++lr) {
        float best = 1e9;
        for (int rep = 0; rep < 4; ++rep) {
            cudaEventRecord(a);
            k_scatter<<<148 * 16, 256>>>(s, d, lg, lr);
            cudaEventRecord(b);
            CKE(cudaEventSynchronize(b));
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            if (rep) best = ms < best ? ms : best;
        }
        printf("run %2d items (%4d B): %7.3f ms  %6.2f TB/s (read+write)\n", 1 << lr, 8 << lr, best,
               2.0 * (8ull << lg) / best / 1e9);
    }
    return 0;
}
