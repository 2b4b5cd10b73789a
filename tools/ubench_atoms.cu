// ubench_atoms.cu -- microbenchmark (not product code): shared-memory histogram update
// throughput on sm_100a.  Digits are pseudo-random in [0, 2^D).  Variants:
//   atoms   : atomicAdd on one CTA-wide histogram (ATOMS)
//   match   : per-warp private histogram; __match_any_sync groups equal digits, the leader
//             does a plain LDS+STS (no atomics)
//   atoms_w : per-warp private histograms with ATOMS (fewer address conflicts)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CKE(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

constexpr int NT = 512, NW = NT / 32, ITERS = 4096;

__device__ __forceinline__ uint32_t digit(uint32_t x, int D) { return (x * 0x9E3779B1u) >> (32 - D); }

template <int MODE>
__global__ void __launch_bounds__(NT) k_hist(int D, uint32_t* out) {
    extern __shared__ uint32_t h[];
    const int nd = 1 << D;
    const int tot = MODE == 0 ? nd : nd * NW;
    for (int i = threadIdx.x; i < tot; i += NT) h[i] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    uint32_t x = blockIdx.x * NT + threadIdx.x;
    uint32_t* hw = h + (MODE == 0 ? 0 : warp * nd);
    for (int it = 0; it < ITERS; ++it) {
        x = x * 1664525u + 1013904223u;
        const uint32_t d = digit(x, D);
        if (MODE == 0 || MODE == 2) {
            atomicAdd(&hw[d], 1u);
        } else {
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            if (lane == __ffs(peers) - 1) hw[d] += __popc(peers);
            __syncwarp();
        }
    }
    __syncthreads();
    uint32_t s = 0;
    for (int i = threadIdx.x; i < tot; i += NT) s += h[i];
    atomicAdd(out, s);
}

int main() {
    uint32_t* out;
    CKE(cudaMalloc(&out, 4));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int grid = 148 * 4;
    for (int D : {5, 8, 10, 12}) {
        const char* names[3] = {"atoms", "match", "atoms_w"};
        for (int m = 0; m < 3; ++m) {
            const size_t sm = (size_t)(m == 0 ? 1 : NW) << D << 2;
            if (sm > 200 * 1024) continue;
            float best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                cudaEventRecord(a);
                if (m == 0) { CKE(cudaFuncSetAttribute(k_hist<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); k_hist<0><<<grid, NT, sm>>>(D, out); }
                if (m == 1) { CKE(cudaFuncSetAttribute(k_hist<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); k_hist<1><<<grid, NT, sm>>>(D, out); }
                if (m == 2) { CKE(cudaFuncSetAttribute(k_hist<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); k_hist<2><<<grid, NT, sm>>>(D, out); }
                cudaEventRecord(b);
                CKE(cudaEventSynchronize(b));
                CKE(cudaGetLastError());
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                if (rep) best = ms < best ? ms : best;
            }
            const double ops = (double)grid * NT * ITERS;
            printf("D=%2d %-8s %7.3f ms  %7.1f Gops/s  %5.2f ops/SM/cycle\n", D, names[m], best, ops / best / 1e6,
                   ops / (best * 1e-3) / 148 / 1.965e9);
        }
    }
    return 0;
}
