// ubench_dsmem.cu -- microbenchmark (not product code): counting 64-bit keys in hash tables
// spread over the shared memories of a thread-block cluster (DSMEM), with remote
// atomicCAS/atomicAdd, versus the same insert into the CTA's own table.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/ub_dsmem tools/ubench_dsmem.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;

constexpr int NT = 1024;
constexpr int TS = 8192;  // slots per CTA: 64 KB keys + 32 KB counts
constexpr unsigned long long EMPTY = ~0ull;

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
    x ^= x >> 33;
    x *= 0xff51afd7ed558ccdull;
    x ^= x >> 33;
    x *= 0xc4ceb9fe1a85ec53ull;
    x ^= x >> 33;
    return x;
}

// MODE 0: own table through a plain shared pointer; 1: own table through map_shared_rank;
// 2: owner = hash bits (remote for (CL-1)/CL of the keys)
template <int CL, int MODE>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(NT, 2)
k_count(uint64_t n_per_cta, uint64_t distinct, unsigned long long* out) {
    extern __shared__ __align__(16) uint8_t smem[];
    unsigned long long* tk = reinterpret_cast<unsigned long long*>(smem);
    unsigned int* tc = reinterpret_cast<unsigned int*>(tk + TS);
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    for (int i = threadIdx.x; i < TS; i += NT) {
        tk[i] = EMPTY;
        tc[i] = 0;
    }
    cl.sync();
    const uint64_t cid = blockIdx.x / CL;
    unsigned long long probes = 0;
    for (uint64_t i = threadIdx.x; i < n_per_cta; i += NT) {
        const uint64_t g = (uint64_t)rank * n_per_cta + i;
        const uint64_t key = mix64(mix64(g + 0x1234567ull * cid) % distinct + cid * 0x9E3779B97F4A7C15ull);
        const uint64_t h = mix64(key ^ 0xabcdefull);
        unsigned owner = MODE == 2 ? (unsigned)((h >> 40) % CL) : rank;
        if (MODE == 2 && CL == 1) owner = 0;
        unsigned long long* k_ = tk;
        unsigned int* c_ = tc;
        if (MODE != 0) {
            k_ = cl.map_shared_rank(tk, owner);
            c_ = cl.map_shared_rank(tc, owner);
        }
        uint32_t s = (uint32_t)h & (TS - 1);
        for (;;) {
            ++probes;
            const unsigned long long old = atomicCAS(k_ + s, EMPTY, (unsigned long long)key);
            if (old == EMPTY || old == key) {
                atomicAdd(c_ + s, 1u);
                break;
            }
            s = (s + 1) & (TS - 1);
        }
    }
    cl.sync();
    unsigned long long tot = 0, used = 0;
    for (int i = threadIdx.x; i < TS; i += NT) {
        tot += tc[i];
        used += tc[i] != 0;
    }
    atomicAdd(out + 0, tot);
    atomicAdd(out + 1, used);
    atomicAdd(out + 2, probes);
}

template <int CL, int MODE>
void run(int n_sms, uint64_t n_per_cta, double load) {
    const int smem = TS * 12;
    cudaFuncSetAttribute(k_count<CL, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (CL > 8) cudaFuncSetAttribute(k_count<CL, MODE>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    int grid = n_sms * 2;
    grid -= grid % CL;
    const uint64_t distinct = (uint64_t)(load * TS * (MODE == 2 ? CL : 1));
    unsigned long long* out;
    cudaMalloc(&out, 24);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    float best = 1e30f;
    unsigned long long h[3] = {0, 0, 0};
    for (int rep = 0; rep < 4; ++rep) {
        cudaMemset(out, 0, 24);
        cudaEventRecord(a);
        k_count<CL, MODE><<<grid, NT, smem>>>(n_per_cta, distinct, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        if (ms < best) best = ms;
        cudaMemcpy(h, out, 24, cudaMemcpyDeviceToHost);
    }
    cudaError_t e = cudaGetLastError();
    const double keys = (double)grid * n_per_cta;
    printf("CL=%2d mode=%d grid=%d  %.3f ms  %.1f G keys/s  (sum %llu of %.0f, used %llu, probes/key %.2f) %s\n", CL, MODE,
           grid, best, keys / best / 1e6, h[0], keys, h[1], (double)h[2] / keys, cudaGetErrorString(e));
    cudaFree(out);
}

int main() {
    int n_sms;
    cudaDeviceGetAttribute(&n_sms, cudaDevAttrMultiProcessorCount, 0);
    const uint64_t n = 1 << 20;
    const double load = 0.5;
    run<1, 0>(n_sms, n, load);
    run<2, 0>(n_sms, n, load);
    run<2, 1>(n_sms, n, load);
    run<2, 2>(n_sms, n, load);
    run<4, 2>(n_sms, n, load);
    run<8, 1>(n_sms, n, load);
    run<8, 2>(n_sms, n, load);
    run<16, 2>(n_sms, n, load);
    return 0;
}
