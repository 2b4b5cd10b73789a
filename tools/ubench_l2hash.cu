// ubench_l2hash.cu -- microbenchmark (not product code): counting 64-bit keys in global-memory
// hash tables that stay resident in L2, vs table size.  Keys carry the C4 duplication
// profile (~26% distinct).  Each "bin" owns a table of TS slots (u64 key, u32 count).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include <cuda_runtime.h>

#define CKE(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

constexpr unsigned long long EMPTY = ~0ull;

__device__ __forceinline__ uint32_t slot_of(uint64_t key, int lg) {
    return (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> (64 - lg));
}

// keys of bin b are keys[b*per .. (b+1)*per); table of bin b at T + b*TS (TS = 1 << lg)
template <int UNR>
__global__ void k_insert(const uint64_t* __restrict__ keys, uint64_t per, int lg, unsigned long long* T, uint32_t* C,
                         uint64_t nbins_keys) {
    const uint64_t TS = 1ull << lg;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x * UNR + threadIdx.x; i0 < nbins_keys;
         i0 += (uint64_t)gridDim.x * blockDim.x * UNR) {
        uint64_t kk[UNR];
        uint32_t s[UNR];
        uint64_t tb[UNR];
        unsigned long long old[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint64_t i = i0 + (uint64_t)u * blockDim.x;
            kk[u] = i < nbins_keys ? __ldcs(keys + i) : EMPTY;
            tb[u] = (i / per) * TS;
            s[u] = slot_of(kk[u], lg);
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u)
            old[u] = kk[u] != EMPTY ? atomicCAS(&T[tb[u] + s[u]], EMPTY, (unsigned long long)kk[u]) : 0ull;
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            if (kk[u] == EMPTY) continue;
            uint32_t ss = s[u];
            unsigned long long o = old[u];
            while (o != EMPTY && o != kk[u]) {
                ss = (ss + 1) & (uint32_t)(TS - 1);
                o = atomicCAS(&T[tb[u] + ss], EMPTY, (unsigned long long)kk[u]);
            }
            atomicAdd(&C[tb[u] + ss], 1u);
        }
    }
}

int main(int argc, char** argv) {
    const uint64_t total = argc > 1 ? strtoull(argv[1], 0, 10) : (1ull << 28);
    std::mt19937_64 rng(7);
    std::vector<uint64_t> keys;
    keys.reserve(total);
    // multiplicities: 70% of distinct keys once, 30% 10..34 times -> ~22% distinct
    while (keys.size() < total) {
        uint64_t key = rng() & ((1ull << 56) - 1);
        int cnt = (rng() % 10) < 7 ? 1 : 10 + (int)(rng() % 25);
        for (int t = 0; t < cnt && keys.size() < total; ++t) keys.push_back(key);
    }
    uint64_t* dk;
    CKE(cudaMalloc(&dk, total * 8));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    unsigned long long* T;
    uint32_t* C;
    CKE(cudaMalloc(&T, (total / 2 + (1 << 22)) * 8));
    CKE(cudaMalloc(&C, (total / 2 + (1 << 22)) * 4));
    // per-bin key counts: "per" keys per bin -> table of next_pow2(per/2) slots
    for (uint64_t per : {1ull << 14, 1ull << 16, 1ull << 18, 1ull << 20, 1ull << 22}) {
        // shuffle within bins (keys of one bin arrive in random order)
        std::vector<uint64_t> kk = keys;
        for (uint64_t b0 = 0; b0 < total; b0 += per)
            std::shuffle(kk.begin() + b0, kk.begin() + std::min(total, b0 + per), rng);
        CKE(cudaMemcpy(dk, kk.data(), total * 8, cudaMemcpyHostToDevice));
        int lg = 0;
        while ((1ull << lg) < per / 2) ++lg;
        const uint64_t nb = total / per;
        const uint64_t slots = nb << lg;
        // bins are processed in waves whose tables fit a budget; here: all at once vs waves
        for (uint64_t wave_bytes : {16ull << 20, 48ull << 20, 1ull << 40}) {
            const uint64_t bins_per_wave = std::max<uint64_t>(1, wave_bytes / ((12ull << lg)));
            float best = 1e9;
            for (int rep = 0; rep < 3; ++rep) {
                CKE(cudaMemset(T, 0xFF, slots * 8));
                CKE(cudaMemset(C, 0, slots * 4));
                cudaEventRecord(a);
                for (uint64_t b0 = 0; b0 < nb; b0 += bins_per_wave) {
                    const uint64_t b1 = std::min(nb, b0 + bins_per_wave);
                    const uint64_t n = (b1 - b0) * per;
                    const unsigned grid = (unsigned)std::min<uint64_t>(148 * 8, (n + 256 * 4 - 1) / (256 * 4));
                    k_insert<4><<<grid, 256>>>(dk + b0 * per, per, lg, T + (b0 << lg), C + (b0 << lg), n);
                }
                cudaEventRecord(b);
                CKE(cudaEventSynchronize(b));
                CKE(cudaGetLastError());
                float ms;
                cudaEventElapsedTime(&ms, a, b);
                best = std::min(best, ms);
            }
            std::vector<uint32_t> hc(slots);
            CKE(cudaMemcpy(hc.data(), C, slots * 4, cudaMemcpyDeviceToHost));
            uint64_t sum = 0, used = 0;
            for (auto c : hc) { sum += c; used += c != 0; }
            printf("per %8llu table %6.1f MB  wave %6.0f MB  %8.3f ms  %6.2f Gkeys/s  (sum %llu used %llu)\n",
                   (unsigned long long)per, (12.0 * (1ull << lg)) / 1e6,
                   std::min<double>(wave_bytes, 12.0 * slots) / 1e6, best, total / best / 1e6,
                   (unsigned long long)sum, (unsigned long long)used);
        }
    }
    return 0;
}
