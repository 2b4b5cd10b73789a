// ubench_chunk.cu -- microbenchmark of per-chunk counting strategies (not product code).
// Chunks of ~5.5K 56-bit keys with the C4 duplication profile (~27% distinct) are counted
// by (a) the product's in-place SMEM LSD radix sort + bitmask RLE and (b) SMEM hash tables.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I../paper_1407_1507_b200/csrc
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <random>
#include <algorithm>
#include "kmc_device.cuh"

using namespace kmc;

constexpr int NT = 512;
constexpr int CAP = 6144;

struct Chunk { uint64_t begin; uint32_t n, pad; };

template <int NB>
__global__ void __launch_bounds__(NT, 2) k_sort(const uint64_t* keys, const Chunk* chunks, uint32_t ci,
                                                 uint64_t* sk, uint32_t* sc, unsigned long long* gs) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t* A = reinterpret_cast<uint64_t*>(smem);
    uint64_t* B = A + CAP;
    uint32_t* whist = reinterpret_cast<uint32_t*>(B + CAP);
    uint32_t* wsum = whist + RADIX * (NT / 32);
    unsigned long long* red = reinterpret_cast<unsigned long long*>(wsum + 24);
    unsigned long long* bcast = red + 4;
    unsigned int* scnt = reinterpret_cast<unsigned int*>(bcast + 1);
    const Chunk c = chunks[blockIdx.x];
    const int n = (int)c.n;
    for (int i = threadIdx.x; i < n; i += NT) A[i] = keys[c.begin + i];
    __syncthreads();
    block_sort_inplace<uint64_t, NT, CAP / NT, false>(A, nullptr, n, NB, whist, wsum, red);
    block_rle_bitmask<uint64_t, NT>(A, n, reinterpret_cast<uint32_t*>(B), ci, 0xFFFFFFFFu, sk, sc, gs, wsum, scnt,
                                    bcast, 0, 1, 2, 3);
}

// ---- hash table count: TS slots of (u64 key, u32 count), linear probing
template <int TS, int UNR>
__global__ void __launch_bounds__(NT, 2) k_hash(const uint64_t* keys, const Chunk* chunks, uint32_t ci,
                                                 uint64_t* sk, uint32_t* sc, unsigned long long* gs) {
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t* T = reinterpret_cast<uint64_t*>(smem);
    uint32_t* C = reinterpret_cast<uint32_t*>(T + TS);
    __shared__ unsigned int scnt[4];
    const Chunk c = chunks[blockIdx.x];
    const int n = (int)c.n;
    const uint64_t EMPTY = ~0ull;
    for (int i = threadIdx.x; i < TS / 2; i += NT) {
        reinterpret_cast<uint4*>(T)[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
    }
    for (int i = threadIdx.x; i < TS / 4; i += NT) reinterpret_cast<uint4*>(C)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x < 4) scnt[threadIdx.x] = 0;
    __syncthreads();
    const uint64_t* src = keys + c.begin;
    constexpr int SH = 64 - __builtin_ctz(TS);
    for (int i0 = threadIdx.x; i0 < n; i0 += NT * UNR) {
        uint64_t kk[UNR];
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const int i = i0 + u * NT;
            kk[u] = i < n ? __ldcs(src + i) : EMPTY;
        }
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint64_t key = kk[u];
            if (key == EMPTY) continue;
            uint32_t s = (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> SH);
            while (true) {
                const uint64_t cur = *reinterpret_cast<volatile uint64_t*>(&T[s]);
                if (cur == key) break;
                if (cur == EMPTY) {
                    const unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long*>(&T[s]), EMPTY, key);
                    if (old == EMPTY || old == key) break;
                }
                s = (s + 1) & (TS - 1);
            }
            atomicAdd(&C[s], 1u);
        }
    }
    __syncthreads();
    const int lane = threadIdx.x & 31;
    const uint32_t ltm = lanemask_lt();
    uint32_t uniq = 0, below = 0;
    for (int s = threadIdx.x; s < TS; s += NT) {
        const uint32_t cnt = C[s];
        uniq += cnt != 0;
        const bool keep = cnt >= ci;
        below += (cnt != 0 && !keep);
        const uint32_t b = __ballot_sync(0xffffffffu, keep);
        if (b) {
            unsigned long long slot = 0;
            if (lane == 0) slot = atomicAdd(&gs[0], (unsigned long long)__popc(b));
            slot = __shfl_sync(0xffffffffu, slot, 0) + __popc(b & ltm);
            if (keep) { sk[slot] = T[s]; sc[slot] = cnt; }
        }
    }
    uniq = __reduce_add_sync(0xffffffffu, uniq);
    below = __reduce_add_sync(0xffffffffu, below);
    if (lane == 0) { atomicAdd(&scnt[1], uniq); atomicAdd(&scnt[2], below); }
    __syncthreads();
    if (threadIdx.x == 0) { atomicAdd(&gs[1], (unsigned long long)scnt[1]); atomicAdd(&gs[2], (unsigned long long)scnt[2]); }
}


// ---- partition into NG warp-owned groups (one SMEM pass), then warp-private hash tables
template <int NTT, int TS, int CAPK>
__global__ void __launch_bounds__(NTT, 1) k_whash(const uint64_t* keys, const Chunk* chunks, uint32_t ci,
                                                  uint64_t* sk, uint32_t* sc, unsigned long long* gs) {
    constexpr int NW = NTT / 32, KPT = CAPK / NTT, SAFE = TS - TS / 8;
    extern __shared__ __align__(16) uint8_t smem[];
    uint64_t* K = reinterpret_cast<uint64_t*>(smem);                  // CAPK
    uint64_t* T = K + CAPK;                                            // NW * TS
    uint32_t* C = reinterpret_cast<uint32_t*>(T + NW * TS);            // NW * TS
    __shared__ uint32_t wh[NW * NW];                                   // [warp][group] counters
    __shared__ uint32_t gstart[NW + 1];
    __shared__ uint32_t wsum[NW + 1];
    __shared__ unsigned int scnt[4];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t ltm = lanemask_lt();
    const uint64_t EMPTY = ~0ull;
    const Chunk c = chunks[blockIdx.x];
    const int n = (int)c.n;
    const int rounds = (n + NTT - 1) / NTT;
    const int wbase = warp * rounds * 32;
    for (int i = threadIdx.x; i < NW * NW; i += NTT) wh[i] = 0;
    for (int i = threadIdx.x; i < NW * TS / 2; i += NTT) reinterpret_cast<uint4*>(T)[i] = make_uint4(~0u, ~0u, ~0u, ~0u);
    for (int i = threadIdx.x; i < NW * TS / 4; i += NTT) reinterpret_cast<uint4*>(C)[i] = make_uint4(0, 0, 0, 0);
    if (threadIdx.x < 4) scnt[threadIdx.x] = 0;
    __syncthreads();
    uint64_t key[KPT];
    uint32_t rank[KPT];
    const uint64_t* src = keys + c.begin;
#pragma unroll
    for (int r = 0; r < KPT; ++r) {
        if (r >= rounds) break;
        const int i = wbase + r * 32 + lane;
        key[r] = i < n ? src[i] : EMPTY;
    }
    uint32_t* myh = wh + warp * NW;
#pragma unroll
    for (int r = 0; r < KPT; ++r) {
        if (r >= rounds) break;
        const bool ok = key[r] != EMPTY;
        const uint32_t g = ok ? (uint32_t)((key[r] * 0x9E3779B97F4A7C15ull) >> 60) % NW : (uint32_t)(NW + lane);
        const uint32_t peers = __match_any_sync(0xffffffffu, g);
        const uint32_t below = __popc(peers & ltm);
        uint32_t pre = 0;
        if (ok) pre = myh[g];
        __syncwarp();
        if (ok && below == 0) myh[g] = pre + __popc(peers);
        __syncwarp();
        rank[r] = ok ? ((pre + below) << 8) | g : 0xFFFFFFFFu;
    }
    __syncthreads();
    // group-major exclusive scan of wh: thread t < NW owns group t
    if (threadIdx.x < 32) {
        uint32_t tot = 0;
        uint32_t cw[NW];
        if (lane < NW) {
#pragma unroll
            for (int w = 0; w < NW; ++w) { cw[w] = wh[w * NW + lane]; tot += cw[w]; }
        }
        uint32_t inc = warp_incl_sum(lane < NW ? tot : 0u);
        uint32_t run = inc - (lane < NW ? tot : 0u);
        if (lane < NW) {
            gstart[lane] = run;
#pragma unroll
            for (int w = 0; w < NW; ++w) { wh[w * NW + lane] = run; run += cw[w]; }
        }
        if (lane == NW - 1) gstart[NW] = inc;
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < KPT; ++r) {
        if (r >= rounds) break;
        if (rank[r] != 0xFFFFFFFFu) K[myh[rank[r] & 0xFF] + (rank[r] >> 8)] = key[r];
    }
    __syncthreads();
    // warp w: group w into its table
    const int g0 = gstart[warp], m = gstart[warp + 1] - g0;
    uint64_t* TT = T + warp * TS;
    uint32_t* CC = C + warp * TS;
    if (m > SAFE) { if (lane == 0) atomicAdd(&gs[3], 1ull); }
    else {
        for (int b = 0; b < m; b += 32) {
            const bool valid = b + lane < m;
            const uint64_t kk = valid ? K[g0 + b + lane] : EMPTY;
            const uint32_t peers = __match_any_sync(0xffffffffu, kk);
            bool todo = valid && (peers & ltm) == 0;
            const uint32_t cnt = __popc(peers);
            uint32_t s = (uint32_t)((kk * 0x9E3779B97F4A7C15ull) >> 40) & (TS - 1);
            while (__any_sync(0xffffffffu, todo)) {
                const uint32_t sp = __match_any_sync(0xffffffffu, todo ? s : (0x80000000u | lane));
                if (todo && (sp & ltm) == 0) {
                    const uint64_t cur = TT[s];
                    if (cur == kk) { CC[s] += cnt; todo = false; }
                    else if (cur == EMPTY) { TT[s] = kk; CC[s] = cnt; todo = false; }
                    else s = (s + 1) & (TS - 1);
                }
                __syncwarp();
            }
        }
    }
    __syncwarp();
    uint32_t uniq = 0, below = 0;
    for (int s = lane; s < TS; s += 32) {
        const uint32_t cnt = CC[s];
        uniq += cnt != 0;
        const bool keep = cnt >= ci;
        below += (cnt != 0 && !keep);
        const uint32_t bb = __ballot_sync(0xffffffffu, keep);
        if (bb) {
            unsigned long long slot = 0;
            if (lane == 0) slot = atomicAdd(&gs[0], (unsigned long long)__popc(bb));
            slot = __shfl_sync(0xffffffffu, slot, 0) + __popc(bb & ltm);
            if (keep) { sk[slot] = TT[s]; sc[slot] = cnt; }
        }
    }
    uniq = __reduce_add_sync(0xffffffffu, uniq);
    below = __reduce_add_sync(0xffffffffu, below);
    if (lane == 0) { atomicAdd(&scnt[1], uniq); atomicAdd(&scnt[2], below); }
    __syncthreads();
    if (threadIdx.x == 0) { atomicAdd(&gs[1], (unsigned long long)scnt[1]); atomicAdd(&gs[2], (unsigned long long)scnt[2]); }
}


// ---- TMA-prefetched, persistent CTA hash count (1 CTA/SM, double-buffered chunk staging)
__device__ __forceinline__ uint32_t ub_smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void ub_mbar_init(uint64_t* m, uint32_t cnt) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(ub_smem_u32(m)), "r"(cnt) : "memory");
}
__device__ __forceinline__ void ub_mbar_expect_tx(uint64_t* m, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(ub_smem_u32(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"(ub_smem_u32(dst)), "l"(src), "r"(bytes), "r"(ub_smem_u32(m)) : "memory");
}
__device__ __forceinline__ void ub_mbar_wait(uint64_t* m, uint32_t parity) {
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra W;\n}"
                 :: "r"(ub_smem_u32(m)), "r"(parity) : "memory");
}

template <int NTT, int TSMAX>
__global__ void __launch_bounds__(NTT, 1) k_hash_tma(const uint64_t* keys, const Chunk* chunks, int nch, uint32_t ci,
                                                     uint64_t* sk, uint32_t* sc, unsigned long long* gs) {
    constexpr int NW = NTT / 32, SPT = TSMAX / NTT;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* T = reinterpret_cast<uint64_t*>(smem);
    uint32_t* C = reinterpret_cast<uint32_t*>(T + TSMAX);
    uint64_t* S[2] = {reinterpret_cast<uint64_t*>(C + TSMAX), reinterpret_cast<uint64_t*>(C + TSMAX) + CAP + 2};
    uint64_t* mbar = S[1] + CAP + 2;
    __shared__ uint32_t wk[NW];
    __shared__ unsigned long long wb[NW];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t ltm = lanemask_lt();
    const uint64_t EMPTY = ~0ull;
    for (int i = threadIdx.x; i < TSMAX; i += NTT) { T[i] = EMPTY; C[i] = 0; }
    auto issue = [&](int cc, int b) {
        const Chunk ch = chunks[cc];
        const uint64_t a0 = ch.begin & ~1ull;  // 16-byte aligned start
        const uint32_t bytes = (uint32_t)(((ch.begin + ch.n - a0) * 8 + 15) & ~15ull);
        ub_mbar_expect_tx(mbar + b, bytes);
        bulk_g2s(S[b], keys + a0, bytes, mbar + b);
    };
    if (threadIdx.x == 0) {
        ub_mbar_init(mbar, 1);
        ub_mbar_init(mbar + 1, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0 && (int)blockIdx.x < nch) issue(blockIdx.x, 0);
    uint32_t uniq = 0, below = 0;
    for (int it = 0;; ++it) {
        const int cc = blockIdx.x + it * gridDim.x;
        if (cc >= nch) break;
        const int b = it & 1;
        if (threadIdx.x == 0 && cc + (int)gridDim.x < nch) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(cc + gridDim.x, b ^ 1);
        }
        const Chunk ch = chunks[cc];
        const int n = (int)ch.n, off = (int)(ch.begin & 1);
        int lg = 6;
        while ((1 << lg) < n + n / 3) ++lg;
        const int TS = 1 << lg;
        ub_mbar_wait(mbar + b, (it >> 1) & 1);
        const uint64_t* src = S[b] + off;
        for (int i = threadIdx.x; i < n; i += NTT) {
            const uint64_t key = src[i];
            uint32_t s = (uint32_t)((key * 0x9E3779B97F4A7C15ull) >> (64 - lg));
            while (true) {
                const uint64_t cur = *reinterpret_cast<volatile uint64_t*>(&T[s]);
                if (cur == key) break;
                if (cur == EMPTY) {
                    const unsigned long long old = atomicCAS(reinterpret_cast<unsigned long long*>(&T[s]), EMPTY, key);
                    if (old == EMPTY || old == key) break;
                }
                s = (s + 1) & (TS - 1);
            }
            atomicAdd(&C[s], 1u);
        }
        __syncthreads();
        // emission: count kept per warp, one global reservation per CTA, then write + clear
        uint32_t cv[SPT];
        uint32_t keep = 0;
#pragma unroll
        for (int j = 0; j < SPT; ++j) {
            const int s = j * NTT + threadIdx.x;
            cv[j] = s < TS ? C[s] : 0u;
            uniq += cv[j] != 0;
            const bool kp = cv[j] >= ci;
            below += (cv[j] != 0 && !kp);
            keep += kp;
        }
        keep = __reduce_add_sync(0xffffffffu, keep);
        if (lane == 0) wk[warp] = keep;
        __syncthreads();
        if (warp == 0) {
            const uint32_t kw = lane < NW ? wk[lane] : 0u;
            const uint32_t inc = warp_incl_sum(kw);
            unsigned long long b0 = 0;
            if (lane == NW - 1 && inc) b0 = atomicAdd(&gs[0], (unsigned long long)inc);
            b0 = __shfl_sync(0xffffffffu, b0, NW - 1);
            if (lane < NW) wb[lane] = b0 + inc - kw;
        }
        __syncthreads();
        unsigned long long o = wb[warp];
#pragma unroll
        for (int j = 0; j < SPT; ++j) {
            const int s = j * NTT + threadIdx.x;
            if (j * NTT >= TS) break;
            const bool kp = cv[j] >= ci;
            const uint32_t bb = __ballot_sync(0xffffffffu, kp);
            if (kp) { sk[o + __popc(bb & ltm)] = T[s]; sc[o + __popc(bb & ltm)] = cv[j]; }
            o += __popc(bb);
            if (s < TS) { T[s] = EMPTY; C[s] = 0; }
        }
        __syncthreads();
    }
    uniq = __reduce_add_sync(0xffffffffu, uniq);
    below = __reduce_add_sync(0xffffffffu, below);
    if (lane == 0) { atomicAdd(&gs[1], (unsigned long long)uniq); atomicAdd(&gs[2], (unsigned long long)below); }
}

#define CKE(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

int main(int argc, char** argv) {
    const int nch = argc > 1 ? atoi(argv[1]) : 20000;
    std::mt19937_64 rng(12345);
    std::vector<uint64_t> keys;
    std::vector<Chunk> chunks;
    uint64_t tot_uniq = 0, tot_keep = 0;
    for (int c = 0; c < nch; ++c) {
        Chunk ch{keys.size(), 0, 0};
        std::vector<uint64_t> v;
        // 70% of distinct keys: errors (count 1); 30%: true k-mers ~ Poisson(22)-ish
        while (v.size() < 5400) {
            uint64_t key = rng() & ((1ull << 56) - 1);
            int cnt = (rng() % 10) < 7 ? 1 : 10 + (int)(rng() % 25);
            if (v.size() + cnt > CAP) break;
            for (int t = 0; t < cnt; ++t) v.push_back(key);
            ++tot_uniq;
            tot_keep += cnt >= 2;
        }
        std::shuffle(v.begin(), v.end(), rng);
        ch.n = (uint32_t)v.size();
        keys.insert(keys.end(), v.begin(), v.end());
        chunks.push_back(ch);
    }
    printf("chunks %d keys %zu unique %llu keep %llu\n", nch, keys.size(), (unsigned long long)tot_uniq,
           (unsigned long long)tot_keep);
    uint64_t *dk, *sk;
    uint32_t* sc;
    Chunk* dc;
    unsigned long long* gs;
    CKE(cudaMalloc(&dk, keys.size() * 8));
    CKE(cudaMalloc(&sk, keys.size() * 8));
    CKE(cudaMalloc(&sc, keys.size() * 4));
    CKE(cudaMalloc(&dc, chunks.size() * sizeof(Chunk)));
    CKE(cudaMalloc(&gs, 64));
    CKE(cudaMemcpy(dk, keys.data(), keys.size() * 8, cudaMemcpyHostToDevice));
    CKE(cudaMemcpy(dc, chunks.data(), chunks.size() * sizeof(Chunk), cudaMemcpyHostToDevice));
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto launch) {
        float best = 1e9;
        unsigned long long h[4] = {0, 0, 0, 0};
        for (int rep = 0; rep < 5; ++rep) {
            CKE(cudaMemset(gs, 0, 64));
            cudaEventRecord(a);
            launch();
            cudaEventRecord(b);
            CKE(cudaEventSynchronize(b));
            CKE(cudaGetLastError());
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = std::min(best, ms);
            CKE(cudaMemcpy(h, gs, 32, cudaMemcpyDeviceToHost));
        }
        printf("%-16s %8.3f ms  %6.2f Gkeys/s  surv %llu uniq %llu below %llu fallback %llu\n", name, best,
               keys.size() / best / 1e6, h[0], h[1], h[2], h[3]);
    };
    const size_t sm_sort = 2 * (size_t)CAP * 8 + RADIX * (NT / 32) * 4 + 128 + 64;
#define SORTV(NB) CKE(cudaFuncSetAttribute(k_sort<NB>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_sort)); \
    run("sort" #NB, [&] { k_sort<NB><<<nch, NT, sm_sort>>>(dk, dc, 2, sk, sc, gs); });
    SORTV(0) SORTV(8) SORTV(16) SORTV(32) SORTV(56)
    const size_t sm_h = 8192 * 12;
    CKE(cudaFuncSetAttribute(k_hash<8192, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_h));
    CKE(cudaFuncSetAttribute(k_hash<8192, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm_h));
    run("hash8k u1", [&] { k_hash<8192, 1><<<nch, NT, sm_h>>>(dk, dc, 2, sk, sc, gs); });
    run("hash8k u4", [&] { k_hash<8192, 4><<<nch, NT, sm_h>>>(dk, dc, 2, sk, sc, gs); });

    {
        const size_t sm = 6144 * 8 + 16 * 512 * 12;
        CKE(cudaFuncSetAttribute(k_whash<512, 512, 6144>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        run("whash 16w512", [&] { k_whash<512, 512, 6144><<<nch, 512, sm>>>(dk, dc, 2, sk, sc, gs); });
    }

    {
        const size_t sm = 8192 * 12 + 2 * (CAP + 2) * 8 + 16;
        CKE(cudaFuncSetAttribute(k_hash_tma<1024, 8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        run("hash_tma 1024", [&] { k_hash_tma<1024, 8192><<<148, 1024, sm>>>(dk, dc, nch, 2, sk, sc, gs); });
        CKE(cudaFuncSetAttribute(k_hash_tma<512, 8192>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
        run("hash_tma 512", [&] { k_hash_tma<512, 8192><<<148, 512, sm>>>(dk, dc, nch, 2, sk, sc, gs); });
    }
    return 0;
}
