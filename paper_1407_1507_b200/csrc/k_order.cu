// k_order.cu -- S9: global ascending order of the survivors (reading R8).
//
// The survivors of all bins are distinct keys, so their top D bits make a good
// most-significant digit: (1) count the digit of every survivor, (2) exclusive scan of
// the 2^D digit counts, (3) pack consecutive digits greedily into chunks of at most CAP
// pairs (k_greedy_chunks) and initialise the scatter cursors, (4) scatter every (key,
// count) pair into its digit's range, (5) sort every chunk in shared memory and write it
// straight into the caller's output at the chunk's offset -- chunks are key ranges in
// ascending order, so the concatenation is the globally sorted list.  A digit holding
// more than CAP survivors is returned to the caller for the device-wide LSD path.
#include <algorithm>
#include <vector>

#include "kmc_device.cuh"
#include "kmc_internal.h"
#include "kmc_scan.cuh"

namespace kmc {

namespace {

constexpr int OR_NT = 256;
constexpr int OC_NT = 512;
constexpr int OC_NW = OC_NT / 32;

template <class K> struct OrderCap;
template <> struct OrderCap<uint64_t> { static constexpr int v = 4096; };
template <> struct OrderCap<K128> { static constexpr int v = 2048; };

template <class K> constexpr size_t order_smem() {
    return 2 * (size_t)OrderCap<K>::v * (sizeof(K) + 4) + RADIX * OC_NW * 4 + 192;
}

__device__ __forceinline__ uint32_t hi_digit(uint64_t key, int twok, int D) {
    return (uint32_t)(key >> (twok - D)) & ((1u << D) - 1);
}
__device__ __forceinline__ uint32_t hi_digit(const K128& key, int twok, int D) {
    const int sh = twok - D;
    uint64_t v;
    if (sh >= 64) v = key.hi >> (sh - 64);
    else if (sh == 0) v = key.lo;
    else v = (key.lo >> sh) | (key.hi << (64 - sh));
    return (uint32_t)v & ((1u << D) - 1);
}

template <class K>
__global__ void __launch_bounds__(OR_NT) k_order_count(const K* __restrict__ keys, uint64_t n, int twok, int D,
                                                       uint32_t* __restrict__ cnt) {
    const uint32_t lane = threadIdx.x & 31;
    for (uint64_t base = (uint64_t)blockIdx.x * OR_NT; base < n; base += (uint64_t)gridDim.x * OR_NT) {
        const uint64_t i = base + threadIdx.x;
        if (i < n) atomicAdd(&cnt[hi_digit(keys[i], twok, D)], 1u);
    }
}

constexpr int OS_U = 4;  // pairs per thread per step, carried together through the dependent steps
template <class K>
__global__ void __launch_bounds__(OR_NT) k_order_scatter(const K* __restrict__ keys, const uint32_t* __restrict__ vals,
                                                         uint64_t n, int twok, int D, uint32_t* __restrict__ cursor,
                                                         K* __restrict__ okeys, uint32_t* __restrict__ ovals) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t ltm = lanemask_lt();
    constexpr uint64_t STEP = (uint64_t)OR_NT * OS_U;
    for (uint64_t base = (uint64_t)blockIdx.x * STEP; base < n; base += (uint64_t)gridDim.x * STEP) {
        K key[OS_U];
        uint32_t val[OS_U], d[OS_U], slot[OS_U];
#pragma unroll
        for (int u = 0; u < OS_U; ++u) {
            const uint64_t i = base + (uint64_t)u * OR_NT + threadIdx.x;
            d[u] = 0xFFFFFFFFu;
            if (i < n) {
                key[u] = ld_stream(keys + i);
                val[u] = __ldcs(vals + i);
                d[u] = hi_digit(key[u], twok, D);
            }
        }
#pragma unroll
        for (int u = 0; u < OS_U; ++u) slot[u] = d[u] != 0xFFFFFFFFu ? atomicAdd(&cursor[d[u]], 1u) : 0u;
#pragma unroll
        for (int u = 0; u < OS_U; ++u) {
            if (d[u] == 0xFFFFFFFFu) continue;
            okeys[slot[u]] = key[u];
            ovals[slot[u]] = val[u];
        }
    }
}

template <class K>
__global__ void __launch_bounds__(OC_NT, 2) k_order_chunk_sort(const K* __restrict__ keys,
                                                               const uint32_t* __restrict__ vals,
                                                               const Chunk* __restrict__ chunks, int twok,
                                                               K* __restrict__ out_keys,
                                                               uint32_t* __restrict__ out_vals) {
    constexpr int CAP = OrderCap<K>::v;
    extern __shared__ __align__(16) uint8_t smem[];
    K* A = reinterpret_cast<K*>(smem);
    uint32_t* VA = reinterpret_cast<uint32_t*>(A + 2 * CAP);
    uint32_t* whist = VA + 2 * CAP;
    uint32_t* wsum = whist + RADIX * OC_NW;
    unsigned long long* red = reinterpret_cast<unsigned long long*>(wsum + 24);
    const Chunk c = chunks[blockIdx.x];
    const int n = (int)c.n;
    for (int i = threadIdx.x; i < n; i += OC_NT) {
        A[i] = keys[c.begin + i];
        VA[i] = vals[c.begin + i];
    }
    __syncthreads();
    block_sort_inplace<K, OC_NT, CAP / OC_NT, true>(A, VA, n, twok, whist, wsum, red);
    for (int i = threadIdx.x; i < n; i += OC_NT) {
        out_keys[c.begin + i] = A[i];
        out_vals[c.begin + i] = VA[i];
    }
}

template <class K>
cudaError_t order_t(const K* keys, const uint32_t* vals, uint64_t n, int k, K* out_keys, uint32_t* out_vals,
                    const OrderScratch& os, cudaStream_t s, int* launches, std::vector<OrderSegment>* oversize) {
    const int twok = 2 * k;
    const int D = order_digit_bits(n, k);
    const uint64_t nd = 1ull << D;
    cudaError_t e;
    if ((e = cudaMemsetAsync(os.cnt, 0, nd * 4, s))) return e;
    if ((e = cudaMemsetAsync(os.counters, 0, 16, s))) return e;
    const unsigned grid = (unsigned)std::min<uint64_t>((n + OR_NT - 1) / OR_NT, 148ull * 16);
    k_order_count<K><<<grid, OR_NT, 0, s>>>(keys, n, twok, D, os.cnt);
    if ((e = cudaGetLastError())) return e;
    if ((e = scan_detail::scan_generic<uint32_t>(scan_detail::ArrayIn<uint32_t>{os.cnt}, nd, os.start,
                                                 (uint32_t*)os.scan_temp, s, launches)))
        return e;
    GreedyArgs ga{};
    ga.cnt = os.cnt;
    ga.gstart = os.start;
    ga.n_digits = nd;
    ga.cursor = os.cursor;
    ga.cursor_abs = 1;
    ga.chunks = os.chunks;
    ga.oversize = os.oversize;
    ga.counters = os.counters;
    ga.cap = OrderCap<K>::v;
    if ((e = launch_greedy_chunks(ga, greedy_segments(nd), s))) return e;
    const unsigned sgrid = (unsigned)std::min<uint64_t>((n + OR_NT * OS_U - 1) / (OR_NT * OS_U), 148ull * 8);
    k_order_scatter<K><<<sgrid, OR_NT, 0, s>>>(keys, vals, n, twok, D, os.cursor, (K*)os.tmp_keys, os.tmp_vals);
    if ((e = cudaGetLastError())) return e;
    if ((e = cudaMemcpyAsync(os.host, os.counters, 16, cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    const uint64_t n_chunks = os.host[0], n_over = os.host[1];
    const size_t sm = order_smem<K>();
    if ((e = cudaFuncSetAttribute(k_order_chunk_sort<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm))) return e;
    if (n_chunks)
        k_order_chunk_sort<K><<<(unsigned)n_chunks, OC_NT, sm, s>>>((const K*)os.tmp_keys, os.tmp_vals, os.chunks,
                                                                   twok, out_keys, out_vals);
    if ((e = cudaGetLastError())) return e;
    *launches += 5;
    oversize->clear();
    if (n_over) {
        std::vector<Chunk> ov(n_over);
        if ((e = cudaMemcpyAsync(ov.data(), os.oversize, n_over * sizeof(Chunk), cudaMemcpyDeviceToHost, s))) return e;
        if ((e = cudaStreamSynchronize(s))) return e;
        for (auto& c : ov) oversize->push_back(OrderSegment{c.begin, c.n});
    }
    return cudaSuccess;
}

}  // namespace

int order_digit_bits(uint64_t n, int k) {
    // about cap/64 survivors per digit on average (canonical keys of AT-rich genomes put
    // ~10x the mean on prefixes like A^9); 1 <= D <= min(24, 2k)
    const uint64_t per = (uint64_t)(k <= 32 ? OrderCap<uint64_t>::v : OrderCap<K128>::v) / 64;
    int D = 1;
    while (D < 24 && (n >> D) > per) ++D;
    return std::min(D, 2 * k);
}

size_t order_scan_temp_bytes(uint64_t n_digits) { return scan_detail::scan_temp_elems<uint64_t>(n_digits) * 8; }

cudaError_t launch_order(int key_words, const void* keys, const uint32_t* vals, uint64_t n, int k, void* out_keys,
                         uint32_t* out_vals, const OrderScratch& os, cudaStream_t s, int* launches,
                         std::vector<OrderSegment>* oversize) {
    oversize->clear();
    if (n == 0) return cudaSuccess;
    if (n >= (1ull << 32)) return cudaErrorInvalidValue;
    if (key_words == 1)
        return order_t<uint64_t>((const uint64_t*)keys, vals, n, k, (uint64_t*)out_keys, out_vals, os, s, launches,
                                 oversize);
    return order_t<K128>((const K128*)keys, vals, n, k, (K128*)out_keys, out_vals, os, s, launches, oversize);
}

}  // namespace kmc
