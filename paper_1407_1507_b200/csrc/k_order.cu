// k_order.cu -- S9: global ascending order of the survivors (reading R8).
//
// The survivors of all bins are distinct keys in no particular order.  Up to four
// most-significant-digit passes partition them into key-ordered buckets: pass l takes the
// next D_l <= 8 bits of the 2k-bit key, over tiles that stay inside one bucket of pass l-1,
// until the average bucket holds at most cap/8 survivors (C4: 3 passes, 24 bits; canonical
// keys are skewed towards A-rich prefixes, so 16 bits leave ~28% of them in buckets above
// one chunk).  Every pass is a histogram (per-tile shared-memory counters, one global atomic per digit
// and tile), a scan, and a scatter in which each tile is first sorted by its digit in
// shared memory, so that it leaves as runs of consecutive addresses (an unsorted scatter
// of 8-12 byte items into millions of buckets is bound by partial-sector writes).  Then
// consecutive buckets are packed greedily into chunks of at most CAP pairs
// (k_greedy_chunks) and every chunk is sorted in shared memory and written straight into
// the caller's output at its offset.  A bucket holding more than CAP survivors is returned
// to the caller for the device-wide LSD path.
#include <algorithm>
#include <vector>

#include "kmc_device.cuh"
#include "kmc_internal.h"
#include "kmc_scan.cuh"

namespace kmc {

namespace {

constexpr int OC_NT = 512;
constexpr int OC_NW = OC_NT / 32;
constexpr int OT_NT = 512;

template <class K> struct OrderCap;
template <> struct OrderCap<uint64_t> { static constexpr int v = 4096; };
template <> struct OrderCap<K128> { static constexpr int v = 2048; };
template <class K> struct OrderTile;
template <> struct OrderTile<uint64_t> { static constexpr int v = 4096; };
template <> struct OrderTile<K128> { static constexpr int v = 2048; };

template <class K> constexpr size_t order_smem() {
    return 2 * (size_t)OrderCap<K>::v * (sizeof(K) + 4) + RADIX * OC_NW * 4 + 192;
}
template <class K> constexpr size_t otile_smem() {
    return (size_t)OrderTile<K>::v * (sizeof(K) + 4 + 1) + 3 * 256 * 4 + 64;
}

// bits [twok - D, twok) of a key (D <= 24)
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

// Histogram of the digit (bits [top - D, top)) over one tile per CTA.
template <class K>
__global__ void __launch_bounds__(OT_NT) k_ord_hist(const K* __restrict__ keys, const OrdTile* __restrict__ tiles,
                                                    int top, int D, uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[256];
    const OrdTile t = tiles[blockIdx.x];
    for (int d = threadIdx.x; d < (1 << D); d += OT_NT) h[d] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < t.n; i += OT_NT) atomicAdd(&h[hi_digit(ld_stream(keys + t.begin + i), top, D)], 1u);
    __syncthreads();
    for (int d = threadIdx.x; d < (1 << D); d += OT_NT)
        if (h[d]) atomicAdd(&hist[((uint64_t)t.bucket << D) + d], h[d]);
}

// Scatter of one tile per CTA by the digit: local counting sort in shared memory (shared
// atomics rank the items, a scan places the digits), one global atomic per digit reserves
// the tile's run, then the tile is written in digit order -- consecutive addresses per run.
template <class K>
__global__ void __launch_bounds__(OT_NT) k_ord_scatter(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                       const OrdTile* __restrict__ tiles, int top, int D,
                                                       uint32_t* __restrict__ cursor, K* __restrict__ kout,
                                                       uint32_t* __restrict__ vout) {
    constexpr int TI = OrderTile<K>::v, IPT = TI / OT_NT;
    extern __shared__ __align__(16) uint8_t osm[];
    K* sk = reinterpret_cast<K*>(osm);
    uint32_t* sv = reinterpret_cast<uint32_t*>(sk + TI);
    uint32_t* lh = sv + TI;     // 256: counts, then local offsets
    uint32_t* gb = lh + 256;    // 256: global base of the tile's run per digit
    uint32_t* wsum = gb + 256;  // scan scratch
    uint8_t* sd = reinterpret_cast<uint8_t*>(wsum + 64);
    const OrdTile t = tiles[blockIdx.x];
    const int nd = 1 << D;
    for (int d = threadIdx.x; d < 256; d += OT_NT) lh[d] = 0;
    __syncthreads();
    K key[IPT];
    uint32_t val[IPT], dr[IPT];
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
        const uint32_t i = threadIdx.x + u * OT_NT;
        dr[u] = 0xFFFFFFFFu;
        if (i < t.n) {
            key[u] = ld_stream(kin + t.begin + i);
            val[u] = __ldcs(vin + t.begin + i);
            const uint32_t d = hi_digit(key[u], top, D);
            dr[u] = (d << 16) | atomicAdd(&lh[d], 1u);  // rank < TI <= 4096
        }
    }
    __syncthreads();
    {
        const uint32_t c = threadIdx.x < (unsigned)nd ? lh[threadIdx.x] : 0u;
        const uint32_t ex = block_excl_sum<OT_NT, uint32_t>(c, wsum, nullptr);
        if (threadIdx.x < (unsigned)nd) {
            gb[threadIdx.x] = c ? atomicAdd(&cursor[((uint64_t)t.bucket << D) + threadIdx.x], c) : 0u;
            lh[threadIdx.x] = ex;
        }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
        if (dr[u] == 0xFFFFFFFFu) continue;
        const uint32_t d = dr[u] >> 16, pos = lh[d] + (dr[u] & 0xFFFFu);
        sk[pos] = key[u];
        sv[pos] = val[u];
        sd[pos] = (uint8_t)d;
    }
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < t.n; i += OT_NT) {
        const uint32_t d = sd[i];
        const uint64_t o = (uint64_t)gb[d] + (i - lh[d]);
        kout[o] = sk[i];
        vout[o] = sv[i];
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

// MSD levels: D_l <= 8 bits each, until the average bucket holds at most cap/8 survivors
int order_levels(uint64_t n, int k, int cap, int* D) {
    const int twok = 2 * k;
    int L = 0, bits = 0;
    do {
        D[L] = std::min(8, twok - bits);
        bits += D[L++];
    } while (bits < twok && L < 4 && (n >> bits) > (uint64_t)cap / 8);
    return L;
}

template <class K>
cudaError_t order_t(K* keys, uint32_t* vals, uint64_t n, int k, K* out_keys, uint32_t* out_vals,
                    const OrderScratch& os, cudaStream_t s, int* launches, std::vector<OrderSegment>* oversize,
                    void** seg_keys, uint32_t** seg_vals) {
    constexpr uint64_t TI = OrderTile<K>::v;
    const int twok = 2 * k;
    int D[4];
    const int L = order_levels(n, k, OrderCap<K>::v, D);
    cudaError_t e;
    const int osm = (int)otile_smem<K>();
    if ((e = cudaFuncSetAttribute(k_ord_scatter<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, osm))) return e;
    K* ck = keys;  // current layout
    uint32_t* cv = vals;
    K* ok = (K*)os.tmp_keys;  // the other buffers
    uint32_t* ov = os.tmp_vals;
    std::vector<uint32_t> counts(1, (uint32_t)n);  // items per bucket of the previous level
    uint64_t nbk = 1;                               // buckets of the previous level
    int top = twok;
    std::vector<OrdTile> tl;
    for (int l = 0; l < L; ++l) {
        // tiles of at most TI items inside each bucket of the previous level
        tl.clear();
        uint64_t b0 = 0;
        for (uint64_t b = 0; b < nbk; ++b) {
            const uint64_t c = counts[b];
            for (uint64_t o = 0; o < c; o += TI)
                tl.push_back(OrdTile{b0 + o, (uint32_t)std::min<uint64_t>(TI, c - o), (uint32_t)b});
            b0 += c;
        }
        const uint64_t nd = nbk << D[l];
        if (tl.empty()) continue;  // (n > 0, so only a pass after an empty previous one)
        if ((e = cudaMemcpyAsync(os.tiles, tl.data(), tl.size() * sizeof(OrdTile), cudaMemcpyHostToDevice, s)))
            return e;
        if ((e = cudaMemsetAsync(os.hist, 0, nd * 4, s))) return e;
        k_ord_hist<K><<<(unsigned)tl.size(), OT_NT, 0, s>>>(ck, os.tiles, top, D[l], os.hist);
        if ((e = cudaGetLastError())) return e;
        if ((e = scan_detail::scan_generic<uint32_t>(scan_detail::ArrayIn<uint32_t>{os.hist}, nd, os.start,
                                                     (uint32_t*)os.scan_temp, s, launches)))
            return e;
        if ((e = cudaMemcpyAsync(os.cursor, os.start, nd * 4, cudaMemcpyDeviceToDevice, s))) return e;
        k_ord_scatter<K><<<(unsigned)tl.size(), OT_NT, osm, s>>>(ck, cv, os.tiles, top, D[l], os.cursor, ok, ov);
        if ((e = cudaGetLastError())) return e;
        *launches += 2;
        std::swap(ck, ok);
        std::swap(cv, ov);
        top -= D[l];
        nbk = nd;
        if (l + 1 < L) {
            counts.resize(nd);
            if ((e = cudaMemcpyAsync(counts.data(), os.hist, nd * 4, cudaMemcpyDeviceToHost, s))) return e;
            if ((e = cudaStreamSynchronize(s))) return e;
        }
    }
    // ---- chunks of consecutive buckets, sorted in shared memory into the output
    if ((e = cudaMemsetAsync(os.counters, 0, 16, s))) return e;
    GreedyArgs ga{};
    ga.cnt = os.hist;
    ga.gstart = os.start;
    ga.n_digits = nbk;
    ga.chunks = os.chunks;
    ga.oversize = os.oversize;
    ga.counters = os.counters;
    ga.cap = OrderCap<K>::v;
    if ((e = launch_greedy_chunks(ga, n, s))) return e;
    if ((e = cudaMemcpyAsync(os.host, os.counters, 16, cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    const uint64_t n_chunks = os.host[0], n_over = os.host[1];
    const size_t sm = order_smem<K>();
    if ((e = cudaFuncSetAttribute(k_order_chunk_sort<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm))) return e;
    if (n_chunks)
        k_order_chunk_sort<K><<<(unsigned)n_chunks, OC_NT, sm, s>>>(ck, cv, os.chunks, twok, out_keys, out_vals);
    if ((e = cudaGetLastError())) return e;
    *launches += 2;
    oversize->clear();
    *seg_keys = ck;
    *seg_vals = cv;
    if (n_over) {
        std::vector<Chunk> ovs(n_over);
        if ((e = cudaMemcpyAsync(ovs.data(), os.oversize, n_over * sizeof(Chunk), cudaMemcpyDeviceToHost, s))) return e;
        if ((e = cudaStreamSynchronize(s))) return e;
        for (auto& c : ovs) oversize->push_back(OrderSegment{c.begin, c.n});
    }
    return cudaSuccess;
}

}  // namespace

int order_digit_bits(uint64_t n, int k) {
    int D[4];
    const int L = order_levels(n, k, k <= 32 ? OrderCap<uint64_t>::v : OrderCap<K128>::v, D);
    int bits = 0;
    for (int l = 0; l < L; ++l) bits += D[l];
    return bits;
}

uint64_t order_tile_items(int key_words) { return key_words == 1 ? OrderTile<uint64_t>::v : OrderTile<K128>::v; }

uint64_t order_max_tiles(uint64_t n, int k) {
    // at most one partial tile per bucket of the previous level beyond n / tile
    int D[4];
    const int L = order_levels(n, k, k <= 32 ? OrderCap<uint64_t>::v : OrderCap<K128>::v, D);
    int prev = 0;
    for (int l = 0; l + 1 < L; ++l) prev += D[l];
    return n / order_tile_items(k <= 32 ? 1 : 2) + (1ull << prev) + 1;
}

size_t order_scan_temp_bytes(uint64_t n_digits) { return scan_detail::scan_temp_elems<uint64_t>(n_digits) * 8; }

cudaError_t launch_order(int key_words, void* keys, uint32_t* vals, uint64_t n, int k, void* out_keys,
                         uint32_t* out_vals, const OrderScratch& os, cudaStream_t s, int* launches,
                         std::vector<OrderSegment>* oversize, void** seg_keys, uint32_t** seg_vals) {
    oversize->clear();
    *seg_keys = keys;
    *seg_vals = vals;
    if (n == 0) return cudaSuccess;
    if (n >= (1ull << 32)) return cudaErrorInvalidValue;
    if (key_words == 1)
        return order_t<uint64_t>((uint64_t*)keys, vals, n, k, (uint64_t*)out_keys, out_vals, os, s, launches, oversize,
                                 seg_keys, seg_vals);
    return order_t<K128>((K128*)keys, vals, n, k, (K128*)out_keys, out_vals, os, s, launches, oversize, seg_keys,
                         seg_vals);
}

}  // namespace kmc
