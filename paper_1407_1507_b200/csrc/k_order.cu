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
#ifndef KMC_ORD_TILE
#define KMC_ORD_TILE 6144  // C4 S9: 2048 -> 5.97 ms, 4096 -> 5.75, 6144 -> 5.63
#endif
template <> struct OrderTile<uint64_t> { static constexpr int v = KMC_ORD_TILE; };
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
                                                    const uint64_t* __restrict__ n_tiles, int top, int D,
                                                    uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[256];
    if (blockIdx.x >= *n_tiles) return;
    const OrdTile t = tiles[blockIdx.x];
    for (int d = threadIdx.x; d < (1 << D); d += OT_NT) h[d] = 0;
    __syncthreads();
    constexpr int HU = 4;  // loads in flight per thread
    for (uint32_t i0 = threadIdx.x; i0 < t.n; i0 += HU * OT_NT) {
        K kk[HU];
#pragma unroll
        for (int u = 0; u < HU; ++u) {
            const uint32_t i = i0 + u * OT_NT;
            if (i < t.n) kk[u] = ld_stream(keys + t.begin + i);
        }
#pragma unroll
        for (int u = 0; u < HU; ++u)
            if (i0 + u * OT_NT < t.n) atomicAdd(&h[hi_digit(kk[u], top, D)], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < (1 << D); d += OT_NT)
        if (h[d]) atomicAdd(&hist[((uint64_t)t.bucket << D) + d], h[d]);
}

// Scatter of one tile per CTA by the digit: local counting sort in shared memory (shared
// atomics rank the items, a scan places the digits), one global atomic per digit reserves
// the tile's run, then the tile is written in digit order -- consecutive addresses per run.
template <class K>
__global__ void __launch_bounds__(OT_NT) k_ord_scatter(const K* __restrict__ kin, const uint32_t* __restrict__ vin,
                                                       const OrdTile* __restrict__ tiles,
                                                       const uint64_t* __restrict__ n_tiles, int top, int D,
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
    if (blockIdx.x >= *n_tiles) return;
    const OrdTile t = tiles[blockIdx.x];
    const int nd = 1 << D;
    for (int d = threadIdx.x; d < 256; d += OT_NT) lh[d] = 0;
    __syncthreads();
    K key[IPT];
    uint32_t val[IPT], dr[IPT];
#pragma unroll
    for (int u = 0; u < IPT; ++u) {  // every load of the tile in flight before the first use
        const uint32_t i = threadIdx.x + u * OT_NT;
        if (i < t.n) {
            key[u] = ld_stream(kin + t.begin + i);
            val[u] = __ldcs(vin + t.begin + i);
        }
    }
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
        const uint32_t i = threadIdx.x + u * OT_NT;
        dr[u] = 0xFFFFFFFFu;
        if (i < t.n) {
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

// ---- after the MSD passes (64-bit keys): most buckets hold a few survivors (7 on average
// at C4, 221 at most), so they are sorted by warps in registers instead of by CTA radix
// sorts.  k_ord_classify puts every bucket into a list by size: "groups" of consecutive
// buckets of <= 32 survivors that start in the same 32-item window of the array (so a
// group holds < 64 items; sorting the union of whole, consecutive buckets by the full key
// is the same as sorting each bucket), buckets of 33-64 / 65-128 / 129-256 survivors, up to
// the chunk capacity (CTA radix sort), and above it (oversize, device LSD).  Lists are
// appended with one atomic per CTA and list; their order is irrelevant.
constexpr int WS_NT = 256;
constexpr uint64_t ORD_GROUPS = 8;  // S9's final sorts in this many bucket groups (copy overlap)

// Buckets [b0, b1) of nbk (a group of consecutive buckets: runs of small buckets stop at b1);
// the group's warp-sort lists in wl[0, 2 (b1 - b0)), its CTA chunks in big[0, b1 - b0), its
// class counters in counters[0..4]; oversize buckets of every group share one list (over_ctr).
__global__ void __launch_bounds__(WS_NT) k_ord_classify(const uint32_t* __restrict__ cnt,
                                                        const uint32_t* __restrict__ start, uint64_t nbk,
                                                        uint32_t n, uint32_t cap, uint2* __restrict__ wl,
                                                        Chunk* __restrict__ big, Chunk* __restrict__ over,
                                                        unsigned long long* __restrict__ counters, uint64_t b0,
                                                        uint64_t b1, unsigned long long* __restrict__ over_ctr) {
    const uint64_t wn = b1 - b0;
    __shared__ unsigned long long wsum64[WS_NT / 32 + 1];
    __shared__ unsigned long long base[6];
    const uint64_t d = b0 + (uint64_t)blockIdx.x * WS_NT + threadIdx.x;
    int cls = -1;  // 0/1/2/3: warp sort of 32/64/128/256 items, 4: CTA sort, 5: oversize
    uint32_t st = 0, sz = 0;
    if (d < b1) {
        const uint32_t c = cnt[d];
        st = start[d];
        if (c > 32) {
            sz = c;
            cls = c <= 64 ? 1 : c <= 128 ? 2 : c <= 256 ? 3 : c <= cap ? 4 : 5;
        } else {
            const bool lead = d == b0 || cnt[d - 1] > 32 || (start[d - 1] >> 5) != (st >> 5);
            if (lead) {
                uint64_t e = d + 1;
                while (e < b1 && cnt[e] <= 32 && (start[e] >> 5) == (st >> 5)) ++e;
                sz = (e < nbk ? start[e] : n) - st;
                if (sz) cls = sz <= 32 ? 0 : 1;
            }
        }
    }
    // one block scan of the six class counters packed in 10-bit fields of a uint64
    unsigned long long tot;
    const unsigned long long off =
        block_excl_sum<WS_NT, unsigned long long>(cls >= 0 ? 1ull << (10 * cls) : 0ull, wsum64, &tot);
    if (threadIdx.x < 6) {
        const uint32_t t = (uint32_t)(tot >> (10 * threadIdx.x)) & 1023u;
        unsigned long long* ctr = threadIdx.x == 5 ? over_ctr : &counters[threadIdx.x];
        base[threadIdx.x] = t ? atomicAdd(ctr, (unsigned long long)t) : 0ull;
    }
    __syncthreads();
    if (cls >= 0) {
        const Chunk ch{st, sz, 0};
        const uint64_t q = base[cls] + ((off >> (10 * cls)) & 1023u);
        // warp-sort lists in 2 nbk slots: sizes <= 32 / <= 64 from both ends of the first half
        // (together at most one item per bucket), <= 128 / <= 256 from both ends of the second
        if (cls == 0) wl[q] = make_uint2(st, sz);
        else if (cls == 1) wl[wn - 1 - q] = make_uint2(st, sz);
        else if (cls == 2) wl[wn + q] = make_uint2(st, sz);
        else if (cls == 3) wl[2 * wn - 1 - q] = make_uint2(st, sz);
        else if (cls == 4) big[q] = ch;
        else over[q] = ch;
    }
}

// One warp sorts one list item of <= 32 R (key, count) pairs in registers: element
// i = lane + 32 r, padded with the all-ones key (never a canonical k-mer); bitonic network,
// exchanges across lanes by shuffles (distance < 32) or between a lane's registers.
// PACK (2k <= 56): the network sorts key << 8 | i (one 64-bit word per element) and the
// counts follow through a shared-memory permutation afterwards.
template <int R, bool PACK>
__global__ void __launch_bounds__(WS_NT) k_ord_wsort(const uint64_t* __restrict__ keys,
                                                     const uint32_t* __restrict__ vals, const uint2* __restrict__ items,
                                                     uint64_t n_items, int dir, uint64_t* __restrict__ out_keys,
                                                     uint32_t* __restrict__ out_vals) {
    constexpr int N = 32 * R;
    __shared__ uint32_t svals[PACK ? WS_NT / 32 : 1][PACK ? N : 1];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const uint64_t w = (uint64_t)blockIdx.x * (WS_NT / 32) + wid;
    if (w >= n_items) return;
    const uint2 it = items[dir * (int64_t)w];  // dir = -1: the list grows downwards from items
    const Chunk c{it.x, it.y, 0};
    uint64_t k[R];
    uint32_t v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t i = lane + 32 * r;
        const uint64_t key = i < c.n ? ld_stream(keys + c.begin + i) : ~0ull;
        const uint32_t val = i < c.n ? __ldcs(vals + c.begin + i) : 0u;
        if (PACK) {
            k[r] = i < c.n ? (key << 8) | i : ~0ull;
            svals[wid][i] = val;
        } else {
            k[r] = key;
            v[r] = val;
        }
    }
#pragma unroll
    for (int sz = 2; sz <= N; sz <<= 1) {
#pragma unroll
        for (int j = sz >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
                const int jr = j / 32;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    if (r & jr) continue;
                    const int h = r | jr;
                    const bool up = ((lane + 32 * r) & sz) == 0;
                    const uint64_t lo = k[r] < k[h] ? k[r] : k[h], hi = k[r] < k[h] ? k[h] : k[r];
                    if (PACK) {
                        k[r] = up ? lo : hi;
                        k[h] = up ? hi : lo;
                    } else if (up ? k[r] > k[h] : k[r] < k[h]) {
                        k[r] = up ? lo : hi;
                        k[h] = up ? hi : lo;
                        const uint32_t tv = v[r];
                        v[r] = v[h];
                        v[h] = tv;
                    }
                }
            } else {
                const bool lower = (lane & j) == 0;
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const uint64_t pk = __shfl_xor_sync(0xffffffffu, k[r], j);
                    const bool want_min = (((lane + 32 * r) & sz) == 0) == lower;
                    if (PACK) {
                        k[r] = want_min ? (pk < k[r] ? pk : k[r]) : (pk > k[r] ? pk : k[r]);
                    } else {
                        const uint32_t pv = __shfl_xor_sync(0xffffffffu, v[r], j);
                        const bool take = want_min ? pk < k[r] : pk > k[r];
                        if (take) {
                            k[r] = pk;
                            v[r] = pv;
                        }
                    }
                }
            }
        }
    }
    if (PACK) __syncwarp();
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t i = lane + 32 * r;
        if (i < c.n) {
            if (PACK) {
                out_keys[c.begin + i] = k[r] >> 8;
                out_vals[c.begin + i] = svals[wid][k[r] & 0xFF];
            } else {
                out_keys[c.begin + i] = k[r];
                out_vals[c.begin + i] = v[r];
            }
        }
    }
}

// MSD levels: D_l <= 8 bits each, until the average bucket holds at most cap/8 survivors
// 64-bit keys end in warp sorts of buckets of a few tens: the last level takes only the
// bits that bring the average bucket to ~20 (fewer, fuller buckets to classify and sort).
int order_levels(uint64_t n, int k, int cap, int* D) {
    const int twok = 2 * k;
    int L = 0, bits = 0;
    do {
        D[L] = std::min(8, twok - bits);
        bits += D[L++];
    } while (bits < twok && L < 4 && (n >> bits) > (uint64_t)cap / 8);
    if (k <= 32) {
        const uint64_t before = n >> (bits - D[L - 1]);
        int d = 1;
#ifndef KMC_ORD_LAST
#define KMC_ORD_LAST 20
#endif
        while (d < D[L - 1] && (before >> d) > KMC_ORD_LAST) ++d;
        D[L - 1] = d;
    }
    return L;
}

// A few counters straight into pinned (mapped) host memory: a read-back that does not queue
// on the device-to-host copy engine behind the output copies of the groups before it.
__global__ void k_counters_to_host(const unsigned long long* __restrict__ src, unsigned long long* dst, int n) {
    if ((int)threadIdx.x < n) dst[threadIdx.x] = src[threadIdx.x];
}

// Host outputs (range_done, 64-bit keys): S9 depth first.  The top level partitions all
// survivors; then the top buckets are taken in ORD_GROUPS groups of about n / ORD_GROUPS
// survivors each, and every group runs its lower levels, its classification and its final
// sorts on its own item range (tiles from the top-level starts, offset to the range).  The
// caller's copy of a group's output can start after one pass over all survivors plus the
// first group's work, and runs while the later groups are sorted (breadth first, every
// level over all survivors came before the first copy).
cudaError_t order_groups64(uint64_t* keys, uint32_t* vals, uint64_t n, int k, const int* D, int L,
                           uint64_t* out_keys, uint32_t* out_vals, const OrderScratch& os, cudaStream_t s,
                           int* launches, std::vector<OrderSegment>* oversize, void** seg_keys,
                           uint32_t** seg_vals, const OrderRangeFn& range_done) {
    using K = uint64_t;
    constexpr uint64_t TI = OrderTile<K>::v;
    const int twok = 2 * k;
    const int osm = (int)otile_smem<K>();
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_ord_scatter<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, osm))) return e;
    const size_t sm = order_smem<K>();
    if ((e = cudaFuncSetAttribute(k_order_chunk_sort<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm))) return e;
    // one MSD level over items [0, m) of (kin, vin) into (kout, vout): tiles of src's nbk
    // buckets, digit = the D_l bits below top; leaves the level's counts / starts in hist / start
    auto level = [&](const TileSrc& src, uint64_t nbk, uint64_t m, int top, int Dl, const K* kin,
                     const uint32_t* vin, K* kout, uint32_t* vout) -> cudaError_t {
        const uint64_t mt = m / TI + nbk;
        cudaError_t e2;
        if ((e2 = launch_make_tiles(src, nbk, (uint32_t)TI, mt, os.tprefix, os.ttemp,
                                    reinterpret_cast<RecTile2*>(os.tiles), s)))
            return e2;
        const uint64_t* ntl = os.tprefix + nbk;
        const uint64_t nd = nbk << Dl;
        if ((e2 = cudaMemsetAsync(os.hist, 0, nd * 4, s))) return e2;
        k_ord_hist<K><<<(unsigned)mt, OT_NT, 0, s>>>(kin, os.tiles, ntl, top, Dl, os.hist);
        if ((e2 = cudaGetLastError())) return e2;
        if ((e2 = scan_detail::scan_generic<uint32_t>(scan_detail::ArrayIn<uint32_t>{os.hist}, nd, os.start,
                                                      (uint32_t*)os.scan_temp, s, launches)))
            return e2;
        if ((e2 = cudaMemcpyAsync(os.cursor, os.start, nd * 4, cudaMemcpyDeviceToDevice, s))) return e2;
        k_ord_scatter<K><<<(unsigned)mt, OT_NT, osm, s>>>(kin, vin, os.tiles, ntl, top, Dl, os.cursor, kout, vout);
        *launches += 5;
        return cudaGetLastError();
    };
    K* ck = keys;
    uint32_t* cv = vals;
    K* ok = (K*)os.tmp_keys;
    uint32_t* ov = os.tmp_vals;
    if ((e = level(TileSrc{nullptr, 0, 0, 0, n}, 1, n, twok, D[0], ck, cv, ok, ov))) return e;
    std::swap(ck, ok);
    std::swap(cv, ov);
    const uint64_t nb0 = 1ull << D[0];
    if ((e = cudaMemcpyAsync(os.start0, os.start, nb0 * 4, cudaMemcpyDeviceToDevice, s))) return e;
    std::vector<uint32_t> h0(nb0 + 1);
    if ((e = cudaMemcpyAsync(h0.data(), os.start, nb0 * 4, cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s))) return e;
    h0[nb0] = (uint32_t)n;
    // the group of every top bucket: about n / G survivors each
    const uint64_t G = std::min<uint64_t>(ORD_GROUPS, nb0);
    std::vector<uint64_t> B(G + 1, nb0);
    B[0] = 0;
    for (uint64_t g = 1, b = 0; g < G; ++g) {
        while (b < nb0 && (uint64_t)h0[b] < g * n / G) ++b;
        B[g] = std::max(b, B[g - 1]);
    }
    // after level 0 and L - 1 levels per group, every group's items are in the same buffer
    K* fk = (L - 1) % 2 == 0 ? ck : ok;
    uint32_t* fv = (L - 1) % 2 == 0 ? cv : ov;
    uint2* wlist = reinterpret_cast<uint2*>(os.chunks);
    Chunk* big = os.oversize;
    Chunk* over = reinterpret_cast<Chunk*>(os.cursor);
    unsigned long long* H = os.host;
    constexpr int WPB = WS_NT / 32;
    const int dir[4] = {1, -1, 1, -1};
    const bool pack = twok <= 56;
    oversize->clear();
    // the counters of every group's classification reach the host through mapped memory
    // written by a kernel, waited for with an event: a copy would wait behind the output
    // copies of the previous groups on the copy engine (and the next group behind it)
    cudaEvent_t ev = nullptr;
    if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming))) return e;
    struct EvGuard {
        cudaEvent_t e;
        ~EvGuard() { cudaEventDestroy(e); }
    } ev_guard{ev};
    for (uint64_t g = 0; g < G; ++g) {
        const uint64_t b0 = B[g], b1 = B[g + 1];
        if (b1 <= b0) continue;
        const uint64_t s0 = h0[b0], s1 = h0[b1], m = s1 - s0;
        if (m == 0) continue;
        K* ak = ck + s0;
        uint32_t* av = cv + s0;
        K* bk = ok + s0;
        uint32_t* bv = ov + s0;
        uint64_t nbk = b1 - b0;
        int top = twok - D[0];
        for (int l = 1; l < L; ++l) {
            const TileSrc src = l == 1 ? TileSrc{os.start0 + b0, 0, nbk, 0, m, s0} : TileSrc{os.start, 0, nbk, 0, m};
            if ((e = level(src, nbk, m, top, D[l], ak, av, bk, bv))) return e;
            std::swap(ak, bk);
            std::swap(av, bv);
            top -= D[l];
            nbk <<= D[l];
        }
        // the group's final buckets [0, nbk): counts in hist, starts (from s0) in start
        if ((e = cudaMemsetAsync(os.counters, 0, 9 * 8, s))) return e;
        k_ord_classify<<<(unsigned)((nbk + WS_NT - 1) / WS_NT), WS_NT, 0, s>>>(
            os.hist, os.start, nbk, (uint32_t)m, OrderCap<K>::v, wlist, big, over, os.counters, 0, nbk,
            os.counters + 8);
        *launches += 1;
        if ((e = cudaGetLastError())) return e;
        k_counters_to_host<<<1, 32, 0, s>>>(os.counters, H, 9);
        *launches += 1;
        if ((e = cudaGetLastError())) return e;
        if ((e = cudaEventRecord(ev, s))) return e;
        if ((e = cudaEventSynchronize(ev))) return e;
        const uint64_t nov = *(volatile unsigned long long*)&H[8];
        bool has_over = false;
        if (nov) {
            std::vector<Chunk> ovs(nov);
            if ((e = cudaMemcpyAsync(ovs.data(), over, nov * sizeof(Chunk), cudaMemcpyDeviceToHost, s))) return e;
            if ((e = cudaStreamSynchronize(s))) return e;
            for (auto& c : ovs) oversize->push_back(OrderSegment{s0 + c.begin, c.n});
            has_over = true;
        }
        const uint64_t wn = nbk;
        const uint2* wl[4] = {wlist, wlist + wn - 1, wlist + wn, wlist + 2 * wn - 1};
        for (int q = 0; q < 4; ++q) {
            const uint64_t nw = H[q];
            if (!nw) continue;
            const unsigned gr = (unsigned)((nw + WPB - 1) / WPB);
#define KMC_WSORT(R)                                                                                               \
    (pack ? k_ord_wsort<R, true><<<gr, WS_NT, 0, s>>>(ak, av, wl[q], nw, dir[q], out_keys + s0, out_vals + s0)      \
          : k_ord_wsort<R, false><<<gr, WS_NT, 0, s>>>(ak, av, wl[q], nw, dir[q], out_keys + s0, out_vals + s0))
            if (q == 0) KMC_WSORT(1);
            if (q == 1) KMC_WSORT(2);
            if (q == 2) KMC_WSORT(4);
            if (q == 3) KMC_WSORT(8);
#undef KMC_WSORT
            *launches += 1;
        }
        if (H[4]) {
            k_order_chunk_sort<K><<<(unsigned)H[4], OC_NT, sm, s>>>(ak, av, big, twok, out_keys + s0, out_vals + s0);
            *launches += 1;
        }
        if ((e = cudaGetLastError())) return e;
        range_done(s0, s1, !has_over);
    }
    *seg_keys = fk;
    *seg_vals = fv;
    return cudaSuccess;
}

template <class K>
cudaError_t order_t(K* keys, uint32_t* vals, uint64_t n, int k, K* out_keys, uint32_t* out_vals,
                    const OrderScratch& os, cudaStream_t s, int* launches, std::vector<OrderSegment>* oversize,
                    void** seg_keys, uint32_t** seg_vals, const OrderRangeFn* range_done) {
    constexpr uint64_t TI = OrderTile<K>::v;
    const int twok = 2 * k;
    int D[4];
    const int L = order_levels(n, k, OrderCap<K>::v, D);
    if constexpr (sizeof(K) == 8)
        if (range_done && L >= 2 && os.start0)
            return order_groups64(keys, vals, n, k, D, L, out_keys, out_vals, os, s, launches, oversize, seg_keys,
                                  seg_vals, *range_done);
    cudaError_t e;
    const int osm = (int)otile_smem<K>();
    if ((e = cudaFuncSetAttribute(k_ord_scatter<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, osm))) return e;
    K* ck = keys;  // current layout
    uint32_t* cv = vals;
    K* ok = (K*)os.tmp_keys;  // the other buffers
    uint32_t* ov = os.tmp_vals;
    uint64_t nbk = 1;  // buckets of the previous level
    int top = twok;
    static_assert(sizeof(OrdTile) == sizeof(RecTile2), "tiles share the generator");
    for (int l = 0; l < L; ++l) {
        // tiles of at most TI items inside each bucket of the previous level, built on the
        // device from the previous level's bucket starts (before this level's scan
        // overwrites them)
        const uint64_t mt = n / TI + nbk;
        const TileSrc src = l == 0 ? TileSrc{nullptr, 0, 0, 0, n} : TileSrc{os.start, 0, nbk, 0, n};
        if ((e = launch_make_tiles(src, nbk, (uint32_t)TI, mt, os.tprefix, os.ttemp,
                                   reinterpret_cast<RecTile2*>(os.tiles), s)))
            return e;
        const uint64_t* ntl = os.tprefix + nbk;
        const uint64_t nd = nbk << D[l];
        if ((e = cudaMemsetAsync(os.hist, 0, nd * 4, s))) return e;
        k_ord_hist<K><<<(unsigned)mt, OT_NT, 0, s>>>(ck, os.tiles, ntl, top, D[l], os.hist);
        if ((e = cudaGetLastError())) return e;
        if ((e = scan_detail::scan_generic<uint32_t>(scan_detail::ArrayIn<uint32_t>{os.hist}, nd, os.start,
                                                     (uint32_t*)os.scan_temp, s, launches)))
            return e;
        if ((e = cudaMemcpyAsync(os.cursor, os.start, nd * 4, cudaMemcpyDeviceToDevice, s))) return e;
        k_ord_scatter<K><<<(unsigned)mt, OT_NT, osm, s>>>(ck, cv, os.tiles, ntl, top, D[l], os.cursor, ok, ov);
        if ((e = cudaGetLastError())) return e;
        *launches += 5;
        std::swap(ck, ok);
        std::swap(cv, ov);
        top -= D[l];
        nbk = nd;
    }
    // ---- the buckets, sorted into the output: by warps (64-bit keys, buckets <= 256 items),
    //      by CTAs in shared memory (chunks of consecutive buckets), or returned as oversize
    if ((e = cudaMemsetAsync(os.counters, 0, 64, s))) return e;
    uint64_t n_chunks = 0, n_over = 0;
    const Chunk* chunk_list = os.chunks;
    const Chunk* over_list = os.oversize;
    const size_t sm = order_smem<K>();
    if ((e = cudaFuncSetAttribute(k_order_chunk_sort<K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm))) return e;
    oversize->clear();
    if constexpr (sizeof(K) == 8) {
        // lists in buffers the MSD passes are done with: the warp-sort lists {begin, n} in
        // os.chunks (2 nbk uint2: 64-item sorts from the front of the first half, 128 / 256
        // from both ends of the second), CTA chunks in os.oversize, oversize buckets (at
        // most n / cap + 1 of them) in os.cursor.  With range_done, the buckets are taken in
        // G groups of consecutive buckets, so that the caller can copy a group's output
        // while the next one is sorted.
        uint2* wlist = reinterpret_cast<uint2*>(os.chunks);
        Chunk* big = os.oversize;
        Chunk* over = reinterpret_cast<Chunk*>(os.cursor);
        static_assert(sizeof(Chunk) == 2 * sizeof(uint2), "two list entries per chunk slot");
        // every group is classified first (its lists in its own slice of the buffers, one
        // read-back for all), then the groups' sorts are launched in order: the caller's copy
        // of a group can start while the next group sorts, with no read-back behind it
        const uint64_t G = range_done ? std::min<uint64_t>(ORD_GROUPS, nbk) : 1;
        unsigned long long* over_ctr = os.counters + 8 * ORD_GROUPS;
        if ((e = cudaMemsetAsync(os.counters, 0, (8 * ORD_GROUPS + 1) * 8, s))) return e;
        std::vector<uint64_t> bb(G + 1);
        for (uint64_t g = 0; g <= G; ++g) bb[g] = g * nbk / G;
        for (uint64_t g = 0; g < G; ++g) {
            const uint64_t b0 = bb[g], b1 = bb[g + 1];
            if (b1 <= b0) continue;
            k_ord_classify<<<(unsigned)((b1 - b0 + WS_NT - 1) / WS_NT), WS_NT, 0, s>>>(
                os.hist, os.start, nbk, (uint32_t)n, OrderCap<K>::v, wlist + 2 * b0, big + b0, over,
                os.counters + 8 * g, b0, b1, over_ctr);
            *launches += 1;
        }
        if ((e = cudaGetLastError())) return e;
        unsigned long long* H = os.host;  // [8 G counters][over count][G + 1 group starts]
        if ((e = cudaMemcpyAsync(H, os.counters, (8 * ORD_GROUPS + 1) * 8, cudaMemcpyDeviceToHost, s))) return e;
        uint32_t* hstart = reinterpret_cast<uint32_t*>(H + 8 * ORD_GROUPS + 1);
        for (uint64_t g = 1; g < G; ++g)
            if ((e = cudaMemcpyAsync(hstart + g, os.start + bb[g], 4, cudaMemcpyDeviceToHost, s))) return e;
        if ((e = cudaStreamSynchronize(s))) return e;
        const uint64_t nov = H[8 * ORD_GROUPS];
        std::vector<Chunk> ovs(nov);
        if (nov) {
            if ((e = cudaMemcpyAsync(ovs.data(), over, nov * sizeof(Chunk), cudaMemcpyDeviceToHost, s))) return e;
            if ((e = cudaStreamSynchronize(s))) return e;
            for (auto& c : ovs) oversize->push_back(OrderSegment{c.begin, c.n});
        }
        std::vector<uint64_t> ist(G + 1);
        ist[0] = 0;
        ist[G] = n;
        for (uint64_t g = 1; g < G; ++g) ist[g] = hstart[g];
        constexpr int WPB = WS_NT / 32;
        const int dir[4] = {1, -1, 1, -1};
        const bool pack = twok <= 56;
        for (uint64_t g = 0; g < G; ++g) {
            const uint64_t b0 = bb[g], b1 = bb[g + 1], wn = b1 - b0;
            if (wn == 0) continue;
            const unsigned long long* c = H + 8 * g;
            uint2* w = wlist + 2 * b0;
            const uint2* wl[4] = {w, w + wn - 1, w + wn, w + 2 * wn - 1};
            for (int q = 0; q < 4; ++q) {
                const uint64_t nw = c[q];
                if (!nw) continue;
                const unsigned gr = (unsigned)((nw + WPB - 1) / WPB);
#define KMC_WSORT(R)                                                                                          \
    (pack ? k_ord_wsort<R, true><<<gr, WS_NT, 0, s>>>(ck, cv, wl[q], nw, dir[q], out_keys, out_vals)            \
          : k_ord_wsort<R, false><<<gr, WS_NT, 0, s>>>(ck, cv, wl[q], nw, dir[q], out_keys, out_vals))
                if (q == 0) KMC_WSORT(1);
                if (q == 1) KMC_WSORT(2);
                if (q == 2) KMC_WSORT(4);
                if (q == 3) KMC_WSORT(8);
#undef KMC_WSORT
                *launches += 1;
            }
            if (c[4]) {
                k_order_chunk_sort<K><<<(unsigned)c[4], OC_NT, sm, s>>>(ck, cv, big + b0, twok, out_keys, out_vals);
                *launches += 1;
            }
            if ((e = cudaGetLastError())) return e;
            if (range_done) {
                bool has_over = false;
                for (auto& o : ovs) has_over |= o.begin >= ist[g] && o.begin < ist[g + 1];
                (*range_done)(ist[g], ist[g + 1], !has_over);
            }
        }
        *seg_keys = ck;
        *seg_vals = cv;
        return cudaSuccess;
    } else {
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
        n_chunks = os.host[0];
        n_over = os.host[1];
        *launches += 1;
    }
    if (n_chunks)
        k_order_chunk_sort<K><<<(unsigned)n_chunks, OC_NT, sm, s>>>(ck, cv, chunk_list, twok, out_keys, out_vals);
    if ((e = cudaGetLastError())) return e;
    *launches += n_chunks > 0;
    *seg_keys = ck;
    *seg_vals = cv;
    if (n_over) {
        std::vector<Chunk> ovs(n_over);
        if ((e = cudaMemcpyAsync(ovs.data(), over_list, n_over * sizeof(Chunk), cudaMemcpyDeviceToHost, s))) return e;
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

uint64_t order_prev_buckets(uint64_t n, int k) {
    int D[4];
    const int L = order_levels(n, k, k <= 32 ? OrderCap<uint64_t>::v : OrderCap<K128>::v, D);
    int prev = 0;
    for (int l = 0; l + 1 < L; ++l) prev += D[l];
    return 1ull << prev;
}

size_t order_scan_temp_bytes(uint64_t n_digits) { return scan_detail::scan_temp_elems<uint64_t>(n_digits) * 8; }

cudaError_t launch_order(int key_words, void* keys, uint32_t* vals, uint64_t n, int k, void* out_keys,
                         uint32_t* out_vals, const OrderScratch& os, cudaStream_t s, int* launches,
                         std::vector<OrderSegment>* oversize, void** seg_keys, uint32_t** seg_vals,
                         const OrderRangeFn* range_done) {
    oversize->clear();
    *seg_keys = keys;
    *seg_vals = vals;
    if (n == 0) return cudaSuccess;
    if (n >= (1ull << 32)) return cudaErrorInvalidValue;
    if (key_words == 1)
        return order_t<uint64_t>((uint64_t*)keys, vals, n, k, (uint64_t*)out_keys, out_vals, os, s, launches, oversize,
                                 seg_keys, seg_vals, range_done);
    return order_t<K128>((K128*)keys, vals, n, k, (K128*)out_keys, out_vals, os, s, launches, oversize, seg_keys,
                         seg_vals, nullptr);
}

}  // namespace kmc
