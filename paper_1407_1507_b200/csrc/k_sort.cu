// k_sort.cu -- phase 2 of KMC 2 on the B200 (Sec. 2.4 "sorting"; appendix
// "Sorter": uncompact super-k-mers, sort, merge identical k-mers with the
// cutoffs) and S9 (global ascending order of the survivors, reading R8).
//
//   k_small_bins  one CTA per bin that fits shared memory: records -> canonical keys
//                 (S6) -> LSD radix sort in SMEM (S7) -> run-length compaction with
//                 ci <= count <= cx (S8) -> survivors appended to the survivor buffer.
//   k_large_expand  S6 for bins above CTA capacity: keys into HBM.
//   k_upsweep / k_downsweep  device-wide LSD radix sort (8-bit digits, constant digits
//                 skipped) -- S7 for large bins and S9 for the survivors.
//   k_rle         S8 over a globally sorted HBM key array.
#include <algorithm>
#include <vector>

#include "kmc_device.cuh"
#include "kmc_internal.h"

namespace kmc {

namespace {

constexpr int SB_NT = 512;
constexpr int SB_NW = SB_NT / 32;
constexpr int SB_CAP64 = 6144;  // keys per small bin (u64); 2 CTAs per SM
constexpr int SB_CAP128 = 3072;

template <class K> struct SmallCap;
template <> struct SmallCap<uint64_t> { static constexpr int v = SB_CAP64; };
template <> struct SmallCap<K128> { static constexpr int v = SB_CAP128; };

template <class K> __host__ __device__ constexpr size_t small_smem_bytes() {
    return 2 * (size_t)SmallCap<K>::v * sizeof(K) + RADIX * SB_NW * 4 + 128 + 64;
}

// Expand one record into n canonical keys at dst[0..n) (min(fwd, rc)).
template <class K>
__device__ __forceinline__ void expand_record(const uint32_t* rec, int k, bool canonical, K* dst) {
    constexpr int RW = RecWords<K>::v;
    uint32_t wd[RW];
    load_record<RW>(rec, wd);
    for_each_window<K, RW>(wd, k, canonical, [&](int w, const K& key) { dst[w] = key; });
}

// Run-length compaction of the sorted keys S[0..n) with the cutoffs (S8); cnt is a free
// uint32 scratch of n entries.  Survivors are appended at a CTA-reserved range.
template <class K, int NT>
__device__ __forceinline__ void block_rle_emit(const K* S, int n, uint32_t* cnt, uint32_t ci, uint32_t cx,
                                               K* out_keys, uint32_t* out_counts, unsigned long long* gstats,
                                               uint32_t* wsum, unsigned long long* bcast) {
    const int seg = (n + NT - 1) / NT;
    const int b0 = threadIdx.x * seg, b1 = min(n, b0 + seg);
    uint32_t uniq = 0, below = 0, above = 0, keep = 0;
    for (int i = b0; i < b1; ++i) {
        uint32_t c = 0;
        if (i == 0 || !key_eq(S[i], S[i - 1])) {
            int j = i + 1;
            while (j < n && key_eq(S[j], S[i])) ++j;
            const uint32_t run = (uint32_t)(j - i);
            ++uniq;
            if (run < ci) ++below;
            else if (run > cx) ++above;
            else {
                c = run;
                ++keep;
            }
        }
        cnt[i] = c;
    }
    uint32_t total;
    uint32_t ex = block_excl_sum<NT, uint32_t>(keep, wsum, &total);
    const uint32_t tu = block_sum<NT, uint32_t>(uniq, wsum);
    const uint32_t tb = block_sum<NT, uint32_t>(below, wsum);
    const uint32_t ta = block_sum<NT, uint32_t>(above, wsum);
    if (threadIdx.x == 0) {
        *bcast = total ? atomicAdd(&gstats[GS_SURV], (unsigned long long)total) : 0ull;
        if (tu) atomicAdd(&gstats[GS_UNIQUE], (unsigned long long)tu);
        if (tb) atomicAdd(&gstats[GS_BELOW], (unsigned long long)tb);
        if (ta) atomicAdd(&gstats[GS_ABOVE], (unsigned long long)ta);
    }
    __syncthreads();
    const uint64_t base = *bcast + ex;
    uint64_t o = 0;
    for (int i = b0; i < b1; ++i) {
        const uint32_t c = cnt[i];
        if (c) {
            out_keys[base + o] = S[i];
            out_counts[base + o] = c;
            ++o;
        }
    }
}

// Small-bin table: the B region (CAP keys) once the records are expanded, as 2^lg key slots +
// 2^lg uint32 counters.
template <class K> struct SmallSlots;
template <> struct SmallSlots<uint64_t> { static constexpr int lg = 12; };  // 4096 x 12 B = 48 KB
template <> struct SmallSlots<K128> { static constexpr int lg = 11; };      // 2048 x 20 B = 40 KB
static_assert((1 << 12) * 12 <= SB_CAP64 * 8 && (1 << 11) * 20 <= SB_CAP128 * 16, "table fits the B region");

template <class K>
__global__ void __launch_bounds__(SB_NT, 2) k_small_bins(SmallArgs a) {
    constexpr int CAP = SmallCap<K>::v;
    extern __shared__ __align__(16) uint8_t smem[];
    K* A = reinterpret_cast<K*>(smem);
    K* B = A + CAP;
    uint32_t* whist = reinterpret_cast<uint32_t*>(B + CAP);
    uint32_t* wsum = whist + RADIX * SB_NW;                                      // 17 used
    unsigned long long* red = reinterpret_cast<unsigned long long*>(wsum + 24);  // 4
    unsigned long long* bcast = red + 4;
    unsigned int* scnt = reinterpret_cast<unsigned int*>(bcast + 1);

    const uint32_t bin = a.small_list[blockIdx.x];
    const uint64_t rec0 = a.bin_rec_off[bin];
    const int nrec = (int)a.bin_nrec[bin];
    const int n = (int)a.bin_w[bin];
    const int k = a.k;
    const int RW = record_words(k);

    // ---- load the bin's records (16-byte vectors) into B
    uint32_t* R = reinterpret_cast<uint32_t*>(B);
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.bins + rec0 * RW);
        uint4* dst = reinterpret_cast<uint4*>(R);
        const int nv = nrec * RW / 4;
#pragma unroll 4
        for (int v = threadIdx.x; v < nv; v += SB_NT) dst[v] = src[v];
    }
    __syncthreads();
    // ---- S6: expand records into canonical keys in A (record prefix sums by block scan)
    {
        const int rpt = (nrec + SB_NT - 1) / SB_NT;
        const int r0 = threadIdx.x * rpt, r1 = min(nrec, r0 + rpt);
        uint32_t s = 0;
        for (int r = r0; r < r1; ++r) s += rec_nwin(R + r * RW);
        uint32_t pos = block_excl_sum<SB_NT, uint32_t>(s, wsum, nullptr);
        for (int r = r0; r < r1; ++r) {
            const uint32_t* rec = R + r * RW;
            expand_record<K>(rec, k, a.canonical, A + pos);
            pos += rec_nwin(rec);
        }
    }
    __syncthreads();
    // ---- S7-S8 by counting: the bin's keys into a hash table in the B region (one shared
    // CAS per probe claims a slot or finds the key, atomicAdd counts), then one scan of the
    // table emits the survivors (S9 orders them).  Same counts as sorting + run-length
    // compaction; a bin whose distinct keys overfill the table (a probe sequence longer
    // than PROBE_MAX) is sorted instead.
    {
        constexpr int LGMAX = SmallSlots<K>::lg;
        int lg = 6;
        while (lg < LGMAX && (1 << lg) < n + n / 3) ++lg;
        const int TS = 1 << lg;
        K* T = reinterpret_cast<K*>(B);
        uint32_t* C = reinterpret_cast<uint32_t*>(T + (1 << LGMAX));
        const K E = key_empty<K>();
        for (int i = threadIdx.x; i < TS; i += SB_NT) {
            T[i] = E;
            C[i] = 0;
        }
        if (threadIdx.x == 0) *scnt = 0;
        __syncthreads();
        bool ok = true;
        for (int i = threadIdx.x; i < n; i += SB_NT) ok &= table_insert_bounded<K>(T, C, lg, A[i]);
        if (!ok) *scnt = 1;
        __syncthreads();
        if (*scnt != 0 && threadIdx.x == 0) atomicAdd(&a.gstats[GS_SMALL_SORTED], 1ull);
        if (*scnt == 0) {
            uint32_t uniq = 0, below = 0, above = 0, keep = 0;
            for (int i = threadIdx.x; i < TS; i += SB_NT) {
                const uint32_t c = C[i];
                if (c) {
                    ++uniq;
                    if (c < a.ci) ++below;
                    else if (c > a.cx) ++above;
                    else ++keep;
                }
            }
            // per-warp reservations and statistics (the warp writes the slots it counted): no
            // block reductions, no barriers
            const uint32_t kin = warp_incl_sum(keep);
            const uint32_t ktot = __shfl_sync(0xffffffffu, kin, 31);
            const uint32_t tu = __reduce_add_sync(0xffffffffu, uniq);
            const uint32_t tb = __reduce_add_sync(0xffffffffu, below);
            const uint32_t ta = __reduce_add_sync(0xffffffffu, above);
            unsigned long long base = 0;
            if ((threadIdx.x & 31) == 0) {
                if (ktot) base = atomicAdd(&a.gstats[GS_SURV], (unsigned long long)ktot);
                if (tu) atomicAdd(&a.gstats[GS_UNIQUE], (unsigned long long)tu);
                if (tb) atomicAdd(&a.gstats[GS_BELOW], (unsigned long long)tb);
                if (ta) atomicAdd(&a.gstats[GS_ABOVE], (unsigned long long)ta);
            }
            uint64_t o = __shfl_sync(0xffffffffu, base, 0) + kin - keep;
            K* ok_keys = reinterpret_cast<K*>(a.surv_keys);
            for (int i = threadIdx.x; i < TS; i += SB_NT) {
                const uint32_t c = C[i];
                if (c >= a.ci && c <= a.cx && c != 0) {
                    ok_keys[o] = T[i];
                    a.surv_counts[o] = c;
                    ++o;
                }
            }
            return;
        }
        __syncthreads();
    }
    // ---- S7: LSD radix sort in shared memory (in place)
    block_sort_inplace<K, SB_NT, CAP / SB_NT, false>(A, nullptr, n, 2 * k, whist, wsum, red);
    // ---- S8: run-length compaction + cutoffs
    block_rle_bitmask<K, SB_NT>(A, n, reinterpret_cast<uint32_t*>(B), a.ci, a.cx, reinterpret_cast<K*>(a.surv_keys),
                                a.surv_counts, a.gstats, wsum, scnt, bcast, GS_SURV, GS_UNIQUE, GS_BELOW, GS_ABOVE);
}

// ---------------------------------------------------------------- large-bin expansion
constexpr int LE_NT = 256;

template <class K>
__global__ void __launch_bounds__(LE_NT) k_large_expand(const uint32_t* __restrict__ bins,
                                                        const Piece* __restrict__ pieces, int k, int canonical,
                                                        K* keys, unsigned long long* gstats) {
    __shared__ __align__(16) uint32_t R[PIECE_RECORDS * 8];
    __shared__ uint32_t wsum[LE_NT / 32 + 1];
    __shared__ unsigned long long bcast;
    const Piece pc = pieces[blockIdx.x];
    const int RW = record_words(k);
    {
        const uint4* src = reinterpret_cast<const uint4*>(bins + pc.rec_begin * RW);
        uint4* dst = reinterpret_cast<uint4*>(R);
        const int nv = (int)pc.nrec * RW / 4;
        for (int v = threadIdx.x; v < nv; v += LE_NT) dst[v] = src[v];
    }
    __syncthreads();
    const int nrec = (int)pc.nrec;
    const int rpt = (nrec + LE_NT - 1) / LE_NT;
    const int r0 = threadIdx.x * rpt, r1 = min(nrec, r0 + rpt);
    uint32_t s = 0;
    for (int r = r0; r < r1; ++r) s += rec_nwin(R + r * RW);
    uint32_t total;
    uint32_t pos = block_excl_sum<LE_NT, uint32_t>(s, wsum, &total);
    if (threadIdx.x == 0) bcast = atomicAdd(&gstats[GS_LARGE_KEYS], (unsigned long long)total);
    __syncthreads();
    K* out = keys + bcast;
    for (int r = r0; r < r1; ++r) {
        const uint32_t* rec = R + r * RW;
        expand_record<K>(rec, k, canonical != 0, out + pos);
        pos += rec_nwin(rec);
    }
}

// ---------------------------------------------------------------- device radix sort
template <class K> struct RadixTile;
template <> struct RadixTile<uint64_t> { static constexpr int NT = 256, TI = 4096; };
template <> struct RadixTile<K128> { static constexpr int NT = 256, TI = 2048; };

// Onesweep-style LSD radix sort (north star: "a device-wide onesweep-style radix pass for
// large ones"): ONE histogram pass over the keys gives the digit counts of every 8-bit digit
// position at once (constant digits are skipped); then every varying digit takes ONE kernel:
// a CTA claims the next tile in order (atomic counter), ranks its keys by the digit in shared
// memory (stable), publishes its per-digit counts and finds the keys of its digits in all
// earlier tiles by decoupled look-back (status words flag | pass tag | value: an aggregate, or
// the inclusive prefix once known), then writes its keys at digit base + prefix + rank.
constexpr uint64_t OS_AGG = 1ull << 62, OS_PRE = 2ull << 62, OS_VAL = (1ull << 56) - 1;

template <class K>
__global__ void __launch_bounds__(256) k_digit_hist_all(const K* __restrict__ keys, uint64_t n, int npass,
                                                        uint32_t* __restrict__ hist) {
    __shared__ uint32_t h[16 * RADIX];
    for (int i = threadIdx.x; i < npass * RADIX; i += 256) h[i] = 0;
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (uint64_t)gridDim.x * 256) {
        const K key = keys[i];
        for (int p = 0; p < npass; ++p) atomicAdd(&h[p * RADIX + key_digit(key, p * RADIX_BITS)], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < npass * RADIX; i += 256)
        if (h[i]) atomicAdd(&hist[i], h[i]);
}

// bases[p][d] = exclusive scan over d of hist[p][d]; one CTA per digit position
__global__ void __launch_bounds__(RADIX) k_digit_bases(const uint32_t* __restrict__ hist, uint32_t* __restrict__ bases) {
    __shared__ uint32_t wsum[RADIX / 32 + 1];
    const uint32_t c = hist[blockIdx.x * RADIX + threadIdx.x];
    bases[blockIdx.x * RADIX + threadIdx.x] = block_excl_sum<RADIX, uint32_t>(c, wsum, nullptr);
}

template <class K, bool VALS>
__global__ void __launch_bounds__(RadixTile<K>::NT) k_onesweep(const K* __restrict__ kin,
                                                               const uint32_t* __restrict__ vin, K* __restrict__ kout,
                                                               uint32_t* __restrict__ vout, uint64_t n, int shift,
                                                               uint64_t tag, const uint32_t* __restrict__ bases,
                                                               unsigned long long* status, uint32_t* tile_ctr) {
    constexpr int NT = RadixTile<K>::NT, TI = RadixTile<K>::TI, NW = NT / 32;
    static_assert(NT == RADIX, "one thread per digit in the look-back");
    extern __shared__ __align__(16) uint8_t smem[];
    K* A = reinterpret_cast<K*>(smem);
    K* B = A + TI;
    uint32_t* VA = reinterpret_cast<uint32_t*>(B + TI);
    uint32_t* VB = VA + (VALS ? TI : 0);
    uint32_t* whist = VB + (VALS ? TI : 0);
    uint32_t* wsum = whist + RADIX * NW;
    uint32_t* dstart = wsum + NW + 1;  // RADIX + 1
    uint32_t* goff = dstart + RADIX + 1;
    __shared__ uint32_t s_tile;
    if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);  // tiles claimed in order: look-back never waits on an unscheduled tile
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t base = tile * TI;
    const int cnt = (int)((n - base) < (uint64_t)TI ? (n - base) : (uint64_t)TI);
    for (int j = threadIdx.x; j < cnt; j += NT) {
        A[j] = kin[base + j];
        if (VALS) VA[j] = vin[base + j];
    }
    __syncthreads();
    block_digit_pass<K, NT, VALS>(A, B, VA, VB, cnt, shift, whist, wsum, dstart);
    {
        const int d = threadIdx.x;
        const uint64_t mine = dstart[d + 1] - dstart[d];
        volatile unsigned long long* st = status + tile * RADIX + d;
        const uint64_t tg = tag << 56;
        uint64_t excl = 0;
        if (tile == 0) {
            *st = OS_PRE | tg | mine;
        } else {
            *st = OS_AGG | tg | mine;
            for (int64_t t = (int64_t)tile - 1; t >= 0;) {
                // volatile: re-read from L2 on every spin (a plain load may be served by a stale L1 line)
                const uint64_t v = *reinterpret_cast<volatile unsigned long long*>(status + (uint64_t)t * RADIX + d);
                if (((v >> 56) & 63) != tag || (v >> 62) == 0) continue;  // not published in this pass yet
                excl += v & OS_VAL;
                if ((v >> 62) == 2) break;  // an inclusive prefix: done
                --t;
            }
            *st = OS_PRE | tg | (excl + mine);
        }
        goff[d] = bases[d] + (uint32_t)excl;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < cnt; j += NT) {
        const K key = B[j];
        const uint32_t d = key_digit(key, shift);
        const uint64_t pos = (uint64_t)goff[d] + (uint32_t)(j - dstart[d]);
        kout[pos] = key;
        if (VALS) vout[pos] = VB[j];
    }
}

template <class K, bool VALS> constexpr size_t downsweep_smem() {
    constexpr int NT = RadixTile<K>::NT, TI = RadixTile<K>::TI, NW = NT / 32;
    return 2 * (size_t)TI * sizeof(K) + (VALS ? 2 * (size_t)TI * 4 : 0) + (RADIX * NW + NW + 1 + 2 * RADIX + 1) * 4 + 16;
}

template <class K>
cudaError_t radix_sort_t(K* keys, uint32_t* vals, uint64_t n, int nbits, const RadixScratch& rs, cudaStream_t s,
                         void** res_keys, uint32_t** res_vals, int* launches) {
    constexpr int NT = RadixTile<K>::NT, TI = RadixTile<K>::TI;
    *res_keys = keys;
    *res_vals = vals;
    if (n <= 1) return cudaSuccess;
    if (n >= (1ull << 32)) return cudaErrorInvalidValue;
    cudaError_t e;
    const int npass = (nbits + RADIX_BITS - 1) / RADIX_BITS;  // <= 16
    const uint64_t ntiles = (n + TI - 1) / TI;
    // scratch: tile_off = hist [16][RADIX] | bases [16][RADIX] | tile counters [16];
    //          tile_hist = look-back status, ntiles x RADIX uint64
    uint32_t* hist = rs.tile_off;
    uint32_t* bases = hist + 16 * RADIX;
    uint32_t* ctrs = bases + 16 * RADIX;
    unsigned long long* status = reinterpret_cast<unsigned long long*>(rs.tile_hist);
    if ((e = cudaMemsetAsync(hist, 0, (32 * RADIX + 16) * 4, s))) return e;
    if ((e = cudaMemsetAsync(status, 0, ntiles * RADIX * 8, s))) return e;
    const unsigned hg = (unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 4);
    k_digit_hist_all<K><<<hg, 256, 0, s>>>(keys, n, npass, hist);
    k_digit_bases<<<npass, RADIX, 0, s>>>(hist, bases);
    *launches += 2;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    // a digit position is constant iff one digit holds every key: skipped
    std::vector<uint32_t> hv((size_t)npass * RADIX);
    if ((e = cudaMemcpyAsync(hv.data(), hist, hv.size() * 4, cudaMemcpyDeviceToHost, s))) return e;
    if ((e = cudaStreamSynchronize(s)) != cudaSuccess) return e;
    K* src = keys;
    K* dst = reinterpret_cast<K*>(rs.keys_alt);
    uint32_t* vsrc = vals;
    uint32_t* vdst = rs.vals_alt;
    const bool has_vals = vals != nullptr;
    const size_t sm = has_vals ? downsweep_smem<K, true>() : downsweep_smem<K, false>();
    if (has_vals) {
        if ((e = cudaFuncSetAttribute(k_onesweep<K, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)))
            return e;
    } else {
        if ((e = cudaFuncSetAttribute(k_onesweep<K, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)))
            return e;
    }
    for (int p = 0; p < npass; ++p) {
        bool varies = true;
        for (int d = 0; d < RADIX; ++d)
            if (hv[(size_t)p * RADIX + d] == n) varies = false;
        if (!varies) continue;
        const int shift = p * RADIX_BITS;
        const uint64_t tag = (uint64_t)p + 1;
        if (has_vals)
            k_onesweep<K, true><<<(unsigned)ntiles, NT, sm, s>>>(src, vsrc, dst, vdst, n, shift, tag,
                                                                 bases + p * RADIX, status, ctrs + p);
        else
            k_onesweep<K, false><<<(unsigned)ntiles, NT, sm, s>>>(src, nullptr, dst, nullptr, n, shift, tag,
                                                                  bases + p * RADIX, status, ctrs + p);
        *launches += 1;
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
        std::swap(src, dst);
        std::swap(vsrc, vdst);
    }
    *res_keys = src;
    *res_vals = has_vals ? vsrc : nullptr;
    return cudaSuccess;
}

// ---------------------------------------------------------------- RLE over HBM keys
constexpr int RLE_NT = 256, RLE_IPT = 8;

template <class K>
__global__ void __launch_bounds__(RLE_NT) k_rle(const K* __restrict__ keys, uint64_t n, uint32_t ci, uint32_t cx,
                                                K* __restrict__ sk, uint32_t* __restrict__ sc,
                                                unsigned long long* gstats) {
    __shared__ uint32_t wsum[RLE_NT / 32 + 1];
    __shared__ unsigned long long bcast;
    const uint64_t base = (uint64_t)blockIdx.x * (RLE_NT * RLE_IPT);
    uint32_t cnts[RLE_IPT];
    uint32_t uniq = 0, below = 0, above = 0, keep = 0;
#pragma unroll
    for (int j = 0; j < RLE_IPT; ++j) {
        const uint64_t i = base + (uint64_t)j * RLE_NT + threadIdx.x;
        cnts[j] = 0;
        if (i >= n) continue;
        const K key = keys[i];
        if (i > 0 && key_eq(keys[i - 1], key)) continue;
        if (key_eq(key, key_empty<K>())) continue;  // pads of the one-pass split (never a k-mer)
        // galloping search for the end of the run
        uint64_t lo = i, hi, step = 1;
        for (;;) {
            const uint64_t pr = lo + step;
            if (pr >= n || !key_eq(keys[pr], key)) {
                hi = pr < n ? pr : n;
                break;
            }
            lo = pr;
            step <<= 1;
        }
        while (hi - lo > 1) {
            const uint64_t mid = lo + ((hi - lo) >> 1);
            if (key_eq(keys[mid], key)) lo = mid;
            else hi = mid;
        }
        const uint64_t run = hi - i;
        ++uniq;
        if (run < ci) ++below;
        else if (run > cx) ++above;
        else {
            cnts[j] = (uint32_t)(run > 0xFFFFFFFFull ? 0xFFFFFFFFull : run);
            ++keep;
        }
    }
    uint32_t total;
    uint32_t ex = block_excl_sum<RLE_NT, uint32_t>(keep, wsum, &total);
    const uint32_t tu = block_sum<RLE_NT, uint32_t>(uniq, wsum);
    const uint32_t tb = block_sum<RLE_NT, uint32_t>(below, wsum);
    const uint32_t ta = block_sum<RLE_NT, uint32_t>(above, wsum);
    if (threadIdx.x == 0) {
        bcast = total ? atomicAdd(&gstats[GS_SURV], (unsigned long long)total) : 0ull;
        if (tu) atomicAdd(&gstats[GS_UNIQUE], (unsigned long long)tu);
        if (tb) atomicAdd(&gstats[GS_BELOW], (unsigned long long)tb);
        if (ta) atomicAdd(&gstats[GS_ABOVE], (unsigned long long)ta);
    }
    __syncthreads();
    uint64_t o = bcast + ex;
#pragma unroll
    for (int j = 0; j < RLE_IPT; ++j) {
        if (cnts[j]) {
            const uint64_t i = base + (uint64_t)j * RLE_NT + threadIdx.x;
            sk[o] = keys[i];
            sc[o] = cnts[j];
            ++o;
        }
    }
}

// ---------------------------------------------------------------- partition split of large bins
// A bin above one CTA's capacity is sorted by a multi-CTA split followed by per-chunk
// shared-memory sorts: (1) count a D-bit digit of every key of the bin,
// (2) scan the digit counts per bin and group consecutive digits into chunks of at most
// CAP keys, (3) re-expand the records and scatter every key to its digit's range in HBM,
// (4) sort + compact every chunk in shared memory (k_chunk_sort).  The digit is a
// multiplicative hash of the whole key: a chunk only has to hold every copy of its keys
// (S9 orders the survivors globally), and the top bits of a key are a poor digit -- about
// 1/(k-p+1) of a bin's windows start with the bin's own signature.  A digit holding more
// than CAP keys (identical-key pile-ups, e.g. poly-A) becomes an "oversize" chunk sorted
// by the device-wide LSD path.
constexpr int MSD_NT = 256;
constexpr int MSD_MAXD = 12;

template <class K> struct MsdPiece;
template <> struct MsdPiece<uint64_t> { static constexpr int REC = 512, MAXW = 60; };
template <> struct MsdPiece<K128> { static constexpr int REC = 512, MAXW = 92; };

// Chunk planner over a flat sequence of digits (consecutive key ranges: digit d holds
// cnt[d] keys from gstart[d]; the large bins' digits bin after bin, or S9's buckets).
// Consecutive digits are packed greedily into chunks of at most cap keys; a digit above cap
// becomes an "oversize" chunk of its own.  Any contiguous key range is a valid chunk: a
// k-mer's keys share one bin and one digit.  One CTA per segment of g.seg digits: a block
// scan gives the prefix P of the segment's counts, then one thread walks the greedy chain
// -- each chunk's end is found by a galloping search on P, so the serial work is
// O(chunks x log(digits per chunk)) -- and the CTA appends its chunks with one atomic per
// list.  The host sizes segments to hold ~64 chunks.
constexpr int GP_NT = 256;
constexpr int GP_SEGMAX = 8192;

__global__ void __launch_bounds__(GP_NT) k_greedy_chunks(GreedyArgs g) {
    extern __shared__ __align__(16) uint32_t gsm[];
    const int seg = (int)g.seg;
    uint32_t* P = gsm;              // seg + 1
    uint32_t* cs = P + seg + 1;     // chunk starts (segment-relative)
    uint32_t* cn = cs + seg;        // chunk sizes; bit 31: oversize
    __shared__ uint32_t wsum[GP_NT / 32 + 1];
    __shared__ uint32_t nl_s, nreg_s;
    __shared__ unsigned long long base_reg, base_over;
    const uint64_t dbase = (uint64_t)blockIdx.x * seg;
    const int nd = (int)((g.n_digits - dbase) < (uint64_t)seg ? (g.n_digits - dbase) : (uint64_t)seg);
    const int ipt = (nd + GP_NT - 1) / GP_NT;
    const int d0 = threadIdx.x * ipt, d1 = min(nd, d0 + ipt);
    uint32_t sum = 0;
    for (int d = d0; d < d1; ++d) sum += g.cnt[dbase + d];
    uint32_t total;
    uint32_t run = block_excl_sum<GP_NT, uint32_t>(sum, wsum, &total);
    for (int d = d0; d < d1; ++d) {
        P[d] = run;
        run += g.cnt[dbase + d];
    }
    if (threadIdx.x == 0) P[nd] = total;
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t cap = g.cap;
        int nl = 0, nreg = 0;
        for (int d = 0; d < nd;) {
            const uint32_t pd = P[d];
            if (P[d + 1] - pd > cap) {
                cs[nl] = pd;
                cn[nl++] = (P[d + 1] - pd) | 0x80000000u;
                ++d;
                continue;
            }
            // largest e in (d, nd] with P[e] - P[d] <= cap: gallop, then bisect
            int lo = d + 1, step = 1;
            while (lo + step <= nd && P[lo + step] - pd <= cap) {
                lo += step;
                step *= 2;
            }
            int hi = min(lo + step, nd + 1);  // P[hi] - pd > cap, or hi = nd + 1
            while (hi - lo > 1) {
                const int mid = (lo + hi) >> 1;
                if (P[mid] - pd <= cap) lo = mid;
                else hi = mid;
            }
            if (P[lo] != pd) {
                cs[nl] = pd;
                cn[nl++] = P[lo] - pd;
                ++nreg;
            }
            d = lo;
        }
        nl_s = nl;
        nreg_s = nreg;
        base_reg = nreg ? atomicAdd(&g.counters[0], (unsigned long long)nreg) : 0ull;
        base_over = nl - nreg ? atomicAdd(&g.counters[1], (unsigned long long)(nl - nreg)) : 0ull;
    }
    __syncthreads();
    // append in chain order (ballot ranks per list)
    const uint64_t kbase = g.gstart[dbase];
    const int nl = (int)nl_s;
    __shared__ uint32_t run_reg, run_over, wr[GP_NT / 32], wo[GP_NT / 32];
    if (threadIdx.x == 0) { run_reg = 0; run_over = 0; }
    __syncthreads();
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, lt = lanemask_lt();
    for (int i0 = 0; i0 < nl; i0 += GP_NT) {
        const int i = i0 + threadIdx.x;
        const uint32_t c = i < nl ? cn[i] : 0u;
        const bool over = i < nl && (c & 0x80000000u), reg = i < nl && !over;
        const uint32_t br = __ballot_sync(0xffffffffu, reg), bo = __ballot_sync(0xffffffffu, over);
        if (lane == 0) { wr[warp] = __popc(br); wo[warp] = __popc(bo); }
        __syncthreads();
        uint32_t orr = run_reg, oo = run_over;
        for (uint32_t w = 0; w < warp; ++w) { orr += wr[w]; oo += wo[w]; }
        if (reg) g.chunks[base_reg + orr + __popc(br & lt)] = Chunk{kbase + cs[i], c, 0};
        if (over) g.oversize[base_over + oo + __popc(bo & lt)] = Chunk{kbase + cs[i], c & 0x7FFFFFFFu, 0};
        __syncthreads();
        if (threadIdx.x == 0)
            for (uint32_t w = 0; w < GP_NT / 32; ++w) { run_reg += wr[w]; run_over += wo[w]; }
        __syncthreads();
    }
}

// Split of the large bins, upsweep/downsweep style over CTA "ranges".  The
// pieces of all large bins (in bin order) are cut into R contiguous ranges, one per CTA.
// A bin's keys are counted per "segment" and digit: the count kernel histograms the split
// digit of every window of a segment in shared memory and stores it, without atomics, at
// table[lb.tb + d * lb.nseg + j] (j = segment index within the bin).  An exclusive scan of
// the table (bin-major, then digit, then segment) gives every segment the position of its
// first key of digit d in the digit-contiguous layout of the bin's keys; the scatter
// kernel re-expands the segment and places every key -- no global atomics.
// Segments are either (range, bin) pairs ("range mode": the scatter places every key at a
// shared-memory cursor seeded from the table, each CTA writing every digit as one run) or,
// for 64-bit keys and bins with D <= SP_PM_DMAX, single pieces ("piece mode", lb.pad = 1):
// the scatter then knows every digit's key count in the piece before expanding it, stages
// the piece's keys in shared memory grouped by digit and writes them out coalesced
// (consecutive threads, consecutive addresses) instead of 8-byte stores scattered over up
// to 2^D runs.  Pieces stream through a double-buffered TMA staging area (one 1-D bulk copy
// each).
constexpr int SP_NT = 512;      // split CTA: one record of a piece per thread
constexpr int SP_PM_DMAX = 8;   // piece mode: digits per bin <= 256 (<= SP_NT)
constexpr int SP_STAGE = 8192;  // keys of a piece staged in shared memory (more: direct stores)
// digit counters, padded to 128 bytes (the TMA staging buffers that follow need 16-byte alignment)
__host__ __device__ constexpr int split_hwords(int dmax) { return ((1 << dmax) + 31) & ~31; }
template <class K> __host__ __device__ constexpr int split_unit(int k) {
    return sizeof(K) == 8 ? (k + 3 <= 32 ? 4 : 33 - k) : 1;  // windows per lane unit
}
template <class K, bool SC> __host__ __device__ int split_own_bytes(int k) {  // unit -> lane map per warp
    const int U = split_unit<K>(k);
    const int upr = (record_max_windows(k) + U - 1) / U;  // units per record, at most
    if (sizeof(K) == 8 && U == 4 && !SC)  // count pass, block-balanced: uint16 unit -> record map + record info
        return ((SP_NT * upr * 2 + SP_NT * 4) / (SP_NT / 32) + 15) & ~15;
    return (32 * upr + 15) & ~15;
}
// bytes of the counter region; the scatter of 64-bit keys aliases it with the piece stage
template <class K, bool SC> __host__ __device__ int split_hreg(int dmax) {
    const int hb = split_hwords(dmax) * 4;
    const int st = (SC && sizeof(K) == 8) ? SP_STAGE * 8 : 0;  // staged keys
    return hb > st ? hb : st;
}
template <class K, bool SC> size_t split_smem(int k, int dmax) {
    return (size_t)split_hreg<K, SC>(dmax) + 3 * 256 * 4 + 2 * (size_t)(MsdPiece<K>::REC * RecWords<K>::v + 8) * 4 +
           (size_t)(SP_NT / 32) * split_own_bytes<K, SC>(k) + 16;
}

template <class K, bool SCATTER, bool CANON>
__global__ void __launch_bounds__(SP_NT) k_split(const uint32_t* __restrict__ bins, const Piece* __restrict__ pieces,
                                                 uint64_t n_pieces, const LargeBin* __restrict__ lbins, int k,
                                                 int dmax, uint32_t* __restrict__ table, K* __restrict__ out) {
    constexpr int REC = MsdPiece<K>::REC, RW = RecWords<K>::v;
    constexpr int RBUF = REC * RW + 8;  // words per staging buffer (+ readable slack for funnel reads)
    static_assert(REC == SP_NT, "one record per thread");
    static_assert((1 << SP_PM_DMAX) <= SP_NT, "one thread per digit in piece mode");
    extern __shared__ __align__(128) uint8_t smem[];
    __shared__ uint32_t wsum[SP_NT / 32 + 1];
    __shared__ uint32_t wtot[SP_NT / 32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int OWN = split_own_bytes<K, SCATTER>(k);
    const int HREG = split_hreg<K, SCATTER>(dmax);
    uint32_t* h = reinterpret_cast<uint32_t*>(smem);
    K* stage = reinterpret_cast<K*>(smem);  // piece mode (scatter): keys by digit
    uint32_t* gst = reinterpret_cast<uint32_t*>(smem + HREG);  // piece mode: first position of digit d
    uint32_t* lof = gst + 256;                                 // ... its offset in the stage
    uint32_t* lc = lof + 256;                                  // ... keys placed so far
    uint32_t* RB = lc + 256;
    uint8_t* own = reinterpret_cast<uint8_t*>(RB + 2 * RBUF) + warp * OWN;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(RB + 2 * RBUF) + (SP_NT / 32) * OWN);
    const uint32_t R = gridDim.x, r = blockIdx.x;
    const int U = split_unit<K>(k);
    const uint64_t p0 = (uint64_t)r * n_pieces / R, p1 = (uint64_t)(r + 1) * n_pieces / R;
    if (p0 >= p1) return;
    auto issue = [&](uint64_t p, int b) {
        const Piece pc = pieces[p];
        const uint32_t bytes = pc.nrec * RW * 4;
        mbar_expect_tx(mbar + b, bytes);
        tma_load_1d_hint(RB + b * RBUF, bins + pc.rec_begin * RW, bytes, mbar + b, l2_policy_evict_first());
    };
    if (threadIdx.x == 0) {
        mbar_init(mbar, 1);
        mbar_init(mbar + 1, 1);
        mbar_init_fence();
    }
    __syncthreads();
    if (threadIdx.x == 0) issue(p0, 0);
    uint32_t cur = 0xFFFFFFFFu;
    LargeBin lb{};
    uint64_t tab = 0;  // table index of digit 0 of the current segment
    bool pm = false, staged = false;
    uint32_t npk = 0;  // piece mode: keys of the piece
    bool bulk_pending = false;        // scatter: this thread's bulk copy may still read the stage
    uint32_t pf0 = 0, pf1 = 0;        // scatter, piece mode: prefetched table entries ...
    uint64_t pf_piece = ~0ull;        // ... of this piece
    __shared__ uint32_t s_npk;
    uint32_t* hp = lof;               // count, piece mode: this piece's digit counters (lof / lc)
    if (!SCATTER) {
        for (int d = threadIdx.x; d < 512; d += SP_NT) lof[d] = 0;  // lof and lc (adjacent)
        __syncthreads();
    }
    Piece pnext = pieces[p0];  // piece descriptors are loaded one iteration ahead
    for (uint64_t p = p0; p < p1; ++p) {
        const uint32_t it = (uint32_t)(p - p0);
        const int b = it & 1;
        if (threadIdx.x == 0 && p + 1 < p1) {
            fence_proxy_async_smem();  // buffer b^1 was released by the previous iteration's barrier
            issue(p + 1, b ^ 1);
        }
        const Piece pc = pnext;
        if (p + 1 < p1) pnext = pieces[p + 1];
        if (SCATTER && bulk_pending) {  // the previous piece's stage has been read out
            bulk_wait_read();
            bulk_pending = false;
        }
        if (pc.lbin != cur) {
            if (SCATTER) __syncthreads();  // h aliases the stage: every copy has read it
            if (!SCATTER && cur != 0xFFFFFFFFu && !pm) {
                for (int d = threadIdx.x; d < (1 << lb.D); d += SP_NT) table[tab + (uint64_t)d * lb.nseg] = h[d];
                __syncthreads();
            }
            cur = pc.lbin;
            lb = lbins[cur];
            pm = sizeof(K) == 8 && lb.pad != 0;
            if (!pm) {
                tab = lb.tb + (r - lb.first_range);
                for (int d = threadIdx.x; d < (1 << lb.D); d += SP_NT)
                    h[d] = SCATTER ? table[tab + (uint64_t)d * lb.nseg] : 0u;
            }
            __syncthreads();
        }
        const int D = (int)lb.D;
        if (pm) {
            // segment = this piece (first_range holds the bin's first piece)
            tab = lb.tb + (p - lb.first_range);
            const bool mine = threadIdx.x < (1u << D);
            if (SCATTER) {
                uint32_t c = 0;
                if (mine) {
                    uint32_t g0, g1;
                    if (pf_piece == p) {  // prefetched during the previous piece
                        g0 = pf0;
                        g1 = pf1;
                    } else {
                        const uint64_t ix = tab + (uint64_t)threadIdx.x * lb.nseg;
                        g0 = table[ix];
                        g1 = table[ix + 1];  // next entry: same digit, next piece (or next digit)
                    }
                    c = g1 - g0;
                    gst[threadIdx.x] = g0;
                }
                // stage layout: one spare slot per digit so that every digit's run starts at
                // the parity of its global position (16-byte aligned bulk copies out)
                const uint32_t cp = mine ? c + 1 : 0u;
                uint32_t P;
                if (D <= 5) {  // every digit in warp 0: shuffle scan, one barrier
                    if (warp == 0) {
                        const uint32_t inc = warp_incl_sum(cp);
                        P = inc - cp;
                        if (lane == 31) s_npk = inc;
                        if (mine) lof[lane] = lc[lane] = P + ((P ^ gst[lane]) & 1u);
                    }
                    __syncthreads();
                    npk = s_npk;
                } else {
                    P = block_excl_sum<SP_NT, uint32_t>(cp, wsum, &npk);
                    if (mine) lof[threadIdx.x] = lc[threadIdx.x] = P + ((P ^ gst[threadIdx.x]) & 1u);
                    __syncthreads();
                }
                staged = npk <= (uint32_t)SP_STAGE;  // npk: keys + one spare slot per digit
            }
            // count: the piece's counters (lof / lc alternately) were zeroed after their last use
        }
        if (SCATTER && sizeof(K) == 8 && p + 1 < p1) {
            // the next piece's table entries are loaded now and used after this piece
            const Piece pn = pnext;
            if (pn.lbin == cur && pm && threadIdx.x < (1u << D)) {
                const uint64_t ix = lb.tb + (p + 1 - lb.first_range) + (uint64_t)threadIdx.x * lb.nseg;
                pf0 = table[ix];
                pf1 = table[ix + 1];
                pf_piece = p + 1;
            }
        }
        mbar_wait(mbar + b, (it >> 1) & 1);
        // warp w expands records [32w, 32w+32) of the piece (S6): a lane takes a unit of up
        // to U consecutive windows of one record (warp scan of the records' unit counts, then
        // a unit -> lane map in SMEM).  64-bit keys: one 64-bit field holds the unit's
        // k + U - 1 <= 32 symbols; the windows' forward keys are shifts of it and their reverse
        // complements shifts of its one reversal.
        const uint32_t* Rp = RB + b * RBUF;
        const int rec = threadIdx.x;
        const uint32_t n = rec < (int)pc.nrec ? rec_nwin(Rp + rec * RW) : 0u;
        if constexpr (sizeof(K) == 8) {
            const uint32_t nu = U == 4 ? (n + 3) >> 2 : U == 2 ? (n + 1) >> 1 : U == 1 ? n : (n + 2) / 3;
          if (U == 4 && !SCATTER) {
            // count pass, block-balanced: the piece's units are numbered across the CTA (warp
            // totals -> warp offsets, one barrier; unit -> record map, a second one) and every
            // warp takes an equal share, so no warp waits at the barrier below for a warp with
            // long records (C4: 7.78 -> 7.65 ms; the scatter pass, which already has a barrier
            // before its expansion, gained nothing and keeps the per-warp map)
            constexpr int NW = SP_NT / 32;
            uint16_t* umap = reinterpret_cast<uint16_t*>(RB + 2 * RBUF);
            uint32_t* rinfo = reinterpret_cast<uint32_t*>(umap + SP_NT * ((record_max_windows(k) + 3) / 4));
            const uint32_t inc = warp_incl_sum(nu);
            if (lane == 31) wtot[warp] = inc;
            __syncthreads();
            const uint32_t wt = lane < NW ? wtot[lane] : 0u;
            const uint32_t wi = warp_incl_sum(wt);
            const uint32_t T = __shfl_sync(0xffffffffu, wi, NW - 1);
            const uint32_t pre = __shfl_sync(0xffffffffu, wi - wt, warp) + inc - nu;
            for (uint32_t j = 0; j < nu; ++j) umap[pre + j] = (uint16_t)rec;
            rinfo[rec] = pre | (n << 16);
            __syncthreads();
            const uint32_t u1 = (uint32_t)(warp + 1) * T / NW;
            for (uint32_t w = (uint32_t)warp * T / NW + lane; w < u1; w += 32) {
                {
                    const int l = umap[w];
                    const uint32_t ri = rinfo[l];
                    const int first = 4 * (int)(w - (ri & 0xFFFFu));
                    const int cnt = min(4, (int)(ri >> 16) - first);
                    const uint64_t g = bits64_be(Rp + l * RW, 8 + 2 * first);
                    const uint64_t rg = rev2_64(~g);
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        if (t < cnt) {
                            const uint64_t f = (g << (2 * t)) >> (64 - 2 * k);
                            const uint64_t rc = (rg << (64 - 2 * t - 2 * k)) >> (64 - 2 * k);
                            const uint64_t key = (f < rc || !CANON) ? f : rc;
                            const uint32_t dg = part_digit(key, D);
                            if (!pm) {
                                const uint32_t slot = atomicAdd(&h[dg], 1u);
                                if (SCATTER) out[slot] = (K)key;
                            } else if (!SCATTER) {
                                atomicAdd(&hp[dg], 1u);
                            } else {
                                const uint32_t q = atomicAdd(&lc[dg], 1u);  // stage slot (lc starts at lof)
                                if (staged) {
                                    stage[q] = (K)key;
                                } else {
                                    out[gst[dg] + (q - lof[dg])] = (K)key;
                                }
                            }
                        }
                    }
                }
            }
          } else {
            const uint32_t inc = warp_incl_sum(nu);
            const uint32_t pre = inc - nu;
            const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
            for (uint32_t j = 0; j < nu; ++j) own[pre + j] = (uint8_t)lane;
            __syncwarp();
            for (uint32_t w0 = 0; w0 < tot; w0 += 32) {
                const uint32_t w = w0 + lane;
                const int l = w < tot ? own[w] : 0;
                const uint32_t pl = __shfl_sync(0xffffffffu, pre, l), nl = __shfl_sync(0xffffffffu, n, l);
                if (w < tot) {
                    const int first = U * (int)(w - pl);
                    const int cnt = min(U, (int)nl - first);
                    const uint64_t g = bits64_be(Rp + (warp * 32 + l) * RW, 8 + 2 * first);
                    const uint64_t rg = rev2_64(~g);
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        if (t < cnt) {
                            const uint64_t f = (g << (2 * t)) >> (64 - 2 * k);
                            const uint64_t rc = (rg << (64 - 2 * t - 2 * k)) >> (64 - 2 * k);
                            const uint64_t key = (f < rc || !CANON) ? f : rc;
                            const uint32_t dg = part_digit(key, D);
                            if (!pm) {
                                const uint32_t slot = atomicAdd(&h[dg], 1u);
                                if (SCATTER) out[slot] = (K)key;
                            } else if (!SCATTER) {
                                atomicAdd(&hp[dg], 1u);
                            } else {
                                const uint32_t q = atomicAdd(&lc[dg], 1u);  // stage slot (lc starts at lof)
                                if (staged) {
                                    stage[q] = (K)key;
                                } else {
                                    out[gst[dg] + (q - lof[dg])] = (K)key;
                                }
                            }
                        }
                    }
                }
            }
          }
        } else {
            const uint32_t inc = warp_incl_sum(n);
            const uint32_t pre = inc - n;
            const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
            for (uint32_t j = 0; j < n; ++j) own[pre + j] = (uint8_t)lane;
            __syncwarp();
            for (uint32_t w0 = 0; w0 < tot; w0 += 32) {
                const uint32_t w = w0 + lane;
                const int l = w < tot ? own[w] : 0;
                const uint32_t pl = __shfl_sync(0xffffffffu, pre, l);
                if (w < tot) {
                    const K key = window_key<K>(Rp + (warp * 32 + l) * RW, (int)(w - pl), k, CANON);
                    const uint32_t slot = atomicAdd(&h[part_digit(key, D)], 1u);
                    if (SCATTER) out[slot] = key;
                }
            }
        }
        if (SCATTER && pm && staged) fence_proxy_async_smem();  // stage writes -> the bulk copies
        __syncthreads();
        if (pm) {
            if (SCATTER) {
                if (staged && threadIdx.x < (1u << D)) {
                    // digit d's run leaves by one TMA bulk copy (its aligned body) and at most
                    // two single stores (an odd head / tail element)
                    const uint32_t d = threadIdx.x, s0 = lof[d], c = lc[d] - s0;
                    const uint64_t g = gst[d];
                    if (c) {
                        uint32_t i = 0;
                        if (s0 & 1u) {
                            out[g] = stage[s0];
                            i = 1;
                        }
                        const uint32_t m = (c - i) & ~1u;
                        if (m) {
                            tma_store_1d(out + g + i, stage + s0 + i, m * (uint32_t)sizeof(K));
                            bulk_commit();
                            bulk_pending = true;
                        }
                        if (i + m < c) out[g + i + m] = stage[s0 + i + m];
                    }
                }
            } else {
                if (threadIdx.x < (1u << D)) {
                    // written and zeroed for the piece after next (double-buffered counters)
                    table[tab + (uint64_t)threadIdx.x * lb.nseg] = hp[threadIdx.x];
                    hp[threadIdx.x] = 0;
                }
                hp = (hp == lof) ? lc : lof;
            }
        }
    }
    if (!SCATTER && !pm)
        for (int d = threadIdx.x; d < (1 << lb.D); d += SP_NT) table[tab + (uint64_t)d * lb.nseg] = h[d];
    if (SCATTER && bulk_pending) bulk_wait_all();
}

// Per-digit key counts of the large bins from the scanned segment table.
__global__ void k_digit_totals(const LargeBin* __restrict__ lbins, const uint32_t* __restrict__ pos,
                               uint32_t* __restrict__ cnt, uint32_t* __restrict__ start) {
    const LargeBin lb = lbins[blockIdx.x];
    for (int d = threadIdx.x; d < (1 << lb.D); d += blockDim.x) {
        const uint32_t s0 = pos[lb.tb + (uint64_t)d * lb.nseg];
        cnt[lb.digit_base + d] = pos[lb.tb + (uint64_t)(d + 1) * lb.nseg] - s0;
        start[lb.digit_base + d] = s0;
    }
}

__global__ void k_make_pieces(const LargeBin* __restrict__ lbins, const uint64_t* __restrict__ piece_prefix,
                              uint32_t rpp, Piece* __restrict__ pieces) {
    const LargeBin lb = lbins[blockIdx.x];
    if (rpp == 0) rpp = lb.nseg;  // per-bin records per piece (k_split1 pieces sized by windows)
    const uint64_t p0 = piece_prefix[blockIdx.x], np = piece_prefix[blockIdx.x + 1] - p0;
    for (uint64_t j = threadIdx.x; j < np; j += blockDim.x) {
        const uint64_t r = j * rpp;
        const uint64_t left = lb.nrec - r;
        pieces[p0 + j] = Piece{lb.rec_off + r, (uint32_t)(left < rpp ? left : rpp), blockIdx.x};
    }
}

template <class K>
__global__ void __launch_bounds__(SB_NT, 2) k_chunk_sort(const K* __restrict__ keys, const Chunk* __restrict__ chunks,
                                                      int k, uint32_t ci, uint32_t cx, K* sk, uint32_t* sc,
                                                      unsigned long long* gstats) {
    constexpr int CAP = SmallCap<K>::v;
    extern __shared__ __align__(16) uint8_t smem[];
    K* A = reinterpret_cast<K*>(smem);
    K* B = A + CAP;
    uint32_t* whist = reinterpret_cast<uint32_t*>(B + CAP);
    uint32_t* wsum = whist + RADIX * SB_NW;
    unsigned long long* red = reinterpret_cast<unsigned long long*>(wsum + 24);
    unsigned long long* bcast = red + 4;
    unsigned int* scnt = reinterpret_cast<unsigned int*>(bcast + 1);
    const Chunk c = chunks[blockIdx.x];
    const int n = (int)c.n;
    const K* src = keys + c.begin;
    for (int i = threadIdx.x; i < n; i += SB_NT) A[i] = src[i];
    __syncthreads();
    block_sort_inplace<K, SB_NT, CAP / SB_NT, false>(A, nullptr, n, 2 * k, whist, wsum, red);
    block_rle_bitmask<K, SB_NT>(A, n, reinterpret_cast<uint32_t*>(B), ci, cx, sk, sc, gstats, wsum, scnt, bcast,
                                GS_SURV, GS_UNIQUE, GS_BELOW, GS_ABOVE);
}

// ---------------------------------------------------------------- S7-S8 by counting in SMEM
// Default counting of the large-bin chunks ("count_path 0").  The paper
// sorts a bin's k-mers and merges equal neighbours; that only
// has to produce, per distinct k-mer, its number of occurrences, and S9 sorts the
// survivors globally anyway.  Here a persistent CTA (one per SM) counts each chunk in an
// open-addressing hash table in shared memory (CAS claims a slot, atomicAdd counts).  The
// chunk's keys stream through a ring of NBUF staging buffers filled by the TMA engine
// (1-D bulk copies, evict-first), NBUF-1 sub-pieces ahead of the consumer, across chunk
// boundaries.  After a chunk, the table is scanned once: every key with
// ci <= count <= cx is a survivor; the CTA reserves its output range with one global
// atomic, writes the survivors, and clears the slots.  A chunk holds up to
// chunk_hash_cap() keys but the table only ~3/4 of its slots in distinct keys: a probe
// sequence longer than PROBE_MAX marks the chunk "overflowed" -- its partial counts are
// dropped and the chunk is listed for the device radix-sort fallback.
#ifndef KMC_CH_NT
#define KMC_CH_NT 1024
#endif
constexpr int CH_NT = KMC_CH_NT;        // threads per CTA; 1024 / CH_NT CTAs per SM
constexpr int CH_CPS = 1024 / CH_NT;
template <class K> struct HashCfg;
// slots: a multiple of CH_NT, as many as shared memory holds (the slot of a key: its 32-bit
// hash scaled to the table, so any size works).  C4: 16384 -> 18432 slots, with chunks
// planned for them, 52.6 -> 52.35 ms/step
template <> struct HashCfg<uint64_t> { static constexpr int slots = 18 * CH_NT; };
template <> struct HashCfg<K128> { static constexpr int slots = 11 * CH_NT; };

template <class K> constexpr size_t chunk_hash_smem() { return (size_t)HashCfg<K>::slots * (sizeof(K) + 4); }

template <class K>
__global__ void __launch_bounds__(CH_NT, CH_CPS) k_chunk_hash(const K* __restrict__ keys, const Chunk* __restrict__ chunks,
                                                         uint32_t n_chunks, uint32_t ci, uint32_t cx, K* sk,
                                                         uint32_t* sc, unsigned long long* gstats,
                                                         Chunk* __restrict__ overflow,
                                                         unsigned long long* __restrict__ n_overflow) {
    // Keys stream straight from HBM into registers: thread t takes the chunk's keys
    // t, t + CH_NT, ...; UNR of them are in flight while the previous UNR are inserted, and
    // the next chunk's first UNR are issued before the table of the current one is scanned.
    #ifndef KMC_CH_UNR
#define KMC_CH_UNR 2
#endif
    constexpr int TSMAX = HashCfg<K>::slots, UNR = KMC_CH_UNR;
    constexpr int NW = CH_NT / 32;
    extern __shared__ __align__(128) uint8_t smem[];
    K* T = reinterpret_cast<K*>(smem);
    uint32_t* C = reinterpret_cast<uint32_t*>(T + TSMAX);
    __shared__ int ovf;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t ltm = lanemask_lt();
    const K E = key_empty<K>();
    for (int i = threadIdx.x; i < TSMAX; i += CH_NT) {
        T[i] = E;
        C[i] = 0;
    }
    if (threadIdx.x == 0) ovf = 0;
    __syncthreads();
    const int t = threadIdx.x;
    auto fetch = [&](const Chunk& ch, uint32_t u0, K (&buf)[UNR]) {
#pragma unroll
        for (int u = 0; u < UNR; ++u) {
            const uint32_t i = t + (u0 + u) * CH_NT;
            if (i < ch.n) buf[u] = ld_stream(keys + ch.begin + i + (i >= (ch.pad & 0xFFFFu) ? ch.pad >> 16 : 0u));
        }
    };
    uint32_t uniq = 0, below = 0, above = 0;
    K cur[UNR], nxt[UNR];
    Chunk ch{};
    if (blockIdx.x < n_chunks) {
        ch = chunks[blockIdx.x];
        fetch(ch, 0, cur);
    }
    for (uint32_t cc = blockIdx.x; cc < n_chunks; cc += gridDim.x) {
        const uint32_t want = ch.n + ch.n / 3 < (uint32_t)TSMAX ? ch.n + ch.n / 3 : (uint32_t)TSMAX;
        const uint32_t TS = (want + CH_NT - 1) / CH_NT * CH_NT;  // (a multiple of CH_NT, <= TSMAX)
        const uint32_t per = (ch.n + CH_NT - 1) / CH_NT;  // keys per thread (rounded up)
        bool ok = true;
        for (uint32_t u0 = 0; u0 < per; u0 += UNR) {
            if (u0 + UNR < per) fetch(ch, u0 + UNR, nxt);
#pragma unroll
            for (int u = 0; u < UNR; ++u) {
                const uint32_t i = t + (u0 + u) * CH_NT;
                // (the one-pass split pads odd runs with EMPTY keys: skipped)
                if (i < ch.n && !key_eq(cur[u], E)) ok &= table_insert_ts<K>(T, C, TS, cur[u]);
            }
#pragma unroll
            for (int u = 0; u < UNR; ++u) cur[u] = nxt[u];
        }
        if (!ok) ovf = 1;
        // the next chunk's first keys are in flight while this table is scanned
        const Chunk done = ch;
        const uint32_t cn = cc + gridDim.x;
        if (cn < n_chunks) {
            ch = chunks[cn];
            fetch(ch, 0, cur);
        }
        __syncthreads();
        if (ovf) {
            // too many distinct keys for the table: drop the partial counts, list the chunk
            if (t == 0) overflow[atomicAdd(n_overflow, 1ull)] = done;
            for (int s = t; s < TS; s += CH_NT) {
                T[s] = E;
                C[s] = 0;
            }
            __syncthreads();
            if (t == 0) ovf = 0;
            __syncthreads();
            continue;
        }
        // the thread's slots t + i CH_NT (i < TS / CH_NT: the same for the whole block): their
        // counts stay in registers between the two passes
        constexpr int SPT = TSMAX / CH_NT;
        static_assert(TSMAX % CH_NT == 0, "whole rounds of slots");
        uint32_t cv[SPT];
        uint32_t keep = 0;
#pragma unroll
        for (int i = 0; i < SPT; ++i) {
            const uint32_t s = t + i * CH_NT;
            cv[i] = s < TS ? C[s] : 0u;
            const uint32_t c = cv[i];
            uniq += c != 0;
            below += c != 0 && c < ci;
            above += c > cx;
            keep += c != 0 && c >= ci && c <= cx;
        }
        // every warp reserves the output range of the survivors it counted (it writes the same
        // slots below): no barrier, and the atomic's round trip overlaps the other warps' work
        keep = __reduce_add_sync(0xffffffffu, keep);
        unsigned long long o = 0;
        if (lane == 0 && keep) o = atomicAdd(&gstats[GS_SURV], (unsigned long long)keep);
        o = __shfl_sync(0xffffffffu, o, 0);
#pragma unroll
        for (int i = 0; i < SPT; ++i) {
            const uint32_t s = t + i * CH_NT;
            if (s >= TS) break;  // (uniform)
            const uint32_t c = cv[i];
            const bool kp = c >= ci && c <= cx && c != 0;
            const uint32_t bb = __ballot_sync(0xffffffffu, kp);
            if (kp) {
                const unsigned long long qq = o + __popc(bb & ltm);
                sk[qq] = T[s];
                sc[qq] = c;
            }
            o += __popc(bb);
            T[s] = E;
            C[s] = 0;
        }
        __syncthreads();
    }
    uniq = __reduce_add_sync(0xffffffffu, uniq);
    below = __reduce_add_sync(0xffffffffu, below);
    above = __reduce_add_sync(0xffffffffu, above);
    if (lane == 0) {
        if (uniq) atomicAdd(&gstats[GS_UNIQUE], (unsigned long long)uniq);
        if (below) atomicAdd(&gstats[GS_BELOW], (unsigned long long)below);
        if (above) atomicAdd(&gstats[GS_ABOVE], (unsigned long long)above);
    }
}

}  // namespace

size_t chunk_key_slack_bytes() { return 16; }

int chunk_hash_cap(int k) { return k <= 32 ? HashCfg<uint64_t>::slots : HashCfg<K128>::slots; }

cudaError_t launch_chunk_hash(const void* keys, const Chunk* chunks, uint64_t n_chunks, int k, uint32_t ci,
                              uint32_t cx, void* surv_keys, uint32_t* surv_counts, unsigned long long* gstats,
                              Chunk* overflow, unsigned long long* n_overflow, int n_sms, cudaStream_t s) {
    if (n_chunks == 0) return cudaSuccess;
    if (n_chunks >= (1ull << 32)) return cudaErrorInvalidValue;
    const unsigned grid = (unsigned)std::min<uint64_t>(n_chunks, (uint64_t)std::max(1, n_sms) * CH_CPS);
    cudaError_t e;
    if (k <= 32) {
        const size_t sm = chunk_hash_smem<uint64_t>();
        if ((e = cudaFuncSetAttribute(k_chunk_hash<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)))
            return e;
        k_chunk_hash<uint64_t><<<grid, CH_NT, sm, s>>>((const uint64_t*)keys, chunks, (uint32_t)n_chunks, ci, cx,
                                                       (uint64_t*)surv_keys, surv_counts, gstats, overflow,
                                                       n_overflow);
    } else {
        const size_t sm = chunk_hash_smem<K128>();
        if ((e = cudaFuncSetAttribute(k_chunk_hash<K128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)))
            return e;
        k_chunk_hash<K128><<<grid, CH_NT, sm, s>>>((const K128*)keys, chunks, (uint32_t)n_chunks, ci, cx,
                                                   (K128*)surv_keys, surv_counts, gstats, overflow, n_overflow);
    }
    return cudaGetLastError();
}

int small_capacity(int k) { return k <= 32 ? SB_CAP64 : SB_CAP128; }

cudaError_t launch_small_bins(const SmallArgs& a, uint64_t n_small, cudaStream_t s) {
    if (n_small == 0) return cudaSuccess;
    cudaError_t e;
    if (a.k <= 32) {
        const size_t sm = small_smem_bytes<uint64_t>();
        if ((e = cudaFuncSetAttribute(k_small_bins<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)) !=
            cudaSuccess)
            return e;
        k_small_bins<uint64_t><<<(unsigned)n_small, SB_NT, sm, s>>>(a);
    } else {
        const size_t sm = small_smem_bytes<K128>();
        if ((e = cudaFuncSetAttribute(k_small_bins<K128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)) !=
            cudaSuccess)
            return e;
        k_small_bins<K128><<<(unsigned)n_small, SB_NT, sm, s>>>(a);
    }
    return cudaGetLastError();
}

cudaError_t launch_large_expand(const uint32_t* bins, const Piece* pieces, uint64_t n_pieces, int k, int canonical,
                                void* keys,
                                unsigned long long* gstats, cudaStream_t s) {
    if (n_pieces == 0) return cudaSuccess;
    if (k <= 32)
        k_large_expand<uint64_t><<<(unsigned)n_pieces, LE_NT, 0, s>>>(bins, pieces, k, canonical, (uint64_t*)keys, gstats);
    else
        k_large_expand<K128><<<(unsigned)n_pieces, LE_NT, 0, s>>>(bins, pieces, k, canonical, (K128*)keys, gstats);
    return cudaGetLastError();
}

cudaError_t launch_make_pieces(const LargeBin* lbins, const uint64_t* piece_prefix, uint64_t n_lbins,
                               uint32_t rec_per_piece, Piece* pieces, cudaStream_t s) {
    if (n_lbins == 0) return cudaSuccess;
    k_make_pieces<<<(unsigned)n_lbins, 256, 0, s>>>(lbins, piece_prefix, rec_per_piece, pieces);
    return cudaGetLastError();
}

int split_piece_mode_dmax(int k) { return k <= 32 ? SP_PM_DMAX : -1; }

int msd_piece_records(int k) { return k <= 32 ? MsdPiece<uint64_t>::REC : MsdPiece<K128>::REC; }

int msd_digit_bits(uint64_t bin_windows, int k, int cap) {
    // about cap/4 keys per digit on average (hashed digits are near-uniform, so chunks of
    // 3-4 digits fill a CTA); 1 <= D <= 12
    (void)k;
    int D = 1;
    while (D < MSD_MAXD && (bin_windows >> D) > (uint64_t)std::max(1, cap / 4)) ++D;
    return D;
}

cudaError_t launch_greedy_chunks(GreedyArgs g, uint64_t n_keys, cudaStream_t s) {
    if (g.n_digits == 0) return cudaSuccess;
    // ~64 chunks per segment: seg ~ 64 cap / (keys per digit), a power of two in [256, 8192]
    const double per = std::max(1.0, (double)n_keys / (double)g.n_digits);
    const double want = 64.0 * g.cap / per;
    int seg = 256;
    while (seg < GP_SEGMAX && seg < want) seg *= 2;
    g.seg = (uint32_t)seg;
    const uint64_t n_segments = (g.n_digits + seg - 1) / seg;
    const int sm = (int)((3 * (size_t)seg + 1) * 4);
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_greedy_chunks, cudaFuncAttributeMaxDynamicSharedMemorySize, sm))) return e;
    k_greedy_chunks<<<(unsigned)n_segments, GP_NT, sm, s>>>(g);
    return cudaGetLastError();
}

template <class K, bool SC>
cudaError_t split_t(const uint32_t* bins, const Piece* pieces, uint64_t n_pieces, const LargeBin* lbins, int k,
                    int canonical, int dmax, uint32_t n_ranges, uint32_t* table, void* keys, cudaStream_t s) {
    const int sm = (int)split_smem<K, SC>(k, dmax);
    cudaError_t e;
    if (canonical) {
        if ((e = cudaFuncSetAttribute(k_split<K, SC, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm))) return e;
        k_split<K, SC, true><<<n_ranges, SP_NT, sm, s>>>(bins, pieces, n_pieces, lbins, k, dmax, table, (K*)keys);
    } else {
        if ((e = cudaFuncSetAttribute(k_split<K, SC, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm))) return e;
        k_split<K, SC, false><<<n_ranges, SP_NT, sm, s>>>(bins, pieces, n_pieces, lbins, k, dmax, table, (K*)keys);
    }
    return cudaGetLastError();
}

cudaError_t launch_split(bool scatter, const uint32_t* bins, const Piece* pieces, uint64_t n_pieces,
                         const LargeBin* lbins, int k, int canonical, int dmax, uint32_t n_ranges, uint32_t* table,
                         void* keys, cudaStream_t s) {
    if (n_pieces == 0) return cudaSuccess;
    if (k <= 32)
        return scatter ? split_t<uint64_t, true>(bins, pieces, n_pieces, lbins, k, canonical, dmax, n_ranges, table,
                                                 keys, s)
                       : split_t<uint64_t, false>(bins, pieces, n_pieces, lbins, k, canonical, dmax, n_ranges, table,
                                                  keys, s);
    return scatter ? split_t<K128, true>(bins, pieces, n_pieces, lbins, k, canonical, dmax, n_ranges, table, keys, s)
                   : split_t<K128, false>(bins, pieces, n_pieces, lbins, k, canonical, dmax, n_ranges, table, keys, s);
}

cudaError_t launch_digit_totals(const LargeBin* lbins, uint64_t n_lbins, const uint32_t* pos, uint32_t* cnt,
                                uint32_t* start,
                                cudaStream_t s) {
    if (n_lbins == 0) return cudaSuccess;
    k_digit_totals<<<(unsigned)n_lbins, 256, 0, s>>>(lbins, pos, cnt, start);
    return cudaGetLastError();
}

cudaError_t launch_chunk_sort(const void* keys, const Chunk* chunks, uint64_t n_chunks, int k, uint32_t ci,
                              uint32_t cx, void* surv_keys, uint32_t* surv_counts, unsigned long long* gstats,
                              cudaStream_t s) {
    if (n_chunks == 0) return cudaSuccess;
    cudaError_t e;
    if (k <= 32) {
        const size_t sm = small_smem_bytes<uint64_t>();
        if ((e = cudaFuncSetAttribute(k_chunk_sort<uint64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)))
            return e;
        k_chunk_sort<uint64_t><<<(unsigned)n_chunks, SB_NT, sm, s>>>((const uint64_t*)keys, chunks, k, ci, cx,
                                                                     (uint64_t*)surv_keys, surv_counts, gstats);
    } else {
        const size_t sm = small_smem_bytes<K128>();
        if ((e = cudaFuncSetAttribute(k_chunk_sort<K128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)))
            return e;
        k_chunk_sort<K128><<<(unsigned)n_chunks, SB_NT, sm, s>>>((const K128*)keys, chunks, k, ci, cx,
                                                                 (K128*)surv_keys, surv_counts, gstats);
    }
    return cudaGetLastError();
}

uint64_t radix_tile_items(int key_words) { return key_words == 1 ? RadixTile<uint64_t>::TI : RadixTile<K128>::TI; }

size_t radix_scan_temp_bytes(uint64_t n, int key_words) {
    (void)n;
    (void)key_words;
    return 16;  // the onesweep sort needs no scan scratch
}
uint64_t radix_status_words(uint64_t n, int key_words) {
    const uint64_t ntiles = (n + radix_tile_items(key_words) - 1) / radix_tile_items(key_words);
    return 2 * RADIX * ntiles + 64;
}
uint64_t radix_aux_words() { return 32 * RADIX + 64; }

cudaError_t device_radix_sort(int key_words, void* keys, uint32_t* vals, uint64_t n, int nbits,
                              const RadixScratch& rs, cudaStream_t s, void** res_keys, uint32_t** res_vals,
                              int* n_launches) {
    if (key_words == 1)
        return radix_sort_t<uint64_t>((uint64_t*)keys, vals, n, nbits, rs, s, res_keys, res_vals, n_launches);
    return radix_sort_t<K128>((K128*)keys, vals, n, nbits, rs, s, res_keys, res_vals, n_launches);
}

cudaError_t launch_rle(int key_words, const void* keys, uint64_t n, uint32_t ci, uint32_t cx, void* surv_keys,
                       uint32_t* surv_counts, unsigned long long* gstats, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned grid = (unsigned)((n + RLE_NT * RLE_IPT - 1) / (RLE_NT * RLE_IPT));
    if (key_words == 1)
        k_rle<uint64_t><<<grid, RLE_NT, 0, s>>>((const uint64_t*)keys, n, ci, cx, (uint64_t*)surv_keys, surv_counts,
                                                gstats);
    else
        k_rle<K128><<<grid, RLE_NT, 0, s>>>((const K128*)keys, n, ci, cx, (K128*)surv_keys, surv_counts, gstats);
    return cudaGetLastError();
}

}  // namespace kmc
