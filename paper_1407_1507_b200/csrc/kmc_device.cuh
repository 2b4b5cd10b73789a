// kmc_device.cuh -- device building blocks shared by the kmcgpu kernels (sm_100a).
//
// Keys: canonical k-mer values, 2 bits per symbol, leftmost symbol most significant
// (Suppl. Sec. 4).  k <= 32 -> uint64_t; 33 <= k <= 64 -> K128 {lo, hi}.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace kmc {

constexpr int RADIX_BITS = 8;
constexpr int RADIX = 1 << RADIX_BITS;

struct __align__(16) K128 {
    uint64_t lo, hi;
};

// ---------------------------------------------------------------- key operations
__device__ __forceinline__ bool key_lt(uint64_t a, uint64_t b) { return a < b; }
__device__ __forceinline__ bool key_lt(const K128& a, const K128& b) {
    return a.hi < b.hi || (a.hi == b.hi && a.lo < b.lo);
}
__device__ __forceinline__ bool key_eq(uint64_t a, uint64_t b) { return a == b; }
__device__ __forceinline__ bool key_eq(const K128& a, const K128& b) { return a.hi == b.hi && a.lo == b.lo; }
__device__ __forceinline__ uint32_t key_digit(uint64_t a, int shift) { return (uint32_t)(a >> shift) & (RADIX - 1); }
__device__ __forceinline__ uint32_t key_digit(const K128& a, int shift) {
    return shift < 64 ? (uint32_t)(a.lo >> shift) & (RADIX - 1) : (uint32_t)(a.hi >> (shift - 64)) & (RADIX - 1);
}
// 32-bit word w (0 = least significant) of a key
__device__ __forceinline__ uint32_t key_word(uint64_t a, int w) { return w ? (uint32_t)(a >> 32) : (uint32_t)a; }
__device__ __forceinline__ uint32_t key_word(const K128& a, int w) {
    const uint64_t x = (w & 2) ? a.hi : a.lo;
    return (w & 1) ? (uint32_t)(x >> 32) : (uint32_t)x;
}
__device__ __forceinline__ uint64_t key_min(uint64_t a, uint64_t b) { return a < b ? a : b; }
__device__ __forceinline__ K128 key_min(const K128& a, const K128& b) { return key_lt(b, a) ? b : a; }

// Rolling forward / reverse-complement values of a k-mer: pushing symbol c
// (0..3) at the right end: fwd = fwd*4 + c (mod 4^k); the reverse complement gains the
// complement 3-c at its most significant position: rc = rc/4 + (3-c)*4^(k-1).
struct Roll64 {
    uint64_t fwd = 0, rc = 0, mask;
    int top;  // 2k-2
    __device__ __forceinline__ explicit Roll64(int k) {
        mask = (k >= 32) ? ~0ull : ((1ull << (2 * k)) - 1);
        top = 2 * k - 2;
    }
    __device__ __forceinline__ void push(uint32_t c) {
        fwd = ((fwd << 2) | c) & mask;
        rc = (rc >> 2) | ((uint64_t)(3u - c) << top);
    }
    __device__ __forceinline__ uint64_t canon() const { return fwd < rc ? fwd : rc; }
    __device__ __forceinline__ uint64_t key(bool canonical) const { return canonical ? canon() : fwd; }
};

struct Roll128 {  // 33 <= k <= 64
    uint64_t flo = 0, fhi = 0, rlo = 0, rhi = 0, hmask;
    int htop;  // 2k-2-64
    __device__ __forceinline__ explicit Roll128(int k) {
        int hb = 2 * k - 64;
        hmask = (hb >= 64) ? ~0ull : ((1ull << hb) - 1);
        htop = 2 * k - 2 - 64;
    }
    __device__ __forceinline__ void push(uint32_t c) {
        fhi = ((fhi << 2) | (flo >> 62)) & hmask;
        flo = (flo << 2) | c;
        rlo = (rlo >> 2) | (rhi << 62);
        rhi = (rhi >> 2) | ((uint64_t)(3u - c) << htop);
    }
    __device__ __forceinline__ K128 canon() const {
        K128 f{flo, fhi}, r{rlo, rhi};
        return key_lt(r, f) ? r : f;
    }
    __device__ __forceinline__ K128 key(bool canonical) const { return canonical ? canon() : K128{flo, fhi}; }
};

template <class K> struct RollFor;
template <> struct RollFor<uint64_t> { using T = Roll64; };
template <> struct RollFor<K128> { using T = Roll128; };

// ---------------------------------------------------------------- signature rule
// P:L206-208 (Sec. 2.2): canonical minimizers that "do not start with AAA, neither start
// with ACA, neither contain AA anywhere except at their beginning" -- applied to the
// canonical p-mer x (2p bits, leftmost symbol most significant).  isA marks the low bit
// of every 2-bit group equal to 00; aa marks adjacent A pairs, the pair at positions
// (0,1) removed.
__device__ __forceinline__ bool sig_allowed(uint32_t x, int p) {
    if (p < 3) return true;  // no 3-symbol prefix and no AA pair after position 0 exist
    uint32_t m2 = (p >= 16) ? 0xFFFFFFFFu : ((1u << (2 * p)) - 1);
    uint32_t isA = ~(x | (x >> 1)) & 0x55555555u & m2;
    uint32_t aa = isA & (isA >> 2) & ~(1u << (2 * (p - 2)));
    uint32_t pre3 = x >> (2 * (p - 3));
    return aa == 0 && pre3 != 0u && pre3 != 4u;
}

// ---------------------------------------------------------------- record format (bins)
// A bin record holds a piece of one super-k-mer: RW 32-bit words, big-endian bit string:
// bits [0,8) = number of windows n (1..255); bits [8+2j, 10+2j) = symbol j.
// RW = 4 (60 symbols) for k <= 32, RW = 8 (124 symbols) for k >= 33.
__host__ __device__ __forceinline__ int record_words(int k) { return k <= 32 ? 4 : 8; }
__host__ __device__ __forceinline__ int record_max_windows(int k) { return 16 * record_words(k) - 4 - k + 1; }

__device__ __forceinline__ uint32_t rec_nwin(const uint32_t* rec) { return rec[0] >> 24; }

template <class K> struct RecWords;
template <> struct RecWords<uint64_t> { static constexpr int v = 4; };
template <> struct RecWords<K128> { static constexpr int v = 8; };

// Calls emit(w, key) for the windows w = 0..n-1 of a record held in registers: the
// canonical key min(fwd, rc) of every window.  The symbol loop is fully
// unrolled so every symbol's word and shift are compile-time constants.
template <class K, int RW, class F>
__device__ __forceinline__ void for_each_window(const uint32_t (&wd)[RW], int k, bool canonical, F&& emit) {
    typename RollFor<K>::T roll(k);
    const int nb = (int)(wd[0] >> 24) + k - 1;
#pragma unroll
    for (int j = 0; j < 16 * RW - 4; ++j) {
        if (j >= nb) break;
        const int g = 8 + 2 * j;
        roll.push((wd[g >> 5] >> (30 - (g & 31))) & 3u);
        if (j >= k - 1) emit(j - (k - 1), roll.key(canonical));
    }
}

// ---------------------------------------------------------------- window-parallel expansion
// Canonical key of window j of a record in shared memory, computed directly from the
// packed bits (no rolling): fwd = the 2k-bit field at bit 8+2j of the record's big-endian
// bit string; rc = complement, 2-bit groups reversed.  One lane per window, so
// records of different lengths do not idle the lanes of a warp.
__device__ __forceinline__ uint64_t rev2_64(uint64_t x) {  // reverse the order of the 2-bit groups
    x = __brevll(x);
    return ((x >> 1) & 0x5555555555555555ull) | ((x & 0x5555555555555555ull) << 1);
}
// bits [b, b+64) of a big-endian bit string in shared memory words (b + 64 <= 32 * words)
__device__ __forceinline__ uint64_t bits64_be(const uint32_t* w, int b) {
    const int q = b >> 5, r = b & 31;
    const uint32_t w0 = w[q], w1 = w[q + 1], w2 = w[q + 2];
    const uint32_t hi = __funnelshift_l(w1, w0, r), lo = __funnelshift_l(w2, w1, r);
    return ((uint64_t)hi << 32) | lo;
}
template <class K> __device__ __forceinline__ K window_key(const uint32_t* rec, int j, int k, bool canonical);
template <>
__device__ __forceinline__ uint64_t window_key<uint64_t>(const uint32_t* rec, int j, int k, bool canonical) {
    // field of 2k <= 64 bits starting at bit 8+2j; the record has 4 words (+1 readable pad)
    const uint64_t f = bits64_be(rec, 8 + 2 * j) >> (64 - 2 * k);
    const uint64_t r = rev2_64(~f) >> (64 - 2 * k);
    return (f < r || !canonical) ? f : r;
}
template <> __device__ __forceinline__ K128 window_key<K128>(const uint32_t* rec, int j, int k, bool canonical) {
    // 2k in (64, 128] bits at bit b = 8+2j: hi part = first 2k-64 bits, lo part = next 64
    const int b = 8 + 2 * j, hb = 2 * k - 64;
    K128 f;
    f.hi = bits64_be(rec, b) >> (64 - hb);
    f.lo = bits64_be(rec, b + hb);
    // rc: reverse the 2k-bit string of complemented groups: lo' = rev of hi.. parts
    const uint64_t nl = ~f.lo, nh = ~f.hi;  // complement (upper bits of nh beyond hb are junk)
    // full 128-bit value V = nh:nl (hb + 64 bits used).  rev2 over 128 bits = (rev2(nl), rev2(nh)),
    // then shift right by 128 - 2k = 64 - hb.
    const uint64_t a = rev2_64(nl), c = rev2_64(nh);  // a = high word of reversed, c = low word
    const int sh = 64 - hb;                           // 0 <= sh < 64
    K128 r;
    r.lo = sh ? ((c >> sh) | (a << (64 - sh))) : c;
    r.hi = sh ? (a >> sh) : a;
    return (key_lt(r, f) && canonical) ? r : f;
}

// Digit of the large-bin split: a multiplicative hash of the whole key (equal keys share
// a digit; the top bits of a key are a poor digit, see k_sort.cu).  1 <= D <= 12.
__device__ __forceinline__ uint32_t part_digit(uint64_t key, int D) {
    const uint32_t h = (((uint32_t)(key >> 32) * 0x85EBCA6Bu) ^ (uint32_t)key) * 0x9E3779B1u;
    return h >> (32 - D);
}
__device__ __forceinline__ uint32_t part_digit(const K128& key, int D) {
    const uint32_t h = (((uint32_t)(key.hi >> 32) * 0x27D4EB2Fu) ^ ((uint32_t)key.hi * 0xC2B2AE35u) ^
                        ((uint32_t)(key.lo >> 32) * 0x85EBCA6Bu) ^ (uint32_t)key.lo) *
                       0x9E3779B1u;
    return h >> (32 - D);
}

// Loads a record (16-byte aligned, RW words) into registers.
template <int RW>
__device__ __forceinline__ void load_record(const uint32_t* rec, uint32_t (&wd)[RW]) {
#pragma unroll
    for (int q = 0; q < RW / 4; ++q) {
        const uint4 v = reinterpret_cast<const uint4*>(rec)[q];
        wd[4 * q] = v.x;
        wd[4 * q + 1] = v.y;
        wd[4 * q + 2] = v.z;
        wd[4 * q + 3] = v.w;
    }
}
__device__ __forceinline__ uint32_t rec_sym(const uint32_t* rec, int j) {
    int g = 8 + 2 * j;
    return (rec[g >> 5] >> (30 - (g & 31))) & 3u;
}

// ---------------------------------------------------------------- TMA bulk copy + mbarrier
// 1-D bulk copies global -> shared (cp.async.bulk, the TMA engine) completing on an
// mbarrier with a transaction byte count.  src, dst and bytes must be multiples of 16.
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* m, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(m)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_init_fence() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* m, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(m)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tma_load_1d(void* dst, const void* src, uint32_t bytes, uint64_t* m) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_addr(dst)),
                 "l"(src), "r"(bytes), "r"(smem_addr(m))
                 : "memory");
}
// Same, with an L2 eviction-priority hint (a streaming source read once: evict_first, so
// it does not push out lines the kernel still writes, e.g. partial sectors being filled).
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ void tma_load_1d_hint(void* dst, const void* src, uint32_t bytes, uint64_t* m,
                                                 uint64_t policy) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
            smem_addr(dst)),
        "l"(src), "r"(bytes), "r"(smem_addr(m)), "l"(policy)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* m, uint32_t parity) {
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}" ::"r"(
            smem_addr(m)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* m) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_addr(m)) : "memory");
}
// Named barrier over the first nthreads threads (a multiple of 32) of the CTA.
__device__ __forceinline__ void named_bar_sync(int id, int nthreads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}
// Orders earlier generic-proxy shared-memory accesses before later async-proxy (TMA) ones.
// 1-D bulk copy shared -> global by the TMA engine (bulk-group completion): 16-byte aligned
// addresses, bytes a multiple of 16.  bulk_wait_read(): the source may be overwritten.
__device__ __forceinline__ void tma_store_1d(void* gdst, const void* ssrc, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(gdst), "r"(smem_addr(ssrc)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Streaming (evict-first) global loads of keys.
__device__ __forceinline__ uint64_t ld_stream(const uint64_t* p) {
    return __ldcs(reinterpret_cast<const unsigned long long*>(p));
}
__device__ __forceinline__ K128 ld_stream(const K128* p) {
    const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2*>(p));
    return K128{v.x, v.y};
}

// ---------------------------------------------------------------- shared-memory hash table
// Slot hash of a key for a table of 2^lg slots: two multiply-xorshift rounds, independent
// of part_digit (the chunk's keys share their part_digit).
__device__ __forceinline__ uint32_t slot_hash(uint64_t key, int lg) {
    // two 32-bit multiply rounds (the high half mixed in first); constants differ from
    // part_digit's so a chunk's common digit bits do not bias the slots
    const uint32_t h = (((uint32_t)(key >> 32) * 0x2C1B3C6Du) ^ (uint32_t)key) * 0x297A2D39u;
    return (h ^ (h >> 16)) * 0x7FEB352Du >> (32 - lg);
}
__device__ __forceinline__ uint32_t slot_hash(const K128& key, int lg) {
    uint64_t x = (key.lo ^ (key.hi * 0xC2B2AE3D27D4EB4Full)) * 0xFF51AFD7ED558CCDull;
    x ^= x >> 32;
    x *= 0x9E3779B97F4A7C15ull;
    return (uint32_t)(x >> (64 - lg));
}
// Empty-slot marker: all ones.  It is never a canonical key: the all-T k-mer's reverse
// complement (all A = 0) is smaller.
template <class K> __device__ __forceinline__ K key_empty();
template <> __device__ __forceinline__ uint64_t key_empty<uint64_t>() { return ~0ull; }
template <> __device__ __forceinline__ K128 key_empty<K128>() { return K128{~0ull, ~0ull}; }

__device__ __forceinline__ uint64_t smem_load_volatile(const uint64_t* p) {
    return *reinterpret_cast<const volatile uint64_t*>(p);
}
__device__ __forceinline__ K128 smem_load_volatile(const K128* p) {
    K128 r;
    asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(r.lo), "=l"(r.hi) : "r"(smem_addr(p)));
    return r;
}
// Claims an empty slot for key; returns the slot's previous content.
__device__ __forceinline__ uint64_t smem_cas_empty(uint64_t* p, uint64_t key) {
    return atomicCAS(reinterpret_cast<unsigned long long*>(p), ~0ull, (unsigned long long)key);
}
__device__ __forceinline__ K128 smem_cas_empty(K128* p, const K128& key) {
    K128 o;
    const uint64_t e = ~0ull;
    asm volatile(
        "{\n .reg .b128 c, n, o;\n mov.b128 c, {%2, %3};\n mov.b128 n, {%4, %5};\n"
        " atom.shared.cas.b128 o, [%6], c, n;\n mov.b128 {%0, %1}, o;\n}"
        : "=l"(o.lo), "=l"(o.hi)
        : "l"(e), "l"(e), "l"(key.lo), "l"(key.hi), "r"(smem_addr(p))
        : "memory");
    return o;
}

constexpr int PROBE_MAX = 256;

// Counts key; false if no slot was found within PROBE_MAX probes (table too full).
template <class K>
__device__ __forceinline__ bool table_insert_bounded(K* T, uint32_t* C, int lg, const K& key) {
    const uint32_t mask = (1u << lg) - 1;
    const K E = key_empty<K>();
    uint32_t s = slot_hash(key, lg);
    for (int pr = 0; pr < PROBE_MAX; ++pr) {
        // one shared CAS per probe: it claims an empty slot, or returns the key that holds it
        const K old = smem_cas_empty(&T[s], key);
        if (key_eq(old, E) || key_eq(old, key)) {
            atomicAdd(&C[s], 1u);
            return true;
        }
        s = (s + 1) & mask;
    }
    return false;
}
// The same for a table of TS slots (any TS): slot = the 32-bit hash scaled to [0, TS).
// Double hashing: the probe step is 1 + 6 j (j = the hash's low 7 bits; the slot comes from
// its high bits).  The step is odd, so with TS = 1024 m its cycle has TS / gcd(step, m) >= 1024
// slots, more than PROBE_MAX probes visit.
template <class K>
__device__ __forceinline__ bool table_insert_ts(K* T, uint32_t* C, uint32_t TS, const K& key) {
    const K E = key_empty<K>();
    const uint32_t h = slot_hash(key, 32);
    uint32_t s = (uint32_t)(((uint64_t)h * TS) >> 32);
    const uint32_t step = 1u + 6u * (h & 127u);
    for (int pr = 0; pr < PROBE_MAX; ++pr) {
        const K old = smem_cas_empty(&T[s], key);
        if (key_eq(old, E) || key_eq(old, key)) {
            atomicAdd(&C[s], 1u);
            return true;
        }
        s += step;
        if (s >= TS) s -= TS;
    }
    return false;
}

// ---------------------------------------------------------------- warp / block helpers
__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm volatile("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

template <class T> __device__ __forceinline__ T warp_incl_sum(T v) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T n = __shfl_up_sync(0xffffffffu, v, o);
        if (lane >= o) v += n;
    }
    return v;
}

// Exclusive block-wide sum; wsum needs NT/32 + 1 entries of T.  All threads must call.
template <int NT, class T> __device__ __forceinline__ T block_excl_sum(T v, T* wsum, T* total) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    T inc = warp_incl_sum(v);
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        T w = (lane < NW) ? wsum[lane] : T(0);
        T wi = warp_incl_sum(w);
        if (lane < NW) wsum[lane] = wi - w;
        if (lane == NW - 1) wsum[NW] = wi;
    }
    __syncthreads();
    T r = wsum[warp] + inc - v;
    if (total) *total = wsum[NW];
    __syncthreads();
    return r;
}

// Exclusive block-wide sum with ONE barrier: wsum (NT/32 entries) must not be reused by
// another call until every thread has returned from this one (alternate two buffers, or
// separate the calls by a barrier).  All threads must call.
template <int NT, class T> __device__ __forceinline__ T block_excl_sum1(T v, T* wsum, T* total) {
    constexpr int NW = NT / 32;
    static_assert(NW <= 32, "one warp holds the warp totals");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const T inc = warp_incl_sum(v);
    if (lane == 31) wsum[warp] = inc;
    __syncthreads();
    const T wt = lane < NW ? wsum[lane] : T(0);
    const T wi = warp_incl_sum(wt);
    const T before = __shfl_sync(0xffffffffu, wi - wt, warp);
    *total = __shfl_sync(0xffffffffu, wi, NW - 1);
    return before + inc - v;
}

template <int NT, class T> __device__ __forceinline__ T block_sum(T v, T* wsum) {
    T tot;
    block_excl_sum<NT, T>(v, wsum, &tot);
    return tot;
}

// ---------------------------------------------------------------- block radix pass
// One stable counting-sort pass of n (<= 65535*NW) keys (and optional uint32 values)
// from src to dst in shared memory, by the 8-bit digit at `shift`.  Warp w owns the
// contiguous segment [w*seg, (w+1)*seg); within a round of 32 keys, ranks come from
// __match_any_sync peers, so the pass is stable.  whist: RADIX*NW uint32 (digit-major),
// wsum: NT/32+1 uint32.  If dstart != nullptr it receives the start of every digit
// (RADIX+1 entries).
template <class K, int NT, bool VALS>
__device__ __forceinline__ void block_digit_pass(const K* src, K* dst, const uint32_t* vsrc, uint32_t* vdst,
                                                 int n, int shift, uint32_t* whist, uint32_t* wsum,
                                                 uint32_t* dstart) {
    constexpr int NW = NT / 32;
    constexpr int IPT = RADIX * NW / NT;  // 8
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < RADIX * NW; i += NT) whist[i] = 0;
    __syncthreads();
    int seg = (n + NW - 1) / NW;
    seg = (seg + 31) & ~31;
    const int beg = warp * seg, end = min(n, beg + seg);
    for (int base = beg; base < end; base += 32) {
        const int i = base + lane;
        const bool ok = i < end;
        const uint32_t d = ok ? key_digit(src[i], shift) : (uint32_t)(RADIX + lane);
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        if (ok && lane == __ffs(peers) - 1) whist[d * NW + warp] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    uint32_t loc[IPT];
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        loc[j] = whist[threadIdx.x * IPT + j];
        s += loc[j];
    }
    uint32_t ex = block_excl_sum<NT, uint32_t>(s, wsum, nullptr);
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        whist[threadIdx.x * IPT + j] = ex;
        ex += loc[j];
    }
    __syncthreads();
    if (dstart) {
        for (int d = threadIdx.x; d < RADIX; d += NT) dstart[d] = whist[d * NW];
        if (threadIdx.x == 0) dstart[RADIX] = n;
    }
    const uint32_t ltm = lanemask_lt();
    for (int base = beg; base < end; base += 32) {
        const int i = base + lane;
        const bool ok = i < end;
        K key;
        uint32_t d = (uint32_t)(RADIX + lane);
        if (ok) {
            key = src[i];
            d = key_digit(key, shift);
        }
        const uint32_t peers = __match_any_sync(0xffffffffu, d);
        if (ok) {
            const uint32_t off = whist[d * NW + warp] + __popc(peers & ltm);
            dst[off] = key;
            if (VALS) vdst[off] = vsrc[i];
        }
        __syncwarp();
        if (ok && lane == __ffs(peers) - 1) whist[d * NW + warp] += __popc(peers);
        __syncwarp();
    }
    __syncthreads();
}

// Bitwise OR and AND over n keys in shared memory (to skip constant digits).
__device__ __forceinline__ void key_or_and_accum(uint64_t k, uint64_t& o, uint64_t& a, uint64_t&, uint64_t&) {
    o |= k;
    a &= k;
}
__device__ __forceinline__ void key_or_and_accum(const K128& k, uint64_t& o, uint64_t& a, uint64_t& oh, uint64_t& ah) {
    o |= k.lo;
    a &= k.lo;
    oh |= k.hi;
    ah &= k.hi;
}

// Varying-bit mask of the keys (lo word, hi word); red needs 4 uint64 of shared memory.
template <class K, int NT>
__device__ __forceinline__ void block_varying_bits(const K* keys, int n, unsigned long long* red, uint64_t& vlo,
                                                   uint64_t& vhi) {
    if (threadIdx.x == 0) {
        red[0] = 0;
        red[1] = ~0ull;
        red[2] = 0;
        red[3] = ~0ull;
    }
    __syncthreads();
    uint64_t o = 0, a = ~0ull, oh = 0, ah = ~0ull;
    for (int i = threadIdx.x; i < n; i += NT) key_or_and_accum(keys[i], o, a, oh, ah);
    {
        const unsigned FULL = 0xffffffffu;
        o = ((uint64_t)__reduce_or_sync(FULL, (unsigned)(o >> 32)) << 32) | __reduce_or_sync(FULL, (unsigned)o);
        a = ((uint64_t)__reduce_and_sync(FULL, (unsigned)(a >> 32)) << 32) | __reduce_and_sync(FULL, (unsigned)a);
        oh = ((uint64_t)__reduce_or_sync(FULL, (unsigned)(oh >> 32)) << 32) | __reduce_or_sync(FULL, (unsigned)oh);
        ah = ((uint64_t)__reduce_and_sync(FULL, (unsigned)(ah >> 32)) << 32) | __reduce_and_sync(FULL, (unsigned)ah);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicOr(&red[0], (unsigned long long)o);
        atomicAnd(&red[1], (unsigned long long)a);
        atomicOr(&red[2], (unsigned long long)oh);
        atomicAnd(&red[3], (unsigned long long)ah);
    }
    __syncthreads();
    vlo = red[0] ^ red[1];
    vhi = red[2] ^ red[3];
    if (n == 0) vlo = vhi = 0;
    __syncthreads();
}

__device__ __forceinline__ bool digit_varies(uint64_t vlo, uint64_t vhi, int shift) {
    return shift < 64 ? ((vlo >> shift) & (RADIX - 1)) != 0 : ((vhi >> (shift - 64)) & (RADIX - 1)) != 0;
}

// LSD radix sort of n keys (+ optional values) in shared memory over bits [0, nbits),
// skipping digits that are constant across the keys.  Returns 0 if the result is in
// (a, va), 1 if in (b, vb).
template <class K, int NT, bool VALS>
__device__ __forceinline__ int block_radix_sort(K* a, K* b, uint32_t* va, uint32_t* vb, int n, int nbits,
                                                uint32_t* whist, uint32_t* wsum, unsigned long long* red) {
    uint64_t vlo, vhi;
    block_varying_bits<K, NT>(a, n, red, vlo, vhi);
    int cur = 0;
    for (int shift = 0; shift < nbits; shift += RADIX_BITS) {
        if (!digit_varies(vlo, vhi, shift)) continue;
        if (cur == 0)
            block_digit_pass<K, NT, VALS>(a, b, va, vb, n, shift, whist, wsum, nullptr);
        else
            block_digit_pass<K, NT, VALS>(b, a, vb, va, n, shift, whist, wsum, nullptr);
        cur ^= 1;
    }
    return cur;
}

// Exclusive scan, in place, of RADIX*NW digit-major warp counters (IPT per thread).
template <int NT>
__device__ __forceinline__ void block_scan_whist(uint32_t* whist, uint32_t* wsum) {
    constexpr int NW = NT / 32;
    constexpr int IPT = RADIX * NW / NT;
    uint32_t loc[IPT];
    uint32_t s = 0;
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        loc[j] = whist[threadIdx.x * IPT + j];
        s += loc[j];
    }
    uint32_t ex = block_excl_sum<NT, uint32_t>(s, wsum, nullptr);
#pragma unroll
    for (int j = 0; j < IPT; ++j) {
        whist[threadIdx.x * IPT + j] = ex;
        ex += loc[j];
    }
    __syncthreads();
}

// Largest value of a key with nbits bits (sorts after every real key in every digit).
template <class K> __device__ __forceinline__ K key_sentinel(int nbits);
template <> __device__ __forceinline__ uint64_t key_sentinel<uint64_t>(int nbits) {
    return nbits >= 64 ? ~0ull : ((1ull << nbits) - 1);
}
template <> __device__ __forceinline__ K128 key_sentinel<K128>(int nbits) {
    K128 s;
    s.lo = nbits >= 64 ? ~0ull : ((1ull << nbits) - 1);
    s.hi = nbits >= 128 ? ~0ull : (nbits > 64 ? ((1ull << (nbits - 64)) - 1) : 0ull);
    return s;
}

// In-place LSD radix sort of n <= NT*KPT keys (+ optional uint32 values) in shared memory
// over bits [0, nbits), 8-bit digits, constant digits skipped.  The keys are padded with
// sentinels to rounds*NT (A needs that capacity); warp w owns positions
// [w*32*rounds, (w+1)*32*rounds).  Per pass every key is read once into registers and
// ranked once: __match_any_sync gives its peers in the round (the peer with no lower peer
// is the leader), the warp's running digit counter -- read before the leader adds the
// round's peers -- gives the keys of earlier rounds; after the block-wide scan of the
// warp-major counters the key is stored straight to its final position.  Rounds are
// processed in position order, so every pass is stable and the sentinels stay last.
template <class K, int NT, int KPT, bool VALS>
__device__ __forceinline__ void block_sort_inplace(K* A, uint32_t* VA, int n, int nbits, uint32_t* whist,
                                                   uint32_t* wsum, unsigned long long* red) {
    constexpr int NW = NT / 32;
    static_assert(NT >= RADIX, "one thread per digit in the scan");
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t ltm = lanemask_lt();
    uint64_t vlo, vhi;
    block_varying_bits<K, NT>(A, n, red, vlo, vhi);
    const int rounds = (n + NT - 1) / NT;
    const int m = rounds * NT;
    {
        const K sent = key_sentinel<K>(nbits);
        for (int i = n + threadIdx.x; i < m; i += NT) {
            A[i] = sent;
            if (VALS) VA[i] = 0;
        }
    }
    __syncthreads();  // the padding is read by the owners of the warp segments
    const int wbase = warp * rounds * 32;
    uint32_t* wh = whist + warp * RADIX;
    for (int shift = 0; shift < nbits; shift += RADIX_BITS) {
        if (!digit_varies(vlo, vhi, shift)) continue;
        // the digit lives in one 32-bit word of the key: word index and in-word shift
        const int wsel = shift >> 5, wsh = shift & 31;
        for (int i = threadIdx.x; i < RADIX * NW / 4; i += NT) reinterpret_cast<uint4*>(whist)[i] = make_uint4(0, 0, 0, 0);
        K key[KPT];
        uint32_t val[KPT];
        uint32_t rank[KPT];
#pragma unroll
        for (int r = 0; r < KPT; ++r) {
            if (r >= rounds) break;
            key[r] = A[wbase + r * 32 + lane];
            if (VALS) val[r] = VA[wbase + r * 32 + lane];
        }
        __syncthreads();
        // rank: peers of the round from __match_any_sync; the warp's running counter (read
        // by all peers before the round's leader -- the peer with no lower peer -- adds the
        // round's count) gives the keys of earlier rounds.  Rounds in order => stable.
#pragma unroll
        for (int r = 0; r < KPT; ++r) {
            if (r >= rounds) break;
            const uint32_t d = (key_word(key[r], wsel) >> wsh) & (RADIX - 1);
            const uint32_t peers = __match_any_sync(0xffffffffu, d);
            const uint32_t below = __popc(peers & ltm);
            const uint32_t pre = wh[d];
            __syncwarp();
            if (below == 0) wh[d] = pre + __popc(peers);
            __syncwarp();
            rank[r] = ((pre + below) << 8) | d;  // rank < 2^16 (n <= NT*KPT), digit < 2^8
        }
        __syncthreads();
        // digit-major exclusive offsets from the warp-major counters (thread t < RADIX owns digit t)
        {
            uint32_t c[NW];
            uint32_t tot = 0;
            if (threadIdx.x < RADIX) {
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    c[w] = whist[w * RADIX + threadIdx.x];
                    tot += c[w];
                }
            }
            uint32_t run = block_excl_sum<NT, uint32_t>(threadIdx.x < RADIX ? tot : 0u, wsum, nullptr);
            if (threadIdx.x < RADIX) {
#pragma unroll
                for (int w = 0; w < NW; ++w) {
                    whist[w * RADIX + threadIdx.x] = run;
                    run += c[w];
                }
            }
            __syncthreads();
        }
#pragma unroll
        for (int r = 0; r < KPT; ++r) {
            if (r >= rounds) break;
            const uint32_t pos = wh[rank[r] & (RADIX - 1)] + (rank[r] >> 8);
            A[pos] = key[r];
            if (VALS) VA[pos] = val[r];
        }
        __syncthreads();
    }
}

// Length of the run starting at i (its start bit is set): distance to the next start bit.
__device__ __forceinline__ uint32_t rle_run_length(const uint32_t* bits, int i) {
    const int pos = i + 1;
    int wd = pos >> 5;
    uint32_t m = bits[wd] & (0xFFFFFFFFu << (pos & 31));
    while (m == 0) m = bits[++wd];
    return (uint32_t)(wd * 32 + __ffs(m) - 1 - i);
}

// Run-length compaction of the sorted keys S[0..n) with the cutoffs ci <= count <= cx
// (S8).  bits: (n+32)/32 + 4 + 4*NW/32 uint32 of scratch.  Run starts are found with warp ballots; a
// run's length is the distance to the next start bit.  The CTA's survivors are counted
// first and their output range is reserved with ONE global atomic per CTA (a per-warp
// atomic on the shared survivor cursor serialises at one L2 address: it was the bottleneck
// of the chunk kernel); then every warp writes its survivors at its scanned offset.
template <class K, int NT>
__device__ __forceinline__ void block_rle_bitmask(const K* S, int n, uint32_t* bits, uint32_t ci, uint32_t cx,
                                                  K* out_keys, uint32_t* out_counts, unsigned long long* gstats,
                                                  uint32_t* wsum, unsigned int* scnt, unsigned long long* bcast,
                                                  int gs_surv, int gs_unique, int gs_below, int gs_above) {
    constexpr int NW = NT / 32;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int nwords = (n + 32) / 32;  // covers the sentinel bit n
    for (int base = (threadIdx.x & ~31); base < nwords * 32; base += NT) {
        const int i = base + lane;
        const bool st = i < n ? (i == 0 || !key_eq(S[i], S[i - 1])) : (i == n);
        const uint32_t b = __ballot_sync(0xffffffffu, st);
        if (lane == 0) bits[base >> 5] = b;
    }
    __syncthreads();
    // pass A: unique / below / above / kept per warp
    uint32_t uniq = 0, below = 0, above = 0, keep = 0;
    for (int i0 = warp * 32; i0 < n; i0 += NT) {
        const int i = i0 + lane;
        if (i < n && ((bits[i0 >> 5] >> lane) & 1u)) {
            const uint32_t run = rle_run_length(bits, i);
            ++uniq;
            if (run < ci) ++below;
            else if (run > cx) ++above;
            else ++keep;
        }
    }
    uniq = __reduce_add_sync(0xffffffffu, uniq);
    below = __reduce_add_sync(0xffffffffu, below);
    above = __reduce_add_sync(0xffffffffu, above);
    keep = __reduce_add_sync(0xffffffffu, keep);
    // scratch after the bitmask: NW u64 warp offsets, then NW u32 kept + NW u32 unique
    unsigned long long* woff = reinterpret_cast<unsigned long long*>(bits + ((nwords + 2) & ~1));
    uint32_t* wkeep = reinterpret_cast<uint32_t*>(woff + NW);
    if (lane == 0) {
        wkeep[warp] = keep;
        wkeep[NW + warp] = uniq;
    }
    (void)wsum;
    (void)scnt;
    (void)bcast;
    __syncthreads();
    if (warp == 0) {
        const uint32_t kw = lane < NW ? wkeep[lane] : 0u;
        const uint32_t inc = warp_incl_sum(kw);
        const uint32_t tu = __reduce_add_sync(0xffffffffu, lane < NW ? wkeep[NW + lane] : 0u);
        unsigned long long b0 = 0;
        if (lane == NW - 1 && inc) b0 = atomicAdd(&gstats[gs_surv], (unsigned long long)inc);
        b0 = __shfl_sync(0xffffffffu, b0, NW - 1);
        if (lane < NW) woff[lane] = b0 + inc - kw;
        if (lane == 0 && tu) atomicAdd(&gstats[gs_unique], (unsigned long long)tu);
    }
    if (lane == 0) {
        if (below) atomicAdd(&gstats[gs_below], (unsigned long long)below);
        if (above) atomicAdd(&gstats[gs_above], (unsigned long long)above);
    }
    __syncthreads();
    if (keep == 0) return;
    // pass B: write survivors at the warp's reserved offset, in position order
    unsigned long long slot = woff[warp];
    const uint32_t ltm = lanemask_lt();
    for (int i0 = warp * 32; i0 < n; i0 += NT) {
        const int i = i0 + lane;
        uint32_t run = 0;
        if (i < n && ((bits[i0 >> 5] >> lane) & 1u)) {
            run = rle_run_length(bits, i);
            if (run < ci || run > cx) run = 0;
        }
        const uint32_t b = __ballot_sync(0xffffffffu, run != 0);
        if (run) {
            const unsigned long long o = slot + __popc(b & ltm);
            out_keys[o] = S[i];
            out_counts[o] = run;
        }
        slot += __popc(b);
    }
}

// Per-window record lookup for a piece of nrec records (RW words each) in shared memory:
// wpos[r] = first window of record r in the piece, own[w] = record of window w.  Returns the
// piece's window count.  All threads must call; ends with __syncthreads().
template <int NT>
__device__ __forceinline__ int piece_window_map(const uint32_t* R, int nrec, int RW, uint32_t* wpos, uint16_t* own,
                                                uint32_t* wsum) {
    const int rpt = (nrec + NT - 1) / NT;
    const int r0 = threadIdx.x * rpt, r1 = min(nrec, r0 + rpt);
    uint32_t s = 0;
    for (int r = r0; r < r1; ++r) s += rec_nwin(R + r * RW);
    uint32_t total;
    uint32_t pos = block_excl_sum<NT, uint32_t>(s, wsum, &total);
    for (int r = r0; r < r1; ++r) {
        const uint32_t n = rec_nwin(R + r * RW);
        wpos[r] = pos;
        for (uint32_t j = 0; j < n; ++j) own[pos + j] = (uint16_t)r;
        pos += n;
    }
    __syncthreads();
    return (int)total;
}

}  // namespace kmc
