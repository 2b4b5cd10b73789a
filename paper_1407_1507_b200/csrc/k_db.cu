// k_db.cu -- KMC 2 database writer: the (k-mer, count) output of
// kmc_count laid out as the paper's .kmc_pre / .kmc_suf files (Suppl. Sec. 4 "Database
// format").  Off the counting hot path; the device does the
// per-k-mer work (signatures, ordering, prefix arrays, packed records), the host writes
// the bytes.
//
//   k_db_ids      signature of every stored k-mer (Sec. 2.2: smallest allowed
//                 canonical p-mer, else the reserved 4^p) -> prefixes-array id = sig >> G
//   (device LSD radix sort of the ids, stable: k-mers stay ascending within an id)
//   k_db_hist     records per (id, lut-symbol prefix) -> exclusive scan = the prefixes
//                 region (first record of every (id, prefix), + the guard)
//   k_db_records  record = suffix (4 symbols per byte, leftmost in the top bits,
//                 P:L1527-1528) + min(count, cs) on counter_size little-endian bytes
//
// The choices the paper leaves open are DESIGN.md reading R-DB: id = signature >> G with
// G = max(0, 2p - 14); lut_prefix_length = the largest of k mod 4, +4, +8 that is <= k
// with ids x 4^lut <= 2^23; counter_size = the fewest bytes holding cs (-cs).
#include "kmc_device.cuh"
#include "kmc_internal.h"

namespace kmc {

namespace {

constexpr int DB_NT = 256;

__device__ __forceinline__ uint32_t db_rev2_32(uint32_t x) {
    x = __brev(x);
    return ((x >> 1) & 0x55555555u) | ((x & 0x55555555u) << 1);
}

// p-mer starting at symbol j of a k-mer key (leftmost symbol most significant)
__device__ __forceinline__ uint32_t db_pmer(uint64_t key, int k, int p, int j) {
    return (uint32_t)(key >> (2 * (k - p - j))) & ((1u << (2 * p)) - 1);
}
__device__ __forceinline__ uint32_t db_pmer(const K128& key, int k, int p, int j) {
    const int sh = 2 * (k - p - j);
    uint64_t v;
    if (sh >= 64) v = key.hi >> (sh - 64);
    else if (sh == 0) v = key.lo;
    else v = (key.lo >> sh) | (key.hi << (64 - sh));
    return (uint32_t)v & ((1u << (2 * p)) - 1);
}

template <class K>
__device__ uint32_t db_signature(const K& key, int k, int p) {
    uint32_t best = 1u << (2 * p);  // reserved: no allowed p-mer
    for (int j = 0; j + p <= k; ++j) {
        const uint32_t f = db_pmer(key, k, p, j);
        const uint32_t r = db_rev2_32(~f) >> (32 - 2 * p);
        const uint32_t c = f < r ? f : r;
        if (c < best && sig_allowed(c, p)) best = c;
    }
    return best;
}

__device__ __forceinline__ uint64_t db_prefix(uint64_t key, int k, int lut) {
    return lut == 0 ? 0 : key >> (2 * (k - lut));
}
__device__ __forceinline__ uint64_t db_prefix(const K128& key, int k, int lut) {
    if (lut == 0) return 0;
    const int sh = 2 * (k - lut);  // >= 2 (k > 32, lut <= 11)
    return sh >= 64 ? key.hi >> (sh - 64) : (key.lo >> sh) | (key.hi << (64 - sh));
}
// the low 2 (k - lut) bits, as a 128-bit pair
__device__ __forceinline__ void db_suffix(uint64_t key, int k, int lut, uint64_t& lo, uint64_t& hi) {
    const int b = 2 * (k - lut);
    lo = b >= 64 ? key : key & ((1ull << b) - 1);
    hi = 0;
}
__device__ __forceinline__ void db_suffix(const K128& key, int k, int lut, uint64_t& lo, uint64_t& hi) {
    const int b = 2 * (k - lut);
    lo = key.lo;
    hi = b >= 128 ? key.hi : (b > 64 ? key.hi & ((1ull << (b - 64)) - 1) : 0);
    if (b < 64) lo &= (1ull << b) - 1;
}

template <class K>
__global__ void k_db_ids(const K* __restrict__ keys, uint64_t n, int k, int p, int G, uint64_t* __restrict__ ids,
                         uint32_t* __restrict__ idx) {
    const uint64_t i = (uint64_t)blockIdx.x * DB_NT + threadIdx.x;
    if (i >= n) return;
    ids[i] = db_signature(keys[i], k, p) >> G;
    idx[i] = (uint32_t)i;
}

template <class K>
__global__ void k_db_hist(const K* __restrict__ keys, const uint64_t* __restrict__ sids,
                          const uint32_t* __restrict__ perm, uint64_t n, int k, int lut,
                          unsigned long long* __restrict__ cnt) {
    const uint64_t i = (uint64_t)blockIdx.x * DB_NT + threadIdx.x;
    if (i >= n) return;
    atomicAdd(&cnt[(sids[i] << (2 * lut)) + db_prefix(keys[perm[i]], k, lut)], 1ull);
}

template <class K>
__global__ void k_db_records(const K* __restrict__ keys, const uint32_t* __restrict__ counts,
                             const uint32_t* __restrict__ perm, uint64_t n, int k, int lut, int cb, uint32_t cs,
                             uint8_t* __restrict__ out) {
    const uint64_t i = (uint64_t)blockIdx.x * DB_NT + threadIdx.x;
    if (i >= n) return;
    const uint32_t src = perm[i];
    const int nb = (k - lut) / 4;
    uint64_t lo, hi;
    db_suffix(keys[src], k, lut, lo, hi);
    uint8_t* o = out + i * (uint64_t)(nb + cb);
    for (int b = 0; b < nb; ++b) {  // big-endian: byte b holds symbols 4b .. 4b+3 of the suffix
        const int sh = 8 * (nb - 1 - b);
        o[b] = (uint8_t)(sh >= 64 ? hi >> (sh - 64) : lo >> sh);
    }
    const uint32_t c = counts[src] < cs ? counts[src] : cs;
    for (int b = 0; b < cb; ++b) o[nb + b] = (uint8_t)(c >> (8 * b));
}

}  // namespace

int db_group_shift(int p) { return 2 * p - 14 > 0 ? 2 * p - 14 : 0; }
uint64_t db_n_arrays(int p) { return ((1ull << (2 * p)) >> db_group_shift(p)) + 1; }
int db_lut_length(int k, int p) {
    int best = k % 4;
    for (int lut = k % 4; lut <= k % 4 + 8; lut += 4)
        if (lut <= k && (db_n_arrays(p) << (2 * lut)) <= (1ull << 23)) best = lut;
    return best;
}
int db_counter_bytes(uint32_t cs) { return cs < (1u << 8) ? 1 : cs < (1u << 16) ? 2 : cs < (1u << 24) ? 3 : 4; }

cudaError_t launch_db_ids(int key_words, const void* keys, uint64_t n, int k, int p, uint64_t* ids, uint32_t* idx,
                          cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned g = (unsigned)((n + DB_NT - 1) / DB_NT);
    if (key_words == 1) k_db_ids<uint64_t><<<g, DB_NT, 0, s>>>((const uint64_t*)keys, n, k, p, db_group_shift(p), ids, idx);
    else k_db_ids<K128><<<g, DB_NT, 0, s>>>((const K128*)keys, n, k, p, db_group_shift(p), ids, idx);
    return cudaGetLastError();
}

cudaError_t launch_db_hist(int key_words, const void* keys, const uint64_t* sids, const uint32_t* perm, uint64_t n,
                           int k, int lut, unsigned long long* cnt, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned g = (unsigned)((n + DB_NT - 1) / DB_NT);
    if (key_words == 1) k_db_hist<uint64_t><<<g, DB_NT, 0, s>>>((const uint64_t*)keys, sids, perm, n, k, lut, cnt);
    else k_db_hist<K128><<<g, DB_NT, 0, s>>>((const K128*)keys, sids, perm, n, k, lut, cnt);
    return cudaGetLastError();
}

cudaError_t launch_db_records(int key_words, const void* keys, const uint32_t* counts, const uint32_t* perm,
                              uint64_t n, int k, int lut, int cb, uint32_t cs, uint8_t* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned g = (unsigned)((n + DB_NT - 1) / DB_NT);
    if (key_words == 1)
        k_db_records<uint64_t><<<g, DB_NT, 0, s>>>((const uint64_t*)keys, counts, perm, n, k, lut, cb, cs, out);
    else k_db_records<K128><<<g, DB_NT, 0, s>>>((const K128*)keys, counts, perm, n, k, lut, cb, cs, out);
    return cudaGetLastError();
}

}  // namespace kmc
