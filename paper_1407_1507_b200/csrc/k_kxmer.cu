// k_kxmer.cu -- S6-S8 of the small bins with (k,x)-mers (Sec. 2.3,
// P:L223-247, and the merge of Sec. 2.4).
//
// One CTA per bin (<= KX_CAP windows).  The paper's sorter, step by step:
//   1. split every super-k-mer record into (k,x)-mers: the record's k-mers, left to right,
//      are cut greedily into runs of at most x+1 consecutive k-mers of one orientation
//      (forward f < r, reverse f > r; a palindrome joins the run in progress and starts a
//      run as forward -- reading R-KX); a run of x'+1 k-mers is the (k+x')-mer it covers,
//      stored as is (forward) or as its reverse complement (reverse), so every k-mer inside a
//      record is canonical;
//   2. radix-sort the (k,x)-mers (key = x' in the top two bits, then the 2(k+x')-bit value,
//      so each length class is one sorted range) and compact equal ones into (value, weight);
//   3. for every class x' and offset j <= x', the records that agree on their first j symbols
//      form a sub-array whose k-mers (symbols j .. j+k-1) are sorted (R_0, R_1, R_A..R_T for
//      x = 1; at most sum_{x'<=x} sum_{j<=x'} 4^j = 112 for x = 3).  The paper
//      scans the sub-arrays "in parallel", taking the smallest k-mer each step;
//      here the same multi-way merge of the sorted sub-arrays runs as ceil(log2 R) rounds of
//      pairwise merges, every element placed by a binary search in its partner sub-array;
//   4. equal neighbouring k-mers are summed (weights) and the cutoffs applied (S8).
// Restrictions: k + x <= 31 (a (k+x)-mer plus its 2-bit class fits 64 bits), canonical counting.
#include <algorithm>

#include "kmc_device.cuh"
#include "kmc_internal.h"

namespace kmc {

namespace {

constexpr int KX_NT = 512, KX_NW = KX_NT / 32;
constexpr int KX_CAP = 4096;  // windows of a bin on this path (64-bit keys)
constexpr int KX_KPT = KX_CAP / KX_NT;
constexpr int KX_RMAX = 128;  // sub-arrays (<= 112)

constexpr size_t KX_OFF_A = 0;                                      // sort keys (KX_CAP u64)
constexpr size_t KX_OFF_DW = KX_OFF_A + KX_CAP * 8;                 // distinct weights (u32)
constexpr size_t KX_OFF_E0K = KX_OFF_DW + KX_CAP * 4;               // merge buffers
constexpr size_t KX_OFF_E0W = KX_OFF_E0K + KX_CAP * 8;
constexpr size_t KX_OFF_E1K = KX_OFF_E0W + KX_CAP * 4;              // records alias here first, then distinct values
constexpr size_t KX_OFF_E1W = KX_OFF_E1K + KX_CAP * 8;
constexpr size_t KX_OFF_RID = KX_OFF_E1W + KX_CAP * 4;              // 2 x KX_CAP u8 sub-array ids
constexpr size_t KX_OFF_BITS = KX_OFF_RID + 2 * KX_CAP;             // run-start bitmask (+ slack)
constexpr size_t KX_OFF_WHIST = KX_OFF_BITS + (KX_CAP / 32 + 8) * 4;
constexpr size_t KX_OFF_BND = KX_OFF_WHIST + (size_t)RADIX * KX_NW * 4;  // 2 x (KX_RMAX + 1) u32
constexpr size_t KX_OFF_MISC = KX_OFF_BND + 2 * (KX_RMAX + 1) * 4 + 8;
constexpr size_t KX_SMEM = KX_OFF_MISC + 256;
static_assert(KX_OFF_MISC % 8 == 0, "alignment");

__device__ __forceinline__ uint64_t kx_mask(int bits) { return bits >= 64 ? ~0ull : ((1ull << bits) - 1); }

__global__ void __launch_bounds__(KX_NT, 1) k_small_kx(SmallArgs a, int x) {
    extern __shared__ __align__(16) uint8_t sm[];
    uint64_t* A = reinterpret_cast<uint64_t*>(sm + KX_OFF_A);
    uint32_t* DW = reinterpret_cast<uint32_t*>(sm + KX_OFF_DW);
    uint64_t* EK[2] = {reinterpret_cast<uint64_t*>(sm + KX_OFF_E0K), reinterpret_cast<uint64_t*>(sm + KX_OFF_E1K)};
    uint32_t* EW[2] = {reinterpret_cast<uint32_t*>(sm + KX_OFF_E0W), reinterpret_cast<uint32_t*>(sm + KX_OFF_E1W)};
    uint8_t* RID[2] = {sm + KX_OFF_RID, sm + KX_OFF_RID + KX_CAP};
    uint32_t* bits = reinterpret_cast<uint32_t*>(sm + KX_OFF_BITS);
    uint32_t* whist = reinterpret_cast<uint32_t*>(sm + KX_OFF_WHIST);
    uint32_t* BND[2] = {reinterpret_cast<uint32_t*>(sm + KX_OFF_BND),
                        reinterpret_cast<uint32_t*>(sm + KX_OFF_BND) + KX_RMAX + 1};
    uint32_t* wsum = reinterpret_cast<uint32_t*>(sm + KX_OFF_MISC);              // 17
    unsigned long long* red = reinterpret_cast<unsigned long long*>(sm + KX_OFF_MISC + 80);  // 4
    uint32_t* cs = reinterpret_cast<uint32_t*>(sm + KX_OFF_MISC + 112);          // class starts [5]
    uint32_t* sc = cs + 8;                                                       // scalars
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t ltm = lanemask_lt();

    const uint32_t bin = a.small_list[blockIdx.x];
    const uint64_t rec0 = a.bin_rec_off[bin];
    const int nrec = (int)a.bin_nrec[bin];
    const int k = a.k;
    // ---- records into the E1 region (16-byte vectors)
    uint32_t* R = reinterpret_cast<uint32_t*>(EK[1]);
    {
        const uint4* src = reinterpret_cast<const uint4*>(a.bins + rec0 * 4);
        uint4* dst = reinterpret_cast<uint4*>(R);
        for (int v = tid; v < nrec; v += KX_NT) dst[v] = src[v];
        if (tid == 0) reinterpret_cast<uint4*>(R)[nrec] = make_uint4(0, 0, 0, 0);  // funnel-read slack
    }
    __syncthreads();
    // ---- 1. (k,x)-mers: orientation runs of <= x+1 k-mers per record (two passes: count, emit)
    auto orient = [&](const uint32_t* rec, int w) {  // 0 forward, 1 reverse, 2 palindrome
        const uint64_t g = bits64_be(rec, 8 + 2 * w);
        const uint64_t f = g >> (64 - 2 * k);
        const uint64_t r = rev2_64(~g) & kx_mask(2 * k);
        return f < r ? 0 : (f > r ? 1 : 2);
    };
    auto for_runs = [&](const uint32_t* rec, auto&& fn) {  // fn(first window, k-mers in run, orientation)
        const int n = (int)rec_nwin(rec);
        int i = 0;
        while (i < n) {
            const int o0 = orient(rec, i);
            const int run = o0 == 2 ? 0 : o0;
            int j = i + 1;
            while (j < n && j - i <= x) {
                const int oj = orient(rec, j);
                if (oj != run && oj != 2) break;
                ++j;
            }
            fn(i, j - i, run);
            i = j;
        }
    };
    const int rpt = (nrec + KX_NT - 1) / KX_NT;
    const int r0 = tid * rpt, r1 = min(nrec, r0 + rpt);
    uint32_t cnt = 0;
    for (int r = r0; r < r1; ++r) for_runs(R + r * 4, [&](int, int, int) { ++cnt; });
    uint32_t n_kx;
    uint32_t pos = block_excl_sum<KX_NT, uint32_t>(cnt, wsum, &n_kx);
    for (int r = r0; r < r1; ++r) {
        const uint32_t* rec = R + r * 4;
        for_runs(rec, [&](int i, int len, int run) {
            const int L = k + len - 1;  // symbols of the (k+x')-mer
            const uint64_t g = bits64_be(rec, 8 + 2 * i);
            const uint64_t v = run == 0 ? (g >> (64 - 2 * L)) : (rev2_64(~g) & kx_mask(2 * L));
            A[pos++] = ((uint64_t)(len - 1) << 62) | v;
        });
    }
    __syncthreads();
    // ---- 2. sort by (class, value), compact equal (k,x)-mers into (value, weight)
    block_sort_inplace<uint64_t, KX_NT, KX_KPT, false>(A, nullptr, (int)n_kx, 64, whist, wsum, red);
    const int nb = ((int)n_kx + 32) / 32;
    for (int base = warp * 32; base < nb * 32; base += KX_NT) {
        const int i = base + lane;
        const bool st = i < (int)n_kx ? (i == 0 || A[i] != A[i - 1]) : (i == (int)n_kx);
        const uint32_t b = __ballot_sync(0xffffffffu, st);
        if (lane == 0) bits[base >> 5] = b;
    }
    __syncthreads();
    uint64_t* D = EK[1];  // the records are no longer needed
    uint32_t nd;
    {
        const int ipt = KX_KPT;
        const int i0 = tid * ipt, i1 = min((int)n_kx, i0 + ipt);
        uint32_t c = 0;
        for (int i = i0; i < i1; ++i) c += (bits[i >> 5] >> (i & 31)) & 1u;
        uint32_t o = block_excl_sum<KX_NT, uint32_t>(c, wsum, &nd);
        for (int i = i0; i < i1; ++i) {
            if ((bits[i >> 5] >> (i & 31)) & 1u) {
                D[o] = A[i];
                DW[o] = rle_run_length(bits, i);
                ++o;
            }
        }
    }
    if (tid < 5) cs[tid] = nd;
    __syncthreads();
    for (uint32_t i = tid; i < nd; i += KX_NT) {  // class starts (classes are contiguous)
        const uint32_t c = (uint32_t)(D[i] >> 62);
        if (i == 0 || (uint32_t)(D[i - 1] >> 62) != c)
            for (uint32_t q = (i == 0 ? 0u : (uint32_t)(D[i - 1] >> 62) + 1); q <= c; ++q) cs[q] = i;
    }
    __syncthreads();
    // ---- 3. the sub-arrays: (class x', offset j) blocks, each split where the first j symbols change
    // E position of block (x', j): blocks in order of x', then j; class x' has cs[x'+1] - cs[x']
    // elements, each in x'+1 blocks
    auto blk_base = [&](int xp, int j) {
        uint32_t b = 0;
        for (int q = 0; q < xp; ++q) b += (uint32_t)(q + 1) * (cs[q + 1] - cs[q]);
        return b + (uint32_t)j * (cs[xp + 1] - cs[xp]);
    };
    const uint32_t M = blk_base(3, 4);  // past the last block (k-mer occurrences in the sub-arrays)
    for (uint32_t i = tid; i < nd; i += KX_NT) {
        const uint64_t d = D[i];
        const int xp = (int)(d >> 62);
        const int L = k + xp;
        const uint64_t v = d & kx_mask(62);
        const uint32_t r = i - cs[xp];
        const uint64_t pv = r ? (D[i - 1] & kx_mask(62)) : 0ull;
        for (int j = 0; j <= xp; ++j) {
            const uint32_t q = blk_base(xp, j) + r;
            EK[0][q] = (v >> (2 * (xp - j))) & kx_mask(2 * k);
            EW[0][q] = DW[i];
            // a sub-array starts at the block start or where the first j symbols change
            const bool st = r == 0 || (j > 0 && (v >> (2 * (L - j))) != (pv >> (2 * (L - j))));
            RID[1][q] = st ? 1 : 0;  // start flags for now
        }
    }
    __syncthreads();
    // sub-array ids: running count of start flags (block scan over contiguous element ranges)
    uint32_t nrun;
    {
        const int ipt = (int)((M + KX_NT - 1) / KX_NT);
        const int i0 = tid * ipt, i1 = min((int)M, i0 + ipt);
        uint32_t c = 0;
        for (int i = i0; i < i1; ++i) c += RID[1][i];
        uint32_t o = block_excl_sum<KX_NT, uint32_t>(c, wsum, &nrun);
        for (int i = i0; i < i1; ++i) {
            if (RID[1][i]) {
                BND[0][o] = (uint32_t)i;
                ++o;
            }
            RID[0][i] = (uint8_t)(o - 1);
        }
        if (tid == 0) BND[0][nrun] = M;
    }
    __syncthreads();
    // ---- multi-way merge of the sorted sub-arrays: rounds of pairwise merges
    int cur = 0;
    uint32_t R_ = nrun;
    while (R_ > 1) {
        const uint64_t* sk = EK[cur];
        const uint32_t* sw = EW[cur];
        const uint8_t* sr = RID[cur];
        const uint32_t* bnd = BND[cur];
        uint64_t* dk = EK[cur ^ 1];
        uint32_t* dw = EW[cur ^ 1];
        uint8_t* dr = RID[cur ^ 1];
        for (uint32_t q = tid; q < M; q += KX_NT) {
            const uint32_t r = sr[q];
            const uint64_t key = sk[q];
            uint32_t out = q;
            if ((r ^ 1u) < R_) {
                const uint32_t p = r ^ 1u;
                uint32_t lo = bnd[p], hi = bnd[p + 1];
                const bool left = (r & 1u) == 0;
                while (lo < hi) {  // left: partner keys < key; right: partner keys <= key
                    const uint32_t mid = (lo + hi) >> 1;
                    const uint64_t km = sk[mid];
                    if (left ? (km < key) : (km <= key)) lo = mid + 1;
                    else hi = mid;
                }
                out = bnd[r & ~1u] + (q - bnd[r]) + (lo - bnd[p]);
            }
            dk[out] = key;
            dw[out] = sw[q];
            dr[out] = (uint8_t)(r >> 1);
        }
        const uint32_t Rn = (R_ + 1) >> 1;
        for (uint32_t t = tid; t <= Rn; t += KX_NT) BND[cur ^ 1][t] = t < Rn ? bnd[2 * t] : M;
        __syncthreads();
        cur ^= 1;
        R_ = Rn;
    }
    // ---- 4. equal k-mers summed, cutoffs, survivors
    const uint64_t* fk = EK[cur];
    const uint32_t* fw = EW[cur];
    const int nbm = ((int)M + 32) / 32;
    for (int base = warp * 32; base < nbm * 32; base += KX_NT) {
        const int i = base + lane;
        const bool st = i < (int)M ? (i == 0 || fk[i] != fk[i - 1]) : (i == (int)M);
        const uint32_t b = __ballot_sync(0xffffffffu, st);
        if (lane == 0) bits[base >> 5] = b;
    }
    __syncthreads();
    uint32_t uniq = 0, below = 0, above = 0, keep = 0;
    for (int i = tid; i < (int)M; i += KX_NT) {
        if (!((bits[i >> 5] >> (i & 31)) & 1u)) continue;
        const uint32_t len = rle_run_length(bits, i);
        uint32_t c = 0;
        for (uint32_t e = 0; e < len; ++e) c += fw[i + e];
        ++uniq;
        if (c < a.ci) ++below;
        else if (c > a.cx) ++above;
        else ++keep;
    }
    const uint32_t kin = warp_incl_sum(keep);
    const uint32_t ktot = __shfl_sync(0xffffffffu, kin, 31);
    const uint32_t tu = __reduce_add_sync(0xffffffffu, uniq);
    const uint32_t tb = __reduce_add_sync(0xffffffffu, below);
    const uint32_t ta = __reduce_add_sync(0xffffffffu, above);
    unsigned long long base = 0;
    if (lane == 0) {
        if (ktot) base = atomicAdd(&a.gstats[GS_SURV], (unsigned long long)ktot);
        if (tu) atomicAdd(&a.gstats[GS_UNIQUE], (unsigned long long)tu);
        if (tb) atomicAdd(&a.gstats[GS_BELOW], (unsigned long long)tb);
        if (ta) atomicAdd(&a.gstats[GS_ABOVE], (unsigned long long)ta);
    }
    if (tid == 0) {
        atomicAdd(&a.gstats[GS_KX], (unsigned long long)n_kx);
        atomicAdd(&a.gstats[GS_KX_WIN], (unsigned long long)a.bin_w[bin]);
    }
    uint64_t o = __shfl_sync(0xffffffffu, base, 0) + kin - keep;
    uint64_t* out_keys = reinterpret_cast<uint64_t*>(a.surv_keys);
    for (int i = tid; i < (int)M; i += KX_NT) {
        if (!((bits[i >> 5] >> (i & 31)) & 1u)) continue;
        const uint32_t len = rle_run_length(bits, i);
        uint32_t c = 0;
        for (uint32_t e = 0; e < len; ++e) c += fw[i + e];
        if (c >= a.ci && c <= a.cx) {
            out_keys[o] = fk[i];
            a.surv_counts[o] = c;
            ++o;
        }
    }
}

}  // namespace

int kx_capacity() { return KX_CAP; }

cudaError_t launch_small_kx(const SmallArgs& a, uint64_t n_small, int x, cudaStream_t s) {
    if (n_small == 0) return cudaSuccess;
    if (a.k + x > 31 || x < 1 || x > 3 || !a.canonical) return cudaErrorInvalidValue;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_small_kx, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)KX_SMEM))) return e;
    k_small_kx<<<(unsigned)n_small, KX_NT, KX_SMEM, s>>>(a, x);
    return cudaGetLastError();
}

}  // namespace kmc
