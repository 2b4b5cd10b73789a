// k_cluster.cu -- S6-S8 of the large bins (k <= 32) with no key spill to HBM.
//
// The paper's sorter loads one bin, extracts its k-mers, sorts and merges them
// (P:L307-310).  A signature is indivisible, and at C4 most windows sit in
// bins of 10^5-10^6 windows -- far more keys than one SM's shared memory holds.  Here a
// thread-block CLUSTER counts one large bin at a time in the union of its CTAs'
// shared-memory hash tables:
//   * every CTA streams a contiguous slice of the bin's compact records from HBM (TMA 1-D
//     bulk copies, double-buffered pieces of <= 512 records) and expands them into canonical
//     keys min(fwd, rc) (one lane per unit of <= 4 consecutive windows of a
//     record, the unit's symbols one 64-bit field);
//   * a key belongs to the CTA named by a hash of the key.  The keys of a sub-batch (1024
//     units) are staged in owner order in the producer's shared memory (warp match + one
//     block scan of the per-warp owner counts); after a cluster barrier every CTA pulls its
//     segment from each peer through distributed shared memory (ld.shared::cluster) and
//     counts the keys in its own table (one shared CAS per probe claims an empty slot or
//     finds the key, then atomicAdd on the count).  Staging is double-buffered, so one
//     cluster barrier per sub-batch orders both the staging writes and the peers' reads;
//   * a bin whose estimated distinct keys exceed the cluster's tables is counted in R
//     rounds, round r keeping the keys of one hash range (every round re-reads the bin);
//   * bins that fit one table are counted by single CTAs (no exchange) once the cluster
//     items are drained;
//   * after an item, every CTA scans its table: keys with ci <= count <= cx are survivors
//     (S8; S9 orders them globally), then it clears the slots.
// A key whose probe sequence (CL_PROBE slots) finds neither itself nor an empty slot is
// appended to a spill list instead.  Slots are never freed during an item, so every copy of
// such a key fails the same way: the table's counts stay exact and the spilled keys --
// disjoint from the table's -- are counted afterwards by the device radix sort + run pass.
#include <algorithm>

#include <cooperative_groups.h>

#include "kmc_device.cuh"
#include "kmc_internal.h"

namespace cg = cooperative_groups;

namespace kmc {

namespace {

constexpr int CL_NT = 1024, CL_NW = CL_NT / 32;
constexpr int CL_TS = 10240;            // hash slots per CTA (8-byte key + 4-byte count)
constexpr int CL_SB = CL_NT * 4;        // keys per sub-batch at most (1024 units x <= 4 windows)
constexpr int CL_REC = 512;             // records per TMA piece, at most
constexpr int CL_UMAX = 4608;           // units per piece (unit -> record map entries per slot)
constexpr int CL_RBW = CL_REC * 4 + 8;  // words per record buffer (+ slack for 3-word funnel reads)
constexpr int CL_CMAX = 16;             // largest cluster
constexpr int CL_PROBE = 64;
constexpr uint64_t CL_EMPTY = ~0ull;    // never a key: k <= 31 for -b, and the all-T canonical k-mer is not canonical

// scalar slots (uint32) at the end of shared memory
enum { SC_ITEM = 0, SC_MORE = 1 /* 2 entries, by staging buffer */, SC_ITEM1 = 3, SC_N = 16 };

// shared-memory layout (bytes)
constexpr size_t OFF_T = 0;
constexpr size_t OFF_CNT = OFF_T + (size_t)CL_TS * 8;
constexpr size_t OFF_STAGE = OFF_CNT + (size_t)CL_TS * 4;
constexpr size_t OFF_RB = OFF_STAGE + 2 * (size_t)CL_SB * 8;
constexpr size_t OFF_UMAP = OFF_RB + 2 * (size_t)CL_RBW * 4;
constexpr size_t OFF_RINFO = OFF_UMAP + 2 * (size_t)CL_UMAX * 2;
constexpr size_t OFF_WCNT = OFF_RINFO + 2 * (size_t)CL_REC * 4;
constexpr size_t OFF_OSTART = OFF_WCNT + (size_t)CL_NW * CL_CMAX * 4;
constexpr size_t OFF_PSEG = OFF_OSTART + 2 * 20 * 4;
constexpr size_t OFF_WSUM = OFF_PSEG + 3 * CL_CMAX * 4;
constexpr size_t OFF_MBAR = OFF_WSUM + 40 * 4;
constexpr size_t OFF_SC = OFF_MBAR + 2 * 8;
constexpr size_t CL_SMEM = OFF_SC + SC_N * 4;
static_assert(OFF_STAGE % 16 == 0 && OFF_RB % 16 == 0 && OFF_MBAR % 8 == 0, "alignment");
static_assert(CL_SMEM <= 232448, "fits one SM's shared memory");
static_assert(CL_TS % CL_NT == 0, "whole warps scan the table");

// owner / round hash and slot hash (independent multipliers)
__device__ __forceinline__ uint32_t cl_hash(uint64_t key) {
    return (((uint32_t)(key >> 32) * 0x85EBCA6Bu) ^ (uint32_t)key) * 0x9E3779B1u;
}
__device__ __forceinline__ uint32_t cl_slot(uint64_t key) {
    uint32_t h = (((uint32_t)(key >> 32) * 0x2C1B3C6Du) ^ (uint32_t)key) * 0x297A2D39u;
    h = (h ^ (h >> 16)) * 0x7FEB352Du;
    return (uint32_t)(((uint64_t)h * CL_TS) >> 32);
}

struct ClArgs {
    const uint32_t* bins;
    const ClItem* citems;
    uint32_t n_citems;
    const ClItem* sitems;
    uint32_t n_sitems;
    unsigned long long* ctr;  // [0] cluster items taken, [1] single items taken, [2] spilled keys
    uint64_t* spill;
    uint64_t spill_cap;
    int k;
    int unit;  // windows per expansion unit
    int rpp;   // records per piece
    uint32_t ci, cx;
    uint64_t* surv_keys;
    uint32_t* surv_counts;
    unsigned long long* gstats;
};

template <int C, bool CANON>
__global__ void __launch_bounds__(CL_NT, 1) k_clcount(ClArgs a) {
    constexpr int LOGC = C == 16 ? 4 : C == 8 ? 3 : C == 4 ? 2 : C == 2 ? 1 : 0;
    static_assert((1 << LOGC) == C && C <= CL_CMAX, "power-of-two cluster");
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* T = reinterpret_cast<uint64_t*>(sm + OFF_T);
    uint32_t* Cn = reinterpret_cast<uint32_t*>(sm + OFF_CNT);
    uint64_t* stage = reinterpret_cast<uint64_t*>(sm + OFF_STAGE);
    uint32_t* RB = reinterpret_cast<uint32_t*>(sm + OFF_RB);
    uint16_t* umap = reinterpret_cast<uint16_t*>(sm + OFF_UMAP);
    uint32_t* rinfo = reinterpret_cast<uint32_t*>(sm + OFF_RINFO);
    uint32_t* wcnt = reinterpret_cast<uint32_t*>(sm + OFF_WCNT);
    uint32_t* ostart = reinterpret_cast<uint32_t*>(sm + OFF_OSTART);
    uint32_t* pseg = reinterpret_cast<uint32_t*>(sm + OFF_PSEG);
    uint32_t* wsum = reinterpret_cast<uint32_t*>(sm + OFF_WSUM);
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + OFF_MBAR);
    uint32_t* sc = reinterpret_cast<uint32_t*>(sm + OFF_SC);

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t ltm = lanemask_lt();
    const int k = a.k, U = a.unit;
    const uint32_t RPP = (uint32_t)a.rpp;

    for (int i = tid; i < CL_TS; i += CL_NT) {
        T[i] = CL_EMPTY;
        Cn[i] = 0;
    }
    if (tid == 0) {
        mbar_init(mbar, 1);
        mbar_init(mbar + 1, 1);
        mbar_init_fence();
    }
    __syncthreads();

    // ---------------------------------------------------------- record stream (per CTA)
    // records [r0, r0 + nrec) in pieces of RPP records; piece p lives in slot p & 1.
    uint64_t r0 = 0;
    uint32_t nrec = 0, npieces = 0, issued = 0, built = 0, cur = 0, cur_u = 0;
    // per slot (kept as scalars: a dynamically indexed pair would live in local memory)
    uint32_t units0 = 0, units1 = 0;  // units of the piece in the slot
    uint32_t uses0 = 0, uses1 = 0;    // TMA completions requested (mbarrier phase)
    auto units_of = [&](uint32_t slot) { return slot ? units1 : units0; };
    auto piece_nrec = [&](uint32_t p) { return min(RPP, nrec - p * RPP); };
    auto issue = [&](uint32_t p) {  // all threads call (uniform bookkeeping); thread 0 issues
        const int slot = p & 1;
        if (tid == 0) {
            const uint32_t n = piece_nrec(p);
            fence_proxy_async_smem();
            mbar_expect_tx(mbar + slot, n * 16);
            tma_load_1d(RB + slot * CL_RBW, a.bins + (r0 + (uint64_t)p * RPP) * 4, n * 16, mbar + slot);
        }
        if (slot) ++uses1;
        else ++uses0;
    };
    auto build = [&](uint32_t p) {  // unit -> record map of piece p (all threads)
        const int slot = p & 1;
        const uint32_t n = piece_nrec(p);
        mbar_wait(mbar + slot, ((slot ? uses1 : uses0) - 1) & 1);
        uint32_t nw = 0, nu = 0;
        if ((uint32_t)tid < n) {
            nw = rec_nwin(RB + slot * CL_RBW + tid * 4);
            nu = U == 4 ? (nw + 3) >> 2 : U == 2 ? (nw + 1) >> 1 : U == 1 ? nw : (nw + 2) / 3;
        }
        uint32_t tot;
        const uint32_t pre = block_excl_sum<CL_NT, uint32_t>(nu, wsum, &tot);
        for (uint32_t j = 0; j < nu; ++j) umap[slot * CL_UMAX + pre + j] = (uint16_t)tid;
        if ((uint32_t)tid < n) rinfo[slot * CL_REC + tid] = pre | (nw << 16);
        if (slot) units1 = tot;
        else units0 = tot;
        __syncthreads();
    };
    auto stream_begin = [&](uint64_t rec0, uint32_t n) {
        r0 = rec0;
        nrec = n;
        npieces = (n + RPP - 1) / RPP;
        issued = built = cur = cur_u = 0;
        while (issued < npieces && issued < 2) issue(issued++);
    };
    // Expands the next sub-batch (<= 1024 units from the current piece and the next one) into
    // keys[0..cnt) of this thread; returns whether the stream holds more units afterwards.
    // Ends with the cursor advanced; the caller issues the freed slots' copies (issue_free)
    // after a barrier that follows every thread's expansion.
    auto expand = [&](uint64_t (&key)[4], int& cnt) -> bool {
        cnt = 0;
        if (cur >= npieces) return false;
        if (built == cur) {
            build(cur);
            ++built;
        }
        const uint32_t avail = units_of(cur & 1) - cur_u;
        if (avail < (uint32_t)CL_NT && cur + 1 < npieces && built == cur + 1) {
            build(cur + 1);
            ++built;
        }
        const uint32_t n0 = min(avail, (uint32_t)CL_NT);
        const uint32_t n1 = built > cur + 1 ? min(units_of((cur + 1) & 1), (uint32_t)CL_NT - n0) : 0u;
        int slot = -1;
        uint32_t u = 0;
        if ((uint32_t)tid < n0) {
            slot = cur & 1;
            u = cur_u + tid;
        } else if ((uint32_t)tid < n0 + n1) {
            slot = (cur + 1) & 1;
            u = tid - n0;
        }
        if (slot >= 0) {
            const uint32_t* Rp = RB + slot * CL_RBW;
            const uint32_t l = umap[slot * CL_UMAX + u];
            const uint32_t ri = rinfo[slot * CL_REC + l];
            const int first = U * (int)(u - (ri & 0xFFFFu));
            cnt = min(U, (int)(ri >> 16) - first);
            const uint64_t g = bits64_be(Rp + l * 4, 8 + 2 * first);
            const uint64_t rg = rev2_64(~g);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                const uint64_t f = (g << (2 * t)) >> (64 - 2 * k);
                const uint64_t rc = (rg << (64 - 2 * t - 2 * k)) >> (64 - 2 * k);
                key[t] = (CANON && rc < f) ? rc : f;
            }
        }
        // advance the cursor (uniform)
        if (n0 == avail) {
            ++cur;
            cur_u = n1;
            if (cur < npieces && built > cur && cur_u == units_of(cur & 1)) {
                ++cur;
                cur_u = 0;
            }
        } else {
            cur_u += n0;
        }
        return cur < npieces;
    };
    auto issue_free = [&]() {  // pieces whose slot the cursor has released
        while (issued < npieces && issued < cur + 2) issue(issued++);
    };

    auto insert = [&](uint64_t key) {
        uint32_t s = cl_slot(key);
#pragma unroll 1
        for (int pr = 0; pr < CL_PROBE; ++pr) {
            const uint64_t old = atomicCAS(reinterpret_cast<unsigned long long*>(T + s), CL_EMPTY, key);
            if (old == CL_EMPTY || old == key) {
                atomicAdd(Cn + s, 1u);
                return;
            }
            s = (s + 1 == (uint32_t)CL_TS) ? 0u : s + 1;
        }
        const unsigned long long q = atomicAdd(a.ctr + 2, 1ull);  // overfull table: spill
        if (q < a.spill_cap) a.spill[q] = key;
    };

    uint32_t uniq = 0, below = 0, above = 0;
    // scan the table: survivors (S8) with per-warp output reservations, then clear
    auto emit = [&]() {
        uint32_t keep = 0;
        for (int s = tid; s < CL_TS; s += CL_NT) {
            const uint32_t c = Cn[s];
            if (c) {
                ++uniq;
                if (c < a.ci) ++below;
                else if (c > a.cx) ++above;
                else ++keep;
            }
        }
        keep = __reduce_add_sync(0xffffffffu, keep);
        unsigned long long o = 0;
        if (lane == 0 && keep) o = atomicAdd(&a.gstats[GS_SURV], (unsigned long long)keep);
        o = __shfl_sync(0xffffffffu, o, 0);
        for (int s = tid; s < CL_TS; s += CL_NT) {
            const uint32_t c = Cn[s];
            const bool kp = c >= a.ci && c <= a.cx && c != 0;
            const uint32_t bb = __ballot_sync(0xffffffffu, kp);
            if (kp) {
                const unsigned long long q = o + __popc(bb & ltm);
                a.surv_keys[q] = T[s];
                a.surv_counts[q] = c;
            }
            o += __popc(bb);
            T[s] = CL_EMPTY;
            Cn[s] = 0;
        }
        __syncthreads();
    };

    // ---------------------------------------------------------- cluster items
    if constexpr (C > 1) {
        cg::cluster_group cl = cg::this_cluster();
        const uint32_t rank = cl.block_rank();
        cl.sync();  // every CTA of the cluster runs before any distributed shared memory access
        for (;;) {
            if (rank == 0 && tid == 0) {
                const uint32_t it = (uint32_t)atomicAdd(a.ctr, 1ull);
#pragma unroll 1
                for (int q = 0; q < C; ++q) *cl.map_shared_rank(sc + SC_ITEM, q) = it;
            }
            cl.sync();
            const uint32_t it = sc[SC_ITEM];
            if (it >= a.n_citems) break;
            const ClItem item = a.citems[it];
            const uint32_t R = item.nround, rnd = item.round;
            // this CTA's slice of the bin's records
            const uint64_t s0 = (uint64_t)item.nrec * rank / C, s1 = (uint64_t)item.nrec * (rank + 1) / C;
            stream_begin(item.rec_off + s0, (uint32_t)(s1 - s0));
            for (uint32_t sb = 0;; ++sb) {
                const int buf = sb & 1;
                uint64_t key[4];
                int cnt;
                const bool more = expand(key, cnt);
                // owner of each key (keys of other rounds dropped); warp-local ranks per owner
                uint32_t own[4], lpos[4];
                if (lane < CL_CMAX) wcnt[warp * CL_CMAX + lane] = 0;
                __syncwarp();
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    own[t] = 0xFFu;
                    if (t < cnt) {
                        const uint32_t h = cl_hash(key[t]);
                        const bool in_round =
                            R <= 1 || (uint32_t)(((uint64_t)(uint32_t)(h << LOGC) * R) >> 32) == rnd;
                        if (in_round) own[t] = h >> (32 - LOGC);
                    }
                    const uint32_t o = own[t] < (uint32_t)C ? own[t] : (uint32_t)(C + lane);
                    const uint32_t peers = __match_any_sync(0xffffffffu, o);
                    const int leader = __ffs(peers) - 1;
                    uint32_t base = 0;
                    if (lane == leader && own[t] < (uint32_t)C) {
                        base = wcnt[warp * CL_CMAX + o];
                        wcnt[warp * CL_CMAX + o] = base + __popc(peers);
                    }
                    base = __shfl_sync(0xffffffffu, base, leader);
                    lpos[t] = base + __popc(peers & ltm);
                    __syncwarp();
                }
                __syncthreads();
                // per owner: exclusive offsets over the warps, owner segments in owner order
                if (warp == 0) {
                    uint32_t tot = 0;
                    if (lane < C)
                        for (int w = 0; w < CL_NW; ++w) tot += wcnt[w * CL_CMAX + lane];
                    const uint32_t inc = warp_incl_sum(lane < C ? tot : 0u);
                    if (lane < C) {
                        uint32_t run = inc - tot;
                        ostart[buf * 20 + lane] = run;
                        for (int w = 0; w < CL_NW; ++w) {
                            const uint32_t c = wcnt[w * CL_CMAX + lane];
                            wcnt[w * CL_CMAX + lane] = run;
                            run += c;
                        }
                    }
                    if (lane == C - 1) ostart[buf * 20 + C] = inc;
                    if (lane == 0) sc[SC_MORE + buf] = more ? 1u : 0u;
                }
                __syncthreads();
                issue_free();  // every thread is past its expansion reads of released pieces
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (own[t] < (uint32_t)C) stage[buf * CL_SB + wcnt[warp * CL_CMAX + own[t]] + lpos[t]] = key[t];
                cl.sync();  // staging written (release) -> peers may read it (acquire)
                if (tid < C) {
                    const uint32_t* ro = cl.map_shared_rank(ostart + buf * 20, tid);
                    const uint32_t st = ro[rank];
                    pseg[tid] = st;
                    pseg[CL_CMAX + tid] = ro[rank + 1] - st;
                    pseg[2 * CL_CMAX + tid] = *cl.map_shared_rank(sc + SC_MORE + buf, tid);
                }
                __syncthreads();
                uint32_t total = 0, any = 0;
#pragma unroll
                for (int q = 0; q < C; ++q) {
                    total += pseg[CL_CMAX + q];
                    any |= pseg[2 * CL_CMAX + q];
                }
                // pull this CTA's keys from every peer's staging buffer and count them
                for (uint32_t i0 = 0; i0 < total; i0 += 2 * CL_NT) {
                    uint64_t kk[2];
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const uint32_t i = i0 + tid + j * CL_NT;
                        kk[j] = CL_EMPTY;
                        if (i < total) {
                            uint32_t q = 0, pre = 0;
                            while (i >= pre + pseg[CL_CMAX + q]) pre += pseg[CL_CMAX + q++];
                            kk[j] = cl.map_shared_rank(stage + buf * CL_SB, q)[pseg[q] + (i - pre)];
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 2; ++j)
                        if (kk[j] != CL_EMPTY) insert(kk[j]);
                }
                if (!any) break;
            }
            __syncthreads();
            emit();
        }
    }

    // ---------------------------------------------------------- single-CTA items
    for (;;) {
        if (tid == 0) sc[SC_ITEM1] = (uint32_t)atomicAdd(a.ctr + 1, 1ull);
        __syncthreads();
        const uint32_t it = sc[SC_ITEM1];
        if (it >= a.n_sitems) break;
        const ClItem item = a.sitems[it];
        stream_begin(item.rec_off, item.nrec);
        for (;;) {
            uint64_t key[4];
            int cnt;
            const bool more = expand(key, cnt);
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (t < cnt) insert(key[t]);
            __syncthreads();
            issue_free();
            if (!more) break;
        }
        emit();
    }

    uniq = __reduce_add_sync(0xffffffffu, uniq);
    below = __reduce_add_sync(0xffffffffu, below);
    above = __reduce_add_sync(0xffffffffu, above);
    if (lane == 0) {
        if (uniq) atomicAdd(&a.gstats[GS_UNIQUE], (unsigned long long)uniq);
        if (below) atomicAdd(&a.gstats[GS_BELOW], (unsigned long long)below);
        if (above) atomicAdd(&a.gstats[GS_ABOVE], (unsigned long long)above);
    }
    if constexpr (C > 1) cg::this_cluster().sync();
}

// Fallback expansion (S6) of the spilled keys' complement is not needed: spilled keys are
// counted from the spill list itself (device radix sort + run pass).

template <int C, bool CANON>
cudaError_t launch_cl_t(const ClArgs& a, int max_clusters, cudaStream_t s, int* n_ctas) {
    cudaError_t e;
    auto kern = k_clcount<C, CANON>;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CL_SMEM))) return e;
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    cfg.blockDim = dim3(CL_NT, 1, 1);
    cfg.dynamicSmemBytes = CL_SMEM;
    cfg.stream = s;
    int n_cl = 0;
    if (C > 1) {
        if (C > 8 && (e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1))) return e;
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = C;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        cfg.gridDim = dim3(C, 1, 1);
        if ((e = cudaOccupancyMaxActiveClusters(&n_cl, kern, &cfg))) return e;
        if (n_cl < 1) return cudaErrorInvalidConfiguration;
        if (max_clusters > 0) n_cl = std::min(n_cl, max_clusters);
        cfg.gridDim = dim3(n_cl * C, 1, 1);
    } else {
        int dev = 0, nsm = 148;
        if ((e = cudaGetDevice(&dev))) return e;
        if ((e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev))) return e;
        n_cl = max_clusters > 0 ? std::min(max_clusters, nsm) : nsm;
        cfg.gridDim = dim3(n_cl, 1, 1);
    }
    *n_ctas = (int)cfg.gridDim.x;
    if ((e = cudaLaunchKernelEx(&cfg, kern, a))) return e;
    return cudaGetLastError();
}

}  // namespace

int cl_table_slots() { return CL_TS; }

int cl_records_per_piece(int k) {
    const int U = k + 3 <= 32 ? 4 : 33 - k;
    const int upr = (record_max_windows(k) + U - 1) / U;
    return std::min(CL_REC, CL_UMAX / upr);
}

cudaError_t launch_cluster_count(const uint32_t* bins, const ClItem* citems, uint64_t n_citems, const ClItem* sitems,
                                 uint64_t n_sitems, int cluster, int k, int canonical, uint32_t ci, uint32_t cx,
                                 unsigned long long* ctr, uint64_t* spill, uint64_t spill_cap, void* surv_keys,
                                 uint32_t* surv_counts, unsigned long long* gstats, int max_ctas, cudaStream_t s,
                                 int* n_ctas) {
    *n_ctas = 0;
    if (n_citems + n_sitems == 0) return cudaSuccess;
    if (k > 32 || n_citems >= (1ull << 32) || n_sitems >= (1ull << 32)) return cudaErrorInvalidValue;
    ClArgs a{};
    a.bins = bins;
    a.citems = citems;
    a.n_citems = (uint32_t)n_citems;
    a.sitems = sitems;
    a.n_sitems = (uint32_t)n_sitems;
    a.ctr = ctr;
    a.spill = spill;
    a.spill_cap = spill_cap;
    a.k = k;
    a.unit = k + 3 <= 32 ? 4 : 33 - k;
    a.rpp = cl_records_per_piece(k);
    a.ci = ci;
    a.cx = cx;
    a.surv_keys = reinterpret_cast<uint64_t*>(surv_keys);
    a.surv_counts = surv_counts;
    a.gstats = gstats;
    const int mc = max_ctas > 0 ? std::max(1, max_ctas / std::max(1, cluster)) : 0;
    if (n_citems == 0) cluster = 1;
    if (canonical) {
        switch (cluster) {
            case 16: return launch_cl_t<16, true>(a, mc, s, n_ctas);
            case 8: return launch_cl_t<8, true>(a, mc, s, n_ctas);
            case 4: return launch_cl_t<4, true>(a, mc, s, n_ctas);
            case 1: return launch_cl_t<1, true>(a, max_ctas, s, n_ctas);
        }
    } else {
        switch (cluster) {
            case 16: return launch_cl_t<16, false>(a, mc, s, n_ctas);
            case 8: return launch_cl_t<8, false>(a, mc, s, n_ctas);
            case 4: return launch_cl_t<4, false>(a, mc, s, n_ctas);
            case 1: return launch_cl_t<1, false>(a, max_ctas, s, n_ctas);
        }
    }
    return cudaErrorInvalidValue;
}

int cluster_max_active(int cluster) {
    // clusters of this size the device can hold at once (1 CTA per SM), 0 if unsupported
    cudaLaunchConfig_t cfg{};
    cudaLaunchAttribute attr[1];
    cfg.blockDim = dim3(CL_NT, 1, 1);
    cfg.dynamicSmemBytes = CL_SMEM;
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = cluster;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(cluster, 1, 1);
    int n = 0;
    cudaError_t e = cudaSuccess;
    auto q = [&](auto kern) {
        if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CL_SMEM))) return;
        if (cluster > 8 && (e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1))) return;
        e = cudaOccupancyMaxActiveClusters(&n, kern, &cfg);
    };
    switch (cluster) {
        case 16: q(k_clcount<16, true>); break;
        case 8: q(k_clcount<8, true>); break;
        case 4: q(k_clcount<4, true>); break;
        default: return 0;
    }
    if (e != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

}  // namespace kmc
