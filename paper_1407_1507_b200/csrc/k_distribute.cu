// k_distribute.cu -- phase 1 of KMC 2 on the B200 (Sec. 2.4 "distribution"):
// S1 encode + split at non-ACGT and read ends, S2 signatures, S3 super-k-mer cut,
// S4 histogram (pass 1) and S5 scatter of super-k-mer records into HBM bins (pass 2).
//
// One CTA owns a tile of P1_TILE consecutive window starts of the concatenated base
// stream (windows never cross read boundaries: reads are marked from read_offsets).
// Everything between the ASCII load and the histogram / bin write stays in shared
// memory: codes, valid-run lengths, the canonical p-mer key of every position, the
// van Herk / Gil-Werman block prefix/suffix minima, and the per-window signature.
#include <algorithm>

#include "kmc_device.cuh"
#include "kmc_internal.h"

namespace kmc {

namespace {

constexpr int LEFT = 16;                      // halo before the tile (window q0-1 + alignment)
constexpr int NB = P1_TILE + 96;             // loaded bases: LEFT + tile + k-1 (k <= 64); multiple of 32
constexpr int CH = (NB + P1_NT - 1) / P1_NT;  // positions per thread in the scans
constexpr int WPT = P1_TILE / P1_NT;          // windows owned per thread
constexpr uint32_t INV = 0xFFFFFFFFu;
static_assert(NB % 32 == 0 && NB >= LEFT + P1_TILE + 63, "NB");

// A->0, C->1, G->2, T->3; lowercase folded; anything else -> 4 (invalid, R3).
__device__ __forceinline__ uint32_t encode_base(uint32_t ch) {
    uint32_t c = ch & 0xDFu;
    bool ok = (c == 'A') | (c == 'C') | (c == 'G') | (c == 'T');
    return ok ? (((c >> 1) ^ (c >> 2)) & 3u) : 4u;
}

__global__ void k_tile_reads(const uint64_t* __restrict__ offsets, uint64_t n_reads, uint64_t off0,
                             uint64_t n_tiles, uint64_t* __restrict__ tile_r_lo) {
    uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tiles) return;
    // first r in [0, n_reads] with offsets[r] - off0 > left edge of tile t
    int64_t edge = (int64_t)(t * P1_TILE) - LEFT;
    uint64_t lo = 0, hi = n_reads + 1;
    while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if ((int64_t)(offsets[mid] - off0) > edge) hi = mid;
        else lo = mid + 1;
    }
    tile_r_lo[t] = lo;
}

constexpr int NWD = NB / 32 + 8;  // bitmask words (with slack for funnel reads)

struct P1Smem {
    uint32_t pre[NB];            // p-mer keys, then (in place) block prefix minima; later the run-start list
    uint32_t suf[NB];            // block suffix minima, then (in place) per-window signatures
    uint32_t pk[NB / 16 + 8];    // 2-bit packed codes, 16 per word, MSB first
    uint32_t inv[NWD];           // bit x: base x is not A/C/G/T (or outside the stream)
    uint32_t rs[NWD];            // bit x: a read starts at x
    uint32_t ext[NWD];           // bit x: x can extend a run to its left (valid, no read start)
    uint32_t vwin[NWD];          // bit i: window i is valid
    uint32_t vpm[NWD];           // bit j: p-mer j is valid
    uint32_t ebits[P1_TILE / 32 + 8];
    uint32_t wsum32[P1_NT / 32 + 1];
    uint32_t cnt[8];
    unsigned long long tmp_base;
};

// bits [a, a+32) of a bitmask (bit x&31 of word x>>5 is position x)
__device__ __forceinline__ uint32_t bits32_at(const uint32_t* m, int a) {
    return __funnelshift_r(m[a >> 5], m[(a >> 5) + 1], a & 31);
}

template <int MODE>
__global__ void __launch_bounds__(P1_NT) k_pass(P1Args a) {
    extern __shared__ __align__(16) uint8_t p1_smem[];
    P1Smem& S = *reinterpret_cast<P1Smem*>(p1_smem);
    uint32_t* pre = S.pre;
    uint32_t* suf = S.suf;
    uint32_t* pk = S.pk;

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int64_t q0 = (int64_t)blockIdx.x * P1_TILE;
    const int64_t lbase = q0 - LEFT;  // stream position of smem index 0
    const int64_t nb = (int64_t)a.n_bases;
    const int k = a.k, p = a.p;
    const uint64_t r0 = a.tile_r_lo[blockIdx.x];  // issued early: its latency overlaps S1

    // ---- S1: load ASCII (16-byte vectors), encode A0 C1 G2 T3 four bytes at a time
    //      (lowercase folded); non-ACGT bytes and bytes outside the stream -> inv bits
    uint32_t n_invalid = 0;
    for (int v = tid; v < NB / 16; v += P1_NT) {
        const int64_t q = lbase + 16 * v;
        uint32_t wd[4];
        if (a.reads_aligned16 && q >= 0 && q + 16 <= nb) {
            const uint4 w = *reinterpret_cast<const uint4*>(a.reads + q);
            wd[0] = w.x; wd[1] = w.y; wd[2] = w.z; wd[3] = w.w;
        } else {
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                uint32_t x = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int64_t qq = q + 4 * t + j;
                    const uint32_t b = (qq >= 0 && qq < nb) ? a.reads[qq] : (uint32_t)'N';
                    x |= b << (8 * j);
                }
                wd[t] = x;
            }
        }
        uint32_t packed = 0, invbits = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
            const uint32_t c = wd[t] & 0xDFDFDFDFu;
            const uint32_t ok = __vcmpeq4(c, 0x41414141u) | __vcmpeq4(c, 0x43434343u) | __vcmpeq4(c, 0x47474747u) |
                                __vcmpeq4(c, 0x54545454u);
            const uint32_t cd = ((c >> 1) ^ (c >> 2)) & 0x03030303u;  // per byte: A0 C1 G2 T3
            const uint32_t b8 = ((cd & 0xFFu) << 6) | (((cd >> 8) & 0xFFu) << 4) | (((cd >> 16) & 0xFFu) << 2) |
                                (cd >> 24);
            packed |= b8 << (24 - 8 * t);
            const uint32_t bad = (~ok) & 0x01010101u;
            invbits |= (((bad * 0x01020408u) >> 24) & 0xFu) << (4 * t);
        }
        pk[v] = packed;
        reinterpret_cast<uint16_t*>(S.inv)[v] = (uint16_t)invbits;
        // invalid bytes inside the tile's own window starts [LEFT, LEFT+TILE) and the stream
        const int li = 16 * v;
        if (li >= LEFT && li < LEFT + P1_TILE) {
            uint32_t m = invbits;
            if (q + 16 > nb) m &= (q >= nb) ? 0u : ((1u << (uint32_t)(nb - q)) - 1u);
            n_invalid += __popc(m);
        }
    }
    if (tid < NWD - NB / 32) {
        S.inv[NB / 32 + tid] = 0xFFFFFFFFu;
        S.rs[NB / 32 + tid] = 0;
    }
    if (tid < 8) pk[NB / 16 + tid] = 0;
    for (int w = tid; w < NB / 32; w += P1_NT) S.rs[w] = 0;
    __syncthreads();
    // ---- read starts inside (lbase, lbase + NB): segment breaks
    for (uint64_t rb = r0;; rb += P1_NT) {
        const uint64_t r = rb + tid;
        bool inr = false;
        if (r <= a.n_reads) {
            const int64_t st = (int64_t)(a.offsets[r] - a.off0) - lbase;
            if (st < NB) {
                inr = true;
                if (st > 0) atomicOr(&S.rs[st >> 5], 1u << (st & 31));
            }
        }
        if (!__syncthreads_or(inr && tid == P1_NT - 1)) break;
    }
    // ---- validity bitmasks: window i valid iff bases [i, i+k) are all valid and no read
    //      starts in (i, i+k); p-mer j likewise over [j, j+p).  ext(x) = valid(x) & !rs(x).
    for (int w = tid; w < NWD; w += P1_NT) S.ext[w] = ~(S.inv[w] | S.rs[w]);
    __syncthreads();
    // one thread per mask word: AND of ext over the next L positions from three register-
    // held words (window: L = k-1 -> vwin; p-mer: L = p-1 -> vpm), then AND with !inv(i)
    {
        constexpr int NWU = NB / 32 + 1;  // words covering every window / p-mer start we use
        for (int t = tid; t < 2 * NWU; t += P1_NT) {
            const int w = t < NWU ? t : t - NWU;
            const int L = t < NWU ? k - 1 : p - 1;
            const uint32_t x0 = S.ext[w], x1 = S.ext[w + 1], x2 = S.ext[w + 2];
            uint32_t acc = 0xFFFFFFFFu;
            for (int o = 1; o <= L; ++o)
                acc &= o < 32 ? __funnelshift_r(x0, x1, o) : (o == 32 ? x1 : __funnelshift_r(x1, x2, o - 32));
            const uint32_t v = ~S.inv[w] & acc;
            if (t < NWU) S.vwin[w] = v;
            else S.vpm[w] = v;
        }
    }
    __syncthreads();
    // ---- S2a: canonical p-mer key of every position j:
    //      key = min(fwd, rc) if that p-mer is valid and allowed, else the reserved 4^p (R4)
    const uint32_t RES = 1u << (2 * p);
    const int NBK = NB - p + 1;
    {
        const uint32_t pmask = (1u << (2 * p)) - 1;
        const int top = 2 * p - 2;
        const int b0 = tid * CH, b1 = min(NBK, b0 + CH);
        uint32_t fwd = 0, rc = 0;
        if (b0 < b1) {
            for (int j = b0; j < b0 + p - 1; ++j) {
                const uint32_t c = (pk[j >> 4] >> (30 - 2 * (j & 15))) & 3u;
                fwd = ((fwd << 2) | c) & pmask;
                rc = (rc >> 2) | ((3u - c) << top);
            }
        }
        for (int j = b0; j < b1; ++j) {
            const int jj = j + p - 1;
            const uint32_t c = (pk[jj >> 4] >> (30 - 2 * (jj & 15))) & 3u;
            fwd = ((fwd << 2) | c) & pmask;
            rc = (rc >> 2) | ((3u - c) << top);
            const uint32_t cn = fwd < rc ? fwd : rc;
            const bool ok = ((S.vpm[j >> 5] >> (j & 31)) & 1u) && sig_allowed(cn, p);
            pre[j] = ok ? cn : RES;
        }
        for (int j = max(b0, NBK); j < min(NB, b0 + CH); ++j) pre[j] = RES;
    }
    __syncthreads();
    // ---- S2b: sliding-window minimum over W = k-p+1 consecutive p-mers (van Herk /
    //      Gil-Werman): blocks of W; suffix minima into suf[], prefix minima in place in
    //      pre[]; sig(i) = min(suf[i], pre[i+W-1]).
    const int W = k - p + 1;
    {
        const int nblk = (NBK + W - 1) / W;
        for (int b = tid; b < nblk; b += P1_NT) {
            const int s0 = b * W, e = min(NBK, s0 + W);
            uint32_t m = 0xFFFFFFFFu;
            for (int j = e - 1; j >= s0; --j) {
                m = min(m, pre[j]);
                suf[j] = m;
            }
            m = 0xFFFFFFFFu;
            for (int j = s0; j < e; ++j) {
                m = min(m, pre[j]);
                pre[j] = m;
            }
        }
    }
    __syncthreads();
    // signature per window i in [LEFT-1, LEFT+TILE) (window q0-1 only for the run test),
    // INV where the window is not valid (crosses a read end or holds a non-ACGT byte)
    for (int i = LEFT - 1 + tid; i < LEFT + P1_TILE; i += P1_NT) {
        const bool ok = (S.vwin[i >> 5] >> (i & 31)) & 1u;
        suf[i] = ok ? min(suf[i], pre[i + W - 1]) : INV;
    }
    __syncthreads();
    uint32_t* key = suf;

    if (MODE == P1_MODE_DEBUG) {
        for (int w = tid; w < P1_TILE; w += P1_NT) {
            const int64_t q = q0 + w;
            if (q < nb) a.dbg_sig[q] = key[LEFT + w];
        }
        return;
    }

    // ---- S3: super-k-mers = maximal runs of valid windows with equal signature
    //      (Fig. 1); record runs are additionally cut at the tile edge and
    //      into pieces of at most record_max_windows(k) windows.  Warp ballots build a
    //      bitmask of the windows where a run cannot continue (invalid or a new start)
    //      and a compacted list of run starts; a run's length is the distance to the
    //      next set bit.
    const int maxw = record_max_windows(k);
    const int RW = record_words(k);
    uint32_t* ebits = S.ebits;
    uint32_t* list = pre;  // pre[] is free after the signatures are formed
    if (tid < 8) S.cnt[tid] = 0;
    __syncthreads();
    uint32_t l_skm = 0;
#pragma unroll 4
    for (int w = 0; w < WPT; ++w) {
        const int i = LEFT + w * P1_NT + tid;
        const uint32_t s = key[i], prev = key[i - 1];
        const bool valid = s != INV;
        const bool skm = valid && prev != s;
        const bool start = skm || (valid && i == LEFT);
        const uint32_t bE = __ballot_sync(0xffffffffu, !valid || start);
        const uint32_t bS = __ballot_sync(0xffffffffu, start);
        l_skm += skm;
        uint32_t base = 0;
        if (lane == 0) {
            ebits[(w * P1_NT + warp * 32) >> 5] = bE;
            if (bS) base = atomicAdd(&S.cnt[0], (uint32_t)__popc(bS));
        }
        base = __shfl_sync(0xffffffffu, base, 0);
        if (start) list[base + __popc(bS & lanemask_lt())] = (uint32_t)i;
    }
    if (tid == 0) ebits[P1_TILE >> 5] = 1u;  // sentinel: the tile edge ends every run
    __syncthreads();
    const int nstarts = (int)S.cnt[0];
    // record words of the run piece starting at smem index ii with m windows: word 0 =
    // m (8 bits) + symbols [0,12); word u>0 = symbols [12+16(u-1), 12+16u); extracted from
    // the packed tile by funnel shifts
    auto pack = [&](int ii, int m, uint32_t (&wd4)[8]) {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (u >= RW) break;
            const int b = ii + (u == 0 ? 0 : 12 + 16 * (u - 1));
            const uint32_t x = __funnelshift_l(pk[(b >> 4) + 1], pk[b >> 4], 2 * (b & 15));
            wd4[u] = (u == 0) ? (((uint32_t)m << 24) | (x >> 8)) : x;
        }
    };
    auto run_len = [&](int i) {
        const int pos = i - LEFT + 1;
        int wd = pos >> 5;
        uint32_t bits = ebits[wd] & (0xFFFFFFFFu << (pos & 31));
        while (bits == 0) bits = ebits[++wd];
        return (wd * 32 + __ffs(bits) - 1) - (i - LEFT);
    };
    uint32_t l_windows = 0, l_recs = 0;
    for (int idx = tid; idx < nstarts; idx += P1_NT) {
        const int i = (int)list[idx];
        const uint32_t s = key[i];
        const int n = run_len(i);
        const int nrec = n <= maxw ? 1 : (n + maxw - 1) / maxw;
        l_windows += n;
        l_recs += nrec;
        if (MODE == P1_MODE_HIST) {
            atomicAdd(&a.hist_w[s], (unsigned long long)n);
            atomicAdd(&a.hist_r[s], (uint32_t)nrec);
        } else {
            // ---- S5 (recompute path): write each piece as a bin record (P:L258-259:
            //      super-k-mers "are sent to bins ... related to signatures"); bins live in
            //      HBM.
            const uint32_t bin = a.sig2bin[s];
            const uint64_t base = a.bin_rec_off[bin];
            const int j = i + n;
            for (int ii = i; ii < j; ii += maxw) {
                const int m = min(maxw, j - ii);
                uint32_t wd4[8];
                pack(ii, m, wd4);
                const uint32_t slot = atomicAdd(&a.bin_fill[bin], 1u);
                uint4* dst = reinterpret_cast<uint4*>(a.bins + (base + slot) * (uint64_t)RW);
                dst[0] = make_uint4(wd4[0], wd4[1], wd4[2], wd4[3]);
                if (RW == 8) dst[1] = make_uint4(wd4[4], wd4[5], wd4[6], wd4[7]);
            }
        }
    }
    if (MODE == P1_MODE_HIST) {
        // ---- the tile's records are also appended, unbinned and tagged with their
        //      signature, to a temporary stream; S5 then only copies them into their bins
        if (a.tmp_recs) {
            uint32_t tot;
            uint32_t rpos = block_excl_sum<P1_NT, uint32_t>(l_recs, S.wsum32, &tot);
            if (tid == 0) S.tmp_base = tot ? atomicAdd(&a.gstats[GS_TMP_RECS], (unsigned long long)tot) : 0ull;
            __syncthreads();
            const unsigned long long base = S.tmp_base;
            if (base + tot <= a.tmp_cap) {
                for (int idx = tid; idx < nstarts; idx += P1_NT) {
                    const int i = (int)list[idx];
                    const uint32_t s = key[i];
                    const int j = i + run_len(i);
                    for (int ii = i; ii < j; ii += maxw) {
                        uint32_t wd4[8];
                        pack(ii, min(maxw, j - ii), wd4);
                        const uint64_t slot = base + rpos++;
                        uint4* dst = reinterpret_cast<uint4*>(a.tmp_recs + slot * (uint64_t)RW);
                        dst[0] = make_uint4(wd4[0], wd4[1], wd4[2], wd4[3]);
                        if (RW == 8) dst[1] = make_uint4(wd4[4], wd4[5], wd4[6], wd4[7]);
                        a.tmp_sig[slot] = s;
                    }
                }
            }
        }
        const uint32_t tw = __reduce_add_sync(0xffffffffu, l_windows);
        const uint32_t ts = __reduce_add_sync(0xffffffffu, l_skm);
        const uint32_t tr = __reduce_add_sync(0xffffffffu, l_recs);
        const uint32_t ti = __reduce_add_sync(0xffffffffu, n_invalid);
        if (lane == 0) {
            atomicAdd(&S.cnt[1], tw);
            atomicAdd(&S.cnt[2], ts);
            atomicAdd(&S.cnt[3], tr);
            atomicAdd(&S.cnt[4], ti);
        }
        __syncthreads();
        if (tid == 0) {
            if (S.cnt[1]) atomicAdd(&a.gstats[GS_WINDOWS], (unsigned long long)S.cnt[1]);
            if (S.cnt[2]) atomicAdd(&a.gstats[GS_SUPERKMERS], (unsigned long long)S.cnt[2]);
            if (S.cnt[3]) atomicAdd(&a.gstats[GS_RECORDS], (unsigned long long)S.cnt[3]);
            if (S.cnt[4]) atomicAdd(&a.gstats[GS_INVALID], (unsigned long long)S.cnt[4]);
        }
    }
}

// S5 from the temporary stream: every record is copied into its bin (signature -> bin
// map of the plan); one atomic per (warp, bin) reserves the slots.  Each thread carries
// BS_U records through the dependent steps (signature -> bin -> slot -> copy) together,
// so BS_U independent memory round trips are in flight per step instead of one.
constexpr int BS_NT = 256, BS_U = 4;
__global__ void __launch_bounds__(BS_NT) k_bin_scatter(const uint32_t* __restrict__ tmp_recs,
                                                       const uint32_t* __restrict__ tmp_sig, uint64_t n, int RW,
                                                       const uint32_t* __restrict__ sig2bin,
                                                       const uint64_t* __restrict__ bin_rec_off,
                                                       uint32_t* __restrict__ bin_fill, uint32_t* __restrict__ bins) {
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t ltm = lanemask_lt();
    constexpr uint64_t STEP = (uint64_t)BS_NT * BS_U;
    for (uint64_t base = (uint64_t)blockIdx.x * STEP; base < n; base += (uint64_t)gridDim.x * STEP) {
        uint32_t bin[BS_U];
        uint64_t slot[BS_U];
        uint4 r0[BS_U], r1[BS_U];
#pragma unroll
        for (int u = 0; u < BS_U; ++u) {
            const uint64_t i = base + (uint64_t)u * BS_NT + threadIdx.x;
            bin[u] = i < n ? __ldcs(tmp_sig + i) : 0xFFFFFFFFu;
            if (i < n) {
                const uint4* src = reinterpret_cast<const uint4*>(tmp_recs + i * (uint64_t)RW);
                r0[u] = __ldcs(src);
                if (RW == 8) r1[u] = __ldcs(src + 1);
            }
        }
#pragma unroll
        for (int u = 0; u < BS_U; ++u)
            if (bin[u] != 0xFFFFFFFFu) bin[u] = sig2bin[bin[u]];
#pragma unroll
        for (int u = 0; u < BS_U; ++u) {
            const uint32_t peers = __match_any_sync(0xffffffffu, bin[u]);
            const uint32_t leader = __ffs(peers) - 1;
            uint32_t b = 0;
            if (bin[u] != 0xFFFFFFFFu && lane == leader) b = atomicAdd(&bin_fill[bin[u]], (uint32_t)__popc(peers));
            slot[u] = (uint64_t)__shfl_sync(0xffffffffu, b, leader) + __popc(peers & ltm);
        }
#pragma unroll
        for (int u = 0; u < BS_U; ++u)
            if (bin[u] != 0xFFFFFFFFu) slot[u] += bin_rec_off[bin[u]];
#pragma unroll
        for (int u = 0; u < BS_U; ++u) {
            if (bin[u] == 0xFFFFFFFFu) continue;
            uint4* dst = reinterpret_cast<uint4*>(bins + slot[u] * (uint64_t)RW);
            dst[0] = r0[u];
            if (RW == 8) dst[1] = r1[u];
        }
    }
}

__global__ void k_debug_allowed(int p, uint8_t* out) {
    uint64_t n = 1ull << (2 * p);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = sig_allowed((uint32_t)i, p) ? 1 : 0;
}

}  // namespace

uint64_t p1_num_tiles(uint64_t n_bases) { return (n_bases + P1_TILE - 1) / P1_TILE; }

cudaError_t launch_tile_reads(const uint64_t* offsets, uint64_t n_reads, uint64_t off0, uint64_t n_tiles,
                              uint64_t* tile_r_lo, cudaStream_t s) {
    if (n_tiles == 0) return cudaSuccess;
    k_tile_reads<<<(unsigned)((n_tiles + 255) / 256), 256, 0, s>>>(offsets, n_reads, off0, n_tiles, tile_r_lo);
    return cudaGetLastError();
}

cudaError_t launch_p1(int mode, const P1Args& a, uint64_t n_tiles, cudaStream_t s) {
    if (n_tiles == 0) return cudaSuccess;
    dim3 grid((unsigned)n_tiles);
    const int sm = (int)sizeof(P1Smem);
    cudaError_t e;
    if (mode == P1_MODE_HIST) {
        if ((e = cudaFuncSetAttribute(k_pass<P1_MODE_HIST>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm))) return e;
        k_pass<P1_MODE_HIST><<<grid, P1_NT, sm, s>>>(a);
    } else if (mode == P1_MODE_SCATTER) {
        if ((e = cudaFuncSetAttribute(k_pass<P1_MODE_SCATTER>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm))) return e;
        k_pass<P1_MODE_SCATTER><<<grid, P1_NT, sm, s>>>(a);
    } else {
        if ((e = cudaFuncSetAttribute(k_pass<P1_MODE_DEBUG>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm))) return e;
        k_pass<P1_MODE_DEBUG><<<grid, P1_NT, sm, s>>>(a);
    }
    return cudaGetLastError();
}

cudaError_t launch_bin_scatter(const uint32_t* tmp_recs, const uint32_t* tmp_sig, uint64_t n, int k,
                               const uint32_t* sig2bin, const uint64_t* bin_rec_off, uint32_t* bin_fill,
                               uint32_t* bins, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    const unsigned grid = (unsigned)std::min<uint64_t>((n + BS_NT * BS_U - 1) / (BS_NT * BS_U), 148ull * 8);
    k_bin_scatter<<<grid, BS_NT, 0, s>>>(tmp_recs, tmp_sig, n, record_words(k), sig2bin, bin_rec_off, bin_fill, bins);
    return cudaGetLastError();
}

cudaError_t launch_debug_allowed(int p, uint8_t* out, cudaStream_t s) {
    k_debug_allowed<<<256, 256, 0, s>>>(p, out);
    return cudaGetLastError();
}

}  // namespace kmc
