// k_distribute.cu -- phase 1 of KMC 2 on the B200 (Sec. 2.4 "distribution"):
// S1 encode + split at non-ACGT and read ends, S2 signatures, S3 super-k-mer cut,
// S4 histogram (pass 1) and S5 scatter of super-k-mer records into HBM bins (pass 2).
//
// One CTA owns a tile of P1_TILE consecutive window starts of the concatenated base
// stream (windows never cross read boundaries: reads are marked from read_offsets).
// Everything between the ASCII load and the histogram / bin write stays in shared
// memory: codes, valid-run lengths, the canonical p-mer key of every position, the
// van Herk / Gil-Werman block prefix/suffix minima, and the per-window signature.
#include "kmc_device.cuh"
#include "kmc_internal.h"

namespace kmc {

namespace {

constexpr int LEFT = 16;                      // halo before the tile (window q0-1 + alignment)
constexpr int NB = P1_TILE + LEFT + 64;       // loaded bases (k <= 64); multiple of 16
constexpr int CH = (NB + P1_NT - 1) / P1_NT;  // positions per thread in the scans
constexpr int WPT = P1_TILE / P1_NT;          // windows owned per thread
constexpr uint32_t INV = 0xFFFFFFFFu;
static_assert(NB % 16 == 0, "NB");

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

struct P1Smem {
    uint32_t key[NB];            // p-mer keys, then per-window signatures
    uint32_t pre[NB];            // block prefix minima
    uint32_t suf[NB];            // block suffix minima
    uint32_t pk[NB / 16 + 8];    // 2-bit packed codes, 16 per word, MSB first
    uint32_t wsum32[P1_NT / 32 + 1];
    int32_t wmax[P1_NT / 32];
    uint8_t code[NB];            // 0..3 = A,C,G,T; 4 = invalid
    uint8_t rsf[NB];             // 1 where a read starts
    uint8_t run[NB];             // valid-run length ending here (capped at 255)
};

template <int MODE>
__global__ void __launch_bounds__(P1_NT) k_pass(P1Args a) {
    extern __shared__ __align__(16) uint8_t p1_smem[];
    P1Smem& S = *reinterpret_cast<P1Smem*>(p1_smem);
    uint8_t(&code)[NB] = S.code;
    uint8_t(&rsf)[NB] = S.rsf;
    uint8_t(&run)[NB] = S.run;
    uint32_t(&key)[NB] = S.key;
    uint32_t(&pre)[NB] = S.pre;
    uint32_t(&suf)[NB] = S.suf;
    uint32_t(&pk)[NB / 16 + 8] = S.pk;
    uint32_t* wsum32 = S.wsum32;
    int32_t* wmax = S.wmax;

    const int tid = threadIdx.x;
    const int64_t q0 = (int64_t)blockIdx.x * P1_TILE;
    const int64_t lbase = q0 - LEFT;  // stream position of smem index 0
    const int64_t nb = (int64_t)a.n_bases;
    const int k = a.k, p = a.p;

    // ---- S1: load ASCII, encode to 2-bit codes (invalid -> 4), clear read-start flags
    uint32_t n_invalid = 0;
    for (int v = tid; v < NB / 16; v += P1_NT) {
        const int64_t q = lbase + 16 * v;
        uint8_t bytes[16];
        if (a.reads_aligned16 && q >= 0 && q + 16 <= nb) {
            uint4 w = *reinterpret_cast<const uint4*>(a.reads + q);
            *reinterpret_cast<uint4*>(bytes) = w;
        } else {
#pragma unroll
            for (int j = 0; j < 16; ++j) bytes[j] = (q + j >= 0 && q + j < nb) ? a.reads[q + j] : (uint8_t)'N';
        }
        uint32_t packed = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            uint32_t c = encode_base(bytes[j]);
            packed |= (c & 3u) << (30 - 2 * j);
            code[16 * v + j] = (uint8_t)c;
            rsf[16 * v + j] = 0;
            const int li = 16 * v + j;
            if (c == 4u && li >= LEFT && li < LEFT + P1_TILE && q + j < nb) ++n_invalid;
        }
        pk[v] = packed;
    }
    if (tid < 8) pk[NB / 16 + tid] = 0;
    __syncthreads();
    // ---- read starts inside (lbase, lbase + NB): segment breaks
    {
        uint64_t r0 = a.tile_r_lo[blockIdx.x];
        for (uint64_t rb = r0;; rb += P1_NT) {
            uint64_t r = rb + tid;
            bool inr = false;
            if (r <= a.n_reads) {
                int64_t s = (int64_t)(a.offsets[r] - a.off0) - lbase;
                if (s < NB) {
                    inr = true;
                    if (s > 0) rsf[s] = 1;
                }
            }
            if (!__syncthreads_or(inr && tid == P1_NT - 1)) break;
        }
    }
    __syncthreads();
    // ---- valid-run length ending at each position: run(e) = e - max_{x<=e} brk(x) + 1,
    //      brk(x) = x+1 if base x invalid, x if a read starts at x
    {
        const int b0 = tid * CH, b1 = min(NB, b0 + CH);
        int32_t m = 0;
        for (int x = b0; x < b1; ++x) {
            int32_t br = code[x] == 4 ? x + 1 : (rsf[x] ? x : 0);
            m = max(m, br);
        }
        // block exclusive prefix max
        const int lane = tid & 31, warp = tid >> 5;
        int32_t inc = m;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int32_t n = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc = max(inc, n);
        }
        if (lane == 31) wmax[warp] = inc;
        int32_t ex = __shfl_up_sync(0xffffffffu, inc, 1);
        if (lane == 0) ex = 0;
        __syncthreads();
        for (int w = 0; w < warp; ++w) ex = max(ex, wmax[w]);
        int32_t cur = ex;
        for (int x = b0; x < b1; ++x) {
            int32_t br = code[x] == 4 ? x + 1 : (rsf[x] ? x : 0);
            cur = max(cur, br);
            run[x] = (uint8_t)min(255, x - cur + 1);
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
                uint32_t c = code[j] & 3u;
                fwd = ((fwd << 2) | c) & pmask;
                rc = (rc >> 2) | ((3u - c) << top);
            }
        }
        for (int j = b0; j < b1; ++j) {
            uint32_t c = code[j + p - 1] & 3u;
            fwd = ((fwd << 2) | c) & pmask;
            rc = (rc >> 2) | ((3u - c) << top);
            uint32_t cn = fwd < rc ? fwd : rc;
            bool ok = run[j + p - 1] >= p && sig_allowed(cn, p);
            key[j] = ok ? cn : RES;
        }
        for (int j = max(b0, NBK); j < min(NB, b0 + CH); ++j) key[j] = RES;
    }
    __syncthreads();
    // ---- S2b: sliding-window minimum over W = k-p+1 consecutive p-mers (van Herk /
    //      Gil-Werman): blocks of W, prefix minima pre[] and suffix minima suf[];
    //      sig(i) = min(suf[i], pre[i+W-1]).
    const int W = k - p + 1;
    {
        const int nblk = (NBK + W - 1) / W;
        for (int b = tid; b < nblk; b += P1_NT) {
            const int s = b * W, e = min(NBK, s + W);
            uint32_t m = 0xFFFFFFFFu;
            for (int j = s; j < e; ++j) {
                m = min(m, key[j]);
                pre[j] = m;
            }
            m = 0xFFFFFFFFu;
            for (int j = e - 1; j >= s; --j) {
                m = min(m, key[j]);
                suf[j] = m;
            }
        }
    }
    __syncthreads();
    // signature per window i in [LEFT-1, LEFT+TILE) (window q0-1 only for the run test),
    // INV where the window is not valid (crosses a read end or holds a non-ACGT byte)
    for (int i = LEFT - 1 + tid; i < LEFT + P1_TILE; i += P1_NT) {
        const bool ok = run[i + k - 1] >= k;
        key[i] = ok ? min(suf[i], pre[i + W - 1]) : INV;
    }
    __syncthreads();

    if (MODE == P1_MODE_DEBUG) {
        for (int w = tid; w < P1_TILE; w += P1_NT) {
            const int64_t q = q0 + w;
            if (q < nb) a.dbg_sig[q] = key[LEFT + w];
        }
        return;
    }

    // ---- S3: super-k-mers = maximal runs of valid windows with equal signature
    //      (Fig. 1); record runs are additionally cut at the tile edge and
    //      into pieces of at most record_max_windows(k) windows.
    const int maxw = record_max_windows(k);
    const int RW = record_words(k);
    uint32_t l_windows = 0, l_skm = 0, l_recs = 0;
    for (int w = 0; w < WPT; ++w) {
        const int i = LEFT + tid * WPT + w;
        const uint32_t s = key[i];
        if (s == INV) continue;
        const uint32_t prev = key[i - 1];
        const bool skm_start = prev != s;
        if (!skm_start && i != LEFT) continue;
        l_skm += skm_start;
        int j = i + 1;
        while (j < LEFT + P1_TILE && key[j] == s) ++j;
        const int n = j - i;
        const int nrec = (n + maxw - 1) / maxw;
        l_windows += n;
        l_recs += nrec;
        if (MODE == P1_MODE_HIST) {
            atomicAdd(&a.hist_w[s], (unsigned long long)n);
            atomicAdd(&a.hist_r[s], (uint32_t)nrec);
        } else {
            // ---- S5: write each piece as a bin record (super-k-mers "are sent
            //      to bins ... related to signatures"); bins live in HBM.
            const uint32_t bin = a.sig2bin[s];
            const uint64_t base = a.bin_rec_off[bin];
            for (int ii = i; ii < j; ii += maxw) {
                const int m = min(maxw, j - ii);
                // record words: word 0 = n (8 bits) + symbols [0,12); word u>0 = symbols
                // [12+16(u-1), 12+16u); extracted from the packed tile by funnel shifts
                uint32_t wd[8];
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    if (u >= RW) break;
                    const int b = ii + (u == 0 ? 0 : 12 + 16 * (u - 1));
                    const uint32_t x = __funnelshift_l(pk[(b >> 4) + 1], pk[b >> 4], 2 * (b & 15));
                    wd[u] = (u == 0) ? (((uint32_t)m << 24) | (x >> 8)) : x;
                }
                const uint32_t slot = atomicAdd(&a.bin_fill[bin], 1u);
                uint4* dst = reinterpret_cast<uint4*>(a.bins + (base + slot) * (uint64_t)RW);
                dst[0] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
                if (RW == 8) dst[1] = make_uint4(wd[4], wd[5], wd[6], wd[7]);
            }
        }
    }
    if (MODE == P1_MODE_HIST) {
        uint32_t tw = block_sum<P1_NT, uint32_t>(l_windows, wsum32);
        uint32_t ts = block_sum<P1_NT, uint32_t>(l_skm, wsum32);
        uint32_t tr = block_sum<P1_NT, uint32_t>(l_recs, wsum32);
        uint32_t ti = block_sum<P1_NT, uint32_t>(n_invalid, wsum32);
        if (tid == 0) {
            if (tw) atomicAdd(&a.gstats[GS_WINDOWS], (unsigned long long)tw);
            if (ts) atomicAdd(&a.gstats[GS_SUPERKMERS], (unsigned long long)ts);
            if (tr) atomicAdd(&a.gstats[GS_RECORDS], (unsigned long long)tr);
            if (ti) atomicAdd(&a.gstats[GS_INVALID], (unsigned long long)ti);
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

cudaError_t launch_debug_allowed(int p, uint8_t* out, cudaStream_t s) {
    k_debug_allowed<<<256, 256, 0, s>>>(p, out);
    return cudaGetLastError();
}

}  // namespace kmc
