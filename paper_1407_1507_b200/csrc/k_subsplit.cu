// k_subsplit.cu -- S6-S8 of the large bins through sub-signatures (large_path 4, 22 <= k <= 32;
// DESIGN.md 5).
//
// The paper sorts each bin after extracting its k-mers.  A bin
// above one CTA's shared memory must be cut into parts whose k-mers can be counted apart:
// every copy of a k-mer must land in the same part.  The one-pass split (k_split1.cu) cuts by
// a hash of every KEY and writes all 2.8 G keys of C4 to HBM and reads them back.  Here the
// part of a k-mer is a function of its content that is constant along runs of consecutive
// windows -- a second, finer signature, computed the way the paper computes the first one
// (P:L146-147): the minimum, over the k-mer's W2 = k - q + 1 canonical q-mers, of a hash
// of the q-mer (q = min(16, k - 12); the hash order avoids the poly-A skew of a
// lexicographic minimum).  digit = (fmix(sub-signature) x nd) >> 32.  A bin record (a piece
// of one super-k-mer) is cut where the digit changes into SUB-RECORDS -- ~5 windows each at
// C4, in the bin record format -- and every sub-record goes to its digit.  A digit is then
// counted from its sub-records alone: 16 bytes move per ~5 windows instead of 8 per window.
//
//   k_subsplit (persistent, 512 threads, pieces of one bin, TMA double-buffered):
//     D  units of <= 8 windows: q-mer hashes of the unit (+ the window before it), van Herk
//        sliding minimum, digits, sub-record starts (a 64-bit mask per record), SMEM digit
//        histogram;
//     R  one reservation per (piece, digit) on the digit's sub-record counter; pool blocks
//        of SS_BLK sub-records are claimed for the digit's block table by CAS (a digit holds
//        up to SS_MAXB blocks; beyond them sub-records go to the overflow list);
//     E  every start builds its sub-record (length from the record's start mask) and places it
//        in a shared-memory stage grouped by digit;
//     W  every digit's run leaves by TMA bulk copies (one per pool block it touches).
//   k_subcount (persistent CTA per SM, 1024 threads, 16 K-slot SMEM hash table): per digit,
//     warps stream batches of 32 sub-records, split them into units of <= 33-k windows,
//     expand the keys (min(fwd, rc)) and count them in the table; then the table
//     scan applies the cutoffs (S8).  A digit whose distinct keys overflow the table is
//     counted again in R = 2, 4, .. rounds, each inserting only the keys of one hash range
//     (nested ranges: the rounds already emitted stay valid).  A digit whose sub-records
//     overflowed its block table is listed for the device-LSD fallback.
#include <algorithm>

#include "kmc_device.cuh"
#include "kmc_internal.h"

namespace kmc {

namespace {

constexpr int SS_NT = 512;
constexpr int SS_REC = 496;        // records per piece at most
constexpr int SS_U = 8;            // windows per digit unit
constexpr int SS_WMAX = 16384;     // windows per piece at most (digit bytes)
constexpr int SS_UMAX = 2560;      // units per piece at most
constexpr int SS_STAGE = 2048;     // sub-records staged per piece
constexpr int SS_RBW = SS_REC * 4 + 16;  // record buffer words (+ pad: units read past the record)
constexpr int SS_BPR = SS_STAGE / SS_BLK + 2;  // pool blocks one staged run can touch

constexpr size_t SS_OFF_STAGE = 0;
constexpr size_t SS_OFF_RB = SS_OFF_STAGE + (size_t)SS_STAGE * 16;
constexpr size_t SS_OFF_MASK = SS_OFF_RB + 2 * (size_t)SS_RBW * 4;
constexpr size_t SS_OFF_RINFO = SS_OFF_MASK + (size_t)SS_REC * 8;
constexpr size_t SS_OFF_WPRE = SS_OFF_RINFO + (size_t)SS_REC * 4;
constexpr size_t SS_OFF_UMAP = SS_OFF_WPRE + (size_t)SS_REC * 4;
constexpr size_t SS_OFF_DIGS = SS_OFF_UMAP + (size_t)SS_UMAX * 2;
constexpr size_t SS_OFF_DTAB = SS_OFF_DIGS + (size_t)SS_WMAX;            // per digit: h, hw, gst, lof, lc, ovb
constexpr size_t SS_OFF_BIDS = SS_OFF_DTAB + 6 * (size_t)SS_DMAX * 4;     // per digit: SS_BPR block ids
constexpr size_t SS_OFF_MBAR = SS_OFF_BIDS + (size_t)SS_DMAX * SS_BPR * 4;
constexpr size_t SS_SMEM = SS_OFF_MBAR + 16 + 16;
static_assert(SS_OFF_RB % 16 == 0 && SS_OFF_MASK % 8 == 0 && SS_OFF_MBAR % 8 == 0, "alignment");
static_assert(SS_DMAX <= SS_NT, "one thread per digit");
static_assert(SS_DMAX <= 256, "digits are stored as bytes");

// murmur3's 32-bit finaliser: the sub-signature is a MINIMUM of hashes (small values are
// over-represented), so it is mixed again before it picks a digit
__device__ __forceinline__ uint32_t fmix32(uint32_t h) {
    h ^= h >> 16;
    h *= 0x85EBCA6Bu;
    h ^= h >> 13;
    h *= 0xC2B2AE35u;
    h ^= h >> 16;
    return h;
}
__device__ __forceinline__ uint32_t bits32_be(const uint32_t* w, int b) {
    const int q = b >> 5, r = b & 31;
    return __funnelshift_l(w[q + 1], w[q], r);
}

// Digits of windows a-1 .. a+U-1 of a record (D[t] = window a-1+t; t = 0 is garbage when
// a = 0), computed from the record's big-endian symbol string.  KK = k (compile time).
template <int KK>
__device__ __forceinline__ void unit_digits(const uint32_t* rec, int a, uint32_t nd, uint32_t (&D)[SS_U + 1]) {
    constexpr int Q = KK <= 28 ? KK - 12 : 16;  // q-mer length
    constexpr int W2 = KK - Q + 1;              // q-mers per window (13..17)
    constexpr int NP = SS_U + W2;               // q-mer positions of windows a-1 .. a+U-1
    constexpr uint32_t MQ = Q == 16 ? 0xFFFFFFFFu : ((1u << (2 * Q)) - 1u);
    static_assert(NP - 1 + Q <= 48, "positions fit three words");
    // symbols a-1 .. a+46 = bits [6 + 2a, +96) of the record string: the record's 4 words and
    // the next 2 (one 16-byte and one 8-byte shared load; a is a multiple of 8, so the word
    // offset is 0..2 and the bit offset 6 or 22)
    const uint4 v = *reinterpret_cast<const uint4*>(rec);
    const uint2 v2 = *reinterpret_cast<const uint2*>(rec + 4);
    const int b = 6 + 2 * a, q = b >> 5, rs = b & 31;
    const uint32_t w0 = q == 0 ? v.x : q == 1 ? v.y : v.z;
    const uint32_t w1 = q == 0 ? v.y : q == 1 ? v.z : v.w;
    const uint32_t w2 = q == 0 ? v.z : q == 1 ? v.w : v2.x;
    const uint32_t w3 = q == 0 ? v.w : q == 1 ? v2.x : v2.y;
    const uint32_t A0 = __funnelshift_l(w1, w0, rs), A1 = __funnelshift_l(w2, w1, rs), A2 = __funnelshift_l(w3, w2, rs);
    const uint64_t X0 = ((uint64_t)A0 << 32) | A1, X1 = ((uint64_t)A1 << 32) | A2;  // symbols 0..31, 16..47
    const uint64_t R0 = rev2_64(~X0), R1 = rev2_64(~X1);  // complement, symbol 0 (16) at the LSB
    uint32_t h[NP];
#pragma unroll
    for (int o = 0; o < NP; ++o) {
        const bool lo = o + Q <= 32;
        const int off = lo ? o : o - 16;
        const uint64_t X = lo ? X0 : X1, R = lo ? R0 : R1;
        const uint32_t f = (uint32_t)(X >> (64 - 2 * (off + Q))) & MQ;
        const uint32_t r = (uint32_t)(R >> (2 * off)) & MQ;
        h[o] = min(f, r) * 0x9E3779B1u;
    }
    // van Herk / Gil-Werman: window t covers positions [t, t + W2); t <= U < W2, so it is the
    // suffix minimum of block [0, W2) at t and the prefix minimum of [W2, t + W2 - 1]
#pragma unroll
    for (int o = W2 - 2; o >= 0; --o) h[o] = min(h[o], h[o + 1]);
#pragma unroll
    for (int o = W2 + 1; o < NP; ++o) h[o] = min(h[o], h[o - 1]);
#pragma unroll
    for (int t = 0; t <= SS_U; ++t) {
        const uint32_t sub = t == 0 ? h[0] : min(h[t], h[W2 + t - 1]);
        D[t] = (uint32_t)(((uint64_t)fmix32(sub) * nd) >> 32);
    }
}

template <int KK>
__global__ void __launch_bounds__(SS_NT, 2) k_subsplit(const uint32_t* __restrict__ bins, const Piece* __restrict__ pieces,
                                                       uint64_t n_pieces, const SSBin* __restrict__ sbins,
                                                       uint32_t* __restrict__ cur, uint32_t* __restrict__ cur_w,
                                                       uint32_t* __restrict__ btab, uint4* __restrict__ pool,
                                                       uint64_t xbase, uint64_t n_blocks, uint4* __restrict__ ovf,
                                                       uint64_t ovf_cap, unsigned long long* __restrict__ ctr) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint4* stage = reinterpret_cast<uint4*>(sm + SS_OFF_STAGE);
    uint32_t* RB = reinterpret_cast<uint32_t*>(sm + SS_OFF_RB);
    unsigned long long* smask = reinterpret_cast<unsigned long long*>(sm + SS_OFF_MASK);
    uint32_t* rinfo = reinterpret_cast<uint32_t*>(sm + SS_OFF_RINFO);  // first unit | n << 16
    uint32_t* wpre = reinterpret_cast<uint32_t*>(sm + SS_OFF_WPRE);    // first window (piece-relative)
    uint16_t* umap = reinterpret_cast<uint16_t*>(sm + SS_OFF_UMAP);
    uint8_t* digs = sm + SS_OFF_DIGS;                                  // digit of every start window
    uint32_t* hs = reinterpret_cast<uint32_t*>(sm + SS_OFF_DTAB);      // sub-records per digit
    uint32_t* hw = hs + SS_DMAX;   // windows per digit
    uint32_t* gst = hw + SS_DMAX;  // first position of the piece's run in the digit
    uint32_t* lof = gst + SS_DMAX; // run start in the stage
    uint32_t* lc = lof + SS_DMAX;  // stage cursor
    uint32_t* ovb = lc + SS_DMAX;  // first overflow slot of the run's part beyond the block table
    uint32_t* bids = reinterpret_cast<uint32_t*>(sm + SS_OFF_BIDS);  // [d][SS_BPR] extra pool block ids (+1)
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + SS_OFF_MBAR);
    __shared__ uint32_t wsumA[SS_NT / 32], wsumB[SS_NT / 32];
    const int tid = threadIdx.x;
    const uint32_t R = gridDim.x, r = blockIdx.x;
    const uint64_t p0 = (uint64_t)r * n_pieces / R, p1 = (uint64_t)(r + 1) * n_pieces / R;
    if (p0 >= p1) return;
    for (int d = tid; d < SS_DMAX; d += SS_NT) hs[d] = hw[d] = 0;
    if (tid == 0) {
        mbar_init(mbar, 1);
        mbar_init(mbar + 1, 1);
        mbar_init_fence();
    }
    __syncthreads();
    auto issue = [&](uint64_t p, int b) {
        const Piece pc = pieces[p];
        const uint32_t bytes = pc.nrec * 16;
        mbar_expect_tx(mbar + b, bytes);
        tma_load_1d_hint(RB + b * SS_RBW, bins + pc.rec_begin * 4, bytes, mbar + b, l2_policy_evict_first());
    };
    if (tid == 0) issue(p0, 0);
    bool bulk_pending = false;
    Piece pnext = pieces[p0];
    for (uint64_t p = p0; p < p1; ++p) {
        const uint32_t it = (uint32_t)(p - p0);
        const int b = it & 1;
        if (tid == 0 && p + 1 < p1) {
            fence_proxy_async_smem();  // buffer b^1 was released by the previous iteration's barriers
            issue(p + 1, b ^ 1);
        }
        const Piece pc = pnext;
        if (p + 1 < p1) pnext = pieces[p + 1];
        const SSBin sb = sbins[pc.lbin];
        const uint32_t nd = sb.nd;
        mbar_wait(mbar + b, (it >> 1) & 1);
        const uint32_t* Rp = RB + b * SS_RBW;
        // ---- unit and window maps of the piece (one scan: windows << 16 | units)
        uint32_t n = 0, nu = 0;
        if ((uint32_t)tid < pc.nrec) {
            n = rec_nwin(Rp + tid * 4);
            nu = (n + SS_U - 1) / SS_U;
            smask[tid] = 0;
        }
        if (bulk_pending) {  // the previous piece's stage has been read by its bulk copies
            bulk_wait_read();
            bulk_pending = false;
        }
        uint32_t T;
        const uint32_t pre = block_excl_sum1<SS_NT, uint32_t>(nu | (n << 16), wsumA, &T);
        T &= 0xFFFFu;
        const uint32_t upre = pre & 0xFFFFu;
        for (uint32_t j = 0; j < nu; ++j) umap[upre + j] = (uint16_t)tid;
        if ((uint32_t)tid < pc.nrec) {
            rinfo[tid] = upre | (n << 16);
            wpre[tid] = pre >> 16;
        }
        __syncthreads();
        // ---- D: digits of every window, sub-record starts, digit histogram
        for (uint32_t w = tid; w < T; w += SS_NT) {
            const uint32_t l = umap[w];
            const uint32_t ri = rinfo[l];
            const int a = SS_U * (int)(w - (ri & 0xFFFFu));
            const int cnt = min(SS_U, (int)(ri >> 16) - a);
            uint32_t D[SS_U + 1];
            unit_digits<KK>(Rp + l * 4, a, nd, D);
            uint32_t m = 0;
            const uint32_t wp = wpre[l] + a;
#pragma unroll
            for (int i = 0; i < SS_U; ++i) {
                if (i < cnt && (a + i == 0 || D[i + 1] != D[i])) {
                    m |= 1u << i;
                    atomicAdd(&hs[D[i + 1]], 1u);
                    digs[wp + i] = (uint8_t)D[i + 1];
                }
            }
            if (m) atomicOr(&smask[l], (unsigned long long)m << a);
        }
        __syncthreads();
        // ---- R: one reservation per digit: positions [g, g + c) of the digit -- its region,
        // then extra pool blocks (claimed by CAS in the digit's table), then the overflow list
        const uint32_t rc = sb.rc, capd = rc + (uint32_t)SS_MAXB * SS_BLK;
        uint4* region0 = pool + sb.rbase;
        uint32_t c = 0, g = 0;
        if ((uint32_t)tid < nd) {
            c = hs[tid];
            hs[tid] = 0;  // ready for the next piece
            if (c) {
                const uint32_t dg = sb.dbase + tid;
                g = atomicAdd(&cur[dg], c);
                const uint32_t e = g + c;
                if (e > capd) {
                    const uint32_t lo = g > capd ? g : capd;
                    ovb[tid] = (uint32_t)atomicAdd(&ctr[1], (unsigned long long)(e - lo));
                }
                if (e > rc && g < capd) {
                    const uint32_t x0 = (g > rc ? g : rc) - rc;
                    const uint32_t b0 = x0 / SS_BLK, b1 = min((e - 1 - rc) / SS_BLK, (uint32_t)SS_MAXB - 1);
                    for (uint32_t bi = b0; bi <= b1; ++bi) {
                        uint32_t* slot = btab + (uint64_t)dg * SS_MAXB + bi;
                        uint32_t id = *reinterpret_cast<volatile uint32_t*>(slot);
                        if (id == 0) {
                            const uint32_t nb = (uint32_t)atomicAdd(&ctr[0], 1ull);
                            const uint32_t old = atomicCAS(slot, 0u, nb + 1);
                            id = old ? old : nb + 1;  // a block lost to a concurrent claim stays unused
                        }
                        if (bi - b0 < (uint32_t)SS_BPR) bids[tid * SS_BPR + (bi - b0)] = id;
                    }
                }
            }
            gst[tid] = g;
        }
        uint32_t npk;
        const uint32_t P = block_excl_sum1<SS_NT, uint32_t>((uint32_t)tid < nd ? c : 0u, wsumB, &npk);
        if ((uint32_t)tid < nd) lof[tid] = lc[tid] = P;
        __syncthreads();
        const bool staged = npk <= (uint32_t)SS_STAGE;
        // address of position gi of digit d (unstaged path), nullptr if dropped (pool too small)
        auto slot_ptr = [&](uint32_t d, uint32_t gi) -> uint4* {
            if (gi < rc) return region0 + (uint64_t)d * rc + gi;
            if (gi < capd) {
                const uint32_t id = __ldcg(btab + (uint64_t)(sb.dbase + d) * SS_MAXB + (gi - rc) / SS_BLK);
                return (id != 0 && id - 1 < n_blocks) ? pool + xbase + (uint64_t)(id - 1) * SS_BLK + (gi - rc) % SS_BLK
                                                      : nullptr;
            }
            const uint32_t lo = gst[d] > capd ? gst[d] : capd;
            const uint64_t o = (uint64_t)ovb[d] + (gi - lo);
            return o < ovf_cap ? ovf + o : nullptr;
        };
        // ---- E: every start builds its sub-record (bin record format) and places it
        for (uint32_t w = tid; w < T; w += SS_NT) {
            const uint32_t l = umap[w];
            const uint32_t ri = rinfo[l];
            const int a = SS_U * (int)(w - (ri & 0xFFFFu));
            const int nrec_w = (int)(ri >> 16);
            const uint64_t mk = smask[l];
            const uint32_t* rec = Rp + l * 4;
            uint32_t m = (uint32_t)(mk >> a) & 0xFFu;
            while (m) {
                const int v = a + __ffs(m) - 1;
                m &= m - 1;
                const uint64_t rest = v + 1 < 64 ? (mk >> (v + 1)) : 0ull;
                const int len = rest ? __ffsll((long long)rest) : nrec_w - v;
                const uint32_t d = digs[wpre[l] + v];
                atomicAdd(&hw[d], (uint32_t)len);
                const int bb = 8 + 2 * v;
                const uint4 sr = make_uint4(((uint32_t)len << 24) | (bits32_be(rec, bb) >> 8), bits32_be(rec, bb + 24),
                                            bits32_be(rec, bb + 56), bits32_be(rec, bb + 88));
                const uint32_t q = atomicAdd(&lc[d], 1u);
                if (staged) {
                    stage[q] = sr;
                } else {
                    uint4* dst = slot_ptr(d, gst[d] + (q - lof[d]));
                    if (dst) *dst = sr;
                }
            }
        }
        if (staged) fence_proxy_async_smem();  // stage writes -> the bulk copies
        __syncthreads();
        // ---- W: every digit's run leaves by bulk copies: its region part, one per extra
        // pool block it touches, single stores for the overflow list
        if ((uint32_t)tid < nd && hw[tid]) {
            atomicAdd(&cur_w[sb.dbase + tid], hw[tid]);
            hw[tid] = 0;
        }
        if (staged && (uint32_t)tid < nd) {
            const uint32_t s0 = lof[tid], cn = lc[tid] - s0, g0 = gst[tid];
            uint32_t i = 0;
            if (g0 < rc && cn) {
                const uint32_t m = min(cn, rc - g0);
                tma_store_1d(region0 + (uint64_t)tid * rc + g0, stage + s0, m * 16u);
                bulk_pending = true;
                i = m;
            }
            const uint32_t bfirst = (g0 > rc ? g0 : rc) - rc;
            while (i < cn) {
                const uint32_t gi = g0 + i;
                if (gi >= capd) {  // beyond the block table: the overflow list
                    const uint32_t lo = g0 > capd ? g0 : capd;
                    for (; i < cn; ++i) {
                        const uint64_t o = (uint64_t)ovb[tid] + (g0 + i - lo);
                        if (o < ovf_cap) ovf[o] = stage[s0 + i];
                    }
                    break;
                }
                const uint32_t x = gi - rc;
                const uint32_t bi = x / SS_BLK - bfirst / SS_BLK;
                const uint32_t m = min(cn - i, (uint32_t)SS_BLK - x % SS_BLK);
                const uint32_t id = bids[tid * SS_BPR + bi];
                if (id != 0 && id - 1 < n_blocks) {
                    tma_store_1d(pool + xbase + (uint64_t)(id - 1) * SS_BLK + x % SS_BLK, stage + s0 + i, m * 16u);
                    bulk_pending = true;
                }
                i += m;
            }
            if (bulk_pending) bulk_commit();
        }
    }
    if (bulk_pending) bulk_wait_all();
}

// ---------------------------------------------------------------- counting
constexpr int SC_NT = 1024, SC_NW = SC_NT / 32;
constexpr int SC_SLOTS = 16384;
constexpr size_t SC_OFF_C = (size_t)SC_SLOTS * 8;
constexpr size_t SC_WBW = 32 * 4 + 8;                                    // words per warp buffer
constexpr size_t SC_OFF_WB = SC_OFF_C + (size_t)SC_SLOTS * 4;            // per warp: 32 sub-records (+ pad)
constexpr size_t SC_OFF_BT = SC_OFF_WB + (size_t)SC_NW * SC_WBW * 4;
constexpr size_t SC_SMEM = SC_OFF_BT + (size_t)SS_MAXB * 4;
static_assert(SC_SMEM <= 227 * 1024, "fits one CTA per SM");
constexpr int SC_MAXLG = 20;  // log2 of the most rounds a digit is counted in

// the round of a key when a digit is counted in R = 2^j rounds: the top j bits of a hash
// independent of slot_hash (nested: round r of R = rounds 2r, 2r+1 of 2R)
__device__ __forceinline__ uint32_t round_of(uint64_t key, int lgR) {
    const uint32_t h = (uint32_t)((key * 0xD6E8FEB86659FD93ull) >> 32);
    return lgR ? h >> (32 - lgR) : 0u;
}

// Sub-record slot i of a digit: its region [rb, rb + rc), then pool blocks from its table.
__device__ __forceinline__ uint64_t sub_slot(uint32_t i, uint64_t rb, uint32_t rc, const uint32_t* BT, uint64_t xbase) {
    return i < rc ? rb + i : xbase + (uint64_t)BT[(i - rc) / SS_BLK] * SS_BLK + (i - rc) % SS_BLK;
}

// Per digit: its region's first slot (dinfo, as two words) and size (drc); one thread per bin.
__global__ void k_sub_digits(const SSBin* __restrict__ sbins, uint32_t n_bins, uint2* __restrict__ dinfo,
                             uint32_t* __restrict__ drc) {
    const uint32_t b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= n_bins) return;
    const SSBin sb = sbins[b];
    for (uint32_t i = 0; i < sb.nd; ++i) {
        const uint64_t rb = sb.rbase + (uint64_t)i * sb.rc;
        dinfo[sb.dbase + i] = make_uint2((uint32_t)rb, (uint32_t)(rb >> 32));
        drc[sb.dbase + i] = sb.rc;
    }
}

template <bool CANON>
__global__ void __launch_bounds__(SC_NT, 1) k_subcount(const uint4* __restrict__ pool, uint64_t xbase,
                                                       const uint2* __restrict__ dinfo, const uint32_t* __restrict__ drc,
                                                       const uint32_t* __restrict__ cur, const uint32_t* __restrict__ cur_w,
                                                       const uint32_t* __restrict__ btab, uint32_t n_digits, int k,
                                                       uint32_t ci, uint32_t cx, uint64_t* sk, uint32_t* sc,
                                                       unsigned long long* gstats, uint32_t* __restrict__ fb_list,
                                                       unsigned long long* __restrict__ fb_ctr) {
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* T = reinterpret_cast<uint64_t*>(smem);
    uint32_t* C = reinterpret_cast<uint32_t*>(smem + SC_OFF_C);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, t = threadIdx.x;
    uint32_t* WB = reinterpret_cast<uint32_t*>(smem + SC_OFF_WB) + warp * SC_WBW;
    uint32_t* BT = reinterpret_cast<uint32_t*>(smem + SC_OFF_BT);
    __shared__ int ovf;
    __shared__ uint32_t bctr;
    __shared__ uint64_t s_rb;
    __shared__ uint32_t s_rc, s_n, s_nw;
    const uint32_t ltm = lanemask_lt();
    constexpr uint64_t E = ~0ull;
    for (int i = t; i < SC_SLOTS; i += SC_NT) {
        T[i] = E;
        C[i] = 0;
    }
    if (t == 0) ovf = 0;
    uint32_t uniq = 0, below = 0, above = 0;
    // thread 0 fetches the next digit's (region, counts) while the current one is counted
    auto fetch = [&](uint32_t d, uint64_t& rb, uint32_t& rc, uint32_t& n, uint32_t& nw) {
        if (d < n_digits) {
            const uint2 x = dinfo[d];
            rb = ((uint64_t)x.y << 32) | x.x;
            rc = drc[d];
            n = cur[d];
            nw = cur_w[d];
        }
    };
    uint64_t f_rb = 0;
    uint32_t f_rc = 0, f_n = 0, f_nw = 0;
    if (t == 0) fetch(blockIdx.x, f_rb, f_rc, f_n, f_nw);
    for (uint32_t d = blockIdx.x; d < n_digits; d += gridDim.x) {
        __syncthreads();  // the previous digit is over (BT, s_*, bctr reused)
        if (t == 0) {
            s_rb = f_rb;
            s_rc = f_rc;
            s_n = f_n;
            s_nw = f_nw;
            fetch(d + gridDim.x, f_rb, f_rc, f_n, f_nw);
        }
        __syncthreads();
        const uint32_t n = s_n, nw = s_nw, rc = s_rc;
        const uint64_t rb = s_rb;
        if (n == 0) continue;
        if (n > rc + (uint32_t)SS_MAXB * SS_BLK) {  // beyond the block table: the whole digit takes the fallback
            if (t == 0) fb_list[atomicAdd(fb_ctr, 1ull)] = d;
            continue;
        }
        const uint32_t nx = n > rc ? (n - rc + SS_BLK - 1) / SS_BLK : 0u;
        if (t < (int)nx) BT[t] = btab[(uint64_t)d * SS_MAXB + t] - 1;
        int lgR = 0;
        uint32_t r = 0;
        bool failed = false;
        for (;;) {
            const uint32_t want = min((uint32_t)SC_SLOTS, (nw >> lgR) + (nw >> lgR) / 3 + 64);
            int lg = 6;
            while ((1u << lg) < want) ++lg;
            const int TS = 1 << lg;
            if (t == 0) bctr = 0;
            __syncthreads();
            // ---- stream the digit: warps claim batches of 32 sub-records; lane = window
            bool ok = true;
            const uint32_t nb32 = (n + 31) / 32;
            auto claim = [&]() {
                uint32_t b = 0;
                if (lane == 0) b = atomicAdd(&bctr, 1u);
                return __shfl_sync(0xffffffffu, b, 0);
            };
            auto load = [&](uint32_t bt) {
                const uint32_t i = bt * 32 + lane;
                uint4 v = make_uint4(0, 0, 0, 0);
                if (bt < nb32 && i < n) v = __ldcs(pool + sub_slot(i, rb, rc, BT, xbase));
                return v;
            };
            uint32_t bt = claim();
            uint4 v = load(bt);
            while (bt < nb32) {
                const uint32_t bn = claim();
                const uint4 vn = load(bn);
                const uint32_t m = v.x >> 24;
                const uint32_t inc = warp_incl_sum(m);
                const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31), pre = inc - m;
                __syncwarp();  // the previous batch is done with WB
                *reinterpret_cast<uint4*>(WB + lane * 4) = v;
                __syncwarp();
                for (uint32_t u0 = 0; u0 < tot; u0 += 32) {
                    const uint32_t u = u0 + lane;
                    // owner: the last lane whose first window is <= u (binary search over pre)
                    uint32_t l = 0;
#pragma unroll
                    for (int st = 16; st >= 1; st >>= 1) {
                        const uint32_t pc = __shfl_sync(0xffffffffu, pre, l + st);
                        if (pc <= u) l += st;
                    }
                    const uint32_t pl = __shfl_sync(0xffffffffu, pre, l);
                    if (u < tot) {
                        const uint64_t key = window_key<uint64_t>(WB + l * 4, (int)(u - pl), k, CANON);
                        if (lgR == 0 || round_of(key, lgR) == r) ok &= table_insert_bounded<uint64_t>(T, C, lg, key);
                    }
                }
                bt = bn;
                v = vn;
            }
            if (!ok) ovf = 1;
            __syncthreads();
            if (ovf) {
                // too many distinct keys for the table: drop the partial counts of this round,
                // count the rest of the digit in twice as many rounds
                if (t == 0 && lgR == 0) atomicAdd(&gstats[GS_SUB_OVF], 1ull);
                for (int s = t; s < TS; s += SC_NT) {
                    T[s] = E;
                    C[s] = 0;
                }
                __syncthreads();
                if (t == 0) ovf = 0;
                ++lgR;
                r *= 2;
                if (lgR > SC_MAXLG) {  // a hash range of 2^-20 of a digit above the table: not data
                    failed = true;
                    break;
                }
                continue;
            }
            uint32_t keep = 0;
            for (int s = t; s < TS; s += SC_NT) {
                const uint32_t c = C[s];
                if (c) {
                    ++uniq;
                    if (c < ci) ++below;
                    else if (c > cx) ++above;
                    else ++keep;
                }
            }
            keep = __reduce_add_sync(0xffffffffu, keep);
            unsigned long long o = 0;
            if (lane == 0 && keep) o = atomicAdd(&gstats[GS_SURV], (unsigned long long)keep);
            o = __shfl_sync(0xffffffffu, o, 0);
            for (int s = t; s < TS; s += SC_NT) {
                const uint32_t c = C[s];
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
            if (++r == (1u << lgR)) break;
            __syncthreads();  // the table is clear before the next round inserts
        }
        if (failed && t == 0) atomicExch(fb_ctr + 1, 1ull);  // reported as an internal error
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

template <int KK>
cudaError_t subsplit_t(const uint32_t* bins, const Piece* pieces, uint64_t n_pieces, const SSBin* sbins,
                       uint32_t* cur, uint32_t* cur_w, uint32_t* btab, uint4* pool, uint64_t xbase, uint64_t n_blocks,
                       uint4* ovf, uint64_t ovf_cap, unsigned long long* ctr, unsigned grid, cudaStream_t s) {
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_subsplit<KK>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SS_SMEM)))
        return e;
    k_subsplit<KK><<<grid, SS_NT, SS_SMEM, s>>>(bins, pieces, n_pieces, sbins, cur, cur_w, btab, pool, xbase, n_blocks,
                                               ovf, ovf_cap, ctr);
    return cudaGetLastError();
}

}  // namespace

int subsplit_piece_records(int k) {
    const int maxw = record_max_windows(k);
    return std::min({SS_REC, SS_WMAX / maxw, SS_UMAX / ((maxw + SS_U - 1) / SS_U)});
}

cudaError_t launch_subsplit(const uint32_t* bins, const Piece* pieces, uint64_t n_pieces, const SSBin* sbins, int k,
                            uint32_t* cur, uint32_t* cur_w, uint32_t* btab, void* pool, uint64_t xbase,
                            uint64_t n_blocks, void* ovf, uint64_t ovf_cap, unsigned long long* ctr, int n_ctas,
                            cudaStream_t s) {
    if (n_pieces == 0) return cudaSuccess;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(n_pieces, (uint64_t)n_ctas));
    uint4* P = (uint4*)pool;
    uint4* O = (uint4*)ovf;
    switch (k) {
#define SS_CASE(KV)                                                                                               \
    case KV:                                                                                                      \
        return subsplit_t<KV>(bins, pieces, n_pieces, sbins, cur, cur_w, btab, P, xbase, n_blocks, O, ovf_cap, ctr, \
                              grid, s);
        SS_CASE(22) SS_CASE(23) SS_CASE(24) SS_CASE(25) SS_CASE(26) SS_CASE(27)
        SS_CASE(28) SS_CASE(29) SS_CASE(30) SS_CASE(31) SS_CASE(32)
#undef SS_CASE
        default: return cudaErrorInvalidValue;
    }
}

cudaError_t launch_subcount(const void* pool, uint64_t xbase, const SSBin* sbins, uint32_t n_bins, uint2* dinfo,
                            uint32_t* drc, const uint32_t* cur, const uint32_t* cur_w, const uint32_t* btab, uint32_t n_digits, int k, int canonical,
                            uint32_t ci, uint32_t cx, uint64_t* surv_keys, uint32_t* surv_counts,
                            unsigned long long* gstats, uint32_t* fb_list, unsigned long long* fb_ctr, int n_sms,
                            cudaStream_t s) {
    if (n_digits == 0) return cudaSuccess;
    if (k < SS_KMIN || k > SS_KMAX) return cudaErrorInvalidValue;
    const unsigned grid = (unsigned)std::min<uint64_t>(n_digits, (uint64_t)std::max(1, n_sms));
    k_sub_digits<<<(n_bins + 255) / 256, 256, 0, s>>>(sbins, n_bins, dinfo, drc);
    cudaError_t e;
    if (canonical) {
        if ((e = cudaFuncSetAttribute(k_subcount<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SC_SMEM)))
            return e;
        k_subcount<true><<<grid, SC_NT, SC_SMEM, s>>>((const uint4*)pool, xbase, dinfo, drc, cur, cur_w, btab,
                                                      n_digits, k, ci, cx, surv_keys, surv_counts, gstats, fb_list,
                                                      fb_ctr);
    } else {
        if ((e = cudaFuncSetAttribute(k_subcount<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SC_SMEM)))
            return e;
        k_subcount<false><<<grid, SC_NT, SC_SMEM, s>>>((const uint4*)pool, xbase, dinfo, drc, cur, cur_w, btab,
                                                       n_digits, k, ci, cx, surv_keys, surv_counts, gstats, fb_list,
                                                       fb_ctr);
    }
    return cudaGetLastError();
}

}  // namespace kmc
