// k_distribute.cu -- phase 1 of KMC 2 on the B200 (Sec. 2.4 "distribution"):
// S1 encode + split at non-ACGT and read ends, S2 signatures, S3 super-k-mer cut,
// S4 histogram (pass 1) and S5 scatter of super-k-mer records into HBM bins.
//
// Warp-centric and persistent: every warp owns a stream of SEG = 512-window segments of
// the concatenated base stream (windows never cross read boundaries: reads are marked
// from read_offsets) and runs the whole of S1-S4 for a segment inside its own slice of
// shared memory, with __syncwarp between steps and no CTA-wide barrier:
//   A  ASCII (16-byte vectors) -> 2-bit codes, invalid-base bitmask
//   B  read starts -> bitmask (bad = invalid | read start)
//   C  canonical p-mer key of every position, computed directly from the packed bits
//      (fwd = a 2p-bit field, rc = complement with the 2-bit groups reversed), held in
//      registers (row r, lane l = position 32r + l)
//   D  sliding minimum over W = k-p+1 keys with warp shuffles (log-step doubling)
//   E  window signature = that minimum if the window is valid
//   F  super-k-mer runs (ballot bitmask + compacted run starts), histogram atomics, and
//      the records: appended to a temporary stream from per-warp reserved blocks (pass 1)
//      or written into their bins (recompute path)
#include <algorithm>

#include "kmc_device.cuh"
#include "kmc_internal.h"

namespace kmc {

namespace {

constexpr int SEG = P1_SEG;                   // window starts per warp segment
constexpr int HL = 16;                        // bases before the segment (window seg0-1, alignment)
constexpr int NBASE = HL + SEG + 64;          // local bases held (k <= 64 needs HL + SEG + 63)
static_assert(NBASE % 32 == 16, "the invalid mask's last half word is set explicitly");
constexpr int NPK = NBASE / 16 + 8;           // packed words (+ zero slack for record packing)
constexpr int NMW = NBASE / 32 + 4;           // bitmask words (+ slack for 3-word funnel reads)
constexpr int NKEY = SEG + 64;                // p-mer positions 15 .. 15 + SEG + W - 1 (W <= 64)
constexpr int NROW = NKEY / 32;               // register rows of 32 positions
constexpr int SG_WARPS = 8, SG_NT = 32 * SG_WARPS;
constexpr uint32_t INV = 0xFFFFFFFFu;
constexpr uint32_t TMP_BLK = 2048;            // temporary-stream records reserved per warp at a time

struct WarpSmem {
    uint32_t pk[2][NPK]; // 2-bit codes, 16 per word, MSB first (local base x: word x/16); two
                         // segments: runs carried over from the previous one are emitted with
                         // the next one's
    uint32_t inv[NMW];   // bit x: local base x is not A/C/G/T (or outside the stream)
    uint32_t bad[NMW];   // bit x: invalid, or a read starts at x
    uint32_t vwin[NMW];  // bit x: the k-mer window starting at local x is valid
    uint32_t vpm[NMW];   // bit x: the p-mer starting at local x is valid
    uint32_t ebits[SEG / 32 + 2];  // bit v: window v cannot continue a run (invalid / run start)
    // phase D: keys (KS, 18 * 32 positions) and block prefix minima (PS, + overrun slack);
    // phases F-G: signature of each run start (xs[0, SEG)) and run starts (xs[SEG, 2 SEG))
    alignas(16) uint32_t xs[NROW * 32 + NROW * 32 + 64];
    uint32_t pv[32], ps[32], pn[32];  // carried-over runs: first window, signature, windows
};
static_assert(NROW * 32 * 2 + 64 >= 2 * SEG, "run lists fit the phase-D scratch");
static_assert(NROW == 18, "the block minimum uses 32 lanes x 18 positions");

// A->0, C->1, G->2, T->3; lowercase folded; anything else invalid (R3).
// Per 4 bytes: c = byte & 0xDF (case fold); code = ((c >> 1) ^ (c >> 2)) & 3 is 0/1/2/3 for
// A/C/G/T; the byte is valid iff it equals the letter of its own code, looked up with one
// byte permute; the 4 codes are packed by one multiply (byte i lands at bits 6-2i).
// One 4-byte word: the packed 8 bits (first base in the top 2) and the invalid nibble.
__device__ __forceinline__ void encode4(uint32_t w, uint32_t& packed8, uint32_t& inv4) {
    const uint32_t c = w & 0xDFDFDFDFu;
    const uint32_t cd = ((c >> 1) ^ (c >> 2)) & 0x03030303u;         // per byte: A0 C1 G2 T3
    const uint32_t sx = (cd | (cd >> 4)) & 0x00FF00FFu;                // codes as nibbles 0,1 | 2,3
    const uint32_t sel = (sx | (sx >> 8)) & 0xFFFFu;
    const uint32_t diff = __byte_perm(0x54474341u, 0u, sel) ^ c;        // 0 where the byte is its letter
    const uint32_t bad = (((diff & 0x7F7F7F7Fu) + 0x7F7F7F7Fu) | diff) & 0x80808080u;  // bit 7: byte != 0
    packed8 = (cd * 0x40100401u) >> 24;
    inv4 = ((bad >> 7) * 0x01020408u) >> 24 & 0xFu;
}
__device__ __forceinline__ void encode16(const uint32_t (&wd)[4], uint32_t& packed, uint32_t& invbits) {
    packed = 0;
    invbits = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
        uint32_t p8, i4;
        encode4(wd[t], p8, i4);
        packed |= p8 << (24 - 8 * t);
        invbits |= i4 << (4 * t);
    }
}

// Lane w holds word w of a bitmask X (LSB-first; lanes past the mask hold 0, and the mask
// has at most 30 words, so the lanes a shuffle wraps around to hold 0 too).  Word w of "X
// shifted down by s" (bit x <- bit x + s): a compile-time s < 32 needs the next lane only,
// a run-time s < 64 the next two.
static_assert(NMW <= 30, "the wrapped lanes of a shuffle-down by 1 or 2 hold no mask word");
template <int SH>
__device__ __forceinline__ uint32_t shr_words_c(uint32_t x) {
    static_assert(SH > 0 && SH < 32, "one-lane shift");
    return __funnelshift_r(x, __shfl_down_sync(0xffffffffu, x, 1), SH);
}
__device__ __forceinline__ uint32_t shr_words(uint32_t x, int s) {
    const uint32_t x1 = __shfl_down_sync(0xffffffffu, x, 1), x2 = __shfl_down_sync(0xffffffffu, x, 2);
    return s < 32 ? __funnelshift_r(x, x1, s) : __funnelshift_r(x1, x2, s - 32);
}
// Bit x of word w (lane w) of R_L = AND of G over positions [x, x + L), for two run lengths at
// once (L1, L2 <= 63), from one doubling chain R_1, R_2, R_4, .. (R_2a = R_a & R_a >> a):
// R_L = R_a & (R_a >> (L - a)) for the largest power of two a <= L.
__device__ __forceinline__ void run_and2(uint32_t g, int L1, int L2, uint32_t& o1, uint32_t& o2) {
    const int need = max(L1, L2);
    uint32_t r[6];
    r[0] = g;
    r[1] = r[0] & shr_words_c<1>(r[0]);
    r[2] = r[1] & shr_words_c<2>(r[1]);
    r[3] = r[2] & shr_words_c<4>(r[2]);
    r[4] = need >= 16 ? r[3] & shr_words_c<8>(r[3]) : 0u;
    r[5] = need >= 32 ? r[4] & shr_words_c<16>(r[4]) : 0u;
    auto pick = [&](int i) {  // r[i] without dynamic register indexing
        return i == 0 ? r[0] : i == 1 ? r[1] : i == 2 ? r[2] : i == 3 ? r[3] : i == 4 ? r[4] : r[5];
    };
    auto run = [&](int L) -> uint32_t {
        if (L == 0) return 0xFFFFFFFFu;
        const int i = 31 - __clz(L), a = 1 << i;
        const uint32_t ra = pick(i);
        return a == L ? ra : (ra & shr_words(ra, L - a));
    };
    o1 = run(L1);
    o2 = run(L2);
}

__device__ __forceinline__ uint32_t rev2_32(uint32_t x) {  // reverse the order of the 2-bit groups
    x = __brev(x);
    return ((x >> 1) & 0x55555555u) | ((x & 0x55555555u) << 1);
}

__global__ void k_tile_reads(const uint64_t* __restrict__ offsets, uint64_t n_reads, uint64_t off0,
                             uint64_t n_tiles, uint64_t* __restrict__ tile_r_lo) {
    uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= n_tiles) return;
    // first r in [0, n_reads] with offsets[r] - off0 > left edge of segment t (its local 0)
    int64_t edge = (int64_t)(t * SEG) - HL;
    uint64_t lo = 0, hi = n_reads + 1;
    while (lo < hi) {
        uint64_t mid = (lo + hi) >> 1;
        if ((int64_t)(offsets[mid] - off0) > edge) hi = mid;
        else lo = mid + 1;
    }
    tile_r_lo[t] = lo;
}

// The same table from the reads' side: read r (0 <= r <= n_reads + 1) is the first read of
// every tile whose left edge e_t = t SEG - HL satisfies O[r-1] <= e_t < O[r] (O[r] = offsets[r]
// - off0, O[-1] = -inf, O[n_reads + 1] = +inf): exactly the binary search's answer.
__global__ void k_tile_reads_by_read(const uint64_t* __restrict__ offsets, uint64_t n_reads, uint64_t off0,
                                     uint64_t n_tiles, uint64_t* __restrict__ tile_r_lo) {
    const uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (r > n_reads + 1) return;
    // first tile: ceil((O[r-1] + HL) / SEG) (0 for r = 0); end: ceil((O[r] + HL) / SEG)
    const uint64_t t0 = r == 0 ? 0 : (offsets[r - 1] - off0 + HL + SEG - 1) / SEG;
    const uint64_t t1 = r == n_reads + 1 ? n_tiles : (offsets[r] - off0 + HL + SEG - 1) / SEG;
    for (uint64_t t = t0; t < t1 && t < n_tiles; ++t) tile_r_lo[t] = r;
}

// PC: the signature length as a compile-time constant (0: a.p at run time).  The p-mer keys
// (phase C) shift and mask by p; the instances for the common lengths fold those constants.
template <int MODE, int PC = 0, int KC = 0>
__global__ void __launch_bounds__(SG_NT, 4) k_sig(P1Args a, uint64_t n_segs) {
    extern __shared__ __align__(16) uint8_t p1_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    WarpSmem& S = reinterpret_cast<WarpSmem*>(p1_smem)[warp];
    const uint32_t ltm = lanemask_lt();
    const int64_t nb = (int64_t)a.n_bases;
    const int k = KC ? KC : a.k, p = PC ? PC : a.p, W = k - p + 1;  // (KC: with PC, the window length folds too)
    const int RW = record_words(k), maxw = record_max_windows(k);
    const uint32_t maxw_magic = ((1u << 20) + maxw - 1) / maxw;  // ceil(2^20 / maxw)
    const uint32_t RES = 1u << (2 * p);
    const int NK = SEG + W;  // p-mer positions y = 0..NK-1 (local 15 + y)

    uint32_t l_windows = 0, l_skm = 0, l_recs = 0, l_inv = 0;  // per lane (< 2^32: a lane sees < 2^32 bases)
    uint64_t blk_cur = 0, blk_end = 0;  // this warp's reserved temporary-stream slots
    bool tmp_ok = a.tmp_recs != nullptr;

    const uint64_t gw = (uint64_t)blockIdx.x * SG_WARPS + warp, nw = (uint64_t)gridDim.x * SG_WARPS;
    int npend = 0;      // runs of the previous segment waiting for a full round of 32 lanes
    uint32_t pbuf = 0;  // this segment's packed-base buffer
    // the sample pass (seg_step s > 1) visits every s-th segment
    const uint64_t step = a.seg_step > 1 ? a.seg_step : 1;
    const uint64_t n_iter = (n_segs + step - 1) / step;
    for (uint64_t it = gw; it < n_iter; it += nw, pbuf ^= 1u) {
        const uint64_t sg = it * step;
        uint32_t* PK = S.pk[pbuf];
        const uint32_t* PKprev = S.pk[pbuf ^ 1u];
        const int64_t seg0 = (int64_t)sg * SEG;
        const int64_t lbase = seg0 - HL;  // stream position of local base 0
        const uint64_t r_first = a.tile_r_lo[sg];
        // ---- A: load + encode
        {  // chunks 0..31: one 16-byte chunk per lane
            const int t = lane;
            const int64_t q = lbase + 16 * t;
            uint32_t wd[4];
            if (a.reads_aligned16 && q >= 0 && q + 16 <= nb) {
                const uint4 v = __ldcs(reinterpret_cast<const uint4*>(a.reads + q));
                wd[0] = v.x;
                wd[1] = v.y;
                wd[2] = v.z;
                wd[3] = v.w;
            } else {
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    uint32_t x = 0;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int64_t qq = q + 4 * u + j;
                        const uint32_t b = (qq >= 0 && qq < nb) ? a.reads[qq] : (uint32_t)'N';
                        x |= b << (8 * j);
                    }
                    wd[u] = x;
                }
            }
            uint32_t packed, invbits;
            encode16(wd, packed, invbits);
            PK[t] = packed;
            reinterpret_cast<uint16_t*>(S.inv)[t] = (uint16_t)invbits;
            if (t >= 1) {  // the segment's own bases: local [HL, HL + SEG) = chunks 1 .. SEG/16
                uint32_t m = invbits;
                if (q + 16 > nb) m &= (q >= nb) ? 0u : ((1u << (uint32_t)(nb - q)) - 1u);
                l_inv += __popc(m);
            }
        }
        {  // the tail chunks 32 .. NBASE/16 - 1: one 4-byte word per lane
            static_assert(SEG / 16 == 32 && NBASE / 16 - 32 <= 8, "tail chunks fit one word per lane");
            constexpr int NTW = 4 * (NBASE / 16 - 32);
            const int t = 32 + (lane >> 2), u = lane & 3;
            const int64_t q = lbase + 16 * t + 4 * u;
            uint32_t x = 0;
            if (lane < NTW) {
                if (a.reads_aligned16 && q >= 0 && q + 4 <= nb) {
                    x = __ldcs(reinterpret_cast<const unsigned int*>(a.reads + q));
                } else {
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int64_t qq = q + j;
                        const uint32_t b = (qq >= 0 && qq < nb) ? a.reads[qq] : (uint32_t)'N';
                        x |= b << (8 * j);
                    }
                }
            }
            uint32_t p8, i4;
            encode4(x, p8, i4);
            uint32_t iv = lane < NTW ? i4 << (4 * u) : 0u;
            iv |= __shfl_xor_sync(0xffffffffu, iv, 1);
            iv |= __shfl_xor_sync(0xffffffffu, iv, 2);
            if (lane < NTW) {
                reinterpret_cast<uint8_t*>(PK)[4 * t + 3 - u] = (uint8_t)p8;
                if (u == 0) reinterpret_cast<uint16_t*>(S.inv)[t] = (uint16_t)iv;
                if (t == SEG / 16) {  // the last chunk of the segment's own bases
                    uint32_t m = i4;
                    if (q + 4 > nb) m &= (q >= nb) ? 0u : ((1u << (uint32_t)(nb - q)) - 1u);
                    l_inv += __popc(m);
                }
            }
        }
        if (lane < NPK - NBASE / 16) PK[NBASE / 16 + lane] = 0;
        if (lane == 0) reinterpret_cast<uint16_t*>(S.inv)[NBASE / 16] = 0xFFFFu;  // NBASE = 16 mod 32
        __syncwarp();
        for (int w = lane; w < NMW; w += 32) {
            const uint32_t iv = w <= NBASE / 32 ? S.inv[w] : 0xFFFFFFFFu;
            S.inv[w] = iv;
            S.bad[w] = iv;
        }
        __syncwarp();
        // ---- B: read starts inside (lbase, lbase + NBASE)
        for (uint64_t rb = r_first;; rb += 32) {
            const uint64_t r = rb + lane;
            int64_t st = NBASE;
            if (r <= a.n_reads) {
                st = (int64_t)(a.offsets[r] - a.off0) - lbase;
                if (st < NBASE) atomicOr(&S.bad[st >> 5], 1u << (st & 31));
            }
            if (!__all_sync(0xffffffffu, st < NBASE)) break;
        }
        __syncwarp();
        // validity masks by doubling (lane = word): window x valid iff base x is valid and
        // no base in (x, x+k) is invalid or starts a read; p-mer likewise with p
        {
            const uint32_t g = lane < NMW ? ~S.bad[lane] : 0u;
            const uint32_t iv = lane < NMW ? S.inv[lane] : 0xFFFFFFFFu;
            uint32_t rw, rp;
            run_and2(g, k - 1, p - 1, rw, rp);
            const uint32_t vw = ~iv & shr_words_c<1>(rw);
            const uint32_t vp = ~iv & shr_words_c<1>(rp);
            if (lane < NMW) {
                S.vwin[lane] = vw;
                S.vpm[lane] = vp;
            }
        }
        __syncwarp();
        // ---- C: canonical p-mer keys at local 15 + y, in registers:
        //      lane l holds positions y = 18 l + o, o < 18 (NROW * 32 = 576 >= SEG + W).
        //      key = min(fwd, rc) if the p-mer is valid and allowed, else the reserved 4^p (R4).
        //      The lane's 32 symbols from its first position are one 64-bit field X (MSB
        //      first); its complement reversed, R, holds every reverse complement:
        //      rc(o) = (R >> 2o) mod 4^p.  Allowedness (R2) is evaluated for all positions
        //      at once on 2-bit-spaced indicator masks of the LSB-first stream Y = ~R:
        //      forward p-mer at o is excluded iff an AA pair starts in [o+1, o+p-2] or ACA
        //      starts at o; its reverse complement iff a TT pair starts in [o, o+p-3] or TGT
        //      starts at o+p-3.
        const int y0 = 18 * lane;
        uint32_t K[18];
        {
            const int j0 = 15 + y0;  // local base of position y0
            const int w0 = j0 >> 4, sh = 2 * (j0 & 15);
            const uint32_t W0 = PK[w0], W1 = PK[w0 + 1], W2 = PK[w0 + 2];
            const uint32_t sA = __funnelshift_l(W1, W0, sh), sB = __funnelshift_l(W2, W1, sh);  // X = sA:sB
            const uint32_t Rlo = rev2_32(~sA), Rhi = rev2_32(~sB);
            const uint32_t pvb = __funnelshift_r(S.vpm[j0 >> 5], S.vpm[(j0 >> 5) + 1], j0 & 31);
            uint64_t fbad = 0, rbad = 0;  // bit 2o: the forward / reverse p-mer at o is not allowed
            if (p >= 3 && a.rules) {
                constexpr uint64_t M5 = 0x5555555555555555ull;
                const uint64_t Y = ~(((uint64_t)Rhi << 32) | Rlo), y1 = Y >> 1;
                const uint64_t iA = ~(Y | y1) & M5, iT = Y & y1 & M5, iC = Y & ~y1 & M5, iG = ~Y & y1 & M5;
                uint64_t ua = iA & (iA >> 2), ut = iT & (iT >> 2);  // AA / TT pair starts
                const int L = p - 2;  // OR over [i, i + L) by doubling
                int A = 1;
                while (2 * A <= L) {
                    ua |= ua >> (2 * A);
                    ut |= ut >> (2 * A);
                    A *= 2;
                }
                ua |= ua >> (2 * (L - A));
                ut |= ut >> (2 * (L - A));
                fbad = (ua >> 2) | (iA & (iC >> 2) & (iA >> 4));
                rbad = ut | ((iT & (iG >> 2) & (iT >> 4)) >> (2 * (p - 3)));
            }
            {  // invalid p-mers (bit o of pvb clear) count as not allowed in both orientations
                uint64_t x = pvb & 0x3FFFFu;  // spread bit o to bit 2o
                x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
                x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
                x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
                x = (x | (x << 2)) & 0x3333333333333333ull;
                x = (x | (x << 1)) & 0x5555555555555555ull;
                const uint64_t nv = ~x & 0x5555555555555555ull;
                fbad |= nv;
                rbad |= nv;
            }
            const uint32_t mp = (uint32_t)(RES - 1);
#pragma unroll
            for (int o = 0; o < 18; ++o) {
                const uint32_t fwd = (o < 16 ? __funnelshift_l(sB, sA, 2 * o) : (sB << (2 * (o - 16)))) >> (32 - 2 * p);
                const uint32_t rc = (o < 16 ? __funnelshift_r(Rlo, Rhi, 2 * o) : (Rhi >> (2 * (o - 16)))) & mp;
                const bool fw = fwd <= rc;
                const uint32_t bad = (uint32_t)((fw ? fbad : rbad) >> (2 * o)) & 1u;
                K[o] = bad ? RES : (fw ? fwd : rc);
            }
        }
        // ---- D: sliding minimum over W keys: window y = min over keys [y, y + W)
        // ---- E: signature of window local 15 + y (y <= SEG), INV where the window is not
        //      valid (crosses a read start or holds a non-ACGT base); rows M[r] (lane l: y = 32 r + l)
        uint32_t* KS = S.xs;
        uint32_t M[NROW];
        if (W >= 19) {
            // van Herk / Gil-Werman over blocks of 18 positions.  W >= 19 means every window
            // leaves its own block: min = suffix min in the own block, minima of the blocks it
            // covers fully, prefix min of the block it ends in (read from PS).
            uint32_t* PS = S.xs + NROW * 32;
            uint32_t T = 0xFFFFFFFFu;
#pragma unroll
            for (int o = 0; o < 18; o += 2) {  // 64-bit: 9 l + o / 2 is conflict-free per half warp
                const uint32_t p0 = min(T, K[o]), p1 = min(p0, K[o + 1]);
                *reinterpret_cast<uint2*>(PS + y0 + o) = make_uint2(p0, p1);
                T = p1;
            }
#pragma unroll
            for (int o = 16; o >= 0; --o) K[o] = min(K[o], K[o + 1]);  // suffix minima
            const uint32_t T1 = __shfl_sync(0xffffffffu, T, (lane + 1) & 31);
            const uint32_t T2 = min(T1, __shfl_sync(0xffffffffu, T, (lane + 2) & 31));
            const uint32_t T3 = min(T2, __shfl_sync(0xffffffffu, T, (lane + 3) & 31));
            // window i ends in block l + m, m = (i + W - 1) / 18 in {m0, m0 + 1}
            const int m0 = (W - 1) / 18, isplit = 18 * (m0 + 1) - (W - 1);
            const uint32_t midA = m0 == 1 ? 0xFFFFFFFFu : m0 == 2 ? T1 : T2;
            const uint32_t midB = m0 == 1 ? T1 : m0 == 2 ? T2 : T3;
            const int i0 = 15 + y0;  // window y0's local base
            const uint32_t vwb = __funnelshift_r(S.vwin[i0 >> 5], S.vwin[(i0 >> 5) + 1], i0 & 31);
            __syncwarp();
            const uint32_t* pe = PS + y0 + (W - 1);
#pragma unroll
            for (int o = 0; o < 18; o += 2) {
                uint32_t w0 = min(min(K[o], o < isplit ? midA : midB), pe[o]);
                uint32_t w1 = min(min(K[o + 1], o + 1 < isplit ? midA : midB), pe[o + 1]);
                w0 = ((vwb >> o) & 1u) ? w0 : INV;
                w1 = ((vwb >> (o + 1)) & 1u) ? w1 : INV;
                *reinterpret_cast<uint2*>(KS + y0 + o) = make_uint2(w0, w1);
            }
            __syncwarp();
#pragma unroll
            for (int r = 0; r <= SEG / 32; ++r) M[r] = KS[32 * r + lane];
        } else {
            // short windows: doubling with warp shuffles over rows; after the step with shift
            // s, M(y) = min over [y, y + 2s); [y, y + W) = two ranges of length A = 2^floor(log2 W)
#pragma unroll
            for (int o = 0; o < 18; o += 2)
                *reinterpret_cast<uint2*>(KS + y0 + o) = make_uint2(K[o], K[o + 1]);
            __syncwarp();
#pragma unroll
            for (int r = 0; r < NROW; ++r) M[r] = KS[32 * r + lane];
            auto shift_min = [&](int sft) {
                const int src = (lane + sft) & 31;
                const bool hi = lane + sft >= 32;
#pragma unroll
                for (int r = 0; r < NROW; ++r) {
                    const uint32_t a0 = __shfl_sync(0xffffffffu, M[r], src);
                    const uint32_t a1 = __shfl_sync(0xffffffffu, r + 1 < NROW ? M[r + 1] : 0xFFFFFFFFu, src);
                    M[r] = min(M[r], hi ? a1 : a0);
                }
            };
            int A = 1;
            while (2 * A <= W) {
                shift_min(A);
                A *= 2;
            }
            if (W > A) shift_min(W - A);  // W - A < A <= 16
#pragma unroll
            for (int r = 0; r <= SEG / 32; ++r) {
                const int i = 15 + 32 * r + lane;
                const bool ok = (S.vwin[i >> 5] >> (i & 31)) & 1u;
                M[r] = ok ? M[r] : INV;
            }
        }
        __syncwarp();
        // ---- F: super-k-mers = maximal runs of valid windows with equal signature
        //      (Fig. 1); records are additionally cut at the segment edge and into
        //      pieces of at most maxw windows.  Window v (= local y = v + 1) compares its
        //      signature with window v - 1's (y = v): one shuffle per row.
        uint32_t* list = S.xs + SEG;
        uint32_t* lsig = S.xs;
        int nstarts = 0;
#pragma unroll
        for (int r = 0; r < SEG / 32; ++r) {
            const int v = 32 * r + lane;
            const uint32_t s = __shfl_sync(0xffffffffu, lane == 0 ? M[r + 1] : M[r], (lane + 1) & 31);
            const uint32_t prev = M[r];
            if (MODE == P1_MODE_DEBUG) {
                if (seg0 + v < nb) a.dbg_sig[seg0 + v] = s;
                continue;
            }
            const bool valid = s != INV;
            const bool skm = valid && prev != s;
            const bool start = skm || (valid && v == 0);
            const uint32_t bE = __ballot_sync(0xffffffffu, !valid || start);
            const uint32_t bS = __ballot_sync(0xffffffffu, start);
            if (r == 0 && lane == 0) l_skm -= start && !skm;  // the segment-edge start is no new run
            if (lane == 0) S.ebits[r] = bE;
            if (start) {
                const int at = nstarts + __popc(bS & ltm);
                list[at] = (uint32_t)v;
                lsig[at] = s;
            }
            nstarts += __popc(bS);
        }
        if (MODE == P1_MODE_DEBUG) continue;
        if (lane == 0) {
            S.ebits[SEG / 32] = 1u;  // sentinel: the segment edge ends every run
            l_skm += nstarts;        // starts that are super-k-mer starts (the edge one corrected above)
        }
        __syncwarp();
        // G: records of the runs, 32 runs per round.  The runs of this segment follow the ones
        // carried over from the previous segment; only full rounds are emitted, and the rest
        // (< 32 runs of this segment) wait for the next segment -- a segment holds ~37 runs,
        // so a second round per segment would run mostly idle.  The last segment of the warp
        // (or one whose runs do not fill a round together with the carried ones) emits all.
        auto run_windows = [&](int v) {  // distance from window v to the next end mark
            const int pos = v + 1;
            int wd = pos >> 5;
            uint32_t bits = S.ebits[wd] & (0xFFFFFFFFu << (pos & 31));
            while (bits == 0) bits = S.ebits[++wd];
            return (wd * 32 + __ffs(bits) - 1) - v;
        };
        const int total = npend + nstarts;
        int emit_end = (it + nw >= n_iter) ? total : (total / 32) * 32;
        if (emit_end < npend) emit_end = total;
        for (int i0 = 0; i0 < emit_end; i0 += 32) {
            const int idx = i0 + lane;
            uint32_t s = INV;
            int v = 0, n = 0, nrec = 0;
            const uint32_t* pkb = PK;
            uint4 dd = make_uint4(0u, 0xFFFFFFFFu, 0u, 0u);
            if (idx < emit_end) {
                if (idx < npend) {
                    v = (int)S.pv[idx];
                    s = S.ps[idx];
                    n = (int)S.pn[idx];
                    pkb = PKprev;
                    if (MODE == P1_MODE_SCATTER && a.sig_dest) dd = a.sig_dest[s];
                } else {
                    v = (int)list[idx - npend];
                    s = lsig[idx - npend];
                    // the run's (bin, capacity, first slot) load is issued before the walk
                    // over the end marks, which hides its L2 latency
                    if (MODE == P1_MODE_SCATTER && a.sig_dest) dd = a.sig_dest[s];
                    n = run_windows(v);
                }
                nrec = (int)(((uint32_t)(n + maxw - 1) * maxw_magic) >> 20);  // exact: (n+maxw)*maxw < 2^20
                l_windows += n;
                l_recs += nrec;
            }
            if ((MODE == P1_MODE_HIST || (MODE == P1_MODE_SCATTER && a.scatter_hist)) && idx < emit_end) {
                atomicAdd(&a.hist_w[s], (unsigned long long)n);
                // (the sampled scatter's record counts per bin are its bins' fill counters)
                if (MODE == P1_MODE_HIST) atomicAdd(&a.hist_r[s], (uint32_t)nrec);
            }
            // slots: temporary stream (pass 1) from the warp's reserved block, or the bins
            uint64_t slot0 = 0;
            if (MODE == P1_MODE_HIST && tmp_ok) {
                const uint32_t inc = warp_incl_sum((uint32_t)nrec);
                const uint32_t tot = __shfl_sync(0xffffffffu, inc, 31);
                if (blk_cur + tot > blk_end) {
                    // close the current block (unused slots carry no signature) and reserve anew
                    for (uint64_t q = blk_cur + lane; q < blk_end; q += 32) a.tmp_sig[q] = INV;
                    unsigned long long nbase = 0;
                    if (lane == 0) nbase = atomicAdd(&a.gstats[GS_TMP_RECS], (unsigned long long)TMP_BLK);
                    nbase = __shfl_sync(0xffffffffu, nbase, 0);
                    blk_cur = nbase;
                    blk_end = nbase + TMP_BLK;
                    if (blk_end > a.tmp_cap) tmp_ok = false;  // overflow: the host recomputes (S5)
                }
                slot0 = blk_cur + inc - nrec;
                blk_cur += tot;
            }
            if (idx < emit_end && (MODE == P1_MODE_SCATTER || tmp_ok)) {
                const int j = v + n;
                uint32_t bin = 0, cap = 0xFFFFFFFFu, f0 = 0;
                uint64_t bbase = 0;
                if (MODE == P1_MODE_SCATTER) {
                    if (a.sig_dest) {  // (bin, capacity, first slot) in one load
                        bin = dd.x;
                        cap = dd.y;
                        bbase = ((uint64_t)dd.w << 32) | dd.z;
                    } else {
                        bin = a.sig2bin[s];
                        bbase = a.bin_rec_off[bin];
                    }
                }
                // a pass over a range of bins (inputs beyond HBM): other bins' records are skipped
                const bool skip = MODE == P1_MODE_SCATTER && (bin < a.bin_lo || bin >= a.bin_hi);
                if (MODE == P1_MODE_SCATTER && !skip) f0 = atomicAdd(&a.bin_fill[bin], (uint32_t)nrec);
                for (int ii = v; ii < j && !skip; ii += maxw) {
                    const int m = min(maxw, j - ii);
                    // record words: word 0 = m (8 bits) + symbols [0, 12); word u > 0 =
                    // symbols [12 + 16(u-1), 12 + 16u) -- from the packed segment by funnel shifts
                    const int b0 = HL + ii;  // local base of the piece's first window
                    uint32_t wd[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
                        if (u >= RW) break;
                        const int bb = b0 + (u == 0 ? 0 : 12 + 16 * (u - 1));
                        const uint32_t x = __funnelshift_l(pkb[(bb >> 4) + 1], pkb[bb >> 4], 2 * (bb & 15));
                        wd[u] = (u == 0) ? (((uint32_t)m << 24) | (x >> 8)) : x;
                    }
                    uint64_t slot;
                    uint32_t* dstb;
                    if (MODE == P1_MODE_SCATTER) {
                        const uint32_t f = f0++;
                        if (f >= cap) {  // beyond the sampled capacity
                            atomicAdd(&a.gstats[GS_P1_OVF], 1ull);
                            continue;
                        }
                        slot = bbase + f;
                        dstb = a.bins;
                    } else {
                        slot = slot0++;
                        dstb = a.tmp_recs;
                        a.tmp_sig[slot] = s;
                    }
                    uint4* dst = reinterpret_cast<uint4*>(dstb + slot * (uint64_t)RW);
                    dst[0] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
                    if (RW == 8) dst[1] = make_uint4(wd[4], wd[5], wd[6], wd[7]);
                }
            }
        }
        __syncwarp();
        // carry the rest (runs of this segment only: emit_end >= npend) to the next segment
        const int carry = total - emit_end;
        if (lane < carry) {
            const int jj = emit_end + lane - npend;
            const int v = (int)list[jj];
            S.pv[lane] = (uint32_t)v;
            S.ps[lane] = lsig[jj];
            S.pn[lane] = (uint32_t)run_windows(v);
        }
        npend = carry;
        __syncwarp();
    }
    if (MODE == P1_MODE_DEBUG) return;
    if (MODE == P1_MODE_HIST && tmp_ok)
        for (uint64_t q = blk_cur + lane; q < blk_end; q += 32) a.tmp_sig[q] = INV;
    // ---- per-warp statistics (one atomic per counter and warp)
    auto wsum64 = [](uint64_t v) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        return v;
    };
    const uint64_t tw = wsum64(l_windows), ts = wsum64(l_skm), tr = wsum64(l_recs), ti = wsum64(l_inv);
    if (lane == 0) {
        if (tw) atomicAdd(&a.gstats[GS_WINDOWS], (unsigned long long)tw);
        if (ts) atomicAdd(&a.gstats[GS_SUPERKMERS], (unsigned long long)ts);
        if (tr) atomicAdd(&a.gstats[GS_RECORDS], (unsigned long long)tr);
        if (ti) atomicAdd(&a.gstats[GS_INVALID], (unsigned long long)ti);
    }
}

// S5 from the temporary stream: the records are sorted by bin id with most-significant-digit
// passes of <= 8 bits (the bins are laid out in bin-id order, so bucket v of a pass starts
// at bin_rec_off[first bin of v] and the last pass writes the final bins).  Each CTA takes
// a tile of records (within one bucket of the previous pass), sorts it by its digit in
// shared memory and writes it as runs of consecutive records -- an unsorted scatter of
// 16-byte records into ~10^4-10^5 bins is bound by partial-sector writes.  Pass 1 reads the
// signature tags (INV = unused slot) and maps them to bins; later passes carry bin ids.
constexpr int RS_NT = 512;
template <int RW> struct RecTile { static constexpr int v = RW == 4 ? 2048 : 1024; };
template <int RW> constexpr size_t rec_scatter_smem() {
    return (size_t)RecTile<RW>::v * (RW * 4 + 4 + 1) + (3 * 256 + 64) * 4 + 64;
}

template <int RW, bool PEER>
__global__ void __launch_bounds__(RS_NT) k_rec_scatter(const uint32_t* __restrict__ in_recs,
                                                       const uint32_t* __restrict__ in_ids,
                                                       const uint32_t* __restrict__ sig2bin,
                                                       const RecTile2* __restrict__ tiles,
                                                       const uint64_t* __restrict__ n_tiles, int shift, int D,
                                                       unsigned long long* __restrict__ cursor,
                                                       uint32_t* __restrict__ out_recs, uint32_t* __restrict__ out_ids,
                                                       int out_orig_ids, uint32_t* const* __restrict__ peer_recs,
                                                       uint32_t* const* __restrict__ peer_ids) {
    constexpr int TI = RecTile<RW>::v, IPT = TI / RS_NT;
    using V = uint4;
    extern __shared__ __align__(16) uint8_t rsm[];
    V* srec = reinterpret_cast<V*>(rsm);  // TI records
    uint32_t* sid = reinterpret_cast<uint32_t*>(srec + TI * (RW / 4));
    uint32_t* lh = sid + TI;              // 256: counts, then local offsets
    unsigned long long* gb = reinterpret_cast<unsigned long long*>(lh + 256);  // 256 run bases
    uint32_t* wsum = reinterpret_cast<uint32_t*>(gb + 256);
    uint8_t* sd = reinterpret_cast<uint8_t*>(wsum + 64);
    __shared__ uint32_t s_tot;
    if (n_tiles && blockIdx.x >= *n_tiles) return;
    const RecTile2 t = tiles[blockIdx.x];
    const int nd = 1 << D;
    for (int d = threadIdx.x; d < 256; d += RS_NT) lh[d] = 0;
    __syncthreads();
    // all loads of the tile are issued before any is used (ids, records, then the bin lookups)
    V r0[IPT], r1[IPT];
    uint32_t id[IPT], bin[IPT], dr[IPT];
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
        const uint32_t i = threadIdx.x + u * RS_NT;
        id[u] = i < t.n ? __ldcs(in_ids + t.begin + i) : INV;
    }
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
        const uint32_t i = threadIdx.x + u * RS_NT;
        if (i < t.n) {  // slots tagged INV hold no record; loading them is harmless
            const V* src = reinterpret_cast<const V*>(in_recs + (t.begin + i) * (uint64_t)RW);
            r0[u] = __ldcs(src);
            if (RW == 8) r1[u] = __ldcs(src + 1);
        }
    }
#pragma unroll
    for (int u = 0; u < IPT; ++u) bin[u] = (sig2bin && id[u] != INV) ? sig2bin[id[u]] : id[u];
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
        dr[u] = INV;
        if (bin[u] != INV) {
            const uint32_t b = bin[u];
            if (out_orig_ids) bin[u] = id[u];
            const uint32_t d = (b >> shift) & (uint32_t)(nd - 1);
            dr[u] = (d << 16) | atomicAdd(&lh[d], 1u);  // rank < TI
        }
    }
    __syncthreads();
    {
        const uint32_t c = threadIdx.x < (unsigned)nd ? lh[threadIdx.x] : 0u;
        // the run reservation is issued first; its round trip overlaps the block scan
        const unsigned long long g =
            c ? atomicAdd(&cursor[((uint64_t)t.bucket << D) + threadIdx.x], (unsigned long long)c) : 0ull;
        uint32_t tot;
        const uint32_t ex = block_excl_sum<RS_NT, uint32_t>(c, wsum, &tot);
        if (threadIdx.x < (unsigned)nd) {
            gb[threadIdx.x] = g;
            lh[threadIdx.x] = ex;
        }
        if (threadIdx.x == 0) s_tot = tot;
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < IPT; ++u) {
        if (dr[u] == INV) continue;
        const uint32_t d = dr[u] >> 16, pos = lh[d] + (dr[u] & 0xFFFFu);
        srec[pos * (RW / 4)] = r0[u];
        if (RW == 8) srec[pos * 2 + 1] = r1[u];
        sid[pos] = bin[u];
        sd[pos] = (uint8_t)d;
    }
    __syncthreads();
    const uint32_t tot = s_tot;
    for (uint32_t i = threadIdx.x; i < tot; i += RS_NT) {
        const uint32_t d = sd[i];
        const uint64_t o = gb[d] + (i - lh[d]);
        // peer mode (fused exchange): digit d is a destination rank, its run goes straight into
        // that rank's receive buffers (mapped peer memory), cursor d counting in them
        uint32_t* orec = PEER ? peer_recs[d] : out_recs;
        uint32_t* oid = PEER ? peer_ids[d] : out_ids;
        V* dst = reinterpret_cast<V*>(orec + o * (uint64_t)RW);
        dst[0] = srec[i * (RW / 4)];
        if (RW == 8) dst[1] = srec[i * 2 + 1];
        if (oid) oid[o] = sid[i];
    }
}

// cursor[v] = first record of bucket v = bins [v << shift, (v+1) << shift)
__global__ void k_bucket_cursors(const uint64_t* __restrict__ bin_rec_off, uint64_t n_bins, uint64_t n_records,
                                 int shift, uint64_t n_buckets, unsigned long long* __restrict__ cursor) {
    const uint64_t v = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (v >= n_buckets) return;
    const uint64_t b = v << shift;
    cursor[v] = b < n_bins ? bin_rec_off[b] : n_records;
}

// Sharded counting helpers.  map2[s] = map_b[map_a[s]] (signature -> bin -> owner rank).
__global__ void k_compose_map(const uint32_t* __restrict__ map_a, const uint32_t* __restrict__ map_b, uint64_t n,
                              uint32_t* __restrict__ out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = map_b[map_a[i]];
}
// Records of the stream per owner rank (slots tagged INV are skipped).
__global__ void k_owner_count(const uint32_t* __restrict__ sig, uint64_t n, const uint32_t* __restrict__ sig2owner,
                              int world, unsigned long long* __restrict__ counts) {
    __shared__ uint32_t h[256];
    for (int d = threadIdx.x; d < world; d += blockDim.x) h[d] = 0;
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t sg = __ldcs(sig + i);
        if (sg != INV) atomicAdd(&h[sig2owner[sg]], 1u);
    }
    __syncthreads();
    for (int d = threadIdx.x; d < world; d += blockDim.x)
        if (h[d]) atomicAdd(&counts[d], (unsigned long long)h[d]);
}
__global__ void k_widen(const uint32_t* __restrict__ in, uint64_t n, uint64_t* __restrict__ out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = in[i];
}
__global__ void k_narrow(const uint64_t* __restrict__ in, uint64_t n, uint32_t* __restrict__ out) {
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = in[i] < 0xFFFFFFFFull ? (uint32_t)in[i] : 0xFFFFFFFFu;
}

__global__ void k_debug_allowed(int p, uint8_t* out) {
    uint64_t n = 1ull << (2 * p);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        out[i] = sig_allowed((uint32_t)i, p) ? 1 : 0;
}

template <int MODE, int PC, int KC = 0> cudaError_t launch_sig_p(const P1Args& a, uint64_t n_segs, cudaStream_t s) {
    const int sm = (int)(sizeof(WarpSmem) * SG_WARPS);
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_sig<MODE, PC, KC>, cudaFuncAttributeMaxDynamicSharedMemorySize, sm))) return e;
    int dev = 0, nsm = 148, per = 1;
    if ((e = cudaGetDevice(&dev))) return e;
    if ((e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev))) return e;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_sig<MODE, PC, KC>, SG_NT, sm))) return e;
    const uint64_t n_iter = a.seg_step > 1 ? (n_segs + a.seg_step - 1) / a.seg_step : n_segs;
    const uint64_t want = (n_iter + SG_WARPS - 1) / SG_WARPS;
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(want, (uint64_t)nsm * std::max(1, per)));
    k_sig<MODE, PC, KC><<<grid, SG_NT, sm, s>>>(a, n_segs);
    return cudaGetLastError();
}
template <int MODE> cudaError_t launch_sig_t(const P1Args& a, uint64_t n_segs, cudaStream_t s) {
#ifndef KMC_SIG_PSPEC
#define KMC_SIG_PSPEC 1
#endif
    if (KMC_SIG_PSPEC && MODE != P1_MODE_DEBUG) {
        // the (k, p) pairs of the paper's configurations fold the window length as well
#ifndef KMC_SIG_KSPEC
#define KMC_SIG_KSPEC 1
#endif
        if (KMC_SIG_KSPEC && a.k == 25 && a.p == 7) return launch_sig_p<MODE, 7, 25>(a, n_segs, s);
        if (KMC_SIG_KSPEC && a.k == 28 && a.p == 9) return launch_sig_p<MODE, 9, 28>(a, n_segs, s);
        if (KMC_SIG_KSPEC && a.k == 31 && a.p == 9) return launch_sig_p<MODE, 9, 31>(a, n_segs, s);
        if (KMC_SIG_KSPEC && a.k == 55 && a.p == 11) return launch_sig_p<MODE, 11, 55>(a, n_segs, s);
        switch (a.p) {  // the signature lengths of the paper's configurations (7, 9, 11)
            case 7: return launch_sig_p<MODE, 7>(a, n_segs, s);
            case 9: return launch_sig_p<MODE, 9>(a, n_segs, s);
            case 11: return launch_sig_p<MODE, 11>(a, n_segs, s);
            default: break;
        }
    }
    return launch_sig_p<MODE, 0>(a, n_segs, s);
}

}  // namespace

uint64_t p1_num_tiles(uint64_t n_bases) { return (n_bases + SEG - 1) / SEG; }

cudaError_t launch_tile_reads(const uint64_t* offsets, uint64_t n_reads, uint64_t off0, uint64_t n_tiles,
                              uint64_t* tile_r_lo, cudaStream_t s) {
    if (n_tiles == 0) return cudaSuccess;
    if (n_reads + 2 < (1ull << 31) * 256ull && n_reads > 0) {
        // by read: one coalesced pass over the offsets instead of a binary search per tile
        // (C4: 0.25 ms); tiles are zeroed first so that offsets that break the nondecreasing
        // contract leave every tile with a valid first read
        cudaError_t e = cudaMemsetAsync(tile_r_lo, 0, n_tiles * 8, s);
        if (e) return e;
        k_tile_reads_by_read<<<(unsigned)((n_reads + 2 + 255) / 256), 256, 0, s>>>(offsets, n_reads, off0, n_tiles,
                                                                                   tile_r_lo);
        return cudaGetLastError();
    }
    k_tile_reads<<<(unsigned)((n_tiles + 255) / 256), 256, 0, s>>>(offsets, n_reads, off0, n_tiles, tile_r_lo);
    return cudaGetLastError();
}

cudaError_t launch_p1(int mode, const P1Args& a, uint64_t n_tiles, cudaStream_t s) {
    if (n_tiles == 0) return cudaSuccess;
    if (mode == P1_MODE_HIST) return launch_sig_t<P1_MODE_HIST>(a, n_tiles, s);
    if (mode == P1_MODE_SCATTER) return launch_sig_t<P1_MODE_SCATTER>(a, n_tiles, s);
    return launch_sig_t<P1_MODE_DEBUG>(a, n_tiles, s);
}

size_t rec_tile_items(int k) { return record_words(k) == 4 ? RecTile<4>::v : RecTile<8>::v; }

cudaError_t launch_rec_scatter(int k, const uint32_t* in_recs, const uint32_t* in_ids, const uint32_t* sig2bin,
                               const RecTile2* tiles, uint64_t max_tiles, const uint64_t* n_tiles_dev, int shift,
                               int D, unsigned long long* cursor, uint32_t* out_recs, uint32_t* out_ids,
                               cudaStream_t s, int out_orig_ids, uint32_t* const* peer_recs,
                               uint32_t* const* peer_ids) {
    if (max_tiles == 0) return cudaSuccess;
    cudaError_t e;
    auto go = [&](auto kern, int sm) -> cudaError_t {
        cudaError_t e2;
        if ((e2 = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, sm))) return e2;
        kern<<<(unsigned)max_tiles, RS_NT, sm, s>>>(in_recs, in_ids, sig2bin, tiles, n_tiles_dev, shift, D, cursor,
                                                   out_recs, out_ids, out_orig_ids, peer_recs, peer_ids);
        return cudaSuccess;
    };
    const bool peer = peer_recs != nullptr;
    if (record_words(k) == 4)
        e = peer ? go(k_rec_scatter<4, true>, (int)rec_scatter_smem<4>())
                 : go(k_rec_scatter<4, false>, (int)rec_scatter_smem<4>());
    else
        e = peer ? go(k_rec_scatter<8, true>, (int)rec_scatter_smem<8>())
                 : go(k_rec_scatter<8, false>, (int)rec_scatter_smem<8>());
    if (e) return e;
    return cudaGetLastError();
}

cudaError_t launch_bucket_cursors(const uint64_t* bin_rec_off, uint64_t n_bins, uint64_t n_records, int shift,
                                  uint64_t n_buckets, unsigned long long* cursor, cudaStream_t s) {
    if (n_buckets == 0) return cudaSuccess;
    k_bucket_cursors<<<(unsigned)((n_buckets + 255) / 256), 256, 0, s>>>(bin_rec_off, n_bins, n_records, shift,
                                                                         n_buckets, cursor);
    return cudaGetLastError();
}

cudaError_t launch_compose_map(const uint32_t* map_a, const uint32_t* map_b, uint64_t n, uint32_t* out,
                               cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_compose_map<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 4096), 256, 0, s>>>(map_a, map_b, n, out);
    return cudaGetLastError();
}
cudaError_t launch_owner_count(const uint32_t* sig, uint64_t n, const uint32_t* sig2owner, int world,
                               unsigned long long* counts, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_owner_count<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 148 * 8), 256, 0, s>>>(sig, n, sig2owner, world,
                                                                                      counts);
    return cudaGetLastError();
}
cudaError_t launch_widen(const uint32_t* in, uint64_t n, uint64_t* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_widen<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 4096), 256, 0, s>>>(in, n, out);
    return cudaGetLastError();
}
cudaError_t launch_narrow(const uint64_t* in, uint64_t n, uint32_t* out, cudaStream_t s) {
    if (n == 0) return cudaSuccess;
    k_narrow<<<(unsigned)std::min<uint64_t>((n + 255) / 256, 4096), 256, 0, s>>>(in, n, out);
    return cudaGetLastError();
}

cudaError_t launch_debug_allowed(int p, uint8_t* out, cudaStream_t s) {
    k_debug_allowed<<<256, 256, 0, s>>>(p, out);
    return cudaGetLastError();
}

}  // namespace kmc
