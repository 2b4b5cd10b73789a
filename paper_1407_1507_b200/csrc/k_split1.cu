// k_split1.cu -- S6 + the split of S7 for the large bins in ONE pass (k <= 32).
//
// The paper sorts each bin after extracting its k-mers.  A bin
// above one CTA's shared memory is first split by a hash of the key into digits of about one
// counting chunk each (every copy of a k-mer shares its digit, so a digit is counted on its
// own; S9 orders the survivors globally).  Round 1 counted every (piece, digit) in a first
// pass, scanned the counts and re-expanded the bins in a second pass.  Here the digit regions
// are SIZED from the bin's window count instead: a bin of W windows gets nd = W / (chunk
// capacity) digits, digit = (h(key) x nd) >> 32, and each digit a region of rc ~ 1.25 W / nd
// key slots (hashed digits are near-uniform, but a k-mer of multiplicity m moves m keys at
// once, so repeat families can still overfill a digit).  One kernel per piece of 512 records (TMA, double-buffered):
//   A  expand every window (one lane per unit of <= 5 windows: one 64-bit field holds the
//      unit's symbols; keys min(fwd, rc)) and histogram the digits in SMEM;
//   R  reserve each digit's run in its region with one global atomic per (piece, digit);
//   B  expand again and place every key in a shared-memory stage grouped by digit (each run
//      starting at the parity of its global position);
//   W  every digit's run leaves by one TMA bulk copy (cp.async.bulk.global.shared::cta).
// Keys of a digit beyond its region go to an overflow list (one atomic reservation per
// (piece, digit)); such digits -- region part and overflow part -- are counted by the device
// radix-sort fallback, every other digit is one chunk of the SMEM hash count.
#include <algorithm>

#include "kmc_device.cuh"
#include "kmc_internal.h"

namespace kmc {

namespace {

constexpr int S1_NT = 512;
constexpr int S1_REC = 512;       // records per piece at most (the piece buffers)
constexpr int S1_UMAX = 7680;     // units per piece (umap entries)
constexpr int S1_STAGE = 8192;    // keys staged per piece (+ one spare slot per digit)
constexpr int S1_RBW = S1_REC * 4 + 8;
#ifndef KMC_S1_UNIT
#define KMC_S1_UNIT 5
#endif
constexpr int S1_UNIT = KMC_S1_UNIT;  // windows per expansion unit at most (k + unit - 1 <= 32 symbols)

__device__ __forceinline__ uint32_t s1_digit(uint64_t key, uint32_t nd) {
    const uint32_t h = (((uint32_t)(key >> 32) * 0x85EBCA6Bu) ^ (uint32_t)key) * 0x9E3779B1u;
    return (uint32_t)(((uint64_t)h * nd) >> 32);
}

constexpr size_t S1_OFF_STAGE = 0;
constexpr size_t S1_OFF_RB = S1_OFF_STAGE + (size_t)S1_STAGE * 8;
constexpr size_t S1_OFF_UMAP = S1_OFF_RB + 2 * (size_t)S1_RBW * 4;
constexpr size_t S1_OFF_RINFO = S1_OFF_UMAP + (size_t)S1_UMAX * 2;
constexpr size_t S1_OFF_DIG = S1_OFF_RINFO + (size_t)S1_REC * 4;  // h, gst, lof, lc, ovb (+ lim): S1_DMAX each
constexpr int S1_SOVF = 256;      // single-pass mode: keys beyond their digit's stage region
template <bool PAIRED> struct S1Lay {  // the paired layout keeps one more per-digit array (lim)
    static constexpr size_t SOVK = S1_OFF_DIG + (PAIRED ? 6 : 5) * (size_t)S1_DMAX * 4;
    static constexpr size_t SOVI = SOVK + (size_t)S1_SOVF * 8;
    static constexpr size_t MBAR = SOVI + (size_t)S1_SOVF * 4;
    static constexpr size_t SMEM = MBAR + 16 + 16;
    static_assert(S1_OFF_RB % 16 == 0 && MBAR % 8 == 0 && SOVK % 8 == 0, "alignment");
    static_assert(2 * SMEM + 2048 <= 228 * 1024, "two CTAs per SM");
};
static_assert(S1_DMAX <= 512, "digit in 9 bits of an overflow entry");
static_assert(S1_DMAX <= S1_NT, "one thread per digit");

// KC: k as a compile-time constant (0: the argument); the window extraction shifts by 2k
template <bool CANON, bool PAIRED, int KC = 0>
__global__ void __launch_bounds__(S1_NT, 2) k_split1(const uint32_t* __restrict__ bins, const Piece* __restrict__ pieces,
                                                     uint64_t n_pieces, const S1Bin* __restrict__ sbins, int k_arg,
                                                     int unit, uint32_t* __restrict__ cur, uint64_t* __restrict__ keys,
                                                     uint64_t* __restrict__ ovf, unsigned long long* __restrict__ ovf_ctr,
                                                     uint64_t ovf_cap, const unsigned long long* __restrict__ n_pieces_dev,
                                                     uint32_t* __restrict__ fail) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* stage = reinterpret_cast<uint64_t*>(sm + S1_OFF_STAGE);
    uint32_t* RB = reinterpret_cast<uint32_t*>(sm + S1_OFF_RB);
    uint16_t* umap = reinterpret_cast<uint16_t*>(sm + S1_OFF_UMAP);
    uint32_t* rinfo = reinterpret_cast<uint32_t*>(sm + S1_OFF_RINFO);
    uint32_t* h = reinterpret_cast<uint32_t*>(sm + S1_OFF_DIG);
    uint32_t* gst = h + S1_DMAX;   // run start of the digit in its region (this piece)
    uint32_t* lof = gst + S1_DMAX; // run start in the stage
    uint32_t* lc = lof + S1_DMAX;  // stage cursor
    uint32_t* ovb = lc + S1_DMAX;  // first overflow slot of the digit's keys beyond the region
    uint32_t* lim = ovb + S1_DMAX; // paired: positions of the digit below lim are in its region (this piece)
    uint64_t* sovk = reinterpret_cast<uint64_t*>(sm + S1Lay<PAIRED>::SOVK);  // single pass: stage-overflow keys
    uint32_t* sovi = reinterpret_cast<uint32_t*>(sm + S1Lay<PAIRED>::SOVI);  //   their digit | rank << 9
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + S1Lay<PAIRED>::MBAR);
    __shared__ uint32_t wsumA[S1_NT / 32], wsumB[S1_NT / 32];  // alternating scan scratch
    __shared__ uint32_t novf;
    const int tid = threadIdx.x;
    const int k = KC ? KC : k_arg;
    const int U = KC ? (S1_UNIT < 33 - KC ? S1_UNIT : 33 - KC) : unit;
    const uint32_t R = gridDim.x, r = blockIdx.x;
    if (n_pieces_dev) n_pieces = *n_pieces_dev;
    const uint64_t p0 = (uint64_t)r * n_pieces / R, p1 = (uint64_t)(r + 1) * n_pieces / R;
    if (p0 >= p1) return;
    for (int d = tid; d < S1_DMAX; d += S1_NT) h[d] = 0;
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
        tma_load_1d_hint(RB + b * S1_RBW, bins + pc.rec_begin * 4, bytes, mbar + b, l2_policy_evict_first());
    };
    if (tid == 0) issue(p0, 0);
    bool bulk_pending = false;
    uint32_t cur_bin = 0xFFFFFFFFu;
    S1Bin sb{};
    // A bin whose pieces all fall in this CTA's range is OWNED: thread d keeps digit d's cursor
    // in a register (no global atomic -- and no round trip -- between a piece's expansion and
    // its runs' bulk copies) and stores it when the bin ends.  Only the first and the last bin
    // of the range can be shared with a neighbouring CTA (pieces of a bin are consecutive);
    // those reserve with global atomics.  (Unpaired layout; the paired one always reserves.)
    const uint32_t first_lbin = pieces[p0].lbin, last_lbin = pieces[p1 - 1].lbin;
    const bool first_shared = p0 > 0 && pieces[p0 - 1].lbin == first_lbin;
    const bool last_shared = p1 < n_pieces && pieces[p1].lbin == last_lbin;
    bool owned = false;
    uint32_t my_cur = 0;
    uint32_t C1 = 0;  // single pass: stage slots of a digit (even), per bin
    const uint32_t umagic = (65536u + (uint32_t)U - 1) / (uint32_t)U;  // (x / U) = (x * umagic) >> 16, x < 64
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
        if (pc.lbin != cur_bin) {
            if (!PAIRED && owned && (uint32_t)tid < sb.nd) cur[sb.dbase + tid] = my_cur;
            cur_bin = pc.lbin;
            sb = sbins[cur_bin];
            C1 = sb.nd ? ((uint32_t)S1_STAGE / sb.nd) & ~1u : 0u;
            owned = !PAIRED && !(first_shared && cur_bin == first_lbin) && !(last_shared && cur_bin == last_lbin);
            if (owned && (uint32_t)tid < sb.nd) my_cur = cur[sb.dbase + tid];
        }
        const uint32_t nd = sb.nd;
        mbar_wait(mbar + b, (it >> 1) & 1);
        // ---- unit -> record map of the piece (block-balanced: every thread takes units in turn)
        const uint32_t* Rp = RB + b * S1_RBW;
        uint32_t n = 0, nu = 0;
        if ((uint32_t)tid < pc.nrec) {
            n = rec_nwin(Rp + tid * 4);
            nu = ((n + U - 1) * umagic) >> 16;
        }
        if (tid < S1_DMAX) lc[tid] = 0;  // (the same thread read it last: the previous piece's W)
        if (tid == 0) novf = 0;
        uint32_t T;
        const uint32_t pre2 = block_excl_sum1<S1_NT, uint32_t>(nu | (n << 16), wsumA, &T);
        const uint32_t NWIN = T >> 16, pre = pre2 & 0xFFFFu;
        T &= 0xFFFFu;
        for (uint32_t j = 0; j < nu; ++j) umap[pre + j] = (uint16_t)tid;
        if ((uint32_t)tid < pc.nrec) rinfo[tid] = pre | (n << 16);
        // the previous piece's bulk copies have read the stage before anyone writes it again:
        // their issuers wait here, so the copies overlap the block scan and the unit map
        if (bulk_pending) {
            bulk_wait_read();
            bulk_pending = false;
        }
        __syncthreads();
        // expansion of unit w: keys of windows first .. first + cnt - 1 of its record
        auto for_unit_keys = [&](uint32_t w, auto&& fn) {
            const uint32_t l = umap[w];
            const uint32_t ri = rinfo[l];
            const int first = U * (int)(w - (ri & 0xFFFFu));
            const int cnt = min(U, (int)(ri >> 16) - first);
            const uint64_t g = bits64_be(Rp + l * 4, 8 + 2 * first);
            const uint64_t rg = rev2_64(~g);
#pragma unroll
            for (int t = 0; t < S1_UNIT; ++t) {
                if (t < cnt) {
                    const uint64_t f = (g << (2 * t)) >> (64 - 2 * k);
                    const uint64_t rc = (rg << (64 - 2 * t - 2 * k)) >> (64 - 2 * k);
                    fn((CANON && rc < f) ? rc : f);
                }
            }
        };
        uint64_t* region = keys + sb.key_base;
        constexpr bool paired = PAIRED;  // (every bin of a paired launch has S1_PAIRED)
        // slot of position i (< rc) of digit d in the bin's regions (paired layout: odd digits
        // fill their pair's slots downwards), and the first slot of positions [g, g + m)
        auto slot = [&](uint32_t d, uint32_t i) -> uint64_t {
            return (paired && (d & 1u)) ? (uint64_t)(d + 1) * sb.rc - 1 - i : (uint64_t)d * sb.rc + i;
        };
        auto run_dst = [&](uint32_t d, uint32_t g, uint32_t m) -> uint64_t {
            return (paired && (d & 1u)) ? (uint64_t)(d + 1) * sb.rc - g - m : (uint64_t)d * sb.rc + g;
        };
        // place key at position i of digit d: its region, or the overflow list beyond it
        auto put = [&](uint32_t d, uint32_t i, uint64_t key) {
            if constexpr (PAIRED) {
                if (i < lim[d]) {
                    region[slot(d, i)] = key;
                } else {
                    const uint64_t o = (uint64_t)ovb[d] + (i - lim[d]);
                    if (o < ovf_cap) ovf[o] = key;
                }
            } else {
                if (i < sb.rc) {
                    region[(uint64_t)d * sb.rc + i] = key;
                } else {
                    const uint32_t lo = gst[d] > sb.rc ? gst[d] : sb.rc;
                    const uint64_t o = (uint64_t)ovb[d] + (i - lo);
                    if (o < ovf_cap) ovf[o] = key;
                }
            }
        };
        // reserve ce (even) positions for digit d's run of this piece: g = the first, returns how
        // many lie in the region (the rest go to the overflow list).  The digits of a pair share
        // its 2 rc slots through one 64-bit counter (the even digit in the low word): a run fits
        // while the two digits' counts stay within them; the first position of a digit that did
        // not fit is recorded (fail) for the chunk listing.
        auto reserve = [&](uint32_t d, uint32_t ce, uint32_t& g) -> uint32_t {
            uint32_t ra;
            if constexpr (PAIRED) {
                const uint32_t hi = d & 1u;
                const unsigned long long old = atomicAdd(
                    reinterpret_cast<unsigned long long*>(cur + sb.dbase + (d & ~1u)), (unsigned long long)ce << (32 * hi));
                g = (uint32_t)(old >> (32 * hi));
                const uint32_t pn = (uint32_t)(old >> (32 * (hi ^ 1u)));
                const uint32_t L = 2 * sb.rc > pn ? 2 * sb.rc - pn : 0u;
                ra = g >= L ? 0u : min(ce, L - g);
                if (ra < ce) atomicMin(&fail[sb.dbase + d], g + ra);
            } else {
                if (owned) {  // (d == this thread's digit)
                    g = my_cur;
                    my_cur += ce;
                } else {
                    g = atomicAdd(&cur[sb.dbase + d], ce);
                }
                ra = g >= sb.rc ? 0u : min(ce, sb.rc - g);
            }
            if (ra < ce) ovb[d] = (uint32_t)atomicAdd(ovf_ctr, (unsigned long long)(ce - ra));
            return ra;
        };
        // ---- single pass (pieces whose windows fill at most 4/5 of the stage): every key is
        //      expanded once and placed at its rank in its digit's share of the stage (keys
        //      beyond it: a short list with digit and rank); the digits' counts then reserve the
        //      regions -- always an even number of slots, the odd one out an EMPTY key that the
        //      counting skips, so every run starts 16-byte aligned -- and every digit's run leaves
        //      by one TMA bulk copy issued by its thread while the other threads move on
        if (NWIN + NWIN / 8 + 16 * nd <= (uint32_t)S1_STAGE) {
            for (uint32_t w = tid; w < T; w += S1_NT)
                for_unit_keys(w, [&](uint64_t key) {
                    const uint32_t d = s1_digit(key, nd);
                    const uint32_t q = atomicAdd(&lc[d], 1u);
                    if (q < C1) {
                        stage[d * C1 + q] = key;
                    } else {
                        const uint32_t o = atomicAdd(&novf, 1u);
                        if (o < (uint32_t)S1_SOVF) {
                            sovk[o] = key;
                            sovi[o] = d | (q << 9);
                        }
                    }
                });
            fence_proxy_async_smem();  // stage writes -> the bulk copies
            __syncthreads();
            const uint32_t nov = novf;  // (read before the next piece's thread 0 resets it)
            if (nov <= (uint32_t)S1_SOVF) {
                if ((uint32_t)tid < nd) {
                    const uint32_t c = lc[tid], ce = c + (c & 1u);
                    uint32_t g = 0, ra = 0;
                    if (c) ra = reserve(tid, ce, g);
                    gst[tid] = g;
                    if constexpr (PAIRED) lim[tid] = g + ra;
                    lof[tid] = c;
                    if (c) {
                        // the stage part (+ the pad slot when the run ends inside it), even-sized
                        uint32_t sn = c < C1 ? ce : C1;
                        if ((c & 1u) && c < C1) {
                            stage[tid * C1 + c] = ~0ull;
                            fence_proxy_async_smem();
                        }
                        const uint32_t in_reg = min(sn, ra);  // even: g, rc, ra even
                        if (in_reg) {
                            tma_store_1d(region + run_dst(tid, g, in_reg), stage + tid * C1, in_reg * 8u);
                            bulk_commit();
                            bulk_pending = true;
                        }
                        for (uint32_t i = in_reg; i < sn; ++i) put(tid, g + i, stage[tid * C1 + i]);
                        if ((c & 1u) && c >= C1) put(tid, g + c, ~0ull);  // the pad after the overflow part
                    }
                }
                if (nov) {
                    __syncthreads();  // gst / ovb of every digit for the overflow entries
                    for (uint32_t o = tid; o < nov; o += S1_NT) {
                        const uint32_t d = sovi[o] & 511u;
                        put(d, gst[d] + (sovi[o] >> 9), sovk[o]);
                    }
                }
                continue;  // (the next piece waits for its bulk copies before writing the stage)
            }
            // the overflow list itself overflowed: this piece takes the two-pass mode
            if ((uint32_t)tid < nd) lc[tid] = 0;
            __syncthreads();
        }
        // ---- A: digit histogram
        for (uint32_t w = tid; w < T; w += S1_NT) for_unit_keys(w, [&](uint64_t key) { atomicAdd(&h[s1_digit(key, nd)], 1u); });
        __syncthreads();
        // ---- R: one reservation per digit in its region (+ overflow beyond it); stage offsets
        // (the reservation's round trip overlaps the stage-offset scan, which needs only c)
        uint32_t c = 0, g = 0, ra = 0;
        if ((uint32_t)tid < nd) {
            c = h[tid];
            h[tid] = 0;  // ready for the next piece
            if (c) ra = reserve(tid, c + (c & 1u), g);  // even: see the single pass
        }
        uint32_t npk;
        const uint32_t cp = (uint32_t)tid < nd ? c + 1 : 0u;  // one spare slot per digit (parity)
        const uint32_t P = block_excl_sum1<S1_NT, uint32_t>(cp, wsumB, &npk);
        if ((uint32_t)tid < nd) {
            gst[tid] = g;
            if constexpr (PAIRED) lim[tid] = g + ra;
            lof[tid] = lc[tid] = P + ((P ^ g) & 1u);
        }
        __syncthreads();
        const bool staged = npk <= (uint32_t)S1_STAGE;
        // ---- B: place every key (stage, or straight to its region / the overflow list)
        for (uint32_t w = tid; w < T; w += S1_NT)
            for_unit_keys(w, [&](uint64_t key) {
                const uint32_t d = s1_digit(key, nd);
                const uint32_t q = atomicAdd(&lc[d], 1u);
                if (staged) {
                    stage[q] = key;
                } else {
                    put(d, gst[d] + (q - lof[d]), key);
                }
            });
        if (staged) fence_proxy_async_smem();  // stage writes -> the bulk copies
        __syncthreads();
        // ---- W: every digit's run leaves by one bulk copy (+ <= 2 single stores, + overflow)
        if (staged && (uint32_t)tid < nd && paired && (tid & 1)) {
            // a downward run: positions [g0, g0 + in_reg) take the slots [E - in_reg, E) below
            // E = (d + 1) rc - g0 (even; s0 is even as g0 is) -- one bulk copy of an even
            // number of keys to an even slot, the odd one out stored alone
            const uint32_t s0 = lof[tid], cn = lc[tid] - s0, g0 = gst[tid];
            const uint32_t in_reg = min(cn, lim[tid] - g0);
            const uint64_t E = (uint64_t)(tid + 1) * sb.rc - g0;
            const uint32_t m = in_reg & ~1u;
            if (in_reg & 1u) region[E - in_reg] = stage[s0 + m];
            if (m) {
                tma_store_1d(region + E - m, stage + s0, m * 8u);
                bulk_commit();
                bulk_pending = true;
            }
            for (uint32_t e = in_reg; e < cn; ++e) put(tid, g0 + e, stage[s0 + e]);
        } else if (staged && (uint32_t)tid < nd) {
            const uint32_t s0 = lof[tid], cn = lc[tid] - s0, g0 = gst[tid];
            const uint32_t in_reg = PAIRED ? min(cn, lim[tid] - g0) : (g0 >= sb.rc ? 0u : min(cn, sb.rc - g0));
            uint64_t* dst = region + (uint64_t)tid * sb.rc + g0;
            uint32_t i = 0;
            if (in_reg && (s0 & 1u)) {
                dst[0] = stage[s0];
                i = 1;
            }
            const uint32_t m = (in_reg - i) & ~1u;
            if (m) {
                tma_store_1d(dst + i, stage + s0 + i, m * 8u);
                bulk_commit();
                bulk_pending = true;
            }
            if (i + m < in_reg) dst[i + m] = stage[s0 + i + m];
            for (uint32_t e = in_reg; e < cn; ++e) {
                const uint64_t o = (uint64_t)ovb[tid] + (e - in_reg);
                if (o < ovf_cap) ovf[o] = stage[s0 + e];
            }
        }
        if ((uint32_t)tid < nd && (c & 1u)) put(tid, g + c, ~0ull);  // the pad slot of an odd run
    }
    if (!PAIRED && owned && (uint32_t)tid < sb.nd) cur[sb.dbase + tid] = my_cur;
    if (bulk_pending) bulk_wait_all();
}

// Chunks of the split: every digit whose keys fit its region is one chunk (<= hard_cap keys,
// else an "oversize" chunk for the fallback); a digit that overflowed lists its region part
// for the fallback (its other keys are in the overflow list).  One CTA per bin.
__global__ void k_split1_chunks(const S1Bin* __restrict__ sbins, const uint32_t* __restrict__ cur, uint32_t hard_cap,
                                Chunk* __restrict__ chunks, Chunk* __restrict__ over, Chunk* __restrict__ ovd,
                                unsigned long long* __restrict__ ctr, uint32_t pair_cap,
                                const uint32_t* __restrict__ fail) {
    const S1Bin sb = sbins[blockIdx.x];
    if (sb.flags & S1_PAIRED) {
        // pair e: slots [key_base + 2e rc, + 2 rc), digit 2e from the start, 2e + 1 from the end
        const uint64_t rc2 = 2ull * sb.rc;
        for (uint32_t e = threadIdx.x; 2 * e < sb.nd; e += blockDim.x) {
            const uint32_t n0 = cur[sb.dbase + 2 * e], n1 = cur[sb.dbase + 2 * e + 1];
            const uint64_t pb = sb.key_base + 2 * e * (uint64_t)sb.rc;
            if ((uint64_t)n0 + n1 > rc2) {
                // the pair overflowed: the region parts below each digit's first position that
                // did not fit (its other keys are in the overflow list) go to the fallback
                const uint32_t a = min(n0, fail[sb.dbase + 2 * e]), b = min(n1, fail[sb.dbase + 2 * e + 1]);
                if (a) ovd[atomicAdd(&ctr[2], 1ull)] = Chunk{pb, a, 0};
                if (b) ovd[atomicAdd(&ctr[2], 1ull)] = Chunk{pb + rc2 - b, b, 0};
                continue;
            }
            const uint64_t gap = rc2 - n0 - n1;
            if (n0 + n1 <= pair_cap && n0 + n1 <= hard_cap && n0 < 65536u && gap < 65536u) {
                if (n0 + n1) chunks[atomicAdd(&ctr[0], 1ull)] = Chunk{pb, n0 + n1, n0 | (uint32_t)gap << 16};
                continue;
            }
            for (int h = 0; h < 2; ++h) {
                const uint32_t n = h ? n1 : n0;
                if (n == 0) continue;
                const Chunk ch{h ? pb + rc2 - n : pb, n, 0};
                if (n > hard_cap) over[atomicAdd(&ctr[1], 1ull)] = ch;
                else chunks[atomicAdd(&ctr[0], 1ull)] = ch;
            }
        }
        return;
    }
    for (uint32_t d = threadIdx.x; d < sb.nd; d += blockDim.x) {
        const uint32_t n = cur[sb.dbase + d];
        if (n == 0) continue;
        const uint64_t base = sb.key_base + (uint64_t)d * sb.rc;
        if (n > sb.rc) ovd[atomicAdd(&ctr[2], 1ull)] = Chunk{base, sb.rc, 0};
        else if (n > hard_cap) over[atomicAdd(&ctr[1], 1ull)] = Chunk{base, n, 0};
        else chunks[atomicAdd(&ctr[0], 1ull)] = Chunk{base, n, 0};
    }
}

// Pieces of the records appended to the presplit bins since the last call (one CTA).
constexpr int PP_NT = 1024;
__global__ void __launch_bounds__(PP_NT) k_presplit_pieces(const uint32_t* __restrict__ bin_ids, uint32_t n_pb,
                                                           const uint32_t* __restrict__ bin_fill,
                                                           const uint32_t* __restrict__ bin_cap,
                                                           const uint64_t* __restrict__ bin_rec_off,
                                                           uint32_t* __restrict__ done, uint32_t rpp,
                                                           Piece* __restrict__ pieces,
                                                           unsigned long long* __restrict__ n_pieces) {
    __shared__ uint32_t wsum[PP_NT / 32];
    uint64_t base = 0;
    for (uint32_t i0 = 0; i0 < n_pb; i0 += PP_NT) {
        const uint32_t i = i0 + threadIdx.x;
        uint32_t d0 = 0, f = 0, np = 0, b = 0;
        if (i < n_pb) {
            b = bin_ids[i];
            f = min(bin_fill[b], bin_cap[b]);  // (a fill beyond the capacity: the call replans)
            d0 = done[i];
            np = f > d0 ? (f - d0 + rpp - 1) / rpp : 0u;
        }
        uint32_t tot;
        const uint32_t pre = block_excl_sum1<PP_NT, uint32_t>(np, wsum, &tot);
        if (np) {
            const uint64_t ro = bin_rec_off[b];
            for (uint32_t q = 0; q < np; ++q) {
                const uint32_t r0 = d0 + q * rpp;
                pieces[base + pre + q] = Piece{ro + r0, min(rpp, f - r0), i};
            }
            done[i] = f;
        }
        base += tot;
        __syncthreads();  // (wsum is reused)
    }
    if (threadIdx.x == 0) *n_pieces = base;
}

}  // namespace

int split1_piece_records(int k) {
    const int U = std::min(S1_UNIT, 33 - k);
    const int upr = (record_max_windows(k) + U - 1) / U;
    return std::min(S1_REC, S1_UMAX / upr);
}

// Pieces of one records-per-piece for every bin (the presplit, whose bins' windows per record
// are only estimates): 448 records.  C4, one size for all bins: 512 -> 14.5 ms, 464 -> 12.1,
// 448 -> 11.2, 416 -> 11.5 (large-bin records average ~14 windows: bigger pieces often exceed
// the single-pass stage and take the two-pass mode).
int split1_uniform_records(int k) { return std::min(448, split1_piece_records(k)); }

// Records per piece of a bin of W windows in R records split into nd digits: pieces of about
// fill x the windows the single-pass mode takes (NWIN + NWIN / 8 + 16 nd <= S1_STAGE).
#ifndef KMC_S1_FILL
#define KMC_S1_FILL 0.80
#endif
int split1_bin_records(int k, uint64_t W, uint64_t R, uint32_t nd) {
    const int cap = split1_piece_records(k);
    if (W == 0 || R == 0) return cap;
    const double win = ((double)S1_STAGE - 16.0 * nd) / 1.125 * KMC_S1_FILL;
    const double r = win * (double)R / (double)W;
    return (int)std::max(32.0, std::min((double)cap, r));
}

cudaError_t launch_split1(const uint32_t* bins, const Piece* pieces, uint64_t n_pieces, const S1Bin* sbins, int k,
                          int canonical, uint32_t* cur, uint64_t* keys, uint64_t* ovf, unsigned long long* ovf_ctr,
                          uint64_t ovf_cap, int n_ctas, cudaStream_t s, const unsigned long long* n_pieces_dev,
                          uint32_t* fail, bool paired) {
    if (n_pieces == 0 && !n_pieces_dev) return cudaSuccess;
    if (k > 32) return cudaErrorInvalidValue;
    const int unit = std::min(S1_UNIT, 33 - k);
    const unsigned grid =
        n_pieces_dev ? (unsigned)n_ctas : (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(n_pieces, (uint64_t)n_ctas));
    auto go = [&](auto kern, size_t smem) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e) return e;
        kern<<<grid, S1_NT, smem, s>>>(bins, pieces, n_pieces, sbins, k, unit, cur, keys, ovf, ovf_ctr, ovf_cap,
                                      n_pieces_dev, fail);
        return cudaSuccess;
    };
    cudaError_t e;
#ifndef KMC_S1_KSPEC
#define KMC_S1_KSPEC 1
#endif
    // canonical splits of the k-mer lengths of the paper's configurations (25, 28, 31) get
    // instances with k folded into the window extraction; other k at run time
    const int kc = KMC_S1_KSPEC && canonical && (k == 25 || k == 28 || k == 31) ? k : 0;
    if (paired) {
        if (!fail) return cudaErrorInvalidValue;
        const size_t sm = S1Lay<true>::SMEM;
        e = kc == 25   ? go(k_split1<true, true, 25>, sm)
            : kc == 28 ? go(k_split1<true, true, 28>, sm)
            : kc == 31 ? go(k_split1<true, true, 31>, sm)
            : canonical ? go(k_split1<true, true>, sm)
                        : go(k_split1<false, true>, sm);
    } else {
        const size_t sm = S1Lay<false>::SMEM;
        e = kc == 25   ? go(k_split1<true, false, 25>, sm)
            : kc == 28 ? go(k_split1<true, false, 28>, sm)
            : kc == 31 ? go(k_split1<true, false, 31>, sm)
            : canonical ? go(k_split1<true, false>, sm)
                        : go(k_split1<false, false>, sm);
    }
    if (e) return e;
    return cudaGetLastError();
}

cudaError_t launch_split1_chunks(const S1Bin* sbins, uint64_t n_bins, const uint32_t* cur, uint32_t hard_cap,
                                 Chunk* chunks, Chunk* over, Chunk* ovd, unsigned long long* ctr, cudaStream_t s,
                                 uint32_t pair_cap, const uint32_t* fail) {
    if (n_bins == 0) return cudaSuccess;
    k_split1_chunks<<<(unsigned)n_bins, 256, 0, s>>>(sbins, cur, hard_cap, chunks, over, ovd, ctr, pair_cap, fail);
    return cudaGetLastError();
}

cudaError_t launch_presplit_pieces(const uint32_t* bin_ids, uint32_t n_pb, const uint32_t* bin_fill,
                                   const uint32_t* bin_cap, const uint64_t* bin_rec_off, uint32_t* done, uint32_t rpp,
                                   Piece* pieces, unsigned long long* n_pieces, cudaStream_t s) {
    if (rpp == 0) return cudaErrorInvalidValue;
    k_presplit_pieces<<<1, PP_NT, 0, s>>>(bin_ids, n_pb, bin_fill, bin_cap, bin_rec_off, done, rpp, pieces, n_pieces);
    return cudaGetLastError();
}

}  // namespace kmc
