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
constexpr int S1_REC = 512;       // records per piece at most
constexpr int S1_UMAX = 7680;     // units per piece (umap entries)
constexpr int S1_STAGE = 8192;    // keys staged per piece (+ one spare slot per digit)
constexpr int S1_RBW = S1_REC * 4 + 8;
constexpr int S1_UNIT = 5;        // windows per expansion unit at most (k + unit - 1 <= 32 symbols)

__device__ __forceinline__ uint32_t s1_digit(uint64_t key, uint32_t nd) {
    const uint32_t h = (((uint32_t)(key >> 32) * 0x85EBCA6Bu) ^ (uint32_t)key) * 0x9E3779B1u;
    return (uint32_t)(((uint64_t)h * nd) >> 32);
}

constexpr size_t S1_OFF_STAGE = 0;
constexpr size_t S1_OFF_RB = S1_OFF_STAGE + (size_t)S1_STAGE * 8;
constexpr size_t S1_OFF_UMAP = S1_OFF_RB + 2 * (size_t)S1_RBW * 4;
constexpr size_t S1_OFF_RINFO = S1_OFF_UMAP + (size_t)S1_UMAX * 2;
constexpr size_t S1_OFF_DIG = S1_OFF_RINFO + (size_t)S1_REC * 4;  // h, gst, lof, lc, ovb: S1_DMAX each
constexpr int S1_SOVF = 256;      // single-pass mode: keys beyond their digit's stage region
constexpr size_t S1_OFF_SOVK = S1_OFF_DIG + 5 * (size_t)S1_DMAX * 4;
constexpr size_t S1_OFF_SOVI = S1_OFF_SOVK + (size_t)S1_SOVF * 8;
constexpr size_t S1_OFF_MBAR = S1_OFF_SOVI + (size_t)S1_SOVF * 4;
constexpr size_t S1_SMEM = S1_OFF_MBAR + 16 + 16;
static_assert(S1_OFF_RB % 16 == 0 && S1_OFF_MBAR % 8 == 0 && S1_OFF_SOVK % 8 == 0, "alignment");
static_assert(2 * S1_SMEM + 2048 <= 228 * 1024, "two CTAs per SM");
static_assert(S1_DMAX <= 512, "digit in 9 bits of an overflow entry");
static_assert(S1_DMAX <= S1_NT, "one thread per digit");

template <bool CANON>
__global__ void __launch_bounds__(S1_NT, 2) k_split1(const uint32_t* __restrict__ bins, const Piece* __restrict__ pieces,
                                                     uint64_t n_pieces, const S1Bin* __restrict__ sbins, int k,
                                                     int unit, uint32_t* __restrict__ cur, uint64_t* __restrict__ keys,
                                                     uint64_t* __restrict__ ovf, unsigned long long* __restrict__ ovf_ctr,
                                                     uint64_t ovf_cap) {
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
    uint64_t* sovk = reinterpret_cast<uint64_t*>(sm + S1_OFF_SOVK);  // single pass: stage-overflow keys
    uint32_t* sovi = reinterpret_cast<uint32_t*>(sm + S1_OFF_SOVI);  //   their digit | rank << 9
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + S1_OFF_MBAR);
    __shared__ uint32_t wsumA[S1_NT / 32], wsumB[S1_NT / 32];  // alternating scan scratch
    __shared__ uint32_t novf;
    const int tid = threadIdx.x;
    const int U = unit;
    const uint32_t R = gridDim.x, r = blockIdx.x;
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
            cur_bin = pc.lbin;
            sb = sbins[cur_bin];
            C1 = sb.nd ? ((uint32_t)S1_STAGE / sb.nd) & ~1u : 0u;
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
        if (bulk_pending) {  // the previous piece's stage has been read by its bulk copies
            bulk_wait_read();
            bulk_pending = false;
        }
        if (tid < S1_DMAX) lc[tid] = 0;  // (the same thread read it last: the previous piece's W)
        if (tid == 0) novf = 0;
        uint32_t T;
        const uint32_t pre2 = block_excl_sum1<S1_NT, uint32_t>(nu | (n << 16), wsumA, &T);
        const uint32_t NWIN = T >> 16, pre = pre2 & 0xFFFFu;
        T &= 0xFFFFu;
        for (uint32_t j = 0; j < nu; ++j) umap[pre + j] = (uint16_t)tid;
        if ((uint32_t)tid < pc.nrec) rinfo[tid] = pre | (n << 16);
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
        // place key at position i of digit d: its region, or the overflow list beyond it
        auto put = [&](uint32_t d, uint32_t i, uint64_t key) {
            if (i < sb.rc) {
                region[(uint64_t)d * sb.rc + i] = key;
            } else {
                const uint32_t lo = gst[d] > sb.rc ? gst[d] : sb.rc;
                const uint64_t o = (uint64_t)ovb[d] + (i - lo);
                if (o < ovf_cap) ovf[o] = key;
            }
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
                    uint32_t g = 0;
                    if (c) g = atomicAdd(&cur[sb.dbase + tid], ce);
                    if (c && g + ce > sb.rc) {
                        const uint32_t lo = g > sb.rc ? g : sb.rc;
                        ovb[tid] = (uint32_t)atomicAdd(ovf_ctr, (unsigned long long)(g + ce - lo));
                    }
                    gst[tid] = g;
                    lof[tid] = c;
                    if (c) {
                        // the stage part (+ the pad slot when the run ends inside it), even-sized
                        uint32_t sn = c < C1 ? ce : C1;
                        if ((c & 1u) && c < C1) {
                            stage[tid * C1 + c] = ~0ull;
                            fence_proxy_async_smem();
                        }
                        const uint32_t in_reg = g >= sb.rc ? 0u : min(sn, sb.rc - g);  // even: g, rc even
                        if (in_reg) {
                            tma_store_1d(region + (uint64_t)tid * sb.rc + g, stage + tid * C1, in_reg * 8u);
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
        uint32_t c = 0, g = 0;
        if ((uint32_t)tid < nd) {
            c = h[tid];
            h[tid] = 0;  // ready for the next piece
            if (c) g = atomicAdd(&cur[sb.dbase + tid], c + (c & 1u));  // even: see the single pass
        }
        uint32_t npk;
        const uint32_t cp = (uint32_t)tid < nd ? c + 1 : 0u;  // one spare slot per digit (parity)
        const uint32_t P = block_excl_sum1<S1_NT, uint32_t>(cp, wsumB, &npk);
        if ((uint32_t)tid < nd) {
            if (c && g + c + (c & 1u) > sb.rc) {
                const uint32_t lo = g > sb.rc ? g : sb.rc;
                ovb[tid] = (uint32_t)atomicAdd(ovf_ctr, (unsigned long long)(g + c + (c & 1u) - lo));
            }
            gst[tid] = g;
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
                    const uint32_t i = gst[d] + (q - lof[d]);
                    if (i < sb.rc) {
                        region[(uint64_t)d * sb.rc + i] = key;
                    } else {
                        const uint32_t lo = gst[d] > sb.rc ? gst[d] : sb.rc;
                        const uint64_t o = (uint64_t)ovb[d] + (i - lo);
                        if (o < ovf_cap) ovf[o] = key;
                    }
                }
            });
        if (staged) fence_proxy_async_smem();  // stage writes -> the bulk copies
        __syncthreads();
        // ---- W: every digit's run leaves by one bulk copy (+ <= 2 single stores, + overflow)
        if (staged && (uint32_t)tid < nd) {
            const uint32_t s0 = lof[tid], cn = lc[tid] - s0, g0 = gst[tid];
            const uint32_t in_reg = g0 >= sb.rc ? 0u : min(cn, sb.rc - g0);
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
    if (bulk_pending) bulk_wait_all();
}

// Chunks of the split: every digit whose keys fit its region is one chunk (<= hard_cap keys,
// else an "oversize" chunk for the fallback); a digit that overflowed lists its region part
// for the fallback (its other keys are in the overflow list).  One CTA per bin.
__global__ void k_split1_chunks(const S1Bin* __restrict__ sbins, const uint32_t* __restrict__ cur, uint32_t hard_cap,
                                Chunk* __restrict__ chunks, Chunk* __restrict__ over, Chunk* __restrict__ ovd,
                                unsigned long long* __restrict__ ctr) {
    const S1Bin sb = sbins[blockIdx.x];
    for (uint32_t d = threadIdx.x; d < sb.nd; d += blockDim.x) {
        const uint32_t n = cur[sb.dbase + d];
        if (n == 0) continue;
        const uint64_t base = sb.key_base + (uint64_t)d * sb.rc;
        if (n > sb.rc) ovd[atomicAdd(&ctr[2], 1ull)] = Chunk{base, sb.rc, 0};
        else if (n > hard_cap) over[atomicAdd(&ctr[1], 1ull)] = Chunk{base, n, 0};
        else chunks[atomicAdd(&ctr[0], 1ull)] = Chunk{base, n, 0};
    }
}

}  // namespace

int split1_piece_records(int k) {
    const int U = std::min(S1_UNIT, 33 - k);
    const int upr = (record_max_windows(k) + U - 1) / U;
    return std::min(S1_REC, S1_UMAX / upr);
}

cudaError_t launch_split1(const uint32_t* bins, const Piece* pieces, uint64_t n_pieces, const S1Bin* sbins, int k,
                          int canonical, uint32_t* cur, uint64_t* keys, uint64_t* ovf, unsigned long long* ovf_ctr,
                          uint64_t ovf_cap, int n_ctas, cudaStream_t s) {
    if (n_pieces == 0) return cudaSuccess;
    if (k > 32) return cudaErrorInvalidValue;
    const int unit = std::min(S1_UNIT, 33 - k);
    const unsigned grid = (unsigned)std::max<uint64_t>(1, std::min<uint64_t>(n_pieces, (uint64_t)n_ctas));
    cudaError_t e;
    if (canonical) {
        if ((e = cudaFuncSetAttribute(k_split1<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S1_SMEM)))
            return e;
        k_split1<true><<<grid, S1_NT, S1_SMEM, s>>>(bins, pieces, n_pieces, sbins, k, unit, cur, keys, ovf, ovf_ctr,
                                                    ovf_cap);
    } else {
        if ((e = cudaFuncSetAttribute(k_split1<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)S1_SMEM)))
            return e;
        k_split1<false><<<grid, S1_NT, S1_SMEM, s>>>(bins, pieces, n_pieces, sbins, k, unit, cur, keys, ovf, ovf_ctr,
                                                     ovf_cap);
    }
    return cudaGetLastError();
}

cudaError_t launch_split1_chunks(const S1Bin* sbins, uint64_t n_bins, const uint32_t* cur, uint32_t hard_cap,
                                 Chunk* chunks, Chunk* over, Chunk* ovd, unsigned long long* ctr, cudaStream_t s) {
    if (n_bins == 0) return cudaSuccess;
    k_split1_chunks<<<(unsigned)n_bins, 256, 0, s>>>(sbins, cur, hard_cap, chunks, over, ovd, ctr);
    return cudaGetLastError();
}

}  // namespace kmc
