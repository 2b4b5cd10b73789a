// kmc_internal.h -- host-side declarations shared by the kmcgpu translation units.
#pragma once
#include <cstdint>
#include <functional>
#include <vector>

#include <cuda_runtime.h>

namespace kmc {

// global statistics slots (device unsigned long long[GS_N])
enum {
    GS_WINDOWS = 0,
    GS_SUPERKMERS = 1,
    GS_RECORDS = 2,
    GS_INVALID = 3,
    GS_UNIQUE = 4,
    GS_BELOW = 5,
    GS_ABOVE = 6,
    GS_SURV = 7,        // survivor cursor
    GS_LARGE_KEYS = 8,  // large-bin key cursor
    GS_SIGS_USED = 9,
    GS_TMP_RECS = 10,   // slots reserved in the temporary record stream by pass 1
    GS_MAX_SIG = 11,    // windows of the most frequent signature
    GS_SMALL_SORTED = 12,  // small bins whose hash table overflowed (sorted instead)
    GS_KX = 13,            // (k,x)-mers sorted (kx path)
    GS_KX_WIN = 14,        // windows of the bins counted through (k,x)-mers
    GS_SUB_OVF = 15,       // sub-signature digits whose table overflowed (counted in rounds)
    GS_P1_OVF = 16,        // records beyond their bin's sampled capacity (scatter pass)
    GS_N = 24
};

// ------------------------------------------------------------ phase 1 (distribution)
constexpr int P1_SEG = 512;  // window starts per pass-1 warp segment (the "tile" of tile_r_lo)

struct P1Args {
    const uint8_t* reads;
    const uint64_t* offsets;
    uint64_t n_reads;
    uint64_t off0;
    uint64_t n_bases;
    int k, p;
    int rules;  // 1: signatures obey P:L206-208; 0: plain canonical minimizers (diagnostic)
    int reads_aligned16;
    const uint64_t* tile_r_lo;  // first read index whose start lies after each segment's left edge
    // pass 1
    unsigned long long* hist_w;  // [4^p + 1]
    uint32_t* hist_r;            // [4^p + 1]
    unsigned long long* gstats;
    // pass 2
    const uint32_t* sig2bin;
    const uint64_t* bin_rec_off;
    uint32_t* bin_fill;
    uint32_t* bins;
    uint32_t bin_lo, bin_hi;  // pass 2 writes only the records of bins [bin_lo, bin_hi)
    const uint4* sig_dest;    // pass 2 (sampled plan): per signature {bin, capacity, first slot lo, hi};
                              // records beyond the capacity are dropped and counted in GS_P1_OVF
    int scatter_hist;         // pass 2 also accumulates hist_w (sampled plan)
    uint32_t seg_step;        // 0/1: every segment; s > 1: every s-th segment (the sample pass)
    // pass 1: temporary record stream (nullptr = not used)
    uint32_t* tmp_recs;
    uint32_t* tmp_sig;
    uint64_t tmp_cap;  // records (slots; warps reserve blocks of slots, unused ones get signature INV)
    // debug
    uint32_t* dbg_sig;
};

enum { P1_MODE_HIST = 0, P1_MODE_SCATTER = 1, P1_MODE_DEBUG = 2 };

uint64_t p1_num_tiles(uint64_t n_bases);
cudaError_t launch_tile_reads(const uint64_t* offsets, uint64_t n_reads, uint64_t off0, uint64_t n_tiles,
                              uint64_t* tile_r_lo, cudaStream_t s);
cudaError_t launch_p1(int mode, const P1Args& a, uint64_t n_tiles, cudaStream_t s);
cudaError_t launch_debug_allowed(int p, uint8_t* out, cudaStream_t s);
// S5: records of the temporary stream sorted into their bins by MSD passes over the bin id
// (k_rec_scatter).  A tile holds <= rec_tile_items(k) records of one bucket of the previous
// pass; bucket ids of pass l are bin >> shift_l, cursors start at the buckets' first record.
struct RecTile2 {
    uint64_t begin;
    uint32_t n;
    uint32_t bucket;  // bucket of the previous pass (cursor row)
};
size_t rec_tile_items(int k);
// Tiles of <= TI items over nb buckets, generated on the device (no host round trip):
// bucket b holds items [start(b), start(b+1)), start(b) = base[b << sh] (uint64 or uint32
// array of nbase entries; b << sh >= nbase: total; base == nullptr: one bucket [0, total)).
// prefix (nb + 1 uint64) receives the exclusive scan of the tiles per bucket, so
// prefix[nb] is the tile count; consumers launch an upper bound of CTAs and those at or
// past prefix[nb] exit.  temp: scan_temp_bytes(nb + 1).
struct TileSrc {
    const void* base;
    int is64;
    uint64_t nbase;
    int sh;
    uint64_t total;
    uint64_t off = 0;  // subtracted from the base entries (tiles of a sub-range; total is relative)
};
cudaError_t launch_make_tiles(const TileSrc& src, uint64_t nb, uint32_t TI, uint64_t max_tiles, uint64_t* prefix,
                              void* temp, RecTile2* tiles, cudaStream_t s);
// out_orig_ids: write the input ids (not the mapped ones) to out_ids.  n_tiles_dev: the
// tile count in device memory (grid = max_tiles CTAs).
cudaError_t launch_rec_scatter(int k, const uint32_t* in_recs, const uint32_t* in_ids, const uint32_t* sig2bin,
                               const RecTile2* tiles, uint64_t max_tiles, const uint64_t* n_tiles_dev, int shift,
                               int D, unsigned long long* cursor, uint32_t* out_recs, uint32_t* out_ids,
                               cudaStream_t s, int out_orig_ids = 0, uint32_t* const* peer_recs = nullptr,
                               uint32_t* const* peer_ids = nullptr);
// sharded counting helpers
cudaError_t launch_compose_map(const uint32_t* map_a, const uint32_t* map_b, uint64_t n, uint32_t* out,
                               cudaStream_t s);
cudaError_t launch_owner_count(const uint32_t* sig, uint64_t n, const uint32_t* sig2owner, int world,
                               unsigned long long* counts, cudaStream_t s);
cudaError_t launch_widen(const uint32_t* in, uint64_t n, uint64_t* out, cudaStream_t s);
cudaError_t launch_narrow(const uint64_t* in, uint64_t n, uint32_t* out, cudaStream_t s);
cudaError_t launch_bucket_cursors(const uint64_t* bin_rec_off, uint64_t n_bins, uint64_t n_records, int shift,
                                  uint64_t n_buckets, unsigned long long* cursor, cudaStream_t s);

// ------------------------------------------------------------ scans / plan
// out[0..n] exclusive prefix sums (out[n] = total) of in[0..n) (uint64).
size_t scan_temp_bytes(uint64_t n);
cudaError_t scan_u64(const uint64_t* in, uint64_t* out, uint64_t n, void* temp, cudaStream_t s);
cudaError_t scan_u32_to_u32(const uint32_t* in, uint32_t* out, uint64_t n, void* temp, cudaStream_t s);

struct PlanArgs {
    const unsigned long long* hist_w;
    const uint32_t* hist_r;
    uint64_t ns;          // 4^p + 1
    uint64_t half_cap;    // small-bin cost grouping threshold (capacity / 2)
    uint32_t recw;        // record cost in key units
    // outputs / temps (ns + 1 entries each unless noted)
    uint64_t* cost_scan;  // P
    uint64_t* bnd_scan;   // B
    uint64_t* win_scan;   // Wp
    uint64_t* rec_scan;   // Rp
    uint32_t* sig2bin;    // [ns]
    uint64_t* bin_first;  // [ns + 1]
    uint64_t* bin_w;      // [ns]
    uint64_t* bin_nrec;   // [ns]
    uint64_t* bin_rec_off;// [ns]
    unsigned long long* gstats;
    void* temp;
};
size_t plan_temp_bytes(uint64_t ns);
cudaError_t launch_plan(const PlanArgs& a, cudaStream_t s, int* n_launches);
// Sampled plan (the paper's sampling): hist = ceil(hist * num / den) + floor (both
// arrays, in place), so every signature gets room even if the sample missed it.
cudaError_t launch_scale_hist(unsigned long long* hist_w, uint32_t* hist_r, uint64_t ns, uint64_t num, uint64_t den,
                              uint32_t floor_w, uint32_t floor_r, cudaStream_t s);
// bin_cap[b] = est + z * sqrt(F * est) + margin records (est = the sampled plan's bin_nrec; F =
// num / den); out_scan (n_bins + 1 uint64) = exclusive scan of bin_cap (temp: scan_temp_bytes)
// sig_dest[s] = {sig2bin[s], bin_cap[bin], bin_rec_off[bin] (lo, hi)} for s < ns
cudaError_t launch_sig_dest(const uint32_t* sig2bin, const uint32_t* bin_cap, const uint64_t* bin_rec_off, uint64_t ns,
                            uint4* sig_dest, cudaStream_t s);
cudaError_t launch_bin_caps(const uint64_t* bin_nrec, uint64_t n_bins, double F, double z, uint32_t margin,
                            uint32_t* bin_cap, uint64_t* bin_cap_u64, uint64_t* out_scan, void* temp, cudaStream_t s);
// Exact per-bin tables on an existing bin plan (bin_first) after the sampled scatter: the scan
// of the exact hist_w into win_scan, bin_w from it, bin_nrec = the bins' fill counters
// (bin_rec_off untouched), and the histogram statistics (GS_SIGS_USED, GS_MAX_SIG)
cudaError_t launch_exact_tables(const PlanArgs& a, uint64_t n_bins, const uint32_t* bin_fill, cudaStream_t s,
                                int* n_launches);

// ------------------------------------------------------------ phase 2 (sorting)
struct SmallArgs {
    const uint32_t* bins;
    const uint32_t* small_list;   // bin ids
    const uint64_t* bin_rec_off;
    const uint64_t* bin_nrec;
    const uint64_t* bin_w;
    int k;
    int canonical;                // 0: forward k-mers (-b)
    uint32_t ci, cx;
    void* surv_keys;              // K*
    uint32_t* surv_counts;
    unsigned long long* gstats;
};
int small_capacity(int k);  // max windows per small bin for this key width
// (k,x)-mer path of the small bins (k_kxmer.cu): x in 1..3, k + x <= 31, canonical only;
// bins of at most kx_capacity() windows
int kx_capacity();
cudaError_t launch_small_kx(const SmallArgs& a, uint64_t n_small, int x, cudaStream_t s);
cudaError_t launch_small_bins(const SmallArgs& a, uint64_t n_small, cudaStream_t s);

struct Piece {
    uint64_t rec_begin;
    uint32_t nrec;
    uint32_t lbin;  // index into the large-bin table
};
constexpr int PIECE_RECORDS = 1024;  // LSD path expansion
int msd_piece_records(int k);        // MSD path: records per piece (bounded by shared memory)

// Large bin of the MSD path: keys of the bin occupy [key_base, key_base + n) in the large
// key array after the split; its top-D-bit digit counters live at digit_base.
struct LargeBin {
    uint64_t key_base;
    uint64_t digit_base;
    uint64_t rec_off;
    uint64_t tb;           // split table index of (digit 0, segment 0) of this bin
    uint32_t n;
    uint32_t D;
    uint32_t nrec;
    uint32_t first_range;  // range mode: first split range (CTA) holding pieces of this bin;
                           // piece mode: the bin's first piece
    uint32_t nseg;         // split segments of this bin (ranges, or pieces in piece mode)
    uint32_t pad;          // 1: piece mode (segment = one piece; staged coalesced scatter)
};
int split_piece_mode_dmax(int k);  // largest digit bits of a piece-mode bin (-1: none)
// pieces[piece_prefix[i] + j] = records [j*rec_per_piece, ...) of large bin i
cudaError_t launch_make_pieces(const LargeBin* lbins, const uint64_t* piece_prefix, uint64_t n_lbins,
                               uint32_t rec_per_piece, Piece* pieces, cudaStream_t s);
struct Chunk {
    uint64_t begin;  // into the large key array
    uint32_t n;
    // k_chunk_hash: 0, or a two-segment chunk (a pair of split digits counted together),
    // n0 | gap << 16: key i is at begin + i for i < n0, else at begin + i + gap
    uint32_t pad;
};
int msd_digit_bits(uint64_t bin_windows, int k, int cap);
// Greedy chunk planner: segments are either the large bins (lbins != nullptr; one CTA per
// bin, 2^D digits each, chunk keys at key_base + bin-relative offsets) or 4096-digit windows
// of a global digit array (lbins == nullptr; gstart = exclusive scan of cnt).
struct GreedyArgs {
    const uint32_t* cnt;     // keys per digit
    const uint32_t* gstart;  // position of each digit's first key
    uint64_t n_digits;
    Chunk* chunks;
    Chunk* oversize;
    unsigned long long* counters;  // [0] chunks, [1] oversize
    uint32_t cap;
    uint32_t seg;  // digits per CTA (set by launch_greedy_chunks)
};
// n_keys: total keys of the digits (sizes the segments)
cudaError_t launch_greedy_chunks(GreedyArgs g, uint64_t n_keys, cudaStream_t s);
// Split of the large bins into digit-contiguous key ranges (k_split): count pass (table of
// per-(bin, digit, segment) counts), then, after an exclusive scan of the table, the scatter.
cudaError_t launch_split(bool scatter, const uint32_t* bins, const Piece* pieces, uint64_t n_pieces,
                         const LargeBin* lbins, int k, int canonical, int dmax, uint32_t n_ranges, uint32_t* table,
                         void* keys, cudaStream_t s);
cudaError_t launch_digit_totals(const LargeBin* lbins, uint64_t n_lbins, const uint32_t* pos, uint32_t* cnt,
                                uint32_t* start,
                                cudaStream_t s);
cudaError_t launch_chunk_sort(const void* keys, const Chunk* chunks, uint64_t n_chunks, int k, uint32_t ci,
                              uint32_t cx, void* surv_keys, uint32_t* surv_counts, unsigned long long* gstats,
                              cudaStream_t s);
// S7-S8 of the chunks by SMEM hash counting (persistent, one CTA per SM, TMA-prefetched).
// The key buffer must have chunk_key_slack_bytes() of readable slack past its last key.
// Chunks that hold more distinct keys than the table (rare) are appended to overflow[] and
// must be counted by another path.  chunk_hash_cap(k): table slots (distinct keys < 3/4 of it
// are always safe).
size_t chunk_key_slack_bytes();
int chunk_hash_cap(int k);
cudaError_t launch_chunk_hash(const void* keys, const Chunk* chunks, uint64_t n_chunks, int k, uint32_t ci,
                              uint32_t cx, void* surv_keys, uint32_t* surv_counts, unsigned long long* gstats,
                              Chunk* overflow, unsigned long long* n_overflow, int n_sms, cudaStream_t s);
cudaError_t launch_large_expand(const uint32_t* bins, const Piece* pieces, uint64_t n_pieces, int k, int canonical,
                                void* keys, unsigned long long* gstats, cudaStream_t s);

// One-pass sized split of the large bins (k_split1.cu, k <= 32): bin b gets nd digits
// (digit = (hash(key) * nd) >> 32), digit d owns key slots [key_base + d * rc, + rc).
// Paired layout (flags & S1_PAIRED, nd even; needs fail[], UINT_MAX-initialised per digit):
// digits 2e and 2e + 1 share the slots [key_base + 2e rc, + 2 rc), the even one filling them
// upwards from the start, the odd one downwards from the end (their counts are one 64-bit
// word of cur, the even digit low), so that a pair overflows only when both together exceed
// 2 rc, and a pair is one chunk with one gap when it fits the table.
constexpr int S1_DMAX = 512;
constexpr uint32_t S1_PAIRED = 1;
struct S1Bin {
    uint64_t key_base;
    uint32_t nd, rc, dbase, flags;
};
int split1_piece_records(int k);
int split1_uniform_records(int k);  // the presplit's records per piece
int split1_bin_records(int k, uint64_t W, uint64_t R, uint32_t nd);  // per bin, sized by windows
// cur: per-digit key counts (zeroed; may exceed rc: overflow); ovf_ctr: keys beyond their
// region (written to ovf while below ovf_cap)
// n_pieces_dev (optional): the piece count in device memory (pieces built on the device);
// n_pieces is then unused
cudaError_t launch_split1(const uint32_t* bins, const Piece* pieces, uint64_t n_pieces, const S1Bin* sbins, int k,
                          int canonical, uint32_t* cur, uint64_t* keys, uint64_t* ovf, unsigned long long* ovf_ctr,
                          uint64_t ovf_cap, int n_ctas, cudaStream_t s,
                          const unsigned long long* n_pieces_dev = nullptr, uint32_t* fail = nullptr,
                          bool paired = false);
// ctr[0] chunks, ctr[1] oversize (> hard_cap), ctr[2] overflowed digits (region parts in ovd).
// Paired bins: a pair whose digits fit their regions and hold <= pair_cap keys together is one
// two-segment chunk.  Bins with nd = 0 are skipped.
cudaError_t launch_split1_chunks(const S1Bin* sbins, uint64_t n_bins, const uint32_t* cur, uint32_t hard_cap,
                                 Chunk* chunks, Chunk* over, Chunk* ovd, unsigned long long* ctr, cudaStream_t s,
                                 uint32_t pair_cap = 0, const uint32_t* fail = nullptr);
// Pieces of the records that pass 1 appended to the presplit bins since the last call
// (done[i]: records already split; fill: the bins' fill counters, capped by cap): at most
// rpp records each, written to pieces[0, *n_pieces).  One CTA.
cudaError_t launch_presplit_pieces(const uint32_t* bin_ids, uint32_t n_pb, const uint32_t* bin_fill,
                                   const uint32_t* bin_cap, const uint64_t* bin_rec_off, uint32_t* done, uint32_t rpp,
                                   Piece* pieces, unsigned long long* n_pieces, cudaStream_t s);

// S6-S8 of the large bins through sub-signatures (k_subsplit.cu, large_path 4, SS_KMIN <= k <=
// SS_KMAX): bin b gets nd digits, digit = hash of the window's sub-signature (the minimum
// hashed canonical q-mer); the sub-records (bin record format, 16 bytes) of a digit fill its
// region of rc slots, then pool blocks of SS_BLK slots from the digit's block table (at most
// SS_MAXB; btab[digit * SS_MAXB + i] = block id + 1, block j = slots xbase + j * SS_BLK of the
// same array), then the overflow list.
constexpr int SS_KMIN = 22, SS_KMAX = 32;
constexpr int SS_BLK = 512;
constexpr int SS_MAXB = 64;
constexpr int SS_DMAX = 256;
struct SSBin {
    uint64_t rbase;  // slot of the bin's digit 0 region; digit d's region starts at rbase + d * rc
    uint32_t nd, dbase, rc, pad;
};
int subsplit_piece_records(int k);
// cur / cur_w: sub-records / windows per digit (zeroed); btab: zeroed; ctr[0] pool blocks
// claimed (> n_blocks: rerun with a larger pool), ctr[1] sub-records beyond the block tables
// (written to ovf while below ovf_cap)
cudaError_t launch_subsplit(const uint32_t* bins, const Piece* pieces, uint64_t n_pieces, const SSBin* sbins, int k,
                            uint32_t* cur, uint32_t* cur_w, uint32_t* btab, void* pool, uint64_t xbase,
                            uint64_t n_blocks, void* ovf, uint64_t ovf_cap, unsigned long long* ctr, int n_ctas,
                            cudaStream_t s);
// fb_list / fb_ctr[0]: digits whose sub-records overflowed the block table (for the
// fallback); fb_ctr[1] = 1 if a digit could not be counted in 2^20 rounds (internal error)
// dinfo / drc: n_digits scratch entries (each digit's region, filled here)
cudaError_t launch_subcount(const void* pool, uint64_t xbase, const SSBin* sbins, uint32_t n_bins, uint2* dinfo,
                            uint32_t* drc, const uint32_t* cur, const uint32_t* cur_w, const uint32_t* btab, uint32_t n_digits, int k, int canonical,
                            uint32_t ci, uint32_t cx, uint64_t* surv_keys, uint32_t* surv_counts,
                            unsigned long long* gstats, uint32_t* fb_list, unsigned long long* fb_ctr, int n_sms,
                            cudaStream_t s);

// S6-S8 of the large bins by thread-block clusters (k_cluster.cu, k <= 32): a cluster item is
// (bin, round r of R) counted by all CTAs of a cluster with keys routed to their owner CTA
// through distributed shared memory; a single item is a bin counted by one CTA's table.
struct ClItem {
    uint64_t rec_off;  // first record of the bin
    uint32_t nrec;
    uint16_t round, nround;
};
int cl_table_slots();
int cl_records_per_piece(int k);
int cluster_max_active(int cluster);  // 0 if the device cannot hold such clusters
// ctr: 3 zeroed uint64 ([2] = spilled keys on return; spill holds min(ctr[2], spill_cap) keys).
// max_ctas: 0 = every SM; else at most this many CTAs.  *n_ctas: CTAs launched.
cudaError_t launch_cluster_count(const uint32_t* bins, const ClItem* citems, uint64_t n_citems, const ClItem* sitems,
                                 uint64_t n_sitems, int cluster, int k, int canonical, uint32_t ci, uint32_t cx,
                                 unsigned long long* ctr, uint64_t* spill, uint64_t spill_cap, void* surv_keys,
                                 uint32_t* surv_counts, unsigned long long* gstats, int max_ctas, cudaStream_t s,
                                 int* n_ctas);

// Device-wide LSD radix sort of n keys (+ optional uint32 values).  Result lands in
// (*res_keys, *res_vals) which is either the input or the alternate buffers.
struct RadixScratch {
    void* keys_alt;
    uint32_t* vals_alt;
    uint32_t* tile_hist;   // radix_status_words(n): the onesweep look-back status
    uint32_t* tile_off;    // radix_aux_words(): per-pass digit histograms, bases, tile counters
    void* scan_temp;
    unsigned long long* red;  // 4 entries
    unsigned long long* red_host;  // pinned 4 entries
};
uint64_t radix_tile_items(int key_words);
size_t radix_scan_temp_bytes(uint64_t n, int key_words);
// onesweep scratch: tile_hist needs radix_status_words(n) uint32 (look-back status), tile_off
// radix_aux_words() uint32 (per-pass histograms, digit bases, tile counters)
uint64_t radix_status_words(uint64_t n, int key_words);
uint64_t radix_aux_words();
// KMC 2 database writer (k_db.cu; Suppl. Sec. 4; reading R-DB)
int db_group_shift(int p);
uint64_t db_n_arrays(int p);
int db_lut_length(int k, int p);
int db_counter_bytes(uint32_t cs);
cudaError_t launch_db_ids(int key_words, const void* keys, uint64_t n, int k, int p, uint64_t* ids, uint32_t* idx,
                          cudaStream_t s);
cudaError_t launch_db_hist(int key_words, const void* keys, const uint64_t* sids, const uint32_t* perm, uint64_t n,
                           int k, int lut, unsigned long long* cnt, cudaStream_t s);
cudaError_t launch_db_records(int key_words, const void* keys, const uint32_t* counts, const uint32_t* perm,
                              uint64_t n, int k, int lut, int cb, uint32_t cs, uint8_t* out, cudaStream_t s);
cudaError_t device_radix_sort(int key_words, void* keys, uint32_t* vals, uint64_t n, int nbits,
                              const RadixScratch& rs, cudaStream_t s, void** res_keys, uint32_t** res_vals,
                              int* n_launches);

cudaError_t launch_rle(int key_words, const void* keys, uint64_t n, uint32_t ci, uint32_t cx, void* surv_keys,
                       uint32_t* surv_counts, unsigned long long* gstats, cudaStream_t s);

// ------------------------------------------------------------ S9 global order
// Most-significant-digit passes of <= 8 bits each, every tile of survivors sorted by its
// digit in shared memory before it is written (coalesced runs), then one shared-memory sort
// per chunk of consecutive buckets.
struct OrdTile {
    uint64_t begin;   // first item
    uint32_t n;       // items (<= order_tile_items)
    uint32_t bucket;  // histogram / cursor row (pass 2: the pass-1 digit)
};
struct OrderScratch {
    uint32_t* hist;         // [2^order_digit_bits] histogram of the current pass
    uint32_t* start;        // [2^order_digit_bits + 1] exclusive scan of hist
    uint32_t* cursor;       // [2^order_digit_bits] scatter cursors
    Chunk* chunks;          // [2^order_digit_bits]
    Chunk* oversize;        // [2^order_digit_bits]
    unsigned long long* counters;  // [80]
    OrdTile* tiles;         // [order_max_tiles(n, k)]
    uint64_t* tprefix;      // [order_prev_buckets(n, k) + 1] tiles per bucket (device-built tiles)
    void* ttemp;            // scan_temp_bytes(order_prev_buckets(n, k) + 1)
    void* tmp_keys;         // [n] K
    uint32_t* tmp_vals;     // [n]
    void* scan_temp;        // order_scan_temp_bytes(2^(D1+D2) + 1)
    unsigned long long* host;  // pinned, >= 80 entries
    uint32_t* start0 = nullptr;  // [257] top-level bucket starts (host outputs: S9 by groups)
};
struct OrderSegment {
    uint64_t begin, n;  // items of an oversize bucket in (*seg_keys, *seg_vals) after launch_order
};
int order_digit_bits(uint64_t n, int k);  // bits of all MSD passes
uint64_t order_prev_buckets(uint64_t n, int k);  // buckets before the last MSD pass
uint64_t order_tile_items(int key_words);
uint64_t order_max_tiles(uint64_t n, int k);
size_t order_scan_temp_bytes(uint64_t n_digits);
// Sorts (keys, vals) ascending into (out_keys, out_vals); keys/vals are used as scratch.
// Buckets holding more than the chunk capacity are left, grouped, in (*seg_keys, *seg_vals)
// and returned in *oversize for the caller to sort with device_radix_sort and copy out.
// range_done (optional, 64-bit keys): the final sorts run in groups of consecutive buckets;
// after each group's kernels are enqueued on s, range_done(lo, hi, final) names its output
// items [lo, hi) -- final = false when the group holds an oversize bucket (its items are in
// place only after the caller's oversize sort)
using OrderRangeFn = std::function<void(uint64_t lo, uint64_t hi, bool final)>;
cudaError_t launch_order(int key_words, void* keys, uint32_t* vals, uint64_t n, int k, void* out_keys,
                         uint32_t* out_vals, const OrderScratch& os, cudaStream_t s, int* launches,
                         std::vector<OrderSegment>* oversize, void** seg_keys, uint32_t** seg_vals,
                         const OrderRangeFn* range_done = nullptr);

}  // namespace kmc
