/*
 * kmcgpu.h -- C ABI of the B200 (sm_100a) canonical k-mer counter: the
 * data-parallel hot path of KMC 2 (Deorowicz, Kokot, Grabowski,
 * Debudaj-Grabysz, arXiv 1407.1507).  Citations "P:Lnnn" are lines of the
 * paper text with its section.
 *
 * Operation (kmc_count): "Building the histogram of occurrences of every
 * k-symbol long substring of nucleotide data" (Abstract; P:L46-48,
 * Sec. 1), over canonical k-mers -- "lexicographically smaller of the pair:
 * the k-mer and its reverse complement" (Sec. 2.1) -- keeping the
 * k-mers whose count c satisfies cutoff_min <= c <= cutoff_max (P:L523-525,
 * Sec. 2.5, Suppl. Sec. 1 "-ci", "-cx").  The path follows the
 * paper's two phases (Sec. 2.4): reads are 2-bit packed, each
 * k-mer window gets its signature (restricted canonical minimizer of length p,
 * P:L206-208, Sec. 2.2), reads are cut into super-k-mers that are
 * binned by signature in HBM; each bin is expanded into canonical k-mers,
 * radix sorted and run-length compacted into (k-mer, count)
 * pairs with the cutoffs applied (appendix "Sorter").
 *
 * Symbols and keys.  A->0, C->1, G->2, T->3 (Suppl. Sec. 4).  A
 * k-mer's key is its 2k-bit value with the leftmost symbol most significant,
 * so unsigned order = A<C<G<T lexicographic order.  Lowercase a/c/g/t are
 * folded to upper case; any other byte (N, IUPAC codes, newline, ...)
 * invalidates every k-mer window containing it (reading R3).
 * Windows never cross read boundaries.
 *
 * Output.  out_kmers is sorted strictly ascending by key (DESIGN.md reading
 * R8).  k <= 32: one uint64 per k-mer; 33 <= k <= 64: two uint64 per k-mer,
 * [lo, hi] (little-endian unsigned __int128 layout).  out_counts holds the
 * exact uint32 count (saturating at 2^32-1; reading R9).
 *
 * Memory.  All pointers may be device or host memory (the library asks the
 * CUDA driver which); host inputs are copied to the device inside the call,
 * host outputs are written by a device-to-host copy.  The caller owns every
 * buffer passed in; the library never frees caller memory.  Scratch comes from
 * the allocator set by kmc_set_allocator (default: the library's block cache,
 * which keeps cudaMalloc'd blocks between calls, see kmc_empty_cache) and is
 * released to it before return.
 *
 * Streams and blocking.  All work is enqueued on `stream` (cudaStream_t passed
 * as void*, 0 = legacy default stream).  kmc_count_begin synchronizes the
 * stream a few times (to size scratch from the data: input extent, bin plan,
 * survivor count) and returns once the survivor count is known;
 * kmc_count_finish returns after the outputs are complete.
 *
 * Errors.  Every entry point returns a kmc_status; on a non-OK status
 * kmc_last_error() returns a thread-local message.  No partial-output
 * guarantee on error.  Invalid arguments are rejected before any device work.
 *
 * Determinism.  Output bytes are identical across runs and launch
 * configurations; atomics only decide internal placement.
 */
#ifndef KMCGPU_H
#define KMCGPU_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KMCGPU_VERSION 100

typedef enum {
    KMC_OK = 0,
    KMC_ERR_INVALID_ARG = 1,   /* argument outside the documented range */
    KMC_ERR_OUT_CAPACITY = 2,  /* out_capacity < n_out; stats->n_out holds the required count */
    KMC_ERR_ALLOC = 3,         /* scratch allocation failed */
    KMC_ERR_CUDA = 4,          /* a CUDA runtime call or kernel failed */
    KMC_ERR_INTERNAL = 5,      /* internal consistency check failed (a bug) */
    KMC_ERR_IO = 6             /* an output file could not be written (kmc_write_db) */
} kmc_status;

/* Pipeline stages timed with CUDA events when kmc_options.profile != 0. */
enum {
    KMC_STAGE_INPUT = 0,      /* host->device copy of host inputs */
    KMC_STAGE_SIGNATURE = 1,  /* S1-S3: encode + signatures + super-k-mer histogram (pass 1) */
    KMC_STAGE_PLAN = 2,       /* S4: signature->bin map, bin offsets (scans) */
    KMC_STAGE_SCATTER = 3,    /* S5: super-k-mer records into HBM bins (copy of pass 1's record
                                 stream, or S1-S3 recomputed as pass 2) */
    KMC_STAGE_SMALL_BINS = 4, /* S6-S8 for bins that fit one CTA: expand + SMEM radix sort + compact */
    KMC_STAGE_LARGE_SPLIT = 5,  /* S6 + split of S7 for large bins, count half: expand, count the
                                   hash digits per CTA range, scan, plan chunks */
    KMC_STAGE_LARGE_CHUNKS = 6, /* S7-S8 for large bins: per chunk, SMEM hash count (count_path 0)
                                   or SMEM radix sort + compaction (count_path 1) */
    KMC_STAGE_LARGE_FALLBACK = 7,/* S7-S8 for oversize digits (or all large bins with
                                   large_path=1): device-wide LSD radix sort + run-length pass */
    KMC_STAGE_ORDER = 8,      /* S9: global ascending order of survivors */
    KMC_STAGE_OUTPUT = 9,     /* copy of the sorted survivors into the caller's buffers */
    KMC_STAGE_LARGE_SCATTER = 10, /* S6 + split of S7 for large bins, scatter half: re-expand and
                                     place every key in its digit range in HBM */
    KMC_N_STAGES = 11
};

typedef struct {
    uint64_t n_reads;
    uint64_t n_bases;          /* offsets[n_reads] - offsets[0] */
    uint64_t n_invalid_bases;  /* bytes that are not A/C/G/T/a/c/g/t */
    uint64_t n_windows;        /* valid k-mer windows = sum of all counts before cutoffs */
    uint64_t n_superkmers;     /* maximal equal-signature runs of valid windows */
    uint64_t n_records;        /* bin records (super-k-mer pieces) written to HBM bins */
    uint64_t n_signatures_used;/* distinct signature values seen (incl. the reserved 4^p) */
    uint64_t n_bins;           /* bins in the plan */
    uint64_t n_large_bins;     /* bins sorted by the multi-CTA path */
    uint64_t max_bin_windows;  /* windows in the largest bin */
    uint64_t large_windows;    /* windows in large bins */
    uint64_t n_unique;         /* distinct canonical k-mers before cutoffs */
    uint64_t n_below_min;      /* distinct k-mers removed by cutoff_min */
    uint64_t n_above_max;      /* distinct k-mers removed by cutoff_max */
    uint64_t n_out;            /* pairs written; or required, on KMC_ERR_OUT_CAPACITY */
    uint64_t n_launches;       /* kernels this library launched for the call */
    uint64_t n_input_batches;  /* pass-1 batches of host-resident reads (0: reads were on the device) */
    uint64_t n_large_groups;   /* memory-bounded groups the large bins were processed in */
    uint64_t chunk_capacity;   /* max keys per large-bin chunk (set from the measured distinct ratio) */
    uint64_t n_overflow_chunks;/* chunks whose distinct keys overflowed the SMEM hash table
                                  (counted by the device radix-sort fallback instead) */
    uint64_t n_order_oversize; /* survivors in S9 buckets above one chunk (sorted by the device LSD) */
    uint64_t max_signature_windows; /* windows of the most frequent signature (Table 6) */
    uint64_t n_small_sorted;   /* small bins whose distinct keys overfilled the SMEM hash table
                                  (sorted + run-length compacted in SMEM instead) */
    uint64_t n_cluster_items;  /* (bin, round) items counted by thread-block clusters (large_path 3) */
    uint64_t n_single_items;   /* large bins counted by one CTA's table (large_path 3) */
    uint64_t n_spilled_keys;   /* windows whose key found no slot in an overfull table (counted by
                                  the device radix-sort fallback) */
    uint64_t cluster_size;     /* CTAs per cluster of the large-bin path (0: not used) */
    uint64_t cluster_ctas;     /* CTAs the large-bin cluster kernel ran with */
    uint64_t n_split_overflow; /* large-bin keys whose digit overfilled its region in the one-pass
                                  split (counted by the device radix-sort fallback) */
    uint64_t n_kxmers;         /* (k,x)-mers sorted (kx > 0): Table 7's "sorted fraction" is
                                  n_kxmers / kx_windows */
    uint64_t kx_windows;       /* windows of the bins counted through (k,x)-mers (the small bins) */
    uint64_t n_passes;         /* passes over bin ranges (host-resident reads beyond HBM); 1 = one pass */
    uint64_t n_distribute_reruns; /* sampled distribution: 1 if a bin overflowed its sampled capacity
                                  and pass 1 was repeated on the exact plan */
    uint64_t n_presplit_bins;  /* large bins split batch by batch during pass 1 (presplit) */
    float stage_ms[KMC_N_STAGES];   /* per-stage device time (profile != 0), else 0 */
    uint32_t stage_launches[KMC_N_STAGES];
} kmc_stats;

typedef struct {
    uint32_t profile;          /* 1: record CUDA events around every stage (stats.stage_ms) */
    uint32_t small_bin_capacity; /* 0 = default; max windows of a bin sorted by one CTA
                                    (clamped to the kernel maximum); smaller values force
                                    more bins down the large path (testing) */
    uint32_t force_large;      /* 1: every bin takes the large (multi-CTA) path (testing) */
    uint32_t large_path;       /* 0 (default) / 2: hashed split of every large bin into HBM key
                                  chunks, each counted by count_path.
                                  1: device-wide LSD radix sort of all large-bin keys (testing).
                                  3 (k <= 32, count_path 0; measured slower):
                                  thread-block clusters count each large bin in their CTAs'
                                  shared-memory tables, keys routed to their owner CTA through
                                  distributed shared memory -- no key spill to HBM */
    uint32_t distribute_path;  /* 0 (default): inputs of >= 64 Mi bases take the sampled distribution
                                  (2), smaller ones the record stream: pass 1 streams its records
                                  and S5 copies them into bins.  1: S5 recomputes pass 1 from the
                                  reads (testing).  2: always sampled -- the bin plan comes from a
                                  sample of the reads and pass 1 writes every record
                                  straight into its bin (no record stream, no S5 copy) */
    uint32_t input_batch_mb;   /* host-resident reads are streamed through pass 1 in read-aligned
                                  batches of this many MiB (0 = default 256), double-buffered so
                                  the H2D copy of batch i+1 overlaps pass 1 on batch i */
    uint32_t large_group_mkeys;/* large bins are split/sorted in groups of at most this many Mi
                                  keys (0 = auto: as many as fit in free device memory) */
    uint32_t count_path;       /* S7-S8 of the large-bin chunks.  0: count every chunk in a
                                  shared-memory hash table (default; persistent CTAs, TMA-prefetched
                                  chunks); 1: the paper's radix sort + run-length compaction of
                                  every chunk in shared memory.  Same output. */
    uint32_t chunk_capacity;   /* 0 = auto; else max keys per large-bin chunk (testing: large
                                  values force hash-table overflows onto the fallback).  With
                                  count_path 1 it is clamped to the per-chunk sort's shared-memory
                                  capacity (6144 keys for k <= 32, 3072 above). */
    uint32_t non_canonical;    /* 1: count k-mers as they occur in the reads, not their canonical
                                  form (KMC's -b).  Signatures and binning stay canonical
                                  (a k-mer and its reverse complement share a bin either way).
                                  k = 32 and k = 64 are rejected (KMC_ERR_INVALID_ARG): the
                                  all-T k-mer is the all-ones key, the kernels' empty marker. */
    uint32_t plain_minimizers; /* 1 (diagnostic): signatures are plain canonical minimizers, without
                                  the P:L206-208 restrictions -- the "Minimizers" columns of
                                  Table 6.  Same counts; different bins. */
    uint32_t cluster_size;     /* large_path 3: CTAs per cluster, 0 = auto (16 where the device
                                  holds such clusters, else 8), or 1, 4, 8, 16 (1: single-CTA
                                  tables only -- bins above one table spill; testing) */
    uint32_t table_keys;       /* large_path 3, testing: distinct keys one CTA's table is planned
                                  for (0 = 3/4 of its slots); small values force many rounds */
    uint32_t kx;               /* x of (k,x)-mers (Sec. 2.3), 0..3: the small bins are
                                  counted the paper's way -- records split into (k,x)-mers, sorted,
                                  the sorted sub-arrays merged; large bins keep plain
                                  k-mers (their split routes single k-mers by hash).  Needs
                                  k + x <= 31 and canonical counting.  Same output for every x. */
    uint32_t spill_keys;       /* large_path 3, testing: spill list capacity (0 = auto); a spill
                                  beyond it reruns the large bins on the split path */
    uint32_t pass_mb;          /* host-resident reads: count in passes over ranges of bins whose
                                  records take at most this many MiB of device memory (0 = auto:
                                  passes only when the single-pass working set would not fit the
                                  free device memory) -- f2, inputs beyond HBM */
    uint32_t split_tight;      /* testing (one-pass split): 1 = digit regions without slack
                                  (ceil(W / nd) + 2 slots), so digits overflow into the overflow
                                  list and the fallback is exercised */
    uint32_t presplit;         /* sampled distribution, one-pass split path (k <= 32): the large
                                  bins of the sampled plan are split into their digit regions batch
                                  by batch while pass 1 runs (host-resident reads: under the input
                                  copy).  0 (default): for host-resident reads; 1: always; 2: never.
                                  Same output. */
} kmc_options;

/* Allocator hook: alloc(bytes, stream, ctx) -> device pointer or NULL; free(ptr, stream, ctx).
 * Passing NULL restores the default: a process-wide cache of cudaMalloc'd blocks.  A block
 * freed by a call stays cached, tagged with the call's stream, and is handed out again only
 * to allocations on that stream and device (stream order makes the reuse safe); when
 * cudaMalloc runs out of memory the cache is synchronised, emptied and the allocation
 * retried once.  Not a performance detail: a C4-sized call needs ~40 GB of scratch, and
 * mapping it anew every call costs more than the count. */
typedef void* (*kmc_alloc_fn)(uint64_t bytes, void* stream, void* ctx);
typedef void (*kmc_free_fn)(void* ptr, void* stream, void* ctx);
void kmc_set_allocator(kmc_alloc_fn alloc_fn, kmc_free_fn free_fn, void* ctx);

/* Returns every cached block of the default allocator to the driver (after a device
 * synchronisation).  Call it when other code in the process needs the memory.  Safe at
 * any time no kmc call is running; a no-op when the cache is empty. */
void kmc_empty_cache(void);

/* One-call form.  reads: n_bases bytes, read i = reads[offsets[i]-offsets[0] ..
 * offsets[i+1]-offsets[0]); read_offsets: n_reads+1 nondecreasing uint64 (offsets[0] may
 * be any value).  Requires 1 <= k <= 64, 1 <= p <= min(k, 15) (p = signature length,
 * P:L1188 "-p"), cutoff_max >= max(cutoff_min, 1) (cutoff_min 0 is treated as 1).
 * Writes n_out pairs if out_capacity >= n_out, else returns KMC_ERR_OUT_CAPACITY with
 * stats->n_out = required.  A capacity that is always enough is
 * floor(n_windows / max(cutoff_min, 1)).  stats may be NULL; opt may be NULL. */
kmc_status kmc_count(const uint8_t* reads, const uint64_t* read_offsets, uint64_t n_reads,
                     int k, int p, uint32_t cutoff_min, uint32_t cutoff_max,
                     uint64_t* out_kmers, uint32_t* out_counts, uint64_t out_capacity,
                     kmc_stats* stats, void* stream);

kmc_status kmc_count_ex(const uint8_t* reads, const uint64_t* read_offsets, uint64_t n_reads,
                        int k, int p, uint32_t cutoff_min, uint32_t cutoff_max,
                        uint64_t* out_kmers, uint32_t* out_counts, uint64_t out_capacity,
                        kmc_stats* stats, void* stream, const kmc_options* opt);

/* Two-call form, so the caller can allocate outputs of exactly n_out pairs.
 * kmc_count_begin runs phases S1-S8 and returns the survivor count in *n_out and an
 * opaque job; kmc_count_finish runs S9 into the caller's buffers (capacity as above)
 * and frees the job (also on error).  kmc_job_free releases a job without finishing.
 * Input buffers must stay valid until kmc_count_finish returns. */
typedef struct kmc_job kmc_job;
kmc_status kmc_count_begin(const uint8_t* reads, const uint64_t* read_offsets, uint64_t n_reads,
                           int k, int p, uint32_t cutoff_min, uint32_t cutoff_max,
                           void* stream, const kmc_options* opt, kmc_job** job, uint64_t* n_out);
kmc_status kmc_count_finish(kmc_job* job, uint64_t* out_kmers, uint32_t* out_counts,
                            uint64_t out_capacity, kmc_stats* stats);
void kmc_job_free(kmc_job* job);

/* ---- Sharded counting over several GPUs.  Every rank holds a slice of the
 * reads and runs, on its own GPU:
 *   1. kmc_shard_pass1: S1-S4 on the slice -> its per-signature histograms hist_w (windows)
 *      and hist_r (records), [4^p + 1] uint64 each (device or host), and *n_records, the
 *      number of super-k-mer records it holds (the size of its send buffers).
 *   2. the caller sums hist_w and hist_r over all ranks (an all-reduce);
 *   3. kmc_shard_partition with the global histograms: the bin plan (identical on every
 *      rank) gives every bin to one rank (kmc_shard_owners: contiguous bins, balanced by
 *      windows), and the rank's records are written to the caller's send buffers grouped by
 *      destination rank: send_records [n_records * kmc_record_words(k)] uint32,
 *      send_sigs [n_records] uint32 (device), send_counts [world] (host) records per rank;
 *   4. the caller exchanges them (all-to-all) -- records from every rank for this rank's bins;
 *   5. kmc_shard_count on the received records counts the rank's bins (S5-S8) and returns
 *      *n_out; kmc_count_finish writes its (k-mer, count) pairs, ascending.
 * The k-mer sets of different ranks are disjoint and their union is the single-GPU result
 * of all slices together.  The job is freed by kmc_count_finish or kmc_job_free. */
kmc_status kmc_shard_pass1(const uint8_t* reads, const uint64_t* read_offsets, uint64_t n_reads,
                           int k, int p, uint32_t cutoff_min, uint32_t cutoff_max,
                           void* stream, const kmc_options* opt, kmc_job** job,
                           uint64_t* hist_w, uint64_t* hist_r, uint64_t* n_records);
kmc_status kmc_shard_partition(kmc_job* job, const uint64_t* global_hist_w, const uint64_t* global_hist_r,
                               int world, int rank, uint32_t* send_records, uint32_t* send_sigs,
                               uint64_t* send_counts);
kmc_status kmc_shard_count(kmc_job* job, const uint32_t* recv_records, const uint32_t* recv_sigs,
                           uint64_t n_recv, uint64_t* n_out);
/* ---- The same exchange fused into the partition pass over peer memory (
 * DESIGN.md 8).  Instead of grouping records into send buffers for an all-to-all, the
 * partition kernel writes every record straight into its owner rank's receive buffer, mapped
 * from the peer through CUDA IPC (NVLink / NVSwitch between the GPUs of one node), so the
 * transfer overlaps the partition tile by tile and no separate collective moves records:
 *   3a. kmc_shard_plan(job, global_hist_w, global_hist_r, world, rank, send_counts): the plan
 *       and bin owners (as kmc_shard_partition) and this rank's record count per destination
 *       (send_counts [world], host); no record moves;
 *   3b. the caller all-gathers send_counts into C[src][dst] (world x world);
 *   3c. kmc_shard_recv_alloc(job, n_recv, handles): this rank's receive buffers for
 *       n_recv = sum_src C[src][rank] records (records, then signature tags: two cudaMalloc
 *       allocations) and their CUDA IPC handles, 2 x 64 bytes into handles;
 *   3d. the caller all-gathers the handles (world x 128 bytes, rank order);
 *   3e. kmc_shard_send_peers(job, all_handles, dst_offsets): dst_offsets[d] = first slot of
 *       this rank's records in rank d's buffers = sum_{src < rank} C[src][d]; maps every
 *       peer's buffers, writes every record into its owner's buffers and waits for the
 *       writes; the mappings are closed before returning;
 *   3f. the caller barriers (every rank's writes are then complete);
 *   5'. kmc_shard_count_recv(job, n_out): counts this rank's receive buffers (S5-S8).
 * All ranks must be processes on GPUs of one node that can map each other's memory (the same
 * GPU included).  Errors: KMC_ERR_CUDA (e.g. cudaIpcOpenMemHandle refused), INVALID_ARG. */
kmc_status kmc_shard_plan(kmc_job* job, const uint64_t* global_hist_w, const uint64_t* global_hist_r, int world,
                          int rank, uint64_t* send_counts);
kmc_status kmc_shard_recv_alloc(kmc_job* job, uint64_t n_recv, uint8_t* handles /* 128 bytes */);
kmc_status kmc_shard_send_peers(kmc_job* job, const uint8_t* all_handles /* world x 128 bytes */,
                                const uint64_t* dst_offsets /* [world] */);
kmc_status kmc_shard_count_recv(kmc_job* job, uint64_t* n_out);
/* Bin -> rank map of the sharded plan (host only, no GPU): contiguous bins, each rank taking
 * about total/world windows; owner[b] = the rank whose share holds the bin's midpoint. */
void kmc_shard_owners(const uint64_t* bin_windows, uint64_t n_bins, int world, uint32_t* owner);
int kmc_record_words(int k);  /* uint32 words per super-k-mer record: 4 (k <= 32) or 8 */

/* Test hook for S2 parity: out_sig[j] (n_bases uint32, device or host) = signature of
 * the window starting at base j (the minimum over its k-p+1 p-mers of the canonical
 * p-mer value if allowed by P:L206-208, else the reserved value 4^p), or 0xFFFFFFFF if
 * no valid window starts at j. */
kmc_status kmc_debug_signatures(const uint8_t* reads, const uint64_t* read_offsets, uint64_t n_reads,
                                int k, int p, uint32_t* out_sig, void* stream);
/* Same, plain_minimizers = 1: the minimum canonical p-mer with no restriction (Table 6). */
kmc_status kmc_debug_signatures_ex(const uint8_t* reads, const uint64_t* read_offsets, uint64_t n_reads,
                                   int k, int p, int plain_minimizers, uint32_t* out_sig, void* stream);

/* Signature-rule test hook: out[i] = 1 if the p-mer with value i (i < 4^p) is an allowed
 * signature -- evaluated by the same device function the kernels use. */
kmc_status kmc_debug_allowed(int p, uint8_t* out_allowed, void* stream);

/* KMC 2 database files: writes <path>.kmc_pre and <path>.kmc_suf in the
 * layout of the paper's supplement, Sec. 4 "Database format":
 *   .kmc_pre = "KMCP" | prefixes | map | header | header position | "KMCP"; all integers
 *   little-endian; header = uint32 kmer_length, mode (0), counter_size,
 *   lut_prefix_length, signature_length (p), min_count (cutoff_min), max_count (cutoff_max),
 *   uint64 total_kmers (n), uint32 tmp[7] (0), uint32 KMC_VER (0x200), 68 bytes; header
 *   position = 68 (the header's distance from that field); map = uint32
 *   [4^p + 1], the prefixes-array id of every signature (4^p = "no allowed p-mer");
 *   prefixes = per id, uint64[4^lut]: index of the first record with that id and that
 *   lut-symbol prefix, then one guard = n.
 *   .kmc_suf = "KMCS" | n records | "KMCS"; record = the k-mer without its lut-symbol prefix,
 *   4 symbols per byte with the leftmost in the top bits, then
 *   min(count, counter_max) on counter_size little-endian bytes.
 * Records are ordered by (id, k-mer).  Readings (DESIGN.md R-DB): id = signature >> G,
 * G = max(0, 2p - 14); lut = the largest of k mod 4, k mod 4 + 4, k mod 4 + 8 that is <= k
 * and keeps ids * 4^lut <= 2^23; counter_size = the fewest bytes that hold counter_max
 * (-cs).  The signature of a stored k-mer is the smallest allowed canonical p-mer
 * over its k-p+1 p-mers, the same rule as kmc_count's binning.
 * kmers: n canonical keys, strictly ascending, in kmc_count's output layout (k <= 32: one
 * uint64 each; else [lo, hi] pairs); counts: n uint32; both device or host memory, read only.
 * n < 2^32.  Errors: KMC_ERR_INVALID_ARG (NULL path, k outside [1, 64], p outside
 * [1, min(k, 12)], counter_max = 0, NULL arrays with n > 0), KMC_ERR_IO (file not written),
 * KMC_ERR_ALLOC / KMC_ERR_CUDA.  Synchronous on `stream`. */
kmc_status kmc_write_db(const void* kmers, const uint32_t* counts, uint64_t n, int k, int p, uint32_t cutoff_min,
                        uint32_t cutoff_max, uint32_t counter_max, const char* path, void* stream);

const char* kmc_last_error(void);
int kmc_version(void);

#ifdef __cplusplus
}
#endif
#endif /* KMCGPU_H */
