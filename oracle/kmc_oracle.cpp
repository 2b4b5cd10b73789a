/*
 * oracle/kmc_oracle.cpp -- CPU ORACLE for canonical k-mer counting (KMC 2,
 * arXiv 1407.1507).  TEST INFRASTRUCTURE ONLY: only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference
 * legs may load this library.  The product path (paper_1407_1507_b200/) never
 * links, imports or calls it, and this file shares no code, header, table or
 * helper with the CUDA path.
 *
 * What it computes is the PLAIN DEFINITION of the result:
 *   - k-mer counting = "the histogram of occurrences of every k-symbol long
 *     substring" (Abstract; Sec. 1);
 *   - canonical k-mer = "lexicographically smaller of the pair: the k-mer and
 *     its reverse complement" (Sec. 2.1);
 *   - symbol codes A->0, C->1, G->2, T->3, leftmost symbol most significant
 *     (Suppl. Sec. 4 "[map]": ACGAC = 97);
 *   - cutoffs: keep k-mers with ci <= count <= cx (Sec. 2.5;
 *     P:L1191-1193 Suppl. Sec. 1; reading R10 in DESIGN.md);
 *   - non-ACGT symbols (after case folding) make every window containing them
 *     invalid (reading R3; "segment_read").
 * Signatures (used only by the K2 debug-hook parity test) follow Sec. 2.2,
 * canonical minimizers restricted to m-mers that do not start with
 * AAA or ACA and contain no AA except at the beginning (readings R1, R2, R4).
 *
 * Counting: every valid window's canonical value is appended to an array, the
 * array is sorted with std::sort (a library primitive), and equal neighbours
 * are counted -- the histogram by definition.  f and r are recomputed from
 * the characters for every window (no rolling update), in O(k) per window.
 * Status: parity PINNED (tests/test_oracle.py).
 */
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>

typedef unsigned __int128 u128;

/* symbol code by P:L1506: A->0, C->1, G->2, T->3; lowercase folded (R3); -1 = not ACGT */
static inline int sym_code(uint8_t ch) {
    switch (ch) {
        case 'A': case 'a': return 0;
        case 'C': case 'c': return 1;
        case 'G': case 'g': return 2;
        case 'T': case 't': return 3;
        default: return -1;
    }
}

/* true iff every symbol of w[0..k) is A/C/G/T (either case) */
static bool window_valid(const uint8_t* w, int k) {
    for (int j = 0; j < k; ++j)
        if (sym_code(w[j]) < 0) return false;
    return true;
}

/* f = sum_j code(w[j]) * 4^(k-1-j)  (leftmost symbol most significant) */
static u128 forward_value(const uint8_t* w, int k) {
    u128 f = 0;
    for (int j = 0; j < k; ++j) f = f * 4 + (u128)sym_code(w[j]);
    return f;
}

/* r = value of the reverse complement: read w backwards, complement each
 * symbol (A<->T, C<->G, i.e. code -> 3 - code): sum_j (3 - code(w[k-1-j])) * 4^(k-1-j) */
static u128 revcomp_value(const uint8_t* w, int k) {
    u128 r = 0;
    for (int j = 0; j < k; ++j) r = r * 4 + (u128)(3 - sym_code(w[k - 1 - j]));
    return r;
}

/* canonical value = min(f, r) */
static u128 canonical_value(const uint8_t* w, int k) {
    u128 f = forward_value(w, k), r = revcomp_value(w, k);
    return f < r ? f : r;
}

template <typename K>
static int64_t count_impl(const uint8_t* reads, const uint64_t* offsets, uint64_t n_reads, int k,
                          uint32_t ci, uint32_t cx, uint64_t* out_keys, uint32_t* out_counts,
                          uint64_t cap, uint64_t* stats, int canonical) {
    std::vector<K> keys;
    uint64_t n_windows = 0;
    for (uint64_t i = 0; i < n_reads; ++i) {
        uint64_t b = offsets[i], e = offsets[i + 1];
        if (e < b + (uint64_t)k) continue;
        for (uint64_t s = b; s + k <= e; ++s) {
            const uint8_t* w = reads + (s - offsets[0]);
            if (!window_valid(w, k)) continue;
            /* -b: "turn off transformation of k-mers into canonical form" */
            keys.push_back((K)(canonical ? canonical_value(w, k) : forward_value(w, k)));
            ++n_windows;
        }
    }
    std::sort(keys.begin(), keys.end());
    if (ci == 0) ci = 1;
    uint64_t n_unique = 0, n_below = 0, n_above = 0, n_out = 0;
    for (size_t a = 0; a < keys.size();) {
        size_t z = a;
        while (z < keys.size() && keys[z] == keys[a]) ++z;
        uint64_t c = z - a;
        ++n_unique;
        if (c < ci) ++n_below;
        else if (c > cx) ++n_above;
        else {
            if (n_out < cap) {
                u128 v = (u128)keys[a];
                if (sizeof(K) == 8) {
                    out_keys[n_out] = (uint64_t)v;
                } else {
                    out_keys[2 * n_out] = (uint64_t)v;
                    out_keys[2 * n_out + 1] = (uint64_t)(v >> 64);
                }
                out_counts[n_out] = (uint32_t)(c > 0xFFFFFFFFull ? 0xFFFFFFFFull : c);
            }
            ++n_out;
        }
        a = z;
    }
    if (stats) {
        stats[0] = n_windows; stats[1] = n_unique; stats[2] = n_below; stats[3] = n_above; stats[4] = n_out;
    }
    return (int64_t)n_out;
}

/* ---------------------------------------------------------------------------------------
 * Key-range-partitioned, multi-threaded form of the same definition (SURVEY 8(d) "Oracle
 * timing"; used for the full-size configs, where one sorted array of every window would not
 * fit, and for the CPU baseline on all host cores).  The key space is cut into R contiguous
 * ranges [bound[j], bound[j+1]) at quantiles of a sample of the windows' values (every
 * SAMPLE-th valid window).  Equal keys fall into one range, so the sorted per-range
 * histograms, concatenated in range order, are the histogram of all windows.  Ranges are
 * processed T at a time ("rounds", bounding memory): in a round every thread scans its
 * slice of the reads, recomputes f and r per window exactly as count_impl does, and keeps
 * the values that fall into the round's ranges, one vector per range; then thread t owns
 * range t of the round, concatenates the threads' vectors for it, std::sorts them and
 * counts equal neighbours.  Nothing but the partition differs from count_impl.
 * --------------------------------------------------------------------------------------- */
template <typename K>
static int64_t count_par_impl(const uint8_t* reads, const uint64_t* offsets, uint64_t n_reads, int k,
                              uint32_t ci, uint32_t cx, uint64_t** out_keys, uint32_t** out_counts,
                              uint64_t* stats, int canonical, int T, uint64_t round_keys) {
    const uint64_t SAMPLE = 61;
    if (T < 1) T = 1;
    if (ci == 0) ci = 1;
    /* read slices: equal numbers of bases per thread */
    std::vector<uint64_t> rs(T + 1, n_reads);
    {
        const uint64_t nb = offsets[n_reads] - offsets[0];
        uint64_t r = 0;
        for (int t = 0; t <= T; ++t) {
            const uint64_t lim = offsets[0] + (nb * (uint64_t)t) / (uint64_t)T;
            while (r < n_reads && offsets[r] < lim) ++r;
            rs[t] = (t == T) ? n_reads : r;
        }
        rs[0] = 0;
    }
    auto for_windows = [&](int t, auto&& fn) {
        for (uint64_t i = rs[t]; i < rs[t + 1]; ++i) {
            const uint64_t b = offsets[i], e = offsets[i + 1];
            if (e < b + (uint64_t)k) continue;
            for (uint64_t s = b; s + k <= e; ++s) {
                const uint8_t* w = reads + (s - offsets[0]);
                if (!window_valid(w, k)) continue;
                fn((K)(canonical ? canonical_value(w, k) : forward_value(w, k)));
            }
        }
    };
    /* 1: window count and a value sample per thread */
    std::vector<std::vector<K>> samp(T);
    std::vector<uint64_t> nwin(T, 0);
    {
        std::vector<std::thread> th;
        for (int t = 0; t < T; ++t)
            th.emplace_back([&, t] {
                uint64_t c = 0;
                for_windows(t, [&](K v) {
                    if (c % SAMPLE == 0) samp[t].push_back(v);
                    ++c;
                });
                nwin[t] = c;
            });
        for (auto& x : th) x.join();
    }
    uint64_t n_windows = 0;
    std::vector<K> all;
    for (int t = 0; t < T; ++t) {
        n_windows += nwin[t];
        all.insert(all.end(), samp[t].begin(), samp[t].end());
        std::vector<K>().swap(samp[t]);
    }
    std::sort(all.begin(), all.end());
    /* 2: ranges -- a multiple of T, each expected to hold about round_keys / T values */
    uint64_t R = (uint64_t)T;
    if (round_keys == 0) round_keys = 1;
    while (R * (round_keys / (uint64_t)T + 1) < n_windows && R < (1ull << 20)) R += (uint64_t)T;
    std::vector<K> bound;  /* lower bounds of ranges 1..R-1 (range 0 starts at the minimum) */
    for (uint64_t j = 1; j < R && !all.empty(); ++j) {
        const K b = all[(size_t)((all.size() * j) / R)];
        if (bound.empty() || bound.back() < b) bound.push_back(b);
    }
    std::vector<K>().swap(all);
    const uint64_t NR = bound.size() + 1; /* distinct ranges */
    auto range_of = [&](K v) { return (uint64_t)(std::upper_bound(bound.begin(), bound.end(), v) - bound.begin()); };
    /* 3: rounds of T ranges */
    uint64_t n_unique = 0, n_below = 0, n_above = 0, n_out = 0;
    std::vector<uint64_t> ok;  /* survivors: 1 or 2 words per key, as in oracle_count */
    std::vector<uint32_t> oc;
    for (uint64_t r0 = 0; r0 < NR; r0 += (uint64_t)T) {
        const uint64_t r1 = std::min<uint64_t>(NR, r0 + (uint64_t)T);
        const int nr = (int)(r1 - r0);
        std::vector<std::vector<std::vector<K>>> part(T, std::vector<std::vector<K>>(nr));
        {
            std::vector<std::thread> th;
            for (int t = 0; t < T; ++t)
                th.emplace_back([&, t] {
                    for_windows(t, [&](K v) {
                        const uint64_t j = range_of(v);
                        if (j >= r0 && j < r1) part[t][j - r0].push_back(v);
                    });
                });
            for (auto& x : th) x.join();
        }
        /* per range: sort + count equal neighbours (thread j - r0 owns range j) */
        struct RangeOut {
            std::vector<K> keys;
            std::vector<uint32_t> counts;
            uint64_t uniq = 0, below = 0, above = 0;
        };
        std::vector<RangeOut> ro(nr);
        {
            std::vector<std::thread> th;
            for (int q = 0; q < nr; ++q)
                th.emplace_back([&, q] {
                    std::vector<K> keys;
                    size_t tot = 0;
                    for (int t = 0; t < T; ++t) tot += part[t][q].size();
                    keys.reserve(tot);
                    for (int t = 0; t < T; ++t) {
                        keys.insert(keys.end(), part[t][q].begin(), part[t][q].end());
                        std::vector<K>().swap(part[t][q]);
                    }
                    std::sort(keys.begin(), keys.end());
                    RangeOut& o = ro[q];
                    for (size_t a = 0; a < keys.size();) {
                        size_t z = a;
                        while (z < keys.size() && keys[z] == keys[a]) ++z;
                        const uint64_t c = z - a;
                        ++o.uniq;
                        if (c < ci) ++o.below;
                        else if (c > cx) ++o.above;
                        else {
                            o.keys.push_back(keys[a]);
                            o.counts.push_back((uint32_t)(c > 0xFFFFFFFFull ? 0xFFFFFFFFull : c));
                        }
                        a = z;
                    }
                });
            for (auto& x : th) x.join();
        }
        for (int q = 0; q < nr; ++q) {
            RangeOut& o = ro[q];
            n_unique += o.uniq;
            n_below += o.below;
            n_above += o.above;
            for (size_t i = 0; i < o.keys.size(); ++i, ++n_out) {
                const u128 v = (u128)o.keys[i];
                ok.push_back((uint64_t)v);
                if (sizeof(K) == 16) ok.push_back((uint64_t)(v >> 64));
                oc.push_back(o.counts[i]);
            }
            std::vector<K>().swap(o.keys);
            std::vector<uint32_t>().swap(o.counts);
        }
    }
    /* exactly-sized outputs, released by oracle_free */
    *out_keys = (uint64_t*)malloc(std::max<size_t>(1, ok.size()) * 8);
    *out_counts = (uint32_t*)malloc(std::max<size_t>(1, oc.size()) * 4);
    if (!ok.empty()) memcpy(*out_keys, ok.data(), ok.size() * 8);
    if (!oc.empty()) memcpy(*out_counts, oc.data(), oc.size() * 4);
    if (stats) {
        stats[0] = n_windows; stats[1] = n_unique; stats[2] = n_below; stats[3] = n_above; stats[4] = n_out;
    }
    return (int64_t)n_out;
}

extern "C" {

/* Key-range-partitioned, multi-threaded oracle_count (same outputs and stats; see
 * count_par_impl).  threads: host threads (>= 1); round_keys: values held in memory per
 * round (bounds RAM at about 2 x round_keys x key bytes).  *out_keys / *out_counts are
 * malloc'd with exactly n_out entries (keys: 1 or 2 words each); free with oracle_free. */
int64_t oracle_count_par(const uint8_t* reads, const uint64_t* offsets, uint64_t n_reads, int k, uint32_t ci,
                         uint32_t cx, uint64_t** out_keys, uint32_t** out_counts, uint64_t* stats, int canonical,
                         int threads, uint64_t round_keys) {
    if (k < 1 || k > 64) return -1;
    if (k <= 32)
        return count_par_impl<uint64_t>(reads, offsets, n_reads, k, ci, cx, out_keys, out_counts, stats, canonical,
                                        threads, round_keys);
    return count_par_impl<u128>(reads, offsets, n_reads, k, ci, cx, out_keys, out_counts, stats, canonical,
                                threads, round_keys);
}

void oracle_free(void* p) { free(p); }

/* Exact sorted (canonical k-mer, count) list with cutoffs.
 * reads: host ASCII bytes; read i = reads[offsets[i]-offsets[0] .. offsets[i+1]-offsets[0]).
 * out_keys: 1 uint64 per k-mer if k <= 32, else 2 (lo, hi).  Writes at most cap pairs;
 * returns the number of survivors (may exceed cap).  stats[5] = n_windows, n_unique,
 * n_below_min, n_above_max, n_out.  Returns -1 on bad k. */
int64_t oracle_count(const uint8_t* reads, const uint64_t* offsets, uint64_t n_reads, int k,
                     uint32_t ci, uint32_t cx, uint64_t* out_keys, uint32_t* out_counts,
                     uint64_t cap, uint64_t* stats) {
    if (k < 1 || k > 64) return -1;
    if (k <= 32) return count_impl<uint64_t>(reads, offsets, n_reads, k, ci, cx, out_keys, out_counts, cap, stats, 1);
    return count_impl<u128>(reads, offsets, n_reads, k, ci, cx, out_keys, out_counts, cap, stats, 1);
}

/* Same with canonical = 0: forward k-mers as they occur in the reads (-b). */
int64_t oracle_count_ex(const uint8_t* reads, const uint64_t* offsets, uint64_t n_reads, int k,
                        uint32_t ci, uint32_t cx, uint64_t* out_keys, uint32_t* out_counts,
                        uint64_t cap, uint64_t* stats, int canonical) {
    if (k < 1 || k > 64) return -1;
    if (k <= 32)
        return count_impl<uint64_t>(reads, offsets, n_reads, k, ci, cx, out_keys, out_counts, cap, stats, canonical);
    return count_impl<u128>(reads, offsets, n_reads, k, ci, cx, out_keys, out_counts, cap, stats, canonical);
}

/* Number of valid k-windows (upper bound for the survivor list). */
uint64_t oracle_n_windows(const uint8_t* reads, const uint64_t* offsets, uint64_t n_reads, int k) {
    uint64_t n = 0;
    for (uint64_t i = 0; i < n_reads; ++i)
        for (uint64_t s = offsets[i]; s + k <= offsets[i + 1]; ++s)
            if (window_valid(reads + (s - offsets[0]), k)) ++n;
    return n;
}

/* Occurrence counts of given canonical keys (sampled parity at full size):
 * for each query q (sorted ascending, 1 or 2 words per key as in oracle_count),
 * count[q] = number of valid windows whose canonical value equals q. */
void oracle_count_queries(const uint8_t* reads, const uint64_t* offsets, uint64_t n_reads, int k,
                          const uint64_t* queries, uint64_t nq, uint64_t* out_counts) {
    std::vector<u128> q(nq);
    for (uint64_t i = 0; i < nq; ++i)
        q[i] = (k <= 32) ? (u128)queries[i] : ((u128)queries[2 * i + 1] << 64) | (u128)queries[2 * i];
    std::memset(out_counts, 0, nq * sizeof(uint64_t));
    /* reads are independent; threads own disjoint read ranges and private counters */
#pragma omp parallel
    {
        std::vector<uint64_t> local(nq, 0);
#pragma omp for schedule(dynamic, 4096)
        for (int64_t i = 0; i < (int64_t)n_reads; ++i) {
            for (uint64_t s = offsets[i]; s + k <= offsets[i + 1]; ++s) {
                const uint8_t* w = reads + (s - offsets[0]);
                if (!window_valid(w, k)) continue;
                u128 v = canonical_value(w, k);
                auto it = std::lower_bound(q.begin(), q.end(), v);
                if (it != q.end() && *it == v) ++local[it - q.begin()];
            }
        }
#pragma omp critical
        for (uint64_t j = 0; j < nq; ++j) out_counts[j] += local[j];
    }
}

/* Number of valid windows, in parallel over reads (a checker for full-size runs). */
uint64_t oracle_n_windows_par(const uint8_t* reads, const uint64_t* offsets, uint64_t n_reads, int k) {
    uint64_t n = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(+ : n)
    for (int64_t i = 0; i < (int64_t)n_reads; ++i)
        for (uint64_t s = offsets[i]; s + k <= offsets[i + 1]; ++s)
            if (window_valid(reads + (s - offsets[0]), k)) ++n;
    return n;
}

/* Signature rule of Sec. 2.2, applied to the CANONICAL m-mer c[0..m)
 * (reading R1): not starting with AAA, not starting with ACA, and no AA at any
 * position j >= 1 (reading R2: "AA anywhere except at their beginning"). */
int oracle_allowed_codes(const int* c, int m) {
    if (m >= 3 && c[0] == 0 && c[1] == 0 && c[2] == 0) return 0; /* AAA prefix */
    if (m >= 3 && c[0] == 0 && c[1] == 1 && c[2] == 0) return 0; /* ACA prefix */
    for (int j = 1; j + 1 < m; ++j)
        if (c[j] == 0 && c[j + 1] == 0) return 0;                 /* AA not at the beginning */
    return 1;
}

/* Allowed test on an m-mer index (base-4, leftmost most significant). */
int oracle_allowed_index(uint64_t idx, int m) {
    int c[32];
    for (int j = m - 1; j >= 0; --j) { c[j] = (int)(idx & 3); idx >>= 2; }
    return oracle_allowed_codes(c, m);
}

/* Signature of the window w[0..k) with signature length p (Sec. 2.2, P:L206-208;
 * Suppl. Sec. 4 P:L1506 "the smallest 5-mer which satisfies conditions of being a
 * signature"): min over the k-p+1 p-mers of (canonical p-mer value if it is
 * allowed, else the reserved value 4^p (reading R4)).  rules=0 gives the plain
 * canonical minimizer for the Fig. 1 minimizer panel. */
static uint64_t window_signature(const uint8_t* w, int k, int p, int rules) {
    uint64_t reserved = 1ull << (2 * p);
    uint64_t best = reserved;
    int c[32];
    for (int j = 0; j + p <= k; ++j) {
        u128 v = canonical_value(w + j, p);
        uint64_t x = (uint64_t)v;
        for (int t = p - 1; t >= 0; --t) { c[t] = (int)(x & 3); x >>= 2; }
        uint64_t key = (!rules || oracle_allowed_codes(c, p)) ? (uint64_t)v : reserved;
        if (key < best) best = key;
    }
    return best;
}

/* Per-position signatures: out[s - offsets[0]] = signature of the window starting at
 * global position s if that window is valid (inside one read, all ACGT), else
 * 0xFFFFFFFF.  out has offsets[n_reads]-offsets[0] entries. */
void oracle_signatures(const uint8_t* reads, const uint64_t* offsets, uint64_t n_reads, int k, int p,
                       int rules, uint32_t* out) {
    uint64_t n = offsets[n_reads] - offsets[0];
    for (uint64_t i = 0; i < n; ++i) out[i] = 0xFFFFFFFFu;
    for (uint64_t i = 0; i < n_reads; ++i) {
        for (uint64_t s = offsets[i]; s + k <= offsets[i + 1]; ++s) {
            const uint8_t* w = reads + (s - offsets[0]);
            if (!window_valid(w, k)) continue;
            out[s - offsets[0]] = (uint32_t)window_signature(w, k, p, rules);
        }
    }
}

/* Super-k-mers (Fig. 1; reading R5): maximal runs of consecutive
 * valid windows of one read with equal signature.  Writes (start position, number of
 * windows, signature) triples; returns the number of super-k-mers (writes at most cap). */
uint64_t oracle_superkmers(const uint8_t* reads, const uint64_t* offsets, uint64_t n_reads, int k, int p,
                           int rules, uint64_t* out_start, uint32_t* out_nwin, uint32_t* out_sig, uint64_t cap) {
    uint64_t n = 0;
    for (uint64_t i = 0; i < n_reads; ++i) {
        uint64_t prev_sig = ~0ull;
        bool in_run = false;
        for (uint64_t s = offsets[i]; s + k <= offsets[i + 1]; ++s) {
            const uint8_t* w = reads + (s - offsets[0]);
            if (!window_valid(w, k)) { in_run = false; continue; }
            uint64_t sg = window_signature(w, k, p, rules);
            if (in_run && sg == prev_sig) {
                if (n - 1 < cap) out_nwin[n - 1] += 1;
            } else {
                if (n < cap) { out_start[n] = s; out_nwin[n] = 1; out_sig[n] = (uint32_t)sg; }
                ++n;
                in_run = true;
                prev_sig = sg;
            }
        }
    }
    return n;
}

/* Number of (k,x)-mers (Sec. 2.3) the super-k-mers of the reads break into: per
 * super-k-mer (as oracle_superkmers), the k-mers left to right are cut greedily into runs of at
 * most x+1 consecutive k-mers of one orientation (forward: f < r; reverse: f > r; a palindrome
 * f == r joins the run in progress and starts a run as forward -- reading R-KX).  With the
 * number of valid windows this is Table 7's "sorted fraction". */
uint64_t oracle_kx_count(const uint8_t* reads, const uint64_t* offsets, uint64_t n_reads, int k, int p, int x,
                         int rules) {
    uint64_t n_rec = 0;
    for (uint64_t i = 0; i < n_reads; ++i) {
        uint64_t prev_sig = ~0ull;
        bool in_run = false;  /* inside a super-k-mer */
        int run_o = 0, run_len = 0;
        for (uint64_t s = offsets[i]; s + k <= offsets[i + 1]; ++s) {
            const uint8_t* w = reads + (s - offsets[0]);
            if (!window_valid(w, k)) { in_run = false; continue; }
            const uint64_t sg = window_signature(w, k, p, rules);
            const u128 f = forward_value(w, k), r = revcomp_value(w, k);
            const int o = f < r ? 0 : (f > r ? 1 : 2);
            if (!(in_run && sg == prev_sig)) {  /* a new super-k-mer: a new (k,x)-mer */
                in_run = true;
                prev_sig = sg;
                run_o = (o == 2) ? 0 : o;
                run_len = 1;
                ++n_rec;
                continue;
            }
            if (run_len <= x && (o == run_o || o == 2)) {
                ++run_len;
            } else {
                run_o = (o == 2) ? 0 : o;
                run_len = 1;
                ++n_rec;
            }
        }
    }
    return n_rec;
}

}  /* extern "C" */
