/*
 * synth/gen.c -- seeded synthetic read generator (shared INPUT module).
 *
 * This file holds NO arithmetic of the counting method: no k-mers, no
 * canonical forms, no signatures.  It only draws genomes and reads with the
 * shapes of the paper's workloads (Table 1: 100-101 bp
 * Illumina reads at 30-44x; SURVEY.md section 8(d) for the five config
 * recipes).  Both the CUDA path (bench, GPU tests) and the CPU oracle (tests)
 * consume its output; neither side depends on the other.
 *
 * Determinism: every random draw comes from xoshiro256** streams seeded by
 * splitmix64.  Genome stream = seed_genome; read-length stream = seed_reads+1;
 * read content for block b of READS_PER_BLOCK reads = stream seeded with
 * (seed_reads, b).  Output is therefore independent of the thread count.
 */
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct { uint64_t s[4]; } rng_t;

static uint64_t splitmix64(uint64_t* x) {
    uint64_t z = (*x += 0x9E3779B97F4A7C15ull);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}
static void rng_seed(rng_t* r, uint64_t seed) {
    uint64_t x = seed;
    for (int i = 0; i < 4; ++i) r->s[i] = splitmix64(&x);
}
static inline uint64_t rotl(uint64_t x, int k) { return (x << k) | (x >> (64 - k)); }
static inline uint64_t rng_next(rng_t* r) {
    uint64_t* s = r->s;
    uint64_t result = rotl(s[1] * 5, 7) * 9;
    uint64_t t = s[1] << 17;
    s[2] ^= s[0]; s[3] ^= s[1]; s[1] ^= s[2]; s[0] ^= s[3];
    s[2] ^= t; s[3] = rotl(s[3], 45);
    return result;
}
/* uniform integer in [0, n) (n > 0), multiply-shift (bias < 2^-32 for our n) */
static inline uint64_t rng_below(rng_t* r, uint64_t n) {
    return (uint64_t)(((unsigned __int128)rng_next(r) * n) >> 64);
}
/* uniform double in [0,1) */
static inline double rng_unif(rng_t* r) { return (rng_next(r) >> 11) * (1.0 / 9007199254740992.0); }

static const char BASES[4] = {'A', 'C', 'G', 'T'};

/* A draw of one base with P(C)=P(G)=gc/2, P(A)=P(T)=(1-gc)/2, from 16 random bits. */
static inline char base_from16(uint32_t u16, uint32_t tA, uint32_t tC, uint32_t tG) {
    if (u16 < tA) return 'A';
    if (u16 < tC) return 'C';
    if (u16 < tG) return 'G';
    return 'T';
}

/* Strand flip used by the read model: the reverse strand of a DNA string is
 * its reverse, with each base replaced by its Watson-Crick partner.  This is
 * the sequencing model (reads come from both strands), applied
 * to ASCII letters; it is not the counting method's key arithmetic. */
static inline char partner(char c) {
    switch (c) { case 'A': return 'T'; case 'C': return 'G'; case 'G': return 'C'; case 'T': return 'A'; default: return c; }
}

typedef struct {
    uint64_t genome_len;
    double gc;
    /* repeat families: n_fam families of fam_len bp, each placed copies times, per-copy divergence */
    uint64_t n_fam, fam_copies, fam_len;
    double fam_div;
    /* low-complexity tracts: fraction of the genome, length U[tract_min, tract_max], half poly-A, half (AT)n */
    double tract_frac;
    uint64_t tract_min, tract_max;
    uint64_t seed_genome;
} genome_params;

typedef struct {
    uint64_t n_reads;
    uint64_t len_min, len_max;   /* uniform read length in [len_min, len_max] */
    double err;                  /* iid substitution rate */
    double n_iid;                /* iid probability a base is replaced by 'N' */
    double n_run_start;          /* per-position probability an N run starts */
    uint64_t n_run_min, n_run_max;
    int both_strands;
    uint64_t seed_reads;
} read_params;

/* Fill genome[0..genome_len) with uppercase ACGT. */
void synth_genome(const genome_params* P, uint8_t* genome) {
    rng_t r;
    rng_seed(&r, P->seed_genome);
    uint64_t G = P->genome_len;
    double at = (1.0 - P->gc) / 2.0, cg = P->gc / 2.0;
    uint32_t tA = (uint32_t)(at * 65536.0), tC = (uint32_t)((at + cg) * 65536.0), tG = (uint32_t)((at + 2 * cg) * 65536.0);
    uint64_t i = 0;
    while (i < G) {
        uint64_t x = rng_next(&r);
        for (int j = 0; j < 4 && i < G; ++j, ++i) genome[i] = (uint8_t)base_from16((uint32_t)(x >> (16 * j)) & 0xFFFF, tA, tC, tG);
    }
    /* repeat families: consensus drawn with the same composition, copies diverged and oriented at random */
    if (P->n_fam && P->fam_len && P->fam_len < G) {
        char* cons = (char*)malloc(P->fam_len);
        char* copy = (char*)malloc(P->fam_len);
        for (uint64_t f = 0; f < P->n_fam; ++f) {
            for (uint64_t j = 0; j < P->fam_len; ++j) cons[j] = base_from16((uint32_t)(rng_next(&r) & 0xFFFF), tA, tC, tG);
            for (uint64_t c = 0; c < P->fam_copies; ++c) {
                for (uint64_t j = 0; j < P->fam_len; ++j) {
                    char b = cons[j];
                    if (rng_unif(&r) < P->fam_div) b = BASES[((b == 'A' ? 0 : b == 'C' ? 1 : b == 'G' ? 2 : 3) + 1 + rng_below(&r, 3)) & 3];
                    copy[j] = b;
                }
                int rev = (int)(rng_next(&r) & 1);
                uint64_t pos = rng_below(&r, G - P->fam_len + 1);
                for (uint64_t j = 0; j < P->fam_len; ++j)
                    genome[pos + j] = (uint8_t)(rev ? partner(copy[P->fam_len - 1 - j]) : copy[j]);
            }
        }
        free(cons);
        free(copy);
    }
    /* low-complexity tracts */
    if (P->tract_frac > 0 && P->tract_max >= P->tract_min && P->tract_max < G) {
        uint64_t target = (uint64_t)(P->tract_frac * (double)G), placed = 0, t = 0;
        while (placed < target) {
            uint64_t L = P->tract_min + rng_below(&r, P->tract_max - P->tract_min + 1);
            uint64_t pos = rng_below(&r, G - L + 1);
            if ((t++ & 1) == 0) {
                for (uint64_t j = 0; j < L; ++j) genome[pos + j] = 'A';
            } else {
                for (uint64_t j = 0; j < L; ++j) genome[pos + j] = (j & 1) ? 'T' : 'A';
            }
            placed += L;
        }
    }
}

/* Read lengths -> offsets[0..n_reads] (offsets[0] = 0).  Returns total bases. */
uint64_t synth_offsets(const read_params* R, uint64_t* offsets) {
    rng_t r;
    rng_seed(&r, R->seed_reads + 1);
    offsets[0] = 0;
    uint64_t span = R->len_max - R->len_min + 1;
    for (uint64_t i = 0; i < R->n_reads; ++i) {
        uint64_t L = R->len_min + (span > 1 ? rng_below(&r, span) : 0);
        offsets[i + 1] = offsets[i] + L;
    }
    return offsets[R->n_reads];
}

#define READS_PER_BLOCK 4096

/* Sample reads from genome[0..G) into reads[] at offsets[] (from synth_offsets). */
void synth_reads(const read_params* R, const uint8_t* genome, uint64_t G, const uint64_t* offsets, uint8_t* reads, int n_threads) {
    uint64_t n_blocks = (R->n_reads + READS_PER_BLOCK - 1) / READS_PER_BLOCK;
    uint64_t err_t = (uint64_t)(R->err * 4294967296.0);
    uint64_t n_t = (uint64_t)(R->n_iid * 1048576.0);
    double run_p = R->n_run_start;
#ifdef _OPENMP
    if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 4)
#endif
    for (int64_t b = 0; b < (int64_t)n_blocks; ++b) {
        rng_t r;
        rng_seed(&r, R->seed_reads * 0x100000001B3ull + (uint64_t)b * 0x9E3779B97F4A7C15ull + 7);
        uint64_t i0 = (uint64_t)b * READS_PER_BLOCK, i1 = i0 + READS_PER_BLOCK;
        if (i1 > R->n_reads) i1 = R->n_reads;
        for (uint64_t i = i0; i < i1; ++i) {
            uint64_t L = offsets[i + 1] - offsets[i];
            uint8_t* out = reads + offsets[i];
            if (L == 0) continue;
            uint64_t start = (G > L) ? rng_below(&r, G - L + 1) : 0;
            int rev = R->both_strands ? (int)(rng_next(&r) & 1) : 0;
            for (uint64_t j = 0; j < L; ++j) {
                uint64_t src = start + j;
                char c = (src < G) ? (char)genome[rev ? (start + L - 1 - j) : src] : 'A';
                if (rev) c = partner(c);
                uint64_t x = rng_next(&r);
                if ((x & 0xFFFFFFFFull) < err_t) {
                    int code = (c == 'A' ? 0 : c == 'C' ? 1 : c == 'G' ? 2 : 3);
                    c = BASES[(code + 1 + (int)(((x >> 52) & 0xFFF) % 3)) & 3];
                }
                if (((x >> 32) & 0xFFFFF) < n_t) c = 'N';
                out[j] = (uint8_t)c;
            }
            if (run_p > 0) {
                for (uint64_t j = 0; j < L; ++j) {
                    if (rng_unif(&r) < run_p) {
                        uint64_t rl = R->n_run_min + rng_below(&r, R->n_run_max - R->n_run_min + 1);
                        for (uint64_t t = 0; t < rl && j + t < L; ++t) out[j + t] = 'N';
                    }
                }
            }
        }
    }
}
