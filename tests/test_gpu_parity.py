"""GPU parity (-m gpu): the CUDA path through the C ABI vs the CPU oracle, element by element.

Bit-exact is the bar everywhere (integer keys and counts).  Small, reduced and full-size
configs are all compared in full (full-size C4 through the oracle's digest).
"""
import json
import os
import random

import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


def to_dev(w):
    r = torch.from_numpy(w.reads).cuda() if w.reads.size else torch.zeros(0, dtype=torch.uint8, device="cuda")
    o = torch.from_numpy(w.offsets.view(np.uint64)).cuda()
    return r, o


def gpu_count(kmc, w, k=None, p=None, ci=None, cx=None, **kw):
    r, o = to_dev(w)
    res = kmc.count(r, o, k or w.k, p or w.p, w.cutoff_min if ci is None else ci,
                    w.cutoff_max if cx is None else cx, **kw)
    keys = res.kmers.cpu().numpy()
    counts = res.counts.cpu().numpy()
    return keys, counts, res.stats


def assert_same(kmc, w, k=None, p=None, ci=None, cx=None, **kw):
    k = k or w.k
    ci = w.cutoff_min if ci is None else ci
    cx = w.cutoff_max if cx is None else cx
    keys, counts, st = gpu_count(kmc, w, k, p, ci, cx, **kw)
    ref = oracle.count(w.reads, w.offsets, k, ci, cx)
    assert keys.shape[0] == ref.keys.shape[0], (keys.shape, ref.keys.shape)
    assert np.array_equal(keys, ref.keys)
    assert np.array_equal(counts, ref.counts)
    assert st["n_windows"] == ref.n_windows
    assert st["n_unique"] == ref.n_unique
    assert st["n_below_min"] == ref.n_below_min
    assert st["n_above_max"] == ref.n_above_max
    assert st["n_out"] == ref.n_out
    return st


# ---------------------------------------------------------------- S2: signatures

def test_allowed_rule_matches_oracle(gpu):
    for p in range(1, 9):
        dev = gpu.debug_allowed(p)
        ref = np.array([oracle.allowed_index(i, p) for i in range(4 ** p)], dtype=np.uint8)
        assert np.array_equal(dev, ref), p


def _sig_case(gpu, w, k, p):
    r, o = to_dev(w)
    got = gpu.debug_signatures(r, o, k, p).cpu().numpy()
    ref = oracle.signatures(w.reads, w.offsets, k, p, True)
    bad = np.nonzero(got != ref)[0]
    assert bad.size == 0, (k, p, bad[:10], got[bad[:10]], ref[bad[:10]])


def test_signature_fig1_golden(gpu):
    w = synth.from_strings(["CGTTGATCAATTTG"], 8)
    r, o = to_dev(w)
    got = gpu.debug_signatures(r, o, 8, 4).cpu().numpy()
    sig = [oracle.str_value(s) for s in ("AACG", "ATCA", "ATCA", "ATCA", "AATT", "AATT", "AATT")]
    assert got[:7].tolist() == sig and all(x == 0xFFFFFFFF for x in got[7:])


@pytest.mark.parametrize("k,p", [(25, 7), (28, 9), (31, 9), (55, 11), (64, 12), (8, 8), (12, 3), (5, 1), (33, 5), (64, 1), (37, 1), (36, 1), (46, 10),
                                 (28, 13), (40, 14), (31, 15), (15, 15), (64, 15)])
def test_signature_parity_random(gpu, k, p):
    seqs = synth.random_reads(k * 100 + p, 400, 0, 300, n_frac=0.01, lower_frac=0.02)
    _sig_case(gpu, synth.from_strings(seqs, k), k, p)


@pytest.mark.parametrize("name,scale", [("C1", 0.02), ("C5", 0.002), ("C4", 0.0002), ("C3", 0.002)])
def test_signature_parity_configs(gpu, name, scale):
    w = synth.make(name, scale=scale)
    _sig_case(gpu, w, w.k, w.p)


def test_superkmer_count(gpu):
    w = synth.make("C5", scale=0.002)
    _, _, st = gpu_count(gpu, w)
    assert st["n_superkmers"] == len(oracle.superkmers(w.reads, w.offsets, w.k, w.p))


# ---------------------------------------------------------------- end-to-end parity

@pytest.mark.parametrize("name,scale", [("C1", 1.0), ("C2", 0.02), ("C3", 0.02), ("C4", 0.001), ("C5", 0.02)])
def test_count_parity_configs(gpu, name, scale):
    st = assert_same(gpu, synth.make(name, scale=scale))
    assert st["n_superkmers"] > 0 and st["n_bins"] > 0


@pytest.mark.parametrize("opts", [dict(force_large=True), dict(small_bin_capacity=64), dict(small_bin_capacity=1024),
                                  dict(large_path=1), dict(force_large=True, large_path=1),
                                  dict(distribute_path=1), dict(count_path=1),
                                  dict(force_large=True, count_path=1), dict(force_large=True, large_path=2),
                                  dict(force_large=True, large_path=3, cluster_size=4, table_keys=100),
                                  dict(force_large=True, large_path=3, cluster_size=1)])
def test_forced_paths(gpu, opts):
    w = synth.make("C5", scale=0.005)
    st = assert_same(gpu, w, **opts)
    if opts.get("force_large"):
        assert st["large_windows"] == st["n_windows"]


@pytest.mark.parametrize("name,scale,p", [("C5", 0.005, 13), ("C5", 0.005, 15), ("C4", 0.001, 14), ("C4", 0.001, 15)])
def test_long_signatures(gpu, name, scale, p):
    # p up to 15 (4^15 + 1 signature ids in 32 bits); C4 at 0.001 takes the sampled plan
    assert_same(gpu, synth.make(name, scale=scale), p=p)


def test_p_invariance(gpu):
    w = synth.make("C2", scale=0.005)
    outs = []
    for p in (3, 5, 7, 9, 11, 12, 13, 15):
        keys, counts, _ = gpu_count(gpu, w, p=p)
        outs.append((keys, counts))
    for keys, counts in outs[1:]:
        assert np.array_equal(keys, outs[0][0]) and np.array_equal(counts, outs[0][1])


def test_revcomp_and_permutation_invariance(gpu):
    w = synth.make("C1", scale=0.05)
    seqs = [bytes(w.reads[w.offsets[i]:w.offsets[i + 1]]).decode() for i in range(w.n_reads)]
    rnd = random.Random(3)
    flipped = [oracle.revcomp_str(s) if rnd.random() < 0.5 else s for s in seqs]
    rnd.shuffle(flipped)
    w2 = synth.from_strings(flipped, w.k, w.p, 1)
    a = gpu_count(gpu, w, ci=1)
    b = gpu_count(gpu, w2, ci=1)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


@pytest.mark.parametrize("force_large", [False, True])
@pytest.mark.parametrize("k", [1, 2, 3, 15, 16, 17, 31, 32, 33, 47, 63, 64])
def test_k_boundaries(gpu, k, force_large):
    p = min(k, 5)
    seqs = synth.random_reads(k, 600, 0, 200, n_frac=0.01, lower_frac=0.01, alphabet=b"ACGT")
    assert_same(gpu, synth.from_strings(seqs, k, p, 1), force_large=force_large)


def test_chunk_hash_overflow_fallback(gpu):
    # distinct-heavy large bins (random reads, no coverage) with a distinct ratio measured on
    # low-coverage small bins: chunks sized for repeats overflow the table and must fall back
    seqs = synth.random_reads(77, 6000, 100, 150, alphabet=b"ACGT")
    w = synth.from_strings(seqs, 25, 5, 1)
    st = assert_same(gpu, w, force_large=True, chunk_capacity=60000, large_path=2)
    assert st["large_windows"] > 0 and st["n_overflow_chunks"] > 0
    st = assert_same(gpu, w, force_large=True, large_path=2)
    assert st["n_overflow_chunks"] == 0
    # the sort path clamps an oversize chunk capacity to its shared-memory array
    st = assert_same(gpu, w, force_large=True, count_path=1, chunk_capacity=60000)
    assert st["chunk_capacity"] <= 6144


@pytest.mark.parametrize("name,scale,opts", [("C2", 0.005, {}), ("C5", 0.004, {}), ("C4", 0.001, {}),
                                             ("C1", 0.1, dict(chunk_capacity=2000)), ("C2", 0.004, dict(canonical=False))])
def test_split_region_overflow(gpu, name, scale, opts):
    """One-pass split with regions of exactly the mean digit size: digits overflow, their excess
    keys go to the overflow list and the overflowed digits (region part + excess) are counted
    by the device radix-sort fallback -- same bytes as the oracle."""
    w = synth.make(name, scale=scale)
    opts = dict(opts)
    opts.setdefault("chunk_capacity", 512)  # many digits per bin
    keys, counts, st = gpu_count(gpu, w, force_large=True, split_tight=True, **opts)
    ref = oracle.count(w.reads, w.offsets, w.k, w.cutoff_min, w.cutoff_max, canonical=opts.get("canonical", True))
    assert np.array_equal(keys, ref.keys) and np.array_equal(counts, ref.counts)
    assert st["n_split_overflow"] > 0


# ---------------------------------------------------------------- large bins by thread-block clusters

@pytest.mark.parametrize("cluster_size", [1, 4, 8, 16])
@pytest.mark.parametrize("table_keys", [0, 40, 3000])
def test_cluster_path(gpu, cluster_size, table_keys):
    """Large bins counted by clusters of 1-16 CTAs (keys routed to their owner CTA through
    distributed shared memory); small table_keys plans many rounds per bin and cluster items
    whose slices hold fewer records than CTAs."""
    w = synth.make("C2", scale=0.003)
    st = assert_same(gpu, w, force_large=True, large_path=3, cluster_size=cluster_size, table_keys=table_keys)
    assert st["cluster_size"] == cluster_size and st["large_windows"] == st["n_windows"]
    if cluster_size > 1 and table_keys == 40:
        assert st["n_cluster_items"] > 0


@pytest.mark.parametrize("k", [12, 25, 28, 29, 30, 31, 32])
def test_cluster_path_units(gpu, k):
    # every expansion unit width (4 windows for k <= 29, 33 - k above) and records up to maxw
    seqs = ["A" * 400, "AC" * 200] * 20 + [s.decode() for s in synth.random_reads(k, 1500, 30, 300, n_frac=0.01)]
    assert_same(gpu, synth.from_strings(seqs, k, 5, 1), force_large=True, large_path=3, cluster_size=8, table_keys=50)


def test_cluster_spill_and_fallback(gpu):
    # distinct-heavy bins far above one table (p = 3: a few huge signatures, random reads):
    # single-CTA tables overfill, the keys that find no slot are spilled and counted by the
    # device radix sort; a spill list too small for them reruns the large bins on the split path
    seqs = synth.random_reads(5, 8000, 100, 150, alphabet=b"ACGT")
    w = synth.from_strings(seqs, 25, 3, 1)
    st = assert_same(gpu, w, force_large=True, large_path=3, cluster_size=1, spill_keys=1 << 24)
    assert st["n_spilled_keys"] > 0
    st = assert_same(gpu, w, force_large=True, large_path=3, cluster_size=1, spill_keys=1000)
    assert st["n_spilled_keys"] > 1000  # overflowed -> split path
    st = assert_same(gpu, w, force_large=True, large_path=3, cluster_size=16)
    assert st["n_cluster_items"] > 0


def test_small_bin_hash_and_sort_fallback(gpu):
    # small bins are counted in a shared-memory hash table; bins whose distinct keys overfill
    # it (random reads: nearly every k-mer distinct, bins near the small capacity) are
    # sorted instead.  Both in one call, both exact.
    seqs = synth.random_reads(91, 20000, 80, 120, alphabet=b"ACGT")
    for k, p in [(25, 5), (25, 6), (40, 5)]:
        w = synth.from_strings(seqs, k, p, 1)
        st = assert_same(gpu, w)
        assert st["n_small_sorted"] > 0 and st["n_small_sorted"] < st["n_bins"], st
    # repeats: every small bin by the table
    st = assert_same(gpu, synth.make("C2", scale=0.01))
    assert st["n_small_sorted"] == 0 and st["n_bins"] > st["n_large_bins"]


@pytest.mark.parametrize("large_path,count_path", [(3, 0), (0, 0), (0, 1)])
@pytest.mark.parametrize("name,scale", [("C3", 0.005), ("C2", 0.005), ("C1", 0.2)])
def test_chunk_count_paths(gpu, name, scale, large_path, count_path):
    # every bin through the large path: cluster tables (large_path 3, k <= 32), or the hashed
    # split and per-chunk SMEM hash count (count_path 0) or SMEM radix sort + run-length
    # compaction (count_path 1)
    st = assert_same(gpu, synth.make(name, scale=scale), force_large=True, count_path=count_path,
                     large_path=large_path)
    assert st["large_windows"] == st["n_windows"]


def test_split_piece_and_range_modes(gpu):
    # piece-mode bins whose pieces hold more keys than the shared-memory stage (long poly-A /
    # (AC)n super-k-mers: maxw windows per record) next to ordinary ones
    seqs = ["A" * 3000, "AC" * 1500, "ACGTTGCA" * 300] * 40
    seqs += [s.decode() for s in synth.random_reads(21, 3000, 100, 300)]
    assert_same(gpu, synth.from_strings(seqs, 28, 9, 1), force_large=True, large_path=2)
    # tiny chunks: bins with more than 2^8 digits take range mode, the rest piece mode, in
    # the same split launch
    st = assert_same(gpu, synth.make("C2", scale=0.005), force_large=True, chunk_capacity=128, large_path=2)
    assert st["chunk_capacity"] == 128


@pytest.mark.parametrize("large_path,count_path", [(0, 0), (0, 1), (1, 0), (3, 0)])
def test_low_complexity_and_skew(gpu, large_path, count_path):
    # poly-A / (AT)n pile-ups: one k-mer with ~25K copies -> an "oversize" MSD digit
    seqs = ["A" * 300, "T" * 250, "AT" * 120, "ACGT" * 60, "N" * 50, "", "ACG", "CA" * 100] * 50
    seqs += [s.decode() for s in synth.random_reads(9, 200, 50, 250)]
    for k, p in ((31, 9), (28, 7), (55, 11), (21, 3)):
        assert_same(gpu, synth.from_strings(seqs, k, p, 2), large_path=large_path, count_path=count_path)


def test_edge_cases(gpu):
    # empty input
    keys, counts, st = gpu_count(gpu, synth.from_strings([], 25, 7, 1))
    assert keys.shape[0] == 0 and st["n_windows"] == 0
    # all reads shorter than k; all-N
    for seqs in (["ACGT", "ACG", ""], ["N" * 100, "n" * 40]):
        keys, counts, st = gpu_count(gpu, synth.from_strings(seqs, 25, 7, 1))
        assert keys.shape[0] == 0 and st["n_windows"] == 0
    # cutoffs that remove everything
    w = synth.make("C1", scale=0.01)
    keys, counts, st = gpu_count(gpu, w, ci=10**6, cx=10**9)
    assert keys.shape[0] == 0 and st["n_below_min"] == st["n_unique"]
    # cutoff_max removes the frequent ones; ci = 0 treated as 1
    assert_same(gpu, w, ci=0, cx=1)
    # lowercase + non-ACGT bytes
    seqs = synth.random_reads(11, 300, 20, 200, n_frac=0.05, lower_frac=0.3, alphabet=b"ACGTRYacgt")
    assert_same(gpu, synth.from_strings(seqs, 21, 7, 1))


def test_offsets_base_and_misaligned_pointer(gpu):
    w = synth.make("C1", scale=0.01)
    pad = 5
    reads = np.concatenate([np.frombuffer(b"NNNNN", dtype=np.uint8), w.reads])
    r = torch.from_numpy(reads).cuda()[pad:]                      # misaligned device pointer
    o = torch.from_numpy((w.offsets + np.uint64(1000)).view(np.uint64)).cuda()  # offsets[0] != 0
    res = gpu.count(r, o, w.k, w.p, 1, 10**9)
    ref = oracle.count(w.reads, w.offsets, w.k, 1, 10**9)
    assert np.array_equal(res.kmers.cpu().numpy(), ref.keys) and np.array_equal(res.counts.cpu().numpy(), ref.counts)


def test_host_buffers_and_capacity(gpu):
    w = synth.make("C5", scale=0.002)
    rh = torch.from_numpy(w.reads).pin_memory()
    oh = torch.from_numpy(w.offsets.view(np.uint64))
    res = gpu.count(rh, oh, w.k, w.p, 2, 10**9, out_device="cpu")
    ref = oracle.count(w.reads, w.offsets, w.k, 2, 10**9)
    assert np.array_equal(res.kmers.numpy(), ref.keys) and np.array_equal(res.counts.numpy(), ref.counts)
    # one-call form: too small capacity -> KMC_ERR_OUT_CAPACITY with the required count
    r, o = to_dev(w)
    small_k = torch.empty(1, dtype=torch.uint64, device="cuda")
    small_c = torch.empty(1, dtype=torch.uint32, device="cuda")
    with pytest.raises(gpu.KmcError) as ei:
        gpu.count_into(r, o, w.k, w.p, 2, 10**9, small_k, small_c)
    assert ei.value.status == gpu.KMC_ERR_OUT_CAPACITY
    ok_k = torch.empty(ref.n_out, dtype=torch.uint64, device="cuda")
    ok_c = torch.empty(ref.n_out, dtype=torch.uint32, device="cuda")
    st = gpu.count_into(r, o, w.k, w.p, 2, 10**9, ok_k, ok_c)
    assert st["n_out"] == ref.n_out and np.array_equal(ok_k.cpu().numpy(), ref.keys)


def test_invalid_args(gpu):
    w = synth.make("C1", scale=0.001)
    r, o = to_dev(w)
    for k, p, ci, cx in ((0, 1, 1, 10), (65, 9, 1, 10), (25, 16, 1, 10), (12, 13, 1, 10), (5, 7, 1, 10), (25, 7, 5, 4)):
        with pytest.raises(gpu.KmcError) as ei:
            gpu.count(r, o, k, p, ci, cx)
        assert ei.value.status == gpu.KMC_ERR_INVALID_ARG


def test_deterministic(gpu):
    w = synth.make("C5", scale=0.005)
    a = gpu_count(gpu, w)
    b = gpu_count(gpu, w, small_bin_capacity=512)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


# ---------------------------------------------------------------- full-size configs (complete)
# BASELINE.json's five configs at full size, compared in full: C1-C3 and C5 element by element
# against the key-range-partitioned oracle run here (pinned to the plain oracle in
# test_oracle.py), and every config -- C4 included, whose oracle run takes ~10 minutes -- by
# the SHA-256 of the whole sorted (k-mer, count) list and the statistics, written once by
# tools/make_goldens.py from oracle/ alone (tests/golden/full_configs.json).

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "full_configs.json")))["configs"]


def _full(gpu, name, live_oracle):
    w = synth.make(name)
    keys, counts, st = gpu_count(gpu, w)
    g = GOLD[name]
    assert (w.k, w.p, w.cutoff_min, w.cutoff_max, w.n_bases) == (g["k"], g["p"], g["cutoff_min"], g["cutoff_max"],
                                                                   g["n_bases"])
    for f in ("n_windows", "n_unique", "n_below_min", "n_above_max", "n_out"):
        assert st[f] == g[f], (f, st[f], g[f])
    assert int(counts.sum(dtype=np.uint64)) == g["count_sum"]
    assert oracle.digest(keys, counts) == g["sha256"]
    if live_oracle:
        ref = oracle.count_partitioned(w.reads, w.offsets, w.k, w.cutoff_min, w.cutoff_max)
        assert keys.shape == ref.keys.shape
        bad = np.nonzero(np.any((keys != ref.keys).reshape(keys.shape[0], -1), axis=1) | (counts != ref.counts))[0]
        assert bad.size == 0, f"first mismatch at {bad[0]}: gpu {keys[bad[0]]}/{counts[bad[0]]}, " \
                              f"oracle {ref.keys[bad[0]]}/{ref.counts[bad[0]]}"
    return st


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C5"])
def test_full_config_exact(gpu, name):
    _full(gpu, name, live_oracle=True)


def test_full_c4_exact(gpu):
    st = _full(gpu, "C4", live_oracle=False)
    assert st["n_windows"] > 2_500_000_000


@pytest.mark.parametrize("opts", [dict(count_path=1), dict(distribute_path=1)])
def test_full_c4_other_paths(gpu, opts):
    """The paper's per-chunk radix sort (count_path 1) and the recompute distribution path at
    full C4 size give the same bytes."""
    w = synth.make("C4")
    keys, counts, st = gpu_count(gpu, w, **opts)
    assert st["n_out"] == GOLD["C4"]["n_out"] and oracle.digest(keys, counts) == GOLD["C4"]["sha256"]


# ---------------------------------------------------------------- f2: streamed input, bounded groups

@pytest.mark.parametrize("opts", [dict(input_batch_mb=1), dict(input_batch_mb=1, distribute_path=1),
                                  dict(input_batch_mb=2, large_group_mkeys=1, force_large=True)])
def test_streamed_host_input(gpu, opts):
    """Host-resident reads streamed through pass 1 in read-aligned batches (double-buffered
    H2D) and large bins in memory-bounded groups give the oracle's bytes exactly."""
    w = synth.make("C4", scale=0.002)  # 8 Mbases -> several 1-2 MiB batches
    rh = torch.from_numpy(w.reads).pin_memory()
    oh = torch.from_numpy(w.offsets.view(np.uint64))
    res = gpu.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu", **opts)
    ref = oracle.count(w.reads, w.offsets, w.k, w.cutoff_min, w.cutoff_max)
    assert res.stats["n_input_batches"] >= 4
    if opts.get("large_group_mkeys"):
        assert res.stats["n_large_groups"] >= 3
    assert np.array_equal(res.kmers.numpy(), ref.keys) and np.array_equal(res.counts.numpy(), ref.counts)
    assert res.stats["n_windows"] == ref.n_windows


def test_streamed_equals_resident(gpu):
    w = synth.make("C5", scale=0.01)
    a = gpu_count(gpu, w)
    rh = torch.from_numpy(w.reads)  # pageable host memory also works
    oh = torch.from_numpy(w.offsets.view(np.uint64))
    b = gpu.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu", input_batch_mb=1,
                  large_group_mkeys=1)
    assert np.array_equal(a[0], b.kmers.numpy()) and np.array_equal(a[1], b.counts.numpy())


# --- -b: non-canonical counting -----------------------------------------------

@pytest.mark.parametrize("name,scale,k,opts", [
    ("C1", 0.02, None, {}), ("C5", 0.002, None, {}), ("C3", 0.002, None, {}), ("C4", 0.0005, None, {}),
    ("C2", 0.005, None, dict(force_large=True)), ("C2", 0.005, None, dict(force_large=True, count_path=1)),
    ("C1", 0.02, None, dict(large_path=1, force_large=True)), ("C1", 0.01, 31, dict(force_large=True)),
    ("C1", 0.01, 33, {}), ("C1", 0.01, 47, dict(force_large=True)), ("C1", 0.01, 12, dict(small_bin_capacity=64))])
def test_noncanonical_parity(gpu, name, scale, k, opts):
    w = synth.make(name, scale=scale) if k is None else synth.make(name, scale=scale, k=k)
    keys, counts, st = gpu_count(gpu, w, canonical=False, **opts)
    ref = oracle.count(w.reads, w.offsets, w.k, w.cutoff_min, w.cutoff_max, canonical=False)
    assert keys.shape[0] == ref.keys.shape[0]
    assert np.array_equal(keys, ref.keys) and np.array_equal(counts, ref.counts)
    assert st["n_windows"] == ref.n_windows and st["n_unique"] == ref.n_unique


def test_noncanonical_low_complexity(gpu):
    seqs = ["T" * 300, "A" * 250, "AT" * 120, "ACGT" * 60, "CA" * 100, "N" * 40, ""] * 30
    for k, p in ((28, 9), (21, 5), (45, 11)):
        w = synth.from_strings(seqs, k, p, 1)
        keys, counts, _ = gpu_count(gpu, w, canonical=False)
        ref = oracle.count(w.reads, w.offsets, k, 1, 10**9, canonical=False)
        assert np.array_equal(keys, ref.keys) and np.array_equal(counts, ref.counts)


def test_noncanonical_rejects_k32(gpu):
    w = synth.from_strings(["ACGT" * 20], 32, 9, 1)
    r, o = to_dev(w)
    with pytest.raises(Exception):
        gpu.count(r, o, 32, 9, 1, 10**9, canonical=False)


# --- Table 6 diagnostic: plain canonical minimizers vs signatures ---------

@pytest.mark.parametrize("k,p", [(28, 5), (28, 7), (55, 8), (21, 9), (12, 3)])
def test_plain_minimizer_signatures(gpu, k, p):
    seqs = synth.random_reads(k * 7 + p, 300, 0, 300, n_frac=0.01)
    seqs += [b"A" * 200, b"ACA" * 50, b"AAT" * 40]
    w = synth.from_strings(seqs, k, p, 1)
    r, o = to_dev(w)
    got = gpu.debug_signatures(r, o, k, p, plain_minimizers=True).cpu().numpy()
    assert np.array_equal(got, oracle.signatures(w.reads, w.offsets, k, p, rules=False))


@pytest.mark.parametrize("rules", [True, False])
@pytest.mark.parametrize("name,scale", [("C1", 0.02), ("C3", 0.002)])
def test_plain_minimizer_counts_and_stats(gpu, name, scale, rules):
    w = synth.make(name, scale=scale)
    keys, counts, st = gpu_count(gpu, w, plain_minimizers=not rules)
    ref = oracle.count(w.reads, w.offsets, w.k, w.cutoff_min, w.cutoff_max)
    assert np.array_equal(keys, ref.keys) and np.array_equal(counts, ref.counts)  # same counts either way
    sig = oracle.signatures(w.reads, w.offsets, w.k, w.p, rules=rules)
    sig = sig[sig != 0xFFFFFFFF]
    assert st["max_signature_windows"] == int(np.bincount(sig).max())
    assert st["n_superkmers"] == len(oracle.superkmers(w.reads, w.offsets, w.k, w.p, rules=rules))


# --- randomized sweep: random k, p, read shapes and options against the oracle -----------

def _mutated_reads(seed, n, L):
    """Reads from a small random genome with repeats, errors and N runs (duplicated k-mers,
    reverse complements, low complexity) -- cheap shapes the configs do not cover."""
    rng = np.random.default_rng(seed)
    G = rng.choice(np.frombuffer(b"ACGT", dtype=np.uint8), size=4000)
    G[1000:1300] = ord("A")                                     # poly-A tract
    G[2000:2400] = np.tile(np.frombuffer(b"AC", dtype=np.uint8), 200)  # (AC)n
    comp = np.zeros(256, dtype=np.uint8)
    for a, b in zip(b"ACGT", b"TGCA"):
        comp[a] = b
    out = []
    for _ in range(n):
        ln = int(rng.integers(1, L + 1))
        st = int(rng.integers(0, len(G) - ln))
        r = G[st:st + ln].copy()
        if rng.random() < 0.5:
            r = comp[r[::-1]]
        err = rng.random(ln) < 0.01
        r[err] = rng.choice(np.frombuffer(b"ACGTN", dtype=np.uint8), size=int(err.sum()))
        if rng.random() < 0.1:
            r = np.where(rng.random(ln) < 0.3, r + 32, r).astype(np.uint8)  # lowercase stretch
        out.append(r.tobytes())
    return out


@pytest.mark.parametrize("seed", list(range(40)))
def test_random_sweep(gpu, seed):
    rng = random.Random(seed)
    k = rng.choice([1, 2, 5, 11, 16, 17, 21, 25, 28, 31, 33, 40, 47, 55, 63, 64])
    p = rng.randint(1, min(k, 12))
    ci = rng.choice([1, 1, 2, 3])
    cx = rng.choice([10**9, 10**9, 50, 7])
    opts = rng.choice([{}, dict(force_large=True), dict(small_bin_capacity=256), dict(force_large=True, count_path=1),
                       dict(force_large=True, chunk_capacity=512, large_path=2), dict(large_path=1, force_large=True),
                       dict(force_large=True, large_path=3, cluster_size=rng.choice([4, 8, 16]),
                            table_keys=rng.choice([8, 100])),
                       dict(force_large=True, large_path=3, cluster_size=1),
                       dict(canonical=False) if k not in (32, 64) else {}, dict(plain_minimizers=True)])
    seqs = _mutated_reads(seed, rng.randint(50, 400), rng.choice([60, 150, 400]))
    w = synth.from_strings(seqs, k, p, ci, cx)
    keys, counts, st = gpu_count(gpu, w, ci=ci, cx=cx, **opts)
    ref = oracle.count(w.reads, w.offsets, k, ci, cx, canonical=opts.get("canonical", True))
    assert keys.shape[0] == ref.keys.shape[0], (seed, k, p, opts)
    assert np.array_equal(keys, ref.keys) and np.array_equal(counts, ref.counts), (seed, k, p, opts)
    assert st["n_windows"] == ref.n_windows and st["n_unique"] == ref.n_unique


# ---------------------------------------------------------------- f1: (k,x)-mers

@pytest.mark.parametrize("x", [1, 2, 3])
@pytest.mark.parametrize("name,scale,k", [("C1", 0.05, None), ("C2", 0.003, None), ("C4", 0.0005, None),
                                          ("C5", 0.002, 27), ("C1", 0.02, 12), ("C1", 0.02, 28)])
def test_kxmer_parity(gpu, x, name, scale, k):
    """Small bins counted through (k,x)-mers -- records split into orientation runs, sorted,
    the sorted sub-arrays merged -- give the plain counts for every x,
    bit for bit against the oracle."""
    w = synth.make(name, scale=scale) if k is None else synth.make(name, scale=scale, k=k)
    st = assert_same(gpu, w, kx=x)
    assert st["kx_windows"] > 0 and 0 < st["n_kxmers"] <= st["kx_windows"]


def test_kxmer_edge_reads(gpu):
    # palindromes (even k), homopolymers, (AT)n, N runs, lowercase, empty and short reads
    seqs = ["A" * 300, "AT" * 120, "ACGT" * 60, "N" * 50, "", "ACG", "CA" * 100, "acgtTGCA" * 30] * 20
    seqs += [s.decode() for s in synth.random_reads(3, 400, 20, 250, n_frac=0.02, lower_frac=0.05)]
    for k, p, x in ((28, 7, 3), (16, 5, 2), (20, 4, 1), (4, 3, 3), (1, 1, 2)):
        assert_same(gpu, synth.from_strings(seqs, k, p, 1), kx=x)


def test_kxmer_sorted_fraction(gpu):
    """Table 7: at x = 3 about half the k-mers remain to be sorted (0.49 printed
    for G. gallus, k = 28).  The GPU's records are super-k-mer pieces (cut at segment edges and
    every maxw windows), so its fraction sits just above the oracle's super-k-mer figure."""
    w = synth.make("C4", scale=0.0005)
    fr = {}
    for x in (1, 2, 3):
        _, _, st = gpu_count(gpu, w, kx=x, small_bin_capacity=4096)
        fr[x] = st["n_kxmers"] / st["kx_windows"]
    ref3 = oracle.kx_count(w.reads, w.offsets, w.k, w.p, 3) / oracle.n_windows(w.reads, w.offsets, w.k)
    assert fr[1] > fr[2] > fr[3]
    assert 0.40 <= fr[3] <= 0.60 and ref3 <= fr[3] <= ref3 + 0.05, (fr, ref3)


def test_kxmer_invalid(gpu):
    w = synth.make("C1", scale=0.001)
    r, o = to_dev(w)
    for k, x, canon in ((25, 4, True), (30, 2, True), (25, 1, False)):
        with pytest.raises(gpu.KmcError) as ei:
            gpu.count(r, o, k, 7, 1, 10**9, kx=x, canonical=canon)
        assert ei.value.status == gpu.KMC_ERR_INVALID_ARG


# ---------------------------------------------------------------- f2: inputs beyond HBM (passes over bin ranges)

@pytest.mark.parametrize("name,scale,opts", [("C4", 0.002, dict(pass_mb=1)), ("C5", 0.004, dict(pass_mb=1)),
                                             ("C3", 0.005, dict(pass_mb=1)), ("C2", 0.004, dict(pass_mb=1, large_path=1)),
                                             ("C1", 0.3, dict(pass_mb=1, count_path=1, force_large=True)),
                                             ("C2", 0.004, dict(pass_mb=1, kx=3)),
                                             ("C4", 0.001, dict(pass_mb=1, input_batch_mb=1))])
def test_multipass_host_input(gpu, name, scale, opts):
    """Host-resident reads counted in passes over ranges of bins (pass 1 builds only the
    histogram; every pass streams the reads again and keeps its bins' records): the oracle's
    bytes, with several passes."""
    w = synth.make(name, scale=scale)
    rh = torch.from_numpy(w.reads).pin_memory()
    oh = torch.from_numpy(w.offsets.view(np.uint64))
    res = gpu.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu", **opts)
    ref = oracle.count(w.reads, w.offsets, w.k, w.cutoff_min, w.cutoff_max)
    assert res.stats["n_passes"] >= 2, res.stats["n_passes"]
    assert np.array_equal(res.kmers.numpy(), ref.keys) and np.array_equal(res.counts.numpy(), ref.counts)
    for f in ("n_windows", "n_unique", "n_below_min", "n_above_max", "n_out"):
        assert res.stats[f] == getattr(ref, f), f


def test_full_c4_host_buffers_digest(gpu):
    """The bench's end-to-end call: host-resident C4 reads in, pinned host outputs out (S9's
    groups sorted depth first and copied while the next group sorts) -- the oracle's digest."""
    w = synth.make("C4")
    rh = torch.from_numpy(w.reads).pin_memory()
    oh = torch.from_numpy(w.offsets.view(np.uint64)).pin_memory()
    res = gpu.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu")
    g = GOLD["C4"]
    assert res.kmers.is_pinned() and res.counts.is_pinned()
    assert res.stats["n_out"] == g["n_out"] and res.stats["n_unique"] == g["n_unique"]
    assert oracle.digest(res.kmers.numpy(), res.counts.numpy()) == g["sha256"]


def test_multipass_full_c4_digest(gpu):
    """The whole C4 read set (4 G bases, host-resident) counted in forced passes of <= 1 GiB of
    records gives exactly the oracle's digest (tests/golden/full_configs.json)."""
    w = synth.make("C4")
    rh = torch.from_numpy(w.reads).pin_memory()
    oh = torch.from_numpy(w.offsets.view(np.uint64))
    res = gpu.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu", pass_mb=1024)
    g = GOLD["C4"]
    assert res.stats["n_passes"] >= 4
    assert res.stats["n_out"] == g["n_out"] and res.stats["n_unique"] == g["n_unique"]
    assert oracle.digest(res.kmers.numpy(), res.counts.numpy()) == g["sha256"]
