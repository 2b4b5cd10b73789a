"""GPU parity of the large-bin path through sub-signatures (large_path 4): bins
above one CTA are cut into digits by a hashed minimizer of length q = min(16, k - 12) of every
window, records are cut into sub-records where the digit changes, and every digit is counted
from its sub-records in one CTA's SMEM hash table (hash-range rounds when it overflows).  The
partition is internal: the output must be the oracle's, byte for byte, on every path --
configs, every k the path takes, -b, digits counted in rounds, block-table overflow (the
device-LSD fallback), memory-bounded groups and host-resident input."""
import numpy as np
import pytest
import torch

import oracle
import synth
from test_gpu_parity import assert_same, gpu_count

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,scale", [("C1", 0.2), ("C2", 0.01), ("C4", 0.002), ("C5", 0.01)])
def test_subsplit_configs(gpu, name, scale):
    st = assert_same(gpu, synth.make(name, scale=scale), large_path=4)
    st = assert_same(gpu, synth.make(name, scale=scale), large_path=4, force_large=True)
    assert st["large_windows"] == st["n_windows"]


@pytest.mark.parametrize("k", list(range(22, 33)))
def test_subsplit_every_k(gpu, k):
    # every q / W2 instantiation (q = k - 12 up to 16, then W2 = k - 15), records of every
    # length up to maxw (poly-A, (AC)n) next to random reads with N and lowercase
    seqs = ["A" * 400, "AC" * 200, "ACGTTGCA" * 50] * 20
    seqs += [s.decode() for s in synth.random_reads(k, 2500, 20, 300, n_frac=0.01, lower_frac=0.01)]
    st = assert_same(gpu, synth.from_strings(seqs, k, 7, 1), force_large=True, large_path=4)
    assert st["large_windows"] == st["n_windows"]


def test_subsplit_noncanonical(gpu):
    for name, scale in (("C2", 0.005), ("C5", 0.004)):
        w = synth.make(name, scale=scale)
        keys, counts, st = gpu_count(gpu, w, canonical=False, force_large=True, large_path=4)
        ref = oracle.count(w.reads, w.offsets, w.k, w.cutoff_min, w.cutoff_max, canonical=False)
        assert np.array_equal(keys, ref.keys) and np.array_equal(counts, ref.counts)
        assert st["n_unique"] == ref.n_unique


def test_subsplit_rounds(gpu):
    # distinct-heavy digits (random reads, no coverage) with digits of 200 K windows: the
    # table overflows and the digits are counted again in 2, 4, .. hash-range rounds
    seqs = synth.random_reads(77, 12000, 100, 150, alphabet=b"ACGT")
    w = synth.from_strings(seqs, 28, 5, 1)
    st = assert_same(gpu, w, force_large=True, large_path=4, chunk_capacity=200000)
    assert st["large_windows"] > 0


def test_subsplit_block_table_overflow(gpu):
    # one k-mer (poly-A) with > SS_MAXB x SS_BLK sub-records in its digit: the excess goes to
    # the overflow list, the digit to the device radix-sort fallback
    seqs = ["A" * 3000] * 1000 + [s.decode() for s in synth.random_reads(3, 3000, 100, 200)]
    w = synth.from_strings(seqs, 28, 9, 2)
    st = assert_same(gpu, w, large_path=4)
    assert st["n_split_overflow"] > 0


def test_subsplit_groups_and_host_input(gpu):
    w = synth.make("C4", scale=0.002)
    rh = torch.from_numpy(w.reads).pin_memory()
    oh = torch.from_numpy(w.offsets.view(np.uint64))
    res = gpu.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu", input_batch_mb=2,
                    large_group_mkeys=1, force_large=True, large_path=4)
    ref = oracle.count(w.reads, w.offsets, w.k, w.cutoff_min, w.cutoff_max)
    assert res.stats["n_large_groups"] >= 3
    assert np.array_equal(res.kmers.numpy(), ref.keys) and np.array_equal(res.counts.numpy(), ref.counts)


def test_subsplit_other_k_falls_back(gpu):
    # k outside [22, 32]: large_path 4 takes the hashed key split
    for k in (21, 33):
        assert_same(gpu, synth.make("C1", scale=0.05, k=k), force_large=True, large_path=4)
