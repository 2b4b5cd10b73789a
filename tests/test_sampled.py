"""GPU parity of the sampled distribution (distribute_path 2, the default for inputs of >= 64 Mi
bases): the bin plan comes from a sample of the reads, pass 1 writes
every record straight into its bin while it counts the exact histograms, and a bin that
overflows its sampled capacity makes the call plan again from the exact histograms.  The plan
never changes the result: the oracle's bytes on every path."""
import numpy as np
import pytest
import torch

import oracle
import synth
from test_gpu_parity import assert_same, gpu_count

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,scale", [("C1", 0.5), ("C2", 0.01), ("C3", 0.01), ("C4", 0.002), ("C5", 0.01)])
def test_sampled_configs(gpu, name, scale):
    w = synth.make(name, scale=scale)
    st = assert_same(gpu, w, distribute_path=2)
    assert st["n_distribute_reruns"] == 0
    ref = oracle.count(w.reads, w.offsets, w.k, 1, 10**9)
    assert st["n_records"] > 0 and st["n_superkmers"] <= st["n_records"]
    # the plan statistics are the exact ones, not the sample's
    st0 = gpu_count(gpu, w, distribute_path=1)[2]
    for f in ("n_windows", "n_records", "n_superkmers", "max_signature_windows", "n_signatures_used",
              "n_invalid_bases"):
        assert st[f] == st0[f], f
    assert st["n_unique"] == ref.n_unique


@pytest.mark.parametrize("opts", [dict(force_large=True), dict(small_bin_capacity=256), dict(canonical=False),
                                  dict(force_large=True, large_path=4), dict(kx=3), dict(count_path=1)])
def test_sampled_paths(gpu, opts):
    w = synth.make("C2", scale=0.005)
    keys, counts, st = gpu_count(gpu, w, distribute_path=2, **opts)
    ref = oracle.count(w.reads, w.offsets, w.k, w.cutoff_min, w.cutoff_max, canonical=opts.get("canonical", True))
    assert np.array_equal(keys, ref.keys) and np.array_equal(counts, ref.counts)


def test_sampled_host_input_batches(gpu):
    w = synth.make("C4", scale=0.003)
    rh = torch.from_numpy(w.reads).pin_memory()
    oh = torch.from_numpy(w.offsets.view(np.uint64))
    res = gpu.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu", input_batch_mb=2,
                    distribute_path=2)
    ref = oracle.count(w.reads, w.offsets, w.k, w.cutoff_min, w.cutoff_max)
    assert res.stats["n_input_batches"] >= 4
    assert np.array_equal(res.kmers.numpy(), ref.keys) and np.array_equal(res.counts.numpy(), ref.counts)


def test_sampled_overflow_reruns(gpu):
    # the sample (the first batch of host reads) misses the rest of the input: 3000 copies of
    # a few reads of a different composition overflow their bins' sampled capacity, and the
    # call plans again from the exact histograms
    first = [s.decode() for s in synth.random_reads(41, 20000, 100, 100, alphabet=b"ACGT")]
    rest = [s.decode() for s in synth.random_reads(42, 5, 150, 150, alphabet=b"ACGT")] * 3000
    w = synth.from_strings(first + rest, 28, 9, 1)
    rh = torch.from_numpy(w.reads).pin_memory()
    oh = torch.from_numpy(w.offsets.view(np.uint64))
    res = gpu.count(rh, oh, w.k, w.p, 1, 10**9, out_device="cpu", input_batch_mb=1, distribute_path=2)
    ref = oracle.count(w.reads, w.offsets, w.k, 1, 10**9)
    assert res.stats["n_distribute_reruns"] == 1
    assert np.array_equal(res.kmers.numpy(), ref.keys) and np.array_equal(res.counts.numpy(), ref.counts)
    # device-resident: the strided sample sees the repeats, no rerun
    st = assert_same(gpu, w, ci=1, cx=10**9, distribute_path=2)
    assert st["n_distribute_reruns"] == 0


def test_sampled_edge_inputs(gpu):
    for seqs, k, p in (([], 25, 7), (["ACGT"], 5, 3), (["A" * 5000] * 10, 28, 9), (["N" * 300] * 20, 21, 5),
                       (["ACGTNNACGTACGT", "acgtacgt", ""] * 50, 8, 4)):
        w = synth.from_strings(seqs, k, p, 1)
        keys, counts, st = gpu_count(gpu, w, distribute_path=2)
        ref = oracle.count(w.reads, w.offsets, k, 1, 10**9)
        assert np.array_equal(keys, ref.keys) and np.array_equal(counts, ref.counts)


# presplit (kmc_options.presplit): the sampled plan's large bins are split into their digit
# regions batch by batch during pass 1 (paired digit layout, pairs counted as one two-segment
# chunk when they fit the table); same bytes as the oracle on every route through it
@pytest.mark.parametrize("opts", [dict(), dict(small_bin_capacity=256), dict(canonical=False),
                                  dict(force_large=True), dict(split_tight=True), dict(chunk_capacity=40000),
                                  dict(small_bin_capacity=256, split_tight=True, canonical=False)])
def test_presplit_device_reads(gpu, opts):
    w = synth.make("C4", scale=0.004)
    opts = dict(dict(small_bin_capacity=512), **opts)
    keys, counts, st = gpu_count(gpu, w, distribute_path=2, presplit=1, **opts)
    ref = oracle.count(w.reads, w.offsets, w.k, w.cutoff_min, w.cutoff_max, canonical=opts.get("canonical", True))
    assert st["n_presplit_bins"] > 0
    assert np.array_equal(keys, ref.keys) and np.array_equal(counts, ref.counts)
    if opts.get("split_tight"):
        assert st["n_split_overflow"] > 0


@pytest.mark.parametrize("batch_mb,opts", [(2, dict()), (1, dict(small_bin_capacity=256)), (3, dict(split_tight=True)),
                                           (2, dict(presplit=2))])
def test_presplit_host_batches(gpu, batch_mb, opts):
    # host-resident reads take the presplit by default: the split of every batch's new records
    w = synth.make("C4", scale=0.005)
    opts = dict(dict(small_bin_capacity=512), **opts)
    rh = torch.from_numpy(w.reads).pin_memory()
    oh = torch.from_numpy(w.offsets.view(np.uint64))
    res = gpu.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu", input_batch_mb=batch_mb,
                    distribute_path=2, **opts)
    ref = oracle.count(w.reads, w.offsets, w.k, w.cutoff_min, w.cutoff_max)
    assert res.stats["n_input_batches"] >= 4
    assert (res.stats["n_presplit_bins"] > 0) == (opts.get("presplit", 0) != 2)
    assert np.array_equal(res.kmers.numpy(), ref.keys) and np.array_equal(res.counts.numpy(), ref.counts)


def test_presplit_rerun(gpu):
    # a sample that misses part of the input overflows a bin: the presplit is dropped with the
    # rest of the sampled plan and the call replans
    first = [s.decode() for s in synth.random_reads(41, 20000, 100, 100, alphabet=b"ACGT")]
    rest = [s.decode() for s in synth.random_reads(42, 5, 150, 150, alphabet=b"ACGT")] * 3000
    w = synth.from_strings(first + rest, 28, 9, 1)
    rh = torch.from_numpy(w.reads).pin_memory()
    oh = torch.from_numpy(w.offsets.view(np.uint64))
    res = gpu.count(rh, oh, w.k, w.p, 1, 10**9, out_device="cpu", input_batch_mb=1, distribute_path=2,
                    small_bin_capacity=256)
    ref = oracle.count(w.reads, w.offsets, w.k, 1, 10**9)
    assert res.stats["n_distribute_reruns"] == 1
    assert np.array_equal(res.kmers.numpy(), ref.keys) and np.array_equal(res.counts.numpy(), ref.counts)


@pytest.mark.parametrize("out_device", ["cpu", "cuda"])
def test_order_oversize_buckets(gpu, out_device):
    # survivors piling into one S9 bucket (a shared all-A prefix) beyond a CTA sort: the
    # oversize path; with pinned host outputs the groups of S9's final sorts are copied out
    # while the next group sorts, the group holding the oversize bucket after its sort
    tails = [s.decode() for s in synth.random_reads(7, 30000, 88, 88, alphabet=b"ACGT")]
    w = synth.from_strings(["A" * 12 + t for t in tails], 28, 9, 1)
    rh = torch.from_numpy(w.reads)
    oh = torch.from_numpy(w.offsets.view(np.uint64))
    if out_device == "cuda":
        rh, oh = rh.cuda(), oh.cuda()
    else:
        rh = rh.pin_memory()
    res = gpu.count(rh, oh, w.k, w.p, 1, 10**9, out_device=out_device)
    ref = oracle.count(w.reads, w.offsets, w.k, 1, 10**9)
    assert res.stats["n_order_oversize"] > 0
    assert np.array_equal(res.kmers.cpu().numpy(), ref.keys) and np.array_equal(res.counts.cpu().numpy(), ref.counts)
