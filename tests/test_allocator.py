"""Scratch allocators (-m gpu): the default block cache (kmc_set_allocator, include/kmcgpu.h)
and the torch caching-allocator hook give the same counts as the oracle, across repeated
calls, streams, an emptied cache and host-resident inputs."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


def _check(kmc, w, reads, offs, **kw):
    res = kmc.count(reads, offs, w.k, w.p, w.cutoff_min, w.cutoff_max, **kw)
    ref = oracle.count(w.reads, w.offsets, w.k, w.cutoff_min, w.cutoff_max)
    assert np.array_equal(res.kmers.cpu().numpy(), ref.keys)
    assert np.array_equal(res.counts.cpu().numpy(), ref.counts)


def test_block_cache_reuse_and_empty(gpu):
    kmc = gpu
    w = synth.make("C2", scale=0.01, shard=5)
    reads = torch.from_numpy(w.reads).cuda()
    offs = torch.from_numpy(w.offsets.view(np.uint64)).cuda()
    kmc.use_torch_allocator(False)
    try:
        for _ in range(3):  # cached blocks handed out again
            _check(kmc, w, reads, offs)
        s = torch.cuda.Stream()
        _check(kmc, w, reads, offs, stream=s)  # another stream: its own blocks
        kmc.empty_cache()
        _check(kmc, w, reads, offs)
        kmc.empty_cache()
        kmc.empty_cache()  # empty cache: no-op
        # host-resident inputs streamed in small batches (copy stream + two device slots)
        _check(kmc, w, torch.from_numpy(w.reads).pin_memory(), torch.from_numpy(w.offsets.view(np.uint64)),
               input_batch_mb=1, out_device="cpu")
    finally:
        kmc.empty_cache()


def test_torch_allocator_hook(gpu):
    kmc = gpu
    w = synth.make("C1", shard=6)
    reads = torch.from_numpy(w.reads).cuda()
    offs = torch.from_numpy(w.offsets.view(np.uint64)).cuda()
    kmc.use_torch_allocator(True)
    try:
        for _ in range(2):
            _check(kmc, w, reads, offs)
    finally:
        kmc.use_torch_allocator(False)
