"""Sharded counting: host logic on CPU (bin ownership, the all-to-all exchange
under gloo with world size 2) and, on the GPU, the sharded path against the CPU oracle."""
import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------- host logic (CPU)

@pytest.mark.parametrize("world", [1, 2, 3, 8])
def test_shard_owners_contiguous_and_balanced(world):
    import paper_1407_1507_b200 as kmc
    rng = np.random.default_rng(7 + world)
    w = rng.integers(0, 5000, size=4000).astype(np.uint64)
    w[rng.integers(0, 4000, 20)] = 0
    own = kmc.shard_owners(w, world)
    assert own.shape == w.shape and own.max() < world
    assert np.all(np.diff(own.astype(np.int64)) >= 0)  # contiguous ranges of bins
    load = np.bincount(own, weights=w.astype(np.float64), minlength=world)
    assert load.max() <= w.sum() / world + w.max() + 1  # within one bin of the even share
    if world <= 3:
        assert set(own.tolist()) == set(range(world))


def test_shard_owners_degenerate():
    import paper_1407_1507_b200 as kmc
    assert kmc.shard_owners(np.zeros(5, np.uint64), 4).tolist() == [0] * 5
    assert kmc.shard_owners(np.array([], np.uint64), 2).tolist() == []
    assert kmc.shard_owners(np.array([7], np.uint64), 3).tolist() == [1]


def _exchange_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import paper_1407_1507_b200 as kmc
    dist.init_process_group("gloo", rank=rank, world_size=world)
    # rank r sends (r*10 + dest) records to each dest; record words encode (src, dest, index)
    counts = [rank * 10 + d + 1 for d in range(world)]
    rows, sigs = [], []
    for d in range(world):
        for i in range(counts[d]):
            rows.append([rank, d, i, 7])
            sigs.append(1000 * rank + 10 * d + i % 10)
    recs = torch.tensor(rows, dtype=torch.int32)
    sg = torch.tensor(sigs, dtype=torch.int32)
    rr, rs, rc = kmc.exchange(recs, sg, counts)
    q.put((rank, rr.tolist(), rs.tolist(), rc))
    dist.destroy_process_group()


def test_exchange_all_to_all_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, 29541, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
        assert p.exitcode == 0
    got = {r: (rr, rs, rc) for r, rr, rs, rc in (q.get() for _ in range(world))}
    for r in range(world):
        rr, rs, rc = got[r]
        assert rc == [s * 10 + r + 1 for s in range(world)]
        want = [[s, r, i, 7] for s in range(world) for i in range(s * 10 + r + 1)]
        assert rr == want  # source-rank order, each source's records in order
        assert rs == [1000 * s + 10 * r + i % 10 for s in range(world) for i in range(s * 10 + r + 1)]


# ---------------------------------------------------------------- GPU: sharded == oracle

def _slices(w, n):
    """n read-aligned slices of a workload, as device tensors."""
    cuts = np.linspace(0, w.n_reads, n + 1).astype(np.int64)
    out = []
    for a, b in zip(cuts[:-1], cuts[1:]):
        off = w.offsets[a:b + 1]
        reads = w.reads[int(off[0]):int(off[-1])]
        r = torch.from_numpy(np.ascontiguousarray(reads)).cuda() if reads.size else torch.zeros(0, dtype=torch.uint8,
                                                                                                device="cuda")
        out.append((r, torch.from_numpy(np.ascontiguousarray(off).view(np.uint64)).cuda()))
    return out


def _union_matches_oracle(results, w, k, ci, cx):
    keys = [r.kmers.cpu().numpy() for r in results]
    counts = [r.counts.cpu().numpy() for r in results]
    for kk in keys:  # every rank's share is ascending
        if k <= 32:
            assert np.all(np.diff(kk.astype(np.uint64)) > 0) if kk.size > 1 else True
    allk = np.concatenate(keys) if k <= 32 else np.concatenate(keys).reshape(-1, 2)
    allc = np.concatenate(counts)
    if k <= 32:
        order = np.argsort(allk, kind="stable")
    else:
        order = np.lexsort((allk[:, 0], allk[:, 1]))
    allk, allc = allk[order], allc[order]
    ref = oracle.count(w.reads, w.offsets, k, ci, cx)
    assert allk.shape[0] == ref.keys.shape[0]  # disjoint shares: no k-mer counted twice
    assert np.array_equal(allk, ref.keys) and np.array_equal(allc, ref.counts)
    return sum(r.stats["n_windows"] for r in results), ref


@pytest.mark.gpu
@pytest.mark.parametrize("world", [1, 2, 3, 5])
@pytest.mark.parametrize("name,scale", [("C5", 0.004), ("C2", 0.004)])
def test_sharded_local_matches_oracle(gpu, world, name, scale):
    w = synth.make(name, scale=scale)
    res = gpu.count_sharded_local(_slices(w, world), w.k, w.p, w.cutoff_min, w.cutoff_max)
    assert len(res) == world
    nwin, ref = _union_matches_oracle(res, w, w.k, w.cutoff_min, w.cutoff_max)
    assert nwin == ref.n_windows


@pytest.mark.gpu
@pytest.mark.parametrize("opts", [dict(force_large=True), dict(count_path=1), dict(small_bin_capacity=256)])
def test_sharded_local_paths(gpu, opts):
    w = synth.make("C1", scale=0.1)
    res = gpu.count_sharded_local(_slices(w, 3), w.k, w.p, 1, 10**9, **opts)
    _union_matches_oracle(res, w, w.k, 1, 10**9)


@pytest.mark.gpu
def test_sharded_local_k128_and_empty_slice(gpu):
    w = synth.make("C3", scale=0.003)
    sl = _slices(w, 2)
    sl.insert(1, (torch.zeros(0, dtype=torch.uint8, device="cuda"), torch.zeros(1, dtype=torch.int64,
                                                                                 device="cuda").view(torch.uint64)))
    res = gpu.count_sharded_local(sl, w.k, w.p, w.cutoff_min, w.cutoff_max)
    _union_matches_oracle(res, w, w.k, w.cutoff_min, w.cutoff_max)


@pytest.mark.gpu
def test_sharded_world1_equals_count(gpu):
    w = synth.make("C5", scale=0.003)
    r = torch.from_numpy(w.reads).cuda()
    o = torch.from_numpy(w.offsets.view(np.uint64)).cuda()
    a = gpu.count(r, o, w.k, w.p, w.cutoff_min, w.cutoff_max)
    b = gpu.count_sharded(r, o, w.k, w.p, w.cutoff_min, w.cutoff_max)
    assert torch.equal(a.kmers, b.kmers) and torch.equal(a.counts, b.counts)


def _sharded_gpu_worker(rank, world, port, name, scale, q, mode="collective", opts=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    sys.path.insert(0, ROOT)
    import paper_1407_1507_b200 as kmc
    import synth as sy
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    w = sy.make(name, scale=scale)
    cuts = np.linspace(0, w.n_reads, world + 1).astype(np.int64)
    off = w.offsets[cuts[rank]:cuts[rank + 1] + 1]
    reads = torch.from_numpy(np.ascontiguousarray(w.reads[int(off[0]):int(off[-1])])).cuda()
    offs = torch.from_numpy(np.ascontiguousarray(off).view(np.uint64)).cuda()
    res = kmc.count_sharded(reads, offs, w.k, w.p, w.cutoff_min, w.cutoff_max, exchange_mode=mode, **(opts or {}))
    q.put((rank, res.kmers.cpu().numpy(), res.counts.cpu().numpy()))
    dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("mode,world,name,opts", [("collective", 2, "C5", None), ("p2p", 2, "C5", None),
                                                  ("p2p", 3, "C2", dict(force_large=True)),
                                                  ("p2p", 2, "C3", None)])
def test_count_sharded_processes(gpu, mode, world, name, opts):
    # ranks as processes on one GPU (gloo for the host-side exchanges).  "collective": records
    # grouped into send buffers, all-to-all through gloo; "p2p": the fused exchange -- every
    # rank's partition pass writes into the owners' receive buffers mapped through CUDA IPC
    # (here the peers are other processes on the same device; on a node, other GPUs over NVLink)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    scale = 0.003
    port = 29561 + 7 * world + (mode == "p2p") + 3 * (name == "C3")
    procs = [ctx.Process(target=_sharded_gpu_worker, args=(r, world, port, name, scale, q, mode, opts))
             for r in range(world)]
    for p in procs:
        p.start()
    got = sorted(q.get(timeout=600) for _ in range(world))
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    w = synth.make(name, scale=scale)
    keys = np.concatenate([g[1] for g in got])
    counts = np.concatenate([g[2] for g in got])
    if keys.ndim == 1:
        order = np.argsort(keys, kind="stable")
    else:
        keys = keys.reshape(-1, 2)
        order = np.lexsort((keys[:, 0], keys[:, 1]))
    ref = oracle.count(w.reads, w.offsets, w.k, w.cutoff_min, w.cutoff_max)
    assert np.array_equal(keys[order], ref.keys) and np.array_equal(counts[order], ref.counts)
