"""kmcgpu: B200-native (sm_100a) canonical k-mer counting -- the data-parallel hot path of
KMC 2 (Deorowicz et al., arXiv 1407.1507) behind the C ABI in include/kmcgpu.h.

This module is argument marshalling only: every step of the path runs in the CUDA
kernels of ``libkmcgpu.so`` (built in-tree by ``paper_1407_1507_b200.build``).  There
is no CPU fallback; if the library is missing or no GPU is present the calls raise.
PyTorch provides device memory (inputs, outputs and, through the allocator hook, the
library's scratch) and the CUDA stream.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkmcgpu.so")

KMC_OK, KMC_ERR_INVALID_ARG, KMC_ERR_OUT_CAPACITY, KMC_ERR_ALLOC, KMC_ERR_CUDA, KMC_ERR_INTERNAL = range(6)
STAGES = ["input", "signature", "plan", "scatter", "small_bins", "large_split", "large_chunks",
          "large_fallback", "order", "output", "large_scatter"]


class KmcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"kmcgpu status {status}: {msg}")
        self.status = status


class _Stats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_uint64) for n in (
        "n_reads", "n_bases", "n_invalid_bases", "n_windows", "n_superkmers", "n_records",
        "n_signatures_used", "n_bins", "n_large_bins", "max_bin_windows", "large_windows", "n_unique",
        "n_below_min", "n_above_max", "n_out", "n_launches", "n_input_batches", "n_large_groups",
        "chunk_capacity", "n_overflow_chunks", "n_order_oversize", "max_signature_windows", "n_small_sorted",
        "n_cluster_items", "n_single_items", "n_spilled_keys", "cluster_size", "cluster_ctas",
        "n_split_overflow", "n_kxmers", "kx_windows", "n_passes", "n_distribute_reruns", "n_presplit_bins")] + [
        ("stage_ms", ctypes.c_float * len(STAGES)), ("stage_launches", ctypes.c_uint32 * len(STAGES))]

    def to_dict(self) -> dict:
        d = {n: int(getattr(self, n)) for n, _ in self._fields_[:-2]}
        d["stage_ms"] = {s: float(self.stage_ms[i]) for i, s in enumerate(STAGES)}
        d["stage_launches"] = {s: int(self.stage_launches[i]) for i, s in enumerate(STAGES)}
        return d


class _Options(ctypes.Structure):
    _fields_ = [("profile", ctypes.c_uint32), ("small_bin_capacity", ctypes.c_uint32),
                ("force_large", ctypes.c_uint32), ("large_path", ctypes.c_uint32),
                ("distribute_path", ctypes.c_uint32), ("input_batch_mb", ctypes.c_uint32),
                ("large_group_mkeys", ctypes.c_uint32), ("count_path", ctypes.c_uint32),
                ("chunk_capacity", ctypes.c_uint32), ("non_canonical", ctypes.c_uint32),
                ("plain_minimizers", ctypes.c_uint32), ("cluster_size", ctypes.c_uint32),
                ("table_keys", ctypes.c_uint32), ("kx", ctypes.c_uint32), ("spill_keys", ctypes.c_uint32),
                ("pass_mb", ctypes.c_uint32), ("split_tight", ctypes.c_uint32), ("presplit", ctypes.c_uint32)]


_ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p)
_FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)

_lock = threading.Lock()
_lib = None
_cb_refs = []


def load():
    """Load libkmcgpu.so (raises if it is missing -- no fallback)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built; run `python -m paper_1407_1507_b200.build`")
        lib = ctypes.CDLL(LIB_PATH)
        P, U64, U32, I = ctypes.c_void_p, ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int
        lib.kmc_count_begin.argtypes = [P, P, U64, I, I, U32, U32, P, ctypes.POINTER(_Options),
                                        ctypes.POINTER(P), ctypes.POINTER(U64)]
        lib.kmc_count_begin.restype = I
        lib.kmc_count_finish.argtypes = [P, P, P, U64, ctypes.POINTER(_Stats)]
        lib.kmc_count_finish.restype = I
        lib.kmc_job_free.argtypes = [P]
        lib.kmc_job_free.restype = None
        lib.kmc_count.argtypes = [P, P, U64, I, I, U32, U32, P, P, U64, ctypes.POINTER(_Stats), P]
        lib.kmc_count.restype = I
        lib.kmc_count_ex.argtypes = [P, P, U64, I, I, U32, U32, P, P, U64, ctypes.POINTER(_Stats), P,
                                     ctypes.POINTER(_Options)]
        lib.kmc_count_ex.restype = I
        lib.kmc_debug_signatures.argtypes = [P, P, U64, I, I, P, P]
        lib.kmc_debug_signatures_ex.argtypes = [P, P, U64, I, I, I, P, P]
        lib.kmc_debug_signatures_ex.restype = I
        lib.kmc_debug_signatures.restype = I
        lib.kmc_debug_allowed.argtypes = [I, P, P]
        lib.kmc_debug_allowed.restype = I
        lib.kmc_last_error.argtypes = []
        lib.kmc_last_error.restype = ctypes.c_char_p
        lib.kmc_version.restype = I
        lib.kmc_set_allocator.argtypes = [_ALLOC_FN, _FREE_FN, P]
        lib.kmc_set_allocator.restype = None
        lib.kmc_empty_cache.argtypes = []
        lib.kmc_empty_cache.restype = None
        lib.kmc_shard_pass1.argtypes = [P, P, U64, I, I, U32, U32, P, ctypes.POINTER(_Options), ctypes.POINTER(P),
                                        P, P, ctypes.POINTER(U64)]
        lib.kmc_shard_pass1.restype = I
        lib.kmc_shard_partition.argtypes = [P, P, P, I, I, P, P, P]
        lib.kmc_shard_partition.restype = I
        lib.kmc_shard_count.argtypes = [P, P, P, U64, ctypes.POINTER(U64)]
        lib.kmc_shard_count.restype = I
        lib.kmc_shard_plan.argtypes = [P, P, P, I, I, P]
        lib.kmc_shard_plan.restype = I
        lib.kmc_shard_recv_alloc.argtypes = [P, U64, P]
        lib.kmc_shard_recv_alloc.restype = I
        lib.kmc_shard_send_peers.argtypes = [P, P, P]
        lib.kmc_shard_send_peers.restype = I
        lib.kmc_shard_count_recv.argtypes = [P, ctypes.POINTER(U64)]
        lib.kmc_shard_count_recv.restype = I
        lib.kmc_shard_owners.argtypes = [P, U64, I, P]
        lib.kmc_shard_owners.restype = None
        lib.kmc_record_words.argtypes = [I]
        lib.kmc_write_db.argtypes = [P, P, U64, I, I, U32, U32, U32, ctypes.c_char_p, P]
        lib.kmc_write_db.restype = I
        lib.kmc_record_words.restype = I
        _lib = lib
        return lib


def empty_cache():
    """Return the default allocator's cached scratch blocks to the driver (kmc_empty_cache)."""
    load().kmc_empty_cache()


def use_torch_allocator(enable: bool = True):
    """Route the library's scratch allocations through torch's caching allocator."""
    import torch
    lib = load()
    if not enable:
        lib.kmc_set_allocator(_ALLOC_FN(0), _FREE_FN(0), None)
        return

    def _alloc(nbytes, stream, ctx):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes), torch.cuda.current_device(), stream or 0)
        except Exception:  # noqa: BLE001 -- reported to the library as NULL -> KMC_ERR_ALLOC
            return None

    def _free(ptr, stream, ctx):
        torch.cuda.caching_allocator_delete(ptr)

    a, f = _ALLOC_FN(_alloc), _FREE_FN(_free)
    _cb_refs[:] = [a, f]
    lib.kmc_set_allocator(a, f, None)


def _check(st: int):
    if st != KMC_OK:
        raise KmcError(st, load().kmc_last_error().decode(errors="replace"))


def _ptr(x) -> int:
    if x is None:
        return 0
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


def _stream_handle(stream) -> int:
    import torch
    if stream is None:
        stream = torch.cuda.current_stream()
    return int(stream.cuda_stream) if hasattr(stream, "cuda_stream") else int(stream)


@dataclasses.dataclass
class Result:
    kmers: object   # uint64 [n] (k <= 32) or [n, 2] (lo, hi); torch tensor (device or host) or numpy
    counts: object  # uint32 [n]
    stats: dict


def _options(profile, small_bin_capacity, force_large, large_path=0, distribute_path=0, input_batch_mb=0,
             large_group_mkeys=0, count_path=0, chunk_capacity=0, canonical=True, plain_minimizers=False,
             cluster_size=0, table_keys=0, spill_keys=0, kx=0, split_tight=False, pass_mb=0, presplit=0):
    o = _Options()
    o.presplit = int(presplit)
    o.pass_mb = int(pass_mb)
    o.split_tight = int(bool(split_tight))
    o.kx = int(kx)
    o.cluster_size = int(cluster_size)
    o.table_keys = int(table_keys)
    o.spill_keys = int(spill_keys)
    o.non_canonical = 0 if canonical else 1
    o.plain_minimizers = int(bool(plain_minimizers))
    o.count_path = int(count_path)
    o.chunk_capacity = int(chunk_capacity)
    o.distribute_path = int(distribute_path)
    o.input_batch_mb = int(input_batch_mb)
    o.large_group_mkeys = int(large_group_mkeys)
    o.profile = int(bool(profile))
    o.small_bin_capacity = int(small_bin_capacity)
    o.force_large = int(bool(force_large))
    o.large_path = int(large_path)
    return o


def count(reads, offsets, k: int, p: int, cutoff_min: int = 2, cutoff_max: int = 10**9, *, stream=None,
          profile: bool = False, small_bin_capacity: int = 0, force_large: bool = False,
          large_path: int = 0, distribute_path: int = 0, input_batch_mb: int = 0, large_group_mkeys: int = 0,
          count_path: int = 0, chunk_capacity: int = 0, out_device: str | None = None,
          canonical: bool = True, plain_minimizers: bool = False, cluster_size: int = 0, table_keys: int = 0,
          spill_keys: int = 0, kx: int = 0, split_tight: bool = False, pass_mb: int = 0,
          presplit: int = 0) -> Result:
    """Count canonical k-mers (KMC 2 hot path on the GPU); canonical=False counts them as
    they occur in the reads (KMC's -b).

    reads: uint8 tensor (cuda, or pinned/pageable cpu -- copied inside the call), n_bases bytes.
    offsets: uint64/int64 tensor, n_reads+1 read boundaries (same device rules).
    Returns sorted unique canonical k-mers and exact counts with
    cutoff_min <= count <= cutoff_max.  Outputs land on ``out_device`` (default: the
    device of ``reads``).
    """
    import torch
    lib = load()
    n_reads = int(offsets.shape[0]) - 1
    if n_reads < 0:
        raise ValueError("offsets must have n_reads + 1 entries")
    opt = _options(profile, small_bin_capacity, force_large, large_path, distribute_path, input_batch_mb,
                   large_group_mkeys, count_path, chunk_capacity, canonical, plain_minimizers, cluster_size,
                   table_keys, spill_keys, kx, split_tight, pass_mb, presplit)
    job = ctypes.c_void_p()
    n_out = ctypes.c_uint64()
    sh = _stream_handle(stream)
    _check(lib.kmc_count_begin(_ptr(reads), _ptr(offsets), n_reads, k, p, cutoff_min, cutoff_max, sh,
                               ctypes.byref(opt), ctypes.byref(job), ctypes.byref(n_out)))
    dev = out_device or (reads.device if hasattr(reads, "device") else "cpu")
    return _finish(lib, job, int(n_out.value), k, dev)


def _finish(lib, job, n: int, k: int, dev) -> Result:
    import torch
    shape = (n,) if k <= 32 else (n, 2)
    pin = str(dev) == "cpu" and torch.cuda.is_available()
    try:
        kmers = torch.empty(shape, dtype=torch.uint64, device=dev, pin_memory=pin)
        counts = torch.empty((n,), dtype=torch.uint32, device=dev, pin_memory=pin)
    except Exception:
        lib.kmc_job_free(job)
        raise
    st = _Stats()
    _check(lib.kmc_count_finish(job, _ptr(kmers), _ptr(counts), n, ctypes.byref(st)))
    return Result(kmers, counts, st.to_dict())


# ---------------------------------------------------------------- sharded counting

def shard_owners(bin_windows, world: int) -> np.ndarray:
    """Bin -> rank map of the sharded plan (host only; kmc_shard_owners)."""
    w = np.ascontiguousarray(bin_windows, dtype=np.uint64)
    out = np.zeros(w.shape[0], dtype=np.uint32)
    load().kmc_shard_owners(w.ctypes.data, w.shape[0], int(world), out.ctypes.data)
    return out


class _Shard:
    """One rank's sharded job: pass 1 -> (all-reduce) -> partition -> (all-to-all) -> count."""

    def __init__(self, reads, offsets, k, p, cutoff_min, cutoff_max, stream=None, **opts):
        import torch
        self.lib = load()
        self.k = k
        self.dev = reads.device if hasattr(reads, "device") else torch.device("cuda")
        ns = 4 ** p + 1
        self.hist_w = torch.zeros(ns, dtype=torch.int64, device=self.dev)
        self.hist_r = torch.zeros(ns, dtype=torch.int64, device=self.dev)
        self.job = ctypes.c_void_p()
        nrec = ctypes.c_uint64()
        opts = dict(opts)
        self.opt = _options(opts.pop("profile", False), opts.pop("small_bin_capacity", 0),
                            opts.pop("force_large", False), **opts)
        n_reads = int(offsets.shape[0]) - 1
        _check(self.lib.kmc_shard_pass1(_ptr(reads), _ptr(offsets), n_reads, k, p, cutoff_min, cutoff_max,
                                        _stream_handle(stream), ctypes.byref(self.opt), ctypes.byref(self.job),
                                        _ptr(self.hist_w), _ptr(self.hist_r), ctypes.byref(nrec)))
        self.n_records = int(nrec.value)
        self.rw = int(self.lib.kmc_record_words(k))

    def partition(self, global_w, global_r, world: int, rank: int):
        """Records grouped by destination rank: (records int32 [n, rw], signatures int32 [n], counts [world])."""
        import torch
        recs = torch.empty((self.n_records, self.rw), dtype=torch.int32, device=self.dev)
        sigs = torch.empty((self.n_records,), dtype=torch.int32, device=self.dev)
        counts = (ctypes.c_uint64 * world)()
        _check(self.lib.kmc_shard_partition(self.job, _ptr(global_w), _ptr(global_r), world, rank, _ptr(recs),
                                            _ptr(sigs), counts))
        return recs, sigs, [int(c) for c in counts]

    # ---- fused exchange over peer memory (kmc_shard_plan / recv_alloc / send_peers / count_recv)
    def plan(self, global_w, global_r, world: int, rank: int):
        """The shared plan and this rank's record count per destination rank (no record moves)."""
        counts = (ctypes.c_uint64 * world)()
        _check(self.lib.kmc_shard_plan(self.job, _ptr(global_w), _ptr(global_r), world, rank, counts))
        return [int(c) for c in counts]

    def recv_alloc(self, n_recv: int) -> bytes:
        """This rank's receive buffers; returns their CUDA IPC handles (128 bytes)."""
        h = (ctypes.c_uint8 * 128)()
        _check(self.lib.kmc_shard_recv_alloc(self.job, int(n_recv), h))
        return bytes(h)

    def send_peers(self, all_handles: bytes, dst_offsets):
        """The partition pass writing every record into its owner's receive buffers."""
        world = len(dst_offsets)
        hb = (ctypes.c_uint8 * len(all_handles)).from_buffer_copy(all_handles)
        offs = (ctypes.c_uint64 * world)(*[int(x) for x in dst_offsets])
        _check(self.lib.kmc_shard_send_peers(self.job, hb, offs))

    def count_recv(self, out_device=None) -> Result:
        n_out = ctypes.c_uint64()
        _check(self.lib.kmc_shard_count_recv(self.job, ctypes.byref(n_out)))
        job, self.job = self.job, None
        return _finish(self.lib, job, int(n_out.value), self.k, out_device or self.dev)

    def count(self, recv_recs, recv_sigs, out_device=None) -> Result:
        n_out = ctypes.c_uint64()
        _check(self.lib.kmc_shard_count(self.job, _ptr(recv_recs), _ptr(recv_sigs), int(recv_sigs.shape[0]),
                                        ctypes.byref(n_out)))
        job, self.job = self.job, None
        return _finish(self.lib, job, int(n_out.value), self.k, out_device or self.dev)

    def __del__(self):
        if getattr(self, "job", None):
            self.lib.kmc_job_free(self.job)


def exchange(recs, sigs, send_counts, group=None):
    """All-to-all of the partitioned records (torch.distributed, NCCL on GPUs / gloo on CPU):
    rank r receives, in source-rank order, every rank's records for r's bins."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    if dist.get_backend(group) == "gloo" and recs.is_cuda:
        # gloo moves host tensors: stage through the host (tests run several ranks on one GPU)
        rr, rs, rc = exchange(recs.cpu(), sigs.cpu(), send_counts, group)
        return rr.to(recs.device), rs.to(sigs.device), rc
    sc = torch.tensor(send_counts, dtype=torch.int64, device=recs.device)
    rc = torch.empty_like(sc)
    dist.all_to_all_single(rc, sc, group=group)
    recv_counts = [int(x) for x in rc.tolist()]
    rw = recs.shape[1]
    rr = torch.empty((sum(recv_counts), rw), dtype=recs.dtype, device=recs.device)
    rs = torch.empty((sum(recv_counts),), dtype=sigs.dtype, device=sigs.device)
    dist.all_to_all_single(rr, recs, output_split_sizes=recv_counts, input_split_sizes=list(send_counts), group=group)
    dist.all_to_all_single(rs, sigs, output_split_sizes=recv_counts, input_split_sizes=list(send_counts), group=group)
    assert len(recv_counts) == world
    return rr, rs, recv_counts


def exchange_p2p(sh, world: int, rank: int, group=None):
    """Fused partition + exchange over peer memory: the record counts per
    (source, destination) are all-gathered, every rank allocates its receive buffers and
    all-gathers their CUDA IPC handles, then every rank's partition pass writes its records
    straight into the owners' buffers (NVLink / NVSwitch between the GPUs of one node) and a
    barrier ends the exchange.  Only counts and handles travel through torch.distributed."""
    import torch.distributed as dist
    counts = sh.plan(sh.hist_w, sh.hist_r, world, rank)
    allc = [None] * world
    dist.all_gather_object(allc, counts, group=group)
    n_recv = sum(allc[s_][rank] for s_ in range(world))
    handles = [None] * world
    dist.all_gather_object(handles, sh.recv_alloc(n_recv), group=group)
    dst_offsets = [sum(allc[s_][d] for s_ in range(rank)) for d in range(world)]
    import torch
    ok, err = 1, None
    try:
        sh.send_peers(b"".join(handles), dst_offsets)
    except KmcError as e:  # e.g. peer memory not mappable: every rank must learn it
        ok, err = 0, e
    # the barrier that ends the exchange (every rank's writes into this rank's buffers are
    # complete), carrying every rank's success
    flag = torch.tensor([ok], dtype=torch.int32,
                        device="cuda" if dist.get_backend(group) == "nccl" else "cpu")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN, group=group)
    if int(flag.item()) == 0:
        raise KmcError(KMC_ERR_CUDA, f"fused P2P exchange failed on a rank ({err})")


def count_sharded(reads, offsets, k: int, p: int, cutoff_min: int = 2, cutoff_max: int = 10**9, *,
                  group=None, stream=None, out_device=None, exchange_mode: str = "p2p", **opts) -> Result:
    """Sharded count over the ranks of ``group`` (torch.distributed): this rank holds a slice
    of the reads; histograms are all-reduced and super-k-mer records exchanged:
    ``exchange_mode="p2p"`` (default, ranks on one node) fuses the exchange into the
    partition pass over peer memory, ``"collective"`` groups the records into send buffers for
    an all-to-all.  Returns this rank's share of the (k-mer, count) pairs -- disjoint from the
    other ranks', ascending; the union is the count of all slices together."""
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    sh = _Shard(reads, offsets, k, p, cutoff_min, cutoff_max, stream=stream, **opts)
    if world > 1:
        if dist.get_backend(group) == "gloo" and sh.hist_w.is_cuda:
            hw, hr = sh.hist_w.cpu(), sh.hist_r.cpu()
            dist.all_reduce(hw, group=group)
            dist.all_reduce(hr, group=group)
            sh.hist_w.copy_(hw)
            sh.hist_r.copy_(hr)
        else:
            dist.all_reduce(sh.hist_w, group=group)
            dist.all_reduce(sh.hist_r, group=group)
    if world > 1 and exchange_mode == "p2p" and sh.hist_w.is_cuda:
        exchange_p2p(sh, world, rank, group)
        return sh.count_recv(out_device=out_device)
    recs, sigs, counts = sh.partition(sh.hist_w, sh.hist_r, world, rank)
    if world > 1:
        recs, sigs, _ = exchange(recs, sigs, counts, group)
    return sh.count(recs, sigs, out_device=out_device)


def count_sharded_local(slices, k: int, p: int, cutoff_min: int = 2, cutoff_max: int = 10**9, *, stream=None,
                        **opts):
    """The sharded path with W virtual ranks in one process (one GPU, run one after another):
    slices = [(reads, offsets), ...]; the all-reduce is a sum and the all-to-all a regrouping
    of the send buffers.  Returns one Result per virtual rank."""
    import torch
    shards = [_Shard(r, o, k, p, cutoff_min, cutoff_max, stream=stream, **opts) for r, o in slices]
    w = len(shards)
    gw = sum(s.hist_w for s in shards)
    gr = sum(s.hist_r for s in shards)
    parts = [s.partition(gw, gr, w, r) for r, s in enumerate(shards)]
    out = []
    for r, s in enumerate(shards):
        rr, rs = [], []
        for recs, sigs, counts in parts:
            o = sum(counts[:r])
            rr.append(recs[o:o + counts[r]])
            rs.append(sigs[o:o + counts[r]])
        out.append(s.count(torch.cat(rr).contiguous(), torch.cat(rs).contiguous()))
    return out


def count_into(reads, offsets, k: int, p: int, cutoff_min: int, cutoff_max: int, out_kmers, out_counts, *,
               stream=None, profile: bool = False) -> dict:
    """One-call form (kmc_count_ex) into caller buffers (device or host); returns stats."""
    lib = load()
    n_reads = int(offsets.shape[0]) - 1
    opt = _options(profile, 0, False)
    st = _Stats()
    cap = int(out_counts.shape[0])
    _check(lib.kmc_count_ex(_ptr(reads), _ptr(offsets), n_reads, k, p, cutoff_min, cutoff_max, _ptr(out_kmers),
                            _ptr(out_counts), cap, ctypes.byref(st), _stream_handle(stream), ctypes.byref(opt)))
    return st.to_dict()


def debug_signatures(reads, offsets, k: int, p: int, stream=None, plain_minimizers: bool = False):
    """Per-position window signature (S2 test hook): uint32 [n_bases], 0xFFFFFFFF = no window;
    plain_minimizers: without the P:L206-208 restrictions (Table 6 diagnostic)."""
    import torch
    lib = load()
    n_reads = int(offsets.shape[0]) - 1
    n_bases = int(reads.shape[0])
    out = torch.empty((max(n_bases, 1),), dtype=torch.uint32, device=reads.device)
    _check(lib.kmc_debug_signatures_ex(_ptr(reads), _ptr(offsets), n_reads, k, p, int(bool(plain_minimizers)),
                                       _ptr(out), _stream_handle(stream)))
    return out[:n_bases]


def debug_allowed(p: int) -> np.ndarray:
    """Device evaluation of the signature rule for every p-mer value (uint8 [4^p])."""
    lib = load()
    out = np.zeros(4 ** p, dtype=np.uint8)
    import torch
    _check(lib.kmc_debug_allowed(p, out.ctypes.data, _stream_handle(torch.cuda.current_stream())))
    return out


def write_db(path: str, kmers, counts, k: int, p: int, cutoff_min: int, cutoff_max: int,
             counter_max: int = 255) -> None:
    """KMC 2 database files <path>.kmc_pre / <path>.kmc_suf (kmc_write_db, include/kmcgpu.h;
    Suppl. Sec. 4) from count()'s k-mers and counts (torch tensors on cuda or
    cpu, or numpy arrays).  counter_max is KMC's -cs: stored counters saturate there."""
    import torch
    lib = load()
    if isinstance(kmers, np.ndarray):
        kmers = torch.from_numpy(np.ascontiguousarray(kmers))
    if isinstance(counts, np.ndarray):
        counts = torch.from_numpy(np.ascontiguousarray(counts))
    kmers = kmers.contiguous()
    counts = counts.contiguous()
    n = int(counts.shape[0])
    stream = torch.cuda.current_stream() if kmers.is_cuda else None
    _check(lib.kmc_write_db(kmers.data_ptr() if n else None, counts.data_ptr() if n else None, n, k, p,
                            max(0, int(cutoff_min)), int(cutoff_max), int(counter_max), path.encode(),
                            _stream_handle(stream) if stream is not None else None))


def version() -> int:
    return int(load().kmc_version())
