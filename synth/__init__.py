"""Seeded synthetic workloads (shared INPUT module -- no counting arithmetic).

The paper's datasets (Table 1) are not available; these
five configurations stand in for them (BASELINE.json ``configs``; recipe and
readings in SURVEY.md section 8(d) and DESIGN.md section 3).  Both the CUDA
path and the CPU oracle consume the arrays produced here; this module imports
neither of them and contains no k-mer, canonical-form or signature code.

``make(name, scale=1.0)`` returns a :class:`Workload` holding
``reads`` (uint8 ASCII, concatenated), ``offsets`` (uint64, n_reads+1, read i
is ``reads[offsets[i]:offsets[i+1]]``) and the counting parameters
(k, p, cutoff_min, cutoff_max) of the config.
"""
from __future__ import annotations

import ctypes
import dataclasses
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")
_lock = threading.Lock()
_lib = None

BASE_SEED = 0x14071507


class _GenomeParams(ctypes.Structure):
    _fields_ = [
        ("genome_len", ctypes.c_uint64), ("gc", ctypes.c_double),
        ("n_fam", ctypes.c_uint64), ("fam_copies", ctypes.c_uint64), ("fam_len", ctypes.c_uint64),
        ("fam_div", ctypes.c_double),
        ("tract_frac", ctypes.c_double), ("tract_min", ctypes.c_uint64), ("tract_max", ctypes.c_uint64),
        ("seed_genome", ctypes.c_uint64),
    ]


class _ReadParams(ctypes.Structure):
    _fields_ = [
        ("n_reads", ctypes.c_uint64), ("len_min", ctypes.c_uint64), ("len_max", ctypes.c_uint64),
        ("err", ctypes.c_double), ("n_iid", ctypes.c_double),
        ("n_run_start", ctypes.c_double), ("n_run_min", ctypes.c_uint64), ("n_run_max", ctypes.c_uint64),
        ("both_strands", ctypes.c_int), ("seed_reads", ctypes.c_uint64),
    ]


def build(force: bool = False) -> str:
    """Compile libsynth.so in-tree with gcc (OpenMP for the read sampler)."""
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, src])
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            lib.synth_genome.argtypes = [ctypes.POINTER(_GenomeParams), ctypes.c_void_p]
            lib.synth_genome.restype = None
            lib.synth_offsets.argtypes = [ctypes.POINTER(_ReadParams), ctypes.c_void_p]
            lib.synth_offsets.restype = ctypes.c_uint64
            lib.synth_reads.argtypes = [ctypes.POINTER(_ReadParams), ctypes.c_void_p, ctypes.c_uint64,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int]
            lib.synth_reads.restype = None
            _lib = lib
    return _lib


@dataclasses.dataclass
class Config:
    name: str
    desc: str
    k: int
    p: int
    cutoff_min: int
    cutoff_max: int
    genome_id: int
    index: int
    genome_len: int
    gc: float
    n_reads: int
    len_min: int
    len_max: int
    err: float
    n_fam: int = 0
    fam_copies: int = 0
    fam_len: int = 0
    fam_div: float = 0.0
    tract_frac: float = 0.0
    tract_min: int = 0
    tract_max: int = 0
    n_iid: float = 0.0
    n_run_start: float = 0.0
    n_run_min: int = 0
    n_run_max: int = 0


# BASELINE.json "configs", read per SURVEY.md 8(d) (readings listed in DESIGN.md section 3).
CONFIGS = {
    "C1": Config("C1", "tiny: 1 Mbp uniform genome, 100,000 x 100 bp (10x), 0.5% errors, k=25 p=7 ci=1",
                 k=25, p=7, cutoff_min=1, cutoff_max=10**9, genome_id=0, index=0,
                 genome_len=1_000_000, gc=0.5, n_reads=100_000, len_min=100, len_max=100, err=0.005),
    "C2": Config("C2", "10 Mbp 40% GC genome + 5 families x 200 copies x 500 bp (1% div), 2M x 150 bp (30x), 1% errors, k=28 p=9 ci=2",
                 k=28, p=9, cutoff_min=2, cutoff_max=10**9, genome_id=1, index=1,
                 genome_len=10_000_000, gc=0.40, n_reads=2_000_000, len_min=150, len_max=150, err=0.01,
                 n_fam=5, fam_copies=200, fam_len=500, fam_div=0.01),
    "C3": Config("C3", "C2's genome, 3M x 100 bp (30x), 1% errors, k=55 p=11 ci=2 (128-bit keys)",
                 k=55, p=11, cutoff_min=2, cutoff_max=10**9, genome_id=1, index=2,
                 genome_len=10_000_000, gc=0.40, n_reads=3_000_000, len_min=100, len_max=100, err=0.01,
                 n_fam=5, fam_copies=200, fam_len=500, fam_div=0.01),
    "C4": Config("C4", "100 Mbp 41% GC genome + 100 families x 100 copies x 1 kbp (2% div), 40M x 100 bp (40x), 1% errors, 0.1% N, k=28 p=9 ci=2 cx=1e9",
                 k=28, p=9, cutoff_min=2, cutoff_max=10**9, genome_id=3, index=3,
                 genome_len=100_000_000, gc=0.41, n_reads=40_000_000, len_min=100, len_max=100, err=0.01,
                 n_fam=100, fam_copies=100, fam_len=1000, fam_div=0.02, n_iid=0.001),
    "C5": Config("C5", "50 Mbp 30% GC genome + 2% poly-A/(AT)n tracts, 2M x U[50,250] bp, 1% errors, ~1% N in runs, k=31 p=9 ci=2",
                 k=31, p=9, cutoff_min=2, cutoff_max=10**9, genome_id=4, index=4,
                 genome_len=50_000_000, gc=0.30, n_reads=2_000_000, len_min=50, len_max=250, err=0.01,
                 tract_frac=0.02, tract_min=20, tract_max=500,
                 n_run_start=0.01 / 5.5, n_run_min=1, n_run_max=10),
}


@dataclasses.dataclass
class Workload:
    name: str
    reads: np.ndarray      # uint8 [n_bases]
    offsets: np.ndarray    # uint64 [n_reads + 1]
    k: int
    p: int
    cutoff_min: int
    cutoff_max: int
    seeds: dict
    scale: float

    @property
    def n_reads(self) -> int:
        return int(self.offsets.shape[0] - 1)

    @property
    def n_bases(self) -> int:
        return int(self.offsets[-1] - self.offsets[0])


def make(name: str, scale: float = 1.0, n_threads: int = 0, shard: int = 0, **overrides) -> Workload:
    """Generate config ``name`` (C1..C5).  ``scale`` < 1 shrinks genome, read count and
    repeat copies together (coverage and composition are kept).  ``shard`` > 0 draws an
    independent read sample of the same genome (the slice of rank ``shard`` in multi-GPU
    runs); shard 0 is the config itself."""
    cfg = dataclasses.replace(CONFIGS[name], **overrides)
    lib = _load()
    G = max(1000, int(cfg.genome_len * scale))
    gp = _GenomeParams(G, cfg.gc, cfg.n_fam, max(2, int(cfg.fam_copies * scale)) if cfg.n_fam else 0,
                       cfg.fam_len, cfg.fam_div, cfg.tract_frac, cfg.tract_min, cfg.tract_max,
                       BASE_SEED + 16 * cfg.genome_id)
    n_reads = max(1, int(round(cfg.n_reads * scale)))
    rp = _ReadParams(n_reads, cfg.len_min, cfg.len_max, cfg.err, cfg.n_iid, cfg.n_run_start,
                     cfg.n_run_min, cfg.n_run_max, 1, BASE_SEED + 16 * cfg.index + 1 + 1000003 * shard)
    genome = np.empty(G, dtype=np.uint8)
    lib.synth_genome(ctypes.byref(gp), genome.ctypes.data)
    offsets = np.empty(n_reads + 1, dtype=np.uint64)
    total = lib.synth_offsets(ctypes.byref(rp), offsets.ctypes.data)
    reads = np.empty(int(total), dtype=np.uint8)
    lib.synth_reads(ctypes.byref(rp), genome.ctypes.data, G, offsets.ctypes.data, reads.ctypes.data, n_threads)
    return Workload(name, reads, offsets, cfg.k, cfg.p, cfg.cutoff_min, cfg.cutoff_max,
                    {"genome": gp.seed_genome, "reads": rp.seed_reads}, scale)


def from_strings(seqs, k: int, p: int = 5, cutoff_min: int = 1, cutoff_max: int = 10**9) -> Workload:
    """Hand-built reads (tests): list of str/bytes -> Workload."""
    bs = [s.encode() if isinstance(s, str) else bytes(s) for s in seqs]
    offsets = np.zeros(len(bs) + 1, dtype=np.uint64)
    if bs:
        offsets[1:] = np.cumsum([len(b) for b in bs], dtype=np.uint64)
    reads = np.frombuffer(b"".join(bs), dtype=np.uint8).copy() if bs else np.zeros(0, dtype=np.uint8)
    return Workload("strings", reads, offsets, k, p, cutoff_min, cutoff_max, {}, 1.0)


def random_reads(seed: int, n_reads: int, len_min: int, len_max: int, n_frac: float = 0.0,
                 lower_frac: float = 0.0, alphabet: bytes = b"ACGT") -> list:
    """Small iid random reads for property tests (numpy Generator, seeded)."""
    rng = np.random.default_rng(seed)
    al = np.frombuffer(alphabet, dtype=np.uint8)
    out = []
    for _ in range(n_reads):
        L = int(rng.integers(len_min, len_max + 1))
        r = al[rng.integers(0, len(al), L)]
        if n_frac > 0:
            r = np.where(rng.random(L) < n_frac, ord("N"), r).astype(np.uint8)
        if lower_frac > 0:
            low = rng.random(L) < lower_frac
            r = np.where(low & (r != ord("N")), r + 32, r).astype(np.uint8)
        out.append(r.tobytes())
    return out
