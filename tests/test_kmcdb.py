"""KMC 2 database files: pins for the oracle writer/reader (-m "not gpu")
and byte-exact parity of the CUDA writer against it (-m gpu).

Pins: the values the paper prints in its format description (Suppl. Sec. 4, PAPER.md
P:L1448-1544) and the paper's own lookup procedure run over brute-force
string counts -- the writer is checked by reading, not by re-deriving its layout.
"""
import os
import random
import struct

import numpy as np
import pytest

import oracle
import oracle.kmcdb as db
import synth


def test_paper_worked_values():
    # the signature of ATACGACAAATG for signature_length 5 is ACGAC = 97
    assert db.signature_value("ATACGACAAATG", 5) == 97
    # prefix ATAC (lut_prefix_length 4) = 49
    assert oracle.str_value("ATAC") == 49
    # CCACAAAT is stored as 0x51 (CCAC), 0x03 (AAAT)
    assert db.pack_symbols("CCACAAAT") == bytes([0x51, 0x03])
    # header: 7 uint32, uint64, 7 uint32, uint32
    assert db.HEADER_BYTES == 68


def test_counter_bytes():
    # -cs, the maximal counter value: the fewest bytes that hold it
    assert [db.counter_bytes(v) for v in (1, 255, 256, 65535, 65536, (1 << 24) - 1, 1 << 24, (1 << 32) - 1)] == \
        [1, 1, 2, 2, 3, 3, 4, 4]


def _random_reads(seed, n, lo, hi, alphabet="ACGT"):
    rng = random.Random(seed)
    return ["".join(rng.choice(alphabet) for _ in range(rng.randint(lo, hi))) for _ in range(n)]


@pytest.mark.parametrize("k,p,cs", [(12, 5, 255), (28, 9, 255), (13, 7, 3), (5, 3, 65535), (33, 9, 1 << 20),
                                    (3, 1, 255), (8, 8, 255)])
def test_db_lookup_roundtrip(tmp_path, k, p, cs):
    reads = _random_reads(k * 31 + p, 60, k, 160, "ACGT")
    reads += ["ACGT" * 20, "A" * 50, "CA" * 40]  # repeats, palindromes, pile-ups
    counts = oracle.count_strings(reads, k)
    kmers = sorted(counts)
    if k <= 32:
        keys = np.array([oracle.str_value(s) for s in kmers], dtype=np.uint64)
    else:
        v = [oracle.str_value(s) for s in kmers]
        keys = np.array([[x & (2**64 - 1), x >> 64] for x in v], dtype=np.uint64).reshape(-1, 2)
    cnt = np.array([counts[s] for s in kmers], dtype=np.uint32)
    path = str(tmp_path / "db")
    db.write_db(path, keys, cnt, k, p, 1, 10**9, cs)
    r = db.KmcDb(path)
    assert (r.k, r.p, r.mode, r.min_count, r.max_count, r.total, r.version) == (k, p, 0, 1, 10**9, len(kmers), 0x200)
    assert (r.k - r.lut) % 4 == 0 and r.counter_size == db.counter_bytes(cs)
    # file sizes from the layout
    na = db.n_arrays(p)
    pre_size = 4 + 8 * (na * 4 ** r.lut + 1) + 4 * (4 ** p + 1) + 68 + 4 + 4
    assert os.path.getsize(path + ".kmc_pre") == pre_size
    assert os.path.getsize(path + ".kmc_suf") == 8 + len(kmers) * ((k - r.lut) // 4 + r.counter_size)
    # every counted k-mer is found with its (saturated) counter by the paper's lookup
    for s in kmers:
        assert r.lookup(s) == min(counts[s], cs), s
    # k-mers that do not occur are not found
    rng = random.Random(k)
    absent = 0
    for _ in range(200):
        s = oracle.canonical_str("".join(rng.choice("ACGT") for _ in range(k)))
        if s not in counts:
            assert r.lookup(s) is None
            absent += 1
    assert absent > 0 or 4 ** k <= len(counts) * 2


@pytest.mark.parametrize("k,p", [(12, 5), (31, 9), (45, 11), (4, 2)])
def test_db_fast_path_equals_string_path(k, p):
    reads = _random_reads(k + 100 * p, 30, k, 120, "ACGT") + ["A" * 60, "ACGT" * 12]
    counts = oracle.count_strings(reads, k)
    kmers = sorted(counts)
    v = [oracle.str_value(s) for s in kmers]
    keys = (np.array(v, dtype=np.uint64) if k <= 32 else
            np.array([[x & (2**64 - 1), x >> 64] for x in v], dtype=np.uint64).reshape(-1, 2))
    cnt = np.array([counts[s] for s in kmers], dtype=np.uint32)
    assert db.db_bytes(keys, cnt, k, p, 1, 10**9, 255, fast=True) == db.db_bytes(keys, cnt, k, p, 1, 10**9, 255,
                                                                                  fast=False)


def test_db_prefix_array_position_formula(tmp_path):
    # for signature_length 5 the prefixes' array of signature 97 starts at
    # 4 + 97 * 4^lut * 8 (one array per signature when 4^p + 1 arrays fit, G = 0 here)
    k, p = 12, 5
    kmer = "ATACGACAAATG"
    keys = np.array([oracle.str_value(oracle.canonical_str(kmer))], dtype=np.uint64)
    path = str(tmp_path / "one")
    db.write_db(path, keys, np.array([7], dtype=np.uint32), k, p, 1, 10**9, 255)
    r = db.KmcDb(path)
    assert db.group_shift(p) == 0 and int(r.map[97]) == 97
    pre = open(path + ".kmc_pre", "rb").read()
    off = 4 + 97 * 4 ** r.lut * 8
    arr = np.frombuffer(pre[off:off + 8 * (4 ** r.lut + 1)], dtype="<u8")
    x = oracle.str_value(kmer[:r.lut])
    assert int(arr[x]) == 0 and int(arr[x + 1]) == 1  # the single record, under its prefix
    assert r.lookup(kmer) == 7


def _gpu_db(gpu, w, path, cs, ci=None, cx=None):
    import torch
    ci = w.cutoff_min if ci is None else ci
    cx = w.cutoff_max if cx is None else cx
    r = torch.from_numpy(w.reads).cuda()
    o = torch.from_numpy(w.offsets.view(np.uint64)).cuda()
    res = gpu.count(r, o, w.k, w.p, ci, cx)
    gpu.write_db(path, res.kmers, res.counts, w.k, w.p, ci, cx, cs)
    return res


@pytest.mark.gpu
@pytest.mark.parametrize("name,scale,k,cs", [("C1", 0.01, None, 255), ("C5", 0.0005, None, 65535),
                                              ("C3", 0.0005, None, 1 << 20), ("C1", 0.005, 12, 3),
                                              ("C1", 0.005, 31, 255), ("C2", 0.0005, 40, (1 << 32) - 1)])
def test_gpu_db_bytes_match_oracle(gpu, tmp_path, name, scale, k, cs):
    w = synth.make(name, scale=scale) if k is None else synth.make(name, scale=scale, k=k)
    path = str(tmp_path / "gpu")
    _gpu_db(gpu, w, path, cs)
    # the expected files come from the oracle's own counts (not the GPU's), so a counting
    # bug cannot cancel out between the two writers
    ref = oracle.count(w.reads, w.offsets, w.k, w.cutoff_min, w.cutoff_max)
    pre, suf = db.db_bytes(ref.keys, ref.counts, w.k, w.p, w.cutoff_min, w.cutoff_max, cs)
    assert open(path + ".kmc_pre", "rb").read() == pre
    assert open(path + ".kmc_suf", "rb").read() == suf


@pytest.mark.gpu
def test_gpu_db_empty(gpu, tmp_path):
    w = synth.from_strings(["ACG", "N" * 40], 25, 7, 1)
    path = str(tmp_path / "empty")
    res = _gpu_db(gpu, w, path, 255)
    assert res.kmers.shape[0] == 0
    pre, suf = db.db_bytes(np.zeros(0, dtype=np.uint64), np.zeros(0, dtype=np.uint32), 25, 7, 1, w.cutoff_max, 255)
    assert open(path + ".kmc_pre", "rb").read() == pre
    assert open(path + ".kmc_suf", "rb").read() == suf
