"""CPU ORACLE for canonical k-mer counting (KMC 2, arXiv 1407.1507).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product path (``paper_1407_1507_b200``) never imports it and it
never imports the product path; the two share no code.

Two independent implementations of the same plain definition live here:

* ``kmc_oracle.cpp`` (compiled with g++ into ``liboracle.so``): packed-integer
  values recomputed per window from the characters, std::sort + run counting.
* ``count_strings`` / ``signature_str`` below: pure-Python string operations
  (reverse complement by string reversal and letter swap, ``min`` of strings,
  ``collections.Counter``), used for small cases and to cross-check the C++
  oracle ("string-based vs packed-based").

Citations (PAPER.md line numbers, section):
  k-mer counting  P:L14-16 (Abstract), P:L46-48 (Sec. 1)
  canonical form  P:L143-145 (Sec. 2.1)
  signatures      P:L206-208 (Sec. 2.2); Suppl. Sec. 4 P:L1506 (ACGAC = 97)
  super-k-mers    P:L148-151 (Sec. 2.1), Fig. 1
  cutoffs         P:L523-525 (Sec. 2.5), P:L1191-1193 (Suppl. Sec. 1)
Parity status: pinned (tests/test_oracle.py); nothing here is "parity unpinned".
"""
from __future__ import annotations

import collections
import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

_P = ctypes.c_void_p
_U64 = ctypes.c_uint64


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "kmc_oracle.cpp")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        tmp = _SO + f".tmp{os.getpid()}"
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-fopenmp", "-fPIC", "-shared", "-o", tmp, src])
        os.replace(tmp, _SO)
    return _SO


def _load():
    global _lib
    with _lock:
        if _lib is None:
            lib = ctypes.CDLL(build())
            lib.oracle_count.argtypes = [_P, _P, _U64, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32, _P, _P, _U64, _P]
            lib.oracle_count.restype = ctypes.c_int64
            lib.oracle_count_ex.argtypes = [_P, _P, _U64, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32, _P, _P, _U64,
                                            _P, ctypes.c_int]
            lib.oracle_count_ex.restype = ctypes.c_int64
            lib.oracle_count_par.argtypes = [_P, _P, _U64, ctypes.c_int, ctypes.c_uint32, ctypes.c_uint32,
                                             ctypes.POINTER(_P), ctypes.POINTER(_P), _P, ctypes.c_int, ctypes.c_int,
                                             _U64]
            lib.oracle_count_par.restype = ctypes.c_int64
            lib.oracle_free.argtypes = [_P]
            lib.oracle_free.restype = None
            lib.oracle_n_windows.argtypes = [_P, _P, _U64, ctypes.c_int]
            lib.oracle_n_windows.restype = _U64
            lib.oracle_n_windows_par.argtypes = [_P, _P, _U64, ctypes.c_int]
            lib.oracle_n_windows_par.restype = _U64
            lib.oracle_count_queries.argtypes = [_P, _P, _U64, ctypes.c_int, _P, _U64, _P]
            lib.oracle_count_queries.restype = None
            lib.oracle_allowed_index.argtypes = [_U64, ctypes.c_int]
            lib.oracle_allowed_index.restype = ctypes.c_int
            lib.oracle_signatures.argtypes = [_P, _P, _U64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P]
            lib.oracle_signatures.restype = None
            lib.oracle_superkmers.argtypes = [_P, _P, _U64, ctypes.c_int, ctypes.c_int, ctypes.c_int, _P, _P, _P, _U64]
            lib.oracle_superkmers.restype = _U64
            lib.oracle_kx_count.argtypes = [_P, _P, _U64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
            lib.oracle_kx_count.restype = _U64
            _lib = lib
    return _lib


def _arrays(reads, offsets):
    reads = np.ascontiguousarray(reads, dtype=np.uint8)
    offsets = np.ascontiguousarray(offsets, dtype=np.uint64)
    if reads.size == 0:
        reads = np.zeros(1, dtype=np.uint8)
    return reads, offsets


class Result:
    """Sorted survivors.  ``keys`` is uint64 [n] for k <= 32, else uint64 [n, 2] (lo, hi)."""

    def __init__(self, keys, counts, stats):
        self.keys = keys
        self.counts = counts
        self.n_windows, self.n_unique, self.n_below_min, self.n_above_max, self.n_out = (int(x) for x in stats)


def count(reads, offsets, k: int, cutoff_min: int = 1, cutoff_max: int = 10**9, canonical: bool = True) -> Result:
    """Exact canonical k-mer counts with cutoffs (C++ oracle); canonical=False counts the
    k-mers as they occur in the reads (KMC's -b)."""
    lib = _load()
    reads, offsets = _arrays(reads, offsets)
    n_reads = offsets.shape[0] - 1
    cap = int(lib.oracle_n_windows(reads.ctypes.data, offsets.ctypes.data, n_reads, k))
    w = 1 if k <= 32 else 2
    keys = np.zeros((max(cap, 1), w), dtype=np.uint64)
    counts = np.zeros(max(cap, 1), dtype=np.uint32)
    stats = np.zeros(5, dtype=np.uint64)
    n = lib.oracle_count_ex(reads.ctypes.data, offsets.ctypes.data, n_reads, k, cutoff_min, cutoff_max,
                            keys.ctypes.data, counts.ctypes.data, cap, stats.ctypes.data, int(canonical))
    if n < 0:
        raise ValueError("bad k")
    keys = keys[:n, 0].copy() if w == 1 else keys[:n].copy()
    return Result(keys, counts[:n].copy(), stats)


def count_partitioned(reads, offsets, k: int, cutoff_min: int = 1, cutoff_max: int = 10**9, canonical: bool = True,
                      threads: int | None = None, round_keys: int = 1 << 28) -> Result:
    """Same result as :func:`count`, computed over contiguous key ranges by ``threads`` host
    threads (SURVEY 8(d) "Oracle timing"; kmc_oracle.cpp count_par_impl).  ``round_keys``
    bounds the values held in memory at once."""
    lib = _load()
    reads, offsets = _arrays(reads, offsets)
    n_reads = offsets.shape[0] - 1
    T = int(threads or os.cpu_count() or 1)
    kp, cp = _P(), _P()
    stats = np.zeros(5, dtype=np.uint64)
    n = lib.oracle_count_par(reads.ctypes.data, offsets.ctypes.data, n_reads, k, cutoff_min, cutoff_max,
                             ctypes.byref(kp), ctypes.byref(cp), stats.ctypes.data, int(canonical), T,
                             int(round_keys))
    if n < 0:
        raise ValueError("bad k")
    try:
        w = 1 if k <= 32 else 2
        kbuf = (ctypes.c_uint64 * max(1, n * w)).from_address(kp.value)
        cbuf = (ctypes.c_uint32 * max(1, n)).from_address(cp.value)
        keys = np.frombuffer(kbuf, dtype=np.uint64, count=n * w).copy()
        counts = np.frombuffer(cbuf, dtype=np.uint32, count=n).copy()
    finally:
        lib.oracle_free(kp)
        lib.oracle_free(cp)
    if w == 2:
        keys = keys.reshape(n, 2)
    return Result(keys, counts, stats)


def digest(keys, counts) -> str:
    """SHA-256 of the little-endian key words (lo, hi for k > 32) followed by the uint32
    counts: a fingerprint of a sorted (k-mer, count) list (tests/golden/full_configs.json)."""
    import hashlib
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(keys, dtype="<u8").tobytes())
    h.update(np.ascontiguousarray(counts, dtype="<u4").tobytes())
    return h.hexdigest()


def n_windows(reads, offsets, k: int) -> int:
    lib = _load()
    reads, offsets = _arrays(reads, offsets)
    return int(lib.oracle_n_windows(reads.ctypes.data, offsets.ctypes.data, offsets.shape[0] - 1, k))


def n_windows_parallel(reads, offsets, k: int) -> int:
    lib = _load()
    reads, offsets = _arrays(reads, offsets)
    return int(lib.oracle_n_windows_par(reads.ctypes.data, offsets.ctypes.data, offsets.shape[0] - 1, k))


def count_queries(reads, offsets, k: int, queries) -> np.ndarray:
    """Occurrence count of each canonical key in ``queries`` (sorted ascending; uint64 [n] or [n,2])."""
    lib = _load()
    reads, offsets = _arrays(reads, offsets)
    q = np.ascontiguousarray(queries, dtype=np.uint64)
    nq = q.shape[0]
    out = np.zeros(max(nq, 1), dtype=np.uint64)
    lib.oracle_count_queries(reads.ctypes.data, offsets.ctypes.data, offsets.shape[0] - 1, k,
                             q.ctypes.data, nq, out.ctypes.data)
    return out[:nq]


def allowed_index(idx: int, m: int) -> bool:
    return bool(_load().oracle_allowed_index(idx, m))


def signatures(reads, offsets, k: int, p: int, rules: bool = True) -> np.ndarray:
    """uint32 per base position: signature of the window starting there, 0xFFFFFFFF if none."""
    lib = _load()
    reads, offsets = _arrays(reads, offsets)
    n = int(offsets[-1] - offsets[0])
    out = np.zeros(max(n, 1), dtype=np.uint32)
    lib.oracle_signatures(reads.ctypes.data, offsets.ctypes.data, offsets.shape[0] - 1, k, p, int(rules), out.ctypes.data)
    return out[:n]


def superkmers(reads, offsets, k: int, p: int, rules: bool = True):
    """List of (start position, n_windows, signature) for every super-k-mer."""
    lib = _load()
    reads, offsets = _arrays(reads, offsets)
    cap = max(1, int(offsets[-1] - offsets[0]))
    st = np.zeros(cap, dtype=np.uint64)
    nw = np.zeros(cap, dtype=np.uint32)
    sg = np.zeros(cap, dtype=np.uint32)
    n = int(lib.oracle_superkmers(reads.ctypes.data, offsets.ctypes.data, offsets.shape[0] - 1, k, p, int(rules),
                                  st.ctypes.data, nw.ctypes.data, sg.ctypes.data, cap))
    return [(int(st[i]), int(nw[i]), int(sg[i])) for i in range(n)]


def kx_count(reads, offsets, k: int, p: int, x: int, rules: bool = True) -> int:
    """Number of (k,x)-mers the super-k-mers of the reads break into (C++; Table 7's sorted
    fraction is this over the number of valid windows)."""
    lib = _load()
    reads, offsets = _arrays(reads, offsets)
    return int(lib.oracle_kx_count(reads.ctypes.data, offsets.ctypes.data, offsets.shape[0] - 1, k, p, x, int(rules)))


# ---------------------------------------------------------------------------
# Pure-Python string oracle (second, independent implementation; small inputs)
# ---------------------------------------------------------------------------
_PARTNER = str.maketrans("ACGT", "TGCA")
_CODE = {"A": 0, "C": 1, "G": 2, "T": 3}


def revcomp_str(s: str) -> str:
    """Reverse complement as a string: reverse, swap A<->T and C<->G (Fig. 1)."""
    return s[::-1].translate(_PARTNER)


def canonical_str(s: str) -> str:
    """Lexicographically smaller of the string and its reverse complement;
    ASCII order A<C<G<T is the paper's symbol order."""
    r = revcomp_str(s)
    return s if s <= r else r


def str_value(s: str) -> int:
    """Base-4 value, leftmost symbol most significant."""
    v = 0
    for ch in s:
        v = v * 4 + _CODE[ch]
    return v


def value_str(v: int, n: int) -> str:
    out = []
    for _ in range(n):
        out.append("ACGT"[v & 3])
        v >>= 2
    return "".join(reversed(out))


def segments(read: str):
    """Maximal runs of A/C/G/T after upper-casing (reading R3)."""
    cur = []
    for ch in read.upper():
        if ch in _CODE:
            cur.append(ch)
        elif cur:
            yield "".join(cur)
            cur = []
    if cur:
        yield "".join(cur)


def count_strings(reads, k: int, cutoff_min: int = 1, cutoff_max: int = 10**9, canonical: bool = True) -> dict:
    """{canonical k-mer string: count} for ci <= count <= cx (string operations only);
    canonical=False keys the k-mers as they occur (-b)."""
    c = collections.Counter()
    for r in reads:
        r = r.decode() if isinstance(r, (bytes, bytearray)) else r
        for seg in segments(r):
            for i in range(len(seg) - k + 1):
                c[canonical_str(seg[i:i + k]) if canonical else seg[i:i + k]] += 1
    ci = max(1, cutoff_min)
    return {kmer: n for kmer, n in c.items() if ci <= n <= cutoff_max}


def allowed_str(m: str) -> bool:
    """Sec. 2.2 rule on an m-mer string (readings R1/R2)."""
    if m.startswith("AAA") or m.startswith("ACA"):
        return False
    return "AA" not in m[1:]


def signature_str(kmer: str, p: int, rules: bool = True) -> str | None:
    """Smallest allowed canonical p-mer of the k-mer (None = reserved slot 4^p)."""
    best = None
    for j in range(len(kmer) - p + 1):
        c = canonical_str(kmer[j:j + p])
        if rules and not allowed_str(c):
            continue
        if best is None or c < best:
            best = c
    return best


def orientation_str(kmer: str) -> int:
    """0: the k-mer is its own canonical form (forward), 1: its reverse complement is
    (reverse), 2: palindrome (both)."""
    r = revcomp_str(kmer)
    return 0 if kmer < r else (1 if kmer > r else 2)


def kx_split_str(seq: str, k: int, x: int):
    """(k,x)-mers of an ACGT string (Sec. 2.3; Fig. 2): the k-mers of
    seq, left to right, are cut greedily into runs of at most x+1 consecutive k-mers of one
    orientation; a forward run is stored as the stretch it covers, a reverse run as the
    reverse complement of that stretch, so every k-mer inside a record is in canonical form.
    A palindromic k-mer joins the run in progress and starts a run as forward (reading R-KX,
    DESIGN.md).  Returns the records as strings of length k+x', 0 <= x' <= x."""
    n = len(seq) - k + 1
    out = []
    i = 0
    while i < n:
        o = orientation_str(seq[i:i + k])
        run = 0 if o == 2 else o
        j = i + 1
        while j < n and j - i <= x:
            oj = orientation_str(seq[j:j + k])
            if oj != run and oj != 2:
                break
            j += 1
        stretch = seq[i:j - 1 + k]
        out.append(stretch if run == 0 else revcomp_str(stretch))
        i = j
    return out


def kx_merge_counts_str(records, k: int, x: int) -> dict:
    """k-mer counts from (k,x)-mers by the paper's merge (Sec. 2.4, generalised from
    x = 1 to x <= 3): the records are sorted per length class k+x'; for every class x' and
    offset j <= x', the records agreeing on their first j symbols form one sorted sub-array
    whose k-mers (symbols j .. j+k-1) come out in nondecreasing order (R_0, R_1 and R_A..R_T for
    x = 1: 6 cursors; sum_{x'<=x} sum_{j<=x'} 4^j = 112 for x = 3).  All cursors are scanned in
    parallel, the smallest k-mer taken each step; equal k-mers accumulate one count."""
    classes = {}
    for r in records:
        classes.setdefault(len(r) - k, []).append(r)
    cursors = []
    for xp, recs in classes.items():
        recs.sort()
        for j in range(xp + 1):
            groups = {}
            for r in recs:
                groups.setdefault(r[:j], []).append(r[j:j + k])
            for pre in sorted(groups):
                cursors.append(groups[pre])  # each nondecreasing by construction
    for c in cursors:
        assert all(c[i] <= c[i + 1] for i in range(len(c) - 1)), "a sub-array is not sorted"
    pos = [0] * len(cursors)
    out = {}
    last = None
    while True:
        best = None
        for ci, c in enumerate(cursors):
            if pos[ci] < len(c) and (best is None or c[pos[ci]] < cursors[best][pos[best]]):
                best = ci
        if best is None:
            break
        kmer = cursors[best][pos[best]]
        pos[best] += 1
        if kmer != last:
            out[kmer] = 0
            last = kmer
        out[kmer] += 1
    return out, len(cursors)


def count_kx_str(reads, k: int, p: int, x: int, cutoff_min: int = 1, cutoff_max: int = 10**9,
                 rules: bool = True) -> dict:
    """Counting the paper's way with (k,x)-mers (small inputs): every read segment is split into
    super-k-mers (split_str), super-k-mers are binned by signature, and every bin's (k,x)-mers
    are merged (kx_merge_counts_str).  Same result as count_strings for every x."""
    bins = {}
    for r in reads:
        r = r.decode() if isinstance(r, (bytes, bytearray)) else r
        for seg in segments(r):
            for sub, sig in split_str(seg, k, p, rules):
                bins.setdefault(sig, []).extend(kx_split_str(sub, k, x))
    total = {}
    for recs in bins.values():
        counts, _ = kx_merge_counts_str(recs, k, x)
        for km, c in counts.items():
            total[km] = total.get(km, 0) + c
    ci = max(1, cutoff_min)
    return {km: c for km, c in total.items() if ci <= c <= cutoff_max}


def split_str(seg: str, k: int, p: int, rules: bool = True):
    """Super-k-mers of an ACGT segment: [(substring, signature string or None)] (Fig. 1)."""
    out = []
    for i in range(len(seg) - k + 1):
        s = signature_str(seg[i:i + k], p, rules)
        if out and out[-1][1] == s and out[-1][2] == i - 1:
            out[-1] = (out[-1][0] + seg[i + k - 1], s, i)
        else:
            out.append((seg[i:i + k], s, i))
    return [(a, b) for a, b, _ in out]
