"""CPU ORACLE for the KMC 2 database files (.kmc_pre / .kmc_suf), SURVEY 8(f) f4.

TEST INFRASTRUCTURE ONLY (same rule as the rest of ``oracle/``): only ``tests/`` may
import it; the product path never does.

The file layout is written out from the paper's supplement, Sec. 4 "Database format"
(PAPER.md P:L1448-1544), field by field, in plain Python:

* ``.kmc_pre`` = "KMCP" | prefixes | map | header | header position | "KMCP"
  (P:L1456-1463); header fields and sizes P:L1478-1490 (68 bytes); header position =
  the header's distance from the header-position field (reading procedure P:L1469-1474);
  map = uint32[4^p + 1], the prefixes-array id of each signature;
  prefixes = uint64 arrays of 4^lut entries, one per id, + one guard.
* ``.kmc_suf`` = "KMCS" | records | "KMCS"; a record = the k-mer suffix
  after the lut-symbol prefix, 4 symbols per byte, leftmost symbol in the top bits
  (CCACAAAT -> 0x51 0x03), then the counter in counter_size LSB-first bytes
  (P:L1535-1540).  All integers little-endian.

What the paper leaves open (reading R-DB): which signatures share a prefixes
array (here id = signature >> G, G = max(0, 2p - 14), so at most 4^7 + 1 arrays; the
reserved "no allowed p-mer" signature 4^p is the last id), lut_prefix_length (the largest
of k mod 4, +4, +8 that is <= k and keeps ids x 4^lut <= 2^23), and the counter size for a
given maximal counter value cs (-cs: the fewest bytes that hold cs; stored
counters are min(count, cs)).  Records are ordered by (array id, k-mer), k-mers ascending
within an array -- the order the lookup procedure binary-searches.

Signatures of stored k-mers come from ``oracle.signature_str`` (Sec. 2.2).
Parity status: pinned by tests/test_kmcdb.py (the paper's worked values and the lookup
procedure of P:L1497-1517 over brute-force counts).
"""
from __future__ import annotations

import struct

import numpy as np

from . import signature_str, str_value, value_str

KMC_VER = 0x200
HEADER_BYTES = 7 * 4 + 8 + 7 * 4 + 4


def group_shift(p: int) -> int:
    return max(0, 2 * p - 14)


def n_arrays(p: int) -> int:
    return (4 ** p >> group_shift(p)) + 1


def lut_length(k: int, p: int) -> int:
    best = k % 4
    for lut in (k % 4, k % 4 + 4, k % 4 + 8):
        if lut <= k and n_arrays(p) * 4 ** lut <= 1 << 23:
            best = lut
    return best


def counter_bytes(cs: int) -> int:
    for b in (1, 2, 3):
        if cs < 1 << (8 * b):
            return b
    return 4


def pack_symbols(s: str) -> bytes:
    """4 symbols per byte, leftmost symbol in the top 2 bits."""
    assert len(s) % 4 == 0
    return bytes(str_value(s[i:i + 4]) for i in range(0, len(s), 4))


def signature_value(kmer: str, p: int) -> int:
    s = signature_str(kmer, p, True)
    return 4 ** p if s is None else str_value(s)


def _kmer_strings(keys, k: int):
    keys = np.asarray(keys)
    if k <= 32:
        return [value_str(int(v), k) for v in keys.reshape(-1)]
    return [value_str((int(keys[i, 1]) << 64) | int(keys[i, 0]), k) for i in range(keys.shape[0])]


def _signatures_fast(kmers, k: int, p: int):
    """Signature values of k-mer strings through the C++ oracle (each k-mer as a read)."""
    from . import signatures
    if not kmers:
        return []
    reads = np.frombuffer("".join(kmers).encode(), dtype=np.uint8)
    offsets = np.arange(0, (len(kmers) + 1) * k, k, dtype=np.uint64)
    sig = signatures(reads, offsets, k, p, True)[::k]
    return [4 ** p if int(v) == 0xFFFFFFFF else int(v) for v in sig]


def db_bytes(keys, counts, k: int, p: int, ci: int, cx: int, cs: int, fast: bool = True):
    """(pre, suf) file contents for canonical k-mers `keys` (ascending) and their counts.
    fast: signatures from the C++ oracle and suffixes as big-endian integers (pinned equal
    to the string path, fast=False, in tests/test_kmcdb.py)."""
    kmers = _kmer_strings(keys, k)
    counts = [int(c) for c in np.asarray(counts).reshape(-1)]
    G, lut, cb = group_shift(p), lut_length(k, p), counter_bytes(cs)
    na = n_arrays(p)
    sigs = _signatures_fast(kmers, k, p) if fast else [signature_value(s, p) for s in kmers]
    ids = [v >> G for v in sigs]
    order = sorted(range(len(kmers)), key=lambda i: (ids[i], kmers[i]))
    # prefixes: position of the first record with (id, prefix) >= (a, x), + guard
    cnt = np.zeros(na * 4 ** lut, dtype=np.uint64)
    for i in order:
        cnt[ids[i] * 4 ** lut + str_value(kmers[i][:lut])] += 1
    pos = np.zeros(na * 4 ** lut + 1, dtype=np.uint64)
    pos[1:] = np.cumsum(cnt)
    suf = bytearray(b"KMCS")
    nb = (k - lut) // 4
    for i in order:
        if fast:
            suf += (str_value(kmers[i][lut:]) if nb else 0).to_bytes(nb, "big")
        else:
            suf += pack_symbols(kmers[i][lut:])
        suf += min(counts[i], cs).to_bytes(cb, "little")
    suf += b"KMCS"
    amap = np.array([s >> G for s in range(4 ** p + 1)], dtype="<u4")
    header = struct.pack("<7IQ7II", k, 0, cb, lut, p, ci, cx, len(kmers), *([0] * 7), KMC_VER)
    assert len(header) == HEADER_BYTES
    pre = b"KMCP" + pos.astype("<u8").tobytes() + amap.tobytes() + header + struct.pack("<I", HEADER_BYTES) + b"KMCP"
    return pre, bytes(suf)


def write_db(path: str, keys, counts, k: int, p: int, ci: int, cx: int, cs: int = 255):
    pre, suf = db_bytes(keys, counts, k, p, ci, cx, cs)
    with open(path + ".kmc_pre", "wb") as f:
        f.write(pre)
    with open(path + ".kmc_suf", "wb") as f:
        f.write(suf)


class KmcDb:
    """Reader following the paper's procedure."""

    def __init__(self, path: str):
        pre = open(path + ".kmc_pre", "rb").read()
        suf = open(path + ".kmc_suf", "rb").read()
        assert pre[:4] == b"KMCP" and pre[-4:] == b"KMCP"
        assert suf[:4] == b"KMCS" and suf[-4:] == b"KMCS"
        x = struct.unpack("<I", pre[-8:-4])[0]
        h = pre[len(pre) - 8 - x:len(pre) - 8]
        f = struct.unpack("<7IQ7II", h)
        (self.k, self.mode, self.counter_size, self.lut, self.p, self.min_count, self.max_count,
         self.total) = f[:8]
        self.version = f[-1]
        nmap = 4 ** self.p + 1
        map_end = len(pre) - 8 - x
        self.map = np.frombuffer(pre[map_end - 4 * nmap:map_end], dtype="<u4")
        self.prefixes = np.frombuffer(pre[4:map_end - 4 * nmap], dtype="<u8")
        self.rec = (self.k - self.lut) // 4 + self.counter_size
        self.suf = suf[4:-4]
        assert len(self.suf) == self.total * self.rec

    def record(self, i: int):
        r = self.suf[i * self.rec:(i + 1) * self.rec]
        nb = (self.k - self.lut) // 4
        return r[:nb], int.from_bytes(r[nb:], "little")

    def lookup(self, kmer: str):
        """Count of a canonical k-mer, or None."""
        a = int(self.map[signature_value(kmer, self.p)])
        base = a * 4 ** self.lut + str_value(kmer[:self.lut])
        lo, hi = int(self.prefixes[base]), int(self.prefixes[base + 1])
        want = pack_symbols(kmer[self.lut:])
        while lo < hi:
            mid = (lo + hi) // 2
            s, c = self.record(mid)
            if s == want:
                return c
            if s < want:
                lo = mid + 1
            else:
                hi = mid
        return None
