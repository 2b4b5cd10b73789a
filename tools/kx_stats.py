"""(k, x)-mer statistics (Sec. 2.3) on a C4-shaped sample.

The paper replaces the k-mers of a super-k-mer by as few (k, x)-mers as possible: runs of
consecutive windows whose canonical form is read in the same direction become one
(k + x')-mer (x' <= x) in canonical form, so a sorter handles fewer, longer items and the
k-mer counts are recovered by merging the sorted (k, x)-mer arrays.  This tool measures
what that would do to the GPU path, which counts with hash tables instead of sorting:

* items       -- windows (k-mers) vs (k, x)-mers: the keys the split and the chunk hash
                 would handle;
* distinct    -- distinct k-mers vs distinct (k, x)-mers;
* expansion   -- sum over distinct (k, x)-mers of (x' + 1): the weighted k-mer inserts a
                 second counting pass would need to turn (k, x)-mer counts into k-mer
                 counts (the hash path has no sorted arrays to merge).

Uses the oracle's signatures (test infrastructure) and numpy only.
usage: python tools/kx_stats.py [scale] [x]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle
import synth

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.005
X = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = synth.make("C4", scale=scale)
k, p = w.k, w.p
reads, offs = w.reads, w.offsets.astype(np.int64)
n = reads.shape[0]
code = np.full(256, 255, dtype=np.uint8)
for ch, v in zip(b"ACGTacgt", [0, 1, 2, 3, 0, 1, 2, 3]):
    code[ch] = v
s = code[reads]
valid_base = s != 255
s = np.where(valid_base, s, 0).astype(np.uint64)
# window starts inside one read and without invalid bases
read_id = np.repeat(np.arange(len(offs) - 1), np.diff(offs))
nw = n - k + 1
same_read = read_id[:nw] == read_id[k - 1:]
bad = np.concatenate([[0], np.cumsum(~valid_base)])
win_ok = same_read & ((bad[k:] - bad[:nw]) == 0)
# forward and reverse-complement values of every window
fwd = np.zeros(nw, dtype=np.uint64)
rc = np.zeros(nw, dtype=np.uint64)
for j in range(k):
    fwd = (fwd << np.uint64(2)) | s[j:j + nw]
    rc = rc | ((np.uint64(3) - s[j:j + nw]) << np.uint64(2 * j))
orient = fwd <= rc  # canonical read forward (palindromes either way)
sig = oracle.signatures(w.reads, w.offsets, k, p)[:nw]
# (k, x)-mers: runs of valid windows, same signature (one super-k-mer) and same orientation,
# cut into groups of at most X + 1 windows
idx = np.nonzero(win_ok)[0]
brk = np.ones(len(idx), dtype=bool)
brk[1:] = (idx[1:] != idx[:-1] + 1) | (sig[idx[1:]] != sig[idx[:-1]]) | (orient[idx[1:]] != orient[idx[:-1]])
run_id = np.cumsum(brk) - 1
run_start = np.nonzero(brk)[0]
pos_in_run = np.arange(len(idx)) - run_start[run_id]
grp_start = (pos_in_run % (X + 1)) == 0
g_first = idx[grp_start]
# group length x' + 1 = windows in the group
gid = np.cumsum(grp_start) - 1
glen = np.bincount(gid).astype(np.int64)
# group value: the (k + x')-mer in its canonical orientation, plus its length
vals = []
for L in range(1, X + 2):
    sel = glen == L
    st = g_first[sel]
    kk = k + L - 1
    v = np.zeros(len(st), dtype=np.uint64)
    ori = orient[st]
    for j in range(kk):
        fj = s[st + j]
        rj = np.uint64(3) - s[st + kk - 1 - j]
        v = (v << np.uint64(2)) | np.where(ori, fj, rj)
    vals.append((L, v))
n_items = int(win_ok.sum())
n_kx = int(len(g_first))
canon = np.minimum(fwd[win_ok], rc[win_ok])
n_distinct_k = len(np.unique(canon))
n_distinct_kx = 0
expansion = 0
for L, v in vals:
    d = len(np.unique(v))
    n_distinct_kx += d
    expansion += d * L
print(f"C4 scale {scale}: {w.n_reads} reads, {w.n_bases} bases, k={k}, p={p}, x={X}")
print(f"| windows (k-mers) | (k,x)-mers | distinct k-mers | distinct (k,x)-mers | second-pass k-mer inserts |")
print(f"|---|---|---|---|---|")
print(f"| {n_items} | {n_kx} ({n_kx / n_items:.3f}) | {n_distinct_k} | {n_distinct_kx} | {expansion} "
      f"({(n_kx + expansion) / n_items:.3f} x windows in total) |")
