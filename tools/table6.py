"""Table 6 on synthetic data: plain canonical minimizers vs KMC 2 signatures.

For k in {28, 55} and p in {5..8}: average super-k-mers per read and the k-mers (windows)
of the most frequent minimizer / signature -- the lower bound of the largest bin.  The
paper's data (G. gallus) is not in the container; the C4-shaped synthetic genome stands in
(DESIGN.md 3).  Prints a markdown table.
usage: python tools/table6.py [scale]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
import paper_1407_1507_b200 as kmc

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.1
kmc.use_torch_allocator(True)
print(f"C4-shaped synthetic reads, scale {scale}\n")
print("| k | p | minimizers: super-k-mers/read | minimizers: largest (M k-mers) | "
      "signatures: super-k-mers/read | signatures: largest (M k-mers) |")
print("|---|---|---|---|---|---|")
for k in (28, 55):
    w = synth.make("C4", scale=scale, k=k)
    r = torch.from_numpy(w.reads).cuda()
    o = torch.from_numpy(w.offsets.view(np.uint64)).cuda()
    for p in (5, 6, 7, 8):
        row = []
        for plain in (True, False):
            st = kmc.count(r, o, k, p, 2, 10**9, plain_minimizers=plain).stats
            row += [st["n_superkmers"] / w.n_reads, st["max_signature_windows"] / 1e6]
        print(f"| {k} | {p} | {row[0]:.3f} | {row[1]:.2f} | {row[2]:.3f} | {row[3]:.2f} |", flush=True)
