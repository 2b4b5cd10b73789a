import sys, os
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import synth, paper_1407_1507_b200 as kmc
w = synth.make("C4", scale=1.0)
r = torch.from_numpy(w.reads).cuda(); o = torch.from_numpy(w.offsets.view(np.uint64)).cuda()
res = kmc.count(r, o, w.k, w.p, w.cutoff_min, w.cutoff_max)
keys = res.kmers.view(torch.int64)
for bits in (20, 22, 24, 26):
    b = (keys >> (56 - bits)).to(torch.int64)
    h = torch.bincount(b, minlength=1 << bits)
    n = keys.numel()
    hs = h.sort().values
    nz = (h > 0).sum().item()
    print(bits, "buckets", 1 << bits, "nonempty", nz, "max", hs[-1].item(),
          "keys in buckets >32:", h[h > 32].sum().item() / n, ">64:", h[h > 64].sum().item() / n,
          ">512:", h[h > 512].sum().item() / n, "n>32:", (h > 32).sum().item(), "n>64:", (h > 64).sum().item())
