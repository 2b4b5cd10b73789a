"""Run one count on a config and compare with the oracle (debug helper)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, oracle
import paper_1407_1507_b200 as kmc
name = sys.argv[1]; scale = float(sys.argv[2]); check = len(sys.argv) > 3
w = synth.make(name, scale=scale)
r = torch.from_numpy(w.reads).cuda(); o = torch.from_numpy(w.offsets.view(np.uint64)).cuda()
res = kmc.count(r, o, w.k, w.p, w.cutoff_min, w.cutoff_max)
torch.cuda.synchronize()
print(name, scale, res.stats["n_out"], res.stats["n_large_bins"], res.stats["n_bins"])
if check:
    ref = oracle.count(w.reads, w.offsets, w.k, w.cutoff_min, w.cutoff_max)
    print("parity", np.array_equal(res.kmers.cpu().numpy(), ref.keys) and np.array_equal(res.counts.cpu().numpy(), ref.counts))
