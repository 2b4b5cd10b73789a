"""One kmc_count call on a scaled config, for ncu captures (not a benchmark)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_1407_1507_b200 as kmc

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 0.05
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 1
w = synth.make(name, scale=scale)
r = torch.from_numpy(w.reads).cuda()
o = torch.from_numpy(w.offsets.view(np.uint64)).cuda()
kmc.use_torch_allocator(True)
for _ in range(calls):
    res = kmc.count(r, o, w.k, w.p, w.cutoff_min, w.cutoff_max, profile=True, **eval(os.environ.get('KMC_OPTS', 'dict()')))
torch.cuda.synchronize()
print({k: round(v, 3) for k, v in res.stats["stage_ms"].items()}, res.stats["n_out"], res.stats["n_overflow_chunks"])
