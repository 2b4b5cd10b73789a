"""Large-chunk stage time vs chunk capacity on a scaled config (tuning aid, not a benchmark)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_1407_1507_b200 as kmc

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 0.25
caps = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, 8192, 12288, 16384, 24576, 32768]
w = synth.make(name, scale=scale)
r = torch.from_numpy(w.reads).cuda()
o = torch.from_numpy(w.offsets.view(np.uint64)).cuda()
kmc.use_torch_allocator(True)
for cap in caps:
    for rep in range(3):
        res = kmc.count(r, o, w.k, w.p, w.cutoff_min, w.cutoff_max, profile=True, chunk_capacity=cap)
    st = res.stats
    print(cap, st["chunk_capacity"], st.get("n_overflow_chunks"), {k: round(v, 2) for k, v in st["stage_ms"].items()
                                                                  if k.startswith("large")}, st["n_out"], flush=True)
