"""Large-bin cluster path at one config: stage times and item statistics per cluster size
(tools/r2 experiments; not a benchmark).  usage: python tools/cl_sweep.py [C4] [scale] [sizes...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1407_1507_b200 as kmc  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
sizes = [int(x) for x in sys.argv[3:]] or [16, 8, 4]
w = synth.make(name, scale=scale)
r = torch.from_numpy(w.reads).cuda()
o = torch.from_numpy(w.offsets.view(np.uint64)).cuda()
for extra in [dict(cluster_size=c) for c in sizes] + [dict(large_path=2)]:
    for rep in range(2):
        res = kmc.count(r, o, w.k, w.p, w.cutoff_min, w.cutoff_max, profile=True, **extra)
    st = res.stats
    print(extra, {k: round(v, 2) for k, v in st["stage_ms"].items() if v > 0},
          {k: st[k] for k in ("n_cluster_items", "n_single_items", "n_spilled_keys", "cluster_size", "cluster_ctas",
                              "n_unique", "n_out")}, flush=True)
    del res
