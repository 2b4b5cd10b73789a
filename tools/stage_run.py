"""One config through kmc_count with options, stage times and statistics (experiments; not a benchmark).
usage: python tools/stage_run.py C4 1.0 'dict(large_path=2)' ..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1407_1507_b200 as kmc  # noqa: E402

name, scale = sys.argv[1], float(sys.argv[2])
w = synth.make(name, scale=scale)
r = torch.from_numpy(w.reads).cuda()
o = torch.from_numpy(w.offsets.view(np.uint64)).cuda()
KEYS = ("n_split_overflow", "n_overflow_chunks", "chunk_capacity", "n_large_groups", "n_unique", "n_out")
for spec in sys.argv[3:] or ["dict()"]:
    opts = eval(spec)
    for rep in range(3):
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        res = kmc.count(r, o, w.k, w.p, w.cutoff_min, w.cutoff_max, profile=True, **opts)
        ev1.record()
        torch.cuda.synchronize()
    st = res.stats
    print(spec, f"{ev0.elapsed_time(ev1):.2f} ms", {k: round(v, 2) for k, v in st["stage_ms"].items() if v > 0},
          {k: st[k] for k in KEYS}, flush=True)
    del res
