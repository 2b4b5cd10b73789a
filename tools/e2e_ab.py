"""e2e A/B on C4 from pinned host memory: the same call as bench.py's e2e leg with different
kmc_options, alternating, N reps each; prints ms per call and the stage times of one profiled
call.  usage: python tools/e2e_ab.py [scale] [reps] 'dict(presplit=2)' 'dict()' ..."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import paper_1407_1507_b200 as kmc  # noqa: E402
import synth  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
variants = [eval(a) for a in sys.argv[3:]] or [dict(presplit=2), dict()]
w = synth.make("C4", scale=scale)
rh = torch.from_numpy(w.reads).pin_memory()
oh = torch.from_numpy(w.offsets.view(np.uint64)).pin_memory()
res = {i: [] for i in range(len(variants))}
ref = None
for i, v in enumerate(variants):  # warm-up + output check + stage times
    r = kmc.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu", **v)
    digest = (int(r.stats["n_out"]), int(r.kmers[::9973].sum()), int(r.counts.sum()))
    ref = ref or digest
    assert digest == ref, (v, digest, ref)
    rp = kmc.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu", profile=True, **v)
    st = rp.stats
    print(v, {s: round(x, 2) for s, x in st["stage_ms"].items() if x}, "presplit bins", st["n_presplit_bins"],
          "split overflow", st["n_split_overflow"], "table overflows", st["n_overflow_chunks"], flush=True)
    del r, rp
for _ in range(reps):
    for i, v in enumerate(variants):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = kmc.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu", **v)
        torch.cuda.synchronize()
        res[i].append((time.perf_counter() - t0) * 1e3)
        del r
for i, v in enumerate(variants):
    print(v, "e2e ms", [round(x, 1) for x in res[i]], "median", round(float(np.median(res[i])), 1))
