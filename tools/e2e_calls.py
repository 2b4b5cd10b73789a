"""Per-call end-to-end times of C4 through the public API (pinned host inputs, outputs on the
host), to see the spread between calls (experiments; not a benchmark)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_1407_1507_b200 as kmc
w = synth.make("C4", scale=1.0)
rh = torch.from_numpy(w.reads).pin_memory(); oh = torch.from_numpy(w.offsets.view(np.uint64)).pin_memory()
for it in range(10):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = kmc.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu")
    e1.record(); torch.cuda.synchronize()
    print(f"call {it}: {e0.elapsed_time(e1):.1f} ms event, {1e3 * (time.perf_counter() - t0):.1f} ms wall", flush=True)
    del r
