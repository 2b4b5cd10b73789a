"""GPU timeline of one C4 kmc_count call (torch.profiler / kineto CUDA activity): kernels and
copies in order, and the idle gaps between them (experiments; not a benchmark)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
import synth, paper_1407_1507_b200 as kmc
w = synth.make("C4", scale=float(sys.argv[1]) if len(sys.argv) > 1 else 1.0)
r = torch.from_numpy(w.reads).cuda(); o = torch.from_numpy(w.offsets.view(np.uint64)).cuda()
for _ in range(2): kmc.count(r, o, w.k, w.p, w.cutoff_min, w.cutoff_max)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    res = kmc.count(r, o, w.k, w.p, w.cutoff_min, w.cutoff_max)
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/trace.json")
ev = [e for e in json.load(open("/tmp/trace.json"))["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]; end = t0; gaps = []
rows = []
for e in ev:
    g = e["ts"] - end
    rows.append((round((e["ts"] - t0) / 1e3, 3), round(e["dur"] / 1e3, 3), round(g / 1e3, 3), e["name"][:60]))
    end = max(end, e["ts"] + e["dur"])
tot = (end - t0) / 1e3
busy = sum(e["dur"] for e in ev) / 1e3
print(f"span {tot:.2f} ms, {len(ev)} activities, sum of durations {busy:.2f} ms")
for row in rows:
    if row[2] > 0.02 or row[1] > 0.5: print(row)
