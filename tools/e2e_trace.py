"""GPU timeline of the tail of one end-to-end C4 call (pinned host inputs and outputs): the
S9 kernels and the output copies, from torch.profiler (experiments; not a benchmark)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from torch.profiler import profile, ProfilerActivity
import synth, paper_1407_1507_b200 as kmc
w = synth.make("C4", scale=float(sys.argv[1]) if len(sys.argv) > 1 else 1.0)
rh = torch.from_numpy(w.reads).pin_memory(); oh = torch.from_numpy(w.offsets.view(np.uint64)).pin_memory()
for _ in range(2): kmc.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu")
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    res = kmc.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu")
    torch.cuda.synchronize()
prof.export_chrome_trace("/tmp/trace_e2e.json")
ev = [e for e in json.load(open("/tmp/trace_e2e.json"))["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]; tend = max(e["ts"] + e["dur"] for e in ev)
print(f"span {(tend - t0) / 1e3:.2f} ms")
s9 = [e for e in ev if "k_ord" in e["name"] or "k_tile" in e["name"]]
ts9 = s9[0]["ts"] if s9 else t0
for e in ev:
    if e["ts"] < ts9 - 20000: continue
    n = e["name"]
    if e["cat"] == "gpu_memcpy" or e["dur"] > 100 or "k_ord" in n:
        print(f"{(e['ts'] - ts9) / 1e3:9.3f} {e['dur'] / 1e3:8.3f} {n[:70]}")
