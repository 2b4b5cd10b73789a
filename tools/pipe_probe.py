"""Do two kmc_count calls on two host threads / two streams overlap?  Host timestamps of every
call (experiments; not a benchmark)."""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_1407_1507_b200 as kmc
w = synth.make("C4", scale=float(sys.argv[1]) if len(sys.argv) > 1 else 1.0)
rh = torch.from_numpy(w.reads).pin_memory(); oh = torch.from_numpy(w.offsets.view(np.uint64)).pin_memory()
if os.environ.get("KMC_TORCH_ALLOC"): kmc.use_torch_allocator(True)
OPTS = eval(os.environ.get("KMC_OPTS", "dict()"))
hold = torch.empty(int(os.environ.get("KMC_HOLD", "0")) * (20 << 30), dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
T0 = time.perf_counter(); log = []
w2 = synth.make("C4", scale=0.1) if os.environ.get("SMALL2") else w
rh2 = torch.from_numpy(w2.reads).pin_memory(); oh2 = torch.from_numpy(w2.offsets.view(np.uint64)).pin_memory()
def call(i, tag):
    t = time.perf_counter()
    R, O = (rh2, oh2) if i == 1 else (rh, oh)
    r = kmc.count(R, O, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device=os.environ.get("OUTDEV", "cpu"), stream=streams[i], **OPTS)
    log.append((tag, i, round((t - T0) * 1e3, 1), round((time.perf_counter() - T0) * 1e3, 1)))
    del r
for i in range(2): call(i, "warm")
torch.cuda.synchronize(); T0 = time.perf_counter(); log.clear()
for i in range(2): call(0, "serial")
torch.cuda.synchronize(); T0 = time.perf_counter()
def worker(i):
    with torch.cuda.stream(streams[i]):
        for j in range(3): call(i, "pipe")
ths = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
[t.start() for t in ths]; [t.join() for t in ths]; torch.cuda.synchronize()
print(round((time.perf_counter() - T0) * 1e3, 1), "ms for 6 pipelined calls")
for x in log: print(x)
