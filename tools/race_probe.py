"""One kmc_count call on host reads while another thread keeps the GPU busy with torch work
(experiments: does pass 1 depend on timing?)."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_1407_1507_b200 as kmc
w = synth.make("C4", scale=float(sys.argv[1]) if len(sys.argv) > 1 else 1.0)
rh = torch.from_numpy(w.reads).pin_memory(); oh = torch.from_numpy(w.offsets.view(np.uint64)).pin_memory()
r0 = kmc.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu")
stop = False
def busy():
    s = torch.cuda.Stream(); a = torch.randn(8192, 8192, device="cuda"); 
    with torch.cuda.stream(s):
        while not stop:
            for _ in range(20): a = (a @ a).clamp_(-1, 1)
            s.synchronize()
t = threading.Thread(target=busy); t.start()
ok = True
try:
    for i in range(3):
        r = kmc.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu", stream=torch.cuda.Stream())
        same = torch.equal(r.kmers, r0.kmers) and torch.equal(r.counts, r0.counts)
        print("call", i, "same", same); ok &= same
finally:
    stop = True; t.join()
print("OK" if ok else "MISMATCH")
