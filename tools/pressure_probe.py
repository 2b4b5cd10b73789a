"""C4 counts while most of the device memory is taken (experiments: the memory-bounded paths
under pressure, checked against a run without pressure)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_1407_1507_b200 as kmc
w = synth.make("C4", scale=1.0)
rh = torch.from_numpy(w.reads).pin_memory(); oh = torch.from_numpy(w.offsets.view(np.uint64)).pin_memory()
r0 = kmc.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu")
kmc.empty_cache(); torch.cuda.empty_cache()
for hold_gb in [int(x) for x in (sys.argv[1:] or ["100", "130"])]:
    hold = torch.empty(hold_gb << 30, dtype=torch.uint8, device="cuda")
    for dev_in in (False, True):
        R = rh.cuda() if dev_in else rh
        O = oh.cuda() if dev_in else oh
        try:
            r = kmc.count(R, O, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu")
            same = torch.equal(r.kmers, r0.kmers) and torch.equal(r.counts, r0.counts)
            print(f"hold {hold_gb} GB device_input={dev_in}: same={same} groups={r.stats['n_large_groups']} "
                  f"passes={r.stats['n_passes']}", flush=True)
            del r
        except Exception as ex:
            print(f"hold {hold_gb} GB device_input={dev_in}: {type(ex).__name__}: {str(ex)[:200]}", flush=True)
            raise
        del R, O
        kmc.empty_cache(); torch.cuda.empty_cache()
    del hold
    torch.cuda.empty_cache()
