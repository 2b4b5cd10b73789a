"""Per-signature window histogram of a config (pass 1 through kmc_shard_pass1) and the share
of windows per size class: sizes the large-bin design.
usage: python tools/sig_hist.py [C4] [scale]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_1407_1507_b200 as kmc  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
w = synth.make(name, scale=scale)
r = torch.from_numpy(w.reads).cuda()
o = torch.from_numpy(w.offsets.view(np.uint64)).cuda()
sh = kmc._Shard(r, o, w.k, w.p, w.cutoff_min, w.cutoff_max)
h = sh.hist_w.cpu().numpy().astype(np.float64)
hr = sh.hist_r.cpu().numpy().astype(np.float64)
del sh
tot = h.sum()
nz = h[h > 0]
print(f"{name} x{scale}: windows {tot:.4g}, records {hr.sum():.4g}, signatures used {len(nz)}, max {nz.max():.0f}")
for lim in (6144, 20000, 46000, 92000, 184000, 368000, 736000, 1500000):
    print(f"  <= {lim:8d}: {nz[nz <= lim].sum() / tot:.3f} of windows, {int((nz > lim).sum())} signatures above")
ratio = 0.26
for C in (1, 2, 4, 8, 16):
    cap = C * 9200 / ratio  # windows per round at ~9.2K distinct per CTA
    R = np.ceil(nz / cap)
    print(f"  cluster {C:2d}: window-weighted rounds E[R] = {(R * nz).sum() / tot:.2f}, max R {R.max():.0f}")
np.save("/tmp/sig_hist.npy", h)
