#!/usr/bin/env python
"""f2 at scale: a C4-shaped read set several times larger than the C4 config, host-resident,
whose single-pass working set (record stream + bins, ~5.4 bytes per base) exceeds the B200's
HBM, counted in passes over bin ranges.  Reports the time, the passes and the
statistics, and checks the result against the oracle on what the oracle can afford at this
size: the total window count (oracle_n_windows_par) and the exact counts of sampled survivors
(oracle_count_queries).  The byte-exact agreement of the multi-pass path with the in-HBM path
is tested on the full C4 config (tests/test_gpu_parity.py::test_multipass_full_c4_digest).

usage: python tools/beyond_hbm.py [scale=12] [n_sample=200]
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_1407_1507_b200 as kmc  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 12.0
n_sample = int(sys.argv[2]) if len(sys.argv) > 2 else 200
t0 = time.time()
w = synth.make("C4", scale=scale, n_threads=os.cpu_count())
t_gen = time.time() - t0
free, total = torch.cuda.mem_get_info()
t0 = time.time()
rh = torch.from_numpy(w.reads).pin_memory()
oh = torch.from_numpy(w.offsets.view(np.uint64)).pin_memory()
t_pin = time.time() - t0
kmc.load()
runs = []
torch.cuda.synchronize()
t0 = time.perf_counter()
res = kmc.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu", profile=True)
torch.cuda.synchronize()
runs.append(time.perf_counter() - t0)  # includes pinning the output tensors (host)
# again into the same pinned output buffers: the call alone
torch.cuda.synchronize()
t0 = time.perf_counter()
st = kmc.count_into(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, res.kmers, res.counts, profile=True)
torch.cuda.synchronize()
runs.append(time.perf_counter() - t0)
keys, counts = res.kmers.numpy(), res.counts.numpy()
# checks the oracle can afford at this size
t0 = time.time()
nw = oracle.n_windows_parallel(w.reads, w.offsets, w.k)
rng = np.random.default_rng(5)
idx = np.sort(rng.choice(keys.shape[0], min(n_sample, keys.shape[0]), replace=False))
ref = oracle.count_queries(w.reads, w.offsets, w.k, keys[idx])
t_chk = time.time() - t0
out = {
    "workload": f"C4 x{scale}: {w.n_reads} reads, {w.n_bases} bases (host-resident, pinned)",
    "device_free_gb": round(free / 1e9, 1), "device_total_gb": round(total / 1e9, 1),
    "single_pass_working_set_gb_est": round(w.n_bases * 5.4 / 1e9, 1),
    "seconds": [round(x, 3) for x in runs], "bases_per_s": w.n_bases / runs[1],
    "note": "seconds[0] includes pinning the 17 GB output tensors; seconds[1] is kmc_count_ex into them",
    "n_passes": st["n_passes"], "n_input_batches": st["n_input_batches"],
    "stats": {x: st[x] for x in ("n_windows", "n_unique", "n_out", "n_large_bins", "max_bin_windows")},
    "stage_ms": {x: round(v, 1) for x, v in st["stage_ms"].items() if v > 0},
    "check": {"oracle_n_windows": nw, "windows_equal": nw == st["n_windows"],
              "sampled_survivors": int(idx.size), "sampled_counts_equal": bool(np.array_equal(ref, counts[idx].astype(np.uint64))),
              "ascending": bool(np.all(keys[1:] > keys[:-1])), "seconds": round(t_chk, 1)},
    "host_seconds": {"generate": round(t_gen, 1), "pin": round(t_pin, 1)},
}
print(json.dumps(out))
