"""Where the end-to-end (host-buffer) call spends its time on C4: per-stage CUDA events of a
profile=True call with pinned host inputs and a pinned host output, plus host wall clock of
kmc_count_begin and kmc_count_finish.  usage: python tools/e2e_breakdown.py [scale]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ctypes
import numpy as np
import torch

import paper_1407_1507_b200 as kmc
from paper_1407_1507_b200 import _options, _ptr, _check, _finish, load
import synth

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
w = synth.make("C4", scale=scale)
reads = torch.from_numpy(w.reads).pin_memory()
offs = torch.from_numpy(w.offsets.view(np.uint64)).pin_memory()
lib = load()
dbuf = torch.empty(reads.numel(), dtype=torch.uint8, device="cuda")
for _ in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    dbuf.copy_(reads, non_blocking=True); torch.cuda.synchronize()
    print(f"plain H2D of {reads.numel() / 1e9:.2f} GB: {1e3 * (time.perf_counter() - t0):.1f} ms")
del dbuf
for it in range(4):
    torch.cuda.synchronize()
    opt = _options(True, 0, False, 0, 0, 0, 0, 0, 0, True, False)
    job = ctypes.c_void_p()
    n_out = ctypes.c_uint64()
    t0 = time.perf_counter()
    _check(lib.kmc_count_begin(_ptr(reads), _ptr(offs), len(offs) - 1, w.k, w.p, 2, 10**9, None,
                               ctypes.byref(opt), ctypes.byref(job), ctypes.byref(n_out)))
    t1 = time.perf_counter()
    r = _finish(lib, job, int(n_out.value), w.k, "cpu")
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    st = r.stats
    print(f"iter {it}: begin {1e3 * (t1 - t0):.1f} ms, finish {1e3 * (t2 - t1):.1f} ms, total {1e3 * (t2 - t0):.1f} ms;"
          f" batches {st.get('n_input_batches')}")
    print("  stages:", {k_: round(v, 2) for k_, v in st["stage_ms"].items()})
    del r
def timed(tag, n=2, **kw):
    for it in range(n):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = kmc.count(reads, offs, w.k, w.p, 2, 10**9, out_device="cpu", **kw)
        torch.cuda.synchronize()
        print(f"{tag}: {1e3 * (time.perf_counter() - t0):.1f} ms")
        del r


timed("default block cache, legacy stream")
st = torch.cuda.Stream()
timed("default block cache, own stream", stream=st)
kmc.use_torch_allocator(True)
timed("torch allocator, legacy stream")
timed("torch allocator, own stream", stream=st)
kmc.use_torch_allocator(False)
timed("default block cache again, legacy stream")
