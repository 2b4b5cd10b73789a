# two processes, each counting C4 from host reads three times, concurrently on one GPU
cat > /tmp/one.py <<'PY'
import os, sys, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import synth, paper_1407_1507_b200 as kmc
w = synth.make("C4", scale=1.0)
rh = torch.from_numpy(w.reads).pin_memory(); oh = torch.from_numpy(w.offsets.view(np.uint64)).pin_memory()
r0 = kmc.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu")
t = time.time()
for i in range(4):
    r = kmc.count(rh, oh, w.k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu")
    print(sys.argv[1], i, torch.equal(r.kmers, r0.kmers), round(time.time() - t, 2), flush=True)
PY
timeout 600 python /tmp/one.py A & pa=$!
timeout 600 python /tmp/one.py B & pb=$!
wait $pa; echo "A rc $?"; wait $pb; echo "B rc $?"
