#!/usr/bin/env python
"""Small inputs through every path of the CUDA library, each checked against the oracle, for
compute-sanitizer runs (tools/sanitize.sh: memcheck, racecheck, synccheck, initcheck).  The
inputs are tiny so that the instrumented kernels finish in minutes: C1 and the other configs'
shapes at reduced scale, fuzzed random reads (N, lowercase, IUPAC bytes, empty reads), and
every forced path (large bins / split, per-chunk radix sort, device LSD, recompute
distribution, small-bin sort fallback, hash-table overflow fallback, host-streamed input,
k > 32, -b, debug hooks, DB writer).  Exit code 1 on any mismatch.
"""
import os
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_1407_1507_b200 as kmc  # noqa: E402


def check(w, label, k=None, canonical=True, host=False, **opts):
    k = k or w.k
    if host:
        r = torch.from_numpy(w.reads)
        o = torch.from_numpy(w.offsets.view(np.uint64))
        res = kmc.count(r, o, k, w.p, w.cutoff_min, w.cutoff_max, out_device="cpu", canonical=canonical, **opts)
    else:
        r = torch.from_numpy(w.reads).cuda() if w.reads.size else torch.zeros(0, dtype=torch.uint8, device="cuda")
        o = torch.from_numpy(w.offsets.view(np.uint64)).cuda()
        res = kmc.count(r, o, k, w.p, w.cutoff_min, w.cutoff_max, canonical=canonical, **opts)
    ref = oracle.count(w.reads, w.offsets, k, w.cutoff_min, w.cutoff_max, canonical=canonical)
    ok = np.array_equal(res.kmers.cpu().numpy(), ref.keys) and np.array_equal(res.counts.cpu().numpy(), ref.counts)
    print(f"{'ok  ' if ok else 'FAIL'} {label}: n_out={ref.n_out} windows={ref.n_windows}", flush=True)
    return ok


def main():
    only = sys.argv[1:]
    kmc.load()
    cases = []
    c1 = synth.make("C1", scale=0.005)
    cases += [("C1", c1, {}), ("C1 force_large", c1, dict(force_large=True)),
              ("C1 count_path=1", c1, dict(force_large=True, count_path=1)),
              ("C1 large_path=1 (device LSD)", c1, dict(force_large=True, large_path=1)),
              ("C1 distribute_path=1", c1, dict(distribute_path=1)),
              ("C1 small cap 64", c1, dict(small_bin_capacity=64)),
              ("C1 chunk cap 128", c1, dict(force_large=True, chunk_capacity=128)),
              ("C1 -b", c1, dict(canonical=False)),
              ("C1 host streamed", c1, dict(host=True, input_batch_mb=1, large_group_mkeys=1, force_large=True))]
    c3 = synth.make("C3", scale=0.0003)
    cases += [("C3 k=55", c3, {}), ("C3 force_large", c3, dict(force_large=True)),
              ("C3 count_path=1", c3, dict(force_large=True, count_path=1))]
    cases += [("C5", synth.make("C5", scale=0.0005), {}), ("C4", synth.make("C4", scale=0.0001), {}),
              ("C2", synth.make("C2", scale=0.0005), dict(force_large=True))]
    for seed in range(3):
        seqs = synth.random_reads(100 + seed, 300, 0, 180, n_frac=0.02, lower_frac=0.02, alphabet=b"ACGTNRY")
        for k, p in ((21, 5), (33, 7), (64, 9)):
            w = synth.from_strings(seqs, k, p, 1)
            cases.append((f"fuzz seed={seed} k={k}", w, dict(force_large=bool(seed & 1))))
    seqs = synth.random_reads(77, 1500, 100, 150, alphabet=b"ACGT")
    cases.append(("overflow fallback", synth.from_strings(seqs, 25, 5, 1),
                  dict(force_large=True, chunk_capacity=60000)))
    cases.append(("small-bin sort fallback", synth.from_strings(synth.random_reads(91, 2000, 80, 120), 25, 5, 1), {}))
    ok = True
    for label, w, opts in cases:
        if only and not any(x in label for x in only):
            continue
        opts = dict(opts)
        ok &= check(w, label, **opts)
    # debug hooks and the DB writer
    w = synth.make("C1", scale=0.002)
    r = torch.from_numpy(w.reads).cuda()
    o = torch.from_numpy(w.offsets.view(np.uint64)).cuda()
    sig = kmc.debug_signatures(r, o, w.k, w.p)
    ref = oracle.signatures(w.reads, w.offsets, w.k, w.p)
    good = np.array_equal(np.asarray(sig.cpu().numpy() if hasattr(sig, "cpu") else sig), ref)
    print(f"{'ok  ' if good else 'FAIL'} debug_signatures", flush=True)
    ok &= good
    res = kmc.count(r, o, w.k, w.p, 1, 10**9)
    with tempfile.TemporaryDirectory() as d:
        kmc.write_db(os.path.join(d, "db"), res.kmers, res.counts, w.k, w.p, 1, 10**9, 255)
    torch.cuda.synchronize()
    print("ALL OK" if ok else "MISMATCH", flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
