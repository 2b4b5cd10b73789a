#!/usr/bin/env python
"""Writes tests/golden/full_configs.json: the oracle's result on BASELINE.json's five configs
at full size, as a digest (SHA-256 of the sorted keys and counts, oracle.digest) plus the
statistics.  It calls only oracle/ and synth/ (never the CUDA path), so the GPU test that
compares against these values compares against the plain definition.

  python tools/make_goldens.py [C1 C2 ...]   (default: all five; C4 takes ~10 min on 8 cores)
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
import synth  # noqa: E402

OUT = os.path.join(ROOT, "tests", "golden", "full_configs.json")


def main(names):
    data = json.load(open(OUT)) if os.path.exists(OUT) else {
        "source": "tools/make_goldens.py: oracle.count_partitioned on synth.make(name) at full size "
                  "(oracle/ + synth/ only; PAPER.md P:L14-16 plain definition)",
        "configs": {}}
    for name in names:
        t0 = time.time()
        w = synth.make(name)
        r = oracle.count_partitioned(w.reads, w.offsets, w.k, w.cutoff_min, w.cutoff_max,
                                     round_keys=1 << 30)
        data["configs"][name] = {
            "k": w.k, "p": w.p, "cutoff_min": w.cutoff_min, "cutoff_max": w.cutoff_max,
            "n_reads": int(w.n_reads), "n_bases": int(w.n_bases),
            "n_windows": r.n_windows, "n_unique": r.n_unique, "n_below_min": r.n_below_min,
            "n_above_max": r.n_above_max, "n_out": r.n_out,
            "count_sum": int(r.counts.sum(dtype="u8")),
            "sha256": oracle.digest(r.keys, r.counts),
        }
        print(name, data["configs"][name], f"{time.time() - t0:.1f} s", flush=True)
        del w, r
        json.dump(data, open(OUT, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1:] or ["C1", "C2", "C3", "C5", "C4"])
