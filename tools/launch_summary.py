"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv --log-file X):
per-kernel launches and total time, optionally per call (divide by --calls)."""
import csv, sys, collections
path = sys.argv[1]
calls = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
hdr = rows[0]
ki, mi, ui, vi = hdr.index("Kernel Name"), hdr.index("Metric Name"), hdr.index("Metric Unit"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if r[mi] != "gpu__time_duration.sum":
        continue
    v = float(r[vi].replace(",", ""))
    v *= {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(r[ui], 1.0)
    name = r[ki].split("(")[0].replace("void ", "").replace("kmc::", "").replace("<unnamed>::", "")
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
print(f"{'kernel':45s} {'launches':>8s} {'ms/call':>9s} {'share':>6s}")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k[:45]:45s} {n/calls:8.1f} {t/calls:9.3f} {t/tot:6.3f}")
print(f"{'TOTAL':45s} {sum(v[0] for v in agg.values())/calls:8.1f} {tot/calls:9.3f}")
