"""Top SASS lines by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) >= len(hdr) - 1 and r[0] not in ("Address", "Kernel Name")]
tot = sum(float(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
idx = {id(d): i for i, d in enumerate(data)}
top = sorted(data, key=lambda d: -float(d["Warp Stall Sampling (All Samples)"] or 0))[:n]
print(f"total samples {tot:.0f}, instructions {len(data)}")
for d in top:
    s = float(d["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{idx[id(d)]:5d} {s/tot*100:5.1f}%  {d['Instructions Executed']:>10}  {d['Source'].strip()[:80]}")
