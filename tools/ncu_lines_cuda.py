"""Per-source-line totals (instructions executed, stall samples) from
`ncu --page source --csv --print-source cuda,sass` output (CUDA lines carry the totals)."""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr = None
lines = []
fname = None
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) > 4 and r[0] and r[2] == "-":
        d = dict(zip(hdr[4:], r[4:]))
        lines.append((fname, r[0], r[1].strip(), float(d.get("Warp Stall Sampling (All Samples)") or 0),
                      float(d.get("Instructions Executed") or 0)))
ts = sum(l[3] for l in lines) or 1
ti = sum(l[4] for l in lines) or 1
print(f"total stall samples {ts:.0f}  warp instructions {ti:.3e}")
for l in sorted(lines, key=lambda x: -x[3])[:n]:
    print(f"{l[0]:>16}:{l[1]:<5} stall {100*l[3]/ts:5.1f}%  inst {100*l[4]/ti:5.1f}%  {l[2][:90]}")
