"""Warp instructions per kmc_count call from an ncu launch list that carries
smsp__inst_executed.sum (one row per launch and metric), averaged over the calls in the list
(a call = one k_tile_reads launch).  usage: python tools/inst_summary.py LAUNCHES.csv [n_windows]"""
import collections
import csv
import sys

rows = [r for r in csv.reader(open(sys.argv[1])) if r and not r[0].startswith("==")]
h = rows[0]
ki, mi, vi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value"))
inst = collections.Counter()
calls = 0
for r in rows[1:]:
    if r[mi] != "smsp__inst_executed.sum":
        continue
    name = r[ki].split("(")[0].replace("void ", "").replace("kmc::", "").replace("<unnamed>::", "").replace("unnamed>::", "")
    inst[name] += float(r[vi].replace(",", ""))
    calls += name.startswith("k_tile_reads")
n_windows = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
tot = sum(inst.values()) / calls
peak = 148 * 4 * 1.965e9
print(f"# warp instructions per kmc_count call ({calls} calls averaged); issue peak = 148 SMs x 4 schedulers"
      f" x 1.965 GHz = {peak / 1e9:.0f} G warp instructions/s")
print(f"# whole call: {tot:.4g} warp instructions = {1e3 * tot / peak:.1f} ms at full issue")
print(f"{'kernel':52s} {'warp inst':>12s}" + (f" {'per window':>10s}" if n_windows else ""))
for name, v in inst.most_common():
    line = f"{name[:52]:52s} {v / calls:12.4e}"
    if n_windows:
        line += f" {32 * v / calls / n_windows:10.1f}"
    print(line)
