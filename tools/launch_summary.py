"""Summarise an ncu launch list of bench.py / profile_run.py.

usage: python tools/launch_summary.py LAUNCHES.csv [timed_calls]

The CSV comes from `ncu --metrics gpu__time_duration.sum[,dram__bytes_read.sum,
dram__bytes_write.sum] --clock-control none --csv --log-file LAUNCHES.csv <command>`.
Launches are grouped into kmc_count calls (each call starts with k_tile_reads); the last
`timed_calls` calls are averaged (default: all).  Prints per-kernel launches, ms, share,
and DRAM GB per call.  ncu serialises launches and runs them cold: compare SHARES with the
live per-stage CUDA-event times of bench.py, not absolutes.
"""
import collections
import csv
import sys

UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
        "byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0}


def main():
    path = sys.argv[1]
    rows = [r for r in csv.reader(open(path)) if r and not r[0].startswith("==")]
    h = rows[0]
    ki, mi, ui, vi, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    by_id = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        lid = int(r[ii])
        names[lid] = r[ki].split("(")[0].replace("void ", "").replace("kmc::", "").replace("<unnamed>::", "")
        by_id[lid][r[mi]] = float(r[vi].replace(",", "")) * UNIT.get(r[ui], 1.0)
    calls, cur = [], None
    for lid in sorted(by_id):
        if "k_tile_reads" in names[lid]:
            cur = []
            calls.append(cur)
        if cur is not None:
            cur.append(lid)
    n_timed = int(sys.argv[2]) if len(sys.argv) > 2 else len(calls)
    sel = [lid for c in calls[-n_timed:] for lid in c]
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for lid in sel:
        a = agg[names[lid]]
        a[0] += 1
        a[1] += by_id[lid].get("gpu__time_duration.sum", 0.0)
        a[2] += by_id[lid].get("dram__bytes_read.sum", 0.0)
        a[3] += by_id[lid].get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    print(f"# {len(calls)} kmc_count calls in the list, last {n_timed} averaged ({len(sel)} launches)")
    print(f"{'kernel':48s} {'launches':>8s} {'ms/call':>9s} {'share':>6s} {'rd GB':>7s} {'wr GB':>7s}")
    for k, (n, t, rd, wr) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k[:48]:48s} {n / n_timed:8.1f} {t / n_timed:9.3f} {t / tot:6.3f} {rd / n_timed:7.2f} {wr / n_timed:7.2f}")
    print(f"{'TOTAL':48s} {len(sel) / n_timed:8.1f} {tot / n_timed:9.3f}")


if __name__ == "__main__":
    main()
