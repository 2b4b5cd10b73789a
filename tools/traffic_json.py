"""profiles/rNN_traffic.json from an ncu launch list of the bench command that carries
gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum and smsp__inst_executed.sum
(tools/r2_profile_suite.sh).  Per stage: the DRAM bytes and warp instructions per call of its
kernels; per call: the totals over every kernel (B_impl and the call's instruction count).
usage: python tools/traffic_json.py LAUNCHES.csv TIMED_CALLS OUT.json [workload] [scale]"""
import collections
import csv
import json
import sys

UNIT = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
        "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1.0, "warp": 1.0}
STAGE = [("k_sig<", "signature"), ("k_rec_scatter", "scatter"), ("k_small_bins", "small_bins"),
         ("k_small_kx", "small_bins"), ("k_split1<", "large_scatter"), ("k_split1_chunks", "large_scatter"),
         ("k_split<unsigned long, 0", "large_split"), ("k_split<unsigned long, 1", "large_scatter"),
         ("k_chunk_hash", "large_chunks"), ("k_chunk_sort", "large_chunks"), ("k_clcount", "large_chunks"),
         ("k_ord", "order"), ("k_order_chunk_sort", "order")]


def stage_of(name):
    for pre, st in STAGE:
        if pre in name:
            return st
    return None


def main():
    path, n_timed, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    workload = sys.argv[4] if len(sys.argv) > 4 else "C4"
    scale = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
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
    sel = [lid for c in calls[-n_timed:] for lid in c]
    stages = collections.defaultdict(lambda: {"kernels": set(), "dram_bytes_read": 0.0, "dram_bytes_write": 0.0,
                                              "warp_inst": 0.0, "ms": 0.0})
    tot = {"dram_bytes": 0.0, "warp_inst": 0.0, "ms": 0.0}
    for lid in sel:
        m = by_id[lid]
        rd, wr = m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0)
        wi, ms = m.get("smsp__inst_executed.sum", 0.0), m.get("gpu__time_duration.sum", 0.0)
        tot["dram_bytes"] += rd + wr
        tot["warp_inst"] += wi
        tot["ms"] += ms
        st = stage_of(names[lid])
        if st:
            e = stages[st]
            e["kernels"].add(names[lid].split("<")[0])
            e["dram_bytes_read"] += rd
            e["dram_bytes_write"] += wr
            e["warp_inst"] += wi
            e["ms"] += ms
    res = {"note": f"per kmc_count call, averaged over the last {n_timed} calls of the ncu launch list {path} "
                   "(serialised, cold-cache launches: compare shares, not absolutes, with the live stage times)",
           "workload": workload, "scale": scale, "sm_clock_ghz": 1.965,
           "stages": {k: {"kernel": " + ".join(sorted(v["kernels"])), "dram_bytes_read": v["dram_bytes_read"] / n_timed,
                          "dram_bytes_write": v["dram_bytes_write"] / n_timed, "warp_inst": v["warp_inst"] / n_timed,
                          "ncu_ms": v["ms"] / n_timed} for k, v in stages.items()},
           "call": {k: v / n_timed for k, v in tot.items()}}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res["call"]), {k: round(v["ncu_ms"], 2) for k, v in res["stages"].items()})


if __name__ == "__main__":
    main()
