"""Per-kernel summary of an ncu report: time, DRAM bytes, throughput, issue, top stalls."""
import csv, io, subprocess, sys
rep = sys.argv[1]
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
     "sm__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
     "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
     "smsp__inst_executed_op_shared_atom.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread"]
ST = ["barrier", "short_scoreboard", "long_scoreboard", "mio_throttle", "lg_throttle", "wait", "math_pipe_throttle",
      "no_instructions", "selected", "not_selected", "membar", "dispatch_stall", "branch_resolving", "drain", "sleeping"]
mm = M + ["smsp__pcsamp_warps_issue_stalled_" + s for s in ST] + ["smsp__pcsamp_sample_count"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(mm)], capture_output=True,
                     text=True).stdout
r = list(csv.reader(io.StringIO(out)))
h, units = r[0], r[1]
for row in r[2:]:
    d = dict(zip(h, row))
    u = dict(zip(h, units))
    t = float(d["gpu__time_duration.sum"]) * {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3, "s": 1e3}[u["gpu__time_duration.sum"]]
    def gb(x):
        v = float(d[x]); un = u[x]
        return v * {"byte": 1e-9, "Kbyte": 1e-6, "Mbyte": 1e-3, "Gbyte": 1.0, "B": 1e-9, "KB": 1e-6, "MB": 1e-3, "GB": 1.0}.get(un, 1e-9)
    rd, wr = gb("dram__bytes_read.sum"), gb("dram__bytes_write.sum")
    tot = float(d["smsp__pcsamp_sample_count"] or 1)
    stalls = sorted(((float(d["smsp__pcsamp_warps_issue_stalled_" + s] or 0) / tot, s) for s in ST), reverse=True)[:4]
    print(f"{d['Kernel Name'][:60]:60s} {t:8.3f} ms  rd {rd:6.2f} GB wr {wr:6.2f} GB  {(rd+wr)/t:7.1f} GB/s  "
          f"issue {float(d['smsp__issue_active.avg.pct_of_peak_sustained_active']):4.1f}%  "
          f"warps {float(d['sm__warps_active.avg.pct_of_peak_sustained_active']):4.1f}%  "
          f"inst {float(d['smsp__inst_executed.sum'])/1e6:8.1f}M  grid {d['launch__grid_size']}x{d['launch__block_size']} "
          f"regs {d['launch__registers_per_thread']}  atoms {float(d['smsp__inst_executed_op_shared_atom.sum'])/1e6:.1f}M  "
          f"bankc {float(d['l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum'])/1e6:.1f}M")
    print("      stalls: " + ", ".join(f"{s} {v*100:.0f}%" for v, s in stalls))
