#!/usr/bin/env python
"""Aggregate an ncu report's source page (cuda,sass) per CUDA source line.

usage: python tools/ncu_lines.py REPORT.ncu-rep [function-substring] [top-N]
Prints, per function, the source lines with the most executed warp instructions and
warp-stall samples (requires -lineinfo at compile time and --import-source on).
"""
import csv
import io
import subprocess
import sys


def main():
    rep = sys.argv[1]
    fsub = sys.argv[2] if len(sys.argv) > 2 else ""
    top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    func = None
    hdr = None
    agg = {}
    src = {}
    cur_line = None
    for row in csv.reader(io.StringIO(out)):
        if not row:
            continue
        if row[0] == "Function Name":
            func = row[1]
            continue
        if row[0] == "File Path":
            continue
        if row[0] == "Line No":
            hdr = row
            continue
        if hdr is None or func is None or fsub not in func:
            continue
        d = dict(zip(hdr, row))
        addr = d.get("Address", "")
        if row[0].strip().isdigit() and not addr:
            cur_line = int(row[0])
            src[(func, cur_line)] = row[1][:90]
            continue
        if row[0].strip().isdigit():
            cur_line = int(row[0])
            src.setdefault((func, cur_line), row[1][:90])
        key = (func, cur_line)
        a = agg.setdefault(key, [0, 0])
        try:
            a[0] += int(float(d.get("Instructions Executed", "0") or 0))
            a[1] += int(float(d.get("Warp Stall Sampling (All Samples)", "0") or 0))
        except ValueError:
            pass
    funcs = sorted({f for f, _ in agg})
    for f in funcs:
        items = [(k, v) for k, v in agg.items() if k[0] == f]
        ti = sum(v[0] for _, v in items) or 1
        ts = sum(v[1] for _, v in items) or 1
        print(f"== {f}: {ti} warp instr, {ts} stall samples")
        byi = len(sys.argv) > 4 and sys.argv[4] == "instr"
        for (fn, line), (ins, st) in sorted(items, key=lambda kv: -kv[1][0 if byi else 1])[:top]:
            print(f"  L{line:4d} instr {100*ins/ti:5.1f}%  stalls {100*st/ts:5.1f}%  {src.get((fn, line), '')}")


if __name__ == "__main__":
    main()
