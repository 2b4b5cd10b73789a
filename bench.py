#!/usr/bin/env python
"""bench.py -- canonical k-mer counting (KMC 2 hot path) on B200.

Default workload: BASELINE.json configs[3] ("C4": 100 Mbp x 40x, 40M x 100 bp reads,
k=28, p=9, ci=2, cx=1e9), the configuration the metric is quoted on.  One "step" is one
full kmc_count call (S1-S9) over the whole read set, inputs resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl kmcgpu|reference] [--config C4]

N > 1 runs under torchrun, one rank per GPU: rank r holds its own read sample of the same
genome (C4 reads each: weak scaling) and the ranks count the union with the sharded path
(kmc_shard_*): NCCL all-reduce of the signature histograms, the partition pass
writing every super-k-mer record into its bin owner's receive buffer over peer memory (the
fused exchange), each rank counting and outputting its own bins.  The time
is the max over ranks.
``--impl reference`` times the CPU oracle (oracle/) on the host cores, rank 0 only.
Prints ONE JSON line (rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "input bases/s (k-mers counted/s and HBM-roofline fraction alongside)"

# Algorithmic HBM bytes per stage.  Each entry: (bytes per launch, launches)
# computed from the per-call statistics.


def compact_bin_bytes(st: dict, k: int) -> float:
    """Bytes of the bins in SURVEY 8(d)'s model: every super-k-mer stored once as a 1-byte
    length header + its n + k - 1 symbols at 2 bits (n windows).  From the call's statistics:
    sum(n + k - 1) = n_windows + n_superkmers * (k - 1)."""
    return st["n_superkmers"] * 1.0 + 2.0 * (st["n_windows"] + st["n_superkmers"] * (k - 1)) / 8.0


def stage_bytes(st: dict, n_reads: int, k: int, ran: set = frozenset({"large_split"})) -> dict:
    """Algorithmic HBM bytes per stage and call, SURVEY 8(d):
    B_alg = input (ASCII + offsets) + 2 x compact bins (written once, read once) + output.
    Each byte of B_alg is charged to the stage that must move it: pass 1 reads the input and
    writes the bins, the counting stages read them, S9 writes the output.  Passes the model
    does not have (S5's re-sort, the large-bin key split and its re-read) get 0: their traffic
    is implementation overhead, reported as B_impl (ncu), never as algorithmic."""
    ksz = 8 if k <= 32 else 16
    nb = st["n_bases"]
    off = 8 * (n_reads + 1)
    bins = compact_bin_bytes(st, k)
    lw = st["large_windows"]
    lfrac = lw / st["n_windows"] if st["n_windows"] else 0.0
    # the large bins' records are read by the first large stage that ran: the count pass of the
    # two-pass split (large_path 2), else the one-pass split (default), else the cluster kernel
    large_reader = next((x for x in ("large_split", "large_scatter", "large_chunks") if x in ran), "large_split")
    out = {
        "signature": nb + off + bins,        # input read, bins written once
        "scatter": 0.0,                      # implementation pass (record stream -> bins)
        "small_bins": (1 - lfrac) * bins,    # bins read once
        "large_split": 0.0,
        "large_scatter": 0.0,
        "large_chunks": 0.0,                 # implementation pass (re-read of the split keys)
        "large_fallback": 0.0,
        "order": st["n_out"] * (ksz + 4),    # output written once
        "output": 0.0,
    }
    out[large_reader] = lfrac * bins         # large bins read once
    return out


def b_alg(st: dict, n_reads: int, k: int) -> float:
    ksz = 8 if k <= 32 else 16
    return st["n_bases"] + 8 * (n_reads + 1) + 2 * compact_bin_bytes(st, k) + st["n_out"] * (ksz + 4)


def latest_traffic(config: str, scale: float):
    """The newest profiles/r*_traffic.json written from ncu captures of this workload."""
    import glob
    best = None
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json"))):
        try:
            tj = json.load(open(path))
        except (OSError, ValueError):
            continue
        if tj.get("workload") == config and float(tj.get("scale", 0)) == scale:
            best = (path, tj)
    return best


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = "index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active," \
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        self.proc.wait()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        smax = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(rows)}


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_oracle_sample(w, n_reads_sample: int, threads: int):
    """The oracle, as it stands, on the first n_reads_sample reads: the key-range-partitioned
    form (SURVEY 8(d) "Oracle timing") on `threads` host threads."""
    import oracle
    n = min(n_reads_sample, w.n_reads)
    offs = w.offsets[: n + 1]
    reads = w.reads[: int(offs[-1])]
    t0 = time.perf_counter()
    r = oracle.count_partitioned(reads, offs, w.k, w.cutoff_min, w.cutoff_max, threads=threads)
    dt = time.perf_counter() - t0
    return dt, int(offs[-1] - offs[0]), r.n_windows, n




def pipelined_only(args):
    """--e2e-pipelined-only: the two-stream e2e measurement alone, one JSON line."""
    import torch
    import paper_1407_1507_b200 as kmc
    torch.cuda.set_device(0)
    kmc.load()
    w = synth.make(args.config, scale=args.scale, n_threads=os.cpu_count() or 8)
    reads_h = torch.from_numpy(w.reads).pin_memory()
    offs_h = torch.from_numpy(w.offsets.view(np.uint64)).pin_memory()
    r = e2e_pipelined(kmc, reads_h, offs_h, w.k, w.p, w.cutoff_min, w.cutoff_max, args.count_path,
                      max(1, min(args.steps, 3)), w.n_bases)
    print(json.dumps(r))

def e2e_pipelined(kmc, reads_h, offs_h, k, p, ci, cx, count_path, e_steps, n_bases):
    """The e2e call from two host threads on two streams: one call's device stages and output
    copy overlap the next call's input copy (PCIe is full duplex; the library lets the input
    copies of concurrent calls cross the link one after another).  Every call still copies its
    own inputs in and its own output out.  Reported beside e2e, whose single-call figure stays
    the headline."""
    import threading
    import torch
    # two calls in flight need two sets of scratch (~60 GB each at C4): the cache of the calls
    # before (another stream's blocks) and torch's are returned first
    kmc.empty_cache()
    torch.cuda.empty_cache()
    streams = [torch.cuda.Stream(), torch.cuda.Stream()]
    per = max(2, e_steps)
    ev_start = torch.cuda.Event(enable_timing=True)
    ev_end = [torch.cuda.Event(enable_timing=True) for _ in streams]
    errs = []

    def worker(i):
        try:
            with torch.cuda.stream(streams[i]):
                for _ in range(per):
                    rr = kmc.count(reads_h, offs_h, k, p, ci, cx, out_device="cpu", count_path=count_path,
                                   stream=streams[i])
                    del rr
                ev_end[i].record(streams[i])
        except Exception as ex:  # re-raised below
            errs.append(ex)

    for st_ in streams:  # each stream's scratch cache warmed first
        with torch.cuda.stream(st_):
            rr = kmc.count(reads_h, offs_h, k, p, ci, cx, out_device="cpu", count_path=count_path, stream=st_)
            del rr
    torch.cuda.synchronize()
    ev_start.record(torch.cuda.current_stream())
    for st_ in streams:
        st_.wait_event(ev_start)
    ths = [threading.Thread(target=worker, args=(i,)) for i in range(2)]
    for t_ in ths:
        t_.start()
    for t_ in ths:
        t_.join()
    torch.cuda.synchronize()
    if errs:
        raise errs[0]
    p_ms = max(ev_start.elapsed_time(e_) for e_ in ev_end) / (2 * per)
    return {"value": n_bases / (p_ms / 1e3), "unit": "bases/s", "ms_per_step": round(p_ms, 3), "calls": 2 * per,
            "streams": 2, "note": "two host threads, one stream each; every call copies its inputs in and its "
                                  "output out; per-step = time of all calls / calls"}

def reduce_max(value: float, world: int, device=None) -> float:
    """Max over ranks (the timing rule: a multi-GPU step takes as long as its slowest rank)."""
    if world <= 1:
        return value
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="kmcgpu", choices=["kmcgpu", "reference"])
    ap.add_argument("--config", default="C4")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--e2e-pipelined", action="store_true",
                    help="also time the e2e call with two calls in flight (two threads / streams, in a "
                         "subprocess); off by default: concurrent calls in one process are not supported "
                         "yet (DESIGN.md 12)")
    ap.add_argument("--e2e-pipelined-only", action="store_true",
                    help="(internal) run only the two-stream e2e measurement and print its JSON")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-reads", type=int, default=3_000_000)
    ap.add_argument("--no-sort-path", action="store_true",
                    help="skip the second timing of the paper's per-chunk radix sort (count_path 1)")
    ap.add_argument("--count-path", type=int, default=0, choices=[0, 1],
                    help="S7-S8 of large-bin chunks: 0 = SMEM hash count (default), 1 = SMEM radix sort + RLE")
    args = ap.parse_args()
    world, rank, local = dist_setup(args)
    cfg = synth.CONFIGS[args.config]

    if args.impl == "reference":
        return reference_arm(args, world, rank, cfg)
    if args.e2e_pipelined_only:
        return pipelined_only(args)

    import torch
    import torch.distributed as dist
    import paper_1407_1507_b200 as kmc

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    kmc.load()

    gen_threads = max(1, (os.cpu_count() or 8) // max(1, world))
    # N > 1: rank r holds its own read sample of the same genome (weak scaling) and the ranks
    # count the union together: histogram all-reduce + all-to-all of the super-k-mer records
    # by bin owner over NCCL; each rank outputs the k-mers of its bins
    w = synth.make(args.config, scale=args.scale, n_threads=gen_threads, shard=rank)
    n_bases = w.n_bases
    reads_d = torch.from_numpy(w.reads).cuda()
    offs_d = torch.from_numpy(w.offsets.view(np.uint64)).cuda()
    k, p, ci, cx = w.k, w.p, w.cutoff_min, w.cutoff_max
    stream = torch.cuda.current_stream()

    xmode = {"mode": "p2p"}  # N > 1: the fused exchange over peer memory, else the all-to-all

    def step(profile=True):
        if world > 1:
            return kmc.count_sharded(reads_d, offs_d, k, p, ci, cx, profile=profile, count_path=args.count_path,
                                     exchange_mode=xmode["mode"])
        return kmc.count(reads_d, offs_d, k, p, ci, cx, profile=profile, count_path=args.count_path)

    if world > 1:
        try:
            del_res = step()
            del del_res
        except kmc.KmcError as e:  # every rank raises together (the exchange's success is all-reduced)
            print(f"rank {rank}: fused P2P exchange unavailable ({e}); using the NCCL all-to-all", file=sys.stderr)
            xmode["mode"] = "collective"

    for _ in range(max(3, args.warmup)):
        res = step()
        del res
    torch.cuda.synchronize()

    clocks = ClockSampler(local)
    clocks.start()
    stage_ms = {}
    stage_launches = {}
    n_launches = 0
    last = None
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        res = step()
        for s_, v in res.stats["stage_ms"].items():
            stage_ms[s_] = stage_ms.get(s_, 0.0) + v
        for s_, v in res.stats["stage_launches"].items():
            stage_launches[s_] = stage_launches.get(s_, 0) + v
        n_launches += res.stats["n_launches"]
        last = res.stats
        del res
    ev1.record(stream)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    ms = reduce_max(ev0.elapsed_time(ev1) / args.steps, world, "cuda")

    # ---- the paper's method (per-chunk radix sort + run-length compaction, count_path 1) timed
    #      from the same build next to the default hash counting (reading R-S7)
    other = None
    if world == 1 and not args.no_sort_path:
        cp2 = 1 - args.count_path
        for _ in range(2):
            res = kmc.count(reads_d, offs_d, k, p, ci, cx, profile=True, count_path=cp2)
            del res
        torch.cuda.synchronize()
        o_steps = max(1, min(args.steps, 3))
        o_stage = {}
        q0 = torch.cuda.Event(enable_timing=True)
        q1 = torch.cuda.Event(enable_timing=True)
        q0.record(stream)
        for _ in range(o_steps):
            res = kmc.count(reads_d, offs_d, k, p, ci, cx, profile=True, count_path=cp2)
            for s_, v in res.stats["stage_ms"].items():
                o_stage[s_] = o_stage.get(s_, 0.0) + v
            o_out = res.stats["n_out"]
            del res
        q1.record(stream)
        torch.cuda.synchronize()
        o_ms = q0.elapsed_time(q1) / o_steps
        other = {"count_path": ["smem_hash", "smem_radix_sort"][cp2], "ms_per_step": round(o_ms, 3),
                 "value": n_bases / (o_ms / 1e3), "unit": "bases/s", "n_out": o_out,
                 "stages_ms": {s_: round(v / o_steps, 3) for s_, v in o_stage.items() if v > 0}}

    # ---- e2e: same call with pinned HOST buffers (H2D of inputs and D2H of outputs inside)
    e2e = None
    if not args.no_e2e:
        reads_h = torch.from_numpy(w.reads).pin_memory()
        offs_h = torch.from_numpy(w.offsets.view(np.uint64)).pin_memory()
        # the device-resident legs above leave their scratch in the library's block cache and
        # in torch's; the e2e call starts from an empty cache, which its untimed warm-up calls fill
        torch.cuda.synchronize()
        kmc.empty_cache()
        torch.cuda.empty_cache()
        def e2e_step():
            if world > 1:
                return kmc.count_sharded(reads_h, offs_h, k, p, ci, cx, out_device="cpu", count_path=args.count_path,
                                         exchange_mode=xmode["mode"])
            return kmc.count(reads_h, offs_h, k, p, ci, cx, out_device="cpu", count_path=args.count_path)
        for _ in range(2):
            r = e2e_step()
            n_out = r.stats["n_out"]
            del r
        e_steps = max(1, min(args.steps, 5))
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(e_steps):
            r = e2e_step()
            del r
        e1.record(stream)
        torch.cuda.synchronize()
        e_ms = reduce_max(e0.elapsed_time(e1) / e_steps, world, "cuda")
        e2e = {"value": world * n_bases / (e_ms / 1e3), "unit": "bases/s",
               "ms_per_step": e_ms, "h2d_bytes_per_step": int(w.reads.nbytes + w.offsets.nbytes),
               "d2h_bytes_per_step": int(n_out * ((8 if k <= 32 else 16) + 4))}
        # context: the link itself -- one plain copy of the same pinned reads and offsets
        scratch = torch.empty(w.reads.nbytes + w.offsets.nbytes, dtype=torch.uint8, device="cuda")
        l0 = torch.cuda.Event(enable_timing=True)
        l1 = torch.cuda.Event(enable_timing=True)
        l0.record(stream)
        scratch[:w.reads.nbytes].copy_(reads_h, non_blocking=True)
        scratch[w.reads.nbytes:].copy_(offs_h.view(torch.uint8), non_blocking=True)
        l1.record(stream)
        torch.cuda.synchronize()
        link_ms = l0.elapsed_time(l1)
        e2e["link_h2d"] = {"ms": round(link_ms, 2), "gbs": round(e2e["h2d_bytes_per_step"] / (link_ms / 1e3) / 1e9, 1),
                           "note": "one plain copy of the same pinned inputs; the e2e step cannot be faster"}
        del scratch
        if world == 1 and args.e2e_pipelined:
            # in a process of its own (its own CUDA context), after this one's scratch is returned:
            # whatever happens there cannot touch this run's numbers
            kmc.empty_cache()
            torch.cuda.empty_cache()
            try:
                cmd = [sys.executable, os.path.abspath(__file__), "--e2e-pipelined-only", "--config", args.config,
                       "--scale", str(args.scale), "--steps", str(e_steps), "--count-path", str(args.count_path)]
                pr = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
                line = [l_ for l_ in pr.stdout.splitlines() if l_.startswith("{")]
                e2e["pipelined"] = json.loads(line[-1]) if pr.returncode == 0 and line else \
                    {"error": f"rc {pr.returncode}: {pr.stderr.strip()[-300:]}"}
            except Exception as ex:  # the single-call e2e above stands; the failure is reported
                e2e["pipelined"] = {"error": f"{type(ex).__name__}: {ex}"[:300]}

    windows_all = float(last["n_windows"])  # N > 1: this rank's bins; summed over ranks below
    if world > 1:
        t = torch.tensor([windows_all], dtype=torch.float64, device="cuda")
        dist.all_reduce(t)
        windows_all = float(t.item())
    if rank != 0:
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    # ---- roofline of the dominant stage (SURVEY 8(d) bytes)
    peaks = measured_peaks()
    sb = stage_bytes(last, w.n_reads, k, ran={s_ for s_, v in stage_ms.items() if v > 0})
    per_stage = {}
    for s_, tot in stage_ms.items():
        if tot <= 0:
            continue
        per_step = tot / args.steps
        bytes_ = sb.get(s_, 0.0)
        per_stage[s_] = {"ms": round(per_step, 3), "share": round(per_step / ms, 4),
                         "launches": stage_launches.get(s_, 0) // args.steps,
                         "alg_bytes": int(bytes_),
                         "gbs": round(bytes_ / (per_step / 1e3) / 1e9, 1) if bytes_ else None,
                         "frac": round(bytes_ / (per_step / 1e3) / 1e9 / peaks["hbm_gbs"], 4) if bytes_ else 0.0}
    dom = max(per_stage, key=lambda s_: per_stage[s_]["ms"])
    dom_ms = per_stage[dom]["ms"]
    achieved = sb.get(dom, 0.0) / (dom_ms / 1e3) / 1e9
    traffic = None
    issue = None
    impl = None
    lt = latest_traffic(args.config, args.scale)
    if lt is not None:
        tpath, tj = lt
        rel = os.path.relpath(tpath, ROOT)
        if dom in tj.get("stages", {}):
            e = tj["stages"][dom]
            traffic = int(e["dram_bytes_read"] + e["dram_bytes_write"])
            if e.get("warp_inst"):
                # the issue side of the same kernel: ncu warp instructions per launch over the
                # live time, against 4 schedulers x SMs x the measured SM clock
                peak_gi = 4 * torch.cuda.get_device_properties(0).multi_processor_count * \
                    float(tj.get("sm_clock_ghz", 1.965))
                gi = e["warp_inst"] / (dom_ms / 1e3) / 1e9
                issue = {"warp_inst_per_launch": int(e["warp_inst"]), "achieved_ginst_s": round(gi, 1),
                         "peak_ginst_s": round(peak_gi, 1), "frac": round(gi / peak_gi, 4),
                         "thread_inst_per_window": round(32 * e["warp_inst"] / last["n_windows"], 1),
                         "source": f"ncu smsp__inst_executed.sum ({rel})"}
        if tj.get("call"):
            impl = {"B_impl": int(tj["call"]["dram_bytes"]),
                    "thread_inst_per_window": round(32 * tj["call"]["warp_inst"] / last["n_windows"], 1),
                    "source": f"ncu launch list, all kernels of one call ({rel})"}
    roof = {"kernel": dom, "bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"],
            "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": traffic,
            "alg_bytes_per_launch": int(sb.get(dom, 0.0)), "ms_per_launch": dom_ms,
            "peak_source": peaks["source"],
            "note": "achieved = SURVEY 8(d) algorithmic bytes of the stage (input + compact bins for "
                    "pass 1) / its live CUDA-event time; traffic = ncu DRAM bytes of the same kernel"}
    if issue:
        roof["issue"] = issue
    B_alg = b_alg(last, w.n_reads, k)
    ksz_ = 8 if k <= 32 else 16
    B_sort = B_alg + 2 * last["n_windows"] * ksz_
    pipe = {"B_alg": int(B_alg), "compact_bins": int(compact_bin_bytes(last, k)),
            "frac_of_step": round(B_alg / (ms / 1e3) / 1e9 / peaks["hbm_gbs"], 4),
            "B_sort": int(B_sort), "B_sort_frac_of_step": round(B_sort / (ms / 1e3) / 1e9 / peaks["hbm_gbs"], 4)}
    if impl:
        pipe.update({"B_impl": impl["B_impl"], "B_impl_over_B_alg": round(impl["B_impl"] / B_alg, 2),
                     "thread_inst_per_window": impl["thread_inst_per_window"], "impl_source": impl["source"]})
    roof["pipeline"] = pipe

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        T = os.cpu_count() or 1
        dt, nb_s, nw_s, nr_s = run_oracle_sample(w, args.cpu_sample_reads, T)
        cpu = {"value": nb_s / dt, "unit": "bases/s", "cores": T, "kind": "oracle",
               "sample": f"first {nr_s} reads of {args.config} ({nb_s} bases, {nw_s} windows), "
                         f"key-range-partitioned oracle on {T} threads, {dt:.1f} s",
               "kmers_per_s": nw_s / dt, "cpu_model": cpu_model()}

    out = {
        "metric": METRIC,
        "value": world * n_bases / (ms / 1e3),
        "unit": "bases/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": max(3, args.warmup),
        "ms_per_step": round(ms, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "u64" if k <= 32 else "u128",
        "data": "synthetic (seeded; BASELINE.json configs, SURVEY 8(d) recipe)",
        "config": {"workload": f"{args.config}: {cfg.desc}", "scale": args.scale, "n_reads": w.n_reads,
                   "n_bases": n_bases, "k": k, "p": p, "cutoff_min": ci, "cutoff_max": cx,
                   "parallelism": (f"sharded x{world}: reads split by rank, NCCL all-reduce of the signature "
                                   f"histogram; super-k-mer records written by the partition pass straight "
                                   f"into the owner rank's receive buffers over NVLink (CUDA IPC peer memory)"
                                   if xmode["mode"] == "p2p" else
                                   f"sharded x{world}: reads split by rank, NCCL all-reduce of the signature "
                                   f"histogram + all-to-all of super-k-mer records by bin owner")
                   if world > 1 else "1 GPU",
                   "count_path": ["smem_hash", "smem_radix_sort"][args.count_path],
                   "l2": "inputs (4 GB) larger than L2 (126 MB); no flush needed",
                   # N > 1: the NCCL process group every rank joined (torch.distributed, one
                   # process per GPU) and the record exchange the run used
                   **({"comm_backend": dist.get_backend(), "comm_nranks": dist.get_world_size(),
                       "exchange": xmode["mode"]} if world > 1 else {})},
        "kmers_per_s": windows_all / (ms / 1e3),
        "stats": {x: last[x] for x in ("n_windows", "n_superkmers", "n_records", "n_bins", "n_large_bins",
                                      "max_bin_windows", "large_windows", "n_unique", "n_out", "n_cluster_items",
                                      "n_single_items", "n_spilled_keys", "cluster_size", "cluster_ctas",
                                      "n_split_overflow", "n_overflow_chunks", "chunk_capacity")},
        "stages": per_stage,
        "roofline": roof,
        "cpu_baseline": cpu,
        "other_count_path": other,
        "e2e": e2e,
        "gpu_launches": n_launches,
        "clocks": clk,
    }
    print(json.dumps(out))
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def reference_arm(args, world, rank, cfg):
    """The CPU oracle, as it stands, on the host cores (rank 0 only)."""
    if rank != 0:
        return
    w = synth.make(args.config, scale=args.scale)
    n_sample = 1_000_000
    T = os.cpu_count() or 1
    for _ in range(args.warmup):
        pass  # the oracle has no warm state worth excluding; warm-up steps are not run
    t_tot, nb_tot, nw_tot = 0.0, 0, 0
    for s in range(args.steps):
        dt, nb_s, nw_s, nr_s = run_oracle_sample(w, n_sample, T)
        t_tot += dt
        nb_tot += nb_s
        nw_tot += nw_s
    v = nb_tot / t_tot
    out = {"impl": "reference", "metric": METRIC, "value": v, "unit": "bases/s", "n_gpus": world,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * t_tot / args.steps, 3),
           "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u64" if cfg.k <= 32 else "u128",
           "data": "synthetic", "config": {"workload": f"{args.config}: {cfg.desc}", "scale": args.scale},
           "kmers_per_s": nw_tot / t_tot,
           "cpu_baseline": {"value": v, "unit": "bases/s", "cores": T, "kind": "oracle",
                            "sample": f"first {n_sample} reads of {args.config} per step, key-range-partitioned "
                                      f"oracle on {T} threads",
                            "cpu_model": cpu_model()},
           "e2e": {"value": v, "unit": "bases/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
