"""Build libkmcgpu.so in-tree for sm_100a (nvcc, -lineinfo, parallel per-file compile).

Usage: python -m paper_1407_1507_b200.build [--force] [--verbose]
The ptxas resource report (registers, shared memory, spills) of every kernel is
written to build/ptxas_<file>.log.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
BUILD = os.path.join(ROOT, "build")
SO = os.path.join(PKG, "libkmcgpu.so")
SOURCES = ["k_distribute.cu", "k_plan.cu", "k_sort.cu", "k_cluster.cu", "k_split1.cu", "k_subsplit.cu", "k_kxmer.cu", "k_order.cu", "k_db.cu", "kmc_api.cu"]
HEADERS = ["kmc_device.cuh", "kmc_internal.h", "kmc_scan.cuh"]
NVCC = os.environ.get("NVCC", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xptxas", "-v",
         "-I" + os.path.join(ROOT, "include")] + os.environ.get("KMC_NVCC_EXTRA", "").split()  # (experiments)


def _newest_input() -> float:
    files = [os.path.join(CSRC, f) for f in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "kmcgpu.h"),
                                                                   os.path.abspath(__file__)]
    return max(os.path.getmtime(f) for f in files)


def _compile(src: str) -> str:
    obj = os.path.join(BUILD, src.replace(".cu", ".o"))
    log = os.path.join(BUILD, "ptxas_" + src.replace(".cu", ".log"))
    cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    with open(log, "w") as f:
        f.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stderr[-6000:]}")
    return obj


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(SO) and os.path.getmtime(SO) >= _newest_input():
        return SO
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    tmp = SO + f".tmp{os.getpid()}"
    cmd = [NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lcudart_static"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stderr[-4000:]}")
    os.replace(tmp, SO)
    if verbose:
        for s in SOURCES:
            print(open(os.path.join(BUILD, "ptxas_" + s.replace(".cu", ".log"))).read())
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv))
