"""CPU-side checks of the boundary (-m "not gpu"): the C-ABI library builds for sm_100a,
loads, exports every symbol include/kmcgpu.h declares, and the product path shares no code
with the oracle.  No compute calls are made without a GPU."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = open(os.path.join(ROOT, "include", "kmcgpu.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*(kmc_[a-z_]+)\s*\(", txt, flags=re.M)
    return sorted(set(names))


@pytest.fixture(scope="module")
def lib_path():
    from paper_1407_1507_b200 import build
    return build.build()


def test_header_declares_expected_api():
    names = header_functions()
    for n in ("kmc_count", "kmc_count_ex", "kmc_count_begin", "kmc_count_finish", "kmc_job_free",
              "kmc_debug_signatures", "kmc_debug_allowed", "kmc_last_error", "kmc_set_allocator", "kmc_version"):
        assert n in names


def test_library_loads_and_exports_every_symbol(lib_path):
    lib = ctypes.CDLL(lib_path)
    for n in header_functions():
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True).stdout
    exported = set(re.findall(r" T (kmc_[a-z_]+)", out))
    assert set(header_functions()) <= exported
    lib.kmc_version.restype = ctypes.c_int
    assert lib.kmc_version() >= 100


def test_library_is_sm100a_native(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_invalid_args_rejected_before_device_work(lib_path):
    lib = ctypes.CDLL(lib_path)
    lib.kmc_count.restype = ctypes.c_int
    lib.kmc_last_error.restype = ctypes.c_char_p
    # k out of range -> KMC_ERR_INVALID_ARG (1) without touching the device
    st = lib.kmc_count(None, None, ctypes.c_uint64(0), 0, 7, 1, 10, None, None, ctypes.c_uint64(0), None, None)
    assert st == 1 and b"k=" in lib.kmc_last_error()
    st = lib.kmc_count(None, None, ctypes.c_uint64(0), 25, 16, 1, 10, None, None, ctypes.c_uint64(0), None, None)
    assert st == 1
    st = lib.kmc_count(None, None, ctypes.c_uint64(0), 25, 7, 5, 4, None, None, ctypes.c_uint64(0), None, None)
    assert st == 1


def _imports(path):
    src = open(path).read()
    return set(re.findall(r"^\s*(?:from|import)\s+([A-Za-z_][A-Za-z0-9_.]*)", src, flags=re.M))


def test_product_and_oracle_share_nothing():
    pkg = os.path.join(ROOT, "paper_1407_1507_b200")
    orc = os.path.join(ROOT, "oracle")
    for d, forbidden in ((pkg, "oracle"), (orc, "paper_1407_1507_b200")):
        for dirpath, _, files in os.walk(d):
            for f in files:
                p = os.path.join(dirpath, f)
                if f.endswith(".py"):
                    assert not any(m.split(".")[0] == forbidden for m in _imports(p)), p
                if f.endswith((".cu", ".cuh", ".h", ".cpp", ".c")):
                    incs = re.findall(r'^\s*#\s*include\s*[<"]([^>"]+)[>"]', open(p).read(), flags=re.M)
                    assert not any(forbidden in i or "oracle" in i or "kmc_device" in i and d == orc for i in incs), p
    # the oracle never includes the product headers and vice versa
    assert "kmcgpu.h" not in open(os.path.join(orc, "kmc_oracle.cpp")).read()


def test_synth_holds_no_method_arithmetic():
    src = open(os.path.join(ROOT, "synth", "gen.c")).read() + open(os.path.join(ROOT, "synth", "__init__.py")).read()
    for word in ("canonical", "signature", "minimizer"):
        # only allowed inside the module docstring disclaimers
        assert src.count(word) <= 2, word
