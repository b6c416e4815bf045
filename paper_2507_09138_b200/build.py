"""Build libhivf.so (sm_100a) in-tree with nvcc.

    python -m paper_2507_09138_b200.build        # or __graft_entry__.build()

Every .cu under csrc/ is compiled for sm_100a only
(-gencode arch=compute_100a,code=sm_100a) with -lineinfo, then linked into
paper_2507_09138_b200/libhivf.so (static cudart, no torch dependency).
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(PKG, "csrc")
OUT = os.path.join(PKG, "libhivf.so")
BUILD = os.path.join(PKG, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
    "--expt-relaxed-constexpr", "-Xptxas", "-warn-spills",
    "-I" + os.path.join(os.path.dirname(PKG), "include"),
]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def _deps():
    return _sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + glob.glob(
        os.path.join(CSRC, "*.h")) + [os.path.join(os.path.dirname(PKG), "include", "hivf.h")]


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(f) <= t for f in _deps())


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(BUILD, os.path.basename(src)[:-3] + ".o")
    cmd = [NVCC, *NVCC_FLAGS, "-c", src, "-o", obj]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    if verbose and r.stderr:
        sys.stderr.write(r.stderr)
    return obj


HOST_SRC = os.path.join(PKG, "host", "hedra_gpu.cpp")
HOST_OUT = os.path.join(PKG, "libhedra_gpu.so")
ROOT = os.path.dirname(PKG)
CPP_TEST_SRC = os.path.join(ROOT, "tests", "cpp", "test_hedra_gpu.cpp")
CPP_TEST_OUT = os.path.join(ROOT, "tests", "cpp", "build", "test_hedra_gpu")


def _newer(out, deps):
    return os.path.exists(out) and all(os.path.getmtime(d) <= os.path.getmtime(out) for d in deps)


def build_host(force: bool = False) -> str:
    """The C++ drop-in adapter (host/hedra_gpu.*) over libhivf.so."""
    deps = [HOST_SRC, os.path.join(PKG, "host", "hedra_gpu.hpp"), OUT]
    if force or not _newer(HOST_OUT, deps):
        cmd = ["g++", "-std=c++20", "-O2", "-fPIC", "-shared", "-ffp-contract=off", "-Wall",
               "-I" + os.path.join(ROOT, "include"), HOST_SRC, "-L" + PKG, "-lhivf",
               "-Wl,-rpath,$ORIGIN", "-o", HOST_OUT]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"host adapter build failed:\n{r.stderr}")
    return HOST_OUT


def build_cpp_tests(force: bool = False) -> str:
    """C++ parity tests of the adapter (linked against the oracle restatement)."""
    oracle_dir = os.path.join(ROOT, "oracle")
    deps = [CPP_TEST_SRC, HOST_OUT, os.path.join(oracle_dir, "liboracle.so")]
    if force or not _newer(CPP_TEST_OUT, deps):
        os.makedirs(os.path.dirname(CPP_TEST_OUT), exist_ok=True)
        cmd = ["g++", "-std=c++20", "-O2", CPP_TEST_SRC, "-L" + PKG, "-lhedra_gpu", "-lhivf",
               "-L" + oracle_dir, "-loracle",
               "-Wl,-rpath," + PKG + ":" + oracle_dir + ":$ORIGIN/../../../paper_2507_09138_b200"
               ":$ORIGIN/../../../oracle", "-o", CPP_TEST_OUT]
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"C++ test build failed:\n{r.stderr}")
    return CPP_TEST_OUT


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        build_host()
        return OUT
    os.makedirs(BUILD, exist_ok=True)
    with cf.ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 4)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), _sources()))
    tmp = OUT + ".tmp"
    cmd = [NVCC, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
           "-o", tmp, *objs]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, OUT)
    build_host(force=True)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
