"""Build the reference's own callers against the GPU engine (and, beside
them, against the reference's CPU hot path, as the oracle build).

    python -m paper_2507_09138_b200.compat.build    # or __graft_entry__.build()

Two flavours, each linking the UNMODIFIED reference sources that sit around
the hot path (compiled in place from /root/reference/proj, nothing copied into
the repo):

  gpu  compat/include (GPU-backed hedra/vector_index.hpp) first on the include
       path, compat/hedra_ivf_gpu.cpp for the hot-path translation units
       (vector_index.cpp, retrieval_engine.cpp), libhivf.so for the kernels.
  cpu  the reference's own vector_index.cpp / retrieval_engine.cpp -- the
       CPU reference the GPU flavour must agree with.

Around the hot path both flavours compile the reference's scheduler.cpp,
similarity.cpp, tiered_cache.cpp, raggraph.cpp, generation_engine.cpp,
workload.cpp, report.cpp and bench.cpp, and link:

  test_<suite>   the reference unit suites proj/tests/test_*.cpp with the
                 doctest stand-in (tests/cpp/doctest_shim/doctest.h)
  acceptance     proj/tests/acceptance_test.cpp with the one-line fix of its
                 :82 dangling-temporary UB, applied to a
                 build-directory copy
  hedra_c5       compat/hedra_c5.cpp: config 5 through sched::run

Outputs go to compat/_build/{gpu,cpu}/ (git-ignored; they travel to the GPU
box with the snapshot, where /root/reference does not exist).  Reference
flags: -std=c++20 -O2 (proj/CMakeLists.txt), no -march, no fast-math.
"""
from __future__ import annotations

import concurrent.futures as cf
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.dirname(HERE)
ROOT = os.path.dirname(PKG)
REF = os.environ.get("HEDRA_REF", "/root/reference/proj")
OUT = os.path.join(HERE, "_build")
JSON_DIR = None
for cand in (
    "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty/nlohmann",
):
    if os.path.exists(os.path.join(cand, "json.hpp")):
        JSON_DIR = cand

AROUND = ["scheduler", "similarity", "tiered_cache", "raggraph", "generation_engine",
          "workload", "report", "bench"]
HOT = ["vector_index", "retrieval_engine"]
SUITES = ["vector_index", "retrieval_engine", "similarity", "tiered_cache", "scheduler",
          "harness", "raggraph", "generation_engine"]
FLAGS = ["-std=c++20", "-O2", "-Wall", "-Wextra", "-Wno-unused-parameter"]
# acceptance_test.cpp:82 builds a set from begin()/end() of two different
# temporaries (UB; hangs the reference's own build).  The fix keeps the ids.
ACCEPT_FIX = (
    "std::set<DocId> truth_ids(truth.doc_ids().begin(), truth.doc_ids().end());",
    "const auto truth_vec = truth.doc_ids();\n"
    "      std::set<DocId> truth_ids(truth_vec.begin(), truth_vec.end());",
)


def available() -> bool:
    return os.path.isdir(os.path.join(REF, "src")) and JSON_DIR is not None


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("compat build failed:\n" + " ".join(cmd) + "\n" + r.stderr[-4000:])


def _newer(out, deps):
    return os.path.exists(out) and all(os.path.getmtime(d) <= os.path.getmtime(out) for d in deps)


def _includes(flavour):
    inc = []
    if flavour == "gpu":
        inc.append("-I" + os.path.join(HERE, "include"))
    inc += ["-I" + os.path.join(REF, "include"), "-I" + JSON_DIR,
            "-I" + os.path.join(ROOT, "tests", "cpp", "doctest_shim")]
    return inc


def _headers(flavour):
    hs = [os.path.join(REF, "include", "hedra", f) for f in os.listdir(os.path.join(REF, "include", "hedra"))]
    if flavour == "gpu":
        d = os.path.join(HERE, "include", "hedra")
        hs += [os.path.join(d, f) for f in os.listdir(d)]
        hs += [os.path.join(ROOT, "include", "hivf.h"), os.path.join(PKG, "host", "hvec_io.hpp")]
    return hs


def _objects(flavour, ex):
    d = os.path.join(OUT, flavour, "obj")
    os.makedirs(d, exist_ok=True)
    srcs = [os.path.join(REF, "src", s + ".cpp") for s in AROUND]
    if flavour == "gpu":
        srcs.append(os.path.join(HERE, "hedra_ivf_gpu.cpp"))
    else:
        srcs += [os.path.join(REF, "src", s + ".cpp") for s in HOT]
    defs = ["-DHEDRA_GPU_COMPAT"] if flavour == "gpu" else []
    hdrs = _headers(flavour)
    jobs = []
    for s in srcs:
        o = os.path.join(d, os.path.basename(s)[:-4] + ".o")
        if not _newer(o, [s] + hdrs):
            jobs.append(ex.submit(_run, ["g++", *FLAGS, "-fPIC", *defs, *_includes(flavour), "-c", s, "-o", o]))
    for j in jobs:
        j.result()
    return [os.path.join(d, os.path.basename(s)[:-4] + ".o") for s in srcs]


def _acceptance_src():
    src = os.path.join(REF, "tests", "acceptance_test.cpp")
    dst = os.path.join(OUT, "src", "acceptance_test.cpp")
    os.makedirs(os.path.dirname(dst), exist_ok=True)
    text = open(src).read()
    if ACCEPT_FIX[0] not in text:
        raise RuntimeError("acceptance_test.cpp: the :82 line to fix was not found")
    fixed = text.replace(ACCEPT_FIX[0], ACCEPT_FIX[1])
    if not os.path.exists(dst) or open(dst).read() != fixed:
        with open(dst, "w") as f:
            f.write(fixed)
    return dst


def _link(flavour, objs, main_src, name, ex):
    exe = os.path.join(OUT, flavour, name)
    defs = ["-DHEDRA_GPU_COMPAT"] if flavour == "gpu" else []
    libs = ["-lpthread"]
    if flavour == "gpu":
        libs = ["-L" + PKG, "-lhivf", "-Wl,-rpath,$ORIGIN/../../..", "-lpthread"]
        deps = objs + [main_src, os.path.join(PKG, "libhivf.so")] + _headers(flavour)
    else:
        deps = objs + [main_src] + _headers(flavour)
    if _newer(exe, deps):
        return None
    return ex.submit(_run, ["g++", *FLAGS, *defs, *_includes(flavour), main_src, *objs, *libs, "-o", exe])


def build(force: bool = False) -> str:
    if not available():
        print("compat: reference sources or json.hpp absent, using prebuilt _build if present")
        return OUT
    if force:
        import shutil
        shutil.rmtree(OUT, ignore_errors=True)
    accept = _acceptance_src()
    with cf.ThreadPoolExecutor(max_workers=min(16, os.cpu_count() or 4)) as ex:
        for flavour in ("gpu", "cpu"):
            objs = _objects(flavour, ex)
            jobs = [_link(flavour, objs, os.path.join(REF, "tests", f"test_{s}.cpp"), f"test_{s}", ex)
                    for s in SUITES]
            jobs.append(_link(flavour, objs, accept, "acceptance", ex))
            jobs.append(_link(flavour, objs, os.path.join(HERE, "hedra_c5.cpp"), "hedra_c5", ex))
            for j in jobs:
                if j is not None:
                    j.result()
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv))
