"""CPU tests of the C-ABI library: it is built for sm_100a, loads, and exports
every symbol include/hivf.h declares (no compute calls without a GPU)."""
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "hivf.h")


def header_symbols():
    src = open(HEADER).read()
    return sorted(set(re.findall(r"\b(hivf_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def libpath():
    from paper_2507_09138_b200 import build
    return build.build()


def test_header_and_binding_agree():
    from paper_2507_09138_b200 import SYMBOLS
    assert sorted(SYMBOLS) == header_symbols()


def test_library_exports_every_header_symbol(libpath):
    out = subprocess.run(["nm", "-D", "--defined-only", libpath], capture_output=True, text=True,
                         check=True).stdout
    exported = set(re.findall(r"\bT (hivf_[a-z0-9_]+)\b", out))
    missing = [s for s in header_symbols() if s not in exported]
    assert not missing, missing


def test_library_loads_and_reports_version(libpath):
    from paper_2507_09138_b200 import lib
    L = lib()
    assert L.hivf_version().startswith(b"hivf")
    assert L.hivf_last_error() is not None


def test_sm100a_cubin_only(libpath):
    out = subprocess.run(["cuobjdump", "--list-elf", libpath], capture_output=True, text=True).stdout
    archs = set(re.findall(r"sm_(\d+a?)", out))
    assert archs == {"100a"}, archs


def test_scan_kernel_uses_bulk_async_copies(libpath):
    """The list scan streams lists with cp.async.bulk (UBLKCP) + mbarriers."""
    out = subprocess.run(["cuobjdump", "-sass", libpath], capture_output=True, text=True).stdout
    funcs = out.split("Function : ")
    scan = [f for f in funcs if f.split("\n", 1)[0].endswith("k_scanENS0_10ScanParamsE")]
    assert scan, "k_scan not found in SASS"
    assert "UBLKCP" in scan[0]
    assert "SYNCS" in scan[0]


def test_no_gpu_calls_fail_cleanly_without_device():
    """Creating a context without a GPU must fail with a status, not crash."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2507_09138_b200 import Context, HivfError
    with pytest.raises(HivfError):
        Context(0)
