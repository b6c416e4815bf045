"""The C++ drop-in adapter (paper_2507_09138_b200/host/hedra_gpu.*) run through
its C++ parity suite (tests/cpp/test_hedra_gpu.cpp), which ports the reference's
doctest cases (test_vector_index.cpp, test_retrieval_engine.cpp,
test_tiered_cache.cpp) to the hedra_gpu namespace."""
import subprocess

import pytest


@pytest.fixture(scope="module")
def binary():
    import oracle
    from paper_2507_09138_b200 import build
    build.build()
    oracle.build()
    return build.build_cpp_tests()


def _run(binary, *args):
    r = subprocess.run([binary, *args], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failures" in r.stdout
    return r.stdout


def test_cpp_adapter_host_only(binary):
    out = _run(binary, "--cpu-only")
    assert "PASS cache_record_access_counts_once_per_substage" in out


@pytest.mark.gpu
def test_cpp_adapter_full_suite_on_gpu(binary):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    out = _run(binary)
    assert "FAIL" not in out
    assert "PASS engine_batch_equals_sequential_and_lane_transparency" in out
