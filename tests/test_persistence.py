"""HVEC / u32 persistence of the C++ adapter (hedra_gpu::ivf::save_*/load_*)
against the reference's own writers and readers (vector_index.cpp:344-473,
through oracle/_ref): files byte-identical, reference files read back
exactly, and the reference's error cases (bad magic, truncation)."""
import ctypes as C
import os

import numpy as np
import pytest

import oracle

HG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                  "paper_2507_09138_b200", "libhedra_gpu.so")


@pytest.fixture(scope="module")
def hg():
    from paper_2507_09138_b200 import build
    build.build()
    L = C.CDLL(HG)
    vp, u32, u64 = C.c_void_p, C.c_uint32, C.c_uint64
    L.hg_save_corpus.argtypes = [C.c_char_p, vp, vp, u64, u32, C.c_int]
    L.hg_save_centroids.argtypes = [C.c_char_p, vp, u32, u32, C.c_int]
    L.hg_save_assignments.argtypes = [C.c_char_p, vp, u64]
    L.hg_load_corpus.argtypes = [C.c_char_p, C.POINTER(u32), C.POINTER(u64), C.POINTER(C.c_int), vp, vp]
    L.hg_load_centroids.argtypes = [C.c_char_p, C.POINTER(u32), C.POINTER(u64), vp]
    L.hg_load_assignments.argtypes = [C.c_char_p, C.POINTER(u64), vp]
    return L


needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def _load_corpus(fn, path):
    dim, n, m = C.c_uint32(), C.c_uint64(), C.c_int()
    assert fn(path, C.byref(dim), C.byref(n), C.byref(m), None, None) == 0
    X = np.zeros((n.value, dim.value), np.float32)
    ids = np.zeros(n.value, np.uint64)
    assert fn(path, C.byref(dim), C.byref(n), C.byref(m), X.ctypes.data, ids.ctypes.data) == 0
    return X, ids, m.value


@needs_ref
@pytest.mark.parametrize("metric", [0, 1])
def test_files_byte_identical_and_cross_readable(hg, tmp_path, metric):
    rng = np.random.default_rng(metric)
    X = rng.standard_normal((37, 11)).astype(np.float32)
    ids = (rng.permutation(37).astype(np.uint64) << np.uint64(33)) + np.uint64(5)
    cents = rng.standard_normal((6, 11)).astype(np.float32)
    asg = rng.integers(0, 6, 37).astype(np.uint32)
    R = oracle.ref()
    files = {}
    for who, sc, sce, sa in [("ours", hg.hg_save_corpus, hg.hg_save_centroids, hg.hg_save_assignments),
                             ("ref", R.ref_save_corpus, R.ref_save_centroids, R.ref_save_assignments)]:
        pc, pe, pa = (str(tmp_path / f"{who}.{x}").encode() for x in ("corpus", "cents", "assign"))
        if who == "ours":
            assert sc(pc, X.ctypes.data, ids.ctypes.data, 37, 11, metric) == 0
            assert sce(pe, cents.ctypes.data, 6, 11, metric) == 0
            assert sa(pa, asg.ctypes.data, 37) == 0
        else:
            assert sc(pc, X, ids, 37, 11, metric) == 0
            assert sce(pe, cents, 6, 11, metric) == 0
            assert sa(pa, asg, 37) == 0
        files[who] = (pc, pe, pa)
    for a, b in zip(files["ours"], files["ref"]):
        assert open(a, "rb").read() == open(b, "rb").read()
    # the reference's files through our loaders, and ours through the reference's
    Xo, io, mo = _load_corpus(hg.hg_load_corpus, files["ref"][0])
    assert np.array_equal(Xo, X) and np.array_equal(io, ids) and mo == metric
    Xr, ir, mr = _load_corpus(R.ref_load_corpus, files["ours"][0])
    assert np.array_equal(Xr, X) and np.array_equal(ir, ids) and mr == metric
    dim, k = C.c_uint32(), C.c_uint64()
    out = np.zeros((6, 11), np.float32)
    assert hg.hg_load_centroids(files["ref"][1], C.byref(dim), C.byref(k), out.ctypes.data) == 0
    assert np.array_equal(out, cents)
    n = C.c_uint64()
    a2 = np.zeros(37, np.uint32)
    assert hg.hg_load_assignments(files["ref"][2], C.byref(n), a2.ctypes.data) == 0
    assert n.value == 37 and np.array_equal(a2, asg)


def test_load_errors(hg, tmp_path):
    bad = tmp_path / "bad.hvec"
    bad.write_bytes(b"NOPE" + b"\\0" * 40)
    dim, n, m = C.c_uint32(), C.c_uint64(), C.c_int()
    assert hg.hg_load_corpus(str(bad).encode(), C.byref(dim), C.byref(n), C.byref(m), None, None) != 0
    X = np.ones((4, 3), np.float32)
    ids = np.arange(4, dtype=np.uint64)
    p = str(tmp_path / "c.hvec").encode()
    assert hg.hg_save_corpus(p, X.ctypes.data, ids.ctypes.data, 4, 3, 0) == 0
    raw = open(p, "rb").read()
    open(p, "wb").write(raw[:-5])  # truncated
    assert hg.hg_load_corpus(p, C.byref(dim), C.byref(n), C.byref(m), None, None) != 0
    assert hg.hg_load_corpus(str(tmp_path / "missing").encode(), C.byref(dim), C.byref(n), C.byref(m),
                             None, None) != 0
