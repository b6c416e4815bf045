"""Coarse assign on the tensor cores (k_coarse_dist_tc, scan_tc.cu): plans and
plan distances of ivf::select_clusters (vector_index.cpp:261-278) must be
bit-identical to the reference's whatever pass computes the filter distances
-- the kind::f16 GEMM over the fp16 centroid/query copies only decides which
centroids get the exact double.  Covers ragged shapes (K, B, dim not multiples
of the 128-row tiles / 64-dim stages), cosine, nprobe up to K, centroid norms
spread over many binades (small centroids underflow the shared fp16 scale:
the subnormal floor of coarse_bound_h16), out-of-range query scales (exact
streaming path) and the node-split / search paths built on the plans."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_ok():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _index(coarse_tc, X, cents, metric=0):
    from paper_2507_09138_b200 import Context, IvfIndex
    ctx = Context(0)
    ctx.set_option("coarse_tc", 2 if coarse_tc else 0)  # 2: every batch, whatever its size
    ids = np.arange(len(X), dtype=np.uint64) * 7 + 3
    assign = oracle.compute_assignments(X, cents)
    csr = oracle.CsrIndex.from_assignments(X, ids, cents, assign, metric)
    return ctx, IvfIndex.upload(ctx, csr.centroids, csr.off, csr.vectors, csr.ids, metric), csr


def _check_plans(ctx, ix, csr, Q, nprobe, bits=16):
    plans, dists = ix.select_clusters(Q, nprobe, with_dists=True)
    assert ctx.stats()["coarse_filter_bits"] == bits
    op, od = csr.assign(Q, nprobe)
    np.testing.assert_array_equal(plans, op)
    assert np.array_equal(dists.view(np.uint64), od.view(np.uint64))
    return plans


@pytest.mark.parametrize("dim,K,B,metric", [(8, 37, 1, 0), (96, 256, 130, 0), (128, 300, 129, 1),
                                            (200, 1000, 300, 0), (768, 512, 257, 0)])
def test_coarse_tc_plans_bit_exact(torch_ok, dim, K, B, metric):
    rng = np.random.default_rng(dim * 1000 + K)
    topics = rng.standard_normal((max(2, K // 4), dim)).astype(np.float32)
    X = (topics[rng.integers(0, len(topics), 6000)] +
         0.3 * rng.standard_normal((6000, dim))).astype(np.float32)
    if metric == 1:
        X = np.stack([oracle.normalized(r) for r in X])
    cents = X[rng.choice(len(X), K, replace=False)].copy()
    Q = (topics[rng.integers(0, len(topics), B)] + 0.3 * rng.standard_normal((B, dim))).astype(np.float32)
    ctx, ix, csr = _index(1, X, cents, metric)
    for nprobe in sorted({1, min(8, K), min(64, K), K}):
        _check_plans(ctx, ix, csr, Q, nprobe)
    ctx0, ix0, _ = _index(0, X, cents, metric)
    np.testing.assert_array_equal(ix0.select_clusters(Q, min(64, K)), ix.select_clusters(Q, min(64, K)))
    assert ctx0.stats()["coarse_filter_bits"] == 32


def test_coarse_tc_centroid_norms_over_many_binades(torch_ok):
    """One shared fp16 scale: centroids 2^-30 .. 2^10 times the largest norm's
    binade underflow to fp16 subnormals / zero; the bound's subnormal floor
    (relative to the largest norm) keeps the candidate set a superset."""
    rng = np.random.default_rng(77)
    dim, K = 64, 200
    X = rng.standard_normal((4000, dim)).astype(np.float32)
    cents = rng.standard_normal((K, dim)).astype(np.float32)
    cents *= (2.0 ** rng.integers(-30, 4, K)).astype(np.float32)[:, None]
    Q = np.concatenate([rng.standard_normal((40, dim)) * 1e-6, rng.standard_normal((40, dim)),
                        rng.standard_normal((40, dim)) * 1e3]).astype(np.float32)
    ctx, ix, csr = _index(1, X, cents)
    for nprobe in (1, 10, 100):
        _check_plans(ctx, ix, csr, Q, nprobe)


def test_coarse_tc_out_of_range_queries_take_the_exact_path(torch_ok):
    rng = np.random.default_rng(5)
    dim, K = 48, 96
    X = rng.standard_normal((3000, dim)).astype(np.float32)
    cents = X[rng.choice(3000, K, replace=False)].copy()
    Q = rng.standard_normal((30, dim)).astype(np.float32)
    Q[::4] *= np.float32(1e-17)  # |q| ~ 2^-53: the query's fp16 scale is out of range
    ctx, ix, csr = _index(1, X, cents)
    _check_plans(ctx, ix, csr, Q, 12)


def test_coarse_tc_search_equals_reference(torch_ok):
    rng = np.random.default_rng(11)
    dim, K = 128, 256
    topics = rng.standard_normal((64, dim)).astype(np.float32)
    X = (topics[rng.integers(0, 64, 20000)] + 0.2 * rng.standard_normal((20000, dim))).astype(np.float32)
    cents = X[rng.choice(len(X), K, replace=False)].copy()
    Q = (topics[rng.integers(0, 64, 300)] + 0.2 * rng.standard_normal((300, dim))).astype(np.float32)
    ctx, ix, csr = _index(1, X, cents)
    ids, d, cnt = ix.search(Q, 16, 10)
    assert ctx.stats()["coarse_filter_bits"] == 16
    oi, od, oc = csr.search(Q, 16, 10)
    np.testing.assert_array_equal(cnt, oc)
    np.testing.assert_array_equal(ids, oi)
    assert np.array_equal(d.view(np.uint64), od.view(np.uint64))


@pytest.mark.parametrize("coarse_tc", [1, 0])
def test_search_set_mode_duplicate_centroids(torch_ok, coarse_tc):
    """The search's coarse select in set mode (sure centroids skip the exact
    double): duplicated centroids put exact ties on the plan boundary (odd
    nprobe splits a pair), where membership is decided by the lower id; the
    lists differ, so a wrong member changes the results."""
    rng = np.random.default_rng(23)
    dim, K = 64, 64
    base = rng.standard_normal((K // 2, dim)).astype(np.float32)
    cents = np.concatenate([base, base])  # centroid i and i + 32 identical
    X = (base[rng.integers(0, K // 2, 8000)] + 0.4 * rng.standard_normal((8000, dim))).astype(np.float32)
    ids = np.arange(len(X), dtype=np.uint64) * 7 + 3
    assign = rng.integers(0, K, len(X)).astype(np.uint32)  # any assignment is an index
    csr = oracle.CsrIndex.from_assignments(X, ids, cents, assign)
    from paper_2507_09138_b200 import Context, IvfIndex
    ctx = Context(0)
    ctx.set_option("coarse_tc", 2 if coarse_tc else 0)
    ix = IvfIndex.upload(ctx, csr.centroids, csr.off, csr.vectors, csr.ids)
    Q = (base[rng.integers(0, K // 2, 200)] + 0.4 * rng.standard_normal((200, dim))).astype(np.float32)
    for nprobe, k in ((1, 10), (7, 10), (15, 5), (33, 20)):
        for set_mode in (1, 0):
            ctx.set_option("coarse_set", set_mode)
            gi, gd, gc = ix.search(Q, nprobe, k)
            oi, od, oc = csr.search(Q, nprobe, k)
            np.testing.assert_array_equal(gc, oc)
            np.testing.assert_array_equal(gi, oi)
            assert np.array_equal(gd.view(np.uint64), od.view(np.uint64))
    ctx.set_option("coarse_set", 1)


def test_coarse_tc_size_threshold(torch_ok):
    """Default (coarse_tc = 1): the tensor-core pass from 2^26 multiply-adds,
    the FFMA pass below; plans identical either way."""
    rng = np.random.default_rng(3)
    dim, K = 128, 1024
    X = rng.standard_normal((5000, dim)).astype(np.float32)
    cents = X[rng.choice(len(X), K, replace=False)].copy()
    from paper_2507_09138_b200 import Context, IvfIndex
    ctx = Context(0)
    ctx.set_option("coarse_tc", 1)
    ids = np.arange(len(X), dtype=np.uint64)
    csr = oracle.CsrIndex.from_assignments(X, ids, cents, oracle.compute_assignments(X, cents))
    ix = IvfIndex.upload(ctx, csr.centroids, csr.off, csr.vectors, csr.ids)
    for B, bits in ((16, 32), (600, 16)):  # 16 x 1024 x 128 = 2^21; 600 x 1024 x 128 > 2^26
        Q = rng.standard_normal((B, dim)).astype(np.float32)
        _check_plans(ctx, ix, csr, Q, 20, bits=bits)
