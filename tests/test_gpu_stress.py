"""Randomised GPU parity sweep against the C restatement of the reference:
dims (incl. non-multiples of 16 / 64), list-size skew (empty lists, lists
shorter than a 128-row tile, multi-segment lists), k, nprobe up to K, L2 and
cosine, both tensor-core scan modes -- ids and distance bits must match."""
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_09138_b200 import Context
    return Context(0)


def _case(seed):
    rng = np.random.default_rng(seed)
    dim = int(rng.choice([3, 17, 48, 64, 100, 130, 256, 384, 768]))
    K = int(rng.choice([4, 16, 37, 64, 128]))
    n = int(rng.integers(max(K, 200), 30000))
    topics = int(rng.integers(2, 40))
    spread = float(rng.choice([0.02, 0.1, 0.4, 1.0]))
    centers = rng.standard_normal((topics, dim)).astype(np.float32)
    X = (centers[rng.integers(0, topics, n)] + spread * rng.standard_normal((n, dim))).astype(np.float32)
    metric = int(rng.integers(0, 2))
    if metric == 1:
        X = np.stack([oracle.normalized(r) for r in X])
    cents = X[rng.choice(n, K, replace=False)].copy()
    if rng.random() < 0.3:  # skew: a few huge lists, some empty
        cents[1:max(2, K // 4)] = cents[0] + 100.0
    assign = oracle.compute_assignments(X, cents)
    ids = rng.permutation(n).astype(np.uint64) * 7 + 3
    B = int(rng.integers(1, 200))
    Q = (centers[rng.integers(0, topics, B)] + spread * rng.standard_normal((B, dim))).astype(np.float32)
    nprobe = int(rng.integers(1, K + 1))
    k = int(rng.choice([1, 5, 10, 20, 32]))
    return X, ids, cents, assign, metric, Q, nprobe, k


@pytest.mark.parametrize("kernel", [0, 2])
@pytest.mark.parametrize("seed", list(range(int(os.environ.get("HIVF_STRESS_SEEDS", "12")))))
def test_random_configs(ctx, seed, kernel):
    from paper_2507_09138_b200 import IvfIndex
    X, ids, cents, assign, metric, Q, nprobe, k = _case(1000 + seed)
    ctx.set_option("scan_kernel", kernel)
    try:
        csr = oracle.CsrIndex.from_assignments(X, ids, cents, assign, metric)
        ix = IvfIndex.upload(ctx, csr.centroids, csr.off, csr.vectors, csr.ids, metric)
        gi, gd, gc = ix.search(Q, nprobe, k)
        oi, od, oc = csr.search(Q, nprobe, k)
        assert np.array_equal(gc, oc)
        assert np.array_equal(gi, oi)
        assert np.array_equal(gd.view(np.uint64), od.view(np.uint64))
        assert np.array_equal(ix.select_clusters(Q, nprobe), csr.assign(Q, nprobe)[0])
    finally:
        ctx.set_option("scan_kernel", 0)
