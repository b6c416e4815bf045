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


@pytest.mark.parametrize("seed", list(range(int(os.environ.get("HIVF_STRESS_SEEDS", "12")) // 2 + 2)))
def test_random_node_split(ctx, seed):
    """hivf_scan_items over random sub-stage slices with seeded heaps (a full
    seeded heap turns on the per-item drop bound from the first sub-stage) vs
    search_clusters of the C restatement: heaps and per-cluster changed flags."""
    from paper_2507_09138_b200 import IvfIndex
    X, ids, cents, assign, metric, Q, nprobe, k = _case(5000 + seed)
    rng = np.random.default_rng(seed)
    csr = oracle.CsrIndex.from_assignments(X, ids, cents, assign, metric)
    ix = IvfIndex.upload(ctx, csr.centroids, csr.off, csr.vectors, csr.ids, metric)
    Q = Q[:24]
    B = len(Q)
    plans = ix.select_clusters(Q, nprobe)
    qs = np.stack([oracle.normalized(q) if metric == 1 else q for q in Q]).astype(np.float32)
    kv = rng.integers(1, 33, B).astype(np.uint32)
    stride = 32
    hi = np.zeros((B, stride), np.uint64)
    hd = np.zeros((B, stride), np.float64)
    hn = np.zeros(B, np.uint32)
    heaps = [oracle.TopK(int(kv[b])) for b in range(B)]
    # seeds: exact distances to random docs (probe_cache-style), half the cursors
    for b in range(B):
        if rng.random() < 0.5:
            for r in rng.choice(len(X), size=int(kv[b]) + 3, replace=False):
                heaps[b].insert(int(ids[r]), oracle.squared_l2(qs[b], X[r]))
            ent = heaps[b].entries()
            hn[b] = len(ent)
            for j, (i, d) in enumerate(ent):
                hi[b, j], hd[b, j] = i, d
    pos = np.zeros(B, np.int64)
    while (pos < nprobe).any():
        take = [int(min(nprobe - pos[b], rng.integers(1, 6))) if pos[b] < nprobe else 0 for b in range(B)]
        items = [b for b in range(B) if take[b] > 0]
        off = np.zeros(len(items) + 1, np.uint32)
        cl = []
        for i, b in enumerate(items):
            cl.append(plans[b, pos[b]:pos[b] + take[b]])
            off[i + 1] = off[i] + take[b]
        cl = np.concatenate(cl).astype(np.uint32)
        sub_hi, sub_hd, sub_hn = hi[items].copy(), hd[items].copy(), hn[items].copy()
        changed = ix.scan_items(qs[items], off, cl, kv[items], sub_hi, sub_hd, sub_hn)
        for i, b in enumerate(items):
            npos, ch = oracle.search_clusters(csr, qs[b], plans[b], int(pos[b]), heaps[b],
                                              cl[off[i]:off[i + 1]])
            assert list(changed[off[i]:off[i + 1]]) == list(ch)
            ent = heaps[b].entries()
            assert int(sub_hn[i]) == len(ent)
            assert [int(x) for x in sub_hi[i, :len(ent)]] == [e[0] for e in ent]
            assert np.array_equal(sub_hd[i, :len(ent)].view(np.uint64),
                                  np.array([e[1] for e in ent], np.float64).view(np.uint64))
            pos[b] = npos
        hi[items], hd[items], hn[items] = sub_hi, sub_hd, sub_hn
