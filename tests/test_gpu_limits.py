"""The reference's full argument range (vector_index.cpp:264-265, :281): any
nprobe in [1, K] and large k.  Plans longer than the fast path's buffers
(nprobe > 4096) take the exact all-centroid select + stable radix sort
(assign.cu, k_coarse_all) and the exact scan; k up to 4096 runs on the exact
heap kernels.  Everything bit-exact against the C restatement."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def setup():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_09138_b200 import Context, IvfIndex
    rng = np.random.default_rng(5)
    n, dim, K = 30000, 24, 6000
    X = rng.standard_normal((n, dim)).astype(np.float32)
    cents = X[rng.choice(n, K, replace=False)].copy()
    cents[:8] = cents[8:16]  # duplicate centroids: equal distances, ties by id
    assign = oracle.compute_assignments(X, cents)
    ids = rng.permutation(n).astype(np.uint64) + 11
    csr = oracle.CsrIndex.from_assignments(X, ids, cents, assign)
    ctx = Context(0)
    ix = IvfIndex.upload(ctx, csr.centroids, csr.off, csr.vectors, csr.ids)
    Q = rng.standard_normal((6, dim)).astype(np.float32)
    Q[0] = cents[3]  # a query on a duplicated centroid
    return csr, ix, Q


@pytest.mark.parametrize("nprobe", [4097, 5000, 6000])
def test_select_clusters_beyond_4096(setup, nprobe):
    csr, ix, Q = setup
    plans, dists = ix.select_clusters(Q, nprobe, with_dists=True)
    op, od = csr.assign(Q, nprobe)
    assert np.array_equal(plans, op)
    assert np.array_equal(dists.view(np.uint64), od.view(np.uint64))


@pytest.mark.parametrize("nprobe,k", [(4097, 10), (6000, 10), (5000, 40)])
def test_search_beyond_4096(setup, nprobe, k):
    csr, ix, Q = setup
    gi, gd, gc = ix.search(Q, nprobe, k)
    oi, od, oc = csr.search(Q, nprobe, k)
    assert np.array_equal(gc, oc)
    assert np.array_equal(gi, oi)
    assert np.array_equal(gd.view(np.uint64), od.view(np.uint64))


@pytest.mark.parametrize("k", [1025, 2500, 4096])
def test_large_k(setup, k):
    csr, ix, Q = setup
    gi, gd, gc = ix.search(Q, 600, k)
    oi, od, oc = csr.search(Q, 600, k)
    assert np.array_equal(gc, oc)
    assert np.array_equal(gi, oi)
    assert np.array_equal(gd.view(np.uint64), od.view(np.uint64))


def test_scan_items_long_items_and_large_k(setup):
    """node-split items with > 4096 clusters and heaps of k = 2000 (seeded)"""
    csr, ix, Q = setup
    nprobe = 5000
    plans = csr.assign(Q[:3], nprobe)[0]
    k = [2000, 10, 4096]
    stride = max(k)
    hid = np.zeros((3, stride), np.uint64)
    hd = np.zeros((3, stride), np.float64)
    hn = np.zeros(3, np.uint32)
    heaps = [oracle.TopK(kk) for kk in k]
    # seed item 1's heap with the reference's merge of a few exact distances
    for doc in range(5):
        row = csr.vectors[doc]
        heaps[1].insert(int(csr.ids[doc]), oracle.squared_l2(Q[1], row))
    for i, h in enumerate(heaps):
        e = h.entries()
        hn[i] = len(e)
        for j, (doc, d) in enumerate(e):
            hid[i, j], hd[i, j] = doc, d
    cuts = [(0, 4500), (0, 300), (0, 5000)]
    off = np.zeros(4, np.uint32)
    cl = []
    for i, (a, b) in enumerate(cuts):
        cl += list(plans[i][a:b])
        off[i + 1] = len(cl)
    changed = ix.scan_items(Q[:3], off, np.array(cl, np.uint32), np.array(k, np.uint32), hid, hd, hn)
    for i, (a, b) in enumerate(cuts):
        _, ch = oracle.search_clusters(csr, Q[i], plans[i], a, heaps[i], plans[i][a:b])
        e = heaps[i].entries()
        assert hn[i] == len(e), i
        assert [int(x) for x in hid[i, : hn[i]]] == [doc for doc, _ in e], i
        assert np.array_equal(hd[i, : hn[i]], np.array([d for _, d in e], np.float64)), i
        assert np.array_equal(changed[off[i]:off[i + 1]], ch), i


def test_k_beyond_4096_is_reported(setup):
    from paper_2507_09138_b200._lib import HivfError
    csr, ix, Q = setup
    with pytest.raises(HivfError):
        ix.search(Q, 16, 4097)
