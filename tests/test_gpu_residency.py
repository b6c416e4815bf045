"""Tiered residency (hbm_list_budget + hivf_residency_set): lists in a pinned
host backing store, the resident set copied into an HBM pool asynchronously.
Results must be bit-identical whatever is resident or in flight (lane
transparency, proj/tests/test_retrieval_engine.cpp:158-199), evictions are
immediate and a list becomes resident only once its copy completed
(tiered_cache.cpp:23-36,70-80)."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _setup(budget_frac, seed=3, n=30000, dim=96, K=64, options=()):
    import torch
    from paper_2507_09138_b200 import Context, IvfIndex
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((24, dim)).astype(np.float32)
    X = (centers[np.arange(n) % 24] + 0.3 * rng.standard_normal((n, dim))).astype(np.float32)
    cents = X[rng.choice(n, K, replace=False)].copy()
    assign = oracle.compute_assignments(X, cents)
    ids = rng.permutation(n).astype(np.uint64) * 5 + 1
    csr = oracle.CsrIndex.from_assignments(X, ids, cents, assign)
    ctx = Context(0, torch.cuda.current_stream())
    total = int(csr.vectors.shape[0]) * ((dim + 15) // 16 * 16) * 4
    ctx.set_option("hbm_list_budget", max(1, int(total * budget_frac)))
    for name, value in options:
        ctx.set_option(name, value)
    ix = IvfIndex.upload(ctx, csr.centroids, csr.off, csr.vectors, csr.ids)
    Q = (centers[rng.integers(0, 24, 40)] + 0.3 * rng.standard_normal((40, dim))).astype(np.float32)
    return ctx, ix, csr, Q


def _same(ix, csr, Q, nprobe=10, k=10):
    gi, gd, gc = ix.search(Q, nprobe, k)
    oi, od, oc = csr.search(Q, nprobe, k)
    assert np.array_equal(gc, oc)
    assert np.array_equal(gi, oi)
    assert np.array_equal(gd.view(np.uint64), od.view(np.uint64))


def test_tiered_search_from_host_backing_store():
    ctx, ix, csr, Q = _setup(0.25)
    assert not ix.residency().any()
    _same(ix, csr, Q)


def test_residency_swaps_and_evictions():
    ctx, ix, csr, Q = _setup(0.3)
    plans = ix.select_clusters(Q, 10)
    hot = np.argsort(-np.bincount(plans.ravel(), minlength=64), kind="stable")[:40].astype(np.uint32)
    ix.set_residency(hot)
    _same(ix, csr, Q)            # copies possibly in flight: results unchanged
    ix.residency_sync()
    res = ix.residency()
    sizes = np.diff(csr.off.astype(np.int64))
    assert res[hot].any() and not res[np.setdiff1d(np.arange(64), hot)].any()
    # admitted in the caller's order while they fit the budget
    budget = int(sizes.sum() * ((96 + 15) // 16 * 16) * 4 * 0.3)
    used = sum(((int(sizes[c]) * 96 * 4 + 255) // 256) * 256 for c in np.nonzero(res)[0])
    assert used <= budget
    _same(ix, csr, Q)
    _same(ix, csr, Q, nprobe=64, k=20)
    ix.set_residency(hot[:5])    # evictions are immediate
    r2 = ix.residency()
    assert not r2[hot[5:]].any()
    _same(ix, csr, Q)
    ix.set_residency([])
    assert not ix.residency().any()
    _same(ix, csr, Q)


def test_tiered_node_split_sub_search():
    """hivf_scan_items over a half-resident index == the reference engine trace."""
    ctx, ix, csr, Q = _setup(0.5, seed=9)
    plans = ix.select_clusters(Q, 12)
    ix.set_residency(np.unique(plans[:, :3]).astype(np.uint32))
    ix.residency_sync()
    B, k = len(Q), 20
    hi = np.zeros((B, k), np.uint64)
    hd = np.zeros((B, k), np.float64)
    hn = np.zeros(B, np.uint32)
    th = oracle.TopK(k) if hasattr(oracle, "TopK") else None
    for step in range(4):  # 3 clusters per sub-stage
        off = np.arange(B + 1, dtype=np.uint32) * 3
        cl = plans[:, step * 3:(step + 1) * 3].reshape(-1).astype(np.uint32)
        ix.scan_items(Q, off, cl, np.full(B, k, np.uint32), hi, hd, hn)
    oi, od, oc = csr.search(Q, 12, k)
    assert np.array_equal(hn, oc)
    for b in range(B):
        assert np.array_equal(hi[b, :hn[b]], oi[b, :oc[b]])
        assert np.array_equal(hd[b, :hn[b]].view(np.uint64), od[b, :oc[b]].view(np.uint64))


@pytest.mark.parametrize("h16", [1, 0])
def test_tiered_two_lanes_fp16_filter_in_hbm(h16):
    """Tiered index with the fp16 filter copy: the copy of EVERY
    list stays in HBM, so the tensor-core scan never reads the host backing
    store; only the exact re-rank of candidates (and repair / fallback) reads
    cold lists' fp32 rows over PCIe.  Without the copy the scan streams the
    cold fp32 lists from host memory.  Both give the reference's bits, with
    nothing, part or all of the exact rows resident."""
    ctx, ix, csr, Q = _setup(0.3, seed=5, options=(("filter_h16", h16), ("scan_kernel", 3)))
    _same(ix, csr, Q)
    st = ctx.stats()
    assert st["scan_kernel"] == 3 and st["scan_filter_bits"] == (16 if h16 else 32), st
    plans = ix.select_clusters(Q, 10)
    hot = np.argsort(-np.bincount(plans.ravel(), minlength=64), kind="stable").astype(np.uint32)
    ix.set_residency(hot)
    ix.residency_sync()
    assert ix.residency().any()
    _same(ix, csr, Q)
    _same(ix, csr, Q, nprobe=64, k=20)
    assert ctx.stats()["scan_filter_bits"] == (16 if h16 else 32)
