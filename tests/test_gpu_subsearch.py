"""GPU parity of the node-split sub-search (hivf_scan_items) and the shard merge.

Reference: search_clusters (vector_index.cpp:291-317) as RetrievalEngine::execute
runs it (retrieval_engine.cpp:55-152): heaps carried across sub-stages, clusters
in plan order, per-cluster `changed` flags feeding heap_changed and
unchanged_streak.  Oracles: the reference engine's own traces
(tests/golden/*.npz, sub_*) and the C restatement.
"""
import glob
import os

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


@pytest.fixture(scope="module")
def ctx():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_09138_b200 import Context
    return Context(0)


def _golden_index(ctx, g):
    from paper_2507_09138_b200 import IvfIndex
    rows = ((g["list_ids"] - 3) // 7).astype(np.int64)
    vec = g["corpus"][rows]
    if int(g["metric"]) == 1:
        vec = np.stack([oracle.normalized(r) for r in vec])
    return IvfIndex.upload(ctx, g["centroids"], g["list_off"], vec, g["list_ids"], int(g["metric"]))


@pytest.mark.parametrize("kernel", [0, 1, 2])
@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_golden_engine_trace(ctx, path, kernel):
    """Replays the reference engine's uneven sub-stage schedule through
    hivf_scan_items: per-item heap_changed per step, final heaps and
    unchanged_streak must equal the reference's."""
    g = np.load(path)
    ix = _golden_index(ctx, g)
    Q = g["queries"]
    metric = int(g["metric"])
    npb, k = int(g["sub_np"]), int(g["sub_k"])
    plans = ix.select_clusters(Q, npb)
    qs = np.stack([oracle.normalized(q) if metric == 1 else q for q in Q]).astype(np.float32)
    B = len(Q)
    heap_ids = np.zeros((B, k), np.uint64)
    heap_d = np.zeros((B, k), np.float64)
    heap_n = np.zeros(B, np.uint32)
    streak = np.zeros(B, np.int64)
    slices = g["sub_slices"]
    steps = np.unique(slices[:, 0])
    got_changed = []
    ctx.set_option("scan_kernel", kernel)
    try:
        for st in steps:
            rows = slices[slices[:, 0] == st]
            items = rows[:, 1]
            off = [0]
            cl = []
            for _, b, p0, take in rows:
                cl.extend(plans[b][p0:p0 + take].tolist())
                off.append(len(cl))
            hi, hd, hn = heap_ids[items].copy(), heap_d[items].copy(), heap_n[items].copy()
            changed = ix.scan_items(qs[items], off, cl, np.full(len(items), k, np.uint32), hi, hd, hn)
            heap_ids[items], heap_d[items], heap_n[items] = hi, hd, hn
            for j, b in enumerate(items):
                flags = changed[off[j]:off[j + 1]]
                got_changed.append(bool(flags.any()))
                for f in flags:
                    streak[b] = 0 if f else streak[b] + 1
    finally:
        ctx.set_option("scan_kernel", 0)
    np.testing.assert_array_equal(np.array(got_changed), g["sub_changed"][1].astype(bool))
    for b in range(B):
        n = int(heap_n[b])
        np.testing.assert_array_equal(heap_ids[b, :n], g["sub_final_ids"][b, :n])
        assert np.array_equal(heap_d[b, :n].view(np.uint64), g["sub_final_dist"][b, :n].view(np.uint64))
    np.testing.assert_array_equal(streak, g["sub_final_streak"].astype(np.int64))


def _rand_index(ctx, seed, n=6000, dim=32, K=24):
    from paper_2507_09138_b200 import IvfIndex
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((8, dim)).astype(np.float32)
    X = (centers[np.arange(n) % 8] + 0.4 * rng.standard_normal((n, dim))).astype(np.float32)
    cents = X[rng.choice(n, K, replace=False)].copy()
    assign = oracle.compute_assignments(X, cents)
    ids = rng.permutation(n).astype(np.uint64) + 100
    csr = oracle.CsrIndex.from_assignments(X, ids, cents, assign)
    ix = IvfIndex.upload(ctx, csr.centroids, csr.off, csr.vectors, csr.ids)
    return ix, csr, X, centers, rng


@pytest.mark.parametrize("kernel", [0, 1, 2, "wide"])
def test_seeded_reordered_subsearch_vs_oracle(ctx, kernel):
    """Seeded heaps (probe_cache, similarity.cpp:35-55) and reordered plans
    (reorder_clusters, :57-72), mixed k and slice sizes, vs the restatement.
    "wide": the single-pass tensor-core scan forced onto its 64-query variant
    (fixed per-item bounds, bound_update = 0)."""
    wide = kernel == "wide"
    if wide:
        kernel = 3
        ctx.set_option("tc_wide_ppl", 0)
    ix, csr, X, centers, rng = _rand_index(ctx, 41)
    B = 40
    Q = (centers[rng.integers(0, 8, B)] + 0.4 * rng.standard_normal((B, 32))).astype(np.float32)
    nprobe = 12
    plans = ix.select_clusters(Q, nprobe)
    ks = rng.integers(1, 33, B).astype(np.uint32)
    heaps, oheaps = [], []
    for b in range(B):
        p = plans[b].copy()
        tail = p[3:]
        rng.shuffle(tail)  # an arbitrary reorder of the unsearched suffix
        p[3:] = tail
        plans[b] = p
        t = oracle.TopK(int(ks[b]))
        # seeds: exact distances of docs from lists in the plan (result-neutral)
        for r in rng.choice(len(csr.ids), 5, replace=False):
            c = int(np.searchsorted(csr.off, r, side="right") - 1)
            if c in p:
                t.insert(int(csr.ids[r]), oracle.squared_l2(Q[b], csr.vectors[r]))
        oheaps.append(t)
        heaps.append(list(t.entries()))
    kmax = 32
    hi = np.zeros((B, kmax), np.uint64)
    hd = np.zeros((B, kmax), np.float64)
    hn = np.zeros(B, np.uint32)
    for b, e in enumerate(heaps):
        hn[b] = len(e)
        for j, (i, d) in enumerate(e):
            hi[b, j], hd[b, j] = i, d
    pos = np.zeros(B, np.int64)
    ctx.set_option("scan_kernel", kernel)
    try:
        while (pos < nprobe).any():
            items = np.nonzero(pos < nprobe)[0]
            off, cl, takes = [0], [], []
            for b in items:
                take = int(min(nprobe - pos[b], rng.integers(1, 5)))
                cl.extend(plans[b][pos[b]:pos[b] + take].tolist())
                off.append(len(cl))
                takes.append(take)
            a, d_, n_ = hi[items].copy(), hd[items].copy(), hn[items].copy()
            changed = ix.scan_items(Q[items], off, cl, ks[items], a, d_, n_)
            hi[items], hd[items], hn[items] = a, d_, n_
            for j, b in enumerate(items):
                npos, och = oracle.search_clusters(csr, Q[b], plans[b], int(pos[b]), oheaps[b],
                                                   plans[b][pos[b]:pos[b] + takes[j]])
                np.testing.assert_array_equal(changed[off[j]:off[j + 1]], och)
                pos[b] = npos
    finally:
        ctx.set_option("scan_kernel", 0)
        ctx.set_option("tc_wide_ppl", 0)
    for b in range(B):
        e = oheaps[b].entries()
        assert int(hn[b]) == len(e)
        assert [int(x) for x in hi[b, :len(e)]] == [i for i, _ in e]
        assert [float(x) for x in hd[b, :len(e)]] == [d for _, d in e]


def test_large_k_items_exact_path(ctx):
    ix, csr, X, centers, rng = _rand_index(ctx, 43)
    Q = rng.standard_normal((6, 32)).astype(np.float32)
    plans = ix.select_clusters(Q, 5)
    k = 64
    hi = np.zeros((6, k), np.uint64)
    hd = np.zeros((6, k), np.float64)
    hn = np.zeros(6, np.uint32)
    off = np.arange(0, 31, 5, dtype=np.uint32)
    changed = ix.scan_items(Q, off, plans.ravel(), np.full(6, k, np.uint32), hi, hd, hn)
    oi, od, oc = csr.search(Q, 5, k)
    np.testing.assert_array_equal(hn, oc)
    np.testing.assert_array_equal(hi, oi)
    assert np.array_equal(hd.view(np.uint64), od.view(np.uint64))
    assert changed.shape == (30,)


def test_device_merge_parts(ctx):
    """hivf_merge_parts_device == merge_topk over per-shard exact lists."""
    import torch
    rng = np.random.default_rng(5)
    P, B, k = 4, 7, 10
    ids = rng.integers(0, 60, (P, B, k)).astype(np.int64)
    d = np.round(rng.random((P, B, k)) * 8, 1)  # many equal distances
    cnt = rng.integers(0, k + 1, (P, B)).astype(np.int32)
    for p in range(P):  # each part sorted by (d, id) and duplicate-free, like a TopKResult
        for b in range(B):
            e = sorted(set(zip(d[p, b].tolist(), ids[p, b].tolist())))
            seen, uniq = set(), []
            for dd, ii in e:
                if ii not in seen:
                    seen.add(ii)
                    uniq.append((dd, ii))
            c = min(int(cnt[p, b]), len(uniq))
            cnt[p, b] = c
            for j in range(c):
                d[p, b, j], ids[p, b, j] = uniq[j]
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a)).to("cuda", dt)  # noqa: E731
    oi = torch.empty(B, k, dtype=torch.int64, device="cuda")
    od = torch.empty(B, k, dtype=torch.float64, device="cuda")
    oc = torch.empty(B, dtype=torch.int32, device="cuda")
    ctx.merge_parts_device(P, B, k, t(ids, torch.int64), t(d, torch.float64), t(cnt, torch.int32),
                           oi, od, oc)
    ctx.synchronize()
    for b in range(B):
        acc = []
        for p in range(P):
            acc = oracle.merge_topk(acc, [(int(ids[p, b, j]), float(d[p, b, j]))
                                          for j in range(cnt[p, b])], k)
        n = int(oc[b])
        assert n == len(acc)
        assert [int(x) for x in oi[b, :n].cpu()] == [i for i, _ in acc]
        assert [float(x) for x in od[b, :n].cpu()] == [x for _, x in acc]
