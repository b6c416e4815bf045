"""Config-5 stream driver (bench_c5.py): plan_substages restatement
(scheduler.cpp:102-156), closed-loop workflow bookkeeping, and on the GPU the
node-split path (hivf_scan_items) against the reference's RetrievalEngine over
the identical sub-stage batch sequence."""
import numpy as np
import pytest

import bench_c5 as c5
import oracle


def test_plan_substages_progress_and_budget():
    sizes = np.array([10, 20, 30, 40, 50], np.int64)
    # every entry gets its first cluster even past the budget
    assert c5.plan_substages([[0, 1], [4, 3]], sizes, 5) == [1, 1]
    # round-robin fill: 10+50 first, then 20 (80), then 40 would exceed 100
    assert c5.plan_substages([[0, 1, 2], [4, 3]], sizes, 100) == [2, 1]
    # exhausted entries close; empty entries take nothing
    assert c5.plan_substages([[0], [], [1, 2]], sizes, 1000) == [1, 0, 2]


def test_nearest_rank():
    xs = list(range(1, 101))
    assert c5.nearest_rank(xs, 50) == 50
    assert c5.nearest_rank(xs, 99) == 99
    assert c5.nearest_rank([7.0], 99) == 7.0


def _small(seed=11, n=6000, dim=16, K=48):
    rng = np.random.default_rng(seed)
    centers = rng.standard_normal((12, dim)).astype(np.float32)
    X = (centers[np.arange(n) % 12] + 0.4 * rng.standard_normal((n, dim))).astype(np.float32)
    cents = X[rng.choice(n, K, replace=False)].copy()
    assign = oracle.compute_assignments(X, cents)
    Q = (centers[rng.integers(0, 12, 64)] + 0.4 * rng.standard_normal((64, dim))).astype(np.float32)
    return X, cents, assign, Q


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("concurrency", [1, 5, 32])
def test_stream_reference_stages_equal_full_search(concurrency):
    """Every stage completed through the sliced stream equals a one-shot
    search of its query (step-split invariance, test_vector_index.cpp:169-177)."""
    X, cents, assign, Q = _small()
    ids = np.arange(len(X), dtype=np.uint64)
    ri = oracle.RefIndex.from_assignments(X, ids, cents, assign)
    sizes = np.bincount(assign, minlength=len(cents))
    nprobe, k = 8, 20
    r = c5.run_stream(c5.RefArm(ri, nprobe, k), Q, sizes, concurrency, 24, int(3 * sizes.mean()))
    assert len(r["stage_ms"]) == len(r["results"]) >= 24
    assert max(r["batch"]) <= concurrency
    wf = c5.Workflows(Q)
    # recompute each stage's query the same way the stream drew them
    qs = {}
    for _ in range(24):
        req, _, stage_qs = wf.new_request()
        for node, q in enumerate(stage_qs):
            qs[(req, node)] = q
    for key, (gi, gd) in r["results"].items():
        oi, od, oc = ri.search(qs[key][None, :], nprobe, k)
        assert np.array_equal(gi, oi[0, : oc[0]])
        assert np.array_equal(gd.view(np.uint64), od[0, : oc[0]].view(np.uint64))


@pytest.mark.gpu
@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("concurrency", [1, 7, 64])
def test_stream_gpu_equals_reference(concurrency):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_09138_b200 import Context, IvfIndex
    X, cents, assign, Q = _small(seed=12, n=20000, dim=48, K=64)
    ids = np.arange(len(X), dtype=np.uint64)
    ri = oracle.RefIndex.from_assignments(X, ids, cents, assign)
    csr = oracle.CsrIndex.from_assignments(X, ids, cents, assign)
    ix = IvfIndex.upload(Context(0), csr.centroids, csr.off, csr.vectors, csr.ids)
    sizes = np.bincount(assign, minlength=len(cents))
    nprobe, k = 12, 20
    budget = int(4 * sizes.mean())
    g = c5.run_stream(c5.GpuArm(ix, nprobe, k), Q, sizes, concurrency, 40, budget)
    r = c5.run_stream(c5.RefArm(ri, nprobe, k), Q, sizes, concurrency, 40, budget)
    assert g["batch"] == r["batch"]
    assert c5.same_results(g, r)
