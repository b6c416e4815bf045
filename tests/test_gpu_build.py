"""GPU index build vs the reference's own train_kmeans / compute_assignments
(oracle/_ref: proj/src/vector_index.cpp:99-208 compiled unmodified):
centroids and assignments must be bit-identical."""
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
    return Context(0, torch.cuda.current_stream())


def _mixture(seed, n, dim, topics, spread):
    rng = np.random.default_rng(seed)
    c = rng.standard_normal((topics, dim))
    c /= np.linalg.norm(c, axis=1, keepdims=True)
    return (c[np.arange(n) % topics] + spread * rng.standard_normal((n, dim))).astype(np.float32)


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("n,dim,K,iters,seed", [
    (3000, 8, 16, 10, 1),      # small dims, several Lloyd steps, convergence
    (5000, 33, 40, 4, 7),      # odd dim (scalar tail of the row loads)
    (4000, 128, 64, 3, 42),
    (300, 4, 60, 5, 3),        # many clusters per point: empty-cluster re-seeding
])
def test_train_kmeans_bit_exact(ctx, n, dim, K, iters, seed):
    import torch
    X = _mixture(seed, n, dim, max(2, K // 3), 0.3)
    ref = oracle.ref_train_kmeans(X, K, iters, seed)
    dX = torch.from_numpy(X).cuda()
    out = torch.empty(K, dim, dtype=torch.float32, device="cuda")
    ctx.train_kmeans(dX, K, iters, seed, out)
    torch.cuda.synchronize()
    got = out.cpu().numpy()
    assert np.array_equal(got.view(np.uint32), ref.view(np.uint32))


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_train_kmeans_duplicate_points(ctx):
    """All-duplicate corpus: total == 0 -> lowest untaken index (vector_index.cpp:137-151)."""
    import torch
    base = _mixture(5, 6, 16, 3, 0.2)
    X = np.repeat(base, 50, axis=0)
    K = 6
    ref = oracle.ref_train_kmeans(X, K, 5, 11)
    out = torch.empty(K, 16, dtype=torch.float32, device="cuda")
    ctx.train_kmeans(torch.from_numpy(X).cuda(), K, 5, 11, out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().view(np.uint32), ref.view(np.uint32))


@pytest.mark.parametrize("n,dim,K", [(20000, 64, 256), (7000, 17, 33), (50000, 768, 128)])
def test_compute_assignments_bit_exact(ctx, n, dim, K):
    import torch
    X = _mixture(n + dim, n, dim, 24, 0.25)
    rng = np.random.default_rng(0)
    cents = X[rng.choice(n, K, replace=False)].copy()
    cents[1] = cents[0]  # duplicate centroid: ties -> lowest id
    want = oracle.compute_assignments(X, cents)
    out = torch.empty(n, dtype=torch.int32, device="cuda")
    ctx.compute_assignments(torch.from_numpy(X).cuda(), torch.from_numpy(cents).cuda(), out)
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().astype(np.uint32), np.asarray(want, np.uint32))


def test_train_kmeans_invalid_args(ctx):
    import torch
    from paper_2507_09138_b200 import InvalidArgument
    X = torch.zeros(10, 4, device="cuda")
    out = torch.empty(20, 4, device="cuda")
    with pytest.raises(InvalidArgument):
        ctx.train_kmeans(X, 20, 3, 1, out)   # n < K
    with pytest.raises(InvalidArgument):
        ctx.train_kmeans(X, 4, 0, 1, out)    # max_iters == 0


def test_bench_exact_assign_equals_library_and_oracle(ctx):
    """The two assignment paths of bench.py (ours: hivf_compute_assignments;
    the reference arm's torch restatement bench_workload.exact_assign) give
    the reference's compute_assignments, incl. near-ties at D=768."""
    import torch
    from bench_workload import Config, Workload
    cfg = Config("t", 40000, 768, 96, 8, 10, 16, 0.03)
    wl = Workload(cfg, device="cuda")
    cents = wl.train_centroids(iters=2, sample_per_centroid=20)
    cents[5] = cents[4]  # exact tie -> lowest id
    X = wl.chunk(0)[: cfg.n]
    want = np.asarray(oracle.compute_assignments(X.cpu().numpy(), cents.cpu().numpy()), np.int64)
    got_t = wl.exact_assign(cents).cpu().numpy()
    got_l = wl.library_assign(ctx, cents).cpu().numpy()
    assert np.array_equal(got_t, want)
    assert np.array_equal(got_l, want)


def test_train_kmeans_sampled_seeds_lloyd_fixed_point(ctx):
    """Parallel training mode: deterministic, and after convergence every
    centroid is the reference's Lloyd update of its cluster (point-order
    double mean, vector_index.cpp:156-197) under the exact assignment."""
    import torch
    n, dim, K = 6000, 24, 20
    X = _mixture(77, n, dim, 10, 0.3)
    dX = torch.from_numpy(X).cuda()
    a = torch.empty(K, dim, device="cuda")
    b = torch.empty(K, dim, device="cuda")
    ctx.train_kmeans_sampled_seeds(dX, K, 100, 5, a)
    ctx.train_kmeans_sampled_seeds(dX, K, 100, 5, b)
    torch.cuda.synchronize()
    C = a.cpu().numpy()
    assert np.array_equal(C.view(np.uint32), b.cpu().numpy().view(np.uint32))
    asg = np.asarray(oracle.compute_assignments(X, C), np.int64)
    for c in range(K):
        rows = X[asg == c].astype(np.float64)
        assert len(rows) > 0
        s = np.zeros(dim)
        for r in rows:  # point order, double accumulate
            s += r
        assert np.array_equal((s / len(rows)).astype(np.float32).view(np.uint32), C[c].view(np.uint32))
