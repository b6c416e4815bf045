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
