"""GPU parity of the wide tensor-core scans -- the dense-batch path (DESIGN.md
"Dense batches"): k_scan_tc<64> (64-query groups streamed with the list
stages, two epilogue groups of 32 with 32-deep per-warp lists),
k_scan_tc<128> (128-query groups, two epilogue groups of 64 with 16-deep
per-warp lists) and k_scan_pair (256-query groups on CTA pairs, cta_group::2,
two candidate slots per segment).  Forced on with options tc_wide_ppl = 0,
tc_wide2_ppl and tc_pair_ppl (0: always) on the single-pass tf32 kernel;
same bar as test_gpu_parity: ids bit-exact, distances bit-equal
doubles against the C restatement of the reference."""
import numpy as np
import pytest

from test_gpu_parity import _check_search, _random_index

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", params=[(-1, -1), (0, -1), (0, 0)], ids=["groups64", "groups128", "pairs256"])
def ctx(request):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2507_09138_b200 import Context
    c = Context(0)
    c.set_option("scan_kernel", 3)
    c.set_option("tc_wide_ppl", 0)
    c.set_option("tc_wide2_ppl", request.param[0])
    c.set_option("tc_pair_ppl", request.param[1])
    c.expect_group = {(-1, -1): 64, (0, -1): 128, (0, 0): 256}[request.param]
    yield c
    c.set_option("tc_wide_ppl", 0)
    c.set_option("tc_wide2_ppl", 24)
    c.set_option("tc_pair_ppl", 96)
    c.set_option("scan_kernel", 0)


# B x nprobe / K spans groups with < 8, 8..32 (second epilogue group idle),
# 33..64, 65..128 and > 128 (several groups) queries per list
@pytest.mark.parametrize("dim,n,K,nprobe,k,B", [
    (16, 3000, 32, 8, 10, 40),
    (48, 8000, 16, 16, 20, 90),
    (128, 20000, 64, 8, 10, 300),
    (768, 30000, 64, 16, 10, 250),
    (100, 6000, 20, 20, 1, 70),
    (64, 9000, 24, 24, 32, 200),
    (768, 40000, 32, 12, 10, 700),
    (32, 20000, 8, 8, 16, 1000),
    (768, 50000, 16, 8, 10, 800),
])
def test_wide_scan_vs_oracle(ctx, dim, n, K, nprobe, k, B):
    rng = np.random.default_rng(dim * 13 + K + B)
    ix, csr, X, centers = _random_index(ctx, rng, n, dim, K)
    Q = (centers[rng.integers(0, len(centers), B)] +
         rng.standard_normal((B, dim)).astype(np.float32) * 0.3).astype(np.float32)
    _check_search(ix, csr, Q, nprobe, k)
    st = ctx.stats()
    assert st["scan_kernel"] == 3 and st["n_work_items"] > 0, st
    assert st["scan_group"] == ctx.expect_group, st


def test_wide_scan_segments_skew_and_empty_lists(ctx):
    rng = np.random.default_rng(71)
    ctx.set_option("seg_rows", 512)
    try:
        ix, csr, X, centers = _random_index(ctx, rng, 12000, 32, 12, spread=0.5, skew=True)
        Q = (X[rng.choice(len(X), 180)] + 0.01).astype(np.float32)
        for nprobe, k in [(1, 10), (3, 5), (12, 32)]:
            _check_search(ix, csr, Q, nprobe, k)
    finally:
        ctx.set_option("seg_rows", 0)


def test_wide_and_narrow_agree_on_dense_batch(ctx):
    """The same dense batch through the wide and the narrow kernel: identical
    results (both equal the reference)."""
    rng = np.random.default_rng(5)
    ix, csr, X, centers = _random_index(ctx, rng, 40000, 768, 32)
    Q = (centers[rng.integers(0, len(centers), 400)] +
         rng.standard_normal((400, 768)).astype(np.float32) * 0.3).astype(np.float32)
    a = ix.search(Q, 16, 10)
    ctx.set_option("tc_wide_ppl", -1)
    try:
        b = ix.search(Q, 16, 10)
    finally:
        ctx.set_option("tc_wide_ppl", 0)
    for x, y in zip(a, b):
        assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
    _check_search(ix, csr, Q, 16, 10)


def test_drop_bound_seed_same_results(ctx):
    """The drop-bound seed (exact distances of a few rows of each query's
    nearest list) only removes work: seeded and unseeded scans give the
    reference's bits."""
    rng = np.random.default_rng(44)
    ix, csr, X, centers = _random_index(ctx, rng, 30000, 96, 24)
    Q = (centers[rng.integers(0, len(centers), 600)] +
         rng.standard_normal((600, 96)).astype(np.float32) * 0.3).astype(np.float32)
    try:
        for rows, ppl in ((32, 0), (64, 0), (10, 0), (0, 0)):
            ctx.set_option("seed_rows", rows)
            ctx.set_option("seed_ppl", ppl)
            _check_search(ix, csr, Q, 8, 10)
            _check_search(ix, csr, Q, 3, 1)
    finally:
        ctx.set_option("seed_rows", 32)
        ctx.set_option("seed_ppl", 16)
