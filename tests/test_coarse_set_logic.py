"""Host restatement of k_coarse_select's set mode (assign.cu), checked on CPU:
with filter distances d^ = d + e, |e| <= E, upper/lower bounds ub = d^ + E,
lb = d^ - E, tau = the nprobe-th smallest ub and L = the nprobe-th smallest
lb, the plan built as {ub < L} (sure) + the best (nprobe - |sure|) of the band
{lb <= tau, ub >= L} by exact (d, id) is exactly the reference's top-nprobe
(vector_index.cpp:266-277, (distance, id) order) as a set.  Adversarial cases:
exact ties (duplicate centroids), errors at the bound's edge, tiny K."""
import numpy as np
import pytest


def _plan_set_mode(d, dh, E, nprobe):
    ub, lb = dh + E, dh - E
    tau = np.sort(ub)[nprobe - 1]
    L = np.sort(lb)[nprobe - 1]
    cand = lb <= tau
    sure = cand & (ub < L)
    band = np.nonzero(cand & ~sure)[0]
    assert sure.sum() <= nprobe
    order = np.lexsort((band, d[band]))  # (d, id)
    take = band[order[: nprobe - int(sure.sum())]]
    return set(np.nonzero(sure)[0].tolist()) | set(take.tolist())


def _reference_top(d, nprobe):
    ids = np.arange(len(d))
    return set(np.lexsort((ids, d))[:nprobe].tolist())


@pytest.mark.parametrize("seed", range(40))
def test_set_mode_equals_reference_top_nprobe(seed):
    rng = np.random.default_rng(seed)
    K = int(rng.integers(1, 600))
    nprobe = int(rng.integers(1, K + 1))
    d = rng.random(K)
    if seed % 3 == 0:  # exact ties: duplicated centroids
        d[rng.integers(0, K, K // 3)] = d[rng.integers(0, K, K // 3)]
    if seed % 4 == 1:  # coarse distances on a grid: many ties
        d = np.round(d * 16) / 16
    E = rng.random(K) * (10.0 ** rng.uniform(-4, -1))
    e = rng.uniform(-1, 1, K) * E
    if seed % 5 == 2:  # errors at the edge of the bound
        e = np.sign(e) * E
    dh = d + e
    assert _plan_set_mode(d, dh, E, nprobe) == _reference_top(d, nprobe)
