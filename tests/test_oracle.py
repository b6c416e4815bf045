"""CPU tests: pin the oracle (C restatement) against the reference's own
known answers and against the reference sources compiled unmodified
(oracle/_ref, when present)."""
import glob
import os

import numpy as np
import pytest

import oracle

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz")))


def corpus_a():
    # proj/tests/test_support.hpp:11-25
    pts = np.array([[0, 0], [.1, 0], [0, .1], [.1, .1], [10, 10], [10.1, 10], [9.9, 10.05],
                    [10, 10.05]], np.float32)
    return pts, np.arange(8, dtype=np.uint64)


def test_corpus_a_known_answers():
    # proj/tests/test_vector_index.cpp:109-155
    pts, ids = corpus_a()
    cents = np.array([[0.05, 0.05], [10.0, 10.025]], np.float32)
    assign = oracle.compute_assignments(pts, cents)
    assert list(assign) == [0, 0, 0, 0, 1, 1, 1, 1]
    csr = oracle.CsrIndex.from_assignments(pts, ids, cents, assign)
    assert list(csr.select_clusters(np.array([1.0, 0.0], np.float32), 1)) == [0]
    assert list(csr.select_clusters(np.array([1.0, 0.0], np.float32), 2)) == [0, 1]
    with pytest.raises(ValueError):
        csr.select_clusters(np.array([1.0, 0.0], np.float32), 0)
    with pytest.raises(ValueError):
        csr.select_clusters(np.array([1.0, 0.0], np.float32), 3)
    I, D, C = csr.search(np.array([[0.0, 0.0]], np.float32), 2, 1)
    assert C[0] == 1 and I[0, 0] == 0 and D[0, 0] == 0.0
    # brute force basics (test_vector_index.cpp:179-194)
    bi, bd = oracle.brute_force(pts, ids, np.zeros(2, np.float32), 100)
    assert len(bi) == 8 and np.all(np.diff(bd) >= 0)
    bi, bd = oracle.brute_force(np.zeros((0, 2), np.float32), np.zeros(0, np.uint64),
                                np.zeros(2, np.float32), 3)
    assert len(bi) == 0


def test_centroid_tie_lower_id():
    # test_vector_index.cpp:91-102
    a = oracle.compute_assignments(np.array([[0.0]], np.float32),
                                   np.array([[-1.0], [1.0]], np.float32))
    assert a[0] == 0


def test_merge_topk_known_answer():
    # test_vector_index.cpp:227-246
    x = oracle.TopK(3)
    x.insert(1, 0.5)
    x.insert(2, 0.25)
    assert oracle.merge_topk(x.entries(), [], 3) == x.entries()
    assert oracle.merge_topk(x.entries(), [], 1) == x.entries()[:1]
    y = oracle.TopK(3)
    y.insert(3, 0.1)
    y.insert(1, 0.75)
    ab = oracle.merge_topk(x.entries(), y.entries(), 3)
    ba = oracle.merge_topk(y.entries(), x.entries(), 3)
    assert ab == ba
    assert [i for i, _ in ab] == [3, 2, 1]
    assert ab[2][1] == 0.5


def test_topk_insert_semantics():
    t = oracle.TopK(2)
    assert t.insert(5, 1.0)
    assert not t.insert(5, 2.0)  # duplicate, worse
    assert t.insert(5, 0.5)  # duplicate, better
    assert t.insert(6, 0.7)
    assert not t.insert(7, 0.9)  # full, not better
    assert t.insert(8, 0.1)
    assert t.entries() == [(8, 0.1), (5, 0.5)]
    assert not oracle.TopK(0).insert(1, 0.0)


def test_squared_l2_sequential_double():
    a = np.array([1e8, 1.0, -3.0], np.float32)
    b = np.array([0.0, 0.5, 1e-3], np.float32)
    acc = 0.0
    for x, y in zip(a, b):
        d = float(x) - float(y)
        acc += d * d
    assert oracle.squared_l2(a, b) == acc


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_oracle_matches_reference_golden(path):
    """The restatement reproduces the reference's own outputs bit for bit."""
    g = np.load(path)
    metric = int(g["metric"])
    rows = ((g["list_ids"] - 3) // 7).astype(np.int64)
    vec = g["corpus"][rows]
    if metric == 1:
        vec = np.stack([oracle.normalized(r) for r in vec])
    csr = oracle.CsrIndex(g["centroids"], g["list_off"], vec, g["list_ids"], metric)
    Q = g["queries"]
    for key in g.files:
        if key.startswith("plan_np"):
            npb = int(key[len("plan_np"):])
            plans, _ = csr.assign(Q, npb)
            np.testing.assert_array_equal(plans, g[key])
        if key.startswith("ids_np"):
            npb, k = (int(v) for v in key[len("ids_np"):].split("_k"))
            I, D, C = csr.search(Q, npb, k)
            np.testing.assert_array_equal(I, g[key])
            assert np.array_equal(D.view(np.uint64), g[f"dist_np{npb}_k{k}"].view(np.uint64))
            np.testing.assert_array_equal(C, g[f"count_np{npb}_k{k}"])
    # index build: exact assignments (ties -> lowest id) reproduce the lists
    Xn = g["corpus"] if metric == 0 else np.stack([oracle.normalized(r) for r in g["corpus"]])
    assign = oracle.compute_assignments(Xn, g["centroids"])
    csr2 = oracle.CsrIndex.from_assignments(Xn, g["ids"], g["centroids"], assign, metric)
    np.testing.assert_array_equal(csr2.off, g["list_off"])
    np.testing.assert_array_equal(csr2.ids, g["list_ids"])


@pytest.mark.parametrize("path", GOLDEN, ids=[os.path.basename(p) for p in GOLDEN])
def test_oracle_subsearch_trace(path):
    """search_clusters over uneven slices reproduces the reference engine's
    per-item heap_changed flags and final heaps (retrieval_engine.cpp:55-152)."""
    g = np.load(path)
    metric = int(g["metric"])
    rows = ((g["list_ids"] - 3) // 7).astype(np.int64)
    vec = g["corpus"][rows]
    if metric == 1:
        vec = np.stack([oracle.normalized(r) for r in vec])
    csr = oracle.CsrIndex(g["centroids"], g["list_off"], vec, g["list_ids"], metric)
    Q = g["queries"]
    npb, k = int(g["sub_np"]), int(g["sub_k"])
    heaps = [oracle.TopK(k) for _ in Q]
    pos = [0] * len(Q)
    plans = [csr.select_clusters(q, npb) for q in Q]
    qs = [oracle.normalized(q) if metric == 1 else q for q in Q]
    changed_trace = []
    for step, b, p0, take in g["sub_slices"]:
        assert p0 == pos[b]
        npos, ch = oracle.search_clusters(csr, qs[b], plans[b], pos[b], heaps[b],
                                          plans[b][p0:p0 + take])
        pos[b] = npos
        changed_trace.append(bool(ch.any()))
    np.testing.assert_array_equal(np.array(changed_trace), g["sub_changed"][1].astype(bool))
    for b in range(len(Q)):
        e = heaps[b].entries()
        np.testing.assert_array_equal([i for i, _ in e], g["sub_final_ids"][b][:len(e)])
        assert [d for _, d in e] == list(g["sub_final_dist"][b][:len(e)])


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_oracle_vs_reference_random():
    rng = np.random.default_rng(5)
    for trial in range(6):
        dim = int(rng.integers(2, 40))
        n = int(rng.integers(200, 1500))
        K = int(rng.integers(4, 20))
        X = rng.standard_normal((n, dim)).astype(np.float32)
        ids = rng.permutation(n).astype(np.uint64)
        cents = oracle.ref_train_kmeans(X, K, 5, trial)
        ri = oracle.RefIndex.build(X, ids, cents)
        csr = ri.export(cents)
        assign = oracle.compute_assignments(X, cents)
        csr2 = oracle.CsrIndex.from_assignments(X, ids, cents, assign)
        np.testing.assert_array_equal(csr.off, csr2.off)
        np.testing.assert_array_equal(csr.ids, csr2.ids)
        Q = rng.standard_normal((8, dim)).astype(np.float32)
        npb = int(rng.integers(1, K + 1))
        k = int(rng.integers(1, 30))
        a = ri.search(Q, npb, k)
        b = csr.search(Q, npb, k)
        for x, y in zip(a, b):
            assert np.array_equal(np.asarray(x).view(np.uint8), np.asarray(y).view(np.uint8))
