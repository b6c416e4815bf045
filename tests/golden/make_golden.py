"""Generate the golden fixtures under tests/golden/ by running the REFERENCE
itself (oracle/_ref/libhedra_ref.so = /root/reference/proj sources compiled
unmodified).  Run in the dev container (where /root/reference exists):

    python tests/golden/make_golden.py

The fixtures are small .npz files committed to the repo so the GPU box (which
has no /root/reference) checks against the reference's own outputs.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import oracle  # noqa: E402


def mixture(rng, n, dim, topics, spread):
    centers = rng.standard_normal((topics, dim))
    X = centers[np.arange(n) % topics] + rng.standard_normal((n, dim)) * spread
    return X.astype(np.float32), centers.astype(np.float32)


def case(name, seed, n, dim, K, metric, nprobes, ks, n_q=16, spread=0.3, topics=8,
         kmeans_iters=10):
    rng = np.random.default_rng(seed)
    X, centers = mixture(rng, n, dim, topics, spread)
    ids = (np.arange(n, dtype=np.uint64) * 7 + 3)  # non-trivial ids; row = (id-3)/7
    Xn = X
    if metric == 1:
        Xn = np.stack([oracle.normalized(r) for r in X])
    cents = oracle.ref_train_kmeans(Xn, K, kmeans_iters, seed)
    ri = oracle.RefIndex.build(X, ids, cents, metric)
    csr = ri.export(cents, metric)
    Q = (centers[rng.integers(0, topics, n_q)] +
         rng.standard_normal((n_q, dim)) * spread).astype(np.float32)
    out = dict(corpus=X, ids=ids, centroids=cents, metric=np.int32(metric),
               list_off=csr.off, list_ids=csr.ids, queries=Q,
               mean_assigned=np.float64(csr.mean_assigned))
    for npb in nprobes:
        plans = np.stack([ri.select_clusters(q, npb) for q in Q])
        out[f"plan_np{npb}"] = plans
        for k in ks:
            I, D, C = ri.search(Q, npb, k)
            out[f"ids_np{npb}_k{k}"] = I
            out[f"dist_np{npb}_k{k}"] = D
            out[f"count_np{npb}_k{k}"] = C
    # brute force at nprobe = K equivalence (test_vector_index.cpp:196-208)
    bi, bd = [], []
    for q in Q:
        a, b = np.zeros(10, np.uint64), np.zeros(10, np.float64)
        m = oracle.ref().ref_brute_force(X, ids, n, dim, metric, q, 10, a, b)
        assert m == min(10, n)
        bi.append(a)
        bd.append(b)
    out["brute_ids_k10"] = np.stack(bi)
    out["brute_dist_k10"] = np.stack(bd)
    # node-split sub-search trace through the reference RetrievalEngine
    # (retrieval_engine.cpp:55-152): uneven slices, per-item heap_changed,
    # completion, and the final heap + streak.
    R = oracle.ref()
    eng = R.ref_engine_new(ri.h, 10.0, 8.0, 5.0, 0, 50, 16.0, 0.5, 2)
    npb = nprobes[-1]
    k = ks[-1]
    trace_changed, trace_completed, slices = [], [], []
    for b, q in enumerate(Q):
        assert R.ref_engine_submit(eng, b, 1, q, npb, k, None, None, 0, None) == 0
    pos = np.zeros(len(Q), np.int64)
    step = 0
    while (pos < npb).any():
        live = np.nonzero(pos < npb)[0]
        reqs, nodes, offs, cl = [], [], [0], []
        for b in live:
            plan = np.zeros(npb, np.uint32)
            ln = __import__("ctypes").c_uint32()
            R.ref_engine_plan(eng, int(b), 1, plan, __import__("ctypes").byref(ln))
            take = int(min(npb - pos[b], 1 + (step + b) % 3))
            reqs.append(b)
            nodes.append(1)
            cl.extend(plan[pos[b]:pos[b] + take].tolist())
            offs.append(len(cl))
            slices.append((step, int(b), int(pos[b]), take))
            pos[b] += take
        hc = np.zeros(len(live), np.uint8)
        cp = np.zeros(len(live), np.uint8)
        rc = R.ref_engine_execute(eng, len(live), np.array(reqs, np.int64),
                                  np.array(nodes, np.int32), np.array(offs, np.uint32),
                                  np.array(cl, np.uint32), 0.0, 0, hc, cp, None, None, None,
                                  None)
        assert rc == 0
        trace_changed.append(np.stack([live, hc]))
        trace_completed.append(np.stack([live, cp]))
        step += 1
    fin_ids = np.zeros((len(Q), k), np.uint64)
    fin_d = np.zeros((len(Q), k), np.float64)
    fin_streak = np.zeros(len(Q), np.uint64)
    import ctypes as C
    for b in range(len(Q)):
        n_ = C.c_uint32()
        st = C.c_uint64()
        npos = C.c_uint64()
        srch = C.c_uint64()
        R.ref_engine_heap(eng, b, 1, fin_ids[b], fin_d[b], k, C.byref(n_), C.byref(st),
                          C.byref(npos), C.byref(srch))
        fin_streak[b] = st.value
    R.ref_engine_free(eng)
    out["sub_slices"] = np.array(slices, np.int64)
    out["sub_changed"] = np.concatenate(trace_changed, axis=1)
    out["sub_completed"] = np.concatenate(trace_completed, axis=1)
    out["sub_final_ids"] = fin_ids
    out["sub_final_dist"] = fin_d
    out["sub_final_streak"] = fin_streak
    out["sub_np"] = np.int64(npb)
    out["sub_k"] = np.int64(k)
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
    print(name, {k_: v.shape for k_, v in out.items() if hasattr(v, "shape")}.get("corpus"))


def main():
    assert oracle.ref_available(), "build oracle/_ref first (make -C oracle)"
    case("l2_d16", 11, 1500, 16, 16, 0, [1, 4, 16], [1, 10])
    case("l2_d64", 12, 3000, 64, 32, 0, [4, 8, 32], [10, 20])
    case("cos_d8", 13, 400, 8, 8, 1, [2, 8], [5])
    case("l2_d5_odd", 14, 300, 5, 10, 0, [3, 10], [7])
    case("l2_d128_c1", 15, 4000, 128, 64, 0, [8], [10], n_q=32, spread=0.25, topics=16)


if __name__ == "__main__":
    main()
