"""Config 5 of BASELINE.json: a heterogeneous multi-stage RAG retrieval stream
driving node-split sub-searches, batch 1-512, p50/p99 search latency.

Bench infrastructure (not product).  What the reference's scheduler does on the
retrieval side (proj/src/scheduler.cpp), restated without the LLM:

* requests arrive as workflows: one-shot (1 retrieval stage), HyDE (1 stage on
  a hypothetical-document embedding) and iterative / multi-step (3 sequential
  stages, each ready when the previous one completes);
* a retrieval stage is a cursor: make_cursor (select_clusters) with
  k = max(topk, k_cache=20) (scheduler.cpp:917-920);
* every engine step, plan_substages (scheduler.cpp:102-156, restated in
  `plan_substages` below with cost = list rows, i.e. cluster_variable_ms up to
  the constant per_vector_ns) slices each live cursor's remaining plan
  round-robin under a budget -> one SubStageBatch -> RetrievalEngine::execute;
* the stream is closed-loop at a fixed concurrency C (live stages); C sweeps
  1..512, which is the batch-size range of configs[4].

Both arms consume the identical batch sequence (the planning depends only on
plans and list sizes, never on timing): ours through hivf_scan_items (host
buffers, one call per sub-stage), the reference's own RetrievalEngine::execute
(oracle/_ref, live_math=true on all host cores).  Every completed stage's heap
is compared bit-for-bit between the arms.

Latencies are engine time: each arm times its own API calls (wall clock,
synchronous, host buffers in/out) -- `substage` = make_cursor of the stages
admitted at that step + one SubStageBatch execute; `stage` = admission ->
completing sub-stage of a retrieval stage on the clock that advances only by
engine time (the search latency a request sees; generation time and this
driver's own bookkeeping / plan_substages excluded).  Percentiles are
nearest-rank as in proj/src/report.cpp:15-21.
"""
from __future__ import annotations

import math
import time

import numpy as np

K_CACHE = 20  # proj/include/hedra/similarity.hpp:15


def nearest_rank(xs, p):
    """report.cpp:15-21: nearest-rank percentile of a sample."""
    if not len(xs):
        return None
    s = sorted(xs)
    r = max(1, int(math.ceil(p / 100.0 * len(s))))
    return float(s[r - 1])


def plan_substages(remaining, sizes, budget_rows):
    """scheduler.cpp:102-156: every entry gets its first cluster, then a
    round-robin fill while the next cluster fits the budget.  Returns the
    number of clusters taken per entry."""
    n = len(remaining)
    taken = [0] * n
    closed = [False] * n
    planned = 0
    for i, r in enumerate(remaining):
        if len(r) == 0:
            closed[i] = True
            continue
        planned += int(sizes[r[0]])
        taken[i] = 1
        if taken[i] == len(r):
            closed[i] = True
    progressed = True
    while progressed:
        progressed = False
        for i, r in enumerate(remaining):
            if closed[i]:
                continue
            cost = int(sizes[r[taken[i]]])
            if planned + cost > budget_rows:
                closed[i] = True
                continue
            planned += cost
            taken[i] += 1
            progressed = True
            if taken[i] == len(r):
                closed[i] = True
    return taken


class Workflows:
    """Deterministic request stream: (req, node, query) stages with
    dependencies (iterative stages become ready when the previous completes)."""

    MIX = (("one-shot", 1, 0.4), ("hyde", 1, 0.2), ("iterative", 3, 0.4))

    def __init__(self, queries: np.ndarray, seed: int = 5):
        self.Q = queries
        self.rng = np.random.default_rng(seed)
        self.next_req = 0
        self.next_q = 0

    def new_request(self):
        u = self.rng.random()
        acc = 0.0
        for name, stages, p in self.MIX:
            acc += p
            if u <= acc:
                break
        req = self.next_req
        self.next_req += 1
        qs = []
        for _ in range(stages):
            qs.append(self.Q[self.next_q % len(self.Q)])
            self.next_q += 1
        return req, name, qs


class GpuArm:
    """Cursors on the host (plans, next_pos, heaps), sub-stages through
    hivf_scan_items -- what hedra_gpu::ret::RetrievalEngine does."""

    name = "hivf"

    def __init__(self, ix, nprobe, k):
        self.ix, self.nprobe, self.k = ix, nprobe, k
        self.cur = {}
        self.api_ms = []  # time inside hivf_scan_items (the C-ABI call) per sub-stage

    def submit(self, keys, queries):
        Q = np.stack(queries).astype(np.float32)
        t0 = time.perf_counter()
        plans = self.ix.select_clusters(Q, self.nprobe)  # make_cursor's select_clusters, batched
        self.last_ms = (time.perf_counter() - t0) * 1e3
        out = []
        for key, q, p in zip(keys, queries, plans):
            self.cur[key] = {"q": np.asarray(q, np.float32), "plan": p.astype(np.uint32), "pos": 0,
                             "ids": np.zeros(self.k, np.uint64), "d": np.zeros(self.k, np.float64),
                             "n": 0}
            out.append(p)
        return out

    def execute(self, items):
        n = len(items)
        Q = np.stack([self.cur[key]["q"] for key, _ in items])
        off = np.zeros(n + 1, np.uint32)
        cl = []
        for i, (key, m) in enumerate(items):
            c = self.cur[key]
            cl.append(c["plan"][c["pos"]:c["pos"] + m])
            off[i + 1] = off[i] + m
        clusters = np.concatenate(cl).astype(np.uint32)
        hi = np.stack([self.cur[key]["ids"] for key, _ in items])
        hd = np.stack([self.cur[key]["d"] for key, _ in items])
        hn = np.array([self.cur[key]["n"] for key, _ in items], np.uint32)
        kv = np.full(n, self.k, np.uint32)
        t0 = time.perf_counter()
        self.ix.scan_items(Q, off, clusters, kv, hi, hd, hn)
        self.last_ms = (time.perf_counter() - t0) * 1e3
        self.api_ms.append(self.last_ms)
        done = []
        for i, (key, m) in enumerate(items):
            c = self.cur[key]
            c["ids"], c["d"], c["n"] = hi[i], hd[i], int(hn[i])
            c["pos"] += m
            if c["pos"] == len(c["plan"]):
                done.append(key)
        return done

    def position(self, key):
        return self.cur[key]["pos"]

    def result(self, key):
        c = self.cur.pop(key)
        return c["ids"][: c["n"]].copy(), c["d"][: c["n"]].copy()


class RefArm:
    """The reference's RetrievalEngine (oracle/_ref) on the host cores."""

    name = "reference"

    def __init__(self, ref_index, nprobe, k):
        import oracle
        self.eng = oracle.RefEngine(ref_index)
        self.nprobe, self.k = nprobe, k
        self.pos = {}
        self.plans = {}

    def submit(self, keys, queries):
        out = []
        t0 = time.perf_counter()
        for key, q in zip(keys, queries):
            p = self.eng.submit(key[0], key[1], q, self.nprobe, self.k)
            self.plans[key] = p
            self.pos[key] = 0
            out.append(p)
        self.last_ms = (time.perf_counter() - t0) * 1e3
        return out

    def execute(self, items):
        reqs = np.array([key[0] for key, _ in items], np.int64)
        nodes = np.array([key[1] for key, _ in items], np.int32)
        off = np.zeros(len(items) + 1, np.uint32)
        cl = []
        for i, (key, m) in enumerate(items):
            cl.append(self.plans[key][self.pos[key]:self.pos[key] + m])
            off[i + 1] = off[i] + m
        cls = np.concatenate(cl)
        t0 = time.perf_counter()
        _, completed = self.eng.execute(reqs, nodes, off, cls, live=True)
        self.last_ms = (time.perf_counter() - t0) * 1e3
        done = []
        for i, (key, m) in enumerate(items):
            self.pos[key] += m
            if completed[i]:
                done.append(key)
        return done

    def position(self, key):
        return self.pos[key]

    def result(self, key):
        ids, d, _ = self.eng.heap(key[0], key[1])
        self.eng.extract(key[0], key[1])
        del self.plans[key], self.pos[key]
        return ids, d


def run_stream(arm, queries, sizes, concurrency, n_requests, budget_rows, seed=5):
    """Closed-loop stream at `concurrency` live stages until n_requests
    requests have completed all their stages.  Returns latencies, batch sizes,
    the plans seen and every completed stage's heap."""
    wf = Workflows(queries, seed)
    pending = []          # ready stages not yet live: (key, query)
    follow = {}           # req -> remaining stage queries
    live = []             # keys in admission order
    t_start = {}
    results, plans = {}, {}
    sub_ms, stage_ms, batch = [], [], []
    clock = 0.0  # ms of engine time
    started = finished = 0
    while finished < n_requests:
        # admit: ready follow-up stages first, then new requests
        while len(live) + len(pending) < concurrency and started < n_requests:
            req, _, qs = wf.new_request()
            started += 1
            pending.append(((req, 0), qs[0]))
            follow[req] = qs[1:]
        admit = pending[: max(0, concurrency - len(live))]
        pending = pending[len(admit):]
        # engine time only (the arms time their own API calls): make_cursor for the
        # admitted stages + one SubStageBatch execute; the stream's bookkeeping and
        # plan_substages (the scheduler's work) advance no clock
        t0 = clock
        eng = 0.0
        if admit:
            ps = arm.submit([k for k, _ in admit], [q for _, q in admit])
            eng += arm.last_ms
            for (key, _), p in zip(admit, ps):
                plans[key] = np.asarray(p, np.uint32)
                t_start[key] = t0
                live.append(key)
        remaining = [plans[key][arm.position(key):] for key in live]
        taken = plan_substages(remaining, sizes, budget_rows)
        items = [(key, m) for key, m in zip(live, taken) if m > 0]
        done = arm.execute(items)
        eng += arm.last_ms
        clock += eng
        t1 = clock
        sub_ms.append(eng)
        batch.append(len(items))
        for key in done:
            results[key] = arm.result(key)
            stage_ms.append(t1 - t_start.pop(key))
            live.remove(key)
            req, node = key
            if follow.get(req):
                pending.insert(0, ((req, node + 1), follow[req].pop(0)))
            else:
                follow.pop(req, None)
                finished += 1
    return {"substage_ms": sub_ms, "stage_ms": stage_ms, "batch": batch, "results": results,
            "plans": plans, "api_ms": list(getattr(arm, "api_ms", []))}


def summarize(r):
    b = np.asarray(r["batch"])
    return {"substages": len(r["substage_ms"]), "stages": len(r["stage_ms"]),
            "batch_items": {"min": int(b.min()), "p50": int(nearest_rank(b, 50)),
                            "max": int(b.max())},
            "substage_ms": {"p50": round(nearest_rank(r["substage_ms"], 50), 3),
                            "p99": round(nearest_rank(r["substage_ms"], 99), 3)},
            "stage_ms": {"p50": round(nearest_rank(r["stage_ms"], 50), 3),
                         "p99": round(nearest_rank(r["stage_ms"], 99), 3)},
            **({"api_call_ms": {"p50": round(nearest_rank(r["api_ms"], 50), 3),
                                "p99": round(nearest_rank(r["api_ms"], 99), 3)}} if r.get("api_ms") else {})}


def same_results(a, b):
    if set(a["results"]) != set(b["results"]):
        return False
    for key, (ia, da) in a["results"].items():
        ib, db = b["results"][key]
        if not (np.array_equal(ia, ib) and np.array_equal(np.asarray(da).view(np.uint64),
                                                          np.asarray(db).view(np.uint64))):
            return False
        if not np.array_equal(a["plans"][key], b["plans"][key]):
            return False
    return True


__all__ = ["plan_substages", "run_stream", "summarize", "same_results", "GpuArm", "RefArm",
           "nearest_rank", "K_CACHE"]
