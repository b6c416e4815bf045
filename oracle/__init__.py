"""Oracle (TEST INFRASTRUCTURE ONLY).

ctypes bindings over
  * ``liboracle.so``          -- our plain-C restatement (hivf_oracle.c), and
  * ``_ref/libhedra_ref.so``  -- the reference's own sources compiled unmodified
                                 (oracle/Makefile, ref_shim.cpp).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg import this package, and only as the checker or the
timed CPU baseline -- never as the thing measured for the GPU arm.  The product
package (paper_2507_09138_b200/) never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE = os.path.join(HERE, "liboracle.so")
_REF = os.path.join(HERE, "_ref", "libhedra_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


def build() -> None:
    """Compile liboracle.so (and _ref when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class OrcEntry(C.Structure):
    _fields_ = [("id", C.c_uint64), ("d", C.c_double)]


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_ORACLE):
            build()
        L = C.CDLL(_ORACLE)
        L.orc_squared_l2.restype = C.c_double
        L.orc_squared_l2.argtypes = [_f32p, _f32p, C.c_uint64]
        L.orc_select_clusters.restype = C.c_int
        L.orc_select_clusters.argtypes = [_f32p, C.c_uint32, C.c_uint32, C.c_int, _f32p,
                                          C.c_uint32, _u32p, C.c_void_p]
        L.orc_ivf_search.restype = C.c_int
        L.orc_ivf_search.argtypes = [_f32p, C.c_uint32, C.c_uint32, C.c_int, _f32p, _u64p,
                                     _u64p, _f32p, C.c_uint32, C.c_uint32, C.c_uint32, _u64p,
                                     _f64p, _u32p]
        L.orc_brute_force.restype = C.c_uint64
        L.orc_brute_force.argtypes = [_f32p, _u64p, C.c_uint64, C.c_uint32, C.c_int, _f32p,
                                      C.c_uint64, _u64p, _f64p]
        L.orc_compute_assignments.restype = None
        L.orc_compute_assignments.argtypes = [_f32p, C.c_uint64, C.c_uint32, _f32p,
                                              C.c_uint32, _u32p]
        L.orc_normalized.restype = None
        L.orc_normalized.argtypes = [_f32p, C.c_uint64, _f32p]
        L.orc_topk_insert.restype = C.c_int
        L.orc_topk_insert.argtypes = [C.POINTER(OrcEntry), C.POINTER(C.c_uint64), C.c_uint64,
                                      C.c_uint64, C.c_double]
        L.orc_merge_topk.restype = C.c_uint64
        L.orc_merge_topk.argtypes = [C.POINTER(OrcEntry), C.c_uint64, C.POINTER(OrcEntry),
                                     C.c_uint64, C.c_uint64, C.POINTER(OrcEntry)]
        L.orc_search_clusters.restype = C.c_int
        L.orc_search_clusters.argtypes = [_f32p, _u64p, _u64p, C.c_uint32, _f32p, _u32p,
                                          C.c_uint32, C.POINTER(C.c_uint32),
                                          C.POINTER(OrcEntry), C.POINTER(C.c_uint64),
                                          C.c_uint64, _u32p, C.c_uint32, _u8p]
        _lib = L
    return _lib


def ref_available() -> bool:
    return os.path.exists(_REF)


def ref():
    """The reference's own compiled code (None-safe: raises if not built)."""
    global _ref
    if _ref is None:
        if not os.path.exists(_REF):
            build()
        R = C.CDLL(_REF)
        vp = C.c_void_p
        R.ref_index_build.restype = vp
        R.ref_index_build.argtypes = [_f32p, _u64p, C.c_uint64, C.c_uint32, C.c_int, _f32p,
                                      C.c_uint32]
        R.ref_index_from_assign.restype = vp
        R.ref_index_from_assign.argtypes = [_f32p, _u64p, C.c_uint64, C.c_uint32, C.c_int,
                                            _f32p, C.c_uint32, _u32p]
        R.ref_index_from_csr.restype = vp
        R.ref_index_from_csr.argtypes = [_f32p, C.c_uint32, C.c_uint32, C.c_int, _u64p, _f32p, _u64p]
        R.ref_index_free.argtypes = [vp]
        R.ref_index_total.restype = C.c_uint64
        R.ref_index_total.argtypes = [vp]
        R.ref_index_export.argtypes = [vp, _u64p, vp, vp, C.POINTER(C.c_double)]
        R.ref_train_kmeans.restype = C.c_int
        R.ref_train_kmeans.argtypes = [_f32p, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.c_uint64, _f32p]
        R.ref_compute_assignments.restype = C.c_int
        R.ref_compute_assignments.argtypes = [_f32p, C.c_uint64, C.c_uint32, _f32p,
                                              C.c_uint32, _u32p]
        for nm in ("ref_save_corpus", "ref_save_centroids", "ref_save_assignments", "ref_load_corpus"):
            getattr(R, nm).restype = C.c_int
        R.ref_save_corpus.argtypes = [C.c_char_p, _f32p, _u64p, C.c_uint64, C.c_uint32, C.c_int]
        R.ref_save_centroids.argtypes = [C.c_char_p, _f32p, C.c_uint32, C.c_uint32, C.c_int]
        R.ref_save_assignments.argtypes = [C.c_char_p, _u32p, C.c_uint64]
        R.ref_load_corpus.argtypes = [C.c_char_p, C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_int), C.c_void_p, C.c_void_p]
        R.ref_select_clusters.restype = C.c_int
        R.ref_select_clusters.argtypes = [vp, _f32p, C.c_uint32, _u32p]
        R.ref_search.restype = C.c_int
        R.ref_search.argtypes = [vp, _f32p, C.c_uint32, C.c_uint32, C.c_uint32, _u64p, _f64p,
                                 _u32p]
        R.ref_brute_force.restype = C.c_uint64
        R.ref_brute_force.argtypes = [_f32p, _u64p, C.c_uint64, C.c_uint32, C.c_int, _f32p,
                                      C.c_uint64, _u64p, _f64p]
        R.ref_merge_topk.restype = C.c_uint64
        R.ref_merge_topk.argtypes = [_u64p, _f64p, C.c_uint64, _u64p, _f64p, C.c_uint64,
                                     C.c_uint64, _u64p, _f64p]
        R.ref_engine_new.restype = vp
        R.ref_engine_new.argtypes = [vp, C.c_double, C.c_double, C.c_double, C.c_uint64,
                                     C.c_int, C.c_double, C.c_double, C.c_uint64]
        R.ref_engine_free.argtypes = [vp]
        R.ref_engine_submit.restype = C.c_int
        R.ref_engine_submit.argtypes = [vp, C.c_int64, C.c_int32, _f32p, C.c_uint32,
                                        C.c_uint32, vp, vp, C.c_uint32, vp]
        R.ref_engine_plan.restype = C.c_int
        R.ref_engine_plan.argtypes = [vp, C.c_int64, C.c_int32, _u32p, C.POINTER(C.c_uint32)]
        R.ref_engine_execute.restype = C.c_int
        R.ref_engine_execute.argtypes = [vp, C.c_uint32, _i64p, _i32p, _u32p, _u32p,
                                         C.c_double, C.c_int, _u8p, _u8p,
                                         C.POINTER(C.c_double), C.POINTER(C.c_double),
                                         C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        R.ref_engine_heap.restype = C.c_int
        R.ref_engine_heap.argtypes = [vp, C.c_int64, C.c_int32, _u64p, _f64p, C.c_uint32,
                                      C.POINTER(C.c_uint32), C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        R.ref_engine_extract.restype = C.c_int
        R.ref_engine_extract.argtypes = [vp, C.c_int64, C.c_int32]
        R.ref_cache_new.restype = vp
        R.ref_cache_new.argtypes = [C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_uint64]
        R.ref_cache_free.argtypes = [vp]
        R.ref_cache_record_access.argtypes = [vp, _u32p, C.c_uint32]
        R.ref_cache_maybe_update.restype = C.c_uint32
        R.ref_cache_maybe_update.argtypes = [vp, C.c_double, vp, _u32p, _u8p, _f64p,
                                             C.c_uint32]
        R.ref_cache_complete_swaps.argtypes = [vp, C.c_double]
        R.ref_cache_partition.argtypes = [vp, _u32p, C.c_uint32, _u32p, C.POINTER(C.c_uint32),
                                          _u32p, C.POINTER(C.c_uint32)]
        R.ref_cache_count_hits.argtypes = [vp, _u32p, C.c_uint32]
        R.ref_cache_resident.restype = C.c_int
        R.ref_cache_resident.argtypes = [vp, C.c_uint32]
        R.ref_cache_resident_count.restype = C.c_uint64
        R.ref_cache_resident_count.argtypes = [vp]
        R.ref_cache_stats.argtypes = [vp, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64),
                                      C.POINTER(C.c_uint64)]
        R.ref_bench_execute.restype = C.c_double
        R.ref_bench_execute.argtypes = [vp, _f32p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_int,
                                        vp, vp, vp]
        _ref = R
    return _ref


# --------------------------------------------------------------------------
# numpy-level helpers over the C restatement
# --------------------------------------------------------------------------

def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class CsrIndex:
    """CSR view of an IVF index (the layout index_from_assignments builds,
    vector_index.cpp:210-235): list c owns rows [off[c], off[c+1])."""

    def __init__(self, centroids, off, vectors, ids, metric=0, mean_assigned=0.0):
        self.centroids = _f32(centroids)
        self.off = np.ascontiguousarray(off, dtype=np.uint64)
        self.vectors = _f32(vectors)
        self.ids = np.ascontiguousarray(ids, dtype=np.uint64)
        self.metric = int(metric)
        self.dim = int(self.centroids.shape[1])
        self.k_clusters = int(self.centroids.shape[0])
        self.mean_assigned = mean_assigned

    @staticmethod
    def from_assignments(corpus, ids, centroids, assign, metric=0):
        """index_from_assignments restated (vector_index.cpp:210-235): rows keep
        corpus order within each list."""
        corpus = _f32(corpus)
        assign = np.asarray(assign, dtype=np.int64)
        K = int(np.asarray(centroids).shape[0])
        order = np.argsort(assign, kind="stable")
        counts = np.bincount(assign, minlength=K)
        off = np.zeros(K + 1, dtype=np.uint64)
        off[1:] = np.cumsum(counts)
        return CsrIndex(centroids, off, corpus[order], np.asarray(ids, dtype=np.uint64)[order],
                        metric)

    def search(self, queries, nprobe, k):
        q = _f32(queries).reshape(-1, self.dim)
        B = q.shape[0]
        ids = np.zeros(B * k, np.uint64)
        d = np.zeros(B * k, np.float64)
        cnt = np.zeros(B, np.uint32)
        rc = lib().orc_ivf_search(self.centroids, self.k_clusters, self.dim, self.metric,
                                  self.vectors, self.ids, self.off, q, B, nprobe, k, ids, d, cnt)
        if rc != 0:
            raise ValueError("orc_ivf_search: invalid argument")
        return ids.reshape(B, k), d.reshape(B, k), cnt

    def select_clusters(self, query, nprobe, with_dists=False):
        plan = np.zeros(nprobe, np.uint32)
        dists = np.zeros(nprobe, np.float64)
        rc = lib().orc_select_clusters(self.centroids, self.k_clusters, self.dim, self.metric,
                                       _f32(query), nprobe, plan,
                                       dists.ctypes.data if with_dists else None)
        if rc != 0:
            raise ValueError("select_clusters: nprobe out of range")
        return (plan, dists) if with_dists else plan

    def assign(self, queries, nprobe):
        q = _f32(queries).reshape(-1, self.dim)
        plans = np.zeros((q.shape[0], nprobe), np.uint32)
        dists = np.zeros((q.shape[0], nprobe), np.float64)
        for b in range(q.shape[0]):
            plans[b], dists[b] = self.select_clusters(q[b], nprobe, True)
        return plans, dists


def squared_l2(a, b) -> float:
    a = _f32(a)
    return lib().orc_squared_l2(a, _f32(b), a.size)


def normalized(v):
    v = _f32(v)
    out = np.empty_like(v)
    lib().orc_normalized(v, v.size, out)
    return out


def brute_force(corpus, ids, query, k, metric=0):
    corpus = _f32(corpus)
    n, dim = corpus.shape
    oi = np.zeros(k, np.uint64)
    od = np.zeros(k, np.float64)
    m = lib().orc_brute_force(corpus, np.ascontiguousarray(ids, np.uint64), n, dim, metric,
                              _f32(query), k, oi, od)
    return oi[:m], od[:m]


def compute_assignments(corpus, centroids):
    corpus = _f32(corpus)
    c = _f32(centroids)
    out = np.zeros(corpus.shape[0], np.uint32)
    lib().orc_compute_assignments(corpus, corpus.shape[0], corpus.shape[1], c, c.shape[0], out)
    return out


class TopK:
    """TopKResult restated through orc_topk_insert (vector_index.cpp:38-53)."""

    def __init__(self, k):
        self.k = k
        self.buf = (OrcEntry * (k + 1))()
        self.n = C.c_uint64(0)

    def insert(self, doc_id, d) -> bool:
        return bool(lib().orc_topk_insert(self.buf, C.byref(self.n), self.k, int(doc_id),
                                          float(d)))

    def entries(self):
        return [(self.buf[i].id, self.buf[i].d) for i in range(self.n.value)]


def merge_topk(a, b, k):
    """merge_topk (vector_index.cpp:71-91) on lists of (id, d)."""
    A = (OrcEntry * max(1, len(a)))(*[OrcEntry(i, d) for i, d in a])
    Bb = (OrcEntry * max(1, len(b)))(*[OrcEntry(i, d) for i, d in b])
    out = (OrcEntry * (k + 1))()
    n = lib().orc_merge_topk(A, len(a), Bb, len(b), k, out)
    return [(out[i].id, out[i].d) for i in range(n)]


def search_clusters(index: CsrIndex, query, plan, next_pos, heap: TopK, clusters):
    """search_clusters (vector_index.cpp:291-317) with per-cluster changed flags."""
    clusters = np.ascontiguousarray(clusters, np.uint32)
    plan = np.ascontiguousarray(plan, np.uint32)
    changed = np.zeros(max(1, len(clusters)), np.uint8)
    npos = C.c_uint32(next_pos)
    rc = lib().orc_search_clusters(index.vectors, index.ids, index.off, index.dim, _f32(query),
                                   plan, len(plan), C.byref(npos), heap.buf, C.byref(heap.n),
                                   heap.k, clusters, len(clusters), changed)
    if rc != 0:
        raise RuntimeError("search_clusters: cluster does not match plan order")
    return npos.value, changed[: len(clusters)].astype(bool)


# --------------------------------------------------------------------------
# the reference itself (oracle/_ref) -- numpy helpers
# --------------------------------------------------------------------------

class RefIndex:
    """An ivf::IvfIndex built by the reference's own code."""

    def __init__(self, handle, dim, k_clusters):
        if not handle:
            raise ValueError("reference index build failed (invalid argument)")
        self.h = handle
        self.dim = dim
        self.k_clusters = k_clusters

    @staticmethod
    def build(corpus, ids, centroids, metric=0):
        corpus = _f32(corpus)
        c = _f32(centroids)
        h = ref().ref_index_build(corpus, np.ascontiguousarray(ids, np.uint64), corpus.shape[0],
                                  corpus.shape[1], metric, c, c.shape[0])
        return RefIndex(h, corpus.shape[1], c.shape[0])

    @staticmethod
    def from_assignments(corpus, ids, centroids, assign, metric=0):
        corpus = _f32(corpus)
        c = _f32(centroids)
        h = ref().ref_index_from_assign(corpus, np.ascontiguousarray(ids, np.uint64),
                                        corpus.shape[0], corpus.shape[1], metric, c, c.shape[0],
                                        np.ascontiguousarray(assign, np.uint32))
        return RefIndex(h, corpus.shape[1], c.shape[0])

    @staticmethod
    def from_csr(centroids, off, vectors, ids, metric=0):
        """The index index_from_assignments builds for these CSR lists (search
        fields only; see ref_shim.cpp ref_index_from_csr)."""
        c = _f32(centroids)
        off = np.ascontiguousarray(off, np.uint64)
        vectors = _f32(vectors)
        h = ref().ref_index_from_csr(c, c.shape[0], c.shape[1], metric, off, vectors,
                                     np.ascontiguousarray(ids, np.uint64))
        return RefIndex(h, c.shape[1], c.shape[0])

    def __del__(self):
        try:
            if self.h:
                ref().ref_index_free(self.h)
        except Exception:
            pass

    def export(self, centroids, metric=0) -> CsrIndex:
        total = ref().ref_index_total(self.h)
        off = np.zeros(self.k_clusters + 1, np.uint64)
        vec = np.zeros((total, self.dim), np.float32)
        ids = np.zeros(total, np.uint64)
        mad = C.c_double()
        ref().ref_index_export(self.h, off, vec.ctypes.data, ids.ctypes.data, C.byref(mad))
        return CsrIndex(centroids, off, vec, ids, metric, mad.value)

    def search(self, queries, nprobe, k):
        q = _f32(queries).reshape(-1, self.dim)
        B = q.shape[0]
        ids = np.zeros(B * k, np.uint64)
        d = np.zeros(B * k, np.float64)
        cnt = np.zeros(B, np.uint32)
        if ref().ref_search(self.h, q, B, nprobe, k, ids, d, cnt) != 0:
            raise ValueError("ref_search failed")
        return ids.reshape(B, k), d.reshape(B, k), cnt

    def select_clusters(self, query, nprobe):
        plan = np.zeros(nprobe, np.uint32)
        if ref().ref_select_clusters(self.h, _f32(query), nprobe, plan) != 0:
            raise ValueError("select_clusters: invalid argument")
        return plan

    def bench_execute(self, queries, nprobe, k, live=True):
        q = _f32(queries).reshape(-1, self.dim)
        B = q.shape[0]
        ids = np.zeros(B * k, np.uint64)
        d = np.zeros(B * k, np.float64)
        cnt = np.zeros(B, np.uint32)
        ms = ref().ref_bench_execute(self.h, q, B, nprobe, k, 1 if live else 0, ids.ctypes.data,
                                     d.ctypes.data, cnt.ctypes.data)
        return ms, ids.reshape(B, k), d.reshape(B, k), cnt


def ref_train_kmeans(corpus, k_clusters, iters, seed):
    corpus = _f32(corpus)
    out = np.zeros((k_clusters, corpus.shape[1]), np.float32)
    if ref().ref_train_kmeans(corpus, corpus.shape[0], corpus.shape[1], k_clusters, iters, seed,
                              out) != 0:
        raise ValueError("train_kmeans: invalid argument")
    return out


class RefEngine:
    """ret::RetrievalEngine (retrieval_engine.hpp:80-110) built by the reference's
    own code over a RefIndex; used as the CPU arm of the node-split stream bench
    (config 5) and its parity check."""

    def __init__(self, index: "RefIndex", per_vector_ns=1.0, fast_speedup=8.0, fixed_call_us=0.0,
                 capacity_gc=0, update_interval=50, bw_gb_s=16.0, decay=0.5, min_fast=2):
        self.index = index  # keeps the IvfIndex alive (the engine borrows it)
        self.h = ref().ref_engine_new(index.h, per_vector_ns, fast_speedup, fixed_call_us,
                                      capacity_gc, update_interval, bw_gb_s, decay, min_fast)

    def __del__(self):
        try:
            if self.h:
                ref().ref_engine_free(self.h)
        except Exception:
            pass

    def submit(self, req, node, query, nprobe, k):
        """make_cursor + submit (scheduler.cpp:920-944); returns the plan."""
        if ref().ref_engine_submit(self.h, req, node, _f32(query), nprobe, k, None, None, 0,
                                   None) != 0:
            raise ValueError("submit failed")
        plan = np.zeros(nprobe, np.uint32)
        n = C.c_uint32()
        ref().ref_engine_plan(self.h, req, node, plan, C.byref(n))
        return plan[: n.value]

    def execute(self, reqs, nodes, item_off, clusters, live=True):
        """One SubStageBatch; returns (heap_changed, completed) per item."""
        n = len(reqs)
        hc = np.zeros(max(1, n), np.uint8)
        done = np.zeros(max(1, n), np.uint8)
        wall, mod = C.c_double(), C.c_double()
        fa, sl = C.c_uint64(), C.c_uint64()
        rc = ref().ref_engine_execute(self.h, n, np.ascontiguousarray(reqs, np.int64),
                                      np.ascontiguousarray(nodes, np.int32),
                                      np.ascontiguousarray(item_off, np.uint32),
                                      np.ascontiguousarray(clusters, np.uint32), 0.0,
                                      1 if live else 0, hc, done, C.byref(wall), C.byref(mod),
                                      C.byref(fa), C.byref(sl))
        if rc != 0:
            raise RuntimeError("execute failed")
        return hc[:n].astype(bool), done[:n].astype(bool)

    def heap(self, req, node, cap=64):
        ids = np.zeros(cap, np.uint64)
        d = np.zeros(cap, np.float64)
        n = C.c_uint32()
        st, npos, srch = C.c_uint64(), C.c_uint64(), C.c_uint64()
        if ref().ref_engine_heap(self.h, req, node, ids, d, cap, C.byref(n), C.byref(st),
                                 C.byref(npos), C.byref(srch)) != 0:
            raise KeyError((req, node))
        return ids[: n.value], d[: n.value], int(st.value)

    def extract(self, req, node):
        ref().ref_engine_extract(self.h, req, node)
