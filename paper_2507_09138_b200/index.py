"""Python front-end over the C-ABI (bench / tests / torch interop).

Mirrors the reference's retrieval API names where they exist
(/root/reference/proj/include/hedra/vector_index.hpp): ``select_clusters``,
``search`` (make_cursor + search_step over the full plan), ``scan_items``
(search_clusters for many cursors).  All compute goes through libhivf.so.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import Stats, check, lib

METRIC_L2, METRIC_COSINE = 0, 1


def _ptr(a) -> int:
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return a.data_ptr()  # torch tensor


class Context:
    """Owns a device + stream (hivf_ctx)."""

    def __init__(self, device: int = 0, stream=None):
        """stream: None -> the context owns a non-blocking stream; a torch
        stream (or raw handle) -> all work is issued on it.  torch's default
        stream has handle 0, which the C-ABI reads as "create one", so it is
        passed as cudaStreamLegacy (0x1)."""
        h = C.c_void_p()
        s = None
        if stream is not None:
            s = stream if isinstance(stream, int) else stream.cuda_stream
            if s == 0:
                s = 1  # cudaStreamLegacy
        check(lib().hivf_ctx_create(device, s, C.byref(h)))
        self.h = h
        self.device = device

    def set_stream(self, stream):
        s = stream if (stream is None or isinstance(stream, int)) else stream.cuda_stream
        if s == 0:
            s = 1  # cudaStreamLegacy
        check(lib().hivf_ctx_set_stream(self.h, s))

    def synchronize(self):
        check(lib().hivf_ctx_synchronize(self.h))

    def device_info(self) -> dict:
        sm, conv = C.c_int(), C.c_int()
        check(lib().hivf_device_info(self.h, C.byref(sm), C.byref(conv)))
        return {"sm_count": sm.value, "tc_tf32_conversion": ["truncate", "rne", "unknown"][conv.value]
                if 0 <= conv.value <= 2 else "unknown"}

    def set_option(self, name: str, value: int):
        check(lib().hivf_set_option(self.h, name.encode(), int(value)))

    def stats(self) -> dict:
        s = Stats()
        check(lib().hivf_last_stats(self.h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in Stats._fields_}

    def merge_parts_device(self, n_parts, n_queries, k, ids, dists, counts, ids_out, dists_out,
                           counts_out):
        """merge_topk of per-shard lists on device (torch tensors)."""
        check(lib().hivf_merge_parts_device(self.h, n_parts, n_queries, k, _ptr(ids), _ptr(dists),
                                            _ptr(counts), _ptr(ids_out), _ptr(dists_out),
                                            _ptr(counts_out)))

    def compute_assignments(self, d_corpus, d_centroids, d_assign_out):
        """ivf::compute_assignments (vector_index.cpp:202-208) on device tensors:
        corpus [n, dim] f32, centroids [K, dim] f32 -> assign [n] int32."""
        n, dim = d_corpus.shape
        check(lib().hivf_compute_assignments(self.h, _ptr(d_corpus), n, dim, _ptr(d_centroids),
                                             d_centroids.shape[0], _ptr(d_assign_out)))

    def train_kmeans(self, d_corpus, k_clusters, max_iters, seed, d_centroids_out):
        """ivf::train_kmeans (vector_index.cpp:99-200), bit-identical centroids."""
        n, dim = d_corpus.shape
        check(lib().hivf_train_kmeans(self.h, _ptr(d_corpus), n, dim, k_clusters, max_iters, seed,
                                      _ptr(d_centroids_out)))

    def train_kmeans_sampled_seeds(self, d_corpus, k_clusters, max_iters, seed, d_centroids_out):
        """Parallel training mode (hivf_train_kmeans_sampled_seeds): Lloyd from
        K distinct corpus rows instead of k-means++."""
        n, dim = d_corpus.shape
        check(lib().hivf_train_kmeans_sampled_seeds(self.h, _ptr(d_corpus), n, dim, k_clusters, max_iters,
                                                    seed, _ptr(d_centroids_out)))

    def close(self):
        if getattr(self, "h", None):
            lib().hivf_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class IvfIndex:
    """An IVF index resident in HBM (hivf_index)."""

    def __init__(self, ctx: Context, handle, dim, k_clusters, metric):
        self.ctx = ctx
        self.h = handle
        self.dim = dim
        self.k_clusters = k_clusters
        self.metric = metric

    # ---- construction ---------------------------------------------------
    @staticmethod
    def upload(ctx: Context, centroids, list_offsets, vectors, ids, metric=METRIC_L2):
        """index_from_assignments-shaped CSR (host numpy arrays) -> HBM."""
        cents = np.ascontiguousarray(centroids, np.float32)
        off = np.ascontiguousarray(list_offsets, np.uint64)
        vec = np.ascontiguousarray(vectors, np.float32)
        ids = np.ascontiguousarray(ids, np.uint64)
        K, dim = cents.shape
        h = C.c_void_p()
        check(lib().hivf_index_upload(ctx.h, dim, metric, K, cents.ctypes.data, off.ctypes.data,
                                      vec.ctypes.data if vec.size else None,
                                      ids.ctypes.data if ids.size else None, C.byref(h)))
        return IvfIndex(ctx, h, dim, K, metric)

    @staticmethod
    def from_assignments(ctx: Context, corpus, ids, centroids, assign, metric=METRIC_L2):
        """ivf::index_from_assignments (vector_index.cpp:210-235): stable
        grouping of corpus rows by assigned cluster."""
        assign = np.asarray(assign, np.int64)
        K = np.asarray(centroids).shape[0]
        order = np.argsort(assign, kind="stable")
        off = np.zeros(K + 1, np.uint64)
        off[1:] = np.cumsum(np.bincount(assign, minlength=K))
        corpus = np.asarray(corpus, np.float32)
        return IvfIndex.upload(ctx, centroids, off, corpus[order], np.asarray(ids, np.uint64)[order],
                               metric)

    @staticmethod
    def build_device(ctx: Context, centroids, list_offsets, metric, n_rows, row_source,
                     chunk_rows=1 << 20):
        """Incremental HBM build: row_source(first, n) -> (float32 [n,dim], uint64 [n]) torch
        CUDA tensors holding rows [first, first+n) in list order."""
        import torch
        cents = centroids
        dev = isinstance(cents, torch.Tensor) and cents.is_cuda
        if not dev:
            cents = np.ascontiguousarray(cents, np.float32)
        K, dim = cents.shape
        off = np.ascontiguousarray(list_offsets, np.uint64)
        h = C.c_void_p()
        check(lib().hivf_index_begin(ctx.h, dim, metric, K, _ptr(cents), 1 if dev else 0,
                                     off.ctypes.data, C.byref(h)))
        ix = IvfIndex(ctx, h, dim, K, metric)
        for first in range(0, int(n_rows), chunk_rows):
            n = min(chunk_rows, int(n_rows) - first)
            rows, rid = row_source(first, n)
            check(lib().hivf_index_add_rows_device(h, first, n, rows.data_ptr(), rid.data_ptr()))
            ctx.synchronize()
            del rows, rid
        check(lib().hivf_index_finish(h))
        return ix

    @staticmethod
    def build_scatter(ctx: Context, centroids, list_offsets, metric, n_rows, chunks):
        """Incremental HBM build from corpus-order chunks: ``chunks`` yields
        (positions uint64 [n], rows float32 [n,dim], ids uint64 [n]) torch CUDA
        tensors; positions are list-order row indices (index_from_assignments
        order)."""
        import torch
        cents = centroids
        dev = isinstance(cents, torch.Tensor) and cents.is_cuda
        if not dev:
            cents = np.ascontiguousarray(cents, np.float32)
        K, dim = cents.shape
        off = np.ascontiguousarray(list_offsets, np.uint64)
        h = C.c_void_p()
        check(lib().hivf_index_begin(ctx.h, dim, metric, K, _ptr(cents), 1 if dev else 0,
                                     off.ctypes.data, C.byref(h)))
        ix = IvfIndex(ctx, h, dim, K, metric)
        for pos, rows, rid in chunks:
            check(lib().hivf_index_add_rows_at_device(h, pos.shape[0], pos.data_ptr(),
                                                      rows.data_ptr(), rid.data_ptr()))
            ctx.synchronize()
        check(lib().hivf_index_finish(h))
        return ix

    def get_rows(self, first, n):
        """Rows [first, first+n) in list order (row-major float32) + doc ids."""
        rows = np.zeros((n, self.dim), np.float32)
        ids = np.zeros(n, np.uint64)
        check(lib().hivf_index_get_rows(self.h, first, n, rows.ctypes.data, ids.ctypes.data))
        return rows, ids

    def get_rows_into(self, first, n, rows_out, ids_out):
        """get_rows into caller arrays (C-contiguous float32 [n,dim] / uint64 [n] views)."""
        assert rows_out.flags.c_contiguous and ids_out.flags.c_contiguous
        assert rows_out.dtype == np.float32 and ids_out.dtype == np.uint64
        check(lib().hivf_index_get_rows(self.h, first, n, rows_out.ctypes.data, ids_out.ctypes.data))

    def close(self):
        # an index must not outlive its context (the C-ABI contract); if the
        # context was closed first, the device memory went with it.
        if getattr(self, "h", None) and getattr(self.ctx, "h", None):
            lib().hivf_index_destroy(self.h)
        self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- introspection ----------------------------------------------------
    def info(self) -> dict:
        d, k, hb = C.c_uint32(), C.c_uint32(), C.c_uint64()
        n = C.c_uint64()
        check(lib().hivf_index_info(self.h, C.byref(d), C.byref(k), C.byref(n), C.byref(hb), None))
        return {"dim": d.value, "k_clusters": k.value, "n_vectors": n.value, "hbm_bytes": hb.value}

    def mean_assigned_distance(self) -> float:
        m = C.c_double()
        check(lib().hivf_index_info(self.h, None, None, None, None, C.byref(m)))
        return m.value

    def cluster_sizes(self) -> np.ndarray:
        out = np.zeros(self.k_clusters, np.uint64)
        check(lib().hivf_index_cluster_sizes(self.h, out.ctypes.data))
        return out

    # ---- hot path -----------------------------------------------------------
    def select_clusters(self, queries, nprobe, with_dists=False):
        """Batched ivf::select_clusters (vector_index.cpp:261-278)."""
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, self.dim)
        B = q.shape[0]
        plans = np.zeros((B, nprobe), np.uint32)
        dists = np.zeros((B, nprobe), np.float64)
        check(lib().hivf_assign(self.h, q.ctypes.data, B, nprobe, plans.ctypes.data,
                                dists.ctypes.data))
        return (plans, dists) if with_dists else plans

    def search(self, queries, nprobe, k):
        """make_cursor + search_step(full plan) per query; host buffers."""
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, self.dim)
        B = q.shape[0]
        ids = np.zeros((B, k), np.uint64)
        d = np.zeros((B, k), np.float64)
        cnt = np.zeros(B, np.uint32)
        check(lib().hivf_search(self.h, q.ctypes.data, B, nprobe, k, ids.ctypes.data, d.ctypes.data,
                                cnt.ctypes.data))
        return ids, d, cnt

    def search_device(self, d_queries, nprobe, k, ids_out, dists_out, counts_out):
        """Same on HBM-resident torch tensors, async on the context stream."""
        B = d_queries.shape[0]
        check(lib().hivf_search_device(self.h, d_queries.data_ptr(), B, nprobe, k,
                                       ids_out.data_ptr(), dists_out.data_ptr(),
                                       counts_out.data_ptr()))

    def assign_device(self, d_queries, nprobe, plans_out, dists_out=None):
        """select_clusters for a batch of HBM-resident queries (plans_out: int32
        [B, nprobe] tensor on the device), async on the context stream."""
        B = d_queries.shape[0]
        check(lib().hivf_assign_device(self.h, d_queries.data_ptr(), B, nprobe, plans_out.data_ptr(),
                                       dists_out.data_ptr() if dists_out is not None else None))

    def search_planned_device(self, d_queries, nprobe, k, plans, ids_out, dists_out, counts_out):
        """search_device with caller-supplied plans (e.g. all-gathered from the
        ranks that assigned slices of the batch)."""
        B = d_queries.shape[0]
        check(lib().hivf_search_planned_device(self.h, d_queries.data_ptr(), B, nprobe, k,
                                               plans.data_ptr(), ids_out.data_ptr(),
                                               dists_out.data_ptr(), counts_out.data_ptr()))

    def scan_items(self, queries, cluster_off, clusters, k, heap_ids, heap_dists, heap_counts):
        """search_clusters for many cursors (vector_index.cpp:291-317); heaps
        updated in place; returns per-cluster changed flags."""
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, self.dim)
        n = q.shape[0]
        off = np.ascontiguousarray(cluster_off, np.uint32)
        cl = np.ascontiguousarray(clusters, np.uint32)
        kv = np.ascontiguousarray(k, np.uint32)
        assert heap_ids.dtype == np.uint64 and heap_dists.dtype == np.float64
        assert heap_counts.dtype == np.uint32 and heap_ids.flags.c_contiguous
        stride = heap_ids.shape[1]
        changed = np.zeros(max(1, len(cl)), np.uint8)
        check(lib().hivf_scan_items(self.h, q.ctypes.data, n, off.ctypes.data,
                                    cl.ctypes.data if len(cl) else None, kv.ctypes.data,
                                    heap_ids.ctypes.data, heap_dists.ctypes.data,
                                    heap_counts.ctypes.data, stride, changed.ctypes.data))
        return changed[: len(cl)].astype(bool)

    def set_residency(self, clusters):
        cl = np.ascontiguousarray(clusters, np.uint32)
        check(lib().hivf_residency_set(self.h, cl.ctypes.data if len(cl) else None, len(cl)))

    def residency_sync(self):
        check(lib().hivf_residency_sync(self.h))

    def residency(self) -> np.ndarray:
        out = np.zeros(self.k_clusters, np.uint8)
        check(lib().hivf_residency_get(self.h, out.ctypes.data))
        return out.astype(bool)


# ---------------------------------------------------------------------------
# multi-GPU list sharding (include/hivf.h "multi-GPU list sharding")
# ---------------------------------------------------------------------------

def shard_plan(sizes, nranks, weights=None, n_striped=-1) -> np.ndarray:
    """owner[c] = rank holding list c, or SHARD_STRIPED (rows split over all
    ranks); frequency-weighted LPT (hivf_shard_plan)."""
    sz = np.ascontiguousarray(sizes, np.uint64)
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    owner = np.zeros(len(sz), np.uint32)
    check(lib().hivf_shard_plan(sz.ctypes.data, None if w is None else w.ctypes.data, len(sz), nranks,
                                int(n_striped), owner.ctypes.data))
    return owner


def shard_local_lists(list_offsets, owner, nranks, rank):
    """(local_offsets [K+1], src_first [K]): rank's list c holds the global
    list-order rows [src_first[c], src_first[c] + local size)."""
    off = np.ascontiguousarray(list_offsets, np.uint64)
    ow = np.ascontiguousarray(owner, np.uint32)
    K = len(ow)
    loc = np.zeros(K + 1, np.uint64)
    first = np.zeros(K, np.uint64)
    check(lib().hivf_shard_local_lists(off.ctypes.data, ow.ctypes.data, K, nranks, rank, loc.ctypes.data,
                                       first.ctypes.data))
    return loc, first


def upload_shard(ctx: Context, centroids, list_offsets, vectors, ids, owner, nranks, rank,
                 metric=METRIC_L2) -> IvfIndex:
    """Rank `rank`'s shard of a host CSR index (hivf_index_upload_shard)."""
    cents = np.ascontiguousarray(centroids, np.float32)
    off = np.ascontiguousarray(list_offsets, np.uint64)
    vec = np.ascontiguousarray(vectors, np.float32)
    ids = np.ascontiguousarray(ids, np.uint64)
    ow = np.ascontiguousarray(owner, np.uint32)
    K, dim = cents.shape
    h = C.c_void_p()
    check(lib().hivf_index_upload_shard(ctx.h, dim, metric, K, cents.ctypes.data, off.ctypes.data,
                                        vec.ctypes.data if vec.size else None,
                                        ids.ctypes.data if ids.size else None, ow.ctypes.data, nranks, rank,
                                        C.byref(h)))
    return IvfIndex(ctx, h, dim, K, metric)


def nccl_unique_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    check(lib().hivf_nccl_unique_id(buf))
    return bytes(buf)


class ShardGroup:
    """Shards of one logical index searched as one (hivf_group): per batch a
    slice assign per rank, plan all-gather, local exact search, result
    exchange and device merge_topk."""

    def __init__(self, handle, shards, keep=None):
        self.h = handle
        self.shards = shards
        self._keep = keep  # ctypes callback / buffers the C side refers to

    @staticmethod
    def in_process(shards):
        """One host thread drives every shard (one context each)."""
        arr = (C.c_void_p * len(shards))(*[s.h.value for s in shards])
        h = C.c_void_p()
        check(lib().hivf_group_create(arr, len(shards), C.byref(h)))
        return ShardGroup(h, list(shards))

    @staticmethod
    def nccl(shard, nranks, rank, unique_id: bytes):
        buf = (C.c_uint8 * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        check(lib().hivf_group_create_nccl(shard.h, nranks, rank, buf, C.byref(h)))
        return ShardGroup(h, [shard])

    @staticmethod
    def host_allgather(shard, nranks, rank, allgather):
        """allgather(send: bytes) -> bytes of nranks blocks in rank order."""
        from ._lib import ALLGATHER_FN

        def cb(user, send, nbytes, recv):
            try:
                out = allgather(C.string_at(send, nbytes))
                assert len(out) == nbytes * nranks
                C.memmove(recv, out, len(out))
                return 0
            except Exception:  # reported as HIVF_ECOMM
                import traceback
                traceback.print_exc()
                return 1

        fn = ALLGATHER_FN(cb)
        h = C.c_void_p()
        check(lib().hivf_group_create_hostcb(shard.h, nranks, rank, fn, None, C.byref(h)))
        return ShardGroup(h, [shard], keep=fn)

    def search(self, queries, nprobe, k):
        dim = self.shards[0].dim
        q = np.ascontiguousarray(queries, np.float32).reshape(-1, dim)
        B = q.shape[0]
        ids = np.zeros((B, k), np.uint64)
        d = np.zeros((B, k), np.float64)
        cnt = np.zeros(B, np.uint32)
        check(lib().hivf_group_search(self.h, q.ctypes.data, B, nprobe, k, ids.ctypes.data, d.ctypes.data,
                                      cnt.ctypes.data))
        return ids, d, cnt

    def search_device(self, d_queries, nprobe, k, ids_out, dists_out, counts_out):
        check(lib().hivf_group_search_device(self.h, d_queries.data_ptr(), d_queries.shape[0], nprobe, k,
                                             ids_out.data_ptr(), dists_out.data_ptr(), counts_out.data_ptr()))

    def close(self):
        if getattr(self, "h", None):
            lib().hivf_group_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
