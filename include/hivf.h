/*
 * hivf.h -- C-ABI of the B200-native IVF retrieval hot path
 *           (HedraRAG, arXiv 2507.09138: coarse assign -> list scan -> top-k).
 *
 * Plain C: pointers, sizes and status codes only (no C++ types, no torch types,
 * no exceptions cross this boundary).  Every entry point names the reference
 * interface it replaces; reference paths are relative to /root/reference/.
 *
 * Error mapping (reference exceptions -> status):
 *   std::invalid_argument  -> HIVF_EINVAL    (caller misuse: nprobe/k out of range,
 *                                             dim mismatch, duplicate doc id, ...)
 *   std::runtime_error     -> HIVF_EINTERNAL (cluster out of plan order, cursor
 *                                             exhausted mid-batch, ...)
 *   plus HIVF_ECUDA / HIVF_ENOMEM / HIVF_EUNSUPPORTED for the device side.
 * hivf_last_error() returns a thread-local message for the last failure.
 *
 * Threading: an hivf_ctx has one owning host thread at a time (the reference's
 * single retrieval-worker context, proj/include/hedra/retrieval_engine.hpp:76-79).
 * All device work is issued on the context's stream.
 *
 * Arithmetic contract: every distance returned is the bit-exact double the
 * reference computes (proj/include/hedra/embedding.hpp:27-34); ids and plan
 * orders follow the reference's (distance, id) total order
 * (proj/include/hedra/vector_index.hpp:41-44).
 *
 * Argument range: any nprobe in [1, K] (vector_index.cpp:264-265; plans longer
 * than 4096 take an exact all-centroid select and the exact scan), any k in
 * [1, 4096].  Deviations from the reference, all reported, never silent:
 *   - k > 4096                 -> HIVF_EUNSUPPORTED (the reference has no bound)
 *   - non-finite query / corpus / centroid values -> HIVF_EINVAL.  The
 *     reference never checks (check_finite, embedding.hpp:45-49, is unused)
 *     and its NaN comparisons then give an order that depends on the scan
 *     order; the filter bounds here need finite operands, so they are rejected.
 *   - duplicate doc ids in an uploaded index -> HIVF_EINVAL.  build_index
 *     rejects them too (vector_index.cpp:240-244); index_from_assignments and
 *     brute_force_search do not, the device layout's id uniqueness needs it.
 *   - shard groups: nranks * k <= 8192 (the on-device merge buffer).
 */
#ifndef HIVF_H_
#define HIVF_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  HIVF_OK = 0,
  HIVF_EINVAL = 1,
  HIVF_EINTERNAL = 2,
  HIVF_ECUDA = 3,
  HIVF_ENOMEM = 4,
  HIVF_EUNSUPPORTED = 5,
  HIVF_ECOMM = 6  /* multi-GPU exchange failed (NCCL error, all-gather callback error) */
} hivf_status;

/* Metric ids match hedra::Metric (proj/include/hedra/embedding.hpp:14). */
enum { HIVF_METRIC_L2 = 0, HIVF_METRIC_COSINE = 1 };

typedef struct hivf_ctx hivf_ctx;
typedef struct hivf_index hivf_index;

/* Thread-local description of the most recent failure ("" if none). */
const char* hivf_last_error(void);
const char* hivf_version(void);

/* ---- context --------------------------------------------------------------
 * Owns the device, the stream and per-call scratch.  Replaces the retrieval
 * worker context that owns a RetrievalEngine
 * (proj/include/hedra/retrieval_engine.hpp:80-84).  `stream` may be NULL
 * (the context creates its own) or a cudaStream_t the caller owns. */
hivf_status hivf_ctx_create(int device, void* stream, hivf_ctx** out);
hivf_status hivf_ctx_destroy(hivf_ctx* ctx);
hivf_status hivf_ctx_set_stream(hivf_ctx* ctx, void* stream);
hivf_status hivf_ctx_synchronize(hivf_ctx* ctx);
/* SM count and the tensor core's fp32->tf32 operand conversion as probed on
 * this device at first context creation (0 truncation, 1 round-to-nearest-
 * even, 2 unknown -> the FFMA scan is used). */
hivf_status hivf_device_info(hivf_ctx* ctx, int* sm_count, int* tc_tf32_conversion);

/* ---- index ----------------------------------------------------------------
 * Replaces ivf::index_from_assignments (proj/src/vector_index.cpp:210-235) and
 * the IvfIndex it returns (proj/include/hedra/vector_index.hpp:83-113): the
 * caller passes the lists in CSR form (list c owns rows
 * [list_offsets[c], list_offsets[c+1]) of vectors/ids, row-major, list order
 * as index_from_assignments leaves it).  Vectors must already be in search
 * space (normalized for cosine, as build_index does at :245-252).  The
 * library copies everything into HBM (chunk-major 16B-aligned list layout,
 * see DESIGN.md); the caller keeps ownership of its arrays.
 * EINVAL: dim == 0, n_clusters == 0, offsets not monotone, duplicate doc ids
 * (build_index, :240-244), non-finite values. */
hivf_status hivf_index_upload(hivf_ctx* ctx, uint32_t dim, int metric, uint32_t n_clusters,
                              const float* centroids, const uint64_t* list_offsets,
                              const float* vectors, const uint64_t* ids, hivf_index** out);
/* Same, with `vectors`/`ids`/`centroids` in device memory (list_offsets on host).
 * Used to build large indexes directly in HBM. */
hivf_status hivf_index_upload_device(hivf_ctx* ctx, uint32_t dim, int metric,
                                     uint32_t n_clusters, const float* d_centroids,
                                     const uint64_t* list_offsets, const float* d_vectors,
                                     const uint64_t* d_ids, hivf_index** out);
/* Incremental build for indexes too large to stage twice (the same packing,
 * fed in row chunks of the list-ordered CSR): begin (centroids on host or
 * device per `centroids_on_device`, offsets on host), add_rows any number of
 * times with device rows [first_row, first_row+n_rows) in list order, then
 * finish (duplicate-id / finiteness checks, EINVAL on failure). */
hivf_status hivf_index_begin(hivf_ctx* ctx, uint32_t dim, int metric, uint32_t n_clusters,
                             const float* centroids, int centroids_on_device,
                             const uint64_t* list_offsets, hivf_index** out);
hivf_status hivf_index_add_rows_device(hivf_index* idx, uint64_t first_row, uint64_t n_rows,
                                       const float* d_rows, const uint64_t* d_ids);
/* Same, rows scattered to explicit list-order positions d_positions[n_rows]
 * (index_from_assignments order: list offset + rank within the list). */
hivf_status hivf_index_add_rows_at_device(hivf_index* idx, uint64_t n_rows,
                                          const uint64_t* d_positions, const float* d_rows,
                                          const uint64_t* d_ids);
hivf_status hivf_index_finish(hivf_index* idx);
/* Read rows [first_row, first_row+n_rows) back (list order, row-major host
 * floats + doc ids); the IvfIndex::doc_embedding of vector_index.hpp:105-108. */
hivf_status hivf_index_get_rows(hivf_index* idx, uint64_t first_row, uint64_t n_rows,
                                float* rows_out, uint64_t* ids_out);
/* IvfIndex::locate / doc_embedding (vector_index.hpp:98-111; the locator map of
 * vector_index.cpp:226-227): list and list-order row of each doc id
 * (clusters_out = UINT32_MAX, rows_out = UINT64_MAX when unknown), and the
 * rows' vectors (row-major host floats).  Used by the locality helpers
 * (make_locality_record, similarity.cpp:18-33). */
hivf_status hivf_index_locate(hivf_index* idx, const uint64_t* doc_ids, uint32_t n,
                              uint32_t* clusters_out, uint64_t* rows_out);
hivf_status hivf_index_gather_rows(hivf_index* idx, const uint64_t* rows, uint32_t n,
                                   float* rows_out);
hivf_status hivf_index_destroy(hivf_index* idx);
/* k_clusters / cluster_size / total_vectors / mean_assigned_distance
 * (vector_index.hpp:92-98).  Any output pointer may be NULL. */
hivf_status hivf_index_info(const hivf_index* idx, uint32_t* dim, uint32_t* n_clusters,
                            uint64_t* n_vectors, uint64_t* hbm_bytes,
                            double* mean_assigned_distance);
hivf_status hivf_index_cluster_sizes(const hivf_index* idx, uint64_t* sizes_out);
/* The exact double squared_l2(row, its centroid) of every row, in list order
 * (host buffer of n_vectors doubles).  index_from_assignments sums these in
 * corpus order for mean_assigned_distance (vector_index.cpp:222-233); the
 * caller owns that order, so it can reproduce the reference sum bit-exactly. */
hivf_status hivf_index_row_distances(hivf_index* idx, double* dist_out);

/* ---- index build -------------------------------------------------------------
 * Replaces ivf::compute_assignments and ivf::train_kmeans
 * (proj/src/vector_index.cpp:202-208, 99-200) with the reference's exact
 * arithmetic (nearest centroid in double, ties -> lowest id; k-means++ seeding
 * with the reference's Rng stream and sequential running sums; Lloyd means
 * summed in point order in double; empty clusters re-seeded to the farthest
 * point), so the centroids / assignments are bit-identical to the reference's.
 * All arrays in device memory, row-major [n][dim] / [K][dim]; rows already in
 * search space (normalized for cosine, as build_index does at :245-252).
 * train_kmeans: EINVAL for n < K, K == 0, max_iters == 0 (:101-105).  Its
 * k-means++ seeding walks the n running sums once per seed (sequential by
 * definition), so it costs O(K n) serial adds on one thread. */
hivf_status hivf_compute_assignments(hivf_ctx* ctx, const float* d_corpus, uint64_t n, uint32_t dim,
                                     const float* d_centroids, uint32_t n_clusters,
                                     uint32_t* d_assign_out);
hivf_status hivf_train_kmeans(hivf_ctx* ctx, const float* d_corpus, uint64_t n, uint32_t dim,
                              uint32_t n_clusters, uint32_t max_iters, uint64_t seed,
                              float* d_centroids_out);
/* Parallel training mode for large K x n (the C3/C4 bench indexes): the same
 * Lloyd iterations (exact assignment, point-order double means, farthest-point
 * re-seeding of empty clusters) from K distinct corpus rows drawn with the
 * reference's Rng instead of k-means++, whose seeding is a serial chain of K
 * running sums over n points.  Deterministic for a seed, but NOT the
 * reference's train_kmeans result (different seeds); the index built from
 * these centroids with hivf_compute_assignments is still exactly the one the
 * reference's index_from_assignments builds from the same centroids. */
hivf_status hivf_train_kmeans_sampled_seeds(hivf_ctx* ctx, const float* d_corpus, uint64_t n,
                                            uint32_t dim, uint32_t n_clusters, uint32_t max_iters,
                                            uint64_t seed, float* d_centroids_out);
/* Same with host buffers (staged through HBM), as the C++ adapter calls them. */
hivf_status hivf_compute_assignments_host(hivf_ctx* ctx, const float* corpus, uint64_t n, uint32_t dim,
                                          const float* centroids, uint32_t n_clusters,
                                          uint32_t* assign_out);
hivf_status hivf_train_kmeans_host(hivf_ctx* ctx, const float* corpus, uint64_t n, uint32_t dim,
                                   uint32_t n_clusters, uint32_t max_iters, uint64_t seed,
                                   float* centroids_out);

/* ---- coarse assign --------------------------------------------------------
 * Batched ivf::select_clusters (proj/src/vector_index.cpp:261-278): for each
 * query, the nprobe nearest centroids in exact (double distance, cluster id)
 * order.  Queries are raw (normalized internally for cosine, :270).
 * plans_out[n_queries*nprobe]; dists_out (optional) gets the exact doubles.
 * EINVAL: nprobe not in [1, n_clusters] (:264). */
hivf_status hivf_assign(hivf_index* idx, const float* queries, uint32_t n_queries,
                        uint32_t nprobe, uint32_t* plans_out, double* dists_out);

/* ---- per-request search ---------------------------------------------------
 * Batched make_cursor + search_step over the full plan
 * (proj/src/vector_index.cpp:280-289,319-328, per-query top-k with the
 * TopKResult semantics of :38-53).  Host buffers: queries[n_queries*dim];
 * ids_out / dists_out [n_queries*k] (entries past counts_out[b] are zero);
 * counts_out[n_queries] = heap size (min(k, rows probed)).
 * EINVAL: k == 0 (:281), nprobe out of range. */
hivf_status hivf_search(hivf_index* idx, const float* queries, uint32_t n_queries,
                        uint32_t nprobe, uint32_t k, uint64_t* ids_out, double* dists_out,
                        uint32_t* counts_out);
/* Device-pointer variant: all buffers in HBM, asynchronous on the context
 * stream (no host synchronisation; CUDA-graph capturable after one warm call
 * with the same (n_queries, nprobe, k)). */
hivf_status hivf_search_device(hivf_index* idx, const float* d_queries, uint32_t n_queries,
                               uint32_t nprobe, uint32_t k, uint64_t* d_ids_out,
                               double* d_dists_out, uint32_t* d_counts_out);

/* Split form of the same call for multi-GPU list sharding:
 * hivf_assign_device is ivf::select_clusters for a batch (plans in HBM, the
 * same exact order as hivf_assign; each rank may assign a slice of the batch
 * and all-gather the plans), and hivf_search_planned_device runs the search
 * with those plans -- make_cursor with a given plan + search_step over it
 * (proj/src/vector_index.cpp:280-289,319-328).  Plan ids >= n_clusters are
 * replaced by 0 and reported as EINVAL by the host-buffer calls. */
hivf_status hivf_assign_device(hivf_index* idx, const float* d_queries, uint32_t n_queries,
                               uint32_t nprobe, uint32_t* d_plans_out, double* d_dists_out);
hivf_status hivf_search_planned_device(hivf_index* idx, const float* d_queries, uint32_t n_queries,
                                       uint32_t nprobe, uint32_t k, const uint32_t* d_plans,
                                       uint64_t* d_ids_out, double* d_dists_out,
                                       uint32_t* d_counts_out);

/* ---- node-split sub-search --------------------------------------------------
 * Many cursors advanced by one sub-stage: ivf::search_clusters
 * (proj/src/vector_index.cpp:291-317) for every item of a SubStageBatch, as
 * RetrievalEngine::execute runs it (proj/src/retrieval_engine.cpp:94-103).
 *   queries[n_items*dim]     the cursor query of each item, already in search
 *                            space (SearchCursor::query, vector_index.hpp:119)
 *   cluster_off[n_items+1], clusters[]  each item's clusters, in plan order
 *   k[n_items]               each cursor's heap bound (SearchCursor::k)
 *   heap_ids/heap_dists [n_items*heap_stride], heap_counts[n_items]:
 *                            the cursor heaps, read and updated in place
 *                            (entries sorted by (dist, id), size <= k)
 *   changed_out[len(clusters)] per-cluster `changed` flag (:300-313), from
 *                            which the caller derives heap_changed and
 *                            unchanged_streak exactly as the reference does.
 * Validation that clusters match plan order stays with the caller (the
 * adapter), which owns the plans (EINTERNAL there, as :295-298). */
hivf_status hivf_scan_items(hivf_index* idx, const float* queries, uint32_t n_items,
                            const uint32_t* cluster_off, const uint32_t* clusters,
                            const uint32_t* k, uint64_t* heap_ids, double* heap_dists,
                            uint32_t* heap_counts, uint32_t heap_stride,
                            uint8_t* changed_out);

/* ---- multi-GPU merge ------------------------------------------------------
 * merge_topk (proj/src/vector_index.cpp:71-91) of n_parts per-shard top-k
 * lists per query, on device: parts laid out [n_parts][n_queries][k]
 * (ids u64, dists f64, counts u32 [n_parts][n_queries]) as an all-gather
 * leaves them.  Output [n_queries][k] + counts. */
hivf_status hivf_merge_parts_device(hivf_ctx* ctx, uint32_t n_parts, uint32_t n_queries,
                                    uint32_t k, const uint64_t* d_ids, const double* d_dists,
                                    const uint32_t* d_counts, uint64_t* d_ids_out,
                                    double* d_dists_out, uint32_t* d_counts_out);

/* ---- multi-GPU list sharding -----------------
 * The reference searches one in-memory IvfIndex (vector_index.hpp:83-113); here
 * the lists of one logical index are split over GPUs and the per-GPU exact
 * top-k lists are merged with merge_topk (vector_index.cpp:71-91), so results
 * are identical to a single-GPU (or reference) search of the whole index.
 *
 * hivf_shard_plan: owner_out[c] = the rank holding list c, or
 * HIVF_SHARD_STRIPED for lists whose rows are split over all ranks (rank r
 * holds rows [n*r/N, n*(r+1)/N) of the list).  Load of a list = sizes[c] *
 * weights[c] (weights NULL = 1: bytes; pass the list's expected scan passes per
 * batch -- its probe frequency -- for skewed query streams).  The n_striped
 * heaviest lists (load desc, id asc) are striped (n_striped < 0: automatic, the
 * lists heavier than 1/16 of one rank's share), the rest go to ranks by LPT
 * (heaviest list to the least-loaded rank, ties to the lowest rank).
 * hivf_shard_local_lists: rank `rank`'s CSR -- local list c holds the global
 * list-order rows [src_first_out[c], src_first_out[c] + local size), local
 * sizes as offsets [n_clusters+1].  Every rank builds its index with ALL
 * centroids (identical on every rank) and its local lists (others empty);
 * hivf_index_upload_shard does that from host CSR arrays. */
#define HIVF_SHARD_STRIPED 0xFFFFFFFFu
hivf_status hivf_shard_plan(const uint64_t* sizes, const double* weights, uint32_t n_clusters,
                            uint32_t nranks, int32_t n_striped, uint32_t* owner_out);
hivf_status hivf_shard_local_lists(const uint64_t* list_offsets, const uint32_t* owner,
                                   uint32_t n_clusters, uint32_t nranks, uint32_t rank,
                                   uint64_t* local_offsets_out, uint64_t* src_first_out);
hivf_status hivf_index_upload_shard(hivf_ctx* ctx, uint32_t dim, int metric, uint32_t n_clusters,
                                    const float* centroids, const uint64_t* list_offsets,
                                    const float* vectors, const uint64_t* ids,
                                    const uint32_t* owner, uint32_t nranks, uint32_t rank,
                                    hivf_index** out);

/* A shard group searches the shards of one logical index as one: per batch,
 * each rank assigns a slice of the batch (select_clusters), the plans are
 * all-gathered, every rank searches its shard with the full plans, and one
 * packed ids|dists|counts block per rank is exchanged and merged on device
 * (merge_topk).  Three transports:
 *   hivf_group_create        in-process: one host thread drives n shards on n
 *                            contexts (one per GPU; several may share a
 *                            device); exchange by a gather kernel over peer
 *                            pointers (NVLink P2P), event-ordered.  Queries
 *                            and results live on shards[0]'s device/stream.
 *   hivf_group_create_nccl   one process per GPU (torchrun): ncclAllGather on
 *                            the context stream; every rank calls every group
 *                            function collectively with the same batch and
 *                            gets the merged results.  unique_id: 128 bytes
 *                            from hivf_nccl_unique_id on rank 0, broadcast by
 *                            the caller.  NCCL is loaded at run time.
 *   hivf_group_create_hostcb one process per rank, exchange through the
 *                            caller's host all-gather `fn` (recv = nranks
 *                            blocks of `bytes`, rank order; return 0 on
 *                            success) -- e.g. torch.distributed over gloo.
 * The shards must share dim / n_clusters / metric and the centroids, and hold
 * disjoint row sets (hivf_shard_local_lists).  EUNSUPPORTED: nranks*k > 8192,
 * tiered shards.  HIVF_ECOMM: NCCL / callback failure. */
typedef struct hivf_group hivf_group;
typedef int (*hivf_allgather_fn)(void* user, const void* send, size_t bytes, void* recv);
hivf_status hivf_group_create(hivf_index* const* shards, uint32_t n, hivf_group** out);
hivf_status hivf_nccl_unique_id(void* unique_id_out);
hivf_status hivf_group_create_nccl(hivf_index* shard, uint32_t nranks, uint32_t rank,
                                   const void* unique_id, hivf_group** out);
hivf_status hivf_group_create_hostcb(hivf_index* shard, uint32_t nranks, uint32_t rank,
                                     hivf_allgather_fn fn, void* user, hivf_group** out);
hivf_status hivf_group_destroy(hivf_group* g);
/* The sharded hivf_search_device / hivf_search (same arguments and errors). */
hivf_status hivf_group_search_device(hivf_group* g, const float* d_queries, uint32_t n_queries,
                                     uint32_t nprobe, uint32_t k, uint64_t* d_ids_out,
                                     double* d_dists_out, uint32_t* d_counts_out);
hivf_status hivf_group_search(hivf_group* g, const float* queries, uint32_t n_queries,
                              uint32_t nprobe, uint32_t k, uint64_t* ids_out, double* dists_out,
                              uint32_t* counts_out);

/* ---- hot-cluster residency set ---------------------------------------------
 * Device side of cache::ClusterCacheState (proj/include/hedra/tiered_cache.hpp
 * :37-78; the host adapter keeps the reference's counters and target choice).
 * With option "hbm_list_budget" (bytes, set on the context before the index
 * is built) smaller than the index, lists live in a pinned host backing store
 * read by the kernels over PCIe, and only the resident set occupies HBM:
 *   hivf_residency_set  -- make exactly `clusters` resident: evictions take
 *       effect for every later launch (tiered_cache.cpp:23-36), admissions in
 *       the given order while they fit the budget start asynchronous H2D
 *       copies on the index's copy stream; a list stays non-resident (read
 *       from the backing store) until its copy completes -- mid-swap =
 *       non-resident, as complete_swaps (:70-80) models it.
 *   hivf_residency_get  -- resident flags [n_clusters] (completed swaps).
 *   hivf_residency_sync -- wait for the swaps in flight and complete them.
 * Results never depend on residency (lane transparency,
 * proj/tests/test_retrieval_engine.cpp:158-199).  Without a budget every list
 * is in HBM and the set is bookkeeping only. */
hivf_status hivf_residency_set(hivf_index* idx, const uint32_t* clusters, uint32_t n);
hivf_status hivf_residency_get(const hivf_index* idx, uint8_t* resident_out);
hivf_status hivf_residency_sync(hivf_index* idx);

/* ---- introspection (bench / tests) ----------------------------------------- */
typedef struct {
  uint32_t kernels_launched;   /* kernels issued by the last search call */
  uint32_t n_work_items;       /* grouped-scan work items of the last call */
  uint32_t n_fallback;         /* queries that took an exact fallback path (last call) */
  uint32_t n_unique_lists;     /* distinct lists probed by the last batch */
  uint64_t scan_bytes;         /* algorithmic list bytes of the last batch (sum n_c*dim*4, or
                                  n_c*dim*2 when the scan read the fp16 filter copy) */
  uint32_t timed_calls;        /* calls accumulated below (option "time_kernels") */
  double assign_ms;            /* accumulated CUDA-event time: coarse assign kernels */
  double scan_ms;              /* accumulated CUDA-event time: grouped list scan kernel */
  double finalize_ms;          /* accumulated CUDA-event time: re-rank + fallback kernels */
  uint32_t scan_kernel;        /* last call: 0 exact only, 1 FFMA, 2 tcgen05 split, 3 tcgen05 single */
  uint32_t scan_group;         /* last call: queries per scan work item (8..32 narrow, 64 / 128 wide,
                                  256 = the CTA-pair scan) */
  uint32_t scan_filter_bits;   /* last call: 16 = the scan read the fp16 filter copy, 32 = the fp32 lists */
  uint32_t coarse_filter_bits; /* last coarse assign: 16 = tensor-core pass over the fp16 centroid copy,
                                  32 = FFMA pass, 0 = exact distance to every centroid (nprobe > 4096) */
} hivf_stats;
hivf_status hivf_last_stats(hivf_ctx* ctx, hivf_stats* out);
/* Options (0 = default): "seg_rows" rows per scan segment, "force_exact",
 * "hbm_list_budget" (bytes of fp32 list storage an index may keep in HBM; the
 * rest stays in pinned host memory, see residency; with "filter_h16" the fp16
 * filter copy of EVERY list is kept in HBM on top of the budget, so the scan
 * never crosses PCIe -- only the exact re-rank of cold lists' rows does),
 * "coarse_tc" (default 1: indexes created while non-zero get an fp16 copy of
 * the centroids and the coarse assign's distance pass of batches with at
 * least 2^26 multiply-adds (B x K x dim) runs as one tcgen05 kind::f16 GEMM,
 * filtered with the fp16 bound; 2: every batch; 0: FFMA pass; plans identical;
 * process default from env HIVF_COARSE_TC), "coarse_set" (default 1: the
 * batched search's coarse select needs its plans only as sets and re-ranks
 * only the centroids its bound cannot place),
 * "seed_rows" (default 32, 0 = off, <= 64) / "seed_ppl" (default 16): batches
 * with at least seed_ppl probes per list seed each query's shared drop bound
 * with the exact distances of seed_rows rows of its nearest probed list,
 * "filter_h16" (default 1: hivf_index_finish builds the fp16 filter copy of the
 * lists -- 0.5x the fp32 list bytes more HBM -- and single-pass scans stream it;
 * 0: no copy / the scans read the fp32 lists; results identical; process
 * default from env HIVF_FILTER_H16),
 * "scan_ctas", "scan_kernel" (0 auto, 1 FFMA, 2 tcgen05 split-precision,
 * 3 tcgen05 single-pass), "tc_qmax" (queries per scan work item: 8..32 step 8,
 * or 64 / 128 / 256 = the wide scans), "tc_wide_ppl" (probes per list above which a
 * single-pass batch uses the wide 64-query scan; default 0 = every single-pass
 * batch (measured faster at all densities), negative = never;
 * process default from env HIVF_TC_WIDE_PPL), "tc_wide2_ppl" (above it 128-query
 * groups, default 24, env HIVF_TC_WIDE2_PPL), "tc_pair_ppl" (above it 256-query
 * groups on CTA pairs, default 96, env HIVF_TC_PAIR_PPL), "time_kernels" (record events
 * around each phase and accumulate into hivf_stats), "reset_timers",
 * "search_graph" (default 1: hivf_search captures a batch shape seen twice in
 * a row into a CUDA graph and replays it; any option write, buffer growth or
 * index upload/destroy invalidates it; tiered indexes and kernel timing
 * bypass it). */
hivf_status hivf_set_option(hivf_ctx* ctx, const char* name, int64_t value);

/* ---- validation / debug (not on the search path) ---------------------------
 * hivf_debug_tc_dot: the list scan's tensor-core dot product in isolation on
 *   the current device (one CTA; A[128][D], B[n][D] host, n in {8, 16};
 *   split = 1 reproduces the 3-pass split, out[128][2n] = [hi*hi + lo*hi |
 *   hi*lo], split = 2 the fp16 filter's kind::f16 MMA on RN-converted fp16
 *   operands (K = 16 per step), else out[128][n]).  Used to validate the accumulation term of the
 *   filter bound on adversarial data (tests/test_gpu_tc_bound.py).
 * hivf_debug_bound: the filter-bound coefficients (e_a, e_b, e_c) of a scan
 *   kind (0 FFMA, 2 split tensor-core, 3 single-pass tensor-core) at dim D.
 * hivf_debug_tc_prof: per-CTA stall counters of the last k_scan_tc launches. */
int hivf_debug_tc_dot(const float* A, const float* B, unsigned D, unsigned n, int split, float* out);
/* hivf_debug_tc2_dot: the same for a CTA pair (cta_group::2, M = 256): A[256][D],
 *   B[n][D] (n in {16, 32}); bsplit = 1 puts B rows [c*n/2, (c+1)*n/2) in CTA c,
 *   0 puts all of B in both; out[256][n] (row r from CTA r / 128). */
int hivf_debug_tc2_dot(const float* A, const float* B, unsigned D, unsigned n, int bsplit, float* out);
int hivf_debug_bound(int kind, unsigned D, double* e_a, double* e_b, double* e_c);
int hivf_debug_tc_prof(unsigned long long* out, int n_ctas);
/* hivf_debug_mma_rate: cycles per MMA of the scan's step shapes in isolation
 *   (mode 0 f16 SS, 1 tf32 SS, 2 f16 with A in TMEM, 3 tcgen05.cp of the A
 *   k-step + f16 TS MMA, 4 + j f16 SS round robin over 1 + j accumulators;
 *   M = 128, N = n), A[128][32], B[256][32] host;
 *   d_out[128][32] = the accumulator (first 32 columns). */
int hivf_debug_mma_rate(int mode, unsigned n, unsigned reps, const float* A, const float* B, double* cycles_out,
                        float* d_out);

#ifdef __cplusplus
}
#endif

#endif /* HIVF_H_ */
