/*
 * hivf_oracle.c -- CPU restatement of the reference IVF retrieval hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path
 * (paper_2507_09138_b200/) links, loads or calls this file; only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg use it, and only as
 * the checker.
 *
 * Every function restates one reference function of
 *   /root/reference/proj/include/hedra/embedding.hpp
 *   /root/reference/proj/src/vector_index.cpp
 * and cites the file:line it follows.  The arithmetic contract is the one the
 * reference compiles to (proj/CMakeLists.txt: -O2, no -march, no fast-math on
 * x86-64, i.e. SSE2 scalar doubles, no FMA contraction): this file is built
 * with -O2 -ffp-contract=off (oracle/Makefile) so it keeps exactly that
 * rounding sequence.
 *
 * Pinned against: the reference's own known-answer tests (tests/golden/) and
 * the reference sources compiled unmodified into oracle/_ref/libhedra_ref.so
 * (tests/test_oracle.py).
 *
 * Index representation (CSR, the shape index_from_assignments builds,
 * vector_index.cpp:210-235): list c owns rows [off[c], off[c+1]) of the
 * row-major vectors[N*dim] and ids[N].
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

typedef struct {
  uint64_t id;
  double d;
} orc_entry;

/* embedding.hpp:27-34 -- sequential double accumulate of ((double)a-(double)b)^2 */
double orc_squared_l2(const float* a, const float* b, uint64_t dim) {
  double acc = 0.0;
  for (uint64_t i = 0; i < dim; ++i) {
    const double d = (double)a[i] - (double)b[i];
    acc += d * d;
  }
  return acc;
}

/* embedding.hpp:36-43 -- double norm, divide, cast back to float */
void orc_normalized(const float* v, uint64_t dim, float* out) {
  double norm = 0.0;
  for (uint64_t i = 0; i < dim; ++i) norm += (double)v[i] * (double)v[i];
  norm = sqrt(norm);
  if (norm == 0.0) {
    memmove(out, v, dim * sizeof(float));
    return;
  }
  for (uint64_t i = 0; i < dim; ++i) out[i] = (float)(v[i] / norm);
}

/* vector_index.hpp:41-44 -- (distance asc, doc_id asc) */
static int entry_less(const orc_entry* a, const orc_entry* b) {
  if (a->d != b->d) return a->d < b->d;
  return a->id < b->id;
}

/* vector_index.cpp:38-53 -- TopKResult::insert.  Returns 1 when the set changed. */
int orc_topk_insert(orc_entry* e, uint64_t* n, uint64_t k, uint64_t id, double d) {
  if (k == 0) return 0;
  for (uint64_t i = 0; i < *n; ++i) {
    if (e[i].id == id) {
      if (d >= e[i].d) return 0;
      memmove(e + i, e + i + 1, (*n - i - 1) * sizeof(orc_entry));
      *n -= 1;
      break;
    }
  }
  const orc_entry x = {id, d};
  uint64_t lo = 0, hi = *n; /* lower_bound under entry_less */
  while (lo < hi) {
    const uint64_t mid = (lo + hi) / 2;
    if (entry_less(&e[mid], &x)) lo = mid + 1; else hi = mid;
  }
  if (*n >= k && lo == *n) return 0;
  /* the caller's buffer holds k+1 entries so the transient overflow fits */
  memmove(e + lo + 1, e + lo, (*n - lo) * sizeof(orc_entry));
  e[lo] = x;
  *n += 1;
  if (*n > k) *n -= 1;
  return 1;
}

static int cmp_id_then_d(const void* pa, const void* pb) {
  const orc_entry* a = (const orc_entry*)pa;
  const orc_entry* b = (const orc_entry*)pb;
  if (a->id != b->id) return a->id < b->id ? -1 : 1;
  if (a->d != b->d) return a->d < b->d ? -1 : 1;
  return 0;
}

static int cmp_entry(const void* pa, const void* pb) {
  const orc_entry* a = (const orc_entry*)pa;
  const orc_entry* b = (const orc_entry*)pb;
  if (entry_less(a, b)) return -1;
  if (entry_less(b, a)) return 1;
  return 0;
}

/* vector_index.cpp:71-91 -- merge_topk: union, collapse duplicate ids to the
 * min distance, sort (d, id), truncate to k.  out needs room for k+1. */
uint64_t orc_merge_topk(const orc_entry* a, uint64_t na, const orc_entry* b,
                        uint64_t nb, uint64_t k, orc_entry* out) {
  orc_entry* all = (orc_entry*)malloc((na + nb + 1) * sizeof(orc_entry));
  memcpy(all, a, na * sizeof(orc_entry));
  memcpy(all + na, b, nb * sizeof(orc_entry));
  const uint64_t n = na + nb;
  qsort(all, n, sizeof(orc_entry), cmp_id_then_d);
  uint64_t m = 0;
  for (uint64_t i = 0; i < n; ++i)
    if (m == 0 || all[m - 1].id != all[i].id) all[m++] = all[i];
  qsort(all, m, sizeof(orc_entry), cmp_entry);
  if (m > k) m = k;
  uint64_t on = 0;
  for (uint64_t i = 0; i < m; ++i) orc_topk_insert(out, &on, k, all[i].id, all[i].d);
  free(all);
  return on;
}

typedef struct {
  double d;
  uint32_t c;
} dist_cluster;

static int cmp_dist_cluster(const void* pa, const void* pb) {
  const dist_cluster* a = (const dist_cluster*)pa;
  const dist_cluster* b = (const dist_cluster*)pb;
  if (a->d != b->d) return a->d < b->d ? -1 : 1;
  if (a->c != b->c) return a->c < b->c ? -1 : 1;
  return 0;
}

/* vector_index.cpp:261-278 -- select_clusters.  metric 1 = cosine (query
 * normalized first, :270).  Returns 0, or -1 for nprobe out of range (the
 * reference's invalid_argument, :264-265).  dists_out may be NULL. */
int orc_select_clusters(const float* centroids, uint32_t n_clusters, uint32_t dim,
                        int metric, const float* query, uint32_t nprobe,
                        uint32_t* plan_out, double* dists_out) {
  if (nprobe < 1 || nprobe > n_clusters) return -1;
  float* q = (float*)malloc(dim * sizeof(float));
  if (metric == 1) orc_normalized(query, dim, q); else memcpy(q, query, dim * sizeof(float));
  dist_cluster* order = (dist_cluster*)malloc(n_clusters * sizeof(dist_cluster));
  for (uint32_t c = 0; c < n_clusters; ++c) {
    order[c].d = orc_squared_l2(centroids + (uint64_t)c * dim, q, dim);
    order[c].c = c;
  }
  qsort(order, n_clusters, sizeof(dist_cluster), cmp_dist_cluster);
  for (uint32_t i = 0; i < nprobe; ++i) {
    plan_out[i] = order[i].c;
    if (dists_out) dists_out[i] = order[i].d;
  }
  free(order);
  free(q);
  return 0;
}

/* vector_index.cpp:18-29 -- nearest_centroid, ties keep the lowest id */
uint32_t orc_nearest_centroid(const float* centroids, uint32_t n_clusters,
                              uint32_t dim, const float* v) {
  double best = INFINITY;
  uint32_t best_id = 0;
  for (uint32_t c = 0; c < n_clusters; ++c) {
    const double d = orc_squared_l2(centroids + (uint64_t)c * dim, v, dim);
    if (d < best) {
      best = d;
      best_id = c;
    }
  }
  return best_id;
}

/* vector_index.cpp:202-208 -- compute_assignments */
void orc_compute_assignments(const float* corpus, uint64_t n, uint32_t dim,
                             const float* centroids, uint32_t n_clusters,
                             uint32_t* assign_out) {
  for (uint64_t i = 0; i < n; ++i)
    assign_out[i] = orc_nearest_centroid(centroids, n_clusters, dim, corpus + i * dim);
}

/* vector_index.cpp:291-317 -- search_clusters over a CSR index.  The cursor
 * state is (query already normalized for cosine, plan, next_pos, heap).
 * changed_out[j] receives the per-cluster `changed` flag (:300-313) that
 * feeds unchanged_streak.  Returns 0, or -2 when a cluster does not match the
 * plan order / the cursor is exhausted (the reference's runtime_error). */
int orc_search_clusters(const float* vectors, const uint64_t* ids,
                        const uint64_t* list_off, uint32_t dim,
                        const float* query, const uint32_t* plan, uint32_t plan_len,
                        uint32_t* next_pos, orc_entry* heap, uint64_t* heap_n,
                        uint64_t k, const uint32_t* clusters, uint32_t n_clusters,
                        uint8_t* changed_out) {
  for (uint32_t j = 0; j < n_clusters; ++j) {
    const uint32_t c = clusters[j];
    if (*next_pos >= plan_len) return -2;
    if (plan[*next_pos] != c) return -2;
    int changed = 0;
    for (uint64_t r = list_off[c]; r < list_off[c + 1]; ++r) {
      const double d = orc_squared_l2(query, vectors + r * dim, dim);
      changed |= orc_topk_insert(heap, heap_n, k, ids[r], d);
    }
    *next_pos += 1;
    if (changed_out) changed_out[j] = (uint8_t)changed;
  }
  return 0;
}

/* Per-request search: make_cursor (vector_index.cpp:280-289) followed by
 * search_step over the whole plan (:319-328).  Per query: ids_out[k],
 * dists_out[k], counts_out = heap size.  Returns 0 / -1 (invalid_argument). */
int orc_ivf_search(const float* centroids, uint32_t n_clusters, uint32_t dim,
                   int metric, const float* vectors, const uint64_t* ids,
                   const uint64_t* list_off, const float* queries, uint32_t n_queries,
                   uint32_t nprobe, uint32_t k, uint64_t* ids_out, double* dists_out,
                   uint32_t* counts_out) {
  if (k == 0) return -1;
  if (nprobe < 1 || nprobe > n_clusters) return -1;
  uint32_t* plan = (uint32_t*)malloc(nprobe * sizeof(uint32_t));
  float* q = (float*)malloc(dim * sizeof(float));
  orc_entry* heap = (orc_entry*)malloc((k + 1) * sizeof(orc_entry));
  for (uint32_t b = 0; b < n_queries; ++b) {
    const float* query = queries + (uint64_t)b * dim;
    orc_select_clusters(centroids, n_clusters, dim, metric, query, nprobe, plan, NULL);
    if (metric == 1) orc_normalized(query, dim, q); else memcpy(q, query, dim * sizeof(float));
    uint64_t hn = 0;
    uint32_t next = 0;
    orc_search_clusters(vectors, ids, list_off, dim, q, plan, nprobe, &next, heap, &hn, k,
                        plan, nprobe, NULL);
    for (uint32_t i = 0; i < k; ++i) {
      ids_out[(uint64_t)b * k + i] = i < hn ? heap[i].id : 0;
      dists_out[(uint64_t)b * k + i] = i < hn ? heap[i].d : 0.0;
    }
    counts_out[b] = (uint32_t)hn;
  }
  free(heap);
  free(q);
  free(plan);
  return 0;
}

/* vector_index.cpp:330-342 -- brute_force_search over a row-major corpus. */
uint64_t orc_brute_force(const float* corpus, const uint64_t* ids, uint64_t n,
                         uint32_t dim, int metric, const float* query, uint64_t k,
                         uint64_t* ids_out, double* dists_out) {
  orc_entry* heap = (orc_entry*)malloc((k + 1) * sizeof(orc_entry));
  float* q = (float*)malloc(dim * sizeof(float));
  float* row = (float*)malloc(dim * sizeof(float));
  if (metric == 1) orc_normalized(query, dim, q); else memcpy(q, query, dim * sizeof(float));
  uint64_t hn = 0;
  for (uint64_t i = 0; i < n; ++i) {
    if (metric == 1) orc_normalized(corpus + i * dim, dim, row);
    else memcpy(row, corpus + i * dim, dim * sizeof(float));
    orc_topk_insert(heap, &hn, k, ids[i], orc_squared_l2(q, row, dim));
  }
  for (uint64_t i = 0; i < hn; ++i) {
    ids_out[i] = heap[i].id;
    dists_out[i] = heap[i].d;
  }
  free(row);
  free(q);
  free(heap);
  return hn;
}
