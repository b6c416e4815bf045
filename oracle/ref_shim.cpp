// ref_shim.cpp -- extern "C" test shim over the UNMODIFIED reference sources.
//
// TEST INFRASTRUCTURE ONLY (see oracle/hivf_oracle.c header).  oracle/Makefile
// compiles this file together with the reference's own
//   /root/reference/proj/src/{vector_index,retrieval_engine,tiered_cache,similarity}.cpp
// (read in place, never copied) into oracle/_ref/libhedra_ref.so, built with
// the reference's flags (-std=c++20 -O2, no -march, no fast-math;
// proj/CMakeLists.txt:8-10,28).  Python tests and bench.py's cpu_baseline leg
// load it with ctypes.  Nothing in the product path links it.
//
// Exceptions never cross this boundary: invalid_argument -> -1,
// runtime_error / anything else -> -2.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <vector>

#include "hedra/retrieval_engine.hpp"
#include "hedra/similarity.hpp"
#include "hedra/tiered_cache.hpp"
#include "hedra/vector_index.hpp"

using namespace hedra;

namespace {

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  } catch (...) {
    return -2;
  }
}

ivf::Corpus make_corpus(const float* data, const uint64_t* ids, uint64_t n, uint32_t dim,
                        int metric) {
  ivf::Corpus c;
  c.dim = dim;
  c.metric = metric == 1 ? Metric::Cosine : Metric::L2;
  c.data.assign(data, data + n * dim);
  c.doc_ids.assign(ids, ids + n);
  return c;
}

ivf::Centroids make_centroids(const float* rows, uint32_t k, uint32_t dim) {
  ivf::Centroids c;
  c.dim = dim;
  for (uint32_t i = 0; i < k; ++i) c.rows.emplace_back(rows + uint64_t(i) * dim, rows + uint64_t(i + 1) * dim);
  return c;
}

struct Engine {
  std::unique_ptr<ret::RetrievalEngine> eng;
};

}  // namespace

extern "C" {

void* ref_index_build(const float* corpus, const uint64_t* ids, uint64_t n, uint32_t dim,
                      int metric, const float* centroids, uint32_t k_clusters) {
  ivf::IvfIndex* out = nullptr;
  guarded([&] {
    auto c = make_corpus(corpus, ids, n, dim, metric);
    out = new ivf::IvfIndex(ivf::build_index(c, make_centroids(centroids, k_clusters, dim),
                                             c.metric));
  });
  return out;
}

void* ref_index_from_assign(const float* corpus, const uint64_t* ids, uint64_t n, uint32_t dim,
                            int metric, const float* centroids, uint32_t k_clusters,
                            const uint32_t* assign) {
  ivf::IvfIndex* out = nullptr;
  guarded([&] {
    auto c = make_corpus(corpus, ids, n, dim, metric);
    std::vector<ClusterId> a(assign, assign + n);
    out = new ivf::IvfIndex(ivf::index_from_assignments(
        c, make_centroids(centroids, k_clusters, dim), c.metric, a));
  });
  return out;
}

// The IvfIndex index_from_assignments (vector_index.cpp:210-235) builds for
// these lists, filled straight from CSR arrays in its list order (corpus order
// within a list): centroids, metric, dim, list_ids, list_vectors.  locator and
// mean_assigned_distance stay empty -- make_cursor / search_clusters /
// RetrievalEngine::execute never read them (vector_index.cpp:261-328,
// retrieval_engine.cpp:55-152).  bench.py's CPU arm builds its restricted
// timing index this way (tens of GB) instead of through the per-row map
// inserts and distance sums of index_from_assignments.
void* ref_index_from_csr(const float* centroids, uint32_t k_clusters, uint32_t dim, int metric,
                         const uint64_t* off, const float* vectors, const uint64_t* ids) {
  ivf::IvfIndex* out = nullptr;
  guarded([&] {
    auto* ix = new ivf::IvfIndex;
    ix->centroids = make_centroids(centroids, k_clusters, dim);
    ix->metric = metric == 1 ? Metric::Cosine : Metric::L2;
    ix->dim = dim;
    ix->list_ids.resize(k_clusters);
    ix->list_vectors.resize(k_clusters);
    for (uint32_t c = 0; c < k_clusters; ++c) {
      ix->list_ids[c].assign(ids + off[c], ids + off[c + 1]);
      ix->list_vectors[c].assign(vectors + off[c] * dim, vectors + off[c + 1] * dim);
    }
    out = ix;
  });
  return out;
}

void ref_index_free(void* idx) { delete static_cast<ivf::IvfIndex*>(idx); }

uint64_t ref_index_total(void* idx) { return static_cast<ivf::IvfIndex*>(idx)->total_vectors(); }

// CSR export of the lists exactly as index_from_assignments laid them out.
void ref_index_export(void* p, uint64_t* off, float* vectors, uint64_t* ids,
                      double* mean_assigned) {
  auto* idx = static_cast<ivf::IvfIndex*>(p);
  uint64_t pos = 0;
  off[0] = 0;
  for (std::size_t c = 0; c < idx->k_clusters(); ++c) {
    const auto& l = idx->list_ids[c];
    if (vectors)
      std::memcpy(vectors + pos * idx->dim, idx->list_vectors[c].data(),
                  l.size() * idx->dim * sizeof(float));
    if (ids) std::memcpy(ids + pos, l.data(), l.size() * sizeof(uint64_t));
    pos += l.size();
    off[c + 1] = pos;
  }
  if (mean_assigned) *mean_assigned = idx->mean_assigned_distance;
}

int ref_train_kmeans(const float* corpus, uint64_t n, uint32_t dim, uint32_t k_clusters,
                     uint32_t iters, uint64_t seed, float* out) {
  return guarded([&] {
    std::vector<uint64_t> ids(n);
    for (uint64_t i = 0; i < n; ++i) ids[i] = i;
    auto c = make_corpus(corpus, ids.data(), n, dim, 0);
    auto cents = ivf::train_kmeans(c, k_clusters, iters, seed);
    for (uint32_t i = 0; i < k_clusters; ++i)
      std::memcpy(out + uint64_t(i) * dim, cents.rows[i].data(), dim * sizeof(float));
  });
}

// --- persistence (vector_index.cpp:344-473), for byte-level parity tests ------
int ref_save_corpus(const char* path, const float* data, const uint64_t* ids, uint64_t n, uint32_t dim,
                    int metric) {
  return guarded([&] { ivf::save_corpus(path, make_corpus(data, ids, n, dim, metric)); });
}
int ref_save_centroids(const char* path, const float* rows, uint32_t k, uint32_t dim, int metric) {
  return guarded([&] {
    ivf::Centroids c;
    c.dim = dim;
    for (uint32_t i = 0; i < k; ++i) c.rows.emplace_back(rows + uint64_t(i) * dim, rows + uint64_t(i + 1) * dim);
    ivf::save_centroids(path, c, static_cast<Metric>(metric));
  });
}
int ref_save_assignments(const char* path, const uint32_t* a, uint64_t n) {
  return guarded([&] { ivf::save_assignments(path, std::vector<ClusterId>(a, a + n)); });
}
// load_corpus into caller buffers sized by a first call with data == nullptr
int ref_load_corpus(const char* path, uint32_t* dim, uint64_t* n, int* metric, float* data, uint64_t* ids) {
  return guarded([&] {
    auto c = ivf::load_corpus(path);
    *dim = c.dim;
    *n = c.size();
    *metric = static_cast<int>(c.metric);
    if (data) std::memcpy(data, c.data.data(), c.data.size() * sizeof(float));
    if (ids) std::memcpy(ids, c.doc_ids.data(), c.doc_ids.size() * sizeof(uint64_t));
  });
}

int ref_compute_assignments(const float* corpus, uint64_t n, uint32_t dim,
                            const float* centroids, uint32_t k_clusters, uint32_t* out) {
  return guarded([&] {
    std::vector<uint64_t> ids(n);
    for (uint64_t i = 0; i < n; ++i) ids[i] = i;
    auto a = ivf::compute_assignments(make_corpus(corpus, ids.data(), n, dim, 0),
                                      make_centroids(centroids, k_clusters, dim));
    std::memcpy(out, a.data(), n * sizeof(uint32_t));
  });
}

int ref_select_clusters(void* p, const float* q, uint32_t nprobe, uint32_t* plan) {
  auto* idx = static_cast<ivf::IvfIndex*>(p);
  return guarded([&] {
    Embedding query(q, q + idx->dim);
    auto r = ivf::select_clusters(*idx, query, nprobe);
    std::memcpy(plan, r.data(), r.size() * sizeof(uint32_t));
  });
}

// make_cursor + search_step over the full plan, per query.
int ref_search(void* p, const float* queries, uint32_t n_queries, uint32_t nprobe, uint32_t k,
               uint64_t* ids_out, double* d_out, uint32_t* counts) {
  auto* idx = static_cast<ivf::IvfIndex*>(p);
  return guarded([&] {
    for (uint32_t b = 0; b < n_queries; ++b) {
      Embedding query(queries + uint64_t(b) * idx->dim, queries + uint64_t(b + 1) * idx->dim);
      auto cur = ivf::make_cursor(*idx, query, nprobe, k);
      ivf::search_step(*idx, cur, nprobe);
      const auto& e = cur.heap.entries();
      for (uint32_t i = 0; i < k; ++i) {
        ids_out[uint64_t(b) * k + i] = i < e.size() ? e[i].doc_id : 0;
        d_out[uint64_t(b) * k + i] = i < e.size() ? e[i].distance : 0.0;
      }
      counts[b] = static_cast<uint32_t>(e.size());
    }
  });
}

uint64_t ref_brute_force(const float* corpus, const uint64_t* ids, uint64_t n, uint32_t dim,
                         int metric, const float* q, uint64_t k, uint64_t* ids_out,
                         double* d_out) {
  uint64_t cnt = 0;
  guarded([&] {
    auto c = make_corpus(corpus, ids, n, dim, metric);
    auto r = ivf::brute_force_search(c, Embedding(q, q + dim), k);
    for (const auto& e : r.entries()) {
      ids_out[cnt] = e.doc_id;
      d_out[cnt] = e.distance;
      ++cnt;
    }
  });
  return cnt;
}

uint64_t ref_merge_topk(const uint64_t* a_ids, const double* a_d, uint64_t na,
                        const uint64_t* b_ids, const double* b_d, uint64_t nb, uint64_t k,
                        uint64_t* ids_out, double* d_out) {
  ivf::TopKResult a(k + na), b(k + nb);
  for (uint64_t i = 0; i < na; ++i) a.insert(a_ids[i], a_d[i]);
  for (uint64_t i = 0; i < nb; ++i) b.insert(b_ids[i], b_d[i]);
  auto m = ivf::merge_topk(a, b, k);
  uint64_t n = 0;
  for (const auto& e : m.entries()) {
    ids_out[n] = e.doc_id;
    d_out[n] = e.distance;
    ++n;
  }
  return n;
}

// --- RetrievalEngine (retrieval_engine.hpp:80-110) --------------------------

void* ref_engine_new(void* idx, double per_vector_ns, double fast_speedup, double fixed_call_us,
                     uint64_t capacity_gc, int update_interval, double bw_gb_s, double decay,
                     uint64_t min_fast) {
  ret::RetrievalCostModel m;
  m.per_vector_ns = per_vector_ns;
  m.fast_speedup = fast_speedup;
  m.fixed_call_us = fixed_call_us;
  cache::CacheConfig cfg;
  cfg.capacity_gc = capacity_gc;
  cfg.update_interval = update_interval;
  cfg.transfer_bandwidth_gb_s = bw_gb_s;
  cfg.decay = decay;
  cfg.min_fast_clusters = min_fast;
  auto* e = new Engine;
  e->eng = std::make_unique<ret::RetrievalEngine>(static_cast<ivf::IvfIndex*>(idx), m, cfg);
  return e;
}

void ref_engine_free(void* e) { delete static_cast<Engine*>(e); }

// make_cursor + optional seed merge (scheduler.cpp:920-930) + submit.
int ref_engine_submit(void* pe, int64_t req, int32_t node, const float* q, uint32_t nprobe,
                      uint32_t k, const uint64_t* seed_ids, const double* seed_d,
                      uint32_t n_seed, const uint32_t* plan_override) {
  auto* e = static_cast<Engine*>(pe);
  return guarded([&] {
    const auto& idx = e->eng->index();
    ret::RetrievalTask t;
    t.request_id = req;
    t.node_id = node;
    t.cursor = ivf::make_cursor(idx, Embedding(q, q + idx.dim), nprobe, k);
    if (plan_override)
      t.cursor.plan.assign(plan_override, plan_override + t.cursor.plan.size());
    if (n_seed) {
      ivf::TopKResult seed(k);
      for (uint32_t i = 0; i < n_seed; ++i) seed.insert(seed_ids[i], seed_d[i]);
      t.cursor.heap = ivf::merge_topk(t.cursor.heap, seed, k);
    }
    e->eng->submit(std::move(t));
  });
}

int ref_engine_plan(void* pe, int64_t req, int32_t node, uint32_t* plan_out, uint32_t* len) {
  auto* e = static_cast<Engine*>(pe);
  const auto* t = e->eng->find(req, node);
  if (!t) return -1;
  std::memcpy(plan_out, t->cursor.plan.data(), t->cursor.plan.size() * sizeof(uint32_t));
  *len = static_cast<uint32_t>(t->cursor.plan.size());
  return 0;
}

int ref_engine_execute(void* pe, uint32_t n_items, const int64_t* reqs, const int32_t* nodes,
                       const uint32_t* item_off, const uint32_t* clusters, double now_ms,
                       int live, uint8_t* heap_changed, uint8_t* completed, double* wall_ms,
                       double* modeled_ms, uint64_t* fast_clusters, uint64_t* slow_clusters) {
  auto* e = static_cast<Engine*>(pe);
  return guarded([&] {
    ret::SubStageBatch batch;
    for (uint32_t i = 0; i < n_items; ++i) {
      ret::BatchItem it;
      it.request_id = reqs[i];
      it.node_id = nodes[i];
      it.clusters.assign(clusters + item_off[i], clusters + item_off[i + 1]);
      batch.items.push_back(std::move(it));
    }
    auto r = e->eng->execute(batch, now_ms, live != 0);
    for (uint32_t i = 0; i < r.deltas.size(); ++i) {
      if (heap_changed) heap_changed[i] = r.deltas[i].heap_changed;
      if (completed) completed[i] = r.deltas[i].completed;
    }
    if (wall_ms) *wall_ms = r.wall_ms;
    if (modeled_ms) *modeled_ms = r.modeled_ms;
    if (fast_clusters) *fast_clusters = r.fast_clusters;
    if (slow_clusters) *slow_clusters = r.slow_clusters;
  });
}

int ref_engine_heap(void* pe, int64_t req, int32_t node, uint64_t* ids, double* d,
                    uint32_t cap, uint32_t* n, uint64_t* streak, uint64_t* next_pos,
                    uint64_t* searched) {
  auto* e = static_cast<Engine*>(pe);
  const auto* t = e->eng->find(req, node);
  if (!t) return -1;
  const auto& en = t->cursor.heap.entries();
  uint32_t m = 0;
  for (; m < en.size() && m < cap; ++m) {
    ids[m] = en[m].doc_id;
    d[m] = en[m].distance;
  }
  *n = m;
  if (streak) *streak = t->cursor.unchanged_streak;
  if (next_pos) *next_pos = t->cursor.next_pos;
  if (searched) *searched = t->cursor.clusters_searched;
  return 0;
}

int ref_engine_extract(void* pe, int64_t req, int32_t node) {
  auto* e = static_cast<Engine*>(pe);
  return guarded([&] { (void)e->eng->extract(req, node); });
}

// --- ClusterCacheState (tiered_cache.hpp:37-78) -----------------------------

void* ref_cache_new(uint64_t capacity_gc, int update_interval, double bw_gb_s, double decay,
                    uint64_t min_fast) {
  cache::CacheConfig cfg;
  cfg.capacity_gc = capacity_gc;
  cfg.update_interval = update_interval;
  cfg.transfer_bandwidth_gb_s = bw_gb_s;
  cfg.decay = decay;
  cfg.min_fast_clusters = min_fast;
  return new cache::ClusterCacheState(cfg);
}
void ref_cache_free(void* c) { delete static_cast<cache::ClusterCacheState*>(c); }
void ref_cache_record_access(void* c, const uint32_t* ids, uint32_t n) {
  static_cast<cache::ClusterCacheState*>(c)->record_access(std::vector<ClusterId>(ids, ids + n));
}
// Returns the number of swaps; fills clusters / inbound / completes_at (cap entries).
uint32_t ref_cache_maybe_update(void* c, double now_ms, void* idx, uint32_t* clusters,
                                uint8_t* inbound, double* completes, uint32_t cap) {
  auto plan = static_cast<cache::ClusterCacheState*>(c)->maybe_update(
      now_ms, *static_cast<ivf::IvfIndex*>(idx));
  for (uint32_t i = 0; i < plan.size() && i < cap; ++i) {
    clusters[i] = plan[i].cluster;
    inbound[i] = plan[i].inbound;
    completes[i] = plan[i].completes_at_ms;
  }
  return static_cast<uint32_t>(plan.size());
}
void ref_cache_complete_swaps(void* c, double now_ms) {
  static_cast<cache::ClusterCacheState*>(c)->complete_swaps(now_ms);
}
// fast/slow sizes returned; arrays need n entries each.
void ref_cache_partition(void* c, const uint32_t* ids, uint32_t n, uint32_t* fast,
                         uint32_t* n_fast, uint32_t* slow, uint32_t* n_slow) {
  auto p = static_cast<cache::ClusterCacheState*>(c)->partition_batch(
      std::vector<ClusterId>(ids, ids + n));
  std::memcpy(fast, p.fast.data(), p.fast.size() * sizeof(uint32_t));
  std::memcpy(slow, p.slow.data(), p.slow.size() * sizeof(uint32_t));
  *n_fast = static_cast<uint32_t>(p.fast.size());
  *n_slow = static_cast<uint32_t>(p.slow.size());
}
void ref_cache_count_hits(void* c, const uint32_t* ids, uint32_t n) {
  static_cast<cache::ClusterCacheState*>(c)->count_access_hits(
      std::vector<ClusterId>(ids, ids + n));
}
int ref_cache_resident(void* c, uint32_t id) {
  return static_cast<cache::ClusterCacheState*>(c)->resident(id) ? 1 : 0;
}
uint64_t ref_cache_resident_count(void* c) {
  return static_cast<cache::ClusterCacheState*>(c)->resident_count();
}
void ref_cache_stats(void* c, uint64_t* hits, uint64_t* misses, uint64_t* swaps) {
  auto* s = static_cast<cache::ClusterCacheState*>(c);
  *hits = s->hits();
  *misses = s->misses();
  *swaps = s->swap_count();
}

// --- CPU baseline: the coarse/naive scheduler shape -------------------------
// make_cursor per query (serial) + one RetrievalEngine::execute(live_math)
// with one BatchItem per query holding its full plan
// (scheduler.cpp:997-1005,1031-1045; retrieval_engine.cpp:55-152).
// Returns the wall-clock milliseconds of the whole call (cursor build +
// execute); results land in ids/d/counts.
double ref_bench_execute(void* p, const float* queries, uint32_t n_queries, uint32_t nprobe,
                         uint32_t k, int live, uint64_t* ids_out, double* d_out,
                         uint32_t* counts) {
  auto* idx = static_cast<ivf::IvfIndex*>(p);
  double ms = -1.0;
  guarded([&] {
    const auto t0 = std::chrono::steady_clock::now();
    ret::RetrievalCostModel m;
    ret::RetrievalEngine eng(idx, m, cache::CacheConfig{});
    ret::SubStageBatch batch;
    for (uint32_t b = 0; b < n_queries; ++b) {
      ret::RetrievalTask t;
      t.request_id = b;
      t.node_id = 0;
      t.cursor = ivf::make_cursor(
          *idx,
          Embedding(queries + uint64_t(b) * idx->dim, queries + uint64_t(b + 1) * idx->dim),
          nprobe, k);
      ret::BatchItem it;
      it.request_id = b;
      it.node_id = 0;
      it.clusters = t.cursor.plan;
      eng.submit(std::move(t));
      batch.items.push_back(std::move(it));
    }
    eng.execute(batch, 0.0, live != 0);
    ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    for (uint32_t b = 0; b < n_queries; ++b) {
      const auto* t = eng.find(b, 0);
      const auto& e = t->cursor.heap.entries();
      for (uint32_t i = 0; i < k; ++i) {
        if (ids_out) ids_out[uint64_t(b) * k + i] = i < e.size() ? e[i].doc_id : 0;
        if (d_out) d_out[uint64_t(b) * k + i] = i < e.size() ? e[i].distance : 0.0;
      }
      if (counts) counts[b] = static_cast<uint32_t>(e.size());
    }
  });
  return ms;
}

}  // extern "C"
