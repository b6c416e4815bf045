// hedra_ivf_gpu.cpp -- the reference's hot-path translation units
// (proj/src/vector_index.cpp and proj/src/retrieval_engine.cpp) re-implemented
// over libhivf, against the reference headers: compat/include/hedra/
// vector_index.hpp (GPU-backed IvfIndex) and the UNMODIFIED
// proj/include/hedra/retrieval_engine.hpp / tiered_cache.hpp.  Linked with the
// reference's other sources (scheduler.cpp, similarity.cpp, tiered_cache.cpp,
// ...), the reference scheduler, unit suites and acceptance suite run on the
// GPU engine (compat/build.py).
//
// Host work here is bookkeeping only (plans, cursors, heaps of <= k entries,
// the host mirror the reference IvfIndex also carries).  Every distance, coarse
// assignment, list scan and k-means step is a libhivf call: select_clusters ->
// hivf_assign, search_clusters / RetrievalEngine::execute -> hivf_scan_items
// (one call per sub-stage for all items), compute_assignments / train_kmeans
// -> hivf_compute_assignments_host / hivf_train_kmeans_host, brute_force_search
// -> hivf_search over a one-list index, mean_assigned_distance ->
// hivf_index_row_distances summed in the reference's corpus order.
#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <unordered_set>

#include "hedra/retrieval_engine.hpp"
#include "hedra/vector_index.hpp"
#include "../../include/hivf.h"
#include "../host/hvec_io.hpp"

namespace hedra::ivf::gpu {

namespace {

// One libhivf context per device, alive for the whole process (never torn
// down: static destructors would race the CUDA runtime's own teardown).
struct Ctx {
  hivf_ctx* ctx = nullptr;
  std::mutex mu;  // an hivf_ctx has one owning thread at a time
};

std::mutex g_registry_mu;
Ctx* g_ctx[64] = {};
int g_device = -1;
std::atomic<std::size_t> g_calls{0};

void check(hivf_status st) {
  ++g_calls;
  if (st == HIVF_OK) return;
  const std::string msg = hivf_last_error();
  if (st == HIVF_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

int current_device() {
  if (g_device < 0) {
    const char* env = std::getenv("HEDRA_GPU_DEVICE");
    g_device = env ? std::atoi(env) : 0;
  }
  return g_device;
}

Ctx& context() {
  std::lock_guard<std::mutex> g(g_registry_mu);
  const int dev = current_device();
  if (dev < 0 || dev >= 64) throw std::invalid_argument("hedra::gpu: device out of range");
  if (!g_ctx[dev]) {
    auto* c = new Ctx;
    check(hivf_ctx_create(dev, nullptr, &c->ctx));
    g_ctx[dev] = c;
  }
  return *g_ctx[dev];
}

}  // namespace

struct DeviceIndex {
  Ctx* ctx = nullptr;
  hivf_index* ix = nullptr;
  ~DeviceIndex() {
    if (ix) {
      std::lock_guard<std::mutex> g(ctx->mu);
      hivf_index_destroy(ix);
    }
  }
};

namespace {

std::mutex g_lazy_mu;

// HBM copy of `index` from its host lists (list order, CSR).
std::shared_ptr<DeviceIndex> upload(const IvfIndex& index) {
  const std::size_t K = index.k_clusters();
  const std::uint32_t dim = index.dim;
  if (index.centroids.k_clusters() != K)
    throw std::invalid_argument("IvfIndex: centroid count does not match the list count");
  std::vector<std::uint64_t> off(K + 1, 0);
  for (std::size_t c = 0; c < K; ++c) {
    if (index.list_vectors[c].size() != index.list_ids[c].size() * dim)
      throw std::invalid_argument("IvfIndex: list_vectors / list_ids size mismatch");
    off[c + 1] = off[c] + index.list_ids[c].size();
  }
  std::vector<float> cents;
  cents.reserve(K * dim);
  for (const auto& r : index.centroids.rows) {
    if (r.size() != dim) throw std::invalid_argument("build_index: dimension mismatch");
    cents.insert(cents.end(), r.begin(), r.end());
  }
  std::vector<float> rows;
  std::vector<DocId> ids;
  rows.reserve(off[K] * dim);
  ids.reserve(off[K]);
  for (std::size_t c = 0; c < K; ++c) {
    rows.insert(rows.end(), index.list_vectors[c].begin(), index.list_vectors[c].end());
    ids.insert(ids.end(), index.list_ids[c].begin(), index.list_ids[c].end());
  }
  auto dev = std::make_shared<DeviceIndex>();
  dev->ctx = &context();
  std::lock_guard<std::mutex> g(dev->ctx->mu);
  check(hivf_index_upload(dev->ctx->ctx, dim, static_cast<int>(index.metric),
                          static_cast<std::uint32_t>(K), cents.data(), off.data(), rows.data(),
                          ids.data(), &dev->ix));
  return dev;
}

// The device copy every call runs on (uploaded on first use for an index
// assembled by hand).
DeviceIndex& device_of(const IvfIndex& index) {
  std::lock_guard<std::mutex> g(g_lazy_mu);
  if (!index.device) index.device = upload(index);
  return *index.device;
}

}  // namespace

std::vector<SearchStepReport> search_clusters_batch_impl(const IvfIndex& index,
                                                         std::span<SearchCursor* const> cursors,
                                                         std::span<const std::span<const ClusterId>> clusters);
std::vector<TopKResult> brute_force_search_batch_impl(const Corpus& corpus,
                                                      std::span<const std::vector<float>> queries,
                                                      std::size_t k);

void set_device(int device) {
  std::lock_guard<std::mutex> g(g_registry_mu);
  g_device = device;
}
int device() {
  std::lock_guard<std::mutex> g(g_registry_mu);
  return current_device();
}
std::size_t device_calls() { return g_calls.load(); }

}  // namespace hedra::ivf::gpu

namespace hedra::gpu {
void set_device(int d) { ivf::gpu::set_device(d); }
int device() { return ivf::gpu::device(); }
std::size_t device_calls() { return ivf::gpu::device_calls(); }
}  // namespace hedra::gpu

namespace hedra::ivf {

using gpu::check;
using gpu::device_of;

// ---- TopKResult / merge_topk (vector_index.cpp:33-91 semantics) -------------
void TopKResult::set_k(std::size_t k) {
  k_ = k;
  if (entries_.size() > k_) entries_.resize(k_);
}

bool TopKResult::insert(DocId doc_id, double distance) {
  if (k_ == 0) return false;
  const auto dup = std::find_if(entries_.begin(), entries_.end(),
                                [&](const TopKEntry& e) { return e.doc_id == doc_id; });
  if (dup != entries_.end()) {
    if (!(distance < dup->distance)) return false;  // a repeated id keeps its minimum
    entries_.erase(dup);
  }
  const TopKEntry e{doc_id, distance};
  const auto at = std::lower_bound(entries_.begin(), entries_.end(), e, topk_less);
  if (at == entries_.end() && entries_.size() >= k_) return false;
  entries_.insert(at, e);
  if (entries_.size() > k_) entries_.pop_back();
  return true;
}

TopKResult TopKResult::truncated(std::size_t k) const {
  TopKResult out(k);
  out.entries_.assign(entries_.begin(), entries_.begin() + std::min(k, entries_.size()));
  return out;
}

bool TopKResult::operator==(const TopKResult& rhs) const {
  if (entries_.size() != rhs.entries_.size()) return false;
  for (std::size_t i = 0; i < entries_.size(); ++i)
    if (entries_[i].doc_id != rhs.entries_[i].doc_id || entries_[i].distance != rhs.entries_[i].distance)
      return false;
  return true;
}

std::vector<DocId> TopKResult::doc_ids() const {
  std::vector<DocId> out;
  out.reserve(entries_.size());
  for (const auto& e : entries_) out.push_back(e.doc_id);
  return out;
}

TopKResult merge_topk(const TopKResult& a, const TopKResult& b, std::size_t k) {
  std::map<DocId, double> best;  // duplicate ids collapse to their minimum
  for (const TopKResult* r : {&a, &b})
    for (const auto& e : r->entries()) {
      const auto [it, fresh] = best.emplace(e.doc_id, e.distance);
      if (!fresh && e.distance < it->second) it->second = e.distance;
    }
  std::vector<TopKEntry> all;
  all.reserve(best.size());
  for (const auto& [id, d] : best) all.push_back(TopKEntry{id, d});
  std::sort(all.begin(), all.end(), topk_less);
  if (all.size() > k) all.resize(k);
  TopKResult out(k);
  for (const auto& e : all) out.insert(e.doc_id, e.distance);
  return out;
}

std::size_t IvfIndex::total_vectors() const {
  std::size_t n = 0;
  for (const auto& l : list_ids) n += l.size();
  return n;
}

// ---- persistence ---------------------------------------------------------------
void save_corpus(const std::string& path, const Corpus& corpus) { hvec_io::save_corpus(path, corpus); }
Corpus load_corpus(const std::string& path) { return hvec_io::load_corpus<Corpus>(path); }
void save_centroids(const std::string& path, const Centroids& centroids, Metric metric) {
  hvec_io::save_centroids(path, centroids, metric);
}
Centroids load_centroids(const std::string& path) { return hvec_io::load_centroids<Centroids>(path); }
void save_assignments(const std::string& path, const std::vector<ClusterId>& assign) {
  hvec_io::save_assignments(path, assign);
}
std::vector<ClusterId> load_assignments(const std::string& path) { return hvec_io::load_assignments(path); }

// ---- index build (vector_index.cpp:99-259) ----------------------------------------
namespace {
std::vector<float> flat_centroids(const Centroids& c, std::uint32_t dim) {
  std::vector<float> out;
  out.reserve(c.k_clusters() * dim);
  for (const auto& r : c.rows) {
    if (r.size() != dim) throw std::invalid_argument("build_index: dimension mismatch");
    out.insert(out.end(), r.begin(), r.end());
  }
  return out;
}
}  // namespace

Centroids train_kmeans(const Corpus& corpus, std::size_t k_clusters, std::size_t max_iters,
                       std::uint64_t seed) {
  if (corpus.size() < k_clusters) throw std::invalid_argument("train_kmeans: corpus smaller than k_clusters");
  if (k_clusters == 0) throw std::invalid_argument("train_kmeans: k_clusters must be >= 1");
  if (max_iters == 0) throw std::invalid_argument("train_kmeans: max_iters must be >= 1");
  std::vector<float> out(k_clusters * corpus.dim);
  auto& ctx = gpu::context();
  {
    std::lock_guard<std::mutex> g(ctx.mu);
    check(hivf_train_kmeans_host(ctx.ctx, corpus.data.data(), corpus.size(), corpus.dim,
                                 static_cast<std::uint32_t>(k_clusters),
                                 static_cast<std::uint32_t>(max_iters), seed, out.data()));
  }
  Centroids c;
  c.dim = corpus.dim;
  c.rows.reserve(k_clusters);
  for (std::size_t r = 0; r < k_clusters; ++r)
    c.rows.emplace_back(out.begin() + r * corpus.dim, out.begin() + (r + 1) * corpus.dim);
  return c;
}

std::vector<ClusterId> compute_assignments(const Corpus& corpus, const Centroids& centroids) {
  std::vector<ClusterId> assign(corpus.size(), 0);
  // no centroids: nearest_centroid's loop never runs and every row gets 0 (:18-29)
  if (corpus.size() == 0 || centroids.k_clusters() == 0) return assign;
  const auto cents = flat_centroids(centroids, corpus.dim);
  auto& ctx = gpu::context();
  std::lock_guard<std::mutex> g(ctx.mu);
  check(hivf_compute_assignments_host(ctx.ctx, corpus.data.data(), corpus.size(), corpus.dim, cents.data(),
                                      static_cast<std::uint32_t>(centroids.k_clusters()), assign.data()));
  return assign;
}

IvfIndex index_from_assignments(const Corpus& corpus, const Centroids& centroids, Metric metric,
                                const std::vector<ClusterId>& assign) {
  if (assign.size() != corpus.size())
    throw std::invalid_argument("index_from_assignments: assignment count mismatch");
  const std::size_t K = centroids.k_clusters();
  IvfIndex index;
  index.centroids = centroids;
  index.metric = metric;
  index.dim = corpus.dim;
  index.list_ids.resize(K);
  index.list_vectors.resize(K);
  std::vector<std::uint32_t> pos(corpus.size());  // row i's offset inside its list
  for (std::size_t i = 0; i < corpus.size(); ++i) {
    const ClusterId c = assign[i];
    if (c >= K) throw std::invalid_argument("index_from_assignments: cluster id out of range");
    pos[i] = static_cast<std::uint32_t>(index.list_ids[c].size());
    index.locator[corpus.doc_ids[i]] = IvfIndex::DocLocation{c, pos[i]};
    index.list_ids[c].push_back(corpus.doc_ids[i]);
    const float* row = corpus.row(i);
    index.list_vectors[c].insert(index.list_vectors[c].end(), row, row + corpus.dim);
  }
  if (K == 0) return index;  // nothing to search; select_clusters rejects every nprobe
  index.device = gpu::upload(index);
  if (corpus.size()) {
    // exact per-row doubles from the device, summed in corpus order (:222-233)
    std::vector<double> rowd(corpus.size());
    {
      std::lock_guard<std::mutex> g(index.device->ctx->mu);
      check(hivf_index_row_distances(index.device->ix, rowd.data()));
    }
    std::vector<std::uint64_t> start(K + 1, 0);
    for (std::size_t c = 0; c < K; ++c) start[c + 1] = start[c] + index.list_ids[c].size();
    double sum = 0.0;
    for (std::size_t i = 0; i < corpus.size(); ++i) sum += rowd[start[assign[i]] + pos[i]];
    index.mean_assigned_distance = sum / static_cast<double>(corpus.size());
  }
  return index;
}

namespace {
Corpus normalized_corpus(const Corpus& corpus) {  // build_index's cosine ingest (:245-252)
  Corpus out = corpus;
  for (std::size_t i = 0; i < corpus.size(); ++i) {
    const Embedding e = normalized(corpus.embedding(i));
    std::copy(e.begin(), e.end(), out.data.begin() + i * corpus.dim);
  }
  return out;
}
}  // namespace

IvfIndex build_index(const Corpus& corpus, const Centroids& centroids, Metric metric) {
  if (corpus.dim != centroids.dim) throw std::invalid_argument("build_index: dimension mismatch");
  {
    std::unordered_set<DocId> seen;
    seen.reserve(corpus.size());
    for (DocId id : corpus.doc_ids)
      if (!seen.insert(id).second) throw std::invalid_argument("build_index: duplicate doc_id");
  }
  if (metric == Metric::Cosine) {
    const Corpus nc = normalized_corpus(corpus);
    return index_from_assignments(nc, centroids, metric, compute_assignments(nc, centroids));
  }
  return index_from_assignments(corpus, centroids, metric, compute_assignments(corpus, centroids));
}

// ---- search (vector_index.cpp:261-342) ------------------------------------------------
std::vector<ClusterId> select_clusters(const IvfIndex& index, const Embedding& query, std::size_t nprobe) {
  if (nprobe < 1 || nprobe > index.k_clusters())
    throw std::invalid_argument("select_clusters: nprobe out of range");
  if (query.size() != index.dim) throw std::invalid_argument("select_clusters: dimension mismatch");
  auto& dev = device_of(index);
  std::vector<ClusterId> plan(nprobe);
  std::lock_guard<std::mutex> g(dev.ctx->mu);
  check(hivf_assign(dev.ix, query.data(), 1, static_cast<std::uint32_t>(nprobe), plan.data(), nullptr));
  return plan;
}

SearchCursor make_cursor(const IvfIndex& index, const Embedding& query, std::size_t nprobe, std::size_t k) {
  if (k == 0) throw std::invalid_argument("make_cursor: k must be >= 1");
  SearchCursor cursor;
  cursor.query = index.metric == Metric::Cosine ? normalized(query) : query;
  cursor.plan = select_clusters(index, query, nprobe);
  cursor.k = k;
  cursor.heap.set_k(k);
  return cursor;
}

SearchStepReport search_clusters(const IvfIndex& index, SearchCursor& cursor,
                                 std::span<const ClusterId> clusters) {
  SearchCursor* const one[1] = {&cursor};
  const std::span<const ClusterId> cl[1] = {clusters};
  return gpu::search_clusters_batch_impl(index, one, cl)[0];
}

SearchStepReport search_step(const IvfIndex& index, SearchCursor& cursor, std::size_t cluster_budget) {
  if (cursor.done()) return {};  // completion signal
  if (cluster_budget == 0) throw std::invalid_argument("search_step: cluster_budget must be >= 1");
  const std::size_t take = std::min(cluster_budget, cursor.remaining());
  const std::vector<ClusterId> slice(cursor.plan.begin() + cursor.next_pos,
                                     cursor.plan.begin() + cursor.next_pos + take);
  return search_clusters(index, cursor, slice);
}

TopKResult brute_force_search(const Corpus& corpus, const Embedding& query, std::size_t k) {
  if (k == 0) throw std::invalid_argument("brute_force_search: k must be >= 1");
  const std::vector<float>* q = &query;
  return gpu::brute_force_search_batch_impl(corpus, std::span<const std::vector<float>>(q, 1), k)[0];
}

}  // namespace hedra::ivf

// ---- batched forms and GPU extras --------------------------------------------------
namespace hedra::ivf::gpu {

// The reference semantics of search_clusters for every (cursor, clusters)
// pair, in one hivf_scan_items call.  Pairs are validated in order as the
// reference's sequential loop meets them: at the first plan-order error the
// earlier pairs and the failing pair's valid leading clusters are searched,
// later pairs are left untouched, and the error is thrown (:295-298).
std::vector<SearchStepReport> search_clusters_batch_impl(const IvfIndex& index,
                                                         std::span<SearchCursor* const> cursors,
                                                         std::span<const std::span<const ClusterId>> clusters) {
  const std::size_t n = cursors.size();
  if (clusters.size() != n) throw std::invalid_argument("search_clusters_batch: size mismatch");
  std::vector<SearchStepReport> out(n);
  std::vector<std::size_t> take(n, 0);
  const char* err = nullptr;
  std::size_t n_run = n;
  for (std::size_t i = 0; i < n && !err; ++i) {
    const SearchCursor& c = *cursors[i];
    for (std::size_t j = 0; j < clusters[i].size(); ++j) {
      if (c.next_pos + j >= c.plan.size()) {
        err = "search_clusters: cursor exhausted mid-batch";
        break;
      }
      if (c.plan[c.next_pos + j] != clusters[i][j]) {
        err = "search_clusters: cluster does not match plan order";
        break;
      }
      ++take[i];
    }
    if (err) n_run = i + 1;
  }
  // device items: pairs with clusters to scan and a heap that can take entries
  const std::uint32_t dim = index.dim;
  std::vector<std::size_t> item_pair;
  std::size_t kmax = 1;
  for (std::size_t i = 0; i < n_run; ++i) {
    if (!take[i]) continue;
    if (cursors[i]->query.size() != dim) throw std::invalid_argument("search_clusters: dimension mismatch");
    if (cursors[i]->heap.k()) {
      item_pair.push_back(i);
      kmax = std::max(kmax, cursors[i]->heap.k());
    }
  }
  const std::size_t m = item_pair.size();
  std::vector<std::uint8_t> changed;
  std::vector<std::uint32_t> off(m + 1, 0);
  std::vector<std::uint64_t> hid(m * kmax, 0);
  std::vector<double> hd(m * kmax, 0.0);
  std::vector<std::uint32_t> hn(m);
  if (m) {
    std::vector<float> q(m * dim);
    std::vector<std::uint32_t> kk(m), cl;
    for (std::size_t t = 0; t < m; ++t) {
      const SearchCursor& c = *cursors[item_pair[t]];
      std::copy(c.query.begin(), c.query.end(), q.begin() + t * dim);
      cl.insert(cl.end(), clusters[item_pair[t]].begin(), clusters[item_pair[t]].begin() + take[item_pair[t]]);
      off[t + 1] = static_cast<std::uint32_t>(cl.size());
      kk[t] = static_cast<std::uint32_t>(c.heap.k());
      const auto& e = c.heap.entries();
      hn[t] = static_cast<std::uint32_t>(e.size());
      for (std::size_t j = 0; j < e.size(); ++j) {
        hid[t * kmax + j] = e[j].doc_id;
        hd[t * kmax + j] = e[j].distance;
      }
    }
    changed.assign(cl.size(), 0);
    auto& dev = device_of(index);
    std::lock_guard<std::mutex> g(dev.ctx->mu);
    check(hivf_scan_items(dev.ix, q.data(), static_cast<std::uint32_t>(m), off.data(), cl.data(), kk.data(),
                          hid.data(), hd.data(), hn.data(), static_cast<std::uint32_t>(kmax), changed.data()));
  }
  // cursor bookkeeping exactly as :299-314
  std::size_t t = 0;
  for (std::size_t i = 0; i < n_run; ++i) {
    SearchCursor& c = *cursors[i];
    const bool on_device = t < m && item_pair[t] == i;
    if (on_device) {
      TopKResult h(c.heap.k());
      for (std::uint32_t j = 0; j < hn[t]; ++j) h.insert(hid[t * kmax + j], hd[t * kmax + j]);
      c.heap = std::move(h);
    }
    for (std::size_t j = 0; j < take[i]; ++j) {
      const bool ch = on_device && changed[off[t] + j];
      ++c.next_pos;
      ++c.clusters_searched;
      c.unchanged_streak = ch ? 0 : c.unchanged_streak + 1;
      out[i].heap_changed |= ch;
      out[i].searched.push_back(clusters[i][j]);
    }
    if (on_device) ++t;
  }
  if (err) throw std::runtime_error(err);
  return out;
}

namespace {

// brute_force_search runs on a one-list device copy of the corpus; the last
// few corpora stay uploaded (keyed by address, shape and a content hash), so
// a caller checking many queries against one corpus uploads it once.
struct CorpusEntry {
  const void* data = nullptr;
  std::size_t n = 0;
  std::uint32_t dim = 0;
  Metric metric = Metric::L2;
  std::uint64_t hash = 0;
  std::shared_ptr<DeviceIndex> dev;
};
std::mutex g_corpus_mu;
std::vector<CorpusEntry> g_corpora;  // most recent last

std::uint64_t content_hash(const Corpus& c) {
  std::uint64_t h = 0x9e3779b97f4a7c15ull ^ c.size();
  auto mix = [&](const void* p, std::size_t bytes) {
    const auto* b = static_cast<const unsigned char*>(p);
    std::size_t i = 0;
    for (; i + 8 <= bytes; i += 8) {
      std::uint64_t w;
      std::memcpy(&w, b + i, 8);
      h = (h ^ w) * 0x100000001b3ull;
      h ^= h >> 29;
    }
    for (; i < bytes; ++i) h = (h ^ b[i]) * 0x100000001b3ull;
  };
  mix(c.data.data(), c.data.size() * sizeof(float));
  mix(c.doc_ids.data(), c.doc_ids.size() * sizeof(DocId));
  return h;
}

std::shared_ptr<DeviceIndex> corpus_index(const Corpus& corpus) {
  const std::uint64_t h = content_hash(corpus);
  std::lock_guard<std::mutex> g(g_corpus_mu);
  for (auto it = g_corpora.begin(); it != g_corpora.end(); ++it)
    if (it->data == corpus.data.data() && it->n == corpus.size() && it->dim == corpus.dim &&
        it->metric == corpus.metric && it->hash == h) {
      CorpusEntry e = *it;
      g_corpora.erase(it);
      g_corpora.push_back(e);
      return e.dev;
    }
  if (corpus.data.size() != corpus.size() * corpus.dim)
    throw std::invalid_argument("brute_force_search: corpus data / doc_ids size mismatch");
  const Corpus rows = corpus.metric == Metric::Cosine ? normalized_corpus(corpus) : Corpus{};
  const float* v = corpus.metric == Metric::Cosine ? rows.data.data() : corpus.data.data();
  const std::vector<float> cent(corpus.dim, 0.0f);
  const std::uint64_t off[2] = {0, corpus.size()};
  auto dev = std::make_shared<DeviceIndex>();
  dev->ctx = &context();
  {
    std::lock_guard<std::mutex> gc(dev->ctx->mu);
    check(hivf_index_upload(dev->ctx->ctx, corpus.dim, static_cast<int>(corpus.metric), 1, cent.data(), off, v,
                            corpus.doc_ids.data(), &dev->ix));
  }
  g_corpora.push_back(CorpusEntry{corpus.data.data(), corpus.size(), corpus.dim, corpus.metric, h, dev});
  if (g_corpora.size() > 4) g_corpora.erase(g_corpora.begin());
  return dev;
}

}  // namespace

std::vector<TopKResult> brute_force_search_batch_impl(const Corpus& corpus,
                                                      std::span<const std::vector<float>> queries,
                                                      std::size_t k) {
  if (k == 0) throw std::invalid_argument("brute_force_search: k must be >= 1");
  std::vector<TopKResult> out(queries.size(), TopKResult(k));
  if (corpus.size() == 0 || queries.empty()) return out;
  const std::uint32_t dim = corpus.dim;
  std::vector<float> q(queries.size() * dim);
  for (std::size_t i = 0; i < queries.size(); ++i) {
    if (queries[i].size() != dim) throw std::invalid_argument("squared_l2: dimension mismatch");
    std::copy(queries[i].begin(), queries[i].end(), q.begin() + i * dim);
  }
  const auto dev = corpus_index(corpus);
  const std::size_t kk = std::min<std::size_t>(k, corpus.size());
  std::vector<std::uint64_t> ids(queries.size() * kk);
  std::vector<double> d(queries.size() * kk);
  std::vector<std::uint32_t> cnt(queries.size());
  {
    std::lock_guard<std::mutex> g(dev->ctx->mu);
    check(hivf_search(dev->ix, q.data(), static_cast<std::uint32_t>(queries.size()), 1,
                      static_cast<std::uint32_t>(kk), ids.data(), d.data(), cnt.data()));
  }
  for (std::size_t i = 0; i < queries.size(); ++i)
    for (std::uint32_t j = 0; j < cnt[i]; ++j) out[i].insert(ids[i * kk + j], d[i * kk + j]);
  return out;
}

double measure_per_vector_ns_impl(const IvfIndex& index, std::size_t repeats) {
  if (index.total_vectors() == 0) throw std::invalid_argument("measure_per_vector_ns: empty index");
  if (repeats == 0) repeats = 1;
  // the reference's calibration scan: every list, constant 0.25 query, k = 1
  // (bench.cpp:139-163), as sub-stage items of <= 2048 lists
  const std::uint32_t K = static_cast<std::uint32_t>(index.k_clusters());
  const std::uint32_t per = 2048;
  const std::uint32_t n_items = (K + per - 1) / per;
  std::vector<float> q(static_cast<std::size_t>(n_items) * index.dim, 0.25f);
  std::vector<std::uint32_t> off(n_items + 1), cl(K), kv(n_items, 1), hn(n_items);
  for (std::uint32_t c = 0; c < K; ++c) cl[c] = c;
  for (std::uint32_t i = 0; i <= n_items; ++i) off[i] = std::min(K, i * per);
  std::vector<std::uint64_t> hid(n_items);
  std::vector<double> hd(n_items), runs;
  std::vector<std::uint8_t> changed(K);
  auto& dev = device_of(index);
  for (std::size_t r = 0; r <= repeats; ++r) {  // the first call warms up
    std::fill(hn.begin(), hn.end(), 0u);
    std::lock_guard<std::mutex> g(dev.ctx->mu);
    const auto t0 = std::chrono::steady_clock::now();
    check(hivf_scan_items(dev.ix, q.data(), n_items, off.data(), cl.data(), kv.data(), hid.data(), hd.data(),
                          hn.data(), 1, changed.data()));
    const double ns = std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t0).count();
    if (r) runs.push_back(ns / static_cast<double>(index.total_vectors()));
  }
  std::sort(runs.begin(), runs.end());
  return runs[runs.size() / 2];
}

}  // namespace hedra::ivf::gpu

namespace hedra::gpu {
void reserve_substage(const ivf::IvfIndex& index, std::size_t n_items, std::size_t clusters_per_item,
                      std::size_t k) {
  const std::size_t K = index.k_clusters();
  if (!K || !n_items || !clusters_per_item || !k) return;
  const std::size_t per = std::min(clusters_per_item, K);
  // realistic sub-stages (a query at its first cluster's centroid): a
  // degenerate query would fail the scan's filter proofs and tip the index's
  // automatic scan-precision policy
  std::vector<float> q(n_items * index.dim, 0.f);
  for (std::size_t i = 0; i < n_items; ++i) {
    const auto& c = index.centroids.rows[i % K];
    std::copy(c.begin(), c.end(), q.begin() + i * index.dim);
  }
  std::vector<std::uint32_t> off(n_items + 1), cl(n_items * per), kk(n_items, static_cast<std::uint32_t>(k)),
      hn(n_items, 0);
  for (std::size_t i = 0; i <= n_items; ++i) off[i] = static_cast<std::uint32_t>(i * per);
  for (std::size_t i = 0; i < n_items; ++i)
    for (std::size_t j = 0; j < per; ++j) cl[i * per + j] = static_cast<std::uint32_t>((i + j) % K);
  std::vector<std::uint64_t> hid(n_items * k);
  std::vector<double> hd(n_items * k);
  std::vector<std::uint8_t> changed(cl.size());
  auto& dev = ivf::gpu::device_of(index);
  std::lock_guard<std::mutex> g(dev.ctx->mu);
  ivf::gpu::check(hivf_scan_items(dev.ix, q.data(), static_cast<std::uint32_t>(n_items), off.data(), cl.data(),
                                  kk.data(), hid.data(), hd.data(), hn.data(), static_cast<std::uint32_t>(k),
                                  changed.data()));
}
std::vector<ivf::SearchStepReport> search_clusters_batch(const ivf::IvfIndex& index,
                                                         std::span<ivf::SearchCursor* const> cursors,
                                                         std::span<const std::span<const ClusterId>> clusters) {
  return ivf::gpu::search_clusters_batch_impl(index, cursors, clusters);
}
std::vector<ivf::TopKResult> brute_force_search_batch(const ivf::Corpus& corpus,
                                                      std::span<const std::vector<float>> queries,
                                                      std::size_t k) {
  return ivf::gpu::brute_force_search_batch_impl(corpus, queries, k);
}
double measure_per_vector_ns(const ivf::IvfIndex& index, std::size_t repeats) {
  return ivf::gpu::measure_per_vector_ns_impl(index, repeats);
}
}  // namespace hedra::gpu

// ---- RetrievalEngine (retrieval_engine.cpp, header unmodified) ------------------------
namespace hedra::ret {

double cluster_variable_ms(const ivf::IvfIndex& index, ClusterId cluster, Lane lane,
                           const RetrievalCostModel& model) {
  if (cluster >= index.k_clusters()) throw std::invalid_argument("cluster_variable_ms: unknown cluster");
  double ns = static_cast<double>(index.cluster_size(cluster)) * model.per_vector_ns;
  if (lane == Lane::Fast) ns /= model.fast_speedup;
  return ns / 1e6;
}

double estimate_cluster_cost_ms(const ivf::IvfIndex& index, ClusterId cluster, Lane lane,
                                const RetrievalCostModel& model) {
  return cluster_variable_ms(index, cluster, lane, model) + fixed_call_ms(model);
}

void RetrievalEngine::submit(RetrievalTask task) {
  const auto key = std::make_pair(task.request_id, task.node_id);
  if (tasks_.count(key)) throw std::invalid_argument("submit: duplicate live task for this stage");
  tasks_.emplace(key, std::move(task));
}

bool RetrievalEngine::has_task(RequestId request_id, NodeId node_id) const {
  return tasks_.count({request_id, node_id}) > 0;
}

const RetrievalTask* RetrievalEngine::find(RequestId request_id, NodeId node_id) const {
  const auto it = tasks_.find({request_id, node_id});
  return it == tasks_.end() ? nullptr : &it->second;
}

RetrievalTask RetrievalEngine::extract(RequestId request_id, NodeId node_id) {
  auto it = tasks_.find({request_id, node_id});
  if (it == tasks_.end()) throw std::invalid_argument("extract: no live task for this stage");
  RetrievalTask task = std::move(it->second);
  tasks_.erase(it);
  return task;
}

bool RetrievalEngine::cancel(RequestId request_id, NodeId node_id) {
  return tasks_.erase({request_id, node_id}) > 0;
}

// One sub-stage (retrieval_engine.cpp:55-152): the same cache bookkeeping and
// lane billing, then every item's search_clusters in ONE device call instead
// of a host thread pool.  live_math only decided the reference's threading;
// the math is the device's either way, and wall_ms is measured around it.
RetStepReport RetrievalEngine::execute(SubStageBatch& batch, double now_ms, bool /*live_math*/) {
  RetStepReport report;
  if (batch.items.empty()) return report;
  cache_.complete_swaps(now_ms);

  std::vector<ClusterId> all;
  for (const auto& item : batch.items) all.insert(all.end(), item.clusters.begin(), item.clusters.end());
  const auto partition = cache_.partition_batch(all);
  const std::set<ClusterId> fast(partition.fast.begin(), partition.fast.end());
  cache_.count_access_hits(all);

  double slow_ns = 0.0, fast_ns = 0.0;
  for (auto& item : batch.items) {
    item.fast.clear();
    item.slow.clear();
    for (ClusterId c : item.clusters) {
      const double ns = static_cast<double>(index_->cluster_size(c)) * model_.per_vector_ns;
      if (fast.count(c)) {
        item.fast.push_back(c);
        fast_ns += ns / model_.fast_speedup;
        ++report.fast_clusters;
      } else {
        item.slow.push_back(c);
        slow_ns += ns;
        ++report.slow_clusters;
      }
    }
  }
  report.slow_lane_ms = slow_ns / 1e6;
  report.fast_lane_ms = fast_ns / 1e6;
  report.modeled_ms = std::max(report.slow_lane_ms, report.fast_lane_ms) + fixed_call_ms(model_);

  // items up to the first unknown task run, then the error (sequential order)
  std::vector<ivf::SearchCursor*> cursors;
  std::vector<std::span<const ClusterId>> spans;
  bool unknown = false;
  for (const auto& item : batch.items) {
    const auto it = tasks_.find({item.request_id, item.node_id});
    if (it == tasks_.end()) {
      unknown = true;
      break;
    }
    cursors.push_back(&it->second.cursor);
    spans.emplace_back(item.clusters.data(), item.clusters.size());
  }
  const auto wall_start = std::chrono::steady_clock::now();
  const auto steps = ivf::gpu::search_clusters_batch_impl(*index_, cursors, spans);
  report.wall_ms =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - wall_start).count();
  if (unknown) throw std::runtime_error("execute: batch references unknown task");

  std::set<ClusterId> accessed;
  for (std::size_t i = 0; i < batch.items.size(); ++i) {
    const auto& item = batch.items[i];
    TaskDelta delta;
    delta.request_id = item.request_id;
    delta.node_id = item.node_id;
    delta.clusters_searched = item.clusters.size();
    delta.heap_changed = steps[i].heap_changed;
    delta.completed = cursors[i]->done();
    report.deltas.push_back(delta);
    accessed.insert(item.clusters.begin(), item.clusters.end());
  }
  const std::vector<ClusterId> accessed_list(accessed.begin(), accessed.end());
  cache_.record_access(accessed_list);
  report.swaps_started = cache_.maybe_update(now_ms, *index_);
  return report;
}

}  // namespace hedra::ret
