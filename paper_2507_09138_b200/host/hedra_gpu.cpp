// hedra_gpu.cpp -- host side of the drop-in (see hedra_gpu.hpp).  Bookkeeping
// only; every distance, scan and selection is a libhivf (sm_100a) call.
#include "hedra_gpu.hpp"
#include "hvec_io.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <numeric>

namespace hedra_gpu {

double squared_l2(const float* a, const float* b, std::size_t dim) {
  double acc = 0.0;
  for (std::size_t i = 0; i < dim; ++i) {
    const double d = static_cast<double>(a[i]) - static_cast<double>(b[i]);
    acc += d * d;
  }
  return acc;
}

double embedding_distance(const Embedding& a, const Embedding& b) {
  if (a.size() != b.size()) throw std::invalid_argument("squared_l2: dimension mismatch");
  return squared_l2(a.data(), b.data(), a.size());
}

Embedding normalized(Embedding v) {
  double norm = 0.0;
  for (float x : v) norm += static_cast<double>(x) * static_cast<double>(x);
  norm = std::sqrt(norm);
  if (norm == 0.0) return v;
  for (float& x : v) x = static_cast<float>(static_cast<double>(x) / norm);
  return v;
}

void check(hivf_status st) {
  if (st == HIVF_OK) return;
  const std::string msg = hivf_last_error();
  if (st == HIVF_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

namespace ivf {

// ---- TopKResult ------------------------------------------------------------
void TopKResult::set_k(std::size_t k) {
  k_ = k;
  if (entries_.size() > k_) entries_.resize(k_);
}

bool TopKResult::insert(DocId doc_id, double distance) {
  if (k_ == 0) return false;
  auto same = std::find_if(entries_.begin(), entries_.end(),
                           [&](const TopKEntry& e) { return e.doc_id == doc_id; });
  if (same != entries_.end()) {
    if (!(distance < same->distance)) return false;  // keep the minimum
    entries_.erase(same);
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

std::vector<DocId> TopKResult::doc_ids() const {
  std::vector<DocId> out(entries_.size());
  std::transform(entries_.begin(), entries_.end(), out.begin(),
                 [](const TopKEntry& e) { return e.doc_id; });
  return out;
}

bool TopKResult::operator==(const TopKResult& o) const {
  if (entries_.size() != o.entries_.size()) return false;
  for (std::size_t i = 0; i < entries_.size(); ++i)
    if (entries_[i].doc_id != o.entries_[i].doc_id || entries_[i].distance != o.entries_[i].distance)
      return false;
  return true;
}

void TopKResult::assign_sorted(const std::uint64_t* ids, const double* d, std::size_t n) {
  entries_.resize(n);
  for (std::size_t i = 0; i < n; ++i) entries_[i] = TopKEntry{ids[i], d[i]};
}

TopKResult merge_topk(const TopKResult& a, const TopKResult& b, std::size_t k) {
  // best distance per id, then (distance, id) order, first k
  std::map<DocId, double> best;
  for (const auto* r : {&a, &b})
    for (const auto& e : r->entries()) {
      auto it = best.find(e.doc_id);
      if (it == best.end() || e.distance < it->second) best[e.doc_id] = e.distance;
    }
  std::vector<TopKEntry> all;
  all.reserve(best.size());
  for (const auto& [id, d] : best) all.push_back(TopKEntry{id, d});
  std::sort(all.begin(), all.end(), topk_less);
  TopKResult out(k);
  for (std::size_t i = 0; i < all.size() && i < k; ++i) out.insert(all[i].doc_id, all[i].distance);
  return out;
}

// ---- Context / IvfIndex ---------------------------------------------------------
Context::Context(int device, void* stream) { check(hivf_ctx_create(device, stream, &ctx_)); }
Context::~Context() { hivf_ctx_destroy(ctx_); }

std::shared_ptr<IvfIndex> IvfIndex::from_assignments(Context& ctx, const std::vector<float>& corpus,
                                                     const std::vector<DocId>& ids, std::uint32_t dim,
                                                     Metric metric,
                                                     const std::vector<std::vector<float>>& centroids,
                                                     const std::vector<ClusterId>& assign) {
  if (assign.size() != ids.size() || corpus.size() != ids.size() * dim)
    throw std::invalid_argument("index_from_assignments: assignment count mismatch");
  const std::size_t K = centroids.size();
  std::vector<std::uint64_t> off(K + 1, 0);
  for (ClusterId c : assign) {
    if (c >= K) throw std::invalid_argument("index_from_assignments: cluster id out of range");
    ++off[c + 1];
  }
  std::partial_sum(off.begin(), off.end(), off.begin());
  std::vector<std::uint64_t> cursor(off.begin(), off.end() - 1);
  std::vector<float> rows(corpus.size());
  std::vector<DocId> lids(ids.size());
  for (std::size_t i = 0; i < ids.size(); ++i) {  // stable: corpus order inside a list
    const std::uint64_t r = cursor[assign[i]]++;
    std::copy(corpus.begin() + i * dim, corpus.begin() + (i + 1) * dim, rows.begin() + r * dim);
    lids[r] = ids[i];
  }
  std::vector<float> cents;
  cents.reserve(K * dim);
  for (const auto& c : centroids) {
    if (c.size() != dim) throw std::invalid_argument("build_index: dimension mismatch");
    cents.insert(cents.end(), c.begin(), c.end());
  }
  auto ix = std::shared_ptr<IvfIndex>(new IvfIndex);
  ix->ctx_ = &ctx;
  ix->dim_ = dim;
  ix->metric_ = metric;
  ix->total_ = ids.size();
  ix->sizes_.resize(K);
  for (std::size_t c = 0; c < K; ++c) ix->sizes_[c] = off[c + 1] - off[c];
  ix->offsets_.assign(off.begin(), off.end());
  check(hivf_index_upload(ctx.raw(), dim, static_cast<int>(metric), static_cast<std::uint32_t>(K),
                          cents.data(), off.data(), rows.data(), lids.data(), &ix->ix_));
  return ix;
}

IvfIndex::~IvfIndex() { hivf_index_destroy(ix_); }

std::optional<IvfIndex::DocLocation> IvfIndex::locate(DocId id) const {
  std::uint32_t c = 0;
  std::uint64_t row = 0;
  check(hivf_index_locate(ix_, &id, 1, &c, &row));
  if (c == 0xffffffffu) return std::nullopt;
  return DocLocation{c, static_cast<std::uint32_t>(row - offsets_[c])};
}

Embedding IvfIndex::doc_embedding(DocLocation loc) const {
  if (loc.cluster >= sizes_.size() || loc.offset >= sizes_[loc.cluster])
    throw std::out_of_range("doc_embedding: location out of range");
  const std::uint64_t row = offsets_[loc.cluster] + loc.offset;
  Embedding e(dim_);
  check(hivf_index_gather_rows(ix_, &row, 1, e.data()));
  return e;
}

double IvfIndex::mean_assigned_distance() const {
  double m = 0.0;
  check(hivf_index_info(ix_, nullptr, nullptr, nullptr, nullptr, &m));
  return m;
}

// ---- persistence (HVEC / u32, vector_index.cpp:344-473 formats) -----------------------
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

// ---- index build ------------------------------------------------------------------
Centroids train_kmeans(Context& ctx, const Corpus& corpus, std::size_t k_clusters, std::size_t max_iters,
                       std::uint64_t seed) {
  if (corpus.size() < k_clusters) throw std::invalid_argument("train_kmeans: corpus smaller than k_clusters");
  if (k_clusters == 0) throw std::invalid_argument("train_kmeans: k_clusters must be >= 1");
  if (max_iters == 0) throw std::invalid_argument("train_kmeans: max_iters must be >= 1");
  std::vector<float> out(k_clusters * corpus.dim);
  check(hivf_train_kmeans_host(ctx.raw(), corpus.data.data(), corpus.size(), corpus.dim,
                               static_cast<std::uint32_t>(k_clusters), static_cast<std::uint32_t>(max_iters),
                               seed, out.data()));
  Centroids c;
  c.dim = corpus.dim;
  for (std::size_t r = 0; r < k_clusters; ++r)
    c.rows.emplace_back(out.begin() + r * corpus.dim, out.begin() + (r + 1) * corpus.dim);
  return c;
}

std::vector<ClusterId> compute_assignments(Context& ctx, const Corpus& corpus, const Centroids& centroids) {
  std::vector<float> cents;
  for (const auto& r : centroids.rows) {
    if (r.size() != corpus.dim) throw std::invalid_argument("build_index: dimension mismatch");
    cents.insert(cents.end(), r.begin(), r.end());
  }
  std::vector<ClusterId> a(corpus.size());
  check(hivf_compute_assignments_host(ctx.raw(), corpus.data.data(), corpus.size(), corpus.dim, cents.data(),
                                      static_cast<std::uint32_t>(centroids.k_clusters()), a.data()));
  return a;
}

std::shared_ptr<IvfIndex> build_index(Context& ctx, const Corpus& corpus, const Centroids& centroids,
                                      Metric metric) {
  if (corpus.dim != centroids.dim) throw std::invalid_argument("build_index: dimension mismatch");
  if (metric == Metric::Cosine) {  // vector_index.cpp:245-252
    Corpus nc = corpus;
    for (std::size_t i = 0; i < corpus.size(); ++i) {
      Embedding e = normalized(corpus.embedding(i));
      std::copy(e.begin(), e.end(), nc.data.begin() + i * corpus.dim);
    }
    return IvfIndex::from_assignments(ctx, nc.data, nc.doc_ids, nc.dim, metric, centroids.rows,
                                      compute_assignments(ctx, nc, centroids));
  }
  // duplicate doc ids -> invalid_argument (vector_index.cpp:240-244) in hivf_index_finish
  return IvfIndex::from_assignments(ctx, corpus.data, corpus.doc_ids, corpus.dim, metric, centroids.rows,
                                    compute_assignments(ctx, corpus, centroids));
}

// ---- search API ---------------------------------------------------------------
std::vector<ClusterId> select_clusters(const IvfIndex& index, const Embedding& query,
                                       std::size_t nprobe) {
  if (nprobe < 1 || nprobe > index.k_clusters())
    throw std::invalid_argument("select_clusters: nprobe out of range");
  if (query.size() != index.dim()) throw std::invalid_argument("select_clusters: dimension mismatch");
  std::vector<ClusterId> plan(nprobe);
  check(hivf_assign(index.raw(), query.data(), 1, static_cast<std::uint32_t>(nprobe), plan.data(),
                    nullptr));
  return plan;
}

SearchCursor make_cursor(const IvfIndex& index, const Embedding& query, std::size_t nprobe,
                         std::size_t k) {
  if (k == 0) throw std::invalid_argument("make_cursor: k must be >= 1");
  SearchCursor c;
  c.query = index.metric() == Metric::Cosine ? normalized(query) : query;
  c.plan = select_clusters(index, query, nprobe);
  c.k = k;
  c.heap.set_k(k);
  return c;
}

std::vector<SearchStepReport> search_clusters_batch(
    const IvfIndex& index, const std::vector<SearchCursor*>& cursors,
    const std::vector<std::span<const ClusterId>>& clusters) {
  const std::size_t n = cursors.size();
  if (clusters.size() != n) throw std::invalid_argument("search_clusters_batch: size mismatch");
  std::vector<SearchStepReport> out(n);
  if (n == 0) return out;
  // Pairs are validated in order, as the reference's sequential loop meets
  // them (vector_index.cpp:295-298): at the first plan-order error, the earlier
  // pairs and the failing pair's valid leading clusters are searched, later
  // pairs are left untouched, then the error is thrown.
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
  std::vector<std::size_t> item;  // pairs with clusters to scan and a heap that takes entries
  std::size_t kmax = 1;
  for (std::size_t i = 0; i < n_run; ++i) {
    if (!take[i] || !cursors[i]->heap.k()) continue;
    if (cursors[i]->query.size() != index.dim()) throw std::invalid_argument("search_clusters: dimension mismatch");
    item.push_back(i);
    kmax = std::max(kmax, cursors[i]->heap.k());
  }
  const std::size_t m = item.size();
  const std::uint32_t dim = index.dim();
  std::vector<std::uint32_t> off(m + 1, 0), hn(m);
  std::vector<std::uint64_t> hid(m * kmax, 0);
  std::vector<double> hd(m * kmax, 0.0);
  std::vector<std::uint8_t> changed;
  if (m) {
    std::vector<float> q(m * dim);
    std::vector<std::uint32_t> kk(m), cl;
    for (std::size_t t = 0; t < m; ++t) {
      const SearchCursor& c = *cursors[item[t]];
      std::copy(c.query.begin(), c.query.end(), q.begin() + t * dim);
      cl.insert(cl.end(), clusters[item[t]].begin(), clusters[item[t]].begin() + take[item[t]]);
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
    check(hivf_scan_items(index.raw(), q.data(), static_cast<std::uint32_t>(m), off.data(), cl.data(),
                          kk.data(), hid.data(), hd.data(), hn.data(), static_cast<std::uint32_t>(kmax),
                          changed.data()));
  }
  std::size_t t = 0;
  for (std::size_t i = 0; i < n_run; ++i) {
    SearchCursor& c = *cursors[i];
    const bool on_device = t < m && item[t] == i;
    if (on_device) c.heap.assign_sorted(hid.data() + t * kmax, hd.data() + t * kmax, hn[t]);
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

SearchStepReport search_clusters(const IvfIndex& index, SearchCursor& cursor,
                                 std::span<const ClusterId> clusters) {
  return search_clusters_batch(index, {&cursor}, {clusters})[0];
}

SearchStepReport search_step(const IvfIndex& index, SearchCursor& cursor,
                             std::size_t cluster_budget) {
  if (cursor.done()) return {};
  if (cluster_budget == 0) throw std::invalid_argument("search_step: cluster_budget must be >= 1");
  const std::size_t take = std::min(cluster_budget, cursor.remaining());
  const std::vector<ClusterId> slice(cursor.plan.begin() + cursor.next_pos,
                                     cursor.plan.begin() + cursor.next_pos + take);
  return search_clusters(index, cursor, slice);
}

std::vector<TopKResult> search(const IvfIndex& index, const std::vector<Embedding>& queries,
                               std::size_t nprobe, std::size_t k) {
  if (k == 0) throw std::invalid_argument("make_cursor: k must be >= 1");
  const std::uint32_t dim = index.dim();
  const std::size_t n = queries.size();
  std::vector<float> q(n * dim);
  for (std::size_t i = 0; i < n; ++i) {
    if (queries[i].size() != dim) throw std::invalid_argument("select_clusters: dimension mismatch");
    std::copy(queries[i].begin(), queries[i].end(), q.begin() + i * dim);
  }
  std::vector<std::uint64_t> ids(n * k);
  std::vector<double> d(n * k);
  std::vector<std::uint32_t> cnt(n);
  if (n)
    check(hivf_search(index.raw(), q.data(), static_cast<std::uint32_t>(n),
                      static_cast<std::uint32_t>(nprobe), static_cast<std::uint32_t>(k), ids.data(),
                      d.data(), cnt.data()));
  std::vector<TopKResult> out(n, TopKResult(k));
  for (std::size_t i = 0; i < n; ++i) out[i].assign_sorted(ids.data() + i * k, d.data() + i * k, cnt[i]);
  return out;
}

std::vector<TopKResult> brute_force_search(Context& ctx, const Corpus& corpus,
                                           const std::vector<Embedding>& queries, std::size_t k) {
  if (k == 0) throw std::invalid_argument("brute_force_search: k must be >= 1");
  std::vector<TopKResult> out(queries.size(), TopKResult(k));
  if (corpus.size() == 0 || queries.empty()) return out;
  if (corpus.data.size() != corpus.size() * corpus.dim)
    throw std::invalid_argument("brute_force_search: corpus data / doc_ids size mismatch");
  const std::uint32_t dim = corpus.dim;
  std::vector<float> rows;
  const float* v = corpus.data.data();
  if (corpus.metric == Metric::Cosine) {  // the reference normalizes every row it scores
    rows.resize(corpus.data.size());
    for (std::size_t i = 0; i < corpus.size(); ++i) {
      const Embedding e = normalized(corpus.embedding(i));
      std::copy(e.begin(), e.end(), rows.begin() + i * dim);
    }
    v = rows.data();
  }
  const std::vector<float> cent(dim, 0.0f);
  const std::uint64_t off[2] = {0, corpus.size()};
  hivf_index* ix = nullptr;
  check(hivf_index_upload(ctx.raw(), dim, static_cast<int>(corpus.metric), 1, cent.data(), off, v,
                          corpus.doc_ids.data(), &ix));
  std::vector<float> q(queries.size() * dim);
  for (std::size_t i = 0; i < queries.size(); ++i) {
    if (queries[i].size() != dim) {
      hivf_index_destroy(ix);
      throw std::invalid_argument("squared_l2: dimension mismatch");
    }
    std::copy(queries[i].begin(), queries[i].end(), q.begin() + i * dim);
  }
  const std::size_t kk = std::min<std::size_t>(k, corpus.size());
  std::vector<std::uint64_t> ids(queries.size() * kk);
  std::vector<double> d(queries.size() * kk);
  std::vector<std::uint32_t> cnt(queries.size());
  const hivf_status st = hivf_search(ix, q.data(), static_cast<std::uint32_t>(queries.size()), 1,
                                     static_cast<std::uint32_t>(kk), ids.data(), d.data(), cnt.data());
  hivf_index_destroy(ix);
  check(st);
  for (std::size_t i = 0; i < queries.size(); ++i) out[i].assign_sorted(ids.data() + i * kk, d.data() + i * kk, cnt[i]);
  return out;
}

TopKResult brute_force_search(Context& ctx, const Corpus& corpus, const Embedding& query, std::size_t k) {
  return brute_force_search(ctx, corpus, std::vector<Embedding>{query}, k)[0];
}

}  // namespace ivf

// ---- cache::ClusterCacheState ------------------------------------------------------
namespace cache {

void ClusterCacheState::record_access(std::span<const ClusterId> cluster_ids) {
  for (ClusterId c : std::set<ClusterId>(cluster_ids.begin(), cluster_ids.end())) freq_[c] += 1.0;
  ++since_update_;
}

std::vector<SwapOp> ClusterCacheState::maybe_update(double now_ms, const ivf::IvfIndex& index) {
  if (cfg_.capacity_gc == 0 || since_update_ < cfg_.update_interval || !in_flight_.empty()) return {};
  since_update_ = 0;
  std::vector<std::pair<double, ClusterId>> by_freq;
  for (const auto& [c, f] : freq_) by_freq.emplace_back(f, c);
  std::sort(by_freq.begin(), by_freq.end(), [](const auto& x, const auto& y) {
    return x.first != y.first ? x.first > y.first : x.second < y.second;  // ties: lower id
  });
  std::set<ClusterId> want;
  for (std::size_t i = 0; i < by_freq.size() && want.size() < cfg_.capacity_gc; ++i)
    want.insert(by_freq[i].second);
  const double bytes_per_ms = cfg_.transfer_bandwidth_gb_s * 1e6;
  std::vector<SwapOp> plan;
  auto enqueue = [&](ClusterId c, bool inbound) {
    const double bytes = static_cast<double>(index.cluster_size(c)) * index.dim() * sizeof(float);
    const double start = std::max(now_ms, link_free_at_ms_);
    plan.push_back(SwapOp{c, inbound, start + bytes / bytes_per_ms});
    link_free_at_ms_ = plan.back().completes_at_ms;
    ++swaps_;
  };
  std::vector<ClusterId> out, in;
  for (ClusterId c : resident_)
    if (!want.count(c)) out.push_back(c);
  for (ClusterId c : want)
    if (!resident_.count(c)) in.push_back(c);
  for (ClusterId c : out) {  // evictions leave residency at once
    resident_.erase(c);
    enqueue(c, false);
    dirty_ = true;
  }
  for (ClusterId c : in) enqueue(c, true);
  in_flight_ = plan;
  for (auto& kv : freq_) kv.second *= cfg_.decay;
  return plan;
}

void ClusterCacheState::complete_swaps(double now_ms) {
  std::vector<SwapOp> keep;
  for (const auto& op : in_flight_) {
    if (op.completes_at_ms <= now_ms) {
      if (op.inbound) {
        resident_.insert(op.cluster);
        dirty_ = true;
      }
    } else {
      keep.push_back(op);
    }
  }
  in_flight_.swap(keep);
}

LanePartition ClusterCacheState::partition_batch(std::span<const ClusterId> clusters) const {
  LanePartition p;
  std::set<ClusterId> hot;
  if (cfg_.capacity_gc)
    for (ClusterId c : clusters)
      if (resident_.count(c)) hot.insert(c);
  if (cfg_.capacity_gc == 0 || hot.size() < cfg_.min_fast_clusters) {
    p.slow.assign(clusters.begin(), clusters.end());
    return p;
  }
  for (ClusterId c : clusters) (hot.count(c) ? p.fast : p.slow).push_back(c);
  return p;
}

void ClusterCacheState::count_access_hits(std::span<const ClusterId> clusters) {
  for (ClusterId c : std::set<ClusterId>(clusters.begin(), clusters.end()))
    (resident_.count(c) ? hits_ : misses_) += 1;
}

void ClusterCacheState::apply_to(const ivf::IvfIndex& index) {
  if (!dirty_) return;
  const std::vector<ClusterId> res(resident_.begin(), resident_.end());
  check(hivf_residency_set(index.raw(), res.data(), static_cast<std::uint32_t>(res.size())));
  dirty_ = false;
}

}  // namespace cache

// ---- ret::RetrievalEngine ----------------------------------------------------------
namespace ret {

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

bool RetrievalEngine::has_task(RequestId r, NodeId n) const { return tasks_.count({r, n}) > 0; }

const RetrievalTask* RetrievalEngine::find(RequestId r, NodeId n) const {
  const auto it = tasks_.find({r, n});
  return it == tasks_.end() ? nullptr : &it->second;
}

RetrievalTask RetrievalEngine::extract(RequestId r, NodeId n) {
  auto it = tasks_.find({r, n});
  if (it == tasks_.end()) throw std::invalid_argument("extract: no live task for this stage");
  RetrievalTask t = std::move(it->second);
  tasks_.erase(it);
  return t;
}

bool RetrievalEngine::cancel(RequestId r, NodeId n) { return tasks_.erase({r, n}) > 0; }

RetStepReport RetrievalEngine::execute(SubStageBatch& batch, double now_ms, bool /*live_math*/) {
  RetStepReport rep;
  if (batch.items.empty()) return rep;
  cache_.complete_swaps(now_ms);
  cache_.apply_to(*index_);
  std::vector<ClusterId> all;
  for (const auto& it : batch.items) all.insert(all.end(), it.clusters.begin(), it.clusters.end());
  const auto part = cache_.partition_batch(all);
  const std::set<ClusterId> fast(part.fast.begin(), part.fast.end());
  cache_.count_access_hits(all);
  double slow_ns = 0.0, fast_ns = 0.0;  // modeled lane billing, as the reference bills it
  for (auto& it : batch.items) {
    it.fast.clear();
    it.slow.clear();
    for (ClusterId c : it.clusters) {
      const double ns = static_cast<double>(index_->cluster_size(c)) * model_.per_vector_ns;
      if (fast.count(c)) {
        it.fast.push_back(c);
        fast_ns += ns / model_.fast_speedup;
        ++rep.fast_clusters;
      } else {
        it.slow.push_back(c);
        slow_ns += ns;
        ++rep.slow_clusters;
      }
    }
  }
  rep.slow_lane_ms = slow_ns / 1e6;
  rep.fast_lane_ms = fast_ns / 1e6;
  rep.modeled_ms = std::max(rep.slow_lane_ms, rep.fast_lane_ms) + fixed_call_ms(model_);
  // items up to the first unknown task run, then the error (the reference's
  // sequential item order, retrieval_engine.cpp:94-100)
  std::vector<ivf::SearchCursor*> cursors;
  std::vector<std::span<const ClusterId>> spans;
  bool unknown = false;
  for (const auto& it : batch.items) {
    auto t = tasks_.find({it.request_id, it.node_id});
    if (t == tasks_.end()) {
      unknown = true;
      break;
    }
    cursors.push_back(&t->second.cursor);
    spans.emplace_back(it.clusters.data(), it.clusters.size());
  }
  const auto t0 = std::chrono::steady_clock::now();
  const auto steps = ivf::search_clusters_batch(*index_, cursors, spans);  // one GPU sub-stage
  rep.wall_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (unknown) throw std::runtime_error("execute: batch references unknown task");
  std::set<ClusterId> accessed;
  for (std::size_t i = 0; i < batch.items.size(); ++i) {
    const auto& it = batch.items[i];
    rep.deltas.push_back(TaskDelta{it.request_id, it.node_id, it.clusters.size(),
                                   steps[i].heap_changed, cursors[i]->done()});
    accessed.insert(it.clusters.begin(), it.clusters.end());
  }
  const std::vector<ClusterId> acc(accessed.begin(), accessed.end());
  cache_.record_access(acc);
  rep.swaps_started = cache_.maybe_update(now_ms, *index_);
  cache_.apply_to(*index_);
  return rep;
}

}  // namespace ret
}  // namespace hedra_gpu

// ---- bench (bench.cpp:139-163) ------------------------------------------------------
namespace hedra_gpu {
namespace bench {

double measure_per_vector_ns(const ivf::IvfIndex& index, std::size_t repeats) {
  if (index.total_vectors() == 0) throw std::invalid_argument("measure_per_vector_ns: empty index");
  if (repeats == 0) repeats = 1;
  const std::uint32_t K = static_cast<std::uint32_t>(index.k_clusters());
  const std::uint32_t per = 2048;
  const std::uint32_t n_items = (K + per - 1) / per;
  std::vector<float> q(static_cast<std::size_t>(n_items) * index.dim(), 0.25f);
  std::vector<std::uint32_t> off(n_items + 1), cl(K), kv(n_items, 1);
  for (std::uint32_t c = 0; c < K; ++c) cl[c] = c;
  for (std::uint32_t i = 0; i <= n_items; ++i) off[i] = std::min(K, i * per);
  std::vector<std::uint64_t> hid(n_items);
  std::vector<double> hd(n_items);
  std::vector<std::uint32_t> hn(n_items);
  std::vector<std::uint8_t> changed(K);
  std::vector<double> runs;
  for (std::size_t r = 0; r <= repeats; ++r) {  // the first call is a warm-up
    std::fill(hn.begin(), hn.end(), 0u);
    const auto t0 = std::chrono::steady_clock::now();
    check(hivf_scan_items(index.raw(), q.data(), n_items, off.data(), cl.data(), kv.data(), hid.data(),
                          hd.data(), hn.data(), 1, changed.data()));
    const double ns = std::chrono::duration<double, std::nano>(std::chrono::steady_clock::now() - t0).count();
    if (r) runs.push_back(ns / static_cast<double>(index.total_vectors()));
  }
  std::sort(runs.begin(), runs.end());
  return runs[runs.size() / 2];
}

}  // namespace bench
}  // namespace hedra_gpu

// ---- sim (similarity.cpp) -----------------------------------------------------------
namespace hedra_gpu {
namespace sim {

void LocalityCache::record_search(RequestId request_id, LocalityRecord record) {
  records_[request_id] = std::move(record);
}
const LocalityRecord* LocalityCache::find(RequestId request_id) const {
  auto it = records_.find(request_id);
  return it == records_.end() ? nullptr : &it->second;
}
void LocalityCache::evict(RequestId request_id) { records_.erase(request_id); }

LocalityRecord make_locality_record(const ivf::IvfIndex& index, const Embedding& query,
                                    const ivf::TopKResult& extended_topk,
                                    std::span<const ClusterId> searched_plan) {
  LocalityRecord record;
  record.query = query;
  record.searched.insert(searched_plan.begin(), searched_plan.end());
  const auto& en = extended_topk.entries();
  const std::uint32_t n = static_cast<std::uint32_t>(en.size());
  if (!n) return record;
  std::vector<std::uint64_t> ids(n), rows(n);
  std::vector<std::uint32_t> cl(n);
  for (std::uint32_t i = 0; i < n; ++i) ids[i] = en[i].doc_id;
  check(hivf_index_locate(index.raw(), ids.data(), n, cl.data(), rows.data()));
  for (std::uint32_t i = 0; i < n; ++i)
    if (cl[i] == 0xffffffffu) throw std::invalid_argument("make_locality_record: unknown doc id");
  std::vector<float> vec(static_cast<std::size_t>(n) * index.dim());
  check(hivf_index_gather_rows(index.raw(), rows.data(), n, vec.data()));
  for (std::uint32_t i = 0; i < n; ++i) {
    record.candidates.push_back(CachedCandidate{
        ids[i], cl[i], Embedding(vec.begin() + i * index.dim(), vec.begin() + (i + 1) * index.dim())});
    record.result_clusters.insert(cl[i]);
  }
  return record;
}

std::optional<ProbeResult> probe_cache(const LocalityCache& cache, RequestId request_id,
                                       const Embedding& v_prime, std::size_t k, double delta,
                                       std::span<const ClusterId> plan) {
  const LocalityRecord* record = cache.find(request_id);
  if (!record) return std::nullopt;
  if (record->query.size() != v_prime.size()) return std::nullopt;
  if (embedding_distance(record->query, v_prime) > delta) return std::nullopt;
  const std::set<ClusterId> in_plan(plan.begin(), plan.end());
  ProbeResult out;
  out.seed.set_k(k);
  for (const auto& cand : record->candidates)
    if (in_plan.count(cand.cluster))  // seeds stay result-neutral
      out.seed.insert(cand.doc_id, embedding_distance(v_prime, cand.vec));
  out.result_clusters = record->result_clusters;
  out.searched = record->searched;
  return out;
}

std::vector<ClusterId> reorder_clusters(std::span<const ClusterId> c_prime, const std::set<ClusterId>& h_v,
                                        const std::set<ClusterId>& c_v) {
  std::vector<ClusterId> hot, seen, rest;
  for (ClusterId c : c_prime) (h_v.count(c) ? hot : c_v.count(c) ? seen : rest).push_back(c);
  hot.insert(hot.end(), seen.begin(), seen.end());
  hot.insert(hot.end(), rest.begin(), rest.end());
  return hot;
}

bool should_terminate(const ivf::SearchCursor& cursor, std::size_t streak_threshold) {
  return cursor.unchanged_streak >= streak_threshold;
}

SpeculationOutcome validate_speculation(const ivf::TopKResult& partial, const ivf::TopKResult& final_result,
                                        std::size_t k) {
  SpeculationOutcome o;
  o.compared_k = k;
  o.kind = partial.truncated(k).doc_ids() == final_result.truncated(k).doc_ids() ? SpecKind::Valid
                                                                                 : SpecKind::Mismatch;
  return o;
}

double semantic_drift(const Embedding& prev_partial, const Embedding& curr_partial) {
  return embedding_distance(prev_partial, curr_partial);
}

}  // namespace sim
}  // namespace hedra_gpu

// ---- C entry points over the persistence functions (ctypes parity tests) -----------
extern "C" {
int hg_save_corpus(const char* path, const float* data, const std::uint64_t* ids, std::uint64_t n,
                   std::uint32_t dim, int metric) {
  try {
    hedra_gpu::ivf::Corpus c;
    c.dim = dim;
    c.metric = static_cast<hedra_gpu::Metric>(metric);
    c.data.assign(data, data + n * dim);
    c.doc_ids.assign(ids, ids + n);
    hedra_gpu::ivf::save_corpus(path, c);
    return 0;
  } catch (...) {
    return -1;
  }
}
int hg_save_centroids(const char* path, const float* rows, std::uint32_t k, std::uint32_t dim, int metric) {
  try {
    hedra_gpu::ivf::Centroids c;
    c.dim = dim;
    for (std::uint32_t i = 0; i < k; ++i) c.rows.emplace_back(rows + std::uint64_t(i) * dim, rows + std::uint64_t(i + 1) * dim);
    hedra_gpu::ivf::save_centroids(path, c, static_cast<hedra_gpu::Metric>(metric));
    return 0;
  } catch (...) {
    return -1;
  }
}
int hg_save_assignments(const char* path, const std::uint32_t* a, std::uint64_t n) {
  try {
    hedra_gpu::ivf::save_assignments(path, std::vector<hedra_gpu::ClusterId>(a, a + n));
    return 0;
  } catch (...) {
    return -1;
  }
}
// load_corpus / load_centroids / load_assignments: sizes first (data == nullptr)
int hg_load_corpus(const char* path, std::uint32_t* dim, std::uint64_t* n, int* metric, float* data,
                   std::uint64_t* ids) {
  try {
    auto c = hedra_gpu::ivf::load_corpus(path);
    *dim = c.dim;
    *n = c.size();
    *metric = static_cast<int>(c.metric);
    if (data) std::memcpy(data, c.data.data(), c.data.size() * sizeof(float));
    if (ids) std::memcpy(ids, c.doc_ids.data(), c.doc_ids.size() * sizeof(std::uint64_t));
    return 0;
  } catch (...) {
    return -1;
  }
}
int hg_load_centroids(const char* path, std::uint32_t* dim, std::uint64_t* k, float* rows) {
  try {
    auto c = hedra_gpu::ivf::load_centroids(path);
    *dim = c.dim;
    *k = c.k_clusters();
    if (rows)
      for (std::size_t i = 0; i < c.rows.size(); ++i)
        std::memcpy(rows + i * c.dim, c.rows[i].data(), c.dim * sizeof(float));
    return 0;
  } catch (...) {
    return -1;
  }
}
int hg_load_assignments(const char* path, std::uint64_t* n, std::uint32_t* a) {
  try {
    auto v = hedra_gpu::ivf::load_assignments(path);
    *n = v.size();
    if (a) std::memcpy(a, v.data(), v.size() * sizeof(std::uint32_t));
    return 0;
  } catch (...) {
    return -1;
  }
}
}