// hedra_gpu.hpp -- C++ drop-in for the reference's retrieval-stage API, backed by
// the sm_100a kernels behind include/hivf.h.
//
// Mirrors (names, argument meaning, error behaviour):
//   hedra::ivf   proj/include/hedra/vector_index.hpp   (TopKResult, merge_topk,
//                SearchCursor, select_clusters, make_cursor, search_clusters,
//                search_step)
//   hedra::cache proj/include/hedra/tiered_cache.hpp   (ClusterCacheState)
//   hedra::ret   proj/include/hedra/retrieval_engine.hpp (RetrievalEngine)
// This is the self-contained form (its own namespace, an explicit Context, an
// HBM-only IvfIndex without the reference's host members), buildable without
// the reference tree.  The LITERAL drop-in -- the reference's own headers and
// namespaces, IvfIndex with its data members, so the unmodified scheduler,
// unit suites and acceptance suite compile against it -- is
// paper_2507_09138_b200/compat/ (include/hedra/vector_index.hpp +
// hedra_ivf_gpu.cpp).  All distance / scan / selection work runs on the GPU in
// both; the host keeps the reference's bookkeeping (cursors, plans, cache
// counters).
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <set>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/hivf.h"

namespace hedra_gpu {

using DocId = std::uint64_t;
using ClusterId = std::uint32_t;
using RequestId = std::int64_t;
using NodeId = std::int32_t;
using Embedding = std::vector<float>;

enum class Metric : std::uint8_t { L2 = 0, Cosine = 1 };

// embedding.hpp:36-43 (double norm, sequential, divide, cast back to float)
Embedding normalized(Embedding v);
// embedding.hpp:27-34 / :53-55 (sequential double chain, no contraction:
// the adapter is built with -ffp-contract=off)
double squared_l2(const float* a, const float* b, std::size_t dim);
double embedding_distance(const Embedding& a, const Embedding& b);

// Throws the reference's exception type for a failed hivf call.
void check(hivf_status st);

namespace ivf {

struct TopKEntry {
  DocId doc_id = 0;
  double distance = 0.0;
};

inline bool topk_less(const TopKEntry& a, const TopKEntry& b) {
  if (a.distance != b.distance) return a.distance < b.distance;
  return a.doc_id < b.doc_id;
}

// Same contract as hedra::ivf::TopKResult (vector_index.hpp:46-79).
class TopKResult {
 public:
  TopKResult() = default;
  explicit TopKResult(std::size_t k) : k_(k) {}
  std::size_t k() const { return k_; }
  void set_k(std::size_t k);
  bool insert(DocId doc_id, double distance);
  const std::vector<TopKEntry>& entries() const { return entries_; }
  std::size_t size() const { return entries_.size(); }
  bool empty() const { return entries_.empty(); }
  TopKResult truncated(std::size_t k) const;
  std::vector<DocId> doc_ids() const;
  bool operator==(const TopKResult& o) const;
  // device round trip (the heap layout hivf_scan_items reads and writes)
  void assign_sorted(const std::uint64_t* ids, const double* d, std::size_t n);

 private:
  std::size_t k_ = 0;
  std::vector<TopKEntry> entries_;
};

TopKResult merge_topk(const TopKResult& a, const TopKResult& b, std::size_t k);

// RAII device context (one owning host thread, like the reference's retrieval worker).
class Context {
 public:
  explicit Context(int device = 0, void* stream = nullptr);
  ~Context();
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  hivf_ctx* raw() const { return ctx_; }

 private:
  hivf_ctx* ctx_ = nullptr;
};

// vector_index.hpp:14-34
struct Corpus {
  std::uint32_t dim = 0;
  Metric metric = Metric::L2;
  std::vector<float> data;     // count * dim, row-major
  std::vector<DocId> doc_ids;  // count
  std::size_t size() const { return doc_ids.size(); }
  const float* row(std::size_t i) const { return data.data() + i * dim; }
  Embedding embedding(std::size_t i) const { return Embedding(row(i), row(i) + dim); }
};

struct Centroids {
  std::uint32_t dim = 0;
  std::vector<std::vector<float>> rows;
  std::size_t k_clusters() const { return rows.size(); }
};

// The HBM-resident index (vector_index.hpp:83-113 without the host copies).
class IvfIndex {
 public:
  // index_from_assignments (vector_index.cpp:210-235): corpus rows (already in
  // search space: normalized for cosine), doc ids, centroid rows, assignment.
  static std::shared_ptr<IvfIndex> from_assignments(Context& ctx, const std::vector<float>& corpus,
                                                    const std::vector<DocId>& ids,
                                                    std::uint32_t dim, Metric metric,
                                                    const std::vector<std::vector<float>>& centroids,
                                                    const std::vector<ClusterId>& assign);
  ~IvfIndex();
  IvfIndex(const IvfIndex&) = delete;
  IvfIndex& operator=(const IvfIndex&) = delete;

  std::size_t k_clusters() const { return sizes_.size(); }
  std::size_t cluster_size(ClusterId c) const { return sizes_.at(c); }
  std::size_t total_vectors() const { return total_; }
  std::uint32_t dim() const { return dim_; }
  Metric metric() const { return metric_; }
  double mean_assigned_distance() const;
  // IvfIndex::locate / doc_embedding (vector_index.hpp:98-111), served by the
  // device locator (hivf_index_locate / hivf_index_gather_rows)
  struct DocLocation {
    ClusterId cluster = 0;
    std::uint32_t offset = 0;
  };
  std::optional<DocLocation> locate(DocId id) const;
  Embedding doc_embedding(DocLocation loc) const;
  hivf_index* raw() const { return ix_; }
  Context& context() const { return *ctx_; }

 private:
  IvfIndex() = default;
  Context* ctx_ = nullptr;
  hivf_index* ix_ = nullptr;
  std::vector<std::size_t> sizes_;
  std::vector<std::uint64_t> offsets_;  // list start rows (list order)
  std::size_t total_ = 0;
  std::uint32_t dim_ = 0;
  Metric metric_ = Metric::L2;
};

// Persistence in the reference's HVEC / u32 formats (vector_index.hpp:162-175),
// byte-identical files: "HVEC", u32 version 1, u32 dim, u64 count, u8 metric,
// then the rows (+ doc ids for a corpus); assignments: u64 count + u32 ids.
// Errors: std::runtime_error (cannot open, bad magic/version, truncated).
void save_corpus(const std::string& path, const Corpus& corpus);
Corpus load_corpus(const std::string& path);
void save_centroids(const std::string& path, const Centroids& centroids, Metric metric);
Centroids load_centroids(const std::string& path);
void save_assignments(const std::string& path, const std::vector<ClusterId>& assign);
std::vector<ClusterId> load_assignments(const std::string& path);

// Index build on the GPU, bit-identical to the reference
// (vector_index.cpp:99-259): train_kmeans, compute_assignments, build_index
// (duplicate-id check, cosine normalization, assignment, index_from_assignments).
Centroids train_kmeans(Context& ctx, const Corpus& corpus, std::size_t k_clusters,
                       std::size_t max_iters, std::uint64_t seed);
std::vector<ClusterId> compute_assignments(Context& ctx, const Corpus& corpus,
                                           const Centroids& centroids);
std::shared_ptr<IvfIndex> build_index(Context& ctx, const Corpus& corpus, const Centroids& centroids,
                                      Metric metric);

struct SearchCursor {
  Embedding query;
  std::vector<ClusterId> plan;
  std::size_t next_pos = 0;
  TopKResult heap;
  std::size_t k = 0;
  std::size_t clusters_searched = 0;
  std::size_t unchanged_streak = 0;
  bool done() const { return next_pos >= plan.size(); }
  std::size_t remaining() const { return plan.size() - next_pos; }
};

struct SearchStepReport {
  std::vector<ClusterId> searched;
  bool heap_changed = false;
};

std::vector<ClusterId> select_clusters(const IvfIndex& index, const Embedding& query,
                                       std::size_t nprobe);
SearchCursor make_cursor(const IvfIndex& index, const Embedding& query, std::size_t nprobe,
                         std::size_t k);
SearchStepReport search_clusters(const IvfIndex& index, SearchCursor& cursor,
                                 std::span<const ClusterId> clusters);
SearchStepReport search_step(const IvfIndex& index, SearchCursor& cursor,
                             std::size_t cluster_budget);

// Batched forms (one GPU launch sequence for many cursors / requests).
// search_clusters_batch: the reference semantics of search_clusters applied to
// every (cursor, clusters) pair; returns one report per pair.
std::vector<SearchStepReport> search_clusters_batch(
    const IvfIndex& index, const std::vector<SearchCursor*>& cursors,
    const std::vector<std::span<const ClusterId>>& clusters);
// make_cursor + search_step(full plan) for every query.
std::vector<TopKResult> search(const IvfIndex& index, const std::vector<Embedding>& queries,
                               std::size_t nprobe, std::size_t k);

// brute_force_search (vector_index.cpp:330-342): every corpus row, exact
// distances, (distance, id) order -- on the device through a one-list index
// of the corpus (cosine: rows and queries normalized as the reference does).
// Batched form uploads the corpus once.  Duplicate doc ids -> invalid_argument
// (the device index needs unique ids; the reference would keep the minimum).
std::vector<TopKResult> brute_force_search(Context& ctx, const Corpus& corpus,
                                           const std::vector<Embedding>& queries, std::size_t k);
TopKResult brute_force_search(Context& ctx, const Corpus& corpus, const Embedding& query, std::size_t k);

}  // namespace ivf

namespace cache {

struct CacheConfig {
  std::size_t capacity_gc = 0;
  int update_interval = 50;
  double transfer_bandwidth_gb_s = 16.0;
  double decay = 0.5;
  std::size_t min_fast_clusters = 2;
};

struct SwapOp {
  ClusterId cluster = 0;
  bool inbound = false;
  double completes_at_ms = 0.0;
};

struct LanePartition {
  std::vector<ClusterId> fast;
  std::vector<ClusterId> slow;
};

// Same state machine as hedra::cache::ClusterCacheState (tiered_cache.hpp:37-78,
// tiered_cache.cpp:10-113). apply_to() publishes the resident set to the device
// (hivf_residency_set) whenever it changed.
class ClusterCacheState {
 public:
  explicit ClusterCacheState(CacheConfig cfg) : cfg_(cfg) {}
  const CacheConfig& config() const { return cfg_; }
  void record_access(std::span<const ClusterId> cluster_ids);
  std::vector<SwapOp> maybe_update(double now_ms, const ivf::IvfIndex& index);
  void complete_swaps(double now_ms);
  LanePartition partition_batch(std::span<const ClusterId> clusters) const;
  bool resident(ClusterId c) const { return resident_.count(c) > 0; }
  std::size_t resident_count() const { return resident_.size(); }
  const std::map<ClusterId, double>& frequencies() const { return freq_; }
  int substages_since_update() const { return since_update_; }
  void count_access_hits(std::span<const ClusterId> clusters);
  std::uint64_t hits() const { return hits_; }
  std::uint64_t misses() const { return misses_; }
  void reset_hit_stats() { hits_ = misses_ = 0; }
  std::uint64_t swap_count() const { return swaps_; }
  void apply_to(const ivf::IvfIndex& index);

 private:
  CacheConfig cfg_;
  std::set<ClusterId> resident_;
  std::vector<SwapOp> in_flight_;
  std::map<ClusterId, double> freq_;
  int since_update_ = 0;
  double link_free_at_ms_ = 0.0;
  std::uint64_t hits_ = 0, misses_ = 0, swaps_ = 0;
  bool dirty_ = false;
};

}  // namespace cache

namespace ret {

enum class TaskOrigin { Normal, SpeculativeRetrieval };

struct RetrievalTask {
  RequestId request_id = 0;
  NodeId node_id = 0;
  ivf::SearchCursor cursor;
  TaskOrigin origin = TaskOrigin::Normal;
};

struct RetrievalCostModel {
  double per_vector_ns = 2000.0;
  double fast_speedup = 8.0;
  double fixed_call_us = 50.0;
};

enum class Lane { Slow, Fast };

double estimate_cluster_cost_ms(const ivf::IvfIndex& index, ClusterId cluster, Lane lane,
                                const RetrievalCostModel& model);
double cluster_variable_ms(const ivf::IvfIndex& index, ClusterId cluster, Lane lane,
                           const RetrievalCostModel& model);
inline double fixed_call_ms(const RetrievalCostModel& model) { return model.fixed_call_us / 1000.0; }

struct BatchItem {
  RequestId request_id = 0;
  NodeId node_id = 0;
  std::vector<ClusterId> clusters;
  std::vector<ClusterId> fast;
  std::vector<ClusterId> slow;
};

struct SubStageBatch {
  std::vector<BatchItem> items;
  double planned_cost_ms = 0.0;
};

struct TaskDelta {
  RequestId request_id = 0;
  NodeId node_id = 0;
  std::size_t clusters_searched = 0;
  bool heap_changed = false;
  bool completed = false;
};

struct RetStepReport {
  double modeled_ms = 0.0;
  double wall_ms = 0.0;
  double slow_lane_ms = 0.0;
  double fast_lane_ms = 0.0;
  std::size_t fast_clusters = 0;
  std::size_t slow_clusters = 0;
  std::vector<TaskDelta> deltas;
  std::vector<cache::SwapOp> swaps_started;
};

// Same contract as hedra::ret::RetrievalEngine (retrieval_engine.hpp:80-110);
// execute() runs every item of the sub-stage in ONE hivf_scan_items call.
class RetrievalEngine {
 public:
  RetrievalEngine(const ivf::IvfIndex* index, RetrievalCostModel model, cache::CacheConfig cfg)
      : index_(index), model_(model), cache_(cfg) {}
  void submit(RetrievalTask task);
  bool has_task(RequestId request_id, NodeId node_id) const;
  const RetrievalTask* find(RequestId request_id, NodeId node_id) const;
  std::size_t task_count() const { return tasks_.size(); }
  RetrievalTask extract(RequestId request_id, NodeId node_id);
  bool cancel(RequestId request_id, NodeId node_id);
  RetStepReport execute(SubStageBatch& batch, double now_ms, bool live_math);
  cache::ClusterCacheState& cache_state() { return cache_; }
  const cache::ClusterCacheState& cache_state() const { return cache_; }
  const RetrievalCostModel& cost_model() const { return model_; }
  const ivf::IvfIndex& index() const { return *index_; }

 private:
  const ivf::IvfIndex* index_;
  RetrievalCostModel model_;
  cache::ClusterCacheState cache_;
  std::map<std::pair<RequestId, NodeId>, RetrievalTask> tasks_;
};

}  // namespace ret

// hedra::bench::measure_per_vector_ns (proj/src/bench.cpp:139-163) on the GPU:
// the reference's calibration of RetrievalCostModel::per_vector_ns (a full
// scan of every list for a constant 0.25 query, median of `repeats`), so the
// unmodified scheduler plans sub-stage budgets (plan_substages) with the
// device's real cost.  One hivf_scan_items call per repeat (items of <= 2048
// lists, same query), wall clock around the synchronous call.
namespace bench {
double measure_per_vector_ns(const ivf::IvfIndex& index, std::size_t repeats = 3);
}  // namespace bench

// hedra::sim (proj/include/hedra/similarity.hpp): the locality helpers of the
// Hedra mode -- host bookkeeping plus exact re-scoring of <= 20 cached docs;
// the doc lookups go through the device locator.
namespace sim {

inline constexpr std::size_t kExtendedTopK = 20;  // K_cache

struct CachedCandidate {
  DocId doc_id = 0;
  ClusterId cluster = 0;
  Embedding vec;
};

struct LocalityRecord {
  Embedding query;
  std::vector<CachedCandidate> candidates;
  std::set<ClusterId> result_clusters;  // H_v
  std::set<ClusterId> searched;         // C_v
};

class LocalityCache {
 public:
  void record_search(RequestId request_id, LocalityRecord record);
  const LocalityRecord* find(RequestId request_id) const;
  void evict(RequestId request_id);
  std::size_t size() const { return records_.size(); }

 private:
  std::map<RequestId, LocalityRecord> records_;
};

// similarity.cpp:18-33 (one batched locate + gather for all candidates)
LocalityRecord make_locality_record(const ivf::IvfIndex& index, const Embedding& query,
                                    const ivf::TopKResult& extended_topk,
                                    std::span<const ClusterId> searched_plan);

struct ProbeResult {
  ivf::TopKResult seed;
  std::set<ClusterId> result_clusters;
  std::set<ClusterId> searched;
};

// similarity.cpp:35-55
std::optional<ProbeResult> probe_cache(const LocalityCache& cache, RequestId request_id,
                                       const Embedding& v_prime, std::size_t k, double delta,
                                       std::span<const ClusterId> plan);
// similarity.cpp:57-72
std::vector<ClusterId> reorder_clusters(std::span<const ClusterId> c_prime, const std::set<ClusterId>& h_v,
                                        const std::set<ClusterId>& c_v);
bool should_terminate(const ivf::SearchCursor& cursor, std::size_t streak_threshold);

enum class SpecKind { Valid, Mismatch };
struct SpeculationOutcome {
  SpecKind kind = SpecKind::Mismatch;
  std::size_t compared_k = 0;
};
SpeculationOutcome validate_speculation(const ivf::TopKResult& partial, const ivf::TopKResult& final_result,
                                        std::size_t k);
double semantic_drift(const Embedding& prev_partial, const Embedding& curr_partial);

}  // namespace sim
}  // namespace hedra_gpu
