// C++ parity tests of the drop-in adapter (paper_2507_09138_b200/host/hedra_gpu.*)
// written like the reference's own doctest suites
// (proj/tests/test_vector_index.cpp, test_retrieval_engine.cpp,
// test_tiered_cache.cpp), with the oracle (oracle/liboracle.so, the plain-C
// restatement) as the checker.  `--cpu-only` runs the host-only cases
// (ClusterCacheState, TopKResult) without a GPU.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <limits>
#include <set>
#include <random>
#include <string>
#include <vector>

#include "../../paper_2507_09138_b200/host/hedra_gpu.hpp"

extern "C" {
uint64_t orc_brute_force(const float* corpus, const uint64_t* ids, uint64_t n, uint32_t dim, int metric,
                         const float* query, uint64_t k, uint64_t* ids_out, double* dists_out);
void orc_compute_assignments(const float* corpus, uint64_t n, uint32_t dim, const float* centroids,
                             uint32_t n_clusters, uint32_t* assign_out);
int orc_select_clusters(const float* centroids, uint32_t n_clusters, uint32_t dim, int metric,
                        const float* query, uint32_t nprobe, uint32_t* plan_out, double* dists_out);
}

using namespace hedra_gpu;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    ++g_checks;                                                                  \
    if (!(cond)) {                                                               \
      ++g_fail;                                                                  \
      std::printf("  CHECK failed %s:%d: %s\n", __FILE__, __LINE__, #cond);      \
    }                                                                            \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                                 \
  do {                                                                           \
    ++g_checks;                                                                  \
    bool ok_ = false;                                                            \
    try {                                                                        \
      (void)(expr);                                                              \
    } catch (const T&) {                                                         \
      ok_ = true;                                                                \
    } catch (...) {                                                              \
    }                                                                            \
    if (!ok_) {                                                                  \
      ++g_fail;                                                                  \
      std::printf("  CHECK_THROWS_AS failed %s:%d: %s\n", __FILE__, __LINE__, #expr); \
    }                                                                            \
  } while (0)

struct Case {
  const char* name;
  bool gpu;
  std::function<void()> fn;
};
static std::vector<Case>& cases() {
  static std::vector<Case> c;
  return c;
}
struct Reg {
  Reg(const char* n, bool gpu, std::function<void()> f) { cases().push_back({n, gpu, f}); }
};
#define TEST_GPU(name) static void name(); static Reg r_##name(#name, true, name); static void name()
#define TEST_CPU(name) static void name(); static Reg r_##name(#name, false, name); static void name()

// ---- fixtures (test_support.hpp equivalents, our own generator) ------------------
struct Data {
  std::uint32_t dim = 0;
  std::vector<float> x;
  std::vector<DocId> ids;
  std::vector<std::vector<float>> cents;
  std::vector<ClusterId> assign;
  std::size_t n() const { return ids.size(); }
};

static Data random_data(std::uint64_t seed, std::size_t n, std::uint32_t dim, std::size_t K, double scale = 1.0) {
  std::mt19937_64 g(seed);
  std::normal_distribution<double> nd(0.0, 1.0);
  Data d;
  d.dim = dim;
  d.x.resize(n * dim);
  for (auto& v : d.x) v = static_cast<float>(nd(g) * scale);
  for (std::size_t i = 0; i < n; ++i) d.ids.push_back(i);
  for (std::size_t c = 0; c < K; ++c)
    d.cents.emplace_back(d.x.begin() + (c * 7 % n) * dim, d.x.begin() + (c * 7 % n + 1) * dim);
  std::vector<float> flat;
  for (auto& c : d.cents) flat.insert(flat.end(), c.begin(), c.end());
  d.assign.resize(n);
  orc_compute_assignments(d.x.data(), n, dim, flat.data(), static_cast<uint32_t>(K), d.assign.data());
  return d;
}

static Data corpus_a() {  // test_support.hpp:11-25 and test_vector_index.cpp:21-26
  Data d;
  d.dim = 2;
  d.x = {0, 0, .1f, 0, 0, .1f, .1f, .1f, 10, 10, 10.1f, 10, 9.9f, 10.05f, 10, 10.05f};
  for (DocId i = 0; i < 8; ++i) d.ids.push_back(i);
  d.cents = {{0.05f, 0.05f}, {10.0f, 10.025f}};
  d.assign = {0, 0, 0, 0, 1, 1, 1, 1};
  return d;
}

static std::shared_ptr<ivf::IvfIndex> build(ivf::Context& ctx, const Data& d, Metric m = Metric::L2) {
  return ivf::IvfIndex::from_assignments(ctx, d.x, d.ids, d.dim, m, d.cents, d.assign);
}

static ivf::TopKResult brute(const Data& d, const Embedding& q, std::size_t k, int metric = 0) {
  std::vector<uint64_t> i(k);
  std::vector<double> dd(k);
  const uint64_t m = orc_brute_force(d.x.data(), d.ids.data(), d.n(), d.dim, metric, q.data(), k,
                                     i.data(), dd.data());
  ivf::TopKResult r(k);
  r.assign_sorted(i.data(), dd.data(), m);
  return r;
}

static Embedding rand_query(std::mt19937_64& g, std::uint32_t dim, double scale = 1.0) {
  std::normal_distribution<double> nd(0.0, 1.0);
  Embedding q(dim);
  for (auto& v : q) v = static_cast<float>(nd(g) * scale);
  return q;
}

static ivf::Context& ctx() {
  static ivf::Context c(0);
  return c;
}

// ---- ivf ---------------------------------------------------------------------------
TEST_GPU(select_clusters_basics_on_corpus_a) {
  auto ix = build(ctx(), corpus_a());
  CHECK(ivf::select_clusters(*ix, {1.0f, 0.0f}, 1) == std::vector<ClusterId>{0});
  CHECK((ivf::select_clusters(*ix, {1.0f, 0.0f}, 2) == std::vector<ClusterId>{0, 1}));
  CHECK_THROWS_AS(ivf::select_clusters(*ix, {1.0f, 0.0f}, 0), std::invalid_argument);
  CHECK_THROWS_AS(ivf::select_clusters(*ix, {1.0f, 0.0f}, 3), std::invalid_argument);
  CHECK(ix->cluster_size(0) == 4 && ix->cluster_size(1) == 4 && ix->total_vectors() == 8);
}

TEST_GPU(select_clusters_matches_full_sort) {
  const Data d = random_data(21, 640, 16, 32);
  auto ix = build(ctx(), d);
  std::vector<float> flat;
  for (auto& c : d.cents) flat.insert(flat.end(), c.begin(), c.end());
  std::mt19937_64 g(5);
  for (int t = 0; t < 10; ++t) {
    const auto q = rand_query(g, 16);
    std::vector<uint32_t> want(8);
    orc_select_clusters(flat.data(), 32, 16, 0, q.data(), 8, want.data(), nullptr);
    CHECK(ivf::select_clusters(*ix, q, 8) == std::vector<ClusterId>(want.begin(), want.end()));
  }
}

TEST_GPU(search_step_finds_exact_nearest_point) {
  auto ix = build(ctx(), corpus_a());
  auto c = ivf::make_cursor(*ix, {0.0f, 0.0f}, 2, 1);
  const auto rep = ivf::search_step(*ix, c, 2);
  CHECK(rep.searched.size() == 2 && c.next_pos == 2 && c.done());
  CHECK(c.heap.size() == 1 && c.heap.entries()[0].doc_id == 0 && c.heap.entries()[0].distance == 0.0);
  auto c2 = ivf::make_cursor(*ix, {0.0f, 0.0f}, 2, 3);
  CHECK(ivf::search_step(*ix, c2, 100).searched.size() == 2);
  const auto again = ivf::search_step(*ix, c2, 1);  // exhausted cursor: empty report
  CHECK(again.searched.empty() && !again.heap_changed);
  CHECK_THROWS_AS(ivf::make_cursor(*ix, {0.0f, 0.0f}, 2, 0), std::invalid_argument);
  auto c3 = ivf::make_cursor(*ix, {0.0f, 0.0f}, 2, 1);
  CHECK_THROWS_AS(ivf::search_step(*ix, c3, 0), std::invalid_argument);
}

TEST_GPU(budget_split_equals_single_pass) {
  auto ix = build(ctx(), corpus_a());
  auto split = ivf::make_cursor(*ix, {5.0f, 5.0f}, 2, 3);
  auto whole = ivf::make_cursor(*ix, {5.0f, 5.0f}, 2, 3);
  ivf::search_step(*ix, split, 1);
  ivf::search_step(*ix, split, 1);
  ivf::search_step(*ix, whole, 2);
  CHECK(split.heap == whole.heap);
}

TEST_GPU(nprobe_all_equals_brute_force) {
  const Data d = random_data(33, 1000, 12, 16);
  auto ix = build(ctx(), d);
  std::mt19937_64 g(7);
  for (int t = 0; t < 20; ++t) {
    const auto q = rand_query(g, 12);
    auto c = ivf::make_cursor(*ix, q, ix->k_clusters(), 10);
    while (!c.done()) ivf::search_step(*ix, c, 3);
    CHECK(c.heap == brute(d, q, 10));
  }
}

TEST_GPU(cosine_metric_matches_brute_force) {
  Data d = random_data(34, 400, 8, 8);
  Data dn = d;
  for (std::size_t i = 0; i < d.n(); ++i) {
    Embedding r(d.x.begin() + i * 8, d.x.begin() + (i + 1) * 8);
    r = normalized(r);
    std::copy(r.begin(), r.end(), dn.x.begin() + i * 8);
  }
  std::vector<float> flat;
  for (auto& c : dn.cents) flat.insert(flat.end(), c.begin(), c.end());
  orc_compute_assignments(dn.x.data(), dn.n(), 8, flat.data(), 8, dn.assign.data());
  auto ix = build(ctx(), dn, Metric::Cosine);
  std::mt19937_64 g(8);
  const auto q = rand_query(g, 8, 3.0);
  auto c = ivf::make_cursor(*ix, q, ix->k_clusters(), 5);
  while (!c.done()) ivf::search_step(*ix, c, 2);
  CHECK(c.heap == brute(d, q, 5, 1));
}

TEST_GPU(step_split_invariance_and_streak) {
  const Data d = random_data(77, 800, 10, 20);
  auto ix = build(ctx(), d);
  std::mt19937_64 g(9);
  for (int t = 0; t < 25; ++t) {
    const auto q = rand_query(g, 10);
    const std::size_t np = 1 + g() % ix->k_clusters();
    auto whole = ivf::make_cursor(*ix, q, np, 7);
    ivf::search_step(*ix, whole, np);
    auto split = ivf::make_cursor(*ix, q, np, 7);
    double prev_worst = INFINITY;
    while (!split.done()) {
      const auto before = split.unchanged_streak;
      const auto rep = ivf::search_step(*ix, split, 1 + g() % 4);
      CHECK(rep.heap_changed ? split.unchanged_streak <= rep.searched.size() - 1
                             : split.unchanged_streak == before + rep.searched.size());
      if (split.heap.size() == split.k) {
        CHECK(split.heap.entries().back().distance <= prev_worst);
        prev_worst = split.heap.entries().back().distance;
      }
    }
    CHECK(split.heap == whole.heap && split.clusters_searched == whole.clusters_searched);
  }
}

TEST_GPU(search_clusters_out_of_plan_order_is_runtime_error) {
  auto ix = build(ctx(), corpus_a());
  auto c = ivf::make_cursor(*ix, {0.0f, 0.0f}, 2, 1);
  const std::vector<ClusterId> wrong{1};
  CHECK_THROWS_AS(ivf::search_clusters(*ix, c, wrong), std::runtime_error);
  const std::vector<ClusterId> too_many{0, 1, 0};
  CHECK_THROWS_AS(ivf::search_clusters(*ix, c, too_many), std::runtime_error);
}

TEST_GPU(batched_search_equals_cursor_path) {
  const Data d = random_data(35, 3000, 24, 16);
  auto ix = build(ctx(), d);
  std::mt19937_64 g(10);
  std::vector<Embedding> qs;
  for (int i = 0; i < 40; ++i) qs.push_back(rand_query(g, 24));
  const auto res = ivf::search(*ix, qs, 5, 10);
  for (std::size_t i = 0; i < qs.size(); ++i) {
    auto c = ivf::make_cursor(*ix, qs[i], 5, 10);
    ivf::search_step(*ix, c, 5);
    CHECK(res[i] == c.heap);
  }
}

// ---- ret ---------------------------------------------------------------------------
static ret::RetrievalTask task_for(const ivf::IvfIndex& ix, RequestId r, NodeId n, Embedding q,
                                   std::size_t nprobe, std::size_t k) {
  ret::RetrievalTask t;
  t.request_id = r;
  t.node_id = n;
  t.cursor = ivf::make_cursor(ix, q, nprobe, k);
  return t;
}

static ret::RetrievalCostModel model_10ns() { return {10.0, 8.0, 5.0}; }

TEST_GPU(engine_submit_duplicates_and_unknown_task) {
  auto ix = build(ctx(), corpus_a());
  ret::RetrievalEngine eng(ix.get(), model_10ns(), {});
  eng.submit(task_for(*ix, 1, 2, {0.f, 0.f}, 2, 3));
  CHECK(eng.task_count() == 1);
  CHECK_THROWS_AS(eng.submit(task_for(*ix, 1, 2, {0.f, 0.f}, 2, 3)), std::invalid_argument);
  ret::SubStageBatch b;
  b.items.push_back(ret::BatchItem{9, 9, {0}, {}, {}});
  CHECK_THROWS_AS(eng.execute(b, 0.0, false), std::runtime_error);
  CHECK_THROWS_AS(eng.extract(7, 7), std::invalid_argument);
  CHECK(eng.cancel(1, 2) && !eng.has_task(1, 2));
}

TEST_GPU(engine_modeled_latency_and_end_of_plan) {
  const Data d = random_data(11, 400, 8, 8);
  auto ix = build(ctx(), d);
  std::mt19937_64 g(12);
  const auto q = rand_query(g, 8);
  ret::RetrievalEngine eng(ix.get(), model_10ns(), {});
  eng.submit(task_for(*ix, 3, 1, q, 8, 5));
  const auto plan = eng.find(3, 1)->cursor.plan;
  std::size_t pos = 0;
  bool done = false;
  for (std::size_t s : {3, 1, 4}) {
    ret::SubStageBatch b;
    ret::BatchItem it;
    it.request_id = 3;
    it.node_id = 1;
    it.clusters.assign(plan.begin() + pos, plan.begin() + pos + s);
    pos += s;
    double slow = 0;
    for (ClusterId c : it.clusters) slow += ix->cluster_size(c) * 10.0 / 1e6;
    b.items.push_back(it);
    const auto rep = eng.execute(b, 0.0, true);
    CHECK(std::fabs(rep.modeled_ms - (slow + 0.005)) < 1e-12);
    done = rep.deltas[0].completed;
  }
  CHECK(done);
  auto t = eng.extract(3, 1);
  auto whole = ivf::make_cursor(*ix, q, 8, 5);
  ivf::search_step(*ix, whole, 8);
  CHECK(t.cursor.heap == whole.heap && eng.task_count() == 0);
}

TEST_GPU(engine_batch_equals_sequential_and_lane_transparency) {
  const Data d = random_data(13, 2000, 8, 16);
  auto ix = build(ctx(), d);
  cache::CacheConfig cached;
  cached.capacity_gc = 4;
  cached.update_interval = 2;
  cached.min_fast_clusters = 1;
  std::vector<std::vector<ivf::TopKResult>> outs;
  for (const auto& cfg : {cache::CacheConfig{}, cached}) {
    ret::RetrievalEngine eng(ix.get(), model_10ns(), cfg);
    std::vector<ivf::TopKResult> heaps;
    for (int round = 0; round < 3; ++round) {
      ret::SubStageBatch b;
      for (RequestId r = 0; r < 6; ++r) {
        std::mt19937_64 g(40 + r + 100 * round);
        eng.submit(task_for(*ix, r, round, rand_query(g, 8), 4, 5));
        ret::BatchItem it;
        it.request_id = r;
        it.node_id = round;
        it.clusters = eng.find(r, round)->cursor.plan;
        b.items.push_back(it);
      }
      const auto rep = eng.execute(b, 1000.0 * round, true);
      CHECK(rep.deltas.size() == 6);
      for (RequestId r = 0; r < 6; ++r) heaps.push_back(eng.extract(r, round).cursor.heap);
    }
    outs.push_back(heaps);
  }
  CHECK(outs[0] == outs[1]);
  // the batched GPU sub-stage equals per-cursor sequential search
  std::size_t i = 0;
  for (int round = 0; round < 3; ++round)
    for (RequestId r = 0; r < 6; ++r, ++i) {
      std::mt19937_64 g(40 + r + 100 * round);
      auto c = ivf::make_cursor(*ix, rand_query(g, 8), 4, 5);
      ivf::search_step(*ix, c, 4);
      CHECK(c.heap == outs[0][i]);
    }
}

// ---- host-only: TopKResult / merge_topk / ClusterCacheState -----------------------------
TEST_CPU(merge_topk_identity_commutativity_dedup) {  // test_vector_index.cpp:227-246
  ivf::TopKResult x(3);
  x.insert(1, 0.5);
  x.insert(2, 0.25);
  ivf::TopKResult empty(3);
  CHECK(ivf::merge_topk(x, empty, 3) == x);
  CHECK(ivf::merge_topk(x, empty, 1) == x.truncated(1));
  ivf::TopKResult y(3);
  y.insert(3, 0.1);
  y.insert(1, 0.75);
  const auto ab = ivf::merge_topk(x, y, 3), ba = ivf::merge_topk(y, x, 3);
  CHECK(ab == ba && ab.size() == 3);
  CHECK(ab.doc_ids() == (std::vector<DocId>{3, 2, 1}) && ab.entries()[2].distance == 0.5);
}

TEST_CPU(cache_record_access_counts_once_per_substage) {  // test_tiered_cache.cpp:40-53
  cache::CacheConfig cfg;
  cfg.capacity_gc = 2;
  cache::ClusterCacheState st(cfg);
  for (int i = 0; i < 5; ++i) st.record_access(std::vector<ClusterId>{0});
  for (int i = 0; i < 3; ++i) st.record_access(std::vector<ClusterId>{1});
  st.record_access(std::vector<ClusterId>{2, 2, 2});
  CHECK(st.frequencies().at(0) == 5.0 && st.frequencies().at(1) == 3.0 && st.frequencies().at(2) == 1.0);
  const auto before = st.frequencies();
  st.record_access(std::vector<ClusterId>{});
  CHECK(st.frequencies() == before);
}

TEST_CPU(cache_partition_threshold) {  // test_tiered_cache.cpp:102-126 (no swaps needed)
  cache::CacheConfig cfg;
  cfg.capacity_gc = 4;
  cfg.min_fast_clusters = 2;
  cache::ClusterCacheState st(cfg);
  auto p = st.partition_batch(std::vector<ClusterId>{2, 3});
  CHECK(p.fast.empty() && p.slow.size() == 2);
  cache::ClusterCacheState off{cache::CacheConfig{}};
  p = off.partition_batch(std::vector<ClusterId>{0, 1});
  CHECK(p.fast.empty() && p.slow.size() == 2);
}

TEST_GPU(cache_update_swaps_ties_midswap_capacity) {  // test_tiered_cache.cpp:55-150
  Data d;
  d.dim = 2;
  for (std::size_t c = 0; c < 8; ++c) {
    d.cents.push_back({10.0f * c, 0.0f});
    for (std::size_t i = 0; i < 50; ++i) {
      d.x.push_back(10.0f * c);
      d.x.push_back(0.01f * i);
      d.ids.push_back(d.ids.size());
      d.assign.push_back(c);
    }
  }
  auto ix = build(ctx(), d);
  {
    cache::CacheConfig cfg;
    cfg.capacity_gc = 2;
    cfg.update_interval = 5;
    cache::ClusterCacheState st(cfg);
    for (int i = 0; i < 4; ++i) st.record_access(std::vector<ClusterId>{0, 1, 2});
    CHECK(st.maybe_update(0.0, *ix).empty());
    st.record_access(std::vector<ClusterId>{0, 1});
    const auto plan = st.maybe_update(0.0, *ix);
    CHECK(plan.size() == 2 && plan[0].inbound && plan[1].inbound);
    st.complete_swaps(plan[1].completes_at_ms + 1.0);
    CHECK(st.resident(0) && st.resident(1) && !st.resident(2));
    st.apply_to(*ix);
    std::vector<std::uint8_t> res(ix->k_clusters());
    hivf_residency_get(ix->raw(), res.data());
    CHECK(res[0] && res[1] && !res[2]);
  }
  {
    cache::CacheConfig cfg;
    cfg.capacity_gc = 1;
    cfg.update_interval = 1;
    cache::ClusterCacheState st(cfg);
    st.record_access(std::vector<ClusterId>{1, 2});
    const auto plan = st.maybe_update(0.0, *ix);
    CHECK(plan.size() == 1 && plan[0].cluster == 1);  // ties -> lower id
    CHECK(st.partition_batch(std::vector<ClusterId>{1}).fast.empty());  // mid-swap: slow
    st.complete_swaps(plan[0].completes_at_ms);
    CHECK(st.resident(1));
  }
  {
    cache::CacheConfig cfg;
    cfg.capacity_gc = 3;
    cfg.update_interval = 1;
    cache::ClusterCacheState st(cfg);
    std::mt19937_64 g(5);
    double now = 0.0;
    for (int s = 0; s < 200; ++s) {
      std::vector<ClusterId> acc;
      for (int j = 0; j < 3; ++j) acc.push_back(static_cast<ClusterId>(g() % 8));
      st.record_access(acc);
      st.maybe_update(now, *ix);
      CHECK(st.resident_count() <= 3);
      now += 0.01;
      st.complete_swaps(now);
      CHECK(st.resident_count() <= 3);
    }
  }
}

// ---- index build (vector_index.cpp:99-259) ----------------------------------------
TEST_GPU(build_index_equals_from_assignments_and_brute_force) {
  // build_index = compute_assignments + index_from_assignments; with nprobe = K
  // the IVF search equals brute force exactly (test_vector_index.cpp:196-208)
  ivf::Context ctx(0);
  const Data d = random_data(91, 3000, 12, 24);
  ivf::Corpus corpus;
  corpus.dim = d.dim;
  corpus.data = d.x;
  corpus.doc_ids = d.ids;
  ivf::Centroids cents;
  cents.dim = d.dim;
  cents.rows = d.cents;
  const auto asg = ivf::compute_assignments(ctx, corpus, cents);
  CHECK(asg == d.assign);  // the C restatement's nearest_centroid, ties -> lowest id
  auto ix = ivf::build_index(ctx, corpus, cents, Metric::L2);
  std::mt19937_64 g(5);
  for (int t = 0; t < 10; ++t) {
    const Embedding q = rand_query(g, d.dim);
    auto cur = ivf::make_cursor(*ix, q, cents.rows.size(), 10);
    while (!cur.done()) ivf::search_step(*ix, cur, 7);
    CHECK(cur.heap == brute(d, q, 10));
  }
}

TEST_GPU(brute_force_search_matches_reference) {  // vector_index.cpp:330-342
  ivf::Context ctx(0);
  for (int metric = 0; metric < 2; ++metric) {
    const Data d = random_data(400 + metric, 2500, 20, 4);
    ivf::Corpus corpus;
    corpus.dim = d.dim;
    corpus.metric = metric ? Metric::Cosine : Metric::L2;
    corpus.data = d.x;
    corpus.doc_ids = d.ids;
    std::mt19937_64 g(11 + metric);
    std::vector<Embedding> qs;
    for (int t = 0; t < 24; ++t) qs.push_back(rand_query(g, d.dim, metric ? 2.0 : 1.0));
    const auto got = ivf::brute_force_search(ctx, corpus, qs, 10);
    CHECK(got.size() == qs.size());
    for (std::size_t t = 0; t < qs.size(); ++t) CHECK(got[t] == brute(d, qs[t], 10, metric));
    CHECK(ivf::brute_force_search(ctx, corpus, qs[3], 10) == got[3]);
    // k above the corpus size: every row, in order
    ivf::Corpus small = corpus;
    small.data.resize(7 * d.dim);
    small.doc_ids.resize(7);
    Data ds = d;
    ds.x.resize(7 * d.dim);
    ds.ids.resize(7);
    CHECK(ivf::brute_force_search(ctx, small, qs[0], 50) == brute(ds, qs[0], 50, metric));
  }
  ivf::Corpus empty;
  empty.dim = 4;
  CHECK(ivf::brute_force_search(ctx, empty, Embedding(4, 1.0f), 5).empty());
}

TEST_GPU(train_kmeans_contract) {
  ivf::Context ctx(0);
  const Data d = random_data(17, 2000, 8, 4);
  ivf::Corpus corpus;
  corpus.dim = d.dim;
  corpus.data = d.x;
  corpus.doc_ids = d.ids;
  const auto a = ivf::train_kmeans(ctx, corpus, 16, 5, 3);
  const auto b = ivf::train_kmeans(ctx, corpus, 16, 5, 3);
  CHECK(a.k_clusters() == 16 && a.dim == 8);
  CHECK(a.rows == b.rows);  // deterministic for a seed
  // every centroid is a mean of data or a data point: finite
  for (const auto& r : a.rows)
    for (float v : r) CHECK(std::isfinite(v));
  CHECK_THROWS_AS(ivf::train_kmeans(ctx, corpus, 3000, 5, 3), std::invalid_argument);  // n < K
  CHECK_THROWS_AS(ivf::train_kmeans(ctx, corpus, 0, 5, 3), std::invalid_argument);
  CHECK_THROWS_AS(ivf::train_kmeans(ctx, corpus, 4, 0, 3), std::invalid_argument);
}

// ---- sim (ported from proj/tests/test_similarity.cpp) ------------------------------
static ivf::SearchCursor full_search(const ivf::IvfIndex& ix, const Embedding& q, std::size_t nprobe,
                                     std::size_t k) {
  auto cur = ivf::make_cursor(ix, q, nprobe, k);
  while (!cur.done()) ivf::search_step(ix, cur, 3);
  return cur;
}

TEST_GPU(sim_probe_identical_query_rescores_cached_topk) {  // test_similarity.cpp:60-72
  ivf::Context ctx(0);
  const Data d = random_data(33, 400, 8, 8);
  auto ix = build(ctx, d);
  sim::LocalityCache cache;
  std::mt19937_64 g(3);
  const auto q = rand_query(g, 8);
  auto cur = full_search(*ix, q, 8, sim::kExtendedTopK);
  cache.record_search(1, sim::make_locality_record(*ix, cur.query, cur.heap, cur.plan));
  const auto probe = sim::probe_cache(cache, 1, cur.query, 5, 1e-12, cur.plan);
  CHECK(probe.has_value());
  if (probe) CHECK(probe->seed == cur.heap.truncated(5));
  // the record holds the docs' own vectors and clusters (locate + doc_embedding)
  const auto* rec = cache.find(1);
  CHECK(rec && rec->candidates.size() == cur.heap.size());
  for (const auto& c : rec->candidates) {
    const auto loc = ix->locate(c.doc_id);
    CHECK(loc.has_value() && loc->cluster == c.cluster);
    if (loc) CHECK(ix->doc_embedding(*loc) == c.vec);
    const float* row = d.x.data() + c.doc_id * d.dim;
    CHECK(c.vec == Embedding(row, row + d.dim));
  }
  CHECK(!ix->locate(987654321ull).has_value());
}

TEST_GPU(sim_probe_misses_on_drift_or_no_record) {  // :74-88
  ivf::Context ctx(0);
  const Data d = random_data(34, 400, 8, 8);
  auto ix = build(ctx, d);
  sim::LocalityCache cache;
  std::mt19937_64 g(4);
  const auto q = rand_query(g, 8);
  auto cur = full_search(*ix, q, 8, sim::kExtendedTopK);
  cache.record_search(1, sim::make_locality_record(*ix, cur.query, cur.heap, cur.plan));
  Embedding far = cur.query;
  far[0] += 100.0f;
  CHECK(!sim::probe_cache(cache, 1, far, 5, 0.5, cur.plan).has_value());
  CHECK(!sim::probe_cache(cache, 2, cur.query, 5, 0.5, cur.plan).has_value());
}

TEST_GPU(sim_seeding_never_changes_the_result) {  // :90-112
  ivf::Context ctx(0);
  const Data d = random_data(35, 600, 8, 8);
  auto ix = build(ctx, d);
  sim::LocalityCache cache;
  std::mt19937_64 g(6);
  std::normal_distribution<double> nd(0.0, 1.0);
  for (int trial = 0; trial < 20; ++trial) {
    const auto q = rand_query(g, 8);
    auto base = full_search(*ix, q, 6, sim::kExtendedTopK);
    cache.record_search(9, sim::make_locality_record(*ix, base.query, base.heap, base.plan));
    Embedding q2 = q;
    for (auto& x : q2) x += static_cast<float>(nd(g) * 0.05);
    auto unseeded = ivf::make_cursor(*ix, q2, 6, 5);
    auto seeded = ivf::make_cursor(*ix, q2, 6, 5);
    const auto probe = sim::probe_cache(cache, 9, seeded.query, 5,
                                        std::numeric_limits<double>::infinity(), seeded.plan);
    CHECK(probe.has_value());
    if (probe) seeded.heap = ivf::merge_topk(seeded.heap, probe->seed, 5);
    while (!unseeded.done()) ivf::search_step(*ix, unseeded, 2);
    while (!seeded.done()) ivf::search_step(*ix, seeded, 2);
    CHECK(seeded.heap == unseeded.heap);
  }
}

TEST_CPU(sim_reorder_three_group_rule) {  // :114-122 (+ permutation property :124-150)
  const std::vector<ClusterId> c_prime = {5, 3, 8, 1};
  CHECK(sim::reorder_clusters(c_prime, {3}, {3, 8}) == (std::vector<ClusterId>{3, 8, 5, 1}));
  CHECK(sim::reorder_clusters(c_prime, {}, {}) == c_prime);
  std::mt19937_64 g(7);
  for (int t = 0; t < 50; ++t) {
    std::vector<ClusterId> cp;
    for (int i = 0; i < 20; ++i) cp.push_back(static_cast<ClusterId>(g() % 1000));
    std::sort(cp.begin(), cp.end());
    cp.erase(std::unique(cp.begin(), cp.end()), cp.end());
    std::set<ClusterId> h, c;
    for (ClusterId x : cp) {
      const double u = (g() >> 11) * 0x1.0p-53;
      if (u < 0.2) {
        h.insert(x);
        c.insert(x);
      } else if (u < 0.5) {
        c.insert(x);
      }
    }
    auto out = sim::reorder_clusters(cp, h, c);
    auto a = cp, b = out;
    std::sort(a.begin(), a.end());
    std::sort(b.begin(), b.end());
    CHECK(a == b);
    int phase = 0;
    for (ClusterId x : out) {
      const int grp = h.count(x) ? 0 : (c.count(x) ? 1 : 2);
      CHECK(grp >= phase);
      phase = std::max(phase, grp);
    }
  }
}

TEST_GPU(sim_reordered_plan_same_result) {  // :152-170
  ivf::Context ctx(0);
  const Data d = random_data(36, 600, 8, 8);
  auto ix = build(ctx, d);
  std::mt19937_64 g(8);
  for (int t = 0; t < 15; ++t) {
    const auto q = rand_query(g, 8);
    auto plain = ivf::make_cursor(*ix, q, 8, 5);
    auto re = plain;
    std::set<ClusterId> h, c;
    for (ClusterId x : plain.plan) {
      if ((g() >> 11) * 0x1.0p-53 < 0.3) h.insert(x);
      if ((g() >> 11) * 0x1.0p-53 < 0.5) c.insert(x);
    }
    re.plan = sim::reorder_clusters(re.plan, h, c);
    while (!plain.done()) ivf::search_step(*ix, plain, 3);
    while (!re.done()) ivf::search_step(*ix, re, 3);
    CHECK(plain.heap == re.heap);
  }
}

TEST_CPU(sim_should_terminate_and_validate_speculation) {  // :172-196
  ivf::SearchCursor cur;
  cur.unchanged_streak = 3;
  CHECK(!sim::should_terminate(cur, 4));
  cur.unchanged_streak = 4;
  CHECK(sim::should_terminate(cur, 4));
  ivf::TopKResult a(3), b(3);
  a.insert(1, 0.5);
  a.insert(2, 0.7);
  b.insert(1, 0.5);
  b.insert(2, 0.7);
  CHECK(sim::validate_speculation(a, b, 2).kind == sim::SpecKind::Valid);
  b.insert(3, 0.1);
  CHECK(sim::validate_speculation(a, b, 2).kind == sim::SpecKind::Mismatch);
}

TEST_GPU(bench_measure_per_vector_ns) {  // bench.cpp:139-163 contract on the GPU
  ivf::Context ctx(0);
  const Data d = random_data(77, 5000, 16, 32);
  auto ix = build(ctx, d);
  const double ns = bench::measure_per_vector_ns(*ix, 3);
  CHECK(std::isfinite(ns) && ns > 0.0);
  CHECK(ns < 1e6);  // a whole-index GPU scan costs far below a millisecond per vector
}

int main(int argc, char** argv) {
  const bool cpu_only = argc > 1 && std::strcmp(argv[1], "--cpu-only") == 0;
  int ran = 0;
  for (const auto& c : cases()) {
    if (cpu_only && c.gpu) continue;
    const int before = g_fail;
    try {
      c.fn();
    } catch (const std::exception& e) {
      ++g_fail;
      std::printf("  exception in %s: %s\n", c.name, e.what());
    }
    std::printf("%s %s\n", g_fail == before ? "PASS" : "FAIL", c.name);
    ++ran;
  }
  std::printf("%d cases, %d checks, %d failures\n", ran, g_checks, g_fail);
  return g_fail == 0 ? 0 : 1;
}
