// hedra_c5.cpp -- config 5 (heterogeneous multi-stage RAG retrieval stream)
// through the reference's UNMODIFIED scheduler: harness::generate_corpus /
// generate_workload (proj/src/workload.cpp) -> ivf::train_kmeans / build_index
// -> sched::run (proj/src/scheduler.cpp:1751-1757), exactly as `hedra run`
// drives it (proj/tools/hedra_main.cpp:103-131).  Built twice by compat/build.py:
//   hedra_c5_gpu  against the GPU-backed hedra::ivf / RetrievalEngine (compat/)
//   hedra_c5_cpu  against the reference's own vector_index.cpp /
//                 retrieval_engine.cpp (the oracle build)
// so the same command gives the GPU engine's report and the reference's, and
// a Virtual-clock run must produce byte-identical report JSON in both.
//
// Prints one JSON line: the report summary plus the retrieval sub-stage
// latency distribution (p50/p99 of the "substage" trace events, nearest rank
// as proj/src/report.cpp:15-21 computes request percentiles) and the batch
// sizes the scheduler formed.  --report PATH writes report.to_json().
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <map>
#include <sstream>
#include <string>
#include <tuple>
#include <vector>

#include "hedra/bench.hpp"
#include "hedra/scheduler.hpp"
#include "hedra/workload.hpp"

using namespace hedra;

namespace {

struct Args {
  std::size_t n = 20000, topics = 32, clusters = 64, requests = 200, nprobe = 16;
  std::uint32_t dim = 32;
  double spread = 0.25, rate = 40.0, drift = 0.3, per_vector_ns = 0.0, beta_ms = 1.0;
  double slo_ms = 1e12;
  std::size_t kmeans_iters = 10, kmeans_sample = 0;
  std::uint64_t seed = 300;
  std::string mix = "multistep=0.5,irg=0.5", strategy = "hedra", clock = "virtual", report;
  bool cache = true, spec = true;
};

double num(const char* s) { return std::strtod(s, nullptr); }

Args parse(int argc, char** argv) {
  Args a;
  for (int i = 1; i + 1 < argc; i += 2) {
    const std::string k = argv[i];
    const char* v = argv[i + 1];
    if (k == "--n") a.n = static_cast<std::size_t>(num(v));
    else if (k == "--dim") a.dim = static_cast<std::uint32_t>(num(v));
    else if (k == "--topics") a.topics = static_cast<std::size_t>(num(v));
    else if (k == "--clusters") a.clusters = static_cast<std::size_t>(num(v));
    else if (k == "--spread") a.spread = num(v);
    else if (k == "--requests") a.requests = static_cast<std::size_t>(num(v));
    else if (k == "--rate") a.rate = num(v);
    else if (k == "--drift") a.drift = num(v);
    else if (k == "--nprobe") a.nprobe = static_cast<std::size_t>(num(v));
    else if (k == "--seed") a.seed = static_cast<std::uint64_t>(num(v));
    else if (k == "--mix") a.mix = v;
    else if (k == "--strategy") a.strategy = v;
    else if (k == "--clock") a.clock = v;
    else if (k == "--per-vector-ns") a.per_vector_ns = num(v);
    else if (k == "--beta-ms") a.beta_ms = num(v);
    else if (k == "--slo-ms") a.slo_ms = num(v);
    else if (k == "--kmeans-iters") a.kmeans_iters = static_cast<std::size_t>(num(v));
    else if (k == "--kmeans-sample") a.kmeans_sample = static_cast<std::size_t>(num(v));
    else if (k == "--cache") a.cache = num(v) != 0;
    else if (k == "--spec") a.spec = num(v) != 0;
    else if (k == "--report") a.report = v;
    else throw std::invalid_argument("unknown option " + k);
  }
  return a;
}

std::map<std::string, double> parse_mix(const std::string& s) {
  std::map<std::string, double> m;
  std::stringstream ss(s);
  std::string part;
  while (std::getline(ss, part, ',')) {
    const auto eq = part.find('=');
    m[part.substr(0, eq)] = eq == std::string::npos ? 1.0 : std::strtod(part.c_str() + eq + 1, nullptr);
  }
  return m;
}

double nearest_rank(std::vector<double> v, double p) {  // report.cpp:15-21
  if (v.empty()) return 0.0;
  std::sort(v.begin(), v.end());
  const double rank = std::ceil(p / 100.0 * static_cast<double>(v.size()));
  const std::size_t idx = rank < 1.0 ? 0 : static_cast<std::size_t>(rank) - 1;
  return v[std::min(idx, v.size() - 1)];
}

double secs(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

}  // namespace

int main(int argc, char** argv) {
  const Args a = parse(argc, argv);
  harness::WorkloadSpec spec;
  spec.corpus.n_vectors = a.n;
  spec.corpus.dim = a.dim;
  spec.corpus.n_topics = a.topics;
  spec.corpus.topic_spread = a.spread;
  spec.corpus.seed = a.seed;
  spec.queries.n_requests = a.requests;
  spec.queries.arrival = "poisson";
  spec.queries.rate_per_s = a.rate;
  spec.queries.zipf_s = 1.0;
  spec.queries.drift_delta = a.drift;
  spec.queries.min_tokens = 6;
  spec.queries.max_tokens = 24;
  spec.queries.seed = a.seed + 1;
  spec.queries.workflow_mix = parse_mix(a.mix);

  auto t0 = std::chrono::steady_clock::now();
  const ivf::Corpus corpus = harness::generate_corpus(spec.corpus);
  const double t_corpus = secs(t0);

  t0 = std::chrono::steady_clock::now();
  ivf::Centroids centroids;
  if (a.kmeans_sample && a.kmeans_sample < corpus.size()) {
    // every (n / sample)-th row: a deterministic training subset
    ivf::Corpus sample;
    sample.dim = corpus.dim;
    const std::size_t stride = corpus.size() / a.kmeans_sample;
    for (std::size_t i = 0; i < a.kmeans_sample; ++i) {
      const float* r = corpus.row(i * stride);
      sample.data.insert(sample.data.end(), r, r + corpus.dim);
      sample.doc_ids.push_back(corpus.doc_ids[i * stride]);
    }
    centroids = ivf::train_kmeans(sample, a.clusters, a.kmeans_iters, a.seed + 2);
  } else {
    centroids = ivf::train_kmeans(corpus, a.clusters, a.kmeans_iters, a.seed + 2);
  }
  const double t_kmeans = secs(t0);
  t0 = std::chrono::steady_clock::now();
  const ivf::IvfIndex index = ivf::build_index(corpus, centroids, Metric::L2);
  const double t_index = secs(t0);
  const harness::RequestTrace trace = harness::generate_workload(spec, corpus);

  sched::SchedulerConfig cfg;
  cfg.strategy = sched::parse_strategy(a.strategy);
  cfg.clock = a.clock == "live" ? sched::ClockMode::Live : sched::ClockMode::Virtual;
  cfg.nprobe = a.nprobe;
  cfg.beta_ms = a.beta_ms;
  cfg.slo_ms = a.slo_ms;
  cfg.speculation = a.spec;
  cfg.cache_enabled = a.cache;
  if (cfg.cache_enabled) cfg.cache_cfg.capacity_gc = std::max<std::size_t>(1, index.k_clusters() / 5);
  if (cfg.speculation) cfg.calibration = bench::calibrate_generation(cfg.gen_latency);
  cfg.seed = a.seed;
  t0 = std::chrono::steady_clock::now();
  if (a.per_vector_ns > 0) {
    cfg.ret_cost.per_vector_ns = a.per_vector_ns;
  } else {
#ifdef HEDRA_GPU_COMPAT
    cfg.ret_cost.per_vector_ns = gpu::measure_per_vector_ns(index);
#else
    cfg.ret_cost.per_vector_ns = bench::measure_per_vector_ns(index);
#endif
  }
  const double t_calib = secs(t0);
#ifdef HEDRA_GPU_COMPAT
  // serving warm-up: device scratch for sub-stages up to 64 items x nprobe
  gpu::reserve_substage(index, 64, a.nprobe, 32);
#endif

  harness::TraceSink sink;
  t0 = std::chrono::steady_clock::now();
  const harness::ExperimentReport report = sched::run(cfg, trace, index, &sink);
  const double t_run = secs(t0);
  if (!a.report.empty()) report.save(a.report);

  std::map<double, std::size_t> substages;  // start time -> items in the sub-stage
  std::map<double, double> substage_ms;
  for (const auto& e : sink.events())
    if (e.worker == "ret" && e.event == "substage") {
      ++substages[e.t_ms];
      substage_ms[e.t_ms] = e.duration_ms;
    }
  std::vector<double> lat, items;
  for (const auto& [t, ms] : substage_ms) lat.push_back(ms);
  // the slowest sub-stages (start time, duration, items): where the tail comes from
  std::vector<std::tuple<double, double, std::size_t>> slow;
  for (const auto& [t, ms] : substage_ms) slow.emplace_back(ms, t, substages[t]);
  std::sort(slow.rbegin(), slow.rend());
  std::string slowest = "[";
  for (std::size_t i = 0; i < slow.size() && i < 12; ++i) {
    char b[96];
    std::snprintf(b, sizeof(b), "%s[%.1f, %.3f, %zu]", i ? ", " : "", std::get<1>(slow[i]), std::get<0>(slow[i]),
                  std::get<2>(slow[i]));
    slowest += b;
  }
  slowest += "]";
  for (const auto& [t, n] : substages) items.push_back(static_cast<double>(n));
  double item_sum = 0.0;
  for (double v : items) item_sum += v;

  std::printf(
      "{\"engine\": \"%s\", \"strategy\": \"%s\", \"clock\": \"%s\", \"corpus\": \"%zux%u\", "
      "\"clusters\": %zu, \"nprobe\": %zu, \"requests\": %zu, \"completed\": %zu, "
      "\"per_vector_ns\": %.6g, \"makespan_ms\": %.3f, \"latency_p50_ms\": %.3f, \"latency_p99_ms\": %.3f, "
      "\"substages\": %zu, \"substage_ms\": {\"p50\": %.4f, \"p99\": %.4f, \"max\": %.4f}, "
      "\"items_per_substage\": {\"mean\": %.2f, \"p50\": %.0f, \"max\": %.0f}, "
      "\"retrieval_stages\": %llu, \"mean_clusters_searched\": %.3f, \"cache_hit_rate\": %.4f, "
      "\"speculation_accuracy\": %.4f, \"setup_s\": {\"corpus\": %.2f, \"kmeans\": %.2f, \"index\": %.2f, "
      "\"calibrate\": %.2f}, \"run_s\": %.3f, \"report_json_bytes\": %zu, "
      "\"slowest_substages_t_ms_items\": %s}\n",
#ifdef HEDRA_GPU_COMPAT
      "gpu",
#else
      "cpu-reference",
#endif
      report.strategy.c_str(), report.clock.c_str(), corpus.size(), corpus.dim, index.k_clusters(), a.nprobe,
      report.requests_admitted, report.requests_completed, cfg.ret_cost.per_vector_ns, report.makespan_ms,
      report.latency_p50_ms, report.latency_p99_ms, lat.size(), nearest_rank(lat, 50), nearest_rank(lat, 99),
      lat.empty() ? 0.0 : *std::max_element(lat.begin(), lat.end()),
      items.empty() ? 0.0 : item_sum / static_cast<double>(items.size()), nearest_rank(items, 50),
      items.empty() ? 0.0 : *std::max_element(items.begin(), items.end()),
      static_cast<unsigned long long>(report.retrieval_stages), report.mean_clusters_searched,
      report.cache_hit_rate.value_or(-1.0), report.speculation_accuracy.value_or(-1.0), t_corpus, t_kmeans, t_index,
      t_calib, t_run, report.to_json().size(), slowest.c_str());
  return 0;
}
