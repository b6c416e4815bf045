// api.cu -- the C-ABI (include/hivf.h): contexts, HBM index, batched search,
// coarse assign, node-split sub-search, shard merge, residency.
//
// No exceptions and no CPU fallback: every compute entry point runs the
// device kernels of this library; failures come back as hivf_status with a
// thread-local message.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "internal.h"

using namespace hivf;

namespace hivf {
std::atomic<uint64_t> g_state_gen{1};
namespace {
thread_local std::string g_err;
}
hivf_status fail(hivf_status st, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return st;
}
}  // namespace hivf

int hivf_index::scan_kind() const {
  const int k = ctx->opt_scan_kernel;
  if (k == 1) return 1;
  if (ctx->tc_conv > 1) return 1;  // unknown tensor-core conversion: FFMA scan
  const int want = k == 2 ? 2 : k == 3 ? 3 : (auto_split ? 2 : 3);
  if (scan_tc_qmax(dpad, want == 2, 0.f, ctx->tc) > 0) return want;
  return 1;  // too wide for the tensor-core scan
}

// Auto policy: the single-pass tf32 bound is 2^-9|x||q| (Cauchy-Schwarz on the
// operand truncation).  When the data's norms are large against its neighbor
// gaps, queries miss the proof and take the segment repair or the exact
// fallback.  Once more than 10% of the queries seen need it, switch this index
// to the split kernel (8x tighter bound, 1.5x slower scan).
static void adapt_scan(hivf_index* ix, uint32_t n_queries, uint32_t n_fallback) {
  if (ix->ctx->opt_scan_kernel != 0 || ix->auto_split) return;
  ix->adapt_seen += n_queries;
  ix->adapt_fallback += n_fallback;
  if (ix->adapt_fallback * 10 > ix->adapt_seen && ix->adapt_fallback >= 2) ix->auto_split = 1;
}

// Rows per scan segment: long segments amortise the per-item costs of the
// grouped scan (query staging, pipeline refill), short ones balance the
// persistent grid and keep the 32 candidates per (query, segment) enough for
// the completeness proof (fewer in-place repairs).  The longest of
// 4096/2048/1024 that still gives >= 16 segments per SM.  Measured with the
// shared drop bound (C3, ms per batch): 4096 -> scan 8.91 + finalize 0.14,
// 8192 -> 8.89 + 0.20; a C3 shard of an 8-GPU job (2.6M rows) gets 1024:
// step 1.46 ms vs 1.81 ms at 4096 (before the bound).
// Tiny indexes (fewer than 2 segments of 1024 rows per SM) take 512-row
// segments so a batch still spreads over the persistent grid: C1 (100k rows)
// 644k -> 669k q/s; C2 (1M rows) stays at 1024 (512 measured 1.5% slower).
static uint32_t auto_seg_rows(uint64_t n_rows, int sm_count) {
  const uint64_t want = 16ull * (uint64_t)std::max(1, sm_count);
  for (uint32_t seg : {4096u, 2048u})
    if (n_rows / seg >= want) return seg;
  if (n_rows / 1024 < 2ull * (uint64_t)std::max(1, sm_count) && kRowBlock <= 512) return 512;
  return 1024;
}

// ---- tiered residency helpers ------------------------------------------------
namespace {
// first-fit allocator over the pool's free extents (host bookkeeping)
uint64_t pool_alloc(hivf_index* ix, uint64_t bytes) {
  bytes = (bytes + 255) & ~uint64_t(255);
  for (size_t i = 0; i < ix->free_ext.size(); ++i) {
    auto& f = ix->free_ext[i];
    if (f.second >= bytes) {
      const uint64_t off = f.first;
      f.first += bytes;
      f.second -= bytes;
      if (!f.second) ix->free_ext.erase(ix->free_ext.begin() + (long)i);
      return off;
    }
  }
  return ~0ull;
}
void pool_free(hivf_index* ix, uint64_t off, uint64_t bytes) {
  if (off == ~0ull) return;
  bytes = (bytes + 255) & ~uint64_t(255);
  auto& v = ix->free_ext;
  v.push_back({off, bytes});
  std::sort(v.begin(), v.end());
  std::vector<std::pair<uint64_t, uint64_t>> m;
  for (auto& e : v) {
    if (!m.empty() && m.back().first + m.back().second == e.first) m.back().second += e.second;
    else m.push_back(e);
  }
  v.swap(m);
}
}  // namespace

// pointer-table updates ride in kernel arguments (no host buffer lifetime):
// ordered on the context stream, so launches before keep the old address
static hivf_status apply_flips(hivf_index* ix, const std::vector<std::pair<uint32_t, const float*>>& f) {
  g_state_gen.fetch_add(1);
  for (size_t b = 0; b < f.size(); b += kPtrFlipBatch) {
    PtrFlips pf{};
    pf.n = (uint32_t)std::min<size_t>(kPtrFlipBatch, f.size() - b);
    for (uint32_t i = 0; i < pf.n; ++i) {
      pf.list[i] = f[b + i].first;
      pf.ptr[i] = f[b + i].second;
    }
    launch_ptr_flips(ix->d_list_ptr, pf, ix->ctx->stream);
    CKL();
  }
  return HIVF_OK;
}

// complete_swaps (tiered_cache.cpp:70-80) on real copies: lists whose H2D
// copy finished become resident (their table entry points at the HBM slot
// for every launch issued from now on)
static void complete_swaps(hivf_index* ix) {
  std::vector<std::pair<uint32_t, const float*>> flips;
  while (!ix->swaps.empty() && cudaEventQuery(ix->swaps.front().done) == cudaSuccess) {
    for (uint32_t c : ix->swaps.front().lists) {
      if (!ix->swap_in[c]) continue;
      ix->swap_in[c] = 0;
      ix->resident[c] = 1;
      flips.push_back({c, reinterpret_cast<const float*>(reinterpret_cast<uint8_t*>(ix->pool) + ix->slot_off[c])});
    }
    cudaEventDestroy(ix->swaps.front().done);
    ix->swaps.erase(ix->swaps.begin());
  }
  if (!flips.empty()) apply_flips(ix, flips);
}

extern "C" {

const char* hivf_last_error(void) { return g_err.c_str(); }
const char* hivf_version(void) { return "hivf 0.1.0 (sm_100a)"; }

hivf_status hivf_ctx_create(int device, void* stream, hivf_ctx** out) {
  if (!out) return fail(HIVF_EINVAL, "hivf_ctx_create: out is NULL");
  int n = 0;
  CK(cudaGetDeviceCount(&n));
  if (device < 0 || device >= n) return fail(HIVF_EINVAL, "hivf_ctx_create: no device %d", device);
  CK(cudaSetDevice(device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    return fail(HIVF_EUNSUPPORTED, "hivf: device %d is sm_%d%d, this build is sm_100a only", device,
                prop.major, prop.minor);
  auto* c = new hivf_ctx;
  c->device = device;
  c->sm_count = prop.multiProcessorCount;
  if (stream) {
    c->stream = static_cast<cudaStream_t>(stream);
  } else {
    cudaError_t e = cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
      delete c;
      return fail(HIVF_ECUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
    }
    c->own_stream = true;
  }
  c->tc_conv = tc_conversion_mode();  // probed once per device
  // process default of option "filter_h16" (env HIVF_FILTER_H16=0 runs every
  // scan on the fp32 lists, e.g. the whole GPU suite on that path)
  if (const char* e = getenv("HIVF_FILTER_H16")) c->opt_h16 = atoi(e) != 0;
  if (const char* e = getenv("HIVF_COARSE_TC")) c->opt_coarse_tc = std::min(2, std::max(0, atoi(e)));
  if (const char* e = getenv("HIVF_COARSE_SET")) c->opt_coarse_set = atoi(e) != 0;
  *out = c;
  return HIVF_OK;
}

hivf_status hivf_device_info(hivf_ctx* ctx, int* sm_count, int* tc_tf32_conversion) {
  if (!ctx) return fail(HIVF_EINVAL, "ctx is NULL");
  if (sm_count) *sm_count = ctx->sm_count;
  if (tc_tf32_conversion) *tc_tf32_conversion = ctx->tc_conv;
  return HIVF_OK;
}

hivf_status hivf_ctx_destroy(hivf_ctx* ctx) {
  if (!ctx) return HIVF_OK;
  cudaSetDevice(ctx->device);
  cudaStreamSynchronize(ctx->stream);
  delete ctx;
  return HIVF_OK;
}

hivf_status hivf_ctx_set_stream(hivf_ctx* ctx, void* stream) {
  if (!ctx) return fail(HIVF_EINVAL, "ctx is NULL");
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  ctx->own_stream = false;
  ctx->stream = static_cast<cudaStream_t>(stream);
  if (!stream) {
    CK(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
    ctx->own_stream = true;
  }
  return HIVF_OK;
}

hivf_status hivf_ctx_synchronize(hivf_ctx* ctx) {
  if (!ctx) return fail(HIVF_EINVAL, "ctx is NULL");
  CK(cudaStreamSynchronize(ctx->stream));
  return HIVF_OK;
}

hivf_status hivf_set_option(hivf_ctx* ctx, const char* name, int64_t value) {
  if (!ctx || !name) return fail(HIVF_EINVAL, "hivf_set_option: NULL argument");
  g_state_gen.fetch_add(1);  // any option may change what a captured search graph launches
  if (!strcmp(name, "search_graph")) {
    ctx->opt_search_graph = value != 0;
  } else if (!strcmp(name, "seed_rows")) {  // rows per query seeding the drop bound (0 off, <= 64)
    if (value < 0 || value > 64) return fail(HIVF_EINVAL, "seed_rows must be in [0, 64]");
    ctx->opt_seed_rows = (uint32_t)value;
  } else if (!strcmp(name, "seed_ppl")) {  // probes per list from which the seed runs
    ctx->opt_seed_ppl = (float)value;
  } else if (!strcmp(name, "coarse_set")) {  // 1: the search's coarse select re-ranks only its uncertain band
    ctx->opt_coarse_set = value != 0;
  } else if (!strcmp(name, "coarse_tc")) {  // tensor-core coarse pass: 0 never, 1 from 2^26 multiply-adds, 2 always
    if (value < 0 || value > 2) return fail(HIVF_EINVAL, "coarse_tc must be 0, 1 or 2");
    ctx->opt_coarse_tc = (int)value;
  } else if (!strcmp(name, "filter_h16")) {  // 1: fp16 filter copy built at index finish and used
    ctx->opt_h16 = value != 0;
  } else if (!strcmp(name, "seg_rows")) {  // 0: automatic (auto_seg_rows)
    if (value != 0 && (value < kRowBlock || value % kRowBlock))
      return fail(HIVF_EINVAL, "seg_rows must be a multiple of %d", kRowBlock);
    ctx->opt_seg_rows = (uint32_t)value;
  } else if (!strcmp(name, "force_exact")) {
    ctx->opt_force_exact = value != 0;
  } else if (!strcmp(name, "hbm_list_budget")) {  // bytes; applies to indexes created later
    if (value < 0) return fail(HIVF_EINVAL, "hbm_list_budget must be >= 0");
    ctx->opt_hbm_list_budget = (uint64_t)value;
  } else if (!strcmp(name, "no_bound")) {
    ctx->opt_no_bound = value != 0;
  } else if (!strcmp(name, "scan_ctas")) {
    ctx->opt_scan_ctas = (int)value;
  } else if (!strcmp(name, "scan_kernel")) {
    if (value < 0 || value > 3)
      return fail(HIVF_EINVAL, "scan_kernel: 0 auto, 1 ffma, 2 tc split, 3 tc single-pass");
    ctx->opt_scan_kernel = (int)value;
  } else if (!strcmp(name, "tc_prof")) {  // debug: stall counters (hivf_debug_tc_prof)
    set_tc_prof((int)value);
  } else if (!strcmp(name, "tc_variant")) {  // debug only: results are inexact when != 0
    ctx->tc.variant = (int)value;
  } else if (!strcmp(name, "tc_qmax")) {  // tuning: queries per tensor-core work item
    if (value < 0 || (value > 32 && !tc_is_wide((uint32_t)value)) || value % 8)
      return fail(HIVF_EINVAL, "tc_qmax: 0, 8..32 step 8, 64, 128 or 256 (wide)");
    ctx->tc.qmax_override = (uint32_t)value;
  } else if (!strcmp(name, "tc_wide_ppl")) {  // tuning: probes/list above which dense batches use
    ctx->tc.wide_ppl = (float)value;           // the wide (64-query) scan; negative = never
  } else if (!strcmp(name, "tc_wide2_ppl")) {  // tuning: probes/list above which the 128-query
    ctx->tc.wide2_ppl = (float)value;          // groups are used; negative = never
  } else if (!strcmp(name, "tc_pair_ppl")) {   // tuning: probes/list above which 256-query groups
    ctx->tc.pair_ppl = (float)value;           // run on CTA pairs (k_scan_pair); negative = never
  } else if (!strcmp(name, "time_kernels")) {
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->resolve_timers();
    ctx->opt_time = value != 0;
  } else if (!strcmp(name, "reset_timers")) {
    CK(cudaStreamSynchronize(ctx->stream));
    ctx->ev_used = 0;
    ctx->timed_calls = 0;
    ctx->acc_assign = ctx->acc_scan = ctx->acc_fin = 0;
  } else {
    return fail(HIVF_EINVAL, "hivf_set_option: unknown option '%s'", name);
  }
  return HIVF_OK;
}

hivf_status hivf_last_stats(hivf_ctx* ctx, hivf_stats* out) {
  if (!ctx || !out) return fail(HIVF_EINVAL, "NULL argument");
  CK(cudaStreamSynchronize(ctx->stream));
  ctx->resolve_timers();
  hivf_stats s = ctx->stats;
  s.timed_calls = ctx->timed_calls;
  s.assign_ms = ctx->acc_assign;
  s.scan_ms = ctx->acc_scan;
  s.finalize_ms = ctx->acc_fin;
  const DBuf& nit = ctx->n_items;
  const DBuf& lcnt = ctx->list_cnt;
  if (nit.p) CK(cudaMemcpy(&s.n_work_items, nit.p, 4, cudaMemcpyDeviceToHost));
  if (ctx->last_index && lcnt.p && ctx->last_K == ctx->last_index->K) {
    std::vector<uint32_t> cnt(ctx->last_K);
    CK(cudaMemcpy(cnt.data(), lcnt.p, 4ull * ctx->last_K, cudaMemcpyDeviceToHost));
    s.n_unique_lists = 0;
    s.scan_bytes = 0;
    const auto& off = ctx->last_index->list_off;
    for (uint32_t c = 0; c < ctx->last_K; ++c)
      if (cnt[c]) {
        ++s.n_unique_lists;
        s.scan_bytes += (off[c + 1] - off[c]) * (uint64_t)ctx->last_index->dim * (ctx->last_filter_bits / 8);
      }
  }
  if (ctx->last_nq && ctx->flags_f.p && ctx->flags_c.p) {
    std::vector<int> f(ctx->last_nq), g(ctx->last_nq);
    CK(cudaMemcpy(f.data(), ctx->flags_f.p, 4ull * ctx->last_nq, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(g.data(), ctx->flags_c.p, 4ull * ctx->last_nq, cudaMemcpyDeviceToHost));
    s.n_fallback = 0;
    uint32_t scan_fb = 0;
    for (uint32_t i = 0; i < ctx->last_nq; ++i) {
      s.n_fallback += (f[i] != 0) + (g[i] != 0);
      scan_fb += f[i] != 0;
    }
    if (ctx->last_index && !ctx->stats_adapted) {
      adapt_scan(const_cast<hivf_index*>(ctx->last_index), ctx->last_nq, scan_fb);
      ctx->stats_adapted = true;
    }
  }
  s.scan_kernel = ctx->last_kind;
  s.scan_group = ctx->last_group;
  s.scan_filter_bits = ctx->last_filter_bits;
  s.coarse_filter_bits = ctx->last_coarse_bits;
  *out = s;
  return HIVF_OK;
}

// ---------------------------------------------------------------------------
// index build
// ---------------------------------------------------------------------------

// fp16 centroid copy for the tensor-core coarse pass (scan_tc.cu,
// k_coarse_dist_tc): one power-of-2 scale from the largest centroid norm
// bound.  Optional: without it (scale out of range, no memory) the coarse
// distances stay on the FFMA pass.
static void build_coarse_h16(hivf_index* ix) {
  std::vector<float> cn(ix->K);
  if (cudaMemcpy(cn.data(), ix->cnorm, ix->K * 4ull, cudaMemcpyDeviceToHost) != cudaSuccess) return;
  float cmax = 0.f;
  for (float v : cn) cmax = std::max(cmax, v);
  const int e = h16_exp(cmax);
  if (e < -kH16ExpMax || e > kH16ExpMax) return;
  const float csc = std::ldexp(1.f, -e);
  uint8_t* d = nullptr;
  if (cudaMalloc(&d, coarse_tc_bytes(ix->K, ix->dpad)) != cudaSuccess) {
    (void)cudaGetLastError();
    return;
  }
  launch_pack_coarse_tc(ix->cent, ix->K, ix->dpad, nullptr, csc, d, ix->ctx->stream);
  if (cudaStreamSynchronize(ix->ctx->stream) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
    cudaFree(d);
    return;
  }
  ix->centh = d;
  ix->csc = csc;
  ix->cmax = cmax;
}

hivf_status hivf_index_begin(hivf_ctx* ctx, uint32_t dim, int metric, uint32_t n_clusters,
                             const float* centroids, int centroids_on_device,
                             const uint64_t* list_offsets, hivf_index** out) {
  if (!ctx || !out || !centroids || !list_offsets) return fail(HIVF_EINVAL, "hivf_index_begin: NULL argument");
  if (dim == 0) return fail(HIVF_EINVAL, "index: dim must be >= 1");
  if (n_clusters == 0) return fail(HIVF_EINVAL, "index: n_clusters must be >= 1");
  if (metric != HIVF_METRIC_L2 && metric != HIVF_METRIC_COSINE) return fail(HIVF_EINVAL, "index: unknown metric %d", metric);
  if (list_offsets[0] != 0) return fail(HIVF_EINVAL, "index: list_offsets[0] must be 0");
  for (uint32_t c = 0; c < n_clusters; ++c)
    if (list_offsets[c + 1] < list_offsets[c]) return fail(HIVF_EINVAL, "index: list_offsets not monotone at %u", c);
  const uint64_t N = list_offsets[n_clusters];
  if (N >= 0xffffffffull) return fail(HIVF_EUNSUPPORTED, "index: more than 2^32-2 vectors per device");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  auto* ix = new hivf_index;
  ix->ctx = ctx;
  ix->dim = dim;
  ix->dpad = (dim + kChunk - 1) / kChunk * kChunk;
  ix->K = n_clusters;
  ix->metric = metric;
  ix->N = N;
  ix->list_off.assign(list_offsets, list_offsets + n_clusters + 1);
  ix->resident.assign(n_clusters, 0);
  uint64_t maxn = 0;
  for (uint32_t c = 0; c < n_clusters; ++c) maxn = std::max(maxn, list_offsets[c + 1] - list_offsets[c]);
  ix->seg_rows = ctx->opt_seg_rows ? ctx->opt_seg_rows : auto_seg_rows(N, ctx->sm_count);
  ix->s_max = (uint32_t)std::max<uint64_t>(1, (maxn + ix->seg_rows - 1) / ix->seg_rows);
  auto bail = [&](cudaError_t e, const char* what) {
    delete ix;
    return fail(e == cudaErrorMemoryAllocation ? HIVF_ENOMEM : HIVF_ECUDA, "%s: %s", what, cudaGetErrorString(e));
  };
  cudaError_t e;
  const uint64_t vec_bytes = std::max<uint64_t>(16, N * ix->dpad * 4);
  if (ctx->opt_hbm_list_budget && ctx->opt_hbm_list_budget < vec_bytes) {
    // tiered: backing store in pinned, device-mapped host memory (UVA: the same
    // address on both sides; the build kernels write it over PCIe), plus an
    // HBM pool of `budget` bytes for the resident (hot) lists
    ix->tiered = true;
    ix->pool_bytes = ctx->opt_hbm_list_budget & ~uint64_t(255);
    if ((e = cudaHostAlloc(&ix->vec, vec_bytes, cudaHostAllocMapped | cudaHostAllocPortable)) != cudaSuccess) {
      ix->vec = nullptr;
      return bail(e, "alloc host backing store");
    }
    if ((e = cudaMalloc(&ix->pool, std::max<uint64_t>(256, ix->pool_bytes))) != cudaSuccess) return bail(e, "alloc list pool");
    if ((e = cudaMalloc(&ix->d_list_ptr, n_clusters * 8ull)) != cudaSuccess) return bail(e, "alloc list table");
    std::vector<uint64_t> ptr(n_clusters);
    for (uint32_t c = 0; c < n_clusters; ++c)
      ptr[c] = reinterpret_cast<uint64_t>(ix->vec + list_offsets[c] * ix->dpad);
    cudaMemcpy(ix->d_list_ptr, ptr.data(), n_clusters * 8ull, cudaMemcpyHostToDevice);
    ix->slot_off.assign(n_clusters, ~0ull);
    ix->swap_in.assign(n_clusters, 0);
    ix->free_ext.push_back({0, ix->pool_bytes});
    if ((e = cudaStreamCreateWithFlags(&ix->copy_stream, cudaStreamNonBlocking)) != cudaSuccess) return bail(e, "copy stream");
  } else if ((e = cudaMalloc(&ix->vec, vec_bytes)) != cudaSuccess) {
    return bail(e, "alloc lists");
  }
  if ((e = cudaMalloc(&ix->ids, std::max<uint64_t>(8, N * 8))) != cudaSuccess) return bail(e, "alloc ids");
  if ((e = cudaMalloc(&ix->xnorm2, std::max<uint64_t>(4, N * 4))) != cudaSuccess) return bail(e, "alloc norms");
  if ((e = cudaMalloc(&ix->d_list_off, (n_clusters + 1) * 8ull)) != cudaSuccess) return bail(e, "alloc offsets");
  if ((e = cudaMalloc(&ix->maxnorm_bits, n_clusters * 4ull)) != cudaSuccess) return bail(e, "alloc maxnorm");
  if ((e = cudaMalloc(&ix->cent, (uint64_t)n_clusters * ix->dpad * 4)) != cudaSuccess) return bail(e, "alloc centroids");
  if ((e = cudaMalloc(&ix->cnorm2, n_clusters * 4ull)) != cudaSuccess) return bail(e, "alloc cnorm2");
  if ((e = cudaMalloc(&ix->cnorm, n_clusters * 4ull)) != cudaSuccess) return bail(e, "alloc cnorm");
  if ((e = cudaMalloc(&ix->list_order, n_clusters * 4ull)) != cudaSuccess) return bail(e, "alloc order");
  if ((e = cudaMalloc(&ix->d_err, 4)) != cudaSuccess) return bail(e, "alloc err");
  cudaMemsetAsync(ix->d_err, 0, 4, s);
  cudaMemsetAsync(ix->maxnorm_bits, 0, n_clusters * 4ull, s);
  cudaMemcpyAsync(ix->d_list_off, list_offsets, (n_clusters + 1) * 8ull, cudaMemcpyHostToDevice, s);
  // lists by size, descending (LPT order for the scan work list)
  std::vector<uint32_t> order(n_clusters);
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) {
    return list_offsets[a + 1] - list_offsets[a] > list_offsets[b + 1] - list_offsets[b];
  });
  cudaMemcpyAsync(ix->list_order, order.data(), n_clusters * 4ull, cudaMemcpyHostToDevice, s);
  const float* dcent = centroids;
  float* tmp = nullptr;
  if (!centroids_on_device) {
    if ((e = cudaMalloc(&tmp, (uint64_t)n_clusters * dim * 4)) != cudaSuccess) return bail(e, "alloc tmp");
    cudaMemcpyAsync(tmp, centroids, (uint64_t)n_clusters * dim * 4, cudaMemcpyHostToDevice, s);
    dcent = tmp;
  }
  launch_pack_centroids(dcent, n_clusters, dim, ix->dpad, ix->cent, ix->cnorm2, ix->cnorm, ix->d_err, s);
  e = cudaStreamSynchronize(s);
  if (tmp) cudaFree(tmp);
  if (e != cudaSuccess) return bail(e, "pack centroids");
  if ((e = cudaGetLastError()) != cudaSuccess) return bail(e, "pack centroids launch");
  if (ctx->opt_coarse_tc && ctx->tc_conv <= 1) build_coarse_h16(ix);
  *out = ix;
  return HIVF_OK;
}

hivf_status hivf_index_add_rows_device(hivf_index* ix, uint64_t first_row, uint64_t n_rows,
                                       const float* d_rows, const uint64_t* d_ids) {
  if (!ix || (!d_rows && n_rows)) return fail(HIVF_EINVAL, "hivf_index_add_rows_device: NULL argument");
  if (ix->finished) return fail(HIVF_EINVAL, "index already finished");
  if (first_row + n_rows > ix->N) return fail(HIVF_EINVAL, "add_rows: rows [%llu, %llu) beyond N=%llu",
                                               (unsigned long long)first_row,
                                               (unsigned long long)(first_row + n_rows),
                                               (unsigned long long)ix->N);
  if (!n_rows) return HIVF_OK;
  cudaStream_t s = ix->ctx->stream;
  CK(cudaSetDevice(ix->ctx->device));
  launch_pack_lists(d_rows, first_row, nullptr, n_rows, ix->dim, ix->dpad, ix->d_list_off, ix->K,
                    ix->vec, ix->xnorm2, ix->maxnorm_bits, ix->d_err, s);
  CKL();
  if (d_ids) CK(cudaMemcpyAsync(ix->ids + first_row, d_ids, n_rows * 8, cudaMemcpyDeviceToDevice, s));
  ix->rows_added += n_rows;
  return HIVF_OK;
}

hivf_status hivf_index_add_rows_at_device(hivf_index* ix, uint64_t n_rows,
                                          const uint64_t* d_positions, const float* d_rows,
                                          const uint64_t* d_ids) {
  if (!ix || (n_rows && (!d_rows || !d_positions)))
    return fail(HIVF_EINVAL, "hivf_index_add_rows_at_device: NULL argument");
  if (ix->finished) return fail(HIVF_EINVAL, "index already finished");
  if (ix->rows_added + n_rows > ix->N) return fail(HIVF_EINVAL, "add_rows_at: more rows than N");
  if (!n_rows) return HIVF_OK;
  cudaStream_t s = ix->ctx->stream;
  CK(cudaSetDevice(ix->ctx->device));
  launch_pack_lists(d_rows, 0, d_positions, n_rows, ix->dim, ix->dpad, ix->d_list_off, ix->K,
                    ix->vec, ix->xnorm2, ix->maxnorm_bits, ix->d_err, s);
  CKL();
  if (d_ids) {
    launch_scatter_ids(d_ids, d_positions, n_rows, ix->ids, s);
    CKL();
  }
  ix->rows_added += n_rows;
  return HIVF_OK;
}

hivf_status hivf_index_get_rows(hivf_index* ix, uint64_t first_row, uint64_t n_rows,
                                float* rows_out, uint64_t* ids_out) {
  if (!ix) return fail(HIVF_EINVAL, "index is NULL");
  if (first_row + n_rows > ix->N) return fail(HIVF_EINVAL, "get_rows: range beyond N");
  if (!n_rows) return HIVF_OK;
  cudaStream_t s = ix->ctx->stream;
  CK(cudaSetDevice(ix->ctx->device));
  const uint64_t per = std::max<uint64_t>(1, (256ull << 20) / (4ull * ix->dim));
  float* tmp = nullptr;
  CK(cudaMalloc(&tmp, std::min(per, n_rows) * ix->dim * 4));
  for (uint64_t r = 0; r < n_rows; r += per) {
    const uint64_t n = std::min(per, n_rows - r);
    launch_unpack_rows(ix->vec, ix->d_list_off, ix->K, ix->dim, ix->dpad, first_row + r, n, tmp, s);
    if (rows_out) cudaMemcpyAsync(rows_out + r * ix->dim, tmp, n * ix->dim * 4, cudaMemcpyDeviceToHost, s);
    cudaStreamSynchronize(s);
  }
  cudaFree(tmp);
  if (ids_out) CK(cudaMemcpyAsync(ids_out, ix->ids + first_row, n_rows * 8, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return HIVF_OK;
}

// fp16 filter copy: per-list power-of-2 scale
// from the list's norm bound, then the rows rounded to fp16 in the scan layout.
// Optional: skipped -- the scan then reads the fp32 lists -- when a list's
// scale is out of range or HBM is short.  Tiered (host-backed) indexes keep
// the WHOLE filter copy in HBM (half the fp32 bytes, outside hbm_list_budget):
// every scan streams from HBM, and only the exact re-rank / repair / fallback
// reads of cold lists' fp32 rows cross PCIe ("two lanes").
static void build_h16(hivf_index* ix) {
  if (ix->N == 0) return;
  cudaStream_t s = ix->ctx->stream;
  std::vector<float> mx(ix->K);
  if (cudaMemcpy(mx.data(), ix->maxnorm_bits, ix->K * 4ull, cudaMemcpyDeviceToHost) != cudaSuccess) return;
  std::vector<float> sc(ix->K);
  for (uint32_t c = 0; c < ix->K; ++c) {
    const int e = h16_exp(mx[c]);
    if (e < -kH16ExpMax || e > kH16ExpMax) return;
    sc[c] = std::ldexp(1.f, -e);
  }
  const uint32_t dph = (ix->dim + 31) / 32 * 32;
  ix->dpf = dph / 2;
  if (cudaMalloc(&ix->vech, ix->N * ix->dpf * 4ull) != cudaSuccess ||
      cudaMalloc(&ix->lsc, ix->K * 4ull) != cudaSuccess) {
    (void)cudaGetLastError();
    cudaFree(ix->vech);
    cudaFree(ix->lsc);
    ix->vech = ix->lsc = nullptr;
    return;
  }
  cudaMemcpyAsync(ix->lsc, sc.data(), ix->K * 4ull, cudaMemcpyHostToDevice, s);
  launch_pack_h16(ix->vec, ix->d_list_off, ix->K, ix->dpad, ix->dpf, ix->N, ix->lsc, ix->vech, s);
  if (cudaStreamSynchronize(s) != cudaSuccess || cudaGetLastError() != cudaSuccess) {
    cudaFree(ix->vech);
    cudaFree(ix->lsc);
    ix->vech = ix->lsc = nullptr;
  }
}

hivf_status hivf_index_finish(hivf_index* ix) {
  if (!ix) return fail(HIVF_EINVAL, "index is NULL");
  cudaStream_t s = ix->ctx->stream;
  CK(cudaSetDevice(ix->ctx->device));
  if (ix->rows_added != ix->N)
    return fail(HIVF_EINVAL, "index_finish: %llu of %llu rows added", (unsigned long long)ix->rows_added,
                (unsigned long long)ix->N);
  if (ix->N > 1) {  // duplicate doc ids -> invalid_argument (vector_index.cpp:240-244)
    uint64_t* sorted = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
    CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp_bytes, ix->ids, sorted, (int64_t)ix->N, 0, 64, s));
    CK(cudaMalloc(&sorted, ix->N * 8));
    CK(cudaMalloc(&tmp, tmp_bytes));
    CK(cub::DeviceRadixSort::SortKeys(tmp, tmp_bytes, ix->ids, sorted, (int64_t)ix->N, 0, 64, s));
    launch_check_dup_ids(sorted, ix->N, ix->d_err, s);
    CK(cudaStreamSynchronize(s));
    cudaFree(sorted);
    cudaFree(tmp);
  }
  int err = 0;
  CK(cudaMemcpyAsync(&err, ix->d_err, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (err == 1) return fail(HIVF_EINVAL, "index: non-finite value in vectors or centroids");
  if (err == 2) return fail(HIVF_EINVAL, "build_index: duplicate doc_id");
  if (ix->ctx->opt_h16) build_h16(ix);
  ix->finished = true;
  return HIVF_OK;
}

static hivf_status upload_common(hivf_ctx* ctx, uint32_t dim, int metric, uint32_t n_clusters,
                                 const float* centroids, int cent_dev, const uint64_t* list_offsets,
                                 const float* vectors, const uint64_t* ids, bool dev,
                                 hivf_index** out) {
  g_state_gen.fetch_add(1);
  if (!out) return fail(HIVF_EINVAL, "out is NULL");
  hivf_index* ix = nullptr;
  hivf_status st = hivf_index_begin(ctx, dim, metric, n_clusters, centroids, cent_dev, list_offsets, &ix);
  if (st != HIVF_OK) return st;
  const uint64_t N = ix->N;
  if (N && (!vectors || !ids)) {
    hivf_index_destroy(ix);
    return fail(HIVF_EINVAL, "index: vectors/ids NULL");
  }
  if (dev) {
    st = hivf_index_add_rows_device(ix, 0, N, vectors, ids);
  } else {
    // stage host rows through a bounded device buffer (256 MB chunks)
    const uint64_t rows_per = std::max<uint64_t>(1, (256ull << 20) / (4ull * dim));
    float* drows = nullptr;
    uint64_t* dids = nullptr;
    cudaError_t e = cudaMalloc(&drows, std::min(rows_per, std::max<uint64_t>(N, 1)) * dim * 4);
    if (e == cudaSuccess) e = cudaMalloc(&dids, std::min(rows_per, std::max<uint64_t>(N, 1)) * 8);
    if (e != cudaSuccess) {
      if (drows) cudaFree(drows);
      hivf_index_destroy(ix);
      return fail(HIVF_ENOMEM, "index staging: %s", cudaGetErrorString(e));
    }
    for (uint64_t r = 0; r < N && st == HIVF_OK; r += rows_per) {
      const uint64_t n = std::min(rows_per, N - r);
      cudaMemcpyAsync(drows, vectors + r * dim, n * dim * 4, cudaMemcpyHostToDevice, ctx->stream);
      cudaMemcpyAsync(dids, ids + r, n * 8, cudaMemcpyHostToDevice, ctx->stream);
      st = hivf_index_add_rows_device(ix, r, n, drows, dids);
      cudaStreamSynchronize(ctx->stream);
    }
    cudaFree(drows);
    cudaFree(dids);
  }
  if (st == HIVF_OK) st = hivf_index_finish(ix);
  if (st != HIVF_OK) {
    std::string keep = g_err;
    hivf_index_destroy(ix);
    g_err = keep;
    return st;
  }
  *out = ix;
  return HIVF_OK;
}

hivf_status hivf_index_upload(hivf_ctx* ctx, uint32_t dim, int metric, uint32_t n_clusters,
                              const float* centroids, const uint64_t* list_offsets,
                              const float* vectors, const uint64_t* ids, hivf_index** out) {
  return upload_common(ctx, dim, metric, n_clusters, centroids, 0, list_offsets, vectors, ids, false, out);
}

hivf_status hivf_index_upload_device(hivf_ctx* ctx, uint32_t dim, int metric,
                                     uint32_t n_clusters, const float* d_centroids,
                                     const uint64_t* list_offsets, const float* d_vectors,
                                     const uint64_t* d_ids, hivf_index** out) {
  return upload_common(ctx, dim, metric, n_clusters, d_centroids, 1, list_offsets, d_vectors, d_ids, true, out);
}

hivf_status hivf_index_destroy(hivf_index* ix) {
  if (!ix) return HIVF_OK;
  g_state_gen.fetch_add(1);
  cudaSetDevice(ix->ctx->device);
  cudaStreamSynchronize(ix->ctx->stream);
  delete ix;
  return HIVF_OK;
}

hivf_status hivf_index_locate(hivf_index* ix, const uint64_t* doc_ids, uint32_t n, uint32_t* clusters_out,
                              uint64_t* rows_out) {
  if (!ix || (n && (!doc_ids || !clusters_out || !rows_out))) return fail(HIVF_EINVAL, "hivf_index_locate: NULL argument");
  if (!ix->finished) return fail(HIVF_EINVAL, "index not finished");
  if (!n) return HIVF_OK;
  CK(cudaSetDevice(ix->ctx->device));
  cudaStream_t s = ix->ctx->stream;
  if (!ix->loc_ids && ix->N) {  // sorted (id, row) table, once
    uint64_t* rows = nullptr;
    void* tmp = nullptr;
    size_t tb = 0;
    CK(cudaMalloc(&ix->loc_ids, ix->N * 8));
    CK(cudaMalloc(&ix->loc_rows, ix->N * 8));
    CK(cudaMalloc(&rows, ix->N * 8));
    launch_iota64(rows, ix->N, s);
    CK(cub::DeviceRadixSort::SortPairs(nullptr, tb, ix->ids, ix->loc_ids, rows, ix->loc_rows, (int64_t)ix->N, 0, 64, s));
    CK(cudaMalloc(&tmp, tb));
    CK(cub::DeviceRadixSort::SortPairs(tmp, tb, ix->ids, ix->loc_ids, rows, ix->loc_rows, (int64_t)ix->N, 0, 64, s));
    CK(cudaStreamSynchronize(s));
    cudaFree(tmp);
    cudaFree(rows);
  }
  hivf_ctx* c = ix->ctx;
  CK(c->x_ids.ensure((size_t)n * 8 * 2));
  CK(c->x_cnt.ensure((size_t)n * 4));
  uint64_t* dq = c->x_ids.as<uint64_t>();
  CK(cudaMemcpyAsync(dq, doc_ids, n * 8ull, cudaMemcpyHostToDevice, s));
  if (ix->N) {
    launch_locate(ix->loc_ids, ix->loc_rows, ix->N, ix->d_list_off, ix->K, dq, n, c->x_cnt.as<uint32_t>(), dq + n, s);
    CKL();
    CK(cudaMemcpyAsync(clusters_out, c->x_cnt.p, n * 4ull, cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(rows_out, dq + n, n * 8ull, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  } else {
    for (uint32_t i = 0; i < n; ++i) {
      clusters_out[i] = 0xffffffffu;
      rows_out[i] = ~0ull;
    }
  }
  return HIVF_OK;
}

hivf_status hivf_index_gather_rows(hivf_index* ix, const uint64_t* rows, uint32_t n, float* rows_out) {
  if (!ix || (n && (!rows || !rows_out))) return fail(HIVF_EINVAL, "hivf_index_gather_rows: NULL argument");
  for (uint32_t i = 0; i < n; ++i)
    if (rows[i] >= ix->N) return fail(HIVF_EINVAL, "hivf_index_gather_rows: row %llu out of range", (unsigned long long)rows[i]);
  if (!n) return HIVF_OK;
  CK(cudaSetDevice(ix->ctx->device));
  cudaStream_t s = ix->ctx->stream;
  hivf_ctx* c = ix->ctx;
  if (ix->tiered) complete_swaps(ix);
  CK(c->x_ids.ensure((size_t)n * 8));
  CK(c->x_d.ensure((size_t)n * ix->dim * 4));
  CK(cudaMemcpyAsync(c->x_ids.p, rows, n * 8ull, cudaMemcpyHostToDevice, s));
  launch_gather_rows(ix->view(), c->x_ids.as<uint64_t>(), n, c->x_d.as<float>(), s);
  CKL();
  CK(cudaMemcpyAsync(rows_out, c->x_d.p, (size_t)n * ix->dim * 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return HIVF_OK;
}

hivf_status hivf_index_row_distances(hivf_index* ix, double* dist_out) {
  if (!ix || !dist_out) return fail(HIVF_EINVAL, "hivf_index_row_distances: NULL argument");
  if (!ix->N) return HIVF_OK;
  if (ix->tiered) return fail(HIVF_EUNSUPPORTED, "hivf_index_row_distances: index has a host backing store");
  CK(cudaSetDevice(ix->ctx->device));
  cudaStream_t s = ix->ctx->stream;
  const uint32_t np = 1024;
  double* d = nullptr;
  CK(cudaMalloc(&d, (size_t)(ix->N + np) * 8));
  launch_mean_assigned(ix->view(), d + ix->N, np, s, d);
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaMemcpyAsync(dist_out, d, (size_t)ix->N * 8, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  cudaFree(d);
  if (e != cudaSuccess) return fail(HIVF_ECUDA, "hivf_index_row_distances: %s", cudaGetErrorString(e));
  return HIVF_OK;
}

hivf_status hivf_index_info(const hivf_index* cix, uint32_t* dim, uint32_t* n_clusters,
                            uint64_t* n_vectors, uint64_t* hbm_bytes,
                            double* mean_assigned_distance) {
  if (!cix) return fail(HIVF_EINVAL, "index is NULL");
  auto* ix = const_cast<hivf_index*>(cix);
  if (dim) *dim = ix->dim;
  if (n_clusters) *n_clusters = ix->K;
  if (n_vectors) *n_vectors = ix->N;
  if (hbm_bytes)
    *hbm_bytes = ix->N * (ix->dpad * 4ull + 8 + 4) + (uint64_t)ix->K * (ix->dpad * 4ull + 8 + 16);
  if (mean_assigned_distance) {
    if (ix->mean_assigned < 0) {
      const uint32_t np = 1024;
      double* part = nullptr;
      CK(cudaMalloc(&part, np * 8));
      launch_mean_assigned(ix->view(), part, np, ix->ctx->stream);
      std::vector<double> h(np);
      CK(cudaMemcpyAsync(h.data(), part, np * 8, cudaMemcpyDeviceToHost, ix->ctx->stream));
      CK(cudaStreamSynchronize(ix->ctx->stream));
      cudaFree(part);
      double sum = 0;
      for (double v : h) sum += v;
      ix->mean_assigned = ix->N ? sum / (double)ix->N : 0.0;
    }
    *mean_assigned_distance = ix->mean_assigned;
  }
  return HIVF_OK;
}

hivf_status hivf_index_cluster_sizes(const hivf_index* ix, uint64_t* sizes_out) {
  if (!ix || !sizes_out) return fail(HIVF_EINVAL, "NULL argument");
  for (uint32_t c = 0; c < ix->K; ++c) sizes_out[c] = ix->list_off[c + 1] - ix->list_off[c];
  return HIVF_OK;
}

// ---------------------------------------------------------------------------
// search
// ---------------------------------------------------------------------------

static hivf_status prep_queries(hivf_index* ix, const float* d_q, uint32_t n, bool normalize,
                                QueryView* qv) {
  hivf_ctx* c = ix->ctx;
  CK(c->qs.ensure((size_t)n * ix->dpad * 4));
  CK(c->qn2.ensure((size_t)n * 4));
  CK(c->qnorm.ensure((size_t)n * 4));
  CK(c->qsc.ensure((size_t)n * 4));
  CK(c->err.ensure(4));
  launch_prep_queries(d_q, n, ix->dim, ix->dpad, ix->metric, normalize, c->qs.as<float>(),
                      c->qn2.as<float>(), c->qnorm.as<float>(), c->qsc.as<float>(), c->err.as<int>(),
                      c->stream);
  CKL();
  c->stats.kernels_launched += 1;
  qv->qs = c->qs.as<float>();
  qv->qn2 = c->qn2.as<float>();
  qv->qnorm = c->qnorm.as<float>();
  qv->qsc = c->qsc.as<float>();
  qv->n = n;
  return HIVF_OK;
}

// set_mode: the caller needs the plans only as sets (the batched search):
// k_coarse_select then re-ranks only the centroids its bound cannot place
static hivf_status run_assign(hivf_index* ix, const QueryView& qv, uint32_t nprobe, double* d_dists,
                              bool set_mode = false) {
  hivf_ctx* c = ix->ctx;
  const IndexView v = ix->view();
  CK(c->dist32.ensure((size_t)qv.n * ix->K * 4));
  CK(c->plans.ensure((size_t)qv.n * nprobe * 4));
  CK(c->flags_c.ensure((size_t)qv.n * 4));
  if (nprobe > kNprobeMax) {
    // plans longer than the candidate buffers: exact distance to every
    // centroid + a stable per-query radix sort (assign.cu, k_coarse_all)
    size_t need = 0;
    CK(launch_coarse_all(v, qv, nprobe, nullptr, nullptr, nullptr, &need, c->stream));
    CK(c->coarse_all.ensure(need));
    need = c->coarse_all.bytes;
    CK(launch_coarse_all(v, qv, nprobe, c->plans.as<uint32_t>(), d_dists, c->coarse_all.p, &need, c->stream));
    CK(cudaMemsetAsync(c->flags_c.p, 0, (size_t)qv.n * 4, c->stream));
    c->stats.kernels_launched += 4;
    c->last_coarse_bits = 0;
    return HIVF_OK;
  }
  // tensor-core pass from 2^26 multiply-adds (C3 B=256 66 -> 22 us, neutral
  // at C2); below that the FFMA tile GEMM's single launch is faster (C1: 64
  // queries x 256 centroids x 128 dims)
  const bool coarse_tc = ix->centh && (c->opt_coarse_tc == 2 ||
                                       (c->opt_coarse_tc == 1 && (uint64_t)qv.n * ix->K * ix->dpad >= (1ull << 26)));
  const uint32_t splits = coarse_tc ? 1u : coarse_dist_splits(v, qv.n);
  float* part = nullptr;
  if (splits > 1) {
    CK(c->coarse_part.ensure((size_t)splits * qv.n * ix->K * 4));
    part = c->coarse_part.as<float>();
  }
  CoarseBound bd = coarse_bound_ffma(ix->dim);
  if (coarse_tc) {
    // tensor-core pass: the batch's fp16 query copy, then one kind::f16 GEMM
    CK(c->qh16.ensure(coarse_tc_bytes(qv.n, ix->dpad)));
    launch_pack_coarse_tc(qv.qs, qv.n, ix->dpad, qv.qsc, 0.f, c->qh16.as<uint8_t>(), c->stream);
    CKL();
    launch_coarse_dist_tc(v, qv, ix->centh, ix->csc, c->qh16.as<uint8_t>(), c->dist32.as<float>(), c->stream);
    bd = coarse_bound_h16(ix->dim, ix->cmax);
    c->last_coarse_bits = 16;
    c->stats.kernels_launched += 1;  // k_pack_cd
  } else {
    c->last_coarse_bits = 32;
    launch_coarse_dist(v, qv, c->dist32.as<float>(), c->stream, part);
  }
  CKL();
  launch_coarse_select(v, qv, c->dist32.as<float>(), nprobe, bd, c->plans.as<uint32_t>(), d_dists,
                       c->flags_c.as<int>(), c->stream, set_mode && c->opt_coarse_set);
  CKL();
  launch_coarse_fallback(v, qv, nprobe, c->plans.as<uint32_t>(), d_dists, c->flags_c.as<int>(), c->stream);
  CKL();
  c->stats.kernels_launched += 3;
  return HIVF_OK;
}

// Grouped scan over pairs (pair_query/pair_list already in c->pq / c->pl).
// kind_override: 0 -> the index's current scan kernel, else 1/2/3
// topk > 0 (a search for the k nearest): the tensor-core scan shares a per-query
// drop bound across items (scan_tc.cu); 0 (node-split items, seeded heaps) off.
// item_bounds: node-split path -- fixed per-item bounds already in c->qbound
// *slots_view: the view finalize / repair must read the candidate slots with
// (the CTA-pair scan reports two slots per segment, IndexView::seg_split).
static hivf_status run_scan(hivf_index* ix, const QueryView& qv, uint32_t n_pairs, bool timed,
                            int kind_override = 0, uint32_t topk = 0, bool item_bounds = false,
                            IndexView* slots_view = nullptr) {
  hivf_ctx* c = ix->ctx;
  const int kind = kind_override ? kind_override : ix->scan_kind();
  IndexView v = ix->view_kind(kind);
  // batch density estimate (host-side, no sync): pairs per list of the index
  float ppl = (float)n_pairs / (float)std::max<uint32_t>(1, ix->K);
  const bool tc = kind != 1;
  uint32_t group = tc ? scan_tc_qmax(v.dpf, kind == 2, ppl, c->tc) : (uint32_t)kQMax;
  if (group == kTcPairQ) {
    v.seg_split = 2;
    v.s_max = 2 * ix->s_max;
  }
  if (slots_view) *slots_view = v;
  const size_t nslots = (size_t)std::max<uint32_t>(n_pairs, 1) * v.s_max;
  CK(c->list_cnt.ensure(ix->K * 4ull));
  CK(c->list_poff.ensure(ix->K * 4ull));
  CK(c->list_cur.ensure(ix->K * 4ull));
  CK(c->list_ioff.ensure(ix->K * 4ull));
  CK(c->sorted_pairs.ensure((size_t)std::max<uint32_t>(n_pairs, 1) * 4));
  CK(c->items.ensure(nslots * sizeof(ScanItem)));
  CK(c->n_items.ensure(4));
  CK(c->work_ctr.ensure(4));
  CK(c->cand_d.ensure(nslots * kKP * 4));
  CK(c->cand_row.ensure(nslots * kKP * 4));
  CK(c->cand_thr.ensure(nslots * 4));
  CK(c->cand_n.ensure(nslots * 4));
  // slots of empty lists are never written by the scan; zero counts so the
  // finalize pass reads "no candidates" there
  CK(cudaMemsetAsync(c->cand_n.p, 0, nslots * 4, c->stream));
  WideStage ws;
  ws.group = group;
  c->last_group = group;
  c->last_filter_bits = (tc && v.vech) ? 16 : 32;
  if (tc_is_wide(group)) {
    // the restaged queries need (pairs + 7K) x D floats; when HBM is short
    // (index near the budget) the batch takes the narrow kernel instead
    if (c->qshift.ensure(ix->K * 4ull) != cudaSuccess ||
        c->qwide.ensure((size_t)wide_stage_rows(n_pairs, ix->K) * ix->dpad * 4) != cudaSuccess) {
      (void)cudaGetLastError();
      ppl = 0.f;
      group = scan_tc_qmax(v.dpf, kind == 2, ppl, c->tc);
      if (tc_is_wide(group)) return fail(HIVF_ENOMEM, "wide scan: query staging buffer");
      ws.group = group;
      c->last_group = group;
      v.seg_split = 1;  // narrow kernel: one slot per segment
      v.s_max = ix->s_max;
      if (slots_view) *slots_view = v;
    } else {
      ws.qshift = c->qshift.as<uint32_t>();
      ws.qstage = c->qwide.as<uint8_t>();
    }
  }
  launch_build_worklist(v, group, c->pq.as<uint32_t>(), c->pl.as<uint32_t>(), n_pairs, c->list_cnt.as<uint32_t>(),
                        c->list_poff.as<uint32_t>(), c->list_cur.as<uint32_t>(),
                        c->list_ioff.as<uint32_t>(), c->sorted_pairs.as<uint32_t>(),
                        c->items.as<ScanItem>(), c->n_items.as<uint32_t>(), c->work_ctr.as<uint32_t>(),
                        ws.qshift, c->stream);
  CKL();
  if (ws.qstage) {
    launch_stage_wide(v, qv, c->sorted_pairs.as<uint32_t>(), c->pq.as<uint32_t>(), c->pl.as<uint32_t>(),
                      c->list_poff.as<uint32_t>(), c->list_cnt.as<uint32_t>(), n_pairs, ws, c->stream);
    CKL();
  }
  const int ctas = c->opt_scan_ctas > 0 ? c->opt_scan_ctas : c->sm_count;
  if (tc && topk && !item_bounds) {  // shared drop bounds start at "none" (0x7f7f7f7f ~ 3.4e38)
    CK(c->qbound.ensure((size_t)qv.n * 4));
    CK(cudaMemsetAsync(c->qbound.p, 0x7f, (size_t)qv.n * 4, c->stream));
    // dense batches: seed them from exact distances of a few rows of each
    // query's nearest list (options "seed_rows", "seed_ppl")
    if (c->opt_seed_rows >= topk && ppl >= c->opt_seed_ppl && qv.n && n_pairs % qv.n == 0) {
      launch_seed_bounds(v, qv, c->plans.as<uint32_t>(), n_pairs / qv.n, topk, c->opt_seed_rows,
                         c->qbound.as<float>(), c->stream);
      CKL();
    }
  }
  if (timed) c->mark(1);
  if (tc)
    launch_scan_tc(v, qv, c->items.as<ScanItem>(), c->n_items.as<uint32_t>(), c->work_ctr.as<uint32_t>(),
                   c->sorted_pairs.as<uint32_t>(), c->pq.as<uint32_t>(), c->cand_d.as<float>(),
                   c->cand_row.as<uint32_t>(), c->cand_thr.as<float>(), c->cand_n.as<uint32_t>(), ctas,
                   kind == 2, topk ? c->qbound.as<float>() : nullptr, topk, item_bounds ? 0 : 1, ppl,
                   ws, c->tc, c->stream);
  else
    launch_scan(v, qv, c->items.as<ScanItem>(), c->n_items.as<uint32_t>(), c->work_ctr.as<uint32_t>(),
                c->sorted_pairs.as<uint32_t>(), c->pq.as<uint32_t>(), c->cand_d.as<float>(),
                c->cand_row.as<uint32_t>(), c->cand_thr.as<float>(), c->cand_n.as<uint32_t>(), ctas,
                c->stream);
  CKL();
  c->stats.kernels_launched += 5;
  return HIVF_OK;
}

static hivf_status check_search_args(hivf_index* ix, uint32_t n, uint32_t nprobe, uint32_t k) {
  if (!ix) return fail(HIVF_EINVAL, "index is NULL");
  if (!ix->finished) return fail(HIVF_EINVAL, "index not finished");
  if (k == 0) return fail(HIVF_EINVAL, "make_cursor: k must be >= 1");
  if (nprobe < 1 || nprobe > ix->K) return fail(HIVF_EINVAL, "select_clusters: nprobe out of range");
  if (k > kExactMaxK) return fail(HIVF_EUNSUPPORTED, "k > %u", kExactMaxK);
  (void)n;
  return HIVF_OK;
}

// Batched search; d_plans == nullptr runs the coarse assign, otherwise the
// caller's select_clusters plans are used (validated on device).
static hivf_status search_impl(hivf_index* ix, const float* d_queries, uint32_t n, uint32_t nprobe,
                               uint32_t k, const uint32_t* d_plans, uint64_t* d_ids_out,
                               double* d_dists_out, uint32_t* d_counts_out) {
  hivf_status st = check_search_args(ix, n, nprobe, k);
  if (st != HIVF_OK) return st;
  if (n == 0) return HIVF_OK;
  hivf_ctx* c = ix->ctx;
  CK(cudaSetDevice(c->device));
  if (ix->tiered) complete_swaps(ix);
  c->stats = hivf_stats{};
  c->last_nq = n;
  c->last_index = ix;
  c->last_K = ix->K;
  // plans longer than kNprobeMax (the fast path's per-query plan buffers) take
  // the exact path, which streams any number of plan positions
  const bool exact_only = c->opt_force_exact || k > (uint32_t)kKP || nprobe > kNprobeMax;
  c->last_kind = exact_only ? 0 : ix->scan_kind();
  c->stats_adapted = false;
  QueryView qv;
  c->mark(0);
  if ((st = prep_queries(ix, d_queries, n, true, &qv)) != HIVF_OK) return st;
  const uint32_t np = n * nprobe;
  if (!d_plans) {
    if ((st = run_assign(ix, qv, nprobe, nullptr, true)) != HIVF_OK) return st;
  } else {
    CK(c->plans.ensure((size_t)np * 4));
    CK(c->flags_c.ensure((size_t)n * 4));  // no coarse fallback in a planned search
    CK(cudaMemsetAsync(c->flags_c.p, 0, (size_t)n * 4, c->stream));
  }
  CK(c->pq.ensure((size_t)np * 4));
  CK(c->pl.ensure((size_t)np * 4));
  CK(c->flags_f.ensure((size_t)n * 4));
  const IndexView v = ix->view();
  {
    const size_t parts = (size_t)n * exact_search_parts(nprobe, k);
    CK(c->x_ids.ensure(parts * k * 8));
    CK(c->x_d.ensure(parts * k * 8));
    CK(c->x_cnt.ensure(parts * 4));
    CK(c->x_tot.ensure(parts * 8));
  }
  if (d_plans || !exact_only) {
    launch_plans_to_pairs(d_plans ? d_plans : c->plans.as<uint32_t>(), n, nprobe, ix->K, c->pq.as<uint32_t>(),
                          c->pl.as<uint32_t>(), d_plans ? c->plans.as<uint32_t>() : nullptr,
                          c->err.as<int>(), c->stream);
    CKL();
  }
  if (!exact_only) {
    IndexView vs = v;  // the candidate slots' view (two per segment after the CTA-pair scan)
    if ((st = run_scan(ix, qv, np, true, 0, c->opt_no_bound ? 0 : k, false, &vs)) != HIVF_OK) return st;
    c->mark(2);
    CK(c->tau.ensure((size_t)n * 4));
    // in-place repair of segments whose completeness proof failed
    // (finalize.cu: k_repair_segments + k_finalize_repair); queries it cannot
    // settle take the whole-query exact fallback below
    const uint32_t rep_cap = std::max<uint32_t>(1024, n * 4);
    const uint32_t per_q = 512;
    CK(c->rep_entries.ensure((size_t)rep_cap * 8));
    CK(c->rep_n.ensure(4));
    CK(c->rep_cnt.ensure((size_t)n * 4));
    CK(c->rep_d.ensure((size_t)n * per_q * 8));
    CK(c->rep_ids.ensure((size_t)n * per_q * 8));
    CK(cudaMemsetAsync(c->rep_n.p, 0, 4, c->stream));
    RepairState R{c->rep_entries.as<uint64_t>(), c->rep_n.as<uint32_t>(), rep_cap, c->rep_cnt.as<uint32_t>(),
                  c->rep_d.as<double>(), c->rep_ids.as<uint64_t>(), per_q};
    launch_finalize_search(vs, qv, c->plans.as<uint32_t>(), nprobe, k, c->cand_d.as<float>(),
                           c->cand_row.as<uint32_t>(), c->cand_thr.as<float>(), c->cand_n.as<uint32_t>(),
                           d_ids_out, d_dists_out, d_counts_out, c->flags_f.as<int>(), c->tau.as<float>(),
                           &R, c->stream);
    CKL();
    // pass-1 flags survive for the auto policy (flags2 carries the repair outcome)
    CK(c->flags2.ensure((size_t)n * 4));
    CK(cudaMemcpyAsync(c->flags2.p, c->flags_f.p, (size_t)n * 4, cudaMemcpyDeviceToDevice, c->stream));
    launch_repair(vs, qv, c->plans.as<uint32_t>(), nprobe, k, c->cand_d.as<float>(), c->cand_row.as<uint32_t>(),
                  c->cand_thr.as<float>(), c->cand_n.as<uint32_t>(), c->tau.as<float>(), R, c->sm_count * 4,
                  d_ids_out, d_dists_out, d_counts_out, c->flags2.as<int>(), c->stream);
    CKL();
    launch_exact_search(vs, qv, c->plans.as<uint32_t>(), nprobe, k, c->flags2.as<int>(), d_ids_out,
                        d_dists_out, d_counts_out, c->x_ids.as<uint64_t>(), c->x_d.as<double>(),
                        c->x_cnt.as<uint32_t>(), c->x_tot.as<uint64_t>(), c->tau.as<float>(), c->stream);
    CKL();
    c->stats.kernels_launched += 5;
    c->mark(3);
  } else {
    CK(cudaMemsetAsync(c->flags_f.p, 0, (size_t)n * 4, c->stream));
    c->mark(1);
    c->mark(2);
    launch_exact_search(v, qv, c->plans.as<uint32_t>(), nprobe, k, nullptr, d_ids_out, d_dists_out,
                        d_counts_out, c->x_ids.as<uint64_t>(), c->x_d.as<double>(),
                        c->x_cnt.as<uint32_t>(), c->x_tot.as<uint64_t>(), nullptr, c->stream);
    CKL();
    c->stats.kernels_launched += 1;
    c->mark(3);
  }
  return HIVF_OK;
}

hivf_status hivf_search_device(hivf_index* ix, const float* d_queries, uint32_t n,
                               uint32_t nprobe, uint32_t k, uint64_t* d_ids_out,
                               double* d_dists_out, uint32_t* d_counts_out) {
  return search_impl(ix, d_queries, n, nprobe, k, nullptr, d_ids_out, d_dists_out, d_counts_out);
}

hivf_status hivf_search_planned_device(hivf_index* ix, const float* d_queries, uint32_t n,
                                       uint32_t nprobe, uint32_t k, const uint32_t* d_plans,
                                       uint64_t* d_ids_out, double* d_dists_out,
                                       uint32_t* d_counts_out) {
  if (!d_plans) return fail(HIVF_EINVAL, "hivf_search_planned_device: plans NULL");
  return search_impl(ix, d_queries, n, nprobe, k, d_plans, d_ids_out, d_dists_out, d_counts_out);
}

hivf_status hivf_assign_device(hivf_index* ix, const float* d_queries, uint32_t n, uint32_t nprobe,
                               uint32_t* d_plans_out, double* d_dists_out) {
  hivf_status st = check_search_args(ix, n, nprobe, 1);
  if (st != HIVF_OK) return st;
  if (n == 0) return HIVF_OK;
  if (!d_queries || !d_plans_out) return fail(HIVF_EINVAL, "hivf_assign_device: NULL buffer");
  hivf_ctx* c = ix->ctx;
  CK(cudaSetDevice(c->device));
  c->stats = hivf_stats{};
  c->last_nq = 0;
  QueryView qv;
  if ((st = prep_queries(ix, d_queries, n, true, &qv)) != HIVF_OK) return st;
  if ((st = run_assign(ix, qv, nprobe, d_dists_out)) != HIVF_OK) return st;
  CK(cudaMemcpyAsync(d_plans_out, c->plans.p, (size_t)n * nprobe * 4, cudaMemcpyDeviceToDevice, c->stream));
  return HIVF_OK;
}

// hivf_search's device part through a cached CUDA graph: a batch shape seen
// twice in a row (same index, n, nprobe, k, scan kind, buffers, options) is
// captured on its second call and replayed from then on, so the ~15
// dependent launches of a search cost one graph launch (the host-buffer API
// is launch-latency bound on small batches).  The search itself has no host
// decisions that depend on device data (repair / exact fallbacks are
// device-side), so the replay does exactly what the captured call did; the
// host-side bookkeeping it left (stats, last-call fields) is restored.  Any
// reallocation, option change or index upload/destroy bumps g_state_gen and
// invalidates the graph; tiered indexes, kernel timing and profiling bypass it.
static hivf_status search_device_cached(hivf_index* ix, const float* dq, uint32_t n, uint32_t nprobe,
                                        uint32_t k, uint64_t* ids, double* dists, uint32_t* counts) {
  hivf_ctx* c = ix->ctx;
  if (!c->opt_search_graph || ix->tiered || c->opt_time)
    return hivf_search_device(ix, dq, n, nprobe, k, ids, dists, counts);
  const int kind = (c->opt_force_exact || k > (uint32_t)kKP || nprobe > kNprobeMax) ? 0 : ix->scan_kind();
  auto& g = c->sgraph;
  const bool same = g.ix == ix && g.q == dq && g.out == ids && g.n == n && g.nprobe == nprobe && g.k == k &&
                    g.kind == kind && g.gen == g_state_gen.load();
  if (same && g.exec) {
    c->stats = g.stats;
    c->last_nq = n;
    c->last_index = ix;
    c->last_K = ix->K;
    c->last_kind = g.last_kind;
    c->stats_adapted = false;
    CK(cudaGraphLaunch(g.exec, c->stream));
    return HIVF_OK;
  }
  // legacy / per-thread default streams cannot be captured, and a blocking
  // stream's capture fails while other threads use the legacy stream: replay
  // only on non-blocking streams, and never retry a stream whose capture failed
  unsigned int sflags = 0;
  const bool capturable = c->stream && c->stream != cudaStreamLegacy && c->stream != cudaStreamPerThread &&
                          cudaStreamGetFlags(c->stream, &sflags) == cudaSuccess &&
                          (sflags & cudaStreamNonBlocking) && g.failed_stream != c->stream;
  (void)cudaGetLastError();
  if (!capturable) return hivf_search_device(ix, dq, n, nprobe, k, ids, dists, counts);
  if (same && g.seen) {  // second call with this shape: capture it
    const uint64_t gen0 = g_state_gen.load();
    cudaGraph_t graph = nullptr;
    bool ok = cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    hivf_status st = ok ? hivf_search_device(ix, dq, n, nprobe, k, ids, dists, counts) : HIVF_ECUDA;
    if (ok) ok = cudaStreamEndCapture(c->stream, &graph) == cudaSuccess && st == HIVF_OK &&
                 g_state_gen.load() == gen0;
    cudaGraphExec_t ex = nullptr;
    if (ok) ok = cudaGraphInstantiate(&ex, graph, 0) == cudaSuccess;
    if (graph) cudaGraphDestroy(graph);
    (void)cudaGetLastError();
    if (ok) {
      if (g.exec) cudaGraphExecDestroy(g.exec);
      g.exec = ex;
      g.gen = gen0;
      g.stats = c->stats;
      g.last_kind = c->last_kind;
      CK(cudaGraphLaunch(g.exec, c->stream));
      return HIVF_OK;
    }
    g.seen = false;  // not capturable: plain launches from now on for this stream
    g.failed_stream = c->stream;
    return hivf_search_device(ix, dq, n, nprobe, k, ids, dists, counts);
  }
  if (g.exec) cudaGraphExecDestroy(g.exec);
  const cudaStream_t failed = g.failed_stream;
  g = {};
  g.failed_stream = failed;
  hivf_status st = hivf_search_device(ix, dq, n, nprobe, k, ids, dists, counts);
  if (st == HIVF_OK) {
    g.ix = ix;
    g.q = dq;
    g.out = ids;
    g.n = n;
    g.nprobe = nprobe;
    g.k = k;
    g.kind = kind;
    g.gen = g_state_gen.load();
    g.seen = true;
  }
  return st;
}

hivf_status hivf_search(hivf_index* ix, const float* queries, uint32_t n, uint32_t nprobe,
                        uint32_t k, uint64_t* ids_out, double* dists_out, uint32_t* counts_out) {
  hivf_status st = check_search_args(ix, n, nprobe, k);
  if (st != HIVF_OK) return st;
  if (n == 0) return HIVF_OK;
  if (!queries || !ids_out || !dists_out || !counts_out) return fail(HIVF_EINVAL, "hivf_search: NULL buffer");
  hivf_ctx* c = ix->ctx;
  CK(cudaSetDevice(c->device));
  const size_t qb = (size_t)n * ix->dim * 4, ob = (size_t)n * k;
  // results, error flag and fallback flags come back in ONE D2H copy:
  //   ids | dists | counts | err | flags
  const size_t o_d = ob * 8, o_c = 2 * ob * 8, o_e = o_c + (size_t)n * 4, o_f = o_e + 4,
               total = o_f + (size_t)n * 4;
  const bool want_fb = c->opt_scan_kernel == 0 && !ix->auto_split;
  CK(c->qin.ensure(qb));
  CK(c->out_ids.ensure(total));
  CK(c->hstage.ensure(total));
  CK(c->err.ensure(4));
  CK(cudaMemsetAsync(c->err.p, 0, 4, c->stream));
  CK(cudaMemcpyAsync(c->qin.p, queries, qb, cudaMemcpyHostToDevice, c->stream));
  uint8_t* dpk = c->out_ids.as<uint8_t>();
  if ((st = search_device_cached(ix, c->qin.as<float>(), n, nprobe, k, reinterpret_cast<uint64_t*>(dpk),
                                 reinterpret_cast<double*>(dpk + o_d), reinterpret_cast<uint32_t*>(dpk + o_c))) !=
      HIVF_OK)
    return st;
  CK(cudaMemcpyAsync(dpk + o_e, c->err.p, 4, cudaMemcpyDeviceToDevice, c->stream));
  if (want_fb) CK(cudaMemcpyAsync(dpk + o_f, c->flags_f.p, 4ull * n, cudaMemcpyDeviceToDevice, c->stream));
  uint8_t* hpk = c->hstage.as<uint8_t>();
  CK(cudaMemcpyAsync(hpk, dpk, want_fb ? total : o_f, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  int err = 0;
  std::memcpy(&err, hpk + o_e, 4);
  std::memcpy(ids_out, hpk, ob * 8);
  std::memcpy(dists_out, hpk + o_d, ob * 8);
  std::memcpy(counts_out, hpk + o_c, (size_t)n * 4);
  std::vector<int> fb(want_fb ? n : 0);
  if (want_fb) std::memcpy(fb.data(), hpk + o_f, 4ull * n);
  if (err) return fail(HIVF_EINVAL, "hivf_search: non-finite query value");
  if (!fb.empty()) {
    uint32_t nf = 0;
    for (int v : fb) nf += v != 0;
    adapt_scan(ix, n, nf);
    c->stats_adapted = true;
  }
  return HIVF_OK;
}

hivf_status hivf_assign(hivf_index* ix, const float* queries, uint32_t n, uint32_t nprobe,
                        uint32_t* plans_out, double* dists_out) {
  hivf_status st = check_search_args(ix, n, nprobe, 1);
  if (st != HIVF_OK) return st;
  if (n == 0) return HIVF_OK;
  if (!queries || !plans_out) return fail(HIVF_EINVAL, "hivf_assign: NULL buffer");
  hivf_ctx* c = ix->ctx;
  CK(cudaSetDevice(c->device));
  c->stats = hivf_stats{};
  c->last_nq = 0;
  const size_t qb = (size_t)n * ix->dim * 4;
  CK(c->qin.ensure(qb));
  CK(c->pdists.ensure((size_t)n * nprobe * 8));
  CK(c->err.ensure(4));
  CK(cudaMemsetAsync(c->err.p, 0, 4, c->stream));
  CK(cudaMemcpyAsync(c->qin.p, queries, qb, cudaMemcpyHostToDevice, c->stream));
  QueryView qv;
  if ((st = prep_queries(ix, c->qin.as<float>(), n, true, &qv)) != HIVF_OK) return st;
  if ((st = run_assign(ix, qv, nprobe, c->pdists.as<double>())) != HIVF_OK) return st;
  CK(cudaMemcpyAsync(plans_out, c->plans.p, (size_t)n * nprobe * 4, cudaMemcpyDeviceToHost, c->stream));
  if (dists_out)
    CK(cudaMemcpyAsync(dists_out, c->pdists.p, (size_t)n * nprobe * 8, cudaMemcpyDeviceToHost, c->stream));
  int err = 0;
  CK(cudaMemcpyAsync(&err, c->err.p, 4, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (err) return fail(HIVF_EINVAL, "select_clusters: non-finite query value");
  return HIVF_OK;
}

// ---------------------------------------------------------------------------
// index build: compute_assignments / train_kmeans (vector_index.cpp:99-208)
// ---------------------------------------------------------------------------

// nearest_centroid for every row (ties -> lowest id): the exact coarse assign
// with nprobe = 1 against a centroid-only L2 index (rows already in search
// space, so no query normalization).
static hivf_status assign_rows(hivf_ctx* c, const float* X, uint64_t n, uint32_t dim, const float* dcent,
                               uint32_t K, uint32_t* out) {
  std::vector<uint64_t> offs(K + 1, 0);
  hivf_index* ix = nullptr;
  hivf_status st = hivf_index_begin(c, dim, HIVF_METRIC_L2, K, dcent, 1, offs.data(), &ix);
  if (st != HIVF_OK) return st;
  if ((st = hivf_index_finish(ix)) != HIVF_OK) {
    hivf_index_destroy(ix);
    return st;
  }
  const uint64_t chunk = std::max<uint64_t>(1, std::min<uint64_t>(65536, (256ull << 20) / (4ull * K)));
  for (uint64_t b = 0; b < n && st == HIVF_OK; b += chunk) {
    const uint32_t m = (uint32_t)std::min(chunk, n - b);
    QueryView qv;
    if ((st = prep_queries(ix, X + b * dim, m, false, &qv)) != HIVF_OK) break;
    if ((st = run_assign(ix, qv, 1, nullptr)) != HIVF_OK) break;
    if (cudaMemcpyAsync(out + b, c->plans.p, m * 4ull, cudaMemcpyDeviceToDevice, c->stream) != cudaSuccess)
      st = fail(HIVF_ECUDA, "assign copy");
  }
  std::string keep = g_err;
  hivf_index_destroy(ix);
  g_err = keep;
  return st;
}

hivf_status hivf_compute_assignments(hivf_ctx* ctx, const float* d_corpus, uint64_t n, uint32_t dim,
                                     const float* d_centroids, uint32_t K, uint32_t* d_assign_out) {
  if (!ctx || (!d_corpus && n) || !d_centroids || (!d_assign_out && n))
    return fail(HIVF_EINVAL, "compute_assignments: NULL argument");
  if (dim == 0 || K == 0) return fail(HIVF_EINVAL, "compute_assignments: dim and K must be >= 1");
  if (n == 0) return HIVF_OK;
  CK(cudaSetDevice(ctx->device));
  CK(ctx->err.ensure(4));
  CK(cudaMemsetAsync(ctx->err.p, 0, 4, ctx->stream));
  hivf_status st = assign_rows(ctx, d_corpus, n, dim, d_centroids, K, d_assign_out);
  if (st != HIVF_OK) return st;
  int err = 0;
  CK(cudaMemcpyAsync(&err, ctx->err.p, 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  if (err) return fail(HIVF_EINVAL, "compute_assignments: non-finite corpus value");
  return HIVF_OK;
}

namespace {
struct DevScratch {  // RAII cudaMalloc set for the k-means run
  std::vector<void*> p;
  cudaError_t alloc(void** out, size_t bytes) {
    cudaError_t e = cudaMalloc(out, std::max<size_t>(bytes, 16));
    if (e == cudaSuccess) p.push_back(*out);
    return e;
  }
  ~DevScratch() {
    for (void* q : p) cudaFree(q);
  }
};
}  // namespace

// seeding 0: the reference's k-means++ (sequential running sums, one serial
// chain per seed); 1: K distinct corpus rows drawn with the reference's Rng
// (uniform_index, duplicates re-drawn) -- no serial chain, for large K x n.
static hivf_status train_kmeans_impl(hivf_ctx* ctx, const float* d_corpus, uint64_t n, uint32_t dim, uint32_t K,
                                     uint32_t max_iters, uint64_t seed, int seeding, float* d_centroids_out) {
  if (!ctx || !d_corpus || !d_centroids_out) return fail(HIVF_EINVAL, "train_kmeans: NULL argument");
  if (n < K) return fail(HIVF_EINVAL, "train_kmeans: corpus smaller than k_clusters");
  if (K == 0) return fail(HIVF_EINVAL, "train_kmeans: k_clusters must be >= 1");
  if (max_iters == 0) return fail(HIVF_EINVAL, "train_kmeans: max_iters must be >= 1");
  if (dim == 0) return fail(HIVF_EINVAL, "train_kmeans: dim must be >= 1");
  if (n >= 0xffffffffull) return fail(HIVF_EUNSUPPORTED, "train_kmeans: n >= 2^32");
  CK(cudaSetDevice(ctx->device));
  cudaStream_t s = ctx->stream;
  // the reference's Rng (common.hpp:18-76): mt19937_64, uniform_index by
  // rejection, uniform = (x >> 11) * 2^-53; the k-means++ draws are taken in
  // stream order (one per seed whose total > 0, consumed on the device)
  std::mt19937_64 gen(seed);
  const uint64_t limit = UINT64_MAX - UINT64_MAX % n;
  uint64_t x;
  do {
    x = gen();
  } while (x >= limit);
  const uint64_t first = x % n;
  std::vector<double> us(std::max<uint32_t>(1, K));
  for (uint32_t i = 0; i + 1 < K; ++i) us[i] = static_cast<double>(gen() >> 11) * 0x1.0p-53;
  DevScratch S;
  double *dist2, *prefix, *total, *d_us, *dd;
  int *draw, *zero, *differs;
  uint64_t *pick, *off;
  uint32_t *assign, *prev, *idx, *idx_s, *keys_s;
  uint8_t* used;
  float* new_c;
  unsigned long long* sc2;
  cudaError_t e = cudaSuccess;
  for (auto [ptr, bytes] : std::initializer_list<std::pair<void**, size_t>>{
           {(void**)&dist2, n * 8}, {(void**)&prefix, n * 8}, {(void**)&total, 8},
           {(void**)&d_us, us.size() * 8}, {(void**)&dd, n * 8}, {(void**)&draw, 4}, {(void**)&zero, 4},
           {(void**)&differs, 4}, {(void**)&pick, 8}, {(void**)&off, (K + 1) * 8ull},
           {(void**)&assign, n * 4}, {(void**)&prev, n * 4}, {(void**)&idx, n * 4},
           {(void**)&idx_s, n * 4}, {(void**)&keys_s, n * 4}, {(void**)&used, n},
           {(void**)&new_c, (size_t)K * dim * 4}, {(void**)&sc2, 16}})
    if ((e = S.alloc(ptr, bytes)) != cudaSuccess)
      return fail(e == cudaErrorMemoryAllocation ? HIVF_ENOMEM : HIVF_ECUDA, "train_kmeans alloc: %s",
                  cudaGetErrorString(e));
  float* cents = d_centroids_out;
  if (seeding == 0) {
    CK(cudaMemcpyAsync(d_us, us.data(), us.size() * 8, cudaMemcpyHostToDevice, s));
    CK(cudaMemsetAsync(draw, 0, 4, s));
    // k-means++ seeding (vector_index.cpp:114-154)
    CK(cudaMemcpyAsync(cents, d_corpus + first * dim, dim * 4ull, cudaMemcpyDeviceToDevice, s));
    launch_kmeans_dist2(d_corpus, n, dim, cents, dist2, 0, s);
    CKL();
    for (uint32_t m = 1; m < K; ++m) {
      launch_kmeans_prefix(dist2, n, prefix, total, s);
      launch_kmeans_pick(prefix, n, total, d_us, draw, pick, zero, d_corpus, dim, cents, m, s);
      launch_kmeans_dist2(d_corpus, n, dim, cents + (uint64_t)m * dim, dist2, 1, s);
      CKL();
    }
  } else {
    // K distinct rows: the first draw as above, then uniform_index draws from
    // the same stream, a row already taken is drawn again
    std::vector<uint8_t> taken(n, 0);
    std::vector<uint64_t> rows{first};
    taken[first] = 1;
    std::mt19937_64 g2(seed ^ 0x9e3779b97f4a7c15ull);
    while (rows.size() < K) {
      uint64_t y;
      do {
        y = g2();
      } while (y >= limit);
      if (!taken[y % n]) {
        taken[y % n] = 1;
        rows.push_back(y % n);
      }
    }
    for (uint32_t m = 0; m < K; ++m)
      CK(cudaMemcpyAsync(cents + (uint64_t)m * dim, d_corpus + rows[m] * dim, dim * 4ull,
                         cudaMemcpyDeviceToDevice, s));
  }
  // Lloyd iterations (vector_index.cpp:156-197)
  CK(cudaMemsetAsync(prev, 0xff, n * 4, s));
  size_t sort_bytes = 0;
  CK(cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, assign, keys_s, idx, idx_s, (int64_t)n, 0, 32, s));
  void* sort_tmp = nullptr;
  if ((e = S.alloc(&sort_tmp, sort_bytes)) != cudaSuccess) return fail(HIVF_ENOMEM, "train_kmeans sort scratch");
  std::vector<uint64_t> hoff(K + 1);
  for (uint32_t it = 0; it < max_iters; ++it) {
    hivf_status st = assign_rows(ctx, d_corpus, n, dim, cents, K, assign);
    if (st != HIVF_OK) return st;
    int h_diff = 0;
    CK(cudaMemsetAsync(differs, 0, 4, s));
    launch_same_assign(assign, prev, n, differs, s);
    CKL();
    CK(cudaMemcpyAsync(&h_diff, differs, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (!h_diff) break;
    launch_iota(idx, n, s);
    CK(cub::DeviceRadixSort::SortPairs(sort_tmp, sort_bytes, assign, keys_s, idx, idx_s, (int64_t)n, 0, 32, s));
    CK(cudaMemcpyAsync(new_c, cents, (size_t)K * dim * 4, cudaMemcpyDeviceToDevice, s));
    launch_cluster_means(d_corpus, dim, K, keys_s, idx_s, n, off, new_c, s);
    CKL();
    CK(cudaMemcpyAsync(hoff.data(), off, (K + 1) * 8ull, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    bool any_empty = false;
    for (uint32_t c = 0; c < K; ++c) {
      if (hoff[c + 1] != hoff[c]) continue;
      if (!any_empty) CK(cudaMemsetAsync(used, 0, n, s));
      any_empty = true;
      launch_far_point(d_corpus, n, dim, assign, new_c, cents, c, used, dd, sc2, s);
      CKL();
    }
    CK(cudaMemcpyAsync(cents, new_c, (size_t)K * dim * 4, cudaMemcpyDeviceToDevice, s));
  }
  CK(cudaStreamSynchronize(s));
  return HIVF_OK;
}

hivf_status hivf_train_kmeans(hivf_ctx* ctx, const float* d_corpus, uint64_t n, uint32_t dim, uint32_t K,
                              uint32_t max_iters, uint64_t seed, float* d_centroids_out) {
  return train_kmeans_impl(ctx, d_corpus, n, dim, K, max_iters, seed, 0, d_centroids_out);
}

hivf_status hivf_train_kmeans_sampled_seeds(hivf_ctx* ctx, const float* d_corpus, uint64_t n, uint32_t dim,
                                            uint32_t K, uint32_t max_iters, uint64_t seed, float* d_centroids_out) {
  return train_kmeans_impl(ctx, d_corpus, n, dim, K, max_iters, seed, 1, d_centroids_out);
}

// host-buffer forms (the C++ adapter's ivf::train_kmeans / compute_assignments)
hivf_status hivf_train_kmeans_host(hivf_ctx* ctx, const float* corpus, uint64_t n, uint32_t dim, uint32_t K,
                                   uint32_t max_iters, uint64_t seed, float* centroids_out) {
  if (!ctx || !corpus || !centroids_out) return fail(HIVF_EINVAL, "train_kmeans: NULL argument");
  if (n < K) return fail(HIVF_EINVAL, "train_kmeans: corpus smaller than k_clusters");
  CK(cudaSetDevice(ctx->device));
  DevScratch S;
  float *dx = nullptr, *dc = nullptr;
  cudaError_t e;
  if ((e = S.alloc((void**)&dx, n * dim * 4ull)) != cudaSuccess || (e = S.alloc((void**)&dc, (uint64_t)K * dim * 4)) != cudaSuccess)
    return fail(HIVF_ENOMEM, "train_kmeans staging: %s", cudaGetErrorString(e));
  CK(cudaMemcpyAsync(dx, corpus, n * dim * 4ull, cudaMemcpyHostToDevice, ctx->stream));
  hivf_status st = hivf_train_kmeans(ctx, dx, n, dim, K, max_iters, seed, dc);
  if (st != HIVF_OK) return st;
  CK(cudaMemcpyAsync(centroids_out, dc, (uint64_t)K * dim * 4, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return HIVF_OK;
}

hivf_status hivf_compute_assignments_host(hivf_ctx* ctx, const float* corpus, uint64_t n, uint32_t dim,
                                          const float* centroids, uint32_t K, uint32_t* assign_out) {
  if (!ctx || (!corpus && n) || !centroids || (!assign_out && n))
    return fail(HIVF_EINVAL, "compute_assignments: NULL argument");
  if (n == 0) return HIVF_OK;
  CK(cudaSetDevice(ctx->device));
  DevScratch S;
  float *dx = nullptr, *dc = nullptr;
  uint32_t* da = nullptr;
  cudaError_t e;
  if ((e = S.alloc((void**)&dx, n * dim * 4ull)) != cudaSuccess ||
      (e = S.alloc((void**)&dc, (uint64_t)K * dim * 4)) != cudaSuccess || (e = S.alloc((void**)&da, n * 4ull)) != cudaSuccess)
    return fail(HIVF_ENOMEM, "compute_assignments staging: %s", cudaGetErrorString(e));
  CK(cudaMemcpyAsync(dx, corpus, n * dim * 4ull, cudaMemcpyHostToDevice, ctx->stream));
  CK(cudaMemcpyAsync(dc, centroids, (uint64_t)K * dim * 4, cudaMemcpyHostToDevice, ctx->stream));
  hivf_status st = hivf_compute_assignments(ctx, dx, n, dim, dc, K, da);
  if (st != HIVF_OK) return st;
  CK(cudaMemcpyAsync(assign_out, da, n * 4ull, cudaMemcpyDeviceToHost, ctx->stream));
  CK(cudaStreamSynchronize(ctx->stream));
  return HIVF_OK;
}

// ---------------------------------------------------------------------------
// node-split sub-search
// ---------------------------------------------------------------------------

hivf_status hivf_scan_items(hivf_index* ix, const float* queries, uint32_t n_items,
                            const uint32_t* cluster_off, const uint32_t* clusters,
                            const uint32_t* kv, uint64_t* heap_ids, double* heap_dists,
                            uint32_t* heap_counts, uint32_t heap_stride, uint8_t* changed_out) {
  if (!ix) return fail(HIVF_EINVAL, "index is NULL");
  if (!ix->finished) return fail(HIVF_EINVAL, "index not finished");
  if (n_items == 0) return HIVF_OK;
  if (!queries || !cluster_off || !kv || !heap_ids || !heap_dists || !heap_counts)
    return fail(HIVF_EINVAL, "hivf_scan_items: NULL buffer");
  uint32_t kmax = 0;
  for (uint32_t i = 0; i < n_items; ++i) {
    if (kv[i] == 0) return fail(HIVF_EINVAL, "make_cursor: k must be >= 1");
    if (kv[i] > kExactMaxK) return fail(HIVF_EUNSUPPORTED, "k > %u", kExactMaxK);
    if (kv[i] > heap_stride) return fail(HIVF_EINVAL, "heap_stride < k");
    if (heap_counts[i] > kv[i]) return fail(HIVF_EINVAL, "heap larger than k");
    if (cluster_off[i + 1] < cluster_off[i]) return fail(HIVF_EINVAL, "cluster_off not monotone");
    kmax = std::max(kmax, kv[i]);
  }
  const uint32_t n_pairs = cluster_off[n_items] - cluster_off[0];
  if (cluster_off[0] != 0) return fail(HIVF_EINVAL, "cluster_off[0] must be 0");
  if (n_pairs && (!clusters || !changed_out)) return fail(HIVF_EINVAL, "hivf_scan_items: NULL clusters");
  for (uint32_t p = 0; p < n_pairs; ++p)
    if (clusters[p] >= ix->K) return fail(HIVF_EINVAL, "cluster id %u out of range", clusters[p]);
  hivf_ctx* c = ix->ctx;
  CK(cudaSetDevice(c->device));
  if (ix->tiered) complete_swaps(ix);
  c->stats = hivf_stats{};
  c->last_nq = 0;
  c->last_index = ix;
  c->last_K = ix->K;
  cudaStream_t s = c->stream;
  // All inputs go down in ONE pinned H2D copy and all outputs come back in ONE
  // D2H copy (latency of a sub-stage, config 5): staging layout
  //   in : queries | pair->item | clusters | cluster_off | k | heap ids | heap d | heap n
  //   out: heap ids | heap d | heap n | changed | err | fallback flags
  // (the heap segments are shared: updated in place on the device).
  auto al = [](size_t x) { return (x + 15) & ~size_t(15); };
  const size_t qb = (size_t)n_items * ix->dim * 4, pb = (size_t)std::max<uint32_t>(n_pairs, 1) * 4;
  const size_t hb = (size_t)n_items * heap_stride * 8;
  const size_t o_q = 0, o_pq = al(o_q + qb), o_cl = al(o_pq + pb), o_off = al(o_cl + pb),
               o_k = al(o_off + (n_items + 1) * 4ull), o_hi = al(o_k + n_items * 4ull), o_hd = al(o_hi + hb),
               o_hn = al(o_hd + hb), o_ch = al(o_hn + n_items * 4ull), o_err = al(o_ch + std::max<uint32_t>(n_pairs, 1)),
               o_fb = al(o_err + 4), total = al(o_fb + n_items * 4ull);
  CK(c->hstage.ensure(total));
  CK(c->qin.ensure(total));
  uint8_t* h = c->hstage.as<uint8_t>();
  uint8_t* d = c->qin.as<uint8_t>();
  std::memcpy(h + o_q, queries, qb);
  uint32_t* hpq = reinterpret_cast<uint32_t*>(h + o_pq);
  for (uint32_t i = 0; i < n_items; ++i)
    for (uint32_t p = cluster_off[i]; p < cluster_off[i + 1]; ++p) hpq[p] = i;
  if (n_pairs) std::memcpy(h + o_cl, clusters, n_pairs * 4ull);
  std::memcpy(h + o_off, cluster_off, (n_items + 1) * 4ull);
  std::memcpy(h + o_k, kv, n_items * 4ull);
  std::memcpy(h + o_hi, heap_ids, hb);
  std::memcpy(h + o_hd, heap_dists, hb);
  std::memcpy(h + o_hn, heap_counts, n_items * 4ull);
  std::memset(h + o_err, 0, 4);
  CK(cudaMemcpyAsync(d, h, o_ch, cudaMemcpyHostToDevice, s));
  CK(cudaMemsetAsync(d + o_err, 0, 4, s));
  const uint32_t* d_pq = reinterpret_cast<const uint32_t*>(d + o_pq);
  const uint32_t* d_cl = reinterpret_cast<const uint32_t*>(d + o_cl);
  const uint32_t* d_off = reinterpret_cast<const uint32_t*>(d + o_off);
  const uint32_t* d_k = reinterpret_cast<const uint32_t*>(d + o_k);
  uint64_t* d_hi = reinterpret_cast<uint64_t*>(d + o_hi);
  double* d_hd = reinterpret_cast<double*>(d + o_hd);
  uint32_t* d_hn = reinterpret_cast<uint32_t*>(d + o_hn);
  uint8_t* d_ch = d + o_ch;
  int* d_fb = reinterpret_cast<int*>(d + o_fb);
  // the scan's pair arrays (run_scan reads c->pq / c->pl)
  CK(c->pq.ensure(pb));
  CK(c->pl.ensure(pb));
  if (n_pairs) {
    CK(cudaMemcpyAsync(c->pq.p, d_pq, n_pairs * 4ull, cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(c->pl.p, d_cl, n_pairs * 4ull, cudaMemcpyDeviceToDevice, s));
  }
  hivf_status st;
  QueryView qv;
  // cursor queries are already in search space: no re-normalization
  CK(c->err.ensure(4));
  CK(cudaMemsetAsync(c->err.p, 0, 4, s));
  if ((st = prep_queries(ix, reinterpret_cast<const float*>(d + o_q), n_items, false, &qv)) != HIVF_OK) return st;
  CK(cudaMemcpyAsync(d + o_err, c->err.p, 4, cudaMemcpyDeviceToDevice, s));
  const IndexView v = ix->view();
  const bool exact_only = c->opt_force_exact || kmax > (uint32_t)kKP;
  CK(cudaMemsetAsync(d_fb, 0, n_items * 4ull, s));
  if (!exact_only && n_pairs) {
    // drop bound per item: its heap's worst before the sub-stage (fixed)
    const bool use_bounds = !c->opt_no_bound;
    if (use_bounds) {
      CK(c->qbound.ensure((size_t)n_items * 4));
      launch_item_bounds(d_hd, d_hn, d_k, heap_stride, n_items, c->qbound.as<float>(), s);
      CKL();
    }
    IndexView vs = v;  // the candidate slots' view
    if ((st = run_scan(ix, qv, n_pairs, false, 0, use_bounds ? 1u : 0u, use_bounds, &vs)) != HIVF_OK) return st;
    launch_finalize_items(vs, qv, n_items, d_off, d_cl, d_k, c->cand_d.as<float>(), c->cand_row.as<uint32_t>(),
                          c->cand_thr.as<float>(), c->cand_n.as<uint32_t>(), d_hi, d_hd, d_hn, heap_stride, d_ch,
                          d_fb, s);
    CKL();
    launch_exact_items(v, qv, n_items, d_off, d_cl, d_k, d_hi, d_hd, d_hn, heap_stride, d_ch, d_fb, s);
    CKL();
  } else {
    launch_exact_items(v, qv, n_items, d_off, d_cl, d_k, d_hi, d_hd, d_hn, heap_stride, d_ch, nullptr, s);
    CKL();
  }
  CK(cudaMemcpyAsync(h + o_hi, d + o_hi, total - o_hi, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  int err = 0;
  std::memcpy(&err, h + o_err, 4);
  if (err) return fail(HIVF_EINVAL, "hivf_scan_items: non-finite query value");
  std::memcpy(heap_ids, h + o_hi, hb);
  std::memcpy(heap_dists, h + o_hd, hb);
  std::memcpy(heap_counts, h + o_hn, n_items * 4ull);
  if (n_pairs) std::memcpy(changed_out, h + o_ch, n_pairs);
  // auto policy (adapt_scan): items whose filter proof failed took the exact path
  if (!exact_only && n_pairs && c->opt_scan_kernel == 0 && !ix->auto_split) {
    const int* fb = reinterpret_cast<const int*>(h + o_fb);
    uint32_t nf = 0;
    for (uint32_t i = 0; i < n_items; ++i) nf += fb[i] != 0;
    adapt_scan(ix, n_items, nf);
  }
  return HIVF_OK;
}

// ---------------------------------------------------------------------------
// multi-GPU merge + residency
// ---------------------------------------------------------------------------

hivf_status hivf_merge_parts_device(hivf_ctx* ctx, uint32_t n_parts, uint32_t n_queries,
                                    uint32_t k, const uint64_t* d_ids, const double* d_dists,
                                    const uint32_t* d_counts, uint64_t* d_ids_out,
                                    double* d_dists_out, uint32_t* d_counts_out) {
  if (!ctx) return fail(HIVF_EINVAL, "ctx is NULL");
  if (k == 0 || n_parts == 0) return fail(HIVF_EINVAL, "merge: k and n_parts must be >= 1");
  if ((uint64_t)n_parts * k > 8192) return fail(HIVF_EUNSUPPORTED, "merge: n_parts*k > 8192");
  if (!n_queries) return HIVF_OK;
  CK(cudaSetDevice(ctx->device));
  launch_merge_parts(n_parts, n_queries, k, d_ids, d_dists, d_counts, d_ids_out, d_dists_out,
                     d_counts_out, ctx->stream);
  CKL();
  return HIVF_OK;
}

hivf_status hivf_residency_set(hivf_index* ix, const uint32_t* clusters, uint32_t n) {
  if (!ix) return fail(HIVF_EINVAL, "index is NULL");
  if (n && !clusters) return fail(HIVF_EINVAL, "clusters NULL");
  for (uint32_t i = 0; i < n; ++i)
    if (clusters[i] >= ix->K) return fail(HIVF_EINVAL, "cluster %u out of range", clusters[i]);
  if (!ix->tiered) {  // every list already lives in HBM: the set is bookkeeping only
    std::vector<uint8_t> res(ix->K, 0);
    for (uint32_t i = 0; i < n; ++i) res[clusters[i]] = 1;
    ix->resident.swap(res);
    return HIVF_OK;
  }
  CK(cudaSetDevice(ix->ctx->device));
  complete_swaps(ix);
  std::vector<uint8_t> want(ix->K, 0);
  for (uint32_t i = 0; i < n; ++i) want[clusters[i]] = 1;
  // evictions take effect immediately (tiered_cache.cpp:23-36): the list reads
  // from the backing store from the next launch on; its slot is reused only by
  // copies ordered after every launch issued so far
  std::vector<std::pair<uint32_t, const float*>> flips;
  for (uint32_t c = 0; c < ix->K; ++c)
    if (!want[c] && (ix->resident[c] || ix->swap_in[c])) {
      if (ix->swap_in[c]) {  // cancel an in-flight swap: forget it on completion
        for (auto& w : ix->swaps)
          w.lists.erase(std::remove(w.lists.begin(), w.lists.end(), c), w.lists.end());
        ix->swap_in[c] = 0;
      }
      if (ix->resident[c]) flips.push_back({c, ix->vec + ix->list_off[c] * ix->dpad});
      ix->resident[c] = 0;
      pool_free(ix, ix->slot_off[c], ix->list_bytes(c));
      ix->slot_off[c] = ~0ull;
    }
  hivf_status st = apply_flips(ix, flips);
  if (st != HIVF_OK) return st;
  cudaEvent_t after_evict;
  CK(cudaEventCreateWithFlags(&after_evict, cudaEventDisableTiming));
  CK(cudaEventRecord(after_evict, ix->ctx->stream));
  CK(cudaStreamWaitEvent(ix->copy_stream, after_evict, 0));
  cudaEventDestroy(after_evict);
  // admissions in the caller's order while they fit the pool: H2D copies on
  // the copy stream; the list stays non-resident until its copy completes
  hivf_index::Swap w{};
  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t c = clusters[i];
    if (ix->resident[c] || ix->swap_in[c]) continue;
    const uint64_t bytes = ix->list_bytes(c);
    if (bytes == 0) {
      ix->resident[c] = 1;  // an empty list is trivially resident
      continue;
    }
    const uint64_t off = pool_alloc(ix, bytes);
    if (off == ~0ull) continue;  // does not fit the HBM budget
    ix->slot_off[c] = off;
    ix->swap_in[c] = 1;
    CK(cudaMemcpyAsync(reinterpret_cast<uint8_t*>(ix->pool) + off, ix->vec + ix->list_off[c] * ix->dpad, bytes,
                       cudaMemcpyHostToDevice, ix->copy_stream));
    ix->swapped_in_bytes += bytes;
    w.lists.push_back(c);
  }
  if (!w.lists.empty()) {
    CK(cudaEventCreateWithFlags(&w.done, cudaEventDisableTiming));
    CK(cudaEventRecord(w.done, ix->copy_stream));
    ix->swaps.push_back(std::move(w));
  }
  return HIVF_OK;
}

hivf_status hivf_residency_get(const hivf_index* cix, uint8_t* out) {
  if (!cix || !out) return fail(HIVF_EINVAL, "NULL argument");
  hivf_index* ix = const_cast<hivf_index*>(cix);
  if (ix->tiered) complete_swaps(ix);
  std::memcpy(out, ix->resident.data(), ix->K);
  return HIVF_OK;
}

hivf_status hivf_residency_sync(hivf_index* ix) {
  if (!ix) return fail(HIVF_EINVAL, "index is NULL");
  if (!ix->tiered) return HIVF_OK;
  CK(cudaStreamSynchronize(ix->copy_stream));
  complete_swaps(ix);
  return HIVF_OK;
}

}  // extern "C"
