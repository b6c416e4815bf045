// internal.h -- the C-ABI's object definitions (hivf_ctx, hivf_index), the
// grow-only scratch buffers and the error helpers, shared by the C-ABI
// translation units (api.cu, shard.cu).  Host-only C++; not public.
#pragma once

#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/hivf.h"
#include "common.cuh"
#include "kernels.h"

using namespace hivf;

namespace hivf {
// thread-local last-error message (hivf_last_error); returns st
hivf_status fail(hivf_status st, const char* fmt, ...);
}  // namespace hivf

#define CK(call)                                                                         \
  do {                                                                                   \
    cudaError_t e_ = (call);                                                             \
    if (e_ != cudaSuccess)                                                               \
      return fail(e_ == cudaErrorMemoryAllocation ? HIVF_ENOMEM : HIVF_ECUDA, "%s: %s (%s:%d)", \
                  #call, cudaGetErrorString(e_), __FILE__, __LINE__);                    \
  } while (0)

#define CKL()                                                                            \
  do {                                                                                   \
    cudaError_t e_ = cudaGetLastError();                                                 \
    if (e_ != cudaSuccess)                                                               \
      return fail(HIVF_ECUDA, "kernel launch: %s (%s:%d)", cudaGetErrorString(e_), __FILE__, \
                  __LINE__);                                                             \
  } while (0)

namespace hivf {
// Bumped whenever something a captured search graph bakes in may have
// changed: a scratch buffer reallocation, an option, an index upload/destroy
// (see search_device_cached).
extern std::atomic<uint64_t> g_state_gen;

// Grow-only device buffer.
struct DBuf {
  void* p = nullptr;
  size_t bytes = 0;
  // grows by >= 2x from 64 KB: a stream of varying batch shapes (node-split
  // sub-stages) settles after a few calls instead of re-allocating (cudaFree
  // synchronises the device) whenever a batch is a little larger than before
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    want = std::max(want, 2 * bytes);
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    g_state_gen.fetch_add(1);
    want = std::max<size_t>(want, 64 << 10);  // 64 KB floor: small sub-stages never regrow
    cudaError_t e = cudaMalloc(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

struct HBuf {  // grow-only pinned host buffer
  void* p = nullptr;
  size_t bytes = 0;
  cudaError_t ensure(size_t want) {
    if (want <= bytes) return cudaSuccess;
    // pinned allocations cost milliseconds and synchronise: start at 1 MB, double
    want = std::max(std::max(want, 2 * bytes), (size_t)1 << 20);
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMallocHost(&p, want);
    if (e == cudaSuccess) bytes = want;
    return e;
  }
  void release() {
    if (p) cudaFreeHost(p);
    p = nullptr;
    bytes = 0;
  }
  template <typename T>
  T* as() const {
    return reinterpret_cast<T*>(p);
  }
};

}  // namespace hivf

struct hivf_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int sm_count = 148;
  // options
  uint32_t opt_seg_rows = 0;  // 0: chosen per index from its size (auto_seg_rows)
  int opt_force_exact = 0;
  // fp16 filter copy (option "filter_h16"): built at index finish when 1 and
  // used by the single-pass tensor-core scan while 1
  int opt_h16 = 1;
  // coarse distances on the tensor cores (option "coarse_tc", env HIVF_COARSE_TC):
  // kind::f16 over fp16 copies of centroids and queries, for indexes that have
  // the centroid copy (built at index creation unless 0); 1 = batches of at
  // least 2^26 multiply-adds, 2 = always, 0 = never
  int opt_coarse_tc = 1;
  // search path: coarse select in set mode (option "coarse_set", env
  // HIVF_COARSE_SET): only centroids the bound cannot place get the exact double
  int opt_coarse_set = 1;
  // drop-bound seed (launch_seed_bounds): rows per query, and the batch density
  // (pairs per list) from which it runs
  uint32_t opt_seed_rows = 32;
  float opt_seed_ppl = 16.f;
  // 0 auto (tensor cores when the dim fits; single-pass tf32, escalating to the
  // split kernel when the data makes its bound too loose), 1 FFMA, 2 tcgen05
  // split-precision, 3 tcgen05 single-pass
  int opt_scan_kernel = 0;
  int opt_scan_ctas = 0;
  int opt_no_bound = 0;  // debug: disable the scan's shared per-query drop bound
  // tiered residency: list bytes an index may keep in HBM (0 = all lists in HBM);
  // the rest stays in a pinned host backing store read over PCIe
  uint64_t opt_hbm_list_budget = 0;
  int tc_conv = 2;  // this device's fp32->tf32 operand conversion (tc_conversion_mode)
  TcOpts tc{0, tc_wide_ppl_default(), 0, tc_wide2_ppl_default(), tc_pair_ppl_default()};  // tensor-core scan tuning (tc_qmax, tc_wide_ppl, tc_variant)
  // scratch
  DBuf qs, qn2, qnorm, qsc, err, dist32, plans, pdists, flags_c, flags_f, pq, pl, list_cnt, list_poff,
      list_cur, list_ioff, sorted_pairs, items, n_items, work_ctr, cand_d, cand_row, cand_thr,
      cand_n, out_ids, qin, x_ids, x_d, x_cnt, x_tot, tau, flags2, qbound, rep_entries, rep_n, rep_cnt,
      rep_d, rep_ids, qshift, qwide, coarse_all, coarse_part, qh16;
  HBuf hstage;
  hivf_stats stats{};
  uint32_t last_nq = 0;
  uint32_t last_K = 0;
  const hivf_index* last_index = nullptr;
  uint32_t last_kind = 0;
  uint32_t last_group = 0;  // queries per scan work item of the last scan
  uint32_t last_filter_bits = 32;  // 16: the last scan read the fp16 filter copy
  uint32_t last_coarse_bits = 32;  // 16: the last coarse assign ran on the tensor cores
  bool stats_adapted = false;
  // phase timing (option "time_kernels"): one event set per call, resolved lazily
  int opt_time = 0;
  int opt_search_graph = 1;  // hivf_search replays a captured graph for a repeated batch shape
  // the cached search graph (search_device_cached): key, exec, and the host
  // state the captured call left behind
  struct SearchGraph {
    const void* ix = nullptr;
    const float* q = nullptr;
    const void* out = nullptr;
    uint32_t n = 0, nprobe = 0, k = 0;
    int kind = -1;
    uint64_t gen = 0;
    bool seen = false;
    cudaGraphExec_t exec = nullptr;
    hivf_stats stats{};
    int last_kind = 0;
    cudaStream_t failed_stream = nullptr;  // capture failed on it: plain launches there
  } sgraph;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  uint32_t timed_calls = 0;
  double acc_assign = 0, acc_scan = 0, acc_fin = 0;
  cudaEvent_t next_event() {
    if (ev_used == ev_pool.size()) {
      cudaEvent_t e;
      cudaEventCreate(&e);
      ev_pool.push_back(e);
    }
    return ev_pool[ev_used++];
  }
  void mark(int slot) {  // slot 0..3 of the current set
    if (!opt_time) return;
    cudaEventRecord(next_event(), stream);
    (void)slot;
  }
  void resolve_timers() {
    for (size_t i = 0; i + 4 <= ev_used; i += 4) {
      float a = 0, b = 0, c = 0;
      cudaEventSynchronize(ev_pool[i + 3]);
      cudaEventElapsedTime(&a, ev_pool[i], ev_pool[i + 1]);
      cudaEventElapsedTime(&b, ev_pool[i + 1], ev_pool[i + 2]);
      cudaEventElapsedTime(&c, ev_pool[i + 2], ev_pool[i + 3]);
      acc_assign += a;
      acc_scan += b;
      acc_fin += c;
      ++timed_calls;
    }
    ev_used = 0;
  }
  ~hivf_ctx() {
    for (cudaEvent_t e : ev_pool) cudaEventDestroy(e);
    for (DBuf* b : {&qs, &qn2, &qnorm, &qsc, &err, &dist32, &plans, &pdists, &flags_c, &flags_f, &pq,
                    &pl, &list_cnt, &list_poff, &list_cur, &list_ioff, &sorted_pairs, &items,
                    &n_items, &work_ctr, &cand_d, &cand_row, &cand_thr, &cand_n, &out_ids, &qin,
                    &x_ids, &x_d, &x_cnt, &x_tot, &tau, &flags2, &qbound, &rep_entries, &rep_n, &rep_cnt,
                    &rep_d, &rep_ids, &qshift, &qwide})
      b->release();
    hstage.release();
    if (sgraph.exec) cudaGraphExecDestroy(sgraph.exec);
    if (own_stream && stream) cudaStreamDestroy(stream);
  }
};

struct hivf_index {
  hivf_ctx* ctx = nullptr;
  uint32_t dim = 0, dpad = 0, K = 0;
  int metric = 0;
  uint64_t N = 0;
  std::vector<uint64_t> list_off;  // host copy
  float* vec = nullptr;
  // fp16 filter copy (nullptr: none): N rows x dpf floats, per-list unscale lsc
  float* vech = nullptr;
  float* lsc = nullptr;
  uint32_t dpf = 0;
  uint64_t* ids = nullptr;
  float* xnorm2 = nullptr;
  uint64_t* d_list_off = nullptr;
  uint32_t* maxnorm_bits = nullptr;
  float* cent = nullptr;
  float* cnorm2 = nullptr;
  float* cnorm = nullptr;
  // fp16 centroid copy for the tensor-core coarse pass (nullptr: FFMA pass):
  // tile layout of launch_pack_coarse_tc, shared unscale 2^-e_c, largest norm bound
  uint8_t* centh = nullptr;
  float csc = 0.f, cmax = 0.f;
  uint32_t* list_order = nullptr;
  int* d_err = nullptr;
  uint64_t rows_added = 0;
  bool finished = false;
  double mean_assigned = -1.0;
  uint32_t seg_rows = 4096, s_max = 1;
  std::vector<uint8_t> resident;
  // locator (doc id -> row), built on the first hivf_index_locate
  uint64_t* loc_ids = nullptr;
  uint64_t* loc_rows = nullptr;
  // ---- tiered residency (hivf_residency_set) ----
  bool tiered = false;           // vec is pinned host memory, hot lists copied into pool
  float* pool = nullptr;         // HBM slots for resident lists
  uint64_t pool_bytes = 0;
  const float** d_list_ptr = nullptr;  // device table read by the kernels
  std::vector<uint64_t> slot_off;      // per list: byte offset in pool, or ~0
  std::vector<std::pair<uint64_t, uint64_t>> free_ext;  // free (offset, size) extents
  std::vector<uint8_t> swap_in;        // per list: copy in flight
  struct Swap {
    cudaEvent_t done;
    std::vector<uint32_t> lists;
  };
  std::vector<Swap> swaps;             // in flight, oldest first
  cudaStream_t copy_stream = nullptr;
  uint64_t swapped_in_bytes = 0;
  uint64_t list_bytes(uint32_t c) const { return (list_off[c + 1] - list_off[c]) * dpad * 4; }
  int auto_split = 0;  // auto policy: 0 single-pass tf32, 1 split-precision
  uint32_t adapt_seen = 0, adapt_fallback = 0;
  // scan kernel for the next call: 1 FFMA, 2 tensor-core split, 3 tensor-core single pass
  int scan_kind() const;
  IndexView view() const { return view_kind(scan_kind()); }
  // view carrying the filter bound of scan kernel `kind`
  IndexView view_kind(int kind) const {
    IndexView v{};
    const bool h16 = kind == 3 && vech && ctx->opt_h16;
    if (kind == 2) bound_tc(dim, &v.e_a, &v.e_b, &v.e_c);
    else if (h16) bound_h16(dim, &v.e_a, &v.e_b, &v.e_c);
    else if (kind == 3) bound_tc1(dim, &v.e_a, &v.e_b, &v.e_c);
    else bound_ffma(dim, &v.e_a, &v.e_b, &v.e_c);
    v.vech = h16 ? vech : nullptr;
    v.lsc = h16 ? lsc : nullptr;
    v.dpf = h16 ? dpf : dpad;
    v.vec = vec;
    v.list_ptr = tiered ? d_list_ptr : nullptr;
    v.ids = ids;
    v.xnorm2 = xnorm2;
    v.list_off = d_list_off;
    v.maxnorm = reinterpret_cast<const float*>(maxnorm_bits);
    v.cent = cent;
    v.cnorm2 = cnorm2;
    v.cnorm = cnorm;
    v.list_order = list_order;
    v.dim = dim;
    v.dpad = dpad;
    v.K = K;
    v.N = N;
    v.seg_rows = seg_rows;
    v.s_max = s_max;
    v.seg_split = 1;
    v.metric = metric;
    return v;
  }
  ~hivf_index() {
    if (copy_stream) cudaStreamSynchronize(copy_stream);
    for (auto& w : swaps) cudaEventDestroy(w.done);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (tiered && vec) cudaFreeHost(vec);
    else if (vec) cudaFree(vec);
    for (void* p : {(void*)centh, (void*)vech, (void*)lsc, (void*)ids, (void*)xnorm2, (void*)d_list_off, (void*)maxnorm_bits, (void*)cent,
                    (void*)cnorm2, (void*)cnorm, (void*)list_order, (void*)d_err, (void*)pool,
                    (void*)d_list_ptr, (void*)loc_ids, (void*)loc_rows})
      if (p) cudaFree(p);
  }
};

