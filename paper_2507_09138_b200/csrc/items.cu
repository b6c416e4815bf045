// items.cu -- node-split sub-search finalize (hivf_scan_items).
//
// Reference: ivf::search_clusters (/root/reference/proj/src/vector_index.cpp
// :291-317) run per BatchItem by RetrievalEngine::execute
// (/root/reference/proj/src/retrieval_engine.cpp:94-103): the cursor heap is
// carried in, every cluster of the item is scanned IN ORDER, TopKResult::insert
// (:38-53) is applied row by row, and each cluster reports whether any insert
// changed the heap (feeds unchanged_streak, :307-313).
//
// Device algorithm (one CTA per item), exact for unique doc ids:
//  A. prefix bounds: U_j = min(worst(H_0), k-th smallest upper bound over the
//     lists before j) bounds worst(H_{j-1}) from above; within list j only
//     its own top-k can enter, bounded by tau_j (k-th upper bound in list j).
//     Candidates of list j: kept rows with lower bound <= min(U_j, tau_j);
//     completeness checked against each segment's drop threshold.
//  B. exact fp64 distances for all candidates (parallel).
//  C. sequential replay, list by list, of TopKResult::insert on a register
//     heap (warp 0): rows that are not candidates provably never survive in
//     the heap, so the final heap and every per-cluster `changed` flag equal
//     the reference's (a row inserted then evicted inside the same list leaves
//     an inserted successor behind, so `changed` is unaffected).
// Items whose proof fails (or k > 32) run k_exact_items: the reference
// algorithm verbatim (exact distances, in-order inserts) on the GPU.
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace hivf {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kItThreads = 128;
constexpr int kItCand = 2048;
// an item's candidate slots (clusters x s_max) and per-cluster metadata staged
// into smem by all threads before the sequential per-cluster pass (the pass
// then runs on smem instead of a chain of dependent global loads per cluster)
constexpr uint32_t kItStage = 256;
constexpr uint32_t kItStageCl = 128;
constexpr float kInf = __builtin_inff();

__device__ __forceinline__ float it_merge32(float cur, float v) {
  const int lane = threadIdx.x & 31;
  const float o = __shfl_sync(FULL, v, 31 - lane);
  float x = fminf(cur, o);
#pragma unroll
  for (int s = 16; s > 0; s >>= 1) {
    const float p = __shfl_xor_sync(FULL, x, s);
    x = ((lane & s) == 0) ? fminf(x, p) : fmaxf(x, p);
  }
  return x;
}

// Ascending bitonic sort / clean of one (distance, id) pair per lane (pair_less order).
__device__ __forceinline__ void warp_sort_pairs(double& d, uint64_t& id, int lane) {
#pragma unroll
  for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
    for (int jj = kk >> 1; jj > 0; jj >>= 1) {
      const double pd = __shfl_xor_sync(FULL, d, jj);
      const uint64_t pi = __shfl_xor_sync(FULL, id, jj);
      const bool keep_min = ((lane & jj) == 0) == ((lane & kk) == 0);
      if (keep_min == pair_less(pd, pi, d, id)) {
        d = pd;
        id = pi;
      }
    }
  }
}
__device__ __forceinline__ void warp_clean_pairs(double& d, uint64_t& id, int lane) {
#pragma unroll
  for (int jj = 16; jj > 0; jj >>= 1) {
    const double pd = __shfl_xor_sync(FULL, d, jj);
    const uint64_t pi = __shfl_xor_sync(FULL, id, jj);
    const bool keep_min = (lane & jj) == 0;
    if (keep_min == pair_less(pd, pi, d, id)) {
      d = pd;
      id = pi;
    }
  }
}

// TopKResult::insert (vector_index.cpp:38-53) on a warp-register heap:
// lane t holds entry t (t < n).  Returns true when the set changed.
__device__ __forceinline__ bool warp_heap_insert(double& hd, uint64_t& hid, uint32_t& n, uint32_t k,
                                                 uint64_t id, double d) {
  const int lane = threadIdx.x & 31;
  if (k == 0) return false;
  const unsigned dup = __ballot_sync(FULL, lane < (int)n && hid == id);
  if (dup) {
    const int at = __ffs(dup) - 1;
    const double old = __shfl_sync(FULL, hd, at);
    if (d >= old) return false;
    // erase entry `at` (shift the tail left by one)
    const double nd = __shfl_down_sync(FULL, hd, 1);
    const uint64_t ni = __shfl_down_sync(FULL, hid, 1);
    if (lane >= at) {
      hd = nd;
      hid = ni;
    }
    n -= 1;
  }
  const int pos = __popc(__ballot_sync(FULL, lane < (int)n && pair_less(hd, hid, d, id)));
  if (n >= k && pos == (int)n) return false;
  const double ud = __shfl_up_sync(FULL, hd, 1);
  const uint64_t ui = __shfl_up_sync(FULL, hid, 1);
  if (lane > pos) {
    hd = ud;
    hid = ui;
  } else if (lane == pos) {
    hd = d;
    hid = id;
  }
  n = min(n + 1, k);
  return true;
}

__global__ void __launch_bounds__(kItThreads) k_finalize_items(
    IndexView ix, QueryView qv, uint32_t n_items, const uint32_t* __restrict__ item_off,
    const uint32_t* __restrict__ clusters, const uint32_t* __restrict__ kv,
    const float* __restrict__ cand_d, const uint32_t* __restrict__ cand_row,
    const float* __restrict__ cand_thr, const uint32_t* __restrict__ cand_n, double eps,
    double ab, uint64_t* heap_ids, double* heap_d, uint32_t* heap_n, uint32_t stride,
    uint8_t* changed, int* flags) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t sm[];
  double* cdist = reinterpret_cast<double*>(sm);                // kItCand
  uint64_t* cid = reinterpret_cast<uint64_t*>(cdist + kItCand);  // kItCand
  uint32_t* crow = reinterpret_cast<uint32_t*>(cid + kItCand);   // kItCand
  uint32_t* clist = crow + kItCand;                              // kItCand
  uint32_t* cj_off = clist + kItCand;                            // (m_items+1) candidate offsets per cluster
  float* qsh = reinterpret_cast<float*>(cj_off + kNprobeMax + 1);  // dpad
  float* st_d = qsh + ix.dpad;                                   // kItStage x 32
  float* st_thr = st_d + kItStage * kKP;                         // kItStage
  uint32_t* st_n = reinterpret_cast<uint32_t*>(st_thr + kItStage);  // kItStage
  uint32_t* st_c = st_n + kItStage;                              // kItStageCl: cluster id
  uint32_t* st_ns = st_c + kItStageCl;                           // kItStageCl: slots
  float* st_E = reinterpret_cast<float*>(st_ns + kItStageCl);    // kItStageCl: filter bound
  __shared__ int s_bad;
  const uint32_t it = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t j0 = item_off[it], j1 = item_off[it + 1];
  const uint32_t mcl = j1 - j0;
  const uint32_t k = kv[it];
  const float qn = qv.qnorm[it];
  for (uint32_t d = threadIdx.x; d < ix.dpad; d += blockDim.x) qsh[d] = qv.qs[(uint64_t)it * ix.dpad + d];
  if (threadIdx.x == 0) s_bad = (k > 32u || mcl > kNprobeMax) ? 1 : 0;
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) flags[it] = 1;
    return;
  }
  const bool staged = mcl <= kItStageCl && mcl * ix.s_max <= kItStage;
  if (staged) {
    const uint64_t sbase = (uint64_t)j0 * ix.s_max;
    const uint32_t S = mcl * ix.s_max;
    for (uint32_t j = threadIdx.x; j < mcl; j += blockDim.x) {
      const uint32_t c = clusters[j0 + j];
      st_c[j] = c;
      st_ns[j] = slots_of(ix, ix.list_off[c + 1] - ix.list_off[c]);
      st_E[j] = seg_bound(ix, qn, ix.maxnorm[c]);
    }
    for (uint32_t i = threadIdx.x; i < S; i += blockDim.x) {
      st_n[i] = cand_n[sbase + i];
      st_thr[i] = cand_thr[sbase + i];
    }
    for (uint32_t i = threadIdx.x; i < S * kKP; i += blockDim.x) st_d[i] = cand_d[sbase * kKP + i];
    __syncthreads();
  }
  // A + candidate collection (warp 0, in plan order -> candidates grouped by cluster)
  if (warp == 0) {
    const uint32_t n0 = heap_n[it];
    float U0 = kInf;
    if (n0 >= k && n0 > 0) U0 = __double2float_ru(heap_d[(uint64_t)it * stride + n0 - 1]);
    float cur = kInf;  // top-32 upper bounds of the lists before j
    uint32_t cnt = 0;
    bool bad = false;
    for (uint32_t j = 0; j < mcl; ++j) {
      const uint32_t c = staged ? st_c[j] : clusters[j0 + j];
      const float E = staged ? st_E[j] : seg_bound(ix, qn, ix.maxnorm[c]);
      const uint32_t ns = staged ? st_ns[j] : slots_of(ix, ix.list_off[c + 1] - ix.list_off[c]);
      float lj = kInf;
      for (uint32_t s = 0; s < ns; ++s) {
        const uint64_t slot = (uint64_t)(j0 + j) * ix.s_max + s;
        const uint32_t si = j * ix.s_max + s;
        const uint32_t n = staged ? st_n[si] : cand_n[slot];
        const float v =
            lane < (int)n ? __fadd_ru(staged ? st_d[si * kKP + lane] : cand_d[slot * kKP + lane], E) : kInf;
        lj = it_merge32(lj, v);
      }
      const float tau_j = __shfl_sync(FULL, lj, (int)k - 1);
      const float u_prev = __shfl_sync(FULL, cur, (int)k - 1);
      const float lim = fminf(fminf(U0, u_prev), tau_j);
      if (lane == 0) cj_off[j] = cnt;
      for (uint32_t s = 0; s < ns; ++s) {
        const uint64_t slot = (uint64_t)(j0 + j) * ix.s_max + s;
        const uint32_t si = j * ix.s_max + s;
        const uint32_t n = staged ? st_n[si] : cand_n[slot];
        const bool take =
            lane < (int)n && __fsub_rd(staged ? st_d[si * kKP + lane] : cand_d[slot * kKP + lane], E) <= lim;
        const unsigned m = __ballot_sync(FULL, take);
        if (take) {
          const uint32_t pos = cnt + __popc(m & ((1u << lane) - 1));
          if (pos < kItCand) {
            crow[pos] = cand_row[slot * kKP + lane];
            clist[pos] = c;
          }
        }
        cnt += __popc(m);
        if (__fsub_rd(staged ? st_thr[si] : cand_thr[slot], E) <= lim) bad = true;
      }
      cur = it_merge32(cur, lj);
    }
    if (lane == 0) {
      cj_off[mcl] = cnt;
      if (bad || cnt > kItCand) s_bad = 1;
    }
  }
  __syncthreads();
  if (s_bad) {
    if (threadIdx.x == 0) flags[it] = 1;
    return;
  }
  const uint32_t m = cj_off[mcl];
  // B. exact distances (loads pipelined ahead of each sequential chain)
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
    const uint32_t c = clist[i];
    const uint64_t lbeg = ix.list_off[c];
    const uint64_t n_c = ix.list_off[c + 1] - lbeg;
    const uint64_t lr = crow[i] - lbeg;
    const float* lb = list_base(ix, c, lbeg);
    cdist[i] = exact_row_pipelined(ix.dim, qsh, [&](uint32_t g) {
      return __ldg(reinterpret_cast<const float4*>(lb + swz_offset(0, n_c, lr, g * 4, ix.dpad)));
    });
    cid[i] = ix.ids[crow[i]];
  }
  __syncthreads();
  // C. replay, cluster by cluster (vector_index.cpp:296-317 inserting the
  // cluster's rows into TopKResult, :38-53).  The heap after cluster j is the
  // top-k of the heap before it and the cluster's rows (a set in the
  // (distance, id) order, whatever the insertion order), and the cluster
  // changed the heap iff one of its rows entered -- its last accepted row is
  // never evicted within the cluster, so that is: a row beats the worst of a
  // full heap (or the heap is not full) -- or it lowered a duplicate id's
  // distance.  So each round of <= 32 candidates is one warp-wide merge:
  // bitonic sort, reversed min against the heap, bitonic clean.
  if (warp == 0) {
    uint32_t n = heap_n[it];
    double hd = lane < (int)n ? heap_d[(uint64_t)it * stride + lane] : DBL_MAX;
    uint64_t hid = lane < (int)n ? heap_ids[(uint64_t)it * stride + lane] : ~0ull;
    for (uint32_t j = 0; j < mcl; ++j) {
      bool ch = false;
      const uint32_t b0 = cj_off[j], b1 = cj_off[j + 1];
      for (uint32_t a0 = b0; k && a0 < b1; a0 += 32) {  // k = 0: nothing can enter
        bool valid = a0 + lane < b1;
        double cd = valid ? cdist[a0 + lane] : DBL_MAX;
        uint64_t ci = valid ? cid[a0 + lane] : ~0ull;
        // ids already in the heap: a smaller distance replaces the entry, else the row is a no-op
        bool removed = false;
        for (uint32_t t = 0; t < n; ++t) {
          const uint64_t ht = __shfl_sync(FULL, hid, t);
          const double hdt = __shfl_sync(FULL, hd, t);
          const unsigned dm = __ballot_sync(FULL, valid && ci == ht);
          if (!dm) continue;
          const int src = __ffs(dm) - 1;
          if (__shfl_sync(FULL, cd, src) < hdt) {
            if (lane == (int)t) {
              hd = DBL_MAX;
              hid = ~0ull;
            }
            removed = true;
            ch = true;
          } else if (lane == src) {
            valid = false;
            cd = DBL_MAX;
            ci = ~0ull;
          }
        }
        if (removed) {
          warp_sort_pairs(hd, hid, lane);
          n = __popc(__ballot_sync(FULL, lane < (int)n && !(hd == DBL_MAX && hid == ~0ull)));
        }
        const double wd = __shfl_sync(FULL, hd, (int)k - 1);
        const uint64_t wi = __shfl_sync(FULL, hid, (int)k - 1);
        const uint32_t nv = __popc(__ballot_sync(FULL, valid));
        ch |= __any_sync(FULL, valid && (n < k || pair_less(cd, ci, wd, wi)));
        warp_sort_pairs(cd, ci, lane);
        const double rd = __shfl_sync(FULL, cd, 31 - lane);
        const uint64_t ri = __shfl_sync(FULL, ci, 31 - lane);
        if (pair_less(rd, ri, hd, hid)) {
          hd = rd;
          hid = ri;
        }
        warp_clean_pairs(hd, hid, lane);
        if (lane >= (int)k) {
          hd = DBL_MAX;
          hid = ~0ull;
        }
        n = min(k, n + nv);
      }
      if (lane == 0) changed[j0 + j] = ch ? 1 : 0;
    }
    if (lane < (int)n) {
      heap_d[(uint64_t)it * stride + lane] = hd;
      heap_ids[(uint64_t)it * stride + lane] = hid;
    }
    if (lane == 0) {
      heap_n[it] = n;
      flags[it] = 0;
    }
  }
}

// The reference algorithm verbatim for flagged items / k > 32: every row of
// every cluster, exact distance, TopKResult::insert in row order.
__global__ void __launch_bounds__(256) k_exact_items(IndexView ix, QueryView qv, uint32_t n_items,
                                                     const uint32_t* __restrict__ item_off,
                                                     const uint32_t* __restrict__ clusters,
                                                     const uint32_t* __restrict__ kv,
                                                     uint64_t* heap_ids, double* heap_d,
                                                     uint32_t* heap_n, uint32_t stride,
                                                     uint8_t* changed, const int* flags) {
  pdl_wait();
  const uint32_t it = blockIdx.x;
  if (flags && !flags[it]) return;
  extern __shared__ __align__(16) uint8_t sm[];
  const uint32_t k = kv[it];
  double* hd = reinterpret_cast<double*>(sm);            // k+1
  uint64_t* hi = reinterpret_cast<uint64_t*>(hd + k + 1);  // k+1
  double* td = reinterpret_cast<double*>(hi + k + 1);     // 256
  uint64_t* ti = reinterpret_cast<uint64_t*>(td + 256);   // 256
  float* qsh = reinterpret_cast<float*>(ti + 256);        // dpad
  __shared__ uint32_t s_n;
  __shared__ int s_ch;
  for (uint32_t d = threadIdx.x; d < ix.dpad; d += blockDim.x) qsh[d] = qv.qs[(uint64_t)it * ix.dpad + d];
  if (threadIdx.x == 0) {
    s_n = heap_n[it];
    for (uint32_t i = 0; i < s_n; ++i) {
      hd[i] = heap_d[(uint64_t)it * stride + i];
      hi[i] = heap_ids[(uint64_t)it * stride + i];
    }
  }
  __syncthreads();
  for (uint32_t j = item_off[it]; j < item_off[it + 1]; ++j) {
    const uint32_t c = clusters[j];
    const uint64_t beg = ix.list_off[c], end = ix.list_off[c + 1];
    if (threadIdx.x == 0) s_ch = 0;
    for (uint64_t r0 = beg; r0 < end; r0 += blockDim.x) {
      const uint64_t r = r0 + threadIdx.x;
      if (r < end) {
        const uint64_t n_c = end - beg, lr = r - beg;
        const float* lb = list_base(ix, c, beg);
        td[threadIdx.x] = exact_row_pipelined(ix.dim, qsh, [&](uint32_t g) {
          return __ldg(reinterpret_cast<const float4*>(lb + swz_offset(0, n_c, lr, g * 4, ix.dpad)));
        });
        ti[threadIdx.x] = ix.ids[r];
      }
      // Only rows that beat the heap's current worst can change it (the worst
      // only improves while this round is replayed, and a duplicate id already
      // in a full heap has distance <= worst): a block-wide prefilter against
      // the worst at the start of the round leaves the serial replay a handful
      // of rows instead of 256.
      const uint32_t lim = (uint32_t)min((uint64_t)blockDim.x, end - r0);
      bool cand = false;
      if (threadIdx.x < lim) {
        const uint32_t n0 = s_n;
        cand = n0 < k || pair_less(td[threadIdx.x], ti[threadIdx.x], hd[n0 - 1], hi[n0 - 1]);
      }
      const int any = __syncthreads_or(cand);
      if (any && threadIdx.x == 0) {
        uint32_t n = s_n;
        for (uint32_t t = 0; t < lim; ++t) {
          const double d = td[t];
          const uint64_t id = ti[t];
          if (k == 0) break;
          if (n >= k && !pair_less(d, id, hd[n - 1], hi[n - 1])) continue;
          // TopKResult::insert
          bool skip = false;
          for (uint32_t i = 0; i < n; ++i) {
            if (hi[i] == id) {
              if (d >= hd[i]) {
                skip = true;
              } else {
                for (uint32_t q = i; q + 1 < n; ++q) {
                  hd[q] = hd[q + 1];
                  hi[q] = hi[q + 1];
                }
                --n;
              }
              break;
            }
          }
          if (skip) continue;
          uint32_t lo = 0, up = n;
          while (lo < up) {
            const uint32_t mid = (lo + up) >> 1;
            if (pair_less(hd[mid], hi[mid], d, id)) lo = mid + 1; else up = mid;
          }
          if (n >= k && lo == n) continue;
          for (uint32_t q = n; q > lo; --q) {
            hd[q] = hd[q - 1];
            hi[q] = hi[q - 1];
          }
          hd[lo] = d;
          hi[lo] = id;
          ++n;
          if (n > k) n = k;
          s_ch = 1;
        }
        s_n = n;
      }
      __syncthreads();
    }
    if (threadIdx.x == 0) changed[j] = (uint8_t)s_ch;
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    heap_n[it] = s_n;
    for (uint32_t i = 0; i < s_n; ++i) {
      heap_d[(uint64_t)it * stride + i] = hd[i];
      heap_ids[(uint64_t)it * stride + i] = hi[i];
    }
  }
}

}  // namespace

void launch_finalize_items(const IndexView& ix, const QueryView& qv, uint32_t n_items,
                           const uint32_t* item_off, const uint32_t* clusters, const uint32_t* k,
                           const float* cand_d, const uint32_t* cand_row, const float* cand_thr,
                           const uint32_t* cand_n, uint64_t* heap_ids, double* heap_d,
                           uint32_t* heap_n, uint32_t heap_stride, uint8_t* changed, int* flags,
                           cudaStream_t s) {
  if (!n_items) return;
  const size_t smem = (size_t)kItCand * (8 + 8 + 4 + 4) + (kNprobeMax + 1) * 4 + (size_t)ix.dpad * 4 +
                      (size_t)kItStage * (kKP + 2) * 4 + (size_t)kItStageCl * 12;
  smem_optin((const void*)k_finalize_items, 220 * 1024);
  launch_pdl(k_finalize_items, dim3(n_items), dim3(kItThreads), smem, s, ix, qv, n_items, item_off, clusters, k, cand_d,
                                                     cand_row, cand_thr, cand_n, filter_eps(ix.dim),
                                                     filter_abs(ix.dim), heap_ids, heap_d, heap_n,
                                                     heap_stride, changed, flags);
}

void launch_exact_items(const IndexView& ix, const QueryView& qv, uint32_t n_items,
                        const uint32_t* item_off, const uint32_t* clusters, const uint32_t* k,
                        uint64_t* heap_ids, double* heap_d, uint32_t* heap_n,
                        uint32_t heap_stride, uint8_t* changed, const int* flags,
                        cudaStream_t s) {
  if (!n_items) return;
  const size_t smem = (size_t)(kExactMaxK + 1) * 16 + 256 * 16 + (size_t)ix.dpad * 4;
  smem_optin((const void*)k_exact_items, 200 * 1024);
  launch_pdl(k_exact_items, dim3(n_items), dim3(256), smem, s, ix, qv, n_items, item_off, clusters, k, heap_ids, heap_d,
                                           heap_n, heap_stride, changed, flags);
}

namespace {
// Rows with d^ >= float_ru(worst) + E can never enter a full heap at any step
// of the sub-stage (its worst only decreases), so the scan may drop them
// without touching the per-cluster `changed` semantics.
__global__ void k_item_bounds(const double* heap_d, const uint32_t* heap_n, const uint32_t* k, uint32_t stride,
                              uint32_t n_items, float* out) {
  pdl_wait();
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_items) return;
  const uint32_t n = heap_n[i];
  float u = 3.3e38f;  // "none" (the scan treats >= 3e38 as no bound)
  if (n > 0 && n >= k[i]) {
    const double w = heap_d[(uint64_t)i * stride + n - 1];
    if (w < 3.0e38) u = __double2float_ru(w);
    if (!(u > 0.f)) u = 0.f;
  }
  out[i] = u;
}
}  // namespace

void launch_item_bounds(const double* heap_d, const uint32_t* heap_n, const uint32_t* k, uint32_t stride,
                        uint32_t n_items, float* out, cudaStream_t s) {
  if (n_items) launch_pdl(k_item_bounds, dim3((n_items + 255) / 256), dim3(256), 0, s, heap_d, heap_n, k, stride, n_items, out);
}

}  // namespace hivf
