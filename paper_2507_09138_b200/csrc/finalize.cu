// finalize.cu -- K4/K5: exact fp64 re-rank and top-k assembly.
//
// The scan kept, per (query, segment), the 32 best rows by the fp32 distance
// d32 plus a "drop threshold" T (every row NOT kept has d32 >= T).  With the
// per-(query, list) error bound E (common.cuh):
//   tau = k-th smallest of (d32 + E) over all kept rows of the query  ->
//         the reference's k-th distance is <= tau;
//   candidates = kept rows with d32 - E <= tau  -> superset of the true top-k;
//   proof of completeness: every segment has T - E > tau (else the query is
//   flagged and redone by the exact streaming kernel).
// Candidates get the reference's exact double (embedding.hpp:27-34, sequential,
// no FMA) and are ordered by (distance, doc id) (vector_index.hpp:41-44), so
// ids AND distances are bit-identical to TopKResult after the full plan
// (vector_index.cpp:38-53,291-317).
#include <algorithm>
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace hivf {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kFinThreads = 256;
constexpr int kCandMax = 512;
constexpr uint32_t kSlotCap = 320;  // staged (plan position, segment) slots per query and chunk
constexpr uint32_t kSpCap = 2048;   // (plan position, segment) slot ids per query held in smem
constexpr uint32_t kRepMax = 64;    // failing segments per query repaired in place
constexpr int kRepChunk = 256;      // rows per repair work unit
constexpr float kInf = __builtin_inff();

// Merge a sorted-ascending 32-lane list `v` into sorted-ascending `cur`
// (keeps the 32 smallest).
__device__ __forceinline__ float warp_merge32(float cur, float v) {
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

template <typename IdT>
__device__ void block_sort_pairs(double* d, IdT* id, uint32_t n) {
  for (uint32_t size = 2; size <= n; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < n / 2; i += blockDim.x) {
        const uint32_t lo = 2 * i - (i & (stride - 1));
        const uint32_t hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const bool gt = pair_less(d[hi], (uint64_t)id[hi], d[lo], (uint64_t)id[lo]);
        if (gt == up) {
          const double td = d[lo];
          d[lo] = d[hi];
          d[hi] = td;
          const IdT ti = id[lo];
          id[lo] = id[hi];
          id[hi] = ti;
        }
      }
    }
  }
  __syncthreads();
}

__device__ __forceinline__ uint32_t nseg_of(const IndexView& ix, uint32_t c) {
  return slots_of(ix, ix.list_off[c + 1] - ix.list_off[c]);
}

// One CTA per query.
__global__ void __launch_bounds__(kFinThreads) k_finalize_search(
    IndexView ix, QueryView qv, const uint32_t* __restrict__ plans, uint32_t nprobe, uint32_t k,
    const float* __restrict__ cand_d, const uint32_t* __restrict__ cand_row,
    const float* __restrict__ cand_thr, const uint32_t* __restrict__ cand_n, double eps,
    double ab, uint64_t* __restrict__ ids_out, double* __restrict__ d_out,
    uint32_t* __restrict__ counts_out, int* flags, float* __restrict__ tau_out,
    RepairState rep) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t sm[];
  double* cdist = reinterpret_cast<double*>(sm);                 // kCandMax
  uint64_t* cid = reinterpret_cast<uint64_t*>(cdist + kCandMax);  // kCandMax
  uint32_t* crow = reinterpret_cast<uint32_t*>(cid + kCandMax);   // kCandMax
  uint32_t* clist = crow + kCandMax;                              // kCandMax
  double* qsh = reinterpret_cast<double*>(clist + kCandMax);      // dpad (widened once)
  __shared__ float wl[kFinThreads / 32][32];
  __shared__ float s_tau;
  __shared__ uint32_t s_cnt;
  __shared__ int s_bad;
  __shared__ unsigned long long s_total;
  __shared__ uint32_t s_nfail;
  __shared__ uint32_t s_fail[kRepMax];  // failing slots (plan position * s_max + segment)
  const uint32_t b = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NW = kFinThreads / 32;
  const float qn = qv.qnorm[b];
  for (uint32_t d = threadIdx.x; d < ix.dpad; d += blockDim.x) qsh[d] = qv.qs[(uint64_t)b * ix.dpad + d];
  if (threadIdx.x == 0) {
    s_cnt = 0;
    s_bad = 0;
    s_total = 0;
    s_nfail = 0;
  }
  __syncthreads();
  // 0. per plan position metadata (list, segment count, bound) -> smem, in parallel
  float* pE = reinterpret_cast<float*>(qsh + ix.dpad);   // nprobe
  uint32_t* pc = reinterpret_cast<uint32_t*>(pE + nprobe);  // nprobe
  uint32_t* pns = pc + nprobe;                            // nprobe
  {
    unsigned long long tot = 0;
    for (uint32_t p = threadIdx.x; p < nprobe; p += blockDim.x) {
      const uint32_t c = plans[(uint64_t)b * nprobe + p];
      const uint64_t rows = ix.list_off[c + 1] - ix.list_off[c];
      pc[p] = c;
      pns[p] = slots_of(ix, rows);
      pE[p] = seg_bound(ix, qn, ix.maxnorm[c]);
      tot += rows;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) tot += __shfl_xor_sync(FULL, tot, o);
    if (lane == 0 && tot) atomicAdd(&s_total, tot);  // one 64-bit smem atomic (a CAS loop) per warp
  }
  __syncthreads();
  // Compacted list of the query's valid (plan position, segment) slots, and
  // their candidate lists staged into smem with all threads' loads in flight
  // (the scan's outputs are read once, latency paid once).
  uint32_t* soff = pns + nprobe;                              // nprobe + 1
  uint32_t* sp = soff + nprobe + 1;                           // kSpCap
  uint32_t* sn = sp + kSpCap;                                 // kSlotCap
  float* sthr = reinterpret_cast<float*>(sn + kSlotCap);      // kSlotCap
  float* sdv = sthr + kSlotCap;                               // kSlotCap x 32
  __shared__ uint32_t s_nslots;
  if (warp == 0) {  // exclusive scan of pns (nprobe <= kNprobeMax) by one warp
    const uint32_t per = (nprobe + 31) / 32;
    const uint32_t p0 = min(nprobe, lane * per), p1 = min(nprobe, p0 + per);
    uint32_t local = 0;
    for (uint32_t p = p0; p < p1; ++p) local += pns[p];
    uint32_t incl = local;
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += y;
    }
    uint32_t run = incl - local;
    for (uint32_t p = p0; p < p1; ++p) {
      soff[p] = run;
      run += pns[p];
    }
    if (lane == 31) {
      soff[nprobe] = incl;
      s_nslots = incl;
    }
  }
  __syncthreads();
  const uint32_t V = s_nslots;
  const uint64_t slot0 = (uint64_t)b * nprobe * ix.s_max;
  if (V <= kSpCap) {
    // staged in chunks of kSlotCap slots: every thread's loads of a chunk in
    // flight at once (the CTA-pair scan's two slots per segment take V past
    // one chunk at C3: 128 probes x ~4 slots)
    for (uint32_t p = threadIdx.x; p < nprobe; p += blockDim.x)
      for (uint32_t t = 0; t < pns[p]; ++t) sp[soff[p] + t] = p * ix.s_max + t;  // p*s_max+s
    __syncthreads();
    auto stage = [&](uint32_t v0, uint32_t nv) {
      for (uint32_t v = threadIdx.x; v < nv; v += blockDim.x) {
        sn[v] = cand_n[slot0 + sp[v0 + v]];
        sthr[v] = cand_thr[slot0 + sp[v0 + v]];
      }
      // 8 independent loads per thread in flight before the stores (one load
      // per iteration left every thread waiting out the full latency each time)
      const uint32_t tot = nv * kKP;
      for (uint32_t i0 = threadIdx.x; i0 < tot; i0 += 8 * blockDim.x) {
        float t[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t idx = i0 + u * blockDim.x;
          t[u] = idx < tot ? __ldg(cand_d + (slot0 + sp[v0 + idx / kKP]) * kKP + (idx % kKP)) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const uint32_t idx = i0 + u * blockDim.x;
          if (idx < tot) sdv[idx] = t[u];
        }
      }
      __syncthreads();
    };
    // 1. tau = k-th smallest upper bound
    float cur = kInf;
    for (uint32_t v0 = 0; v0 < V; v0 += kSlotCap) {
      const uint32_t nv = min(kSlotCap, V - v0);
      stage(v0, nv);
      for (uint32_t v = warp; v < nv; v += NW) {
        const float E = pE[sp[v0 + v] / ix.s_max];
        cur = warp_merge32(cur, lane < (int)sn[v] ? __fadd_ru(sdv[v * kKP + lane], E) : kInf);
      }
      __syncthreads();
    }
    wl[warp][lane] = cur;
    __syncthreads();
    if (warp == 0) {
      float x = wl[0][lane];
      for (int w = 1; w < NW; ++w) x = warp_merge32(x, wl[w][lane]);
      const float t = __shfl_sync(FULL, x, (int)min(k, 32u) - 1);
      if (lane == 0) s_tau = t;
    }
    __syncthreads();
    const float tau = s_tau;
    // 2. candidates + completeness (one chunk: still staged from pass 1)
    for (uint32_t v0 = 0; v0 < V; v0 += kSlotCap) {
      const uint32_t nv = min(kSlotCap, V - v0);
      if (V > kSlotCap) stage(v0, nv);
      for (uint32_t v = warp; v < nv; v += NW) {
        const uint32_t sv = sp[v0 + v];
        const uint32_t p = sv / ix.s_max;
        const float E = pE[p];
        const bool take = lane < (int)sn[v] && __fsub_rd(sdv[v * kKP + lane], E) <= tau;
        const unsigned msk = __ballot_sync(FULL, take);
        uint32_t base = 0;
        if (lane == 0 && msk) base = atomicAdd(&s_cnt, (uint32_t)__popc(msk));
        base = __shfl_sync(FULL, base, 0);
        if (take) {
          const uint32_t pos = base + __popc(msk & ((1u << lane) - 1));
          if (pos < kCandMax) {
            crow[pos] = cand_row[(slot0 + sv) * kKP + lane];
            clist[pos] = pc[p];
          }
        }
        if (lane == 0 && __fsub_rd(sthr[v], E) <= tau) {
          s_bad = 1;
          const uint32_t f = atomicAdd(&s_nfail, 1u);
          if (f < kRepMax) s_fail[f] = sv;
        }
      }
      __syncthreads();
    }
  } else {
    // more segments than fit in smem: read the scan's outputs from global
    const uint32_t T = nprobe * ix.s_max;
    float cur = kInf;
    for (uint32_t t = warp; t < T; t += NW) {
      if ((t % ix.s_max) >= pns[t / ix.s_max]) continue;
      const uint32_t n = cand_n[slot0 + t];
      const float v = lane < (int)n ? __fadd_ru(cand_d[(slot0 + t) * kKP + lane], pE[t / ix.s_max]) : kInf;
      cur = warp_merge32(cur, v);
    }
    wl[warp][lane] = cur;
    __syncthreads();
    if (warp == 0) {
      float x = wl[0][lane];
      for (int w = 1; w < NW; ++w) x = warp_merge32(x, wl[w][lane]);
      const float t = __shfl_sync(FULL, x, (int)min(k, 32u) - 1);
      if (lane == 0) s_tau = t;
    }
    __syncthreads();
    const float tau = s_tau;
    for (uint32_t t = warp; t < T; t += NW) {
      const uint32_t p = t / ix.s_max;
      if ((t % ix.s_max) >= pns[p]) continue;
      const float E = pE[p];
      const uint64_t slot = slot0 + t;
      const uint32_t n = cand_n[slot];
      const bool take = lane < (int)n && __fsub_rd(cand_d[slot * kKP + lane], E) <= tau;
      const unsigned msk = __ballot_sync(FULL, take);
      uint32_t base = 0;
      if (lane == 0 && msk) base = atomicAdd(&s_cnt, (uint32_t)__popc(msk));
      base = __shfl_sync(FULL, base, 0);
      if (take) {
        const uint32_t pos = base + __popc(msk & ((1u << lane) - 1));
        if (pos < kCandMax) {
          crow[pos] = cand_row[slot * kKP + lane];
          clist[pos] = pc[p];
        }
      }
      if (lane == 0 && __fsub_rd(cand_thr[slot], E) <= tau) {
        s_bad = 1;
        const uint32_t f = atomicAdd(&s_nfail, 1u);
        if (f < kRepMax) s_fail[f] = t;
      }
    }
  }
  __syncthreads();
  const uint32_t m = s_cnt;
  const float tau = s_tau;
  // tau bounds the true k-th distance from above even when the completeness
  // proof fails: the exact fallback re-filters every row against it
  if (threadIdx.x == 0 && tau_out) tau_out[b] = tau;
  const bool tau_ok = tau < kInf && tau >= -FLT_MAX;
  if (s_bad && rep.entries && m <= kCandMax && tau_ok && s_nfail <= kRepMax) {
    // proof failed on a few segments only: queue them for the in-place repair
    // (every row of the segment re-filtered against tau, k_repair_segments)
    for (uint32_t f = threadIdx.x; f < s_nfail; f += blockDim.x) {
      const uint32_t e = atomicAdd(rep.n, 1u);
      if (e < rep.cap) rep.entries[e] = ((uint64_t)b << 32) | s_fail[f];
      else flags[b] = 1;  // repair list full: whole-query exact fallback
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (flags[b] != 1) flags[b] = 2;
      rep.cnt[b] = 0;
    }
    return;
  }
  if (s_bad || m > kCandMax || !tau_ok && s_total >= k) {
    if (threadIdx.x == 0) flags[b] = 1;
    return;
  }
  // 3. exact distances: one candidate per thread, loads pipelined ahead of the chain
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
  const uint32_t cnt = (uint32_t)min((unsigned long long)k, s_total);
  if (m <= blockDim.x) {
    // rank placement (doc ids of distinct rows are distinct, so ranks are):
    // one barrier instead of the bitonic network's log^2 barriers
    __syncthreads();
    if (threadIdx.x < m) {
      const double di = cdist[threadIdx.x];
      const uint64_t ii = cid[threadIdx.x];
      uint32_t r = 0;
      for (uint32_t j = 0; j < m; ++j) r += pair_less(cdist[j], cid[j], di, ii) ? 1u : 0u;
      if (r < cnt) {
        ids_out[(uint64_t)b * k + r] = ii;
        d_out[(uint64_t)b * k + r] = di;
      }
    }
    for (uint32_t i = cnt + threadIdx.x; i < k; i += blockDim.x) {
      ids_out[(uint64_t)b * k + i] = 0;
      d_out[(uint64_t)b * k + i] = 0.0;
    }
  } else {
    uint32_t mp = 1;
    while (mp < m) mp <<= 1;
    for (uint32_t i = m + threadIdx.x; i < mp; i += blockDim.x) {
      cdist[i] = DBL_MAX;
      cid[i] = ~0ull;
    }
    block_sort_pairs(cdist, cid, mp);
    for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
      ids_out[(uint64_t)b * k + i] = i < cnt ? cid[i] : 0;
      d_out[(uint64_t)b * k + i] = i < cnt ? cdist[i] : 0.0;
    }
  }
  if (threadIdx.x == 0) {
    counts_out[b] = cnt;
    flags[b] = 0;
  }
}

// ---- in-place repair of failing segments ---------------------------------------
// A query whose completeness proof failed on a few (plan position, segment)
// slots only: every row of those segments is re-tested with the FFMA filter
// (d^ - E_ffma > tau cannot be in the top-k; tau = finalize's upper bound on the
// true k-th distance) and the survivors get the exact double.  Work units are
// (entry, 256-row chunk) over the whole GPU, so one long segment does not
// serialise on one SM.
__global__ void __launch_bounds__(256) k_repair_segments(IndexView ix, QueryView qv,
                                                         const uint32_t* __restrict__ plans,
                                                         uint32_t nprobe, RepairState R,
                                                         const float* __restrict__ tau, double fa,
                                                         double fb, double fc, int* flags) {
  pdl_wait();
  const uint32_t chunks = (ix.seg_rows + kRepChunk - 1) / kRepChunk;
  const uint32_t n_units = min(*R.n, R.cap) * chunks;
  for (uint32_t u = blockIdx.x; u < n_units; u += gridDim.x) {
    const uint64_t e = R.entries[u / chunks];
    const uint32_t ch = u % chunks;
    const uint32_t b = (uint32_t)(e >> 32), t = (uint32_t)e;
    const uint32_t p = t / ix.s_max, sg = t % ix.s_max;
    const uint32_t c = plans[(uint64_t)b * nprobe + p];
    const uint64_t beg = ix.list_off[c], n_c = ix.list_off[c + 1] - beg;
    const uint64_t s0 = (uint64_t)(sg / ix.seg_split) * ix.seg_rows;
    if (s0 + (uint64_t)ch * kRepChunk * ix.seg_split >= n_c) continue;  // chunk past the list
    const uint64_t lr = slot_row(ix, sg, n_c, (uint64_t)ch * kRepChunk + threadIdx.x);
    const float tq = tau[b];
    const float* qs = qv.qs + (uint64_t)b * ix.dpad;
    double E;
    {
      const double q = qv.qnorm[b], x = ix.maxnorm[c];
      E = fa * q * x + fb * (q * q + x * x) + fc;
    }
    if (lr == ~0ull) continue;
    const float* lb = list_base(ix, c, beg);
    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 16
    for (uint32_t g = 0; g < ix.dpad / 4; ++g) {
      const float4 x = __ldg(reinterpret_cast<const float4*>(lb + swz_offset(0, n_c, lr, g * 4, ix.dpad)));
      const float4 q4 = __ldg(reinterpret_cast<const float4*>(qs + g * 4));
      a0 = __fmaf_rn(x.x, q4.x, a0);
      a1 = __fmaf_rn(x.y, q4.y, a1);
      a2 = __fmaf_rn(x.z, q4.z, a2);
      a3 = __fmaf_rn(x.w, q4.w, a3);
    }
    const float dot = __fadd_rn(__fadd_rn(a0, a1), __fadd_rn(a2, a3));
    const float dh = __fmaf_rn(-2.f, dot, __fadd_rn(ix.xnorm2[beg + lr], qv.qn2[b]));
    if (__fsub_rd(dh, __double2float_ru(E)) > tq) continue;  // NaN keeps the row
    const double d = exact_row_pipelined(ix.dim, qs, [&](uint32_t g) {
      return __ldg(reinterpret_cast<const float4*>(lb + swz_offset(0, n_c, lr, g * 4, ix.dpad)));
    });
    const uint32_t pos = atomicAdd(&R.cnt[b], 1u);
    if (pos < R.per_query) {
      R.d[(uint64_t)b * R.per_query + pos] = d;
      R.ids[(uint64_t)b * R.per_query + pos] = ix.ids[beg + lr];
    } else {
      flags[b] = 1;  // too many survivors: whole-query exact fallback
    }
  }
}

// Repaired queries (flag 2): candidates of the slots that passed the proof
// (recomputed with the same tau, so the same slots) + the repaired segments'
// exact survivors -> (d, id) sort -> top-k.
__global__ void __launch_bounds__(kFinThreads) k_finalize_repair(
    IndexView ix, QueryView qv, const uint32_t* __restrict__ plans, uint32_t nprobe, uint32_t k,
    const float* __restrict__ cand_d, const uint32_t* __restrict__ cand_row,
    const float* __restrict__ cand_thr, const uint32_t* __restrict__ cand_n,
    const float* __restrict__ tau, RepairState R, uint64_t* __restrict__ ids_out,
    double* __restrict__ d_out, uint32_t* __restrict__ counts_out, int* flags) {
  pdl_wait();
  const uint32_t b = blockIdx.x;
  if (flags[b] != 2) return;
  extern __shared__ __align__(16) uint8_t sm[];
  constexpr uint32_t kCap = 2 * kCandMax;
  double* cdist = reinterpret_cast<double*>(sm);               // kCap
  uint64_t* cid = reinterpret_cast<uint64_t*>(cdist + kCap);    // kCap
  uint32_t* crow = reinterpret_cast<uint32_t*>(cid + kCap);     // kCandMax
  uint32_t* clist = crow + kCandMax;                            // kCandMax
  float* qsh = reinterpret_cast<float*>(clist + kCandMax);      // dpad
  __shared__ uint32_t s_cnt;
  __shared__ int s_over;
  __shared__ unsigned long long s_total;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NW = kFinThreads / 32;
  for (uint32_t d = threadIdx.x; d < ix.dpad; d += blockDim.x) qsh[d] = qv.qs[(uint64_t)b * ix.dpad + d];
  if (threadIdx.x == 0) {
    s_cnt = 0;
    s_over = 0;
    s_total = 0;
  }
  __syncthreads();
  const float tq = tau[b], qn = qv.qnorm[b];
  const uint64_t slot0 = (uint64_t)b * nprobe * ix.s_max;
  for (uint32_t p = warp; p < nprobe; p += NW) {
    const uint32_t c = plans[(uint64_t)b * nprobe + p];
    const uint64_t rows = ix.list_off[c + 1] - ix.list_off[c];
    if (lane == 0) atomicAdd(&s_total, (unsigned long long)rows);
    const uint32_t ns = slots_of(ix, rows);
    const float E = seg_bound(ix, qn, ix.maxnorm[c]);
    for (uint32_t sg = 0; sg < ns; ++sg) {
      const uint64_t slot = slot0 + (uint64_t)p * ix.s_max + sg;
      if (__fsub_rd(cand_thr[slot], E) <= tq) continue;  // repaired segment
      const uint32_t n = cand_n[slot];
      const bool take = lane < (int)n && __fsub_rd(cand_d[slot * kKP + lane], E) <= tq;
      const unsigned msk = __ballot_sync(FULL, take);
      uint32_t base = 0;
      if (lane == 0 && msk) base = atomicAdd(&s_cnt, (uint32_t)__popc(msk));
      base = __shfl_sync(FULL, base, 0);
      if (take) {
        const uint32_t pos = base + __popc(msk & ((1u << lane) - 1));
        if (pos < kCandMax) {
          crow[pos] = cand_row[slot * kKP + lane];
          clist[pos] = c;
        } else {
          s_over = 1;
        }
      }
    }
  }
  __syncthreads();
  const uint32_t m = min(s_cnt, (uint32_t)kCandMax);
  const uint32_t r = min(R.cnt[b], R.per_query);
  if (s_over || m + r > kCap) {
    if (threadIdx.x == 0) flags[b] = 1;
    return;
  }
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
  for (uint32_t i = threadIdx.x; i < r; i += blockDim.x) {
    cdist[m + i] = R.d[(uint64_t)b * R.per_query + i];
    cid[m + i] = R.ids[(uint64_t)b * R.per_query + i];
  }
  uint32_t mp = 1;
  while (mp < m + r) mp <<= 1;
  for (uint32_t i = m + r + threadIdx.x; i < mp; i += blockDim.x) {
    cdist[i] = DBL_MAX;
    cid[i] = ~0ull;
  }
  block_sort_pairs(cdist, cid, mp);
  const uint32_t cnt = (uint32_t)min((unsigned long long)k, s_total);
  for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
    ids_out[(uint64_t)b * k + i] = i < cnt ? cid[i] : 0;
    d_out[(uint64_t)b * k + i] = i < cnt ? cdist[i] : 0.0;
  }
  if (threadIdx.x == 0) {
    counts_out[b] = cnt;
    flags[b] = 0;
  }
}

// Exact streaming top-k (the reference algorithm on the GPU: every row of the
// plan, exact distance, (d, id) order) for flagged queries and k > 32.
// Grid (query, part): part y covers plan positions [y*per, (y+1)*per); with
// more than one part each CTA writes its exact partial top-k and
// k_exact_merge combines them (lists are disjoint, so the merge is exact).
// Buffer of `cap` (d, id) pairs filtered by the running k-th.
// With `tau` (finalize's upper bound on the query's true k-th distance), a
// row whose FFMA filter distance d^ satisfies d^ - E > tau (E: the FFMA bound of
// scan.cu, any summation order) cannot be in the top-k and skips the fp64 chain.
__global__ void __launch_bounds__(256) k_exact_search(IndexView ix, QueryView qv,
                                                      const uint32_t* __restrict__ plans,
                                                      uint32_t nprobe, uint32_t k, uint32_t cap,
                                                      const int* flags, uint64_t* ids_out,
                                                      double* d_out, uint32_t* counts_out,
                                                      uint64_t* part_total, const float* tau,
                                                      double fa, double fb, double fc) {
  pdl_wait();
  // grid-stride over queries: the grid is sized for ~one wave, so a batch
  // with no flagged query costs a few hundred idle CTAs, not B x nsplit; each
  // CTA checks the flags of its next blockDim.x queries at once and works
  // through the flagged ones
  __shared__ uint32_t s_list[256];
  __shared__ uint32_t s_nl;
  for (uint64_t base = blockIdx.x; base < qv.n; base += (uint64_t)gridDim.x * blockDim.x) {
  __syncthreads();  // the previous chunk's list is consumed
  if (threadIdx.x == 0) s_nl = 0;
  __syncthreads();
  {
    const uint64_t bb = base + (uint64_t)threadIdx.x * gridDim.x;
    if (bb < qv.n && (!flags || flags[bb])) s_list[atomicAdd(&s_nl, 1u)] = (uint32_t)bb;
  }
  __syncthreads();
  const uint32_t nl = s_nl;
  for (uint32_t li = 0; li < nl; ++li) {
  const uint32_t b = s_list[li];
  const uint32_t nsplit = gridDim.y, y = blockIdx.y;
  const uint32_t per = (nprobe + nsplit - 1) / nsplit;
  const uint32_t p_beg = min(nprobe, y * per), p_end = min(nprobe, p_beg + per);
  const uint64_t out_row = nsplit > 1 ? (uint64_t)b * nsplit + y : b;
  extern __shared__ __align__(16) uint8_t sm[];
  double* bd = reinterpret_cast<double*>(sm);
  uint64_t* bi = reinterpret_cast<uint64_t*>(bd + cap);
  float* qsh = reinterpret_cast<float*>(bi + cap);
  __shared__ uint32_t s_cnt;
  __shared__ double s_thr_d;
  __shared__ uint64_t s_thr_i;
  __shared__ unsigned long long s_total;
  for (uint32_t d = threadIdx.x; d < ix.dpad; d += blockDim.x) qsh[d] = qv.qs[(uint64_t)b * ix.dpad + d];
  if (threadIdx.x == 0) {
    s_cnt = 0;
    s_thr_d = DBL_MAX;
    s_thr_i = ~0ull;
    s_total = 0;
  }
  __syncthreads();
  const float tq = tau ? tau[b] : __int_as_float(0x7f800000);
  const bool filt = tq < __int_as_float(0x7f800000) && tq >= -FLT_MAX;
  const float qn = qv.qnorm[b], qn2 = qv.qn2[b];
  for (uint32_t p = p_beg; p < p_end; ++p) {
    const uint32_t c = plans[(uint64_t)b * nprobe + p];
    const uint64_t beg = ix.list_off[c], end = ix.list_off[c + 1];
    if (threadIdx.x == 0) s_total += end - beg;
    float E = 0.f;
    if (filt) {
      const double q = qn, x = ix.maxnorm[c];
      E = __double2float_ru(fa * q * x + fb * (q * q + x * x) + fc);
    }
    for (uint64_t r0 = beg; r0 < end; r0 += blockDim.x) {
      const uint64_t r = r0 + threadIdx.x;
      double dist = DBL_MAX;
      uint64_t id = ~0ull;
      if (r < end) {
        const uint64_t n_c = end - beg, lr = r - beg;
        const float* lb = list_base(ix, c, beg);
        bool need = true;
        if (filt) {
          float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll 16
          for (uint32_t g = 0; g < ix.dpad / 4; ++g) {
            const float4 x = __ldg(reinterpret_cast<const float4*>(lb + swz_offset(0, n_c, lr, g * 4, ix.dpad)));
            const float4 q4 = *reinterpret_cast<const float4*>(qsh + g * 4);
            a0 = __fmaf_rn(x.x, q4.x, a0);
            a1 = __fmaf_rn(x.y, q4.y, a1);
            a2 = __fmaf_rn(x.z, q4.z, a2);
            a3 = __fmaf_rn(x.w, q4.w, a3);
          }
          const float dot = __fadd_rn(__fadd_rn(a0, a1), __fadd_rn(a2, a3));
          const float dh = __fmaf_rn(-2.f, dot, __fadd_rn(ix.xnorm2[r], qn2));
          need = !(__fsub_rd(dh, E) > tq);  // NaN keeps the row (exact path decides)
        }
        if (need) {
          dist = exact_row_pipelined(ix.dim, qsh, [&](uint32_t g) {
            return __ldg(reinterpret_cast<const float4*>(lb + swz_offset(0, n_c, lr, g * 4, ix.dpad)));
          });
          id = ix.ids[r];
        }
      }
      const uint32_t cnt_now = s_cnt;
      __syncthreads();  // every thread has read s_cnt before any append
      if (cnt_now + blockDim.x > cap) {
        for (uint32_t i = s_cnt + threadIdx.x; i < cap; i += blockDim.x) {
          bd[i] = DBL_MAX;
          bi[i] = ~0ull;
        }
        block_sort_pairs(bd, bi, cap);
        if (threadIdx.x == 0) {
          s_cnt = k;
          s_thr_d = bd[k - 1];
          s_thr_i = bi[k - 1];
        }
        __syncthreads();
      }
      if (r < end && pair_less(dist, id, s_thr_d, s_thr_i)) {
        const uint32_t pos = atomicAdd(&s_cnt, 1u);
        bd[pos] = dist;
        bi[pos] = id;
      }
      __syncthreads();
    }
  }
  for (uint32_t i = s_cnt + threadIdx.x; i < cap; i += blockDim.x) {
    bd[i] = DBL_MAX;
    bi[i] = ~0ull;
  }
  block_sort_pairs(bd, bi, cap);
  const uint32_t cnt = (uint32_t)min((unsigned long long)k, s_total);
  for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
    ids_out[out_row * k + i] = i < cnt ? bi[i] : 0;
    d_out[out_row * k + i] = i < cnt ? bd[i] : 0.0;
  }
  if (threadIdx.x == 0) {
    counts_out[out_row] = cnt;
    if (part_total) part_total[out_row] = s_total;
  }
  __syncthreads();  // shared state is re-initialised by the next query
  }
  }
}

// Combine the exact partial top-k lists of k_exact_search (nsplit parts).
__global__ void __launch_bounds__(256) k_exact_merge(uint32_t nsplit, uint32_t k, uint32_t cap,
                                                     const int* flags, const uint64_t* part_ids,
                                                     const double* part_d,
                                                     const uint32_t* part_cnt,
                                                     const uint64_t* part_total,
                                                     uint64_t* ids_out, double* d_out,
                                                     uint32_t* counts_out) {
  pdl_wait();
  const uint32_t b = blockIdx.x;
  if (flags && !flags[b]) return;
  extern __shared__ __align__(16) uint8_t sm[];
  double* bd = reinterpret_cast<double*>(sm);
  uint64_t* bi = reinterpret_cast<uint64_t*>(bd + cap);
  __shared__ unsigned long long s_total;
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (uint32_t y = 0; y < nsplit; ++y) t += part_total[(uint64_t)b * nsplit + y];
    s_total = t;
  }
  for (uint32_t i = threadIdx.x; i < cap; i += blockDim.x) {
    const uint32_t y = i / k, e = i % k;
    const uint64_t row = (uint64_t)b * nsplit + y;
    const bool ok = y < nsplit && e < part_cnt[row];
    bd[i] = ok ? part_d[row * k + e] : DBL_MAX;
    bi[i] = ok ? part_ids[row * k + e] : ~0ull;
  }
  block_sort_pairs(bd, bi, cap);
  const uint32_t cnt = (uint32_t)min((unsigned long long)k, s_total);
  for (uint32_t i = threadIdx.x; i < k; i += blockDim.x) {
    ids_out[(uint64_t)b * k + i] = i < cnt ? bi[i] : 0;
    d_out[(uint64_t)b * k + i] = i < cnt ? bd[i] : 0.0;
  }
  if (threadIdx.x == 0) counts_out[b] = cnt;
}

// (query, list) pairs of the plans.  Caller-supplied plans (planned search)
// are validated: an id >= K is replaced by 0 in the working copy and flags err.
__global__ void k_plans_to_pairs(const uint32_t* plans, uint32_t n, uint32_t nprobe, uint32_t K,
                                 uint32_t* pq, uint32_t* pl, uint32_t* plans_out, int* err) {
  pdl_wait();
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n * nprobe) return;
  uint32_t c = plans[p];
  if (c >= K) {
    c = 0;
    if (err) atomicOr(err, 2);
  }
  pq[p] = p / nprobe;
  pl[p] = c;
  if (plans_out) plans_out[p] = c;
}

// merge_topk (vector_index.cpp:71-91) over n_parts exact per-shard lists.
// Part p's arrays start at ids + p*s_ids, d + p*s_d, counts + p*s_cnt (an
// all-gather of separate arrays, or of one packed ids|dists|counts block per rank).
__global__ void k_merge_parts(uint32_t n_parts, uint32_t nq, uint32_t k, const uint64_t* ids,
                              const double* d, const uint32_t* counts, uint64_t* ids_out,
                              double* d_out, uint32_t* counts_out, uint32_t cap, uint64_t s_ids,
                              uint64_t s_d, uint64_t s_cnt) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t sm[];
  double* bd = reinterpret_cast<double*>(sm);
  uint64_t* bi = reinterpret_cast<uint64_t*>(bd + cap);
  const uint32_t b = blockIdx.x;
  for (uint32_t i = threadIdx.x; i < cap; i += blockDim.x) {
    const uint32_t part = i / k, e = i % k;
    bool ok = part < n_parts && e < counts[(uint64_t)part * s_cnt + b];
    bd[i] = ok ? d[(uint64_t)part * s_d + (uint64_t)b * k + e] : DBL_MAX;
    bi[i] = ok ? ids[(uint64_t)part * s_ids + (uint64_t)b * k + e] : ~0ull;
  }
  block_sort_pairs(bd, bi, cap);
  // collapse duplicate ids to the minimum distance: after the (d, id) sort the
  // first occurrence of an id is its minimum; drop later ones.
  __shared__ uint32_t s_n;
  if (threadIdx.x == 0) {
    uint32_t n = 0;
    for (uint32_t i = 0; i < cap && n < k; ++i) {
      if (bi[i] == ~0ull && bd[i] == DBL_MAX) break;
      bool dup = false;
      for (uint32_t j = 0; j < n; ++j)
        if (ids_out[(uint64_t)b * k + j] == bi[i]) dup = true;
      if (dup) continue;
      ids_out[(uint64_t)b * k + n] = bi[i];
      d_out[(uint64_t)b * k + n] = bd[i];
      ++n;
    }
    for (uint32_t j = n; j < k; ++j) {
      ids_out[(uint64_t)b * k + j] = 0;
      d_out[(uint64_t)b * k + j] = 0.0;
    }
    s_n = n;
    counts_out[b] = n;
  }
}

}  // namespace

void launch_plans_to_pairs(const uint32_t* plans, uint32_t n_queries, uint32_t nprobe, uint32_t K,
                           uint32_t* pair_query, uint32_t* pair_list, uint32_t* plans_out, int* err,
                           cudaStream_t s) {
  const uint32_t n = n_queries * nprobe;
  if (!n) return;
  launch_pdl(k_plans_to_pairs, dim3((n + 255) / 256), dim3(256), 0, s, plans, n_queries, nprobe, K, pair_query, pair_list,
                                                    plans_out, err);
}

void launch_finalize_search(const IndexView& ix, const QueryView& qv, const uint32_t* plans,
                            uint32_t nprobe, uint32_t k, const float* cand_d,
                            const uint32_t* cand_row, const float* cand_thr,
                            const uint32_t* cand_n, uint64_t* ids_out, double* d_out,
                            uint32_t* counts_out, int* flags, float* tau_out,
                            const RepairState* rep, cudaStream_t s) {
  const RepairState R = rep ? *rep : RepairState{};
  const size_t smem = (size_t)kCandMax * (8 + 8 + 4 + 4) + (size_t)ix.dpad * 8 + (size_t)nprobe * 16 + 4 +
                      (size_t)kSpCap * 4 + (size_t)kSlotCap * (4 + 4 + kKP * 4);
  smem_optin((const void*)k_finalize_search, 200 * 1024);
  launch_pdl(k_finalize_search, dim3(qv.n), dim3(kFinThreads), smem, s, ix, qv, plans, nprobe, k, cand_d, cand_row,
                                                    cand_thr, cand_n, filter_eps(ix.dim),
                                                    filter_abs(ix.dim), ids_out, d_out,
                                                    counts_out, flags, tau_out, R);
}

uint32_t exact_search_parts(uint32_t nprobe, uint32_t k) {
  uint32_t ns = nprobe < 64 ? nprobe : 64;
  while (ns > 1 && (uint64_t)ns * k > 8192) ns >>= 1;
  return ns ? ns : 1;
}

namespace {
// Seed of the shared drop bound: per query, the
// exact double distance (the reference's sequential arithmetic, exact_step) of
// the first `rows` rows of its nearest probed list with at least that many
// rows (first 4 plan positions); the k-th smallest, rounded up, is an upper
// bound on the query's true k-th distance over its probes (k distinct probed
// rows), so the scan can drop rows from its first tile on instead of after the
// query's first finished item.  One CTA (64 threads, one row each) per query.
__global__ void __launch_bounds__(64) k_seed_bounds(IndexView ix, QueryView qv, const uint32_t* __restrict__ plans,
                                                    uint32_t nprobe, uint32_t k, uint32_t rows,
                                                    float* __restrict__ qbound) {
  pdl_wait();
  const uint32_t b = blockIdx.x, t = threadIdx.x;
  __shared__ double sd[64];
  uint32_t c = ~0u;
  uint64_t lbeg = 0, n_c = 0;
  for (uint32_t p = 0; p < nprobe && p < 4; ++p) {
    const uint32_t cc = plans[(uint64_t)b * nprobe + p];
    if (cc >= ix.K) continue;
    const uint64_t lb = ix.list_off[cc], n = ix.list_off[cc + 1] - lb;
    if (n >= rows) {
      c = cc;
      lbeg = lb;
      n_c = n;
      break;
    }
  }
  if (c == ~0u) return;  // uniform: no list with enough rows, no seed
  const float* q = qv.qs + (uint64_t)b * ix.dpad;
  const float* base = list_base(ix, c, lbeg);
  double acc = __longlong_as_double(0x7ff0000000000000ll);
  if (t < rows) {
    // 16-B loads of the row's swizzled granules, double-buffered ahead of the
    // sequential chain ((x - q)^2 == (q - x)^2 exactly: the reference's
    // squared_l2 operand order does not matter)
    acc = exact_row_pipelined(ix.dim, q, [&](uint32_t g) {
      return __ldg(reinterpret_cast<const float4*>(base + swz_offset(0, n_c, t, g * 4, ix.dpad)));
    });
  }
  sd[t] = acc;
  __syncthreads();
  if (t == 0) {  // k-th smallest of <= 64 values
    double kth = 0.0;
    for (uint32_t j = 0; j < rows; ++j) {
      uint32_t below = 0;
      for (uint32_t i = 0; i < rows; ++i) below += sd[i] < sd[j] || (sd[i] == sd[j] && i < j);
      if (below == k - 1) kth = sd[j];
    }
    const float u = __double2float_ru(kth);
    if (u < 3.0e38f) atomicMin(reinterpret_cast<int*>(qbound + b), __float_as_int(u));
  }
}
}  // namespace

void launch_seed_bounds(const IndexView& ix, const QueryView& qv, const uint32_t* plans, uint32_t nprobe,
                        uint32_t k, uint32_t rows, float* qbound, cudaStream_t s) {
  if (!qv.n || rows < k || rows > 64) return;
  launch_pdl(k_seed_bounds, dim3(qv.n), dim3(64), 0, s, ix, qv, plans, nprobe, k, rows, qbound);
}

void launch_exact_search(const IndexView& ix, const QueryView& qv, const uint32_t* plans,
                         uint32_t nprobe, uint32_t k, const int* flags, uint64_t* ids_out,
                         double* d_out, uint32_t* counts_out, uint64_t* part_ids,
                         double* part_d, uint32_t* part_cnt, uint64_t* part_total,
                         const float* tau, cudaStream_t s) {
  double fa = 0, fb = 0, fc = 0;
  bound_ffma(ix.dim, &fa, &fb, &fc);
  uint32_t cap = 512;
  while (cap < k + 256) cap <<= 1;
  const size_t smem = (size_t)cap * 16 + (size_t)ix.dpad * 4;
  smem_optin((const void*)k_exact_search, 200 * 1024);
  smem_optin((const void*)k_exact_merge, 200 * 1024);
  const uint32_t ns = part_ids ? exact_search_parts(nprobe, k) : 1;
  const int sms = device_sm_count();
  // grid-strided over the queries: a full wave at the kernel's occupancy (an
  // exact-only search sends every query here; the flagged fallback few)
  static thread_local int occ_dev = -1, occ = 0;
  static thread_local size_t occ_smem = 0;
  if (occ_dev != current_device() || occ_smem != smem) {
    occ = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_exact_search, 256, smem);
    occ_dev = current_device();
    occ_smem = smem;
  }
  const uint32_t wave = (uint32_t)std::max(1, occ) * (uint32_t)sms;
  const uint32_t gx = std::max(1u, std::min(qv.n, wave / ns));
  if (ns <= 1) {
    launch_pdl(k_exact_search, dim3(dim3(gx, 1)), dim3(256), smem, s, ix, qv, plans, nprobe, k, cap, flags, ids_out,
                                                    d_out, counts_out, nullptr, tau, fa, fb, fc);
    return;
  }
  launch_pdl(k_exact_search, dim3(dim3(gx, ns)), dim3(256), smem, s, ix, qv, plans, nprobe, k, cap, flags, part_ids,
                                                   part_d, part_cnt, part_total, tau, fa, fb, fc);
  uint32_t mcap = 1;
  while (mcap < ns * k) mcap <<= 1;
  launch_pdl(k_exact_merge, dim3(qv.n), dim3(256), (size_t)mcap * 16, s, ns, k, mcap, flags, part_ids, part_d,
                                                     part_cnt, part_total, ids_out, d_out,
                                                     counts_out);
}

void launch_merge_parts(uint32_t n_parts, uint32_t n_queries, uint32_t k, const uint64_t* ids,
                        const double* d, const uint32_t* counts, uint64_t* ids_out,
                        double* d_out, uint32_t* counts_out, cudaStream_t s) {
  uint32_t cap = 1;
  while (cap < n_parts * k) cap <<= 1;
  const size_t smem = (size_t)cap * 16;
  smem_optin((const void*)k_merge_parts, 200 * 1024);
  launch_pdl(k_merge_parts, dim3(n_queries), dim3(256), smem, s, n_parts, n_queries, k, ids, d, counts, ids_out, d_out,
                                             counts_out, cap, (uint64_t)n_queries * k,
                                             (uint64_t)n_queries * k, n_queries);
}

void launch_merge_parts_strided(uint32_t n_parts, uint32_t n_queries, uint32_t k, const uint64_t* ids,
                                const double* d, const uint32_t* counts, uint64_t s_ids, uint64_t s_d,
                                uint64_t s_cnt, uint64_t* ids_out, double* d_out, uint32_t* counts_out,
                                cudaStream_t s) {
  uint32_t cap = 1;
  while (cap < n_parts * k) cap <<= 1;
  smem_optin((const void*)k_merge_parts, 200 * 1024);
  launch_pdl(k_merge_parts, dim3(n_queries), dim3(256), (size_t)cap * 16, s, n_parts, n_queries, k, ids, d, counts, ids_out,
                                                         d_out, counts_out, cap, s_ids, s_d, s_cnt);
}

// Node-split sub-search finalize lives in items.cu.


void launch_repair(const IndexView& ix, const QueryView& qv, const uint32_t* plans, uint32_t nprobe,
                   uint32_t k, const float* cand_d, const uint32_t* cand_row, const float* cand_thr,
                   const uint32_t* cand_n, const float* tau, const RepairState& R, int n_ctas,
                   uint64_t* ids_out, double* d_out, uint32_t* counts_out, int* flags, cudaStream_t s) {
  double fa = 0, fb = 0, fc = 0;
  bound_ffma(ix.dim, &fa, &fb, &fc);
  launch_pdl(k_repair_segments, dim3(n_ctas), dim3(256), 0, s, ix, qv, plans, nprobe, R, tau, fa, fb, fc, flags);
  const size_t smem = (size_t)2 * kCandMax * 16 + (size_t)kCandMax * 8 + (size_t)ix.dpad * 4;
  smem_optin((const void*)k_finalize_repair, 200 * 1024);
  launch_pdl(k_finalize_repair, dim3(qv.n), dim3(kFinThreads), smem, s, ix, qv, plans, nprobe, k, cand_d, cand_row, cand_thr,
                                                    cand_n, tau, R, ids_out, d_out, counts_out, flags);
}

}  // namespace hivf
