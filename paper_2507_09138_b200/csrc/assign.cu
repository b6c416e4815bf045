// assign.cu -- K1: exact coarse assign (batched ivf::select_clusters).
//
// Reference: /root/reference/proj/src/vector_index.cpp:261-278 -- for every
// centroid the double distance of embedding.hpp:27-34, std::sort by
// (distance, cluster id), first nprobe.  Plan ORDER is API-visible (cursor
// plans, node-split slicing), so the output must equal the reference order
// bit for bit.
//
// B200 design: (1) fp32 expansion distances for all B x K pairs on FFMA (a
// small GEMM, 1.6 GFLOP at B=256/K=4096/D=768); (2) per query, the nprobe-th
// smallest *upper* bound tau (radix select); every centroid whose *lower*
// bound is <= tau is a candidate (provably a superset of the true top-nprobe);
// (3) candidates get the exact fp64 distance in the reference's sequential
// order and are sorted by (distance, id).  Degenerate inputs (more than
// kCandCap candidates) take an exact streaming path over all K.
#include <cfloat>
#include <cmath>

#include <cub/device/device_segmented_radix_sort.cuh>

#include "common.cuh"
#include "kernels.h"

namespace hivf {

namespace {

constexpr int kCandCap = 4096;

// Search-space queries: cosine normalization exactly as embedding.hpp:36-43
// (double norm, sequential, divide, cast back to float), then fp32 |q|^2 and
// an upper bound of |q| for the filter bound.
__global__ void k_prep_queries(const float* __restrict__ qin, uint32_t n, uint32_t dim,
                               uint32_t dpad, int metric, int normalize, float* __restrict__ qs,
                               float* __restrict__ qn2, float* __restrict__ qnorm, float* __restrict__ qsc,
                               int* err) {
  pdl_wait();
  const uint32_t b = blockIdx.x;
  if (b >= n) return;
  __shared__ double s_norm;
  __shared__ double s_part[4];
  const float* q = qin + (uint64_t)b * dim;
  const bool do_norm_metric = metric == 1 && normalize;
  if (do_norm_metric && threadIdx.x == 0) {
    // cosine: the reference's sequential double norm (embedding.hpp:36-43), exactly
    double nrm = 0.0;
    for (uint32_t d = 0; d < dim; ++d) {
      const double x = (double)q[d];
      nrm = __dadd_rn(nrm, __dmul_rn(x, x));
    }
    s_norm = __dsqrt_rn(nrm);
  }
  __syncthreads();
  const double nrm = do_norm_metric ? s_norm : 0.0;
  const bool do_norm = do_norm_metric && nrm != 0.0;
  double part = 0.0;  // |q|^2 for the filter bound only: any summation order is fine
  for (uint32_t d = threadIdx.x; d < dpad; d += blockDim.x) {
    float v = d < dim ? q[d] : 0.f;
    if (d < dim && !isfinite(v)) *err = 1;
    if (do_norm) v = __double2float_rn(__ddiv_rn((double)v, nrm));
    qs[(uint64_t)b * dpad + d] = v;
    part += (double)v * (double)v;
  }
  for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
  if ((threadIdx.x & 31) == 0) s_part[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (uint32_t w = 0; w < (blockDim.x + 31) / 32; ++w) acc += s_part[w];
    qn2[b] = __double2float_rn(acc);
    const float qb = __double2float_ru(sqrt(acc) * (1.0 + 1e-6));
    qnorm[b] = qb;
    const int e = h16_exp(qb);  // fp16 filter: q 2^e has every |element| < 2^15
    qsc[b] = (e < -kH16ExpMax || e > kH16ExpMax) ? 0.f : ldexpf(1.f, -e);
  }
}

// dist32[b][c] = fma(-2, <q_b, c>, |c|^2 + |q_b|^2); the dot accumulates in
// ascending dim order with one FMA per term (the order the error bound
// assumes).  Tile: CTC centroids x 32 queries, 4x4 per thread (CTC*2 threads);
// CTC shrinks (128 -> 64 -> 32) until the grid covers the SMs twice, so
// small-K / small-B batches (C1, C2) are not run on a fraction of the GPU.
constexpr int CT_Q = 32, CT_K = 16;

// kSplit: blockIdx.z takes dims [z * kspan, (z + 1) * kspan) and writes its
// partial dot product to out[z][q][c] (combined by k_coarse_combine): small
// batches on small codebooks (C2: 256 x 1024 centroids) fill the GPU through
// the reduction dimension.  The dot product is then a different summation
// tree of the same D terms, which filter_eps (gamma_D, any order) covers.
template <int CTC, bool kSplit = false>
__global__ void __launch_bounds__(CTC * 2) k_coarse_dist(IndexView ix, QueryView qv,
                                                         float* __restrict__ out, uint32_t kspan = 0) {
  pdl_wait();
  constexpr int NT = CTC * 2;  // threads
  constexpr int NA = CTC * CT_K / 4;  // float4 loads per A k-tile
  constexpr int NB = CT_Q * CT_K / 4;  // float4 loads per B k-tile
  __shared__ __align__(16) float As[CT_K][CTC + 4];
  __shared__ __align__(16) float Bs[CT_K][CT_Q + 4];
  const int tid = threadIdx.x;
  const int tc = tid % (CTC / 4);  // centroid group (4 centroids)
  const int tq = tid / (CTC / 4);  // query group (4 queries)
  const uint32_t c0 = blockIdx.x * CTC, q0 = blockIdx.y * CT_Q;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  // register-prefetched k-tiles: tile k0+CT_K is loaded from global while tile
  // k0 is multiplied out of shared memory
  constexpr int PA = NA / NT, PB = (NB + NT - 1) / NT;
  float4 pa[PA], pb[PB];
  auto fetch = [&](uint32_t k0) {
#pragma unroll
    for (int t = 0; t < PA; ++t) {
      const int f = tid + t * NT;
      const uint32_t c = c0 + (f >> 2);
      pa[t] = (c < ix.K && k0 < ix.dpad)
                  ? __ldg(reinterpret_cast<const float4*>(ix.cent + (uint64_t)c * ix.dpad + k0 + (f & 3) * 4))
                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int t = 0; t < PB; ++t) {
      const int f = tid + t * NT;
      const uint32_t q = q0 + (f >> 2);
      pb[t] = (f < NB && q < qv.n && k0 < ix.dpad)
                  ? __ldg(reinterpret_cast<const float4*>(qv.qs + (uint64_t)q * ix.dpad + k0 + (f & 3) * 4))
                  : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  const uint32_t kb = kSplit ? blockIdx.z * kspan : 0u;
  const uint32_t ke = kSplit ? min(ix.dpad, kb + kspan) : ix.dpad;
  fetch(kb);
  for (uint32_t k0 = kb; k0 < ke; k0 += CT_K) {
#pragma unroll
    for (int t = 0; t < PA; ++t) {
      const int f = tid + t * NT;
      const int row = f >> 2, g = f & 3;
      As[g * 4 + 0][row] = pa[t].x;
      As[g * 4 + 1][row] = pa[t].y;
      As[g * 4 + 2][row] = pa[t].z;
      As[g * 4 + 3][row] = pa[t].w;
    }
#pragma unroll
    for (int t = 0; t < PB; ++t) {
      const int f = tid + t * NT;
      if (f < NB) {
        const int row = f >> 2, g = f & 3;
        Bs[g * 4 + 0][row] = pb[t].x;
        Bs[g * 4 + 1][row] = pb[t].y;
        Bs[g * 4 + 2][row] = pb[t].z;
        Bs[g * 4 + 3][row] = pb[t].w;
      }
    }
    __syncthreads();
    if (k0 + CT_K < ke) fetch(k0 + CT_K);
#pragma unroll
    for (int kk = 0; kk < CT_K; ++kk) {
      const float4 a = *reinterpret_cast<const float4*>(&As[kk][tc * 4]);
      const float4 b = *reinterpret_cast<const float4*>(&Bs[kk][tq * 4]);
      const float av[4] = {a.x, a.y, a.z, a.w};
      const float bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const uint32_t q = q0 + tq * 4 + j;
    if (q >= qv.n) continue;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint32_t c = c0 + tc * 4 + i;
      if (c >= ix.K) continue;
      if (kSplit) {
        out[((uint64_t)blockIdx.z * qv.n + q) * ix.K + c] = acc[i][j];
      } else {
        const float s = __fadd_rn(ix.cnorm2[c], qv.qn2[q]);
        out[(uint64_t)q * ix.K + c] = __fmaf_rn(-2.f, acc[i][j], s);
      }
    }
  }
}

// Partial dot products (z = 0..S-1, summed in z order: deterministic) ->
// fp32 expansion distance, as the unsplit kernel forms it.
__global__ void k_coarse_combine(IndexView ix, QueryView qv, const float* __restrict__ part, uint32_t S,
                                 float* __restrict__ out) {
  pdl_wait();
  const uint64_t n = (uint64_t)qv.n * ix.K;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
    float dot = part[i];
    for (uint32_t z = 1; z < S; ++z) dot = __fadd_rn(dot, part[(uint64_t)z * n + i]);
    const uint32_t q = (uint32_t)(i / ix.K), c = (uint32_t)(i % ix.K);
    out[i] = __fmaf_rn(-2.f, dot, __fadd_rn(ix.cnorm2[c], qv.qn2[q]));
  }
}


// Block-wide radix select: the `want`-th smallest (1-based) of n keys
// produced by key_of(i).  512 threads.
template <typename KeyOf>
__device__ uint32_t block_radix_select(uint32_t n, uint32_t want, KeyOf key_of, uint32_t* hist) {
  uint32_t prefix = 0, mask = 0;
  for (int shift = 24; shift >= 0; shift -= 8) {
    for (int i = threadIdx.x; i < 256; i += blockDim.x) hist[i] = 0;
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < n; i += blockDim.x) {
      const uint32_t key = key_of(i);
      if ((key & mask) == prefix) atomicAdd(&hist[(key >> shift) & 255u], 1u);
    }
    __syncthreads();
    __shared__ uint32_t s_digit, s_before;
    if (threadIdx.x < 32) {  // warp 0: 8 bins per lane, warp prefix sum, first bin reaching `want`
      const uint32_t lane = threadIdx.x;
      uint32_t h[8], local = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        h[j] = hist[lane * 8 + j];
        local += h[j];
      }
      uint32_t incl = local;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
      }
      const uint32_t excl = incl - local;
      const unsigned hit = __ballot_sync(0xffffffffu, incl >= want && excl < want);
      const uint32_t src = hit ? __ffs(hit) - 1 : 31;
      if (lane == src) {
        uint32_t cum = excl, dig = lane * 8 + 7;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (cum + h[j] >= want) {
            dig = lane * 8 + j;
            break;
          }
          cum += h[j];
        }
        s_digit = dig;
        s_before = cum;
      }
    }
    __syncthreads();
    prefix |= s_digit << shift;
    mask |= 255u << shift;
    want -= s_before;
    __syncthreads();
  }
  return prefix;
}

// Bitonic sort of (d, id) pairs in shared memory, n a power of two.
__device__ void block_sort_pairs(double* d, uint32_t* id, uint32_t n) {
  for (uint32_t size = 2; size <= n; size <<= 1) {
    for (uint32_t stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (uint32_t i = threadIdx.x; i < n / 2; i += blockDim.x) {
        const uint32_t lo = 2 * i - (i & (stride - 1));
        const uint32_t hi = lo + stride;
        const bool up = ((lo & size) == 0);
        const bool gt = pair_less(d[hi], id[hi], d[lo], id[lo]);
        if (gt == up) {
          const double td = d[lo];
          d[lo] = d[hi];
          d[hi] = td;
          const uint32_t ti = id[lo];
          id[lo] = id[hi];
          id[hi] = ti;
        }
      }
    }
  }
  __syncthreads();
}

// One CTA (512 threads) per query.
__global__ void __launch_bounds__(512) k_coarse_select(IndexView ix, QueryView qv,
                                                       const float* __restrict__ dist32,
                                                       uint32_t nprobe, CoarseBound bd,
                                                       uint32_t* __restrict__ plans,
                                                       double* __restrict__ dists, int* flags,
                                                       uint32_t set_mode, uint32_t cap) {
  pdl_wait();
  extern __shared__ __align__(16) uint8_t sm[];
  double* cd = reinterpret_cast<double*>(sm);                       // cap
  uint32_t* cid = reinterpret_cast<uint32_t*>(cd + cap);              // cap
  double* qsh = reinterpret_cast<double*>(cid + cap);                 // dpad (widened once)
  __shared__ uint32_t hist[256];
  __shared__ uint32_t s_cnt, s_ns, s_wcnt[16];
  __shared__ unsigned long long s_min;
  const uint32_t b = blockIdx.x;
  const float* row = dist32 + (uint64_t)b * ix.K;
  const float qn = qv.qnorm[b];
  for (uint32_t d = threadIdx.x; d < ix.dpad; d += blockDim.x) qsh[d] = qv.qs[(uint64_t)b * ix.dpad + d];
  if (threadIdx.x == 0) {
    s_cnt = 0;
    s_ns = 0;
    s_min = ~0ull;
  }
  // E(c) = ea q c + eb (q^2 + c^2) + ec + es q = c (c B + A) + C with the
  // query's constants rounded up once: two round-up fp32 FMAs per key (every
  // term is >= 0, so each rounding up keeps an upper bound) instead of the
  // double evaluation per key and radix pass (fp64 issues at ~1/30 the rate)
  const double qd = qn;
  const float cA = __double2float_ru(bd.ea * qd), cB = __double2float_ru(bd.eb),
              cC = __double2float_ru(bd.eb * qd * qd + bd.ec + bd.es * qd);
  auto E_of = [&](float cn) { return __fmaf_ru(cn, __fmaf_ru(cn, cB, cA), cC); };
  auto ub_key = [&](uint32_t c) {
    return f2key(__fadd_ru(row[c], E_of(ix.cnorm[c])));
  };
  const uint32_t tau_key = block_radix_select(ix.K, nprobe, ub_key, hist);
  const float tau = key2f(tau_key);
  // Set mode (the search path: plan order and plan distances unused): L = the
  // nprobe-th smallest LOWER bound.  A centroid with ub < L is in the top
  // nprobe for sure -- every centroid at or before it in (d, id) order has
  // lb <= d <= ub < L, and at most nprobe - 1 centroids have lb < L -- so only
  // the uncertain band (lb <= tau, ub >= L) needs the exact double; the plan
  // is the sure set plus the best (nprobe - |sure|) of the band by (d, id),
  // which is the reference's top-nprobe as a set.
  float L = -FLT_MAX;
  if (set_mode) {
    auto lb_key = [&](uint32_t c) {
      return f2key(__fsub_rd(row[c], E_of(ix.cnorm[c])));
    };
    L = key2f(block_radix_select(ix.K, nprobe, lb_key, hist));
  }
  for (uint32_t c = threadIdx.x; c < ix.K; c += blockDim.x) {
    const float E = E_of(ix.cnorm[c]);
    const float lb = __fsub_rd(row[c], E);
    if (lb <= tau) {
      if (set_mode && __fadd_ru(row[c], E) < L) {  // sure
        atomicAdd(&s_ns, 1u);
        atomicMin(&s_min, ((unsigned long long)f2key(row[c]) << 32) | c);
      } else {
        const uint32_t pos = atomicAdd(&s_cnt, 1u);
        if (pos < cap) cid[pos] = c;
      }
    }
  }
  __syncthreads();
  const uint32_t m = s_cnt, ns = s_ns;
  if (m > cap || !(tau <= FLT_MAX) || ns > nprobe || m + ns < nprobe) {  // degenerate: exact streaming path
    if (threadIdx.x == 0) flags[b] = 1;
    return;
  }
  // exact fp64 distances in the reference's order (select_clusters uses
  // squared_l2(centroid, query), :272); the candidates' rows are warmed into
  // L1 by all threads first (every 128-B line in flight at once)
  for (uint32_t idx = threadIdx.x; idx < m * (ix.dpad / 32); idx += blockDim.x) {
    const uint32_t i = idx / (ix.dpad / 32), l = idx - i * (ix.dpad / 32);
    prefetch_l1(ix.cent + (uint64_t)cid[i] * ix.dpad + l * 32);
  }
  for (uint32_t i = threadIdx.x; i < m; i += blockDim.x) {
    const float4* crow = reinterpret_cast<const float4*>(ix.cent + (uint64_t)cid[i] * ix.dpad);
    cd[i] = exact_row_pipelined(ix.dim, qsh, [&](uint32_t g) { return __ldg(crow + g); });
  }
  // the band's best (nprobe - ns) by (d, id) -> plan positions [ns, nprobe)
  const uint32_t take = nprobe - ns;
  uint32_t* out = plans + (uint64_t)b * nprobe;
  if (m <= blockDim.x) {
    // rank placement: each candidate counts the candidates before it in
    // (d, id) order (centroid ids are distinct, so ranks are) -- one barrier
    // instead of the bitonic network's log^2 barriers (which dominated this
    // kernel's stall samples)
    __syncthreads();
    if (threadIdx.x < m) {
      const double di = cd[threadIdx.x];
      const uint32_t ii = cid[threadIdx.x];
      uint32_t r = 0;
      for (uint32_t j = 0; j < m; ++j) r += pair_less(cd[j], cid[j], di, ii) ? 1u : 0u;
      if (r < take) {
        out[ns + r] = ii;
        if (dists) dists[(uint64_t)b * nprobe + r] = di;
      }
    }
  } else {
    uint32_t mp = 1;
    while (mp < m) mp <<= 1;
    for (uint32_t i = m + threadIdx.x; i < mp; i += blockDim.x) {
      cd[i] = DBL_MAX;
      cid[i] = 0xffffffffu;
    }
    block_sort_pairs(cd, cid, mp);
    for (uint32_t i = threadIdx.x; i < take; i += blockDim.x) {
      out[ns + i] = cid[i];
      if (dists) dists[(uint64_t)b * nprobe + i] = cd[i];
    }
  }
  if (ns > 0) {
    // set mode: the sure centroid with the smallest d^ first (the likely
    // nearest list, which the drop-bound seed reads), the other sure ones in
    // id order (deterministic), then the band's best by (d, id)
    const uint32_t cmin = (uint32_t)(s_min & 0xffffffffu);
    const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t base_pos = 1;
    for (uint32_t base = 0; base < ix.K; base += blockDim.x) {
      const uint32_t c = base + threadIdx.x;
      bool sure = false;
      if (c < ix.K && c != cmin) {
        const float E = E_of(ix.cnorm[c]);
        sure = __fsub_rd(row[c], E) <= tau && __fadd_ru(row[c], E) < L;
      }
      const unsigned bal = __ballot_sync(0xffffffffu, sure);
      if (lane == 0) s_wcnt[warp] = __popc(bal);
      __syncthreads();
      uint32_t before = base_pos, total = base_pos;
      for (uint32_t w = 0; w < nw; ++w) {
        if (w < warp) before += s_wcnt[w];
        total += s_wcnt[w];
      }
      if (sure) out[before + __popc(bal & ((1u << lane) - 1u))] = c;
      base_pos = total;
      __syncthreads();
    }
    if (threadIdx.x == 0) out[0] = cmin;
  }
  if (threadIdx.x == 0) flags[b] = 0;
}

// Exact streaming top-nprobe over all K centroids (degenerate inputs only).
// Buffer of `cap` (d, id) pairs; filter against the running nprobe-th pair.
__global__ void __launch_bounds__(512) k_coarse_fallback(IndexView ix, QueryView qv,
                                                         uint32_t nprobe, uint32_t cap,
                                                         uint32_t* __restrict__ plans,
                                                         double* __restrict__ dists,
                                                         const int* flags) {
  pdl_wait();
  const uint32_t b = blockIdx.x;
  if (!flags[b]) return;
  extern __shared__ __align__(16) uint8_t sm[];
  double* bd = reinterpret_cast<double*>(sm);
  uint32_t* bi = reinterpret_cast<uint32_t*>(bd + cap);
  float* qsh = reinterpret_cast<float*>(bi + cap);
  __shared__ uint32_t s_cnt;
  __shared__ double s_thr_d;
  __shared__ uint32_t s_thr_i;
  for (uint32_t d = threadIdx.x; d < ix.dpad; d += blockDim.x) qsh[d] = qv.qs[(uint64_t)b * ix.dpad + d];
  if (threadIdx.x == 0) {
    s_cnt = 0;
    s_thr_d = DBL_MAX;
    s_thr_i = 0xffffffffu;
  }
  __syncthreads();
  for (uint32_t base = 0; base < ix.K; base += blockDim.x) {
    const uint32_t c = base + threadIdx.x;
    double acc = DBL_MAX;
    if (c < ix.K) {
      acc = 0.0;
      const float4* crow = reinterpret_cast<const float4*>(ix.cent + (uint64_t)c * ix.dpad);
      acc = exact_row_pipelined(ix.dim, qsh, [&](uint32_t g) { return __ldg(crow + g); });
    }
    const uint32_t cnt_now = s_cnt;
    __syncthreads();  // every thread has read s_cnt before any append
    if (cnt_now + blockDim.x > cap) {  // compact: sort, keep nprobe
      for (uint32_t i = s_cnt + threadIdx.x; i < cap; i += blockDim.x) {
        bd[i] = DBL_MAX;
        bi[i] = 0xffffffffu;
      }
      block_sort_pairs(bd, bi, cap);
      if (threadIdx.x == 0) {
        s_cnt = nprobe;
        s_thr_d = bd[nprobe - 1];
        s_thr_i = bi[nprobe - 1];
      }
      __syncthreads();
    }
    if (c < ix.K && pair_less(acc, c, s_thr_d, s_thr_i)) {
      const uint32_t pos = atomicAdd(&s_cnt, 1u);
      bd[pos] = acc;
      bi[pos] = c;
    }
    __syncthreads();
  }
  for (uint32_t i = s_cnt + threadIdx.x; i < cap; i += blockDim.x) {
    bd[i] = DBL_MAX;
    bi[i] = 0xffffffffu;
  }
  block_sort_pairs(bd, bi, cap);
  for (uint32_t i = threadIdx.x; i < nprobe; i += blockDim.x) {
    plans[(uint64_t)b * nprobe + i] = bi[i];
    if (dists) dists[(uint64_t)b * nprobe + i] = bd[i];
  }
}

// nprobe > kNprobeMax (a plan longer than the candidate buffers hold): the
// exact fp64 distance to EVERY centroid, one thread each, written as
// order-preserving keys (distances are >= +0, so their bit patterns order as
// unsigned integers) with the centroid id as value; a stable radix sort per
// query then leaves (distance, id) order because equal keys keep the
// ascending-id input order (vector_index.cpp:272-275).
__global__ void __launch_bounds__(256) k_coarse_all(IndexView ix, QueryView qv, unsigned long long* keys,
                                                    uint32_t* vals) {
  extern __shared__ __align__(16) uint8_t sm[];
  float* qsh = reinterpret_cast<float*>(sm);
  const uint32_t b = blockIdx.y;
  for (uint32_t d = threadIdx.x; d < ix.dpad; d += blockDim.x) qsh[d] = qv.qs[(uint64_t)b * ix.dpad + d];
  __syncthreads();
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ix.K) return;
  const float4* crow = reinterpret_cast<const float4*>(ix.cent + (uint64_t)c * ix.dpad);
  const double d = exact_row_pipelined(ix.dim, qsh, [&](uint32_t g) { return __ldg(crow + g); });
  keys[(uint64_t)b * ix.K + c] = (unsigned long long)__double_as_longlong(d);
  vals[(uint64_t)b * ix.K + c] = c;
}

__global__ void k_seg_offsets(uint32_t* off, uint32_t n, uint32_t K) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= n) off[i] = i * K;
}

__global__ void k_take_plans(const unsigned long long* keys, const uint32_t* vals, uint32_t K, uint32_t nprobe,
                             uint32_t* plans, double* dists) {
  const uint32_t b = blockIdx.y;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nprobe; i += gridDim.x * blockDim.x) {
    plans[(uint64_t)b * nprobe + i] = vals[(uint64_t)b * K + i];
    if (dists) dists[(uint64_t)b * nprobe + i] = __longlong_as_double((long long)keys[(uint64_t)b * K + i]);
  }
}

}  // namespace

void launch_prep_queries(const float* q_in, uint32_t n, uint32_t dim, uint32_t dpad, int metric,
                         bool normalize, float* qs, float* qn2, float* qnorm, float* qsc, int* err,
                         cudaStream_t s) {
  if (n == 0) return;
  launch_pdl(k_prep_queries, dim3(n), dim3(128), 0, s, q_in, n, dim, dpad, metric, normalize ? 1 : 0, qs, qn2, qnorm, qsc,
                                   err);
}

uint32_t coarse_dist_splits(const IndexView& ix, uint32_t n_queries) {
  const int sms = device_sm_count();
  const uint64_t t32 = (uint64_t)((ix.K + 31) / 32) * ((n_queries + CT_Q - 1) / CT_Q);
  if (t32 >= 2ull * sms || ix.dpad < 256) return 1;
  uint32_t S = 1;
  while (S * 2 <= ix.dpad / 64 && t32 * S < 4ull * sms) S *= 2;  // >= 64 dims per split
  return S;
}

void launch_coarse_dist(const IndexView& ix, const QueryView& qv, float* dist32, cudaStream_t s,
                        float* part) {
  const int sms = device_sm_count();
  const uint32_t qt = (qv.n + CT_Q - 1) / CT_Q;
  auto tiles = [&](uint32_t ctc) { return (uint64_t)((ix.K + ctc - 1) / ctc) * qt; };
  const uint32_t S = part ? coarse_dist_splits(ix, qv.n) : 1u;
  if (S > 1) {
    const uint32_t span = (ix.dpad / S + CT_K - 1) / CT_K * CT_K;
    launch_pdl(k_coarse_dist<32, true>, dim3(dim3((ix.K + 31) / 32, qt, S)), dim3(64), 0, s, ix, qv, part, span);
    const uint64_t n = (uint64_t)qv.n * ix.K;
    launch_pdl(k_coarse_combine, dim3((unsigned)std::min<uint64_t>((n + 255) / 256, 4ull * sms)), dim3(256), 0, s, ix, qv, part, S, dist32);
    return;
  }
  if (tiles(128) >= 2ull * sms)
    launch_pdl(k_coarse_dist<128>, dim3(dim3((ix.K + 127) / 128, qt)), dim3(256), 0, s, ix, qv, dist32, 0u);
  else if (tiles(64) >= 2ull * sms)
    launch_pdl(k_coarse_dist<64>, dim3(dim3((ix.K + 63) / 64, qt)), dim3(128), 0, s, ix, qv, dist32, 0u);
  else
    launch_pdl(k_coarse_dist<32>, dim3(dim3((ix.K + 31) / 32, qt)), dim3(64), 0, s, ix, qv, dist32, 0u);
}

// eps (|q| + |c|)^2 + abs, expanded
CoarseBound coarse_bound_ffma(uint32_t dim) {
  const double e = filter_eps(dim);
  return {2.0 * e, e, filter_abs(dim), 0.0};
}
// bound_h16 with x = the centroid (its own norm bound cnorm[c]); bound_h16's
// subnormal floor 2 sqrt(D) 2^-38 |x||q| is relative to the norm the SCALE was
// taken from -- here the largest centroid norm cmax, shared by all centroids --
// so that term is added with cmax (x1.5 headroom and the factor 2 of the
// distance, as bound_h16 carries it).
CoarseBound coarse_bound_h16(uint32_t dim, float cmax) {
  CoarseBound b{};
  bound_h16(dim, &b.ea, &b.eb, &b.ec);
  b.es = 1.5 * 2.0 * 2.0 * std::sqrt((double)dim) * 0x1p-38 * 1.01 * (double)cmax;
  return b;
}

void launch_coarse_select(const IndexView& ix, const QueryView& qv, const float* dist32,
                          uint32_t nprobe, const CoarseBound& bd, uint32_t* plans, double* dists, int* flags,
                          cudaStream_t s, bool set_mode) {
  // candidate buffer: 4x the plan (>= 1024) -- more candidates take the
  // exact streaming path -- instead of a fixed kCandCap, so dense batches keep
  // several CTAs per SM resident while one's exact fp64 chains run
  uint32_t cap = 1024;
  while (cap < 4 * nprobe && cap < (uint32_t)kCandCap) cap <<= 1;
  if (cap < nprobe) cap = nprobe;  // nprobe <= kNprobeMax = kCandCap
  const size_t smem = (size_t)cap * (8 + 4) + (size_t)ix.dpad * 8;
  smem_optin((const void*)k_coarse_select, 220 * 1024);
  smem_optin((const void*)k_coarse_fallback, 200 * 1024);
  // 512 threads for batches up to ~4 per SM (a query's latency is the step's:
  // fewer threads measured slower, C2 41 -> 61 us, C3 59 -> 75 us); 256 for
  // dense batches (twice the CTAs resident to cover the fp64 chains)
  const int threads = qv.n > 4u * (uint32_t)device_sm_count() ? 256 : 512;
  launch_pdl(k_coarse_select, dim3(qv.n), dim3(threads), smem, s, ix, qv, dist32, nprobe, bd, plans, dists, flags,
             (set_mode && !dists) ? 1u : 0u, cap);
}

void launch_coarse_fallback(const IndexView& ix, const QueryView& qv, uint32_t nprobe,
                            uint32_t* plans, double* dists, const int* flags, cudaStream_t s) {
  uint32_t cap = 1024;
  while (cap < nprobe + 512) cap <<= 1;
  const size_t smem = (size_t)cap * 12 + (size_t)ix.dpad * 4;
  launch_pdl(k_coarse_fallback, dim3(qv.n), dim3(512), smem, s, ix, qv, nprobe, cap, plans, dists, flags);
}

}  // namespace hivf

namespace hivf {
// Exact select for plans longer than kNprobeMax (see k_coarse_all).  scratch
// holds keys/values twice, the segment offsets and CUB's temporary storage;
// *scratch_bytes returns the size needed when scratch == nullptr.
cudaError_t launch_coarse_all(const IndexView& ix, const QueryView& qv, uint32_t nprobe, uint32_t* plans,
                              double* dists, void* scratch, size_t* scratch_bytes, cudaStream_t s) {
  const size_t n = (size_t)qv.n * ix.K;
  auto al = [](size_t x) { return (x + 255) & ~size_t(255); };
  size_t cub_bytes = 0;
  cudaError_t e = cub::DeviceSegmentedRadixSort::SortPairs(
      nullptr, cub_bytes, (const unsigned long long*)nullptr, (unsigned long long*)nullptr,
      (const uint32_t*)nullptr, (uint32_t*)nullptr, (int)n, (int)qv.n, (const uint32_t*)nullptr,
      (const uint32_t*)nullptr, 0, 64, s);
  if (e != cudaSuccess) return e;
  const size_t o_k0 = 0, o_k1 = al(o_k0 + n * 8), o_v0 = al(o_k1 + n * 8), o_v1 = al(o_v0 + n * 4),
               o_off = al(o_v1 + n * 4), o_tmp = al(o_off + (qv.n + 1) * 4ull), total = al(o_tmp + cub_bytes);
  if (!scratch) {
    *scratch_bytes = total;
    return cudaSuccess;
  }
  if (*scratch_bytes < total) return cudaErrorInvalidValue;
  uint8_t* base = static_cast<uint8_t*>(scratch);
  auto* k0 = reinterpret_cast<unsigned long long*>(base + o_k0);
  auto* k1 = reinterpret_cast<unsigned long long*>(base + o_k1);
  auto* v0 = reinterpret_cast<uint32_t*>(base + o_v0);
  auto* v1 = reinterpret_cast<uint32_t*>(base + o_v1);
  auto* off = reinterpret_cast<uint32_t*>(base + o_off);
  k_coarse_all<<<dim3((ix.K + 255) / 256, qv.n), 256, (size_t)ix.dpad * 4, s>>>(ix, qv, k0, v0);
  k_seg_offsets<<<(qv.n + 256) / 256, 256, 0, s>>>(off, qv.n, ix.K);
  size_t tb = cub_bytes;
  e = cub::DeviceSegmentedRadixSort::SortPairs(base + o_tmp, tb, k0, k1, v0, v1, (int)n, (int)qv.n, off, off + 1,
                                               0, 64, s);
  if (e != cudaSuccess) return e;
  k_take_plans<<<dim3((nprobe + 255) / 256, qv.n), 256, 0, s>>>(k1, v1, ix.K, nprobe, plans, dists);
  return cudaGetLastError();
}
}  // namespace hivf
