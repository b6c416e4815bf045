// kmeans.cu -- index build on the GPU: ivf::train_kmeans and the Lloyd
// update of /root/reference/proj/src/vector_index.cpp:99-200, with the
// reference's arithmetic reproduced exactly:
//   * every distance is squared_l2 (embedding.hpp:27-34: sequential fp64
//     chain, no FMA) -- exact_step;
//   * k-means++ sampling uses the sequentially rounded running sum of dist2
//     (vector_index.cpp:123-134): one thread walks the n values in index order
//     and stores every prefix; the prefix is monotone (dist2 >= 0), so the
//     first index with acc > target is an exact binary search;
//   * Lloyd sums `sum[d] += row[d]` run per (cluster, dim) over the cluster's
//     points in increasing index order (a stable sort by cluster), then
//     (float)(sum / count) (vector_index.cpp:164-180);
//   * empty clusters take the farthest unused point from its assigned
//     centroid, ties to the lowest index, in cluster order (:181-196).
// Assignment (nearest_centroid, ties -> lowest id, :18-29) is the coarse
// assign of assign.cu with nprobe = 1 (api.cu, hivf_compute_assignments).
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace hivf {
namespace {

// squared_l2(row, c) of the reference, row-major corpus
__device__ __forceinline__ double sq_row(const float* __restrict__ row, const float* __restrict__ c,
                                         uint32_t dim) {
  double acc = 0.0;
  uint32_t d = 0;
  if (((reinterpret_cast<uintptr_t>(row) | reinterpret_cast<uintptr_t>(c)) & 15) == 0) {
    for (; d + 4 <= dim; d += 4) {
      const float4 a = *reinterpret_cast<const float4*>(row + d);
      const float4 b = *reinterpret_cast<const float4*>(c + d);
      acc = exact_step(acc, a.x, b.x);
      acc = exact_step(acc, a.y, b.y);
      acc = exact_step(acc, a.z, b.z);
      acc = exact_step(acc, a.w, b.w);
    }
  }
  for (; d < dim; ++d) acc = exact_step(acc, row[d], c[d]);
  return acc;
}

// dist2[i] = d(row i, c) (mode 0) or min(dist2[i], d) (mode 1, vector_index.cpp:146-149)
__global__ void k_dist2(const float* __restrict__ X, uint64_t n, uint32_t dim, const float* __restrict__ c,
                        double* __restrict__ dist2, int mode) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double d = sq_row(X + i * dim, c, dim);
  if (mode == 0 || d < dist2[i]) dist2[i] = d;
}

// running sum in index order (total += d, :123-124) with every prefix kept;
// the walk is the reference's own left-to-right chain of rounded adds.  One
// thread owns the chain; the other warps of the block stream dist2 tiles into
// shared memory ahead of it and write the finished prefixes back, so the
// serial thread only sees shared-memory latency.
constexpr int kScanTile = 2048;  // doubles per tile (16 KB), double-buffered
__global__ void __launch_bounds__(512, 1) k_prefix_seq(const double* __restrict__ dist2, uint64_t n,
                                                       double* __restrict__ prefix,
                                                       double* __restrict__ total) {
  __shared__ double buf[2][kScanTile];
  const uint64_t ntile = (n + kScanTile - 1) / kScanTile;
  double acc = 0.0;
  // prologue: tile 0
  for (uint32_t e = threadIdx.x; e < kScanTile; e += blockDim.x) {
    const uint64_t i = e;
    buf[0][e] = i < n ? dist2[i] : 0.0;
  }
  __syncthreads();
  for (uint64_t t = 0; t < ntile; ++t) {
    const int cur = (int)(t & 1), nxt = cur ^ 1;
    const uint64_t base = t * kScanTile;
    const uint32_t len = (uint32_t)min((uint64_t)kScanTile, n - base);
    if (threadIdx.x == 0) {
      double* b = buf[cur];
      uint32_t e = 0;
      for (; e + 8 <= len; e += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = b[e + u];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          acc = __dadd_rn(acc, v[u]);
          b[e + u] = acc;
        }
      }
      for (; e < len; ++e) {
        acc = __dadd_rn(acc, b[e]);
        b[e] = acc;
      }
    } else if (t + 1 < ntile) {
      // helpers (threads 32..): stage the next tile while the chain runs
      const uint64_t nb = base + kScanTile;
      for (uint32_t e = threadIdx.x - 32; threadIdx.x >= 32 && e < kScanTile; e += blockDim.x - 32) {
        const uint64_t i = nb + e;
        buf[nxt][e] = i < n ? dist2[i] : 0.0;
      }
    }
    __syncthreads();
    for (uint32_t e = threadIdx.x; e < len; e += blockDim.x) prefix[base + e] = buf[cur][e];
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = acc;
}

// k-means++ pick (vector_index.cpp:125-135): target = u * total, first i with
// prefix[i] > target (pick = n-1 if none).  total == 0 -> *zero = 1 and the
// pick is resolved by k_pick_zero.  `us` holds the pre-drawn uniforms; a draw
// is consumed only when total > 0, exactly as the reference consumes its Rng.
__global__ void k_pick(const double* __restrict__ prefix, uint64_t n, const double* __restrict__ total,
                       const double* __restrict__ us, int* __restrict__ draw, uint64_t* __restrict__ pick,
                       int* __restrict__ zero) {
  if (threadIdx.x || blockIdx.x) return;
  const double t = *total;
  if (t > 0.0) {
    const double target = __dmul_rn(us[*draw], t);
    *draw += 1;
    uint64_t lo = 0, hi = n;  // first index with prefix > target
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (prefix[mid] > target) hi = mid; else lo = mid + 1;
    }
    *pick = lo < n ? lo : n - 1;
    *zero = 0;
  } else {
    *pick = ~0ull;  // lowest not-yet-chosen row, via atomicMin in k_pick_zero
    *zero = 1;
  }
}

// total == 0: the lowest index whose row differs bytewise from every chosen
// center (vector_index.cpp:137-151); none -> 0
__global__ void k_pick_zero(const float* __restrict__ X, uint64_t n, uint32_t dim,
                            const float* __restrict__ cents, uint32_t m, const int* __restrict__ zero,
                            unsigned long long* __restrict__ pick) {
  if (!*zero) return;
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t* r = reinterpret_cast<const uint32_t*>(X + i * dim);
  for (uint32_t c = 0; c < m; ++c) {
    const uint32_t* q = reinterpret_cast<const uint32_t*>(cents + (uint64_t)c * dim);
    bool same = true;
    for (uint32_t d = 0; d < dim && same; ++d) same = r[d] == q[d];
    if (same) return;
  }
  atomicMin(pick, (unsigned long long)i);
}

// centroid m <- row pick (raw copy)
__global__ void k_take_row(const float* __restrict__ X, uint64_t n, uint32_t dim, const uint64_t* pick,
                           float* __restrict__ cents, uint32_t m) {
  uint64_t p = *pick;
  if (p >= n) p = 0;
  for (uint32_t d = threadIdx.x; d < dim; d += blockDim.x) cents[(uint64_t)m * dim + d] = X[p * dim + d];
}

__global__ void k_iota(uint32_t* v, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = (uint32_t)i;
}

// assign == prev ?  (vector_index.cpp:158) and prev <- assign
__global__ void k_same_assign(const uint32_t* __restrict__ a, uint32_t* __restrict__ prev, uint64_t n,
                              int* __restrict__ differs) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (a[i] != prev[i]) {
    *differs = 1;
    prev[i] = a[i];
  }
}

// cluster c's points are sorted[off[c], off[c+1]); off from the sorted keys
__global__ void k_cluster_bounds(const uint32_t* __restrict__ keys, uint64_t n, uint32_t K,
                                 uint64_t* __restrict__ off) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > n) return;
  const uint32_t cur = i < n ? keys[i] : K;
  const uint32_t prv = i > 0 ? keys[i - 1] : 0xffffffffu;
  if (i == 0) {
    for (uint32_t c = 0; c <= cur && c <= K; ++c) off[c] = 0;
  } else if (cur != prv) {
    for (uint32_t c = prv + 1; c <= cur && c <= K; ++c) off[c] = i;
  }
}

// new centroid (float)(sum / count) per (cluster, dim), sums in point order
__global__ void k_cluster_means(const float* __restrict__ X, uint32_t dim, uint32_t K,
                                const uint32_t* __restrict__ sorted_idx, const uint64_t* __restrict__ off,
                                float* __restrict__ cents) {
  const uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (uint64_t)K * dim) return;
  const uint32_t c = (uint32_t)(t / dim), d = (uint32_t)(t % dim);
  const uint64_t b = off[c], e = off[c + 1];
  if (b == e) return;  // empty: re-seeded by the host loop
  double s = 0.0;
  for (uint64_t p = b; p < e; ++p) s = __dadd_rn(s, (double)X[(uint64_t)sorted_idx[p] * dim + d]);
  cents[t] = __double2float_rn(__ddiv_rn(s, (double)(e - b)));
}

// empty cluster c (vector_index.cpp:183-195): distance of every unused point
// to its assigned centroid as the reference's loop sees it at cluster c
// (clusters < c already updated, > c not yet); max over d, then min index
__global__ void k_far_dist(const float* __restrict__ X, uint64_t n, uint32_t dim,
                           const uint32_t* __restrict__ assign, const float* __restrict__ new_c,
                           const float* __restrict__ old_c, uint32_t c, const uint8_t* __restrict__ used,
                           double* __restrict__ dd, unsigned long long* __restrict__ dmax) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (used[i]) {
    dd[i] = -1.0;
    return;
  }
  const uint32_t a = assign[i];
  const float* cen = (a < c ? new_c : old_c) + (uint64_t)a * dim;
  const double d = sq_row(X + i * dim, cen, dim);
  dd[i] = d;
  // d >= 0 (or NaN, never selected by `d > far_d`): bit patterns order like values
  if (d >= 0.0) atomicMax(dmax, (unsigned long long)__double_as_longlong(d));
}

__global__ void k_far_pick(const double* __restrict__ dd, uint64_t n, const unsigned long long* dmax,
                           unsigned long long* __restrict__ pick) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (dd[i] >= 0.0 && (unsigned long long)__double_as_longlong(dd[i]) == *dmax) atomicMin(pick, (unsigned long long)i);
}

__global__ void k_far_take(const float* __restrict__ X, uint64_t n, uint32_t dim,
                           const unsigned long long* pick, uint8_t* used, float* __restrict__ new_c,
                           uint32_t c) {
  uint64_t p = *pick;
  if (p >= n) p = 0;  // every point used: far_i stays 0 (vector_index.cpp:183-184)
  if (threadIdx.x == 0) used[p] = 1;
  for (uint32_t d = threadIdx.x; d < dim; d += blockDim.x) new_c[(uint64_t)c * dim + d] = X[p * dim + d];
}

inline unsigned grid(uint64_t n, unsigned b) { return (unsigned)((n + b - 1) / b); }

}  // namespace

void launch_kmeans_dist2(const float* X, uint64_t n, uint32_t dim, const float* c, double* dist2, int mode,
                         cudaStream_t s) {
  k_dist2<<<grid(n, 128), 128, 0, s>>>(X, n, dim, c, dist2, mode);
}
void launch_kmeans_prefix(const double* dist2, uint64_t n, double* prefix, double* total, cudaStream_t s) {
  k_prefix_seq<<<1, 512, 0, s>>>(dist2, n, prefix, total);
}
void launch_kmeans_pick(const double* prefix, uint64_t n, const double* total, const double* us, int* draw,
                        uint64_t* pick, int* zero, const float* X, uint32_t dim, float* cents, uint32_t m,
                        cudaStream_t s) {
  k_pick<<<1, 1, 0, s>>>(prefix, n, total, us, draw, pick, zero);
  k_pick_zero<<<grid(n, 256), 256, 0, s>>>(X, n, dim, cents, m, zero,
                                           reinterpret_cast<unsigned long long*>(pick));
  k_take_row<<<1, 256, 0, s>>>(X, n, dim, pick, cents, m);
}
void launch_iota(uint32_t* v, uint64_t n, cudaStream_t s) { k_iota<<<grid(n, 256), 256, 0, s>>>(v, n); }
void launch_same_assign(const uint32_t* a, uint32_t* prev, uint64_t n, int* differs, cudaStream_t s) {
  k_same_assign<<<grid(n, 256), 256, 0, s>>>(a, prev, n, differs);
}
void launch_cluster_means(const float* X, uint32_t dim, uint32_t K, const uint32_t* sorted_keys,
                          const uint32_t* sorted_idx, uint64_t n, uint64_t* off, float* cents,
                          cudaStream_t s) {
  k_cluster_bounds<<<grid(n + 1, 256), 256, 0, s>>>(sorted_keys, n, K, off);
  k_cluster_means<<<grid((uint64_t)K * dim, 128), 128, 0, s>>>(X, dim, K, sorted_idx, off, cents);
}
void launch_far_point(const float* X, uint64_t n, uint32_t dim, const uint32_t* assign, const float* new_c,
                      const float* old_c, uint32_t c, uint8_t* used, double* dd, unsigned long long* scratch2,
                      cudaStream_t s) {
  cudaMemsetAsync(scratch2, 0, 8, s);                 // dmax = +0.0 bits
  cudaMemsetAsync(scratch2 + 1, 0xff, 8, s);          // pick = ~0
  k_far_dist<<<grid(n, 128), 128, 0, s>>>(X, n, dim, assign, new_c, old_c, c, used, dd, scratch2);
  k_far_pick<<<grid(n, 256), 256, 0, s>>>(dd, n, scratch2, scratch2 + 1);
  k_far_take<<<1, 256, 0, s>>>(X, n, dim, scratch2 + 1, used, const_cast<float*>(new_c), c);
}

}  // namespace hivf
