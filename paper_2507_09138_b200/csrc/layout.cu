// layout.cu -- K6: inverted-list packing into HBM.
//
// Replaces the host-side list building of ivf::index_from_assignments
// (/root/reference/proj/src/vector_index.cpp:210-235).  Input rows arrive
// row-major in list order (exactly the order index_from_assignments appends
// them); output is the chunk-major, 16B-group-swizzled layout the scan kernel
// streams with 1-D bulk copies (common.cuh).
#include <cuda_fp16.h>
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace hivf {

namespace {

// One thread per (row, 4-dim group).  Also computes fp32 |x|^2 (from an fp64
// sum; only used by the error-bounded filter) and the per-list max |x|.
__global__ void k_pack_lists(const float* __restrict__ src, uint64_t r_first,
                             const uint64_t* __restrict__ pos, uint64_t n_rows, uint32_t dim,
                             uint32_t dpad, const uint64_t* __restrict__ list_off, uint32_t K,
                             float* __restrict__ dst, float* __restrict__ xnorm2,
                             uint32_t* __restrict__ maxnorm_bits, int* err) {
  const uint32_t groups = dpad / 4;
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= n_rows * groups) return;
  const uint64_t lrow = gid / groups;        // row within this chunk
  const uint64_t r = pos ? pos[lrow] : r_first + lrow;  // global row (list order)
  const uint32_t g = (uint32_t)(gid % groups);
  // list of row r: upper_bound(list_off, r) - 1
  uint32_t lo = 0, hi = K;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (list_off[mid + 1] <= r) lo = mid + 1; else hi = mid;
  }
  const uint32_t c = lo;
  const uint64_t base = list_off[c] * (uint64_t)dpad;
  const uint64_t n_c = list_off[c + 1] - list_off[c];
  const uint64_t lr = r - list_off[c];
  float v[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const uint32_t d = g * 4 + e;
    v[e] = d < dim ? src[lrow * dim + d] : 0.f;
    if (!isfinite(v[e])) *err = 1;
  }
  const uint64_t o = swz_offset(base, n_c, lr, g * 4, dpad);
  *reinterpret_cast<float4*>(dst + o) = make_float4(v[0], v[1], v[2], v[3]);
  if (g == 0) {
    double acc = 0.0;
    for (uint32_t d = 0; d < dim; ++d) {
      const double x = (double)src[lrow * dim + d];
      acc = __dadd_rn(acc, __dmul_rn(x, x));
    }
    xnorm2[r] = __double2float_rn(acc);
    const float nrm = __double2float_ru(sqrt(acc) * (1.0 + 1e-6));
    atomicMax(maxnorm_bits + c, __float_as_uint(nrm));  // non-negative floats order as uints
  }
}

// fp16 filter copy: one thread per 16-B
// granule (8 dims) of a row, read from the fp32 tile-major copy, scaled by the
// list's 2^e_l (exact) and rounded to fp16 (RN) into the same tile-major
// SWIZZLE_64B pattern with 32-dim chunks (dpf floats = 2 dpf halfs per row).
__global__ void k_pack_h16(const float* __restrict__ vec, const uint64_t* __restrict__ list_off, uint32_t K,
                           uint32_t dpad, uint32_t dpf, uint64_t N, const float* __restrict__ lsc,
                           float* __restrict__ vech) {
  const uint32_t gpr = dpf / 4;  // granules per row
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= N * gpr) return;
  const uint64_t r = gid / gpr;
  const uint32_t G = (uint32_t)(gid % gpr), ch = G >> 2, gi = G & 3;
  uint32_t lo = 0, hi = K;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (list_off[mid + 1] <= r) lo = mid + 1; else hi = mid;
  }
  const uint32_t c = lo;
  const uint64_t n_c = list_off[c + 1] - list_off[c];
  const uint64_t lr = r - list_off[c];
  const float up = 1.f / lsc[c];  // 2^e_l
  __align__(16) __half h[8];
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const uint32_t d = ch * 32 + gi * 8 + p * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (d < dpad) v = *reinterpret_cast<const float4*>(vec + swz_offset(list_off[c] * (uint64_t)dpad, n_c, lr, d, dpad));
    h[p * 4 + 0] = __float2half_rn(v.x * up);
    h[p * 4 + 1] = __float2half_rn(v.y * up);
    h[p * 4 + 2] = __float2half_rn(v.z * up);
    h[p * 4 + 3] = __float2half_rn(v.w * up);
  }
  const uint64_t r0 = lr - lr % kTileRows;
  const uint64_t o = list_off[c] * (uint64_t)dpf + tile_chunk_offset(n_c, dpf, r0, ch) + (lr - r0) * kChunk +
                     (uint64_t)((gi ^ ((uint32_t)(lr >> 1) & 3u)) * 4);
  *reinterpret_cast<uint4*>(vech + o) = *reinterpret_cast<const uint4*>(h);
}


// Inverse of the packing: rows [first, first+n) back to row-major.
__global__ void k_unpack_rows(const float* __restrict__ vec, const uint64_t* __restrict__ list_off,
                              uint32_t K, uint32_t dim, uint32_t dpad, uint64_t first, uint64_t n,
                              float* __restrict__ out) {
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= n * dim) return;
  const uint64_t lrow = gid / dim;
  const uint32_t d = (uint32_t)(gid % dim);
  const uint64_t r = first + lrow;
  uint32_t lo = 0, hi = K;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (list_off[mid + 1] <= r) lo = mid + 1; else hi = mid;
  }
  const uint64_t n_c = list_off[lo + 1] - list_off[lo];
  out[gid] = vec[swz_offset(list_off[lo] * (uint64_t)dpad, n_c, r - list_off[lo], d, dpad)];
}

__global__ void k_pack_centroids(const float* __restrict__ src, uint32_t K, uint32_t dim,
                                 uint32_t dpad, float* __restrict__ dst, float* cnorm2,
                                 float* cnorm, int* err) {
  const uint32_t c = blockIdx.x;
  for (uint32_t d = threadIdx.x; d < dpad; d += blockDim.x) {
    const float v = d < dim ? src[(uint64_t)c * dim + d] : 0.f;
    if (!isfinite(v)) *err = 1;
    dst[(uint64_t)c * dpad + d] = v;
  }
  if (threadIdx.x == 0) {
    double acc = 0.0;
    for (uint32_t d = 0; d < dim; ++d) {
      const double x = (double)src[(uint64_t)c * dim + d];
      acc = __dadd_rn(acc, __dmul_rn(x, x));
    }
    cnorm2[c] = __double2float_rn(acc);
    cnorm[c] = __double2float_ru(sqrt(acc) * (1.0 + 1e-6));
  }
}

// mean_assigned_distance (vector_index.cpp:222-233): exact per-row distance to
// its centroid, reduced in a fixed tree (deterministic; the reference sums in
// corpus order, so the last bits may differ -- the value is informational).
// With row_dist the exact per-row doubles are also written (list order), so a
// caller can form the reference's corpus-order sum bit-exactly
// (hivf_index_row_distances).
__global__ void k_mean_assigned(IndexView ix, double* partial, double* row_dist) {
  __shared__ double red[256];
  double acc = 0.0;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < ix.N;
       r += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t lo = 0, hi = ix.K;
    while (lo < hi) {
      const uint32_t mid = (lo + hi) >> 1;
      if (ix.list_off[mid + 1] <= r) lo = mid + 1; else hi = mid;
    }
    const uint64_t base = ix.list_off[lo] * (uint64_t)ix.dpad;
    const uint64_t n_c = ix.list_off[lo + 1] - ix.list_off[lo];
    const uint64_t lr = r - ix.list_off[lo];
    double d = 0.0;
    for (uint32_t k = 0; k < ix.dim; ++k)
      d = exact_step(d, ix.vec[swz_offset(base, n_c, lr, k, ix.dpad)], ix.cent[(uint64_t)lo * ix.dpad + k]);
    if (row_dist) row_dist[r] = d;
    acc += d;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) partial[blockIdx.x] = red[0];
}

__global__ void k_check_dup(const uint64_t* sorted, uint64_t n, int* err) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x + 1;
  if (i < n && sorted[i] == sorted[i - 1]) *err = 2;
}

}  // namespace

void launch_pack_h16(const float* vec, const uint64_t* d_list_off, uint32_t K, uint32_t dpad, uint32_t dpf,
                     uint64_t N, const float* lsc, float* vech, cudaStream_t s) {
  const uint64_t total = N * (dpf / 4);
  if (!total) return;
  k_pack_h16<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(vec, d_list_off, K, dpad, dpf, N, lsc, vech);
}

void launch_pack_lists(const float* src_rows, uint64_t r_first, const uint64_t* pos,
                       uint64_t n_rows, uint32_t dim, uint32_t dpad, const uint64_t* d_list_off,
                       uint32_t K, float* dst, float* xnorm2, uint32_t* maxnorm_bits, int* err,
                       cudaStream_t s) {
  const uint64_t total = n_rows * (dpad / 4);
  if (total == 0) return;
  const uint32_t bs = 256;
  k_pack_lists<<<(unsigned)((total + bs - 1) / bs), bs, 0, s>>>(
      src_rows, r_first, pos, n_rows, dim, dpad, d_list_off, K, dst, xnorm2, maxnorm_bits, err);
}

void launch_unpack_rows(const float* vec, const uint64_t* d_list_off, uint32_t K, uint32_t dim,
                        uint32_t dpad, uint64_t first, uint64_t n, float* out, cudaStream_t s) {
  const uint64_t total = n * dim;
  if (!total) return;
  k_unpack_rows<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(vec, d_list_off, K, dim, dpad, first,
                                                               n, out);
}

void launch_pack_centroids(const float* src, uint32_t K, uint32_t dim, uint32_t dpad, float* dst,
                           float* cnorm2, float* cnorm, int* err, cudaStream_t s) {
  k_pack_centroids<<<K, 128, 0, s>>>(src, K, dim, dpad, dst, cnorm2, cnorm, err);
}

void launch_mean_assigned(const IndexView& ix, double* partial, uint32_t n_partial,
                          cudaStream_t s, double* row_dist) {
  k_mean_assigned<<<n_partial, 256, 0, s>>>(ix, partial, row_dist);
}

void launch_check_dup_ids(const uint64_t* sorted_ids, uint64_t n, int* err, cudaStream_t s) {
  if (n < 2) return;
  k_check_dup<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(sorted_ids, n, err);
}

}  // namespace hivf

namespace hivf {
namespace {
__global__ void k_scatter_ids(const uint64_t* ids, const uint64_t* pos, uint64_t n, uint64_t* out) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[pos[i]] = ids[i];
}
}  // namespace
void launch_scatter_ids(const uint64_t* ids, const uint64_t* pos, uint64_t n, uint64_t* out,
                        cudaStream_t s) {
  if (n) k_scatter_ids<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(ids, pos, n, out);
}
namespace {
__global__ void k_ptr_flips(const float** table, PtrFlips f) {
  if (threadIdx.x < f.n) table[f.list[threadIdx.x]] = f.ptr[threadIdx.x];
}
}  // namespace

void launch_ptr_flips(const float** table, const PtrFlips& f, cudaStream_t s) {
  if (f.n) k_ptr_flips<<<1, kPtrFlipBatch, 0, s>>>(table, f);
}

namespace {
// locator (vector_index.cpp:226-227): binary search of doc ids in the sorted
// (id, row) table built on first use
__global__ void k_locate(const uint64_t* __restrict__ sid, const uint64_t* __restrict__ srow, uint64_t N,
                         const uint64_t* __restrict__ list_off, uint32_t K, const uint64_t* __restrict__ q,
                         uint32_t n, uint32_t* __restrict__ cl_out, uint64_t* __restrict__ row_out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint64_t id = q[i];
  uint64_t lo = 0, hi = N;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (sid[mid] < id) lo = mid + 1; else hi = mid;
  }
  if (lo >= N || sid[lo] != id) {
    cl_out[i] = 0xffffffffu;
    row_out[i] = ~0ull;
    return;
  }
  const uint64_t r = srow[lo];
  uint32_t a = 0, b = K;
  while (a < b) {
    const uint32_t mid = (a + b) >> 1;
    if (list_off[mid + 1] <= r) a = mid + 1; else b = mid;
  }
  cl_out[i] = a;
  row_out[i] = r;
}

// doc_embedding for arbitrary rows (list order): out[i][d]
__global__ void k_gather_rows(IndexView ix, const uint64_t* __restrict__ rows, uint32_t n, float* __restrict__ out) {
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (uint64_t)n * ix.dim) return;
  const uint32_t i = (uint32_t)(gid / ix.dim), d = (uint32_t)(gid % ix.dim);
  const uint64_t r = rows[i];
  uint32_t a = 0, b = ix.K;
  while (a < b) {
    const uint32_t mid = (a + b) >> 1;
    if (ix.list_off[mid + 1] <= r) a = mid + 1; else b = mid;
  }
  const uint64_t beg = ix.list_off[a], n_c = ix.list_off[a + 1] - beg;
  out[gid] = list_base(ix, a, beg)[swz_offset(0, n_c, r - beg, d, ix.dpad)];
}

__global__ void k_iota64(uint64_t* v, uint64_t n) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) v[i] = i;
}
}  // namespace

void launch_locate(const uint64_t* sid, const uint64_t* srow, uint64_t N, const uint64_t* list_off, uint32_t K,
                   const uint64_t* q, uint32_t n, uint32_t* cl_out, uint64_t* row_out, cudaStream_t s) {
  if (n) k_locate<<<(n + 127) / 128, 128, 0, s>>>(sid, srow, N, list_off, K, q, n, cl_out, row_out);
}
void launch_gather_rows(const IndexView& ix, const uint64_t* rows, uint32_t n, float* out, cudaStream_t s) {
  const uint64_t t = (uint64_t)n * ix.dim;
  if (t) k_gather_rows<<<(unsigned)((t + 255) / 256), 256, 0, s>>>(ix, rows, n, out);
}
void launch_iota64(uint64_t* v, uint64_t n, cudaStream_t s) {
  if (n) k_iota64<<<(unsigned)((n + 255) / 256), 256, 0, s>>>(v, n);
}

}  // namespace hivf
