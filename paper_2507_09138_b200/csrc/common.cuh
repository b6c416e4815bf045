// common.cuh -- shared constants, PTX wrappers and exact-arithmetic helpers
// for the hivf kernels (sm_100a only).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#ifndef __CUDA_ARCH__
#define HIVF_HOST_ONLY 1
#endif

namespace hivf {

// ---- layout constants ------------------------------------------------------
// Lists live in HBM tile-major, chunk-major inside a tile: list c's rows
// [R_c, R_c+n_c) (list order) form tiles of kTileRows rows (the last one may
// be short, nt rows); a tile occupies nt*dpad floats, and inside it the 16-dim
// chunk `ch` of its rows is one contiguous plane of nt*64 B.  Inside a 64-B
// row slice the four 16-B groups are XOR-swizzled by ((row>>1)&3).  So a
// (full tile x 64 dims) pipeline stage of the tensor-core scan is ONE
// contiguous 32 KB span already in the canonical SWIZZLE_64B K-major UMMA
// layout, and a warp reading 8 consecutive rows at one group is
// bank-conflict-free in shared memory.
constexpr int kChunk = 16;            // dims per chunk (64 B per row slice)
constexpr uint32_t kTileRows = 128;   // rows per layout tile (= the MMA's M)
constexpr int kQMax = 16;             // queries per scan work item
constexpr int kKP = 32;               // candidates kept per (query, segment)
constexpr int kScanWarps = 8;         // consumer warps per scan CTA
constexpr int kRowsPerWarp = 64;
constexpr int kRowBlock = kScanWarps * kRowsPerWarp;  // 512 rows per row-block
constexpr int kStages = 4;
constexpr int kStageBytes = kRowBlock * kChunk * 4;  // 32 KB
constexpr uint32_t kNoRow = 0xffffffffu;

// Rows in the tile that starts at (tile-aligned) list row r0.
__host__ __device__ inline uint64_t tile_rows(uint64_t n_rows, uint64_t r0) {
  const uint64_t left = n_rows - r0;
  return left < kTileRows ? left : kTileRows;
}
// Float offset (from the list base) of chunk `ch` of the tile starting at row r0.
__host__ __device__ inline uint64_t tile_chunk_offset(uint64_t n_rows, uint32_t dpad, uint64_t r0,
                                                      uint32_t ch) {
  return r0 * dpad + (uint64_t)ch * tile_rows(n_rows, r0) * kChunk;
}
// Float offset of element d of list row r.
__host__ __device__ inline uint64_t swz_offset(uint64_t list_base_floats, uint64_t n_rows, uint64_t r,
                                               uint32_t d, uint32_t dpad) {
  const uint32_t ch = d >> 4, e = d & 15;
  const uint32_t g = (e >> 2) ^ ((uint32_t)(r >> 1) & 3u);
  const uint64_t r0 = r - r % kTileRows;
  return list_base_floats + tile_chunk_offset(n_rows, dpad, r0, ch) + (r - r0) * kChunk + g * 4 + (e & 3);
}

// ---- error bound of the fp32 filter -------------------------------------------
// |d32 - delta| <= eps(D) * (|x| + |q|)^2 + abs_floor, where d32 is the fp32
// expansion distance (|x|^2 + |q|^2 - 2 x.q, sequential FMA dot) and delta the
// reference's double (embedding.hpp:27-34).  Derivation in DESIGN.md; the
// factor 2 is headroom over the analytic bound.
__host__ __device__ inline double filter_eps(uint32_t dim) {
  const double u = 5.9604644775390625e-08;      // 2^-24
  const double u53 = 1.1102230246251565e-16;    // 2^-53
  const double Du = (double)dim * u;
  return 2.0 * (Du / (1.0 - Du) + 3.0001 * u + (3.0 * dim + 6.0) * u53) * 1.001;
}
__host__ __device__ inline double filter_abs(uint32_t dim) { return 1e-36 * (dim + 8.0); }

// Per-(query, list) filter bound from the IndexView coefficients (rounded up).
template <typename View>
__device__ __forceinline__ float seg_bound(const View& ix, float qn, float xn) {
  const double q = qn, x = xn;
  return __double2float_ru(ix.e_a * q * x + ix.e_b * (q * q + x * x) + ix.e_c);
}

// ---- exact reference arithmetic (embedding.hpp:27-34) -------------------------
// d = (double)a - (double)b ; acc += d * d  -- sequential, every op rounded,
// never contracted into an FMA.
__device__ __forceinline__ double exact_step(double acc, float a, float b) {
  const double d = __dsub_rn((double)a, (double)b);
  return __dadd_rn(acc, __dmul_rn(d, d));
}
// Same step with the query element already widened (exact: every float is a
// double), one conversion fewer per dim: a single chain measured 20.7 vs
// 29.5 cycles per dim on B200 (fp64 chains are latency-bound).
__device__ __forceinline__ double exact_step(double acc, double a, float b) {
  const double d = __dsub_rn(a, (double)b);
  return __dadd_rn(acc, __dmul_rn(d, d));
}

// Exact distance of one row to the query in smem, loads double-buffered 32
// dims (8 x 16 B) ahead so the memory latency overlaps the sequential fp64
// chain.  load(g) returns dims 4g..4g+3 of the row (zero past dim).
template <typename Q, typename Load>
__device__ __forceinline__ double exact_row_pipelined(uint32_t dim, const Q* qsh, Load load) {
  const uint32_t ng = (dim + 3) / 4;
  double acc = 0.0;
  float4 cur[8], nxt[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) cur[e] = (uint32_t)e < ng ? load(e) : make_float4(0.f, 0.f, 0.f, 0.f);
  for (uint32_t g0 = 0; g0 < ng; g0 += 8) {
#pragma unroll
    for (int e = 0; e < 8; ++e)
      nxt[e] = g0 + 8 + e < ng ? load(g0 + 8 + e) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const uint32_t d = (g0 + e) * 4;
      if (d + 0 < dim) acc = exact_step(acc, qsh[d + 0], cur[e].x);
      if (d + 1 < dim) acc = exact_step(acc, qsh[d + 1], cur[e].y);
      if (d + 2 < dim) acc = exact_step(acc, qsh[d + 2], cur[e].z);
      if (d + 3 < dim) acc = exact_step(acc, qsh[d + 3], cur[e].w);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) cur[e] = nxt[e];
  }
  return acc;
}

// Warm a line into L1 ahead of a latency-bound sequential consumer (the exact
// fp64 chains read their rows 128 B at a time).
__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}

// ---- orderable float keys ----------------------------------------------------
__device__ __forceinline__ uint32_t f2key(float f) {
  uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key2f(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

// (dist, id) total order of the reference (vector_index.hpp:41-44)
__device__ __forceinline__ bool pair_less(double da, uint64_t ia, double db, uint64_t ib) {
  return da < db || (da == db && ia < ib);
}

// ---- mbarrier / bulk-copy PTX --------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_barrier_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.release.cta.shared::cta.b64 st, [%0];\n\t}" ::"r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile(
      "{\n\t.reg .b64 st;\n\t"
      "mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 st, [%0], %1;\n\t}" ::"r"(
          smem_u32(bar)),
      "r"(bytes)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// Same, for waiters off the critical path: the suspend-time hint lets the
// hardware park the warp until the phase completes (or ~the hint elapses)
// instead of re-issuing try_wait, so spinning consumers do not steal issue
// slots from the producer / MMA warps sharing their SM sub-partition.
__device__ __forceinline__ void mbar_wait_parked(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITP_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAITP_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity), "r"(0x989680)
      : "memory");
}
// 1-D bulk async copy global -> shared, completion reported as tx bytes on bar.
__device__ __forceinline__ void bulk_g2s(void* smem_dst, const void* gmem_src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(smem_dst)),
      "l"(gmem_src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void named_bar_sync(uint32_t id, uint32_t nthreads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
}

__device__ __forceinline__ float4 lds128(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}

}  // namespace hivf
