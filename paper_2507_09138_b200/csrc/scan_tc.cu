// scan_tc.cu -- K2 on the 5th-gen tensor cores: grouped inverted-list scan
// with tcgen05.mma (kind::tf32), TMEM accumulators and a bulk-copy/mbarrier
// pipeline.  Same work items and same output contract as scan.cu (32 best
// (dist32, row) per (query, segment) + drop threshold), so finalize.cu /
// items.cu re-rank its candidates exactly as for the FFMA kernel.
//
// Replaces the inner loop of ivf::search_clusters
// (/root/reference/proj/src/vector_index.cpp:302-306).  Why tensor cores: the
// FFMA scan (scan.cu) is issue-bound at ~50% of HBM (profiles/); here the
// B x rows dot products run on tcgen05 and the SMs only stream + select.
//
// Precision: error-compensated split.  The tensor core reads every fp32
// operand x as hi = tf32(x) (its own conversion, measured once per process by
// hivf_tc_probe: truncation or RNE); splitter warps write lo = x - hi (exact in
// fp32) for the list rows, the query group carries [q ; lo(q)] rows, and each
// 8-dim k-step issues A x [q ; lo(q)] (N = 2 npad: hi*hi and hi*lo in separate
// TMEM columns) and lo(A) x q (accumulated onto hi*hi; lo(A) is written by the
// splitters straight into TMEM and read from there by the MMA, so the split
// costs one extra smem read of the stage and no smem writes).  The
// dropped lo*lo term and the tf32 conversion of lo are each <= 2^-20 per
// element, so by Cauchy-Schwarz the operand error is <= 4*2^-20 |x||q|; the
// fp32 tensor-core accumulation is bounded at 4x the round-to-nearest bound
// per MMA step ((3D/2) * 2^-22 |x||q|).  finalize.cu uses that bound
// (IndexView::e_*), so every id/distance is still the reference's exact double.
//
// CTA (1 per SM, persistent) = 6 warps:
//   warp 0   producer: ONE 1-D bulk copy per (128-row tile x 64 dims) stage --
//            contiguous in the tile-major HBM layout, whose 16-B XOR swizzle
//            IS the canonical SWIZZLE_64B K-major UMMA layout -- into a deep
//            ring (3-8 stages of 4 chunks = 64 dims) sized from the smem left
//            after the resident query group
//   warp 1   TMEM allocator + single-thread MMA issuer: per 128-row tile and
//            per 8-dim k-step one tcgen05.mma M=128 x N=ceil8(nq) x K=8 into
//            a double-buffered TMEM accumulator; tcgen05.commit frees smem
//            stages and publishes finished tiles
//   warps 2-5 splitters: lo(A) of each stage, one row per thread, into TMEM
//   warps 6-9 epilogue: tcgen05.ld of the tile (one row per thread, one column
//            per query), fp32 expansion distance, per-warp register top-32 per
//            query; at item end a bitonic merge across the four warps.
#include <mutex>
#include <algorithm>
#include <cstdlib>
#include <cfloat>

#include <cuda_fp16.h>

#include "common.cuh"
#include "kernels.h"

namespace hivf {

namespace {

constexpr unsigned FULL = 0xffffffffu;
constexpr int kTcTile = 128;       // rows per MMA tile (M)
constexpr int kTcCps = 4;          // 16-dim chunks per pipeline stage (64 dims)
constexpr int kTcMaxA = 8;         // max depth of the A landing ring
constexpr int kTcLo = 4;           // depth of the A_lo ring (in TMEM, 64 columns per slot)
constexpr int kMergeQ = 16;        // queries per round of the item-end cross-warp merge (wide: 8)
constexpr int kItemQ = 4;          // published work items in flight (producer runs ahead)
constexpr int kTcChunkBytes = kTcTile * kChunk * 4;       // 8 KB
constexpr int kTcStageBytes = kTcCps * kTcChunkBytes;     // 32 KB
constexpr int kTcSplitWarps = 4;
constexpr int kTcEpiWarps = 4;
constexpr int kTcThreads = (2 + kTcSplitWarps + kTcEpiWarps) * 32;
constexpr uint32_t kTmemAcc = 128;  // split mode: 2 accumulator buffers x 64 columns ([hi*hi|hi*lo]), A_lo after
constexpr int kAccMax = 8;          // single mode: up to 8 x 64 accumulator columns (the A_lo ring is unused)
constexpr uint32_t kTmemLoCols = kTcCps * kChunk;            // 64 columns of A_lo per slot
constexpr uint32_t kTmemCols = 512;  // 128 accumulator + kTcLo x 64 lo columns (pow2)

struct TcParams {
  IndexView ix;
  QueryView qv;
  const ScanItem* items;
  const uint32_t* n_items;
  uint32_t* work_ctr;
  const uint32_t* sorted_pairs;
  const uint32_t* pair_query;
  float* out_d;
  uint32_t* out_row;
  float* out_thr;
  uint32_t* out_n;
  uint32_t qmax;  // queries per item (8..32)
  uint32_t sa;    // A landing-ring depth (16 KB stages)
  int conv;       // tensor-core tf32 conversion (0 trunc, 1 RNE)
  int variant;    // debug: bit0 skip split math, bit1 skip lo(A) MMA, bit2 skip all MMAs, bit3 skip odd k-steps (results then inexact), bit4 spin-wait epilogue, bit5 skip the pair scan's tile epilogue
  int split;      // 1: 3-pass split precision, 0: single-pass tf32 (looser bound)
  unsigned long long* prof;  // debug: per-CTA stall counters [gridDim.x][16] (nullptr = off)
  // shared per-query drop bound: U_q = min over
  // finished items of their k-th smallest (d^ + E); rows with d^ >= U_q + E
  // cannot reach the top-k and are not kept.  topk == 0 disables it.
  float* qbound;
  uint32_t topk;
  // 0: the bounds are fixed inputs (node-split items: the heap's worst before
  // the sub-stage -- updating them from later clusters would change the
  // reference's per-cluster `changed` flags), 1: items publish their k-th
  uint32_t bound_update;
  // wide mode (k_scan_tc<64|128>): query groups of up
  // to 64 / 128 streamed with the list stages from a restaged copy (launch_stage_wide):
  // group block at staged row (pair0 + qshift[list]), chunk-major [ch][npad
  // rows][64 B] in the SWIZZLE_64B pattern, so a stage's query slice is one copy
  const uint8_t* qstage;
  const uint32_t* qshift;
};

// ---- tcgen05 PTX wrappers ------------------------------------------------------
__device__ __forceinline__ uint64_t sw64_kmajor_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFFu);  // start address (16-B units)
  d |= (uint64_t)1u << 16;                  // LBO (unused for swizzled K-major)
  d |= (uint64_t)(512u >> 4) << 32;         // SBO: 8 rows x 64 B between row groups
  d |= (uint64_t)1u << 46;                  // descriptor version (sm_100)
  d |= (uint64_t)4u << 61;                  // SWIZZLE_64B
  return d;
}
__device__ __forceinline__ uint32_t tf32_idesc(uint32_t n) {
  return (1u << 4)            // D = f32
         | (2u << 7)          // A = tf32
         | (2u << 10)         // B = tf32
         | ((n >> 3) << 17)   // N
         | ((uint32_t)(kTcTile >> 4) << 24);  // M = 128
}
__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
// kind::f16 with fp16 operands (A, B type 0) and an f32 accumulator: K = 16 per
// instruction, i.e. the same 32 B of each operand row per k-step as tf32's K = 8
__device__ __forceinline__ uint32_t f16_idesc_m(uint32_t m, uint32_t n) {
  return (1u << 4) | ((n >> 3) << 17) | ((m >> 4) << 24);
}
__device__ __forceinline__ void mma_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_f16_elect(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                              uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

// One pipeline stage's MMAs (cn <= 4 chunks x 2 k-steps) in ONE warp-collective
// asm block: elect.sync once, descriptors advanced with 64-bit adds inside the
// block (A: +512 per 8 KB chunk, +2 per 32-B k-step; B: +qs per chunk), so the
// issuing warp moves its operands to uniform registers once per stage instead
// of once per instruction (the per-instruction R2UR / elect sequence cost
// ~130 cycles per MMA, profiles/r2_mma_rate.txt).  acc0: accumulate into D on
// the stage's first k-step.
#define HIVF_MMA_STAGE8(CG, KIND)                                                            \
  asm volatile(                                                                            \
      "{\n\t.reg .pred p, t, e, c1, c2, c3;\n\t.reg .b64 a, b, bq, q;\n\t"                 \
      "setp.ne.b32 p, %4, 0;\n\t"                                                          \
      "setp.eq.u32 t, 0, 0;\n\t"                                                           \
      "cvt.u64.u32 q, %6;\n\t"                                                             \
      "elect.sync _|e, 0xffffffff;\n\t"                                                    \
      "setp.gt.and.u32 c1, %5, 1, e;\n\t"                                                  \
      "setp.gt.and.u32 c2, %5, 2, e;\n\t"                                                  \
      "setp.gt.and.u32 c3, %5, 3, e;\n\t"                                                  \
      "@e tcgen05.mma.cta_group::" CG ".kind::" KIND " [%0], %1, %2, %3, p;\n\t"                \
      "add.s64 a, %1, 2;\n\tadd.s64 b, %2, 2;\n\t"                                         \
      "@e tcgen05.mma.cta_group::" CG ".kind::" KIND " [%0], a, b, %3, t;\n\t"                  \
      "add.s64 a, %1, 512;\n\tadd.s64 bq, %2, q;\n\t"                                      \
      "@c1 tcgen05.mma.cta_group::" CG ".kind::" KIND " [%0], a, bq, %3, t;\n\t"                \
      "add.s64 a, a, 2;\n\tadd.s64 b, bq, 2;\n\t"                                          \
      "@c1 tcgen05.mma.cta_group::" CG ".kind::" KIND " [%0], a, b, %3, t;\n\t"                 \
      "add.s64 a, %1, 1024;\n\tadd.s64 bq, bq, q;\n\t"                                     \
      "@c2 tcgen05.mma.cta_group::" CG ".kind::" KIND " [%0], a, bq, %3, t;\n\t"                \
      "add.s64 a, a, 2;\n\tadd.s64 b, bq, 2;\n\t"                                          \
      "@c2 tcgen05.mma.cta_group::" CG ".kind::" KIND " [%0], a, b, %3, t;\n\t"                 \
      "add.s64 a, %1, 1536;\n\tadd.s64 bq, bq, q;\n\t"                                     \
      "@c3 tcgen05.mma.cta_group::" CG ".kind::" KIND " [%0], a, bq, %3, t;\n\t"                \
      "add.s64 a, a, 2;\n\tadd.s64 b, bq, 2;\n\t"                                          \
      "@c3 tcgen05.mma.cta_group::" CG ".kind::" KIND " [%0], a, b, %3, t;\n\t}" ::"r"(d_tmem), \
      "l"(a0), "l"(b0), "r"(idesc), "r"(acc0), "r"(cn), "r"(qs))
__device__ __forceinline__ void mma_stage8_tf32(uint32_t d_tmem, uint64_t a0, uint64_t b0, uint32_t idesc,
                                                uint32_t acc0, uint32_t cn, uint32_t qs) {
  HIVF_MMA_STAGE8("1", "tf32");
}
__device__ __forceinline__ void mma_stage8_f16(uint32_t d_tmem, uint64_t a0, uint64_t b0, uint32_t idesc,
                                               uint32_t acc0, uint32_t cn, uint32_t qs) {
  HIVF_MMA_STAGE8("1", "f16");
}
// the same for a CTA pair (cta_group::2, issued by the leader CTA's MMA warp)
__device__ __forceinline__ void mma2_stage8_tf32(uint32_t d_tmem, uint64_t a0, uint64_t b0, uint32_t idesc,
                                                 uint32_t acc0, uint32_t cn, uint32_t qs) {
  HIVF_MMA_STAGE8("2", "tf32");
}
__device__ __forceinline__ void mma2_stage8_f16(uint32_t d_tmem, uint64_t a0, uint64_t b0, uint32_t idesc,
                                                uint32_t acc0, uint32_t cn, uint32_t qs) {
  HIVF_MMA_STAGE8("2", "f16");
}
__device__ __forceinline__ void mma_tf32_ta(uint32_t d_tmem, uint32_t a_tmem, uint64_t b,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate));
}
// Warp-collective variants: every lane executes the asm with the same
// (warp-uniform) operands, elect.sync picks the single issuing lane.
__device__ __forceinline__ void mma_tf32_elect(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                               uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma_tf32_ta_elect(uint32_t d_tmem, uint32_t a_tmem, uint64_t b,
                                                  uint32_t idesc) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.eq.u32 p, %0, %0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc));
}
__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
          smem_u32(bar))
      : "memory");
}
#define TMEM_ST32(taddr, r)                                                                    \
  asm volatile(                                                                                \
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,"  \
      "%13,%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};"     \
      ::"r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]),         \
      "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]),          \
      "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]), "r"(r[19]),      \
      "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]),      \
      "r"(r[27]), "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31]))
__device__ __forceinline__ void tmem_wait_st() {
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

#define TMEM_LD32(taddr, r)                                                                    \
  asm volatile(                                                                                \
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13," \
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"      \
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),    \
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),             \
        "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]),          \
        "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),          \
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]),          \
        "=r"(r[31])                                                                            \
      : "r"(taddr))

__device__ __forceinline__ void tmem_wait_ld() {
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// ---- the kernel ------------------------------------------------------------------
// smem carve-out (1024-B aligned): per stage [A_hi 16K | A_lo 16K | B_hi | B_lo],
// then the resident (unsplit) query group, then the mbarriers.
constexpr float kInfF = __builtin_inff();
// Drop bound for a query from its shared upper bound u on the true k-th
// distance: rows with d^ >= u + E (rounded up, plus two ulps) satisfy
// d^ - E > u >= tau, so they are neither top-k nor finalize candidates.
__device__ __forceinline__ float drop_bound(float u, float E) {
  const float g = __fadd_ru(u, E);
  return nextafterf(nextafterf(g, kInfF), kInfF);
}
__device__ __forceinline__ float tf32_trunc(float x) {
  return __uint_as_float(__float_as_uint(x) & 0xffffe000u);
}
// The tensor core's own fp32 -> tf32 operand conversion, as measured by
// hivf_tc_probe (mode 0: truncation, 1: round-to-nearest-even).
__device__ __forceinline__ float tf32_conv(float x, int mode) {
  if (mode == 0) return tf32_trunc(x);
  const uint32_t u = __float_as_uint(x);
  if ((u & 0x7f800000u) == 0x7f800000u) return x;  // inf / nan untouched
  const uint32_t r = (u + 0xfffu + ((u >> 13) & 1u)) & 0xffffe000u;
  return __uint_as_float(r);
}

// fp16 filter copy (IndexView::vech): list
// c's filter rows (dpf floats each), and the distance's dot coefficient
// -2 2^-(e_q + e_l) (exact power of 2; -2 on the fp32 copy).  0 marks a query
// whose scale is out of range: its segments report no candidates and a -inf
// threshold, so finalize re-scans them exactly.
__device__ __forceinline__ const float* filter_base(const IndexView& ix, uint32_t c, uint64_t lbeg) {
  return ix.vech ? ix.vech + lbeg * ix.dpf : list_base(ix, c, lbeg);
}
__device__ __forceinline__ float dot_coef(const IndexView& ix, const QueryView& qv, uint32_t qi, uint32_t c) {
  return ix.vech ? -2.f * qv.qsc[qi] * ix.lsc[c] : -2.f;
}
// a query is out of the fp16 filter's range (its coefficient is 0)
__device__ __forceinline__ bool coef_bad(float m2) { return m2 == 0.f; }
// fp16 query row: the 8 dims [8 gh, 8 gh + 8) of q 2^e_q (zero past dpad) as one 16-B granule
__device__ __forceinline__ uint4 h16_granule(const float* qrow, uint32_t dpad, uint32_t gh, float up) {
  __align__(16) __half h[8];
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    const uint32_t d = gh * 8 + p * 4;
    const float4 v = d < dpad ? *reinterpret_cast<const float4*>(qrow + d) : make_float4(0.f, 0.f, 0.f, 0.f);
    h[p * 4 + 0] = __float2half_rn(v.x * up);
    h[p * 4 + 1] = __float2half_rn(v.y * up);
    h[p * 4 + 2] = __float2half_rn(v.z * up);
    h[p * 4 + 3] = __float2half_rn(v.w * up);
  }
  return *reinterpret_cast<const uint4*>(h);
}
// the query's up-scale 2^e_q (1 when out of range: its results are discarded)
__device__ __forceinline__ float h16_up(const QueryView& qv, uint32_t qi) {
  const float sc = qv.qsc[qi];
  return sc > 0.f ? 1.f / sc : 1.f;
}

// debug profiling (P.prof != nullptr): cycles spent in selected waits, per CTA
#define TC_PROF_T0() const long long _t0 = P.prof ? clock64() : 0
#define TC_PROF_ADD(slot) \
  if (P.prof) atomicAdd(&P.prof[blockIdx.x * 16 + (slot)], (unsigned long long)(clock64() - _t0))

// (d^, row) order of the candidate lists
__device__ __forceinline__ bool cand_less(float a, uint32_t ar, float b, uint32_t br) {
  return a < b || (a == b && ar < br);
}
// Ascending bitonic sort of one (d^, row) pair per lane across the warp.
__device__ __forceinline__ void warp_sort32(float& v, uint32_t& r, int lane) {
#pragma unroll
  for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
    for (int jj = kk >> 1; jj > 0; jj >>= 1) {
      const float pv = __shfl_xor_sync(FULL, v, jj);
      const uint32_t pr = __shfl_xor_sync(FULL, r, jj);
      const bool keep_min = ((lane & jj) == 0) == ((lane & kk) == 0);
      if (keep_min == cand_less(pv, pr, v, r)) {
        v = pv;
        r = pr;
      }
    }
  }
}
// Bitonic clean over lanes (xor steps from `top` down to 1): a bitonic
// sequence per (2*top)-lane block becomes ascending.
__device__ __forceinline__ void warp_clean(float& v, uint32_t& r, int lane, int top) {
#pragma unroll
  for (int jj = 16; jj > 0; jj >>= 1) {
    if (jj > top) continue;
    const float pv = __shfl_xor_sync(FULL, v, jj);
    const uint32_t pr = __shfl_xor_sync(FULL, r, jj);
    const bool keep_min = (lane & jj) == 0;
    if (keep_min == cand_less(pv, pr, v, r)) {
      v = pv;
      r = pr;
    }
  }
}

// One tile's candidates of a query pair (a: lanes' va, b: vb; inf = none)
// merged into the pair's 16-deep lists (lanes 0-15: a, 16-31: b).  Out of
// line: the per-pair loop around it stays small enough to unroll, so the
// lists stay in registers.
struct Cand {
  float v;
  uint32_t r;
};
__device__ __noinline__ Cand merge_pair16(float sa, float sb, uint32_t grow, float yv, uint32_t yr, int lane) {
  uint32_t ra = sa < kInfF ? grow : kNoRow, rb = sb < kInfF ? grow : kNoRow;
  if (__any_sync(FULL, ra != kNoRow)) warp_sort32(sa, ra, lane);
  if (__any_sync(FULL, rb != kNoRow)) warp_sort32(sb, rb, lane);
  // best 16 of query a in lanes 0-15, of query b in lanes 16-31
  const float sb16 = __shfl_sync(FULL, sb, lane & 15);
  const uint32_t rb16 = __shfl_sync(FULL, rb, lane & 15);
  const bool upper = lane >= 16;
  const float xv = upper ? sb16 : sa;
  const uint32_t xr = upper ? rb16 : ra;
  // per half: min(list, reversed candidates) is bitonic -> clean 8..1
  const float rv = __shfl_xor_sync(FULL, xv, 15);
  const uint32_t rr = __shfl_xor_sync(FULL, xr, 15);
  if (cand_less(rv, rr, yv, yr)) {
    yv = rv;
    yr = rr;
  }
  warp_clean(yv, yr, lane, 8);
  return Cand{yv, yr};
}

// Epilogue of k_scan_tc<128>: group h = 0 (warps 6-9) takes the item's
// queries 0..63, h = 1 (warps 2-5) queries 64..127 (TMEM columns
// 128*buffer + 64h + [0, 64)), each warp its lane quadrant of the tile.  Per
// warp and query the best 16 rows are kept: register slot s holds local
// queries 2s (lanes 0-15) and 2s+1 (lanes 16-31), ascending (d^, row); a tile's
// candidates of a query pair are bitonic-sorted across the warp and the best
// 16 merged into each half.  Item end: the four warps' 16-lists of a query
// merge into the (query, segment) output of 32 with the drop threshold
//   T = min(32nd kept when 32 are kept, each full warp list's 16th, the
//       smallest drop bound used)
// -- every row not reported has d^ >= T (rows a full 16-list dropped are >=
// its 16th; rows the bound dropped are >= that bound).
__device__ __forceinline__ void epilogue128(const TcParams& P, uint32_t tmem_base, uint32_t nacc, uint32_t& tb,
                                         uint32_t& tph, uint64_t* ifull, uint64_t* iempty, uint64_t* tfull,
                                         uint64_t* tempty, const ScanItem* s_item, const int* s_valid,
                                         float* md, uint32_t* mr, int warp, int lane) {
  __shared__ float s_gm[2][kTcEpiWarps][64];   // smallest drop bound used, per warp and query
  __shared__ float s_w16[2][kTcEpiWarps][64];  // 16th of a full warp list (else inf)
  const uint32_t quad = warp & 3;
  const uint32_t ew = (warp - 2) & 3;
  const uint32_t h = warp < 2 + kTcSplitWarps ? 1u : 0u;
  const bool upper = lane >= 16;
  float* gmd = md + h * (kTcEpiWarps * 8 * 16);
  uint32_t* gmr = mr + h * (kTcEpiWarps * 8 * 16);
  for (uint32_t i = 0;; ++i) {
    const uint32_t slot = i % kItemQ, iph = (i / kItemQ) & 1;
    mbar_wait_parked(&ifull[slot], iph);
    if (!s_valid[slot]) break;
    const ScanItem item = s_item[slot];
    const uint32_t nq = item.nq > 64 * h ? min(64u, item.nq - 64 * h) : 0u;
    // lane j: metadata of local queries j (m = 0) and 32 + j (m = 1)
    float w_qn2[2] = {0.f, 0.f}, w_E[2] = {0.f, 0.f}, w_m2[2] = {-2.f, -2.f};
    uint32_t w_qi[2] = {0, 0}, w_slot[2] = {0, 0};
#pragma unroll
    for (int m = 0; m < 2; ++m) {
      const uint32_t q = 32 * m + lane;
      if (q < nq) {
        const uint32_t pair = P.sorted_pairs[item.pair0 + 64 * h + q];
        w_qi[m] = P.pair_query[pair];
        w_qn2[m] = P.qv.qn2[w_qi[m]];
        w_slot[m] = pair * P.ix.s_max + item.seg;
        w_E[m] = seg_bound(P.ix, P.qv.qnorm[w_qi[m]], P.ix.maxnorm[item.list]);
        w_m2[m] = dot_coef(P.ix, P.qv, w_qi[m], item.list);
      }
    }
    const uint32_t ntiles = (item.nrows + kTcTile - 1) / kTcTile;
    const uint64_t lbeg = P.ix.list_off[item.list];
    float ld[32];
    uint32_t lr[32];
#pragma unroll
    for (int j = 0; j < 32; ++j) {
      ld[j] = kInfF;
      lr[j] = kNoRow;
    }
    float xn_next = 0.f;
    {
      const uint32_t srow0 = quad * 32 + lane;
      if (srow0 < item.nrows) xn_next = __ldg(P.ix.xnorm2 + lbeg + item.row0 + srow0);
    }
    float gmin[2] = {kInfF, kInfF};
    for (uint32_t t = 0; t < ntiles; ++t) {
      const uint32_t srow = t * kTcTile + quad * 32 + lane;
      const bool valid = srow < item.nrows;
      const float xn = xn_next;
      {
        const uint32_t nrow = srow + kTcTile;
        xn_next = (nrow < item.nrows) ? __ldg(P.ix.xnorm2 + lbeg + item.row0 + nrow) : 0.f;
      }
      {
        TC_PROF_T0();
        mbar_wait_parked(&tfull[tb], tph);
        if (lane == 0) TC_PROF_ADD(8);
      }
      tc_fence_after();
      const uint32_t ta = tmem_base + ((quad * 32) << 16) + tb * 128 + 64 * h;
      float gl[2] = {kInfF, kInfF};
#pragma unroll
      for (int m = 0; m < 2; ++m) {
        if (P.topk && 32 * m + lane < nq) {
          const float u = __ldcg(P.qbound + w_qi[m]);
          if (u < 3.0e38f) gl[m] = drop_bound(u, w_E[m]);
        }
        gmin[m] = fminf(gmin[m], gl[m]);
      }
      const uint32_t grow = (uint32_t)(lbeg + item.row0 + srow);
      // two halves of 32 query columns (32 accumulator registers live at a time);
      // the buffer is released after the second load
      if (nq == 0) {  // nothing of this item in the group's columns: free the buffer
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[tb]);
      }
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        if (32 * hh >= (int)nq) break;
        uint32_t acc[32];
        TMEM_LD32(ta + 32 * hh, acc);
        tmem_wait_ld();
        if (hh == 1 || nq <= 32) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&tempty[tb]);
        }
#pragma unroll
        for (int sl = 0; sl < 16; ++sl) {  // query pair (2sp, 2sp+1), sp = 16hh + sl
          const int sp = 16 * hh + sl;
          const int qa = 2 * sp, qb = 2 * sp + 1;
          if (qa >= (int)nq) break;
          const float qa2 = __shfl_sync(FULL, w_qn2[hh], qa & 31);
          const float qb2 = __shfl_sync(FULL, w_qn2[hh], qb & 31);
          const float ma = __shfl_sync(FULL, w_m2[hh], qa & 31);
          const float mb = __shfl_sync(FULL, w_m2[hh], qb & 31);
          const float va = valid ? __fmaf_rn(ma, __uint_as_float(acc[qa & 31]), __fadd_rn(xn, qa2)) : kInfF;
          const float vb = (valid && qb < (int)nq)
                               ? __fmaf_rn(mb, __uint_as_float(acc[qb & 31]), __fadd_rn(xn, qb2))
                               : kInfF;
          const float ga = __shfl_sync(FULL, gl[hh], qa & 31);
          const float gb = __shfl_sync(FULL, gl[hh], qb & 31);
          const float tha = fminf(__shfl_sync(FULL, ld[sp], 15), ga);
          const float thb = fminf(__shfl_sync(FULL, ld[sp], 31), gb);
          const bool ca = va < tha, cb = vb < thb;
          if (!__any_sync(FULL, ca || cb)) continue;
          const Cand m = merge_pair16(ca ? va : kInfF, cb ? vb : kInfF, grow, ld[sp], lr[sp], lane);
          ld[sp] = m.v;
          lr[sp] = m.r;
        }
      }
      if (++tb == nacc) {
        tb = 0;
        tph ^= 1;
      }
    }
    // ---- item end: merge the four warps' 16-lists of each query, 8 queries per round ----
    const long long _tm = P.prof ? clock64() : 0;
#pragma unroll
    for (int h0 = 0; h0 < 64; h0 += 8) {
      if (h0 >= (int)nq) break;
      named_bar_sync(2 + h, kTcEpiWarps * 32);  // the previous round's reads are done
      if (h0 == 0) {
        s_gm[h][ew][lane] = gmin[0];
        s_gm[h][ew][32 + lane] = gmin[1];
      }
#pragma unroll
      for (int jj = 0; jj < 8; ++jj) {
        const int q = h0 + jj;
        const int sp = q >> 1;
        if ((q & 1) == (int)upper) {
          gmd[(ew * 8 + jj) * 16 + (lane & 15)] = ld[sp];
          gmr[(ew * 8 + jj) * 16 + (lane & 15)] = lr[sp];
          if ((lane & 15) == 15) s_w16[h][ew][q] = lr[sp] != kNoRow ? ld[sp] : kInfF;
        }
      }
      named_bar_sync(2 + h, kTcEpiWarps * 32);
      for (uint32_t jj = ew; jj < 8 && h0 + jj < nq; jj += kTcEpiWarps) {
        const uint32_t q = h0 + jj;
        // warps 0|1 and 2|3: ascending 16 + reversed 16 = bitonic 32 -> clean
        float x, y;
        uint32_t xr, yr;
        {
          const int w0 = 0, w1 = 1;
          const int src = upper ? 31 - lane : lane;
          x = gmd[((upper ? w1 : w0) * 8 + jj) * 16 + (src & 15)];
          xr = gmr[((upper ? w1 : w0) * 8 + jj) * 16 + (src & 15)];
          y = gmd[((upper ? 3 : 2) * 8 + jj) * 16 + (src & 15)];
          yr = gmr[((upper ? 3 : 2) * 8 + jj) * 16 + (src & 15)];
        }
        warp_clean(x, xr, lane, 16);
        warp_clean(y, yr, lane, 16);
        // best 32 of both: min(x, reversed y) is bitonic -> clean
        const float ry = __shfl_sync(FULL, y, 31 - lane);
        const uint32_t ryr = __shfl_sync(FULL, yr, 31 - lane);
        if (cand_less(ry, ryr, x, xr)) {
          x = ry;
          xr = ryr;
        }
        warp_clean(x, xr, lane, 16);
        const uint32_t m = q >> 5;
        const uint32_t oslot = __shfl_sync(FULL, m ? w_slot[1] : w_slot[0], q & 31);
        const float Ej = __shfl_sync(FULL, m ? w_E[1] : w_E[0], q & 31);
        const uint32_t qij = __shfl_sync(FULL, m ? w_qi[1] : w_qi[0], q & 31);
        const bool bad = coef_bad(__shfl_sync(FULL, m ? w_m2[1] : w_m2[0], q & 31));
        P.out_d[(uint64_t)oslot * kKP + lane] = x;
        P.out_row[(uint64_t)oslot * kKP + lane] = xr;
        const uint32_t n_kept = __popc(__ballot_sync(FULL, xr != kNoRow));
        const uint32_t n_valid = bad ? 0u : n_kept;
        const float last = __shfl_sync(FULL, x, 31);
        const float gm = fminf(fminf(s_gm[h][0][q], s_gm[h][1][q]), fminf(s_gm[h][2][q], s_gm[h][3][q]));
        const float w16 = fminf(fminf(s_w16[h][0][q], s_w16[h][1][q]), fminf(s_w16[h][2][q], s_w16[h][3][q]));
        const float vk = __shfl_sync(FULL, x, (int)(P.topk ? P.topk - 1 : 0));
        if (lane == 0) {
          P.out_thr[oslot] = bad ? -kInfF : fminf(fminf(n_valid == kKP ? last : kInfF, gm), w16);
          P.out_n[oslot] = n_valid;
          if (P.bound_update && !bad && n_valid >= P.topk) {  // this item's k-th upper bound
            float u = __fadd_ru(vk, Ej);
            if (!(u > 0.f)) u = 0.f;
            atomicMin(reinterpret_cast<int*>(P.qbound + qij), __float_as_int(u));
          }
        }
      }
    }
    __syncwarp();
    if (lane == 0) {
      mbar_arrive(&iempty[slot]);
      if (P.prof) atomicAdd(&P.prof[blockIdx.x * 16 + 9], (unsigned long long)(clock64() - _tm));
    }
  }
}

// kQ = 0: narrow (resident query group of <= 32, split precision possible);
// kQ = 64 / 128: wide (query groups streamed with the list stages, single-pass
// tf32; 128: 16-deep per-warp lists, two epilogue groups of 64 queries)
template <int kQ>
__global__ void __launch_bounds__(kTcThreads, 1) k_scan_tc(TcParams P) {
  pdl_wait();
  // wide: warps 2-5 are a second epilogue group (queries kQ/2.. of the item)
  // instead of stagers/splitters; single-pass tf32 only
  constexpr bool kWide = kQ != 0;
  constexpr int kMQ = kWide ? 8 : kMergeQ;
  constexpr uint32_t kSB = kTcStageBytes + kTcCps * kQ * 64;  // ring stage bytes (A tile [+ query slice])
  constexpr uint32_t kAccW = kQ == 128 ? 128u : 64u;          // TMEM columns per accumulator buffer
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  const uint32_t dpad = P.ix.dpad;
  // list / query rows as the MMA reads them: fp32 (tf32) or the fp16 filter copy
  const bool h16 = P.ix.vech != nullptr;
  const uint32_t dpf = P.ix.dpf;
  const uint32_t nch = dpf / kChunk;
  const uint32_t qmax = P.qmax;
  const uint32_t SA = P.sa;
  const bool split = !kWide && P.split != 0;
  // TMEM accumulator ring: split mode shares TMEM with the A_lo ring; single
  // mode spreads over the whole 512 columns to absorb epilogue jitter
  const uint32_t nacc = split ? 2u : (kQ == 128 ? 4u : (uint32_t)kAccMax);
  const uint32_t qblk = (split ? 2 : 1) * qmax * 64;                // per chunk: [raw rows | lo rows]
  uint8_t* aring = smem;                                            // SA x kSB (raw A [| query slice])
  uint8_t* qsm = smem + SA * kSB;                                   // nch x qblk (narrow only)
  float* md = reinterpret_cast<float*>(qsm + (kWide ? 0 : (size_t)nch * qblk));  // merge scratch [groups][4][kMQ][32]
  constexpr int kGroups = kWide ? 2 : 1;
  uint32_t* mr = reinterpret_cast<uint32_t*>(md + kGroups * kTcEpiWarps * kMQ * 32);
  uint64_t* bars = reinterpret_cast<uint64_t*>(mr + kGroups * kTcEpiWarps * kMQ * 32);
  uint64_t* full = bars;                        // [SA] TMA -> splitter / MMA
  uint64_t* empty = bars + kTcMaxA;             // [SA] MMA -> TMA
  uint64_t* lfull = bars + 2 * kTcMaxA;         // [kTcLo] splitter -> MMA
  uint64_t* lempty = lfull + kTcLo;             // [kTcLo] MMA -> splitter
  uint64_t* tfull = lempty + kTcLo;             // [nacc] MMA -> epilogue
  uint64_t* tempty = tfull + kAccMax;           // [nacc] epilogue -> MMA
  uint64_t* ifull = tempty + kAccMax;                 // [kItemQ] producer -> all roles (item published)
  uint64_t* iempty = ifull + kItemQ;            // [kItemQ] roles -> producer (slot consumed)
  uint64_t* qfull = iempty + kItemQ;            // stagers -> MMA (query group staged)
  uint64_t* qempty = qfull + 1;                 // MMA commit -> stagers (query group free)
  __shared__ ScanItem s_item[kItemQ];
  __shared__ int s_valid[kItemQ];
  __shared__ uint32_t s_tmem;
  float (*s_qn2)[32] = reinterpret_cast<float (*)[32]>(qempty + 1);            // [kItemQ][32]
  uint32_t (*s_slot)[32] = reinterpret_cast<uint32_t (*)[32]>(s_qn2 + kItemQ);  // [kItemQ][32]
  float (*s_E)[32] = reinterpret_cast<float (*)[32]>(s_slot + kItemQ);            // [kItemQ][32]
  uint32_t (*s_qi)[32] = reinterpret_cast<uint32_t (*)[32]>(s_E + kItemQ);        // [kItemQ][32]
  float (*s_g)[32] = reinterpret_cast<float (*)[32]>(s_qi + kItemQ);              // [groups*4][32]
  float (*s_m2)[32] = reinterpret_cast<float (*)[32]>(s_g + kGroups * 4);         // [kItemQ][32] dot coefficients

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < SA; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < kTcLo; ++i) {
      mbar_init(&lfull[i], kTcSplitWarps);
      mbar_init(&lempty[i], 1);
    }
    for (int i = 0; i < kAccMax; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], kGroups * kTcEpiWarps);
    }
    for (int i = 0; i < kItemQ; ++i) {
      mbar_init(&ifull[i], 1);
      mbar_init(&iempty[i], 1 + kTcSplitWarps + kTcEpiWarps);
    }
    mbar_init(qfull, kTcSplitWarps);
    mbar_init(qempty, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s_tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = s_tmem;
  const uint32_t nstg = (nch + kTcCps - 1) / kTcCps;
  if (P.prof && threadIdx.x == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    P.prof[blockIdx.x * 16 + 5] = g;
  }

  // Every role walks the same item sequence: the producer claims work items
  // (atomic counter) into a kItemQ-deep queue of published items, so the bulk
  // copies of item i+1 start while the MMA / epilogue still finish item i (no
  // CTA-wide barrier between items).  ring positions are per role.
  uint32_t ra = 0, rpa = 0, rl = 0, rpl = 0;
  uint32_t tb = 0, tph = 0;   // TMEM accumulator ring
  if (warp == 0) {
    // ---------------- producer: claims items, list slices -> A ring ----------------
    // The next item is claimed while the current one streams (atomic at item
    // start, its descriptor and list bounds loaded after the first stages), so
    // no global round trip sits between the last copy of one item and the
    // first copy of the next.
    if (lane == 0) {
      const uint32_t n_items = *P.n_items;
      uint32_t it = atomicAdd(P.work_ctr, 1u);
      bool valid = it < n_items;
      ScanItem item{};
      uint64_t lbeg = 0, lend = 0;
      uint32_t qsh = 0;
      if (valid) {
        item = P.items[it];
        lbeg = P.ix.list_off[item.list];
        lend = P.ix.list_off[item.list + 1];
        if (kWide) qsh = P.qshift[item.list];
      }
      for (uint32_t i = 0;; ++i) {
        const uint32_t slot = i % kItemQ, iph = (i / kItemQ) & 1;
        {
          TC_PROF_T0();
          mbar_wait(&iempty[slot], iph ^ 1);
          TC_PROF_ADD(4);
        }
        s_item[slot] = item;
        s_valid[slot] = valid;
        mbar_arrive(&ifull[slot]);
        if (!valid) break;
        if (P.prof) P.prof[blockIdx.x * 16 + 7] += 1;
        const uint32_t it_n = atomicAdd(P.work_ctr, 1u);
        const bool valid_n = it_n < n_items;
        ScanItem item_n{};
        uint64_t lbeg_n = 0, lend_n = 0;
        uint32_t qsh_n = 0;
        uint32_t pf = valid_n ? 0 : 2;  // prefetch progress of the next item
        const uint32_t ntiles = (item.nrows + kTcTile - 1) / kTcTile;
        const uint64_t n_c = lend - lbeg;
        const float* lbase = filter_base(P.ix, item.list, lbeg);
        const uint32_t qbytes = kWide ? ((item.nq + 7) & ~7u) * 64 : 0;  // per chunk
        const uint8_t* qsrc = kWide ? P.qstage + (uint64_t)(item.pair0 + qsh) * dpf * 4 : nullptr;
        for (uint32_t t = 0; t < ntiles; ++t) {
          const uint32_t r0 = item.row0 + t * kTcTile;
          const uint32_t nr = min((uint32_t)kTcTile, item.nrows - t * kTcTile);
          for (uint32_t sg = 0; sg < nstg; ++sg) {
            const uint32_t c0 = sg * kTcCps, cn = min((uint32_t)kTcCps, nch - c0);
            const uint32_t a = ra, pa = rpa;
            {
              TC_PROF_T0();
              mbar_wait(&empty[a], pa ^ 1);
              TC_PROF_ADD(3);
            }
            const long long _tp = P.prof ? clock64() : 0;
            mbar_arrive_expect_tx(&full[a], cn * nr * kChunk * 4 + cn * qbytes);
            if (nr == kTcTile) {  // full tile: the stage is one contiguous span
              bulk_g2s(aring + a * kSB, lbase + tile_chunk_offset(n_c, dpf, r0, c0),
                       cn * kTcChunkBytes, &full[a]);
            } else {  // short last tile: its chunk planes are nr rows apart
              for (uint32_t c = 0; c < cn; ++c)
                bulk_g2s(aring + a * kSB + c * kTcChunkBytes,
                         lbase + tile_chunk_offset(n_c, dpf, r0, c0 + c), nr * kChunk * 4, &full[a]);
            }
            if (kWide)  // the group's query rows of these chunks (L2-resident restaged copy)
              bulk_g2s(aring + a * kSB + kTcStageBytes, qsrc + (uint64_t)c0 * qbytes, cn * qbytes, &full[a]);
            if (P.prof) atomicAdd(&P.prof[blockIdx.x * 16 + 14], (unsigned long long)(clock64() - _tp));
            if (++ra == SA) { ra = 0; rpa ^= 1; }
            if (pf == 1) {
              lbeg_n = P.ix.list_off[item_n.list];
              lend_n = P.ix.list_off[item_n.list + 1];
              if (kWide) qsh_n = P.qshift[item_n.list];
              pf = 2;
            } else if (pf == 0) {
              item_n = P.items[it_n];
              pf = 1;
            }
          }
        }
        if (pf == 0) {
          item_n = P.items[it_n];
          pf = 1;
        }
        if (pf == 1) {
          lbeg_n = P.ix.list_off[item_n.list];
          lend_n = P.ix.list_off[item_n.list + 1];
          if (kWide) qsh_n = P.qshift[item_n.list];
        }
        valid = valid_n;
        item = item_n;
        lbeg = lbeg_n;
        lend = lend_n;
        qsh = qsh_n;
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: tf32, single pass or 3-pass split ----------------
    // The whole warp walks the issue loop with warp-uniform operands (so the
    // descriptors live in uniform registers); elect.sync inside each tcgen05
    // instruction picks the one issuing lane -- no per-instruction waterfall.
    for (uint32_t i = 0;; ++i) {
      const uint32_t slot = i % kItemQ, iph = (i / kItemQ) & 1;
      mbar_wait(&ifull[slot], iph);
      if (!__shfl_sync(FULL, s_valid[slot], 0)) break;
      const uint32_t nq_i = __shfl_sync(FULL, s_item[slot].nq, 0);
      const uint32_t nrows_i = __shfl_sync(FULL, s_item[slot].nrows, 0);
      __syncwarp();
      if (lane == 0) mbar_arrive(&iempty[slot]);
      const uint32_t npad = (nq_i + 7) & ~7u;
      const uint32_t ntiles = (nrows_i + kTcTile - 1) / kTcTile;
      const uint32_t idesc2 = h16 ? f16_idesc_m(kTcTile, npad) : tf32_idesc(split ? 2 * npad : npad);
      const uint32_t idesc1 = tf32_idesc(npad);
      const uint64_t qdesc0 = sw64_kmajor_desc(smem_u32(qsm));
      const uint64_t adesc0 = sw64_kmajor_desc(smem_u32(aring));
      if (!kWide) {
        TC_PROF_T0();
        mbar_wait(qfull, i & 1);  // this item's query group is staged
        if (lane == 0) TC_PROF_ADD(0);
      }
      tc_fence_after();
      for (uint32_t t = 0; t < ntiles; ++t) {
        {
          TC_PROF_T0();
          mbar_wait(&tempty[tb], tph ^ 1);
          if (lane == 0) TC_PROF_ADD(2);
        }
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + tb * kAccW;  // this tile's accumulator columns
        for (uint32_t sg = 0; sg < nstg; ++sg) {
          const uint32_t cn = min((uint32_t)kTcCps, nch - sg * kTcCps);
          const uint32_t a = ra, pa = rpa, l = rl, pl = rpl;
          {
            TC_PROF_T0();
            if (split) mbar_wait(&lfull[l], pl);  // split done (implies A landed)
            else mbar_wait(&full[a], pa);
            if (lane == 0) TC_PROF_ADD(1);
          }
          tc_fence_after();
          const long long _ti = P.prof ? clock64() : 0;
          // descriptor start addresses are in 16-B units: +32 B == +2
          const uint64_t adesc = adesc0 + (uint64_t)(a * (kSB >> 4));
          // wide: this stage's query slice follows its A tile (64 rows per chunk)
          const uint64_t qdw = adesc + (uint64_t)(kTcStageBytes >> 4);
          const uint32_t alo = tmem_base + kTmemAcc + l * kTmemLoCols;  // A_lo in TMEM, lane = row
          const uint32_t c0 = sg * kTcCps;
          if (!(P.variant & 4) && !split && !(P.variant & 8)) {
            // single pass: the stage's MMAs in one asm block (operands to uniform registers once)
            const uint64_t qd0 = kWide ? qdw : qdesc0 + (uint64_t)(c0 * (qblk >> 4));
            const uint32_t qs = kWide ? npad * 4 : (qblk >> 4);
            if (h16) mma_stage8_f16(d_tmem, adesc, qd0, idesc2, sg != 0, cn, qs);
            else mma_stage8_tf32(d_tmem, adesc, qd0, idesc2, sg != 0, cn, qs);
          } else if (!(P.variant & 4)) {
#pragma unroll
            for (uint32_t c = 0; c < (uint32_t)kTcCps; ++c) {
              if (c >= cn) break;
              const uint64_t qd = kWide ? qdw + (uint64_t)(c * (npad * 4))  // npad*64 B per chunk
                                        : qdesc0 + (uint64_t)((c0 + c) * (qblk >> 4));
#pragma unroll
              for (uint32_t k2 = 0; k2 < 2; ++k2) {
                const uint64_t ad = adesc + (uint64_t)((c * kTcChunkBytes + k2 * 32) >> 4);
                const uint32_t accum = (sg | c | k2) != 0;
                // cols [0,npad): hi(A) hi(q);  cols [npad,2npad): hi(A) lo(q)
                if (!(P.variant & 8) || k2 == 0) {
                  if (h16) mma_f16_elect(d_tmem, ad, qd + 2 * k2, idesc2, accum);
                  else mma_tf32_elect(d_tmem, ad, qd + 2 * k2, idesc2, accum);
                }
                // cols [0,npad) += lo(A) hi(q), A from TMEM (8 columns per k-step)
                if (split && !(P.variant & 2))
                  mma_tf32_ta_elect(d_tmem, alo + c * 16 + k2 * 8, qd + 2 * k2, idesc1);
              }
            }
          }
          mma_commit_elect(&empty[a]);   // A slot reusable by TMA
          if (P.prof && lane == 0) {
            atomicAdd(&P.prof[blockIdx.x * 16 + 12], (unsigned long long)(clock64() - _ti));
            atomicAdd(&P.prof[blockIdx.x * 16 + 13], 1ull);
          }
          if (split) {
            mma_commit_elect(&lempty[l]);  // lo slot reusable by the splitters
            if (++rl == kTcLo) { rl = 0; rpl ^= 1; }
          }
          if (++ra == SA) { ra = 0; rpa ^= 1; }
        }
        mma_commit_elect(&tfull[tb]);
        if (++tb == nacc) {
          tb = 0;
          tph ^= 1;
        }
      }
      if (!kWide) mma_commit_elect(qempty);  // query group free once this item's MMAs retire
    }
  } else if (!kWide && warp < 2 + kTcSplitWarps) {
    // -------- stagers (query group of each item) + splitters (lo(A) rows -> TMEM) --------
    const uint32_t sw = warp - 2;                // 0..3
    const uint32_t quad = warp & 3;              // TMEM lane quadrant of this warp
    const uint32_t row = quad * 32 + lane;       // tile row owned by this thread
    const uint32_t swz = (row >> 1) & 3;
    const int cm = P.conv;
    const uint32_t ng = dpad / 4;                // float4 groups per query row
    for (uint32_t i = 0;; ++i) {
      const uint32_t slot = i % kItemQ, iph = (i / kItemQ) & 1;
      mbar_wait_parked(&ifull[slot], iph);
      if (!s_valid[slot]) break;
      const ScanItem item = s_item[slot];
      const uint32_t nq = item.nq;
      const uint32_t npad = (nq + 7) & ~7u;
      // rows n = sw + 4m of the query group belong to this warp; lane m < 8 resolves
      // row m's query id / output slot / |q|^2 (two dependent L2 loads, once)
      uint32_t my_qi = 0;
      {
        const uint32_t n = sw + 4 * lane;
        if (lane < 8 && n < nq) {
          const uint32_t pair = P.sorted_pairs[item.pair0 + n];
          my_qi = P.pair_query[pair];
          s_qn2[slot][n] = P.qv.qn2[my_qi];
          s_slot[slot][n] = pair * P.ix.s_max + item.seg;
          s_E[slot][n] = seg_bound(P.ix, P.qv.qnorm[my_qi], P.ix.maxnorm[item.list]);
          s_qi[slot][n] = my_qi;
          s_m2[slot][n] = dot_coef(P.ix, P.qv, my_qi, item.list);
        }
      }
      const long long _ts = P.prof ? clock64() : 0;
      if (i > 0) {
        TC_PROF_T0();
        mbar_wait_parked(qempty, (i - 1) & 1);  // previous item's MMAs retired
        if (lane == 0) TC_PROF_ADD(10);
      }
      const uint32_t nmine = npad > sw ? (npad - sw + 3) / 4 : 0;
      if (h16) {  // fp16 filter: the query rows scaled by 2^e_q, 8 dims per 16-B granule
        for (uint32_t m = 0; m < nmine; ++m) {
          const uint32_t n = sw + 4 * m;
          const uint32_t qi = __shfl_sync(FULL, my_qi, m & 7);
          const float up = n < nq ? h16_up(P.qv, qi) : 1.f;
          const float* qrow = P.qv.qs + (uint64_t)qi * dpad;
          for (uint32_t gh = lane; gh < dpf / 4; gh += 32) {
            const uint32_t ch = gh >> 2, g = gh & 3;
            const uint4 x = n < nq ? h16_granule(qrow, dpad, gh, up) : make_uint4(0u, 0u, 0u, 0u);
            *reinterpret_cast<uint4*>(qsm + ch * qblk + n * 64 + ((g ^ ((n >> 1) & 3)) << 4)) = x;
          }
        }
      }
      for (uint32_t m0 = 0; !h16 && m0 < nmine; m0 += 2) {
        for (uint32_t e0 = 0; e0 * 32 < ng; e0 += 8) {
          float4 v[2][8];
#pragma unroll
          for (uint32_t r = 0; r < 2; ++r) {
            const uint32_t m = m0 + r, n = sw + 4 * m;
            const uint32_t qi = __shfl_sync(FULL, my_qi, m & 7);
            const float* qrow = P.qv.qs + (uint64_t)qi * dpad;
#pragma unroll
            for (uint32_t e = 0; e < 8; ++e) {
              const uint32_t g4 = lane + 32 * (e0 + e);
              v[r][e] = (m < nmine && n < nq && g4 < ng) ? *reinterpret_cast<const float4*>(qrow + g4 * 4)
                                                          : make_float4(0.f, 0.f, 0.f, 0.f);
            }
          }
#pragma unroll
          for (uint32_t r = 0; r < 2; ++r) {
            const uint32_t m = m0 + r, n = sw + 4 * m;
            if (m >= nmine) break;
#pragma unroll
            for (uint32_t e = 0; e < 8; ++e) {
              const uint32_t g4 = lane + 32 * (e0 + e);
              if (g4 >= ng) break;
              const uint32_t ch = g4 >> 2, g = g4 & 3;
              uint8_t* blk = qsm + ch * qblk;
              const float4 x = v[r][e];
              *reinterpret_cast<float4*>(blk + n * 64 + ((g ^ ((n >> 1) & 3)) << 4)) = x;
              if (split) {
                const float4 lo = make_float4(x.x - tf32_conv(x.x, cm), x.y - tf32_conv(x.y, cm),
                                              x.z - tf32_conv(x.z, cm), x.w - tf32_conv(x.w, cm));
                const uint32_t nl = npad + n;  // lo rows follow the npad raw rows
                *reinterpret_cast<float4*>(blk + nl * 64 + ((g ^ ((nl >> 1) & 3)) << 4)) = lo;
              }
            }
          }
        }
      }
      fence_proxy_async_smem();  // generic-proxy writes -> visible to the tensor core
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(qfull);
        mbar_arrive(&iempty[slot]);
        if (P.prof) atomicAdd(&P.prof[blockIdx.x * 16 + 11], (unsigned long long)(clock64() - _ts));
      }
      const uint32_t ntiles = (item.nrows + kTcTile - 1) / kTcTile;
      for (uint32_t t = 0; split && t < ntiles; ++t) {
        for (uint32_t sg = 0; sg < nstg; ++sg) {
          const uint32_t cn = min((uint32_t)kTcCps, nch - sg * kTcCps);
          const uint32_t a = ra, pa = rpa, l = rl, pl = rpl;
          mbar_wait(&full[a], pa);
          mbar_wait(&lempty[l], pl ^ 1);
          tc_fence_after();
          const uint8_t* sb = aring + a * kTcStageBytes + row * 64;
          if (!(P.variant & 1))
#pragma unroll
          for (uint32_t h2 = 0; h2 < kTcCps / 2; ++h2) {  // 2 chunks (32 columns) per TMEM store
            uint32_t lo[32];
#pragma unroll
            for (uint32_t cc = 0; cc < 2; ++cc) {
              const uint32_t c = h2 * 2 + cc;
#pragma unroll
              for (uint32_t g = 0; g < 4; ++g) {
                float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
                if (c < cn) v = *reinterpret_cast<const float4*>(sb + c * kTcChunkBytes + ((g ^ swz) << 4));
                lo[cc * 16 + g * 4 + 0] = __float_as_uint(v.x - tf32_conv(v.x, cm));
                lo[cc * 16 + g * 4 + 1] = __float_as_uint(v.y - tf32_conv(v.y, cm));
                lo[cc * 16 + g * 4 + 2] = __float_as_uint(v.z - tf32_conv(v.z, cm));
                lo[cc * 16 + g * 4 + 3] = __float_as_uint(v.w - tf32_conv(v.w, cm));
              }
            }
            TMEM_ST32(tmem_base + ((quad * 32) << 16) + kTmemAcc + l * kTmemLoCols + h2 * 32, lo);
          }
          tmem_wait_st();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&lfull[l]);
          if (++ra == SA) { ra = 0; rpa ^= 1; }
          if (++rl == kTcLo) { rl = 0; rpl ^= 1; }
        }
      }
    }
  } else if constexpr (kQ == 128) {
    epilogue128(P, tmem_base, nacc, tb, tph, ifull, iempty, tfull, tempty, s_item, s_valid,
                reinterpret_cast<float*>(md), reinterpret_cast<uint32_t*>(mr), warp, lane);
  } else {
    // ---------------- epilogue warps ----------------
    // narrow: warps 6-9, queries 0..31.  wide: group h = 0 (warps 6-9) takes
    // queries 0..31, group h = 1 (warps 2-5) queries 32..63 -- TMEM columns
    // 32h.., each warp its lane quadrant
    const uint32_t quad = warp & 3;  // TMEM lane quadrant this warp may access
    const uint32_t ew = (warp - 2) & 3;
    const uint32_t h = (kWide && warp < 2 + kTcSplitWarps) ? 1u : 0u;
    for (uint32_t i = 0;; ++i) {
      const uint32_t slot = i % kItemQ, iph = (i / kItemQ) & 1;
      mbar_wait_parked(&ifull[slot], iph);
      if (!s_valid[slot]) break;
      const ScanItem item = s_item[slot];
      const uint32_t nq = kWide ? (item.nq > 32 * h ? min(32u, item.nq - 32 * h) : 0u) : item.nq;
      const uint32_t npad = (nq + 7) & ~7u;
      // wide: per-query metadata in registers (lane j = query 32h + j), loaded
      // here instead of by stager warps
      float w_qn2 = 0.f, w_E = 0.f, w_m2 = -2.f;
      uint32_t w_qi = 0, w_slot = 0;
      if (kWide && lane < nq) {
        const uint32_t pair = P.sorted_pairs[item.pair0 + 32 * h + lane];
        w_qi = P.pair_query[pair];
        w_qn2 = P.qv.qn2[w_qi];
        w_slot = pair * P.ix.s_max + item.seg;
        w_E = seg_bound(P.ix, P.qv.qnorm[w_qi], P.ix.maxnorm[item.list]);
        w_m2 = dot_coef(P.ix, P.qv, w_qi, item.list);
      }
      const uint32_t ntiles = (item.nrows + kTcTile - 1) / kTcTile;
      const uint64_t lbeg = P.ix.list_off[item.list];
      float ld[32];
      uint32_t lr[32];
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        ld[j] = __int_as_float(0x7f800000);
        lr[j] = kNoRow;
      }
      // row norms for tile t are fetched one tile ahead (global latency off the
      // critical path)
      float xn_next = 0.f;
      {
        const uint32_t srow0 = quad * 32 + lane;
        if (srow0 < item.nrows) xn_next = __ldg(P.ix.xnorm2 + lbeg + item.row0 + srow0);
      }
      float gmin = kInfF;  // lane j: smallest drop bound used for query j in this item
      for (uint32_t t = 0; t < ntiles; ++t) {
        const uint32_t srow = t * kTcTile + quad * 32 + lane;
        const bool valid = srow < item.nrows;
        const float xn = xn_next;
        {
          const uint32_t nrow = srow + kTcTile;
          xn_next = (nrow < item.nrows) ? __ldg(P.ix.xnorm2 + lbeg + item.row0 + nrow) : 0.f;
        }
        {
          TC_PROF_T0();
          if (P.variant & 16) mbar_wait(&tfull[tb], tph);
          else mbar_wait_parked(&tfull[tb], tph);
          if (lane == 0) TC_PROF_ADD(8);
        }
        tc_fence_after();
        uint32_t acc[32], acc2[32];
        TMEM_LD32(tmem_base + ((quad * 32) << 16) + tb * 64 + 32 * h, acc);
        if (split) TMEM_LD32(tmem_base + ((quad * 32) << 16) + tb * 64 + npad, acc2);
        tmem_wait_ld();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&tempty[tb]);
        if (++tb == nacc) {
          tb = 0;
          tph ^= 1;
        }
        // lane j: this tile's drop bound for query j (read through L2: other
        // CTAs lower it as their items finish).  After the tfull wait: the
        // stagers' per-item s_qi / s_E writes are ordered before it.
        float gl = kInfF;
        if (P.topk && lane < (int)nq) {
          const float u = __ldcg(P.qbound + (kWide ? w_qi : s_qi[slot][lane]));
          if (u < 3.0e38f) gl = drop_bound(u, kWide ? w_E : s_E[slot][lane]);
        }
        gmin = fminf(gmin, gl);
        const uint32_t grow = (uint32_t)(lbeg + item.row0 + srow);
#pragma unroll
        for (int j = 0; j < 32; ++j) {
          if (j >= (int)nq) break;
          const float dot = split ? __fadd_rn(__uint_as_float(acc[j]), __uint_as_float(acc2[j]))
                                  : __uint_as_float(acc[j]);
          const float qn2j = kWide ? __shfl_sync(FULL, w_qn2, j) : s_qn2[slot][j];
          const float m2j = kWide ? __shfl_sync(FULL, w_m2, j) : (h16 ? s_m2[slot][j] : -2.f);
          const float v = valid ? __fmaf_rn(m2j, dot, __fadd_rn(xn, qn2j))
                                : __int_as_float(0x7f800000);
          const float gj = __shfl_sync(FULL, gl, j);
          float th = fminf(__shfl_sync(FULL, ld[j], 31), gj);
          unsigned m = __ballot_sync(FULL, v < th);
          if (__popc(m) > 2) {
            // many candidates (early tiles): bitonic-sort this tile's 32 values and
            // min-merge them into the running top-32 (about 25 shuffle steps instead
            // of up to 32 serial insertions)
            float sv = (v < th) ? v : __int_as_float(0x7f800000);
            uint32_t sr = (v < th) ? grow : kNoRow;
#pragma unroll
            for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
              for (int jj = kk >> 1; jj > 0; jj >>= 1) {
                const float pv = __shfl_xor_sync(FULL, sv, jj);
                const uint32_t pr = __shfl_xor_sync(FULL, sr, jj);
                const bool keep_min = ((lane & jj) == 0) == ((lane & kk) == 0);
                const bool p_less = (pv < sv) || (pv == sv && pr < sr);
                if (keep_min == p_less) {
                  sv = pv;
                  sr = pr;
                }
              }
            }
            const float ov = __shfl_sync(FULL, sv, 31 - lane);
            const uint32_t orr = __shfl_sync(FULL, sr, 31 - lane);
            float xv = ld[j];
            uint32_t xr = lr[j];
            if (ov < xv || (ov == xv && orr < xr)) {
              xv = ov;
              xr = orr;
            }
#pragma unroll
            for (int jj = 16; jj > 0; jj >>= 1) {
              const float pv = __shfl_xor_sync(FULL, xv, jj);
              const uint32_t pr = __shfl_xor_sync(FULL, xr, jj);
              const bool keep_min = (lane & jj) == 0;
              const bool p_less = (pv < xv) || (pv == xv && pr < xr);
              if (keep_min == p_less) {
                xv = pv;
                xr = pr;
              }
            }
            ld[j] = xv;
            lr[j] = xr;
            continue;
          }
          while (m) {
            const int src = __ffs(m) - 1;
            const float cv = __shfl_sync(FULL, v, src);
            const uint32_t crow = __shfl_sync(FULL, grow, src);
            const bool before = (ld[j] < cv) || (ld[j] == cv && lr[j] < crow);
            const int pos = __popc(__ballot_sync(FULL, before));
            const float upd = __shfl_up_sync(FULL, ld[j], 1);
            const uint32_t upr = __shfl_up_sync(FULL, lr[j], 1);
            if (lane > pos) {
              ld[j] = upd;
              lr[j] = upr;
            } else if (lane == pos) {
              ld[j] = cv;
              lr[j] = crow;
            }
            th = fminf(__shfl_sync(FULL, ld[j], 31), gj);
            m &= ~(1u << src);
            m &= __ballot_sync(FULL, v < th);
          }
        }
      }
      // cross-warp merge through the dedicated scratch (the MMA / producer are
      // already on the next item), kMergeQ queries per round
      const long long _tm = P.prof ? clock64() : 0;
      float* gmd = md + h * (kTcEpiWarps * kMQ * 32);  // this group's scratch
      uint32_t* gmr = mr + h * (kTcEpiWarps * kMQ * 32);
      float (*gs_g)[32] = s_g + 4 * h;
#pragma unroll
      for (int h0 = 0; h0 < 32; h0 += kMQ) {
        if (h0 >= (int)nq) break;
        named_bar_sync(2 + h, kTcEpiWarps * 32);  // previous round's reads are done
        if (h0 == 0) gs_g[ew][lane] = gmin;
#pragma unroll
        for (int jj = 0; jj < kMQ; ++jj) {
          if (h0 + jj >= (int)nq) break;
          gmd[(ew * kMQ + jj) * 32 + lane] = ld[h0 + jj];
          gmr[(ew * kMQ + jj) * 32 + lane] = lr[h0 + jj];
        }
        named_bar_sync(2 + h, kTcEpiWarps * 32);
        for (uint32_t jj = ew; jj < (uint32_t)kMQ && h0 + jj < nq; jj += kTcEpiWarps) {
          const uint32_t j = h0 + jj;
          float v = gmd[jj * 32 + lane];
          uint32_t r = gmr[jj * 32 + lane];
          for (uint32_t w2 = 1; w2 < kTcEpiWarps; ++w2) {
            const float o = gmd[(w2 * kMQ + jj) * 32 + 31 - lane];
            const uint32_t orr = gmr[(w2 * kMQ + jj) * 32 + 31 - lane];
            if (o < v || (o == v && orr < r)) {
              v = o;
              r = orr;
            }
#pragma unroll
            for (int s = 16; s > 0; s >>= 1) {
              const float pv = __shfl_xor_sync(FULL, v, s);
              const uint32_t pr = __shfl_xor_sync(FULL, r, s);
              const bool keep_min = (lane & s) == 0;
              const bool p_less = (pv < v) || (pv == v && pr < r);
              if (keep_min == p_less) {
                v = pv;
                r = pr;
              }
            }
          }
          const uint32_t oslot = kWide ? __shfl_sync(FULL, w_slot, j) : s_slot[slot][j];
          const float Ej = kWide ? __shfl_sync(FULL, w_E, j) : s_E[slot][j];
          const uint32_t qij = kWide ? __shfl_sync(FULL, w_qi, j) : s_qi[slot][j];
          const float m2o = kWide ? __shfl_sync(FULL, w_m2, j) : s_m2[slot][j];
          const bool bad = h16 && coef_bad(m2o);
          P.out_d[(uint64_t)oslot * kKP + lane] = v;
          P.out_row[(uint64_t)oslot * kKP + lane] = r;
          const uint32_t n_kept = __popc(__ballot_sync(FULL, r != kNoRow));
          const uint32_t n_valid = bad ? 0u : n_kept;
          const float last = __shfl_sync(FULL, v, 31);
          // every row not kept has d^ >= the 32nd kept value (when 32 are kept)
          // or >= a drop bound this item used (bounds only decrease)
          const float gm = fminf(fminf(gs_g[0][j], gs_g[1][j]), fminf(gs_g[2][j], gs_g[3][j]));
          const float vk = __shfl_sync(FULL, v, (int)(P.topk ? P.topk - 1 : 0));
          if (lane == 0) {
            P.out_thr[oslot] = bad ? -kInfF : fminf(n_valid == kKP ? last : kInfF, gm);
            P.out_n[oslot] = n_valid;
            if (P.bound_update && !bad && n_valid >= P.topk) {  // this item's k-th upper bound
              float u = __fadd_ru(vk, Ej);
              if (!(u > 0.f)) u = 0.f;
              atomicMin(reinterpret_cast<int*>(P.qbound + qij), __float_as_int(u));
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&iempty[slot]);
        if (P.prof) atomicAdd(&P.prof[blockIdx.x * 16 + 9], (unsigned long long)(clock64() - _tm));
      }
    }
  }
  if (P.prof && threadIdx.x == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    P.prof[blockIdx.x * 16 + 6] = g;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(kTmemCols));
  }
}

}  // namespace

// ===========================================================================
// k_scan_pair: the wide scan on a CTA PAIR (cluster of 2, tcgen05 cta_group::2)
// for the densest batches -- query groups of up to 256 per list tile.
//
// One tcgen05.mma.cta_group::2 (issued by the leader CTA) multiplies M = 256
// rows x N = 256 queries x K = 8: CTA c supplies its own 128 rows (A) and
// queries [c*N/2, (c+1)*N/2) of the group (its half of B), and receives its
// 128 rows x all N columns in its own TMEM (layout measured by
// hivf_debug_tc2_dot).  So each SM streams 32 KB of list + 32 KB of query
// slice per 64-dim stage for 128 x 256 dot products -- half the SM ingress per
// dot product of the single-CTA 128-query scan, and one list pass for up to
// 256 probing queries.
//
// Rows: CTA c takes the 128-row tiles of parity c of each segment and reports
// them as candidate slot 2*segment + c (IndexView::seg_split = 2: finalize and
// repair address the same rows through slots_of / slot_row), so the two CTAs
// never merge candidates.  Work: pair p walks items p, p + P, ... (P pairs;
// both CTAs compute the same sequence, the work list is LPT-ordered).
//
// Per CTA, 10 warps: warp 0 producer (own A tile + own half of the query
// slice per stage into a 3-deep 64 KB ring); warp 1 = MMA issuer in the
// leader, relay in the peer (forwards "my stage landed" to the leader's pfull
// barrier); warps 2-9 = two epilogue groups of 128 queries with 8-deep
// per-warp lists (register slot s: queries 4s..4s+3, 8 lanes each).
// Cross-CTA barriers: the leader's tcgen05.commit multicasts `empty` and
// `tfull` to both CTAs; the peer's relay and epilogue arrive remotely on the
// leader's `pfull` / `tempty`.
// ===========================================================================
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t tf32_idesc_m(uint32_t m, uint32_t n) {
  return (1u << 4) | (2u << 7) | (2u << 10) | ((n >> 3) << 17) | ((m >> 4) << 24);
}
constexpr uint32_t kPairQ = 256;
constexpr int kPG = 4;                        // epilogue groups (4 warps each, one per TMEM lane quadrant)
constexpr int kPQ = (int)kPairQ / kPG;        // query columns per group
constexpr int kPairThreads = (2 + kPG * kTcEpiWarps) * 32;
// 64-dim pipeline stages (4 chunks), as the single-CTA scans.  32-dim stages
// (6 slots instead of 3, same bytes in flight) measured 1.5x slower at C3
// B=4096 (31.9 vs 20.8 ms): the pair's per-stage handshakes (relay,
// multicast commit) cost more than the finer slots win.
constexpr int kPCps = 4;
constexpr int kPairStageA = kPCps * kTcChunkBytes;  // 16 KB of list rows
constexpr int kPairQB = kPCps * 128 * 64;           // one CTA's half of a 256-query slice (16 KB)

__device__ __forceinline__ uint32_t mapa_peer(const void* p, uint32_t cta) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(cta));
  return r;
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
}
__device__ __forceinline__ void mbar_wait_cl(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAITC_%=:\n\t"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAITC_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void mma2_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma2_f16(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void mma2_commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}

// One tile's candidates of a query quad (4 queries, inf = not a candidate)
// merged into the quad's 8-deep lists (lanes 8j..8j+7: query j).
__device__ __noinline__ Cand merge_quad8(float s0, float s1, float s2, float s3, uint32_t grow, float yv,
                                         uint32_t yr, int lane) {
  float xv = kInfF;
  uint32_t xr = kNoRow;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float sv = j == 0 ? s0 : j == 1 ? s1 : j == 2 ? s2 : s3;
    uint32_t sr = sv < kInfF ? grow : kNoRow;
    if (__any_sync(FULL, sr != kNoRow)) warp_sort32(sv, sr, lane);
    const float bv = __shfl_sync(FULL, sv, lane & 7);  // best 8 of query j
    const uint32_t br = __shfl_sync(FULL, sr, lane & 7);
    if ((lane >> 3) == j) {
      xv = bv;
      xr = br;
    }
  }
  // per 8-lane group: min(list, reversed candidates) is bitonic -> clean 4..1
  const float rv = __shfl_xor_sync(FULL, xv, 7);
  const uint32_t rr = __shfl_xor_sync(FULL, xr, 7);
  if (cand_less(rv, rr, yv, yr)) {
    yv = rv;
    yr = rr;
  }
  warp_clean(yv, yr, lane, 4);
  return Cand{yv, yr};
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kPairThreads, 1) k_scan_pair(TcParams P) {
  pdl_wait();
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr uint32_t kSB = kPairStageA + kPairQB;  // A tile stage + this CTA's half query slice
  const bool h16 = P.ix.vech != nullptr;        // fp16 filter copy (dpf floats per row) or fp32
  const uint32_t dpf = P.ix.dpf;
  const uint32_t nch = dpf / kChunk;
  const uint32_t nstg = (nch + kPCps - 1) / kPCps;
  const uint32_t SA = P.sa;
  uint8_t* aring = smem;
  float* md = reinterpret_cast<float*>(smem + SA * kSB);  // merge scratch [kPG groups][4 warps][8 q][8]
  uint32_t* mr = reinterpret_cast<uint32_t*>(md + kPG * kTcEpiWarps * 8 * 8);
  // TMEM: 4 slots of 128 columns; a tile takes 1 slot (npad <= 128) or 2 (an
  // even-aligned pair; an odd slot is skipped), so tiles of <= 128 queries
  // get 4-deep accumulator buffering instead of 2
  __shared__ uint64_t full[kTcMaxA], empty[kTcMaxA], pfull[kTcMaxA], tfull[4], tempty[4];
  __shared__ uint64_t ifull[kItemQ], iempty[kItemQ];
  __shared__ ScanItem s_item[kItemQ];
  __shared__ int s_valid[kItemQ];
  __shared__ uint32_t s_tmem;
  __shared__ float s_gm[kPG][kTcEpiWarps][kPQ];
  __shared__ float s_w8[kPG][kTcEpiWarps][kPQ];
  // per-query metadata of the current item, [item parity][group][query]
  __shared__ float s_qn2[2][kPG][kPQ], s_E[2][kPG][kPQ];
  __shared__ uint32_t s_qi[2][kPG][kPQ], s_oslot[2][kPG][kPQ];
  __shared__ float s_m2[2][kPG][kPQ];  // dot coefficient (dot_coef)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t crank = cluster_rank();
  const bool leader = crank == 0;
  const uint32_t pair_id = blockIdx.x >> 1, n_pairs_grid = gridDim.x >> 1;
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < SA; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
      mbar_init(&pfull[i], 1);
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 2 * kPG * kTcEpiWarps);  // both CTAs' epilogue warps
    }
    for (int i = 0; i < kItemQ; ++i) {
      mbar_init(&ifull[i], 1);
      mbar_init(&iempty[i], 1 + kPG * kTcEpiWarps);
    }
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(kTmemCols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();  // barriers initialised and TMEM allocated in both CTAs
  tc_fence_after();
  const uint32_t tmem_base = s_tmem;
  if (P.prof && threadIdx.x == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    P.prof[blockIdx.x * 16 + 5] = g;
  }

  uint32_t ra = 0, rpa = 0;
  uint32_t tu = 0;  // TMEM slot uses so far: slot tu & 3, phase (tu >> 2) & 1
  if (warp == 0) {
    // ---------------- producer: static item sequence, own A tiles + own query half ----------------
    if (lane == 0) {
      const uint32_t n_items = *P.n_items;
      for (uint32_t i = 0;; ++i) {
        const uint32_t it = pair_id + i * n_pairs_grid;
        const bool valid = it < n_items;
        const uint32_t slot = i % kItemQ, iph = (i / kItemQ) & 1;
        mbar_wait(&iempty[slot], iph ^ 1);
        ScanItem item{};
        if (valid) item = P.items[it];
        s_item[slot] = item;
        s_valid[slot] = valid;
        mbar_arrive(&ifull[slot]);
        if (!valid) break;
        if (P.prof) P.prof[blockIdx.x * 16 + 7] += 1;
        const uint64_t lbeg = P.ix.list_off[item.list];
        const uint64_t n_c = P.ix.list_off[item.list + 1] - lbeg;
        const float* lbase = filter_base(P.ix, item.list, lbeg);
        const uint32_t npad = (item.nq + 15) & ~15u, hrows = npad / 2;
        const uint32_t qbytes = hrows * 64;  // per chunk, this CTA's half
        // the group's staged block: [half][ch][hrows][64 B]
        const uint8_t* qsrc = P.qstage + (uint64_t)(item.pair0 + P.qshift[item.list]) * dpf * 4 +
                              (uint64_t)crank * nch * qbytes;
        const uint32_t ntiles = (item.nrows + kTcTile - 1) / kTcTile;
        const uint32_t npt = (ntiles + 1) / 2;
        for (uint32_t pt = 0; pt < npt; ++pt) {
          const uint32_t t = 2 * pt + crank;  // this CTA's tile of the pair-tile
          const uint32_t r0 = item.row0 + t * kTcTile;
          const uint32_t nr = t < ntiles ? min((uint32_t)kTcTile, item.nrows - t * kTcTile) : 0u;
          for (uint32_t sg = 0; sg < nstg; ++sg) {
            const uint32_t c0 = sg * kPCps, cn = min((uint32_t)kPCps, nch - c0);
            const uint32_t a = ra, pa = rpa;
            {
              TC_PROF_T0();
              mbar_wait(&empty[a], pa ^ 1);
              TC_PROF_ADD(3);
            }
            mbar_arrive_expect_tx(&full[a], cn * nr * kChunk * 4 + cn * qbytes);
            if (nr == kTcTile) {
              bulk_g2s(aring + a * kSB, lbase + tile_chunk_offset(n_c, dpf, r0, c0), cn * kTcChunkBytes,
                       &full[a]);
            } else if (nr) {
              for (uint32_t c = 0; c < cn; ++c)
                bulk_g2s(aring + a * kSB + c * kTcChunkBytes, lbase + tile_chunk_offset(n_c, dpf, r0, c0 + c),
                         nr * kChunk * 4, &full[a]);
            }
            bulk_g2s(aring + a * kSB + kPairStageA, qsrc + (uint64_t)c0 * qbytes, cn * qbytes, &full[a]);
            if (++ra == SA) { ra = 0; rpa ^= 1; }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- leader: MMA issuer; peer: relay of landed stages ----------------
    const uint32_t pfull_peer0 = leader ? 0u : mapa_peer(&pfull[0], 0);
    const uint32_t tmask_idesc = 0;  // (unused)
    (void)tmask_idesc;
    for (uint32_t i = 0;; ++i) {
      const uint32_t slot = i % kItemQ, iph = (i / kItemQ) & 1;
      mbar_wait(&ifull[slot], iph);
      if (!__shfl_sync(FULL, s_valid[slot], 0)) break;
      const uint32_t nq_i = __shfl_sync(FULL, s_item[slot].nq, 0);
      const uint32_t nrows_i = __shfl_sync(FULL, s_item[slot].nrows, 0);
      __syncwarp();
      if (lane == 0) mbar_arrive(&iempty[slot]);
      const uint32_t npad = (nq_i + 15) & ~15u;
      const uint32_t ntiles = (nrows_i + kTcTile - 1) / kTcTile;
      const uint32_t npt = (ntiles + 1) / 2;
      const uint32_t idesc = h16 ? f16_idesc_m(256, npad) : tf32_idesc_m(256, npad);
      const uint64_t adesc0 = sw64_kmajor_desc(smem_u32(aring));
      const uint32_t tw = npad > 128 ? 2u : 1u;  // TMEM slots per tile
      for (uint32_t pt = 0; pt < npt; ++pt) {
        if (tw == 2 && (tu & 1)) {  // a two-slot tile starts on an even slot: skip one
          if (leader) {
            mbar_wait_cl(&tempty[tu & 3], ((tu >> 2) & 1) ^ 1);
            tc_fence_after();
            if (lane == 0) mma2_commit_both(&tfull[tu & 3]);
            __syncwarp();
          }
          ++tu;
        }
        if (leader) {
          TC_PROF_T0();
          mbar_wait_cl(&tempty[tu & 3], ((tu >> 2) & 1) ^ 1);
          if (tw == 2) mbar_wait_cl(&tempty[(tu + 1) & 3], (((tu + 1) >> 2) & 1) ^ 1);
          if (lane == 0) TC_PROF_ADD(2);
          tc_fence_after();
        }
        const uint32_t d_tmem = tmem_base + (tu & 3) * 128;
        for (uint32_t sg = 0; sg < nstg; ++sg) {
          const uint32_t cn = min((uint32_t)kPCps, nch - sg * kPCps);
          const uint32_t a = ra, pa = rpa;
          if (leader) {
            {
              TC_PROF_T0();
              mbar_wait(&full[a], pa);        // own stage landed
              if (lane == 0) TC_PROF_ADD(1);
            }
            {
              TC_PROF_T0();
              mbar_wait_cl(&pfull[a], pa);    // the peer's stage landed
              if (lane == 0) TC_PROF_ADD(0);
            }
            tc_fence_after();
            const long long _ti = P.prof ? clock64() : 0;
            const uint64_t adesc = adesc0 + (uint64_t)(a * (kSB >> 4));
            const uint64_t qd0 = adesc + (uint64_t)(kPairStageA >> 4);
            // the stage's MMAs in one warp-collective asm block; (npad/2)*64 B of queries per chunk
            if (!(P.variant & 4)) {
              if (h16) mma2_stage8_f16(d_tmem, adesc, qd0, idesc, sg != 0, cn, npad * 2);
              else mma2_stage8_tf32(d_tmem, adesc, qd0, idesc, sg != 0, cn, npad * 2);
            }
            if (lane == 0) mma2_commit_both(&empty[a]);  // the slot is free in both CTAs
            __syncwarp();
            if (P.prof && lane == 0) {
              atomicAdd(&P.prof[blockIdx.x * 16 + 12], (unsigned long long)(clock64() - _ti));
              atomicAdd(&P.prof[blockIdx.x * 16 + 13], 1ull);
            }
          } else {
            mbar_wait(&full[a], pa);
            if (lane == 0) mbar_arrive_remote(pfull_peer0 + a * 8);
            __syncwarp();
          }
          if (++ra == SA) { ra = 0; rpa ^= 1; }
        }
        if (leader) {
          if (lane == 0) {
            mma2_commit_both(&tfull[tu & 3]);
            if (tw == 2) mma2_commit_both(&tfull[(tu + 1) & 3]);
          }
          __syncwarp();
        }
        tu += tw;
      }
    }
  } else {
    // ---------------- epilogue: two groups of 128 queries, 8-deep per-warp lists ----------------
    const uint32_t quad = warp & 3;                 // TMEM lane quadrant of this warp
    const uint32_t ew = (warp - 2) & 3;             // warp within its group
    const uint32_t h = (uint32_t)(warp - 2) >> 2;   // group: query columns [kPQ h, kPQ (h+1))
    const uint32_t tempty_leader = mapa_peer(&tempty[0], 0);
    float* gmd = md + h * (kTcEpiWarps * 8 * 8);
    uint32_t* gmr = mr + h * (kTcEpiWarps * 8 * 8);
    for (uint32_t i = 0;; ++i) {
      const uint32_t slot = i % kItemQ, iph = (i / kItemQ) & 1;
      mbar_wait_parked(&ifull[slot], iph);
      if (!s_valid[slot]) break;
      const ScanItem item = s_item[slot];
      const uint32_t nq = item.nq > kPQ * h ? min((uint32_t)kPQ, item.nq - kPQ * h) : 0u;
      const uint32_t ip = i & 1;
      float* m_qn2 = s_qn2[ip][h];
      float* m_E = s_E[ip][h];
      float* m_m2 = s_m2[ip][h];
      uint32_t* m_qi = s_qi[ip][h];
      uint32_t* m_oslot = s_oslot[ip][h];
      {  // the group's per-query metadata (warp ew owns queries 16 ew .. 16 ew + 15)
        const uint32_t q = 16 * ew + lane;
        if (lane < 16 && q < nq) {
          const uint32_t pair = P.sorted_pairs[item.pair0 + kPQ * h + q];
          const uint32_t qi = P.pair_query[pair];
          m_qi[q] = qi;
          m_qn2[q] = P.qv.qn2[qi];
          m_oslot[q] = pair * P.ix.s_max + 2 * item.seg + crank;
          m_E[q] = seg_bound(P.ix, P.qv.qnorm[qi], P.ix.maxnorm[item.list]);
          m_m2[q] = dot_coef(P.ix, P.qv, qi, item.list);
        }
        named_bar_sync(2 + h, kTcEpiWarps * 32);
      }
      const uint32_t ntiles = (item.nrows + kTcTile - 1) / kTcTile;
      const uint32_t npt = (ntiles + 1) / 2;
      const uint64_t lbeg = P.ix.list_off[item.list];
      float ld[kPQ / 4];  // slot s: queries 4s..4s+3, 8 lanes each
      uint32_t lr[kPQ / 4];
#pragma unroll
      for (int j = 0; j < kPQ / 4; ++j) {
        ld[j] = kInfF;
        lr[j] = kNoRow;
      }
      float gmin[2] = {kInfF, kInfF};
      const uint32_t tw = ((item.nq + 15) & ~15u) > 128 ? 2u : 1u;  // TMEM slots per tile (as the MMA warp)
      for (uint32_t pt = 0; pt < npt; ++pt) {
        const uint32_t t = 2 * pt + crank;
        const uint32_t srow = t * kTcTile + quad * 32 + lane;  // segment-local row
        const bool valid = srow < item.nrows;
        const float xn = valid ? __ldg(P.ix.xnorm2 + lbeg + item.row0 + srow) : 0.f;
        if (tw == 2 && (tu & 1)) {  // the skipped odd slot: pass it back
          mbar_wait_parked(&tfull[tu & 3], (tu >> 2) & 1);
          tc_fence_after();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (leader) mbar_arrive(&tempty[tu & 3]);
            else mbar_arrive_remote(tempty_leader + (tu & 3) * 8);
          }
          ++tu;
        }
        {
          TC_PROF_T0();
          mbar_wait_parked(&tfull[tu & 3], (tu >> 2) & 1);
          if (tw == 2) mbar_wait_parked(&tfull[(tu + 1) & 3], ((tu + 1) >> 2) & 1);
          if (lane == 0) TC_PROF_ADD(8);
        }
        tc_fence_after();
        const long long _te = P.prof ? clock64() : 0;
        float gl[2] = {kInfF, kInfF};
        if (!(P.variant & 32)) {  // debug bit5: skip the tile's epilogue math
#pragma unroll
        for (int m = 0; m < 2; ++m) {
          if (P.topk && 32 * m + lane < nq) {
            const float u = __ldcg(P.qbound + m_qi[32 * m + lane]);
            if (u < 3.0e38f) gl[m] = drop_bound(u, m_E[32 * m + lane]);
          }
          gmin[m] = fminf(gmin[m], gl[m]);
        }
        const uint32_t grow = (uint32_t)(lbeg + item.row0 + srow);
        const uint32_t ta = tmem_base + ((quad * 32) << 16) + (tu & 3) * 128 + kPQ * h;
#pragma unroll
        for (int m = 0; m < 2; ++m) {  // 32 query columns at a time
          if (32 * m >= (int)nq) break;
          uint32_t acc[32];
          TMEM_LD32(ta + 32 * m, acc);
          tmem_wait_ld();
#pragma unroll
          for (int sl = 0; sl < 8; ++sl) {  // query quad (4sp .. 4sp+3), sp = 8m + sl
            const int sp = 8 * m + sl;
            if (4 * sp >= (int)nq) break;
            float v[4];
            bool any = false;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int q = 4 * sp + j;  // group-local query; acc column q & 31
              const float q2 = q < (int)nq ? m_qn2[q] : 0.f;
              const float m2 = q < (int)nq ? m_m2[q] : -2.f;
              const float g = __shfl_sync(FULL, gl[m], q & 31);
              const float th = fminf(__shfl_sync(FULL, ld[sp], 8 * j + 7), g);
              const float x = (valid && q < (int)nq)
                                  ? __fmaf_rn(m2, __uint_as_float(acc[q & 31]), __fadd_rn(xn, q2))
                                  : kInfF;
              v[j] = x < th ? x : kInfF;
              any |= x < th;
            }
            if (!__any_sync(FULL, any)) continue;
            const Cand r = merge_quad8(v[0], v[1], v[2], v[3], grow, ld[sp], lr[sp], lane);
            ld[sp] = r.v;
            lr[sp] = r.r;
          }
        }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          for (uint32_t u = tu; u < tu + tw; ++u) {
            if (leader) mbar_arrive(&tempty[u & 3]);
            else mbar_arrive_remote(tempty_leader + (u & 3) * 8);
          }
          if (P.prof) atomicAdd(&P.prof[blockIdx.x * 16 + 11], (unsigned long long)(clock64() - _te));
        }
        tu += tw;
      }
      // ---- item end: the four warps' 8-lists of each query -> its 32 candidates ----
      const long long _tm = P.prof ? clock64() : 0;
#pragma unroll
      for (int h0 = 0; h0 < kPQ; h0 += 8) {
        if (h0 >= (int)nq) break;
        named_bar_sync(2 + h, kTcEpiWarps * 32);
        if (h0 == 0) {
#pragma unroll
          for (int m = 0; m < 2; ++m) s_gm[h][ew][32 * m + lane] = gmin[m];
        }
#pragma unroll
        for (int jj = 0; jj < 8; ++jj) {
          const int q = h0 + jj;
          const int sp = q >> 2;
          if ((lane >> 3) == (q & 3)) {
            gmd[(ew * 8 + jj) * 8 + (lane & 7)] = ld[sp];
            gmr[(ew * 8 + jj) * 8 + (lane & 7)] = lr[sp];
            if ((lane & 7) == 7) s_w8[h][ew][q] = lr[sp] != kNoRow ? ld[sp] : kInfF;
          }
        }
        named_bar_sync(2 + h, kTcEpiWarps * 32);
        for (uint32_t jj = ew; jj < 8 && h0 + jj < nq; jj += kTcEpiWarps) {
          const uint32_t q = h0 + jj;
          float x = gmd[((lane >> 3) * 8 + jj) * 8 + (lane & 7)];
          uint32_t xr = gmr[((lane >> 3) * 8 + jj) * 8 + (lane & 7)];
          warp_sort32(x, xr, lane);
          const uint32_t oslot = m_oslot[q];
          const float Ej = m_E[q];
          const uint32_t qij = m_qi[q];
          const bool bad = coef_bad(m_m2[q]);
          P.out_d[(uint64_t)oslot * kKP + lane] = x;
          P.out_row[(uint64_t)oslot * kKP + lane] = xr;
          const uint32_t n_kept = __popc(__ballot_sync(FULL, xr != kNoRow));
          const uint32_t n_valid = bad ? 0u : n_kept;
          const float gm = fminf(fminf(s_gm[h][0][q], s_gm[h][1][q]), fminf(s_gm[h][2][q], s_gm[h][3][q]));
          const float w8 = fminf(fminf(s_w8[h][0][q], s_w8[h][1][q]), fminf(s_w8[h][2][q], s_w8[h][3][q]));
          const float vk = __shfl_sync(FULL, x, (int)(P.topk ? P.topk - 1 : 0));
          if (lane == 0) {
            P.out_thr[oslot] = bad ? -kInfF : fminf(gm, w8);
            P.out_n[oslot] = n_valid;
            if (P.bound_update && !bad && n_valid >= P.topk) {
              float u = __fadd_ru(vk, Ej);
              if (!(u > 0.f)) u = 0.f;
              atomicMin(reinterpret_cast<int*>(P.qbound + qij), __float_as_int(u));
            }
          }
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&iempty[slot]);
        if (P.prof) atomicAdd(&P.prof[blockIdx.x * 16 + 9], (unsigned long long)(clock64() - _tm));
      }
    }
  }
  if (P.prof && threadIdx.x == 0) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    P.prof[blockIdx.x * 16 + 6] = g;
  }
  tc_fence_before();
  cluster_sync_all();  // both CTAs done with TMEM and the cross-CTA barriers
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(kTmemCols));
  }
}

// Shared-memory plan: the unsplit query group stays resident for the whole
// item; what is left feeds the A landing ring (bytes in flight per SM).
// Dynamic smem budget = the device's opt-in per-block maximum (227 KB on B200)
// minus the kernel's static __shared__ variables, queried once.
// Per kernel (by its query-group size q): narrow 8..32, wide 64 / 128, pair 256.
static int tc_budget(uint32_t q) {
  static int budget[kMaxDevices][4];
  static bool have[kMaxDevices] = {};
  const int dev = current_device();
  if (dev < 0 || dev >= kMaxDevices) return 0;
  if (!have[dev]) {  // benign race: every thread computes the same value
    int optin = 232448;
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev) != cudaSuccess)
      optin = 232448;
    const void* fns[4] = {(const void*)k_scan_tc<0>, (const void*)k_scan_tc<64>, (const void*)k_scan_tc<128>,
                          (const void*)k_scan_pair};
    for (int i = 0; i < 4; ++i) {
      cudaFuncAttributes fa{};
      size_t st = 16384;
      if (cudaFuncGetAttributes(&fa, fns[i]) == cudaSuccess) st = fa.sharedSizeBytes;
      budget[dev][i] = optin - (int)st;
    }
    have[dev] = true;
  }
  return budget[dev][q == kTcPairQ ? 3 : q == kTcWide2Q ? 2 : q == kTcWideQ ? 1 : 0];
}
static int tc_fixed_bytes(uint32_t dpad, uint32_t qmax, int split) {
  const bool wide = tc_is_wide(qmax);  // no resident query group; two merge groups of 8
  if (qmax == kTcPairQ)  // alignment + merge scratch [4 groups][4 warps][8 queries][8] x (d, row)
    return 1024 + 4 * kTcEpiWarps * 8 * 8 * 8;
  return 1024 + (wide ? 0 : (int)(dpad / kChunk) * (split ? 2 : 1) * (int)qmax * 64) +
         (wide ? 2 * 8 : kMergeQ) * kTcEpiWarps * 32 * 8 +       // merge scratch
         8 * (2 * kTcMaxA + 2 * kTcLo + 2 * kAccMax + 2 * kItemQ + 2) + kItemQ * 32 * 16 +
         (wide ? 8 : 4) * 32 * 4 + kItemQ * 32 * 4;
}
static uint32_t tc_ring(uint32_t dpad, uint32_t qmax, int split) {
  const int left = tc_budget(qmax) - tc_fixed_bytes(dpad, qmax, split);
  // wide: the stage carries the group's query slice (the pair scan: this CTA's half)
  const int sb = qmax == kTcPairQ ? kPairStageA + kPairQB
                                  : kTcStageBytes + (tc_is_wide(qmax) ? kTcCps * (int)qmax * 64 : 0);
  return left <= 0 ? 0 : (uint32_t)min(kTcMaxA, left / sb);
}
// option "tc_wide_ppl" (env HIVF_TC_WIDE_PPL sets the process default): the
// probes-per-list density above which single-pass batches use the wide scan
// (< 0: never).  Default 0: alternating A/B runs on one box measured the wide
// scan faster at every density (C1 scan 36.6 -> 33.2 us, C2 0.463 -> 0.450 ms,
// C3 B=64 8.01 -> 7.94 ms, B=256 8.81 -> 8.72 ms, B=1024 16.3 -> 10.3 ms).
float tc_wide_ppl_default() {
  const char* e = getenv("HIVF_TC_WIDE_PPL");
  return e ? (float)atof(e) : 0.f;
}
// option "tc_wide2_ppl" (env HIVF_TC_WIDE2_PPL): the density above which the
// wide scan takes 128-query groups (k_scan_tc<128>: a list probed by 65-128
// queries is streamed once instead of twice; 3 ring stages of 64 KB).  C3
// measured (profiles/r2_c3_batch_sweep.txt): B=512 (16/list) equal, B=1024
// (32/list) 91.2k -> 93.4k q/s, B=2048 110k -> 151k.
// option "tc_pair_ppl" (env HIVF_TC_PAIR_PPL): the density above which the
// wide scan runs 256-query groups on CTA pairs (k_scan_pair).  C3 A/B on one
// box (profiles/r2_pair_ab.txt): B=4096 (128 probes/list) 162.8k -> 167.0k q/s,
// B=2048 (64/list) 151k -> 103k -- the pair's MMA floor (~120 cycles per
// M=256 K=8 step at any N) and cross-CTA waits cost more than the saved
// passes until lists carry > ~96 probes.
float tc_pair_ppl_default() {
  const char* e = getenv("HIVF_TC_PAIR_PPL");
  return e ? (float)atof(e) : 96.f;
}
float tc_wide2_ppl_default() {
  const char* e = getenv("HIVF_TC_WIDE2_PPL");
  return e ? (float)atof(e) : 24.f;
}

uint32_t scan_tc_qmax(uint32_t dpad, int split, float probes_per_list, const TcOpts& opt) {
  const uint32_t o = opt.qmax_override;
  if (o && (!tc_is_wide(o) || !split) && tc_ring(dpad, o, split) >= 2) return o;
  if (!split && opt.pair_ppl >= 0.f && opt.wide_ppl >= 0.f && probes_per_list > opt.pair_ppl &&
      tc_ring(dpad, kTcPairQ, 0) >= 3)
    return kTcPairQ;
  if (!split && opt.wide2_ppl >= 0.f && opt.wide_ppl >= 0.f && probes_per_list > opt.wide2_ppl &&
      tc_ring(dpad, kTcWide2Q, 0) >= 3)
    return kTcWide2Q;
  // dense batches, single pass: 64-query groups streamed with the list stages
  // (k_scan_tc<64>) -- each list tile crosses HBM->smem once per 64 probes
  if (!split && opt.wide_ppl >= 0.f && probes_per_list > opt.wide_ppl && tc_ring(dpad, kTcWideQ, 0) >= 3)
    return kTcWideQ;
  // HBM-bound batches (few probes per list): the widest group that still
  // leaves a 4-stage (128 KB) landing ring -- ring depth (bytes in flight per
  // SM) wins (C3, B=256, ~8 probes/list: q=24/4 stages 8.81 ms vs q=32/3
  // stages 9.03 ms).  Dense batches (> 12 probes per list): fewer groups per
  // list win (B=512: q=32 9.74 ms vs q=24 10.85 ms; B=1024: 60.6k vs 53.7k q/s).
  if (probes_per_list <= 12.f)
    for (uint32_t q : {32u, 24u, 16u})
      if (tc_ring(dpad, q, split) >= 4) return q;
  for (uint32_t q : {32u, 24u, 16u})
    if (tc_ring(dpad, q, split) >= 3) return q;
  if (tc_ring(dpad, 8, split) >= 2) return 8;
  return 0;  // too wide for the tensor-core scan: caller uses the FFMA scan
}
static unsigned long long* g_tc_prof = nullptr;  // debug stall counters (option "tc_prof")
void set_tc_prof(int on) {
  if (on && !g_tc_prof) cudaMalloc(&g_tc_prof, 1024 * 16 * sizeof(unsigned long long));
  if (on) cudaMemset(g_tc_prof, 0, 1024 * 16 * sizeof(unsigned long long));
  if (!on && g_tc_prof) {
    cudaFree(g_tc_prof);
    g_tc_prof = nullptr;
  }
}
int get_tc_prof(unsigned long long* host, int n_ctas) {
  if (!g_tc_prof) return 0;
  cudaDeviceSynchronize();
  cudaMemcpy(host, g_tc_prof, (size_t)n_ctas * 16 * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
  return 1;
}

int scan_tc_smem_bytes(uint32_t dpad, int split, float probes_per_list, const TcOpts& o) {
  const uint32_t q = scan_tc_qmax(dpad, split, probes_per_list, o);
  return tc_fixed_bytes(dpad, q, split) +
         (int)tc_ring(dpad, q, split) *
             (q == kTcPairQ ? kPairStageA + kPairQB
                            : kTcStageBytes + (tc_is_wide(q) ? kTcCps * (int)q * 64 : 0));
}

void launch_scan_tc(const IndexView& ix, const QueryView& qv, const ScanItem* items,
                    const uint32_t* n_items, uint32_t* work_ctr, const uint32_t* sorted_pairs,
                    const uint32_t* pair_query, float* out_d, uint32_t* out_row, float* out_thr,
                    uint32_t* out_n, int n_ctas, int split, float* qbound, uint32_t topk,
                    int bound_update, float probes_per_list, const WideStage& ws, const TcOpts& o,
                    cudaStream_t s) {
  const uint32_t q = scan_tc_qmax(ix.dpf, split, probes_per_list, o);
  const int conv = tc_conversion_mode();
  const bool wide = tc_is_wide(q);
  TcParams P{ix, qv, items, n_items, work_ctr, sorted_pairs, pair_query, out_d, out_row, out_thr,
             out_n, q, tc_ring(ix.dpf, q, split), conv > 1 ? 0 : conv, o.variant,
             wide ? 0 : split, g_tc_prof, qbound, qbound ? topk : 0u, (qbound && bound_update) ? 1u : 0u,
             ws.qstage, ws.qshift};
  const int smem = scan_tc_smem_bytes(ix.dpf, split, probes_per_list, o);
  if (q == kTcPairQ) {
    smem_optin((const void*)k_scan_pair, smem);
    launch_pdl(k_scan_pair, dim3(std::max(2, n_ctas & ~1)), dim3(kPairThreads), smem, s, P);
  } else if (q == kTcWide2Q) {
    smem_optin((const void*)k_scan_tc<128>, smem);
    launch_pdl(k_scan_tc<128>, dim3(n_ctas), dim3(kTcThreads), smem, s, P);
  } else if (wide) {
    smem_optin((const void*)k_scan_tc<64>, smem);
    launch_pdl(k_scan_tc<64>, dim3(n_ctas), dim3(kTcThreads), smem, s, P);
  } else {
    smem_optin((const void*)k_scan_tc<0>, smem);
    launch_pdl(k_scan_tc<0>, dim3(n_ctas), dim3(kTcThreads), smem, s, P);
  }
}

namespace {
// Restage the pairs' query rows for the wide scan.  List c's pairs occupy
// staged rows [pair_off[c] + qshift[c], +ceil8(n_c)) (8-row aligned); its
// query group g (64 pairs, the last one npad = ceil8(rest) rows) is one block
// of dpad*4*npad bytes laid out chunk-major [ch][npad rows][64 B] with the
// SWIZZLE_64B XOR, so a stage's 4-chunk slice is one contiguous bulk copy
// that lands in UMMA K-major layout.
__global__ void __launch_bounds__(256) k_stage_wide(const float* __restrict__ qs, uint32_t dpad, uint32_t dpf,
                                                    const float* __restrict__ qsc,
                                                    const uint32_t* __restrict__ sorted_pairs,
                                                    const uint32_t* __restrict__ pair_query,
                                                    const uint32_t* __restrict__ pair_list,
                                                    const uint32_t* __restrict__ pair_off,
                                                    const uint32_t* __restrict__ list_cnt,
                                                    const uint32_t* __restrict__ qshift, uint8_t* qstage,
                                                    uint32_t n_pairs, uint32_t G) {
  pdl_wait();
  const uint32_t p = blockIdx.x * 8 + (threadIdx.x >> 5);  // one warp per pair
  if (p >= n_pairs) return;
  const uint32_t pair = sorted_pairs[p];
  const uint32_t c = pair_list[pair];
  const uint32_t local = p - pair_off[c], n = list_cnt[c];
  const uint32_t g = local / G, row = local % G;
  uint8_t* blk = qstage + (uint64_t)(pair_off[c] + qshift[c] + g * G) * dpf * 4;
  const uint32_t qi = pair_query[pair];
  const float4* src = reinterpret_cast<const float4*>(qs + (uint64_t)qi * dpad);
  if (qsc) {  // fp16 filter copy: q 2^e_q in fp16, 32-dim chunks (16-B granules of 8 dims)
    const float up = qsc[qi] > 0.f ? 1.f / qsc[qi] : 1.f;
    const float* qrow = qs + (uint64_t)qi * dpad;
    uint32_t nrow = 0, r = row;
    uint8_t* base = blk;
    if (G == kPairQ) {
      const uint32_t npad = min(G, ((n - g * G) + 15) & ~15u), hr = npad / 2;
      const uint32_t half = row / hr;
      r = row % hr;
      nrow = hr;
      base = blk + (uint64_t)half * (dpf / 16) * hr * 64;
    } else {
      nrow = min(G, ((n - g * G) + 7) & ~7u);
    }
    for (uint32_t gh = threadIdx.x & 31; gh < dpf / 4; gh += 32) {
      const uint32_t ch = gh >> 2, q4 = gh & 3;
      *reinterpret_cast<uint4*>(base + (uint64_t)ch * nrow * 64 + r * 64 + ((q4 ^ ((r >> 1) & 3)) << 4)) =
          h16_granule(qrow, dpad, gh, up);
    }
    return;
  }
  if (G == kPairQ) {  // CTA-pair groups: [half][ch][npad/2 rows][64 B], npad = ceil16
    const uint32_t npad = min(G, ((n - g * G) + 15) & ~15u), hr = npad / 2;
    const uint32_t half = row / hr, r = row % hr;
    uint8_t* hb = blk + (uint64_t)half * (dpad / 16) * hr * 64;
    for (uint32_t g4 = threadIdx.x & 31; g4 < dpad / 4; g4 += 32) {
      const uint32_t ch = g4 >> 2, q4 = g4 & 3;
      *reinterpret_cast<float4*>(hb + (uint64_t)ch * hr * 64 + r * 64 + ((q4 ^ ((r >> 1) & 3)) << 4)) = src[g4];
    }
    return;
  }
  const uint32_t npad = min(G, ((n - g * G) + 7) & ~7u);
  for (uint32_t g4 = threadIdx.x & 31; g4 < dpad / 4; g4 += 32) {
    const uint32_t ch = g4 >> 2, q4 = g4 & 3;
    *reinterpret_cast<float4*>(blk + (uint64_t)ch * npad * 64 + row * 64 + ((q4 ^ ((row >> 1) & 3)) << 4)) =
        src[g4];
  }
}
}  // namespace

uint64_t wide_stage_rows(uint32_t n_pairs, uint32_t n_lists) {
  return (uint64_t)n_pairs + 15ull * n_lists + 16;  // 16-row aligned per list (pair groups)
}

void launch_stage_wide(const IndexView& ix, const QueryView& qv, const uint32_t* sorted_pairs,
                       const uint32_t* pair_query, const uint32_t* pair_list, const uint32_t* pair_off,
                       const uint32_t* list_cnt, uint32_t n_pairs, const WideStage& ws, cudaStream_t s) {
  if (n_pairs)
    launch_pdl(k_stage_wide, dim3((n_pairs + 7) / 8), dim3(256), 0, s, qv.qs, ix.dpad, ix.vech ? ix.dpf : ix.dpad,
               ix.vech ? qv.qsc : nullptr, sorted_pairs, pair_query, pair_list,
                                                   pair_off, list_cnt, ws.qshift, ws.qstage, n_pairs, ws.group);
}

}  // namespace hivf

// ---------------------------------------------------------------------------
// hivf_tc_probe: how does this tensor core convert fp32 operands to tf32?
// One M=128 x N=8 x K=8 MMA with A[r][0] = probe value, B[0][0] = 1: the
// accumulator then holds conv(v_r) exactly.  Result: 0 truncation, 1 RNE,
// 2 neither (the split-precision scan is then disabled).
// ---------------------------------------------------------------------------
namespace hivf {
namespace {
__global__ void __launch_bounds__(128, 1) k_tc_probe(int* out) {
  __shared__ __align__(1024) uint8_t a[kTcChunkBytes];
  __shared__ __align__(1024) uint8_t b[8 * 64];
  __shared__ uint64_t bar;
  __shared__ uint32_t s_tmem;
  __shared__ int votes[3];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // probe values: 1.x with every interesting low-13-bit pattern (below, at, above the tie)
  const uint32_t lows[8] = {0x0000u, 0x0001u, 0x0fffu, 0x1000u, 0x1001u, 0x1fffu, 0x0800u, 0x17ffu};
  const uint32_t u = 0x3f800000u | ((uint32_t)(tid >> 3) << 13) | lows[tid & 7];
  const float v = __uint_as_float(u);
  for (int i = tid; i < kTcChunkBytes / 4; i += 128) reinterpret_cast<float*>(a)[i] = 0.f;
  for (int i = tid; i < 8 * 16; i += 128) reinterpret_cast<float*>(b)[i] = 0.f;
  if (tid < 3) votes[tid] = 0;
  __syncthreads();
  // row tid, dim 0 -> 16-B group 0 at swizzled position (0 ^ ((r>>1)&3))
  reinterpret_cast<float*>(a + tid * 64 + (((tid >> 1) & 3) << 4))[0] = v;
  if (tid == 0) reinterpret_cast<float*>(b)[0] = 1.0f;  // B row 0, group 0 (swizzle 0)
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s_tmem)),
                 "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  if (tid == 0) {
    mma_tf32(tmem, sw64_kmajor_desc(smem_u32(a)), sw64_kmajor_desc(smem_u32(b)), tf32_idesc(8), 0);
    mma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  uint32_t r[32];
  TMEM_LD32(tmem + ((warp * 32) << 16), r);
  tmem_wait_ld();
  const float got = __uint_as_float(r[0]);
  const uint32_t rne = (u + 0xfffu + ((u >> 13) & 1u)) & 0xffffe000u;
  if (got == tf32_trunc(v)) atomicAdd(&votes[0], 1);
  if (__float_as_uint(got) == rne) atomicAdd(&votes[1], 1);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
  }
  if (tid == 0) *out = votes[0] == 128 ? 0 : (votes[1] == 128 ? 1 : 2);
}
}  // namespace

static int tc_probe_conversion() {
  int* d = nullptr;
  int h = 2;
  cudaStream_t s = nullptr;
  if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess) return 2;
  if (cudaMalloc(&d, sizeof(int)) == cudaSuccess) {
    k_tc_probe<<<1, 128, 0, s>>>(d);
    if (cudaMemcpyAsync(&h, d, sizeof(int), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      h = 2;
    cudaFree(d);
  }
  cudaStreamDestroy(s);
  (void)cudaGetLastError();
  return h;
}

// probed once per device, on first use (hivf_ctx_create triggers it)
int tc_conversion_mode() {
  static std::mutex mu;
  static int conv[kMaxDevices];
  static bool have[kMaxDevices] = {};
  const int dev = current_device();
  if (dev < 0 || dev >= kMaxDevices) return 2;
  std::lock_guard<std::mutex> lk(mu);
  if (!have[dev]) {
    conv[dev] = tc_probe_conversion();
    have[dev] = true;
  }
  return conv[dev];
}
}  // namespace hivf

// ---------------------------------------------------------------------------
// hivf_debug_tc_dot: the scan's tensor-core dot product in isolation, to
// validate the accumulation term of the filter bound (DESIGN.md §3,
// bound_tc / bound_tc1) against adversarial data.  One CTA computes
// out[r][j] = sum_d A[r][d] * B[j][d] for 128 rows and n <= 16 columns with
// exactly the scan's MMA sequence: 64-dim stages in the SWIZZLE_64B K-major
// layout, one tcgen05.mma M=128 x N x K=8 per 8-dim k-step, accumulating in
// TMEM in dim order.  split = 1 reproduces the 3-pass split: the k-step
// issues A x [q ; lo(q)] (N = 2n) and lo(A) x q onto the first n columns,
// lo = x - conv(x) as the splitters form it; out then holds 2n columns
// ([hi*hi + lo*hi | hi*lo]) that the epilogue adds in fp32.
// ---------------------------------------------------------------------------
namespace hivf {
namespace {
__global__ void __launch_bounds__(128, 1) k_tc_dot(const float* __restrict__ A, const float* __restrict__ B,
                                                   uint32_t D, uint32_t n, int split, int conv,
                                                   float* __restrict__ out) {
  // one 16-dim chunk plane at a time (the stage's chunks are consumed in the
  // same dim order, so the accumulation sequence is the scan's)
  __shared__ __align__(1024) uint8_t a[kTcChunkBytes];
  __shared__ __align__(1024) uint8_t alo[kTcChunkBytes];
  __shared__ __align__(1024) uint8_t b[32 * 64];  // <= 32 B rows
  __shared__ uint64_t bar;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t nb = split == 1 ? 2 * n : n;  // B rows: [q ; lo(q)]
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(&s_tmem)),
                 "r"(32));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  if (split == 2) {  // kind::f16: fp16 operands (RN conversion here), 32-dim chunks, K = 16 per MMA
    const uint32_t nch16 = (D + 31) / 32;
    for (uint32_t ch = 0; ch < nch16; ++ch) {
      for (int g = 0; g < 4; ++g)
        for (int e = 0; e < 8; ++e) {
          const uint32_t d = ch * 32 + g * 8 + e;
          const uint32_t off = tid * 64 + ((g ^ ((tid >> 1) & 3)) << 4) + e * 2;
          *reinterpret_cast<__half*>(a + off) = __float2half_rn(d < D ? A[(size_t)tid * D + d] : 0.f);
          if ((uint32_t)tid < n) *reinterpret_cast<__half*>(b + off) = __float2half_rn(d < D ? B[(size_t)tid * D + d] : 0.f);
        }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
      if (tid == 0) {
        tc_fence_after();
        for (int k2 = 0; k2 < 2; ++k2) {
          const uint64_t ad = sw64_kmajor_desc(smem_u32(a)) + (uint64_t)(k2 * 2);
          const uint64_t bd = sw64_kmajor_desc(smem_u32(b)) + (uint64_t)(k2 * 2);
          mma_f16(tmem, ad, bd, f16_idesc_m(128, n), (ch | k2) != 0);
        }
        mma_commit(&bar);
      }
      mbar_wait(&bar, ch & 1);
      tc_fence_after();
      __syncthreads();
    }
  }
  const uint32_t nch = split == 2 ? 0u : (D + 15) / 16;
  for (uint32_t ch = 0; ch < nch; ++ch) {
    // A row `tid` (and lo(A)); B rows for tid < nb; zero past D
    for (int g = 0; g < 4; ++g)
      for (int e = 0; e < 4; ++e) {
        const uint32_t d = ch * 16 + g * 4 + e;
        const uint32_t off = tid * 64 + ((g ^ ((tid >> 1) & 3)) << 4) + e * 4;
        const float x = d < D ? A[(size_t)tid * D + d] : 0.f;
        *reinterpret_cast<float*>(a + off) = x;
        *reinterpret_cast<float*>(alo + off) = x - tf32_conv(x, conv);
        if ((uint32_t)tid < nb) {
          const uint32_t j = (uint32_t)tid < n ? tid : tid - n;
          float y = d < D ? B[(size_t)j * D + d] : 0.f;
          if ((uint32_t)tid >= n) y = y - tf32_conv(y, conv);
          *reinterpret_cast<float*>(b + off) = y;
        }
      }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      tc_fence_after();
      for (int k2 = 0; k2 < 2; ++k2) {
        const uint64_t ad = sw64_kmajor_desc(smem_u32(a)) + (uint64_t)(k2 * 2);
        const uint64_t ld = sw64_kmajor_desc(smem_u32(alo)) + (uint64_t)(k2 * 2);
        const uint64_t bd = sw64_kmajor_desc(smem_u32(b)) + (uint64_t)(k2 * 2);
        mma_tf32(tmem, ad, bd, tf32_idesc(nb), (ch | k2) != 0);
        if (split) mma_tf32(tmem, ld, bd, tf32_idesc(n), 1);
      }
      mma_commit(&bar);
    }
    mbar_wait(&bar, ch & 1);
    tc_fence_after();
    __syncthreads();
  }
  uint32_t r[32];
  TMEM_LD32(tmem + ((warp * 32) << 16), r);
  tmem_wait_ld();
  for (uint32_t j = 0; j < nb; ++j) out[(size_t)tid * nb + j] = __uint_as_float(r[j]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(32));
  }
}
}  // namespace
}  // namespace hivf

// ---------------------------------------------------------------------------
// hivf_debug_tc2_dot: a CTA pair (cluster of 2, tcgen05 cta_group::2) computes
// out[r][j] = sum_d A[r][d] B[j][d] for 256 rows (CTA c holds rows 128c..) and
// n columns with M=256 MMAs issued by the leader CTA.  Which CTA's shared
// memory holds which half of B is the layout question this probe answers:
// bsplit = 1 puts B rows [c*n/2, (c+1)*n/2) in CTA c (N split across the
// pair), bsplit = 0 puts all n rows in both CTAs.
// ---------------------------------------------------------------------------
namespace hivf {
namespace {
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    k_tc2_dot(const float* __restrict__ A, const float* __restrict__ B, uint32_t D, uint32_t n, int bsplit,
              float* __restrict__ out) {
  __shared__ __align__(1024) uint8_t a[kTcChunkBytes];
  __shared__ __align__(1024) uint8_t b[64 * 64];  // <= 64 B rows of one 16-dim chunk
  __shared__ uint64_t bar;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5;
  const uint32_t rank = cluster_rank();
  const uint32_t nb = bsplit ? n / 2 : n;  // B rows in this CTA's smem
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)),
                 "r"(64));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync_all();
  tc_fence_after();
  const uint32_t tmem = s_tmem;
  const uint32_t nch = (D + 15) / 16;
  for (uint32_t ch = 0; ch < nch; ++ch) {
    for (int g = 0; g < 4; ++g)
      for (int e = 0; e < 4; ++e) {
        const uint32_t d = ch * 16 + g * 4 + e;
        const uint32_t off = tid * 64 + ((g ^ ((tid >> 1) & 3)) << 4) + e * 4;
        *reinterpret_cast<float*>(a + off) = d < D ? A[(size_t)(rank * 128 + tid) * D + d] : 0.f;
        if ((uint32_t)tid < nb) {
          const uint32_t j = (bsplit ? rank * nb : 0) + tid;
          *reinterpret_cast<float*>(b + off) = d < D ? B[(size_t)j * D + d] : 0.f;
        }
      }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    cluster_sync_all();  // both CTAs' operands are in place
    if (rank == 0 && tid == 0) {
      tc_fence_after();
      for (int k2 = 0; k2 < 2; ++k2) {
        const uint64_t ad = sw64_kmajor_desc(smem_u32(a)) + (uint64_t)(k2 * 2);
        const uint64_t bd = sw64_kmajor_desc(smem_u32(b)) + (uint64_t)(k2 * 2);
        const uint32_t acc = (ch | k2) != 0;
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
            "l"(ad), "l"(bd), "r"(tf32_idesc_m(256, n)), "r"(acc));
      }
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              smem_u32(&bar)),
          "h"((uint16_t)3)
          : "memory");
    }
    mbar_wait(&bar, ch & 1);
    tc_fence_after();
    cluster_sync_all();  // both CTAs done with this chunk's smem
  }
  uint32_t r[32];
  TMEM_LD32(tmem + ((warp * 32) << 16), r);
  tmem_wait_ld();
  for (uint32_t j = 0; j < n && j < 32; ++j) out[(size_t)(rank * 128 + tid) * n + j] = __uint_as_float(r[j]);
  tc_fence_before();
  cluster_sync_all();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(64));
  }
}
}  // namespace
}  // namespace hivf

// Debug / validation: host A[256][D], B[n][D] (n in {16, 32}), out[256][n].
extern "C" int hivf_debug_tc2_dot(const float* A, const float* B, unsigned D, unsigned n, int bsplit,
                                  float* out) {
  using namespace hivf;
  if (!A || !B || !out || D == 0 || (n != 16 && n != 32)) return 1;
  float *dA = nullptr, *dB = nullptr, *dO = nullptr;
  int rc = 0;
  if (cudaMalloc(&dA, 256ull * D * 4) != cudaSuccess || cudaMalloc(&dB, (size_t)n * D * 4) != cudaSuccess ||
      cudaMalloc(&dO, 256ull * n * 4) != cudaSuccess)
    rc = 3;
  if (!rc && (cudaMemcpy(dA, A, 256ull * D * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
              cudaMemcpy(dB, B, (size_t)n * D * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
              cudaMemset(dO, 0xff, 256ull * n * 4) != cudaSuccess))
    rc = 3;
  if (!rc) {
    k_tc2_dot<<<2, 128>>>(dA, dB, D, n, bsplit, dO);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) rc = 10 + (int)e;
    else if (cudaMemcpy(out, dO, 256ull * n * 4, cudaMemcpyDeviceToHost) != cudaSuccess) rc = 4;
  }
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dO);
  return rc;
}

// Debug / validation: host A[128][D], B[n][D] (n in {8, 16}), out[128][split ? 2n : n].
extern "C" int hivf_debug_tc_dot(const float* A, const float* B, unsigned D, unsigned n, int split,
                                 float* out) {
  using namespace hivf;
  if (!A || !B || !out || D == 0 || (n != 8 && n != 16)) return 1;
  const int conv = tc_conversion_mode();
  if (conv > 1) return 2;
  const size_t nb = split == 1 ? 2 * n : n;
  float *dA = nullptr, *dB = nullptr, *dO = nullptr;
  int rc = 0;
  if (cudaMalloc(&dA, 128ull * D * 4) != cudaSuccess || cudaMalloc(&dB, (size_t)n * D * 4) != cudaSuccess ||
      cudaMalloc(&dO, 128 * nb * 4) != cudaSuccess)
    rc = 3;
  if (!rc && (cudaMemcpy(dA, A, 128ull * D * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
              cudaMemcpy(dB, B, (size_t)n * D * 4, cudaMemcpyHostToDevice) != cudaSuccess))
    rc = 3;
  if (!rc) {
    k_tc_dot<<<1, 128>>>(dA, dB, D, n, split, conv, dO);
    if (cudaMemcpy(out, dO, 128 * nb * 4, cudaMemcpyDeviceToHost) != cudaSuccess) rc = 4;
  }
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dO);
  return rc;
}

// ---------------------------------------------------------------------------
// hivf_debug_mma_rate: issue rate of the scan's MMA step shapes in isolation
// (one CTA, operands resident, `reps` back-to-back MMAs into one accumulator):
//   mode 0  kind::f16  M=128 x N x K=16, A and B from shared memory (SS)
//   mode 1  kind::tf32 M=128 x N x K=8,  SS
//   mode 2  kind::f16, A from TMEM (TS), A written once
//   mode 3  tcgen05.cp 128x256b (A k-step smem -> TMEM) + TS MMA per k-step
//   mode 4+j  f16 SS round robin over 1+j independent accumulators (n <= 32)
//   mode 12 f16 SS, whole stages of 8 MMAs per asm block (mma_stage8_f16)
// cycles_out[0] = cycles per MMA; d_out[128][min(n,32)] = the accumulator
// (A rows = a[r][0..31], B rows = b[j][0..31] fp16 / tf32 values cycled
// over the reps), so modes 0, 2 and 3 can be compared bit for bit.
// ---------------------------------------------------------------------------
namespace hivf {
namespace {
__device__ __forceinline__ void mma_f16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t b, uint32_t idesc,
                                           uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d_tmem),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void tc_cp_128x256(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc));
}
__global__ void __launch_bounds__(128, 1) k_mma_rate(int mode, uint32_t n, uint32_t reps, const float* A,
                                                     const float* B, double* cyc, float* dout) {
  extern __shared__ __align__(1024) uint8_t mr_smem[];
  uint8_t* a = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(mr_smem) + 1023) & ~uintptr_t(1023));
  uint8_t* b = a + 4 * 128 * 64;  // a: 4 chunk planes (mode 12 walks them), b: 256 rows
  __shared__ uint64_t bar;
  __shared__ uint32_t s_tmem;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int i = tid; i < 4 * 128 * 64 / 4; i += 128) reinterpret_cast<uint32_t*>(a)[i] = 0u;
  __syncthreads();
  // one 64-B row slice per operand row: f16 -> 32 dims, tf32 -> 16 dims
  for (int g = 0; g < 4; ++g) {
    const uint32_t off = tid * 64 + ((g ^ ((tid >> 1) & 3)) << 4);
    for (int e = 0; e < (mode == 1 ? 4 : 8); ++e) {
      if (mode == 1) {
        reinterpret_cast<float*>(a + off)[e] = A[tid * 32 + g * 4 + e];
      } else {
        reinterpret_cast<__half*>(a + off)[e] = __float2half_rn(A[tid * 32 + g * 8 + e]);
      }
    }
  }
  for (uint32_t j = tid; j < 256; j += 128)
    for (int g = 0; g < 4; ++g) {
      const uint32_t off = j * 64 + ((g ^ ((j >> 1) & 3)) << 4);
      for (int e = 0; e < (mode == 1 ? 4 : 8); ++e) {
        const float v = j < n ? B[j * 32 + (mode == 1 ? g * 4 : g * 8) + e] : 0.f;
        if (mode == 1) reinterpret_cast<float*>(b + off)[e] = v;
        else reinterpret_cast<__half*>(b + off)[e] = __float2half_rn(v);
      }
    }
  if (tid == 0) {
    mbar_init(&bar, 1);
    fence_barrier_init();
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&s_tmem)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = s_tmem, atm = tmem + 256;  // D: columns [0, n); A in TMEM: columns 256.. (8 per k-step)
  const uint64_t ad0 = sw64_kmajor_desc(smem_u32(a)), bd0 = sw64_kmajor_desc(smem_u32(b));
  const uint32_t idesc = mode == 1 ? tf32_idesc(n) : f16_idesc_m(128, n);
  if (mode == 12 && warp == 0) {  // whole stages (4 chunks x 2 k-steps) per asm block, warp-collective
    const long long t0 = clock64();
    for (uint32_t r = 0; r < reps; r += 8) mma_stage8_f16(tmem, ad0, bd0, idesc, r != 0, 4, 0);
    if (lane == 0) {
      mma_commit(&bar);
      mbar_wait(&bar, 0);
      cyc[0] = (double)(clock64() - t0) / reps;
    }
    __syncwarp();
  }
  if (tid == 0 && mode != 12) {
    if (mode == 2) {  // A once into TMEM (both k-steps of the slice)
      tc_cp_128x256(atm, ad0);
      tc_cp_128x256(atm + 8, ad0 + 2);
    }
    tc_fence_after();
    const long long t0 = clock64();
    for (uint32_t r = 0; r < reps; ++r) {
      const uint32_t k2 = r & 1;
      if (mode >= 4) {  // f16 SS into (mode - 3) independent accumulators, round robin (32 columns apart)
        const uint32_t nd = (uint32_t)mode - 3, di = r % nd;
        mma_f16(tmem + 32 * di, ad0 + 2 * k2, bd0 + 2 * k2, idesc, r >= nd);
      } else if (mode == 0) mma_f16(tmem, ad0 + 2 * k2, bd0 + 2 * k2, idesc, r != 0);
      else if (mode == 1) mma_tf32(tmem, ad0 + 2 * k2, bd0 + 2 * k2, idesc, r != 0);
      else if (mode == 2) mma_f16_ts(tmem, atm + 8 * k2, bd0 + 2 * k2, idesc, r != 0);
      else {
        const uint32_t slot = atm + 8 * (r & 7);
        tc_cp_128x256(slot, ad0 + 2 * k2);
        mma_f16_ts(tmem, slot, bd0 + 2 * k2, idesc, r != 0);
      }
    }
    mma_commit(&bar);
    mbar_wait(&bar, 0);
    const long long t1 = clock64();
    cyc[0] = (double)(t1 - t0) / reps;
  }
  __syncthreads();
  tc_fence_after();
  uint32_t r32[32];
  TMEM_LD32(tmem + ((warp * 32) << 16), r32);
  tmem_wait_ld();
  for (uint32_t j = 0; j < 32 && j < n; ++j) dout[tid * 32 + j] = __uint_as_float(r32[j]);
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}
}  // namespace
}  // namespace hivf

extern "C" int hivf_debug_mma_rate(int mode, unsigned n, unsigned reps, const float* A, const float* B,
                                   double* cycles_out, float* d_out) {
  using namespace hivf;
  if (mode < 0 || mode > 12 || n < 8 || n > 256 || n % 8 || !A || !B || !cycles_out || !d_out) return 1;
  if (mode >= 4 && mode < 12 && n > 32) return 1;
  float *dA = nullptr, *dB = nullptr, *dO = nullptr;
  double* dC = nullptr;
  int rc = 0;
  if (cudaMalloc(&dA, 128 * 32 * 4) != cudaSuccess || cudaMalloc(&dB, 256 * 32 * 4) != cudaSuccess ||
      cudaMalloc(&dO, 128 * 32 * 4) != cudaSuccess || cudaMalloc(&dC, 8) != cudaSuccess)
    rc = 3;
  if (!rc) {
    cudaMemcpy(dA, A, 128 * 32 * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B, 256 * 32 * 4, cudaMemcpyHostToDevice);
    cudaMemset(dO, 0, 128 * 32 * 4);
    const int smem = 1024 + 4 * 128 * 64 + 256 * 64;
    cudaFuncSetAttribute(k_mma_rate, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    k_mma_rate<<<1, 128, smem>>>(mode, n, reps, dA, dB, dC, dO);
    if (cudaMemcpy(cycles_out, dC, 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(d_out, dO, 128 * 32 * 4, cudaMemcpyDeviceToHost) != cudaSuccess)
      rc = 4;
  }
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dO);
  cudaFree(dC);
  return rc;
}

// Debug: the filter-bound coefficients of a scan kind (0 FFMA, 2 split TC,
// 3 single-pass TC) at dimension D: E = e_a |q||x| + e_b (|q|^2+|x|^2) + e_c.
extern "C" int hivf_debug_bound(int kind, unsigned D, double* e_a, double* e_b, double* e_c) {
  if (kind == 2) hivf::bound_tc(D, e_a, e_b, e_c);
  else if (kind == 3) hivf::bound_tc1(D, e_a, e_b, e_c);
  else if (kind == 4) hivf::bound_h16(D, e_a, e_b, e_c);
  else hivf::bound_ffma(D, e_a, e_b, e_c);
  return 0;
}

// Debug: per-CTA stall counters of the last k_scan_tc launches (accumulated
// since option tc_prof=1): [n_ctas][16] cycles / timestamps, see TC_PROF_*.
extern "C" int hivf_debug_tc_prof(unsigned long long* out, int n_ctas) {
  return hivf::get_tc_prof(out, n_ctas);
}

// ===========================================================================
// Coarse assign on the tensor cores: the distance pass of ivf::select_clusters
// (/root/reference/proj/src/vector_index.cpp:266-273) for all B x K (query,
// centroid) pairs as one kind::f16 GEMM over fp16 copies of the centroids and
// the queries, scaled by powers of two exactly like the fp16 filter copy
// (DESIGN.md 3a): the centroids share one scale (from the largest centroid
// norm), each query has its own (qsc, k_prep_queries).  d^ = fma(-2 2^-(e_q+e_c),
// acc, |c|^2 + |q|^2) -- the scan's fp16 distance, so the scan's bound
// (bound_h16) holds with x = the centroid; k_coarse_select then filters with it
// and re-ranks every candidate in the reference's exact double arithmetic, so
// plans are bit-identical to the FFMA pass (only the candidate superset differs).
//
// Tile: 128 centroids (M, TMEM lanes) x 128 queries (N, TMEM columns); 64-dim
// pipeline stages (two 32-dim SWIZZLE_64B chunk planes per operand, 16 KB
// each) in a 3-deep ring, one bulk copy per operand per stage.  192 threads:
// warp 0 producer, warp 1 TMEM allocator + MMA issuer, warps 2-5 epilogue
// (warp w reads TMEM lane quadrant w % 4).  96 KB of smem: 2 CTAs per SM,
// so one tile's epilogue overlaps the other's loads.
// ===========================================================================
namespace hivf {
namespace {
constexpr uint32_t kCdTile = 128;                          // centroids / queries per tile
constexpr uint32_t kCdCps = 2;                             // 32-dim chunks per stage
constexpr uint32_t kCdStageDims = kCdCps * 32;             // 64
constexpr uint32_t kCdOpBytes = kCdTile * kCdStageDims * 2;  // 16 KB per operand per stage
// ring depth: 3 stages (96 KB, 2 CTAs per SM) for grids that fill the GPU, 6
// (192 KB, one CTA per SM) for small grids, where each CTA's chain of stage
// loads is the kernel's latency (C2 / C3 B=256: 16-64 CTAs, 12 stages each)
template <uint32_t kCdRing>
constexpr uint32_t cd_smem() { return kCdRing * 2 * kCdOpBytes + 1024 + 128; }

// byte offset of the 16-B granule holding dims [d, d + 8) of row r of a tile
// (layout [tile][stage][chunk][row 0..127][64 B, SWIZZLE_64B: granule g at g ^ ((r >> 1) & 3)])
__device__ __forceinline__ uint64_t cd_offset(uint32_t tile, uint32_t S, uint32_t r, uint32_t d) {
  const uint32_t s = d / kCdStageDims, j = (d % kCdStageDims) / 32, g = (d % 32) / 8;
  return (((uint64_t)tile * S + s) * kCdCps + j) * (kCdTile * 64) + r * 64 + ((g ^ ((r >> 1) & 3u)) << 4);
}

// rows [0, n_pad) x dims [0, 64 S) of src ([n][dpad] fp32, zero past n / dpad),
// scaled by 2^e (1 / unscale; per row when rsc != nullptr, else 1 / sc) and
// rounded to fp16, into the tile layout.  One thread per 16-B granule.
__global__ void k_pack_cd(const float* __restrict__ src, uint32_t n, uint32_t dpad, uint32_t S, uint32_t n_pad,
                          const float* __restrict__ rsc, float sc, uint8_t* __restrict__ dst) {
  pdl_wait();
  const uint32_t gpr = S * kCdStageDims / 8;
  const uint64_t gid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (gid >= (uint64_t)n_pad * gpr) return;
  const uint32_t row = (uint32_t)(gid / gpr), d = (uint32_t)(gid % gpr) * 8;
  float up = 1.f;
  if (row < n) {
    const float u = rsc ? rsc[row] : sc;
    up = u > 0.f ? 1.f / u : 1.f;  // out-of-range query: results discarded (k_coarse_dist_tc)
  }
  __align__(16) __half h[8];
#pragma unroll
  for (int p = 0; p < 2; ++p) {
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (row < n && d + p * 4 < dpad) v = *reinterpret_cast<const float4*>(src + (uint64_t)row * dpad + d + p * 4);
    h[p * 4 + 0] = __float2half_rn(v.x * up);
    h[p * 4 + 1] = __float2half_rn(v.y * up);
    h[p * 4 + 2] = __float2half_rn(v.z * up);
    h[p * 4 + 3] = __float2half_rn(v.w * up);
  }
  *reinterpret_cast<uint4*>(dst + cd_offset(row / kCdTile, S, row % kCdTile, d)) = *reinterpret_cast<const uint4*>(h);
}

struct CdParams {
  const uint8_t* a;     // centroid copy (tile layout)
  const uint8_t* b;     // query copy (tile layout)
  const float* cnorm2;  // [K]
  const float* qn2;     // [n]
  const float* qsc;     // [n] 2^-e_q (0: out of range)
  float csc;            // 2^-e_c
  float* out;           // [n][K]
  uint32_t K, n, S;
};

template <uint32_t kCdRing>
__global__ void __launch_bounds__(192, 1) k_coarse_dist_tc(CdParams P) {
  pdl_wait();
  extern __shared__ uint8_t cd_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(cd_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + kCdRing * 2 * kCdOpBytes);
  uint64_t* empty = full + kCdRing;
  uint64_t* accf = empty + kCdRing;
  uint32_t* s_tmem = reinterpret_cast<uint32_t*>(accf + 1);
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t ct = blockIdx.x, qt = blockIdx.y, S = P.S;
  if (tid == 0) {
    for (uint32_t i = 0; i < kCdRing; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(accf, 1);
    fence_barrier_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(s_tmem)),
                 "r"(kCdTile));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *s_tmem;
  auto stage_a = [&](uint32_t slot) { return sm + slot * 2 * kCdOpBytes; };
  auto stage_b = [&](uint32_t slot) { return sm + slot * 2 * kCdOpBytes + kCdOpBytes; };
  if (warp == 0) {
    if (lane == 0) {
      for (uint32_t s = 0; s < S; ++s) {
        const uint32_t slot = s % kCdRing;
        if (s >= kCdRing) mbar_wait(&empty[slot], ((s / kCdRing) - 1) & 1);
        mbar_arrive_expect_tx(&full[slot], 2 * kCdOpBytes);
        bulk_g2s(stage_a(slot), P.a + ((uint64_t)ct * S + s) * kCdOpBytes, kCdOpBytes, &full[slot]);
        bulk_g2s(stage_b(slot), P.b + ((uint64_t)qt * S + s) * kCdOpBytes, kCdOpBytes, &full[slot]);
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = f16_idesc_m(kCdTile, kCdTile);
    for (uint32_t s = 0; s < S; ++s) {
      const uint32_t slot = s % kCdRing;
      mbar_wait(&full[slot], (s / kCdRing) & 1);
      tc_fence_after();
      // chunk planes are 8 KB apart in both operands (+512 in 16-B descriptor units)
      mma_stage8_f16(tmem, sw64_kmajor_desc(smem_u32(stage_a(slot))), sw64_kmajor_desc(smem_u32(stage_b(slot))),
                     idesc, s > 0 ? 1u : 0u, kCdCps, 512u);
      mma_commit_elect(&empty[slot]);
    }
    mma_commit_elect(accf);
  } else {
    mbar_wait_parked(accf, 0);
    tc_fence_after();
    const uint32_t quad = warp & 3;
    const uint32_t c = ct * kCdTile + quad * 32 + lane;
    const float cn2 = c < P.K ? P.cnorm2[c] : 0.f;
#pragma unroll 1
    for (uint32_t j = 0; j < kCdTile / 32; ++j) {
      const uint32_t q0 = qt * kCdTile + j * 32;
      if (q0 >= P.n) break;
      uint32_t r[32];
      TMEM_LD32(tmem + ((quad * 32) << 16) + j * 32, r);
      tmem_wait_ld();
      if (c < P.K) {
#pragma unroll
        for (int i = 0; i < 32; ++i) {
          const uint32_t q = q0 + i;
          if (q < P.n) {
            const float qs = P.qsc[q];
            // out-of-range query scale: +inf everywhere sends it to the exact path
            P.out[(uint64_t)q * P.K + c] =
                qs > 0.f ? __fmaf_rn(-2.f * qs * P.csc, __uint_as_float(r[i]), __fadd_rn(cn2, P.qn2[q])) : kInfF;
          }
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(kCdTile));
  }
}
}  // namespace

uint32_t coarse_tc_stages(uint32_t dpad) { return (dpad + kCdStageDims - 1) / kCdStageDims; }
uint64_t coarse_tc_bytes(uint32_t rows, uint32_t dpad) {
  return (uint64_t)((rows + kCdTile - 1) / kCdTile) * kCdTile * coarse_tc_stages(dpad) * kCdStageDims * 2;
}

void launch_pack_coarse_tc(const float* src, uint32_t n, uint32_t dpad, const float* rsc, float sc, uint8_t* dst,
                           cudaStream_t s) {
  const uint32_t S = coarse_tc_stages(dpad), n_pad = (n + kCdTile - 1) / kCdTile * kCdTile;
  const uint64_t total = (uint64_t)n_pad * S * kCdStageDims / 8;
  if (!total) return;
  launch_pdl(k_pack_cd, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, s, src, n, dpad, S, n_pad, rsc, sc, dst);
}

void launch_coarse_dist_tc(const IndexView& ix, const QueryView& qv, const uint8_t* cent_h16, float csc,
                           const uint8_t* q_h16, float* dist32, cudaStream_t s) {
  if (!qv.n) return;
  CdParams P{cent_h16, q_h16, ix.cnorm2, qv.qn2, qv.qsc, csc, dist32, ix.K, qv.n, coarse_tc_stages(ix.dpad)};
  const dim3 grid((ix.K + kCdTile - 1) / kCdTile, (qv.n + kCdTile - 1) / kCdTile);
  if ((uint64_t)grid.x * grid.y <= (uint64_t)device_sm_count()) {
    smem_optin((const void*)k_coarse_dist_tc<6>, cd_smem<6>());
    launch_pdl(k_coarse_dist_tc<6>, grid, dim3(192), (size_t)cd_smem<6>(), s, P);
  } else {
    smem_optin((const void*)k_coarse_dist_tc<3>, cd_smem<3>());
    launch_pdl(k_coarse_dist_tc<3>, grid, dim3(192), (size_t)cd_smem<3>(), s, P);
  }
}
}  // namespace hivf
