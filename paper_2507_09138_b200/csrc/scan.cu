// scan.cu -- K2/K3: grouped inverted-list scan with per-(query, segment)
// candidate selection.
//
// Replaces the inner loop of ivf::search_clusters
// (/root/reference/proj/src/vector_index.cpp:302-306: squared_l2 of
// embedding.hpp:27-34 per row, then TopKResult::insert of :38-53).  The
// reference scans one (query, list) pair at a time on a CPU core; here every
// list probed by ANY query of the batch is streamed from HBM once per batch
// (per query group of <= 16) and scored against all its probing queries.
//
// Work item = (list, segment of <= seg_rows rows, group of <= 16 queries).
// Persistent CTAs (one per SM) pull items from a global counter; items are
// generated largest-list-first (LPT).  Inside a CTA:
//   warp 8 (lane 0)  producer: 1-D cp.async.bulk of one (row-block x 16-dim
//                    chunk) slice per stage -- contiguous thanks to the
//                    chunk-major HBM layout -- into a 4-stage smem ring,
//                    completion via mbarrier tx-count;
//   warps 0..7       consumers: FFMA dot products, lane-owns-rows x
//                    query-group register tiling (8 rows x 4 queries per lane
//                    for 9-16 queries), conflict-free thanks to the XOR swizzle;
//                    epilogue = fp32 expansion distance, per-warp register
//                    top-32 per query (ballot + shuffle insertion);
//   item end         cross-warp bitonic merge -> 32 (dist32, row) per
//                    (query, segment) + drop threshold, for the exact re-rank
//                    in finalize.cu.
#include <cmath>
#include <cfloat>

#include "common.cuh"
#include "kernels.h"

namespace hivf {

namespace {

struct ScanParams {
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
};

constexpr unsigned FULL = 0xffffffffu;

template <int NQG>
__device__ __forceinline__ void consume_item(const ScanParams& P, const ScanItem& item,
                                             const float* __restrict__ stage,
                                             const float* __restrict__ qsm, uint64_t* full,
                                             uint64_t* empty, const float* s_qn2,
                                             const uint32_t* s_slot, uint32_t& st, uint32_t& ph,
                                             int warp, int lane, float* merge_buf) {
  constexpr int RG = 32 / NQG;            // row groups per warp
  constexpr int RPL = kRowsPerWarp / RG;  // rows per lane
  const int qg = lane % NQG;
  const int rg = lane / NQG;
  const uint32_t nq = item.nq;
  const uint32_t nch = P.ix.dpad / kChunk;
  const uint64_t row_base = P.ix.list_off[item.list] + item.row0;  // global row of segment row 0
  float ld[kQMax];
  uint32_t lr[kQMax];
#pragma unroll
  for (int q = 0; q < kQMax; ++q) {
    ld[q] = FLT_MAX * 2.f;  // +inf
    lr[q] = kNoRow;
  }
  const uint32_t nrb = (item.nrows + kRowBlock - 1) / kRowBlock;
  for (uint32_t rb = 0; rb < nrb; ++rb) {
    float acc[RPL][4];
#pragma unroll
    for (int i = 0; i < RPL; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    for (uint32_t ch = 0; ch < nch; ++ch) {
      mbar_wait(&full[st], ph);
      const float* sb = stage + st * (kStageBytes / 4);
#pragma unroll
      for (int s4 = 0; s4 < 4; ++s4) {
        float4 qv[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) qv[j] = lds128(qsm + (((ch * 4 + s4) * 16) + j * 4 + qg) * 4);
#pragma unroll
        for (int i = 0; i < RPL; ++i) {
          const int r = warp * kRowsPerWarp + rg + RG * i;
          const float4 xv = lds128(sb + r * kChunk + ((s4 ^ ((r >> 1) & 3)) << 2));
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            acc[i][j] = __fmaf_rn(xv.x, qv[j].x, acc[i][j]);
            acc[i][j] = __fmaf_rn(xv.y, qv[j].y, acc[i][j]);
            acc[i][j] = __fmaf_rn(xv.z, qv[j].z, acc[i][j]);
            acc[i][j] = __fmaf_rn(xv.w, qv[j].w, acc[i][j]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[st]);
      if (++st == kStages) {
        st = 0;
        ph ^= 1;
      }
    }
    // epilogue: fp32 expansion distance, masked rows -> +inf
    const uint32_t rbase = rb * kRowBlock + warp * kRowsPerWarp;
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const uint32_t srow = rbase + rg + RG * i;
      const bool valid = srow < item.nrows;
      const float xn = valid ? P.ix.xnorm2[row_base + srow] : 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const uint32_t q = qg * 4 + j;
        acc[i][j] = (valid && q < nq) ? __fmaf_rn(-2.f, acc[i][j], __fadd_rn(xn, s_qn2[q < kQMax ? q : 0]))
                                      : FLT_MAX * 2.f;
      }
    }
#pragma unroll
    for (int q = 0; q < kQMax; ++q) {
      if (q >= (int)nq) break;
      const bool own = (qg == (q >> 2));
      float th = __shfl_sync(FULL, ld[q], 31);
#pragma unroll
      for (int i = 0; i < RPL; ++i) {
        const float v = own ? acc[i][q & 3] : FLT_MAX * 2.f;
        unsigned m = __ballot_sync(FULL, v < th);
        while (m) {
          const int src = __ffs(m) - 1;
          const float cv = __shfl_sync(FULL, v, src);
          const uint32_t crow = (uint32_t)(row_base + rbase + (src / NQG) + RG * i);
          const bool before = (ld[q] < cv) || (ld[q] == cv && lr[q] < crow);
          const int pos = __popc(__ballot_sync(FULL, before));
          const float upd = __shfl_up_sync(FULL, ld[q], 1);
          const uint32_t upr = __shfl_up_sync(FULL, lr[q], 1);
          if (lane > pos) {
            ld[q] = upd;
            lr[q] = upr;
          } else if (lane == pos) {
            ld[q] = cv;
            lr[q] = crow;
          }
          th = __shfl_sync(FULL, ld[q], 31);
          m &= ~(1u << src);
          m &= __ballot_sync(FULL, v < th);
        }
      }
    }
  }
  // cross-warp merge of the per-warp top-32 lists (bitonic min-merge)
  named_bar_sync(1, kScanWarps * 32);
  float* md = merge_buf;
  uint32_t* mr = reinterpret_cast<uint32_t*>(merge_buf + kScanWarps * kQMax * 32);
#pragma unroll
  for (int q = 0; q < kQMax; ++q) {
    if (q >= (int)nq) break;
    md[(warp * kQMax + q) * 32 + lane] = ld[q];
    mr[(warp * kQMax + q) * 32 + lane] = lr[q];
  }
  named_bar_sync(1, kScanWarps * 32);
  for (uint32_t q = warp; q < nq; q += kScanWarps) {
    float v = md[q * 32 + lane];
    uint32_t r = mr[q * 32 + lane];
    for (int w2 = 1; w2 < kScanWarps; ++w2) {
      const float o = md[(w2 * kQMax + q) * 32 + 31 - lane];
      const uint32_t orr = mr[(w2 * kQMax + q) * 32 + 31 - lane];
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
    const uint32_t slot = s_slot[q];
    P.out_d[(uint64_t)slot * kKP + lane] = v;
    P.out_row[(uint64_t)slot * kKP + lane] = r;
    const uint32_t n_valid = __popc(__ballot_sync(FULL, r != kNoRow));
    const float last = __shfl_sync(FULL, v, 31);
    if (lane == 0) {
      P.out_thr[slot] = n_valid == kKP ? last : FLT_MAX * 2.f;
      P.out_n[slot] = n_valid;
    }
  }
}

__global__ void __launch_bounds__((kScanWarps + 1) * 32, 1) k_scan(ScanParams P) {
  pdl_wait();
  extern __shared__ __align__(128) uint8_t smem[];
  float* stage = reinterpret_cast<float*>(smem);
  float* qsm = reinterpret_cast<float*>(smem + kStages * kStageBytes);
  uint64_t* full = reinterpret_cast<uint64_t*>(qsm + (size_t)P.ix.dpad * kQMax);
  uint64_t* empty = full + kStages;
  __shared__ ScanItem s_item;
  __shared__ int s_valid;
  __shared__ float s_qn2[kQMax];
  __shared__ uint32_t s_slot[kQMax];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < kStages; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kScanWarps);
    }
    fence_barrier_init();
  }
  __syncthreads();
  uint32_t st = 0, ph = 0;
  const uint32_t dpad = P.ix.dpad;
  const uint32_t nch = dpad / kChunk;
  for (;;) {
    if (threadIdx.x == 0) {
      const uint32_t it = atomicAdd(P.work_ctr, 1u);
      s_valid = it < *P.n_items;
      if (s_valid) s_item = P.items[it];
    }
    __syncthreads();
    if (!s_valid) break;
    const ScanItem item = s_item;
    if (warp == kScanWarps) {
      if (lane == 0) {
        const uint64_t lbeg = P.ix.list_off[item.list];
        const uint64_t n_c = P.ix.list_off[item.list + 1] - lbeg;
        const float* lbase = list_base(P.ix, item.list, lbeg);
        for (uint32_t r0 = 0; r0 < item.nrows; r0 += kRowBlock) {
          const uint32_t nr = min((uint32_t)kRowBlock, item.nrows - r0);
          const uint32_t bytes = nr * kChunk * 4;
          for (uint32_t ch = 0; ch < nch; ++ch) {
            mbar_wait(&empty[st], ph ^ 1);
            mbar_arrive_expect_tx(&full[st], bytes);
            // the row block spans up to 4 layout tiles: one copy per tile piece,
            // landing back to back (row order) in the stage
            for (uint32_t t0 = 0; t0 < nr; t0 += kTileRows) {
              const uint64_t rt = (uint64_t)item.row0 + r0 + t0;
              const uint32_t tn = (uint32_t)tile_rows(n_c, rt);
              bulk_g2s(stage + st * (kStageBytes / 4) + t0 * kChunk, lbase + tile_chunk_offset(n_c, dpad, rt, ch),
                       tn * kChunk * 4, &full[st]);
            }
            if (++st == kStages) {
              st = 0;
              ph ^= 1;
            }
          }
        }
      }
    } else {
      const int tid = threadIdx.x;
      const uint32_t ng = dpad / 4;
      for (uint32_t idx = tid; idx < item.nq * ng; idx += kScanWarps * 32) {
        const uint32_t q = idx / ng, s = idx % ng;
        const uint32_t pair = P.sorted_pairs[item.pair0 + q];
        const uint32_t qi = P.pair_query[pair];
        const float4 v = *reinterpret_cast<const float4*>(P.qv.qs + (uint64_t)qi * dpad + s * 4);
        *reinterpret_cast<float4*>(qsm + ((s * 16) + (q & 3) * 4 + (q >> 2)) * 4) = v;
      }
      if (tid < (int)item.nq) {
        const uint32_t pair = P.sorted_pairs[item.pair0 + tid];
        s_qn2[tid] = P.qv.qn2[P.pair_query[pair]];
        s_slot[tid] = pair * P.ix.s_max + item.seg;
      }
      named_bar_sync(1, kScanWarps * 32);
      float* merge_buf = stage;  // stage ring is idle once every consumer passed the barrier
      if (item.nq <= 4)
        consume_item<1>(P, item, stage, qsm, full, empty, s_qn2, s_slot, st, ph, warp, lane, merge_buf);
      else if (item.nq <= 8)
        consume_item<2>(P, item, stage, qsm, full, empty, s_qn2, s_slot, st, ph, warp, lane, merge_buf);
      else
        consume_item<4>(P, item, stage, qsm, full, empty, s_qn2, s_slot, st, ph, warp, lane, merge_buf);
    }
    __syncthreads();
  }
}

// ---- work-list construction (all on device: no host round trip) -------------

__global__ void k_count_pairs(const uint32_t* pair_list, uint32_t n_pairs, uint32_t* cnt) {
  pdl_wait();
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p < n_pairs) atomicAdd(&cnt[pair_list[p]], 1u);
}

// Staged query rows a list reserves for the wide scans: 8-row aligned blocks,
// 16-row aligned for the CTA-pair scan's 256-query groups (each CTA of the
// pair takes half of a group's padded rows).
__device__ __forceinline__ uint32_t qpad(uint32_t n, uint32_t group) {
  return group >= 256 ? (n + 15) & ~15u : (n + 7) & ~7u;
}

// Single CTA: exclusive scans (in list_order, largest lists first) of the pair
// counts and of the work items each list generates.
__global__ void __launch_bounds__(1024) k_list_offsets(IndexView ix, uint32_t group,
                                                       const uint32_t* cnt,
                                                       uint32_t* pair_off, uint32_t* cursor,
                                                       uint32_t* item_off, uint32_t* n_items,
                                                       uint32_t* work_ctr, uint32_t* qshift) {
  pdl_wait();
  // qshift (wide tensor-core scan, optional): each list's pair range restaged
  // at an 8-row aligned offset, staged row = pair position + qshift[c]
  __shared__ uint32_t sp[1024], si[1024], sq[1024];
  const uint32_t per = (ix.K + 1023) / 1024;
  const uint32_t b = threadIdx.x * per, e = min(ix.K, b + per);
  uint32_t tp = 0, ti = 0, tq = 0;
  for (uint32_t t = b; t < e; ++t) {
    const uint32_t c = ix.list_order[t];
    const uint32_t n = cnt[c];
    const uint64_t rows = ix.list_off[c + 1] - ix.list_off[c];
    const uint32_t nseg = (uint32_t)((rows + ix.seg_rows - 1) / ix.seg_rows);
    tp += n;
    ti += n ? nseg * ((n + group - 1) / group) : 0;
    tq += qpad(n, group);
  }
  sp[threadIdx.x] = tp;
  si[threadIdx.x] = ti;
  sq[threadIdx.x] = tq;
  __syncthreads();
  for (int s = 1; s < 1024; s <<= 1) {  // Hillis-Steele inclusive scan
    const uint32_t a = threadIdx.x >= s ? sp[threadIdx.x - s] : 0;
    const uint32_t c2 = threadIdx.x >= s ? si[threadIdx.x - s] : 0;
    const uint32_t c3 = threadIdx.x >= s ? sq[threadIdx.x - s] : 0;
    __syncthreads();
    sp[threadIdx.x] += a;
    si[threadIdx.x] += c2;
    sq[threadIdx.x] += c3;
    __syncthreads();
  }
  uint32_t op = sp[threadIdx.x] - tp, oi = si[threadIdx.x] - ti, oq = sq[threadIdx.x] - tq;
  for (uint32_t t = b; t < e; ++t) {
    const uint32_t c = ix.list_order[t];
    const uint32_t n = cnt[c];
    const uint64_t rows = ix.list_off[c + 1] - ix.list_off[c];
    const uint32_t nseg = (uint32_t)((rows + ix.seg_rows - 1) / ix.seg_rows);
    pair_off[c] = op;
    item_off[c] = oi;
    cursor[c] = 0;
    if (qshift) qshift[c] = oq - op;
    op += n;
    oi += n ? nseg * ((n + group - 1) / group) : 0;
    oq += qpad(n, group);
  }
  if (threadIdx.x == 1023) {
    *n_items = si[1023];
    *work_ctr = 0;
  }
}

__global__ void k_scatter_pairs(const uint32_t* pair_list, uint32_t n_pairs, const uint32_t* pair_off,
                                uint32_t* cursor, uint32_t* sorted_pairs) {
  pdl_wait();
  const uint32_t p = blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n_pairs) return;
  const uint32_t c = pair_list[p];
  const uint32_t pos = atomicAdd(&cursor[c], 1u);
  sorted_pairs[pair_off[c] + pos] = p;
}

__global__ void k_make_items(IndexView ix, uint32_t group, const uint32_t* cnt,
                             const uint32_t* pair_off,
                             const uint32_t* item_off, ScanItem* items) {
  pdl_wait();
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ix.K) return;
  const uint32_t n = cnt[c];
  if (!n) return;
  const uint64_t rows = ix.list_off[c + 1] - ix.list_off[c];
  const uint32_t nseg = (uint32_t)((rows + ix.seg_rows - 1) / ix.seg_rows);
  const uint32_t ng = (n + group - 1) / group;
  uint32_t o = item_off[c];
  for (uint32_t s = 0; s < nseg; ++s) {
    const uint32_t row0 = s * ix.seg_rows;
    const uint32_t nr = (uint32_t)min((uint64_t)ix.seg_rows, rows - row0);
    for (uint32_t g = 0; g < ng; ++g) {
      ScanItem it;
      it.list = c;
      it.seg = s;
      it.row0 = row0;
      it.nrows = nr;
      it.pair0 = pair_off[c] + g * group;
      it.nq = min(group, n - g * group);
      items[o++] = it;
    }
  }
}

// Small batches, K <= kFusedK: the whole work list in ONE single-CTA kernel
// (count -> scans in list_order -> scatter -> items) with the per-list
// counters in shared memory -- the same outputs as the four-kernel chain
// above, four launches (and a memset) fewer on the latency-bound configs
// (C1, node-split sub-stages).
constexpr uint32_t kFusedK = 4096;

__global__ void __launch_bounds__(1024) k_worklist_fused(IndexView ix, uint32_t group,
                                                         const uint32_t* __restrict__ pair_list,
                                                         uint32_t n_pairs, uint32_t* cnt_out,
                                                         uint32_t* pair_off_out, uint32_t* item_off_out,
                                                         uint32_t* sorted_pairs, ScanItem* items,
                                                         uint32_t* n_items, uint32_t* work_ctr,
                                                         uint32_t* qshift) {
  pdl_wait();
  extern __shared__ uint32_t wsm[];
  uint32_t* cnt = wsm;            // [K]
  uint32_t* poff = cnt + ix.K;    // [K]
  uint32_t* cur = poff + ix.K;    // [K]
  __shared__ uint32_t sp[1024], si[1024], sq[1024];
  for (uint32_t c = threadIdx.x; c < ix.K; c += blockDim.x) {
    cnt[c] = 0;
    cur[c] = 0;
  }
  __syncthreads();
  for (uint32_t p = threadIdx.x; p < n_pairs; p += blockDim.x) atomicAdd(&cnt[pair_list[p]], 1u);
  __syncthreads();
  // exclusive scans in list_order (largest lists first), as k_list_offsets
  const uint32_t per = (ix.K + 1023) / 1024;
  const uint32_t b = threadIdx.x * per, e = min(ix.K, b + per);
  uint32_t tp = 0, ti = 0, tq = 0;
  for (uint32_t t = b; t < e; ++t) {
    const uint32_t c = ix.list_order[t];
    const uint32_t n = cnt[c];
    const uint64_t rows = ix.list_off[c + 1] - ix.list_off[c];
    const uint32_t nseg = (uint32_t)((rows + ix.seg_rows - 1) / ix.seg_rows);
    tp += n;
    ti += n ? nseg * ((n + group - 1) / group) : 0;
    tq += qpad(n, group);
  }
  sp[threadIdx.x] = tp;
  si[threadIdx.x] = ti;
  sq[threadIdx.x] = tq;
  __syncthreads();
  for (int o = 1; o < 1024; o <<= 1) {
    const uint32_t a = threadIdx.x >= o ? sp[threadIdx.x - o] : 0;
    const uint32_t c2 = threadIdx.x >= o ? si[threadIdx.x - o] : 0;
    const uint32_t c3 = threadIdx.x >= o ? sq[threadIdx.x - o] : 0;
    __syncthreads();
    sp[threadIdx.x] += a;
    si[threadIdx.x] += c2;
    sq[threadIdx.x] += c3;
    __syncthreads();
  }
  uint32_t op = sp[threadIdx.x] - tp, oi = si[threadIdx.x] - ti, oq = sq[threadIdx.x] - tq;
  for (uint32_t t = b; t < e; ++t) {
    const uint32_t c = ix.list_order[t];
    const uint32_t n = cnt[c];
    const uint64_t rows = ix.list_off[c + 1] - ix.list_off[c];
    const uint32_t nseg = (uint32_t)((rows + ix.seg_rows - 1) / ix.seg_rows);
    poff[c] = op;
    cnt_out[c] = n;
    pair_off_out[c] = op;
    item_off_out[c] = oi;
    if (qshift) qshift[c] = oq - op;
    // this list's work items (segment-major, query groups inside), as k_make_items
    if (n) {
      const uint32_t ng = (n + group - 1) / group;
      uint32_t o = oi;
      for (uint32_t sgi = 0; sgi < nseg; ++sgi) {
        const uint32_t row0 = sgi * ix.seg_rows;
        const uint32_t nr = (uint32_t)min((uint64_t)ix.seg_rows, rows - row0);
        for (uint32_t g = 0; g < ng; ++g) {
          ScanItem it;
          it.list = c;
          it.seg = sgi;
          it.row0 = row0;
          it.nrows = nr;
          it.pair0 = op + g * group;
          it.nq = min(group, n - g * group);
          items[o++] = it;
        }
      }
    }
    op += n;
    oi += n ? nseg * ((n + group - 1) / group) : 0;
    oq += qpad(n, group);
  }
  if (threadIdx.x == 1023) {
    *n_items = si[1023];
    *work_ctr = 0;
  }
  __syncthreads();
  for (uint32_t p = threadIdx.x; p < n_pairs; p += blockDim.x) {
    const uint32_t c = pair_list[p];
    sorted_pairs[poff[c] + atomicAdd(&cur[c], 1u)] = p;
  }
}

}  // namespace

int scan_smem_bytes(uint32_t dpad) {
  return kStages * kStageBytes + (int)dpad * kQMax * 4 + 2 * kStages * 8;
}

void launch_build_worklist(const IndexView& ix, uint32_t group, const uint32_t* pair_query,
                           const uint32_t* pair_list, uint32_t n_pairs, uint32_t* list_cnt,
                           uint32_t* list_pair_off, uint32_t* list_cursor,
                           uint32_t* list_item_off, uint32_t* sorted_pairs, ScanItem* items,
                           uint32_t* n_items, uint32_t* work_ctr, uint32_t* qshift, cudaStream_t s) {
  (void)pair_query;
  (void)list_cursor;
  if (ix.K <= kFusedK && n_pairs <= 8192u) {  // C3 (32k pairs) is faster on the 4-kernel chain
    const size_t smem = (size_t)ix.K * 12;
    smem_optin((const void*)k_worklist_fused, (int)(kFusedK * 12));
    launch_pdl(k_worklist_fused, dim3(1), dim3(1024), smem, s, ix, group, pair_list, n_pairs, list_cnt, list_pair_off,
                                           list_item_off, sorted_pairs, items, n_items, work_ctr, qshift);
    return;
  }
  cudaMemsetAsync(list_cnt, 0, sizeof(uint32_t) * ix.K, s);
  if (n_pairs) launch_pdl(k_count_pairs, dim3((n_pairs + 255) / 256), dim3(256), 0, s, pair_list, n_pairs, list_cnt);
  launch_pdl(k_list_offsets, dim3(1), dim3(1024), 0, s, ix, group, list_cnt, list_pair_off, list_cursor, list_item_off,
                                    n_items, work_ctr, qshift);
  if (n_pairs)
    launch_pdl(k_scatter_pairs, dim3((n_pairs + 255) / 256), dim3(256), 0, s, pair_list, n_pairs, list_pair_off,
                                                          list_cursor, sorted_pairs);
  launch_pdl(k_make_items, dim3((ix.K + 255) / 256), dim3(256), 0, s, ix, group, list_cnt, list_pair_off, list_item_off, items);
}

void launch_scan(const IndexView& ix, const QueryView& qv, const ScanItem* items,
                 const uint32_t* n_items, uint32_t* work_ctr, const uint32_t* sorted_pairs,
                 const uint32_t* pair_query, float* out_d, uint32_t* out_row, float* out_thr,
                 uint32_t* out_n, int n_ctas, cudaStream_t s) {
  ScanParams P{ix, qv, items, n_items, work_ctr, sorted_pairs, pair_query, out_d, out_row, out_thr, out_n};
  const int smem = scan_smem_bytes(ix.dpad);
  smem_optin((const void*)k_scan, smem);
  launch_pdl(k_scan, dim3(n_ctas), dim3((kScanWarps + 1) * 32), smem, s, P);
}

}  // namespace hivf

namespace hivf {
// Filter bounds: coefficients of
//   |d32 - delta| <= a*|q|*|x| + b*(|q|^2 + |x|^2) + c.
// FFMA scan: sequential fp32 FMA dot, eps(D)*(|q|+|x|)^2 (common.cuh).
void bound_ffma(uint32_t dim, double* a, double* b, double* c) {
  const double e = filter_eps(dim);
  *a = 2.0 * e;
  *b = e;
  *c = filter_abs(dim);
}
// Tensor-core scan (3-pass split tf32): dropped lo*lo and lo conversion
// (4*2^-20 |x||q| by Cauchy-Schwarz) + fp32 tensor-core accumulation bounded at
// 4x round-to-nearest per MMA step over 3*D/8 steps, plus the norm/combine
// roundings; x1.5 headroom.
void bound_tc(uint32_t dim, double* a, double* b, double* c) {
  const double u = 5.9604644775390625e-08, u53 = 1.1102230246251565e-16;
  const double alpha = (4.0 * 0x1p-20 + 1.5 * (double)dim * 0x1p-22) * 1.01;
  *a = 1.5 * (2.0 * alpha + 4.0 * u + 2.0 * (3.0 * dim + 6.0) * u53);
  *b = 1.5 * (4.0 * u + (3.0 * dim + 6.0) * u53);
  *c = filter_abs(dim);
}
}  // namespace hivf

namespace hivf {
// Tensor-core scan, single pass: tf32 operand truncation (<= 2^-10 relative
// per element, both operands) bounded by Cauchy-Schwarz: (2^-9 + 2^-20)|x||q|,
// plus fp32 accumulation at 4x round-to-nearest per MMA step (D/8 steps) and
// the norm/combine roundings; x1.5 headroom.
void bound_tc1(uint32_t dim, double* a, double* b, double* c) {
  const double u = 5.9604644775390625e-08, u53 = 1.1102230246251565e-16;
  const double alpha = (0x1p-9 + 0x1p-20 + 0.5 * (double)dim * 0x1p-22) * 1.01;
  *a = 1.5 * (2.0 * alpha + 4.0 * u + 2.0 * (3.0 * dim + 6.0) * u53);
  *b = 1.5 * (4.0 * u + (3.0 * dim + 6.0) * u53);
  *c = filter_abs(dim);
}
// Tensor-core scan over the fp16 filter copy (kind::f16): every row and query
// is scaled by a power of two (exact) so |element| < 2^15, then rounded to
// fp16 (RN: <= 2^-11 relative per element, both operands -> (2^-10 + 2^-22)
// |x||q| by Cauchy-Schwarz); elements below the fp16 normal range carry at
// most 2^-25 absolute in scaled units, <= 2^-39 |v| after unscaling, summing
// to <= 2 sqrt(D) 2^-38 |x||q|; the fp32 accumulation keeps the single-pass
// tf32 allowance (D/16 k-steps here, D/8 there).  Unscaling is a power-of-2
// multiply folded into the distance's fma (exact).  x1.5 headroom.
void bound_h16(uint32_t dim, double* a, double* b, double* c) {
  const double u = 5.9604644775390625e-08, u53 = 1.1102230246251565e-16;
  const double alpha =
      (0x1p-10 + 0x1p-22 + 2.0 * std::sqrt((double)dim) * 0x1p-38 + 0.5 * (double)dim * 0x1p-22) * 1.01;
  *a = 1.5 * (2.0 * alpha + 4.0 * u + 2.0 * (3.0 * dim + 6.0) * u53);
  *b = 1.5 * (4.0 * u + (3.0 * dim + 6.0) * u53);
  *c = filter_abs(dim);
}
}  // namespace hivf
