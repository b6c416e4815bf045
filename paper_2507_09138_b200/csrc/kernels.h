// kernels.h -- internal launcher interface between the C-ABI (api.cu) and the
// kernel translation units.  Host-only C++; not part of the public ABI.
#pragma once

#include <cmath>
#include <cstdint>
#include <cuda_runtime.h>

namespace hivf {

// ---- devattr.cu: per-device launch attributes (a process may drive several
// GPUs; the opt-in and the SM count are per device, keyed by the current one)
constexpr int kMaxDevices = 64;
int current_device();
int device_sm_count();
cudaError_t smem_optin(const void* kernel, int bytes);

// Tensor-core scan options of one context (hivf_set_option), passed by value
// to the scan launcher -- never process globals, so contexts on different
// devices (or with different tuning) do not interfere.
struct TcOpts {
  uint32_t qmax_override = 0;  // "tc_qmax": 0 auto
  float wide_ppl = 0.f;        // "tc_wide_ppl": probes/list above which the wide scan runs; < 0 never
  int variant = 0;             // "tc_variant" (debug, inexact when nonzero)
  float wide2_ppl = 24.f;      // "tc_wide2_ppl": above it, 128-query groups; < 0 never
  float pair_ppl = 96.f;       // "tc_pair_ppl": above it, 256-query groups on CTA pairs; < 0 never
};
float tc_wide_ppl_default();   // env HIVF_TC_WIDE_PPL, else 0
float tc_wide2_ppl_default();  // env HIVF_TC_WIDE2_PPL, else 24
float tc_pair_ppl_default();   // env HIVF_TC_PAIR_PPL, else 96

// One grouped-scan work item: rows [row0, row0+nrows) of list `list` (local
// row numbers) against up to kQMax queries listed in item_pairs[pair0, pair0+nq).
struct ScanItem {
  uint32_t list;
  uint32_t seg;    // segment index within the list
  uint32_t row0;   // first local row of the segment
  uint32_t nrows;  // rows in the segment
  uint32_t pair0;  // offset into the list-sorted pair array
  uint32_t nq;     // queries in the group (1..kQMax)
};

// Device view of an uploaded index.
struct IndexView {
  const float* vec;         // chunk-major swizzled lists (the backing store)
  // tiered index (option hbm_list_budget): per-list base address -- an HBM
  // pool slot for resident lists, the pinned host backing store otherwise;
  // nullptr when every list lives in HBM at vec + list_off[c] * dpad
  const float* const* list_ptr;
  const uint64_t* ids;      // [N] doc ids, list order
  const float* xnorm2;      // [N] fp32(|x|^2)
  const uint64_t* list_off; // [K+1] row offsets
  const float* maxnorm;     // [K] upper bound of max |x| in the list
  const float* cent;        // [K][dpad] row-major, zero padded
  const float* cnorm2;      // [K] fp32(|c|^2)
  const float* cnorm;       // [K] upper bound of |c|
  const uint32_t* list_order;  // [K] lists by size, descending
  uint32_t dim, dpad, K;
  uint64_t N;
  uint32_t seg_rows;        // rows per scan segment (multiple of kRowBlock)
  uint32_t s_max;           // max candidate slots per list (segments x seg_split)
  // candidate slots per segment: 1, or 2 for the CTA-pair scan (k_scan_pair),
  // whose CTA c reports the segment's 128-row tiles of parity c as slot
  // 2*segment + c (slot_rows below)
  uint32_t seg_split;
  int metric;
  // filter bound of the scan kernel that produced the candidates:
  // |d32 - delta| <= e_a*|q|*|x| + e_b*(|q|^2 + |x|^2) + e_c
  double e_a, e_b, e_c;
  // fp16 filter copy: the lists again, each row
  // scaled by its list's power of two 2^e_l and rounded to fp16, in the same
  // tile-major SWIZZLE_64B layout (64 B = 32 dims per chunk row).  Set only in
  // views of the single-pass tensor-core scan over an index that has it (the
  // bound above is then bound_h16); nullptr otherwise.
  const float* vech;        // addressed in float units: dpf floats per row
  const float* lsc;         // [K] 2^-e_l (unscale of the list's rows)
  uint32_t dpf;             // floats per filter row: dpad, or ceil32(dim) / 2 with vech
};

// Programmatic dependent launch on the search path: each kernel is launched
// with cudaLaunchAttributeProgrammaticStreamSerialization and waits for its
// predecessor's completion (griddepcontrol.wait) as its first instruction, so
// the launch of kernel i+1 overlaps the tail of kernel i instead of following
// it.  No early trigger: dependents never occupy SM slots while they wait.
// Env HIVF_PDL=0 turns it off (plain stream order).
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  (void)cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...);
}

#ifdef __CUDACC__
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// candidate slots of a list of `rows` rows
__device__ __forceinline__ uint32_t slots_of(const IndexView& ix, uint64_t rows) {
  return (uint32_t)((rows + ix.seg_rows - 1) / ix.seg_rows) * ix.seg_split;
}
// i-th row (list-local) of slot `slot` of a list with n_c rows, or ~0 past its end
__device__ __forceinline__ uint64_t slot_row(const IndexView& ix, uint32_t slot, uint64_t n_c, uint64_t i) {
  const uint64_t s0 = (uint64_t)(slot / ix.seg_split) * ix.seg_rows;
  const uint64_t s1 = n_c < s0 + ix.seg_rows ? n_c : s0 + ix.seg_rows;
  uint64_t r;
  if (ix.seg_split == 1) {
    r = s0 + i;
  } else {  // tiles of parity slot % 2
    r = s0 + ((i >> 7) * 2 + (slot & 1)) * 128 + (i & 127);
  }
  return r < s1 ? r : ~0ull;
}
// base of list c's chunk-major block (swz_offset(0, n_c, row, d) indexes into it)
__device__ __forceinline__ const float* list_base(const IndexView& ix, uint32_t c, uint64_t lbeg) {
  return ix.list_ptr ? ix.list_ptr[c] : ix.vec + lbeg * ix.dpad;
}
#endif

// Per-batch query state (search space).
struct QueryView {
  const float* qs;      // [nq][dpad] search-space queries, zero padded
  const float* qn2;     // [nq] fp32(|q|^2)
  const float* qnorm;   // [nq] upper bound of |q|
  const float* qsc;     // [nq] 2^-e_q, the fp16 filter's unscale of the query (0: out of range)
  uint32_t n;
};

// ---- layout.cu
// tiered residency: list-table entries updated by value through kernel args
constexpr int kPtrFlipBatch = 64;
struct PtrFlips {
  uint32_t n;
  uint32_t list[kPtrFlipBatch];
  const float* ptr[kPtrFlipBatch];
};
void launch_ptr_flips(const float** table, const PtrFlips& f, cudaStream_t s);
void launch_locate(const uint64_t* sorted_ids, const uint64_t* sorted_rows, uint64_t N, const uint64_t* list_off,
                   uint32_t K, const uint64_t* q, uint32_t n, uint32_t* cl_out, uint64_t* row_out, cudaStream_t s);
void launch_gather_rows(const IndexView& ix, const uint64_t* rows, uint32_t n, float* out, cudaStream_t s);
void launch_iota64(uint64_t* v, uint64_t n, cudaStream_t s);
void launch_pack_lists(const float* src_rows, uint64_t r_first, const uint64_t* pos,
                       uint64_t n_rows, uint32_t dim, uint32_t dpad, const uint64_t* d_list_off,
                       uint32_t K, float* dst, float* xnorm2, uint32_t* maxnorm_bits, int* err,
                       cudaStream_t s);
void launch_unpack_rows(const float* vec, const uint64_t* d_list_off, uint32_t K, uint32_t dim,
                        uint32_t dpad, uint64_t first, uint64_t n, float* out, cudaStream_t s);
void launch_pack_centroids(const float* src, uint32_t K, uint32_t dim, uint32_t dpad, float* dst,
                           float* cnorm2, float* cnorm, int* err, cudaStream_t s);
void launch_mean_assigned(const IndexView& ix, double* partial, uint32_t n_partial,
                          cudaStream_t s, double* row_dist = nullptr);
void launch_scatter_ids(const uint64_t* ids, const uint64_t* pos, uint64_t n, uint64_t* out,
                        cudaStream_t s);
void launch_check_dup_ids(const uint64_t* sorted_ids, uint64_t n, int* err, cudaStream_t s);

// ---- assign.cu
void launch_prep_queries(const float* q_in, uint32_t n, uint32_t dim, uint32_t dpad, int metric,
                         bool normalize, float* qs, float* qn2, float* qnorm, float* qsc, int* err,
                         cudaStream_t s);
// fp16 filter copy: per-list scale exponent from the list's norm bound
// (|x_i| 2^e < 2^15), 0 for empty lists; the same rule per query (h16_exp)
__host__ __device__ inline int h16_exp(float norm_bound) {
  if (!(norm_bound > 0.f)) return 0;
  int e2 = 0;
#ifdef __CUDA_ARCH__
  e2 = ilogbf(norm_bound);
#else
  e2 = std::ilogb(norm_bound);
#endif
  return 14 - e2;
}
constexpr int kH16ExpMax = 60;  // |e| beyond this: the scale products could leave the fp32 normal range
void launch_pack_h16(const float* vec, const uint64_t* d_list_off, uint32_t K, uint32_t dpad, uint32_t dpf,
                     uint64_t N, const float* lsc, float* vech, cudaStream_t s);
// part (optional, coarse_dist_splits() x n_queries x K floats): scratch for the
// split-K form on small batches / codebooks
uint32_t coarse_dist_splits(const IndexView& ix, uint32_t n_queries);
void launch_coarse_dist(const IndexView& ix, const QueryView& qv, float* dist32, cudaStream_t s,
                        float* part = nullptr);
// Filter bound of the coarse distances: |d^ - delta| <= ea |q||c| + eb (|q|^2 + |c|^2)
// + ec + es |q| (rounded up).  FFMA pass: the fp32 filter's eps (coarse_bound_ffma);
// tensor-core pass: bound_h16 + the fp16 subnormal floor of the shared centroid
// scale (coarse_bound_h16).
struct CoarseBound {
  double ea, eb, ec, es;
};
CoarseBound coarse_bound_ffma(uint32_t dim);
CoarseBound coarse_bound_h16(uint32_t dim, float cmax);
void launch_coarse_select(const IndexView& ix, const QueryView& qv, const float* dist32,
                          uint32_t nprobe, const CoarseBound& bd, uint32_t* plans, double* dists, int* flags,
                          cudaStream_t s, bool set_mode = false);
// ---- scan_tc.cu: coarse distances on the tensor cores (kind::f16 GEMM over
// fp16 copies of the centroids and the queries in a 128-row tile layout)
uint32_t coarse_tc_stages(uint32_t dpad);
uint64_t coarse_tc_bytes(uint32_t rows, uint32_t dpad);
void launch_pack_coarse_tc(const float* src, uint32_t n, uint32_t dpad, const float* rsc, float sc, uint8_t* dst,
                           cudaStream_t s);
void launch_coarse_dist_tc(const IndexView& ix, const QueryView& qv, const uint8_t* cent_h16, float csc,
                           const uint8_t* q_h16, float* dist32, cudaStream_t s);
cudaError_t launch_coarse_all(const IndexView& ix, const QueryView& qv, uint32_t nprobe, uint32_t* plans,
                              double* dists, void* scratch, size_t* scratch_bytes, cudaStream_t s);
void launch_coarse_fallback(const IndexView& ix, const QueryView& qv, uint32_t nprobe,
                            uint32_t* plans, double* dists, const int* flags, cudaStream_t s);

// ---- scan.cu
// Pair p = (query pair_query[p], cluster pair_list[p]); output slots
// [p*s_max, p*s_max + nseg(list)).
void launch_build_worklist(const IndexView& ix, uint32_t group, const uint32_t* pair_query,
                           const uint32_t* pair_list, uint32_t n_pairs, uint32_t* list_cnt,
                           uint32_t* list_pair_off, uint32_t* list_cursor,
                           uint32_t* list_item_off, uint32_t* sorted_pairs, ScanItem* items,
                           uint32_t* n_items, uint32_t* work_ctr, uint32_t* qshift, cudaStream_t s);
void launch_scan(const IndexView& ix, const QueryView& qv, const ScanItem* items,
                 const uint32_t* n_items, uint32_t* work_ctr, const uint32_t* sorted_pairs,
                 const uint32_t* pair_query, float* out_d, uint32_t* out_row, float* out_thr,
                 uint32_t* out_n, int n_ctas, cudaStream_t s);
int scan_smem_bytes(uint32_t dpad);
// ---- scan_tc.cu (tcgen05 tensor-core scan)
// Wide tensor-core scan (query groups of kTcWideQ, dense batches): the
// restaged query rows (launch_stage_wide) and per-list staging shifts
// (launch_build_worklist's qshift).  Unused (zeros) for the narrow scan.
constexpr uint32_t kTcWideQ = 64;
// 128-query groups (k_scan_tc<128>, dense batches): half as many list passes
// as 64-query groups, 16-deep per-warp candidate lists
constexpr uint32_t kTcWide2Q = 128;
// 256-query groups on a CTA pair (k_scan_pair, cta_group::2), densest batches;
// candidate slots per segment x2 (IndexView::seg_split)
constexpr uint32_t kTcPairQ = 256;
inline bool tc_is_wide(uint32_t q) { return q == kTcWideQ || q == kTcWide2Q || q == kTcPairQ; }
struct WideStage {
  uint8_t* qstage = nullptr;  // wide_stage_rows() x dpad floats
  uint32_t* qshift = nullptr;
  uint32_t group = kTcWideQ;  // staged query-group size (the scan's qmax)
};
uint64_t wide_stage_rows(uint32_t n_pairs, uint32_t n_lists);
void launch_stage_wide(const IndexView& ix, const QueryView& qv, const uint32_t* sorted_pairs,
                       const uint32_t* pair_query, const uint32_t* pair_list, const uint32_t* pair_off,
                       const uint32_t* list_cnt, uint32_t n_pairs, const WideStage& ws, cudaStream_t s);
void launch_scan_tc(const IndexView& ix, const QueryView& qv, const ScanItem* items,
                    const uint32_t* n_items, uint32_t* work_ctr, const uint32_t* sorted_pairs,
                    const uint32_t* pair_query, float* out_d, uint32_t* out_row, float* out_thr,
                    uint32_t* out_n, int n_ctas, int split, float* qbound, uint32_t topk,
                    int bound_update, float probes_per_list, const WideStage& ws, const TcOpts& o,
                    cudaStream_t s);
// queries per tensor-core work item; probes_per_list = the batch's pairs / lists
uint32_t scan_tc_qmax(uint32_t dpad, int split, float probes_per_list, const TcOpts& o);
// fp32->tf32 operand conversion of the current device's tensor cores, probed
// once per device (0 trunc, 1 RNE, 2 unsupported -> FFMA scan)
int tc_conversion_mode();
void set_tc_prof(int on);    // debug: per-CTA stall counters in k_scan_tc (process-wide)
int scan_tc_smem_bytes(uint32_t dpad, int split, float probes_per_list, const TcOpts& o);
void bound_ffma(uint32_t dim, double* a, double* b, double* c);
void bound_tc(uint32_t dim, double* a, double* b, double* c);   // 3-pass split
void bound_tc1(uint32_t dim, double* a, double* b, double* c);  // single pass
void bound_h16(uint32_t dim, double* a, double* b, double* c);  // single pass over the fp16 filter copy

// ---- kmeans.cu (index build: train_kmeans / Lloyd, vector_index.cpp:99-200)
void launch_kmeans_dist2(const float* X, uint64_t n, uint32_t dim, const float* c, double* dist2, int mode,
                         cudaStream_t s);
void launch_kmeans_prefix(const double* dist2, uint64_t n, double* prefix, double* total, cudaStream_t s);
void launch_kmeans_pick(const double* prefix, uint64_t n, const double* total, const double* us, int* draw,
                        uint64_t* pick, int* zero, const float* X, uint32_t dim, float* cents, uint32_t m,
                        cudaStream_t s);
void launch_iota(uint32_t* v, uint64_t n, cudaStream_t s);
void launch_same_assign(const uint32_t* a, uint32_t* prev, uint64_t n, int* differs, cudaStream_t s);
void launch_cluster_means(const float* X, uint32_t dim, uint32_t K, const uint32_t* sorted_keys,
                          const uint32_t* sorted_idx, uint64_t n, uint64_t* off, float* cents,
                          cudaStream_t s);
void launch_far_point(const float* X, uint64_t n, uint32_t dim, const uint32_t* assign, const float* new_c,
                      const float* old_c, uint32_t c, uint8_t* used, double* dd, unsigned long long* scratch2,
                      cudaStream_t s);

// ---- finalize.cu
// In-place repair of segments whose completeness proof failed (finalize.cu).
struct RepairState {
  uint64_t* entries;  // (query << 32 | plan position * s_max + segment)
  uint32_t* n;        // entries used (device counter, zeroed per call)
  uint32_t cap;       // entries capacity
  uint32_t* cnt;      // [n_queries] exact survivors per query
  double* d;          // [n_queries][per_query]
  uint64_t* ids;      // [n_queries][per_query]
  uint32_t per_query;
};
void launch_repair(const IndexView& ix, const QueryView& qv, const uint32_t* plans, uint32_t nprobe,
                   uint32_t k, const float* cand_d, const uint32_t* cand_row, const float* cand_thr,
                   const uint32_t* cand_n, const float* tau, const RepairState& R, int n_ctas,
                   uint64_t* ids_out, double* d_out, uint32_t* counts_out, int* flags, cudaStream_t s);
void launch_plans_to_pairs(const uint32_t* plans, uint32_t n_queries, uint32_t nprobe, uint32_t K,
                           uint32_t* pair_query, uint32_t* pair_list, uint32_t* plans_out, int* err,
                           cudaStream_t s);
void launch_finalize_search(const IndexView& ix, const QueryView& qv, const uint32_t* plans,
                            uint32_t nprobe, uint32_t k, const float* cand_d,
                            const uint32_t* cand_row, const float* cand_thr,
                            const uint32_t* cand_n, uint64_t* ids_out, double* d_out,
                            uint32_t* counts_out, int* flags, float* tau_out,
                            const RepairState* rep, cudaStream_t s);
// part_* scratch (n_queries x exact_search_parts() x k) enables the multi-CTA
// path; pass nullptr for one CTA per query.
uint32_t exact_search_parts(uint32_t nprobe, uint32_t k);
// seed of the shared drop bound: exact distances of `rows` (<= 64) rows of each
// query's nearest probed list (finalize.cu)
void launch_seed_bounds(const IndexView& ix, const QueryView& qv, const uint32_t* plans, uint32_t nprobe,
                        uint32_t k, uint32_t rows, float* qbound, cudaStream_t s);
void launch_exact_search(const IndexView& ix, const QueryView& qv, const uint32_t* plans,
                         uint32_t nprobe, uint32_t k, const int* flags, uint64_t* ids_out,
                         double* d_out, uint32_t* counts_out, uint64_t* part_ids,
                         double* part_d, uint32_t* part_cnt, uint64_t* part_total,
                         const float* tau, cudaStream_t s);
// node-split drop bounds: float_ru(heap worst) for full heaps, "none" otherwise
void launch_item_bounds(const double* heap_d, const uint32_t* heap_n, const uint32_t* k, uint32_t stride,
                        uint32_t n_items, float* out, cudaStream_t s);
void launch_finalize_items(const IndexView& ix, const QueryView& qv, uint32_t n_items,
                           const uint32_t* item_off, const uint32_t* clusters, const uint32_t* k,
                           const float* cand_d, const uint32_t* cand_row, const float* cand_thr,
                           const uint32_t* cand_n, uint64_t* heap_ids, double* heap_d,
                           uint32_t* heap_n, uint32_t heap_stride, uint8_t* changed, int* flags,
                           cudaStream_t s);
void launch_exact_items(const IndexView& ix, const QueryView& qv, uint32_t n_items,
                        const uint32_t* item_off, const uint32_t* clusters, const uint32_t* k,
                        uint64_t* heap_ids, double* heap_d, uint32_t* heap_n,
                        uint32_t heap_stride, uint8_t* changed, const int* flags,
                        cudaStream_t s);
void launch_merge_parts(uint32_t n_parts, uint32_t n_queries, uint32_t k, const uint64_t* ids,
                        const double* d, const uint32_t* counts, uint64_t* ids_out,
                        double* d_out, uint32_t* counts_out, cudaStream_t s);

void launch_merge_parts_strided(uint32_t n_parts, uint32_t n_queries, uint32_t k, const uint64_t* ids,
                                const double* d, const uint32_t* counts, uint64_t s_ids, uint64_t s_d,
                                uint64_t s_cnt, uint64_t* ids_out, double* d_out, uint32_t* counts_out,
                                cudaStream_t s);
// shard.cu: device-side all-gather over peer pointers (in-process shard group)
constexpr int kMaxGroup = 16;
struct PeerSrc {
  const void* src[kMaxGroup];
};
void launch_gather_peer(const PeerSrc& src, uint32_t n_src, uint64_t bytes_each, void* dst, cudaStream_t s);

constexpr uint32_t kExactMaxK = 4096;     // exact-path heap bound
constexpr uint32_t kNprobeMax = 4096;     // exact coarse-assign bound

}  // namespace hivf
