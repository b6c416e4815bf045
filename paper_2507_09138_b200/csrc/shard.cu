// shard.cu -- multi-GPU list sharding.
//
// Inverted lists are independent units: every GPU holds the centroids and a
// disjoint share of the list rows (whole lists by frequency-weighted LPT, the
// hottest lists striped by rows over all GPUs), searches its share exactly,
// and the per-GPU top-k lists are merged with merge_topk
// (/root/reference/proj/src/vector_index.cpp:71-91).  Per batch:
//
//   1. rank r assigns its slice of the batch (ivf::select_clusters,
//      vector_index.cpp:261-278) -- the plans are identical to a full assign;
//   2. all-gather of the plans;
//   3. every rank searches its share with the full plans
//      (hivf_search_planned_device: make_cursor + search_step, :280-328);
//   4. all-gather (in-process: gather to member 0) of one packed
//      ids|dists|counts block per rank, then k_merge_parts on device.
//
// Exact because the shares are disjoint and every row of a probed list is on
// exactly one GPU.  Three exchange transports behind the same steps:
//   * in-process group (one host thread drives N contexts, e.g. one per GPU of
//     the box): a gather kernel that reads the other members' buffers through
//     peer pointers (NVLink P2P; plain loads when two members share a device),
//     ordered with events -- no NCCL needed;
//   * NCCL (one process per GPU, torchrun): ncclAllGather on the context
//     stream; libnccl is dlopen'ed on first use (the copy torch already
//     loaded, else the system one), so the library has no link-time NCCL
//     dependency;
//   * host callback (one process per rank, any all-gather the caller has, e.g.
//     torch.distributed over gloo): staged through pinned host memory.  Lets
//     the per-rank path run with several ranks on one GPU, which NCCL refuses.
#include <dlfcn.h>
#include <nccl.h>

#include <mutex>
#include <numeric>

#include "internal.h"

namespace hivf {
namespace {

__global__ void __launch_bounds__(256) k_gather_peer(PeerSrc src, uint32_t n_src, uint64_t n16, uint4* dst) {
  const uint64_t total = (uint64_t)n_src * n16;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t j = (uint32_t)(i / n16);
    dst[i] = reinterpret_cast<const uint4*>(src.src[j])[i - (uint64_t)j * n16];
  }
}

}  // namespace

void launch_gather_peer(const PeerSrc& src, uint32_t n_src, uint64_t bytes_each, void* dst, cudaStream_t s) {
  const uint64_t n16 = bytes_each / 16, total = n16 * n_src;
  if (!total) return;
  const int blocks = (int)std::min<uint64_t>((total + 255) / 256, 2ull * device_sm_count());
  k_gather_peer<<<blocks, 256, 0, s>>>(src, n_src, n16, reinterpret_cast<uint4*>(dst));
}

}  // namespace hivf

namespace {

// ---- NCCL, loaded at run time ----------------------------------------------
struct NcclApi {
  bool loaded = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi* nccl() {
  static std::once_flag once;
  static NcclApi api;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("dlopen libnccl.so.2: ") + dlerror();
      return;
    }
    api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
    api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
    api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
    api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
    api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
    api.loaded = api.GetUniqueId && api.CommInitRank && api.AllGather && api.CommDestroy && api.GetErrorString;
    if (!api.loaded) api.why = "libnccl.so.2 lacks a required symbol";
  });
  return &api;
}

#define NCK(call)                                                                                  \
  do {                                                                                             \
    ncclResult_t r_ = (call);                                                                      \
    if (r_ != ncclSuccess)                                                                         \
      return fail(HIVF_ECOMM, "%s: %s (%s:%d)", #call, nccl()->GetErrorString(r_), __FILE__, __LINE__); \
  } while (0)

}  // namespace

struct hivf_group {
  enum Kind { kPeer, kNccl, kHostCb } kind = kPeer;
  uint32_t nranks = 1, rank = 0;  // in-process: nranks = members, rank 0 = the caller's member
  struct Member {
    hivf_index* ix = nullptr;
    DBuf q, plans_loc, plans_all, packed, gathered, out;
    cudaEvent_t ready = nullptr, done = nullptr;
  };
  std::vector<Member> m;  // local members (in-process: all; per-rank: this rank)
  bool p2p_loads = true;  // in-process: every member pair can load each other's memory
  bool first = true;
  cudaEvent_t start = nullptr;
  ncclComm_t comm = nullptr;
  hivf_allgather_fn cb = nullptr;
  void* cb_user = nullptr;
  HBuf hs, hr, hio;
  ~hivf_group() {
    for (auto& x : m) {
      cudaSetDevice(x.ix->ctx->device);
      cudaStreamSynchronize(x.ix->ctx->stream);
      for (DBuf* b : {&x.q, &x.plans_loc, &x.plans_all, &x.packed, &x.gathered, &x.out}) b->release();
      if (x.ready) cudaEventDestroy(x.ready);
      if (x.done) cudaEventDestroy(x.done);
    }
    if (start) cudaEventDestroy(start);
    if (comm) nccl()->CommDestroy(comm);
    hs.release();
    hr.release();
    hio.release();
  }
};

namespace {

hivf_status check_member(hivf_index* ix) {
  if (!ix) return fail(HIVF_EINVAL, "shard group: NULL index");
  if (!ix->finished) return fail(HIVF_EINVAL, "shard group: index not finished");
  if (ix->tiered) return fail(HIVF_EUNSUPPORTED, "shard group: tiered (hbm_list_budget) shards");
  return HIVF_OK;
}

hivf_status new_events(hivf_group::Member& x) {
  CK(cudaSetDevice(x.ix->ctx->device));
  CK(cudaEventCreateWithFlags(&x.ready, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&x.done, cudaEventDisableTiming));
  return HIVF_OK;
}

// per-rank all-gather of `bytes` (multiple of 16) from send into recv[nranks][bytes]
hivf_status rank_allgather(hivf_group* g, const void* send, size_t bytes, void* recv) {
  hivf_ctx* c = g->m[0].ix->ctx;
  if (g->kind == hivf_group::kNccl) {
    NCK(nccl()->AllGather(send, recv, bytes, ncclUint8, g->comm, c->stream));
    return HIVF_OK;
  }
  CK(g->hs.ensure(bytes));
  CK(g->hr.ensure(bytes * g->nranks));
  CK(cudaMemcpyAsync(g->hs.p, send, bytes, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (g->cb(g->cb_user, g->hs.p, bytes, g->hr.p) != 0)
    return fail(HIVF_ECOMM, "shard group: all-gather callback failed");
  CK(cudaMemcpyAsync(recv, g->hr.p, bytes * g->nranks, cudaMemcpyHostToDevice, c->stream));
  return HIVF_OK;
}

// member m's recv[j] <- member j's buffer `which` (in-process group)
hivf_status peer_gather(hivf_group* g, uint32_t mi, DBuf hivf_group::Member::*which, size_t bytes,
                        void* recv) {
  auto& x = g->m[mi];
  hivf_ctx* c = x.ix->ctx;
  CK(cudaSetDevice(c->device));
  for (auto& y : g->m) CK(cudaStreamWaitEvent(c->stream, y.ready, 0));
  if (g->p2p_loads) {
    PeerSrc src{};
    for (uint32_t j = 0; j < g->m.size(); ++j) src.src[j] = (g->m[j].*which).p;
    launch_gather_peer(src, (uint32_t)g->m.size(), bytes, recv, c->stream);
    CKL();
    c->stats.kernels_launched += 1;
  } else {
    for (uint32_t j = 0; j < g->m.size(); ++j)
      CK(cudaMemcpyPeerAsync(static_cast<uint8_t*>(recv) + j * bytes, c->device, (g->m[j].*which).p,
                             g->m[j].ix->ctx->device, bytes, c->stream));
  }
  return HIVF_OK;
}

inline size_t up16(size_t b) { return (b + 15) & ~size_t(15); }

// The sharded search (steps 1-4 above).  d_queries / outputs live on member
// 0's device (in-process) or this rank's device (per-rank), in the stream
// order of that member's context stream.
hivf_status group_search(hivf_group* g, const float* d_queries, uint32_t n, uint32_t nprobe, uint32_t k,
                         uint64_t* d_ids, double* d_dists, uint32_t* d_counts) {
  const uint32_t N = g->nranks, L = (uint32_t)g->m.size();
  hivf_index* ix0 = g->m[0].ix;
  const uint32_t dim = ix0->dim;
  // rank r assigns rows [r*bs, min(n, (r+1)*bs)); bs is a multiple of 4 so a
  // plan slice is 16-byte aligned and the gathered slices are one [N*bs][nprobe] array
  const uint32_t bs = ((n + N - 1) / N + 3) & ~3u;
  const size_t plan_bytes = (size_t)bs * nprobe * 4;
  const size_t nk = (size_t)n * k;
  const size_t part_bytes = up16(16 * nk + 4 * (size_t)n);
  hivf_status st;
  if (g->kind == hivf_group::kPeer) {
    // previous call's readers are done before any member overwrites a buffer
    // they read (stream 0 waits for every member, the others wait for stream 0)
    hivf_ctx* c0 = ix0->ctx;
    CK(cudaSetDevice(c0->device));
    if (!g->first)
      for (auto& y : g->m) CK(cudaStreamWaitEvent(c0->stream, y.done, 0));
    CK(cudaEventRecord(g->start, c0->stream));
  }
  g->first = false;
  for (uint32_t mi = 0; mi < L; ++mi) {  // 1. queries on every member, slice assign
    auto& x = g->m[mi];
    hivf_ctx* c = x.ix->ctx;
    const uint32_t r = g->kind == hivf_group::kPeer ? mi : g->rank;
    CK(cudaSetDevice(c->device));
    const float* q = d_queries;
    if (g->kind == hivf_group::kPeer && mi > 0) {
      CK(cudaStreamWaitEvent(c->stream, g->start, 0));
      CK(x.q.ensure((size_t)n * dim * 4));
      CK(cudaMemcpyPeerAsync(x.q.p, c->device, d_queries, ix0->ctx->device, (size_t)n * dim * 4, c->stream));
      q = x.q.as<float>();
    }
    CK(x.plans_loc.ensure(plan_bytes));
    CK(x.plans_all.ensure(plan_bytes * N));
    CK(x.packed.ensure(part_bytes));
    const uint32_t lo = std::min(n, r * bs), hi = std::min(n, lo + bs);
    if (hi > lo)
      if ((st = hivf_assign_device(x.ix, q + (size_t)lo * dim, hi - lo, nprobe, x.plans_loc.as<uint32_t>(),
                                   nullptr)) != HIVF_OK)
        return st;
    if (g->kind == hivf_group::kPeer) CK(cudaEventRecord(x.ready, c->stream));
  }
  for (uint32_t mi = 0; mi < L; ++mi) {  // 2. plan all-gather
    auto& x = g->m[mi];
    if (g->kind == hivf_group::kPeer) {
      if ((st = peer_gather(g, mi, &hivf_group::Member::plans_loc, plan_bytes, x.plans_all.p)) != HIVF_OK)
        return st;
    } else if ((st = rank_allgather(g, x.plans_loc.p, plan_bytes, x.plans_all.p)) != HIVF_OK) {
      return st;
    }
  }
  for (uint32_t mi = 0; mi < L; ++mi) {  // 3. local exact search of this member's share
    auto& x = g->m[mi];
    hivf_ctx* c = x.ix->ctx;
    const float* q = (g->kind == hivf_group::kPeer && mi > 0) ? x.q.as<float>() : d_queries;
    uint8_t* pk = x.packed.as<uint8_t>();
    if ((st = hivf_search_planned_device(x.ix, q, n, nprobe, k, x.plans_all.as<uint32_t>(),
                                         reinterpret_cast<uint64_t*>(pk), reinterpret_cast<double*>(pk + 8 * nk),
                                         reinterpret_cast<uint32_t*>(pk + 16 * nk))) != HIVF_OK)
      return st;
    if (g->kind == hivf_group::kPeer) {
      CK(cudaSetDevice(c->device));
      CK(cudaEventRecord(x.ready, c->stream));
    }
  }
  // 4. result exchange + merge_topk on device (in-process: member 0 only)
  auto& x = g->m[0];
  hivf_ctx* c = x.ix->ctx;
  CK(cudaSetDevice(c->device));
  CK(x.gathered.ensure(part_bytes * N));
  if (g->kind == hivf_group::kPeer) {
    if ((st = peer_gather(g, 0, &hivf_group::Member::packed, part_bytes, x.gathered.p)) != HIVF_OK) return st;
  } else if ((st = rank_allgather(g, x.packed.p, part_bytes, x.gathered.p)) != HIVF_OK) {
    return st;
  }
  CK(cudaSetDevice(c->device));
  const uint8_t* gb = x.gathered.as<uint8_t>();
  launch_merge_parts_strided(N, n, k, reinterpret_cast<const uint64_t*>(gb),
                             reinterpret_cast<const double*>(gb + 8 * nk),
                             reinterpret_cast<const uint32_t*>(gb + 16 * nk), part_bytes / 8, part_bytes / 8,
                             part_bytes / 4, d_ids, d_dists, d_counts, c->stream);
  CKL();
  c->stats.kernels_launched += 1;
  if (g->kind == hivf_group::kPeer)
    for (auto& y : g->m) {
      CK(cudaSetDevice(y.ix->ctx->device));
      CK(cudaEventRecord(y.done, y.ix->ctx->stream));
    }
  CK(cudaSetDevice(c->device));
  return HIVF_OK;
}

hivf_status check_group_args(hivf_group* g, uint32_t nprobe, uint32_t k) {
  if (!g) return fail(HIVF_EINVAL, "shard group is NULL");
  hivf_index* ix = g->m[0].ix;
  if (k == 0) return fail(HIVF_EINVAL, "make_cursor: k must be >= 1");
  if (nprobe < 1 || nprobe > ix->K) return fail(HIVF_EINVAL, "select_clusters: nprobe out of range");
  if ((uint64_t)g->nranks * k > 8192) return fail(HIVF_EUNSUPPORTED, "shard group: nranks * k > 8192");
  return HIVF_OK;
}

}  // namespace

extern "C" {

hivf_status hivf_shard_plan(const uint64_t* sizes, const double* weights, uint32_t n_clusters, uint32_t nranks,
                            int32_t n_striped, uint32_t* owner_out) {
  if (!sizes || !owner_out || !n_clusters || !nranks) return fail(HIVF_EINVAL, "hivf_shard_plan: bad argument");
  const uint32_t K = n_clusters;
  std::vector<double> load(K);
  double total = 0;
  for (uint32_t c = 0; c < K; ++c) {
    const double w = weights ? weights[c] : 1.0;
    if (!(w >= 0.0)) return fail(HIVF_EINVAL, "hivf_shard_plan: weights must be finite and >= 0");
    load[c] = (double)sizes[c] * w;
    total += load[c];
  }
  // hottest first: (load desc, id asc)
  std::vector<uint32_t> order(K);
  std::iota(order.begin(), order.end(), 0u);
  std::stable_sort(order.begin(), order.end(), [&](uint32_t a, uint32_t b) { return load[a] > load[b]; });
  uint32_t n_str = 0;
  if (nranks > 1) {
    if (n_striped < 0) {  // auto: stripe lists heavier than 1/16 of one rank's share
      const double cut = total / nranks / 16.0;
      while (n_str < K && load[order[n_str]] > cut) ++n_str;
    } else {
      n_str = std::min<uint32_t>((uint32_t)n_striped, K);
    }
  }
  std::vector<double> rank_load(nranks, 0.0);
  for (uint32_t i = 0; i < n_str; ++i) {
    owner_out[order[i]] = HIVF_SHARD_STRIPED;
    for (auto& r : rank_load) r += load[order[i]] / nranks;
  }
  // LPT: heaviest remaining list to the least-loaded rank (ties: lowest rank)
  for (uint32_t i = n_str; i < K; ++i) {
    uint32_t best = 0;
    for (uint32_t r = 1; r < nranks; ++r)
      if (rank_load[r] < rank_load[best]) best = r;
    owner_out[order[i]] = best;
    rank_load[best] += load[order[i]];
  }
  return HIVF_OK;
}

hivf_status hivf_shard_local_lists(const uint64_t* list_offsets, const uint32_t* owner, uint32_t n_clusters,
                                   uint32_t nranks, uint32_t rank, uint64_t* local_offsets_out,
                                   uint64_t* src_first_out) {
  if (!list_offsets || !owner || !local_offsets_out || !src_first_out || !nranks || rank >= nranks)
    return fail(HIVF_EINVAL, "hivf_shard_local_lists: bad argument");
  local_offsets_out[0] = 0;
  for (uint32_t c = 0; c < n_clusters; ++c) {
    const uint64_t b = list_offsets[c], n = list_offsets[c + 1] - b;
    if (list_offsets[c + 1] < b) return fail(HIVF_EINVAL, "hivf_shard_local_lists: offsets not monotone");
    uint64_t lo = 0, hi = 0;
    if (owner[c] == HIVF_SHARD_STRIPED) {
      lo = n * rank / nranks;
      hi = n * (rank + 1) / nranks;
    } else if (owner[c] == rank) {
      hi = n;
    } else if (owner[c] >= nranks) {
      return fail(HIVF_EINVAL, "hivf_shard_local_lists: owner[%u] = %u out of range", c, owner[c]);
    }
    src_first_out[c] = b + lo;
    local_offsets_out[c + 1] = local_offsets_out[c] + (hi - lo);
  }
  return HIVF_OK;
}

hivf_status hivf_index_upload_shard(hivf_ctx* ctx, uint32_t dim, int metric, uint32_t n_clusters,
                                    const float* centroids, const uint64_t* list_offsets, const float* vectors,
                                    const uint64_t* ids, const uint32_t* owner, uint32_t nranks, uint32_t rank,
                                    hivf_index** out) {
  if (!ctx || !list_offsets || !owner || !out) return fail(HIVF_EINVAL, "hivf_index_upload_shard: NULL argument");
  std::vector<uint64_t> loff(n_clusters + 1), first(n_clusters);
  hivf_status st = hivf_shard_local_lists(list_offsets, owner, n_clusters, nranks, rank, loff.data(), first.data());
  if (st != HIVF_OK) return st;
  const uint64_t nl = loff[n_clusters];
  if (nl && (!vectors || !ids)) return fail(HIVF_EINVAL, "hivf_index_upload_shard: NULL rows");
  std::vector<float> v(nl * dim);
  std::vector<uint64_t> id(nl);
  for (uint32_t c = 0; c < n_clusters; ++c) {
    const uint64_t m = loff[c + 1] - loff[c];
    if (!m) continue;
    std::memcpy(v.data() + loff[c] * dim, vectors + first[c] * dim, m * dim * 4);
    std::memcpy(id.data() + loff[c], ids + first[c], m * 8);
  }
  return hivf_index_upload(ctx, dim, metric, n_clusters, centroids, loff.data(), nl ? v.data() : nullptr,
                           nl ? id.data() : nullptr, out);
}

hivf_status hivf_group_create(hivf_index* const* shards, uint32_t n, hivf_group** out) {
  if (!shards || !out || n == 0) return fail(HIVF_EINVAL, "hivf_group_create: bad argument");
  if (n > (uint32_t)kMaxGroup) return fail(HIVF_EUNSUPPORTED, "hivf_group_create: more than %d members", kMaxGroup);
  hivf_status st;
  for (uint32_t i = 0; i < n; ++i) {
    if ((st = check_member(shards[i])) != HIVF_OK) return st;
    if (shards[i]->dim != shards[0]->dim || shards[i]->K != shards[0]->K || shards[i]->metric != shards[0]->metric)
      return fail(HIVF_EINVAL, "hivf_group_create: shards differ in dim / n_clusters / metric");
    for (uint32_t j = 0; j < i; ++j)
      if (shards[j]->ctx == shards[i]->ctx)
        return fail(HIVF_EINVAL, "hivf_group_create: two shards share a context (one context per member)");
  }
  auto* g = new hivf_group;
  g->kind = hivf_group::kPeer;
  g->nranks = n;
  g->m.resize(n);
  for (uint32_t i = 0; i < n; ++i) {
    g->m[i].ix = shards[i];
    if ((st = new_events(g->m[i])) != HIVF_OK) {
      delete g;
      return st;
    }
  }
  // direct peer loads need P2P access between every pair of distinct devices
  for (uint32_t i = 0; i < n; ++i)
    for (uint32_t j = 0; j < n; ++j) {
      const int a = shards[i]->ctx->device, b = shards[j]->ctx->device;
      if (a == b) continue;
      int can = 0;
      cudaDeviceCanAccessPeer(&can, a, b);
      if (!can) {
        g->p2p_loads = false;
        continue;
      }
      cudaSetDevice(a);
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) g->p2p_loads = false;
      (void)cudaGetLastError();
    }
  cudaSetDevice(shards[0]->ctx->device);
  if (cudaEventCreateWithFlags(&g->start, cudaEventDisableTiming) != cudaSuccess) {
    delete g;
    return fail(HIVF_ECUDA, "hivf_group_create: event");
  }
  *out = g;
  return HIVF_OK;
}

hivf_status hivf_nccl_unique_id(void* id_out) {
  if (!id_out) return fail(HIVF_EINVAL, "hivf_nccl_unique_id: NULL");
  NcclApi* api = nccl();
  if (!api->loaded) return fail(HIVF_EUNSUPPORTED, "NCCL unavailable: %s", api->why.c_str());
  ncclUniqueId id;
  NCK(api->GetUniqueId(&id));
  std::memcpy(id_out, &id, sizeof id);
  return HIVF_OK;
}

hivf_status hivf_group_create_nccl(hivf_index* shard, uint32_t nranks, uint32_t rank, const void* unique_id,
                                   hivf_group** out) {
  hivf_status st;
  if (!out || !unique_id || !nranks || rank >= nranks) return fail(HIVF_EINVAL, "hivf_group_create_nccl: bad argument");
  if ((st = check_member(shard)) != HIVF_OK) return st;
  NcclApi* api = nccl();
  if (!api->loaded) return fail(HIVF_EUNSUPPORTED, "NCCL unavailable: %s", api->why.c_str());
  CK(cudaSetDevice(shard->ctx->device));
  ncclUniqueId id;
  std::memcpy(&id, unique_id, sizeof id);
  ncclComm_t comm = nullptr;
  NCK(api->CommInitRank(&comm, (int)nranks, id, (int)rank));
  auto* g = new hivf_group;
  g->kind = hivf_group::kNccl;
  g->nranks = nranks;
  g->rank = rank;
  g->comm = comm;
  g->m.resize(1);
  g->m[0].ix = shard;
  *out = g;
  return HIVF_OK;
}

hivf_status hivf_group_create_hostcb(hivf_index* shard, uint32_t nranks, uint32_t rank, hivf_allgather_fn fn,
                                     void* user, hivf_group** out) {
  hivf_status st;
  if (!out || !fn || !nranks || rank >= nranks) return fail(HIVF_EINVAL, "hivf_group_create_hostcb: bad argument");
  if ((st = check_member(shard)) != HIVF_OK) return st;
  auto* g = new hivf_group;
  g->kind = hivf_group::kHostCb;
  g->nranks = nranks;
  g->rank = rank;
  g->cb = fn;
  g->cb_user = user;
  g->m.resize(1);
  g->m[0].ix = shard;
  *out = g;
  return HIVF_OK;
}

hivf_status hivf_group_destroy(hivf_group* g) {
  delete g;
  return HIVF_OK;
}

hivf_status hivf_group_search_device(hivf_group* g, const float* d_queries, uint32_t n, uint32_t nprobe,
                                     uint32_t k, uint64_t* d_ids_out, double* d_dists_out,
                                     uint32_t* d_counts_out) {
  hivf_status st = check_group_args(g, nprobe, k);
  if (st != HIVF_OK) return st;
  if (n == 0) return HIVF_OK;
  if (!d_queries || !d_ids_out || !d_dists_out || !d_counts_out)
    return fail(HIVF_EINVAL, "hivf_group_search_device: NULL buffer");
  return group_search(g, d_queries, n, nprobe, k, d_ids_out, d_dists_out, d_counts_out);
}

hivf_status hivf_group_search(hivf_group* g, const float* queries, uint32_t n, uint32_t nprobe, uint32_t k,
                              uint64_t* ids_out, double* dists_out, uint32_t* counts_out) {
  hivf_status st = check_group_args(g, nprobe, k);
  if (st != HIVF_OK) return st;
  if (n == 0) return HIVF_OK;
  if (!queries || !ids_out || !dists_out || !counts_out) return fail(HIVF_EINVAL, "hivf_group_search: NULL buffer");
  auto& x = g->m[0];
  hivf_ctx* c = x.ix->ctx;
  CK(cudaSetDevice(c->device));
  const size_t qb = (size_t)n * x.ix->dim * 4, nk = (size_t)n * k, ob = 16 * nk + 4 * (size_t)n;
  // one pinned staging block: queries in, ids|dists|counts out
  CK(g->hio.ensure(std::max(qb, ob)));
  CK(x.out.ensure(up16(qb) + ob));
  std::memcpy(g->hio.p, queries, qb);
  uint8_t* dq = x.out.as<uint8_t>();
  uint8_t* dres = dq + up16(qb);
  CK(cudaMemcpyAsync(dq, g->hio.p, qb, cudaMemcpyHostToDevice, c->stream));
  if ((st = group_search(g, reinterpret_cast<const float*>(dq), n, nprobe, k, reinterpret_cast<uint64_t*>(dres),
                         reinterpret_cast<double*>(dres + 8 * nk), reinterpret_cast<uint32_t*>(dres + 16 * nk))) !=
      HIVF_OK)
    return st;
  CK(cudaMemcpyAsync(g->hio.p, dres, ob, cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const uint8_t* h = g->hio.as<uint8_t>();
  std::memcpy(ids_out, h, 8 * nk);
  std::memcpy(dists_out, h + 8 * nk, 8 * nk);
  std::memcpy(counts_out, h + 16 * nk, 4 * (size_t)n);
  return HIVF_OK;
}

}  // extern "C"
