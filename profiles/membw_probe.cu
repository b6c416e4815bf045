// Read-bandwidth ceiling probe: persistent CTAs stream a large buffer through a
// bulk-copy smem ring (the k_scan_tc producer pattern) and release stages
// immediately.  Sweeps ring depth / copy size / CTAs per SM.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
#include "../paper_2507_09138_b200/csrc/common.cuh"
using namespace hivf;

struct P { const uint8_t* src; uint64_t bytes; uint32_t copy; uint32_t stages; uint32_t per_stage; uint32_t* ctr; uint64_t chunk_per_item; uint32_t* sink; int planes; };

__global__ void k_stream(P p) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint64_t full[16];
  __shared__ uint64_t empty[16];
  __shared__ uint64_t s_it;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < p.stages; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
    fence_barrier_init();
  }
  __syncthreads();
  const uint64_t stage_bytes = (uint64_t)p.copy * p.per_stage;
  const uint64_t n_items = p.bytes / p.chunk_per_item;
  const uint32_t stages_per_item = (uint32_t)(p.chunk_per_item / stage_bytes);
  uint32_t s = 0, ph = 0;
  uint32_t acc = 0;
  for (;;) {
    if (threadIdx.x == 0) s_it = atomicAdd(p.ctr, 1u);
    __syncthreads();
    const uint64_t it = s_it;
    __syncthreads();
    if (it >= n_items) break;
    const uint8_t* base = p.src + it * p.chunk_per_item;
    if (warp == 0) {
      if (lane == 0) {
        for (uint32_t st = 0; st < stages_per_item; ++st) {
          mbar_wait(&empty[s], ph ^ 1);
          mbar_arrive_expect_tx(&full[s], (uint32_t)stage_bytes);
          if (p.planes) {  // chunk-major list layout: 48 planes of n_rows*64 B, tile = 128 rows
            const uint64_t n_rows = p.chunk_per_item / 3072;
            const uint32_t spt = 12;  // stages per 128-row tile (768 dims / 64)
            const uint32_t t = st / spt, sg = st % spt;
            for (uint32_t c = 0; c < 4; ++c)
              bulk_g2s(sm + s * stage_bytes + c * 8192, base + (uint64_t)(sg * 4 + c) * n_rows * 64 + (uint64_t)t * 8192, 8192, &full[s]);
          } else
          for (uint32_t c = 0; c < p.per_stage; ++c)
            bulk_g2s(sm + s * stage_bytes + c * p.copy, base + (uint64_t)st * stage_bytes + (uint64_t)c * p.copy, p.copy, &full[s]);
          if (++s == p.stages) { s = 0; ph ^= 1; }
        }
      }
    } else if (warp == 1) {
      for (uint32_t st = 0; st < stages_per_item; ++st) {
        mbar_wait(&full[s], ph);
        acc += reinterpret_cast<const uint32_t*>(sm + s * stage_bytes)[lane];
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[s]);
        if (++s == p.stages) { s = 0; ph ^= 1; }
      }
    }
  }
  if (acc == 0x12345678u) *p.sink = acc;
}

__global__ void k_ldg(const float4* __restrict__ src, uint64_t n4, uint32_t* sink) {
  float acc = 0.f;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  for (; i + 3 * stride < n4; i += 4 * stride) {
    float4 a = __ldcs(src + i), b = __ldcs(src + i + stride), c = __ldcs(src + i + 2 * stride), d = __ldcs(src + i + 3 * stride);
    acc += a.x + b.y + c.z + d.w;
  }
  for (; i < n4; i += stride) acc += __ldcs(src + i).x;
  if (acc == 1234.5f) *sink = 1;
}

int main(int argc, char** argv) {
  const uint64_t bytes = 16ull << 30;
  uint8_t* d; cudaMalloc(&d, bytes); cudaMemset(d, 1, bytes);
  uint32_t* ctr; cudaMalloc(&ctr, 4);
  uint32_t* sink; cudaMalloc(&sink, 4);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaFuncSetAttribute(k_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  struct Cfg { uint32_t copy, per_stage, stages, ctas_per_sm; uint64_t item; int planes = 0; };
  std::vector<Cfg> cfgs;
  cfgs.push_back({8192, 4, 3, 1, 2u << 20});
  cfgs.push_back({8192, 4, 3, 1, 3072ull * 4096, 0});
  cfgs.push_back({8192, 4, 3, 1, 3072ull * 4096, 1});
  cfgs.push_back({8192, 4, 6, 1, 3072ull * 4096, 1});
  cfgs.push_back({8192, 4, 3, 1, 3072ull * 1024, 1});
  for (auto c : cfgs) {
    const uint32_t smem = c.copy * c.per_stage * c.stages;
    if (smem > 200 * 1024 || (c.ctas_per_sm == 2 && smem > 100 * 1024)) continue;
    P p{d, bytes, c.copy, c.stages, c.per_stage, ctr, c.item, sink, c.planes};
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaMemset(ctr, 0, 4);
      cudaEventRecord(a);
      k_stream<<<sms * c.ctas_per_sm, 64, smem>>>(p);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    cudaError_t e = cudaGetLastError();
    printf("planes=%d copy=%6u x%u stages=%u ctas/sm=%u item=%lluKB inflight/SM=%3u KB : %.1f GB/s %s\n", c.planes, c.copy, c.per_stage, c.stages,
           c.ctas_per_sm, (unsigned long long)(c.item >> 10), smem * c.ctas_per_sm / 1024,
           (bytes / 1e9) / (best / 1e3), e == cudaSuccess ? "" : cudaGetErrorString(e));
  }
  for (int mult : {2, 4, 8}) {
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(a);
      k_ldg<<<sms * mult, 512>>>(reinterpret_cast<const float4*>(d), bytes / 16, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    printf("ldg.v4 grid=%d x 512 : %.1f GB/s\n", sms * mult, (bytes / 1e9) / (best / 1e3));
  }
  return 0;
}
