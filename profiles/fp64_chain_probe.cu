// fp64 exact-chain latency probe: cycles per sequential step for one thread
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double step(double acc, float a, float b) {
  const double d = __dsub_rn((double)a, (double)b);
  return __dadd_rn(acc, __dmul_rn(d, d));
}
__global__ void k(const float* q, const float* x, int dim, double* out, long long* cyc, int mode) {
  __shared__ float qs[1024], xs[1024 * 8];
  __shared__ double qd[1024];
  for (int i = threadIdx.x; i < dim; i += blockDim.x) { qs[i] = q[i]; qd[i] = q[i]; }
  for (int i = threadIdx.x; i < dim * 8; i += blockDim.x) xs[i] = x[i];
  __syncthreads();
  const float* row = xs + (threadIdx.x & 7) * dim;
  long long t0 = clock64();
  double acc = 0.0;
  if (mode == 0) {
    for (int d = 0; d < dim; ++d) acc = step(acc, qs[d], row[d]);
  } else if (mode == 1) {
#pragma unroll 8
    for (int d = 0; d < dim; ++d) acc = step(acc, qs[d], row[d]);
  } else {
#pragma unroll 8
    for (int d = 0; d < dim; ++d) { const double t = __dsub_rn(qd[d], (double)row[d]); acc = __dadd_rn(acc, __dmul_rn(t, t)); }
  }
  long long t1 = clock64();
  out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  const int dim = 768;
  float *q, *x; double* out; long long* cyc;
  cudaMalloc(&q, 4 * 1024); cudaMalloc(&x, 4 * 8192); cudaMalloc(&out, 8 * 1 << 20); cudaMalloc(&cyc, 8 * 4096);
  cudaMemset(q, 0, 4096); cudaMemset(x, 0, 32768);
  for (int mode = 0; mode < 3; ++mode)
    for (int threads : {1, 32, 256}) for (int blocks : {1, 148, 592}) {
      k<<<blocks, threads>>>(q, x, dim, out, cyc, mode);
      k<<<blocks, threads>>>(q, x, dim, out, cyc, mode);
      long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
      printf("mode %d threads %3d blocks %3d: %.1f cycles/step\n", mode, threads, blocks, (double)h / dim);
    }
  return 0;
}
