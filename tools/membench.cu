// Streaming-read microbenchmark: achievable HBM bandwidth when reading K columns at once
// (the fill pass's access pattern).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 membench.cu
#include <cstdio>
#include <cuda_runtime.h>
template <int K>
__global__ void sumk(const double* __restrict__ base, long long stride, long long n, double* __restrict__ out) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    double v[K];
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = __ldg(base + k * stride + e);
    double s = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) s += v[k];
    out[e] = s;
  }
}
template <int K>
__global__ void sumk_chunk(const double* __restrict__ base, long long stride, long long n, double* __restrict__ out) {
  // each warp streams a contiguous chunk of 32*8 elements per column (like a tile)
  const long long nchunk = n / 256;
  const int lane = threadIdx.x & 31;
  for (long long c = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32; c < nchunk; c += (long long)gridDim.x * blockDim.x / 32) {
    for (int j = 0; j < 8; ++j) {
      const long long e = c * 256 + j * 32 + lane;
      double v[K];
#pragma unroll
      for (int k = 0; k < K; ++k) v[k] = __ldg(base + k * stride + e);
      double s = 0;
#pragma unroll
      for (int k = 0; k < K; ++k) s += v[k];
      out[e] = s;
    }
  }
}
int main() {
  const long long n = 16777216;  // config-4 DOFs
  const int K = 66;
  double *ring, *out;
  cudaMalloc(&ring, (size_t)K * n * 8);
  cudaMalloc(&out, n * 8);
  cudaMemset(ring, 0, (size_t)K * n * 8);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  for (int cfg = 0; cfg < 6; ++cfg) {
    int threads = 256, blocks;
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(a);
      if (cfg == 0) { blocks = nsm * 4; sumk<1><<<blocks, threads>>>(ring, n, n, out); }
      if (cfg == 1) { blocks = nsm * 4; sumk<K><<<blocks, threads>>>(ring, n, n, out); }
      if (cfg == 2) { blocks = nsm * 2; sumk<K><<<blocks, threads>>>(ring, n, n, out); }
      if (cfg == 3) { threads = 128; blocks = nsm * 4; sumk<K><<<blocks, threads>>>(ring, n, n, out); }
      if (cfg == 4) { blocks = nsm * 4; sumk<16><<<blocks, threads>>>(ring, n, n, out); }
      if (cfg == 5) { blocks = nsm * 4; sumk_chunk<K><<<blocks, threads>>>(ring, n, n, out); }
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    const int kk = (cfg == 0) ? 1 : (cfg == 4 ? 16 : K);
    const double bytes = (double)(kk + 1) * n * 8;
    printf("cfg %d K=%d: %.3f ms  %.1f GB/s  err=%s\n", cfg, kk, best, bytes / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
