// TMA bulk-copy streaming microbenchmark: many small copies vs one big copy per tile.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ unsigned su(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mb_init(unsigned long long* b, int c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su(b)), "r"(c)); }
__device__ __forceinline__ void mb_expect(unsigned long long* b, unsigned n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mb_arrive(unsigned long long* b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su(b)) : "memory"); }
__device__ __forceinline__ void mb_wait(unsigned long long* b, unsigned p) {
  asm volatile("{\n.reg .pred q;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 q, [%0], %1;\n@!q bra W_%=;\n}\n" ::"r"(su(b)), "r"(p) : "memory"); }
__device__ __forceinline__ void bulk(void* d, const void* s, unsigned n, unsigned long long* b) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su(d)), "l"(s), "r"(n), "r"(su(b)) : "memory"); }
// tile = TE doubles x K columns; layout 0: columns far apart (stride n), 1: tile-interleaved (contiguous)
template <int TE>
__global__ void __launch_bounds__(160, 1) stream(const double* base, long long n, int K, int layout, int nstage, double* out) {
  extern __shared__ __align__(128) unsigned char sm[];
  double* st0 = (double*)sm;
  unsigned long long* full = (unsigned long long*)(st0 + (size_t)nstage * K * TE);
  unsigned long long* empty = full + nstage;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) { for (int s = 0; s < nstage; ++s) { mb_init(&full[s], 1); mb_init(&empty[s], 4); } asm volatile("fence.mbarrier_init.release.cluster;"); }
  __syncthreads();
  const long long ntiles = n / TE;
  if (warp == 4) {
    int it = 0;
    for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int st = it % nstage;
      if (it >= nstage) mb_wait(&empty[st], ((it / nstage) - 1) & 1);
      double* dst = st0 + (size_t)st * K * TE;
      if (layout == 1) {
        if (lane == 0) { mb_expect(&full[st], K * TE * 8); bulk(dst, base + t * K * TE, K * TE * 8, &full[st]); }
      } else {
        if (lane == 0) mb_expect(&full[st], K * TE * 8);
        __syncwarp();
        for (int k = lane; k < K; k += 32) bulk(dst + k * TE, base + k * n + t * TE, TE * 8, &full[st]);
      }
    }
    return;
  }
  double acc = 0;
  int it = 0;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int st = it % nstage;
    mb_wait(&full[st], (it / nstage) & 1);
    const double* T = st0 + (size_t)st * K * TE;
    for (int k = 0; k < K; ++k) acc += T[k * TE + threadIdx.x % TE];
    __syncwarp();
    if (lane == 0) mb_arrive(&empty[st]);
  }
  if (acc == 12345.0) out[0] = acc;
}
int main() {
  const long long n = 16777216; const int K = 66;
  double* buf; cudaMalloc(&buf, (size_t)K * n * 8); cudaMemset(buf, 0, (size_t)K * n * 8);
  double* out; cudaMalloc(&out, 8);
  int nsm; cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  for (int layout = 0; layout < 2; ++layout)
    for (int ns = 2; ns <= 3; ++ns) {
      const size_t smem = (size_t)ns * K * 128 * 8 + 64;
      cudaFuncSetAttribute(stream<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      float best = 1e9;
      for (int r = 0; r < 4; ++r) {
        cudaEventRecord(a);
        stream<128><<<nsm, 160, smem>>>(buf, n, K, layout, ns, out);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b); if (ms < best) best = ms;
      }
      printf("layout %d (%s) stages %d: %.3f ms %.1f GB/s err=%s\n", layout, layout ? "1 copy of 66KB/tile" : "66 copies of 1KB/tile", ns, best,
             (double)K * n * 8 / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
