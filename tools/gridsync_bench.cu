// Micro-benchmark: cost of a grid-wide barrier in a cooperative kernel (cg::grid.sync vs a
// sense-reversing counter barrier with acquire/release).  nvcc -arch=sm_100a -O3 gridsync_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, double* sink) {
  cg::grid_group g = cg::this_grid();
  double x = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    x = x * 1.0000001 + 1.0;
    g.sync();
  }
  if (x == -1.0) *sink = x;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void gbar(unsigned* count, unsigned* gen, unsigned nblk) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned g0 = ld_acquire(gen);
    unsigned prev;
    asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], 1;" : "=r"(prev) : "l"(count) : "memory");
    if (prev == nblk - 1) {
      *count = 0;
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g0 + 1) : "memory");
    } else {
      while (ld_acquire(gen) == g0) {
      }
    }
  }
  __syncthreads();
}

__global__ void k_own(int iters, double* sink, unsigned* bar) {
  double x = threadIdx.x;
  for (int i = 0; i < iters; ++i) {
    x = x * 1.0000001 + 1.0;
    gbar(bar, bar + 32, gridDim.x);
  }
  if (x == -1.0) *sink = x;
}

int main() {
  int nsm;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  double* sink;
  unsigned* bar;
  cudaMalloc(&sink, 8);
  cudaMalloc(&bar, 256);
  cudaMemset(bar, 0, 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 2000;
  int threads_list[] = {128, 256, 512, 1024};
  for (int bpsm = 1; bpsm <= 2; ++bpsm)
    for (int t : threads_list) {
      if (bpsm * t > 1024) continue;
      const int grid = nsm * bpsm;
      int it = iters;
      void* args[] = {&it, &sink};
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)k_cg, grid, t, args, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      void* args2[] = {&it, &sink, &bar};
      float ms2 = 0;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        cudaLaunchCooperativeKernel((void*)k_own, grid, t, args2, 0, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
      }
      cudaEventElapsedTime(&ms2, e0, e1);
      printf("grid %4d x %4d: cg %.2f us/sync   own %.2f us/sync  (%s)\n", grid, t, 1000.0 * ms / iters,
             1000.0 * ms2 / iters, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
