// FP64 tensor-core (DMMA) peak on this GPU: back-to-back mma.sync.m8n8k4.f64 with independent
// accumulators in registers (no memory traffic).  Flops per mma = 2 * 8 * 8 * 4 = 512.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dmma_peak tools/dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int ACC>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed - threadIdx.x * 1e-3;
  double c0[ACC], c1[ACC];
#pragma unroll
  for (int k = 0; k < ACC; ++k) c0[k] = c1[k] = 0.0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int k = 0; k < ACC; ++k)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c0[k]), "+d"(c1[k]) : "d"(a), "d"(b));
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < ACC; ++k) s += c0[k] + c1[k];
  if (s == 12345.678) out[0] = s;
}

// FFMA f64 peak (non-tensor pipe) for comparison: 2 flops per fma
template <int ACC>
__global__ void ffma_loop(double* out, int iters, double seed) {
  double x[ACC];
  const double m = 1.0 + 1e-9 * threadIdx.x, ad = seed;
#pragma unroll
  for (int k = 0; k < ACC; ++k) x[k] = k;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int k = 0; k < ACC; ++k) x[k] = fma(x[k], m, ad);
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < ACC; ++k) s += x[k];
  if (s == 12345.678) out[0] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int nsm = p.multiProcessorCount;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"results\": [\n", p.name, nsm);
  bool first = true;
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) dmma_loop<8><<<nsm, 32 * warps>>>(out, iters, 1.0);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      dmma_loop<8><<<nsm, 32 * warps>>>(out, iters, 1.0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double fl = 512.0 * 8 * iters * (double)warps * nsm;
    printf("%s {\"kind\": \"dmma_m8n8k4\", \"warps_per_sm\": %d, \"tflops\": %.3f}", first ? "" : ",\n", warps,
           fl / (best * 1e-3) / 1e12);
    first = false;
  }
  for (int warps : {8, 16, 32}) {
    const int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) ffma_loop<16><<<nsm, 32 * warps>>>(out, iters, 1.0);
    float best = 1e30f;
    for (int rep = 0; rep < 5; ++rep) {
      cudaEventRecord(e0);
      ffma_loop<16><<<nsm, 32 * warps>>>(out, iters, 1.0);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    const double fl = 2.0 * 16 * iters * 32.0 * warps * nsm;
    printf(",\n {\"kind\": \"ffma_f64\", \"warps_per_sm\": %d, \"tflops\": %.3f}", warps, fl / (best * 1e-3) / 1e12);
  }
  printf("\n]}\n");
  return 0;
}
