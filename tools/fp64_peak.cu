// FP64 peak microbenchmarks for the roofline denominators (DMMA.8x8x4 and DFMA issue rate).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters) {
  double acc[CHAINS][2];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-9;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) { acc[c][0] = 0; acc[c][1] = 0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[c][0]), "+d"(acc[c][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c][0] + acc[c][1];
  if (s == 12345.0) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters) {
  double acc[CHAINS];
  double a = 1.0 + threadIdx.x * 1e-9, b = 1.0 - threadIdx.x * 1e-12;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) acc[c] = c;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += acc[c];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int iters = 20000;
  for (int threads : {128, 256, 512}) {
    for (int bps : {1, 2, 4}) {
      int grid = sms * bps;
      dmma_loop<8><<<grid, threads>>>(out, 100);
      cudaEventRecord(e0);
      dmma_loop<8><<<grid, threads>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      float ms; cudaEventElapsedTime(&ms, e0, e1);
      double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (threads / 32) * (double)grid;
      printf("{\"kind\":\"dmma\",\"threads\":%d,\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", threads, bps, flops / ms / 1e9);
      dfma_loop<8><<<grid, threads>>>(out, 100);
      cudaEventRecord(e0);
      dfma_loop<8><<<grid, threads>>>(out, iters);
      cudaEventRecord(e1); cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      flops = 2.0 * 8.0 * iters * threads * (double)grid;
      printf("{\"kind\":\"dfma\",\"threads\":%d,\"blocks_per_sm\":%d,\"tflops\":%.3f}\n", threads, bps, flops / ms / 1e9);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
