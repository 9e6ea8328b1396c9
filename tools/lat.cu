// fp64 dependent-chain latencies on the B200 (cycles per op)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_dfma(double* o, long long* t, double x) {
  double a = x; long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 1024; ++i) a = fma(a, 1.0000001, 1e-9);
  long long t1 = clock64(); o[threadIdx.x] = a; t[0] = (t1 - t0);
}
__global__ void k_ddiv(double* o, long long* t, double x) {
  double a = x; long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 256; ++i) a = 1.0001 / (a + 1.0);
  long long t1 = clock64(); o[threadIdx.x] = a; t[0] = (t1 - t0);
}
__global__ void k_dsqrt(double* o, long long* t, double x) {
  double a = x; long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 256; ++i) a = sqrt(a + 1.0);
  long long t1 = clock64(); o[threadIdx.x] = a; t[0] = (t1 - t0);
}
__global__ void k_drsqrt(double* o, long long* t, double x) {
  double a = x; long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 256; ++i) a = rsqrt(a + 1.0);
  long long t1 = clock64(); o[threadIdx.x] = a; t[0] = (t1 - t0);
}
__global__ void k_shfl(double* o, long long* t, double x) {
  double a = x + threadIdx.x; long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 256; ++i) a += __shfl_xor_sync(0xffffffff, a, 1);
  long long t1 = clock64(); o[threadIdx.x] = a; t[0] = (t1 - t0);
}
__global__ void k_lds(double* o, long long* t, double x) {
  __shared__ double s[64];
  s[threadIdx.x] = x; __syncthreads();
  double a = x; long long t0 = clock64(); int j = threadIdx.x;
  #pragma unroll 1
  for (int i = 0; i < 256; ++i) { a += s[j]; j = (j + (int)(a == 12345.0)) & 31; }
  long long t1 = clock64(); o[threadIdx.x] = a; t[0] = (t1 - t0);
}
__global__ void k_bar(double* o, long long* t, double x) {
  double a = x; long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 256; ++i) { a += 1.0; __syncthreads(); }
  long long t1 = clock64(); o[threadIdx.x] = a; if (threadIdx.x == 0) t[0] = (t1 - t0);
}
__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1]) : "d"(a), "d"(b));
}
// dependent DMMA chain (same accumulator) and four independent accumulators per step
__global__ void k_dmma(double* o, long long* t, double x) {
  double c[2] = {x, x}; long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 256; ++i) dmma(c, 1.0000001, 1e-3);
  long long t1 = clock64(); o[threadIdx.x] = c[0] + c[1]; t[0] = (t1 - t0);
}
__global__ void k_dmma4(double* o, long long* t, double x) {
  double c0[2] = {x, x}, c1[2] = {x, x}, c2[2] = {x, x}, c3[2] = {x, x}; long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 256; ++i) { dmma(c0, 1.0000001, 1e-3); dmma(c1, 1.0000001, 1e-3); dmma(c2, 1.0000001, 1e-3); dmma(c3, 1.0000001, 1e-3); }
  long long t1 = clock64(); o[threadIdx.x] = c0[0] + c1[1] + c2[0] + c3[1]; t[0] = (t1 - t0);
}
// DMMA whose result feeds a dependent DFMA that feeds the next DMMA's operand
__global__ void k_dmma_dep_op(double* o, long long* t, double x) {
  double a = x; long long t0 = clock64();
  #pragma unroll 1
  for (int i = 0; i < 256; ++i) { double c[2] = {0.0, 0.0}; dmma(c, a, 1e-3); a = c[0] + 1.0; }
  long long t1 = clock64(); o[threadIdx.x] = a; t[0] = (t1 - t0);
}
int main() {
  double* o; long long* t; cudaMalloc(&o, 8192); cudaMalloc(&t, 8);
  long long h;
  k_dfma<<<1, 32>>>(o, t, 1.0); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("dfma %.1f\n", h / 1024.0);
  k_ddiv<<<1, 32>>>(o, t, 1.0); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("ddiv %.1f\n", h / 256.0);
  k_dsqrt<<<1, 32>>>(o, t, 1.0); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("dsqrt %.1f\n", h / 256.0);
  k_drsqrt<<<1, 32>>>(o, t, 1.0); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("drsqrt %.1f\n", h / 256.0);
  k_shfl<<<1, 32>>>(o, t, 1.0); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("shfl+dadd %.1f\n", h / 256.0);
  k_lds<<<1, 32>>>(o, t, 1.0); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("lds+dadd %.1f\n", h / 256.0);
  k_bar<<<1, 512>>>(o, t, 1.0); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("bar512+dadd %.1f\n", h / 256.0);
  k_bar<<<1, 1024>>>(o, t, 1.0); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("bar1024+dadd %.1f\n", h / 256.0);
  k_dmma<<<1, 32>>>(o, t, 1.0); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("dmma dependent accumulator %.1f\n", h / 256.0);
  k_dmma4<<<1, 32>>>(o, t, 1.0); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("4 independent dmma per step %.1f\n", h / 256.0);
  k_dmma_dep_op<<<1, 32>>>(o, t, 1.0); cudaMemcpy(&h, t, 8, cudaMemcpyDeviceToHost); printf("dmma -> dadd -> dmma operand %.1f\n", h / 256.0);
  return 0;
}
