// Accuracy of the fp64 hardware reciprocal-square-root seed (rsqrt.approx.ftz.f64)
// over the rotation formula's argument range: decides how many Newton steps the
// Jacobi rotation needs.  nvcc -gencode arch=compute_100a,code=sm_100a -o tools/rsqrt_acc tools/rsqrt_acc.cu
#include <cstdio>
#include <cmath>
__global__ void k(double* err, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // p spans 1e-30 .. 16 log-uniformly plus mantissa jitter
  double p = exp(-69.0 + 71.8 * (i / (double)n)) * (1.0 + 0.37 * ((i * 2654435761u) % 1000) / 1000.0);
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(p));
  double ex = 1.0 / sqrt(p);
  err[i] = fabs(y - ex) / ex;
}
int main() {
  const int n = 1 << 22;
  double* d; cudaMalloc(&d, n * 8);
  k<<<n / 256, 256>>>(d, n);
  double* h = new double[n];
  cudaMemcpy(h, d, n * 8, cudaMemcpyDeviceToHost);
  double mx = 0; for (int i = 0; i < n; ++i) mx = fmax(mx, h[i]);
  printf("rsqrt.approx.ftz.f64 max rel error %.3e = 2^%.2f\n", mx, log2(mx));
  return 0;
}
