// Counter-based Gaussian TT-DRM on the device (the solver's randomized-rounding
// sketch; the reference has no RTO).
//
// Entry (i, j, l) of core k is a pure function of (seed, k, i, j, l) in the
// FULL index space (r0_full x n x r1_full): Philox4x32-10 of the counter
// ((k * r0_full + i) * n + j) * r1_full + l under key = seed, two 53-bit
// uniforms, Box-Muller (cosine branch), times `scale`.  Any leading block
// (r0 <= r0_full, r1 <= r1_full) is therefore generated on demand and equals
// the same block of the full map -- the solver grows its sketch ranks by one
// per iteration without ever drawing the whole cap-sized DRM.
#include "common.cuh"
#include "../../include/ttk_b200.h"

#include <algorithm>
#include <cstdint>

namespace ttk {

__device__ __forceinline__ void philox_round(uint32_t& c0, uint32_t& c1, uint32_t& c2, uint32_t& c3, uint32_t k0,
                                             uint32_t k1) {
  const uint32_t M0 = 0xD2511F53u, M1 = 0xCD9E8D57u;
  const uint32_t hi0 = __umulhi(M0, c0), lo0 = M0 * c0;
  const uint32_t hi1 = __umulhi(M1, c2), lo1 = M1 * c2;
  const uint32_t n0 = hi1 ^ c1 ^ k0, n1 = lo1, n2 = hi0 ^ c3 ^ k1, n3 = lo0;
  c0 = n0; c1 = n1; c2 = n2; c3 = n3;
}

__device__ __forceinline__ void philox4x32_10(uint64_t ctr, uint64_t key, uint32_t (&out)[4]) {
  uint32_t c0 = (uint32_t)ctr, c1 = (uint32_t)(ctr >> 32), c2 = 0x9E3779B9u, c3 = 0x7F4A7C15u;
  uint32_t k0 = (uint32_t)key, k1 = (uint32_t)(key >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    philox_round(c0, c1, c2, c3, k0, k1);
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

__global__ void drm_gaussian_kernel(uint64_t seed, int core, int n, int r0_full, int r1_full, int r0, int r1,
                                    double scale, double* __restrict__ out) {
  const long long total = (long long)r0 * n * r1;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long i = e / ((long long)n * r1);
    const long long rem = e - i * n * r1;
    const long long j = rem / r1, l = rem - j * r1;
    const uint64_t ctr = ((((uint64_t)core * r0_full + i) * n + j) * r1_full + l);
    uint32_t x[4];
    philox4x32_10(ctr, seed, x);
    const uint64_t a = (((uint64_t)x[1] << 32) | x[0]) >> 11;
    const uint64_t b = (((uint64_t)x[3] << 32) | x[2]) >> 11;
    const double u1 = ((double)a + 0.5) * (1.0 / 9007199254740992.0);  // (0, 1)
    const double u2 = (double)b * (1.0 / 9007199254740992.0);          // [0, 1)
    out[e] = scale * sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
}

}  // namespace ttk

using namespace ttk;

extern "C" {

int ttk_drm_gaussian(unsigned long long seed, int core, int n, int r0_full, int r1_full, int r0, int r1,
                     double scale, double* out, void* stream) {
  TTK_REQUIRE(n > 0 && r0 > 0 && r1 > 0 && r0 <= r0_full && r1 <= r1_full && core >= 0, kInvalidValue,
              "drm_gaussian: bad block (%d x %d x %d of %d x %d x %d)", r0, n, r1, r0_full, n, r1_full);
  const long long total = (long long)r0 * n * r1;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 8LL * kNumSMs);
  drm_gaussian_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>((uint64_t)seed, core, n, r0_full, r1_full, r0, r1,
                                                                 scale, out);
  TTK_CHECK_LAUNCH();
  return kOk;
}

}  // extern "C"
