// Left-to-right interface sweeps built on the grouped DMMA GEMM:
//   * tt_dot (reference tt.py:285-294), batched over several partners
//   * stream_sketch partial contractions (reference streaming.py:214-239)
#include "gemm.cuh"
#include "../../include/ttk_b200.h"

#include <algorithm>
#include <vector>

using namespace ttk;

namespace {

// per-core contraction step of the dot sweep; m: (ra x rb) row-major
//   T[rb, i, ra'] = sum_ra m[ra, rb] X_k[ra, i, ra']          (M=rb, K=ra, N=n ra')
//   m'[ra', rb']  = sum_{rb,i} T[rb, i, ra'] Y_k[rb, i, rb']  (M=ra', K=rb n, N=rb')
GemmProblem dot_step1(const double* m, int ra, int rb, const double* X, int n, int ra1, double* T) {
  GemmProblem p = make_gemm(rb, n * ra1, ra, m, /*a_ms=*/1, /*a_ks=*/rb, X, /*b_ks=*/(long long)n * ra1,
                            /*b_ns=*/1, T, (long long)n * ra1, 1);
  return p;
}
GemmProblem dot_step2(const double* T, int rb, int n, int ra1, const double* Y, int rb1, double* m1) {
  GemmProblem p = make_gemm(ra1, rb1, rb * n, T, /*a_ms=*/1, /*a_ks=*/ra1, Y, /*b_ks=*/rb1,
                            /*b_ns=*/1, m1, rb1, 1);
  return p;
}

}  // namespace

extern "C" {

size_t ttk_tt_dots_ws_bytes(int d, const int* dims, const int* xr, int p, const int* yr) {
  size_t tmax = 0, mmax = 1;
  for (int i = 0; i < p; ++i)
    for (int k = 0; k < d; ++k) {
      tmax = std::max(tmax, (size_t)yr[i * (d + 1) + k] * dims[k] * xr[k + 1]);
      mmax = std::max(mmax, (size_t)xr[k + 1] * yr[i * (d + 1) + k + 1]);
    }
  // per partner: T + 2 m buffers; plus split-K partials (bounded by the GEMM planner)
  size_t per = align_up(tmax * 8, 256) + 2 * align_up(mmax * 8, 256) + 256;
  return per * p + (size_t)64 * tmax * 8 + (size_t)64 * mmax * 8 + 4096;
}

// out_dev[i] = <x, y_i> for i < p (device doubles).  Reference tt_dot, tt.py:285-294.
int ttk_tt_dots(int d, const int* dims, const int* xr, const double* const* x, int p,
                const int* yr, const double* const* y, double* out_dev, void* ws, size_t ws_bytes,
                void* stream) {
  TTK_REQUIRE(d >= 1 && p >= 0, kInvalidValue, "tt_dots: bad sizes");
  if (p == 0) return kOk;
  cudaStream_t st = (cudaStream_t)stream;
  size_t tmax = 0, mmax = 1;
  for (int i = 0; i < p; ++i) {
    TTK_REQUIRE(yr[i * (d + 1)] == 1 && yr[i * (d + 1) + d] == 1, kShapeMismatch,
                "tt_dots: boundary ranks must equal 1");
    for (int k = 0; k < d; ++k) {
      tmax = std::max(tmax, (size_t)yr[i * (d + 1) + k] * dims[k] * xr[k + 1]);
      mmax = std::max(mmax, (size_t)xr[k + 1] * yr[i * (d + 1) + k + 1]);
    }
  }
  Arena ar(ws, ws_bytes);
  std::vector<double*> T(p), m0(p), m1(p);
  for (int i = 0; i < p; ++i) {
    T[i] = ar.take<double>(tmax);
    m0[i] = ar.take<double>(mmax);
    m1[i] = ar.take<double>(mmax);
  }
  size_t rest_off = align_up(ar.used, 256);
  TTK_REQUIRE(ar.used <= ws_bytes && ws != nullptr, kWorkspace, "tt_dots: workspace too small");
  void* split_ws = (char*)ws + rest_off;
  size_t split_bytes = ws_bytes > rest_off ? ws_bytes - rest_off : 0;
  // initial m = [[1]]: run core 0 with "m" = identity-of-size-1, i.e. T = X_0 directly
  std::vector<GemmProblem> probs(p);
  for (int k = 0; k < d; ++k) {
    const int n = dims[k], ra = xr[k], ra1 = xr[k + 1];
    // step 1 (skipped at k == 0: m = [[1]] so T = X_0 viewed as (1 x n ra1))
    if (k > 0) {
      for (int i = 0; i < p; ++i) {
        const int rb = yr[i * (d + 1) + k];
        probs[i] = dot_step1(m0[i], ra, rb, x[k], n, ra1, T[i]);
      }
      TTK_TRY(gemm_group_launch(probs.data(), p, split_ws, split_bytes, st));
    }
    for (int i = 0; i < p; ++i) {
      const int rb = yr[i * (d + 1) + k], rb1 = yr[i * (d + 1) + k + 1];
      const double* Tin = (k == 0) ? x[0] : T[i];
      double* dst = (k == d - 1) ? out_dev + i : m0[i];
      probs[i] = dot_step2(Tin, rb, n, ra1, y[(size_t)i * d + k], rb1, (k == d - 1) ? dst : m1[i]);
    }
    TTK_TRY(gemm_group_launch(probs.data(), p, split_ws, split_bytes, st));
    if (k < d - 1)
      for (int i = 0; i < p; ++i) std::swap(m0[i], m1[i]);
  }
  return kOk;
}

}  // extern "C"
