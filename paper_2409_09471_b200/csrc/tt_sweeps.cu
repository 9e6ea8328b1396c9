// Left-to-right interface sweeps built on the grouped DMMA GEMM:
//   * tt_dot (reference tt.py:285-294), batched over several partners
//   * stream_sketch partial contractions (reference streaming.py:117-142)
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

// ---------------------------------------------------------------------------
// stream_sketch (reference streaming.py:117-142).  Left partial contractions
// L_{k+1} = Y_k^T (L_k x_1 C_k) and right partial contractions
// R_k = (C_k x_3 R_{k+1}) X_k^T run as two independent chains; step j of the
// left chain and step j of the right chain share one grouped GEMM launch.
// Then every Psi_mu = (L_mu C_mu) R_{mu+1} and Omega_mu = L_mu R_mu is formed
// with grouped launches.
extern "C" {

size_t ttk_stream_sketch_ws_bytes(int d, const int* dims, const int* tr, const int* lr, const int* rr) {
  size_t tot = 0;
  for (int k = 0; k <= d; ++k) {
    tot += align_up((size_t)lr[k] * tr[k] * 8, 256);  // L_k (l_k x t_k)
    tot += align_up((size_t)tr[k] * rr[k] * 8, 256);  // R_k (t_k x r_k)
  }
  size_t tmax = 0;
  for (int k = 0; k < d; ++k) {
    tmax = std::max(tmax, (size_t)lr[k] * dims[k] * tr[k + 1]);
    tmax = std::max(tmax, (size_t)tr[k] * dims[k] * rr[k + 1]);
  }
  // two chain temporaries + d psi temporaries
  size_t tsum = 0;
  for (int k = 0; k < d; ++k) tsum += align_up((size_t)lr[k] * dims[k] * tr[k + 1] * 8, 256);
  return tot + 2 * align_up(tmax * 8, 256) + tsum + (16u << 20) + 65536;
}

// psi[mu]: (lr[mu]*dims[mu]) x rr[mu+1]; omega[mu-1]: lr[mu] x rr[mu] for mu=1..d-1.
// tr: ranks of the sketched TT (d+1); lr / rr: ranks of the left (Y) and right (X) DRMs.
int ttk_stream_sketch(int d, const int* dims, const int* tr, const double* const* C, const int* lr,
                      const double* const* Y, const int* rr, const double* const* X,
                      double* const* psi, double* const* omega, void* ws, size_t ws_bytes,
                      void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  TTK_REQUIRE(d >= 1, kInvalidValue, "stream_sketch: d must be >= 1");
  const size_t need = ttk_stream_sketch_ws_bytes(d, dims, tr, lr, rr);
  TTK_REQUIRE(ws != nullptr && ws_bytes >= need, kWorkspace, "stream_sketch: workspace %zu < %zu",
              ws_bytes, need);
  Arena ar(ws, ws_bytes);
  std::vector<double*> L(d + 1), R(d + 1);
  for (int k = 0; k <= d; ++k) {
    L[k] = ar.take<double>((size_t)lr[k] * tr[k]);
    R[k] = ar.take<double>((size_t)tr[k] * rr[k]);
  }
  size_t tmax = 0;
  for (int k = 0; k < d; ++k) {
    tmax = std::max(tmax, (size_t)lr[k] * dims[k] * tr[k + 1]);
    tmax = std::max(tmax, (size_t)tr[k] * dims[k] * rr[k + 1]);
  }
  double* TL = ar.take<double>(tmax);
  double* TR = ar.take<double>(tmax);
  std::vector<double*> TP(d);
  for (int k = 0; k < d; ++k) TP[k] = ar.take<double>((size_t)lr[k] * dims[k] * tr[k + 1]);
  void* split_ws = ar.take<char>(16u << 20);
  TTK_REQUIRE(split_ws != nullptr, kWorkspace, "stream_sketch: workspace too small");
  const double one = 1.0;
  TTK_CHECK_CUDA(cudaMemcpyAsync(L[0], &one, sizeof(double), cudaMemcpyHostToDevice, st));
  TTK_CHECK_CUDA(cudaMemcpyAsync(R[d], &one, sizeof(double), cudaMemcpyHostToDevice, st));
  // chains: step s of the left chain computes L_{s+1}; of the right chain R_{d-1-s}
  for (int s = 0; s < d - 1; ++s) {
    GemmProblem pr[2];
    int np = 0;
    {  // left: T = L_k (l x t) C_k (t x n t')  -> (l, n, t')
      const int k = s, l = lr[k], t = tr[k], n = dims[k], t1 = tr[k + 1];
      pr[np++] = make_gemm(l, n * t1, t, L[k], t, 1, C[k], (long long)n * t1, 1, TL, (long long)n * t1, 1);
    }
    {  // right: T = C_k (t n x t') R_{k+1} (t' x r')  -> (t, n, r')
      const int k = d - 1 - s, t = tr[k], n = dims[k], t1 = tr[k + 1], r1 = rr[k + 1];
      pr[np++] = make_gemm(t * n, r1, t1, C[k], t1, 1, R[k + 1], r1, 1, TR, r1, 1);
    }
    TTK_TRY(gemm_group_launch(pr, np, split_ws, 16u << 20, st));
    np = 0;
    {  // L_{k+1} (l' x t') = Y_k^T (l' x l n) T (l n x t')
      const int k = s, l = lr[k], n = dims[k], t1 = tr[k + 1], l1 = lr[k + 1];
      pr[np++] = make_gemm(l1, t1, l * n, Y[k], 1, l1, TL, t1, 1, L[k + 1], t1, 1);
    }
    {  // R_k (t x r) = T (t x n r') X_k^T (n r' x r)
      const int k = d - 1 - s, t = tr[k], n = dims[k], r1 = rr[k + 1], r = rr[k];
      const long long K = (long long)n * r1;
      pr[np++] = make_gemm(t, r, (int)K, TR, K, 1, X[k], 1, K, R[k], r, 1);
    }
    TTK_TRY(gemm_group_launch(pr, np, split_ws, 16u << 20, st));
  }
  // Psi_mu = (L_mu C_mu) R_{mu+1}: two grouped launches over mu
  std::vector<GemmProblem> pp(d);
  for (int mu = 0; mu < d; ++mu) {
    const int l = lr[mu], t = tr[mu], n = dims[mu], t1 = tr[mu + 1];
    pp[mu] = make_gemm(l, n * t1, t, L[mu], t, 1, C[mu], (long long)n * t1, 1, TP[mu], (long long)n * t1, 1);
  }
  TTK_TRY(gemm_group_launch(pp.data(), d, split_ws, 16u << 20, st));
  for (int mu = 0; mu < d; ++mu) {
    const int l = lr[mu], n = dims[mu], t1 = tr[mu + 1], r1 = rr[mu + 1];
    pp[mu] = make_gemm(l * n, r1, t1, TP[mu], t1, 1, R[mu + 1], r1, 1, psi[mu], r1, 1);
  }
  TTK_TRY(gemm_group_launch(pp.data(), d, split_ws, 16u << 20, st));
  if (d > 1) {
    std::vector<GemmProblem> po(d - 1);
    for (int mu = 1; mu < d; ++mu)
      po[mu - 1] = make_gemm(lr[mu], rr[mu], tr[mu], L[mu], tr[mu], 1, R[mu], rr[mu], 1, omega[mu - 1],
                             rr[mu], 1);
    TTK_TRY(gemm_group_launch(po.data(), d - 1, split_ws, 16u << 20, st));
  }
  return kOk;
}

}  // extern "C"
