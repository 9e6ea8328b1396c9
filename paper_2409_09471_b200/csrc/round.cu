// TT rounding drivers (host-orchestrated sequences of device kernels):
//  * ttk_tt_round   -- TT-SVD (reference tt_round, tt.py:337-368): right-to-left
//                      Householder-QR orthogonalisation sweep, then left-to-right
//                      truncated SVDs (QR + Jacobi SVD of the small R factor).
//  * ttk_rto_sweeps -- randomize-then-orthogonalize (absent from the reference,
//                      SPEC.md:313; restated in oracle/ttoracle.py:rto_sweeps):
//                      right partial contractions with a Gaussian TT-DRM, then
//                      the left-to-right sketch / TSQR / project sweep.
#include "gemm.cuh"
#include "qr.cuh"
#include "../../include/ttk_b200.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <mutex>
#include <cmath>
#include <cstring>
#include <unordered_map>
#include <vector>

namespace ttk {

namespace {

constexpr size_t kSplitKBytes = 32u << 20;

#ifdef TTK_DEBUG_KNOBS
// diagnostics (TTK_TMA_VERIFY): every TMA GEMM is recomputed by the grouped kernel and compared on the device
__global__ void gemm_verify_kernel(int M, int N, int K, const double* __restrict__ C, long long c_ms, long long c_ns,
                                   const double* __restrict__ S, int* __restrict__ count) {
  double worst = 0.0;
  long long at = -1;
  const long long mn = (long long)M * N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < mn; e += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(e / N), n = (int)(e % N);
    const double d = fabs(C[m * c_ms + n * c_ns] - S[e]);
    if (d > worst || !(d == d)) { worst = d; at = e; }
  }
  if (worst > 1e-6 || !(worst == worst)) {
    if (atomicAdd(count, 1) < 4)
      printf("TMA GEMM mismatch M=%d N=%d K=%d at (%lld, %lld): |diff| %g (tma %g, grouped %g)\n", M, N, K, at / N,
             at % N, worst, C[(at / N) * c_ms + (at % N) * c_ns], S[at]);
  }
}
#endif

// The TMA-staged GEMM is used only while ONE problem owns the GPU.  With two
// independent problems in flight on different streams (bench.py's in-flight
// mode, concurrent solves) sweeps that route contractions through it were
// measured to return corrupted cores now and then (tools/inflight_repro.py:
// 4 of 12 two-thread runs, 0 of 12 with the grouped cp.async kernel; the TMA
// kernel alone passes every overlap test in tools/gemm_overlap.py,
// gemm_fresh.py, overlap_mix.py -- root cause not found, DESIGN 6.2).  So:
// ttk_gemm_tma_enable(0) turns it off, and a call that sees another caller
// stream active within the last half second takes the grouped kernel.
std::atomic<int> g_tma_enabled{1};
std::mutex g_tma_mu;
cudaStream_t g_tma_last_stream = nullptr;
long long g_tma_last_ns = 0, g_tma_conc_until_ns = 0;
constexpr long long kTmaQuietNs = 500000000LL;

// set while a sweep runs next to work of the same problem on other streams
// (the host pipeline's matvec chunks overlap the RTO right sweep)
thread_local int g_tma_suppress = 0;

bool tma_allowed(cudaStream_t st, bool internal_stream) {
  if (!g_tma_enabled.load(std::memory_order_relaxed) || g_tma_suppress > 0) return false;
  const long long now =
      std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now().time_since_epoch()).count();
  std::lock_guard<std::mutex> lock(g_tma_mu);
  if (!internal_stream) {
    if (g_tma_last_stream != st && g_tma_last_ns != 0 && now - g_tma_last_ns < kTmaQuietNs)
      g_tma_conc_until_ns = now + kTmaQuietNs;
    g_tma_last_stream = st;
    g_tma_last_ns = now;
  }
  return now >= g_tma_conc_until_ns;
}

int gemm1(int M, int N, int K, const double* A, long long a_ms, long long a_ks, const double* B,
          long long b_ks, long long b_ns, double* C, long long c_ms, long long c_ns, void* split_ws,
          cudaStream_t st, double alpha = 1.0, double beta = 0.0, bool internal_stream = false) {
  // row-major operands or their transposes (every contraction of the RTO sweeps
  // and of the truncation): the TMA-staged kernel, K split over split_ws when
  // the tiles leave SMs idle; anything else: the grouped cp.async kernel
  int status = kOk;
  static const int tma_off = knob_env("TTK_NO_TMA") ? atoi(knob_env("TTK_NO_TMA")) : 0;  // A/B: shape-class mask
  const bool no_tma = !tma_allowed(st, internal_stream) || (tma_off & 1) || ((tma_off & 2) && M > N) || ((tma_off & 4) && M <= N && N <= 12000) ||
                      ((tma_off & 8) && M <= N && N > 12000);
  if (!no_tma && gemm_tma_try(M, N, K, alpha, A, a_ms, a_ks, B, b_ks, b_ns, beta, C, c_ms, c_ns, split_ws,
                              split_ws ? kSplitKBytes : 0, st, &status)) {
#ifdef TTK_DEBUG_KNOBS
    static const bool verify = knob_env("TTK_TMA_VERIFY") != nullptr;
    if (verify && status == kOk && beta == 0.0) {
      double* S = nullptr;
      int* cnt = nullptr;
      TTK_TRY(scratch_alloc((void**)&S, sizeof(double) * (size_t)M * N + 256, st));
      cnt = reinterpret_cast<int*>(S + (size_t)M * N);
      TTK_CHECK_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int), st));
      GemmProblem q = make_gemm(M, N, K, A, a_ms, a_ks, B, b_ks, b_ns, S, N, 1, alpha, 0.0);
      TTK_TRY(gemm_group_launch(&q, 1, nullptr, 0, st));
      gemm_verify_kernel<<<148, 256, 0, st>>>(M, N, K, C, c_ms, c_ns, S, cnt);
      TTK_CHECK_LAUNCH();
      TTK_TRY(scratch_free(S, st));
    }
#endif
    return status;
  }
  GemmProblem p = make_gemm(M, N, K, A, a_ms, a_ks, B, b_ks, b_ns, C, c_ms, c_ns, alpha, beta);
  return gemm_group_launch(&p, 1, split_ws, split_ws ? kSplitKBytes : 0, st);
}

__global__ void sumsq_multi_kernel(const double* const* ptrs, const long long* sizes, double* out) {
  __shared__ double red[32];
  const double* x = ptrs[blockIdx.x];
  const long long n = sizes[blockIdx.x];
  double s = 0.0;
  for (long long e = threadIdx.x; e < n; e += blockDim.x) s += x[e] * x[e];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) out[blockIdx.x] = v;
  }
}

// T1[i][c] = L[i][c] / S[c]^2 (c < r): the right-factor map of the Gram truncation
__global__ void scale_cols_inv_sq_kernel(int rows, int r, const double* __restrict__ L, int ld,
                                         const double* __restrict__ S, double* __restrict__ T1) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < rows * r; e += gridDim.x * blockDim.x) {
    const int i = e / r, c = e - i * r;
    const double s = S[c];
    T1[i * ld + c] = L[i * ld + c] / (s * s);
  }
}

// certificate of one Gram-path core: Cholesky succeeded and the kept singular
// values stay >= sqrt(1e-3) of the largest (so the rank is min(cap, r0), as the
// reference's budget-0 rule gives, and the squared condition number costs <= ~1e3 eps)
__global__ void gram_cert_kernel(const double* __restrict__ S, int rk, const int* __restrict__ cstat,
                                 int* __restrict__ flag) {
  if (threadIdx.x == 0) {
    const double s0 = S[0], sr = S[rk - 1];
    *flag = (*cstat == 0 && s0 > 0.0 && sr * sr >= 1e-3 * s0 * s0) ? 1 : 0;
  }
}

struct PinnedScratch {
  void* p = nullptr;
  size_t cap = 0;
  void* get(size_t bytes) {
    if (bytes > cap) {
      if (p) cudaFreeHost(p);
      if (cudaMallocHost(&p, bytes) != cudaSuccess) { p = nullptr; cap = 0; return nullptr; }
      cap = bytes;
    }
    return p;
  }
};
thread_local PinnedScratch g_pinned;

// cores truncated by the Gram path / by the QR path (ttk_debug_truncate_paths)
std::atomic<long long> g_trunc_gram{0}, g_trunc_qr{0}, g_trunc_redo{0};
// cores factored by the gap-certified subspace kernel, and sweeps of it redone
// through the Jacobi Gram path after a failed certificate
std::atomic<long long> g_trunc_fast{0}, g_trunc_fast_redo{0};
// RTO left sweeps accepted with the deferred CholeskyQR2 check / redone with the per-core check
std::atomic<long long> g_rto_deferred{0}, g_rto_defer_redo{0};

// Shapes whose subspace sweep failed its certificate skip the subspace kernel
// for the next kFastSkip truncations of the same shape (a gap-free spectrum,
// e.g. config 2, would otherwise pay a wasted sweep on every call).
constexpr int kFastSkip = 16;
uint64_t trunc_shape_key(int d, const int* dims, const int* ranks, int max_rank) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](uint64_t v) { h = (h ^ v) * 1099511628211ull; };
  mix((uint64_t)d);
  mix((uint64_t)(uint32_t)max_rank);
  for (int k = 0; k < d; ++k) mix((uint64_t)dims[k]);
  for (int k = 0; k <= d; ++k) mix((uint64_t)ranks[k]);
  return h;
}
thread_local std::unordered_map<uint64_t, int> g_fast_skip;

size_t core_elems(const int* dims, const int* ranks, int k) {
  return (size_t)ranks[k] * dims[k] * ranks[k + 1];
}

}  // namespace

// --------------------------------------------------------------------------
// TT-SVD workspace plan
static size_t round_ws_bytes(int d, const int* dims, const int* ranks) {
  size_t sum = 0, mx = 0, qrws = 0;
  int rmax = 1;
  for (int k = 0; k < d; ++k) {
    size_t e = core_elems(dims, ranks, k);
    sum += align_up(e * 8, 256);
    mx = std::max(mx, e);
    rmax = std::max(rmax, std::max(ranks[k], ranks[k + 1]));
  }
  for (int k = 0; k < d; ++k) {
    int r0 = ranks[k], r1 = ranks[k + 1], n = dims[k];
    if (k > 0) qrws = std::max(qrws, qr_auto_ws_bytes(n * r1, r0));
    qrws = std::max(qrws, qr_auto_ws_bytes(r0 * n, r1));
  }
  size_t small = (size_t)rmax * rmax;
  return sum + 3 * align_up(mx * 8, 256) + 4 * align_up(small * 8, 256) + align_up(qrws, 256) +
         kSplitKBytes + (size_t)(d + 8) * 256 + 65536 + 4096;
}

}  // namespace ttk

using namespace ttk;

extern "C" {

size_t ttk_tt_round_ws_bytes(int d, const int* dims, const int* ranks) {
  return round_ws_bytes(d, dims, ranks);
}

// TT-SVD rounding.  out[k] must hold ranks[k]*dims[k]*ranks[k+1] doubles (the
// result never exceeds the input ranks); out_ranks (host, d+1) receives the
// result ranks; result core k occupies the first out_ranks[k]*dims[k]*out_ranks[k+1]
// entries of out[k], C-order.  max_rank <= 0: no cap.  zero_rel < 0 disables
// the reference's cancellation test (tt.py:348-356).  Synchronises `stream`.
int ttk_tt_round(int d, const int* dims, const int* ranks, const double* const* cores,
                 double rel_tol, int max_rank, double zero_rel, double* const* out, int* out_ranks,
                 void* ws, size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  TTK_REQUIRE(d >= 1, kInvalidValue, "tt_round: d must be >= 1");
  TTK_REQUIRE(rel_tol >= 0.0, kInvalidValue, "rel_tol must be nonnegative");
  for (int k = 0; k <= d; ++k) out_ranks[k] = ranks[k];
  if (d == 1) {
    TTK_CHECK_CUDA(cudaMemcpyAsync(out[0], cores[0], sizeof(double) * core_elems(dims, ranks, 0),
                                   cudaMemcpyDeviceToDevice, st));
    TTK_SYNC(st);
    return kOk;
  }
  const size_t need = round_ws_bytes(d, dims, ranks);
  TTK_REQUIRE(ws != nullptr && ws_bytes >= need, kWorkspace, "tt_round: workspace %zu < %zu", ws_bytes,
              need);
  Arena ar(ws, ws_bytes);
  size_t mx = 0;
  int rmax = 1;
  for (int k = 0; k < d; ++k) {
    mx = std::max(mx, core_elems(dims, ranks, k));
    rmax = std::max(rmax, std::max(ranks[k], ranks[k + 1]));
  }
  std::vector<double*> wk(d);
  for (int k = 0; k < d; ++k) wk[k] = ar.take<double>(core_elems(dims, ranks, k));
  double* alt[2] = {ar.take<double>(mx), ar.take<double>(mx)};
  double* tq = ar.take<double>(mx);
  double* tR = ar.take<double>((size_t)rmax * rmax);
  double* tU = ar.take<double>((size_t)rmax * rmax);
  double* tS = ar.take<double>((size_t)rmax + 8);
  double* tC = ar.take<double>((size_t)rmax * rmax);
  double* red = ar.take<double>((size_t)d + 8);
  double* part = ar.take<double>(256);
  int* rdev = ar.take<int>(8);
  const double** pdev = ar.take<const double*>((size_t)d);
  long long* sdev = ar.take<long long>((size_t)d);
  size_t qr_off = align_up(ar.used, 256);
  size_t qr_bytes = 0;
  for (int k = 0; k < d; ++k) {
    int r0 = ranks[k], r1 = ranks[k + 1], n = dims[k];
    if (k > 0) qr_bytes = std::max(qr_bytes, qr_auto_ws_bytes(n * r1, r0));
    qr_bytes = std::max(qr_bytes, qr_auto_ws_bytes(r0 * n, r1));
  }
  void* qws = (char*)ws + qr_off;
  ar.used = qr_off + qr_bytes;
  void* split_ws = ar.take<char>(kSplitKBytes);
  TTK_REQUIRE(split_ws != nullptr, kWorkspace, "tt_round: workspace too small");

  double* pin = (double*)g_pinned.get(sizeof(double) * (d + 8));
  TTK_REQUIRE(pin != nullptr, kCudaError, "tt_round: cannot allocate pinned scratch");

  // optional zero test: prod_k ||C_k||_F of the INPUT cores
  std::vector<int> r(ranks, ranks + d + 1);
  double prod_norm = 1.0;
  if (zero_rel >= 0.0) {
    std::vector<const double*> hp(cores, cores + d);
    std::vector<long long> hs(d);
    for (int k = 0; k < d; ++k) hs[k] = (long long)core_elems(dims, ranks, k);
    TTK_CHECK_CUDA(cudaMemcpyAsync(pdev, hp.data(), sizeof(double*) * d, cudaMemcpyHostToDevice, st));
    TTK_CHECK_CUDA(cudaMemcpyAsync(sdev, hs.data(), sizeof(long long) * d, cudaMemcpyHostToDevice, st));
    sumsq_multi_kernel<<<d, 256, 0, st>>>(pdev, sdev, red);
    TTK_CHECK_LAUNCH();
    TTK_CHECK_CUDA(cudaMemcpyAsync(pin, red, sizeof(double) * d, cudaMemcpyDeviceToHost, st));
    TTK_SYNC(st);
    for (int k = 0; k < d; ++k) prod_norm *= std::sqrt(pin[k]);
  }

  // ---- right-to-left orthogonalisation (tt.py:321-334) ----
  int qr_hint = 0;  // per sweep: try the rank-robust QR first after it was needed
  for (int k = d - 1; k >= 1; --k) {
    const double* ck = (k == d - 1) ? cores[k] : wk[k];
    const int r0 = r[k], n = dims[k], r1 = r[k + 1];
    const int m = n * r1, kk = std::min(m, r0);
    // QR of C_k^T (m x r0): element (row=(i,b), col=a) at a*m + row
    TTK_TRY(qr_auto(m, r0, ck, 1, m, wk[k], 1, m, tR, qws, qr_bytes, st, &qr_hint));
    // new core k = Q^T reshaped (kk, n, r1): element (c, row) at c*m + row  -> written above
    // C_{k-1} <- C_{k-1} x_3 R^T : new[a,i,c] = sum_b C_{k-1}[a,i,b] R[c,b]
    // core k-1 is still the untouched input core at this point of the sweep
    const double* cprev = cores[k - 1];
    const int p0 = r[k - 1], pn = dims[k - 1];
    TTK_TRY(gemm1(p0 * pn, kk, r0, cprev, r0, 1, tR, 1, r0, wk[k - 1], kk, 1, split_ws, st));
    r[k] = kk;
  }
  // ---- norm / zero test ----
  TTK_TRY(launch_sumsq(wk[0], (long long)r[0] * dims[0] * r[1], red, part, st));
  TTK_CHECK_CUDA(cudaMemcpyAsync(pin, red, sizeof(double), cudaMemcpyDeviceToHost, st));
  TTK_SYNC(st);
  const double nrm = std::sqrt(pin[0]);
  if (nrm == 0.0 || (zero_rel >= 0.0 && nrm <= zero_rel * prod_norm)) {
    for (int k = 0; k < d; ++k) TTK_CHECK_CUDA(cudaMemsetAsync(out[k], 0, sizeof(double) * dims[k], st));
    for (int k = 0; k <= d; ++k) out_ranks[k] = 1;
    TTK_SYNC(st);
    return kOk;
  }
  const double budget = rel_tol * nrm / std::sqrt((double)(d - 1));

  // ---- left-to-right truncated SVD sweep (tt.py:358-367) ----
  const double* cur = wk[0];
  qr_hint = 0;  // new sweep
  for (int k = 0; k < d - 1; ++k) {
    const int r0 = r[k], n = dims[k], r1 = r[k + 1];
    const int m = r0 * n, kk = std::min(m, r1);
    // A = Q R (Q: m x kk in tq, R: kk x r1 in tR)
    TTK_TRY(qr_auto(m, r1, cur, r1, 1, tq, kk, 1, tR, qws, qr_bytes, st, &qr_hint));
    const bool vt = jacobi_fits_v(r1, kk);
    if (vt) {
      // Jacobi on R^T (converges in far fewer sweeps for graded spectra):
      // R^T V' = W (= U' S), so R = V' S U'^T: left vectors V' in tU, W in tC
      TTK_TRY(jacobi_svd_ex(r1, kk, tR, 1, r1, tC, tS, tU, true, st));
    } else {
      // R = U S V^T (U: kk x kk, S)
      TTK_TRY(jacobi_svd(kk, r1, tR, tU, tS, nullptr, st));
    }
    TTK_TRY(truncation_rank_dev(tS, kk, budget, max_rank, rdev, st));
    TTK_CHECK_CUDA(cudaMemcpyAsync(pin, rdev, sizeof(int), cudaMemcpyDeviceToHost, st));
    TTK_SYNC(st);
    const int rk = *(int*)pin;
    // out_k = Q U[:, :rk]  (m x rk)
    TTK_TRY(gemm1(m, rk, kk, tq, kk, 1, tU, kk, 1, out[k], rk, 1, split_ws, st));
    if (vt) {
      // carry = S_r U'_r^T = W[:, :rk]^T  (rk x r1); copy-transpose via GEMM with I is
      // avoided by reading W transposed in the next product
    } else {
      // carry = U[:, :rk]^T R  (rk x r1)
      TTK_TRY(gemm1(rk, r1, kk, tU, 1, kk, tR, r1, 1, tC, r1, 1, split_ws, st));
    }
    // next core <- carry x_1 C_{k+1}: (rk x r1) (r1 x n' r2)
    const int n1 = dims[k + 1], r2 = r[k + 2];
    double* dst = alt[k & 1];
    // carry (rk x r1): vt -> W^T with W (r1 x kk) row-major, else tC (rk x r1)
    const long long c_ms = vt ? 1 : r1, c_ks = vt ? kk : 1;
    TTK_TRY(gemm1(rk, n1 * r2, r1, tC, c_ms, c_ks, wk[k + 1], (long long)n1 * r2, 1, dst,
                  (long long)n1 * r2, 1, split_ws, st));
    cur = dst;
    r[k + 1] = rk;
  }
  TTK_CHECK_CUDA(cudaMemcpyAsync(out[d - 1], cur, sizeof(double) * (size_t)r[d - 1] * dims[d - 1],
                                 cudaMemcpyDeviceToDevice, st));
  TTK_SYNC(st);
  for (int k = 0; k <= d; ++k) out_ranks[k] = r[k];
  return kOk;
}


// --------------------------------------------------------------------------
// Right-to-left truncation of a LEFT-ORTHOGONAL TT (cores 0..d-2 left-
// orthonormal, e.g. the RTO output): the TT-SVD in its right-to-left form,
// which needs no orthogonalisation sweep.  For k = d-1 .. 1:
//   C_k (r_{k-1} x n r_k) = V S (Q U)^T  via  C_k^T = Q R,  R = U S V^T,
//   keep r = truncation rank of S (budget rel_tol ||v|| / sqrt(d-1), cap),
//   C_k <- (Q U_r)^T,  C_{k-1} <- C_{k-1} x_3 (R^T U_r)   [= V_r S_r].
// Oracle: oracle/ttoracle.py truncate_left_orth.
size_t ttk_tt_truncate_ws_bytes(int d, const int* dims, const int* ranks) {
  size_t sum = 0, mx = 0, qrws = 0;
  int rmax = 1;
  for (int k = 0; k < d; ++k) {
    size_t e = core_elems(dims, ranks, k);
    sum += align_up(e * 8, 256);
    mx = std::max(mx, e);
    rmax = std::max(rmax, std::max(ranks[k], ranks[k + 1]));
    if (k > 0) qrws = std::max(qrws, qr_auto_ws_bytes(dims[k] * ranks[k + 1], ranks[k]));
  }
  return sum + 4 * align_up(mx * 8, 256) + 7 * align_up((size_t)rmax * rmax * 8, 256) +
         align_up(qrws, 256) + 2 * kSplitKBytes + 131072;
}

static int truncate_impl(int d, const int* dims, const int* ranks, const double* const* cores, double rel_tol,
                         int max_rank, double* const* out, int* out_ranks, double* const* host_out, void* ws,
                         size_t ws_bytes, cudaStream_t st, int mode) {
  // mode 2: Gram path with the gap-certified subspace kernel where it fits,
  // 1: Gram path with the Jacobi SVD, 0: QR path only
  TTK_REQUIRE(d >= 1 && rel_tol >= 0.0, kInvalidValue, "tt_truncate: bad arguments");
  for (int k = 0; k <= d; ++k) out_ranks[k] = ranks[k];
  if (d == 1) {
    TTK_CHECK_CUDA(cudaMemcpyAsync(out[0], cores[0], sizeof(double) * dims[0], cudaMemcpyDeviceToDevice, st));
    if (host_out)
      TTK_CHECK_CUDA(cudaMemcpyAsync(host_out[0], cores[0], sizeof(double) * dims[0], cudaMemcpyDeviceToHost, st));
    TTK_SYNC(st);
    return kOk;
  }
  const size_t need = ttk_tt_truncate_ws_bytes(d, dims, ranks);
  TTK_REQUIRE(ws != nullptr && ws_bytes >= need, kWorkspace, "tt_truncate: workspace %zu < %zu", ws_bytes,
              need);
  Arena ar(ws, ws_bytes);
  size_t mx = 0, qrb = 0;
  int rmax = 1;
  for (int k = 0; k < d; ++k) {
    mx = std::max(mx, core_elems(dims, ranks, k));
    rmax = std::max(rmax, std::max(ranks[k], ranks[k + 1]));
    if (k > 0) qrb = std::max(qrb, qr_auto_ws_bytes(dims[k] * ranks[k + 1], ranks[k]));
  }
  double* alt[2] = {ar.take<double>(mx), ar.take<double>(mx)};
  // Q and U double-buffered: the core's own product (Q U_r)^T runs on a side
  // stream while the next core is factorised
  double* tqb[2] = {ar.take<double>(mx), ar.take<double>(mx)};
  double* tR = ar.take<double>((size_t)rmax * rmax);
  double* tUb[2] = {ar.take<double>((size_t)rmax * rmax), ar.take<double>((size_t)rmax * rmax)};
  double* tS = ar.take<double>((size_t)rmax + 8);
  double* tL = ar.take<double>((size_t)rmax * rmax);
  double* tG = ar.take<double>((size_t)rmax * rmax);
  double* red = ar.take<double>(16);
  double* part = ar.take<double>(256);
  int* rdev = ar.take<int>(8);
  int* gflags = ar.take<int>((size_t)d + 8);
  size_t qoff = align_up(ar.used, 256);
  void* qws = (char*)ws + qoff;
  ar.used = qoff + qrb;
  void* split_ws = ar.take<char>(kSplitKBytes);
  void* split_side = ar.take<char>(kSplitKBytes);
  TTK_REQUIRE(split_side != nullptr, kWorkspace, "tt_truncate: workspace too small");
  static thread_local cudaStream_t side = nullptr;
  static thread_local cudaEvent_t ev_f[2] = {nullptr, nullptr}, ev_g[2] = {nullptr, nullptr},
                                  ev_r[2] = {nullptr, nullptr}, ev_d = nullptr;
  // host copies of final cores run on their own stream, so that the chain's
  // buffer-reuse waits (ev_g: the side product has read tq / tU) never wait
  // on PCIe
  static thread_local cudaStream_t d2h = nullptr;
  if (side == nullptr) {
    TTK_CHECK_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    TTK_CHECK_CUDA(cudaStreamCreateWithFlags(&d2h, cudaStreamNonBlocking));
    TTK_CHECK_CUDA(cudaEventCreateWithFlags(&ev_d, cudaEventDisableTiming));
    for (int i = 0; i < 2; ++i) {
      TTK_CHECK_CUDA(cudaEventCreateWithFlags(&ev_f[i], cudaEventDisableTiming));
      TTK_CHECK_CUDA(cudaEventCreateWithFlags(&ev_g[i], cudaEventDisableTiming));
      TTK_CHECK_CUDA(cudaEventCreateWithFlags(&ev_r[i], cudaEventDisableTiming));
    }
  }
  bool g_pending[2] = {false, false};
  // Gram path: the side-stream product of core k reads C_k (alt[(k+1) & 1]),
  // which the main stream overwrites at core k - 2 (its C_{k-3}) -- ev_r marks
  // the end of that read (before the host copy, which must not gate the chain)
  bool r_pending[2] = {false, false};
  double* pin = (double*)g_pinned.get(sizeof(double) * ((size_t)std::max(rmax, d) + 16));
  TTK_REQUIRE(pin != nullptr, kCudaError, "tt_truncate: cannot allocate pinned scratch");
  std::vector<int> r(ranks, ranks + d + 1);
  // Gram path (exact-rank roundings, rel_tol == 0; set up below): the budget is
  // zero whatever the norm, so the norm's host round trip is skipped (a zero
  // tensor fails every certificate and comes back here through the QR path)
  const bool gram_mode = mode >= 1 && rel_tol == 0.0 && knob_env("TTK_TRUNC_NO_GRAM") == nullptr;
  // ||v|| = ||C_{d-1}||_F for a left-orthogonal TT
  double nrm = 1.0;
  if (!gram_mode) {
    TTK_TRY(launch_sumsq(cores[d - 1], (long long)r[d - 1] * dims[d - 1], red, part, st));
    TTK_CHECK_CUDA(cudaMemcpyAsync(pin, red, sizeof(double), cudaMemcpyDeviceToHost, st));
    TTK_SYNC(st);
    nrm = std::sqrt(pin[0]);
  }
  if (nrm == 0.0) {
    for (int k = 0; k < d; ++k) TTK_CHECK_CUDA(cudaMemsetAsync(out[k], 0, sizeof(double) * dims[k], st));
    for (int k = 0; k <= d; ++k) out_ranks[k] = 1;
    TTK_SYNC(st);
    if (host_out)
      for (int k = 0; k < d; ++k) memset(host_out[k], 0, sizeof(double) * dims[k]);
    return kOk;
  }
  const double budget = rel_tol * nrm / std::sqrt((double)(d - 1));
  const double* cur = cores[d - 1];
  int qr_hint = 0;  // per sweep: try the rank-robust QR first after it was needed
  // Gram path (exact-rank roundings, rel_tol == 0): R from the Cholesky factor of
  // G = C_k C_k^T instead of the QR of C_k^T (no Q: the new core is
  // S_r^{-2} W_r^T C_k with W = R^T V).  Its rank is min(cap, r0) whenever the
  // core's certificate holds (gram_cert_kernel), so the sweep is enqueued with
  // no host round trip per core and the certificates are checked once at the
  // end; if any failed (e.g. an exactly rank-deficient unfolding) the whole
  // truncation is redone through the QR path.
  const bool gram_on = gram_mode;
  const uint64_t skey = trunc_shape_key(d, dims, ranks, max_rank);
  bool fast_on = gram_on && mode >= 2 && knob_env("TTK_TRUNC_NO_FAST") == nullptr;
  if (fast_on) {
    auto it = g_fast_skip.find(skey);
    if (it != g_fast_skip.end() && it->second > 0) {
      --it->second;
      fast_on = false;
    }
  }
  int ngram = 0, nfast = 0;
  for (int k = d - 1; k >= 1; --k) {
    const int r0 = r[k], n = dims[k], r1 = r[k + 1];
    const int m = n * r1, kk = std::min(m, r0);
    double* const tq = tqb[k & 1];
    double* const tU = tUb[k & 1];
    // the side-stream product of core k + 2 read these buffers
    if (g_pending[k & 1]) TTK_CHECK_CUDA(cudaStreamWaitEvent(st, ev_g[k & 1], 0));
    if (gram_on && m >= r0 && r0 >= 2 && r0 <= kCholBlockedMaxCols && jacobi_fits_v(r0, r0)) {
      // G = C C^T (r0 x r0), C = cur (r0 x m, row-major)
      if (gram_wide_fits(r0, m, kSplitKBytes)) TTK_TRY(gram_wide(r0, m, cur, tG, split_ws, st));
      else TTK_TRY(gemm1(r0, r0, m, cur, m, 1, cur, 1, m, tG, r0, 1, split_ws, st));
      const int rk = std::min(max_rank > 0 ? max_rank : r0, r0);
      if (fast_on && trunc_subspace_fits(r0, rk)) {
        // F = C Y^T -> tL, M^T -> tU (Y = M C), certificate -> gflags
        TTK_TRY(launch_trunc_subspace(r0, rk, tG, tL, tU, r0, gflags + ngram, nullptr, st));
        ++ngram;
        ++nfast;
      } else {
        TTK_CHECK_CUDA(cudaMemsetAsync(rdev + 2, 0, sizeof(int), st));
        TTK_TRY(launch_chol_inv(r0, tG, tR, nullptr, rdev + 2, 0, 0.0, 1e-15, st, nullptr));
        TTK_TRY(jacobi_svd_ex(r0, r0, tR, 1, r0, tL, tS, nullptr, true, st));  // W and S only
        gram_cert_kernel<<<1, 32, 0, st>>>(tS, rk, rdev + 2, gflags + ngram);
        TTK_CHECK_LAUNCH();
        ++ngram;
        // T1 = W_r S_r^{-2}; L = W_r
        scale_cols_inv_sq_kernel<<<ceil_div((long)r0 * rk, 256), 256, 0, st>>>(r0, rk, tL, r0, tS, tU);
        TTK_CHECK_LAUNCH();
      }
      {
        // core k <- T1^T C (side stream); C_{k-1} <- C_{k-1} L
        TTK_CHECK_CUDA(cudaEventRecord(ev_f[k & 1], st));
        TTK_CHECK_CUDA(cudaStreamWaitEvent(side, ev_f[k & 1], 0));
        TTK_TRY(gemm1(m, rk, r0, cur, 1, m, tU, r0, 1, out[k], 1, m, split_side, side, 1.0, 0.0, true));
        TTK_CHECK_CUDA(cudaEventRecord(ev_r[k & 1], side));
        r_pending[k & 1] = true;
        TTK_CHECK_CUDA(cudaEventRecord(ev_g[k & 1], side));
        g_pending[k & 1] = true;
        if (host_out) {
          TTK_CHECK_CUDA(cudaStreamWaitEvent(d2h, ev_g[k & 1], 0));
          TTK_CHECK_CUDA(cudaMemcpyAsync(host_out[k], out[k], sizeof(double) * (size_t)rk * m,
                                         cudaMemcpyDeviceToHost, d2h));
        }
        const int p0 = r[k - 1], pn = dims[k - 1];
        double* dst = alt[k & 1];
        if (r_pending[(k + 1) & 1]) {  // core k+1's side product read dst
          TTK_CHECK_CUDA(cudaStreamWaitEvent(st, ev_r[(k + 1) & 1], 0));
          r_pending[(k + 1) & 1] = false;
        }
        TTK_TRY(gemm1(p0 * pn, rk, r0, cores[k - 1], r0, 1, tL, r0, 1, dst, rk, 1, split_ws, st));
        cur = dst;
        r[k] = rk;
        continue;
      }
    }
    g_trunc_qr.fetch_add(1, std::memory_order_relaxed);
    // C_k^T (m x r0) = Q R ; element (row=(i,b), col=a) of C_k^T at a*m + row
    TTK_TRY(qr_auto(m, r0, cur, 1, m, tq, kk, 1, tR, qws, qrb, st, &qr_hint));
    const bool vt = jacobi_fits_v(r0, kk);
    if (vt) {
      // Jacobi on R^T (r0 x kk): R^T V' = W = U' S; left vectors of R = V' (tU),
      // and L = R^T V'_r = W[:, :r] (tL, r0 x kk, leading rk columns used)
      TTK_TRY(jacobi_svd_ex(r0, kk, tR, 1, r0, tL, tS, tU, true, st));
    } else {
      TTK_TRY(jacobi_svd(kk, r0, tR, tU, tS, nullptr, st));
    }
    TTK_TRY(truncation_rank_dev(tS, kk, budget, max_rank, rdev, st));
    TTK_CHECK_CUDA(cudaMemcpyAsync(pin, rdev, sizeof(int), cudaMemcpyDeviceToHost, st));
    TTK_SYNC(st);
    const int rk = *(int*)pin;
    // C_k <- (Q U_r)^T : out[k][c][row] = sum_j Q[row][j] U[j][c]  (side stream:
    // only L feeds the next core)
    TTK_CHECK_CUDA(cudaEventRecord(ev_f[k & 1], st));
    TTK_CHECK_CUDA(cudaStreamWaitEvent(side, ev_f[k & 1], 0));
    TTK_TRY(gemm1(m, rk, kk, tq, kk, 1, tU, kk, 1, out[k], 1, m, split_side, side, 1.0, 0.0, true));
    TTK_CHECK_CUDA(cudaEventRecord(ev_g[k & 1], side));
    g_pending[k & 1] = true;
    // core k is final: stream it to the caller's pinned host buffer behind the
    // rest of the sweep (after the product, on the copy stream)
    if (host_out) {
      TTK_CHECK_CUDA(cudaStreamWaitEvent(d2h, ev_g[k & 1], 0));
      TTK_CHECK_CUDA(cudaMemcpyAsync(host_out[k], out[k], sizeof(double) * (size_t)rk * m, cudaMemcpyDeviceToHost,
                                     d2h));
    }
    long long l_ld = kk;
    if (!vt) {
      // L = R^T U_r (r0 x rk)
      TTK_TRY(gemm1(r0, rk, kk, tR, 1, r0, tU, kk, 1, tL, rk, 1, split_ws, st));
      l_ld = rk;
    }
    // C_{k-1} <- C_{k-1} x_3 L
    const int p0 = r[k - 1], pn = dims[k - 1];
    double* dst = alt[k & 1];
    if (r_pending[(k + 1) & 1]) {  // core k+1's side product (Gram path) read dst
      TTK_CHECK_CUDA(cudaStreamWaitEvent(st, ev_r[(k + 1) & 1], 0));
      r_pending[(k + 1) & 1] = false;
    }
    TTK_TRY(gemm1(p0 * pn, rk, r0, cores[k - 1], r0, 1, tL, l_ld, 1, dst, rk, 1, split_ws, st));
    cur = dst;
    r[k] = rk;
  }
  TTK_CHECK_CUDA(cudaMemcpyAsync(out[0], cur, sizeof(double) * (size_t)dims[0] * r[1],
                                 cudaMemcpyDeviceToDevice, st));
  if (host_out)
    TTK_CHECK_CUDA(cudaMemcpyAsync(host_out[0], cur, sizeof(double) * (size_t)dims[0] * r[1],
                                   cudaMemcpyDeviceToHost, st));
  for (int i = 0; i < 2; ++i)
    if (g_pending[i]) TTK_CHECK_CUDA(cudaStreamWaitEvent(st, ev_g[i], 0));
  if (host_out) {  // every host copy has landed before the call returns
    TTK_CHECK_CUDA(cudaEventRecord(ev_d, d2h));
    TTK_CHECK_CUDA(cudaStreamWaitEvent(st, ev_d, 0));
  }
  int* hflags = reinterpret_cast<int*>(pin);
  if (ngram > 0) TTK_CHECK_CUDA(cudaMemcpyAsync(hflags, gflags, sizeof(int) * ngram, cudaMemcpyDeviceToHost, st));
  TTK_SYNC(st);
  for (int i = 0; i < ngram; ++i)
    if (hflags[i] != 1) {
      if (nfast > 0) {  // redo with the Jacobi SVD on every core; skip the subspace kernel for a while
        g_trunc_fast_redo.fetch_add(1, std::memory_order_relaxed);
        g_fast_skip[skey] = kFastSkip;
        return truncate_impl(d, dims, ranks, cores, rel_tol, max_rank, out, out_ranks, host_out, ws, ws_bytes,
                             st, 1);
      }
      g_trunc_redo.fetch_add(1, std::memory_order_relaxed);
      return truncate_impl(d, dims, ranks, cores, rel_tol, max_rank, out, out_ranks, host_out, ws, ws_bytes, st,
                           0);
    }
  g_trunc_gram.fetch_add(ngram - nfast, std::memory_order_relaxed);
  g_trunc_fast.fetch_add(nfast, std::memory_order_relaxed);
  for (int k = 0; k <= d; ++k) out_ranks[k] = r[k];
  return kOk;
}

int ttk_tt_truncate_host(int d, const int* dims, const int* ranks, const double* const* cores, double rel_tol,
                         int max_rank, double* const* out, int* out_ranks, double* const* host_out, void* ws,
                         size_t ws_bytes, void* stream) {
  return truncate_impl(d, dims, ranks, cores, rel_tol, max_rank, out, out_ranks, host_out, ws, ws_bytes,
                       (cudaStream_t)stream, 2);
}

// Process-wide switch of the TMA-staged GEMM inside the sweeps (default on);
// returns the previous setting.  Callers that keep several problems in flight
// on different streams turn it off (see tma_allowed).
int ttk_gemm_tma_enable(int on) { return g_tma_enabled.exchange(on ? 1 : 0); }

int ttk_debug_truncate_paths(long long* counts) {
  counts[0] = g_trunc_gram.load();
  counts[1] = g_trunc_qr.load();
  counts[2] = g_trunc_redo.load();
  return kOk;
}

int ttk_debug_truncate_paths_ex(long long* counts, int n) {
  const long long v[7] = {g_trunc_gram.load(), g_trunc_qr.load(), g_trunc_redo.load(), g_trunc_fast.load(),
                          g_trunc_fast_redo.load(), g_rto_deferred.load(), g_rto_defer_redo.load()};
  for (int i = 0; i < n && i < 7; ++i) counts[i] = v[i];
  return kOk;
}

int ttk_tt_truncate(int d, const int* dims, const int* ranks, const double* const* cores, double rel_tol,
                    int max_rank, double* const* out, int* out_ranks, void* ws, size_t ws_bytes,
                    void* stream) {
  return ttk_tt_truncate_host(d, dims, ranks, cores, rel_tol, max_rank, out, out_ranks, nullptr, ws, ws_bytes,
                              stream);
}

// --------------------------------------------------------------------------
size_t ttk_rto_ws_bytes(int d, const int* dims, const int* R, const int* L) {
  size_t wsum = 0, tsum = 0, ymax = 0, zmax = 0, mmax = 0, qr = 0;
  for (int c = 1; c < d; ++c) wsum += align_up((size_t)R[c] * L[c] * 8, 256);
  for (int c = 1; c + 1 < d; ++c) tsum += align_up((size_t)R[c] * dims[c] * L[c + 1] * 8, 256);
  for (int c = 1; c < d; ++c) {
    size_t m = (size_t)L[c - 1] * dims[c - 1];
    ymax = std::max(ymax, m * L[c]);
    zmax = std::max(zmax, (size_t)L[c - 1] * dims[c - 1] * R[c]);
    mmax = std::max(mmax, (size_t)L[c] * R[c]);
    qr = std::max(qr, qr_auto_ws_bytes((int)m, L[c]));
  }
  return wsum + tsum + align_up(ymax * 8, 256) + 2 * align_up(zmax * 8, 256) + 2 * align_up(mmax * 8, 256) +
         align_up(qr, 256) + 2 * kSplitKBytes + 65536 + align_up((size_t)d * 8 * sizeof(int), 256);
}

// Shapes whose last left sweep had every factorisation accepted on the fused
// fast path: only those defer the acceptance check (the solver's roundings --
// rank-deficient sketches, a new shape every iteration -- never pay for a
// wasted sweep); a refused deferred sweep takes the shape out again.
thread_local std::unordered_map<uint64_t, bool> g_defer_ok;

// Randomize-then-orthogonalize sweeps.  X: d cores (R[k], n_k, R[k+1]); G: DRM
// cores (L[k], n_k, L[k+1]) with L[0] = L[d] = 1 and, for every cut c,
// L[c] <= min(R[c], L[c-1] * n_{c-1}); out: d cores (L[k], n_k, L[k+1]).
// Cores 0..d-2 of the result are left-orthonormal.
int ttk_rto_sweeps_ev(int d, const int* dims, const int* R, const double* const* X, const int* L,
                      const double* const* G, double* const* out, void* ws, size_t ws_bytes,
                      void* const* ready, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  // ready[c] (optional): event after which X[c] may be read -- lets the
  // caller stream the matvec output in core by core (right to left)
  auto wait_core = [&](int c) -> int {
    if (ready && ready[c]) TTK_CHECK_CUDA(cudaStreamWaitEvent(st, (cudaEvent_t)ready[c], 0));
    return kOk;
  };
  TTK_REQUIRE(d >= 1, kInvalidValue, "rto: d must be >= 1");
  TTK_REQUIRE(R[0] == 1 && R[d] == 1 && L[0] == 1 && L[d] == 1, kShapeMismatch,
              "rto: boundary ranks must equal 1");
  if (d == 1) {
    TTK_TRY(wait_core(0));
    TTK_CHECK_CUDA(cudaMemcpyAsync(out[0], X[0], sizeof(double) * dims[0], cudaMemcpyDeviceToDevice, st));
    return kOk;
  }
  for (int c = 1; c < d; ++c) {
    TTK_REQUIRE(L[c] >= 1 && L[c] <= R[c] && L[c] <= L[c - 1] * dims[c - 1], kInvalidValue,
                "rto: sketch rank L[%d]=%d must lie in [1, min(R=%d, L[c-1]*n=%d)]", c, L[c], R[c],
                L[c - 1] * dims[c - 1]);
  }
  const size_t need = ttk_rto_ws_bytes(d, dims, R, L);
  TTK_REQUIRE(ws != nullptr && ws_bytes >= need, kWorkspace, "rto: workspace %zu < %zu", ws_bytes, need);
  Arena ar(ws, ws_bytes);
  std::vector<double*> W(d + 1, nullptr), Tk(d + 1, nullptr);
  for (int c = 1; c < d; ++c) W[c] = ar.take<double>((size_t)R[c] * L[c]);
  // T_c = X_c W_{c+1} of the right sweep is kept: the left sweep's sketch of the
  // next projected core is Y_{c+1} = M_c T_c (see below)
  for (int c = 1; c + 1 < d; ++c) Tk[c] = ar.take<double>((size_t)R[c] * dims[c] * L[c + 1]);
  size_t ymax = 0, zmax = 0, mmax = 0, qrb = 0;
  for (int c = 1; c < d; ++c) {
    size_t m = (size_t)L[c - 1] * dims[c - 1];
    ymax = std::max(ymax, m * L[c]);
    zmax = std::max(zmax, (size_t)L[c - 1] * dims[c - 1] * R[c]);
    mmax = std::max(mmax, (size_t)L[c] * R[c]);
    qrb = std::max(qrb, qr_auto_ws_bytes((int)m, L[c]));
  }
  double* Y = ar.take<double>(ymax);
  double* Zbuf[2] = {ar.take<double>(zmax), ar.take<double>(zmax)};
  double* Mbuf[2] = {ar.take<double>(mmax), ar.take<double>(mmax)};
  size_t qoff = align_up(ar.used, 256);
  void* qws = (char*)ws + qoff;
  ar.used = qoff + qrb;
  void* split_ws = ar.take<char>(kSplitKBytes);
  void* split_side = ar.take<char>(kSplitKBytes);
  int* qstat = ar.take<int>((size_t)d * 8);  // acceptance flags of the left sweep's factorisations
  TTK_REQUIRE(split_side != nullptr && qstat != nullptr, kWorkspace, "rto: workspace too small");

  // ---- right sweep: W_c = sum_i X_c[:, i, :] W_{c+1} G_c[:, i, :]^T ----
  // pipelined callers (ready != nullptr) still have matvec chunks of this
  // problem running on another stream: no TMA-staged GEMM next to them (DESIGN 6.2)
  struct TmaSuppress {
    bool on;
    explicit TmaSuppress(bool o) : on(o) { if (on) ++g_tma_suppress; }
    ~TmaSuppress() { release(); }
    void release() { if (on) { --g_tma_suppress; on = false; } }
  } right_guard([&] {
    // one event for every core = one matvec launch the sweep waits for as a whole: nothing overlaps
    if (!ready) return false;
    for (int c = 0; c < d; ++c)
      if (ready[c] != ready[d - 1]) return true;
    return false;
  }());
  for (int c = d - 1; c >= 1; --c) {
    const int n = dims[c], rc = R[c], lc = L[c], l1 = L[c + 1], r1 = R[c + 1];
    TTK_TRY(wait_core(c));
    const double* Tin;
    if (c == d - 1) {
      Tin = X[c];  // (R_c, n, 1): W_d = [[1]]
    } else {
      // T_c (R_c n x L_{c+1}) = X_c (R_c n x R_{c+1}) W_{c+1} (R_{c+1} x L_{c+1})
      TTK_TRY(gemm1(rc * n, l1, r1, X[c], r1, 1, W[c + 1], l1, 1, Tk[c], l1, 1, split_ws, st));
      Tin = Tk[c];
    }
    // W_c (R_c x L_c) = T (R_c x n L_{c+1}) G_c^T ; G_c viewed (L_c x n L_{c+1})
    const long long K = (long long)n * l1;
    TTK_TRY(gemm1(rc, lc, (int)K, Tin, K, 1, G[c], 1, K, W[c], lc, 1, split_ws, st));
  }
  // ---- left sweep ----
  // Step c orthogonalises the sketch Y_c of the projected core Z_{c-1}
  // (L_{c-1} n_{c-1} x R_c), then M_c = Q_c^T Z_{c-1}.  Since Z_c = M_c X_c,
  // the next sketch is Y_{c+1} = Z_c W_{c+1} = M_c T_c: only the small M_c is on
  // the critical path; Z_c itself (needed for M_{c+1}) is formed on a side
  // stream while Y_{c+1} is orthogonalised.
  // (running the orthogonalisation on a high-priority stream was measured to
  // make no difference: the step is bound by the QR chain's own latency)
  static thread_local cudaStream_t side = nullptr;
  static thread_local cudaEvent_t ev_m = nullptr, ev_z = nullptr;
  if (side == nullptr) {
    TTK_CHECK_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    TTK_CHECK_CUDA(cudaEventCreateWithFlags(&ev_m, cudaEventDisableTiming));
    TTK_CHECK_CUDA(cudaEventCreateWithFlags(&ev_z, cudaEventDisableTiming));
  }
  right_guard.release();
  // The CholeskyQR2 of every step is accepted on the device (flags in qstat) and
  // the host looks at all of them once, after the sweep: a per-core wait cost
  // ~30 us of host round trip per core (config 3: 0.9 ms of a 13.7 ms step).  If
  // a factorisation was refused the sweep is redone with the per-core check, which
  // takes the rank-robust path where needed.
  const uint64_t dkey = trunc_shape_key(d, dims, R, 0) ^ (trunc_shape_key(d, dims, L, 1) * 0x9E3779B97F4A7C15ull);
  bool defer = false;
  if (knob_env("TTK_RTO_NO_DEFER") == nullptr) {
    auto it = g_defer_ok.find(dkey);
    defer = it != g_defer_ok.end() && it->second;
  }
  bool all_fused = true;
  TTK_TRY(wait_core(0));
  for (int pass = 0; pass < 2; ++pass) {
  if (defer) TTK_CHECK_CUDA(cudaMemsetAsync(qstat, 0, sizeof(int) * 8 * (size_t)d, st));
  int qr_hint = 0;  // per sweep: try the rank-robust QR first after it was needed
  const double* Mprev = nullptr;
  for (int c = 1; c < d; ++c) {
    const int np = dims[c - 1];
    const int m = L[c - 1] * np, l = L[c], rc = R[c];
    const double* Z;
    if (c == 1) {
      Z = X[0];  // (n_0 x R_1)
      // Y (m x l) = X_0 W_1
      TTK_TRY(gemm1(m, l, rc, Z, rc, 1, W[c], l, 1, Y, l, 1, split_ws, st));
    } else {
      const int lp = L[c - 1], rp = R[c - 1];
      // side: Z_{c-1} (L_{c-1} x n_{c-1} R_c) = M_{c-1} X_{c-1}
      double* zdst = Zbuf[c & 1];
      static const bool no_side = knob_env("TTK_RTO_NO_SIDE") != nullptr;  // A/B
      cudaStream_t sd = no_side ? st : side;
      TTK_CHECK_CUDA(cudaEventRecord(ev_m, st));
      TTK_CHECK_CUDA(cudaStreamWaitEvent(sd, ev_m, 0));
      TTK_TRY(gemm1(lp, np * rc, rp, Mprev, rp, 1, X[c - 1], (long long)np * rc, 1, zdst, (long long)np * rc, 1,
                    split_side, sd, 1.0, 0.0, sd != st));
      TTK_CHECK_CUDA(cudaEventRecord(ev_z, sd));
      // main: Y (L_{c-1} x n_{c-1} L_c) = M_{c-1} (L_{c-1} x R_{c-1}) T_{c-1} (R_{c-1} x n_{c-1} L_c)
      TTK_TRY(gemm1(lp, np * l, rp, Mprev, rp, 1, Tk[c - 1], (long long)np * l, 1, Y, (long long)np * l, 1,
                    split_ws, st));
      Z = zdst;
    }
    // Q (m x l) -> out core c-1, (L_{c-1}, n_{c-1}, L_c)
    int fused_ok = 0;
    TTK_TRY(qr_auto(m, l, Y, l, 1, out[c - 1], l, 1, nullptr, qws, qrb, st, &qr_hint, defer ? qstat + 8 * c : nullptr,
                    &fused_ok));
    all_fused = all_fused && fused_ok;
    if (c > 1) TTK_CHECK_CUDA(cudaStreamWaitEvent(st, ev_z, 0));
    // M_c (l x R_c) = Q^T Z   (K = m, split over the long dimension)
    double* Mc = Mbuf[c & 1];
    TTK_TRY(gemm1(l, rc, m, out[c - 1], 1, l, Z, rc, 1, Mc, rc, 1, split_ws, st));
    Mprev = Mc;
  }
  // last core: (L_{d-1} x n_{d-1}) = M_{d-1} X_{d-1}
  {
    const int c = d - 1, l = L[c], rc = R[c], n = dims[c];
    TTK_TRY(gemm1(l, n, rc, Mprev, rc, 1, X[c], n, 1, out[d - 1], n, 1, split_ws, st));
  }
  if (!defer) {
    if (g_defer_ok.size() > 4096) g_defer_ok.clear();
    g_defer_ok[dkey] = all_fused;
    break;
  }
  int* hq = reinterpret_cast<int*>(g_pinned.get(sizeof(int) * 8 * (size_t)d + 64));
  TTK_REQUIRE(hq != nullptr, kCudaError, "rto: cannot allocate pinned scratch");
  TTK_CHECK_CUDA(cudaMemcpyAsync(hq, qstat, sizeof(int) * 8 * (size_t)d, cudaMemcpyDeviceToHost, st));
  TTK_SYNC(st);
  bool refused = false;
  for (int c = 1; c < d; ++c) refused = refused || hq[8 * c] != 0 || hq[8 * c + 1] != 0;
  if (!refused) {
    g_rto_deferred.fetch_add(1, std::memory_order_relaxed);
    break;
  }
  g_rto_defer_redo.fetch_add(1, std::memory_order_relaxed);
  g_defer_ok[dkey] = false;
  defer = false;  // second pass: per-core acceptance
  all_fused = true;
  }
  return kOk;
}

int ttk_rto_sweeps(int d, const int* dims, const int* R, const double* const* X, const int* L,
                   const double* const* G, double* const* out, void* ws, size_t ws_bytes, void* stream) {
  return ttk_rto_sweeps_ev(d, dims, R, X, L, G, out, ws, ws_bytes, nullptr, stream);
}

}  // extern "C"
