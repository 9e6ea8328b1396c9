// STTA recovery (reference stream_recover, streaming.py:166-205) and the
// entrywise sketch-pair combination (combine_pairs, streaming.py:145-163).
#include "gemm.cuh"
#include "qr.cuh"
#include "../../include/ttk_b200.h"

#include <algorithm>
#include <cmath>
#include <vector>

namespace ttk {

constexpr int kMaxAxpyTerms = 64;
struct AxpyParams {
  int nterms;
  long long n;
  double coeff[kMaxAxpyTerms];
  const double* in[kMaxAxpyTerms];
  double* out;
};

// out = c0*in0 + c1*in1 + ... accumulated left to right with separate
// multiply and add roundings (numpy's `psi += a * m`, streaming.py:158,259)
__global__ void axpy_multi_kernel(const __grid_constant__ AxpyParams P) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < P.n;
       e += (long long)gridDim.x * blockDim.x) {
    double acc = __dmul_rn(P.in[0][e], P.coeff[0]);
    for (int t = 1; t < P.nterms; ++t) acc = __dadd_rn(acc, __dmul_rn(P.coeff[t], P.in[t][e]));
    P.out[e] = acc;
  }
}

// keep count and the two half pseudo-inverse factors of one Omega (k x l):
//   LH = S^{-1/2} U^T (kept x k),  RH = V S^{-1/2} (l x kept)
// copy of X (n entries) scaled by an exact power of two
__global__ void scale_copy_kernel(long long n, const double* __restrict__ X, double s, double* __restrict__ Y) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x)
    Y[e] = X[e] * s;
}

// S, U, V: SVD of the cross matrix scaled by 2^e (unscale = 2^(e/2) restores
// 1/sqrt of the true singular values)
__global__ void recover_halves_kernel(int k, int l, const double* U, const double* S, const double* V,
                                      double rcond, double unscale, double* LH, double* RH, int* kept_out) {
  const int kn = min(k, l);
  __shared__ int kept;
  if (threadIdx.x == 0) {
    int c = 0;
    const double s0 = S[0];
    for (int i = 0; i < kn; ++i) c += (S[i] > rcond * s0) ? 1 : 0;
    kept = c;
    *kept_out = c;
  }
  __syncthreads();
  const int c = kept;
  for (int e = threadIdx.x; e < c * k; e += blockDim.x) {
    int i = e / k, j = e - i * k;
    LH[e] = U[(long long)j * kn + i] * (unscale / sqrt(S[i]));
  }
  for (int e = threadIdx.x; e < l * c; e += blockDim.x) {
    int j = e / c, i = e - j * c;
    RH[e] = V[(long long)j * kn + i] * (unscale / sqrt(S[i]));
  }
}

__global__ void sumsq_list_kernel(const double* const* ptrs, const long long* sizes, double* out) {
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

}  // namespace ttk

using namespace ttk;

extern "C" {

// out[e] = sum_t coeff[t] * in_t[e] for e < n, t < nterms (<= 64 per launch; longer lists chain)
int ttk_axpy_multi(int nterms, const double* coeff, const double* const* in, long long n, double* out,
                   void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  TTK_REQUIRE(nterms >= 1, kInvalidValue, "axpy_multi: need at least one term");
  if (n <= 0) return kOk;
  static thread_local AxpyParams P;
  int done = 0;
  while (done < nterms) {
    int take = std::min(kMaxAxpyTerms - (done ? 1 : 0), nterms - done);
    int t = 0;
    if (done) { P.coeff[t] = 1.0; P.in[t] = out; ++t; }
    for (int i = 0; i < take; ++i, ++t) { P.coeff[t] = coeff[done + i]; P.in[t] = in[done + i]; }
    P.nterms = t;
    P.n = n;
    P.out = out;
    int blocks = (int)std::min<long long>((n + 255) / 256, 8LL * kNumSMs);
    axpy_multi_kernel<<<blocks, 256, 0, st>>>(P);
    TTK_CHECK_LAUNCH();
    done += take;
  }
  return kOk;
}

size_t ttk_stream_recover_ws_bytes(int d, const int* dims, const int* lr, const int* rr) {
  size_t tot = 0, tmax = 0;
  for (int mu = 1; mu < d; ++mu) {
    const size_t k = lr[mu], l = rr[mu], kn = std::min(k, l);
    tot += align_up(k * kn * 8, 256) + align_up(kn * 8, 256) + align_up(l * kn * 8, 256) +
           align_up(kn * k * 8, 256) + align_up(l * kn * 8, 256);
  }
  for (int mu = 0; mu < d; ++mu)
    tmax = std::max(tmax, std::max((size_t)std::max(lr[mu], rr[mu]) * dims[mu] * rr[mu + 1], (size_t)lr[mu] * rr[mu]));
  return tot + align_up(tmax * 8, 256) + (size_t)(4 * d + 16) * 256 + (16u << 20) + 65536;
}

// STTA core recovery: psi[mu] ((lr[mu] n_mu) x rr[mu+1]), omega[mu-1] (lr[mu] x rr[mu]).
// Writes the (unrounded) recovered cores into out[mu] (capacity
// max(lr[mu], rr[mu]) * n_mu * rr[mu+1]) and their ranks into out_ranks (host).
// Returns TTK_DEGENERATE for an all-zero Omega with nonzero Psi; an all-zero
// Psi list gives out_ranks all 1 and a zero flag in *is_zero (reference
// streaming.py:179-180).  Synchronises `stream`.
int ttk_stream_recover_cores(int d, const int* dims, const int* lr, const int* rr,
                             const double* const* psi, const double* const* omega, double rcond,
                             double* const* out, int* out_ranks, int* is_zero, void* ws,
                             size_t ws_bytes, void* stream) {
  cudaStream_t st = (cudaStream_t)stream;
  const size_t need = ttk_stream_recover_ws_bytes(d, dims, lr, rr);
  TTK_REQUIRE(ws != nullptr && ws_bytes >= need, kWorkspace, "stream_recover: workspace %zu < %zu",
              ws_bytes, need);
  Arena ar(ws, ws_bytes);
  std::vector<double*> U(d), S(d), V(d), LH(d), RH(d);
  for (int mu = 1; mu < d; ++mu) {
    const size_t k = lr[mu], l = rr[mu], kn = std::min(k, l);
    U[mu] = ar.take<double>(k * kn);
    S[mu] = ar.take<double>(kn);
    V[mu] = ar.take<double>(l * kn);
    LH[mu] = ar.take<double>(kn * k);
    RH[mu] = ar.take<double>(l * kn);
  }
  size_t tmax = 0;
  for (int mu = 0; mu < d; ++mu)
    tmax = std::max(tmax, std::max((size_t)std::max(lr[mu], rr[mu]) * dims[mu] * rr[mu + 1], (size_t)lr[mu] * rr[mu]));
  double* T = ar.take<double>(tmax);
  double* red = ar.take<double>(2 * (size_t)d + 8);
  int* kept = ar.take<int>((size_t)d + 8);
  const double** pdev = ar.take<const double*>(2 * (size_t)d);
  long long* sdev = ar.take<long long>(2 * (size_t)d);
  void* split_ws = ar.take<char>(16u << 20);
  TTK_REQUIRE(split_ws != nullptr, kWorkspace, "stream_recover: workspace too small");

  // zero / degenerate checks: sum of squares of every Psi and Omega
  std::vector<const double*> hp;
  std::vector<long long> hs;
  for (int mu = 0; mu < d; ++mu) { hp.push_back(psi[mu]); hs.push_back((long long)lr[mu] * dims[mu] * rr[mu + 1]); }
  for (int mu = 1; mu < d; ++mu) { hp.push_back(omega[mu - 1]); hs.push_back((long long)lr[mu] * rr[mu]); }
  const int nl = (int)hp.size();
  TTK_CHECK_CUDA(cudaMemcpyAsync(pdev, hp.data(), sizeof(double*) * nl, cudaMemcpyHostToDevice, st));
  TTK_CHECK_CUDA(cudaMemcpyAsync(sdev, hs.data(), sizeof(long long) * nl, cudaMemcpyHostToDevice, st));
  sumsq_list_kernel<<<nl, 256, 0, st>>>(pdev, sdev, red);
  TTK_CHECK_LAUNCH();
  std::vector<double> hred(nl);
  TTK_CHECK_CUDA(cudaMemcpyAsync(hred.data(), red, sizeof(double) * nl, cudaMemcpyDeviceToHost, st));
  TTK_SYNC(st);
  bool all_zero = true;
  for (int mu = 0; mu < d; ++mu) all_zero = all_zero && hred[mu] == 0.0;
  *is_zero = all_zero ? 1 : 0;
  if (all_zero) {
    for (int k = 0; k <= d; ++k) out_ranks[k] = 1;
    return kOk;
  }
  for (int mu = 1; mu < d; ++mu)
    TTK_REQUIRE(hred[d + mu - 1] != 0.0, kDegenerate, "zero cross matrix at mode %d", mu);

  // truncated SVDs of the cross matrices and their symmetric half inverses.
  // Omega is scaled by an exact power of two to unit size first (as LAPACK's
  // dgesdd scales): at d = 50 its entries are ~1e-106, the Jacobi rotation
  // tests square the products (~1e-424) and underflow, leaving noise singular
  // values at the level of the large ones (config-5 solutions blew up to 1e71)
  for (int mu = 1; mu < d; ++mu) {
    const int k = lr[mu], l = rr[mu];
    const double fro = std::sqrt(hred[d + mu - 1]);
    const int e = -std::ilogb(fro);              // fro * 2^e in [1, 2)
    const double sc = std::ldexp(1.0, e);
    const double unscale = (e % 2 == 0) ? std::ldexp(1.0, e / 2) : std::ldexp(std::sqrt(2.0), (e - 1) / 2);
    scale_copy_kernel<<<std::min(ceil_div((long)k * l, 256), 4 * kNumSMs), 256, 0, st>>>((long long)k * l,
                                                                                        omega[mu - 1], sc, T);
    TTK_CHECK_LAUNCH();
    TTK_TRY(jacobi_svd(k, l, T, U[mu], S[mu], V[mu], st));
    recover_halves_kernel<<<1, 256, 0, st>>>(k, l, U[mu], S[mu], V[mu], rcond, unscale, LH[mu], RH[mu], kept + mu);
    TTK_CHECK_LAUNCH();
  }
  std::vector<int> hk(d + 1, 1);
  if (d > 1) {
    TTK_CHECK_CUDA(cudaMemcpyAsync(hk.data() + 1, kept + 1, sizeof(int) * (d - 1), cudaMemcpyDeviceToHost, st));
    TTK_SYNC(st);
  }
  hk[0] = 1;
  hk[d] = 1;
  // cores: LH[mu] (c_{mu} x l_mu) x_1 Psi_mu (l_mu, n, r_{mu+1}) x_3 RH[mu+1] (r_{mu+1} x c_{mu+1})
  for (int mu = 0; mu < d; ++mu) {
    const int l = lr[mu], n = dims[mu], r1 = rr[mu + 1];
    const int c0 = hk[mu], c1 = hk[mu + 1];
    const double* blk = psi[mu];
    int rows = l;
    if (mu > 0) {
      GemmProblem p = make_gemm(c0, n * r1, l, LH[mu], l, 1, psi[mu], (long long)n * r1, 1, T,
                                (long long)n * r1, 1);
      TTK_TRY(gemm_group_launch(&p, 1, split_ws, 16u << 20, st));
      blk = T;
      rows = c0;
    }
    if (mu < d - 1) {
      GemmProblem p = make_gemm(rows * n, c1, r1, blk, r1, 1, RH[mu + 1], c1, 1, out[mu], c1, 1);
      TTK_TRY(gemm_group_launch(&p, 1, split_ws, 16u << 20, st));
    } else {
      TTK_CHECK_CUDA(cudaMemcpyAsync(out[mu], blk, sizeof(double) * (size_t)rows * n * r1,
                                     cudaMemcpyDeviceToDevice, st));
    }
  }
  for (int k = 0; k <= d; ++k) out_ranks[k] = hk[k];
  return kOk;
}

}  // extern "C"
