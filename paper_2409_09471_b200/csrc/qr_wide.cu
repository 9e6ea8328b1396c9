// Factorisations for rank profiles above the register-resident kernels'
// kQrMaxCols (160) columns -- the reference rounds at any rank through LAPACK
// (tt.py:330 np.linalg.qr, tt.py:361 np.linalg.svd), e.g. BASELINE config 2
// (rank 200) and config 3 (rank 192) under TT-SVD rounding:
//
//  * qr_blocked: column-blocked QR.  Panels of <= 96 columns; each panel is
//    projected against the Q columns already formed twice (block classical
//    Gram-Schmidt with re-orthogonalisation, BCGS2: two GEMM pairs per panel),
//    factored by qr_auto (CholeskyQR2 / rank-robust CholeskyQR3 / Householder
//    TSQR), and its unit-norm Q block projected and re-factored once more
//    (an ill-conditioned panel amplifies the projection residual by kappa).  Wide inputs (m < l) factor the leading m columns and
//    form R's trailing columns as Q^T A.
//  * jacobi_svd_global: one-sided (Hestenes) Jacobi with the columns in global
//    memory (L2-resident: 200 x 200 fp64 is 320 KB), one warp per column pair,
//    the round-robin pairing computed from the round index (no data moves),
//    one grid-wide barrier per round in a single cooperative launch.
#include <cooperative_groups.h>

#include "gemm.cuh"
#include "qr.cuh"

#include <algorithm>
#include <cmath>

namespace cg = cooperative_groups;

namespace ttk {

namespace {

constexpr int kWidePanel = 96;     // <= the fused CholeskyQR2's column limit
constexpr int kJgThreads = 256;    // 8 warps per CTA
constexpr int kJgMaxSweeps = 40;
constexpr size_t kWideSplitBytes = 32u << 20;

__global__ void add_block_kernel(int rows, int cols, const double* __restrict__ X, long long x_rs, double* Y,
                                 long long y_rs, int accumulate) {
  const long long n = (long long)rows * cols;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int r = (int)(e / cols), c = (int)(e % cols);
    const double v = X[r * x_rs + c];
    Y[r * y_rs + c] = accumulate ? Y[r * y_rs + c] + v : v;
  }
}

// Columns of a projected unit-norm block that vanished (they lay in the span
// of the Q columns already formed: completion directions of a rank-deficient
// panel) are refilled with a deterministic pseudo-random vector; they carry an
// O(eps) weight in R, so the factorisation stays backward stable, and the next
// projection + QR makes them orthonormal to everything before.
__global__ void refill_vanished_kernel(int m, double* X, long long x_rs, long long x_cs, unsigned long long seed) {
  __shared__ double red[32];
  __shared__ int vanished;
  double* x = X + blockIdx.x * x_cs;
  double s = 0.0;
  for (int i = threadIdx.x; i < m; i += blockDim.x) s = fma(x[i * x_rs], x[i * x_rs], s);
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += red[w];
    vanished = t < 1e-16;
  }
  __syncthreads();
  if (!vanished) return;
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    unsigned long long z = ((unsigned long long)i + 1) * 0x9E3779B97F4A7C15ull + seed * 0xD1B54A32D192ED03ull +
                           blockIdx.x;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    x[i * x_rs] = ((double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0) / sqrt((double)m);
  }
}

inline int grid_for(long long n) { return (int)std::max(1LL, std::min<long long>((n + 255) / 256, 4 * kNumSMs)); }

}  // namespace

size_t qr_blocked_ws_bytes(int m, int l) {
  const int k = std::min(m, l);
  const int np = (k + kWidePanel - 1) / kWidePanel;
  const int w = (k + np - 1) / np;
  return align_up((size_t)m * w * 8, 256) + 2 * align_up((size_t)k * w * 8, 256) + 2 * align_up((size_t)w * w * 8, 256) +
         kWideSplitBytes + qr_auto_ws_bytes(m, w) + 4096;
}

int qr_blocked(int m, int l, const double* A, long long a_rs, long long a_cs, double* Q, long long q_rs,
               long long q_cs, double* R, void* ws, size_t ws_bytes, cudaStream_t st) {
  const int k = std::min(m, l);
  const int np = (k + kWidePanel - 1) / kWidePanel;
  const int w = (k + np - 1) / np;
  TTK_REQUIRE((const void*)A != (const void*)Q || (a_rs == q_rs && a_cs == q_cs), kInvalidValue,
              "qr_blocked: an in-place call needs equal strides");
  TTK_REQUIRE(ws != nullptr && ws_bytes >= qr_blocked_ws_bytes(m, l), kWorkspace,
              "qr_blocked: workspace %zu < %zu", ws_bytes, qr_blocked_ws_bytes(m, l));
  Arena ar(ws, ws_bytes);
  double* P = ar.take<double>((size_t)m * w);      // panel, row-major (m x w)
  double* C = ar.take<double>((size_t)k * w);      // projection coefficients (c0 x w)
  double* C2 = ar.take<double>((size_t)k * w);
  double* Rp = ar.take<double>((size_t)w * w);     // panel R
  double* R2 = ar.take<double>((size_t)w * w);     // re-factorisation R
  void* split = ar.take<char>(kWideSplitBytes);
  const size_t used = align_up(ar.used, 256);
  void* qws = (char*)ws + used;
  const size_t qbytes = ws_bytes - used;
  if (R) TTK_CHECK_CUDA(cudaMemsetAsync(R, 0, sizeof(double) * (size_t)k * l, st));
  GemmProblem g;
  for (int c0 = 0; c0 < k; c0 += w) {
    const int wj = std::min(w, k - c0);
    // P = A[:, c0:c0+wj]
    TTK_TRY(copy_strided(m, wj, A + (long long)c0 * a_cs, a_rs, a_cs, P, wj, 1, st));
    for (int pass = 0; pass < 2 && c0 > 0; ++pass) {
      // C = Q[:, :c0]^T P ;  P -= Q[:, :c0] C ;  R[:c0, c0:c0+wj] += C
      g = make_gemm(c0, wj, m, Q, q_cs, q_rs, P, wj, 1, C, wj, 1);
      TTK_TRY(gemm_group_launch(&g, 1, split, kWideSplitBytes, st));
      g = make_gemm(m, wj, c0, Q, q_rs, q_cs, C, wj, 1, P, wj, 1, -1.0, 1.0);
      TTK_TRY(gemm_group_launch(&g, 1, split, kWideSplitBytes, st));
      if (R) {
        add_block_kernel<<<grid_for((long long)c0 * wj), 256, 0, st>>>(c0, wj, C, wj, R + c0, l, pass);
        TTK_CHECK_LAUNCH();
      }
    }
    double* Qj = Q + (long long)c0 * q_cs;
    TTK_TRY(qr_auto(m, wj, P, wj, 1, Qj, q_rs, q_cs, Rp, qws, qbytes, st));
    if (c0 > 0) {
      // Q_j = P R_jj^{-1} amplifies P's O(eps |A_j|) residual along Q[:, :c0] by
      // kappa(P) (graded inputs: 1e-10 instead of 1e-16): project the unit-norm
      // Q_j once more and re-factor the now well-conditioned block,
      //   Q_j = Q C2 + Q_j' R2  ->  R[:c0, j] += C2 R_jj,  R_jj <- R2 R_jj
      g = make_gemm(c0, wj, m, Q, q_cs, q_rs, Qj, q_rs, q_cs, C, wj, 1);
      TTK_TRY(gemm_group_launch(&g, 1, split, kWideSplitBytes, st));
      g = make_gemm(m, wj, c0, Q, q_rs, q_cs, C, wj, 1, Qj, q_rs, q_cs, -1.0, 1.0);
      TTK_TRY(gemm_group_launch(&g, 1, split, kWideSplitBytes, st));
      refill_vanished_kernel<<<wj, 256, 0, st>>>(m, Qj, q_rs, q_cs, (unsigned long long)c0);
      TTK_CHECK_LAUNCH();
      // second projection (C accumulates it: Q_j = Q (C + C') + Q_j'' exactly)
      g = make_gemm(c0, wj, m, Q, q_cs, q_rs, Qj, q_rs, q_cs, C2, wj, 1);
      TTK_TRY(gemm_group_launch(&g, 1, split, kWideSplitBytes, st));
      g = make_gemm(m, wj, c0, Q, q_rs, q_cs, C2, wj, 1, Qj, q_rs, q_cs, -1.0, 1.0);
      TTK_TRY(gemm_group_launch(&g, 1, split, kWideSplitBytes, st));
      add_block_kernel<<<grid_for((long long)c0 * wj), 256, 0, st>>>(c0, wj, C2, wj, C, wj, 1);
      TTK_CHECK_LAUNCH();
      TTK_TRY(copy_strided(m, wj, Qj, q_rs, q_cs, P, wj, 1, st));
      TTK_TRY(qr_auto(m, wj, P, wj, 1, Qj, q_rs, q_cs, R2, qws, qbytes, st));
      if (R) {
        g = make_gemm(c0, wj, wj, C, wj, 1, Rp, wj, 1, R + c0, l, 1, 1.0, 1.0);
        TTK_TRY(gemm_group_launch(&g, 1, split, kWideSplitBytes, st));
        g = make_gemm(wj, wj, wj, R2, wj, 1, Rp, wj, 1, R + (size_t)c0 * l + c0, l, 1);
        TTK_TRY(gemm_group_launch(&g, 1, split, kWideSplitBytes, st));
      }
    } else if (R) {
      add_block_kernel<<<grid_for((long long)wj * wj), 256, 0, st>>>(wj, wj, Rp, wj, R + (size_t)c0 * l + c0, l, 0);
      TTK_CHECK_LAUNCH();
    }
  }
  if (R && l > k) {
    // wide input: R[:, k:] = Q^T A[:, k:]
    g = make_gemm(k, l - k, m, Q, q_cs, q_rs, A + (long long)k * a_cs, a_rs, a_cs, R + k, l, 1);
    TTK_TRY(gemm_group_launch(&g, 1, split, kWideSplitBytes, st));
  }
  // R is block upper triangular (zero below the diagonal panels); a panel's
  // diagonal block is upper triangular unless the panel took the rank-robust
  // path, whose R = Q^T Y is full (qr_auto's contract: A = Q R, Q orthonormal)
  return kOk;
}

// -------------------------------------------------------------------------
// grid-cooperative one-sided Jacobi

struct JgParams {
  int k, l, le;
  const double* B;
  long long b_rs, b_cs;
  double* X;    // le columns of k rows, column j at X + j*k
  double* W;    // le columns of le rows (V), column j at W + j*le
  double* nrm;  // le
  int* order;   // le
  int* flags;   // kJgMaxSweeps
  double* U;
  double* S;
  double* V;
  int want_v, scaled_u;
  double skip2;
};

// round-robin (circle method) pairing of le players in round t: player le-1
// stays, the others rotate; pair q of round t
__device__ __forceinline__ void jg_pair(int t, int q, int le, int& a, int& b) {
  const int n1 = le - 1;
  if (q == 0) {
    a = t;
    b = n1;
  } else {
    a = (t + q) % n1;
    b = (t - q + n1) % n1;
  }
  if (a > b) { const int x = a; a = b; b = x; }
}

__global__ void __launch_bounds__(kJgThreads) jacobi_global_kernel(const JgParams p) {
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int warp = (int)((blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5);
  const int nwarps = (int)((gridDim.x * (long long)blockDim.x) >> 5);
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nth = gridDim.x * (long long)blockDim.x;
  const int k = p.k, l = p.l, le = p.le;
  for (long long e = tid; e < (long long)le * k; e += nth) {
    const int j = (int)(e / k), i = (int)(e % k);
    p.X[e] = j < l ? p.B[i * p.b_rs + j * p.b_cs] : 0.0;
  }
  if (p.want_v)
    for (long long e = tid; e < (long long)le * le; e += nth) p.W[e] = (e / le == e % le) ? 1.0 : 0.0;
  grid.sync();
  const int npairs = le / 2;
  for (int sweep = 0; sweep < kJgMaxSweeps; ++sweep) {
    for (int t = 0; t < le - 1; ++t) {
      for (int q = warp; q < npairs; q += nwarps) {
        int a, b;
        jg_pair(t, q, le, a, b);
        if (b >= l) continue;  // padding column (zero)
        double* xa = p.X + (size_t)a * k;
        double* xb = p.X + (size_t)b * k;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < k; i += 32) {
          const double u = xa[i], v = xb[i];
          al = fma(u, u, al);
          be = fma(v, v, be);
          ga = fma(u, v, ga);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        // rotate unless the pair is orthogonal to working precision
        if (ga == 0.0 || al == 0.0 || be == 0.0 || fabs(ga) <= 1e-17 * sqrt(al) * sqrt(be)) continue;
        if (lane == 0 && ga * ga > p.skip2 * al * be) p.flags[sweep] = 1;
        const double zeta = (be - al) / (2.0 * ga);
        const double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + tt * tt), s = c * tt;
        for (int i = lane; i < k; i += 32) {
          const double u = xa[i], v = xb[i];
          xa[i] = c * u - s * v;
          xb[i] = s * u + c * v;
        }
        if (p.want_v) {
          double* va = p.W + (size_t)a * le;
          double* vb = p.W + (size_t)b * le;
          for (int i = lane; i < l; i += 32) {
            const double u = va[i], v = vb[i];
            va[i] = c * u - s * v;
            vb[i] = s * u + c * v;
          }
        }
      }
      grid.sync();
    }
    // flags[sweep] was written before the last barrier of this sweep
    if (p.flags[sweep] == 0) break;
  }
  // column norms, ordering by decreasing norm (ties by index), outputs
  for (int j = warp; j < le; j += nwarps) {
    const double* x = p.X + (size_t)j * k;
    double s = 0.0;
    for (int i = lane; i < k; i += 32) s = fma(x[i], x[i], s);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) p.nrm[j] = j < l ? sqrt(s) : -1.0;
  }
  grid.sync();
  for (long long j = tid; j < le; j += nth) {
    const double v = p.nrm[j];
    int pos = 0;
    for (int i = 0; i < le; ++i) {
      const double w = p.nrm[i];
      pos += (w > v) || (w == v && i < j);
    }
    p.order[pos] = (int)j;
  }
  grid.sync();
  const int kout = min(k, l);
  for (long long e = tid; e < (long long)kout * k; e += nth) {
    const int r = (int)(e % kout), i = (int)(e / kout);
    const int j = p.order[r];
    const double n = p.nrm[j];
    const double x = p.X[(size_t)j * k + i];
    p.U[(size_t)i * kout + r] = p.scaled_u ? x : (n > 0.0 ? x / n : 0.0);
  }
  for (long long r = tid; r < kout; r += nth) p.S[r] = p.nrm[p.order[r]];
  if (p.want_v && p.V)
    for (long long e = tid; e < (long long)kout * l; e += nth) {
      const int r = (int)(e % kout), i = (int)(e / kout);
      p.V[(size_t)i * kout + r] = p.W[(size_t)p.order[r] * le + i];
    }
}

int jacobi_svd_global(int k, int l, const double* B, long long b_rs, long long b_cs, double* U, double* S,
                      double* V, bool scaled_u, double skip2, cudaStream_t st) {
  const int le = l + (l & 1);
  const size_t xb = align_up((size_t)le * k * 8, 256);
  const size_t wb = V ? align_up((size_t)le * le * 8, 256) : 0;
  const size_t bytes = xb + wb + align_up((size_t)le * 8, 256) + align_up((size_t)le * 4, 256) + 256;
  char* buf = nullptr;
  TTK_TRY(scratch_alloc((void**)&buf, bytes, st));
  JgParams p{};
  p.k = k; p.l = l; p.le = le; p.B = B; p.b_rs = b_rs; p.b_cs = b_cs;
  p.X = (double*)buf;
  p.W = V ? (double*)(buf + xb) : nullptr;
  p.nrm = (double*)(buf + xb + wb);
  p.order = (int*)(buf + xb + wb + align_up((size_t)le * 8, 256));
  p.flags = (int*)(buf + xb + wb + align_up((size_t)le * 8, 256) + align_up((size_t)le * 4, 256));
  p.U = U; p.S = S; p.V = V; p.want_v = V != nullptr; p.scaled_u = scaled_u; p.skip2 = skip2;
  TTK_CHECK_CUDA(cudaMemsetAsync(p.flags, 0, sizeof(int) * kJgMaxSweeps, st));
  int dev = 0, sms = kNumSMs, per_sm = 1;
  TTK_CHECK_CUDA(cudaGetDevice(&dev));
  TTK_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  TTK_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, jacobi_global_kernel, kJgThreads, 0));
  const int want = std::max(1, (le / 2 + (kJgThreads / 32) - 1) / (kJgThreads / 32));
  const int grid = std::max(1, std::min(want, sms * std::max(per_sm, 1)));
  void* args[] = {(void*)&p};
  TTK_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)jacobi_global_kernel, dim3(grid), dim3(kJgThreads), args,
                                             0, st));
  TTK_CHECK_LAUNCH();
  TTK_TRY(scratch_free(buf, st));
  return kOk;
}

}  // namespace ttk
