// Tall-skinny Householder QR (TSQR) and one-sided Jacobi SVD for the
// rounding sweeps.  Replaces np.linalg.qr / np.linalg.svd (LAPACK) at the
// reference call sites tt.py:330, tt.py:361, streaming.py:187.
#pragma once
#include "common.cuh"

namespace ttk {

// Largest column count handled by the register-resident panel kernels.
constexpr int kQrMaxCols = 160;

struct QrPlan {
  int m, l, k;       // k = min(m, l) columns of Q / rows of R
  int cpw, rpl, h;   // panel config (h = 32 * rpl rows per panel)
  int levels;
  int rows[16];      // rows of the level-i input
  int panels[16];
  // tree mode (H < 2l): one leaf level, then a binary tree of triangle pairs
  int tree;
  int depth;
  int nodes[24];     // nodes per tree level (nodes[0] = leaf panels)
  size_t ws_bytes;
};

int qr_plan(int m, int l, QrPlan* plan);

// Householder TSQR of A (m x l), A(i,j) = A[i*a_rs + j*a_cs].  Writes the
// explicit Q (m x k) to Q(i,j) = Q[i*q_rs + j*q_cs] and, when R != nullptr,
// the upper-trapezoidal R (k x l, row-major, ldr = l).  Q may alias nothing
// of A.  Sign convention: Householder reflectors as LAPACK dgeqrf (R is
// unique up to the signs of its rows, Q up to the signs of its columns).
int tsqr(int m, int l, const double* A, long long a_rs, long long a_cs, double* Q, long long q_rs,
         long long q_cs, double* R, void* ws, size_t ws_bytes, cudaStream_t st);
size_t tsqr_ws_bytes(int m, int l);

// QR front door: CholeskyQR2 (GEMM-based) when it is accepted, else Householder TSQR
// hint (in/out, optional): 1 = the previous factorisation of this sweep needed
// the rank-robust path, try it first (one fast-path attempt and host sync less)
int qr_auto(int m, int l, const double* A, long long a_rs, long long a_cs, double* Q, long long q_rs,
            long long q_cs, double* R, void* ws, size_t ws_bytes, cudaStream_t st, int* hint = nullptr,
            int* defer_status = nullptr, int* fused_ok = nullptr);
size_t qr_auto_ws_bytes(int m, int l);

// One-sided (Hestenes) Jacobi SVD of B (k x l, row-major, ldb = l), k, l <= kWideMaxCols:
// B V = U S.  Outputs, columns sorted by decreasing singular value:
//   S[min(k,l)], U (k x min(k,l), row-major, ld = min(k,l)), and optionally
//   V (l x min(k,l), row-major) when V != nullptr (needs l*l + k*l <= 26624 doubles).
// Columns with zero norm give zero singular vectors.
int jacobi_svd(int k, int l, const double* B, double* U, double* S, double* V, cudaStream_t st);
// general form: B(i,j) = B[i*b_rs + j*b_cs]; scaled_u returns U*S (the rotated
// columns) instead of U
int jacobi_svd_ex(int k, int l, const double* B, long long b_rs, long long b_cs, double* U, double* S,
                  double* V, bool scaled_u, cudaStream_t st);
// whether the V-accumulating variant fits in shared memory
bool jacobi_fits_v(int k, int l);

// Above kQrMaxCols columns (qr_wide.cu): column-blocked QR (BCGS2 over <= 96-column
// panels factored by qr_auto) and the grid-cooperative one-sided Jacobi SVD.
constexpr int kWideMaxCols = 4096;
int qr_blocked(int m, int l, const double* A, long long a_rs, long long a_cs, double* Q, long long q_rs,
               long long q_cs, double* R, void* ws, size_t ws_bytes, cudaStream_t st);
size_t qr_blocked_ws_bytes(int m, int l);
int jacobi_svd_global(int k, int l, const double* B, long long b_rs, long long b_cs, double* U, double* S,
                      double* V, bool scaled_u, double skip2, cudaStream_t st);
// Y(i,j) = X(i,j) for an m x l strided block
int copy_strided(int m, int l, const double* X, long long x_rs, long long x_cs, double* Y, long long y_rs,
                 long long y_cs, cudaStream_t st);

// Cholesky factor R (upper, l x l row-major) of G (+ shift_rel * trace), optional
// R^{-1}; status bit set on a non-positive or tiny pivot (qr.cu)
int launch_chol_inv(int l, const double* G, double* R, double* Rinv, int* status, int check_identity,
                    double shift_rel, double tiny_rel, cudaStream_t st, int* near_id_flag);
constexpr int kCholBlockedMaxCols = 112;

// gap-certified dominant-subspace factor of the exact-rank truncation (qr.cu):
// F (l x r) and M^T (l x r), row stride ldo; *flag = 1 when certified
bool trunc_subspace_fits(int l, int r);
// G = C C^T for a wide row-major C (l x m): staged-slab partials + fixed-order reduce
bool gram_wide_fits(int l, long long m, size_t ws_bytes);
int gram_wide(int l, long long m, const double* C, double* G, void* ws, cudaStream_t st);
int launch_trunc_subspace(int l, int r, const double* G, double* F, double* Mt, int ldo, int* flag, double* info,
                          cudaStream_t st, long long* prof = nullptr);

// r = max(1, first index with sqrt(sum_{i>=r} S_i^2) <= budget) capped by
// max_rank (<= 0: no cap) and by n; reference _truncation_rank (tt.py:203-211).
int truncation_rank_dev(const double* S, int n, double budget, int max_rank, int* r_dev,
                        cudaStream_t st);

}  // namespace ttk
