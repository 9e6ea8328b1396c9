/*
 * ttk_b200.h -- C ABI of the B200-native (sm_100a, fp64) TT-sGMRES hot path.
 *
 * Drop-in boundary for the reference package `ttkrylov` (arXiv 2409.09471
 * companion code, /root/reference/pkg/src/ttkrylov).  The reference has no
 * FFI: its boundary is the module-level Python API over lists of float64
 * C-order cores (ttkrylov/__init__.py:3-69).  Each entry point below replaces
 * the arithmetic of one reference function; the Python mirror in
 * paper_2409_09471_b200/ binds them with ctypes.
 *
 * Conventions
 *  - all double pointers are DEVICE pointers to fp64 C-order cores:
 *      TT vector core k   : (r[k], n[k], r[k+1])         r[0] = r[d] = 1
 *      TT operator core k : (rho[k], m[k], n[k], rho[k+1]) rho[0] = rho[d] = 1
 *  - shape/rank arrays and pointer arrays are HOST arrays;
 *  - `stream` is a cudaStream_t (NULL = legacy default stream); all work is
 *    stream-ordered; functions that return host-side results (ranks,
 *    scalars) synchronise the stream before returning;
 *  - `ws`/`ws_bytes` is caller-owned device scratch; size it with the
 *    matching *_ws_bytes query (the library keeps no global device state);
 *  - return 0 on success; nonzero status codes:
 *      1 TTK_SHAPE_MISMATCH  (reference ShapeMismatch, tt.py:22-23)
 *      2 TTK_INVALID_VALUE   (reference ValueError)
 *      3 TTK_CUDA_ERROR
 *      4 TTK_WORKSPACE       (workspace too small)
 *      5 TTK_DEGENERATE      (reference DegenerateRecovery, streaming.py:20-21)
 *    ttk_last_error() returns the message of the last failure on this thread.
 */
#ifndef TTK_B200_H_
#define TTK_B200_H_

#include <stddef.h>

#define TTK_ABI_VERSION 1

#define TTK_OK 0
#define TTK_SHAPE_MISMATCH 1
#define TTK_INVALID_VALUE 2
#define TTK_CUDA_ERROR 3
#define TTK_WORKSPACE 4
#define TTK_DEGENERATE 5

#ifdef __cplusplus
extern "C" {
#endif

/* ---- library ------------------------------------------------------------ */
const char* ttk_last_error(void);
int ttk_version(void);
int ttk_device_arch(void); /* compute capability of the current device, e.g. 100 */
long long ttk_launch_count(void); /* kernels launched by this library so far (all threads) */

/* ---- dense building block ------------------------------------------------
 * Strided batched fp64 GEMM on the DMMA tensor pipe:
 *   C_b(m,n) = alpha * sum_k A_b(m,k) B_b(k,n) + beta * C_b(m,n)
 *   A_b(m,k) = A[b*a_bs + m*a_ms + k*a_ks], B_b(k,n) = B[b*b_bs + k*b_ks + n*b_ns],
 *   C_b(m,n) = C[b*c_bs + m*c_ms + n*c_ns].
 * Replaces the np.tensordot / einsum contractions of the reference
 * (tt.py:292-293,311,333,367; streaming.py:131,136,139). */
int ttk_gemm_strided(int batch, int M, int N, int K, double alpha, const double* A,
                     long long a_ms, long long a_ks, long long a_bs, const double* B,
                     long long b_ks, long long b_ns, long long b_bs, double beta, double* C,
                     long long c_ms, long long c_ns, long long c_bs, void* ws, size_t ws_bytes,
                     void* stream);
size_t ttk_gemm_strided_ws_bytes(int batch, int M, int N, int K);

/* ---- tt_matvec (reference tt.py:302-314) -----------------------------------
 * G_k[(a*rho[k]+al), i, (b*rho[k+1]+be)] = sum_j D_k[al,i,j,be] * C_k[a,j,b]
 * One grouped launch over all d cores; G_k must hold r[k]*rho[k]*m[k]*r[k+1]*rho[k+1]. */
int ttk_matvec(int d, const int* rho, const int* m, const int* n, const int* r,
               const double* const* D, const double* const* C, double* const* G, void* stream);
/* cores k0 <= k < k1 only (shapes are those of the full TT): lets a caller
 * contract cores as their uploads land (tt_matvec_round_rto pipeline) */
int ttk_matvec_range(int d, const int* rho, const int* m, const int* n, const int* r,
                     const double* const* D, const double* const* C, double* const* G, int k0, int k1,
                     void* stream);

/* ---- structure-aware tt_matvec (reference tt.py:302-314) --
 * Same result and output layout as ttk_matvec for square operator cores whose
 * blocks D_k[al, :, :, be] have half-bandwidth <= w (w in 0..2: zero / scaled
 * identity / tridiagonal / pentadiagonal blocks).  band[k] holds
 * band_k[((al*rho[k+1]+be)*n[k] + i)*(2w+1) + t] = D_k[al, i, i+t-w, be] (zero
 * outside the matrix).  kinds (host, optional): per core rho[k]*rho[k+1] bytes
 * (concatenated over k), 0 = zero block, 1 = diagonal block (only t = w
 * nonzero), 2 = banded; NULL treats every block as banded.  An HBM write
 * stream instead of a DMMA contraction. */
int ttk_matvec_banded(int d, const int* rho, const int* n, const int* r, int w, const double* const* band,
                      const unsigned char* kinds, const double* const* C, double* const* G, void* stream);

/* ---- mode_multiply (reference precond.py:189-200, exp-sum terms :266-273) --
 * For each of nterms matrix lists sharing one TT X (ranks r[0..d], mode sizes
 * n[k]): O_{t,k}[a, i, b] = s * sum_j M_{t,k}[i, j] * X_k[a, j, b], with
 * s = alpha[t] on the last core (tt_scale convention) and 1 elsewhere
 * (alpha NULL: all 1).  mats[t*d+k]: m[k] x n[k] row-major; out[t*d+k]:
 * (r[k], m[k], r[k+1]).  Ranks are unchanged.  One grouped DMMA launch (per
 * 96 products). */
int ttk_mode_multiply(int nterms, int d, const int* n, const int* m, const int* r, const double* alpha,
                      const double* const* mats, const double* const* X, double* const* out,
                      void* stream);

/* ---- TT-axpy / concatenation (reference tt_add + tt_scale, tt.py:254-282) --
 * out = sum_t coeff[t] * term_t as ONE block-diagonal concatenation: first core
 * concatenated along axis 2, last along axis 0 (scaled by coeff[t], the factor
 * the reference's tt_scale puts in the last core), interior cores block
 * diagonal; d == 1 sums entrywise.  Equal to the explicit Arnoldi update
 * tt_add(vt, tt_scale(v_i, -h_i)) chained left to right (solvers.py:361-366).
 * ranks: nterms x (d+1); in: nterms x d (term-major); out: d, preallocated with
 * ranks (1, sum_t r_t[1], ..., sum_t r_t[d-1], 1).  nterms <= 16, d <= 64. */
int ttk_tt_concat(int d, int nterms, const double* coeff, const int* dims, const int* ranks,
                  const double* const* in, double* const* out, void* stream);
/* y[i] = alpha * x[i] (last-core scaling of tt_scale, tt.py:278-282) */
int ttk_scale(double* y, const double* x, long long n, double alpha, void* stream);
/* out_dev[0] = sum x[i]^2, fixed reduction order; ws >= 2048 bytes */
int ttk_sumsq(const double* x, long long n, double* out_dev, void* ws, size_t ws_bytes,
              void* stream);

/* ---- tt_dot (reference tt.py:285-294), batched over p partners -----------
 * out_dev[i] = <x, y_i>, left-to-right interface sweep, grouped DMMA GEMMs
 * per core.  xr: d+1 ranks of x; yr: p x (d+1); y: p x d pointers. */
int ttk_tt_dots(int d, const int* dims, const int* xr, const double* const* x, int p,
                const int* yr, const double* const* y, double* out_dev, void* ws, size_t ws_bytes,
                void* stream);
size_t ttk_tt_dots_ws_bytes(int d, const int* dims, const int* xr, int p, const int* yr);

/* ---- Khatri-Rao sketch (reference kr_apply, sketch.py:50-70) ---------------
 * out[v, j - s_lo] = (row j of the Khatri-Rao product of F_1..F_d) . vec(x_v)
 * for rows j in [s_lo, s_hi) and nvec TT vectors x_v (row-shardable: every GPU
 * passes its own [s_lo, s_hi)).  F: d pointers to the full (s x n_k)
 * row-major factors; ranks: nvec x (d+1); cores: nvec x d; out row-major
 * nvec x (s_hi - s_lo). */
int ttk_kr_sketch(int d, const int* n, int s_lo, int s_hi, const double* const* F, int nvec,
                  const int* ranks, const double* const* cores, double* out, void* ws,
                  size_t ws_bytes, void* stream);
size_t ttk_kr_sketch_ws_bytes(int d, const int* n, int s_lo, int s_hi, int nvec, const int* ranks);
/* fused matvec -> sketch: out[j] = KR row j . vec(A x), A x
 * never materialised.  Ft[k]: the operator-premultiplied factors
 * Ft_k[j, al, i', be] = sum_i F_k[j, i] D_k[al, i, i', be]  (S x rho[k] x n[k] x
 * rho[k+1], row-major; built once per (sketch, operator) pair, e.g. with
 * ttk_gemm_strided); C: d cores of x with ranks r; out: S values. */
int ttk_kr_sketch_matvec(int d, const int* n, int S, const double* const* Ft, const int* rho, const int* r,
                         const double* const* C, double* out, void* ws, size_t ws_bytes, void* stream);
size_t ttk_kr_sketch_matvec_ws_bytes(int d, int S, const int* rho, const int* r);
/* same, forcing the fused (path 0) or two-phase (path 1) kernel; for tests */
int ttk_kr_sketch_path(int path, int d, const int* n, int s_lo, int s_hi, const double* const* F,
                       int nvec, const int* ranks, const double* const* cores, double* out,
                       void* ws, size_t ws_bytes, void* stream);

/* ---- dense factorisations (replace np.linalg.qr/svd at tt.py:330,361) ------
 * Householder TSQR of A (m x l), A(i,j) = A[i*a_rs + j*a_cs]: explicit Q (m x k,
 * k = min(m,l)) at Q[i*q_rs + j*q_cs] and, if R != NULL, R (k x l, row-major).
 * Multi-panel inputs (m above one shared-memory panel) need l <= 112. */
int ttk_qr(int m, int l, const double* A, long long a_rs, long long a_cs, double* Q, long long q_rs,
           long long q_cs, double* R, void* ws, size_t ws_bytes, void* stream);
size_t ttk_qr_ws_bytes(int m, int l);
/* the rounding drivers' QR: shifted CholeskyQR2/3 (GEMM-based, accepted only if the
 * Gram of the computed Q is within 1e-3 of I before the last pass), Householder
 * TSQR otherwise (exactly rank-deficient inputs).  Same contract as ttk_qr;
 * synchronises `stream` for the acceptance test. */
int ttk_qr_auto(int m, int l, const double* A, long long a_rs, long long a_cs, double* Q, long long q_rs,
                long long q_cs, double* R, void* ws, size_t ws_bytes, void* stream);
/* one-sided Jacobi SVD of B (k x l, row-major, k,l <= 128): B V = U S with
 * S[min(k,l)] descending, U (k x min(k,l)), V (l x min(k,l)) if V != NULL. */
int ttk_svd_small(int k, int l, const double* B, double* U, double* S, double* V, void* stream);
/* C = alpha A B + beta C for row-major fp64 A (M x K, lda), B (K x N, ldb), C (M x N,
 * ldc) on the TMA-staged DMMA kernel (cp.async.bulk.tensor tiles with the 128-byte
 * swizzle, mbarrier ring): the plain skinny contractions of the RTO sweeps
 * (tt.py's tensordot chains restated in oracle/ttoracle.py rto_sweeps).
 * Requires 16-byte aligned bases, even leading dimensions and K >= 16. */
int ttk_gemm_tma(int M, int N, int K, double alpha, const double* A, long long lda, const double* B, long long ldb,
                 double beta, double* C, long long ldc, void* stream);
/* general strided form: A(m,k) = A[m*a_ms + k*a_ks], B(k,n) = B[k*b_ks + n*b_ns],
 * C(m,n) = C[m*c_ms + n*c_ns] with row-major operands or transposes of row-major
 * operands (a column-major C is computed as the transposed problem); K is split
 * over ws (ws_bytes) when the output tiles leave SMs idle.  Returns
 * TTK_INVALID_VALUE without launching when the operands do not fit TMA. */
int ttk_gemm_tma_strided(int M, int N, int K, double alpha, const double* A, long long a_ms, long long a_ks,
                         const double* B, long long b_ks, long long b_ns, double beta, double* C, long long c_ms,
                         long long c_ns, void* ws, size_t ws_bytes, void* stream);
/* Process-wide switch of the TMA-staged GEMM inside the rounding sweeps (default 1); returns the
 * previous setting.  Independent problems kept in flight on several streams must run with it off
 * (the library also drops to the cp.async kernel while it sees two caller streams active within
 * 0.5 s of each other); DESIGN.md 6.2. */
int ttk_gemm_tma_enable(int on);
/* diagnostics: a shared-memory-holding neighbour kernel for overlap experiments:
 * blocks x threads, smem_bytes dynamic shared memory filled from src (4096 doubles; mode & 1:
 * through cp.async), re-read for `spin` clocks, corrupted words counted into *bad */
int ttk_debug_occupy(int blocks, int threads, int smem_bytes, long long spin, int mode, const double* src, int* bad,
                     void* stream);
/* diagnostics: subsequent Jacobi SVDs store their sweep count in *dev_counter (NULL: off) */
int ttk_debug_svd_sweeps(int* dev_counter);
/* diagnostics: the cluster Jacobi adds per-CTA phase clocks (rotate, send, wait,
 * pull, rounds; 5 int64 per CTA, 8 CTAs) into dev_acc (NULL: off) */
int ttk_debug_jacobi_profile(long long* dev_acc);
/* diagnostics: the blocked Cholesky adds per-call phase clocks (load, diagonal
 * blocks, panels, trailing updates, epilogue, call count) into dev_acc[6] (NULL: off) */
/* diagnostics: one blocked Cholesky R^T R = G (l x l, device; status: device int) */
int ttk_debug_chol(int l, const double* G, double* R, int* status, void* stream);
int ttk_debug_chol_profile(long long* dev_acc);
/* diagnostics: one gap-certified subspace factorisation (truncation, DESIGN 2.2) of the l x l Gram G
 * for rank r: F, Mt (l x r, row stride l), flag (1 = certified), info[3] = {angle bound, tau / lmin,
 * iterations}; prof[5] (or NULL) accumulates phase clocks */
int ttk_debug_trunc_subspace(int l, int r, const double* G, double* F, double* Mt, int* flag, double* info,
                             long long* prof, void* stream);
/* diagnostics: phase timestamps (%globaltimer, ns) of the fused CholeskyQR2 kernel into dev_ts[16]; NULL = off */
int ttk_debug_fused_qr_profile(long long* dev_ts);
/* diagnostics: host synchronisation points (rank / path decisions) so far:
 * out[0] = count, out[1] = total wait in ns (timed only when TTK_HOST_PROF is set) */
int ttk_debug_host_profile(long long* out);

/* ---- tt_round, TT-SVD (reference tt.py:337-368) ----------------------------
 * out[k] holds ranks[k]*dims[k]*ranks[k+1] doubles; out_ranks (host, d+1)
 * receives the result ranks and core k fills the first
 * out_ranks[k]*dims[k]*out_ranks[k+1] entries of out[k].  max_rank <= 0: no
 * cap; zero_rel < 0: no cancellation test (reference tt.py:348-356, quirk Q1).
 * Synchronises `stream` (rank decisions are read back per core). */
int ttk_tt_round(int d, const int* dims, const int* ranks, const double* const* cores,
                 double rel_tol, int max_rank, double zero_rel, double* const* out, int* out_ranks,
                 void* ws, size_t ws_bytes, void* stream);
size_t ttk_tt_round_ws_bytes(int d, const int* dims, const int* ranks);

/* ---- randomize-then-orthogonalize sweeps (absent from the reference,
 * SPEC.md:313; restated in oracle/ttoracle.py rto_sweeps) --------------------
 * X: cores (R[k], n_k, R[k+1]); G: Gaussian TT-DRM cores (L[k], n_k, L[k+1])
 * (reference tt_drm_new, streaming.py:38-53) with L[c] <= min(R[c],
 * L[c-1] n_{c-1}); out: cores (L[k], n_k, L[k+1]), cores 0..d-2 left-orthonormal. */
int ttk_rto_sweeps(int d, const int* dims, const int* R, const double* const* X, const int* L,
                   const double* const* G, double* const* out, void* ws, size_t ws_bytes, void* stream);
/* same, with ready[k] (cudaEvent_t, entries may be NULL) awaited on `stream`
 * before core X[k] is first read: the right sweep starts on the last cores
 * while earlier ones are still being produced */
int ttk_rto_sweeps_ev(int d, const int* dims, const int* R, const double* const* X, const int* L,
                      const double* const* G, double* const* out, void* ws, size_t ws_bytes,
                      void* const* ready, void* stream);
size_t ttk_rto_ws_bytes(int d, const int* dims, const int* R, const int* L);

/* ---- TT containers (reference save_/load_vector, save_/load_operator,
 * tt.py:451-520): magic "TTKVEC01" / "TTKOPR01", int64 LE header
 * (vector: d, dims[d], ranks[d+1]; operator: d, row_dims[d], col_dims[d],
 * ranks[d+1]), then row-major float64 LE cores.  Device transfers are staged
 * through two pinned buffers (file I/O overlaps the copies).
 * Errors: 2 (ValueError) for a bad magic, truncated file or bad header. */
/* kind: 0 vector, 1 operator; header[0..] as laid out in the file (incl. d) */
int ttk_io_read_header(const char* path, int* kind, int* d, long long* header, int cap);
/* cores: d pointers (host if !to_device) sized from the header */
int ttk_io_read_cores(const char* path, int to_device, double* const* cores, void* stream);
int ttk_io_write(const char* path, int kind, int d, const long long* header, int from_device,
                 const double* const* cores, void* stream);

/* ---- counter-based Gaussian TT-DRM (the solver's randomized-rounding sketch;
 * no reference counterpart, SPEC.md:313 -- replaces the host draw of
 * streaming.py:38-53 for that one use).  Writes the leading r0 x n x r1 block of
 * core `core` of a Gaussian TT with full ranks (r0_full, r1_full): entry
 * (i, j, l) = scale * N(Philox4x32-10(seed; ((core*r0_full + i)*n + j)*r1_full + l)),
 * so every leading block equals the same block of the full map.
 * out: device, r0 x n x r1 row-major.  Stream-ordered. */
int ttk_drm_gaussian(unsigned long long seed, int core, int n, int r0_full, int r1_full, int r0, int r1,
                     double scale, double* out, void* stream);

/* ---- streaming sketches (reference streaming.py:117-205) -------------------
 * stream_sketch: psi[mu] ((lr[mu] n_mu) x rr[mu+1]) and omega[mu-1]
 * (lr[mu] x rr[mu]) of a TT with ranks tr against the frame's left (Y, ranks
 * lr) and right (X, ranks rr) TT-DRMs. */
int ttk_stream_sketch(int d, const int* dims, const int* tr, const double* const* C, const int* lr,
                      const double* const* Y, const int* rr, const double* const* X,
                      double* const* psi, double* const* omega, void* ws, size_t ws_bytes,
                      void* stream);
size_t ttk_stream_sketch_ws_bytes(int d, const int* dims, const int* tr, const int* lr, const int* rr);
/* combine_pairs kernel: out = sum_t coeff[t] in_t, left-to-right (streaming.py:145-163) */
int ttk_axpy_multi(int nterms, const double* coeff, const double* const* in, long long n, double* out,
                   void* stream);
/* stream_recover up to its final tt_round: truncated-SVD pseudo-inverse halves
 * of every Omega (relative cutoff rcond) applied to the Psi blocks; writes the
 * recovered cores (capacity max(lr,rr)*n*rr[mu+1]) and their ranks (host).
 * *is_zero = 1 when every Psi is zero; TTK_DEGENERATE on a zero Omega. */
int ttk_stream_recover_cores(int d, const int* dims, const int* lr, const int* rr,
                             const double* const* psi, const double* const* omega, double rcond,
                             double* const* out, int* out_ranks, int* is_zero, void* ws,
                             size_t ws_bytes, void* stream);
size_t ttk_stream_recover_ws_bytes(int d, const int* dims, const int* lr, const int* rr);

/* ---- truncation of a LEFT-orthogonal TT (the RTO output), right to left ------
 * TT-SVD without an orthogonalisation sweep; same budget rule
 * rel_tol*||v||/sqrt(d-1) and cap as tt_round (tt.py:357-364); output layout as
 * ttk_tt_round.  Oracle: oracle/ttoracle.py truncate_left_orth.  Synchronises.
 * Exact-rank roundings (rel_tol == 0) factor each unfolding through its Gram
 * matrix (Cholesky, then the Jacobi SVD of R) when the kept singular values
 * are >= sqrt(1e-3) of the largest; otherwise (and for rel_tol > 0) through
 * the QR of C_k^T, as np.linalg.svd at tt.py:361. */
int ttk_tt_truncate(int d, const int* dims, const int* ranks, const double* const* cores, double rel_tol,
                    int max_rank, double* const* out, int* out_ranks, void* ws, size_t ws_bytes,
                    void* stream);
/* same, and every result core is also copied to host_out[k] (pinned host
 * memory, room for ranks[k]*dims[k]*ranks[k+1] doubles) as soon as it is
 * final, overlapping the copies with the rest of the sweep; returns after all
 * copies completed */
int ttk_tt_truncate_host(int d, const int* dims, const int* ranks, const double* const* cores, double rel_tol,
                         int max_rank, double* const* out, int* out_ranks, double* const* host_out, void* ws,
                         size_t ws_bytes, void* stream);
/* diagnostics: cores truncated so far through the Gram path [0] and the QR path [1], and
 * truncations redone through the QR path after a failed Gram certificate [2] */
int ttk_debug_truncate_paths(long long* counts);
/* the same plus [3] cores factored by the gap-certified subspace kernel and [4] truncations
 * redone through the Jacobi Gram path after a failed subspace certificate, [5] RTO left sweeps
 * accepted with the deferred CholeskyQR2 check, [6] RTO left sweeps redone with the per-core
 * check; writes min(n, 7) */
int ttk_debug_truncate_paths_ex(long long* counts, int n);
size_t ttk_tt_truncate_ws_bytes(int d, const int* dims, const int* ranks);

#ifdef __cplusplus
}
#endif

#endif /* TTK_B200_H_ */
