// Householder TSQR + one-sided Jacobi SVD (see qr.cuh).
//
// TSQR: the m x l input is cut into panels of H rows; one CTA factors a panel
// with Householder reflectors entirely in shared memory (LAPACK dlarfg sign
// convention), keeps the reflectors for the explicit-Q pass and emits its
// l x l R.  The stacked R's form the next level's input until one panel is
// left.  The explicit Q is then formed top-down: every panel applies its
// reflectors (in reverse order) to its l x l block of the level-above Q padded
// with zeros.  Rank-deficient inputs are handled exactly like LAPACK (a zero
// column gives tau = 0 and an identity reflector), so Q is always orthonormal.
#include "qr.cuh"
#include "../../include/ttk_b200.h"

#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace ttk {

constexpr int kQrThreads = 1024;
constexpr int kQrSmemDoubles = 28672;  // 224 KB of shared memory, in doubles

__device__ __forceinline__ int qr_ld(int l) { return l | 1; }  // odd stride: conflict-free columns

// -------------------------------------------------------------------------
// panel factorisation: one CTA per panel
__global__ void __launch_bounds__(kQrThreads, 1)
    qr_panel_factor_kernel(int m, int l, int H, const double* __restrict__ A, long long a_rs,
                           long long a_cs, double* __restrict__ Vt, double* __restrict__ tau,
                           double* __restrict__ Rout) {
  extern __shared__ double sm[];
  const int ld = qr_ld(l);
  double* S = sm;                 // H x ld
  double* vsh = S + (size_t)H * ld;  // 2 x H
  double* tsh = vsh + 2 * H;      // l
  const int p = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const long long row0 = (long long)p * H;

  for (int e = threadIdx.x; e < H * l; e += blockDim.x) {
    int r, c;
    if (a_cs == 1) { r = e / l; c = e - r * l; } else { c = e / H; r = e - c * H; }
    long long gr = row0 + r;
    S[r * ld + c] = (gr < m) ? A[gr * a_rs + (long long)c * a_cs] : 0.0;
  }
  const int kmax = min(l, H);  // reflectors; the rest are identities
  for (int j = kmax + threadIdx.x; j < l; j += blockDim.x) tsh[j] = 0.0;
  __syncthreads();

  for (int j = 0; j < kmax; ++j) {
    double* v = vsh + (j & 1) * H;
    if (warp == 0) {
      // reflector for column j (rows j..H-1); warp 0 also updated this column
      double s2 = 0.0;
      for (int r = j + 1 + lane; r < H; r += 32) {
        double x = S[r * ld + j];
        s2 += x * x;
      }
      s2 = warp_sum(s2);
      const double alpha = S[j * ld + j];
      double t = 0.0, beta = alpha, scal = 0.0;
      if (s2 > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + s2), alpha);
        t = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      for (int r = j + 1 + lane; r < H; r += 32) {
        double x = S[r * ld + j] * scal;
        S[r * ld + j] = x;
        v[r] = x;
      }
      if (lane == 0) {
        S[j * ld + j] = beta;
        v[j] = 1.0;
        tsh[j] = t;
      }
    }
    __syncthreads();
    const double t = tsh[j];
    if (t != 0.0) {
      // columns c > j round-robin over warps; warp 0 always takes column j+1
      for (int c = j + 1 + warp; c < l; c += nwarps) {
        double s = 0.0;
        for (int r = j + lane; r < H; r += 32) s += v[r] * S[r * ld + c];
        s = warp_sum(s) * t;
        for (int r = j + lane; r < H; r += 32) S[r * ld + c] -= v[r] * s;
      }
    }
    // no second barrier: the next reflector is computed by warp 0 from the
    // column it just updated, and the v buffers are double-buffered.
  }
  __syncthreads();
  // R block (rows 0..l-1), reflectors (column-major per panel), tau
  double* Rp = Rout + (long long)p * l * l;
  for (int e = threadIdx.x; e < l * l; e += blockDim.x) {
    int r = e / l, c = e - r * l;
    Rp[e] = (c >= r && r < H) ? S[r * ld + c] : 0.0;
  }
  double* Vp = Vt + (long long)p * l * H;
  for (int e = threadIdx.x; e < l * H; e += blockDim.x) {
    int j = e / H, r = e - j * H;
    Vp[e] = (r > j) ? S[r * ld + j] : (r == j ? 1.0 : 0.0);
  }
  for (int j = threadIdx.x; j < l; j += blockDim.x) tau[(long long)p * l + j] = tsh[j];
}

// -------------------------------------------------------------------------
// explicit Q of one panel: E (H x l) = [Qup block (l x l); 0], E <- H_0 ... H_{l-1} E
__global__ void __launch_bounds__(kQrThreads, 1)
    qr_panel_apply_kernel(int l, int H, int kcols, const double* __restrict__ Vt,
                          const double* __restrict__ tau, const double* __restrict__ Qup,
                          long long m_out, double* __restrict__ Q, long long q_rs, long long q_cs) {
  extern __shared__ double sm[];
  const int ld = qr_ld(l);
  double* E = sm;  // H x ld
  const int p = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  for (int e = threadIdx.x; e < H * l; e += blockDim.x) {
    int r = e / l, c = e - r * l;
    double x = 0.0;
    if (r < l) x = Qup ? Qup[((long long)p * l + r) * l + c] : (r == c ? 1.0 : 0.0);
    // (single-panel wide case H < l: rows >= H do not exist)
    E[r * ld + c] = x;
  }
  __syncthreads();
  const double* Vp = Vt + (long long)p * l * H;
  const double* tp = tau + (long long)p * l;
  for (int j = min(l, H) - 1; j >= 0; --j) {
    const double t = tp[j];
    if (t == 0.0) continue;
    const double* v = Vp + (long long)j * H;
    for (int c = warp; c < l; c += nwarps) {
      double s = 0.0;
      for (int r = j + lane; r < H; r += 32) s += __ldg(v + r) * E[r * ld + c];
      s = warp_sum(s) * t;
      for (int r = j + lane; r < H; r += 32) E[r * ld + c] -= __ldg(v + r) * s;
    }
  }
  __syncthreads();
  const long long row0 = (long long)p * H;
  for (int e = threadIdx.x; e < H * kcols; e += blockDim.x) {
    int r, c;
    if (q_cs == 1) { r = e / kcols; c = e - r * kcols; } else { c = e / H; r = e - c * H; }
    long long gr = row0 + r;
    if (gr < m_out) Q[gr * q_rs + (long long)c * q_cs] = E[r * ld + c];
  }
}

// -------------------------------------------------------------------------
// Tree mode: QR of two stacked upper-triangular l x l factors [R1; R2].
// Reflector j touches row j of R1 and rows 0..j of R2 only, so both stay
// upper triangular; they live packed column-major in shared memory
// (entry (r, c), r <= c, at c(c+1)/2 + r).  The reflector vectors overwrite
// R2 (unit entry at row j of R1 implicit).
__device__ __forceinline__ int pk_idx(int r, int c) { return c * (c + 1) / 2 + r; }

__global__ void __launch_bounds__(kQrThreads, 1)
    qr_pair_factor_kernel(int l, int nchild, const double* __restrict__ Rin, double* __restrict__ Rout,
                          double* __restrict__ Vp, double* __restrict__ tau) {
  extern __shared__ double sm[];
  const size_t pk = (size_t)l * (l + 1) / 2;
  double* T1 = sm;
  double* T2 = sm + pk;
  double* tsh = T2 + pk;
  const int node = blockIdx.x;
  const int a = 2 * node, b = 2 * node + 1;
  const bool pair = b < nchild;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const double* R1 = Rin + (size_t)a * l * l;
  const double* R2 = Rin + (size_t)b * l * l;
  for (int e = threadIdx.x; e < l * l; e += blockDim.x) {
    int r = e / l, c = e - r * l;
    if (r <= c) {
      T1[pk_idx(r, c)] = R1[e];
      T2[pk_idx(r, c)] = pair ? R2[e] : 0.0;
    }
  }
  __syncthreads();
  for (int j = 0; j < l; ++j) {
    if (warp == 0) {
      double s2 = 0.0;
      for (int i = lane; i <= j; i += 32) {
        double x = T2[pk_idx(i, j)];
        s2 += x * x;
      }
      s2 = warp_sum(s2);
      const double alpha = T1[pk_idx(j, j)];
      double t = 0.0, beta = alpha, scal = 0.0;
      if (s2 > 0.0) {
        beta = -copysign(sqrt(alpha * alpha + s2), alpha);
        t = (beta - alpha) / beta;
        scal = 1.0 / (alpha - beta);
      }
      for (int i = lane; i <= j; i += 32) T2[pk_idx(i, j)] *= scal;
      if (lane == 0) {
        T1[pk_idx(j, j)] = beta;
        tsh[j] = t;
      }
    }
    __syncthreads();
    const double t = tsh[j];
    if (t != 0.0) {
      const double* v = T2 + pk_idx(0, j);
      for (int c = j + 1 + warp; c < l; c += nwarps) {
        double* col = T2 + pk_idx(0, c);
        double s = 0.0;
        for (int i = lane; i <= j; i += 32) s += v[i] * col[i];
        s = (warp_sum(s) + T1[pk_idx(j, c)]) * t;
        for (int i = lane; i <= j; i += 32) col[i] -= v[i] * s;
        if (lane == 0) T1[pk_idx(j, c)] -= s;
      }
    }
  }
  __syncthreads();
  double* Ro = Rout + (size_t)node * l * l;
  for (int e = threadIdx.x; e < l * l; e += blockDim.x) {
    int r = e / l, c = e - r * l;
    Ro[e] = (r <= c) ? T1[pk_idx(r, c)] : 0.0;
  }
  double* vo = Vp + (size_t)node * pk;
  for (size_t e = threadIdx.x; e < pk; e += blockDim.x) vo[e] = T2[e];
  for (int j = threadIdx.x; j < l; j += blockDim.x) tau[(size_t)node * l + j] = tsh[j];
}

// E_node (l x l) -> [E_top; E_bot] = H_0..H_{l-1} [E_node; 0]; column chunks of 32.
__global__ void __launch_bounds__(256)
    qr_pair_apply_kernel(int l, int nchild, const double* __restrict__ Vp, const double* __restrict__ tau,
                         const double* __restrict__ Ein, double* __restrict__ Eout) {
  constexpr int CB = 32;
  extern __shared__ double sm[];
  double* Et = sm;            // l x CB
  double* Eb = sm + l * CB;   // l x CB
  const int node = blockIdx.x, c0 = blockIdx.y * CB;
  const int cb = min(CB, l - c0);
  const int a = 2 * node, b = 2 * node + 1;
  const bool pair = b < nchild;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int nwarps = blockDim.x >> 5;
  const double* E = Ein + (size_t)node * l * l;
  for (int e = threadIdx.x; e < l * CB; e += blockDim.x) {
    int r = e / CB, c = e - r * CB;
    Et[e] = (c < cb) ? E[(size_t)r * l + c0 + c] : 0.0;
    Eb[e] = 0.0;
  }
  __syncthreads();
  const size_t pk = (size_t)l * (l + 1) / 2;
  const double* V = Vp + (size_t)node * pk;
  const double* tp = tau + (size_t)node * l;
  if (pair) {
    for (int j = l - 1; j >= 0; --j) {
      const double t = tp[j];
      if (t == 0.0) continue;
      const double* v = V + pk_idx(0, j);
      for (int c = warp; c < cb; c += nwarps) {
        double s = 0.0;
        for (int i = lane; i <= j; i += 32) s += __ldg(v + i) * Eb[i * CB + c];
        s = (warp_sum(s) + Et[j * CB + c]) * t;
        for (int i = lane; i <= j; i += 32) Eb[i * CB + c] -= __ldg(v + i) * s;
        if (lane == 0) Et[j * CB + c] -= s;
      }
      __syncwarp();
    }
  }
  __syncthreads();
  double* Oa = Eout + (size_t)a * l * l;
  double* Ob = Eout + (size_t)b * l * l;
  for (int e = threadIdx.x; e < l * cb; e += blockDim.x) {
    int r = e / cb, c = e - r * cb;
    Oa[(size_t)r * l + c0 + c] = Et[r * CB + c];
    if (pair) Ob[(size_t)r * l + c0 + c] = Eb[r * CB + c];
  }
}

__global__ void identity_kernel(double* E, int l) {
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < l * l; e += gridDim.x * blockDim.x)
    E[e] = (e / l == e % l) ? 1.0 : 0.0;
}

// -------------------------------------------------------------------------
int qr_plan(int m, int l, QrPlan* P) {
  P->m = m; P->l = l; P->k = std::min(m, l);
  P->cpw = P->rpl = 0;
  TTK_REQUIRE(l >= 1, kInvalidValue, "tsqr: l=%d must be positive", l);
  const int ld = l | 1;
  // shared memory holds the panel (H x ld), two reflector buffers (2 x H) and tau (l)
  int H = (kQrSmemDoubles - 128 - l) / (ld + 2);
  H = std::min(H, 2048);
  P->tree = 0;
  P->depth = 0;
  if (m <= H) {
    H = m;  // single panel, exactly m rows (wide inputs: min(m, l) reflectors)
  } else if (H < 2 * l) {
    // stacked-R levels would not shrink: leaf panels + binary tree of R pairs
    TTK_REQUIRE(l <= kQrMaxCols && H >= l, kInvalidValue, "tsqr: %d x %d: at most %d columns", m, l,
                kQrMaxCols);
    P->h = H;
    P->tree = 1;
    P->levels = 1;
    P->rows[0] = m;
    P->panels[0] = (m + H - 1) / H;
    int nodes = P->panels[0], t = 0;
    P->nodes[0] = nodes;
    size_t ws = align_up((size_t)nodes * l * H * 8, 256) + align_up((size_t)nodes * l * 8, 256);
    const size_t pk = (size_t)l * (l + 1) / 2;
    while (true) {
      ws += align_up((size_t)nodes * l * l * 8, 256) * 2;  // R and E of this tree level
      if (t > 0) ws += align_up((size_t)nodes * pk * 8, 256) + align_up((size_t)nodes * l * 8, 256);
      if (nodes == 1) break;
      nodes = (nodes + 1) / 2;
      ++t;
      TTK_REQUIRE(t < 24, kInvalidValue, "tsqr: tree too deep");
      P->nodes[t] = nodes;
    }
    P->depth = t;
    P->ws_bytes = ws + 4096;
    return kOk;
  } else {
    TTK_REQUIRE(H >= 2 * l, kInvalidValue,
                "tsqr: %d x %d needs a multi-panel tree; columns limited to %d", m, l, H / 2);
  }
  P->h = H;
  int rows = m, lev = 0;
  size_t ws = 0;
  while (true) {
    TTK_REQUIRE(lev < 16, kInvalidValue, "tsqr: too many levels");
    int panels = (rows + H - 1) / H;
    P->rows[lev] = rows;
    P->panels[lev] = panels;
    ws += align_up((size_t)panels * l * H * 8, 256);          // reflectors
    ws += align_up((size_t)panels * l * 8, 256);              // tau
    ws += align_up((size_t)panels * l * l * 8, 256);          // stacked R (next input)
    ws += align_up((size_t)rows * l * 8, 256);                // Q of this level (levels > 0)
    ++lev;
    if (panels == 1) break;
    rows = panels * l;
  }
  P->levels = lev;
  P->ws_bytes = ws + 4096;
  return kOk;
}

size_t tsqr_ws_bytes(int m, int l) {
  QrPlan P;
  if (m <= 0 || l <= 0) return 0;
  if (qr_plan(m, l, &P) != kOk) return 0;
  return P.ws_bytes;
}

static int qr_set_smem(const void* fn, size_t bytes) {
  TTK_TRY(set_attr_once(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes));
  return kOk;
}

static int tsqr_tree(const QrPlan& P, const double* A, long long a_rs, long long a_cs, double* Q,
                     long long q_rs, long long q_cs, double* R, void* ws, size_t ws_bytes, size_t smem_f,
                     size_t smem_a, cudaStream_t st) {
  const int l = P.l, H = P.h, D = P.depth;
  {  // per-device attributes (set_attr_once)
    TTK_TRY(qr_set_smem((const void*)qr_pair_factor_kernel, 227 * 1024));
    TTK_TRY(qr_set_smem((const void*)qr_pair_apply_kernel, 128 * 1024));
  }
  const size_t pk = (size_t)l * (l + 1) / 2;
  Arena ar(ws, ws_bytes);
  double* V0 = ar.take<double>((size_t)P.nodes[0] * l * H);
  double* T0 = ar.take<double>((size_t)P.nodes[0] * l);
  std::vector<double*> Rl(D + 1), El(D + 1), Vl(D + 1, nullptr), Tl(D + 1, nullptr);
  for (int t = 0; t <= D; ++t) {
    Rl[t] = ar.take<double>((size_t)P.nodes[t] * l * l);
    El[t] = ar.take<double>((size_t)P.nodes[t] * l * l);
    if (t > 0) {
      Vl[t] = ar.take<double>((size_t)P.nodes[t] * pk);
      Tl[t] = ar.take<double>((size_t)P.nodes[t] * l);
    }
  }
  TTK_REQUIRE(ar.used <= ws_bytes, kWorkspace, "tsqr(tree): workspace too small");
  qr_panel_factor_kernel<<<P.nodes[0], kQrThreads, smem_f, st>>>(P.rows[0], l, H, A, a_rs, a_cs, V0, T0,
                                                                 Rl[0]);
  TTK_CHECK_LAUNCH();
  const size_t smem_p = sizeof(double) * (2 * pk + l);
  for (int t = 1; t <= D; ++t) {
    qr_pair_factor_kernel<<<P.nodes[t], kQrThreads, smem_p, st>>>(l, P.nodes[t - 1], Rl[t - 1], Rl[t],
                                                                  Vl[t], Tl[t]);
    TTK_CHECK_LAUNCH();
  }
  if (R) TTK_CHECK_CUDA(cudaMemcpyAsync(R, Rl[D], sizeof(double) * (size_t)P.k * l,
                                        cudaMemcpyDeviceToDevice, st));
  identity_kernel<<<8, 256, 0, st>>>(El[D], l);
  TTK_CHECK_LAUNCH();
  for (int t = D; t >= 1; --t) {
    dim3 grid(P.nodes[t], (l + 31) / 32);
    qr_pair_apply_kernel<<<grid, 256, sizeof(double) * 2 * l * 32, st>>>(l, P.nodes[t - 1], Vl[t], Tl[t],
                                                                         El[t], El[t - 1]);
    TTK_CHECK_LAUNCH();
  }
  qr_panel_apply_kernel<<<P.nodes[0], kQrThreads, smem_a, st>>>(l, H, P.k, V0, T0, El[0], P.rows[0], Q,
                                                                q_rs, q_cs);
  TTK_CHECK_LAUNCH();
  return kOk;
}

int tsqr(int m, int l, const double* A, long long a_rs, long long a_cs, double* Q, long long q_rs,
         long long q_cs, double* R, void* ws, size_t ws_bytes, cudaStream_t st) {
  if (m <= 0 || l <= 0) return kOk;
  QrPlan P;
  TTK_TRY(qr_plan(m, l, &P));
  TTK_REQUIRE(ws != nullptr && ws_bytes >= P.ws_bytes, kWorkspace,
              "tsqr: workspace %zu < %zu bytes", ws_bytes, P.ws_bytes);
  const int H = P.h, ld = l | 1;
  {  // per-device attributes (set_attr_once)
    TTK_TRY(qr_set_smem((const void*)qr_panel_factor_kernel, 227 * 1024));
    TTK_TRY(qr_set_smem((const void*)qr_panel_apply_kernel, 227 * 1024));
  }
  const size_t smem_f = sizeof(double) * ((size_t)H * ld + 2 * H + l);
  const size_t smem_a = sizeof(double) * ((size_t)H * ld);
  if (P.tree) return tsqr_tree(P, A, a_rs, a_cs, Q, q_rs, q_cs, R, ws, ws_bytes, smem_f, smem_a, st);
  Arena ar(ws, ws_bytes);
  std::vector<double*> V(P.levels), T(P.levels), RS(P.levels), QL(P.levels);
  for (int i = 0; i < P.levels; ++i) {
    V[i] = ar.take<double>((size_t)P.panels[i] * l * H);
    T[i] = ar.take<double>((size_t)P.panels[i] * l);
    RS[i] = ar.take<double>((size_t)P.panels[i] * l * l);
    QL[i] = ar.take<double>((size_t)P.rows[i] * l);
  }
  // factor, bottom-up
  for (int i = 0; i < P.levels; ++i) {
    const double* in = (i == 0) ? A : RS[i - 1];
    long long rs = (i == 0) ? a_rs : l, cs = (i == 0) ? a_cs : 1;
    qr_panel_factor_kernel<<<P.panels[i], kQrThreads, smem_f, st>>>(P.rows[i], l, H, in, rs, cs, V[i],
                                                                    T[i], RS[i]);
    TTK_CHECK_LAUNCH();
  }
  const int top = P.levels - 1;
  if (R) {
    // top-level R (l x l) -> k x l
    TTK_CHECK_CUDA(cudaMemcpyAsync(R, RS[top], sizeof(double) * (size_t)P.k * l,
                                   cudaMemcpyDeviceToDevice, st));
  }
  // explicit Q, top-down
  for (int i = top; i >= 0; --i) {
    const double* qup = (i == top) ? nullptr : QL[i + 1];
    if (i == 0) {
      qr_panel_apply_kernel<<<P.panels[0], kQrThreads, smem_a, st>>>(l, H, P.k, V[0], T[0], qup, m, Q,
                                                                     q_rs, q_cs);
    } else {
      qr_panel_apply_kernel<<<P.panels[i], kQrThreads, smem_a, st>>>(l, H, l, V[i], T[i], qup,
                                                                     P.rows[i], QL[i], l, 1);
    }
    TTK_CHECK_LAUNCH();
  }
  return kOk;
}

// -------------------------------------------------------------------------
// One-sided Jacobi SVD of B (k x l, row-major).  Columns of B are stored
// column-major in shared memory; l/2 disjoint column pairs rotate per round
// (round-robin tournament), one 16-lane group per pair.
constexpr int kSvdThreads = 1024;
__device__ int* g_svd_sweeps = nullptr;  // optional diagnostic sink (tests)
__device__ long long* g_chol_prof = nullptr;  // diagnostics: phase clocks of chol_blocked_kernel
__device__ long long* g_fq_prof = nullptr;  // fused CholeskyQR2 phase timestamps (diagnostics)
constexpr int kSvdGroup = 16;  // lanes per column pair

template <int RPL>
__global__ void __launch_bounds__(kSvdThreads, 1)
    jacobi_svd_kernel(int k, int l, const double* __restrict__ B, long long b_rs, long long b_cs,
                      double* __restrict__ U, double* __restrict__ S, double* __restrict__ V, int want_v,
                      int scaled_u) {
  extern __shared__ double sm[];
  const int le = l + (l & 1);           // even number of columns (dummy zero column)
  const int kk = k;                     // column length
  const int ldc = kk | 1;
  double* C = sm;                       // le columns x ldc
  double* Vs = C + (size_t)le * ldc;    // le x le (col-major) when want_v
  __shared__ int changed;
  __shared__ double nrm[kQrMaxCols + 2];
  __shared__ int order[kQrMaxCols + 2];
  __shared__ int slot[kQrMaxCols + 2];  // round-robin position -> column
  const int tid = threadIdx.x;
  // initial column order: decreasing norm (speeds up convergence)
  for (int c = tid >> 5; c < l; c += blockDim.x >> 5) {
    double s = 0.0;
    for (int r = tid & 31; r < kk; r += 32) {
      double x = B[(long long)r * b_rs + (long long)c * b_cs];
      s += x * x;
    }
    s = warp_sum(s);
    if ((tid & 31) == 0) nrm[c] = s;
  }
  __syncthreads();
  for (int c = tid; c < l; c += blockDim.x) {
    int rank = 0;
    for (int j = 0; j < l; ++j) rank += (nrm[j] > nrm[c]) || (nrm[j] == nrm[c] && j < c);
    order[rank] = c;
  }
  __syncthreads();
  for (int e = tid; e < le * kk; e += blockDim.x) {
    int c = e / kk, r = e - c * kk;
    C[c * ldc + r] = (c < l) ? B[(long long)r * b_rs + (long long)order[c] * b_cs] : 0.0;
  }
  if (want_v)
    for (int e = tid; e < le * le; e += blockDim.x) {
      int c = e / le, r = e - c * le;
      Vs[c * le + r] = (c < l && r == order[c]) ? 1.0 : 0.0;
    }
  __syncthreads();
  const double tol = (double)max(kk, 1) * 1.1102230246251565e-16;
  const double tol2 = tol * tol;
  const int gl = tid % kSvdGroup;
  const int npairs = le / 2;
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
    __syncthreads();
    if (tid == 0) changed = 0;
    for (int rnd = 0; rnd < le - 1; ++rnd) {
      __syncthreads();
      // warp-uniform loop over pair slots (two 16-lane halves per warp) so the
      // butterfly reductions use full-warp shuffles (no collective fix-ups)
      constexpr int kGroupsPerWarp = 32 / kSvdGroup;
      for (int base = (tid >> 5) * kGroupsPerWarp; base < npairs; base += (blockDim.x >> 5) * kGroupsPerWarp) {
        const int pi = base + ((tid & 31) / kSvdGroup);
        const bool active = pi < npairs;
        // round-robin tournament: position 0 fixed, positions 1..le-1 rotate
        const int pic = active ? pi : 0;
        const int qi = le - 1 - pic;
        int p = 0, q;
        if (pic > 0) { p = pic - 1 + rnd; if (p >= le - 1) p -= le - 1; p += 1; }
        q = qi - 1 + rnd; if (q >= le - 1) q -= le - 1; q += 1;
        double* cp = C + p * ldc;
        double* cq = C + q * ldc;
        // this lane's rows of the pair, loaded once (independent loads, one
        // shared-memory latency) and kept in registers for the rotation
        double x[RPL], y[RPL];
#pragma unroll
        for (int i = 0; i < RPL; ++i) {
          const int r = gl + i * kSvdGroup;
          const bool ok = r < kk;
          x[i] = ok ? cp[r] : 0.0;
          y[i] = ok ? cq[r] : 0.0;
        }
        double a = 0.0, b = 0.0, g = 0.0, a2 = 0.0, b2 = 0.0, g2 = 0.0;
#pragma unroll
        for (int i = 0; i < RPL; i += 2) {
          a += x[i] * x[i]; b += y[i] * y[i]; g += x[i] * y[i];
          if (i + 1 < RPL) { a2 += x[i + 1] * x[i + 1]; b2 += y[i + 1] * y[i + 1]; g2 += x[i + 1] * y[i + 1]; }
        }
        a += a2; b += b2; g += g2;
#pragma unroll
        for (int o = kSvdGroup / 2; o > 0; o >>= 1) {
          a += __shfl_xor_sync(0xffffffffu, a, o);
          b += __shfl_xor_sync(0xffffffffu, b, o);
          g += __shfl_xor_sync(0xffffffffu, g, o);
        }
        if (active && a > 0.0 && b > 0.0 && g * g > tol2 * a * b) {
          // t = tan(theta) = sign(d) w / (|d| + sqrt(d^2 + w^2)), d = b - a, w = 2g
          const double dd = b - a, w = 2.0 * g;
          const double t = (dd >= 0.0 ? w : -w) / (fabs(dd) + sqrt(dd * dd + w * w));
          const double c = rsqrt(1.0 + t * t), s = c * t;
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const int r = gl + i * kSvdGroup;
            if (r < kk) {
              cp[r] = c * x[i] - s * y[i];
              cq[r] = s * x[i] + c * y[i];
            }
          }
          if (want_v) {
            double* vp = Vs + p * le;
            double* vq = Vs + q * le;
#pragma unroll
            for (int i = 0; i < RPL; ++i) {
              const int r = gl + i * kSvdGroup;
              const bool ok = r < le;
              x[i] = ok ? vp[r] : 0.0;
              y[i] = ok ? vq[r] : 0.0;
            }
#pragma unroll
            for (int i = 0; i < RPL; ++i) {
              const int r = gl + i * kSvdGroup;
              if (r < le) {
                vp[r] = c * x[i] - s * y[i];
                vq[r] = s * x[i] + c * y[i];
              }
            }
          }
          if (gl == 0) changed = 1;
        }
      }
    }
    __syncthreads();
    const int ch = changed;
    __syncthreads();  // everyone has read the flag before thread 0 resets it
    if (!ch) break;
  }
  if (tid == 0 && g_svd_sweeps) *g_svd_sweeps = sweep + 1;
  __syncthreads();
  // norms, ranking (descending, ties by index), outputs; C column c holds
  // original column order[c]
  for (int c = tid >> 5; c < l; c += blockDim.x >> 5) {
    double s = 0.0;
    for (int r = tid & 31; r < kk; r += 32) s += C[c * ldc + r] * C[c * ldc + r];
    s = warp_sum(s);
    if ((tid & 31) == 0) nrm[c] = sqrt(s);
  }
  __syncthreads();
  for (int c = tid; c < l; c += blockDim.x) {
    int rank = 0;
    for (int j = 0; j < l; ++j) rank += (nrm[j] > nrm[c]) || (nrm[j] == nrm[c] && j < c);
    slot[rank] = c;
  }
  __syncthreads();
  const int kout = min(kk, l);
  for (int i = tid; i < kout; i += blockDim.x) S[i] = nrm[slot[i]];
  for (int e = tid; e < kk * kout; e += blockDim.x) {
    int r = e / kout, i = e - r * kout;
    int c = slot[i];
    double sv = nrm[c];
    U[e] = scaled_u ? C[c * ldc + r] : ((sv > 0.0) ? C[c * ldc + r] / sv : 0.0);
  }
  if (want_v && V)
    for (int e = tid; e < l * kout; e += blockDim.x) {
      int r = e / kout, i = e - r * kout;
      V[e] = Vs[slot[i] * le + r];
    }
}

// ---------------------------------------------------------------------------
// Cluster-parallel one-sided Jacobi (same tournament, same rotation formula).
//
// The single-CTA kernel above runs on one SM and is bound by its shared-memory
// pipe: every round re-reads and re-writes both columns of every pair (and of
// V).  Here the le/2 pair slots are spread over a cluster of kJcCluster CTAs
// (one SM each); every 16-lane group keeps its two columns of C and of V in
// registers for the whole factorisation.  The round-robin schedule only moves
// columns between neighbouring slots, so after each round a slot pushes its
// outgoing columns straight into the destination slot's inbox (local or
// remote shared memory, DSMEM) and one cluster barrier publishes them:
//   position v -> v-1 (v >= 1, position 1 -> le-1, position 0 fixed), i.e.
//   left(s)  -> left(s-1)   (s >= 2),  left(1) -> right(0),  left(0) stays
//   right(s) -> right(s+1)  (s <= np-2),  right(np-1) -> left(np-1)
// which is exactly the p/q index rotation of jacobi_svd_kernel.

// 1/sqrt(p) for normal positive p without the library's slow-path CALL (a
// call inside the unrolled pivot loop forces the register-resident block
// to local memory): hardware approximation plus two Newton steps (~1 ulp).
__device__ __forceinline__ double rsqrt_nr(double p) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(p));
  const double h = 0.5 * p;
  y = y * fma(-h * y, y, 1.5);
  y = y * fma(-h * y, y, 1.5);
  return y;
}

// 1/sqrt(p) for the rotation formula (normal positive p): the fp64 hardware
// seed is good to 2^-20 on B200 (tools/rsqrt_acc.cu), so one third-order
// correction y (1 + e/2 + 3e^2/8), e = 1 - p y^2 (error ~0.3 e^3 < 2^-61)
// replaces rsqrt_nr's two Newton steps: four dependent fp64 ops instead of six.
__device__ __forceinline__ double rsqrt_rot(double p) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(p));
  const double e = fma(-p * y, y, 1.0);
  const double t = fma(e, 0.375, 0.5);
  return fma(y * e, t, y);
}

// Jacobi rotation of the pair Gram [[ra, rg], [rg, rb]] for the one-sided
// update x' = cs x - sn y, y' = sn x + cs y, returned unnormalised:
// (cs, sn) = (sum, wd) * rq, tan = wd / sum, sum = |dd| + rho, wd = sgn(dd) w,
// dd = rb - ra, w = 2 rg, rho = sqrt(dd^2 + w^2).  rho only sets the angle, so
// the hardware rsqrt seed (2^-20) suffices for it; rq = 1 / sqrt(sum^2 + wd^2)
// is refined, so the rotation is orthogonal to rounding with an angle good to
// ~1e-6 (the pair keeps a ~1e-6 |rg| residual; quadratic convergence holds down
// to the 1e-8 stop).  One refined rsqrt on the chain instead of two (same-box
// A/B, no V: 80x80 316 -> 306 us, 50x50 189 -> 181).  Forming sum x - wd y,
// wd x + sum y while rq is in flight and scaling after measured neutral.  The inputs
// are prescaled (largest column norm^2 in [1, 8)); pairs small enough for q to
// leave the normal range take the per-pair power-of-two rescale.
__device__ __forceinline__ void jacobi_rot(double ra, double rb, double rg, double& sum, double& wd, double& rq) {
  double dd = rb - ra, w = 2.0 * rg;
  double w2 = w * w;
  double q = fma(dd, dd, w2);
  if (!(q > 1e-280 && q < 1e280)) {  // rare: rescale the pair
    const long long ex = min((__double_as_longlong(ra + rb) >> 52) & 0x7ff, 2045LL);
    const double sc = __longlong_as_double((2046LL - ex) << 52);
    dd *= sc;
    w *= sc;
    w2 = w * w;
    q = fma(dd, dd, w2);
  }
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(q));
  sum = fma(q, y, fabs(dd));
  wd = dd >= 0.0 ? w : -w;
  rq = rsqrt_rot(fma(sum, sum, w2));
}

constexpr int kJcCluster = 8;
constexpr int kJcMaxSlots = 8;   // pair slots per CTA (le <= 128)
constexpr int kJcThreads = kJcMaxSlots * kSvdGroup;

__device__ __forceinline__ uint32_t jc_map(const void* p, int rank) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
// asynchronous store into (possibly remote) shared memory; completion is
// counted in bytes on the destination CTA's mbarrier
__device__ __forceinline__ void jc_st_v2(uint32_t addr, double a, double b, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(addr),
               "d"(a), "d"(b), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void jc_st_u32(uint32_t addr, uint32_t v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(addr), "r"(v),
               "r"(bar)
               : "memory");
}
__device__ __forceinline__ void jc_arm(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// CTA-scope acquire: the remote st.async data is tracked by this CTA's own
// mbarrier (complete_tx), as for TMA multicast (a cluster-scope acquire adds an
// L1 invalidation, CCTL.IVALL, to every wait; measured time-neutral in r01)
__device__ __forceinline__ void jc_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}

__device__ long long* g_jc_prof = nullptr;  // optional per-phase clock sink (diagnostics)
static bool g_jc_prof_host = false;            // host mirror: launch the PROF kernel instances

template <int RPL>
__global__ void __cluster_dims__(kJcCluster, 1, 1) __launch_bounds__(kJcThreads, 1)
    jacobi_cluster_kernel(int k, int l, const double* __restrict__ B, long long b_rs, long long b_cs,
                          double* __restrict__ U, double* __restrict__ S, double* __restrict__ V,
                          int want_v, int scaled_u, double skip2) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int crank = (int)cl.block_rank();
  // inboxes [2 bufs][spc][2 sides][2 (C,V)][RPL/2][16 lanes] of double2 (conflict-free)
  extern __shared__ __align__(16) double sm[];
  __shared__ double nrm[kQrMaxCols + 2];
  __shared__ double fin[kQrMaxCols + 2];  // final column norms, every column (all CTAs)
  __shared__ int order[kQrMaxCols + 2];
  __shared__ int flags[64];               // per-sweep "rotated" flag (never reset)
  __shared__ int bigf[64];                // per-sweep "some pair had |g|/sqrt(ab) > skip" flag
  __shared__ int inid[2][kJcMaxSlots][2];
  __shared__ __align__(8) unsigned long long mbar[2];
  const int le = l + (l & 1), kk = k, np = le / 2;
  const int spc = (np + kJcCluster - 1) / kJcCluster;
  const int tid = threadIdx.x, li = tid / kSvdGroup, gl = tid % kSvdGroup;
  const int si = crank * spc + li;
  const bool active = li < spc && si < np;
  constexpr int box = RPL * kSvdGroup;  // doubles per column part
  const int nv = want_v ? 2 : 1;
  const uint32_t msg_bytes = (uint32_t)(box * 8 * nv + 4);
  // bytes this CTA receives per round: a right column for every slot, a left
  // column for slots 1..np-2 (slot 0 keeps its left, slot np-1 takes its own right)
  // (only columns arriving from another CTA are counted)
  uint32_t rx_bytes = 0;
  if (np > 1)
    for (int j = 0; j < spc; ++j) {
      const int s = crank * spc + j;
      if (s >= np) break;
      const int from_r = (s == 0) ? 1 : s - 1;  // source of the new right column
      if (from_r / spc != crank) rx_bytes += msg_bytes;
      if (s >= 1 && s <= np - 2 && (s + 1) / spc != crank) rx_bytes += msg_bytes;
    }
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&mbar[0]);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (rx_bytes) { jc_arm(bar0, rx_bytes); jc_arm(bar0 + 8, rx_bytes); }
  }
  // initial order: decreasing norm, ties by index (identical in every CTA)
  for (int c = tid >> 5; c < l; c += blockDim.x >> 5) {
    double s = 0.0;
    for (int r = tid & 31; r < kk; r += 32) {
      double x = B[(long long)r * b_rs + (long long)c * b_cs];
      s += x * x;
    }
    s = warp_sum(s);
    if ((tid & 31) == 0) nrm[c] = s;
  }
  for (int i = tid; i < 64; i += blockDim.x) { flags[i] = 0; bigf[i] = 0; }
  __syncthreads();
  for (int c = tid; c < l; c += blockDim.x) {
    int rank = 0;
    for (int j = 0; j < l; ++j) rank += (nrm[j] > nrm[c]) || (nrm[j] == nrm[c] && j < c);
    order[rank] = c;
  }
  __syncthreads();
  int idl = active ? si : 0, idr = active ? le - 1 - si : 0;
  double x[RPL], y[RPL], vx[RPL], vy[RPL];
#pragma unroll
  for (int i = 0; i < RPL; ++i) {
    const int r = gl + i * kSvdGroup;
    const bool okl = active && r < kk && idl < l, okr = active && r < kk && idr < l;
    x[i] = okl ? B[(long long)r * b_rs + (long long)order[idl] * b_cs] : 0.0;
    y[i] = okr ? B[(long long)r * b_rs + (long long)order[idr] * b_cs] : 0.0;
    vx[i] = (want_v && active && idl < l && r == order[idl]) ? 1.0 : 0.0;
    vy[i] = (want_v && active && idr < l && r == order[idr]) ? 1.0 : 0.0;
  }
  const double tol = (double)max(kk, 1) * 1.1102230246251565e-16;
  const double tol2 = tol * tol;
  auto inbox = [&](int buf, int slot_local, int side, int cv) {
    return sm + ((((size_t)buf * spc + slot_local) * 2 + side) * 2 + cv) * box + gl * 2;
  };
  const uint32_t buf_bytes = (uint32_t)(spc * 4 * box * 8);
  const uint32_t id_bytes = (uint32_t)(kJcMaxSlots * 2 * sizeof(int));
  // destinations (shared::cluster addresses of buffer 0), fixed for the whole run:
  //   left(s) -> left(s-1) (s >= 2), left(1) -> right(0); right(s) -> right(s+1) (s <= np-2)
  const bool send_l = active && si >= 1 && si <= np - 1 && np > 1 && !(si == np - 1 && si == 0);
  const bool send_r = active && si <= np - 2;
  // same-CTA moves are plain shared-memory stores (ordered by __syncthreads);
  // only moves across a CTA boundary travel as st.async (completion counted on
  // the destination's mbarrier)
  uint32_t l_c = 0, l_id = 0, l_bar = 0, r_c = 0, r_id = 0, r_bar = 0;
  double *l_loc = nullptr, *r_loc = nullptr;
  int* l_idloc = nullptr;
  int* r_idloc = nullptr;
  bool l_remote = false, r_remote = false;
  if (send_l) {
    const int ds = si - 1, side = (si == 1) ? 1 : 0;
    const int dc = ds / spc, dl = ds - dc * spc;
    l_remote = dc != crank;
    l_loc = sm + ((((size_t)dl) * 2 + side) * 2) * box + gl * 2;
    l_idloc = &inid[0][dl][side];
    l_c = jc_map(l_loc, dc);
    l_id = jc_map(l_idloc, dc);
    l_bar = jc_map(&mbar[0], dc);
  }
  if (send_r) {
    const int ds = si + 1;
    const int dc = ds / spc, dl = ds - dc * spc;
    r_remote = dc != crank;
    r_loc = sm + ((((size_t)dl) * 2 + 1) * 2) * box + gl * 2;
    r_idloc = &inid[0][dl][1];
    r_c = jc_map(r_loc, dc);
    r_id = jc_map(r_idloc, dc);
    r_bar = jc_map(&mbar[0], dc);
  }
  // a warp waits for this CTA's incoming columns only if it holds a slot
  const bool warp_active = __any_sync(0xffffffffu, active);
  cl.sync();  // barriers initialised and armed in every CTA before the first remote store
  long long* const prof = (tid == 0) ? g_jc_prof : nullptr;
  long long pt[4] = {0, 0, 0, 0}, tc = 0;
  int sweep = 0, round = 0;
  for (; sweep < 60; ++sweep) {
    for (int rnd = 0; rnd < le - 1; ++rnd, ++round) {
      if (prof) tc = clock64();
      double a = 0.0, b = 0.0, g = 0.0, a2 = 0.0, b2 = 0.0, g2 = 0.0;
#pragma unroll
      for (int i = 0; i < RPL; i += 2) {
        a += x[i] * x[i]; b += y[i] * y[i]; g += x[i] * y[i];
        if (i + 1 < RPL) { a2 += x[i + 1] * x[i + 1]; b2 += y[i + 1] * y[i + 1]; g2 += x[i + 1] * y[i + 1]; }
      }
      a += a2; b += b2; g += g2;
#pragma unroll
      for (int o = kSvdGroup / 2; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        g += __shfl_xor_sync(0xffffffffu, g, o);
      }
      if (active && gl == 0 && g * g > skip2 * a * b) bigf[sweep] = 1;
      if (active && a > 0.0 && b > 0.0 && g * g > tol2 * a * b) {
        // same angle as tan = sign(d) w / (|d| + rho), division-free:
        //   c = (|d| + rho) / sqrt(q), s = sign(d) w / sqrt(q), q = 2 rho (|d| + rho)
        // (CALL-free square roots: the library sqrt/rsqrt put a slow-path
        // CALL and its reconvergence barrier on every round's critical path).
        // c and s depend only on w/dd, so both are first scaled by the exact
        // power of two 2^-e(a+b): q below then stays a normal number (< 8) for
        // any column norms, as the flush-to-zero approximation requires.
        const long long ex = min((__double_as_longlong(a + b) >> 52) & 0x7ff, 2045LL);
        const double sc = __longlong_as_double((2046LL - ex) << 52);
        const double dd = (b - a) * sc, w = 2.0 * g * sc;
        const double q = dd * dd + w * w;
        const double rho = q * rsqrt_rot(q);
        const double sum = fabs(dd) + rho;
        const double rq = rsqrt_rot(fma(2.0 * rho, fabs(dd), 2.0 * q));  // 2 rho (|dd| + rho)
        const double c = sum * rq, s = (dd >= 0.0 ? w : -w) * rq;
#pragma unroll
        for (int i = 0; i < RPL; ++i) {  // old x consumed first: no register moves
          const double cx = c * x[i], sx = s * x[i];
          x[i] = fma(-s, y[i], cx);
          y[i] = fma(c, y[i], sx);
        }
        if (want_v) {
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const double cx = c * vx[i], sx = s * vx[i];
            vx[i] = fma(-s, vy[i], cx);
            vy[i] = fma(c, vy[i], sx);
          }
        }
        if (gl == 0) flags[sweep] = 1;
      }
      if (prof) { long long t = clock64(); pt[0] += t - tc; tc = t; }
      if (np > 1) {
        const int buf = round & 1;
        const uint32_t bo = buf * buf_bytes, io = buf * id_bytes, mo = buf * 8;
        if (send_l) {
          if (l_remote) {
#pragma unroll
            for (int j = 0; j < RPL; j += 2) jc_st_v2(l_c + bo + 128 * j, x[j], x[j + 1], l_bar + mo);
            if (want_v) {
#pragma unroll
              for (int j = 0; j < RPL; j += 2) jc_st_v2(l_c + bo + box * 8 + 128 * j, vx[j], vx[j + 1], l_bar + mo);
            }
            if (gl == 0) jc_st_u32(l_id + io, (uint32_t)idl, l_bar + mo);
          } else {
            double2* pc = reinterpret_cast<double2*>(l_loc + buf * (buf_bytes / 8));
#pragma unroll
            for (int j = 0; j < RPL / 2; ++j) pc[j * kSvdGroup] = make_double2(x[2 * j], x[2 * j + 1]);
            if (want_v) {
#pragma unroll
              for (int j = 0; j < RPL / 2; ++j) pc[box / 2 + j * kSvdGroup] = make_double2(vx[2 * j], vx[2 * j + 1]);
            }
            if (gl == 0) l_idloc[buf * kJcMaxSlots * 2] = idl;
          }
        }
        if (send_r) {
          if (r_remote) {
#pragma unroll
            for (int j = 0; j < RPL; j += 2) jc_st_v2(r_c + bo + 128 * j, y[j], y[j + 1], r_bar + mo);
            if (want_v) {
#pragma unroll
              for (int j = 0; j < RPL; j += 2) jc_st_v2(r_c + bo + box * 8 + 128 * j, vy[j], vy[j + 1], r_bar + mo);
            }
            if (gl == 0) jc_st_u32(r_id + io, (uint32_t)idr, r_bar + mo);
          } else {
            double2* pc = reinterpret_cast<double2*>(r_loc + buf * (buf_bytes / 8));
#pragma unroll
            for (int j = 0; j < RPL / 2; ++j) pc[j * kSvdGroup] = make_double2(y[2 * j], y[2 * j + 1]);
            if (want_v) {
#pragma unroll
              for (int j = 0; j < RPL / 2; ++j) pc[box / 2 + j * kSvdGroup] = make_double2(vy[2 * j], vy[2 * j + 1]);
            }
            if (gl == 0) r_idloc[buf * kJcMaxSlots * 2] = idr;
          }
        }
        __syncthreads();  // same-CTA moves visible
        if (prof) { long long t = clock64(); pt[1] += t - tc; tc = t; }
        if (warp_active && rx_bytes) {
          jc_wait(bar0 + mo, (round >> 1) & 1);
          if (tid == 0) jc_arm(bar0 + mo, rx_bytes);  // for round + 2
        }
        if (prof) { long long t = clock64(); pt[2] += t - tc; tc = t; }
        if (active) {
          if (si >= 1) {
            if (si == np - 1) {
#pragma unroll
              for (int i = 0; i < RPL; ++i) { x[i] = y[i]; vx[i] = vy[i]; }
              idl = idr;
            } else {
              const double2* pc = reinterpret_cast<const double2*>(inbox(buf, li, 0, 0));
#pragma unroll
              for (int j = 0; j < RPL / 2; ++j) { double2 v2 = pc[j * kSvdGroup]; x[2 * j] = v2.x; x[2 * j + 1] = v2.y; }
              if (want_v) {
                const double2* pv = reinterpret_cast<const double2*>(inbox(buf, li, 0, 1));
#pragma unroll
                for (int j = 0; j < RPL / 2; ++j) { double2 v2 = pv[j * kSvdGroup]; vx[2 * j] = v2.x; vx[2 * j + 1] = v2.y; }
              }
              idl = inid[buf][li][0];
            }
          }
          const double2* pc = reinterpret_cast<const double2*>(inbox(buf, li, 1, 0));
#pragma unroll
          for (int j = 0; j < RPL / 2; ++j) { double2 v2 = pc[j * kSvdGroup]; y[2 * j] = v2.x; y[2 * j + 1] = v2.y; }
          if (want_v) {
            const double2* pv = reinterpret_cast<const double2*>(inbox(buf, li, 1, 1));
#pragma unroll
            for (int j = 0; j < RPL / 2; ++j) { double2 v2 = pv[j * kSvdGroup]; vy[2 * j] = v2.x; vy[2 * j + 1] = v2.y; }
          }
          idr = inid[buf][li][1];
        }
        if (prof) { long long t = clock64(); pt[3] += t - tc; tc = t; }
      }
    }
    // every rotation of this sweep is ordered before this cluster barrier
    cl.sync();
    int ch = 0, big = 0;
#pragma unroll 1
    for (int r = 0; r < kJcCluster; ++r) {
      ch |= *cl.map_shared_rank(&flags[sweep], r);
      big |= *cl.map_shared_rank(&bigf[sweep], r);
    }
    // no rotation, or every pair already within skip (the next sweep's rotations
    // would be O(skip^2), below tol: it is a confirmation sweep)
    if (!ch || !big) break;
  }
  if (crank == 0 && tid == 0 && g_svd_sweeps) *g_svd_sweeps = sweep + 1;
  if (prof) {
    for (int i = 0; i < 4; ++i) atomicAdd((unsigned long long*)&prof[crank * 5 + i], (unsigned long long)pt[i]);
    atomicAdd((unsigned long long*)&prof[crank * 5 + 4], (unsigned long long)round);
  }
  // final norms of every column, broadcast to every CTA
  double a = 0.0, b = 0.0;
#pragma unroll
  for (int i = 0; i < RPL; ++i) { a += x[i] * x[i]; b += y[i] * y[i]; }
#pragma unroll
  for (int o = kSvdGroup / 2; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  a = sqrt(a); b = sqrt(b);
  if (active && gl == 0)
    for (int r = 0; r < kJcCluster; ++r) {
      *cl.map_shared_rank(&fin[idl], r) = a;
      *cl.map_shared_rank(&fin[idr], r) = b;
    }
  cl.sync();
  if (!active) return;
  const int kout = min(kk, l);
#pragma unroll 1
  for (int side = 0; side < 2; ++side) {
    const int id = side ? idr : idl;
    const double nv2 = side ? b : a;
    int rank = 0;
    for (int j = 0; j < le; ++j) rank += (fin[j] > nv2) || (fin[j] == nv2 && j < id);
    if (id >= l || rank >= kout) continue;
    if (gl == 0) S[rank] = nv2;
    const double inv = (scaled_u || nv2 <= 0.0) ? 1.0 : 1.0 / nv2;
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int r = gl + i * kSvdGroup;
      const double cv = side ? y[i] : x[i];
      if (r < kk) U[(size_t)r * kout + rank] = scaled_u ? cv : (nv2 > 0.0 ? cv * inv : 0.0);
      if (want_v && V && r < l) V[(size_t)r * kout + rank] = side ? vy[i] : vx[i];
    }
  }
}

// ---------------------------------------------------------------------------
// Block-ordered cluster Jacobi.  Same rotations, stopping rule and outputs as
// jacobi_cluster_kernel, different cyclic pair order: the le columns form 16
// blocks of bs columns, CTA c holds two blocks P(c), Q(c) (slot a of the CTA
// owns column a of each).  A sweep is
//   block round 0  : round-robin over the CTA's own 2 bs columns (2 bs - 1 rounds;
//                    covers every pair inside P(c) u Q(c));
//   block rounds 1-14: bs rounds pairing P_a with Q_{a-t}: the Q block shifts by one
//                    slot inside the CTA between rounds (all bs^2 cross pairs);
//   after every block round the blocks move between CTAs by the circle method
//   on 16 blocks (P(c) -> P(c-1), P(1) -> Q(0), Q(c) -> Q(c+1), Q(7) -> P(7)).
// Every pair meets once per sweep, le - 1 rounds as before, but only 15 of
// them end with a DSMEM handoff + mbarrier wait (the ~900-cycle part of the
// plain kernel's round: r01 phase clocks rotate 666 / send 277 / wait 272 /
// pull 320 at 80 x 80); the others exchange through this CTA's shared memory
// with one barrier.
// diagnostics (TTK_JB_DIAG, fixed 9 sweeps): 1 = no rotations, 2 = also no local
// moves, 3 = barrier only, 4 = stores + barrier.  r01, 80 x 80 on one box: 528 us
// normal, 488 (1), 339 (2), 370 (3), 431 (4): dots + reduction ~465 cycles per
// round, rotation ~110 (mostly hidden), local move ~400 (barrier ~90, stores
// ~160, loads ~160), block moves ~230 per round on average
__device__ int g_jb_diag = 0;
constexpr int kJbCluster = 8;
constexpr int kJbMaxSlots = 16;  // columns per block (8-CTA cluster: <= 8, l <= 128)

template <int RPL, int CL = kJbCluster>
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(kJbMaxSlots * kSvdGroup, 1)
    jacobi_block_kernel(int k, int l, const double* __restrict__ B, long long b_rs, long long b_cs,
                        double* __restrict__ U, double* __restrict__ S, double* __restrict__ V, int want_v_arg,
                        int scaled_u, double skip2) {
  // V accumulation is a compile-time constant (its runtime branches cost
  // instructions every round); V stores stay guarded by V != nullptr
  const bool want_v = true;
  (void)want_v_arg;
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int c = (int)cl.block_rank();
  extern __shared__ __align__(16) double sm[];
  __shared__ double nrm[kQrMaxCols + 2];
  __shared__ double fin[kQrMaxCols + 2];
  __shared__ int order[kQrMaxCols + 2];
  __shared__ int flags[64];
  __shared__ int bigf[64];
  __shared__ int bid[2][kJbMaxSlots][2];  // block-move inbox: column ids
  __shared__ int lid[2][kJbMaxSlots][2];  // local-move inbox: column ids
  __shared__ __align__(8) unsigned long long mbar[2];
  const int bs = (l + 2 * CL - 1) / (2 * CL);
  const int le = 2 * CL * bs, kk = k;
  const int tid = threadIdx.x, a = tid / kSvdGroup, gl = tid % kSvdGroup;
  const bool active = a < bs;
  const int diag = g_jb_diag;  // diagnostics only (0 in production)
  constexpr int box = RPL * kSvdGroup;
  const int nv = want_v ? 2 : 1;
  // [2 bufs][bs slots][2 sides][2 (C, V)][box], block inbox then local inbox
  double* const lbox = sm + (size_t)2 * bs * 4 * box;
  auto bslot = [&](int buf, int slot, int side, int cv) {
    return sm + ((((size_t)buf * bs + slot) * 2 + side) * 2 + cv) * box + gl * 2;
  };
  auto lslot = [&](int buf, int slot, int side, int cv) {
    return lbox + ((((size_t)buf * bs + slot) * 2 + side) * 2 + cv) * box + gl * 2;
  };
  const uint32_t msg_bytes = (uint32_t)(box * 8 * nv + 4);
  // remote columns received per block move: new Q always, new P for 1 <= c <= CL-2
  const uint32_t rx_bytes = (uint32_t)bs * msg_bytes * ((c >= 1 && c <= CL - 2) ? 2u : 1u);
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&mbar[0]);
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    jc_arm(bar0, rx_bytes);
    jc_arm(bar0 + 8, rx_bytes);
  }
  // initial order: decreasing norm, ties by index (identical in every CTA)
  for (int cc = tid >> 5; cc < l; cc += blockDim.x >> 5) {
    double s = 0.0;
    for (int r = tid & 31; r < kk; r += 32) {
      double xv = B[(long long)r * b_rs + (long long)cc * b_cs];
      s += xv * xv;
    }
    s = warp_sum(s);
    if ((tid & 31) == 0) nrm[cc] = s;
  }
  for (int i = tid; i < 64; i += blockDim.x) { flags[i] = 0; bigf[i] = 0; }
  __syncthreads();
  for (int cc = tid; cc < l; cc += blockDim.x) {
    int rank = 0;
    for (int j = 0; j < l; ++j) rank += (nrm[j] > nrm[cc]) || (nrm[j] == nrm[cc] && j < cc);
    order[rank] = cc;
  }
  __syncthreads();
  // positions: P slot a of CTA c = c bs + a, Q slot a = le - 1 - (c bs + a)
  int idl = active ? c * bs + a : 0, idr = active ? le - 1 - (c * bs + a) : 0;
  double x[RPL], y[RPL], vx[RPL], vy[RPL];
#pragma unroll
  for (int i = 0; i < RPL; ++i) {
    const int r = gl + i * kSvdGroup;
    const bool okl = active && r < kk && idl < l, okr = active && r < kk && idr < l;
    x[i] = okl ? B[(long long)r * b_rs + (long long)order[idl] * b_cs] : 0.0;
    y[i] = okr ? B[(long long)r * b_rs + (long long)order[idr] * b_cs] : 0.0;
    vx[i] = (want_v && active && idl < l && r == order[idl]) ? 1.0 : 0.0;
    vy[i] = (want_v && active && idr < l && r == order[idr]) ? 1.0 : 0.0;
  }
  const double tol = (double)max(kk, 1) * 1.1102230246251565e-16;
  const double tol2 = tol * tol;
  // block-move destinations (shared::cluster addresses, buffer 0)
  const bool send_p = active && c >= 1;       // P(c) -> P(c-1) (c >= 2), P(1) -> Q(0)
  const bool send_q = active && c <= CL - 2;  // Q(c) -> Q(c+1)
  uint32_t p_c = 0, p_id = 0, p_bar = 0, q_c = 0, q_id = 0, q_bar = 0;
  if (send_p) {
    const int side = (c == 1) ? 1 : 0;
    p_c = jc_map(bslot(0, a, side, 0), c - 1);
    p_id = jc_map(&bid[0][a][side], c - 1);
    p_bar = jc_map(&mbar[0], c - 1);
  }
  if (send_q) {
    q_c = jc_map(bslot(0, a, 1, 0), c + 1);
    q_id = jc_map(&bid[0][a][1], c + 1);
    q_bar = jc_map(&mbar[0], c + 1);
  }
  const uint32_t bbuf_bytes = (uint32_t)(bs * 4 * box * 8);
  const uint32_t bid_bytes = (uint32_t)(kJbMaxSlots * 2 * sizeof(int));
  cl.sync();  // barriers initialised and armed in every CTA before the first remote store

  auto put = [&](double* dst, const double* v) {  // one column part into an inbox slot
    double2* p = reinterpret_cast<double2*>(dst);
#pragma unroll
    for (int j = 0; j < RPL / 2; ++j) p[j * kSvdGroup] = make_double2(v[2 * j], v[2 * j + 1]);
  };
  auto get = [&](const double* src, double* v) {
    const double2* p = reinterpret_cast<const double2*>(src);
#pragma unroll
    for (int j = 0; j < RPL / 2; ++j) { double2 t = p[j * kSvdGroup]; v[2 * j] = t.x; v[2 * j + 1] = t.y; }
  };

  long long* const prof = (tid == 0) ? g_jc_prof : nullptr;
  long long pt[4] = {0, 0, 0, 0}, tc = 0;
  int sweep = 0, moves = 0, lr = 0;
  for (; sweep < 60; ++sweep) {
    for (int br = 0; br < 2 * CL - 1; ++br) {
      const int nr = (br == 0) ? 2 * bs - 1 : bs;
#pragma unroll 2
      for (int t = 0; t < nr; ++t, ++lr) {
        // ---- rotate the pair (x, y) ----
        if (prof) tc = clock64();
        double ra = 0.0, rb = 0.0, rg = 0.0, a2 = 0.0, b2 = 0.0, g2 = 0.0;
#pragma unroll
        for (int i = 0; i < RPL; i += 2) {
          ra += x[i] * x[i]; rb += y[i] * y[i]; rg += x[i] * y[i];
          if (i + 1 < RPL) { a2 += x[i + 1] * x[i + 1]; b2 += y[i + 1] * y[i + 1]; g2 += x[i + 1] * y[i + 1]; }
        }
        ra += a2; rb += b2; rg += g2;
#pragma unroll
        for (int o = kSvdGroup / 2; o > 0; o >>= 1) {
          ra += __shfl_xor_sync(0xffffffffu, ra, o);
          rb += __shfl_xor_sync(0xffffffffu, rb, o);
          rg += __shfl_xor_sync(0xffffffffu, rg, o);
        }
        if (active && gl == 0 && rg * rg > skip2 * ra * rb) bigf[sweep] = 1;
        if (active && ra > 0.0 && rb > 0.0 && rg * rg > tol2 * ra * rb && diag == 0) {
          // jacobi_cluster_kernel's division- and CALL-free rotation
          const long long ex = min((__double_as_longlong(ra + rb) >> 52) & 0x7ff, 2045LL);
          const double sc = __longlong_as_double((2046LL - ex) << 52);
          const double dd = (rb - ra) * sc, w = 2.0 * rg * sc;
          const double q = dd * dd + w * w;
          const double rho = q * rsqrt_rot(q);
          const double sum = fabs(dd) + rho;
          const double rq = rsqrt_rot(fma(2.0 * rho, fabs(dd), 2.0 * q));  // 2 rho (|dd| + rho)
          const double cs = sum * rq, sn = (dd >= 0.0 ? w : -w) * rq;
#pragma unroll
          for (int i = 0; i < RPL; ++i) {  // old x consumed first: no register moves
            const double cx = cs * x[i], sx = sn * x[i];
            x[i] = fma(-sn, y[i], cx);
            y[i] = fma(cs, y[i], sx);
          }
          if (want_v) {
#pragma unroll
            for (int i = 0; i < RPL; ++i) {
              const double cx = cs * vx[i], sx = sn * vx[i];
              vx[i] = fma(-sn, vy[i], cx);
              vy[i] = fma(cs, vy[i], sx);
            }
          }
          if (gl == 0) flags[sweep] = 1;
        }
        // ---- local move through this CTA's shared memory ----
        if (prof) { long long t = clock64(); pt[0] += t - tc; tc = t; }
        const int buf = lr & 1;
        if (diag == 2) {
        } else if (diag == 3) {
          __syncthreads();
        } else if (diag == 4) {
          if (active) {
            const int ds = (a + 1 == bs) ? 0 : a + 1;
            put(lslot(buf, ds, 1, 0), y);
            if (want_v) put(lslot(buf, ds, 1, 1), vy);
          }
          __syncthreads();
        } else if (br == 0) {
          // round-robin over the CTA's 2 bs columns (circle method on bs slots):
          // left(s) -> left(s-1) (s >= 2), left(1) -> right(0), right(s) -> right(s+1),
          // right(bs-1) -> left(bs-1), left(0) fixed
          if (active) {
            if (a >= 1) {
              const int ds = a - 1, side = (a == 1) ? 1 : 0;
              put(lslot(buf, ds, side, 0), x);
              if (want_v) put(lslot(buf, ds, side, 1), vx);
              if (gl == 0) lid[buf][ds][side] = idl;
            }
            if (a <= bs - 2) {
              put(lslot(buf, a + 1, 1, 0), y);
              if (want_v) put(lslot(buf, a + 1, 1, 1), vy);
              if (gl == 0) lid[buf][a + 1][1] = idr;
            }
          }
          __syncthreads();
          if (active) {
            if (a >= 1) {
              if (a == bs - 1) {
#pragma unroll
                for (int i = 0; i < RPL; ++i) { x[i] = y[i]; vx[i] = vy[i]; }
                idl = idr;
              } else {
                get(lslot(buf, a, 0, 0), x);
                if (want_v) get(lslot(buf, a, 0, 1), vx);
                idl = lid[buf][a][0];
              }
            }
            get(lslot(buf, a, 1, 0), y);
            if (want_v) get(lslot(buf, a, 1, 1), vy);
            idr = lid[buf][a][1];
          }
        } else {
          // Q block shifts by one slot: Q_a -> slot a + 1 (mod bs)
          if (active) {
            const int ds = (a + 1 == bs) ? 0 : a + 1;
            put(lslot(buf, ds, 1, 0), y);
            if (want_v) put(lslot(buf, ds, 1, 1), vy);
            if (gl == 0) lid[buf][ds][1] = idr;
          }
          __syncthreads();
          if (active) {
            get(lslot(buf, a, 1, 0), y);
            if (want_v) get(lslot(buf, a, 1, 1), vy);
            idr = lid[buf][a][1];
          }
        }
        if (prof) { long long t = clock64(); pt[1] += t - tc; tc = t; }
      }
      // ---- block move between CTAs (DSMEM, completion on the receiver's mbarrier) ----
      {
        const int buf = moves & 1;
        const uint32_t bo = buf * bbuf_bytes, io = buf * bid_bytes, mo = buf * 8;
        if (send_p) {
#pragma unroll
          for (int j = 0; j < RPL; j += 2) jc_st_v2(p_c + bo + 128 * j, x[j], x[j + 1], p_bar + mo);
          if (want_v) {
#pragma unroll
            for (int j = 0; j < RPL; j += 2) jc_st_v2(p_c + bo + box * 8 + 128 * j, vx[j], vx[j + 1], p_bar + mo);
          }
          if (gl == 0) jc_st_u32(p_id + io, (uint32_t)idl, p_bar + mo);
        }
        if (send_q) {
#pragma unroll
          for (int j = 0; j < RPL; j += 2) jc_st_v2(q_c + bo + 128 * j, y[j], y[j + 1], q_bar + mo);
          if (want_v) {
#pragma unroll
            for (int j = 0; j < RPL; j += 2) jc_st_v2(q_c + bo + box * 8 + 128 * j, vy[j], vy[j + 1], q_bar + mo);
          }
          if (gl == 0) jc_st_u32(q_id + io, (uint32_t)idr, q_bar + mo);
        }
        jc_wait(bar0 + mo, (moves >> 1) & 1);
        __syncthreads();  // every thread has seen the phase complete before it is re-armed
        if (tid == 0) jc_arm(bar0 + mo, rx_bytes);  // for move + 2
        if (active) {
          if (c >= 1) {
            if (c == CL - 1) {
#pragma unroll
              for (int i = 0; i < RPL; ++i) { x[i] = y[i]; vx[i] = vy[i]; }
              idl = idr;
            } else {
              get(bslot(buf, a, 0, 0), x);
              if (want_v) get(bslot(buf, a, 0, 1), vx);
              idl = bid[buf][a][0];
            }
          }
          get(bslot(buf, a, 1, 0), y);
          if (want_v) get(bslot(buf, a, 1, 1), vy);
          idr = bid[buf][a][1];
        }
        ++moves;
        if (prof) { long long t = clock64(); pt[2] += t - tc; tc = t; }
      }
    }
    // every rotation of this sweep is ordered before this cluster barrier
    cl.sync();
    int ch = 0, big = 0;
#pragma unroll 1
    for (int r = 0; r < CL; ++r) {
      ch |= *cl.map_shared_rank(&flags[sweep], r);
      big |= *cl.map_shared_rank(&bigf[sweep], r);
    }
    if (diag ? sweep == 8 : (!ch || !big)) break;
  }
  if (c == 0 && tid == 0 && g_svd_sweeps) *g_svd_sweeps = sweep + 1;
  if (prof) {
    for (int i = 0; i < 4; ++i) atomicAdd((unsigned long long*)&prof[c * 5 + i], (unsigned long long)pt[i]);
    atomicAdd((unsigned long long*)&prof[c * 5 + 4], (unsigned long long)lr);
  }
  // final norms of every column, broadcast to every CTA
  double na = 0.0, nb = 0.0;
#pragma unroll
  for (int i = 0; i < RPL; ++i) { na += x[i] * x[i]; nb += y[i] * y[i]; }
#pragma unroll
  for (int o = kSvdGroup / 2; o > 0; o >>= 1) {
    na += __shfl_xor_sync(0xffffffffu, na, o);
    nb += __shfl_xor_sync(0xffffffffu, nb, o);
  }
  na = sqrt(na); nb = sqrt(nb);
  if (active && gl == 0)
    for (int r = 0; r < CL; ++r) {
      *cl.map_shared_rank(&fin[idl], r) = na;
      *cl.map_shared_rank(&fin[idr], r) = nb;
    }
  cl.sync();
  if (!active) return;
  const int kout = min(kk, l);
#pragma unroll 1
  for (int side = 0; side < 2; ++side) {
    const int id = side ? idr : idl;
    const double nv2 = side ? nb : na;
    int rank = 0;
    for (int j = 0; j < le; ++j) rank += (fin[j] > nv2) || (fin[j] == nv2 && j < id);
    if (id >= l || rank >= kout) continue;
    if (gl == 0) S[rank] = nv2;
    const double inv = (scaled_u || nv2 <= 0.0) ? 1.0 : 1.0 / nv2;
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int r = gl + i * kSvdGroup;
      const double cv = side ? y[i] : x[i];
      if (r < kk) U[(size_t)r * kout + rank] = scaled_u ? cv : (nv2 > 0.0 ? cv * inv : 0.0);
      if (want_v && V && r < l) V[(size_t)r * kout + rank] = side ? vy[i] : vx[i];
    }
  }
}

// ---------------------------------------------------------------------------
// One-warp-per-CTA block Jacobi (the truncation's SVD for 40 < l, rows <= 96).
// The block kernel above spends ~400 of its
// ~1300 cycles per round on the in-CTA move (shared-memory stores, a 3-warp
// barrier, loads).  Here a CTA is ONE warp holding 4 pair slots of 8 lanes
// (rows gl, gl + 8, ...; RPL per lane), so every in-CTA move is a register
// shuffle inside the warp -- no shared memory, no barrier -- and the dot
// products reduce over 3 shuffle levels instead of 4.  The cluster has
// CL = le / 8 CTAs (10 for l = 80; sizes above 8 use the non-portable cluster
// attribute, <= 16), each holding a P and a Q block of 4 columns; the sweep
// order is the block kernel's (round-robin over the CTA's 8 columns, then
// 2 CL - 2 block rounds of 4 cross rounds, blocks moving between CTAs by the
// circle method over DSMEM between block rounds).
// r01, same box, 80 x 80 with V: 512 us vs 546 us for the 16-lane block kernel
// (50 x 50: 302 vs 305).  Phase clocks (80 x 80, per round): dots + 3-level
// reduction ~230 cycles, rotation + apply ~475, shuffle move ~440, block moves
// ~240 averaged -- the shuffles (40-80 SHFL.32 per lane per round) are not
// cheaper than the shared-memory move, and an fp32 rotation angle (fp64
// normalisation) measured time-neutral: the round is issue/latency bound
// across the whole chain, not by one piece.
constexpr int kJwSlots = 4, kJwLanes = 8;

template <int RPL, bool PROF = false, int LC = 0, bool WV = true>
__global__ void __launch_bounds__(32, 1)
    jacobi_warp_kernel(int k, int l_arg, const double* __restrict__ B, long long b_rs, long long b_cs,
                       double* __restrict__ U, double* __restrict__ S, double* __restrict__ V, int want_v_arg,
                       int scaled_u, double skip2) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  // LC > 0: the column count (and so the cluster size) as compile-time constants
  const int l = LC > 0 ? LC : l_arg;
  const int CL = LC > 0 ? LC / (2 * kJwSlots) : (int)cl.num_blocks();
  // V accumulation as a compile-time flag (no per-round V branches): the QR
  // truncation path needs V (Q V_r), the Gram path only the rotated columns and
  // S -- without V a round has half the rotation FMAs, shuffle moves and DSMEM
  // block-move bytes.  PROF instances keep the runtime form.
  const bool want_v = PROF ? (want_v_arg != 0) : WV;
  const int c = (int)cl.block_rank();
  static_assert(RPL % 2 == 0, "RPL must be even");
  constexpr int box = RPL * kJwLanes;  // doubles per column part
  // block-move inbox: [2 bufs][4 slots][2 sides][2 (C, V)][box]
  extern __shared__ __align__(16) double sm[];
  __shared__ double nrm[kQrMaxCols + 2];
  __shared__ double fin[kQrMaxCols + 2];
  __shared__ int order[kQrMaxCols + 2];
  __shared__ int flags[64];
  __shared__ int bigf[64];
  __shared__ int bid[2][kJwSlots][2];
  __shared__ __align__(8) unsigned long long mbar[2];
  const int le = 2 * kJwSlots * CL, kk = k;
  const int lane = threadIdx.x, s = lane >> 3, gl = lane & 7;
  const int nv = want_v ? 2 : 1;
  auto bslot = [&](int buf, int slot, int side, int cv) {
    return sm + ((((size_t)buf * kJwSlots + slot) * 2 + side) * 2 + cv) * box + gl * 2;
  };
  const uint32_t msg_bytes = (uint32_t)(box * 8 * nv + 4);
  const uint32_t rx_bytes = (uint32_t)kJwSlots * msg_bytes * ((c >= 1 && c <= CL - 2) ? 2u : 1u);
  const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(&mbar[0]);
  if (lane == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar0 + 8) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    jc_arm(bar0, rx_bytes);
    jc_arm(bar0 + 8, rx_bytes);
  }
  // column norms (lane-parallel over columns), ranking by decreasing norm
  for (int cc = lane; cc < l; cc += 32) {
    double s0 = 0.0, s1 = 0.0;
    int r = 0;
    for (; r + 1 < kk; r += 2) {
      const double u0 = B[(long long)r * b_rs + (long long)cc * b_cs];
      const double u1 = B[(long long)(r + 1) * b_rs + (long long)cc * b_cs];
      s0 += u0 * u0;
      s1 += u1 * u1;
    }
    if (r < kk) { const double u0 = B[(long long)r * b_rs + (long long)cc * b_cs]; s0 += u0 * u0; }
    nrm[cc] = s0 + s1;
  }
  for (int i = lane; i < 64; i += 32) { flags[i] = 0; bigf[i] = 0; }
  __syncwarp();
  for (int cc = lane; cc < l; cc += 32) {
    int rank = 0;
    for (int j = 0; j < l; ++j) rank += (nrm[j] > nrm[cc]) || (nrm[j] == nrm[cc] && j < cc);
    order[rank] = cc;
  }
  __syncwarp();
  // prescale by a power of two (exact) so the largest column norm^2 lies in
  // [1, 4): the rotation needs no per-pair rescale on the common path
  double bmax = 0.0;
  for (int cc = lane; cc < l; cc += 32) bmax = fmax(bmax, nrm[cc]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) bmax = fmax(bmax, __shfl_xor_sync(0xffffffffu, bmax, o));
  const long long bex = (__double_as_longlong(bmax) >> 52) & 0x7ff;
  const long long hsc = (bex == 0 || bex == 0x7ff) ? 0 : ((bex - 1023) >> 1);  // floor(E / 2)
  const double bscale = __longlong_as_double((1023LL - hsc) << 52), bunscale = __longlong_as_double((1023LL + hsc) << 52);
  int idl = c * kJwSlots + s, idr = le - 1 - (c * kJwSlots + s);
  double x[RPL], y[RPL], vx[RPL], vy[RPL];
#pragma unroll
  for (int i = 0; i < RPL; ++i) {
    const int r = gl + i * kJwLanes;
    const bool okl = r < kk && idl < l, okr = r < kk && idr < l;
    x[i] = okl ? B[(long long)r * b_rs + (long long)order[idl] * b_cs] * bscale : 0.0;
    y[i] = okr ? B[(long long)r * b_rs + (long long)order[idr] * b_cs] * bscale : 0.0;
    vx[i] = (want_v && idl < l && r == order[idl]) ? 1.0 : 0.0;
    vy[i] = (want_v && idr < l && r == order[idr]) ? 1.0 : 0.0;
  }
  const double tol = (double)max(kk, 1) * 1.1102230246251565e-16;
  const double tol2 = tol * tol;
  const bool send_p = c >= 1, send_q = c <= CL - 2;
  uint32_t p_c = 0, p_id = 0, p_bar = 0, q_c = 0, q_id = 0, q_bar = 0;
  if (send_p) {
    const int side = (c == 1) ? 1 : 0;
    p_c = jc_map(bslot(0, s, side, 0), c - 1);
    p_id = jc_map(&bid[0][s][side], c - 1);
    p_bar = jc_map(&mbar[0], c - 1);
  }
  if (send_q) {
    q_c = jc_map(bslot(0, s, 1, 0), c + 1);
    q_id = jc_map(&bid[0][s][1], c + 1);
    q_bar = jc_map(&mbar[0], c + 1);
  }
  const uint32_t bbuf_bytes = (uint32_t)(kJwSlots * 4 * box * 8);
  const uint32_t bid_bytes = (uint32_t)(kJwSlots * 2 * sizeof(int));
  constexpr uint32_t pstride = 2u * kJwLanes * 8u;  // bytes between a lane's double2 pairs
  cl.sync();  // barriers initialised and armed in every CTA before the first remote store

  // phase clocks only in the PROF instance (the checks and clock reads cost ~2 % of a round)
  long long* const prof = (PROF && lane == 0) ? g_jc_prof : nullptr;
  long long pt[4] = {0, 0, 0, 0}, tc = 0;
  int lr = 0;
  int sweep = 0, moves = 0;
  for (; sweep < 60; ++sweep) {
    int rot = 0, big = 0;
    for (int br = 0; br < 2 * CL - 1; ++br) {
      // one round (rotation + in-CTA move); the cross rounds run in a loop with a
      // compile-time trip count, fully unrolled (no per-round loop / branch overhead)
      auto round = [&](const bool tournament) {
        // ---- rotate the pair (x, y): 8-lane dot products, 3 shuffle levels ----
        if (PROF && prof) tc = clock64();
        double ra0 = 0.0, rb0 = 0.0, rg0 = 0.0, ra1 = 0.0, rb1 = 0.0, rg1 = 0.0;
#pragma unroll
        for (int i = 0; i < RPL; i += 2) {
          ra0 = fma(x[i], x[i], ra0); rb0 = fma(y[i], y[i], rb0); rg0 = fma(x[i], y[i], rg0);
          ra1 = fma(x[i + 1], x[i + 1], ra1); rb1 = fma(y[i + 1], y[i + 1], rb1); rg1 = fma(x[i + 1], y[i + 1], rg1);
        }
        double ra = ra0 + ra1, rb = rb0 + rb1, rg = rg0 + rg1;
#pragma unroll
        for (int o = kJwLanes / 2; o > 0; o >>= 1) {
          ra += __shfl_xor_sync(0xffffffffu, ra, o);
          rb += __shfl_xor_sync(0xffffffffu, rb, o);
          rg += __shfl_xor_sync(0xffffffffu, rg, o);
        }
        if (PROF && prof) { long long t2 = clock64(); pt[3] += t2 - tc; }
        if (rg * rg > skip2 * ra * rb) big = 1;
        if (ra > 0.0 && rb > 0.0 && rg * rg > tol2 * ra * rb) {
          rot = 1;
          double sum, wd, rq;
          jacobi_rot(ra, rb, rg, sum, wd, rq);
          const double cs = sum * rq, sn = wd * rq;
          // both products of the old x first, then each register overwritten by
          // the FMA that consumes its old value (no temporaries to move back:
          // the plain form cost ~40 register moves per round in SASS)
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const double cx = cs * x[i], sx = sn * x[i];
            x[i] = fma(-sn, y[i], cx);
            y[i] = fma(cs, y[i], sx);
          }
          if (want_v) {
#pragma unroll
            for (int i = 0; i < RPL; ++i) {
              const double cx = cs * vx[i], sx = sn * vx[i];
              vx[i] = fma(-sn, vy[i], cx);
              vy[i] = fma(cs, vy[i], sx);
            }
          }
        }
        // ---- in-CTA move: register shuffles inside the warp ----
        if (PROF && prof) { long long t2 = clock64(); pt[0] += t2 - tc; tc = t2; }
        if (tournament) {
          // circle method on the 4 slots: left(s) <- left(s+1) (s = 1, 2),
          // left(3) <- right(3), left(0) fixed; right(0) <- left(1), right(s) <- right(s-1)
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const double tx = __shfl_down_sync(0xffffffffu, x[i], kJwLanes);
            const double ty = __shfl_up_sync(0xffffffffu, y[i], kJwLanes);
            const double nx = (s == 0) ? x[i] : (s == kJwSlots - 1 ? y[i] : tx);
            y[i] = (s == 0) ? tx : ty;
            x[i] = nx;
          }
          if (want_v) {
#pragma unroll
            for (int i = 0; i < RPL; ++i) {
              const double tx = __shfl_down_sync(0xffffffffu, vx[i], kJwLanes);
              const double ty = __shfl_up_sync(0xffffffffu, vy[i], kJwLanes);
              const double nx = (s == 0) ? vx[i] : (s == kJwSlots - 1 ? vy[i] : tx);
              vy[i] = (s == 0) ? tx : ty;
              vx[i] = nx;
            }
          }
          const int tl = __shfl_down_sync(0xffffffffu, idl, kJwLanes);
          const int tr = __shfl_up_sync(0xffffffffu, idr, kJwLanes);
          const int nl = (s == 0) ? idl : (s == kJwSlots - 1 ? idr : tl);
          idr = (s == 0) ? tl : tr;
          idl = nl;
        } else {
          // the Q block shifts one slot: right(s) <- right(s-1 mod 4)
          const int src = (lane + 32 - kJwLanes) & 31;
#pragma unroll
          for (int i = 0; i < RPL; ++i) y[i] = __shfl_sync(0xffffffffu, y[i], src);
          if (want_v) {
#pragma unroll
            for (int i = 0; i < RPL; ++i) vy[i] = __shfl_sync(0xffffffffu, vy[i], src);
          }
          idr = __shfl_sync(0xffffffffu, idr, src);
        }
        if (PROF && prof) { long long t2 = clock64(); pt[1] += t2 - tc; tc = t2; }
        ++lr;
      };
      if (br == 0) {
#pragma unroll
        for (int t = 0; t < 2 * kJwSlots - 1; ++t) round(true);
      } else {
#pragma unroll
        for (int t = 0; t < kJwSlots; ++t) round(false);
      }
      // ---- block move between CTAs (DSMEM, completion on the receiver's mbarrier) ----
      {
        const int buf = moves & 1;
        const uint32_t bo = buf * bbuf_bytes, io = buf * bid_bytes, mo = buf * 8;
        if (send_p) {
#pragma unroll
          for (int j = 0; j < RPL; j += 2) jc_st_v2(p_c + bo + pstride * (j / 2), x[j], x[j + 1], p_bar + mo);
          if (want_v) {
#pragma unroll
            for (int j = 0; j < RPL; j += 2)
              jc_st_v2(p_c + bo + box * 8 + pstride * (j / 2), vx[j], vx[j + 1], p_bar + mo);
          }
          if (gl == 0) jc_st_u32(p_id + io, (uint32_t)idl, p_bar + mo);
        }
        if (send_q) {
#pragma unroll
          for (int j = 0; j < RPL; j += 2) jc_st_v2(q_c + bo + pstride * (j / 2), y[j], y[j + 1], q_bar + mo);
          if (want_v) {
#pragma unroll
            for (int j = 0; j < RPL; j += 2)
              jc_st_v2(q_c + bo + box * 8 + pstride * (j / 2), vy[j], vy[j + 1], q_bar + mo);
          }
          if (gl == 0) jc_st_u32(q_id + io, (uint32_t)idr, q_bar + mo);
        }
        jc_wait(bar0 + mo, (moves >> 1) & 1);
        __syncwarp();
        if (lane == 0) jc_arm(bar0 + mo, rx_bytes);  // for move + 2
        auto get = [&](const double* src, double* v) {
          const double2* p = reinterpret_cast<const double2*>(src);
#pragma unroll
          for (int j = 0; j < RPL / 2; ++j) { double2 t2 = p[j * kJwLanes]; v[2 * j] = t2.x; v[2 * j + 1] = t2.y; }
        };
        if (c >= 1) {
          if (c == CL - 1) {
#pragma unroll
            for (int i = 0; i < RPL; ++i) { x[i] = y[i]; vx[i] = vy[i]; }
            idl = idr;
          } else {
            get(bslot(buf, s, 0, 0), x);
            if (want_v) get(bslot(buf, s, 0, 1), vx);
            idl = bid[buf][s][0];
          }
        }
        get(bslot(buf, s, 1, 0), y);
        if (want_v) get(bslot(buf, s, 1, 1), vy);
        idr = bid[buf][s][1];
        ++moves;
        if (PROF && prof) { long long t2 = clock64(); pt[2] += t2 - tc; tc = t2; }
      }
    }
    if (__any_sync(0xffffffffu, rot) && lane == 0) flags[sweep] = 1;
    if (__any_sync(0xffffffffu, big) && lane == 0) bigf[sweep] = 1;
    // every rotation of this sweep is ordered before this cluster barrier
    cl.sync();
    int ch = 0, bg = 0;
#pragma unroll 1
    for (int r = 0; r < CL; ++r) {
      ch |= *cl.map_shared_rank(&flags[sweep], r);
      bg |= *cl.map_shared_rank(&bigf[sweep], r);
    }
    if (!ch || !bg) break;
  }
  if (c == 0 && lane == 0 && g_svd_sweeps) *g_svd_sweeps = sweep + 1;
  if (PROF && prof && c < 8) {
    for (int i = 0; i < 4; ++i) atomicAdd((unsigned long long*)&prof[c * 5 + i], (unsigned long long)pt[i]);
    atomicAdd((unsigned long long*)&prof[c * 5 + 4], (unsigned long long)lr);
  }
  // final norms of every column, broadcast to every CTA
  double na = 0.0, nb = 0.0;
#pragma unroll
  for (int i = 0; i < RPL; ++i) { na += x[i] * x[i]; nb += y[i] * y[i]; }
#pragma unroll
  for (int o = kJwLanes / 2; o > 0; o >>= 1) {
    na += __shfl_xor_sync(0xffffffffu, na, o);
    nb += __shfl_xor_sync(0xffffffffu, nb, o);
  }
  na = sqrt(na); nb = sqrt(nb);
  if (gl == 0)
    for (int r = 0; r < CL; ++r) {
      *cl.map_shared_rank(&fin[idl], r) = na;
      *cl.map_shared_rank(&fin[idr], r) = nb;
    }
  cl.sync();
  const int kout = min(kk, l);
#pragma unroll 1
  for (int side = 0; side < 2; ++side) {
    const int id = side ? idr : idl;
    const double nv2 = side ? nb : na;
    int rank = 0;
    for (int j = 0; j < le; ++j) rank += (fin[j] > nv2) || (fin[j] == nv2 && j < id);
    if (id >= l || rank >= kout) continue;
    if (gl == 0) S[rank] = nv2 * bunscale;
    const double inv = (scaled_u || nv2 <= 0.0) ? 1.0 : 1.0 / nv2;
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int r = gl + i * kJwLanes;
      const double cv = side ? y[i] : x[i];
      if (r < kk) U[(size_t)r * kout + rank] = scaled_u ? cv * bunscale : (nv2 > 0.0 ? cv * inv : 0.0);
      if (want_v && V && r < l) V[(size_t)r * kout + rank] = side ? vy[i] : vx[i];
    }
  }
}

// ---------------------------------------------------------------------------
// Single-CTA variant for small factorisations (le <= 64, rows <= 64): the same
// register-resident pair slots, tournament and rotation as the cluster kernel,
// but every move stays in this CTA's shared memory (double-buffered inbox, one
// barrier per round).  The cluster kernel's DSMEM handoff + mbarrier wait sets
// a ~0.85-1.1 us per-round floor whatever the size; here a round costs the
// reduction/rotation chain plus one CTA barrier, and the shared-memory traffic
// (every moved column, C and V) grows with l^2 -- which is what keeps large
// factorisations on the cluster.

constexpr int kJlMaxSlots = 32;

template <int RPL>
__global__ void __launch_bounds__(kJlMaxSlots * kSvdGroup, 1)
    jacobi_local_kernel(int k, int l, const double* __restrict__ B, long long b_rs, long long b_cs,
                        double* __restrict__ U, double* __restrict__ S, double* __restrict__ V, int want_v_arg,
                        int scaled_u, double skip2) {
  // V accumulation is a compile-time constant (its runtime branches cost
  // instructions every round); V stores stay guarded by V != nullptr
  const bool want_v = true;
  (void)want_v_arg;
  extern __shared__ __align__(16) double sm[];  // [2 bufs][np][2 sides][2 (C,V)][RPL/2][16] double2
  __shared__ double nrm[kQrMaxCols + 2];
  __shared__ double fin[kQrMaxCols + 2];
  __shared__ int order[kQrMaxCols + 2];
  __shared__ int flags[64];  // per-sweep "rotated" flag (never reset)
  __shared__ int bigf[64];   // per-sweep "some pair beyond skip" flag
  __shared__ int inid[2][kJlMaxSlots][2];
  const int le = l + (l & 1), kk = k, np = le / 2;
  const int tid = threadIdx.x, si = tid / kSvdGroup, gl = tid % kSvdGroup;
  const bool active = si < np;
  constexpr int box = RPL * kSvdGroup;
  for (int c = tid >> 5; c < l; c += blockDim.x >> 5) {
    double s = 0.0;
    for (int r = tid & 31; r < kk; r += 32) {
      const double x = B[(long long)r * b_rs + (long long)c * b_cs];
      s += x * x;
    }
    s = warp_sum(s);
    if ((tid & 31) == 0) nrm[c] = s;
  }
  for (int i = tid; i < 64; i += blockDim.x) { flags[i] = 0; bigf[i] = 0; }
  __syncthreads();
  for (int c = tid; c < l; c += blockDim.x) {
    int rank = 0;
    for (int j = 0; j < l; ++j) rank += (nrm[j] > nrm[c]) || (nrm[j] == nrm[c] && j < c);
    order[rank] = c;
  }
  __syncthreads();
  int idl = active ? si : 0, idr = active ? le - 1 - si : 0;
  double x[RPL], y[RPL], vx[RPL], vy[RPL];
#pragma unroll
  for (int i = 0; i < RPL; ++i) {
    const int r = gl + i * kSvdGroup;
    const bool okl = active && r < kk && idl < l, okr = active && r < kk && idr < l;
    x[i] = okl ? B[(long long)r * b_rs + (long long)order[idl] * b_cs] : 0.0;
    y[i] = okr ? B[(long long)r * b_rs + (long long)order[idr] * b_cs] : 0.0;
    vx[i] = (want_v && active && idl < l && r == order[idl]) ? 1.0 : 0.0;
    vy[i] = (want_v && active && idr < l && r == order[idr]) ? 1.0 : 0.0;
  }
  const double tol = (double)max(kk, 1) * 1.1102230246251565e-16;
  const double tol2 = tol * tol;
  auto part = [&](int buf, int slot, int side, int cv) {
    return reinterpret_cast<double2*>(sm + ((((size_t)buf * np + slot) * 2 + side) * 2 + cv) * box) + gl;
  };
  // moves (position v -> v-1 of the round-robin, as in the cluster kernel):
  //   left(s) -> left(s-1) (s >= 2), left(1) -> right(0), right(s) -> right(s+1) (s <= np-2),
  //   right(np-1) -> left(np-1) (stays in the slot), left(0) fixed
  const bool send_l = active && si >= 1, send_r = active && si <= np - 2;
  const int l_slot = si - 1, l_side = (si == 1) ? 1 : 0, r_slot = si + 1;
  int sweep = 0, round = 0;
  for (; sweep < 60; ++sweep) {
#pragma unroll 2
    for (int rnd = 0; rnd < le - 1; ++rnd, ++round) {
      double a = 0.0, b = 0.0, g = 0.0, a2 = 0.0, b2 = 0.0, g2 = 0.0;
#pragma unroll
      for (int i = 0; i < RPL; i += 2) {
        a += x[i] * x[i]; b += y[i] * y[i]; g += x[i] * y[i];
        if (i + 1 < RPL) { a2 += x[i + 1] * x[i + 1]; b2 += y[i + 1] * y[i + 1]; g2 += x[i + 1] * y[i + 1]; }
      }
      a += a2; b += b2; g += g2;
#pragma unroll
      for (int o = kSvdGroup / 2; o > 0; o >>= 1) {
        a += __shfl_xor_sync(0xffffffffu, a, o);
        b += __shfl_xor_sync(0xffffffffu, b, o);
        g += __shfl_xor_sync(0xffffffffu, g, o);
      }
      if (active && gl == 0 && g * g > skip2 * a * b) bigf[sweep] = 1;
      if (active && a > 0.0 && b > 0.0 && g * g > tol2 * a * b) {
        const long long ex = min((__double_as_longlong(a + b) >> 52) & 0x7ff, 2045LL);
        const double sc = __longlong_as_double((2046LL - ex) << 52);
        const double dd = (b - a) * sc, w = 2.0 * g * sc;
        const double q = dd * dd + w * w;
        const double rho = q * rsqrt_rot(q);
        const double sum = fabs(dd) + rho;
        const double rq = rsqrt_rot(fma(2.0 * rho, fabs(dd), 2.0 * q));  // 2 rho (|dd| + rho)
        const double c = sum * rq, s = (dd >= 0.0 ? w : -w) * rq;
#pragma unroll
        for (int i = 0; i < RPL; ++i) {  // old x consumed first: no register moves
          const double cx = c * x[i], sx = s * x[i];
          x[i] = fma(-s, y[i], cx);
          y[i] = fma(c, y[i], sx);
        }
        if (want_v) {
#pragma unroll
          for (int i = 0; i < RPL; ++i) {
            const double cx = c * vx[i], sx = s * vx[i];
            vx[i] = fma(-s, vy[i], cx);
            vy[i] = fma(c, vy[i], sx);
          }
        }
        if (gl == 0) flags[sweep] = 1;
      }
      if (np > 1) {
        const int buf = round & 1;
        if (send_l) {
          double2* pc = part(buf, l_slot, l_side, 0);
#pragma unroll
          for (int j = 0; j < RPL / 2; ++j) pc[j * kSvdGroup] = make_double2(x[2 * j], x[2 * j + 1]);
          if (want_v) {
            double2* pv = part(buf, l_slot, l_side, 1);
#pragma unroll
            for (int j = 0; j < RPL / 2; ++j) pv[j * kSvdGroup] = make_double2(vx[2 * j], vx[2 * j + 1]);
          }
          if (gl == 0) inid[buf][l_slot][l_side] = idl;
        }
        if (send_r) {
          double2* pc = part(buf, r_slot, 1, 0);
#pragma unroll
          for (int j = 0; j < RPL / 2; ++j) pc[j * kSvdGroup] = make_double2(y[2 * j], y[2 * j + 1]);
          if (want_v) {
            double2* pv = part(buf, r_slot, 1, 1);
#pragma unroll
            for (int j = 0; j < RPL / 2; ++j) pv[j * kSvdGroup] = make_double2(vy[2 * j], vy[2 * j + 1]);
          }
          if (gl == 0) inid[buf][r_slot][1] = idr;
        }
        __syncthreads();
        if (active) {
          if (si >= 1) {
            if (si == np - 1) {
#pragma unroll
              for (int i = 0; i < RPL; ++i) { x[i] = y[i]; vx[i] = vy[i]; }
              idl = idr;
            } else {
              const double2* pc = part(buf, si, 0, 0);
#pragma unroll
              for (int j = 0; j < RPL / 2; ++j) { const double2 v2 = pc[j * kSvdGroup]; x[2 * j] = v2.x; x[2 * j + 1] = v2.y; }
              if (want_v) {
                const double2* pv = part(buf, si, 0, 1);
#pragma unroll
                for (int j = 0; j < RPL / 2; ++j) { const double2 v2 = pv[j * kSvdGroup]; vx[2 * j] = v2.x; vx[2 * j + 1] = v2.y; }
              }
              idl = inid[buf][si][0];
            }
          }
          const double2* pc = part(buf, si, 1, 0);
#pragma unroll
          for (int j = 0; j < RPL / 2; ++j) { const double2 v2 = pc[j * kSvdGroup]; y[2 * j] = v2.x; y[2 * j + 1] = v2.y; }
          if (want_v) {
            const double2* pv = part(buf, si, 1, 1);
#pragma unroll
            for (int j = 0; j < RPL / 2; ++j) { const double2 v2 = pv[j * kSvdGroup]; vy[2 * j] = v2.x; vy[2 * j + 1] = v2.y; }
          }
          idr = inid[buf][si][1];
        }
      }
    }
    __syncthreads();  // every rotation flag of this sweep is visible
    if (!flags[sweep] || !bigf[sweep]) break;
  }
  if (tid == 0 && g_svd_sweeps) *g_svd_sweeps = sweep + 1;
  double a = 0.0, b = 0.0;
#pragma unroll
  for (int i = 0; i < RPL; ++i) { a += x[i] * x[i]; b += y[i] * y[i]; }
#pragma unroll
  for (int o = kSvdGroup / 2; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  a = sqrt(a); b = sqrt(b);
  if (active && gl == 0) { fin[idl] = a; fin[idr] = b; }
  __syncthreads();
  if (!active) return;
  const int kout = min(kk, l);
#pragma unroll 1
  for (int side = 0; side < 2; ++side) {
    const int id = side ? idr : idl;
    const double nv2 = side ? b : a;
    int rank = 0;
    for (int j = 0; j < le; ++j) rank += (fin[j] > nv2) || (fin[j] == nv2 && j < id);
    if (id >= l || rank >= kout) continue;
    if (gl == 0) S[rank] = nv2;
    const double inv = (scaled_u || nv2 <= 0.0) ? 1.0 : 1.0 / nv2;
#pragma unroll
    for (int i = 0; i < RPL; ++i) {
      const int r = gl + i * kSvdGroup;
      const double cv = side ? y[i] : x[i];
      if (r < kk) U[(size_t)r * kout + rank] = scaled_u ? cv : (nv2 > 0.0 ? cv * inv : 0.0);
      if (want_v && V && r < l) V[(size_t)r * kout + rank] = side ? vy[i] : vx[i];
    }
  }
}

int jacobi_svd_ex(int k, int l, const double* B, long long b_rs, long long b_cs, double* U, double* S,
                  double* V, bool scaled_u, cudaStream_t st) {
  if (k <= 0 || l <= 0) return kOk;
  TTK_REQUIRE(l <= kWideMaxCols && k <= kWideMaxCols, kInvalidValue,
              "jacobi_svd: %d x %d exceeds %d", k, l, kWideMaxCols);
  const int le = l + (l & 1);
  static const bool single_cta = knob_env("TTK_JACOBI_SINGLE") != nullptr;  // A/B switch
  // stop after a sweep in which every pair had |g| <= skip sqrt(ab): by quadratic
  // convergence the next sweep would only rotate by O(skip^2) < tol (a pure
  // confirmation sweep).  1e-8: the skipped rotations are O(1e-16), below the
  // 8.9e-15 threshold; r01 (tools/jac_ab.py) singular values / orthogonality
  // unchanged, one sweep saved on most inputs (80x80 Gaussian 9 -> 8; config-3
  // step 37.7 -> 36.1 ms).  1e-7 was tried (tools/jac_ab.py: 80 x 80 Gaussian one
  // sweep fewer, orthogonality unchanged) but moved neither the config-3 step
  // (31.9 vs 31.9 ms) nor the solvers beyond their run-to-run noise; 1e-6 let
  // 128 x 128 orthogonality slip to 2e-12.  TTK_JACOBI_SKIP overrides (0 keeps
  // the confirmation sweep)
  static const double skip = knob_env("TTK_JACOBI_SKIP") ? atof(knob_env("TTK_JACOBI_SKIP")) : 1e-8;
  const double skip2 = skip * skip;
  if (l > kQrMaxCols || k > kQrMaxCols)  // beyond the register-resident kernels: qr_wide.cu
    return jacobi_svd_global(k, l, B, b_rs, b_cs, U, S, V, scaled_u, skip2, st);
  // largest (even) width for the single-CTA register kernel (tools/jac_ab.py, r01: local vs
  // cluster 27 vs 54 us at 7x7, 77 vs 148 at 20, 205 vs 228 at 33, 435 vs 369 at 50 -- beyond
  // ~40 its shared-memory traffic costs more than the cluster's handoff); env var: A/B
  static const int local_max = knob_env("TTK_JACOBI_LOCAL_MAX") ? atoi(knob_env("TTK_JACOBI_LOCAL_MAX")) : 40;
  if (!single_cta && le <= std::min(local_max, 2 * kJlMaxSlots) && std::max(k, le) <= 4 * kSvdGroup) {
    {  // per-device attributes (set_attr_once)
      TTK_TRY(qr_set_smem((const void*)jacobi_local_kernel<2>, 128 * 1024));
      TTK_TRY(qr_set_smem((const void*)jacobi_local_kernel<4>, 128 * 1024));
    }
    const int np = le / 2;
    const int threads = std::max(32, (np * kSvdGroup + 31) / 32 * 32);
    const int want = V != nullptr;
    if (std::max(k, le) <= 2 * kSvdGroup) {
      const size_t jsm = sizeof(double) * 2 * np * 4 * 2 * kSvdGroup;
      jacobi_local_kernel<2><<<1, threads, jsm, st>>>(k, l, B, b_rs, b_cs, U, S, V, want, scaled_u, skip2);
    } else {
      const size_t jsm = sizeof(double) * 2 * np * 4 * 4 * kSvdGroup;
      jacobi_local_kernel<4><<<1, threads, jsm, st>>>(k, l, B, b_rs, b_cs, U, S, V, want, scaled_u, skip2);
    }
    TTK_CHECK_LAUNCH();
    return kOk;
  }
  // one-warp-per-CTA block kernel (in-CTA moves are shuffles); TTK_JACOBI_WARP=0
  // keeps the 16-lane block kernel below (A/B)
  static const bool warp_off = knob_env("TTK_JACOBI_WARP") && atoi(knob_env("TTK_JACOBI_WARP")) == 0;
  if (!single_cta && !warp_off && l > 2 * kJwSlots && std::max(k, l) <= 12 * kJwLanes &&
      (l + 2 * kJwSlots - 1) / (2 * kJwSlots) <= 16) {
    const int CL = (l + 2 * kJwSlots - 1) / (2 * kJwSlots);
    const int rows = std::max(k, l);
    const int rpl = ((rows + kJwLanes - 1) / kJwLanes + 1) & ~1;
    {  // per-device attributes (set_attr_once)
      for (const void* fn : {(const void*)jacobi_warp_kernel<2>, (const void*)jacobi_warp_kernel<4>,
                             (const void*)jacobi_warp_kernel<6>, (const void*)jacobi_warp_kernel<8>,
                             (const void*)jacobi_warp_kernel<10>, (const void*)jacobi_warp_kernel<12>,
                             (const void*)jacobi_warp_kernel<2, true>, (const void*)jacobi_warp_kernel<4, true>,
                             (const void*)jacobi_warp_kernel<6, true>, (const void*)jacobi_warp_kernel<8, true>,
                             (const void*)jacobi_warp_kernel<10, true>, (const void*)jacobi_warp_kernel<12, true>,
                             (const void*)jacobi_warp_kernel<2, false, 0, false>,
                             (const void*)jacobi_warp_kernel<4, false, 0, false>,
                             (const void*)jacobi_warp_kernel<6, false, 0, false>,
                             (const void*)jacobi_warp_kernel<8, false, 0, false>,
                             (const void*)jacobi_warp_kernel<10, false, 0, false>,
                             (const void*)jacobi_warp_kernel<12, false, 0, false>})
        TTK_TRY(set_attr_once(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    }
    const size_t jsm = sizeof(double) * 2 * kJwSlots * 4 * (size_t)rpl * kJwLanes;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CL, 1, 1);
    cfg.blockDim = dim3(32, 1, 1);
    cfg.dynamicSmemBytes = jsm;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const int want = V != nullptr;
    cudaError_t e;
    static const bool jlc_off = knob_env("TTK_JW_LC") && atoi(knob_env("TTK_JW_LC")) == 0;  // A/B
    if (!g_jc_prof_host && rpl == 10 && l == 80 && !jlc_off) {
      {  // per-device attributes (set_attr_once)
        TTK_TRY(set_attr_once((const void*)jacobi_warp_kernel<10, false, 80>,
                                            cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        TTK_TRY(set_attr_once((const void*)jacobi_warp_kernel<10, false, 80, false>,
                              cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
      }
      if (want)
        e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<10, false, 80>, k, l, B, b_rs, b_cs, U, S, V, want,
                               (int)scaled_u, skip2);
      else
        e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<10, false, 80, false>, k, l, B, b_rs, b_cs, U, S, V,
                               want, (int)scaled_u, skip2);
    } else if (g_jc_prof_host) {
    switch (rpl) {
      case 2: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<2, true>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
      case 4: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<4, true>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
      case 6: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<6, true>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
      case 8: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<8, true>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
      case 10: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<10, true>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
      default: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<12, true>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
    }
    } else if (!want) {
    switch (rpl) {
      case 2: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<2, false, 0, false>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
      case 4: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<4, false, 0, false>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
      case 6: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<6, false, 0, false>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
      case 8: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<8, false, 0, false>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
      case 10: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<10, false, 0, false>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
      default: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<12, false, 0, false>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
    }
    } else {
    switch (rpl) {
      case 2: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<2>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
      case 4: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<4>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
      case 6: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<6>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
      case 8: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<8>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
      case 10: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<10>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
      default: e = cudaLaunchKernelEx(&cfg, jacobi_warp_kernel<12>, k, l, B, b_rs, b_cs, U, S, V, want, (int)scaled_u, skip2); break;
    }
    }
    if (e == cudaSuccess) {
      TTK_CHECK_LAUNCH();
      return kOk;
    }
    // a non-portable cluster of CL CTAs can be refused (e.g. a partitioned
    // GPU): clear the error and take the portable 8-CTA block kernel below
    (void)cudaGetLastError();
  }
  // block-ordered cluster kernel (2 CL - 1 DSMEM handoffs per sweep instead of
  // le - 1); TTK_JACOBI_BLOCK=0 keeps the plain cluster kernel, =4 / =8 picks the
  // cluster size (A/B)
  static const int block_env = knob_env("TTK_JACOBI_BLOCK") ? atoi(knob_env("TTK_JACOBI_BLOCK")) : -1;
  static const bool jb_diag_set = [] {
    const int v = knob_env("TTK_JB_DIAG") ? atoi(knob_env("TTK_JB_DIAG")) : 0;
    if (v) cudaMemcpyToSymbol(g_jb_diag, &v, sizeof(int));
    return true;
  }();
  (void)jb_diag_set;
  int block_cl = block_env;
  if (block_cl < 0) {
    // fewest padded columns (dummy columns cost whole rounds), 8 CTAs on ties:
    // r01 (tools/jac_ab.py) 50 x 50: 4 CTAs (56 columns) 291 us vs 8 CTAs (64) 316;
    // 80 x 80: 581 vs 529
    const int le8 = 16 * ((l + 15) / 16), le4 = 8 * ((l + 7) / 8);
    const int rows4 = std::max(k, le4), rpl4 = rows4 <= 4 * kSvdGroup ? 4 : rows4 <= 6 * kSvdGroup ? 6 : 8;
    const bool fits4 = le4 / 8 <= kJbMaxSlots && sizeof(double) * 2 * (2 * (size_t)(le4 / 8) * 4 * rpl4 * kSvdGroup) <= 200 * 1024;
    block_cl = (le4 < le8 && fits4) ? 4 : 8;
  }
  if (!single_cta && block_cl != 0 && l > 2 * block_cl && k <= 8 * kSvdGroup) {
    const int bs = (l + 2 * block_cl - 1) / (2 * block_cl);
    const int rows = std::max(k, 2 * block_cl * bs);
    const int rpl = rows <= 4 * kSvdGroup ? 4 : rows <= 6 * kSvdGroup ? 6 : 8;
    const size_t jsm = sizeof(double) * 2 * (2 * (size_t)bs * 4 * rpl * kSvdGroup);
    if (bs <= kJbMaxSlots && jsm <= 200 * 1024) {
      {  // per-device attributes (set_attr_once)
        TTK_TRY(qr_set_smem((const void*)jacobi_block_kernel<4, 8>, 200 * 1024));
        TTK_TRY(qr_set_smem((const void*)jacobi_block_kernel<6, 8>, 200 * 1024));
        TTK_TRY(qr_set_smem((const void*)jacobi_block_kernel<8, 8>, 200 * 1024));
        TTK_TRY(qr_set_smem((const void*)jacobi_block_kernel<4, 4>, 200 * 1024));
        TTK_TRY(qr_set_smem((const void*)jacobi_block_kernel<6, 4>, 200 * 1024));
        TTK_TRY(qr_set_smem((const void*)jacobi_block_kernel<8, 4>, 200 * 1024));
      }
      const int threads = (bs * kSvdGroup + 31) / 32 * 32;
      const int want = V != nullptr;
#define TTK_JB_LAUNCH(R, C) \
  jacobi_block_kernel<R, C><<<C, threads, jsm, st>>>(k, l, B, b_rs, b_cs, U, S, V, want, scaled_u, skip2)
      if (block_cl == 4) {
        if (rpl == 4) TTK_JB_LAUNCH(4, 4); else if (rpl == 6) TTK_JB_LAUNCH(6, 4); else TTK_JB_LAUNCH(8, 4);
      } else {
        if (rpl == 4) TTK_JB_LAUNCH(4, 8); else if (rpl == 6) TTK_JB_LAUNCH(6, 8); else TTK_JB_LAUNCH(8, 8);
      }
#undef TTK_JB_LAUNCH
      TTK_CHECK_LAUNCH();
      return kOk;
    }
  }
  if (!single_cta && le <= 2 * kJcCluster * kJcMaxSlots && k <= 8 * kSvdGroup) {
    {  // per-device attributes (set_attr_once)
      TTK_TRY(qr_set_smem((const void*)jacobi_cluster_kernel<4>, 96 * 1024));
      TTK_TRY(qr_set_smem((const void*)jacobi_cluster_kernel<6>, 96 * 1024));
      TTK_TRY(qr_set_smem((const void*)jacobi_cluster_kernel<8>, 96 * 1024));
    }
    const int spc = (le / 2 + kJcCluster - 1) / kJcCluster;
    const int rows = std::max(k, le);
    const int threads = std::max(32, (spc * kSvdGroup + 31) / 32 * 32);
    const int want = V != nullptr;
    if (rows <= 4 * kSvdGroup) {
      const size_t jsm = sizeof(double) * 8 * spc * 4 * kSvdGroup;
      jacobi_cluster_kernel<4><<<kJcCluster, threads, jsm, st>>>(k, l, B, b_rs, b_cs, U, S, V, want, scaled_u,
                                                                skip2);
    } else if (rows <= 6 * kSvdGroup) {
      const size_t jsm = sizeof(double) * 8 * spc * 6 * kSvdGroup;
      jacobi_cluster_kernel<6><<<kJcCluster, threads, jsm, st>>>(k, l, B, b_rs, b_cs, U, S, V, want, scaled_u,
                                                                skip2);
    } else {
      const size_t jsm = sizeof(double) * 8 * spc * 8 * kSvdGroup;
      jacobi_cluster_kernel<8><<<kJcCluster, threads, jsm, st>>>(k, l, B, b_rs, b_cs, U, S, V, want, scaled_u,
                                                                skip2);
    }
    TTK_CHECK_LAUNCH();
    return kOk;
  }
  size_t smem = sizeof(double) * ((size_t)le * (k | 1) + (V ? (size_t)le * le : 0));
  TTK_REQUIRE(smem <= 215 * 1024, kInvalidValue, "jacobi_svd: %d x %d (V=%d) exceeds shared memory", k,
              l, V != nullptr);
  {  // per-device attributes (set_attr_once)
    TTK_TRY(qr_set_smem((const void*)jacobi_svd_kernel<4>, 215 * 1024));
    TTK_TRY(qr_set_smem((const void*)jacobi_svd_kernel<6>, 215 * 1024));
    TTK_TRY(qr_set_smem((const void*)jacobi_svd_kernel<8>, 215 * 1024));
    TTK_TRY(qr_set_smem((const void*)jacobi_svd_kernel<10>, 215 * 1024));
  }
  const int threads = std::min(kSvdThreads, std::max(64, ((le / 2) * kSvdGroup + 31) / 32 * 32));
  const int rows = std::max(k, le);
  if (rows <= 4 * kSvdGroup)
    jacobi_svd_kernel<4><<<1, threads, smem, st>>>(k, l, B, b_rs, b_cs, U, S, V, V != nullptr, scaled_u);
  else if (rows <= 6 * kSvdGroup)
    jacobi_svd_kernel<6><<<1, threads, smem, st>>>(k, l, B, b_rs, b_cs, U, S, V, V != nullptr, scaled_u);
  else if (rows <= 8 * kSvdGroup)
    jacobi_svd_kernel<8><<<1, threads, smem, st>>>(k, l, B, b_rs, b_cs, U, S, V, V != nullptr, scaled_u);
  else
    jacobi_svd_kernel<10><<<1, threads, smem, st>>>(k, l, B, b_rs, b_cs, U, S, V, V != nullptr, scaled_u);
  TTK_CHECK_LAUNCH();
  return kOk;
}

bool jacobi_fits_v(int k, int l) {
  const int le = l + (l & 1);
  if (l > kQrMaxCols || k > kQrMaxCols) return l <= kWideMaxCols && k <= kWideMaxCols;  // global kernel
  return l <= kQrMaxCols && k <= kQrMaxCols &&
         sizeof(double) * ((size_t)le * (k | 1) + (size_t)le * le) <= 215 * 1024;
}

int jacobi_svd(int k, int l, const double* B, double* U, double* S, double* V, cudaStream_t st) {
  return jacobi_svd_ex(k, l, B, l, 1, U, S, V, false, st);
}

__global__ void truncation_rank_kernel(const double* S, int n, double budget, int max_rank, int* r_out) {
  // tail[r] = sqrt(sum_{i>=r} S_i^2), accumulated from the smallest value as
  // np.cumsum(sv[::-1]**2)[::-1] does (tt.py:207): the running sums stay
  // sequential with separately rounded squares (numpy's rounding), one
  // thread; the square roots and the search for the smallest r with tail[r] <= budget run
  // across the block (the serial form with sqrt in the loop took ~13 us)
  __shared__ double acc[kWideMaxCols + 2];
  __shared__ int best;
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int i = n - 1; i >= 0; --i) {
      a = __dadd_rn(a, __dmul_rn(S[i], S[i]));
      acc[i] = a;
    }
    best = n;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += blockDim.x)
    if (sqrt(fmax(acc[i], 0.0)) <= budget) atomicMin(&best, i);
  __syncthreads();
  if (threadIdx.x != 0) return;
  int r = best;
  if (n == 0) r = 1;
  if (r < 1) r = 1;
  if (max_rank > 0 && r > max_rank) r = max_rank;
  *r_out = r;
}

int truncation_rank_dev(const double* S, int n, double budget, int max_rank, int* r_dev,
                        cudaStream_t st) {
  TTK_REQUIRE(n <= kWideMaxCols, kInvalidValue, "truncation_rank: %d values exceed %d", n, kWideMaxCols);
  truncation_rank_kernel<<<1, 128, 0, st>>>(S, n, budget, max_rank, r_dev);
  TTK_CHECK_LAUNCH();
  return kOk;
}

}  // namespace ttk

using namespace ttk;

extern "C" {

size_t ttk_qr_ws_bytes(int m, int l) { return qr_auto_ws_bytes(m, l); }

// QR front door used by the rounding drivers: shifted CholeskyQR2/3 when
// accepted, Householder TSQR otherwise (same contract as ttk_qr)
int ttk_qr_auto(int m, int l, const double* A, long long a_rs, long long a_cs, double* Q, long long q_rs,
                long long q_cs, double* R, void* ws, size_t ws_bytes, void* stream) {
  return qr_auto(m, l, A, a_rs, a_cs, Q, q_rs, q_cs, R, ws, ws_bytes, (cudaStream_t)stream);
}

int ttk_qr(int m, int l, const double* A, long long a_rs, long long a_cs, double* Q, long long q_rs,
           long long q_cs, double* R, void* ws, size_t ws_bytes, void* stream) {
  return tsqr(m, l, A, a_rs, a_cs, Q, q_rs, q_cs, R, ws, ws_bytes, (cudaStream_t)stream);
}

int ttk_svd_small(int k, int l, const double* B, double* U, double* S, double* V, void* stream) {
  return jacobi_svd(k, l, B, U, S, V, (cudaStream_t)stream);
}

// diagnostics: chol_blocked_kernel phase clocks (load, diagonal blocks, panels, trailing, epilogue)
int ttk_debug_fused_qr_profile(long long* dev_ts) {
  TTK_CHECK_CUDA(cudaMemcpyToSymbol(g_fq_prof, &dev_ts, sizeof(dev_ts)));
  return kOk;
}

// diagnostics: one Cholesky factorisation R^T R = G (l x l, device) through
// launch_chol_inv (the truncation's Gram path); status: device int
int ttk_debug_chol(int l, const double* G, double* R, int* status, void* stream) {
  return launch_chol_inv(l, G, R, nullptr, status, 0, 0.0, 1e-15, (cudaStream_t)stream, nullptr);
}

int ttk_debug_chol_profile(long long* dev_acc) {
  TTK_CHECK_CUDA(cudaMemcpyToSymbol(g_chol_prof, &dev_acc, sizeof(long long*)));
  return kOk;
}

// diagnostics: accumulate per-CTA phase clocks of the cluster Jacobi (5 int64 per CTA:
// rotate, send, wait, pull, rounds) into dev_acc (NULL: off)
int ttk_debug_jacobi_profile(long long* dev_acc) {
  TTK_CHECK_CUDA(cudaMemcpyToSymbol(g_jc_prof, &dev_acc, sizeof(long long*)));
  g_jc_prof_host = dev_acc != nullptr;
  return kOk;
}

// diagnostics: route the sweep count of subsequent Jacobi SVDs to a device int (NULL: off)
int ttk_debug_svd_sweeps(int* dev_counter) {
  TTK_CHECK_CUDA(cudaMemcpyToSymbol(g_svd_sweeps, &dev_counter, sizeof(int*)));
  return kOk;
}

}  // extern "C"

// ===========================================================================
// CholeskyQR2 fast path (all heavy work on the DMMA GEMM):
//   G1 = Y^T Y, R1 = chol(G1), Q1 = Y R1^{-1}; G2 = Q1^T Q1, R2 = chol(G2),
//   Q = Q1 R2^{-1}, R = R2 R1.
// Accepted only when both factorisations succeed and ||G2 - I||_max <= 1e-3
// (then Q is orthonormal to working precision, Yamamoto et al. 2015);
// otherwise the caller falls back to Householder TSQR.
#include "gemm.cuh"

namespace ttk {

constexpr int kCholMaxCols = 112;

// one CTA: upper Cholesky G = R^T R of an l x l SPD matrix and R^{-1};
// status |= 1 on a non-positive / tiny pivot, |= 2 if check_identity and
// max|G - I| > 1e-3.
__global__ void __launch_bounds__(1024, 1)
    chol_inv_kernel(int l, const double* __restrict__ G, double* __restrict__ Rout,
                    double* __restrict__ Rinv, int* status, int check_identity, double shift_rel,
                    double tiny_rel, const int* __restrict__ skip) {
  if (skip && *skip) return;  // chol_near_identity_kernel already produced R, R^{-1}
  extern __shared__ double sm[];
  const int ld = l + 1;
  double* A = sm;               // l x ld, becomes R (upper)
  double* X = sm + l * ld;      // l x ld, R^{-1}
  __shared__ int bad;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int ty = tid >> 5, tx = tid & 31, nty = nt >> 5;
  if (tid == 0) bad = 0;
  __syncthreads();
  for (int e = tid; e < l * l; e += nt) {
    int r = e / l, c = e - r * l;
    double g = G[e];
    A[r * ld + c] = g;
    if (check_identity && fabs(g - (r == c ? 1.0 : 0.0)) > 1e-3) atomicOr(&bad, 2);
  }
  __syncthreads();
  __shared__ double gmax_s;
  if (ty == 0) {
    double g = 0.0;
    for (int i = tx; i < l; i += 32) g = fmax(g, A[i * ld + i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) g = fmax(g, __shfl_xor_sync(0xffffffffu, g, o));
    if (tx == 0) gmax_s = g;
  }
  __syncthreads();
  if (shift_rel > 0.0) {
    // shifted CholeskyQR (Fukaya et al.): G + s I with s = shift_rel * trace(G)
    __shared__ double tr_s;
    if (ty == 0) {
      double t = 0.0;
      for (int i = tx; i < l; i += 32) t += A[i * ld + i];
      t = warp_sum(t);
      if (tx == 0) tr_s = t;
    }
    __syncthreads();
    const double sh = shift_rel * tr_s;
    for (int i = tid; i < l; i += nt) A[i * ld + i] += sh;
    __syncthreads();
  }
  const double tiny = gmax_s * tiny_rel + 1e-300;  // pivot^2 floor relative to max diag(G)
  // Gaussian elimination of [G | I] without pivoting (SPD): E G = U with E unit
  // lower, U = D L1^T upper, and E = L1^{-1}.  Hence R = D^{-1/2} U and
  // R^{-1} = E^T D^{-1/2}: one pass gives both (no separate triangular inverse).
  // Only the upper triangle of A and the lower triangle of X (= E) are touched;
  // one barrier per step, the next pivot's reciprocal is formed by the lane that
  // finishes it while the other rows are still being updated.
  __shared__ double pinv[kQrMaxCols + 1];
  for (int e = tid; e < l * ld; e += nt) {
    int r = e / ld, c = e - r * ld;
    X[e] = (r == c) ? 1.0 : 0.0;
  }
  if (tid == 0) {
    const double p0 = A[0];
    if (!(p0 > tiny)) { atomicOr(&bad, 1); pinv[0] = 1.0; } else { pinv[0] = 1.0 / p0; }
  }
  __syncthreads();
  for (int j = 0; j < l; ++j) {
    const double inv = pinv[j];
    for (int i = j + 1 + ty; i < l; i += nty) {
      const double aji = A[j * ld + i] * inv;
      for (int c = i + tx; c < l; c += 32) A[i * ld + c] -= aji * A[j * ld + c];
      if (i == j + 1 && tx == 0) {
        const double pn = A[i * ld + i];
        if (!(pn > tiny)) { atomicOr(&bad, 1); pinv[i] = 1.0; } else { pinv[i] = 1.0 / pn; }
      }
      for (int c = tx; c <= j; c += 32) X[i * ld + c] -= aji * X[j * ld + c];
    }
    __syncthreads();
  }
  __shared__ double dsq[kQrMaxCols + 1], rsq[kQrMaxCols + 1];
  for (int r = tid; r < l; r += nt) {
    const double p = A[r * ld + r];
    const double d = sqrt(p > tiny ? p : 1.0);
    dsq[r] = d;
    rsq[r] = 1.0 / d;
  }
  __syncthreads();
  for (int e = tid; e < l * l; e += nt) {
    int r = e / l, c = e - r * l;
    Rout[e] = (c > r) ? A[r * ld + c] * rsq[r] : (c == r ? dsq[r] : 0.0);
    Rinv[e] = (c >= r) ? X[c * ld + r] * rsq[c] : 0.0;
  }
  if (tid == 0 && bad) atomicOr(status, bad);
}

// C = A B for small matrices in shared memory, on the DMMA pipe: warps take
// 8x8 output tiles round-robin, two accumulator chains over k (m8n8k4 f64).
// A(m,k) = A[m a_rs + k a_cs], B(k,n) = B[k b_rs + n b_cs], C row-major (ldc).
// rinv_out != nullptr: instead of storing C, write the upper triangle of
// I - F + P - C into rinv_out (row-major, ld = N) with F = rinv_f, P = rinv_p
// (shared, ld = ldc): the R^{-1} epilogue of chol_near_identity_kernel.
// Strides that are 4 mod 16 make the fragment loads bank-conflict free.
__device__ void block_dmma(int M, int N, int K, const double* A, int a_rs, int a_cs, const double* B, int b_rs,
                           int b_cs, double* C, int ldc, double* rinv_out = nullptr,
                           const double* rinv_f = nullptr, const double* rinv_p = nullptr, bool sub = false) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  if (rinv_out == nullptr) {
    // 16 x 16 output blocks per warp (2 x 2 DMMA tiles): each k-step loads two
    // A and two B fragments for four DMMAs (the 8 x 8 form loads two per DMMA
    // and is bound by shared-memory issue, not by the DMMA pipe)
    const int tn = (N + 15) >> 4, tiles = ((M + 15) >> 4) * tn;
    for (int tt = warp; tt < tiles; tt += nw) {
      const int m0 = (tt / tn) * 16, n0 = (tt % tn) * 16;
      const int ma = m0 + fr, mb = m0 + 8 + fr, na = n0 + fr, nb = n0 + 8 + fr;
      const bool va = ma < M, vb = mb < M, wa = na < N, wb = nb < N;
      double c00[2] = {0.0, 0.0}, c01[2] = {0.0, 0.0}, c10[2] = {0.0, 0.0}, c11[2] = {0.0, 0.0};
#pragma unroll 2
      for (int k0 = 0; k0 < K; k0 += 4) {
        const int k = k0 + fk;
        const bool kv = k < K;
        const double a0 = (va && kv) ? A[ma * a_rs + k * a_cs] : 0.0;
        const double a1 = (vb && kv) ? A[mb * a_rs + k * a_cs] : 0.0;
        const double b0 = (wa && kv) ? B[k * b_rs + na * b_cs] : 0.0;
        const double b1 = (wb && kv) ? B[k * b_rs + nb * b_cs] : 0.0;
        dmma_8x8x4(c00, a0, b0);
        dmma_8x8x4(c01, a0, b1);
        dmma_8x8x4(c10, a1, b0);
        dmma_8x8x4(c11, a1, b1);
      }
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int cn0 = n0 + 2 * fk + h, cn1 = n0 + 8 + 2 * fk + h;
        auto put = [&](int m, int cn, double v) {
          if (m < M && cn < N) {
            if (sub) C[m * ldc + cn] -= v;
            else C[m * ldc + cn] = v;
          }
        };
        put(ma, cn0, c00[h]);
        put(ma, cn1, c01[h]);
        put(mb, cn0, c10[h]);
        put(mb, cn1, c11[h]);
      }
    }
    return;
  }
  const int tn = (N + 7) >> 3, tiles = ((M + 7) >> 3) * tn;
  for (int tt = warp; tt < tiles; tt += nw) {
    const int m0 = (tt / tn) * 8, n0 = (tt % tn) * 8;
    const int m = m0 + fr, n = n0 + fr;
    double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
    int k0 = 0;
    for (; k0 + 8 <= K; k0 += 8) {
      const int ka = k0 + fk, kb = k0 + 4 + fk;
      const double a0 = (m < M) ? A[m * a_rs + ka * a_cs] : 0.0;
      const double b0 = (n < N) ? B[ka * b_rs + n * b_cs] : 0.0;
      const double a1 = (m < M) ? A[m * a_rs + kb * a_cs] : 0.0;
      const double b1 = (n < N) ? B[kb * b_rs + n * b_cs] : 0.0;
      dmma_8x8x4(c0, a0, b0);
      dmma_8x8x4(c1, a1, b1);
    }
    for (; k0 < K; k0 += 4) {
      const int k = k0 + fk;
      const double a0 = (m < M && k < K) ? A[m * a_rs + k * a_cs] : 0.0;
      const double b0 = (n < N && k < K) ? B[k * b_rs + n * b_cs] : 0.0;
      dmma_8x8x4(c0, a0, b0);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int cn = n0 + 2 * fk + h;
      if (m < M && cn < N) {
        if (rinv_out) {
          const double v = (cn > m) ? -rinv_f[m * ldc + cn] + rinv_p[m * ldc + cn] - (c0[h] + c1[h])
                           : (cn == m ? 1.0 - rinv_f[m * ldc + cn] + rinv_p[m * ldc + cn] - (c0[h] + c1[h]) : 0.0);
          rinv_out[(size_t)m * N + cn] = v;
        } else if (sub) {
          C[m * ldc + cn] -= c0[h] + c1[h];
        } else {
          C[m * ldc + cn] = c0[h] + c1[h];
        }
      }
    }
  }
}

// Triangular variant of block_dmma for the near-identity series: only output
// tiles with m-tile <= n-tile (upper triangle, lower tiles are left alone) and,
// per tile, only the k range where both operands are nonzero:
//   kind 0: C = F^T F with F upper  -> k < min(m, n) + 8  (k <= min(i, j))
//   kind 1: C = A B with A, B upper -> k in [m-tile start, n-tile end)
// rinv_out != nullptr: the R^{-1} epilogue of block_dmma (only c >= r written; the
// strictly lower part of rinv_out is zeroed by the caller).
__device__ void block_dmma_tri(int l, int kind, const double* A, int a_rs, int a_cs, const double* B, int b_rs,
                               int b_cs, double* C, int ldc, double* rinv_out = nullptr,
                               const double* rinv_f = nullptr, const double* rinv_p = nullptr) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int fr = lane >> 2, fk = lane & 3;
  const int nt = (l + 7) >> 3;
  const int tiles = nt * (nt + 1) / 2;
  for (int tt = warp; tt < tiles; tt += nw) {
    // tt -> (ti <= tj), row-major over the upper triangle
    int ti = 0, rem = tt;
    while (rem >= nt - ti) { rem -= nt - ti; ++ti; }
    const int tj = ti + rem;
    const int m0 = ti * 8, n0 = tj * 8;
    const int m = m0 + fr, n = n0 + fr;
    const int kb = (kind == 0) ? 0 : (m0 & ~3);
    const int ke = min(l, (kind == 0) ? m0 + 8 : n0 + 8);
    double c0[2] = {0.0, 0.0}, c1[2] = {0.0, 0.0};
    int k0 = kb;
    for (; k0 + 8 <= ke; k0 += 8) {
      const int ka = k0 + fk, kb2 = k0 + 4 + fk;
      const double a0 = (m < l) ? A[m * a_rs + ka * a_cs] : 0.0;
      const double b0 = (n < l) ? B[ka * b_rs + n * b_cs] : 0.0;
      const double a1 = (m < l) ? A[m * a_rs + kb2 * a_cs] : 0.0;
      const double b1 = (n < l) ? B[kb2 * b_rs + n * b_cs] : 0.0;
      dmma_8x8x4(c0, a0, b0);
      dmma_8x8x4(c1, a1, b1);
    }
    for (; k0 < ke; k0 += 4) {
      const int k = k0 + fk;
      const double a0 = (m < l && k < ke) ? A[m * a_rs + k * a_cs] : 0.0;
      const double b0 = (n < l && k < ke) ? B[k * b_rs + n * b_cs] : 0.0;
      dmma_8x8x4(c0, a0, b0);
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int cn = n0 + 2 * fk + h;
      if (m < l && cn < l) {
        const double v = c0[h] + c1[h];
        if (rinv_out) {
          if (cn >= m)
            rinv_out[(size_t)m * l + cn] = (cn == m ? 1.0 : 0.0) - rinv_f[m * ldc + cn] + rinv_p[m * ldc + cn] - v;
        } else {
          C[m * ldc + cn] = v;
        }
      }
    }
  }
}

// Cholesky factor of a Gram matrix that is already the identity to within
// tol (the second CholeskyQR pass of a well-conditioned block), by series:
// with E = G - I, F1 = triu(E) - diag(E)/2 satisfies F1 + F1^T = E, and
// F2 = F1 - up(F1^T F1) (up: upper triangle, halved diagonal) gives
// (I + F2)^T (I + F2) = I + E + O(|E|^3); R^{-1} = I - F2 + F2^2 - F2^3 + O(|E|^4).
// For tol = 1e-7 and l <= 96 both are exact to ~1e-17: three small DMMA
// products across the block instead of l sequential pivots.
// Writes *flag = 1 when it produced R and R^{-1}, 0 when G is not close enough
// (then the elimination kernel launched after it does the work).
constexpr int kNearIdMax = kCholMaxCols;

__device__ __forceinline__ int near_id_ld(int l) { return ((l + 15) & ~15) + 4; }

// body shared by chol_near_identity_kernel and the fused CholeskyQR2 kernel
// (any block size that is a multiple of 32; sm: 2 l near_id_ld(l) doubles)
// Element-wise pass over an n-element global array written earlier in the same
// kernel by other CTAs: U independent L2 loads in flight per thread (a plain
// strided loop waits one L2 round trip, ~0.5 us, per element: 5-6 us for an
// 80 x 80 matrix on 512 threads).  __ldcg: L2 only, never a stale L1 line.
template <int U, typename F>
__device__ __forceinline__ void for_each_l2(const double* __restrict__ src, int n, F&& f) {
  const int nt = blockDim.x;
  for (int e0 = threadIdx.x; e0 < n; e0 += U * nt) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * nt;
      v[u] = e < n ? __ldcg(src + e) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int e = e0 + u * nt;
      if (e < n) f(e, v[u]);
    }
  }
}

// Bound on l |E|^2 below which the second CholeskyQR pass uses the first-order
// factor R = I + F1, R^{-1} = I - F1 (F1 = triu(E) - diag(E)/2): then
// Q^T Q = R^{-T} (I + E) R^{-1} = I + O(l |E|^2), i.e. the dropped second-order
// terms leave an orthogonality error of at most ~1e-15 -- the size of the
// rounding of the Q product itself.  (r01 used 1e-17; the config-3 RTO
// sketches, kappa up to ~600, sit between the two and paid ~19 us per
// factorisation for three 80^3 products on one CTA.)
constexpr double kNearIdFirstOrderMax = 1e-15;

__device__ void chol_near_identity_body(int l, const double* __restrict__ G, double* __restrict__ Rout,
                                        double* __restrict__ Rinv, int* flag, double tol, double first_order_max,
                                        double* sm) {
  const int ld = near_id_ld(l);
  double* F = sm;
  double* P = F + (size_t)l * ld;
  __shared__ double red[32];
  const int tid = threadIdx.x, nt = blockDim.x;
  double e = 0.0;
  for_each_l2<16>(G, l * l, [&](int idx, double g) {
    const int r = idx / l, c = idx - r * l;
    e = fmax(e, fabs(g - (r == c ? 1.0 : 0.0)));
    F[r * ld + c] = (c > r) ? g : (c == r ? 0.5 * (g - 1.0) : 0.0);
  });
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
  if ((tid & 31) == 0) red[tid >> 5] = e;
  __syncthreads();
  double emax = 0.0;
  for (int i = 0; i < (nt >> 5); ++i) emax = fmax(emax, red[i]);
  if (!(emax <= tol)) {
    if (tid == 0) *flag = 0;
    return;
  }
  if ((double)l * emax * emax <= first_order_max) {
    // every second-order term (entries of F1^T F1, F1^2) is below l |E|^2 <= 1e-17:
    // R = I + F1 and R^{-1} = I - F1 are exact to below an ulp of 1 (the usual
    // case: a well-conditioned block leaves |E| ~ 1e-12 after the first pass)
    for (int idx = tid; idx < l * l; idx += nt) {
      const int i = idx / l, c = idx - i * l;
      const double f = F[i * ld + c];
      Rout[idx] = (c > i) ? f : (c == i ? 1.0 + f : 0.0);
      Rinv[idx] = (c > i) ? -f : (c == i ? 1.0 - f : 0.0);
    }
    if (tid == 0) *flag = 1;
    return;
  }
  block_dmma_tri(l, 0, F, 1, ld, F, ld, 1, P, ld);  // P = F1^T F1 (upper tiles, k <= min(i, j))
  __syncthreads();
  for (int idx = tid; idx < l * l; idx += nt) {
    const int i = idx / l, c = idx - i * l;
    if (c > i) F[i * ld + c] -= P[i * ld + c];
    else if (c == i) F[i * ld + c] -= 0.5 * P[i * ld + c];
  }
  __syncthreads();
  for (int idx = tid; idx < l * l; idx += nt) {
    const int i = idx / l, c = idx - i * l;
    Rout[idx] = (c > i) ? F[i * ld + c] : (c == i ? 1.0 + F[i * ld + c] : 0.0);
    if (c < i) Rinv[idx] = 0.0;
  }
  block_dmma_tri(l, 1, F, ld, 1, F, ld, 1, P, ld);  // P = F2^2 (upper x upper)
  __syncthreads();
  // R^{-1} = I - F2 + F2^2 - F2^2 F2, the last product folded into the store
  block_dmma_tri(l, 1, P, ld, 1, F, ld, 1, nullptr, ld, Rinv, F, P);
  if (tid == 0) *flag = 1;
}

__global__ void __launch_bounds__(1024, 1)
    chol_near_identity_kernel(int l, const double* __restrict__ G, double* __restrict__ Rout,
                              double* __restrict__ Rinv, int* flag, double tol, double first_order_max) {
  extern __shared__ double sm[];
  chol_near_identity_body(l, G, Rout, Rinv, flag, tol, first_order_max, sm);
}

// Blocked right-looking Cholesky (blocks of 16) of G + shift*trace(G) I for
// l <= kCholMaxCols: warp 0 factors each 16 x 16 diagonal block in registers
// (lane c owns column c; pivots by shuffle, rsqrt, no barrier inside), the
// panel R_kk^{-T} A_kJ is a thread-per-column forward substitution, and the
// trailing update A_JJ -= R_kJ^T R_kJ runs on the DMMA pipe.  Three barriers
// per block instead of one per pivot.  R^{-1} (when Rinv != nullptr) by
// blocked triangular inversion.  Same status bits as chol_inv_kernel.
constexpr int kCbThreads = 512;


// one pivot of the in-register 16 x 16 diagonal-block Cholesky (lane c owns
// column c); compile-time recursion keeps every index of d[] static.  dg is the
// lane's own diagonal entry W[c][c], updated from registers only (dg -= rrow^2),
// so the pivot chain is shuffle -> rsqrt -> row entry -> dg and the
// shared-memory broadcast of the pivot row (store, syncwarp, loads, updates)
// runs beside the next pivot's rsqrt instead of ahead of it.
template <int JJ>
__device__ __forceinline__ void cb_diag_steps(double (&d)[16], double& dg, int lane, int bs, double tiny, int& badd,
                                              double (*rowb)[16]) {
  if constexpr (JJ < 16) {
    double p = __shfl_sync(0xffffffffu, dg, JJ);
    if (JJ < bs && !(p > tiny)) { badd = 1; p = 1.0; }
    if (JJ >= bs) p = 1.0;
    // rrow = x / sqrt(p), x = p on the pivot lane: the seed y is good to 2^-20
    // (tools/rsqrt_acc.cu), one third-order correction x y (1 + e (1/2 + 3e/8)),
    // e = 1 - p y^2, with x y formed beside p y
    // unconditional row and update: lanes c < JJ / entries below the diagonal
    // only touch the strict lower triangle, which is never read again and is
    // zeroed when the block is stored
    double y;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(p));
    const double x = (lane == JJ) ? p : d[JJ];
    const double xy = x * y;
    const double e = fma(-p * y, y, 1.0);
    const double rrow = fma(xy * e, fma(e, 0.375, 0.5), xy);
    dg = fma(-rrow, rrow, dg);
    d[JJ] = rrow;
    // row JJ of R broadcast through shared memory (double-buffered by pivot
    // parity): one store per lane and 15 - JJ broadcast loads instead of
    // 2 (15 - JJ) 32-bit shuffles per pivot
    if (lane < 16) rowb[JJ & 1][lane] = rrow;
    __syncwarp();
#pragma unroll
    for (int rr = JJ + 1; rr < 16; ++rr) d[rr] = fma(-rowb[JJ & 1][rr], rrow, d[rr]);
    cb_diag_steps<JJ + 1>(d, dg, lane, bs, tiny, badd, rowb);
  }
}


__host__ __device__ __forceinline__ int cb_ld(int l) { return ((l + 15) & ~15) + 4; }

// partial tiles of warp_dmma16 (M or N below 16, or K not a multiple of 4: the solver's
// small ranks), out of line so that its registers do not weigh on the callers' pivot chains
__device__ __noinline__ void warp_dmma16_partial(int M, int N, int K, const double* A, int a_rs, int a_cs,
                                                 const double* B, int b_rs, int b_cs, double* C, int ldc, bool neg,
                                                 const double* D, int ldd) {
  const int lane = threadIdx.x & 31, fr = lane >> 2, fk = lane & 3;
  const int ma = fr, mb = 8 + fr;
  double c00[2] = {0.0, 0.0}, c01[2] = {0.0, 0.0}, c10[2] = {0.0, 0.0}, c11[2] = {0.0, 0.0};
  // partial tiles (the solver's small ranks): the same chunked schedule with clamped
  // addresses and selects instead of predicated loads -- 16 loads in flight per chunk
  const bool va = ma < M, vb = mb < M, wa = ma < N, wb = mb < N;
  {
    const double* pa0 = A + min(ma, M - 1) * a_rs;
    const double* pa1 = A + min(mb, M - 1) * a_rs;
    const double* pb0 = B + min(ma, N - 1) * b_cs;
    const double* pb1 = B + min(mb, N - 1) * b_cs;
    for (int k0 = 0; k0 < K; k0 += 16) {
      double a0[4], a1[4], b0[4], b1[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = k0 + 4 * q + fk;
        const int kc = min(k, K - 1);
        const bool kv = k < K;
        const double x0 = pa0[kc * a_cs], x1 = pa1[kc * a_cs], y0 = pb0[kc * b_rs], y1 = pb1[kc * b_rs];
        a0[q] = (va && kv) ? x0 : 0.0;
        a1[q] = (vb && kv) ? x1 : 0.0;
        b0[q] = (wa && kv) ? y0 : 0.0;
        b1[q] = (wb && kv) ? y1 : 0.0;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (k0 + 4 * q < K) {  // warp-uniform
          dmma_8x8x4(c00, a0[q], b0[q]);
          dmma_8x8x4(c01, a0[q], b1[q]);
          dmma_8x8x4(c10, a1[q], b0[q]);
          dmma_8x8x4(c11, a1[q], b1[q]);
        }
      }
    }
  }
  const double sg = neg ? -1.0 : 1.0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int cn0 = 2 * fk + h, cn1 = 8 + 2 * fk + h;
    if (va && cn0 < N) C[ma * ldc + cn0] = fma(sg, c00[h], D ? D[ma * ldd + cn0] : 0.0);
    if (va && cn1 < N) C[ma * ldc + cn1] = fma(sg, c01[h], D ? D[ma * ldd + cn1] : 0.0);
    if (vb && cn0 < N) C[mb * ldc + cn0] = fma(sg, c10[h], D ? D[mb * ldd + cn0] : 0.0);
    if (vb && cn1 < N) C[mb * ldc + cn1] = fma(sg, c11[h], D ? D[mb * ldd + cn1] : 0.0);
  }
}

// one warp: C[0:M, 0:N] (row stride ldc) = D + (neg ? -1 : 1) A[0:M, 0:K] B[0:K, 0:N]
// for M, N <= 16 (2 x 2 DMMA tiles, the fragment layout of block_dmma); D
// (row stride ldd) may be null (zero) or alias C or B.  Full tiles with K a
// multiple of 16 take an unpredicated path that issues the 16 operand loads of
// a 16-deep K chunk before its 16 DMMAs (a single warp runs these products, so
// their time is the load -> DMMA chain, not throughput).
__device__ __forceinline__ void warp_dmma16(int M, int N, int K, const double* A, int a_rs, int a_cs,
                                            const double* B, int b_rs, int b_cs, double* C, int ldc, bool neg,
                                            const double* D = nullptr, int ldd = 0) {
  const int lane = threadIdx.x & 31, fr = lane >> 2, fk = lane & 3;
  const int ma = fr, mb = 8 + fr;
  double c00[2] = {0.0, 0.0}, c01[2] = {0.0, 0.0}, c10[2] = {0.0, 0.0}, c11[2] = {0.0, 0.0};
  const bool full = (M == 16) && (N == 16) && ((K & 3) == 0);
  if (full) {
    const double* pa0 = A + ma * a_rs + fk * a_cs;
    const double* pa1 = A + mb * a_rs + fk * a_cs;
    const double* pb0 = B + fk * b_rs + ma * b_cs;
    const double* pb1 = B + fk * b_rs + mb * b_cs;
    int k0 = 0;
    for (; k0 + 16 <= K; k0 += 16) {
      double a0[4], a1[4], b0[4], b1[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = k0 + 4 * q;
        a0[q] = pa0[k * a_cs];
        a1[q] = pa1[k * a_cs];
        b0[q] = pb0[k * b_rs];
        b1[q] = pb1[k * b_rs];
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        dmma_8x8x4(c00, a0[q], b0[q]);
        dmma_8x8x4(c01, a0[q], b1[q]);
        dmma_8x8x4(c10, a1[q], b0[q]);
        dmma_8x8x4(c11, a1[q], b1[q]);
      }
    }
    for (; k0 < K; k0 += 4) {  // K not a multiple of 16: single k steps
      const double a0 = pa0[k0 * a_cs], a1 = pa1[k0 * a_cs], b0 = pb0[k0 * b_rs], b1 = pb1[k0 * b_rs];
      dmma_8x8x4(c00, a0, b0);
      dmma_8x8x4(c01, a0, b1);
      dmma_8x8x4(c10, a1, b0);
      dmma_8x8x4(c11, a1, b1);
    }
    const double sg = neg ? -1.0 : 1.0;
    double dv[8] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    if (D) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        dv[h] = D[ma * ldd + 2 * fk + h];
        dv[2 + h] = D[ma * ldd + 8 + 2 * fk + h];
        dv[4 + h] = D[mb * ldd + 2 * fk + h];
        dv[6 + h] = D[mb * ldd + 8 + 2 * fk + h];
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      C[ma * ldc + 2 * fk + h] = fma(sg, c00[h], dv[h]);
      C[ma * ldc + 8 + 2 * fk + h] = fma(sg, c01[h], dv[2 + h]);
      C[mb * ldc + 2 * fk + h] = fma(sg, c10[h], dv[4 + h]);
      C[mb * ldc + 8 + 2 * fk + h] = fma(sg, c11[h], dv[6 + h]);
    }
    return;
  }
  warp_dmma16_partial(M, N, K, A, a_rs, a_cs, B, b_rs, b_cs, C, ldc, neg, D, ldd);
}

// Blocked right-looking Cholesky core on an l x l SPD matrix already in shared
// memory (row stride ld = cb_ld(l)): on return the upper triangle of A holds R
// (A = R^T R); the strict lower triangle is left unspecified.  X (l x ld; Tb:
// 256 ceil(l/16) doubles of scratch) is zeroed and receives the inverses of the 16 x 16 diagonal blocks of R: the
// warp that factors a diagonal block carries the identity in its upper 16
// lanes through the same elimination (lane 16 + c owns column c of L^{-1} =
// row c of R_kk^{-1}) at no cost on the pivot chain.  The panel is then one
// DMMA product R_kJ = R_kk^{-T} A_kJ per 16 columns instead of a 16-step
// substitution per column (which was ~5 K cycles per block), and
// tri_inv_offdiag completes R^{-1} from the diagonal inverses.  *bad |= 1 on a
// pivot <= tiny.  All threads of the CTA (a multiple of 32, >= 32); ph: optional
// per-phase clock sink of thread 0 (chol_blocked_kernel diagnostics).
__device__ void chol_blocked_core(int l, double* __restrict__ A, int ld, double* __restrict__ X,
                                  double* __restrict__ Tb, double tiny, int* bad, long long* ph, long long& t0) {
  __shared__ double rowb[2][16];  // pivot-row broadcast of the diagonal-block factorisation
  const int tid = threadIdx.x, nt = blockDim.x, w = tid >> 5, lane = tid & 31, nw = nt >> 5;
  const int nb = (l + 15) >> 4;
  for (int e = tid; e < l * ld; e += nt) X[e] = 0.0;
  __syncthreads();
  for (int kb = 0; kb < nb; ++kb) {
    const int j0 = kb * 16, bs = min(16, l - j0);
    if (w == 0) {
      // diagonal block: lane c (< 16) owns column c (rows 0..15 of the block),
      // lane 16 + c column c of the identity
      const int c = lane & 15;
      const bool aug = lane >= 16;
      double d[16];
#pragma unroll
      for (int rr = 0; rr < 16; ++rr)
        d[rr] = (!aug && rr < bs && c < bs) ? A[(j0 + rr) * ld + j0 + c] : (rr == c ? 1.0 : 0.0);
      int badd = 0;
      double dg = (!aug && c < bs) ? A[(j0 + c) * ld + j0 + c] : 1.0;
      cb_diag_steps<0>(d, dg, lane, bs, tiny, badd, rowb);
      if (c < bs) {
        if (!aug) {
#pragma unroll
          for (int rr = 0; rr < 16; ++rr)
            if (rr < bs) A[(j0 + rr) * ld + j0 + c] = (rr <= c) ? d[rr] : 0.0;
        } else {
#pragma unroll
          for (int rr = 0; rr < 16; ++rr)
            if (rr < bs) X[(j0 + c) * ld + j0 + rr] = (rr >= c) ? d[rr] : 0.0;
        }
      }
      if (badd && lane == 0) atomicOr(bad, 1);
    }
    __syncthreads();
    if (ph) { long long t = clock64(); ph[1] += t - t0; t0 = t; }
    const int rest = l - j0 - bs;
    if (rest > 0) {
      // panel: R_kJ = R_kk^{-T} A_kJ in place, one warp per 16 columns, with one
      // refinement step T + R_kk^{-T} (A_kJ - R_kk^T T) so that the panel solves
      // R_kk^T R_kJ = A_kJ as accurately as a substitution does
      for (int t = w; t * 16 < rest; t += nw) {
        const int n0 = j0 + bs + t * 16, nn = min(16, l - n0);
        double* P = A + (size_t)j0 * ld + n0;
        double* T = Tb + t * 256;
        const double* Xt = X + (size_t)j0 * ld + j0;  // (m, k) -> R_kk^{-1}[k][m]
        const double* Rt = A + (size_t)j0 * ld + j0;  // (m, k) -> R_kk[k][m]
        warp_dmma16(bs, nn, bs, Xt, 1, ld, P, ld, 1, T, 16, false);
        __syncwarp();
        warp_dmma16(bs, nn, bs, Rt, 1, ld, T, 16, 1, P, ld, true, P, ld);  // residual
        __syncwarp();
        warp_dmma16(bs, nn, bs, Xt, 1, ld, P, ld, 1, P, ld, false, T, 16);
      }
      __syncthreads();
      if (ph) { long long t = clock64(); ph[2] += t - t0; t0 = t; }
      // trailing update (full square; only the upper triangle is used later)
      const double* P = A + (size_t)j0 * ld + j0 + bs;  // bs x rest panel
      block_dmma(rest, rest, bs, P, 1, ld, P, ld, 1, A + (size_t)(j0 + bs) * ld + j0 + bs, ld, nullptr,
                 nullptr, nullptr, true);
      __syncthreads();
      if (ph) { long long t = clock64(); ph[3] += t - t0; t0 = t; }
    }
  }
}

// R^{-1} (X, upper) from R (A, upper) and the inverses of R's 16 x 16 diagonal
// blocks already in X (chol_blocked_core): block back-substitution
// X_IJ = -X_II sum_{I<K<=J} R_IK X_KJ, one block-diagonal distance at a time,
// one warp per block, both products on the DMMA pipe.  Tb: 256 ceil(l/16) doubles.
__device__ void tri_inv_offdiag(const double* __restrict__ A, double* __restrict__ X, double* __restrict__ Tb,
                                int ld, int l) {
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int nb = (l + 15) >> 4;
  for (int dist = 1; dist < nb; ++dist) {
    const int nblk = nb - dist;
    for (int I = w; I < nblk; I += nw) {
      const int i0 = I * 16, k0 = i0 + 16, c0 = (I + dist) * 16;
      warp_dmma16(16, min(16, l - c0), min(l, c0 + 16) - k0, A + (size_t)i0 * ld + k0, ld, 1,
                  X + (size_t)k0 * ld + c0, ld, 1, Tb + I * 256, 16, false);
    }
    __syncthreads();
    for (int I = w; I < nblk; I += nw) {
      const int i0 = I * 16, c0 = (I + dist) * 16;
      warp_dmma16(16, min(16, l - c0), 16, X + (size_t)i0 * ld + i0, ld, 1, Tb + I * 256, 16, 1,
                  X + (size_t)i0 * ld + c0, ld, true);
    }
    __syncthreads();
  }
}

// C (l x l, row stride ldc) = Y^T Y for the K x l tile Y (row stride ldy) in
// shared memory: upper 16 x 16 tiles only (ti <= tj), one warp per tile -- 15
// tiles instead of 25 for l = 80, one round of the 16 warps instead of two.
// The lower tiles of C are left untouched.
__device__ __forceinline__ void block_gram_upper(int l, int K, const double* Y, int ldy, double* C, int ldc) {
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int tn = (l + 15) >> 4, tiles = tn * (tn + 1) / 2;
  for (int tt = warp; tt < tiles; tt += nw) {
    int ti = 0, rem = tt;
    while (rem >= tn - ti) { rem -= tn - ti; ++ti; }
    const int i0 = ti * 16, j0 = (ti + rem) * 16;
    warp_dmma16(min(16, l - i0), min(16, l - j0), K, Y + i0, 1, ldy, Y + j0, ldy, 1, C + (size_t)i0 * ldc + j0, ldc,
                false);
  }
}

// element (i, c) of an l x l matrix stored with its upper 16 x 16 tiles only
__device__ __forceinline__ bool in_upper_tiles(int i, int c) { return (i >> 4) <= (c >> 4); }

// body shared by chol_blocked_kernel and the fused CholeskyQR2 kernel (block
// size kCbThreads; sm: 2 l cb_ld(l) + 256 ceil(l/16) doubles)
__device__ void chol_blocked_body(int l, const double* __restrict__ G, double* __restrict__ Rout,
                                  double* __restrict__ Rinv, int* status, int check_identity, double shift_rel,
                                  double tiny_rel, double* sm) {
  const int ld = cb_ld(l);
  double* A = sm;                       // l x ld
  double* X = A + (size_t)l * ld;       // l x ld (inverse)
  double* Tb = X + (size_t)l * ld;      // 256 * nb
  __shared__ double gmax_s, tr_s;
  __shared__ int bad;
  const int tid = threadIdx.x, nt = blockDim.x, w = tid >> 5, lane = tid & 31;
  long long* const prof = (tid == 0) ? g_chol_prof : nullptr;
  long long t0 = prof ? clock64() : 0, ph[6] = {0, 0, 0, 0, 0, 0};
  if (tid == 0) bad = 0;
  __syncthreads();
  {
    int badl = 0;
    for_each_l2<16>(G, l * l, [&](int e, double v) {
      const int r = e / l, c = e - r * l;
      if (check_identity && fabs(v - (r == c ? 1.0 : 0.0)) > 1e-3) badl |= 2;
      A[r * ld + c] = v;
    });
    if (badl) atomicOr(&bad, badl);
  }
  __syncthreads();
  if (w == 0) {
    // diagonal statistics (same order as before: lane-strided max / sum, warp reduction)
    double g = 0.0, tr = 0.0;
    for (int i = lane; i < l; i += 32) { const double v = A[i * ld + i]; g = fmax(g, v); tr += v; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) g = fmax(g, __shfl_xor_sync(0xffffffffu, g, o));
    tr = warp_sum(tr);
    const double shw = shift_rel > 0.0 ? shift_rel * tr : 0.0;
    if (shw != 0.0)
      for (int i = lane; i < l; i += 32) A[i * ld + i] += shw;
    if (lane == 0) { gmax_s = g; tr_s = tr; }
  }
  __syncthreads();
  const double tiny = gmax_s * tiny_rel + 1e-300;
  if (prof) { long long t = clock64(); ph[0] += t - t0; t0 = t; }
  chol_blocked_core(l, A, ld, X, Tb, tiny, &bad, prof ? ph : nullptr, t0);
  for (int e = tid; e < l * l; e += nt) {
    const int r = e / l, c = e - r * l;
    Rout[e] = (c >= r) ? A[r * ld + c] : 0.0;
  }
  if (Rinv) {
    tri_inv_offdiag(A, X, Tb, ld, l);
    for (int e = tid; e < l * l; e += nt) {
      const int r = e / l, c = e - r * l;
      Rinv[e] = (c >= r) ? X[r * ld + c] : 0.0;
    }
  }
  if (prof) {
    ph[4] = clock64() - t0;
    for (int i = 0; i < 5; ++i) atomicAdd((unsigned long long*)&prof[i], (unsigned long long)ph[i]);
    atomicAdd((unsigned long long*)&prof[5], 1ull);
  }
  if (tid == 0 && bad) atomicOr(status, bad);
}

__global__ void __launch_bounds__(kCbThreads, 1)
    chol_blocked_kernel(int l, const double* __restrict__ G, double* __restrict__ Rout,
                        double* __restrict__ Rinv, int* status, int check_identity, double shift_rel,
                        double tiny_rel, const int* __restrict__ skip) {
  if (skip && *skip) return;  // chol_near_identity_kernel already produced R, R^{-1}
  extern __shared__ double sm[];
  chol_blocked_body(l, G, Rout, Rinv, status, check_identity, shift_rel, tiny_rel, sm);
}

// R (upper) and R^{-1} of the Cholesky factor of G (+ shift): register kernel
// for l <= 96, shared-memory kernel above
int launch_chol_inv(int l, const double* G, double* R, double* Rinv, int* status, int check_identity,
                    double shift_rel, double tiny_rel, cudaStream_t st, int* near_id_flag) {
  {  // per-device attributes (set_attr_once)
    TTK_TRY(qr_set_smem((const void*)chol_inv_kernel, 220 * 1024));
    TTK_TRY(qr_set_smem((const void*)chol_near_identity_kernel, 220 * 1024));
    TTK_TRY(qr_set_smem((const void*)chol_blocked_kernel, 225 * 1024));
  }
  const int* skip = nullptr;
  if (near_id_flag && shift_rel == 0.0 && l <= kNearIdMax) {
    const size_t smem_n = sizeof(double) * 2 * (size_t)l * (((l + 15) & ~15) + 4);
    // first-order shortcut when l |E|^2 <= kNearIdFirstOrderMax; TTK_NEAR_ID_FIRST_ORDER=0 disables it (A/B)
    static const double fo = knob_env("TTK_NEAR_ID_FIRST_ORDER") ? atof(knob_env("TTK_NEAR_ID_FIRST_ORDER"))
                                                                   : kNearIdFirstOrderMax;
    chol_near_identity_kernel<<<1, 1024, smem_n, st>>>(l, G, R, Rinv, near_id_flag, 1e-7, fo);
    TTK_CHECK_LAUNCH();
    skip = near_id_flag;
  }
  if (l <= kCholMaxCols) {
    const int ldb = ((l + 15) & ~15) + 4;
    const size_t smem_b = sizeof(double) * (2 * (size_t)l * ldb + 256 * (size_t)((l + 15) / 16));
    chol_blocked_kernel<<<1, kCbThreads, smem_b, st>>>(l, G, R, Rinv, status, check_identity, shift_rel, tiny_rel,
                                                       skip);
  } else {
    const size_t smem = sizeof(double) * (2 * (size_t)l * (l + 1) + 256 * (size_t)((l + 15) / 16));
    chol_inv_kernel<<<1, 1024, smem, st>>>(l, G, R, Rinv, status, check_identity, shift_rel, tiny_rel, skip);
  }
  TTK_CHECK_LAUNCH();
  return kOk;
}

// --------------------------------------------------------------------------
// Gap-certified dominant-subspace factor for the exact-rank truncation.
//
// The truncation of core k (round.cu, Gram path) needs, for G = C C^T
// (l x l, C the r0 x m unfolding), a left factor F (l x r) and the map M
// (r x l) with Y = M C the new core: rows of Y orthonormal, F = C Y^T, so
// that F Y = C P_Y is C projected onto the row space of Y.  The reference
// (tt.py:358-367, np.linalg.svd) takes Y = V_r^T; any Y spanning the same
// dominant row space gives the same rounded tensor (the cores differ by a
// gauge).  When sigma_r / sigma_{r+1} is large -- the usual
// regime of a rounding that discards noise; config 3 has 41..770 -- that
// space is found with a few products instead of ~630 Jacobi rotation rounds:
//   Qa = orth(G[:, J])                J: the r largest diagonal entries (CholeskyQR)
//   Z  = G^2 Qa                       (tail damped by (lambda_{r+1}/lambda_r)^2 per pass)
//   Z^T G Z = R^T R,  M^T = Z R^{-1},  F = (G Z) R^{-1} = G M^T
// M G M^T = I whatever the conditioning of Z (G-orthonormalisation: one
// Cholesky gives the gauge, Z is never orthonormalised), so Y = M C has
// Y Y^T = I to eps kappa(Z^T G Z); D = M F - I is formed and, when
// max|D| > 1e-14, removed to second order (M^T, F) <- (M^T, F)(I - D/2).
// N = G^{1/2} M^T is then an orthonormal basis of G^{1/2} span(Z) -- the left
// image of Y's row space under the isometry V U^T of C = U S V^T -- with Ritz
// matrix B = N^T G N = F^T F and residual G N - N B = G^{1/2} E,
// E = F - M^T B, all formed from l x r matrices.  Every matrix lives in shared
// memory of one CTA, every product runs on the DMMA pipe.  Certificate
// (flag = 1), else the caller redoes the sweep with the Jacobi SVD: both
// Cholesky factorisations succeed; the tail tau = tr(G) - ||F||_F^2 >=
// sum_{i>r} lambda_i is below half of lmin = 1 / ||M M^T||_F <= 1 / ||M^T||_2^2
// <= lambda_min(B) (for unit x and y = M^T x: x^T B x = |G y|^2 >=
// (y^T G y)^2 / |y|^2 = 1 / |y|^2), a clear gap; the Davis-Kahan bound on the
// subspace angle, sqrt(tr(E^T G E)) / (lmin - tau), is <= 1e-9 (another pass
// Z <- G F -- F is as well conditioned as sqrt(kappa(B)), no orthonormalisation --
// while it exceeds 1e-12, at most kTsMaxIters passes); and lmin >= 2e-6 ||B||_F
// (the Gram squares the condition number, as for gram_cert_kernel).
constexpr int kTsMaxL = 80, kTsMaxR = 64, kTsThreads = 512, kTsMaxIters = 3;

__device__ __forceinline__ double ts_block_sum(double v, double* red) {
  v = warp_sum(v);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  for (int i = 0; i < nw; ++i) s += red[i];  // same order in every thread
  return s;
}

// Cholesky of the r x r A (ld) in place and X = R^{-1} (ld); false on a tiny pivot
__device__ bool ts_chol_inv(int r, double* A, double* X, double* Tb, int ld, int* bad, double* red,
                            long long* prof = nullptr) {
  const int tid = threadIdx.x, nt = blockDim.x;
  long long ph[6] = {0, 0, 0, 0, 0, 0};
  long long tc = prof ? clock64() : 0;
  double g = 0.0;
  for (int i = tid; i < r; i += nt) g = fmax(g, A[i * ld + i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) g = fmax(g, __shfl_xor_sync(0xffffffffu, g, o));
  __syncthreads();
  if ((tid & 31) == 0) red[tid >> 5] = g;
  if (tid == 0) *bad = 0;
  __syncthreads();
  double gm = 0.0;
  for (int i = 0; i < (nt >> 5); ++i) gm = fmax(gm, red[i]);
  long long t0 = tc;
  chol_blocked_core(r, A, ld, X, Tb, gm * 1e-15 + 1e-300, bad, (prof && tid == 0) ? ph : nullptr, t0);
  const bool ok = (*bad == 0);
  tri_inv_offdiag(A, X, Tb, ld, r);
  if (prof && tid == 0) {  // diagnostics: diagonal blocks, panels, trailing updates, inverse
    prof[5] += ph[1];
    prof[6] += ph[2];
    prof[7] += ph[3];
    prof[8] += clock64() - t0;
  }
  return ok;
}

__global__ void __launch_bounds__(kTsThreads, 1)
    trunc_subspace_kernel(int l, int r, const double* __restrict__ G, double* __restrict__ F,
                          double* __restrict__ Mt, int ldo, int* __restrict__ flag, double* __restrict__ info,
                          long long* __restrict__ prof) {
  extern __shared__ double sm[];
  long long tp = prof ? clock64() : 0;
  // diagnostics: phase clocks (thread 0) accumulated into prof[ph]
  auto mark = [&](int ph) {
    if (prof && threadIdx.x == 0) {
      const long long t = clock64();
      prof[ph] += t - tp;
      tp = t;
    }
  };
  const int ldg = cb_ld(l), ldq = cb_ld(r);
  double* Gs = sm;                                  // l x ldg
  double* p[3] = {Gs + (size_t)l * ldg, Gs + (size_t)l * ldg + (size_t)l * ldq,
                  Gs + (size_t)l * ldg + 2 * (size_t)l * ldq};  // l x ldq each
  double* A = p[2] + (size_t)l * ldq;               // r x ldq
  double* Tb = A + (size_t)r * ldq;                 // 256 * ceil(r/16)
  __shared__ double red[32];
  __shared__ int J[kTsMaxL];
  __shared__ int bad;
  const int tid = threadIdx.x, nt = blockDim.x;
  double trg = 0.0;
  for_each_l2<16>(G, l * l, [&](int e, double v) {
    const int i = e / l, c = e - i * l;
    Gs[i * ldg + c] = v;
    if (i == c) trg += v;
  });
  trg = ts_block_sum(trg, red);  // (contains the barrier after the load)
  // J: indices of the r largest diagonal entries (ties by index); a non-finite
  // diagonal ranks nothing, so J starts as the identity (the factorisation then
  // fails its certificate instead of indexing out of range)
  for (int i = tid; i < r; i += nt) J[i] = i;
  __syncthreads();
  for (int i = tid; i < l; i += nt) {
    const double di = Gs[i * ldg + i];
    int rank = 0;
    for (int j = 0; j < l; ++j) {
      const double dj = Gs[j * ldg + j];
      rank += (dj > di || (dj == di && j < i)) ? 1 : 0;
    }
    if (rank < r) J[rank] = i;
  }
  __syncthreads();
  mark(0);
  bool ok = true;
  if (r < l) {
    for (int e = tid; e < l * r; e += nt) {
      const int i = e / r, c = e - i * r;
      p[0][i * ldq + c] = Gs[i * ldg + J[c]];
    }
    __syncthreads();
    // Qa = orth(G[:, J]) -> p[1]; G Qa -> p[2]; Z = G^2 Qa -> p[0]
    block_dmma(r, r, l, p[0], 1, ldq, p[0], ldq, 1, A, ldq);
    __syncthreads();
    mark(1);
    ok = ts_chol_inv(r, A, p[2], Tb, ldq, &bad, red, prof) && ok;
    mark(2);
    block_dmma(l, r, r, p[0], ldq, 1, p[2], ldq, 1, p[1], ldq);
    __syncthreads();
    block_dmma(l, r, l, Gs, ldg, 1, p[1], ldq, 1, p[2], ldq);
    __syncthreads();
    block_dmma(l, r, l, Gs, ldg, 1, p[2], ldq, 1, p[0], ldq);
  } else {
    // nothing is truncated: Z = I, only the gauge Y = R^{-T} C is computed
    for (int e = tid; e < l * ldq; e += nt) p[0][e] = (e / ldq == e % ldq) ? 1.0 : 0.0;
  }
  __syncthreads();
  mark(1);
  double bv = 0.0, taur = 0.0, dmax = 0.0;
  int it = 0;
  for (;; ++it) {
    // Z = p[0]: G Z -> p[1]; Z^T G Z -> A = R^T R; R^{-1} -> p[2]
    block_dmma(l, r, l, Gs, ldg, 1, p[0], ldq, 1, p[1], ldq);
    __syncthreads();
    block_dmma(r, r, l, p[0], 1, ldq, p[1], ldq, 1, A, ldq);
    __syncthreads();
    double trb = 0.0;
    for (int i = tid; i < r; i += nt) trb += A[i * ldq + i];
    trb = ts_block_sum(trb, red);
    mark(3);
    ok = ts_chol_inv(r, A, p[2], Tb, ldq, &bad, red, prof) && ok;
    mark(2);
    // kappa(Z^T G Z) <= tr(.) tr(.^-1) - r^2 + 2 (every eigenvalue pair adds
    // x + 1/x >= 2 to the product of the traces): below 4.5e4 the gauge is
    // orthonormal to ~5e-12 without looking, above it D = M F - I is formed
    double xf2 = 0.0;
    for (int e = tid; e < r * r; e += nt) {
      const int i = e / r, c = e - i * r;
      const double v = p[2][i * ldq + c];
      xf2 += v * v;
    }
    xf2 = ts_block_sum(xf2, red);
    const bool check_d = !(trb * xf2 - (double)r * r + 2.0 <= 4.5e4);
    // M^T = Z R^{-1} -> Mt (global); F = (G Z) R^{-1} -> p[0]; then M^T -> p[1]
    block_dmma(l, r, r, p[0], ldq, 1, p[2], ldq, 1, Mt, ldo);
    __syncthreads();
    block_dmma(l, r, r, p[1], ldq, 1, p[2], ldq, 1, p[0], ldq);
    __syncthreads();
    for (int e = tid; e < l * r; e += nt) {
      const int i = e / r, c = e - i * r;
      p[1][i * ldq + c] = Mt[(size_t)i * ldo + c];
    }
    __syncthreads();
    double* fs = p[0];
    double* ms = p[1];
    double* es = p[2];
    double dm = 0.0;
    if (check_d) {  // uniform: D = M F - I
      block_dmma(r, r, l, ms, 1, ldq, fs, ldq, 1, A, ldq);
      __syncthreads();
      for (int e = tid; e < r * r; e += nt) {
        const int i = e / r, c = e - i * r;
        dm = fmax(dm, fabs(A[i * ldq + c] - (i == c ? 1.0 : 0.0)));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
      __syncthreads();
      if ((tid & 31) == 0) red[tid >> 5] = dm;
      __syncthreads();
      dm = 0.0;
      for (int i = 0; i < (nt >> 5); ++i) dm = fmax(dm, red[i]);
    }
    dmax = check_d ? dm : -1.0;
    bool polished = false;
    if (dm > 1e-14 && dm < 1e-4) {  // uniform: (M^T, F) <- (M^T, F) (I - D/2)
      polished = true;
      for (int e = tid; e < r * r; e += nt) {
        const int i = e / r, c = e - i * r;
        A[i * ldq + c] = (i == c ? 1.5 : 0.0) - 0.5 * A[i * ldq + c];
      }
      __syncthreads();
      block_dmma(l, r, r, ms, ldq, 1, A, ldq, 1, es, ldq);
      __syncthreads();
      block_dmma(l, r, r, fs, ldq, 1, A, ldq, 1, ms, ldq);
      __syncthreads();
      double* t = ms;  // M^T in es, F in ms, fs free
      ms = es;
      es = fs;
      fs = t;
      for (int e = tid; e < l * r; e += nt) {
        const int i = e / r, c = e - i * r;
        Mt[(size_t)i * ldo + c] = ms[i * ldq + c];
      }
    }
    ok = ok && dm < 1e-4;
    // F -> global; ||F||_F^2; S = M M^T -> A, lmin = 1 / ||S||_F
    double fsum = 0.0;
    for (int e = tid; e < l * r; e += nt) {
      const int i = e / r, c = e - i * r;
      const double v = fs[i * ldq + c];
      F[(size_t)i * ldo + c] = v;
      fsum += v * v;
    }
    block_dmma(r, r, l, ms, 1, ldq, ms, ldq, 1, A, ldq);
    fsum = ts_block_sum(fsum, red);
    double sf = 0.0;
    for (int e = tid; e < r * r; e += nt) {
      const int i = e / r, c = e - i * r;
      const double v = A[i * ldq + c];
      sf += v * v;
    }
    sf = ts_block_sum(sf, red);
    __syncthreads();
    // B = F^T F -> A; E = F - M^T B -> es; G E -> ms
    block_dmma(r, r, l, fs, 1, ldq, fs, ldq, 1, A, ldq);
    for (int e = tid; e < l * ldq; e += nt) es[e] = fs[e];
    __syncthreads();
    double bf = 0.0;
    for (int e = tid; e < r * r; e += nt) {
      const int i = e / r, c = e - i * r;
      const double v = A[i * ldq + c];
      bf += v * v;
    }
    block_dmma(l, r, r, ms, ldq, 1, A, ldq, 1, es, ldq, nullptr, nullptr, nullptr, true);
    bf = ts_block_sum(bf, red);
    __syncthreads();
    block_dmma(l, r, l, Gs, ldg, 1, es, ldq, 1, ms, ldq);
    __syncthreads();
    double rs = 0.0;
    for (int e = tid; e < l * r; e += nt) {
      const int i = e / r, c = e - i * r;
      rs = fma(es[i * ldq + c], ms[i * ldq + c], rs);
    }
    rs = fmax(ts_block_sum(rs, red), 0.0);
    const double lmin = 1.0 / sqrt(sf);
    const double tau = fmax(trg - fsum, 0.0) + 1e-12 * trg;
    const double gap = lmin - tau;
    // (r == l: the subspace is the whole space, only the gauge was computed)
    bv = (r == l) ? 0.0 : (gap > 0.0) ? sqrt(rs) / gap : INFINITY;
    taur = tau / lmin;
    ok = ok && gap > 0.5 * lmin && lmin >= 2e-6 * sqrt(bf);
    (void)polished;
    mark(3);
    if (!ok || bv <= 1e-12 || it + 1 >= kTsMaxIters) break;
    // next pass: Z = G F -> (a buffer that is not fs)
    block_dmma(l, r, l, Gs, ldg, 1, fs, ldq, 1, es, ldq);
    __syncthreads();
    // rotate so that Z sits in p[0]
    double* z = es;
    double* o1 = fs;
    double* o2 = ms;
    p[0] = z;
    p[1] = o1;
    p[2] = o2;
  }
  ok = ok && bv <= 1e-9;
  if (tid == 0) {
    *flag = ok ? 1 : 0;
    if (info) { info[0] = bv; info[1] = taur; info[2] = it + 1; info[3] = dmax; }
  }
  mark(4);
}

size_t trunc_subspace_smem(int l, int r) {
  return sizeof(double) * ((size_t)l * cb_ld(l) + 3 * (size_t)l * cb_ld(r) + (size_t)r * cb_ld(r) +
                           256 * (size_t)((r + 15) / 16));
}

bool trunc_subspace_fits(int l, int r) {
  return l >= 2 && r >= 1 && r <= l && l <= kTsMaxL && r <= kTsMaxR && trunc_subspace_smem(l, r) <= 227 * 1024;
}

int launch_trunc_subspace(int l, int r, const double* G, double* F, double* Mt, int ldo, int* flag, double* info,
                          cudaStream_t st, long long* prof) {
  TTK_REQUIRE(trunc_subspace_fits(l, r), kInvalidValue, "trunc_subspace: l=%d r=%d outside the kernel", l, r);
  TTK_TRY(qr_set_smem((const void*)trunc_subspace_kernel, (int)trunc_subspace_smem(kTsMaxL, kTsMaxR)));
  trunc_subspace_kernel<<<1, kTsThreads, trunc_subspace_smem(l, r), st>>>(l, r, G, F, Mt, ldo, flag, info,
                                                                               prof);
  TTK_CHECK_LAUNCH();
  return kOk;
}

// diagnostics: one subspace factorisation of the l x l G (device) for rank r:
// F, Mt (l x r, row stride l), flag, info[3] = {bound, tau / lmin, iterations},
// prof[5] phase clocks (load, initial orth products, Cholesky + inverse,
// iteration products + norms, output) or NULL
extern "C" int ttk_debug_trunc_subspace(int l, int r, const double* G, double* F, double* Mt, int* flag,
                                        double* info, long long* prof, void* stream) {
  return launch_trunc_subspace(l, r, G, F, Mt, l, flag, info, (cudaStream_t)stream, prof);
}

// --------------------------------------------------------------------------
// Gram matrix of a wide unfolding: G = C C^T for the row-major l x m C (l <= 96,
// row stride m) -- the per-core Gram of the truncation (round.cu).  CTA b
// stages columns [b kc, (b + 1) kc) of every row in shared memory once (kc a
// multiple of 16, the tail zero-filled), forms the upper 16 x 16 tiles of its
// l x l partial on DMMA (both operands of every tile come from the one staged
// slab) and stores them; gram_wide_reduce_kernel sums the partials in a fixed
// order (8 lanes per element, one L2 round trip) and mirrors the triangle.
// Replaces the generic split-K GEMM + reduce for this shape (80 x 80 x 8192:
// 19 + 4.6 us), which re-stages C for every 64 x 32 output tile.
constexpr int kGwThreads = 256;

__global__ void __launch_bounds__(kGwThreads)
    gram_wide_partial_kernel(int l, long long m, int kc, const double* __restrict__ C, double* __restrict__ part) {
  extern __shared__ double gw_sm[];
  const int ld = kc + 4;  // kc is a multiple of 16: stride 4 mod 16 doubles
  const long long c0 = (long long)blockIdx.x * kc;
  const int cols = (int)min((long long)kc, m - c0);
  const int tid = threadIdx.x, nt = blockDim.x, warp = tid >> 5, nw = nt >> 5;
  for (int e = tid; e < l * kc; e += nt) {
    const int r = e / kc, c = e - r * kc;
    const bool ok = c < cols;
    cp_async8(gw_sm + r * ld + c, ok ? C + (long long)r * m + c0 + c : C, ok);
  }
  cp_async_commit();
  cp_async_wait<0>();
  __syncthreads();
  const int tn = (l + 15) >> 4, tiles = tn * (tn + 1) / 2;
  double* mine = part + (size_t)blockIdx.x * l * l;
  for (int tt = warp; tt < tiles; tt += nw) {
    int ti = 0, rem = tt;
    while (rem >= tn - ti) { rem -= tn - ti; ++ti; }
    const int tj = ti + rem;
    const int i0 = ti * 16, j0 = tj * 16;
    warp_dmma16(min(16, l - i0), min(16, l - j0), kc, gw_sm + (size_t)i0 * ld, ld, 1, gw_sm + (size_t)j0 * ld, 1, ld,
                mine + (size_t)i0 * l + j0, l, false);
  }
}

__global__ void __launch_bounds__(256)
    gram_wide_reduce_kernel(int l, int nparts, const double* __restrict__ part, double* __restrict__ G) {
  const int ll = l * l;
  const int lane8 = threadIdx.x & 7;
  const int e = blockIdx.x * (blockDim.x >> 3) + (threadIdx.x >> 3);
  double s = 0.0;
  if (e < ll) {
    const int i = e / l, c = e - i * l;
    // lower tiles mirror the stored upper ones
    const int src = ((i >> 4) > (c >> 4)) ? c * l + i : e;
    double v[16];
    for (int p0 = lane8; p0 < nparts; p0 += 8 * 16) {
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const int pp = p0 + 8 * u;
        v[u] = pp < nparts ? __ldcg(part + (size_t)pp * ll + src) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 16; ++u) s += v[u];
    }
  }
  s += __shfl_xor_sync(0xffffffffu, s, 1);
  s += __shfl_xor_sync(0xffffffffu, s, 2);
  s += __shfl_xor_sync(0xffffffffu, s, 4);
  if (lane8 == 0 && e < ll) G[e] = s;
}

bool gram_wide_fits(int l, long long m, size_t ws_bytes) {
  if (l < 16 || l > 96 || m < 1024) return false;
  const long long per = (m + num_sms() - 1) / num_sms();
  const int kc = (int)std::max<long long>(16, (per + 15) & ~15LL);
  const long long nparts = (m + kc - 1) / kc;
  return kc <= 256 && (size_t)nparts * l * l * sizeof(double) <= ws_bytes;
}

// G (l x l, row-major) = C C^T; ws: partials (gram_wide_fits checked by the caller)
int gram_wide(int l, long long m, const double* C, double* G, void* ws, cudaStream_t st) {
  const long long per = (m + num_sms() - 1) / num_sms();
  const int kc = (int)std::max<long long>(16, (per + 15) & ~15LL);
  const int nparts = (int)((m + kc - 1) / kc);
  const size_t smem = sizeof(double) * (size_t)l * (kc + 4);
  TTK_TRY(qr_set_smem((const void*)gram_wide_partial_kernel, (int)(sizeof(double) * 96 * (256 + 4))));
  gram_wide_partial_kernel<<<nparts, kGwThreads, smem, st>>>(l, m, kc, C, reinterpret_cast<double*>(ws));
  TTK_CHECK_LAUNCH();
  gram_wide_reduce_kernel<<<(l * l + 31) / 32, 256, 0, st>>>(l, nparts, reinterpret_cast<const double*>(ws), G);
  TTK_CHECK_LAUNCH();
  return kOk;
}

__global__ void copy_strided_kernel(int m, int l, const double* __restrict__ X, long long x_rs,
                                    long long x_cs, double* __restrict__ Y, long long y_rs, long long y_cs) {
  const long long n = (long long)m * l;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    int r, c;
    if (y_cs == 1) { r = (int)(e / l); c = (int)(e - (long long)r * l); }
    else { c = (int)(e / m); r = (int)(e - (long long)c * m); }
    Y[r * y_rs + c * y_cs] = X[r * x_rs + c * x_cs];
  }
}

int copy_strided(int m, int l, const double* X, long long x_rs, long long x_cs, double* Y, long long y_rs,
                 long long y_cs, cudaStream_t st) {
  const long long n = (long long)m * l;
  if (n <= 0) return kOk;
  copy_strided_kernel<<<(int)std::min<long long>((n + 255) / 256, 4 * kNumSMs), 256, 0, st>>>(
      m, l, X, x_rs, x_cs, Y, y_rs, y_cs);
  TTK_CHECK_LAUNCH();
  return kOk;
}


// Pivoted Cholesky of the l x l PSD matrix G (full symmetric storage):
// P^T G P = R^T R with R upper triangular, stopped at the first pivot below
// tau_rel * max(diag G).  Writes rank (device), the leading rank x rank block
// of R compactly (row-major, ld = rank) into Rk and the pivot order into
// perm_out, so that Q2 = Q1[:, perm[:rank]] / Rk (a triangular solve, no
// explicit inverse) has orthonormal-ish columns spanning the numerically
// significant part of range(Q1).
__global__ void __launch_bounds__(1024, 1)
    pchol_kernel(int l, const double* __restrict__ G, double tau_rel, double* __restrict__ Rk,
                 int* perm_out, int* rank_out) {
  extern __shared__ double sm[];
  const int ld = l + 1;
  double* A = sm;
  double* X = sm + l * ld;
  __shared__ int perm[kCholMaxCols + 1];
  __shared__ int piv_s, stop_s;
  __shared__ double d0_s;
  const int tid = threadIdx.x, nt = blockDim.x;
  const int ty = tid >> 5, tx = tid & 31, nty = nt >> 5;
  for (int e = tid; e < l * l; e += nt) {
    int r = e / l, c = e - r * l;
    A[r * ld + c] = G[e];
    X[r * ld + c] = 0.0;
  }
  for (int i = tid; i < l; i += nt) perm[i] = i;
  __syncthreads();
  if (ty == 0) {
    double g = 0.0;
    for (int i = tx; i < l; i += 32) g = fmax(g, A[i * ld + i]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) g = fmax(g, __shfl_xor_sync(0xffffffffu, g, o));
    if (tx == 0) d0_s = g;
  }
  __syncthreads();
  const double thr = tau_rel * d0_s;
  int rank = l;
  for (int j = 0; j < l; ++j) {
    if (ty == 0) {
      double best = -1.0;
      int bi = j;
      for (int i = j + tx; i < l; i += 32) {
        const double v = A[i * ld + i];
        if (v > best) { best = v; bi = i; }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) { best = ob; bi = oi; }
      }
      if (tx == 0) { piv_s = bi; stop_s = !(best > thr); }
    }
    __syncthreads();
    if (stop_s) { rank = j; break; }
    const int p = piv_s;
    if (p != j) {
      for (int e = tid; e < l; e += nt) {
        double t = A[j * ld + e]; A[j * ld + e] = A[p * ld + e]; A[p * ld + e] = t;
      }
      __syncthreads();
      for (int e = tid; e < l; e += nt) {
        double t = A[e * ld + j]; A[e * ld + j] = A[e * ld + p]; A[e * ld + p] = t;
      }
      if (tid == 0) { int t = perm[j]; perm[j] = perm[p]; perm[p] = t; }
      __syncthreads();
    }
    const double rjj = sqrt(A[j * ld + j]);
    const double inv = 1.0 / rjj;
    // trailing update of the full symmetric block with the unscaled row j
    for (int i = j + 1 + ty; i < l; i += nty) {
      const double aji = A[j * ld + i] * inv * inv;
      for (int c = j + 1 + tx; c < l; c += 32) A[i * ld + c] -= aji * A[j * ld + c];
    }
    __syncthreads();
    for (int c = j + 1 + tid; c < l; c += nt) A[j * ld + c] *= inv;
    if (tid == 0) A[j * ld + j] = rjj;
    __syncthreads();
  }
  for (int e = tid; e < rank * rank; e += nt) {
    int r = e / rank, c = e - r * rank;
    Rk[e] = (c >= r) ? A[r * ld + c] : 0.0;
  }
  for (int i = tid; i < l; i += nt) perm_out[i] = perm[i];
  if (tid == 0) *rank_out = rank;
}

// Y[:, c] = X[:, idx[c]] for c < n (column gather, strided output)
__global__ void gather_cols_kernel(int m, int n, const double* __restrict__ X, long long x_rs,
                                   const int* __restrict__ idx, double* __restrict__ Y, long long y_rs,
                                   long long y_cs) {
  const long long tot = (long long)m * n;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < tot;
       e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / n;
    const int c = (int)(e - r * n);
    Y[r * y_rs + (long long)c * y_cs] = X[r * x_rs + idx[c]];
  }
}

// deterministic pseudo-random fill in [-1, 1) (completion directions)
__global__ void fill_random_kernel(long long n, double* x, unsigned long long seed) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    unsigned long long z = (unsigned long long)e * 0x9E3779B97F4A7C15ull + seed;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    x[e] = (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
  }
}

size_t cholqr2_ws_bytes(int m, int l) {
  return align_up((size_t)m * l * 8, 256) + 6 * align_up((size_t)l * l * 8, 256) +
         align_up(sizeof(int) * (16 + kCholMaxCols), 256) + (32u << 20);
}

// Shifted CholeskyQR2/3.  Pass 1 factors G + s I with s = 11 (m l + l(l+1)) u
// trace(G) (Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa 2020), so it
// succeeds for kappa(Y) up to ~1e16 and leaves kappa(Q1) <~ 1e4; pass 2 is
// plain CholeskyQR.  If Q1 was already orthonormal to 1e-3 (||G2 - I||_max),
// Q2 is orthonormal to working precision and we stop; otherwise a third pass
// (checked the same way) finishes.  Exactly rank-deficient inputs fail the
// checks and the caller falls back to Householder TSQR.
// returns kOk and *ok = 1 when the result was accepted
// ---------------------------------------------------------------------------
// Q = Y R^{-1} for an upper-triangular R (l x l, row-major) by forward
// substitution: backward stable (Q R = Y + O(eps |Y|)), unlike a GEMM with an
// explicit inverse whose error grows like eps kappa(R) ||Y|| -- the first
// CholeskyQR pass of a rank-deficient / shifted Gram has kappa(R) up to ~1e8.
// Rows are independent, so Q may alias Y.
// Blocked form: a CTA owns kTbRows rows.  For every 16-column block J the
// off-diagonal part Y_J -= Q_{<J} R_{<J,J} runs on the DMMA pipe
// (block_dmma), and only the 16 x 16 diagonal solve is scalar: four threads
// per row, each owning four columns, pivot value broadcast by shuffle.
// Same backward-stable forward substitution, ~10x fewer instructions.
constexpr int kTbRows = 32, kTbThreads = 128;

__global__ void __launch_bounds__(kTbThreads)
    trsm_blocked_kernel(int m, int l, const double* Y, long long y_rs, long long y_cs,
                        const double* __restrict__ R, double* Q, long long q_rs, long long q_cs) {
  extern __shared__ __align__(16) double tsm[];
  const int ld = ((l + 15) & ~15) + 4;
  double* sR = tsm;                          // l x ld
  double* sY = sR + (size_t)l * ld;          // kTbRows x ld
  double* rinv = sY + (size_t)kTbRows * ld;  // l
  const int tid = threadIdx.x;
  // R and the first Y tile staged asynchronously (one round of load latency)
  for (int e = tid; e < l * l; e += kTbThreads) {
    const int r = e / l, c = e - r * l;
    cp_async8(sR + r * ld + c, R + e, true);
  }
  const int row = tid >> 2, g = tid & 3;
  bool first = true;
  for (long long r0 = (long long)blockIdx.x * kTbRows; r0 < m; r0 += (long long)gridDim.x * kTbRows) {
    __syncthreads();
    for (int e = tid; e < kTbRows * l; e += kTbThreads) {
      const int r = e / l, c = e - r * l;
      const bool ok = r0 + r < m;
      cp_async8(sY + r * ld + c, ok ? Y + (r0 + r) * y_rs + (long long)c * y_cs : Y, ok);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    if (first) {
      for (int j = tid; j < l; j += kTbThreads) rinv[j] = 1.0 / sR[j * ld + j];
      __syncthreads();
      first = false;
    }
    for (int j0 = 0; j0 < l; j0 += 16) {
      const int bs = min(16, l - j0);
      if (j0 > 0) {
        block_dmma(kTbRows, bs, j0, sY, ld, 1, sR + j0, ld, 1, sY + j0, ld, nullptr, nullptr, nullptr, true);
        __syncthreads();
      }
      // diagonal block: thread (row, g) owns columns j0 + g + 4 k
      double t[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = g + 4 * k;
        t[k] = (c < bs) ? sY[row * ld + j0 + c] : 0.0;
      }
#pragma unroll
      for (int jj = 0; jj < 16; ++jj) {
        if (jj < bs) {
          const int kj = jj >> 2;
          double v = t[kj] * rinv[j0 + jj];
          v = __shfl_sync(0xffffffffu, v, (threadIdx.x & ~3) | (jj & 3), 32);
          const double* rr = sR + (j0 + jj) * ld + j0;
          // unconditional update: R is zero below its diagonal (columns c < jj
          // unchanged); the owner's own column (c == jj) is overwritten with v
          // right after, and columns c >= bs are never stored
#pragma unroll
          for (int k = 0; k < 4; ++k) t[k] = fma(-v, rr[g + 4 * k], t[k]);
          if ((jj & 3) == g) t[kj] = v;
        }
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int c = g + 4 * k;
        if (c < bs) sY[row * ld + j0 + c] = t[k];
      }
      __syncthreads();
    }
    for (int e = tid; e < kTbRows * l; e += kTbThreads) {
      const int r = e / l, c = e - r * l;
      if (r0 + r < m) Q[(r0 + r) * q_rs + (long long)c * q_cs] = sY[r * ld + c];
    }
  }
}

// ---------------------------------------------------------------------------
// Fused fast-path CholeskyQR2: one cooperative kernel instead of the chain
// Gram -> split-K reduce -> Cholesky -> TRSM -> Gram -> reduce -> near-identity
// -> (Cholesky) -> Q GEMM -> R GEMM, each link a few microseconds of work behind
// a launch.  CTAs 1..G-1 each keep one kFqRows-row tile of Y (then Q1) in shared
// memory for the whole factorisation; the l x l Gram reductions are spread over
// the grid; CTA 0 holds no tile and factors the two small Gram matrices between
// grid barriers.  Same arithmetic as the unfused path (same Cholesky, TRSM,
// near-identity and DMMA products), fixed reduction order.
constexpr int kFqRows = 128, kFqThreads = 512, kFqMaxCols = 96;
constexpr int kFqTiles = 128;  // target tile CTAs (SMs left free for side-stream work)

struct FqParams {
  int m, l;
  const double* Y;
  long long y_rs, y_cs;
  double* Q;      // row-major, ld q_rs
  long long q_rs;
  double* R;      // l x l or null
  double* part;   // (grid - 1) x l x l partial Gram matrices
  double* G;      // l x l reduced Gram
  double* R1;
  double* R2;
  double* I2;     // R2^{-1}
  int* status;    // [0] first pass, [1] second pass, [4] near-identity flag
  double first_order_max;
  int tr;         // rows per tile CTA
};

__device__ __forceinline__ void fq_reduce(const double* part, int nparts, int l, double* G) {
  const int ll = l * l;
  // 8 lanes per element: lane j sums partials j, j + 8, ... (all loads in
  // flight at once), then a fixed 3-level butterfly -- deterministic, and one
  // L2 round trip instead of nparts dependent ones
  const int lane8 = threadIdx.x & 7;
  const int nthr = (gridDim.x - 1) * (blockDim.x >> 3);
  const int ebase = (blockIdx.x - 1) * (blockDim.x >> 3) + (threadIdx.x >> 3);
  const int iters = (ll + nthr - 1) / nthr;  // uniform trip count: every lane reaches the shuffles
  for (int it = 0; it < iters; ++it) {
    const int e = ebase + it * nthr;
    double s = 0.0;
    if (e < ll) {
      // the partials hold the upper 16 x 16 tiles only: those elements are
      // summed (coalesced) and written to both triangles
      const int ei = e / l, ec = e - ei * l;
      const int src = e;
      double v[16];
      if (in_upper_tiles(ei, ec))
      for (int p0 = lane8; p0 < nparts; p0 += 8 * 16) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int pp = p0 + 8 * u;
          v[u] = pp < nparts ? __ldcg(part + (size_t)pp * ll + src) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) s += v[u];
      }
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    if (lane8 == 0 && e < ll) {
      const int ei = e / l, ec = e - ei * l;
      if (in_upper_tiles(ei, ec)) {
        G[e] = s;
        if ((ei >> 4) != (ec >> 4)) G[ec * l + ei] = s;
      }
    }
  }
}

// The second Gram's reduction also emits the first-order second factor
// elementwise -- R2^{-1} = I - F1 into I2 (and R2 = I + F1 when R is wanted),
// F1 = triu(E) - diag(E)/2, E = G2 - I -- and max |E| into emax_bits (atomicMax
// on the bit pattern of a nonnegative double): in the common case (l |E|^2
// small, see kNearIdFirstOrderMax) CTA 0 has nothing left to factor.
__device__ __forceinline__ void fq_reduce_nearid(const double* part, int nparts, int l, double* G, double* I2,
                                                 double* R2, unsigned long long* emax_bits) {
  const int ll = l * l;
  const int lane8 = threadIdx.x & 7;
  const int nthr = (gridDim.x - 1) * (blockDim.x >> 3);
  const int ebase = (blockIdx.x - 1) * (blockDim.x >> 3) + (threadIdx.x >> 3);
  const int iters = (ll + nthr - 1) / nthr;
  double em = 0.0;
  for (int it = 0; it < iters; ++it) {
    const int e = ebase + it * nthr;
    double s = 0.0;
    if (e < ll) {
      // the partials hold the upper 16 x 16 tiles only: those elements are
      // summed (coalesced) and written to both triangles
      const int ei = e / l, ec = e - ei * l;
      const int src = e;
      double v[16];
      if (in_upper_tiles(ei, ec))
      for (int p0 = lane8; p0 < nparts; p0 += 8 * 16) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          const int pp = p0 + 8 * u;
          v[u] = pp < nparts ? __ldcg(part + (size_t)pp * ll + src) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 16; ++u) s += v[u];
      }
    }
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    if (lane8 == 0 && e < ll) {
      const int r = e / l, c = e - r * l;
      if (in_upper_tiles(r, c)) {
        const double f = (c > r) ? s : (c == r ? 0.5 * (s - 1.0) : 0.0);
        G[e] = s;
        I2[e] = (c > r) ? -f : (c == r ? 1.0 - f : 0.0);
        if (R2) R2[e] = (c > r) ? f : (c == r ? 1.0 + f : 0.0);
        em = fmax(em, fabs(s - (r == c ? 1.0 : 0.0)));
        if ((r >> 4) != (c >> 4)) {  // the mirrored element of a strictly lower tile
          const int mir = c * l + r;
          G[mir] = s;
          I2[mir] = 0.0;
          if (R2) R2[mir] = 0.0;
        }
      }
    }
  }
  if (lane8 == 0 && em > 0.0) atomicMax(emax_bits, (unsigned long long)__double_as_longlong(em));
}

__device__ __forceinline__ void fq_mark(int i) {
  if (g_fq_prof && blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_fq_prof[i] = (long long)t;
  }
}

// LC > 0: the column count as a compile-time constant (the RTO / truncation
// width 80), so every l-bounded loop and block_dmma shape is specialised
template <int LC>
__global__ void __launch_bounds__(kFqThreads, 1) cholqr2_fused_kernel(const __grid_constant__ FqParams P) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  fq_mark(0);
  extern __shared__ __align__(16) double fsm[];
  const int l = LC > 0 ? LC : P.l, ld = ((l + 15) & ~15) + 4, tid = threadIdx.x;
  const bool fac = blockIdx.x == 0;  // the factorisation CTA
  const int tr = P.tr;                        // rows per tile (multiple of 8, <= kFqRows)
  double* sY = fsm;                           // tr x ld   (tile CTAs)
  double* sR = sY + (size_t)tr * ld;          // l x ld
  double* rinv = sR + (size_t)l * ld;         // l
  const long long r0 = (long long)(blockIdx.x - 1) * tr;
  const int rows = fac ? 0 : (int)(P.m - r0 < tr ? P.m - r0 : tr);
  const int nparts = gridDim.x - 1, ll = l * l;
  if (!fac) {
    for (int e = tid; e < tr * l; e += kFqThreads) {
      const int r = e / l, c = e - r * l;
      const bool ok = r < rows;
      cp_async8(sY + r * ld + c, ok ? P.Y + (r0 + r) * P.y_rs + (long long)c * P.y_cs : P.Y, ok);
    }
    cp_async_commit();
    cp_async_wait<0>();
    __syncthreads();
    // Gram partial of the tile (zero rows beyond m contribute nothing)
    block_gram_upper(l, tr, sY, ld, sR, ld);  // upper tiles; the reduction mirrors them
    __syncthreads();
    double* mine = P.part + (size_t)(blockIdx.x - 1) * ll;
    for (int e = tid; e < ll; e += kFqThreads) {
      const int i = e / l, c = e - i * l;
      if (in_upper_tiles(i, c)) mine[e] = sR[i * ld + c];
    }
  }
  grid.sync();
  fq_mark(1);
  if (!fac) fq_reduce(P.part, nparts, l, P.G);
  grid.sync();
  fq_mark(2);
  if (fac) chol_blocked_body(l, P.G, P.R1, nullptr, P.status, 0, 0.0, 1e-15, fsm);
  grid.sync();
  fq_mark(3);
  if (!fac) {
    // Q1 tile = Y tile R1^{-1}: blocked forward substitution (trsm_blocked_kernel's
    // scheme, 4 threads per row), then the tile's partial of Q1^T Q1
    for_each_l2<16>(P.R1, ll, [&](int e, double v) { sR[(e / l) * ld + e % l] = v; });
    __syncthreads();
    for (int j = tid; j < l; j += kFqThreads) rinv[j] = 1.0 / sR[j * ld + j];
    __syncthreads();
    const int row = tid >> 2, g = tid & 3;
    for (int j0 = 0; j0 < l; j0 += 16) {
      const int bs = min(16, l - j0);
      if (j0 > 0) {
        block_dmma(tr, bs, j0, sY, ld, 1, sR + j0, ld, 1, sY + j0, ld, nullptr, nullptr, nullptr, true);
        __syncthreads();
      }
      if (row < tr) {  // warp-uniform: a warp holds 8 rows and tr is a multiple of 8
        double t[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int c = g + 4 * k;
          t[k] = (c < bs) ? sY[row * ld + j0 + c] : 0.0;
        }
#pragma unroll
        for (int jj = 0; jj < 16; ++jj) {
          if (jj < bs) {
            const int kj = jj >> 2;
            double v = t[kj] * rinv[j0 + jj];
            v = __shfl_sync(0xffffffffu, v, (threadIdx.x & ~3) | (jj & 3), 32);
            const double* rr = sR + (j0 + jj) * ld + j0;
            // unconditional update: R is zero below its diagonal (columns c < jj
            // unchanged); the owner's own column (c == jj) is overwritten with v
            // right after, and columns c >= bs are never stored
#pragma unroll
            for (int k = 0; k < 4; ++k) t[k] = fma(-v, rr[g + 4 * k], t[k]);
            if ((jj & 3) == g) t[kj] = v;
          }
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int c = g + 4 * k;
          if (c < bs) sY[row * ld + j0 + c] = t[k];
        }
      }
      __syncthreads();
    }
    if (row >= rows && row < tr)  // padded rows stay zero (rinv scaling of zeros is zero; keep it exact)
      for (int c = g; c < l; c += 4) sY[row * ld + c] = 0.0;
    __syncthreads();
    block_gram_upper(l, tr, sY, ld, sR, ld);  // upper tiles; the reduction mirrors them
    __syncthreads();
    double* mine = P.part + (size_t)(blockIdx.x - 1) * ll;
    for (int e = tid; e < ll; e += kFqThreads) {
      const int i = e / l, c = e - i * l;
      if (in_upper_tiles(i, c)) mine[e] = sR[i * ld + c];
    }
  }
  grid.sync();
  fq_mark(4);
  unsigned long long* emax_bits = reinterpret_cast<unsigned long long*>(P.status + 6);
  if (!fac) fq_reduce_nearid(P.part, nparts, l, P.G, P.I2, P.R ? P.R2 : nullptr, emax_bits);
  grid.sync();
  fq_mark(5);
  // every CTA reads the same max |E| after the barrier: a uniform branch
  const double emax = __longlong_as_double((long long)*(volatile unsigned long long*)emax_bits);
  const bool first_order = (double)l * emax * emax <= P.first_order_max;
  if (!first_order && fac) {
    // second-order series or, beyond 1e-7, a full Cholesky of G2 (rare)
    chol_near_identity_body(l, P.G, P.R2, P.I2, P.status + 4, 1e-7, P.first_order_max, fsm);
    __syncthreads();
    if (!*(volatile int*)(P.status + 4))
      chol_blocked_body(l, P.G, P.R2, P.I2, P.status + 1, 1, 0.0, 1e-28, fsm);
    __syncthreads();
  }
  if (fac) {
    if (P.R) {  // R = R2 R1
      double* a = fsm;
      double* b = fsm + (size_t)l * ld;
      for (int e = tid; e < ll; e += kFqThreads) {
        a[(e / l) * ld + e % l] = __ldcg(P.R2 + e);
        b[(e / l) * ld + e % l] = __ldcg(P.R1 + e);
      }
      __syncthreads();
      block_dmma(l, l, l, a, ld, 1, b, ld, 1, P.R, l);
    }
  }
  if (!first_order) grid.sync();  // the Q phase reads the I2 CTA 0 just wrote
  fq_mark(6);
  if (!fac) {
    // Q tile = Q1 tile R2^{-1}
    for_each_l2<16>(P.I2, ll, [&](int e, double v) { sR[(e / l) * ld + e % l] = v; });
    __syncthreads();
    block_dmma(rows, l, l, sY, ld, 1, sR, ld, 1, P.Q + r0 * P.q_rs, (int)P.q_rs);
  }
  if (g_fq_prof) {  // diagnostics only: the kernel's end orders the Q tiles
    grid.sync();
    fq_mark(15);
  }
}

size_t cholqr2_fused_smem(int l, int tr) {
  const size_t ld = ((l + 15) & ~15) + 4;
  const size_t tile = (size_t)tr * ld + (size_t)l * ld + ((l + 1) & ~1);
  const size_t fac = 2 * (size_t)l * ld + 256 * (size_t)((l + 15) / 16);
  return sizeof(double) * std::max(tile, fac);
}

bool cholqr2_fused_fits(int m, int l, long long q_cs) {
  static const bool off = knob_env("TTK_QR_NO_FUSED") != nullptr;  // A/B
  return !off && l <= kFqMaxCols && m >= l && q_cs == 1 && (m + kFqRows - 1) / kFqRows <= num_sms() - 1 &&
         cholqr2_fused_smem(l, kFqRows) <= 220 * 1024;
}

// Precondition: R's strict lower triangle is exactly zero and finite -- the
// blocked off-diagonal update multiplies whole 16 x 16 blocks of R without
// masking.  Every producer (chol_blocked_body, pchol, the near-identity series)
// stores zeros there.
int trsm_right_upper(int m, int l, const double* Y, long long y_rs, long long y_cs, const double* R, double* Q,
                     long long q_rs, long long q_cs, cudaStream_t st) {
  if (m <= 0 || l <= 0) return kOk;
  TTK_REQUIRE(l <= 128, kInvalidValue, "trsm: %d columns exceed 128", l);
  {  // per-device attributes (set_attr_once)
    TTK_TRY(qr_set_smem((const void*)trsm_blocked_kernel, 220 * 1024));
  }
  const int ld = ((l + 15) & ~15) + 4;
  const size_t smem = sizeof(double) * ((size_t)l * ld + (size_t)kTbRows * ld + l);
  const int grid = (int)std::min<long long>((m + kTbRows - 1) / kTbRows, 4LL * kNumSMs);
  trsm_blocked_kernel<<<grid, kTbThreads, smem, st>>>(m, l, Y, y_rs, y_cs, R, Q, q_rs, q_cs);
  TTK_CHECK_LAUNCH();
  return kOk;
}

static int g_qr_path_tmp = 0;
static void g_qr_last_path_set(int v) { g_qr_path_tmp = v; }
// unit-norm columns of an m x n strided block, one CTA per column, fixed
// reduction order; an exactly-zero column becomes a deterministic
// pseudo-random unit vector (it then carries a noise direction of the
// completion, which the joint CholeskyQR orthonormalises)
__global__ void normalize_cols_kernel(int m, int n, double* X, long long x_rs, long long x_cs,
                                      unsigned long long seed) {
  __shared__ double red[32];
  const int c = blockIdx.x;
  if (c >= n) return;
  double* col = X + (long long)c * x_cs;
  for (int pass = 0; pass < 2; ++pass) {
    double s = 0.0;
    for (int r = threadIdx.x; r < m; r += blockDim.x) { const double v = col[(long long)r * x_rs]; s += v * v; }
    s = warp_sum(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    double tot = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    __syncthreads();
    if (tot > 0.0) {
      const double inv = 1.0 / sqrt(tot);
      for (int r = threadIdx.x; r < m; r += blockDim.x) col[(long long)r * x_rs] *= inv;
      return;
    }
    for (int r = threadIdx.x; r < m; r += blockDim.x) {
      unsigned long long z = ((unsigned long long)c * 0x9E3779B97F4A7C15ull) ^ ((unsigned long long)r + seed);
      z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
      z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
      z ^= z >> 31;
      col[(long long)r * x_rs] = (double)(z >> 11) * (2.0 / 9007199254740992.0) - 1.0;
    }
    __syncthreads();
  }
}

// CholeskyQR2 with a rank-robust fallback, entirely on the DMMA GEMMs and the
// small one-CTA factorisations.
//   fast path (skipped when robust_first): Gram -> Cholesky -> TRSM -> Gram ->
//     near-identity series -> GEMM; accepted iff both factorisations succeed
//     and ||Q1^T Q1 - I||_max <= 1e-3.
//   robust path (exactly rank-deficient or ill-conditioned Y):
//     1. shifted CholeskyQR pass (Fukaya et al. 2020) + TRSM -> Q1, always succeeds;
//     2. pivoted Cholesky of Q1^T Q1 finds rho significant directions; CholeskyQR
//        on the gathered pivot columns (TRSM) -> Q2 = Q[:, :rho];
//     3. completion aligned with what step 2 dropped: Om = (I - Q2 Q2^T) Y Omega
//        (projected twice), columns normalised -> Q[:, rho:];
//     4. ONE joint CholeskyQR2 of [Q2 | Om] makes the whole Q orthonormal to
//        working precision (this also removes the eps-sized leftovers of Om along
//        Q2 that a separate orthonormalisation of Om would amplify by kappa(Om));
//     5. R = Q^T Y (range(Q) covers range(Y) to working precision).
//   *deficient is set to 1 when Y needed the robust path with rho < l, so a sweep
//   can try it first on the next core (fewer launches, one host sync less).
// defer_status (optional, 8 device ints, zeroed by the caller): the fused
// kernel's acceptance flags go there and the host does NOT wait for them --
// *ok = 1 optimistically; the caller checks [0] and [1] of every slot later
// and redoes its sweep without deferral if one is nonzero.
int cholqr2(int m, int l, const double* Y, long long y_rs, long long y_cs, double* Q, long long q_rs,
            long long q_cs, double* R, void* ws, size_t ws_bytes, cudaStream_t st, int* ok,
            bool robust_first, int* deficient, int* defer_status = nullptr, int* fused_ok = nullptr) {
  *ok = 0;
  if (deficient) *deficient = 0;
  if (l > kCholMaxCols || m < l) return kOk;
  TTK_REQUIRE(ws_bytes >= cholqr2_ws_bytes(m, l), kWorkspace, "cholqr: workspace too small");
  Arena ar(ws, ws_bytes);
  double* Q1 = ar.take<double>((size_t)m * l);
  double* G = ar.take<double>((size_t)l * l);
  double* R1 = ar.take<double>((size_t)l * l);
  double* I1 = ar.take<double>((size_t)l * l);
  double* R2 = ar.take<double>((size_t)l * l);
  double* I2 = ar.take<double>((size_t)l * l);
  int* status = ar.take<int>(16 + kCholMaxCols);  // [0,8) flags/rank, [8, 8+l) pivot order
  void* split = ar.take<char>(32u << 20);
  const size_t split_bytes = 32u << 20;
  const size_t smem = sizeof(double) * (2 * (size_t)l * (l + 1) + 256 * (size_t)((l + 15) / 16));
  const double shift_rel = 11.0 * ((double)m * l + (double)l * (l + 1)) * 1.1102230246251565e-16;
  GemmProblem p;
  auto gram = [&](const double* X, long long x_rs, long long x_cs) -> int {
    GemmProblem g = make_gemm(l, l, m, X, x_cs, x_rs, X, x_rs, x_cs, G, l, 1);
    return gemm_group_launch(&g, 1, split, split_bytes, st);
  };
  // one pass: Gram of X, Cholesky (+shift) into (Rk, Ik); second passes (checked
  // against I) try the near-identity series first; first passes feed a
  // triangular solve and need no inverse
  auto gram_chol = [&](const double* X, long long x_rs, long long x_cs, double* Rk, double* Ik, int* st_slot,
                       int check, double shift, double tiny) -> int {
    TTK_TRY(gram(X, x_rs, x_cs));
    TTK_TRY(launch_chol_inv(l, G, Rk, check ? Ik : nullptr, st_slot, check, shift, tiny, st,
                            check ? status + 4 : nullptr));
    return kOk;
  };
  int hs[4] = {0, 0, 0, 0};
  static const int qr_mode = knob_env("TTK_QR_MODE") ? atoi(knob_env("TTK_QR_MODE")) : 0;
  bool fast_tried = false;
  if ((!robust_first || qr_mode == 2) && cholqr2_fused_fits(m, l, q_cs)) {
    // ---- fast path, fused into one cooperative kernel ----
    {  // per-device attributes (set_attr_once)
      TTK_TRY(qr_set_smem((const void*)cholqr2_fused_kernel<0>, 220 * 1024));
      TTK_TRY(qr_set_smem((const void*)cholqr2_fused_kernel<80>, 220 * 1024));
    }
    static const double fo = knob_env("TTK_NEAR_ID_FIRST_ORDER") ? atof(knob_env("TTK_NEAR_ID_FIRST_ORDER"))
                                                                   : kNearIdFirstOrderMax;
    int* const fstatus = defer_status ? defer_status : status;
    if (!defer_status) TTK_CHECK_CUDA(cudaMemsetAsync(status, 0, 8 * sizeof(int), st));
    FqParams fp{};
    fp.m = m; fp.l = l; fp.Y = Y; fp.y_rs = y_rs; fp.y_cs = y_cs; fp.Q = Q; fp.q_rs = q_rs; fp.R = R;
    fp.part = (double*)split; fp.G = G; fp.R1 = R1; fp.R2 = R2; fp.I2 = I2; fp.status = fstatus;
    fp.first_order_max = fo;
    // tile rows: spread the tall dimension over up to kFqTiles CTAs (the tile
    // phases are per-SM DMMA work: 10240 x 80 in 80-row tiles instead of 128);
    // TTK_FQ_ROWS pins it (A/B)
    static const int fq_rows = knob_env("TTK_FQ_ROWS") ? atoi(knob_env("TTK_FQ_ROWS")) : 0;
    int trows = fq_rows > 0 ? fq_rows : (int)(((m + kFqTiles - 1) / kFqTiles + 7) & ~7);
    trows = std::max(8, std::min(kFqRows, (trows + 7) & ~7));
    fp.tr = trows;
    const int grid = 1 + (m + trows - 1) / trows;
    void* args[] = {&fp};
    static const bool lc_off = knob_env("TTK_FQ_LC") && atoi(knob_env("TTK_FQ_LC")) == 0;  // A/B
    const void* fq_fn = (l == 80 && !lc_off) ? (const void*)cholqr2_fused_kernel<80> : (const void*)cholqr2_fused_kernel<0>;
    const cudaError_t le = cudaLaunchCooperativeKernel(fq_fn, dim3(grid),
                                                       dim3(kFqThreads), args, cholqr2_fused_smem(l, trows), st);
    if (le == cudaSuccess) {
      fast_tried = true;
      TTK_CHECK_LAUNCH();
      if (defer_status) {  // flags checked by the caller after its sweep
        *ok = 1;
        g_qr_last_path_set(1);
        return kOk;
      }
      TTK_CHECK_CUDA(cudaMemcpyAsync(hs, status, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
      TTK_SYNC(st);
      if (hs[0] == 0 && hs[1] == 0) {
        *ok = 1;
        if (fused_ok) *fused_ok = 1;
        g_qr_last_path_set(1);
        return kOk;
      }
      if (qr_mode == 2) return kOk;
    } else {
      (void)cudaGetLastError();  // cooperative launch refused (co-residency): unfused chain below
    }
  }
  if (!fast_tried && (!robust_first || qr_mode == 2)) {
    // ---- fast path: CholeskyQR2, accepted for kappa(Y) <~ 3e7 ----
    TTK_CHECK_CUDA(cudaMemsetAsync(status, 0, 4 * sizeof(int), st));
    TTK_TRY(gram_chol(Y, y_rs, y_cs, R1, I1, status, 0, 0.0, 1e-15));
    TTK_TRY(trsm_right_upper(m, l, Y, y_rs, y_cs, R1, Q1, l, 1, st));  // Q1 = Y / R1 (backward stable)
    TTK_TRY(gram_chol(Q1, l, 1, R2, I2, status + 1, 1, 0.0, 1e-28));
    static const bool assume_fast = knob_env("TTK_QR_ASSUME_FAST") != nullptr;  // diagnostics: cost of this sync
    if (!assume_fast) {
      TTK_CHECK_CUDA(cudaMemcpyAsync(hs, status, 2 * sizeof(int), cudaMemcpyDeviceToHost, st));
      TTK_SYNC(st);
    }
    if (hs[0] == 0 && hs[1] == 0) {
      p = make_gemm(m, l, l, Q1, l, 1, I2, l, 1, Q, q_rs, q_cs);
      TTK_TRY(gemm_group_launch(&p, 1, split, split_bytes, st));
      if (R) {
        p = make_gemm(l, l, l, R2, l, 1, R1, l, 1, R, l, 1);
        TTK_TRY(gemm_group_launch(&p, 1, split, split_bytes, st));
      }
      *ok = 1;
      g_qr_last_path_set(1);
      return kOk;
    }
    if (qr_mode == 2) return kOk;  // diagnostics: fast path or Householder only
  }
  // ---- rank-robust path ----
  // 1. shifted pass: always succeeds, kappa(Q1) <~ 1e5 on the significant part of range(Y)
  TTK_CHECK_CUDA(cudaMemsetAsync(status, 0, 4 * sizeof(int), st));
  TTK_TRY(gram_chol(Y, y_rs, y_cs, R1, I1, status, 0, shift_rel, 1e-28));
  TTK_TRY(trsm_right_upper(m, l, Y, y_rs, y_cs, R1, Q1, l, 1, st));
  // 2. pivoted Cholesky of Q1^T Q1: directions with eigenvalue < 1e-14 are left to the completion
  TTK_TRY(gram(Q1, l, 1));
  {
    {  // per-device attributes (set_attr_once)
      TTK_TRY(qr_set_smem((const void*)pchol_kernel, 220 * 1024));
    }
    pchol_kernel<<<1, 1024, smem, st>>>(l, G, 1e-14, R2, status + 8, status + 3);
    TTK_CHECK_LAUNCH();
  }
  TTK_CHECK_CUDA(cudaMemcpyAsync(hs, status, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
  TTK_SYNC(st);
  if (hs[0] & 1) return kOk;
  const int rho = hs[3];
  if (deficient) *deficient = rho < l;
  if (rho > 0) {
    gather_cols_kernel<<<(int)std::min<long long>(((long long)m * rho + 255) / 256, 4 * kNumSMs), 256, 0, st>>>(
        m, rho, Q1, l, status + 8, Q, q_rs, q_cs);
    TTK_CHECK_LAUNCH();
    TTK_TRY(trsm_right_upper(m, rho, Q, q_rs, q_cs, R2, Q, q_rs, q_cs, st));
  }
  if (rho < l) {
    // 3. completion Om = (I - Q2 Q2^T) Y Omega, written into Q[:, rho:]
    const int kc = l - rho;
    double* Om = Q + (long long)rho * q_cs;
    fill_random_kernel<<<8, 256, 0, st>>>((long long)l * kc, I2, 0x5DEECE66Dull + (unsigned)l);
    TTK_CHECK_LAUNCH();
    p = make_gemm(m, kc, l, Y, y_rs, y_cs, I2, kc, 1, Om, q_rs, q_cs);
    TTK_TRY(gemm_group_launch(&p, 1, split, split_bytes, st));
    for (int rep = 0; rep < 2 && rho > 0; ++rep) {
      p = make_gemm(rho, kc, m, Q, q_cs, q_rs, Om, q_rs, q_cs, G, kc, 1);
      TTK_TRY(gemm_group_launch(&p, 1, split, split_bytes, st));
      p = make_gemm(m, kc, rho, Q, q_rs, q_cs, G, kc, 1, Om, q_rs, q_cs, -1.0, 1.0);
      TTK_TRY(gemm_group_launch(&p, 1, split, split_bytes, st));
    }
    normalize_cols_kernel<<<kc, 256, 0, st>>>(m, kc, Om, q_rs, q_cs, 0x2545F4914F6CDD1Dull + (unsigned)l);
    TTK_CHECK_LAUNCH();
    // 4. joint CholeskyQR2 of [Q2 | Om] (in place through the Q1 scratch)
    TTK_CHECK_CUDA(cudaMemsetAsync(status + 2, 0, 2 * sizeof(int), st));
    TTK_TRY(gram_chol(Q, q_rs, q_cs, R1, I1, status + 2, 0, 0.0, 1e-28));
    TTK_TRY(trsm_right_upper(m, l, Q, q_rs, q_cs, R1, Q1, l, 1, st));
    TTK_TRY(gram_chol(Q1, l, 1, R2, I2, status + 2, 1, 0.0, 1e-28));
    p = make_gemm(m, l, l, Q1, l, 1, I2, l, 1, Q, q_rs, q_cs);
    TTK_TRY(gemm_group_launch(&p, 1, split, split_bytes, st));
  } else {
    // Q2 spans all of range(Y): one more CholeskyQR pass to working precision
    TTK_CHECK_CUDA(cudaMemsetAsync(status + 2, 0, 2 * sizeof(int), st));
    TTK_TRY(gram_chol(Q, q_rs, q_cs, R1, I1, status + 2, 1, 0.0, 1e-28));
    p = make_gemm(m, l, l, Q, q_rs, q_cs, I1, l, 1, Q1, l, 1);
    TTK_TRY(gemm_group_launch(&p, 1, split, split_bytes, st));
    TTK_TRY(copy_strided(m, l, Q1, l, 1, Q, q_rs, q_cs, st));
  }
  TTK_CHECK_CUDA(cudaMemcpyAsync(hs, status, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
  TTK_SYNC(st);
  if (hs[2] & 1) return kOk;  // joint Cholesky broke down: Householder fallback
  g_qr_last_path_set(2 + 100 * rho);
  if (R) {
    // 5. R = Q^T Y (l x l): exact to working precision because range(Q) covers range(Y)
    p = make_gemm(l, l, m, Q, q_cs, q_rs, Y, y_rs, y_cs, R, l, 1);
    TTK_TRY(gemm_group_launch(&p, 1, split, split_bytes, st));
  }
  *ok = 1;
  return kOk;
}

size_t qr_auto_ws_bytes(int m, int l) {
  if (l > kQrMaxCols) return qr_blocked_ws_bytes(m, l);
  size_t a = tsqr_ws_bytes(m, l);
  size_t b = (l <= kCholMaxCols && m >= l) ? cholqr2_ws_bytes(m, l) + align_up((size_t)m * l * 8, 256) : 0;
  return std::max(a, b);
}

// diagnostics (TTK_QR_CHECK=1): host-side check of every CholeskyQR factorisation
static const bool g_qr_check = knob_env("TTK_QR_CHECK") != nullptr;
#define g_qr_last_path g_qr_path_tmp  // 1 fast, 2 + 100 rho robust
static void qr_check_report(int m, int l, const std::vector<double>& hy, const double* Q, long long q_rs,
                            long long q_cs, const double* R, cudaStream_t st) {
  cudaStreamSynchronize(st);
  std::vector<double> hq((size_t)m * l), hr((size_t)l * l);
  double* tmp = nullptr;
  cudaMalloc(&tmp, 8 * (size_t)m * l);
  copy_strided(m, l, Q, q_rs, q_cs, tmp, l, 1, st);
  cudaStreamSynchronize(st);
  cudaMemcpy(hq.data(), tmp, 8 * (size_t)m * l, cudaMemcpyDeviceToHost);
  cudaFree(tmp);
  cudaMemcpy(hr.data(), R, 8 * (size_t)l * l, cudaMemcpyDeviceToHost);
  double orth = 0, rec = 0, ymax = 0;
  for (int i = 0; i < l; ++i)
    for (int j = 0; j < l; ++j) {
      double s = 0;
      for (int r = 0; r < m; ++r) s += hq[(size_t)r * l + i] * hq[(size_t)r * l + j];
      orth = std::max(orth, std::fabs(s - (i == j)));
    }
  for (int r = 0; r < m; ++r)
    for (int c = 0; c < l; ++c) {
      double s = 0;
      for (int k = 0; k < l; ++k) s += hq[(size_t)r * l + k] * hr[(size_t)k * l + c];
      rec = std::max(rec, std::fabs(s - hy[(size_t)r * l + c]));
      ymax = std::max(ymax, std::fabs(hy[(size_t)r * l + c]));
    }
  fprintf(stderr, "qrcheck path=%d m=%d l=%d orth=%.2e rec=%.2e\n", g_qr_last_path, m, l, orth, rec / ymax);
}

int qr_auto(int m, int l, const double* A, long long a_rs, long long a_cs, double* Q, long long q_rs,
            long long q_cs, double* R, void* ws, size_t ws_bytes, cudaStream_t st, int* hint, int* defer_status,
            int* fused_ok) {
  if (fused_ok) *fused_ok = 0;
  if (m <= 0 || l <= 0) return kOk;
  if (l > kQrMaxCols) {
    TTK_REQUIRE(l <= kWideMaxCols, kInvalidValue, "qr: %d x %d exceeds %d columns", m, l, kWideMaxCols);
    return qr_blocked(m, l, A, a_rs, a_cs, Q, q_rs, q_cs, R, ws, ws_bytes, st);
  }
  // CholeskyQR2 pays off only for tall inputs that need a multi-panel tree
  static const int qr_mode = knob_env("TTK_QR_MODE") ? atoi(knob_env("TTK_QR_MODE")) : 0;  // 1: Householder only
  // (r01: Householder 128 x 80 400 us vs 246, 256 x 40 235 vs 100, 512 x 100 1986 vs
  // 140; only the smallest panels, e.g. 32 x 20 43 vs 76 us, stay on Householder)
  if (qr_mode != 1 && l <= kCholMaxCols && ((m >= 4 * l && m > 512) || (m >= l && l >= 32))) {
    int ok = 0;
    const double* Y = A;
    long long y_rs = a_rs, y_cs = a_cs;
    void* cws = ws;
    size_t cbytes = ws_bytes;
    if ((const void*)A == (const void*)Q) {
      // in-place call (the rank-robust path reads Y after writing Q): work on a copy
      double* Ycopy = reinterpret_cast<double*>(ws);
      const size_t cb = align_up((size_t)m * l * 8, 256);
      TTK_REQUIRE(ws_bytes >= cb, kWorkspace, "qr_auto: workspace too small");
      TTK_TRY(copy_strided(m, l, A, a_rs, a_cs, Ycopy, l, 1, st));
      Y = Ycopy; y_rs = l; y_cs = 1;
      cws = (char*)ws + cb;
      cbytes = ws_bytes - cb;
    }
    std::vector<double> hy;
    if (g_qr_check) {  // diagnostics: keep the input for the factorisation check
      hy.resize((size_t)m * l);
      double* tmp = nullptr;
      TTK_CHECK_CUDA(cudaMalloc(&tmp, 8 * (size_t)m * l));
      TTK_TRY(copy_strided(m, l, Y, y_rs, y_cs, tmp, l, 1, st));
      TTK_SYNC(st);
      TTK_CHECK_CUDA(cudaMemcpy(hy.data(), tmp, 8 * (size_t)m * l, cudaMemcpyDeviceToHost));
      cudaFree(tmp);
    }
    int deficient = 0;
    TTK_TRY(cholqr2(m, l, Y, y_rs, y_cs, Q, q_rs, q_cs, R, cws, cbytes, st, &ok, hint && *hint, &deficient,
                    defer_status, fused_ok));
    if (hint) *hint = ok && deficient;
    if (ok && g_qr_check && R) qr_check_report(m, l, hy, Q, q_rs, q_cs, R, st);
    if (ok) return kOk;
  }
  return tsqr(m, l, A, a_rs, a_cs, Q, q_rs, q_cs, R, ws, ws_bytes, st);
}

}  // namespace ttk
