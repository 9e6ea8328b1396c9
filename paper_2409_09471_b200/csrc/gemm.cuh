// Grouped fp64 GEMM on the FP64 tensor pipe (DMMA.8x8x4 via mma.sync.m8n8k4.f64).
//
// Every TT contraction on the hot path (matvec cores, RTO partial
// contractions, projections, Gram/dot sweeps, stream-sketch sweeps) reduces to
//   C(m,n) = alpha * sum_k A(m,k) B(k,n) + beta * C(m,n)
// where the row/column index maps are *two-level affine*:
//   A(m,k) = A[(m / a_mdiv) * a_ms1 + (m % a_mdiv) * a_ms0 + k * a_ks]
//   B(k,n) = B[(n / b_ndiv) * b_ns1 + (n % b_ndiv) * b_ns0 + k * b_ks]
//   C(m,n) = C[(m / c_mdiv) * c_ms1 + (m % c_mdiv) * c_ms0
//              + (n / c_ndiv) * c_ns1 + (n % c_ndiv) * c_ns0]
// which covers plain/transposed/strided GEMMs and the rank-merged
// (vector-rank major, operator-rank minor) output layout of tt_matvec.
// Operands are staged through a 3-stage cp.async shared-memory pipeline; the
// per-row/column offsets are tabulated once per tile in shared memory.
#pragma once
#include "common.cuh"

namespace ttk {

struct GemmProblem {
  const double* A;
  const double* B;
  double* C;
  double* partial;  // split-K partials: splits * M * N (row-major), nullptr if splits == 1
  long long a_ms0, a_ms1, a_ks;
  long long b_ns0, b_ns1, b_ks;
  long long c_ms0, c_ms1, c_ns0, c_ns1;
  double alpha, beta;
  int M, N, K;
  int a_mdiv, b_ndiv, c_mdiv, c_ndiv;
  int splits, k_per_split;
  int tiles_m, tiles_n;
  int tile_begin;  // first CTA index of this problem within the group launch
};

constexpr int kMaxGroup = 96;
constexpr int kSmallGroup = 4;  // kernel-parameter size ~0.7 KB instead of ~17 KB

template <int CAP>
struct GemmGroupT {
  int count;
  int total_tiles;
  GemmProblem p[CAP];
};
using GemmGroup = GemmGroupT<kMaxGroup>;
using GemmGroupSmall = GemmGroupT<kSmallGroup>;

__device__ __forceinline__ long long amap(const GemmProblem& P, int m) {
  int q = m / P.a_mdiv;
  return (long long)q * P.a_ms1 + (long long)(m - q * P.a_mdiv) * P.a_ms0;
}
__device__ __forceinline__ long long bmap(const GemmProblem& P, int n) {
  int q = n / P.b_ndiv;
  return (long long)q * P.b_ns1 + (long long)(n - q * P.b_ndiv) * P.b_ns0;
}
__device__ __forceinline__ long long cmap_m(const GemmProblem& P, int m) {
  int q = m / P.c_mdiv;
  return (long long)q * P.c_ms1 + (long long)(m - q * P.c_mdiv) * P.c_ms0;
}
__device__ __forceinline__ long long cmap_n(const GemmProblem& P, int n) {
  int q = n / P.c_ndiv;
  return (long long)q * P.c_ns1 + (long long)(n - q * P.c_ndiv) * P.c_ns0;
}

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES>
struct GemmCfg {
  static constexpr int kThreads = 32 * WARPS_M * WARPS_N;
  static constexpr int WM = BM / WARPS_M;  // rows per warp
  static constexpr int WN = BN / WARPS_N;  // cols per warp
  static constexpr int FM = WM / 8;        // 8x8 fragments per warp along m
  static constexpr int FN = WN / 8;
  static constexpr int SA = BM + 4;  // smem row stride (doubles) of the k-major A tile
  static constexpr int SB = BN + 4;
  // rows m and m + 8 of every 16-row group stored side by side, so fragment
  // pairs (i, i + 1) come from one 16-byte shared load (needs even FM / FN)
  static constexpr bool kPairA = (FM % 2 == 0);
  static constexpr bool kPairB = (FN % 2 == 0);
  static constexpr int NA = (BM * BK + kThreads - 1) / kThreads;  // A elements per thread per stage
  static constexpr int NB = (BN * BK + kThreads - 1) / kThreads;
  static constexpr size_t kSmemBytes =
      sizeof(double) * (size_t)STAGES * BK * (SA + SB) + sizeof(long long) * (BM + BN) * 2;
  static_assert(BM % (8 * WARPS_M) == 0 && BN % (8 * WARPS_N) == 0, "tile");
  static_assert(BK % 4 == 0, "bk");
  static_assert(SA % 16 == 4 && SB % 16 == 4, "bank-conflict-free fragment loads");
};

// position of tile row m in a paired shared layout
template <bool PAIR>
__device__ __forceinline__ int pair_pos(int m) {
  if constexpr (PAIR) return (m & ~15) | ((m & 7) << 1) | ((m >> 3) & 1);
  else return m;
}

// Per-thread load plan for one operand tile (E x BK elements, E = BM or BN):
// each thread always copies the same (row, k) slots, so its source offsets
// (32-bit element offsets from the operand base; the host checks that every
// operand fits) and shared destinations (byte offsets within a stage) are
// computed once per tile.  Per stage and element: one 64-bit add, one 32-bit
// add and the cp.async; rows outside the problem and (on the last stage) k
// beyond the slice are zero-filled through cp.async's src-size operand, so the
// source pointer never needs a select.
template <int E, int BK, int T, int NE, bool PAIR, int S>
struct TileLoader {
  const double* base;
  int off[NE];
  int dk[NE];      // (dst byte offset << 8) | k, -1 if the slot is unused
  unsigned valid;  // bit i: row in range
  __device__ __forceinline__ void init(const double* b, const long long* rowoff, long long ks, int r0, int rows) {
    base = b;
    valid = 0;
    const int tid = threadIdx.x;
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      const int e = tid + i * T;
      int r, k;
      if (ks == 1) { k = e % BK; r = e / BK; } else { r = e % E; k = e / E; }
      const bool used = e < E * BK;
      const bool ok = used && (r0 + r < rows);
      off[i] = ok ? (int)(rowoff[r] + (long long)k * ks) : 0;
      dk[i] = used ? ((((k * S + pair_pos<PAIR>(r)) * 8) << 8) | k) : -1;
      if (ok) valid |= 1u << i;
    }
  }
  // full = every k of the stage lies inside the slice (all but the last stage)
  template <bool FULL>
  __device__ __forceinline__ void load(uint32_t smem_stage, long long koff, int kleft) const {
    const double* gb = base + koff;
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      if ((i + 1) * T > E * BK && dk[i] < 0) continue;  // only the last slot can be unused
      bool ok = (valid >> i) & 1u;
      if constexpr (!FULL) ok = ok && ((dk[i] & 255) < kleft);
      cp_async8_s(smem_stage + (uint32_t)(dk[i] >> 8), gb + off[i], ok);
    }
  }
  // the per-element form (k bound tested on every stage, source selected):
  // measured faster for the grouped tt_matvec launch (24.4 vs 22.5 TF/s, its
  // L2-bound operand stream), slower on single large GEMMs
  __device__ __forceinline__ void load_classic(uint32_t smem_stage, long long koff, int kleft) const {
#pragma unroll
    for (int i = 0; i < NE; ++i) {
      if ((i + 1) * T > E * BK && dk[i] < 0) continue;
      const bool ok = ((valid >> i) & 1u) && ((dk[i] & 255) < kleft);
      const double* src = base + koff + off[i];
      cp_async8_s(smem_stage + (uint32_t)(dk[i] >> 8), ok ? src : base, ok);
    }
  }
};

// at most ~128 registers per thread: >= 16 resident warps per SM keep the
// DMMA pipe fed (a warp cannot issue DMMAs back to back)
// (full-width rank-80 warps with >= 20 fragments keep their registers)
template <int BM, int BN, int WARPS_M, int WARPS_N>
constexpr int gemm_min_blocks() {
  constexpr int frags = (BM / WARPS_M / 8) * (BN / WARPS_N / 8);
  constexpr int mb = 65536 / (32 * WARPS_M * WARPS_N * 128);
  return (frags >= 20 || mb < 1) ? 1 : mb;
}

template <int BM, int BN, int BK, int WARPS_M, int WARPS_N, int STAGES, int CAP>
__global__ void __launch_bounds__(32 * WARPS_M * WARPS_N, gemm_min_blocks<BM, BN, WARPS_M, WARPS_N>())
    gemm_group_kernel(const __grid_constant__ GemmGroupT<CAP> G) {
  using Cfg = GemmCfg<BM, BN, BK, WARPS_M, WARPS_N, STAGES>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* As = reinterpret_cast<double*>(smem_raw);
  double* Bs = As + STAGES * BK * Cfg::SA;
  long long* rowA = reinterpret_cast<long long*>(Bs + STAGES * BK * Cfg::SB);
  long long* colB = rowA + BM;
  long long* rowC = colB + BN;
  long long* colC = rowC + BM;

  // locate the problem owning this CTA
  int bid = blockIdx.x;
  int pi = 0;
  {
    int lo = 0, hi = G.count - 1;
    while (lo < hi) {
      int mid = (lo + hi + 1) >> 1;
      if (G.p[mid].tile_begin <= bid) lo = mid; else hi = mid - 1;
    }
    pi = lo;
  }
  const GemmProblem& P = G.p[pi];
  int t = bid - P.tile_begin;
  const int split = t % P.splits;
  t /= P.splits;
  const int tn = t % P.tiles_n;
  const int tm = t / P.tiles_n;
  const int m0 = tm * BM, n0 = tn * BN;
  const int kbeg = split * P.k_per_split;
  const int kend = min(P.K, kbeg + P.k_per_split);
  const long long a_ks = P.a_ks, b_ks = P.b_ks;

  for (int i = threadIdx.x; i < BM; i += Cfg::kThreads) {
    int m = min(m0 + i, P.M - 1);
    rowA[i] = amap(P, m);
    rowC[i] = cmap_m(P, m);
  }
  for (int i = threadIdx.x; i < BN; i += Cfg::kThreads) {
    int n = min(n0 + i, P.N - 1);
    colB[i] = bmap(P, n);
    colC[i] = cmap_n(P, n);
  }
  __syncthreads();

  TileLoader<BM, BK, Cfg::kThreads, Cfg::NA, Cfg::kPairA, Cfg::SA> la;
  TileLoader<BN, BK, Cfg::kThreads, Cfg::NB, Cfg::kPairB, Cfg::SB> lb;
  la.init(P.A + (long long)kbeg * a_ks, rowA, a_ks, m0, P.M);
  lb.init(P.B + (long long)kbeg * b_ks, colB, b_ks, n0, P.N);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int wm0 = (warp / WARPS_N) * Cfg::WM;
  const int wn0 = (warp % WARPS_N) * Cfg::WN;

  double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int klen = kend - kbeg;
  const int nk = (klen > 0) ? (klen + BK - 1) / BK : 0;
  const uint32_t as0 = smem_u32(As), bs0 = smem_u32(Bs);
  auto load_stage = [&](int kt, int buf) {
    const uint32_t sa = as0 + (uint32_t)(buf * BK * Cfg::SA * 8), sb = bs0 + (uint32_t)(buf * BK * Cfg::SB * 8);
    const int kleft = klen - kt * BK;
    if constexpr (CAP > kSmallGroup) {
      la.load_classic(sa, (long long)kt * BK * a_ks, kleft);
      lb.load_classic(sb, (long long)kt * BK * b_ks, kleft);
    } else if (kleft >= BK) {
      la.template load<true>(sa, (long long)kt * BK * a_ks, kleft);
      lb.template load<true>(sb, (long long)kt * BK * b_ks, kleft);
    } else {
      la.template load<false>(sa, (long long)kt * BK * a_ks, kleft);
      lb.template load<false>(sb, (long long)kt * BK * b_ks, kleft);
    }
  };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nk) load_stage(s, s);
    cp_async_commit();
  }

  const int fr = lane >> 2, fk = lane & 3;
  for (int kt = 0; kt < nk; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = kt + STAGES - 1;
      if (nxt < nk) load_stage(nxt, nxt % STAGES);
      cp_async_commit();
    }
    const double* as = As + (kt % STAGES) * BK * Cfg::SA;
    const double* bs = Bs + (kt % STAGES) * BK * Cfg::SB;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[Cfg::FM], bf[Cfg::FN];
      if constexpr (Cfg::kPairA) {
#pragma unroll
        for (int i = 0; i < Cfg::FM; i += 2) {
          const double2 v = *reinterpret_cast<const double2*>(as + (kk + fk) * Cfg::SA + wm0 + i * 8 + 2 * fr);
          af[i] = v.x; af[i + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int i = 0; i < Cfg::FM; ++i) af[i] = as[(kk + fk) * Cfg::SA + wm0 + i * 8 + fr];
      }
      if constexpr (Cfg::kPairB) {
#pragma unroll
        for (int j = 0; j < Cfg::FN; j += 2) {
          const double2 v = *reinterpret_cast<const double2*>(bs + (kk + fk) * Cfg::SB + wn0 + j * 8 + 2 * fr);
          bf[j] = v.x; bf[j + 1] = v.y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) bf[j] = bs[(kk + fk) * Cfg::SB + wn0 + j * 8 + fr];
      }
#pragma unroll
      for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
        for (int j = 0; j < Cfg::FN; ++j) dmma_8x8x4(acc[i][j], af[i], bf[j]);
    }
  }
  cp_async_wait<0>();

  // epilogue
  if (P.splits > 1) {
    double* part = P.partial + (size_t)split * P.M * P.N;
#pragma unroll
    for (int i = 0; i < Cfg::FM; ++i) {
      int ml = wm0 + i * 8 + fr;
      int m = m0 + ml;
      if (m >= P.M) continue;
#pragma unroll
      for (int j = 0; j < Cfg::FN; ++j) {
        int nl = wn0 + j * 8 + 2 * fk;
        int n = n0 + nl;
        if (n < P.N) part[(size_t)m * P.N + n] = acc[i][j][0];
        if (n + 1 < P.N) part[(size_t)m * P.N + n + 1] = acc[i][j][1];
      }
    }
    return;
  }
  const double alpha = P.alpha, beta = P.beta;
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i) {
    int ml = wm0 + i * 8 + fr;
    if (m0 + ml >= P.M) continue;
    long long ro = rowC[ml];
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) {
      int nl = wn0 + j * 8 + 2 * fk;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (n0 + nl + h < P.N) {
          double* dst = P.C + ro + colC[nl + h];
          double v = alpha * acc[i][j][h];
          if (beta != 0.0) v += beta * *dst;
          *dst = v;
        }
      }
    }
  }
}


// Host-side helpers ----------------------------------------------------------

// Fill tile bookkeeping of a problem; returns CTA count. split-K factor decided here.
struct GemmPlan {
  int bm, bn;
  size_t partial_elems;  // total split-K workspace (doubles)
};

// Launch a group of problems (count <= kMaxGroup, same tile config chosen
// internally). `ws` provides the split-K partial buffers (may be null when no
// split is needed; query with gemm_group_ws_bytes).
int gemm_group_launch(GemmProblem* probs, int count, void* ws, size_t ws_bytes, cudaStream_t st,
                      bool allow_split = true);

// TMA-staged DMMA GEMM for plain row-major operands (gemm_tma.cu):
// C = alpha A B + beta C, A (M x K, lda), B (K x N, ldb), C (M x N, ldc).
// gemm_tma_ok: 16-byte aligned bases, even leading dimensions, K >= 16.
bool gemm_tma_ok(int M, int N, int K, const double* A, long long lda, const double* B, long long ldb);
// strided form (A(m,k) = A[m*a_ms + k*a_ks], ...): row-major operands or
// transposes of row-major ones, column-major C as the transposed problem, K
// split over ws when the tiles leave SMs idle (only with force_split_ok: the
// grouped kernel's split-K is as fast); false = not taken, nothing launched
bool gemm_tma_try(int M, int N, int K, double alpha, const double* A, long long a_ms, long long a_ks,
                  const double* B, long long b_ks, long long b_ns, double beta, double* C, long long c_ms,
                  long long c_ns, void* ws, size_t ws_bytes, cudaStream_t st, int* status,
                  bool force_split_ok = false);
int gemm_tma(int M, int N, int K, double alpha, const double* A, long long lda, const double* B, long long ldb,
             double beta, double* C, long long ldc, cudaStream_t st);
size_t gemm_group_ws_bytes(const GemmProblem* probs, int count, bool allow_split = true);

// Convenience: plain strided problem, C(m,n) = alpha*sum_k A(m,k)B(k,n) + beta*C
inline GemmProblem make_gemm(int M, int N, int K, const double* A, long long a_ms, long long a_ks,
                             const double* B, long long b_ks, long long b_ns, double* C,
                             long long c_ms, long long c_ns, double alpha = 1.0, double beta = 0.0) {
  GemmProblem p{};
  p.A = A; p.B = B; p.C = C; p.partial = nullptr;
  p.M = M; p.N = N; p.K = K;
  p.a_ms0 = a_ms; p.a_ms1 = 0; p.a_mdiv = 1 << 30; p.a_ks = a_ks;
  p.b_ns0 = b_ns; p.b_ns1 = 0; p.b_ndiv = 1 << 30; p.b_ks = b_ks;
  p.c_ms0 = c_ms; p.c_ms1 = 0; p.c_mdiv = 1 << 30;
  p.c_ns0 = c_ns; p.c_ns1 = 0; p.c_ndiv = 1 << 30;
  p.alpha = alpha; p.beta = beta;
  p.splits = 1;
  return p;
}

}  // namespace ttk
