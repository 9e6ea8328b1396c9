// Khatri-Rao structured sketch of TT vectors (reference kr_apply, sketch.py:50-70).
//
//   y_j = sum_{i_1..i_d} prod_k F_k[j, i_k] * v[i_1, ..., i_d]
//
// Per row j a running state s_j (1 x r_k) advances mode by mode:
//   s_j <- sum_{a, i} s_j[a] F_k[j, i] C_k[a, i, :]
// which is a GEMM with M = rows, K = r_{k-1} n_k, N = r_k whose A operand
// A[j, (a,i)] = s_j[a] * F_k[j, i] is a Khatri-Rao product formed on the fly.
//
// Two device paths:
//  * fused (many rows, ranks <= 128): one CTA owns 128 rows of one vector and
//    runs all d modes with the state resident in shared memory; F and C_k tiles
//    are staged by a 3-stage cp.async pipeline and contracted on the DMMA pipe.
//  * two-phase (few rows, e.g. the solver's s = 2*maxit sketch of one vector):
//    phase 1 computes every M_k = F_k x_2 C_k (s x r_{k-1} x r_k) for all modes
//    at once with the grouped GEMM (all FLOPs, fully parallel); phase 2 walks
//    the per-row state through the d small matrices (rows are independent).
// Output rows stay in their fixed positions (SPEC: deterministic row order).
#include <cooperative_groups.h>

#include "gemm.cuh"
#include "../../include/ttk_b200.h"

#include <algorithm>
#include <vector>

namespace ttk {

constexpr int kKrMaxModes = 64;
constexpr int kKrMaxSlots = 1536;  // (vector, mode) core pointers per launch

struct KrParams {
  int d;
  int S;         // rows handled (s_hi - s_lo)
  int nvec;
  int rmax;
  const double* F[kKrMaxModes];  // row s_lo of factor k, row stride ldF[k] = n_k
  int n[kKrMaxModes];
  double* out;                   // nvec x S
  const double* core[kKrMaxSlots];   // vec * d + k
  short rank[kKrMaxSlots + 64];      // vec * (d+1) + k
};

namespace kr {
// 64 rows of one vector per CTA; 8 warps = 4 row groups (16 rows) x 2 column
// halves (64 state columns each).  The K loop of mode k runs over (a, i-chunk)
// so the state value s_j[a] is uniform per stage (no index divisions), the
// F_k tile (64 x n) stays resident in shared memory for the whole mode, and
// only the core rows C_k[a, i0:i0+16, :] are streamed.
constexpr int WARPS = 8;
constexpr int BM = 64;                // rows per CTA
constexpr int BN = 128;               // max rank handled by the fused path
constexpr int FNH = 10;               // max fragments per warp along n (fn - 2*(fn/4) <= 10 for fn <= 16)
constexpr int BK = 32;
constexpr int STAGES = 3;
constexpr int NMAX = 96;              // mode size handled by the fused path (smem: state + F tile + 3 stages)
constexpr int SST = BN + 1;           // odd stride: conflict-free state reads
constexpr int SFT = BM + 4;           // F tile, i-major: Ft[i][row], 4 mod 16
constexpr int SB = BN + 4;
constexpr int CPT = BK * BN / (WARPS * 32);  // C elements per thread per stage
// F tile sized by the largest mode of the launch (smem_bytes(nmax))
constexpr size_t smem_bytes(int nmax) {
  return sizeof(double) * ((size_t)BM * SST + (size_t)((nmax + BK - 1) / BK * BK) * SFT + (size_t)STAGES * BK * SB);
}
}  // namespace kr

// One mode of the fused sketch for a warp owning FNW state-column fragments
// (compile-time: no branches around the warp-synchronous DMMAs).
template <int FNW>
__device__ __forceinline__ void kr_mode(double* St, const double* Ft, double* Bs, const double* Ck, int r1,
                                        int n, int nic, int s_lo, int s_hi, int wrow, int wcol,
                                        const int (&ckk)[kr::CPT], const int (&ccol)[kr::CPT], double* Dst) {
  using namespace kr;
  const int tid = threadIdx.x, lane = tid & 31;
  const int fr = lane >> 2, fk = lane & 3;
  auto load_c = [&](int s, int buf) {
    const int a = s / nic, ic = s - a * nic;
    const long long kb = (long long)a * n + ic * BK;
#pragma unroll
    for (int q = 0; q < CPT; ++q) {
      const bool ok = (ic * BK + ckk[q] < n) && (ccol[q] < r1);
      const double* src = ok ? Ck + (kb + ckk[q]) * r1 + ccol[q] : Ck;
      cp_async8(Bs + (size_t)buf * BK * SB + ckk[q] * SB + pair_pos<true>(ccol[q]), src, ok);
    }
  };
  const int nst = s_hi - s_lo;  // this CTA's stages (a cluster splits the K range)
  auto load_c_rel = [&](int s, int buf) { load_c(s_lo + s, buf); };
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < nst) load_c_rel(s, s);
    cp_async_commit();
  }
  double acc[2][FNW > 0 ? FNW : 1][2];
#pragma unroll
  for (int i = 0; i < 2; ++i)
#pragma unroll
    for (int j = 0; j < FNW; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double sa0 = 0.0, sa1 = 0.0;
  int a_cur = -1;
  for (int s = 0; s < nst; ++s) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nxt = s + STAGES - 1;
      if (nxt < nst) load_c_rel(nxt, nxt % STAGES);
      cp_async_commit();
    }
    const int sg = s_lo + s;
    const int a = sg / nic, ic = sg - a * nic;
    if (a != a_cur) {  // state values of this lane's two rows for the new a
      a_cur = a;
      sa0 = St[(wrow + fr) * SST + a];
      sa1 = St[(wrow + 8 + fr) * SST + a];
    }
    if constexpr (FNW > 0) {
      const double* bs = Bs + (size_t)(s % STAGES) * BK * SB + wcol + 2 * fr;
      const double* ft = Ft + (size_t)(ic * BK) * SFT + wrow + 2 * fr;
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) {
        const double2 fv = *reinterpret_cast<const double2*>(ft + (kk + fk) * SFT);
        const double af0 = fv.x * sa0, af1 = fv.y * sa1;
#pragma unroll
        for (int j = 0; j < FNW; j += 2) {
          const double2 bv = *reinterpret_cast<const double2*>(bs + (kk + fk) * SB + j * 8);
          dmma_8x8x4(acc[0][j], af0, bv.x);
          dmma_8x8x4(acc[1][j], af1, bv.x);
          if constexpr (true) {
            if (j + 1 < FNW) {
              dmma_8x8x4(acc[0][j + 1], af0, bv.y);
              dmma_8x8x4(acc[1][j + 1], af1, bv.y);
            }
          }
        }
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // every warp is done reading the old state (and the stage buffers)
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    const int row = wrow + i * 8 + fr;
#pragma unroll
    for (int j = 0; j < FNW; ++j) {
      const int col = wcol + j * 8 + 2 * fk;
      if (col < r1) Dst[row * SST + col] = acc[i][j][0];
      if (col + 1 < r1) Dst[row * SST + col + 1] = acc[i][j][1];
    }
  }
}

__global__ void __launch_bounds__(kr::WARPS * 32, 1)
    kr_fused_kernel(const __grid_constant__ KrParams P) {
  using namespace kr;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int nmax = 0;
  for (int k = 0; k < P.d; ++k) nmax = max(nmax, P.n[k]);
  const int nft = (nmax + BK - 1) / BK * BK;
  double* St = reinterpret_cast<double*>(smem_raw);   // BM x SST
  double* Ft = St + BM * SST;                          // nft x SFT
  double* Bs = Ft + (size_t)nft * SFT;                 // STAGES x BK x SB

  // a cluster of CL CTAs shares one (vector, 64-row) item: each contracts a
  // contiguous slice of the mode's K stages into a partial state, the partials
  // are summed over DSMEM in a fixed order (every CTA then holds the full state)
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int CL = (int)cl.num_blocks(), crank = (int)cl.block_rank();
  double* Pbuf = Bs;  // partial state (BM x SST) in the stage buffers once the K loop is done
  const int vec = blockIdx.y;
  const int j0 = (blockIdx.x / CL) * BM;
  const int tid = threadIdx.x, warp = tid >> 5;
  const int wrow = (warp >> 1) * 16;     // 16 rows = fragment pair (rows r, r + 8)

  for (int e = tid; e < BM; e += WARPS * 32) St[e * SST] = 1.0;

  // per-thread C-chunk slots: (kk, col) fixed for the whole kernel
  int ckk[CPT], ccol[CPT];
#pragma unroll
  for (int q = 0; q < CPT; ++q) {
    const int e = tid + q * WARPS * 32;
    ckk[q] = e / BN;
    ccol[q] = e % BN;
  }

  for (int k = 0; k < P.d; ++k) {
    const int r0 = P.rank[vec * (P.d + 1) + k];
    const int r1 = P.rank[vec * (P.d + 1) + k + 1];
    const int n = P.n[k];
    const int nic = (n + BK - 1) / BK;   // i-chunks per a
    const int nst = r0 * nic;            // stages of this mode
    const double* Fk = P.F[k];
    const double* Ck = P.core[vec * P.d + k];
    // column halves split at an even fragment count (pairs stay 16-aligned) as
    // evenly as possible: r1 = 100 -> 6 + 7 fragments
    const int fn = (r1 + 7) / 8;
    const int f0 = 2 * (fn / 4);
    const int wcol = (warp & 1) ? f0 * 8 : 0;
    const int fnh = (warp & 1) ? fn - f0 : f0;

    __syncthreads();  // previous mode's state written; F tile / stage buffers free
    // F tile of this row block, i-major, rows paired (r, r + 8) side by side
    for (int e = tid; e < BM * n; e += WARPS * 32) {
      const int row = e / n, i = e - row * n;
      const bool ok = j0 + row < P.S;
      cp_async8(Ft + i * SFT + pair_pos<true>(row), ok ? Fk + (long long)(j0 + row) * n + i : Fk, ok);
    }
    for (int e = tid; e < (nic * BK - n) * BM; e += WARPS * 32) {
      // zero rows i >= n of the F tile used by the last, partial i-chunk
      const int i = n + e / BM, row = e % BM;
      Ft[i * SFT + row] = 0.0;
    }
    const int s_lo = (int)((long long)nst * crank / CL), s_hi = (int)((long long)nst * (crank + 1) / CL);
    double* Dst = CL > 1 ? Pbuf : St;
#define KR_MODE(F) kr_mode<F>(St, Ft, Bs, Ck, r1, n, nic, s_lo, s_hi, wrow, wcol, ckk, ccol, Dst)
    switch (fnh) {  // warp-uniform
      case 0: KR_MODE(0); break;
      case 1: KR_MODE(1); break;
      case 2: KR_MODE(2); break;
      case 3: KR_MODE(3); break;
      case 4: KR_MODE(4); break;
      case 5: KR_MODE(5); break;
      case 6: KR_MODE(6); break;
      case 7: KR_MODE(7); break;
      case 8: KR_MODE(8); break;
      case 9: KR_MODE(9); break;
      default: KR_MODE(10); break;
    }
#undef KR_MODE
    if (CL > 1) {
      cl.sync();  // every CTA's partial written
      for (int e = tid; e < BM * r1; e += WARPS * 32) {
        const int row = e / r1, col = e - row * r1;
        double v = 0.0;
        for (int q = 0; q < CL; ++q) v += *cl.map_shared_rank(Pbuf + row * SST + col, q);
        St[row * SST + col] = v;
      }
      cl.sync();  // partials read everywhere before the next mode reuses the stage buffers
    }
  }
  __syncthreads();
  if (crank == 0)
    for (int row = tid; row < BM; row += WARPS * 32)
      if (j0 + row < P.S) P.out[(long long)vec * P.S + j0 + row] = St[row * SST];
}

// phase 2 of the two-phase path: per (vector, row) walk the state through
// M_k[j] (r0 x r1), M stored as [vec][k] blocks of S x r0 x r1.
struct KrChainParams {
  int d, S, nvec, rmax;
  const double* M;            // base of the M buffer
  long long moff[kKrMaxSlots];  // offset of block (vec, k)
  short rank[kKrMaxSlots + 64];
  double* out;
};

__global__ void kr_chain_kernel(const __grid_constant__ KrChainParams P) {
  extern __shared__ double sm[];
  const int rows_per_cta = blockDim.x >> 5;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int vec = blockIdx.y;
  const int j = blockIdx.x * rows_per_cta + warp;
  double* st = sm + warp * 2 * P.rmax;
  double* nx = st + P.rmax;
  if (lane == 0) st[0] = 1.0;
  __syncwarp();
  for (int k = 0; k < P.d; ++k) {
    const int r0 = P.rank[vec * (P.d + 1) + k];
    const int r1 = P.rank[vec * (P.d + 1) + k + 1];
    if (j < P.S) {
      const double* Mk = P.M + P.moff[vec * P.d + k] + (long long)j * r0 * r1;
      for (int b = lane; b < r1; b += 32) {
        double s = 0.0;
        for (int a = 0; a < r0; ++a) s += st[a] * Mk[(long long)a * r1 + b];
        nx[b] = s;
      }
    }
    __syncwarp();
    double* t = st; st = nx; nx = t;
  }
  if (j < P.S && lane == 0) P.out[(long long)vec * P.S + j] = st[0];
}

}  // namespace ttk

using namespace ttk;

namespace {

int kr_fused(int d, const int* n, int S, const double* const* F, int nvec, const int* ranks,
             const double* const* cores, double* out, cudaStream_t st) {
  {  // per-device attributes (set_attr_once)
    TTK_TRY(set_attr_once(kr_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)kr::smem_bytes(kr::NMAX)));
  }
  const int per = std::max(1, std::min(kKrMaxSlots / d, 64));
  for (int v0 = 0; v0 < nvec; v0 += per) {
    int nv = std::min(per, nvec - v0);
    static thread_local KrParams P;
    P.d = d; P.S = S; P.nvec = nv; P.rmax = 0;
    for (int k = 0; k < d; ++k) { P.F[k] = F[k]; P.n[k] = n[k]; }
    P.out = out + (long long)v0 * S;
    for (int v = 0; v < nv; ++v) {
      for (int k = 0; k < d; ++k) P.core[v * d + k] = cores[(long long)(v0 + v) * d + k];
      for (int k = 0; k <= d; ++k) P.rank[v * (d + 1) + k] = (short)ranks[(long long)(v0 + v) * (d + 1) + k];
    }
    // cluster split of the K stages: at least 2 CTAs per (vector, row-block)
    // item (config 4, 512 items: 3.46 -> 6.9 waves, 19.1 -> 20.7 TF/s), more
    // when the items alone would leave SMs idle (a row shard of the
    // 1/2/4/8-GPU partition: 64 rows x 64 vectors 10.2 -> 5.5 ms, 0.90 of the
    // full-row per-row rate; CL 4 / 8 measured 5.7 / 8.1 ms, tools/kr_rows.py):
    // the smallest CL in {2, 4, 8} with items * CL >= 0.8 SMs
    const int items = ceil_div(S, kr::BM) * nv;
    int CL = 2;
    while (CL < 8 && (long)items * CL * 5 < 4L * num_sms()) CL *= 2;
    static const int cl_knob = knob_env("TTK_KR_CL") ? atoi(knob_env("TTK_KR_CL")) : 0;  // A/B
    if (cl_knob > 0) CL = cl_knob;
    int nmax = 0;
    for (int k = 0; k < d; ++k) nmax = std::max(nmax, n[k]);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(ceil_div(S, kr::BM) * CL, nv, 1);
    cfg.blockDim = dim3(kr::WARPS * 32, 1, 1);
    cfg.dynamicSmemBytes = kr::smem_bytes(nmax);
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    TTK_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kr_fused_kernel, P));
    TTK_CHECK_LAUNCH();
  }
  return kOk;
}

size_t kr_two_phase_elems(int d, int S, int nvec, const int* ranks) {
  size_t tot = 0;
  for (int v = 0; v < nvec; ++v)
    for (int k = 0; k < d; ++k)
      tot += (size_t)S * ranks[v * (d + 1) + k] * ranks[v * (d + 1) + k + 1];
  return tot;
}

int kr_two_phase(int d, const int* n, int S, const double* const* F, int nvec, const int* ranks,
                 const double* const* cores, double* out, void* ws, size_t ws_bytes,
                 cudaStream_t st) {
  size_t melems = kr_two_phase_elems(d, S, nvec, ranks);
  Arena ar(ws, ws_bytes);
  double* M = ar.take<double>(melems);
  std::vector<GemmProblem> probs;
  probs.reserve((size_t)nvec * d);
  std::vector<long long> moff((size_t)nvec * d);
  long long off = 0;
  int rmax = 1;
  for (int v = 0; v < nvec; ++v) {
    for (int k = 0; k < d; ++k) {
      const int r0 = ranks[v * (d + 1) + k], r1 = ranks[v * (d + 1) + k + 1];
      rmax = std::max(rmax, std::max(r0, r1));
      moff[(size_t)v * d + k] = off;
      GemmProblem p{};
      p.M = S; p.N = r0 * r1; p.K = n[k];
      p.A = F[k]; p.a_ms0 = n[k]; p.a_ms1 = 0; p.a_mdiv = 1 << 30; p.a_ks = 1;
      p.B = cores[(size_t)v * d + k];
      p.b_ndiv = r1; p.b_ns1 = (long long)n[k] * r1; p.b_ns0 = 1; p.b_ks = r1;
      p.C = M ? M + off : nullptr;
      p.c_mdiv = 1 << 30; p.c_ms0 = (long long)r0 * r1; p.c_ms1 = 0;
      p.c_ndiv = 1 << 30; p.c_ns0 = 1; p.c_ns1 = 0;
      p.alpha = 1.0; p.beta = 0.0; p.splits = 1;
      probs.push_back(p);
      off += (long long)S * r0 * r1;
    }
  }
  TTK_REQUIRE(M != nullptr, kWorkspace, "kr_sketch: workspace too small (%zu bytes needed)",
              ar.used);
  TTK_TRY(gemm_group_launch(probs.data(), (int)probs.size(), nullptr, 0, st, false));
  const int per = std::max(1, std::min(kKrMaxSlots / d, 1024));
  for (int v0 = 0; v0 < nvec; v0 += per) {
    int nv = std::min(per, nvec - v0);
    static thread_local KrChainParams C;
    C.d = d; C.S = S; C.nvec = nv; C.rmax = rmax; C.M = M;
    C.out = out + (long long)v0 * S;
    for (int v = 0; v < nv; ++v) {
      for (int k = 0; k < d; ++k) C.moff[v * d + k] = moff[(size_t)(v0 + v) * d + k];
      for (int k = 0; k <= d; ++k) C.rank[v * (d + 1) + k] = (short)ranks[(v0 + v) * (d + 1) + k];
    }
    const int rows_per_cta = 4;
    dim3 grid(ceil_div(S, rows_per_cta), nv);
    size_t smem = sizeof(double) * 2 * rmax * rows_per_cta;
    if (smem > 48 * 1024)
      TTK_TRY(set_attr_once(kr_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
    kr_chain_kernel<<<grid, 32 * rows_per_cta, smem, st>>>(C);
    TTK_CHECK_LAUNCH();
  }
  return kOk;
}

bool use_fused(int d, const int* n, int S, int nvec, const int* ranks) {
  for (int k = 0; k < d; ++k)
    if (n[k] > kr::NMAX) return false;
  for (int v = 0; v < nvec; ++v)
    for (int k = 0; k <= d; ++k)
      if (ranks[v * (d + 1) + k] > kr::BN) return false;
  // the fused path needs enough CTAs to fill the machine: (vector, row-block)
  // items, each split over a cluster of up to 8 CTAs
  long ctas = (long)nvec * ceil_div(S, kr::BM) * 8;
  return ctas >= num_sms();
}

}  // namespace

extern "C" {

// Sketch rows [s_lo, s_hi) of nvec TT vectors.  F: d device pointers to the
// FULL factors (s_total x n_k row-major); out: nvec x (s_hi - s_lo) row-major.
// ranks: nvec x (d+1); cores: nvec x d device pointers.
size_t ttk_kr_sketch_ws_bytes(int d, const int* n, int s_lo, int s_hi, int nvec, const int* ranks) {
  const int S = s_hi - s_lo;
  if (S <= 0 || nvec <= 0) return 0;
  if (use_fused(d, n, S, nvec, ranks)) return 0;
  return kr_two_phase_elems(d, S, nvec, ranks) * sizeof(double) + 4096;
}

int ttk_kr_sketch(int d, const int* n, int s_lo, int s_hi, const double* const* F, int nvec,
                  const int* ranks, const double* const* cores, double* out, void* ws,
                  size_t ws_bytes, void* stream) {
  TTK_REQUIRE(d >= 1 && d <= kKrMaxModes, kInvalidValue, "kr_sketch: d=%d out of range", d);
  TTK_REQUIRE(s_hi >= s_lo && s_lo >= 0, kInvalidValue, "kr_sketch: bad row range");
  const int S = s_hi - s_lo;
  if (S == 0 || nvec == 0) return kOk;
  for (int v = 0; v < nvec; ++v)
    TTK_REQUIRE(ranks[v * (d + 1)] == 1 && ranks[v * (d + 1) + d] == 1, kShapeMismatch,
                "kr_sketch: boundary ranks must equal 1");
  std::vector<const double*> Fo(d);
  for (int k = 0; k < d; ++k) Fo[k] = F[k] + (long long)s_lo * n[k];
  cudaStream_t st = (cudaStream_t)stream;
  if (use_fused(d, n, S, nvec, ranks)) return kr_fused(d, n, S, Fo.data(), nvec, ranks, cores, out, st);
  return kr_two_phase(d, n, S, Fo.data(), nvec, ranks, cores, out, ws, ws_bytes, st);
}

// Fused matvec -> sketch: out[j] = (row j of the Khatri-Rao
// product) . vec(A x) without materialising A x.  With the operator-premultiplied
// factors Ft_k[j, al, i', be] = sum_i F_k[j, i] D_k[al, i, i', be] (S x rho_k x
// n_k x rho_{k+1}, computed once per (sketch, operator) pair by the caller), phase
// 1 forms M_k[j, (a*rho+al), (b*rho'+be)] = sum_i' Ft_k[j, al, i', be] C_k[a, i', b]
// -- one grouped-GEMM problem per (core, al, be) writing straight into the merged
// rank order of tt_matvec's output -- and phase 2 is the same per-row chain as the
// two-phase sketch over ranks r_k * rho_k.  Same flops as sketching A x, minus
// the write and re-read of A x.
size_t ttk_kr_sketch_matvec_ws_bytes(int d, int S, const int* rho, const int* r) {
  if (S <= 0 || d <= 0) return 0;
  size_t tot = 0;
  for (int k = 0; k < d; ++k) tot += (size_t)S * r[k] * rho[k] * r[k + 1] * rho[k + 1];
  return tot * sizeof(double) + 4096;
}

int ttk_kr_sketch_matvec(int d, const int* n, int S, const double* const* Ft, const int* rho, const int* r,
                         const double* const* C, double* out, void* ws, size_t ws_bytes, void* stream) {
  TTK_REQUIRE(d >= 1 && d <= kKrMaxModes, kInvalidValue, "kr_sketch_matvec: d=%d out of range", d);
  TTK_REQUIRE(S >= 0, kInvalidValue, "kr_sketch_matvec: negative row count");
  TTK_REQUIRE(r[0] == 1 && r[d] == 1 && rho[0] == 1 && rho[d] == 1, kShapeMismatch,
              "kr_sketch_matvec: boundary ranks must equal 1");
  if (S == 0) return kOk;
  cudaStream_t st = (cudaStream_t)stream;
  std::vector<int> R(d + 1);
  for (int k = 0; k <= d; ++k) R[k] = r[k] * rho[k];
  size_t melems = 0;
  for (int k = 0; k < d; ++k) melems += (size_t)S * R[k] * R[k + 1];
  Arena ar(ws, ws_bytes);
  double* M = ar.take<double>(melems);
  TTK_REQUIRE(M != nullptr, kWorkspace, "kr_sketch_matvec: workspace too small (%zu bytes needed)", ar.used);
  std::vector<GemmProblem> probs;
  std::vector<long long> moff(d);
  long long off = 0;
  int rmax = 1;
  for (int k = 0; k < d; ++k) {
    const int r0 = r[k], r1 = r[k + 1], p0 = rho[k], p1 = rho[k + 1], nk = n[k];
    moff[k] = off;
    rmax = std::max(rmax, std::max(R[k], R[k + 1]));
    if (r0 > 0 && r1 > 0)
      for (int al = 0; al < p0; ++al)
        for (int be = 0; be < p1; ++be) {
          GemmProblem p{};
          p.M = S; p.N = r0 * r1; p.K = nk;
          p.A = Ft[k] + (long long)al * nk * p1 + be;  // A(j, i') = Ft[j, al, i', be]
          p.a_ms0 = (long long)p0 * nk * p1; p.a_ms1 = 0; p.a_mdiv = 1 << 30; p.a_ks = p1;
          p.B = C[k];  // B(i', (a, b)) = C[a, i', b]
          p.b_ndiv = r1; p.b_ns1 = (long long)nk * r1; p.b_ns0 = 1; p.b_ks = r1;
          p.C = M + off + (long long)al * R[k + 1] + be;  // M_k[j, a*p0+al, b*p1+be]
          p.c_mdiv = 1 << 30; p.c_ms0 = (long long)R[k] * R[k + 1]; p.c_ms1 = 0;
          p.c_ndiv = r1; p.c_ns0 = p1; p.c_ns1 = (long long)p0 * R[k + 1];
          p.alpha = 1.0; p.beta = 0.0; p.splits = 1;
          probs.push_back(p);
        }
    off += (long long)S * R[k] * R[k + 1];
  }
  TTK_REQUIRE(d <= kKrMaxSlots, kInvalidValue, "kr_sketch_matvec: d too large");
  TTK_TRY(gemm_group_launch(probs.data(), (int)probs.size(), nullptr, 0, st, false));
  static thread_local KrChainParams CP;
  CP.d = d; CP.S = S; CP.nvec = 1; CP.rmax = rmax; CP.M = M; CP.out = out;
  for (int k = 0; k < d; ++k) CP.moff[k] = moff[k];
  for (int k = 0; k <= d; ++k) CP.rank[k] = (short)R[k];
  const int rows_per_cta = 4;
  dim3 grid(ceil_div(S, rows_per_cta), 1);
  const size_t smem = sizeof(double) * 2 * rmax * rows_per_cta;
  if (smem > 48 * 1024)
    TTK_TRY(set_attr_once(kr_chain_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  kr_chain_kernel<<<grid, 32 * rows_per_cta, smem, st>>>(CP);
  TTK_CHECK_LAUNCH();
  return kOk;
}

// Force a path (testing): path 0 = fused, 1 = two-phase.
int ttk_kr_sketch_path(int path, int d, const int* n, int s_lo, int s_hi, const double* const* F,
                       int nvec, const int* ranks, const double* const* cores, double* out,
                       void* ws, size_t ws_bytes, void* stream) {
  const int S = s_hi - s_lo;
  if (S <= 0 || nvec == 0) return kOk;
  std::vector<const double*> Fo(d);
  for (int k = 0; k < d; ++k) Fo[k] = F[k] + (long long)s_lo * n[k];
  cudaStream_t st = (cudaStream_t)stream;
  if (path == 0) {
    for (int k = 0; k < d; ++k)
      TTK_REQUIRE(n[k] <= kr::NMAX, kInvalidValue, "fused path needs mode sizes <= %d", kr::NMAX);
    for (int v = 0; v < nvec; ++v)
      for (int k = 0; k <= d; ++k)
        TTK_REQUIRE(ranks[v * (d + 1) + k] <= kr::BN, kInvalidValue, "fused path needs ranks <= %d",
                    kr::BN);
    return kr_fused(d, n, S, Fo.data(), nvec, ranks, cores, out, st);
  }
  return kr_two_phase(d, n, S, Fo.data(), nvec, ranks, cores, out, ws, ws_bytes, st);
}

}  // extern "C"
