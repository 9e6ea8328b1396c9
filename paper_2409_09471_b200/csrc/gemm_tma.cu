// TMA-staged fp64 DMMA GEMM: C = alpha op(A) op(B) + beta C for the skinny
// contractions of the randomize-then-orthogonalize sweeps and the truncation
// (round.cu): the right sweep's T_c = X_c W_{c+1} and W_c = T_c G_c^T, the
// left sweep's sketches Y = M_{c-1} T_{c-1}, projections Z = M_{c-1} X_{c-1}
// and M_c = Q_c^T Z, the truncation's Gram C C^T and its core products.
//
// Operands are row-major matrices or transposes of row-major matrices (TA:
// A given as A^T, row-major K x M; TB: B given as B^T, row-major N x K).
// Staging: one producer warp issues cp.async.bulk.tensor (TMA) loads of a
// BM x 16 slice of op(A) and a 16 x BN slice of op(B) per stage (boxes of 16
// doubles = one 128-byte row) into a ring of STAGES buffers, completion counted
// in bytes on the stage's "full" mbarrier; the four consumer warps release a
// stage on its "empty" mbarrier as soon as its last fragments are in
// registers.  Every box uses the 128-byte swizzle (16-byte chunk index XOR row
// mod 8).  The DMMA m8n8k4 fragments read 8 rows x 4 k of A and 4 k x 8 columns
// of B, one double per lane: from a tile stored [m][k] (row-major A, or B^T)
// the 8 rows differ in (row mod 8) and from a tile stored [k][n] (row-major B,
// or A^T) the 4 k rows do -- either way each 128-byte bank row is hit by
// exactly two lanes, the two-wavefront minimum of a 64-bit warp access.  No
// per-thread load plan or cp.async address arithmetic in the consumer warps;
// fragments are double-buffered in registers (the loads of k-step kk + 1, or
// of the next stage's first k-step behind its wait, are issued before the
// DMMAs of k-step kk).  Out-of-range rows / columns / k are zero-filled by TMA.
//
// Tiles: 64 x 80 (tall, N = 80: one column tile covers N) and 80 x 64 (wide,
// M = 80), halved along the long side (32 x 80 / 80 x 32) when the full tiles
// leave fewer than two CTAs per SM; 2 x 2 consumer warps.  Long-K problems
// with few tiles split K over grid.z (~one wave, >= 8 k tiles per split); the partial
// tiles are reduced in a fixed order (deterministic).
#include "common.cuh"
#include "gemm.cuh"
#include "../../include/ttk_b200.h"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <algorithm>
#include <mutex>

namespace ttk {

namespace {

constexpr int kTmBK = 16;  // k per stage

template <int BM, int BN, int STAGES>
struct TmCfg {
  static constexpr int kConsumers = 4;
  static constexpr int kThreads = 32 * (kConsumers + 1);
  static constexpr int WM = BM / 2, WN = BN / 2;
  static constexpr int FM = WM / 8, FN = WN / 8;
  static constexpr int A_BYTES = BM * kTmBK * 8;
  static constexpr int B_BYTES = kTmBK * BN * 8;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024;  // + alignment slack
  static_assert(BM % 16 == 0 && BN % 16 == 0, "tile shape");
  static_assert(A_BYTES % 1024 == 0 && B_BYTES % 1024 == 0, "swizzle-128B buffers need 1024-byte alignment");
};

struct TmParams {
  int M, N, K;
  int kt_per_split;  // k tiles per grid.z slice
  double alpha, beta;
  double* C;  // output (splits == 1) or the partial buffer (splits x M x N, row-major)
  long long c_ms, c_ns;
  int splits;
};

__device__ __forceinline__ void tm_mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void tm_arrive_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void tm_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void tm_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done);
}
__device__ __forceinline__ void tm_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(map), "r"(x), "r"(y), "r"(bar)
      : "memory");
}

// byte offset of an element in the swizzled tiles: a "row-stored" tile holds
// 128-byte rows of 16 k values ([m][k] or [n][k]); a "k-stored" tile holds
// 16-column boxes of 16 k rows ([k][m] or [k][n])
__device__ __forceinline__ uint32_t sw_rows(int r, int k) {
  return (uint32_t)(r * 128 + ((((k >> 1) ^ r) & 7) << 4) + ((k & 1) << 3));
}
__device__ __forceinline__ uint32_t sw_kboxes(int k, int c) {
  return (uint32_t)((c >> 4) * 2048 + k * 128 + (((((c & 15) >> 1) ^ k) & 7) << 4) + ((c & 1) << 3));
}

template <int BM, int BN, int STAGES, bool TA, bool TB>
__global__ void __launch_bounds__(TmCfg<BM, BN, STAGES>::kThreads)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                    const __grid_constant__ TmParams P) {
  using Cfg = TmCfg<BM, BN, STAGES>;
  extern __shared__ unsigned char tm_smem_raw[];
  __shared__ __align__(8) unsigned long long full[STAGES], empty[STAGES];
  const uint32_t raw = smem_u32(tm_smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int KTall = (P.K + kTmBK - 1) / kTmBK;
  const int kt0 = blockIdx.z * P.kt_per_split;
  const int KT = max(0, min(KTall, kt0 + P.kt_per_split) - kt0);
  auto a_buf = [&](int s) { return base + (uint32_t)(s * Cfg::STAGE_BYTES); };
  auto b_buf = [&](int s) { return base + (uint32_t)(s * Cfg::STAGE_BYTES + Cfg::A_BYTES); };
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tm_mbar_init(smem_u32(&full[s]), 1);
      tm_mbar_init(smem_u32(&empty[s]), Cfg::kConsumers);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();

  if (warp == Cfg::kConsumers) {
    // ---- producer: one elected lane streams this slice's k tiles ----
    if (lane == 0) {
#ifndef TTK_TMA_NO_PREFETCH
      asm volatile("prefetch.tensormap [%0];" ::"l"(&ma) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mb) : "memory");
#endif
      for (int it = 0; it < KT; ++it) {
        const int s = it % STAGES;
        if (it >= STAGES) tm_wait(smem_u32(&empty[s]), (uint32_t)(((it / STAGES) - 1) & 1));
        const uint32_t fb = smem_u32(&full[s]);
        const int k0 = (kt0 + it) * kTmBK;
        tm_arrive_tx(fb, (uint32_t)Cfg::STAGE_BYTES);
        if (!TA) {
          tm_load_2d(a_buf(s), &ma, k0, m0, fb);  // [m][k] rows
        } else {
#pragma unroll
          for (int j = 0; j < BM / 16; ++j) tm_load_2d(a_buf(s) + j * 2048, &ma, m0 + 16 * j, k0, fb);  // [k][m]
        }
        if (!TB) {
#pragma unroll
          for (int j = 0; j < BN / 16; ++j) tm_load_2d(b_buf(s) + j * 2048, &mb, n0 + 16 * j, k0, fb);  // [k][n]
        } else {
          tm_load_2d(b_buf(s), &mb, k0, n0, fb);  // [n][k] rows
        }
      }
    }
    return;
  }

  // ---- consumers: 2 x 2 warps, warp tile WM x WN ----
  const int wm = warp >> 1, wn = warp & 1;
  const int lr = lane >> 2, lk = lane & 3;
  double acc[Cfg::FM][Cfg::FN][2];
#pragma unroll
  for (int i = 0; i < Cfg::FM; ++i)
#pragma unroll
    for (int j = 0; j < Cfg::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // lane-constant offsets (fragment row / column offsets are multiples of 8)
  uint32_t a_off[4][Cfg::FM], b_off[4][Cfg::FN];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const int k = kk * 4 + lk;
#pragma unroll
    for (int fm = 0; fm < Cfg::FM; ++fm) {
      const int m = wm * Cfg::WM + fm * 8 + lr;
      a_off[kk][fm] = TA ? sw_kboxes(k, m) : sw_rows(m, k);
    }
#pragma unroll
    for (int fn = 0; fn < Cfg::FN; ++fn) {
      const int n = wn * Cfg::WN + fn * 8 + lr;
      b_off[kk][fn] = (uint32_t)Cfg::A_BYTES + (TB ? sw_rows(n, k) : sw_kboxes(k, n));
    }
  }
  // generic pointer to the aligned ring: ordinary loads, which the "memory"
  // clobber of the mbarrier wait keeps below it (a volatile asm load without a
  // clobber could be hoisted above the wait and read a stage not yet landed)
  const unsigned char* ring = tm_smem_raw + (base - raw);
  double af[2][Cfg::FM], bf[2][Cfg::FN];
  auto load_frags = [&](int buf, int s, int kk) {
    const unsigned char* sb = ring + s * Cfg::STAGE_BYTES;
#pragma unroll
    for (int fm = 0; fm < Cfg::FM; ++fm) af[buf][fm] = *reinterpret_cast<const double*>(sb + a_off[kk][fm]);
#pragma unroll
    for (int fn = 0; fn < Cfg::FN; ++fn) bf[buf][fn] = *reinterpret_cast<const double*>(sb + b_off[kk][fn]);
  };
  if (KT > 0) {
    tm_wait(smem_u32(&full[0]), 0u);
    load_frags(0, 0, 0);
  }
  for (int it = 0; it < KT; ++it) {
    const int s = it % STAGES;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int cur = kk & 1, nxt = cur ^ 1;
      if (kk < 3) {
        load_frags(nxt, s, kk + 1);
      } else if (it + 1 < KT) {
        const int s1 = (it + 1) % STAGES;
        tm_wait(smem_u32(&full[s1]), (uint32_t)(((it + 1) / STAGES) & 1));
        load_frags(nxt, s1, 0);
      }
#pragma unroll
      for (int fm = 0; fm < Cfg::FM; ++fm)
#pragma unroll
        for (int fn = 0; fn < Cfg::FN; ++fn) dmma_8x8x4(acc[fm][fn], af[cur][fm], bf[cur][fn]);
      if (kk == 3) {
        // release the stage only after the DMMAs that consume its last fragments have been
        // issued: their operands are then in registers, i.e. every shared-memory read of
        // the stage has completed.  Releasing right after ISSUING those reads (one k step
        // earlier) let the next TMA write overtake them whenever another kernel's traffic
        // delayed this CTA's shared-memory pipeline: corrupted tiles next to any heavy
        // neighbour (tools/overlap_tma_grouped.py, DESIGN 6.2)
        __syncwarp();
        if (lane == 0) tm_arrive(smem_u32(&empty[s]));
      }
    }
  }
  // ---- epilogue ----
  if (P.splits > 1) {  // this K slice's partial tile (row-major M x N slab)
    double* part = P.C + (size_t)blockIdx.z * P.M * P.N;
#pragma unroll
    for (int fm = 0; fm < Cfg::FM; ++fm) {
      const int m = m0 + wm * Cfg::WM + fm * 8 + lr;
      if (m >= P.M) continue;
#pragma unroll
      for (int fn = 0; fn < Cfg::FN; ++fn) {
        const int n = n0 + wn * Cfg::WN + fn * 8 + 2 * lk;
        if (n < P.N) part[(size_t)m * P.N + n] = acc[fm][fn][0];
        if (n + 1 < P.N) part[(size_t)m * P.N + n + 1] = acc[fm][fn][1];
      }
    }
    return;
  }
#pragma unroll
  for (int fm = 0; fm < Cfg::FM; ++fm) {
    const int m = m0 + wm * Cfg::WM + fm * 8 + lr;
    if (m >= P.M) continue;
#pragma unroll
    for (int fn = 0; fn < Cfg::FN; ++fn) {
      const int n = n0 + wn * Cfg::WN + fn * 8 + 2 * lk;
      double* c = P.C + (long long)m * P.c_ms + (long long)n * P.c_ns;
      double v0 = P.alpha * acc[fm][fn][0], v1 = P.alpha * acc[fm][fn][1];
      if (P.beta != 0.0) {
        if (n < P.N) v0 = fma(P.beta, c[0], v0);
        if (n + 1 < P.N) v1 = fma(P.beta, c[P.c_ns], v1);
      }
      if (P.c_ns == 1 && n + 1 < P.N && ((reinterpret_cast<uintptr_t>(c) & 15) == 0)) {
        *reinterpret_cast<double2*>(c) = make_double2(v0, v1);
      } else {
        if (n < P.N) c[0] = v0;
        if (n + 1 < P.N) c[P.c_ns] = v1;
      }
    }
  }
}

// C = alpha sum_z part[z] + beta C, fixed order over the splits
__global__ void tma_splitk_reduce_kernel(int M, int N, int splits, const double* __restrict__ part, double alpha,
                                         double beta, double* __restrict__ C, long long c_ms, long long c_ns) {
  const long long mn = (long long)M * N;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < mn; e += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += __ldcg(part + (size_t)z * mn + e);
    const int m = (int)(e / N), n = (int)(e - (long long)m * N);
    double* c = C + (long long)m * c_ms + (long long)n * c_ns;
    *c = beta != 0.0 ? fma(beta, *c, alpha * s) : alpha * s;
  }
}

constexpr int kTmStages = 4;

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D fp64 tensor map of a row-major matrix (rows x cols, ld) with a box of
// box_cols x box_rows (box_cols * 8 = 128 bytes), 128-byte swizzle, zero OOB fill
int make_map(CUtensorMap* map, const double* ptr, long long rows, long long cols, long long ld, int box_cols,
             int box_rows) {
  auto fn = encode_fn();
  TTK_REQUIRE(fn != nullptr, kCudaError, "gemm_tma: cuTensorMapEncodeTiled unavailable");
  const cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ld * 8};
  const cuuint32_t box[2] = {(cuuint32_t)box_cols, (cuuint32_t)box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(ptr), dims, strides, box, estr,
                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TTK_REQUIRE(r == CUDA_SUCCESS, kCudaError, "gemm_tma: cuTensorMapEncodeTiled failed (%d)", (int)r);
  return kOk;
}

// row-major storage of op(X) (trans = false) or of op(X)^T (trans = true)
struct TmOperand {
  const double* ptr;
  long long ld;
  bool trans;
};

template <int BM, int BN, bool TA, bool TB>
int launch_tma(int M, int N, int K, double alpha, TmOperand A, TmOperand B, double beta, double* C, long long c_ms,
               long long c_ns, int splits, double* part, cudaStream_t st) {
  using Cfg = TmCfg<BM, BN, kTmStages>;
  auto kern = gemm_tma_kernel<BM, BN, kTmStages, TA, TB>;
  TTK_TRY(set_attr_once(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
  CUtensorMap ma, mb;
  if (!TA) TTK_TRY(make_map(&ma, A.ptr, M, K, A.ld, kTmBK, BM));  // [m][k]
  else TTK_TRY(make_map(&ma, A.ptr, K, M, A.ld, 16, kTmBK));       // A^T: [k][m]
  if (!TB) TTK_TRY(make_map(&mb, B.ptr, K, N, B.ld, 16, kTmBK));  // [k][n]
  else TTK_TRY(make_map(&mb, B.ptr, N, K, B.ld, kTmBK, BN));       // B^T: [n][k]
  const int KT = (K + kTmBK - 1) / kTmBK;
  const int per = (KT + splits - 1) / splits;
  splits = (KT + per - 1) / per;
  TmParams p{M, N, K, per, alpha, beta, splits > 1 ? part : C, c_ms, c_ns, splits};
  dim3 grid((M + BM - 1) / BM, (N + BN - 1) / BN, splits);
  static const int pad = knob_env("TTK_TMA_SMEM_PAD") ? atoi(knob_env("TTK_TMA_SMEM_PAD")) : 0;  // A/B
  if (pad > 0) {
    static std::once_flag once;
    std::call_once(once, [&] { cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM + pad); });
  }
  kern<<<grid, Cfg::kThreads, Cfg::SMEM + pad, st>>>(ma, mb, p);
  TTK_CHECK_LAUNCH();
  if (splits > 1) {
    const long long mn = (long long)M * N;
    const int blocks = (int)std::min<long long>((mn + 255) / 256, 4LL * num_sms());
    tma_splitk_reduce_kernel<<<blocks, 256, 0, st>>>(M, N, splits, part, alpha, beta, C, c_ms, c_ns);
    TTK_CHECK_LAUNCH();
  }
  return kOk;
}

template <bool TA, bool TB>
int dispatch_tiles(int M, int N, int K, double alpha, TmOperand A, TmOperand B, double beta, double* C,
                   long long c_ms, long long c_ns, void* ws, size_t ws_bytes, cudaStream_t st) {
  const long long two_waves = 2LL * num_sms();
  const bool wide = M <= N;
  int bm = wide ? 80 : 64, bn = wide ? 64 : 80;
  long long tiles = (long long)((M + bm - 1) / bm) * ((N + bn - 1) / bn);
  if (tiles < two_waves && (wide ? N : M) > 64) {  // halve the long side
    if (wide) bn = 32;
    else bm = 32;
    tiles = (long long)((M + bm - 1) / bm) * ((N + bn - 1) / bn);
  }
  // split K when the tiles alone leave SMs idle (>= 4 k tiles per split)
  const int KT = (K + kTmBK - 1) / kTmBK;
  int splits = 1;
  if (tiles < two_waves && KT >= 16 && ws != nullptr) {
    // about one wave of CTAs, >= 8 k tiles each (short slices are all pipeline
    // fill, and every split adds an M x N slab to the reduction)
    splits = (int)std::min<long long>(((long long)num_sms() + tiles - 1) / tiles, KT / 8);
    const size_t per = (size_t)M * N * sizeof(double);
    splits = (int)std::min<size_t>((size_t)splits, ws_bytes / std::max<size_t>(per, 1));
    splits = std::max(splits, 1);
  }
  double* part = reinterpret_cast<double*>(ws);
  if (wide && bn == 32) return launch_tma<80, 32, TA, TB>(M, N, K, alpha, A, B, beta, C, c_ms, c_ns, splits, part, st);
  if (wide) return launch_tma<80, 64, TA, TB>(M, N, K, alpha, A, B, beta, C, c_ms, c_ns, splits, part, st);
  if (bm == 32) return launch_tma<32, 80, TA, TB>(M, N, K, alpha, A, B, beta, C, c_ms, c_ns, splits, part, st);
  return launch_tma<64, 80, TA, TB>(M, N, K, alpha, A, B, beta, C, c_ms, c_ns, splits, part, st);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

// Strided front door (gemm1's convention): A(m,k) = A[m*a_ms + k*a_ks],
// B(k,n) = B[k*b_ks + n*b_ns], C(m,n) = C[m*c_ms + n*c_ns].  Handles row-major
// operands and transposes of row-major operands; a column-major C is computed
// as the transposed problem.  Returns false (nothing launched) when the
// operands do not fit TMA (alignment, odd pitches, K < 16, other layouts).
bool gemm_tma_try(int M, int N, int K, double alpha, const double* A, long long a_ms, long long a_ks,
                  const double* B, long long b_ks, long long b_ns, double beta, double* C, long long c_ms,
                  long long c_ns, void* ws, size_t ws_bytes, cudaStream_t st, int* status, bool force_split_ok) {
  *status = kOk;
  if (M < 2 || N < 2 || K < kTmBK || encode_fn() == nullptr) return false;
  if (c_ms == 1 && c_ns != 1) {
    // column-major C: compute C^T (N x M, row-major) = op(B)^T op(A)^T, i.e. the
    // new A(n,k) = old B(k,n) and the new B(k,m) = old A(m,k)
    std::swap(M, N);
    std::swap(A, B);
    std::swap(a_ms, b_ns);
    std::swap(a_ks, b_ks);
    std::swap(c_ms, c_ns);
  }
  // long-K problems whose tiles leave SMs idle need split K; measured no better
  // than the grouped cp.async kernel's split-K (192x80x10240 25.2 vs 25.1 us,
  // 80x192x10240 24.9 vs 23.0, tools/gemm_tma_check.py) -- leave them to it
  {
    const bool wide = M <= N;
    const long long tiles = wide ? (long long)((M + 79) / 80) * ((N + 31) / 32) : (long long)((M + 31) / 32) * ((N + 79) / 80);
    if (tiles < 2LL * num_sms() && (K + kTmBK - 1) / kTmBK >= 16 && ws != nullptr && !force_split_ok) return false;
  }
  TmOperand oa, ob;
  if (a_ks == 1 && a_ms >= K) oa = {A, a_ms, false};
  else if (a_ms == 1 && a_ks >= M) oa = {A, a_ks, true};
  else return false;
  if (b_ns == 1 && b_ks >= N) ob = {B, b_ks, false};
  else if (b_ks == 1 && b_ns >= K) ob = {B, b_ns, true};
  else return false;
  if (!aligned16(A) || !aligned16(B) || (oa.ld & 1) || (ob.ld & 1)) return false;
  int s;
  if (!oa.trans && !ob.trans)
    s = dispatch_tiles<false, false>(M, N, K, alpha, oa, ob, beta, C, c_ms, c_ns, ws, ws_bytes, st);
  else if (oa.trans && !ob.trans)
    s = dispatch_tiles<true, false>(M, N, K, alpha, oa, ob, beta, C, c_ms, c_ns, ws, ws_bytes, st);
  else if (!oa.trans && ob.trans)
    s = dispatch_tiles<false, true>(M, N, K, alpha, oa, ob, beta, C, c_ms, c_ns, ws, ws_bytes, st);
  else
    s = dispatch_tiles<true, true>(M, N, K, alpha, oa, ob, beta, C, c_ms, c_ns, ws, ws_bytes, st);
  *status = s;
  return true;
}

bool gemm_tma_ok(int M, int N, int K, const double* A, long long lda, const double* B, long long ldb) {
  return M > 1 && N > 1 && K >= kTmBK && aligned16(A) && aligned16(B) && (lda % 2) == 0 && (ldb % 2) == 0 &&
         lda >= K && ldb >= N && encode_fn() != nullptr;
}

int gemm_tma(int M, int N, int K, double alpha, const double* A, long long lda, const double* B, long long ldb,
             double beta, double* C, long long ldc, cudaStream_t st) {
  TTK_REQUIRE(gemm_tma_ok(M, N, K, A, lda, B, ldb), kInvalidValue, "gemm_tma: unsupported operands");
  int status = kOk;
  gemm_tma_try(M, N, K, alpha, A, lda, 1, B, ldb, 1, beta, C, ldc, 1, nullptr, 0, st, &status);
  return status;
}

}  // namespace ttk

using namespace ttk;

extern "C" {

// diagnostics (DESIGN 6.2): a neighbour for overlap experiments -- `blocks` CTAs of
// `threads` threads holding `smem_bytes` of dynamic shared memory; every CTA fills its
// shared memory with a pattern (mode & 1: through cp.async from `src`, else plain
// stores), spins `spin` clocks re-reading it, and counts corrupted words into *bad
__global__ void occupy_kernel(int smem_words, long long spin, int mode, const double* __restrict__ src,
                              int* __restrict__ bad) {
  extern __shared__ double oc_sm[];
  const int tid = threadIdx.x, nt = blockDim.x;
  if (mode & 1) {
    for (int e = tid; e < smem_words; e += nt) cp_async8(oc_sm + e, src + (e & 4095), true);
    cp_async_commit();
    cp_async_wait<0>();
  } else {
    for (int e = tid; e < smem_words; e += nt) oc_sm[e] = src[e & 4095];
  }
  __syncthreads();
  const long long t0 = clock64();
  int wrong = 0;
  do {
    for (int e = tid; e < smem_words; e += nt) wrong += (oc_sm[e] != src[e & 4095]) ? 1 : 0;
  } while (clock64() - t0 < spin);
  if (wrong) atomicAdd(bad, wrong);
}

int ttk_debug_occupy(int blocks, int threads, int smem_bytes, long long spin, int mode, const double* src, int* bad,
                     void* stream) {
  static std::mutex mu;
  {
    std::lock_guard<std::mutex> lock(mu);
    TTK_CHECK_CUDA(cudaFuncSetAttribute(occupy_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  }
  occupy_kernel<<<blocks, threads, smem_bytes, (cudaStream_t)stream>>>(smem_bytes / 8, spin, mode, src, bad);
  TTK_CHECK_LAUNCH();
  return kOk;
}

// C = alpha A B + beta C for row-major fp64 A (M x K, lda), B (K x N, ldb),
// C (M x N, ldc): the TMA-staged DMMA kernel (16-byte aligned bases, even
// leading dimensions, K >= 16).  Asynchronous on `stream`.
int ttk_gemm_tma(int M, int N, int K, double alpha, const double* A, long long lda, const double* B, long long ldb,
                 double beta, double* C, long long ldc, void* stream) {
  return gemm_tma(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, (cudaStream_t)stream);
}

// general strided form (A(m,k) = A[m*a_ms + k*a_ks] etc.; row-major operands or
// transposes of row-major operands; K split over `ws` when it pays); returns
// TTK_INVALID_VALUE without launching when the operands do not fit TMA
int ttk_gemm_tma_strided(int M, int N, int K, double alpha, const double* A, long long a_ms, long long a_ks,
                         const double* B, long long b_ks, long long b_ns, double beta, double* C, long long c_ms,
                         long long c_ns, void* ws, size_t ws_bytes, void* stream) {
  int status = kOk;
  if (!gemm_tma_try(M, N, K, alpha, A, a_ms, a_ks, B, b_ks, b_ns, beta, C, c_ms, c_ns, ws, ws_bytes,
                    (cudaStream_t)stream, &status, true)) {
    set_error("gemm_tma: operands do not fit the TMA kernel");
    return kInvalidValue;
  }
  return status;
}

}  // extern "C"
