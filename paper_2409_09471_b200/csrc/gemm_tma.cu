// TMA-staged fp64 DMMA GEMM for plain row-major operands: C = alpha A B + beta C,
// A (M x K, lda), B (K x N, ldb), C (M x N, ldc).  Used for the skinny
// contractions of the randomize-then-orthogonalize sweeps and the truncation
// (round.cu), whose operands are plain row-major matrices: the right-sweep
// T_c = X_c W_{c+1} (M = R n, N = l, K = R), the left-sweep sketches
// Y = M_{c-1} T_{c-1} and projections Z = M_{c-1} X_{c-1} (M = l).
//
// Operand staging: one producer warp issues cp.async.bulk.tensor (TMA) loads
// of a BM x 16 tile of A and a 16 x BN tile of B (boxes of 16 doubles = one
// 128-byte row) per stage into a ring of STAGES buffers, completion counted in
// bytes on the stage's "full" mbarrier; the four consumer warps release a stage
// on its "empty" mbarrier.  Both tiles use the 128-byte swizzle (16-byte chunk
// index XOR row mod 8), which makes the DMMA m8n8k4 fragment loads -- 8 rows x
// 4 k of A, 4 k x 8 columns of B, one double per lane -- bank-conflict free
// (each 128-byte bank row is hit by exactly two lanes: the two-wavefront
// minimum of a 64-bit warp access).  No per-thread load plan, no cp.async
// address arithmetic in the consumer warps.  Out-of-range rows / columns / k
// are zero-filled by TMA; the epilogue masks the stores.
//
// Tiles: 64 x 80 (tall, N = 80: one column tile covers N, A is read once) and
// 80 x 64 (wide, M = 80), halved along the long side (32 x 80 / 80 x 32) when
// the full tiles would leave fewer than two CTAs per SM; 2 x 2 consumer warps,
// warp tiles up to 32 x 40 / 40 x 32 (20 accumulator fragments).
#include "common.cuh"
#include "gemm.cuh"
#include "../../include/ttk_b200.h"

#include <cuda.h>
#include <cudaTypedefs.h>
#include <mutex>

namespace ttk {

namespace {

constexpr int kTmBK = 16;  // k per stage (one 128-byte swizzle row of A)

template <int BM, int BN, int STAGES>
struct TmCfg {
  static constexpr int kConsumers = 4;
  static constexpr int kThreads = 32 * (kConsumers + 1);
  static constexpr int WM = BM / 2, WN = BN / 2;
  static constexpr int FM = WM / 8, FN = WN / 8;
  static constexpr int A_BYTES = BM * kTmBK * 8;
  static constexpr int B_BYTES = kTmBK * BN * 8;
  static constexpr int NB = BN / 16;  // 16-column boxes of B per stage
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr size_t SMEM = (size_t)STAGES * STAGE_BYTES + 1024;  // + alignment slack
  static_assert(BM % 8 == 0 && BN % 16 == 0, "tile shape");
  static_assert(A_BYTES % 1024 == 0 && B_BYTES % 1024 == 0, "swizzle-128B buffers need 1024-byte alignment");
};

struct TmParams {
  int M, N, K;
  double alpha, beta;
  double* C;
  long long ldc;
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

template <int BM, int BN, int STAGES>
#ifndef TTK_TMA_MINB
#define TTK_TMA_MINB 1
#endif
__global__ void __launch_bounds__(TmCfg<BM, BN, STAGES>::kThreads, TTK_TMA_MINB)
    gemm_tma_kernel(const __grid_constant__ CUtensorMap ma, const __grid_constant__ CUtensorMap mb,
                    const __grid_constant__ TmParams P) {
  using Cfg = TmCfg<BM, BN, STAGES>;
  extern __shared__ unsigned char tm_smem_raw[];
  __shared__ __align__(8) unsigned long long full[STAGES], empty[STAGES];
  const uint32_t raw = smem_u32(tm_smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * BM, n0 = blockIdx.y * BN;
  const int KT = (P.K + kTmBK - 1) / kTmBK;
  auto a_buf = [&](int s) { return base + (uint32_t)(s * Cfg::STAGE_BYTES); };
  auto b_buf = [&](int s, int j) { return base + (uint32_t)(s * Cfg::STAGE_BYTES + Cfg::A_BYTES + j * 2048); };
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
    // ---- producer: one elected lane streams the k tiles ----
    if (lane == 0) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&ma) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&mb) : "memory");
      for (int kt = 0; kt < KT; ++kt) {
        const int s = kt % STAGES;
        if (kt >= STAGES) tm_wait(smem_u32(&empty[s]), (uint32_t)(((kt / STAGES) - 1) & 1));
        const uint32_t fb = smem_u32(&full[s]);
        tm_arrive_tx(fb, (uint32_t)Cfg::STAGE_BYTES);
        tm_load_2d(a_buf(s), &ma, kt * kTmBK, m0, fb);
#pragma unroll
        for (int j = 0; j < Cfg::NB; ++j) tm_load_2d(b_buf(s, j), &mb, n0 + 16 * j, kt * kTmBK, fb);
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
  // lane-constant swizzled offsets.  A (row r, k): r*128 + (((k>>1) ^ (r&7)) << 4) + (k&1)*8,
  // r & 7 = lr for every fragment row; B box (k, nn): k*128 + (((nn>>1) ^ (k&7)) << 4) + (nn&1)*8
  uint32_t a_off[4], b_off[4][Cfg::FN];
#pragma unroll
  for (int kk = 0; kk < 4; ++kk) {
    const int k = kk * 4 + lk;
    a_off[kk] = (uint32_t)((wm * Cfg::WM + lr) * 128 + ((((k >> 1) ^ lr) & 7) << 4) + ((k & 1) << 3));
#pragma unroll
    for (int fn = 0; fn < Cfg::FN; ++fn) {
      const int n = wn * Cfg::WN + fn * 8 + lr;
      const int j = n >> 4, nn = n & 15;
      b_off[kk][fn] = (uint32_t)(Cfg::A_BYTES + j * 2048 + k * 128 + ((((nn >> 1) ^ (k & 7)) & 7) << 4) + ((nn & 1) << 3));
    }
  }
  // generic pointer to the aligned ring: ordinary loads, which the "memory"
  // clobber of the mbarrier wait keeps below it (a volatile asm load without a
  // clobber could be hoisted above the wait and read a stage not yet landed).
  // Fragments are double-buffered in registers: the loads of k-step kk + 1 --
  // or, after the last k-step of a stage, of the next stage's first k-step
  // (behind that stage's wait) -- are issued before the DMMAs of k-step kk, and
  // a stage is released as soon as its last fragments are in registers.
  const unsigned char* ring = tm_smem_raw + (base - raw);
  double af[2][Cfg::FM], bf[2][Cfg::FN];
  auto load_frags = [&](int buf, int s, int kk) {
    const unsigned char* sb = ring + s * Cfg::STAGE_BYTES;
#pragma unroll
    for (int fm = 0; fm < Cfg::FM; ++fm)
      af[buf][fm] = *reinterpret_cast<const double*>(sb + a_off[kk] + fm * 8 * 128);
#pragma unroll
    for (int fn = 0; fn < Cfg::FN; ++fn) bf[buf][fn] = *reinterpret_cast<const double*>(sb + b_off[kk][fn]);
  };
  if (KT > 0) {
    tm_wait(smem_u32(&full[0]), 0u);
    load_frags(0, 0, 0);
  }
  for (int kt = 0; kt < KT; ++kt) {
    const int s = kt % STAGES;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
      const int cur = kk & 1, nxt = cur ^ 1;
      if (kk < 3) {
        load_frags(nxt, s, kk + 1);
        if (kk == 2) {  // the stage's last fragments are loaded: release it
          __syncwarp();
          if (lane == 0) tm_arrive(smem_u32(&empty[s]));
        }
      } else if (kt + 1 < KT) {
        const int s1 = (kt + 1) % STAGES;
        tm_wait(smem_u32(&full[s1]), (uint32_t)(((kt + 1) / STAGES) & 1));
        load_frags(nxt, s1, 0);
      }
#pragma unroll
      for (int fm = 0; fm < Cfg::FM; ++fm)
#pragma unroll
        for (int fn = 0; fn < Cfg::FN; ++fn) dmma_8x8x4(acc[fm][fn], af[cur][fm], bf[cur][fn]);
    }
  }
  // ---- epilogue: C[m][n, n+1] = alpha acc + beta C ----
#pragma unroll
  for (int fm = 0; fm < Cfg::FM; ++fm) {
    const int m = m0 + wm * Cfg::WM + fm * 8 + lr;
    if (m >= P.M) continue;
#pragma unroll
    for (int fn = 0; fn < Cfg::FN; ++fn) {
      const int n = n0 + wn * Cfg::WN + fn * 8 + 2 * lk;
      double* c = P.C + (long long)m * P.ldc + n;
      double v0 = P.alpha * acc[fm][fn][0], v1 = P.alpha * acc[fm][fn][1];
      if (P.beta != 0.0) {
        if (n < P.N) v0 = fma(P.beta, c[0], v0);
        if (n + 1 < P.N) v1 = fma(P.beta, c[1], v1);
      }
      if (n + 1 < P.N && ((reinterpret_cast<uintptr_t>(c) & 15) == 0)) {
        *reinterpret_cast<double2*>(c) = make_double2(v0, v1);
      } else {
        if (n < P.N) c[0] = v0;
        if (n + 1 < P.N) c[1] = v1;
      }
    }
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

template <int BM, int BN>
int launch_tma(int M, int N, int K, double alpha, const double* A, long long lda, const double* B, long long ldb,
               double beta, double* C, long long ldc, cudaStream_t st) {
  using Cfg = TmCfg<BM, BN, kTmStages>;
  auto kern = gemm_tma_kernel<BM, BN, kTmStages>;
  TTK_TRY(set_attr_once(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Cfg::SMEM));
  CUtensorMap ma, mb;
  TTK_TRY(make_map(&ma, A, M, K, lda, kTmBK, BM));
  TTK_TRY(make_map(&mb, B, K, N, ldb, 16, kTmBK));
  TmParams p{M, N, K, alpha, beta, C, ldc};
  dim3 grid((M + BM - 1) / BM, (N + BN - 1) / BN);
  kern<<<grid, Cfg::kThreads, Cfg::SMEM, st>>>(ma, mb, p);
  TTK_CHECK_LAUNCH();
  return kOk;
}

}  // namespace

bool gemm_tma_ok(int M, int N, int K, const double* A, long long lda, const double* B, long long ldb) {
  // TMA: 16-byte aligned bases, row pitches multiple of 16 bytes; skinny shapes only
  auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
  return M > 0 && N > 0 && K >= kTmBK && al(A) && al(B) && (lda % 2) == 0 && (ldb % 2) == 0 && lda >= K &&
         ldb >= N && encode_fn() != nullptr;
}

int gemm_tma(int M, int N, int K, double alpha, const double* A, long long lda, const double* B, long long ldb,
             double beta, double* C, long long ldc, cudaStream_t st) {
  TTK_REQUIRE(gemm_tma_ok(M, N, K, A, lda, B, ldb), kInvalidValue, "gemm_tma: unsupported operands");
  // full-width tiles along the short side; halve the long-side tile when that
  // leaves fewer than two CTAs per SM
  const long long two_waves = 2LL * num_sms();
  if (M <= N) {
    const long long tiles = (long long)((M + 79) / 80) * ((N + 63) / 64);
    if (tiles < two_waves) return launch_tma<80, 32>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, st);
    return launch_tma<80, 64>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, st);
  }
  const long long tiles = (long long)((M + 63) / 64) * ((N + 79) / 80);
  if (tiles < two_waves) return launch_tma<32, 80>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, st);
  return launch_tma<64, 80>(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, st);
}

}  // namespace ttk

using namespace ttk;

extern "C" {

// C = alpha A B + beta C for row-major fp64 A (M x K, lda), B (K x N, ldb),
// C (M x N, ldc): the TMA-staged DMMA kernel (16-byte aligned bases, even
// leading dimensions, K >= 16).  Asynchronous on `stream`.
int ttk_gemm_tma(int M, int N, int K, double alpha, const double* A, long long lda, const double* B, long long ldb,
                 double beta, double* C, long long ldc, void* stream) {
  return gemm_tma(M, N, K, alpha, A, lda, B, ldb, beta, C, ldc, (cudaStream_t)stream);
}

}  // extern "C"
