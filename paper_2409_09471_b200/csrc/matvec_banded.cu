// Structure-aware tt_matvec for operators whose blocks D_k[alpha, :, :, beta]
// are banded (zero, scaled identity, tridiagonal, pentadiagonal): SURVEY
// section 8(f) #3 -- the identity / tridiagonal operator cores that the
// reference contracts densely (tt.py:302-314).  Same output layout as
// ttk_matvec (vector-rank major, operator-rank minor):
//   G_k[(a*rho0+al), i, (b*rho1+be)] = sum_{|j-i|<=w} D_k[al,i,j,be] * C_k[a,j,b]
// With 2w+1 <= 5 terms per output this is a write stream.  A CTA owns R whole
// output row pairs (a, i) x a chunk of BW vector columns b (R*BW <= 256): one
// thread per input element (a, i, b) loads its 2w+1 band neighbours
// C_k[a, i-w..i+w, b] once (coalesced across b) and computes all rho0*rho1
// outputs that use them into a shared-memory tile; warps then write every
// (row, al) segment -- contiguous in G -- with consecutive 8-byte stores.
// (Storing straight from registers strides the warp's stores by rho1: 3.2x
// the L1 store sectors, L1-bound at 56 % of HBM in ncu.)  The band table is
// band_k[((al*rho1+be)*n + i)*(2w+1) + t] = D_k[al, i, i+t-w, be].
#include "common.cuh"
#include "../../include/ttk_b200.h"

#include <algorithm>

namespace ttk {

constexpr int kBandMaxCores = 64;
constexpr int kBandThreads = 256;
constexpr int kBandMaxBlocks = 16;  // rho0 * rho1 block kinds kept per core (more: all banded)

struct BandCore {
  const double* C;
  double* G;
  const double* band;
  int rows;       // r0 * n output row pairs (a, i)
  int nblocks;    // CTAs of this core
  int r1, n, rho0, rho1;
  int R, BW, nbchunk;  // rows per CTA, columns per CTA, column chunks per row group
  unsigned char kind[kBandMaxBlocks];  // per (al, be) block: 0 zero, 1 diagonal, 2 banded
};

struct BandParams {
  int ncores;
  BandCore c[kBandMaxCores];
};

// one thread's outputs: all (al, be) for input element (a, i, b); RHO0/RHO1 > 0
// unroll the block loops for the common operator ranks (0 = runtime bounds)
template <int W, int RHO0, int RHO1>
__device__ __forceinline__ void banded_outputs(const BandCore& K, const double (&c)[2 * W + 1], int i,
                                               double* o, int BW) {
  constexpr int T = 2 * W + 1;
  const int rho0 = RHO0 ? RHO0 : K.rho0, rho1 = RHO1 ? RHO1 : K.rho1, n = K.n;
  const bool kinds = rho0 * rho1 <= kBandMaxBlocks;
#pragma unroll
  for (int al = 0; al < rho0; ++al) {
#pragma unroll
    for (int be = 0; be < rho1; ++be) {
      const int kd = kinds ? K.kind[al * rho1 + be] : 2;  // uniform over the CTA
      const double* bp = K.band + ((al * rho1 + be) * n + i) * T;
      double s = 0.0;
      if (kd == 1) {
        s = __ldg(bp + W) * c[W];
      } else if (kd == 2) {
#pragma unroll
        for (int t = 0; t < T; ++t) s = fma(__ldg(bp + t), c[t], s);
      }
      o[al * BW * rho1 + be] = s;
    }
  }
}

template <int W>
__global__ void __launch_bounds__(kBandThreads) matvec_banded_kernel(const __grid_constant__ BandParams P) {
  extern __shared__ __align__(16) double tile[];  // [R][rho0][BW][rho1]
  const BandCore& K = P.c[blockIdx.y];  // grid.y = core, grid.x = CTAs of the largest core
  const int blk = blockIdx.x;
  if (blk >= K.nblocks) return;
  const int r1 = K.r1, n = K.n, rho0 = K.rho0, rho1 = K.rho1, R = K.R, BW = K.BW;
  const int rg = K.nbchunk == 1 ? blk : blk / K.nbchunk;
  const int row0 = rg * R, b0 = (blk - rg * K.nbchunk) * BW;
  const int nrows = min(R, K.rows - row0), ncols = min(BW, r1 - b0);
  constexpr int T = 2 * W + 1;
  const int tid = threadIdx.x, rl = tid / BW, bl = tid - rl * BW;
  if (rl < nrows && bl < ncols) {
    const int row = row0 + rl, b = b0 + bl;
    const int a = row / n, i = row - a * n;
    double c[T];
#pragma unroll
    for (int t = 0; t < T; ++t) {
      const int j = i + t - W;
      c[t] = (j >= 0 && j < n) ? __ldg(K.C + (a * n + j) * r1 + b) : 0.0;
    }
    double* o = tile + (rl * rho0 * BW + bl) * rho1;
    switch (rho0 * 8 + rho1) {
      case 1 * 8 + 1: banded_outputs<W, 1, 1>(K, c, i, o, BW); break;
      case 1 * 8 + 2: banded_outputs<W, 1, 2>(K, c, i, o, BW); break;
      case 2 * 8 + 1: banded_outputs<W, 2, 1>(K, c, i, o, BW); break;
      case 2 * 8 + 2: banded_outputs<W, 2, 2>(K, c, i, o, BW); break;
      case 1 * 8 + 3: banded_outputs<W, 1, 3>(K, c, i, o, BW); break;
      case 3 * 8 + 1: banded_outputs<W, 3, 1>(K, c, i, o, BW); break;
      case 3 * 8 + 3: banded_outputs<W, 3, 3>(K, c, i, o, BW); break;
      default: banded_outputs<W, 0, 0>(K, c, i, o, BW);
    }
  }
  __syncthreads();
  // write-out: every (row, al) segment is contiguous in G and in the tile
  const int ldg = r1 * rho1;
  const int seg_len = ncols * rho1, warp = tid >> 5, lane = tid & 31;
  for (int seg = warp; seg < nrows * rho0; seg += kBandThreads / 32) {
    const int sr = seg / rho0, al = seg - sr * rho0;
    const int row = row0 + sr, a = row / n, i = row - a * n;
    double* g = K.G + ((a * rho0 + al) * n + i) * ldg + b0 * rho1;
    const double* src = tile + (sr * rho0 + al) * BW * rho1;
    int off = 0;
    if ((((size_t)g | (size_t)src) & 15) == 0) {  // both 16-byte aligned: paired stores
      const int npair = seg_len >> 1;
      for (int p = lane; p < npair; p += 32)
        reinterpret_cast<double2*>(g)[p] = reinterpret_cast<const double2*>(src)[p];
      off = npair * 2;
    }
    for (int q = off + lane; q < seg_len; q += 32) g[q] = src[q];
  }
}

}  // namespace ttk

using namespace ttk;

extern "C" {

int ttk_matvec_banded(int d, const int* rho, const int* n, const int* r, int w, const double* const* band,
                      const unsigned char* kinds, const double* const* C, double* const* G, void* stream) {
  TTK_REQUIRE(d >= 1 && d <= kBandMaxCores, kInvalidValue, "d must be in [1, %d]", kBandMaxCores);
  TTK_REQUIRE(w >= 0 && w <= 2, kInvalidValue, "half-bandwidth %d outside [0, 2]", w);
  TTK_REQUIRE(rho[0] == 1 && rho[d] == 1 && r[0] == 1 && r[d] == 1, kShapeMismatch,
              "boundary ranks must equal 1");
  static thread_local BandParams P;
  P.ncores = 0;
  long long blocks = 0;  // CTAs of the largest core
  int rho_prod = 1;
  long long kind_off = 0;
  for (int k = 0; k < d; ++k, kind_off += (long long)rho[k - 1] * rho[k]) {
    TTK_REQUIRE(r[k] >= 0 && r[k + 1] >= 0 && rho[k] >= 1 && rho[k + 1] >= 1 && n[k] >= 1, kShapeMismatch,
                "bad shapes at core %d", k);
    const long long rows = (long long)r[k] * n[k];
    // 32-bit offsets inside the kernel: output core and band table below 2^31 elements
    TTK_REQUIRE(rows * rho[k] * r[k + 1] * rho[k + 1] < (1LL << 31), kInvalidValue,
                "core %d output has %lld elements (limit 2^31)", k, rows * rho[k] * r[k + 1] * rho[k + 1]);
    if (rows == 0 || r[k + 1] == 0) continue;
    BandCore& K = P.c[P.ncores++];
    K.C = C[k]; K.G = G[k]; K.band = band[k];
    K.rows = (int)rows;
    K.r1 = r[k + 1]; K.n = n[k]; K.rho0 = rho[k]; K.rho1 = rho[k + 1];
    K.BW = std::min(r[k + 1], kBandThreads);
    K.R = kBandThreads / K.BW;
    K.nbchunk = (r[k + 1] + K.BW - 1) / K.BW;
    rho_prod = std::max(rho_prod, rho[k] * rho[k + 1]);
    for (int q = 0; q < kBandMaxBlocks; ++q)
      K.kind[q] = (kinds != nullptr && q < rho[k] * rho[k + 1]) ? kinds[kind_off + q] : 2;
    const long long nb = (rows + K.R - 1) / K.R * K.nbchunk;
    K.nblocks = (int)nb;
    blocks = std::max(blocks, nb);
  }
  if (P.ncores == 0) return kOk;
  TTK_REQUIRE(blocks < (1LL << 31), kInvalidValue, "grid too large");
  const size_t smem = sizeof(double) * kBandThreads * rho_prod;
  TTK_REQUIRE(smem <= 200 * 1024, kInvalidValue, "operator ranks too large for the banded tile (%d)", rho_prod);
  {  // per-device attributes (set_attr_once)
    for (const void* f : {(const void*)matvec_banded_kernel<0>, (const void*)matvec_banded_kernel<1>,
                          (const void*)matvec_banded_kernel<2>})
      TTK_TRY(set_attr_once(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  }
  cudaStream_t st = (cudaStream_t)stream;
  const dim3 grid((unsigned)blocks, (unsigned)P.ncores);
  if (w == 0) matvec_banded_kernel<0><<<grid, kBandThreads, smem, st>>>(P);
  else if (w == 1) matvec_banded_kernel<1><<<grid, kBandThreads, smem, st>>>(P);
  else matvec_banded_kernel<2><<<grid, kBandThreads, smem, st>>>(P);
  TTK_CHECK_LAUNCH();
  return kOk;
}

}  // extern "C"
