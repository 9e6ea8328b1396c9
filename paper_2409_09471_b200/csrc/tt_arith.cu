// TT-axpy / concatenation (reference tt_add + tt_scale, tt.py:254-282) and
// small elementwise helpers.  HBM-streaming kernels: every output element is
// written exactly once, every input element read exactly once.
#include "common.cuh"
#include "../../include/ttk_b200.h"

#include <vector>

namespace ttk {

constexpr int kMaxConcatTerms = 16;
constexpr int kMaxConcatCores = 64;

struct ConcatCore {
  double* out;
  long long rows;     // R0_total * n   (output rows, each of length R1_total)
  long long row_begin;  // prefix over cores (in rows)
  int blk_begin;        // first CTA of this core
  int R0, R1, n;
  int kind;  // 0 first (concat along axis 2), 1 middle (block diagonal), 2 last (axis 0), 3 d==1 (sum)
  const double* in[kMaxConcatTerms];
  int r0_off[kMaxConcatTerms + 1];  // row-block offsets (prefix of r0 over terms)
  int r1_off[kMaxConcatTerms + 1];  // col-block offsets
};

struct ConcatParams {
  int nterms;
  int ncores;
  long long total_rows;
  double coeff[kMaxConcatTerms];
  ConcatCore c[kMaxConcatCores];
};

// Block-diagonal concatenation (tt_add generalised to a linear combination,
// tt.py:254-275 + tt_scale tt.py:278-282).  Each CTA owns kConcatRows output
// rows of ONE core (found once by binary search over per-core CTA offsets):
// first/middle cores are written warp-per-row with 16-byte stores (zeros
// outside the term's column block), last cores and d == 1 thread-per-element.
// Multiply and add stay separate (no FMA contraction): bit-exact with numpy.
constexpr int kConcatRows = 64;

__device__ __forceinline__ double concat_elem(const ConcatCore& C, const double* src, int c0, int w, int col) {
  return (col >= c0 && col < c0 + w) ? src[col - c0] : 0.0;
}

__global__ void __launch_bounds__(256) concat_kernel(const __grid_constant__ ConcatParams P) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  int lo = 0, hi = P.ncores - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (P.c[mid].blk_begin <= (int)blockIdx.x) lo = mid; else hi = mid - 1;
  }
  const ConcatCore& C = P.c[lo];
  const long long r_begin = (long long)(blockIdx.x - C.blk_begin) * kConcatRows;
  const long long r_end = min(C.rows, r_begin + kConcatRows);
  if (C.kind == 2 || C.kind == 3) {
    // one output element per row: thread per element
    for (long long row = r_begin + threadIdx.x; row < r_end; row += blockDim.x) {
      const int r = (int)(row / C.n);
      const int i = (int)(row - (long long)r * C.n);
      if (C.kind == 3) {
        for (int col = 0; col < C.R1; ++col) {  // d == 1: R1 == 1 after normalisation
          double acc = P.coeff[0] == 1.0 ? C.in[0][(long long)i * C.R1 + col]
                                         : __dmul_rn(P.coeff[0], C.in[0][(long long)i * C.R1 + col]);
          for (int t = 1; t < P.nterms; ++t)
            acc = __dadd_rn(acc, __dmul_rn(P.coeff[t], C.in[t][(long long)i * C.R1 + col]));
          C.out[row * C.R1 + col] = acc;
        }
      } else {
        int t = 0;
        while (t + 1 < P.nterms && C.r0_off[t + 1] <= r) ++t;
        const double v = C.in[t][(long long)(r - C.r0_off[t]) * C.n + i];
        C.out[row] = (P.coeff[t] == 1.0) ? v : v * P.coeff[t];
      }
    }
    return;
  }
  const bool vec = (C.R1 % 2 == 0) && ((reinterpret_cast<uintptr_t>(C.out) & 15) == 0);
  for (long long row = r_begin + warp; row < r_end; row += nwarps) {
    const int r = (int)(row / C.n);
    const int i = (int)(row - (long long)r * C.n);
    double* dst = C.out + row * C.R1;
    if (C.kind == 0) {
      // first core: R0 == 1, the terms' columns side by side (axis 2)
      for (int col = lane; col < C.R1; col += 32) {
        int tt = 0;
        while (tt + 1 < P.nterms && C.r1_off[tt + 1] <= col) ++tt;
        const int w = C.r1_off[tt + 1] - C.r1_off[tt];
        dst[col] = C.in[tt][(long long)i * w + (col - C.r1_off[tt])];
      }
      continue;
    }
    int t = 0;
    while (t + 1 < P.nterms && C.r0_off[t + 1] <= r) ++t;
    const int c0 = C.r1_off[t], w = C.r1_off[t + 1] - c0;
    const double* src = C.in[t] + ((long long)(r - C.r0_off[t]) * C.n + i) * w;
    if (vec) {
      double2* d2 = reinterpret_cast<double2*>(dst);
      for (int cp = lane; cp < (C.R1 >> 1); cp += 32) {
        const int col = cp << 1;
        d2[cp] = make_double2(concat_elem(C, src, c0, w, col), concat_elem(C, src, c0, w, col + 1));
      }
    } else {
      for (int col = lane; col < C.R1; col += 32) dst[col] = concat_elem(C, src, c0, w, col);
    }
  }
}

__global__ void scale_kernel(double* y, const double* x, long long n, double alpha) {
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    y[e] = x[e] * alpha;
}

// sum of squares, fixed-order two-level reduction (block partials then one block)
__global__ void sumsq_partial_kernel(const double* x, long long n, double* part) {
  __shared__ double red[32];
  double s = 0.0;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x)
    s += x[e] * x[e];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) part[blockIdx.x] = v;
  }
}

__global__ void sum_final_kernel(const double* part, int n, double* out) {
  __shared__ double red[32];
  double s = 0.0;
  for (int e = threadIdx.x; e < n; e += blockDim.x) s += part[e];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) out[0] = v;
  }
}

int launch_sumsq(const double* x, long long n, double* out_dev, double* part, cudaStream_t st) {
  const int blocks = 256;
  sumsq_partial_kernel<<<blocks, 256, 0, st>>>(x, n, part);
  TTK_CHECK_LAUNCH();
  sum_final_kernel<<<1, 256, 0, st>>>(part, blocks, out_dev);
  TTK_CHECK_LAUNCH();
  return kOk;
}

}  // namespace ttk

using namespace ttk;

extern "C" {

// out = sum_t coeff[t] * term_t, block-diagonal TT concatenation (reference
// solvers.py:361-366: tt_add(vt, tt_scale(v_i, -h_i)) chained left to right).
// ranks: nterms x (d+1) host array; in: nterms x d device pointers (row-major,
// term-major); out: d device pointers, core k of shape (sum_t r_t[k], n[k], sum_t r_t[k+1])
// (interior), with the boundary ranks 1 for k = 0 / d-1.
int ttk_tt_concat(int d, int nterms, const double* coeff, const int* dims, const int* ranks,
                  const double* const* in, double* const* out, void* stream) {
  TTK_REQUIRE(d >= 1 && d <= kMaxConcatCores, kInvalidValue, "d=%d out of range [1,%d]", d,
              kMaxConcatCores);
  TTK_REQUIRE(nterms >= 1 && nterms <= kMaxConcatTerms, kInvalidValue,
              "nterms=%d out of range [1,%d]", nterms, kMaxConcatTerms);
  static thread_local ConcatParams P;
  P.nterms = nterms;
  P.ncores = d;
  for (int t = 0; t < nterms; ++t) {
    P.coeff[t] = coeff[t];
    TTK_REQUIRE(ranks[t * (d + 1)] == 1 && ranks[t * (d + 1) + d] == 1, kShapeMismatch,
                "term %d: boundary ranks must equal 1", t);
  }
  long long rows = 0, blocks_total = 0;
  for (int k = 0; k < d; ++k) {
    ConcatCore& C = P.c[k];
    C.out = out[k];
    C.n = dims[k];
    C.kind = (d == 1) ? 3 : (k == 0 ? 0 : (k == d - 1 ? 2 : 1));
    C.r0_off[0] = 0;
    C.r1_off[0] = 0;
    for (int t = 0; t < nterms; ++t) {
      C.in[t] = in[t * d + k];
      C.r0_off[t + 1] = C.r0_off[t] + ranks[t * (d + 1) + k];
      C.r1_off[t + 1] = C.r1_off[t] + ranks[t * (d + 1) + k + 1];
    }
    C.R0 = (C.kind == 0 || C.kind == 3) ? 1 : C.r0_off[nterms];
    C.R1 = (C.kind == 2 || C.kind == 3) ? 1 : C.r1_off[nterms];
    C.rows = (long long)C.R0 * C.n;
    C.row_begin = rows;
    C.blk_begin = (int)blocks_total;
    blocks_total += (C.rows + kConcatRows - 1) / kConcatRows;
    rows += C.rows;
  }
  P.total_rows = rows;
  if (rows == 0) return kOk;
  TTK_REQUIRE(blocks_total < (1LL << 31), kInvalidValue, "tt_concat: output too large");
  const int blocks = (int)blocks_total;
  concat_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(P);
  TTK_CHECK_LAUNCH();
  return kOk;
}

int ttk_scale(double* y, const double* x, long long n, double alpha, void* stream) {
  if (n <= 0) return kOk;
  int blocks = (int)std::min<long long>((n + 255) / 256, 4LL * kNumSMs);
  scale_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(y, x, n, alpha);
  TTK_CHECK_LAUNCH();
  return kOk;
}

// out_dev[0] = sum x^2 (fixed reduction order; deterministic). ws >= 256 doubles.
int ttk_sumsq(const double* x, long long n, double* out_dev, void* ws, size_t ws_bytes,
              void* stream) {
  TTK_REQUIRE(ws_bytes >= 256 * sizeof(double) && ws != nullptr, kWorkspace, "sumsq workspace too small");
  return launch_sumsq(x, n, out_dev, (double*)ws, (cudaStream_t)stream);
}

}  // extern "C"
