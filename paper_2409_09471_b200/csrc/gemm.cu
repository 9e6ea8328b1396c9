// Host launch logic for the grouped fp64 DMMA GEMM (see gemm.cuh).
#include "gemm.cuh"

#include <algorithm>
#include <cstdio>
#include <cstdlib>

namespace ttk {

// Deterministic split-K reduction.  A block owns 32 consecutive output
// elements of one problem; its kRedGroups thread groups each sum a fixed,
// interleaved subset of the splits (group g: splits g, g+G, ...), then group 0
// adds the group sums in order.  The summation order depends only on `splits`.
constexpr int kRedGroups = 8;

// Few splits (<= kRedGroups): one thread per output element, partials summed
// in split order; fully parallel, no barriers.  Problems with more splits are
// left to gemm_splitk_reduce_kernel.
template <int CAP>
__global__ void gemm_splitk_reduce_small_kernel(const __grid_constant__ GemmGroupT<CAP> G) {
  long long total = 0;
  for (int pi = 0; pi < G.count; ++pi)
    if (G.p[pi].splits > 1 && G.p[pi].splits <= kRedGroups) total += (long long)G.p[pi].M * G.p[pi].N;
  for (long long ge = blockIdx.x * (long long)blockDim.x + threadIdx.x; ge < total;
       ge += (long long)gridDim.x * blockDim.x) {
    long long e = ge;
    int pi = 0;
    for (; pi < G.count; ++pi) {
      if (G.p[pi].splits <= 1 || G.p[pi].splits > kRedGroups) continue;
      const long long n = (long long)G.p[pi].M * G.p[pi].N;
      if (e < n) break;
      e -= n;
    }
    const GemmProblem& P = G.p[pi];
    const size_t mn = (size_t)P.M * P.N;
    double v[kRedGroups];
#pragma unroll
    for (int k = 0; k < kRedGroups; ++k) v[k] = (k < P.splits) ? __ldcg(P.partial + (size_t)k * mn + e) : 0.0;
    double t = v[0];
#pragma unroll
    for (int k = 1; k < kRedGroups; ++k)
      if (k < P.splits) t += v[k];
    const int m = (int)(e / P.N), n = (int)(e % P.N);
    double* dst = P.C + cmap_m(P, m) + cmap_n(P, n);
    double out = P.alpha * t;
    if (P.beta != 0.0) out += P.beta * *dst;
    *dst = out;
  }
}

template <int CAP>
__global__ void gemm_splitk_reduce_kernel(const __grid_constant__ GemmGroupT<CAP> G) {
  __shared__ double part[kRedGroups][33];
  const int lane = threadIdx.x & 31, grp = threadIdx.x >> 5;
  long long total = 0;
  for (int pi = 0; pi < G.count; ++pi)
    if (G.p[pi].splits > kRedGroups) total += ((long long)G.p[pi].M * G.p[pi].N + 31) / 32;
  for (long long gc = blockIdx.x; gc < total; gc += gridDim.x) {
    // locate the problem and chunk (block-uniform)
    long long c = gc;
    int pi = 0;
    for (; pi < G.count; ++pi) {
      if (G.p[pi].splits <= kRedGroups) continue;
      const long long n = ((long long)G.p[pi].M * G.p[pi].N + 31) / 32;
      if (c < n) break;
      c -= n;
    }
    const GemmProblem& P = G.p[pi];
    const size_t mn = (size_t)P.M * P.N;
    const size_t e = (size_t)c * 32 + lane;
    double s = 0.0;
    if (e < mn) {
      int k = grp;
      for (; k + 3 * kRedGroups < P.splits; k += 4 * kRedGroups) {
        const double v0 = __ldcg(P.partial + (size_t)k * mn + e);
        const double v1 = __ldcg(P.partial + (size_t)(k + kRedGroups) * mn + e);
        const double v2 = __ldcg(P.partial + (size_t)(k + 2 * kRedGroups) * mn + e);
        const double v3 = __ldcg(P.partial + (size_t)(k + 3 * kRedGroups) * mn + e);
        s += v0; s += v1; s += v2; s += v3;
      }
      for (; k < P.splits; k += kRedGroups) s += __ldcg(P.partial + (size_t)k * mn + e);
    }
    part[grp][lane] = s;
    __syncthreads();
    if (grp == 0 && e < mn) {
      double t = part[0][lane];
#pragma unroll
      for (int g = 1; g < kRedGroups; ++g) t += part[g][lane];
      const int m = (int)(e / P.N), n = (int)(e % P.N);
      double* dst = P.C + cmap_m(P, m) + cmap_n(P, n);
      double v = P.alpha * t;
      if (P.beta != 0.0) v += P.beta * *dst;
      *dst = v;
    }
    __syncthreads();
  }
}

namespace {

enum TileCfg { kT128x128 = 0, kT128x64 = 1, kT64x64 = 2, kT64x32 = 3, kT128x80 = 4, kT64x80 = 5,
               kT80x64 = 6, kT80x80 = 7, kX64x32w4 = 8, kX64x64w4s4 = 9, kX128x64w8s4 = 10, kX32x64w4 = 11 };

struct CfgDims { int bm, bn; };
constexpr CfgDims kDims[] = {{128, 128}, {128, 64}, {64, 64}, {64, 32}, {128, 80}, {64, 80},
                             {80, 64},   {80, 80},  {64, 32}, {64, 64}, {128, 64}, {32, 64}};

// C = A B  <=>  C^T = B^T A^T: make the output's contiguous direction the
// column (n) index so the epilogue stores are coalesced (1-level maps only)
void normalize_output(GemmProblem& p) {
  const int big = 1 << 30;
  if (!(p.c_ns0 != 1 && p.c_ms0 == 1)) return;
  if (p.a_mdiv != big || p.b_ndiv != big || p.c_mdiv != big || p.c_ndiv != big) return;
  GemmProblem q = p;
  q.M = p.N; q.N = p.M;
  q.A = p.B; q.a_ms0 = p.b_ns0; q.a_ks = p.b_ks;
  q.B = p.A; q.b_ns0 = p.a_ms0; q.b_ks = p.a_ks;
  q.c_ms0 = p.c_ns0; q.c_ns0 = p.c_ms0;
  p = q;
}

TileCfg pick_cfg(const GemmProblem* probs, int count) {
  // Light 64 x 32 (tall output) / 32 x 64 (wide output) tiles, 4 warps, 4
  // stages, ~16 resident warps per SM -- the cuBLAS DGEMM shape.  Measured on
  // every GEMM shape of the workload (tools/gemm_cfg_sweep.py): they win or tie
  // the larger tiles everywhere, including 4096^3 (30.7 TF/s) and the grouped
  // matvec (24.4 TF/s).
  long best = 0; int bm = 0, bn = 0;
  for (int i = 0; i < count; ++i) {
    long mn = (long)probs[i].M * probs[i].N;
    if (mn > best) { best = mn; bm = probs[i].M; bn = probs[i].N; }
  }
  return (bm >= bn) ? kX64x32w4 : kX32x64w4;
}

constexpr int kBK = 16;
constexpr int kStages = 3;

void plan(GemmProblem* probs, int count, TileCfg c, bool allow_split, size_t* partial_elems, int* total) {
  int bm = kDims[c].bm, bn = kDims[c].bn;
  long tiles = 0;
  for (int i = 0; i < count; ++i) {
    probs[i].tiles_m = ceil_div(probs[i].M, bm);
    probs[i].tiles_n = ceil_div(probs[i].N, bn);
    tiles += (long)probs[i].tiles_m * probs[i].tiles_n;
  }
  size_t pe = 0;
  int t = 0;
  for (int i = 0; i < count; ++i) {
    GemmProblem& p = probs[i];
    int s = 1;
    long mytiles = (long)p.tiles_m * p.tiles_n;
    if (allow_split && tiles < 2L * kNumSMs && p.K >= 8 * kBK && mytiles > 0) {
      // spread the K reduction so the whole group covers ~2 waves
      long want = (2L * kNumSMs + tiles - 1) / tiles;
      long maxs = p.K / (4 * kBK);
      s = (int)std::max(1L, std::min(want, std::min(maxs, 192L)));
    }
    p.splits = s;
    p.k_per_split = ceil_div(ceil_div(p.K, s), kBK) * kBK;
    if (p.k_per_split <= 0) p.k_per_split = kBK;
    // recompute the effective number of splits after rounding
    p.splits = std::max(1, ceil_div(p.K, p.k_per_split));
    if (p.splits > 1) pe += (size_t)p.splits * p.M * p.N;
    p.tile_begin = t;
    t += p.tiles_m * p.tiles_n * p.splits;
  }
  *partial_elems = pe;
  *total = t;
}

template <int BM, int BN, int WM, int WN, int ST, int CAP>
int launch_cfg(GemmGroupT<CAP>& g, cudaStream_t st) {
  using Cfg = GemmCfg<BM, BN, kBK, WM, WN, ST>;
  auto kern = gemm_group_kernel<BM, BN, kBK, WM, WN, ST, CAP>;
  {  // per-device attributes (set_attr_once)
    TTK_TRY(set_attr_once(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)Cfg::kSmemBytes));
  }
  kern<<<g.total_tiles, Cfg::kThreads, Cfg::kSmemBytes, st>>>(g);
  TTK_CHECK_LAUNCH();
  return kOk;
}

}  // namespace

// tile kernel + split-K reduction for one planned group; the group's kernel
// parameter is CAP problems wide (single-problem launches pass ~0.7 KB, not 17 KB)
template <int CAP>
int launch_group(GemmGroupT<CAP>& g, TileCfg cfg, size_t pe, cudaStream_t st) {
  int rc;
  if constexpr (CAP > kSmallGroup) {
    // grouped launches (tt_matvec, sketches) use the default light tiles
    if (cfg != kX32x64w4) cfg = kX64x32w4;
  }
  switch (cfg) {
    case kX64x32w4: rc = launch_cfg<64, 32, 2, 2, 4>(g, st); break;
    case kX32x64w4: rc = launch_cfg<32, 64, 2, 2, 4>(g, st); break;
    // experiment-only configurations (TTK_GEMM_FORCE_CFG), single-problem launches
    case kT128x128: rc = launch_cfg<128, 128, 4, 4, 3>(g, st); break;
    case kT128x64: case kX128x64w8s4: rc = launch_cfg<128, 64, 4, 2, 4>(g, st); break;
    case kT64x64: case kX64x64w4s4: rc = launch_cfg<64, 64, 2, 2, 4>(g, st); break;
    case kT128x80: rc = launch_cfg<128, 80, 8, 1, 3>(g, st); break;
    case kT64x80: rc = launch_cfg<64, 80, 4, 1, 3>(g, st); break;
    case kT80x64: rc = launch_cfg<80, 64, 5, 1, 3>(g, st); break;
    case kT80x80: rc = launch_cfg<80, 80, 5, 1, 3>(g, st); break;
    default: rc = launch_cfg<64, 32, 2, 2, 4>(g, st); break;
  }
  if (rc != kOk) return rc;
  if (pe > 0) {
    size_t chunks = 0, small = 0;
    for (int i = 0; i < g.count; ++i) {
      if (g.p[i].splits > kRedGroups) chunks += ((size_t)g.p[i].M * g.p[i].N + 31) / 32;
      else if (g.p[i].splits > 1) small += (size_t)g.p[i].M * g.p[i].N;
    }
    if (small > 0) {
      const int sblocks = (int)std::min<size_t>((small + 255) / 256, 8 * kNumSMs);
      gemm_splitk_reduce_small_kernel<CAP><<<sblocks, 256, 0, st>>>(g);
      TTK_CHECK_LAUNCH();
    }
    if (chunks > 0) {
      const int rblocks = (int)std::min<size_t>(chunks, 8 * kNumSMs);
      gemm_splitk_reduce_kernel<CAP><<<rblocks, 32 * kRedGroups, 0, st>>>(g);
      TTK_CHECK_LAUNCH();
    }
  }
  return kOk;
}

size_t gemm_group_ws_bytes(const GemmProblem* probs_in, int count, bool allow_split) {
  size_t total = 0;
  for (int base = 0; base < count; base += kMaxGroup) {
    int c = std::min(kMaxGroup, count - base);
    GemmProblem tmp[kMaxGroup];
    for (int i = 0; i < c; ++i) { tmp[i] = probs_in[base + i]; normalize_output(tmp[i]); }
    TileCfg cfg = pick_cfg(tmp, c);
    size_t pe; int tt;
    plan(tmp, c, cfg, allow_split, &pe, &tt);
    total = std::max(total, pe * sizeof(double));
  }
  return total;
}

int gemm_group_launch(GemmProblem* probs, int count, void* ws, size_t ws_bytes, cudaStream_t st,
                      bool allow_split) {
  for (int base = 0; base < count; base += kMaxGroup) {
    int c = std::min(kMaxGroup, count - base);
    static thread_local GemmGroup g;
    int nonempty = 0;
    for (int i = 0; i < c; ++i) {
      const GemmProblem& p = probs[base + i];
      if (p.M <= 0 || p.N <= 0) continue;
      g.p[nonempty] = p;
      normalize_output(g.p[nonempty]);
      ++nonempty;
    }
    if (nonempty == 0) continue;
    g.count = nonempty;
    TileCfg cfg = pick_cfg(g.p, g.count);
    static const int force = knob_env("TTK_GEMM_FORCE_CFG") ? atoi(knob_env("TTK_GEMM_FORCE_CFG")) : -1;  // experiments
    if (force >= 0) cfg = (TileCfg)force;
    size_t pe; int total;
    plan(g.p, g.count, cfg, allow_split && ws != nullptr, &pe, &total);
    if (pe * sizeof(double) > ws_bytes) {
      // not enough workspace: fall back to unsplit launch
      plan(g.p, g.count, cfg, false, &pe, &total);
    }
    double* part = reinterpret_cast<double*>(ws);
    size_t off = 0;
    for (int i = 0; i < g.count; ++i) {
      GemmProblem& p = g.p[i];
      if (p.K <= 0) {  // empty contraction: C = beta*C (alpha*0)
        p.splits = 1;
      }
      if (p.splits > 1) { p.partial = part + off; off += (size_t)p.splits * p.M * p.N; }
    }
    g.total_tiles = total;
    for (int i = 0; i < g.count; ++i) {
      // operand offsets are 32-bit inside the kernel (see TileLoader)
      const GemmProblem& q = g.p[i];
      auto span = [](long long s0, long long s1, int div, int n) {
        const long long d = std::min<long long>(div, n);
        return (long long)((n + d - 1) / d) * (s1 < 0 ? -s1 : s1) + d * (s0 < 0 ? -s0 : s0);
      };
      const long long sa = span(q.a_ms0, q.a_ms1, q.a_mdiv, q.M) + (long long)q.K * (q.a_ks < 0 ? -q.a_ks : q.a_ks);
      const long long sb = span(q.b_ns0, q.b_ns1, q.b_ndiv, q.N) + (long long)q.K * (q.b_ks < 0 ? -q.b_ks : q.b_ks);
      TTK_REQUIRE(sa < (1LL << 31) && sb < (1LL << 31), kInvalidValue,
                  "gemm: operand spans %lld / %lld elements, limit 2^31", sa, sb);
    }
    static const bool trace = knob_env("TTK_GEMM_TRACE") != nullptr;  // shape log (diagnostics)
    if (trace) fprintf(stderr, "gemm-launch count=%d\n", g.count);
    if (trace)
      for (int i = 0; i < g.count; ++i)
        fprintf(stderr, "gemm cfg=%d M=%d N=%d K=%d splits=%d tiles=%d a_ks=%lld b_ks=%lld\n", (int)cfg,
                g.p[i].M, g.p[i].N, g.p[i].K, g.p[i].splits, g.p[i].tiles_m * g.p[i].tiles_n,
                g.p[i].a_ks, g.p[i].b_ks);
    int rc;
    if (g.count <= kSmallGroup) {
      static thread_local GemmGroupSmall gs;
      gs.count = g.count;
      gs.total_tiles = g.total_tiles;
      for (int i = 0; i < g.count; ++i) gs.p[i] = g.p[i];
      rc = launch_group(gs, cfg, pe, st);
    } else {
      rc = launch_group(g, cfg, pe, st);
    }
    if (rc != kOk) return rc;
  }
  return kOk;
}

}  // namespace ttk
