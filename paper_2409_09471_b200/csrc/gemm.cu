// Host launch logic for the grouped fp64 DMMA GEMM (see gemm.cuh).
#include "gemm.cuh"

#include <algorithm>

namespace ttk {

__global__ void gemm_splitk_reduce_kernel(const __grid_constant__ GemmGroup G) {
  // one CTA-strided pass over every problem that was split
  for (int pi = 0; pi < G.count; ++pi) {
    const GemmProblem& P = G.p[pi];
    if (P.splits <= 1) continue;
    const size_t mn = (size_t)P.M * P.N;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < mn;
         e += (size_t)gridDim.x * blockDim.x) {
      // fixed summation order; loads issued 8 at a time so the L2 latency of the
      // partials overlaps instead of chaining
      double s = 0.0;
      int k = 0;
      for (; k + 8 <= P.splits; k += 8) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) v[u] = __ldcg(P.partial + (size_t)(k + u) * mn + e);
#pragma unroll
        for (int u = 0; u < 8; ++u) s += v[u];
      }
      for (; k < P.splits; ++k) s += __ldcg(P.partial + (size_t)k * mn + e);
      int m = (int)(e / P.N), n = (int)(e % P.N);
      double* dst = P.C + cmap_m(P, m) + cmap_n(P, n);
      double v = P.alpha * s;
      if (P.beta != 0.0) v += P.beta * *dst;
      *dst = v;
    }
  }
}

namespace {

enum TileCfg { kT128x128 = 0, kT128x64 = 1, kT64x64 = 2, kT64x32 = 3, kT128x80 = 4 };

struct CfgDims { int bm, bn; };
constexpr CfgDims kDims[] = {{128, 128}, {128, 64}, {64, 64}, {64, 32}, {128, 80}};

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
  // pick by the largest problem; small-N problems use narrower tiles
  long best = 0; int bm = 0, bn = 0;
  for (int i = 0; i < count; ++i) {
    long mn = (long)probs[i].M * probs[i].N;
    if (mn > best) { best = mn; bm = probs[i].M; bn = probs[i].N; }
  }
  long tiles128 = 0;
  for (int i = 0; i < count; ++i) tiles128 += (long)ceil_div(probs[i].M, 128) * ceil_div(probs[i].N, 128);
  if (bn <= 32 && bm >= 64) return kT64x32;
  if (bm >= 512 && bn > 64 && bn <= 80) return kT128x80;
  if (bm >= 128 && bn >= 128 && tiles128 >= kNumSMs) return kT128x128;
  if (bm >= 128 && bn > 32 && bn <= 64) return kT128x64;
  if (bm >= 128 && bn >= 96) return tiles128 >= kNumSMs / 2 ? kT128x128 : kT64x64;
  return kT64x64;
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
      s = (int)std::max(1L, std::min(want, std::min(maxs, 64L)));
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

template <int BM, int BN, int WM, int WN>
int launch_cfg(GemmGroup& g, cudaStream_t st) {
  using Cfg = GemmCfg<BM, BN, kBK, WM, WN, kStages>;
  auto kern = gemm_group_kernel<BM, BN, kBK, WM, WN, kStages>;
  static bool attr_set = false;
  if (!attr_set) {
    TTK_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        (int)Cfg::kSmemBytes));
    attr_set = true;
  }
  kern<<<g.total_tiles, Cfg::kThreads, Cfg::kSmemBytes, st>>>(g);
  TTK_CHECK_LAUNCH();
  return kOk;
}

}  // namespace

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
    int rc;
    switch (cfg) {
      case kT128x128: rc = launch_cfg<128, 128, 2, 4>(g, st); break;
      case kT128x64: rc = launch_cfg<128, 64, 2, 2>(g, st); break;
      case kT64x64: rc = launch_cfg<64, 64, 2, 2>(g, st); break;
      case kT128x80: rc = launch_cfg<128, 80, 4, 2>(g, st); break;
      default: rc = launch_cfg<64, 32, 2, 1>(g, st); break;
    }
    if (rc != kOk) return rc;
    if (pe > 0) {
      size_t maxmn = 0;
      for (int i = 0; i < g.count; ++i)
        if (g.p[i].splits > 1) maxmn = std::max(maxmn, (size_t)g.p[i].M * g.p[i].N);
      const int rblocks = (int)std::min<size_t>((maxmn + 127) / 128, 4 * kNumSMs);
      gemm_splitk_reduce_kernel<<<std::max(rblocks, 1), 128, 0, st>>>(g);
      TTK_CHECK_LAUNCH();
    }
  }
  return kOk;
}

}  // namespace ttk
