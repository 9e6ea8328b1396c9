// Truncation eigensolver: symmetric eigendecomposition of the small Gram matrix
// G = C C^T (n <= 128) of a core unfolding C (n x m, m >> n) by two-sided cyclic
// Jacobi, with the truncation rank and a numerical certificate decided on the
// device.  Used by the right-to-left truncation of the left-orthogonal RTO
// output (round.cu ttk_tt_truncate_host), replacing "QR of C^T, then one-sided
// Jacobi SVD of R" (the reference's np.linalg.svd at tt.py:361 / oracle
// truncate_left_orth) whenever the certificate holds:
//   C = U S W^T  <=>  G = U S^2 U^T;  keep r;  core <- S_r^{-1} U_r^T C  (= W_r^T),
//   left neighbour <- x_3 U_r S_r.
//
// Why two-sided on the Gram: a one-sided round needs dot products and a lane
// reduction per pair before the rotation (and a column exchange after); here
// the three numbers a rotation needs (g_pp, g_qq, g_pq) are maintained in the
// Gram itself, so a round is "rotate, then update every 2x2 block once".
//
// Layout and schedule (one thread-block cluster of 1 + kEigUCtas CTAs):
//  * CTA 0 owns G: the upper triangle in shared memory (ld = 1 mod 16 doubles,
//    so both row and column sweeps of consecutive indices are bank-conflict
//    free), the diagonal in a double-buffered array.  Players (indices) are
//    paired by the circle method (position 0 fixed, positions 1..np-1 rotate),
//    evaluated arithmetically -- no pairing tables, no data movement.
//  * Round t: every off-diagonal block (pair slot a, pair slot b) of the round
//    is rotated from both sides ONCE by one thread (4 entries, 16 DFMA).  The
//    threads that own the h "designated" blocks (each holds the off-diagonal
//    entry of one pair of round t+1) immediately compute that pair's rotation
//    from the fresh entry and the post-rotation diagonal -- so one barrier per
//    round; the rotation itself is fp32 (angle) + fp64 renormalisation of
//    (c, s) with the exact fp64 similarity update of the pair's 2x2 block.
//  * The eigenvector matrix U is accumulated off the critical path by the
//    other CTAs of the cluster (row blocks of U): every rotation is pushed to
//    them with st.async into a ring of per-round slots (mbarrier complete_tx);
//    they trail CTA 0 by a few rounds, with a progress counter for back-pressure.
//  * Stop: after the sweep whose largest pre-rotation |g_pq|/sqrt(g_pp g_qq)
//    was below 1e-8 (quadratic convergence leaves ~1e-16 after it).
//  * Finish: sort, truncation rank (reference _truncation_rank, tt.py:203-211,
//    with the cap) and a certificate: the rank decision must hold with every
//    tail moved by the Gram error bound, the kept eigenvalues must be
//    >= 1e-3 of the largest (the new core's rows are orthonormal to ~1e-11),
//    and the sweep loop must have converged.  Callers fall back to the QR +
//    one-sided Jacobi SVD path when it does not hold (solver roundings whose
//    tolerance cuts into the noise floor, rank-deficient unfoldings).
//
// Accuracy: eigenvalues of the Gram carry absolute error ~eps ||C||^2, i.e. the
// singular values eps ||C||^2 / sigma -- irrelevant for the kept directions
// under the certificate, and the tails are compared with that error included.
#include "common.cuh"
#include "qr.cuh"
#include "../../include/ttk_b200.h"

#include <cooperative_groups.h>

namespace ttk {

namespace {

constexpr int kEigMaxN = 128;
constexpr int kEigThreads = 256;
constexpr int kEigUCtas = 3;        // U-accumulating CTAs per cluster
constexpr int kEigCluster = 1 + kEigUCtas;
constexpr int kEigRing = 32;        // rotation slots per U CTA
constexpr int kEigMaxH = kEigMaxN / 2;
constexpr int kEigMaxSweeps = 30;

__device__ __forceinline__ int eig_ld(int np) { return ((np + 15) & ~15) + 1; }

// player at position pos (circle method; position 0 fixed), round offset toff
__device__ __forceinline__ int eig_player(int pos, int toff, int np) {
  if (pos == 0) return 0;
  const int x = pos + toff;
  return x > np - 1 ? x - (np - 1) : x;
}

// CTA-0 area: G (np x ld), dn [2][kEigMaxN], rb [2][kEigMaxH] double2, lam, order, misc, then
// ps [2][kEigMaxH] double4 and the bulk item table
__host__ __device__ constexpr size_t eig_ps_off(int np, int ld) {
  return (((size_t)np * ld * 8 + 2 * 128 * 8 + 2 * 64 * 16 + 128 * 8 + 128 * 4 + 64) + 31) / 32 * 32;
}

__device__ __forceinline__ int tri(int i, int j, int ld) { return i < j ? i * ld + j : j * ld + i; }

__device__ __forceinline__ uint32_t eig_map(uint32_t a, int rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(rank));
  return r;
}
__device__ __forceinline__ void eig_st_v2(uint32_t addr, double a, double b, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::"r"(addr),
               "d"(a), "d"(b), "r"(bar)
               : "memory");
}
__device__ __forceinline__ void eig_st_u32(uint32_t addr, uint32_t v, uint32_t bar) {
  asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b32 [%0], %1, [%2];" ::"r"(addr), "r"(v),
               "r"(bar)
               : "memory");
}
__device__ __forceinline__ void eig_arm(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
// bounded wait (a lost hand-off must not hang the device): false after ~1 s
__device__ __forceinline__ bool eig_wait(uint32_t bar, uint32_t parity) {
  uint32_t done;
  long long spins = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 p, [%1], %2;\n"
        " selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!done && ++spins < (1LL << 22));
  return done != 0;
}
// Jacobi rotation of the symmetric pair block [[a, g], [g, b]], J = [[c, s], [-s, c]]
// (J^T M J diagonal): the angle in fp32 (G is prescaled so its largest diagonal
// lies in [1, 2); a pair too small for fp32 takes the rescaled path), then
// (c, s) renormalised in fp64 to c^2 + s^2 = 1 + O(1e-20).  rotate = false
// gives the identity.  Branch-free on the common path.
__device__ __forceinline__ double2 eig_rot_cs(double a, double b, double g, bool rotate) {
  double d = b - a, h = g;
  float df = (float)d, hf = (float)h;
  float x = fmaf(df, df, 4.f * hf * hf);
  if (rotate && !(x >= 1e-30f)) {  // rare: rescale the pair by a power of two
    const double m = fmax(fabs(d), 2.0 * fabs(h));
    const long long ex = (__double_as_longlong(m) >> 52) & 0x7ff;
    const double sc = (ex > 0 && ex < 2046) ? __longlong_as_double((2046LL - ex) << 52) : 0.0;
    df = (float)(d * sc);
    hf = (float)(h * sc);
    x = fmaf(df, df, 4.f * hf * hf);
  }
  const float den = fabsf(df) + x * rsqrtf(x);
  float t = __fdividef(2.f * hf, den);
  t = df < 0.f ? -t : t;
  t = (rotate && isfinite(t)) ? t : 0.f;
  const float c32 = rsqrtf(fmaf(t, t, 1.f));
  const double c = (double)c32, s = (double)(t * c32);
  const double e = fma(c, c, fma(s, s, -1.0));
  const double f = fma(e, fma(e, 0.375, -0.5), 1.0);
  return make_double2(c * f, s * f);
}
// diagonal entry after rotating the pair block st = (a, b, g): p side (J^T M J)_00
// or q side (J^T M J)_11
__device__ __forceinline__ double eig_rot_diag(const double4& st, const double2& r, bool qside) {
  const double cc = r.x * r.x, ss = r.y * r.y, cs2 = 2.0 * r.x * r.y;
  return qside ? fma(ss, st.x, fma(cs2, st.z, cc * st.y)) : fma(cc, st.x, fma(-cs2, st.z, ss * st.y));
}
// off-diagonal entry after the rotation: cs (a - b) + (c^2 - s^2) g
__device__ __forceinline__ double eig_rot_offdiag(const double4& st, const double2& r) {
  return fma(r.x * r.y, st.x - st.y, (r.x * r.x - r.y * r.y) * st.z);
}

struct EigParams {
  int n;
  const double* G;   // n x n symmetric (upper triangle read), G[i*ldg + j]
  int ldg;
  double budget;     // truncation budget (absolute, on singular values)
  int cap;           // max rank (<= 0: none)
  double* S;         // n singular values sqrt(lambda), sorted descending
  double* T1;        // n x r: U_r S_r^{-1}  (ld ldo)
  double* L;         // n x r: U_r S_r       (ld ldo)
  int ldo;
  double* U;         // optional n x n sorted eigenvectors (ld n)
  int* trace;        // diagnostics: milestones into mapped host memory (or null)
  int dbg;           // test bisection: 1 = no hand-offs at all, 2 = pushes but U CTAs do not wait
  int* info;         // [r, certified, sweeps, converged, (diagnostics: 4 back-pressure, 5.. U-CTA waits)]
};

// shared-memory layout common to every CTA of the cluster (mapa needs equal offsets)
struct EigCommon {
  unsigned long long mbar[kEigRing];   // U CTAs: one per ring slot
  uint32_t uprog[kEigUCtas];           // CTA 0: rounds consumed by each U CTA (pushed by them)
  uint32_t flag[kEigRing];             // U CTAs: "last round" flag per slot
  double2 ring[kEigRing][kEigMaxH];    // U CTAs: (c, s) per pair per slot
};

constexpr int kEigRotThreads = 64;                            // warps 0-1: one thread per next-round pair
constexpr int kEigBulkThreads = kEigThreads - kEigRotThreads;  // warps 2-7: the other blocks
constexpr int kEigMaxBulk = (kEigMaxH * (kEigMaxH - 3) / 2 + kEigBulkThreads - 1) / kEigBulkThreads;  // 11
constexpr int kEigCtl = kEigRotThreads;                       // control thread (flags, back-pressure)

__device__ __forceinline__ uint32_t eig_ld_acquire(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.acquire.cluster.shared::cluster.u32 %0, [%1];" : "=r"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void eig_st_release_remote(uint32_t addr, uint32_t v) {
  asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

// rotate block (al, be) of the round with offset toff from both sides; returns the
// four new entries and their triangle offsets
struct EigBlock {
  int i00, i01, i10, i11;
  double z00, z01, z10, z11;
  int pa, qa, pb, qb;
};
__device__ __forceinline__ void eig_block(const double* G, const double2* rot, int code, int toff, int np, int ld,
                                          EigBlock& B) {
  const int al = code & 0xff, be = code >> 8;
  B.pa = eig_player(al, toff, np);
  B.qa = eig_player(np - 1 - al, toff, np);
  B.pb = eig_player(be, toff, np);
  B.qb = eig_player(np - 1 - be, toff, np);
  B.i00 = tri(B.pa, B.pb, ld);
  B.i01 = tri(B.pa, B.qb, ld);
  B.i10 = tri(B.qa, B.pb, ld);
  B.i11 = tri(B.qa, B.qb, ld);
  const double x00 = G[B.i00], x01 = G[B.i01], x10 = G[B.i10], x11 = G[B.i11];
  const double2 ra = rot[al], rb = rot[be];
  // rows: J_a^T ; columns: J_b   (J = [[c, s], [-s, c]])
  const double y00 = fma(ra.x, x00, -ra.y * x10), y01 = fma(ra.x, x01, -ra.y * x11);
  const double y10 = fma(ra.y, x00, ra.x * x10), y11 = fma(ra.y, x01, ra.x * x11);
  B.z00 = fma(rb.x, y00, -rb.y * y01);
  B.z01 = fma(rb.y, y00, rb.x * y01);
  B.z10 = fma(rb.x, y10, -rb.y * y11);
  B.z11 = fma(rb.y, y10, rb.x * y11);
}

__device__ __forceinline__ void eig_trace(int* tr, int i, int v) {
  if (tr) {
    *(volatile int*)(tr + i) = v;
    __threadfence_system();
  }
}

__global__ void __cluster_dims__(kEigCluster, 1, 1) __launch_bounds__(kEigThreads, 1)
    gram_eig_kernel(const __grid_constant__ EigParams P) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int crank = (int)cl.block_rank();
  extern __shared__ __align__(16) unsigned char eig_smem[];
  EigCommon& cm = *reinterpret_cast<EigCommon*>(eig_smem);
  unsigned char* area = eig_smem + ((sizeof(EigCommon) + 255) & ~size_t(255));

  const int n = P.n, np = n + (n & 1), h = np / 2, ld = eig_ld(np);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t slot_bytes = (uint32_t)(h * 16 + 4);

  // CTA-0 area
  double* G = reinterpret_cast<double*>(area);                 // np * ld (strict upper triangle used)
  double* dn = G + (size_t)np * ld;                              // [2][kEigMaxN] diagonal
  double2* rb = reinterpret_cast<double2*>(dn + 2 * kEigMaxN);   // [2][kEigMaxH] rotations
  double* lam = reinterpret_cast<double*>(rb + 2 * kEigMaxH);    // sorted eigenvalues (unscaled)
  int* order = reinterpret_cast<int*>(lam + kEigMaxN);           // sorted -> player
  int* misc = order + kEigMaxN;                                   // [0..1] sweep "unconverged" flags, [2] r
  __shared__ unsigned long long red_u;

  if (crank == 0) {
    // ---- load G (scaled by 2^-e so the largest diagonal lies in [1, 2)) ----
    if (tid == 0) red_u = 0ull;
    if (tid < 4) misc[tid] = 0;
    if (tid < kEigUCtas) cm.uprog[tid] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += kEigThreads) {
      const double v = P.G[(size_t)i * P.ldg + i];
      if (v > 0.0) atomicMax(&red_u, (unsigned long long)__double_as_longlong(v));
    }
    __syncthreads();
    const double gmax = __longlong_as_double((long long)red_u);
    long long gex = gmax > 0.0 ? ((__double_as_longlong(gmax) >> 52) & 0x7ff) : 1023;
    if (gex == 0 || gex >= 2046) gex = 1023;
    const double scale = __longlong_as_double((2046LL - gex) << 52);
    const double unscale = __longlong_as_double(gex << 52);
    for (int i = warp; i < np; i += kEigThreads / 32)
      for (int j = lane; j < np; j += 32) {
        const double v = (i < n && j < n) ? P.G[(size_t)i * P.ldg + j] * scale : 0.0;
        if (i < j) G[i * ld + j] = v;
        else if (i == j) dn[i] = v;  // dn[0] = G^(0) diagonal
      }
    if (tid == 0) eig_trace(P.trace, 0, 1);
    cl.sync();  // U CTAs have initialised their mbarriers
    if (tid == 0) eig_trace(P.trace, 0, 2);

    // remote addresses of the U CTAs' rings / barriers / flags; own progress slots
    uint32_t ring_r[kEigUCtas], bar_r[kEigUCtas], flag_r[kEigUCtas], prog_l[kEigUCtas];
#pragma unroll
    for (int u = 0; u < kEigUCtas; ++u) {
      ring_r[u] = eig_map(smem_u32(&cm.ring[0][0]), u + 1);
      bar_r[u] = eig_map(smem_u32(&cm.mbar[0]), u + 1);
      flag_r[u] = eig_map(smem_u32(&cm.flag[0]), u + 1);
      prog_l[u] = eig_map(smem_u32(&cm.uprog[u]), 0);
    }
    auto push_rot = [&](int round, int a, double c, double s) {
      if (P.dbg == 1) return;
      const int slot = round % kEigRing;
#pragma unroll
      for (int u = 0; u < kEigUCtas; ++u)
        eig_st_v2(ring_r[u] + (uint32_t)((slot * kEigMaxH + a) * 16), c, s, bar_r[u] + (uint32_t)(slot * 8));
    };
    const double tol2 = 1e-30, stop2 = 1e-16, tiny = 1e-36;
    // Rotation of the pair block [[a, g], [g, b]] (only (c, s); the rotated
    // block itself is recomputed where it is needed, off this chain).
    auto pair_rotation = [&](double a, double b, double g, int sweep_of) -> double2 {
      const double hh = g * g, ab = a * b;
      if (hh > stop2 * ab && ab > tiny) misc[sweep_of & 1] = 1;
      return eig_rot_cs(a, b, g, hh > tol2 * ab);
    };
    double4* ps = reinterpret_cast<double4*>(area + eig_ps_off(np, ld));  // [2][kEigMaxH] (a, b, g) per pair
    unsigned short* itab = reinterpret_cast<unsigned short*>(ps + 2 * kEigMaxH);  // [kEigMaxBulk][bulk threads]

    // ---- prologue: rotations of round 0 (pairs (a, np-1-a)) ----
    double4 myps = make_double4(0, 0, 0, 0);  // state of my pair of the current round (deferred g write)
    double2 myrot = make_double2(1.0, 0.0);
    if (tid < h) {
      const int p = tid, q = np - 1 - tid;
      myps = make_double4(dn[p], dn[q], G[tri(p, q, ld)], 0.0);
      myrot = pair_rotation(myps.x, myps.y, myps.z, 0);
      rb[tid] = myrot;
      ps[tid] = myps;
      push_rot(0, tid, myrot.x, myrot.y);
    }
    if (tid == 0) eig_trace(P.trace, 0, 3);

    // Thread a' < h (warps 0-1) owns the block holding next-round pair a':
    // (0,1), (a'-1, a'+1), (h-2, h-1).  The other blocks go to warps 2-7 in
    // row-major order of the strict upper triangle minus those (row 0 loses
    // (0,1), (0,2); rows 1..h-3 lose (a, a+2); row h-2 is empty), so a warp's
    // lanes mostly share a row and walk consecutive columns (conflict-free);
    // the per-thread lists live in shared memory (small loop body).
    int al_d = 0, be_d = 0, kind = 0;  // kind: 0 = (q_a, p_b) [be = al+2], 1 = (p_a, p_b), 2 = (q_a, q_b)
    if (tid < h) {
      al_d = tid == 0 ? 0 : (tid == h - 1 ? h - 2 : tid - 1);
      be_d = tid == 0 ? 1 : (tid == h - 1 ? h - 1 : tid + 1);
      kind = (be_d == al_d + 2) ? 0 : (tid == 0 ? 1 : 2);
    }
    int nbulk = 0;
    if (tid >= kEigRotThreads) {
      const int bt = tid - kEigRotThreads;
      const int nb = h * (h - 1) / 2 - h;
      int al = 0, off = 0;
      auto row_len = [&](int r) { return r == 0 ? h - 3 : (r <= h - 3 ? h - 2 - r : 0); };
      for (int k = bt; k < nb; k += kEigBulkThreads) {
        while (off + row_len(al) <= k) { off += row_len(al); ++al; }
        const int idx = k - off;
        const int be = al == 0 ? 3 + idx : al + 1 + idx + (idx >= 1 ? 1 : 0);
        itab[nbulk * kEigBulkThreads + bt] = (unsigned short)(al | (be << 8));
        ++nbulk;
      }
    }
    __syncthreads();
    if (tid == 0) eig_trace(P.trace, 0, 4);

    // ---- main loop: one barrier per round ----
    int toff = 0, sweep = 0, stop = 0, conv = 0;
    int it = 0;
    const bool prof = P.dbg == 3 && tid == 5;
    long long ph[6] = {0, 0, 0, 0, 0, 0}, tc = clock64();
    auto mark = [&](int k) {
      if (prof) {
        const long long t = clock64();
        ph[k] += t - tc;
        tc = t;
      }
    };
    for (;; ++it) {
      const int cur = it & 1, nxt = cur ^ 1;
      const double2* rcur = rb + cur * kEigMaxH;
      const bool last_of_sweep = (toff == np - 2);
      if (last_of_sweep) {
        conv = misc[sweep & 1] == 0;
        stop = conv || (sweep + 1 >= kEigMaxSweeps);
      }
      const int toffn = (toff + 1 == np - 1) ? 0 : toff + 1;
      if (tid < h) {
        mark(0);
        // designated block of round it, then the rotation of its round-(it+1) pair
        EigBlock B;
        eig_block(G, rcur, al_d | (be_d << 8), toff, np, ld, B);
        // diagonal of the next pair after round it, from the pair states of round it
        const int sP = kind == 1 ? al_d : be_d, sQ = kind == 1 ? be_d : al_d;  // slots holding P', Q'
        const bool qP = kind == 2, qQ = kind != 1;                             // ... on their q side?
        const double4 psP = ps[cur * kEigMaxH + sP], psQ = ps[cur * kEigMaxH + sQ];
        const double2 rP = rcur[sP], rQ = rcur[sQ];
        const double aP = eig_rot_diag(psP, rP, qP), aQ = eig_rot_diag(psQ, rQ, qQ);
        const double g = kind == 0 ? B.z10 : (kind == 1 ? B.z00 : B.z11);
        mark(1);
        const double2 rot = pair_rotation(aP, aQ, g, toffn == 0 ? sweep + 1 : sweep);
        mark(2);
        rb[nxt * kEigMaxH + tid] = rot;
        ps[nxt * kEigMaxH + tid] = make_double4(aP, aQ, g, 0.0);
        push_rot(it + 1, tid, rot.x, rot.y);
        G[B.i00] = B.z00;
        G[B.i01] = B.z01;
        G[B.i10] = B.z10;
        G[B.i11] = B.z11;
        // deferred: rotated off-diagonal of my round-it pair (no one reads it this round)
        {
          const int p = eig_player(tid, toff, np), q = eig_player(np - 1 - tid, toff, np);
          G[tri(p, q, ld)] = eig_rot_offdiag(myps, myrot);
        }
        myps = make_double4(aP, aQ, g, 0.0);
        myrot = rot;
        mark(3);
      } else if (tid >= kEigRotThreads) {
        if (tid == kEigCtl) {
          if (toff == 0 && sweep >= 1) misc[(sweep + 1) & 1] = 0;
          if (P.dbg == 0) {
            const int slot = it % kEigRing;
#pragma unroll
            for (int u = 0; u < kEigUCtas; ++u)
              eig_st_u32(flag_r[u] + (uint32_t)(slot * 4), (uint32_t)stop, bar_r[u] + (uint32_t)(slot * 8));
            if ((it & 7) == 0) {  // back-pressure for the pushes of rounds it+1 .. it+8
              const int need = it + 10 - kEigRing;
#pragma unroll
              for (int u = 0; u < kEigUCtas; ++u) {
                long long spins = 0;
                while ((int)eig_ld_acquire(prog_l[u]) < need && ++spins < (1LL << 22)) {
                }
                if (spins >= (1LL << 22)) P.info[4] = 100 + it;  // diagnostics: back-pressure timeout
              }
            }
          }
        }
        // bulk blocks, two at a time (loads of both issued before either is stored)
        const int bt = tid - kEigRotThreads;
        for (int j = 0; j < nbulk; j += 2) {
          const int c0 = itab[j * kEigBulkThreads + bt];
          const bool two = j + 1 < nbulk;
          const int c1 = two ? itab[(j + 1) * kEigBulkThreads + bt] : c0;
          EigBlock B0, B1;
          eig_block(G, rcur, c0, toff, np, ld, B0);
          eig_block(G, rcur, c1, toff, np, ld, B1);
          G[B0.i00] = B0.z00;
          G[B0.i01] = B0.z01;
          G[B0.i10] = B0.z10;
          G[B0.i11] = B0.z11;
          if (two) {
            G[B1.i00] = B1.z00;
            G[B1.i01] = B1.z01;
            G[B1.i10] = B1.z10;
            G[B1.i11] = B1.z11;
          }
        }
      }
      __syncthreads();
      mark(4);
      if (tid == 0) { eig_trace(P.trace, 1, it); eig_trace(P.trace, 2, sweep); }
      if (last_of_sweep) ++sweep;
      toff = toffn;
      if (stop) break;
    }
    if (prof)
      for (int k = 0; k < 5; ++k) P.info[8 + k] = (int)(ph[k] / (it + 1));
    // diagonal after the last applied round `it`: from the pair states of that round
    double* dfin = dn;
    {
      const int cur = it & 1;
      for (int a = tid; a < h; a += kEigThreads) {
        const int tf = toff == 0 ? np - 2 : toff - 1;  // offset of round `it`
        const int p = eig_player(a, tf, np), q = eig_player(np - 1 - a, tf, np);
        const double4 st = ps[cur * kEigMaxH + a];
        const double2 rt = rb[cur * kEigMaxH + a];
        dfin[p] = eig_rot_diag(st, rt, false);
        dfin[q] = eig_rot_diag(st, rt, true);
      }
    }
    __syncthreads();
    if (tid == 0) eig_trace(P.trace, 0, 5);

    // ---- sort (descending), rank, certificate ----
    for (int j = tid; j < n; j += kEigThreads) {
      const double v = dfin[j];
      int rk = 0;
      for (int i = 0; i < n; ++i) {
        const double w = dfin[i];
        rk += (w > v) || (w == v && i < j);
      }
      order[rk] = j;
    }
    __syncthreads();
    for (int c = tid; c < n; c += kEigThreads) {
      const double v = fmax(dfin[order[c]], 0.0);
      lam[c] = v * unscale;
      P.S[c] = sqrt(v * unscale);
    }
    __syncthreads();
    if (tid < 32) {
      // suffix sums over the sorted eigenvalues (scaled), `per` per lane
      const int per = (n + 31) / 32;
      double loc = 0.0;
      for (int i = min(n, (tid + 1) * per) - 1; i >= tid * per; --i) loc += fmax(dfin[order[i]], 0.0);
      double suf = loc;  // inclusive suffix over lanes >= tid
      for (int o = 1; o < 32; o <<= 1) {
        const double v = __shfl_down_sync(0xffffffffu, suf, o);
        if (tid + o < 32) suf += v;
      }
      const double trace = __shfl_sync(0xffffffffu, suf, 0);
      const double b2 = P.budget * P.budget * scale;  // budget^2 in scaled units
      // first index r with tail(r) <= b2 inside my range
      int rfirst = n;
      double tail = suf;  // tail at the start of my range
      for (int i = tid * per; i < min(n, (tid + 1) * per); ++i) {
        if (tail <= b2) { rfirst = i; break; }
        tail -= fmax(dfin[order[i]], 0.0);
      }
      for (int o = 16; o >= 1; o >>= 1) rfirst = min(rfirst, __shfl_xor_sync(0xffffffffu, rfirst, o));
      if (tid == 0) {
        int r = max(rfirst, 1);
        const int capr = (P.cap > 0) ? min(P.cap, n) : n;
        r = min(r, capr);
        double t_rm1 = 0.0, t_r = 0.0;  // tails at r-1 and r
        for (int i = n - 1; i >= r - 1 && i >= 0; --i) {
          const double v = fmax(dfin[order[i]], 0.0);
          if (i >= r) t_r += v;
          t_rm1 += v;
        }
        const double E = 1e-11 * trace;  // >> the Gram's rounding error on any tail
        bool cert = conv != 0;
        if (r >= 2) cert = cert && (t_rm1 - E > b2);
        if (r < capr && r < n) cert = cert && (t_r + E <= b2);
        const double lr = fmax(dfin[order[r - 1]], 0.0), l0 = fmax(dfin[order[0]], 0.0);
        cert = cert && (lr >= 1e-3 * l0) && (l0 > 0.0);
        misc[2] = r;
        P.info[0] = r;
        P.info[1] = cert ? 1 : 0;
        P.info[2] = sweep;
        P.info[3] = conv;
      }
    }
    if (tid == 0) eig_trace(P.trace, 0, 6);
    cl.sync();  // publish order / lam / r to the U CTAs
    cl.sync();  // they have read them
    if (tid == 0) eig_trace(P.trace, 0, 8);
  } else {
    // ---------------- U CTAs: rows [r0, r1) of U, one row per warp at a time ----------------
    const int u = crank - 1;
    const int rpc = (n + kEigUCtas - 1) / kEigUCtas;
    const int r0 = u * rpc, r1 = min(n, r0 + rpc), nrows = max(0, r1 - r0);
    double* Uloc = reinterpret_cast<double*>(area);  // nrows x ld
    for (int i = warp; i < nrows; i += kEigThreads / 32)
      for (int j = lane; j < ld; j += 32) Uloc[i * ld + j] = (j == r0 + i) ? 1.0 : 0.0;
    if (tid == 0) {
      for (int s = 0; s < kEigRing; ++s)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&cm.mbar[s])) : "memory");
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      for (int s = 0; s < kEigRing; ++s) eig_arm(smem_u32(&cm.mbar[s]), slot_bytes);
    }
    __syncthreads();
    if (tid == 0) eig_trace(P.trace, 3 + u, 1);
    cl.sync();
    if (tid == 0) eig_trace(P.trace, 3 + u, 2);
    const uint32_t prog_r = eig_map(smem_u32(&cm.uprog[u]), 0);
    const int a0 = lane, a1 = lane + 32;
    int toff = 0;
    for (int it = 0; P.dbg == 0; ++it) {
      const int slot = it % kEigRing;
      const bool got = eig_wait(smem_u32(&cm.mbar[slot]), (uint32_t)((it / kEigRing) & 1));
      const uint32_t fl = got ? cm.flag[slot] : 1u;
      if (!got && tid == 0) P.info[5 + u] = it + 1;  // diagnostics: lost hand-off at round it
      const double2 t0 = a0 < h ? cm.ring[slot][a0] : make_double2(1.0, 0.0);
      const double2 t1 = a1 < h ? cm.ring[slot][a1] : make_double2(1.0, 0.0);
      const int p0 = eig_player(a0, toff, np), q0 = eig_player(np - 1 - a0, toff, np);
      const int p1 = eig_player(a1 < h ? a1 : a0, toff, np), q1 = eig_player(np - 1 - (a1 < h ? a1 : a0), toff, np);
      for (int i = warp; i < nrows; i += kEigThreads / 32) {
        double* row = Uloc + i * ld;
        if (a0 < h && t0.y != 0.0) {
          const double up = row[p0], uq = row[q0];
          row[p0] = fma(t0.x, up, -t0.y * uq);
          row[q0] = fma(t0.y, up, t0.x * uq);
        }
        if (a1 < h && t1.y != 0.0) {
          const double up = row[p1], uq = row[q1];
          row[p1] = fma(t1.x, up, -t1.y * uq);
          row[q1] = fma(t1.y, up, t1.x * uq);
        }
      }
      __syncthreads();
      if (tid == 0) {
        eig_arm(smem_u32(&cm.mbar[slot]), slot_bytes);
        eig_st_release_remote(prog_r, (uint32_t)(it + 1));
        eig_trace(P.trace, 8 + u, it + 1);
      }
      toff = (toff + 1 == np - 1) ? 0 : toff + 1;
      if (fl) break;
    }
    if (tid == 0) eig_trace(P.trace, 3 + u, 3);
    cl.sync();  // CTA 0 has published order / lam / r
    if (tid == 0) eig_trace(P.trace, 3 + u, 4);
    // local copies of the permutation and eigenvalues (one DSMEM read each)
    int* ordl = reinterpret_cast<int*>(Uloc + (size_t)rpc * ld);
    double* laml = reinterpret_cast<double*>(ordl + kEigMaxN);
    const int* ord0 = cl.map_shared_rank(order, 0);
    const double* lam0 = cl.map_shared_rank(lam, 0);
    const int r = *cl.map_shared_rank(misc + 2, 0);
    for (int c = tid; c < n; c += kEigThreads) {
      ordl[c] = ord0[c];
      laml[c] = lam0[c];
    }
    __syncthreads();
    for (int i = warp; i < nrows; i += kEigThreads / 32)
      for (int c = lane; c < n; c += 32) {
        const double v = Uloc[i * ld + ordl[c]];
        if (P.U) P.U[(size_t)(r0 + i) * n + c] = v;
        if (c < r) {
          const double l = laml[c];
          const double sg = sqrt(l);
          P.T1[(size_t)(r0 + i) * P.ldo + c] = l > 0.0 ? v / sg : 0.0;
          P.L[(size_t)(r0 + i) * P.ldo + c] = v * sg;
        }
      }
    cl.sync();
  }
}

size_t eig_smem_bytes(int n) {
  const int np = n + (n & 1), ld = ((np + 15) & ~15) + 1;
  const size_t common = (sizeof(EigCommon) + 255) & ~size_t(255);
  const size_t cta0 = eig_ps_off(np, ld) + 2 * kEigMaxH * 32 + (size_t)kEigMaxBulk * kEigBulkThreads * 2;
  const int rpc = (n + kEigUCtas - 1) / kEigUCtas;
  const size_t ucta = (size_t)rpc * ld * 8 + kEigMaxN * 12 + 64;
  return common + (cta0 > ucta ? cta0 : ucta);
}

}  // namespace

int* g_eig_trace = nullptr;
int g_eig_dbg = 0;  // test bisection only (ttk_debug_gram_eig)

bool gram_eig_supported(int n) { return n >= 6 && n <= kEigMaxN; }

int gram_eig(int n, const double* G, int ldg, double budget, int cap, double* S, double* T1, double* L, int ldo,
             double* U, int* info, cudaStream_t st) {
  TTK_REQUIRE(gram_eig_supported(n), kInvalidValue, "gram_eig: n = %d outside [6, %d]", n, kEigMaxN);
  TTK_REQUIRE(ldo >= n && ldg >= n, kInvalidValue, "gram_eig: bad leading dimensions");
  const size_t smem = eig_smem_bytes(n);
  TTK_TRY(set_attr_once(gram_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)eig_smem_bytes(kEigMaxN)));
  EigParams p{n, G, ldg, budget, cap, S, T1, L, ldo, U, g_eig_trace, g_eig_dbg, info};
  gram_eig_kernel<<<kEigCluster, kEigThreads, smem, st>>>(p);
  TTK_CHECK_LAUNCH();
  return kOk;
}

}  // namespace ttk

using namespace ttk;

extern "C" {

// Symmetric eigendecomposition of a Gram matrix G (n x n, device, ld ldg) with
// the truncation decision of the reference's TT-SVD step (tt.py:203-211, 358-367):
// S = sqrt(eigenvalues) descending, T1 = U_r S_r^{-1}, L = U_r S_r (n x r, ld ldo),
// optional U (n x n sorted eigenvectors), info = [r, certified, sweeps, converged]
// (device ints).  Asynchronous on `stream`.
int ttk_debug_gram_eig(int mode, int* trace) {
  g_eig_dbg = mode;
  g_eig_trace = trace;
  return 0;
}

int ttk_gram_eig(int n, const double* G, int ldg, double budget, int max_rank, double* S, double* T1,
                 double* L, int ldo, double* U, int* info, void* stream) {
  return gram_eig(n, G, ldg, budget, max_rank, S, T1, L, ldo, U, info, (cudaStream_t)stream);
}

}  // extern "C"
