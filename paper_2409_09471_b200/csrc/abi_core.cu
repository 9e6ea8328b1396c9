// C-ABI entry points: library info, error channel, grouped GEMM, TT matvec.
#include "gemm.cuh"
#include "../../include/ttk_b200.h"

#include <chrono>
#include <mutex>
#include <set>
#include <tuple>
#include <cstdlib>
#include <string>
#include <vector>

namespace ttk {

static thread_local char g_err[1024] = {0};
std::atomic<long long> g_launches{0};

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

const char* last_error() { return g_err; }

namespace {
std::mutex g_attr_mu;
std::set<std::tuple<int, const void*, int>> g_attr_done;
int g_sms[64] = {0};
}  // namespace

int num_sms() {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return kNumSMs;
  if (g_sms[dev] == 0) {
    int n = kNumSMs;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = kNumSMs;
    g_sms[dev] = n;  // benign race: every writer stores the same value
  }
  return g_sms[dev];
}

int scratch_alloc(void** p, size_t bytes, cudaStream_t st) {
  static bool pool_set[64] = {false};
  int dev = 0;
  TTK_CHECK_CUDA(cudaGetDevice(&dev));
  if (dev >= 0 && dev < 64 && !pool_set[dev]) {
    std::lock_guard<std::mutex> lock(g_attr_mu);
    if (!pool_set[dev]) {
      cudaMemPool_t pool;
      TTK_CHECK_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
      unsigned long long thr = ~0ULL;
      TTK_CHECK_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
      pool_set[dev] = true;
    }
  }
  TTK_CHECK_CUDA(cudaMallocAsync(p, bytes, st));
  return kOk;
}

int scratch_free(void* p, cudaStream_t st) {
  TTK_CHECK_CUDA(cudaFreeAsync(p, st));
  return kOk;
}

int set_attr_once(const void* fn, cudaFuncAttribute attr, int value) {
  int dev = 0;
  TTK_CHECK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(g_attr_mu);
  const auto key = std::make_tuple(dev, fn, (int)attr);
  if (g_attr_done.count(key)) return kOk;
  TTK_CHECK_CUDA(cudaFuncSetAttribute(fn, attr, value));
  g_attr_done.insert(key);
  return kOk;
}

static const bool g_host_prof = knob_env("TTK_HOST_PROF") != nullptr;
std::atomic<long long> g_syncs{0}, g_sync_ns{0};

int host_sync(cudaStream_t st) {
  if (!g_host_prof) {
    TTK_CHECK_CUDA(cudaStreamSynchronize(st));
    return kOk;
  }
  const auto t0 = std::chrono::steady_clock::now();
  TTK_CHECK_CUDA(cudaStreamSynchronize(st));
  g_sync_ns += std::chrono::duration_cast<std::chrono::nanoseconds>(std::chrono::steady_clock::now() - t0).count();
  ++g_syncs;
  return kOk;
}

}  // namespace ttk

using namespace ttk;

extern "C" {

const char* ttk_last_error(void) { return ttk::last_error(); }

int ttk_version(void) { return TTK_ABI_VERSION; }

long long ttk_launch_count(void) { return ttk::g_launches.load(); }

int ttk_debug_host_profile(long long* out) {
  out[0] = ttk::g_syncs.load();
  out[1] = ttk::g_sync_ns.load();
  return 0;
}

int ttk_device_arch(void) {
  int dev = 0, major = 0, minor = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return -1;
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(&minor, cudaDevAttrComputeCapabilityMinor, dev);
  return major * 10 + minor;
}

int ttk_gemm_strided(int batch, int M, int N, int K, double alpha, const double* A,
                     long long a_ms, long long a_ks, long long a_bs, const double* B,
                     long long b_ks, long long b_ns, long long b_bs, double beta, double* C,
                     long long c_ms, long long c_ns, long long c_bs, void* ws, size_t ws_bytes,
                     void* stream) {
  TTK_REQUIRE(batch >= 0 && M >= 0 && N >= 0 && K >= 0, kInvalidValue, "negative GEMM size");
  if (batch == 0 || M == 0 || N == 0) return kOk;
  std::vector<GemmProblem> probs(batch);
  for (int b = 0; b < batch; ++b)
    probs[b] = make_gemm(M, N, K, A + b * a_bs, a_ms, a_ks, B + b * b_bs, b_ks, b_ns, C + b * c_bs,
                         c_ms, c_ns, alpha, beta);
  return gemm_group_launch(probs.data(), batch, ws, ws_bytes, (cudaStream_t)stream);
}

size_t ttk_gemm_strided_ws_bytes(int batch, int M, int N, int K) {
  if (batch <= 0 || M <= 0 || N <= 0) return 0;
  std::vector<GemmProblem> probs(batch);
  for (int b = 0; b < batch; ++b)
    probs[b] = make_gemm(M, N, K, nullptr, 1, 1, nullptr, 1, 1, nullptr, 1, 1);
  return gemm_group_ws_bytes(probs.data(), batch);
}

// tt_matvec: G_k[(a*rho0+al), i, (b*rho1+be)] = sum_j D_k[al,i,j,be] * C_k[a,j,b]
// Reference: ttkrylov/tt.py:302-314 (tensordot over j, transpose (0,2,3,1,4),
// reshape to (r0*rho0, m, r1*rho1): vector-rank major, operator-rank minor).
int ttk_matvec_range(int d, const int* rho, const int* m, const int* n, const int* r,
                     const double* const* D, const double* const* C, double* const* G, int k0, int k1,
                     void* stream) {
  TTK_REQUIRE(d >= 1, kInvalidValue, "d must be >= 1");
  TTK_REQUIRE(rho[0] == 1 && rho[d] == 1 && r[0] == 1 && r[d] == 1, kShapeMismatch,
              "boundary ranks must equal 1");
  TTK_REQUIRE(0 <= k0 && k0 <= k1 && k1 <= d, kInvalidValue, "core range [%d, %d) outside [0, %d)", k0, k1, d);
  std::vector<GemmProblem> probs;
  probs.reserve(64);
  for (int k = k0; k < k1; ++k) {
    const int r0 = r[k], r1 = r[k + 1], p0 = rho[k], p1 = rho[k + 1];
    const int mk = m[k], nk = n[k];
    TTK_REQUIRE(r0 >= 0 && r1 >= 0 && p0 >= 1 && p1 >= 1 && mk >= 1 && nk >= 1, kShapeMismatch,
                "bad shapes at core %d", k);
    if (r0 == 0 || r1 == 0) continue;
    const long long rr1 = (long long)r1 * p1;
    for (int al = 0; al < p0; ++al) {
      GemmProblem p{};
      // rows  (a,b)   : A(p,j) = C[a, j, b]
      // cols  (i,be)  : B(j,q) = D[al, i, j, be]
      p.M = r0 * r1;
      p.N = mk * p1;
      p.K = nk;
      p.A = C[k];
      p.a_mdiv = r1; p.a_ms1 = (long long)nk * r1; p.a_ms0 = 1; p.a_ks = r1;
      p.B = D[k] + (long long)al * mk * nk * p1;
      p.b_ndiv = p1; p.b_ns1 = (long long)nk * p1; p.b_ns0 = 1; p.b_ks = p1;
      p.C = G[k] + (long long)al * mk * rr1;
      p.c_mdiv = r1; p.c_ms1 = (long long)p0 * mk * rr1; p.c_ms0 = p1;
      p.c_ndiv = p1; p.c_ns1 = rr1; p.c_ns0 = 1;
      p.alpha = 1.0; p.beta = 0.0; p.splits = 1;
      probs.push_back(p);
    }
  }
  if (probs.empty()) return kOk;
  return gemm_group_launch(probs.data(), (int)probs.size(), nullptr, 0, (cudaStream_t)stream,
                           /*allow_split=*/false);
}

int ttk_matvec(int d, const int* rho, const int* m, const int* n, const int* r,
               const double* const* D, const double* const* C, double* const* G, void* stream) {
  return ttk_matvec_range(d, rho, m, n, r, D, C, G, 0, d, stream);
}

// mode_multiply for nterms matrix lists sharing one TT (the exp-sum terms):
// O_{t,k}[a, i, b] = s_{t,k} * sum_j M_{t,k}[i, j] * X_k[a, j, b], s = alpha[t] on
// the last core (tt_scale's convention), 1 elsewhere.  Reference:
// ttkrylov/precond.py:189-200 (tensordot over the mode index, transpose back)
// and the term scaling precond.py:270-272 / tt.py:278-282.  Every (term, core)
// product is one problem of a single grouped DMMA launch (rows (a,b), cols i).
int ttk_mode_multiply(int nterms, int d, const int* n, const int* m, const int* r, const double* alpha,
                      const double* const* mats, const double* const* X, double* const* out,
                      void* stream) {
  TTK_REQUIRE(nterms >= 0 && d >= 1, kInvalidValue, "need nterms >= 0 and d >= 1");
  TTK_REQUIRE(r[0] == 1 && r[d] == 1, kShapeMismatch, "boundary ranks must equal 1");
  std::vector<GemmProblem> probs;
  probs.reserve((size_t)nterms * d);
  for (int t = 0; t < nterms; ++t) {
    for (int k = 0; k < d; ++k) {
      const int r0 = r[k], r1 = r[k + 1], nk = n[k], mk = m[k];
      TTK_REQUIRE(r0 >= 0 && r1 >= 0 && nk >= 1 && mk >= 1, kShapeMismatch, "bad shapes at core %d", k);
      TTK_REQUIRE(mats[(size_t)t * d + k] != nullptr && out[(size_t)t * d + k] != nullptr, kInvalidValue,
                  "null matrix or output at term %d core %d", t, k);
      if (r0 == 0 || r1 == 0) continue;
      GemmProblem p{};
      p.M = r0 * r1;
      p.N = mk;
      p.K = nk;
      p.A = X[k];  // A((a,b), j) = X[a, j, b]
      p.a_mdiv = r1; p.a_ms1 = (long long)nk * r1; p.a_ms0 = 1; p.a_ks = r1;
      p.B = mats[(size_t)t * d + k];  // B(j, i) = M[i, j]
      p.b_ndiv = 1 << 30; p.b_ns1 = 0; p.b_ns0 = nk; p.b_ks = 1;
      p.C = out[(size_t)t * d + k];  // C((a,b), i) = O[a, i, b]
      p.c_mdiv = r1; p.c_ms1 = (long long)mk * r1; p.c_ms0 = 1;
      p.c_ndiv = 1 << 30; p.c_ns1 = 0; p.c_ns0 = r1;
      p.alpha = (alpha != nullptr && k == d - 1) ? alpha[t] : 1.0;
      p.beta = 0.0; p.splits = 1;
      probs.push_back(p);
    }
  }
  if (probs.empty()) return kOk;
  return gemm_group_launch(probs.data(), (int)probs.size(), nullptr, 0, (cudaStream_t)stream,
                           /*allow_split=*/false);
}

}  // extern "C"
