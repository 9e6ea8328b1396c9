// Shared device/host helpers for the TT-sGMRES B200 kernels (sm_100a, fp64).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdlib>
#include <cstdio>
#include <cstdarg>
#include <cmath>
#include <atomic>

namespace ttk {

// number of kernels this library has launched (ttk_launch_count); bumped by
// TTK_CHECK_LAUNCH, which follows every <<<...>>> launch site
extern std::atomic<long long> g_launches;

// ---------------------------------------------------------------------------
// error reporting: every extern "C" entry point returns 0 on success and a
// nonzero status otherwise; the message is kept per host thread.
enum Status : int {
  kOk = 0,
  kShapeMismatch = 1,   // maps to ShapeMismatch (ValueError) on the Python side
  kInvalidValue = 2,    // maps to ValueError
  kCudaError = 3,       // maps to RuntimeError
  kWorkspace = 4,       // caller-provided workspace too small
  kDegenerate = 5,      // DegenerateRecovery
};

void set_error(const char* fmt, ...);
const char* last_error();

#define TTK_CHECK_CUDA(expr)                                                     \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess) {                                                     \
      ::ttk::set_error("%s:%d: %s -> %s", __FILE__, __LINE__, #expr,            \
                       cudaGetErrorString(_e));                                  \
      return ::ttk::kCudaError;                                                  \
    }                                                                            \
  } while (0)

#define TTK_CHECK_LAUNCH()                                                       \
  do {                                                                           \
    ::ttk::g_launches.fetch_add(1, std::memory_order_relaxed);                   \
    cudaError_t _e = cudaGetLastError();                                         \
    if (_e != cudaSuccess) {                                                     \
      ::ttk::set_error("%s:%d: launch failed -> %s", __FILE__, __LINE__,        \
                       cudaGetErrorString(_e));                                  \
      return ::ttk::kCudaError;                                                  \
    }                                                                            \
  } while (0)

#define TTK_REQUIRE(cond, status, ...)                                           \
  do {                                                                           \
    if (!(cond)) {                                                               \
      ::ttk::set_error(__VA_ARGS__);                                             \
      return (status);                                                           \
    }                                                                            \
  } while (0)

#define TTK_TRY(expr)                                                            \
  do {                                                                           \
    int _s = (expr);                                                             \
    if (_s != ::ttk::kOk) return _s;                                             \
  } while (0)

// grid-size cap for grid-stride loops (B200: 148 SMs); residency decisions use num_sms()
constexpr int kNumSMs = 148;

// SM count of the current device (queried once per device)
int num_sms();

// Stream-ordered scratch (cudaMallocAsync / cudaFreeAsync on the device's
// default memory pool, whose release threshold is raised once per device so
// freed blocks stay cached instead of going back to the driver at every sync)
int scratch_alloc(void** p, size_t bytes, cudaStream_t st);
int scratch_free(void* p, cudaStream_t st);

// Kernel attributes are per device: set (fn, attr) = value once per device.
int set_attr_once(const void* fn, cudaFuncAttribute attr, int value);
template <class F>
inline int set_attr_once(F* fn, cudaFuncAttribute attr, int value) {
  return set_attr_once((const void*)fn, attr, value);
}

// Experiment / diagnostic knobs (A/B switches, tracing) are read from the
// environment only in builds with -DTTK_DEBUG_KNOBS; the shipped library
// ignores them, so no environment variable changes its numerics or control flow.
#ifdef TTK_DEBUG_KNOBS
inline const char* knob_env(const char* name) { return getenv(name); }
#else
inline const char* knob_env(const char*) { return nullptr; }
#endif

inline int ceil_div(long a, long b) { return (int)((a + b - 1) / b); }
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// simple bump allocator over a caller-provided workspace
struct Arena {
  char* base;
  size_t cap;
  size_t used = 0;
  Arena(void* b, size_t c) : base((char*)b), cap(c) {}
  template <class T>
  T* take(size_t count) {
    size_t off = align_up(used, 256);
    size_t bytes = count * sizeof(T);
    if (base == nullptr || off + bytes > cap) { used = off + bytes; return nullptr; }
    used = off + bytes;
    return reinterpret_cast<T*>(base + off);
  }
};

// ---------------------------------------------------------------------------
// device helpers

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  // D(8x8) += A(8x4, row) * B(4x8, col); lane l holds A[l/4][l%4], B[l%4][l/4],
  // and C[l/4][2*(l%4) + {0,1}].
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// 8-byte async global->shared copy; src_bytes = 0 zero-fills the destination
// shared destination given as a 32-bit shared-window address
__device__ __forceinline__ void cp_async8_s(uint32_t smem_dst, const void* gmem_src, bool valid) {
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_dst), "l"(gmem_src), "r"(sz));
}

__device__ __forceinline__ void cp_async8(void* smem_dst, const void* gmem_src, bool valid) {
  int sz = valid ? 8 : 0;
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(smem_u32(smem_dst)),
               "l"(gmem_src), "r"(sz));
}

// 16-byte async copy (both addresses 16B aligned)
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src, bool valid) {
  int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(smem_dst)),
               "l"(gmem_src), "r"(sz));
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }

template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// sum of squares of x[0..n) into out_dev[0] (fixed-order reduction; part >= 256 doubles)
int launch_sumsq(const double* x, long long n, double* out_dev, double* part, cudaStream_t st);


// ---------------------------------------------------------------------------
// host synchronisation points (a rank or path decision read back to the host);
// counted and timed when TTK_HOST_PROF is set (ttk_debug_host_profile)
int host_sync(cudaStream_t st);
#define TTK_SYNC(st) TTK_TRY(::ttk::host_sync(st))

}  // namespace ttk
