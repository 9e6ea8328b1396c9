// TT containers (reference tt.py:451-520, test_tt.py:363-387): 8-byte magic
// "TTKVEC01" (vector) / "TTKOPR01" (operator), int64 little-endian header
//   vector:   d, dims[d], ranks[d+1]
//   operator: d, row_dims[d], col_dims[d], ranks[d+1]
// then every core as row-major float64 little-endian.
// Cores move between the file and host or device memory; device transfers go
// through two pinned staging buffers so file reads/writes overlap the copies.
#include "common.cuh"
#include "../../include/ttk_b200.h"

#include <cstdio>
#include <cstring>
#include <vector>

namespace ttk {
namespace {

constexpr char kVecMagic[9] = "TTKVEC01";
constexpr char kOpMagic[9] = "TTKOPR01";
constexpr size_t kStage = 32u << 20;  // bytes per pinned staging buffer

struct File {
  FILE* f = nullptr;
  explicit File(const char* path, const char* mode) { f = fopen(path, mode); }
  ~File() { if (f) fclose(f); }
};

// header ints after the magic: d, then dims (1 or 2 lists of d), then d+1 ranks
int header_len(int kind, int d) { return 1 + (kind ? 2 : 1) * d + d + 1; }

long long core_elems(int kind, int d, const long long* h, int k) {
  const long long* dims = h + 1;
  const long long* ranks = h + 1 + (kind ? 2 : 1) * d;
  long long e = ranks[k] * dims[k] * ranks[k + 1];
  if (kind) e *= dims[d + k];
  return e;
}

int check_header(int kind, int d, const long long* h) {
  TTK_REQUIRE(d >= 1 && d <= 4096, kInvalidValue, "TT container: bad order d=%d", d);
  const int nd = (kind ? 2 : 1) * d;
  for (int i = 0; i < nd; ++i) TTK_REQUIRE(h[1 + i] >= 1, kInvalidValue, "TT container: bad mode size");
  for (int i = 0; i <= d; ++i) TTK_REQUIRE(h[1 + nd + i] >= 1, kInvalidValue, "TT container: bad rank");
  return kOk;
}

struct Pinned {
  void* p[2] = {nullptr, nullptr};
  cudaEvent_t ev[2] = {nullptr, nullptr};
  int init() {
    for (int i = 0; i < 2; ++i) {
      TTK_CHECK_CUDA(cudaMallocHost(&p[i], kStage));
      TTK_CHECK_CUDA(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    }
    return kOk;
  }
  ~Pinned() {
    for (int i = 0; i < 2; ++i) {
      if (ev[i]) { cudaEventSynchronize(ev[i]); cudaEventDestroy(ev[i]); }
      if (p[i]) cudaFreeHost(p[i]);
    }
  }
};

}  // namespace
}  // namespace ttk

using namespace ttk;

extern "C" {

int ttk_io_read_header(const char* path, int* kind, int* d, long long* header, int cap) {
  File fh(path, "rb");
  TTK_REQUIRE(fh.f != nullptr, kInvalidValue, "cannot open %s", path);
  char magic[8];
  TTK_REQUIRE(fread(magic, 1, 8, fh.f) == 8, kInvalidValue, "truncated TT container");
  if (memcmp(magic, kVecMagic, 8) == 0) *kind = 0;
  else if (memcmp(magic, kOpMagic, 8) == 0) *kind = 1;
  else { set_error("not a TT vector or operator container"); return kInvalidValue; }
  long long dd = 0;
  TTK_REQUIRE(fread(&dd, 8, 1, fh.f) == 1, kInvalidValue, "truncated TT container");
  TTK_REQUIRE(dd >= 1 && dd <= 4096, kInvalidValue, "TT container: bad order d=%lld", dd);
  *d = (int)dd;
  const int n = header_len(*kind, *d);
  TTK_REQUIRE(n <= cap, kInvalidValue, "header buffer too small (%d < %d)", cap, n);
  header[0] = dd;
  TTK_REQUIRE(fread(header + 1, 8, n - 1, fh.f) == (size_t)(n - 1), kInvalidValue, "truncated TT container");
  return check_header(*kind, *d, header);
}

int ttk_io_read_cores(const char* path, int to_device, double* const* cores, void* stream) {
  int kind = 0, d = 0;
  std::vector<long long> h(1 + 3 * 4096 + 1);
  TTK_TRY(ttk_io_read_header(path, &kind, &d, h.data(), (int)h.size()));
  File fh(path, "rb");
  TTK_REQUIRE(fh.f != nullptr, kInvalidValue, "cannot open %s", path);
  TTK_REQUIRE(fseek(fh.f, 8 + 8L * header_len(kind, d), SEEK_SET) == 0, kInvalidValue, "seek failed");
  cudaStream_t st = (cudaStream_t)stream;
  Pinned pin;
  if (to_device) TTK_TRY(pin.init());
  int buf = 0;
  for (int k = 0; k < d; ++k) {
    const size_t bytes = (size_t)core_elems(kind, d, h.data(), k) * 8;
    if (!to_device) {
      TTK_REQUIRE(fread(cores[k], 1, bytes, fh.f) == bytes, kInvalidValue, "truncated TT container");
      continue;
    }
    for (size_t off = 0; off < bytes; off += kStage) {
      const size_t chunk = std::min(kStage, bytes - off);
      TTK_CHECK_CUDA(cudaEventSynchronize(pin.ev[buf]));  // previous copy out of this buffer done
      TTK_REQUIRE(fread(pin.p[buf], 1, chunk, fh.f) == chunk, kInvalidValue, "truncated TT container");
      TTK_CHECK_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(cores[k]) + off, pin.p[buf], chunk,
                                     cudaMemcpyHostToDevice, st));
      TTK_CHECK_CUDA(cudaEventRecord(pin.ev[buf], st));
      buf ^= 1;
    }
  }
  if (to_device) TTK_SYNC(st);
  return kOk;
}

int ttk_io_write(const char* path, int kind, int d, const long long* header, int from_device,
                 const double* const* cores, void* stream) {
  TTK_REQUIRE(kind == 0 || kind == 1, kInvalidValue, "kind must be 0 (vector) or 1 (operator)");
  TTK_REQUIRE(header[0] == d, kInvalidValue, "header[0] must equal d");
  TTK_TRY(check_header(kind, d, header));
  File fh(path, "wb");
  TTK_REQUIRE(fh.f != nullptr, kInvalidValue, "cannot open %s for writing", path);
  TTK_REQUIRE(fwrite(kind ? kOpMagic : kVecMagic, 1, 8, fh.f) == 8, kInvalidValue, "write failed");
  const int n = header_len(kind, d);
  TTK_REQUIRE(fwrite(header, 8, n, fh.f) == (size_t)n, kInvalidValue, "write failed");
  cudaStream_t st = (cudaStream_t)stream;
  Pinned pin;
  if (from_device) TTK_TRY(pin.init());
  // device -> pinned copy of chunk i+1 overlaps the file write of chunk i
  struct Pending { size_t bytes = 0; int buf = 0; bool live = false; } prev;
  int buf = 0;
  for (int k = 0; k < d; ++k) {
    const size_t bytes = (size_t)core_elems(kind, d, header, k) * 8;
    if (!from_device) {
      TTK_REQUIRE(fwrite(cores[k], 1, bytes, fh.f) == bytes, kInvalidValue, "write failed");
      continue;
    }
    for (size_t off = 0; off < bytes; off += kStage) {
      const size_t chunk = std::min(kStage, bytes - off);
      TTK_CHECK_CUDA(cudaMemcpyAsync(pin.p[buf], reinterpret_cast<const char*>(cores[k]) + off, chunk,
                                     cudaMemcpyDeviceToHost, st));
      TTK_CHECK_CUDA(cudaEventRecord(pin.ev[buf], st));
      if (prev.live) {
        TTK_CHECK_CUDA(cudaEventSynchronize(pin.ev[prev.buf]));
        TTK_REQUIRE(fwrite(pin.p[prev.buf], 1, prev.bytes, fh.f) == prev.bytes, kInvalidValue, "write failed");
      }
      prev.bytes = chunk; prev.buf = buf; prev.live = true;
      buf ^= 1;
    }
  }
  if (prev.live) {
    TTK_CHECK_CUDA(cudaEventSynchronize(pin.ev[prev.buf]));
    TTK_REQUIRE(fwrite(pin.p[prev.buf], 1, prev.bytes, fh.f) == prev.bytes, kInvalidValue, "write failed");
  }
  return kOk;
}

}  // extern "C"
