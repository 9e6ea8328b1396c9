// Cluster ping-pong latency of one Jacobi-sized message (16 lanes x 6 doubles
// + an id) between two CTAs of a cluster, for the exchange variants the
// cluster Jacobi could use.  Build: nvcc -gencode arch=compute_100a,code=sm_100a
// -o tools/dsmem_lat tools/dsmem_lat.cu ; run on the GPU box.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
namespace cg = cooperative_groups;

__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t map_rank(uint32_t a, int r) {
  uint32_t o; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(o) : "r"(a), "r"(r)); return o;
}
__device__ __forceinline__ void wait_parity(uint32_t bar, uint32_t par) {
  uint32_t done;
  do {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n"
                 " selp.u32 %0, 1, 0, p;\n}\n" : "=r"(done) : "r"(bar), "r"(par) : "memory");
  } while (!done);
}

// mode 0: st.async v2 per lane with complete_tx (current kernel)
// mode 1: plain st.shared::cluster v2 per lane, __syncwarp, lane 0 remote arrive.release.cluster
template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) pingpong(int iters, long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  const int rank = cl.block_rank(), lane = threadIdx.x;
  __shared__ __align__(16) double box[2][96];
  __shared__ __align__(8) unsigned long long bar[2];
  const uint32_t b0 = smem_addr(&bar[0]);
  const int peer = rank ^ 1;
  const uint32_t msg_bytes = 16 * 6 * 8;
  if (lane == 0) {
    if (MODE == 0) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0 + 8));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b0), "r"(msg_bytes) : "memory");
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b0 + 8), "r"(msg_bytes) : "memory");
    } else {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0 + 8));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
  }
  cl.sync();
  const uint32_t rbox = map_rank(smem_addr(&box[0][0]), peer);
  const uint32_t rbar = map_rank(b0, peer);
  double v[6];
  for (int i = 0; i < 6; ++i) v[i] = lane + i;
  long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const int buf = it & 1;
    const bool my_turn = ((it & 1) == rank);
    if (my_turn) {
      if (lane < 16) {
        if (MODE == 0) {
          for (int j = 0; j < 6; j += 2)
            asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.f64 [%0], {%1, %2}, [%3];" ::
                             "r"(rbox + buf * 768 + (j * 16 + lane * 2) * 8), "d"(v[j]), "d"(v[j + 1]), "r"(rbar + buf * 8) : "memory");
        } else {
          for (int j = 0; j < 6; j += 2)
            asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(rbox + buf * 768 + (j * 16 + lane * 2) * 8),
                         "d"(v[j]), "d"(v[j + 1]) : "memory");
        }
      }
      if (MODE == 1) {
        __syncwarp();
        if (lane == 0)
          asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar + buf * 8) : "memory");
      }
    } else {
      wait_parity(b0 + buf * 8, (it >> 1) & 1);
      if (MODE == 0 && lane == 0)
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b0 + buf * 8), "r"(msg_bytes) : "memory");
      for (int i = 0; i < 6; ++i) v[i] += box[buf][(i & ~1) * 16 + lane * 2 % 32 + (i & 1)];
    }
  }
  long long t1 = clock64();
  cl.sync();
  if (rank == 0 && lane == 0) { out[MODE * 2] = t1 - t0; out[MODE * 2 + 1] = (long long)v[0]; }
}

int main() {
  long long* d; cudaMalloc(&d, 64);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    pingpong<0><<<2, 32>>>(iters, d);
    pingpong<1><<<2, 32>>>(iters, d);
  }
  cudaDeviceSynchronize();
  long long h[8]; cudaMemcpy(h, d, 64, cudaMemcpyDeviceToHost);
  printf("{\"st_async_oneway_cycles\": %.1f, \"plain_store_release_arrive_oneway_cycles\": %.1f, \"err\": \"%s\"}\n",
         (double)h[0] / iters, (double)h[2] / iters, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
