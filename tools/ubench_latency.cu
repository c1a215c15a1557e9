// Latency micro-benchmark on B200 (sm_100a): cycles per iteration of
//   cluster.sync() (8 CTAs), cluster.sync() + dependent DSMEM load, __syncthreads(),
//   and dependent chains of FP64 div / sqrt / rsqrt and 64-bit warp shuffles.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_latency tools/ubench_latency.cu
#include <cooperative_groups.h>
#include <cstdio>

#include "../paratime_b200/csrc/ptb_dsmem.h"
using namespace ptb;

namespace cg = cooperative_groups;
constexpr int ITERS = 4096;

__global__ void __cluster_dims__(8, 1, 1) k_cluster_sync(long long* out, int mode) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double buf[64];
  buf[threadIdx.x & 63] = threadIdx.x;
  cl.sync();
  double acc = 0.0;
  const unsigned peer = (cl.block_rank() + 1) % 8;
  double* remote = cl.map_shared_rank(buf, peer);
  const long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
    if (mode == 0) {
      cl.sync();
    } else if (mode == 1) {
      cl.sync();
      acc += remote[(i + int(acc)) & 63];  // dependent DSMEM load after the barrier
    } else {
      __syncthreads();
    }
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[mode] = (t1 - t0) / ITERS + (acc == -1.0 ? 1 : 0);
}

__global__ void k_fp64_chain(long long* out, double seed) {
  double x = seed + threadIdx.x * 1e-9, y = 1.5;
  long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) x = 1.0 / (x + 1.0);
  long long t1 = clock64();
  if (threadIdx.x == 0) out[0] = (t1 - t0) / ITERS;
  t0 = clock64();
  for (int i = 0; i < ITERS; ++i) y = sqrt(y + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) out[1] = (t1 - t0) / ITERS;
  double z = 1.25;
  t0 = clock64();
  for (int i = 0; i < ITERS; ++i) z = rsqrt(z + 1.0);
  t1 = clock64();
  if (threadIdx.x == 0) out[2] = (t1 - t0) / ITERS;
  double w = 0.5 + threadIdx.x;  // lane-dependent: a uniform value lets the compiler drop the shuffle
  t0 = clock64();
  for (int i = 0; i < ITERS; ++i) w = __shfl_xor_sync(0xffffffffu, w, 1 + (i & 3)) * 0.999 + 0.001;
  t1 = clock64();
  if (threadIdx.x == 0) out[3] = (t1 - t0) / ITERS;
  double v = 0.5;
  t0 = clock64();
  for (int i = 0; i < ITERS; ++i) v = fma(v, 0.999, 0.001);
  t1 = clock64();
  if (threadIdx.x == 0) out[4] = (t1 - t0) / ITERS;
  if (x + y + z + w + v == -1.0) out[5] = 1;
}

// issue cost of one st.async (16 B) to the next rank + mapa, no waiting (ITERS sends, one
// mbarrier wait for all bytes at the end)
__global__ void __cluster_dims__(8, 1, 1) k_st_async_issue(long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double buf[2];
  __shared__ __align__(8) unsigned long long bar;
  const unsigned b0 = smem_addr(&bar);
  if (threadIdx.x == 0) {
    mbar_init(b0, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  cl.sync();
  const int peer = (cl.block_rank() + 1) % 8;
  if (threadIdx.x == 0) mbar_expect(b0, 16u * ITERS);
  const long long t0 = clock64();
  if (threadIdx.x == 0)
    for (int i = 0; i < ITERS; ++i) st_async2(cluster_map(smem_addr(&buf[0]), peer), 1.0, double(i), cluster_map(b0, peer));
  const long long t1 = clock64();
  mbar_wait(b0, 0);
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = (t1 - t0) / ITERS;
  cl.sync();
}

// st.async ring: every CTA sends 16 bytes to the next rank and waits for its own 16 bytes
// (mbarrier transaction count), ITERS times; cycles per hop
__global__ void __cluster_dims__(8, 1, 1) k_st_async_ring(long long* out) {
  cg::cluster_group cl = cg::this_cluster();
  __shared__ double buf[2][2];
  __shared__ __align__(8) unsigned long long bars[2];
  const unsigned bar0 = smem_addr(&bars[0]);
  if (threadIdx.x == 0) {
    mbar_init(bar0, 1);
    mbar_init(bar0 + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  cl.sync();
  const int peer = (cl.block_rank() + 1) % 8;
  double acc = 0.0;
  const long long t0 = clock64();
  for (int i = 0; i < ITERS; ++i) {
    const unsigned bar = bar0 + 8u * unsigned(i & 1);
    if (threadIdx.x == 0) {
      mbar_expect(bar, 16);
      st_async2(cluster_map(smem_addr(&buf[i & 1][0]), peer), acc, 1.0, cluster_map(bar, peer));
    }
    mbar_wait(bar, unsigned(i >> 1) & 1u);
    acc += buf[i & 1][1];
    __syncthreads();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0 && cl.block_rank() == 0) out[0] = (t1 - t0) / ITERS + (acc == -1.0 ? 1 : 0);
  cl.sync();
}

int main() {
  long long* d;
  long long h[8] = {};
  cudaMalloc(&d, sizeof(h));
  for (int mode = 0; mode < 3; ++mode) k_cluster_sync<<<8, 256>>>(d, mode);
  cudaMemcpy(h, d, 3 * sizeof(long long), cudaMemcpyDeviceToHost);
  std::printf("cycles/iter: cluster.sync %lld, cluster.sync+DSMEM load %lld, __syncthreads(256) %lld\n", h[0], h[1],
              h[2]);
  k_st_async_ring<<<8, 256>>>(d);
  cudaMemcpy(h, d, sizeof(long long), cudaMemcpyDeviceToHost);
  std::printf("st.async + mbarrier ring hop: %lld cycles\n", h[0]);
  k_st_async_issue<<<8, 32>>>(d);
  cudaMemcpy(h, d, sizeof(long long), cudaMemcpyDeviceToHost);
  std::printf("st.async issue (one thread, back to back): %lld cycles each\n", h[0]);
  k_fp64_chain<<<1, 32>>>(d, 1.0);
  cudaMemcpy(h, d, 5 * sizeof(long long), cudaMemcpyDeviceToHost);
  std::printf("dependent cycles: ddiv %lld, dsqrt %lld, drsqrt %lld, 64-bit shfl+dfma %lld, dfma %lld\n", h[0], h[1],
              h[2], h[3], h[4]);
  return cudaGetLastError() != cudaSuccess;
}
