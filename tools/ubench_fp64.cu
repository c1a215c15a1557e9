// Microbenchmark: fp64 pipe latency/throughput, shared-memory latency, barrier cost.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ubench_fp64 tools/ubench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_latency(double* out, long long* cyc, int n) {
  double a = out[0], m = 0.9999, c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 32; ++k) a = fma(a, m, c);
  }
  long long t1 = clock64();
  out[1] = a;
  cyc[0] = t1 - t0;
}

__global__ void dadd_latency(double* out, long long* cyc, int n) {
  double a = out[0], c = 1e-9;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 32; ++k) a = a + c;
  }
  long long t1 = clock64();
  out[1] = a;
  cyc[0] = t1 - t0;
}

__global__ void lds_latency(double* out, long long* cyc, int n) {
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) % 1024;
  __syncthreads();
  int p = 0;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 32; ++k) p = idx[p];
  }
  long long t1 = clock64();
  out[1] = p;
  cyc[0] = t1 - t0;
}

// per-warp chain of `chains` independent dfma sequences: throughput vs ILP
template <int CH>
__global__ void dfma_ilp(double* out, long long* cyc, int n) {
  double a[CH];
#pragma unroll
  for (int k = 0; k < CH; ++k) a[k] = out[0] + k;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int k = 0; k < CH; ++k) a[k] = fma(a[k], 0.9999, 1e-9);
  }
  long long t1 = clock64();
  double s = 0;
#pragma unroll
  for (int k = 0; k < CH; ++k) s += a[k];
  if (threadIdx.x == 0 && blockIdx.x == 0) { out[1] = s; cyc[0] = t1 - t0; }
}

__global__ void bar_cost(double* out, long long* cyc, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

int main() {
  double* d; long long* c; long long h;
  cudaMalloc(&d, 64); cudaMalloc(&c, 64);
  cudaMemset(d, 0, 64);
  const int n = 1000;
  dfma_latency<<<1, 1>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", double(h) / (n * 32));
  dadd_latency<<<1, 1>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("DADD dependent latency: %.2f cycles\n", double(h) / (n * 32));
  lds_latency<<<1, 32>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("LDS dependent latency: %.2f cycles\n", double(h) / (n * 32));
  for (int w : {1, 2, 4, 8, 16}) {
    dfma_ilp<1><<<1, 32 * w>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double per = double(h) / (n * 8);
    dfma_ilp<4><<<1, 32 * w>>>(d, c, n); long long h4; cudaMemcpy(&h4, c, 8, cudaMemcpyDeviceToHost);
    dfma_ilp<8><<<1, 32 * w>>>(d, c, n); long long h8; cudaMemcpy(&h8, c, 8, cudaMemcpyDeviceToHost);
    printf("warps/SM %2d: ILP1 %.2f cyc/dfma-round, ILP4 %.2f, ILP8 %.2f  (per warp-instr: %.2f %.2f %.2f)\n", w, per,
           double(h4) / (n * 8), double(h8) / (n * 8), per / w, double(h4) / (n * 8) / (4 * w), double(h8) / (n * 8) / (8 * w));
  }
  for (int w : {4, 8, 16}) {
    bar_cost<<<1, 32 * w>>>(d, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    printf("__syncthreads with %d warps: %.1f cycles\n", w, double(h) / n);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
}
