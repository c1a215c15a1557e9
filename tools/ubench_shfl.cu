// Throughput of SHFL vs LDS.64 vs mixed, per SM (cycles per warp-instruction).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void shfl_tp(double* out, long long* cyc, int n) {
  double a = threadIdx.x, b = a + 1, c = a + 2, d = a + 3;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a += __shfl_up_sync(0xffffffffu, b, 1);
      b += __shfl_down_sync(0xffffffffu, c, 1);
      c += __shfl_up_sync(0xffffffffu, d, 1);
      d += __shfl_down_sync(0xffffffffu, a, 1);
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) { cyc[blockIdx.x] = t1 - t0; }
  out[threadIdx.x] = a + b + c + d;
}

__global__ void lds_tp(double* out, long long* cyc, int n) {
  __shared__ double s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
  __syncthreads();
  double a = 0, b = 0, c = 0, d = 0;
  int j = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a += s[(j + 1) & 4095];
      b += s[(j + 33) & 4095];
      c += s[(j + 65) & 4095];
      d += s[(j + 97) & 4095];
      j = (j + 128) & 4095;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[threadIdx.x] = a + b + c + d;
}

__global__ void mix_tp(double* out, long long* cyc, int n) {
  __shared__ double s[4096];
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i;
  __syncthreads();
  double a = 0, b = 1, c = 2, d = 3;
  int j = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      a += s[(j + 1) & 4095];
      b += s[(j + 33) & 4095];
      c += __shfl_up_sync(0xffffffffu, d, 1);
      d += __shfl_down_sync(0xffffffffu, a, 1);
      j = (j + 128) & 4095;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
  out[threadIdx.x] = a + b + c + d;
}

int main() {
  double* o; long long* c; cudaMalloc(&o, 8 * 1024); cudaMalloc(&c, 8 * 64);
  const int n = 2000;
  for (int w : {8, 16, 32}) {
    long long h;
    shfl_tp<<<1, 32 * w>>>(o, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double shfl = double(h) / (n * 32.0 * w);  // 32 shfl instr (of a 64-bit value = 2 SHFL each) per iter per warp
    lds_tp<<<1, 32 * w>>>(o, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double lds = double(h) / (n * 32.0 * w);
    mix_tp<<<1, 32 * w>>>(o, c, n); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
    double mix = double(h) / (n * 32.0 * w);
    printf("warps %2d: cycles per warp-op (64-bit): shfl %.3f  lds.64 %.3f  mixed(half/half) %.3f\n", w, shfl, lds, mix);
  }
  printf("%s\n", cudaGetErrorString(cudaDeviceSynchronize()));
}
