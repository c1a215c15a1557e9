// FP64 latency / throughput micro-benchmark (B200): dependent DFMA / DADD chains timed with
// clock64 in one warp, and the per-SM DFMA rate with ILP chains x warps.
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void k_lat(double* out, double a, double b, int n, long long* cyc) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      if (OP == 0) x = fma(x, a, b);
      else if (OP == 1) x = x + b;
      else x = x * a;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = t1 - t0;
}

template <int ILP>
__global__ void k_tput(double* out, double a, double b, int n) {
  double x[ILP];
#pragma unroll
  for (int k = 0; k < ILP; ++k) x[k] = a + threadIdx.x + k;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int k = 0; k < ILP; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < ILP; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 1 << 26);
  cudaMalloc(&cyc, 8);
  const int n = 4096;
  const char* names[3] = {"DFMA", "DADD", "DMUL"};
  for (int op = 0; op < 3; ++op) {
    for (int rep = 0; rep < 2; ++rep) {
      if (op == 0) k_lat<0><<<1, 32>>>(out, 0.999, 1e-3, n, cyc);
      if (op == 1) k_lat<1><<<1, 32>>>(out, 0.999, 1e-3, n, cyc);
      if (op == 2) k_lat<2><<<1, 32>>>(out, 0.999, 1e-3, n, cyc);
    }
    long long c;
    cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%s dependent latency: %.2f cycles\n", names[op], double(c) / (16.0 * n));
  }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 1 << 14;
  for (int warps : {1, 2, 4, 8, 16, 32}) {
    for (int ilp : {1, 2, 4, 8}) {
      auto launch = [&] {
        if (ilp == 1) k_tput<1><<<sms, 32 * warps>>>(out, 0.999, 1e-3, iters);
        if (ilp == 2) k_tput<2><<<sms, 32 * warps>>>(out, 0.999, 1e-3, iters);
        if (ilp == 4) k_tput<4><<<sms, 32 * warps>>>(out, 0.999, 1e-3, iters);
        if (ilp == 8) k_tput<8><<<sms, 32 * warps>>>(out, 0.999, 1e-3, iters);
      };
      launch();
      cudaEventRecord(e0);
      launch();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double fmas = double(sms) * 32 * warps * ilp * iters;
      printf("warps/SM %2d ilp %d: %.2f TFLOP/s  (%.2f DFMA warp-instr/clk/SM at %d MHz)\n", warps, ilp,
             2 * fmas / (ms * 1e-3) / 1e12, fmas / 32 / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
  }
  return 0;
}
