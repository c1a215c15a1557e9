// Device probes used by bench.py to obtain live roofline denominators.
#include "ptb_internal.h"

namespace ptb {
namespace {

// 8 independent DFMA chains per thread; the result is stored so nothing is elided.
__global__ void __launch_bounds__(256) k_dfma_peak(int iters, double seed, double* sink) {
  double a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3, a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6,
         a7 = a0 + 7;
  const double m = 0.999999, c = 1e-7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      a0 = fma(a0, m, c); a1 = fma(a1, m, c); a2 = fma(a2, m, c); a3 = fma(a3, m, c);
      a4 = fma(a4, m, c); a5 = fma(a5, m, c); a6 = fma(a6, m, c); a7 = fma(a7, m, c);
    }
  }
  const double r = ((a0 + a1) + (a2 + a3)) + ((a4 + a5) + (a6 + a7));
  if (r == 12345.678) sink[threadIdx.x] = r;
}

}  // namespace
}  // namespace ptb

using namespace ptb;

extern "C" ptb_status ptb_probe_fp64_peak(ptb_context* ctx, double* tflops, double* ms) {
  try {
    cudaSetDevice(ctx->device);
    double* sink = static_cast<double*>(ctx->scratch[3].get(256 * sizeof(double)));
    const int blocks = ctx->num_sms * 8, threads = 256, iters = 4096;
    k_dfma_peak<<<blocks, threads, 0, ctx->stream>>>(64, 1.0, sink);  // warm-up
    cudaEvent_t e0, e1;
    PTB_CUDA_CHECK(cudaEventCreate(&e0));
    PTB_CUDA_CHECK(cudaEventCreate(&e1));
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      PTB_CUDA_CHECK(cudaEventRecord(e0, ctx->stream));
      k_dfma_peak<<<blocks, threads, 0, ctx->stream>>>(iters, 1.0, sink);
      PTB_CUDA_CHECK(cudaEventRecord(e1, ctx->stream));
      PTB_CUDA_CHECK(cudaEventSynchronize(e1));
      float t = 0;
      PTB_CUDA_CHECK(cudaEventElapsedTime(&t, e0, e1));
      best = std::min(best, t);
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double flops = 2.0 * 8 * 16 * double(iters) * blocks * threads;
    *ms = best;
    *tflops = flops / (best * 1e-3) / 1e12;
    return PTB_OK;
  } catch (const Error& e) {
    return e.status;
  }
}
