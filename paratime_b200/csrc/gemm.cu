// Hand-written fp64 GEMM / GEMV for the Procrustes step and the theta sweep (sm_100a).
//
// Every matrix product of the reference's corrector (procrustes.cpp:65-66 R_F R_G^T and the
// Q U / Q V rotations, :201-207 U^T F / V^T G and the projections, :217 H, :233-234 the new
// factors, :251 the residual; PhaseCorrector::apply :82-86) and of the sweep restructure
// (Z dz, Y^T Lambda w) goes through ptb::gemm below — column-major BLAS semantics,
// C = alpha op(A) op(B) + beta C.
//
// Why DFMA and not the fp64 tensor path: a DMMA m8n8k4 fragment gives every lane a distinct
// operand element, so a warp streams 512 B of shared memory per 512 flops with no broadcast;
// at B200's 128 B/clk/SM that caps a shared-memory-fed DMMA kernel near the DFMA pipe's own
// 64 FMA/clk/SM unless the per-warp tile is 64 x 64 (256 accumulator registers).  A DFMA
// register tile whose warp shares A rows by broadcast needs ~576 B per 16 warp-DFMA, well
// under the pipe's rate.  profiles/r02_gemm_ncu.md compares this kernel with cuBLAS's DMMA
// (sm80 d884) kernels on the corrector's shapes.
//
// Kernels
//   k_dgemm<TA, TB>  64 x 64 CTA tile, BK = 16, 256 threads, 4 x 4 outputs per thread
//                    (rows {2ty, 2ty+1, 32+2ty, 33+2ty}, columns likewise from tx: every
//                    LDS.128 of a quarter warp is 128 contiguous bytes), global loads staged in
//                    registers one k-tile ahead (double-buffered shared memory, one barrier per
//                    k-tile).  Split-K over blockIdx.z for the corrector's tall-skinny
//                    products (k = 3 N_c up to 196608, m, n <= ~1100): partial tiles go to a
//                    workspace and k_splitk_reduce sums them in split order — deterministic,
//                    independent of timing.
//   k_gemv_n         y = alpha A x + beta y, one thread per row (coalesced columns of A).
//   k_gemv_t         y = alpha A^T x + beta y: column dot products split over row chunks,
//                    fixed-order partial sums (k_splitk_reduce with n = 1).
//   k_geam_sub       D = F - D (relative_residual, procrustes.cpp:251).

#include <algorithm>

#include "ptb_internal.h"
#include "ptb_procrustes.h"

namespace ptb {
namespace {

constexpr int BM = 64, BN = 64, BK = 16, GT = 256;
constexpr int LDS_A = BM + 2, LDS_B = BN + 2;  // padded rows, 16-byte aligned

struct GemmArgs {
  int m, n, k;
  const double* A;
  int lda;
  const double* B;
  int ldb;
  double* C;
  int ldc;
  double alpha, beta;
  int kchunk;  // k-range per blockIdx.z
  double* ws;  // split-K partials [z][n][m] (null: write C)
};

// op(A) tile (BM x BK) of k-tile k0 into registers: 4 values per thread
template <bool TA>
__device__ __forceinline__ void load_a(const GemmArgs& a, int i0, int k0, int kend, double (&r)[4]) {
  const int t = threadIdx.x;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int i, kk;
    if (!TA) {  // A(i, kk) = A[i + kk lda]: a warp reads 32 consecutive rows
      i = t % BM;
      kk = t / BM + 4 * j;
    } else {  // op(A)(i, kk) = A[kk + i lda]: a warp reads 2 x 16 consecutive k
      kk = t % BK;
      i = t / BK + 16 * j;
    }
    const int gi = i0 + i, gk = k0 + kk;
    r[j] = (gi < a.m && gk < kend) ? (TA ? a.A[gk + size_t(gi) * a.lda] : a.A[gi + size_t(gk) * a.lda]) : 0.0;
  }
}
template <bool TA>
__device__ __forceinline__ void store_a(double* As, const double (&r)[4]) {
  const int t = threadIdx.x;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int i = TA ? t / BK + 16 * j : t % BM, kk = TA ? t % BK : t / BM + 4 * j;
    As[kk * LDS_A + i] = r[j];
  }
}
// op(B) tile (BK x BN)
template <bool TB>
__device__ __forceinline__ void load_b(const GemmArgs& a, int j0, int k0, int kend, double (&r)[4]) {
  const int t = threadIdx.x;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    int c, kk;
    if (TB) {  // op(B)(kk, c) = B[c + kk ldb]: contiguous in c
      c = t % BN;
      kk = t / BN + 4 * j;
    } else {  // B(kk, c) = B[kk + c ldb]: contiguous in kk
      kk = t % BK;
      c = t / BK + 16 * j;
    }
    const int gc = j0 + c, gk = k0 + kk;
    r[j] = (gc < a.n && gk < kend) ? (TB ? a.B[gc + size_t(gk) * a.ldb] : a.B[gk + size_t(gc) * a.ldb]) : 0.0;
  }
}
template <bool TB>
__device__ __forceinline__ void store_b(double* Bs, const double (&r)[4]) {
  const int t = threadIdx.x;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int c = TB ? t % BN : t / BK + 16 * j, kk = TB ? t / BN + 4 * j : t % BK;
    Bs[kk * LDS_B + c] = r[j];
  }
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(GT) k_dgemm(const GemmArgs a) {
  __shared__ __align__(16) double As[2][BK * LDS_A];
  __shared__ __align__(16) double Bs[2][BK * LDS_B];
  const int i0 = blockIdx.x * BM, j0 = blockIdx.y * BN;
  const int kbeg = blockIdx.z * a.kchunk, kend = min(a.k, kbeg + a.kchunk);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[4][4];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[p][q] = 0.0;
  double ra[4], rb[4];
  load_a<TA>(a, i0, kbeg, kend, ra);
  load_b<TB>(a, j0, kbeg, kend, rb);
  store_a<TA>(As[0], ra);
  store_b<TB>(Bs[0], rb);
  __syncthreads();
  int buf = 0;
  for (int k0 = kbeg; k0 < kend; k0 += BK) {
    const bool more = k0 + BK < kend;
    if (more) {  // next k-tile in flight while this one is multiplied
      load_a<TA>(a, i0, k0 + BK, kend, ra);
      load_b<TB>(a, j0, k0 + BK, kend, rb);
    }
    const double* as = As[buf];
    const double* bs = Bs[buf];
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      const double2 a0 = *reinterpret_cast<const double2*>(as + kk * LDS_A + 2 * ty);
      const double2 a1 = *reinterpret_cast<const double2*>(as + kk * LDS_A + 32 + 2 * ty);
      const double2 b0 = *reinterpret_cast<const double2*>(bs + kk * LDS_B + 2 * tx);
      const double2 b1 = *reinterpret_cast<const double2*>(bs + kk * LDS_B + 32 + 2 * tx);
      const double av[4] = {a0.x, a0.y, a1.x, a1.y}, bv[4] = {b0.x, b0.y, b1.x, b1.y};
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fma(av[p], bv[q], acc[p][q]);
    }
    if (more) {
      store_a<TA>(As[buf ^ 1], ra);
      store_b<TB>(Bs[buf ^ 1], rb);
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int i = i0 + (p < 2 ? 2 * ty + p : 32 + 2 * ty + p - 2);
    if (i >= a.m) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + (q < 2 ? 2 * tx + q : 32 + 2 * tx + q - 2);
      if (j >= a.n) continue;
      if (a.ws) {
        a.ws[(size_t(blockIdx.z) * a.n + j) * a.m + i] = acc[p][q];
      } else {
        double* c = a.C + i + size_t(j) * a.ldc;
        *c = a.beta == 0.0 ? a.alpha * acc[p][q] : a.alpha * acc[p][q] + a.beta * *c;
      }
    }
  }
}

// C = alpha sum_z ws[z] + beta C, partials summed in split order (deterministic)
__global__ void k_splitk_reduce(int m, int n, int splits, const double* __restrict__ ws, double alpha, double beta,
                                double* C, int ldc) {
  const size_t total = size_t(m) * n;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += ws[size_t(z) * total + e];
    const size_t i = e % m, j = e / m;
    double* c = C + i + j * ldc;
    *c = beta == 0.0 ? alpha * s : alpha * s + beta * *c;
  }
}

// y = alpha A x + beta y (A m x k column-major): one thread per row, k sequential
__global__ void k_gemv_n(int m, int k, double alpha, const double* __restrict__ A, int lda,
                         const double* __restrict__ x, double beta, double* y) {
  extern __shared__ double xs[];
  for (int j = threadIdx.x; j < k; j += blockDim.x) xs[j] = x[j];
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  double s0 = 0.0, s1 = 0.0;  // two chains: even / odd columns (more loads in flight)
  int j = 0;
  for (; j + 1 < k; j += 2) {
    s0 = fma(A[i + size_t(j) * lda], xs[j], s0);
    s1 = fma(A[i + size_t(j + 1) * lda], xs[j + 1], s1);
  }
  if (j < k) s0 = fma(A[i + size_t(j) * lda], xs[j], s0);
  const double s = s0 + s1;
  y[i] = beta == 0.0 ? alpha * s : alpha * s + beta * y[i];
}

// partial[z][j] = sum over rows [z chunk) of A(:, j) . x  (A rows x m column-major)
__global__ void __launch_bounds__(256) k_gemv_t_part(int rows, int m, int chunk, const double* __restrict__ A, int lda,
                                                     const double* __restrict__ x, double* __restrict__ part) {
  const int j = blockIdx.x, z = blockIdx.y;
  const int r0 = z * chunk, r1 = min(rows, r0 + chunk);
  const double* col = A + size_t(j) * lda;
  double s = 0.0;
  for (int r = r0 + threadIdx.x; r < r1; r += blockDim.x) s = fma(col[r], x[r], s);
  __shared__ double red[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[size_t(z) * m + j] = t;
  }
}

__global__ void k_geam_sub(size_t total, const double* __restrict__ F, double* D) {
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x)
    D[e] = F[e] - D[e];
}

unsigned ew_grid(ptb_context* ctx, size_t total) {
  return unsigned(std::min<size_t>((total + 255) / 256, size_t(ctx->num_sms) * 8));
}

double* workspace(ptb_context* ctx, size_t doubles) {
  return static_cast<double*>(ctx->gemm_ws.get(std::max<size_t>(1, doubles) * sizeof(double)));
}

}  // namespace

// C (m x n) = alpha op(A) op(B) + beta C, all column-major (BLAS dgemm semantics)
void gemm(ptb_context* ctx, bool ta, bool tb, int m, int n, int k, double alpha, const double* A, int lda,
          const double* B, int ldb, double beta, double* C, int ldc) {
  if (m == 0 || n == 0) return;
  cudaStream_t st = ctx->stream;
  if (k == 0) {
    if (beta == 0.0) {
      for (int j = 0; j < n; ++j) PTB_CUDA_CHECK(cudaMemsetAsync(C + size_t(j) * ldc, 0, size_t(m) * sizeof(double), st));
    } else if (beta != 1.0) {
      gemm(ctx, false, false, m, n, 1, 0.0, C, ldc, C, 1, beta, C, ldc);  // C = beta C
    }
    return;
  }
  if (n == 1 && !tb) {  // matrix-vector products (the sweep's Z dz, the single apply)
    if (!ta) {
      const int T = 256;
      k_gemv_n<<<unsigned((m + T - 1) / T), T, size_t(k) * sizeof(double), st>>>(m, k, alpha, A, lda, B, beta, C);
      PTB_LAUNCH_CHECK(ctx);
      return;
    }
    const int chunk = std::max(2048, (k + 63) / 64), splits = (k + chunk - 1) / chunk;
    double* part = workspace(ctx, size_t(splits) * m);
    k_gemv_t_part<<<dim3(unsigned(m), unsigned(splits)), 256, 0, st>>>(k, m, chunk, A, lda, B, part);
    PTB_LAUNCH_CHECK(ctx);
    k_splitk_reduce<<<ew_grid(ctx, size_t(m)), 256, 0, st>>>(m, 1, splits, part, alpha, beta, C, ldc);
    PTB_LAUNCH_CHECK(ctx);
    return;
  }
  const int tm = (m + BM - 1) / BM, tn = (n + BN - 1) / BN, tiles = tm * tn;
  // split K so the grid covers >= 2 CTAs per SM, keeping >= 4 k-tiles per split
  int splits = 1;
  const int want = 2 * ctx->num_sms;
  if (tiles < want) splits = std::min({(want + tiles - 1) / tiles, (k + 4 * BK - 1) / (4 * BK), 128});
  int kchunk = ((k + splits - 1) / splits + BK - 1) / BK * BK;
  splits = (k + kchunk - 1) / kchunk;
  GemmArgs a{m, n, k, A, lda, B, ldb, C, ldc, alpha, beta, kchunk, nullptr};
  if (splits > 1) a.ws = workspace(ctx, size_t(splits) * m * n);
  const dim3 grid{unsigned(tm), unsigned(tn), unsigned(splits)};
  if (!ta && !tb) k_dgemm<false, false><<<grid, GT, 0, st>>>(a);
  else if (ta && !tb) k_dgemm<true, false><<<grid, GT, 0, st>>>(a);
  else if (!ta && tb) k_dgemm<false, true><<<grid, GT, 0, st>>>(a);
  else k_dgemm<true, true><<<grid, GT, 0, st>>>(a);
  PTB_LAUNCH_CHECK(ctx);
  if (splits > 1) {
    k_splitk_reduce<<<ew_grid(ctx, size_t(m) * n), 256, 0, st>>>(m, n, splits, a.ws, alpha, beta, C, ldc);
    PTB_LAUNCH_CHECK(ctx);
  }
}

// D = F - D, rows x cols contiguous (relative_residual)
void geam_sub(ptb_context* ctx, size_t total, const double* F, double* D) {
  if (total == 0) return;
  k_geam_sub<<<ew_grid(ctx, total), 256, 0, ctx->stream>>>(total, F, D);
  PTB_LAUNCH_CHECK(ctx);
}

}  // namespace ptb
