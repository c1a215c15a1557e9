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
//   k_dgemm<TA, TB>  128 x 64 CTA tile, BK = 16, 256 threads, 8 x 4 outputs per thread
//                    (rows 32p + 2ty + {0,1}, columns 32q + 2tx + {0,1}: every LDS.128 of a
//                    quarter warp is 128 contiguous bytes or a broadcast), global loads staged in
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
#include <functional>
#include <cstdlib>
#include <string>

#include "ptb_internal.h"
#include "ptb_procrustes.h"

namespace ptb {
namespace {

constexpr int BM = 128, BN = 64, BK = 16, GT = 256;
constexpr int LDS_A = BM + 2, LDS_B = BN + 2;  // padded rows, 16-byte aligned
constexpr int AL = BM * BK / GT, BL = BN * BK / GT;  // staged global loads per thread: 8 of A, 4 of B
constexpr size_t GEMM_SMEM = size_t(2) * BK * (LDS_A + LDS_B) * sizeof(double);  // 49 KB: dynamic

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
  int tc = 0;  // 1: the kernel computes C^T (m x n here = C's n x m): element (i, j) goes to C[j + i ldc]
  int zbase = 0;  // k-range of split z starts at (z + zbase) kchunk (row-slab products)
};

// op(A) tile (BM x BK) of k-tile k0 into registers.  !TA: A(i, kk) = A[i + kk lda], a warp reads
// 32 consecutive rows; TA: op(A)(i, kk) = A[kk + i lda], a half warp reads 16 consecutive k.  One
// base pointer per thread, constant strides; bounds checks only on edge tiles.
template <bool TA>
__device__ __forceinline__ void load_a(const GemmArgs& a, int i0, int k0, int kend, double (&r)[AL]) {
  const int t = threadIdx.x;
  const int ib = TA ? t / BK : t % BM, kb = TA ? t % BK : t / BM;  // element j: (ib + di j, kb + dk j)
  constexpr int di = TA ? GT / BK : 0, dk = TA ? 0 : GT / BM;
  const size_t lda = size_t(a.lda);
  const double* p = TA ? a.A + (k0 + kb) + size_t(i0 + ib) * lda : a.A + (i0 + ib) + size_t(k0 + kb) * lda;
  const size_t step = TA ? size_t(di) * lda : size_t(dk) * lda;
  if (i0 + BM <= a.m && k0 + BK <= kend) {
#pragma unroll
    for (int j = 0; j < AL; ++j) r[j] = p[j * step];
  } else {
#pragma unroll
    for (int j = 0; j < AL; ++j)
      r[j] = (i0 + ib + di * j < a.m && k0 + kb + dk * j < kend) ? p[j * step] : 0.0;
  }
}
template <bool TA>
__device__ __forceinline__ void store_a(double* As, const double (&r)[AL]) {
  const int t = threadIdx.x;
#pragma unroll
  for (int j = 0; j < AL; ++j) {
    const int i = TA ? t / BK + (GT / BK) * j : t % BM, kk = TA ? t % BK : t / BM + (GT / BM) * j;
    As[kk * LDS_A + i] = r[j];
  }
}
// op(B) tile (BK x BN).  TB: op(B)(kk, c) = B[c + kk ldb], contiguous in c; else B(kk, c) =
// B[kk + c ldb], contiguous in kk
template <bool TB>
__device__ __forceinline__ void load_b(const GemmArgs& a, int j0, int k0, int kend, double (&r)[BL]) {
  const int t = threadIdx.x;
  const int cb = TB ? t % BN : t / BK, kb = TB ? t / BN : t % BK;
  constexpr int dc = TB ? 0 : GT / BK, dk = TB ? GT / BN : 0;
  const size_t ldb = size_t(a.ldb);
  const double* p = TB ? a.B + (j0 + cb) + size_t(k0 + kb) * ldb : a.B + (k0 + kb) + size_t(j0 + cb) * ldb;
  const size_t step = TB ? size_t(dk) * ldb : size_t(dc) * ldb;
  if (j0 + BN <= a.n && k0 + BK <= kend) {
#pragma unroll
    for (int j = 0; j < BL; ++j) r[j] = p[j * step];
  } else {
#pragma unroll
    for (int j = 0; j < BL; ++j)
      r[j] = (j0 + cb + dc * j < a.n && k0 + kb + dk * j < kend) ? p[j * step] : 0.0;
  }
}
template <bool TB>
__device__ __forceinline__ void store_b(double* Bs, const double (&r)[BL]) {
  const int t = threadIdx.x;
#pragma unroll
  for (int j = 0; j < BL; ++j) {
    const int c = TB ? t % BN : t / BK + (GT / BK) * j, kk = TB ? t / BN + (GT / BN) * j : t % BK;
    Bs[kk * LDS_B + c] = r[j];
  }
}

// thread (tx, ty) = (t % 16, t / 16) owns rows 32 p + 2 ty + h (p < 4) and columns 32 q + 2 tx + h
// (q < 2), h in {0, 1}: 8 x 4 accumulators; per k step 4 + 2 LDS.128, the A ones shared by the
// 16 lanes of a row group (broadcast), the B ones 128 contiguous bytes per quarter warp
template <bool TA, bool TB>
__global__ void __launch_bounds__(GT, 1) k_dgemm(const GemmArgs a) {
  extern __shared__ __align__(16) double gsm[];  // A stages [2][BK][LDS_A], then B stages [2][BK][LDS_B]
  double* const Asm = gsm;
  double* const Bsm = gsm + 2 * BK * LDS_A;
  const int i0 = blockIdx.x * BM, j0 = blockIdx.y * BN;
  const int kbeg = (int(blockIdx.z) + a.zbase) * a.kchunk, kend = min(a.k, kbeg + a.kchunk);
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  double acc[8][4];
#pragma unroll
  for (int p = 0; p < 8; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[p][q] = 0.0;
  double ra[AL], rb[BL];
  load_a<TA>(a, i0, kbeg, kend, ra);
  load_b<TB>(a, j0, kbeg, kend, rb);
  store_a<TA>(Asm, ra);
  store_b<TB>(Bsm, rb);
  __syncthreads();
  int buf = 0;
  for (int k0 = kbeg; k0 < kend; k0 += BK) {
    const bool more = k0 + BK < kend;
    if (more) {  // next k-tile in flight while this one is multiplied
      load_a<TA>(a, i0, k0 + BK, kend, ra);
      load_b<TB>(a, j0, k0 + BK, kend, rb);
    }
    const double* as = Asm + buf * (BK * LDS_A);
    const double* bs = Bsm + buf * (BK * LDS_B);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double av[8], bv[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) {
        const double2 t2 = *reinterpret_cast<const double2*>(as + kk * LDS_A + 32 * p + 2 * ty);
        av[2 * p] = t2.x;
        av[2 * p + 1] = t2.y;
      }
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const double2 t2 = *reinterpret_cast<const double2*>(bs + kk * LDS_B + 32 * q + 2 * tx);
        bv[2 * q] = t2.x;
        bv[2 * q + 1] = t2.y;
      }
#pragma unroll
      for (int p = 0; p < 8; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[p][q] = fma(av[p], bv[q], acc[p][q]);
    }
    if (more) {
      store_a<TA>(Asm + (buf ^ 1) * (BK * LDS_A), ra);
      store_b<TB>(Bsm + (buf ^ 1) * (BK * LDS_B), rb);
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int i = i0 + 32 * (p / 2) + 2 * ty + (p & 1);
    if (i >= a.m) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int j = j0 + 32 * (q / 2) + 2 * tx + (q & 1);
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

// ---- the fp64 tensor-core variant (DMMA, mma.sync m8n8k4 f64) ----------------------------------
// Same CTA tile (128 x 64, BK = 16, split-K, register-staged double-buffered shared memory) and the
// same global->shared staging as k_dgemm; 8 warps in a 4 x 2 grid, each a 32 x 32 block = 4 x 4
// m8n8k4 tiles (32 accumulator doubles per lane).  Per 4-deep k step a warp loads 4 A and 4 B
// fragments (LDS.64: lane l holds A(8p + l/4, kk + l%4) / B(kk + l%4, 8q + l/4)) and issues 16
// DMMA.  Row strides of 136 / 72 doubles (= 8 mod 16) put the four k rows of a fragment load on
// disjoint bank halves: two wavefronts per LDS.64, the minimum for 256 bytes.  Each output is one
// fixed-order accumulation over k (the DMMA's internal order), independent of the launch shape.
constexpr int MLDS_A = BM + 8, MLDS_B = BN + 8;
constexpr size_t MMA_SMEM = size_t(2) * BK * (MLDS_A + MLDS_B) * sizeof(double);

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// Staging for the DMMA kernel.  Where op(A) / op(B) is contiguous along k in memory (TA, !TB) a
// warp covers 8 rows x 4 consecutive k (one 32-byte sector per row) instead of 2 rows x 16 k: the
// shared-memory store of a fixed k-row then hits 8 consecutive addresses in each of 4 k-rows, whose
// bank halves alternate (row stride 8 mod 16 doubles) -- 2 wavefronts per STS.64 instead of 8.
// Where op(A) / op(B) is contiguous along m / n the layout of load_a / load_b is kept.
template <bool TA>
__device__ __forceinline__ void load_a_m(const GemmArgs& a, int i0, int k0, int kend, double (&r)[AL]) {
  if constexpr (!TA) {
    load_a<false>(a, i0, k0, kend, r);
  } else {
    const int t = threadIdx.x, kb = t % 4, ib = t / 4;  // element j: (ib + 64 (j & 1), kb + 4 (j >> 1))
    const size_t lda = size_t(a.lda);
    const double* p = a.A + (k0 + kb) + size_t(i0 + ib) * lda;
    if (i0 + BM <= a.m && k0 + BK <= kend) {
#pragma unroll
      for (int j = 0; j < AL; ++j) r[j] = p[4 * (j >> 1) + size_t(64 * (j & 1)) * lda];
    } else {
#pragma unroll
      for (int j = 0; j < AL; ++j)
        r[j] = (i0 + ib + 64 * (j & 1) < a.m && k0 + kb + 4 * (j >> 1) < kend)
                   ? p[4 * (j >> 1) + size_t(64 * (j & 1)) * lda]
                   : 0.0;
    }
  }
}
template <bool TA>
__device__ __forceinline__ void store_a_m(double* As, const double (&r)[AL]) {
  const int t = threadIdx.x;
#pragma unroll
  for (int j = 0; j < AL; ++j) {
    const int i = TA ? t / 4 + 64 * (j & 1) : t % BM, kk = TA ? t % 4 + 4 * (j >> 1) : t / BM + (GT / BM) * j;
    As[kk * MLDS_A + i] = r[j];
  }
}
template <bool TB>
__device__ __forceinline__ void load_b_m(const GemmArgs& a, int j0, int k0, int kend, double (&r)[BL]) {
  if constexpr (TB) {
    load_b<true>(a, j0, k0, kend, r);
  } else {
    const int t = threadIdx.x, kb = t % 4, cb = t / 4;  // element j: (kb + 4 j, cb)
    const double* p = a.B + (k0 + kb) + size_t(j0 + cb) * size_t(a.ldb);
    if (j0 + BN <= a.n && k0 + BK <= kend) {
#pragma unroll
      for (int j = 0; j < BL; ++j) r[j] = p[4 * j];
    } else {
#pragma unroll
      for (int j = 0; j < BL; ++j) r[j] = (j0 + cb < a.n && k0 + kb + 4 * j < kend) ? p[4 * j] : 0.0;
    }
  }
}
template <bool TB>
__device__ __forceinline__ void store_b_m(double* Bs, const double (&r)[BL]) {
  const int t = threadIdx.x;
#pragma unroll
  for (int j = 0; j < BL; ++j) {
    const int c = TB ? t % BN : t / 4, kk = TB ? t / BN + (GT / BN) * j : t % 4 + 4 * j;
    Bs[kk * MLDS_B + c] = r[j];
  }
}

template <bool TA, bool TB>
__global__ void __launch_bounds__(GT, 2) k_dgemm_mma(const GemmArgs a) {
  extern __shared__ __align__(16) double gsm[];
  double* const Asm = gsm;
  double* const Bsm = gsm + 2 * BK * MLDS_A;
  const int i0 = blockIdx.x * BM, j0 = blockIdx.y * BN;
  const int kbeg = (int(blockIdx.z) + a.zbase) * a.kchunk, kend = min(a.k, kbeg + a.kchunk);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int wm = (warp & 3) * 32, wn = (warp >> 2) * 32;  // the warp's 32 x 32 block
  const int fr = lane >> 2, fk = lane & 3;                 // fragment row (or column) / k index
  double acc[4][4][2];
#pragma unroll
  for (int p = 0; p < 4; ++p)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[p][q][0] = acc[p][q][1] = 0.0;
  double ra[AL], rb[BL];
  load_a_m<TA>(a, i0, kbeg, kend, ra);
  load_b_m<TB>(a, j0, kbeg, kend, rb);
  store_a_m<TA>(Asm, ra);
  store_b_m<TB>(Bsm, rb);
  __syncthreads();
  int buf = 0;
  for (int k0 = kbeg; k0 < kend; k0 += BK) {
    const bool more = k0 + BK < kend;
    if (more) {
      load_a_m<TA>(a, i0, k0 + BK, kend, ra);
      load_b_m<TB>(a, j0, k0 + BK, kend, rb);
    }
    const double* as = Asm + buf * (BK * MLDS_A) + fk * MLDS_A + wm + fr;
    const double* bs = Bsm + buf * (BK * MLDS_B) + fk * MLDS_B + wn + fr;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int p = 0; p < 4; ++p) af[p] = as[kk * MLDS_A + 8 * p];
#pragma unroll
      for (int q = 0; q < 4; ++q) bf[q] = bs[kk * MLDS_B + 8 * q];
#pragma unroll
      for (int p = 0; p < 4; ++p)
#pragma unroll
        for (int q = 0; q < 4; ++q) dmma884(acc[p][q], af[p], bf[q]);
    }
    if (more) {
      store_a_m<TA>(Asm + (buf ^ 1) * (BK * MLDS_A), ra);
      store_b_m<TB>(Bsm + (buf ^ 1) * (BK * MLDS_B), rb);
    }
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int p = 0; p < 4; ++p) {
    const int i = i0 + wm + 8 * p + fr;
    if (i >= a.m) continue;
#pragma unroll
    for (int q = 0; q < 4; ++q)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int j = j0 + wn + 8 * q + 2 * fk + h;
        if (j >= a.n) continue;
        if (a.ws) {
          a.ws[(size_t(blockIdx.z) * a.n + j) * a.m + i] = acc[p][q][h];
        } else {
          double* c = a.tc ? a.C + j + size_t(i) * a.ldc : a.C + i + size_t(j) * a.ldc;
          *c = a.beta == 0.0 ? a.alpha * acc[p][q][h] : a.alpha * acc[p][q][h] + a.beta * *c;
        }
      }
  }
}

// C = alpha sum_z ws[z] + beta C, partials summed in split order (deterministic)
__global__ void k_splitk_reduce(int m, int n, int splits, const double* __restrict__ ws, double alpha, double beta,
                                double* C, int ldc, int tc = 0) {
  const size_t total = size_t(m) * n;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (int z = 0; z < splits; ++z) s += ws[size_t(z) * total + e];
    const size_t i = e % m, j = e / m;
    double* c = tc ? C + j + i * ldc : C + i + j * ldc;
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
  // one sequential chain per row (a fixed order), loads issued 8 columns ahead of the FMAs
  double s = 0.0;
  const double* a = A + i;
  int j = 0;
  for (; j + 8 <= k; j += 8) {
    double t[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) t[q] = a[size_t(j + q) * lda];
#pragma unroll
    for (int q = 0; q < 8; ++q) s = fma(t[q], xs[j + q], s);
  }
  for (; j < k; ++j) s = fma(a[size_t(j) * lda], xs[j], s);
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

// PTB_DGEMM=dfma|dmma selects the kernel family (A/B measurements); default: DMMA
bool use_dmma() {
  const char* e = std::getenv("PTB_DGEMM");  // read per call: tests switch it with monkeypatch
  return !(e && std::string(e) == "dfma");
}

double* workspace(ptb_context* ctx, size_t doubles) {
  return static_cast<double*>(ctx->gemm_ws.get(std::max<size_t>(1, doubles) * sizeof(double)));
}

}  // namespace

void gemm_core(ptb_context* ctx, bool ta, bool tb, int m, int n, int k, double alpha, const double* A, int lda,
               const double* B, int ldb, double beta, double* C, int ldc, int tc, int max_splits = 128);

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
  // DMMA: a short m that the 128-row tile would pad badly (the corrector's U^T F, r x N') is
  // computed as C^T = op(B)^T op(A)^T with a transposed store when that pads less
  if (use_dmma() && m <= 1024 && n <= 1024) {
    const auto padded = [](int rows, int cols) { return size_t((rows + BM - 1) / BM * BM) * ((cols + BN - 1) / BN * BN); };
    if (padded(n, m) < padded(m, n)) {
      std::swap(m, n);
      std::swap(A, B);
      std::swap(lda, ldb);
      std::swap(ta, tb);
      ta = !ta;
      tb = !tb;
      return gemm_core(ctx, ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, 1);
    }
  }
  return gemm_core(ctx, ta, tb, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, 0);
}

void gemm_core(ptb_context* ctx, bool ta, bool tb, int m, int n, int k, double alpha, const double* A, int lda,
               const double* B, int ldb, double beta, double* C, int ldc, int tc, int max_splits) {
  cudaStream_t st = ctx->stream;
  const int tm = (m + BM - 1) / BM, tn = (n + BN - 1) / BN, tiles = tm * tn;
  // split K so the grid covers >= 2 CTAs per SM, keeping >= 4 k-tiles per split
  int splits = 1;
  const int want = 2 * ctx->num_sms;
  if (tiles < want) splits = std::min({(want + tiles - 1) / tiles, (k + 4 * BK - 1) / (4 * BK), max_splits});
  int kchunk = ((k + splits - 1) / splits + BK - 1) / BK * BK;
  splits = (k + kchunk - 1) / kchunk;
  GemmArgs a{m, n, k, A, lda, B, ldb, C, ldc, alpha, beta, kchunk, nullptr, tc};
  if (splits > 1) a.ws = workspace(ctx, size_t(splits) * m * n);
  const dim3 grid{unsigned(tm), unsigned(tn), unsigned(splits)};
  static const bool attrs = [] {
    for (const void* f : {reinterpret_cast<const void*>(k_dgemm<false, false>),
                          reinterpret_cast<const void*>(k_dgemm<true, false>),
                          reinterpret_cast<const void*>(k_dgemm<false, true>),
                          reinterpret_cast<const void*>(k_dgemm<true, true>)})
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(GEMM_SMEM));
    for (const void* f : {reinterpret_cast<const void*>(k_dgemm_mma<false, false>),
                          reinterpret_cast<const void*>(k_dgemm_mma<true, false>),
                          reinterpret_cast<const void*>(k_dgemm_mma<false, true>),
                          reinterpret_cast<const void*>(k_dgemm_mma<true, true>)})
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(MMA_SMEM));
    return true;
  }();
  (void)attrs;
  if (use_dmma()) {
    if (!ta && !tb) k_dgemm_mma<false, false><<<grid, GT, MMA_SMEM, st>>>(a);
    else if (ta && !tb) k_dgemm_mma<true, false><<<grid, GT, MMA_SMEM, st>>>(a);
    else if (!ta && tb) k_dgemm_mma<false, true><<<grid, GT, MMA_SMEM, st>>>(a);
    else k_dgemm_mma<true, true><<<grid, GT, MMA_SMEM, st>>>(a);
  } else if (!ta && !tb) k_dgemm<false, false><<<grid, GT, GEMM_SMEM, st>>>(a);
  else if (ta && !tb) k_dgemm<true, false><<<grid, GT, GEMM_SMEM, st>>>(a);
  else if (!ta && tb) k_dgemm<false, true><<<grid, GT, GEMM_SMEM, st>>>(a);
  else k_dgemm<true, true><<<grid, GT, GEMM_SMEM, st>>>(a);
  PTB_LAUNCH_CHECK(ctx);
  if (splits > 1) {
    k_splitk_reduce<<<ew_grid(ctx, size_t(m) * n), 256, 0, st>>>(m, n, splits, a.ws, alpha, beta, C, ldc, tc);
    PTB_LAUNCH_CHECK(ctx);
  }
}

// Row-local product for row-sharded matrices: C = alpha A B + beta C on a range of rows, never
// split over k, so every output row has the same value whatever range (rank) computes it.
void gemm_rows(ptb_context* ctx, int m, int n, int k, double alpha, const double* A, int lda, const double* B, int ldb,
               double beta, double* C, int ldc) {
  if (m == 0 || n == 0) return;
  if (k == 0 || n == 1) {  // the general entry handles these shapes (no split over rows either way)
    gemm(ctx, false, false, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc);
    return;
  }
  gemm_core(ctx, false, false, m, n, k, alpha, A, lda, B, ldb, beta, C, ldc, 0, 1);
}

// Row-slab reduction C (m x n) = A^T B over `rows` = P slabs of `slab` rows (A: rows x m, B: rows x n,
// column-major).  This process computes the partials of slabs [z0, z0 + nz) (k-split z of the DMMA
// kernel = one slab) into ws_own (nz x n x m), `gather` assembles all P partials in slab order into
// ws_all (it may be ws_own itself when nz == P), and they are summed in slab order: the value is
// the same whichever process computed which slabs.  A short m is computed as C^T exactly as gemm().
void gemm_tn_slabs(ptb_context* ctx, int m, int n, const double* A, int lda, const double* B, int ldb, double* C,
                   int ldc, int P, int slab, int z0, int nz, double* ws_own, double* ws_all,
                   const std::function<void()>& gather) {
  cudaStream_t st = ctx->stream;
  int tc = 0;
  if (use_dmma() && m <= 1024 && n <= 1024) {
    const auto padded = [](int rows, int cols) { return size_t((rows + BM - 1) / BM * BM) * ((cols + BN - 1) / BN * BN); };
    if (padded(n, m) < padded(m, n)) {
      std::swap(m, n);
      std::swap(A, B);
      std::swap(lda, ldb);
      tc = 1;
    }
  }
  static const bool attrs = [] {
    cudaFuncSetAttribute(reinterpret_cast<const void*>(k_dgemm_mma<true, false>),
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(MMA_SMEM));
    cudaFuncSetAttribute(reinterpret_cast<const void*>(k_dgemm<true, false>),
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(GEMM_SMEM));
    return true;
  }();
  (void)attrs;
  if (nz > 0) {
    GemmArgs a{m, n, P * slab, A, lda, B, ldb, C, ldc, 1.0, 0.0, slab, ws_own, tc, z0};
    const dim3 grid{unsigned((m + BM - 1) / BM), unsigned((n + BN - 1) / BN), unsigned(nz)};
    if (use_dmma())
      k_dgemm_mma<true, false><<<grid, GT, MMA_SMEM, st>>>(a);
    else
      k_dgemm<true, false><<<grid, GT, GEMM_SMEM, st>>>(a);
    PTB_LAUNCH_CHECK(ctx);
  }
  gather();
  k_splitk_reduce<<<ew_grid(ctx, size_t(m) * n), 256, 0, st>>>(m, n, P, ws_all, 1.0, 0.0, C, ldc, tc);
  PTB_LAUNCH_CHECK(ctx);
}

// D = F - D, rows x cols contiguous (relative_residual)
void geam_sub(ptb_context* ctx, size_t total, const double* F, double* D) {
  if (total == 0) return;
  k_geam_sub<<<ew_grid(ctx, total), 256, 0, ctx->stream>>>(total, F, D);
  PTB_LAUNCH_CHECK(ctx);
}

}  // namespace ptb
