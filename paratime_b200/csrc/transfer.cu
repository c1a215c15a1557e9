// Grid transfer between nested coarse/fine grids — restriction R and interpolation I.
//
// Reference: /root/reference/proj/src/grid.cpp
//   GridTransfer          :100-119  integer ratio per axis, equal extents
//   restrict_field        :121-139  out[j] = in[ratio*j]           (exact, pointwise)
//   fourier_interp_line   :151-177  zero-padded spectrum * (m/n), Nyquist split 1/2-1/2
//   linear_interp_line    :179-191  (1-t)*a + t*b, t = rem/r, periodic wrap
//   interpolate_field     :201-230  2D: along x within rows, then along y within columns
//
// Linear I is evaluated with explicitly rounded intrinsics in the reference's order,
// fused over both axes in one pass (bitwise equal to the reference).
// Fourier I is the same linear map written as circulant weights: for fine index
// i = q*r + rem on an axis of n coarse points,
//   out[i] = sum_d W[rem][d] * in[(q - d) mod n],
//   W[rem][d] = K(d + rem/r),  K(delta) = (1/n)[1 + 2 sum_{s=1}^{ceil(n/2)-1} cos(2 pi s delta/n)
//                                              + (n even) cos(pi delta)],
// which is exactly what the padded-spectrum construction computes (the split Nyquist
// bin contributes cos(pi delta)).  W is tabulated on the host with exact integer
// argument reduction, so the device path is a two-pass (x then y) dense stencil with
// no FFT; R(I(U)) = U holds to round-off like the reference's FFT route.
// On large 2D grids the two passes are matrix products with the dense forms
//   Mx[j][q*r + rem] = W[rem][(q - j) mod n]   (x: half = in . Mx)
//   My[q*r + rem][j] = W[rem][(q - j) mod n]   (y: out = My . half)
// issued as cuBLAS DGEMMs of one fixed shape per field, so each slice's result does not
// depend on how many slices a call (or a rank) carries.
// Default on 2D fine grids >= 256^2 (measured: faster than the DGEMMs from 256^2 up; the
// DGEMM route stays for PTB_INTERP_FFT=0) is the reference's own construction done with cuFFT (fft.cpp wraps
// FFTW): 2D D2Z of the coarse field, the zero-padded spectrum (Nyquist bins split 1/2-1/2 per
// axis as grid.cpp:161-166; the x split comes from the implicit Hermitian mirror of the
// half-spectrum), 2D Z2D on the fine grid.  The 2D DFT is separable, so this equals the
// reference's x-then-y line interpolation; plans are for one field, executed per field (same
// determinism argument as the DGEMMs).  Memory-bound instead of 2 n_c flops per output point.

#include <cmath>
#include <cstdlib>
#include <vector>

#include <cufft.h>

#include "ptb_internal.h"
#include "ptb_procrustes.h"  // gemm (cuBLAS DGEMM on the context stream)

namespace ptb {
namespace {

struct TGeom {
  int cy, cx;  // coarse points (1D: cy = 1)
  int fy, fx;  // fine points
  int ry, rx;  // ratios
};

TGeom geom(const ptb_transfer* t) {
  TGeom g{};
  if (t->coarse.dim == 1) {
    g.cy = g.fy = g.ry = 1;
    g.cx = int(t->coarse.n[0]);
    g.fx = int(t->fine.n[0]);
    g.rx = int(t->ratio[0]);
  } else {
    g.cy = int(t->coarse.n[0]);
    g.cx = int(t->coarse.n[1]);
    g.fy = int(t->fine.n[0]);
    g.fx = int(t->fine.n[1]);
    g.ry = int(t->ratio[0]);
    g.rx = int(t->ratio[1]);
  }
  return g;
}

__global__ void k_restrict(TGeom g, size_t batch, const double* __restrict__ fine, double* __restrict__ coarse) {
  const size_t nc = size_t(g.cy) * g.cx, nf = size_t(g.fy) * g.fx, total = batch * nc;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t b = e / nc, c = e - b * nc;
    const int jy = int(c / g.cx), jx = int(c - size_t(jy) * g.cx);
    coarse[e] = fine[b * nf + size_t(jy) * g.ry * g.fx + size_t(jx) * g.rx];
  }
}

// linear_interp_line value at fine index i of a periodic line (grid.cpp:184-188)
__device__ __forceinline__ double lin_at(const double* line, int stride, int n, int r, int i) {
  const int q = i / r, rem = i - q * r;
  const double a = line[size_t(q) * stride];
  if (r == 1) return a;
  const double b = line[size_t((q + 1) % n) * stride];
  const double t = double(rem) / double(r);
  return __dadd_rn(__dmul_rn(__dsub_rn(1.0, t), a), __dmul_rn(t, b));
}

// 2D (or 1D with cy = 1) linear interpolation, x then y, fused.
__global__ void k_interp_linear(TGeom g, size_t batch, const double* __restrict__ coarse, double* __restrict__ fine) {
  const size_t nc = size_t(g.cy) * g.cx, nf = size_t(g.fy) * g.fx, total = batch * nf;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t b = e / nf, f = e - b * nf;
    const int iy = int(f / g.fx), ix = int(f - size_t(iy) * g.fx);
    const double* C = coarse + b * nc;
    const int qy = iy / g.ry, remy = iy - qy * g.ry;
    const double h0 = lin_at(C + size_t(qy) * g.cx, 1, g.cx, g.rx, ix);
    double v = h0;
    if (g.ry > 1) {
      const double h1 = lin_at(C + size_t((qy + 1) % g.cy) * g.cx, 1, g.cx, g.rx, ix);
      const double t = double(remy) / double(g.ry);
      v = __dadd_rn(__dmul_rn(__dsub_rn(1.0, t), h0), __dmul_rn(t, h1));
    }
    fine[e] = v;
  }
}

// linear I at the coarse nodes (fine index r*j), same arithmetic as k_interp_linear
__global__ void k_interp_linear_nodes(TGeom g, size_t batch, const double* __restrict__ coarse,
                                      double* __restrict__ out) {
  const size_t nc = size_t(g.cy) * g.cx, total = batch * nc;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t b = e / nc;
    const int p = int(e - b * nc);
    const int jy = p / g.cx, jx = p - jy * g.cx;
    const double* C = coarse + b * nc;
    const int ix = jx * g.rx;
    const double h0 = lin_at(C + size_t(jy) * g.cx, 1, g.cx, g.rx, ix);
    double v = h0;
    if (g.ry > 1) {
      const double h1 = lin_at(C + size_t((jy + 1) % g.cy) * g.cx, 1, g.cx, g.rx, ix);
      const double t = 0.0;
      v = __dadd_rn(__dmul_rn(__dsub_rn(1.0, t), h0), __dmul_rn(t, h1));
    }
    out[e] = v;
  }
}

// Fourier pass along x: in (rows x n) -> out (rows x n*r), weights W[r][n]
__global__ void k_fourier_x(int rows, int n, int r, size_t batch, const double* __restrict__ w,
                            const double* __restrict__ in, double* __restrict__ out) {
  const size_t m = size_t(n) * r, total = batch * rows * m;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t line = e / m;
    const int i = int(e - line * m);
    const int q = i / r, rem = i - q * r;
    const double* L = in + line * n;
    const double* Wr = w + size_t(rem) * n;
    double acc = 0.0;
    int idx = q;
    for (int d = 0; d < n; ++d) {
      acc = fma(Wr[d], L[idx], acc);
      idx = idx == 0 ? n - 1 : idx - 1;
    }
    out[e] = acc;
  }
}

// Fourier pass along y: in (n x cols) -> out (n*r x cols)
__global__ void k_fourier_y(int n, int cols, int r, size_t batch, const double* __restrict__ w,
                            const double* __restrict__ in, double* __restrict__ out) {
  const size_t m = size_t(n) * r, plane_in = size_t(n) * cols, plane_out = m * cols;
  const size_t total = batch * plane_out;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t b = e / plane_out, f = e - b * plane_out;
    const int i = int(f / cols), x = int(f - size_t(i) * cols);
    const int q = i / r, rem = i - q * r;
    const double* P = in + b * plane_in + x;
    const double* Wr = w + size_t(rem) * n;
    double acc = 0.0;
    int idx = q;
    for (int d = 0; d < n; ++d) {
      acc = fma(Wr[d], P[size_t(idx) * cols], acc);
      idx = idx == 0 ? n - 1 : idx - 1;
    }
    out[e] = acc;
  }
}

__global__ void k_copy(size_t total, const double* in, double* out) {
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x)
    out[e] = in[e];
}

unsigned blocks_for(ptb_context* ctx, size_t total) {
  const size_t want = (total + 255) / 256;
  return unsigned(std::max<size_t>(1, std::min<size_t>(want, size_t(ctx->num_sms) * 32)));
}

// W[rem][d] = K(d + rem/r) on an axis of n coarse points, ratio r.
std::vector<double> fourier_weights(int n, int r) {
  std::vector<double> w(size_t(n) * r);
  const long long nr = (long long)n * r;
  const int smax = (n % 2 == 0) ? n / 2 - 1 : (n - 1) / 2;
  for (int rem = 0; rem < r; ++rem)
    for (int d = 0; d < n; ++d) {
      if (rem == 0) {  // K(integer d) = delta(d) exactly: the interpolant passes through the nodes
        w[size_t(d)] = d == 0 ? 1.0 : 0.0;
        continue;
      }
      const long long num = (long long)d * r + rem;  // delta = num / r
      long double acc = 1.0L;
      for (int s = 1; s <= smax; ++s) {
        const long long ph = (s * num) % nr;  // s*delta/n = ph / (n r) mod 1
        acc += 2.0L * std::cos(2.0L * 3.14159265358979323846264338327950288L * (long double)ph / (long double)nr);
      }
      if (n % 2 == 0) {
        const long long ph = num % (2LL * r);  // cos(pi delta) = cos(pi num / r), period 2r in num
        acc += std::cos(3.14159265358979323846264338327950288L * (long double)ph / (long double)r);
      }
      w[size_t(rem) * n + d] = double(acc / (long double)n);
    }
  return w;
}

}  // namespace

void transfer_init(ptb_transfer* t) {
  if (t->kind != PTB_INTERP_FOURIER) return;
  const TGeom g = geom(t);
  auto upload = [&](int n, int r) -> double* {
    if (r == 1) return nullptr;
    const std::vector<double> w = fourier_weights(n, r);
    double* d = nullptr;
    PTB_CUDA_CHECK(cudaMalloc(&d, w.size() * sizeof(double)));
    PTB_CUDA_CHECK(cudaMemcpy(d, w.data(), w.size() * sizeof(double), cudaMemcpyHostToDevice));
    return d;
  };
  t->wx = upload(g.cx, g.rx);
  if (t->coarse.dim == 2) t->wy = upload(g.cy, g.ry);
}

void transfer_release(ptb_transfer* t) {
  if (t->fft_fwd) cufftDestroy(cufftHandle(t->fft_fwd));
  if (t->fft_inv) cufftDestroy(cufftHandle(t->fft_inv));
  t->fft_fwd = t->fft_inv = 0;
}

void restrict_fields(ptb_transfer* t, size_t batch, const double* fine, double* coarse) {
  ptb_context* ctx = t->ctx;
  const TGeom g = geom(t);
  const size_t total = batch * size_t(g.cy) * g.cx;
  if (total == 0) return;
  k_restrict<<<blocks_for(ctx, total), 256, 0, ctx->stream>>>(g, batch, fine, coarse);
  PTB_LAUNCH_CHECK(ctx);
}

namespace {
// dense circulant matrix of one axis: rows x cols row-major, TRANSPOSED selects the x form
std::vector<double> dense_axis(int n, int r, bool x_form) {
  const std::vector<double> w = fourier_weights(n, r);
  const size_t m = size_t(n) * r;
  std::vector<double> d(m * n);
  for (size_t i = 0; i < m; ++i) {
    const int q = int(i / r), rem = int(i % r);
    for (int j = 0; j < n; ++j) {
      const double v = w[size_t(rem) * n + size_t(((q - j) % n + n) % n)];
      if (x_form)
        d[size_t(j) * m + i] = v;  // Mx[j][i]
      else
        d[i * n + size_t(j)] = v;  // My[i][j]
    }
  }
  return d;
}

bool use_gemm(const TGeom& g) {
  static const int env = [] {
    const char* e = std::getenv("PTB_INTERP_GEMM");
    return e ? std::atoi(e) : -1;
  }();
  if (env == 0) return false;
  const bool ok = g.cy > 1 && g.rx > 1 && g.ry > 1;
  return ok && (env == 1 || size_t(g.fy) * g.fx >= size_t(512) * 512);
}

__global__ void k_pad_spectrum(int cy, int cx, int fy, int fx, double scale, const double2* __restrict__ in_all,
                               double2* __restrict__ out_all) {
  const int hc = cx / 2 + 1, hf = fx / 2 + 1;
  const size_t total = size_t(fy) * hf;
  const double2* __restrict__ in = in_all + size_t(blockIdx.y) * cy * hc;
  double2* __restrict__ out = out_all + size_t(blockIdx.y) * total;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const int ky = int(e / hf), kx = int(e - size_t(ky) * hf);
    double2 v = make_double2(0.0, 0.0);
    // source row: fine row ky <-> signed frequency sy (coarse row sy mod cy)
    int sy;
    double wgt = scale;
    if (ky < (cy + 1) / 2) {
      sy = ky;
    } else if (ky > fy - (cy + 1) / 2) {
      sy = ky - fy + cy;
    } else if (cy % 2 == 0 && (ky == cy / 2 || ky == fy - cy / 2)) {
      sy = cy / 2;  // Nyquist row split between +cy/2 and -cy/2
      wgt *= 0.5;
    } else {
      sy = -1;
    }
    if (sy >= 0 && kx <= cx / 2) {
      if (cx % 2 == 0 && kx == cx / 2) wgt *= 0.5;  // mirror (implicit) carries the other half
      const double2 f = in[size_t(sy) * hc + kx];
      v = make_double2(f.x * wgt, f.y * wgt);
    }
    out[e] = v;
  }
}

void check_fft(cufftResult r, const char* what) {
  if (r != CUFFT_SUCCESS) fail(PTB_CUDA, std::string("cuFFT ") + what + " failed (" + std::to_string(int(r)) + ")");
}

bool use_fft(const TGeom& g) {
  static const int env = [] {
    const char* e = std::getenv("PTB_INTERP_FFT");
    return e ? std::atoi(e) : -1;
  }();
  if (env == 0) return false;
  const bool ok = g.cy > 1 && g.rx > 1 && g.ry > 1;
  return ok && (env == 1 || size_t(g.fy) * g.fx >= size_t(256) * 256);
}

constexpr int FFT_CHUNK = 8;  // fields per cuFFT execution (fixed: a partial chunk is padded)

void interpolate_fft(ptb_transfer* t, const TGeom& g, size_t batch, const double* coarse, double* fine) {
  ptb_context* ctx = t->ctx;
  cudaStream_t st = ctx->stream;
  const int hc = g.cx / 2 + 1, hf = g.fx / 2 + 1;
  const size_t nc = size_t(g.cy) * g.cx, nf = size_t(g.fy) * g.fx;
  const size_t sc_n = size_t(g.cy) * hc, sf_n = size_t(g.fy) * hf;
  if (!t->fft_fwd) {
    cufftHandle f = 0, b = 0;
    int nC[2] = {g.cy, g.cx}, nF[2] = {g.fy, g.fx};
    check_fft(cufftPlanMany(&f, 2, nC, nullptr, 1, int(nc), nullptr, 1, int(sc_n), CUFFT_D2Z, FFT_CHUNK),
              "plan D2Z");
    check_fft(cufftPlanMany(&b, 2, nF, nullptr, 1, int(sf_n), nullptr, 1, int(nf), CUFFT_Z2D, FFT_CHUNK),
              "plan Z2D");
    t->fft_fwd = int(f);
    t->fft_inv = int(b);
  }
  const cufftHandle f = cufftHandle(t->fft_fwd), b = cufftHandle(t->fft_inv);
  check_fft(cufftSetStream(f, st), "set stream");
  check_fft(cufftSetStream(b, st), "set stream");
  double2* sc = static_cast<double2*>(t->spec_c.get(FFT_CHUNK * sc_n * sizeof(double2)));
  double2* sf = static_cast<double2*>(t->spec_f.get(FFT_CHUNK * sf_n * sizeof(double2)));
  const double scale = 1.0 / double(nc);
  for (size_t i0 = 0; i0 < batch; i0 += FFT_CHUNK) {
    const size_t cnt = std::min<size_t>(FFT_CHUNK, batch - i0);
    const double* in = coarse + i0 * nc;
    double* out = fine + i0 * nf;
    double* stage_in = nullptr;
    double* stage_out = nullptr;
    if (cnt < FFT_CHUNK) {  // partial chunk: same plan on a zero-padded staging copy
      stage_in = static_cast<double*>(ctx->scratch[2].get(FFT_CHUNK * nc * sizeof(double)));
      stage_out = static_cast<double*>(ctx->scratch[3].get(FFT_CHUNK * nf * sizeof(double)));
      PTB_CUDA_CHECK(cudaMemsetAsync(stage_in, 0, FFT_CHUNK * nc * sizeof(double), st));
      PTB_CUDA_CHECK(cudaMemcpyAsync(stage_in, in, cnt * nc * sizeof(double), cudaMemcpyDeviceToDevice, st));
      in = stage_in;
    }
    // cuFFT's D2Z takes its input as non-const
    check_fft(cufftExecD2Z(f, const_cast<double*>(in), reinterpret_cast<cufftDoubleComplex*>(sc)), "exec D2Z");
    k_pad_spectrum<<<dim3(blocks_for(ctx, sf_n), FFT_CHUNK), 256, 0, st>>>(g.cy, g.cx, g.fy, g.fx, scale, sc, sf);
    PTB_LAUNCH_CHECK(ctx);
    check_fft(cufftExecZ2D(b, reinterpret_cast<cufftDoubleComplex*>(sf), stage_out ? stage_out : out), "exec Z2D");
    ctx->launches.fetch_add(2, std::memory_order_relaxed);
    if (stage_out)
      PTB_CUDA_CHECK(cudaMemcpyAsync(out, stage_out, cnt * nf * sizeof(double), cudaMemcpyDeviceToDevice, st));
  }
}

void interpolate_gemm(ptb_transfer* t, const TGeom& g, size_t batch, const double* coarse, double* fine) {
  ptb_context* ctx = t->ctx;
  if (!t->mx) {
    const std::vector<double> mx = dense_axis(g.cx, g.rx, true), my = dense_axis(g.cy, g.ry, false);
    PTB_CUDA_CHECK(cudaMalloc(&t->mx, mx.size() * sizeof(double)));
    PTB_CUDA_CHECK(cudaMalloc(&t->my, my.size() * sizeof(double)));
    PTB_CUDA_CHECK(cudaMemcpy(t->mx, mx.data(), mx.size() * sizeof(double), cudaMemcpyHostToDevice));
    PTB_CUDA_CHECK(cudaMemcpy(t->my, my.data(), my.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  const size_t nc = size_t(g.cy) * g.cx, nh = size_t(g.cy) * g.fx, nf = size_t(g.fy) * g.fx;
  double* half = static_cast<double*>(ctx->scratch[3].get(batch * nh * sizeof(double)));
  // row-major products as column-major GEMMs: half_b^T (fx x cy) = Mx^T (fx x cx) . in_b^T (cx x cy)
  for (size_t b = 0; b < batch; ++b)
    gemm(ctx, false, false, g.fx, g.cy, g.cx, 1.0, t->mx, g.fx, coarse + b * nc, g.cx, 0.0, half + b * nh, g.fx);
  // out_b^T (fx x fy) = half_b^T (fx x cy) . My^T (cy x fy)
  for (size_t b = 0; b < batch; ++b)
    gemm(ctx, false, false, g.fx, g.fy, g.cy, 1.0, half + b * nh, g.fx, t->my, g.cy, 0.0, fine + b * nf, g.fx);
}
}  // namespace

void interpolate_fields(ptb_transfer* t, size_t batch, const double* coarse, double* fine) {
  ptb_context* ctx = t->ctx;
  const TGeom g = geom(t);
  const size_t nf = size_t(g.fy) * g.fx;
  if (batch == 0) return;
  if (t->kind == PTB_INTERP_LINEAR || (g.rx == 1 && g.ry == 1)) {
    k_interp_linear<<<blocks_for(ctx, batch * nf), 256, 0, ctx->stream>>>(g, batch, coarse, fine);
    PTB_LAUNCH_CHECK(ctx);
    return;
  }
  if (use_fft(g)) {
    interpolate_fft(t, g, batch, coarse, fine);
    return;
  }
  if (use_gemm(g)) {
    interpolate_gemm(t, g, batch, coarse, fine);
    return;
  }
  // Fourier: x pass into scratch (cy x fx), then y pass (fy x fx)
  const double* src = coarse;
  double* half = nullptr;
  if (g.rx > 1) {
    const size_t hn = batch * size_t(g.cy) * g.fx;
    half = (g.ry > 1) ? static_cast<double*>(ctx->scratch[3].get(hn * sizeof(double))) : fine;
    k_fourier_x<<<blocks_for(ctx, hn), 256, 0, ctx->stream>>>(g.cy, g.cx, g.rx, batch, t->wx, coarse, half);
    PTB_LAUNCH_CHECK(ctx);
    src = half;
  }
  if (g.ry > 1) {
    k_fourier_y<<<blocks_for(ctx, batch * nf), 256, 0, ctx->stream>>>(g.cy, g.fx, g.ry, batch, t->wy, src, fine);
    PTB_LAUNCH_CHECK(ctx);
  } else if (g.rx == 1) {
    k_copy<<<blocks_for(ctx, batch * nf), 256, 0, ctx->stream>>>(batch * nf, coarse, fine);
    PTB_LAUNCH_CHECK(ctx);
  }
}

void interpolate_at_coarse_nodes(ptb_transfer* t, size_t batch, const double* coarse, double* out) {
  ptb_context* ctx = t->ctx;
  const TGeom g = geom(t);
  const size_t nc = size_t(g.cy) * g.cx;
  if (batch == 0) return;
  if (t->kind == PTB_INTERP_LINEAR || (g.rx == 1 && g.ry == 1)) {
    k_interp_linear_nodes<<<blocks_for(ctx, batch * nc), 256, 0, ctx->stream>>>(g, batch, coarse, out);
    PTB_LAUNCH_CHECK(ctx);
    return;
  }
  // Fourier: W[0][d] = delta(d) exactly (fourier_weights), so both passes reproduce the node
  // values bit for bit (adding exact zeros) for finite data, and so does the dense GEMM route:
  // R(I(d)) = d.  (Non-finite d: the coarse step that follows turns the state all-NaN, as the
  // reference's nan_state does, so NaN spreading inside I is not observable.)
  const size_t total = batch * nc;
  k_copy<<<blocks_for(ctx, total), 256, 0, ctx->stream>>>(total, coarse, out);
  PTB_LAUNCH_CHECK(ctx);
}

}  // namespace ptb
