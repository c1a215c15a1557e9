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
// On 2D fine grids >= 256^2 with power-of-two coarse axes (32..256 points) the same map runs as
// warp FFTs (k_fourier_fft_x / k_fourier_fft_y below): O(n log n) per line instead of n taps per
// output point, phase 0 copied so the nodes stay exact.  Every field is transformed on its own,
// so a slice's result never depends on how many slices a call or a rank carries.

#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <vector>

#include "ptb_internal.h"

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
  t->spec_c.release();
  t->nodes_half.release();
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
// ------------------------------------------------------------------ Fourier I by warp FFTs
//
// fourier_interp_line (grid.cpp:151-177) maps n coarse values x to m = n r fine values
//   out[i] = (1/n) sum_k X_k e^{2 pi i kappa(k) i / m},   X = DFT_n(x),
// kappa(k) the signed frequency, the Nyquist bin k = n/2 split half/half between +-n/2.  At
// i = q r + s this is a length-n inverse DFT of the phase-shifted spectrum
//   Y^(s)_k = X_k e^{2 pi i kappa s / m}   (Nyquist: X_{n/2} cos(pi s / r)),
// so one forward DFT_n and r-1 inverse DFT_n per line give all r phases, and s = 0 is the
// line itself (the interpolant passes through the nodes exactly, as the circulant weights
// do).  Y^(s) is Hermitian, so two phases share one complex inverse transform (real part:
// phase s1, imaginary part: phase s2).  n = 32 E (E <= 8) points live in one warp, lane L
// holding x[L + 32 e]: an E-point DFT in registers, a twiddle, then a 32-point DFT across the
// lanes by shuffles (DIF, bit-reversed lane order); the inverse runs the same network backwards
// (DIT), so the spectrum is never permuted.  x pass: a warp per coarse row, the r n outputs
// staged in shared memory phase-major and written as one contiguous row; y pass: a CTA per 16
// adjacent fine columns (128-byte rows), a warp per column.  Optionally fused with the fine
// combine: out = base + I(coarse).

__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {  // a * conj(b)
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }

constexpr int bitrev_c(int v, int bits) {
  int r = 0;
  for (int i = 0; i < bits; ++i) r |= ((v >> i) & 1) << (bits - 1 - i);
  return r;
}
constexpr int log2_c(int v) { return v <= 1 ? 0 : 1 + log2_c(v / 2); }

// e^{-2 pi i p / q} for the compile-time register DFTs (q <= 8)
__device__ __forceinline__ double2 tw_const(int p, int q, bool inv) {
  constexpr double h = 0.70710678118654752440;
  double2 w;
  switch ((p * 8) / q) {  // angle in units of pi/4
    case 0: w = make_double2(1.0, 0.0); break;
    case 1: w = make_double2(h, -h); break;
    case 2: w = make_double2(0.0, -1.0); break;
    default: w = make_double2(-h, -h); break;  // 3 pi / 4
  }
  if (inv) w.y = -w.y;
  return w;
}

// E-point DFT in registers, natural order in and out (unnormalised; INV: e^{+})
template <int E, bool INV>
__device__ __forceinline__ void dft_reg(double2 (&v)[E]) {
  if constexpr (E > 1) {
#pragma unroll
    for (int h = E / 2; h >= 1; h /= 2)
#pragma unroll
      for (int i = 0; i < E; ++i)
        if ((i & h) == 0) {
          const double2 a = v[i], b = v[i + h];
          v[i] = cadd(a, b);
          const int p = i & (h - 1);
          v[i + h] = p == 0 ? csub(a, b) : cmul(csub(a, b), tw_const(p, 2 * h, INV));
        }
    double2 t[E];
#pragma unroll
    for (int i = 0; i < E; ++i) t[bitrev_c(i, log2_c(E))] = v[i];
#pragma unroll
    for (int i = 0; i < E; ++i) v[i] = t[i];
  }
}

__device__ __forceinline__ double2 shfl_xor2(double2 v, int m) {
  return make_double2(__shfl_xor_sync(0xffffffffu, v.x, m), __shfl_xor_sync(0xffffffffu, v.y, m));
}

// per-lane twiddles of the transforms: lane network w_{2h}^{lane & (h-1)} (h = 16 >> st) and the
// register-to-lane twiddle w_n^{lane k1}
template <int E>
struct LaneTw {
  double2 net[5];
  double2 mid[E];
  __device__ void init(int lane) {
#pragma unroll
    for (int st = 0; st < 5; ++st) {
      const int h = 16 >> st;
      double sn, cs;
      sincospi(-double(lane & (h - 1)) / double(h), &sn, &cs);  // e^{-2 pi i p / (2h)}
      net[st] = make_double2(cs, sn);
    }
#pragma unroll
    for (int k1 = 0; k1 < E; ++k1) {
      double sn, cs;
      sincospi(-2.0 * double(lane * k1) / double(32 * E), &sn, &cs);
      mid[k1] = make_double2(cs, sn);
    }
  }
};

// forward DFT of n = 32 E points: in lane L slot e = x[L + 32 e]; out lane L slot k1 = X[k1 + E rev5(L)]
template <int E>
__device__ __forceinline__ void fft_fwd(double2 (&v)[E], const LaneTw<E>& tw, int lane) {
  dft_reg<E, false>(v);
#pragma unroll
  for (int k1 = 1; k1 < E; ++k1) v[k1] = cmul(v[k1], tw.mid[k1]);
#pragma unroll
  for (int st = 0; st < 5; ++st) {
    const int h = 16 >> st;
    const bool up = lane & h;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const double2 o = shfl_xor2(v[e], h);
      v[e] = up ? cmul(csub(o, v[e]), tw.net[st]) : cadd(v[e], o);
    }
  }
}

// inverse (unnormalised, e^{+}): in lane L slot k1 = Z[k1 + E rev5(L)]; out lane L slot e = z[L + 32 e]
template <int E>
__device__ __forceinline__ void fft_inv(double2 (&v)[E], const LaneTw<E>& tw, int lane) {
#pragma unroll
  for (int st = 4; st >= 0; --st) {
    const int h = 16 >> st;
    const bool up = lane & h;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      if (up) v[e] = cmulc(v[e], tw.net[st]);
      const double2 o = shfl_xor2(v[e], h);
      v[e] = up ? csub(o, v[e]) : cadd(v[e], o);
    }
  }
#pragma unroll
  for (int k1 = 1; k1 < E; ++k1) v[k1] = cmulc(v[k1], tw.mid[k1]);
  dft_reg<E, true>(v);
}

// The r phases of one line.  Per lane: the spectrum X (layout of fft_fwd) and the unit phase
// steps e^{2 pi i kappa / m} of its bins; emit(s, e, value) receives out[(L + 32 e) r + s].
template <int E, typename Emit>
__device__ __forceinline__ void interp_line(double2 (&x)[E], int r, const LaneTw<E>& tw, const double2 (&step)[E],
                                            int lane, Emit&& emit) {
  constexpr int n = 32 * E;
#pragma unroll
  for (int e = 0; e < E; ++e) emit(0, e, x[e].x);  // phase 0: the nodes themselves
  fft_fwd<E>(x, tw, lane);
  const double inv_n = 1.0 / double(n);  // power of two: exact
  // Nyquist bin (k = n/2): lane 1 (rev5(1) = 16), slot 0
  const bool nyq_lane = lane == 1;
  double2 ph[E];  // e^{2 pi i kappa s / m} for the current s
#pragma unroll
  for (int e = 0; e < E; ++e) ph[e] = make_double2(1.0, 0.0);
  for (int s1 = 1; s1 < r; s1 += 2) {
    const int s2 = s1 + 1;
    double2 z[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const double2 p1 = cmul(ph[e], step[e]);
      const double2 p2 = cmul(p1, step[e]);
      ph[e] = p2;
      double2 a = p1, b = s2 < r ? p2 : make_double2(0.0, 0.0);
      if (nyq_lane && e == 0) {  // split Nyquist: X_{n/2} cos(pi s / r)
        a = make_double2(a.x, 0.0);
        b = make_double2(b.x, 0.0);
      }
      const double2 y1 = cmul(x[e], a), y2 = cmul(x[e], b);
      z[e] = make_double2((y1.x - y2.y) * inv_n, (y1.y + y2.x) * inv_n);  // (Y1 + i Y2) / n
    }
    fft_inv<E>(z, tw, lane);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      emit(s1, e, z[e].x);
      if (s2 < r) emit(s2, e, z[e].y);
    }
  }
}

// unit phase steps of the bins a lane holds after fft_fwd: e^{2 pi i kappa / m}
template <int E>
__device__ __forceinline__ void phase_steps(double2 (&step)[E], int lane, int r) {
  constexpr int n = 32 * E;
  const int k2 = __brev(unsigned(lane)) >> 27;
#pragma unroll
  for (int k1 = 0; k1 < E; ++k1) {
    const int k = k1 + E * k2;
    const int kap = k <= n / 2 ? k : k - n;  // Nyquist (k = n/2): +n/2, only its real part is used
    double sn, cs;
    sincospi(2.0 * double(kap) / double(n * r), &sn, &cs);
    step[k1] = make_double2(cs, sn);
  }
}

constexpr int FX_WARPS = 4;

// x pass: rows of `lines` coarse lines (length n = 32E, row stride n) -> rows of n r values
template <int E>
__global__ void __launch_bounds__(32 * FX_WARPS) k_fourier_fft_x(size_t lines, int r, const double* __restrict__ in,
                                                                   double* __restrict__ out) {
  constexpr int n = 32 * E, PITCH = n + 4;  // phase-major staging, pitch n+4: conflict-free row reads
  extern __shared__ double stage_x[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* sb = stage_x + size_t(warp) * r * PITCH;
  LaneTw<E> tw;
  tw.init(lane);
  double2 step[E];
  phase_steps<E>(step, lane, r);
  const size_t m = size_t(n) * r;
  for (size_t line = size_t(blockIdx.x) * FX_WARPS + warp; line < lines; line += size_t(gridDim.x) * FX_WARPS) {
    double2 x[E];
#pragma unroll
    for (int e = 0; e < E; ++e) x[e] = make_double2(in[line * n + lane + 32 * e], 0.0);
    interp_line<E>(x, r, tw, step, lane, [&](int s, int e, double val) { sb[s * PITCH + lane + 32 * e] = val; });
    __syncwarp();
    double* o = out + line * m;
    for (int i = lane; i < int(m); i += 32) o[i] = sb[(i % r) * PITCH + i / r];
    __syncwarp();
  }
}

constexpr int FY_COLS = 8;  // columns (= warps) per CTA: 64-byte row segments, <= 255 registers

__device__ __forceinline__ void cp_async16_y(double* smem_dst, const double* gmem_src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit_y() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_y() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// y pass: plane (n x w) per field -> (n r x w), columns [16 blockIdx.x, +16) of field blockIdx.y;
// out = base + I (base nullable, may alias out)
template <int E>
__global__ void __launch_bounds__(32 * FY_COLS) k_fourier_fft_y(int w, int r, const double* __restrict__ in,
                                                                  const double* base, double* out) {
  constexpr int n = 32 * E, IP = n + 1, OP = FY_COLS + 1;
  extern __shared__ __align__(16) double smem_y[];
  double* tin = smem_y;                  // [FY_COLS][n + 1]
  double* tout = smem_y + FY_COLS * IP;  // [2][n][FY_COLS + 1]: one phase pair
  double* bsm = tout + 2 * n * OP + 1;   // [2 buffers][2 phases][n][FY_COLS]: base rows (16-byte aligned)
  bsm += (reinterpret_cast<uintptr_t>(bsm) & 15) ? 1 : 0;
  const int tid = threadIdx.x, lane = tid & 31, col = tid >> 5;
  const int x0 = blockIdx.x * FY_COLS;
  const double* src = in + size_t(blockIdx.y) * n * w + x0;
  const size_t off = size_t(blockIdx.y) * n * r * w + x0;
  {  // the plane's coarse columns: all loads of a thread in flight together, then the stores
    constexpr int PER = n / 32;  // = n * FY_COLS / (32 * FY_COLS)
    double t[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int i = tid + e * 32 * FY_COLS;
      t[e] = src[size_t(i / FY_COLS) * w + i % FY_COLS];
    }
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int i = tid + e * 32 * FY_COLS;
      tin[(i % FY_COLS) * IP + i / FY_COLS] = t[e];
    }
  }
  __syncthreads();
  // phase 0: the coarse rows themselves (loads first, as below)
  {
    constexpr int PER = n / 32;
    double bv[PER];
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int i = tid + e * 32 * FY_COLS, q = i / FY_COLS, c = i % FY_COLS;
      bv[e] = base ? base[off + size_t(q) * r * w + c] : 0.0;
    }
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int i = tid + e * 32 * FY_COLS, q = i / FY_COLS, c = i % FY_COLS;
      out[off + size_t(q) * r * w + c] = bv[e] + tin[c * IP + q];
    }
  }
  // base rows q r + s1 + {0, 1} (8 columns each) of a phase pair -> bsm[b], 16-byte cp.async
  auto prefetch = [&](int b, int s1) {
    double* d = bsm + b * (2 * n * FY_COLS);
    for (int k = tid; k < n * FY_COLS; k += 32 * FY_COLS) {  // 2n rows x 4 chunks
      const int qq = k / (FY_COLS / 2), ch = k % (FY_COLS / 2), slot = qq / n, q = qq % n;
      if (s1 + slot < r) cp_async16_y(d + qq * FY_COLS + 2 * ch, base + off + (size_t(q) * r + s1 + slot) * w + 2 * ch);
    }
  };
  int buf = 0;
  if (base && r > 1) prefetch(0, 1);
  cp_async_commit_y();
  LaneTw<E> tw;
  tw.init(lane);
  double2 step[E];
  phase_steps<E>(step, lane, r);
  double2 x[E];
#pragma unroll
  for (int e = 0; e < E; ++e) x[e] = make_double2(tin[col * IP + lane + 32 * e], 0.0);
  fft_fwd<E>(x, tw, lane);
  const double inv_n = 1.0 / double(n);
  const bool nyq_lane = lane == 1;
  double2 ph[E];
#pragma unroll
  for (int e = 0; e < E; ++e) ph[e] = make_double2(1.0, 0.0);
  for (int s1 = 1; s1 < r; s1 += 2) {
    const int s2 = s1 + 1, cnt = s2 < r ? 2 : 1;
    double2 z[E];
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const double2 p1 = cmul(ph[e], step[e]);
      const double2 p2 = cmul(p1, step[e]);
      ph[e] = p2;
      double2 a = p1, b = cnt == 2 ? p2 : make_double2(0.0, 0.0);
      if (nyq_lane && e == 0) {
        a = make_double2(a.x, 0.0);
        b = make_double2(b.x, 0.0);
      }
      const double2 y1 = cmul(x[e], a), y2 = cmul(x[e], b);
      z[e] = make_double2((y1.x - y2.y) * inv_n, (y1.y + y2.x) * inv_n);
    }
    fft_inv<E>(z, tw, lane);
#pragma unroll
    for (int e = 0; e < E; ++e) {
      tout[(lane + 32 * e) * OP + col] = z[e].x;
      tout[(n + lane + 32 * e) * OP + col] = z[e].y;
    }
    // the next phase pair's base rows start moving while this pair's are added and stored
    if (base && s1 + 2 < r) prefetch(buf ^ 1, s1 + 2);
    cp_async_commit_y();
    cp_async_wait_y<1>();
    __syncthreads();  // tout and this pair's base rows complete
    constexpr int PER = 2 * n * FY_COLS / (32 * FY_COLS);  // = 2n/32 elements per thread
    const double* bs = bsm + buf * (2 * n * FY_COLS);
#pragma unroll
    for (int e = 0; e < PER; ++e) {
      const int i = tid + e * 32 * FY_COLS, c = i % FY_COLS, qq = i / FY_COLS, slot = qq / n, q = qq % n;
      if (slot < cnt)
        out[off + (size_t(q) * r + s1 + slot) * w + c] = (base ? bs[qq * FY_COLS + c] : 0.0) + tout[(slot * n + q) * OP + c];
    }
    __syncthreads();
    buf ^= 1;
  }
}

// E = n / 32 for the warp FFT route, 0 when n is not 32, 64, 128 or 256
int fft_e(int n) { return (n == 32 || n == 64 || n == 128 || n == 256) ? n / 32 : 0; }

bool use_fft(const TGeom& g) {
  static const int env = [] {
    const char* e = std::getenv("PTB_INTERP_FFT");
    return e ? std::atoi(e) : -1;
  }();
  if (env == 0) return false;
  const bool ok = g.cy > 1 && g.rx > 1 && g.ry > 1 && fft_e(g.cx) && fft_e(g.cy) && g.fx % FY_COLS == 0;
  return ok && (env == 1 || size_t(g.fy) * g.fx >= size_t(256) * 256);
}

template <int E>
void launch_fft_x(ptb_context* ctx, size_t lines, int r, const double* in, double* out) {
  const size_t smem = size_t(FX_WARPS) * r * (32 * E + 4) * sizeof(double);
  PTB_CUDA_CHECK(cudaFuncSetAttribute(k_fourier_fft_x<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  const unsigned grid = unsigned(std::min<size_t>((lines + FX_WARPS - 1) / FX_WARPS, size_t(ctx->num_sms) * 16));
  k_fourier_fft_x<E><<<grid, 32 * FX_WARPS, smem, ctx->stream>>>(lines, r, in, out);
  PTB_LAUNCH_CHECK(ctx);
}

template <int E>
void launch_fft_y(ptb_context* ctx, size_t planes, int w, int r, const double* in, const double* base, double* out) {
  constexpr int n = 32 * E;
  const size_t smem =
      (size_t(FY_COLS) * (n + 1) + size_t(2) * n * (FY_COLS + 1) + 2 + size_t(2) * 2 * n * FY_COLS) * sizeof(double);
  PTB_CUDA_CHECK(cudaFuncSetAttribute(k_fourier_fft_y<E>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  for (size_t p0 = 0; p0 < planes; p0 += 65535) {  // gridDim.y limit
    const size_t np = std::min<size_t>(65535, planes - p0);
    k_fourier_fft_y<E><<<dim3(unsigned(w / FY_COLS), unsigned(np)), 32 * FY_COLS, smem, ctx->stream>>>(
        w, r, in + p0 * size_t(n) * w, base ? base + p0 * size_t(n) * r * w : nullptr, out + p0 * size_t(n) * r * w);
    PTB_LAUNCH_CHECK(ctx);
  }
}

// fine = [base +] I(coarse) for `batch` fields, x pass into a scratch plane, then y pass
void interpolate_fft(ptb_transfer* t, const TGeom& g, size_t batch, const double* coarse, const double* base,
                     double* fine) {
  ptb_context* ctx = t->ctx;
  double* half = static_cast<double*>(t->spec_c.get(batch * size_t(g.cy) * g.fx * sizeof(double)));
  const size_t lines = batch * size_t(g.cy);
  switch (fft_e(g.cx)) {
    case 1: launch_fft_x<1>(ctx, lines, g.rx, coarse, half); break;
    case 2: launch_fft_x<2>(ctx, lines, g.rx, coarse, half); break;
    case 4: launch_fft_x<4>(ctx, lines, g.rx, coarse, half); break;
    default: launch_fft_x<8>(ctx, lines, g.rx, coarse, half); break;
  }
  switch (fft_e(g.cy)) {
    case 1: launch_fft_y<1>(ctx, batch, g.fx, g.ry, half, base, fine); break;
    case 2: launch_fft_y<2>(ctx, batch, g.fx, g.ry, half, base, fine); break;
    case 4: launch_fft_y<4>(ctx, batch, g.fx, g.ry, half, base, fine); break;
    default: launch_fft_y<8>(ctx, batch, g.fx, g.ry, half, base, fine); break;
  }
}

__global__ void k_add_base(size_t total, const double* __restrict__ base, double* out) {
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x)
    out[e] = base[e] + out[e];
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
    interpolate_fft(t, g, batch, coarse, nullptr, fine);
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

// out = base + I(coarse): the fine combine next = fine_next + I(d) (base may alias out); fused
// into the y pass on the warp-FFT route, a separate add otherwise
void interpolate_fields_add(ptb_transfer* t, size_t batch, const double* coarse, const double* base, double* out,
                            double* scratch) {
  ptb_context* ctx = t->ctx;
  const TGeom g = geom(t);
  if (batch == 0) return;
  if (t->kind == PTB_INTERP_FOURIER && !(g.rx == 1 && g.ry == 1) && use_fft(g)) {
    interpolate_fft(t, g, batch, coarse, base, out);
    return;
  }
  const size_t total = batch * size_t(g.fy) * g.fx;
  interpolate_fields(t, batch, coarse, scratch);
  k_add_base<<<blocks_for(ctx, total), 256, 0, ctx->stream>>>(total, base, scratch);
  PTB_LAUNCH_CHECK(ctx);
  if (scratch != out) PTB_CUDA_CHECK(cudaMemcpyAsync(out, scratch, total * sizeof(double), cudaMemcpyDeviceToDevice,
                                                     ctx->stream));
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
