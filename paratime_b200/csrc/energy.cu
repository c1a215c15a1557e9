// Energy map: components Lambda, reconstruction Lambda-dagger, energies and error sums.
//
// Reference: /root/reference/proj/src/energy_map.cpp
//   stencil_coefficients   :31-44   fd2..fd8 half-stencils beta_j
//   fd_gradient_axis       :50-90   acc = sum_j beta_j (f[i+j] - f[i-j]) in j order; * (1/h)
//   spectral_gradient_axis :95-122  FFT derivative, unmatched Nyquist bin zeroed
//   to_energy_components   :137-150 [grad_0; ...; grad_{d-1}; udot/c], mean_u = sum(u)
//   from_energy_components :152-214 u_hat = -i (xi . g_hat)/|xi|^2, u_hat(0) = mean_u,
//                                    both-Nyquist bin 0; udot = c * momentum
//   energy / energy_error / l2_error :216-249
//
// Stacked layout = stack_components (procrustes.cpp:129-142): column b of a column-major
// matrix with leading dimension ld holds [grad axis 0 (N); grad axis 1 (N); momentum (N)].
// Finite-difference gradients and the momentum use explicitly rounded intrinsics in the
// reference's order (bitwise equal).  Sums use deterministic fixed-order tree reductions.

#include <cmath>
#include <vector>

#include <cstdlib>

#include "ptb_energy.h"
#include "ptb_fft.h"

namespace ptb {
namespace {

struct Beta {
  int m;
  double b[4];
};

Beta beta_of(int scheme) {
  switch (scheme) {  // energy_map.cpp:32-35
    case PTB_FD2: return Beta{1, {1.0 / 2.0, 0, 0, 0}};
    case PTB_FD4: return Beta{2, {2.0 / 3.0, -1.0 / 12.0, 0, 0}};
    case PTB_FD6: return Beta{3, {3.0 / 4.0, -3.0 / 20.0, 1.0 / 60.0, 0}};
    case PTB_FD8: return Beta{4, {4.0 / 5.0, -1.0 / 5.0, 4.0 / 105.0, -1.0 / 280.0}};
  }
  fail(PTB_INVALID_ARGUMENT, "stencil_coefficients: spectral scheme has no stencil");
}

struct Geo {
  int dim, ny, nx;  // 1D: ny = 1
  double ih[2];     // 1/h per axis (axis 0 = y in 2D, x in 1D)
};

Geo geo_of(const ptb_grid& g) {
  Geo o{};
  o.dim = g.dim;
  if (g.dim == 1) {
    o.ny = 1;
    o.nx = int(g.n[0]);
    o.ih[0] = 1.0 / g.h[0];
  } else {
    o.ny = int(g.n[0]);
    o.nx = int(g.n[1]);
    o.ih[0] = 1.0 / g.h[0];
    o.ih[1] = 1.0 / g.h[1];
  }
  return o;
}

// fd derivative of f along `axis` at flat point p (energy_map.cpp:50-90, reference order);
// DIFF: f = fa - fb evaluated per access (same rounding as a precomputed difference)
template <bool DIFF>
__device__ __forceinline__ double fd_grad(const double* fa, const double* fb, const Geo& G, const Beta& B, int axis,
                                          int p) {
  const int iy = p / G.nx, ix = p - iy * G.nx;
  double acc = 0.0;
  for (int j = 1; j <= B.m; ++j) {
    int pp, pm;
    if (G.dim == 1 || axis == 1) {
      pp = iy * G.nx + (ix + j) % G.nx;
      pm = iy * G.nx + (ix + G.nx - j) % G.nx;
    } else {
      pp = ((iy + j) % G.ny) * G.nx + ix;
      pm = ((iy + G.ny - j) % G.ny) * G.nx + ix;
    }
    const double a = DIFF ? __dsub_rn(fa[pp], fb[pp]) : fa[pp];
    const double b = DIFF ? __dsub_rn(fa[pm], fb[pm]) : fa[pm];
    acc = __dadd_rn(acc, __dmul_rn(B.b[j - 1], __dsub_rn(a, b)));
  }
  const double ih = (G.dim == 1) ? G.ih[0] : G.ih[axis];
  return __dmul_rn(acc, ih);
}

struct CompArgs {
  Geo G;
  Beta B;
  int n;  // points
  const double* u;
  const double* v;
  size_t sstride;      // state stride (u and v share it)
  const int* index;    // optional gather: state b reads source index[b]
  const double* c;
  double* out;
  size_t ld;
};

__global__ void k_components_fd(const CompArgs a, size_t batch) {
  const size_t total = batch * a.n;
  const int d = a.G.dim;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t b = e / a.n;
    const int p = int(e - b * a.n);
    const size_t src = a.index ? size_t(a.index[b]) : b;
    const double* U = a.u + src * a.sstride;
    const double* V = a.v + src * a.sstride;
    double* O = a.out + b * a.ld;
    for (int ax = 0; ax < d; ++ax) O[size_t(ax) * a.n + p] = fd_grad<false>(U, nullptr, a.G, a.B, ax, p);
    O[size_t(d) * a.n + p] = __ddiv_rn(V[p], a.c[p]);
  }
}

__global__ void k_momentum(const CompArgs a, size_t batch) {
  const size_t total = batch * a.n;
  const int d = a.G.dim;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t b = e / a.n;
    const int p = int(e - b * a.n);
    const size_t src = a.index ? size_t(a.index[b]) : b;
    a.out[b * a.ld + size_t(d) * a.n + p] = __ddiv_rn(a.v[src * a.sstride + p], a.c[p]);
  }
}

// deterministic per-state sum: one CTA per state, fixed thread->element map, tree reduce
// fixed-order block reduction: xor-butterfly inside each warp, then the T/32 warp sums by warp 0
// (two barriers instead of log2 T); the result is returned to every thread
template <int T>
__device__ double block_sum(double x) {
  static_assert(T % 32 == 0 && T <= 1024, "block size");
  __shared__ double red[T / 32];
  __shared__ double tot;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    double y = threadIdx.x < T / 32 ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
    if (threadIdx.x == 0) tot = y;
  }
  __syncthreads();
  const double r = tot;
  __syncthreads();  // red / tot are reused by the next call
  return r;
}

// mean_u partials: grid (P, batch); block p sums the points p, p + P*256, ... of its state, so
// the partial layout (and the result) depends only on n and P = state_sum_parts(n)
__global__ void __launch_bounds__(256) k_state_sum(int n, const double* f, size_t sstride, const int* index,
                                                   double* part) {
  const size_t b = blockIdx.y;
  const size_t src = index ? size_t(index[b]) : b;
  const double* F = f + src * sstride;
  // four independent accumulators (four loads in flight per thread), combined in fixed order
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const int step = gridDim.x * 256;
  int i = blockIdx.x * 256 + threadIdx.x;
  for (; i + 3 * step < n; i += 4 * step) {
    a0 += F[i];
    a1 += F[i + step];
    a2 += F[i + 2 * step];
    a3 += F[i + 3 * step];
  }
  for (; i < n; i += step) a0 += F[i];
  const double s = block_sum<256>((a0 + a1) + (a2 + a3));
  if (threadIdx.x == 0) part[b * gridDim.x + blockIdx.x] = s;
}

__global__ void k_state_sum_final(size_t batch, int P, const double* part, double* out) {
  for (size_t b = blockIdx.x * size_t(blockDim.x) + threadIdx.x; b < batch; b += size_t(gridDim.x) * blockDim.x) {
    double acc = 0.0;
    for (int q = 0; q < P; ++q) acc += part[b * P + q];
    out[b] = acc;
  }
}

// The sweep step's z = Y^T Lambda(w) for ONE coarse state without materialising Lambda(w):
// block (j, p), j < r, reduces rows [p chunk, (p + 1) chunk) of column j of Y against the
// components evaluated on the fly (fd gradients / momentum of k_components_fd, bitwise the same
// values; w is L2-resident); blocks (r, p < Psum) are k_state_sum's partials of sum(u) (same
// partition and order, so mean_u is bitwise energy_components'), one launch for both.
__global__ void __launch_bounds__(256) k_comp_gemv(const CompArgs a, int r, size_t rows, size_t chunk, const double* Y,
                                                   size_t ldy, double* z, int Psum, double* mean_part) {
  pdl_wait();  // w comes from the coarse propagation launched just before
  pdl_trigger();
  const int n = a.n, d = a.G.dim;
  if (int(blockIdx.x) == r) {  // sum(u) partials
    if (int(blockIdx.y) >= Psum) return;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
    const int step = Psum * 256;
    int i = blockIdx.y * 256 + threadIdx.x;
    for (; i + 3 * step < n; i += 4 * step) {
      a0 += a.u[i];
      a1 += a.u[i + step];
      a2 += a.u[i + 2 * step];
      a3 += a.u[i + 3 * step];
    }
    for (; i < n; i += step) a0 += a.u[i];
    const double s = block_sum<256>((a0 + a1) + (a2 + a3));
    if (threadIdx.x == 0) mean_part[blockIdx.y] = s;
    return;
  }
  const double* Yj = Y + size_t(blockIdx.x) * ldy;
  const size_t r0 = size_t(blockIdx.y) * chunk, r1 = min(rows, r0 + chunk);
  auto comp = [&](size_t row) {
    const int ax = int(row / size_t(n)), pt = int(row - size_t(ax) * n);
    return ax < d ? fd_grad<false>(a.u, nullptr, a.G, a.B, ax, pt) : __ddiv_rn(a.v[pt], a.c[pt]);
  };
  double s0 = 0.0, s1 = 0.0;
  size_t i = r0 + threadIdx.x;
  for (; i + 256 < r1; i += 512) {
    s0 += Yj[i] * comp(i);
    s1 += Yj[i + 256] * comp(i + 256);
  }
  if (i < r1) s0 += Yj[i] * comp(i);
  const double t = block_sum<256>(s0 + s1);
  if (threadIdx.x == 0) z[size_t(blockIdx.x) * gridDim.y + blockIdx.y] = t;
}

int state_sum_parts(int n) { return std::max(1, std::min(64, n / 4096)); }

// complex staging for spectral maps
__global__ void k_real_to_complex(size_t total, int n, const double* src, size_t sstride, const int* index,
                                  double2* dst) {
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t b = e / n;
    const int p = int(e - b * n);
    const size_t s = index ? size_t(index[b]) : b;
    dst[e] = make_double2(src[s * sstride + p], 0.0);
  }
}

// spectral derivative multiplier along axis (energy_map.cpp:95-122)
__global__ void k_spectral_mult(size_t total, Geo G, int axis, const double* xi, double2* spec, double2* out) {
  const int n = G.ny * G.nx;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const int p = int(e % n);
    const int ky = p / G.nx, kx = p - ky * G.nx;
    int k, nn;
    if (G.dim == 1 || axis == 1) {
      k = kx;
      nn = G.nx;
    } else {
      k = ky;
      nn = G.ny;
    }
    const double2 v = spec[e];
    if (nn % 2 == 0 && k == nn / 2) {
      out[e] = make_double2(0.0, 0.0);
    } else {
      const double w = xi[k];  // v * (0 + i w) = (-w v.y, w v.x)
      out[e] = make_double2(0.0 * v.x - w * v.y, 0.0 * v.y + w * v.x);
    }
  }
}

__global__ void k_complex_real_to(size_t total, int n, const double2* src, double* out, size_t ld, size_t off) {
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t b = e / n;
    const int p = int(e - b * n);
    out[b * ld + off + p] = src[e].x;
  }
}

// Lambda-dagger spectrum (energy_map.cpp:158-208): gather g blocks into complex buffers
__global__ void k_stack_to_complex(size_t total, int n, int axis, const double* stacked, size_t ld, double2* dst) {
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t b = e / n;
    const int p = int(e - b * n);
    dst[e] = make_double2(stacked[b * ld + size_t(axis) * n + p], 0.0);
  }
}

__global__ void k_uhat(size_t total, Geo G, const double* xiy, const double* xix, const double2* gy, const double2* gx,
                       const double* mean, double2* uhat) {
  const int n = G.ny * G.nx;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t b = e / n;
    const int p = int(e - b * n);
    const int ky = p / G.nx, kx = p - ky * G.nx;
    double2 r;
    if (G.dim == 1) {
      if (kx == 0) {
        r = make_double2(mean[b], 0.0);
      } else {
        const double xi = xix[kx];
        const double2 num = make_double2(0.0 + xi * gx[e].x, 0.0 + xi * gx[e].y);
        const double den = xi * xi;
        r = make_double2(num.y / den, -num.x / den);  // (0,-1)*num / den
      }
    } else if (ky == 0 && kx == 0) {
      r = make_double2(mean[b], 0.0);
    } else if ((G.ny % 2 == 0 && ky == G.ny / 2) && (G.nx % 2 == 0 && kx == G.nx / 2)) {
      r = make_double2(0.0, 0.0);
    } else {
      const double a = xiy[ky], c = xix[kx];
      const double2 num = make_double2(__dadd_rn(0.0 + a * gy[e].x, c * gx[e].x), __dadd_rn(0.0 + a * gy[e].y, c * gx[e].y));
      const double den = __dadd_rn(__dmul_rn(a, a), __dmul_rn(c, c));
      r = make_double2(num.y / den, -num.x / den);
    }
    uhat[e] = r;
  }
}

__global__ void k_finish_inverse(size_t total, int n, int d, const double2* uhat, const double* stacked, size_t ld,
                                 const double* c, double* u, double* v, size_t sstride) {
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t b = e / n;
    const int p = int(e - b * n);
    u[b * sstride + p] = uhat[e].x;
    v[b * sstride + p] = __dmul_rn(c[p], stacked[b * ld + size_t(d) * n + p]);
  }
}

// fused fd energy sums of a state pair: S_diff = |Lambda(a-b)|^2, S_ref = |Lambda(b)|^2,
// L_diff = sum (ua-ub)^2, L_ref = sum ub^2 (energy_map.cpp:216-249).  grid = (PB, pairs):
// fixed per-block partials, then k_pair_final sums them in block order (deterministic).
constexpr int PAIR_BLOCKS = 32;

__global__ void __launch_bounds__(256) k_pair_sums(Geo G, Beta B, int n, const double* ua, const double* va,
                                                   size_t sa, const double* ub, const double* vb, size_t sb,
                                                   const double* c, double* part, int32_t* nonfinite) {
  bool ok = true;
  const size_t pr = blockIdx.y;
  const double* UA = ua + pr * sa;
  const double* VA = va + pr * sa;
  const double* UB = ub + pr * sb;
  const double* VB = vb + pr * sb;
  double sd = 0.0, sr = 0.0, ld = 0.0, lr = 0.0;
  for (int p = blockIdx.x * 256 + threadIdx.x; p < n; p += gridDim.x * 256) {
    for (int ax = 0; ax < G.dim; ++ax) {
      const double gd = fd_grad<true>(UA, UB, G, B, ax, p);
      const double gr = fd_grad<false>(UB, nullptr, G, B, ax, p);
      sd += gd * gd;
      sr += gr * gr;
    }
    const double md = __ddiv_rn(__dsub_rn(VA[p], VB[p]), c[p]);
    const double mr = __ddiv_rn(VB[p], c[p]);
    sd += md * md;
    sr += mr * mr;
    const double du = __dsub_rn(UA[p], UB[p]);
    ld += du * du;
    lr += UB[p] * UB[p];
    ok &= isfinite(UA[p]) && isfinite(VA[p]);
  }
  if (nonfinite && __syncthreads_or(!ok) && threadIdx.x == 0) atomicOr(&nonfinite[pr], 1);
  sd = block_sum<256>(sd);
  sr = block_sum<256>(sr);
  ld = block_sum<256>(ld);
  lr = block_sum<256>(lr);
  if (threadIdx.x == 0) {
    double* o = part + (pr * gridDim.x + blockIdx.x) * 4;
    o[0] = sd;
    o[1] = sr;
    o[2] = ld;
    o[3] = lr;
  }
}

// 2D variant: block rows r = blockIdx.x (+ k * gridDim.x), threads along x; periodic neighbour
// offsets resolved once per row instead of integer div/mod per access.  Per-point arithmetic is
// that of fd_grad / k_pair_sums (same rounding), only the grouping of the partial sums differs.
__device__ __forceinline__ double grad_x(const double* ra, const double* rb, int x, int nx, const Beta& B, double ih,
                                         bool diff) {
  double acc = 0.0;
#pragma unroll
  for (int j = 1; j <= 4; ++j) {
    if (j > B.m) break;
    const int xp = x + j >= nx ? x + j - nx : x + j;
    const int xm = x - j < 0 ? x - j + nx : x - j;
    const double a = diff ? __dsub_rn(ra[xp], rb[xp]) : ra[xp];
    const double b = diff ? __dsub_rn(ra[xm], rb[xm]) : ra[xm];
    acc = __dadd_rn(acc, __dmul_rn(B.b[j - 1], __dsub_rn(a, b)));
  }
  return __dmul_rn(acc, ih);
}

__global__ void __launch_bounds__(256) k_pair_sums2d(Geo G, Beta B, const double* ua, const double* va, size_t sa,
                                                     const double* ub, const double* vb, size_t sb, const double* c,
                                                     double* part, int32_t* nonfinite) {
  bool ok = true;
  const size_t pr = blockIdx.y;
  const double* UA = ua + pr * sa;
  const double* VA = va + pr * sa;
  const double* UB = ub + pr * sb;
  const double* VB = vb + pr * sb;
  const int nx = G.nx, ny = G.ny;
  double sd = 0.0, sr = 0.0, ld = 0.0, lr = 0.0;
  // a contiguous band of rows per block: the y-neighbour rows of row r were rows of the band's
  // previous iterations, so they come from this SM's L1 instead of L2
  const int band = (ny + int(gridDim.x) - 1) / int(gridDim.x);
  const int r_end = min(ny, (int(blockIdx.x) + 1) * band);
  for (int r = int(blockIdx.x) * band; r < r_end; ++r) {
    int rp[4], rm[4];
#pragma unroll
    for (int j = 1; j <= 4; ++j) {
      rp[j - 1] = ((r + j) % ny) * nx;
      rm[j - 1] = ((r + ny * 4 - j) % ny) * nx;
    }
    const size_t row = size_t(r) * nx;
    for (int x = threadIdx.x; x < nx; x += 256) {
      const size_t p = row + x;
      // axis 0 (y)
      double ady = 0.0, ary = 0.0;
#pragma unroll
      for (int j = 1; j <= 4; ++j) {
        if (j > B.m) break;
        const size_t pp = size_t(rp[j - 1]) + x, pm = size_t(rm[j - 1]) + x;
        const double bp = UB[pp], bm = UB[pm];
        ady = __dadd_rn(ady, __dmul_rn(B.b[j - 1], __dsub_rn(__dsub_rn(UA[pp], bp), __dsub_rn(UA[pm], bm))));
        ary = __dadd_rn(ary, __dmul_rn(B.b[j - 1], __dsub_rn(bp, bm)));
      }
      const double gdy = __dmul_rn(ady, G.ih[0]), gry = __dmul_rn(ary, G.ih[0]);
      sd += gdy * gdy;
      sr += gry * gry;
      // axis 1 (x)
      const double gdx = grad_x(UA + row, UB + row, x, nx, B, G.ih[1], true);
      const double grx = grad_x(UB + row, nullptr, x, nx, B, G.ih[1], false);
      sd += gdx * gdx;
      sr += grx * grx;
      const double cp = c[p], vbp = VB[p], ubp = UB[p], vap = VA[p];
      ok &= isfinite(UA[p]) && isfinite(vap);
      const double md = __ddiv_rn(__dsub_rn(vap, vbp), cp);
      const double mr = __ddiv_rn(vbp, cp);
      sd += md * md;
      sr += mr * mr;
      const double du = __dsub_rn(UA[p], ubp);
      ld += du * du;
      lr += ubp * ubp;
    }
  }
  if (nonfinite && __syncthreads_or(!ok) && threadIdx.x == 0) atomicOr(&nonfinite[pr], 1);
  sd = block_sum<256>(sd);
  sr = block_sum<256>(sr);
  ld = block_sum<256>(ld);
  lr = block_sum<256>(lr);
  if (threadIdx.x == 0) {
    double* o = part + (pr * gridDim.x + blockIdx.x) * 4;
    o[0] = sd;
    o[1] = sr;
    o[2] = ld;
    o[3] = lr;
  }
}

// Streaming variant for wide 2D grids (nx % 256 == 0): block = a 256-column strip x a band of rows
// of one pair; each thread owns one column and marches down the band with the (2M+1)-row windows
// of u_a and u_b in registers, so every u value is loaded once (the y-neighbours come from the
// window, the x-neighbours from a shared row of the band's current row, halo columns of the
// neighbouring strips loaded by the edge threads).  Per-point arithmetic is k_pair_sums2d's (same
// rounding: the x-term differences u_a - u_b are formed before they are shared); only the grouping
// of the partial sums differs (fixed: thread, then block, then k_pair_final in block order).
constexpr int PS_T = 256;
template <int M>
__global__ void __launch_bounds__(PS_T) k_pair_sums_stream(Geo G, Beta B, int bands, const double* ua,
                                                          const double* va, size_t sa, const double* ub,
                                                          const double* vb, size_t sb, const double* c, double* part,
                                                          int32_t* nonfinite) {
  __shared__ double sdif[2][PS_T + 2 * M], sref[2][PS_T + 2 * M];
  const int nx = G.nx, ny = G.ny, strips = nx / PS_T;
  const int strip = int(blockIdx.x) % strips, band = int(blockIdx.x) / strips;
  const size_t pr = blockIdx.y;
  const double* UA = ua + pr * sa;
  const double* VA = va + pr * sa;
  const double* UB = ub + pr * sb;
  const double* VB = vb + pr * sb;
  const int t = threadIdx.x, x = strip * PS_T + t;
  const int rows = (ny + bands - 1) / bands, r0 = band * rows, r1 = min(ny, r0 + rows);
  // halo columns: thread t < 2M loads column x_h of the left (t < M) or right halo
  const int hx = t < M ? (strip * PS_T - M + t + nx) % nx : ((strip + 1) * PS_T + (t - M)) % nx;
  const int hslot = t < M ? t : PS_T + t;
  double wa[2 * M + 1], wb[2 * M + 1];
#pragma unroll
  for (int k = 0; k < 2 * M; ++k) {  // rows r0 - M .. r0 + M - 1
    const size_t o = size_t((r0 - M + k + ny) % ny) * nx + x;
    wa[k] = UA[o];
    wb[k] = UB[o];
  }
  double sd = 0.0, sr = 0.0, ld = 0.0, lr = 0.0;
  bool ok = true;
  int buf = 0;
  for (int r = r0; r < r1; ++r) {
    {
      const size_t o = size_t((r + M) % ny) * nx + x;
      wa[2 * M] = UA[o];
      wb[2 * M] = UB[o];
    }
    const size_t p = size_t(r) * nx + x;
    sdif[buf][M + t] = __dsub_rn(wa[M], wb[M]);
    sref[buf][M + t] = wb[M];
    if (t < 2 * M) {
      const size_t ho = size_t(r) * nx + hx;
      sdif[buf][hslot] = __dsub_rn(UA[ho], UB[ho]);
      sref[buf][hslot] = UB[ho];
    }
    const double cp = c[p], vbp = VB[p], vap = VA[p];
    // axis 0 (y) from the windows
    double ady = 0.0, ary = 0.0;
#pragma unroll
    for (int j = 1; j <= M; ++j) {
      ady = __dadd_rn(ady, __dmul_rn(B.b[j - 1], __dsub_rn(__dsub_rn(wa[M + j], wb[M + j]),
                                                            __dsub_rn(wa[M - j], wb[M - j]))));
      ary = __dadd_rn(ary, __dmul_rn(B.b[j - 1], __dsub_rn(wb[M + j], wb[M - j])));
    }
    const double gdy = __dmul_rn(ady, G.ih[0]), gry = __dmul_rn(ary, G.ih[0]);
    sd += gdy * gdy;
    sr += gry * gry;
    __syncthreads();  // the shared row (and its halo) of this r complete
    double adx = 0.0, arx = 0.0;
#pragma unroll
    for (int j = 1; j <= M; ++j) {
      adx = __dadd_rn(adx, __dmul_rn(B.b[j - 1], __dsub_rn(sdif[buf][M + t + j], sdif[buf][M + t - j])));
      arx = __dadd_rn(arx, __dmul_rn(B.b[j - 1], __dsub_rn(sref[buf][M + t + j], sref[buf][M + t - j])));
    }
    const double gdx = __dmul_rn(adx, G.ih[1]), grx = __dmul_rn(arx, G.ih[1]);
    sd += gdx * gdx;
    sr += grx * grx;
    ok &= isfinite(wa[M]) && isfinite(vap);
    const double md = __ddiv_rn(__dsub_rn(vap, vbp), cp);
    const double mr = __ddiv_rn(vbp, cp);
    sd += md * md;
    sr += mr * mr;
    const double du = __dsub_rn(wa[M], wb[M]);
    ld += du * du;
    lr += wb[M] * wb[M];
#pragma unroll
    for (int k = 0; k < 2 * M; ++k) {
      wa[k] = wa[k + 1];
      wb[k] = wb[k + 1];
    }
    buf ^= 1;  // the other shared row next: its previous readers passed this row's barrier
  }
  if (nonfinite && __syncthreads_or(!ok) && threadIdx.x == 0) atomicOr(&nonfinite[pr], 1);
  sd = block_sum<256>(sd);
  sr = block_sum<256>(sr);
  ld = block_sum<256>(ld);
  lr = block_sum<256>(lr);
  if (threadIdx.x == 0) {
    double* o = part + (pr * gridDim.x + blockIdx.x) * 4;
    o[0] = sd;
    o[1] = sr;
    o[2] = ld;
    o[3] = lr;
  }
}

__global__ void k_pair_final(size_t pairs, int nb, const double* part, double* out) {
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < pairs * 4; e += size_t(gridDim.x) * blockDim.x) {
    const size_t pr = e / 4, q = e % 4;
    double acc = 0.0;
    for (int b = 0; b < nb; ++b) acc += part[(pr * nb + b) * 4 + q];
    out[e] = acc;
  }
}

__global__ void __launch_bounds__(256) k_sumsq_cols(int rows, const double* m, size_t ld, double* out) {
  const double* M = m + blockIdx.x * ld;
  double acc = 0.0;
  for (int i = threadIdx.x; i < rows; i += 256) acc += M[i] * M[i];
  const double s = block_sum<256>(acc);
  if (threadIdx.x == 0) out[blockIdx.x] = s;
}

__global__ void k_sub_states(size_t total, int n, const double* ua, const double* va, size_t sa, const double* ub,
                             const double* vb, size_t sb, double* uo, double* vo) {
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t b = e / n;
    const int p = int(e - b * n);
    uo[e] = __dsub_rn(ua[b * sa + p], ub[b * sb + p]);
    vo[e] = __dsub_rn(va[b * sa + p], vb[b * sb + p]);
  }
}

unsigned nblk(ptb_context* ctx, size_t total) {
  return unsigned(std::max<size_t>(1, std::min<size_t>((total + 255) / 256, size_t(ctx->num_sms) * 32)));
}

// per-grid wavenumber tables (fft.cpp:97-100 evaluated on the host, bitwise)
struct Xi {
  double* y = nullptr;
  double* x = nullptr;
};

std::vector<double> xi_table(size_t n, double h) {
  std::vector<double> t(n);
  const double extent = static_cast<double>(n) * h;
  for (size_t k = 0; k < n; ++k) {
    const long sf = k <= (n - 1) / 2 ? long(k) : long(k) - long(n);
    t[k] = 2.0 * M_PI * static_cast<double>(sf) / extent;
  }
  return t;
}

Xi xi_for(ptb_context* ctx, const ptb_grid& g, DeviceBuffer& buf) {
  const size_t ny = g.dim == 1 ? 1 : g.n[0], nx = g.dim == 1 ? g.n[0] : g.n[1];
  std::vector<double> host;
  if (g.dim == 2) {
    host = xi_table(g.n[0], g.h[0]);
    const std::vector<double> hx = xi_table(g.n[1], g.h[1]);
    host.insert(host.end(), hx.begin(), hx.end());
  } else {
    host = xi_table(g.n[0], g.h[0]);
  }
  double* d = static_cast<double*>(buf.get(host.size() * sizeof(double)));
  PTB_CUDA_CHECK(cudaMemcpyAsync(d, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice, ctx->stream));
  Xi xi;
  if (g.dim == 2) {
    xi.y = d;
    xi.x = d + ny;
  } else {
    xi.x = d;
  }
  (void)nx;
  return xi;
}

}  // namespace

EnergyWork::~EnergyWork() {
  for (auto& b : buf) b.release();
}

void energy_components(EnergyWork& w, const ptb_grid& g, int scheme, size_t batch, const double* u, const double* v,
                       size_t sstride, const int* index, const double* c, double* stacked, size_t ld, double* mean) {
  ptb_context* ctx = w.ctx;
  cudaStream_t st = ctx->stream;
  if (batch == 0) return;
  const Geo G = geo_of(g);
  const int n = G.ny * G.nx;
  const size_t total = batch * n;
  if (scheme != PTB_SPECTRAL) {
    CompArgs a{G, beta_of(scheme), n, u, v, sstride, index, c, stacked, ld};
    k_components_fd<<<nblk(ctx, total), 256, 0, st>>>(a, batch);
    PTB_LAUNCH_CHECK(ctx);
  } else {
    require(scheme == PTB_SPECTRAL, "gradient scheme");
    const Xi xi = xi_for(ctx, g, w.buf[0]);
    double2* spec = static_cast<double2*>(w.buf[1].get(total * sizeof(double2)));
    double2* tmp = static_cast<double2*>(w.buf[2].get(total * sizeof(double2)));
    k_real_to_complex<<<nblk(ctx, total), 256, 0, st>>>(total, n, u, sstride, index, spec);
    PTB_LAUNCH_CHECK(ctx);
    fft_field(ctx, st, g, batch, spec, false);
    for (int ax = 0; ax < G.dim; ++ax) {
      const double* xa = (G.dim == 1 || ax == 1) ? xi.x : xi.y;
      k_spectral_mult<<<nblk(ctx, total), 256, 0, st>>>(total, G, ax, xa, spec, tmp);
      PTB_LAUNCH_CHECK(ctx);
      fft_field(ctx, st, g, batch, tmp, true);
      k_complex_real_to<<<nblk(ctx, total), 256, 0, st>>>(total, n, tmp, stacked, ld, size_t(ax) * n);
      PTB_LAUNCH_CHECK(ctx);
    }
    CompArgs a{G, Beta{}, n, u, v, sstride, index, c, stacked, ld};
    k_momentum<<<nblk(ctx, total), 256, 0, st>>>(a, batch);
    PTB_LAUNCH_CHECK(ctx);
  }
  if (mean) {
    const int P = state_sum_parts(n);
    double* part = static_cast<double*>(w.buf[8].get(batch * P * sizeof(double)));
    // one partial per state: the block writes the sum directly (0 + x == x, same bits)
    k_state_sum<<<dim3(unsigned(P), unsigned(batch)), 256, 0, st>>>(n, u, sstride, index, P == 1 ? mean : part);
    PTB_LAUNCH_CHECK(ctx);
    if (P > 1) {
      k_state_sum_final<<<unsigned(std::min<size_t>((batch + 255) / 256, 1024)), 256, 0, st>>>(batch, P, part,
                                                                                              mean);
      PTB_LAUNCH_CHECK(ctx);
    }
  }
}

int comp_gemv_parts(size_t rows) { return int(std::max<size_t>(1, std::min<size_t>(64, rows / 2048))); }
int sweep_mean_parts(int n) { return state_sum_parts(n); }

void comp_gemv(EnergyWork& w, const ptb_grid& g, int scheme, const double* u, const double* v, const double* c,
               const double* Y, size_t ldy, int r, double* z, int P, double* mean_part) {
  ptb_context* ctx = w.ctx;
  require(scheme != PTB_SPECTRAL, "comp_gemv: finite-difference schemes only");
  const Geo G = geo_of(g);
  const int n = G.ny * G.nx;
  const size_t rows = size_t(G.dim + 1) * n;
  const int Psum = state_sum_parts(n);
  CompArgs a{G, beta_of(scheme), n, u, v, size_t(n), nullptr, c, nullptr, 0};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(unsigned(r + 1), unsigned(std::max(P, Psum)));
  cfg.blockDim = dim3(256);
  cfg.stream = ctx->stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  PTB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_comp_gemv, a, r, rows, (rows + P - 1) / P, Y, ldy, z, Psum, mean_part));
  PTB_LAUNCH_CHECK(ctx);
}

void from_energy_components(EnergyWork& w, const ptb_grid& g, size_t batch, const double* stacked, size_t ld,
                            const double* mean, const double* c, double* u, double* v, size_t sstride) {
  ptb_context* ctx = w.ctx;
  cudaStream_t st = ctx->stream;
  if (batch == 0) return;
  const Geo G = geo_of(g);
  const int n = G.ny * G.nx;
  const size_t total = batch * n;
  const Xi xi = xi_for(ctx, g, w.buf[0]);
  double2* gx = static_cast<double2*>(w.buf[1].get(total * sizeof(double2)));
  double2* gy = static_cast<double2*>(w.buf[2].get(total * sizeof(double2)));
  double2* uh = static_cast<double2*>(w.buf[3].get(total * sizeof(double2)));
  if (G.dim == 2) {
    k_stack_to_complex<<<nblk(ctx, total), 256, 0, st>>>(total, n, 0, stacked, ld, gy);
    PTB_LAUNCH_CHECK(ctx);
    fft_field(ctx, st, g, batch, gy, false);
    k_stack_to_complex<<<nblk(ctx, total), 256, 0, st>>>(total, n, 1, stacked, ld, gx);
  } else {
    k_stack_to_complex<<<nblk(ctx, total), 256, 0, st>>>(total, n, 0, stacked, ld, gx);
  }
  PTB_LAUNCH_CHECK(ctx);
  fft_field(ctx, st, g, batch, gx, false);
  k_uhat<<<nblk(ctx, total), 256, 0, st>>>(total, G, xi.y, xi.x, gy, gx, mean, uh);
  PTB_LAUNCH_CHECK(ctx);
  fft_field(ctx, st, g, batch, uh, true);
  k_finish_inverse<<<nblk(ctx, total), 256, 0, st>>>(total, n, G.dim, uh, stacked, ld, c, u, v, sstride);
  PTB_LAUNCH_CHECK(ctx);
}

__global__ void k_nonfinite_states(int n, const double* u, const double* v, size_t stride, int32_t* flags) {
  const size_t b = blockIdx.y;
  bool ok = true;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    ok &= isfinite(u[b * stride + i]) && isfinite(v[b * stride + i]);
  if (__syncthreads_or(!ok) && threadIdx.x == 0) atomicOr(&flags[b], 1);
}

// PTB_PAIR_STREAM=0: the row-per-block kernel (A/B measurements, tests)
bool pair_stream_enabled() {
  const char* e = std::getenv("PTB_PAIR_STREAM");
  return !(e && std::atoi(e) == 0);
}

void pair_energy_sums(EnergyWork& w, const ptb_grid& g, int scheme, size_t batch, const double* ua, const double* va,
                      size_t sa, const double* ub, const double* vb, size_t sb, const double* c, double* out4,
                      int32_t* nonfinite_a) {
  ptb_context* ctx = w.ctx;
  cudaStream_t st = ctx->stream;
  if (batch == 0) return;
  const Geo G = geo_of(g);
  const int n = G.ny * G.nx;
  if (scheme != PTB_SPECTRAL && G.dim == 2 && G.nx % PS_T == 0 && G.ny >= 64 && pair_stream_enabled()) {
    const int strips = G.nx / PS_T, bands = std::max(1, std::min(G.ny / 32, 64 / strips));
    const int nb = strips * bands;
    double* part = static_cast<double*>(w.buf[7].get(batch * nb * 4 * sizeof(double)));
    const dim3 grid{unsigned(nb), unsigned(batch)};
    const Beta bt = beta_of(scheme);
    switch (bt.m) {
      case 1: k_pair_sums_stream<1><<<grid, PS_T, 0, st>>>(G, bt, bands, ua, va, sa, ub, vb, sb, c, part, nonfinite_a); break;
      case 2: k_pair_sums_stream<2><<<grid, PS_T, 0, st>>>(G, bt, bands, ua, va, sa, ub, vb, sb, c, part, nonfinite_a); break;
      case 3: k_pair_sums_stream<3><<<grid, PS_T, 0, st>>>(G, bt, bands, ua, va, sa, ub, vb, sb, c, part, nonfinite_a); break;
      default: k_pair_sums_stream<4><<<grid, PS_T, 0, st>>>(G, bt, bands, ua, va, sa, ub, vb, sb, c, part, nonfinite_a); break;
    }
    PTB_LAUNCH_CHECK(ctx);
    k_pair_final<<<nblk(ctx, batch * 4), 256, 0, st>>>(batch, nb, part, out4);
    PTB_LAUNCH_CHECK(ctx);
    return;
  }
  if (scheme != PTB_SPECTRAL) {
    const int nb = std::max(1, std::min(PAIR_BLOCKS, (n + 255) / 256));
    double* part = static_cast<double*>(w.buf[7].get(batch * nb * 4 * sizeof(double)));
    if (G.dim == 2 && G.nx >= 256)
      k_pair_sums2d<<<dim3(nb, unsigned(batch)), 256, 0, st>>>(G, beta_of(scheme), ua, va, sa, ub, vb, sb, c, part,
                                                                 nonfinite_a);
    else
      k_pair_sums<<<dim3(nb, unsigned(batch)), 256, 0, st>>>(G, beta_of(scheme), n, ua, va, sa, ub, vb, sb, c, part,
                                                               nonfinite_a);
    PTB_LAUNCH_CHECK(ctx);
    k_pair_final<<<nblk(ctx, batch * 4), 256, 0, st>>>(batch, nb, part, out4);
    PTB_LAUNCH_CHECK(ctx);
    return;
  }
  if (nonfinite_a) {
    k_nonfinite_states<<<dim3(unsigned(std::max(1, std::min(64, (n + 255) / 256))), unsigned(batch)), 256, 0, st>>>(
        n, ua, va, sa, nonfinite_a);
    PTB_LAUNCH_CHECK(ctx);
  }
  // spectral: components of (a - b) and b, then sums of squares (chunked over states)
  const size_t rows = size_t(G.dim + 1) * n;
  std::vector<double> dummy;
  const size_t chunk = std::max<size_t>(1, std::min<size_t>(batch, (size_t(256) << 20) / (rows * 8 * 4)));
  double* du = static_cast<double*>(w.buf[4].get(chunk * n * sizeof(double)));
  double* dv = static_cast<double*>(w.buf[5].get(chunk * n * sizeof(double)));
  double* comp = static_cast<double*>(w.buf[6].get(chunk * rows * sizeof(double)));
  double* sums = static_cast<double*>(w.buf[7].get(chunk * sizeof(double)));
  for (size_t b0 = 0; b0 < batch; b0 += chunk) {
    const size_t nb = std::min(chunk, batch - b0);
    k_sub_states<<<nblk(ctx, nb * n), 256, 0, st>>>(nb * n, n, ua + b0 * sa, va + b0 * sa, sa, ub + b0 * sb,
                                                    vb + b0 * sb, sb, du, dv);
    PTB_LAUNCH_CHECK(ctx);
    for (int which = 0; which < 2; ++which) {
      if (which == 0)
        energy_components(w, g, scheme, nb, du, dv, n, nullptr, c, comp, rows, nullptr);
      else
        energy_components(w, g, scheme, nb, ub + b0 * sb, vb + b0 * sb, sb, nullptr, c, comp, rows, nullptr);
      k_sumsq_cols<<<unsigned(nb), 256, 0, st>>>(int(rows), comp, rows, sums);
      PTB_LAUNCH_CHECK(ctx);
      PTB_CUDA_CHECK(cudaMemcpy2DAsync(out4 + b0 * 4 + which, 4 * sizeof(double), sums, sizeof(double),
                                       sizeof(double), nb, cudaMemcpyDeviceToDevice, st));
    }
    // l2 sums: reuse the fd kernel path on u only is not needed; compute with sumsq
    k_sumsq_cols<<<unsigned(nb), 256, 0, st>>>(n, du, size_t(n), sums);
    PTB_LAUNCH_CHECK(ctx);
    PTB_CUDA_CHECK(cudaMemcpy2DAsync(out4 + b0 * 4 + 2, 4 * sizeof(double), sums, sizeof(double), sizeof(double), nb,
                                     cudaMemcpyDeviceToDevice, st));
    k_sumsq_cols<<<unsigned(nb), 256, 0, st>>>(n, ub + b0 * sb, sb, sums);
    PTB_LAUNCH_CHECK(ctx);
    PTB_CUDA_CHECK(cudaMemcpy2DAsync(out4 + b0 * 4 + 3, 4 * sizeof(double), sums, sizeof(double), sizeof(double), nb,
                                     cudaMemcpyDeviceToDevice, st));
  }
}

void column_sumsq(ptb_context* ctx, int rows, size_t cols, const double* m, size_t ld, double* out) {
  if (cols == 0) return;
  k_sumsq_cols<<<unsigned(cols), 256, 0, ctx->stream>>>(rows, m, ld, out);
  PTB_LAUNCH_CHECK(ctx);
}

}  // namespace ptb
