// Absorbing-layer (PML) fine propagator for BASELINE.json config 4 — not in the reference.
//
// The reference propagator is periodic only (propagator.cpp:31-105); SPEC.md:8,97 lists a PML as
// future work and SURVEY.md 8(f) rank 4 asks for one for config 4 ("32-cell perfectly-matched
// absorbing layer on all sides").  The scheme is specified, with its derivation, by the CPU
// oracle oracle/pml_np.py (parity unpinned by the reference: pinned by self-consistency, see
// there and tests/test_pml_*.py):
//   u_tt + (zx+zy) u_t + zx zy u = c^2 (Lap u + Dx px + Dy py)
//   px_t = -zx px + (zy - zx) Dx u,  py_t = -zy py + (zx - zy) Dy u
// velocity Verlet with the damping split trapezoidally over the two half kicks, auxiliary
// fields advanced by the trapezoidal rule.  State per slice: u, udot, px, py (SoA, slice-major,
// row-major fields as everywhere else).  px, py must be zero wherever zx = zy = 0 (they stay
// zero there); the kernel never touches them on tiles without layer cells.
//
// Kernel k_pml<LAYER>: overlapped temporal tiling.  A CTA owns a TY x TX output tile of one slice
// and loads it with a halo of H = 2S+1 cells (periodic wrap, so any grid size works) into shared
// memory, then runs up to S steps on chip: the initial half kick shrinks the valid region by one
// cell, each step by 2 more in the layer (the auxiliary update reads new u neighbours, the force
// reads new auxiliary neighbours) and by 1 elsewhere; after S steps the central tile is exact.  The carried velocity is the half
// kick vh (as the FAST kernel), so the drift is pointwise.  Tiles with no layer cell in their
// halo run the plain FAST step (bitwise the periodic kernels' arithmetic, bfast<true> below);
// the two tile classes are two launches (LAYER = false / true) so the plain tiles need only the
// u plane in shared memory (more CTAs per SM).  Out of place (halo reads of other tiles' inputs):
// passes ping-pong between the caller's buffers and the propagator's scratch.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "ptb_internal.h"

namespace ptb {
namespace {

constexpr int PS = 4;           // steps per pass
constexpr int HL = 2 * PS + 1;  // layer-tile halo: the first half kick costs 1 cell, each step 2
constexpr int HP = PS + 1;      // plain-tile halo: 1 cell per step + 1
constexpr int BT = 96;          // plain tiles are BT x BT; layer tiles BT/2 (4 per big tile)

struct PmlArgs {
  int ny, nx;
  size_t n;
  double dt, hd, ry, cc, gx, gy;
  const double* kx;                          // hd c^2 / hx^2 (N)
  const double *zx, *ax, *qx;                // per column
  const double *zy, *ay, *qy;                // per row
  const double *ui, *vi, *pxi, *pyi;
  double *uo, *vo, *pxo, *pyo;
  int steps;                                 // steps of this pass (<= PS)
  int32_t* flags;
};

template <int T, int H, int NT>
struct Geo {
  static constexpr int E = T + 2 * H, EXT = E * E, NPT = (EXT + NT - 1) / NT, EXTP = NPT * NT;
  static constexpr int PAD = E + 1;            // stencil reads of padded points stay in bounds
  static constexpr int PLANE = EXTP + 2 * PAD;
};

// FAST half kick, the association of propagate.cu's bfast<true> (must stay identical so a zero
// profile reproduces the periodic kernels bitwise; tests/test_gpu_pml.py checks it)
__device__ __forceinline__ double bfast_y(double uc, double ul, double ur, double uu, double ud, double kx,
                                          double ry, double cc) {
  const double s1 = ul + ur;
  return fma(kx * ry, uu, kx * fma(cc, uc, fma(ry, ud, s1)));
}

// The layer terms with every operation rounded separately, in oracle/pml_np.py's order (one
// code path for the first kick of a pass and the kicks inside it: a fused coupling then equals
// repeated single steps bitwise).
__device__ __forceinline__ double kick_layer(double v, double f, double u, double zx, double zy, double hd) {
  const double d = __dadd_rn(__dmul_rn(__dmul_rn(zy, zx), u), __dmul_rn(__dadd_rn(zy, zx), v));
  return __dadd_rn(v, __dsub_rn(f, __dmul_rn(hd, d)));  // v + (F - hd (pi u + sg v))
}
__device__ __forceinline__ double force_layer(double fb, double kx, double gx, double gy, double pxe, double pxw,
                                              double pyn, double pys) {
  return __dadd_rn(fb, __dmul_rn(kx, __dadd_rn(__dmul_rn(gx, __dsub_rn(pxe, pxw)), __dmul_rn(gy, __dsub_rn(pyn, pys)))));
}

__device__ __forceinline__ int wrap(int i, int n) {
  i %= n;
  return i < 0 ? i + n : i;
}

// Does big tile (by, bx) have a layer cell within HL cells?  Both launches classify with this
// one rule, so every tile is processed by exactly one of them.  Called by all threads.
template <int NT>
__device__ bool big_tile_has_layer(const PmlArgs& a, int by, int bx) {
  bool any = false;
  for (int j = threadIdx.x; j < BT + 2 * HL; j += NT) {
    any |= a.zx[wrap(bx * BT - HL + j, a.nx)] > 0.0;
    any |= a.zy[wrap(by * BT - HL + j, a.ny)] > 0.0;
  }
  return __syncthreads_or(any) != 0;
}

template <bool LAYER, int NT>
__global__ void __launch_bounds__(NT, 1) k_pml(const PmlArgs a) {
  constexpr int T = LAYER ? BT / 2 : BT, H = LAYER ? HL : HP;
  using G = Geo<T, H, NT>;
  constexpr int E = G::E, NPT = G::NPT;
  extern __shared__ double sm[];
  double* us = sm + G::PAD;
  double* pxs = sm + G::PLANE + G::PAD;      // LAYER: px; plain: the coefficient kx
  double* pys = sm + 2 * G::PLANE + G::PAD;  // LAYER only
  double* ks = pxs;
  double* zxs = sm + (LAYER ? 3 : 2) * G::PLANE;  // E each: zx ax qx zy ay qy (LAYER only)
  double* axs = zxs + E;
  double* qxs = axs + E;
  double* zys = qxs + E;
  double* ays = zys + E;
  double* qys = ays + E;
  int* colg = reinterpret_cast<int*>(zxs + (LAYER ? 6 * E : 0));  // E: global column
  int* rowg = colg + E;                                             // E: global row offset

  const int tid = threadIdx.x, b = blockIdx.z;
  const int ty0 = blockIdx.y * T, tx0 = blockIdx.x * T;
  if (ty0 >= a.ny || tx0 >= a.nx) return;
  const int by = LAYER ? blockIdx.y / 2 : blockIdx.y, bx = LAYER ? blockIdx.x / 2 : blockIdx.x;
  if (big_tile_has_layer<NT>(a, by, bx) != LAYER) return;  // the other launch owns this tile

  for (int j = tid; j < E; j += NT) {
    const int gx = wrap(tx0 - H + j, a.nx), gy = wrap(ty0 - H + j, a.ny);
    colg[j] = gx;
    rowg[j] = gy * a.nx;
    if constexpr (LAYER) {
      zxs[j] = a.zx[gx];
      axs[j] = a.ax[gx];
      qxs[j] = a.qx[gx];
      zys[j] = a.zy[gy];
      ays[j] = a.ay[gy];
      qys[j] = a.qy[gy];
    }
  }
  for (int j = tid; j < G::PAD; j += NT) {  // the pads are read (rim stencils) but never matter
    us[j - G::PAD] = 0.0;
    us[G::EXTP + j] = 0.0;
    pxs[j - G::PAD] = pxs[G::EXTP + j] = 0.0;
    if constexpr (LAYER) pys[j - G::PAD] = pys[G::EXTP + j] = 0.0;
  }
  __syncthreads();

  const size_t base = size_t(b) * a.n;
  double hv[NPT];                  // v on load, then the carried half kick vh, then v at the end
  double kr[LAYER ? NPT : 1];      // layer tiles: kx in registers (plain tiles: the ks plane)
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    const int e = tid + i * NT;
    double u = 0.0, v = 0.0, k = 0.0, px = 0.0, py = 0.0;
    if (e < G::EXT) {
      const int ey = e / E, ex = e - ey * E;
      const size_t g = size_t(rowg[ey]) + colg[ex];
      u = a.ui[base + g];
      v = a.vi[base + g];
      k = a.kx[g];
      if constexpr (LAYER) {
        px = a.pxi[base + g];
        py = a.pyi[base + g];
      }
    }
    us[e] = u;
    hv[i] = v;
    if constexpr (LAYER) {
      kr[i] = k;
      pxs[e] = px;
      pys[e] = py;
    } else {
      ks[e] = k;
    }
  }
  __syncthreads();

  // Every stage runs over all padded points without branches: rim and pad values are garbage
  // that moves inward one cell per dependent stage, never into the central tile (halo H).
  auto force = [&](int e, double kl) {
    const double k = LAYER ? kl : ks[e];
    const double fb = bfast_y(us[e], us[e - 1], us[e + 1], us[e + E], us[e - E], k, a.ry, a.cc);
    if constexpr (!LAYER) return fb;
    return force_layer(fb, k, a.gx, a.gy, pxs[e + 1], pxs[e - 1], pys[e + E], pys[e - E]);
  };
  auto col = [](int e) { return e % E; };
  auto row = [](int e) { return min(e / E, E - 1); };

#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    const int e = tid + i * NT;
    const double f = force(e, kr[LAYER ? i : 0]);
    if constexpr (LAYER)
      hv[i] = kick_layer(hv[i], f, us[e], zxs[col(e)], zys[row(e)], a.hd);
    else
      hv[i] = hv[i] + f;
  }
  for (int s = 0; s < a.steps; ++s) {
    __syncthreads();  // force reads of u are done
#pragma unroll
    for (int i = 0; i < NPT; ++i) {
      const int e = tid + i * NT;
      us[e] = us[e] + a.dt * hv[i];  // drift (pointwise)
    }
    __syncthreads();
    if constexpr (LAYER) {
#pragma unroll
      for (int i = 0; i < NPT; ++i) {
        const int e = tid + i * NT;
        const int ex = col(e), ey = row(e);
        const double zx = zxs[ex], zy = zys[ey];
        pxs[e] = __dadd_rn(__dmul_rn(axs[ex], pxs[e]),
                           __dmul_rn(__dmul_rn(__dsub_rn(zy, zx), qxs[ex]), __dsub_rn(us[e + 1], us[e - 1])));
        pys[e] = __dadd_rn(__dmul_rn(ays[ey], pys[e]),
                           __dmul_rn(__dmul_rn(__dsub_rn(zx, zy), qys[ey]), __dsub_rn(us[e + E], us[e - E])));
      }
      __syncthreads();
    }
    const bool last = s + 1 == a.steps;
#pragma unroll
    for (int i = 0; i < NPT; ++i) {
      const int e = tid + i * NT;
      const double f = force(e, kr[LAYER ? i : 0]);
      if constexpr (LAYER) {
        const double zx = zxs[col(e)], zy = zys[row(e)];
        const double pi = __dmul_rn(zy, zx), sg = __dadd_rn(zy, zx);
        const double inv = __ddiv_rn(1.0, __dadd_rn(1.0, __dmul_rn(a.hd, sg)));
        const double v1 = __dmul_rn(__dadd_rn(hv[i], __dsub_rn(f, __dmul_rn(a.hd, __dmul_rn(pi, us[e])))), inv);
        hv[i] = last ? v1 : kick_layer(v1, f, us[e], zx, zy, a.hd);
      } else {
        const double v1 = hv[i] + f;
        hv[i] = last ? v1 : v1 + f;
      }
    }
  }

  // store the central tile
  bool bad = false;
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    const int e = tid + i * NT;
    if (e < G::EXT) {
      const int ey = e / E, ex = e - ey * E;
      const int oy = ey - H, ox = ex - H;
      if (oy >= 0 && oy < T && ox >= 0 && ox < T && ty0 + oy < a.ny && tx0 + ox < a.nx) {
        const size_t g = base + size_t(ty0 + oy) * a.nx + (tx0 + ox);
        a.uo[g] = us[e];
        a.vo[g] = hv[i];
        bad |= !(isfinite(us[e]) && isfinite(hv[i]));
        if constexpr (LAYER) {
          a.pxo[g] = pxs[e];
          a.pyo[g] = pys[e];
          bad |= !(isfinite(pxs[e]) && isfinite(pys[e]));
        }
      }
    }
  }
  if (a.flags) {
    bad = __syncthreads_or(bad);
    if (bad && tid == 0) atomicOr(&a.flags[b], 1);
  }
}

constexpr int kPlainThreads = 512, kLayerThreads = 512;

template <bool LAYER>
size_t pml_smem() {
  using G = Geo<LAYER ? BT / 2 : BT, LAYER ? HL : HP, LAYER ? kLayerThreads : kPlainThreads>;
  return size_t(G::PLANE) * (LAYER ? 3 : 2) * sizeof(double) + (LAYER ? 6 * G::E * sizeof(double) : 0) +
         2 * G::E * sizeof(int);
}

struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    cudaGetDevice(&prev);
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace
}  // namespace ptb

struct ptb_pml {
  ptb_context* ctx = nullptr;
  ptb_grid grid{};
  size_t n = 0, steps = 0;
  double dt = 0, hd = 0, ry = 0, cc = 0, gx = 0, gy = 0;
  double* coef = nullptr;  // kx (n) | zx ax qx (nx) | zy ay qy (ny)
  ptb::DeviceBuffer scratch;  // 4 fields x batch (ping-pong partner; phi planes zeroed once)
  size_t scratch_batch = 0;
};

namespace ptb {

void pml_propagate(ptb_pml* p, size_t steps, size_t batch, double* u, double* v, double* px, double* py,
                   int32_t* flags) {
  ptb_context* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  if (batch == 0 || steps == 0) return;
  const int ny = int(p->grid.n[0]), nx = int(p->grid.n[1]);
  const size_t n = p->n, fb = batch * n * sizeof(double);
  if (p->scratch_batch < batch) {
    double* s = static_cast<double*>(p->scratch.get(4 * fb));
    PTB_CUDA_CHECK(cudaMemsetAsync(s, 0, 4 * fb, st));  // phi planes: zero off the layer, for good
    p->scratch_batch = batch;
  }
  double* s = static_cast<double*>(p->scratch.ptr);
  const size_t sb = p->scratch_batch * n;
  double* bufs[2][4] = {{u, v, px, py}, {s, s + sb, s + 2 * sb, s + 3 * sb}};
  PmlArgs a{};
  a.ny = ny;
  a.nx = nx;
  a.n = n;
  a.dt = p->dt;
  a.hd = p->hd;
  a.ry = p->ry;
  a.cc = p->cc;
  a.gx = p->gx;
  a.gy = p->gy;
  a.kx = p->coef;
  a.zx = p->coef + n;
  a.ax = a.zx + nx;
  a.qx = a.ax + nx;
  a.zy = a.qx + nx;
  a.ay = a.zy + ny;
  a.qy = a.ay + ny;
  static bool attr = false;
  if (!attr) {
    PTB_CUDA_CHECK(cudaFuncSetAttribute(k_pml<false, kPlainThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(pml_smem<false>())));
    PTB_CUDA_CHECK(cudaFuncSetAttribute(k_pml<true, kLayerThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(pml_smem<true>())));
    attr = true;
  }
  // plain launch: big tiles; layer launch: the four half-size tiles of every big tile
  const dim3 gplain((nx + BT - 1) / BT, (ny + BT - 1) / BT, unsigned(batch));
  const dim3 glayer(2 * gplain.x, 2 * gplain.y, unsigned(batch));
  int cur = 0;
  for (size_t done = 0; done < steps;) {
    const int ns = int(std::min<size_t>(PS, steps - done));
    done += ns;
    a.ui = bufs[cur][0];
    a.vi = bufs[cur][1];
    a.pxi = bufs[cur][2];
    a.pyi = bufs[cur][3];
    a.uo = bufs[1 - cur][0];
    a.vo = bufs[1 - cur][1];
    a.pxo = bufs[1 - cur][2];
    a.pyo = bufs[1 - cur][3];
    a.steps = ns;
    a.flags = done == steps ? flags : nullptr;
    k_pml<false, kPlainThreads><<<gplain, kPlainThreads, pml_smem<false>(), st>>>(a);
    PTB_LAUNCH_CHECK(ctx);
    k_pml<true, kLayerThreads><<<glayer, kLayerThreads, pml_smem<true>(), st>>>(a);
    PTB_LAUNCH_CHECK(ctx);
    cur = 1 - cur;
  }
  if (cur == 1)  // odd number of passes: the result is in the scratch
    for (int f = 0; f < 4; ++f)
      PTB_CUDA_CHECK(cudaMemcpyAsync(bufs[0][f], bufs[1][f], fb, cudaMemcpyDeviceToDevice, st));
}

}  // namespace ptb

using namespace ptb;

extern "C" {

ptb_status ptb_pml_damping_profile(size_t n, size_t width, double h, double cmax, double reflection,
                                   double* out_host) {
  return guarded([&] {
    require(out_host, "pml: null output");
    require(n >= 4 && h > 0.0 && cmax > 0.0 && reflection > 0.0 && reflection < 1.0, "pml: bad profile argument");
    require(2 * width < n, "pml: layer wider than half the axis");
    std::fill(out_host, out_host + n, 0.0);
    if (width == 0) return;
    const double L = double(width) * h;
    const double z0 = 1.5 * cmax * std::log(1.0 / reflection) / L;  // oracle/pml_np.py damping_profile
    for (size_t i = 0; i < width; ++i) {
      const double t = (double(width - i) - 0.5) / double(width);
      out_host[i] = z0 * (t * t);
      out_host[n - 1 - i] = z0 * (t * t);
    }
  });
}

ptb_status ptb_pml_create(ptb_context* ctx, const ptb_grid* grid, const double* c_host, const double* zeta_y_host,
                          const double* zeta_x_host, double dt, size_t steps, ptb_pml** out) {
  return guarded([&] {
    require(ctx && grid && c_host && zeta_y_host && zeta_x_host && out, "PmlConfig: null argument");
    validate_grid(*grid);
    require(grid->dim == 2, "PmlConfig: the absorbing layer is two-dimensional");
    const size_t ny = grid->n[0], nx = grid->n[1], n = ny * nx;
    for (size_t i = 0; i < n; ++i)
      require(c_host[i] > 0.0 && std::isfinite(c_host[i]), "SpeedField: wave speed must be strictly positive and finite");
    for (size_t i = 0; i < ny; ++i) require(zeta_y_host[i] >= 0.0 && std::isfinite(zeta_y_host[i]), "PmlConfig: bad damping");
    for (size_t i = 0; i < nx; ++i) require(zeta_x_host[i] >= 0.0 && std::isfinite(zeta_x_host[i]), "PmlConfig: bad damping");
    require(dt > 0.0 && std::isfinite(dt), "PropagatorConfig: dt must be positive");
    require(steps > 0, "PropagatorConfig: steps_per_coupling must be positive");
    const double cmax = *std::max_element(c_host, c_host + n);
    const double hy = grid->h[0], hx = grid->h[1];
    const double cfl = dt * cmax / std::min(hy, hx), bound = 1.0 / std::sqrt(2.0);
    if (cfl > bound * (1.0 + 1e-12))
      fail(PTB_INVALID_ARGUMENT, "PropagatorConfig: CFL violated, dt*max(c)/min(h) = " + std::to_string(cfl) +
                                     " > " + std::to_string(bound));
    DevGuard g(ctx->device);
    auto* p = new ptb_pml();
    p->ctx = ctx;
    p->grid = *grid;
    p->n = n;
    p->steps = steps;
    // the expressions of oracle/pml_np.py PmlCoefficients, in the same order
    p->dt = dt;
    p->hd = 0.5 * dt;
    const double ihx2 = 1.0 / (hx * hx), ihy2 = 1.0 / (hy * hy);
    p->ry = ihy2 / ihx2;
    p->cc = -2.0 * (1.0 + p->ry);
    p->gx = 0.5 * hx;
    p->gy = (hx * hx) / (2.0 * hy);
    std::vector<double> h(n + 3 * nx + 3 * ny);
    for (size_t i = 0; i < n; ++i) h[i] = p->hd * (c_host[i] * c_host[i]) * ihx2;
    double* zx = h.data() + n;
    double* zy = zx + 3 * nx;
    for (size_t i = 0; i < nx; ++i) {
      const double z = zeta_x_host[i];
      zx[i] = z;
      zx[nx + i] = (1.0 - p->hd * z) / (1.0 + p->hd * z);
      zx[2 * nx + i] = dt / (2.0 * hx * (1.0 + p->hd * z));
    }
    for (size_t i = 0; i < ny; ++i) {
      const double z = zeta_y_host[i];
      zy[i] = z;
      zy[ny + i] = (1.0 - p->hd * z) / (1.0 + p->hd * z);
      zy[2 * ny + i] = dt / (2.0 * hy * (1.0 + p->hd * z));
    }
    PTB_CUDA_CHECK(cudaMalloc(&p->coef, h.size() * sizeof(double)));
    PTB_CUDA_CHECK(cudaMemcpy(p->coef, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
    *out = p;
  });
}

ptb_status ptb_pml_destroy(ptb_pml* p) {
  return guarded([&] {
    if (!p) return;
    DevGuard g(p->ctx->device);
    cudaFree(p->coef);
    delete p;
  });
}

ptb_status ptb_pml_propagate_batch(ptb_pml* p, size_t steps, size_t batch, double* u_dev, double* udot_dev,
                                   double* px_dev, double* py_dev, int32_t* nonfinite_dev) {
  return guarded([&] {
    require(p && u_dev && udot_dev && px_dev && py_dev, "pml propagate: null argument");
    DevGuard g(p->ctx->device);
    std::lock_guard<std::recursive_mutex> lock(p->ctx->mutex);
    pml_propagate(p, steps ? steps : p->steps, batch, u_dev, udot_dev, px_dev, py_dev, nonfinite_dev);
  });
}

}  // extern "C"
