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
// Overlapped temporal tiling, 4 steps per pass, 70 x 54 output tiles in two classes fixed per
// propagator (host tile lists built at create):
//   k_pml<true> (layer tiles: damping within 9 cells) — the tile plus a halo of H = 2S+1 cells
//     (periodic wrap, so any grid size works) in shared memory (u, px, py planes): the initial half
//     kick shrinks the valid region by one cell, each step by 2 more (the auxiliary update reads
//     new u neighbours, the force reads new auxiliary neighbours); after S steps the central tile
//     is exact.  Branch-free stages over the padded box; undamped points take the plain arithmetic.
//   k_pml_plain (all other tiles) — halo S+1, the periodic FAST step on register columns (below),
//     bitwise the periodic kernels' arithmetic (bfast<true>); two CTAs per SM.
// The carried velocity is the half kick vh (as the FAST kernel), so the drift is pointwise.  Out
// of place (halo reads of other tiles' inputs): passes ping-pong between the caller's buffers and
// the propagator's scratch.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <cstdint>
#include <limits>

#include "ptb_comm.h"
#include "ptb_driver.h"
#include "ptb_energy.h"
#include "ptb_internal.h"
#include "ptb_procrustes.h"

namespace ptb {
namespace {

constexpr int PS = 4;           // steps per pass
constexpr int HL = 2 * PS + 1;  // layer-tile halo: the first half kick costs 1 cell, each step 2
constexpr int HP = PS + 1;      // plain-tile halo: 1 cell per step + 1
constexpr int PTY = 70, PTX = 54;  // output tile (both classes): plain ext 80 x 64 = 4 x 64 threads x 20 rows

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
  const int2* tiles;                         // (ty0, tx0) of the tiles of this launch's class
  int ylim, xlim;                            // outputs only on rows < ylim, columns < xlim (0: the grid's)
};

template <int TY, int TX, int H, int NT, int HY0 = H, int HY1 = H, int HX0 = H, int HX1 = H>
struct Geo {
  static constexpr int EY = TY + HY0 + HY1, EX = TX + HX0 + HX1, EXT = EY * EX, NPT = (EXT + NT - 1) / NT;
  static constexpr int EXTP = NPT * NT;
  static constexpr int PAD = EX + 1;           // stencil reads of padded points stay in bounds
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

// 8-byte global -> shared asynchronous copy (LDGSTS)
__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gmem_src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

__device__ __forceinline__ int wrap(int i, int n) {
  i %= n;
  return i < 0 ? i + n : i;
}

// HY0/HY1/HX0/HX1 (default: the class halo H on every side): halo rows before / after the tile and
// halo columns before / after it.  A side whose rim cells are all undamped — no damping within the
// halo and the margin behind it — needs only the plain halo HP there: garbage moves one cell per
// step through undamped cells (their px, py are never updated), two through damped ones.
template <bool LAYER, int NT, int TY = PTY, int TX = PTX, int HY0 = -1, int HY1 = -1, int HX0 = -1, int HX1 = -1>
__global__ void __launch_bounds__(NT, LAYER ? 1 : 2) k_pml(const PmlArgs a) {
  constexpr int H = LAYER ? HL : HP;
  constexpr int hy0 = HY0 < 0 ? H : HY0, hy1 = HY1 < 0 ? H : HY1, hx0 = HX0 < 0 ? H : HX0, hx1 = HX1 < 0 ? H : HX1;
  using G = Geo<TY, TX, H, NT, hy0, hy1, hx0, hx1>;
  constexpr int E = G::EX, EY = G::EY, NPT = G::NPT;
  extern __shared__ double sm[];
  double* us = sm + G::PAD;
  double* pxs = sm + G::PLANE + G::PAD;      // LAYER: px; plain: the coefficient kx
  double* pys = sm + 2 * G::PLANE + G::PAD;  // LAYER only
  double* ks = pxs;
  // LAYER only: 1 / (1 + hd (zy + zx)) per point, formed once per pass (the same correctly rounded
  // quotient the second half kick would form at every step)
  [[maybe_unused]] double* ivs = sm + 3 * G::PLANE;
  double* zxs = sm + (LAYER ? 4 : 2) * G::PLANE;  // EX each: zx ax qx; EY each: zy ay qy (LAYER only)
  double* axs = zxs + E;
  double* qxs = axs + E;
  double* zys = qxs + E;
  double* ays = zys + EY;
  double* qys = ays + EY;
  int* colg = reinterpret_cast<int*>(zxs + (LAYER ? 3 * (E + EY) : 0));  // EX: global column
  int* rowg = colg + E;                                                    // EY: global row offset

  const int tid = threadIdx.x, b = blockIdx.y;
  const int2 t0 = a.tiles[blockIdx.x];
  const int ty0 = t0.x, tx0 = t0.y;

  for (int j = tid; j < E; j += NT) {
    const int gx = wrap(tx0 - hx0 + j, a.nx);
    colg[j] = gx;
    if constexpr (LAYER) {
      zxs[j] = a.zx[gx];
      axs[j] = a.ax[gx];
      qxs[j] = a.qx[gx];
    }
  }
  for (int j = tid; j < EY; j += NT) {
    const int gy = wrap(ty0 - hy0 + j, a.ny);
    rowg[j] = gy * a.nx;
    if constexpr (LAYER) {
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
  // shared planes filled with cp.async (all copies in flight together), v and k into registers
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    const int e = tid + i * NT;
    double v = 0.0, k = 0.0;
    if (e < G::EXT) {
      const int ey = e / E, ex = e - ey * E;
      const size_t g = size_t(rowg[ey]) + colg[ex];
      cp_async8(&us[e], a.ui + base + g);
      v = a.vi[base + g];
      k = a.kx[g];
      if constexpr (LAYER) {
        cp_async8(&pxs[e], a.pxi + base + g);
        cp_async8(&pys[e], a.pyi + base + g);
      }
    } else {
      us[e] = 0.0;
      if constexpr (LAYER) pxs[e] = pys[e] = 0.0;
    }
    hv[i] = v;
    if constexpr (LAYER) {
      kr[i] = k;
    } else {
      ks[e] = k;
    }
  }
  cp_async_wait_all();
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
  auto row = [](int e) { return min(e / E, EY - 1); };
  if constexpr (LAYER) {
#pragma unroll 1
    for (int i = 0; i < NPT; ++i) {
      const int e = tid + i * NT;
      const double sg = __dadd_rn(zys[row(e)], zxs[col(e)]);
      ivs[e] = __ddiv_rn(1.0, __dadd_rn(1.0, __dmul_rn(a.hd, sg)));
    }
  }

#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    const int e = tid + i * NT;
    const double f = force(e, kr[LAYER ? i : 0]);
    if constexpr (LAYER) {
      const double zx = zxs[col(e)], zy = zys[row(e)];
      hv[i] = (zx != 0.0 || zy != 0.0) ? kick_layer(hv[i], f, us[e], zx, zy, a.hd) : __dadd_rn(hv[i], f);
    } else
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
        if (zx != 0.0 || zy != 0.0) {  // undamped points: px' = 1 * px + 0 * (...) = px
          pxs[e] = __dadd_rn(__dmul_rn(axs[ex], pxs[e]),
                             __dmul_rn(__dmul_rn(__dsub_rn(zy, zx), qxs[ex]), __dsub_rn(us[e + 1], us[e - 1])));
          pys[e] = __dadd_rn(__dmul_rn(ays[ey], pys[e]),
                             __dmul_rn(__dmul_rn(__dsub_rn(zx, zy), qys[ey]), __dsub_rn(us[e + E], us[e - E])));
        }
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
        if (zx != 0.0 || zy != 0.0) {
          const double pi = __dmul_rn(zy, zx);
          const double v1 = __dmul_rn(__dadd_rn(hv[i], __dsub_rn(f, __dmul_rn(a.hd, __dmul_rn(pi, us[e])))), ivs[e]);
          hv[i] = last ? v1 : kick_layer(v1, f, us[e], zx, zy, a.hd);
        } else {  // the same values for finite fields: pi = sg = 0, inv = 1
          const double v1 = __dadd_rn(hv[i], f);
          hv[i] = last ? v1 : __dadd_rn(v1, f);
        }
      } else {
        const double v1 = hv[i] + f;
        hv[i] = last ? v1 : v1 + f;
      }
    }
  }

  // store the central tile
  const int ylim = a.ylim ? a.ylim : a.ny, xlim = a.xlim ? a.xlim : a.nx;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < NPT; ++i) {
    const int e = tid + i * NT;
    if (e < G::EXT) {
      const int ey = e / E, ex = e - ey * E;
      const int oy = ey - hy0, ox = ex - hx0;
      if (oy >= 0 && oy < TY && ox >= 0 && ox < TX && ty0 + oy < ylim && tx0 + ox < xlim) {
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

// Plain tiles (no damping within the halo): the periodic FAST step on a register column.  Thread
// t owns column t % 64 of the 80 x 64 ext box and PR = 20 consecutive rows of it: u and the
// carried half kick live in registers, so the y-neighbours come from registers (the segment ends
// and the x-neighbours from the shared u plane) — about 4 shared-memory accesses per point-step
// instead of 8 for the generic kernel.  Same arithmetic as k_pml<false> and the periodic kernels.
constexpr int PR = 20;
__global__ void __launch_bounds__(256, 2) k_pml_plain(const PmlArgs a) {
  constexpr int EX = PTX + 2 * HP, EY = PTY + 2 * HP, H = HP, PAD = EX + 1, PLANE = EY * EX + 2 * PAD;
  static_assert(EX == 64 && EY == 4 * PR, "plain tile geometry");
  extern __shared__ double sm[];
  double* us = sm + PAD;
  double* ks = sm + PLANE + PAD;
  int* colg = reinterpret_cast<int*>(sm + 2 * PLANE);  // EX
  int* rowg = colg + EX;                               // EY
  const int tid = threadIdx.x, c = tid & (EX - 1), r0 = (tid / EX) * PR;
  const int2 t0 = a.tiles[blockIdx.x];
  const int ty0 = t0.x, tx0 = t0.y;
  if (tid < EX) colg[tid] = wrap(tx0 - H + tid, a.nx);
  if (tid < EY) rowg[tid] = wrap(ty0 - H + tid, a.ny) * a.nx;
  if (tid < PAD) {
    us[tid - PAD] = us[EY * EX + tid] = 0.0;
    ks[tid - PAD] = ks[EY * EX + tid] = 0.0;
  }
  __syncthreads();
  const size_t base = size_t(blockIdx.y) * a.n;
  double u[PR], hv[PR];
  // u and the coefficient go global -> shared with cp.async (no register round trip, so all 40
  // copies of a thread are in flight together; ncu: a register-staged kx store per row
  // serialised the loads), the velocity straight into registers
#pragma unroll
  for (int r = 0; r < PR; ++r) {
    const size_t g = size_t(rowg[r0 + r]) + colg[c];
    cp_async8(&us[(r0 + r) * EX + c], a.ui + base + g);
    cp_async8(&ks[(r0 + r) * EX + c], a.kx + g);
    hv[r] = a.vi[base + g];
  }
  cp_async_wait_all();
  __syncthreads();
#pragma unroll
  for (int r = 0; r < PR; ++r) u[r] = us[(r0 + r) * EX + c];
  auto force = [&](int r, const double* uu) {
    const int e = (r0 + r) * EX + c;
    const double un = r < PR - 1 ? uu[r + 1] : us[e + EX];
    const double ud = r > 0 ? uu[r - 1] : us[e - EX];
    return bfast_y(uu[r], us[e - 1], us[e + 1], un, ud, ks[e], a.ry, a.cc);
  };
#pragma unroll
  for (int r = 0; r < PR; ++r) hv[r] = hv[r] + force(r, u);
  for (int s = 0; s < a.steps; ++s) {
    __syncthreads();  // force reads of u are done
#pragma unroll
    for (int r = 0; r < PR; ++r) {
      u[r] = u[r] + a.dt * hv[r];
      us[(r0 + r) * EX + c] = u[r];
    }
    __syncthreads();
    const bool last = s + 1 == a.steps;
#pragma unroll
    for (int r = 0; r < PR; ++r) {
      const double f = force(r, u);
      const double v1 = hv[r] + f;
      hv[r] = last ? v1 : v1 + f;
    }
  }
  bool bad = false;
  const int ox = c - H;
#pragma unroll
  for (int r = 0; r < PR; ++r) {
    const int oy = r0 + r - H;
    if (oy >= 0 && oy < PTY && ox >= 0 && ox < PTX && ty0 + oy < a.ny && tx0 + ox < a.nx) {
      const size_t g = base + size_t(ty0 + oy) * a.nx + (tx0 + ox);
      a.uo[g] = u[r];
      a.vo[g] = hv[r];
      bad |= !(isfinite(u[r]) && isfinite(hv[r]));
    }
  }
  if (a.flags) {
    bad = __syncthreads_or(bad);
    if (bad && tid == 0) atomicOr(&a.flags[blockIdx.y], 1);
  }
}
size_t pml_plain_smem() {
  constexpr int EX = PTX + 2 * HP, EY = PTY + 2 * HP;
  return size_t(2 * (EY * EX + 2 * (EX + 1))) * sizeof(double) + (EX + EY) * sizeof(int);
}

constexpr int kPlainThreads = 256, kLayerThreads = 512;

// frame mode (a standard layer: damped bands at both ends of each axis, undamped interior): the
// interior rectangle runs k_wave2, the four bands run the layer kernel on band-shaped tiles —
// FB rows x PTX columns (top and bottom), PTY rows x FB columns (left and right)
constexpr int FB = 40;
constexpr int FRAME_MARGIN = PS + 2;  // interior rectangle starts this far from the last damped cell
// super-pass (2 PS steps): the interior runs ONE 2 PS-step wavefront launch on the rectangle
// SUPER_MARGIN cells from the damped bands, the bands two PS-step passes — pass A into a third
// buffer set (its outputs feed pass B's halo), pass B into the output.  Pass B covers bands FBB
// wide.  Band tile classes of a pass:
//   corner tiles (the band ends, where the cells beyond the band's inner edge are damped by the
//     crossing band): the layer halo HL on every side; pass A's are FBA = FBB + HL wide and
//     two tiles long, so pass B's corner tiles (one tile long) find all their inputs;
//   mid tiles (top/bottom between the corners) and left/right tiles: the cells beyond the inner
//     edge are undamped for SUPER_MARGIN + HP cells, so the plain halo HP suffices there (k_pml's
//     HY0..HX1); pass A's are FBM = FBB + HP wide.  Their tile lengths fill 10 points per thread.
constexpr int SUPER_MARGIN = 2 * PS + 2;
constexpr int FBB = 32 + SUPER_MARGIN, FBA = FBB + HL, FBM = FBB + HP;  // 42, 51, 47 (layers up to 32 cells)
constexpr int LA = 64, LB = 72;                                         // mid / left-right tile lengths, pass A / B
constexpr int XCA = 2 * PTX, XCB = PTX;                                 // corner-class extent along the band

template <bool LAYER, int TY = PTY, int TX = PTX, int HY0 = -1, int HY1 = -1, int HX0 = -1, int HX1 = -1>
size_t pml_smem() {
  constexpr int H = LAYER ? HL : HP;
  using G = Geo<TY, TX, H, LAYER ? kLayerThreads : kPlainThreads, (HY0 < 0 ? H : HY0), (HY1 < 0 ? H : HY1),
                (HX0 < 0 ? H : HX0), (HX1 < 0 ? H : HX1)>;
  return size_t(G::PLANE) * (LAYER ? 4 : 2) * sizeof(double) + (LAYER ? 3 * (G::EX + G::EY) * sizeof(double) : 0) +
         (G::EX + G::EY) * sizeof(int);
}

// the super-pass band kernels (fixed instantiations; BandLaunch::kern indexes this table)
struct BandKernel {
  const void* fn;
  size_t smem;
};
template <int TY, int TX, int HY0 = -1, int HY1 = -1, int HX0 = -1, int HX1 = -1>
BandKernel band_kernel() {
  return {reinterpret_cast<const void*>(k_pml<true, kLayerThreads, TY, TX, HY0, HY1, HX0, HX1>),
          pml_smem<true, TY, TX, HY0, HY1, HX0, HX1>()};
}
enum { BK_A_CORNER, BK_A_TOP, BK_A_BOT, BK_A_LEFT, BK_A_RIGHT, BK_B_CORNER, BK_B_TOP, BK_B_BOT, BK_B_LEFT, BK_B_RIGHT, BK_COUNT };
const BandKernel* band_kernels() {
  static const BandKernel k[BK_COUNT] = {
      band_kernel<FBA, PTX>(),
      band_kernel<FBM, LA, HL, HP, HL, HL>(),  // top: the inner side is below
      band_kernel<FBM, LA, HP, HL, HL, HL>(),  // bottom: above
      band_kernel<LA, FBM, HL, HL, HL, HP>(),  // left: to the right
      band_kernel<LA, FBM, HL, HL, HP, HL>(),  // right: to the left
      band_kernel<FBB, PTX>(),
      band_kernel<FBB, LB, HL, HP, HL, HL>(),
      band_kernel<FBB, LB, HP, HL, HL, HL>(),
      band_kernel<LB, FBB, HL, HL, HL, HP>(),
      band_kernel<LB, FBB, HL, HL, HP, HL>(),
  };
  return k;
}
struct BandLaunch {
  int kern, first, count, ylim, xlim;  // kernel, tile range in ptb_pml::stiles, output clips (0: none)
};

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
  double* speed = nullptr;  // c (n): the energy map of the theta coupling
  ptb::DeviceBuffer scratch;  // 4 fields x batch (ping-pong partner; phi planes zeroed once)
  size_t scratch_batch = 0;
  int2* tiles = nullptr;       // plain tiles, then layer tiles (PT x PT, classified at create)
  int nplain = 0, nlayer = 0;
  // the plain tiles as one rectangle (rows [ry0, ry0 + rny), columns [rx0, rx0 + rnx)) when they
  // form one: the interior then runs the periodic wavefront kernel (k_wave2) instead of k_pml_plain
  int ry0 = 0, rny = 0, rx0 = 0, rnx = 0;
  ptb::StepParams prm{};
  // frame mode: interior rectangle and the band tiles (top/bottom FB x PTX, then left/right PTY x FB)
  int frame = 0, fy0 = 0, fny = 0, fx0 = 0, fnx = 0, ntb = 0, nlr = 0;
  int2* ftiles = nullptr;
  // super-pass geometry (see SUPER_MARGIN): interior rectangle, pass-A and pass-B band tiles
  // (top/bottom then left/right in each list), and the buffer set pass A writes
  int super = 0, sy0 = 0, sny = 0, sx0 = 0, snx = 0;
  int2* stiles = nullptr;                       // the band tiles of both passes
  std::vector<ptb::BandLaunch> pass_a, pass_b;  // band launches of pass A / pass B
  // a pass's band launches are independent one-CTA-per-SM kernels: each class on its own stream, so
  // one class's last partial round overlaps the next class's first
  static constexpr int NBS = 5;
  cudaStream_t bstream[NBS] = {};
  cudaEvent_t bfork = nullptr, bev[NBS] = {};
  ptb::DeviceBuffer mid;
  size_t mid_batch = 0;
};

namespace ptb {

// PTB_PML_WAVE=0: interior tiles through k_pml_plain (A/B measurements, tests)
bool pml_wave_enabled() {
  const char* e = std::getenv("PTB_PML_WAVE");
  return !(e && std::atoi(e) == 0);
}
// PTB_PML_FRAME=0: the 70 x 54 tile classes instead of the frame (A/B measurements, tests)
bool pml_frame_enabled() {
  const char* e = std::getenv("PTB_PML_FRAME");
  return !(e && std::atoi(e) == 0);
}

// PTB_PML_SUPER=0: PS-step passes only (A/B measurements, tests)
bool pml_super_enabled() {
  const char* e = std::getenv("PTB_PML_SUPER");
  return !(e && std::atoi(e) == 0);
}

// Size the propagator's ping-pong scratch (and the super-pass's third buffer set) for `batch` slices
// now, so that a later, larger batch does not reallocate them inside a timed region (a cudaFree +
// cudaMalloc pair of this size synchronises the device and was measured at 2-700 ms).
void pml_reserve(ptb_pml* p, size_t batch) {
  if (batch == 0) return;
  const size_t fb = batch * p->n * sizeof(double);
  if (p->scratch_batch < batch) {
    double* s = static_cast<double*>(p->scratch.get(4 * fb));
    PTB_CUDA_CHECK(cudaMemsetAsync(s, 0, 4 * fb, p->ctx->stream));  // phi planes: zero off the layer, for good
    p->scratch_batch = batch;
  }
  if (p->super && p->mid_batch < batch) {
    p->mid.get(4 * fb);
    p->mid_batch = batch;
  }
}

// `src` (optional): the input state (u, udot, px, py); the result still goes to u, v, px, py, whose
// px, py must then already be zero off the layer (the interior kernels never write them).  Saves
// the caller a copy of the whole state when it keeps the input.
void pml_propagate(ptb_pml* p, size_t steps, size_t batch, double* u, double* v, double* px, double* py,
                   int32_t* flags, const double* const* src = nullptr) {
  ptb_context* ctx = p->ctx;
  cudaStream_t st = ctx->stream;
  if (batch == 0 || steps == 0) return;
  const int ny = int(p->grid.n[0]), nx = int(p->grid.n[1]);
  const size_t n = p->n, fb = batch * n * sizeof(double);
  pml_reserve(p, batch);
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
  // the dynamic shared-memory opt-in is per device
  static std::atomic<uint64_t> attr_done{0};
  const uint64_t bit = uint64_t(1) << (ctx->device & 63);
  if (!(attr_done.load() & bit)) {
    PTB_CUDA_CHECK(cudaFuncSetAttribute(k_pml_plain, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(pml_plain_smem())));
    PTB_CUDA_CHECK(cudaFuncSetAttribute(k_pml<true, kLayerThreads>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(pml_smem<true>())));
    PTB_CUDA_CHECK(cudaFuncSetAttribute(k_pml<true, kLayerThreads, FB, PTX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(pml_smem<true, FB, PTX>())));
    PTB_CUDA_CHECK(cudaFuncSetAttribute(k_pml<true, kLayerThreads, PTY, FB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        int(pml_smem<true, PTY, FB>())));
    for (int i = 0; i < BK_COUNT; ++i)
      PTB_CUDA_CHECK(cudaFuncSetAttribute(band_kernels()[i].fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(band_kernels()[i].smem)));
    attr_done.fetch_or(bit);
  }
  require(batch <= 65535, "pml propagate: at most 65535 slices per call");
  // PTB_PML_LANES=0: every launch of a pass on the one stream (A/B measurements)
  static const bool lanes_env = [] {
    const char* e = std::getenv("PTB_PML_LANES");
    return !(e && std::atoi(e) == 0);
  }();
  const bool lanes = lanes_env && p->frame;
  const bool super = p->super && steps >= size_t(2 * PS) && pml_wave_enabled() && pml_frame_enabled() &&
                     pml_super_enabled();
  double* mid[4] = {nullptr, nullptr, nullptr, nullptr};
  if (super) {
    double* m = static_cast<double*>(p->mid.ptr);
    const size_t mb = p->mid_batch * n;
    for (int f = 0; f < 4; ++f) mid[f] = m + f * mb;
  }
  constexpr int NBS = ptb_pml::NBS;
  if (lanes && !p->bfork) {
    PTB_CUDA_CHECK(cudaEventCreateWithFlags(&p->bfork, cudaEventDisableTiming));
    for (int i = 0; i < NBS; ++i) {
      PTB_CUDA_CHECK(cudaStreamCreateWithFlags(&p->bstream[i], cudaStreamNonBlocking));
      PTB_CUDA_CHECK(cudaEventCreateWithFlags(&p->bev[i], cudaEventDisableTiming));
    }
  }
  int cur = 0;
  bool first = true;  // the first pass reads `src` when given
  for (size_t done = 0; done < steps;) {
    if (super && steps - done >= size_t(2 * PS)) {
      // One super-pass = 2 PS steps.  Band pass A (PS steps, bands FBA wide) reads the input and writes
      // the third buffer set; band pass B (PS steps, bands FBB wide) reads that — its halo ends where
      // pass A's outputs end — and writes the output; the interior rectangle advances 2 PS steps in
      // one wavefront launch (its cone stays SUPER_MARGIN - 2 PS cells away from damped cells).  The
      // band passes go to the lane stream, the interior to the caller's.
      done += 2 * PS;
      a.flags = done == steps ? flags : nullptr;
      a.steps = PS;
      if (lanes) {
        PTB_CUDA_CHECK(cudaEventRecord(p->bfork, st));
        for (int i = 0; i < NBS; ++i) PTB_CUDA_CHECK(cudaStreamWaitEvent(p->bstream[i], p->bfork, 0));
      }
      const double* in[4];
      for (int f = 0; f < 4; ++f) in[f] = (first && src) ? src[f] : bufs[cur][f];
      first = false;
      PmlArgs pa = a;
      pa.flags = nullptr;
      pa.ui = in[0], pa.vi = in[1], pa.pxi = in[2], pa.pyi = in[3];
      pa.uo = mid[0], pa.vo = mid[1], pa.pxo = mid[2], pa.pyo = mid[3];
      PmlArgs pb = a;
      pb.ui = mid[0], pb.vi = mid[1], pb.pxi = mid[2], pb.pyi = mid[3];
      pb.uo = bufs[1 - cur][0], pb.vo = bufs[1 - cur][1], pb.pxo = bufs[1 - cur][2], pb.pyo = bufs[1 - cur][3];
      auto run = [&](const std::vector<BandLaunch>& pass, PmlArgs& args) {
        for (size_t i = 0; i < pass.size(); ++i) {
          const BandLaunch& bl = pass[i];
          if (bl.count == 0) continue;
          args.tiles = p->stiles + bl.first;
          args.ylim = bl.ylim;
          args.xlim = bl.xlim;
          void* kargs[] = {&args};
          const BandKernel& bk = band_kernels()[bl.kern];
          PTB_CUDA_CHECK(cudaLaunchKernel(bk.fn, dim3(unsigned(bl.count), unsigned(batch)), dim3(kLayerThreads), kargs,
                                          bk.smem, lanes ? p->bstream[i % NBS] : st));
          PTB_LAUNCH_CHECK(ctx);
        }
      };
      // every band stream sees all of the pass's launches before the next pass / the join
      auto barrier = [&](bool join) {
        if (!lanes) return;
        for (int i = 0; i < NBS; ++i) PTB_CUDA_CHECK(cudaEventRecord(p->bev[i], p->bstream[i]));
        for (int i = 0; i < NBS; ++i) {
          if (join) {
            PTB_CUDA_CHECK(cudaStreamWaitEvent(st, p->bev[i], 0));
          } else {
            for (int j = 0; j < NBS; ++j)
              if (j != i) PTB_CUDA_CHECK(cudaStreamWaitEvent(p->bstream[j], p->bev[i], 0));
          }
        }
      };
      run(p->pass_a, pa);
      barrier(false);
      run(p->pass_b, pb);
      wave_rect_fast(ctx, st, 2 * PS, p->prm, batch, in[0], in[1], bufs[1 - cur][0], bufs[1 - cur][1],
                     a.kx, a.flags, p->sy0, p->sny, p->sx0, p->snx);
      barrier(true);
      cur = 1 - cur;
      continue;
    }
    const int ns = int(std::min<size_t>(PS, steps - done));
    done += ns;
    a.ui = (first && src) ? src[0] : bufs[cur][0];
    a.vi = (first && src) ? src[1] : bufs[cur][1];
    a.pxi = (first && src) ? src[2] : bufs[cur][2];
    a.pyi = (first && src) ? src[3] : bufs[cur][3];
    first = false;
    a.uo = bufs[1 - cur][0];
    a.vo = bufs[1 - cur][1];
    a.pxo = bufs[1 - cur][2];
    a.pyo = bufs[1 - cur][3];
    a.steps = ns;
    a.flags = done == steps ? flags : nullptr;
    if (p->frame && (ns == 4 || ns == 2 || ns == 1) && pml_wave_enabled() && pml_frame_enabled()) {
      // frame mode: the interior rectangle through k_wave2, the bands through band-shaped layer tiles
      // The three launches of a pass read the same input and write disjoint parts of the output.
      // Band tiles: top/bottom and left/right on their own streams (independent one-CTA-per-SM
      // kernels; on a small grid each is one CTA latency long), the interior on the caller's
      cudaStream_t bs0 = st, bs1 = st;
      if (lanes) {
        PTB_CUDA_CHECK(cudaEventRecord(p->bfork, st));
        PTB_CUDA_CHECK(cudaStreamWaitEvent(p->bstream[0], p->bfork, 0));
        PTB_CUDA_CHECK(cudaStreamWaitEvent(p->bstream[1], p->bfork, 0));
        bs0 = p->bstream[0];
        bs1 = p->bstream[1];
      }
      a.tiles = p->ftiles;
      k_pml<true, kLayerThreads, FB, PTX><<<dim3(p->ntb, unsigned(batch)), kLayerThreads, pml_smem<true, FB, PTX>(),
                                            bs0>>>(a);
      PTB_LAUNCH_CHECK(ctx);
      a.tiles = p->ftiles + p->ntb;
      k_pml<true, kLayerThreads, PTY, FB><<<dim3(p->nlr, unsigned(batch)), kLayerThreads, pml_smem<true, PTY, FB>(),
                                            bs1>>>(a);
      PTB_LAUNCH_CHECK(ctx);
      wave_rect_fast(ctx, st, ns, p->prm, batch, a.ui, a.vi, a.uo, a.vo, a.kx, a.flags, p->fy0, p->fny, p->fx0,
                     p->fnx);
      if (lanes) {
        for (int i = 0; i < 2; ++i) {
          PTB_CUDA_CHECK(cudaEventRecord(p->bev[i], p->bstream[i]));
          PTB_CUDA_CHECK(cudaStreamWaitEvent(st, p->bev[i], 0));
        }
      }
      cur = 1 - cur;
      continue;
    }
    if (p->nplain && p->rnx && (ns == 4 || ns == 2 || ns == 1) && pml_wave_enabled()) {
      // the undamped interior: the periodic FAST wavefront kernel on the plain-tile rectangle
      // (bitwise k_pml_plain's arithmetic; its S-step cone stays in undamped cells, px = py = 0)
      wave_rect_fast(ctx, st, ns, p->prm, batch, a.ui, a.vi, a.uo, a.vo, a.kx, a.flags, p->ry0, p->rny, p->rx0,
                     p->rnx);
    } else if (p->nplain) {
      a.tiles = p->tiles;
      k_pml_plain<<<dim3(p->nplain, unsigned(batch)), 256, pml_plain_smem(), st>>>(a);
      PTB_LAUNCH_CHECK(ctx);
    }
    if (p->nlayer) {
      a.tiles = p->tiles + p->nplain;
      k_pml<true, kLayerThreads><<<dim3(p->nlayer, unsigned(batch)), kLayerThreads, pml_smem<true>(), st>>>(a);
      PTB_LAUNCH_CHECK(ctx);
    }
    cur = 1 - cur;
  }
  if (cur == 1)  // odd number of passes: the result is in the scratch
    for (int f = 0; f < 4; ++f)
      PTB_CUDA_CHECK(cudaMemcpyAsync(bufs[0][f], bufs[1][f], fb, cudaMemcpyDeviceToDevice, st));
}


// ---------------------------------------------------------------- plain parareal with the layer
namespace {

__global__ void k_sweep_diff(size_t n, const double* g, const double* old, const double* rf, double* d, double* w) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const double di = g[i] - old[i];
    d[i] = di;
    w[i] = rf[i] + di;
  }
}
__global__ void k_add_into(size_t n, double* x, const double* y) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    x[i] = x[i] + y[i];
}
// auxiliary fields of an interpolated correction: px, py vanish identically where the cell is
// undamped (zx = zy = 0: px_t = py_t = 0 from a zero start), so the interpolant's spread into
// the interior (Fourier I rings across the whole row) is cut back to the layer; x += mask * y
__global__ void k_aux_mask_add(size_t total, int ny, int nx, const double* __restrict__ zx,
                               const double* __restrict__ zy, double* x, const double* __restrict__ y) {
  const size_t n = size_t(ny) * nx;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
    const size_t p = i % n;
    const int iy = int(p / nx), ix = int(p - size_t(iy) * nx);
    if (zx[ix] != 0.0 || zy[iy] != 0.0) x[i] = x[i] + y[i];
  }
}
// x = 0 where undamped (iterate 0's interpolated auxiliary fields)
__global__ void k_aux_mask(size_t total, int ny, int nx, const double* __restrict__ zx, const double* __restrict__ zy,
                           double* x) {
  const size_t n = size_t(ny) * nx;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
    const size_t p = i % n;
    const int iy = int(p / nx), ix = int(p - size_t(iy) * nx);
    if (zx[ix] == 0.0 && zy[iy] == 0.0) x[i] = 0.0;
  }
}
// finalize_iteration (parareal.cpp:117-124) on the layered state: slice s of `next` with any
// non-finite entry in its four fields is flagged (bad[s], and the divergence flags) ...
// (px, py null: their finiteness is known already — `known_bad`, the fine stage's flag of the slice,
// whose px, py the iterate carries unchanged)
__global__ void __launch_bounds__(256) k_state_bad(size_t n, const double* u, const double* v, const double* px,
                                                    const double* py, const int32_t* known_bad, int32_t* bad,
                                                    int32_t* flags) {
  const size_t o = size_t(blockIdx.y) * n;
  bool ok = !(known_bad && known_bad[blockIdx.y]);
  if (px) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
      ok &= isfinite(u[o + i]) && isfinite(v[o + i]) && isfinite(px[o + i]) && isfinite(py[o + i]);
  } else {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
      ok &= isfinite(u[o + i]) && isfinite(v[o + i]);
  }
  if (__syncthreads_or(!ok) && threadIdx.x == 0) {
    atomicOr(bad + blockIdx.y, 1);
    atomicOr(flags + blockIdx.y, 1);
  }
}
// ... and clamped to the previous iterate
__global__ void k_clamp_bad(size_t n, const int32_t* bad, double* const* dst, const double* const* src) {
  if (!bad[blockIdx.y]) return;
  const size_t o = size_t(blockIdx.y) * n;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
#pragma unroll
    for (int f = 0; f < 4; ++f) dst[f][o + i] = src[f][o + i];
}

// per slice (one block each, fixed-order reduction): out[2b] = sum (a-b)^2, out[2b+1] = sum b^2 over [u; udot]
__global__ void __launch_bounds__(512) k_err_sums(size_t n, const double* au, const double* av, const double* bu,
                                                  const double* bv, double* out) {
  const size_t o = size_t(blockIdx.x) * n;
  double e = 0.0, r = 0.0;
  for (size_t i = threadIdx.x; i < n; i += 512) {
    const double du = au[o + i] - bu[o + i], dv = av[o + i] - bv[o + i];
    e += du * du + dv * dv;
    r += bu[o + i] * bu[o + i] + bv[o + i] * bv[o + i];
  }
  __shared__ double se[512], sr[512];
  se[threadIdx.x] = e;
  sr[threadIdx.x] = r;
  __syncthreads();
  for (int k = 256; k > 0; k >>= 1) {
    if (int(threadIdx.x) < k) {
      se[threadIdx.x] += se[threadIdx.x + k];
      sr[threadIdx.x] += sr[threadIdx.x + k];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = se[0];
    out[2 * blockIdx.x + 1] = sr[0];
  }
}

// theta coupling, one sweep step's tail on the layered coarse state (one launch): the (u, udot)
// part d = Z dz + (m_w - m_old)/N_c (dl: Z dz as [du; dv], null when the corrector is empty); the
// auxiliary fields are not corrected (d = 0: next[n]'s px, py are fine_next[n]'s — correcting them
// additively, as plain parareal does, is unstable: DESIGN.md 3.7); d := NaN when g, old[n] or
// fine_next[n] is non-finite (parareal.cpp:323-326); then w = R(fine_next[n]) + d for all four
// fields (the next step's R(next[n]), R(I(d)) = d at the coarse nodes).  g and w share storage.
struct Fields4 {
  double* f[4];
};
__global__ void k_theta_tail(size_t nc, const double* __restrict__ dl, const double* __restrict__ mw,
                             const double* __restrict__ mold, const int32_t* gbad, const int32_t* obad,
                             const int32_t* fbad, Fields4 g, Fields4 rf, Fields4 d) {
  const bool nan = *gbad || *obad || *fbad;
  const double dm = (*mw - *mold) / double(nc);
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < nc; i += size_t(gridDim.x) * blockDim.x) {
    double di[4];
    di[0] = (dl ? dl[i] : 0.0) + dm;
    di[1] = dl ? dl[nc + i] : 0.0;
    di[2] = 0.0;
    di[3] = 0.0;
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const double x = nan ? __longlong_as_double(0x7ff8000000000000LL) : di[f];
      d.f[f][i] = x;
      g.f[f][i] = rf.f[f][i] + x;
    }
  }
}
__global__ void k_sub_small(int n, const double* a, const double* b, double* out) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) out[i] = a[i] - b[i];
}
__global__ void k_or_flags(size_t n, const int32_t* src, int32_t* dst) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    dst[i] |= src[i];
}

unsigned ew_blocks(ptb_context* ctx, size_t n) {
  return unsigned(std::max<size_t>(1, std::min<size_t>((n + 255) / 256, size_t(ctx->num_sms) * 8)));
}

// a set of (N+1) states of 4 fields each: field f of state s at base + (f*(N+1) + s)*n
struct States {
  double* base = nullptr;
  size_t n = 0, count = 0;
  double* f(int field, size_t s = 0) const { return base + (size_t(field) * count + s) * n; }
};

}  // namespace

// Slices block-sharded over the ranks of `comm` (null: one GPU), as the periodic driver
// (driver.cu): rank r owns couplings n in [a, b) and the fine states a-1 .. b-1; per iteration one
// all-gather of the coarse payload (C(R cur[n-1]) and R(fine_next[n]), 4 fields each) feeds the
// replicated, deterministic coarse sweep, and the last own state goes to rank r+1.  Results are
// bitwise independent of the world size.
// th (nullable): the theta (Procrustes) coupling instead of plain parareal — oracle/pml_np.py
// theta_parareal: (u, udot) corrected through Lambda-dagger Omega Lambda with the coarse speed, the
// auxiliary fields additively; the corrector is fitted on the (u, udot) snapshots of the slices
// whose four fields are finite.
struct PmlTheta {
  double tol = 1e-4;
  int scheme = PTB_FD2;
  int* ranks = nullptr;        // [K] corrector rank per iteration (nullable)
  double* residual = nullptr;  // [K] relative_residual of the fit (nullable)
};

void pml_parareal(ptb_pml* fine, ptb_pml* coarse, ptb_transfer* t, const Comm* comm, size_t N, int K,
                  const double* u0, const double* v0, double* err_out, double* ms_out, double* states_out,
                  int32_t* diverged_out, const PmlTheta* th = nullptr) {
  ptb_context* ctx = fine->ctx;
  cudaStream_t st = ctx->stream;
  const size_t nf = fine->n, nc = coarse->n;
  auto same = [](const ptb_grid& a, const ptb_grid& b) {
    return a.dim == b.dim && a.n[0] == b.n[0] && a.n[1] == b.n[1] && a.h[0] == b.h[0] && a.h[1] == b.h[1];
  };
  require(same(fine->grid, t->fine) && same(coarse->grid, t->coarse), "pml parareal: grids do not match the transfer");
  const double tf = fine->dt * double(fine->steps), tc = coarse->dt * double(coarse->steps);
  require(std::fabs(tf - tc) <= 1e-12 * std::max(tf, tc), "CouplingSchedule: fine and coarse couplings differ");
  require(N >= 1 && K >= 0, "pml parareal: need N >= 1 couplings and K >= 0 iterations");
  const int rank = comm ? comm->rank : 0, world = comm ? comm->world : 1;
  const size_t chunk = (N + size_t(world) - 1) / size_t(world);
  const size_t a = std::min(N + 1, 1 + size_t(rank) * chunk), b = std::min(N + 1, a + chunk), L = b - a;
  const size_t P = size_t(world) * chunk;  // padded global coarse slots (slot n-1 <-> coupling n)
  // device state: own fine states a-1 .. b-1 (local 0 .. L), the init state, coarse work
  DeviceBuffer bcur, bnext, bref, bini, bc, bflag, bsum, bchunk, bpay, ball, bgs;
  States cur{static_cast<double*>(bcur.get(4 * (L + 1) * nf * sizeof(double))), nf, L + 1};
  States nxt{static_cast<double*>(bnext.get(4 * (L + 1) * nf * sizeof(double))), nf, L + 1};
  States ref{static_cast<double*>(bref.get(4 * (L + 1) * nf * sizeof(double))), nf, L + 1};
  States ini{static_cast<double*>(bini.get(4 * 2 * nf * sizeof(double))), nf, 2};  // init + a work state
  double* cw = static_cast<double*>(bc.get(4 * (3 * P + 2) * nc * sizeof(double)));
  States cold{cw, nc, P}, crf{cw + 4 * P * nc, nc, P}, cd{cw + 8 * P * nc, nc, P};
  States cwv{cw + 12 * P * nc, nc, 1}, cg{cw + 12 * P * nc + 4 * nc, nc, 1};
  int32_t* flags = static_cast<int32_t*>(bflag.get((L + 1) * sizeof(int32_t)));
  // theta: per-iteration stage flags (own fine, own coarse), their global copies, the corrector
  const bool theta = th != nullptr;
  const size_t rows = 3 * nc;  // stacked (c dx u, c dy u, udot) on the coarse grid
  DeviceBuffer bsf, bgf, bth, bZ, bidx, bsw;
  int32_t *ffl = nullptr, *cfl = nullptr, *gff = nullptr, *gcf = nullptr, *swf = nullptr;
  double *Fm = nullptr, *Gm = nullptr, *cmp = nullptr, *zold = nullptr, *mold = nullptr, *zw = nullptr,
         *mw = nullptr, *dl = nullptr, *dz = nullptr;
  int* idx_d = nullptr;
  DevCorrector corr;
  EnergyWork ew(ctx);
  if (theta) {
    check_tol(th->tol);
    require(th->scheme >= PTB_FD2 && th->scheme <= PTB_SPECTRAL, "pml theta: unknown gradient scheme");
    ffl = static_cast<int32_t*>(bsf.get(2 * (chunk + 1) * sizeof(int32_t)));
    cfl = ffl + chunk + 1;
    gff = static_cast<int32_t*>(bgf.get(2 * P * sizeof(int32_t)));
    gcf = gff + P;
    swf = static_cast<int32_t*>(bsw.get((N + 1) * sizeof(int32_t)));
    double* w = static_cast<double*>(bth.get((3 * rows * N + 4 * N + 2) * sizeof(double)));
    Fm = w;
    Gm = Fm + rows * N;
    cmp = Gm + rows * N;   // Lambda of the old terms (rows x (N-1)), then of w (batch 1)
    mold = cmp + rows * N;  // N
    mw = mold + N;          // 1 (+1 pad)
    idx_d = static_cast<int*>(bidx.get(N * sizeof(int)));
    require(ctx->num_sms > 0, "pml theta: context");
    {  // the rank-sized buffers for a corrector of up to 2 N columns now: their growth inside an
       // iteration is a cudaFree + cudaMalloc pair each (device synchronisation, measured 2-700 ms);
       // a larger rank still grows them geometrically
      const size_t rcap = std::min<size_t>(rows, 2 * N);
      ProcWork& w0 = context_proc_work(ctx);
      for (DeviceBuffer* bf : {&corr.X, &corr.Y, &w0.SX, &w0.SY}) bf->get(rows * rcap * sizeof(double));
      bZ.get((2 * nc * rcap + 2 * nc + rcap * (N + 2)) * sizeof(double));
      for (int i = 1; i <= 3; ++i) ew.buf[i].get(nc * rcap * 2 * sizeof(double));  // Lambda-dagger of X (complex planes)
    }
  }
  const double* ccs = coarse->speed;
  double* sums = static_cast<double*>(bsum.get(2 * (chunk + 2) * sizeof(double)));
  const size_t ichunk = std::max<size_t>(1, std::min<size_t>(L, 8));
  DeviceBuffer bbad, bptr;
  int32_t* bad = static_cast<int32_t*>(bbad.get((L + 1) * sizeof(int32_t)));
  double** dptr = static_cast<double**>(bptr.get(8 * sizeof(double*)));
  double* hptr[8];
  double* fchunk = static_cast<double*>(bchunk.get(ichunk * nf * sizeof(double)));
  auto cpy = [&](double* dst, const double* src, size_t count) {
    if (count) PTB_CUDA_CHECK(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyDeviceToDevice, st));
  };
  auto cpy_state = [&](const States& D, size_t ds, const States& S, size_t ss) {
    for (int f = 0; f < 4; ++f) cpy(D.f(f, ds), S.f(f, ss), D.n);
  };
  PTB_CUDA_CHECK(cudaMemcpyAsync(ini.f(0), u0, nf * sizeof(double), cudaMemcpyHostToDevice, st));
  PTB_CUDA_CHECK(cudaMemcpyAsync(ini.f(1), v0, nf * sizeof(double), cudaMemcpyHostToDevice, st));
  PTB_CUDA_CHECK(cudaMemsetAsync(ini.f(2), 0, 2 * nf * sizeof(double), st));  // px, py of state 0
  PTB_CUDA_CHECK(cudaMemsetAsync(ini.f(3), 0, 2 * nf * sizeof(double), st));
  PTB_CUDA_CHECK(cudaMemsetAsync(flags, 0, (L + 1) * sizeof(int32_t), st));
  PTB_CUDA_CHECK(cudaMemsetAsync(cw, 0, 4 * (3 * P + 2) * nc * sizeof(double), st));
  pml_reserve(fine, L);  // the batched stages' buffers now, not inside the first iteration
  pml_reserve(coarse, L);
  // serial fine reference (parareal.cpp:190-199): the chain up to b-1, own states kept
  cpy_state(ini, 1, ini, 0);
  for (size_t n = 0; n < b; ++n) {
    if (n > 0) pml_propagate(fine, fine->steps, 1, ini.f(0, 1), ini.f(1, 1), ini.f(2, 1), ini.f(3, 1), nullptr);
    if (n + 1 >= a) cpy_state(ref, n + 1 - a, ini, 1);
  }
  // iterate 0: the serial coarse chain, interpolated (parareal.cpp:139-145), own states
  for (int f = 0; f < 4; ++f) restrict_fields(t, 1, ini.f(f, 0), cwv.f(f));
  if (a == 1) cpy_state(cur, 0, ini, 0);
  const int fny = int(fine->grid.n[0]), fnx = int(fine->grid.n[1]);
  const double* fzx = fine->coef + nf;             // coef layout: kx (n) | zx ax qx (nx) | zy ay qy (ny)
  const double* fzy = fine->coef + nf + 3 * size_t(fnx);
  for (size_t n = 1; n < b; ++n) {
    pml_propagate(coarse, coarse->steps, 1, cwv.f(0), cwv.f(1), cwv.f(2), cwv.f(3), nullptr);
    if (n + 1 >= a) {
      for (int f = 0; f < 4; ++f) interpolate_fields(t, 1, cwv.f(f), cur.f(f, n + 1 - a));
      for (int f = 2; f < 4; ++f) {
        k_aux_mask<<<ew_blocks(ctx, nf), 256, 0, st>>>(nf, fny, fnx, fzx, fzy, cur.f(f, n + 1 - a));
        PTB_LAUNCH_CHECK(ctx);
      }
    }
  }
  // init norm (errors are relative to it)
  k_err_sums<<<1, 512, 0, st>>>(nf, ini.f(0), ini.f(1), ini.f(0), ini.f(1), sums);
  PTB_LAUNCH_CHECK(ctx);
  double init_sums[2];
  PTB_CUDA_CHECK(cudaMemcpyAsync(init_sums, sums, sizeof(init_sums), cudaMemcpyDeviceToHost, st));
  PTB_CUDA_CHECK(cudaStreamSynchronize(st));
  const double init_norm2 = init_sums[1];

  cudaEvent_t e0, e1;
  PTB_CUDA_CHECK(cudaEventCreate(&e0));
  PTB_CUDA_CHECK(cudaEventCreate(&e1));
  const size_t per = 8 * chunk * nc;  // payload doubles per rank: cold and crf, 4 fields each
  const size_t per_b = per * sizeof(double) + (theta ? 2 * chunk * sizeof(int32_t) + 8 : 0);  // + flags
  double* own = static_cast<double*>(bpay.get(per_b));
  double* all = static_cast<double*>(ball.get(per_b * size_t(world)));
  std::vector<double> hs(2 * (chunk + 1) * size_t(world));
  double* gsums = static_cast<double*>(bgs.get(hs.size() * sizeof(double)));
  ProcWork* pw = theta ? &context_proc_work(ctx) : nullptr;
  const ptb_grid& cgr = coarse->grid;
  // theta: fit the corrector on this iteration's snapshots, then the replicated coarse sweep -> cd
  HostProf* hp_it = nullptr;  // the running iteration's PTB_PROF timeline
  auto theta_iteration = [&](int k) {
    std::vector<int32_t> hf(2 * N);
    PTB_CUDA_CHECK(cudaMemcpyAsync(hf.data(), gff, N * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    PTB_CUDA_CHECK(cudaMemcpyAsync(hf.data() + N, gcf, N * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    PTB_CUDA_CHECK(cudaStreamSynchronize(st));
    std::vector<int> keep;
    for (size_t n = 1; n <= N; ++n)
      if (!hf[n - 1] && !hf[N + n - 1]) keep.push_back(int(n - 1));
    double res = std::numeric_limits<double>::quiet_NaN();
    if (!keep.empty()) {  // assemble_snapshots (procrustes.cpp:158-175) on the (u, udot) part
      const int cols = int(keep.size());
      PTB_CUDA_CHECK(cudaMemcpyAsync(idx_d, keep.data(), keep.size() * sizeof(int), cudaMemcpyHostToDevice, st));
      energy_components(ew, cgr, th->scheme, size_t(cols), crf.f(0), crf.f(1), nc, idx_d, ccs, Fm, rows, nullptr);
      energy_components(ew, cgr, th->scheme, size_t(cols), cold.f(0), cold.f(1), nc, idx_d, ccs, Gm, rows, nullptr);
      pw->comm = comm;
      update_svd(*pw, corr, Fm, Gm, int(rows), cols, th->tol);
      pw->comm = nullptr;
      if (th->residual) res = relative_residual(*pw, corr, Fm, Gm, int(rows), cols);
    }
    if (th->ranks) th->ranks[k - 1] = corr.rank;
    if (th->residual) th->residual[k - 1] = res;
    const int r = corr.rank;
    // Z = Lambda-dagger(X, 0) as one (2 N_c x r) matrix [Zu; Zv]; z_old = Y^T Lambda(old[n]), n >= 2
    if (r > 0) {
      dl = static_cast<double*>(bZ.get((2 * nc * size_t(r) + 2 * nc + size_t(r) * (N + 2)) * sizeof(double)));
      double* Z = dl + 2 * nc;
      zold = Z + 2 * nc * size_t(r);
      zw = zold + size_t(r) * N;
      dz = zw + r;
      PTB_CUDA_CHECK(cudaMemsetAsync(zw, 0, size_t(r) * sizeof(double), st));
      from_energy_components(ew, cgr, size_t(r), corr.Xp(), rows, zw, ccs, Z, Z + nc, 2 * nc);
      if (N >= 2) {
        energy_components(ew, cgr, th->scheme, N - 1, cold.f(0, 1), cold.f(1, 1), nc, nullptr, ccs, cmp, rows, mold + 1);
        gemm(ctx, true, false, r, int(N - 1), int(rows), 1.0, corr.Yp(), int(rows), cmp, int(rows), 0.0, zold, r);
      }
    } else if (N >= 2) {
      energy_components(ew, cgr, th->scheme, N - 1, cold.f(0, 1), cold.f(1, 1), nc, nullptr, ccs, cmp, rows, mold + 1);
    }
    const double* Z = r > 0 ? dl + 2 * nc : nullptr;
    if (hp_it) hp_it->mark("pml theta:  fit, Z, old terms");
    PTB_CUDA_CHECK(cudaMemsetAsync(swf, 0, (N + 1) * sizeof(int32_t), st));
    // n = 1: next[1] = fine_next[1] (both corrected terms cancel, parareal.cpp:315-318): d_1 = 0
    for (int f = 0; f < 4; ++f) {
      PTB_CUDA_CHECK(cudaMemsetAsync(cd.f(f, 0), 0, nc * sizeof(double), st));
      cpy(cwv.f(f), crf.f(f, 0), nc);
    }
    Fields4 G{{cwv.f(0), cwv.f(1), cwv.f(2), cwv.f(3)}};
    for (size_t n = 2; n <= N; ++n) {
      pml_propagate(coarse, coarse->steps, 1, cwv.f(0), cwv.f(1), cwv.f(2), cwv.f(3), swf + n);  // g = C(w)
      energy_components(ew, cgr, th->scheme, 1, cwv.f(0), cwv.f(1), nc, nullptr, ccs, cmp, rows, mw);
      if (r > 0) {
        gemm(ctx, true, false, r, 1, int(rows), 1.0, corr.Yp(), int(rows), cmp, int(rows), 0.0, zw, r);
        k_sub_small<<<1, 256, 0, st>>>(r, zw, zold + (n - 2) * size_t(r), dz);
        PTB_LAUNCH_CHECK(ctx);
        gemm(ctx, false, false, int(2 * nc), 1, r, 1.0, Z, int(2 * nc), dz, r, 0.0, dl, int(2 * nc));
      }
      Fields4 RF{{crf.f(0, n - 1), crf.f(1, n - 1), crf.f(2, n - 1), crf.f(3, n - 1)}};
      Fields4 D{{cd.f(0, n - 1), cd.f(1, n - 1), cd.f(2, n - 1), cd.f(3, n - 1)}};
      k_theta_tail<<<ew_blocks(ctx, nc), 256, 0, st>>>(nc, r > 0 ? dl : nullptr, mw, mold + (n - 1), swf + n,
                                                      gcf + (n - 1), gff + (n - 1), G, RF, D);
      PTB_LAUNCH_CHECK(ctx);
    }
  };
  for (int f = 2; f < 4; ++f) PTB_CUDA_CHECK(cudaMemsetAsync(nxt.f(f, 0), 0, (L + 1) * nf * sizeof(double), st));
  for (int k = 1; k <= K; ++k) {
    HostProf hp_(st);
    hp_it = &hp_;
    PTB_CUDA_CHECK(cudaEventRecord(e0, st));
    // parallel stage on the own couplings: next[n] = F(cur[n-1]), old[n] = C(R cur[n-1])
    if (L) {
      for (int f = 0; f < 4; ++f) restrict_fields(t, L, cur.f(f, 0), cold.f(f, a - 1));
      // next[n] = F(cur[n-1]) straight from cur into nxt (no copy of the state; nxt's px, py are
      // zero off the layer: zeroed before the first iteration, valid iterates afterwards)
      const double* fsrc[4] = {cur.f(0, 0), cur.f(1, 0), cur.f(2, 0), cur.f(3, 0)};
      if (theta) {
        PTB_CUDA_CHECK(cudaMemsetAsync(ffl, 0, 2 * (chunk + 1) * sizeof(int32_t), st));
        pml_propagate(fine, fine->steps, L, nxt.f(0, 1), nxt.f(1, 1), nxt.f(2, 1), nxt.f(3, 1), ffl, fsrc);
        k_or_flags<<<1, 256, 0, st>>>(L, ffl, flags + 1);
        PTB_LAUNCH_CHECK(ctx);
      } else {
        pml_propagate(fine, fine->steps, L, nxt.f(0, 1), nxt.f(1, 1), nxt.f(2, 1), nxt.f(3, 1), flags + 1, fsrc);
      }
      pml_propagate(coarse, coarse->steps, L, cold.f(0, a - 1), cold.f(1, a - 1), cold.f(2, a - 1), cold.f(3, a - 1),
                    theta ? cfl : nullptr);
      for (int f = 0; f < 4; ++f) restrict_fields(t, L, nxt.f(f, 1), crf.f(f, a - 1));
    }
    hp_.mark("pml theta: parallel stage");
    if (world > 1) {  // one all-gather of the coarse payload (theta: and the stage flags)
      for (int f = 0; f < 4; ++f) {
        cpy(own + size_t(f) * chunk * nc, cold.f(f, a - 1), L * nc);
        cpy(own + size_t(4 + f) * chunk * nc, crf.f(f, a - 1), L * nc);
      }
      if (theta && L) {  // two int32 rows of `chunk` after the fields (per_b counts them)
        int32_t* of = reinterpret_cast<int32_t*>(own + per);
        PTB_CUDA_CHECK(cudaMemcpyAsync(of, ffl, L * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        PTB_CUDA_CHECK(cudaMemcpyAsync(of + chunk, cfl, L * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
      }
      comm->allgather(own, all, per_b, st);
      for (int r = 0; r < world; ++r) {
        const size_t ra = 1 + size_t(r) * chunk;
        if (ra > N) continue;
        const size_t rl = std::min(N + 1, ra + chunk) - ra;
        const double* src = reinterpret_cast<const double*>(reinterpret_cast<const char*>(all) + size_t(r) * per_b);
        if (theta) {
          const int32_t* rf_ = reinterpret_cast<const int32_t*>(src + per);
          PTB_CUDA_CHECK(cudaMemcpyAsync(gff + (ra - 1), rf_, rl * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
          PTB_CUDA_CHECK(cudaMemcpyAsync(gcf + (ra - 1), rf_ + chunk, rl * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
        }
        if (r == rank) continue;
        for (int f = 0; f < 4; ++f) {
          cpy(cold.f(f, ra - 1), src + size_t(f) * chunk * nc, rl * nc);
          cpy(crf.f(f, ra - 1), src + size_t(4 + f) * chunk * nc, rl * nc);
        }
      }
    } else if (theta && L) {
      PTB_CUDA_CHECK(cudaMemcpyAsync(gff, ffl, L * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
      PTB_CUDA_CHECK(cudaMemcpyAsync(gcf, cfl, L * sizeof(int32_t), cudaMemcpyDeviceToDevice, st));
    }
    if (theta) {
      theta_iteration(k);
    } else {
    // replicated sequential sweep on the coarse grid: w_0 = R(init); g = C(w_{n-1});
    // d_n = g - old[n]; w_n = R(fine_next[n]) + d_n  (= R(next[n]): R(I(d)) = d at the coarse nodes)
    for (int f = 0; f < 4; ++f) restrict_fields(t, 1, ini.f(f, 0), cwv.f(f));
    for (size_t n = 1; n <= N; ++n) {
      for (int f = 0; f < 4; ++f) cpy(cg.f(f), cwv.f(f), nc);
      pml_propagate(coarse, coarse->steps, 1, cg.f(0), cg.f(1), cg.f(2), cg.f(3), nullptr);
      for (int f = 0; f < 4; ++f) {
        k_sweep_diff<<<ew_blocks(ctx, nc), 256, 0, st>>>(nc, cg.f(f), cold.f(f, n - 1), crf.f(f, n - 1),
                                                         cd.f(f, n - 1), cwv.f(f));
        PTB_LAUNCH_CHECK(ctx);
      }
    }
    }
    hp_.mark("pml theta: fit + sweep");
    // own combine: next[n] = fine_next[n] + I(d_n), in chunks of slices (u, udot: fused into the
    // interpolation; px, py: the correction masked to the layer)
    // (theta leaves px, py uncorrected: their d is zero — or NaN together with d_u, d_udot on a
    // flagged coupling, which the clamp below catches through u — so only u, udot are combined)
    for (int f = 0; f < (theta ? 2 : 4); ++f)
      for (size_t c0 = 0; c0 < L; c0 += ichunk) {
        const size_t m = std::min(ichunk, L - c0);
        if (f < 2) {
          interpolate_fields_add(t, m, cd.f(f, a - 1 + c0), nxt.f(f, 1 + c0), nxt.f(f, 1 + c0), fchunk);
        } else {
          interpolate_fields(t, m, cd.f(f, a - 1 + c0), fchunk);
          k_aux_mask_add<<<ew_blocks(ctx, m * nf), 256, 0, st>>>(m * nf, fny, fnx, fzx, fzy, nxt.f(f, 1 + c0), fchunk);
          PTB_LAUNCH_CHECK(ctx);
        }
      }
    hp_.mark("pml theta: combine");
    // non-finite iterates: flag and clamp to the previous iterate (parareal.cpp:117-124)
    if (L) {
      PTB_CUDA_CHECK(cudaMemsetAsync(bad, 0, (L + 1) * sizeof(int32_t), st));
      const dim3 g(unsigned(std::min<size_t>((nf + 255) / 256, 64)), unsigned(L));
      if (theta)  // px, py are fine_next's, checked by the fine stage (ffl)
        k_state_bad<<<g, 256, 0, st>>>(nf, nxt.f(0, 1), nxt.f(1, 1), nullptr, nullptr, ffl, bad, flags + 1);
      else
        k_state_bad<<<g, 256, 0, st>>>(nf, nxt.f(0, 1), nxt.f(1, 1), nxt.f(2, 1), nxt.f(3, 1), nullptr, bad, flags + 1);
      PTB_LAUNCH_CHECK(ctx);
      for (int f = 0; f < 4; ++f) {
        hptr[f] = nxt.f(f, 1);
        hptr[4 + f] = cur.f(f, 1);
      }
      PTB_CUDA_CHECK(cudaMemcpyAsync(dptr, hptr, sizeof(hptr), cudaMemcpyHostToDevice, st));
      k_clamp_bad<<<g, 256, 0, st>>>(nf, bad, dptr, dptr + 4);
      PTB_LAUNCH_CHECK(ctx);
    }
    // state a-1: the initial state on rank 0, the previous rank's last state elsewhere
    if (a == 1) cpy_state(nxt, 0, ini, 0);
    if (world > 1) {
      const bool has_next = rank + 1 < world && b <= N && L > 0, has_prev = rank > 0 && a <= N;
      for (int f = 0; f < 4; ++f)
        comm->shift_right(nxt.f(f, L), nf * sizeof(double), has_next, nxt.f(f, 0), nf * sizeof(double), has_prev, st);
    }
    hp_.mark("pml theta: flags + clamp");
    PTB_CUDA_CHECK(cudaEventRecord(e1, st));
    // metric (outside the timed body): L2 distance of [u; udot] to the serial fine run
    if (err_out) {
      PTB_CUDA_CHECK(cudaMemsetAsync(sums, 0, 2 * (chunk + 1) * sizeof(double), st));
      k_err_sums<<<unsigned(L + 1), 512, 0, st>>>(nf, nxt.f(0), nxt.f(1), ref.f(0), ref.f(1), sums);
      PTB_LAUNCH_CHECK(ctx);
      if (world > 1) {
        comm->allgather(sums, gsums, 2 * (chunk + 1) * sizeof(double), st);
        PTB_CUDA_CHECK(cudaMemcpyAsync(hs.data(), gsums, hs.size() * sizeof(double), cudaMemcpyDeviceToHost, st));
      } else {
        PTB_CUDA_CHECK(cudaMemcpyAsync(hs.data(), sums, 2 * (L + 1) * sizeof(double), cudaMemcpyDeviceToHost, st));
      }
    }
    PTB_CUDA_CHECK(cudaStreamSynchronize(st));
    if (ms_out) {
      float ms = 0.f;
      PTB_CUDA_CHECK(cudaEventElapsedTime(&ms, e0, e1));
      ms_out[k - 1] = ms;
    }
    if (err_out)
      for (size_t n = 0; n <= N; ++n) {  // state n from the rank owning coupling n (state 0: rank 0)
        const size_t r = n == 0 ? 0 : (n - 1) / chunk, local = n == 0 ? 0 : n - (1 + r * chunk) + 1;
        const double* h = hs.data() + 2 * (r * (chunk + 1) + local);
        err_out[size_t(k - 1) * (N + 1) + n] = init_norm2 > 0 ? std::sqrt(h[0] / init_norm2) : std::sqrt(h[0]);
      }
    std::swap(cur, nxt);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (diverged_out) {
    std::vector<int32_t> hf(L + 1);
    PTB_CUDA_CHECK(cudaMemcpyAsync(hf.data(), flags, (L + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    PTB_CUDA_CHECK(cudaStreamSynchronize(st));
    int32_t any = 0;
    for (auto x : hf) any |= x;
    if (world > 1) {  // any rank
      int32_t* d = reinterpret_cast<int32_t*>(sums);
      std::vector<int32_t> gv(static_cast<size_t>(world));
      PTB_CUDA_CHECK(cudaMemcpyAsync(d, &any, sizeof(int32_t), cudaMemcpyHostToDevice, st));
      comm->allgather(d, gsums, sizeof(int32_t), st);
      PTB_CUDA_CHECK(cudaMemcpyAsync(gv.data(), gsums, gv.size() * sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      PTB_CUDA_CHECK(cudaStreamSynchronize(st));
      for (auto x : gv) any |= x;
    }
    *diverged_out = any;
  }
  if (states_out) {  // the last iterate, [field][state][point]: own states a-1 .. b-1 (all on one GPU)
    for (int f = 0; f < 4; ++f)
      PTB_CUDA_CHECK(cudaMemcpyAsync(states_out + (size_t(f) * (N + 1) + (a - 1)) * nf, cur.f(f, 0),
                                     (L + 1) * nf * sizeof(double), cudaMemcpyDeviceToHost, st));
    PTB_CUDA_CHECK(cudaStreamSynchronize(st));
  }
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
    PTB_CUDA_CHECK(cudaMalloc(&p->speed, n * sizeof(double)));
    PTB_CUDA_CHECK(cudaMemcpy(p->speed, c_host, n * sizeof(double), cudaMemcpyHostToDevice));
    PTB_CUDA_CHECK(cudaMalloc(&p->coef, h.size() * sizeof(double)));
    PTB_CUDA_CHECK(cudaMemcpy(p->coef, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice));
    // tile classes: a tile is a layer tile when a damped row or column lies within HL cells of
    // it (the halo the layer kernel reads); the plain kernel's smaller halo then sees none
    std::vector<int2> plain, layer;
    auto damped = [](const double* z, long n, long lo, long hi) {
      for (long i = lo; i < hi; ++i)
        if (z[((i % n) + n) % n] > 0.0) return true;
      return false;
    };
    for (long ty = 0; ty < long(ny); ty += PTY)
      for (long tx = 0; tx < long(nx); tx += PTX) {
        const bool l = damped(zeta_y_host, long(ny), ty - HL, ty + PTY + HL) ||
                       damped(zeta_x_host, long(nx), tx - HL, tx + PTX + HL);
        (l ? layer : plain).push_back(make_int2(int(ty), int(tx)));
      }
    p->nplain = int(plain.size());
    p->nlayer = int(layer.size());
    if (!plain.empty()) {  // do the plain tiles tile a rectangle?
      int y0 = INT32_MAX, y1 = 0, x0 = INT32_MAX, x1 = 0;
      for (const int2& t : plain) {
        y0 = std::min(y0, t.x);
        y1 = std::max(y1, std::min(t.x + PTY, int(ny)));
        x0 = std::min(x0, t.y);
        x1 = std::max(x1, std::min(t.y + PTX, int(nx)));
      }
      const size_t rows = size_t((y1 - y0 + PTY - 1) / PTY), cols = size_t((x1 - x0 + PTX - 1) / PTX);
      if (rows * cols == plain.size() && nx % 2 == 0 && x0 % 2 == 0 && (x1 - x0) % 2 == 0) {
        p->ry0 = y0;
        p->rny = y1 - y0;
        p->rx0 = x0;
        p->rnx = x1 - x0;
      }
    }
    {  // frame mode: damped cells only in bands [0, lo) and [n - hi, n) of each axis
      auto bands = [](const double* z, long n, long& lo, long& hi) {
        lo = 0;
        while (lo < n && z[lo] > 0.0) ++lo;
        hi = 0;
        while (hi < n - lo && z[n - 1 - hi] > 0.0) ++hi;
        for (long i = lo; i < n - hi; ++i)
          if (z[i] > 0.0) return false;  // damping inside: not a layer
        return true;
      };
      long ylo, yhi, xlo, xhi;
      if (bands(zeta_y_host, long(ny), ylo, yhi) && bands(zeta_x_host, long(nx), xlo, xhi)) {
        const long m = FRAME_MARGIN;
        const long y0 = ylo + m, y1 = long(ny) - yhi - m;
        const long x0 = (xlo + m + 1) & ~1L, x1 = (long(nx) - xhi - m) & ~1L;
        const bool fits = y0 <= FB && long(ny) - y1 <= FB && x0 <= FB && long(nx) - x1 <= FB;
        if (fits && nx % 2 == 0 && y1 - y0 >= 4 * FB && x1 - x0 >= 4 * FB) {
          std::vector<int2> ft;
          for (long tx = 0; tx < long(nx); tx += PTX) {  // top and bottom bands, FB rows
            ft.push_back(make_int2(0, int(tx)));
            ft.push_back(make_int2(int(ny) - FB, int(tx)));
          }
          const int ntb = int(ft.size());
          for (long ty = y0; ty < y1; ty += PTY) {  // left and right bands between them, FB columns
            ft.push_back(make_int2(int(ty), 0));
            ft.push_back(make_int2(int(ty), int(nx) - FB));
          }
          // the super-pass needs the wider margin and the band tiles of both passes
          const long sy0 = ylo + SUPER_MARGIN, sy1 = long(ny) - yhi - SUPER_MARGIN;
          const long sx0 = (xlo + SUPER_MARGIN + 1) & ~1L, sx1 = (long(nx) - xhi - SUPER_MARGIN) & ~1L;
          if (sy0 <= FBB && long(ny) - sy1 <= FBB && sx0 <= FBB && long(nx) - sx1 <= FBB && sy1 - sy0 >= 4 * FBA &&
              sx1 - sx0 >= 4 * FBA && long(nx) >= 2 * XCA + LA && long(ny) >= 2 * FBA + LA) {
            std::vector<int2> stl;
            // one pass: corner tiles at both ends of the top and bottom bands (wc wide, xc long), mid
            // tiles between them (wm wide, len long, clipped at nx - xc), left/right tiles between the
            // bands' corner rows (wm wide, len long, clipped at ny - wc)
            auto pass_tiles = [&](std::vector<ptb::BandLaunch>& pass, int kbase, int wc, int wm, int xc, int len) {
              const int NX = int(nx), NY = int(ny);
              int first = int(stl.size());
              for (int tx = 0; tx < xc; tx += PTX)
                for (int x : {tx, NX - xc + tx}) {
                  stl.push_back(make_int2(0, x));
                  stl.push_back(make_int2(NY - wc, x));
                }
              pass.push_back({kbase + 0, first, int(stl.size()) - first, 0, 0});
              first = int(stl.size());
              for (int tx = xc; tx < NX - xc; tx += len) stl.push_back(make_int2(0, tx));
              pass.push_back({kbase + 1, first, int(stl.size()) - first, 0, NX - xc});
              first = int(stl.size());
              for (int tx = xc; tx < NX - xc; tx += len) stl.push_back(make_int2(NY - wm, tx));
              pass.push_back({kbase + 2, first, int(stl.size()) - first, 0, NX - xc});
              first = int(stl.size());
              for (int ty = wc; ty < NY - wc; ty += len) stl.push_back(make_int2(ty, 0));
              pass.push_back({kbase + 3, first, int(stl.size()) - first, NY - wc, 0});
              first = int(stl.size());
              for (int ty = wc; ty < NY - wc; ty += len) stl.push_back(make_int2(ty, NX - wm));
              pass.push_back({kbase + 4, first, int(stl.size()) - first, NY - wc, 0});
            };
            pass_tiles(p->pass_a, ptb::BK_A_CORNER, FBA, FBM, XCA, LA);
            pass_tiles(p->pass_b, ptb::BK_B_CORNER, FBB, FBB, XCB, LB);
            p->super = 1;
            p->sy0 = int(sy0);
            p->sny = int(sy1 - sy0);
            p->sx0 = int(sx0);
            p->snx = int(sx1 - sx0);
            PTB_CUDA_CHECK(cudaMalloc(&p->stiles, stl.size() * sizeof(int2)));
            PTB_CUDA_CHECK(cudaMemcpy(p->stiles, stl.data(), stl.size() * sizeof(int2), cudaMemcpyHostToDevice));
          }
          p->frame = 1;
          p->fy0 = int(y0);
          p->fny = int(y1 - y0);
          p->fx0 = int(x0);
          p->fnx = int(x1 - x0);
          p->ntb = ntb;
          p->nlr = int(ft.size()) - ntb;
          PTB_CUDA_CHECK(cudaMalloc(&p->ftiles, ft.size() * sizeof(int2)));
          PTB_CUDA_CHECK(cudaMemcpy(p->ftiles, ft.data(), ft.size() * sizeof(int2), cudaMemcpyHostToDevice));
        }
      }
    }
    p->prm.dim = 2;
    p->prm.ny = int(ny);
    p->prm.nx = int(nx);
    p->prm.ihx2 = ihx2;
    p->prm.ihy2 = ihy2;
    p->prm.dt = dt;
    p->prm.hd = p->hd;
    p->prm.hdt2 = 0.5 * dt * dt;
    p->prm.ry = p->ry;
    p->prm.cc = p->cc;
    plain.insert(plain.end(), layer.begin(), layer.end());
    PTB_CUDA_CHECK(cudaMalloc(&p->tiles, plain.size() * sizeof(int2)));
    PTB_CUDA_CHECK(cudaMemcpy(p->tiles, plain.data(), plain.size() * sizeof(int2), cudaMemcpyHostToDevice));
    *out = p;
  });
}

ptb_status ptb_pml_destroy(ptb_pml* p) {
  return guarded([&] {
    if (!p) return;
    DevGuard g(p->ctx->device);
    cudaFree(p->coef);
    cudaFree(p->speed);
    cudaFree(p->tiles);
    cudaFree(p->ftiles);
    cudaFree(p->stiles);
    if (p->bfork) cudaEventDestroy(p->bfork);
    for (int i = 0; i < ptb_pml::NBS; ++i) {
      if (p->bstream[i]) cudaStreamDestroy(p->bstream[i]);
      if (p->bev[i]) cudaEventDestroy(p->bev[i]);
    }
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

ptb_status ptb_pml_parareal_run(ptb_pml* fine, ptb_pml* coarse, ptb_transfer* t, size_t n_couplings, int iterations,
                                const double* u0_host, const double* udot0_host, double* rel_err_host,
                                double* iteration_ms_host, double* states_host, int32_t* diverged_host) {
  return guarded([&] {
    require(fine && coarse && t && u0_host && udot0_host, "pml parareal: null argument");
    require(fine->ctx == coarse->ctx && t->ctx == fine->ctx, "pml parareal: objects of different contexts");
    DevGuard g(fine->ctx->device);
    std::lock_guard<std::recursive_mutex> lock(fine->ctx->mutex);
    pml_parareal(fine, coarse, t, nullptr, n_couplings, iterations, u0_host, udot0_host, rel_err_host,
                 iteration_ms_host, states_host, diverged_host);
  });
}

ptb_status ptb_pml_parareal_run_sharded(ptb_pml* fine, ptb_pml* coarse, ptb_transfer* t, ptb_comm* comm,
                                        size_t n_couplings, int iterations, const double* u0_host,
                                        const double* udot0_host, double* rel_err_host, double* iteration_ms_host,
                                        double* states_host, int32_t* diverged_host) {
  return guarded([&] {
    require(fine && coarse && t && u0_host && udot0_host, "pml parareal: null argument");
    require(fine->ctx == coarse->ctx && t->ctx == fine->ctx, "pml parareal: objects of different contexts");
    DevGuard g(fine->ctx->device);
    std::lock_guard<std::recursive_mutex> lock(fine->ctx->mutex);
    pml_parareal(fine, coarse, t, comm_of(comm), n_couplings, iterations, u0_host, udot0_host, rel_err_host,
                 iteration_ms_host, states_host, diverged_host);
  });
}

ptb_status ptb_pml_theta_run(ptb_pml* fine, ptb_pml* coarse, ptb_transfer* t, ptb_comm* comm, size_t n_couplings,
                             int iterations, double tol, int scheme, const double* u0_host, const double* udot0_host,
                             double* rel_err_host, double* iteration_ms_host, double* states_host, int32_t* ranks_host,
                             double* residual_host, int32_t* diverged_host) {
  return guarded([&] {
    require(fine && coarse && t && u0_host && udot0_host, "pml parareal: null argument");
    require(fine->ctx == coarse->ctx && t->ctx == fine->ctx, "pml parareal: objects of different contexts");
    DevGuard g(fine->ctx->device);
    std::lock_guard<std::recursive_mutex> lock(fine->ctx->mutex);
    PmlTheta th;
    th.tol = tol;
    th.scheme = scheme;
    th.ranks = ranks_host;
    th.residual = residual_host;
    pml_parareal(fine, coarse, t, comm_of(comm), n_couplings, iterations, u0_host, udot0_host, rel_err_host,
                 iteration_ms_host, states_host, diverged_host, &th);
  });
}

}  // extern "C"
