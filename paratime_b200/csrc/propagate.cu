// K1 — batched fp64 velocity-Verlet propagator for u_tt = c^2 Lap u (periodic 5-point).
//
// Reference: /root/reference/proj/src/propagator.cpp
//   laplacian_into        :31-58   (x term first, (f[x+1] - 2 f[x]) + f[x-1], times 1/h^2)
//   verlet_step_inplace   :60-73   a0 = c^2 Lap u; u += dt*udot + dt^2/2 a0;
//                                  a1 = Lap u; udot += dt/2 (a0 + c^2 a1)
//   propagate_coupling    :95-105  m steps, finite check once at the end
//
// Two arithmetic modes share every kernel below:
//   EXACT — the reference's operations in the reference's order with explicitly
//           rounded intrinsics (__dadd_rn/__dmul_rn never contract to FMA), carrying
//           (u, udot, a = c^2 Lap u).  Bitwise equal to the reference.  Reusing a from
//           the previous step instead of recomputing Lap is bitwise neutral: the
//           reference's a0 of step s+1 is Lap(u_s+1)*c^2, the very product used as
//           c^2*a1 in step s.
//   FAST  — the same Verlet step in kick-drift-kick form carrying (u, vh = udot + b),
//           b = (dt/2) c^2 Lap u:  u' = u + dt vh;  b' = Kx*(cc*u' + ry*(uN+uS) + (uW+uE));
//           udot' = vh + b';  vh' = udot' + b'.  Kx = (dt/2) c^2 / hx^2 is precomputed per
//           point.  Keeping the two half kicks as separate adds makes a fused coupling
//           bitwise equal to repeated single steps, as in the reference.
//
// Kernel families:
//   k_small   — one CTA owns a whole slice (N <= 4096: 1D fields, coarse 2D grids);
//               u double-buffered in shared memory, all steps on chip, one barrier/step.
//   k_cluster — a thread-block cluster owns a slice (2D, 4096 < N <= 32768, nx % 128 == 0):
//               rows split over the CTAs, halo rows exchanged through DSMEM (st.async +
//               mbarrier transaction counts), all steps on chip.
//   k_wave2   — FAST-mode wavefront (below) with two columns per thread (even nx).
//   k_wave    — 2D wavefront temporal blocking: a CTA owns a column strip (+ S+1 halo
//               columns each side) of one slice and marches along y; S+1 time levels
//               are in flight, level t one row behind level t-1.  Each thread owns one
//               column: its u window (rows r-1, r) and carried velocity sit in registers,
//               the current row of every level sits in shared memory (x-neighbours).
//               S steps per HBM round trip (read u, udot, coef once; write u, udot once).
//   k_stream  — generic fallback (large 1D): one kernel per half step, HBM streaming.
//
// Layout: slice-major SoA, u[b*N + iy*nx + ix], axis 0 = y (grid.hpp:8-13).

#include <algorithm>
#include <cmath>
#include <cstdlib>

#include <cooperative_groups.h>

#include "ptb_dsmem.h"

#include "ptb_internal.h"

// k_wave2's level-0 ring (A/B builds; see DESIGN.md 3.1 for the measurements):
//   0: per-thread 16-byte cp.async (LDGSTS, L1-allocating .ca)   1: the same with .cg (L2 only)
//   2: bulk copies (cp.async.bulk, TMA engine) of the CTA's rows by one thread, one mbarrier per slot
//   3: bulk copies of each warp's 64-column segment by its lane 0, one mbarrier per slot and warp
//   4, 5: no ring: 16-byte loads straight into registers 2 (4) or 3 (5) rows ahead
#ifndef PTB_WAVE2_RING
#define PTB_WAVE2_RING 0
#endif
// full-row strips of at least this many threads take the bulk-copy ring (variant 2) instead:
// 512^2 x 64 (W = 256) 7.0 -> 7.7e11 updates/s; narrower full-row strips and haloed strips lose
#ifndef PTB_WAVE2_BULK_FROM
#define PTB_WAVE2_BULK_FROM 256
#endif

namespace ptb {

namespace cg = cooperative_groups;

void nonfinite_on(ptb_context* ctx, cudaStream_t st, size_t n, size_t batch, const double* f, int32_t* flags);

namespace {

using namespace std;

// ------------------------------------------------------------------ arithmetic

// propagator.cpp:44-56 in reference order.  1D: only the x term (propagator.cpp:32-40).
template <bool HASY>
__device__ __forceinline__ double lap_exact(double uc, double ul, double ur, double uu, double ud,
                                            const StepParams& p) {
  double x = __dadd_rn(__dsub_rn(ur, __dmul_rn(2.0, uc)), ul);
  x = __dmul_rn(x, p.ihx2);
  if (!HASY) return x;
  double y = __dadd_rn(__dsub_rn(uu, __dmul_rn(2.0, uc)), ud);
  return __dadd_rn(x, __dmul_rn(y, p.ihy2));
}

// FAST half-kick b = Kx*ry*uu + Kx*(cc*uc + ry*ud + (ul+ur)).  One canonical association is
// used by every kernel and every time level, so b depends on its inputs only: a fused
// coupling then equals the same number of single steps bitwise (test_propagator.cpp:135-149),
// and only the last fma waits on uu (the level below in the wavefront kernel).
template <bool HASY>
__device__ __forceinline__ double bfast(double uc, double ul, double ur, double uu, double ud, double kx,
                                        const StepParams& p) {
  const double s1 = ul + ur;
  if (!HASY) return kx * fma(p.cc, uc, s1);
  return fma(kx * p.ry, uu, kx * fma(p.cc, uc, fma(p.ry, ud, s1)));
}

// bfast<true> when ry == 1 (square cells): fma(1, ud, s1) == ud + s1 and kx * 1 == kx exactly,
// so this is the same value with one multiply fewer
template <bool RY1>
__device__ __forceinline__ double bfast2(double uc, double ul, double ur, double uu, double ud, double kx,
                                         const StepParams& p) {
  if (!RY1) return bfast<true>(uc, ul, ur, uu, ud, kx, p);
  return fma(kx, uu, kx * fma(p.cc, uc, ud + (ul + ur)));
}

__device__ __forceinline__ bool finite2(double a, double b) { return isfinite(a) && isfinite(b); }

// 8-byte global -> shared asynchronous copy (LDGSTS), grouped by commit/wait
__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gmem_src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// periodic neighbour offsets of point p in an ny x nx slice
struct Nb {
  int l, r, u, d;
};
__device__ __forceinline__ Nb neighbours(int p, int ny, int nx) {
  const int iy = p / nx, ix = p - iy * nx;
  Nb n;
  n.l = ix == 0 ? p + nx - 1 : p - 1;
  n.r = ix == nx - 1 ? p - nx + 1 : p + 1;
  n.u = iy == ny - 1 ? ix : p + nx;
  n.d = iy == 0 ? p + (ny - 1) * nx : p - nx;
  return n;
}

// ------------------------------------------------------------------ k_small

struct SmallArgs {
  StepParams p;
  int n;  // points per slice
  int steps;
  double* u;
  double* v;
  const double* coef;  // EXACT: c2, FAST: kx
  int32_t* flags;
};

template <int PPT, bool EXACT, bool HASY>
__global__ void __launch_bounds__(1024) k_small(const SmallArgs a) {
  pdl_wait();  // PDL launches (the theta sweep's coarse steps): the state comes from the previous kernel
  pdl_trigger();
  extern __shared__ double buf[];  // [2][n]
  const int n = a.n, T = blockDim.x, tid = threadIdx.x;
  const size_t off = static_cast<size_t>(blockIdx.x) * n;
  double* __restrict__ U = a.u + off;
  double* __restrict__ V = a.v + off;
  const StepParams& p = a.p;
  double u[PPT], v[PPT], k[PPT], acc[PPT];
  Nb nbq[PPT];  // periodic neighbour offsets, computed once (integer div/mod off the step loop)
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int i = tid + q * T;
    u[q] = v[q] = k[q] = acc[q] = 0.0;
    nbq[q] = Nb{0, 0, 0, 0};
    if (i < n) {
      u[q] = U[i];
      v[q] = V[i];
      k[q] = a.coef[i];
      buf[i] = u[q];
      nbq[q] = neighbours(i, p.ny, p.nx);
    }
  }
  __syncthreads();
  // initial acceleration (EXACT: a0 = Lap(u)*c^2) / half kick (FAST: vh = udot + b)
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int i = tid + q * T;
    if (i < n) {
      const Nb nb = nbq[q];
      if (EXACT) {
        acc[q] = __dmul_rn(lap_exact<HASY>(u[q], buf[nb.l], buf[nb.r], buf[nb.u], buf[nb.d], p), k[q]);
      } else {
        const double b = bfast<HASY>(u[q], buf[nb.l], buf[nb.r], buf[nb.u], buf[nb.d], k[q], p);
        v[q] = v[q] + b;
      }
    }
  }
  for (int s = 0; s < a.steps; ++s) {
    double* dst = buf + ((s + 1) & 1) * n;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int i = tid + q * T;
      if (i < n) {
        if (EXACT)
          u[q] = __dadd_rn(u[q], __dadd_rn(__dmul_rn(p.dt, v[q]), __dmul_rn(p.hdt2, acc[q])));
        else
          u[q] = fma(p.dt, v[q], u[q]);
        dst[i] = u[q];
      }
    }
    __syncthreads();
    const bool last = s + 1 == a.steps;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
      const int i = tid + q * T;
      if (i < n) {
        const Nb nb = nbq[q];
        if (EXACT) {
          const double an = __dmul_rn(lap_exact<HASY>(u[q], dst[nb.l], dst[nb.r], dst[nb.u], dst[nb.d], p), k[q]);
          v[q] = __dadd_rn(v[q], __dmul_rn(p.hd, __dadd_rn(acc[q], an)));
          acc[q] = an;
        } else {
          const double b = bfast<HASY>(u[q], dst[nb.l], dst[nb.r], dst[nb.u], dst[nb.d], k[q], p);
          v[q] = v[q] + b;
          if (!last) v[q] = v[q] + b;
        }
      }
    }
  }
  bool ok = true;
#pragma unroll
  for (int q = 0; q < PPT; ++q) {
    const int i = tid + q * T;
    if (i < n) {
      U[i] = u[q];
      V[i] = v[q];
      ok &= finite2(u[q], v[q]);
    }
  }
  if (a.flags) {
    const int bad = __syncthreads_or(!ok);
    if (bad && tid == 0) atomicOr(&a.flags[blockIdx.x], 1);
  }
}

// ------------------------------------------------------------------ k_cluster
//
// On-chip path for 2D slices of 4096 < N <= 32768 points (cfg1 / cfg5 128^2 fine slices):
// one thread-block cluster of CS <= 8 CTAs owns a slice for all its steps.  CTA c holds
// rows [c R, (c+1) R) (R = ny / CS); every thread keeps a 4-point row segment's u, vh and
// coefficient (EXACT: also a) in registers.  u is double-buffered in shared memory with one
// halo row above and below.  Per step: drift, publish the segment to shared memory, and the
// CTA's first / last row go straight into the neighbouring CTAs' halo rows with st.async,
// which completes bytes on the receiver's mbarrier (periodic ring, DSMEM).  A CTA barrier
// covers its own rows; only the boundary-row threads wait on the mbarrier phase.  x
// neighbours inside a warp come by shuffle.  No HBM traffic between the first load and the
// last store.  Arithmetic identical to k_small / k_wave(2).
//
// Buffer reuse: halo rows of buffer P are rewritten two steps later, by a neighbour that
// first had to receive this CTA's next-step rows, which it sends only after finishing the
// reads of this step, so one mbarrier per buffer and no cluster-wide barrier per step.

// smem_addr, cluster_map, st_async2, mbar_*: ptb_dsmem.h

// Thread mapping: the CTA's rows are cut into 128-point chunks (nx % 128 == 0, so a chunk
// lies in one row); warp w owns chunks RW w .. RW w + RW - 1 and in each chunk lane l owns the
// pairs A = chunk + 2l and B = chunk + 64 + 2l, so every 16-byte shared/global access of a
// warp is contiguous (4 wavefronts).  x neighbours come by shuffle; only the chunk's outer
// neighbours (lane 0 left, lane 31 right) are read from shared memory.
constexpr int CL_RW = 2;        // chunks per warp
constexpr int CL_THREADS = 512;  // 4096 points per CTA

template <bool EXACT>
__global__ void __launch_bounds__(CL_THREADS, 1) k_cluster(const SmallArgs a) {
  pdl_wait();
  pdl_trigger();
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ double cbuf[];  // [2][R + 2][nx]
  __shared__ alignas(8) unsigned long long bars[2];
  const int CS = int(cluster.num_blocks()), c = int(cluster.block_rank());
  const int nx = a.p.nx, ny = a.p.ny, R = ny / CS;
  const int plane = (R + 2) * nx;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const size_t slice = blockIdx.x / CS;
  const StepParams& p = a.p;
  int lr[CL_RW], xa[CL_RW], xl[CL_RW], xr[CL_RW];
#pragma unroll
  for (int i = 0; i < CL_RW; ++i) {
    const int g = 128 * (CL_RW * warp + i);  // first point of the chunk in the CTA's block
    lr[i] = g / nx;
    const int xc = g - lr[i] * nx;
    xa[i] = xc + 2 * lane;
    xl[i] = xc == 0 ? nx - 1 : xc - 1;
    xr[i] = xc + 128 == nx ? 0 : xc + 128;
  }
  auto gidx = [&](int i, int half) {  // offset of pair (i, half) within the slice
    return size_t(c * R + lr[i]) * nx + xa[i] + 64 * half;
  };
  double* __restrict__ U = a.u + slice * size_t(a.n);
  double* __restrict__ V = a.v + slice * size_t(a.n);
  // u, v, k, acc per point: index 4 i + {A0, A1, B0, B1}
  double u[4 * CL_RW], v[4 * CL_RW], k[4 * CL_RW], acc[4 * CL_RW];
#pragma unroll
  for (int i = 0; i < CL_RW; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const size_t o = gidx(i, h);
      const double2 uu = *reinterpret_cast<const double2*>(U + o);
      const double2 vv = *reinterpret_cast<const double2*>(V + o);
      const double2 kk = *reinterpret_cast<const double2*>(a.coef + o);
      u[4 * i + 2 * h] = uu.x, u[4 * i + 2 * h + 1] = uu.y;
      v[4 * i + 2 * h] = vv.x, v[4 * i + 2 * h + 1] = vv.y;
      k[4 * i + 2 * h] = kk.x, k[4 * i + 2 * h + 1] = kk.y;
      acc[4 * i + 2 * h] = acc[4 * i + 2 * h + 1] = 0.0;
    }
  // ranks owning the rows above (c+1: larger y) and below (c-1)
  const int up_rank = c + 1 == CS ? 0 : c + 1, dn_rank = c == 0 ? CS - 1 : c - 1;
  const unsigned bar0 = smem_addr(&bars[0]);
  const unsigned halo_bytes = 2u * unsigned(nx) * sizeof(double);
  bool waiter = false;
#pragma unroll
  for (int i = 0; i < CL_RW; ++i) waiter |= lr[i] == 0 || lr[i] == R - 1;
  if (tid == 0) {
    mbar_init(bar0, 1);
    mbar_init(bar0 + 8, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  cluster.sync();  // barriers initialised before any neighbour sends
  // use index q: buffer q & 1, mbarrier phase (q >> 1) & 1
  auto publish = [&](int q) {
    double* buf = cbuf + (q & 1) * plane;
    const unsigned bar = bar0 + 8u * unsigned(q & 1);
#pragma unroll
    for (int i = 0; i < CL_RW; ++i) {
      double* row = buf + (lr[i] + 1) * nx;
      *reinterpret_cast<double2*>(row + xa[i]) = make_double2(u[4 * i], u[4 * i + 1]);
      *reinterpret_cast<double2*>(row + xa[i] + 64) = make_double2(u[4 * i + 2], u[4 * i + 3]);
      if (lr[i] == 0) {  // first own row = top halo (row R+1) of the CTA below
        const unsigned dst = cluster_map(smem_addr(buf + (R + 1) * nx), dn_rank);
        const unsigned rb = cluster_map(bar, dn_rank);
        st_async2(dst + 8u * unsigned(xa[i]), u[4 * i], u[4 * i + 1], rb);
        st_async2(dst + 8u * unsigned(xa[i] + 64), u[4 * i + 2], u[4 * i + 3], rb);
      }
      if (lr[i] == R - 1) {  // last own row = bottom halo (row 0) of the CTA above
        const unsigned dst = cluster_map(smem_addr(buf), up_rank);
        const unsigned rb = cluster_map(bar, up_rank);
        st_async2(dst + 8u * unsigned(xa[i]), u[4 * i], u[4 * i + 1], rb);
        st_async2(dst + 8u * unsigned(xa[i] + 64), u[4 * i + 2], u[4 * i + 3], rb);
      }
    }
    if (tid == 0) mbar_expect(bar, halo_bytes);
    __syncthreads();  // own rows of buf complete
    if (waiter) mbar_wait(bar, unsigned(q >> 1) & 1u);
  };
  // b (FAST) or c^2 Lap u (EXACT) for the points from buffer q & 1
  auto kick = [&](int q, double (&out)[4 * CL_RW]) {
#pragma unroll
    for (int i = 0; i < CL_RW; ++i) {
      const double* row = cbuf + (q & 1) * plane + (lr[i] + 1) * nx;
      const double* w = u + 4 * i;
      const double2 upa = *reinterpret_cast<const double2*>(row + nx + xa[i]);
      const double2 upb = *reinterpret_cast<const double2*>(row + nx + xa[i] + 64);
      const double2 dna = *reinterpret_cast<const double2*>(row - nx + xa[i]);
      const double2 dnb = *reinterpret_cast<const double2*>(row - nx + xa[i] + 64);
      // right of A1: lane+1's A0 (lane 31: lane 0's B0); right of B1: lane+1's B0 (lane 31: next chunk)
      const double ra = __shfl_sync(0xffffffffu, lane == 0 ? w[2] : w[0], (lane + 1) & 31);
      const double rbv = __shfl_down_sync(0xffffffffu, w[2], 1);
      // left of A0: lane-1's A1 (lane 0: previous chunk); left of B0: lane-1's B1 (lane 0: lane 31's A1)
      const double la = __shfl_up_sync(0xffffffffu, w[1], 1);
      const double lbv = __shfl_sync(0xffffffffu, lane == 31 ? w[1] : w[3], (lane + 31) & 31);
      const double left_a = lane == 0 ? row[xl[i]] : la;
      const double right_b = lane == 31 ? row[xr[i]] : rbv;
      const double ul[4] = {left_a, w[0], lbv, w[2]}, ur[4] = {w[1], ra, w[3], right_b};
      const double ups[4] = {upa.x, upa.y, upb.x, upb.y}, dns[4] = {dna.x, dna.y, dnb.x, dnb.y};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (EXACT)
          out[4 * i + j] = __dmul_rn(lap_exact<true>(w[j], ul[j], ur[j], ups[j], dns[j], p), k[4 * i + j]);
        else
          out[4 * i + j] = bfast<true>(w[j], ul[j], ur[j], ups[j], dns[j], k[4 * i + j], p);
      }
    }
  };
  publish(0);
  {
    double b[4 * CL_RW];
    kick(0, b);
#pragma unroll
    for (int j = 0; j < 4 * CL_RW; ++j) {
      if (EXACT)
        acc[j] = b[j];
      else
        v[j] = v[j] + b[j];
    }
  }
  for (int s = 0; s < a.steps; ++s) {
#pragma unroll
    for (int j = 0; j < 4 * CL_RW; ++j) {
      if (EXACT)
        u[j] = __dadd_rn(u[j], __dadd_rn(__dmul_rn(p.dt, v[j]), __dmul_rn(p.hdt2, acc[j])));
      else
        u[j] = fma(p.dt, v[j], u[j]);
    }
    publish(s + 1);
    const bool last = s + 1 == a.steps;
    double b[4 * CL_RW];
    kick(s + 1, b);
#pragma unroll
    for (int j = 0; j < 4 * CL_RW; ++j) {
      if (EXACT) {
        v[j] = __dadd_rn(v[j], __dmul_rn(p.hd, __dadd_rn(acc[j], b[j])));
        acc[j] = b[j];
      } else {
        v[j] = v[j] + b[j];
        if (!last) v[j] = v[j] + b[j];
      }
    }
  }
  bool ok = true;
#pragma unroll
  for (int i = 0; i < CL_RW; ++i)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const size_t o = gidx(i, h);
      *reinterpret_cast<double2*>(U + o) = make_double2(u[4 * i + 2 * h], u[4 * i + 2 * h + 1]);
      *reinterpret_cast<double2*>(V + o) = make_double2(v[4 * i + 2 * h], v[4 * i + 2 * h + 1]);
      ok &= finite2(u[4 * i + 2 * h], v[4 * i + 2 * h]) && finite2(u[4 * i + 2 * h + 1], v[4 * i + 2 * h + 1]);
    }
  if (a.flags) {
    const int bad = __syncthreads_or(!ok);
    if (bad && tid == 0) atomicOr(&a.flags[slice], 1);
  }
  cluster.sync();  // no CTA exits while a neighbour may still address its shared memory
}

// ------------------------------------------------------------------ k_stream

struct StreamArgs {
  StepParams p;
  size_t n, total;  // points per slice, batch*n
  double* u;
  double* v;
  double* acc;      // EXACT: a (N per slice) — FAST: unused
  const double* coef;
  int last;
};

template <bool EXACT, bool HASY>
__global__ void k_stream_init(const StreamArgs a) {
  for (size_t g = blockIdx.x * size_t(blockDim.x) + threadIdx.x; g < a.total; g += size_t(gridDim.x) * blockDim.x) {
    const size_t s = g / a.n, i = g - s * a.n;
    const double* U = a.u + s * a.n;
    const Nb nb = neighbours(int(i), a.p.ny, a.p.nx);
    if (EXACT)
      a.acc[g] = __dmul_rn(lap_exact<HASY>(U[i], U[nb.l], U[nb.r], U[nb.u], U[nb.d], a.p), a.coef[i]);
    else
      a.v[g] = a.v[g] + bfast<HASY>(U[i], U[nb.l], U[nb.r], U[nb.u], U[nb.d], a.coef[i], a.p);
  }
}

template <bool EXACT>
__global__ void k_stream_drift(const StreamArgs a) {
  for (size_t g = blockIdx.x * size_t(blockDim.x) + threadIdx.x; g < a.total; g += size_t(gridDim.x) * blockDim.x) {
    if (EXACT)
      a.u[g] = __dadd_rn(a.u[g], __dadd_rn(__dmul_rn(a.p.dt, a.v[g]), __dmul_rn(a.p.hdt2, a.acc[g])));
    else
      a.u[g] = fma(a.p.dt, a.v[g], a.u[g]);
  }
}

template <bool EXACT, bool HASY>
__global__ void k_stream_kick(const StreamArgs a) {
  for (size_t g = blockIdx.x * size_t(blockDim.x) + threadIdx.x; g < a.total; g += size_t(gridDim.x) * blockDim.x) {
    const size_t s = g / a.n, i = g - s * a.n;
    const double* U = a.u + s * a.n;
    const Nb nb = neighbours(int(i), a.p.ny, a.p.nx);
    if (EXACT) {
      const double an = __dmul_rn(lap_exact<HASY>(U[i], U[nb.l], U[nb.r], U[nb.u], U[nb.d], a.p), a.coef[i]);
      a.v[g] = __dadd_rn(a.v[g], __dmul_rn(a.p.hd, __dadd_rn(a.acc[g], an)));
      a.acc[g] = an;
    } else {
      const double b = bfast<HASY>(U[i], U[nb.l], U[nb.r], U[nb.u], U[nb.d], a.coef[i], a.p);
      const double vt = a.v[g] + b;
      a.v[g] = a.last ? vt : vt + b;
    }
  }
}

// ------------------------------------------------------------------ k_wave

struct WaveArgs {
  StepParams p;
  const double* __restrict__ u_in;
  const double* __restrict__ v_in;
  double* __restrict__ u_out;
  double* __restrict__ v_out;
  const double* __restrict__ coef;  // EXACT: c2, FAST: kx
  size_t stride;                    // points per slice
  int wu;                           // useful (output) columns per strip
  int rb;                           // output rows per row block
  int32_t* flags;                   // nonfinite flags (nullable)
  int full = 0;                     // k_wave2: the strip is the whole periodic row (2W == nx)
  // k_wave2 output rectangle (rows [ry0, ry0 + rny), columns [rx0, rx0 + rnx)); inputs are read
  // with the periodic wrap of the whole ny x nx slice.  Default (rnx = 0): the whole slice.
  int ry0 = 0, rny = 0, rx0 = 0, rnx = 0;
  int lanes = 0;  // host-side planning hint: launched from the two-lane chunk loop
};

// One iteration of the wavefront: level 0 loads row r0 = ystart+i (+ look-ahead row), levels
// 1..S finalise step t at row ystart+i-t.  PAR (iteration parity) is a template parameter so
// shared-memory addresses are base + immediate.  The per-level register "shifts" below are
// SSA renames: the caller unrolls by 6 (lcm of the window period 3 and the carry period 2),
// so they compile to no moves.
template <int S, bool EXACT, int PAR>
__device__ __forceinline__ void wave_iter(double* __restrict__ sbase, int sstride_par, const StepParams& p,
                                          double (&ulo)[S + 1], double (&uce)[S + 1], double (&vin)[S + 1],
                                          double (&kin)[S + 1], double (&ain)[S + 1], double uu0, double v0,
                                          double k0, double& out_u, double& out_v) {
  constexpr int NLP = (S + 1) | 1;  // odd stride per column: conflict-free 8-byte accesses
  // reads of parity PAR, writes of parity PAR^1
  const double* __restrict__ rd = sbase + PAR * sstride_par;
  double* __restrict__ wr = sbase + (PAR ^ 1) * sstride_par;
  // All x-neighbour loads first: they depend only on the previous iteration, so issuing
  // them ahead of this iteration's stores keeps shared-memory latency off the level chain.
  double ul[S + 1], ur[S + 1];
#pragma unroll
  for (int t = 0; t <= S; ++t) {
    ul[t] = rd[t - NLP];
    ur[t] = rd[t + NLP];
  }
  double up, cv, ck, ca;
  {
    const double uc = uce[0], ud = ulo[0];
    if (EXACT) {
      const double a0 = __dmul_rn(lap_exact<true>(uc, ul[0], ur[0], uu0, ud, p), k0);
      up = __dadd_rn(uc, __dadd_rn(__dmul_rn(p.dt, v0), __dmul_rn(p.hdt2, a0)));
      cv = v0;
      ca = a0;
    } else {
      const double vh = v0 + bfast<true>(uc, ul[0], ur[0], uu0, ud, k0, p);
      up = fma(p.dt, vh, uc);
      cv = vh;
      ca = 0.0;
    }
    ck = k0;
    wr[0] = uu0;
    wr[1] = up;
    ulo[0] = uc;
    uce[0] = uu0;
  }
  // FAST: the part of b independent of the level below, b = fma(Kx*ry, uu, q)
  double q[S + 1], kr[S + 1];
  if (!EXACT) {
#pragma unroll
    for (int t = 1; t <= S; ++t) {
      q[t] = kin[t] * fma(p.cc, uce[t], fma(p.ry, ulo[t], ul[t] + ur[t]));
      kr[t] = kin[t] * p.ry;
    }
  }
#pragma unroll
  for (int t = 1; t <= S; ++t) {
    const double vprev = vin[t], kt = kin[t], aprev = ain[t];
    vin[t] = cv;
    kin[t] = ck;
    ain[t] = ca;
    const double uu = up;
    const double uc = uce[t], ud = ulo[t];
    if (EXACT) {
      const double an = __dmul_rn(lap_exact<true>(uc, ul[t], ur[t], uu, ud, p), kt);
      const double vn = __dadd_rn(vprev, __dmul_rn(p.hd, __dadd_rn(aprev, an)));
      if (t < S) {
        up = __dadd_rn(uc, __dadd_rn(__dmul_rn(p.dt, vn), __dmul_rn(p.hdt2, an)));
        cv = vn;
        ca = an;
        ck = kt;
        wr[t + 1] = up;
      } else {
        out_u = uc;
        out_v = vn;
      }
    } else {
      const double b = fma(kr[t], uu, q[t]);
      if (t < S) {
        const double vh = (vprev + b) + b;
        up = fma(p.dt, vh, uc);
        cv = vh;
        ck = kt;
        wr[t + 1] = up;
      } else {
        out_u = uc;
        out_v = vprev + b;
      }
    }
    ulo[t] = uce[t];
    uce[t] = uu;
  }
}

template <int S, bool EXACT>
__global__ void __launch_bounds__(512) k_wave(const WaveArgs a) {
  constexpr int HX = S + 1;  // halo columns each side: level 0 (a_0 stencil) + S levels
  constexpr int NL = S + 1;  // time levels 0..S in flight
  constexpr int NLP = NL | 1;
  constexpr int UNROLL = 6;
  constexpr int RING = 6;  // must divide UNROLL so ring slots are compile-time
  extern __shared__ double sm[];  // [2 parity][W + 2 pad columns][NLP] + [RING][3][W]
  const int W = blockDim.x, j = threadIdx.x;
  const int nx = a.p.nx, ny = a.p.ny;
  const int npts = nx * ny;
  // blockIdx.x = slice (fastest: concurrent CTAs share coef rows in L2), y = strip, z = row block
  const int x0 = blockIdx.y * a.wu;
  int gx = (x0 - HX + j) % nx;
  if (gx < 0) gx += nx;
  const int Y0 = blockIdx.z * a.rb;
  const int nrows = min(a.rb, ny - Y0);
  const int ystart = Y0 - S;  // level S is valid from row ystart + S = Y0
  const int n_iter = ((nrows + 2 * S + UNROLL - 1) / UNROLL) * UNROLL;
  const int oc = j - HX;
  const bool col_out = oc >= 0 && j < W - HX && oc < a.wu && x0 + oc < nx;
  const size_t off = static_cast<size_t>(blockIdx.x) * a.stride;
  const double* __restrict__ U = a.u_in + off;
  const double* __restrict__ V = a.v_in + off;
  double* __restrict__ UO = a.u_out + off;
  double* __restrict__ VO = a.v_out + off;
  const double* __restrict__ K = a.coef;
  const StepParams p = a.p;
  // pad column on each side keeps j-1 / j+1 in bounds for the edge threads (values unused)
  const int sstride_par = (W + 2) * NLP;
  double* sbase = sm + (j + 1) * NLP;
  auto wrap = [&](int y) -> int {  // flat offset of row y (any integer) at column gx
    int r = y % ny;
    if (r < 0) r += ny;
    return r * nx + gx;
  };
  double ulo[NL], uce[NL], vin[NL], kin[NL], ain[NL];
#pragma unroll
  for (int t = 0; t < NL; ++t) ulo[t] = uce[t] = vin[t] = kin[t] = ain[t] = 0.0;
  ulo[0] = U[wrap(ystart - 1)];
  uce[0] = U[wrap(ystart)];
  sbase[0] = uce[0];  // parity 0, level 0
  // running offsets: look-ahead u row (ystart+i+1), v/k row (ystart+i), output row (ystart+i-S)
  int ou = wrap(ystart + 1), ov = wrap(ystart), oo = wrap(ystart - S);
  auto adv = [npts, nx](int& o) {
    o += nx;
    if (o >= npts) o -= npts;
  };
  // level-0 inputs stream through a cp.async ring of RING rows (prefetch distance RING-1):
  // slot s holds {u_0[ystart+i+1], udot_0[ystart+i], coef[ystart+i]} for iteration i = s mod RING
  double* ring = sm + 2 * sstride_par;  // [RING][3][W]
  auto issue = [&](int slot) {
    double* d = ring + (slot * 3) * W + j;
    cp_async8(d, U + ou);
    cp_async8(d + W, V + ov);
    cp_async8(d + 2 * W, K + ov);
    cp_async_commit();
    adv(ou);
    adv(ov);
  };
#pragma unroll
  for (int s0 = 0; s0 < RING - 1; ++s0) issue(s0);
  __syncthreads();
  bool ok = true;
  const int last_out = nrows + 2 * S;  // outputs are iterations [2S, nrows+2S)
  for (int i0 = 0; i0 < n_iter; i0 += UNROLL) {
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) {
      const int i = i0 + k;
      cp_async_wait<RING - 2>();
      const double* src = ring + ((k % RING) * 3) * W + j;
      const double uu0 = src[0], v0 = src[W], k0 = src[2 * W];
      issue((k + RING - 1) % RING);
      double out_u, out_v;
      if (k & 1)
        wave_iter<S, EXACT, 1>(sbase, sstride_par, p, ulo, uce, vin, kin, ain, uu0, v0, k0, out_u, out_v);
      else
        wave_iter<S, EXACT, 0>(sbase, sstride_par, p, ulo, uce, vin, kin, ain, uu0, v0, k0, out_u, out_v);
      if (col_out && i >= 2 * S && i < last_out) {
        UO[oo] = out_u;
        VO[oo] = out_v;
        ok &= finite2(out_u, out_v);
      }
      adv(oo);
      __syncthreads();
    }
  }
  cp_async_wait<0>();
  if (a.flags) {
    const int bad = __syncthreads_or(!ok);
    if (bad && j == 0) atomicOr(&a.flags[blockIdx.x], 1);
  }
}

// ------------------------------------------------------------------ k_wave2 (FAST, 2 columns/thread)
//
// Same wavefront as k_wave, but every thread owns the column PAIR (2j, 2j+1): the x-neighbours
// inside the pair stay in registers and only the pair's edge values go through shared memory
// (separate left-edge / right-edge rows, conflict-free 8-byte accesses), halving crossbar
// traffic per update.  Level-0 inputs stream as 16-byte cp.async pairs, outputs are 16-byte
// stores.  Requires even nx (pairs never straddle the periodic wrap); the strip halo is the
// even HXE = S + 2 columns per side.  Arithmetic identical to k_wave/k_small FAST.

template <bool CG = false>
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  if constexpr (CG)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(gmem_src) : "memory");
}
// 16-byte streaming load (read-only path, no L1 allocation)
__device__ __forceinline__ double2 ldg_stream2(const double* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];\n" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
// bulk-copy issuers per CTA for k_wave2's ring variants 2 (one) and 3 (one per warp)
template <int RINGV, int T>
constexpr int RING_ISSUERS = RINGV == 3 ? T / 32 : 1;

template <int S, int W, int PAR, bool RY1>
__device__ __forceinline__ void wave2_iter(double* __restrict__ eL, double* __restrict__ eR, const int offl,
                                           const int offr,
                                           const StepParams& p, double (&ulo)[S + 1][2], double (&uce)[S + 1][2],
                                           double (&vin)[S + 1][2], double (&kin)[S + 1][2], const double2 uu0,
                                           const double2 v0, const double2 k0, double2& out_u, double2& out_v) {
  // edge rows: eL/eR + parity*pstride + level*lstride + j (+1 padding)
  constexpr int lstride = W + 2, pstride = (S + 1) * lstride;
  const double* __restrict__ rL = eL + PAR * pstride;
  const double* __restrict__ rR = eR + PAR * pstride;
  double* __restrict__ wL = eL + (PAR ^ 1) * pstride;
  double* __restrict__ wR = eR + (PAR ^ 1) * pstride;
  double nl[S + 1], nr[S + 1];  // left neighbour of col 0, right neighbour of col 1, per level
#pragma unroll
  for (int t = 0; t <= S; ++t) {
    nl[t] = rR[t * lstride + offl];
    nr[t] = rL[t * lstride + offr];
  }
  double up0, up1, cv0, cv1, ck0, ck1;
  {
    const double uc0 = uce[0][0], uc1 = uce[0][1];
    wL[0] = uu0.x;
    wR[0] = uu0.y;
    const double vh0 = v0.x + bfast2<RY1>(uc0, nl[0], uc1, uu0.x, ulo[0][0], k0.x, p);
    const double vh1 = v0.y + bfast2<RY1>(uc1, uc0, nr[0], uu0.y, ulo[0][1], k0.y, p);
    up0 = fma(p.dt, vh0, uc0);
    up1 = fma(p.dt, vh1, uc1);
    cv0 = vh0;
    cv1 = vh1;
    ck0 = k0.x;
    ck1 = k0.y;
    wL[lstride] = up0;
    wR[lstride] = up1;
    ulo[0][0] = uc0;
    ulo[0][1] = uc1;
    uce[0][0] = uu0.x;
    uce[0][1] = uu0.y;
  }
  // parts of b independent of the level below: b = fma(K ry, uu, K (cc uc + ry ud + (ul + ur)))
  double q0[S + 1], q1[S + 1];
#pragma unroll
  for (int t = 1; t <= S; ++t) {
    if (RY1) {
      q0[t] = kin[t][0] * fma(p.cc, uce[t][0], ulo[t][0] + (nl[t] + uce[t][1]));
      q1[t] = kin[t][1] * fma(p.cc, uce[t][1], ulo[t][1] + (uce[t][0] + nr[t]));
    } else {
      q0[t] = kin[t][0] * fma(p.cc, uce[t][0], fma(p.ry, ulo[t][0], nl[t] + uce[t][1]));
      q1[t] = kin[t][1] * fma(p.cc, uce[t][1], fma(p.ry, ulo[t][1], uce[t][0] + nr[t]));
    }
  }
#pragma unroll
  for (int t = 1; t <= S; ++t) {
    const double vp0 = vin[t][0], vp1 = vin[t][1], k0t = kin[t][0], k1t = kin[t][1];
    vin[t][0] = cv0;
    vin[t][1] = cv1;
    kin[t][0] = ck0;
    kin[t][1] = ck1;
    const double uu_0 = up0, uu_1 = up1;
    const double uc0 = uce[t][0], uc1 = uce[t][1];
    const double b0 = fma(RY1 ? k0t : k0t * p.ry, uu_0, q0[t]);
    const double b1 = fma(RY1 ? k1t : k1t * p.ry, uu_1, q1[t]);
    if (t < S) {
      const double vh0 = (vp0 + b0) + b0;
      const double vh1 = (vp1 + b1) + b1;
      up0 = fma(p.dt, vh0, uc0);
      up1 = fma(p.dt, vh1, uc1);
      cv0 = vh0;
      cv1 = vh1;
      ck0 = k0t;
      ck1 = k1t;
      wL[(t + 1) * lstride] = up0;
      wR[(t + 1) * lstride] = up1;
    } else {
      out_u = make_double2(uc0, uc1);
      out_v = make_double2(vp0 + b0, vp1 + b1);
    }
    ulo[t][0] = uc0;
    ulo[t][1] = uc1;
    uce[t][0] = uu_0;
    uce[t][1] = uu_1;
  }
}

// VAR: bit 0 = FULL (one strip spans the periodic row), bit 1 = RY1 (hy == hx)
template <int S, int W, int VAR>
__global__ void __launch_bounds__(W, 1) k_wave2(const WaveArgs a) {
  constexpr bool FULL = VAR & 1, RY1 = (VAR & 2) != 0;
  // even halo >= S + 1 (16-byte aligned pairs); none when the strip is the whole periodic row
  constexpr int HXE = FULL ? 0 : (S + 3) & ~1;
  constexpr int NL = S + 1;
  constexpr int UNROLL = 6, RING = 6;
  extern __shared__ double sm[];
  constexpr int T = W;
  const int j = threadIdx.x;
  // x-neighbour offsets into the edge rows: the left neighbour of column 2j is thread j-1's
  // right edge, the right neighbour of column 2j+1 thread j+1's left edge; a full-width strip
  // wraps them inside the CTA (thread 0 <-> thread W-1) instead of through halo columns
  const int offl = FULL && j == 0 ? W - 1 : -1;
  const int offr = FULL && j == W - 1 ? -(W - 1) : 1;
  const int nx = a.p.nx, ny = a.p.ny;
  const int npts = nx * ny;
  const int rnx = a.rnx ? a.rnx : nx, rny = a.rnx ? a.rny : ny;  // output rectangle
  const int x0 = a.rx0 + blockIdx.y * a.wu;  // even
  int gx = (x0 - HXE + 2 * j) % nx;
  if (gx < 0) gx += nx;
  const int Y0 = a.ry0 + blockIdx.z * a.rb;
  const int nrows = min(a.rb, a.ry0 + rny - Y0);
  const int ystart = Y0 - S;
  const int n_iter = ((nrows + 2 * S + UNROLL - 1) / UNROLL) * UNROLL;
  const int oc = 2 * j - HXE;  // output column offset of col 0 within the strip
  const bool col_out = oc >= 0 && 2 * j + 1 < 2 * T - HXE && oc < a.wu && x0 + oc < a.rx0 + rnx;
  const size_t off = static_cast<size_t>(blockIdx.x) * a.stride;
  const double* __restrict__ U = a.u_in + off;
  const double* __restrict__ V = a.v_in + off;
  double* __restrict__ UO = a.u_out + off;
  double* __restrict__ VO = a.v_out + off;
  const double* __restrict__ K = a.coef;
  const StepParams p = a.p;
  // shared: edges [2 parity][NL][T+2] for L and R, then ring [RING][3][T] double2
  constexpr int pstride = NL * (T + 2);
  double* eL = sm + 1 + j;  // +1: pad so j-1 >= 0
  double* eR = sm + 2 * pstride + 1 + j;
  double2* ring = reinterpret_cast<double2*>(sm + 4 * pstride);
  auto wrap = [&](int y) -> int {
    int r = y % ny;
    if (r < 0) r += ny;
    return r * nx + gx;
  };
  double ulo[NL][2], uce[NL][2], vin[NL][2], kin[NL][2];
#pragma unroll
  for (int t = 0; t < NL; ++t)
#pragma unroll
    for (int c = 0; c < 2; ++c) ulo[t][c] = uce[t][c] = vin[t][c] = kin[t][c] = 0.0;
  {
    const double2 lo = *reinterpret_cast<const double2*>(U + wrap(ystart - 1));
    const double2 ce = *reinterpret_cast<const double2*>(U + wrap(ystart));
    ulo[0][0] = lo.x;
    ulo[0][1] = lo.y;
    uce[0][0] = ce.x;
    uce[0][1] = ce.y;
    eL[0] = ce.x;  // parity 0, level 0
    eR[0] = ce.y;
  }
  int ou = wrap(ystart + 1), ov = wrap(ystart), oo = wrap(ystart - S);
  auto adv = [npts, nx](int& o) {
    o += nx;
    if (o >= npts) o -= npts;
  };
  // ring variant of this instantiation (see the top of the file): the bulk-copy ring pays on wide
  // full-row strips only (one aligned copy per row for 8 warps), cp.async everywhere else
  constexpr int RINGV = (FULL && W >= PTB_WAVE2_BULK_FROM && PTB_WAVE2_RING <= 1) ? 2 : PTB_WAVE2_RING;
  constexpr bool R_ASYNC = RINGV <= 1, R_REGS = RINGV >= 4, R_BULK = !R_ASYNC && !R_REGS;
  // R_REGS: level-0 inputs straight into registers, PD rows ahead (no shared-memory ring)
  constexpr int PD = R_REGS ? RINGV - 2 : 1;
  [[maybe_unused]] double2 pu[PD], pv[PD], pk[PD];
  // R_BULK: level-0 rows arrive by bulk copies (the TMA engine, cp.async.bulk) that complete on an
  // mbarrier; every thread waits on the barrier's phase and reads its pair from the slot.
  //   RING 2: one thread moves the CTA's three row segments (2W doubles each, split where the strip
  //           wraps the periodic x boundary), one barrier per slot;
  //   RING 3: lane 0 of each warp moves the warp's 64-column segments, one barrier per slot and warp
  //           (no cross-warp dependency: a warp only waits for its own bytes).
  constexpr int NW = RING_ISSUERS<RINGV, T>;
  constexpr int SEG = 2 * T / NW;  // doubles per issuer and row
  [[maybe_unused]] uint64_t* bars = reinterpret_cast<uint64_t*>(ring + RING * 3 * T);
  [[maybe_unused]] const int wid = RINGV == 3 ? (j >> 5) : 0;
  [[maybe_unused]] const bool issuer = RINGV == 3 ? (j & 31) == 0 : j == 0;
  // first column of the issuer's segment
  [[maybe_unused]] const int gx0 = ((FULL ? 0 : ((x0 - HXE) % nx + nx) % nx) + SEG * wid) % nx;
  [[maybe_unused]] int ru = 0, rv = 0;  // next u row / udot,coef row (issuers)
  if constexpr (R_BULK) {
    if (issuer) {
      ru = ((ystart + 1) % ny + ny) % ny;
      rv = ((ystart) % ny + ny) % ny;
#pragma unroll
      for (int s0 = 0; s0 < RING; ++s0) mbar_init(smem_addr(&bars[s0 * NW + wid]), 1);
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    __syncthreads();
  }
  [[maybe_unused]] auto copy_row = [&](double* dst, const double* row, unsigned bar) {
    int col = gx0, rem = SEG;
    while (rem > 0) {
      const int len = min(rem, nx - col);
      bulk_from_global(smem_addr(dst), row + col, unsigned(len) * 8u, bar);
      dst += len;
      rem -= len;
      col = 0;
    }
  };
  auto issue = [&](int slot, [[maybe_unused]] int iter) {
    if constexpr (R_ASYNC) {
      double2* d = ring + (slot * 3) * T + j;
      cp_async16<RINGV == 1>(d, U + ou);
      cp_async16<RINGV == 1>(d + T, V + ov);
      cp_async16<RINGV == 1>(d + 2 * T, K + ov);
      cp_async_commit();
      adv(ou);
      adv(ov);
    } else if constexpr (R_REGS) {
      pu[slot] = ldg_stream2(U + ou);
      pv[slot] = ldg_stream2(V + ov);
      pk[slot] = ldg_stream2(K + ov);
      adv(ou);
      adv(ov);
    } else {
      if (issuer && iter < n_iter) {
        const unsigned bar = smem_addr(&bars[slot * NW + wid]);
        mbar_expect(bar, unsigned(3 * SEG) * 8u);
        double* d = reinterpret_cast<double*>(ring + (slot * 3) * T) + SEG * wid;
        copy_row(d, U + size_t(ru) * nx, bar);
        copy_row(d + 2 * T, V + size_t(rv) * nx, bar);
        copy_row(d + 4 * T, K + size_t(rv) * nx, bar);
        if (++ru == ny) ru = 0;
        if (++rv == ny) rv = 0;
      }
    }
  };
#pragma unroll
  for (int s0 = 0; s0 < (R_REGS ? PD : RING - 1); ++s0) issue(s0, s0);
  __syncthreads();
  bool ok = true;
  const int last_out = nrows + 2 * S;
  for (int i0 = 0; i0 < n_iter; i0 += UNROLL) {
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) {
      const int i = i0 + k;
      double2 uu0, v0, k0;
      if constexpr (R_REGS) {
        uu0 = pu[k % PD], v0 = pv[k % PD], k0 = pk[k % PD];
        issue(k % PD, i + PD);
      } else {
        if constexpr (R_ASYNC)
          cp_async_wait<RING - 2>();
        else
          mbar_wait(smem_addr(&bars[k * NW + wid]), unsigned(i0 / UNROLL) & 1u);
        const double2* src = ring + ((k % RING) * 3) * T + j;
        uu0 = src[0], v0 = src[T], k0 = src[2 * T];
        issue((k + RING - 1) % RING, i + RING - 1);
      }
      double2 out_u, out_v;
      if (k & 1)
        wave2_iter<S, W, 1, RY1>(eL, eR, offl, offr, p, ulo, uce, vin, kin, uu0, v0, k0, out_u, out_v);
      else
        wave2_iter<S, W, 0, RY1>(eL, eR, offl, offr, p, ulo, uce, vin, kin, uu0, v0, k0, out_u, out_v);
      if (col_out && i >= 2 * S && i < last_out) {
        *reinterpret_cast<double2*>(UO + oo) = out_u;
        *reinterpret_cast<double2*>(VO + oo) = out_v;
        ok &= finite2(out_u.x, out_v.x) && finite2(out_u.y, out_v.y);
      }
      adv(oo);
      __syncthreads();
    }
  }
  if constexpr (R_ASYNC) cp_async_wait<0>();
  if (a.flags) {
    const int bad = __syncthreads_or(!ok);
    if (bad && j == 0) atomicOr(&a.flags[blockIdx.x], 1);
  }
}

// ------------------------------------------------------------------ misc kernels

__global__ void k_laplacian(StepParams p, size_t n, size_t total, const double* f, double* out) {
  for (size_t g = blockIdx.x * size_t(blockDim.x) + threadIdx.x; g < total; g += size_t(gridDim.x) * blockDim.x) {
    const size_t s = g / n, i = g - s * n;
    const double* F = f + s * n;
    const Nb nb = neighbours(int(i), p.ny, p.nx);
    out[g] = p.dim == 1 ? lap_exact<false>(F[i], F[nb.l], F[nb.r], 0, 0, p)
                        : lap_exact<true>(F[i], F[nb.l], F[nb.r], F[nb.u], F[nb.d], p);
  }
}

__global__ void k_nonfinite(size_t n, const double* f, int32_t* flags) {
  const double* F = f + blockIdx.y * n;
  bool ok = true;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    ok &= isfinite(F[i]);
  const int bad = __syncthreads_or(!ok);
  if (bad && threadIdx.x == 0) atomicOr(&flags[blockIdx.y], 1);
}

__global__ void k_copy2(size_t total, const double* a, const double* b, double* ao, double* bo) {
  for (size_t g = blockIdx.x * size_t(blockDim.x) + threadIdx.x; g < total; g += size_t(gridDim.x) * blockDim.x) {
    ao[g] = a[g];
    bo[g] = b[g];
  }
}

unsigned grid_for(ptb_context* ctx, size_t total, int block) {
  const size_t want = (total + block - 1) / block;
  return static_cast<unsigned>(std::max<size_t>(1, std::min<size_t>(want, size_t(ctx->num_sms) * 16)));
}

// ------------------------------------------------------------------ dispatch

template <int PPT, bool EXACT, bool HASY>
void launch_small(ptb_context* ctx, cudaStream_t st, const SmallArgs& a, int threads, size_t batch) {
  const size_t smem = 2 * size_t(a.n) * sizeof(double);
  auto kern = k_small<PPT, EXACT, HASY>;
  PTB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(batch));
  cfg.blockDim = dim3(unsigned(threads));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  PTB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, a));
  PTB_LAUNCH_CHECK(ctx);
}

// cluster size for k_cluster (0 = not applicable): smallest CS with ny % CS == 0 and at most
// 4096 points (1024 threads x 4) per CTA
int cluster_size(const StepParams& p, size_t n, size_t batch) {
  static const int env = [] {
    const char* e = std::getenv("PTB_CLUSTER");
    return e ? std::atoi(e) : 1;
  }();
  if (env == 0 || p.dim != 2 || n <= 4096 || n > 32768 || p.nx % 128 != 0) return 0;
  // measured crossover (128^2, scripts/sweep_w.py): the cluster kernel wins below ~128 slices
  // (0.44e12 vs 0.31e12 at 64); with more slices the full-row wavefront fills the GPU without
  // row splitting and wins (0.48e12 at 128, 0.61e12 at 512, 0.73e12 at 2048)
  if (env == 1 && batch >= 128) return 0;
  // measured (scripts/sweep_w.py): ahead of k_wave2 up to clusters of 8 (128^2: 0.41-0.45e12
  // vs 0.27-0.42e12 upd/s); at 16 CTAs (256^2) the wavefront kernel is as fast or faster
  for (int cs : {2, 4, 8}) {
    if (p.ny % cs) continue;
    const size_t per = size_t(p.ny / cs) * p.nx;
    if (per == size_t(128) * CL_RW * (CL_THREADS / 32)) return cs;  // exactly one full CTA
  }
  return 0;
}

template <bool EXACT>
void launch_cluster(ptb_context* ctx, cudaStream_t st, const SmallArgs& a, int cs, size_t batch) {
  const int R = a.p.ny / cs, threads = CL_THREADS;
  const size_t smem = size_t(2) * (R + 2) * a.p.nx * sizeof(double);
  auto kern = k_cluster<EXACT>;
  PTB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  if (cs > 8) PTB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(batch * cs));
  cfg.blockDim = dim3(threads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = cs;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  PTB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kern, a));
  PTB_LAUNCH_CHECK(ctx);
}

template <bool EXACT, bool HASY>
void small_dispatch(ptb_context* ctx, cudaStream_t st, const SmallArgs& a, size_t batch) {
  const int n = a.n;
  int ppt = 1;
  while (ppt < 4 && n > ppt * 1024) ppt *= 2;
  int threads = (n + ppt - 1) / ppt;
  threads = ((threads + 31) / 32) * 32;
  switch (ppt) {
    case 1: launch_small<1, EXACT, HASY>(ctx, st, a, threads, batch); break;
    case 2: launch_small<2, EXACT, HASY>(ctx, st, a, threads, batch); break;
    default: launch_small<4, EXACT, HASY>(ctx, st, a, threads, batch); break;
  }
}

struct WavePlan {
  int W, wu, strips, rb, nrb;
  int full = 0;  // k_wave2: one strip spanning the periodic row, no halo columns
};

// Choose strip width W (threads) and row-block height rb.  Cost model: per-SM work in
// warp-iterations = ceil(CTAs / SMs) * (W/32) * (rb + 2S) — halo columns and warm-up rows
// are both paid for — with a latency penalty when fewer than 2 CTAs land on each SM.
WavePlan plan_wave(ptb_context* ctx, int ny, int nx, int S, size_t batch) {
  const int HX = S + 1;
  WavePlan best{};
  double best_cost = 1e300;
  for (int W = 64; W <= 512; W += 32) {
    const int wu_max = W - 2 * HX;
    if (wu_max < 16) continue;
    const int strips = (nx + wu_max - 1) / wu_max;
    const int wu = (nx + strips - 1) / strips;
    for (int div = 1;; div *= 2) {
      const int rb = (ny + div - 1) / div;
      if (div > 1 && rb < 2 * S) break;
      const int nrb = (ny + rb - 1) / rb;
      const size_t ctas = size_t(strips) * nrb * batch;
      const double rounds = std::ceil(double(ctas) / ctx->num_sms);
      const double lat = ctas < size_t(2 * ctx->num_sms) ? 1.5 : 1.0;
      const double cost = rounds * (W / 32.0) * (rb + 2.0 * S) * lat;
      if (cost < best_cost) {
        best_cost = cost;
        best = WavePlan{W, wu, strips, rb, nrb};
      }
      if (rb <= 1) break;
    }
  }
  // tuning overrides (measurement only): PTB_WAVE_W=<threads>, PTB_WAVE_DIV=<row blocks>
  if (const char* e = std::getenv("PTB_WAVE_W"); e && std::atoi(e) > 0) {
    const int W = std::atoi(e);
    const int wu_max = W - 2 * HX;
    if (W >= 64 && W <= 512 && wu_max >= 16) {
      best.W = W;
      best.strips = (nx + wu_max - 1) / wu_max;
      best.wu = (nx + best.strips - 1) / best.strips;
    }
  }
  if (const char* e = std::getenv("PTB_WAVE_DIV"); e && std::atoi(e) > 0) {
    const int div = std::atoi(e);
    best.rb = (ny + div - 1) / div;
    best.nrb = (ny + best.rb - 1) / best.rb;
  }
  return best;
}

template <int S, bool EXACT>
void launch_wave(ptb_context* ctx, cudaStream_t st, const WavePlan& pl, WaveArgs a, size_t batch) {
  const size_t smem = (size_t((S + 1) | 1) * 2 * (pl.W + 2) + size_t(6) * 3 * pl.W) * sizeof(double);
  auto kern = k_wave<S, EXACT>;
  PTB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  a.wu = pl.wu;
  a.rb = pl.rb;
  dim3 grid(static_cast<unsigned>(batch), pl.strips, pl.nrb);
  kern<<<grid, pl.W, smem, st>>>(a);
  PTB_LAUNCH_CHECK(ctx);
}

// k_wave2: W threads cover 2W columns; useful width even; occupancy from the runtime.
size_t wave2_smem(int S, int W) {
  // edges [L,R][2 parity][S+1][W+2], ring [6][3][2W], ring mbarriers (bulk variants)
  return (size_t(4) * (S + 1) * (W + 2) + size_t(6) * 3 * 2 * W) * sizeof(double) +
         size_t(6) * (W / 32 + 1) * sizeof(uint64_t);
}

// strip widths (threads) k_wave2 is instantiated for; each thread covers 2 columns
constexpr int kWave2Widths[] = {64, 96, 128, 160, 192, 256};

template <int S, int W>
const void* wave2_fn(int v) {
  switch (v) {
    case 0: return reinterpret_cast<const void*>(k_wave2<S, W, 0>);
    case 1: return reinterpret_cast<const void*>(k_wave2<S, W, 1>);
    case 2: return reinterpret_cast<const void*>(k_wave2<S, W, 2>);
    default: return reinterpret_cast<const void*>(k_wave2<S, W, 3>);
  }
}
// variant bits: FULL | RY1 << 1 (see k_wave2)
template <int S>
const void* wave2_kernel(int W, int v) {
  switch (W) {
    case 64: return wave2_fn<S, 64>(v);
    case 96: return wave2_fn<S, 96>(v);
    case 128: return wave2_fn<S, 128>(v);
    case 160: return wave2_fn<S, 160>(v);
    case 192: return wave2_fn<S, 192>(v);
    case 256: return wave2_fn<S, 256>(v);
  }
  fail(PTB_UNSUPPORTED, "k_wave2 width");
}
inline int wave2_variant(const StepParams& p, int full) {
  static const bool ry1_env = [] {  // PTB_WAVE_RY1=0: general-ry kernels only (diagnostics)
    const char* e = std::getenv("PTB_WAVE_RY1");
    return !e || std::atoi(e) != 0;
  }();
  return (full ? 1 : 0) | (ry1_env && p.ry == 1.0 ? 2 : 0);
}

template <int S>
WavePlan plan_wave2(ptb_context* ctx, int ny, int nx, size_t batch, bool no_full = false, bool lanes = false) {
  const int HXE = (S + 3) & ~1;
  WavePlan best{};
  double best_cost = 1e300;
  size_t best_slots = 0;
  int forceW = 0;
  if (const char* e = std::getenv("PTB_WAVE_W"); e && std::atoi(e) > 0) forceW = std::atoi(e);
  static const int full_env = [] {
    const char* e = std::getenv("PTB_WAVE_FULL");
    return e ? std::atoi(e) : 1;
  }();
  for (int W : kWave2Widths)
   for (int full = 0; full < 2; ++full) {
    if (forceW && W != forceW) continue;
    if (full && (nx != 2 * W || !full_env || no_full)) continue;
    const int wu_max = full ? nx : (2 * W - 2 * HXE) & ~1;
    if (wu_max < 16) continue;
    int occ = 0;
    const size_t smem = wave2_smem(S, W);
    const void* kern = wave2_kernel<S>(W, full);  // occupancy: same registers for both RY variants
    PTB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    PTB_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, W, smem));
    if (occ < 1) continue;
    const int strips = full ? 1 : (nx + wu_max - 1) / wu_max;
    const int wu = full ? nx : (((nx + strips - 1) / strips) + 1) & ~1;
    for (int div = 1;; div *= 2) {
      const int rb = (ny + div - 1) / div;
      if (div > 1 && rb < 2 * S) break;
      const int nrb = (ny + rb - 1) / rb;
      const size_t ctas = size_t(strips) * nrb * batch;
      const size_t slots = size_t(ctx->num_sms) * occ;
      // time of one round on its busiest SM ~ rows x max(warps, 8) / 8: the kernel is
      // latency-bound below 8 warps per SM (ncu: W=160, 5 warps/SM, runs ~1.6x slower per
      // warp-row than 2 x W=128), throughput-bound above.  Full rounds hold `occ` CTAs per SM;
      // a partial last round ceil(rest / SMs) on its busiest SM (idle SMs cost nothing).
      const auto round_time = [&](size_t ctas_per_sm) {
        return (rb + 2.0 * S) * std::max(1.0, double(ctas_per_sm) * (W / 32.0) / 8.0);
      };
      const size_t full_rounds = ctas / slots, rest = ctas - full_rounds * slots;
      double cost = double(full_rounds) * round_time(size_t(occ)) +
                    (rest ? round_time((rest + ctx->num_sms - 1) / ctx->num_sms) : 0.0);
      if (full && full_env == 2) cost *= 1e-6;  // PTB_WAVE_FULL=2 (tests): prefer full-row strips
      if (cost < best_cost) {
        best_cost = cost;
        best = WavePlan{W, wu, strips, rb, nrb, full};
        best_slots = slots;
      }
      if (rb <= 1) break;
    }
  }
  if (best.W == 0) fail(PTB_UNSUPPORTED, "k_wave2: no feasible strip width");
  // Two-lane chunk loop (wave_propagate): the other lane's CTAs fill a pass's partial last round, so
  // the rounds need no balancing by extra row blocks — each costs 2S warm-up rows.  Keep the strip
  // width and take the fewest row blocks that still give the launch ~one full round of CTAs
  // (measured, scripts/sweep_div.py: 1024^2 x 64 0.74 -> 0.80e12, 512^2 x 512 0.86 -> 0.94e12).
  if (lanes) {
    for (int div = 1; div <= best.nrb; ++div) {
      const int rb = (ny + div - 1) / div, nrb = (ny + rb - 1) / rb;
      if (size_t(best.strips) * nrb * batch * 20 >= best_slots * 17 || nrb >= best.nrb) {
        best.rb = rb;
        best.nrb = nrb;
        break;
      }
    }
  }
  if (const char* e = std::getenv("PTB_WAVE_DIV"); e && std::atoi(e) > 0) {
    const int div = std::atoi(e);
    best.rb = (ny + div - 1) / div;
    best.nrb = (ny + best.rb - 1) / best.rb;
  }
  return best;
}

template <int S>
void launch_wave2(ptb_context* ctx, cudaStream_t st, WaveArgs a, size_t batch) {
  // a rectangle narrower than the row is covered by haloed strips (full-row needs rnx == nx)
  const bool rect = a.rnx != 0;
  const WavePlan pl = plan_wave2<S>(ctx, rect ? a.rny : a.p.ny, rect ? a.rnx : a.p.nx, batch,
                                    rect && a.rnx != a.p.nx, a.lanes != 0);
  const size_t smem = wave2_smem(S, pl.W);
  a.wu = pl.wu;
  a.rb = pl.rb;
  a.full = pl.full;
  dim3 grid(static_cast<unsigned>(batch), pl.strips, pl.nrb);
  void* args[] = {&a};
  const void* kern = wave2_kernel<S>(pl.W, wave2_variant(a.p, pl.full));
  PTB_CUDA_CHECK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  PTB_CUDA_CHECK(cudaLaunchKernel(kern, grid, dim3(pl.W), args, smem, st));
  PTB_LAUNCH_CHECK(ctx);
}

bool use_wave2(const StepParams& p) {
  static const int env = [] {
    const char* e = std::getenv("PTB_WAVE2");
    return e ? std::atoi(e) : 1;
  }();
  return env != 0 && p.nx % 2 == 0 && p.nx >= 32;
}

template <bool EXACT>
void wave_pass(ptb_context* ctx, cudaStream_t st, int S, const StepParams& p, size_t batch, const double* ui,
               const double* vi, double* uo, double* vo, const double* coef, int32_t* flags, bool lanes) {
  WaveArgs a{p, ui, vi, uo, vo, coef, size_t(p.ny) * p.nx, 0, 0, flags};
  a.lanes = lanes ? 1 : 0;
  if constexpr (!EXACT) {
    if (use_wave2(p)) {
      switch (S) {
        case 1: launch_wave2<1>(ctx, st, a, batch); return;
        case 2: launch_wave2<2>(ctx, st, a, batch); return;
        case 4: launch_wave2<4>(ctx, st, a, batch); return;
        case 8: launch_wave2<8>(ctx, st, a, batch); return;
        default: fail(PTB_UNSUPPORTED, "wavefront depth");
      }
    }
  }
  const WavePlan pl = plan_wave(ctx, p.ny, p.nx, S, batch);
  switch (S) {
    case 1: launch_wave<1, EXACT>(ctx, st, pl, a, batch); break;
    case 2: launch_wave<2, EXACT>(ctx, st, pl, a, batch); break;
    case 4: launch_wave<4, EXACT>(ctx, st, pl, a, batch); break;
    case 8: launch_wave<8, EXACT>(ctx, st, pl, a, batch); break;
    default: fail(PTB_UNSUPPORTED, "wavefront depth");
  }
}

// two-lane chunk loop of wave_propagate: PTB_LANES=0 turns it off, PTB_LANE_MIN_POINTS sets the
// smallest batch x grid size that takes it (default 2^22 points:
// 256^2 x 64 slices +10 %, 512^2 / 1024^2 x 64 +4 %, 2048^2 x 64..128 +3 %, 4096^2 x 512 +1 %)
bool lanes_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PTB_LANES");
    return !(e && std::atoi(e) == 0);
  }();
  return on;
}
size_t lane_min_points() {
  static const size_t v = [] {
    const char* e = std::getenv("PTB_LANE_MIN_POINTS");
    return e && std::atoll(e) > 0 ? size_t(std::atoll(e)) : size_t(1) << 22;
  }();
  return v;
}

// slices per ping-pong chunk of the context scratch (see wave_propagate)
size_t scratch_chunk(size_t n, size_t batch) {
  static const size_t cap = [] {
    const char* e = std::getenv("PTB_SCRATCH_MIB");
    return (e && std::atoll(e) > 0 ? size_t(std::atoll(e)) : size_t(16384)) << 20;
  }();
  return std::min(batch, std::max<size_t>(1, cap / (2 * n * sizeof(double))));
}

// slices per launch of wave_propagate on the context scratch, and whether the chunks alternate
// between two lanes (each lane owns half of the scratch)
size_t lane_chunk(size_t n, size_t batch, bool& lanes) {
  const size_t chunk0 = scratch_chunk(n, batch);
  lanes = lanes_enabled() && batch >= 4 && batch * n >= lane_min_points();
  return lanes ? std::max<size_t>(1, std::min((batch + 1) / 2, chunk0 / 2)) : chunk0;
}

template <bool EXACT>
void wave_propagate(ptb_propagator* pr, size_t steps, size_t batch, double* u, double* v, int32_t* flags,
                    const LaunchSlot& slot) {
  ptb_context* ctx = pr->ctx;
  const StepParams& p = pr->prm;
  const size_t n = pr->n;
  const double* coef = EXACT ? pr->c2 : pr->kx;
  // decompose steps into passes of 8,4,2,1 levels; ping-pong between (u,v) and scratch
  std::vector<int> passes;
  size_t rem = steps;
  while (rem >= 8) { passes.push_back(8); rem -= 8; }
  for (int s : {4, 2, 1})
    if (rem >= size_t(s)) { passes.push_back(s); rem -= size_t(s); }
  // The context scratch holds at most `chunk` slices (PTB_SCRATCH_MIB, default 16 GiB for the
  // pair): larger batches run the whole coupling chunk by chunk, each chunk ping-ponging between
  // its own slices and the shared scratch, so a batch can use ~all of HBM for its state (cfg5
  // 4096^2 x 512 slices: 137 GB of state + 17 GB of scratch).  A slice's arithmetic does not
  // depend on the plan, so chunking never changes results.
  // Two lanes: with the context scratch and enough work, alternate chunks run on the caller's
  // stream and on the context's lane stream, each lane ping-ponging into its own half of the
  // scratch.  A pass is a few rounds of long-running CTAs (4096^2: ~3 ms each), so a single
  // in-order stream idles SMs through every pass's last partial round; the other lane's CTAs fill
  // them (fork/join by events: the caller's stream still orders the whole call).
  bool lanes = false;
  const size_t chunk = slot.su ? batch : lane_chunk(n, batch, lanes);
  const size_t lane_stride = chunk * n;
  double* su = slot.su ? slot.su : static_cast<double*>(ctx->scratch[0].get((lanes ? 2 : 1) * lane_stride * sizeof(double)));
  double* sv = slot.sv ? slot.sv : static_cast<double*>(ctx->scratch[1].get((lanes ? 2 : 1) * lane_stride * sizeof(double)));
  cudaStream_t st[2] = {slot.stream, slot.stream};
  if (lanes) {
    if (!ctx->lane) {
      PTB_CUDA_CHECK(cudaStreamCreateWithFlags(&ctx->lane, cudaStreamNonBlocking));
      PTB_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->lane_fork, cudaEventDisableTiming));
      PTB_CUDA_CHECK(cudaEventCreateWithFlags(&ctx->lane_join, cudaEventDisableTiming));
    }
    st[1] = ctx->lane;
    PTB_CUDA_CHECK(cudaEventRecord(ctx->lane_fork, slot.stream));
    PTB_CUDA_CHECK(cudaStreamWaitEvent(ctx->lane, ctx->lane_fork, 0));
  }
  size_t ci_ = 0;
  for (size_t b0 = 0; b0 < batch; b0 += chunk, ++ci_) {
    const size_t nb = std::min(chunk, batch - b0);
    const int lane = lanes ? int(ci_ & 1) : 0;
    double* lu = su + lane * lane_stride;
    double* lv = sv + lane * lane_stride;
    double* hu = u + b0 * n;
    double* hv = v + b0 * n;
    const double* ci = slot.src_u ? slot.src_u + b0 * n : hu;
    const double* cvi = slot.src_u ? slot.src_v + b0 * n : hv;
    for (size_t k = 0; k < passes.size(); ++k) {
      const bool to_scratch = (k % 2) == 0;
      double* uo = to_scratch ? lu : hu;
      double* vo = to_scratch ? lv : hv;
      wave_pass<EXACT>(ctx, st[lane], passes[k], p, nb, ci, cvi, uo, vo, coef,
                       k + 1 == passes.size() && flags ? flags + b0 : nullptr, lanes);
      ci = uo;
      cvi = vo;
    }
    if (ci != hu) {
      const size_t total = nb * n;
      k_copy2<<<grid_for(ctx, total, 256), 256, 0, st[lane]>>>(total, lu, lv, hu, hv);
      PTB_LAUNCH_CHECK(ctx);
    }
  }
  if (lanes) {
    PTB_CUDA_CHECK(cudaEventRecord(ctx->lane_join, ctx->lane));
    PTB_CUDA_CHECK(cudaStreamWaitEvent(slot.stream, ctx->lane_join, 0));
  }
}

template <bool EXACT, bool HASY>
void stream_propagate(ptb_propagator* pr, size_t steps, size_t batch, double* u, double* v, int32_t* flags,
                      const LaunchSlot& slot) {
  ptb_context* ctx = pr->ctx;
  const size_t n = pr->n, total = batch * n;
  double* acc = !EXACT ? nullptr
                : slot.su ? slot.su
                          : static_cast<double*>(ctx->scratch[2].get(total * sizeof(double)));
  const cudaStream_t st = slot.stream;
  StreamArgs a{pr->prm, n, total, u, v, acc, EXACT ? pr->c2 : pr->kx, 0};
  const unsigned g = grid_for(ctx, total, 256);
  k_stream_init<EXACT, HASY><<<g, 256, 0, st>>>(a);
  PTB_LAUNCH_CHECK(ctx);
  for (size_t s = 0; s < steps; ++s) {
    a.last = s + 1 == steps;
    k_stream_drift<EXACT><<<g, 256, 0, st>>>(a);
    PTB_LAUNCH_CHECK(ctx);
    k_stream_kick<EXACT, HASY><<<g, 256, 0, st>>>(a);
    PTB_LAUNCH_CHECK(ctx);
  }
  if (flags) {
    nonfinite_on(ctx, st, n, batch, u, flags);
    nonfinite_on(ctx, st, n, batch, v, flags);
  }
}

}  // namespace

// FAST steps on the rectangle [y0, y0 + rny) x [x0, x0 + rnx) of every slice (out of place; points
// outside the rectangle are neither computed nor written).  The caller guarantees that the S-step
// dependency cone of the rectangle lies where the periodic FAST step is the right one (the
// absorbing-layer propagator's undamped interior).  S in {1, 2, 4, 8}, even nx.
void wave_rect_fast(ptb_context* ctx, cudaStream_t st, int S, const StepParams& p, size_t batch, const double* ui,
                    const double* vi, double* uo, double* vo, const double* kx, int32_t* flags, int y0, int rny,
                    int x0, int rnx) {
  require(p.nx % 2 == 0 && x0 % 2 == 0 && rnx % 2 == 0 && rnx > 0 && rny > 0, "wave rect: bad rectangle");
  WaveArgs a{p, ui, vi, uo, vo, kx, size_t(p.ny) * p.nx, 0, 0, flags};
  a.ry0 = y0;
  a.rny = rny;
  a.rx0 = x0;
  a.rnx = rnx;
  switch (S) {
    case 1: launch_wave2<1>(ctx, st, a, batch); return;
    case 2: launch_wave2<2>(ctx, st, a, batch); return;
    case 4: launch_wave2<4>(ctx, st, a, batch); return;
    case 8: launch_wave2<8>(ctx, st, a, batch); return;
    default: fail(PTB_UNSUPPORTED, "wave rect: depth");
  }
}


void propagate(ptb_propagator* pr, size_t steps, size_t batch, double* u, double* v, int32_t* flags, int mode,
               const LaunchSlot* slot_in) {
  if (batch == 0 || steps == 0) return;
  ptb_context* ctx = pr->ctx;
  LaunchSlot slot;
  if (slot_in) slot = *slot_in;
  if (!slot.stream) slot.stream = ctx->stream;
  const bool exact = mode == PTB_MODE_EXACT;
  const StepParams& p = pr->prm;
  const size_t n = pr->n;
  if (slot.src_u && !(n > 4096 && !cluster_size(p, n, batch) && p.dim == 2)) {
    // every family but the wavefront works in place: copy the source state first
    const size_t total = batch * n;
    k_copy2<<<grid_for(ctx, total, 256), 256, 0, slot.stream>>>(total, slot.src_u, slot.src_v, u, v);
    PTB_LAUNCH_CHECK(ctx);
    slot.src_u = slot.src_v = nullptr;
  }
  if (n <= 4096) {
    SmallArgs a{p, int(n), int(steps), u, v, exact ? pr->c2 : pr->kx, flags};
    const cudaStream_t st = slot.stream;
    if (p.dim == 1) {
      exact ? small_dispatch<true, false>(ctx, st, a, batch) : small_dispatch<false, false>(ctx, st, a, batch);
    } else {
      exact ? small_dispatch<true, true>(ctx, st, a, batch) : small_dispatch<false, true>(ctx, st, a, batch);
    }
    return;
  }
  if (const int cs = cluster_size(p, n, batch)) {
    SmallArgs a{p, int(n), int(steps), u, v, exact ? pr->c2 : pr->kx, flags};
    exact ? launch_cluster<true>(ctx, slot.stream, a, cs, batch) : launch_cluster<false>(ctx, slot.stream, a, cs, batch);
    return;
  }
  if (p.dim == 2) {
    exact ? wave_propagate<true>(pr, steps, batch, u, v, flags, slot)
          : wave_propagate<false>(pr, steps, batch, u, v, flags, slot);
    return;
  }
  exact ? stream_propagate<true, false>(pr, steps, batch, u, v, flags, slot)
        : stream_propagate<false, false>(pr, steps, batch, u, v, flags, slot);
}

std::string describe_plan(ptb_propagator* pr, size_t steps, size_t batch, int mode) {
  const bool exact = mode == PTB_MODE_EXACT;
  const StepParams& p = pr->prm;
  const char* m = exact ? "EXACT" : "FAST";
  if (batch == 0 || steps == 0) return "none";
  if (pr->n <= 4096) return std::string("k_small<") + m + "> x1 launch, one CTA per slice";
  if (const int cs = cluster_size(p, pr->n, batch))
    return std::string("k_cluster<") + m + "> x1 launch, cluster of " + std::to_string(cs) + " CTAs x " +
           std::to_string(CL_THREADS) + " threads per slice";
  if (p.dim != 2) return std::string("k_stream_drift/kick<") + m + "> 2 launches per step";
  const size_t full_batch = batch;
  bool lanes = false;
  batch = lane_chunk(pr->n, batch, lanes);
  std::string out;
  size_t rem = steps;
  int passes = 0;
  for (int S : {8, 4, 2, 1}) {
    const size_t k = S == 8 ? rem / 8 : (rem >= size_t(S) ? 1 : 0);
    if (!k) continue;
    rem -= k * S;
    passes += int(k);
    std::string d;
    if (!exact && use_wave2(p)) {
      WavePlan pl;
      switch (S) {
        case 8: pl = plan_wave2<8>(pr->ctx, p.ny, p.nx, batch, false, lanes); break;
        case 4: pl = plan_wave2<4>(pr->ctx, p.ny, p.nx, batch, false, lanes); break;
        case 2: pl = plan_wave2<2>(pr->ctx, p.ny, p.nx, batch, false, lanes); break;
        default: pl = plan_wave2<1>(pr->ctx, p.ny, p.nx, batch, false, lanes); break;
      }
      d = "k_wave2<" + std::to_string(S) + "," + std::to_string(pl.W) + ">" + (pl.full ? " full-row" : "") +
          ((wave2_variant(p, pl.full) & 2) ? " ry1" : "");
      d += " grid " + std::to_string(batch) + "x" + std::to_string(pl.strips) + "x" + std::to_string(pl.nrb);
    } else {
      const WavePlan pl = plan_wave(pr->ctx, p.ny, p.nx, S, batch);
      d = "k_wave<" + std::to_string(S) + "," + m + "> W " + std::to_string(pl.W);
      d += " grid " + std::to_string(batch) + "x" + std::to_string(pl.strips) + "x" + std::to_string(pl.nrb);
    }
    out += (out.empty() ? "" : " + ") + std::to_string(k) + " x " + d;
  }
  if (passes % 2) out += " + k_copy2";
  if (batch < full_batch)
    out = "(" + out + ") per chunk of " + std::to_string(batch) + " slices x " +
          std::to_string((full_batch + batch - 1) / batch) + (lanes ? " on two lanes" : "");
  return out;
}

void laplacian(ptb_context* ctx, const ptb_grid& g, size_t batch, const double* f, double* out) {
  StepParams p{};
  p.dim = g.dim;
  p.ny = g.dim == 1 ? 1 : int(g.n[0]);
  p.nx = g.dim == 1 ? int(g.n[0]) : int(g.n[1]);
  if (g.dim == 1) {
    p.ihx2 = 1.0 / (g.h[0] * g.h[0]);
  } else {
    p.ihy2 = 1.0 / (g.h[0] * g.h[0]);
    p.ihx2 = 1.0 / (g.h[1] * g.h[1]);
  }
  const size_t n = grid_size(g), total = n * batch;
  if (total == 0) return;
  k_laplacian<<<grid_for(ctx, total, 256), 256, 0, ctx->stream>>>(p, n, total, f, out);
  PTB_LAUNCH_CHECK(ctx);
}

void nonfinite_on(ptb_context* ctx, cudaStream_t st, size_t n, size_t batch, const double* f, int32_t* flags) {
  if (batch == 0 || n == 0) return;
  const unsigned gx = static_cast<unsigned>(std::min<size_t>((n + 255) / 256, 64));
  k_nonfinite<<<dim3(gx, static_cast<unsigned>(batch)), 256, 0, st>>>(n, f, flags);
  PTB_LAUNCH_CHECK(ctx);
}

void nonfinite(ptb_context* ctx, size_t n, size_t batch, const double* f, int32_t* flags) {
  nonfinite_on(ctx, ctx->stream, n, batch, f, flags);
}

}  // namespace ptb
