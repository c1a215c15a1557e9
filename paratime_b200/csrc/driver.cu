// Device-resident parareal drivers: serial fine reference, plain parareal, theta
// (data-driven Procrustes) parareal and the corrected-coarse-only ablation, with the
// N time slices block-sharded over one or more GPUs.
//
// Reference: /root/reference/proj/src/parareal.cpp
//   nan_state / fine_stage / coarse_stage   :49-73   divergence -> NaN state
//   measure / finalize_iteration            :80-128  errors vs the serial fine run,
//                                                    flag + clamp non-finite iterates
//   reference_or_nan / serial_coarse_init   :133-159
//   CouplingSchedule                        :172-188
//   plain_parareal                          :201-237
//   corrected_coarse_state / theta_engine   :245-350
//
// Structure.  The reference's sweep is sequential in n and
// works on fine states: next[n] = fine_next[n] + I(corrected(C R next[n-1]) - corrected(
// coarse_next[n])).  Restriction is pointwise, so R(next[n-1]) = R(fine_next[n-1]) +
// R(I(d_{n-1})) exactly (interpolate_at_coarse_nodes evaluates the interpolant at the
// shared nodes with the same arithmetic as the full I).  The sequential part therefore
// runs on coarse vectors only and the fine combine next[n] = fine_next[n] + I(d_n) is one
// batched pass afterwards.  Lambda-dagger is linear with a separate zero mode, so the
// corrected difference is Z (z_w - z_old) + (mean_w - mean_old)/N_c with Z = Lambda-dagger(X)
// computed once per iteration and z = Y^T Lambda(.) — two GEMVs per sweep step instead of
// three 2D FFTs.  The "old" terms do not depend on the sweep and are one GEMM for all n.
//
// Sharding: rank r owns slices [a_r, b_r) and keeps the fine states [a_r-1, b_r).  After
// the parallel stage the coarse payload of every slice is all-gathered (NCCL); the
// Procrustes update and the coarse sweep are then replicated (deterministic, identical on
// every rank), each rank forms its own fine iterates, and the last own state is sent to
// the next rank.  No fine-grid data crosses GPUs except that one boundary state.

#include <math_constants.h>

#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

#include "ptb_comm.h"
#include "ptb_driver.h"
#include "ptb_energy.h"
#include "ptb_procrustes.h"

namespace ptb {
namespace {

constexpr double kNaN = std::numeric_limits<double>::quiet_NaN();
constexpr double kInf = std::numeric_limits<double>::infinity();

unsigned blocks(ptb_context* ctx, size_t n) {
  return unsigned(std::max<size_t>(1, std::min<size_t>((n + 255) / 256, size_t(ctx->num_sms) * 16)));
}

template <typename T>
T* dalloc(DeviceBuffer& b, size_t count) {
  return static_cast<T*>(b.get(std::max<size_t>(1, count) * sizeof(T)));
}

#define GRID_STRIDE(i, n) \
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < (n); i += size_t(gridDim.x) * blockDim.x)

__global__ void k_fill(size_t n, double v, double* a) {
  GRID_STRIDE(i, n) a[i] = v;
}

// states b of `n` values where flags[b] (or any of the optional flag arrays) is set -> NaN
// theta sweep step tail: d_n := NaN where w, coarse_next[n] or fine_next[n] is non-finite
// (parareal.cpp:323-326), then R(next[n]) = R(fine_next[n]) + R(I(d_n)) = R(fine_next[n]) + d_n:
// the interpolant passes through the coarse nodes (Fourier: W[0] = delta exactly; linear: t = 0),
// bitwise for finite d, and a NaN d gives a NaN R(next) as in the reference.
__global__ void k_sweep_tail(size_t n, const int32_t* f0, const int32_t* f1, const int32_t* f2, double* du,
                             double* dv, const double* rfu, const double* rfv, double* ru, double* rv) {
  const bool bad = (*f0) || (*f1) || (*f2);
  GRID_STRIDE(e, n) {
    double a = du[e], b = dv[e];
    if (bad) {
      a = b = CUDART_NAN;
      du[e] = a;
      dv[e] = b;
    }
    if (ru) {
      ru[e] = rfu[e] + a;
      rv[e] = rfv[e] + b;
    }
  }
}

// slice blockIdx.y: a clean slice's CTAs leave at once (the flags are almost always clean)
__global__ void k_nan_where(size_t n, const int32_t* f0, const int32_t* f1, const int32_t* f2, double* u, double* v) {
  const size_t b = blockIdx.y;
  const bool bad = (f0 && f0[b]) || (f1 && f1[b]) || (f2 && f2[b]);
  if (!bad) return;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    u[b * n + i] = CUDART_NAN;
    if (v) v[b * n + i] = CUDART_NAN;
  }
}

__global__ void k_axpby(size_t n, double a, const double* x, double b, const double* y, double* out) {
  GRID_STRIDE(i, n) out[i] = a * x[i] + b * y[i];
}

__global__ void k_add(size_t n, const double* x, const double* y, double* out) {
  GRID_STRIDE(i, n) out[i] = __dadd_rn(x[i], y[i]);
}

__global__ void k_sub(size_t n, const double* x, const double* y, double* out) {
  GRID_STRIDE(i, n) out[i] = __dsub_rn(x[i], y[i]);
}

// (x + y) - z, reference order of plain parareal (parareal.cpp:230)
__global__ void k_add_sub(size_t n, const double* x, const double* y, const double* z, double* out) {
  GRID_STRIDE(i, n) out[i] = __dsub_rn(__dadd_rn(x[i], y[i]), z[i]);
}

// u-part of Lambda-dagger(X z, m): u += (m_new - m_old) / Nc  (zero mode of the inverse DFT)
__device__ __forceinline__ double drv_block_sum256(double x) {  // as energy.cu's block_sum<256>
  __shared__ double red[8];
  __shared__ double tot;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x < 32) {
    double y = threadIdx.x < 8 ? red[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) y += __shfl_xor_sync(0xffffffffu, y, o);
    if (threadIdx.x == 0) tot = y;
  }
  __syncthreads();
  const double r = tot;
  __syncthreads();
  return r;
}

// z = Y^T x for ONE vector (the sweep's z_w = Y^T Lambda(w)): block j reduces column j in a
// fixed order (four accumulators, tree), one launch instead of cuBLAS's gemv + reductions
// grid (r, P): block (j, p) reduces rows [p*chunk, (p+1)*chunk) of column j -> z[j*P + p]; the P
// partials are summed in order by k_assemble_d (fixed layout for a given row count)
__global__ void __launch_bounds__(256) k_gemv_t1(size_t rows, size_t chunk, const double* Y, size_t ld,
                                                 const double* x, double* z) {
  const double* Yj = Y + size_t(blockIdx.x) * ld;
  const size_t r0 = size_t(blockIdx.y) * chunk, r1 = min(rows, r0 + chunk);
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  size_t i = r0 + threadIdx.x;
  for (; i + 768 < r1; i += 1024) {
    a0 += Yj[i] * x[i];
    a1 += Yj[i + 256] * x[i + 256];
    a2 += Yj[i + 512] * x[i + 512];
    a3 += Yj[i + 768] * x[i + 768];
  }
  for (; i < r1; i += 256) a0 += Yj[i] * x[i];
  const double s = drv_block_sum256((a0 + a1) + (a2 + a3));
  if (threadIdx.x == 0) z[size_t(blockIdx.x) * gridDim.y + blockIdx.y] = s;
}

int gemv_parts(size_t rows) { return int(std::max<size_t>(1, std::min<size_t>(64, rows / 2048))); }

// corrected difference on the coarse grid (one launch): dz = z_w - z_old (z_old nullable),
// du = Zu dz + (m_w - m_old)/N_c, dv = Zv dz  (Zu, Zv: N_c x r column-major).
// Block = AD_I consecutive points x AD_J column groups: group g sums columns j = g, g + AD_J, ...
// (all loads of a thread independent, coalesced across the AD_I points), then the AD_J partials
// are added in a fixed tree order -- the result depends on (nc, r) only.
constexpr int AD_I = 32, AD_J = 8;
// mw: mparts partials of m_w, summed in order (k_state_sum_final's order: bitwise the same m_w).
// Optional sweep-step tail (f0 non-null): d := NaN where w, coarse_next[n] or fine_next[n] is
// non-finite (parareal.cpp:323-326), then R(next[n]) = R(fine_next[n]) + d (k_sweep_tail).
struct SweepTail {
  const int32_t *f0, *f1, *f2;
  const double *rfu, *rfv;
  double *ru, *rv;
};
__global__ void __launch_bounds__(AD_I * AD_J) k_assemble_d(size_t nc, int r, const double* Zu, const double* Zv,
                                                          const double* zw, int zparts, const double* zold,
                                                          const double* mw, int mparts, const double* mold,
                                                          double* du, double* dv, const SweepTail tl) {
  pdl_wait();  // z_w and sum(u) come from k_comp_gemv launched just before
  pdl_trigger();
  extern __shared__ double dz[];  // r, then [2][AD_J][AD_I] partials
  const int tid = threadIdx.y * AD_I + threadIdx.x;
  for (int j = tid; j < r; j += AD_I * AD_J) {
    double zj = 0.0;  // z_w[j] = sum of its partials, in order
    for (int q = 0; q < zparts; ++q) zj += zw[size_t(j) * zparts + q];
    dz[j] = zold ? __dsub_rn(zj, zold[j]) : zj;
  }
  __syncthreads();
  double* pu = dz + ((r + 1) & ~1);
  double* pv = pu + AD_J * AD_I;
  const size_t i = size_t(blockIdx.x) * AD_I + threadIdx.x;
  double su0 = 0.0, su1 = 0.0, sv0 = 0.0, sv1 = 0.0;
  if (i < nc) {
    int j = threadIdx.y;
    for (; j + AD_J < r; j += 2 * AD_J) {
      su0 = fma(Zu[size_t(j) * nc + i], dz[j], su0);
      sv0 = fma(Zv[size_t(j) * nc + i], dz[j], sv0);
      su1 = fma(Zu[size_t(j + AD_J) * nc + i], dz[j + AD_J], su1);
      sv1 = fma(Zv[size_t(j + AD_J) * nc + i], dz[j + AD_J], sv1);
    }
    if (j < r) {
      su0 = fma(Zu[size_t(j) * nc + i], dz[j], su0);
      sv0 = fma(Zv[size_t(j) * nc + i], dz[j], sv0);
    }
  }
  pu[threadIdx.y * AD_I + threadIdx.x] = su0 + su1;
  pv[threadIdx.y * AD_I + threadIdx.x] = sv0 + sv1;
  __syncthreads();
  if (threadIdx.y == 0 && i < nc) {
    double a[AD_J], b[AD_J];
#pragma unroll
    for (int g = 0; g < AD_J; ++g) {
      a[g] = pu[g * AD_I + threadIdx.x];
      b[g] = pv[g * AD_I + threadIdx.x];
    }
#pragma unroll
    for (int w = AD_J / 2; w > 0; w >>= 1)
#pragma unroll
      for (int g = 0; g < w; ++g) {
        a[g] += a[g + w];
        b[g] += b[g + w];
      }
    double m = 0.0;
    for (int q = 0; q < mparts; ++q) m += mw[q];
    const double dm = mold ? __dsub_rn(m, *mold) : m;
    double ou = a[0] + dm / double(nc), ov = b[0];
    if (tl.f0) {
      if (*tl.f0 || *tl.f1 || *tl.f2) ou = ov = CUDART_NAN;
      if (tl.ru) {
        tl.ru[i] = tl.rfu[i] + ou;
        tl.rv[i] = tl.rfv[i] + ov;
      }
    }
    du[i] = ou;
    dv[i] = ov;
  }
}

// Row-sharded sweep products of a large corrector (3 N_c x r, cfg4): the rows of Y are cut into
// SWEEP_BLOCKS fixed blocks; block b belongs to rank b % world.  part[b][j] = Y[rows_b, j] . x[rows_b]
// (fixed-order tree per block), then z[j] = sum_b part[b][j] in block order on every rank: the
// value does not depend on the world size.
constexpr int SWEEP_BLOCKS = 8;
__global__ void __launch_bounds__(256) k_zt_blocks(size_t rows, size_t bl, const double* __restrict__ Y, size_t ld,
                                                   const double* __restrict__ x, int r, int rank, int world,
                                                   double* __restrict__ part) {
  pdl_wait();  // x (Lambda(w)) comes from the launch just before
  pdl_trigger();
  const int j = blockIdx.x, b = blockIdx.y;
  if (b % world != rank) return;
  const size_t r0 = size_t(b) * bl, r1 = min(rows, r0 + bl);
  const double* col = Y + size_t(j) * ld;
  double s = 0.0;
  for (size_t i = r0 + threadIdx.x; i < r1; i += 256) s = fma(col[i], x[i], s);
  __shared__ double red[8];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += red[w];
    part[size_t(b) * r + j] = t;
  }
}
// z[j] = sum_b part_of_owner(b)[b][j]; `all` holds world copies of the [SWEEP_BLOCKS][r] array
__global__ void k_zt_sum(int r, int world, const double* __restrict__ all, double* z) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < r; j += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int b = 0; b < SWEEP_BLOCKS; ++b) s += all[(size_t(b % world) * SWEEP_BLOCKS + b) * r + j];
    z[j] = s;
  }
}
// d rows [i0, i1) of both blocks: seg = [du rows | dv rows] of this rank, sg rows each
__global__ void k_zd_rows(int i0, int i1, int sg, int r, const double* __restrict__ Zu, const double* __restrict__ Zv,
                          size_t ld, const double* __restrict__ dz, double* seg) {
  extern __shared__ double dzs[];
  for (int k = threadIdx.x; k < r; k += blockDim.x) dzs[k] = dz[k];
  __syncthreads();
  const int i = i0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= i1) return;
  double su = 0.0, sv = 0.0;  // sequential in k (fixed order), loads issued 8 columns ahead
  int k = 0;
  for (; k + 8 <= r; k += 8) {
    double tu[8], tv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      tu[q] = Zu[i + size_t(k + q) * ld];
      tv[q] = Zv[i + size_t(k + q) * ld];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      su = fma(tu[q], dzs[k + q], su);
      sv = fma(tv[q], dzs[k + q], sv);
    }
  }
  for (; k < r; ++k) {
    su = fma(Zu[i + size_t(k) * ld], dzs[k], su);
    sv = fma(Zv[i + size_t(k) * ld], dzs[k], sv);
  }
  seg[i - i0] = su;
  seg[sg + i - i0] = sv;
}
// One GPU, large corrector: the whole sweep-step tail in one launch — z_w = sum of the
// SWEEP_BLOCKS partials in block order (k_zt_sum), dz = z_w - z_old (k_sub), d = Z dz row by row
// (k_zd_rows' sequential order), the zero mode (m_w - m_old)/N_c (k_add_mean), the NaN rule and
// R(next[n]) = R(fine_next[n]) + d (k_sweep_tail): the same operations in the same order as the
// multi-rank path, so results stay bitwise independent of the world size.
__global__ void k_zd_fused(int n, int r, const double* __restrict__ Zu, const double* __restrict__ Zv, size_t ld,
                           const double* __restrict__ part, const double* __restrict__ zold, const double* mw,
                           const double* mold, double* du, double* dv, const SweepTail tl) {
  pdl_wait();  // the partials come from k_zt_blocks launched just before
  pdl_trigger();
  extern __shared__ double dzs[];
  for (int j = threadIdx.x; j < r; j += blockDim.x) {
    double z = 0.0;
    for (int b = 0; b < SWEEP_BLOCKS; ++b) z += part[size_t(b) * r + j];
    dzs[j] = zold ? __dsub_rn(z, zold[j]) : z;
  }
  __syncthreads();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double su = 0.0, sv = 0.0;
  int k = 0;
  for (; k + 8 <= r; k += 8) {
    double tu[8], tv[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      tu[q] = Zu[i + size_t(k + q) * ld];
      tv[q] = Zv[i + size_t(k + q) * ld];
    }
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      su = fma(tu[q], dzs[k + q], su);
      sv = fma(tv[q], dzs[k + q], sv);
    }
  }
  for (; k < r; ++k) {
    su = fma(Zu[i + size_t(k) * ld], dzs[k], su);
    sv = fma(Zv[i + size_t(k) * ld], dzs[k], sv);
  }
  const double dm = mold ? __dsub_rn(*mw, *mold) : *mw;
  su += dm / double(n);
  if (tl.f0 && (*tl.f0 || *tl.f1 || *tl.f2)) su = sv = CUDART_NAN;
  du[i] = su;
  dv[i] = sv;
  if (tl.ru) {
    tl.ru[i] = tl.rfu[i] + su;
    tl.rv[i] = tl.rfv[i] + sv;
  }
}

// gathered segments (world x [du sg | dv sg]) -> du, dv (n rows)
__global__ void k_zd_unpack(size_t n, int sg, const double* __restrict__ all, double* du, double* dv) {
  GRID_STRIDE(i, n) {
    const size_t rr = i / size_t(sg), o = i - rr * size_t(sg);
    du[i] = all[rr * 2 * size_t(sg) + o];
    dv[i] = all[rr * 2 * size_t(sg) + sg + o];
  }
}

__global__ void k_add_mean(size_t n, const double* mnew, const double* mold, double* u) {
  const double dm = mold ? __dsub_rn(*mnew, *mold) : *mnew;
  const double v = dm / double(n);
  GRID_STRIDE(i, n) u[i] += v;
}

__global__ void k_state_flags(size_t n, const double* u, const double* v, size_t stride, int32_t* flags) {
  const size_t b = blockIdx.y;
  bool ok = true;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    ok &= isfinite(u[b * stride + i]) && isfinite(v[b * stride + i]);
  const int bad = __syncthreads_or(!ok);
  if (bad && threadIdx.x == 0) atomicOr(&flags[b], 1);
}

__global__ void k_or_flags(int32_t* out, const int32_t* a, const int32_t* b, const int32_t* c) {
  *out = (*a ? 1 : 0) | (b && *b ? 1 : 0) | (c && *c ? 1 : 0);
}

}  // namespace

// Work buffers reused by successive runs on one context (ptb_context::driver_cache).
constexpr int kDriverBuffers = 64;
struct DriverCache {
  EnergyWork ew;
  ProcWork pw;
  DeviceBuffer bufs[kDriverBuffers];
  DeviceBuffer corr_x, corr_y;
  explicit DriverCache(ptb_context* c) : ew(c), pw(c) {}
};

DriverCache& driver_cache(ptb_context* ctx) {
  if (!ctx->driver_cache) ctx->driver_cache = std::make_shared<DriverCache>(ctx);
  return *static_cast<DriverCache*>(ctx->driver_cache.get());
}

ProcWork& context_proc_work(ptb_context* ctx) { return driver_cache(ctx).pw; }
EnergyWork& context_energy_work(ptb_context* ctx) { return driver_cache(ctx).ew; }

struct Driver {
  ptb_context* ctx;
  const ptb_run_spec& s;
  Comm single;
  const Comm* comm;
  ptb_grid fg{}, cg{};
  size_t nf = 0, nc = 0, N = 0, chunk = 0, a = 1, b = 1, L = 0;  // own slices [a, b), L = b - a
  int K = 0;
  ptb_propagator* pf = nullptr;
  ptb_propagator* pc = nullptr;
  ptb_transfer* tr = nullptr;
  DriverCache& cache;
  EnergyWork& ew;
  ProcWork& pw;
  DevCorrector corr;
  ptb_phase_times* times = nullptr;
  // fine, own: states [a-1, b) -> index 0..L
  DeviceBuffer cur_u, cur_v, nxt_u, nxt_v, ref_u, ref_v, fn_u, fn_v, fine_u, fine_v, fine2_u, fine2_v;
  // coarse, one slot per slice n = 1..N at index (n-1) (padded to world*chunk)
  DeviceBuffer rf_u, rf_v, kn_u, kn_v, d_u, d_v, w_u, w_v, rik_u, rik_v, own_pay, all_pay;
  DeviceBuffer ff, cf, wf, bad, sflags, sums_own, sums_all, own_sc, all_sc;
  DeviceBuffer rn_u, rn_v, ri_u, ri_v, init_u, init_v, init_cu, init_cv;
  DeviceBuffer comp, mean, comp_old, mean_old, zold, zw, Zu, Zv, Fm, Gm, idx, tmpc;
  DeviceBuffer zpart, zpart_all, dseg, dseg_all;  // row-sharded large-corrector sweep
  std::vector<int32_t> ref_bad;
  int zw_parts = 1;  // partials per z_w entry written by corrected_batch (batch 1)

  // per-step sweep products as single fused launches (k_gemv_t1 + k_assemble_d) for small and mid
  // correctors (latency-bound: cfg1-3); cuBLAS GEMVs for large ones (HBM-bound: cfg4)
  bool fused_sweep(const DevCorrector& c) const {
    // PTB_FUSED_SWEEP_MAX: corrector entries (tests force the large-corrector branch with it)
    const char* e = std::getenv("PTB_FUSED_SWEEP_MAX");
    const long long limit = e ? std::atoll(e) : (4LL << 20);
    return (long long)(size_t(cg.dim + 1) * nc * size_t(std::max(c.rank, 1))) <= limit;
  }
  const double* cf_dev = nullptr;  // coarse speed

  std::vector<DeviceBuffer*> owned() {
    return {&cur_u, &cur_v, &nxt_u, &nxt_v, &ref_u, &ref_v, &fn_u, &fn_v, &fine_u, &fine_v, &fine2_u, &fine2_v,
            &rf_u, &rf_v, &kn_u, &kn_v, &d_u, &d_v, &w_u, &w_v, &rik_u, &rik_v, &own_pay, &all_pay,
            &ff, &cf, &wf, &bad, &sflags, &sums_own, &sums_all, &own_sc, &all_sc,
            &rn_u, &rn_v, &ri_u, &ri_v, &init_u, &init_v, &init_cu, &init_cv,
            &comp, &mean, &comp_old, &mean_old, &zold, &zw, &Zu, &Zv, &Fm, &Gm, &idx, &tmpc,
            &zpart, &zpart_all, &dseg, &dseg_all};
  }

  Driver(ptb_context* c, const Comm* cm, const ptb_run_spec& spec)
      : ctx(c), s(spec), comm(cm), cache(driver_cache(c)), ew(cache.ew), pw(cache.pw) {
    if (!comm) comm = &single;
    const std::vector<DeviceBuffer*> b = owned();
    if (b.size() > size_t(kDriverBuffers)) fail(PTB_UNSUPPORTED, "driver cache too small");
    for (size_t i = 0; i < b.size(); ++i) *b[i] = std::move(cache.bufs[i]);
    corr.X = std::move(cache.corr_x);
    corr.Y = std::move(cache.corr_y);
  }
  ~Driver() {
    const std::vector<DeviceBuffer*> b = owned();
    for (size_t i = 0; i < b.size(); ++i) cache.bufs[i] = std::move(*b[i]);
    cache.corr_x = std::move(corr.X);
    cache.corr_y = std::move(corr.Y);
    ptb_propagator_destroy(pf);
    ptb_propagator_destroy(pc);
    ptb_transfer_destroy(tr);
  }

  cudaStream_t st() const { return ctx->stream; }
  void copy(double* dst, const double* src, size_t n) {
    if (n) PTB_CUDA_CHECK(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, st()));
  }
  void nan_fill(double* p, size_t n) {
    if (!n) return;
    k_fill<<<blocks(ctx, n), 256, 0, st()>>>(n, kNaN, p);
    PTB_LAUNCH_CHECK(ctx);
  }
  void nan_where(size_t n, size_t batch, const int32_t* f0, const int32_t* f1, const int32_t* f2, double* u,
                 double* v) {
    if (!n || !batch) return;
    for (size_t b0 = 0; b0 < batch; b0 += 65535) {  // grid.y limit
      const size_t nb = std::min<size_t>(65535, batch - b0);
      const unsigned gx = unsigned(std::min<size_t>((n + 255) / 256, 64));
      k_nan_where<<<dim3(gx, unsigned(nb)), 256, 0, st()>>>(n, f0 ? f0 + b0 : nullptr, f1 ? f1 + b0 : nullptr,
                                                         f2 ? f2 + b0 : nullptr, u + b0 * n, v ? v + b0 * n : nullptr);
    }
    PTB_LAUNCH_CHECK(ctx);
  }
  template <typename T>
  std::vector<T> to_host(const T* d, size_t n) {
    std::vector<T> h(n);
    if (n) PTB_CUDA_CHECK(cudaMemcpyAsync(h.data(), d, n * sizeof(T), cudaMemcpyDeviceToHost, st()));
    PTB_CUDA_CHECK(cudaStreamSynchronize(st()));
    return h;
  }

  // own-index accessors (fine): state m in [a-1, b) at index m - (a-1)
  double* CU(size_t m) { return static_cast<double*>(cur_u.ptr) + (m - (a - 1)) * nf; }
  double* CV(size_t m) { return static_cast<double*>(cur_v.ptr) + (m - (a - 1)) * nf; }
  double* NU(size_t m) { return static_cast<double*>(nxt_u.ptr) + (m - (a - 1)) * nf; }
  double* NV(size_t m) { return static_cast<double*>(nxt_v.ptr) + (m - (a - 1)) * nf; }
  double* RU(size_t m) { return static_cast<double*>(ref_u.ptr) + (m - (a - 1)) * nf; }
  double* RV(size_t m) { return static_cast<double*>(ref_v.ptr) + (m - (a - 1)) * nf; }
  double* FU(size_t n) { return static_cast<double*>(fn_u.ptr) + (n - a) * nf; }  // own slices
  double* FV(size_t n) { return static_cast<double*>(fn_v.ptr) + (n - a) * nf; }
  // coarse per-slice slots (n = 1..N)
  static double* slot(DeviceBuffer& bf, size_t n, size_t nc_) { return static_cast<double*>(bf.ptr) + (n - 1) * nc_; }
  int32_t* fl(DeviceBuffer& bf) { return static_cast<int32_t*>(bf.ptr); }

  void setup(const double* cfh, const double* cch) {
    fg.dim = cg.dim = s.dim;
    for (int k = 0; k < 2; ++k) {
      fg.n[k] = s.fine_n[k];
      fg.h[k] = s.fine_h[k];
      cg.n[k] = s.coarse_n[k];
      cg.h[k] = s.coarse_h[k];
    }
    validate_grid(fg);
    validate_grid(cg);
    nf = grid_size(fg);
    nc = grid_size(cg);
    N = s.n_couplings;
    K = s.iterations;
    ptb_status e1 = ptb_propagator_create(ctx, &fg, cfh, s.dt_fine, s.m_fine, &pf);
    if (e1 != PTB_OK) fail(e1, g_last_error);
    ptb_status e2 = ptb_propagator_create(ctx, &cg, cch, s.dt_coarse, s.m_coarse, &pc);
    if (e2 != PTB_OK) fail(e2, g_last_error);
    require(s.T > 0.0 && s.dt_com > 0.0 && N > 0, "CouplingSchedule: T, dt_com, N must be positive");
    require(std::abs(double(N) * s.dt_com - s.T) <= 1e-9 * s.T, "CouplingSchedule: N * dt_com must equal T");
    require(std::abs(double(s.m_fine) * s.dt_fine - s.dt_com) <= 1e-12 * s.dt_com,
            "CouplingSchedule: fine steps_per_coupling * dt != dt_com");
    require(std::abs(double(s.m_coarse) * s.dt_coarse - s.dt_com) <= 1e-12 * s.dt_com,
            "CouplingSchedule: coarse steps_per_coupling * dt != dt_com");
    ptb_status e3 = ptb_transfer_create(ctx, &cg, &fg, s.interp, &tr);
    if (e3 != PTB_OK) fail(e3, g_last_error);
    require(K >= 0, "parareal: negative iteration count");
    require(s.variant >= 0 && s.variant <= 3, "parareal: unknown variant");
    require(s.mode == PTB_MODE_FAST || s.mode == PTB_MODE_EXACT, "parareal: unknown propagator mode");
    cf_dev = ptb_propagator_speed(pc);
    // static block partition of slices 1..N (parareal.cpp:25-47 chunking)
    const size_t W = size_t(comm->world);
    chunk = (N + W - 1) / W;
    a = std::min(N + 1, 1 + size_t(comm->rank) * chunk);
    b = std::min(N + 1, a + chunk);
    L = b - a;
    const size_t S = (L + 1) * nf;
    for (DeviceBuffer* bf : {&cur_u, &cur_v, &nxt_u, &nxt_v, &ref_u, &ref_v}) dalloc<double>(*bf, S);
    for (DeviceBuffer* bf : {&fn_u, &fn_v, &fine_u, &fine_v, &fine2_u, &fine2_v}) dalloc<double>(*bf, L * nf);
    const size_t P = W * chunk;  // padded slice slots
    for (DeviceBuffer* bf : {&rf_u, &rf_v, &kn_u, &kn_v, &d_u, &d_v, &w_u, &w_v, &rik_u, &rik_v})
      dalloc<double>(*bf, P * nc);
    for (DeviceBuffer* bf : {&ff, &cf, &wf, &bad, &sflags}) dalloc<int32_t>(*bf, P + 1);
    for (DeviceBuffer* bf : {&rn_u, &rn_v, &ri_u, &ri_v, &init_cu, &init_cv}) dalloc<double>(*bf, nc);
    dalloc<double>(init_u, nf);
    dalloc<double>(init_v, nf);
  }

  // ---- collectives -------------------------------------------------------------------
  // Gather the coarse payload of the own slices: R(fine_next), coarse_next, flags.
  void gather_payload() {
    const size_t per = chunk * (4 * nc) * sizeof(double) + 2 * chunk * sizeof(int32_t);
    char* own = static_cast<char*>(own_pay.get(per));
    char* all = static_cast<char*>(all_pay.get(per * size_t(comm->world)));
    const size_t bc = chunk * nc * sizeof(double);
    if (comm->world == 1) return;  // single GPU: the own slots are the global slots
    // pack own slots (slice a..b-1 live at global slots a-1..)
    auto pack = [&](DeviceBuffer& src, size_t k) {
      if (L) PTB_CUDA_CHECK(cudaMemcpyAsync(own + k * bc, slot(src, a, nc), L * nc * sizeof(double),
                                            cudaMemcpyDeviceToDevice, st()));
    };
    pack(rf_u, 0);
    pack(rf_v, 1);
    pack(kn_u, 2);
    pack(kn_v, 3);
    int32_t* of = reinterpret_cast<int32_t*>(own + 4 * bc);
    if (L) {
      PTB_CUDA_CHECK(cudaMemcpyAsync(of, fl(ff) + (a - 1), L * sizeof(int32_t), cudaMemcpyDeviceToDevice, st()));
      PTB_CUDA_CHECK(cudaMemcpyAsync(of + chunk, fl(cf) + (a - 1), L * sizeof(int32_t), cudaMemcpyDeviceToDevice, st()));
    }
    comm->allgather(own, all, per, st());
    for (int r = 0; r < comm->world; ++r) {
      const size_t ra = 1 + size_t(r) * chunk;
      if (ra > N) break;
      const size_t rl = std::min(N + 1, ra + chunk) - ra;
      const char* src = all + size_t(r) * per;
      auto unpack = [&](DeviceBuffer& dst, size_t k) {
        PTB_CUDA_CHECK(cudaMemcpyAsync(slot(dst, ra, nc), src + k * bc, rl * nc * sizeof(double),
                                       cudaMemcpyDeviceToDevice, st()));
      };
      unpack(rf_u, 0);
      unpack(rf_v, 1);
      unpack(kn_u, 2);
      unpack(kn_v, 3);
      const int32_t* rfl = reinterpret_cast<const int32_t*>(src + 4 * bc);
      PTB_CUDA_CHECK(cudaMemcpyAsync(fl(ff) + (ra - 1), rfl, rl * sizeof(int32_t), cudaMemcpyDeviceToDevice, st()));
      PTB_CUDA_CHECK(cudaMemcpyAsync(fl(cf) + (ra - 1), rfl + chunk, rl * sizeof(int32_t), cudaMemcpyDeviceToDevice, st()));
    }
  }

  // gather per-slice scalars: `own` (chunk * per) -> `all` slots n = 1..N
  std::vector<double> gather_scalars(const double* own_dev, size_t per) {
    std::vector<double> h;
    if (comm->world == 1) {
      h = to_host(own_dev, N * per);
      return h;
    }
    double* all = dalloc<double>(all_sc, size_t(comm->world) * chunk * per);
    comm->allgather(own_dev, all, chunk * per * sizeof(double), st());
    h = to_host(all, size_t(comm->world) * chunk * per);
    h.resize(N * per);
    return h;
  }

  // ---- stages ------------------------------------------------------------------------
  // C on `batch` coarse states with the NaN-state rule (coarse_stage, parareal.cpp:64-73).
  // sweep_step: flags pre-zeroed by the caller and the state consumed only through the theta
  // sweep's tail, which turns d_n into NaN on this same flag -> no memset, no NaN fill here.
  void coarse_propagate(double* u, double* v, size_t batch, int32_t* flags, bool sweep_step = false) {
    if (!batch) return;
    if (!sweep_step) PTB_CUDA_CHECK(cudaMemsetAsync(flags, 0, batch * sizeof(int32_t), st()));
    propagate(pc, pc->steps, batch, u, v, flags, s.mode);
    if (!sweep_step) nan_where(nc, batch, flags, nullptr, nullptr, u, v);
  }

  // reference_or_nan (parareal.cpp:133-145): chain on every rank up to its last slice
  void serial_reference() {
    copy(static_cast<double*>(ref_u.ptr), fl_init_u(), nf);
    copy(static_cast<double*>(ref_v.ptr), fl_init_v(), nf);
    int32_t* f = fl(sflags);
    PTB_CUDA_CHECK(cudaMemsetAsync(f, 0, (N + 1) * sizeof(int32_t), st()));
    // walk the chain 1..b-1 with a rolling state, storing the own states [a-1, b)
    double* pu = dalloc<double>(fine2_u, std::max<size_t>(L, 1) * nf);
    double* pv = dalloc<double>(fine2_v, std::max<size_t>(L, 1) * nf);
    copy(pu, fl_init_u(), nf);
    copy(pv, fl_init_v(), nf);
    for (size_t n = 1; n < b; ++n) {
      propagate(pf, pf->steps, 1, pu, pv, f + n, s.mode);
      if (n >= a - 1) {
        copy(RU(n), pu, nf);
        copy(RV(n), pv, nf);
      }
    }
    // any divergence anywhere in 1..N makes every reference slot n >= 1 NaN
    std::vector<int32_t> h = to_host(f, N + 1);
    double any = 0.0;
    for (size_t n = 1; n < b; ++n) any = std::max(any, double(h[n]));
    double* sc = dalloc<double>(own_sc, chunk);
    std::vector<double> mine(chunk, 0.0);
    mine[0] = any;
    PTB_CUDA_CHECK(cudaMemcpyAsync(sc, mine.data(), chunk * sizeof(double), cudaMemcpyHostToDevice, st()));
    double global_any = any;
    if (comm->world > 1) {
      double* all = dalloc<double>(all_sc, size_t(comm->world) * chunk);
      comm->allgather(sc, all, chunk * sizeof(double), st());
      std::vector<double> g = to_host(all, size_t(comm->world) * chunk);
      for (int r = 0; r < comm->world; ++r) global_any = std::max(global_any, g[size_t(r) * chunk]);
    }
    if (global_any > 0.0) {
      const size_t first = std::max<size_t>(a - 1, 1);
      if (b > first) {
        nan_fill(RU(first), (b - first) * nf);
        nan_fill(RV(first), (b - first) * nf);
      }
    }
    // reference finiteness of own slots (for measure) — every rank keeps the full vector
    PTB_CUDA_CHECK(cudaMemsetAsync(f, 0, (N + 1) * sizeof(int32_t), st()));
    if (L) {
      k_state_flags<<<dim3(std::min(64u, blocks(ctx, nf)), unsigned(L)), 256, 0, st()>>>(nf, RU(a), RV(a), nf, f + a);
      PTB_LAUNCH_CHECK(ctx);
    }
    ref_bad = to_host(f, N + 1);  // own entries valid; others unused
  }

  double* fl_init_u() { return static_cast<double*>(init_u.ptr); }
  double* fl_init_v() { return static_cast<double*>(init_v.ptr); }

  // finalize_iteration (parareal.cpp:107-128) on own states (su, sv) [a-1, b); prev may be null
  void finalize(DeviceBuffer& su_b, DeviceBuffer& sv_b, DeviceBuffer* pu_b, DeviceBuffer* pv_b, double* ee, double* l2,
                int* diverged, double* states_out) {
    double* su = static_cast<double*>(su_b.ptr);
    double* sv = static_cast<double*>(sv_b.ptr);
    HostProf hp_(st());
    int32_t* f = fl(sflags);
    PTB_CUDA_CHECK(cudaMemsetAsync(f, 0, (L + 1) * sizeof(int32_t), st()));
    // state 0 (index a-1) here; states 1..L are checked by the error sums, which read them anyway
    k_state_flags<<<dim3(std::min(64u, blocks(ctx, nf)), 1u), 256, 0, st()>>>(nf, su, sv, nf, f);
    PTB_LAUNCH_CHECK(ctx);
    double* own = dalloc<double>(sums_own, chunk * 5);
    PTB_CUDA_CHECK(cudaMemsetAsync(own, 0, chunk * 5 * sizeof(double), st()));
    if (L) {
      double* tmp = dalloc<double>(sums_all, L * 4);
      hp_.mark("finalize: flags");
      pair_energy_sums(ew, fg, s.metric_scheme, L, su + nf, sv + nf, nf, RU(a), RV(a), nf, ptb_propagator_speed(pf),
                       tmp, f + 1);
      hp_.mark("finalize: error sums");
      // pack [flag, s0..s3] per own slice
      PTB_CUDA_CHECK(cudaMemcpy2DAsync(own + 1, 5 * sizeof(double), tmp, 4 * sizeof(double), 4 * sizeof(double), L,
                                       cudaMemcpyDeviceToDevice, st()));
    }
    std::vector<int32_t> hf = to_host(f, L + 1);
    {  // flags as doubles into column 0
      std::vector<double> fd(L);
      for (size_t i = 0; i < L; ++i) fd[i] = hf[i + 1];
      if (L)
        PTB_CUDA_CHECK(cudaMemcpy2DAsync(own, 5 * sizeof(double), fd.data(), sizeof(double), sizeof(double), L,
                                         cudaMemcpyHostToDevice, st()));
    }
    const std::vector<double> g = gather_scalars(own, 5);
    const double vol = [&] {
      double v = 1.0;
      for (int k = 0; k < fg.dim; ++k) v *= fg.h[k];
      return v;
    }();
    // n = 0: the initial condition (identical on every rank)
    bool dv = init_bad;
    ee[0] = 0.0;
    l2[0] = 0.0;
    for (size_t n = 1; n <= N; ++n) {
      const double* q = &g[(n - 1) * 5];
      const bool bad_n = q[0] != 0.0;
      double e, l;
      if (bad_n || ref_bad_global[n]) {
        e = l = kInf;
      } else {
        const double e_ref = 0.5 * q[2] * vol, e_diff = 0.5 * q[1] * vol;
        e = (e_ref == 0.0) ? (e_diff == 0.0 ? 0.0 : kInf) : std::sqrt(e_diff / e_ref);
        l = (q[4] == 0.0) ? (q[3] == 0.0 ? 0.0 : kInf) : std::sqrt(q[3] / q[4]);
      }
      ee[n] = e;
      l2[n] = l;
      if (bad_n) dv = true;
    }
    *diverged = dv ? 1 : 0;
    // clamp own non-finite states to the previous iterate
    if (pu_b) {
      for (size_t i = 1; i <= L; ++i)
        if (hf[i]) {
          copy(su + i * nf, static_cast<double*>(pu_b->ptr) + i * nf, nf);
          copy(sv + i * nf, static_cast<double*>(pv_b->ptr) + i * nf, nf);
        }
    }
    if (states_out) {
      for (size_t m = (a == 1 ? 0 : a); m < b; ++m) {
        const size_t i = m - (a - 1);
        PTB_CUDA_CHECK(cudaMemcpyAsync(states_out + (2 * m) * nf, su + i * nf, nf * sizeof(double),
                                       cudaMemcpyDeviceToHost, st()));
        PTB_CUDA_CHECK(cudaMemcpyAsync(states_out + (2 * m + 1) * nf, sv + i * nf, nf * sizeof(double),
                                       cudaMemcpyDeviceToHost, st()));
      }
      PTB_CUDA_CHECK(cudaStreamSynchronize(st()));
    }
  }

  bool init_bad = false;
  std::vector<int32_t> ref_bad_global;

  void gather_ref_flags() {
    // every rank needs reference finiteness of all n for the error table
    double* own = dalloc<double>(own_sc, chunk);
    std::vector<double> h(chunk, 0.0);
    for (size_t n = a; n < b; ++n) h[n - a] = ref_bad[n];
    PTB_CUDA_CHECK(cudaMemcpyAsync(own, h.data(), chunk * sizeof(double), cudaMemcpyHostToDevice, st()));
    const std::vector<double> g = gather_scalars(own, 1);
    ref_bad_global.assign(N + 1, 0);
    for (size_t n = 1; n <= N; ++n) ref_bad_global[n] = g[n - 1] != 0.0;
  }

  // parallel stage on own slices: fine_next[n] = F(cur[n-1]), coarse_next[n] = C(R cur[n-1])
  void parallel_stage() {
    if (!L) return;
    int32_t* ffo = fl(ff) + (a - 1);
    int32_t* cfo = fl(cf) + (a - 1);
    PTB_CUDA_CHECK(cudaMemsetAsync(ffo, 0, L * sizeof(int32_t), st()));
    // fine_next[n] = F(cur[n-1]) read straight from cur (the wavefront path's first pass; no copy)
    LaunchSlot fs;
    fs.stream = st();
    fs.src_u = CU(a - 1);
    fs.src_v = CV(a - 1);
    propagate(pf, pf->steps, L, FU(a), FV(a), ffo, s.mode, &fs);
    nan_where(nf, L, ffo, nullptr, nullptr, FU(a), FV(a));
    restrict_fields(tr, L, CU(a - 1), slot(kn_u, a, nc));
    restrict_fields(tr, L, CV(a - 1), slot(kn_v, a, nc));
    coarse_propagate(slot(kn_u, a, nc), slot(kn_v, a, nc), L, cfo);
    restrict_fields(tr, L, FU(a), slot(rf_u, a, nc));
    restrict_fields(tr, L, FV(a), slot(rf_v, a, nc));
  }

  // Z = Lambda-dagger(X, 0): u and udot blocks (Nc x r each)
  void precompute_Z(const DevCorrector& c) {
    const int r = c.rank;
    if (r == 0) return;
    const size_t rows = size_t(cg.dim + 1) * nc;
    double* zu = dalloc<double>(Zu, nc * r);
    double* zv = dalloc<double>(Zv, nc * r);
    double* m0 = dalloc<double>(mean_old, std::max<size_t>(N, size_t(r)));
    PTB_CUDA_CHECK(cudaMemsetAsync(m0, 0, size_t(r) * sizeof(double), st()));
    from_energy_components(ew, cg, size_t(r), c.Xp(), rows, m0, cf_dev, zu, zv, nc);
  }

  // corrected coarse vectors for `batch` coarse states: Z (Y^T Lambda(.)) + mean/Nc, stored to (ou, ov)
  // (omega_identity: Lambda-dagger(Lambda(.)))
  void corrected_batch(const DevCorrector& c, bool omega_identity, size_t batch, const double* u, const double* v,
                       double* ou, double* ov, double* zout, double* mout) {
    const size_t rows = size_t(cg.dim + 1) * nc;
    double* cp = dalloc<double>(comp, rows * batch);
    energy_components(ew, cg, s.scheme, batch, u, v, nc, nullptr, cf_dev, cp, rows, mout);
    if (omega_identity) {
      if (ou) from_energy_components(ew, cg, batch, cp, rows, mout, cf_dev, ou, ov, nc);
      return;
    }
    if (c.rank == 0) {
      if (zout) PTB_CUDA_CHECK(cudaMemsetAsync(zout, 0, sizeof(double), st()));
      return;
    }
    if (batch == 1 && fused_sweep(c)) {  // the sweep's per-step product: one launch, fixed order, P partials
      const int P = gemv_parts(rows);
      zw_parts = P;
      k_gemv_t1<<<dim3(unsigned(c.rank), unsigned(P)), 256, 0, st()>>>(rows, (rows + P - 1) / P, c.Yp(), rows, cp,
                                                                       zout);
      PTB_LAUNCH_CHECK(ctx);
    } else if (batch == 1) {  // large corrector: the row-sharded product (bitwise the same at any world)
      zw_parts = 1;
      sharded_zt(c, cp, zout);
    } else {
      gemm(ctx, true, false, c.rank, int(batch), int(rows), 1.0, c.Yp(), int(rows), cp, int(rows), 0.0, zout,
           c.rank);
    }
  }

  // z = Y^T x for a large corrector, rows split over the ranks in SWEEP_BLOCKS fixed blocks
  void sharded_zt(const DevCorrector& c, const double* x, double* z) {
    const size_t rows = size_t(cg.dim + 1) * nc;
    const int r = c.rank, W = comm->world;
    const size_t bl = (rows + SWEEP_BLOCKS - 1) / SWEEP_BLOCKS, arr = size_t(SWEEP_BLOCKS) * r;
    double* part = dalloc<double>(zpart, arr);
    k_zt_blocks<<<dim3(unsigned(r), SWEEP_BLOCKS), 256, 0, st()>>>(rows, bl, c.Yp(), rows, x, r, comm->rank, W, part);
    PTB_LAUNCH_CHECK(ctx);
    const double* all = part;
    if (W > 1) {
      double* g = dalloc<double>(zpart_all, arr * size_t(W));
      comm->allgather(part, g, arr * sizeof(double), st());
      all = g;
    }
    k_zt_sum<<<unsigned((r + 255) / 256), 256, 0, st()>>>(r, W, all, z);
    PTB_LAUNCH_CHECK(ctx);
  }

  // du = Zu dz, dv = Zv dz for a large corrector: each rank its own row segment, one all-gather
  void sharded_zd(int r, const double* dz, double* du, double* dv) {
    const int W = comm->world, sg = int((nc + size_t(W) - 1) / size_t(W));
    const int i0 = std::min(int(nc), comm->rank * sg), i1 = std::min(int(nc), i0 + sg);
    double* seg = dalloc<double>(dseg, 2 * size_t(sg));
    if (i1 > i0)
      k_zd_rows<<<unsigned((i1 - i0 + 255) / 256), 256, size_t(r) * sizeof(double), st()>>>(
          i0, i1, sg, r, static_cast<const double*>(Zu.ptr), static_cast<const double*>(Zv.ptr), nc, dz, seg);
    PTB_LAUNCH_CHECK(ctx);
    const double* all = seg;
    if (W > 1) {
      double* g = dalloc<double>(dseg_all, 2 * size_t(sg) * size_t(W));
      comm->allgather(seg, g, 2 * size_t(sg) * sizeof(double), st());
      all = g;
    }
    k_zd_unpack<<<blocks(ctx, nc), 256, 0, st()>>>(nc, sg, all, du, dv);
    PTB_LAUNCH_CHECK(ctx);
  }

  // ---- sweeps (coarse, replicated) --------------------------------------------------------

  // R(next) for the first step: R(init)
  void restrict_init(double* ou, double* ov) {
    restrict_fields(tr, 1, fl_init_u(), ou);
    restrict_fields(tr, 1, fl_init_v(), ov);
  }

  // d (coarse) = Z (z_w - z_old) + (m_w - m_old)/Nc  [u], Zv (z_w - z_old) [udot]
  void assemble_d(const DevCorrector& c, const double* zw_, const double* zold_, const double* mw, const double* mold,
                  double* du, double* dv, int mparts = 1, const SweepTail& tail = SweepTail{}) {
    const int r = c.rank;
    if (fused_sweep(c)) {
      const size_t smem = (size_t(r + 1) + 2 * AD_J * AD_I) * sizeof(double);
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(unsigned((nc + AD_I - 1) / AD_I));
      cfg.blockDim = dim3(AD_I, AD_J);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st();
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = pdl_enabled() ? 1 : 0;
      PTB_CUDA_CHECK(cudaLaunchKernelEx(&cfg, k_assemble_d, nc, r, static_cast<const double*>(Zu.ptr),
                                        static_cast<const double*>(Zv.ptr), zw_, zw_parts, zold_, mw, mparts, mold, du,
                                        dv, tail));
      PTB_LAUNCH_CHECK(ctx);
      return;
    }
    // large corrector (cfg4: 3 N_c x r up to ~200 M entries): HBM-bound GEMVs, rows sharded
    // over the ranks (each streams 1/world of Zu, Zv), d all-gathered
    double* dz = dalloc<double>(tmpc, std::max(r, 1));
    if (r > 0) {
      if (zold_) {
        k_sub<<<1, 256, 0, st()>>>(size_t(r), zw_, zold_, dz);
        PTB_LAUNCH_CHECK(ctx);
      } else {
        copy(dz, zw_, size_t(r));
      }
      sharded_zd(r, dz, du, dv);
    } else {
      PTB_CUDA_CHECK(cudaMemsetAsync(du, 0, nc * sizeof(double), st()));
      PTB_CUDA_CHECK(cudaMemsetAsync(dv, 0, nc * sizeof(double), st()));
    }
    k_add_mean<<<blocks(ctx, nc), 256, 0, st()>>>(nc, mw, mold, du);
    PTB_LAUNCH_CHECK(ctx);
  }

  // theta sweep, additive (parareal.cpp:311-331) on coarse vectors -> d[n], bad[n]
  void theta_sweep(const DevCorrector& c, bool omega_identity) {
    const size_t rows = size_t(cg.dim + 1) * nc;
    int32_t* wfl = fl(wf);
    PTB_CUDA_CHECK(cudaMemsetAsync(wfl, 0, (N + 1) * sizeof(int32_t), st()));
    // "old" terms for n = 2..N, one batch
    double* zo = nullptr;
    double* mo = dalloc<double>(mean_old, std::max<size_t>(N, size_t(c.rank)));
    double* cold = nullptr;
    if (N >= 2) {
      if (omega_identity) {
        cold = dalloc<double>(comp_old, rows * (N - 1));
        energy_components(ew, cg, s.scheme, N - 1, slot(kn_u, 2, nc), slot(kn_v, 2, nc), nc, nullptr, cf_dev, cold,
                          rows, mo + 1);
      } else {
        precompute_Z(c);
        zo = dalloc<double>(zold, std::max<size_t>(1, size_t(c.rank) * N));
        corrected_batch(c, false, N - 1, slot(kn_u, 2, nc), slot(kn_v, 2, nc), nullptr, nullptr,
                        zo + size_t(c.rank), mo + 1);
      }
    }
    double* zwp = dalloc<double>(zw, size_t(std::max(c.rank, 1)) * 64);  // r x P partials
    double* mw = dalloc<double>(mean, std::max<size_t>(N, 64));  // >= 64: sum(u) partials of comp_gemv
    double* ru = static_cast<double*>(rn_u.ptr);
    double* rv = static_cast<double*>(rn_v.ptr);
    // n = 1: next[1] = fine_next[1]  ->  d_1 = 0, R(next[1]) = R(fine_next[1])
    PTB_CUDA_CHECK(cudaMemsetAsync(slot(d_u, 1, nc), 0, nc * sizeof(double), st()));
    PTB_CUDA_CHECK(cudaMemsetAsync(slot(d_v, 1, nc), 0, nc * sizeof(double), st()));
    copy(ru, slot(rf_u, 1, nc), nc);
    copy(rv, slot(rf_v, 1, nc), nc);
    for (size_t n = 2; n <= N; ++n) {
      coarse_propagate(ru, rv, 1, wfl + n, /*sweep_step=*/true);  // w = C(R next[n-1]) in place
      double* du = slot(d_u, n, nc);
      double* dv = slot(d_v, n, nc);
      if (omega_identity) {
        double* cw = dalloc<double>(comp, rows);
        energy_components(ew, cg, s.scheme, 1, ru, rv, nc, nullptr, cf_dev, cw, rows, mw);
        k_sub<<<blocks(ctx, rows), 256, 0, st()>>>(rows, cw, cold + (n - 2) * rows, cw);
        k_sub<<<1, 32, 0, st()>>>(1, mw, mo + (n - 1), mw + 1);
        PTB_LAUNCH_CHECK(ctx);
        from_energy_components(ew, cg, 1, cw, rows, mw + 1, cf_dev, du, dv, nc);
      } else if (fused_sweep(c) && s.scheme != PTB_SPECTRAL) {
        // one launch for Lambda(w), z_w = Y^T Lambda(w) and sum(u); one for d, the NaN rule and
        // R(next[n]) = R(fine_next[n]) + d_n
        const int P = comp_gemv_parts(rows);
        zw_parts = P;
        comp_gemv(ew, cg, s.scheme, ru, rv, cf_dev, c.Yp(), rows, c.rank, zwp, P, mw);
        const bool more = n < N;
        const SweepTail tail{wfl + n, fl(cf) + (n - 1), fl(ff) + (n - 1), more ? slot(rf_u, n, nc) : nullptr,
                             more ? slot(rf_v, n, nc) : nullptr, more ? ru : nullptr, more ? rv : nullptr};
        assemble_d(c, zwp, zo + (n - 1) * size_t(c.rank), mw, mo + (n - 1), du, dv, sweep_mean_parts(int(nc)), tail);
        continue;
      } else if (comm->world == 1 && s.scheme != PTB_SPECTRAL) {
        // one GPU, large corrector: Lambda(w) and sum(u); the row-block partials of z_w; one launch
        // for the rest of the step (k_zd_fused: bitwise the multi-rank path's operations)
        double* cp = dalloc<double>(comp, rows);
        energy_components(ew, cg, s.scheme, 1, ru, rv, nc, nullptr, cf_dev, cp, rows, mw);
        const int r = c.rank;
        double* part = dalloc<double>(zpart, size_t(SWEEP_BLOCKS) * std::max(r, 1));
        if (r > 0)
          launch_pdl(k_zt_blocks, dim3(unsigned(r), SWEEP_BLOCKS), dim3(256), 0, st(), rows,
                     (rows + SWEEP_BLOCKS - 1) / SWEEP_BLOCKS, c.Yp(), rows, static_cast<const double*>(cp), r, 0, 1,
                     part);
        const bool more = n < N;
        const SweepTail tail{wfl + n, fl(cf) + (n - 1), fl(ff) + (n - 1), more ? slot(rf_u, n, nc) : nullptr,
                             more ? slot(rf_v, n, nc) : nullptr, more ? ru : nullptr, more ? rv : nullptr};
        launch_pdl(k_zd_fused, dim3(unsigned((nc + 255) / 256)), dim3(256), size_t(std::max(r, 1)) * sizeof(double),
                   st(), int(nc), r, static_cast<const double*>(Zu.ptr), static_cast<const double*>(Zv.ptr), nc,
                   static_cast<const double*>(part), static_cast<const double*>(zo + (n - 1) * size_t(r)),
                   static_cast<const double*>(mw), static_cast<const double*>(mo + (n - 1)), du, dv, tail);
        PTB_LAUNCH_CHECK(ctx);
        continue;
      } else {
        corrected_batch(c, false, 1, ru, rv, nullptr, nullptr, zwp, mw);
        assemble_d(c, zwp, zo + (n - 1) * size_t(c.rank), mw, mo + (n - 1), du, dv);
      }
      // NaN flags (parareal.cpp:323-326) and R(next[n]) = R(fine_next[n]) + d_n, one launch
      const bool more = n < N;
      k_sweep_tail<<<blocks(ctx, nc), 256, 0, st()>>>(nc, wfl + n, fl(cf) + (n - 1), fl(ff) + (n - 1), du, dv,
                                                      more ? slot(rf_u, n, nc) : nullptr,
                                                      more ? slot(rf_v, n, nc) : nullptr, more ? ru : nullptr,
                                                      more ? rv : nullptr);
      PTB_LAUNCH_CHECK(ctx);
    }
  }

  // corrected-coarse-only sweep (parareal.cpp:332-338): d[n] = corrected(C R next[n-1])
  void corrected_only_sweep(const DevCorrector& c, bool omega_identity) {
    int32_t* wfl = fl(wf);
    PTB_CUDA_CHECK(cudaMemsetAsync(wfl, 0, (N + 1) * sizeof(int32_t), st()));
    if (!omega_identity) precompute_Z(c);
    double* zwp = dalloc<double>(zw, size_t(std::max(c.rank, 1)) * 64);  // r x P partials
    double* mw = dalloc<double>(mean, std::max<size_t>(N, 1));
    double* ru = static_cast<double*>(rn_u.ptr);
    double* rv = static_cast<double*>(rn_v.ptr);
    restrict_init(ru, rv);
    for (size_t n = 1; n <= N; ++n) {
      coarse_propagate(ru, rv, 1, wfl + n);
      double* du = slot(d_u, n, nc);
      double* dv = slot(d_v, n, nc);
      if (omega_identity) {
        corrected_batch(c, true, 1, ru, rv, du, dv, nullptr, mw);
      } else {
        corrected_batch(c, false, 1, ru, rv, nullptr, nullptr, zwp, mw);
        assemble_d(c, zwp, nullptr, mw, nullptr, du, dv);
      }
      nan_where(nc, 1, wfl + n, nullptr, nullptr, du, dv);
      interpolate_at_coarse_nodes(tr, 1, du, ru);
      interpolate_at_coarse_nodes(tr, 1, dv, rv);
    }
  }

  // plain sweep (parareal.cpp:222-231): w[n] = C(R next[n-1]); R next[n] = (RI w + RF) - RI K
  void plain_sweep() {
    int32_t* wfl = fl(wf);
    PTB_CUDA_CHECK(cudaMemsetAsync(wfl, 0, (N + 1) * sizeof(int32_t), st()));
    interpolate_at_coarse_nodes(tr, N, slot(kn_u, 1, nc), slot(rik_u, 1, nc));
    interpolate_at_coarse_nodes(tr, N, slot(kn_v, 1, nc), slot(rik_v, 1, nc));
    double* ru = static_cast<double*>(rn_u.ptr);
    double* rv = static_cast<double*>(rn_v.ptr);
    restrict_init(ru, rv);
    for (size_t n = 1; n <= N; ++n) {
      double* wu = slot(w_u, n, nc);
      double* wv = slot(w_v, n, nc);
      copy(wu, ru, nc);
      copy(wv, rv, nc);
      coarse_propagate(wu, wv, 1, wfl + n);
      if (n < N) {
        interpolate_at_coarse_nodes(tr, 1, wu, static_cast<double*>(ri_u.ptr));
        interpolate_at_coarse_nodes(tr, 1, wv, static_cast<double*>(ri_v.ptr));
        k_add_sub<<<blocks(ctx, nc), 256, 0, st()>>>(nc, static_cast<double*>(ri_u.ptr), slot(rf_u, n, nc),
                                                       slot(rik_u, n, nc), ru);
        k_add_sub<<<blocks(ctx, nc), 256, 0, st()>>>(nc, static_cast<double*>(ri_v.ptr), slot(rf_v, n, nc),
                                                       slot(rik_v, n, nc), rv);
        PTB_LAUNCH_CHECK(ctx);
      }
    }
  }

  // serial_coarse_init (parareal.cpp:147-159): cur[n] = I(C R cur[n-1]) via the coarse chain
  void serial_coarse_init() {
    int32_t* wfl = fl(wf);
    PTB_CUDA_CHECK(cudaMemsetAsync(wfl, 0, (N + 1) * sizeof(int32_t), st()));
    double* ru = static_cast<double*>(rn_u.ptr);
    double* rv = static_cast<double*>(rn_v.ptr);
    restrict_init(ru, rv);
    for (size_t n = 1; n <= N; ++n) {
      double* wu = slot(w_u, n, nc);
      double* wv = slot(w_v, n, nc);
      copy(wu, ru, nc);
      copy(wv, rv, nc);
      coarse_propagate(wu, wv, 1, wfl + n);
      if (n < N) {
        interpolate_at_coarse_nodes(tr, 1, wu, ru);
        interpolate_at_coarse_nodes(tr, 1, wv, rv);
      }
    }
    if (a == 1) {
      copy(CU(0), fl_init_u(), nf);
      copy(CV(0), fl_init_v(), nf);
    }
    if (L) {
      interpolate_fields(tr, L, slot(w_u, a, nc), CU(a));
      interpolate_fields(tr, L, slot(w_v, a, nc), CV(a));
      nan_where(nf, L, wfl + a, nullptr, nullptr, CU(a), CV(a));
    }
  }

  // fine combine on own slices -> nxt
  void fine_combine(bool theta, bool additive) {
    if (a == 1) {
      copy(NU(0), fl_init_u(), nf);
      copy(NV(0), fl_init_v(), nf);
    }
    if (!L) return;
    HostProf hp_(st());
    double* iu = dalloc<double>(fine_u, L * nf);
    double* iv = dalloc<double>(fine_v, L * nf);
    if (theta && additive) {
      // next = fine_next + I(d): fused into the interpolation's last pass on the FFT route
      interpolate_fields_add(tr, L, slot(d_u, a, nc), FU(a), NU(a), iu);
      interpolate_fields_add(tr, L, slot(d_v, a, nc), FV(a), NV(a), iv);
      hp_.mark("combine: interpolate + add");
      {
        if (a == 1) {  // next[1] = fine_next[1] exactly
          copy(NU(1), FU(1), nf);
          copy(NV(1), FV(1), nf);
        }
        nan_where(nf, L, fl(wf) + a, fl(cf) + (a - 1), fl(ff) + (a - 1), NU(a), NV(a));
        if (a == 1) {  // n = 1 carries fine_next[1] as is, whatever its finiteness
          copy(NU(1), FU(1), nf);
          copy(NV(1), FV(1), nf);
        }
      }
    } else if (theta) {
      interpolate_fields(tr, L, slot(d_u, a, nc), NU(a));
      interpolate_fields(tr, L, slot(d_v, a, nc), NV(a));
      nan_where(nf, L, fl(wf) + a, nullptr, nullptr, NU(a), NV(a));
    } else {
      // (I(w) + fine_next) - I(coarse_next), with NaN states where w / coarse_next diverged
      double* ku = dalloc<double>(fine2_u, L * nf);
      double* kv = dalloc<double>(fine2_v, L * nf);
      interpolate_fields(tr, L, slot(w_u, a, nc), iu);
      interpolate_fields(tr, L, slot(w_v, a, nc), iv);
      nan_where(nf, L, fl(wf) + a, nullptr, nullptr, iu, iv);
      interpolate_fields(tr, L, slot(kn_u, a, nc), ku);
      interpolate_fields(tr, L, slot(kn_v, a, nc), kv);
      nan_where(nf, L, fl(cf) + (a - 1), nullptr, nullptr, ku, kv);
      k_add_sub<<<blocks(ctx, L * nf), 256, 0, st()>>>(L * nf, iu, FU(a), ku, NU(a));
      k_add_sub<<<blocks(ctx, L * nf), 256, 0, st()>>>(L * nf, iv, FV(a), kv, NV(a));
      PTB_LAUNCH_CHECK(ctx);
    }
  }

  // boundary: state b-1 -> next rank's slot a'-1
  void exchange_boundary(DeviceBuffer& u_b, DeviceBuffer& v_b) {
    if (comm->world == 1) return;
    const bool has_next = comm->rank + 1 < comm->world && b <= N;
    const bool has_prev = comm->rank > 0 && a <= N;
    double* u = static_cast<double*>(u_b.ptr);
    double* v = static_cast<double*>(v_b.ptr);
    comm->shift_right(u + L * nf, nf * sizeof(double), has_next && L > 0, u, nf * sizeof(double), has_prev, st());
    comm->shift_right(v + L * nf, nf * sizeof(double), has_next && L > 0, v, nf * sizeof(double), has_prev, st());
  }

  void run(const double* u0h, const double* v0h, double* ee, double* l2, double* residual, int* rank, int* diverged,
           double* states, double* reference) {
    PTB_CUDA_CHECK(cudaMemcpyAsync(fl_init_u(), u0h, nf * sizeof(double), cudaMemcpyHostToDevice, st()));
    PTB_CUDA_CHECK(cudaMemcpyAsync(fl_init_v(), v0h, nf * sizeof(double), cudaMemcpyHostToDevice, st()));
    init_bad = false;
    for (size_t i = 0; i < nf; ++i)
      if (!std::isfinite(u0h[i]) || !std::isfinite(v0h[i])) {
        init_bad = true;
        break;
      }
    cudaEvent_t ev[7];
    for (auto& e : ev) PTB_CUDA_CHECK(cudaEventCreate(&e));
    auto ms = [&](cudaEvent_t x, cudaEvent_t y) {
      float t = 0;
      cudaEventElapsedTime(&t, x, y);
      return double(t);
    };
    PTB_CUDA_CHECK(cudaEventRecord(ev[0], st()));
    serial_reference();
    PTB_CUDA_CHECK(cudaEventRecord(ev[1], st()));
    PTB_CUDA_CHECK(cudaEventSynchronize(ev[1]));
    if (times) times->reference_ms = ms(ev[0], ev[1]);
    gather_ref_flags();
    if (reference) {
      for (size_t m = (a == 1 ? 0 : a); m < b; ++m) {
        PTB_CUDA_CHECK(cudaMemcpyAsync(reference + 2 * m * nf, RU(m), nf * sizeof(double), cudaMemcpyDeviceToHost, st()));
        PTB_CUDA_CHECK(
            cudaMemcpyAsync(reference + (2 * m + 1) * nf, RV(m), nf * sizeof(double), cudaMemcpyDeviceToHost, st()));
      }
      PTB_CUDA_CHECK(cudaStreamSynchronize(st()));
    }
    serial_coarse_init();
    residual[0] = kNaN;
    rank[0] = 0;
    finalize(cur_u, cur_v, nullptr, nullptr, ee, l2, diverged, states);
    exchange_boundary(cur_u, cur_v);

    const bool theta = s.variant != PTB_PLAIN;
    const bool omega_identity = s.variant == PTB_OMEGA_IDENTITY;
    const bool additive = s.variant != PTB_CORRECTED_COARSE_ONLY;
    const size_t rows = size_t(cg.dim + 1) * nc;
    double* Fp = dalloc<double>(Fm, rows * N);
    double* Gp = dalloc<double>(Gm, rows * N);
    int* idx_d = dalloc<int>(idx, N);
    if (theta) {
      // the rank-sized buffers for a corrector of up to 2 N columns now: inside an iteration their
      // growth is a cudaFree + cudaMalloc pair each, which synchronises the device and was measured
      // at 2-700 ms; a larger rank still grows them geometrically
      const size_t rcap = std::min<size_t>(rows, 2 * N);
      for (DeviceBuffer* bf : {&corr.X, &corr.Y, &pw.SX, &pw.SY}) bf->get(rows * rcap * sizeof(double));
      dalloc<double>(Zu, nc * rcap);
      dalloc<double>(Zv, nc * rcap);
      for (int i = 1; i <= 3; ++i) ew.buf[i].get(nc * rcap * 2 * sizeof(double));  // Lambda-dagger planes
    }
    DevCorrector dropped;
    for (int k = 1; k <= K; ++k) {
      PTB_CUDA_CHECK(cudaEventRecord(ev[0], st()));
      parallel_stage();
      PTB_CUDA_CHECK(cudaEventRecord(ev[1], st()));
      gather_payload();
      PTB_CUDA_CHECK(cudaEventRecord(ev[2], st()));
      double res = kNaN;
      int rk = 0;
      const DevCorrector* applied = &corr;
      if (theta) {
        const std::vector<int32_t> ffh = to_host(fl(ff), N), cfh = to_host(fl(cf), N);
        std::vector<int> keep;
        for (size_t n = 1; n <= N; ++n)
          if (!ffh[n - 1] && !cfh[n - 1]) keep.push_back(int(n - 1));
        if (!keep.empty()) {
          const int cols = int(keep.size());
          PTB_CUDA_CHECK(cudaMemcpyAsync(idx_d, keep.data(), keep.size() * sizeof(int), cudaMemcpyHostToDevice, st()));
          // assemble_snapshots (procrustes.cpp:158-175) from the gathered coarse payload
          energy_components(ew, cg, s.scheme, size_t(cols), slot(rf_u, 1, nc), slot(rf_v, 1, nc), nc, idx_d, cf_dev,
                            Fp, rows, nullptr);
          energy_components(ew, cg, s.scheme, size_t(cols), slot(kn_u, 1, nc), slot(kn_v, 1, nc), nc, idx_d, cf_dev,
                            Gp, rows, nullptr);
          if (omega_identity) {
            std::vector<double> nrm(2);
            double* d2 = dalloc<double>(tmpc, 2);
            column_sumsq(ctx, int(rows * cols), 1, Fp, rows * cols, d2);
            double* D = dalloc<double>(comp_old, rows * cols);
            k_sub<<<blocks(ctx, rows * cols), 256, 0, st()>>>(rows * cols, Fp, Gp, D);
            PTB_LAUNCH_CHECK(ctx);
            column_sumsq(ctx, int(rows * cols), 1, D, rows * cols, d2 + 1);
            nrm = to_host(d2, 2);
            res = nrm[0] > 0.0 ? std::sqrt(nrm[1]) / std::sqrt(nrm[0]) : 0.0;
          } else {
            HostProf hp_(st());
            pw.comm = comm;  // the factor update's tall products and QRs are row-sharded over the ranks
            update_svd(pw, corr, Fp, Gp, int(rows), cols, s.tol);
            pw.comm = nullptr;
            hp_.mark("driver: update_svd total");
            if (s.remove_leading > 0) {
              drop_leading(corr, size_t(s.remove_leading), dropped, ctx);
              applied = &dropped;
            }
            res = relative_residual(pw, *applied, Fp, Gp, int(rows), cols);
            hp_.mark("driver: residual");
            rk = applied->rank;
          }
        } else if (!omega_identity) {
          drop_leading(corr, size_t(std::max(0, s.remove_leading)), dropped, ctx);
          applied = &dropped;
          rk = applied->rank;
        }
      }
      PTB_CUDA_CHECK(cudaEventRecord(ev[3], st()));
      if (!theta)
        plain_sweep();
      else if (additive)
        theta_sweep(*applied, omega_identity);
      else
        corrected_only_sweep(*applied, omega_identity);
      PTB_CUDA_CHECK(cudaEventRecord(ev[4], st()));
      fine_combine(theta, additive);
      residual[k] = res;
      rank[k] = rk;
      finalize(nxt_u, nxt_v, &cur_u, &cur_v, ee + size_t(k) * (N + 1), l2 + size_t(k) * (N + 1), diverged + k,
               states ? states + size_t(k) * (N + 1) * 2 * nf : nullptr);
      exchange_boundary(nxt_u, nxt_v);
      PTB_CUDA_CHECK(cudaEventRecord(ev[5], st()));
      PTB_CUDA_CHECK(cudaEventSynchronize(ev[5]));
      if (times && k <= PTB_MAX_TIMED_ITERS) {
        times->parallel_ms[k - 1] = ms(ev[0], ev[1]);
        times->gather_ms[k - 1] = ms(ev[1], ev[2]);
        times->procrustes_ms[k - 1] = ms(ev[2], ev[3]);
        times->sweep_ms[k - 1] = ms(ev[3], ev[4]);
        times->finalize_ms[k - 1] = ms(ev[4], ev[5]);
        times->iteration_ms[k - 1] = ms(ev[0], ev[5]);
      }
      std::swap(cur_u, nxt_u);
      std::swap(cur_v, nxt_v);
    }
    for (auto& e : ev) cudaEventDestroy(e);
  }
};

void run_parareal(ptb_context* ctx, const Comm* comm, const ptb_run_spec& spec, const double* cf, const double* cc,
                  const double* u0, const double* v0, double* ee, double* l2, double* residual, int* rank,
                  int* diverged, double* states, double* reference, ptb_phase_times* times) {
  std::lock_guard<std::recursive_mutex> lock(ctx->mutex);
  Driver d(ctx, comm, spec);
  d.times = times;
  d.setup(cf, cc);
  d.run(u0, v0, ee, l2, residual, rank, diverged, states, reference);
}

}  // namespace ptb
