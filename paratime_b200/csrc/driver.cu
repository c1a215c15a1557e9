// Device-resident parareal drivers: serial fine reference, plain parareal, theta
// (data-driven Procrustes) parareal and the corrected-coarse-only ablation.
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
// Every fine/coarse state, snapshot matrix and corrector factor stays in HBM for the whole
// run.  The parallel stage is one batched K1 call over all N slices (fine) plus one over
// their restrictions (coarse); snapshot assembly is a batched Lambda into the columns of
// F and G; the corrector update is ptb::update_svd; the corrected "old" coarse states of
// the sweep do not depend on the sweep and are computed for all n in one batch before it.
// Host control flow reads back only per-slice flags and scalar sums.

#include <cmath>
#include <cstring>
#include <limits>
#include <vector>

#include <math_constants.h>

#include "ptb_driver.h"
#include "ptb_energy.h"
#include "ptb_procrustes.h"

namespace ptb {
namespace {

constexpr double kNaN = std::numeric_limits<double>::quiet_NaN();
constexpr double kInf = std::numeric_limits<double>::infinity();

__global__ void k_fill(size_t n, double v, double* a) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) a[i] = v;
}

// per-state NaN fill where flags[b] != 0 (fine_stage/coarse_stage NaN states)
__global__ void k_nan_where(size_t n, size_t batch, const int32_t* flags, double* u, double* v) {
  const size_t total = n * batch;
  for (size_t e = blockIdx.x * size_t(blockDim.x) + threadIdx.x; e < total; e += size_t(gridDim.x) * blockDim.x) {
    const size_t b = e / n;
    if (flags[b]) {
      u[e] = CUDART_NAN;
      v[e] = CUDART_NAN;
    }
  }
}

// theta sweep combine (parareal.cpp:321-331): next = fine + I(diff), or NaN when any of
// w, coarse_next[n], fine_next[n] is non-finite.
__global__ void k_combine_theta(size_t n, const int32_t* wflag, const int32_t* cflag, const int32_t* fflag,
                                const double* fu, const double* fv, const double* du, const double* dv, double* ou,
                                double* ov) {
  const bool bad = *wflag || *cflag || *fflag;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    if (bad) {
      ou[i] = CUDART_NAN;
      ov[i] = CUDART_NAN;
    } else {
      ou[i] = __dadd_rn(fu[i], du[i]);
      ov[i] = __dadd_rn(fv[i], dv[i]);
    }
  }
}

// corrected-coarse-only: next = I(corrected) or NaN when w is non-finite
__global__ void k_nan_if(size_t n, const int32_t* flag, double* u, double* v) {
  if (!*flag) return;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    u[i] = CUDART_NAN;
    v[i] = CUDART_NAN;
  }
}

// plain sweep (parareal.cpp:224-230): next = (I C R next[n-1] + fine_next[n]) - coarse_next[n]
__global__ void k_combine_plain(size_t n, const int32_t* wflag, const double* cu, const double* cv, const double* fu,
                                const double* fv, const double* ou_, const double* ov_, double* nu, double* nv) {
  const bool bad = *wflag;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x) {
    const double a = bad ? CUDART_NAN : cu[i];
    const double b = bad ? CUDART_NAN : cv[i];
    nu[i] = __dsub_rn(__dadd_rn(a, fu[i]), ou_[i]);
    nv[i] = __dsub_rn(__dadd_rn(b, fv[i]), ov_[i]);
  }
}

__global__ void k_sub(size_t n, const double* a, const double* b, double* o) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    o[i] = __dsub_rn(a[i], b[i]);
}

__global__ void k_state_flags(size_t n, size_t batch, const double* u, const double* v, size_t stride, int32_t* flags) {
  const size_t b = blockIdx.y;
  bool ok = true;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n; i += size_t(gridDim.x) * blockDim.x)
    ok &= isfinite(u[b * stride + i]) && isfinite(v[b * stride + i]);
  const int bad = __syncthreads_or(!ok);
  if (bad && threadIdx.x == 0) atomicOr(&flags[b], 1);
}

unsigned blocks(ptb_context* ctx, size_t n) {
  return unsigned(std::max<size_t>(1, std::min<size_t>((n + 255) / 256, size_t(ctx->num_sms) * 16)));
}

template <typename T>
T* dalloc(DeviceBuffer& b, size_t count) {
  return static_cast<T*>(b.get(std::max<size_t>(1, count) * sizeof(T)));
}

}  // namespace

// ------------------------------------------------------------------------------------

struct Driver {
  ptb_context* ctx;
  const ptb_run_spec& s;
  ptb_grid fg{}, cg{};
  size_t nf = 0, nc = 0, N = 0;
  int K = 0;
  ptb_propagator* pf = nullptr;
  ptb_propagator* pc = nullptr;
  ptb_transfer* tr = nullptr;
  EnergyWork ew;
  ProcWork pw;
  // device arrays
  DeviceBuffer ref_u, ref_v, cur_u, cur_v, nxt_u, nxt_v, fn_u, fn_v, cn_u, cn_v, cold_u, cold_v;
  DeviceBuffer flags_f, flags_c, flags_w, flags_s, flags_ref, sums, Fm, Gm, idx, comp, mean, comp2, mean2, wc_u,
      wc_v, tmp_u, tmp_v, fine_tmp_u, fine_tmp_v, cnew_u, cnew_v, cof_u, cof_v;
  std::vector<int32_t> ref_bad;  // per n (host)
  DevCorrector corr;
  ptb_phase_times* times = nullptr;

  Driver(ptb_context* c, const ptb_run_spec& spec) : ctx(c), s(spec), ew(c), pw(c) {}
  ~Driver() {
    ptb_propagator_destroy(pf);
    ptb_propagator_destroy(pc);
    ptb_transfer_destroy(tr);
  }

  cudaStream_t st() const { return ctx->stream; }

  void nan_fill(double* p, size_t n) {
    k_fill<<<blocks(ctx, n), 256, 0, st()>>>(n, kNaN, p);
    PTB_LAUNCH_CHECK(ctx);
  }

  void copy(double* dst, const double* src, size_t n) {
    PTB_CUDA_CHECK(cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyDeviceToDevice, st()));
  }

  void setup(const double* cf, const double* cc) {
    fg.dim = cg.dim = s.dim;
    for (int a = 0; a < 2; ++a) {
      fg.n[a] = s.fine_n[a];
      fg.h[a] = s.fine_h[a];
      cg.n[a] = s.coarse_n[a];
      cg.h[a] = s.coarse_h[a];
    }
    validate_grid(fg);
    validate_grid(cg);
    nf = grid_size(fg);
    nc = grid_size(cg);
    N = s.n_couplings;
    K = s.iterations;
    // PropagatorConfig x2 (propagator.cpp:11-27)
    ptb_status st1 = ptb_propagator_create(ctx, &fg, cf, s.dt_fine, s.m_fine, &pf);
    if (st1 != PTB_OK) fail(st1, g_last_error);
    ptb_status st2 = ptb_propagator_create(ctx, &cg, cc, s.dt_coarse, s.m_coarse, &pc);
    if (st2 != PTB_OK) fail(st2, g_last_error);
    // CouplingSchedule (parareal.cpp:172-188)
    require(s.T > 0.0 && s.dt_com > 0.0 && N > 0, "CouplingSchedule: T, dt_com, N must be positive");
    require(std::abs(double(N) * s.dt_com - s.T) <= 1e-9 * s.T, "CouplingSchedule: N * dt_com must equal T");
    require(std::abs(double(s.m_fine) * s.dt_fine - s.dt_com) <= 1e-12 * s.dt_com,
            "CouplingSchedule: fine steps_per_coupling * dt != dt_com");
    require(std::abs(double(s.m_coarse) * s.dt_coarse - s.dt_com) <= 1e-12 * s.dt_com,
            "CouplingSchedule: coarse steps_per_coupling * dt != dt_com");
    ptb_status st3 = ptb_transfer_create(ctx, &cg, &fg, s.interp, &tr);
    if (st3 != PTB_OK) fail(st3, g_last_error);
    require(K >= 0, "parareal: negative iteration count");
    require(s.variant >= 0 && s.variant <= 3, "parareal: unknown variant");
    require(s.mode == PTB_MODE_FAST || s.mode == PTB_MODE_EXACT, "parareal: unknown propagator mode");
    const size_t S = (N + 1) * nf;
    dalloc<double>(ref_u, S);
    dalloc<double>(ref_v, S);
    dalloc<double>(cur_u, S);
    dalloc<double>(cur_v, S);
    dalloc<double>(nxt_u, S);
    dalloc<double>(nxt_v, S);
    dalloc<double>(fn_u, N * nf);
    dalloc<double>(fn_v, N * nf);
    dalloc<double>(cn_u, N * nc);
    dalloc<double>(cn_v, N * nc);
    dalloc<int32_t>(flags_f, N);
    dalloc<int32_t>(flags_c, N);
    dalloc<int32_t>(flags_w, N + 1);
    dalloc<int32_t>(flags_s, N + 1);
    dalloc<double>(sums, 4 * (N + 1));
    dalloc<double>(wc_u, nc);
    dalloc<double>(wc_v, nc);
  }

  double* RU(size_t n) { return static_cast<double*>(ref_u.ptr) + n * nf; }
  double* RV(size_t n) { return static_cast<double*>(ref_v.ptr) + n * nf; }
  double* CU(size_t n) { return static_cast<double*>(cur_u.ptr) + n * nf; }
  double* CV(size_t n) { return static_cast<double*>(cur_v.ptr) + n * nf; }
  double* NU(size_t n) { return static_cast<double*>(nxt_u.ptr) + n * nf; }
  double* NV(size_t n) { return static_cast<double*>(nxt_v.ptr) + n * nf; }
  double* FU(size_t n) { return static_cast<double*>(fn_u.ptr) + (n - 1) * nf; }  // n = 1..N
  double* FV(size_t n) { return static_cast<double*>(fn_v.ptr) + (n - 1) * nf; }
  double* KU(size_t n) { return static_cast<double*>(cn_u.ptr) + (n - 1) * nc; }
  double* KV(size_t n) { return static_cast<double*>(cn_v.ptr) + (n - 1) * nc; }
  int32_t* fl(DeviceBuffer& b) { return static_cast<int32_t*>(b.ptr); }

  // coarse_stage on one fine state (parareal.cpp:66-73) into (wu, wv); flag -> *flag
  void coarse_stage(const double* u, const double* v, double* wu, double* wv, int32_t* flag) {
    restrict_fields(tr, 1, u, wu);
    restrict_fields(tr, 1, v, wv);
    PTB_CUDA_CHECK(cudaMemsetAsync(flag, 0, sizeof(int32_t), st()));
    propagate(pc, pc->steps, 1, wu, wv, flag, s.mode);
    k_nan_where<<<blocks(ctx, nc), 256, 0, st()>>>(nc, 1, flag, wu, wv);
    PTB_LAUNCH_CHECK(ctx);
  }

  // reference_or_nan (parareal.cpp:133-145)
  void serial_reference() {
    copy(RU(0), s_u0, nf);
    copy(RV(0), s_v0, nf);
    int32_t* f = fl(flags_w);
    PTB_CUDA_CHECK(cudaMemsetAsync(f, 0, (N + 1) * sizeof(int32_t), st()));
    for (size_t n = 1; n <= N; ++n) {
      copy(RU(n), RU(n - 1), nf);
      copy(RV(n), RV(n - 1), nf);
      propagate(pf, pf->steps, 1, RU(n), RV(n), f + n, s.mode);
    }
    std::vector<int32_t> h(N + 1);
    PTB_CUDA_CHECK(cudaMemcpyAsync(h.data(), f, (N + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, st()));
    PTB_CUDA_CHECK(cudaStreamSynchronize(st()));
    bool any = false;
    for (size_t n = 1; n <= N; ++n) any |= h[n] != 0;
    if (any) {  // serial_fine threw: every n >= 1 becomes NaN
      nan_fill(RU(1), N * nf);
      nan_fill(RV(1), N * nf);
    }
    // reference finiteness per n (init may itself be non-finite)
    int32_t* rf = dalloc<int32_t>(flags_ref, N + 1);
    PTB_CUDA_CHECK(cudaMemsetAsync(rf, 0, (N + 1) * sizeof(int32_t), st()));
    k_state_flags<<<dim3(blocks(ctx, nf) > 64 ? 64 : blocks(ctx, nf), unsigned(N + 1)), 256, 0, st()>>>(
        nf, N + 1, RU(0), RV(0), nf, rf);
    PTB_LAUNCH_CHECK(ctx);
    ref_bad.assign(N + 1, 0);
    PTB_CUDA_CHECK(cudaMemcpyAsync(ref_bad.data(), rf, (N + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, st()));
    PTB_CUDA_CHECK(cudaStreamSynchronize(st()));
  }

  const double* s_u0 = nullptr;
  const double* s_v0 = nullptr;

  // serial_coarse_init (parareal.cpp:147-159) into cur
  void serial_coarse_init() {
    copy(CU(0), s_u0, nf);
    copy(CV(0), s_v0, nf);
    int32_t* f = fl(flags_w);
    for (size_t n = 1; n <= N; ++n) {
      coarse_stage(CU(n - 1), CV(n - 1), wcu(), wcv(), f + n);
      interpolate_fields(tr, 1, wcu(), CU(n));
      interpolate_fields(tr, 1, wcv(), CV(n));
      k_nan_where<<<blocks(ctx, nf), 256, 0, st()>>>(nf, 1, f + n, CU(n), CV(n));
      PTB_LAUNCH_CHECK(ctx);
    }
  }
  double* wcu() { return static_cast<double*>(wc_u.ptr); }
  double* wcv() { return static_cast<double*>(wc_v.ptr); }

  // finalize_iteration (parareal.cpp:107-128) on states (su, sv); previous may be null
  void finalize(double* su, double* sv, double* pu, double* pv, double* ee, double* l2, int* diverged,
                double* states_out) {
    int32_t* sf = fl(flags_s);
    PTB_CUDA_CHECK(cudaMemsetAsync(sf, 0, (N + 1) * sizeof(int32_t), st()));
    k_state_flags<<<dim3(std::min(64u, blocks(ctx, nf)), unsigned(N + 1)), 256, 0, st()>>>(nf, N + 1, su, sv, nf, sf);
    PTB_LAUNCH_CHECK(ctx);
    double* sm = static_cast<double*>(sums.ptr);
    pair_energy_sums(ew, fg, s.metric_scheme, N, su + nf, sv + nf, nf, RU(1), RV(1), nf, ptb_propagator_speed(pf),
                     sm + 4);
    std::vector<int32_t> bad(N + 1);
    std::vector<double> h(4 * (N + 1));
    PTB_CUDA_CHECK(cudaMemcpyAsync(bad.data(), sf, (N + 1) * sizeof(int32_t), cudaMemcpyDeviceToHost, st()));
    PTB_CUDA_CHECK(cudaMemcpyAsync(h.data() + 4, sm + 4, 4 * N * sizeof(double), cudaMemcpyDeviceToHost, st()));
    PTB_CUDA_CHECK(cudaStreamSynchronize(st()));
    const double vol = [&] {
      double v = 1.0;
      for (int a = 0; a < fg.dim; ++a) v *= fg.h[a];
      return v;
    }();
    bool dv = false;
    for (size_t n = 0; n <= N; ++n) {
      double e = 0.0, l = 0.0;
      if (n > 0) {  // measure (parareal.cpp:80-103)
        if (bad[n] || ref_bad[n]) {
          e = l = kInf;
        } else {
          const double sd = h[4 * n], sr = h[4 * n + 1], ld = h[4 * n + 2], lr = h[4 * n + 3];
          const double e_ref = 0.5 * sr * vol, e_diff = 0.5 * sd * vol;
          e = (e_ref == 0.0) ? (e_diff == 0.0 ? 0.0 : kInf) : std::sqrt(e_diff / e_ref);
          l = (lr == 0.0) ? (ld == 0.0 ? 0.0 : kInf) : std::sqrt(ld / lr);
        }
      }
      ee[n] = e;
      l2[n] = l;
      if (bad[n]) {
        dv = true;
        if (pu) {
          copy(su + n * nf, pu + n * nf, nf);
          copy(sv + n * nf, pv + n * nf, nf);
        }
      }
    }
    *diverged = dv ? 1 : 0;
    if (states_out) {
      for (size_t n = 0; n <= N; ++n) {
        PTB_CUDA_CHECK(cudaMemcpyAsync(states_out + (2 * n) * nf, su + n * nf, nf * sizeof(double),
                                       cudaMemcpyDeviceToHost, st()));
        PTB_CUDA_CHECK(cudaMemcpyAsync(states_out + (2 * n + 1) * nf, sv + n * nf, nf * sizeof(double),
                                       cudaMemcpyDeviceToHost, st()));
      }
      PTB_CUDA_CHECK(cudaStreamSynchronize(st()));
    }
  }

  // parallel stage: fine_next[n] = F(cur[n-1]), coarse_next[n] = C(R(cur[n-1])), n = 1..N
  void parallel_stage() {
    copy(FU(1), CU(0), N * nf);
    copy(FV(1), CV(0), N * nf);
    PTB_CUDA_CHECK(cudaMemsetAsync(fl(flags_f), 0, N * sizeof(int32_t), st()));
    PTB_CUDA_CHECK(cudaMemsetAsync(fl(flags_c), 0, N * sizeof(int32_t), st()));
    propagate(pf, pf->steps, N, FU(1), FV(1), fl(flags_f), s.mode);
    k_nan_where<<<blocks(ctx, N * nf), 256, 0, st()>>>(nf, N, fl(flags_f), FU(1), FV(1));
    PTB_LAUNCH_CHECK(ctx);
    restrict_fields(tr, N, CU(0), KU(1));
    restrict_fields(tr, N, CV(0), KV(1));
    propagate(pc, pc->steps, N, KU(1), KV(1), fl(flags_c), s.mode);
    k_nan_where<<<blocks(ctx, N * nc), 256, 0, st()>>>(nc, N, fl(flags_c), KU(1), KV(1));
    PTB_LAUNCH_CHECK(ctx);
  }

  void run(const double* u0h, const double* v0h, double* ee, double* l2, double* residual, int* rank, int* diverged,
           double* states, double* reference) {
    // upload the initial state into nxt[0] as staging
    PTB_CUDA_CHECK(cudaMemcpyAsync(NU(0), u0h, nf * sizeof(double), cudaMemcpyHostToDevice, st()));
    PTB_CUDA_CHECK(cudaMemcpyAsync(NV(0), v0h, nf * sizeof(double), cudaMemcpyHostToDevice, st()));
    // keep a pristine copy of init in the reference slot 0 (serial_reference copies from s_u0)
    double* init_u = dalloc<double>(tmp_u, nf);
    double* init_v = dalloc<double>(tmp_v, nf);
    copy(init_u, NU(0), nf);
    copy(init_v, NV(0), nf);
    s_u0 = init_u;
    s_v0 = init_v;
    cudaEvent_t ev[6];
    for (auto& e : ev) PTB_CUDA_CHECK(cudaEventCreate(&e));
    auto elapsed = [&](cudaEvent_t a, cudaEvent_t b) {
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      return double(ms);
    };
    PTB_CUDA_CHECK(cudaEventRecord(ev[0], st()));
    serial_reference();
    PTB_CUDA_CHECK(cudaEventRecord(ev[1], st()));
    PTB_CUDA_CHECK(cudaEventSynchronize(ev[1]));
    if (times) times->reference_ms = elapsed(ev[0], ev[1]);
    if (reference) {
      for (size_t n = 0; n <= N; ++n) {
        PTB_CUDA_CHECK(cudaMemcpyAsync(reference + 2 * n * nf, RU(n), nf * sizeof(double), cudaMemcpyDeviceToHost, st()));
        PTB_CUDA_CHECK(
            cudaMemcpyAsync(reference + (2 * n + 1) * nf, RV(n), nf * sizeof(double), cudaMemcpyDeviceToHost, st()));
      }
    }
    serial_coarse_init();
    residual[0] = kNaN;
    rank[0] = 0;
    finalize(CU(0), CV(0), nullptr, nullptr, ee, l2, diverged, states);

    const bool theta = s.variant != 0;
    const bool omega_identity = s.variant == 3;
    const bool additive = s.variant != 2;
    const int d = cg.dim;
    const size_t rows = size_t(d + 1) * nc;
    double* Fp = dalloc<double>(Fm, rows * N);
    double* Gp = dalloc<double>(Gm, rows * N);
    int* idx_d = dalloc<int>(idx, N);
    DevCorrector applied_drop;
    for (int k = 1; k <= K; ++k) {
      PTB_CUDA_CHECK(cudaEventRecord(ev[0], st()));
      parallel_stage();
      PTB_CUDA_CHECK(cudaEventRecord(ev[1], st()));
      double res = kNaN;
      int rk = 0;
      const DevCorrector* applied = &corr;
      std::vector<int32_t> ffl(N), cfl(N);
      PTB_CUDA_CHECK(cudaMemcpyAsync(ffl.data(), fl(flags_f), N * sizeof(int32_t), cudaMemcpyDeviceToHost, st()));
      PTB_CUDA_CHECK(cudaMemcpyAsync(cfl.data(), fl(flags_c), N * sizeof(int32_t), cudaMemcpyDeviceToHost, st()));
      PTB_CUDA_CHECK(cudaStreamSynchronize(st()));
      if (theta) {
        std::vector<int> keep;
        for (size_t n = 1; n <= N; ++n)
          if (!ffl[n - 1] && !cfl[n - 1]) keep.push_back(int(n - 1));
        if (!keep.empty()) {
          const int cols = int(keep.size());
          PTB_CUDA_CHECK(cudaMemcpyAsync(idx_d, keep.data(), keep.size() * sizeof(int), cudaMemcpyHostToDevice, st()));
          // assemble_snapshots (procrustes.cpp:158-175): F = Lambda(R fine_next), G = Lambda(coarse_next)
          double* ru = dalloc<double>(cof_u, N * nc);
          double* rv = dalloc<double>(cof_v, N * nc);
          restrict_fields(tr, N, FU(1), ru);
          restrict_fields(tr, N, FV(1), rv);
          energy_components(ew, cg, s.scheme, size_t(cols), ru, rv, nc, idx_d, ptb_propagator_speed(pc), Fp, rows,
                            nullptr);
          energy_components(ew, cg, s.scheme, size_t(cols), KU(1), KV(1), nc, idx_d, ptb_propagator_speed(pc), Gp,
                            rows, nullptr);
          if (omega_identity) {
            const double fn2 = std::sqrt(frob2(Fp, rows * cols));
            if (fn2 > 0.0) {
              double* D = dalloc<double>(comp2, rows * cols);
              k_sub<<<blocks(ctx, rows * cols), 256, 0, st()>>>(rows * cols, Fp, Gp, D);
              PTB_LAUNCH_CHECK(ctx);
              res = std::sqrt(frob2(D, rows * cols)) / fn2;
            } else {
              res = 0.0;
            }
          } else {
            update_svd(pw, corr, Fp, Gp, int(rows), cols, s.tol);
            if (s.remove_leading > 0) {
              drop_leading(corr, size_t(s.remove_leading), applied_drop, ctx);
              applied = &applied_drop;
            }
            res = relative_residual(pw, *applied, Fp, Gp, int(rows), cols);
            rk = applied->rank;
          }
        } else if (!omega_identity) {
          drop_leading(corr, size_t(std::max(0, s.remove_leading)), applied_drop, ctx);
          applied = &applied_drop;
          rk = applied->rank;
        }
      }
      PTB_CUDA_CHECK(cudaEventRecord(ev[2], st()));
      if (theta)
        theta_sweep(*applied, additive, omega_identity);
      else
        plain_sweep();
      PTB_CUDA_CHECK(cudaEventRecord(ev[3], st()));
      residual[k] = res;
      rank[k] = rk;
      finalize(NU(0), NV(0), CU(0), CV(0), ee + size_t(k) * (N + 1), l2 + size_t(k) * (N + 1), diverged + k,
               states ? states + size_t(k) * (N + 1) * 2 * nf : nullptr);
      PTB_CUDA_CHECK(cudaEventRecord(ev[4], st()));
      PTB_CUDA_CHECK(cudaEventSynchronize(ev[4]));
      if (times && k <= PTB_MAX_TIMED_ITERS) {
        times->parallel_ms[k - 1] = elapsed(ev[0], ev[1]);
        times->procrustes_ms[k - 1] = elapsed(ev[1], ev[2]);
        times->sweep_ms[k - 1] = elapsed(ev[2], ev[3]);
        times->finalize_ms[k - 1] = elapsed(ev[3], ev[4]);
        times->iteration_ms[k - 1] = elapsed(ev[0], ev[4]);
      }
      std::swap(cur_u, nxt_u);
      std::swap(cur_v, nxt_v);
    }
    for (auto& e : ev) cudaEventDestroy(e);
  }

  double frob2(const double* p, size_t n) {
    double* d = dalloc<double>(mean2, 1);
    column_sumsq(ctx, int(n), 1, p, n, d);
    double h = 0;
    PTB_CUDA_CHECK(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, st()));
    PTB_CUDA_CHECK(cudaStreamSynchronize(st()));
    return h;
  }

  // corrected_coarse_state (parareal.cpp:245-253) for `batch` coarse states -> (ou, ov)
  void corrected(const DevCorrector& applied, bool omega_identity, size_t batch, const double* u, const double* v,
                 double* ou, double* ov) {
    const size_t rows = size_t(cg.dim + 1) * nc;
    double* cp = dalloc<double>(comp, rows * batch);
    double* mp = dalloc<double>(mean, batch);
    energy_components(ew, cg, s.scheme, batch, u, v, nc, nullptr, ptb_propagator_speed(pc), cp, rows, mp);
    const double* src = cp;
    if (!omega_identity) {
      double* c2 = dalloc<double>(comp2, rows * batch);
      apply_corrector(pw, applied, batch, cp, rows, c2, rows);
      src = c2;
    }
    from_energy_components(ew, cg, batch, src, rows, mp, ptb_propagator_speed(pc), ou, ov, nc);
  }

  // theta sweep (parareal.cpp:311-340), writes nxt
  void theta_sweep(const DevCorrector& applied, bool additive, bool omega_identity) {
    copy(NU(0), s_u0, nf);
    copy(NV(0), s_v0, nf);
    int32_t* wf = fl(flags_w);
    PTB_CUDA_CHECK(cudaMemsetAsync(wf, 0, (N + 1) * sizeof(int32_t), st()));
    double* ou = dalloc<double>(cold_u, N * nc);
    double* ov = dalloc<double>(cold_v, N * nc);
    if (additive && N >= 2) corrected(applied, omega_identity, N - 1, KU(2), KV(2), ou + nc, ov + nc);
    double* du = dalloc<double>(cnew_u, nc);
    double* dv = dalloc<double>(cnew_v, nc);
    double* iu = dalloc<double>(fine_tmp_u, nf);
    double* iv = dalloc<double>(fine_tmp_v, nf);
    for (size_t n = 1; n <= N; ++n) {
      if (additive && n == 1) {  // the two theta terms cancel exactly at the first coupling
        copy(NU(1), FU(1), nf);
        copy(NV(1), FV(1), nf);
        continue;
      }
      coarse_stage(NU(n - 1), NV(n - 1), wcu(), wcv(), wf + n);
      corrected(applied, omega_identity, 1, wcu(), wcv(), du, dv);
      if (additive) {
        const double* cou = ou + (n - 1) * nc;
        const double* cov = ov + (n - 1) * nc;
        k_sub<<<blocks(ctx, nc), 256, 0, st()>>>(nc, du, cou, du);
        k_sub<<<blocks(ctx, nc), 256, 0, st()>>>(nc, dv, cov, dv);
        PTB_LAUNCH_CHECK(ctx);
        interpolate_fields(tr, 1, du, iu);
        interpolate_fields(tr, 1, dv, iv);
        k_combine_theta<<<blocks(ctx, nf), 256, 0, st()>>>(nf, wf + n, fl(flags_c) + (n - 1), fl(flags_f) + (n - 1),
                                                            FU(n), FV(n), iu, iv, NU(n), NV(n));
        PTB_LAUNCH_CHECK(ctx);
      } else {
        interpolate_fields(tr, 1, du, NU(n));
        interpolate_fields(tr, 1, dv, NV(n));
        k_nan_if<<<blocks(ctx, nf), 256, 0, st()>>>(nf, wf + n, NU(n), NV(n));
        PTB_LAUNCH_CHECK(ctx);
      }
    }
  }

  // plain sweep (parareal.cpp:222-231), writes nxt
  void plain_sweep() {
    copy(NU(0), s_u0, nf);
    copy(NV(0), s_v0, nf);
    int32_t* wf = fl(flags_w);
    PTB_CUDA_CHECK(cudaMemsetAsync(wf, 0, (N + 1) * sizeof(int32_t), st()));
    // coarse_next on the fine grid: I(C R cur[n-1]) or NaN (parareal.cpp:218-220)
    double* cfu = dalloc<double>(cof_u, N * nf);
    double* cfv = dalloc<double>(cof_v, N * nf);
    interpolate_fields(tr, N, KU(1), cfu);
    interpolate_fields(tr, N, KV(1), cfv);
    k_nan_where<<<blocks(ctx, N * nf), 256, 0, st()>>>(nf, N, fl(flags_c), cfu, cfv);
    PTB_LAUNCH_CHECK(ctx);
    double* iu = dalloc<double>(fine_tmp_u, nf);
    double* iv = dalloc<double>(fine_tmp_v, nf);
    for (size_t n = 1; n <= N; ++n) {
      coarse_stage(NU(n - 1), NV(n - 1), wcu(), wcv(), wf + n);
      interpolate_fields(tr, 1, wcu(), iu);
      interpolate_fields(tr, 1, wcv(), iv);
      k_combine_plain<<<blocks(ctx, nf), 256, 0, st()>>>(nf, wf + n, iu, iv, FU(n), FV(n), cfu + (n - 1) * nf,
                                                          cfv + (n - 1) * nf, NU(n), NV(n));
      PTB_LAUNCH_CHECK(ctx);
    }
  }
};

void run_parareal(ptb_context* ctx, const ptb_run_spec& spec, const double* cf, const double* cc, const double* u0,
                  const double* v0, double* ee, double* l2, double* residual, int* rank, int* diverged, double* states,
                  double* reference, ptb_phase_times* times) {
  std::lock_guard<std::recursive_mutex> lock(ctx->mutex);
  Driver d(ctx, spec);
  d.times = times;
  d.setup(cf, cc);
  d.run(u0, v0, ee, l2, residual, rank, diverged, states, reference);
}

}  // namespace ptb
