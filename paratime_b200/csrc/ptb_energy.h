#pragma once
#include "ptb_internal.h"

namespace ptb {

// Scratch owned by whoever runs energy-map work (driver, C ABI calls).
struct EnergyWork {
  ptb_context* ctx = nullptr;
  DeviceBuffer buf[9];  // [8]: mean_u partials
  explicit EnergyWork(ptb_context* c) : ctx(c) {}
  ~EnergyWork();
};

// Lambda: `batch` states (u, v at state stride sstride, optional gather index) ->
// stacked columns (column b at stacked + b*ld) and mean_u[b] (nullable).
void energy_components(EnergyWork& w, const ptb_grid& g, int scheme, size_t batch, const double* u, const double* v,
                       size_t sstride, const int* index, const double* c, double* stacked, size_t ld, double* mean);

// Sweep step of the theta sweep (finite-difference schemes): z[j P + p] = partial p of
// Y[:, j]^T Lambda(w) (P = comp_gemv_parts(rows) chunks), mean_part[q] = partial q of sum(u)
// (sweep_mean_parts(n) partials, k_state_sum's) -- one launch, Lambda(w) never stored.
int comp_gemv_parts(size_t rows);
int sweep_mean_parts(int n);
void comp_gemv(EnergyWork& w, const ptb_grid& g, int scheme, const double* u, const double* v, const double* c,
               const double* Y, size_t ldy, int r, double* z, int P, double* mean_part);

// Lambda-dagger: stacked columns + mean_u -> states (u, v at stride sstride).
void from_energy_components(EnergyWork& w, const ptb_grid& g, size_t batch, const double* stacked, size_t ld,
                            const double* mean, const double* c, double* u, double* v, size_t sstride);

// Per state pair b: out4[4b..4b+3] = { |Lambda(a-b)|^2, |Lambda(b)|^2, |u_a-u_b|^2, |u_b|^2 }.
void pair_energy_sums(EnergyWork& w, const ptb_grid& g, int scheme, size_t batch, const double* ua, const double* va,
                      size_t sa, const double* ub, const double* vb, size_t sb, const double* c, double* out4,
                      int32_t* nonfinite_a = nullptr);  // optional: OR 1 into [b] if state a_b is non-finite

// out[j] = sum_i m[j*ld + i]^2, i < rows (deterministic).
void column_sumsq(ptb_context* ctx, int rows, size_t cols, const double* m, size_t ld, double* out);

}  // namespace ptb
