#pragma once
#include "ptb_comm.h"
#include "ptb_internal.h"

namespace ptb {

struct ProcWork;
// the context's cached Procrustes workspace (shared with the driver; callers hold ctx->mutex)
ProcWork& context_proc_work(ptb_context* ctx);
struct EnergyWork;
// the context's cached energy-map workspace (C ABI calls; callers hold ctx->mutex)
EnergyWork& context_energy_work(ptb_context* ctx);

void run_parareal(ptb_context* ctx, const Comm* comm, const ptb_run_spec& spec, const double* cf, const double* cc,
                  const double* u0, const double* v0, double* ee, double* l2, double* residual, int* rank,
                  int* diverged, double* states, double* reference, ptb_phase_times* times);

}  // namespace ptb
