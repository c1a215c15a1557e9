#pragma once
#include "ptb_comm.h"
#include "ptb_internal.h"

namespace ptb {

void run_parareal(ptb_context* ctx, const Comm* comm, const ptb_run_spec& spec, const double* cf, const double* cc,
                  const double* u0, const double* v0, double* ee, double* l2, double* residual, int* rank,
                  int* diverged, double* states, double* reference, ptb_phase_times* times);

}  // namespace ptb
