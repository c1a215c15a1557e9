#pragma once
#include <cuda_runtime.h>

#include "ptb_internal.h"

namespace ptb {

// In-place batched DFT of `batch` complex fields on grid g (fft.cu).
void fft_field(ptb_context* ctx, cudaStream_t st, const ptb_grid& g, size_t batch, double2* data, bool inverse);

}  // namespace ptb
