// error_norms on the device (mms.cu).
#pragma once

#include <cuda_runtime.h>

#include "errnorm_kernel.cuh"

namespace tsb {

size_t error_norms_smem(const GridG& micro);
// blocks = false: the per-cell partials are already there (jit.cu ran the compiled kernel)
void launch_error_norms(const ErrNormArgs& a, double* partials, double* out, cudaStream_t s, bool blocks = true);

}  // namespace tsb
