// Run-time compiled tapes (jit.cu).
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "errnorm_kernel.cuh"

namespace tsb {

// A tape as straight-line device code: double name(double x0, double x1, double y0, double y1).
std::string tape_function(const ts_tape& t, const std::string& name);
// error_norms' block kernel with the 12 tapes compiled in; false (nothing launched) when
// NVRTC is unavailable, TS_JIT=0, or compilation failed — the caller runs the interpreter.
bool launch_error_norms_jit(const ErrNormArgs& a, const ts_tape* tapes, double* partials, cudaStream_t s);
// "compiled" / "interpreter (why)" for the last error_norms call, with counters.
std::string jit_status();

}  // namespace tsb
