// error_norms on the device (mms.cu).
#pragma once

#include <cuda_runtime.h>

#include "device_common.cuh"

namespace tsb {

// Tapes: 0 u, 1 w, 2 u_x0, 3 u_x1, 4 w_x0, 5 w_x1, 6 v_hat, 7 v_hat_x0, 8 v_hat_x1,
// 9 v_hat_y0, 10 v_hat_y1, 11 det grad_y zeta (mms.cpp:250-266).
struct ErrNormArgs {
    GridG macro, micro;
    const int* op;
    const int* arg;
    const double* val;
    TapeRef t[12];
    const double* u;
    const double* w;
    const double* V;
    double S[9], T[9], W[9];   // Gauss-3 cell rule (grid.cpp:142-147), i fastest
    double N[9][4], dN[9][4][2];
};

size_t error_norms_smem(const GridG& micro);
void launch_error_norms(const ErrNormArgs& a, double* partials, double* out, cudaStream_t s);

}  // namespace tsb
