// error_norms (mms.cpp:247-377) as a batched device reduction.  The
// block body is errnorm_kernel.cuh; this file instantiates it with the tape interpreter
// (the run-time compiled variant with straight-line tapes is in jit.cu).
#include <cmath>

#include "mms.h"

namespace tsb {

namespace {

struct InterpTapes {
    const ErrNormArgs* a;
    __device__ __forceinline__ double operator()(int k, double x0, double x1, double y0, double y1) const {
        return tape_eval(a->op, a->arg, a->val, a->t[k], x0, x1, y0, y1, nullptr);
    }
};

__global__ void __launch_bounds__(256) k_error_norms(const ErrNormArgs a, double* partials) {
    extern __shared__ double sm[];
    error_norms_block(a, partials, sm, InterpTapes{&a});
}

__global__ void k_error_norms_final(int ncells, const double* partials, double* out) {
    __shared__ double red[32 * 6];
    double acc[6] = {0, 0, 0, 0, 0, 0};
    for (int c = threadIdx.x; c < ncells; c += blockDim.x)
        for (int k = 0; k < 6; ++k) acc[k] += partials[(size_t)c * 6 + k];
    en_block_sum6(acc, red);
    if (threadIdx.x == 0) {  // mms.cpp:371-376
        out[0] = sqrt(acc[0]) + sqrt(acc[2]);
        out[1] = sqrt(acc[0] + acc[1]) + sqrt(acc[2] + acc[3]);
        out[2] = sqrt(acc[4]);
        out[3] = sqrt(acc[5]);
    }
}

}  // namespace

size_t error_norms_smem(const GridG& micro) { return (3 * (size_t)micro.nodes() + 32 * 6) * sizeof(double); }

void launch_error_norms(const ErrNormArgs& a, double* partials, double* out, cudaStream_t s, bool blocks) {
    if (blocks) {
        const size_t smem = error_norms_smem(a.micro);
        cudaFuncSetAttribute(k_error_norms, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_error_norms<<<a.macro.cells(), 256, smem, s>>>(a, partials);
    }
    k_error_norms_final<<<1, 1024, 0, s>>>(a.macro.cells(), partials, out);
}

}  // namespace tsb
