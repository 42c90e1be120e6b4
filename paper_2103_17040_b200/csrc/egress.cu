// Pushforward and byte-order kernels of the micro-state egress (egress.h).
// Compiled with -fmad=false: point coordinates round like the reference's
// x.x + scale * y.x (vtk.cpp:66) on its x86-64 build.
#include "egress.h"

namespace tsb {

namespace {

constexpr int kThreads = 256;

__device__ __constant__ int kPK[8] = {1, 1, 2, 2, 1, 3, 2, 3};
__device__ __constant__ int kPL[8] = {1, 2, 1, 2, 3, 1, 3, 2};

__device__ __forceinline__ double bswap_d(double v) {
    const unsigned long long u = (unsigned long long)__double_as_longlong(v);
    const unsigned lo = (unsigned)u, hi = (unsigned)(u >> 32);
    const unsigned long long r =
        ((unsigned long long)__byte_perm(lo, 0, 0x0123) << 32) | (unsigned long long)__byte_perm(hi, 0, 0x0123);
    return __longlong_as_double((long long)r);
}

// zeta(x_node, yhat) for every map family (mapping.hpp CompiledDiffeo::map and the
// tabulated extensions of include/twoscale_b200.h).
__device__ void push_zeta(const PushG& g, int node, double x0, double x1, const double* y, double* z,
                          unsigned* err) {
    if (g.kind == TS_MAP_TAPE) {
        z[0] = tape_eval(g.op, g.arg, g.val, g.zeta[0], x0, x1, y[0], y[1], err);
        z[1] = tape_eval(g.op, g.arg, g.val, g.zeta[1], x0, x1, y[0], y[1], err);
        z[2] = 0.0;
        return;
    }
    const double* T = g.table + (size_t)node * g.tstride;
    if (g.kind == TS_MAP_AFFINE_BUBBLE_TABLE) {
        const int d = g.dim;
        double beta = d == 2 ? 16.0 : 64.0;
        for (int k = 0; k < d; ++k) beta *= y[k] * (1.0 - y[k]);
        const double ab = g.amp * s_of_x(g.s_kind, x0, x1) * beta;
        for (int a = 0; a < d; ++a) {
            double v = 0.0;
            for (int b = 0; b < d; ++b) v += T[a * d + b] * y[b];
            z[a] = v + ab;
        }
        if (d == 2) z[2] = 0.0;
        return;
    }
    const double pi = 3.141592653589793;  // FOURIER_TABLE
    for (int a = 0; a < 2; ++a) {
        double v = y[a];
        for (int m = 0; m < 8; ++m) v += T[a * 8 + m] * sin(pi * kPK[m] * y[0]) * sin(pi * kPL[m] * y[1]);
        z[a] = v;
    }
    z[2] = 0.0;
}

__global__ void __launch_bounds__(kThreads) k_vtk_points(const PushG g, int first_node, long long npts,
                                                         int big_endian, double* __restrict__ out,
                                                         unsigned* err) {
    const long long np = (long long)g.nn[0] * g.nn[1] * g.nn[2];
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < npts;
         k += (long long)gridDim.x * blockDim.x) {
        const int node = first_node + (int)(k / np);
        const int j = (int)(k % np);
        const int i0 = j % g.nn[0], i1 = (j / g.nn[0]) % g.nn[1], i2 = j / (g.nn[0] * g.nn[1]);
        double y[3] = {TS_ADD(g.lo[0], TS_MUL((double)i0, g.hp[0])), TS_ADD(g.lo[1], TS_MUL((double)i1, g.hp[1])),
                       TS_ADD(g.lo[2], TS_MUL((double)i2, g.hp[2]))};
        double x0, x1;
        node_xy(g.macro, node, x0, x1);
        double z[3];
        push_zeta(g, node, x0, x1, y, z, err);
        const double p0 = TS_ADD(x0, TS_MUL(g.scale, z[0]));
        const double p1 = TS_ADD(x1, TS_MUL(g.scale, z[1]));
        const double p2 = TS_MUL(g.scale, z[2]);
        if (big_endian) {
            out[3 * k] = bswap_d(p0);
            out[3 * k + 1] = bswap_d(p1);
            out[3 * k + 2] = bswap_d(g.dim == 3 ? p2 : 0.0);
        } else if (g.dim == 3) {
            out[3 * k] = p0;
            out[3 * k + 1] = p1;
            out[3 * k + 2] = p2;
        } else {
            out[2 * k] = p0;
            out[2 * k + 1] = p1;
        }
    }
}

__global__ void __launch_bounds__(kThreads) k_vtk_swap(const double* __restrict__ in, long long n,
                                                       double* __restrict__ out) {
    for (long long k = blockIdx.x * (long long)blockDim.x + threadIdx.x; k < n; k += (long long)gridDim.x * blockDim.x)
        out[k] = bswap_d(in[k]);
}

int blocks_for(long long n) {
    long long b = (n + kThreads - 1) / kThreads;
    if (b > 148LL * 16) b = 148LL * 16;
    return (int)(b < 1 ? 1 : b);
}

}  // namespace

void launch_vtk_points(const PushG& g, int first_node, int n_nodes, int big_endian, double* out, unsigned* err,
                       cudaStream_t s) {
    const long long npts = (long long)n_nodes * g.nn[0] * g.nn[1] * g.nn[2];
    k_vtk_points<<<blocks_for(npts), kThreads, 0, s>>>(g, first_node, npts, big_endian, out, err);
}

void launch_vtk_swap(const double* in, size_t n, double* out, cudaStream_t s) {
    k_vtk_swap<<<blocks_for((long long)n), kThreads, 0, s>>>(in, (long long)n, out);
}

}  // namespace tsb
