// error_norms (mms.cpp:247-377) as a batched device reduction:
// one block per macro cell; per macro Gauss-3 point the block combines the four
// nodal micro solutions through the macro basis into SMEM (value and both macro
// gradients, 3 x n_micro doubles), then every thread integrates its share of the
// micro cells x Gauss-3 points against the manufactured solution (device tapes).
// Per-cell partials are summed in a fixed order by a second single-block kernel,
// so the result is deterministic (the reference also reduces per-cell partials
// serially, mms.cpp:362-370).
#include <cmath>

#include "mms.h"

namespace tsb {

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block sum of 6 values into out (thread 0 only valid); red has >= 32*6 doubles.
__device__ void block_sum6(double (&v)[6], double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int k = 0; k < 6; ++k) v[k] = warp_sum(v[k]);
    if (lane == 0)
        for (int k = 0; k < 6; ++k) red[warp * 6 + k] = v[k];
    __syncthreads();
    if (warp == 0)
        for (int k = 0; k < 6; ++k) v[k] = warp_sum(lane < nw ? red[lane * 6 + k] : 0.0);
    __syncthreads();
}

__global__ void __launch_bounds__(256) k_error_norms(const ErrNormArgs a, double* partials) {
    extern __shared__ double sm[];
    const GridG& M = a.macro;
    const GridG& g = a.micro;
    const int nm = g.nodes();
    double* vc = sm;
    double* vgx = vc + nm;
    double* vgy = vgx + nm;
    double* red = vgy + nm;
    const int cM = blockIdx.x;
    const int ci = cM % M.n0, cj = cM / M.n0;
    const int nx = M.n0 + 1;
    const int nodesM[4] = {cj * nx + ci, cj * nx + ci + 1, (cj + 1) * nx + ci + 1, (cj + 1) * nx + ci};
    const double detM = 0.25 * M.h0 * M.h1, detm = 0.25 * g.h0 * g.h1;
    const double Mgx = 2.0 / M.h0, Mgy = 2.0 / M.h1, mgx = 2.0 / g.h0, mgy = 2.0 / g.h1;
    const int* op = a.op;
    const int* arg = a.arg;
    const double* val = a.val;
    double acc[6] = {0, 0, 0, 0, 0, 0};  // eu2, egu2, ew2, egw2, ev2, evg2
    for (int qM = 0; qM < 9; ++qM) {
        double x0, x1;
        cell_pt(M, cM, a.S[qM], a.T[qM], x0, x1);
        const double wM = a.W[qM] * detM;
        if (threadIdx.x == 0) {  // macro errors (mms.cpp:307-325)
            double uh = 0, wh = 0, gux = 0, guy = 0, gwx = 0, gwy = 0;
            for (int k = 0; k < 4; ++k) {
                const double cu = a.u[nodesM[k]], cw = a.w[nodesM[k]];
                uh += a.N[qM][k] * cu;
                wh += a.N[qM][k] * cw;
                gux += a.dN[qM][k][0] * Mgx * cu;
                guy += a.dN[qM][k][1] * Mgy * cu;
                gwx += a.dN[qM][k][0] * Mgx * cw;
                gwy += a.dN[qM][k][1] * Mgy * cw;
            }
            const double du = tape_eval(op, arg, val, a.t[0], x0, x1, 0, 0, nullptr) - uh;
            const double dw = tape_eval(op, arg, val, a.t[1], x0, x1, 0, 0, nullptr) - wh;
            const double dux = tape_eval(op, arg, val, a.t[2], x0, x1, 0, 0, nullptr) - gux;
            const double duy = tape_eval(op, arg, val, a.t[3], x0, x1, 0, 0, nullptr) - guy;
            const double dwx = tape_eval(op, arg, val, a.t[4], x0, x1, 0, 0, nullptr) - gwx;
            const double dwy = tape_eval(op, arg, val, a.t[5], x0, x1, 0, 0, nullptr) - gwy;
            acc[0] += wM * du * du;
            acc[2] += wM * dw * dw;
            acc[1] += wM * (dux * dux + duy * duy);
            acc[3] += wM * (dwx * dwx + dwy * dwy);
        }
        // micro field through the macro basis at this point (mms.cpp:327-340)
        const double* V0 = a.V + (size_t)nodesM[0] * nm;
        const double* V1 = a.V + (size_t)nodesM[1] * nm;
        const double* V2 = a.V + (size_t)nodesM[2] * nm;
        const double* V3 = a.V + (size_t)nodesM[3] * nm;
        for (int j = threadIdx.x; j < nm; j += blockDim.x) {
            const double v[4] = {V0[j], V1[j], V2[j], V3[j]};
            double c = 0, gx = 0, gy = 0;
            for (int k = 0; k < 4; ++k) {
                c += a.N[qM][k] * v[k];
                gx += a.dN[qM][k][0] * Mgx * v[k];
                gy += a.dN[qM][k][1] * Mgy * v[k];
            }
            vc[j] = c;
            vgx[j] = gx;
            vgy[j] = gy;
        }
        __syncthreads();
        const int total = g.cells() * 9;
        for (int idx = threadIdx.x; idx < total; idx += blockDim.x) {
            const int cm = idx / 9, qm = idx % 9;
            const int mi = cm % g.n0, mj = cm / g.n0, mnx = g.n0 + 1;
            const int nd[4] = {mj * mnx + mi, mj * mnx + mi + 1, (mj + 1) * mnx + mi + 1, (mj + 1) * mnx + mi};
            double y0, y1;
            cell_pt(g, cm, a.S[qm], a.T[qm], y0, y1);
            const double wq = wM * a.W[qm] * detm;
            double vh = 0, vhx = 0, vhy = 0, vh0 = 0, vh1 = 0;
            for (int b = 0; b < 4; ++b) {
                const int j = nd[b];
                vh += a.N[qm][b] * vc[j];
                vhx += a.N[qm][b] * vgx[j];
                vhy += a.N[qm][b] * vgy[j];
                vh0 += a.dN[qm][b][0] * mgx * vc[j];
                vh1 += a.dN[qm][b][1] * mgy * vc[j];
            }
            const double J = tape_eval(op, arg, val, a.t[11], x0, x1, y0, y1, nullptr);
            const double D = tape_eval(op, arg, val, a.t[6], x0, x1, y0, y1, nullptr) - vh;
            const double Dx0 = tape_eval(op, arg, val, a.t[7], x0, x1, y0, y1, nullptr) - vhx;
            const double Dx1 = tape_eval(op, arg, val, a.t[8], x0, x1, y0, y1, nullptr) - vhy;
            const double Dy0 = tape_eval(op, arg, val, a.t[9], x0, x1, y0, y1, nullptr) - vh0;
            const double Dy1 = tape_eval(op, arg, val, a.t[10], x0, x1, y0, y1, nullptr) - vh1;
            acc[4] += wq * D * D * J;
            acc[5] += wq * (D * D + Dx0 * Dx0 + Dx1 * Dx1 + Dy0 * Dy0 + Dy1 * Dy1) * J;
        }
        __syncthreads();
    }
    block_sum6(acc, red);
    if (threadIdx.x == 0)
        for (int k = 0; k < 6; ++k) partials[(size_t)cM * 6 + k] = acc[k];
}

__global__ void k_error_norms_final(int ncells, const double* partials, double* out) {
    __shared__ double red[32 * 6];
    double acc[6] = {0, 0, 0, 0, 0, 0};
    for (int c = threadIdx.x; c < ncells; c += blockDim.x)
        for (int k = 0; k < 6; ++k) acc[k] += partials[(size_t)c * 6 + k];
    block_sum6(acc, red);
    if (threadIdx.x == 0) {  // mms.cpp:371-376
        out[0] = sqrt(acc[0]) + sqrt(acc[2]);
        out[1] = sqrt(acc[0] + acc[1]) + sqrt(acc[2] + acc[3]);
        out[2] = sqrt(acc[4]);
        out[3] = sqrt(acc[5]);
    }
}

}  // namespace

size_t error_norms_smem(const GridG& micro) { return (3 * (size_t)micro.nodes() + 32 * 6) * sizeof(double); }

void launch_error_norms(const ErrNormArgs& a, double* partials, double* out, cudaStream_t s) {
    const size_t smem = error_norms_smem(a.micro);
    cudaFuncSetAttribute(k_error_norms, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_error_norms<<<a.macro.cells(), 256, smem, s>>>(a, partials);
    k_error_norms_final<<<1, 1024, 0, s>>>(a.macro.cells(), partials, out);
}

}  // namespace tsb
