// error_norms (mms.cpp:247-377), the per-macro-cell block body shared by the statically
// compiled kernel (tapes interpreted, mms.cu) and the run-time compiled one (tapes as
// straight-line code, jit.cu).  Plain device code, so NVRTC compiles it unchanged.
//
// One block per macro cell; per macro Gauss-3 point the block combines the four nodal
// micro solutions through the macro basis into SMEM (value and both macro gradients,
// 3 x n_micro doubles), then every thread integrates its share of the micro cells x
// Gauss-3 points against the manufactured solution.  Per-cell partials are summed in a
// fixed order by a second kernel (the reference also reduces per-cell partials serially,
// mms.cpp:362-370).
#pragma once

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

__device__ __forceinline__ double en_warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block sum of 6 values (thread 0's result valid); red has >= 32*6 doubles.
__device__ __forceinline__ void en_block_sum6(double (&v)[6], double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int k = 0; k < 6; ++k) v[k] = en_warp_sum(v[k]);
    if (lane == 0)
        for (int k = 0; k < 6; ++k) red[warp * 6 + k] = v[k];
    __syncthreads();
    if (warp == 0)
        for (int k = 0; k < 6; ++k) v[k] = en_warp_sum(lane < nw ? red[lane * 6 + k] : 0.0);
    __syncthreads();
}

// tape(k, x0, x1, y0, y1): the value of tape k (the table above).
template <class TE>
__device__ __forceinline__ void error_norms_block(const ErrNormArgs& a, double* partials, double* sm, const TE& tape) {
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
            const double du = tape(0, x0, x1, 0, 0) - uh;
            const double dw = tape(1, x0, x1, 0, 0) - wh;
            const double dux = tape(2, x0, x1, 0, 0) - gux;
            const double duy = tape(3, x0, x1, 0, 0) - guy;
            const double dwx = tape(4, x0, x1, 0, 0) - gwx;
            const double dwy = tape(5, x0, x1, 0, 0) - gwy;
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
            const double J = tape(11, x0, x1, y0, y1);
            const double D = tape(6, x0, x1, y0, y1) - vh;
            const double Dx0 = tape(7, x0, x1, y0, y1) - vhx;
            const double Dx1 = tape(8, x0, x1, y0, y1) - vhy;
            const double Dy0 = tape(9, x0, x1, y0, y1) - vh0;
            const double Dy1 = tape(10, x0, x1, y0, y1) - vh1;
            acc[4] += wq * D * D * J;
            acc[5] += wq * (D * D + Dx0 * Dx0 + Dx1 * Dx1 + Dy0 * Dy0 + Dy1 * Dy1) * J;
        }
        __syncthreads();
    }
    en_block_sum6(acc, red);
    if (threadIdx.x == 0)
        for (int k = 0; k < 6; ++k) partials[(size_t)cM * 6 + k] = acc[k];
}

}  // namespace tsb
