// Generic (Q2 / 3D micro) versions of kernels (1) and (2): map caches, micro
// operator assembly (node-centric gather in the reference's scatter order) and rhs
// parts, plus the macro quadrature-point integrals over the generic micro faces.
// Compiled with -fmad=false; arithmetic mirrors oracle/twoscale_oracle_gen.c
// operation by operation.
#include <algorithm>
#include <cstdlib>

#include "generic.h"

namespace tsb {

__constant__ GenTables cG;  // this translation unit only

void upload_gen_tables(const GenTables& t) { cudaMemcpyToSymbol(cG, &t, sizeof(GenTables)); }

namespace {

constexpr int kThreads = 256;

int grid_for(long long total) {
    long long b = (total + kThreads - 1) / kThreads;
    if (b > 148LL * 64) b = 148LL * 64;
    return (int)(b < 1 ? 1 : b);
}

__device__ __forceinline__ void table_row(const GenMap& m, int node, double x0, double x1, double* out) {
    const int ts = m.tstride;
    if (node >= 0) {
        for (int k = 0; k < ts; ++k) out[k] = m.table[(size_t)node * ts + k];
        return;
    }
    const GridG& g = m.macro;
    const double fx = (x0 - g.lo0) / g.h0, fy = (x1 - g.lo1) / g.h1;
    int ci = (int)floor(fx), cj = (int)floor(fy);
    ci = ci < 0 ? 0 : (ci > g.n0 - 1 ? g.n0 - 1 : ci);
    cj = cj < 0 ? 0 : (cj > g.n1 - 1 ? g.n1 - 1 : cj);
    const double s = fx - ci, t = fy - cj;
    const int nx = g.n0 + 1;
    const double* T00 = m.table + (size_t)(cj * nx + ci) * ts;
    const double* T10 = m.table + (size_t)(cj * nx + ci + 1) * ts;
    const double* T11 = m.table + (size_t)((cj + 1) * nx + ci + 1) * ts;
    const double* T01 = m.table + (size_t)((cj + 1) * nx + ci) * ts;
    for (int k = 0; k < ts; ++k)
        out[k] = (1.0 - s) * (1.0 - t) * T00[k] + s * (1.0 - t) * T10[k] + s * t * T11[k] + (1.0 - s) * t * T01[k];
}

__device__ __constant__ int kFK[8] = {1, 1, 2, 2, 1, 3, 2, 3};
__device__ __constant__ int kFL[8] = {1, 2, 1, 2, 3, 1, 3, 2};

__device__ __forceinline__ void gen_jac_row(const GenMap& m, int d, const double* T, double x0, double x1,
                                            const double* y, double* F);

__device__ void gen_jac(const GenMap& m, int d, int node, double x0, double x1, const double* y, double* F,
                        unsigned* err) {
    if (m.kind == TS_MAP_TAPE) {
        for (int k = 0; k < 4; ++k) F[k] = tape_eval(m.op, m.arg, m.val, m.jac[k], x0, x1, y[0], y[1], err);
        return;
    }
    double T[16];
    table_row(m, node, x0, x1, T);
    gen_jac_row(m, d, T, x0, x1, y, F);
}

// The Jacobian of a tabulated map from its (node or interpolated) table row T.
__device__ __forceinline__ void gen_jac_row(const GenMap& m, int d, const double* T, double x0, double x1,
                                            const double* y, double* F) {
    if (m.kind == TS_MAP_AFFINE_BUBBLE_TABLE) {
        const double as = m.amp * s_of_x(m.s_kind, x0, x1);
        const double cd = d == 2 ? 16.0 : 64.0;
        double gb[3];
        for (int k = 0; k < d; ++k) {
            double v = cd * (1.0 - 2.0 * y[k]);
            for (int l = 0; l < d; ++l)
                if (l != k) v *= y[l] * (1.0 - y[l]);
            gb[k] = v;
        }
        for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b) F[a * d + b] = T[a * d + b] + as * gb[b];
        return;
    }
    const double pi = 3.141592653589793;
    double s0[4], c0[4], s1[4], c1[4];
    for (int k = 1; k <= 3; ++k) {
        s0[k] = sin(pi * k * y[0]);
        c0[k] = cos(pi * k * y[0]);
        s1[k] = sin(pi * k * y[1]);
        c1[k] = cos(pi * k * y[1]);
    }
    for (int a = 0; a < 2; ++a) {
        double g0 = 0.0, g1 = 0.0;
        for (int mm = 0; mm < 8; ++mm) {
            const double cm = T[a * 8 + mm];
            g0 += cm * (pi * kFK[mm]) * c0[kFK[mm]] * s1[kFL[mm]];
            g1 += cm * (pi * kFL[mm]) * s0[kFK[mm]] * c1[kFL[mm]];
        }
        F[a * 2 + 0] = (a == 0 ? 1.0 : 0.0) + g0;
        F[a * 2 + 1] = (a == 1 ? 1.0 : 0.0) + g1;
    }
}

__device__ __forceinline__ double gen_cofactor(int d, const double* F, double* C) {
    if (d == 2) {
        C[0] = F[3];
        C[1] = -F[2];
        C[2] = -F[1];
        C[3] = F[0];
        return F[0] * F[3] - F[1] * F[2];
    }
#define f(i, j) F[(i) * 3 + (j)]
    C[0] = f(1, 1) * f(2, 2) - f(1, 2) * f(2, 1);
    C[1] = -(f(1, 0) * f(2, 2) - f(1, 2) * f(2, 0));
    C[2] = f(1, 0) * f(2, 1) - f(1, 1) * f(2, 0);
    C[3] = -(f(0, 1) * f(2, 2) - f(0, 2) * f(2, 1));
    C[4] = f(0, 0) * f(2, 2) - f(0, 2) * f(2, 0);
    C[5] = -(f(0, 0) * f(2, 1) - f(0, 1) * f(2, 0));
    C[6] = f(0, 1) * f(1, 2) - f(0, 2) * f(1, 1);
    C[7] = -(f(0, 0) * f(1, 2) - f(0, 2) * f(1, 0));
    C[8] = f(0, 0) * f(1, 1) - f(0, 1) * f(1, 0);
#undef f
    return F[0] * C[0] + F[1] * C[1] + F[2] * C[2];
}

// J then A = C^T D C / det (upper triangle, row-major); returns det > 1e-12.
__device__ bool gen_cell_entry(const GenMap& m, int d, int node, double x0, double x1, const double* y,
                               double* e, unsigned* err) {
    double F[9], C[9], DC[9];
    gen_jac(m, d, node, x0, x1, y, F, err);
    const double det = gen_cofactor(d, F, C);
    for (int k = 0; k < d; ++k)
        for (int b = 0; b < d; ++b) {
            double s = m.D[k * d + 0] * C[0 * d + b];
            for (int l = 1; l < d; ++l) s += m.D[k * d + l] * C[l * d + b];
            DC[k * d + b] = s;
        }
    e[0] = det;
    int idx = 1;
    const bool ident = d == 2 && m.D_identity;
    for (int a = 0; a < d; ++a)
        for (int b = a; b < d; ++b) {
            double s;
            if (ident) {
                s = C[0 * d + a] * C[0 * d + b] + C[1 * d + a] * C[1 * d + b];
            } else {
                s = C[0 * d + a] * DC[0 * d + b];
                for (int k = 1; k < d; ++k) s += C[k * d + a] * DC[k * d + b];
            }
            e[idx++] = s / det;
        }
    return det > 1e-12;
}

__device__ __forceinline__ bool gen_face_len(const GenMap& m, int d, int node, double x0, double x1, const double* y,
                             const double* nrm, double& len, double& det_out, unsigned* err,
                             const double* row = nullptr) {
    double F[9], C[9];
    if (row) gen_jac_row(m, d, row, x0, x1, y, F);
    else gen_jac(m, d, node, x0, x1, y, F, err);
    const double det = gen_cofactor(d, F, C);
    double s = 0.0;
    for (int i = 0; i < d; ++i) {
        double nu = C[i * d + 0] * nrm[0];
        for (int k = 1; k < d; ++k) nu += C[i * d + k] * nrm[k];
        s += nu * nu;
    }
    len = sqrt(s);
    det_out = det;
    return det > 1e-12;
}

__device__ __forceinline__ void row_x(const GenProblem& P, int row, const double* points, double& x0, double& x1,
                                      int& node, int row0 = 0) {
    if (points) {
        x0 = points[2 * row];
        x1 = points[2 * row + 1];
        node = -1;
    } else {
        node = row0 + row;
        node_xy(P.macro, node, x0, x1);
    }
}

__global__ void k_gcell_cache(GenProblem P, int rows, const double* points, double* out,
                              unsigned long long* first_bad, unsigned* err, int row0) {
    const GenGeom& g = P.g;
    const int nc = 1 + g.d * (g.d + 1) / 2;
    const long long total = (long long)rows * g.ncells * g.nq;
    const long long stride = (long long)g.ncells * g.nq + (long long)g.nfaces * g.nqf;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(t % g.ncells);  // planar layout, as k_gcell_cache_t
        const long long rq = t / g.ncells;
        const int q = (int)(rq % g.nq);
        const int row = (int)(rq / g.nq);
        double x0, x1, y[3];
        int node, cc[3];
        row_x(P, row, points, x0, x1, node, row0);
        gen_cell_idx(g, c, cc);
        gen_cell_qpoint(g, cG, cc, q, y);
        double e[7];
        if (!gen_cell_entry(P.map, g.d, node, x0, x1, y, e, err))
            atomicMin(first_bad, (unsigned long long)(row * stride + (long long)c * g.nq + q));
        for (int k = 0; k < nc; ++k) out[((size_t)rq * nc + k) * g.ncells + c] = e[k];
    }
}

// k_gcell_cache with the dimension at compile time (loops unrolled, arrays in registers);
// same operations in the same order as gen_cell_entry, so the same bits.
template <int D>
__global__ void __launch_bounds__(256) k_gcell_cache_t(GenProblem P, int rows, const double* points, double* out,
                                                       unsigned long long* first_bad, unsigned* err, int row0) {
    const GenGeom& g = P.g;
    constexpr int NC = 1 + D * (D + 1) / 2;
    const long long total = (long long)rows * g.ncells * g.nq;
    const long long stride = (long long)g.ncells * g.nq + (long long)g.nfaces * g.nqf;
    const GenMap& m = P.map;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
        // planar layout [row][q][k][cell] (generic.h): consecutive threads, consecutive cells
        const int c = (int)(t % g.ncells);
        const long long rq = t / g.ncells;
        const int q = (int)(rq % g.nq);
        const int row = (int)(rq / g.nq);
        double x0, x1, y[3];
        int node, cc[3];
        row_x(P, row, points, x0, x1, node, row0);
        gen_cell_idx(g, c, cc);
        gen_cell_qpoint(g, cG, cc, q, y);
        double F[D * D], C[D * D], DC[D * D];
        gen_jac(m, D, node, x0, x1, y, F, err);
        double det;
        if constexpr (D == 2) {
            C[0] = F[3];
            C[1] = -F[2];
            C[2] = -F[1];
            C[3] = F[0];
            det = F[0] * F[3] - F[1] * F[2];
        } else {
            det = gen_cofactor(3, F, C);
        }
#pragma unroll
        for (int k = 0; k < D; ++k)
#pragma unroll
            for (int b = 0; b < D; ++b) {
                double sum = m.D[k * D + 0] * C[0 * D + b];
#pragma unroll
                for (int l = 1; l < D; ++l) sum += m.D[k * D + l] * C[l * D + b];
                DC[k * D + b] = sum;
            }
        double e[NC];
        e[0] = det;
        int idx = 1;
        const bool ident = D == 2 && m.D_identity;
#pragma unroll
        for (int a = 0; a < D; ++a)
#pragma unroll
            for (int b = a; b < D; ++b) {
                double sum;
                if (ident) {
                    sum = C[0 * D + a] * C[0 * D + b] + C[1 * D + a] * C[1 * D + b];
                } else {
                    sum = C[0 * D + a] * DC[0 * D + b];
#pragma unroll
                    for (int k = 1; k < D; ++k) sum += C[k * D + a] * DC[k * D + b];
                }
                e[idx++] = sum / det;
            }
        if (!(det > 1e-12)) atomicMin(first_bad, (unsigned long long)(row * stride + (long long)c * g.nq + q));
        double* o = out + ((size_t)rq * NC) * g.ncells + c;
#pragma unroll
        for (int k = 0; k < NC; ++k) o[(size_t)k * g.ncells] = e[k];
    }
}

__global__ void k_gface_cache(GenProblem P, int rows, const double* points, int with_cells, double* out,
                              unsigned long long* first_bad, unsigned* err) {
    const GenGeom& g = P.g;
    const long long total = (long long)rows * g.nfaces * g.nqf;
    const long long cpart = with_cells ? (long long)g.ncells * g.nq : 0;
    const long long stride = cpart + (long long)g.nfaces * g.nqf;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
        const int q = (int)(t % g.nqf);
        const long long rf = t / g.nqf;
        const int f = (int)(rf % g.nfaces);
        const int row = (int)(rf / g.nfaces);
        double x0, x1, y[3], nrm[3], sc, len, det;
        int node, axis, side, cc[3], tr[2];
        row_x(P, row, points, x0, x1, node);
        gen_face(g, f, axis, side, cc, tr);
        gen_face_geom(g, cG, axis, side, cc, q, y, sc, nrm);
        if (!gen_face_len(P.map, g.d, node, x0, x1, y, nrm, len, det, err))
            atomicMin(first_bad, (unsigned long long)(row * stride + cpart + (long long)f * g.nqf + q));
        out[t] = len;
    }
}

__global__ void k_gprobe(GenProblem P, const double* points, int with_cells, unsigned long long index, double* out) {
    const GenGeom& g = P.g;
    const long long cpart = with_cells ? (long long)g.ncells * g.nq : 0;
    const long long stride = cpart + (long long)g.nfaces * g.nqf;
    const int row = (int)(index / stride);
    const long long r = index % stride;
    double x0, x1, y[3] = {0, 0, 0}, det = 0.0;
    int node;
    row_x(P, row, points, x0, x1, node);
    if (r < cpart) {
        int cc[3];
        gen_cell_idx(g, (int)(r / g.nq), cc);
        gen_cell_qpoint(g, cG, cc, (int)(r % g.nq), y);
        double e[7];
        gen_cell_entry(P.map, g.d, node, x0, x1, y, e, nullptr);
        det = e[0];
    } else {
        const int f = (int)((r - cpart) / g.nqf), q = (int)((r - cpart) % g.nqf);
        int axis, side, cc[3], tr[2];
        double nrm[3], sc, len;
        gen_face(g, f, axis, side, cc, tr);
        gen_face_geom(g, cG, axis, side, cc, q, y, sc, nrm);
        gen_face_len(P.map, g.d, node, x0, x1, y, nrm, len, det, nullptr);
    }
    out[0] = det;
    out[1] = x0;
    out[2] = x1;
    out[3] = y[0];
    out[4] = y[1];
    out[5] = y[2];
}

// cells along axis a whose closure contains lattice index i: [c0, c1]
__device__ __forceinline__ void cells_of(const GenGeom& g, int a, int i, int& c0, int& c1) {
    c0 = i > 0 ? (i - 1) / g.p : 0;
    c1 = i / g.p;
    if (c1 > g.nc[a] - 1) c1 = g.nc[a] - 1;
}

// Boundary faces containing lattice node ii, ascending face index, with the node's
// face-local index.  Returns the count (<= 12).
__device__ int gen_node_faces(const GenGeom& g, const int* ii, int* fl, int* pl) {
    int k = 0;
    const int q1 = g.p + 1;
    for (int a = 0; a < g.d; ++a) {
        for (int side = 0; side < 2; ++side) {
            if (ii[a] != (side ? g.nn[a] - 1 : 0)) continue;
            int tr[2], nt = 0;
            for (int t = 0; t < g.d; ++t)
                if (t != a) tr[nt++] = t;
            int a0, a1, b0 = 0, b1 = 0;
            cells_of(g, tr[0], ii[tr[0]], a0, a1);
            if (g.d == 3) cells_of(g, tr[1], ii[tr[1]], b0, b1);
            for (int cb = b0; cb <= b1; ++cb)
                for (int ca = a0; ca <= a1; ++ca) {
                    const int tlin = ca + (g.d == 3 ? g.nc[tr[0]] * cb : 0);
                    fl[k] = g.face_off[a] + 2 * tlin + side;
                    pl[k] = (ii[tr[0]] - g.p * ca) + (g.d == 3 ? q1 * (ii[tr[1]] - g.p * cb) : 0);
                    ++k;
                }
        }
    }
    for (int x = 1; x < k; ++x)
        for (int y = x; y > 0 && fl[y] < fl[y - 1]; --y) {
            int t = fl[y]; fl[y] = fl[y - 1]; fl[y - 1] = t;
            t = pl[y]; pl[y] = pl[y - 1]; pl[y - 1] = t;
        }
    return k;
}

__device__ __forceinline__ double reaction_k(const GenProblem& P, const double* y) {
    if (P.reaction_kind == TS_REACTION_DISC) {
        double s = 0.0;
        for (int k = 0; k < P.g.d; ++k) {
            const double t = y[k] - P.reaction_c[k];
            s += t * t;
        }
        return sqrt(s) < P.reaction_r ? P.reaction_in : P.reaction_out;
    }
    return P.reaction_in;
}

// build_micro_matrices (generalised) as a gather: thread = (system, node).
__global__ void k_gassemble(GenProblem P, int srows, const double* __restrict__ cells,
                            const double* __restrict__ faces, double* __restrict__ stencil) {
    const GenGeom& g = P.g;
    const int d = g.d, p = g.p, q1 = p + 1, nc = 1 + d * (d + 1) / 2;
    const int n = g.nnodes, span = 2 * p + 1;
    const long long total = (long long)srows * n;
    const double det_elem = d == 2 ? 0.25 * g.h[0] * g.h[1] : 0.125 * g.h[0] * g.h[1] * g.h[2];
    double gs[3];
    for (int k = 0; k < d; ++k) gs[k] = 2.0 / g.h[k];
    const bool react = !(P.reaction_kind == TS_REACTION_CONST && P.reaction_in == 0.0);
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
        const int node = (int)(t % n);
        const int sys = (int)(t / n);
        int ii[3];
        gen_node_idx(g, node, ii);
        double acc[kGenMaxDirs];
        for (int k = 0; k < g.ndirs; ++k) acc[k] = 0.0;
        const double* crow = cells + (size_t)sys * g.ncells * g.nq * nc;
        const double* frow = faces + (size_t)sys * g.nfaces * g.nqf;
        auto add_faces = [&]() {
            int fl[12], pl[12];
            const int nf = gen_node_faces(g, ii, fl, pl);
            for (int k = 0; k < nf; ++k) {
                int axis, side, cc[3], tr[2];
                gen_face(g, fl[k], axis, side, cc, tr);
                const int role = P.role[2 * axis + side];
                if (role == TS_GAMMA_N) continue;
                const double kappa = role == TS_GAMMA_I ? P.kappa[1] : P.kappa[3];
                if (kappa == 0.0) continue;
                double y[3], sc, nrm[3];
                gen_face_geom(g, cG, axis, side, cc, 0, y, sc, nrm);
                const int a = pl[k];
                double loc[kGenMaxFQ];
                for (int b = 0; b < g.npf; ++b) loc[b] = 0.0;
                for (int q = 0; q < g.nqf; ++q) {
                    const double wq = cG.FW[q] * kappa * frow[(size_t)fl[k] * g.nqf + q] * sc;
                    for (int b = 0; b < g.npf; ++b) loc[b] += wq * cG.Nf[q][a] * cG.Nf[q][b];
                }
                for (int b = 0; b < g.npf; ++b) {
                    const int nb = gen_face_node(g, axis, side, cc, tr, b);
                    int jj[3];
                    gen_node_idx(g, nb, jj);
                    int dir = 0, mul = 1;
                    for (int k2 = 0; k2 < d; ++k2) {
                        dir += (jj[k2] - ii[k2] + p) * mul;
                        mul *= span;
                    }
                    acc[dir] += loc[b];
                }
            }
        };
        int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
        for (int a = 0; a < d; ++a) cells_of(g, a, ii[a], lo[a], hi[a]);
        bool faces_done = false;
        for (int c2 = lo[2]; c2 <= hi[2]; ++c2)
            for (int c1 = lo[1]; c1 <= hi[1]; ++c1)
                for (int c0 = lo[0]; c0 <= hi[0]; ++c0) {
                    const int cc[3] = {c0, c1, c2};
                    const int c = gen_cell(g, cc);
                    if (!faces_done && c >= 512) {
                        add_faces();
                        faces_done = true;
                    }
                    int ai[3] = {0, 0, 0};
                    for (int k = 0; k < d; ++k) ai[k] = ii[k] - p * cc[k];
                    const int a = ai[0] + q1 * (ai[1] + q1 * ai[2]);
                    double loc[kGenMaxQ];
                    for (int b = 0; b < g.npe; ++b) loc[b] = 0.0;
                    for (int q = 0; q < g.nq; ++q) {
                        const double* e = crow + (size_t)q * nc * g.ncells + c;  // planar layout
                        double A[3][3];
                        int idx = 1;
                        for (int r = 0; r < d; ++r)
                            for (int s = r; s < d; ++s) A[r][s] = A[s][r] = e[(size_t)(idx++) * g.ncells];
                        const double wq = cG.W[q] * det_elem * P.Dv;
                        double ga[3], Ag[3];
                        for (int k = 0; k < d; ++k) ga[k] = cG.dN[q][a][k] * gs[k];
                        for (int r = 0; r < d; ++r) {
                            double s = A[r][0] * ga[0];
                            for (int k = 1; k < d; ++k) s += A[r][k] * ga[k];
                            Ag[r] = s;
                        }
                        for (int b = 0; b < g.npe; ++b) {
                            double s = Ag[0] * (cG.dN[q][b][0] * gs[0]);
                            for (int r = 1; r < d; ++r) s += Ag[r] * (cG.dN[q][b][r] * gs[r]);
                            loc[b] += wq * s;
                        }
                        if (react) {
                            double y[3];
                            gen_cell_qpoint(g, cG, cc, q, y);
                            const double wr = cG.W[q] * det_elem * reaction_k(P, y) * e[0];
                            for (int b = 0; b < g.npe; ++b) loc[b] += wr * cG.N[q][a] * cG.N[q][b];
                        }
                    }
                    for (int b = 0; b < g.npe; ++b) {
                        const int bi[3] = {b % q1, (b / q1) % q1, b / (q1 * q1)};
                        int dir = 0, mul = 1;
                        for (int k = 0; k < d; ++k) {
                            dir += (p * cc[k] + bi[k] - ii[k] + p) * mul;
                            mul *= span;
                        }
                        acc[dir] += loc[b];
                    }
                }
        if (!faces_done) add_faces();
        // stored: the centre and the upper half of the directions (plane k - ctr); the lower
        // half is the neighbours' upper entries by symmetry
        const int ctr = g.ndirs / 2;
        double* out = stencil + (size_t)sys * (ctr + 1) * n + node;
        for (int k = ctr; k < g.ndirs; ++k) out[(size_t)(k - ctr) * n] = acc[k];
    }
}

// k_gassemble with the element structure at compile time.  Along each axis a lattice node
// is either a cell vertex position (C = 0: the lower cell holds it as local node P, the
// upper as local node 0) or, for P = 2, an interior position (C = 1: one cell, local node
// 1).  With the class (CX, CY, CZ) fixed, every (cell position, element node) pair maps to a
// compile-time stencil direction, so the row stays in registers instead of local memory.
// Same arithmetic, same order (cells ascending in 512-cell chunks, faces merged after chunk
// 0) as k_gassemble, so bitwise the same values.
template <int ND>
__device__ __forceinline__ void acc_at(double (&acc)[ND], int dir, double v) {
#pragma unroll
    for (int k = 0; k < ND; ++k)
        if (k == dir) acc[k] += v;
}

// Per-block quadrature tables in shared memory (the rolled q loop would otherwise index
// __constant__ arrays at run time: LDC traffic, ncu short_scoreboard 34 %).  Each entry is
// the same single product the loop formed before, so the bits are unchanged:
//   GB[q][b][k] = dN[q][b][k] * (2 / h_k),  WD[q] = W[q] * det_elem,  NN[q][b] = N[q][b].
template <int D, int P>
struct AsmTables {
    static constexpr int Q1 = P + 1, NPE = D == 2 ? Q1 * Q1 : Q1 * Q1 * Q1;
    double GB[NPE][NPE][D];
    double WD[NPE];
    double NN[NPE][NPE];
};

// The boundary faces of a lattice node that carry a Robin term (assembly.cpp:149-169), in the
// order the reference adds them: face index, the node's face-local index, the face's role,
// the face scale and the stencil direction of every face node.  The same for every system,
// so it is tabulated once per context build (k_gface_table) instead of being re-derived by
// every (system, node) thread: the face lookups were a third of the assembly kernel's
// instructions, executed by nearly every warp for a few boundary lanes each.
constexpr int kMaxNodeFaces = 12;
struct GFaceRef {
    int f, a, role, pad;
    double sc;
    int dirs[kGenMaxFQ + 1];
};

template <int D, int P>
__global__ void k_gface_table(GenProblem Pr, int* __restrict__ fcount, GFaceRef* __restrict__ ftab) {
    const GenGeom& g = Pr.g;
    constexpr int Q1 = P + 1, SPAN = 2 * P + 1, NFQ = D == 2 ? Q1 : Q1 * Q1;
    const int node = blockIdx.x * blockDim.x + threadIdx.x;
    if (node >= g.nnodes) return;
    int ii[3] = {0, 0, 0};
    gen_node_idx(g, node, ii);
    int fl[kMaxNodeFaces], pl[kMaxNodeFaces];
    const int nf = gen_node_faces(g, ii, fl, pl);
    int cnt = 0;
    for (int k = 0; k < nf; ++k) {
        int axis, side, cc[3], tr[2];
        gen_face(g, fl[k], axis, side, cc, tr);
        const int role = Pr.role[2 * axis + side];
        if (role == TS_GAMMA_N) continue;
        const double kappa = role == TS_GAMMA_I ? Pr.kappa[1] : Pr.kappa[3];
        if (kappa == 0.0) continue;
        double y[3], sc, nrm[3];
        gen_face_geom(g, cG, axis, side, cc, 0, y, sc, nrm);
        GFaceRef R;
        R.f = fl[k];
        R.a = pl[k];
        R.role = role;
        R.pad = 0;
        R.sc = sc;
        for (int b = 0; b <= kGenMaxFQ; ++b) R.dirs[b] = -1;
        for (int b = 0; b < NFQ; ++b) {
            const int nb = gen_face_node(g, axis, side, cc, tr, b);
            int jj[3];
            gen_node_idx(g, nb, jj);
            int dir = 0, mul = 1;
            for (int k2 = 0; k2 < D; ++k2) {
                dir += (jj[k2] - ii[k2] + P) * mul;
                mul *= SPAN;
            }
            R.dirs[b] = dir;
        }
        ftab[(size_t)node * kMaxNodeFaces + cnt++] = R;
    }
    fcount[node] = cnt;
}

template <int D, int P, int CX, int CY, int CZ>
__device__ __forceinline__ void gassemble_node(const GenProblem& Pr, int sys, const int* ii,
                                               const double* __restrict__ cells, const double* __restrict__ faces,
                                               double* __restrict__ stencil, const AsmTables<D, P>& T,
                                               const int* __restrict__ fcount, const GFaceRef* __restrict__ ftab) {
    const GenGeom& g = Pr.g;
    constexpr int Q1 = P + 1, NC = 1 + D * (D + 1) / 2, SPAN = 2 * P + 1;
    constexpr int NPE = D == 2 ? Q1 * Q1 : Q1 * Q1 * Q1, NQ = NPE, ND = D == 2 ? SPAN * SPAN : SPAN * SPAN * SPAN;
    constexpr int NFQ = D == 2 ? Q1 : Q1 * Q1;
    // Only the centre and the upper half of the row are formed and stored (directions
    // CTR .. ND - 1 at planes 0 .. NUP - 1): the solvers read the lower half as the neighbours'
    // upper entries (the operator is symmetric), so the other (a, b) products of a cell —
    // 28 of 64 for trilinear hexahedra — are never needed.
    constexpr int CTR = ND / 2, NUP = CTR + 1;
    const int n = g.nnodes;
    const bool react = !(Pr.reaction_kind == TS_REACTION_CONST && Pr.reaction_in == 0.0);
    double acc[NUP];
#pragma unroll
    for (int k = 0; k < NUP; ++k) acc[k] = 0.0;
    const double* crow = cells + (size_t)sys * g.ncells * NQ * NC;
    const double* frow = faces + (size_t)sys * g.nfaces * NFQ;
    const int node = gen_node(g, ii[0], ii[1], ii[2]);
    auto add_faces = [&]() {  // the node's Robin face rows in the reference's order (k_gface_table)
        const int nfr = fcount[node];
        for (int k = 0; k < nfr; ++k) {
            const GFaceRef& R = ftab[(size_t)node * kMaxNodeFaces + k];
            const double kappa = R.role == TS_GAMMA_I ? Pr.kappa[1] : Pr.kappa[3];
            const int a = R.a;
            double loc[NFQ];
#pragma unroll
            for (int b = 0; b < NFQ; ++b) loc[b] = 0.0;
#pragma unroll
            for (int q = 0; q < NFQ; ++q) {
                const double wq = cG.FW[q] * kappa * frow[(size_t)R.f * NFQ + q] * R.sc;
#pragma unroll
                for (int b = 0; b < NFQ; ++b) loc[b] += wq * cG.Nf[q][a] * cG.Nf[q][b];
            }
#pragma unroll
            for (int b = 0; b < NFQ; ++b) acc_at(acc, R.dirs[b] - CTR, loc[b]);  // lower directions match nothing
        }
    };
    constexpr int C3[3] = {CX, CY, CZ};
    constexpr int NO0 = CX ? 1 : 2, NO1 = CY ? 1 : 2, NO2 = D == 3 ? (CZ ? 1 : 2) : 1;
    bool faces_done = false;
    // Loops stay rolled (an unrolled cell-position x NQ body thrashes the instruction cache, ncu:
    // 81 % of stalls "no instruction"; unrolling the positions alone measured 2x slower, too);
    // the row stays in registers through acc_at.  Per cell position the needed element nodes b
    // (direction >= CTR) are a warp-uniform bit mask.
    constexpr int NOT = NO0 * NO1 * NO2;
#pragma unroll 1
    for (int o = 0; o < NOT; ++o) {
        const int oo[3] = {o % NO0, (o / NO0) % NO1, o / (NO0 * NO1)};
        int cc[3] = {0, 0, 0}, al[3] = {0, 0, 0};
        bool valid = true;
#pragma unroll
        for (int k = 0; k < D; ++k) {
            // local node index along k: interior position 1, lower cell P, upper cell 0
            al[k] = C3[k] ? 1 : (oo[k] == 0 ? P : 0);
            cc[k] = (ii[k] - al[k]) / P;
            valid = valid && ii[k] - al[k] >= 0 && cc[k] < g.nc[k];
        }
        const int c = valid ? gen_cell(g, cc) : 0;
        if (!faces_done && valid && c >= 512) {  // the faces follow the first 512-cell chunk
            add_faces();
            faces_done = true;
        }
        if (!valid) continue;
        const int a = al[0] + Q1 * (al[1] + Q1 * al[2]);
        int base = 0, mul = 1;  // direction of element node b = base + sum_k bi_k SPAN^k
#pragma unroll
        for (int k = 0; k < D; ++k) {
            base += (P - al[k]) * mul;
            mul *= SPAN;
        }
        auto off_of = [&](int b) { return (b % Q1) + SPAN * ((b / Q1) % Q1) + SPAN * SPAN * (b / (Q1 * Q1)); };
        unsigned need = 0;
#pragma unroll
        for (int b = 0; b < NPE; ++b)
            if (base + off_of(b) >= CTR) need |= 1u << b;
        double loc[NPE];
#pragma unroll
        for (int b = 0; b < NPE; ++b) loc[b] = 0.0;
        // the cell's cache entries, planar: entry k of point q at ce[(q * NC + k) * ncells]; point
        // q + 1 is fetched while point q is used (the loads are L2 latency: ncu had
        // long_scoreboard as the top stall with the loads at the head of each iteration)
        const double* ce = crow + c;
        const size_t cs = (size_t)g.ncells;
        double en[NC];
#pragma unroll
        for (int k = 0; k < NC; ++k) en[k] = ce[k * cs];
#pragma unroll 1
        for (int q = 0; q < NQ; ++q) {
            double ev[NC];
#pragma unroll
            for (int k = 0; k < NC; ++k) ev[k] = en[k];
            if (q + 1 < NQ) {
                ce += NC * cs;
#pragma unroll
                for (int k = 0; k < NC; ++k) en[k] = ce[k * cs];
            }
            double A[3][3];
            int idx = 1;
#pragma unroll
            for (int r = 0; r < D; ++r)
#pragma unroll
                for (int s2 = r; s2 < D; ++s2) A[r][s2] = A[s2][r] = ev[idx++];
            const double wq = T.WD[q] * Pr.Dv;  // = W[q] * det_elem * Dv
            double ga[3], Ag[3];
#pragma unroll
            for (int k = 0; k < D; ++k) ga[k] = T.GB[q][a][k];
#pragma unroll
            for (int r = 0; r < D; ++r) {
                double sum = A[r][0] * ga[0];
#pragma unroll
                for (int k = 1; k < D; ++k) sum += A[r][k] * ga[k];
                Ag[r] = sum;
            }
            double wa = 0.0;
            if (react) {
                double kq = Pr.reaction_in;  // constant reaction: no quadrature-point coordinates needed
                if (Pr.reaction_kind != TS_REACTION_CONST) {
                    double y[3];
                    gen_cell_qpoint(g, cG, cc, q, y);
                    kq = reaction_k(Pr, y);
                }
                const double wr = T.WD[q] * kq * ev[0];
                wa = wr * T.NN[q][a];
            }
#pragma unroll
            for (int b = 0; b < NPE; ++b) {
                if (!((need >> b) & 1u)) continue;  // warp-uniform
                double sum = Ag[0] * T.GB[q][b][0];
#pragma unroll
                for (int r = 1; r < D; ++r) sum += Ag[r] * T.GB[q][b][r];
                loc[b] += wq * sum;
                if (react) loc[b] += wa * T.NN[q][b];
            }
        }
#pragma unroll
        for (int b = 0; b < NPE; ++b) acc_at(acc, base + off_of(b) - CTR, loc[b]);  // unneeded b: no match
    }
    if (!faces_done) add_faces();
    double* out = stencil + (size_t)sys * NUP * n + node;
#pragma unroll
    for (int k = 0; k < NUP; ++k) out[(size_t)k * n] = acc[k];
}

// Thread t -> (system, node) with the nodes of each system enumerated class-major for
// P = 2 (so a warp runs one compile-time class), lattice order for P = 1.
template <int D, int P>
__global__ void __launch_bounds__(128) k_gassemble_t(GenProblem Pr, int srows, const double* __restrict__ cells,
                                                      const double* __restrict__ faces, double* __restrict__ stencil,
                                                      const int* __restrict__ fcount,
                                                      const GFaceRef* __restrict__ ftab) {
    const GenGeom& g = Pr.g;
    const int n = g.nnodes;
    const long long total = (long long)srows * n;
    __shared__ AsmTables<D, P> T;
    {
        constexpr int NPE = AsmTables<D, P>::NPE;
        const double det_elem = D == 2 ? 0.25 * g.h[0] * g.h[1] : 0.125 * g.h[0] * g.h[1] * g.h[2];
        for (int t = threadIdx.x; t < NPE * NPE; t += blockDim.x) {
            const int q = t / NPE, b = t % NPE;
            for (int k = 0; k < D; ++k) T.GB[q][b][k] = cG.dN[q][b][k] * (2.0 / g.h[k]);
            T.NN[q][b] = cG.N[q][b];
            if (b == 0) T.WD[q] = cG.W[q] * det_elem;
        }
        __syncthreads();
    }
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
        const int sys = (int)(t / n);
        int K = (int)(t % n);
        int ii[3] = {0, 0, 0};
        if constexpr (P == 1) {
            gen_node_idx(g, K, ii);
            gassemble_node<D, 1, 0, 0, 0>(Pr, sys, ii, cells, faces, stencil, T, fcount, ftab);
        } else {
        // 2D, P = 2: classes (i odd, j odd) = 00, 10, 01, 11; counts ci[a] x cj[b]
        const int ci0 = (g.nn[0] + 1) / 2, ci1 = g.nn[0] / 2, cj0 = (g.nn[1] + 1) / 2, cj1 = g.nn[1] / 2;
        const int cnt[4] = {ci0 * cj0, ci1 * cj0, ci0 * cj1, ci1 * cj1};
        int c = 0;
        while (c < 3 && K >= cnt[c]) K -= cnt[c++];
        const int a = c & 1, b = c >> 1, w = a ? ci1 : ci0;
        ii[0] = 2 * (K % w) + a;
        ii[1] = 2 * (K / w) + b;
        switch (c) {
            case 0: gassemble_node<2, P, 0, 0, 0>(Pr, sys, ii, cells, faces, stencil, T, fcount, ftab); break;
            case 1: gassemble_node<2, P, 1, 0, 0>(Pr, sys, ii, cells, faces, stencil, T, fcount, ftab); break;
            case 2: gassemble_node<2, P, 0, 1, 0>(Pr, sys, ii, cells, faces, stencil, T, fcount, ftab); break;
            default: gassemble_node<2, P, 1, 1, 0>(Pr, sys, ii, cells, faces, stencil, T, fcount, ftab); break;
        }
        }
    }
}

__global__ void k_grhs_parts(GenProblem P, int n_nodes, int shared, const double* __restrict__ faces, double* rin,
                             double* rout) {
    const GenGeom& g = P.g;
    const int n = g.nnodes;
    const long long total = (long long)n_nodes * n;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(t % n);
        const int node = (int)(t / n);
        const double* frow = faces + (size_t)(shared ? 0 : node) * g.nfaces * g.nqf;
        int ii[3], fl[12], pl[12];
        gen_node_idx(g, k, ii);
        const int nf = gen_node_faces(g, ii, fl, pl);
        double ri = 0.0, ro = 0.0;
        for (int j = 0; j < nf; ++j) {
            int axis, side, cc[3], tr[2];
            gen_face(g, fl[j], axis, side, cc, tr);
            const int role = P.role[2 * axis + side];
            double y[3], sc, nrm[3];
            gen_face_geom(g, cG, axis, side, cc, 0, y, sc, nrm);
            for (int q = 0; q < g.nqf; ++q) {
                const double w_meas = cG.FW[q] * frow[(size_t)fl[j] * g.nqf + q] * sc;
                if (role == TS_GAMMA_I)
                    ri += w_meas * cG.Nf[q][pl[j]];
                else if (role == TS_GAMMA_O)
                    ro += w_meas * cG.Nf[q][pl[j]];
            }
        }
        rin[t] = ri;
        rout[t] = ro;
    }
}

// gamma_in/out and rhs integrands per macro quadrature point (assembly.cpp:237-281).  One
// block per quadrature point: the threads evaluate the micro face points into shared memory,
// thread 0 adds them in the serial loop's order (faces ascending, q inner) — the same bits
// as one thread doing it all, with the map evaluations spread over the block.
constexpr int kGmqThreads = 128;
constexpr int kGmqChunk = 512;

// D: the micro dimension at compile time (a local copy of the geometry carries it, so the
// inlined face helpers unroll their per-axis loops).  One block per macro cell: the micro
// face point geometry (face lookup, point, scale, normal) is the same for every macro point,
// so a thread derives it once and evaluates the map at the cell's four quadrature points; four
// threads then add the four points' terms in the serial loop's order.
template <int D>
__global__ void __launch_bounds__(kGmqThreads) k_gmacro_qpoints(GenProblem P, QuadTables Q, double* gamma_in,
                                                                double* gamma_out, double* rhs_u_q, double* rhs_w_q,
                                                                double* dw_q, unsigned long long* first_bad,
                                                                unsigned* err) {
    __shared__ double s_w[4][kGmqChunk];
    __shared__ signed char s_role[kGmqChunk];
    __shared__ double s_scalar[4][3];
    __shared__ double s_row[4][16];  // tabulated maps: the table interpolated at each macro point, once
    GenGeom g = P.g;
    g.d = D;
    const int ncell = P.macro.cells();
    const int npts = g.nfaces * g.nqf;
    const bool tab = P.map.kind != TS_MAP_TAPE;
    const int* op = P.map.op;
    const int* arg = P.map.arg;
    const double* val = P.map.val;
    for (int cell = blockIdx.x; cell < ncell; cell += gridDim.x) {
        double x0[4], x1[4];
#pragma unroll
        for (int m = 0; m < 4; ++m) cell_pt(P.macro, cell, Q.QS[m], Q.QT[m], x0[m], x1[m]);
        if (threadIdx.x < 12) {
            const int m = threadIdx.x / 3, which = threadIdx.x % 3;
            const TapeRef t = which == 0 ? P.data.fu : which == 1 ? P.data.fw : P.data.Dw;
            double xa = x0[0], xb = x1[0];
#pragma unroll
            for (int mm = 1; mm < 4; ++mm)
                if (mm == m) {
                    xa = x0[mm];
                    xb = x1[mm];
                }
            s_scalar[m][which] = tape_eval(op, arg, val, t, xa, xb, 0.0, 0.0, err);
        }
        if (tab && threadIdx.x >= 32 && threadIdx.x < 36) {
            const int m = threadIdx.x - 32;
            double xa = x0[0], xb = x1[0];
#pragma unroll
            for (int mm = 1; mm < 4; ++mm)
                if (mm == m) {
                    xa = x0[mm];
                    xb = x1[mm];
                }
            table_row(P.map, -1, xa, xb, s_row[m]);
        }
        __syncthreads();
        double g_in = 0.0, g_out = 0.0;  // threads 0..3: macro point threadIdx.x
        for (int c0 = 0; c0 < npts; c0 += kGmqChunk) {
            const int cn = min(kGmqChunk, npts - c0);
            for (int k = threadIdx.x; k < cn; k += kGmqThreads) {
                const int f = (c0 + k) / g.nqf, q = (c0 + k) % g.nqf;
                int axis, side, cc[3], tr[2];
                gen_face(g, f, axis, side, cc, tr);
                double y[3], sc, nrm[3];
                gen_face_geom(g, cG, axis, side, cc, q, y, sc, nrm);
                const double w = cG.FW[q] * sc;
#pragma unroll
                for (int m = 0; m < 4; ++m) {
                    double len, det;
                    if (!gen_face_len(P.map, D, -1, x0[m], x1[m], y, nrm, len, det, err, tab ? s_row[m] : nullptr))
                        atomicMin(first_bad, (unsigned long long)(cell * 4 + m) * npts + f * g.nqf + q);
                    s_w[m][k] = w * len;
                }
                s_role[k] = (signed char)P.role[2 * axis + side];
            }
            __syncthreads();
            if (threadIdx.x < 4)
                for (int k = 0; k < cn; ++k) {
                    if (s_role[k] == TS_GAMMA_I) g_in += s_w[threadIdx.x][k];
                    else if (s_role[k] == TS_GAMMA_O) g_out += s_w[threadIdx.x][k];
                }
            __syncthreads();
        }
        if (threadIdx.x < 4) {
            const int qg = cell * 4 + threadIdx.x;
            gamma_in[qg] = g_in;
            gamma_out[qg] = g_out;
            rhs_u_q[qg] = s_scalar[threadIdx.x][0] + 0.0 - 0.0;
            rhs_w_q[qg] = s_scalar[threadIdx.x][1] + 0.0 - 0.0;
            dw_q[qg] = s_scalar[threadIdx.x][2];
        }
        __syncthreads();
    }
}

// Coefficient tensors of the matrix-free Q2 operator (gpcg.cu k_gen_pcg_q2t) from the cell
// and face caches: per cell quadrature point T0 = w Dv A00 s0^2, T1 = w Dv A01 s0 s1,
// T2 = w Dv A11 s1^2 (w = W_q det_elem, s = 2/h: the factors build_micro_matrices applies,
// src/assembly.cpp:129-147, folded into the coefficient) and T3 = w k(y_q) J (the reaction
// extension); per face point F = FW_q kappa |nu| scale (assembly.cpp:149-169; 0 on Gamma^N
// or kappa = 0).  Layout [colour][k][q][cell of colour], colour = (ci & 1) + 2 (cj & 1).
__global__ void k_q2_tensor_pack(GenProblem P, int rows, const double* __restrict__ cells,
                                 const double* __restrict__ faces, double* __restrict__ tens) {
    const GenGeom& g = P.g;
    const long long per_row = 36LL * g.ncells + 3LL * g.nfaces;
    const long long total = (long long)rows * per_row;
    const double det_elem = 0.25 * g.h[0] * g.h[1];
    const double s0 = 2.0 / g.h[0], s1 = 2.0 / g.h[1];
    int cw[4], cnt[4], cbase[4], base = 0;
    for (int c = 0; c < 4; ++c) {
        const int a = c & 1, b = c >> 1;
        cw[c] = (g.nc[0] + 1 - a) / 2;
        cnt[c] = cw[c] * ((g.nc[1] + 1 - b) / 2);
        cbase[c] = base;
        base += 36 * cnt[c];
    }
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(t / per_row);
        const int e = (int)(t % per_row);
        double v;
        if (e < 36 * g.ncells) {
            int c = 0;
            while (c < 3 && e >= cbase[c + 1]) ++c;
            const int w = e - cbase[c], l = w % cnt[c], kq = w / cnt[c], k = kq / 9, q = kq % 9;
            const int ci = 2 * (l % cw[c]) + (c & 1), cj = 2 * (l / cw[c]) + (c >> 1);
            const int cell = ci + g.nc[0] * cj;
            const double* ce = cells + ((size_t)row * 9 + q) * 4 * g.ncells + cell;  // planar: J, A00, A01, A11
            const size_t cs = g.ncells;
            const double wq = cG.W[q] * det_elem;
            if (k == 0) v = wq * P.Dv * ce[cs] * s0 * s0;
            else if (k == 1) v = wq * P.Dv * ce[2 * cs] * s0 * s1;
            else if (k == 2) v = wq * P.Dv * ce[3 * cs] * s1 * s1;
            else {
                const bool react = !(P.reaction_kind == TS_REACTION_CONST && P.reaction_in == 0.0);
                double y[3];
                const int cc[3] = {ci, cj, 0};
                gen_cell_qpoint(g, cG, cc, q, y);
                v = react ? wq * reaction_k(P, y) * ce[0] : 0.0;
            }
        } else {
            const int fq = e - 36 * g.ncells, f = fq / 3, q = fq % 3;
            int axis, side, cc[3], tr[2];
            gen_face(g, f, axis, side, cc, tr);
            const int role = P.role[2 * axis + side];
            const double kappa = role == TS_GAMMA_I ? P.kappa[1] : role == TS_GAMMA_O ? P.kappa[3] : 0.0;
            double y[3], sc, nrm[3];
            gen_face_geom(g, cG, axis, side, cc, 0, y, sc, nrm);
            v = cG.FW[q] * kappa * faces[((size_t)row * g.nfaces + f) * 3 + q] * sc;
        }
        tens[t] = v;
    }
}

}  // namespace

void launch_gcell_cache(const GenProblem& P, int rows, const double* points, double* out,
                        unsigned long long* first_bad, unsigned* err, cudaStream_t s, int row0) {
    const long long total = (long long)rows * P.g.ncells * P.g.nq;
    if (P.g.d == 3) return (void)(k_gcell_cache_t<3><<<grid_for(total), kThreads, 0, s>>>(P, rows, points, out, first_bad, err, row0));
    if (P.g.d == 2) return (void)(k_gcell_cache_t<2><<<grid_for(total), kThreads, 0, s>>>(P, rows, points, out, first_bad, err, row0));
    k_gcell_cache<<<grid_for(total), kThreads, 0, s>>>(P, rows, points, out, first_bad, err, row0);
}

void launch_gface_cache(const GenProblem& P, int rows, const double* points, int with_cells, double* out,
                        unsigned long long* first_bad, unsigned* err, cudaStream_t s) {
    const long long total = (long long)rows * P.g.nfaces * P.g.nqf;
    k_gface_cache<<<grid_for(total), kThreads, 0, s>>>(P, rows, points, with_cells, out, first_bad, err);
}

void launch_gprobe(const GenProblem& P, const double* points, int with_cells, unsigned long long index, double* out,
                   cudaStream_t s) {
    k_gprobe<<<1, 1, 0, s>>>(P, points, with_cells, index, out);
}

void launch_gassemble(const GenProblem& P, int srows, const double* cells, const double* faces, double* stencil,
                      cudaStream_t s) {
    const long long total = (long long)srows * P.g.nnodes;
    const int grid = std::max(1, (int)std::min<long long>(148LL * 64, (total + 127) / 128));
    if (std::getenv("TS_GASSEMBLE_RT") == nullptr) {  // runtime-structure kernel kept for A/B checks
        auto run = [&](auto table, auto kern) {
            int* fcount = nullptr;
            GFaceRef* ftab = nullptr;
            const int n = P.g.nnodes;
            if (cudaMallocAsync(&fcount, sizeof(int) * n, s) != cudaSuccess ||
                cudaMallocAsync(&ftab, sizeof(GFaceRef) * (size_t)n * kMaxNodeFaces, s) != cudaSuccess) {
                if (fcount) cudaFreeAsync(fcount, s);
                cudaGetLastError();
                return false;  // no table: the runtime-structure kernel below assembles instead
            }
            table<<<(n + 127) / 128, 128, 0, s>>>(P, fcount, ftab);
            kern<<<grid, 128, 0, s>>>(P, srows, cells, faces, stencil, fcount, ftab);
            cudaFreeAsync(ftab, s);
            cudaFreeAsync(fcount, s);
            return true;
        };
        if (P.g.d == 3 && P.g.p == 1 && run(k_gface_table<3, 1>, k_gassemble_t<3, 1>)) return;
        if (P.g.d == 2 && P.g.p == 2 && run(k_gface_table<2, 2>, k_gassemble_t<2, 2>)) return;
        if (P.g.d == 2 && P.g.p == 1 && run(k_gface_table<2, 1>, k_gassemble_t<2, 1>)) return;
    }
    k_gassemble<<<grid_for(total), 128, 0, s>>>(P, srows, cells, faces, stencil);
}

void launch_q2_tensor_pack(const GenProblem& P, int rows, const double* cells, const double* faces, double* tensor,
                           cudaStream_t s) {
    const long long total = (long long)rows * (36LL * P.g.ncells + 3LL * P.g.nfaces);
    k_q2_tensor_pack<<<grid_for(total), kThreads, 0, s>>>(P, rows, cells, faces, tensor);
}

void launch_grhs_parts(const GenProblem& P, int n_nodes, int shared, const double* faces, double* rin, double* rout,
                       cudaStream_t s) {
    const long long total = (long long)n_nodes * P.g.nnodes;
    k_grhs_parts<<<grid_for(total), kThreads, 0, s>>>(P, n_nodes, shared, faces, rin, rout);
}

void launch_gmacro_qpoints(const GenProblem& P, const QuadTables& Q, double* gamma_in, double* gamma_out,
                           double* rhs_u_q, double* rhs_w_q, double* dw_q, unsigned long long* first_bad,
                           unsigned* err, cudaStream_t s) {
    const int total = P.macro.cells();  // one block per macro cell (its four quadrature points)
    if (P.g.d == 3)
        k_gmacro_qpoints<3><<<std::min(total, 148 * 16), kGmqThreads, 0, s>>>(P, Q, gamma_in, gamma_out, rhs_u_q,
                                                                              rhs_w_q, dw_q, first_bad, err);
    else
        k_gmacro_qpoints<2><<<std::min(total, 148 * 16), kGmqThreads, 0, s>>>(P, Q, gamma_in, gamma_out, rhs_u_q,
                                                                              rhs_w_q, dw_q, first_bad, err);
}

}  // namespace tsb
