// Kernels (1) and (2) and the macro-system build: everything the reference does
// in the AssemblyContext constructor (assembly.cpp:52-99).  Compiled with
// -fmad=false: each product/sum is rounded separately and, where the reference
// has a fixed serial order, accumulated in that order, so the results reproduce
// the reference's 1-worker build to the last bit whenever the map values agree.
//
// Work decomposition is node-centric gather (one thread per output entry), never
// scatter: no FP64 atomics, deterministic, and the per-entry summation order is
// exactly the reference's scatter order.
#include <math_constants.h>

#include <algorithm>
#include <cstdio>

#include "kernels.h"

namespace tsb {

__constant__ QuadTables cQ;  // used by this translation unit only (no -rdc)

void upload_quad_tables(const QuadTables& q) { cudaMemcpyToSymbol(cQ, &q, sizeof(QuadTables)); }

namespace {

constexpr int kThreads = 256;

struct FaceP {
    double mx, my, tx, ty, nx, ny;
};

__device__ __forceinline__ FaceP face_param(const GridG& g, int f, int& side, int& a, int& b) {
    face_info(g, f, side, a, b);
    double ax, ay, bx, by;
    node_xy(g, a, ax, ay);
    node_xy(g, b, bx, by);
    FaceP p;
    p.mx = 0.5 * (ax + bx);
    p.my = 0.5 * (ay + by);
    p.tx = 0.5 * (bx - ax);
    p.ty = 0.5 * (by - ay);
    p.nx = side == 0 ? -1.0 : side == 1 ? 1.0 : 0.0;  // side_normal, grid.cpp:18-26
    p.ny = side == 2 ? -1.0 : side == 3 ? 1.0 : 0.0;
    return p;
}

__device__ __forceinline__ double face_scale(const FaceP& p) { return sqrt(p.tx * p.tx + p.ty * p.ty); }

__device__ __forceinline__ void row_point(const ProblemG& p, int row, const double* points, double& x0,
                                          double& x1, int& node, int row0 = 0) {
    if (points) {
        x0 = points[2 * row];
        x1 = points[2 * row + 1];
        node = -1;
    } else {
        node = row0 + row;
        node_xy(p.macro, node, x0, x1);
    }
}

// mapping.cpp:96-110 with the D-tensor extension A = C^T D C / det.
__device__ __forceinline__ bool cell_coef(const MapG& m, int node, double x0, double x1, double y0,
                                          double y1, double4& e, unsigned* err) {
    double F[4];
    map_jac(m, node, x0, x1, y0, y1, F, err);
    const double det = F[0] * F[3] - F[1] * F[2];
    const double C00 = F[3], C01 = -F[2], C10 = -F[1], C11 = F[0];
    e.x = det;
    if (m.D_identity) {
        e.y = (C00 * C00 + C10 * C10) / det;
        e.z = (C00 * C01 + C10 * C11) / det;
        e.w = (C01 * C01 + C11 * C11) / det;
    } else {
        const double DC00 = m.D[0] * C00 + m.D[1] * C10, DC01 = m.D[0] * C01 + m.D[1] * C11;
        const double DC10 = m.D[2] * C00 + m.D[3] * C10, DC11 = m.D[2] * C01 + m.D[3] * C11;
        e.y = (C00 * DC00 + C10 * DC10) / det;
        e.z = (C00 * DC01 + C10 * DC11) / det;
        e.w = (C01 * DC01 + C11 * DC11) / det;
    }
    return det > 1e-12;
}

// mapping.cpp:112-126
__device__ __forceinline__ bool face_coef(const MapG& m, int node, double x0, double x1, double y0,
                                          double y1, double nx, double ny, double4& e, unsigned* err) {
    double F[4];
    map_jac(m, node, x0, x1, y0, y1, F, err);
    const double det = F[0] * F[3] - F[1] * F[2];
    const double C00 = F[3], C01 = -F[2], C10 = -F[1], C11 = F[0];
    e.x = det;
    e.y = C00 * nx + C01 * ny;
    e.z = C10 * nx + C11 * ny;
    e.w = sqrt(e.y * e.y + e.z * e.z);
    return det > 1e-12;
}

__global__ void k_cell_cache(ProblemG p, int rows, const double* points, double4* out,
                             unsigned long long* first_bad, unsigned* err, int row0) {
    const int cells = p.micro.cells();
    const long long total = (long long)rows * cells * 4;
    const long long stride_row = (long long)cells * 4 + (long long)p.micro.faces() * 2;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int q = (int)(t & 3);
        const long long rc = t >> 2;
        const int c = (int)(rc % cells);
        const int row = (int)(rc / cells);
        double x0, x1, y0, y1;
        int node;
        row_point(p, row, points, x0, x1, node, row0);
        cell_pt(p.micro, c, cQ.QS[q], cQ.QT[q], y0, y1);
        double4 e;
        if (!cell_coef(p.map, node, x0, x1, y0, y1, e, err))
            atomicMin(first_bad, (unsigned long long)(row * stride_row + (long long)c * 4 + q));
        out[t] = e;
    }
}

__global__ void k_face_cache(ProblemG p, int rows, const double* points, int with_cells,
                             double4* out, unsigned long long* first_bad, unsigned* err, int row0) {
    const int faces = p.micro.faces();
    const long long total = (long long)rows * faces * 2;
    const long long cpart = with_cells ? (long long)p.micro.cells() * 4 : 0;
    const long long stride_row = cpart + (long long)faces * 2;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int q = (int)(t & 1);
        const long long rf = t >> 1;
        const int f = (int)(rf % faces);
        const int row = (int)(rf / faces);
        double x0, x1;
        int node;
        row_point(p, row, points, x0, x1, node, row0);
        int side, a, b;
        const FaceP fp = face_param(p.micro, f, side, a, b);
        const double y0 = fp.mx + fp.tx * cQ.GP[q], y1 = fp.my + fp.ty * cQ.GP[q];
        double4 e;
        if (!face_coef(p.map, node, x0, x1, y0, y1, fp.nx, fp.ny, e, err))
            atomicMin(first_bad, (unsigned long long)(row * stride_row + cpart + (long long)f * 2 + q));
        out[t] = e;
    }
}

__global__ void k_probe(ProblemG p, const double* points, int with_cells, unsigned long long index,
                        double* out) {
    const long long cells4 = with_cells ? (long long)p.micro.cells() * 4 : 0;
    const long long stride_row = cells4 + (long long)p.micro.faces() * 2;
    const int row = (int)(index / stride_row);
    const long long r = index % stride_row;
    double x0, x1, y0, y1;
    int node;
    unsigned* err = nullptr;
    row_point(p, row, points, x0, x1, node);
    double4 e;
    if (r < cells4) {
        cell_pt(p.micro, (int)(r / 4), cQ.QS[r % 4], cQ.QT[r % 4], y0, y1);
        cell_coef(p.map, node, x0, x1, y0, y1, e, err);
    } else {
        const int f = (int)((r - cells4) / 2), q = (int)((r - cells4) % 2);
        int side, a, b;
        const FaceP fp = face_param(p.micro, f, side, a, b);
        y0 = fp.mx + fp.tx * cQ.GP[q];
        y1 = fp.my + fp.ty * cQ.GP[q];
        face_coef(p.map, node, x0, x1, y0, y1, fp.nx, fp.ny, e, err);
    }
    out[0] = e.x;
    out[1] = x0;
    out[2] = x1;
    out[3] = y0;
    out[4] = y1;
}

// validate_diffeo (mapping.cpp:131-156): det grad_y zeta (Mat2::det, linalg.hpp:29) at every
// pair of xs x ys, pair t = ix * ny + iy (x outer, as the reference's loops).  Per block: the
// minimum with the first pair index reaching it, and the maximum; the host folds the block
// partials in index order, so `worst` is the reference's first strict minimum.
constexpr int kValThreads = 256;

__global__ void __launch_bounds__(kValThreads) k_validate_pairs(MapG m, const double* xs, int nx, const double* ys,
                                                                int ny, double* part, unsigned* err) {
    __shared__ double s_mn[kValThreads], s_mx[kValThreads];
    __shared__ long long s_at[kValThreads];
    const long long total = (long long)nx * ny;
    double mn = CUDART_INF, mx = -CUDART_INF;
    long long at = -1;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const long long ix = t / ny, iy = t % ny;
        double F[4];
        map_jac(m, -1, xs[2 * ix], xs[2 * ix + 1], ys[2 * iy], ys[2 * iy + 1], F, err);
        const double det = F[0] * F[3] - F[1] * F[2];
        if (at < 0 || det < mn) {  // indices rise within a thread: strict < keeps the first
            mn = det;
            at = t;
        }
        mx = fmax(mx, det);
    }
    s_mn[threadIdx.x] = mn;
    s_mx[threadIdx.x] = mx;
    s_at[threadIdx.x] = at;
    __syncthreads();
    for (int w = kValThreads / 2; w > 0; w >>= 1) {
        if (threadIdx.x < w) {
            const int o = threadIdx.x + w;
            const long long ao = s_at[o], am = s_at[threadIdx.x];
            if (ao >= 0 && (am < 0 || s_mn[o] < s_mn[threadIdx.x] || (s_mn[o] == s_mn[threadIdx.x] && ao < am))) {
                s_mn[threadIdx.x] = s_mn[o];
                s_at[threadIdx.x] = ao;
            }
            s_mx[threadIdx.x] = fmax(s_mx[threadIdx.x], s_mx[o]);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        part[3 * blockIdx.x + 0] = s_mn[0];
        part[3 * blockIdx.x + 1] = (double)s_at[0];
        part[3 * blockIdx.x + 2] = s_mx[0];
    }
}

// check_assumption6 (mapping.cpp:158-195): per macro point, the physical measures of
// Gamma^I and Gamma^O, len_f = sum_q w_q |nu|_{f,q} scale_f summed over the faces in the
// reference's face order (grid.cpp:35-45) — one thread per point, serial in that order, so
// the sums are the reference's bits.  |nu| at [(point * faces + f) * 2 + q] * stride + offset
// (a MapCache's compact |nu| or kernel (1)'s double4 face entries).
__global__ void k_boundary_measures(GridG micro, int4 role, int n, const double* nu, int stride, int offset,
                                    double* gamma) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const int faces = micro.faces();
    const int roles[4] = {role.x, role.y, role.z, role.w};
    double g_in = 0.0, g_out = 0.0;
    for (int f = 0; f < faces; ++f) {
        int side, a, b;
        const FaceP fp = face_param(micro, f, side, a, b);
        const int r = roles[side];
        if (r == TS_GAMMA_N) continue;
        const double scale = face_scale(fp);
        double len = 0.0;
        for (int q = 0; q < 2; ++q)
            len += cQ.GW[q] * nu[(((long long)i * faces + f) * 2 + q) * stride + offset] * scale;
        if (r == TS_GAMMA_I) g_in += len;
        else g_out += len;
    }
    gamma[2 * i] = g_in;
    gamma[2 * i + 1] = g_out;
}

// A data tape (e.g. D^w) at macro points: out[i] = tape(x_i, 0, 0).
__global__ void k_tape_at_points(const int* op, const int* arg, const double* val, TapeRef t, int n,
                                 const double* points, double* out, unsigned* err) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) out[i] = tape_eval(op, arg, val, t, points[2 * i], points[2 * i + 1], 0.0, 0.0, err);
}

__device__ __forceinline__ double reaction_k(const ProblemG& p, double y0, double y1) {
    if (p.reaction_kind == TS_REACTION_DISC) {
        const double dx = y0 - p.reaction[2], dy = y1 - p.reaction[3];
        return sqrt(dx * dx + dy * dy) < p.reaction[4] ? p.reaction[0] : p.reaction[1];
    }
    return p.reaction[0];
}

__device__ __forceinline__ bool has_reaction(const ProblemG& p) {
    return !(p.reaction_kind == TS_REACTION_CONST && p.reaction[0] == 0.0);
}

// Boundary faces (reference order) that contain node (i, j) of grid g; returns count (<= 2 per
// side pair, <= 2 in total for a rectangle) sorted ascending.
__device__ __forceinline__ int node_faces(const GridG& g, int i, int j, int* f, int* pos) {
    int k = 0;
    // Left/right faces come first in the order (indices < 2*n1), then bottom/top.
    if (i == 0 || i == g.n0) {
        const int side = i == 0 ? 0 : 1;
        if (j > 0) { f[k] = 2 * (j - 1) + side; pos[k] = 1; ++k; }
        if (j < g.n1) { f[k] = 2 * j + side; pos[k] = 0; ++k; }
    }
    if (j == 0 || j == g.n1) {
        const int side = j == 0 ? 0 : 1;
        if (i > 0) { f[k] = 2 * g.n1 + 2 * (i - 1) + side; pos[k] = 1; ++k; }
        if (i < g.n0) { f[k] = 2 * g.n1 + 2 * i + side; pos[k] = 0; ++k; }
    }
    // insertion sort (k <= 4)
    for (int a = 1; a < k; ++a)
        for (int b = a; b > 0 && f[b] < f[b - 1]; --b) {
            int t = f[b]; f[b] = f[b - 1]; f[b - 1] = t;
            t = pos[b]; pos[b] = pos[b - 1]; pos[b - 1] = t;
        }
    return k;
}

// acc[idx] += v for a runtime idx without dynamic register indexing (which would put the
// 9-entry row in local memory): one predicated add per entry, bitwise the plain add.
__device__ __forceinline__ void acc_add(double (&acc)[9], int idx, double v) {
#pragma unroll
    for (int d = 0; d < 9; ++d)
        if (d == idx) acc[d] += v;
}

// Corner offsets of the four cell nodes (grid.cpp:54-59), CCW from (ci, cj).
__device__ __constant__ int kCornerDi[4] = {0, 1, 1, 0};
__device__ __constant__ int kCornerDj[4] = {0, 0, 1, 1};

// build_micro_matrices (assembly.cpp:101-174) as a gather: thread = (system, node) row.
__global__ void __launch_bounds__(256, 3) k_assemble_micro(ProblemG p, int srows, const double4* __restrict__ cells,
                                 const double4* __restrict__ faces, double* __restrict__ stencil) {
    const GridG& g = p.micro;
    const int n = g.nodes(), ncell = g.cells(), nface = g.faces();
    const long long total = (long long)srows * n;
    const double det_elem = 0.25 * g.h0 * g.h1;
    const double gx = 2.0 / g.h0, gy = 2.0 / g.h1;
    const bool react = has_reaction(p);
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int node = (int)(t % n);
        const int sys = (int)(t / n);
        const int i = node % (g.n0 + 1), j = node / (g.n0 + 1);
        double acc[9];
#pragma unroll
        for (int d = 0; d < 9; ++d) acc[d] = 0.0;
        const double4* crow = cells + (size_t)sys * ncell * 4;
        const double4* frow = faces + (size_t)sys * nface * 2;

        auto add_faces = [&]() {
            int fl[4], pl[4];
            const int nf = node_faces(g, i, j, fl, pl);
            for (int k = 0; k < nf; ++k) {
                int side, na, nb;
                const FaceP fp = face_param(g, fl[k], side, na, nb);
                const int role = p.micro_role[side];
                if (role == TS_GAMMA_N) continue;
                const double kappa = role == TS_GAMMA_I ? p.kappa[1] : p.kappa[3];
                if (kappa == 0.0) continue;
                const double scale = face_scale(fp);
                const int a = pl[k];
                double loc0 = 0.0, loc1 = 0.0;
                for (int q = 0; q < 2; ++q) {
                    const double wq = cQ.GW[q] * kappa * frow[fl[k] * 2 + q].w * scale;
                    loc0 += wq * cQ.Nf[q][a] * cQ.Nf[q][0];
                    loc1 += wq * cQ.Nf[q][a] * cQ.Nf[q][1];
                }
                // neighbour of node along the face: node a -> node b
                const int other = a == 0 ? nb : na;
                const int oi = other % (g.n0 + 1), oj = other / (g.n0 + 1);
                const int dself = 4;
                const int doth = (oj - j + 1) * 3 + (oi - i + 1);
                acc_add(acc, a == 0 ? dself : doth, loc0);
                acc_add(acc, a == 0 ? doth : dself, loc1);
            }
        };

        bool faces_done = false;
        // adjacent cells in ascending index: (i-1,j-1), (i,j-1), (i-1,j), (i,j)
        for (int k = 0; k < 4; ++k) {
            const int ci = i - 1 + (k & 1), cj = j - 1 + (k >> 1);
            if (ci < 0 || ci >= g.n0 || cj < 0 || cj >= g.n1) continue;
            const int c = cj * g.n0 + ci;
            if (!faces_done && c >= 512) {  // faces are merged after cell chunk 0 (512 cells)
                add_faces();
                faces_done = true;
            }
            // corner index of (i,j) in cell (ci,cj): (0,0)->0, (1,0)->1, (1,1)->2, (0,1)->3
            const int di = i - ci, dj = j - cj;
            const int corner = dj == 0 ? di : (di == 1 ? 2 : 3);
            double loc[4] = {0.0, 0.0, 0.0, 0.0};
            for (int q = 0; q < 4; ++q) {
                const double4 e = crow[c * 4 + q];
                const double wq = cQ.QW[q] * det_elem * p.Dv;
                const double gax = cQ.dN[q][corner][0] * gx, gay = cQ.dN[q][corner][1] * gy;
                const double Agx = e.y * gax + e.z * gay;
                const double Agy = e.z * gax + e.w * gay;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const double gbx = cQ.dN[q][b][0] * gx, gby = cQ.dN[q][b][1] * gy;
                    loc[b] += wq * (Agx * gbx + Agy * gby);
                }
                if (react) {
                    double y0, y1;
                    cell_pt(g, c, cQ.QS[q], cQ.QT[q], y0, y1);
                    const double wr = cQ.QW[q] * det_elem * reaction_k(p, y0, y1) * e.x;
#pragma unroll
                    for (int b = 0; b < 4; ++b) loc[b] += wr * cQ.N[q][corner] * cQ.N[q][b];
                }
            }
            // acc[(bj - j + 1) * 3 + (bi - i + 1)] += loc[b] with a compile-time index per cell
            // position k (keeps the 9-entry row in registers instead of local memory)
            switch (k) {
                case 0: acc[0] += loc[0]; acc[1] += loc[1]; acc[4] += loc[2]; acc[3] += loc[3]; break;
                case 1: acc[1] += loc[0]; acc[2] += loc[1]; acc[5] += loc[2]; acc[4] += loc[3]; break;
                case 2: acc[3] += loc[0]; acc[4] += loc[1]; acc[7] += loc[2]; acc[6] += loc[3]; break;
                default: acc[4] += loc[0]; acc[5] += loc[1]; acc[8] += loc[2]; acc[7] += loc[3]; break;
            }
        }
        if (!faces_done) add_faces();
        double* out = stencil + (size_t)sys * 5 * n + node;  // upper half: C, E, NW, N, NE (dirs 4..8)
#pragma unroll
        for (int d = 4; d < 9; ++d) out[(size_t)(d - 4) * n] = acc[d];
    }
}

// build_micro_rhs_parts (assembly.cpp:176-231): thread = (macro node, micro node).
__global__ void k_rhs_parts(ProblemG p, int n_nodes, int cache_shared,
                            const double4* __restrict__ cells, const double4* __restrict__ faces,
                            double* fixed, double* rin, double* rout, int has_fixed, unsigned* err) {
    const GridG& g = p.micro;
    const int n = g.nodes(), ncell = g.cells(), nface = g.faces();
    const long long total = (long long)n_nodes * n;
    const double det_elem = 0.25 * g.h0 * g.h1;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int k = (int)(t % n);
        const int node = (int)(t / n);
        const int row = cache_shared ? 0 : node;
        double x0, x1;
        node_xy(p.macro, node, x0, x1);
        const int i = k % (g.n0 + 1), j = k / (g.n0 + 1);
        double fx = 0.0, ri = 0.0, ro = 0.0;
        if (has_fixed && p.data.fv_hat.n) {
            const double4* crow = cells + (size_t)row * ncell * 4;
            for (int kk = 0; kk < 4; ++kk) {
                const int ci = i - 1 + (kk & 1), cj = j - 1 + (kk >> 1);
                if (ci < 0 || ci >= g.n0 || cj < 0 || cj >= g.n1) continue;
                const int c = cj * g.n0 + ci;
                const int di = i - ci, dj = j - cj;
                const int corner = dj == 0 ? di : (di == 1 ? 2 : 3);
                for (int q = 0; q < 4; ++q) {
                    double y0, y1;
                    cell_pt(g, c, cQ.QS[q], cQ.QT[q], y0, y1);
                    const double fv = tape_eval(p.map.op, p.map.arg, p.map.val, p.data.fv_hat, x0, x1, y0, y1, err);
                    const double wq = cQ.QW[q] * det_elem * fv * crow[c * 4 + q].x;
                    fx += wq * cQ.N[q][corner];
                }
            }
        }
        int fl[4], pl[4];
        const int nf = node_faces(g, i, j, fl, pl);
        const double4* frow = faces + (size_t)row * nface * 2;
        for (int kk = 0; kk < nf; ++kk) {
            int side, na, nb;
            const FaceP fp = face_param(g, fl[kk], side, na, nb);
            const int role = p.micro_role[side];
            const double scale = face_scale(fp);
            const int a = pl[kk];
            for (int q = 0; q < 2; ++q) {
                const double w_meas = cQ.GW[q] * frow[fl[kk] * 2 + q].w * scale;
                if (role == TS_GAMMA_I)
                    ri += w_meas * cQ.Nf[q][a];
                else if (role == TS_GAMMA_O)
                    ro += w_meas * cQ.Nf[q][a];
                if (has_fixed && p.data.gv[side].n) {
                    const double y0 = fp.mx + fp.tx * cQ.GP[q], y1 = fp.my + fp.ty * cQ.GP[q];
                    const double gval = tape_eval(p.map.op, p.map.arg, p.map.val, p.data.gv[side], x0, x1, y0, y1, err);
                    fx += w_meas * gval * cQ.Nf[q][a];
                }
            }
        }
        if (has_fixed) fixed[t] = fx;
        rin[t] = ri;
        rout[t] = ro;
    }
}

__global__ void k_face_len(long long total, const double4* faces, double* len) {
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x)
        len[t] = faces[t].w;
}

// Per macro quadrature point: gamma_in/out, iterate-independent rhs integrands, D^w
// (assembly.cpp:237-281).  The face entries of the qpoint cache (assembly.cpp:69) are
// evaluated on the fly.
// Per macro quadrature point (assembly.cpp:244-276): gamma_in / gamma_out, the flux and
// g^v corrections of the macro rhs, f^u, f^w and D^w.  One block per quadrature point: the
// block's threads evaluate the micro face points (kernel (1) + data tapes) into shared
// memory, one thread then adds the per-point terms in the reference's order (faces
// ascending, q inner), so every sum is the serial loop's bits while the tape work is spread
// over the block.  Faces are handled in chunks of kMqChunk (face, q) points.
constexpr int kMqThreads = 128;
constexpr int kMqChunk = 512;

__global__ void __launch_bounds__(kMqThreads) k_macro_qpoints(ProblemG p, double* gamma_in, double* gamma_out,
                                                              double* rhs_u_q, double* rhs_w_q, double* dw_q,
                                                              unsigned long long* first_bad, unsigned* err) {
    __shared__ double s_len[kMqChunk], s_flux[kMqChunk], s_corr[kMqChunk];
    __shared__ signed char s_role[kMqChunk];
    __shared__ double s_scalar[3];
    const GridG& M = p.macro;
    const GridG& g = p.micro;
    const int nq_total = M.cells() * 4;
    const int npts = g.faces() * 2;
    const int* op = p.map.op;
    const int* arg = p.map.arg;
    const double* val = p.map.val;
    for (int qg = blockIdx.x; qg < nq_total; qg += gridDim.x) {
        double x0, x1;
        cell_pt(M, qg >> 2, cQ.QS[qg & 3], cQ.QT[qg & 3], x0, x1);
        if (threadIdx.x < 3) {  // f^u, f^w, D^w at the macro point (tapes in x only)
            const TapeRef t = threadIdx.x == 0 ? p.data.fu : threadIdx.x == 1 ? p.data.fw : p.data.Dw;
            s_scalar[threadIdx.x] = tape_eval(op, arg, val, t, x0, x1, 0.0, 0.0, err);
        }
        double g_in = 0.0, g_out = 0.0, flux_u = 0.0, flux_w = 0.0, corr_u = 0.0, corr_w = 0.0;
        for (int c0 = 0; c0 < npts; c0 += kMqChunk) {
            const int cn = min(kMqChunk, npts - c0);
            for (int k = threadIdx.x; k < cn; k += kMqThreads) {
                const int f = (c0 + k) >> 1, q = (c0 + k) & 1;
                int side, a, b;
                const FaceP fp = face_param(g, f, side, a, b);
                const int role = p.micro_role[side];
                const double y0 = fp.mx + fp.tx * cQ.GP[q], y1 = fp.my + fp.ty * cQ.GP[q];
                double4 e;
                if (!face_coef(p.map, -1, x0, x1, y0, y1, fp.nx, fp.ny, e, err))
                    atomicMin(first_bad, (unsigned long long)qg * npts + f * 2 + q);
                const double w = cQ.GW[q] * face_scale(fp);
                const double len = w * e.w;
                double flux = 0.0, corr = 0.0;
                const bool in = role == TS_GAMMA_I, out = role == TS_GAMMA_O;
                if ((in && p.data.has_fu_flux) || (out && p.data.has_fw_flux)) {
                    const TapeRef* fl = in ? p.data.fu_flux : p.data.fw_flux;
                    flux = w * (tape_eval(op, arg, val, fl[0], x0, x1, y0, y1, err) * e.y +
                                tape_eval(op, arg, val, fl[1], x0, x1, y0, y1, err) * e.z);
                }
                if ((in || out) && p.data.gv[side].n)
                    corr = len * tape_eval(op, arg, val, p.data.gv[side], x0, x1, y0, y1, err);
                s_len[k] = len;
                s_flux[k] = flux;
                s_corr[k] = corr;
                s_role[k] = (signed char)role;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                // adding the +0.0 of absent terms leaves a sum that started at +0.0 unchanged
                for (int k = 0; k < cn; ++k) {
                    if (s_role[k] == TS_GAMMA_I) {
                        g_in += s_len[k];
                        flux_u += s_flux[k];
                        corr_u += s_corr[k];
                    } else if (s_role[k] == TS_GAMMA_O) {
                        g_out += s_len[k];
                        flux_w += s_flux[k];
                        corr_w += s_corr[k];
                    }
                }
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            gamma_in[qg] = g_in;
            gamma_out[qg] = g_out;
            rhs_u_q[qg] = s_scalar[0] + flux_u - corr_u;
            rhs_w_q[qg] = s_scalar[1] + flux_w - corr_w;
            dw_q[qg] = s_scalar[2];
        }
        __syncthreads();
    }
}

// Macro cell loop (assembly.cpp:287-320) + Neumann boundary terms (323-342) as a
// gather over the <= 4 cells / 2 faces of each macro node, in the reference order.
__global__ void k_macro_assemble(ProblemG p, const int* row_ptr, const double* gamma_in,
                                 const double* gamma_out, const double* rhs_u_q,
                                 const double* rhs_w_q, const double* dw_q, double* Au, double* Aw,
                                 double* M0, double* bu_out, double* bw_out, unsigned* err) {
    const GridG& M = p.macro;
    const int n = M.nodes();
    const double det_elem = 0.25 * M.h0 * M.h1;
    const double gx = 2.0 / M.h0, gy = 2.0 / M.h1;
    for (int node = blockIdx.x * blockDim.x + threadIdx.x; node < n; node += gridDim.x * blockDim.x) {
        const int i = node % (M.n0 + 1), j = node / (M.n0 + 1);
        double au[9], aw[9], am[9];
#pragma unroll
        for (int d = 0; d < 9; ++d) au[d] = aw[d] = am[d] = 0.0;
        double bu = 0.0, bw = 0.0;
        for (int k = 0; k < 4; ++k) {
            const int ci = i - 1 + (k & 1), cj = j - 1 + (k >> 1);
            if (ci < 0 || ci >= M.n0 || cj < 0 || cj >= M.n1) continue;
            const int c = cj * M.n0 + ci;
            const int di = i - ci, dj = j - cj;
            const int a = dj == 0 ? di : (di == 1 ? 2 : 3);
            double lu[4] = {0, 0, 0, 0}, lw[4] = {0, 0, 0, 0}, lm[4] = {0, 0, 0, 0}, lbu = 0.0, lbw = 0.0;
            for (int q = 0; q < 4; ++q) {
                const int qg = c * 4 + q;
                const double wq = cQ.QW[q] * det_elem;
                const double mass_u = p.kappa[0] * gamma_in[qg];
                const double mass_w = p.kappa[2] * gamma_out[qg];
                const double dw = dw_q[qg];
                const double gax = cQ.dN[q][a][0] * gx, gay = cQ.dN[q][a][1] * gy;
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const double gbx = cQ.dN[q][b][0] * gx, gby = cQ.dN[q][b][1] * gy;
                    const double stiff = gax * gbx + gay * gby;
                    const double mass = cQ.N[q][a] * cQ.N[q][b];
                    lu[b] += wq * (stiff + mass_u * mass);
                    lw[b] += wq * (dw * stiff + mass_w * mass);
                    lm[b] += wq * mass;
                }
                lbu += wq * rhs_u_q[qg] * cQ.N[q][a];
                lbw += wq * rhs_w_q[qg] * cQ.N[q][a];
            }
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                const int bi = ci + kCornerDi[b], bj = cj + kCornerDj[b];
                const int d = (bj - j + 1) * 3 + (bi - i + 1);
                au[d] += lu[b];
                aw[d] += lw[b];
                am[d] += lm[b];
            }
            bu += lbu;
            bw += lbw;
        }
        // Neumann data (assembly.cpp:323-342), faces ascending
        int fl[4], pl[4];
        const int nf = node_faces(M, i, j, fl, pl);
        const int* op = p.map.op;
        const int* arg = p.map.arg;
        const double* val = p.map.val;
        for (int k = 0; k < nf; ++k) {
            int side, na, nb;
            const FaceP fp = face_param(M, fl[k], side, na, nb);
            const bool u_neu = p.macro_bc[side] == TS_NEUMANN;
            const bool has_u = u_neu && p.data.gu2[side].n;
            const bool has_w = p.data.gw[side].n != 0;
            if (!has_u && !has_w) continue;
            const double scale = face_scale(fp);
            for (int q = 0; q < 2; ++q) {
                const double x0 = fp.mx + fp.tx * cQ.GP[q], x1 = fp.my + fp.ty * cQ.GP[q];
                const double w = cQ.GW[q] * scale;
                if (has_u) bu += w * tape_eval(op, arg, val, p.data.gu2[side], x0, x1, 0, 0, err) * cQ.Nf[q][pl[k]];
                if (has_w) bw += w * tape_eval(op, arg, val, p.data.gw[side], x0, x1, 0, 0, err) * cQ.Nf[q][pl[k]];
            }
        }
        int kk = row_ptr[node];
        for (int d = 0; d < 9; ++d) {
            const int di = d % 3 - 1, dj = d / 3 - 1;
            if (i + di < 0 || i + di > M.n0 || j + dj < 0 || j + dj > M.n1) continue;
            Au[kk] = au[d];
            Aw[kk] = aw[d];
            M0[kk] = am[d];
            ++kk;
        }
        bu_out[node] = bu;
        bw_out[node] = bw;
    }
}

__global__ void k_dirichlet_values(ProblemG p, int n, const int* dofs, double* vals, unsigned* err) {
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        double x0, x1;
        node_xy(p.macro, dofs[k], x0, x1);
        vals[k] = tape_eval(p.map.op, p.map.arg, p.map.val, p.data.dirichlet_value, x0, x1, 0, 0, err);
    }
}

__global__ void k_eliminate(int n, const int* row_ptr, const int* col_idx, const double* A,
                            const unsigned char* cmask, const double* cval, double* A_e,
                            double* shift) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
        double s = 0.0;
        for (int k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
            const int c = col_idx[k];
            s += A[k] * (cmask[c] ? cval[c] : 0.0);  // A_orig * g_ext (solver.cpp:22-24)
            if (cmask[r])
                A_e[k] = (c == r) ? 1.0 : 0.0;      // linalg.cpp:66-69
            else
                A_e[k] = cmask[c] ? 0.0 : A[k];      // linalg.cpp:70-76
        }
        shift[r] = s;
    }
}

int grid_for(long long total) {
    long long b = (total + kThreads - 1) / kThreads;
    if (b > 148LL * 64) b = 148LL * 64;
    if (b < 1) b = 1;
    return (int)b;
}

}  // namespace

// min / max of det J over a strided array of cache entries (first double of each entry);
// per-block results {min, argmin, max, argmax} in out[block*4 .. +3].
// value t = e[(t / blk) * bstride + (t % blk) * stride] (blk = count: one strided run)
__global__ void k_det_minmax(const double* e, long long count, int stride, long long blk, long long bstride,
                             double* out) {
    __shared__ double smin[256], smax[256];
    __shared__ long long imin[256], imax[256];
    double mn = 1e300, mx = -1e300;
    long long an = -1, ax = -1;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < count; t += (long long)gridDim.x * blockDim.x) {
        const double v = e[(t / blk) * bstride + (t % blk) * stride];
        if (v < mn) { mn = v; an = t; }
        if (v > mx) { mx = v; ax = t; }
    }
    smin[threadIdx.x] = mn; imin[threadIdx.x] = an;
    smax[threadIdx.x] = mx; imax[threadIdx.x] = ax;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            const int j = threadIdx.x + o;
            if (smin[j] < smin[threadIdx.x] || (smin[j] == smin[threadIdx.x] && imin[j] >= 0 && imin[j] < imin[threadIdx.x])) {
                smin[threadIdx.x] = smin[j]; imin[threadIdx.x] = imin[j];
            }
            if (smax[j] > smax[threadIdx.x] || (smax[j] == smax[threadIdx.x] && imax[j] >= 0 && imax[j] < imax[threadIdx.x])) {
                smax[threadIdx.x] = smax[j]; imax[threadIdx.x] = imax[j];
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[blockIdx.x * 4 + 0] = smin[0];
        out[blockIdx.x * 4 + 1] = (double)imin[0];
        out[blockIdx.x * 4 + 2] = smax[0];
        out[blockIdx.x * 4 + 3] = (double)imax[0];
    }
}

void launch_det_minmax(const double* e, long long count, int stride, double* out, int blocks, cudaStream_t s,
                       long long blk, long long bstride) {
    if (blk <= 0) blk = count > 0 ? count : 1;
    k_det_minmax<<<blocks, 256, 0, s>>>(e, count, stride, blk, bstride, out);
}

void launch_cell_cache(const ProblemG& p, int rows, const double* points, double4* cells,
                       unsigned long long* first_bad, unsigned* err, cudaStream_t s, int row0) {
    const long long total = (long long)rows * p.micro.cells() * 4;
    k_cell_cache<<<grid_for(total), kThreads, 0, s>>>(p, rows, points, cells, first_bad, err, row0);
}

void launch_face_cache(const ProblemG& p, int rows, const double* points, int with_cells,
                       double4* faces, unsigned long long* first_bad, unsigned* err, cudaStream_t s, int row0) {
    const long long total = (long long)rows * p.micro.faces() * 2;
    k_face_cache<<<grid_for(total), kThreads, 0, s>>>(p, rows, points, with_cells, faces, first_bad, err, row0);
}

int launch_validate_pairs(const MapG& m, const double* xs, int nx, const double* ys, int ny, double* part,
                          unsigned* err, cudaStream_t s) {
    const long long total = (long long)nx * ny;
    const int blocks = (int)std::max(1LL, std::min<long long>(148LL * 8, (total + kValThreads - 1) / kValThreads));
    k_validate_pairs<<<blocks, kValThreads, 0, s>>>(m, xs, nx, ys, ny, part, err);
    return blocks;
}

void launch_boundary_measures(const GridG& micro, const int* role, int n, const double* nu, int stride, int offset,
                              double* gamma, cudaStream_t s) {
    if (n > 0)
        k_boundary_measures<<<(n + 127) / 128, 128, 0, s>>>(micro, make_int4(role[0], role[1], role[2], role[3]), n,
                                                             nu, stride, offset, gamma);
}

void launch_tape_at_points(const int* op, const int* arg, const double* val, TapeRef t, int n,
                           const double* points, double* out, unsigned* err, cudaStream_t s) {
    if (n > 0) k_tape_at_points<<<(n + 127) / 128, 128, 0, s>>>(op, arg, val, t, n, points, out, err);
}

void launch_degenerate_probe(const ProblemG& p, const double* points, int with_cells,
                             unsigned long long index, double* out, cudaStream_t s) {
    k_probe<<<1, 1, 0, s>>>(p, points, with_cells, index, out);
}

void launch_assemble_micro(const ProblemG& p, int srows, const double4* cells, const double4* faces,
                           double* stencil, cudaStream_t s) {
    const long long total = (long long)srows * p.micro.nodes();
    k_assemble_micro<<<grid_for(total), kThreads, 0, s>>>(p, srows, cells, faces, stencil);
}

void launch_rhs_parts(const ProblemG& p, int n_nodes, int cache_shared, const double4* cells,
                      const double4* faces, double* fixed, double* rin, double* rout, int has_fixed,
                      unsigned* err, cudaStream_t s) {
    const long long total = (long long)n_nodes * p.micro.nodes();
    k_rhs_parts<<<grid_for(total), kThreads, 0, s>>>(p, n_nodes, cache_shared, cells, faces, fixed,
                                                     rin, rout, has_fixed, err);
}

void launch_face_len(int rows, int n_faces, const double4* faces, double* len, cudaStream_t s) {
    const long long total = (long long)rows * n_faces * 2;
    k_face_len<<<grid_for(total), kThreads, 0, s>>>(total, faces, len);
}

void launch_macro_qpoints(const ProblemG& p, double* gamma_in, double* gamma_out, double* rhs_u_q,
                          double* rhs_w_q, double* dw_q, unsigned long long* first_bad,
                          unsigned* err, cudaStream_t s) {
    const int total = p.macro.cells() * 4;
    k_macro_qpoints<<<std::min(total, 148 * 16), kMqThreads, 0, s>>>(p, gamma_in, gamma_out, rhs_u_q, rhs_w_q,
                                                                     dw_q, first_bad, err);
}

void launch_macro_assemble(const ProblemG& p, const int* row_ptr, const double* gamma_in,
                           const double* gamma_out, const double* rhs_u_q, const double* rhs_w_q,
                           const double* dw_q, double* Au, double* Aw, double* M0, double* bu,
                           double* bw, unsigned* err, cudaStream_t s) {
    k_macro_assemble<<<grid_for(p.macro.nodes()), kThreads, 0, s>>>(p, row_ptr, gamma_in, gamma_out,
                                                                     rhs_u_q, rhs_w_q, dw_q, Au, Aw,
                                                                     M0, bu, bw, err);
}

void launch_dirichlet_values(const ProblemG& p, int n, const int* dofs, double* vals, unsigned* err,
                             cudaStream_t s) {
    if (n <= 0) return;
    k_dirichlet_values<<<grid_for(n), kThreads, 0, s>>>(p, n, dofs, vals, err);
}

void launch_eliminate(int n, const int* row_ptr, const int* col_idx, const double* A,
                      const unsigned char* cmask, const double* cval, double* A_e, double* shift,
                      cudaStream_t s) {
    k_eliminate<<<grid_for(n), kThreads, 0, s>>>(n, row_ptr, col_idx, A, cmask, cval, A_e, shift);
}

}  // namespace tsb
