// Dimension/order-generic micro geometry for BASELINE configs 4 (Q2 micro) and 5
// (3D Q1 micro): tensor-product Lagrange elements of order p on a d-dimensional box,
// the same conventions as the generic oracle (oracle/twoscale_oracle_gen.c):
// lattice spacing h/p, element-local nodes and quadrature lexicographic (axis 0
// fastest), Gauss-(p+1) rules, boundary faces ordered by axis, transverse cell
// index, then side (for d = 2 this is the reference order, grid.cpp:34-45).
#pragma once

#include "device_common.cuh"

namespace tsb {

constexpr int kGenMaxQ = 27;   // (p+1)^d element nodes / cell quadrature points
constexpr int kGenMaxFQ = 9;   // (p+1)^(d-1) face nodes / face quadrature points
constexpr int kGenMaxDirs = 27;

struct GenGeom {
    int d, p;
    double lo[3], hi[3], h[3], hp[3];
    int nc[3], nn[3];
    int nnodes, ncells, nfaces, npe, npf, nq, nqf, ndirs;
    int face_off[4];
};

struct GenTables {
    double W[kGenMaxQ], S[kGenMaxQ][3];
    double N[kGenMaxQ][kGenMaxQ], dN[kGenMaxQ][kGenMaxQ][3];
    double FW[kGenMaxFQ], FT[kGenMaxFQ][2], Nf[kGenMaxFQ][kGenMaxFQ];
};

struct GenMap {
    int kind;  // TS_MAP_TAPE (2D only), TS_MAP_AFFINE_BUBBLE_TABLE, TS_MAP_FOURIER_TABLE (2D)
    const int* op;
    const int* arg;
    const double* val;
    TapeRef jac[4];
    const double* table;
    int tstride;
    int s_kind;
    double amp;
    GridG macro;
    double D[9];
    int D_identity;
};

__host__ __device__ __forceinline__ int gen_node(const GenGeom& g, int i0, int i1, int i2) {
    return g.d == 2 ? i0 + g.nn[0] * i1 : i0 + g.nn[0] * (i1 + g.nn[1] * i2);
}

__host__ __device__ __forceinline__ void gen_node_idx(const GenGeom& g, int n, int* ii) {
    ii[0] = n % g.nn[0];
    ii[1] = (n / g.nn[0]) % g.nn[1];
    ii[2] = g.d == 3 ? n / (g.nn[0] * g.nn[1]) : 0;
}

__host__ __device__ __forceinline__ double gen_coord(const GenGeom& g, int a, int i) {
    return TS_ADD(g.lo[a], TS_MUL((double)i, g.hp[a]));
}

__host__ __device__ __forceinline__ void gen_cell_idx(const GenGeom& g, int c, int* cc) {
    cc[0] = c % g.nc[0];
    cc[1] = (c / g.nc[0]) % g.nc[1];
    cc[2] = g.d == 3 ? c / (g.nc[0] * g.nc[1]) : 0;
}

__host__ __device__ __forceinline__ int gen_cell(const GenGeom& g, const int* cc) {
    return g.d == 2 ? cc[0] + g.nc[0] * cc[1] : cc[0] + g.nc[0] * (cc[1] + g.nc[1] * cc[2]);
}

// Face f -> axis, side (0 = minus, 1 = plus), cell coordinates, transverse axes.
__host__ __device__ __forceinline__ void gen_face(const GenGeom& g, int f, int& axis, int& side, int* cc,
                                                  int* tr) {
    axis = 0;
    while (axis < g.d - 1 && f >= g.face_off[axis + 1]) ++axis;
    const int idx = f - g.face_off[axis];
    side = idx & 1;
    const int t = idx >> 1;
    int nt = 0;
    for (int k = 0; k < g.d; ++k)
        if (k != axis) tr[nt++] = k;
    if (g.d == 2) tr[1] = tr[0];
    cc[tr[0]] = t % g.nc[tr[0]];
    if (g.d == 3) cc[tr[1]] = t / g.nc[tr[0]];
    cc[axis] = side ? g.nc[axis] - 1 : 0;
}

// Lattice node of face-local node fa.
__host__ __device__ __forceinline__ int gen_face_node(const GenGeom& g, int axis, int side, const int* cc,
                                                      const int* tr, int fa) {
    int ii[3] = {0, 0, 0};
    const int q1 = g.p + 1;
    ii[axis] = side ? g.nn[axis] - 1 : 0;
    ii[tr[0]] = g.p * cc[tr[0]] + fa % q1;
    if (g.d == 3) ii[tr[1]] = g.p * cc[tr[1]] + fa / q1;
    return gen_node(g, ii[0], ii[1], ii[2]);
}

// Face quadrature point q (y[3]), the face scale (product of half extents) and normal.
__host__ __device__ __forceinline__ void gen_face_geom(const GenGeom& g, const GenTables& T, int axis, int side,
                                                       const int* cc, int q, double* y, double& scale,
                                                       double* nrm) {
    double sc = 1.0;
    int t = 0;
    for (int k = 0; k < g.d; ++k) {
        nrm[k] = 0.0;
        if (k == axis) {
            y[k] = side ? gen_coord(g, k, g.nn[k] - 1) : g.lo[k];
            continue;
        }
        const double x0 = gen_coord(g, k, g.p * cc[k]), x1 = gen_coord(g, k, g.p * (cc[k] + 1));
        const double mid = TS_MUL(0.5, TS_ADD(x0, x1)), tan = TS_MUL(0.5, TS_SUB(x1, x0));
        y[k] = TS_ADD(mid, TS_MUL(T.FT[q][t], tan));
        sc = TS_MUL(sc, tan);
        ++t;
    }
    nrm[axis] = side ? 1.0 : -1.0;
    scale = g.d == 2 ? sqrt(TS_MUL(sc, sc)) : sc;
}

__host__ __device__ __forceinline__ void gen_cell_qpoint(const GenGeom& g, const GenTables& T, const int* cc,
                                                         int q, double* y) {
    for (int k = 0; k < g.d; ++k)
        y[k] = TS_ADD(TS_ADD(g.lo[k], TS_MUL(cc[k] + 0.5, g.h[k])), TS_MUL(TS_MUL(0.5, g.h[k]), T.S[q][k]));
}

}  // namespace tsb
