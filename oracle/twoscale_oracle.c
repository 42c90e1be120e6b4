/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference's micro-solve path.
 * See twoscale_oracle.h for scope.  Each routine cites the reference file:line it
 * restates (paths relative to /root/reference/proj).  Compiled with
 * -ffp-contract=off so that, like the reference's x86-64 -O3 build (no -march, so
 * no FMA), every product and sum is rounded separately and in the same order. */
#define _GNU_SOURCE
#include "twoscale_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static __thread char g_err[512];

const char* or_last_error(void) { return g_err; }

/* ------------------------------------------------------------------ grid ---- */
/* grid.cpp:28-70 — lexicographic nodes, CCW cells, faces L,R per row then B,T. */
typedef struct {
    double lo[2], hi[2], h[2];
    int n[2];
    int n_faces;
    int* face_side;  /* 0 L, 1 R, 2 B, 3 T */
    int* face_nodes; /* 2 per face */
} grid_t;

static int node_index(const grid_t* g, int i, int j) { return j * (g->n[0] + 1) + i; }
static int node_count(const grid_t* g) { return (g->n[0] + 1) * (g->n[1] + 1); }
static int cell_count(const grid_t* g) { return g->n[0] * g->n[1]; }

static void grid_init(grid_t* g, const double lo[2], const double hi[2], const int n[2]) {
    for (int a = 0; a < 2; ++a) {
        g->lo[a] = lo[a];
        g->hi[a] = hi[a];
        g->n[a] = n[a];
        g->h[a] = (hi[a] - lo[a]) / n[a]; /* grid.cpp:31-32 */
    }
    g->n_faces = 2 * n[1] + 2 * n[0];
    g->face_side = malloc(sizeof(int) * g->n_faces);
    g->face_nodes = malloc(sizeof(int) * 2 * g->n_faces);
    int f = 0;
    for (int cj = 0; cj < n[1]; ++cj) { /* grid.cpp:34-38 */
        g->face_side[f] = 0;
        g->face_nodes[2 * f] = node_index(g, 0, cj);
        g->face_nodes[2 * f + 1] = node_index(g, 0, cj + 1);
        ++f;
        g->face_side[f] = 1;
        g->face_nodes[2 * f] = node_index(g, n[0], cj);
        g->face_nodes[2 * f + 1] = node_index(g, n[0], cj + 1);
        ++f;
    }
    for (int ci = 0; ci < n[0]; ++ci) { /* grid.cpp:39-44 */
        g->face_side[f] = 2;
        g->face_nodes[2 * f] = node_index(g, ci, 0);
        g->face_nodes[2 * f + 1] = node_index(g, ci + 1, 0);
        ++f;
        g->face_side[f] = 3;
        g->face_nodes[2 * f] = node_index(g, ci, n[1]);
        g->face_nodes[2 * f + 1] = node_index(g, ci + 1, n[1]);
        ++f;
    }
}

static void grid_free(grid_t* g) {
    free(g->face_side);
    free(g->face_nodes);
}

static void grid_node(const grid_t* g, int idx, double* p) { /* grid.cpp:47-52 */
    const int i = idx % (g->n[0] + 1), j = idx / (g->n[0] + 1);
    p[0] = g->lo[0] + i * g->h[0];
    p[1] = g->lo[1] + j * g->h[1];
}

static void cell_nodes(const grid_t* g, int c, int* nd) { /* grid.cpp:54-59 */
    const int ci = c % g->n[0], cj = c / g->n[0];
    nd[0] = node_index(g, ci, cj);
    nd[1] = node_index(g, ci + 1, cj);
    nd[2] = node_index(g, ci + 1, cj + 1);
    nd[3] = node_index(g, ci, cj + 1);
}

static void cell_point(const grid_t* g, int c, double s, double t, double* p) { /* grid.cpp:61-71 */
    const int ci = c % g->n[0], cj = c / g->n[0];
    const double mx = g->lo[0] + (ci + 0.5) * g->h[0];
    const double my = g->lo[1] + (cj + 0.5) * g->h[1];
    p[0] = mx + 0.5 * g->h[0] * s;
    p[1] = my + 0.5 * g->h[1] * t;
}

typedef struct {
    double mid[2], tan[2], nrm[2];
} faceparam_t;

static faceparam_t face_param(const grid_t* g, int f) { /* grid.cpp:121-127 */
    double a[2], b[2];
    grid_node(g, g->face_nodes[2 * f], a);
    grid_node(g, g->face_nodes[2 * f + 1], b);
    faceparam_t fp;
    fp.mid[0] = 0.5 * (a[0] + b[0]);
    fp.mid[1] = 0.5 * (a[1] + b[1]);
    fp.tan[0] = 0.5 * (b[0] - a[0]);
    fp.tan[1] = 0.5 * (b[1] - a[1]);
    static const double normals[4][2] = {{-1, 0}, {1, 0}, {0, -1}, {0, 1}}; /* grid.cpp:18-26 */
    fp.nrm[0] = normals[g->face_side[f]][0];
    fp.nrm[1] = normals[g->face_side[f]][1];
    return fp;
}

static double face_scale(const faceparam_t* fp) { /* Vec2::norm, linalg.hpp:19 */
    return sqrt(fp->tan[0] * fp->tan[0] + fp->tan[1] * fp->tan[1]);
}

/* Gauss-2 (grid.cpp:134-141, 170-177): points +-1/sqrt(3), weights 1, i fastest. */
static double GP[2], GW[2];
static double QS[4], QT[4], QW[4];
static double SHN[4][4], SHG[4][4][2], SHF[2][2];

static void rule_init(void) {
    const double gq = 1.0 / sqrt(3.0);
    GP[0] = -gq;
    GP[1] = gq;
    GW[0] = 1.0;
    GW[1] = 1.0;
    for (int j = 0; j < 2; ++j)
        for (int i = 0; i < 2; ++i) {
            QS[j * 2 + i] = GP[i];
            QT[j * 2 + i] = GP[j];
            QW[j * 2 + i] = GW[i] * GW[j];
        }
    for (int q = 0; q < 4; ++q) { /* shape_eval / shape_grad, grid.cpp:109-119 */
        const double s = QS[q], t = QT[q];
        SHN[q][0] = 0.25 * (1.0 - s) * (1.0 - t);
        SHN[q][1] = 0.25 * (1.0 + s) * (1.0 - t);
        SHN[q][2] = 0.25 * (1.0 + s) * (1.0 + t);
        SHN[q][3] = 0.25 * (1.0 - s) * (1.0 + t);
        SHG[q][0][0] = -0.25 * (1.0 - t);
        SHG[q][0][1] = -0.25 * (1.0 - s);
        SHG[q][1][0] = 0.25 * (1.0 - t);
        SHG[q][1][1] = -0.25 * (1.0 + s);
        SHG[q][2][0] = 0.25 * (1.0 + t);
        SHG[q][2][1] = 0.25 * (1.0 + s);
        SHG[q][3][0] = -0.25 * (1.0 + t);
        SHG[q][3][1] = 0.25 * (1.0 - s);
    }
    for (int q = 0; q < 2; ++q) { /* face_shape, grid.hpp:83-85 */
        SHF[q][0] = 0.5 * (1.0 - GP[q]);
        SHF[q][1] = 0.5 * (1.0 + GP[q]);
    }
}

/* ------------------------------------------------------------------- CSR ---- */
typedef struct {
    int n, nnz;
    int* rp;
    int* ci;
} pattern_t;

/* make_q1_matrix (assembly.cpp:34-50) + CsrMatrix ctor (linalg.cpp:8-18) */
static void q1_pattern(const grid_t* g, pattern_t* P) {
    const int n0 = g->n[0], n1 = g->n[1];
    P->n = node_count(g);
    P->rp = malloc(sizeof(int) * (P->n + 1));
    P->ci = malloc(sizeof(int) * 9 * P->n);
    int k = 0;
    P->rp[0] = 0;
    for (int j = 0; j <= n1; ++j)
        for (int i = 0; i <= n0; ++i) {
            for (int dj = -1; dj <= 1; ++dj) {
                if (j + dj < 0 || j + dj > n1) continue;
                for (int di = -1; di <= 1; ++di) {
                    if (i + di < 0 || i + di > n0) continue;
                    P->ci[k++] = node_index(g, i + di, j + dj);
                }
            }
            P->rp[node_index(g, i, j) + 1] = k;
        }
    P->nnz = k;
}

static int csr_find(const int* rp, const int* ci, int row, int col) { /* linalg.cpp:22-27 */
    int lo = rp[row], hi = rp[row + 1];
    while (lo < hi) {
        const int mid = (lo + hi) / 2;
        if (ci[mid] < col)
            lo = mid + 1;
        else
            hi = mid;
    }
    return (lo < rp[row + 1] && ci[lo] == col) ? lo : -1;
}

static void csr_apply(int n, const int* rp, const int* ci, const double* v, const double* x,
                      double* y) { /* linalg.cpp:40-47 */
    for (int r = 0; r < n; ++r) {
        double s = 0.0;
        for (int k = rp[r]; k < rp[r + 1]; ++k) s += v[k] * x[ci[k]];
        y[r] = s;
    }
}

static double norm2(const double* v, int n) { /* linalg.cpp:93-97 */
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += v[i] * v[i];
    return sqrt(s);
}

/* cg_solve (linalg.cpp:103-161), op order preserved. */
int or_cg_solve(int n, const int* rp, const int* ci, const double* A, const double* b, double* x,
                double tol, int maxit, int* res, double* resid) {
    res[0] = 0;
    res[1] = 0;
    res[2] = 0;
    *resid = 0.0;
    const double bnorm = norm2(b, n);
    if (bnorm == 0.0) {
        memset(x, 0, sizeof(double) * n);
        res[0] = 1;
        return 0;
    }
    double* inv_diag = malloc(sizeof(double) * n * 5);
    double *r = inv_diag + n, *z = r + n, *p = z + n, *Ap = p + n;
    for (int i = 0; i < n; ++i) {
        const int k = csr_find(rp, ci, i, i);
        const double d = k < 0 ? 0.0 : A[k];
        inv_diag[i] = (d != 0.0) ? 1.0 / d : 1.0;
    }
    csr_apply(n, rp, ci, A, x, Ap);
    for (int i = 0; i < n; ++i) r[i] = b[i] - Ap[i];
    for (int i = 0; i < n; ++i) z[i] = inv_diag[i] * r[i];
    memcpy(p, z, sizeof(double) * n);
    double rz = 0.0;
    for (int i = 0; i < n; ++i) rz += r[i] * z[i];
    double rnorm = norm2(r, n);
    *resid = rnorm / bnorm;
    if (*resid <= tol) {
        res[0] = 1;
        free(inv_diag);
        return 0;
    }
    for (int it = 1; it <= maxit; ++it) {
        csr_apply(n, rp, ci, A, p, Ap);
        double pAp = 0.0;
        for (int i = 0; i < n; ++i) pAp += p[i] * Ap[i];
        if (pAp <= 0.0) {
            res[2] = 1;
            res[1] = it;
            free(inv_diag);
            return 0;
        }
        const double alpha = rz / pAp;
        for (int i = 0; i < n; ++i) x[i] += alpha * p[i];
        for (int i = 0; i < n; ++i) r[i] -= alpha * Ap[i];
        rnorm = norm2(r, n);
        res[1] = it;
        *resid = rnorm / bnorm;
        if (*resid <= tol) {
            res[0] = 1;
            free(inv_diag);
            return 0;
        }
        for (int i = 0; i < n; ++i) z[i] = inv_diag[i] * r[i];
        double rz_new = 0.0;
        for (int i = 0; i < n; ++i) rz_new += r[i] * z[i];
        const double beta = rz_new / rz;
        rz = rz_new;
        for (int i = 0; i < n; ++i) p[i] = z[i] + beta * p[i];
    }
    free(inv_diag);
    return 0;
}

/* ------------------------------------------------------------------- ctx ---- */
struct or_ctx {
    or_problem p;
    double* A_table; /* owned copy */
    grid_t macro, micro;
    pattern_t mp, Mp; /* micro / macro patterns */
    int D_identity;
    /* per-node robin parts (lazily built) and matrices (lazily built) */
    double* robin_in;
    double* robin_out;
    double* micro_vals;
    /* per-node face |nu| (for coupling) */
    double* node_face_len; /* [n_macro][faces][2] */
    /* macro systems */
    double *Au, *Aw, *M0, *bu, *bw;
    int n_dir_u;
    int* dir_u;
    double* dir_u_val;
    int w_pinned;
};

static double s_of_x(const or_problem* p, double x0, double x1) {
    const double tp = 2.0 * 3.141592653589793;
    switch (p->s_kind) {
        case OR_S_SINCOS: return sin(tp * x0) * cos(tp * x1);
        case OR_S_PRODUCT: return x0 * x1;
        default: return 0.0;
    }
}

/* A(x): node index >= 0 uses the table row directly; otherwise bilinear interpolation
 * of the nodal table on the macro grid (decision recorded in DESIGN.md). */
static void A_of_x(const or_ctx* c, int node, double x0, double x1, double* A) {
    const or_problem* p = &c->p;
    if (p->A_kind == OR_A_IDENTITY) {
        A[0] = 1.0; A[1] = 0.0; A[2] = 0.0; A[3] = 1.0;
    } else if (p->A_kind == OR_A_TRIG) {
        const double tp = 2.0 * 3.141592653589793;
        A[0] = 1.0 + p->A_eps * sin(tp * x0);
        A[1] = p->A_eps * cos(tp * x1);
        A[2] = p->A_eps * cos(tp * x0);
        A[3] = 1.0 + p->A_eps * sin(tp * x1);
    } else if (node >= 0) {
        memcpy(A, c->A_table + 4 * (size_t)node, 4 * sizeof(double));
    } else {
        const grid_t* g = &c->macro;
        double fx = (x0 - g->lo[0]) / g->h[0], fy = (x1 - g->lo[1]) / g->h[1];
        int ci = (int)floor(fx), cj = (int)floor(fy);
        if (ci < 0) ci = 0;
        if (ci > g->n[0] - 1) ci = g->n[0] - 1;
        if (cj < 0) cj = 0;
        if (cj > g->n[1] - 1) cj = g->n[1] - 1;
        const double s = fx - ci, t = fy - cj;
        const double* T00 = c->A_table + 4 * (size_t)node_index(g, ci, cj);
        const double* T10 = c->A_table + 4 * (size_t)node_index(g, ci + 1, cj);
        const double* T11 = c->A_table + 4 * (size_t)node_index(g, ci + 1, cj + 1);
        const double* T01 = c->A_table + 4 * (size_t)node_index(g, ci, cj + 1);
        for (int k = 0; k < 4; ++k)
            A[k] = (1.0 - s) * (1.0 - t) * T00[k] + s * (1.0 - t) * T10[k] + s * t * T11[k] +
                   (1.0 - s) * t * T01[k];
    }
}

/* grad_y zeta for zeta = A(x) y + amp s(x) beta(y) (1,1). */
static void jac_eval(const or_ctx* c, int node, double x0, double x1, double y0, double y1,
                     double* F) {
    double A[4];
    A_of_x(c, node, x0, x1, A);
    const double as = c->p.amp * s_of_x(&c->p, x0, x1);
    const double db0 = 16.0 * (1.0 - 2.0 * y0) * y1 * (1.0 - y1);
    const double db1 = 16.0 * y0 * (1.0 - y0) * (1.0 - 2.0 * y1);
    F[0] = A[0] + as * db0;
    F[1] = A[1] + as * db1;
    F[2] = A[2] + as * db0;
    F[3] = A[3] + as * db1;
}

int or_jac(const or_ctx* c, double x0, double x1, double y0, double y1, double* F) {
    jac_eval(c, -1, x0, x1, y0, y1, F);
    return 0;
}

/* build_cache cell entry (mapping.cpp:96-110) with the D-tensor extension
 * A = C^T D C / det (reduces to mapping.cpp:106-108 at D = I). */
static int cell_entry(const or_ctx* c, int node, const double* x, const double* y, double* e) {
    double F[4];
    jac_eval(c, node, x[0], x[1], y[0], y[1], F);
    const double det = F[0] * F[3] - F[1] * F[2];
    if (det <= 1e-12) {
        snprintf(g_err, sizeof g_err,
                 "degenerate map in cache build: det grad_y zeta = %g at x = (%g, %g), yhat = (%g, %g)",
                 det, x[0], x[1], y[0], y[1]);
        return 3;
    }
    const double C00 = F[3], C01 = -F[2], C10 = -F[1], C11 = F[0]; /* linalg.hpp:36 */
    e[0] = det;
    if (c->D_identity) {
        e[1] = (C00 * C00 + C10 * C10) / det;
        e[2] = (C00 * C01 + C10 * C11) / det;
        e[3] = (C01 * C01 + C11 * C11) / det;
    } else {
        const double* D = c->p.D;
        const double DC00 = D[0] * C00 + D[1] * C10, DC01 = D[0] * C01 + D[1] * C11;
        const double DC10 = D[2] * C00 + D[3] * C10, DC11 = D[2] * C01 + D[3] * C11;
        e[1] = (C00 * DC00 + C10 * DC10) / det;
        e[2] = (C00 * DC01 + C10 * DC11) / det;
        e[3] = (C01 * DC01 + C11 * DC11) / det;
    }
    return 0;
}

/* build_cache face entry (mapping.cpp:112-126). */
static int face_entry(const or_ctx* c, int node, const double* x, const double* y,
                      const double* nrm, double* e) {
    double F[4];
    jac_eval(c, node, x[0], x[1], y[0], y[1], F);
    const double det = F[0] * F[3] - F[1] * F[2];
    if (det <= 1e-12) {
        snprintf(g_err, sizeof g_err,
                 "degenerate map in cache build: det grad_y zeta = %g at x = (%g, %g), yhat = (%g, %g)",
                 det, x[0], x[1], y[0], y[1]);
        return 3;
    }
    const double C00 = F[3], C01 = -F[2], C10 = -F[1], C11 = F[0];
    e[0] = det;
    e[1] = C00 * nrm[0] + C01 * nrm[1];
    e[2] = C10 * nrm[0] + C11 * nrm[1];
    e[3] = sqrt(e[1] * e[1] + e[2] * e[2]);
    return 0;
}

static int node_cache_row(const or_ctx* c, int node, double* cells, double* faces) {
    double x[2];
    grid_node(&c->macro, node, x);
    if (cells)
        for (int cc = 0; cc < cell_count(&c->micro); ++cc)
            for (int q = 0; q < 4; ++q) {
                double y[2];
                cell_point(&c->micro, cc, QS[q], QT[q], y);
                const int rc = cell_entry(c, node, x, y, cells + (cc * 4 + q) * 4);
                if (rc) return rc;
            }
    if (faces)
        for (int f = 0; f < c->micro.n_faces; ++f) {
            const faceparam_t fp = face_param(&c->micro, f);
            for (int q = 0; q < 2; ++q) {
                double y[2] = {fp.mid[0] + fp.tan[0] * GP[q], fp.mid[1] + fp.tan[1] * GP[q]};
                const int rc = face_entry(c, node, x, y, fp.nrm, faces + (f * 2 + q) * 4);
                if (rc) return rc;
            }
        }
    return 0;
}

int or_node_cache(const or_ctx* c, int node, double* cells, double* faces) {
    return node_cache_row(c, node, cells, faces);
}

static double k_of_y(const or_problem* p, const double* y) {
    if (p->k_kind == OR_K_DISC) {
        const double dx = y[0] - p->k_par[2], dy = y[1] - p->k_par[3];
        return sqrt(dx * dx + dy * dy) < p->k_par[4] ? p->k_par[0] : p->k_par[1];
    }
    return p->k_par[0];
}

static int has_reaction(const or_problem* p) {
    return !(p->k_kind == OR_K_CONST && p->k_par[0] == 0.0);
}

/* build_micro_matrices (assembly.cpp:101-174) for one system, 1-worker scatter order:
 * chunks of 512 cells in order, the boundary faces appended to chunk 0.  Extension:
 * reaction mass  w_q det_elem k(yhat_q) J_q N_a N_b  inside the cell loop. */
static int assemble_micro(const or_ctx* c, int node, double* vals) {
    const grid_t* g = &c->micro;
    const int cells = cell_count(g);
    double* cache = malloc(sizeof(double) * (size_t)cells * 16);
    double* fcache = malloc(sizeof(double) * (size_t)g->n_faces * 8);
    int rc = node_cache_row(c, node, cache, fcache);
    if (rc) {
        free(cache);
        free(fcache);
        return rc;
    }
    memset(vals, 0, sizeof(double) * c->mp.nnz);
    const double det_elem = 0.25 * g->h[0] * g->h[1];
    const double gx = 2.0 / g->h[0], gy = 2.0 / g->h[1];
    const int chunk = 512, nchunks = (cells + chunk - 1) / chunk;
    const int react = has_reaction(&c->p);
    for (int ck = 0; ck < nchunks; ++ck) {
        const int cb = ck * chunk, ce = cells < cb + chunk ? cells : cb + chunk;
        for (int cc = cb; cc < ce; ++cc) {
            int nd[4];
            cell_nodes(g, cc, nd);
            double local[4][4] = {{0}};
            for (int q = 0; q < 4; ++q) {
                const double* e = cache + (cc * 4 + q) * 4;
                const double wq = QW[q] * det_elem * c->p.Dv;
                double gg[4][2];
                for (int a = 0; a < 4; ++a) {
                    gg[a][0] = SHG[q][a][0] * gx;
                    gg[a][1] = SHG[q][a][1] * gy;
                }
                for (int a = 0; a < 4; ++a) {
                    const double Agx = e[1] * gg[a][0] + e[2] * gg[a][1];
                    const double Agy = e[2] * gg[a][0] + e[3] * gg[a][1];
                    for (int b = 0; b < 4; ++b) local[a][b] += wq * (Agx * gg[b][0] + Agy * gg[b][1]);
                }
                if (react) {
                    double y[2];
                    cell_point(g, cc, QS[q], QT[q], y);
                    const double wr = QW[q] * det_elem * k_of_y(&c->p, y) * e[0];
                    for (int a = 0; a < 4; ++a)
                        for (int b = 0; b < 4; ++b) local[a][b] += wr * SHN[q][a] * SHN[q][b];
                }
            }
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b)
                    vals[csr_find(c->mp.rp, c->mp.ci, nd[a], nd[b])] += local[a][b];
        }
        if (ck == 0) {
            for (int f = 0; f < g->n_faces; ++f) {
                const int role = c->p.micro_role[g->face_side[f]];
                if (role == OR_GAMMA_N) continue;
                const double kappa = role == OR_GAMMA_I ? c->p.kappa[1] : c->p.kappa[3];
                if (kappa == 0.0) continue;
                const faceparam_t fp = face_param(g, f);
                const double scale = face_scale(&fp);
                double local[2][2] = {{0}};
                for (int q = 0; q < 2; ++q) {
                    const double wq = GW[q] * kappa * fcache[(f * 2 + q) * 4 + 3] * scale;
                    for (int a = 0; a < 2; ++a)
                        for (int b = 0; b < 2; ++b) local[a][b] += wq * SHF[q][a] * SHF[q][b];
                }
                const int* fn = g->face_nodes + 2 * f;
                for (int a = 0; a < 2; ++a)
                    for (int b = 0; b < 2; ++b)
                        vals[csr_find(c->mp.rp, c->mp.ci, fn[a], fn[b])] += local[a][b];
            }
        }
    }
    free(cache);
    free(fcache);
    return 0;
}

int or_micro_values(const or_ctx* c, int node, double* vals) { return assemble_micro(c, node, vals); }

/* build_micro_rhs_parts (assembly.cpp:176-231) with f^v = 0 and no g^v. */
static int rhs_parts(const or_ctx* c, int node, double* fixed, double* rin, double* rout) {
    const grid_t* g = &c->micro;
    const int n = node_count(g);
    double* fcache = malloc(sizeof(double) * (size_t)g->n_faces * 8);
    int rc = node_cache_row(c, node, NULL, fcache);
    if (rc) {
        free(fcache);
        return rc;
    }
    if (fixed) memset(fixed, 0, sizeof(double) * n);
    memset(rin, 0, sizeof(double) * n);
    memset(rout, 0, sizeof(double) * n);
    for (int f = 0; f < g->n_faces; ++f) {
        const int role = c->p.micro_role[g->face_side[f]];
        const faceparam_t fp = face_param(g, f);
        const double scale = face_scale(&fp);
        const int* fn = g->face_nodes + 2 * f;
        for (int q = 0; q < 2; ++q) {
            const double w_meas = GW[q] * fcache[(f * 2 + q) * 4 + 3] * scale;
            if (role == OR_GAMMA_I)
                for (int a = 0; a < 2; ++a) rin[fn[a]] += w_meas * SHF[q][a];
            else if (role == OR_GAMMA_O)
                for (int a = 0; a < 2; ++a) rout[fn[a]] += w_meas * SHF[q][a];
        }
    }
    free(fcache);
    return 0;
}

int or_micro_rhs_parts(const or_ctx* c, int node, double* fixed, double* rin, double* rout) {
    return rhs_parts(c, node, fixed, rin, rout);
}

/* surface_coupling (assembly.cpp:377-393) using the cached per-node |nu|. */
static double coupling(const or_ctx* c, const double* v, int node, int role) {
    const grid_t* g = &c->micro;
    const double* len = c->node_face_len + (size_t)node * g->n_faces * 2;
    double total = 0.0;
    for (int f = 0; f < g->n_faces; ++f) {
        if (c->p.micro_role[g->face_side[f]] != role) continue;
        const faceparam_t fp = face_param(g, f);
        const double scale = face_scale(&fp);
        const int* fn = g->face_nodes + 2 * f;
        for (int q = 0; q < 2; ++q) {
            const double vq = v[fn[0]] * SHF[q][0] + v[fn[1]] * SHF[q][1];
            total += GW[q] * vq * len[f * 2 + q] * scale;
        }
    }
    return total;
}

double or_surface_coupling(const or_ctx* c, const double* v, int node, int role) {
    return coupling(c, v, node, role);
}

/* build_macro_systems (assembly.cpp:233-361) with constant data, no Neumann data. */
static int build_macro(or_ctx* c) {
    const grid_t* M = &c->macro;
    const grid_t* g = &c->micro;
    const int ncell = cell_count(M), nq = 4;
    const size_t n_q = (size_t)ncell * nq;
    double* gin = calloc(n_q, sizeof(double));
    double* gout = calloc(n_q, sizeof(double));
    double e[4];
    for (size_t qg = 0; qg < n_q; ++qg) {
        double x[2];
        cell_point(M, (int)(qg / nq), QS[qg % nq], QT[qg % nq], x);
        double g_in = 0.0, g_out = 0.0;
        for (int f = 0; f < g->n_faces; ++f) {
            const int role = c->p.micro_role[g->face_side[f]];
            const faceparam_t fp = face_param(g, f);
            const double scale = face_scale(&fp);
            for (int q = 0; q < 2; ++q) {
                double y[2] = {fp.mid[0] + fp.tan[0] * GP[q], fp.mid[1] + fp.tan[1] * GP[q]};
                const int rc = face_entry(c, -1, x, y, fp.nrm, e); /* qpoint_cache, assembly.cpp:69 */
                if (rc) {
                    free(gin);
                    free(gout);
                    return rc;
                }
                const double w = GW[q] * scale;
                if (role == OR_GAMMA_I)
                    g_in += w * e[3];
                else if (role == OR_GAMMA_O)
                    g_out += w * e[3];
            }
        }
        gin[qg] = g_in;
        gout[qg] = g_out;
    }
    const int nM = node_count(M);
    c->Au = calloc(c->Mp.nnz, sizeof(double));
    c->Aw = calloc(c->Mp.nnz, sizeof(double));
    c->M0 = calloc(c->Mp.nnz, sizeof(double));
    c->bu = calloc(nM, sizeof(double));
    c->bw = calloc(nM, sizeof(double));
    const double det_elem = 0.25 * M->h[0] * M->h[1];
    const double gx = 2.0 / M->h[0], gy = 2.0 / M->h[1];
    const double rhs_u = c->p.fu + 0.0 - 0.0, rhs_w = c->p.fw + 0.0 - 0.0;
    for (int cc = 0; cc < ncell; ++cc) {
        int nd[4];
        cell_nodes(M, cc, nd);
        double lu[4][4] = {{0}}, lw[4][4] = {{0}}, lm[4][4] = {{0}}, bu[4] = {0}, bw[4] = {0};
        for (int q = 0; q < nq; ++q) {
            const size_t qg = (size_t)cc * nq + q;
            const double wq = QW[q] * det_elem;
            const double mass_u = c->p.kappa[0] * gin[qg];
            const double mass_w = c->p.kappa[2] * gout[qg];
            const double dw = c->p.Dw;
            double gg[4][2];
            for (int a = 0; a < 4; ++a) {
                gg[a][0] = SHG[q][a][0] * gx;
                gg[a][1] = SHG[q][a][1] * gy;
            }
            for (int a = 0; a < 4; ++a) {
                for (int b = 0; b < 4; ++b) {
                    const double stiff = gg[a][0] * gg[b][0] + gg[a][1] * gg[b][1];
                    const double mass = SHN[q][a] * SHN[q][b];
                    lu[a][b] += wq * (stiff + mass_u * mass);
                    lw[a][b] += wq * (dw * stiff + mass_w * mass);
                    lm[a][b] += wq * mass;
                }
                bu[a] += wq * rhs_u * SHN[q][a];
                bw[a] += wq * rhs_w * SHN[q][a];
            }
        }
        for (int a = 0; a < 4; ++a) {
            for (int b = 0; b < 4; ++b) {
                const int k = csr_find(c->Mp.rp, c->Mp.ci, nd[a], nd[b]);
                c->Au[k] += lu[a][b];
                c->Aw[k] += lw[a][b];
                c->M0[k] += lm[a][b];
            }
            c->bu[nd[a]] += bu[a];
            c->bw[nd[a]] += bw[a];
        }
    }
    free(gin);
    free(gout);
    /* Dirichlet list: ascending nodes on Dirichlet sides (assembly.cpp:345-353). */
    char* mark = calloc(nM, 1);
    for (int f = 0; f < M->n_faces; ++f)
        if (c->p.macro_dirichlet[M->face_side[f]]) {
            mark[M->face_nodes[2 * f]] = 1;
            mark[M->face_nodes[2 * f + 1]] = 1;
        }
    c->n_dir_u = 0;
    for (int i = 0; i < nM; ++i) c->n_dir_u += mark[i];
    c->dir_u = malloc(sizeof(int) * (c->n_dir_u + 1));
    c->dir_u_val = malloc(sizeof(double) * (c->n_dir_u + 1));
    for (int i = 0, k = 0; i < nM; ++i)
        if (mark[i]) {
            c->dir_u[k] = i;
            c->dir_u_val[k] = c->p.u0;
            ++k;
        }
    free(mark);
    c->w_pinned = c->p.kappa[2] == 0.0; /* assembly.cpp:357-360 */
    return 0;
}

int or_create(const or_problem* p, or_ctx** out) {
    *out = NULL;
    static pthread_once_t once = PTHREAD_ONCE_INIT;
    pthread_once(&once, rule_init);
    or_ctx* c = calloc(1, sizeof(or_ctx));
    c->p = *p;
    grid_init(&c->macro, p->macro_lo, p->macro_hi, p->macro_n);
    grid_init(&c->micro, p->micro_lo, p->micro_hi, p->micro_n);
    const int nM = node_count(&c->macro);
    if (p->A_kind == OR_A_TABLE) {
        c->A_table = malloc(sizeof(double) * 4 * nM);
        memcpy(c->A_table, p->A_table, sizeof(double) * 4 * nM);
        c->p.A_table = c->A_table;
    }
    c->D_identity = p->D[0] == 1.0 && p->D[1] == 0.0 && p->D[2] == 0.0 && p->D[3] == 1.0;
    q1_pattern(&c->micro, &c->mp);
    q1_pattern(&c->macro, &c->Mp);
    const int nf = c->micro.n_faces;
    c->node_face_len = malloc(sizeof(double) * (size_t)nM * nf * 2);
    double* fc = malloc(sizeof(double) * nf * 8);
    for (int i = 0; i < nM; ++i) {
        int rc = node_cache_row(c, i, NULL, fc);
        if (rc) {
            free(fc);
            or_destroy(c);
            return rc;
        }
        for (int k = 0; k < nf * 2; ++k) c->node_face_len[(size_t)i * nf * 2 + k] = fc[k * 4 + 3];
    }
    free(fc);
    int rc = build_macro(c);
    if (rc) {
        or_destroy(c);
        return rc;
    }
    *out = c;
    return 0;
}

void or_destroy(or_ctx* c) {
    if (!c) return;
    grid_free(&c->macro);
    grid_free(&c->micro);
    free(c->mp.rp);
    free(c->mp.ci);
    free(c->Mp.rp);
    free(c->Mp.ci);
    free(c->A_table);
    free(c->robin_in);
    free(c->robin_out);
    free(c->micro_vals);
    free(c->node_face_len);
    free(c->Au);
    free(c->Aw);
    free(c->M0);
    free(c->bu);
    free(c->bw);
    free(c->dir_u);
    free(c->dir_u_val);
    free(c);
}

int or_sizes(const or_ctx* c, int* s) {
    s[0] = node_count(&c->macro);
    s[1] = node_count(&c->micro);
    s[2] = c->mp.nnz;
    s[3] = c->Mp.nnz;
    s[4] = c->micro.n_faces;
    s[5] = cell_count(&c->micro);
    return 0;
}

int or_micro_pattern(const or_ctx* c, int* rp, int* ci) {
    memcpy(rp, c->mp.rp, sizeof(int) * (c->mp.n + 1));
    memcpy(ci, c->mp.ci, sizeof(int) * c->mp.nnz);
    return 0;
}

int or_macro_pattern(const or_ctx* c, int* rp, int* ci) {
    memcpy(rp, c->Mp.rp, sizeof(int) * (c->Mp.n + 1));
    memcpy(ci, c->Mp.ci, sizeof(int) * c->Mp.nnz);
    return 0;
}

int or_macro_matrix(const or_ctx* c, int which, double* vals) {
    const double* src = which == 0 ? c->Au : which == 1 ? c->Aw : c->M0;
    memcpy(vals, src, sizeof(double) * c->Mp.nnz);
    return 0;
}

int or_macro_fixed_rhs(const or_ctx* c, double* bu, double* bw) {
    memcpy(bu, c->bu, sizeof(double) * c->Mp.n);
    memcpy(bw, c->bw, sizeof(double) * c->Mp.n);
    return 0;
}

/* ---------------------------------------------------------- micro loop ---- */
/* Per-problem operators and Robin parts of every micro problem, `threads` workers over
 * the problems (one problem per thread at a time: values independent of the count). */
typedef struct {
    or_ctx* c;
    atomic_int next, rc;
} asm_job;

static void* asm_worker(void* arg) {
    asm_job* J = arg;
    or_ctx* c = J->c;
    const int nM = node_count(&c->macro), n = c->mp.n, nnz = c->mp.nnz;
    for (;;) {
        const int i = atomic_fetch_add(&J->next, 1);
        if (i >= nM) break;
        int rc = assemble_micro(c, i, c->micro_vals + (size_t)i * nnz);
        if (!rc) rc = rhs_parts(c, i, NULL, c->robin_in + (size_t)i * n, c->robin_out + (size_t)i * n);
        if (rc) {
            atomic_store(&J->rc, rc);
            break;
        }
    }
    return NULL;
}

static int ensure_micro_t(or_ctx* c, int threads) {
    if (c->micro_vals) return 0;
    const int nM = node_count(&c->macro), n = c->mp.n, nnz = c->mp.nnz;
    c->micro_vals = malloc(sizeof(double) * (size_t)nM * nnz);
    c->robin_in = malloc(sizeof(double) * (size_t)nM * n);
    c->robin_out = malloc(sizeof(double) * (size_t)nM * n);
    asm_job J = {.c = c};
    atomic_store(&J.next, 0);
    atomic_store(&J.rc, 0);
    if (threads <= 1) {
        asm_worker(&J);
    } else {
        pthread_t* th = malloc(sizeof(pthread_t) * threads);
        for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, asm_worker, &J);
        for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
        free(th);
    }
    const int rc = atomic_load(&J.rc);
    if (rc) {
        free(c->micro_vals);
        free(c->robin_in);
        free(c->robin_out);
        c->micro_vals = c->robin_in = c->robin_out = NULL;
    }
    return rc;
}


typedef struct {
    or_ctx* c;
    const double *u, *w;
    double tol;
    int maxit, n_nodes;
    const int* nodes;
    double* V;
    int* iters;
    int use_cached; /* 1: matrices/rhs parts from ctx; 0: assemble per node */
    atomic_int next;
} sweep_job;

/* micro_rhs (assembly.cpp:370-375) */
static void micro_rhs(const or_ctx* c, const double* rin, const double* rout, double u, double w,
                      double* b, int n) {
    memset(b, 0, sizeof(double) * n); /* fixed = 0 (f^v = 0, no g^v) */
    if (c->p.kappa[0] != 0.0 && u != 0.0) {
        const double a = c->p.kappa[0] * u;
        for (int k = 0; k < n; ++k) b[k] += a * rin[k];
    }
    if (c->p.kappa[2] != 0.0 && w != 0.0) {
        const double a = c->p.kappa[2] * w;
        for (int k = 0; k < n; ++k) b[k] += a * rout[k];
    }
}

static void* sweep_worker(void* arg) {
    sweep_job* J = arg;
    or_ctx* c = J->c;
    const int n = c->mp.n, nnz = c->mp.nnz;
    double* b = malloc(sizeof(double) * n);
    double* vals = J->use_cached ? NULL : malloc(sizeof(double) * nnz);
    double* rin = J->use_cached ? NULL : malloc(sizeof(double) * n * 2);
    for (;;) {
        const int k = atomic_fetch_add(&J->next, 1);
        if (k >= J->n_nodes) break;
        const int i = J->nodes ? J->nodes[k] : k;
        const double *A, *ri, *ro;
        if (J->use_cached) {
            A = c->micro_vals + (size_t)i * nnz;
            ri = c->robin_in + (size_t)i * n;
            ro = c->robin_out + (size_t)i * n;
        } else {
            if (assemble_micro(c, i, vals) || rhs_parts(c, i, NULL, rin, rin + n)) {
                J->iters[k] = -2;
                continue;
            }
            A = vals;
            ri = rin;
            ro = rin + n;
        }
        micro_rhs(c, ri, ro, J->u[i], J->w[i], b, n);
        int res[3];
        double resid;
        or_cg_solve(n, c->mp.rp, c->mp.ci, A, b, J->V + (size_t)k * n, J->tol, J->maxit, res, &resid);
        J->iters[k] = res[0] ? res[1] : (res[2] ? -3 : -1);
    }
    free(b);
    free(vals);
    free(rin);
    return NULL;
}

static void run_sweep(sweep_job* J, int threads) {
    atomic_store(&J->next, 0);
    if (threads <= 1) {
        sweep_worker(J);
        return;
    }
    pthread_t* th = malloc(sizeof(pthread_t) * threads);
    for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, sweep_worker, J);
    for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
    free(th);
}

int or_micro_sweep(or_ctx* c, const double* u, const double* w, double tol, int maxit, int threads,
                   int n_nodes, const int* nodes, double* V, int* iters) {
    sweep_job J = {.c = c, .u = u, .w = w, .tol = tol, .maxit = maxit, .n_nodes = n_nodes,
                   .nodes = nodes, .V = V, .iters = iters, .use_cached = c->micro_vals != NULL};
    run_sweep(&J, threads);
    for (int k = 0; k < n_nodes; ++k)
        if (iters[k] < 0) {
            snprintf(g_err, sizeof g_err, "micro system %d: CG failed (code %d)",
                     nodes ? nodes[k] : k, iters[k]);
            return 4;
        }
    return 0;
}

/* EliminatedOperator (solver.cpp:14-46) */
typedef struct {
    double* A;
    double* shift;
    int nc;
    const int* dofs;
    const double* vals;
} elim_t;

static void elim_init(elim_t* E, const pattern_t* P, const double* orig, int nc, const int* dofs,
                      const double* vals) {
    const int n = P->n;
    E->nc = nc;
    E->dofs = dofs;
    E->vals = vals;
    E->A = malloc(sizeof(double) * P->nnz);
    memcpy(E->A, orig, sizeof(double) * P->nnz);
    E->shift = malloc(sizeof(double) * n);
    double* gext = calloc(n, sizeof(double));
    for (int k = 0; k < nc; ++k) gext[dofs[k]] = vals[k];
    csr_apply(n, P->rp, P->ci, orig, gext, E->shift);
    /* CsrMatrix::eliminate (linalg.cpp:55-79) — rhs side-effects go to a dummy. */
    char* is_c = calloc(n, 1);
    double* value = calloc(n, sizeof(double));
    for (int k = 0; k < nc; ++k) {
        is_c[dofs[k]] = 1;
        value[dofs[k]] = vals[k];
    }
    if (nc > 0)
        for (int r = 0; r < n; ++r) {
            if (is_c[r]) {
                for (int k = P->rp[r]; k < P->rp[r + 1]; ++k) E->A[k] = (P->ci[k] == r) ? 1.0 : 0.0;
            } else {
                for (int k = P->rp[r]; k < P->rp[r + 1]; ++k)
                    if (is_c[P->ci[k]]) E->A[k] = 0.0;
            }
        }
    free(is_c);
    free(value);
    free(gext);
}

static void elim_rhs(const elim_t* E, const double* b, double* out, int n) {
    for (int i = 0; i < n; ++i) out[i] = b[i] - E->shift[i];
    for (int k = 0; k < E->nc; ++k) out[E->dofs[k]] = E->vals[k];
}

static double elim_residual(const elim_t* E, const pattern_t* P, const double* raw, const double* x) {
    const int n = P->n;
    double* b = malloc(sizeof(double) * n * 2);
    double* Ax = b + n;
    elim_rhs(E, raw, b, n);
    csr_apply(n, P->rp, P->ci, E->A, x, Ax);
    double s = 0.0;
    for (int i = 0; i < n; ++i) {
        const double r = b[i] - Ax[i];
        s += r * r;
    }
    free(b);
    return sqrt(s);
}

/* macro_u_rhs / macro_w_rhs (assembly.cpp:402-422) */
static void macro_rhs(const or_ctx* c, int which, const double* V, double* out) {
    const int nM = c->Mp.n, n = c->mp.n;
    memcpy(out, which == 0 ? c->bu : c->bw, sizeof(double) * nM);
    const double kap = which == 0 ? c->p.kappa[1] : c->p.kappa[3];
    if (kap == 0.0) return;
    double* bI = malloc(sizeof(double) * nM * 2);
    double* mb = bI + nM;
    for (int i = 0; i < nM; ++i)
        bI[i] = coupling(c, V + (size_t)i * n, i, which == 0 ? OR_GAMMA_I : OR_GAMMA_O);
    csr_apply(nM, c->Mp.rp, c->Mp.ci, c->M0, bI, mb);
    for (int i = 0; i < nM; ++i) out[i] += kap * mb[i];
    free(bI);
}

int or_fixed_point_solve(or_ctx* c, double inner_tol, int inner_maxit, double outer_tol,
                         int max_outer, int threads, double* u, double* w, double* V, double* hist,
                         int hist_cap, int* info, double* micro_dof_iters) {
    int rc = ensure_micro_t(c, threads);
    if (rc) return rc;
    const int nM = c->Mp.n, n = c->mp.n, nnz = c->mp.nnz;
    memset(u, 0, sizeof(double) * nM);
    memset(w, 0, sizeof(double) * nM);
    memset(V, 0, sizeof(double) * (size_t)nM * n);
    info[0] = info[1] = info[3] = 0;
    info[2] = c->w_pinned;
    *micro_dof_iters = 0.0;
    elim_t Eu, Ew;
    static const int pin_dof[1] = {0};
    static const double pin_val[1] = {0.0};
    elim_init(&Eu, &c->Mp, c->Au, c->n_dir_u, c->dir_u, c->dir_u_val);
    elim_init(&Ew, &c->Mp, c->Aw, c->w_pinned ? 1 : 0, pin_dof, pin_val);
    double* raw = malloc(sizeof(double) * nM * 2);
    double* bb = raw + nM;
    int* iters = malloc(sizeof(int) * nM);
    double* res_v = malloc(sizeof(double) * nM);
    double* b = malloc(sizeof(double) * n * 2);
    double* Av = b + n;
    double prev = 0.0;
    int ok = 0;
    for (int sweep = 1; sweep <= max_outer; ++sweep) {
        int res[3];
        double resid;
        macro_rhs(c, 0, V, raw);
        elim_rhs(&Eu, raw, bb, nM);
        or_cg_solve(nM, c->Mp.rp, c->Mp.ci, Eu.A, bb, u, inner_tol, inner_maxit, res, &resid);
        if (!res[0]) {
            snprintf(g_err, sizeof g_err, "macro u-system: CG %s", res[2] ? "negative curvature" : "failed");
            rc = 4;
            break;
        }
        macro_rhs(c, 1, V, raw);
        elim_rhs(&Ew, raw, bb, nM);
        or_cg_solve(nM, c->Mp.rp, c->Mp.ci, Ew.A, bb, w, inner_tol, inner_maxit, res, &resid);
        if (!res[0]) {
            snprintf(g_err, sizeof g_err, "macro w-system: CG %s", res[2] ? "negative curvature" : "failed");
            rc = 4;
            break;
        }
        sweep_job J = {.c = c, .u = u, .w = w, .tol = inner_tol, .maxit = inner_maxit, .n_nodes = nM,
                       .nodes = NULL, .V = V, .iters = iters, .use_cached = 1};
        run_sweep(&J, threads);
        for (int i = 0; i < nM; ++i) {
            if (iters[i] < 0) {
                snprintf(g_err, sizeof g_err, "micro system %d: CG failed (code %d)", i, iters[i]);
                rc = 4;
                break;
            }
            *micro_dof_iters += (double)n * iters[i];
        }
        if (rc) break;
        macro_rhs(c, 0, V, raw);
        const double res_u = elim_residual(&Eu, &c->Mp, raw, u);
        macro_rhs(c, 1, V, raw);
        const double res_w = elim_residual(&Ew, &c->Mp, raw, w);
        for (int i = 0; i < nM; ++i) {
            micro_rhs(c, c->robin_in + (size_t)i * n, c->robin_out + (size_t)i * n, u[i], w[i], b, n);
            csr_apply(n, c->mp.rp, c->mp.ci, c->micro_vals + (size_t)i * nnz, V + (size_t)i * n, Av);
            double s = 0.0;
            for (int k = 0; k < n; ++k) {
                const double r = b[k] - Av[k];
                s += r * r;
            }
            res_v[i] = sqrt(s);
        }
        double avg = 0.0;
        for (int i = 0; i < nM; ++i) avg += res_v[i];
        avg /= nM;
        const double residual = res_u + res_w + avg;
        if (info[3] < hist_cap) hist[info[3]] = residual;
        info[3] += 1;
        info[0] = sweep;
        if (residual < outer_tol || (sweep >= 2 && fabs(residual - prev) < outer_tol)) {
            ok = 1;
            break;
        }
        prev = residual;
    }
    info[1] = ok;
    free(raw);
    free(iters);
    free(res_v);
    free(b);
    free(Eu.A);
    free(Eu.shift);
    free(Ew.A);
    free(Ew.shift);
    return rc;
}
