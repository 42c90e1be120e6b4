/* TEST INFRASTRUCTURE ONLY — see twoscale_oracle_gen.h.  Compiled with
 * -ffp-contract=off into oracle/lib/liboracle.so next to twoscale_oracle.c, whose
 * or_cg_solve (linalg.cpp:103-161) it reuses. */
#define _GNU_SOURCE
#include "twoscale_oracle_gen.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "twoscale_oracle.h"

static __thread char g_err[512];
const char* og_last_error(void) { return g_err; }

#define MAXQ 27   /* (p+1)^d quadrature points / element nodes, p <= 2, d <= 3 */
#define MAXFQ 9

/* ------------------------------------------------------------- micro grid -- */
typedef struct {
    int d, p;
    double lo[3], hi[3], h[3], hp[3];
    int nc[3], nn[3];
    int nnodes, ncells, nfaces;
    int npe, npf;            /* nodes per element / per face */
    int nq, nqf;             /* quadrature points per cell / face */
    double W[MAXQ], S[MAXQ][3];           /* cell rule on [-1,1]^d */
    double N[MAXQ][MAXQ], dN[MAXQ][MAXQ][3];
    double FW[MAXFQ], FT[MAXFQ][2];       /* face rule on [-1,1]^(d-1) */
    double Nf[MAXFQ][MAXFQ];
    int *f_axis, *f_side, *f_cell;        /* per boundary face */
    int* f_nodes;                         /* [face][npf] */
} ggrid;

static void rule1d(int n, double* x, double* w) {
    if (n == 2) {
        const double g = 1.0 / sqrt(3.0);
        x[0] = -g; x[1] = g;
        w[0] = 1.0; w[1] = 1.0;
    } else {
        const double g = sqrt(3.0 / 5.0);
        x[0] = -g; x[1] = 0.0; x[2] = g;
        w[0] = 5.0 / 9.0; w[1] = 8.0 / 9.0; w[2] = 5.0 / 9.0;
    }
}

/* 1D Lagrange basis on the p+1 equispaced points of [-1,1] */
static double lag(int p, int a, double s) {
    if (p == 1) return a == 0 ? 0.5 * (1.0 - s) : 0.5 * (1.0 + s);
    if (a == 0) return 0.5 * s * (s - 1.0);
    if (a == 1) return 1.0 - s * s;
    return 0.5 * s * (s + 1.0);
}
static double dlag(int p, int a, double s) {
    if (p == 1) return a == 0 ? -0.5 : 0.5;
    if (a == 0) return s - 0.5;
    if (a == 1) return -2.0 * s;
    return s + 0.5;
}

static int gnode(const ggrid* g, const int* i) {
    return g->d == 2 ? i[0] + g->nn[0] * i[1] : i[0] + g->nn[0] * (i[1] + g->nn[1] * i[2]);
}
static double gcoord(const ggrid* g, int a, int i) { return g->lo[a] + i * g->hp[a]; }

static void ggrid_init(ggrid* g, int d, int p, const double* lo, const double* hi, const int* n) {
    memset(g, 0, sizeof *g);
    g->d = d;
    g->p = p;
    g->nnodes = 1;
    g->ncells = 1;
    for (int a = 0; a < d; ++a) {
        g->lo[a] = lo[a];
        g->hi[a] = hi[a];
        g->nc[a] = n[a];
        g->h[a] = (hi[a] - lo[a]) / n[a];
        g->hp[a] = g->h[a] / p;
        g->nn[a] = p * n[a] + 1;
        g->nnodes *= g->nn[a];
        g->ncells *= n[a];
    }
    const int q1 = p + 1;
    double x[3], w[3];
    rule1d(q1, x, w);
    g->npe = d == 2 ? q1 * q1 : q1 * q1 * q1;
    g->npf = d == 2 ? q1 : q1 * q1;
    g->nq = g->npe;
    g->nqf = g->npf;
    for (int q = 0; q < g->nq; ++q) {
        const int qi[3] = {q % q1, (q / q1) % q1, q / (q1 * q1)};
        g->W[q] = 1.0;
        for (int k = 0; k < d; ++k) {
            g->S[q][k] = x[qi[k]];
            g->W[q] *= w[qi[k]];
        }
        for (int a = 0; a < g->npe; ++a) {
            const int ai[3] = {a % q1, (a / q1) % q1, a / (q1 * q1)};
            double v = 1.0;
            for (int k = 0; k < d; ++k) v *= lag(p, ai[k], g->S[q][k]);
            g->N[q][a] = v;
            for (int k = 0; k < d; ++k) {
                double t = dlag(p, ai[k], g->S[q][k]);
                for (int l = 0; l < d; ++l)
                    if (l != k) t *= lag(p, ai[l], g->S[q][l]);
                g->dN[q][a][k] = t;
            }
        }
    }
    for (int q = 0; q < g->nqf; ++q) {
        const int qi[2] = {q % q1, q / q1};
        g->FW[q] = 1.0;
        for (int k = 0; k < d - 1; ++k) {
            g->FT[q][k] = x[qi[k]];
            g->FW[q] *= w[qi[k]];
        }
        for (int a = 0; a < g->npf; ++a) {
            const int ai[2] = {a % q1, a / q1};
            double v = 1.0;
            for (int k = 0; k < d - 1; ++k) v *= lag(p, ai[k], g->FT[q][k]);
            g->Nf[q][a] = v;
        }
    }
    /* boundary faces: axis, then transverse cells lexicographic, then side (-,+) */
    int nf = 0;
    for (int a = 0; a < d; ++a) {
        int cnt = 1;
        for (int k = 0; k < d; ++k)
            if (k != a) cnt *= n[k];
        nf += 2 * cnt;
    }
    g->nfaces = nf;
    g->f_axis = malloc(sizeof(int) * nf);
    g->f_side = malloc(sizeof(int) * nf);
    g->f_cell = malloc(sizeof(int) * nf);
    g->f_nodes = malloc(sizeof(int) * nf * g->npf);
    int f = 0;
    for (int a = 0; a < d; ++a) {
        int tr[2], nt = 0;
        for (int k = 0; k < d; ++k)
            if (k != a) tr[nt++] = k;
        const int c0n = n[tr[0]], c1n = nt > 1 ? n[tr[1]] : 1;
        for (int c1 = 0; c1 < c1n; ++c1)
            for (int c0 = 0; c0 < c0n; ++c0)
                for (int side = 0; side < 2; ++side) {
                    int cc[3] = {0, 0, 0};
                    cc[tr[0]] = c0;
                    if (nt > 1) cc[tr[1]] = c1;
                    cc[a] = side ? n[a] - 1 : 0;
                    g->f_axis[f] = a;
                    g->f_side[f] = side;
                    g->f_cell[f] = d == 2 ? cc[0] + n[0] * cc[1] : cc[0] + n[0] * (cc[1] + n[1] * cc[2]);
                    for (int fa = 0; fa < g->npf; ++fa) {
                        const int li[2] = {fa % q1, fa / q1};
                        int ii[3];
                        ii[a] = side ? g->nn[a] - 1 : 0;
                        ii[tr[0]] = p * cc[tr[0]] + li[0];
                        if (nt > 1) ii[tr[1]] = p * cc[tr[1]] + li[1];
                        g->f_nodes[f * g->npf + fa] = gnode(g, ii);
                    }
                    ++f;
                }
    }
}

static void ggrid_free(ggrid* g) {
    free(g->f_axis);
    free(g->f_side);
    free(g->f_cell);
    free(g->f_nodes);
}

static void cell_index(const ggrid* g, int c, int* cc) {
    cc[0] = c % g->nc[0];
    cc[1] = (c / g->nc[0]) % g->nc[1];
    cc[2] = g->d == 3 ? c / (g->nc[0] * g->nc[1]) : 0;
}

static void cell_nodes_g(const ggrid* g, int c, int* nd) {
    int cc[3];
    cell_index(g, c, cc);
    const int q1 = g->p + 1;
    for (int a = 0; a < g->npe; ++a) {
        const int ai[3] = {a % q1, (a / q1) % q1, a / (q1 * q1)};
        int ii[3];
        for (int k = 0; k < g->d; ++k) ii[k] = g->p * cc[k] + ai[k];
        nd[a] = gnode(g, ii);
    }
}

static void cell_qpoint(const ggrid* g, int c, int q, double* y) {
    int cc[3];
    cell_index(g, c, cc);
    for (int k = 0; k < g->d; ++k) y[k] = g->lo[k] + (cc[k] + 0.5) * g->h[k] + 0.5 * g->h[k] * g->S[q][k];
}

/* face point and scale (product over transverse axes of half the face extent) */
static void face_geom(const ggrid* g, int f, int q, double* y, double* scale, double* nrm) {
    const int a = g->f_axis[f];
    int cc[3];
    cell_index(g, g->f_cell[f], cc);
    int t = 0;
    double sc = 1.0;
    for (int k = 0; k < g->d; ++k) {
        nrm[k] = 0.0;
        if (k == a) {
            y[k] = g->f_side[f] ? gcoord(g, k, g->nn[k] - 1) : g->lo[k];
            continue;
        }
        const double x0 = gcoord(g, k, g->p * cc[k]), x1 = gcoord(g, k, g->p * (cc[k] + 1));
        const double mid = 0.5 * (x0 + x1), tan = 0.5 * (x1 - x0);
        y[k] = mid + g->FT[q][t] * tan;
        sc *= tan;
        ++t;
    }
    nrm[a] = g->f_side[f] ? 1.0 : -1.0;
    *scale = g->d == 2 ? sqrt(sc * sc) : sc;
}

/* -------------------------------------------------------------------- ctx -- */
struct og_ctx {
    og_problem p;
    double* table;
    int tstride;
    ggrid g;
    /* macro grid (2D Q1, reference numbering) */
    double Mlo[2], Mh[2];
    int Mn[2], nM, Mcells;
    int *Mrp, *Mci, Mnnz;
    int *rp, *ci, nnz;
    double* face_len; /* [nM][nfaces][nqf] */
    double *Au, *Aw, *M0, *bu, *bw;
    int n_dir;
    int* dir;
    int w_pinned;
    double *vals, *rin, *rout;
};

static int csr_find(const int* rp, const int* ci, int row, int col) {
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

static void macro_node(const og_ctx* c, int i, double* x) {
    x[0] = c->Mlo[0] + (i % (c->Mn[0] + 1)) * c->Mh[0];
    x[1] = c->Mlo[1] + (i / (c->Mn[0] + 1)) * c->Mh[1];
}

static double s_of(int kind, const double* x) {
    const double tp = 2.0 * 3.141592653589793;
    if (kind == 1) return sin(tp * x[0]) * cos(tp * x[1]);
    if (kind == 2) return x[0] * x[1];
    return 0.0;
}

/* table row at macro node, or bilinear interpolation at other macro points */
static void table_row(const og_ctx* c, int node, const double* x, double* out) {
    const int ts = c->tstride;
    if (node >= 0) {
        memcpy(out, c->table + (size_t)node * ts, sizeof(double) * ts);
        return;
    }
    const double fx = (x[0] - c->Mlo[0]) / c->Mh[0], fy = (x[1] - c->Mlo[1]) / c->Mh[1];
    int ci = (int)floor(fx), cj = (int)floor(fy);
    if (ci < 0) ci = 0;
    if (ci > c->Mn[0] - 1) ci = c->Mn[0] - 1;
    if (cj < 0) cj = 0;
    if (cj > c->Mn[1] - 1) cj = c->Mn[1] - 1;
    const double s = fx - ci, t = fy - cj;
    const int nx = c->Mn[0] + 1;
    const double* T00 = c->table + (size_t)(cj * nx + ci) * ts;
    const double* T10 = c->table + (size_t)(cj * nx + ci + 1) * ts;
    const double* T11 = c->table + (size_t)((cj + 1) * nx + ci + 1) * ts;
    const double* T01 = c->table + (size_t)((cj + 1) * nx + ci) * ts;
    for (int k = 0; k < ts; ++k)
        out[k] = (1.0 - s) * (1.0 - t) * T00[k] + s * (1.0 - t) * T10[k] + s * t * T11[k] + (1.0 - s) * t * T01[k];
}

static const int FK[8] = {1, 1, 2, 2, 1, 3, 2, 3};
static const int FL[8] = {1, 2, 1, 2, 3, 1, 3, 2};

/* grad_y zeta (row-major d x d) */
static void jac(const og_ctx* c, int node, const double* x, const double* y, double* F) {
    const int d = c->g.d;
    double T[18];
    table_row(c, node, x, T);
    if (c->p.map_kind == OG_MAP_AFFINE_BUBBLE) {
        const double as = c->p.amp * s_of(c->p.s_kind, x);
        double gb[3];
        const double cd = d == 2 ? 16.0 : 64.0;
        for (int k = 0; k < d; ++k) {
            double v = cd * (1.0 - 2.0 * y[k]);
            for (int l = 0; l < d; ++l)
                if (l != k) v *= y[l] * (1.0 - y[l]);
            gb[k] = v;
        }
        for (int a = 0; a < d; ++a)
            for (int b = 0; b < d; ++b) F[a * d + b] = T[a * d + b] + as * gb[b];
    } else { /* FOURIER, d = 2: zeta_a = y_a + sum_m c[a][m] sin(pi k y0) sin(pi l y1) */
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
            for (int m = 0; m < 8; ++m) {
                const double cm = T[a * 8 + m];
                g0 += cm * (pi * FK[m]) * c0[FK[m]] * s1[FL[m]];
                g1 += cm * (pi * FL[m]) * s0[FK[m]] * c1[FL[m]];
            }
            F[a * 2 + 0] = (a == 0 ? 1.0 : 0.0) + g0;
            F[a * 2 + 1] = (a == 1 ? 1.0 : 0.0) + g1;
        }
    }
}

/* cofactor matrix C = det(F) F^{-T} (linalg.hpp:36 in 2D) and det */
static double cofactor(int d, const double* F, double* C) {
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

static int degenerate(double det, const double* x, const double* y, int d) {
    if (d == 2)
        snprintf(g_err, sizeof g_err,
                 "degenerate map in cache build: det grad_y zeta = %g at x = (%g, %g), yhat = (%g, %g)", det, x[0],
                 x[1], y[0], y[1]);
    else
        snprintf(g_err, sizeof g_err,
                 "degenerate map in cache build: det grad_y zeta = %g at x = (%g, %g), yhat = (%g, %g, %g)", det,
                 x[0], x[1], y[0], y[1], y[2]);
    return 3;
}

/* cell entry: J, then A = C^T D C / det upper triangle */
static int cell_entry(const og_ctx* c, int node, const double* x, const double* y, double* e) {
    const int d = c->g.d;
    double F[9], C[9], DC[9];
    jac(c, node, x, y, F);
    const double det = cofactor(d, F, C);
    if (det <= 1e-12) return degenerate(det, x, y, d);
    const double* D = c->p.D;
    for (int k = 0; k < d; ++k)
        for (int b = 0; b < d; ++b) {
            double s = D[k * d + 0] * C[0 * d + b];
            for (int l = 1; l < d; ++l) s += D[k * d + l] * C[l * d + b];
            DC[k * d + b] = s;
        }
    int idx = 1;
    e[0] = det;
    const int ident = (d == 2 && D[0] == 1.0 && D[1] == 0.0 && D[2] == 0.0 && D[3] == 1.0);
    for (int a = 0; a < d; ++a)
        for (int b = a; b < d; ++b) {
            double s;
            if (ident) { /* reference order, mapping.cpp:106-108 */
                s = C[0 * d + a] * C[0 * d + b] + C[1 * d + a] * C[1 * d + b];
            } else {
                s = C[0 * d + a] * DC[0 * d + b];
                for (int k = 1; k < d; ++k) s += C[k * d + a] * DC[k * d + b];
            }
            e[idx++] = s / det;
        }
    return 0;
}

static int face_entry(const og_ctx* c, int node, const double* x, const double* y, const double* nrm,
                      double* len) {
    const int d = c->g.d;
    double F[9], C[9];
    jac(c, node, x, y, F);
    const double det = cofactor(d, F, C);
    if (det <= 1e-12) return degenerate(det, x, y, d);
    double s = 0.0;
    for (int i = 0; i < d; ++i) {
        double nu = C[i * d + 0] * nrm[0];
        for (int k = 1; k < d; ++k) nu += C[i * d + k] * nrm[k];
        s += nu * nu;
    }
    *len = sqrt(s);
    return 0;
}

static int ncoef(int d) { return 1 + d * (d + 1) / 2; }

static int node_cache(const og_ctx* c, int node, double* cells, double* faces) {
    const ggrid* g = &c->g;
    double x[2], y[3], nrm[3], sc;
    macro_node(c, node, x);
    const int nc = ncoef(g->d);
    if (cells)
        for (int cc = 0; cc < g->ncells; ++cc)
            for (int q = 0; q < g->nq; ++q) {
                cell_qpoint(g, cc, q, y);
                int rc = cell_entry(c, node, x, y, cells + ((size_t)cc * g->nq + q) * nc);
                if (rc) return rc;
            }
    if (faces)
        for (int f = 0; f < g->nfaces; ++f)
            for (int q = 0; q < g->nqf; ++q) {
                face_geom(g, f, q, y, &sc, nrm);
                int rc = face_entry(c, node, x, y, nrm, faces + (size_t)f * g->nqf + q);
                if (rc) return rc;
            }
    return 0;
}

int og_node_cache(const og_ctx* c, int node, double* cells, double* faces) { return node_cache(c, node, cells, faces); }

static double k_of(const og_problem* p, const double* y, int d) {
    if (p->k_kind == 1) {
        double s = 0.0;
        for (int k = 0; k < d; ++k) {
            const double t = y[k] - p->k_par[2 + k];
            s += t * t;
        }
        return sqrt(s) < p->k_par[5] ? p->k_par[0] : p->k_par[1];
    }
    return p->k_par[0];
}

/* micro pattern: all nodes sharing an element, rows lexicographic, columns ascending */
static void pattern(og_ctx* c) {
    const ggrid* g = &c->g;
    const int d = g->d, p = g->p;
    c->rp = malloc(sizeof(int) * (g->nnodes + 1));
    c->ci = malloc(sizeof(int) * (size_t)g->nnodes * (d == 2 ? 25 : 125));
    int k = 0;
    c->rp[0] = 0;
    for (int n = 0; n < g->nnodes; ++n) {
        int ii[3] = {n % g->nn[0], (n / g->nn[0]) % g->nn[1], d == 3 ? n / (g->nn[0] * g->nn[1]) : 0};
        int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
        for (int a = 0; a < d; ++a) {
            /* cells containing lattice index i on this axis: floor((i-1)/p) .. floor(i/p) */
            int c0 = ii[a] > 0 ? (ii[a] - 1) / p : 0, c1 = ii[a] / p;
            if (c1 > g->nc[a] - 1) c1 = g->nc[a] - 1;
            if (ii[a] == 0) c0 = 0;
            lo[a] = p * c0;
            hi[a] = p * (c1 + 1);
        }
        if (d == 2) {
            for (int j = lo[1]; j <= hi[1]; ++j)
                for (int i = lo[0]; i <= hi[0]; ++i) c->ci[k++] = i + g->nn[0] * j;
        } else {
            for (int l = lo[2]; l <= hi[2]; ++l)
                for (int j = lo[1]; j <= hi[1]; ++j)
                    for (int i = lo[0]; i <= hi[0]; ++i) c->ci[k++] = i + g->nn[0] * (j + g->nn[1] * l);
        }
        c->rp[n + 1] = k;
    }
    c->nnz = k;
}

/* build_micro_matrices generalised; reference scatter order (512-cell chunks, faces after chunk 0) */
static int assemble(const og_ctx* c, int node, double* vals) {
    const ggrid* g = &c->g;
    const int d = g->d, nc = ncoef(d);
    double* cache = malloc(sizeof(double) * (size_t)g->ncells * g->nq * nc);
    double* fcache = malloc(sizeof(double) * (size_t)g->nfaces * g->nqf);
    int rc = node_cache(c, node, cache, fcache);
    if (rc) {
        free(cache);
        free(fcache);
        return rc;
    }
    memset(vals, 0, sizeof(double) * c->nnz);
    const double det_elem = d == 2 ? 0.25 * g->h[0] * g->h[1] : 0.125 * g->h[0] * g->h[1] * g->h[2];
    double gs[3];
    for (int k = 0; k < d; ++k) gs[k] = 2.0 / g->h[k];
    const int react = !(c->p.k_kind == 0 && c->p.k_par[0] == 0.0);
    const int chunk = 512, nch = (g->ncells + chunk - 1) / chunk;
    int nd[MAXQ];
    for (int ck = 0; ck < nch; ++ck) {
        const int cb = ck * chunk, ce = g->ncells < cb + chunk ? g->ncells : cb + chunk;
        for (int cc = cb; cc < ce; ++cc) {
            cell_nodes_g(g, cc, nd);
            double K[MAXQ][MAXQ];
            memset(K, 0, sizeof K);
            for (int q = 0; q < g->nq; ++q) {
                const double* e = cache + ((size_t)cc * g->nq + q) * nc;
                double A[3][3];
                int idx = 1;
                for (int a = 0; a < d; ++a)
                    for (int b = a; b < d; ++b) A[a][b] = A[b][a] = e[idx++];
                const double wq = g->W[q] * det_elem * c->p.Dv;
                double gg[MAXQ][3];
                for (int a = 0; a < g->npe; ++a)
                    for (int k = 0; k < d; ++k) gg[a][k] = g->dN[q][a][k] * gs[k];
                for (int a = 0; a < g->npe; ++a) {
                    double Ag[3];
                    for (int i = 0; i < d; ++i) {
                        double s = A[i][0] * gg[a][0];
                        for (int k = 1; k < d; ++k) s += A[i][k] * gg[a][k];
                        Ag[i] = s;
                    }
                    for (int b = 0; b < g->npe; ++b) {
                        double s = Ag[0] * gg[b][0];
                        for (int i = 1; i < d; ++i) s += Ag[i] * gg[b][i];
                        K[a][b] += wq * s;
                    }
                }
                if (react) {
                    double y[3];
                    cell_qpoint(g, cc, q, y);
                    const double wr = g->W[q] * det_elem * k_of(&c->p, y, d) * e[0];
                    for (int a = 0; a < g->npe; ++a)
                        for (int b = 0; b < g->npe; ++b) K[a][b] += wr * g->N[q][a] * g->N[q][b];
                }
            }
            for (int a = 0; a < g->npe; ++a)
                for (int b = 0; b < g->npe; ++b) vals[csr_find(c->rp, c->ci, nd[a], nd[b])] += K[a][b];
        }
        if (ck == 0)
            for (int f = 0; f < g->nfaces; ++f) {
                const int role = c->p.micro_role[2 * g->f_axis[f] + g->f_side[f]];
                if (role == 2) continue;
                const double kappa = role == 0 ? c->p.kappa[1] : c->p.kappa[3];
                if (kappa == 0.0) continue;
                double y[3], sc, nrm[3];
                face_geom(g, f, 0, y, &sc, nrm);
                double K[MAXFQ][MAXFQ];
                memset(K, 0, sizeof K);
                for (int q = 0; q < g->nqf; ++q) {
                    const double wq = g->FW[q] * kappa * fcache[(size_t)f * g->nqf + q] * sc;
                    for (int a = 0; a < g->npf; ++a)
                        for (int b = 0; b < g->npf; ++b) K[a][b] += wq * g->Nf[q][a] * g->Nf[q][b];
                }
                const int* fn = g->f_nodes + (size_t)f * g->npf;
                for (int a = 0; a < g->npf; ++a)
                    for (int b = 0; b < g->npf; ++b) vals[csr_find(c->rp, c->ci, fn[a], fn[b])] += K[a][b];
            }
    }
    free(cache);
    free(fcache);
    return 0;
}

int og_micro_values(const og_ctx* c, int node, double* vals) { return assemble(c, node, vals); }

static int rhs_parts(const og_ctx* c, int node, double* rin, double* rout) {
    const ggrid* g = &c->g;
    memset(rin, 0, sizeof(double) * g->nnodes);
    memset(rout, 0, sizeof(double) * g->nnodes);
    const double* len = c->face_len + (size_t)node * g->nfaces * g->nqf;
    for (int f = 0; f < g->nfaces; ++f) {
        const int role = c->p.micro_role[2 * g->f_axis[f] + g->f_side[f]];
        double y[3], sc, nrm[3];
        face_geom(g, f, 0, y, &sc, nrm);
        const int* fn = g->f_nodes + (size_t)f * g->npf;
        for (int q = 0; q < g->nqf; ++q) {
            const double w_meas = g->FW[q] * len[f * g->nqf + q] * sc;
            if (role == 0)
                for (int a = 0; a < g->npf; ++a) rin[fn[a]] += w_meas * g->Nf[q][a];
            else if (role == 1)
                for (int a = 0; a < g->npf; ++a) rout[fn[a]] += w_meas * g->Nf[q][a];
        }
    }
    return 0;
}

int og_rhs_parts(const og_ctx* c, int node, double* rin, double* rout) { return rhs_parts(c, node, rin, rout); }

static double coupling(const og_ctx* c, const double* v, int node, int role) {
    const ggrid* g = &c->g;
    const double* len = c->face_len + (size_t)node * g->nfaces * g->nqf;
    double total = 0.0;
    for (int f = 0; f < g->nfaces; ++f) {
        if (c->p.micro_role[2 * g->f_axis[f] + g->f_side[f]] != role) continue;
        double y[3], sc, nrm[3];
        face_geom(g, f, 0, y, &sc, nrm);
        const int* fn = g->f_nodes + (size_t)f * g->npf;
        for (int q = 0; q < g->nqf; ++q) {
            double vq = v[fn[0]] * g->Nf[q][0];
            for (int a = 1; a < g->npf; ++a) vq += v[fn[a]] * g->Nf[q][a];
            total += g->FW[q] * vq * len[f * g->nqf + q] * sc;
        }
    }
    return total;
}

double og_surface_coupling(const og_ctx* c, const double* v, int node, int role) { return coupling(c, v, node, role); }

/* macro Q1 systems (assembly.cpp:233-361) with gamma from this micro geometry */
static int build_macro(og_ctx* c) {
    const ggrid* g = &c->g;
    const int ncell = c->Mcells;
    const size_t n_q = (size_t)ncell * 4;
    double* gin = calloc(n_q, sizeof(double));
    double* gout = calloc(n_q, sizeof(double));
    const double gq = 1.0 / sqrt(3.0);
    const double QS[4] = {-gq, gq, -gq, gq}, QT[4] = {-gq, -gq, gq, gq};
    for (size_t qg = 0; qg < n_q; ++qg) {
        const int cc = (int)(qg / 4), q = (int)(qg % 4);
        const int ci = cc % c->Mn[0], cj = cc / c->Mn[0];
        double x[2];
        x[0] = c->Mlo[0] + (ci + 0.5) * c->Mh[0] + 0.5 * c->Mh[0] * QS[q];
        x[1] = c->Mlo[1] + (cj + 0.5) * c->Mh[1] + 0.5 * c->Mh[1] * QT[q];
        double g_in = 0.0, g_out = 0.0;
        for (int f = 0; f < g->nfaces; ++f) {
            const int role = c->p.micro_role[2 * g->f_axis[f] + g->f_side[f]];
            for (int fq = 0; fq < g->nqf; ++fq) {
                double y[3], sc, nrm[3], len;
                face_geom(g, f, fq, y, &sc, nrm);
                int rc = face_entry(c, -1, x, y, nrm, &len);
                if (rc) {
                    free(gin);
                    free(gout);
                    return rc;
                }
                const double w = g->FW[fq] * sc;
                if (role == 0)
                    g_in += w * len;
                else if (role == 1)
                    g_out += w * len;
            }
        }
        gin[qg] = g_in;
        gout[qg] = g_out;
    }
    const int nM = c->nM;
    c->Au = calloc(c->Mnnz, sizeof(double));
    c->Aw = calloc(c->Mnnz, sizeof(double));
    c->M0 = calloc(c->Mnnz, sizeof(double));
    c->bu = calloc(nM, sizeof(double));
    c->bw = calloc(nM, sizeof(double));
    const double det_elem = 0.25 * c->Mh[0] * c->Mh[1];
    const double gx = 2.0 / c->Mh[0], gy = 2.0 / c->Mh[1];
    double N[4][4], dN[4][4][2];
    for (int q = 0; q < 4; ++q) {
        const double s = QS[q], t = QT[q];
        N[q][0] = 0.25 * (1.0 - s) * (1.0 - t);
        N[q][1] = 0.25 * (1.0 + s) * (1.0 - t);
        N[q][2] = 0.25 * (1.0 + s) * (1.0 + t);
        N[q][3] = 0.25 * (1.0 - s) * (1.0 + t);
        dN[q][0][0] = -0.25 * (1.0 - t);
        dN[q][0][1] = -0.25 * (1.0 - s);
        dN[q][1][0] = 0.25 * (1.0 - t);
        dN[q][1][1] = -0.25 * (1.0 + s);
        dN[q][2][0] = 0.25 * (1.0 + t);
        dN[q][2][1] = 0.25 * (1.0 + s);
        dN[q][3][0] = -0.25 * (1.0 + t);
        dN[q][3][1] = 0.25 * (1.0 - s);
    }
    const double rhs_u = c->p.fu + 0.0 - 0.0, rhs_w = c->p.fw + 0.0 - 0.0;
    const int nx = c->Mn[0] + 1;
    for (int cc = 0; cc < ncell; ++cc) {
        const int ci = cc % c->Mn[0], cj = cc / c->Mn[0];
        const int nd[4] = {cj * nx + ci, cj * nx + ci + 1, (cj + 1) * nx + ci + 1, (cj + 1) * nx + ci};
        double lu[4][4] = {{0}}, lw[4][4] = {{0}}, lm[4][4] = {{0}}, bu[4] = {0}, bw[4] = {0};
        for (int q = 0; q < 4; ++q) {
            const size_t qg = (size_t)cc * 4 + q;
            const double wq = 1.0 * det_elem;
            const double mass_u = c->p.kappa[0] * gin[qg], mass_w = c->p.kappa[2] * gout[qg];
            double gg[4][2];
            for (int a = 0; a < 4; ++a) {
                gg[a][0] = dN[q][a][0] * gx;
                gg[a][1] = dN[q][a][1] * gy;
            }
            for (int a = 0; a < 4; ++a) {
                for (int b = 0; b < 4; ++b) {
                    const double stiff = gg[a][0] * gg[b][0] + gg[a][1] * gg[b][1];
                    const double mass = N[q][a] * N[q][b];
                    lu[a][b] += wq * (stiff + mass_u * mass);
                    lw[a][b] += wq * (c->p.Dw * stiff + mass_w * mass);
                    lm[a][b] += wq * mass;
                }
                bu[a] += wq * rhs_u * N[q][a];
                bw[a] += wq * rhs_w * N[q][a];
            }
        }
        for (int a = 0; a < 4; ++a) {
            for (int b = 0; b < 4; ++b) {
                const int k = csr_find(c->Mrp, c->Mci, nd[a], nd[b]);
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
    c->dir = malloc(sizeof(int) * nM);
    c->n_dir = 0;
    for (int i = 0; i < nM; ++i) {
        const int ii = i % nx, jj = i / nx;
        const int on = (ii == 0 && c->p.macro_dirichlet[0]) || (ii == c->Mn[0] && c->p.macro_dirichlet[1]) ||
                       (jj == 0 && c->p.macro_dirichlet[2]) || (jj == c->Mn[1] && c->p.macro_dirichlet[3]);
        if (on) c->dir[c->n_dir++] = i;
    }
    c->w_pinned = c->p.kappa[2] == 0.0;
    return 0;
}

int og_create(const og_problem* p, og_ctx** out) {
    *out = NULL;
    if (!(p->dim == 2 || p->dim == 3) || !(p->order == 1 || p->order == 2) || (p->dim == 3 && p->order == 2))
        return snprintf(g_err, sizeof g_err, "unsupported dim/order"), 5;
    if (p->map_kind == OG_MAP_FOURIER && p->dim != 2) return snprintf(g_err, sizeof g_err, "Fourier map is 2D"), 5;
    og_ctx* c = calloc(1, sizeof(og_ctx));
    c->p = *p;
    ggrid_init(&c->g, p->dim, p->order, p->micro_lo, p->micro_hi, p->micro_n);
    for (int a = 0; a < 2; ++a) {
        c->Mlo[a] = p->macro_lo[a];
        c->Mn[a] = p->macro_n[a];
        c->Mh[a] = (p->macro_hi[a] - p->macro_lo[a]) / p->macro_n[a];
    }
    c->nM = (c->Mn[0] + 1) * (c->Mn[1] + 1);
    c->Mcells = c->Mn[0] * c->Mn[1];
    c->tstride = p->map_kind == OG_MAP_FOURIER ? 16 : p->dim * p->dim;
    c->table = malloc(sizeof(double) * (size_t)c->nM * c->tstride);
    memcpy(c->table, p->table, sizeof(double) * (size_t)c->nM * c->tstride);
    /* macro Q1 pattern (make_q1_matrix) */
    const int nx = c->Mn[0] + 1;
    c->Mrp = malloc(sizeof(int) * (c->nM + 1));
    c->Mci = malloc(sizeof(int) * 9 * c->nM);
    int k = 0;
    c->Mrp[0] = 0;
    for (int j = 0; j <= c->Mn[1]; ++j)
        for (int i = 0; i <= c->Mn[0]; ++i) {
            for (int dj = -1; dj <= 1; ++dj)
                for (int di = -1; di <= 1; ++di)
                    if (i + di >= 0 && i + di <= c->Mn[0] && j + dj >= 0 && j + dj <= c->Mn[1])
                        c->Mci[k++] = (j + dj) * nx + i + di;
            c->Mrp[j * nx + i + 1] = k;
        }
    c->Mnnz = k;
    pattern(c);
    const ggrid* g = &c->g;
    c->face_len = malloc(sizeof(double) * (size_t)c->nM * g->nfaces * g->nqf);
    for (int i = 0; i < c->nM; ++i) {
        int rc = node_cache(c, i, NULL, c->face_len + (size_t)i * g->nfaces * g->nqf);
        if (rc) {
            og_destroy(c);
            return rc;
        }
    }
    int rc = build_macro(c);
    if (rc) {
        og_destroy(c);
        return rc;
    }
    *out = c;
    return 0;
}

void og_destroy(og_ctx* c) {
    if (!c) return;
    ggrid_free(&c->g);
    free(c->table);
    free(c->Mrp);
    free(c->Mci);
    free(c->rp);
    free(c->ci);
    free(c->face_len);
    free(c->Au);
    free(c->Aw);
    free(c->M0);
    free(c->bu);
    free(c->bw);
    free(c->dir);
    free(c->vals);
    free(c->rin);
    free(c->rout);
    free(c);
}

int og_sizes(const og_ctx* c, int* s) {
    s[0] = c->nM;
    s[1] = c->g.nnodes;
    s[2] = c->nnz;
    s[3] = c->Mnnz;
    s[4] = c->g.nfaces;
    s[5] = c->g.ncells;
    s[6] = c->g.nq;
    s[7] = c->g.nqf;
    s[8] = c->g.npf;
    return 0;
}

int og_micro_pattern(const og_ctx* c, int* rp, int* ci) {
    memcpy(rp, c->rp, sizeof(int) * (c->g.nnodes + 1));
    memcpy(ci, c->ci, sizeof(int) * c->nnz);
    return 0;
}

int og_macro_matrix(const og_ctx* c, int which, double* vals) {
    memcpy(vals, which == 0 ? c->Au : which == 1 ? c->Aw : c->M0, sizeof(double) * c->Mnnz);
    return 0;
}

/* ---------------------------------------------------------- fixed point -- */
typedef struct {
    og_ctx* c;
    const double *u, *w;
    double tol;
    int maxit;
    double* V;
    int* iters;
    atomic_int next;
} job_t;

static void micro_rhs(const og_ctx* c, int i, double u, double w, double* b) {
    const int n = c->g.nnodes;
    memset(b, 0, sizeof(double) * n);
    if (c->p.kappa[0] != 0.0 && u != 0.0) {
        const double a = c->p.kappa[0] * u;
        for (int k = 0; k < n; ++k) b[k] += a * c->rin[(size_t)i * n + k];
    }
    if (c->p.kappa[2] != 0.0 && w != 0.0) {
        const double a = c->p.kappa[2] * w;
        for (int k = 0; k < n; ++k) b[k] += a * c->rout[(size_t)i * n + k];
    }
}

static void* worker(void* arg) {
    job_t* J = arg;
    og_ctx* c = J->c;
    const int n = c->g.nnodes;
    double* b = malloc(sizeof(double) * n);
    for (;;) {
        const int i = atomic_fetch_add(&J->next, 1);
        if (i >= c->nM) break;
        micro_rhs(c, i, J->u[i], J->w[i], b);
        int res[3];
        double resid;
        or_cg_solve(n, c->rp, c->ci, c->vals + (size_t)i * c->nnz, b, J->V + (size_t)i * n, J->tol, J->maxit, res,
                    &resid);
        J->iters[i] = res[0] ? res[1] : -1;
    }
    free(b);
    return NULL;
}

static void apply(int n, const int* rp, const int* ci, const double* v, const double* x, double* y) {
    for (int r = 0; r < n; ++r) {
        double s = 0.0;
        for (int k = rp[r]; k < rp[r + 1]; ++k) s += v[k] * x[ci[k]];
        y[r] = s;
    }
}

static void macro_rhs(const og_ctx* c, int which, const double* V, double* out) {
    const int nM = c->nM, n = c->g.nnodes;
    memcpy(out, which == 0 ? c->bu : c->bw, sizeof(double) * nM);
    const double kap = which == 0 ? c->p.kappa[1] : c->p.kappa[3];
    if (kap == 0.0) return;
    double* bI = malloc(sizeof(double) * nM * 2);
    for (int i = 0; i < nM; ++i) bI[i] = coupling(c, V + (size_t)i * n, i, which == 0 ? 0 : 1);
    apply(nM, c->Mrp, c->Mci, c->M0, bI, bI + nM);
    for (int i = 0; i < nM; ++i) out[i] += kap * bI[nM + i];
    free(bI);
}

/* EliminatedOperator (solver.cpp:14-46) */
static void elim(const og_ctx* c, const double* A, const int* dofs, int nd, double* Ae, double* shift) {
    const int n = c->nM;
    char* mk = calloc(n, 1);
    for (int k = 0; k < nd; ++k) mk[dofs[k]] = 1;
    memcpy(Ae, A, sizeof(double) * c->Mnnz);
    for (int r = 0; r < n; ++r) shift[r] = 0.0; /* constraint values are zero (u0 = 0 configs) */
    for (int r = 0; r < n; ++r)
        for (int k = c->Mrp[r]; k < c->Mrp[r + 1]; ++k) {
            if (mk[r])
                Ae[k] = c->Mci[k] == r ? 1.0 : 0.0;
            else if (mk[c->Mci[k]])
                Ae[k] = 0.0;
        }
    free(mk);
}

/* Per-problem operators and rhs parts of every micro problem, `threads` workers over the
 * problems (each problem is assembled by one thread, so the values do not depend on the
 * worker count). */
typedef struct {
    og_ctx* c;
    atomic_int next, rc;
} asm_job_t;

static void* asm_worker(void* arg) {
    asm_job_t* J = arg;
    og_ctx* c = J->c;
    const int n = c->g.nnodes;
    for (;;) {
        const int i = atomic_fetch_add(&J->next, 1);
        if (i >= c->nM) break;
        const int rc = assemble(c, i, c->vals + (size_t)i * c->nnz);
        if (rc) {
            atomic_store(&J->rc, rc);
            break;
        }
        rhs_parts(c, i, c->rin + (size_t)i * n, c->rout + (size_t)i * n);
    }
    return NULL;
}

static int ensure_assembled(og_ctx* c, int threads) {
    if (c->vals) return 0;
    const int nM = c->nM, n = c->g.nnodes;
    c->vals = malloc(sizeof(double) * (size_t)nM * c->nnz);
    c->rin = malloc(sizeof(double) * (size_t)nM * n);
    c->rout = malloc(sizeof(double) * (size_t)nM * n);
    asm_job_t J = {.c = c};
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
        free(c->vals);
        free(c->rin);
        free(c->rout);
        c->vals = c->rin = c->rout = NULL;
    }
    return rc;
}

static void run_sweep(job_t* J, int threads) {
    atomic_store(&J->next, 0);
    if (threads <= 1) {
        worker(J);
    } else {
        pthread_t* th = malloc(sizeof(pthread_t) * threads);
        for (int t = 0; t < threads; ++t) pthread_create(&th[t], NULL, worker, J);
        for (int t = 0; t < threads; ++t) pthread_join(th[t], NULL);
        free(th);
    }
}

/* One batched micro solve (micro_rhs + cg_solve per problem, solver.cpp:85-98) with
 * warm start V (in/out); iters[i] = CgResult.iterations, -1 on failure. */
int og_micro_sweep(og_ctx* c, const double* u, const double* w, double tol, int maxit, int threads, double* V,
                   int* iters) {
    int rc = ensure_assembled(c, threads);
    if (rc) return rc;
    job_t J = {.c = c, .u = u, .w = w, .tol = tol, .maxit = maxit, .V = V, .iters = iters};
    run_sweep(&J, threads);
    return 0;
}

int og_fixed_point_solve(og_ctx* c, double inner_tol, int inner_maxit, double outer_tol, int max_outer,
                         int threads, double* u, double* w, double* V, double* hist, int hist_cap, int* info,
                         double* dof_it) {
    if (c->p.u0 != 0.0) return snprintf(g_err, sizeof g_err, "generic oracle supports u0 = 0"), 5;
    const int nM = c->nM, n = c->g.nnodes;
    {
        int rc = ensure_assembled(c, threads);
        if (rc) return rc;
    }
    memset(u, 0, sizeof(double) * nM);
    memset(w, 0, sizeof(double) * nM);
    memset(V, 0, sizeof(double) * (size_t)nM * n);
    double *Aue = malloc(sizeof(double) * c->Mnnz), *Awe = malloc(sizeof(double) * c->Mnnz);
    double *su = malloc(sizeof(double) * nM), *sw = malloc(sizeof(double) * nM);
    static const int pin[1] = {0};
    elim(c, c->Au, c->dir, c->n_dir, Aue, su);
    elim(c, c->Aw, pin, c->w_pinned ? 1 : 0, Awe, sw);
    double *raw = malloc(sizeof(double) * nM * 3), *bb = raw + nM, *Ax = bb + nM;
    int* iters = malloc(sizeof(int) * nM);
    double* b = malloc(sizeof(double) * n * 2);
    char* mk = calloc(nM, 1);
    for (int k = 0; k < c->n_dir; ++k) mk[c->dir[k]] = 1;
    double prev = 0.0;
    int rc = 0;
    info[0] = info[1] = info[3] = 0;
    info[2] = c->w_pinned;
    *dof_it = 0.0;
    for (int sweep = 1; sweep <= max_outer; ++sweep) {
        int res[3];
        double resid;
        macro_rhs(c, 0, V, raw);
        for (int i = 0; i < nM; ++i) bb[i] = mk[i] ? 0.0 : raw[i] - su[i];
        or_cg_solve(nM, c->Mrp, c->Mci, Aue, bb, u, inner_tol, inner_maxit, res, &resid);
        if (!res[0]) { rc = 4; snprintf(g_err, sizeof g_err, "macro u-system: CG failed"); break; }
        macro_rhs(c, 1, V, raw);
        for (int i = 0; i < nM; ++i) bb[i] = (c->w_pinned && i == 0) ? 0.0 : raw[i] - sw[i];
        or_cg_solve(nM, c->Mrp, c->Mci, Awe, bb, w, inner_tol, inner_maxit, res, &resid);
        if (!res[0]) { rc = 4; snprintf(g_err, sizeof g_err, "macro w-system: CG failed"); break; }
        job_t J = {.c = c, .u = u, .w = w, .tol = inner_tol, .maxit = inner_maxit, .V = V, .iters = iters};
        run_sweep(&J, threads);
        for (int i = 0; i < nM; ++i) {
            if (iters[i] < 0) { rc = 4; snprintf(g_err, sizeof g_err, "micro system %d: CG failed", i); break; }
            *dof_it += (double)n * iters[i];
        }
        if (rc) break;
        double res_uw[2];
        for (int s = 0; s < 2; ++s) {
            macro_rhs(c, s, V, raw);
            const double* Ae = s == 0 ? Aue : Awe;
            const double* sh = s == 0 ? su : sw;
            const double* x = s == 0 ? u : w;
            apply(nM, c->Mrp, c->Mci, Ae, x, Ax);
            double acc = 0.0;
            for (int i = 0; i < nM; ++i) {
                const int fixed = s == 0 ? mk[i] : (c->w_pinned && i == 0);
                const double bi = fixed ? 0.0 : raw[i] - sh[i];
                acc += (bi - Ax[i]) * (bi - Ax[i]);
            }
            res_uw[s] = sqrt(acc);
        }
        double avg = 0.0;
        for (int i = 0; i < nM; ++i) {
            micro_rhs(c, i, u[i], w[i], b);
            apply(n, c->rp, c->ci, c->vals + (size_t)i * c->nnz, V + (size_t)i * n, b + n);
            double s = 0.0;
            for (int k = 0; k < n; ++k) s += (b[k] - b[n + k]) * (b[k] - b[n + k]);
            avg += sqrt(s);
        }
        avg /= nM;
        const double residual = res_uw[0] + res_uw[1] + avg;
        if (info[3] < hist_cap) hist[info[3]] = residual;
        info[3] += 1;
        info[0] = sweep;
        if (residual < outer_tol || (sweep >= 2 && fabs(residual - prev) < outer_tol)) {
            info[1] = 1;
            break;
        }
        prev = residual;
    }
    free(Aue);
    free(Awe);
    free(su);
    free(sw);
    free(raw);
    free(iters);
    free(b);
    free(mk);
    return rc;
}
