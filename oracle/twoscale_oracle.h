/* TEST INFRASTRUCTURE ONLY — CPU restatement ("oracle port") of the reference's
 * batched micro-solve path, used by tests/ as the checker and by bench.py's
 * cpu_baseline leg.  Never linked into or called by the product path.
 *
 * Parity pin: at the reference-expressible reduction (reaction k = 0, D = I,
 * symbolic affine+bubble map) every routine here reproduces the reference
 * library (oracle/_ref, built from /root/reference/proj/src) — see
 * tests/test_oracle_vs_ref.py — so the extensions below (reaction term,
 * anisotropic D, per-node tabulated A(x)) rest on a pinned base.
 *
 * Map family (covers BASELINE.json configs 1-3):
 *   zeta(x, y) = A(x) y + amp * s(x) * beta(y) * (1, 1),
 *   beta(y)    = 16 y0 (1 - y0) y1 (1 - y1)
 * A(x): OR_A_IDENTITY, OR_A_TRIG (I + eps [[sin 2 pi x0, cos 2 pi x1],
 *       [cos 2 pi x0, sin 2 pi x1]]) or OR_A_TABLE (per macro node, bilinear
 *       interpolation between nodes for non-node points, e.g. macro qpoints).
 * s(x): OR_S_SINCOS (sin 2 pi x0 cos 2 pi x1) or OR_S_PRODUCT (x0 x1).
 * Data: constant f^u, f^w, D^w, u0; f^v = 0 and no MMS corrections (g^u, g^v,
 * g^w, flux functionals) — the BASELINE configs use none of them.
 */
#ifndef TWOSCALE_ORACLE_H
#define TWOSCALE_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_A_IDENTITY = 0, OR_A_TRIG = 1, OR_A_TABLE = 2 };
enum { OR_S_NONE = 0, OR_S_SINCOS = 1, OR_S_PRODUCT = 2 };
enum { OR_K_CONST = 0, OR_K_DISC = 1 };
enum { OR_GAMMA_I = 0, OR_GAMMA_O = 1, OR_GAMMA_N = 2 };

typedef struct or_problem {
    double macro_lo[2], macro_hi[2];
    int macro_n[2];
    double micro_lo[2], micro_hi[2];
    int micro_n[2];
    double kappa[4];
    double Dv;
    double D[4];          /* physical-frame micro diffusion tensor (row-major, symmetric) */
    int k_kind;           /* reaction k(yhat) */
    double k_par[5];      /* CONST: k0 | DISC: k_in, k_out, cx, cy, radius */
    int micro_role[4];    /* per side Left, Right, Bottom, Top */
    int macro_dirichlet[4];
    int A_kind;
    double A_eps;
    const double* A_table; /* [n_macro_nodes][4], row-major 2x2 per node */
    int s_kind;
    double amp;
    double fu, fw, Dw, u0;
} or_problem;

typedef struct or_ctx or_ctx;

int or_create(const or_problem* p, or_ctx** out);
void or_destroy(or_ctx* c);
const char* or_last_error(void);

int or_sizes(const or_ctx* c, int* sizes); /* n_macro, n_micro, micro_nnz, macro_nnz, n_faces, n_cells */

int or_micro_pattern(const or_ctx* c, int* row_ptr, int* col_idx);
/* CSR values of micro system `node` (assembly.cpp:101-174 + reaction extension) */
int or_micro_values(const or_ctx* c, int node, double* vals);
/* fixed, robin_in, robin_out (assembly.cpp:176-231) */
int or_micro_rhs_parts(const or_ctx* c, int node, double* fixed, double* rin, double* rout);
/* node cache row: cells [cell][q][J,A00,A01,A11], faces [face][q][J,nux,nuy,len] */
int or_node_cache(const or_ctx* c, int node, double* cells, double* faces);
int or_jac(const or_ctx* c, double x0, double x1, double y0, double y1, double* F);

int or_macro_matrix(const or_ctx* c, int which, double* vals); /* 0 A_u, 1 A_w, 2 M0 */
int or_macro_pattern(const or_ctx* c, int* row_ptr, int* col_idx);
int or_macro_fixed_rhs(const or_ctx* c, double* bu, double* bw);
double or_surface_coupling(const or_ctx* c, const double* v, int node, int role);

/* cg_solve (linalg.cpp:103-161); res = {converged, iterations, indefinite}, *resid */
int or_cg_solve(int n, const int* row_ptr, const int* col_idx, const double* vals, const double* b,
                double* x, double tol, int maxit, int* res, double* resid);

/* fixed_point_solve (solver.cpp:61-132).  V row-major [n_macro][n_micro].
 * info = {sweeps, converged, w_pinned, n_hist}; micro_dof_iters = sum over sweeps of
 * n_micro * iterations (the north-star work unit); threads >= 1 for the micro loop. */
int or_fixed_point_solve(or_ctx* c, double inner_tol, int inner_maxit, double outer_tol,
                         int max_outer, int threads, double* u, double* w, double* V, double* hist,
                         int hist_cap, int* info, double* micro_dof_iters);

/* Micro loop only (solver.cpp:85-98) for a subset of nodes with fixed u, w.
 * V [n_nodes][n_micro] in/out; iters per node (-1 on failure). */
int or_micro_sweep(or_ctx* c, const double* u, const double* w, double tol, int maxit,
                   int threads, int n_nodes, const int* nodes, double* V, int* iters);

#ifdef __cplusplus
}
#endif
#endif
