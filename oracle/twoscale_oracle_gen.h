/* TEST INFRASTRUCTURE ONLY — dimension/order-generic CPU restatement of the
 * micro-solve path for BASELINE configs 4 (Q2 micro) and 5 (3D Q1 micro), which the
 * reference cannot express (it is 2D Q1 only: grid.cpp:109-119, assembly.cpp:57).
 *
 * It restates the same algorithm as twoscale_oracle.c (assembly.cpp:101-361,
 * mapping.cpp:79-129, linalg.cpp:103-161, solver.cpp:61-132) for tensor-product
 * Lagrange elements of order p in {1,2} on a d-dimensional micro box, d in {2,3};
 * the macro problem stays 2D Q1 as in the reference.  Pinning: at d = 2, p = 1 it
 * is checked against the reference binary (tests/test_oracle_gen.py); beyond that
 * it is pinned only by that reduction.
 *
 * Decisions: node lattice spacing h/p; element-local nodes and cell
 * quadrature lexicographic (axis 0 fastest); Gauss-(p+1) per axis for cells and
 * faces; boundary faces ordered by axis, then transverse cell index, then (-,+)
 * side, which for d = 2 is the reference order (grid.cpp:34-45).
 */
#ifndef TWOSCALE_ORACLE_GEN_H
#define TWOSCALE_ORACLE_GEN_H

#ifdef __cplusplus
extern "C" {
#endif

enum { OG_MAP_AFFINE_BUBBLE = 0, OG_MAP_FOURIER = 1 };

typedef struct og_problem {
    double macro_lo[2], macro_hi[2];
    int macro_n[2];
    int dim, order;
    double micro_lo[3], micro_hi[3];
    int micro_n[3];
    double kappa[4];
    double Dv;
    double D[9];          /* dim x dim physical diffusion tensor, row-major */
    int k_kind;           /* 0 const k_par[0]; 1 disc/ball: k_in, k_out, cx, cy, cz, r */
    double k_par[6];
    int micro_role[6];    /* per side (axis a: 2a = minus, 2a+1 = plus); 0 I, 1 O, 2 N */
    int macro_dirichlet[4];
    int map_kind;
    const double* table; /* AFFINE_BUBBLE: [nodes][dim*dim]; FOURIER: [nodes][2][8] */
    int s_kind;           /* 0 none, 1 sin(2 pi x0) cos(2 pi x1), 2 x0 x1 */
    double amp;
    double fu, fw, Dw, u0;
} og_problem;

typedef struct og_ctx og_ctx;

int og_create(const og_problem* p, og_ctx** out);
void og_destroy(og_ctx* c);
const char* og_last_error(void);
/* n_macro, n_micro, micro_nnz, macro_nnz, n_faces, n_cells, nq_cell, nq_face, face_nodes */
int og_sizes(const og_ctx* c, int* s);
int og_micro_pattern(const og_ctx* c, int* row_ptr, int* col_idx);
int og_micro_values(const og_ctx* c, int node, double* vals);
int og_rhs_parts(const og_ctx* c, int node, double* rin, double* rout);
/* cells [cell][q][1 + dim*(dim+1)/2] (J then A upper triangle row-major), faces [face][q] |nu| */
int og_node_cache(const og_ctx* c, int node, double* cells, double* faces);
int og_macro_matrix(const og_ctx* c, int which, double* vals);
double og_surface_coupling(const og_ctx* c, const double* v, int node, int role);
/* one batched micro solve (micro_rhs + cg_solve per problem), V in/out, iters[-1 = failed] */
int og_micro_sweep(og_ctx* c, const double* u, const double* w, double tol, int maxit, int threads, double* V,
                   int* iters);
int og_fixed_point_solve(og_ctx* c, double inner_tol, int inner_maxit, double outer_tol, int max_outer,
                         int threads, double* u, double* w, double* V, double* hist, int hist_cap, int* info,
                         double* micro_dof_iters);

#ifdef __cplusplus
}
#endif
#endif
