// Host-side launch interface of the device kernels (setup.cu, pcg.cu).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "device_common.cuh"

namespace tsb {

// Data tapes used by the setup kernels (packed in the same buffer as the map tapes).
struct DataTapes {
    TapeRef fv_hat, fu, fw, Dw, dirichlet_value;
    TapeRef gv[4], gu2[4], gw[4];
    TapeRef fu_flux[2], fw_flux[2];
    int has_fu_flux, has_fw_flux;
};

struct ProblemG {
    GridG macro, micro;
    double kappa[4];
    double Dv;
    int macro_bc[4];
    int micro_role[4];
    int reaction_kind;
    double reaction[5];
    MapG map;
    DataTapes data;
};

void upload_quad_tables(const QuadTables& q);

// ---- kernel (1): map cache ------------------------------------------------
// cells out [rows][cells][4] (double4 J,A00,A01,A11); faces out [rows][faces][2]
// (double4 J,nu0,nu1,|nu|).  points == nullptr: row r is macro node r.
// first_bad: atomicMin of the reference's evaluation order index of a degenerate point.
// row0: first macro node when points == nullptr (on-demand single rows for inspection).
void launch_cell_cache(const ProblemG& p, int rows, const double* points, double4* cells,
                       unsigned long long* first_bad, unsigned* err, cudaStream_t s, int row0 = 0);
void launch_face_cache(const ProblemG& p, int rows, const double* points, int with_cells,
                       double4* faces, unsigned long long* first_bad, unsigned* err, cudaStream_t s,
                       int row0 = 0);
// Re-evaluates a single (row, entry) for the error message: out = det, x0, x1, y0, y1.
void launch_degenerate_probe(const ProblemG& p, const double* points, int with_cells,
                             unsigned long long index, double* out, cudaStream_t s);

// min/max of det J over `count` cache entries spaced `stride` doubles apart; per-block
// {min, argmin, max, argmax} into out[4*blocks].
// validate_diffeo over xs x ys (block partials [blocks][min, first index of min, max]; returns
// the block count), check_assumption6's boundary measures, a data tape at macro points.
int launch_validate_pairs(const MapG& m, const double* xs, int nx, const double* ys, int ny, double* part,
                          unsigned* err, cudaStream_t s);
void launch_boundary_measures(const GridG& micro, const int* role, int n, const double* nu, int stride, int offset,
                              double* gamma, cudaStream_t s);
void launch_tape_at_points(const int* op, const int* arg, const double* val, TapeRef t, int n,
                           const double* points, double* out, unsigned* err, cudaStream_t s);
void launch_det_minmax(const double* e, long long count, int stride, double* out, int blocks, cudaStream_t s,
                       long long blk = 0, long long bstride = 0);

// ---- kernel (2): micro operator + rhs parts ---------------------------------
// stencil out [srows][9][n_micro], directions (dj,di) row-major = CSR column order.
void launch_assemble_micro(const ProblemG& p, int srows, const double4* cells, const double4* faces,
                           double* stencil, cudaStream_t s);
void launch_rhs_parts(const ProblemG& p, int n_nodes, int cache_shared, const double4* cells,
                      const double4* faces, double* fixed, double* rin, double* rout, int has_fixed,
                      unsigned* err, cudaStream_t s);
// face |nu| per (row, face, q) for the coupling reduction
void launch_face_len(int rows, int n_faces, const double4* faces, double* len, cudaStream_t s);

// ---- macro systems (assembly.cpp:233-361) ----------------------------------
void launch_macro_qpoints(const ProblemG& p, double* gamma_in, double* gamma_out, double* rhs_u_q,
                          double* rhs_w_q, double* dw_q, unsigned long long* first_bad,
                          unsigned* err, cudaStream_t s);
void launch_macro_assemble(const ProblemG& p, const int* row_ptr, const double* gamma_in,
                           const double* gamma_out, const double* rhs_u_q, const double* rhs_w_q,
                           const double* dw_q, double* Au, double* Aw, double* M0, double* bu,
                           double* bw, unsigned* err, cudaStream_t s);
void launch_dirichlet_values(const ProblemG& p, int n, const int* dofs, double* vals, unsigned* err,
                             cudaStream_t s);
// EliminatedOperator (solver.cpp:14-33): A_e and shift = A * g_ext.
void launch_eliminate(int n, const int* row_ptr, const int* col_idx, const double* A,
                      const unsigned char* cmask, const double* cval, double* A_e, double* shift,
                      cudaStream_t s);

// ---- sweep kernels (pcg.cu) ------------------------------------------------
struct MicroPcgArgs {
    int n_problems;
    GridG micro;
    const double* stencil;   // [srows][planes][n]: the upper half C, E, NW, N, NE at planes plane_base..+4
    long long stencil_stride; // 0 when shared
    int plane_base;           // 0: 5-plane micro operators (upper half only); 4: full 9-plane stencils (macro)
    const double* fixed;     // [n_problems][n]
    const double* rin;
    const double* rout;
    int has_fixed;
    double kappa1, kappa3;
    const double* u;         // [n_problems]
    const double* w;
    double* V;               // [n_problems][n] in: warm start, out: solution
    int warm;                // 0: start from zero
    double tol;
    int maxit;
    int* iters;              // [n_problems]
    int* status;             // [n_problems]: 0 ok, 1 indefinite, 2 maxit
    double* final_rel;       // [n_problems] relative residual at exit
    // epilogue (fixed-point loop): residual norm and coupling integrals
    int epilogue;
    double* res_v;           // [n_problems] ||b - A V||
    double* bI;              // [n_problems] surface_coupling(V, i, GammaI)
    double* bO;
    const double* face_len;  // [rows][faces*2]
    long long face_len_stride;
    int micro_role[4];
    double GW[2];            // face Gauss weights and traces (grid.hpp:83-85)
    double Nf[2][2];
    int* counter;            // persistent-scheduler ticket (zeroed before launch)
    int rows_per_thread;     // 0 = automatic
    const int* order;        // ticket -> problem (longest first); nullptr = identity
};

// Returns the number of kernel launches issued.
int launch_micro_pcg(const MicroPcgArgs& a, cudaStream_t s);
// order = problems sorted by the previous sweep's iteration counts, descending (bucketed
// counting sort, one block; order within a bucket is arbitrary — results do not depend on it).
void launch_order_by_iters(int n, const int* iters, int* order, cudaStream_t s);
size_t micro_pcg_smem_bytes(const GridG& g);
// Which SMEM-resident kernel launch_micro_pcg runs for this grid (env overrides included).
struct MicroPlan {
    int kernel;            // 0 column strips, 1 column pairs
    int R, threads;
    double smem_bytes;     // SMEM bytes per DoF-iteration (loads + stores)
};
MicroPlan plan_micro_pcg(const GridG& g, int forced_rows, int n_problems);
bool micro_pcg_fits(const GridG& g);

// One thread block per system: Jacobi-PCG on CSR (linalg.cpp:103-161), vectors in
// global scratch (4n per system).  systems share the pattern; vals/b/x strided by nnz/n.
struct CsrPcgArgs {
    int n, n_sys;
    const int* row_ptr;
    const int* col_idx;
    const double* vals;
    long long vals_stride;
    const double* b;
    double* x;
    double* scratch;  // [n_sys][6n] (single-block path uses 5n)
    double tol;
    int maxit;
    int* result_i;    // [n_sys][3] converged, iterations, indefinite
    double* result_d; // [n_sys] relative residual
    double* partials; // cooperative path: [3][4][grid] per-block dot-product partials (may be null
                      // for n <= 8192, which use one block per system)
};
// Macro systems on the SMEM-resident stencil PCG: CSR rows of a Q1 matrix on grid g
// (make_q1_matrix pattern) -> 9 direction planes [dir][n] (dir = (dj+1)*3 + (di+1)).
void launch_csr_to_stencil(int n_sys, const GridG& g, const int* row_ptr, const int* col_idx, const double* vals,
                           long long vals_stride, double* planes, cudaStream_t s);
// micro-kernel status/iters/final_rel of the two macro systems -> CsrPcgArgs result layout
void launch_macro_cg_result(const int* status, const int* iters, const double* rel, int* result_i,
                            double* result_d, cudaStream_t s);
// Grid size the cooperative CG uses on the current device (for sizing `partials`).
int csr_pcg_coop_blocks();
// Macro u/w systems on a thread-block cluster (mcluster.cu) when the macro grid exceeds one
// SM's SMEM: a.stencil = 9 planes per system (k_csr_to_stencil), a.fixed = rhs, a.V = x
// (warm start in, solution out), iters/status/final_rel per system.  macro_cluster_size()
// returns the preferred cluster size (0: not applicable); launch tries that size, then smaller
// ones, and returns the size it launched with (0: none).
// ---- device-side sweep loop (CUDA graph with a conditional while node, ctx.cu) ----
// Control state of the loop: sweeps completed, previous residual, per-sweep logs in the
// host's D2H layout (sweep_out[8], cg_res_d[2], cg_res_i[6] packed into 3 doubles) and
// globaltimer stamps (before macro, after macro, after micro, after residual).
struct SweepCtl {
    int sweep;
    int pad;
    double prev;
};
constexpr int kSweepLog = 16;
void launch_sweep_stamp(SweepCtl* ctl, unsigned long long* stamps, int idx, cudaStream_t s);
void launch_sweep_control(SweepCtl* ctl, const double* sweep_out, const double* cg_res_d, const int* cg_res_i,
                          double* log, double outer_tol, int max_outer, cudaGraphConditionalHandle h,
                          cudaStream_t s);
int macro_cluster_size(const GridG& g);
int launch_macro_cluster(const MicroPcgArgs& a, int CL, cudaStream_t s);
void launch_csr_pcg(const CsrPcgArgs& a, cudaStream_t s);

// macro rhs for u and w (assembly.cpp:402-422) + constrain_rhs (solver.cpp:28-33).
struct MacroRhsArgs {
    int n;
    const int* row_ptr;
    const int* col_idx;
    const double* M0;
    const double* b_fixed[2];
    const double* coupling[2];  // bI, bO
    double kappa[2];            // kappa2, kappa4
    const double* shift[2];
    const unsigned char* cmask[2];
    const double* cval[2];
    double* raw[2];
    double* constrained[2];
};
void launch_macro_rhs(const MacroRhsArgs& a, cudaStream_t s);

// residual of a sweep (solver.cpp:100-117) -> out[0] = r_k, out[1] = sum of
// micro DoF-iterations of this sweep, out[2]/out[3] = max/min iterations.
struct SweepResidualArgs {
    int n_macro, n_micro;
    const int* row_ptr;
    const int* col_idx;
    const double* A_e[2];
    const double* constrained[2];
    const double* x[2];
    const double* res_v;
    const int* iters;
    const int* status;       // micro status per problem (0 ok)
    const double* final_rel;
    double* out;             // [8]: r_k, dof_iters, max_it, min_it, first_bad, its status, its rel
};
void launch_sweep_residual(const SweepResidualArgs& a, cudaStream_t s);

// micro_rhs (assembly.cpp:370-375) for one node into b.
void launch_micro_rhs(int n, const double* fixed, const double* rin, const double* rout,
                      int has_fixed, double kappa1, double kappa3, double u, double w, double* b,
                      cudaStream_t s);
// surface_coupling (assembly.cpp:377-393) for n_vec vectors (one warp each):
// out[i] = coupling(v + i*n_micro, face_len + i*len_stride, role).
void launch_coupling(const GridG& micro, const int* micro_role, int role, int n_vec, const double* v,
                     const double* face_len, long long len_stride, const double* GW,
                     const double (*Nf)[2], double* out, cudaStream_t s);

}  // namespace tsb
