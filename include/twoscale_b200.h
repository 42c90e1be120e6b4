/* twoscale_b200.h — C ABI of the B200-native micro-solve path.
 *
 * Drop-in boundary for the reference's hot path (arXiv 2103.17040 artifact,
 * /root/reference/proj).  The reference exposes this path only as a C++ API
 * (the headers under proj/include/twoscale); it has no FFI.  The host C++ mirror shipped
 * with this library (include/twoscale, same class/function names) implements that
 * API on top of the entry points below, and any other host (ctypes, cgo, JNI)
 * binds them directly.  Each entry point cites the reference interface it replaces.
 *
 * Conventions: plain pointers + sizes, no C++ or torch types.  All arrays are
 * host memory unless stated; every call is synchronous at return.  Return value
 * is a ts_status; on error ts_last_error() gives the message (same text shape as
 * the reference's exception) and ts_last_error_index() the failing micro system
 * or -1.  Floating point is IEEE FP64 throughout.
 */
#ifndef TWOSCALE_B200_H
#define TWOSCALE_B200_H

#ifdef __CUDACC_RTC__  /* device code compiled at run time (NVRTC): no host headers */
typedef int int32_t;
typedef long long int64_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
#else
#include <stdint.h>
#endif

#ifdef __cplusplus
extern "C" {
#endif

#define TS_ABI_VERSION 3  /* 2: ts_ctx_info gained macro_solver, macro_cluster; 3: ts_validate_diffeo, ts_assumption6 */

typedef enum ts_status {
    TS_OK = 0,
    TS_ERR_CONFIG = 1,         /* ConfigError            (config.hpp:10-12)   */
    TS_ERR_EXPR = 2,           /* ParseError / EvalError (expr.hpp:36-47)     */
    TS_ERR_DEGENERATE_MAP = 3, /* DegenerateMapError     (mapping.hpp:12-14)  */
    TS_ERR_SOLVER = 4,         /* SolverError: CG indefinite / maxit (linalg.hpp:90-92) */
    TS_ERR_INVALID = 5,        /* bad argument / unsupported shape              */
    TS_ERR_CUDA = 6,           /* CUDA runtime failure or no device             */
    TS_ERR_IO = 7,             /* file output (vtk.cpp:11-15 "cannot write '<path>'") */
} ts_status;

/* Postfix program, same instruction set and semantics as CompiledExpr::Instr
 * (expr.hpp:109-116, expr.cpp:663-701): variables x0,x1,y0,y1 = 0..3, parameters
 * already folded to constants.  n == 0 means the constant 0 (the reference's
 * "is_zero" data, assembly.cpp:13-16). */
enum {
    TS_OP_PUSH_CONST = 0, TS_OP_PUSH_VAR = 1, TS_OP_NEG = 2, TS_OP_ADD = 3, TS_OP_SUB = 4,
    TS_OP_MUL = 5, TS_OP_DIV = 6, TS_OP_POW = 7, TS_OP_SIN = 8, TS_OP_COS = 9, TS_OP_EXP = 10,
    TS_OP_SQRT = 11
};
#define TS_MAX_TAPE_STACK 32

typedef struct ts_tape {
    int32_t n;           /* instruction count */
    int32_t max_stack;   /* <= TS_MAX_TAPE_STACK */
    const int32_t* op;
    const int32_t* arg;  /* variable index (PUSH_VAR) or exponent (POW) */
    const double* val;   /* constant (PUSH_CONST) */
} ts_tape;

typedef struct ts_grid_desc {  /* Grid(RectDomain, n0, n1) (grid.hpp:32-40) */
    double lo[2], hi[2];
    int32_t n[2];
} ts_grid_desc;

enum { TS_DIRICHLET = 0, TS_NEUMANN = 1 };               /* MacroBC   (grid.hpp:97) */
enum { TS_GAMMA_I = 0, TS_GAMMA_O = 1, TS_GAMMA_N = 2 }; /* MicroRole (grid.hpp:98) */

/* Micro map families.  TAPE: symbolic zeta, Jacobian as four tapes
 * d zeta_a / d yhat_b (mapping.cpp:10-18).  AFFINE_BUBBLE_TABLE (extension, BASELINE
 * config 3): zeta = A_i yhat + amp s(x) beta(yhat) (1,1), beta = 16 y0(1-y0)y1(1-y1),
 * A_i tabulated per macro node, bilinearly interpolated at non-node macro points; in 3D
 * (config 5) A_i is 3x3, beta = 64 prod y_k(1-y_k) and the direction is (1,1,1).
 * FOURIER_TABLE (config 4, 2D): zeta_a = y_a + sum_{m<8} c[a][m] sin(pi k_m y0) sin(pi l_m y1),
 * (k,l) = (1,1),(1,2),(2,1),(2,2),(1,3),(3,1),(2,3),(3,2), c tabulated per node [2][8]. */
enum { TS_MAP_TAPE = 0, TS_MAP_AFFINE_BUBBLE_TABLE = 1, TS_MAP_FOURIER_TABLE = 2 };
enum { TS_S_NONE = 0, TS_S_SINCOS = 1, TS_S_PRODUCT = 2 };
enum { TS_REACTION_CONST = 0, TS_REACTION_DISC = 1 };

/* ProblemData (problem.hpp:16-40) in flat form, plus the BASELINE extensions.
 * With D = I and reaction 0 it is exactly the reference's problem. */
typedef struct ts_problem_desc {
    int32_t abi_version;           /* TS_ABI_VERSION */
    ts_grid_desc macro, micro;
    double kappa[4];
    double Dv;
    int32_t macro_bc[4];           /* per side Left, Right, Bottom, Top */
    int32_t micro_role[4];
    int32_t map_kind;
    ts_tape jac[4];                /* TAPE: dzeta[0][0], [0][1], [1][0], [1][1] */
    int32_t jac_depends_on_x;      /* Diffeo::jacobian_depends_on_x (mapping.cpp:24-29) */
    const double* A_table;         /* TABLE: [n_macro_nodes][4] row-major */
    int32_t s_kind;
    double amp;
    ts_tape fv_hat;                /* f^v composed with zeta, in (x, yhat) (assembly.cpp:72-75) */
    ts_tape fu, fw, Dw, dirichlet_value; /* dirichlet_value = u0 + gu1 */
    ts_tape gv[4], gu2[4], gw[4];
    ts_tape fu_flux[2], fw_flux[2];
    int32_t has_fu_flux, has_fw_flux;
    double D[4];                   /* extension: physical-frame micro diffusion tensor */
    int32_t reaction_kind;         /* extension: reaction k(yhat) J v phi in the micro operator */
    double reaction[5];            /* CONST: k | DISC: k_in, k_out, cx, cy, radius */
    /* generic micro geometry (configs 4-5).  micro_dim 0/2 + micro_order 0/1 = reference 2D Q1. */
    int32_t micro_dim;             /* 2 or 3 */
    int32_t micro_order;           /* 1 (Q1) or 2 (Q2, 2D only) */
    int32_t micro_n2;              /* 3D: cells along y2 */
    double micro_lo2, micro_hi2;   /* 3D: extent along y2 */
    double D3[9];                  /* 3D: physical-frame diffusion tensor (row-major) */
    int32_t micro_role3[2];        /* 3D: roles of the y2 = lo / hi faces */
    double reaction_cz;            /* 3D: third centre coordinate of the reaction ball */
    int32_t force_generic;         /* run a 2D Q1 problem through the generic path (tests) */
    ts_tape zeta[2];               /* TAPE: zeta itself (optional; the VTK pushforward needs it) */
} ts_problem_desc;

/* Extension block for the INI front-end (keys the reference grammar cannot express). */
typedef struct ts_ext_desc {
    double D[4];
    int32_t reaction_kind;
    double reaction[5];
    int32_t map_kind;              /* TS_MAP_TAPE: use [micro] zeta0/zeta1 */
    const double* A_table;         /* 4 (2D affine), 9 (3D affine) or 16 (Fourier) per macro node */
    int32_t s_kind;
    double amp;
    int32_t micro_dim, micro_order, micro_n2;
    double micro_lo2, micro_hi2;
    double D3[9];
    int32_t micro_role3[2];
    double reaction_cz;
    int32_t force_generic;
} ts_ext_desc;

typedef struct ts_ctx ts_ctx;

typedef struct ts_ctx_info {
    int32_t n_macro, n_micro, micro_nnz, macro_nnz;
    int32_t n_micro_faces, n_micro_cells, n_macro_cells;
    int32_t shared_operator;       /* one micro matrix for all nodes (assembly.cpp:102) */
    int32_t w_pinned;              /* assembly.cpp:357-360 */
    int32_t n_dirichlet_u;
    double setup_ms;               /* device time of the context build (CUDA events) */
    int64_t device_bytes;          /* HBM held by the context */
    int32_t micro_kernel;          /* batched PCG: 0 column strips, 1 column pairs, 2 generic, 3 generic Q2 class-compact */
    int32_t micro_rows;            /* strip height R of variants 0/1 */
    double micro_smem_bytes;       /* SMEM bytes per micro DoF-iteration of variants 0/1 (loads+stores) */
    int32_t macro_solver;          /* macro u/w PCG: 0 one-SM stencil kernel, 1 thread-block cluster, 2 cooperative CSR */
    int32_t macro_cluster;         /* cluster size of macro_solver 1 (CTAs per system), else 0 */
} ts_ctx_info;

typedef struct ts_solve_opts {     /* SolveOptions (solver.hpp:9-15); workers ignored */
    double inner_tol;
    int32_t inner_maxit;
    double outer_tol;
    int32_t max_outer;
} ts_solve_opts;

typedef struct ts_solve_report {   /* SolveReport (solver.hpp:23-28) + measurements */
    int32_t converged, sweeps, w_pinned;
    double final_residual;
    double micro_dof_iters;        /* sum over sweeps/problems of n_micro * PCG iterations */
    double micro_ms;               /* device time of the batched micro PCG launches */
    double macro_ms;               /* device time of the macro rhs/solve/residual launches */
    double total_ms;               /* device time of the whole solve */
    int32_t micro_iters_max, micro_iters_min;
    int32_t gpu_launches;          /* kernels launched by this call */
} ts_solve_report;

typedef struct ts_cg_result {      /* CgResult (linalg.hpp:94-99) */
    int32_t converged, iterations, indefinite;
    double residual;
} ts_cg_result;

#ifndef __CUDACC_RTC__  /* entry points: host code only */
const char* ts_last_error(void);
int32_t ts_last_error_index(void);
int32_t ts_abi_version(void);
/* 1 if a CUDA device of compute capability 10.0 is visible. */
int32_t ts_device_ok(void);
/* Selects the device used by contexts created afterwards on this thread (one process
 * per GPU: rank r calls ts_select_device(local_rank)). */
int32_t ts_select_device(int32_t device);
/* Contexts return their device memory to a process-wide cache that the next context of
 * the same shape reuses; this releases everything cached (e.g. before handing the GPU to
 * another library). */
void ts_trim_device_cache(void);
/* Page-locked host buffers for the host<->device copies of the C ABI. */
void* ts_host_alloc(int64_t bytes);
void ts_host_free(void* p);

/* AssemblyContext(data, macro, micro, workers) (assembly.hpp:24, assembly.cpp:52-99):
 * builds map caches (kernel 1), micro operators + rhs parts (kernel 2) and macro
 * systems on the device. */
int32_t ts_ctx_create(const ts_problem_desc* desc, ts_ctx** out);
/* parse_config + make_problem (config.cpp:126-266, problem.cpp:30-66) then
 * ts_ctx_create; `ext` may be NULL (pure reference problem). */
int32_t ts_ctx_create_ini(const char* ini_text, const ts_ext_desc* ext, ts_ctx** out);
void ts_ctx_destroy(ts_ctx* ctx);
int32_t ts_ctx_get_info(const ts_ctx* ctx, ts_ctx_info* info);
/* Solver options parsed from the INI [solver] section (defaults otherwise). */
int32_t ts_ctx_default_opts(const ts_ctx* ctx, ts_solve_opts* opts);

/* fixed_point_solve(ctx, opts) (solver.hpp:41, solver.cpp:61-132).  State stays on
 * the device; fetch it with ts_download_state.  history may be NULL. */
int32_t ts_fixed_point_solve(ts_ctx* ctx, const ts_solve_opts* opts, ts_solve_report* report,
                             double* residual_history, int32_t history_cap);
/* TwoScaleState (solver.hpp:17-21): u, w [n_macro], V row-major [n_macro][n_micro].
 * Any pointer may be NULL. */
int32_t ts_download_state(ts_ctx* ctx, double* u, double* w, double* V);

/* The micro loop of fixed_point_solve alone (solver.cpp:85-98): every micro system i
 * with b = micro_rhs(i, u[i], w[i]) solved by Jacobi-PCG, warm-started from V_in
 * (NULL = zeros).  V_out [n_macro][n_micro], iters [n_macro] (may be NULL). */
int32_t ts_micro_solve(ts_ctx* ctx, const double* u, const double* w, const double* V_in,
                       double tol, int32_t maxit, double* V_out, int32_t* iters,
                       ts_solve_report* report);

/* Inspection (parity) — CSR in the reference's make_q1_matrix pattern.  The device keeps the
 * centre and the upper half of every operator row (the solvers read a_ij, j < i, as a_ji);
 * ts_micro_values expands a row set to full CSR with the lower entries mirrored, so the
 * returned matrix is exactly symmetric and agrees with the reference's separately
 * assembled lower entries to rounding (src/assembly.cpp:129-147 is symmetric in (a, b)). */
int32_t ts_micro_pattern(const ts_ctx* ctx, int32_t* row_ptr, int32_t* col_idx);
int32_t ts_micro_values(const ts_ctx* ctx, int32_t node, double* vals);       /* micro_matrix(node) */
int32_t ts_micro_rhs(const ts_ctx* ctx, int32_t node, double u, double w, double* b); /* micro_rhs */
/* MapCache row (mapping.hpp:60-94): cells [cell][q][J,A00,A01,A11], faces [face][q][J,nu0,nu1,|nu|] */
int32_t ts_node_cache(const ts_ctx* ctx, int32_t node, double* cells, double* faces);
/* which: 0 A_u, 1 A_w, 2 M0 (macro_u_matrix / macro_w_matrix / macro_mass) */
int32_t ts_macro_matrix(const ts_ctx* ctx, int32_t which, int32_t* row_ptr, int32_t* col_idx,
                        double* vals);
/* macro_u_rhs / macro_w_rhs (assembly.cpp:402-422); V NULL = zero field */
int32_t ts_macro_rhs(ts_ctx* ctx, int32_t which, const double* V, double* out);
/* dirichlet_u / dirichlet_w; dofs/vals may be NULL to query the count */
int32_t ts_dirichlet(const ts_ctx* ctx, int32_t which, int32_t* n, int32_t* dofs, double* vals);
/* surface_coupling(v_node, node, role) (assembly.cpp:377-393) */
int32_t ts_surface_coupling(ts_ctx* ctx, const double* v, int32_t node, int32_t role, double* out);

/* cg_solve(A, b, x, tol, maxit) (linalg.hpp:105-106, linalg.cpp:103-161) on a general
 * CSR matrix, one thread block on the device.  x in/out. */
int32_t ts_cg_solve(int32_t n, const int32_t* row_ptr, const int32_t* col_idx, const double* vals,
                    const double* b, double* x, double tol, int32_t maxit, ts_cg_result* result);

/* build_cache(d, points, micro, gauss(2), workers, with_cells) (mapping.hpp:99-101) for
 * the map and micro grid of `desc` at arbitrary macro points (kernel 1 alone).  cells may
 * be NULL (with_cells = false).  Layout as ts_node_cache, points-major. */
int32_t ts_build_cache(const ts_problem_desc* desc, int32_t n_points, const double* points,
                       double* cells, double* faces);

/* validate_diffeo (mapping.hpp:108-113, mapping.cpp:131-156) for arbitrary lattices: det grad_y
 * zeta of desc's (TAPE) map at every pair of xs x ys ([nx][2], [ny][2]), x outer, on the device.
 * out[3] = min, max, pair index ix * ny + iy of the first minimum (-1: no pairs).  The C++
 * mirror's validate_diffeo applies MapBounds and formats the reference's message. */
int32_t ts_validate_diffeo(const ts_problem_desc* desc, int32_t nx, const double* xs, int32_t ny,
                           const double* ys, double* out);

/* check_assumption6 (mapping.hpp:119-133, mapping.cpp:158-195) at macro points ([n_points][2]):
 * gamma[2i], gamma[2i+1] = the physical measures of Gamma^I and Gamma^O at point i (roles from
 * desc->micro_role, faces in the reference order, Gauss-2 face rule), summed on the device from
 * |nu| at the micro face quadrature points — nu_len ([n_points][n_faces][2], a MapCache's face
 * entries) when given, else kernel (1) on desc's map; dw[i] = desc->Dw(x_i) when dw != NULL.
 * The per-point inequalities and maxima are the mirror's (O(n_points) host work). */
int32_t ts_assumption6(const ts_problem_desc* desc, int32_t n_points, const double* points,
                       const double* nu_len, double* gamma, double* dw);

/* validate_diffeo (mapping.hpp:108-117, mapping.cpp:131-156) at every point the solve uses:
 * det grad_y zeta over all macro nodes x all micro cell and face quadrature points, by
 * kernel (1).  out[6] = min_det, max_det, node, kind (0 cell, 1 face), cell/face index, q
 * of the minimum; *pass = min >= lo && max <= hi && min > 0. */
int32_t ts_validate_map(ts_ctx* ctx, double lo, double hi, double* out, int32_t* pass);

/* error_norms(state, case, macro, micro, workers) (mms.hpp:40, mms.cpp:247-377) on the
 * device, 2D Q1 grids.  tapes[12]: u, w, du/dx0, du/dx1, dw/dx0, dw/dx1, v_hat = v o zeta,
 * dv_hat/dx0, dv_hat/dx1, dv_hat/dy0, dv_hat/dy1, det grad_y zeta.  State from host arrays
 * (u, w [n_macro], V [n_macro][n_micro]).  out[4] = e_uw, e_uw_grad, e_v, e_v_grad. */
int32_t ts_error_norms(const ts_grid_desc* macro, const ts_grid_desc* micro, const ts_tape* tapes,
                       const double* u, const double* w, const double* V, double* out);
/* The same on the device-resident state of a context after ts_fixed_point_solve. */
/* Tape evaluation path of the last error_norms call on this thread: "compiled" (the tapes as
 * straight-line code compiled at run time with NVRTC) or
 * "interpreter (<why>)"; with process-wide compile / launch counters.  TS_JIT=0 forces the
 * interpreter. */
const char* ts_jit_status(void);
int32_t ts_ctx_error_norms(ts_ctx* ctx, const ts_tape* tapes, double* out);
/* Manufactured-solution sweep (convergence_sweep, mms.cpp:384-418): INI with an [mms]
 * section -> derive_data -> per n: n x n macro and micro grids, device solve, device error
 * norms.  rows [n_ns][13]: n, macro_dofs, micro_dofs, H, h, e_uw, e_uw_grad, e_v, e_v_grad,
 * p_macro, q_macro, p_micro, q_micro (orders NaN in the first row). */
int32_t ts_mms_sweep_ini(const char* ini_text, const int32_t* ns, int32_t n_ns, double* rows);
/* Context for the manufactured problem of an INI with an [mms] section: parse_config +
 * make_problem + derive_data (mms.cpp:30-83) + ts_ctx_create, on the INI's own grids. */
int32_t ts_ctx_create_mms_ini(const char* ini_text, ts_ctx** out);
/* error_norms for a host state on the INI's grids against its [mms] solution. */
int32_t ts_error_norms_ini(const char* ini_text, const double* u, const double* w, const double* V, double* out);

/* Micro-state egress.  Legacy VTK unstructured grids written
 * from the device-resident state of the last ts_fixed_point_solve.  TS_VTK_ASCII is the
 * reference's byte layout (vtk.cpp, ostream precision 16); TS_VTK_BINARY is the legacy
 * BINARY variant (big-endian doubles / int32), same sections.  Points and values stream
 * device -> pinned host in chunks overlapped with a multi-threaded ordered formatter. */
enum { TS_VTK_ASCII = 0, TS_VTK_BINARY = 1 };
/* write_vtk_macro(macro, {{"u", u}, {"w", w}}, path) (vtk.hpp:14-16, vtk.cpp:36-54). */
int32_t ts_write_vtk_macro(ts_ctx* ctx, int32_t format, const char* path);
/* write_vtk_micro(V, macro, micro, map, scale, path) (vtk.hpp:21-22, vtk.cpp:56-85): every
 * micro patch pushed forward through zeta(x_i, .), scaled and translated to its macro
 * node.  Q2 patches are written on their node lattice (2n x 2n quads), 3D patches as
 * hexahedra (VTK type 12) with z = scale * zeta_2.  TAPE maps need desc.zeta. */
int32_t ts_write_vtk_micro(ts_ctx* ctx, double scale, int32_t format, const char* path);
/* The C++ mirror's host writers (include/twoscale/vtk.hpp) for a HOST state on the INI's
 * grids and map, as the reference CLI calls them (tools/twoscale.cpp:139-143): u, w
 * [n_macro], V [n_macro][n_micro]; either path may be NULL.  ASCII only. */
int32_t ts_write_vtk_ini(const char* ini_text, const double* u, const double* w, const double* V, double scale,
                         const char* macro_path, const char* micro_path);

#endif /* !__CUDACC_RTC__ */
#ifdef __cplusplus
}
#endif
#endif /* TWOSCALE_B200_H */
