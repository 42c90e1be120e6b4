// Launch interface of the generic (Q2 / 3D micro) kernels: gsetup.cu, gpcg.cu.
#pragma once

#include "generic_common.cuh"
#include "kernels.h"

namespace tsb {

struct GenProblem {
    GenGeom g;
    GridG macro;
    GenMap map;
    double kappa[4];
    double Dv;
    int role[6];
    int reaction_kind;
    double reaction_in, reaction_out, reaction_c[3], reaction_r;
    DataTapes data;  // macro-side tapes (fu, fw, Dw, dirichlet value)
};

void upload_gen_tables(const GenTables& t);      // gsetup.cu copy
void upload_gen_tables_pcg(const GenTables& t);  // gpcg.cu copy
GenTables make_gen_tables(int d, int p);
GenGeom make_gen_geom(int d, int p, const double* lo, const double* hi, const int* n);

// Generic cell cache, planar: out[((row * nq + q) * ncoef + k) * ncells + cell], k = J, A (upper
// triangle) — a warp's loads and stores of one (q, k) are contiguous across cells.
void launch_gcell_cache(const GenProblem& P, int rows, const double* points, double* out,
                        unsigned long long* first_bad, unsigned* err, cudaStream_t s, int row0 = 0);
void launch_gface_cache(const GenProblem& P, int rows, const double* points, int with_cells, double* out,
                        unsigned long long* first_bad, unsigned* err, cudaStream_t s);
void launch_gprobe(const GenProblem& P, const double* points, int with_cells, unsigned long long index, double* out,
                   cudaStream_t s);
void launch_gassemble(const GenProblem& P, int srows, const double* cells, const double* faces, double* stencil,
                      cudaStream_t s);
void launch_grhs_parts(const GenProblem& P, int n_nodes, int shared, const double* faces, double* rin, double* rout,
                       cudaStream_t s);
void launch_gmacro_qpoints(const GenProblem& P, const QuadTables& Q, double* gamma_in, double* gamma_out,
                           double* rhs_u_q, double* rhs_w_q, double* dw_q, unsigned long long* first_bad,
                           unsigned* err, cudaStream_t s);

// Streaming-stencil batched PCG for the generic path (operators too large for SMEM):
// coefficient planes stream from HBM every iteration, all CG vectors live in SMEM.
struct GenPcgArgs {
    int n_problems;
    GenGeom g;
    const double* stencil;     // [srows][ndirs / 2 + 1][n]: the centre and the upper half of the direction planes
    long long stencil_stride;  // 0 when shared
    const double* rin;
    const double* rout;
    double kappa1, kappa3;
    const double* u;
    const double* w;
    double* V;
    int warm;
    double tol;
    int maxit;
    int* iters;
    int* status;
    double* final_rel;
    int epilogue;
    double* res_v;
    double* bI;
    double* bO;
    const double* face_len;    // [rows][faces][nqf]
    long long face_len_stride;
    int role[6];
    int* counter;
    double* scratch;           // per-block vector storage when the problem exceeds SMEM
    const double* qstencil;    // 2D Q2: class-compact operator (q2_compact_doubles per row), or null
    long long qstencil_stride; // 0 when shared
    const double* tensor;      // 2D Q2: coefficient tensors (q2_tensor_doubles per row), or null
    long long tensor_stride;   // 0 when shared
};
int launch_gen_pcg(const GenPcgArgs& a, cudaStream_t s);  // returns launches issued (0 = does not fit)
// 2D Q2 class-compact operator: nodes grouped by lattice parity class (vertex, two edge
// kinds, cell interior), each class storing only its structurally nonzero directions
// (25 / 15 / 15 / 9), class-major.  Doubles per operator row (0 = not applicable).
size_t q2_compact_doubles(const GenGeom& g);
void launch_q2_repack(const GenGeom& g, int rows, const double* stencil, double* qstencil, cudaStream_t s);
// 2D Q2 matrix-free operator: per row 36 coefficient-tensor doubles per cell (colour-major,
// [colour][k][q][cell]) + 3 Robin face weights per face; 0 = not applicable or disabled
// (TS_GEN_Q2T=0).  Packed from the cell / face caches by launch_q2_tensor_pack (gsetup.cu).
size_t q2_tensor_doubles(const GenGeom& g);
void launch_q2_tensor_pack(const GenProblem& P, int rows, const double* cells, const double* faces, double* tensor,
                           cudaStream_t s);
void upload_q2t_tables();
// doubles of per-block global scratch the generic PCG needs (0 when it runs in SMEM)
size_t gen_pcg_scratch_doubles(const GenGeom& g);
size_t gen_pcg_smem_bytes(const GenGeom& g);

// surface_coupling over the generic faces for n_vec vectors (one warp each).
void launch_gcoupling(const GenGeom& g, const int* role6, int role, int n_vec, const double* v, const double* len,
                      long long len_stride, double* out, cudaStream_t s);
// micro_rhs for one node (generic: no fixed part).
void launch_gmicro_rhs(int n, const double* rin, const double* rout, double kappa1, double kappa3, double u, double w,
                       double* b, cudaStream_t s);

}  // namespace tsb
