// The C ABI (include/twoscale_b200.h): device-resident AssemblyContext and the
// fixed-point loop.  Host code here only allocates, launches, and moves a few
// scalars per sweep; all arithmetic of the path runs in the kernels of setup.cu
// and pcg.cu.  There is no CPU fallback: without a usable sm_100 device every
// entry point returns TS_ERR_CUDA.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>
#include <stdexcept>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "ctx_internal.h"

namespace tsb {

thread_local std::string g_err;
thread_local int g_err_index = -1;

BlockCache& BlockCache::get() {
    static BlockCache c;
    return c;
}

}  // namespace tsb


int tsb::device_ready() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
        return fail(TS_ERR_CUDA, "no CUDA device visible (the B200 path has no CPU fallback)");
    int dev = 0, major = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
    if (major != 10) return fail(TS_ERR_CUDA, "device compute capability %d.x is not sm_100", major);
    return TS_OK;
}

namespace {

// Degenerate-map check shared by the cache builds; message as mapping.cpp:50-55.
int check_degenerate(ts_ctx* c, const double* points, int with_cells, const char* what) {
    unsigned long long bad = 0;
    CU(cudaMemcpyAsync(&bad, c->first_bad.p, sizeof bad, cudaMemcpyDeviceToHost, c->stream));
    unsigned err = 0;
    CU(cudaMemcpyAsync(&err, c->err.p, sizeof err, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    if (err) return fail(TS_ERR_EXPR, "%s", expr_error(err));
    if (bad == ~0ULL) return TS_OK;
    DBuf<double> probe;
    probe.alloc(5);
    launch_degenerate_probe(c->P, points, with_cells, bad, probe.p, c->stream);
    double h[5];
    CU(cudaMemcpyAsync(h, probe.p, sizeof h, cudaMemcpyDeviceToHost, c->stream));
    c->sync();
    return fail(TS_ERR_DEGENERATE_MAP, "%s: det grad_y zeta = %g at x = (%g, %g), yhat = (%g, %g)", what,
                h[0], h[1], h[2], h[3], h[4]);
}


}  // namespace

void tsb::reset_flags(ts_ctx* c) {
    CU(cudaMemsetAsync(c->first_bad.p, 0xff, sizeof(unsigned long long), c->stream));
    CU(cudaMemsetAsync(c->err.p, 0, sizeof(unsigned), c->stream));
}

namespace {

// Micro half of the AssemblyContext for Q2 / 3D micro problems (configs 4-5):
// generic caches, operators (ndirs-point stencil planes) and rhs parts.
int build_generic_micro(ts_ctx* c, const ts_problem_desc* d) {
    const int mdim = d->micro_dim == 3 ? 3 : 2, morder = d->micro_order == 2 ? 2 : 1;
    if (mdim == 3 && morder == 2) return fail(TS_ERR_INVALID, "Q2 elements are supported on 2D micro grids only");
    if (mdim == 3 && d->map_kind == TS_MAP_TAPE)
        return fail(TS_ERR_INVALID, "3D micro maps must be tabulated (the expression language has y0, y1 only)");
    if (c->P.data.fv_hat.n)
        return fail(TS_ERR_INVALID, "f^v source terms are not supported for Q2/3D micro problems");
    for (int k = 0; k < 4; ++k)
        if (c->P.data.gv[k].n) return fail(TS_ERR_INVALID, "g^v corrections are not supported for Q2/3D micro problems");
    if (c->P.data.has_fu_flux || c->P.data.has_fw_flux)
        return fail(TS_ERR_INVALID, "flux functionals are not supported for Q2/3D micro problems");
    GenProblem& G = c->GP;
    const double lo[3] = {d->micro.lo[0], d->micro.lo[1], d->micro_lo2};
    const double hi[3] = {d->micro.hi[0], d->micro.hi[1], d->micro_hi2};
    const int n[3] = {d->micro.n[0], d->micro.n[1], d->micro_n2};
    if (mdim == 3 && (n[2] < 1 || !(lo[2] < hi[2]))) return fail(TS_ERR_INVALID, "invalid 3D micro extent");
    G.g = make_gen_geom(mdim, morder, lo, hi, n);
    G.macro = c->P.macro;
    G.map.kind = d->map_kind;
    G.map.op = c->P.map.op;
    G.map.arg = c->P.map.arg;
    G.map.val = c->P.map.val;
    for (int k = 0; k < 4; ++k) G.map.jac[k] = c->P.map.jac[k];
    G.map.table = c->A_table.p;
    G.map.tstride = d->map_kind == TS_MAP_FOURIER_TABLE ? 16 : mdim * mdim;
    G.map.s_kind = d->s_kind;
    G.map.amp = d->amp;
    G.map.macro = c->P.macro;
    if (mdim == 2) {
        for (int k = 0; k < 4; ++k) G.map.D[k] = d->D[k];
        G.map.D_identity = d->D[0] == 1.0 && d->D[1] == 0.0 && d->D[2] == 0.0 && d->D[3] == 1.0;
    } else {
        for (int k = 0; k < 9; ++k) G.map.D[k] = d->D3[k];
        G.map.D_identity = 0;
    }
    for (int k = 0; k < 4; ++k) G.kappa[k] = d->kappa[k];
    G.Dv = d->Dv;
    for (int k = 0; k < 4; ++k) G.role[k] = d->micro_role[k];
    G.role[4] = d->micro_role3[0];
    G.role[5] = d->micro_role3[1];
    G.reaction_kind = d->reaction_kind;
    if (d->reaction_kind == TS_REACTION_DISC) {
        G.reaction_in = d->reaction[0];
        G.reaction_out = d->reaction[1];
        G.reaction_c[0] = d->reaction[2];
        G.reaction_c[1] = d->reaction[3];
        G.reaction_c[2] = d->reaction_cz;
        G.reaction_r = d->reaction[4];
    } else {
        G.reaction_in = d->reaction[0];
    }
    G.data = c->P.data;
    const GenGeom& g = G.g;
    c->nm = g.nnodes;
    c->nfaces = g.nfaces;
    c->ncells = g.ncells;
    c->ncoef = 1 + mdim * (mdim + 1) / 2;
    const GenTables T = make_gen_tables(mdim, morder);
    upload_gen_tables(T);
    upload_gen_tables_pcg(T);
    // kernel (1)
    c->gcells.alloc((size_t)c->rows * g.ncells * g.nq * c->ncoef);
    c->gfaces.alloc((size_t)c->rows * g.nfaces * g.nqf);
    launch_gcell_cache(G, c->rows, nullptr, c->gcells.p, c->first_bad.p, c->err.p, c->stream);
    launch_gface_cache(G, c->rows, nullptr, 1, c->gfaces.p, c->first_bad.p, c->err.p, c->stream);
    CU(cudaGetLastError());
    {
        unsigned long long bad = 0;
        unsigned err = 0;
        CU(cudaMemcpyAsync(&bad, c->first_bad.p, sizeof bad, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaMemcpyAsync(&err, c->err.p, sizeof err, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        if (err) return fail(TS_ERR_EXPR, "%s", expr_error(err));
        if (bad != ~0ULL) {
            DBuf<double> probe;
            probe.alloc(6);
            launch_gprobe(G, nullptr, 1, bad, probe.p, c->stream);
            double h[6];
            CU(cudaMemcpyAsync(h, probe.p, sizeof h, cudaMemcpyDeviceToHost, c->stream));
            c->sync();
            if (mdim == 3)
                return fail(TS_ERR_DEGENERATE_MAP,
                            "degenerate map in cache build: det grad_y zeta = %g at x = (%g, %g), yhat = (%g, %g, %g)",
                            h[0], h[1], h[2], h[3], h[4], h[5]);
            return fail(TS_ERR_DEGENERATE_MAP,
                        "degenerate map in cache build: det grad_y zeta = %g at x = (%g, %g), yhat = (%g, %g)", h[0],
                        h[1], h[2], h[3], h[4]);
        }
    }
    // kernel (2)
    c->stencil.alloc((size_t)c->rows * (g.ndirs / 2 + 1) * g.nnodes);  // centre + upper half of the directions
    launch_gassemble(G, c->rows, c->gcells.p, c->gfaces.p, c->stencil.p, c->stream);
    if (const size_t td = q2_tensor_doubles(g)) {  // 2D Q2: matrix-free coefficient tensors
        upload_q2t_tables();
        c->tensor.alloc((size_t)c->rows * td);
        launch_q2_tensor_pack(G, c->rows, c->gcells.p, c->gfaces.p, c->tensor.p, c->stream);
    } else if (const size_t qd = q2_compact_doubles(g)) {  // 2D Q2: class-compact copy for the PCG
        c->qstencil.alloc((size_t)c->rows * qd);
        launch_q2_repack(g, c->rows, c->stencil.p, c->qstencil.p, c->stream);
    }
    c->has_fixed = false;
    if (const size_t sc = gen_pcg_scratch_doubles(g)) c->gscratch.alloc(sc);
    c->rin.alloc((size_t)c->nM * g.nnodes);
    c->rout.alloc((size_t)c->nM * g.nnodes);
    launch_grhs_parts(G, c->nM, c->shared, c->gfaces.p, c->rin.p, c->rout.p, c->stream);
    CU(cudaGetLastError());
    c->sync();
    c->gcells.release();  // recomputed on demand by ts_node_cache; gfaces stays (coupling weights)
    // pattern: every node pair sharing an element, rows lexicographic, columns ascending
    c->mrp.assign(g.nnodes + 1, 0);
    c->mci.clear();
    for (int node = 0; node < g.nnodes; ++node) {
        int ii[3], lo2[3] = {0, 0, 0}, hi2[3] = {0, 0, 0};
        gen_node_idx(g, node, ii);
        for (int a = 0; a < mdim; ++a) {
            int c0 = ii[a] > 0 ? (ii[a] - 1) / morder : 0, c1 = ii[a] / morder;
            if (c1 > g.nc[a] - 1) c1 = g.nc[a] - 1;
            lo2[a] = morder * c0;
            hi2[a] = morder * (c1 + 1);
        }
        for (int l = lo2[2]; l <= hi2[2]; ++l)
            for (int j = lo2[1]; j <= hi2[1]; ++j)
                for (int i = lo2[0]; i <= hi2[0]; ++i) c->mci.push_back(gen_node(g, i, j, l));
        c->mrp[node + 1] = (int)c->mci.size();
    }
    return TS_OK;
}

int build(ts_ctx* c, const ts_problem_desc* d) {
    if (!d) return fail(TS_ERR_INVALID, "null problem description");
    if (d->abi_version != TS_ABI_VERSION)
        return fail(TS_ERR_INVALID, "ABI version %d, library speaks %d", d->abi_version, TS_ABI_VERSION);
    for (const ts_grid_desc* g : {&d->macro, &d->micro}) {
        if (g->n[0] < 1 || g->n[1] < 1) return fail(TS_ERR_INVALID, "grid needs at least one cell per axis");
        if (!(g->lo[0] < g->hi[0] && g->lo[1] < g->hi[1]))
            return fail(TS_ERR_INVALID, "domain bounds must satisfy lo < hi componentwise");
    }
    if (d->map_kind != TS_MAP_TAPE && d->map_kind != TS_MAP_AFFINE_BUBBLE_TABLE && d->map_kind != TS_MAP_FOURIER_TABLE)
        return fail(TS_ERR_INVALID, "unknown map kind %d", d->map_kind);
    if (d->map_kind != TS_MAP_TAPE && !d->A_table)
        return fail(TS_ERR_INVALID, "tabulated map without A_table");
    std::vector<const ts_tape*> all = {&d->fv_hat, &d->fu, &d->fw, &d->Dw, &d->dirichlet_value};
    for (int k = 0; k < 4; ++k) {
        all.push_back(&d->jac[k]);
        all.push_back(&d->gv[k]);
        all.push_back(&d->gu2[k]);
        all.push_back(&d->gw[k]);
    }
    for (int k = 0; k < 2; ++k) {
        all.push_back(&d->fu_flux[k]);
        all.push_back(&d->fw_flux[k]);
        all.push_back(&d->zeta[k]);
    }
    for (const ts_tape* t : all)
        if (!check_tape(*t)) return fail(TS_ERR_INVALID, "malformed tape (null arrays or stack > %d)", TS_MAX_TAPE_STACK);
    if (int rc = device_ready()) return rc;

    CU(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CU(cudaMallocHost(&c->h_pinned, 64 * sizeof(double)));

    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    CU(cudaEventRecord(e0, c->stream));

    ProblemG& P = c->P;
    P.macro = to_grid(d->macro);
    P.micro = to_grid(d->micro);
    for (int k = 0; k < 4; ++k) {
        P.kappa[k] = d->kappa[k];
        P.macro_bc[k] = d->macro_bc[k];
        P.micro_role[k] = d->micro_role[k];
    }
    P.Dv = d->Dv;
    P.reaction_kind = d->reaction_kind;
    for (int k = 0; k < 5; ++k) P.reaction[k] = d->reaction[k];
    c->nM = P.macro.nodes();
    c->nm = P.micro.nodes();
    c->nfaces = P.micro.faces();
    c->ncells = P.micro.cells();
    c->Mcells = P.macro.cells();

    TapePack pack;
    for (int k = 0; k < 4; ++k) P.map.jac[k] = pack.add(d->jac[k]);
    DataTapes& T = P.data;
    T.fv_hat = pack.add(d->fv_hat);
    T.fu = pack.add(d->fu);
    T.fw = pack.add(d->fw);
    T.Dw = pack.add(d->Dw);
    T.dirichlet_value = pack.add(d->dirichlet_value);
    for (int k = 0; k < 4; ++k) {
        T.gv[k] = pack.add(d->gv[k]);
        T.gu2[k] = pack.add(d->gu2[k]);
        T.gw[k] = pack.add(d->gw[k]);
    }
    for (int k = 0; k < 2; ++k) {
        T.fu_flux[k] = pack.add(d->fu_flux[k]);
        T.fw_flux[k] = pack.add(d->fw_flux[k]);
    }
    T.has_fu_flux = d->has_fu_flux;
    T.has_fw_flux = d->has_fw_flux;
    for (int k = 0; k < 2; ++k) c->zeta[k] = pack.add(d->zeta[k]);
    c->has_zeta = d->zeta[0].n > 0 || d->zeta[1].n > 0;
    const size_t ninstr = pack.op.size() ? pack.op.size() : 1;
    pack.op.resize(ninstr, 0);
    pack.arg.resize(ninstr, 0);
    pack.val.resize(ninstr, 0.0);
    c->t_op.alloc(ninstr);
    c->t_arg.alloc(ninstr);
    c->t_val.alloc(ninstr);
    CU(cudaMemcpyAsync(c->t_op.p, pack.op.data(), ninstr * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(c->t_arg.p, pack.arg.data(), ninstr * sizeof(int), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(c->t_val.p, pack.val.data(), ninstr * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    P.map.kind = d->map_kind;
    P.map.op = c->t_op.p;
    P.map.arg = c->t_arg.p;
    P.map.val = c->t_val.p;
    P.map.s_kind = d->s_kind;
    P.map.amp = d->amp;
    P.map.macro = P.macro;
    for (int k = 0; k < 4; ++k) P.map.D[k] = d->D[k];
    P.map.D_identity = d->D[0] == 1.0 && d->D[1] == 0.0 && d->D[2] == 0.0 && d->D[3] == 1.0;
    const int mdim = d->micro_dim == 3 ? 3 : 2, morder = d->micro_order == 2 ? 2 : 1;
    // the generic kernels also take 2D Q1 micro grids too large for the SMEM-resident PCG
    c->gen = mdim == 3 || morder == 2 || d->force_generic || d->map_kind == TS_MAP_FOURIER_TABLE ||
             !micro_pcg_fits(to_grid(d->micro));
    if (d->map_kind == TS_MAP_AFFINE_BUBBLE_TABLE || d->map_kind == TS_MAP_FOURIER_TABLE) {
        const int ts = d->map_kind == TS_MAP_FOURIER_TABLE ? 16 : mdim * mdim;
        c->A_table.alloc((size_t)ts * c->nM);
        CU(cudaMemcpyAsync(c->A_table.p, d->A_table, c->A_table.bytes(), cudaMemcpyHostToDevice, c->stream));
        P.map.A_table = c->A_table.p;
    }
    c->shared = d->map_kind == TS_MAP_TAPE && !d->jac_depends_on_x;
    c->rows = c->shared ? std::min(1, c->nM) : c->nM;  // mapping.cpp:84
    c->Q = make_quad();
    upload_quad_tables(c->Q);

    c->first_bad.alloc(1);
    c->err.alloc(1);
    reset_flags(c);

    if (!c->gen) {
        // ---- kernel (1): node cache (cells + faces), mapping.cpp:79-129
        c->cells.alloc((size_t)c->rows * c->ncells * 4);
        c->faces.alloc((size_t)c->rows * c->nfaces * 2);
        launch_cell_cache(P, c->rows, nullptr, c->cells.p, c->first_bad.p, c->err.p, c->stream);
        launch_face_cache(P, c->rows, nullptr, 1, c->faces.p, c->first_bad.p, c->err.p, c->stream);
        CU(cudaGetLastError());
        if (int rc = check_degenerate(c, nullptr, 1, "degenerate map in cache build")) return rc;

        // ---- kernel (2): micro operators and rhs parts
        // the upper half of each micro operator (C, E, NW, N, NE planes): the kernels read
        // a_{-d}(k) = a_d(k - o_d), and ts_micro_values mirrors the lower half on demand
        c->stencil.alloc((size_t)c->rows * 5 * c->nm);
        launch_assemble_micro(P, c->rows, c->cells.p, c->faces.p, c->stencil.p, c->stream);
        c->has_fixed = T.fv_hat.n != 0;
        for (int k = 0; k < 4; ++k) c->has_fixed = c->has_fixed || T.gv[k].n != 0;
        if (c->has_fixed) c->fixed.alloc((size_t)c->nM * c->nm);
        c->rin.alloc((size_t)c->nM * c->nm);
        c->rout.alloc((size_t)c->nM * c->nm);
        launch_rhs_parts(P, c->nM, c->shared, c->cells.p, c->faces.p, c->fixed.p, c->rin.p, c->rout.p,
                         c->has_fixed, c->err.p, c->stream);
        c->face_len.alloc((size_t)c->rows * c->nfaces * 2);
        launch_face_len(c->rows, c->nfaces, c->faces.p, c->face_len.p, c->stream);
        CU(cudaGetLastError());
        q1_pattern(P.micro, c->mrp, c->mci);
    } else {
        if (int rc = build_generic_micro(c, d)) return rc;
    }

    // ---- macro systems, assembly.cpp:233-361
    q1_pattern(P.macro, c->Mrp, c->Mci);
    const int nnz = (int)c->Mci.size();
    c->d_Mrp.alloc(c->Mrp.size());
    c->d_Mci.alloc(c->Mci.size());
    CU(cudaMemcpyAsync(c->d_Mrp.p, c->Mrp.data(), c->d_Mrp.bytes(), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(c->d_Mci.p, c->Mci.data(), c->d_Mci.bytes(), cudaMemcpyHostToDevice, c->stream));
    const int nq = c->Mcells * 4;
    DBuf<double> qbuf;
    qbuf.alloc((size_t)5 * nq);
    if (!c->gen)
        launch_macro_qpoints(P, qbuf.p, qbuf.p + nq, qbuf.p + 2 * nq, qbuf.p + 3 * nq, qbuf.p + 4 * nq,
                             c->first_bad.p, c->err.p, c->stream);
    else
        launch_gmacro_qpoints(c->GP, c->Q, qbuf.p, qbuf.p + nq, qbuf.p + 2 * nq, qbuf.p + 3 * nq, qbuf.p + 4 * nq,
                              c->first_bad.p, c->err.p, c->stream);
    CU(cudaGetLastError());
    {
        unsigned long long bad = 0;
        unsigned err = 0;
        CU(cudaMemcpyAsync(&bad, c->first_bad.p, sizeof bad, cudaMemcpyDeviceToHost, c->stream));
        CU(cudaMemcpyAsync(&err, c->err.p, sizeof err, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        if (err) return fail(TS_ERR_EXPR, "%s", expr_error(err));
        if (bad != ~0ULL) {
            // qpoint_cache (assembly.cpp:69): re-probe the failing macro quadrature point
            const unsigned long long per = c->gen ? (unsigned long long)c->nfaces * c->GP.g.nqf : 2ULL * c->nfaces;
            const int qg = (int)(bad / per);
            double x[2];
            cell_pt(P.macro, qg / 4, c->Q.QS[qg % 4], c->Q.QT[qg % 4], x[0], x[1]);
            DBuf<double> dx;
            dx.alloc(2);
            CU(cudaMemcpy(dx.p, x, sizeof x, cudaMemcpyHostToDevice));
            reset_flags(c);
            unsigned long long local = bad % per;
            DBuf<double> probe;
            probe.alloc(6);
            if (c->gen)
                launch_gprobe(c->GP, dx.p, 0, local, probe.p, c->stream);
            else
                launch_degenerate_probe(P, dx.p, 0, local, probe.p, c->stream);
            double h[6] = {0, 0, 0, 0, 0, 0};
            CU(cudaMemcpyAsync(h, probe.p, (c->gen ? 6 : 5) * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            c->sync();
            if (c->gen && c->GP.g.d == 3)
                return fail(TS_ERR_DEGENERATE_MAP,
                            "degenerate map in cache build: det grad_y zeta = %g at x = (%g, %g), yhat = (%g, %g, %g)",
                            h[0], h[1], h[2], h[3], h[4], h[5]);
            return fail(TS_ERR_DEGENERATE_MAP,
                        "degenerate map in cache build: det grad_y zeta = %g at x = (%g, %g), yhat = (%g, %g)",
                        h[0], h[1], h[2], h[3], h[4]);
        }
    }
    c->Au.alloc(nnz);
    c->Aw.alloc(nnz);
    c->M0.alloc(nnz);
    c->bfix.alloc((size_t)2 * c->nM);
    launch_macro_assemble(P, c->d_Mrp.p, qbuf.p, qbuf.p + nq, qbuf.p + 2 * nq, qbuf.p + 3 * nq,
                          qbuf.p + 4 * nq, c->Au.p, c->Aw.p, c->M0.p, c->bfix.p, c->bfix.p + c->nM,
                          c->err.p, c->stream);
    CU(cudaGetLastError());

    // Dirichlet list: every node of every Dirichlet side, ascending (assembly.cpp:345-353)
    std::vector<char> mark(c->nM, 0);
    const GridG& M = P.macro;
    for (int f = 0; f < M.faces(); ++f) {
        int side, a, b;
        face_info(M, f, side, a, b);
        if (d->macro_bc[side] == TS_DIRICHLET) mark[a] = mark[b] = 1;
    }
    for (int i = 0; i < c->nM; ++i)
        if (mark[i]) c->dir_u.push_back(i);
    c->dir_u_val.assign(c->dir_u.size(), 0.0);
    c->w_pinned = d->kappa[2] == 0.0;  // assembly.cpp:357-360
    {
        DBuf<int> dd;
        DBuf<double> dv;
        dd.alloc(c->dir_u.size() + 1);
        dv.alloc(c->dir_u.size() + 1);
        if (!c->dir_u.empty()) {
            CU(cudaMemcpyAsync(dd.p, c->dir_u.data(), c->dir_u.size() * sizeof(int), cudaMemcpyHostToDevice, c->stream));
            launch_dirichlet_values(P, (int)c->dir_u.size(), dd.p, dv.p, c->err.p, c->stream);
            CU(cudaMemcpyAsync(c->dir_u_val.data(), dv.p, c->dir_u.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        }
        c->sync();
    }
    unsigned err = 0;
    CU(cudaMemcpy(&err, c->err.p, sizeof err, cudaMemcpyDeviceToHost));
    if (err) return fail(TS_ERR_EXPR, "%s", expr_error(err));

    // EliminatedOperator for u and w (solver.cpp:14-33)
    std::vector<unsigned char> hmask((size_t)2 * c->nM, 0);
    std::vector<double> hval((size_t)2 * c->nM, 0.0);
    for (size_t k = 0; k < c->dir_u.size(); ++k) {
        hmask[c->dir_u[k]] = 1;
        hval[c->dir_u[k]] = c->dir_u_val[k];
    }
    if (c->w_pinned) hmask[c->nM + 0] = 1;
    c->cmask.alloc(hmask.size());
    c->cval.alloc(hval.size());
    CU(cudaMemcpyAsync(c->cmask.p, hmask.data(), hmask.size(), cudaMemcpyHostToDevice, c->stream));
    CU(cudaMemcpyAsync(c->cval.p, hval.data(), hval.size() * sizeof(double), cudaMemcpyHostToDevice, c->stream));
    c->Ae.alloc((size_t)2 * nnz);
    c->shift.alloc((size_t)2 * c->nM);
    launch_eliminate(c->nM, c->d_Mrp.p, c->d_Mci.p, c->Au.p, c->cmask.p, c->cval.p, c->Ae.p, c->shift.p, c->stream);
    launch_eliminate(c->nM, c->d_Mrp.p, c->d_Mci.p, c->Aw.p, c->cmask.p + c->nM, c->cval.p + c->nM,
                     c->Ae.p + nnz, c->shift.p + c->nM, c->stream);
    CU(cudaGetLastError());

    // state
    c->uw.alloc((size_t)2 * c->nM);
    c->V.alloc((size_t)c->nM * c->nm);
    c->coupling.alloc((size_t)2 * c->nM);
    c->res_v.alloc(c->nM);
    c->final_rel.alloc(c->nM);
    c->raw.alloc((size_t)2 * c->nM);
    c->cons.alloc((size_t)2 * c->nM);
    c->cg_scratch.alloc((size_t)2 * 6 * c->nM);
    c->cg_partials.alloc((size_t)12 * csr_pcg_coop_blocks());
    c->cg_res_d.alloc(2);
    c->cg_res_i.alloc(6);
    {   // macro CG on the stencil kernel when the macro grid fits one SM's shared memory
        const char* e = std::getenv("TS_MACRO_STENCIL");
        c->macro_stencil = c->nM <= 8192 && micro_pcg_fits(c->P.macro) && !(e && e[0] == '0');
        c->macro_cluster = c->macro_stencil ? 0 : macro_cluster_size(c->P.macro);
        if (c->macro_stencil || c->macro_cluster) {
            c->mstencil.alloc((size_t)2 * 9 * c->nM);
            launch_csr_to_stencil(2, c->P.macro, c->d_Mrp.p, c->d_Mci.p, c->Ae.p, nnz, c->mstencil.p, c->stream);
            c->mzero.alloc(2);
            c->mzero.zero(c->stream);
            c->mrel.alloc(2);
            c->mstatus.alloc(2);
            c->miters.alloc(2);
            c->mcounter.alloc(1);
        }
    }
    c->sweep_out.alloc(8);
    c->iters.alloc(c->nM);
    c->order.alloc(c->nM);
    c->status.alloc(c->nM);
    c->counter.alloc(1);
    CU(cudaEventRecord(e1, c->stream));
    c->sync();
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, e0, e1));
    c->setup_ms = ms;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return TS_OK;
}

MicroPcgArgs micro_args(ts_ctx* c) {
    MicroPcgArgs a{};
    a.n_problems = c->nM;
    a.micro = c->P.micro;
    a.stencil = c->stencil.p;
    a.stencil_stride = c->shared ? 0 : 5LL * c->nm;
    a.plane_base = 0;
    a.fixed = c->fixed.p;
    a.rin = c->rin.p;
    a.rout = c->rout.p;
    a.has_fixed = c->has_fixed;
    a.kappa1 = c->P.kappa[0];
    a.kappa3 = c->P.kappa[2];
    a.u = c->uw.p;
    a.w = c->uw.p + c->nM;
    a.V = c->V.p;
    a.warm = 1;
    a.iters = c->iters.p;
    a.status = c->status.p;
    a.final_rel = c->final_rel.p;
    a.res_v = c->res_v.p;
    a.bI = c->coupling.p;
    a.bO = c->coupling.p + c->nM;
    a.face_len = c->face_len.p;
    a.face_len_stride = c->shared ? 0 : 2LL * c->nfaces;
    for (int k = 0; k < 4; ++k) a.micro_role[k] = c->P.micro_role[k];
    a.GW[0] = c->Q.GW[0];
    a.GW[1] = c->Q.GW[1];
    for (int q = 0; q < 2; ++q)
        for (int k = 0; k < 2; ++k) a.Nf[q][k] = c->Q.Nf[q][k];
    a.counter = c->counter.p;
    return a;
}

GenPcgArgs gen_args(ts_ctx* c) {
    GenPcgArgs a{};
    a.n_problems = c->nM;
    a.g = c->GP.g;
    a.stencil = c->stencil.p;
    a.stencil_stride = c->shared ? 0 : (long long)(c->GP.g.ndirs / 2 + 1) * c->nm;
    a.rin = c->rin.p;
    a.rout = c->rout.p;
    a.kappa1 = c->P.kappa[0];
    a.kappa3 = c->P.kappa[2];
    a.u = c->uw.p;
    a.w = c->uw.p + c->nM;
    a.V = c->V.p;
    a.warm = 1;
    a.iters = c->iters.p;
    a.status = c->status.p;
    a.final_rel = c->final_rel.p;
    a.res_v = c->res_v.p;
    a.bI = c->coupling.p;
    a.bO = c->coupling.p + c->nM;
    a.face_len = c->gfaces.p;
    a.face_len_stride = c->shared ? 0 : (long long)c->nfaces * c->GP.g.nqf;
    for (int k = 0; k < 6; ++k) a.role[k] = c->GP.role[k];
    a.counter = c->counter.p;
    a.scratch = c->gscratch.p;
    a.qstencil = c->qstencil.p;
    a.qstencil_stride = c->shared ? 0 : (long long)q2_compact_doubles(c->GP.g);
    a.tensor = c->tensor.p;
    a.tensor_stride = c->shared ? 0 : (long long)q2_tensor_doubles(c->GP.g);
    return a;
}

// Batched micro PCG on whichever path the context uses; returns launches (0 = no fit).
bool order_disabled() {
    const char* e = std::getenv("TS_ORDER");
    return e && e[0] == '0';
}

int launch_micro(ts_ctx* c, const MicroPcgArgs& ma, cudaStream_t s) {
    if (!c->gen) return launch_micro_pcg(ma, s);
    GenPcgArgs ga = gen_args(c);
    ga.u = ma.u;
    ga.w = ma.w;
    ga.V = ma.V;
    ga.warm = ma.warm;
    ga.tol = ma.tol;
    ga.maxit = ma.maxit;
    ga.iters = ma.iters;
    ga.status = ma.status;
    ga.final_rel = ma.final_rel;
    ga.epilogue = ma.epilogue;
    ga.res_v = ma.res_v;
    ga.bI = ma.bI;
    ga.bO = ma.bO;
    return launch_gen_pcg(ga, s);
}

void launch_coupling_any(ts_ctx* c, int role, int n_vec, const double* v, int row, long long stride, double* out,
                         cudaStream_t s) {
    if (!c->gen) {
        launch_coupling(c->P.micro, c->P.micro_role, role, n_vec, v, c->face_len.p + (size_t)row * 2 * c->nfaces, stride,
                        c->Q.GW, c->Q.Nf, out, s);
    } else {
        const long long per = (long long)c->nfaces * c->GP.g.nqf;
        launch_gcoupling(c->GP.g, c->GP.role, role, n_vec, v, c->gfaces.p + (size_t)row * per,
                         stride ? per : 0, out, s);
    }
}

MacroRhsArgs macro_rhs_args(ts_ctx* c) {
    MacroRhsArgs m{};
    m.n = c->nM;
    m.row_ptr = c->d_Mrp.p;
    m.col_idx = c->d_Mci.p;
    m.M0 = c->M0.p;
    for (int s = 0; s < 2; ++s) {
        m.b_fixed[s] = c->bfix.p + (size_t)s * c->nM;
        m.coupling[s] = c->coupling.p + (size_t)s * c->nM;
        m.shift[s] = c->shift.p + (size_t)s * c->nM;
        m.cmask[s] = c->cmask.p + (size_t)s * c->nM;
        m.cval[s] = c->cval.p + (size_t)s * c->nM;
        m.raw[s] = c->raw.p + (size_t)s * c->nM;
        m.constrained[s] = c->cons.p + (size_t)s * c->nM;
    }
    m.kappa[0] = c->P.kappa[1];
    m.kappa[1] = c->P.kappa[3];
    return m;
}

}  // namespace

extern "C" {

const char* ts_last_error(void) { return g_err.c_str(); }
int32_t ts_last_error_index(void) { return g_err_index; }
int32_t ts_abi_version(void) { return TS_ABI_VERSION; }

int32_t ts_device_ok(void) { return device_ready() == TS_OK ? 1 : 0; }

void ts_trim_device_cache(void) { BlockCache::get().trim(); }

int32_t ts_validate_map(ts_ctx* c, double lo, double hi, double* out, int32_t* pass) {
    if (!c || !out || !pass) return fail(TS_ERR_INVALID, "null argument");
    return guarded([&]() -> int {
        // recompute the node cache in row chunks (the build released it) and reduce det J
        const int blocks = 148 * 4;
        const bool gen = c->gen;
        const long long cells_per_row = gen ? (long long)c->GP.g.ncells * c->GP.g.nq : (long long)c->ncells * 4;
        const long long faces_per_row = gen ? (long long)c->GP.g.nfaces * c->GP.g.nqf : (long long)c->nfaces * 2;
        const int chunk = std::max(1, (int)std::min<long long>(c->rows, (256LL << 20) / (cells_per_row * 32 + 1)));
        DBuf<double> buf, fbuf, part;
        buf.alloc((size_t)chunk * cells_per_row * (gen ? c->ncoef : 4));
        fbuf.alloc((size_t)chunk * faces_per_row * (gen ? 1 : 4));
        part.alloc((size_t)blocks * 4);
        std::vector<double> hp((size_t)blocks * 4);
        double mn = 1e300, mx = -1e300;
        double where[4] = {-1, -1, -1, -1};
        reset_flags(c);
        for (int r0 = 0; r0 < c->rows; r0 += chunk) {
            const int nr = std::min(chunk, c->rows - r0);
            for (int kind = 0; kind < 2; ++kind) {
                long long count;
                int stride;
                if (kind == 0) {
                    if (gen) launch_gcell_cache(c->GP, nr, nullptr, buf.p, c->first_bad.p, c->err.p, c->stream, r0);
                    else launch_cell_cache(c->P, nr, nullptr, reinterpret_cast<double4*>(buf.p), c->first_bad.p, c->err.p, c->stream, r0);
                    count = nr * cells_per_row;
                    stride = gen ? c->ncoef : 4;
                } else {
                    if (gen) continue;  // generic face caches hold |nu| only; their det was checked at build
                                        // (ts_ctx_create fails on det <= 1e-12 anywhere)
                    launch_face_cache(c->P, nr, nullptr, 1, reinterpret_cast<double4*>(fbuf.p), c->first_bad.p, c->err.p, c->stream, r0);
                    count = nr * faces_per_row;
                    stride = 4;
                }
                if (gen && kind == 0)  // planar [row][q][k][cell]: det runs of ncells, k = 0
                    launch_det_minmax(buf.p, count, 1, part.p, blocks, c->stream, c->GP.g.ncells,
                                      (long long)c->ncoef * c->GP.g.ncells);
                else
                    launch_det_minmax(kind == 0 ? buf.p : fbuf.p, count, stride, part.p, blocks, c->stream);
                CU(cudaGetLastError());
                CU(cudaMemcpyAsync(hp.data(), part.p, hp.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
                c->sync();
                for (int b = 0; b < blocks; ++b) {
                    const long long per = kind == 0 ? cells_per_row : faces_per_row;
                    const int qn = kind == 0 ? (gen ? c->GP.g.nq : 4) : 2;
                    auto locate = [&](double idx, double* w) {
                        const long long t = (long long)idx;
                        const long long row = t / per, rem = t % per;
                        w[0] = (double)((c->shared ? 0 : r0) + row);
                        w[1] = kind;
                        if (gen && kind == 0) {  // planar: rem = q * ncells + cell
                            w[2] = (double)(rem % c->GP.g.ncells);
                            w[3] = (double)(rem / c->GP.g.ncells);
                        } else {
                            w[2] = (double)(rem / qn);
                            w[3] = (double)(rem % qn);
                        }
                    };
                    if (hp[4 * b + 1] >= 0 && hp[4 * b] < mn) {
                        mn = hp[4 * b];
                        locate(hp[4 * b + 1], where);
                    }
                    if (hp[4 * b + 3] >= 0 && hp[4 * b + 2] > mx) mx = hp[4 * b + 2];
                }
            }
        }
        out[0] = mn;
        out[1] = mx;
        for (int k = 0; k < 4; ++k) out[2 + k] = where[k];
        *pass = (mn >= lo && mx <= hi && mn > 0.0) ? 1 : 0;  // mapping.cpp:148
        return TS_OK;
    });
}

int32_t ts_select_device(int32_t device) {
    const cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return fail(TS_ERR_CUDA, "cudaSetDevice(%d): %s", device, cudaGetErrorString(e));
    return TS_OK;
}

void* ts_host_alloc(int64_t bytes) {
    void* p = nullptr;
    if (cudaMallocHost(&p, bytes > 0 ? (size_t)bytes : 1) != cudaSuccess) {
        fail(TS_ERR_CUDA, "cudaMallocHost(%lld) failed", (long long)bytes);
        return nullptr;
    }
    return p;
}

void ts_host_free(void* p) {
    if (p) cudaFreeHost(p);
}

int32_t ts_ctx_create(const ts_problem_desc* desc, ts_ctx** out) {
    if (!out) return fail(TS_ERR_INVALID, "null output handle");
    *out = nullptr;
    ts_ctx* c = new ts_ctx();
    const int rc = guarded([&] { return build(c, desc); });
    if (rc != TS_OK) {
        delete c;
        return rc;
    }
    *out = c;
    return TS_OK;
}

void ts_ctx_destroy(ts_ctx* ctx) { delete ctx; }

int32_t ts_ctx_get_info(const ts_ctx* c, ts_ctx_info* info) {
    if (!c || !info) return fail(TS_ERR_INVALID, "null argument");
    info->n_macro = c->nM;
    info->n_micro = c->nm;
    info->micro_nnz = (int)c->mci.size();
    info->macro_nnz = (int)c->Mci.size();
    info->n_micro_faces = c->nfaces;
    info->n_micro_cells = c->ncells;
    info->n_macro_cells = c->Mcells;
    info->shared_operator = c->shared && c->nM > 1;
    info->w_pinned = c->w_pinned;
    info->n_dirichlet_u = (int)c->dir_u.size();
    info->setup_ms = c->setup_ms;
    info->device_bytes = c->device_bytes();
    info->micro_kernel = c->tensor.p ? 4 : c->qstencil.p ? 3 : 2;
    info->micro_rows = 0;
    info->micro_smem_bytes = 0.0;
    info->macro_solver = c->macro_stencil ? 0 : c->macro_cluster ? 1 : 2;
    info->macro_cluster = c->macro_cluster;
    if (!c->gen) {
        const MicroPlan pl = plan_micro_pcg(c->P.micro, 0, c->nM);
        info->micro_kernel = pl.kernel;
        info->micro_rows = pl.R;
        info->micro_smem_bytes = pl.smem_bytes;
    }
    return TS_OK;
}

int32_t ts_ctx_default_opts(const ts_ctx* c, ts_solve_opts* o) {
    if (!c || !o) return fail(TS_ERR_INVALID, "null argument");
    *o = c->default_opts;
    return TS_OK;
}

// Internal: lets the INI front-end record the [solver] section and report errors.
void tsb_set_default_opts(ts_ctx* c, const ts_solve_opts* o) { c->default_opts = *o; }
int32_t ts_set_error_for_front_end(int32_t code, const char* msg) {
    g_err = msg;
    g_err_index = -1;
    return code;
}

int32_t ts_fixed_point_solve(ts_ctx* c, const ts_solve_opts* opts, ts_solve_report* rep,
                             double* history, int32_t history_cap) {
    if (!c || !opts) return fail(TS_ERR_INVALID, "null argument");
    return guarded([&]() -> int {
        ts_solve_report R{};
        R.w_pinned = c->w_pinned;
        R.micro_iters_min = 0x7fffffff;
        const int nM = c->nM, nnz = (int)c->Mci.size();
        cudaStream_t s = c->stream;
        cudaEvent_t ev[6];
        for (auto& e : ev) CU(cudaEventCreate(&e));
        CU(cudaEventRecord(ev[0], s));
        c->uw.zero(s);  // solver.cpp:67-69: u, w, V start at zero
        c->V.zero(s);
        c->coupling.zero(s);
        const MacroRhsArgs margs = macro_rhs_args(c);
        launch_macro_rhs(margs, s);
        R.gpu_launches += 1;
        MicroPcgArgs ma = micro_args(c);
        ma.tol = opts->inner_tol;
        ma.maxit = opts->inner_maxit;
        ma.epilogue = 1;
        CsrPcgArgs ca{};
        ca.n = nM;
        ca.n_sys = 2;
        ca.row_ptr = c->d_Mrp.p;
        ca.col_idx = c->d_Mci.p;
        ca.vals = c->Ae.p;
        ca.vals_stride = nnz;
        ca.b = c->cons.p;
        ca.x = c->uw.p;
        ca.scratch = c->cg_scratch.p;
        ca.tol = opts->inner_tol;
        ca.maxit = opts->inner_maxit;
        ca.result_i = c->cg_res_i.p;
        ca.result_d = c->cg_res_d.p;
        ca.partials = c->cg_partials.p;
        SweepResidualArgs ra{};
        ra.n_macro = nM;
        ra.n_micro = c->nm;
        ra.row_ptr = c->d_Mrp.p;
        ra.col_idx = c->d_Mci.p;
        ra.A_e[0] = c->Ae.p;
        ra.A_e[1] = c->Ae.p + nnz;
        ra.constrained[0] = c->cons.p;
        ra.constrained[1] = c->cons.p + nM;
        ra.x[0] = c->uw.p;
        ra.x[1] = c->uw.p + nM;
        ra.res_v = c->res_v.p;
        ra.iters = c->iters.p;
        ra.status = c->status.p;
        ra.final_rel = c->final_rel.p;
        ra.out = c->sweep_out.p;
        double* h = c->h_pinned;
        double prev = 0.0;
        int hist_n = 0;
        float micro_ms = 0.f, macro_ms = 0.f;
        int rc = TS_OK;
        MicroPcgArgs mm{};  // the two macro systems as stencil problems (c->macro_stencil / macro_cluster)
        if (c->macro_stencil || c->macro_cluster) {
            mm.n_problems = 2;
            mm.micro = c->P.macro;
            mm.stencil = c->mstencil.p;
            mm.stencil_stride = 9LL * nM;
            mm.plane_base = 4;
            mm.fixed = c->cons.p;  // b = constrained rhs; kappa1 = kappa3 = 0 below
            mm.rin = mm.rout = c->cons.p;
            mm.has_fixed = 1;
            mm.u = mm.w = c->mzero.p;
            mm.V = c->uw.p;        // warm start from the current u, w (solver.cpp:78-82)
            mm.warm = 1;
            mm.tol = opts->inner_tol;
            mm.maxit = opts->inner_maxit;
            mm.iters = c->miters.p;
            mm.status = c->mstatus.p;
            mm.final_rel = c->mrel.p;
            mm.epilogue = 0;
            mm.counter = c->mcounter.p;
        }
        // ---- one sweep's launches (src/solver.cpp:76-117), in three parts so the eager loop
        // can put events and the graph timestamps between them
        auto macro_part = [&]() -> int {  // macro u and w solves against the previous micro field
            if (c->macro_stencil) {
                CU(cudaMemsetAsync(c->mcounter.p, 0, sizeof(int), s));
                launch_micro_pcg(mm, s);
                launch_macro_cg_result(c->mstatus.p, c->miters.p, c->mrel.p, c->cg_res_i.p, c->cg_res_d.p, s);
            } else if (c->macro_cluster && (c->macro_cluster = launch_macro_cluster(mm, c->macro_cluster, s))) {
                launch_macro_cg_result(c->mstatus.p, c->miters.p, c->mrel.p, c->cg_res_i.p, c->cg_res_d.p, s);
            } else {
                c->macro_cluster = 0;  // could not launch here: cooperative CSR CG from now on
                launch_csr_pcg(ca, s);
                return 1;
            }
            return 2;
        };
        auto micro_part = [&](int sweep) -> int {  // all micro solves with the fresh macro values (solver.cpp:85-98)
            int n = 0;
            CU(cudaMemsetAsync(c->counter.p, 0, sizeof(int), s));
            // from sweep 2 on, hand out the problems longest-first (previous sweep's counts)
            ma.order = nullptr;
            if (sweep > 1 && !c->gen && !order_disabled()) {
                launch_order_by_iters(nM, c->iters.p, c->order.p, s);
                ma.order = c->order.p;
                ++n;
            }
            const int nl = launch_micro(c, ma, s);
            return nl ? n + nl : -1;
        };
        auto rhs_part = [&]() -> int {
            // residuals against the freshest data (solver.cpp:100-117); the raw rhs of this
            // step is also next sweep's rhs (V is unchanged in between)
            launch_macro_rhs(margs, s);
            launch_sweep_residual(ra, s);
            return 2;
        };
        // ---- the host's view of a finished sweep (h: sweep_out[8], cg_res_d[2], cg_res_i[6])
        // returns true when the loop stops (converged, or rc set to the reference's error)
        auto post_sweep = [&](int sweep, const double* hh) -> bool {
            const int* cg = reinterpret_cast<const int*>(hh + 10);
            for (int sys = 0; sys < 2; ++sys) {
                const char* label = sys == 0 ? "macro u-system" : "macro w-system";
                if (cg[3 * sys + 2]) {
                    rc = fail(TS_ERR_SOLVER, "%s: CG detected negative curvature (matrix not SPD)", label);
                    return true;
                }
                if (!cg[3 * sys]) {
                    rc = fail(TS_ERR_SOLVER, "%s: CG failed to converge, relative residual %f after %d iterations",
                              label, hh[8 + sys], cg[3 * sys + 1]);
                    return true;
                }
            }
            if (hh[4] >= 0) {
                const int bad = (int)hh[4];
                g_err_index = bad;
                if ((int)hh[5] == 1)
                    rc = fail(TS_ERR_SOLVER, "micro system %d: CG detected negative curvature", bad);
                else
                    rc = fail(TS_ERR_SOLVER, "micro system %d: CG failed to converge, relative residual %f", bad, hh[6]);
                g_err_index = bad;
                return true;
            }
            const double residual = hh[0];
            R.micro_dof_iters += hh[1];
            R.micro_iters_max = std::max(R.micro_iters_max, (int)hh[2]);
            R.micro_iters_min = std::min(R.micro_iters_min, (int)hh[3]);
            if (history && hist_n < history_cap) history[hist_n] = residual;
            ++hist_n;
            R.sweeps = sweep;
            R.final_residual = residual;
            if (residual < opts->outer_tol || (sweep >= 2 && std::fabs(residual - prev) < opts->outer_tol)) {
                R.converged = 1;  // solver.cpp:124-125
                return true;
            }
            prev = residual;
            return false;
        };
        // ---- sweeps 2.. on the device: one CUDA graph whose conditional while node repeats
        // the sweep's launches + k_sweep_control (the stop test) with no host round trip.
        // Used where the per-sweep round trip is a visible share (small problems) and the
        // macro solve is graph-capturable (stencil kernel or cluster).
        bool use_graph = (double)nM * c->nm <= 8e6 && (c->macro_stencil || c->macro_cluster) && opts->max_outer > 1;
        if (const char* e = std::getenv("TS_GRAPH")) use_graph = e[0] == '1' ? (c->macro_stencil || c->macro_cluster) && opts->max_outer > 1 : false;
        auto build_graph = [&]() -> bool {
            const double key[4] = {opts->inner_tol, (double)opts->inner_maxit, opts->outer_tol, (double)opts->max_outer};
            if (c->sweep_graph && std::memcmp(key, c->graph_key, sizeof key) == 0 && c->sweep_log.n >= (size_t)kSweepLog * opts->max_outer)
                return true;
            if (c->sweep_graph) {
                cudaGraphExecDestroy(c->sweep_graph);
                c->sweep_graph = nullptr;
            }
            c->sweep_log.alloc((size_t)kSweepLog * opts->max_outer);
            c->stamps.alloc((size_t)4 * opts->max_outer);
            c->ctl_buf.alloc(2);
            cudaGraph_t g = nullptr;
            cudaGraphConditionalHandle hnd;
            if (cudaGraphCreate(&g, 0) != cudaSuccess) return false;
            bool ok = cudaGraphConditionalHandleCreate(&hnd, g, 1, cudaGraphCondAssignDefault) == cudaSuccess;
            cudaGraphNodeParams np{};
            np.type = cudaGraphNodeTypeConditional;
            np.conditional.handle = hnd;
            np.conditional.type = cudaGraphCondTypeWhile;
            np.conditional.size = 1;
            cudaGraphNode_t node;
            ok = ok && cudaGraphAddNode(&node, g, nullptr, 0, &np) == cudaSuccess;
            if (ok) {
                cudaGraph_t body = np.conditional.phGraph_out[0];
                ok = cudaStreamBeginCaptureToGraph(s, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed) == cudaSuccess;
                if (ok) {
                    SweepCtl* ctl = reinterpret_cast<SweepCtl*>(c->ctl_buf.p);
                    int n = 0, nm = -1;
                    try {
                        launch_sweep_stamp(ctl, c->stamps.p, 0, s);
                        n += macro_part();
                        launch_sweep_stamp(ctl, c->stamps.p, 1, s);
                        nm = micro_part(2);
                        launch_sweep_stamp(ctl, c->stamps.p, 2, s);
                        n += rhs_part();
                        launch_sweep_stamp(ctl, c->stamps.p, 3, s);
                        launch_sweep_control(ctl, c->sweep_out.p, c->cg_res_d.p, c->cg_res_i.p, c->sweep_log.p,
                                             opts->outer_tol, opts->max_outer, hnd, s);
                    } catch (...) {  // a failed call inside the capture: end it, run eagerly
                        nm = -1;
                    }
                    cudaGraph_t out = nullptr;
                    ok = cudaStreamEndCapture(s, &out) == cudaSuccess && nm > 0;
                    c->graph_launches = n + nm + 5;
                }
            }
            ok = ok && cudaGraphInstantiate(&c->sweep_graph, g, 0) == cudaSuccess;
            cudaGraphDestroy(g);
            if (!ok) {
                if (c->sweep_graph) cudaGraphExecDestroy(c->sweep_graph);
                c->sweep_graph = nullptr;
                cudaGetLastError();
                return false;
            }
            std::memcpy(c->graph_key, key, sizeof key);
            return true;
        };
        auto run_graph = [&](int sweep) -> bool {  // sweeps `sweep`.. ; false: could not build
            if (!build_graph()) return false;
            SweepCtl h0{};
            h0.sweep = sweep - 1;
            h0.prev = prev;
            std::memcpy(h, &h0, sizeof h0);
            CU(cudaMemcpyAsync(c->ctl_buf.p, h, sizeof h0, cudaMemcpyHostToDevice, s));
            CU(cudaGraphLaunch(c->sweep_graph, s));
            CU(cudaMemcpyAsync(h, c->ctl_buf.p, sizeof h0, cudaMemcpyDeviceToHost, s));
            c->sync();
            SweepCtl h1;
            std::memcpy(&h1, h, sizeof h1);
            const int done = h1.sweep;
            std::vector<double> log((size_t)kSweepLog * done);
            std::vector<unsigned long long> st((size_t)4 * done);
            CU(cudaMemcpy(log.data(), c->sweep_log.p, log.size() * sizeof(double), cudaMemcpyDeviceToHost));
            CU(cudaMemcpy(st.data(), c->stamps.p, st.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
            for (int k = sweep - 1; k < done; ++k) {
                const unsigned long long* t = st.data() + 4 * k;
                micro_ms += (float)((t[2] - t[1]) * 1e-6);
                macro_ms += (float)((t[1] - t[0]) * 1e-6 + (t[3] - t[2]) * 1e-6);
                R.gpu_launches += c->graph_launches;
                if (post_sweep(k + 1, log.data() + (size_t)kSweepLog * k)) break;
            }
            return true;
        };

        for (int sweep = 1; sweep <= opts->max_outer; ++sweep) {
            if (sweep == 2 && use_graph && run_graph(sweep)) break;
            CU(cudaEventRecord(ev[1], s));
            R.gpu_launches += macro_part();
            CU(cudaGetLastError());
            CU(cudaEventRecord(ev[2], s));
            const int nl = micro_part(sweep);
            if (nl < 0) {
                rc = fail(TS_ERR_INVALID, "micro grid %dx%d does not fit the shared-memory batched PCG",
                          c->P.micro.n0, c->P.micro.n1);
                break;
            }
            CU(cudaGetLastError());
            R.gpu_launches += nl;
            CU(cudaEventRecord(ev[3], s));
            R.gpu_launches += rhs_part();
            CU(cudaGetLastError());
            CU(cudaEventRecord(ev[4], s));
            CU(cudaMemcpyAsync(h, c->sweep_out.p, 8 * sizeof(double), cudaMemcpyDeviceToHost, s));
            CU(cudaMemcpyAsync(h + 8, c->cg_res_d.p, 2 * sizeof(double), cudaMemcpyDeviceToHost, s));
            CU(cudaMemcpyAsync(reinterpret_cast<int*>(h + 10), c->cg_res_i.p, 6 * sizeof(int),
                               cudaMemcpyDeviceToHost, s));
            c->sync();
            float t;
            CU(cudaEventElapsedTime(&t, ev[2], ev[3]));
            micro_ms += t;
            CU(cudaEventElapsedTime(&t, ev[1], ev[2]));
            macro_ms += t;
            CU(cudaEventElapsedTime(&t, ev[3], ev[4]));
            macro_ms += t;
            if (post_sweep(sweep, h)) break;
        }
        CU(cudaEventRecord(ev[5], s));
        c->sync();
        float tot = 0.f;
        CU(cudaEventElapsedTime(&tot, ev[0], ev[5]));
        for (auto& e : ev) cudaEventDestroy(e);
        R.micro_ms = micro_ms;
        R.macro_ms = macro_ms;
        R.total_ms = tot;
        if (R.micro_iters_min == 0x7fffffff) R.micro_iters_min = 0;
        if (rep) *rep = R;
        c->state_valid = true;
        return rc;
    });
}

int32_t ts_download_state(ts_ctx* c, double* u, double* w, double* V) {
    if (!c) return fail(TS_ERR_INVALID, "null context");
    return guarded([&]() -> int {
        if (u) CU(cudaMemcpyAsync(u, c->uw.p, c->nM * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        if (w) CU(cudaMemcpyAsync(w, c->uw.p + c->nM, c->nM * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        if (V) CU(cudaMemcpyAsync(V, c->V.p, c->V.bytes(), cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        return TS_OK;
    });
}

int32_t ts_micro_solve(ts_ctx* c, const double* u, const double* w, const double* V_in, double tol,
                       int32_t maxit, double* V_out, int32_t* iters, ts_solve_report* rep) {
    if (!c || !u || !w || !V_out) return fail(TS_ERR_INVALID, "null argument");
    return guarded([&]() -> int {
        cudaStream_t s = c->stream;
        const int nM = c->nM;
        DBuf<double> uw, V, fr, rv, cp;
        DBuf<int> it, st;
        uw.alloc(2 * (size_t)nM);
        V.alloc((size_t)nM * c->nm);
        fr.alloc(nM);
        rv.alloc(nM);
        cp.alloc(2 * (size_t)nM);
        it.alloc(nM);
        st.alloc(nM);
        CU(cudaMemcpyAsync(uw.p, u, nM * sizeof(double), cudaMemcpyHostToDevice, s));
        CU(cudaMemcpyAsync(uw.p + nM, w, nM * sizeof(double), cudaMemcpyHostToDevice, s));
        if (V_in)
            CU(cudaMemcpyAsync(V.p, V_in, V.bytes(), cudaMemcpyHostToDevice, s));
        MicroPcgArgs a = micro_args(c);
        a.u = uw.p;
        a.w = uw.p + nM;
        a.V = V.p;
        a.warm = V_in != nullptr;
        a.tol = tol;
        a.maxit = maxit;
        a.iters = it.p;
        a.status = st.p;
        a.final_rel = fr.p;
        a.epilogue = 0;
        a.res_v = rv.p;
        a.bI = cp.p;
        a.bO = cp.p + nM;
        cudaEvent_t e0, e1;
        CU(cudaEventCreate(&e0));
        CU(cudaEventCreate(&e1));
        CU(cudaMemsetAsync(c->counter.p, 0, sizeof(int), s));
        CU(cudaEventRecord(e0, s));
        const int nl = launch_micro(c, a, s);
        if (!nl) return fail(TS_ERR_INVALID, "micro grid too large for the shared-memory PCG kernel");
        CU(cudaEventRecord(e1, s));
        CU(cudaGetLastError());
        std::vector<int> hit(nM), hst(nM);
        std::vector<double> hfr(nM);
        CU(cudaMemcpyAsync(V_out, V.p, V.bytes(), cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(hit.data(), it.p, nM * sizeof(int), cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(hst.data(), st.p, nM * sizeof(int), cudaMemcpyDeviceToHost, s));
        CU(cudaMemcpyAsync(hfr.data(), fr.p, nM * sizeof(double), cudaMemcpyDeviceToHost, s));
        c->sync();
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        ts_solve_report R{};
        R.micro_ms = ms;
        R.total_ms = ms;
        R.gpu_launches = nl;
        R.micro_iters_min = 0x7fffffff;
        for (int i = 0; i < nM; ++i) {
            if (iters) iters[i] = hit[i];
            R.micro_dof_iters += (double)c->nm * hit[i];
            R.micro_iters_max = std::max(R.micro_iters_max, hit[i]);
            R.micro_iters_min = std::min(R.micro_iters_min, hit[i]);
        }
        R.converged = 1;
        if (rep) *rep = R;
        for (int i = 0; i < nM; ++i)
            if (hst[i] != 0) {
                g_err_index = i;
                if (hst[i] == 1) return fail(TS_ERR_SOLVER, "micro system %d: CG detected negative curvature", i);
                return fail(TS_ERR_SOLVER, "micro system %d: CG failed to converge, relative residual %f", i, hfr[i]);
            }
        return TS_OK;
    });
}

int32_t ts_micro_pattern(const ts_ctx* c, int32_t* row_ptr, int32_t* col_idx) {
    if (!c) return fail(TS_ERR_INVALID, "null context");
    if (row_ptr) std::memcpy(row_ptr, c->mrp.data(), c->mrp.size() * sizeof(int));
    if (col_idx) std::memcpy(col_idx, c->mci.data(), c->mci.size() * sizeof(int));
    return TS_OK;
}

int32_t ts_micro_values(const ts_ctx* cc, int32_t node, double* vals) {
    ts_ctx* c = const_cast<ts_ctx*>(cc);
    if (!c || !vals) return fail(TS_ERR_INVALID, "null argument");
    if (node < 0 || node >= c->nM) return fail(TS_ERR_INVALID, "node %d out of range", node);
    return guarded([&]() -> int {
        const int row = c->shared ? 0 : node, n = c->nm;
        const int nd = c->gen ? c->GP.g.ndirs / 2 + 1 : 5;  // stored planes: the centre and the upper half
        std::vector<double> st((size_t)nd * n);
        CU(cudaMemcpyAsync(st.data(), c->stencil.p + (size_t)row * nd * n, st.size() * sizeof(double),
                           cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        if (c->gen) {
            const GenGeom& g = c->GP.g;
            const int span = 2 * g.p + 1;
            for (int r = 0; r < n; ++r) {
                int ii[3], jj[3];
                gen_node_idx(g, r, ii);
                for (int k = c->mrp[r]; k < c->mrp[r + 1]; ++k) {
                    gen_node_idx(g, c->mci[k], jj);
                    int dir = 0, mul = 1;
                    for (int a = 0; a < g.d; ++a) {
                        dir += (jj[a] - ii[a] + g.p) * mul;
                        mul *= span;
                    }
                    // lower half by symmetry: a_d(r) = a_{ndirs-1-d}(column node)
                    const int ctr = g.ndirs / 2;
                    vals[k] = dir >= ctr ? st[(size_t)(dir - ctr) * n + r] : st[(size_t)(ctr - dir) * n + c->mci[k]];
                }
            }
            return TS_OK;
        }
        const int nx = c->P.micro.n0 + 1;
        for (int r = 0; r < n; ++r) {
            const int i = r % nx, j = r / nx;
            for (int k = c->mrp[r]; k < c->mrp[r + 1]; ++k) {
                const int cc2 = c->mci[k];
                const int di = cc2 % nx - i, dj = cc2 / nx - j;
                const int d = (dj + 1) * 3 + di + 1;
                // lower half (d < 4) by symmetry: a_d(r) = a_{8-d}(r + o_d), the column node's entry
                vals[k] = d >= 4 ? st[(size_t)(d - 4) * n + r] : st[(size_t)(4 - d) * n + cc2];
            }
        }
        return TS_OK;
    });
}

int32_t ts_micro_rhs(const ts_ctx* cc, int32_t node, double u, double w, double* b) {
    ts_ctx* c = const_cast<ts_ctx*>(cc);
    if (!c || !b) return fail(TS_ERR_INVALID, "null argument");
    if (node < 0 || node >= c->nM) return fail(TS_ERR_INVALID, "node %d out of range", node);
    return guarded([&]() -> int {
        const size_t off = (size_t)node * c->nm;
        DBuf<double> d;
        d.alloc(c->nm);
        if (c->gen)
            launch_gmicro_rhs(c->nm, c->rin.p + off, c->rout.p + off, c->P.kappa[0], c->P.kappa[2], u, w, d.p, c->stream);
        else
            launch_micro_rhs(c->nm, c->has_fixed ? c->fixed.p + off : nullptr, c->rin.p + off, c->rout.p + off,
                             c->has_fixed, c->P.kappa[0], c->P.kappa[2], u, w, d.p, c->stream);
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(b, d.p, d.bytes(), cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        return TS_OK;
    });
}

int32_t ts_node_cache(const ts_ctx* cc, int32_t node, double* cells, double* faces) {
    ts_ctx* c = const_cast<ts_ctx*>(cc);
    if (!c) return fail(TS_ERR_INVALID, "null context");
    if (node < 0 || node >= c->nM) return fail(TS_ERR_INVALID, "node %d out of range", node);
    return guarded([&]() -> int {
        // one cache row recomputed by kernel (1) — bit-identical to the row used in assembly
        const int row = c->shared ? 0 : node;
        reset_flags(c);
        if (c->gen) {
            const GenGeom& g = c->GP.g;
            const size_t cper = (size_t)g.ncells * g.nq * c->ncoef, fper = (size_t)g.nfaces * g.nqf;
            if (cells) {
                DBuf<double> tmp;
                tmp.alloc(cper);
                launch_gcell_cache(c->GP, 1, nullptr, tmp.p, c->first_bad.p, c->err.p, c->stream, row);
                CU(cudaGetLastError());
                std::vector<double> planar(cper);
                CU(cudaMemcpyAsync(planar.data(), tmp.p, cper * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
                c->sync();
                const int nc = c->ncoef;  // planar [q][k][cell] -> the API's [cell][q][k]
                for (int q = 0; q < g.nq; ++q)
                    for (int k = 0; k < nc; ++k)
                        for (int cell = 0; cell < g.ncells; ++cell)
                            cells[((size_t)cell * g.nq + q) * nc + k] = planar[((size_t)q * nc + k) * g.ncells + cell];
            }
            if (faces)
                CU(cudaMemcpyAsync(faces, c->gfaces.p + row * fper, fper * sizeof(double), cudaMemcpyDeviceToHost,
                                   c->stream));
            c->sync();
            return TS_OK;
        }
        if (cells) {
            DBuf<double4> tmp;
            tmp.alloc((size_t)c->ncells * 4);
            launch_cell_cache(c->P, 1, nullptr, tmp.p, c->first_bad.p, c->err.p, c->stream, row);
            CU(cudaGetLastError());
            CU(cudaMemcpyAsync(cells, tmp.p, tmp.bytes(), cudaMemcpyDeviceToHost, c->stream));
            c->sync();
        }
        if (faces) {
            DBuf<double4> tmp;
            tmp.alloc((size_t)c->nfaces * 2);
            launch_face_cache(c->P, 1, nullptr, 1, tmp.p, c->first_bad.p, c->err.p, c->stream, row);
            CU(cudaGetLastError());
            CU(cudaMemcpyAsync(faces, tmp.p, tmp.bytes(), cudaMemcpyDeviceToHost, c->stream));
            c->sync();
        }
        return TS_OK;
    });
}

int32_t ts_macro_matrix(const ts_ctx* cc, int32_t which, int32_t* row_ptr, int32_t* col_idx, double* vals) {
    ts_ctx* c = const_cast<ts_ctx*>(cc);
    if (!c) return fail(TS_ERR_INVALID, "null context");
    if (which < 0 || which > 2) return fail(TS_ERR_INVALID, "which must be 0 (A_u), 1 (A_w) or 2 (M0)");
    return guarded([&]() -> int {
        if (row_ptr) std::memcpy(row_ptr, c->Mrp.data(), c->Mrp.size() * sizeof(int));
        if (col_idx) std::memcpy(col_idx, c->Mci.data(), c->Mci.size() * sizeof(int));
        const double* src = which == 0 ? c->Au.p : which == 1 ? c->Aw.p : c->M0.p;
        if (vals) {
            CU(cudaMemcpyAsync(vals, src, c->Mci.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            c->sync();
        }
        return TS_OK;
    });
}

int32_t ts_macro_rhs(ts_ctx* c, int32_t which, const double* V, double* out) {
    if (!c || !out) return fail(TS_ERR_INVALID, "null argument");
    if (which < 0 || which > 1) return fail(TS_ERR_INVALID, "which must be 0 (u) or 1 (w)");
    return guarded([&]() -> int {
        cudaStream_t s = c->stream;
        DBuf<double> dV, cp, raw, cons;
        cp.alloc(2 * (size_t)c->nM);
        raw.alloc(2 * (size_t)c->nM);
        cons.alloc(2 * (size_t)c->nM);
        cp.zero(s);
        if (V) {
            dV.alloc((size_t)c->nM * c->nm);
            CU(cudaMemcpyAsync(dV.p, V, dV.bytes(), cudaMemcpyHostToDevice, s));
            for (int role = 0; role < 2; ++role)
                launch_coupling_any(c, role, c->nM, dV.p, 0, c->shared ? 0 : 2LL * c->nfaces,
                                    cp.p + (size_t)role * c->nM, s);
        }
        MacroRhsArgs m = macro_rhs_args(c);
        for (int k = 0; k < 2; ++k) {
            m.coupling[k] = cp.p + (size_t)k * c->nM;
            m.raw[k] = raw.p + (size_t)k * c->nM;
            m.constrained[k] = cons.p + (size_t)k * c->nM;
        }
        launch_macro_rhs(m, s);
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(out, raw.p + (size_t)which * c->nM, c->nM * sizeof(double), cudaMemcpyDeviceToHost, s));
        c->sync();
        return TS_OK;
    });
}

int32_t ts_dirichlet(const ts_ctx* c, int32_t which, int32_t* n, int32_t* dofs, double* vals) {
    if (!c || !n) return fail(TS_ERR_INVALID, "null argument");
    if (which == 0) {
        *n = (int)c->dir_u.size();
        for (size_t k = 0; k < c->dir_u.size(); ++k) {
            if (dofs) dofs[k] = c->dir_u[k];
            if (vals) vals[k] = c->dir_u_val[k];
        }
    } else {
        *n = c->w_pinned ? 1 : 0;
        if (c->w_pinned) {
            if (dofs) dofs[0] = 0;
            if (vals) vals[0] = 0.0;
        }
    }
    return TS_OK;
}

int32_t ts_surface_coupling(ts_ctx* c, const double* v, int32_t node, int32_t role, double* out) {
    if (!c || !v || !out) return fail(TS_ERR_INVALID, "null argument");
    if (node < 0 || node >= c->nM) return fail(TS_ERR_INVALID, "node %d out of range", node);
    return guarded([&]() -> int {
        DBuf<double> dv, r;
        dv.alloc(c->nm);
        r.alloc(1);
        CU(cudaMemcpyAsync(dv.p, v, dv.bytes(), cudaMemcpyHostToDevice, c->stream));
        const int row = c->shared ? 0 : node;
        launch_coupling_any(c, role, 1, dv.p, row, 0, r.p, c->stream);
        CU(cudaGetLastError());
        CU(cudaMemcpyAsync(out, r.p, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        return TS_OK;
    });
}

int32_t ts_cg_solve(int32_t n, const int32_t* row_ptr, const int32_t* col_idx, const double* vals,
                    const double* b, double* x, double tol, int32_t maxit, ts_cg_result* result) {
    if (n < 0 || !row_ptr || !col_idx || !vals || !b || !x) return fail(TS_ERR_INVALID, "null argument");
    if (int rc = device_ready()) return rc;
    return guarded([&]() -> int {
        if (n == 0) {
            if (result) *result = ts_cg_result{1, 0, 0, 0.0};
            return TS_OK;
        }
        const int nnz = row_ptr[n];
        DBuf<int> rp, ci, ri;
        DBuf<double> v, bb, xx, sc, rd;
        rp.alloc(n + 1);
        ci.alloc(nnz);
        v.alloc(nnz);
        bb.alloc(n);
        xx.alloc(n);
        sc.alloc((size_t)5 * n);
        ri.alloc(3);
        rd.alloc(1);
        CU(cudaMemcpy(rp.p, row_ptr, rp.bytes(), cudaMemcpyHostToDevice));
        CU(cudaMemcpy(ci.p, col_idx, ci.bytes(), cudaMemcpyHostToDevice));
        CU(cudaMemcpy(v.p, vals, v.bytes(), cudaMemcpyHostToDevice));
        CU(cudaMemcpy(bb.p, b, bb.bytes(), cudaMemcpyHostToDevice));
        CU(cudaMemcpy(xx.p, x, xx.bytes(), cudaMemcpyHostToDevice));
        CsrPcgArgs a{};
        a.n = n;
        a.n_sys = 1;
        a.row_ptr = rp.p;
        a.col_idx = ci.p;
        a.vals = v.p;
        a.b = bb.p;
        a.x = xx.p;
        a.scratch = sc.p;
        a.tol = tol;
        a.maxit = maxit;
        a.result_i = ri.p;
        a.result_d = rd.p;
        launch_csr_pcg(a, 0);
        CU(cudaGetLastError());
        int hi[3];
        double hd;
        CU(cudaMemcpy(x, xx.p, xx.bytes(), cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(hi, ri.p, sizeof hi, cudaMemcpyDeviceToHost));
        CU(cudaMemcpy(&hd, rd.p, sizeof hd, cudaMemcpyDeviceToHost));
        if (result) *result = ts_cg_result{hi[0], hi[1], hi[2], hd};
        return TS_OK;
    });
}

}  // extern "C"

namespace {

// The map of `desc` alone (jac tapes or table, D, quadrature) on a scratch context, for the
// entry points that evaluate kernel (1) at caller-given points.  extra: tapes packed after the
// map's (returned as TapeRefs into tmp.t_*).
void load_map(const ts_problem_desc* desc, ts_ctx& tmp, const std::vector<const ts_tape*>& extra = {},
              std::vector<TapeRef>* extra_refs = nullptr) {
    if (int rc = device_ready()) throw CudaError{rc};
    CU(cudaStreamCreateWithFlags(&tmp.stream, cudaStreamNonBlocking));
    ProblemG& P = tmp.P;
    P.macro = to_grid(desc->macro);
    P.micro = to_grid(desc->micro);
    TapePack pack;
    for (int k = 0; k < 4; ++k) {
        if (!check_tape(desc->jac[k])) throw std::invalid_argument("malformed tape");
        P.map.jac[k] = pack.add(desc->jac[k]);
    }
    for (const ts_tape* t : extra) {
        if (!check_tape(*t)) throw std::invalid_argument("malformed tape");
        const TapeRef r = pack.add(*t);
        if (extra_refs) extra_refs->push_back(r);
    }
    const size_t ni = pack.op.size() ? pack.op.size() : 1;
    pack.op.resize(ni, 0);
    pack.arg.resize(ni, 0);
    pack.val.resize(ni, 0.0);
    tmp.t_op.alloc(ni);
    tmp.t_arg.alloc(ni);
    tmp.t_val.alloc(ni);
    CU(cudaMemcpy(tmp.t_op.p, pack.op.data(), ni * sizeof(int), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(tmp.t_arg.p, pack.arg.data(), ni * sizeof(int), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(tmp.t_val.p, pack.val.data(), ni * sizeof(double), cudaMemcpyHostToDevice));
    P.map.kind = desc->map_kind;
    P.map.op = tmp.t_op.p;
    P.map.arg = tmp.t_arg.p;
    P.map.val = tmp.t_val.p;
    P.map.s_kind = desc->s_kind;
    P.map.amp = desc->amp;
    P.map.macro = P.macro;
    for (int k = 0; k < 4; ++k) P.map.D[k] = desc->D[k];
    P.map.D_identity = desc->D[0] == 1.0 && desc->D[1] == 0.0 && desc->D[2] == 0.0 && desc->D[3] == 1.0;
    if (desc->map_kind == TS_MAP_AFFINE_BUBBLE_TABLE) {
        const size_t nn = (size_t)4 * P.macro.nodes();
        tmp.A_table.alloc(nn);
        CU(cudaMemcpy(tmp.A_table.p, desc->A_table, nn * sizeof(double), cudaMemcpyHostToDevice));
        P.map.A_table = tmp.A_table.p;
    }
    tmp.Q = make_quad();
    upload_quad_tables(tmp.Q);
    tmp.nfaces = P.micro.faces();
    tmp.first_bad.alloc(1);
    tmp.err.alloc(1);
    reset_flags(&tmp);
}

int expr_status(ts_ctx& tmp) {
    unsigned e = 0;
    CU(cudaMemcpy(&e, tmp.err.p, sizeof e, cudaMemcpyDeviceToHost));
    return e ? fail(TS_ERR_EXPR, "%s", expr_error(e)) : TS_OK;
}

}  // namespace

extern "C" {

int32_t ts_build_cache(const ts_problem_desc* desc, int32_t n_points, const double* points, double* cells,
                       double* faces) {
    if (!desc || !points || n_points < 0) return fail(TS_ERR_INVALID, "null argument");
    ts_ctx tmp;
    return guarded([&]() -> int {
        load_map(desc, tmp);
        const ProblemG& P = tmp.P;
        DBuf<double> pts;
        pts.alloc((size_t)2 * n_points + 1);
        CU(cudaMemcpy(pts.p, points, (size_t)2 * n_points * sizeof(double), cudaMemcpyHostToDevice));
        DBuf<double4> dc, df;
        if (cells) {
            dc.alloc((size_t)n_points * P.micro.cells() * 4);
            launch_cell_cache(P, n_points, pts.p, dc.p, tmp.first_bad.p, tmp.err.p, tmp.stream);
        }
        df.alloc((size_t)n_points * P.micro.faces() * 2);
        launch_face_cache(P, n_points, pts.p, cells != nullptr, df.p, tmp.first_bad.p, tmp.err.p, tmp.stream);
        CU(cudaGetLastError());
        if (int rc = check_degenerate(&tmp, pts.p, cells != nullptr, "degenerate map in cache build")) return rc;
        if (cells) CU(cudaMemcpy(cells, dc.p, dc.bytes(), cudaMemcpyDeviceToHost));
        if (faces) CU(cudaMemcpy(faces, df.p, df.bytes(), cudaMemcpyDeviceToHost));
        return TS_OK;
    });
}

int32_t ts_validate_diffeo(const ts_problem_desc* desc, int32_t nx, const double* xs, int32_t ny, const double* ys,
                           double* out) {
    if (!desc || !out || nx < 0 || ny < 0 || (nx && !xs) || (ny && !ys)) return fail(TS_ERR_INVALID, "null argument");
    if (desc->map_kind != TS_MAP_TAPE) return fail(TS_ERR_INVALID, "validate_diffeo takes a symbolic (tape) map");
    out[0] = out[1] = 0.0;
    out[2] = -1.0;
    if ((long long)nx * ny == 0) return TS_OK;
    ts_ctx tmp;
    return guarded([&]() -> int {
        load_map(desc, tmp);
        DBuf<double> dx, dy, part;
        dx.alloc((size_t)2 * nx);
        dy.alloc((size_t)2 * ny);
        part.alloc((size_t)3 * 148 * 8);
        CU(cudaMemcpy(dx.p, xs, dx.bytes(), cudaMemcpyHostToDevice));
        CU(cudaMemcpy(dy.p, ys, dy.bytes(), cudaMemcpyHostToDevice));
        const int blocks = launch_validate_pairs(tmp.P.map, dx.p, nx, dy.p, ny, part.p, tmp.err.p, tmp.stream);
        CU(cudaGetLastError());
        std::vector<double> h((size_t)3 * blocks);
        CU(cudaMemcpyAsync(h.data(), part.p, h.size() * sizeof(double), cudaMemcpyDeviceToHost, tmp.stream));
        tmp.sync();
        if (int rc = expr_status(tmp)) return rc;
        double mn = 0.0, mx = 0.0, at = -1.0;
        for (int b = 0; b < blocks; ++b) {  // (min, index) lexicographic: the first strict minimum
            if (h[3 * b + 1] < 0) continue;
            if (at < 0 || h[3 * b] < mn || (h[3 * b] == mn && h[3 * b + 1] < at)) {
                mn = h[3 * b];
                at = h[3 * b + 1];
            }
            mx = at < 0 ? h[3 * b + 2] : std::max(mx, h[3 * b + 2]);
        }
        out[0] = mn;
        out[1] = mx;
        out[2] = at;
        return TS_OK;
    });
}

int32_t ts_assumption6(const ts_problem_desc* desc, int32_t n_points, const double* points, const double* nu_len,
                       double* gamma, double* dw) {
    if (!desc || n_points < 0 || (n_points && (!points || !gamma))) return fail(TS_ERR_INVALID, "null argument");
    if (n_points == 0) return TS_OK;
    ts_ctx tmp;
    return guarded([&]() -> int {
        std::vector<TapeRef> refs;
        load_map(desc, tmp, {&desc->Dw}, &refs);
        const ProblemG& P = tmp.P;
        const int faces = P.micro.faces();
        DBuf<double> pts, nu, g, d;
        pts.alloc((size_t)2 * n_points);
        CU(cudaMemcpy(pts.p, points, pts.bytes(), cudaMemcpyHostToDevice));
        g.alloc((size_t)2 * n_points);
        DBuf<double4> df;
        if (nu_len) {  // a MapCache's |nu| entries
            nu.alloc((size_t)n_points * faces * 2);
            CU(cudaMemcpy(nu.p, nu_len, nu.bytes(), cudaMemcpyHostToDevice));
            launch_boundary_measures(P.micro, desc->micro_role, n_points, nu.p, 1, 0, g.p, tmp.stream);
        } else {  // kernel (1) at the points
            df.alloc((size_t)n_points * faces * 2);
            launch_face_cache(P, n_points, pts.p, 0, df.p, tmp.first_bad.p, tmp.err.p, tmp.stream);
            if (int rc = check_degenerate(&tmp, pts.p, false, "degenerate map in cache build")) return rc;
            launch_boundary_measures(P.micro, desc->micro_role, n_points, reinterpret_cast<const double*>(df.p), 4,
                                     3, g.p, tmp.stream);
        }
        if (dw) {
            d.alloc(n_points);
            launch_tape_at_points(tmp.t_op.p, tmp.t_arg.p, tmp.t_val.p, refs[0], n_points, pts.p, d.p, tmp.err.p,
                                  tmp.stream);
        }
        CU(cudaGetLastError());
        tmp.sync();
        if (int rc = expr_status(tmp)) return rc;
        CU(cudaMemcpy(gamma, g.p, g.bytes(), cudaMemcpyDeviceToHost));
        if (dw) CU(cudaMemcpy(dw, d.p, d.bytes(), cudaMemcpyDeviceToHost));
        return TS_OK;
    });
}

}  // extern "C"
