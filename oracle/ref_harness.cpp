// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" harness over the UNMODIFIED reference library (the twelve
// /root/reference/proj/src/*.cpp files compiled by oracle/Makefile into
// oracle/_ref/libtwoscale_ref.so).  Every function below calls only the
// reference's public C++ API (proj/include/twoscale/*.hpp); nothing of the
// reference's algorithm is restated here.  Used by tests/ as the parity oracle
// and by bench.py's cpu_baseline / --impl reference legs.
//
// Error protocol: 0 = ok, 1 = ConfigError, 2 = ParseError/EvalError,
// 3 = DegenerateMapError, 4 = SolverError, 9 = anything else; the message is
// available from ref_last_error().

#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "twoscale/assembly.hpp"
#include "twoscale/config.hpp"
#include "twoscale/linalg.hpp"
#include "twoscale/mapping.hpp"
#include "twoscale/mms.hpp"
#include "twoscale/parallel.hpp"
#include "twoscale/solver.hpp"
#include "twoscale/vtk.hpp"

using namespace twoscale;

namespace {

thread_local std::string g_err;

struct RefCtx {
    Config cfg;
    std::unique_ptr<ProblemSetup> setup;        // grids must outlive ctx (assembly.hpp:73-75)
    std::unique_ptr<AssemblyContext> ctx;
    double build_seconds = 0.0;
};

template <class F>
int guarded(F&& f) {
    try {
        f();
        return 0;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 1;
    } catch (const ParseError& e) {
        g_err = e.what();
        return 2;
    } catch (const EvalError& e) {
        g_err = e.what();
        return 2;
    } catch (const DegenerateMapError& e) {
        g_err = e.what();
        return 3;
    } catch (const SolverError& e) {
        g_err = e.what();
        return 4;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

// parse_config -> make_problem -> AssemblyContext (config.cpp:126, problem.cpp:30,
// assembly.cpp:52).  workers as in AssemblyContext(..., workers).
int ref_create(const char* ini, int workers, void** out) {
    *out = nullptr;
    return guarded([&] {
        auto rc = std::make_unique<RefCtx>();
        rc->cfg = parse_config(ini);
        rc->setup = std::make_unique<ProblemSetup>(make_problem(rc->cfg));
        auto t0 = std::chrono::steady_clock::now();
        rc->ctx = std::make_unique<AssemblyContext>(rc->setup->data, rc->setup->macro,
                                                    rc->setup->micro, workers);
        rc->build_seconds =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *out = rc.release();
    });
}

// Same for the manufactured problem of an INI with [mms]: derive_data (mms.cpp:30-83).
int ref_create_mms(const char* ini, int workers, void** out) {
    *out = nullptr;
    return guarded([&] {
        auto rc = std::make_unique<RefCtx>();
        rc->cfg = parse_config(ini);
        rc->setup = std::make_unique<ProblemSetup>(make_problem(rc->cfg));
        rc->setup->data = derive_data(rc->setup->mms);
        rc->ctx = std::make_unique<AssemblyContext>(rc->setup->data, rc->setup->macro, rc->setup->micro, workers);
        *out = rc.release();
    });
}

void ref_destroy(void* h) { delete static_cast<RefCtx*>(h); }

double ref_build_seconds(void* h) { return static_cast<RefCtx*>(h)->build_seconds; }

// sizes[0..7] = n_macro, n_micro, micro_nnz, macro_nnz, n_micro_faces, shared_matrix,
//               n_macro_cells, n_micro_cells
int ref_sizes(void* h, int* sizes) {
    auto* rc = static_cast<RefCtx*>(h);
    return guarded([&] {
        const AssemblyContext& c = *rc->ctx;
        sizes[0] = c.macro_grid().node_count();
        sizes[1] = c.micro_grid().node_count();
        sizes[2] = static_cast<int>(c.micro_matrix(0).col_idx().size());
        sizes[3] = static_cast<int>(c.macro_u_matrix().col_idx().size());
        sizes[4] = static_cast<int>(c.micro_grid().boundary_faces().size());
        sizes[5] = (&c.micro_matrix(0) == &c.micro_matrix(sizes[0] > 1 ? 1 : 0)) ? 1 : 0;
        sizes[6] = c.macro_grid().cell_count();
        sizes[7] = c.micro_grid().cell_count();
    });
}

int ref_micro_pattern(void* h, int* row_ptr, int* col_idx) {
    auto* rc = static_cast<RefCtx*>(h);
    return guarded([&] {
        const CsrMatrix& A = rc->ctx->micro_matrix(0);
        std::memcpy(row_ptr, A.row_ptr().data(), A.row_ptr().size() * sizeof(int));
        std::memcpy(col_idx, A.col_idx().data(), A.col_idx().size() * sizeof(int));
    });
}

int ref_micro_values(void* h, int node, double* vals) {
    auto* rc = static_cast<RefCtx*>(h);
    return guarded([&] {
        const CsrMatrix& A = rc->ctx->micro_matrix(node);
        std::memcpy(vals, A.values().data(), A.values().size() * sizeof(double));
    });
}

int ref_micro_rhs(void* h, int node, double u, double w, double* out) {
    auto* rc = static_cast<RefCtx*>(h);
    return guarded([&] {
        std::vector<double> b;
        rc->ctx->micro_rhs(node, u, w, b);
        std::memcpy(out, b.data(), b.size() * sizeof(double));
    });
}

// cells: [cell][q][J, A00, A01, A11]; faces: [face][q][J, nu.x, nu.y, nu_len]
int ref_node_cache(void* h, int node, double* cells, double* faces) {
    auto* rc = static_cast<RefCtx*>(h);
    return guarded([&] {
        const AssemblyContext& c = *rc->ctx;
        const MapCache& m = c.node_cache();
        const int nq = c.rule().n_cell(), nqf = c.rule().n_face();
        if (cells) {
            for (int cell = 0; cell < c.micro_grid().cell_count(); ++cell)
                for (int q = 0; q < nq; ++q) {
                    const auto& e = m.cell(node, cell, q);
                    double* o = cells + (std::size_t(cell) * nq + q) * 4;
                    o[0] = e.J;
                    o[1] = e.A00;
                    o[2] = e.A01;
                    o[3] = e.A11;
                }
        }
        if (faces) {
            const int nf = static_cast<int>(c.micro_grid().boundary_faces().size());
            for (int f = 0; f < nf; ++f)
                for (int q = 0; q < nqf; ++q) {
                    const auto& e = m.face(node, f, q);
                    double* o = faces + (std::size_t(f) * nqf + q) * 4;
                    o[0] = e.J;
                    o[1] = e.nu.x;
                    o[2] = e.nu.y;
                    o[3] = e.nu_len;
                }
        }
    });
}

// CompiledDiffeo::jac (mapping.cpp:44-47) at arbitrary points; out = 4 per point.
int ref_jac(void* h, int npts, const double* x, const double* y, double* out) {
    auto* rc = static_cast<RefCtx*>(h);
    return guarded([&] {
        for (int p = 0; p < npts; ++p) {
            const Mat2 F = rc->ctx->diffeo().jac({x[2 * p], x[2 * p + 1]}, {y[2 * p], y[2 * p + 1]});
            out[4 * p + 0] = F.a00;
            out[4 * p + 1] = F.a01;
            out[4 * p + 2] = F.a10;
            out[4 * p + 3] = F.a11;
        }
    });
}

// build_cache (mapping.cpp:79-129) of the context's map at arbitrary macro points, on the
// context's micro grid and rule.  rows_out = cache rows (1 when the Jacobian has no x).
// cells [row][cell][q][J, A00, A01, A11] (may be NULL: with_cells = false),
// faces [row][face][q][J, nu.x, nu.y, nu_len].
int ref_build_cache(void* h, int npts, const double* pts, double* cells, double* faces, int* rows_out) {
    auto* rc = static_cast<RefCtx*>(h);
    return guarded([&] {
        const AssemblyContext& c = *rc->ctx;
        std::vector<Vec2> xs(npts);
        for (int p = 0; p < npts; ++p) xs[p] = {pts[2 * p], pts[2 * p + 1]};
        const MapCache m = build_cache(c.diffeo(), xs, c.micro_grid(), c.rule(), 1, cells != nullptr);
        const int rows = c.diffeo().jacobian_depends_on_x() ? npts : std::min(1, npts);
        *rows_out = rows;
        const int nq = c.rule().n_cell(), nqf = c.rule().n_face();
        const int nc = c.micro_grid().cell_count(), nf = static_cast<int>(c.micro_grid().boundary_faces().size());
        for (int r = 0; r < rows; ++r) {
            if (cells)
                for (int cell = 0; cell < nc; ++cell)
                    for (int q = 0; q < nq; ++q) {
                        const auto& e = m.cell(r, cell, q);
                        double* o = cells + ((std::size_t(r) * nc + cell) * nq + q) * 4;
                        o[0] = e.J;
                        o[1] = e.A00;
                        o[2] = e.A01;
                        o[3] = e.A11;
                    }
            for (int f = 0; f < nf; ++f)
                for (int q = 0; q < nqf; ++q) {
                    const auto& e = m.face(r, f, q);
                    double* o = faces + ((std::size_t(r) * nf + f) * nqf + q) * 4;
                    o[0] = e.J;
                    o[1] = e.nu.x;
                    o[2] = e.nu.y;
                    o[3] = e.nu_len;
                }
        }
    });
}

// validate_diffeo (mapping.cpp:131-156) of the context's map over xs x ys.
// out = pass, min_det, max_det, worst x (2), worst yhat (2); msg receives the message.
int ref_validate_diffeo(void* h, int nx, const double* xs, int ny, const double* ys, double lo, double hi,
                        double* out, char* msg, int msg_cap) {
    auto* rc = static_cast<RefCtx*>(h);
    return guarded([&] {
        std::vector<Vec2> X(nx), Y(ny);
        for (int p = 0; p < nx; ++p) X[p] = {xs[2 * p], xs[2 * p + 1]};
        for (int p = 0; p < ny; ++p) Y[p] = {ys[2 * p], ys[2 * p + 1]};
        MapBounds b;
        b.lo = lo;
        b.hi = hi;
        const DiffeoValidation v = validate_diffeo(rc->ctx->diffeo(), b, X, Y);
        out[0] = v.pass ? 1.0 : 0.0;
        out[1] = v.min_det;
        out[2] = v.max_det;
        out[3] = v.worst_x.x;
        out[4] = v.worst_x.y;
        out[5] = v.worst_yhat.x;
        out[6] = v.worst_yhat.y;
        std::snprintf(msg, msg_cap, "%s", v.message.c_str());
    });
}

// check_assumption6 (mapping.cpp:158-195) at arbitrary macro points: the cache is
// build_cache(points, faces only) of the context's map, D^w is the INI's dw, the roles and
// kappas are the context's.  rows [n][4] = gamma_in, gamma_out, ok1, ok2;
// summary = min_dw, lhs1_max, lhs2_max, ok1, ok2.
int ref_check_assumption6(void* h, int npts, const double* pts, double* rows, double* summary) {
    auto* rc = static_cast<RefCtx*>(h);
    return guarded([&] {
        const AssemblyContext& c = *rc->ctx;
        const ProblemData& d = c.data();
        std::vector<Vec2> xs(npts);
        for (int p = 0; p < npts; ++p) xs[p] = {pts[2 * p], pts[2 * p + 1]};
        const MapCache m = build_cache(c.diffeo(), xs, c.micro_grid(), c.rule(), 1, false);
        const CompiledExpr dw(d.Dw, d.params);
        const Assumption6Report r = check_assumption6(d.kappa1, d.kappa2, d.kappa3, d.kappa4, dw, m,
                                                      c.micro_grid(), c.rule(), d.roles, xs);
        for (int p = 0; p < npts; ++p) {
            rows[4 * p + 0] = r.rows[p].gamma_in;
            rows[4 * p + 1] = r.rows[p].gamma_out;
            rows[4 * p + 2] = r.rows[p].ok1 ? 1.0 : 0.0;
            rows[4 * p + 3] = r.rows[p].ok2 ? 1.0 : 0.0;
        }
        summary[0] = r.min_dw;
        summary[1] = r.lhs1_max;
        summary[2] = r.lhs2_max;
        summary[3] = r.ok1 ? 1.0 : 0.0;
        summary[4] = r.ok2 ? 1.0 : 0.0;
    });
}

// which: 0 = A_u, 1 = A_w, 2 = M0 (values in the shared macro Q1 pattern)
int ref_macro_matrix(void* h, int which, int* row_ptr, int* col_idx, double* vals) {
    auto* rc = static_cast<RefCtx*>(h);
    return guarded([&] {
        const AssemblyContext& c = *rc->ctx;
        const CsrMatrix& A =
            which == 0 ? c.macro_u_matrix() : which == 1 ? c.macro_w_matrix() : c.macro_mass();
        if (row_ptr) std::memcpy(row_ptr, A.row_ptr().data(), A.row_ptr().size() * sizeof(int));
        if (col_idx) std::memcpy(col_idx, A.col_idx().data(), A.col_idx().size() * sizeof(int));
        if (vals) std::memcpy(vals, A.values().data(), A.values().size() * sizeof(double));
    });
}

// macro_u_rhs / macro_w_rhs (assembly.cpp:402-422) for a row-major V[n_macro][n_micro].
int ref_macro_rhs(void* h, int which, const double* V, double* out) {
    auto* rc = static_cast<RefCtx*>(h);
    return guarded([&] {
        const AssemblyContext& c = *rc->ctx;
        const int nM = c.macro_grid().node_count(), nm = c.micro_grid().node_count();
        MicroField F(nM, std::vector<double>(nm, 0.0));
        if (V)
            for (int i = 0; i < nM; ++i)
                std::memcpy(F[i].data(), V + std::size_t(i) * nm, nm * sizeof(double));
        const std::vector<double> b = which == 0 ? c.macro_u_rhs(F) : c.macro_w_rhs(F);
        std::memcpy(out, b.data(), b.size() * sizeof(double));
    });
}

// which: 0 = u, 1 = w.  Returns count in *n; dofs/vals may be null to query.
int ref_dirichlet(void* h, int which, int* n, int* dofs, double* vals) {
    auto* rc = static_cast<RefCtx*>(h);
    return guarded([&] {
        const auto& d = which == 0 ? rc->ctx->dirichlet_u() : rc->ctx->dirichlet_w();
        *n = static_cast<int>(d.size());
        for (std::size_t k = 0; k < d.size(); ++k) {
            if (dofs) dofs[k] = d[k].first;
            if (vals) vals[k] = d[k].second;
        }
    });
}

// role: 0 = GammaI, 1 = GammaO, 2 = GammaN (assembly.cpp:377-393)
int ref_surface_coupling(void* h, const double* v, int node, int role, double* out) {
    auto* rc = static_cast<RefCtx*>(h);
    return guarded([&] {
        const int nm = rc->ctx->micro_grid().node_count();
        std::vector<double> vv(v, v + nm);
        *out = rc->ctx->surface_coupling(vv, node, static_cast<MicroRole>(role));
    });
}

// fixed_point_solve(ctx, opts) (solver.cpp:61-132).  V is row-major [n_macro][n_micro].
// info[0..3] = sweeps, converged, w_pinned, n_hist; info_d[0..1] = final_residual, seconds
int ref_solve(void* h, double inner_tol, int inner_maxit, double outer_tol, int max_outer,
              int workers, double* u, double* w, double* V, double* hist, int hist_cap, int* info,
              double* info_d) {
    auto* rc = static_cast<RefCtx*>(h);
    return guarded([&] {
        SolveOptions o;
        o.inner_tol = inner_tol;
        o.inner_maxit = inner_maxit;
        o.outer_tol = outer_tol;
        o.max_outer = max_outer;
        o.workers = workers;
        auto t0 = std::chrono::steady_clock::now();
        SolveResult r = fixed_point_solve(*rc->ctx, o);
        const double secs =
            std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        const int nM = static_cast<int>(r.state.u.size());
        if (u) std::memcpy(u, r.state.u.data(), nM * sizeof(double));
        if (w) std::memcpy(w, r.state.w.data(), nM * sizeof(double));
        if (V)
            for (int i = 0; i < nM; ++i)
                std::memcpy(V + std::size_t(i) * r.state.V[i].size(), r.state.V[i].data(),
                            r.state.V[i].size() * sizeof(double));
        const int nh = static_cast<int>(r.state.residual_history.size());
        for (int k = 0; k < nh && k < hist_cap; ++k) hist[k] = r.state.residual_history[k];
        info[0] = r.report.sweeps;
        info[1] = r.report.converged ? 1 : 0;
        info[2] = r.report.w_pinned ? 1 : 0;
        info[3] = nh;
        info_d[0] = r.report.final_residual;
        info_d[1] = secs;
    });
}

// cg_solve (linalg.cpp:103-161) on a caller-provided CSR matrix.
// res[0..3] = converged, iterations, indefinite; resd[0] = residual
int ref_cg_solve(int n, const int* row_ptr, const int* col_idx, const double* vals,
                 const double* b, double* x, double tol, int maxit, int* res, double* resd) {
    return guarded([&] {
        std::vector<std::vector<int>> pattern(n);
        for (int r = 0; r < n; ++r) pattern[r].assign(col_idx + row_ptr[r], col_idx + row_ptr[r + 1]);
        CsrMatrix A(n, pattern);
        std::memcpy(A.values().data(), vals, sizeof(double) * row_ptr[n]);
        std::vector<double> bb(b, b + n), xx(x, x + n);
        const CgResult r = cg_solve(A, bb, xx, tol, maxit);
        std::memcpy(x, xx.data(), n * sizeof(double));
        res[0] = r.converged ? 1 : 0;
        res[1] = r.iterations;
        res[2] = r.indefinite ? 1 : 0;
        resd[0] = r.residual;
    });
}

// Many systems on one shared pattern, one reference cg_solve per system, spread over
// `workers` threads with the reference's own parallel_for (solver.cpp:85-98 pattern).
// vals: [n_sys][nnz]; b, x: [n_sys][n]; iters: [n_sys].  *seconds = wall time of the
// solve loop only (pattern/matrix construction excluded).
int ref_batched_cg(int n, const int* row_ptr, const int* col_idx, int n_sys, const double* vals,
                   const double* b, double* x, double tol, int maxit, int workers, int* iters,
                   double* seconds) {
    return guarded([&] {
        std::vector<std::vector<int>> pattern(n);
        for (int r = 0; r < n; ++r) pattern[r].assign(col_idx + row_ptr[r], col_idx + row_ptr[r + 1]);
        const CsrMatrix proto(n, pattern);
        const int nnz = row_ptr[n];
        std::vector<CsrMatrix> As(n_sys, proto);
        for (int s = 0; s < n_sys; ++s)
            std::memcpy(As[s].values().data(), vals + std::size_t(s) * nnz, sizeof(double) * nnz);
        std::vector<std::vector<double>> B(n_sys), X(n_sys);
        for (int s = 0; s < n_sys; ++s) {
            B[s].assign(b + std::size_t(s) * n, b + std::size_t(s + 1) * n);
            X[s].assign(x + std::size_t(s) * n, x + std::size_t(s + 1) * n);
        }
        auto t0 = std::chrono::steady_clock::now();
        parallel_for(workers, n_sys, [&](std::int64_t s) {
            const CgResult r = cg_solve(As[s], B[s], X[s], tol, maxit);
            iters[s] = r.converged ? r.iterations : -1;
        });
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        for (int s = 0; s < n_sys; ++s)
            std::memcpy(x + std::size_t(s) * n, X[s].data(), n * sizeof(double));
    });
}

// Instrumented replica of the micro loop of fixed_point_solve (solver.cpp:85-98):
// micro_rhs + cg_solve per macro node, with fixed u, w.  V in/out (warm start),
// iters per node; *seconds = wall time.  nodes==nullptr means all nodes.
int ref_micro_sweep(void* h, const double* u, const double* w, double tol, int maxit,
                    int workers, int n_nodes, const int* nodes, double* V, int* iters,
                    double* seconds) {
    auto* rc = static_cast<RefCtx*>(h);
    return guarded([&] {
        const AssemblyContext& c = *rc->ctx;
        const int nm = c.micro_grid().node_count();
        auto t0 = std::chrono::steady_clock::now();
        parallel_for(workers, n_nodes, [&](std::int64_t k) {
            const int i = nodes ? nodes[k] : static_cast<int>(k);
            std::vector<double> b;
            c.micro_rhs(i, u[i], w[i], b);
            std::vector<double> x(V + std::size_t(k) * nm, V + std::size_t(k + 1) * nm);
            const CgResult r = cg_solve(c.micro_matrix(i), b, x, tol, maxit);
            std::memcpy(V + std::size_t(k) * nm, x.data(), nm * sizeof(double));
            iters[k] = r.converged ? r.iterations : -1;
        });
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    });
}

int ref_hardware_threads() { return resolve_worker_count(0); }

// derive_data + convergence_sweep (mms.cpp:30-83, 384-418) from an INI with [mms];
// rows [n_ns][13] as ts_mms_sweep_ini.
int ref_mms_sweep(const char* ini, const int* ns, int n_ns, double* rows, int workers) {
    return guarded([&] {
        const Config cfg = parse_config(ini);
        const ProblemSetup setup = make_problem(cfg);
        SolveOptions o;
        o.workers = workers;
        o.inner_tol = cfg.inner_tol;
        o.inner_maxit = cfg.inner_maxit;
        o.outer_tol = cfg.outer_tol;
        o.max_outer = cfg.max_outer;
        const ErrorReport rep = convergence_sweep(setup.mms, std::vector<int>(ns, ns + n_ns), o);
        for (std::size_t k = 0; k < rep.size(); ++k) {
            const ErrorReportRow& r = rep[k];
            const double v[13] = {double(r.n), double(r.macro_dofs), double(r.micro_dofs), r.H, r.h, r.e_uw,
                                  r.e_uw_grad, r.e_v, r.e_v_grad, r.p_macro, r.q_macro, r.p_micro, r.q_micro};
            std::memcpy(rows + 13 * k, v, sizeof v);
        }
    });
}

// error_norms (mms.cpp:247-377) for a given state on the INI's grids.
int ref_error_norms(const char* ini, const double* u, const double* w, const double* V, double* out, int workers) {
    return guarded([&] {
        const Config cfg = parse_config(ini);
        const ProblemSetup setup = make_problem(cfg);
        const int nM = setup.macro.node_count(), nm = setup.micro.node_count();
        TwoScaleState st;
        st.u.assign(u, u + nM);
        st.w.assign(w, w + nM);
        st.V.resize(nM);
        for (int i = 0; i < nM; ++i) st.V[i].assign(V + std::size_t(i) * nm, V + std::size_t(i + 1) * nm);
        const ErrorNorms e = error_norms(st, setup.mms, setup.macro, setup.micro, workers);
        out[0] = e.e_uw;
        out[1] = e.e_uw_grad;
        out[2] = e.e_v;
        out[3] = e.e_v_grad;
    });
}

// derive_data (mms.cpp:30-83) then AssemblyContext + fixed_point_solve on the INI's grids:
// the MMS problem as a plain solve (exercises every data term of the path).
int ref_mms_solve(const char* ini, double* u, double* w, double* V, int* sweeps) {
    return guarded([&] {
        const Config cfg = parse_config(ini);
        const ProblemSetup setup = make_problem(cfg);
        const ProblemData derived = derive_data(setup.mms);
        SolveOptions o;
        o.inner_tol = cfg.inner_tol;
        o.inner_maxit = cfg.inner_maxit;
        o.outer_tol = cfg.outer_tol;
        o.max_outer = cfg.max_outer;
        const SolveResult r = fixed_point_solve(derived, setup.macro, setup.micro, o);
        const int nM = static_cast<int>(r.state.u.size());
        std::memcpy(u, r.state.u.data(), nM * sizeof(double));
        std::memcpy(w, r.state.w.data(), nM * sizeof(double));
        for (int i = 0; i < nM; ++i)
            std::memcpy(V + std::size_t(i) * r.state.V[i].size(), r.state.V[i].data(), r.state.V[i].size() * sizeof(double));
        *sweeps = r.report.sweeps;
    });
}

// write_vtk_macro + write_vtk_micro (vtk.cpp:36-85) for a given host state on the
// INI's grids and map, as tools/twoscale.cpp:139-143 calls them.  Either path may be null.
int ref_write_vtk(const char* ini, const double* u, const double* w, const double* V, double scale,
                  const char* macro_path, const char* micro_path) {
    return guarded([&] {
        const Config cfg = parse_config(ini);
        const ProblemSetup setup = make_problem(cfg);
        const int nM = setup.macro.node_count(), nm = setup.micro.node_count();
        if (macro_path) {
            const std::vector<double> uu(u, u + nM), ww(w, w + nM);
            write_vtk_macro(setup.macro, {{"u", &uu}, {"w", &ww}}, macro_path);
        }
        if (micro_path) {
            MicroField F(nM);
            for (int i = 0; i < nM; ++i) F[i].assign(V + std::size_t(i) * nm, V + std::size_t(i + 1) * nm);
            const CompiledDiffeo map(setup.data.diffeo, setup.data.params);
            write_vtk_micro(F, setup.macro, setup.micro, map, scale, micro_path);
        }
    });
}

}  // extern "C"
