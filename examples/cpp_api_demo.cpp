// Drop-in check of the host C++ mirror: the same calls the reference's CLI makes
// (tools/twoscale.cpp:115-143 cmd_solve) against include/twoscale/*.hpp, linked to
// libtwoscale_b200.so.  Usage: cpp_api_demo <config.ini> <out.bin> [vtk_dir]
// Writes u, w, V (row-major) as raw float64 and prints a one-line JSON summary; with
// vtk_dir also macro.vtk / micro.vtk exactly as cmd_solve does (tools/twoscale.cpp:139-143).
#include <cstdio>
#include <fstream>

#include "twoscale/config.hpp"
#include "twoscale/solver.hpp"
#include "twoscale/vtk.hpp"

int main(int argc, char** argv) {
    if (argc < 3) {
        std::fprintf(stderr, "usage: %s config.ini out.bin\n", argv[0]);
        return 2;
    }
    try {
        const twoscale::Config cfg = twoscale::load_config(argv[1]);
        twoscale::ProblemSetup setup = twoscale::make_problem(cfg);
        twoscale::SolveOptions opts;
        opts.inner_tol = cfg.inner_tol;
        opts.inner_maxit = cfg.inner_maxit;
        opts.outer_tol = cfg.outer_tol;
        opts.max_outer = cfg.max_outer;
        twoscale::AssemblyContext ctx(setup.data, setup.macro, setup.micro, 1);
        const twoscale::SolveResult r = twoscale::fixed_point_solve(ctx, opts);
        // API spot checks a caller of the reference relies on
        const twoscale::CsrMatrix& A0 = ctx.micro_matrix(0);
        std::vector<double> b;
        ctx.micro_rhs(setup.macro.node_count() / 2, 1.0, 0.0, b);
        std::vector<double> x(A0.size(), 0.0);
        const twoscale::CgResult cg = twoscale::cg_solve(ctx.micro_matrix(setup.macro.node_count() / 2), b, x,
                                                          opts.inner_tol, opts.inner_maxit);
        if (argc > 3) {  // cmd_solve's VTK output (tools/twoscale.cpp:139-143)
            const std::string dir = argv[3];
            twoscale::write_vtk_macro(setup.macro, {{"u", &r.state.u}, {"w", &r.state.w}}, dir + "/macro.vtk");
            const twoscale::CompiledDiffeo map(setup.data.diffeo, setup.data.params);
            twoscale::write_vtk_micro(r.state.V, setup.macro, setup.micro, map, cfg.micro_viz_scale,
                                      dir + "/micro.vtk");
        }
        std::ofstream out(argv[2], std::ios::binary);
        out.write(reinterpret_cast<const char*>(r.state.u.data()), r.state.u.size() * sizeof(double));
        out.write(reinterpret_cast<const char*>(r.state.w.data()), r.state.w.size() * sizeof(double));
        for (const auto& row : r.state.V) out.write(reinterpret_cast<const char*>(row.data()), row.size() * sizeof(double));
        std::printf("{\"sweeps\": %d, \"converged\": %d, \"final_residual\": %.17g, \"micro_nnz\": %zu, "
                    "\"cg_converged\": %d, \"cg_iterations\": %d, \"dirichlet_u\": %zu, \"w_pinned\": %d}\n",
                    r.report.sweeps, r.report.converged ? 1 : 0, r.report.final_residual, A0.values().size(),
                    cg.converged ? 1 : 0, cg.iterations, ctx.dirichlet_u().size(), ctx.w_pinned() ? 1 : 0);
        return r.report.converged ? 0 : 1;
    } catch (const twoscale::SolverError& e) {
        std::fprintf(stderr, "solver error: %s\n", e.what());
        return 4;
    } catch (const twoscale::DegenerateMapError& e) {
        std::fprintf(stderr, "degenerate map: %s\n", e.what());
        return 3;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    }
}
