// fixed_point_solve on the device (see include/twoscale/solver.hpp).
#include "twoscale/solver.hpp"

#include <cstring>

namespace twoscale {

SolveResult fixed_point_solve(const AssemblyContext& ctx, const SolveOptions& opts) {
    const int nM = ctx.macro_grid().node_count(), nm = ctx.micro_grid().node_count();
    ts_solve_opts o{opts.inner_tol, opts.inner_maxit, opts.outer_tol, opts.max_outer};
    ts_solve_report rep{};
    std::vector<double> hist(std::max(opts.max_outer, 1));
    throw_status(ts_fixed_point_solve(ctx.handle(), &o, &rep, hist.data(), static_cast<int>(hist.size())));
    SolveResult r;
    r.state.u.resize(nM);
    r.state.w.resize(nM);
    std::vector<double> V(static_cast<std::size_t>(nM) * nm);
    throw_status(ts_download_state(ctx.handle(), r.state.u.data(), r.state.w.data(), V.data()));
    r.state.V.assign(nM, std::vector<double>(nm));
    for (int i = 0; i < nM; ++i) std::memcpy(r.state.V[i].data(), V.data() + static_cast<std::size_t>(i) * nm, nm * sizeof(double));
    hist.resize(std::min(rep.sweeps, static_cast<int>(hist.size())));
    r.state.residual_history = hist;
    r.report.converged = rep.converged != 0;
    r.report.sweeps = rep.sweeps;
    r.report.w_pinned = rep.w_pinned != 0;
    r.report.final_residual = rep.final_residual;
    return r;
}

SolveResult fixed_point_solve(const ProblemData& data, const Grid& macro, const Grid& micro, const SolveOptions& opts) {
    AssemblyContext ctx(data, macro, micro, opts.workers);
    return fixed_point_solve(ctx, opts);
}

}  // namespace twoscale
