// Manufactured-solution pipeline (see include/twoscale/mms.hpp).  derive_data follows
// the reference's formulation (mms.cpp:30-83): sources from the strong form, Robin /
// Neumann corrections from the covector nu = cof(grad_y zeta) n^, all composed with
// zeta so the micro data live on the reference cell.
#include "twoscale/mms.hpp"

#include <cstring>

#include "../internal.h"

namespace twoscale {

namespace {

// Outward normal axis and sign of a macro side (Left/Right: x0, Bottom/Top: x1).
void side_axis(Side s, Var& v, double& sign) {
    v = (s == Side::Left || s == Side::Right) ? Var::x0 : Var::x1;
    sign = (s == Side::Left || s == Side::Bottom) ? -1.0 : 1.0;
}

std::array<std::optional<Expr>, 4> pullback_of(const Diffeo& d) {
    return {std::nullopt, std::nullopt, d.zeta.c0, d.zeta.c1};
}

}  // namespace

ProblemData derive_data(const ManufacturedCase& c) {
    ProblemData d = c.base;
    const Expr &u = c.u, &w = c.w, &v = c.v;
    const Expr Dv(d.Dv);
    d.gu1 = (u - d.u0).simplified();
    for (int s = 0; s < 4; ++s) {
        Var ax;
        double sign;
        side_axis(static_cast<Side>(s), ax, sign);
        d.gu2[s] = (Expr(sign) * u.diff(ax)).simplified();
        d.gw[s] = (Expr(sign) * (d.Dw * w.diff(ax))).simplified();
    }
    const Expr lap_u = u.diff(Var::x0).diff(Var::x0) + u.diff(Var::x1).diff(Var::x1);
    d.fu = (Expr(0.0) - lap_u).simplified();
    const Expr div_w = (d.Dw * w.diff(Var::x0)).diff(Var::x0) + (d.Dw * w.diff(Var::x1)).diff(Var::x1);
    d.fw = (Expr(0.0) - div_w).simplified();
    d.fv = (Expr(0.0) - Dv * (v.diff(Var::y0).diff(Var::y0) + v.diff(Var::y1).diff(Var::y1))).simplified();

    const auto pb = pullback_of(d.diffeo);
    const Expr v_hat = v.subst(pb).simplified();
    const Expr dv0 = v.diff(Var::y0).subst(pb).simplified();
    const Expr dv1 = v.diff(Var::y1).subst(pb).simplified();
    d.fu_flux = VecExpr{(Dv * dv0).simplified(), (Dv * dv1).simplified()};
    d.fw_flux = d.fu_flux;

    const auto& dz = d.diffeo.dzeta;
    for (int s = 0; s < 4; ++s) {
        const Vec2 n = side_normal(static_cast<Side>(s));
        // nu = cof(F) n^  with cof(F) = [[F11, -F10], [-F01, F00]]
        const Expr nu0 = (dz[1][1] * Expr(n.x) - dz[1][0] * Expr(n.y)).simplified();
        const Expr nu1 = (dz[0][0] * Expr(n.y) - dz[0][1] * Expr(n.x)).simplified();
        const Expr len = sqrt(nu0 * nu0 + nu1 * nu1);
        const Expr flux = (Dv * (dv0 * nu0 + dv1 * nu1) / len).simplified();
        switch (d.roles.micro_side(static_cast<Side>(s))) {
            case MicroRole::GammaI: d.gv[s] = (flux - Expr(d.kappa1) * u + Expr(d.kappa2) * v_hat).simplified(); break;
            case MicroRole::GammaO: d.gv[s] = (flux - Expr(d.kappa3) * w + Expr(d.kappa4) * v_hat).simplified(); break;
            case MicroRole::GammaN: d.gv[s] = flux; break;
        }
    }
    return d;
}

namespace {

// The twelve tapes ts_error_norms expects (mms.cpp:250-266).
std::vector<CompiledExpr> error_tapes(const ManufacturedCase& c) {
    const ParamMap& pm = c.base.params;
    const Expr v_hat = c.v.subst(pullback_of(c.base.diffeo)).simplified();
    const auto& dz = c.base.diffeo.dzeta;
    std::vector<CompiledExpr> t;
    t.reserve(12);
    t.emplace_back(c.u, pm);
    t.emplace_back(c.w, pm);
    t.emplace_back(c.u.diff(Var::x0).simplified(), pm);
    t.emplace_back(c.u.diff(Var::x1).simplified(), pm);
    t.emplace_back(c.w.diff(Var::x0).simplified(), pm);
    t.emplace_back(c.w.diff(Var::x1).simplified(), pm);
    t.emplace_back(v_hat, pm);
    t.emplace_back(v_hat.diff(Var::x0).simplified(), pm);
    t.emplace_back(v_hat.diff(Var::x1).simplified(), pm);
    t.emplace_back(v_hat.diff(Var::y0).simplified(), pm);
    t.emplace_back(v_hat.diff(Var::y1).simplified(), pm);
    t.emplace_back((dz[0][0] * dz[1][1] - dz[0][1] * dz[1][0]).simplified(), pm);
    return t;
}

ts_grid_desc desc_of(const Grid& g) {
    ts_grid_desc d{};
    d.lo[0] = g.domain().lo.x;
    d.lo[1] = g.domain().lo.y;
    d.hi[0] = g.domain().hi.x;
    d.hi[1] = g.domain().hi.y;
    d.n[0] = g.n0();
    d.n[1] = g.n1();
    return d;
}

}  // namespace

ErrorNorms error_norms(const TwoScaleState& state, const ManufacturedCase& c, const Grid& macro, const Grid& micro,
                       int /*workers*/) {
    const std::vector<CompiledExpr> tapes = error_tapes(c);
    std::vector<ts_tape> tt;
    for (const auto& e : tapes) tt.push_back(e.tape());
    const int nM = macro.node_count(), nm = micro.node_count();
    std::vector<double> V(static_cast<std::size_t>(nM) * nm);
    for (int i = 0; i < nM; ++i) std::memcpy(V.data() + static_cast<std::size_t>(i) * nm, state.V[i].data(), nm * sizeof(double));
    const ts_grid_desc Md = desc_of(macro), md = desc_of(micro);
    double out[4];
    throw_status(ts_error_norms(&Md, &md, tt.data(), state.u.data(), state.w.data(), V.data(), out));
    return ErrorNorms{out[0], out[1], out[2], out[3]};
}

double observed_order(double e1, double n1, double e2, double n2) {
    if (!(e1 > 0.0) || !(e2 > 0.0) || !(n1 > 0.0) || !(n2 > 0.0) || n1 == n2) return NAN;
    return std::log(e1 / e2) / std::log(std::sqrt(n2 / n1));
}

ErrorReport convergence_sweep(const ManufacturedCase& c, const std::vector<int>& ns, const SolveOptions& opts) {
    const ProblemData derived = derive_data(c);
    const std::vector<CompiledExpr> tapes = error_tapes(c);
    std::vector<ts_tape> tt;
    for (const auto& e : tapes) tt.push_back(e.tape());
    ErrorReport report;
    for (int n : ns) {
        const Grid macro(c.macro_domain, n, n);
        const Grid micro(c.micro_domain, n, n);
        AssemblyContext ctx(derived, macro, micro, opts.workers);
        ts_solve_opts o{opts.inner_tol, opts.inner_maxit, opts.outer_tol, opts.max_outer};
        ts_solve_report rep{};
        throw_status(ts_fixed_point_solve(ctx.handle(), &o, &rep, nullptr, 0));
        if (!rep.converged)
            throw SolverError("outer iteration did not converge at n = " + std::to_string(n) + ", last residual " +
                              std::to_string(rep.final_residual));
        double out[4];
        throw_status(ts_ctx_error_norms(ctx.handle(), tt.data(), out));  // device-resident state
        ErrorReportRow row;
        row.n = n;
        row.macro_dofs = macro.node_count();
        row.micro_dofs = micro.node_count();
        row.H = (c.macro_domain.hi.x - c.macro_domain.lo.x) / n;
        row.h = (c.micro_domain.hi.x - c.micro_domain.lo.x) / n;
        row.e_uw = out[0];
        row.e_uw_grad = out[1];
        row.e_v = out[2];
        row.e_v_grad = out[3];
        if (!report.empty()) {
            const ErrorReportRow& prev = report.back();
            row.p_macro = observed_order(prev.e_uw, prev.macro_dofs, row.e_uw, row.macro_dofs);
            row.q_macro = observed_order(prev.e_uw_grad, prev.macro_dofs, row.e_uw_grad, row.macro_dofs);
            row.p_micro = observed_order(prev.e_v, prev.micro_dofs, row.e_v, row.micro_dofs);
            row.q_micro = observed_order(prev.e_v_grad, prev.micro_dofs, row.e_v_grad, row.micro_dofs);
        }
        report.push_back(row);
    }
    return report;
}

}  // namespace twoscale

extern "C" int32_t ts_mms_sweep_ini(const char* ini_text, const int32_t* ns, int32_t n_ns, double* rows) {
    using namespace twoscale;
    if (!ini_text || !ns || !rows || n_ns < 0) return ts_set_error_for_front_end(TS_ERR_INVALID, "null argument");
    try {
        const Config cfg = parse_config(ini_text);
        if (!cfg.has_mms) throw ConfigError("mms subcommand needs an [mms] section");
        const ProblemSetup setup = make_problem(cfg);
        SolveOptions o;
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
        return TS_OK;
    } catch (const ConfigError& e) {
        return ts_set_error_for_front_end(TS_ERR_CONFIG, e.what());
    } catch (const DegenerateMapError& e) {
        return ts_set_error_for_front_end(TS_ERR_DEGENERATE_MAP, e.what());
    } catch (const SolverError& e) {
        return ts_set_error_for_front_end(TS_ERR_SOLVER, e.what());
    } catch (const EvalError& e) {
        return ts_set_error_for_front_end(TS_ERR_EXPR, e.what());
    } catch (const std::exception& e) {
        return ts_set_error_for_front_end(TS_ERR_INVALID, e.what());
    }
}

extern "C" int32_t ts_ctx_create_mms_ini(const char* ini_text, ts_ctx** out) {
    using namespace twoscale;
    if (!ini_text || !out) return ts_set_error_for_front_end(TS_ERR_INVALID, "null argument");
    *out = nullptr;
    try {
        const Config cfg = parse_config(ini_text);
        if (!cfg.has_mms) throw ConfigError("mms subcommand needs an [mms] section");
        const ProblemSetup setup = make_problem(cfg);
        const ProblemData derived = derive_data(setup.mms);
        LoweredProblem L = lower_problem(derived, setup.macro, setup.micro);
        const int rc = ts_ctx_create(&L.desc, out);
        if (rc != TS_OK) return rc;
        const ts_solve_opts o{cfg.inner_tol, cfg.inner_maxit, cfg.outer_tol, cfg.max_outer};
        tsb_set_default_opts(*out, &o);
        return TS_OK;
    } catch (const ConfigError& e) {
        return ts_set_error_for_front_end(TS_ERR_CONFIG, e.what());
    } catch (const EvalError& e) {
        return ts_set_error_for_front_end(TS_ERR_EXPR, e.what());
    } catch (const std::exception& e) {
        return ts_set_error_for_front_end(TS_ERR_INVALID, e.what());
    }
}

extern "C" int32_t ts_error_norms_ini(const char* ini_text, const double* u, const double* w, const double* V,
                                      double* out) {
    using namespace twoscale;
    if (!ini_text || !u || !w || !V || !out) return ts_set_error_for_front_end(TS_ERR_INVALID, "null argument");
    try {
        const Config cfg = parse_config(ini_text);
        if (!cfg.has_mms) throw ConfigError("mms subcommand needs an [mms] section");
        const ProblemSetup setup = make_problem(cfg);
        const std::vector<CompiledExpr> tapes = twoscale::error_tapes(setup.mms);
        std::vector<ts_tape> tt;
        for (const auto& e : tapes) tt.push_back(e.tape());
        const ts_grid_desc Md = twoscale::desc_of(setup.macro), md = twoscale::desc_of(setup.micro);
        return ts_error_norms(&Md, &md, tt.data(), u, w, V, out);
    } catch (const ConfigError& e) {
        return ts_set_error_for_front_end(TS_ERR_CONFIG, e.what());
    } catch (const std::exception& e) {
        return ts_set_error_for_front_end(TS_ERR_INVALID, e.what());
    }
}
