// ProblemData -> ts_problem_desc (tapes compiled the way the reference's
// AssemblyContext constructor compiles them, assembly.cpp:52-99).
#include "twoscale/problem.hpp"

namespace twoscale {

namespace {
bool is_zero(const Expr& e) {
    double c;
    return e.is_constant(&c) && c == 0.0;
}
ts_grid_desc grid_desc(const Grid& g) {
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

LoweredProblem lower_problem(const ProblemData& data, const Grid& macro, const Grid& micro) {
    LoweredProblem L;
    L.tapes.reserve(40);
    ts_problem_desc& d = L.desc;
    d.abi_version = TS_ABI_VERSION;
    d.macro = grid_desc(macro);
    d.micro = grid_desc(micro);
    d.kappa[0] = data.kappa1;
    d.kappa[1] = data.kappa2;
    d.kappa[2] = data.kappa3;
    d.kappa[3] = data.kappa4;
    d.Dv = data.Dv;
    for (int s = 0; s < 4; ++s) {
        d.macro_bc[s] = data.roles.macro[s] == MacroBC::Dirichlet ? TS_DIRICHLET : TS_NEUMANN;
        d.micro_role[s] = data.roles.micro[s] == MicroRole::GammaI   ? TS_GAMMA_I
                          : data.roles.micro[s] == MicroRole::GammaO ? TS_GAMMA_O
                                                                     : TS_GAMMA_N;
    }
    auto tape = [&](const Expr& e) {
        L.tapes.emplace_back(e, data.params);
        return L.tapes.back().tape();
    };
    if (data.table.empty()) {
        d.map_kind = TS_MAP_TAPE;
        for (int a = 0; a < 2; ++a)
            for (int b = 0; b < 2; ++b) d.jac[2 * a + b] = tape(data.diffeo.dzeta[a][b]);
        d.zeta[0] = tape(data.diffeo.zeta.c0);
        d.zeta[1] = tape(data.diffeo.zeta.c1);
        d.jac_depends_on_x = data.diffeo.jacobian_depends_on_x();
    } else {
        const std::size_t stride = data.table.kind == TS_MAP_FOURIER_TABLE ? 16
                                   : data.micro_dim == 3                    ? 9
                                                                            : 4;
        if (data.table.A.size() != stride * static_cast<std::size_t>(macro.node_count()))
            throw std::invalid_argument("tabulated map needs " + std::to_string(stride) + " entries per macro node");
        d.map_kind = data.table.kind;
        d.A_table = data.table.A.data();
        d.s_kind = data.table.s_kind;
        d.amp = data.table.amp;
        d.jac_depends_on_x = 1;
    }
    // fv composed with zeta so the tape takes (x, yhat) (assembly.cpp:72-75)
    if (!is_zero(data.fv)) {
        const std::array<std::optional<Expr>, 4> pull{std::nullopt, std::nullopt, data.diffeo.zeta.c0,
                                                      data.diffeo.zeta.c1};
        d.fv_hat = tape(data.fv.subst(pull).simplified());
    }
    d.fu = tape(data.fu);
    d.fw = tape(data.fw);
    d.Dw = tape(data.Dw);
    d.dirichlet_value = tape((data.u0 + data.gu1).simplified());
    for (int s = 0; s < 4; ++s) {
        if (!is_zero(data.gv[s])) d.gv[s] = tape(data.gv[s]);
        if (!is_zero(data.gu2[s])) d.gu2[s] = tape(data.gu2[s]);
        if (!is_zero(data.gw[s])) d.gw[s] = tape(data.gw[s]);
    }
    if (data.fu_flux) {
        d.fu_flux[0] = tape(data.fu_flux->c0);
        d.fu_flux[1] = tape(data.fu_flux->c1);
        d.has_fu_flux = 1;
    }
    if (data.fw_flux) {
        d.fw_flux[0] = tape(data.fw_flux->c0);
        d.fw_flux[1] = tape(data.fw_flux->c1);
        d.has_fw_flux = 1;
    }
    d.D[0] = data.D.a00;
    d.D[1] = data.D.a01;
    d.D[2] = data.D.a10;
    d.D[3] = data.D.a11;
    d.reaction_kind = data.reaction_kind;
    for (int k = 0; k < 5; ++k) d.reaction[k] = data.reaction[k];
    d.micro_dim = data.micro_dim;
    d.micro_order = data.micro_order;
    d.micro_n2 = data.micro_n2;
    d.micro_lo2 = data.micro_lo2;
    d.micro_hi2 = data.micro_hi2;
    for (int k = 0; k < 9; ++k) d.D3[k] = data.D3[k];
    for (int k = 0; k < 2; ++k)
        d.micro_role3[k] = data.micro_role3[k] == MicroRole::GammaI   ? TS_GAMMA_I
                           : data.micro_role3[k] == MicroRole::GammaO ? TS_GAMMA_O
                                                                      : TS_GAMMA_N;
    d.reaction_cz = data.reaction_cz;
    d.force_generic = data.force_generic ? 1 : 0;
    return L;
}

}  // namespace twoscale
