// Problem data — drop-in for proj/include/twoscale/problem.hpp, plus the B200
// extensions needed by the BASELINE configs.  With the extension fields at their
// defaults (D = I, no reaction, no table) the problem is exactly the reference's.
#pragma once

#include <array>
#include <optional>

#include "twoscale/expr.hpp"
#include "twoscale/grid.hpp"
#include "twoscale/mapping.hpp"

namespace twoscale {

struct ProblemData {
    double kappa1 = 1.0, kappa2 = 1.0, kappa3 = 1.0, kappa4 = 1.0;
    double Dv = 1.0;
    Expr Dw{1.0};
    Expr fu{0.0}, fv{0.0}, fw{0.0}, u0{0.0};
    Expr gu1{0.0};
    std::array<Expr, 4> gu2{}, gw{}, gv{};
    std::optional<VecExpr> fu_flux, fw_flux;
    Diffeo diffeo = Diffeo::identity();
    BoundaryRoles roles;
    MapBounds bounds;
    ParamMap params;

    // ---- B200 extensions (not expressible in the reference) -------------------
    Mat2 D = Mat2::identity();        // physical-frame micro diffusion tensor: A = C^T D C / det
    int reaction_kind = TS_REACTION_CONST;
    std::array<double, 5> reaction{0.0, 0.0, 0.0, 0.0, 0.0};  // k | k_in, k_out, cx, cy, r
    TabulatedMap table;               // non-empty: replaces `diffeo` for the micro map
    // generic micro geometry (configs 4-5): dimension, element order, third axis
    int micro_dim = 2, micro_order = 1;
    int micro_n2 = 0;
    double micro_lo2 = 0.0, micro_hi2 = 1.0;
    std::array<double, 9> D3{1, 0, 0, 0, 1, 0, 0, 0, 1};
    std::array<MicroRole, 2> micro_role3{MicroRole::GammaI, MicroRole::GammaI};
    double reaction_cz = 0.0;
    bool force_generic = false;       // route 2D Q1 through the generic kernels (tests)
};

// Lowers ProblemData + grids to the flat C ABI description.  The returned object
// owns every tape the description points into.
struct LoweredProblem {
    ts_problem_desc desc{};
    std::vector<CompiledExpr> tapes;  // storage
};
LoweredProblem lower_problem(const ProblemData& data, const Grid& macro, const Grid& micro);

}  // namespace twoscale
