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
};

// Lowers ProblemData + grids to the flat C ABI description.  The returned object
// owns every tape the description points into.
struct LoweredProblem {
    ts_problem_desc desc{};
    std::vector<CompiledExpr> tapes;  // storage
};
LoweredProblem lower_problem(const ProblemData& data, const Grid& macro, const Grid& micro);

}  // namespace twoscale
