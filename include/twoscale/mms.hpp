// Manufactured-solution pipeline — drop-in for proj/include/twoscale/mms.hpp
// (derive_data, error_norms, observed_order, convergence_sweep).  The symbolic
// derivation runs on the host; the solves and the error quadrature run on the
// device (ts_fixed_point_solve, ts_error_norms).  residual_check (a host sampling
// diagnostic) is not part of the B200 library.
#pragma once

#include <cmath>
#include <vector>

#include "twoscale/config.hpp"
#include "twoscale/solver.hpp"

namespace twoscale {

ProblemData derive_data(const ManufacturedCase& c);

struct ErrorNorms {
    double e_uw = 0.0;
    double e_uw_grad = 0.0;
    double e_v = 0.0;
    double e_v_grad = 0.0;
};

ErrorNorms error_norms(const TwoScaleState& state, const ManufacturedCase& c, const Grid& macro, const Grid& micro,
                       int workers);

double observed_order(double e1, double n1, double e2, double n2);

struct ErrorReportRow {
    int n = 0;
    int macro_dofs = 0, micro_dofs = 0;
    double H = 0.0, h = 0.0;
    double e_uw = 0.0, e_uw_grad = 0.0, e_v = 0.0, e_v_grad = 0.0;
    double p_macro = NAN, q_macro = NAN;
    double p_micro = NAN, q_micro = NAN;
};
using ErrorReport = std::vector<ErrorReportRow>;

ErrorReport convergence_sweep(const ManufacturedCase& c, const std::vector<int>& ns, const SolveOptions& opts);

}  // namespace twoscale
