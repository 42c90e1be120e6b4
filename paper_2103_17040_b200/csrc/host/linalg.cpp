// Host CSR container + device-backed cg_solve (see include/twoscale/linalg.hpp).
#include "twoscale/linalg.hpp"

#include <algorithm>

#include "twoscale/assembly.hpp"
#include "twoscale_b200.h"

namespace twoscale {

CsrMatrix::CsrMatrix(int n, const std::vector<std::vector<int>>& pattern) : n_(n) {
    row_ptr_.assign(n + 1, 0);
    for (int r = 0; r < n; ++r) {
        row_ptr_[r + 1] = row_ptr_[r] + static_cast<int>(pattern[r].size());
        col_idx_.insert(col_idx_.end(), pattern[r].begin(), pattern[r].end());
    }
    vals_.assign(col_idx_.size(), 0.0);
}

CsrMatrix::CsrMatrix(int n, std::vector<int> row_ptr, std::vector<int> col_idx, std::vector<double> vals)
    : n_(n), row_ptr_(std::move(row_ptr)), col_idx_(std::move(col_idx)), vals_(std::move(vals)) {}

void CsrMatrix::zero() { std::fill(vals_.begin(), vals_.end(), 0.0); }

int CsrMatrix::find(int row, int col) const {
    const auto b = col_idx_.begin() + row_ptr_[row], e = col_idx_.begin() + row_ptr_[row + 1];
    const auto it = std::lower_bound(b, e, col);
    return (it != e && *it == col) ? static_cast<int>(it - col_idx_.begin()) : -1;
}

void CsrMatrix::add(int row, int col, double v) {
    const int k = find(row, col);
    if (k < 0) throw SolverError("matrix entry outside sparsity pattern");
    vals_[k] += v;
}

double CsrMatrix::get(int row, int col) const {
    const int k = find(row, col);
    return k < 0 ? 0.0 : vals_[k];
}

void CsrMatrix::apply(const std::vector<double>& x, std::vector<double>& y) const {
    y.assign(n_, 0.0);
    for (int r = 0; r < n_; ++r) {
        double s = 0.0;
        for (int k = row_ptr_[r]; k < row_ptr_[r + 1]; ++k) s += vals_[k] * x[col_idx_[k]];
        y[r] = s;
    }
}

std::vector<double> CsrMatrix::diagonal() const {
    std::vector<double> d(n_);
    for (int r = 0; r < n_; ++r) d[r] = get(r, r);
    return d;
}

void CsrMatrix::eliminate(const std::vector<std::pair<int, double>>& constraints, std::vector<double>& b) {
    if (constraints.empty()) return;
    std::vector<char> fixed(n_, 0);
    std::vector<double> g(n_, 0.0);
    for (const auto& [dof, val] : constraints) {
        fixed[dof] = 1;
        g[dof] = val;
    }
    for (int r = 0; r < n_; ++r) {
        for (int k = row_ptr_[r]; k < row_ptr_[r + 1]; ++k) {
            const int c = col_idx_[k];
            if (fixed[r]) {
                vals_[k] = c == r ? 1.0 : 0.0;
            } else if (fixed[c]) {
                b[r] -= vals_[k] * g[c];
                vals_[k] = 0.0;
            }
        }
        if (fixed[r]) b[r] = g[r];
    }
}

double CsrMatrix::symmetry_error() const {
    double big = 0.0, diff = 0.0;
    for (int r = 0; r < n_; ++r)
        for (int k = row_ptr_[r]; k < row_ptr_[r + 1]; ++k) {
            big = std::max(big, std::abs(vals_[k]));
            if (col_idx_[k] > r) diff = std::max(diff, std::abs(vals_[k] - get(col_idx_[k], r)));
        }
    return big > 0.0 ? diff / big : 0.0;
}

double norm2(const std::vector<double>& v) {
    double s = 0.0;
    for (double a : v) s += a * a;
    return std::sqrt(s);
}

void axpy(double a, const std::vector<double>& x, std::vector<double>& y) {
    for (std::size_t i = 0; i < y.size(); ++i) y[i] += a * x[i];
}

CgResult cg_solve(const CsrMatrix& A, const std::vector<double>& b, std::vector<double>& x, double tol,
                  int maxit) {
    x.resize(A.size(), 0.0);
    ts_cg_result r{};
    throw_status(ts_cg_solve(A.size(), A.row_ptr().data(), A.col_idx().data(), A.values().data(), b.data(),
                             x.data(), tol, maxit, &r));
    CgResult out;
    out.converged = r.converged != 0;
    out.iterations = r.iterations;
    out.residual = r.residual;
    out.indefinite = r.indefinite != 0;
    return out;
}

}  // namespace twoscale
