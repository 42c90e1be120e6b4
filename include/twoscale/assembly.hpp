// AssemblyContext — drop-in for proj/include/twoscale/assembly.hpp.  The context
// lives on the B200 (ts_ctx): map caches, micro operators, rhs parts and macro
// systems are built there by kernels (1)-(2); the accessors below download what a
// caller asks for, on demand.
#pragma once

#include <map>
#include <memory>
#include <mutex>
#include <vector>

#include "twoscale/grid.hpp"
#include "twoscale/linalg.hpp"
#include "twoscale/mapping.hpp"
#include "twoscale/problem.hpp"

namespace twoscale {

using MicroField = std::vector<std::vector<double>>;

class AssemblyContext {
public:
    AssemblyContext(const ProblemData& data, const Grid& macro, const Grid& micro, int workers);
    ~AssemblyContext();
    AssemblyContext(const AssemblyContext&) = delete;
    AssemblyContext& operator=(const AssemblyContext&) = delete;

    const Grid& macro_grid() const { return macro_; }
    const Grid& micro_grid() const { return micro_; }
    const QuadratureRule& rule() const { return rule_; }
    const ProblemData& data() const { return data_; }
    const CompiledDiffeo& diffeo() const { return diffeo_; }
    const MapCache& node_cache() const;  // downloaded on first use
    const std::vector<Vec2>& macro_nodes() const { return macro_nodes_; }

    SparseSystem assemble_micro(int node, double u_i, double w_i) const;
    SparseSystem assemble_macro_u(const MicroField& V) const;
    SparseSystem assemble_macro_w(const MicroField& V) const;
    double surface_coupling(const std::vector<double>& v_node, int node, MicroRole role) const;

    const CsrMatrix& micro_matrix(int node) const;  // downloaded on first use
    void micro_rhs(int node, double u_i, double w_i, std::vector<double>& out) const;

    const CsrMatrix& macro_u_matrix() const { return A_u_; }
    const CsrMatrix& macro_w_matrix() const { return A_w_; }
    const CsrMatrix& macro_mass() const { return M0_; }
    const std::vector<std::pair<int, double>>& dirichlet_u() const { return dirichlet_u_; }
    const std::vector<std::pair<int, double>>& dirichlet_w() const { return dirichlet_w_; }
    bool w_pinned() const { return w_pinned_; }

    std::vector<double> macro_u_rhs(const MicroField& V) const;
    std::vector<double> macro_w_rhs(const MicroField& V) const;

    // B200 additions
    ts_ctx* handle() const { return ctx_; }
    bool shared_operator() const { return shared_; }

private:
    ProblemData data_;
    const Grid& macro_;
    const Grid& micro_;
    QuadratureRule rule_;
    CompiledDiffeo diffeo_;
    std::vector<Vec2> macro_nodes_;
    ts_ctx* ctx_ = nullptr;
    bool shared_ = false;
    CsrMatrix A_u_, A_w_, M0_;
    std::vector<std::pair<int, double>> dirichlet_u_, dirichlet_w_;
    bool w_pinned_ = false;
    mutable std::mutex mu_;
    mutable std::map<int, CsrMatrix> micro_cache_;
    mutable std::unique_ptr<MapCache> node_cache_;
    std::vector<double> macro_rhs(int which, const MicroField& V) const;
};

CsrMatrix make_q1_matrix(const Grid& grid);

// Throws the reference exception type matching a ts_status (no-op on TS_OK).
void throw_status(int status);

}  // namespace twoscale
