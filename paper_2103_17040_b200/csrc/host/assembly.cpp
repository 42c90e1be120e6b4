// AssemblyContext over the device context (see include/twoscale/assembly.hpp).
#include "twoscale/assembly.hpp"

#include <cstring>

#include "twoscale/config.hpp"

namespace twoscale {

void throw_status(int status) {
    switch (status) {
        case TS_OK: return;
        case TS_ERR_CONFIG: throw ConfigError(ts_last_error());
        case TS_ERR_EXPR: throw EvalError(ts_last_error());
        case TS_ERR_DEGENERATE_MAP: throw DegenerateMapError(ts_last_error());
        case TS_ERR_SOLVER: throw SolverError(ts_last_error());
        case TS_ERR_INVALID: throw std::invalid_argument(ts_last_error());
        default: throw std::runtime_error(ts_last_error());
    }
}

CsrMatrix make_q1_matrix(const Grid& grid) {
    std::vector<std::vector<int>> pattern(grid.node_count());
    for (int j = 0; j <= grid.n1(); ++j)
        for (int i = 0; i <= grid.n0(); ++i) {
            auto& row = pattern[grid.node_index(i, j)];
            for (int dj = -1; dj <= 1; ++dj)
                for (int di = -1; di <= 1; ++di) {
                    const int ii = i + di, jj = j + dj;
                    if (ii >= 0 && ii <= grid.n0() && jj >= 0 && jj <= grid.n1()) row.push_back(grid.node_index(ii, jj));
                }
        }
    return CsrMatrix(grid.node_count(), pattern);
}

AssemblyContext::AssemblyContext(const ProblemData& data, const Grid& macro, const Grid& micro, int /*workers*/)
    : data_(data), macro_(macro), micro_(micro), rule_(QuadratureRule::gauss(2)), diffeo_(data_.diffeo, data_.params) {
    macro_nodes_.resize(macro_.node_count());
    for (int i = 0; i < macro_.node_count(); ++i) macro_nodes_[i] = macro_.node(i);
    LoweredProblem L = lower_problem(data_, macro_, micro_);
    throw_status(ts_ctx_create(&L.desc, &ctx_));
    ts_ctx_info info{};
    ts_ctx_get_info(ctx_, &info);
    shared_ = info.shared_operator != 0;
    w_pinned_ = info.w_pinned != 0;
    const CsrMatrix pat = make_q1_matrix(macro_);
    CsrMatrix* mats[3] = {&A_u_, &A_w_, &M0_};
    for (int k = 0; k < 3; ++k) {
        *mats[k] = pat;
        throw_status(ts_macro_matrix(ctx_, k, nullptr, nullptr, mats[k]->values().data()));
    }
    for (int which = 0; which < 2; ++which) {
        int n = 0;
        throw_status(ts_dirichlet(ctx_, which, &n, nullptr, nullptr));
        std::vector<int> dofs(n);
        std::vector<double> vals(n);
        throw_status(ts_dirichlet(ctx_, which, &n, dofs.data(), vals.data()));
        auto& dst = which == 0 ? dirichlet_u_ : dirichlet_w_;
        for (int k = 0; k < n; ++k) dst.emplace_back(dofs[k], vals[k]);
    }
}

AssemblyContext::~AssemblyContext() { ts_ctx_destroy(ctx_); }

const CsrMatrix& AssemblyContext::micro_matrix(int node) const {
    const int key = shared_ ? 0 : node;
    std::lock_guard<std::mutex> lock(mu_);
    auto it = micro_cache_.find(key);
    if (it != micro_cache_.end()) return it->second;
    CsrMatrix A = make_q1_matrix(micro_);
    throw_status(ts_micro_values(ctx_, key, A.values().data()));
    return micro_cache_.emplace(key, std::move(A)).first->second;
}

void AssemblyContext::micro_rhs(int node, double u_i, double w_i, std::vector<double>& out) const {
    out.assign(micro_.node_count(), 0.0);
    throw_status(ts_micro_rhs(ctx_, node, u_i, w_i, out.data()));
}

SparseSystem AssemblyContext::assemble_micro(int node, double u_i, double w_i) const {
    SparseSystem s;
    s.A = micro_matrix(node);
    micro_rhs(node, u_i, w_i, s.b);
    return s;
}

double AssemblyContext::surface_coupling(const std::vector<double>& v, int node, MicroRole role) const {
    double out = 0.0;
    const int r = role == MicroRole::GammaI ? TS_GAMMA_I : role == MicroRole::GammaO ? TS_GAMMA_O : TS_GAMMA_N;
    throw_status(ts_surface_coupling(ctx_, v.data(), node, r, &out));
    return out;
}

std::vector<double> AssemblyContext::macro_rhs(int which, const MicroField& V) const {
    const int nM = macro_.node_count(), nm = micro_.node_count();
    std::vector<double> flat(static_cast<std::size_t>(nM) * nm);
    for (int i = 0; i < nM; ++i) std::memcpy(flat.data() + static_cast<std::size_t>(i) * nm, V[i].data(), nm * sizeof(double));
    std::vector<double> out(nM);
    throw_status(ts_macro_rhs(ctx_, which, flat.data(), out.data()));
    return out;
}

std::vector<double> AssemblyContext::macro_u_rhs(const MicroField& V) const { return macro_rhs(0, V); }
std::vector<double> AssemblyContext::macro_w_rhs(const MicroField& V) const { return macro_rhs(1, V); }

SparseSystem AssemblyContext::assemble_macro_u(const MicroField& V) const {
    return SparseSystem{A_u_, macro_u_rhs(V), dirichlet_u_};
}

SparseSystem AssemblyContext::assemble_macro_w(const MicroField& V) const {
    return SparseSystem{A_w_, macro_w_rhs(V), dirichlet_w_};
}

const MapCache& AssemblyContext::node_cache() const {
    std::lock_guard<std::mutex> lock(mu_);
    if (node_cache_) return *node_cache_;
    auto m = std::make_unique<MapCache>();
    m->points_ = macro_.node_count();
    m->rows_ = shared_ || m->points_ == 1 ? 1 : m->points_;
    m->nq_cell_ = 4;
    m->nq_face_ = 2;
    m->cell_stride_ = static_cast<std::size_t>(micro_.cell_count()) * 4;
    m->face_stride_ = micro_.boundary_faces().size() * 2;
    m->cells_.resize(m->cell_stride_ * m->rows_);
    m->faces_.resize(m->face_stride_ * m->rows_);
    std::vector<double> c(m->cell_stride_ * 4), f(m->face_stride_ * 4);
    for (int r = 0; r < m->rows_; ++r) {
        throw_status(ts_node_cache(ctx_, r, c.data(), f.data()));
        for (std::size_t k = 0; k < m->cell_stride_; ++k)
            m->cells_[r * m->cell_stride_ + k] = {c[4 * k], c[4 * k + 1], c[4 * k + 2], c[4 * k + 3]};
        for (std::size_t k = 0; k < m->face_stride_; ++k)
            m->faces_[r * m->face_stride_ + k] = {f[4 * k], {f[4 * k + 1], f[4 * k + 2]}, f[4 * k + 3]};
    }
    node_cache_ = std::move(m);
    return *node_cache_;
}

}  // namespace twoscale
