// Internal declarations shared by the translation units of the C ABI (ctx.cu: context
// build and solve; ctx_io.cu: error norms and VTK egress).  Not part of the ABI.
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "generic.h"
#include "internal.h"
#include "kernels.h"
#include "twoscale_b200.h"

namespace tsb {

extern thread_local std::string g_err;
extern thread_local int g_err_index;

inline int fail(int code, const char* fmt, ...) {
    char buf[1024];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

struct CudaError {
    int code;
};

#define CU(call)                                                                               \
    do {                                                                                       \
        cudaError_t e_ = (call);                                                               \
        if (e_ != cudaSuccess) {                                                               \
            fail(TS_ERR_CUDA, "CUDA error %s at %s:%d: %s", cudaGetErrorName(e_), __FILE__,    \
                 __LINE__, cudaGetErrorString(e_));                                            \
            throw CudaError{TS_ERR_CUDA};                                                      \
        }                                                                                      \
    } while (0)

// Device buffers of contexts go through a small process-wide caching allocator:
// freed blocks are kept (per device, by exact size, up to kCacheCap bytes) and handed
// to the next context asking for the same size.  The C ABI's end-to-end path builds
// and destroys a multi-GB context per solve; without the cache every build re-maps
// ~7 GB and the driver's lazy unmapping of the previous context shows up as
// 0.1-0.5 s stalls in cudaMalloc.
class BlockCache {
public:
    static BlockCache& get();
    void* take(size_t bytes) {
        int dev = 0;
        cudaGetDevice(&dev);
        {
            std::lock_guard<std::mutex> lock(mu_);
            auto it = free_.find({dev, bytes});
            if (it != free_.end() && !it->second.empty()) {
                void* p = it->second.back();
                it->second.pop_back();
                cached_ -= bytes;
                return p;
            }
        }
        void* p = nullptr;
        if (cudaMalloc(&p, bytes) != cudaSuccess) {
            cudaGetLastError();  // clear, then retry once with the cache emptied
            trim();
            if (cudaMalloc(&p, bytes) != cudaSuccess) return nullptr;
        }
        return p;
    }
    void give(void* p, size_t bytes) {
        int dev = 0;
        cudaGetDevice(&dev);
        std::lock_guard<std::mutex> lock(mu_);
        if (cached_ + bytes > kCacheCap) {
            cudaFree(p);
            return;
        }
        free_[{dev, bytes}].push_back(p);
        cached_ += bytes;
    }
    void trim() {
        std::lock_guard<std::mutex> lock(mu_);
        int cur = 0;
        cudaGetDevice(&cur);
        for (auto& kv : free_) {
            cudaSetDevice(kv.first.first);
            for (void* p : kv.second) cudaFree(p);
        }
        cudaSetDevice(cur);
        free_.clear();
        cached_ = 0;
    }

private:
    static constexpr size_t kCacheCap = size_t(48) << 30;
    std::mutex mu_;
    std::map<std::pair<int, size_t>, std::vector<void*>> free_;
    size_t cached_ = 0;
};

template <class T>
struct DBuf {
    T* p = nullptr;
    size_t n = 0;
    void alloc(size_t count) {
        release();
        n = count;
        if (!count) return;
        p = static_cast<T*>(BlockCache::get().take(count * sizeof(T)));
        if (!p) {
            n = 0;
            fail(TS_ERR_CUDA, "device allocation of %zu bytes failed", count * sizeof(T));
            throw CudaError{TS_ERR_CUDA};
        }
    }
    void zero(cudaStream_t s) {
        if (n) CU(cudaMemsetAsync(p, 0, n * sizeof(T), s));
    }
    void release() {
        if (p) BlockCache::get().give(p, n * sizeof(T));  // callers have synchronised their stream
        p = nullptr;
        n = 0;
    }
    size_t bytes() const { return n * sizeof(T); }
    ~DBuf() { release(); }
};

// Gauss-2 + Q1 tables built exactly like the reference (grid.cpp:109-119, 134-141).
inline QuadTables make_quad() {
    QuadTables q{};
    const double g = 1.0 / std::sqrt(3.0);
    q.GP[0] = -g;
    q.GP[1] = g;
    q.GW[0] = 1.0;
    q.GW[1] = 1.0;
    for (int j = 0; j < 2; ++j)
        for (int i = 0; i < 2; ++i) {
            q.QS[j * 2 + i] = q.GP[i];
            q.QT[j * 2 + i] = q.GP[j];
            q.QW[j * 2 + i] = q.GW[i] * q.GW[j];
        }
    for (int k = 0; k < 4; ++k) {
        const double s = q.QS[k], t = q.QT[k];
        q.N[k][0] = 0.25 * (1.0 - s) * (1.0 - t);
        q.N[k][1] = 0.25 * (1.0 + s) * (1.0 - t);
        q.N[k][2] = 0.25 * (1.0 + s) * (1.0 + t);
        q.N[k][3] = 0.25 * (1.0 - s) * (1.0 + t);
        q.dN[k][0][0] = -0.25 * (1.0 - t);
        q.dN[k][0][1] = -0.25 * (1.0 - s);
        q.dN[k][1][0] = 0.25 * (1.0 - t);
        q.dN[k][1][1] = -0.25 * (1.0 + s);
        q.dN[k][2][0] = 0.25 * (1.0 + t);
        q.dN[k][2][1] = 0.25 * (1.0 + s);
        q.dN[k][3][0] = -0.25 * (1.0 + t);
        q.dN[k][3][1] = 0.25 * (1.0 - s);
    }
    for (int k = 0; k < 2; ++k) {
        q.Nf[k][0] = 0.5 * (1.0 - q.GP[k]);
        q.Nf[k][1] = 0.5 * (1.0 + q.GP[k]);
    }
    return q;
}

inline GridG to_grid(const ts_grid_desc& d) {
    GridG g;
    g.lo0 = d.lo[0];
    g.lo1 = d.lo[1];
    g.n0 = d.n[0];
    g.n1 = d.n[1];
    g.h0 = (d.hi[0] - d.lo[0]) / d.n[0];  // grid.cpp:31-32
    g.h1 = (d.hi[1] - d.lo[1]) / d.n[1];
    return g;
}

// make_q1_matrix pattern (assembly.cpp:34-50): rows lexicographic, dj outer, di inner.
inline void q1_pattern(const GridG& g, std::vector<int>& rp, std::vector<int>& ci) {
    const int n = g.nodes();
    rp.assign(n + 1, 0);
    ci.clear();
    ci.reserve((size_t)9 * n);
    for (int j = 0; j <= g.n1; ++j)
        for (int i = 0; i <= g.n0; ++i) {
            for (int dj = -1; dj <= 1; ++dj) {
                if (j + dj < 0 || j + dj > g.n1) continue;
                for (int di = -1; di <= 1; ++di) {
                    if (i + di < 0 || i + di > g.n0) continue;
                    ci.push_back((j + dj) * (g.n0 + 1) + i + di);
                }
            }
            rp[j * (g.n0 + 1) + i + 1] = (int)ci.size();
        }
}

// Packs host tapes into one instruction stream.
struct TapePack {
    std::vector<int> op, arg;
    std::vector<double> val;
    TapeRef add(const ts_tape& t) {
        TapeRef r{(int)op.size(), t.n};
        for (int k = 0; k < t.n; ++k) {
            op.push_back(t.op[k]);
            arg.push_back(t.arg[k]);
            val.push_back(t.val[k]);
        }
        return r;
    }
};

inline bool check_tape(const ts_tape& t) { return t.n == 0 || (t.op && t.arg && t.val && t.max_stack <= TS_MAX_TAPE_STACK); }

inline const char* expr_error(unsigned e) {
    if (e & ERR_DIV0) return "division by zero";
    if (e & ERR_SQRT) return "sqrt of negative value";
    return "expression evaluation error";
}

}  // namespace tsb

using namespace tsb;

struct ts_ctx {
    ProblemG P{};
    bool gen = false;      // Q2 / 3D micro problems (configs 4-5): generic kernels
    GenProblem GP{};
    int ncoef = 4;
    int nM = 0, nm = 0, rows = 0, nfaces = 0, ncells = 0, Mcells = 0;
    bool shared = false, has_fixed = false;
    std::vector<int> mrp, mci, Mrp, Mci;
    std::vector<int> dir_u;
    std::vector<double> dir_u_val;
    int w_pinned = 0;
    QuadTables Q{};
    double setup_ms = 0.0;
    ts_solve_opts default_opts{1e-10, 20000, 1e-8, 100};

    cudaStream_t stream = nullptr;
    DBuf<int> t_op, t_arg;
    DBuf<double> t_val, A_table;
    DBuf<double4> cells, faces;
    DBuf<double> gcells, gfaces;  // generic caches: [row][cell][q][ncoef], [row][face][qf] |nu|
    DBuf<double> gscratch;        // generic PCG vectors when a micro problem exceeds SMEM
    DBuf<double> stencil, qstencil, tensor, fixed, rin, rout, face_len;
    DBuf<int> d_Mrp, d_Mci;
    DBuf<double> Au, Aw, M0, bfix;   // bfix [2][nM]: b_u_fixed, b_w_fixed
    DBuf<double> Ae, shift;          // Ae [2][nnz], shift [2][nM]
    DBuf<unsigned char> cmask;       // [2][nM]
    DBuf<double> cval;               // [2][nM]
    // state
    DBuf<double> uw, V, coupling, res_v, final_rel, raw, cons, cg_scratch, cg_res_d, sweep_out, cg_partials;
    DBuf<int> iters, status, cg_res_i, counter, order;
    // macro u/w solves on the SMEM-resident stencil PCG (macro grids that fit one SM)
    bool macro_stencil = false;
    int macro_cluster = 0;  // cluster size of the macro solve (mcluster.cu), 0: cooperative CSR CG
    DBuf<double> mstencil, mzero, mrel;  // [2][9][nM], [2], [2]
    DBuf<int> mstatus, miters, mcounter;
    DBuf<unsigned long long> first_bad;
    DBuf<unsigned> err;
    // device-side sweep loop (sweeps 2.. as one CUDA graph with a conditional while node)
    DBuf<double> sweep_log;             // [max_outer][kSweepLog]
    DBuf<unsigned long long> stamps;    // [max_outer][4]
    DBuf<double> ctl_buf;               // SweepCtl
    cudaGraphExec_t sweep_graph = nullptr;
    int graph_launches = 0;             // kernels one graph sweep launches
    double graph_key[4] = {0, 0, 0, 0};  // inner_tol, inner_maxit, outer_tol, max_outer it was built for
    double* h_pinned = nullptr;  // small pinned staging block
    bool state_valid = false;
    TapeRef zeta[2]{};           // TAPE map values (VTK pushforward only)
    bool has_zeta = false;
    double* h_stage[2] = {nullptr, nullptr};  // pinned VTK staging, kept for later writes
    size_t h_stage_bytes = 0;

    ~ts_ctx() {
        if (stream) cudaStreamSynchronize(stream);  // members return their blocks to the cache
        if (sweep_graph) cudaGraphExecDestroy(sweep_graph);
        if (h_pinned) cudaFreeHost(h_pinned);
        for (double* p : h_stage)
            if (p) cudaFreeHost(p);
        if (stream) cudaStreamDestroy(stream);
    }

    long long device_bytes() const {
        return (long long)(gcells.bytes() + gfaces.bytes() + t_op.bytes() + t_arg.bytes() + t_val.bytes() + A_table.bytes() + cells.bytes() +
                           faces.bytes() + stencil.bytes() + qstencil.bytes() + fixed.bytes() + rin.bytes() + rout.bytes() +
                           face_len.bytes() + tensor.bytes() + d_Mrp.bytes() + d_Mci.bytes() + Au.bytes() + Aw.bytes() +
                           M0.bytes() + bfix.bytes() + Ae.bytes() + shift.bytes() + cmask.bytes() +
                           cval.bytes() + uw.bytes() + V.bytes() + coupling.bytes() + res_v.bytes() +
                           final_rel.bytes() + raw.bytes() + cons.bytes() + cg_scratch.bytes() +
                           cg_res_d.bytes() + sweep_out.bytes() + iters.bytes() + status.bytes() +
                           cg_res_i.bytes() + counter.bytes());
    }

    void sync() { CU(cudaStreamSynchronize(stream)); }
};

namespace tsb {

int device_ready();
void reset_flags(ts_ctx* c);

// Runs f, mapping CUDA failures (thrown by CU) and C++ exceptions to a ts_status.
template <class F>
int guarded(F&& f) {
    try {
        g_err_index = -1;
        return f();
    } catch (const CudaError& e) {
        return e.code;
    } catch (const std::exception& e) {
        return fail(TS_ERR_INVALID, "%s", e.what());
    }
}

}  // namespace tsb
