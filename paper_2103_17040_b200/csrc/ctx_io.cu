// C ABI, part 2: error norms on the device and the micro-state
// egress (§8f rank 2: VTK writers fed from the device state).
#include "ctx_internal.h"
#include "egress.h"
#include "jit.h"
#include "mms.h"
#include "vtk_stream.h"

// ------------------------------------------------------------- error norms --
namespace {

int error_norms_impl(const GridG& macro, const GridG& micro, const ts_tape* tapes, const double* du,
                     const double* dw, const double* dV, double* out, cudaStream_t s) {
    ErrNormArgs a{};
    a.macro = macro;
    a.micro = micro;
    TapePack pack;
    for (int k = 0; k < 12; ++k) {
        if (!check_tape(tapes[k])) return fail(TS_ERR_INVALID, "malformed tape %d", k);
        a.t[k] = pack.add(tapes[k]);
    }
    const size_t ni = pack.op.size() ? pack.op.size() : 1;
    pack.op.resize(ni, 0);
    pack.arg.resize(ni, 0);
    pack.val.resize(ni, 0.0);
    DBuf<int> op, arg;
    DBuf<double> val, partials, dout;
    op.alloc(ni);
    arg.alloc(ni);
    val.alloc(ni);
    CU(cudaMemcpyAsync(op.p, pack.op.data(), ni * sizeof(int), cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(arg.p, pack.arg.data(), ni * sizeof(int), cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(val.p, pack.val.data(), ni * sizeof(double), cudaMemcpyHostToDevice, s));
    a.op = op.p;
    a.arg = arg.p;
    a.val = val.p;
    a.u = du;
    a.w = dw;
    a.V = dV;
    // Gauss-3 rule and Q1 shapes, built like grid.cpp:109-119, 142-147
    const double gq = std::sqrt(3.0 / 5.0);
    const double p[3] = {-gq, 0.0, gq}, wt[3] = {5.0 / 9.0, 8.0 / 9.0, 5.0 / 9.0};
    for (int j = 0; j < 3; ++j)
        for (int i = 0; i < 3; ++i) {
            const int q = j * 3 + i;
            const double S = p[i], T = p[j];
            a.S[q] = S;
            a.T[q] = T;
            a.W[q] = wt[i] * wt[j];
            a.N[q][0] = 0.25 * (1.0 - S) * (1.0 - T);
            a.N[q][1] = 0.25 * (1.0 + S) * (1.0 - T);
            a.N[q][2] = 0.25 * (1.0 + S) * (1.0 + T);
            a.N[q][3] = 0.25 * (1.0 - S) * (1.0 + T);
            a.dN[q][0][0] = -0.25 * (1.0 - T);
            a.dN[q][0][1] = -0.25 * (1.0 - S);
            a.dN[q][1][0] = 0.25 * (1.0 - T);
            a.dN[q][1][1] = -0.25 * (1.0 + S);
            a.dN[q][2][0] = 0.25 * (1.0 + T);
            a.dN[q][2][1] = 0.25 * (1.0 + S);
            a.dN[q][3][0] = -0.25 * (1.0 + T);
            a.dN[q][3][1] = 0.25 * (1.0 - S);
        }
    if (error_norms_smem(micro) > 232448) return fail(TS_ERR_INVALID, "micro grid too large for error_norms");
    partials.alloc((size_t)6 * macro.cells());
    dout.alloc(4);
    const bool compiled = launch_error_norms_jit(a, tapes, partials.p, s);  // tapes as code (jit.cu)
    launch_error_norms(a, partials.p, dout.p, s, !compiled);
    CU(cudaGetLastError());
    CU(cudaMemcpyAsync(out, dout.p, 4 * sizeof(double), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    return TS_OK;
}

}  // namespace

extern "C" {

int32_t ts_error_norms(const ts_grid_desc* macro, const ts_grid_desc* micro, const ts_tape* tapes,
                       const double* u, const double* w, const double* V, double* out) {
    if (!macro || !micro || !tapes || !u || !w || !V || !out) return fail(TS_ERR_INVALID, "null argument");
    if (int rc = device_ready()) return rc;
    return guarded([&]() -> int {
        const GridG M = to_grid(*macro), g = to_grid(*micro);
        DBuf<double> du, dw, dV;
        du.alloc(M.nodes());
        dw.alloc(M.nodes());
        dV.alloc((size_t)M.nodes() * g.nodes());
        CU(cudaMemcpy(du.p, u, du.bytes(), cudaMemcpyHostToDevice));
        CU(cudaMemcpy(dw.p, w, dw.bytes(), cudaMemcpyHostToDevice));
        CU(cudaMemcpy(dV.p, V, dV.bytes(), cudaMemcpyHostToDevice));
        return error_norms_impl(M, g, tapes, du.p, dw.p, dV.p, out, 0);
    });
}

const char* ts_jit_status(void) {
    static thread_local std::string s;
    s = jit_status();
    return s.c_str();
}

int32_t ts_ctx_error_norms(ts_ctx* c, const ts_tape* tapes, double* out) {
    if (!c || !tapes || !out) return fail(TS_ERR_INVALID, "null argument");
    if (c->gen) return fail(TS_ERR_INVALID, "error_norms is defined for 2D Q1 micro grids");
    return guarded([&]() -> int {
        return error_norms_impl(c->P.macro, c->P.micro, tapes, c->uw.p, c->uw.p + c->nM, c->V.p, out, c->stream);
    });
}

}  // extern "C"

// ---- micro-state egress (host formatter in host/vtk.cpp) ----

namespace {

template <class F>
int io_guarded(F&& f) {
    return guarded([&]() -> int {
        try {
            return f();
        } catch (const std::runtime_error& e) {
            return fail(TS_ERR_IO, "%s", e.what());
        }
    });
}

int check_vtk_args(const ts_ctx* c, int32_t format, const char* path) {
    if (!c || !path) return fail(TS_ERR_INVALID, "null argument");
    if (format != TS_VTK_ASCII && format != TS_VTK_BINARY) return fail(TS_ERR_INVALID, "unknown VTK format %d", format);
    if (!c->state_valid) return fail(TS_ERR_INVALID, "no device state: run ts_fixed_point_solve first");
    return TS_OK;
}

}  // namespace

extern "C" {

int32_t ts_write_vtk_macro(ts_ctx* c, int32_t format, const char* path) {
    if (int rc = check_vtk_args(c, format, path)) return rc;
    return io_guarded([&]() -> int {
        const int nM = c->nM;
        std::vector<double> uw(2 * (size_t)nM), xy(2 * (size_t)nM);
        CU(cudaMemcpyAsync(uw.data(), c->uw.p, uw.size() * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        for (int i = 0; i < nM; ++i) node_xy(c->P.macro, i, xy[2 * i], xy[2 * i + 1]);  // grid.cpp:47-52
        tsb::vtk::write_macro(c->P.macro.n0, c->P.macro.n1, xy.data(), {{"u", uw.data()}, {"w", uw.data() + nM}},
                              format == TS_VTK_BINARY ? tsb::vtk::BINARY : tsb::vtk::ASCII, path);
        return TS_OK;
    });
}

int32_t ts_write_vtk_micro(ts_ctx* c, double scale, int32_t format, const char* path) {
    if (int rc = check_vtk_args(c, format, path)) return rc;
    if (c->P.map.kind == TS_MAP_TAPE && !c->has_zeta)
        return fail(TS_ERR_INVALID, "TAPE map without desc.zeta: the pushforward needs zeta itself");
    return io_guarded([&]() -> int {
        const bool bin = format == TS_VTK_BINARY;
        PushG g{};
        g.kind = c->P.map.kind;
        g.op = c->t_op.p;
        g.arg = c->t_arg.p;
        g.val = c->t_val.p;
        g.zeta[0] = c->zeta[0];
        g.zeta[1] = c->zeta[1];
        g.s_kind = c->P.map.s_kind;
        g.amp = c->P.map.amp;
        g.macro = c->P.macro;
        g.scale = scale;
        tsb::vtk::MicroSource src;
        src.n_macro = c->nM;
        if (c->gen) {
            const GenGeom& G = c->GP.g;
            g.table = c->GP.map.table;
            g.tstride = c->GP.map.tstride;
            g.dim = G.d;
            for (int a = 0; a < 3; ++a) {
                g.nn[a] = G.nn[a];
                g.lo[a] = G.lo[a];
                g.hp[a] = G.hp[a];
            }
        } else {
            g.table = c->A_table.p;
            g.tstride = 4;
            g.dim = 2;
            g.nn[0] = c->P.micro.nx();
            g.nn[1] = c->P.micro.ny();
            g.nn[2] = 1;
            g.lo[0] = c->P.micro.lo0;
            g.lo[1] = c->P.micro.lo1;
            g.hp[0] = c->P.micro.h0;
            g.hp[1] = c->P.micro.h1;
        }
        src.lat.dim = g.dim;
        for (int a = 0; a < 3; ++a) src.lat.nn[a] = g.nn[a];
        const long long np = src.lat.nodes();
        if (np != c->nm) return fail(TS_ERR_INVALID, "micro lattice does not match the state");
        src.chunk_nodes = (int)std::min<long long>(c->nM, std::max<long long>(1, (1ll << 20) / np));  // ~1M points
        const size_t cap = (size_t)src.chunk_nodes * np;
        const int pdim = bin || g.dim == 3 ? 3 : 2;
        DBuf<double> dbuf;
        dbuf.alloc(pdim * cap);
        if (c->h_stage_bytes < pdim * cap * sizeof(double)) {
            for (double*& p : c->h_stage) {
                if (p) cudaFreeHost(p);
                p = nullptr;
            }
            c->h_stage_bytes = 0;
            for (double*& p : c->h_stage) CU(cudaMallocHost(&p, pdim * cap * sizeof(double)));
            c->h_stage_bytes = pdim * cap * sizeof(double);
        }
        double* const* host = c->h_stage;
        cudaEvent_t ev[2] = {nullptr, nullptr};
        struct Cleanup {
            cudaEvent_t* e;
            ~Cleanup() {
                for (int k = 0; k < 2; ++k)
                    if (e[k]) cudaEventSynchronize(e[k]), cudaEventDestroy(e[k]);
            }
        } cleanup{ev};
        for (int k = 0; k < 2; ++k) CU(cudaEventCreateWithFlags(&ev[k], cudaEventDisableTiming));
        reset_flags(c);
        src.start = [&](int chunk, int slot, int what) {
            const int first = chunk * src.chunk_nodes;
            const int cnt = (int)std::min<long long>(c->nM - first, src.chunk_nodes);
            const size_t n = (size_t)cnt * np;
            if (what == 0) {
                launch_vtk_points(g, first, cnt, bin, dbuf.p, c->err.p, c->stream);
                CU(cudaGetLastError());
                CU(cudaMemcpyAsync(host[slot], dbuf.p, pdim * n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            } else if (bin) {
                launch_vtk_swap(c->V.p + (size_t)first * np, n, dbuf.p, c->stream);
                CU(cudaGetLastError());
                CU(cudaMemcpyAsync(host[slot], dbuf.p, n * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
            } else {
                CU(cudaMemcpyAsync(host[slot], c->V.p + (size_t)first * np, n * sizeof(double),
                                   cudaMemcpyDeviceToHost, c->stream));
            }
            CU(cudaEventRecord(ev[slot], c->stream));
        };
        src.wait = [&](int slot) -> const double* {
            CU(cudaEventSynchronize(ev[slot]));
            return host[slot];
        };
        tsb::vtk::write_micro(src, bin ? tsb::vtk::BINARY : tsb::vtk::ASCII, path);
        unsigned err = 0;
        CU(cudaMemcpyAsync(&err, c->err.p, sizeof err, cudaMemcpyDeviceToHost, c->stream));
        c->sync();
        if (err) return fail(TS_ERR_EXPR, "%s", expr_error(err));
        return TS_OK;
    });
}

}  // extern "C"
