// Legacy VTK writers — drop-in for proj/src/vtk.cpp (write_vtk_macro, vtk.cpp:36-54;
// write_vtk_micro, vtk.cpp:56-85) plus the streaming engine behind the C ABI's
// ts_write_vtk_macro / ts_write_vtk_micro.
//
// Byte layout: the reference streams through std::ofstream with precision(16) in the
// default float format, i.e. printf "%.16g"; std::to_chars(general, 16) produces the
// identical characters (checked in tests/test_vtk.py against the reference writer)
// at ~3x the speed, and lines are formatted by all host threads into per-thread
// buffers that a writer thread appends in order, so the file is identical to a
// serial run.  The micro dataset arrives in chunks of macro nodes (MicroSource): the
// next chunk is produced (device kernel + D2H into pinned memory, or host map
// evaluation for the C++ mirror) while the current one is formatted.
#include "twoscale/vtk.hpp"

#include <algorithm>
#include <charconv>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <deque>
#include <mutex>
#include <stdexcept>
#include <thread>

#include "../internal.h"
#include "../vtk_stream.h"
#include "twoscale/config.hpp"

namespace tsb::vtk {

int threads() {
    if (const char* e = std::getenv("TS_VTK_THREADS")) {
        const int n = std::atoi(e);
        if (n > 0) return n;
    }
    const unsigned h = std::thread::hardware_concurrency();
    return h ? static_cast<int>(h) : 1;
}

namespace {

// Ordered output with one background writer; the producer blocks when more than
// kMaxQueued bytes are waiting.
class Sink {
public:
    explicit Sink(const std::string& path) : path_(path) {
        f_ = std::fopen(path.c_str(), "wb");
        if (!f_) throw std::runtime_error("cannot write '" + path + "'");
        th_ = std::thread([this] { run(); });
    }
    ~Sink() {
        if (th_.joinable()) {
            {
                std::lock_guard<std::mutex> g(m_);
                done_ = true;
            }
            cv_.notify_all();
            th_.join();
        }
        if (f_) std::fclose(f_);
    }
    void text(const std::string& s) { push(std::vector<char>(s.begin(), s.end())); }
    // Large raw block written from the caller's buffer once the queue has drained (no copy).
    void raw(const void* p, size_t n) {
        std::unique_lock<std::mutex> g(m_);
        space_.wait(g, [&] { return queued_ == 0 || failed_; });
        if (failed_ || std::fwrite(p, 1, n, f_) != n) {
            failed_ = true;
            throw std::runtime_error("cannot write '" + path_ + "'");
        }
    }
    void push(std::vector<char>&& b) {
        std::unique_lock<std::mutex> g(m_);
        space_.wait(g, [&] { return queued_ < kMaxQueued || failed_; });
        if (failed_) throw std::runtime_error("cannot write '" + path_ + "'");
        queued_ += b.size();
        q_.push_back(std::move(b));
        cv_.notify_all();
    }
    void close() {
        {
            std::lock_guard<std::mutex> g(m_);
            done_ = true;
        }
        cv_.notify_all();
        th_.join();
        const bool bad = failed_ || std::fflush(f_) != 0;
        const bool bad_close = std::fclose(f_) != 0;
        f_ = nullptr;
        if (bad || bad_close) throw std::runtime_error("cannot write '" + path_ + "'");
    }

private:
    static constexpr size_t kMaxQueued = size_t(1) << 30;
    void run() {
        for (;;) {
            std::vector<char> b;
            {
                std::unique_lock<std::mutex> g(m_);
                cv_.wait(g, [&] { return done_ || !q_.empty(); });
                if (q_.empty()) return;
                b = std::move(q_.front());
                q_.pop_front();
            }
            const bool ok = failed_ || std::fwrite(b.data(), 1, b.size(), f_) == b.size();
            std::lock_guard<std::mutex> g(m_);
            if (!ok) failed_ = true;
            queued_ -= b.size();
            space_.notify_all();
        }
    }
    std::string path_;
    std::FILE* f_ = nullptr;
    std::thread th_;
    std::mutex m_;
    std::condition_variable cv_, space_;
    std::deque<std::vector<char>> q_;
    size_t queued_ = 0;
    bool done_ = false, failed_ = false;
};

inline char* put_d(char* p, double v) { return std::to_chars(p, p + 32, v, std::chars_format::general, 16).ptr; }
inline char* put_i(char* p, long long v) { return std::to_chars(p, p + 24, v).ptr; }
inline char* put_s(char* p, const char* s, size_t n) {
    std::memcpy(p, s, n);
    return p + n;
}

// Lines [0, n) formatted by fn(begin, end, dst) -> new end, at most max_line bytes
// per line, split over all threads in rounds of bounded memory, pushed in order.
template <class Fn>
void emit(Sink& sink, long long n, size_t max_line, Fn fn) {
    const int T = threads();
    const long long per_thread = std::max<long long>(1, std::min<long long>((n + T - 1) / T, (16ll << 20) / (long long)max_line));
    long long done = 0;
    while (done < n) {
        const long long round = std::min<long long>(n - done, per_thread * T);
        const long long slice = (round + T - 1) / T;
        std::vector<std::vector<char>> bufs(T);
        std::vector<std::thread> ws;
        for (int t = 0; t < T; ++t) {
            const long long b = done + t * slice, e = std::min(done + round, b + slice);
            if (b >= e) break;
            ws.emplace_back([&, t, b, e] {
                auto& buf = bufs[t];
                buf.resize(static_cast<size_t>(e - b) * max_line);
                buf.resize(fn(b, e, buf.data()) - buf.data());
            });
        }
        for (auto& w : ws) w.join();
        for (auto& b : bufs)
            if (!b.empty()) sink.push(std::move(b));
        done += round;
    }
}

// Big-endian int32 runs for the BINARY cell sections.
inline void put_be32(char* p, int32_t v) {
    const uint32_t u = static_cast<uint32_t>(v);
    p[0] = static_cast<char>(u >> 24);
    p[1] = static_cast<char>(u >> 16);
    p[2] = static_cast<char>(u >> 8);
    p[3] = static_cast<char>(u);
}
inline void put_be64(char* p, double v) {
    uint64_t u;
    std::memcpy(&u, &v, 8);
    for (int k = 0; k < 8; ++k) p[k] = static_cast<char>(u >> (56 - 8 * k));
}

template <class Fn>
void emit_bin(Sink& sink, long long n, size_t bytes_per, Fn fn) {
    emit(sink, n, bytes_per, [&](long long b, long long e, char* p) {
        for (long long k = b; k < e; ++k) p = fn(k, p);
        return p;
    });
}

void header(Sink& s, const char* title, long long n_points, Format fmt) {
    s.text(std::string("# vtk DataFile Version 3.0\n") + title + "\n" + (fmt == BINARY ? "BINARY" : "ASCII") +
           "\nDATASET UNSTRUCTURED_GRID\nPOINTS " + std::to_string(n_points) + " double\n");
}

// Cell c of a patch lattice, VTK node order; returns node count (4 or 8).
inline int cell_nodes(const Lattice& L, long long c, long long off, long long* nd) {
    const long long nx = L.nn[0], ny = L.nn[1];
    const long long cx = L.nn[0] - 1, cy = L.nn[1] - 1;
    const long long i = c % cx, j = (c / cx) % cy, k = c / (cx * cy);
    const long long n0 = off + k * nx * ny + j * nx + i;
    nd[0] = n0;
    nd[1] = n0 + 1;
    nd[2] = n0 + nx + 1;
    nd[3] = n0 + nx;
    if (L.dim == 2) return 4;
    for (int q = 0; q < 4; ++q) nd[4 + q] = nd[q] + nx * ny;
    return 8;
}

// CELLS / CELL_TYPES sections for n_patches copies of the lattice (vtk.cpp:22-27, 70-80).
void cells(Sink& s, const Lattice& L, long long n_patches, Format fmt) {
    const long long cpp = L.cells(), np = L.nodes(), nc = cpp * n_patches;
    const int npc = L.dim == 2 ? 4 : 8;
    s.text("CELLS " + std::to_string(nc) + " " + std::to_string(nc * (npc + 1)) + "\n");
    if (fmt == ASCII) {
        emit(s, nc, 12 + 21 * (size_t)npc, [&](long long b, long long e, char* p) {
            long long nd[8];
            for (long long c = b; c < e; ++c) {
                const int m = cell_nodes(L, c % cpp, (c / cpp) * np, nd);
                *p++ = m == 4 ? '4' : '8';
                for (int q = 0; q < m; ++q) {
                    *p++ = ' ';
                    p = put_i(p, nd[q]);
                }
                *p++ = '\n';
            }
            return p;
        });
    } else {
        if (np * n_patches > 0x7fffffffLL) throw std::runtime_error("BINARY VTK node index exceeds int32");
        emit_bin(s, nc, 4 * (size_t)(npc + 1), [&](long long c, char* p) {
            long long nd[8];
            const int m = cell_nodes(L, c % cpp, (c / cpp) * np, nd);
            put_be32(p, m);
            for (int q = 0; q < m; ++q) put_be32(p + 4 * (q + 1), static_cast<int32_t>(nd[q]));
            return p + 4 * (m + 1);
        });
        s.text("\n");
    }
    const char* ty = L.dim == 2 ? "9\n" : "12\n";
    s.text("CELL_TYPES " + std::to_string(nc) + "\n");
    if (fmt == ASCII) {
        const size_t tl = std::strlen(ty);
        emit(s, nc, tl, [&](long long b, long long e, char* p) {
            for (long long c = b; c < e; ++c) p = put_s(p, ty, tl);
            return p;
        });
    } else {
        const int32_t t = L.dim == 2 ? 9 : 12;
        emit_bin(s, nc, 4, [&](long long, char* p) {
            put_be32(p, t);
            return p + 4;
        });
        s.text("\n");
    }
}

void scalars_head(Sink& s, const std::string& name) { s.text("SCALARS " + name + " double 1\nLOOKUP_TABLE default\n"); }

// n values: ASCII "%.16g\n" each, or BINARY raw (v already big-endian if pre_swapped).
void values(Sink& s, const double* v, long long n, Format fmt, bool pre_swapped) {
    if (fmt == ASCII) {
        emit(s, n, 26, [&](long long b, long long e, char* p) {
            for (long long k = b; k < e; ++k) {
                p = put_d(p, v[k]);
                *p++ = '\n';
            }
            return p;
        });
    } else if (pre_swapped) {
        s.raw(v, n * sizeof(double));
    } else {
        emit_bin(s, n, 8, [&](long long k, char* p) {
            put_be64(p, v[k]);
            return p + 8;
        });
    }
}

}  // namespace

void write_micro(const MicroSource& src, Format fmt, const std::string& path) {
    const Lattice& L = src.lat;
    const long long np = L.nodes(), n_points = src.n_macro * np;
    const int nchunks = static_cast<int>((src.n_macro + src.chunk_nodes - 1) / src.chunk_nodes);
    const int pdim = fmt == BINARY ? 3 : (L.dim == 3 ? 3 : 2);
    Sink s(path);
    header(s, "micro solutions (pushed forward)", n_points, fmt);
    // pass 1: points (vtk.cpp:62-68); pass 2 (after cells): values (vtk.cpp:81-84)
    for (int pass = 0; pass < 2; ++pass) {
        if (pass == 1) {
            if (fmt == BINARY) s.text("\n");
            cells(s, L, src.n_macro, fmt);
            s.text("POINT_DATA " + std::to_string(n_points) + "\n");
            scalars_head(s, "v");
        }
        if (nchunks > 0) src.start(0, 0, pass);
        for (int c = 0; c < nchunks; ++c) {
            if (c + 1 < nchunks) src.start(c + 1, (c + 1) & 1, pass);
            const double* buf = src.wait(c & 1);
            const double* pos = buf;
            const double* v = buf;
            const long long first = (long long)c * src.chunk_nodes;
            const long long cnt = (std::min<long long>(src.n_macro, first + src.chunk_nodes) - first) * np;
            if (pass == 1) {
                values(s, v, cnt, fmt, true);
            } else if (fmt == BINARY) {
                s.raw(pos, 3 * cnt * sizeof(double));
            } else {
                emit(s, cnt, pdim == 2 ? 2 * 25 + 4 : 3 * 25 + 3, [&](long long b, long long e, char* p) {
                    for (long long k = b; k < e; ++k) {
                        p = put_d(p, pos[pdim * k]);
                        *p++ = ' ';
                        p = put_d(p, pos[pdim * k + 1]);
                        *p++ = ' ';
                        if (pdim == 3) {
                            p = put_d(p, pos[pdim * k + 2]);
                        } else {
                            *p++ = '0';
                        }
                        *p++ = '\n';
                    }
                    return p;
                });
            }
        }
    }
    if (fmt == BINARY) s.text("\n");
    s.close();
}

void write_macro(int n0, int n1, const double* xy, const std::vector<std::pair<std::string, const double*>>& fields,
                 Format fmt, const std::string& path) {
    const long long nn = (long long)(n0 + 1) * (n1 + 1);
    Sink s(path);
    header(s, "macro solution", nn, fmt);
    if (fmt == ASCII) {
        emit(s, nn, 2 * 25 + 4, [&](long long b, long long e, char* p) {
            for (long long k = b; k < e; ++k) {
                p = put_d(p, xy[2 * k]);
                *p++ = ' ';
                p = put_d(p, xy[2 * k + 1]);
                p = put_s(p, " 0\n", 3);
            }
            return p;
        });
    } else {
        emit_bin(s, nn, 24, [&](long long k, char* p) {
            put_be64(p, xy[2 * k]);
            put_be64(p + 8, xy[2 * k + 1]);
            put_be64(p + 16, 0.0);
            return p + 24;
        });
        s.text("\n");
    }
    Lattice L;
    L.dim = 2;
    L.nn[0] = n0 + 1;
    L.nn[1] = n1 + 1;
    cells(s, L, 1, fmt);
    s.text("POINT_DATA " + std::to_string(nn) + "\n");
    for (const auto& [name, v] : fields) {
        scalars_head(s, name);
        values(s, v, nn, fmt, false);
        if (fmt == BINARY) s.text("\n");
    }
    s.close();
}

}  // namespace tsb::vtk

namespace twoscale {

void write_vtk_macro(const Grid& grid, const std::vector<std::pair<std::string, const std::vector<double>*>>& fields,
                     const std::string& path) {
    for (const auto& [name, values] : fields)  // vtk.cpp:39-41
        if (static_cast<int>(values->size()) != grid.node_count())
            throw std::runtime_error("field '" + name + "' does not match the node count");
    std::vector<double> xy(2 * static_cast<size_t>(grid.node_count()));
    for (int i = 0; i < grid.node_count(); ++i) {
        const Vec2 p = grid.node(i);
        xy[2 * i] = p.x;
        xy[2 * i + 1] = p.y;
    }
    std::vector<std::pair<std::string, const double*>> f;
    for (const auto& [name, values] : fields) f.emplace_back(name, values->data());
    tsb::vtk::write_macro(grid.n0(), grid.n1(), xy.data(), f, tsb::vtk::ASCII, path);
}

void write_vtk_micro(const MicroField& V, const Grid& macro, const Grid& micro, const CompiledDiffeo& map,
                     double scale, const std::string& path) {
    const int n_patch = micro.node_count();
    tsb::vtk::MicroSource src;
    src.n_macro = macro.node_count();
    src.lat.dim = 2;
    src.lat.nn[0] = micro.n0() + 1;
    src.lat.nn[1] = micro.n1() + 1;
    src.chunk_nodes = std::max(1, (1 << 21) / std::max(1, n_patch));
    std::vector<double> buf[2];
    src.start = [&](int chunk, int slot, int what) {
        const int first = chunk * src.chunk_nodes;
        const int cnt = std::min<int>(macro.node_count() - first, src.chunk_nodes);
        auto& B = buf[slot];
        B.resize((what == 0 ? 2 : 1) * static_cast<size_t>(cnt) * n_patch);
        const int T = tsb::vtk::threads();
        std::vector<std::thread> ws;
        for (int t = 0; t < T; ++t)
            ws.emplace_back([&, t] {
                for (int i = t; i < cnt; i += T) {
                    const size_t k0 = static_cast<size_t>(i) * n_patch;
                    if (what == 1) {  // vtk.cpp:81-84
                        const auto& row = V.at(first + i);
                        for (int j = 0; j < n_patch; ++j) B[k0 + j] = row.at(j);
                        continue;
                    }
                    const Vec2 x = macro.node(first + i);  // vtk.cpp:62-68
                    for (int j = 0; j < n_patch; ++j) {
                        const Vec2 y = map.map(x, micro.node(j));
                        B[2 * (k0 + j)] = x.x + scale * y.x;
                        B[2 * (k0 + j) + 1] = x.y + scale * y.y;
                    }
                }
            });
        for (auto& w : ws) w.join();
    };
    src.wait = [&](int slot) -> const double* { return buf[slot].data(); };
    tsb::vtk::write_micro(src, tsb::vtk::ASCII, path);
}

void write_vtk_macro(const AssemblyContext& ctx, const std::string& path, bool binary) {
    throw_status(ts_write_vtk_macro(ctx.handle(), binary ? TS_VTK_BINARY : TS_VTK_ASCII, path.c_str()));
}

void write_vtk_micro(const AssemblyContext& ctx, double scale, const std::string& path, bool binary) {
    throw_status(ts_write_vtk_micro(ctx.handle(), scale, binary ? TS_VTK_BINARY : TS_VTK_ASCII, path.c_str()));
}

}  // namespace twoscale

extern "C" int32_t ts_write_vtk_ini(const char* ini_text, const double* u, const double* w, const double* V,
                                   double scale, const char* macro_path, const char* micro_path) {
    using namespace twoscale;
    if (!ini_text || (macro_path && (!u || !w)) || (micro_path && !V))
        return ts_set_error_for_front_end(TS_ERR_INVALID, "null argument");
    try {
        const ProblemSetup setup = make_problem(parse_config(ini_text));
        const int nM = setup.macro.node_count(), nm = setup.micro.node_count();
        if (macro_path) {
            const std::vector<double> uu(u, u + nM), ww(w, w + nM);
            write_vtk_macro(setup.macro, {{"u", &uu}, {"w", &ww}}, macro_path);
        }
        if (micro_path) {
            MicroField F(nM);
            for (int i = 0; i < nM; ++i) F[i].assign(V + static_cast<size_t>(i) * nm, V + static_cast<size_t>(i + 1) * nm);
            const CompiledDiffeo map(setup.data.diffeo, setup.data.params);
            write_vtk_micro(F, setup.macro, setup.micro, map, scale, micro_path);
        }
        return TS_OK;
    } catch (const ConfigError& e) {
        return ts_set_error_for_front_end(TS_ERR_CONFIG, e.what());
    } catch (const EvalError& e) {
        return ts_set_error_for_front_end(TS_ERR_EXPR, e.what());
    } catch (const ParseError& e) {
        return ts_set_error_for_front_end(TS_ERR_EXPR, e.what());
    } catch (const std::runtime_error& e) {
        return ts_set_error_for_front_end(TS_ERR_IO, e.what());
    } catch (const std::exception& e) {
        return ts_set_error_for_front_end(TS_ERR_INVALID, e.what());
    }
}
