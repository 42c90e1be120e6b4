// Host half of the micro-state egress (see egress.h): the parallel ordered VTK
// formatter shared by the C++ mirror (include/twoscale/vtk.hpp) and the C ABI.
// Plain C++ (no CUDA types) so host/*.cpp can include it.
#pragma once

#include <functional>
#include <string>
#include <utility>
#include <vector>

namespace tsb::vtk {

enum Format { ASCII = 0, BINARY = 1 };

// One patch's node lattice (nn[2] = 1 in 2D); cells are the lattice cells, written as
// VTK quads (9) in 2D with the reference's node order (grid.cpp:45-48) and as
// hexahedra (12) in 3D.
struct Lattice {
    int dim = 2;
    int nn[3] = {1, 1, 1};
    long long nodes() const { return (long long)nn[0] * nn[1] * nn[2]; }
    long long cells() const {
        return dim == 2 ? (long long)(nn[0] - 1) * (nn[1] - 1) : (long long)(nn[0] - 1) * (nn[1] - 1) * (nn[2] - 1);
    }
};

// Chunked source of the micro dataset.  start(c, slot, what) enqueues chunk c (macro
// nodes [c*chunk_nodes, ...)) of the points (what 0) or the micro values (what 1) into
// host buffer slot 0/1; wait(slot) blocks until it is on the host and returns it.
// Points: 2 (2D ASCII), 3 (3D ASCII) or 3 big-endian (BINARY) doubles per point;
// values: native (ASCII) or big-endian (BINARY) doubles.
struct MicroSource {
    long long n_macro = 0;
    Lattice lat;
    int chunk_nodes = 1;
    std::function<void(int chunk, int slot, int what)> start;
    std::function<const double*(int slot)> wait;
};

// Throws std::runtime_error("cannot write '<path>'") like vtk.cpp:11-15.
void write_micro(const MicroSource& src, Format fmt, const std::string& path);
void write_macro(int n0, int n1, const double* xy, const std::vector<std::pair<std::string, const double*>>& fields,
                 Format fmt, const std::string& path);
int threads();

}  // namespace tsb::vtk
