// Micro-state egress: the reference's write_vtk_macro /
// write_vtk_micro (proj/src/vtk.cpp:36-85) fed straight from the device state.
//
// Device side (egress.cu): one kernel pushes every micro patch forward through
// zeta(x_i, .) (vtk.cpp:64-67) in chunks of macro nodes, writing either native
// (x, y[, z]) doubles for the ASCII formatter or big-endian (x, y, z) triples that
// go to the file unchanged (legacy BINARY); a second kernel byte-swaps V chunks.
// Host side (host/vtk.cpp): a parallel, ordered formatter that writes the
// reference's byte layout (std::to_chars general/16 == ostream precision 16).
#pragma once

#include <cstddef>

#include "device_common.cuh"

namespace tsb {

// zeta evaluation for the pushforward, all map families of the context.
struct PushG {
    int kind;             // TS_MAP_*
    const int* op;
    const int* arg;
    const double* val;
    TapeRef zeta[2];      // TAPE maps
    const double* table;  // table maps: row per macro node
    int tstride, s_kind;
    double amp;
    GridG macro;
    int dim;              // micro dimension (2 / 3)
    int nn[3];            // node lattice of one patch
    double lo[3], hp[3];  // lattice coordinates lo + i * hp
    double scale;
};

void launch_vtk_points(const PushG& g, int first_node, int n_nodes, int big_endian, double* out,
                       unsigned* err, cudaStream_t s);
void launch_vtk_swap(const double* in, size_t n, double* out, cudaStream_t s);

}  // namespace tsb
