// Macro u/w solves on a thread-block cluster (solver.cpp:76-82, Jacobi-PCG of
// linalg.cpp:103-161 on the eliminated macro systems) for macro grids too large for one
// SM's shared memory (config 3: 129 x 129 nodes).  One cluster of CL CTAs per system;
// CTA `rank` owns a band of grid rows: the 9 stencil planes of its rows (k_csr_to_stencil
// output, CSR column order) and its slice of p live in SMEM, x/r/D^-1/Ap in registers.
// Per PCG iteration three cluster barriers: two dot-product exchanges (each CTA writes
// its block total into every peer's slot over DSMEM, then all sum the CL slots in rank
// order: identical bits everywhere) and the p halo rows (written straight into the
// neighbours' SMEM).  This replaces the grid-wide cooperative CSR CG (k_csr_pcg_coop),
// whose two grid.sync() per iteration cost ~4 us against ~1 us here.
#include <cooperative_groups.h>

#include <cstdlib>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace tsb {

namespace {

constexpr int kMcThreads = 512;
constexpr int kMcSlots = 3;

struct McGeom {
    int nx, ny, rp, planes_doubles, p_doubles;
};

__host__ __device__ __forceinline__ McGeom mc_geom(const GridG& g, int CL) {
    McGeom m;
    m.nx = g.n0 + 1;
    m.ny = g.n1 + 1;
    m.rp = (m.ny + CL - 1) / CL;
    m.planes_doubles = 9 * m.rp * m.nx;
    // p: halo row above, rp own rows, halo row below, one margin double at each end (a
    // neighbour column that wraps into the next row carries a zero coefficient)
    m.p_doubles = (m.rp + 2) * m.nx + 2;
    return m;
}

__host__ __device__ __forceinline__ size_t mc_smem_bytes(const GridG& g, int CL) {
    const McGeom m = mc_geom(g, CL);
    return ((size_t)m.planes_doubles + m.p_doubles + (m.p_doubles & 1) + kMcSlots * 32 * 4 +
            kMcSlots * 16 * 4) * sizeof(double);
}

// Block total of K values in every thread (warp DMMA sums + one SMEM exchange).
template <int K>
__device__ __forceinline__ void mc_block_sum(double (&v)[K], double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = warp_sum_tc(v[k]);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) red[k * 32 + warp] = v[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = warp_sum_tc(lane < nw ? red[k * 32 + lane] : 0.0);
}

// Cluster total: block totals exchanged over DSMEM, summed in rank order by every CTA.
template <int K>
__device__ __forceinline__ void mc_cluster_sum(double (&v)[K], double* red, double* xch, cg::cluster_group& cl,
                                               int CL) {
    mc_block_sum<K>(v, red);
    const int rank = (int)cl.block_rank();
    if ((int)threadIdx.x < CL) {  // thread q writes this CTA's totals into CTA q's slot `rank`
        double* dst = cl.map_shared_rank(xch, threadIdx.x);
#pragma unroll
        for (int k = 0; k < K; ++k) dst[rank * 4 + k] = v[k];
    }
    cl.sync();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double s = 0.0;
        for (int q = 0; q < CL; ++q) s += xch[q * 4 + k];
        v[k] = s;
    }
}

template <int KM>
__global__ void __launch_bounds__(kMcThreads, 1) k_macro_cluster(const MicroPcgArgs a, int CL) {
    extern __shared__ double smem[];
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const int sys = blockIdx.x / CL;
    const McGeom G = mc_geom(a.micro, CL);
    const int nx = G.nx, n = nx * G.ny;
    const int r0 = rank * G.rp, r1 = min(G.ny, r0 + G.rp), nloc = max(0, r1 - r0) * nx;
    double* sA = smem;                                   // [9][rp * nx]
    double* sP = sA + G.planes_doubles;                  // p with halo rows
    double* red = sP + G.p_doubles + (G.p_doubles & 1);  // block reduction slots
    double* xch = red + kMcSlots * 32 * 4;               // cluster exchange slots [3][16][4]
    const int tid = threadIdx.x;
    const int pbase = 1 + nx;  // p index of local node 0 (first own row)

    const double* st = a.stencil + (size_t)sys * a.stencil_stride;
    const double* b = a.fixed + (size_t)sys * n;
    double* xg = a.V + (size_t)sys * n;

    for (int k = tid; k < G.p_doubles; k += blockDim.x) sP[k] = 0.0;
    for (int d = 0; d < 9; ++d)
        for (int k = tid; k < nloc; k += blockDim.x) sA[d * G.rp * nx + k] = st[(size_t)d * n + r0 * nx + k];

    double x[KM], r[KM], dinv[KM], ap[KM];
#pragma unroll
    for (int j = 0; j < KM; ++j) {
        const int k = tid + j * kMcThreads;
        x[j] = r[j] = ap[j] = 0.0;
        dinv[j] = 1.0;
        if (k < nloc) {
            const double dg = sA[4 * G.rp * nx + k];
            dinv[j] = dg != 0.0 ? 1.0 / dg : 1.0;  // linalg.cpp:116-117
            r[j] = b[r0 * nx + k];
            x[j] = a.warm ? xg[r0 * nx + k] : 0.0;
        }
    }
    // own p values into SMEM and the boundary rows into the neighbours' halo rows
    auto publish = [&](const double (&v)[KM]) {
        double* up = rank > 0 ? cl.map_shared_rank(sP, rank - 1) : nullptr;        // its bottom halo
        double* down = rank < CL - 1 ? cl.map_shared_rank(sP, rank + 1) : nullptr;  // its top halo
#pragma unroll
        for (int j = 0; j < KM; ++j) {
            const int k = tid + j * kMcThreads;
            if (k >= nloc) continue;
            sP[pbase + k] = v[j];
            if (up && k < nx) up[1 + (G.rp + 1) * nx + k] = v[j];
            if (down && k >= nloc - nx) down[1 + (k - (nloc - nx))] = v[j];
        }
        cl.sync();
    };
    // y = A v over the own nodes (CSR column order: dy outer, dx inner)
    auto spmv = [&](int j) {
        const int k = tid + j * kMcThreads;
        double y = 0.0;
#pragma unroll
        for (int d = 0; d < 9; ++d) {
            const int off = (d / 3 - 1) * nx + (d % 3 - 1);
            y = fma(sA[d * G.rp * nx + k], sP[pbase + k + off], y);
        }
        return y;
    };

    int slot = 0;  // rotating reduction / exchange slots (a slot is reused 3 barriers later)
    auto csum = [&](auto& v) {
        mc_cluster_sum(v, red + slot * 128, xch + slot * 64, cl, CL);
        slot = slot == kMcSlots - 1 ? 0 : slot + 1;
    };

    // Every CTA of the cluster has started and zero-filled its p halo before any peer
    // writes into it over DSMEM (the first publish stores the warm start's boundary rows).
    cl.sync();
    publish(x);
    double s3[3] = {0.0, 0.0, 0.0};  // b.b, r.z, r.r with r = b - A x0 (linalg.cpp:108-129)
#pragma unroll
    for (int j = 0; j < KM; ++j) {
        if (tid + j * kMcThreads >= nloc) continue;
        const double bk = r[j];
        s3[0] = fma(bk, bk, s3[0]);
        r[j] = bk - spmv(j);
        ap[j] = dinv[j] * r[j];
        s3[1] = fma(r[j], ap[j], s3[1]);
        s3[2] = fma(r[j], r[j], s3[2]);
    }
    csum(s3);
    const double bnorm = sqrt(s3[0]);
    int status = 0, iters = 0;
    double rel = 0.0;
    if (bnorm == 0.0) {  // linalg.cpp:110-114
#pragma unroll
        for (int j = 0; j < KM; ++j) x[j] = 0.0;
    } else {
        double rz = s3[1];
        rel = sqrt(s3[2]) / bnorm;
        if (rel > a.tol) {
            const double thr = rel_threshold(bnorm, a.tol);  // rr <= thr <=> sqrt(rr) / bnorm <= tol
            double rr_last = s3[2];
            double p[KM];
#pragma unroll
            for (int j = 0; j < KM; ++j) p[j] = ap[j];  // p0 = z0
            publish(p);
            status = 2;
            for (int it = 1; it <= a.maxit; ++it) {
                double t1[1] = {0.0};
#pragma unroll
                for (int j = 0; j < KM; ++j) {
                    if (tid + j * kMcThreads >= nloc) continue;
                    ap[j] = spmv(j);
                    t1[0] = fma(p[j], ap[j], t1[0]);
                }
                const double yrz = div_recip(rz);
                csum(t1);
                iters = it;
                if (t1[0] <= 0.0) {  // linalg.cpp:138-142
                    status = 1;
                    break;
                }
                const double alpha = rz / t1[0];
                double t2[2] = {0.0, 0.0};
#pragma unroll
                for (int j = 0; j < KM; ++j) {
                    x[j] = fma(alpha, p[j], x[j]);
                    r[j] = fma(-alpha, ap[j], r[j]);
                    t2[0] = fma(r[j], r[j], t2[0]);
                    ap[j] = dinv[j] * r[j];  // z
                    t2[1] = fma(r[j], ap[j], t2[1]);
                }
                csum(t2);
                rr_last = t2[0];
                if (t2[0] <= thr) {
                    status = 0;
                    break;
                }
                const double beta = div_finish(t2[1], rz, yrz);  // == t2[1] / rz bitwise
                rz = t2[1];
#pragma unroll
                for (int j = 0; j < KM; ++j) p[j] = fma(beta, p[j], ap[j]);
                publish(p);
            }
            rel = sqrt(rr_last) / bnorm;
        }
    }
#pragma unroll
    for (int j = 0; j < KM; ++j) {
        const int k = tid + j * kMcThreads;
        if (k < nloc) xg[r0 * nx + k] = x[j];
    }
    if (rank == 0 && tid == 0) {
        a.iters[sys] = iters;
        a.status[sys] = status;
        a.final_rel[sys] = rel;
    }
}

template <int KM>
int launch_km(const MicroPcgArgs& a, int CL, size_t smem, cudaStream_t s) {
    auto kern = k_macro_cluster<KM>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
    if (CL > 8 && cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess)
        return 0;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(a.n_problems * CL);
    cfg.blockDim = dim3(kMcThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess || nclusters < a.n_problems) {
        cudaGetLastError();
        return 0;
    }
    return cudaLaunchKernelEx(&cfg, kern, a, CL) == cudaSuccess ? 1 : 0;
}

}  // namespace

namespace {
bool mc_fits(const GridG& g, int CL) {
    const McGeom m = mc_geom(g, CL);
    return g.n1 + 1 >= 2 * CL && (m.rp * m.nx + kMcThreads - 1) / kMcThreads <= 8 &&
           mc_smem_bytes(g, CL) <= 232448;
}
}  // namespace

// Largest cluster (16 where the device allows non-portable sizes, else 8) whose row bands
// fit SMEM; TS_MACRO_CLUSTER=0 disables, =8/16 forces a size.
int macro_cluster_size(const GridG& g) {
    int want = 16;
    if (const char* e = std::getenv("TS_MACRO_CLUSTER")) {
        want = std::atoi(e);
        if (want <= 0) return 0;
    }
    for (int CL : {16, 8})
        if (CL <= want && mc_fits(g, CL)) return CL;
    return 0;
}

int launch_macro_cluster_cl(const MicroPcgArgs& a, int CL, cudaStream_t s) {
    if (CL <= 0) return 0;
    const McGeom m = mc_geom(a.micro, CL);
    const size_t smem = mc_smem_bytes(a.micro, CL);
    switch ((m.rp * m.nx + kMcThreads - 1) / kMcThreads) {
        case 1: return launch_km<1>(a, CL, smem, s);
        case 2: return launch_km<2>(a, CL, smem, s);
        case 3: return launch_km<3>(a, CL, smem, s);
        case 4: return launch_km<4>(a, CL, smem, s);
        case 5: return launch_km<5>(a, CL, smem, s);
        case 6: return launch_km<6>(a, CL, smem, s);
        case 7: return launch_km<7>(a, CL, smem, s);
        case 8: return launch_km<8>(a, CL, smem, s);
    }
    return 0;
}

// Launch with cluster size CL, or the next smaller one that fits and launches; returns the
// size used (0: none).
int launch_macro_cluster(const MicroPcgArgs& a, int CL, cudaStream_t s) {
    for (int c : {16, 8})
        if (c <= CL && mc_fits(a.micro, c) && launch_macro_cluster_cl(a, c, s)) return c;
    return 0;
}

}  // namespace tsb
