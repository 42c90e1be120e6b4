// Generic batched Jacobi-PCG (configs 4 and 5).  The Q2 (25-direction) and 3D Q1
// (27-direction) operators of one micro problem are 0.8-1.1 MB, too large for SMEM,
// so here the coefficient planes stream from HBM/L2 every iteration (coalesced:
// consecutive threads read consecutive nodes of one direction plane) while every
// CG vector of the problem (p with a zero halo, x, r, D^-1, Ap/z) stays in SMEM.
// Same persistent ticket scheduling, reduction scheme and fused prologue/epilogue
// as the SMEM-resident 2D kernel (pcg.cu).
#include <cooperative_groups.h>
#include <cstdio>

#include <cmath>
#include <mutex>
#include <type_traits>
#include <cstdlib>

#include "generic.h"

namespace cg = cooperative_groups;

namespace tsb {

namespace {

__constant__ GenTables cGP;  // this translation unit's copy of the generic tables

constexpr int kThreadsG = 512;  // 128 registers per thread: the direction offset tables stay in registers
constexpr int kMaxK = 10;       // nodes per thread (n <= 5120)
constexpr int kRedStride = 32 * 4;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block sum, identical bits in every thread (warp sums on the FP64 tensor core,
// device_common.cuh warp_sum_tc; k-major warp partials).  One barrier.
template <int K>
__device__ __forceinline__ void block_sum(double (&v)[K], double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = warp_sum_tc(v[k]);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) red[k * 32 + warp] = v[k];
    }
    __syncthreads();
    if (K == 2 && nw <= 16) {  // both second stages in one DMMA pair (as pcg.cu's block_sum)
        const int src = (lane & 15) < nw ? (lane >> 4) * 32 + (lane & 15) : -1;
        const double t = src >= 0 ? red[src] : 0.0;
        double g0, g1, s0, s1;
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};\n"
                     : "=d"(g0), "=d"(g1)
                     : "d"(1.0), "d"(t), "d"(0.0), "d"(0.0));
        const double h = g0 + g1;
        const double bsel = (((lane & 3) < 2) == (((lane >> 2) & 1) == 0)) ? 1.0 : 0.0;
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};\n"
                     : "=d"(s0), "=d"(s1)
                     : "d"(h), "d"(bsel), "d"(0.0), "d"(0.0));
        if (isfinite(s0) && isfinite(s1)) {  // inf * 0 in the selector: redo as two chains
            v[0] = s0;
            v[K - 1] = s1;
            return;
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = warp_sum_tc(lane < nw ? red[k * 32 + lane] : 0.0);
}

struct PadGeom {
    int PN0, PN1, PN2, Lp;
};

__host__ __device__ __forceinline__ PadGeom pad_geom(const GenGeom& g) {
    PadGeom q;
    q.PN0 = g.nn[0] + 2 * g.p;
    q.PN1 = g.nn[1] + 2 * g.p;
    q.PN2 = g.d == 3 ? g.nn[2] + 2 * g.p : 1;
    q.Lp = q.PN0 * q.PN1 * q.PN2;
    return q;
}

// y_k = sum_d a_d(k) p(k + o_d).  The operator is symmetric, so only the centre and
// the upper half of the direction planes are read: a_{-d}(k) = a_d(k - o_d).  That
// halves the distinct bytes a problem streams (config 5: 0.55 of 1.06 MB), which
// keeps the 148 concurrently solved problems' operators L2-resident.  Node indices
// k - o_d that fall outside the lattice are clamped: the matching p entry is the
// zero halo, and wrapped in-range indices carry a zero coefficient for the wrapped
// direction (no neighbour there), so both contribute exactly 0.
template <int ND>
__device__ __forceinline__ double gen_spmv(const double* __restrict__ st, int n, int k, const double* sP, int pk,
                                           const int* off, const int* lin) {
    constexpr int C = (ND - 1) / 2;  // the operator stores planes C .. ND - 1 only (plane d - C)
    double acc = __ldg(st + k) * sP[pk];
#pragma unroll
    for (int d = C + 1; d < ND; ++d) {
        const double* plane = st + (size_t)(d - C) * n;
        int m = k - lin[d];
        m = m < 0 ? 0 : m;
        acc = fma(__ldg(plane + k), sP[pk + off[d]], acc);
        acc = fma(__ldg(plane + m), sP[pk - off[d]], acc);
    }
    return acc;
}

// GLOBAL = false: every CG vector in dynamic SMEM, the thread's nodes precomputed in
// registers (n <= kMaxK * kThreadsG).  GLOBAL = true: the vectors live in a per-block
// global scratch slice (L2-resident), for micro grids beyond SMEM; nodes are visited
// with a block-stride loop.
template <int DIM, int P, bool GLOBAL>
__global__ void __launch_bounds__(kThreadsG, 1) k_gen_pcg(const GenPcgArgs a) {
    constexpr int SPAN = 2 * P + 1;
    constexpr int ND = DIM == 2 ? SPAN * SPAN : SPAN * SPAN * SPAN;
    extern __shared__ double smem[];
    __shared__ double gred[GLOBAL ? 3 * kRedStride : 1];
    __shared__ int gticket[GLOBAL ? 1 : 1];
    const GenGeom& g = a.g;
    const PadGeom pg = pad_geom(g);
    const int n = g.nnodes;
    double* sP = GLOBAL ? a.scratch + (size_t)blockIdx.x * ((size_t)pg.Lp + 4 * (size_t)n) : smem;
    double* sx = sP + pg.Lp;
    double* sr = sx + n;
    double* sd = sr + n;
    double* sz = sd + n;
    double* red = GLOBAL ? gred : sz + n;
    int* sTicket = GLOBAL ? gticket : reinterpret_cast<int*>(red + 3 * kRedStride);
    const int tid = threadIdx.x;

    // padded-p offset and lattice (linear node) offset per direction; uniform across the
    // block, read as SMEM broadcasts
    __shared__ int off[ND], lin[ND];
    if (tid < ND) {
        const int d = tid;
        const int o0 = d % SPAN - P, o1 = (d / SPAN) % SPAN - P, o2 = DIM == 3 ? d / (SPAN * SPAN) - P : 0;
        off[d] = o0 + pg.PN0 * (o1 + pg.PN1 * o2);
        lin[d] = o0 + g.nn[0] * (o1 + g.nn[1] * o2);
    }
    constexpr int KM = GLOBAL ? 1 : kMaxK;
    int kk[KM], pk[KM];
    auto pad_of = [&](int k) {
        int ii[3];
        gen_node_idx(g, k, ii);
        return (ii[0] + P) + pg.PN0 * ((ii[1] + P) + pg.PN1 * (DIM == 3 ? ii[2] + P : 0));
    };
    if (!GLOBAL) {
#pragma unroll
        for (int j = 0; j < KM; ++j) {
            const int k = tid + j * blockDim.x;
            kk[j] = k < n ? k : -1;
            pk[j] = pad_of(k < n ? k : 0);
        }
    }
    // visit this thread's nodes: f(node, padded index)
    auto for_nodes = [&](auto&& f) {
        if (GLOBAL) {
            for (int k = tid; k < n; k += blockDim.x) f(k, pad_of(k));
        } else {
#pragma unroll
            for (int j = 0; j < KM; ++j)
                if (kk[j] >= 0) f(kk[j], pk[j]);
        }
    };
    for (int k = tid; k < pg.Lp; k += blockDim.x) sP[k] = 0.0;

    for (;;) {
        __syncthreads();
        if (tid == 0) *sTicket = atomicAdd(a.counter, 1);
        __syncthreads();
        const int Pb = *sTicket;
        if (Pb >= a.n_problems) break;
        const double* st = a.stencil + (size_t)Pb * a.stencil_stride;
        const double uP = a.u[Pb], wP = a.w[Pb];
        const bool use_u = a.kappa1 != 0.0 && uP != 0.0, use_w = a.kappa3 != 0.0 && wP != 0.0;
        const double cu = a.kappa1 * uP, cw = a.kappa3 * wP;
        const size_t vrow = (size_t)Pb * n;
        for_nodes([&](int k, int pkk) {
            const double dg = __ldg(st + k);  // plane 0 = the centre direction
            sd[k] = dg != 0.0 ? 1.0 / dg : 1.0;
            double bk = 0.0;
            if (use_u) bk = fma(cu, __ldg(a.rin + vrow + k), bk);
            if (use_w) bk = fma(cw, __ldg(a.rout + vrow + k), bk);
            sr[k] = bk;
            const double x0 = a.warm ? a.V[vrow + k] : 0.0;
            sx[k] = x0;
            sP[pkk] = x0;
        });
        __syncthreads();
        double s3[3] = {0.0, 0.0, 0.0};
        for_nodes([&](int k, int pkk) {
            const double y = gen_spmv<ND>(st, n, k, sP, pkk, off, lin);
            const double bk = sr[k];
            s3[0] = fma(bk, bk, s3[0]);
            const double r = bk - y;
            sr[k] = r;
            const double z = sd[k] * r;
            sz[k] = z;
            s3[1] = fma(r, z, s3[1]);
            s3[2] = fma(r, r, s3[2]);
        });
        block_sum<3>(s3, red);
        int slot = 1;
        const double bnorm = sqrt(s3[0]);
        int status = 0, iters = 0;
        double rel = 0.0;
        if (bnorm == 0.0) {
            for_nodes([&](int k, int) { sx[k] = 0.0; });
        } else {
            double rz = s3[1];
            rel = sqrt(s3[2]) / bnorm;
            if (rel > a.tol) {
                const double thr = rel_threshold(bnorm, a.tol);  // rr <= thr <=> sqrt(rr) / bnorm <= tol
                double rr_last = s3[2];
                for_nodes([&](int k, int pkk) { sP[pkk] = sz[k]; });
                __syncthreads();
                status = 2;
                for (int it = 1; it <= a.maxit; ++it) {
                    double t1[1] = {0.0};
                    for_nodes([&](int k, int pkk) {
                        const double y = gen_spmv<ND>(st, n, k, sP, pkk, off, lin);
                        sz[k] = y;
                        t1[0] = fma(sP[pkk], y, t1[0]);
                    });
                    const double yrz = div_recip(rz);  // divisor part of beta = rz_new / rz, overlaps the reduction
                    block_sum<1>(t1, red + slot * kRedStride);
                    slot = slot == 2 ? 0 : slot + 1;
                    iters = it;
                    if (t1[0] <= 0.0) {
                        status = 1;
                        break;
                    }
                    const double alpha = rz / t1[0];
                    double t2[2] = {0.0, 0.0};
                    for_nodes([&](int k, int) {
                        const double r = fma(-alpha, sz[k], sr[k]);
                        sr[k] = r;
                        const double z = sd[k] * r;
                        sz[k] = z;
                        t2[0] = fma(r, r, t2[0]);
                        t2[1] = fma(r, z, t2[1]);
                    });
                    block_sum<2>(t2, red + slot * kRedStride);
                    slot = slot == 2 ? 0 : slot + 1;
                    rr_last = t2[0];
                    const bool done = t2[0] <= thr;
                    const double beta = div_finish(t2[1], rz, yrz);  // == t2[1] / rz bitwise
                    rz = t2[1];
                    for_nodes([&](int k, int pkk) {
                        const double p = sP[pkk];
                        sx[k] = fma(alpha, p, sx[k]);
                        if (!done) sP[pkk] = fma(beta, p, sz[k]);
                    });
                    if (done) {
                        status = 0;
                        break;
                    }
                    __syncthreads();
                }
                rel = sqrt(rr_last) / bnorm;  // the last relative residual, as the loop computed it
            }
        }
        for_nodes([&](int k, int) { a.V[vrow + k] = sx[k]; });
        if (a.epilogue) {
            __syncthreads();
            for_nodes([&](int k, int pkk) { sP[pkk] = sx[k]; });
            __syncthreads();
            double t1[1] = {0.0};
            for_nodes([&](int k, int pkk) {
                const double y = gen_spmv<ND>(st, n, k, sP, pkk, off, lin);
                double bk = 0.0;
                if (use_u) bk = fma(cu, __ldg(a.rin + vrow + k), bk);
                if (use_w) bk = fma(cw, __ldg(a.rout + vrow + k), bk);
                const double rr = bk - y;
                t1[0] = fma(rr, rr, t1[0]);
            });
            block_sum<1>(t1, red + slot * kRedStride);
            const int warp = tid >> 5, lane = tid & 31;
            // one warp per role (a single-warp block does both in turn)
            for (int rw = warp; rw < 2; rw += (int)(blockDim.x >> 5)) {
                const int role = rw == 0 ? TS_GAMMA_I : TS_GAMMA_O;
                const double* len = a.face_len + (size_t)Pb * a.face_len_stride;
                double tot = 0.0;
                for (int f = lane; f < g.nfaces; f += 32) {
                    int axis, side, cc[3], tr[2];
                    gen_face(g, f, axis, side, cc, tr);
                    if (a.role[2 * axis + side] != role) continue;
                    double y[3], sc, nrm[3];
                    gen_face_geom(g, cGP, axis, side, cc, 0, y, sc, nrm);
                    for (int q = 0; q < g.nqf; ++q) {
                        double vq = 0.0;
                        for (int fa = 0; fa < g.npf; ++fa)
                            vq = fma(sx[gen_face_node(g, axis, side, cc, tr, fa)], cGP.Nf[q][fa], vq);
                        tot += cGP.FW[q] * vq * len[(size_t)f * g.nqf + q] * sc;
                    }
                }
                tot = warp_sum(tot);
                if (lane == 0) (rw == 0 ? a.bI : a.bO)[Pb] = tot;
            }
            if (tid == 0) a.res_v[Pb] = sqrt(t1[0]);
        }
        if (tid == 0) {
            a.iters[Pb] = iters;
            a.status[Pb] = status;
            a.final_rel[Pb] = rel;
        }
    }
}

// ------------------------------------- 3D Q1 on a 4-CTA cluster (config 5) --------
// The 27-point operator of one 17^3 problem is 1.06 MB (0.55 MB as centre + upper half),
// beyond one SM; streamed from L2 every iteration (k_gen_pcg) the kernel is bound by
// L2->SM latency and traffic.  Here one problem runs on a cluster of kGcCL CTAs: CTA r owns
// a contiguous range of lattice nodes [k0, k1) (balanced, ~1229 nodes) and holds in SMEM the
// centre + upper-half planes of [k0 - H, k1) (H = largest |node offset| = nx*ny + nx + 1; the
// first H only for the lower-half lookups a_{-d}(k) = a_d(k - o_d)) and p on [k0 - H, k1 + H);
// the operator is read from HBM once per solve.  x, r, D^-1, Ap live in registers.  The p
// halos (H nodes each way) are written into the neighbours' SMEM, and the barrier that
// publishes them is split: arrive, SpMV of the interior nodes (which need no halo), wait,
// SpMV of the rest.  Dot products: block totals written into every peer's slot over DSMEM,
// summed in rank order (identical bits in every CTA).  SpMV in k_gen_pcg's order.
namespace {

constexpr int kGcCL = 4;
constexpr int kGcThreads = 512;
constexpr int kGcSlots = 3;

struct GcGeom {
    int nxy, H, chunk, coef_len, p_len, coef_doubles, p_doubles;
};

__host__ __device__ __forceinline__ GcGeom gc_geom(const GenGeom& g) {
    GcGeom m;
    m.nxy = g.nn[0] * g.nn[1];
    m.H = m.nxy + g.nn[0] + 1;
    m.chunk = (g.nnodes + kGcCL - 1) / kGcCL;
    m.coef_len = m.chunk + m.H;
    m.p_len = m.chunk + 2 * m.H;
    m.coef_doubles = 14 * m.coef_len;
    m.p_doubles = m.p_len + (m.p_len & 1);
    m.coef_doubles += m.coef_doubles & 1;
    return m;
}

__host__ __device__ __forceinline__ size_t gc_smem_bytes(const GenGeom& g) {
    const GcGeom m = gc_geom(g);
    return ((size_t)m.coef_doubles + m.p_doubles + kGcSlots * 32 * 4 + kGcSlots * 16 * 4 + kGcSlots + 2) *
           sizeof(double);
}

__device__ __forceinline__ void gc_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void gc_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory"); }

// mbarrier helpers for the dot-product exchange: each CTA's slot barrier expects one
// remote release-arrive per CTA of the cluster (after that CTA's DSMEM store of its totals);
// waiting is an acquire at cluster scope — no full cluster barrier, no CTA-wide fence.
__device__ __forceinline__ void gc_mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void gc_mbar_arrive_remote(unsigned long long* bar, unsigned cta) {
    const unsigned laddr = (unsigned)__cvta_generic_to_shared(bar);
    unsigned raddr;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(laddr), "r"(cta));
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(raddr) : "memory");
}
// The data behind these barriers is shared memory only (DSMEM stores from the peers), so
// the wait is relaxed and followed by an acquire fence restricted to shared::cluster: the
// cluster-scope acquire of try_wait.acquire.cluster also invalidates L1 (CCTL.IVALL: 16 %
// of the z-column kernel's stall samples in ncu), which shared memory does not need.
__device__ __forceinline__ void gc_mbar_wait(unsigned long long* bar, unsigned parity) {
    const unsigned laddr = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n .reg .pred p;\n GC_WAIT_%=:\n"
        " mbarrier.try_wait.parity.relaxed.cluster.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra GC_WAIT_%=;\n}\n" ::"r"(laddr),
        "r"(parity)
        : "memory");
    asm volatile("fence.acquire.sync_restrict::shared::cluster.cluster;" ::: "memory");
}

template <int K>
__device__ __forceinline__ void gc_cluster_sum(double (&v)[K], double* red, double* xch, unsigned long long* bar,
                                               unsigned parity, cg::cluster_group& cl) {
    block_sum<K>(v, red);
    const int rank = (int)cl.block_rank();
    if ((int)threadIdx.x < kGcCL) {  // thread q: totals into CTA q's slot, then arrive on its barrier
        double* dst = cl.map_shared_rank(xch, threadIdx.x);
#pragma unroll
        for (int k = 0; k < K; ++k) dst[rank * 4 + k] = v[k];
        gc_mbar_arrive_remote(bar, threadIdx.x);
    }
    gc_mbar_wait(bar, parity);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < kGcCL; ++q) s += xch[q * 4 + k];
        v[k] = s;
    }
}

template <int KM>
__global__ void __launch_bounds__(kGcThreads, 1) k_gen_pcg3_cluster(const GenPcgArgs a) {
    extern __shared__ double smem[];
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const GenGeom& g = a.g;
    const GcGeom G = gc_geom(g);
    const int n = g.nnodes, H = G.H;
    const int k0 = rank * G.chunk, k1 = min(n, k0 + G.chunk), nloc = max(0, k1 - k0);
    double* sA = smem;                         // [14][chunk + H], node k at (k - k0 + H)
    double* sP = sA + G.coef_doubles;          // [chunk + 2H], node k at (k - k0 + H)
    double* red = sP + G.p_doubles;
    double* xch = red + kGcSlots * 32 * 4;
    unsigned long long* sBar = reinterpret_cast<unsigned long long*>(xch + kGcSlots * 16 * 4);  // [kGcSlots]
    int* sTicket = reinterpret_cast<int*>(sBar + kGcSlots);  // [current, next]
    const int tid = threadIdx.x;
    if (tid < kGcSlots) gc_mbar_init(sBar + tid, kGcCL);
    if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    unsigned phase = 0;  // parity bit per slot
    int lin[14];
#pragma unroll
    for (int e = 0; e < 14; ++e) {
        const int d = 13 + e;
        lin[e] = (d % 3 - 1) + g.nn[0] * ((d / 3) % 3 - 1) + G.nxy * (d / 9 - 1);
    }
    for (int k = tid; k < G.p_doubles; k += blockDim.x) sP[k] = 0.0;

    auto csum = [&](auto& v, int& slot) {
        gc_cluster_sum(v, red + slot * 128, xch + slot * 64, sBar + slot, (phase >> slot) & 1u, cl);
        phase ^= 1u << slot;
        slot = slot == kGcSlots - 1 ? 0 : slot + 1;
    };
    // own values into p, the first / last H into the neighbours' halos; then a CTA barrier
    // and the cluster arrive — the caller waits (gc_wait) before touching halo nodes
    auto publish = [&](const double (&v)[KM]) {
        double* below = rank > 0 ? cl.map_shared_rank(sP, rank - 1) : nullptr;
        double* above = rank < kGcCL - 1 ? cl.map_shared_rank(sP, rank + 1) : nullptr;
#pragma unroll
        for (int j = 0; j < KM; ++j) {
            const int k = tid + j * kGcThreads;
            if (k >= nloc) continue;
            sP[H + k] = v[j];
            if (below && k < H) below[G.chunk + H + k] = v[j];
            if (above && k >= nloc - H) above[k - nloc + H] = v[j];
        }
        __syncthreads();
        gc_arrive();
    };
    auto spmv = [&](int k) {  // local node k
        const int c = H + k;
        double acc = sA[c] * sP[c];
#pragma unroll
        for (int e = 1; e < 14; ++e) {
            const double* plane = sA + e * G.coef_len;
            acc = fma(plane[c], sP[c + lin[e]], acc);
            acc = fma(plane[c - lin[e]], sP[c - lin[e]], acc);
        }
        return acc;
    };
    auto interior = [&](int k) { return k >= H && k < nloc - H; };

    int slot = 0;
    // All CTAs of the cluster have started (mbarriers initialised, p halos zeroed) before the
    // first remote shared-memory write below.
    cl.sync();
    // Tickets: the cluster holds the next problem's ticket while it solves the current one and
    // prefetches that problem's operator range into L2, so the per-problem load (config 5
    // averages ~60 PCG iterations per solve) comes from L2 instead of HBM.
    if (rank == 0 && tid == 0) {
        const int t = atomicAdd(a.counter, 1);
        for (int q = 0; q < kGcCL; ++q) cl.map_shared_rank(sTicket, q)[1] = t;
    }
    for (;;) {
        if (rank == 0 && tid == 0) {
            const int cur = sTicket[1];
            const int nxt = cur < a.n_problems ? atomicAdd(a.counter, 1) : cur;
            for (int q = 0; q < kGcCL; ++q) {
                int* t = cl.map_shared_rank(sTicket, q);
                t[0] = cur;
                t[1] = nxt;
            }
        }
        cl.sync();
        const int Pb = sTicket[0];
        if (Pb >= a.n_problems) break;
        if (sTicket[1] < a.n_problems && a.stencil_stride) {
            const char* nst = reinterpret_cast<const char*>(a.stencil + (size_t)sTicket[1] * a.stencil_stride);
            const int lo = max(0, k0 - H), bytes = (k1 - lo) * 8;
            const int lines = (bytes + 127) / 128 + 1;
            for (int t = tid; t < 14 * lines; t += blockDim.x) {
                const int e = t / lines, l = t % lines;
                const size_t off = ((size_t)e * n + lo) * 8 + (size_t)l * 128;
                if (off < ((size_t)e * n + k1) * 8)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(nst + off));
            }
        }
        const double* st = a.stencil + (size_t)Pb * a.stencil_stride;
        const double uP = a.u[Pb], wP = a.w[Pb];
        const bool use_u = a.kappa1 != 0.0 && uP != 0.0, use_w = a.kappa3 != 0.0 && wP != 0.0;
        const double cu = a.kappa1 * uP, cw = a.kappa3 * wP;
        const size_t vrow = (size_t)Pb * n;
        for (int e = 0; e < 14; ++e) {
            const double* src = st + (size_t)e * n;
            for (int k = tid; k < nloc + H; k += blockDim.x) {
                const int gk = k0 - H + k;
                sA[e * G.coef_len + k] = gk >= 0 ? __ldg(src + gk) : 0.0;
            }
        }
        double x[KM], r[KM], dv[KM], z[KM];
#pragma unroll
        for (int j = 0; j < KM; ++j) {
            const int k = tid + j * kGcThreads;
            x[j] = r[j] = z[j] = 0.0;
            dv[j] = 1.0;
            if (k < nloc) {
                const double dg = __ldg(st + k0 + k);
                dv[j] = dg != 0.0 ? 1.0 / dg : 1.0;
                double bk = 0.0;
                if (use_u) bk = fma(cu, __ldg(a.rin + vrow + k0 + k), bk);
                if (use_w) bk = fma(cw, __ldg(a.rout + vrow + k0 + k), bk);
                r[j] = bk;
                x[j] = a.warm ? a.V[vrow + k0 + k] : 0.0;
            }
        }
        publish(x);  // (its CTA barrier also completes sA)
        gc_wait();
        double s3[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int j = 0; j < KM; ++j) {
            const int k = tid + j * kGcThreads;
            if (k >= nloc) continue;
            const double bk = r[j];
            s3[0] = fma(bk, bk, s3[0]);
            r[j] = bk - spmv(k);
            z[j] = dv[j] * r[j];
            s3[1] = fma(r[j], z[j], s3[1]);
            s3[2] = fma(r[j], r[j], s3[2]);
        }
        csum(s3, slot);
        const double bnorm = sqrt(s3[0]);
        int status = 0, iters = 0;
        double rel = 0.0;
        if (bnorm == 0.0) {
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
                for (int j = 0; j < KM; ++j) p[j] = z[j];  // p0 = z0
                publish(p);
                bool pending = true;  // a publish's cluster arrive awaits its wait
                status = 2;
                for (int it = 1; it <= a.maxit; ++it) {
                    // interior nodes while the halos are in flight, then the rest
#pragma unroll
                    for (int j = 0; j < KM; ++j) {
                        const int k = tid + j * kGcThreads;
                        if (k < nloc && interior(k)) z[j] = spmv(k);
                    }
                    gc_wait();
                    pending = false;
                    double t1[1] = {0.0};
#pragma unroll
                    for (int j = 0; j < KM; ++j) {
                        const int k = tid + j * kGcThreads;
                        if (k >= nloc) continue;
                        if (!interior(k)) z[j] = spmv(k);  // z holds Ap until the r update
                        t1[0] = fma(p[j], z[j], t1[0]);
                    }
                    const double yrz = div_recip(rz);
                    csum(t1, slot);
                    iters = it;
                    if (t1[0] <= 0.0) {
                        status = 1;
                        break;
                    }
                    const double alpha = rz / t1[0];
                    double t2[2] = {0.0, 0.0};
#pragma unroll
                    for (int j = 0; j < KM; ++j) {
                        r[j] = fma(-alpha, z[j], r[j]);
                        z[j] = dv[j] * r[j];
                        t2[0] = fma(r[j], r[j], t2[0]);
                        t2[1] = fma(r[j], z[j], t2[1]);
                    }
                    csum(t2, slot);
                    rr_last = t2[0];
                    const bool done = t2[0] <= thr;
                    const double beta = div_finish(t2[1], rz, yrz);  // == t2[1] / rz bitwise
                    rz = t2[1];
#pragma unroll
                    for (int j = 0; j < KM; ++j) {
                        x[j] = fma(alpha, p[j], x[j]);
                        p[j] = fma(beta, p[j], z[j]);
                    }
                    if (done) {
                        status = 0;
                        break;
                    }
                    publish(p);
                    pending = true;
                }
                if (pending) gc_wait();  // maxit reached right after a publish
                rel = sqrt(rr_last) / bnorm;
            }
        }
#pragma unroll
        for (int j = 0; j < KM; ++j) {
            const int k = tid + j * kGcThreads;
            if (k < nloc) a.V[vrow + k0 + k] = x[j];
        }
        if (a.epilogue) {
            publish(x);  // x with halos: true residual and the face integrals
            gc_wait();
            double t3[3] = {0.0, 0.0, 0.0};
#pragma unroll
            for (int j = 0; j < KM; ++j) {
                const int k = tid + j * kGcThreads;
                if (k >= nloc) continue;
                const double y = spmv(k);
                double bk = 0.0;
                if (use_u) bk = fma(cu, __ldg(a.rin + vrow + k0 + k), bk);
                if (use_w) bk = fma(cw, __ldg(a.rout + vrow + k0 + k), bk);
                const double rr = bk - y;
                t3[0] = fma(rr, rr, t3[0]);
            }
            // surface_coupling (src/assembly.cpp:377-393) over the faces whose lowest node this CTA owns
            const double* len = a.face_len + (size_t)Pb * a.face_len_stride;
            for (int f = tid; f < g.nfaces; f += blockDim.x) {
                int axis, side, cc[3], tr[2];
                gen_face(g, f, axis, side, cc, tr);
                const int role = a.role[2 * axis + side];
                if (role != TS_GAMMA_I && role != TS_GAMMA_O) continue;
                int lo = n;
                for (int fa = 0; fa < g.npf; ++fa) lo = min(lo, gen_face_node(g, axis, side, cc, tr, fa));
                if (lo < k0 || lo >= k1) continue;
                double y[3], sc, nrm[3];
                gen_face_geom(g, cGP, axis, side, cc, 0, y, sc, nrm);
                double tot = 0.0;
                for (int q = 0; q < g.nqf; ++q) {
                    double vq = 0.0;
                    for (int fa = 0; fa < g.npf; ++fa)
                        vq = fma(sP[H + gen_face_node(g, axis, side, cc, tr, fa) - k0], cGP.Nf[q][fa], vq);
                    tot += cGP.FW[q] * vq * len[(size_t)f * g.nqf + q] * sc;
                }
                t3[role == TS_GAMMA_I ? 1 : 2] += tot;
            }
            csum(t3, slot);
            if (rank == 0 && tid == 0) {
                a.res_v[Pb] = sqrt(t3[0]);
                a.bI[Pb] = t3[1];
                a.bO[Pb] = t3[2];
            }
        }
        if (rank == 0 && tid == 0) {
            a.iters[Pb] = iters;
            a.status[Pb] = status;
            a.final_rel[Pb] = rel;
        }
        cl.sync();  // the next ticket's operator load overwrites SMEM the peers may still read
    }
}

// ---------------------------------------------- 3D Q1: z-column cluster kernel ------
// Config 5's operator (symmetric half: 14 direction planes, 0.55 MB per problem) held in the
// shared memory of a 4-CTA cluster for the whole solve, split into z-slabs (CTA r owns
// lattice planes [z0, z1), 5 + 4 + 4 + 4 of 17), plus one halo coefficient plane below (the
// lower-half lookups a_{-d}(k) = a_d(k - o_d) reach one plane down).  A thread owns one
// (x, y) column of its slab and walks it in z with a sliding 3x3x3 window of p in registers:
// 9 new p loads per node instead of 27, and every access is unit-stride across the warp.
// p lives in a zero-padded (NX+2)^2 x (nz+2) block; the slab's boundary planes go into the
// neighbours' halo planes over DSMEM, followed by a split cluster barrier (arrive after the
// stores, wait before the first node that needs a halo plane — the interior nodes of each
// column run in between).  Dot products: block sums + one DSMEM exchange on per-slot
// mbarriers (gc_cluster_sum).  Same PCG, stop test and epilogue as k_gen_pcg3_cluster.
constexpr int kZcCL = kGcCL;
constexpr int kZcCLx = kZcCL;

// Transaction-counted DSMEM signalling for the z-column kernel: st.async writes a double
// into a peer CTA's shared memory and completes 8 bytes on that CTA's mbarrier; the waiting
// CTA arms each phase with one arrive.expect_tx for the bytes it expects and waits with a
// plain (CTA-scope) try_wait — the transaction mechanism orders the data, so no release /
// acquire fences at cluster scope (ncu on the fence version: CCTL.IVALL + ERRBAR ~22 % of
// stall samples).
__device__ __forceinline__ unsigned zc_mapa(const void* p, unsigned cta) {
    unsigned r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((unsigned)__cvta_generic_to_shared(p)), "r"(cta));
    return r;
}
__device__ __forceinline__ void zc_st_async(unsigned raddr, double v, unsigned rbar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(raddr),
                 "l"(__double_as_longlong(v)), "r"(rbar)
                 : "memory");
}
__device__ __forceinline__ void zc_expect(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void zc_wait(unsigned long long* bar, unsigned parity) {
    const unsigned laddr = (unsigned)__cvta_generic_to_shared(bar);
    asm volatile(
        "{\n .reg .pred p;\n ZC_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra ZC_WAIT_%=;\n}\n" ::"r"(laddr),
        "r"(parity)
        : "memory");
}

// Cluster total of K values: block sums, then thread q sends this CTA's totals into CTA q's
// exchange slot (st.async, completing on CTA q's slot barrier); every CTA sums the slots in
// rank order (identical bits everywhere).
struct ZcNoop {
    __device__ __forceinline__ void operator()() const {}
};

// between(): work that does not depend on the totals, run after the sends and before the wait
// (it overlaps the exchange's DSMEM round trip)
template <int K, int CL = kZcCLx, class F = ZcNoop>
__device__ __forceinline__ void zc_cluster_sum(double (&v)[K], double* red, double* xch, unsigned long long* bar,
                                               unsigned parity, int rank, F between = F()) {
    if (threadIdx.x == 0) zc_expect(bar, CL * K * 8);
    block_sum<K>(v, red);
    if ((int)threadIdx.x < CL) {
        const unsigned rb = zc_mapa(bar, threadIdx.x);
#pragma unroll
        for (int k = 0; k < K; ++k) zc_st_async(zc_mapa(xch + rank * 4 + k, threadIdx.x), v[k], rb);
    }
    between();
    zc_wait(bar, parity);
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < CL; ++q) t += xch[q * 4 + k];
        v[k] = t;
    }
}

// Cluster total of K values without the CTA stage: every warp sends its K warp sums straight
// into all CTAs' exchange buffers (entry k * 32 + rank * (32 / CL) + warp; unused entries stay
// zero), every thread waits on its CTA's slot barrier and re-reduces the same 32 entries per
// value in the same order (identical bits in every thread of the cluster).  One exchange
// instead of CTA barrier + second stage + exchange.  Needs warps per CTA <= 32 / CL.
template <int K, int CL, class F = ZcNoop>
__device__ __forceinline__ void zc_cluster_sum_direct(double (&v)[K], double* xch, unsigned long long* bar,
                                                      unsigned parity, int rank, F between = F()) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    if (threadIdx.x == 0) zc_expect(bar, CL * nw * K * 8);
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = warp_sum_tc(v[k]);
    if (lane < CL) {
        const unsigned rb = zc_mapa(bar, lane);
#pragma unroll
        for (int k = 0; k < K; ++k) zc_st_async(zc_mapa(xch + k * 32 + rank * (32 / CL) + warp, lane), v[k], rb);
    }
    between();
    zc_wait(bar, parity);  // (one polling warp + a CTA barrier measured slower: 9.79e10 vs 1.005e11 on C4)
#pragma unroll
    for (int k = 0; k < K; ++k) v[k] = warp_sum_tc(xch[k * 32 + lane]);
}

template <int NX, int NZ>
struct ZcGeom {
    static constexpr int NXY = NX * NX;
    static constexpr int HALO = NXY + NX + 1;  // reach of a node's neighbours in node index
    static constexpr int NOWN = NZ * NXY;      // nodes a CTA owns at most (NZ * NX lattice rows)
    static constexpr int ASTR = NOWN + HALO;   // per direction: coefficients of nodes [k0 - HALO, k1)
    static constexpr int COEF = 14 * ASTR;
    static constexpr int PD = NOWN + 2 * HALO;  // p of nodes [k0 - HALO, k1 + HALO)
    static constexpr int EXMAX = 5 * NX;  // top nodes of NZ-node columns that get threads of their own
    static constexpr int THREADS = ((NXY + EXMAX + 31) / 32) * 32;
    static constexpr size_t SMEM =
        ((size_t)COEF + PD + (PD & 1) + kGcSlots * 32 * 4 + kGcSlots * 16 * 4 + kGcSlots + 1 + 2) * sizeof(double);
};

// The lattice rows (z * NX + y) CTA `rank` owns: an even split of all nz * NX rows, so the
// four CTAs differ by at most one row of NX nodes (whole z-planes would give 5 + 4 + 4 + 4 on
// a 17^3 lattice: three CTAs idle for ~20 % of every SpMV).
__host__ __device__ __forceinline__ void zc_rows(int rows_total, int rank, int& r0, int& r1) {
    const int base = rows_total / kZcCL, rem = rows_total % kZcCL;
    r0 = rank * base + min(rank, rem);
    r1 = r0 + base + (rank < rem ? 1 : 0);
}

template <int NX, int NZ, bool CGX>
__global__ void __launch_bounds__(ZcGeom<NX, NZ>::THREADS, 1) k_gen_pcg3_zcol(const GenPcgArgs a) {
    constexpr bool CG1 = CGX;
    using G = ZcGeom<NX, NZ>;
    constexpr int NXY = G::NXY, HALO = G::HALO, ASTR = G::ASTR;
    extern __shared__ double smem[];
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank();
    const GenGeom& g = a.g;
    const int n = g.nnodes, rows_total = g.nn[2] * NX;
    int R0, R1;
    zc_rows(rows_total, rank, R0, R1);
    const int k0 = R0 * NX, k1 = R1 * NX;  // the CTA owns nodes [k0, k1) (lexicographic, z-major)
    // p and the coefficients keep the lattice's own lexicographic order, so a warp's accesses are
    // unit-stride (conflict-free); both are indexed by node - (k0 - HALO).  Out-of-lattice
    // neighbours wrap to another row or plane: there the coefficient of the wrapped direction
    // is exactly zero (no neighbour on that side), so the product vanishes; nodes below 0 or
    // beyond the lattice hit zero entries.
    double* sA = smem;            // [14][ASTR]: coefficient e of node k at sA[e * ASTR + k - k0 + HALO]
    double* sP = smem + G::COEF;  // p of node k at sP[k - k0 + HALO]
    double* red = smem + G::COEF + G::PD + (G::PD & 1);
    double* xch = red + kGcSlots * 32 * 4;
    unsigned long long* sBar = reinterpret_cast<unsigned long long*>(xch + kGcSlots * 16 * 4);  // [kGcSlots + 1]
    unsigned long long* hBar = sBar + kGcSlots;  // halos: the bytes both neighbours send per publish
    int* sTicket = reinterpret_cast<int*>(hBar + 1);
    const int tid = threadIdx.x;
    // One thread per (x, y) column: its nodes in the CTA's row range are z = zf .. zf + nzo - 1.
    // A column's nodes are serial in the sweep, and the SpMV phase is bound by that latency
    // (equalising the CTAs' node counts alone changed nothing), so when the range is NZ - 1
    // full planes plus a few rows, the columns of those rows (NZ nodes) keep NZ - 1 and their top
    // nodes go to threads of their own (tid >= NXY, one node each): every warp's sweep is at most
    // NZ - 1 nodes long.
    constexpr int NZH = NZ;
    const int full = (R1 - R0) / NX, remr = (R1 - R0) % NX, ys = R0 % NX;
    const bool split = full == NZ - 1 && remr > 0 && remr * NX <= G::EXMAX;
    int ct = tid, zskip = 0;
    if (tid >= NXY) {
        const int j = tid - NXY;
        ct = split && j < remr * NX ? (ys * NX + j) % NXY : NXY;  // NXY: no column
        zskip = NZ - 1;
    }
    const int cy = ct / NX;
    const int zf = (R0 > cy ? (R0 - cy + NX - 1) / NX : 0) + zskip;
    const int zl = R1 > cy ? (R1 - cy + NX - 1) / NX : 0;
    const int nzo = ct < NXY ? max(0, min(zl - zf, tid < NXY && split ? NZ - 1 : NZ)) : 0;
    const bool col = nzo > 0;
    const int kf = zf * NXY + ct;     // the thread's first own node
    const int pf = kf - k0 + HALO;    // its sP / sA index; the node above is NXY further
    const int nbrs = (rank > 0) + (rank < kZcCL - 1);
    if (tid <= kGcSlots) gc_mbar_init(sBar + tid, 1);  // slot barriers + the halo barrier: one local arrival
    if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    if (tid == 0) zc_expect(hBar, nbrs * HALO * 8);  // arm the first halo phase
    unsigned phase = 0, hphase = 0;
    // zero everything once: entries no load or publish ever writes (nodes below 0 / beyond the
    // lattice, the tail of a short range) are read against zero coefficients or as zero p
    for (int k = tid; k < G::COEF + G::PD; k += blockDim.x) smem[k] = 0.0;
    auto csum_with = [&](auto& v, int& slot, auto between) {
        zc_cluster_sum<sizeof(v) / sizeof(double), kZcCLx>(v, red + slot * 128, xch + slot * 64, sBar + slot,
                                                           (phase >> slot) & 1u, rank, between);
        phase ^= 1u << slot;
        slot = slot == kGcSlots - 1 ? 0 : slot + 1;
    };
    auto csum = [&](auto& v, int& slot) { csum_with(v, slot, ZcNoop()); };
    // Own values into the p block; the first HALO own nodes into the lower neighbour's upper
    // halo and the last HALO into the upper neighbour's lower halo (st.async, completing on the
    // neighbour's halo barrier); then a CTA barrier.  A column's first / last node always
    // travels, its second / second-to-last one for the NX + 1 columns at the range's ends.  A
    // neighbour is never overwritten while it still reads: every publish is preceded by a
    // cluster dot-product exchange that the neighbour joins only after its SpMV.
    int kb0 = 0;  // first node of the CTA below
    {
        int b0, b1;
        zc_rows(rows_total, rank > 0 ? rank - 1 : 0, b0, b1);
        kb0 = b0 * NX;
    }
    auto publish = [&](const double (&v)[NZH]) {
        if (col) {
#pragma unroll
            for (int sl = 0; sl < NZH; ++sl)
                if (sl < nzo) sP[pf + sl * NXY] = v[sl];
            if (rank > 0) {
                const unsigned rb = zc_mapa(hBar, rank - 1);
#pragma unroll
                for (int sl = 0; sl < (NZH < 2 ? NZH : 2); ++sl) {
                    const int k = kf + sl * NXY;
                    if (sl < nzo && k < k0 + HALO) zc_st_async(zc_mapa(sP + (k - kb0 + HALO), rank - 1), v[sl], rb);
                }
            }
            if (rank < kZcCL - 1) {
                const unsigned rb = zc_mapa(hBar, rank + 1);
#pragma unroll
                for (int sl = 0; sl < NZH; ++sl) {
                    const int k = kf + sl * NXY;
                    if (sl < nzo && k >= k1 - HALO) zc_st_async(zc_mapa(sP + (k - k1 + HALO), rank + 1), v[sl], rb);
                }
            }
        }
        __syncthreads();  // own entries complete
    };
    auto hwait = [&] {
        zc_wait(hBar, hphase);
        hphase ^= 1u;
        if (tid == 0) zc_expect(hBar, nbrs * HALO * 8);  // arm the next phase (no peer sends before we read)
    };
    auto load_plane = [&](int pc, double (&w)[9]) {  // the 3 x 3 (x, y) neighbourhood around sP index pc
        const double* pp = sP + pc;
#pragma unroll
        for (int j = 0; j < 3; ++j)
#pragma unroll
            for (int i = 0; i < 3; ++i) w[i + 3 * j] = pp[(j - 1) * NX + (i - 1)];
    };
    // y = A p at the node with SMEM index pc, window w[plane][3x3] = p planes z-1, z, z+1.
    // cz: the pure-z coefficient a_(0,0,1) of the node below (its lower-half lookup), kept from
    // the previous node of the sweep.
    auto node_yz = [&](int pc, const double (&w)[3][9], double& cz, bool have_cz) {
        const double* A0 = sA + pc;  // own coefficient, direction e at A0[e * ASTR]
        // one partial sum per p plane (z-1, z, z+1): three chains of nine dependent FMAs instead
        // of one of 27 (a column's nodes are serial in the sweep, so the chain is latency)
        double acc[3] = {0.0, A0[0] * w[1][4], 0.0};
#pragma unroll
        for (int e = 1; e < 14; ++e) {
            const int d = 13 + e, dx = d % 3 - 1, dy = (d / 3) % 3 - 1, dz = d / 9 - 1;
            const int wi = (dx + 1) + 3 * (dy + 1);
            const double* Ae = A0 + e * ASTR;
            const bool purez = dx == 0 && dy == 0 && dz == 1;
            const double up = Ae[0];                                                    // a_d(k)
            const double lo = purez && have_cz ? cz : Ae[-(dz * NXY + dy * NX + dx)];  // a_d(k - o_d)
            acc[1 + dz] = fma(up, w[1 + dz][wi], acc[1 + dz]);
            acc[1 - dz] = fma(lo, w[1 - dz][8 - wi], acc[1 - dz]);
            if (purez) cz = up;
        }
        return (acc[0] + acc[2]) + acc[1];
    };
    // One upward sweep over the column after the halo wait, so every p plane is loaded once.
    // The thread's own entries (window centres of its own nodes) come from the registers v:
    // 189 LDS.64 per 5-node column (234 with separate interior / boundary passes).  The halo
    // wait is no longer hidden behind interior nodes; the sweep is SMEM-bound, so the loads it
    // saves outweigh that.
    auto spmv_col = [&](double (&y)[NZH], const double (&v)[NZH]) {
        hwait();
        if (!col) return;
        double w[3][9];
        double cz = 0.0;
        load_plane(pf - NXY, w[0]);
        load_plane(pf, w[1]);
        w[1][4] = v[0];
#pragma unroll
        for (int sl = 0; sl < NZH; ++sl) {
            if (sl >= nzo) break;
            load_plane(pf + (sl + 1) * NXY, w[2]);
            if (sl + 1 < nzo) w[2][4] = v[sl + 1 < NZH ? sl + 1 : 0];  // own node: centre from the register
            y[sl] = node_yz(pf + sl * NXY, w, cz, sl > 0);
#pragma unroll
            for (int k = 0; k < 9; ++k) {
                w[0][k] = w[1][k];
                w[1][k] = w[2][k];
            }
        }
    };

    int slot = 0;
    cl.sync();  // every CTA started (mbarriers initialised, halos zeroed) before remote writes
    if (rank == 0 && tid == 0) {
        const int t = atomicAdd(a.counter, 1);
        for (int q = 0; q < kZcCL; ++q) cl.map_shared_rank(sTicket, q)[1] = t;
    }
    for (;;) {
        if (rank == 0 && tid == 0) {
            const int cur = sTicket[1];
            const int nxt = cur < a.n_problems ? atomicAdd(a.counter, 1) : cur;
            for (int q = 0; q < kZcCL; ++q) {
                int* t = cl.map_shared_rank(sTicket, q);
                t[0] = cur;
                t[1] = nxt;
            }
        }
        cl.sync();
        const int Pb = sTicket[0];
        if (Pb >= a.n_problems) break;
        if (sTicket[1] < a.n_problems && a.stencil_stride) {  // next problem's slab into L2
            const char* nst = reinterpret_cast<const char*>(a.stencil + (size_t)sTicket[1] * a.stencil_stride);
            const int lo = max(0, k0 - HALO), hi = k1;
            const int lines = ((hi - lo) * 8 + 127) / 128 + 1;
            for (int t = tid; t < 14 * lines; t += blockDim.x) {
                const int e = t / lines, l = t % lines;
                const size_t off = ((size_t)e * n + lo) * 8 + (size_t)l * 128;
                if (off < ((size_t)e * n + hi) * 8) asm volatile("prefetch.global.L2 [%0];" ::"l"(nst + off));
            }
        }
        const double* st = a.stencil + (size_t)Pb * a.stencil_stride;
        const double uP = a.u[Pb], wP = a.w[Pb];
        const bool use_u = a.kappa1 != 0.0 && uP != 0.0, use_w = a.kappa3 != 0.0 && wP != 0.0;
        const double cu = a.kappa1 * uP, cw = a.kappa3 * wP;
        const size_t vrow = (size_t)Pb * n;
        // coefficients of nodes [k0 - HALO, k1) (zero below node 0)
        for (int e = 0; e < 14; ++e) {
            const double* src = st + (size_t)e * n;
            for (int k = tid; k < k1 - k0 + HALO; k += blockDim.x) {
                const int gk = k0 - HALO + k;
                sA[e * ASTR + k] = gk >= 0 ? __ldg(src + gk) : 0.0;
            }
        }
        double x[NZH], r[NZH], dv[NZH], z[NZH];
#pragma unroll
        for (int zi = 0; zi < NZH; ++zi) {
            x[zi] = r[zi] = z[zi] = 0.0;
            dv[zi] = 1.0;
            if (col && zi < nzo) {
                const int k = kf + zi * NXY;
                const double dg = __ldg(st + k);
                dv[zi] = dg != 0.0 ? 1.0 / dg : 1.0;
                double bk = 0.0;
                if (use_u) bk = fma(cu, __ldg(a.rin + vrow + k), bk);
                if (use_w) bk = fma(cw, __ldg(a.rout + vrow + k), bk);
                r[zi] = bk;
                x[zi] = a.warm ? a.V[vrow + k] : 0.0;
            }
        }
        auto own = [&](int zi) { return col && zi < nzo; };  // zi: the thread's slot
        publish(x);  // (its CTA barrier also completes sA)
        double s3[3] = {0.0, 0.0, 0.0};
        {
            double y[NZH];
            spmv_col(y, x);
#pragma unroll
            for (int zi = 0; zi < NZH; ++zi) {
                if (!own(zi)) continue;
                const double bk = r[zi];
                s3[0] = fma(bk, bk, s3[0]);
                r[zi] = bk - y[zi];
                z[zi] = dv[zi] * r[zi];
                s3[1] = fma(r[zi], z[zi], s3[1]);
                s3[2] = fma(r[zi], r[zi], s3[2]);
            }
        }
        csum(s3, slot);
        const double bnorm = sqrt(s3[0]);
        int status = 0, iters = 0;
        double rel = 0.0;
        if (bnorm == 0.0) {
#pragma unroll
            for (int zi = 0; zi < NZH; ++zi) x[zi] = 0.0;
        } else {
            double rz = s3[1];
            rel = sqrt(s3[2]) / bnorm;
            if (rel > a.tol && CG1) {
                // Single-reduction PCG (Chronopoulos & Gear): s = A p is carried by the
                // recurrence s = w + beta s with w = A u, u = D^-1 r, so one SpMV and ONE cluster
                // reduction {(r,u), (w,u), (r,r)} per iteration instead of two.  Same iterates as
                // src/linalg.cpp:103-161 in exact arithmetic (rounding differs): x, r, the stop
                // test on the recursive ||r||, p.Ap = delta - beta gamma / alpha_prev <= 0 ->
                // indefinite, iteration counts as the reference's loop SpMVs.
                const double thr = rel_threshold(bnorm, a.tol);
                double rr_last = s3[2];
                double p[NZH], sv[NZH], w[NZH];
                double gamma = rz;
                publish(z);  // u0 = z0
                spmv_col(w, z);  // w0 = A u0
                double t1[1] = {0.0};
#pragma unroll
                for (int zi = 0; zi < NZH; ++zi) {
                    if (!own(zi)) w[zi] = 0.0;
                    t1[0] = fma(w[zi], z[zi], t1[0]);
                }
                csum(t1, slot);
                status = 2;
                iters = 1;
                double pAp = t1[0], alpha = 0.0;
                if (pAp <= 0.0) {
                    status = 1;
                } else {
                    alpha = gamma / pAp;
#pragma unroll
                    for (int zi = 0; zi < NZH; ++zi) {
                        p[zi] = z[zi];
                        sv[zi] = w[zi];
                    }
#ifdef TSB_PHASE_TIMING
                    long long ph[6] = {0, 0, 0, 0, 0, 0}, tc = clock64();
#define TSB_PHZ(i)                      \
    {                                   \
        const long long tn = clock64(); \
        ph[i] += tn - tc;               \
        tc = tn;                        \
    }
#else
#define TSB_PHZ(i)
#endif
                    for (int it = 1; it <= a.maxit; ++it) {
                        iters = it;
                        double t3[3] = {0.0, 0.0, 0.0};  // (r,u), (r,r), then (w,u)
#pragma unroll
                        for (int zi = 0; zi < NZH; ++zi) {
                            x[zi] = fma(alpha, p[zi], x[zi]);
                            r[zi] = fma(-alpha, sv[zi], r[zi]);
                            z[zi] = dv[zi] * r[zi];  // u
                            t3[0] = fma(r[zi], z[zi], t3[0]);
                            t3[1] = fma(r[zi], r[zi], t3[1]);
                        }
                        TSB_PHZ(0)
                        publish(z);
                        TSB_PHZ(1)
                        spmv_col(w, z);
                        TSB_PHZ(2)
#pragma unroll
                        for (int zi = 0; zi < NZH; ++zi) {
                            if (!own(zi)) w[zi] = 0.0;
                            t3[2] = fma(w[zi], z[zi], t3[2]);
                        }
                        // divisor-only parts of the two quotients whose divisors are known
                        // before the reduction (bitwise a / b, device_common.cuh)
                        // divisor-only parts of the two quotients whose divisors are known
                        // before the reduction (bitwise a / b, device_common.cuh).  (The Q2
                        // kernel's shorter chain through c = 1 / (gamma alpha) measured -1 % here.)
                        const double yg = div_recip(gamma), ya = div_recip(alpha);
                        csum(t3, slot);
                        TSB_PHZ(3)
                        rr_last = t3[1];
                        if (t3[1] <= thr) {  // iteration it converged (its x is final)
                            status = 0;
                            break;
                        }
                        if (it == a.maxit) break;
                        const double beta = div_finish(t3[0], gamma, yg);
                        gamma = t3[0];
                        pAp = t3[2] - div_finish(beta * gamma, alpha, ya);
                        if (pAp <= 0.0) {  // iteration it + 1's p.Ap (src/linalg.cpp:138-142)
                            iters = it + 1;
                            status = 1;
                            break;
                        }
                        alpha = gamma / pAp;
#pragma unroll
                        for (int zi = 0; zi < NZH; ++zi) {
                            p[zi] = fma(beta, p[zi], z[zi]);
                            sv[zi] = fma(beta, sv[zi], w[zi]);
                        }
                        TSB_PHZ(4)
                    }
#ifdef TSB_PHASE_TIMING
                    if ((tid == 0 || tid == 288) && Pb % 41 == 0 && Pb < 160)
                        printf("P %d rank %d tid %d iters %d: update %lld publish %lld spmv(+hwait) %lld dots+csum %lld scalars+ps %lld (cycles per iteration)\n",
                               Pb, rank, tid, iters, ph[0] / iters, ph[1] / iters, ph[2] / iters, ph[3] / iters, ph[4] / iters);
#endif
                }
                rel = sqrt(rr_last) / bnorm;
            } else if (rel > a.tol) {
                const double thr = rel_threshold(bnorm, a.tol);
                double rr_last = s3[2];
                double p[NZH];
#pragma unroll
                for (int zi = 0; zi < NZH; ++zi) p[zi] = z[zi];
                publish(p);
                bool pending = true;
                status = 2;
                for (int it = 1; it <= a.maxit; ++it) {
                    double y[NZH];
                    spmv_col(y, p);
                    pending = false;
                    double t1[1] = {0.0};
#pragma unroll
                    for (int zi = 0; zi < NZH; ++zi) {
                        z[zi] = own(zi) ? y[zi] : 0.0;  // z holds Ap until the r update
                        t1[0] = fma(p[zi], z[zi], t1[0]);
                    }
                    const double yrz = div_recip(rz);
                    csum(t1, slot);
                    iters = it;
                    if (t1[0] <= 0.0) {
                        status = 1;
                        break;
                    }
                    const double alpha = rz / t1[0];
                    double t2[2] = {0.0, 0.0};
#pragma unroll
                    for (int zi = 0; zi < NZH; ++zi) {
                        r[zi] = fma(-alpha, z[zi], r[zi]);
                        z[zi] = dv[zi] * r[zi];
                        t2[0] = fma(r[zi], r[zi], t2[0]);
                        t2[1] = fma(r[zi], z[zi], t2[1]);
                    }
                    csum(t2, slot);
                    rr_last = t2[0];
                    const bool done = t2[0] <= thr;
                    const double beta = div_finish(t2[1], rz, yrz);
                    rz = t2[1];
#pragma unroll
                    for (int zi = 0; zi < NZH; ++zi) {
                        x[zi] = fma(alpha, p[zi], x[zi]);
                        p[zi] = fma(beta, p[zi], z[zi]);
                    }
                    if (done) {
                        status = 0;
                        break;
                    }
                    publish(p);
                    pending = true;
                }
                if (pending) hwait();
                rel = sqrt(rr_last) / bnorm;
            }
        }
#pragma unroll
        for (int zi = 0; zi < NZH; ++zi)
            if (own(zi)) a.V[vrow + kf + zi * NXY] = x[zi];
        if (a.epilogue) {
            publish(x);  // x with halos: true residual and the face integrals
            double t3[3] = {0.0, 0.0, 0.0};
            {
                double y[NZH];
                spmv_col(y, x);
#pragma unroll
                for (int zi = 0; zi < NZH; ++zi) {
                    if (!own(zi)) continue;
                    const int k = kf + zi * NXY;
                    double bk = 0.0;
                    if (use_u) bk = fma(cu, __ldg(a.rin + vrow + k), bk);
                    if (use_w) bk = fma(cw, __ldg(a.rout + vrow + k), bk);
                    const double rr = bk - y[zi];
                    t3[0] = fma(rr, rr, t3[0]);
                }
            }
            // surface_coupling (src/assembly.cpp:377-393) over the faces whose lowest node this CTA owns
            const double* len = a.face_len + (size_t)Pb * a.face_len_stride;
            for (int f = tid; f < g.nfaces; f += blockDim.x) {
                int axis, side, cc[3], tr[2];
                gen_face(g, f, axis, side, cc, tr);
                const int role = a.role[2 * axis + side];
                if (role != TS_GAMMA_I && role != TS_GAMMA_O) continue;
                int lo = n;
                for (int fa = 0; fa < g.npf; ++fa) lo = min(lo, gen_face_node(g, axis, side, cc, tr, fa));
                if (lo < k0 || lo >= k1) continue;
                double yq[3], sc, nrm[3];
                gen_face_geom(g, cGP, axis, side, cc, 0, yq, sc, nrm);
                double tot = 0.0;
                for (int q = 0; q < g.nqf; ++q) {
                    double vq = 0.0;
                    for (int fa = 0; fa < g.npf; ++fa) {
                        const int nd = gen_face_node(g, axis, side, cc, tr, fa);
                        const double xv = sP[nd - k0 + HALO];
                        vq = fma(xv, cGP.Nf[q][fa], vq);
                    }
                    tot += cGP.FW[q] * vq * len[(size_t)f * g.nqf + q] * sc;
                }
                t3[role == TS_GAMMA_I ? 1 : 2] += tot;
            }
            csum(t3, slot);
            if (rank == 0 && tid == 0) {
                a.res_v[Pb] = sqrt(t3[0]);
                a.bI[Pb] = t3[1];
                a.bO[Pb] = t3[2];
            }
        }
        if (rank == 0 && tid == 0) {
            a.iters[Pb] = iters;
            a.status[Pb] = status;
            a.final_rel[Pb] = rel;
        }
        cl.sync();  // the next ticket's operator load overwrites SMEM the peers may still read
    }
}

// 4-CTA clusters cannot use every SM (GPC sizes: 132 of 148 SMs on B200), so the SMs the
// cluster kernel leaves idle run the streaming kernel (k_gen_pcg<3, 1>) on a side stream,
// pulling tickets from the same counter: both drain one queue of problems.  Fork / join by
// events, so this also works inside a stream capture.  TS_GEN_ZFILL=0 disables it.
struct ZcSide {
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr;
};

ZcSide* zc_side() {
    // one side stream and event pair per host thread and device: contexts on different host
    // threads never share the fork/join events
    static thread_local ZcSide side[16];
    int dev = 0;
    cudaGetDevice(&dev);
    ZcSide& sd = side[dev & 15];
    if (!sd.s) {
        if (cudaStreamCreateWithFlags(&sd.s, cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&sd.fork, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&sd.join, cudaEventDisableTiming) != cudaSuccess) {
            cudaGetLastError();
            sd.s = nullptr;
            return nullptr;
        }
    }
    return &sd;
}

int zc_idle_sms(const GenPcgArgs& a, int cluster_ctas) {
    if (const char* e = std::getenv("TS_GEN_ZFILL"))
        if (e[0] == '0') return 0;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int idle = sms - cluster_ctas;
    if (idle <= 0 || a.n_problems <= cluster_ctas / kZcCL || gen_pcg_smem_bytes(a.g) > 232448 ||
        a.g.nnodes > kMaxK * kThreadsG)
        return 0;
    return idle;
}

bool zc_fill_fork(const GenPcgArgs& a, int cluster_ctas, cudaStream_t s) {
    if (!zc_idle_sms(a, cluster_ctas)) return false;
    ZcSide* sd = zc_side();
    if (!sd) return false;
    cudaEventRecord(sd->fork, s);
    cudaStreamWaitEvent(sd->s, sd->fork, 0);
    return true;
}

void zc_fill_launch(const GenPcgArgs& a, int cluster_ctas, cudaStream_t s) {
    ZcSide* sd = zc_side();
    const size_t smem = gen_pcg_smem_bytes(a.g);
    cudaFuncSetAttribute(k_gen_pcg<3, 1, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_gen_pcg<3, 1, false><<<zc_idle_sms(a, cluster_ctas), kThreadsG, smem, sd->s>>>(a);
    cudaEventRecord(sd->join, sd->s);
    cudaStreamWaitEvent(s, sd->join, 0);
}

template <int NX, int NZ>
bool zc_launch_t(const GenPcgArgs& a, cudaStream_t s) {
    using G = ZcGeom<NX, NZ>;
    // single-reduction loop by default (measured +2.6 % on config 5); TS_GEN_CG1=0: the
    // two-reduction loop with the reference's operation order
    const char* e = std::getenv("TS_GEN_CG1");
    const bool cg1 = !(e && e[0] == '0');
    auto kern = cg1 ? k_gen_pcg3_zcol<NX, NZ, true> : k_gen_pcg3_zcol<NX, NZ, false>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(G::THREADS);
    cfg.dynamicSmemBytes = G::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kZcCL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(kZcCL);
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess || nclusters < 1) {
        cudaGetLastError();
        return false;
    }
    if (nclusters > a.n_problems) nclusters = a.n_problems;
    cfg.gridDim = dim3(kZcCL * nclusters);
    // the side stream forks before the cluster launch (an event recorded after it would
    // complete only when the cluster kernel does)
    const bool fill = zc_fill_fork(a, kZcCL * nclusters, s);
    if (cudaLaunchKernelEx(&cfg, kern, a) != cudaSuccess) return false;
    if (fill) zc_fill_launch(a, kZcCL * nclusters, s);
    return true;
}

// The z-column kernel for the lattices it is instantiated for (17^3: config 5; 13^3), unless
// TS_GEN_ZCOL=0.  Slab heights: ceil(nz / 4) <= NZ.
bool zc_launch(const GenPcgArgs& a, cudaStream_t s) {
    if (const char* e = std::getenv("TS_GEN_ZCOL"))
        if (e[0] == '0') return false;
    const GenGeom& g = a.g;
    if (g.d != 3 || g.p != 1 || g.nn[0] != g.nn[1]) return false;
    if (g.nn[0] == 17 && g.nn[2] >= 2 * kZcCL && (g.nn[2] + kZcCL - 1) / kZcCL <= 5) return zc_launch_t<17, 5>(a, s);
    if (g.nn[0] == 13 && g.nn[2] >= 2 * kZcCL && (g.nn[2] + kZcCL - 1) / kZcCL <= 4) return zc_launch_t<13, 4>(a, s);
    return false;
}

// Used when the lattice fits and the batch is too small to fill the GPU with one problem
// per SM (n_problems * kGcCL <= #SMs): there the cluster puts 4x the SMs on the batch
// (c5 at 4x4 macro / 12^3 micro: 4.8e9 vs 1.5e9 DoF*it/s).  On full config 5 (4225
// problems) it measured 3.14e10 vs 3.22e10 for the streaming kernel (three cluster
// barriers per iteration, 16 SMs stranded by 4-CTA clusters), so it is not used there.
// TS_GEN_CLUSTER=1 forces it wherever it fits, 0 disables it.
bool gc_fits(const GenGeom& g, int n_problems) {
    int want = -1;
    if (const char* e = std::getenv("TS_GEN_CLUSTER")) want = std::atoi(e);
    if (want == 0 || g.d != 3 || g.p != 1) return false;
    const GcGeom m = gc_geom(g);
    if (!(m.chunk >= 2 * m.H && m.chunk <= 4 * kGcThreads && gc_smem_bytes(g) <= 232448)) return false;
    if (want == 1) return true;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    return (long long)n_problems * kGcCL <= sms;
}

template <int KM>
bool gc_launch_km(const GenPcgArgs& a, cudaStream_t s) {
    auto kern = k_gen_pcg3_cluster<KM>;
    const size_t smem = gc_smem_bytes(a.g);
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return false;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(kGcThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kGcCL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(kGcCL);
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess || nclusters < 1) {
        cudaGetLastError();
        return false;
    }
    if (nclusters > a.n_problems) nclusters = a.n_problems;
    cfg.gridDim = dim3(kGcCL * nclusters);
    return cudaLaunchKernelEx(&cfg, kern, a) == cudaSuccess;
}

bool gc_launch(const GenPcgArgs& a, cudaStream_t s) {
    switch ((gc_geom(a.g).chunk + kGcThreads - 1) / kGcThreads) {
        case 1: return gc_launch_km<1>(a, s);
        case 2: return gc_launch_km<2>(a, s);
        case 3: return gc_launch_km<3>(a, s);
        case 4: return gc_launch_km<4>(a, s);
    }
    return false;
}

}  // namespace

// ------------------------------------------------- 2D Q2, class-compact operator --
// Lattice nodes (i, j) fall into four parity classes c = (i & 1) + 2 (j & 1): vertices
// (couple to the 5x5 box), horizontal / vertical edge midpoints (3x5 / 5x3) and cell
// interiors (3x3).  The compact operator stores, per class and class-major, only those
// directions (25/15/15/9 planes, ~16 per node instead of 25), and p lives in four
// class planes with a one-node zero halo; a warp of one class then reads consecutive
// coefficients and consecutive p entries for every direction.  Same PCG as k_gen_pcg.
struct Q2Geom {
    int nn0, nn1, ci[2], cj[2], nc[4], KB[5], QB[5], PPi, PS;
};

// Slots: class c's slots cover its padded p plane row by row at the plane pitch PPi (the
// halo columns are dead slots), so slot K and its p entry advance together: a warp's p
// accesses — own and every neighbour offset — are one contiguous run, free of bank
// conflicts (the compact enumeration wrapped rows at ci[a] < PPi: 26 % of the kernel's SMEM
// wavefronts were conflicts, profiles/r01/prof_q2_c4_raw.csv).
__host__ __device__ __forceinline__ Q2Geom q2_geom(const GenGeom& g) {
    Q2Geom q;
    q.nn0 = g.nn[0];
    q.nn1 = g.nn[1];
    q.ci[0] = (q.nn0 + 1) / 2;
    q.ci[1] = q.nn0 / 2;
    q.cj[0] = (q.nn1 + 1) / 2;
    q.cj[1] = q.nn1 / 2;
    q.PPi = q.ci[0] + 2;
    q.PS = q.PPi * (q.cj[0] + 2);
    q.KB[0] = 0;
    q.QB[0] = 0;
    for (int c = 0; c < 4; ++c) {
        const int a = c & 1, b = c >> 1;
        q.nc[c] = q.ci[a] * q.cj[b];
        q.KB[c + 1] = q.KB[c] + q.PPi * q.cj[b];
        q.QB[c + 1] = q.QB[c] + (a ? 3 : 5) * (b ? 3 : 5) * q.nc[c];
    }
    return q;
}

// class-major slot K -> class, compact local index, node, class-plane p index; false for a
// dead (halo-column) slot
__device__ __forceinline__ bool q2_slot(const Q2Geom& q, int K, int& c, int& l, int& node, int& pa) {
    c = K < q.KB[1] ? 0 : K < q.KB[2] ? 1 : K < q.KB[3] ? 2 : 3;
    const int a = c & 1, b = c >> 1;
    const int w = K - q.KB[c], col = w % q.PPi, jj = w / q.PPi, ii = col - 1;
    pa = c * q.PS + (jj + 1) * q.PPi + col;
    l = ii + q.ci[a] * jj;
    node = (2 * ii + a) + q.nn0 * (2 * jj + b);
    return ii >= 0 && ii < q.ci[a];
}

// node -> class-major slot
__device__ __forceinline__ int q2_slot_of(const Q2Geom& q, int node) {
    const int i = node % q.nn0, j = node / q.nn0;
    const int a = i & 1, b = j & 1, c = a + 2 * b;
    return q.KB[c] + (i >> 1) + 1 + q.PPi * (j >> 1);
}

__global__ void k_q2_repack(const GenGeom g, int rows, const double* __restrict__ st, double* __restrict__ qst) {
    const Q2Geom q = q2_geom(g);
    const int n = g.nnodes;
    const long long per = q.QB[4];
    const long long total = (long long)rows * per;
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
         t += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(t / per);
        const int e = (int)(t % per);
        int c = 0;
        while (c < 3 && e >= q.QB[c + 1]) ++c;
        const int a = c & 1, b = c >> 1, Lx = a ? 1 : 2, Ly = b ? 1 : 2;
        const int w = e - q.QB[c];
        const int dd = w / q.nc[c], l = w % q.nc[c];
        const int dx = dd % (2 * Lx + 1) - Lx, dy = dd / (2 * Lx + 1) - Ly;
        const int ii = l % q.ci[a], jj = l / q.ci[a];
        const int node = (2 * ii + a) + q.nn0 * (2 * jj + b);
        // generic direction index (P = 2) d = (dx + 2) + 5 (dy + 2); the operator stores the
        // upper half (planes d - 12 for d >= 12), the lower half is the neighbour's entry:
        // a_d(k) = a_{24 - d}(k + o_d) (zero where k + o_d is outside the lattice)
        const int d = (dx + 2) + 5 * (dy + 2);
        double v;
        if (d >= 12) {
            v = st[((size_t)row * 13 + (d - 12)) * n + node];
        } else {
            const int i2 = 2 * ii + a + dx, j2 = 2 * jj + b + dy;
            v = i2 >= 0 && i2 < q.nn0 && j2 >= 0 && j2 < q.nn1
                    ? st[((size_t)row * 13 + (12 - d)) * n + i2 + q.nn0 * j2]
                    : 0.0;
        }
        qst[(size_t)row * per + e] = v;
    }
}

constexpr int kQ2Slots = 9;  // n <= 9 * 512

// Compact-operator SpMV for one node of parity class (A, B) (A = i & 1, B = j & 1).
template <int A, int B>
__device__ __forceinline__ double q2_spmv(const double* __restrict__ base, size_t ncl, const double* __restrict__ p,
                                          int PS, int PPi) {
    constexpr int Lx = A ? 1 : 2, Ly = B ? 1 : 2, C = A + 2 * B;
    double acc = 0.0;
#pragma unroll
    for (int dy = -Ly; dy <= Ly; ++dy) {
#pragma unroll
        for (int dx = -Lx; dx <= Lx; ++dx) {
            constexpr int dummy = 0;
            (void)dummy;
            const int dd = (dy + Ly) * (2 * Lx + 1) + (dx + Lx);
            const int c2 = ((A + dx) & 1) + 2 * ((B + dy) & 1);
            const int off = (c2 - C) * PS + ((B + dy) >> 1) * PPi + ((A + dx) >> 1);
            acc = fma(__ldg(base + dd * ncl), p[off], acc);
        }
    }
    return acc;
}

__global__ void __launch_bounds__(kThreadsG, 1) k_gen_pcg_q2(const GenPcgArgs a) {
    extern __shared__ double smem[];
    const GenGeom& g = a.g;
    const Q2Geom q = q2_geom(g);
    const int n = g.nnodes;
    double* sP = smem;                 // 4 class planes
    const int ns = q.KB[4];            // slots (live nodes + dead halo-column slots)
    double* sx = sP + 4 * q.PS;        // vectors in slot order
    double* sr = sx + ns;
    double* sd = sr + ns;
    double* sz = sd + ns;
    double* red = sz + ns;
    int* sTicket = reinterpret_cast<int*>(red + 3 * kRedStride);
    const int tid = threadIdx.x;
    int cl[kQ2Slots], pa[kQ2Slots];  // packed (class << 28 | local index), p index; cl < 0: none
#pragma unroll
    for (int j = 0; j < kQ2Slots; ++j) {
        const int K = tid + j * blockDim.x;
        int c = 0, l = 0, node = 0, p = 0;
        const bool live = K < q.KB[4] && q2_slot(q, K, c, l, node, p);
        cl[j] = live ? (c << 28) | l : -1;
        pa[j] = p;
    }
    auto node_of = [&](int c, int l) {
        const int aa = c & 1, bb = c >> 1;
        return (2 * (l % q.ci[aa]) + aa) + q.nn0 * (2 * (l / q.ci[aa]) + bb);
    };
    // visit slots: f(slot K, class, local, p index)
    auto for_slots = [&](auto&& f) {
#pragma unroll
        for (int j = 0; j < kQ2Slots; ++j)
            if (cl[j] >= 0) f(tid + j * (int)blockDim.x, cl[j] >> 28, cl[j] & 0x0fffffff, pa[j]);
    };
    // y = (A p) at one slot; directions in CSR order (dy outer, dx inner); the class is
    // warp-uniform, so the switch picks one fully compile-time direction set
    auto spmv_at = [&](const double* __restrict__ qs, int c, int l, int p) {
        const double* base = qs + q.QB[c] + l;
        const size_t ncl = (size_t)q.nc[c];
        switch (c) {
            case 0: return q2_spmv<0, 0>(base, ncl, sP + p, q.PS, q.PPi);
            case 1: return q2_spmv<1, 0>(base, ncl, sP + p, q.PS, q.PPi);
            case 2: return q2_spmv<0, 1>(base, ncl, sP + p, q.PS, q.PPi);
            default: return q2_spmv<1, 1>(base, ncl, sP + p, q.PS, q.PPi);
        }
    };
    for (int k = tid; k < 4 * q.PS; k += blockDim.x) sP[k] = 0.0;

    for (;;) {
        __syncthreads();
        if (tid == 0) *sTicket = atomicAdd(a.counter, 1);
        __syncthreads();
        const int Pb = *sTicket;
        if (Pb >= a.n_problems) break;
        const double* qs = a.qstencil + (size_t)Pb * a.qstencil_stride;
        const double uP = a.u[Pb], wP = a.w[Pb];
        const bool use_u = a.kappa1 != 0.0 && uP != 0.0, use_w = a.kappa3 != 0.0 && wP != 0.0;
        const double cu = a.kappa1 * uP, cw = a.kappa3 * wP;
        const size_t vrow = (size_t)Pb * n;
        for_slots([&](int K, int c, int l, int p) {
            const int aa = c & 1, bb = c >> 1, Lx = aa ? 1 : 2, Ly = bb ? 1 : 2;
            const double dg = __ldg(qs + q.QB[c] + (size_t)(Ly * (2 * Lx + 1) + Lx) * q.nc[c] + l);
            sd[K] = dg != 0.0 ? 1.0 / dg : 1.0;
            const int k = node_of(c, l);
            double bk = 0.0;
            if (use_u) bk = fma(cu, __ldg(a.rin + vrow + k), bk);
            if (use_w) bk = fma(cw, __ldg(a.rout + vrow + k), bk);
            sr[K] = bk;
            const double x0 = a.warm ? a.V[vrow + k] : 0.0;
            sx[K] = x0;
            sP[p] = x0;
        });
        __syncthreads();
        double s3[3] = {0.0, 0.0, 0.0};
        for_slots([&](int K, int c, int l, int p) {
            const double y = spmv_at(qs, c, l, p);
            const double bk = sr[K];
            s3[0] = fma(bk, bk, s3[0]);
            const double r = bk - y;
            sr[K] = r;
            const double z = sd[K] * r;
            sz[K] = z;
            s3[1] = fma(r, z, s3[1]);
            s3[2] = fma(r, r, s3[2]);
        });
        block_sum<3>(s3, red);
        int slot = 1;
        const double bnorm = sqrt(s3[0]);
        int status = 0, iters = 0;
        double rel = 0.0;
        if (bnorm == 0.0) {
            for_slots([&](int K, int, int, int) { sx[K] = 0.0; });
        } else {
            double rz = s3[1];
            rel = sqrt(s3[2]) / bnorm;
            if (rel > a.tol) {
                const double thr = rel_threshold(bnorm, a.tol);  // rr <= thr <=> sqrt(rr) / bnorm <= tol
                double rr_last = s3[2];
                for_slots([&](int K, int, int, int p) { sP[p] = sz[K]; });
                __syncthreads();
                status = 2;
                for (int it = 1; it <= a.maxit; ++it) {
                    double t1[1] = {0.0};
                    for_slots([&](int K, int c, int l, int p) {
                        const double y = spmv_at(qs, c, l, p);
                        sz[K] = y;
                        t1[0] = fma(sP[p], y, t1[0]);
                    });
                    const double yrz = div_recip(rz);  // divisor part of beta = rz_new / rz, overlaps the reduction
                    block_sum<1>(t1, red + slot * kRedStride);
                    slot = slot == 2 ? 0 : slot + 1;
                    iters = it;
                    if (t1[0] <= 0.0) {
                        status = 1;
                        break;
                    }
                    const double alpha = rz / t1[0];
                    double t2[2] = {0.0, 0.0};
                    for_slots([&](int K, int, int, int) {
                        const double r = fma(-alpha, sz[K], sr[K]);
                        sr[K] = r;
                        const double z = sd[K] * r;
                        sz[K] = z;
                        t2[0] = fma(r, r, t2[0]);
                        t2[1] = fma(r, z, t2[1]);
                    });
                    block_sum<2>(t2, red + slot * kRedStride);
                    slot = slot == 2 ? 0 : slot + 1;
                    rr_last = t2[0];
                    const bool done = t2[0] <= thr;
                    const double beta = div_finish(t2[1], rz, yrz);  // == t2[1] / rz bitwise
                    rz = t2[1];
                    for_slots([&](int K, int, int, int p) {
                        const double pv = sP[p];
                        sx[K] = fma(alpha, pv, sx[K]);
                        if (!done) sP[p] = fma(beta, pv, sz[K]);
                    });
                    if (done) {
                        status = 0;
                        break;
                    }
                    __syncthreads();
                }
                rel = sqrt(rr_last) / bnorm;  // the last relative residual, as the loop computed it
            }
        }
        for_slots([&](int K, int c, int l, int) { a.V[vrow + node_of(c, l)] = sx[K]; });
        if (a.epilogue) {
            __syncthreads();
            for_slots([&](int K, int, int, int p) { sP[p] = sx[K]; });
            __syncthreads();
            double t1[1] = {0.0};
            for_slots([&](int K, int c, int l, int p) {
                const double y = spmv_at(qs, c, l, p);
                const int k = node_of(c, l);
                double bk = 0.0;
                if (use_u) bk = fma(cu, __ldg(a.rin + vrow + k), bk);
                if (use_w) bk = fma(cw, __ldg(a.rout + vrow + k), bk);
                const double rr = bk - y;
                t1[0] = fma(rr, rr, t1[0]);
            });
            block_sum<1>(t1, red + slot * kRedStride);
            const int warp = tid >> 5, lane = tid & 31;
            for (int rw = warp; rw < 2; rw += (int)(blockDim.x >> 5)) {
                const int role = rw == 0 ? TS_GAMMA_I : TS_GAMMA_O;
                const double* len = a.face_len + (size_t)Pb * a.face_len_stride;
                double tot = 0.0;
                for (int f = lane; f < g.nfaces; f += 32) {
                    int axis, side, cc[3], tr[2];
                    gen_face(g, f, axis, side, cc, tr);
                    if (a.role[2 * axis + side] != role) continue;
                    double y[3], sc, nrm[3];
                    gen_face_geom(g, cGP, axis, side, cc, 0, y, sc, nrm);
                    for (int qq = 0; qq < g.nqf; ++qq) {
                        double vq = 0.0;
                        for (int fa = 0; fa < g.npf; ++fa)
                            vq = fma(sx[q2_slot_of(q, gen_face_node(g, axis, side, cc, tr, fa))], cGP.Nf[qq][fa], vq);
                        tot += cGP.FW[qq] * vq * len[(size_t)f * g.nqf + qq] * sc;
                    }
                }
                tot = warp_sum(tot);
                if (lane == 0) (rw == 0 ? a.bI : a.bO)[Pb] = tot;
            }
            if (tid == 0) a.res_v[Pb] = sqrt(t1[0]);
        }
        if (tid == 0) {
            a.iters[Pb] = iters;
            a.status[Pb] = status;
            a.final_rel[Pb] = rel;
        }
    }
}

// ------------------------------------- 2D Q2, matrix-free from coefficient tensors --
// The north star's second operator representation (BASELINE.json): instead
// of the assembled operator, the PCG reads per cell quadrature point the pulled-back
// coefficient tensor (the three entries of A = C^T D C / det scaled by the quadrature weight
// and the gradient scales, plus J k w for the reaction term) — 36 doubles per cell, 70.53 B
// per DoF on config 4 against 125 B for CSR values (~129 B class-compact) — and applies the
// bilinear form of src/assembly.cpp:129-147 by sum factorisation: 1-D Lagrange tables
// along each axis (Gauss-3 points, nodes -1, 0, 1), 315 FMA per cell.  Cells are visited in
// four colours (cell parities) so a colour's cells share no node: each adds its element
// vector into y without atomics, in a fixed colour order (deterministic).  The Robin face
// mass (assembly.cpp:149-169) is a per-boundary-node gather over <= 2 faces per side.
// The Jacobi diagonal comes from the assembled operator's centre plane.  CG vectors in SMEM,
// lattice order.  Tensors: [row][colour][k][q][cell of colour] (coalesced), then
// [face][q] face weights FW_q kappa |nu| scale.
struct Q2T {
    double L[3][3], D[3][3];  // L[q][a] = l_a(s_q), D[q][a] = l_a'(s_q), Gauss-3 points
};
__constant__ Q2T cQ2T;

constexpr int kQ2tThreads = 256;

struct Q2tGeom {
    int nn0, nn1, nc0, nc1, cw[4], cnt[4], cbase[4];  // colour c = (ci & 1) + 2 (cj & 1)
};

__host__ __device__ __forceinline__ Q2tGeom q2t_geom(const GenGeom& g) {
    Q2tGeom q;
    q.nn0 = g.nn[0];
    q.nn1 = g.nn[1];
    q.nc0 = g.nc[0];
    q.nc1 = g.nc[1];
    int base = 0;
    for (int c = 0; c < 4; ++c) {
        const int a = c & 1, b = c >> 1;
        q.cw[c] = (q.nc0 + 1 - a) / 2;
        q.cnt[c] = q.cw[c] * ((q.nc1 + 1 - b) / 2);
        q.cbase[c] = base;
        base += 36 * q.cnt[c];
    }
    return q;
}

// y_e = K_e p_e for one cell: p[a1][a0] element values, T = the cell's tensors
// (T0 T1 T2 T3 at stride `cs`, q = q0 + 3 q1).
__device__ __forceinline__ void q2t_cell(const double (&p)[3][3], const double* __restrict__ T, int cs,
                                         double (&y)[3][3]) {
    double u[3][3], du[3][3];
#pragma unroll
    for (int a1 = 0; a1 < 3; ++a1)
#pragma unroll
        for (int q0 = 0; q0 < 3; ++q0) {
            u[a1][q0] = cQ2T.L[q0][0] * p[a1][0] + cQ2T.L[q0][1] * p[a1][1] + cQ2T.L[q0][2] * p[a1][2];
            du[a1][q0] = cQ2T.D[q0][0] * p[a1][0] + cQ2T.D[q0][1] * p[a1][1] + cQ2T.D[q0][2] * p[a1][2];
        }
    double f0[3][3], f1[3][3], sv[3][3];
#pragma unroll
    for (int q1 = 0; q1 < 3; ++q1)
#pragma unroll
        for (int q0 = 0; q0 < 3; ++q0) {
            const double v = cQ2T.L[q1][0] * u[0][q0] + cQ2T.L[q1][1] * u[1][q0] + cQ2T.L[q1][2] * u[2][q0];
            const double g0 = cQ2T.L[q1][0] * du[0][q0] + cQ2T.L[q1][1] * du[1][q0] + cQ2T.L[q1][2] * du[2][q0];
            const double g1 = cQ2T.D[q1][0] * u[0][q0] + cQ2T.D[q1][1] * u[1][q0] + cQ2T.D[q1][2] * u[2][q0];
            const int q = q0 + 3 * q1;
            const double t0 = __ldg(T + (0 * 9 + q) * cs), t1 = __ldg(T + (1 * 9 + q) * cs);
            const double t2 = __ldg(T + (2 * 9 + q) * cs), t3 = __ldg(T + (3 * 9 + q) * cs);
            f0[q1][q0] = t0 * g0 + t1 * g1;
            f1[q1][q0] = t1 * g0 + t2 * g1;
            sv[q1][q0] = t3 * v;
        }
    double X[3][3], Y[3][3];
#pragma unroll
    for (int a1 = 0; a1 < 3; ++a1)
#pragma unroll
        for (int q0 = 0; q0 < 3; ++q0) {
            X[a1][q0] = cQ2T.L[0][a1] * f0[0][q0] + cQ2T.L[1][a1] * f0[1][q0] + cQ2T.L[2][a1] * f0[2][q0];
            Y[a1][q0] = cQ2T.D[0][a1] * f1[0][q0] + cQ2T.D[1][a1] * f1[1][q0] + cQ2T.D[2][a1] * f1[2][q0] +
                        cQ2T.L[0][a1] * sv[0][q0] + cQ2T.L[1][a1] * sv[1][q0] + cQ2T.L[2][a1] * sv[2][q0];
        }
#pragma unroll
    for (int a1 = 0; a1 < 3; ++a1)
#pragma unroll
        for (int a0 = 0; a0 < 3; ++a0)
            y[a1][a0] = cQ2T.D[0][a0] * X[a1][0] + cQ2T.D[1][a0] * X[a1][1] + cQ2T.D[2][a0] * X[a1][2] +
                        cQ2T.L[0][a0] * Y[a1][0] + cQ2T.L[1][a0] * Y[a1][1] + cQ2T.L[2][a0] * Y[a1][2];
}

// Boundary nodes' Robin face mass rows (assembly.cpp:149-169): node (i, j) on side(s) of
// the lattice gathers over the <= 2 faces per side that contain it, sides in face order.
__device__ __forceinline__ double q2t_face_row(const GenGeom& g, const int* role, const double* __restrict__ F,
                                               const double* __restrict__ src, int i, int j) {
    double acc = 0.0;
    const int ii[2] = {i, j};
#pragma unroll
    for (int axis = 0; axis < 2; ++axis)
#pragma unroll
        for (int side = 0; side < 2; ++side) {
            if (ii[axis] != (side ? g.nn[axis] - 1 : 0)) continue;
            if (role[2 * axis + side] == TS_GAMMA_N) continue;
            const int tr = 1 - axis, it = ii[tr];
            int t0 = it > 0 ? (it - 1) / 2 : 0, t1 = it / 2;
            if (t1 > g.nc[tr] - 1) t1 = g.nc[tr] - 1;
            for (int t = t0; t <= t1; ++t) {
                const int f = g.face_off[axis] + 2 * t + side, a = it - 2 * t;
                double row = 0.0;
#pragma unroll
                for (int b = 0; b < 3; ++b) {
                    double kab = 0.0;
#pragma unroll
                    for (int q = 0; q < 3; ++q) kab += __ldg(F + f * 3 + q) * cGP.Nf[q][a] * cGP.Nf[q][b];
                    const int lb = 2 * t + b;
                    const int node = axis == 0 ? (side ? g.nn[0] - 1 : 0) + g.nn[0] * lb : lb + g.nn[0] * (side ? g.nn[1] - 1 : 0);
                    row = fma(kab, src[node], row);
                }
                acc += row;
            }
        }
    return acc;
}

__global__ void __launch_bounds__(kQ2tThreads, 1) k_gen_pcg_q2t(const GenPcgArgs a) {
    extern __shared__ double smem[];
    const GenGeom& g = a.g;
    const Q2tGeom q = q2t_geom(g);
    const int n = g.nnodes, nn0 = q.nn0;
    double* sp = smem;
    double* sx = sp + n;
    double* sr = sx + n;
    double* sd = sr + n;
    double* sy = sd + n;
    double* red = sy + n;
    int* sTicket = reinterpret_cast<int*>(red + 3 * kRedStride);
    const int tid = threadIdx.x;
    const int CDIR = 12;  // centre of the 5 x 5 direction set
    for (;;) {
        __syncthreads();
        if (tid == 0) *sTicket = atomicAdd(a.counter, 1);
        __syncthreads();
        const int Pb = *sTicket;
        if (Pb >= a.n_problems) break;
        const double* T = a.tensor + (size_t)Pb * a.tensor_stride;
        const double* F = T + 36 * (size_t)g.ncells;
        const double* st = a.stencil + (size_t)Pb * a.stencil_stride;
        const double uP = a.u[Pb], wP = a.w[Pb];
        const bool use_u = a.kappa1 != 0.0 && uP != 0.0, use_w = a.kappa3 != 0.0 && wP != 0.0;
        const double cu = a.kappa1 * uP, cw = a.kappa3 * wP;
        const size_t vrow = (size_t)Pb * n;
        // y = A src (colours in order, then the boundary face rows); ends with a barrier
        auto apply = [&](const double* src, double* y) {
            for (int k = tid; k < n; k += blockDim.x) y[k] = 0.0;
            __syncthreads();
#pragma unroll 1
            for (int c = 0; c < 4; ++c) {
                const int ca = c & 1, cb = c >> 1;
                for (int l = tid; l < q.cnt[c]; l += blockDim.x) {
                    const int ci = 2 * (l % q.cw[c]) + ca, cj = 2 * (l / q.cw[c]) + cb;
                    const int base = 2 * ci + nn0 * 2 * cj;
                    double pe[3][3], ye[3][3];
#pragma unroll
                    for (int a1 = 0; a1 < 3; ++a1)
#pragma unroll
                        for (int a0 = 0; a0 < 3; ++a0) pe[a1][a0] = src[base + a0 + nn0 * a1];
                    q2t_cell(pe, T + q.cbase[c] + l, q.cnt[c], ye);
#pragma unroll
                    for (int a1 = 0; a1 < 3; ++a1)
#pragma unroll
                        for (int a0 = 0; a0 < 3; ++a0) y[base + a0 + nn0 * a1] += ye[a1][a0];
                }
                __syncthreads();
            }
            const int nb = 2 * (q.nn0 + q.nn1) - 4;  // boundary nodes, walked around the lattice
            for (int k = tid; k < nb; k += blockDim.x) {
                int i, j;
                if (k < q.nn0) { i = k; j = 0; }
                else if (k < 2 * q.nn0) { i = k - q.nn0; j = q.nn1 - 1; }
                else if (k < 2 * q.nn0 + q.nn1 - 2) { i = 0; j = k - 2 * q.nn0 + 1; }
                else { i = q.nn0 - 1; j = k - (2 * q.nn0 + q.nn1 - 2) + 1; }
                y[i + nn0 * j] += q2t_face_row(g, a.role, F, src, i, j);
            }
            __syncthreads();
        };
        for (int k = tid; k < n; k += blockDim.x) {
            const double dg = __ldg(st + k);  // plane 0 = the centre direction
            sd[k] = dg != 0.0 ? 1.0 / dg : 1.0;
            double bk = 0.0;
            if (use_u) bk = fma(cu, __ldg(a.rin + vrow + k), bk);
            if (use_w) bk = fma(cw, __ldg(a.rout + vrow + k), bk);
            sr[k] = bk;
            const double x0 = a.warm ? a.V[vrow + k] : 0.0;
            sx[k] = x0;
            sp[k] = x0;
        }
        __syncthreads();
        apply(sp, sy);
        double s3[3] = {0.0, 0.0, 0.0};
        for (int k = tid; k < n; k += blockDim.x) {
            const double bk = sr[k];
            s3[0] = fma(bk, bk, s3[0]);
            const double r = bk - sy[k];
            sr[k] = r;
            const double z = sd[k] * r;
            sy[k] = z;
            s3[1] = fma(r, z, s3[1]);
            s3[2] = fma(r, r, s3[2]);
        }
        block_sum<3>(s3, red);
        int slot = 1;
        const double bnorm = sqrt(s3[0]);
        int status = 0, iters = 0;
        double rel = 0.0;
        if (bnorm == 0.0) {
            for (int k = tid; k < n; k += blockDim.x) sx[k] = 0.0;
        } else {
            double rz = s3[1];
            rel = sqrt(s3[2]) / bnorm;
            if (rel > a.tol) {
                const double thr = rel_threshold(bnorm, a.tol);
                double rr_last = s3[2];
                for (int k = tid; k < n; k += blockDim.x) sp[k] = sy[k];
                __syncthreads();
                status = 2;
                for (int it = 1; it <= a.maxit; ++it) {
                    apply(sp, sy);
                    double t1[1] = {0.0};
                    for (int k = tid; k < n; k += blockDim.x) t1[0] = fma(sp[k], sy[k], t1[0]);
                    const double yrz = div_recip(rz);
                    block_sum<1>(t1, red + slot * kRedStride);
                    slot = slot == 2 ? 0 : slot + 1;
                    iters = it;
                    if (t1[0] <= 0.0) {
                        status = 1;
                        break;
                    }
                    const double alpha = rz / t1[0];
                    double t2[2] = {0.0, 0.0};
                    for (int k = tid; k < n; k += blockDim.x) {
                        const double r = fma(-alpha, sy[k], sr[k]);
                        sr[k] = r;
                        const double z = sd[k] * r;
                        sy[k] = z;
                        t2[0] = fma(r, r, t2[0]);
                        t2[1] = fma(r, z, t2[1]);
                    }
                    block_sum<2>(t2, red + slot * kRedStride);
                    slot = slot == 2 ? 0 : slot + 1;
                    rr_last = t2[0];
                    const bool done = t2[0] <= thr;
                    const double beta = div_finish(t2[1], rz, yrz);
                    rz = t2[1];
                    for (int k = tid; k < n; k += blockDim.x) {
                        const double pv = sp[k];
                        sx[k] = fma(alpha, pv, sx[k]);
                        if (!done) sp[k] = fma(beta, pv, sy[k]);
                    }
                    if (done) {
                        status = 0;
                        break;
                    }
                    __syncthreads();
                }
                rel = sqrt(rr_last) / bnorm;
            }
        }
        for (int k = tid; k < n; k += blockDim.x) a.V[vrow + k] = sx[k];
        if (a.epilogue) {
            __syncthreads();
            apply(sx, sy);
            double t1[1] = {0.0};
            for (int k = tid; k < n; k += blockDim.x) {
                double bk = 0.0;
                if (use_u) bk = fma(cu, __ldg(a.rin + vrow + k), bk);
                if (use_w) bk = fma(cw, __ldg(a.rout + vrow + k), bk);
                const double rr = bk - sy[k];
                t1[0] = fma(rr, rr, t1[0]);
            }
            block_sum<1>(t1, red + slot * kRedStride);
            const int warp = tid >> 5, lane = tid & 31;
            for (int rw = warp; rw < 2; rw += (int)(blockDim.x >> 5)) {
                const int role = rw == 0 ? TS_GAMMA_I : TS_GAMMA_O;
                const double* len = a.face_len + (size_t)Pb * a.face_len_stride;
                double tot = 0.0;
                for (int f = lane; f < g.nfaces; f += 32) {
                    int axis, side, cc[3], tr[2];
                    gen_face(g, f, axis, side, cc, tr);
                    if (a.role[2 * axis + side] != role) continue;
                    double y[3], sc, nrm[3];
                    gen_face_geom(g, cGP, axis, side, cc, 0, y, sc, nrm);
                    for (int qq = 0; qq < g.nqf; ++qq) {
                        double vq = 0.0;
                        for (int fa = 0; fa < g.npf; ++fa)
                            vq = fma(sx[gen_face_node(g, axis, side, cc, tr, fa)], cGP.Nf[qq][fa], vq);
                        tot += cGP.FW[qq] * vq * len[(size_t)f * g.nqf + qq] * sc;
                    }
                }
                tot = warp_sum(tot);
                if (lane == 0) (rw == 0 ? a.bI : a.bO)[Pb] = tot;
            }
            if (tid == 0) a.res_v[Pb] = sqrt(t1[0]);
        }
        if (tid == 0) {
            a.iters[Pb] = iters;
            a.status[Pb] = status;
            a.final_rel[Pb] = rel;
        }
    }
}

// ------------------------------- 2D Q2, class-compact operator on a 2-CTA cluster --
// Config 4's class-compact operator (§4 (3')) halved by symmetry — each node stores only
// its upper directions (dy > 0, or dy = 0 and dx >= 0: 13 / 8 / 8 / 5 per class), the
// lower ones are the neighbours' (a_{-d}(k) = a_d(k + d)) — is 0.29 MB per problem: it
// stays in the shared memory of a 2-CTA cluster for the whole solve (CTA r owns lattice rows
// [0, JS) / [JS, NN), plus one class row of coefficients below).  No global loads remain in
// the iteration (the streaming kernel is L2-latency bound: long_scoreboard 33 %, L1TEX 74 %).
// p: four class planes per CTA with one halo class row above and below and a zero column on
// each side; slots run over the padded planes at the plane pitch, class-major and
// warp-aligned, so every access of a warp is one contiguous run.  CG vectors in registers.
// Halo rows and dot products travel by st.async + transaction mbarriers (as the z-column
// kernel).  Single-reduction (Chronopoulos-Gear) loop or the two-reduction loop (CG1).
constexpr int kQcCL = 2;
constexpr int kQcThreads = 512;
constexpr int kQcKMClass = 5;  // slots per thread of the class-per-warp mapping

__host__ __device__ constexpr int qc_floor2(int v) { return v >= 0 ? v / 2 : -((1 - v) / 2); }

// index of direction (dx, dy) in class (A, B)'s upper set: dy = 0: dx = 0..Lx, then
// dy = 1..Ly: dx = -Lx..Lx
__host__ __device__ constexpr int qc_ue(int A, int B, int dx, int dy) {
    return dy == 0 ? dx : ((A ? 1 : 2) + 1) + (dy - 1) * (2 * (A ? 1 : 2) + 1) + dx + (A ? 1 : 2);
}
__host__ __device__ constexpr int qc_nu(int A, int B) { return ((A ? 1 : 2) + 1) + (B ? 1 : 2) * (2 * (A ? 1 : 2) + 1); }

// Block mapping: thread t -> (pair row t / TP, column t % TP).  Consecutive lanes must hit
// consecutive SMEM words also across a pair-row break (the next pair row starts 2 PPI
// further), or a straddling half-warp sees 2-way bank conflicts (ncu: 30 % of the
// wavefronts with PPI = 35, TP = 35): 2 PPI - (TP - 1) = 1 (mod 16), i.e. TP = 2 PPI (mod 16).
__host__ __device__ constexpr int qb_tp(int ppi, int ci0) {
    int tp = ci0;
    while ((2 * ppi - tp) % 16 != 0) ++tp;
    return tp;
}
// plane pitch of the block mapping: the pitch >= CI0 + 2 whose TP needs the fewest warps
__host__ __device__ constexpr int qb_ppi(int ci0, int pair_rows) {
    int best = ci0 + 2, best_w = 1 << 30;
    for (int ppi = ci0 + 2; ppi < ci0 + 18; ++ppi) {
        const int w = (pair_rows * qb_tp(ppi, ci0) + 31) / 32;
        if (w < best_w) {
            best_w = w;
            best = ppi;
        }
    }
    return best;
}

template <int NN, bool BLK = false>
struct QcGeom {
    static constexpr int CI0 = (NN + 1) / 2, CI1 = NN / 2;  // class columns / rows, parity 0 / 1
    static constexpr int JS = (NN / 2) & ~1;                // rank 0: lattice rows [0, JS)
    static constexpr int PAIRS = (CI0 - JS / 2 + 1) / 2;    // block mapping: pair rows (rank 1 has the most)
    static constexpr int PPI = BLK ? qb_ppi(CI0, PAIRS) : CI0 + 2;  // plane pitch
    static constexpr int TP = qb_tp(PPI, CI0);              // block mapping: thread-row pitch
    static constexpr int THREADS = BLK ? ((PAIRS * TP + 31) / 32) * 32 : kQcThreads;
    static constexpr int RP = (CI0 - JS / 2) + 2;           // p rows per plane (max own class rows + halos)
    static constexpr int RA = (CI0 - JS / 2) + 1;           // coefficient rows per plane (+ the row below)
    static constexpr int PPL = RP * PPI, APL = RA * PPI;
    static constexpr int NU = qc_nu(0, 0) + qc_nu(1, 0) + qc_nu(0, 1) + qc_nu(1, 1);  // 34
    static constexpr int GUARD = PPI + 2;
    static constexpr int PD = 4 * PPL + 2 * GUARD;
    static constexpr int AD = NU * APL + 2 * GUARD;
    static constexpr size_t SMEM =
        ((size_t)PD + AD + kGcSlots * 32 * 4 + kGcSlots * 16 * 4 + kGcSlots + 1 + 2) * sizeof(double);
};

__host__ __device__ __forceinline__ void qc_rows(int NN, int JS, int rank, int b, int& jb0, int& jb1) {
    const int J0 = rank ? JS : 0, J1 = rank ? NN : JS;
    jb0 = (J0 - b + 1) / 2;
    jb1 = (J1 - b + 1) / 2;
}

// y_k for a slot of class (A, B) at class position q = jj * PPI + ii; pb / ab: per-class
// plane bases (runtime, one per class), everything else compile-time
template <int NN, int A, int B>
__device__ __forceinline__ double qc_spmv(const double* __restrict__ sP, const double* __restrict__ sA,
                                          const int (&pb)[4], const int (&ab)[4], int q) {
    using G = QcGeom<NN, false>;
    constexpr int Lx = A ? 1 : 2, Ly = B ? 1 : 2, C = A + 2 * B;
    double acc[3] = {0.0, 0.0, 0.0};
#pragma unroll
    for (int dy = -Ly; dy <= Ly; ++dy)
#pragma unroll
        for (int dx = -Lx; dx <= Lx; ++dx) {
            const int A2 = (A + dx) & 1, B2 = (B + dy) & 1, C2 = A2 + 2 * B2;
            const int off = qc_floor2(B + dy) * G::PPI + qc_floor2(A + dx);
            const double pv = sP[pb[C2] + q + off];
            const bool upper = dy > 0 || (dy == 0 && dx >= 0);
            const double cf = upper ? sA[ab[C] + qc_ue(A, B, dx, dy) * G::APL + q]
                                    : sA[ab[C2] + qc_ue(A2, B2, -dx, -dy) * G::APL + q + off];
            acc[dy + Ly < 3 ? (dy + Ly) % 3 : 2] = fma(cf, pv, acc[dy + Ly < 3 ? (dy + Ly) % 3 : 2]);
        }
    return (acc[0] + acc[1]) + acc[2];
}

// Block mapping (BLK): a thread owns the eight nodes of two vertically adjacent 2x2 node blocks
// of the Q2 lattice — lattice columns X, X+1 and rows Y..Y+3 (X = 2 bi, Y = 2 bj):
// two nodes of every parity class, so every thread has the same work (the class-per-warp
// mapping leaves the vertex-class warps with 25 products per node against 9 for interiors).
// The eight coupling boxes overlap: their union is 5 x 7 lattice nodes, of which the eight
// own values are already in registers (27 p loads for 8 nodes instead of 128), and the 20
// couplings between two own nodes load their coefficient once (108 instead of 128): 16.9
// LDS.64 per node against 32.  Rows are walked bottom to top so only one 5-wide p row is
// live.  Node n = 2 ay + ax, ax = 0/1, ay = 0..3; class (ax, ay & 1), class position
// (bi, bj + (ay >> 1)).
constexpr int kQbKM = 8;

template <int NN, unsigned MASK = 0xffu>
__device__ __forceinline__ void qb_spmv(const double* __restrict__ sP, const double* __restrict__ sA,
                                        const int (&pb)[4], const int (&ab)[4], int q0,
                                        const double (&pin)[kQbKM], double (&y)[kQbKM]) {
    using G = QcGeom<NN, true>;
    constexpr int PPI = G::PPI;
    double acc[kQbKM];
#pragma unroll
    for (int n = 0; n < kQbKM; ++n) acc[n] = 0.0;
#pragma unroll
    for (int ry = -2; ry <= 4; ++ry) {
        double pr[5];
#pragma unroll
        for (int cx = -2; cx <= 2; ++cx) {
            const bool own = ry >= 0 && ry <= 3 && cx >= 0 && cx <= 1;
            const int C2 = (cx & 1) + 2 * (ry & 1);
            pr[cx + 2] = own ? pin[own ? 2 * ry + cx : 0] : sP[pb[C2] + q0 + qc_floor2(ry) * PPI + qc_floor2(cx)];
        }
#pragma unroll
        for (int n = 0; n < kQbKM; ++n) {
            const int ax = n & 1, ay = n >> 1, A = ax, B = ay & 1, C = A + 2 * B;
            const int Lx = A ? 1 : 2, Ly = B ? 1 : 2, dy = ry - ay;
            if (!((MASK >> n) & 1u) || dy < -Ly || dy > Ly) continue;
#pragma unroll
            for (int cx = -2; cx <= 2; ++cx) {
                const int dx = cx - ax;
                if (dx < -Lx || dx > Lx) continue;
                const int A2 = cx & 1, B2 = ry & 1, C2 = A2 + 2 * B2;
                const bool upper = dy > 0 || (dy == 0 && dx >= 0);
                const double cf = upper ? sA[ab[C] + qc_ue(A, B, dx, dy) * G::APL + q0 + (ay >> 1) * PPI]
                                        : sA[ab[C2] + qc_ue(A2, B2, -dx, -dy) * G::APL + q0 + qc_floor2(ry) * PPI +
                                             qc_floor2(cx)];
                acc[n] = fma(cf, pr[cx + 2], acc[n]);
            }
        }
    }
#pragma unroll
    for (int n = 0; n < kQbKM; ++n) y[n] = acc[n];
}

template <int NN, bool CG1, bool BLK>
__global__ void __launch_bounds__(QcGeom<NN, BLK>::THREADS, 1) k_gen_pcg_q2c(const GenPcgArgs a) {
    using G = QcGeom<NN, BLK>;
    constexpr int PPI = G::PPI;
    constexpr int kQcKM = BLK ? kQbKM : kQcKMClass;
    // per-class values are selected with compile-time indices only, so the small arrays stay
    // in registers (a runtime index would put them in local memory, read by every SpMV)
    auto sel = [](const int (&v)[4], int c) { return c == 0 ? v[0] : c == 1 ? v[1] : c == 2 ? v[2] : v[3]; };
    extern __shared__ double smem[];
    cg::cluster_group cl = cg::this_cluster();
    const int rank = (int)cl.block_rank(), other = 1 - rank;
    const GenGeom& g = a.g;
    const Q2Geom q2 = q2_geom(g);
    const int n = g.nnodes;
    double* sP = smem + G::GUARD;
    double* sA = smem + G::PD + G::GUARD;
    double* red = smem + G::PD + G::AD;
    double* xch = red + kGcSlots * 32 * 4;
    unsigned long long* sBar = reinterpret_cast<unsigned long long*>(xch + kGcSlots * 16 * 4);
    unsigned long long* hBar = sBar + kGcSlots;
    int* sTicket = reinterpret_cast<int*>(hBar + 1);
    const int tid = threadIdx.x;
    // per-class geometry of this CTA and of the other one
    int jb0[4], jb1[4], pb[4], ab[4], pbo[4];
    {
        int abase = 0;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int b = c >> 1;
            int o0, o1;
            qc_rows(NN, G::JS, rank, b, jb0[c], jb1[c]);
            qc_rows(NN, G::JS, other, b, o0, o1);
            pb[c] = c * G::PPL - (jb0[c] - 1) * PPI + 1;
            pbo[c] = c * G::PPL - (o0 - 1) * PPI + 1;
            ab[c] = abase - (jb0[c] - 1) * PPI + 1;
            abase += qc_nu(c & 1, c >> 1) * G::APL;
        }
    }
    // Class mapping: the thread's slots are all of one class: warp w serves class w / 4 and
    // takes that class's 32-slot chunks (w % 4) * KM .. + KM - 1, so the SpMV dispatches on the
    // class once and runs the KM slots as one compile-time loop (loads of all slots in flight
    // together).  Block mapping (BLK): see qb_spmv; slot m = node 2 ay + ax of the block pair.
    const int wcls = BLK ? 0 : (tid >> 5) >> 2;
    int qpos_[kQcKM], node_[kQcKM];
    bool live_[kQcKM];
    int q0 = 0, node0 = 0;  // BLK: class position / lattice node of the pair's first block
    // BLK: bits 0-7 live(m), bits 8-15 node m is on the boundary class row (sent to the peer),
    // bits 16-17 the nodes any lane of this warp holds (3: full blocks, 1: nodes 0, 1 only — the
    // single first lattice row of an odd class-row count —, 0: none)
    unsigned flags = 0;
    if constexpr (BLK) {
        const int row = tid / G::TP, bi = tid % G::TP;
        const bool in = row < G::PAIRS;  // threads past the last pair row: dead, parked on pair row 0
        const int bjr = jb0[0] + 2 * (in ? row : 0);
        q0 = bjr * PPI + bi;
        node0 = 2 * bi + NN * 2 * bjr;
#pragma unroll
        for (int m = 0; m < kQcKM; ++m) {
            const int c = (m & 1) + 2 * ((m >> 1) & 1), jj = bjr + (m >> 2);
            const bool lv = in && bi < ((m & 1) ? G::CI1 : G::CI0) && jj < jb1[c];
            const int brow = rank ? jb0[c] : jb1[c] - 1;
            if (lv) flags |= 1u << m;
            if (lv && jj == brow) flags |= 0x100u << m;
        }
        const bool any_hi = __any_sync(0xffffffffu, (flags & 0xfcu) != 0);
        const bool any_lo = __any_sync(0xffffffffu, (flags & 0x03u) != 0);
        flags |= (any_hi ? 3u : any_lo ? 1u : 0u) << 16;
    } else {
#pragma unroll
        for (int m = 0; m < kQcKM; ++m) {
            const int c = wcls;
            const int w = 32 * (((tid >> 5) & 3) * kQcKM + m) + (tid & 31);
            const int row = w / PPI, col = w % PPI, ii = col - 1, jj = sel(jb0, c) + row;
            const int A = c & 1, B = c >> 1, ci = A ? G::CI1 : G::CI0;
            live_[m] = jj < sel(jb1, c) && ii >= 0 && ii < ci;
            qpos_[m] = live_[m] ? jj * PPI + ii : 0;
            node_[m] = live_[m] ? (2 * ii + A) + NN * (2 * jj + B) : 0;
        }
    }
    // slot accessors (m is a compile-time index after unrolling)
    auto cls = [&](int m) { return BLK ? (m & 1) + 2 * ((m >> 1) & 1) : wcls; };
    auto live = [&](int m) {
        if constexpr (BLK)
            return ((flags >> m) & 1u) != 0;
        else
            return live_[m];
    };
    auto qpos = [&](int m) { return BLK ? q0 + (m >> 2) * PPI : qpos_[m]; };
    auto node = [&](int m) { return BLK ? node0 + (m & 1) + NN * (m >> 1) : node_[m]; };
    const int nbr_bytes = 8 * (G::CI0 + G::CI1 + G::CI0 + G::CI1);  // one class row per class
    if (tid <= kGcSlots) gc_mbar_init(sBar + tid, 1);
    if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int k = tid; k < G::PD + G::AD + kGcSlots * 32 * 4; k += blockDim.x) smem[k] = 0.0;  // + red (exchange entries)
    __syncthreads();
    if (tid == 0) zc_expect(hBar, nbr_bytes);
    unsigned phase = 0, hphase = 0;
    int slot = 0;
    auto csum_with = [&](auto& v, auto between) {
        if constexpr (BLK && G::THREADS / 32 <= 32 / kQcCL)
            zc_cluster_sum_direct<sizeof(v) / sizeof(double), kQcCL>(v, red + slot * 128, sBar + slot,
                                                                     (phase >> slot) & 1u, rank, between);
        else
            zc_cluster_sum<sizeof(v) / sizeof(double), kQcCL>(v, red + slot * 128, xch + slot * 64, sBar + slot,
                                                              (phase >> slot) & 1u, rank, between);
        phase ^= 1u << slot;
        slot = slot == kGcSlots - 1 ? 0 : slot + 1;
    };
    auto csum = [&](auto& v) { csum_with(v, ZcNoop()); };
    // own values into the class planes, the boundary class row into the other CTA's halo
    auto publish = [&](const double (&v)[kQcKM]) {
        if constexpr (BLK) {
            // predicated stores (no branches), then the sends of the one boundary pair row
#pragma unroll
            for (int m = 0; m < kQcKM; ++m)
                if (live(m)) sP[pb[cls(m)] + qpos(m)] = v[m];
            if (flags & 0xff00u) {
                const unsigned rb = zc_mapa(hBar, other);
#pragma unroll
                for (int m = 0; m < kQcKM; ++m)
                    if ((flags >> (8 + m)) & 1u) zc_st_async(zc_mapa(sP + pbo[cls(m)] + qpos(m), other), v[m], rb);
            }
        } else {
#pragma unroll
            for (int m = 0; m < kQcKM; ++m) {
                if (!live(m)) continue;
                const int c = cls(m);
                const int brow = rank ? sel(jb0, c) : sel(jb1, c) - 1;
                sP[sel(pb, c) + qpos(m)] = v[m];
                if (qpos(m) / PPI == brow)
                    zc_st_async(zc_mapa(sP + sel(pbo, c) + qpos(m), other), v[m], zc_mapa(hBar, other));
            }
        }
        __syncthreads();
    };
    auto hwait = [&] {
        zc_wait(hBar, hphase);
        hphase ^= 1u;
        if (tid == 0) zc_expect(hBar, nbr_bytes);
    };
    // y = A v for the vector v the last publish stored (BLK reads its own entries from v)
    auto spmv = [&](double (&y)[kQcKM], const double (&v)[kQcKM]) {
        hwait();
        if constexpr (BLK) {
            // warp-uniform: the last pair row of an odd class-row count holds only its first
            // lattice row (nodes 0, 1); warps past the last pair row hold nothing
            if ((flags >> 17) & 1u)
                qb_spmv<NN, 0xffu>(sP, sA, pb, ab, q0, v, y);
            else if ((flags >> 16) & 1u)
                qb_spmv<NN, 0x03u>(sP, sA, pb, ab, q0, v, y);
#pragma unroll
            for (int m = 0; m < kQcKM; ++m)
                if (!live(m)) y[m] = 0.0;
        } else {
            auto run = [&](auto A_, auto B_) {
#pragma unroll
                for (int m = 0; m < kQcKM; ++m)
                    y[m] = live(m) ? qc_spmv<NN, decltype(A_)::value, decltype(B_)::value>(sP, sA, pb, ab, qpos(m))
                                   : 0.0;
            };
            switch (wcls) {  // warp-uniform
                case 0: run(std::integral_constant<int, 0>{}, std::integral_constant<int, 0>{}); break;
                case 1: run(std::integral_constant<int, 1>{}, std::integral_constant<int, 0>{}); break;
                case 2: run(std::integral_constant<int, 0>{}, std::integral_constant<int, 1>{}); break;
                default: run(std::integral_constant<int, 1>{}, std::integral_constant<int, 1>{}); break;
            }
        }
    };

    cl.sync();
    if (rank == 0 && tid == 0) {
        const int t = atomicAdd(a.counter, 1);
        for (int q = 0; q < kQcCL; ++q) cl.map_shared_rank(sTicket, q)[1] = t;
    }
    for (;;) {
        if (rank == 0 && tid == 0) {
            const int cur = sTicket[1];
            const int nxt = cur < a.n_problems ? atomicAdd(a.counter, 1) : cur;
            for (int q = 0; q < kQcCL; ++q) {
                int* t = cl.map_shared_rank(sTicket, q);
                t[0] = cur;
                t[1] = nxt;
            }
        }
        cl.sync();
        const int Pb = sTicket[0];
        if (Pb >= a.n_problems) break;
        const double* qs = a.qstencil + (size_t)Pb * a.qstencil_stride;
        // upper-direction coefficient planes, own class rows + one below
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const int A = c & 1, B = c >> 1, Lx = A ? 1 : 2, Ly = B ? 1 : 2, ci = A ? G::CI1 : G::CI0;
            const int r0 = max(0, jb0[c] - 1), nr = jb1[c] - r0, nu = qc_nu(A, B);
            for (int t = tid; t < nu * nr * ci; t += blockDim.x) {
                const int e = t / (nr * ci), rr = (t / ci) % nr, ii = t % ci, jj = r0 + rr;
                const int dy = e <= Lx ? 0 : 1 + (e - (Lx + 1)) / (2 * Lx + 1);
                const int dx = e <= Lx ? e : (e - (Lx + 1)) % (2 * Lx + 1) - Lx;
                const int dd = (dy + Ly) * (2 * Lx + 1) + (dx + Lx);
                sA[ab[c] + e * G::APL + jj * PPI + ii] = __ldg(qs + q2.QB[c] + (size_t)dd * q2.nc[c] + ii + ci * jj);
            }
        }
        const double uP = a.u[Pb], wP = a.w[Pb];
        const bool use_u = a.kappa1 != 0.0 && uP != 0.0, use_w = a.kappa3 != 0.0 && wP != 0.0;
        const double cu = a.kappa1 * uP, cw = a.kappa3 * wP;
        const size_t vrow = (size_t)Pb * n;
        double x[kQcKM], r[kQcKM], dv[kQcKM], z[kQcKM];
#pragma unroll
        for (int m = 0; m < kQcKM; ++m) {
            x[m] = r[m] = z[m] = 0.0;
            dv[m] = 1.0;
            if (live(m)) {
                const int c = cls(m), A = c & 1, B = c >> 1, Lx = A ? 1 : 2, Ly = B ? 1 : 2;
                const int ci = A ? G::CI1 : G::CI0, ii = qpos(m) % PPI, jj = qpos(m) / PPI;
                const int QBc = c == 0 ? q2.QB[0] : c == 1 ? q2.QB[1] : c == 2 ? q2.QB[2] : q2.QB[3];
                const int NCc = c == 0 ? q2.nc[0] : c == 1 ? q2.nc[1] : c == 2 ? q2.nc[2] : q2.nc[3];
                const double dg = __ldg(qs + QBc + (size_t)(Ly * (2 * Lx + 1) + Lx) * NCc + ii + ci * jj);
                dv[m] = dg != 0.0 ? 1.0 / dg : 1.0;
                const int k = node(m);
                double bk = 0.0;
                if (use_u) bk = fma(cu, __ldg(a.rin + vrow + k), bk);
                if (use_w) bk = fma(cw, __ldg(a.rout + vrow + k), bk);
                r[m] = bk;
                x[m] = a.warm ? a.V[vrow + k] : 0.0;
            }
        }
        publish(x);  // (its CTA barrier also completes sA)
        double s3[3] = {0.0, 0.0, 0.0};
        {
            double y[kQcKM];
            spmv(y, x);
#pragma unroll
            for (int m = 0; m < kQcKM; ++m) {
                if (!live(m)) continue;
                const double bk = r[m];
                s3[0] = fma(bk, bk, s3[0]);
                r[m] = bk - y[m];
                z[m] = dv[m] * r[m];
                s3[1] = fma(r[m], z[m], s3[1]);
                s3[2] = fma(r[m], r[m], s3[2]);
            }
        }
        csum(s3);
        const double bnorm = sqrt(s3[0]);
        int status = 0, iters = 0;
        double rel = 0.0;
        if (bnorm == 0.0) {
#pragma unroll
            for (int m = 0; m < kQcKM; ++m) x[m] = 0.0;
        } else {
            double rz = s3[1];
            rel = sqrt(s3[2]) / bnorm;
            if (rel > a.tol && CG1) {  // single-reduction loop (as k_gen_pcg3_zcol)
                const double thr = rel_threshold(bnorm, a.tol);
                double rr_last = s3[2];
                double p[kQcKM], sv[kQcKM], w[kQcKM];
                double gamma = rz;
                publish(z);
                spmv(w, z);
                double t1[1] = {0.0};
#pragma unroll
                for (int m = 0; m < kQcKM; ++m) {
                    if (!live(m)) w[m] = 0.0;
                    t1[0] = fma(w[m], z[m], t1[0]);
                }
                csum(t1);
                status = 2;
                iters = 1;
                double pAp = t1[0], alpha = 0.0;
                if (pAp <= 0.0) {
                    status = 1;
                } else {
                    alpha = gamma / pAp;
#pragma unroll
                    for (int m = 0; m < kQcKM; ++m) {
                        p[m] = z[m];
                        sv[m] = w[m];
                    }
#ifdef TSB_PHASE_TIMING
                    long long ph[6] = {0, 0, 0, 0, 0, 0}, tc = clock64();
#define TSB_PH(i)                     \
    {                                 \
        const long long tn = clock64(); \
        ph[i] += tn - tc;             \
        tc = tn;                      \
    }
#else
#define TSB_PH(i)
#endif
                    for (int it = 1; it <= a.maxit; ++it) {
                        iters = it;
                        double t3[3] = {0.0, 0.0, 0.0};
#pragma unroll
                        for (int m = 0; m < kQcKM; ++m) {
                            x[m] = fma(alpha, p[m], x[m]);
                            r[m] = fma(-alpha, sv[m], r[m]);
                            z[m] = dv[m] * r[m];
                            t3[0] = fma(r[m], z[m], t3[0]);
                            t3[1] = fma(r[m], r[m], t3[1]);
                        }
                        TSB_PH(0)
                        publish(z);
                        TSB_PH(1)
                        spmv(w, z);
                        TSB_PH(2)
#pragma unroll
                        for (int m = 0; m < kQcKM; ++m) {
                            if (!live(m)) w[m] = 0.0;
                            t3[2] = fma(w[m], z[m], t3[2]);
                        }
                        // divisor-only parts of the two quotients whose divisors are known
                        // before the reduction (bitwise a / b, device_common.cuh)
                        // Scalars off the critical path, computed while the totals travel:
                        // p.Ap = delta - beta gamma' / alpha = delta - gamma'^2 c with
                        // c = 1 / (gamma alpha) from the previous iteration's values, and the
                        // divisor-only part of beta = gamma' / gamma (device_common.cuh).  After
                        // the exchange p.Ap is two dependent operations instead of two divisions.
                        double yg = 0.0, cinv = 0.0;
                        csum_with(t3, [&] {
                            yg = div_recip(gamma);
                            cinv = 1.0 / (gamma * alpha);
                        });
                        TSB_PH(3)
                        rr_last = t3[1];
                        if (t3[1] <= thr) {
                            status = 0;
                            break;
                        }
                        if (it == a.maxit) break;
                        const double beta = div_finish(t3[0], gamma, yg);
                        const bool fast = isfinite(cinv) && cinv != 0.0;  // gamma alpha neither under- nor overflowed
                        pAp = fast ? fma(-(t3[0] * t3[0]), cinv, t3[2]) : t3[2] - beta * t3[0] / alpha;
                        gamma = t3[0];
                        if (pAp <= 0.0) {
                            iters = it + 1;
                            status = 1;
                            break;
                        }
                        alpha = gamma / pAp;
#pragma unroll
                        for (int m = 0; m < kQcKM; ++m) {
                            p[m] = fma(beta, p[m], z[m]);
                            sv[m] = fma(beta, sv[m], w[m]);
                        }
                        TSB_PH(4)
                    }
#ifdef TSB_PHASE_TIMING
                    if (BLK && (tid == 0 || tid == 300) && Pb < 2 * (int)(gridDim.x / kQcCL) && Pb % 37 == 0)
                        printf("P %d rank %d tid %d iters %d: update %lld publish %lld spmv(+hwait) %lld dots+csum %lld scalars+ps %lld (cycles per iteration)\n",
                               Pb, rank, tid, iters, ph[0] / iters, ph[1] / iters, ph[2] / iters, ph[3] / iters, ph[4] / iters);
#endif
                }
                rel = sqrt(rr_last) / bnorm;
            } else if (rel > a.tol) {  // two-reduction loop, src/linalg.cpp:103-161 order
                const double thr = rel_threshold(bnorm, a.tol);
                double rr_last = s3[2];
                double p[kQcKM];
#pragma unroll
                for (int m = 0; m < kQcKM; ++m) p[m] = z[m];
                publish(p);
                status = 2;
                for (int it = 1; it <= a.maxit; ++it) {
                    double y[kQcKM];
                    spmv(y, p);
                    double t1[1] = {0.0};
#pragma unroll
                    for (int m = 0; m < kQcKM; ++m) {
                        z[m] = live(m) ? y[m] : 0.0;
                        t1[0] = fma(p[m], z[m], t1[0]);
                    }
                    const double yrz = div_recip(rz);
                    csum(t1);
                    iters = it;
                    if (t1[0] <= 0.0) {
                        status = 1;
                        break;
                    }
                    const double alpha = rz / t1[0];
                    double t2[2] = {0.0, 0.0};
#pragma unroll
                    for (int m = 0; m < kQcKM; ++m) {
                        r[m] = fma(-alpha, z[m], r[m]);
                        z[m] = dv[m] * r[m];
                        t2[0] = fma(r[m], r[m], t2[0]);
                        t2[1] = fma(r[m], z[m], t2[1]);
                    }
                    csum(t2);
                    rr_last = t2[0];
                    const bool done = t2[0] <= thr;
                    const double beta = div_finish(t2[1], rz, yrz);
                    rz = t2[1];
#pragma unroll
                    for (int m = 0; m < kQcKM; ++m) {
                        x[m] = fma(alpha, p[m], x[m]);
                        p[m] = fma(beta, p[m], z[m]);
                    }
                    if (done) {
                        status = 0;
                        break;
                    }
                    publish(p);
                }
                rel = sqrt(rr_last) / bnorm;
            }
        }
        // a publish not consumed (the two-reduction loop's last publish is always consumed;
        // every spmv waits on exactly one publish)
#pragma unroll
        for (int m = 0; m < kQcKM; ++m)
            if (live(m)) a.V[vrow + node(m)] = x[m];
        if (a.epilogue) {
            publish(x);
            double t3[3] = {0.0, 0.0, 0.0};
            {
                double y[kQcKM];
                spmv(y, x);
#pragma unroll
                for (int m = 0; m < kQcKM; ++m) {
                    if (!live(m)) continue;
                    const int k = node(m);
                    double bk = 0.0;
                    if (use_u) bk = fma(cu, __ldg(a.rin + vrow + k), bk);
                    if (use_w) bk = fma(cw, __ldg(a.rout + vrow + k), bk);
                    const double rr = bk - y[m];
                    t3[0] = fma(rr, rr, t3[0]);
                }
            }
            // surface_coupling (src/assembly.cpp:377-393): faces whose first node row this CTA owns
            const double* len = a.face_len + (size_t)Pb * a.face_len_stride;
            const int J0 = rank ? G::JS : 0, J1 = rank ? NN : G::JS;
            for (int f = tid; f < g.nfaces; f += blockDim.x) {
                int axis, side, cc[3], tr[2];
                gen_face(g, f, axis, side, cc, tr);
                const int role = a.role[2 * axis + side];
                if (role != TS_GAMMA_I && role != TS_GAMMA_O) continue;
                int lo = n;
                for (int fa = 0; fa < g.npf; ++fa) lo = min(lo, gen_face_node(g, axis, side, cc, tr, fa));
                if (lo / NN < J0 || lo / NN >= J1) continue;
                double yq[3], sc, nrm[3];
                gen_face_geom(g, cGP, axis, side, cc, 0, yq, sc, nrm);
                double tot = 0.0;
                for (int qq = 0; qq < g.nqf; ++qq) {
                    double vq = 0.0;
                    for (int fa = 0; fa < g.npf; ++fa) {
                        const int nd = gen_face_node(g, axis, side, cc, tr, fa);
                        const int i = nd % NN, j = nd / NN, c = (i & 1) + 2 * (j & 1);
                        vq = fma(sP[sel(pb, c) + (j >> 1) * PPI + (i >> 1)], cGP.Nf[qq][fa], vq);
                    }
                    tot += cGP.FW[qq] * vq * len[(size_t)f * g.nqf + qq] * sc;
                }
                t3[role == TS_GAMMA_I ? 1 : 2] += tot;
            }
            csum(t3);
            if (rank == 0 && tid == 0) {
                a.res_v[Pb] = sqrt(t3[0]);
                a.bI[Pb] = t3[1];
                a.bO[Pb] = t3[2];
            }
        }
        if (rank == 0 && tid == 0) {
            a.iters[Pb] = iters;
            a.status[Pb] = status;
            a.final_rel[Pb] = rel;
        }
        cl.sync();  // the next ticket's operator load overwrites SMEM the peer may still read
    }
}

template <int NN, bool BLK>
bool qc_launch_t(const GenPcgArgs& a, cudaStream_t s) {
    using G = QcGeom<NN, BLK>;
    const char* e = std::getenv("TS_GEN_CG1");
    const bool cg1 = !(e && e[0] == '0');
    auto kern = cg1 ? k_gen_pcg_q2c<NN, true, BLK> : k_gen_pcg_q2c<NN, false, BLK>;
    if (G::SMEM > 232448) return false;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(G::THREADS);
    cfg.dynamicSmemBytes = G::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = kQcCL;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(kQcCL);
    int nclusters = 0;
    if (cudaOccupancyMaxActiveClusters(&nclusters, kern, &cfg) != cudaSuccess || nclusters < 1) {
        cudaGetLastError();
        return false;
    }
    if (nclusters > a.n_problems) nclusters = a.n_problems;
    cfg.gridDim = dim3(kQcCL * nclusters);
    return cudaLaunchKernelEx(&cfg, kern, a) == cudaSuccess;
}

// 2-CTA cluster kernel for square Q2 lattices it is instantiated for (65: config 4; 41), with
// the class-compact operator available; TS_GEN_Q2CL=0 keeps the streaming kernel.
bool qc_launch(const GenPcgArgs& a, cudaStream_t s) {
    if (const char* e = std::getenv("TS_GEN_Q2CL"))
        if (e[0] == '0') return false;
    const GenGeom& g = a.g;
    if (g.d != 2 || g.p != 2 || g.nn[0] != g.nn[1] || !a.qstencil) return false;
    // TS_GEN_Q2B=0: the class-per-warp thread mapping instead of the block mapping
    const char* eb = std::getenv("TS_GEN_Q2B");
    const bool blk = !(eb && eb[0] == '0');
    if (g.nn[0] == 65) return (blk && qc_launch_t<65, true>(a, s)) || qc_launch_t<65, false>(a, s);
    if (g.nn[0] == 41) return (blk && qc_launch_t<41, true>(a, s)) || qc_launch_t<41, false>(a, s);
    return false;
}

size_t q2t_smem_bytes(const GenGeom& g) { return ((size_t)5 * g.nnodes + 3 * kRedStride) * sizeof(double) + 16; }

bool q2t_fits(const GenGeom& g) { return g.d == 2 && g.p == 2 && q2t_smem_bytes(g) <= 232448; }

size_t q2_smem_bytes(const GenGeom& g) {
    const Q2Geom q = q2_geom(g);
    return ((size_t)4 * q.PS + 4 * (size_t)q.KB[4] + 3 * kRedStride) * sizeof(double) + 16;
}

bool q2_fits(const GenGeom& g) {
    return g.d == 2 && g.p == 2 && q2_geom(g).KB[4] <= kQ2Slots * kThreadsG && q2_smem_bytes(g) <= 232448;
}

template <int DIM, int P>
void launch_dp(const GenPcgArgs& a, size_t smem, cudaStream_t s) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int grid = a.n_problems < sms ? a.n_problems : sms;
    if (grid > 148) grid = 148;  // the global-scratch variant is sized for 148 blocks
    if (DIM == 3 && P == 1 && zc_launch(a, s)) return;
    if (DIM == 3 && P == 1 && gc_fits(a.g, a.n_problems) && gc_launch(a, s)) return;
    if (DIM == 2 && P == 2 && a.tensor && q2t_fits(a.g)) {
        const size_t tsm = q2t_smem_bytes(a.g);
        cudaFuncSetAttribute(k_gen_pcg_q2t, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tsm);
        k_gen_pcg_q2t<<<grid, kQ2tThreads, tsm, s>>>(a);
        return;
    }
    if (DIM == 2 && P == 2 && qc_launch(a, s)) return;
    if (DIM == 2 && P == 2 && a.qstencil && q2_fits(a.g)) {
        const size_t qsm = q2_smem_bytes(a.g);
        cudaFuncSetAttribute(k_gen_pcg_q2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)qsm);
        k_gen_pcg_q2<<<grid, kThreadsG, qsm, s>>>(a);
        return;
    }
    if (smem <= 232448 && a.g.nnodes <= kMaxK * kThreadsG) {
        cudaFuncSetAttribute(k_gen_pcg<DIM, P, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        k_gen_pcg<DIM, P, false><<<grid, kThreadsG, smem, s>>>(a);
    } else {
        k_gen_pcg<DIM, P, true><<<grid, kThreadsG, 0, s>>>(a);
    }
}

__global__ void k_gcoupling(GenGeom g, int role, int r0, int r1, int r2, int r3, int r4, int r5, int n_vec,
                            const double* v, const double* len, long long len_stride, double* out) {
    const int roles[6] = {r0, r1, r2, r3, r4, r5};
    const int lane = threadIdx.x & 31;
    for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n_vec; i += gridDim.x * (blockDim.x >> 5)) {
        const double* vi = v + (size_t)i * g.nnodes;
        const double* li = len + (size_t)i * len_stride;
        double tot = 0.0;
        for (int f = lane; f < g.nfaces; f += 32) {
            int axis, side, cc[3], tr[2];
            gen_face(g, f, axis, side, cc, tr);
            if (roles[2 * axis + side] != role) continue;
            double y[3], sc, nrm[3];
            gen_face_geom(g, cGP, axis, side, cc, 0, y, sc, nrm);
            for (int q = 0; q < g.nqf; ++q) {
                double vq = 0.0;
                for (int fa = 0; fa < g.npf; ++fa) vq = fma(vi[gen_face_node(g, axis, side, cc, tr, fa)], cGP.Nf[q][fa], vq);
                tot += cGP.FW[q] * vq * li[(size_t)f * g.nqf + q] * sc;
            }
        }
        tot = warp_sum(tot);
        if (lane == 0) out[i] = tot;
    }
}

__global__ void k_gmicro_rhs(int n, const double* rin, const double* rout, double kappa1, double kappa3, double u,
                             double w, double* b) {
    const bool use_u = kappa1 != 0.0 && u != 0.0, use_w = kappa3 != 0.0 && w != 0.0;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        double bk = 0.0;
        if (use_u) bk = fma(kappa1 * u, rin[k], bk);
        if (use_w) bk = fma(kappa3 * w, rout[k], bk);
        b[k] = bk;
    }
}

}  // namespace

void upload_gen_tables_pcg(const GenTables& t) { cudaMemcpyToSymbol(cGP, &t, sizeof(GenTables)); }

size_t gen_pcg_smem_bytes(const GenGeom& g) {
    const PadGeom pg = pad_geom(g);
    return ((size_t)pg.Lp + 4 * (size_t)g.nnodes + 3 * kRedStride) * sizeof(double) + 16;
}

size_t gen_pcg_scratch_doubles(const GenGeom& g) {
    const size_t smem = gen_pcg_smem_bytes(g);
    if (smem <= 232448 && g.nnodes <= kMaxK * kThreadsG) return 0;
    const PadGeom pg = pad_geom(g);
    return 148 * ((size_t)pg.Lp + 4 * (size_t)g.nnodes);
}

size_t q2_tensor_doubles(const GenGeom& g) {
    const char* e = std::getenv("TS_GEN_Q2T");
    if (!(e && e[0] == '1') || !q2t_fits(g)) return 0;  // opt-in (DESIGN.md §4 (3'): measured choice)
    return (size_t)36 * g.ncells + 3 * (size_t)g.nfaces;
}

size_t q2_compact_doubles(const GenGeom& g) {
    if (!q2_fits(g)) return 0;
    if (const char* e = std::getenv("TS_GEN_Q2C"))
        if (e[0] == '0') return 0;
    return (size_t)q2_geom(g).QB[4];
}

void launch_q2_repack(const GenGeom& g, int rows, const double* stencil, double* qstencil, cudaStream_t s) {
    const long long total = (long long)rows * q2_geom(g).QB[4];
    long long b = (total + 255) / 256;
    if (b > 148LL * 64) b = 148LL * 64;
    k_q2_repack<<<(int)(b < 1 ? 1 : b), 256, 0, s>>>(g, rows, stencil, qstencil);
}

int launch_gen_pcg(const GenPcgArgs& a, cudaStream_t s) {
    const size_t smem = gen_pcg_smem_bytes(a.g);
    if (gen_pcg_scratch_doubles(a.g) && !a.scratch) return 0;
    if (a.g.d == 2 && a.g.p == 1) launch_dp<2, 1>(a, smem, s);
    else if (a.g.d == 2 && a.g.p == 2) launch_dp<2, 2>(a, smem, s);
    else if (a.g.d == 3 && a.g.p == 1) launch_dp<3, 1>(a, smem, s);
    else return 0;
    return 1;
}

void launch_gcoupling(const GenGeom& g, const int* role6, int role, int n_vec, const double* v, const double* len,
                      long long len_stride, double* out, cudaStream_t s) {
    k_gcoupling<<<(n_vec + 7) / 8, 256, 0, s>>>(g, role, role6[0], role6[1], role6[2], role6[3], role6[4], role6[5],
                                                n_vec, v, len, len_stride, out);
}

void launch_gmicro_rhs(int n, const double* rin, const double* rout, double kappa1, double kappa3, double u, double w,
                       double* b, cudaStream_t s) {
    k_gmicro_rhs<<<(n + 255) / 256, 256, 0, s>>>(n, rin, rout, kappa1, kappa3, u, w, b);
}

// ------------------------------------------------------------ host tables --
namespace {
void rule1d(int n, double* x, double* w) {
    if (n == 2) {
        const double gg = 1.0 / std::sqrt(3.0);
        x[0] = -gg; x[1] = gg;
        w[0] = 1.0; w[1] = 1.0;
    } else {
        const double gg = std::sqrt(3.0 / 5.0);
        x[0] = -gg; x[1] = 0.0; x[2] = gg;
        w[0] = 5.0 / 9.0; w[1] = 8.0 / 9.0; w[2] = 5.0 / 9.0;
    }
}
double lag(int p, int a, double s) {
    if (p == 1) return a == 0 ? 0.5 * (1.0 - s) : 0.5 * (1.0 + s);
    if (a == 0) return 0.5 * s * (s - 1.0);
    if (a == 1) return 1.0 - s * s;
    return 0.5 * s * (s + 1.0);
}
double dlag(int p, int a, double s) {
    if (p == 1) return a == 0 ? -0.5 : 0.5;
    if (a == 0) return s - 0.5;
    if (a == 1) return -2.0 * s;
    return s + 0.5;
}
}  // namespace

GenTables make_gen_tables(int d, int p) {
    GenTables T{};
    const int q1 = p + 1;
    double x[3], w[3];
    rule1d(q1, x, w);
    const int npe = d == 2 ? q1 * q1 : q1 * q1 * q1, npf = d == 2 ? q1 : q1 * q1;
    for (int q = 0; q < npe; ++q) {
        const int qi[3] = {q % q1, (q / q1) % q1, q / (q1 * q1)};
        T.W[q] = 1.0;
        for (int k = 0; k < d; ++k) {
            T.S[q][k] = x[qi[k]];
            T.W[q] *= w[qi[k]];
        }
        for (int a = 0; a < npe; ++a) {
            const int ai[3] = {a % q1, (a / q1) % q1, a / (q1 * q1)};
            double v = 1.0;
            for (int k = 0; k < d; ++k) v *= lag(p, ai[k], T.S[q][k]);
            T.N[q][a] = v;
            for (int k = 0; k < d; ++k) {
                double t = dlag(p, ai[k], T.S[q][k]);
                for (int l = 0; l < d; ++l)
                    if (l != k) t *= lag(p, ai[l], T.S[q][l]);
                T.dN[q][a][k] = t;
            }
        }
    }
    for (int q = 0; q < npf; ++q) {
        const int qi[2] = {q % q1, q / q1};
        T.FW[q] = 1.0;
        for (int k = 0; k < d - 1; ++k) {
            T.FT[q][k] = x[qi[k]];
            T.FW[q] *= w[qi[k]];
        }
        for (int a = 0; a < npf; ++a) {
            const int ai[2] = {a % q1, a / q1};
            double v = 1.0;
            for (int k = 0; k < d - 1; ++k) v *= lag(p, ai[k], T.FT[q][k]);
            T.Nf[q][a] = v;
        }
    }
    return T;
}

GenGeom make_gen_geom(int d, int p, const double* lo, const double* hi, const int* n) {
    GenGeom g{};
    g.d = d;
    g.p = p;
    g.nnodes = 1;
    g.ncells = 1;
    for (int a = 0; a < 3; ++a) {
        g.nc[a] = a < d ? n[a] : 1;
        g.nn[a] = a < d ? p * n[a] + 1 : 1;
        g.lo[a] = a < d ? lo[a] : 0.0;
        g.hi[a] = a < d ? hi[a] : 0.0;
        g.h[a] = a < d ? (hi[a] - lo[a]) / n[a] : 1.0;
        g.hp[a] = g.h[a] / p;
        if (a < d) {
            g.nnodes *= g.nn[a];
            g.ncells *= g.nc[a];
        }
    }
    const int q1 = p + 1;
    g.npe = d == 2 ? q1 * q1 : q1 * q1 * q1;
    g.npf = d == 2 ? q1 : q1 * q1;
    g.nq = g.npe;
    g.nqf = g.npf;
    g.ndirs = d == 2 ? (2 * p + 1) * (2 * p + 1) : (2 * p + 1) * (2 * p + 1) * (2 * p + 1);
    g.face_off[0] = 0;
    for (int a = 0; a < d; ++a) {
        int cnt = 1;
        for (int k = 0; k < d; ++k)
            if (k != a) cnt *= g.nc[k];
        g.face_off[a + 1] = g.face_off[a] + 2 * cnt;
    }
    for (int a = d + 1; a < 4; ++a) g.face_off[a] = g.face_off[d];
    g.nfaces = g.face_off[d];
    return g;
}

void upload_q2t_tables() {
    Q2T t{};
    double x[3], w[3];
    rule1d(3, x, w);
    for (int q = 0; q < 3; ++q)
        for (int a = 0; a < 3; ++a) {
            t.L[q][a] = lag(2, a, x[q]);
            t.D[q][a] = dlag(2, a, x[q]);
        }
    cudaMemcpyToSymbol(cQ2T, &t, sizeof t);
}

}  // namespace tsb
