// Kernel (3): batched Jacobi-PCG over all micro problems — the hot path — plus the
// small per-sweep kernels of the fixed-point loop (kernel 4).
//
// Design: one thread block owns one micro problem at a time
// (persistent grid, atomic ticket queue handed out longest-first, so per-problem
// iteration counts balance themselves).  The problem's operator is loaded ONCE per
// solve into shared memory as the symmetric half of the 9-point stencil (C, E, NW, N,
// NE planes, zero halos); the search direction p lives in shared memory; x, r, D^-1
// and Ap live in registers.  Two thread layouts:
//   k_micro_pcg       thread = column strip of R rows; the SpMV slides a 3x3 window of
//                     p down the strip and reuses N as the next row's S;
//   k_micro_pcg_pair  thread = column pair x strip, planes split into even/odd
//                     half-rows (unit-stride, conflict-free), shared horizontal data
//                     read once, own p kept from the window for the update.
// HBM is touched only in the prologue/epilogue; every PCG iteration runs out of SMEM.
// Dot products: per-warp sums on the FP64 tensor core (two DMMA m8n8k4) + one SMEM
// exchange re-reduced by every warp (identical bits in every thread, one barrier each).
// The same SMEM-resident kernels also solve the macro u/w systems when the macro grid
// fits one SM (ctx.cu); larger macro grids use the cooperative CSR CG below.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace tsb {

namespace {

constexpr int kRedSlots = 3;
constexpr int kRedStride = 32 * 4;  // doubles per reduction slot

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Sum K values over the block; every thread returns the same bits.  One barrier.
// Warp partials are stored k-major (red[k * 32 + warp]) so the second stage reads
// them conflict-free.
// MERGE2: K = 2 second stage as one DMMA pair (below); measured +2.2 % on C3, +0.8 % on
// C1, -1 % on C2's 33-wide pair kernel (3 blocks per SM), which keeps the separate chains.
// PRE1: v[1] arrives already warp-reduced (its warp stage ran earlier, off the burst).
template <int K, bool MERGE2 = true, bool PRE1 = false>
__device__ __forceinline__ void block_sum(double (&v)[K], double* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int k = 0; k < K; ++k)
        if (!(PRE1 && k == 1)) v[k] = warp_sum_tc(v[k]);
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) red[k * 32 + warp] = v[k];
    }
    __syncthreads();
    if (MERGE2 && K == 2 && nw <= 16) {
        // Both components' second stage in one DMMA pair: lanes 0-15 carry component 0's
        // warp partials (B columns 0-3), lanes 16-31 component 1's (columns 4-7); the
        // second MMA's B selects k = 0,1 for even and k = 2,3 for odd output columns, so
        // every lane gets (total 0, total 1).  Same partial sums in the same positions as
        // two separate warp_sum_tc (the extra terms are exact zeros): identical bits, half
        // the DMMAs on the FP64 tensor pipe all warps share.
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
        // The zero B entries multiply the other component's sums: an inf there would give
        // inf * 0 = NaN in this one.  Every thread holds the same bits, so this branch is
        // block-uniform; non-finite totals redo the stage as two separate chains.
        if (isfinite(s0) && isfinite(s1)) {
            v[0] = s0;
            v[K - 1] = s1;
            return;
        }
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const double t = lane < nw ? red[k * 32 + lane] : 0.0;
        v[k] = warp_sum_tc(t);
    }
}

// Shared-memory geometry of one micro problem for strip height R: pitch nx+1 (one
// zero column doubles as left/right halo), rows padded to a multiple of R plus a
// zero halo row above and below.  Padded rows carry zero coefficients and zero rhs,
// so they stay exactly zero through the iteration and need no guards.
struct SmemGeom {
    int nx, ny, W, rows, L;
};

__host__ __device__ __forceinline__ SmemGeom smem_geom(const GridG& g, int R) {
    SmemGeom s;
    s.nx = g.n0 + 1;
    s.ny = g.n1 + 1;
    s.W = s.nx + 1;
    s.rows = ((s.ny + R - 1) / R) * R;
    s.L = (s.rows + 2) * s.W + 2;
    return s;
}

__host__ __device__ __forceinline__ size_t smem_bytes_for(const GridG& g, int R) {
    const SmemGeom s = smem_geom(g, R);
    return (6 * (size_t)s.L + kRedSlots * kRedStride) * sizeof(double) + 16;
}

// y = A p over the thread's strip (symmetric 9-point stencil in smem, 3x3 window of
// p sliding down the strip; the N coefficient of row j is the S coefficient of j+1).
// Also returns sum_k p_k y_k.
template <int R>
__device__ __forceinline__ double strip_spmv(const double* __restrict__ sP, const double* __restrict__ sC,
                                             const double* __restrict__ sE, const double* __restrict__ sNW,
                                             const double* __restrict__ sN, const double* __restrict__ sNE,
                                             int base, int W, double (&y)[R]) {
    double pmL = sP[base - W - 1], pmC = sP[base - W], pmR = sP[base - W + 1];
    double p0L = sP[base - 1], p0C = sP[base], p0R = sP[base + 1];
    double cS = sN[base - W];
    double py = 0.0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int id = base + k * W;
        const double ppL = sP[id + W - 1], ppC = sP[id + W], ppR = sP[id + W + 1];
        const double cW = sE[id - 1], cSW = sNE[id - W - 1], cSE = sNW[id - W + 1];
        const double cN = sN[id];
        double acc = cSW * pmL;
        acc = fma(cS, pmC, acc);
        acc = fma(cSE, pmR, acc);
        acc = fma(cW, p0L, acc);
        acc = fma(sC[id], p0C, acc);
        acc = fma(sE[id], p0R, acc);
        acc = fma(sNW[id], ppL, acc);
        acc = fma(cN, ppC, acc);
        acc = fma(sNE[id], ppR, acc);
        y[k] = acc;
        py = fma(p0C, acc, py);
        pmL = p0L; pmC = p0C; pmR = p0R;
        p0L = ppL; p0C = ppC; p0R = ppR;
        cS = cN;
    }
    return py;
}

// Max block size per strip height: bounds the register budget the compiler may use.
template <int R> struct StripCfg;
template <> struct StripCfg<2> { static constexpr int kMaxThreads = 1024; };
template <> struct StripCfg<3> { static constexpr int kMaxThreads = 1024; };
template <> struct StripCfg<4> { static constexpr int kMaxThreads = 1024; };
template <> struct StripCfg<5> { static constexpr int kMaxThreads = 896; };
template <> struct StripCfg<7> { static constexpr int kMaxThreads = 672; };
template <> struct StripCfg<9> { static constexpr int kMaxThreads = 576; };
template <> struct StripCfg<13> { static constexpr int kMaxThreads = 352; };
template <> struct StripCfg<17> { static constexpr int kMaxThreads = 256; };
template <> struct StripCfg<22> { static constexpr int kMaxThreads = 224; };

int max_threads_for(int R) {
    switch (R) {
        case 2: case 3: case 4: return 1024;
        case 5: return 896;
        case 7: return 672;
        case 9: return 576;
        case 13: return 352;
        case 17: return 256;
        case 22: return 224;
    }
    return 0;
}

// Thread -> (column, strip) map.  Full warps cover 32 consecutive columns of one
// strip (conflict-free 256-B SMEM rows).  If 16..31 columns are left per strip, their
// first 16 go to half-warps, two strips per warp (each half reads 16 consecutive
// doubles = all 32 banks once, so the pair of halves still needs only the ideal two
// wavefronts); the remaining < 16 columns of all strips are packed into tail warps.
struct StripMap {
    int F, H, Lc, nstrips, full_warps, half_warps, threads;
};

__host__ __device__ __forceinline__ StripMap strip_map(int nx, int ny, int R) {
    StripMap m;
    m.F = nx / 32;
    const int rem = nx - 32 * m.F;
    m.H = rem >= 16 ? 1 : 0;
    m.Lc = rem - 16 * m.H;
    m.nstrips = (ny + R - 1) / R;
    m.full_warps = m.F * m.nstrips;
    m.half_warps = m.H ? (m.nstrips + 1) / 2 : 0;
    const int tail = (m.Lc * m.nstrips + 31) / 32;
    m.threads = 32 * (m.full_warps + m.half_warps + tail);
    return m;
}

__device__ __forceinline__ bool thread_cell(const StripMap& m, int tid, int& col, int& strip) {
    const int warp = tid >> 5, lane = tid & 31;
    if (warp < m.full_warps) {
        strip = warp / m.F;
        col = (warp % m.F) * 32 + lane;
        return true;
    }
    if (warp < m.full_warps + m.half_warps) {
        strip = 2 * (warp - m.full_warps) + (lane >> 4);
        col = 32 * m.F + (lane & 15);
        if (strip < m.nstrips) return true;
        col = 0;
        return false;  // idle half of the last warp (odd strip count)
    }
    const int q = (warp - m.full_warps - m.half_warps) * 32 + lane;
    if (m.Lc == 0 || q >= m.Lc * m.nstrips) {
        col = 0;
        strip = m.nstrips;  // idle
        return false;
    }
    col = 32 * m.F + 16 * m.H + q % m.Lc;
    strip = q / m.Lc;
    return true;
}

// NXC > 0 fixes the micro grid width at compile time (SMEM offsets become immediates).
template <int R, int NXC>
__global__ void __launch_bounds__(StripCfg<R>::kMaxThreads, 1) k_micro_pcg(const MicroPcgArgs a) {
    extern __shared__ double smem[];
    const SmemGeom G = smem_geom(a.micro, R);
    const int nx = NXC ? NXC : G.nx;
    const int ny = G.ny, n = nx * ny;
    const int W = NXC ? NXC + 1 : G.W;
    const int L = G.L;
    double* sP = smem;
    double* sC = sP + L;
    double* sE = sC + L;
    double* sNW = sE + L;
    double* sN = sNW + L;
    double* sNE = sN + L;
    double* red = sNE + L;
    int* sTicket = reinterpret_cast<int*>(red + kRedSlots * kRedStride);

    const int tid = threadIdx.x;
    int col, strip;
    const bool active = thread_cell(strip_map(nx, ny, R), tid, col, strip);
    const int j0 = strip * R;
    const int nvalid = active ? min(R, ny - j0) : 0;  // real (non-padded) rows of the strip
    const int base = 1 + (j0 + 1) * W + col;

    for (int k = tid; k < 6 * L; k += blockDim.x) smem[k] = 0.0;  // halos/padding stay zero

    for (;;) {
        __syncthreads();
        if (tid == 0) *sTicket = atomicAdd(a.counter, 1);
        __syncthreads();
        const int T = *sTicket;
        if (T >= a.n_problems) break;
        const int P = a.order ? __ldg(a.order + T) : T;

        // ---------------- prologue: operator -> smem, b, x0 ------------------
        const double* st = a.stencil + (size_t)P * a.stencil_stride;
        const double uP = a.u[P], wP = a.w[P];
        const bool use_u = a.kappa1 != 0.0 && uP != 0.0;  // micro_rhs, assembly.cpp:373-374
        const bool use_w = a.kappa3 != 0.0 && wP != 0.0;
        const double cu = a.kappa1 * uP, cw = a.kappa3 * wP;
        const size_t vrow = (size_t)P * n;
        double x[R], r[R], dinv[R], ap[R];
#pragma unroll
        for (int k = 0; k < R; ++k) {
            x[k] = r[k] = ap[k] = 0.0;
            dinv[k] = 1.0;
            if (k < nvalid) {
                const int node = (j0 + k) * nx + col;
                const int id = base + k * W;
                const double cC = __ldg(st + (size_t)(a.plane_base + 0) * n + node);
                sC[id] = cC;
                sE[id] = __ldg(st + (size_t)(a.plane_base + 1) * n + node);
                sNW[id] = __ldg(st + (size_t)(a.plane_base + 2) * n + node);
                sN[id] = __ldg(st + (size_t)(a.plane_base + 3) * n + node);
                sNE[id] = __ldg(st + (size_t)(a.plane_base + 4) * n + node);
                dinv[k] = cC != 0.0 ? 1.0 / cC : 1.0;  // linalg.cpp:116-117
                double bk = a.has_fixed ? __ldg(a.fixed + vrow + node) : 0.0;
                if (use_u) bk = fma(cu, __ldg(a.rin + vrow + node), bk);
                if (use_w) bk = fma(cw, __ldg(a.rout + vrow + node), bk);
                r[k] = bk;
                x[k] = a.warm ? a.V[vrow + node] : 0.0;
                sP[id] = x[k];
            }
        }
        __syncthreads();
        if (active) strip_spmv<R>(sP, sC, sE, sNW, sN, sNE, base, W, ap);
        double s3[3] = {0.0, 0.0, 0.0};  // |b|^2, r.z, |r|^2
#pragma unroll
        for (int k = 0; k < R; ++k) {
            s3[0] = fma(r[k], r[k], s3[0]);
            r[k] -= ap[k];
            const double z = dinv[k] * r[k];
            ap[k] = z;
            s3[1] = fma(r[k], z, s3[1]);
            s3[2] = fma(r[k], r[k], s3[2]);
        }
        block_sum<3>(s3, red);
        int slot = 1;
        const double bnorm = sqrt(s3[0]);
        int status = 0, iters = 0;
        double rel = 0.0;
        if (bnorm == 0.0) {  // linalg.cpp:110-114: x := 0, converged, 0 iterations
#pragma unroll
            for (int k = 0; k < R; ++k) x[k] = 0.0;
        } else {
            double rz = s3[1];
            rel = sqrt(s3[2]) / bnorm;
            if (rel > a.tol) {
                const double thr = rel_threshold(bnorm, a.tol);  // rr <= thr <=> sqrt(rr) / bnorm <= tol
                double rr_last = s3[2];
                if (active) {
#pragma unroll
                    for (int k = 0; k < R; ++k) sP[base + k * W] = ap[k];  // p0 = z0
                }
                __syncthreads();
                status = 2;  // maxit unless converged below
                for (int it = 1; it <= a.maxit; ++it) {
                    double t1[1] = {0.0};
                    if (active) t1[0] = strip_spmv<R>(sP, sC, sE, sNW, sN, sNE, base, W, ap);
                    const double yrz = div_recip(rz);  // divisor part of beta = rz_new / rz, overlaps the reduction
                    block_sum<1>(t1, red + slot * kRedStride);
                    slot = slot == kRedSlots - 1 ? 0 : slot + 1;
                    const double pAp = t1[0];
                    iters = it;
                    if (pAp <= 0.0) {  // linalg.cpp:138-142
                        status = 1;
                        break;
                    }
                    const double alpha = rz / pAp;
                    double t2[2] = {0.0, 0.0};
#pragma unroll
                    for (int k = 0; k < R; ++k) {
                        r[k] = fma(-alpha, ap[k], r[k]);
                        t2[0] = fma(r[k], r[k], t2[0]);
                        const double z = dinv[k] * r[k];
                        ap[k] = z;  // ap now holds z
                        t2[1] = fma(r[k], z, t2[1]);
                    }
                    block_sum<2>(t2, red + slot * kRedStride);
                    slot = slot == kRedSlots - 1 ? 0 : slot + 1;
                    rr_last = t2[0];
                    const bool done = t2[0] <= thr;
                    const double beta = div_finish(t2[1], rz, yrz);  // == t2[1] / rz bitwise
                    rz = t2[1];
                    // x += alpha p, deferred past the reduction (p re-read once from smem)
                    if (active) {
#pragma unroll
                        for (int k = 0; k < R; ++k) {
                            const int id = base + k * W;
                            const double pk = sP[id];
                            x[k] = fma(alpha, pk, x[k]);
                            if (!done) sP[id] = fma(beta, pk, ap[k]);
                        }
                    }
                    if (done) {
                        status = 0;
                        break;
                    }
                    __syncthreads();
                }
                rel = sqrt(rr_last) / bnorm;  // the last relative residual, as the loop computed it
            }
        }

        // ---------------- epilogue ------------------------------------------
#pragma unroll
        for (int k = 0; k < R; ++k)
            if (k < nvalid) a.V[vrow + (j0 + k) * nx + col] = x[k];
        if (a.epilogue) {
            // true residual ||b - A V|| (solver.cpp:104-113) and coupling (assembly.cpp:377-393)
            if (active) {
#pragma unroll
                for (int k = 0; k < R; ++k) sP[base + k * W] = x[k];
            }
            __syncthreads();
            if (active) strip_spmv<R>(sP, sC, sE, sNW, sN, sNE, base, W, ap);
            double t1[1] = {0.0};
#pragma unroll
            for (int k = 0; k < R; ++k) {
                if (k < nvalid) {
                    const int node = (j0 + k) * nx + col;
                    double bk = a.has_fixed ? __ldg(a.fixed + vrow + node) : 0.0;
                    if (use_u) bk = fma(cu, __ldg(a.rin + vrow + node), bk);
                    if (use_w) bk = fma(cw, __ldg(a.rout + vrow + node), bk);
                    const double rr = bk - ap[k];
                    t1[0] = fma(rr, rr, t1[0]);
                }
            }
            block_sum<1>(t1, red + slot * kRedStride);
            const int warp = tid >> 5, lane = tid & 31;
            // one warp per role (a single-warp block does both in turn)
            for (int rw = warp; rw < 2; rw += (int)(blockDim.x >> 5)) {
                const int role = rw == 0 ? TS_GAMMA_I : TS_GAMMA_O;
                const double* len = a.face_len + (size_t)P * a.face_len_stride;
                const int nf = a.micro.faces();
                double tot = 0.0;
                for (int f = lane; f < nf; f += 32) {
                    int side, n0, n1;
                    face_info(a.micro, f, side, n0, n1);
                    if (a.micro_role[side] != role) continue;
                    const double scale = face_scale_of(a.micro, f);
                    const double v0 = sP[1 + (n0 / nx + 1) * W + n0 % nx];
                    const double v1 = sP[1 + (n1 / nx + 1) * W + n1 % nx];
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const double vq = v0 * a.Nf[q][0] + v1 * a.Nf[q][1];
                        tot += a.GW[q] * vq * len[f * 2 + q] * scale;
                    }
                }
                tot = warp_sum(tot);
                if (lane == 0) (rw == 0 ? a.bI : a.bO)[P] = tot;
            }
            if (tid == 0) a.res_v[P] = sqrt(t1[0]);
        }
        if (tid == 0) {
            a.iters[P] = iters;
            a.status[P] = status;
            a.final_rel[P] = rel;
        }
    }
}

struct Choice {
    int R, threads;
};

// Strip height: tall strips amortise the window and barrier overhead per row and
// were measured fastest for the 33- and 65-wide BASELINE grids (profiles/r01); when
// there are fewer problems than two per SM, shorter strips (more threads per
// problem) win instead.
Choice choose(const GridG& g, int forced, int n_problems) {
    const int nx = g.n0 + 1, ny = g.n1 + 1;
    static const int cands[] = {2, 3, 4, 5, 7, 9, 13, 17, 22};
    const bool few = n_problems < 2 * 148;
    Choice best{0, 0};
    double best_score = 1e30;
    for (int R : cands) {
        if (forced && R != forced) continue;
        if (!forced && R > 13) continue;  // 17/22 measured slower than 13 on 33- and 65-wide grids
        const StripMap m = strip_map(nx, ny, R);
        if (m.threads > max_threads_for(R)) continue;
        if (smem_bytes_for(g, R) > 232448) continue;
        const double waste = double(m.nstrips * R - ny) / ny;
        const double score = few ? waste * 4.0 + 0.01 * R : waste * 10.0 - R;
        if (score < best_score) {
            best_score = score;
            best = {R, m.threads};
        }
    }
    return best;
}

template <int R, int NXC>
void launch_R(const MicroPcgArgs& a, int threads, cudaStream_t s) {
    const size_t smem = smem_bytes_for(a.micro, R);
    cudaFuncSetAttribute(k_micro_pcg<R, NXC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_micro_pcg<R, NXC>, threads, smem);
    if (per_sm < 1) per_sm = 1;
    int grid = sms * per_sm;
    if (grid > a.n_problems) grid = a.n_problems;
    if (grid < 1) grid = 1;
    k_micro_pcg<R, NXC><<<grid, threads, smem, s>>>(a);
}

// Compile-time grid widths for the BASELINE micro grids (17, 33, 65 nodes per row);
// any other width runs the runtime-width instantiation.
template <int R>
void launch_width(const MicroPcgArgs& a, int threads, cudaStream_t s) {
    switch (a.micro.n0 + 1) {
        case 17: launch_R<R, 17>(a, threads, s); break;
        case 33: launch_R<R, 33>(a, threads, s); break;
        case 65: launch_R<R, 65>(a, threads, s); break;
        default: launch_R<R, 0>(a, threads, s); break;
    }
}

// ------------------------------------------------------------ column pairs --
// Variant for compile-time grid widths: each thread owns the column pair (2t, 2t+1)
// of a strip of R rows.  Every plane is stored split into an even and an odd
// half-row (pitch PP = NP + 2, zero halos at t = -1 and t = NP), so every SMEM
// access a warp makes is unit-stride (conflict-free), and the horizontal neighbour
// data the two columns share is read once: per row pair 4 p + 10 own + 3 neighbour
// coefficient loads (17) instead of 2 x 11 for two single-column threads.
template <int NXC>
struct PairDims {
    static constexpr int NP = (NXC + 1) / 2, PP = NP + 2, RS = 2 * PP;
};

__host__ __device__ __forceinline__ int pair_rows(int ny, int R) { return ((ny + R - 1) / R) * R; }

__host__ __device__ __forceinline__ size_t pair_smem_bytes(const GridG& g, int R) {
    const int nx = g.n0 + 1, ny = g.n1 + 1;
    const int RS = 2 * ((nx + 1) / 2 + 2);
    const size_t L = (size_t)(pair_rows(ny, R) + 2) * RS + pair_rows(ny, R) / R + 2;  // + strip skews
    return (6 * L + kRedSlots * kRedStride) * sizeof(double) + 16;
}

template <int R> struct PairCfg;
template <> struct PairCfg<4> { static constexpr int kMaxThreads = 576; };
template <> struct PairCfg<5> { static constexpr int kMaxThreads = 448; };
template <> struct PairCfg<6> { static constexpr int kMaxThreads = 384; };

int pair_max_threads(int R) { return R == 4 ? 576 : R == 5 ? 448 : R == 6 ? 384 : 0; }

// Row offsets inside a pair strip.  Each strip's rows are shifted by one more double
// than the strip above (skew), so the tail warp — one lane per strip on the same
// column pair — hits distinct banks (strip stride R*RS+1 is odd mod 16 doubles).
// k = -1 / R are the rows of the neighbouring strips.
template <int R, int RS>
__host__ __device__ constexpr int pair_ro(int k) { return k * RS + (k < 0 ? -1 : (k >= R ? 1 : 0)); }

// y = A p over the pair strip; be / bo = SMEM index of (2t, j0) / (2t+1, j0).
// Per node the nine products go into CH independent partial sums (see below).
// KEEP_P: also return the thread's own p values (the window's centre columns), so the
// update needs no SMEM reload of p.
template <int R, int PP, bool KEEP_P = false, int CH = (2 * PP - 4 > 64 ? 2 : 3)>
__device__ __forceinline__ double pair_spmv(const double* __restrict__ sP, const double* __restrict__ sC,
                                            const double* __restrict__ sE, const double* __restrict__ sNW,
                                            const double* __restrict__ sN, const double* __restrict__ sNE,
                                            int be, double (&y)[2 * R], double* pown = nullptr,
                                            const double* cdg = nullptr, const double* pin = nullptr) {
    // pin: the thread's own p values from registers (it computed them in the previous p
    // update), so only the neighbour columns' and the strip halo rows' p come from SMEM
    constexpr int RS = 2 * PP;
    const int bo = be + PP;
    constexpr int rm = pair_ro<R, RS>(-1);
    double pmL = sP[bo + rm - 1], pmE = sP[be + rm], pmO = sP[bo + rm], pmR = sP[be + rm + 1];
    double p0L = sP[bo - 1], p0E = pin ? pin[0] : sP[be], p0O = pin ? pin[1] : sP[bo], p0R = sP[be + 1];
    double cSe = sN[be + rm], cSo = sN[bo + rm];  // S of this row = N of the row below
    double cSEe = sNW[bo + rm];                   // SE of (2t) = NW of (2t+1, j-1)
    double cSWo = sNE[be + rm];                   // SW of (2t+1) = NE of (2t, j-1)
    double py = 0.0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
        const int r0 = pair_ro<R, RS>(k), rp = pair_ro<R, RS>(k + 1), rd = pair_ro<R, RS>(k - 1);
        const int ie = be + r0, io = bo + r0;
        const bool own_next = pin && k + 1 < R;
        const double ppL = sP[bo + rp - 1], ppE = own_next ? pin[2 * k + 2] : sP[be + rp],
                     ppO = own_next ? pin[2 * k + 3] : sP[bo + rp], ppR = sP[be + rp + 1];
        const double cWe = sE[io - 1];         // E of (2t-1, j)
        const double cSWe = sNE[bo + rd - 1];  // NE of (2t-1, j-1)
        const double cSEo = sNW[be + rd + 1];  // NW of (2t+2, j-1)
        // cdg: the thread's own diagonal from registers (the pair kernel keeps C there and
        // D^-1 in the SMEM plane, moving those loads out of the SMEM-bound SpMV)
        const double Ce = cdg ? cdg[2 * k] : sC[ie], Ee = sE[ie], NWe = sNW[ie], Ne = sN[ie], NEe = sNE[ie];
        const double Co = cdg ? cdg[2 * k + 1] : sC[io], Eo = sE[io], NWo = sNW[io], No = sN[io], NEo = sNE[io];
        // Independent partial sums per node shorten the dependent FMA chain (the order
        // differs from CSR order only in rounding).  CH = 3: one per stencil row
        // (j-1, j, j+1); CH = 2: rows j-1..j | j+1 (fewer registers; measured best on
        // the 65-wide grid, CH = 3 on the 33-wide one).
        double ye, yo;
        if (CH == 3) {
            double ye0 = cSWe * pmL, ye1 = cWe * p0L, ye2 = NWe * ppL;
            ye0 = fma(cSe, pmE, ye0);
            ye1 = fma(Ce, p0E, ye1);
            ye2 = fma(Ne, ppE, ye2);
            ye0 = fma(cSEe, pmO, ye0);
            ye1 = fma(Ee, p0O, ye1);
            ye2 = fma(NEe, ppO, ye2);
            ye = (ye0 + ye1) + ye2;
            double yo0 = cSWo * pmE, yo1 = Ee * p0E, yo2 = NWo * ppE;  // W of (2t+1) = E of (2t)
            yo0 = fma(cSo, pmO, yo0);
            yo1 = fma(Co, p0O, yo1);
            yo2 = fma(No, ppO, yo2);
            yo0 = fma(cSEo, pmR, yo0);
            yo1 = fma(Eo, p0R, yo1);
            yo2 = fma(NEo, ppR, yo2);
            yo = (yo0 + yo1) + yo2;
        } else {
            double ye0 = cSWe * pmL, ye2 = NWe * ppL;
            ye0 = fma(cSe, pmE, ye0);
            ye2 = fma(Ne, ppE, ye2);
            ye0 = fma(cSEe, pmO, ye0);
            ye2 = fma(NEe, ppO, ye2);
            ye0 = fma(cWe, p0L, ye0);
            ye0 = fma(Ce, p0E, ye0);
            ye0 = fma(Ee, p0O, ye0);
            ye = ye0 + ye2;
            double yo0 = cSWo * pmE, yo2 = NWo * ppE;
            yo0 = fma(cSo, pmO, yo0);
            yo2 = fma(No, ppO, yo2);
            yo0 = fma(cSEo, pmR, yo0);
            yo2 = fma(NEo, ppR, yo2);
            yo0 = fma(Ee, p0E, yo0);  // W of (2t+1) = E of (2t)
            yo0 = fma(Co, p0O, yo0);
            yo0 = fma(Eo, p0R, yo0);
            yo = yo0 + yo2;
        }
        y[2 * k] = ye;
        y[2 * k + 1] = yo;
        if (KEEP_P) {
            pown[2 * k] = p0E;
            pown[2 * k + 1] = p0O;
        }
        py = fma(p0E, ye, py);
        py = fma(p0O, yo, py);
        pmL = p0L; pmE = p0E; pmO = p0O; pmR = p0R;
        p0L = ppL; p0E = ppE; p0O = ppO; p0R = ppR;
        cSe = Ne; cSo = No; cSEe = NWo; cSWo = NEe;
    }
    return py;
}

// sum_m r[m]^2 over the thread's 2R nodes as two interleaved chains (even / odd column of
// the pair): ptxas places this after the SpMV, so chain depth is latency on the critical
// path (R instead of 2R dependent FMAs).
template <int R>
__device__ __forceinline__ double pair_rr(const double (&r)[2 * R]) {
    double e = 0.0, o = 0.0;
#pragma unroll
    for (int k = 0; k < R; ++k) {
        e = fma(r[2 * k], r[2 * k], e);
        o = fma(r[2 * k + 1], r[2 * k + 1], o);
    }
    return e + o;
}

template <int R, int NXC, bool CG1 = false>
__global__ void __launch_bounds__(PairCfg<R>::kMaxThreads, 1) k_micro_pcg_pair(const MicroPcgArgs a) {
    extern __shared__ double smem[];
    constexpr int nx = NXC, NP = PairDims<NXC>::NP, PP = PairDims<NXC>::PP, RS = PairDims<NXC>::RS;
    const int ny = a.micro.n1 + 1, n = nx * ny;
    const int L = (pair_rows(ny, R) + 2) * RS + pair_rows(ny, R) / R + 2;
    double* sP = smem;
    double* sC = sP + L;
    double* sE = sC + L;
    double* sNW = sE + L;
    double* sN = sNW + L;
    double* sNE = sN + L;
    double* red = sNE + L;
    int* sTicket = reinterpret_cast<int*>(red + kRedSlots * kRedStride);

    const int tid = threadIdx.x;
    int t, strip;
    const bool active = thread_cell(strip_map(NP, ny, R), tid, t, strip);
    const int j0 = strip * R;
    const int nvalid = active ? min(R, ny - j0) : 0;
    const int be = (j0 + 1) * RS + (strip + 1) + t + 1;  // strip s rows carry skew s + 1
    const int ncols = min(2, nx - 2 * t);  // 1 when 2t+1 is the virtual column
    auto sidx = [&](int m) { return be + (m & 1) * PP + (m >> 1) * RS; };  // m = 2k + (0 even | 1 odd)

    for (int k = tid; k < 6 * L; k += blockDim.x) smem[k] = 0.0;

    for (;;) {
        __syncthreads();
        if (tid == 0) *sTicket = atomicAdd(a.counter, 1);
        __syncthreads();
        const int T = *sTicket;
        if (T >= a.n_problems) break;
        const int P = a.order ? __ldg(a.order + T) : T;

        const double* st = a.stencil + (size_t)P * a.stencil_stride;
        const double uP = a.u[P], wP = a.w[P];
        const bool use_u = a.kappa1 != 0.0 && uP != 0.0;  // micro_rhs, assembly.cpp:373-374
        const bool use_w = a.kappa3 != 0.0 && wP != 0.0;
        const double cu = a.kappa1 * uP, cw = a.kappa3 * wP;
        const size_t vrow = (size_t)P * n;
        // CREG (65-wide grids): registers hold the diagonal C (read by every SpMV) and the sC
        // plane holds D^-1 (read once per iteration in the latency-bound r/z update); measured
        // +2.8 % on C3, -0.8 % on the 33-wide C2 (3 blocks per SM), where the registers keep
        // D^-1 and the plane C as before.
        constexpr bool CREG = NXC >= 65;
        double x[2 * R], r[2 * R], cdg[2 * R], ap[2 * R];  // cdg: C (CREG) or D^-1
#pragma unroll
        for (int m = 0; m < 2 * R; ++m) {
            x[m] = r[m] = ap[m] = 0.0;
            cdg[m] = CREG ? 0.0 : 1.0;
            if ((m >> 1) < nvalid && (m & 1) < ncols) {
                const int node = (j0 + (m >> 1)) * nx + 2 * t + (m & 1);
                const int id = sidx(m);
                const double cC = __ldg(st + (size_t)(a.plane_base + 0) * n + node);
                const double di = cC != 0.0 ? 1.0 / cC : 1.0;  // D^-1, linalg.cpp:116-117
                cdg[m] = CREG ? cC : di;
                sC[id] = CREG ? di : cC;
                sE[id] = __ldg(st + (size_t)(a.plane_base + 1) * n + node);
                sNW[id] = __ldg(st + (size_t)(a.plane_base + 2) * n + node);
                sN[id] = __ldg(st + (size_t)(a.plane_base + 3) * n + node);
                sNE[id] = __ldg(st + (size_t)(a.plane_base + 4) * n + node);
                double bk = a.has_fixed ? __ldg(a.fixed + vrow + node) : 0.0;
                if (use_u) bk = fma(cu, __ldg(a.rin + vrow + node), bk);
                if (use_w) bk = fma(cw, __ldg(a.rout + vrow + node), bk);
                r[m] = bk;
                x[m] = a.warm ? a.V[vrow + node] : 0.0;
                sP[id] = x[m];
            }
        }
        __syncthreads();
        if (active) pair_spmv<R, PP>(sP, sC, sE, sNW, sN, sNE, be, ap, nullptr, CREG ? cdg : nullptr);
        double s3[3] = {0.0, 0.0, 0.0};
#pragma unroll
        for (int m = 0; m < 2 * R; ++m) {
            s3[0] = fma(r[m], r[m], s3[0]);
            r[m] -= ap[m];
            const double z = (CREG ? (active ? sC[sidx(m)] : 0.0) : cdg[m]) * r[m];
            ap[m] = z;
            s3[1] = fma(r[m], z, s3[1]);
            s3[2] = fma(r[m], r[m], s3[2]);
        }
        block_sum<3>(s3, red);
        int slot = 1;
        const double bnorm = sqrt(s3[0]);
        int status = 0, iters = 0;
        double rel = 0.0;
        if (bnorm == 0.0) {  // linalg.cpp:110-114
#pragma unroll
            for (int m = 0; m < 2 * R; ++m) x[m] = 0.0;
        } else {
            double rz = s3[1];
            rel = sqrt(s3[2]) / bnorm;
            if (CG1 && rel > a.tol) {
                // Single-reduction loop (Chronopoulos & Gear), as the cluster kernels (gpcg.cu):
                // s = A p by the recurrence s = w + beta s, w = A u, u = D^-1 r; one SpMV, one
                // barrier for u and one three-value reduction per iteration.  Same iterates in
                // exact arithmetic; the stop test on the recursive ||r||, p.Ap = delta - beta
                // gamma / alpha_prev, iteration counts as the reference's loop SpMVs.
                const double thr = rel_threshold(bnorm, a.tol);
                double rr_last = s3[2];
                double pv[2 * R], sv[2 * R], u[2 * R];
#pragma unroll
                for (int m = 0; m < 2 * R; ++m) u[m] = ap[m];  // u0 = z0
                if (active) {
#pragma unroll
                    for (int m = 0; m < 2 * R; ++m) sP[sidx(m)] = u[m];
                }
                __syncthreads();
                double gamma = rz;
                double t1[1] = {0.0};
                if (active)
                    t1[0] = pair_spmv<R, PP>(sP, sC, sE, sNW, sN, sNE, be, ap, nullptr, CREG ? cdg : nullptr, u);
                block_sum<1>(t1, red + slot * kRedStride);
                slot = slot == kRedSlots - 1 ? 0 : slot + 1;
                status = 2;
                iters = 1;
                double pAp = t1[0], alpha = 0.0;
                if (pAp <= 0.0) {
                    status = 1;
                } else {
                    alpha = gamma / pAp;
#pragma unroll
                    for (int m = 0; m < 2 * R; ++m) {
                        pv[m] = u[m];
                        sv[m] = ap[m];
                    }
                    for (int it = 1; it <= a.maxit; ++it) {
                        iters = it;
                        double t3[3] = {0.0, 0.0, 0.0};  // (r,u), (r,r), (w,u)
#pragma unroll
                        for (int m = 0; m < 2 * R; ++m) {
                            x[m] = fma(alpha, pv[m], x[m]);
                            r[m] = fma(-alpha, sv[m], r[m]);
                            u[m] = (CREG ? (active ? sC[sidx(m)] : 0.0) : cdg[m]) * r[m];
                            t3[0] = fma(r[m], u[m], t3[0]);
                            t3[1] = fma(r[m], r[m], t3[1]);
                        }
                        // (the previous reduction's barrier ended every SpMV of the previous u)
                        if (active) {
#pragma unroll
                            for (int m = 0; m < 2 * R; ++m) sP[sidx(m)] = u[m];
                        }
                        __syncthreads();
                        if (active)
                            t3[2] = pair_spmv<R, PP>(sP, sC, sE, sNW, sN, sNE, be, ap, nullptr, CREG ? cdg : nullptr, u);
                        block_sum<3>(t3, red + slot * kRedStride);
                        slot = slot == kRedSlots - 1 ? 0 : slot + 1;
                        rr_last = t3[1];
                        if (t3[1] <= thr) {
                            status = 0;
                            break;
                        }
                        if (it == a.maxit) break;
                        const double beta = t3[0] / gamma;
                        gamma = t3[0];
                        pAp = t3[2] - beta * gamma / alpha;
                        if (pAp <= 0.0) {
                            iters = it + 1;
                            status = 1;
                            break;
                        }
                        alpha = gamma / pAp;
#pragma unroll
                        for (int m = 0; m < 2 * R; ++m) {
                            pv[m] = fma(beta, pv[m], u[m]);
                            sv[m] = fma(beta, sv[m], ap[m]);
                        }
                    }
                }
                rel = sqrt(rr_last) / bnorm;
            } else if (rel > a.tol) {
                const double thr = rel_threshold(bnorm, a.tol);  // rr <= thr <=> sqrt(rr) / bnorm <= tol
                double rr_last = s3[2];
                double pown[2 * R];  // own p values, kept in registers across iterations
#pragma unroll
                for (int m = 0; m < 2 * R; ++m) pown[m] = ap[m];  // p0 = z0
                if (active) {
#pragma unroll
                    for (int m = 0; m < 2 * R; ++m) sP[sidx(m)] = ap[m];
                }
                __syncthreads();
                status = 2;
                // LAG: the stop test of iteration k (src/linalg.cpp:147-152) runs one reduction
                // late: ||r_k||^2 is summed during SpMV k+1 (SMEM-bound, FP64 slack) and reduced
                // with p.Ap, so the r/z update carries one dot product.  Iteration k's x is final
                // when the test fires (x += alpha p precedes it), so results and counts are
                // unchanged; a converged solve costs one extra SpMV.  Measured: +0.9 % on the
                // 65-wide grid (C3, ~300 iterations per solve), -1 % on the 33-wide one (C2,
                // shorter solves, 3 blocks per SM), so it is on for the 65-wide grid only.
                constexpr bool LAG = NXC >= 65;
#ifdef TSB_PHASE_TIMING
                long long ph[6] = {0, 0, 0, 0, 0, 0}, tc = clock64();
#define TSB_PHP(i)                      \
    {                                   \
        const long long tn = clock64(); \
        ph[i] += tn - tc;               \
        tc = tn;                        \
    }
#else
#define TSB_PHP(i)
#endif
                for (int it = 1; it <= a.maxit; ++it) {
                    double t1[LAG ? 2 : 1] = {0.0};
                    // LAG: ||r||^2's warp stage on the FP64 tensor pipe before the SpMV (idle
                    // then) instead of in the reduction burst where all 12 warps queue on it
                    if constexpr (LAG) t1[1] = warp_sum_tc(pair_rr<R>(r));
                    if (active)
                        t1[0] = pair_spmv<R, PP>(sP, sC, sE, sNW, sN, sNE, be, ap, nullptr, CREG ? cdg : nullptr, pown);
                    TSB_PHP(0)
                    const double yrz = div_recip(rz);  // divisor part of beta = rz_new / rz, overlaps the reduction
                    block_sum<LAG ? 2 : 1, (NXC >= 65), LAG>(t1, red + slot * kRedStride);
                    TSB_PHP(1)
                    slot = slot == kRedSlots - 1 ? 0 : slot + 1;
                    if constexpr (LAG) {
                        if (it > 1) {
                            rr_last = t1[1];
                            if (t1[1] <= thr) {  // iteration it-1 converged
                                status = 0;
                                break;
                            }
                        }
                    }
                    const double pAp = t1[0];
                    iters = it;
                    if (pAp <= 0.0) {  // linalg.cpp:138-142
                        status = 1;
                        break;
                    }
                    const double alpha = rz / pAp;
                    double t2[LAG ? 1 : 2] = {0.0};  // {rz} or {rz, rr}
                    // (r.z as three interleaved chains instead of one measured -1 % on config 3:
                    // 2.72e11 against 2.75e11, so the single chain stays)
#pragma unroll
                    for (int m = 0; m < 2 * R; ++m) {
                        r[m] = fma(-alpha, ap[m], r[m]);
                        if constexpr (!LAG) t2[LAG ? 0 : 1] = fma(r[m], r[m], t2[LAG ? 0 : 1]);
                        const double z = (CREG ? (active ? sC[sidx(m)] : 0.0) : cdg[m]) * r[m];
                        ap[m] = z;
                        t2[0] = fma(r[m], z, t2[0]);
                    }
                    TSB_PHP(2)
                    block_sum<LAG ? 1 : 2, (NXC >= 65)>(t2, red + slot * kRedStride);
                    TSB_PHP(3)
                    slot = slot == kRedSlots - 1 ? 0 : slot + 1;
                    bool done = false;
                    if constexpr (!LAG) {
                        rr_last = t2[LAG ? 0 : 1];
                        done = t2[LAG ? 0 : 1] <= thr;
                    }
                    const double beta = div_finish(t2[0], rz, yrz);  // == t2[0] / rz bitwise
                    rz = t2[0];
                    if (active) {
#pragma unroll
                        for (int m = 0; m < 2 * R; ++m) {
                            const double pk = pown[m];  // this iteration's p, in registers
                            x[m] = fma(alpha, pk, x[m]);
                            pown[m] = fma(beta, pk, ap[m]);
                            if (!done) sP[sidx(m)] = pown[m];
                        }
                    }
                    if (done) {
                        status = 0;
                        break;
                    }
                    TSB_PHP(4)
                    __syncthreads();
                    TSB_PHP(5)
                }
#ifdef TSB_PHASE_TIMING
                if ((tid == 0 || tid == 352) && T % 997 == 0 && iters > 0)
                    printf("P %d tid %d iters %d: spmv %lld reduce1 %lld update %lld reduce2 %lld pupdate %lld barrier %lld\n", P,
                           tid, iters, ph[0] / iters, ph[1] / iters, ph[2] / iters, ph[3] / iters, ph[4] / iters, ph[5] / iters);
#endif
                if (LAG && status == 2 && a.maxit >= 1) {  // the last iteration's stop test
                    double t1[1] = {pair_rr<R>(r)};
                    block_sum<1>(t1, red + slot * kRedStride);
                    slot = slot == kRedSlots - 1 ? 0 : slot + 1;
                    rr_last = t1[0];
                    if (t1[0] <= thr) status = 0;
                }
                rel = sqrt(rr_last) / bnorm;  // the last relative residual, as the loop computed it
            }
        }

        // ---------------- epilogue (as k_micro_pcg) --------------------------
#pragma unroll
        for (int m = 0; m < 2 * R; ++m)
            if ((m >> 1) < nvalid && (m & 1) < ncols) a.V[vrow + (j0 + (m >> 1)) * nx + 2 * t + (m & 1)] = x[m];
        if (a.epilogue) {
            if (active) {
#pragma unroll
                for (int m = 0; m < 2 * R; ++m) sP[sidx(m)] = x[m];
            }
            __syncthreads();
            if (active) pair_spmv<R, PP>(sP, sC, sE, sNW, sN, sNE, be, ap, nullptr, CREG ? cdg : nullptr);
            double t1[1] = {0.0};
#pragma unroll
            for (int m = 0; m < 2 * R; ++m) {
                if ((m >> 1) < nvalid && (m & 1) < ncols) {
                    const int node = (j0 + (m >> 1)) * nx + 2 * t + (m & 1);
                    double bk = a.has_fixed ? __ldg(a.fixed + vrow + node) : 0.0;
                    if (use_u) bk = fma(cu, __ldg(a.rin + vrow + node), bk);
                    if (use_w) bk = fma(cw, __ldg(a.rout + vrow + node), bk);
                    const double rr = bk - ap[m];
                    t1[0] = fma(rr, rr, t1[0]);
                }
            }
            block_sum<1>(t1, red + slot * kRedStride);
            const int warp = tid >> 5, lane = tid & 31;
            for (int rw = warp; rw < 2; rw += (int)(blockDim.x >> 5)) {
                const int role = rw == 0 ? TS_GAMMA_I : TS_GAMMA_O;
                const double* len = a.face_len + (size_t)P * a.face_len_stride;
                const int nf = a.micro.faces();
                double tot = 0.0;
                for (int f = lane; f < nf; f += 32) {
                    int side, n0, n1;
                    face_info(a.micro, f, side, n0, n1);
                    if (a.micro_role[side] != role) continue;
                    const double scale = face_scale_of(a.micro, f);
                    const int c0 = n0 % nx, c1 = n1 % nx, r0 = n0 / nx + 1, r1 = n1 / nx + 1;
                    const double v0 = sP[r0 * RS + (r0 + R - 1) / R + (c0 & 1) * PP + (c0 >> 1) + 1];
                    const double v1 = sP[r1 * RS + (r1 + R - 1) / R + (c1 & 1) * PP + (c1 >> 1) + 1];
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const double vq = v0 * a.Nf[q][0] + v1 * a.Nf[q][1];
                        tot += a.GW[q] * vq * len[f * 2 + q] * scale;
                    }
                }
                tot = warp_sum(tot);
                if (lane == 0) (rw == 0 ? a.bI : a.bO)[P] = tot;
            }
            if (tid == 0) a.res_v[P] = sqrt(t1[0]);
        }
        if (tid == 0) {
            a.iters[P] = iters;
            a.status[P] = status;
            a.final_rel[P] = rel;
        }
    }
}

// Pair strip height for a compile-time width: R in {4, 5, 6} that fits SMEM and the
// thread budget with the least row padding (ties -> taller strips).
Choice choose_pair(const GridG& g, int forced) {
    const int nx = g.n0 + 1, ny = g.n1 + 1;
    Choice best{0, 0};
    double best_score = 1e30;
    for (int R : {6, 5, 4}) {
        if (forced && R != forced) continue;
        const StripMap m = strip_map((nx + 1) / 2, ny, R);
        if (m.threads > pair_max_threads(R)) continue;
        if (pair_smem_bytes(g, R) > 232448) continue;
        const double score = double(pair_rows(ny, R) - ny) / ny * 10.0 - R;
        if (score < best_score) {
            best_score = score;
            best = {R, m.threads};
        }
    }
    return best;
}

template <int R, int NXC>
void launch_pair_R(const MicroPcgArgs& a, int threads, cudaStream_t s) {
    const size_t smem = pair_smem_bytes(a.micro, R);
    // TS_PCG_CG1=1: the single-reduction loop (measured slower on config 3: DESIGN.md §7)
    const char* e = std::getenv("TS_PCG_CG1");
    auto kern = (e && e[0] == '1') ? k_micro_pcg_pair<R, NXC, true> : k_micro_pcg_pair<R, NXC, false>;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int dev = 0, sms = 148, per_sm = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, threads, smem);
    if (per_sm < 1) per_sm = 1;
    int grid = sms * per_sm;
    if (grid > a.n_problems) grid = a.n_problems;
    if (grid < 1) grid = 1;
    kern<<<grid, threads, smem, s>>>(a);
}

template <int NXC>
void launch_pair_width(const MicroPcgArgs& a, const Choice& ch, cudaStream_t s) {
    switch (ch.R) {
        case 4: launch_pair_R<4, NXC>(a, ch.threads, s); break;
        case 5: launch_pair_R<5, NXC>(a, ch.threads, s); break;
        case 6: launch_pair_R<6, NXC>(a, ch.threads, s); break;
    }
}

// Pair variant for the compile-time widths.  Default on the 65- and 33-wide grids
// (config 3: 2.32e11 vs 2.04e11, config 2: 2.05e11 vs 1.70e11 DoF*it/s for column
// strips); on the 17-wide grid (9 pairs, tail warps only) column strips are faster
// (profiles/r01/SUMMARY.md).  TS_PCG_PAIR=1 forces the pair kernel for every
// compile-time width, 0 disables it.
Choice pair_choice(const GridG& g, int forced) {
    const int nx = g.n0 + 1;
    if (nx != 17 && nx != 33 && nx != 65) return {0, 0};
    int want = nx == 65 || nx == 33 ? 1 : 0;
    if (const char* env = std::getenv("TS_PCG_PAIR")) want = std::atoi(env);
    if (!want) return {0, 0};
    Choice ch = choose_pair(g, forced);
    if (!ch.R && forced) ch = choose_pair(g, 0);
    return ch;
}

// ------------------------------------------------------------ scheduling --
// Longest-first ticket order for the next sweep: counting sort of the problems by
// their last iteration count (buckets 0..1023, larger counts share the top bucket).
__global__ void __launch_bounds__(1024) k_order_by_iters(int n, const int* __restrict__ iters,
                                                         int* __restrict__ order) {
    constexpr int B = 1024;
    __shared__ int cnt[B];
    __shared__ int warp_tot[32];
    const int tid = threadIdx.x;
    cnt[tid] = 0;
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) atomicAdd(&cnt[B - 1 - min(iters[i], B - 1)], 1);
    __syncthreads();
    // exclusive scan of the 1024 bucket counts (one per thread)
    const int lane = tid & 31, warp = tid >> 5;
    const int v = cnt[tid];
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int w = warp_tot[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, w, o);
            if (lane >= o) w += y;
        }
        warp_tot[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    cnt[tid] = incl - v + (warp ? warp_tot[warp - 1] : 0);
    __syncthreads();
    for (int i = tid; i < n; i += blockDim.x) {
        const int pos = atomicAdd(&cnt[B - 1 - min(iters[i], B - 1)], 1);
        order[pos] = i;
    }
}

// ---------------------------------------------------------------- CSR PCG --
// cg_solve (linalg.cpp:103-161) for one system per block; vectors in global memory.
__global__ void __launch_bounds__(1024) k_csr_pcg(const CsrPcgArgs a) {
    __shared__ double red[kRedSlots * kRedStride];
    const int sys = blockIdx.x;
    const int n = a.n;
    const int* rp = a.row_ptr;
    const int* ci = a.col_idx;
    const double* A = a.vals + (size_t)sys * a.vals_stride;
    const double* b = a.b + (size_t)sys * n;
    double* x = a.x + (size_t)sys * n;
    double* r = a.scratch + (size_t)sys * 5 * n;
    double* z = r + n;
    double* p = z + n;
    double* Ap = p + n;
    double* dinv = Ap + n;
    int slot = 0;
    auto next = [&]() {
        double* s = red + slot * kRedStride;
        slot = slot == kRedSlots - 1 ? 0 : slot + 1;
        return s;
    };
    double bb[1] = {0.0};
    for (int i = threadIdx.x; i < n; i += blockDim.x) bb[0] = fma(b[i], b[i], bb[0]);
    block_sum<1>(bb, next());
    const double bnorm = sqrt(bb[0]);
    int* res = a.result_i + 3 * sys;
    if (bnorm == 0.0) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) x[i] = 0.0;
        if (threadIdx.x == 0) {
            res[0] = 1; res[1] = 0; res[2] = 0;
            a.result_d[sys] = 0.0;
        }
        return;
    }
    double s2[2] = {0.0, 0.0};
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double d = 0.0, y = 0.0;
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            const int c = ci[k];
            if (c == i) d = A[k];
            y = fma(A[k], x[c], y);
        }
        const double di = d != 0.0 ? 1.0 / d : 1.0;
        dinv[i] = di;
        const double ri = b[i] - y;
        r[i] = ri;
        const double zi = di * ri;
        p[i] = zi;
        s2[0] = fma(ri, zi, s2[0]);
        s2[1] = fma(ri, ri, s2[1]);
    }
    block_sum<2>(s2, next());  // barrier also publishes p
    double rz = s2[0];
    double rel = sqrt(s2[1]) / bnorm;
    int conv = rel <= a.tol, iters = 0, indef = 0;
    for (int it = 1; !conv && it <= a.maxit; ++it) {
        double t1[1] = {0.0};
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            double y = 0.0;
            for (int k = rp[i]; k < rp[i + 1]; ++k) y = fma(A[k], p[ci[k]], y);
            Ap[i] = y;
            t1[0] = fma(p[i], y, t1[0]);
        }
        block_sum<1>(t1, next());
        iters = it;
        if (t1[0] <= 0.0) {
            indef = 1;
            break;
        }
        const double alpha = rz / t1[0];
        double t2[2] = {0.0, 0.0};
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            x[i] = fma(alpha, p[i], x[i]);
            const double ri = fma(-alpha, Ap[i], r[i]);
            r[i] = ri;
            t2[0] = fma(ri, ri, t2[0]);
            const double zi = dinv[i] * ri;
            z[i] = zi;
            t2[1] = fma(ri, zi, t2[1]);
        }
        block_sum<2>(t2, next());
        rel = sqrt(t2[0]) / bnorm;
        if (rel <= a.tol) {
            conv = 1;
            break;
        }
        const double beta = t2[1] / rz;
        rz = t2[1];
        for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = fma(beta, p[i], z[i]);
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        res[0] = conv;
        res[1] = iters;
        res[2] = indef;
        a.result_d[sys] = rel;
    }
}

// cg_solve (linalg.cpp:103-161) on one large system per launch slot, cooperatively over
// the whole GPU (macro grids beyond ~90^2).  Dot products: per-block partials in global
// memory, summed in the same fixed order by every block (deterministic, identical in
// all threads).  The (up to two) systems of a launch — macro u and w — iterate in
// lockstep so they share every grid barrier, and the direction update p = z + beta p is
// folded into the next SpMV (each row recomputes its neighbours' new p from z and the
// previous p, double-buffered), which leaves two grid barriers per iteration.  Every
// value is computed by the same expression as the sequential algorithm, so results are
// unchanged bit for bit.
template <int K>
__device__ __forceinline__ void grid_sumk(double* partial, double (&v)[K], double* red, cg::grid_group& grid) {
    double t[K];
#pragma unroll
    for (int k = 0; k < K; ++k) t[k] = v[k];
    block_sum<K>(t, red);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int k = 0; k < K; ++k) partial[K * blockIdx.x + k] = t[k];
    }
    grid.sync();
#pragma unroll
    for (int k = 0; k < K; ++k) {
        double acc = 0.0;
        for (int b = threadIdx.x & 31; b < (int)gridDim.x; b += 32) acc += partial[K * b + k];
        v[k] = warp_sum(acc);
    }
}

__global__ void __launch_bounds__(512) k_csr_pcg_coop(const CsrPcgArgs a, double* partials) {
    __shared__ double red[kRedSlots * kRedStride];
    cg::grid_group grid = cg::this_grid();
    const int n = a.n;
    const int* rp = a.row_ptr;
    const int* ci = a.col_idx;
    const int gt = blockIdx.x * blockDim.x + threadIdx.x, gs = gridDim.x * blockDim.x;
    int pslot = 0;
    auto next_partial = [&]() {
        double* p = partials + (size_t)pslot * 4 * gridDim.x;
        pslot = pslot == 2 ? 0 : pslot + 1;
        return p;
    };
    for (int s0 = 0; s0 < a.n_sys; s0 += 2) {
        const int m = min(2, a.n_sys - s0);
        const double* A[2];
        const double* b[2];
        double *x[2], *r[2], *z[2], *pb[2][2], *Ap[2], *dinv[2];
        for (int q = 0; q < 2; ++q) {
            const int sys = s0 + min(q, m - 1);
            A[q] = a.vals + (size_t)sys * a.vals_stride;
            b[q] = a.b + (size_t)sys * n;
            x[q] = a.x + (size_t)sys * n;
            r[q] = a.scratch + (size_t)sys * 6 * n;
            z[q] = r[q] + n;
            pb[q][0] = z[q] + n;
            pb[q][1] = pb[q][0] + n;
            Ap[q] = pb[q][1] + n;
            dinv[q] = Ap[q] + n;
        }
        // ||b|| (linalg.cpp:108-114)
        double v4[4] = {0.0, 0.0, 0.0, 0.0};
        for (int q = 0; q < m; ++q)
            for (int i = gt; i < n; i += gs) v4[q] = fma(b[q][i], b[q][i], v4[q]);
        grid_sumk<4>(next_partial(), v4, red, grid);
        double bnorm[2], rz[2], rel[2], beta[2] = {0.0, 0.0};
        int active[2], conv[2] = {0, 0}, iters[2] = {0, 0}, indef[2] = {0, 0};
        for (int q = 0; q < 2; ++q) {
            bnorm[q] = sqrt(v4[q]);
            active[q] = q < m && bnorm[q] != 0.0;
            if (q < m && bnorm[q] == 0.0) conv[q] = 1;  // x := 0, converged, 0 iterations
            rel[q] = 0.0;
        }
        // r = b - A x, z = D^-1 r, p_(-1) = 0 (linalg.cpp:115-129)
        double t4[4] = {0.0, 0.0, 0.0, 0.0};
        for (int q = 0; q < m; ++q) {
            for (int i = gt; i < n; i += gs) {
                if (!active[q]) {
                    x[q][i] = 0.0;
                    continue;
                }
                double d = 0.0, y = 0.0;
                for (int k = rp[i]; k < rp[i + 1]; ++k) {
                    const int c = ci[k];
                    if (c == i) d = A[q][k];
                    y = fma(A[q][k], x[q][c], y);
                }
                const double di = d != 0.0 ? 1.0 / d : 1.0;
                dinv[q][i] = di;
                const double ri = b[q][i] - y;
                r[q][i] = ri;
                const double zi = di * ri;
                z[q][i] = zi;
                pb[q][0][i] = 0.0;  // p_0 = z_0 + 0 * p_(-1) in the first SpMV
                t4[2 * q] = fma(ri, zi, t4[2 * q]);
                t4[2 * q + 1] = fma(ri, ri, t4[2 * q + 1]);
            }
        }
        grid_sumk<4>(next_partial(), t4, red, grid);
        for (int q = 0; q < 2; ++q) {
            if (!active[q]) continue;
            rz[q] = t4[2 * q];
            rel[q] = sqrt(t4[2 * q + 1]) / bnorm[q];
            if (rel[q] <= a.tol) {
                conv[q] = 1;
                active[q] = 0;
            }
        }
        for (int it = 1; (active[0] || active[1]) && it <= a.maxit; ++it) {
            const int cur = it & 1, prv = cur ^ 1;
            // p_it = z + beta p_(it-1) on the fly; Ap = A p_it; pAp (linalg.cpp:131-137)
            double u4[4] = {0.0, 0.0, 0.0, 0.0};
            for (int q = 0; q < 2; ++q) {
                if (!active[q]) continue;
                const double* pp = pb[q][prv];
                const double* zz = z[q];
                const double bq = beta[q];
                for (int i = gt; i < n; i += gs) {
                    double y = 0.0;
                    for (int k = rp[i]; k < rp[i + 1]; ++k) {
                        const int c = ci[k];
                        y = fma(A[q][k], fma(bq, pp[c], zz[c]), y);
                    }
                    const double pi = fma(bq, pp[i], zz[i]);
                    pb[q][cur][i] = pi;
                    Ap[q][i] = y;
                    u4[q] = fma(pi, y, u4[q]);
                }
            }
            grid_sumk<4>(next_partial(), u4, red, grid);
            double alpha[2] = {0.0, 0.0};
            for (int q = 0; q < 2; ++q) {
                if (!active[q]) continue;
                iters[q] = it;
                if (u4[q] <= 0.0) {  // linalg.cpp:138-142
                    indef[q] = 1;
                    active[q] = 0;
                    continue;
                }
                alpha[q] = rz[q] / u4[q];
            }
            double w4[4] = {0.0, 0.0, 0.0, 0.0};
            for (int q = 0; q < 2; ++q) {
                if (!active[q]) continue;
                const double* pc = pb[q][cur];
                for (int i = gt; i < n; i += gs) {
                    x[q][i] = fma(alpha[q], pc[i], x[q][i]);
                    const double ri = fma(-alpha[q], Ap[q][i], r[q][i]);
                    r[q][i] = ri;
                    const double zi = dinv[q][i] * ri;
                    z[q][i] = zi;
                    w4[2 * q] = fma(ri, ri, w4[2 * q]);
                    w4[2 * q + 1] = fma(ri, zi, w4[2 * q + 1]);
                }
            }
            grid_sumk<4>(next_partial(), w4, red, grid);
            for (int q = 0; q < 2; ++q) {
                if (!active[q]) continue;
                rel[q] = sqrt(w4[2 * q]) / bnorm[q];
                if (rel[q] <= a.tol) {  // linalg.cpp:147-152
                    conv[q] = 1;
                    active[q] = 0;
                    continue;
                }
                beta[q] = w4[2 * q + 1] / rz[q];
                rz[q] = w4[2 * q + 1];
            }
        }
        if (gt == 0) {
            for (int q = 0; q < m; ++q) {
                int* res = a.result_i + 3 * (s0 + q);
                res[0] = conv[q];
                res[1] = iters[q];
                res[2] = indef[q];
                a.result_d[s0 + q] = rel[q];
            }
        }
        grid.sync();
    }
}

// macro_u_rhs / macro_w_rhs + constrain_rhs; blockIdx.y selects u (0) or w (1).
__global__ void k_macro_rhs(const MacroRhsArgs a) {
    const int s = blockIdx.y;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < a.n; i += gridDim.x * blockDim.x) {
        double raw = a.b_fixed[s][i];
        if (a.kappa[s] != 0.0) {
            double mb = 0.0;  // M0.apply(bI) row i (linalg.cpp:40-47)
            for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k)
                mb = fma(a.M0[k], a.coupling[s][a.col_idx[k]], mb);
            raw = fma(a.kappa[s], mb, raw);  // axpy (linalg.cpp:99-101)
        }
        a.raw[s][i] = raw;
        a.constrained[s][i] = a.cmask[s][i] ? a.cval[s][i] : raw - a.shift[s][i];
    }
}

// r_k = ||res_u|| + ||res_w|| + mean_i ||res_v,i|| (solver.cpp:100-117); one block.
__global__ void __launch_bounds__(1024) k_sweep_residual(const SweepResidualArgs a) {
    __shared__ double red[kRedSlots * kRedStride];
    double v[3] = {0.0, 0.0, 0.0};
    for (int i = threadIdx.x; i < a.n_macro; i += blockDim.x) {
#pragma unroll
        for (int s = 0; s < 2; ++s) {
            double y = 0.0;
            for (int k = a.row_ptr[i]; k < a.row_ptr[i + 1]; ++k)
                y = fma(a.A_e[s][k], a.x[s][a.col_idx[k]], y);
            const double rr = a.constrained[s][i] - y;
            v[s] = fma(rr, rr, v[s]);
        }
        v[2] += a.res_v[i];
    }
    block_sum<3>(v, red);
    double it[1] = {0.0};
    int mx = 0, mn = 0x7fffffff;
    for (int i = threadIdx.x; i < a.n_macro; i += blockDim.x) {
        const int k = a.iters[i];
        it[0] += (double)k;
        mx = max(mx, k);
        mn = min(mn, k);
    }
    block_sum<1>(it, red + kRedStride);
    int first_bad = 0x7fffffff;  // lowest failing system index (solver.cpp:92-97 reports the first)
    for (int i = threadIdx.x; i < a.n_macro; i += blockDim.x)
        if (a.status[i] != 0) {
            first_bad = i;
            break;
        }
    for (int o = 16; o > 0; o >>= 1) {
        mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
        first_bad = min(first_bad, __shfl_xor_sync(0xffffffffu, first_bad, o));
    }
    __shared__ int smx[32], smn[32], sbad[32];
    if ((threadIdx.x & 31) == 0) {
        smx[threadIdx.x >> 5] = mx;
        smn[threadIdx.x >> 5] = mn;
        sbad[threadIdx.x >> 5] = first_bad;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) {
            mx = max(mx, smx[w]);
            mn = min(mn, smn[w]);
            first_bad = min(first_bad, sbad[w]);
        }
        a.out[0] = sqrt(v[0]) + sqrt(v[1]) + v[2] / a.n_macro;
        a.out[1] = it[0] * a.n_micro;
        a.out[2] = mx;
        a.out[3] = mn;
        const int bad = first_bad == 0x7fffffff ? -1 : first_bad;
        a.out[4] = bad;
        a.out[5] = bad >= 0 ? a.status[bad] : 0;
        a.out[6] = bad >= 0 ? a.final_rel[bad] : 0.0;
    }
}

__global__ void k_micro_rhs(int n, const double* fixed, const double* rin, const double* rout,
                            int has_fixed, double kappa1, double kappa3, double u, double w,
                            double* b) {
    const bool use_u = kappa1 != 0.0 && u != 0.0, use_w = kappa3 != 0.0 && w != 0.0;
    const double cu = kappa1 * u, cw = kappa3 * w;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < n; k += gridDim.x * blockDim.x) {
        double bk = has_fixed ? fixed[k] : 0.0;
        if (use_u) bk = fma(cu, rin[k], bk);
        if (use_w) bk = fma(cw, rout[k], bk);
        b[k] = bk;
    }
}

struct CouplingArgs {
    GridG micro;
    int role;
    int micro_role[4];
    double GW[2];
    double Nf[2][2];
};

__global__ void k_coupling(const CouplingArgs c, int n_vec, const double* v, const double* len,
                           long long len_stride, double* out) {
    const int nf = c.micro.faces();
    const int n = c.micro.nodes();
    const int lane = threadIdx.x & 31;
    for (int i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); i < n_vec;
         i += gridDim.x * (blockDim.x >> 5)) {
        const double* vi = v + (size_t)i * n;
        const double* li = len + (size_t)i * len_stride;
        double tot = 0.0;
        for (int f = lane; f < nf; f += 32) {
            int side, n0, n1;
            face_info(c.micro, f, side, n0, n1);
            if (c.micro_role[side] != c.role) continue;
            const double scale = face_scale_of(c.micro, f);
            for (int q = 0; q < 2; ++q) {
                const double vq = vi[n0] * c.Nf[q][0] + vi[n1] * c.Nf[q][1];
                tot += c.GW[q] * vq * li[f * 2 + q] * scale;
            }
        }
        tot = warp_sum(tot);
        if (lane == 0) out[i] = tot;
    }
}

}  // namespace

size_t micro_pcg_smem_bytes(const GridG& g) {
    const Choice ch = choose(g, 0, 1 << 20);
    return ch.R ? smem_bytes_for(g, ch.R) : 0;
}

bool micro_pcg_fits(const GridG& g) { return choose(g, 0, 1 << 20).R != 0; }

MicroPlan plan_micro_pcg(const GridG& g, int forced, int n_problems) {
    if (!forced) {
        if (const char* env = std::getenv("TS_PCG_ROWS")) forced = std::atoi(env);
    }
    const Choice pc = pair_choice(g, forced);
    if (pc.R) {
        // per strip and pair: 6 halo-row / neighbour p + 4 carried coefficients + 2 p of the
        // next strip; per row pair 2 neighbour p + 3 neighbour coefficients + 10 own
        // coefficients (8 + 2 D^-1 in the r/z update where the diagonal is in registers) +
        // 2 p stores.  Own p never comes from SMEM (registers across iterations).
        const double per = (12.0 + 17.0 * pc.R) / (2.0 * pc.R);
        return {1, pc.R, pc.threads, 8.0 * per};
    }
    Choice ch = choose(g, forced, n_problems);
    if (!ch.R && forced) ch = choose(g, 0, n_problems);  // forced height does not fit
    const double per = (7.0 + 13.0 * ch.R) / (ch.R ? ch.R : 1);
    return {0, ch.R, ch.threads, ch.R ? 8.0 * per : 0.0};
}

int launch_micro_pcg(const MicroPcgArgs& a, cudaStream_t s) {
    const MicroPlan pl = plan_micro_pcg(a.micro, a.rows_per_thread, a.n_problems);
    const Choice ch{pl.R, pl.threads};
    if (pl.kernel == 1) {
        switch (a.micro.n0 + 1) {
            case 17: launch_pair_width<17>(a, ch, s); break;
            case 33: launch_pair_width<33>(a, ch, s); break;
            case 65: launch_pair_width<65>(a, ch, s); break;
        }
        return 1;
    }
    switch (ch.R) {
        case 2: launch_width<2>(a, ch.threads, s); break;
        case 3: launch_width<3>(a, ch.threads, s); break;
        case 4: launch_width<4>(a, ch.threads, s); break;
        case 5: launch_width<5>(a, ch.threads, s); break;
        case 7: launch_width<7>(a, ch.threads, s); break;
        case 9: launch_width<9>(a, ch.threads, s); break;
        case 13: launch_width<13>(a, ch.threads, s); break;
        case 17: launch_width<17>(a, ch.threads, s); break;
        case 22: launch_width<22>(a, ch.threads, s); break;
        default: return 0;
    }
    return 1;
}

constexpr int kCoopThreads = 512;

int csr_pcg_coop_blocks() {
    int dev = 0, sms = 148, per_sm = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_csr_pcg_coop, 512, 0);
    return sms * (per_sm < 1 ? 1 : (per_sm > 2 ? 2 : per_sm));
}

void launch_csr_pcg(const CsrPcgArgs& a, cudaStream_t s) {
    // Small systems: one block each.  Large ones (macro grids beyond ~90^2): the
    // cooperative whole-GPU kernel with the caller's grid-sized partials buffer.
    if (a.n <= 8192 || !a.partials) {
        k_csr_pcg<<<a.n_sys, 1024, 0, s>>>(a);
        return;
    }
    int threads = kCoopThreads;
    if (const char* e = std::getenv("TS_COOP_THREADS")) threads = std::atoi(e);
    if (threads < 64 || threads > 512 || threads % 32) threads = kCoopThreads;
    int nb = (a.n + threads - 1) / threads;
    const int blocks = csr_pcg_coop_blocks();
    if (nb > blocks) nb = blocks;
    CsrPcgArgs args = a;
    double* partials = a.partials;
    void* params[] = {&args, &partials};
    cudaLaunchCooperativeKernel((void*)k_csr_pcg_coop, nb, threads, params, 0, s);
}

void launch_order_by_iters(int n, const int* iters, int* order, cudaStream_t s) {
    k_order_by_iters<<<1, 1024, 0, s>>>(n, iters, order);
}

namespace {

__global__ void k_csr_to_stencil(int n_sys, GridG g, const int* __restrict__ rp, const int* __restrict__ ci,
                                 const double* __restrict__ vals, long long vals_stride, double* __restrict__ planes) {
    const int n = g.nodes(), nx = g.nx();
    for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < (long long)n_sys * n;
         t += (long long)gridDim.x * blockDim.x) {
        const int sys = (int)(t / n), i = (int)(t % n);
        const int ix = i % nx, iy = i / nx;
        double* pl = planes + (size_t)sys * 9 * n;
        for (int d = 0; d < 9; ++d) pl[(size_t)d * n + i] = 0.0;
        for (int k = rp[i]; k < rp[i + 1]; ++k) {
            const int c = ci[k];
            const int d = (c / nx - iy + 1) * 3 + (c % nx - ix + 1);
            pl[(size_t)d * n + i] = vals[(size_t)sys * vals_stride + k];
        }
    }
}

__global__ void k_macro_cg_result(const int* status, const int* iters, const double* rel, int* result_i,
                                  double* result_d) {
    const int s = threadIdx.x;
    if (s < 2) {
        result_i[3 * s + 0] = status[s] == 0;
        result_i[3 * s + 1] = iters[s];
        result_i[3 * s + 2] = status[s] == 1;
        result_d[s] = rel[s];
    }
}

}  // namespace

void launch_csr_to_stencil(int n_sys, const GridG& g, const int* row_ptr, const int* col_idx, const double* vals,
                           long long vals_stride, double* planes, cudaStream_t s) {
    const long long total = (long long)n_sys * g.nodes();
    k_csr_to_stencil<<<(int)((total + 255) / 256), 256, 0, s>>>(n_sys, g, row_ptr, col_idx, vals, vals_stride,
                                                                 planes);
}

namespace {

__global__ void k_sweep_stamp(SweepCtl* ctl, unsigned long long* stamps, int idx) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    stamps[4 * ctl->sweep + idx] = t;
}

// End of one device-side sweep: log the sweep scalars for the host, apply the stop test of
// src/solver.cpp:124-125 and stop on any CG failure (the host replays the logs with the same
// code as the eager loop, so messages and reports are identical), then set the while node.
__global__ void k_sweep_control(SweepCtl* ctl, const double* sweep_out, const double* cg_res_d,
                                const int* cg_res_i, double* log, double outer_tol, int max_outer,
                                cudaGraphConditionalHandle h) {
    const int done_before = ctl->sweep;  // sweeps completed before this one
    double* L = log + (size_t)kSweepLog * done_before;
    for (int k = 0; k < 8; ++k) L[k] = sweep_out[k];
    L[8] = cg_res_d[0];
    L[9] = cg_res_d[1];
    int* Li = reinterpret_cast<int*>(L + 10);
    for (int k = 0; k < 6; ++k) Li[k] = cg_res_i[k];
    bool stop = false;
    for (int q = 0; q < 2; ++q) stop = stop || cg_res_i[3 * q + 2] || !cg_res_i[3 * q];
    if (sweep_out[4] >= 0) stop = true;
    const int sweep = done_before + 1;
    if (!stop) {
        const double residual = sweep_out[0];
        if (residual < outer_tol || (sweep >= 2 && fabs(residual - ctl->prev) < outer_tol)) stop = true;
        ctl->prev = residual;
    }
    ctl->sweep = sweep;
    if (sweep >= max_outer) stop = true;
    cudaGraphSetConditional(h, stop ? 0u : 1u);
}

}  // namespace

void launch_sweep_stamp(SweepCtl* ctl, unsigned long long* stamps, int idx, cudaStream_t s) {
    k_sweep_stamp<<<1, 1, 0, s>>>(ctl, stamps, idx);
}

void launch_sweep_control(SweepCtl* ctl, const double* sweep_out, const double* cg_res_d, const int* cg_res_i,
                          double* log, double outer_tol, int max_outer, cudaGraphConditionalHandle h,
                          cudaStream_t s) {
    k_sweep_control<<<1, 1, 0, s>>>(ctl, sweep_out, cg_res_d, cg_res_i, log, outer_tol, max_outer, h);
}

void launch_macro_cg_result(const int* status, const int* iters, const double* rel, int* result_i,
                            double* result_d, cudaStream_t s) {
    k_macro_cg_result<<<1, 32, 0, s>>>(status, iters, rel, result_i, result_d);
}

void launch_macro_rhs(const MacroRhsArgs& a, cudaStream_t s) {
    dim3 grid((a.n + 255) / 256, 2);
    k_macro_rhs<<<grid, 256, 0, s>>>(a);
}

void launch_sweep_residual(const SweepResidualArgs& a, cudaStream_t s) {
    k_sweep_residual<<<1, 1024, 0, s>>>(a);
}

void launch_micro_rhs(int n, const double* fixed, const double* rin, const double* rout,
                      int has_fixed, double kappa1, double kappa3, double u, double w, double* b,
                      cudaStream_t s) {
    k_micro_rhs<<<(n + 255) / 256, 256, 0, s>>>(n, fixed, rin, rout, has_fixed, kappa1, kappa3, u, w, b);
}

void launch_coupling(const GridG& micro, const int* micro_role, int role, int n_vec, const double* v,
                     const double* face_len, long long len_stride, const double* GW,
                     const double (*Nf)[2], double* out, cudaStream_t s) {
    CouplingArgs c;
    c.micro = micro;
    c.role = role;
    for (int k = 0; k < 4; ++k) c.micro_role[k] = micro_role[k];
    c.GW[0] = GW[0];
    c.GW[1] = GW[1];
    for (int q = 0; q < 2; ++q)
        for (int k = 0; k < 2; ++k) c.Nf[q][k] = Nf[q][k];
    const int blocks = (n_vec + 7) / 8;
    k_coupling<<<blocks, 256, 0, s>>>(c, n_vec, v, face_len, len_stride, out);
}

}  // namespace tsb
