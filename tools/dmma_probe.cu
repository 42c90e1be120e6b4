// Probe: warp-wide FP64 sum with two DMMA m8n8k4 (no shuffles) vs a shuffle butterfly.
// Checks that every lane gets the same bits, the result is within a few ulps of the
// exact sum, and times both in a dependent loop.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double dmma_1x4(double a, double b, double c) {
    double d0, d1;
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};\n"
                 : "=d"(d0), "=d"(d1)
                 : "d"(a), "d"(b), "d"(c), "d"(c));
    return d0 + d1 * 0.0;  // keep both outputs live without changing d0
}

// Sum of v over the 32 lanes; identical bits in every lane.
__device__ __forceinline__ double warp_sum_mma(double v) {
    double g0, g1;
    // step 1: A = ones, B[k][j] = v(lane = 4j + k)  ->  D[i][j] = g_j (sum of lanes 4j..4j+3)
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};\n"
                 : "=d"(g0), "=d"(g1)
                 : "d"(1.0), "d"(v), "d"(0.0), "d"(0.0));
    // lane holds g_{2t}, g_{2t+1} (t = lane % 4)
    const double h = g0 + g1;
    double s0, s1;
    // step 2: A[i][k] = h_k, B = ones  ->  D[i][j] = sum_k h_k
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};\n"
                 : "=d"(s0), "=d"(s1)
                 : "d"(h), "d"(1.0), "d"(0.0), "d"(0.0));
    return s0;
}

__device__ __forceinline__ double warp_sum_shfl(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__global__ void k_check(const double* in, double* out_mma, double* out_shfl, int* mismatch) {
    const int lane = threadIdx.x & 31, w = blockIdx.x;
    const double v = in[w * 32 + lane];
    const double a = warp_sum_mma(v), b = warp_sum_shfl(v);
    const double a0 = __shfl_sync(0xffffffffu, a, 0);
    if (__double_as_longlong(a0) != __double_as_longlong(a)) atomicAdd(mismatch, 1);
    if (lane == 0) {
        out_mma[w] = a;
        out_shfl[w] = b;
    }
}

template <int MODE>
__global__ void k_time(int iters, double* sink, long long* cyc) {
    double v = threadIdx.x * 1e-3 + blockIdx.x;
    const long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
        const double s = MODE ? warp_sum_mma(v) : warp_sum_shfl(v);
        v = v * 0.5 + s * 1e-9;
    }
    const long long t1 = clock64();
    sink[blockIdx.x * blockDim.x + threadIdx.x] = v;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    const int W = 4096;
    double *in, *om, *os, *sink;
    int* mm;
    long long* cyc;
    cudaMallocManaged(&in, W * 32 * 8);
    cudaMallocManaged(&om, W * 8);
    cudaMallocManaged(&os, W * 8);
    cudaMallocManaged(&mm, 4);
    cudaMallocManaged(&sink, 148 * 1024 * 8);
    cudaMallocManaged(&cyc, 148 * 8);
    unsigned long long s = 12345;
    for (int i = 0; i < W * 32; ++i) {
        s = s * 6364136223846793005ULL + 1442695040888963407ULL;
        in[i] = ((double)(s >> 11) / 9007199254740992.0 - 0.5) * ((i % 7) ? 1.0 : 1e6);
    }
    *mm = 0;
    k_check<<<W, 32>>>(in, om, os, mm);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
        printf("error %s\n", cudaGetErrorString(e));
        return 1;
    }
    double maxrel = 0;
    for (int w = 0; w < W; ++w) {
        long double ex = 0;
        for (int l = 0; l < 32; ++l) ex += in[w * 32 + l];
        double sc = 0;
        for (int l = 0; l < 32; ++l) sc += fabs(in[w * 32 + l]);
        const double r = fabs((double)(om[w] - ex)) / sc;
        if (r > maxrel) maxrel = r;
    }
    printf("lane mismatches %d, max |mma - exact| / sum|v| = %.3e\n", *mm, maxrel);
    for (int mode = 0; mode < 2; ++mode)
        for (int warps : {1, 12}) {
            if (mode) k_time<1><<<148, warps * 32>>>(10000, sink, cyc);
            else k_time<0><<<148, warps * 32>>>(10000, sink, cyc);
            cudaDeviceSynchronize();
            double avg = 0;
            for (int b = 0; b < 148; ++b) avg += cyc[b];
            printf("%s warps %2d: %.1f cycles per warp sum (per SM, all warps)\n", mode ? "mma " : "shfl", warps,
                   avg / 148 / 10000);
        }
    return 0;
}
