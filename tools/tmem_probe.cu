// Microbenchmark: tcgen05.ld (TMEM -> registers) throughput per SM on B200, alone and
// mixed with LDS.64, for a non-MMA kernel that keeps per-thread data in TMEM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tmem_probe tmem_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

#define CK(x)                                                                         \
    do {                                                                              \
        cudaError_t e = (x);                                                          \
        if (e != cudaSuccess) {                                                       \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            return 1;                                                                 \
        }                                                                             \
    } while (0)

template <int X>
__device__ __forceinline__ void tld(uint32_t taddr, uint32_t (&v)[X]);

template <>
__device__ __forceinline__ void tld<2>(uint32_t taddr, uint32_t (&v)[2]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];\n" : "=r"(v[0]), "=r"(v[1]) : "r"(taddr));
}
template <>
__device__ __forceinline__ void tld<4>(uint32_t taddr, uint32_t (&v)[4]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3])
                 : "r"(taddr));
}
template <>
__device__ __forceinline__ void tld<8>(uint32_t taddr, uint32_t (&v)[8]) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];\n"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                 : "r"(taddr));
}
template <>
__device__ __forceinline__ void tld<32>(uint32_t taddr, uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
          "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(taddr));
}
template <>
__device__ __forceinline__ void tld<16>(uint32_t taddr, uint32_t (&v)[16]) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]), "=r"(v[8]),
          "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}

__device__ __forceinline__ void tst8(uint32_t taddr, const uint32_t (&v)[8]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};\n" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
}
__device__ __forceinline__ void twait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void twait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }

// mode 0: TMEM loads only; 1: LDS.64 only; 2: both interleaved (same count each).
template <int X>
__global__ void __launch_bounds__(1024, 1) k_probe(int iters, int mode, int lds_per, int batch, unsigned long long* cycles,
                                                    double* sink, int* bad) {
    __shared__ uint32_t s_taddr;
    __shared__ double sbuf[4096];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
    for (int k = threadIdx.x; k < 4096; k += blockDim.x) sbuf[k] = k * 0.5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                         (uint32_t)__cvta_generic_to_shared(&s_taddr)),
                     "n"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t base = s_taddr;
    const int per_sp = (nw + 3) / 4;
    const int cols = 512 / per_sp / 8 * 8;  // columns owned by this warp
    const uint32_t my = base + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * cols);
    // fill own columns with a pattern and verify a round trip
    for (int c = 0; c + 8 <= cols; c += 8) {
        uint32_t v[8];
        for (int q = 0; q < 8; ++q) v[q] = (uint32_t)(warp * 100000 + lane * 1000 + c + q);
        tst8(my + c, v);
    }
    twait_st();
    for (int c = 0; c + 8 <= cols; c += 8) {
        uint32_t v[8];
        tld<8>(my + c, v);
        twait_ld();
        for (int q = 0; q < 8; ++q)
            if (v[q] != (uint32_t)(warp * 100000 + lane * 1000 + c + q)) atomicAdd(bad, 1);
    }
    __syncthreads();
    double acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    uint32_t xacc = 0;
    const int span = cols - 4 * X;  // >= 0 for X <= cols / 4
    const unsigned long long t0 = clock64();
    int c = 0;
    for (int it = 0; it < iters; ++it) {
        if (mode != 1) {
            uint32_t v0[X], v1[X], v2[X], v3[X];
            tld<X>(my + c, v0);
            if (batch > 1) tld<X>(my + c + X, v1);
            if (batch > 2) tld<X>(my + c + 2 * X, v2);
            if (batch > 3) tld<X>(my + c + 3 * X, v3);
            if (mode == 2) {
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    if (q < lds_per) acc[q] += sbuf[(threadIdx.x + q * 256 + it * 32) & 4095];
            }
            twait_ld();
#pragma unroll
            for (int q = 0; q < X; ++q) {
                xacc += v0[q];
                if (batch > 1) xacc ^= v1[q];
                if (batch > 2) xacc += v2[q];
                if (batch > 3) xacc ^= v3[q];
            }
        } else {
#pragma unroll
            for (int q = 0; q < 8; ++q)
                if (q < lds_per) acc[q] += sbuf[(threadIdx.x + q * 256 + it * 32) & 4095];
        }
        c += X;
        if (c > span) c = 0;
    }
    const unsigned long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc[0] + acc[1] + acc[2] + acc[3] + acc[4] + acc[5] + acc[6] + acc[7] + xacc;
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(base), "n"(512));
}

template <int X>
int run(int threads, int mode, int lds_per, int batch = 1) {
    const int blocks = 148, iters = 20000;
    unsigned long long* cyc;
    double* sink;
    int* bad;
    CK(cudaMalloc(&cyc, blocks * 8));
    CK(cudaMalloc(&sink, (size_t)blocks * threads * 8));
    CK(cudaMalloc(&bad, 4));
    CK(cudaMemset(bad, 0, 4));
    k_probe<X><<<blocks, threads>>>(iters, mode, lds_per, batch, cyc, sink, bad);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    unsigned long long h[148];
    int hb = 0;
    CK(cudaMemcpy(h, cyc, sizeof h, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(&hb, bad, 4, cudaMemcpyDeviceToHost));
    double avg = 0;
    for (int b = 0; b < blocks; ++b) avg += h[b];
    avg /= blocks;
    const double tbytes = mode != 1 ? (double)iters * (threads / 32) * 32 * X * 4 * batch : 0.0;
    const double sbytes = mode != 0 ? (double)iters * threads * lds_per * 8 : 0.0;
    printf("x%-2d b%d warps %2d mode %d lds/it %d: %8.0f cyc  TMEM %6.1f B/cyc/SM  SMEM %6.1f B/cyc/SM  bad=%d\n", X, batch,
           threads / 32, mode, lds_per, avg, tbytes / avg, sbytes / avg, hb);
    cudaFree(cyc);
    cudaFree(sink);
    cudaFree(bad);
    return 0;
}

int main() {
    run<2>(32, 0, 0, 1);   // latency: one warp, one load per wait
    run<16>(32, 0, 0, 1);
    for (int w : {4, 8, 12, 16}) {
        run<16>(w * 32, 0, 0, 1);
        run<16>(w * 32, 0, 0, 4);
        run<32>(w * 32, 0, 0, 2);
    }
    for (int w : {8, 12, 16}) {
        run<4>(w * 32, 1, 8);
        run<16>(w * 32, 2, 8, 4);
        run<16>(w * 32, 2, 4, 2);
    }
    return 0;
}
