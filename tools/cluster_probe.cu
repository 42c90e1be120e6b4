// Probe: cost of a 2-CTA cluster exchange step (DSMEM store to the partner + cluster
// barrier) vs a CTA __syncthreads, per iteration, 384 threads per CTA, 1 CTA per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o cluster_probe cluster_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__device__ __forceinline__ void cluster_sync_ar() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n" ::: "memory");
    asm volatile("barrier.cluster.wait.acquire.aligned;\n" ::: "memory");
}

template <int MODE>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(384, 1)
    k_probe(int iters, long long* cyc, double* sink) {
    __shared__ double buf[2][256];
    extern __shared__ double big[];
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    double* peer = cl.map_shared_rank(&buf[0][0], rank ^ 1);
    const int tid = threadIdx.x;
    double acc = tid;
    if (tid < 256) buf[0][tid] = buf[1][tid] = 0.0;
    cl.sync();
    const long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const int s = it & 1;
        if (MODE == 0) {  // CTA barrier only
            if (tid < 65) buf[s][tid] = acc;
            __syncthreads();
            acc += buf[s][(tid + 1) & 63] * 1e-9;
        } else if (MODE == 1) {  // DSMEM row store + cluster barrier
            if (tid < 65) peer[s * 256 + tid] = acc;
            cluster_sync_ar();
            acc += buf[s][(tid + 1) & 63] * 1e-9;
        } else {  // cluster barrier only
            cluster_sync_ar();
            acc += 1e-9;
        }
    }
    const long long t1 = clock64();
    cl.sync();
    if (tid == 0) cyc[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + tid] = acc + big[0] * 0.0;
}

int main() {
    const int blocks = 148, iters = 20000;
    long long* cyc;
    double* sink;
    cudaMallocManaged(&cyc, blocks * 8);
    cudaMallocManaged(&sink, blocks * 384 * 8);
    const size_t dyn = 200 * 1024;  // force one CTA per SM
    const char* names[3] = {"CTA __syncthreads", "DSMEM row + cluster barrier", "cluster barrier only"};
    for (int mode = 0; mode < 3; ++mode) {
        cudaError_t e;
        if (mode == 0) {
            cudaFuncSetAttribute(k_probe<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
            k_probe<0><<<blocks, 384, dyn>>>(iters, cyc, sink);
        } else if (mode == 1) {
            cudaFuncSetAttribute(k_probe<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
            k_probe<1><<<blocks, 384, dyn>>>(iters, cyc, sink);
        } else {
            cudaFuncSetAttribute(k_probe<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dyn);
            k_probe<2><<<blocks, 384, dyn>>>(iters, cyc, sink);
        }
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) {
            printf("%s: error %s\n", names[mode], cudaGetErrorString(e));
            return 1;
        }
        double avg = 0;
        for (int b = 0; b < blocks; ++b) avg += cyc[b];
        printf("%-30s %.1f cycles per iteration\n", names[mode], avg / blocks / iters);
    }
    return 0;
}
