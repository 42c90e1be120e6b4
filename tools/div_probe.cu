// Exhaustive-ish check of the split division (device_common.cuh div_recip/div_finish)
// and the stop threshold (rel_threshold) against the plain IEEE operations.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2103_17040_b200/csrc -I include \
//        tools/div_probe.cu -o /tmp/div_probe && /tmp/div_probe
#include <cstdio>
#include <cstdint>
#include "device_common.cuh"

using namespace tsb;

__device__ __forceinline__ uint64_t mix(uint64_t x) {
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return x;
}

// Random doubles: random sign/mantissa, exponent drawn from [-e, e] (plus specials).
__device__ double rnd(uint64_t s, int e) {
    const uint64_t r = mix(s);
    const int ex = (int)(mix(s ^ 0x9e3779b97f4a7c15ULL) % (uint64_t)(2 * e + 1)) - e;
    const uint64_t bits = (r & 0x800fffffffffffffULL) | ((uint64_t)(ex + 1023) << 52);
    return __longlong_as_double((long long)bits);
}

__global__ void k_div(uint64_t seed, long long n, int e, unsigned long long* bad) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        const double a = rnd(seed + 2 * i, e), b = rnd(seed + 2 * i + 1, e);
        const double q = div_finish(a, b, div_recip(b));
        const double ref = a / b;
        if (__double_as_longlong(q) != __double_as_longlong(ref) && !(isnan(q) && isnan(ref))) atomicAdd(bad, 1ULL);
    }
}

// One (b, tol) pair per warp (rel_threshold is warp-collective); every lane probes one
// point next to T and one random point near (tol*b)^2.
__global__ void k_thr(uint64_t seed, long long n, unsigned long long* bad) {
    const int lane = threadIdx.x & 31;
    const long long warps = (long long)gridDim.x * blockDim.x / 32;
    for (long long i = (blockIdx.x * (long long)blockDim.x + threadIdx.x) / 32; i < n; i += warps) {
        const double b = fabs(rnd(seed + 3 * i, 60));
        const double tol = fabs(rnd(seed + 3 * i + 1, 40));
        const double T = rel_threshold(b, tol);
        if (lane == 0 && (i & 63) == 0 && __double_as_longlong(rel_threshold_bisect(b, tol)) != __double_as_longlong(T) && isfinite(tol))
            atomicAdd(bad, 1ULL);  // the fallback agrees with the window search
        const double t = __longlong_as_double(__double_as_longlong(T) + lane - 16);
        if (t >= 0 && (t <= T) != rel_le_tol(t, b, tol)) atomicAdd(bad, 1ULL);
        const double g = tol * b;
        const double t2 = fabs(g * g * (1.0 + 1e-15 * (double)((int)(mix(seed + 3 * i + 2 + lane) % 2001) - 1000)));
        if ((t2 <= T) != rel_le_tol(t2, b, tol)) atomicAdd(bad, 1ULL);
    }
}

// Special values: one warp per (b, tol) pair, lanes test a list of residual norms.
__global__ void k_thr_special(unsigned long long* bad) {
    const double inf = __longlong_as_double(0x7ff0000000000000LL), nan = __longlong_as_double(0x7ff8000000000000LL);
    const double bs[] = {4.9e-324, 1e-300, 1e-20, 1.0, 3.7e5, 1e300, 1.7976931348623157e308, inf, nan};
    const double tols[] = {0.0, -0.0, 1e-300, 1e-10, 0.5, 1.0, 1e300, inf, nan, -1.0, -inf};
    const int w = blockIdx.x, lane = threadIdx.x;
    const int nb = sizeof(bs) / sizeof(bs[0]), nt = sizeof(tols) / sizeof(tols[0]);
    if (w >= nb * nt) return;
    const double b = bs[w / nt], tol = tols[w % nt];
    const double T = rel_threshold(b, tol);
    const double ts[32] = {0.0, -0.0, 4.9e-324, 1e-310, 1e-300, 1e-200, 1e-40, 1e-30, 1e-20, 1e-10, 0.25, 1.0, 2.0,
                           1e10, 1e100, 1e300, 1.7976931348623157e308, inf, nan, T,
                           __longlong_as_double(__double_as_longlong(T) + 1), __longlong_as_double(__double_as_longlong(T) - 1),
                           tol * tol * b * b, 1e-200 * b, b * b, b, tol, 1e-120, 1e-160, 1e-250, 3.0, 5e-324};
    const double t = ts[lane];
    if (!(t >= 0.0) && !isnan(t)) return;  // the residual norm^2 is never negative
    if ((t <= T) != rel_le_tol(t, b, tol)) {
        atomicAdd(bad, 1ULL);
        printf("special mismatch b=%g tol=%g t=%g T=%g\n", b, tol, t, T);
    }
}

int main(int argc, char** argv) {
    const bool quick = argc > 1;  // any argument: 64x fewer samples (the pytest run)
    unsigned long long* bad;
    cudaMalloc(&bad, sizeof(*bad));
    const long long n = quick ? 1LL << 25 : 1LL << 31;
    int fails = 0;
    for (int e : {4, 60, 300, 440, 460, 600, 1000, 1022}) {
        cudaMemset(bad, 0, sizeof(*bad));
        k_div<<<148 * 8, 256>>>(12345 + e, n, e, bad);
        unsigned long long h = 0;
        cudaMemcpy(&h, bad, sizeof(h), cudaMemcpyDeviceToHost);
        printf("div  exp range +-%4d: %lld samples, %llu mismatches\n", e, n, h);
        fails += h != 0;
    }
    cudaMemset(bad, 0, sizeof(*bad));
    const long long nt = quick ? 1LL << 18 : 1LL << 22;
    k_thr<<<148 * 4, 128>>>(777, nt, bad);
    unsigned long long h = 0;
    cudaMemcpy(&h, bad, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threshold: %lld (b, tol) pairs x 64 probes, %llu mismatches\n", nt, h);
    fails += h != 0;
    cudaMemset(bad, 0, sizeof(*bad));
    k_thr_special<<<128, 32>>>(bad);
    cudaMemcpy(&h, bad, sizeof(h), cudaMemcpyDeviceToHost);
    printf("threshold special values: %llu mismatches\n", h);
    fails += h != 0;
    const cudaError_t err = cudaDeviceSynchronize();
    printf("%s\n", err == cudaSuccess && !fails ? "div_probe OK" : "div_probe FAILED");
    return err == cudaSuccess && !fails ? 0 : 1;
}
