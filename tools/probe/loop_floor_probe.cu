// Probe: per-iteration floor of a single-CTA sweep loop on B200 (the C1
// kernels): (a) __syncthreads only; (b) + a double warp butterfly, a
// cross-warp sum through shared memory and a data-dependent branch; (c) + an
// 8-point per-lane stencil update (10 dependent fp64 ops per point).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/lfp loop_floor_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 10000;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int MODE>
__global__ void k_loop(double* out, double tol) {
    __shared__ double red[2][4];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double x[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = threadIdx.x * 0.001 + j;
    double S = 0.0;
    for (int k = 0; k < ITERS; ++k) {
        double acc = 1e-3;
        if (MODE >= 2) {
            const double pl = __shfl_up_sync(0xffffffffu, x[7], 1);
            const double pr = __shfl_down_sync(0xffffffffu, x[0], 1);
            double nx[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                double y = __dadd_rn(0.0, __dmul_rn(-1.0, j == 0 ? pl : x[j - 1]));
                y = __dadd_rn(y, __dmul_rn(2.0, x[j]));
                y = __dadd_rn(y, __dmul_rn(-1.0, j == 7 ? pr : x[j + 1]));
                const double r = __dadd_rn(1.0, -y);
                nx[j] = __dadd_rn(x[j], __dmul_rn(0.3, __dmul_rn(0.5, r)));
                acc = fma(r, r, acc);
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) x[j] = nx[j];
        }
        if (MODE >= 1) {
            acc = wsum(acc);
            if (lane == 0) red[k & 1][wid] = acc;
        }
        __syncthreads();
        if (MODE >= 1) {
            S = red[k & 1][0] + red[k & 1][1] + red[k & 1][2] + red[k & 1][3];
            if (S < tol) break;
        }
    }
    if (threadIdx.x == 0) out[0] = S + x[0];
}

template <int MODE>
static float run(double* d) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    k_loop<MODE><<<1, 128>>>(d, -1.0);
    cudaEventRecord(a);
    k_loop<MODE><<<1, 128>>>(d, -1.0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

int main() {
    double* d;
    cudaMalloc(&d, 8);
    printf("(a) barrier only        : %.3f us/iter\n", run<0>(d) * 1e3 / ITERS);
    printf("(b) + butterfly + branch: %.3f us/iter\n", run<1>(d) * 1e3 / ITERS);
    printf("(c) + 8-point stencil   : %.3f us/iter\n", run<2>(d) * 1e3 / ITERS);
    return 0;
}
