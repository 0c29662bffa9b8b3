// Probe: latency of a grid-wide barrier on B200 with one CTA per SM -- the
// cooperative_groups grid sync vs a minimal monotonic-counter barrier (one
// atomic add with release per CTA, acquire spin on the counter).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/gbp grid_barrier_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;
constexpr int ITERS = 2000;

__global__ void k_cg(int* sink) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < ITERS; ++i) g.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = 1;
}

__global__ void k_counter(unsigned* counter, int* sink) {
    const unsigned nb = gridDim.x;
    for (int i = 0; i < ITERS; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned v;
            asm volatile("atom.add.release.gpu.u32 %0, [%1], 1;" : "=r"(v) : "l"(counter) : "memory");
            const unsigned target = (unsigned)(i + 1) * nb;
            unsigned cur = v + 1;
            while (cur < target)
                asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(cur) : "l"(counter) : "memory");
        }
        __syncthreads();
    }
    if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = 1;
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int* sink;
    unsigned* counter;
    cudaMalloc(&sink, 4);
    cudaMalloc(&counter, 4);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int threads : {256, 384}) {
        void* args1[] = {&sink};
        cudaLaunchCooperativeKernel((void*)k_cg, dim3(sms), dim3(threads), args1, 0, 0);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_cg, dim3(sms), dim3(threads), args1, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("threads %d  cg grid sync : %.3f us\n", threads, ms * 1e3 / ITERS);
        cudaMemset(counter, 0, 4);
        void* args2[] = {&counter, &sink};
        cudaLaunchCooperativeKernel((void*)k_counter, dim3(sms), dim3(threads), args2, 0, 0);
        cudaMemset(counter, 0, 4);
        cudaEventRecord(a);
        cudaLaunchCooperativeKernel((void*)k_counter, dim3(sms), dim3(threads), args2, 0, 0);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("threads %d  counter barrier: %.3f us  (%s)\n", threads, ms * 1e3 / ITERS,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
