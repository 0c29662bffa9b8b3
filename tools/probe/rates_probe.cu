// Micro-probe: per-SM throughput of SHFL (64-bit), LDS.64, DADD and the
// latency of a dependent DADD chain on this GPU.  Used to pick the exchange
// mechanism of the temporally blocked 2D kernel.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/rates rates_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void k_shfl(double* out, int threads_active) {
    double a = threadIdx.x * 1.0, b = 2.0, c = 3.0, d = 4.0;
#pragma unroll 16
    for (int i = 0; i < ITERS; ++i) {
        a = __shfl_up_sync(0xffffffffu, a, 1);
        b = __shfl_down_sync(0xffffffffu, b, 1);
        c = __shfl_up_sync(0xffffffffu, c, 1);
        d = __shfl_down_sync(0xffffffffu, d, 1);
    }
    if (a + b + c + d == 12345.0) out[0] = a;
}

__global__ void k_lds(double* out) {
    extern __shared__ double sm[];
    for (int i = threadIdx.x; i < 8192; i += blockDim.x) sm[i] = i;
    __syncthreads();
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    int base = threadIdx.x;
#pragma unroll 16
    for (int i = 0; i < ITERS; ++i) {
        const volatile double* v = sm;
        s0 += v[(base + i) & 8191];
        s1 += v[(base + i + 1024) & 8191];
        s2 += v[(base + i + 2048) & 8191];
        s3 += v[(base + i + 3072) & 8191];
    }
    if (s0 + s1 + s2 + s3 == 12345.0) out[0] = s0;
}

template <int CHAINS>
__global__ void k_dadd(double* out, double inc) {
    double s[CHAINS];
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) s[c] = threadIdx.x + c;
    for (int i = 0; i < ITERS; ++i) {
#pragma unroll
        for (int c = 0; c < CHAINS; ++c) s[c] = __dadd_rn(s[c], inc);
    }
    double t = 0;
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) t += s[c];
    if (t == 12345.0) out[0] = t;
}

static float time_it(void (*launch)(), int reps = 5) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    launch();
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
}

static double* g_out;
static int g_blocks, g_threads;

int main() {
    cudaDeviceProp p;
    cudaGetDeviceProperties(&p, 0);
    int clk_khz = 0;
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
    cudaMalloc(&g_out, 64);
    const int sms = p.multiProcessorCount;
    printf("sms %d clock %.0f MHz\n", sms, clk_khz / 1e3);
    for (int threads : {256, 512, 1024}) {
        g_blocks = sms;
        g_threads = threads;
        float ms = time_it([] { k_shfl<<<g_blocks, g_threads>>>(g_out, g_threads); });
        double warp_ops = (double)sms * threads / 32 * ITERS * 4;  // 64-bit shuffles
        double per_sm_clk = warp_ops / sms / (ms * 1e-3 * clk_khz * 1e3);
        printf("shfl64  threads %4d: %.3f ms  warp-shfl64/clk/SM %.3f\n", threads, ms, per_sm_clk);
        cudaFuncSetAttribute(k_lds, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536);
        ms = time_it([] { k_lds<<<g_blocks, g_threads, 65536>>>(g_out); });
        double bytes = (double)sms * threads * ITERS * 4 * 8;
        printf("lds64   threads %4d: %.3f ms  B/clk/SM %.1f\n", threads, ms,
               bytes / sms / (ms * 1e-3 * clk_khz * 1e3));
    }
    for (int threads : {32, 128, 512, 1024}) {
        g_blocks = sms;
        g_threads = threads;
        float ms1 = time_it([] { k_dadd<1><<<g_blocks, g_threads>>>(g_out, 1e-9); });
        float ms8 = time_it([] { k_dadd<8><<<g_blocks, g_threads>>>(g_out, 1e-9); });
        double clk = clk_khz * 1e3;
        printf("dadd threads %4d: 1-chain %.3f ms (%.2f clk/iter/warp)  8-chain lanes/clk/SM %.1f\n",
               threads, ms1, ms1 * 1e-3 * clk / ITERS,
               (double)threads * 8 * ITERS / (ms8 * 1e-3 * clk));
    }
    return 0;
}
