// Batched small-system SRJ cycles: the data-collection workload (SURVEY §8
// f1, reference datacollect._run_trial, datacollect.py:79-117).  A collection
// step runs up to three candidate cycles per trial from the same snapshot, on
// 1D Dirichlet Poisson systems of a few hundred unknowns, for thousands of
// independent trials: one CTA per candidate cycle, the iterate held in shared
// memory for all M sweeps, one launch for the whole step.
//
// Arithmetic per point is the reference's (srj_stencil.cuh recipe); the cycle
// has no stopping rule (run_cycle without `stopping`), so every job applies
// all M sweeps and reports the squared residual of its final iterate.
#include <cuda_runtime.h>

#include "../../include/srj.h"
#include "srj_common.cuh"
#include "srj_stencil.cuh"

namespace srj {

constexpr int kBatchThreads = 256;
constexpr int kBatchMaxN = 12288;  // 2 x n doubles of shared memory per CTA

__global__ void __launch_bounds__(kBatchThreads) k_batch_cycles_1d(
    const srj_batch_job* __restrict__ jobs, const double* __restrict__ omega_pool,
    double* __restrict__ x_pool, const double* __restrict__ b_pool, double* __restrict__ sumsq) {
    extern __shared__ double sm[];
    __shared__ double red[32];
    const srj_batch_job job = jobs[blockIdx.x];
    const int n = job.n;
    double* xa = sm;
    double* xb = sm + n + 2;  // each buffer carries a zero ghost at both ends
    const double* b = b_pool + job.b_off;
    const double dx2 = DMUL(n + 1.0, n + 1.0);  // (N+1.0)**2 (reference problems.py:58)
    const double c = DMUL(-1.0, dx2), d = DMUL(2.0, dx2);
    const double inv = __ddiv_rn(1.0, d);
    for (int i = threadIdx.x; i < n + 2; i += blockDim.x) {
        xa[i] = (i >= 1 && i <= n) ? x_pool[job.x_in_off + i - 1] : 0.0;
        xb[i] = 0.0;
    }
    __syncthreads();
    const double* om = omega_pool + job.omega_off;
    for (int k = 0; k < job.M; ++k) {
        const double w = __ldg(om + k);
        for (int i = threadIdx.x + 1; i <= n; i += blockDim.x) {
            double y = DADD(0.0, DMUL(c, xa[i - 1]));
            y = DADD(y, DMUL(d, xa[i]));
            y = DADD(y, DMUL(c, xa[i + 1]));
            xb[i] = relax(xa[i], inv, DSUB(__ldg(b + i - 1), y), w);
        }
        __syncthreads();
        double* t = xa;
        xa = xb;
        xb = t;
    }
    double acc = 0.0;
    for (int i = threadIdx.x + 1; i <= n; i += blockDim.x) {
        double y = DADD(0.0, DMUL(c, xa[i - 1]));
        y = DADD(y, DMUL(d, xa[i]));
        y = DADD(y, DMUL(c, xa[i + 1]));
        const double r = DSUB(__ldg(b + i - 1), y);
        acc = fma(r, r, acc);
        x_pool[job.x_out_off + i - 1] = xa[i];
    }
    acc = block_allsum(acc, red);
    if (threadIdx.x == 0) sumsq[blockIdx.x] = acc;
}

}  // namespace srj

extern "C" int srj_batch_cycles_1d(const srj_batch_job* jobs_dev, int32_t njobs, int32_t max_n,
                                   const double* omega_pool, double* x_pool,
                                   const double* b_pool, double* sumsq_dev, int32_t device,
                                   void* stream) {
    if (njobs < 0 || max_n < 1 || max_n > srj::kBatchMaxN) return SRJ_BAD_ARGUMENT;
    if (njobs == 0) return SRJ_OK;
    if (!jobs_dev || !omega_pool || !x_pool || !b_pool || !sumsq_dev) return SRJ_BAD_ARGUMENT;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != device) cudaSetDevice(device);
    const size_t smem = 2 * (size_t)(max_n + 2) * sizeof(double);
    cudaError_t e = cudaSuccess;
    if (smem > 48 * 1024)
        e = cudaFuncSetAttribute(srj::k_batch_cycles_1d,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e == cudaSuccess) {
        srj::k_batch_cycles_1d<<<njobs, srj::kBatchThreads, smem, (cudaStream_t)stream>>>(
            jobs_dev, omega_pool, x_pool, b_pool, sumsq_dev);
        e = cudaGetLastError();
    }
    if (prev >= 0 && prev != device) cudaSetDevice(prev);
    return e == cudaSuccess ? SRJ_OK : SRJ_CUDA_ERROR;
}
