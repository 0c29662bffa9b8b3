// Grid-wide building blocks shared by the cycle kernels: the single-sweep
// row walker, the cooperative grid barrier and the deterministic reduction of
// per-CTA residual partials.
#pragma once

#include <cooperative_groups.h>

#include "srj_common.cuh"
#include "srj_stencil.cuh"

namespace srj {

// kSweepDiff: sweep returning max |x' - x| (solution-difference norm,
// reference solver.py:224-228) instead of sum r^2.
enum Mode { kSweep = 0, kResid = 1, kMatvec = 2, kSweepDiff = 3 };

// Walk the 32-point x-row units [u0, u1) of the grid.  Warps take units
// round-robin so a CTA streams through consecutive rows together (coalesced
// rows; the y/z neighbour rows are still hot in L1/L2).  Two units per warp
// iteration keep two independent load groups in flight.
template <int FAM, int MODE>
__device__ __forceinline__ double walk_units(const Geom& g, const double* __restrict__ x,
                                             double* __restrict__ out,
                                             const double* __restrict__ b, double w,
                                             int u0, int u1) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double acc = 0.0;
    for (int u = u0 + warp; u < u1; u += nw) {
        const int row = u / g.upr;
        const int i = (u - row * g.upr) * 32 + lane;
        if (i < g.nx) {
            const int j = (FAM == F3D) ? row % g.ny : row;
            const long long k = (long long)row * g.nx + i;
            double xc, inv;
            const double y = apply_at<FAM>(g, x, k, i, j, xc, inv);
            if constexpr (MODE == kMatvec) {
                out[k] = y;
            } else if constexpr (MODE == kSweepDiff) {
                const double r = DSUB(__ldg(b + k), y);
                const double xn = relax(xc, inv, r, w);
                out[k] = xn;
                acc = nanmax(acc, fabs(DSUB(xn, xc)));
            } else {
                const double r = DSUB(__ldg(b + k), y);
                acc = fma(r, r, acc);
                if constexpr (MODE == kSweep) out[k] = relax(xc, inv, r, w);
            }
        }
    }
    return acc;
}

__device__ __forceinline__ void grid_barrier() {
    SRJ_JITTER(5);
    if (gridDim.x == 1) {
        __syncthreads();
    } else {
        cooperative_groups::this_grid().sync();
    }
}

// Sum of part[0..nb) in a fixed order; identical bits in every thread of
// every CTA (all CTAs run the same code on the same data).
__device__ __forceinline__ double reduce_partials(const double* part, int nb, double* sh) {
    // four independent loads in flight per thread, added in ascending order (an
    // absent entry adds +0)
    double s = 0.0;
    for (int q0 = threadIdx.x; q0 < nb; q0 += 4 * blockDim.x) {
        double v[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int q = q0 + k * (int)blockDim.x;
            v[k] = q < nb ? __ldcg(part + q) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) s += v[k];
    }
    return block_allsum(s, sh);
}

// Non-cooperative grid sum: every CTA contributes `acc`; the last CTA to
// arrive reduces the per-CTA values in a fixed order into *result and re-arms
// the counter (threadfence-reduction pattern).
__device__ __forceinline__ void last_block_sum(double acc, double* block_part, unsigned* counter,
                                               double* result, double* sh) {
    __shared__ int s_last;
    acc = block_allsum(acc, sh);
    if (threadIdx.x == 0) {
        block_part[blockIdx.x] = acc;
        __threadfence();
        const unsigned ticket = atomicAdd(counter, 1u);
        s_last = ticket == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        const double s = reduce_partials(block_part, gridDim.x, sh);
        if (threadIdx.x == 0) {
            *result = s;
            *counter = 0u;
        }
    }
}

// Block sums of h <= H per-thread values at once (two barriers in total):
// out[t] = sum over the block of v[t].  `sh` needs 32*H doubles, `out` H.
template <int H>
__device__ __forceinline__ void block_sums(const double (&v)[H], int h, double* sh, double* out) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int t = 0; t < H; ++t) {
        if (t < h) {
            const double s = warp_allsum(v[t]);
            if (lane == 0) sh[wid * H + t] = s;
        }
    }
    __syncthreads();
    if (wid < h) {
        double s = lane < nw ? sh[lane * H + wid] : 0.0;
        s = warp_allsum(s);
        if (lane == 0) out[wid] = s;
    }
    __syncthreads();
}

// out[t] = sum_q part[t*nb + q] for t < h (h <= warps per block), fixed order:
// warp t strides over the nb partials, then a butterfly.  One barrier.
__device__ __forceinline__ void reduce_partials_multi(const double* part, int nb, int h,
                                                      double* out) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    if (wid < h) {
        // Eight independent loads in flight per lane (one L2 round trip for up to
        // 256 CTAs instead of one per 32), added in the same ascending order; an
        // absent entry adds +0, which leaves a sum of squares unchanged.
        double s = 0.0;
        for (int q0 = 0; q0 < nb; q0 += 256) {
            double v[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int q = q0 + lane + 32 * k;
                v[k] = q < nb ? __ldcg(part + wid * nb + q) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) s += v[k];
        }
        s = warp_allsum(s);
        if (lane == 0) out[wid] = s;
    }
    __syncthreads();
}

}  // namespace srj
