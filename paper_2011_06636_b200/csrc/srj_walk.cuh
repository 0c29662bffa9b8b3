// Grid-wide building blocks shared by the cycle kernels: the single-sweep
// row walker, the cooperative grid barrier and the deterministic reduction of
// per-CTA residual partials.
#pragma once

#include <cooperative_groups.h>

#include "srj_common.cuh"
#include "srj_stencil.cuh"

namespace srj {

enum Mode { kSweep = 0, kResid = 1, kMatvec = 2 };

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
    if (gridDim.x == 1) {
        __syncthreads();
    } else {
        cooperative_groups::this_grid().sync();
    }
}

// Sum of part[0..nb) in a fixed order; identical bits in every thread of
// every CTA (all CTAs run the same code on the same data).
__device__ __forceinline__ double reduce_partials(const double* part, int nb, double* sh) {
    double s = 0.0;
    for (int q = threadIdx.x; q < nb; q += blockDim.x) s += __ldcg(part + q);
    return block_allsum(s, sh);
}

}  // namespace srj
