// Per-cycle driver shared by the persistent temporally blocked kernels
// (srj_tb.cu: constant coefficient, srj_tbvar.cu: variable coefficient).
//
// A cycle of M sweeps runs as ceil(M / s) passes of h <= s sub-sweeps.  Each
// pass accumulates, per sub-sweep t, the squared residual of its INPUT iterate
// x_{k0+t} over the CTA's owned points; after a grid barrier every CTA reduces
// the per-CTA partials in the same fixed order (identical bits in all CTAs)
// and applies the reference's per-sweep stopping rule (solver.py:216-222,
// 235-239): a stop at sweep k0+j, j >= 1, re-runs the pass with j sub-sweeps
// from its intact input buffer (rollback); j = 0 returns the input buffer.
// Without a stop, a residual-only pass gives res(x_M) (solver.py:233-234,
// 248-249).  While the stop test runs, the next pass's first tile is already
// being loaded (speculative TMA, drained on a stop).
#pragma once

#include "srj_common.cuh"
#include "srj_tb.cuh"
#include "srj_walk.cuh"

namespace srj {

struct TbArgs {
    Geom g;
    double* buf0;
    double* buf1;
    const double* b;
    const double* omegas;
    int M, s;
    double tol, baseline;
    double* partials;  // [2][kTbMaxSub][gridDim.x]
    double* hist;
    int* out_i;
    double* out_d;
    int tiles_x, ntiles;
    // Owned rows [row_lo, row_hi) (2D): tiles cover these rows; rows outside
    // them but inside the grid are updated as ring points, never stored or
    // accumulated (slab with deep ghost rows).  Whole grid: 0, ny.
    int row_lo, row_hi;
    // Pass mode (slab kernels): one pass of M <= s sweeps, no stop test and no
    // residual tail; sums[t] = owned sum of r^2 of sub-sweep t (fixed order).
    double* sums;
};

// pass(in, xout, k0, h, acc, accumulate, first_issued): one pass of h
//   sub-sweeps over this CTA's tiles, reading buffer `in` (0: buf0, 1: buf1)
//   and writing xout; acc[t] += owned r^2 of sub-sweep t when accumulating.
// issue(in): (thread 0) start the TMA of this CTA's first tile of buffer `in`.
// drain(): every thread waits for the outstanding TMA.
// has_tiles: this CTA owns at least one tile.
// SLAB: pass mode (the slab instantiation of a kernel; see TbArgs::sums).
// TAIL_PASS: the residual of the cycle's final iterate is a pass with h = 0
// (xout == nullptr; acc[0] = owned sum of r^2) instead of the generic walker.
template <int S, int FAM, bool SLAB, bool TAIL_PASS = false, class Pass, class Issue, class Drain>
__device__ __forceinline__ void tb_run_cycle(const TbArgs& a, bool has_tiles, Pass&& pass,
                                             Issue&& issue, Drain&& drain) {
    __shared__ double sh[32 * S];
    __shared__ double red[S];
    __shared__ double sh1[32];
    const int nb = gridDim.x;
    double* const buf[2] = {a.buf0, a.buf1};
    const int npasses = (a.M + a.s - 1) / a.s;
    int executed = a.M, status = kStatusRan, result = npasses & 1;
    double S2 = 0.0, res = 0.0;
    bool stopped = false, issued = false;
    for (int p = 0; p < npasses && !stopped; ++p) {
        const int k0 = p * a.s;
        const int h = min(a.s, a.M - k0);
        double acc[S];
#pragma unroll
        for (int t = 0; t < S; ++t) acc[t] = 0.0;
        pass(p & 1, buf[(p + 1) & 1], k0, h, acc, true, issued);
        issued = false;
        double* part = a.partials + (size_t)(p & 1) * kTbMaxSub * nb;
        block_sums<S>(acc, h, sh, red);
        if (threadIdx.x < h) part[threadIdx.x * nb + blockIdx.x] = red[threadIdx.x];
        grid_barrier();
        if constexpr (SLAB) {  // pass mode: raw sums, no decision, no tail
            reduce_partials_multi(part, nb, h, red);
            if (blockIdx.x == 0 && threadIdx.x < h) a.sums[threadIdx.x] = red[threadIdx.x];
            if (blockIdx.x == 0 && threadIdx.x == 0) {
                a.out_i[0] = h;
                a.out_i[1] = kStatusRan;
                a.out_i[2] = (p + 1) & 1;
            }
            return;
        }
        // Speculatively start the next pass's first tile while the stop test runs.
        if (p + 1 < npasses && has_tiles) {
            if (threadIdx.x == 0) issue((p + 1) & 1);
            issued = true;
        }
        reduce_partials_multi(part, nb, h, red);
        int stop_t = -1;
        for (int t = 0; t < h; ++t) {
            const int k = k0 + t;
            if (k == 0) continue;  // res(x_0) is known to the host
            S2 = red[t];
            res = sqrt(S2) / a.baseline;
            if (blockIdx.x == 0 && threadIdx.x == 0) a.hist[k] = res;
            if (!isfinite(res)) { status = kStatusDiverged; stop_t = t; break; }
            if (res <= a.tol) { status = kStatusConverged; stop_t = t; break; }
        }
        __syncthreads();  // red[] is reused below
        if (stop_t >= 0) {
            stopped = true;
            executed = k0 + stop_t;
            if (issued) {  // drain the speculative load
                drain();
                issued = false;
                __syncthreads();
            }
            if (stop_t == 0) {
                result = p & 1;
            } else {
                // rollback: x_{k0+stop_t} from the intact pass input
                pass(p & 1, buf[(p + 1) & 1], k0, stop_t, acc, false, false);
                grid_barrier();
                result = (p + 1) & 1;
            }
        }
    }
    if (!stopped) {
        // residual of the cycle's final iterate (solver.py:233-234,248-249)
        const int u0 = (int)((long long)a.g.units * blockIdx.x / nb);
        const int u1 = (int)((long long)a.g.units * (blockIdx.x + 1) / nb);
        double acc;
        if constexpr (TAIL_PASS) {
            double t[S];
#pragma unroll
            for (int q = 0; q < S; ++q) t[q] = 0.0;
            pass(result, nullptr, 0, 0, t, true, false);
            acc = t[0];
        } else {
            acc = walk_units<FAM, kResid>(a.g, buf[result], nullptr, a.b, 0.0, u0, u1);
        }
        double* part = a.partials + (size_t)(npasses & 1) * kTbMaxSub * nb;
        acc = block_allsum(acc, sh1);
        if (threadIdx.x == 0) part[blockIdx.x] = acc;
        grid_barrier();
        S2 = reduce_partials(part, nb, sh1);
        res = sqrt(S2) / a.baseline;
        if (blockIdx.x == 0 && threadIdx.x == 0) a.hist[a.M] = res;
        if (!isfinite(res)) status = kStatusDiverged;
        else if (res <= a.tol) status = kStatusConverged;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.out_i[0] = executed;
        a.out_i[1] = status;
        a.out_i[2] = result;
        a.out_d[0] = S2;
        a.out_d[1] = res;
    }
}

}  // namespace srj
