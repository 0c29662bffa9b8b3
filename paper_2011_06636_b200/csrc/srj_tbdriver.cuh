// Per-cycle driver shared by the persistent temporally blocked kernels
// (srj_tb.cu: 2D constant coefficient, srj_tbvar.cu: 2D variable coefficient,
// srj_tb3d.cu: 3D).
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
//
// Device-resident solve (tb_run_solve): the same cycles back to back in one
// launch, the scheme level chosen on the device between cycles exactly as the
// host loop does (solver.py:305-326: heuristic_next_level on the last finite
// residual ratio, or the increasing / fixed controllers), one record per cycle
// for the host to rebuild the report.  Every CTA takes the same decisions: the
// values they are made from are reduced in the same fixed order everywhere.
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
    // Device-resident solve (the kernels' SOLVE instantiation only).
    SolveCtl ctl;
    // Skewed-tile kernel (srj_tbs.cu): CTA c runs tab[c*tpc .. c*tpc + tpc),
    // {ox, oy, lo, hi} per tile, until an entry with hi <= lo.
    const int4* tab = nullptr;
    int tpc = 0;
};

struct TbCycleResult {
    int executed, status, result;  // result: buffer index holding x_executed
    double S2, res;                // sum of squares / relative residual of x_executed
};

__device__ __forceinline__ int heuristic_level(double ratio, int level, double t_hi, double t_lo,
                                               int max_level) {
    // solver.py:125-140: raise above t_hi, lower strictly between, else keep
    if (ratio > t_hi)
        ++level;
    else if (t_lo < ratio && ratio < t_hi)
        --level;
    return min(max(level, 0), max_level);
}

// One cycle of M sweeps with omegas[0..M) from buffer `cur` (0: buf0, 1: buf1);
// hist[k] = relative residual of x_k, k = 1..executed.  `phase` numbers the
// partial-sum reductions (double-buffered across passes AND cycles).  The
// kernel's arguments stay untouched (no local copy of them); M, omegas and
// hist are references (kernel parameters, or the solve loop's shared state) so
// they need no registers across the passes.
// pass(in, xout, om, h, acc, accumulate, first_issued): one pass of h
//   sub-sweeps with om[0..h) over this CTA's tiles, reading buffer `in` and
//   writing xout; acc[t] += owned r^2 of sub-sweep t when accumulating; h = 0
//   with xout == nullptr (TAIL_PASS): acc[0] = owned r^2 of buffer `in`.
// issue(in): (thread 0) start the TMA of this CTA's first tile of buffer `in`.
// drain(): every thread waits for the outstanding TMA.
// SLAB: pass mode (the slab instantiation of a kernel; see TbArgs::sums).
template <int S, int FAM, bool SLAB, bool TAIL_PASS, class Pass, class Issue, class Drain>
__device__ __forceinline__ TbCycleResult tb_cycle(const TbArgs& a, const int& M,
                                                  const double* const& omegas,
                                                  double* const& hist, int cur, uint32_t& phase,
                                                  bool has_tiles, Pass&& pass, Issue&& issue,
                                                  Drain&& drain) {
    __shared__ double sh[32 * S];
    __shared__ double red[S];
    __shared__ double sh1[32];
    const int nb = gridDim.x;
    double* const buf[2] = {a.buf0, a.buf1};
    const int npasses = (M + a.s - 1) / a.s;
    TbCycleResult r{M, kStatusRan, (cur + npasses) & 1, 0.0, 0.0};
    bool stopped = false, issued = false;
    // fast stop test (see below): usable when sqrt(S2)/baseline cannot overflow
    const double tolb = a.tol * a.baseline;
    const double thr_hi = tolb * tolb * (1.0 + 1e-9);
    const bool fast_ok = a.baseline >= 1e-150 && !(thr_hi != thr_hi);
    int raw_to = 0;  // history entries 1 .. raw_to hold raw sums of squares
    for (int p = 0; p < npasses && !stopped; ++p) {
        const int k0 = p * a.s;
        const int h = min(a.s, M - k0);
        const int in = (cur + p) & 1;
        double acc[S];
#pragma unroll
        for (int t = 0; t < S; ++t) acc[t] = 0.0;
        pass(in, buf[in ^ 1], omegas + k0, h, acc, true, issued);
        issued = false;
        double* part = a.partials + (size_t)(phase++ & 1) * kTbMaxSub * nb;
        {
            // CTA sums of the h sub-sweeps: warp butterflies, then thread t < h
            // adds the warps' values in warp order (one block barrier)
            const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
            const int nw = (blockDim.x + 31) >> 5;
#pragma unroll
            for (int t = 0; t < S; ++t) {
                if (t < h) {
                    const double v = warp_allsum(acc[t]);
                    if (lane == 0) sh[wid * S + t] = v;
                }
            }
            __syncthreads();
            if (threadIdx.x < h) {
                double v = sh[threadIdx.x];
                for (int q = 1; q < nw; ++q) v += sh[q * S + threadIdx.x];
                part[threadIdx.x * nb + blockIdx.x] = v;
            }
        }
        grid_barrier();
        if constexpr (SLAB) {  // pass mode: raw sums, no decision, no tail
            reduce_partials_multi(part, nb, h, red);
            if (blockIdx.x == 0 && threadIdx.x < h) a.sums[threadIdx.x] = red[threadIdx.x];
            r.executed = h;
            r.result = in ^ 1;
            return r;
        }
        // Speculatively start the next pass's first tile while the stop test runs.
        if (p + 1 < npasses && has_tiles) {
            issue(in ^ 1);  // every thread calls; the kernel picks the issuing thread
            issued = true;
        }
        reduce_partials_multi(part, nb, h, red);
        // The reference's per-sweep checks (solver.py:216-222) for the h sub-sweeps at
        // once: lane t of every warp evaluates sub-sweep t; the first lane that stops
        // decides, as the sequential loop would.  Fast path: a sum of squares that is
        // finite and above (tol*baseline)^2 by a margin far beyond the rounding of
        // sqrt and the division cannot stop the cycle, so no sqrt / division sits on
        // the path to the next pass; the history keeps the raw sums until the end of
        // the cycle (hist_raw_to .. converted below).
        int stop_t = -1;
        {
            const int lane = threadIdx.x & 31;
            const bool live = lane < h && k0 + lane != 0;  // res(x_0) is known to the host
            const double S2l = live ? red[lane] : 0.0;
            const bool sure = !live || (fast_ok && S2l > thr_hi && S2l < 1e290);
            if (blockIdx.x == 0 && threadIdx.x < 32 && live) hist[k0 + lane] = S2l;  // raw
            if (live) raw_to = k0 + lane;  // (lane-dependent; the maximum is taken below)
            if (!__all_sync(0xffffffffu, sure)) {
                const double resl = sqrt(S2l) / a.baseline;
                const bool bad = live && !isfinite(resl);
                const bool conv = live && resl <= a.tol;
                const unsigned stops = __ballot_sync(0xffffffffu, bad || conv);
                if (stops) {
                    const int first = __ffs(stops) - 1;
                    stop_t = first;
                    r.S2 = __shfl_sync(0xffffffffu, S2l, first);
                    r.res = __shfl_sync(0xffffffffu, resl, first);
                    r.status = __shfl_sync(0xffffffffu, (int)bad, first) != 0 ? kStatusDiverged
                                                                               : kStatusConverged;
                }
            }
        }
        if (stop_t >= 0) {
            stopped = true;
            r.executed = k0 + stop_t;
            if (issued) {  // drain the speculative load
                drain();
                issued = false;
                __syncthreads();
            }
            if (stop_t == 0) {
                r.result = in;
            } else {
                // rollback: x_{k0+stop_t} from the intact pass input
                pass(in, buf[in ^ 1], omegas + k0, stop_t, acc, false, false);
                grid_barrier();
                r.result = in ^ 1;
            }
        }
    }
    if constexpr (!SLAB) {
        // history: raw sums -> relative residuals (CTA 0; its own stores, made
        // visible by the block barriers of the pass epilogue).  A stop at sub-sweep
        // t leaves entries beyond k0+t that the host never reads (k > executed).
        raw_to = __reduce_max_sync(0xffffffffu, raw_to);
        if (blockIdx.x == 0) {
            __syncthreads();
            for (int k = 1 + (int)threadIdx.x; k <= raw_to; k += blockDim.x)
                hist[k] = sqrt(hist[k]) / a.baseline;
        }
    }
    if (!stopped) {
        // residual of the cycle's final iterate (solver.py:233-234,248-249)
        double acc;
        if constexpr (TAIL_PASS) {
            double t[S];
#pragma unroll
            for (int q = 0; q < S; ++q) t[q] = 0.0;
            pass(r.result, nullptr, omegas, 0, t, true, false);
            acc = t[0];
        } else {
            const int u0 = (int)((long long)a.g.units * blockIdx.x / nb);
            const int u1 = (int)((long long)a.g.units * (blockIdx.x + 1) / nb);
            acc = walk_units<FAM, kResid>(a.g, buf[r.result], nullptr, a.b, 0.0, u0, u1);
        }
        double* part = a.partials + (size_t)(phase++ & 1) * kTbMaxSub * nb;
        acc = block_allsum(acc, sh1);
        if (threadIdx.x == 0) part[blockIdx.x] = acc;
        grid_barrier();
        r.S2 = reduce_partials(part, nb, sh1);
        r.res = sqrt(r.S2) / a.baseline;
        if (blockIdx.x == 0 && threadIdx.x == 0) hist[M] = r.res;
        if (!isfinite(r.res)) r.status = kStatusDiverged;
        else if (r.res <= a.tol) r.status = kStatusConverged;
    }
    return r;
}

// One cycle (srj_run_cycle protocol): out_i = {executed, status, result
// buffer}, out_d = {final sum of squares, res_after}.
template <int S, int FAM, bool SLAB, bool TAIL_PASS = false, class Pass, class Issue, class Drain>
__device__ __forceinline__ void tb_run_cycle(const TbArgs& a, bool has_tiles, Pass&& pass,
                                             Issue&& issue, Drain&& drain) {
    uint32_t phase = 0;
    const TbCycleResult r = tb_cycle<S, FAM, SLAB, TAIL_PASS>(a, a.M, a.omegas, a.hist, 0, phase,
                                                              has_tiles, pass, issue, drain);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.out_i[0] = r.executed;
        a.out_i[1] = r.status;
        a.out_i[2] = r.result;
        a.out_d[0] = r.S2;
        a.out_d[1] = r.res;
    }
}

// Device-resident solve: cycles back to back from buf0 (see SolveCtl).  The
// loop state lives in shared memory (thread 0 updates it between cycles), so
// it costs the register-bound pass code nothing.
struct TbSolveState {
    long long total;
    double res_before, prev;
    const double* omegas;
    double* hist;
    int level, cur, cyc, stop, M, halt;
};

template <int S, int FAM, bool TAIL_PASS = false, class Pass, class Issue, class Drain>
__device__ __forceinline__ void tb_run_solve(const TbArgs& a, bool has_tiles, Pass&& pass,
                                             Issue&& issue, Drain&& drain) {
    const SolveCtl& c = a.ctl;
    __shared__ TbSolveState ss;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    if (threadIdx.x == 0) {
        ss.total = 0;
        ss.res_before = c.res0;
        ss.prev = c.prev_ratio0;
        ss.level = c.level0;
        ss.cur = 0;
        ss.cyc = 0;
        ss.stop = kSolvePaused;
    }
    uint32_t phase = 0;
    for (;;) {
        // thread 0 sets up the next cycle (or ends the loop)
        if (threadIdx.x == 0) {
            ss.halt = 1;
            if (ss.cyc < c.max_cycles) {
                const int off = c.level_off[ss.level];
                const int M = c.level_off[ss.level + 1] - off;
                const int Meff = (int)min((long long)M, max(c.budget - ss.total, 0ll));
                const SolveRec rec{ss.level, M, 0, kStatusConverged, ss.res_before, ss.res_before};
                if (ss.res_before <= a.tol) {
                    // the checks before sweep 0 (solver.py:217-222): the incoming residual is known
                    if (lead) c.recs[ss.cyc] = rec;
                    ss.stop = kSolveConverged;
                    ++ss.cyc;
                } else if (Meff == 0) {
                    if (lead) c.recs[ss.cyc] = SolveRec{rec.level, M, 0, kStatusRan, rec.res_before,
                                                        rec.res_after};
                    ss.stop = kSolveBudget;
                    ++ss.cyc;
                } else if (ss.total + Meff <= c.hist_cap) {  // else: history full, pause
                    ss.M = Meff;
                    ss.omegas = c.omegas_all + off;
                    ss.hist = a.hist + ss.total;
                    ss.halt = 0;
                }
            }
        }
        __syncthreads();
        if (ss.halt) break;
        const int M = ss.M;
        const double* const om = ss.omegas;
        double* const hist = ss.hist;
        const TbCycleResult r = tb_cycle<S, FAM, false, TAIL_PASS>(a, M, om, hist, ss.cur, phase,
                                                                   has_tiles, pass, issue, drain);
        if (threadIdx.x == 0) {
            const double rb = ss.res_before;
            const double ra = r.executed > 0 ? r.res : rb;
            const int off = c.level_off[ss.level];
            if (lead)
                c.recs[ss.cyc] = SolveRec{ss.level, c.level_off[ss.level + 1] - off, r.executed,
                                          r.status, rb, ra};
            ++ss.cyc;
            ss.total += r.executed;
            ss.cur = r.result;
            ss.res_before = ra;
            if (r.status == kStatusDiverged) {
                ss.stop = kSolveDiverged;
            } else if (ra <= a.tol) {
                ss.stop = kSolveConverged;
            } else if (ss.total >= c.budget) {
                ss.stop = kSolveBudget;
            } else {
                // controller update (solver.py:294-299, 320-326)
                if (r.executed > 0 && rb > 0.0 && ra > 0.0) ss.prev = ra / rb;
                if (c.mode == kSolveHeuristic) {
                    if (isfinite(ss.prev))
                        ss.level = heuristic_level(ss.prev, ss.level, c.t_hi, c.t_lo, c.n_levels - 1);
                } else if (c.mode == kSolveIncreasing) {
                    ss.level = min(ss.level + 1, c.n_levels - 1);
                }
            }
        }
        __syncthreads();
        if (ss.stop != kSolvePaused) break;
    }
    if (lead) {
        a.out_i[0] = ss.cyc;
        a.out_i[1] = ss.stop;
        a.out_i[2] = ss.cur;
        a.out_i[3] = ss.level;
        a.out_d[0] = ss.res_before;
        a.out_d[1] = ss.prev;
        a.out_d[2] = (double)ss.total;
    }
}

}  // namespace srj
