// libsrj.so: sm_100a SRJ sweep kernels and the C ABI declared in include/srj.h.
//
// Cycle execution model (one launch per cycle):
//   a persistent cooperative kernel holds one CTA per resident slot on every SM
//   and walks the M sweeps of the cycle itself.  Each sweep reads x_k (ping-pong
//   buffer), writes x_{k+1} and accumulates the squared residual r_k = b - A x_k
//   of its INPUT iterate; after a grid barrier every CTA reduces the per-CTA
//   partials in the same fixed order (bit-identical in all CTAs), so all CTAs
//   agree on res_k = sqrt(sum r_k^2)/baseline without another barrier and stop
//   together before sweep k when res_k <= tol or is non-finite -- the
//   reference's per-sweep stopping rule (solver.py:216-222,235-239).  Because the
//   residual of x_k is produced by the sweep that consumes x_k, x_k is still
//   intact in the input buffer when the cycle stops there.  After the last sweep
//   a residual-only pass gives res(x_M) (solver.py:233-234,248-249).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "../../include/srj.h"
#include "srj_common.cuh"
#include "srj_tbdriver.cuh"
#include "srj_stencil.cuh"
#include "srj_2d.cuh"
#include "srj_3d.cuh"
#include "srj_tb.cuh"
#include "srj_walk.cuh"

namespace cg = cooperative_groups;

namespace srj {

constexpr int kMaxSchemeLength = 10000;  // reference schemes.py:24
constexpr int kTbPassMax = 6;             // sweeps one srj_tb_pass fuses (S = 6 rings)
constexpr int kThreads = 256;       // standalone sweep / matvec kernels
constexpr int kCoopThreads = 512;   // persistent cycle kernel: 2 CTAs per SM
constexpr int kSmallThreads = 1024;
constexpr int kSlots = 2;           // srj_sweep_planes scratch slots
constexpr int kApplyBlocksPerSm = 16;  // grid cap of the non-persistent kernels
constexpr long long kSmallUnits = 256;   // <= 8192 points: one CTA, no grid barrier

struct CycleArgs {
    Geom g;
    const double* xa;      // x_0 (also receives x_2, x_4, ...)
    double* xb;            // receives x_1, x_3, ...
    const double* b;
    const double* omegas;  // application order
    int M;                 // sweeps allowed this cycle (0: residual only)
    double tol, baseline;
    double* partials;      // [2][gridDim.x]
    double* hist;          // [M+1] relative residual of x_k
    int* out_i;            // executed, status
    double* out_d;         // final sum of squares, res_after
    int diff;              // 1: solution-difference infinity norm (no baseline, no lag)
    SolveCtl ctl;          // device-resident solve (k_reg_cycle_1d<.., SOLVE>)
};

// Solution-difference norm cycle (reference solver.py:200-203,224-228,242-243):
// sweep k produces x_{k+1} and d_k = max|x_{k+1} - x_k| (a max: bit-identical
// to numpy in any order); the test before sweep k+1 uses d_k, so there is no
// lag and no residual tail.
template <int FAM>
__device__ __forceinline__ void cycle_diff(const CycleArgs& a, int u0, int u1, double* sh) {
    const int nb = gridDim.x;
    double* const buf[2] = {const_cast<double*>(a.xa), a.xb};
    int executed = a.M, status = kStatusRan;
    double res = 0.0;
    for (int k = 0; k < a.M; ++k) {
        double d = walk_units<FAM, kSweepDiff>(a.g, buf[k & 1], buf[(k + 1) & 1], a.b,
                                               a.omegas[k], u0, u1);
        double* part = a.partials + (k & 1) * nb;
        d = block_allmax(d, sh);
        if (threadIdx.x == 0) part[blockIdx.x] = d;
        grid_barrier();
        double m = 0.0;
        for (int q = threadIdx.x; q < nb; q += blockDim.x) m = nanmax(m, __ldcg(part + q));
        res = block_allmax(m, sh);
        if (blockIdx.x == 0 && threadIdx.x == 0) a.hist[k + 1] = res;
        if (!isfinite(res)) { executed = k + 1; status = kStatusDiverged; break; }
        if (res <= a.tol) { executed = k + 1; status = kStatusConverged; break; }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.out_i[0] = executed;
        a.out_i[1] = status;
        a.out_i[2] = executed & 1;
        a.out_d[0] = res;
        a.out_d[1] = res;
    }
}

template <int FAM>
__global__ void __launch_bounds__(1024) k_cycle(CycleArgs a) {
    __shared__ double sh[32];
    const int nb = gridDim.x;
    const int u0 = (int)((long long)a.g.units * blockIdx.x / nb);
    const int u1 = (int)((long long)a.g.units * (blockIdx.x + 1) / nb);
    if (a.diff) {
        cycle_diff<FAM>(a, u0, u1, sh);
        return;
    }
    double* const buf[2] = {const_cast<double*>(a.xa), a.xb};
    int executed = a.M, status = kStatusRan;
    double S = 0.0, res = 0.0;
    for (int k = 0; k <= a.M; ++k) {
        const bool tail = (k == a.M);
        const double* xin = buf[k & 1];
        double acc = tail ? walk_units<FAM, kResid>(a.g, xin, nullptr, a.b, 0.0, u0, u1)
                          : walk_units<FAM, kSweep>(a.g, xin, buf[(k + 1) & 1], a.b, a.omegas[k], u0, u1);
        double* part = a.partials + (k & 1) * nb;
        acc = block_allsum(acc, sh);
        if (threadIdx.x == 0) part[blockIdx.x] = acc;
        grid_barrier();
        if (k >= 1 || tail) {
            S = reduce_partials(part, nb, sh);
            res = sqrt(S) / a.baseline;
            if (k >= 1) {
                if (blockIdx.x == 0 && threadIdx.x == 0) a.hist[k] = res;
                if (!isfinite(res)) { executed = k; status = kStatusDiverged; break; }
                if (res <= a.tol) { executed = k; status = kStatusConverged; break; }
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.out_i[0] = executed;
        a.out_i[1] = status;
        a.out_i[2] = executed & 1;  // x_executed lives in buf[executed & 1]
        a.out_d[0] = S;
        a.out_d[1] = res;
    }
}

// Small 1D systems (BASELINE config 1, N = 1024): one CTA of 8 warps holds x
// (two ping-pong buffers with zero ghosts) and b in shared memory for the whole
// cycle.  Per sweep: every thread updates its points, warp butterfly sums of
// r^2 land in red[parity][warp], ONE __syncthreads, then every warp reduces
// the 8 warp partials with the same butterfly (identical bits everywhere, no
// second barrier).  The relative norm sqrt(S)/baseline is evaluated exactly
// only when S is within 1e-12 of the stop threshold (or huge); otherwise
// S > ((tol*baseline)(1+1e-12))^2 already proves res > tol.  hist[k] is
// filled with S during the loop and converted in parallel afterwards.  Same
// protocol and outputs as k_cycle.
constexpr int kSmall1dMaxN = 8192;
constexpr int kSmall1dThreads = 256;

__global__ void __launch_bounds__(kSmall1dThreads) k_small_cycle_1d(CycleArgs a) {
    extern __shared__ double sm[];
    __shared__ double red[2][32];
    const int n = a.g.nx;
    // buffer k (ping-pong) starts at offset base(k); ghosts at base-1 and base+n.
    // Offsets, not pointers, keep every access an LDS/STS.
    const int base0 = 1, base1 = n + 3, bso = 2 * (n + 2);
    const double c = a.g.c_off, d = a.g.c_diag, inv = a.g.inv_diag;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = blockDim.x >> 5;
    for (int i = threadIdx.x; i < n + 2; i += blockDim.x) {
        sm[i] = (i >= 1 && i <= n) ? a.xa[i - 1] : 0.0;
        sm[n + 2 + i] = 0.0;
    }
    for (int i = threadIdx.x; i < n; i += blockDim.x) sm[bso + i] = a.b[i];
    // S above `hi2` proves sqrt(S)/baseline > tol (1e-12 relative margin for the
    // two roundings); only S below it (or non-finite / huge) takes the exact path
    const double tb = a.tol * a.baseline;
    const double hi2 = a.tol > 0.0 ? DMUL(DMUL(tb, tb), 1.0 + 1e-12) : -1.0;
    __syncthreads();
    int executed = a.M, status = kStatusRan, last = 0;
    double S = 0.0;
    double w_next = a.M > 0 ? __ldg(a.omegas) : 0.0;  // loaded one sweep ahead
    for (int k = 0; k <= a.M; ++k) {
        const bool tail = (k == a.M);
        const int bi = (k & 1) ? base1 : base0;
        const int bo = (k & 1) ? base0 : base1;
        const double w = w_next;
        if (k + 1 < a.M) w_next = __ldg(a.omegas + k + 1);
        double acc = 0.0;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const double xl = sm[bi + i - 1], xc = sm[bi + i], xr = sm[bi + i + 1];
            double y = DADD(0.0, DMUL(c, xl));
            y = DADD(y, DMUL(d, xc));
            y = DADD(y, DMUL(c, xr));
            const double r = DSUB(sm[bso + i], y);
            if (!tail) sm[bo + i] = relax(xc, inv, r, w);
            acc = fma(r, r, acc);
        }
        acc = warp_allsum(acc);
        if (lane == 0) red[k & 1][wid] = acc;
        __syncthreads();
        S = warp_allsum(lane < nw ? red[k & 1][lane] : 0.0);
        if (k >= 1) {
            last = k;
            if (threadIdx.x == 0) a.hist[k] = S;  // converted below
            if (!(S > hi2 && S < 1e300)) {
                const double res = sqrt(S) / a.baseline;
                if (!isfinite(res)) { executed = k; status = kStatusDiverged; break; }
                if (res <= a.tol) { executed = k; status = kStatusConverged; break; }
            }
        }
    }
    // x_executed lives in buffer executed & 1; it goes to x (even) or x_alt
    // (odd).  executed == 0 leaves x untouched (it is the input).
    if (executed > 0) {
        const int src = (executed & 1) ? base1 : base0;
        double* dst = (executed & 1) ? a.xb : const_cast<double*>(a.xa);
        for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = sm[src + i];
    }
    __syncthreads();  // thread 0's hist stores are visible to the CTA
    for (int k = 1 + threadIdx.x; k <= last; k += blockDim.x) a.hist[k] = sqrt(a.hist[k]) / a.baseline;
    if (threadIdx.x == 0) {
        a.out_i[0] = executed;
        a.out_i[1] = status;
        a.out_i[2] = executed & 1;
        a.out_d[0] = S;
        a.out_d[1] = sqrt(S) / a.baseline;
    }
}

// Register-resident 1D cycle (n <= 32 * kReg1dWarps * 16): NW warps (4 up to
// n = 2048, else 8; reg1d_shape), lane l of warp w holds P consecutive points
// [(32w + l) P, +P) -- x, b and p = c*x in registers for the whole cycle.
// Neighbours inside a lane are registers, across lanes one shuffle each way,
// across warps the edge p of the neighbouring warps
// through shared memory (double-buffered by sweep parity), one __syncthreads
// per sweep.
//
// Batched stop test.  A sweep's only output besides x_{k+1} is the lane's
// partial sum of r_k^2; sweeps run in batches of K = 16 with the partials kept
// in registers, then one transposed warp butterfly reduces all K at once
// (16 shuffles instead of 5 per sweep) and warp 0 applies the reference's
// per-sweep stop test (solver.py:216-222, 235-239) to the K residuals in order.
// A stop at sweep kb+s of the batch restores the batch's input x_kb (a register
// snapshot) and replays s sweeps.  Iterates are bit-identical to the reference
// (the diagonal term is fma(p, -2, y): c_diag = -2 c_off exactly, see srj_tb.cu
// for the identity and the leading "0 +"), residual norms are summed in a
// fixed order.  FULL: n == 256 P (no held points past n).
constexpr int kReg1dWarps = 8;      // most warps (n <= 32 * 8 * 16 = 4096)
constexpr int kReg1dBatch = 32;     // sweeps per stop-test batch (16 for P = 16: registers)

// The register kernel applies c_diag*x as -2*p (exact: c_diag = -2 c_off).
// VAR keeps faces and 1/diag per point in registers as well: at most 8
// points per lane (n <= 2048; 16 per lane spill several KB).
static bool reg1d_ok(const Geom& g) {
    return (g.fam == F1D && g.nx <= 32 * kReg1dWarps * 16 && g.c_diag == -2.0 * g.c_off) ||
           (g.fam == F1DV && g.nx <= 32 * kReg1dWarps * 8);
}

// Warps of the register kernel for n points: 4 up to 2048 (one barrier among
// fewer warps is cheaper: C1 3.56 -> 3.40 ms), else 8; points per lane P.
static void reg1d_shape(int n, int& nw, int& per, bool var = false) {
    nw = n <= 32 * 4 * (var ? 8 : 16) ? 4 : 8;
    per = (n + 32 * nw - 1) / (32 * nw);
    per = per <= 2 ? 2 : per <= 4 ? 4 : per <= 8 ? 8 : 16;
}

//
// VAR (SRJ_STENCIL_1D3_VAR): per point the faces c_w, c_e, the diagonal
// d = c_w + c_e and 1/d (the reference's division) stay in registers; no
// product is shared between neighbours (each face multiplies two different
// x), so x itself crosses lanes and warps and
// y = ((0 + (-c_w) x_w) + d x) + (-c_e) x_e in the reference's order.
template <int NW, int P, bool FULL, bool SOLVE, bool VAR>
__global__ void __launch_bounds__(32 * NW) k_reg_cycle_1d(CycleArgs a) {
    constexpr int K = (P <= 8 && !(VAR && P == 8)) ? kReg1dBatch : 16;
    __shared__ double edge[2][2][NW + 2];  // [parity][first|last][warp + 1]
    __shared__ double red[K][NW + 1];
    __shared__ double stop_sum;
    __shared__ int stop_at, stop_status;
    const int n = a.g.nx;
    const double c = a.g.c_off, inv = a.g.inv_diag;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int i0 = (wid * 32 + lane) * P;
    double x[P], b[P], p_[P], xs[P];
    // the neighbours' view: p = c*x (shared products), or x itself (VAR)
    double (&p)[P] = VAR ? x : p_;
    // VAR: west faces, the lane's last east face and 1/diagonal per point
    double fw[P], iv[VAR ? P : 1], fel = 0.0;
    // the value a neighbour needs: p = c*x (shared product) or x itself (VAR)
    auto pv = [&](double xv) __attribute__((always_inline)) -> double {
        if constexpr (VAR) return xv;
        else return DMUL(c, xv);
    };
#pragma unroll
    for (int j = 0; j < P; ++j) {
        const bool in = FULL || i0 + j < n;
        x[j] = in ? a.xa[i0 + j] : 0.0;
        b[j] = in ? a.b[i0 + j] : 0.0;
        p[j] = pv(x[j]);
        if constexpr (VAR) {
            // faces 0..n exist: the point past the last one still carries the
            // last point's east (boundary) face
            fw[j] = (FULL || i0 + j <= n) ? __ldg(a.g.fx + i0 + j) : 0.0;
            if (j == P - 1) fel = (FULL || i0 + j + 1 <= n) ? __ldg(a.g.fx + i0 + j + 1) : 0.0;
        }
    }
    // east face of point j = west face of j+1; diag = c_w + c_e
    auto fe = [&](int j) __attribute__((always_inline)) -> double {
        return j == P - 1 ? fel : fw[j + 1];
    };
    if constexpr (VAR) {
#pragma unroll
        for (int j = 0; j < P; ++j) {
            const bool in = FULL || i0 + j < n;
            iv[j] = in ? __drcp_rn(DADD(fw[j], fe(j))) : 0.0;  // sparse.py:42-44 (1.0 / diag)
        }
    }
    const double pz = pv(0.0);  // ghost / past-n neighbour: c*0 or 0 (a no-op term)
    if (threadIdx.x < 2 * 2 * (NW + 2)) (&edge[0][0][0])[threadIdx.x] = pz;
    __syncthreads();
    if (lane == 0) edge[0][0][wid + 1] = p[0];
    if (lane == 31) edge[0][1][wid + 1] = p[P - 1];
    const double tb = a.tol * a.baseline;
    const double hi2 = a.tol > 0.0 ? DMUL(DMUL(tb, tb), 1.0 + 1e-12) : -1.0;
    __syncthreads();
    int par = 0;
    // One sweep: residual of the current x (returned as the lane's sum of r^2
    // over its points), and x <- x + w inv r unless `update` is false.
    auto sweep = [&](double w, bool update) __attribute__((always_inline)) -> double {
        // branch-free: every lane reads the two edge words (broadcast) and the
        // warp's end lanes select them
        const double el = edge[par][1][wid];      // last point of warp-1
        const double er = edge[par][0][wid + 2];  // first point of warp+1
        double pl = __shfl_up_sync(0xffffffffu, p[P - 1], 1);
        double pr = __shfl_down_sync(0xffffffffu, p[0], 1);
        pl = lane == 0 ? el : pl;
        pr = lane == 31 ? er : pr;
        double r[P], acc = 0.0;
#pragma unroll
        for (int j = 0; j < P; ++j) {
            double y;
            if constexpr (VAR) {
                y = DADD(0.0, DMUL(-fw[j], j == 0 ? pl : p[j - 1]));
                y = DADD(y, DMUL(DADD(fw[j], fe(j)), x[j]));
                y = DADD(y, DMUL(-fe(j), j == P - 1 ? pr : p[j + 1]));
            } else {
                y = __fma_rn(p[j], -2.0, j == 0 ? pl : p[j - 1]);
                y = DADD(y, j == P - 1 ? pr : p[j + 1]);
            }
            r[j] = DSUB(b[j], y);
            if (FULL || i0 + j < n) acc = fma(r[j], r[j], acc);
        }
        if (update) {
#pragma unroll
            for (int j = 0; j < P; ++j) {
                const double xn = relax(x[j], VAR ? iv[j] : inv, r[j], w);
                x[j] = (FULL || i0 + j < n) ? xn : 0.0;
                if constexpr (!VAR) p[j] = pv(x[j]);
            }
            // one predicated store (lanes 0 and 31), no divergent branch
            if (lane == 0 || lane == 31)
                edge[par ^ 1][lane == 31][wid + 1] = lane == 0 ? p[0] : p[P - 1];
            __syncthreads();
            par ^= 1;
        }
        return acc;
    };
    // One cycle of M sweeps with omegas[0..M): x (registers) ends as
    // x_executed; hist[k] = relative residual of x_k (k = 1..); returns
    // {executed, status} and the last residual's sum of squares in S.
    auto cycle = [&](const int M, const double* __restrict__ omegas, double* __restrict__ hist,
                     int& status, double& S) __attribute__((always_inline)) -> int {
        int executed = M;
        status = kStatusRan;
        S = 0.0;
        for (int kb = 0;; kb = min(kb + K, M)) {
            // sweeps kb .. kb+kk-1 (residual of x_k, then x_{k+1}); at kb == M the
            // residual of x_M alone (the cycle's tail)
            const bool tail = kb == M;
            const int kk = tail ? 1 : min(K, M - kb);
#pragma unroll
            for (int j = 0; j < P; ++j) xs[j] = x[j];
            double v[K], wv[K];  // the batch's omegas, loaded up front (off the sweep chain)
#pragma unroll
            for (int s = 0; s < K; ++s) wv[s] = (!tail && s < kk) ? __ldg(omegas + kb + s) : 0.0;
            if (kk == K) {  // a full batch: no per-sweep guard (uniform, branch-free)
#pragma unroll
                for (int s = 0; s < K; ++s) v[s] = sweep(wv[s], true);
            } else {
#pragma unroll
                for (int s = 0; s < K; ++s) {
                    v[s] = 0.0;
                    if (s < kk) v[s] = sweep(wv[s], !tail);
                }
            }
            // transposed butterfly: log2(K) halving rounds (lane bits 16, 8, ...),
            // then plain butterfly rounds over the remaining low lane bits; lane l
            // ends with the warp sum of sweep (l / (32/K)) (fixed order; the lanes
            // of a group agree)
            constexpr int G = 32 / K;  // lanes per sweep after the halving rounds
#pragma unroll
            for (int h = K / 2, o = 16; h >= 1; h >>= 1, o >>= 1) {
                const bool hi = (lane & o) != 0;
#pragma unroll
                for (int i = 0; i < h; ++i) {
                    const double send = hi ? v[i] : v[i + h];
                    const double keep = hi ? v[i + h] : v[i];
                    v[i] = DADD(keep, __shfl_xor_sync(0xffffffffu, send, o));
                }
            }
#pragma unroll
            for (int o = G / 2; o >= 1; o >>= 1) v[0] = DADD(v[0], __shfl_xor_sync(0xffffffffu, v[0], o));
            if ((lane & (G - 1)) == 0) red[lane / G][wid] = v[0];
            __syncthreads();
            if (wid == 0) {
                // lane s: the residual of x_{kb+s}, warp partials in warp order
                double Ss = 0.0;
                bool stop = false;
                int st = kStatusRan;
                if (lane < kk) {
                    Ss = red[lane][0];
#pragma unroll
                    for (int q = 1; q < NW; ++q) Ss = DADD(Ss, red[lane][q]);
                    const int k = kb + lane;
                    if (k >= 1) {
                        const double res = sqrt(Ss) / a.baseline;
                        hist[k] = res;
                        if (!(Ss > hi2 && Ss < 1e300)) {
                            if (!isfinite(res)) { stop = true; st = kStatusDiverged; }
                            else if (res <= a.tol) { stop = true; st = kStatusConverged; }
                        }
                    }
                }
                const unsigned m = __ballot_sync(0xffffffffu, stop);
                const int first = m ? __ffs(m) - 1 : (tail ? 0 : -1);
                if (first >= 0 && lane == first) {
                    stop_at = first;
                    stop_status = st;
                    stop_sum = Ss;
                } else if (first < 0 && lane == kk - 1) {
                    stop_at = -1;
                    stop_sum = Ss;
                }
            }
            __syncthreads();
            const int s_stop = stop_at;
            S = stop_sum;
            if (s_stop >= 0) {
                if (!tail) {
                    executed = kb + s_stop;
                    // x_{kb+s}: replay s sweeps from the batch's input
#pragma unroll
                    for (int j = 0; j < P; ++j) {
                        x[j] = xs[j];
                        if constexpr (!VAR) p[j] = pv(x[j]);
                    }
                    if (lane == 0) edge[par][0][wid + 1] = p[0];
                    if (lane == 31) edge[par][1][wid + 1] = p[P - 1];
                    __syncthreads();
#pragma unroll
                    for (int s = 0; s < K; ++s)
                        if (s < s_stop) sweep(wv[s], true);
                }
                status = stop_status;
                __syncthreads();  // stop_* are rewritten by the next batch / cycle
                return executed;
            }
            __syncthreads();  // stop_at / stop_sum are rewritten by the next batch
        }
    };
    if constexpr (!SOLVE) {
        int status;
        double S;
        const int executed = cycle(a.M, a.omegas, a.hist, status, S);
        if (executed > 0) {
            double* dst = (executed & 1) ? a.xb : const_cast<double*>(a.xa);
#pragma unroll
            for (int j = 0; j < P; ++j)
                if (FULL || i0 + j < n) dst[i0 + j] = x[j];
        }
        if (threadIdx.x == 0) {
            a.out_i[0] = executed;
            a.out_i[1] = status;
            a.out_i[2] = executed & 1;
            a.out_d[0] = S;
            a.out_d[1] = sqrt(S) / a.baseline;
        }
    } else {
        // Device-resident solve (srj_tbdriver.cuh tb_run_solve, same decisions):
        // every thread runs the controller on identical values; x stays in
        // registers across cycles and ends in xa.
        const SolveCtl& cs = a.ctl;
        int level = cs.level0, stop = kSolvePaused, cyc = 0;
        long long total = 0;
        double res_before = cs.res0, prev = cs.prev_ratio0;
        for (; cyc < cs.max_cycles; ++cyc) {
            const int off = cs.level_off[level];
            const int Mfull = cs.level_off[level + 1] - off;
            if (res_before <= a.tol) {  // solver.py:217-222, checked on the known residual
                if (threadIdx.x == 0)
                    cs.recs[cyc] = SolveRec{level, Mfull, 0, kStatusConverged, res_before, res_before};
                stop = kSolveConverged;
                ++cyc;
                break;
            }
            const int Meff = (int)min((long long)Mfull, max(cs.budget - total, 0ll));
            if (Meff == 0) {
                if (threadIdx.x == 0)
                    cs.recs[cyc] = SolveRec{level, Mfull, 0, kStatusRan, res_before, res_before};
                stop = kSolveBudget;
                ++cyc;
                break;
            }
            if (total + Meff > cs.hist_cap) break;  // history buffer full: pause
            int status;
            double S;
            const int executed = cycle(Meff, cs.omegas_all + off, a.hist + total, status, S);
            const double ra = executed > 0 ? sqrt(S) / a.baseline : res_before;
            if (threadIdx.x == 0)
                cs.recs[cyc] = SolveRec{level, Mfull, executed, status, res_before, ra};
            total += executed;
            if (status == kStatusDiverged) { stop = kSolveDiverged; ++cyc; break; }
            if (ra <= a.tol) { stop = kSolveConverged; res_before = ra; ++cyc; break; }
            if (total >= cs.budget) { stop = kSolveBudget; res_before = ra; ++cyc; break; }
            if (executed > 0 && res_before > 0.0 && ra > 0.0) prev = ra / res_before;
            if (cs.mode == kSolveHeuristic) {
                if (isfinite(prev)) level = heuristic_level(prev, level, cs.t_hi, cs.t_lo, cs.n_levels - 1);
            } else if (cs.mode == kSolveIncreasing) {
                level = min(level + 1, cs.n_levels - 1);
            }
            res_before = ra;
        }
#pragma unroll
        for (int j = 0; j < P; ++j)
            if (FULL || i0 + j < n) const_cast<double*>(a.xa)[i0 + j] = x[j];
        if (threadIdx.x == 0) {
            a.out_i[0] = cyc;
            a.out_i[1] = stop;
            a.out_i[2] = 0;
            a.out_i[3] = level;
            a.out_d[0] = res_before;
            a.out_d[1] = prev;
            a.out_d[2] = (double)total;
        }
    }
}

template <bool SOLVE, bool VAR>
static void reg1d_launch_v(int nw, int per, bool full, const CycleArgs& a, cudaStream_t st) {
#define SRJ_REG1D(NWW, PP)                                                               \
    if (full) k_reg_cycle_1d<NWW, PP, true, SOLVE, VAR><<<1, 32 * NWW, 0, st>>>(a);     \
    else k_reg_cycle_1d<NWW, PP, false, SOLVE, VAR><<<1, 32 * NWW, 0, st>>>(a)
    if (nw == 4) {
        if (per == 2) { SRJ_REG1D(4, 2); }
        else if (per == 4) { SRJ_REG1D(4, 4); }
        else if (per == 8) { SRJ_REG1D(4, 8); }
        else if constexpr (!VAR) { SRJ_REG1D(4, 16); }
    } else {
        if constexpr (VAR) { SRJ_REG1D(8, 8); }
        else { SRJ_REG1D(8, 16); }
    }
#undef SRJ_REG1D
}

template <bool SOLVE>
static void reg1d_launch(int nw, int per, bool full, const CycleArgs& a, cudaStream_t st) {
    if (a.g.fam == F1DV) reg1d_launch_v<SOLVE, true>(nw, per, full, a, st);
    else reg1d_launch_v<SOLVE, false>(nw, per, full, a, st);
}

template <int FAM, int MODE>
__global__ void __launch_bounds__(kThreads) k_apply(Geom g, const double* x, double* out,
                                                    const double* __restrict__ b, double w) {
    const int nb = gridDim.x;
    const int u0 = (int)((long long)g.units * blockIdx.x / nb);
    const int u1 = (int)((long long)g.units * (blockIdx.x + 1) / nb);
    walk_units<FAM, MODE>(g, x, out, b, w, u0, u1);
}

// One sweep / residual over units [ub, ue) (whole x-rows of a plane range)
// with the grid's sum of r^2 reduced into *result.
template <int FAM, int MODE>
__global__ void __launch_bounds__(kThreads) k_apply_range(Geom g, const double* x, double* out,
                                                          const double* __restrict__ b, double w,
                                                          int ub, int ue, double* block_part,
                                                          unsigned* counter, double* result) {
    __shared__ double sh[32];
    const int nb = gridDim.x;
    const int u0 = ub + (int)((long long)(ue - ub) * blockIdx.x / nb);
    const int u1 = ub + (int)((long long)(ue - ub) * (blockIdx.x + 1) / nb);
    const double acc = walk_units<FAM, MODE>(g, x, out, b, w, u0, u1);
    last_block_sum(acc, block_part, counter, result, sh);
}

// SplitMix64 counter form: draw i of a stream seeded with s is
// mix(s + (i+1)*GAMMA) (reference rng.py:25-40), f = 2u - 1.
__global__ void k_fill_rhs(double* out, long long n, unsigned long long seed, long long start) {
    const long long stride = (long long)gridDim.x * blockDim.x;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
        unsigned long long z = seed + (unsigned long long)(start + i + 1) * 0x9E3779B97F4A7C15ull;
        z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
        z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
        z ^= z >> 31;
        const double u = (double)(z >> 11) * 0x1.0p-53;
        out[i] = DSUB(DMUL(2.0, u), 1.0);
    }
}

}  // namespace srj

using namespace srj;

// ----------------------------------------------------------------------------
// Host side
// ----------------------------------------------------------------------------

static thread_local std::string g_last_error;

static int fail(int code, const std::string& msg) {
    g_last_error = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                   \
    do {                                                                                 \
        cudaError_t _e = (expr);                                                         \
        if (_e != cudaSuccess)                                                           \
            return fail(SRJ_CUDA_ERROR, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur = -1;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev) cudaSetDevice(prev);
    }
};

struct srj_op {
    srj_op_desc desc;
    Geom g;
    int device = 0;
    int num_sms = 0;
    int coop_blocks = 0;     // cooperative grid of the cycle kernel
    int coop_threads = 0;
    int sweeps_per_pass = 1;
    double* partials = nullptr;  // device scratch
    double* hist = nullptr;      // device [kMaxSchemeLength + 2]
    int* out_i = nullptr;        // device [4]
    double* out_d = nullptr;     // device [4]
    int* h_out_i = nullptr;      // pinned mirrors
    double* h_out_d = nullptr;
    double* h_hist = nullptr;
    TbPlan tb;                   // temporal-blocking plan (srj_tb.cuh)
    Tb3Plan tb3;                 // 3D temporal-blocking plan (srj_tb3d.cu)
    TbvPlan tbv;                 // var-coef 2D temporal-blocking plan (srj_tbvar.cu)
    Plan3D p3;                   // plane-streaming 3D plan (srj_3d.cuh)
    Plan3V p3v;                  // plane-streaming 3D variable-coefficient plan (srj_3dv.cu)
    Tb3vPlan tb3v;               // 3D variable-coefficient temporal blocking (srj_tb3v.cu)
    Plan2D p2;                   // tile-streaming 2D plan (srj_2d.cuh)
    // srj_sweep_planes scratch, one set per slot (concurrent launches)
    double* slot_part[kSlots] = {nullptr, nullptr};
    unsigned* slot_counter = nullptr;  // device [kSlots], zero between launches
    int slot_capacity = 0;             // doubles per slot_part
    // device-resident solve (srj_solve): per-cycle records and sweep history
    SolveRec* solve_recs = nullptr;
    int solve_recs_cap = 0;
    double* solve_hist = nullptr;
    long long solve_hist_cap = 0;
};

template <int FAM>
static const void* cycle_kernel() { return (const void*)&k_cycle<FAM>; }

static const void* cycle_kernel_for(int fam) {
    switch (fam) {
        case F1D: return cycle_kernel<F1D>();
        case F2D: return cycle_kernel<F2D>();
        case F3D: return cycle_kernel<F3D>();
        case FCSR: return cycle_kernel<FCSR>();
        case F3DV: return cycle_kernel<F3DV>();
        case F1DV: return cycle_kernel<F1DV>();
        default: return cycle_kernel<F2DV>();
    }
}

template <int MODE>
static int launch_apply(srj_op* op, const double* x, double* out, const double* b, double w,
                        cudaStream_t st) {
    const int blocks = (int)std::max<long long>(1, std::min<long long>((op->g.units + 7) / 8, 16ll * op->num_sms));
    switch (op->g.fam) {
        case F1D: k_apply<F1D, MODE><<<blocks, kThreads, 0, st>>>(op->g, x, out, b, w); break;
        case F2D: k_apply<F2D, MODE><<<blocks, kThreads, 0, st>>>(op->g, x, out, b, w); break;
        case F3D: k_apply<F3D, MODE><<<blocks, kThreads, 0, st>>>(op->g, x, out, b, w); break;
        case FCSR: k_apply<FCSR, MODE><<<blocks, kThreads, 0, st>>>(op->g, x, out, b, w); break;
        case F3DV: k_apply<F3DV, MODE><<<blocks, kThreads, 0, st>>>(op->g, x, out, b, w); break;
        case F1DV: k_apply<F1DV, MODE><<<blocks, kThreads, 0, st>>>(op->g, x, out, b, w); break;
        default: k_apply<F2DV, MODE><<<blocks, kThreads, 0, st>>>(op->g, x, out, b, w); break;
    }
    CUDA_TRY(cudaGetLastError());
    return SRJ_OK;
}

extern "C" {

int srj_abi_version(void) { return SRJ_ABI_VERSION; }

const char* srj_last_error(void) { return g_last_error.c_str(); }

int srj_op_create(const srj_op_desc* d, srj_op** out) {
    if (!d || !out) return fail(SRJ_BAD_ARGUMENT, "null argument");
    *out = nullptr;
    if (d->family < SRJ_STENCIL_1D3 || d->family > SRJ_STENCIL_1D3_VAR)
        return fail(SRJ_BAD_ARGUMENT, "unknown stencil family");
    if (d->nx < 1 || d->ny < 1 || d->nz < 1)
        return fail(SRJ_BAD_ARGUMENT, "extents must be positive");
    const bool var = d->family == SRJ_STENCIL_2D5_VAR || d->family == SRJ_STENCIL_3D7_VAR ||
                     d->family == SRJ_STENCIL_1D3_VAR;
    const bool csr = d->family == SRJ_CSR;
    const bool is1d = d->family == SRJ_STENCIL_1D3 || d->family == SRJ_STENCIL_1D3_VAR;
    const bool is3d = d->family == SRJ_STENCIL_3D7 || d->family == SRJ_STENCIL_3D7_VAR;
    if (var && (!d->face_x || (!is1d && !d->face_y) || (is3d && !d->face_z)))
        return fail(SRJ_BAD_ARGUMENT,
                    "variable-coefficient operator needs face_x (and face_y in 2D/3D, face_z in 3D)");
    if (csr && (!d->row_ptr || !d->col_idx || !d->values || !d->inv_diag || d->ny != 1 ||
                d->nz != 1 || d->nnz < 1))
        return fail(SRJ_BAD_ARGUMENT, "CSR operator needs row_ptr, col_idx, values, inv_diag, nnz and ny == nz == 1");
    if (!var && !csr && !(d->dx2 > 0.0))
        return fail(SRJ_BAD_ARGUMENT, "dx2 must be positive");
    if (is1d && (d->ny != 1 || d->nz != 1))
        return fail(SRJ_BAD_ARGUMENT, "1D operator needs ny == nz == 1");
    if ((d->family == SRJ_STENCIL_2D5 || d->family == SRJ_STENCIL_2D5_VAR) && d->nz != 1)
        return fail(SRJ_BAD_ARGUMENT, "2D operator needs nz == 1");
    const long long rows = d->ny * d->nz;
    const long long upr = (d->nx + 31) / 32;
    if (d->nx >= (1ll << 31) || rows * upr >= (1ll << 31))
        return fail(SRJ_BAD_ARGUMENT, "grid too large for one operator (shard it into slabs)");

    DeviceGuard guard(d->device);
    srj_op* op = new srj_op();
    op->desc = *d;
    op->device = d->device;
    Geom& g = op->g;
    g.fam = d->family;
    g.nx = (int)d->nx;
    g.ny = (int)d->ny;
    g.nz = (int)d->nz;
    g.n = d->nx * d->ny * d->nz;
    g.plane = csr ? 0 : is1d ? 1 : (is3d ? d->nx * d->ny : d->nx);
    g.rows = (int)rows;
    g.upr = (int)upr;
    g.units = (int)(rows * upr);
    const double dim = is1d ? 1.0 : (is3d ? 3.0 : 2.0);
    g.c_off = -1.0 * d->dx2;                  // reference problems.py:59,170
    g.c_diag = (2.0 * dim) * d->dx2;          // 2*dx2, 4*dx2, 6*dx2 (problems.py:58,164)
    g.inv_diag = 1.0 / g.c_diag;              // sparse.py:44
    g.fx = d->face_x;
    g.fy = d->face_y;
    g.fz = is3d && var ? d->face_z : nullptr;
    g.rp = reinterpret_cast<const long long*>(d->row_ptr);
    g.ci = d->col_idx;
    g.cv = d->values;
    g.cinv = d->inv_diag;

    cudaDeviceProp prop;
    cudaError_t e = cudaGetDeviceProperties(&prop, d->device);
    if (e != cudaSuccess) { delete op; return fail(SRJ_CUDA_ERROR, cudaGetErrorString(e)); }
    op->num_sms = prop.multiProcessorCount;
    if (!prop.cooperativeLaunch) { delete op; return fail(SRJ_CUDA_ERROR, "device lacks cooperative launch"); }

    if (g.units <= kSmallUnits) {
        op->coop_blocks = 1;
        op->coop_threads = kSmallThreads;
    } else {
        int per_sm = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, cycle_kernel_for(g.fam), kCoopThreads, 0);
        if (e != cudaSuccess || per_sm < 1) { delete op; return fail(SRJ_CUDA_ERROR, "occupancy query failed"); }
        // Few, fat CTAs on mid-size grids (the per-sweep grid barrier and
        // partial reduction cost grows with the CTA count); full occupancy on
        // large, bandwidth-bound grids.
        const bool large = g.units >= (1 << 16);
        long long want = (long long)(large ? per_sm : std::min(per_sm, 2)) * op->num_sms;
        const long long cap = std::max<long long>(1, g.units / (4 * (kCoopThreads / 32)));
        op->coop_blocks = (int)std::min(want, cap);
        op->coop_threads = kCoopThreads;
    }
    const size_t nparts = 2 * (size_t)std::max(op->coop_blocks, 8 * op->num_sms) * kTbMaxSub;
    if ((e = cudaMalloc(&op->partials, nparts * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&op->hist, (kMaxSchemeLength + 2) * sizeof(double))) != cudaSuccess ||
        (e = cudaMalloc(&op->out_i, 4 * sizeof(int))) != cudaSuccess ||
        (e = cudaMalloc(&op->out_d, 4 * sizeof(double))) != cudaSuccess ||
        (e = cudaHostAlloc(&op->h_out_i, 4 * sizeof(int), cudaHostAllocDefault)) != cudaSuccess ||
        (e = cudaHostAlloc(&op->h_out_d, 4 * sizeof(double), cudaHostAllocDefault)) != cudaSuccess ||
        (e = cudaHostAlloc(&op->h_hist, (kMaxSchemeLength + 2) * sizeof(double), cudaHostAllocDefault)) != cudaSuccess) {
        srj_op_destroy(op);
        return fail(SRJ_CUDA_ERROR, std::string("allocation failed: ") + cudaGetErrorString(e));
    }
    if ((e = plan2d_init(op->p2, g, op->num_sms)) != cudaSuccess) {
        srj_op_destroy(op);
        return fail(SRJ_CUDA_ERROR, std::string("2D plan setup failed: ") + cudaGetErrorString(e));
    }
    if ((e = plan3d_init(op->p3, g, op->num_sms)) != cudaSuccess) {
        srj_op_destroy(op);
        return fail(SRJ_CUDA_ERROR, std::string("3D plan setup failed: ") + cudaGetErrorString(e));
    }
    if ((e = plan3v_init(op->p3v, g, op->num_sms)) != cudaSuccess) {
        srj_op_destroy(op);
        return fail(SRJ_CUDA_ERROR, std::string("3D var-coef plan setup failed: ") + cudaGetErrorString(e));
    }
    if (op->p3v.supported &&
        (e = tb3v_plan_init(op->tb3v, g, op->num_sms, op->p3v.fx_pad, op->p3v.fx_pitch)) != cudaSuccess) {
        srj_op_destroy(op);
        return fail(SRJ_CUDA_ERROR, std::string("3D var-coef TB setup failed: ") + cudaGetErrorString(e));
    }
    if ((e = tb_plan_init(op->tb, g, op->num_sms)) != cudaSuccess) {
        srj_op_destroy(op);
        return fail(SRJ_CUDA_ERROR, std::string("temporal-blocking setup failed: ") + cudaGetErrorString(e));
    }
    if (g.fam == F1D &&
        (e = cudaFuncSetAttribute(k_small_cycle_1d, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)((3 * kSmall1dMaxN + 4) * sizeof(double)))) != cudaSuccess) {
        srj_op_destroy(op);
        return fail(SRJ_CUDA_ERROR, std::string("small 1D kernel setup failed: ") + cudaGetErrorString(e));
    }
    if ((e = tbv_plan_init(op->tbv, g, op->num_sms)) != cudaSuccess) {
        srj_op_destroy(op);
        return fail(SRJ_CUDA_ERROR, std::string("var-coef temporal-blocking setup failed: ") + cudaGetErrorString(e));
    }
    if ((e = tb3_plan_init(op->tb3, g, op->num_sms)) != cudaSuccess) {
        srj_op_destroy(op);
        return fail(SRJ_CUDA_ERROR, std::string("3D temporal-blocking setup failed: ") + cudaGetErrorString(e));
    }
    // Default: 6 fused sweeps per pass where a 2D temporally blocked kernel
    // exists (the S=6 rings measured fastest on B200 for constant and variable
    // coefficients), 2 for the 3D temporally blocked kernel (512^3 sweep: 296 us
    // vs 603 for the HBM-bound plane ring), else one per pass.
    op->sweeps_per_pass = (op->tb.supported || op->tbv.supported) ? 6
                          : (op->tb3.supported || op->tb3v.supported) ? 2
                                                                  : 1;
    op->slot_capacity = std::max(op->p3.slots, kApplyBlocksPerSm * op->num_sms);
    for (int s = 0; s < kSlots; ++s) {
        if ((e = cudaMalloc(&op->slot_part[s], op->slot_capacity * sizeof(double))) != cudaSuccess) {
            srj_op_destroy(op);
            return fail(SRJ_CUDA_ERROR, std::string("allocation failed: ") + cudaGetErrorString(e));
        }
    }
    if ((e = cudaMalloc(&op->slot_counter, kSlots * sizeof(unsigned))) != cudaSuccess ||
        (e = cudaMemset(op->slot_counter, 0, kSlots * sizeof(unsigned))) != cudaSuccess) {
        srj_op_destroy(op);
        return fail(SRJ_CUDA_ERROR, std::string("allocation failed: ") + cudaGetErrorString(e));
    }
    *out = op;
    return SRJ_OK;
}

int srj_op_destroy(srj_op* op) {
    if (!op) return SRJ_OK;
    DeviceGuard guard(op->device);
    cudaFree(op->partials);
    cudaFree(op->hist);
    cudaFree(op->out_i);
    cudaFree(op->out_d);
    cudaFreeHost(op->h_out_i);
    cudaFreeHost(op->h_out_d);
    cudaFreeHost(op->h_hist);
    for (int s = 0; s < kSlots; ++s) cudaFree(op->slot_part[s]);
    cudaFree(op->slot_counter);
    cudaFree(op->solve_recs);
    cudaFree(op->solve_hist);
    plan2d_free(op->p2);
    tbv_plan_free(op->tbv);
    tbs_plan_free(op->tb);
    plan3v_free(op->p3v);
    delete op;
    return SRJ_OK;
}

int srj_op_layout(const srj_op* op, int64_t* n, int64_t* halo) {
    if (!op) return fail(SRJ_BAD_ARGUMENT, "null operator");
    if (n) *n = op->g.n;
    if (halo) *halo = op->g.plane;
    return SRJ_OK;
}

int srj_op_diag(const srj_op* op, double* diag, double* inv_diag) {
    if (!op) return fail(SRJ_BAD_ARGUMENT, "null operator");
    if (op->g.fam == F2DV || op->g.fam == F3DV || op->g.fam == F1DV || op->g.fam == FCSR)
        return fail(SRJ_BAD_ARGUMENT, "this operator's diagonal is per point");
    if (diag) *diag = op->g.c_diag;
    if (inv_diag) *inv_diag = op->g.inv_diag;
    return SRJ_OK;
}

int srj_op_set_temporal_kernel(srj_op* op, int32_t kind) {
    if (!op) return fail(SRJ_BAD_ARGUMENT, "null operator");
    // The warp-streaming variant (round 1: 196 vs 555 GLUP/s) was removed; the
    // tile kernel is the only 2D temporally blocked kernel.
    if (kind != SRJ_TB_TILE)
        return fail(SRJ_BAD_ARGUMENT, "unknown temporal-blocking kernel (only SRJ_TB_TILE)");
    return SRJ_OK;
}

int srj_skew_plan(int64_t nx, int64_t ny, int32_t num_ctas, int32_t* tiles_per_cta,
                  int32_t* ctas_used, int32_t* tile_rows, int32_t* tile_cols, int32_t* sweeps,
                  int32_t* table, int64_t capacity) {
    if (nx < 1 || ny < 1 || nx >= (1ll << 30) || ny >= (1ll << 30) || num_ctas < 1 || num_ctas > 65536)
        return fail(SRJ_BAD_ARGUMENT, "skew plan: extents or CTA count out of range");
    int T = 0, used = 0;
    if (tbs_plan_table((int)nx, (int)ny, num_ctas, table, capacity, &T, &used) != 0)
        return fail(SRJ_BAD_ARGUMENT, "skew plan: table capacity too small");
    if (tiles_per_cta) *tiles_per_cta = T;
    if (ctas_used) *ctas_used = used;
    if (tile_rows) *tile_rows = tbs_tile_rows();
    if (tile_cols) *tile_cols = tbs_tile_cols();
    if (sweeps) *sweeps = tbs_sweeps();
    return SRJ_OK;
}

int srj_op_describe(const srj_op* op, srj_op_info* info) {
    if (!op || !info) return fail(SRJ_BAD_ARGUMENT, "null argument");
    info->num_sms = op->num_sms;
    info->cycle_blocks = op->coop_blocks;
    info->cycle_threads = op->coop_threads;
    info->sweeps_per_pass = op->sweeps_per_pass;
    info->tb_supported =
        (op->tb.supported || op->tb3.supported || op->tbv.supported || op->tb3v.supported) ? 1 : 0;
    const int tbk = tb_variant_for(op->tb, op->sweeps_per_pass);
    const bool skew = op->tb.supported && tb_uses_skew(op->tb, op->sweeps_per_pass);
    info->tb_blocks = op->tbv.supported    ? op->tbv.blocks
                      : op->tb3.supported  ? op->tb3.blocks
                      : op->tb3v.supported ? op->tb3v.blocks
                      : skew               ? op->tb.skew_blocks
                                           : op->tb.blocks[tbk];
    info->tb_occupancy =
        (op->tbv.supported || op->tb3.supported || op->tb3v.supported) ? 1 : op->tb.occupancy;
    info->tb_tiles = op->tbv.supported    ? op->tbv.ntiles
                     : op->tb3.supported  ? op->tb3.ntiles
                     : op->tb3v.supported ? op->tb3v.ntiles
                     : skew               ? op->tb.skew_blocks * op->tb.skew_tpc
                                          : op->tb.ntiles[tbk];
    info->cycle_kernel = (op->sweeps_per_pass > 1 && op->tbv.supported)  ? SRJ_KERNEL_TBVAR
                         : (op->sweeps_per_pass > 1 && op->tb3.supported) ? SRJ_KERNEL_TB3D
                         : (op->sweeps_per_pass > 1 && op->tb3v.supported) ? SRJ_KERNEL_TB3DV
                         : op->p3.supported                               ? SRJ_KERNEL_PLANE3D
                         : op->p3v.supported                              ? SRJ_KERNEL_PLANE3DV
                         : (op->sweeps_per_pass > 1 && skew)              ? SRJ_KERNEL_TBS2D
                         : (op->sweeps_per_pass > 1 && op->tb.supported) ? SRJ_KERNEL_TB2D
                         : op->p2.supported                               ? SRJ_KERNEL_TILE2D
                         : reg1d_ok(op->g) ? SRJ_KERNEL_REG1D
                         : (op->g.fam == F1D && op->g.nx <= kSmall1dMaxN) ? SRJ_KERNEL_SMALL1D
                                                                          : SRJ_KERNEL_GENERIC;
    return SRJ_OK;
}

int srj_op_set_sweeps_per_pass(srj_op* op, int32_t s) {
    if (!op) return fail(SRJ_BAD_ARGUMENT, "null operator");
    if (s < 1 || s > kTbMaxSub) return fail(SRJ_BAD_ARGUMENT, "sweeps per pass out of range");
    op->sweeps_per_pass = s;
    return SRJ_OK;
}

static int launch_cycle(srj_op* op, const double* xa, double* xb, const double* b,
                        const double* omegas, int M, double tol, double baseline,
                        cudaStream_t st, int diff = 0) {
    CycleArgs a;
    a.diff = diff;
    a.g = op->g;
    a.xa = xa;
    a.xb = xb;
    a.b = b;
    a.omegas = omegas;
    a.M = M;
    a.tol = tol;
    a.baseline = baseline;
    a.partials = op->partials;
    a.hist = op->hist;
    a.out_i = op->out_i;
    a.out_d = op->out_d;
    if (!diff && reg1d_ok(op->g)) {
        int nw, per;
        reg1d_shape(op->g.nx, nw, per, op->g.fam == F1DV);
        const bool full = op->g.nx == per * 32 * nw;
        reg1d_launch<false>(nw, per, full, a, st);
        CUDA_TRY(cudaGetLastError());
        return SRJ_OK;
    }
    if (!diff && op->g.fam == F1D && op->g.nx <= kSmall1dMaxN) {
        const size_t smem = (size_t)(3 * op->g.nx + 4) * sizeof(double);
        k_small_cycle_1d<<<1, kSmall1dThreads, smem, st>>>(a);
        CUDA_TRY(cudaGetLastError());
        return SRJ_OK;
    }
    void* args[] = {&a};
    CUDA_TRY(cudaLaunchCooperativeKernel(cycle_kernel_for(op->g.fam), dim3(op->coop_blocks),
                                         dim3(op->coop_threads), args, 0, st));
    return SRJ_OK;
}

int srj_residual_sq(srj_op* op, const double* x, const double* b, double* sumsq_host, void* stream) {
    if (!op || !x || !b || !sumsq_host) return fail(SRJ_BAD_ARGUMENT, "null argument");
    DeviceGuard guard(op->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (op->p3.supported) {
        CUDA_TRY(launch3d_cycle(op->p3, op->g, const_cast<double*>(x), nullptr, b, nullptr, 0, 0.0,
                                1.0, op->partials, op->hist, op->out_i, op->out_d, st));
    } else if (op->p3v.supported) {
        CUDA_TRY(launch3v_cycle(op->p3v, op->g, const_cast<double*>(x), nullptr, b, nullptr, 0, 0.0,
                                1.0, op->partials, op->hist, op->out_i, op->out_d, st));
    } else if (op->p2.supported) {
        CUDA_TRY(launch2d_cycle(op->p2, op->g, const_cast<double*>(x), nullptr, b, nullptr, 0, 0.0,
                                1.0, op->partials, op->hist, op->out_i, op->out_d, st));
    } else {
        int rc = launch_cycle(op, x, nullptr, b, nullptr, 0, 0.0, 1.0, st);
        if (rc) return rc;
    }
    CUDA_TRY(cudaMemcpyAsync(op->h_out_d, op->out_d, 2 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    *sumsq_host = op->h_out_d[0];
    return SRJ_OK;
}

int srj_run_cycle(srj_op* op, double* x, double* x_alt, const double* b,
                  const double* omegas_dev, int32_t M, double tol, double baseline,
                  double res_before, int64_t budget, double* history_host,
                  srj_cycle_out* out, void* stream) {
    if (!op || !x || !x_alt || !b || !out) return fail(SRJ_BAD_ARGUMENT, "null argument");
    if (M < 1 || M > kMaxSchemeLength) return fail(SRJ_BAD_ARGUMENT, "scheme length out of range");
    if (M > 0 && !omegas_dev) return fail(SRJ_BAD_ARGUMENT, "null omegas");
    if (!(baseline > 0.0)) return fail(SRJ_BAD_ARGUMENT, "baseline must be positive");
    DeviceGuard guard(op->device);
    cudaStream_t st = (cudaStream_t)stream;
    std::memset(out, 0, sizeof(*out));
    out->res_before = res_before;
    out->res_after = res_before;
    // Checks before sweep 0 are host-side: the incoming residual is known
    // (solver.py:217-222).
    if (res_before <= tol) {
        out->status = SRJ_CYCLE_CONVERGED;
        return SRJ_OK;
    }
    const int Meff = (int)std::min<int64_t>(M, std::max<int64_t>(budget, 0));
    if (Meff == 0) return SRJ_OK;

    if (op->sweeps_per_pass > 1 && op->tbv.supported) {
        CUDA_TRY(tbv_launch_cycle(op->tbv, op->g, x, x_alt, b, omegas_dev, Meff,
                                  op->sweeps_per_pass, tol, baseline, op->partials, op->hist,
                                  op->out_i, op->out_d, st, 0, op->g.ny, nullptr));
        out->launches = 1;
    } else if (op->sweeps_per_pass > 1 && op->tb3.supported) {
        CUDA_TRY(tb3_launch_cycle(op->tb3, op->g, x, x_alt, b, omegas_dev, Meff, tol, baseline,
                                  op->partials, op->hist, op->out_i, op->out_d, st, 0, op->g.nz,
                                  nullptr));
        out->launches = 1;
    } else if (op->sweeps_per_pass > 1 && op->tb3v.supported) {
        CUDA_TRY(tb3v_launch_cycle(op->tb3v, op->g, x, x_alt, b, omegas_dev, Meff, tol, baseline,
                                   op->partials, op->hist, op->out_i, op->out_d, st));
        out->launches = 1;
    } else if (op->p3v.supported) {
        CUDA_TRY(launch3v_cycle(op->p3v, op->g, x, x_alt, b, omegas_dev, Meff, tol, baseline,
                                op->partials, op->hist, op->out_i, op->out_d, st));
        out->launches = 1;
    } else if (op->p3.supported) {
        CUDA_TRY(launch3d_cycle(op->p3, op->g, x, x_alt, b, omegas_dev, Meff, tol, baseline,
                                op->partials, op->hist, op->out_i, op->out_d, st));
        out->launches = 1;
    } else if (op->sweeps_per_pass > 1 && op->tb.supported) {
        CUDA_TRY(tb_launch_cycle(op->tb, op->g, x, x_alt, b, omegas_dev, Meff,
                                 op->sweeps_per_pass, tol, baseline, op->partials, op->hist,
                                 op->out_i, op->out_d, st, 0, op->g.ny, nullptr));
        out->launches = 1;
    } else if (op->p2.supported) {
        CUDA_TRY(launch2d_cycle(op->p2, op->g, x, x_alt, b, omegas_dev, Meff, tol, baseline,
                                op->partials, op->hist, op->out_i, op->out_d, st));
        out->launches = 1;
    } else {
        const int rc = launch_cycle(op, x, x_alt, b, omegas_dev, Meff, tol, baseline, st);
        if (rc) return rc;
        out->launches = 1;
    }
    CUDA_TRY(cudaMemcpyAsync(op->h_out_i, op->out_i, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(op->h_out_d, op->out_d, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (history_host)
        CUDA_TRY(cudaMemcpyAsync(op->h_hist, op->hist, (Meff + 1) * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    const int executed = op->h_out_i[0];
    const int status = op->h_out_i[1];
    out->executed = executed;
    out->status = status;
    out->result_in_alt = op->h_out_i[2];
    out->res_after = op->h_out_d[1];
    if (history_host && executed > 0)
        std::memcpy(history_host, op->h_hist + 1, executed * sizeof(double));
    return SRJ_OK;
}

// Which cycle kernel a device-resident solve runs on (0: none): the
// temporally blocked kernels, whose cycles share one driver (srj_tbdriver.cuh),
// and the register-resident 1D kernel.
static int solve_kernel(const srj_op* op) {
    if (reg1d_ok(op->g)) return SRJ_KERNEL_REG1D;
    if (op->sweeps_per_pass <= 1) return 0;
    if (op->tbv.supported) return SRJ_KERNEL_TBVAR;
    if (op->tb3.supported) return SRJ_KERNEL_TB3D;
    if (op->tb3v.supported) return SRJ_KERNEL_TB3DV;
    if (op->tb.supported) return SRJ_KERNEL_TB2D;
    return 0;
}

int srj_op_set_reserved_sms(srj_op* op, int32_t k) {
    if (!op) return fail(SRJ_BAD_ARGUMENT, "null operator");
    if (k < 0 || k >= op->num_sms) return fail(SRJ_BAD_ARGUMENT, "reserved SMs out of range");
    op->tb.reserved = op->tbv.reserved = op->tb3.reserved = k;
    return SRJ_OK;
}

int srj_op_solve_supported(const srj_op* op) { return op && solve_kernel(op) != 0 ? 1 : 0; }

int srj_solve(srj_op* op, double* x, double* x_alt, const double* b, const srj_solve_args* args,
              double tol, double baseline, srj_solve_rec* recs_host, double* history_host,
              srj_solve_out* out, void* stream) {
    if (!op || !x || !x_alt || !b || !args || !recs_host || !out)
        return fail(SRJ_BAD_ARGUMENT, "null argument");
    const int kern = solve_kernel(op);
    if (!kern) return fail(SRJ_BAD_ARGUMENT, "no device-resident solve for this operator");
    if (!args->omegas_all || !args->level_off || args->n_levels < 1 || args->max_cycles < 1 ||
        args->level0 < 0 || args->level0 >= args->n_levels || args->mode < 0 || args->mode > 2)
        return fail(SRJ_BAD_ARGUMENT, "bad solve arguments");
    if (!(baseline > 0.0)) return fail(SRJ_BAD_ARGUMENT, "baseline must be positive");
    if (args->hist_cap < kMaxSchemeLength) return fail(SRJ_BAD_ARGUMENT, "history capacity too small");
    DeviceGuard guard(op->device);
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e;
    const int max_cycles = std::min(args->max_cycles, 4096);
    if (op->solve_recs_cap < max_cycles) {
        cudaFree(op->solve_recs);
        op->solve_recs = nullptr;
        op->solve_recs_cap = 0;
        if ((e = cudaMalloc(&op->solve_recs, max_cycles * sizeof(SolveRec))) != cudaSuccess)
            return fail(SRJ_CUDA_ERROR, std::string("allocation failed: ") + cudaGetErrorString(e));
        op->solve_recs_cap = max_cycles;
    }
    const long long hist_cap = std::min<long long>(args->hist_cap, 1ll << 22);
    if (op->solve_hist_cap < hist_cap) {
        cudaFree(op->solve_hist);
        op->solve_hist = nullptr;
        op->solve_hist_cap = 0;
        if ((e = cudaMalloc(&op->solve_hist, (hist_cap + 1) * sizeof(double))) != cudaSuccess)
            return fail(SRJ_CUDA_ERROR, std::string("allocation failed: ") + cudaGetErrorString(e));
        op->solve_hist_cap = hist_cap;
    }
    static_assert(sizeof(SolveRec) == sizeof(srj_solve_rec), "srj_solve_rec layout");
    SolveCtl c;
    c.omegas_all = args->omegas_all;
    c.level_off = args->level_off;
    c.n_levels = args->n_levels;
    c.mode = args->mode;
    c.level0 = args->level0;
    c.max_cycles = max_cycles;
    c.t_hi = args->t_hi;
    c.t_lo = args->t_lo;
    c.res0 = args->res0;
    c.prev_ratio0 = args->prev_ratio0;
    c.budget = args->budget;
    c.hist_cap = hist_cap;
    c.recs = op->solve_recs;
    const Geom& g = op->g;
    if (kern == SRJ_KERNEL_REG1D) {
        CycleArgs a = {};
        a.g = g;
        a.xa = x;
        a.xb = x_alt;
        a.b = b;
        a.tol = tol;
        a.baseline = baseline;
        a.hist = op->solve_hist;
        a.out_i = op->out_i;
        a.out_d = op->out_d;
        a.ctl = c;
        int nw, per;
        reg1d_shape(g.nx, nw, per, g.fam == F1DV);
        reg1d_launch<true>(nw, per, g.nx == per * 32 * nw, a, st);
        CUDA_TRY(cudaGetLastError());
    } else if (kern == SRJ_KERNEL_TBVAR)
        CUDA_TRY(tbv_launch_cycle(op->tbv, g, x, x_alt, b, nullptr, 0, op->sweeps_per_pass, tol,
                                  baseline, op->partials, op->solve_hist, op->out_i, op->out_d, st,
                                  0, g.ny, nullptr, &c));
    else if (kern == SRJ_KERNEL_TB3D)
        CUDA_TRY(tb3_launch_cycle(op->tb3, g, x, x_alt, b, nullptr, 0, tol, baseline, op->partials,
                                  op->solve_hist, op->out_i, op->out_d, st, 0, g.nz, nullptr, &c));
    else if (kern == SRJ_KERNEL_TB3DV)
        CUDA_TRY(tb3v_launch_cycle(op->tb3v, g, x, x_alt, b, nullptr, 0, tol, baseline,
                                   op->partials, op->solve_hist, op->out_i, op->out_d, st, &c));
    else
        CUDA_TRY(tb_launch_cycle(op->tb, g, x, x_alt, b, nullptr, 0, op->sweeps_per_pass, tol,
                                 baseline, op->partials, op->solve_hist, op->out_i, op->out_d, st,
                                 0, g.ny, nullptr, &c));
    CUDA_TRY(cudaMemcpyAsync(op->h_out_i, op->out_i, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(op->h_out_d, op->out_d, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    const int cycles = op->h_out_i[0];
    const long long sweeps = (long long)op->h_out_d[2];
    if (cycles > 0)
        CUDA_TRY(cudaMemcpy(recs_host, op->solve_recs, cycles * sizeof(SolveRec),
                            cudaMemcpyDeviceToHost));
    if (history_host && sweeps > 0)
        CUDA_TRY(cudaMemcpy(history_host, op->solve_hist + 1, sweeps * sizeof(double),
                            cudaMemcpyDeviceToHost));
    out->cycles = cycles;
    out->stop = op->h_out_i[1];
    out->result_in_alt = op->h_out_i[2];
    out->next_level = op->h_out_i[3];
    out->res_next = op->h_out_d[0];
    out->prev_ratio = op->h_out_d[1];
    out->sweeps = sweeps;
    return SRJ_OK;
}

int srj_run_cycle_diffinf(srj_op* op, double* x, double* x_alt, const double* b,
                          const double* omegas_dev, int32_t M, double tol, double res_before,
                          int64_t budget, double* history_host, srj_cycle_out* out,
                          void* stream) {
    if (!op || !x || !x_alt || !b || !out) return fail(SRJ_BAD_ARGUMENT, "null argument");
    if (M < 1 || M > kMaxSchemeLength) return fail(SRJ_BAD_ARGUMENT, "scheme length out of range");
    if (!omegas_dev) return fail(SRJ_BAD_ARGUMENT, "null omegas");
    DeviceGuard guard(op->device);
    cudaStream_t st = (cudaStream_t)stream;
    std::memset(out, 0, sizeof(*out));
    out->res_before = res_before;
    out->res_after = res_before;
    // the incoming difference norm, when known (a NaN means unknown), is tested
    // before the first sweep (solver.py:217-220)
    if (res_before == res_before && res_before <= tol) {
        out->status = SRJ_CYCLE_CONVERGED;
        return SRJ_OK;
    }
    const int Meff = (int)std::min<int64_t>(M, std::max<int64_t>(budget, 0));
    if (Meff == 0) return SRJ_OK;
    const int rc = launch_cycle(op, x, x_alt, b, omegas_dev, Meff, tol, 1.0, st, /*diff=*/1);
    if (rc) return rc;
    out->launches = 1;
    CUDA_TRY(cudaMemcpyAsync(op->h_out_i, op->out_i, 4 * sizeof(int), cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaMemcpyAsync(op->h_out_d, op->out_d, 4 * sizeof(double), cudaMemcpyDeviceToHost, st));
    if (history_host)
        CUDA_TRY(cudaMemcpyAsync(op->h_hist, op->hist, (Meff + 1) * sizeof(double),
                                 cudaMemcpyDeviceToHost, st));
    CUDA_TRY(cudaStreamSynchronize(st));
    out->executed = op->h_out_i[0];
    out->status = op->h_out_i[1];
    out->result_in_alt = op->h_out_i[2];
    out->res_after = op->h_out_d[1];
    if (history_host && out->executed > 0)
        std::memcpy(history_host, op->h_hist + 1, out->executed * sizeof(double));
    return SRJ_OK;
}

int srj_tb_pass(srj_op* op, double* x, double* x_alt, const double* b,
                const double* omegas_dev, int32_t h, int64_t row_lo, int64_t row_hi,
                double* sums_dev, void* stream) {
    if (!op || !x || !x_alt || !b || !omegas_dev || !sums_dev)
        return fail(SRJ_BAD_ARGUMENT, "null argument");
    if (!(op->tb.supported || op->tbv.supported || op->tb3.supported))
        return fail(SRJ_BAD_ARGUMENT, "no temporally blocked kernel for this operator");
    const bool is3d = op->tb3.supported;
    if (h < 1 || h > (is3d ? op->tb3.sweeps : kTbPassMax))
        return fail(SRJ_BAD_ARGUMENT, "sweeps per pass out of range");
    // a pass must not fuse more sweeps than the selected ring holds (the
    // SRJ_TB_VARIANT tuning override can pin the S = 4 ring)
    if (!is3d && !op->tbv.supported && h > tb_ring_for(op->tb, h))
        return fail(SRJ_BAD_ARGUMENT, "sweeps per pass exceed the selected ring width");
    if (row_lo < 0 || row_lo >= row_hi || row_hi > (is3d ? op->g.nz : op->g.ny))
        return fail(SRJ_BAD_ARGUMENT, "owned rows out of range");
    DeviceGuard guard(op->device);
    cudaStream_t st = (cudaStream_t)stream;
    if (is3d)
        CUDA_TRY(tb3_launch_cycle(op->tb3, op->g, x, x_alt, b, omegas_dev, h, -1.0, 1.0,
                                  op->partials, op->hist, op->out_i, op->out_d, st, (int)row_lo,
                                  (int)row_hi, sums_dev));
    else if (op->tbv.supported)
        CUDA_TRY(tbv_launch_cycle(op->tbv, op->g, x, x_alt, b, omegas_dev, h, h, -1.0, 1.0,
                                  op->partials, op->hist, op->out_i, op->out_d, st, (int)row_lo,
                                  (int)row_hi, sums_dev));
    else
        CUDA_TRY(tb_launch_cycle(op->tb, op->g, x, x_alt, b, omegas_dev, h, h, -1.0, 1.0,
                                 op->partials, op->hist, op->out_i, op->out_d, st, (int)row_lo,
                                 (int)row_hi, sums_dev));
    return SRJ_OK;
}

int srj_sweep(srj_op* op, const double* x, double* x_out, const double* b, double omega, void* stream) {
    if (!op || !x || !x_out || !b) return fail(SRJ_BAD_ARGUMENT, "null argument");
    DeviceGuard guard(op->device);
    return launch_apply<kSweep>(op, x, x_out, b, omega, (cudaStream_t)stream);
}

int srj_matvec(srj_op* op, const double* x, double* y, void* stream) {
    if (!op || !x || !y) return fail(SRJ_BAD_ARGUMENT, "null argument");
    DeviceGuard guard(op->device);
    return launch_apply<kMatvec>(op, x, y, nullptr, 0.0, (cudaStream_t)stream);
}

int64_t srj_op_planes(const srj_op* op) {
    if (!op) return -1;
    return (op->g.fam == F3D || op->g.fam == F3DV) ? op->g.nz
           : ((op->g.fam == F1D || op->g.fam == F1DV || op->g.fam == FCSR) ? 1 : op->g.ny);
}

int srj_sweep_planes(srj_op* op, const double* x, double* x_out, const double* b, double omega,
                     int64_t z_begin, int64_t z_end, double* partial_dev, int32_t slot,
                     void* stream) {
    if (!op || !x || !b || !partial_dev) return fail(SRJ_BAD_ARGUMENT, "null argument");
    if (slot < 0 || slot >= kSlots) return fail(SRJ_BAD_ARGUMENT, "slot out of range");
    const int64_t planes = srj_op_planes(op);
    if (z_begin < 0 || z_end > planes || z_begin >= z_end)
        return fail(SRJ_BAD_ARGUMENT, "plane range out of bounds");
    DeviceGuard guard(op->device);
    cudaStream_t st = (cudaStream_t)stream;
    const Geom& g = op->g;
    if (g.fam == F3D && op->p3.supported) {
        CUDA_TRY(launch3d_sweep(op->p3, g, x, x_out, b, omega, (int)z_begin, (int)z_end,
                                op->slot_part[slot], op->slot_counter + slot, partial_dev, st));
        return SRJ_OK;
    }
    if (op->p2.supported) {
        CUDA_TRY(launch2d_sweep(op->p2, g, x, x_out, b, omega, (int)z_begin, (int)z_end,
                                op->slot_part[slot], op->slot_counter + slot, partial_dev, st));
        return SRJ_OK;
    }
    const bool is1d = g.fam == F1D || g.fam == F1DV || g.fam == FCSR;
    const long long rows_per_plane = (g.fam == F3D || g.fam == F3DV) ? g.ny : 1;
    const long long per_plane = rows_per_plane * g.upr;
    const int ub = (int)(z_begin * (is1d ? g.units : per_plane));
    const int ue = (int)(z_end * (is1d ? g.units : per_plane));
    const int blocks = (int)std::max<long long>(
        1, std::min<long long>((ue - ub + 7) / 8, (long long)kApplyBlocksPerSm * op->num_sms));
    double* bp = op->slot_part[slot];
    unsigned* ct = op->slot_counter + slot;
#define SRJ_RANGE(FAM)                                                                          \
    if (x_out)                                                                                  \
        k_apply_range<FAM, kSweep><<<blocks, kThreads, 0, st>>>(g, x, x_out, b, omega, ub, ue,  \
                                                                bp, ct, partial_dev);           \
    else                                                                                        \
        k_apply_range<FAM, kResid><<<blocks, kThreads, 0, st>>>(g, x, nullptr, b, 0.0, ub, ue,  \
                                                                bp, ct, partial_dev);
    switch (g.fam) {
        case F1D: SRJ_RANGE(F1D) break;
        case F2D: SRJ_RANGE(F2D) break;
        case F3D: SRJ_RANGE(F3D) break;
        case FCSR: SRJ_RANGE(FCSR) break;
        case F3DV: SRJ_RANGE(F3DV) break;
        case F1DV: SRJ_RANGE(F1DV) break;
        default: SRJ_RANGE(F2DV) break;
    }
#undef SRJ_RANGE
    CUDA_TRY(cudaGetLastError());
    return SRJ_OK;
}

int srj_fill_uniform_rhs(double* out, int64_t n, uint64_t seed, int64_t start, int32_t device,
                         void* stream) {
    if (n < 0 || start < 0) return fail(SRJ_BAD_ARGUMENT, "negative size");
    if (n == 0) return SRJ_OK;
    if (!out) return fail(SRJ_BAD_ARGUMENT, "null output");
    DeviceGuard guard(device);
    const long long blocks = std::min<long long>((n + 255) / 256, 148ll * 16);
    k_fill_rhs<<<(int)blocks, 256, 0, (cudaStream_t)stream>>>(out, n, seed, start);
    CUDA_TRY(cudaGetLastError());
    return SRJ_OK;
}

}  // extern "C"
