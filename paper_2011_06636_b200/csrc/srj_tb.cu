// Temporally blocked SRJ cycle for the 2D 5-point constant-coefficient
// stencil (BASELINE config 2): s consecutive sweeps, each with its own omega,
// per HBM/L2 round trip.
//
// Overlapped ("ghost-zone") tiling: a CTA owns a TX x TY output tile and loads
// the (TX+2S) x (TY+2S) region around it into shared memory once per pass.
// Sub-sweep t (0..h-1) updates the region shrunk by t+1 rings, ping-ponging
// between two shared buffers, so after h sub-sweeps the owned tile holds
// x_{k0+h} exactly -- every value is produced by the same per-point arithmetic
// as the one-sweep kernel (bit-identical iterates).  Points outside the grid
// stay 0 in both buffers, which is the Dirichlet ghost.
//
// Residuals: sub-sweep t accumulates (b - A x_{k0+t})^2 over OWNED points only,
// giving per-sweep partials identical in meaning to the one-sweep kernel.  After
// each pass a grid barrier lets every CTA reduce the s partial vectors in a fixed
// order and apply the reference's per-sweep stopping rule (solver.py:216-222,
// 235-239).  A stop inside the pass at sweep k0+j (j >= 1) is resolved by
// re-running that pass with j sub-sweeps from its intact input buffer
// (rollback); a stop at j = 0 returns the input buffer itself.
#include <cooperative_groups.h>

#include <algorithm>

#include "srj_stencil.cuh"
#include "srj_tb.cuh"
#include "srj_walk.cuh"

namespace srj {
namespace tb2d {
constexpr int TX = 64, TY = 64, SMAX = kTbMaxSub;
constexpr int RX = TX + 2 * SMAX, RY = TY + 2 * SMAX;  // 80 x 80 region
constexpr int THREADS = 640;
constexpr int G = THREADS / RX;          // row groups
constexpr int ROWS = (RY + G - 1) / G;   // region rows per thread
static_assert(THREADS % RX == 0, "thread rows must tile the region width");
constexpr size_t SMEM = 2ull * RX * RY * sizeof(double);
}  // namespace tb2d

struct TbArgs {
    Geom g;
    double* buf0;
    double* buf1;
    const double* b;
    const double* omegas;
    int M, s;
    double tol, baseline;
    double* partials;  // [2][SMAX][gridDim.x]
    double* hist;
    int* out_i;
    double* out_d;
    int tiles_x, ntiles;
};

// One pass (h sub-sweeps) over every tile this CTA owns.
__device__ __forceinline__ void tb2d_pass(const TbArgs& a, const double* __restrict__ xin,
                                          double* __restrict__ xout, int k0, int h,
                                          double (&acc)[tb2d::SMAX], bool accumulate,
                                          double* xs0, double* xs1) {
    using namespace tb2d;
    const int tid = threadIdx.x;
    const int c = tid % RX, gq = tid / RX;
    const int nx = a.g.nx, ny = a.g.ny;
    const double coff = a.g.c_off, cdiag = a.g.c_diag, inv = a.g.inv_diag;
    for (int q = blockIdx.x; q < a.ntiles; q += gridDim.x) {
        const int ox = (q % a.tiles_x) * TX, oy = (q / a.tiles_x) * TY;
        const int gx = ox - SMAX + c;
        const bool colin = gx >= 0 && gx < nx;
        double breg[ROWS];
#pragma unroll
        for (int m = 0; m < ROWS; ++m) {
            const int r = gq + G * m;
            breg[m] = 0.0;
            if (r < RY) {
                const int gy = oy - SMAX + r;
                const bool in = colin && gy >= 0 && gy < ny;
                const long long k = (long long)gy * nx + gx;
                xs0[r * RX + c] = in ? xin[k] : 0.0;
                xs1[r * RX + c] = 0.0;
                if (in) breg[m] = __ldg(a.b + k);
            }
        }
        __syncthreads();
#pragma unroll
        for (int t = 0; t < SMAX; ++t) {
            if (t < h) {
                const double w = __ldg(a.omegas + k0 + t);
                const double* src = (t & 1) ? xs1 : xs0;
                double* dst = (t & 1) ? xs0 : xs1;
                const int lo = SMAX - h + t + 1;
                const int hix = SMAX + TX + h - t - 1, hiy = SMAX + TY + h - t - 1;
                if (c >= lo && c < hix && colin) {
                    const bool ocol = c >= SMAX && c < SMAX + TX;
#pragma unroll
                    for (int m = 0; m < ROWS; ++m) {
                        const int r = gq + G * m;
                        const int gy = oy - SMAX + r;
                        if (r >= lo && r < hiy && gy >= 0 && gy < ny) {
                            const double* s0 = src + r * RX + c;
                            const double xc = s0[0];
                            double y = DADD(0.0, DMUL(coff, s0[-RX]));
                            y = DADD(y, DMUL(coff, s0[-1]));
                            y = DADD(y, DMUL(cdiag, xc));
                            y = DADD(y, DMUL(coff, s0[1]));
                            y = DADD(y, DMUL(coff, s0[RX]));
                            const double rr = DSUB(breg[m], y);
                            dst[r * RX + c] = relax(xc, inv, rr, w);
                            if (accumulate && ocol && r >= SMAX && r < SMAX + TY)
                                acc[t] = fma(rr, rr, acc[t]);
                        }
                    }
                }
                __syncthreads();
            }
        }
        const double* fin = (h & 1) ? xs1 : xs0;
        if (c >= SMAX && c < SMAX + TX && colin) {
#pragma unroll
            for (int m = 0; m < ROWS; ++m) {
                const int r = gq + G * m;
                const int gy = oy - SMAX + r;
                if (r >= SMAX && r < SMAX + TY && gy < ny)
                    xout[(long long)gy * nx + gx] = fin[r * RX + c];
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(tb2d::THREADS, 1) k_tb2d_cycle(TbArgs a) {
    using namespace tb2d;
    extern __shared__ double smem[];
    __shared__ double sh[32];
    double* xs0 = smem;
    double* xs1 = smem + RX * RY;
    const int nb = gridDim.x;
    double* const buf[2] = {a.buf0, a.buf1};
    const int npasses = (a.M + a.s - 1) / a.s;
    int executed = a.M, status = kStatusRan, result = npasses & 1;
    double S = 0.0, res = 0.0;
    bool stopped = false;
    for (int p = 0; p < npasses && !stopped; ++p) {
        const int k0 = p * a.s;
        const int h = min(a.s, a.M - k0);
        const double* xin = buf[p & 1];
        double* xout = buf[(p + 1) & 1];
        double acc[SMAX];
#pragma unroll
        for (int t = 0; t < SMAX; ++t) acc[t] = 0.0;
        tb2d_pass(a, xin, xout, k0, h, acc, true, xs0, xs1);
        double* part = a.partials + (size_t)(p & 1) * SMAX * nb;
#pragma unroll
        for (int t = 0; t < SMAX; ++t) {
            if (t < h) {
                const double v = block_allsum(acc[t], sh);
                if (threadIdx.x == 0) part[t * nb + blockIdx.x] = v;
            }
        }
        grid_barrier();
        int stop_t = -1;
        for (int t = 0; t < h; ++t) {
            const int k = k0 + t;
            if (k == 0) continue;  // res(x_0) is known to the host
            S = reduce_partials(part + t * nb, nb, sh);
            res = sqrt(S) / a.baseline;
            if (blockIdx.x == 0 && threadIdx.x == 0) a.hist[k] = res;
            if (!isfinite(res)) { status = kStatusDiverged; stop_t = t; break; }
            if (res <= a.tol) { status = kStatusConverged; stop_t = t; break; }
        }
        if (stop_t >= 0) {
            stopped = true;
            executed = k0 + stop_t;
            if (stop_t == 0) {
                result = p & 1;
            } else {
                // rollback: x_{k0+stop_t} from the intact pass input
                tb2d_pass(a, xin, xout, k0, stop_t, acc, false, xs0, xs1);
                grid_barrier();
                result = (p + 1) & 1;
            }
        }
    }
    if (!stopped) {
        // residual of the cycle's final iterate (solver.py:233-234,248-249)
        const int u0 = (int)((long long)a.g.units * blockIdx.x / nb);
        const int u1 = (int)((long long)a.g.units * (blockIdx.x + 1) / nb);
        double acc = walk_units<F2D, kResid>(a.g, buf[result], nullptr, a.b, 0.0, u0, u1);
        double* part = a.partials + (size_t)(npasses & 1) * SMAX * nb;
        acc = block_allsum(acc, sh);
        if (threadIdx.x == 0) part[blockIdx.x] = acc;
        grid_barrier();
        S = reduce_partials(part, nb, sh);
        res = sqrt(S) / a.baseline;
        if (blockIdx.x == 0 && threadIdx.x == 0) a.hist[a.M] = res;
        if (!isfinite(res)) status = kStatusDiverged;
        else if (res <= a.tol) status = kStatusConverged;
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.out_i[0] = executed;
        a.out_i[1] = status;
        a.out_i[2] = result;
        a.out_d[0] = S;
        a.out_d[1] = res;
    }
}

cudaError_t tb_plan_init(TbPlan& plan, const Geom& g, int num_sms) {
    plan = TbPlan();
    if (g.fam != F2D) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(k_tb2d_cycle, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)tb2d::SMEM);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tb2d_cycle, tb2d::THREADS,
                                                      tb2d::SMEM);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaSuccess;
    plan.tiles_x = (g.nx + tb2d::TX - 1) / tb2d::TX;
    plan.ntiles = plan.tiles_x * ((g.ny + tb2d::TY - 1) / tb2d::TY);
    plan.blocks = std::max(1, std::min(num_sms * per_sm, plan.ntiles));
    plan.threads = tb2d::THREADS;
    plan.smem = tb2d::SMEM;
    plan.supported = true;
    return cudaSuccess;
}

cudaError_t tb_launch_cycle(const TbPlan& plan, const Geom& g, double* x, double* x_alt,
                            const double* b, const double* omegas, int M, int s, double tol,
                            double baseline, double* partials, double* hist, int* out_i,
                            double* out_d, cudaStream_t st) {
    TbArgs a;
    a.g = g;
    a.buf0 = x;
    a.buf1 = x_alt;
    a.b = b;
    a.omegas = omegas;
    a.M = M;
    a.s = std::max(1, std::min(s, kTbMaxSub));
    a.tol = tol;
    a.baseline = baseline;
    a.partials = partials;
    a.hist = hist;
    a.out_i = out_i;
    a.out_d = out_d;
    a.tiles_x = plan.tiles_x;
    a.ntiles = plan.ntiles;
    void* args[] = {&a};
    return cudaLaunchCooperativeKernel((const void*)k_tb2d_cycle, dim3(plan.blocks),
                                       dim3(plan.threads), args, plan.smem, st);
}

}  // namespace srj
