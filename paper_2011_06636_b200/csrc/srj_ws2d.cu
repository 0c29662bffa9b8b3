// Warp-streaming temporal blocking for the 2D 5-point constant-coefficient
// stencil: S sweeps per pass with no shared memory and no block barriers.
//
// A warp owns a strip of 64 columns (two per lane, columns c0 = base+2l and
// c0+1) and a run of rows [r0, r1).  It streams x_{k0} rows r0-H .. r1+H-1
// from L2/HBM through H sub-sweep stages held in per-lane register rings.  The
// stages are SKEWED: at step tau, stage t produces x_{t+1} at row tau-1-2t from
// its ring (x_t rows tau-2-2t .. tau-2t), all of which were produced in earlier
// steps; stages run from last to first and each writes its new row into the
// next stage's oldest ring slot, already consumed this step.  So the H stages
// of a step are independent (2H fp64 dependency chains per lane) and the ring
// slot of every access is a compile-time index (steps unrolled by 3: no
// register moves).  West/east neighbours come from the adjacent lanes by warp
// shuffles; the strip's outer columns and the run's outer rows turn to garbage
// one ring per stage, so after H stages the inner 64-2S columns of rows
// [r0, r1) hold x_{k0+H} exactly -- each value from the reference's per-point
// arithmetic (bit-identical iterates).  Grid-exterior points are held at 0.
//
// Sub-sweep t accumulates (b - A x_{k0+t})^2 over the strip's owned points;
// per-pass grid barrier, fixed-order reduction and per-sweep stop test (with
// rollback) as the other cycle kernels.
#include <cooperative_groups.h>

#include <algorithm>

#include "srj_stencil.cuh"
#include "srj_walk.cuh"
#include "srj_ws2d.cuh"

namespace srj {

constexpr int kWsThreads = 128;
constexpr int kWsMaxS = 6;

struct WsArgs {
    Geom g;
    double* buf0;
    double* buf1;
    const double* b;
    const double* omegas;
    int M, s;
    double tol, baseline;
    double* partials;  // [2][kWsMaxS][gridDim.x]
    double* hist;
    int* out_i;
    double* out_d;
    int strips, rc, items;  // strips of 64-2S owned columns, rows per item
};

struct Pair {
    double a, b;
};

// Lane-constant data of one item.
struct WsLane {
    int c0;        // global column of the lane's first point
    bool in0, in1; // points inside the grid
    bool own;      // both points are owned columns of the strip (S even)
    bool vec;      // 16-byte aligned pair: one 128-bit access
};

__device__ __forceinline__ Pair ws_load(const double* row, const WsLane& L) {
    if (L.vec && L.in0 && L.in1) {
        const double2 v = *reinterpret_cast<const double2*>(row + L.c0);
        return Pair{v.x, v.y};
    }
    return Pair{L.in0 ? row[L.c0] : 0.0, L.in1 ? row[L.c0 + 1] : 0.0};
}

__device__ __forceinline__ Pair ws_ldg(const double* row, const WsLane& L) {
    if (L.vec && L.in0 && L.in1) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(row + L.c0));
        return Pair{v.x, v.y};
    }
    return Pair{L.in0 ? __ldg(row + L.c0) : 0.0, L.in1 ? __ldg(row + L.c0 + 1) : 0.0};
}

__device__ __forceinline__ Pair ws_row(const double* base, int row, int ny, int nx,
                                       const WsLane& L) {
    return (row >= 0 && row < ny) ? ws_load(base + (long long)row * nx, L) : Pair{0.0, 0.0};
}

// One skewed step at row tau, phase P = (tau - first) mod 3: every ring holds
// its (oldest, middle, newest) rows in slots (P, P+1, P+2) mod 3.
template <int S, int H, int P>
__device__ __forceinline__ void ws_step(const WsArgs& a, const double* __restrict__ xin,
                                        double* __restrict__ xout, int tau, int r0, int r1,
                                        const WsLane& L, const double (&w)[H],
                                        Pair (&ring)[H][3], Pair (&pre)[3], double (&acc)[S],
                                        bool accumulate) {
    constexpr int O = P % 3, C = (P + 1) % 3, N = (P + 2) % 3;
    const int nx = a.g.nx, ny = a.g.ny;
    const double coff = a.g.c_off, cdiag = a.g.c_diag, inv = a.g.inv_diag;
#pragma unroll
    for (int t = H - 1; t >= 0; --t) {
        const int row = tau - 1 - 2 * t;  // row of x_{t+1} produced now
        const Pair s = ring[t][O], cc = ring[t][C], n = ring[t][N];
        // west of point a: lane-1's b; east of point b: lane+1's a
        const double wa = __shfl_up_sync(0xffffffffu, cc.b, 1);
        const double eb = __shfl_down_sync(0xffffffffu, cc.a, 1);
        Pair out{0.0, 0.0};
        if (row >= 0 && row < ny) {
            const Pair bv = ws_ldg(a.b + (long long)row * nx, L);
            double y = DADD(0.0, DMUL(coff, s.a));
            y = DADD(y, DMUL(coff, wa));
            y = DADD(y, DMUL(cdiag, cc.a));
            y = DADD(y, DMUL(coff, cc.b));
            y = DADD(y, DMUL(coff, n.a));
            const double ra = DSUB(bv.a, y);
            double z = DADD(0.0, DMUL(coff, s.b));
            z = DADD(z, DMUL(coff, cc.a));
            z = DADD(z, DMUL(cdiag, cc.b));
            z = DADD(z, DMUL(coff, eb));
            z = DADD(z, DMUL(coff, n.b));
            const double rb = DSUB(bv.b, z);
            out.a = L.in0 ? relax(cc.a, inv, ra, w[t]) : 0.0;
            out.b = L.in1 ? relax(cc.b, inv, rb, w[t]) : 0.0;
            if (accumulate && L.own && row >= r0 && row < r1) {
                if (L.in0) acc[t] = fma(ra, ra, acc[t]);
                if (L.in1) acc[t] = fma(rb, rb, acc[t]);
            }
        }
        if (t + 1 < H) {
            ring[t + 1][O] = out;  // the next stage's newest row for step tau+1
        } else if (L.own && row >= r0 && row < r1) {
            double* dst = xout + (long long)row * nx + L.c0;
            if (L.vec && L.in0 && L.in1) {
                *reinterpret_cast<double2*>(dst) = make_double2(out.a, out.b);
            } else {
                if (L.in0) dst[0] = out.a;
                if (L.in1) dst[1] = out.b;
            }
        }
    }
    // stage 0's next newest row (tau+1) from the prefetch queue; refill it
    ring[0][O] = pre[P];
    pre[P] = ws_row(xin, tau + 4, ny, nx, L);
}

template <int S, int H>
__device__ __forceinline__ void ws_item(const WsArgs& a, const double* __restrict__ xin,
                                        double* __restrict__ xout, int k0, int strip, int r0,
                                        int r1, double (&acc)[S], bool accumulate) {
    const int lane = threadIdx.x & 31;
    const int nx = a.g.nx, ny = a.g.ny;
    constexpr int VW = 64 - 2 * S;
    WsLane L;
    L.c0 = strip * VW - S + 2 * lane;
    L.in0 = L.c0 >= 0 && L.c0 < nx;
    L.in1 = L.c0 + 1 >= 0 && L.c0 + 1 < nx;
    L.own = 2 * lane >= S && 2 * lane < 64 - S;
    L.vec = (nx & 1) == 0 && ((((uintptr_t)xin) | ((uintptr_t)xout) | ((uintptr_t)a.b)) & 15) == 0;
    double w[H];
#pragma unroll
    for (int t = 0; t < H; ++t) w[t] = __ldg(a.omegas + k0 + t);
    Pair ring[H][3];
#pragma unroll
    for (int t = 0; t < H; ++t)
#pragma unroll
        for (int q = 0; q < 3; ++q) ring[t][q] = Pair{0.0, 0.0};
    // first step: stage 0 sees x_{k0} rows r0-H .. r0-H+2, the last H rows of
    // output come H-1 skew steps after the last input row
    const int first = r0 - H + 2, last = r1 + 2 * H - 2;
    ring[0][0] = ws_row(xin, first - 2, ny, nx, L);
    ring[0][1] = ws_row(xin, first - 1, ny, nx, L);
    ring[0][2] = ws_row(xin, first, ny, nx, L);
    Pair pre[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) pre[q] = ws_row(xin, first + 1 + q, ny, nx, L);
    for (int tau = first; tau <= last; tau += 3) {
        ws_step<S, H, 0>(a, xin, xout, tau, r0, r1, L, w, ring, pre, acc, accumulate);
        if (tau + 1 <= last)
            ws_step<S, H, 1>(a, xin, xout, tau + 1, r0, r1, L, w, ring, pre, acc, accumulate);
        if (tau + 2 <= last)
            ws_step<S, H, 2>(a, xin, xout, tau + 2, r0, r1, L, w, ring, pre, acc, accumulate);
    }
}

template <int S, int H>
__device__ __forceinline__ void ws_pass_h(const WsArgs& a, const double* xin, double* xout,
                                          int k0, double (&acc)[S], bool accumulate) {
    const int warps = gridDim.x * (blockDim.x >> 5);
    const int wid = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    for (int item = wid; item < a.items; item += warps) {
        const int strip = item % a.strips, chunk = item / a.strips;
        const int r0 = chunk * a.rc, r1 = min(r0 + a.rc, a.g.ny);
        ws_item<S, H>(a, xin, xout, k0, strip, r0, r1, acc, accumulate);
    }
}

// h sub-sweeps (1 <= h <= S) with a compile-time stage count.
template <int S>
__device__ __forceinline__ void ws_pass(const WsArgs& a, const double* xin, double* xout,
                                        int k0, int h, double (&acc)[S], bool accumulate) {
#define SRJ_WS_CASE(HH)                                                          \
    case HH:                                                                     \
        if constexpr (HH <= S) ws_pass_h<S, HH>(a, xin, xout, k0, acc, accumulate); \
        break;
    switch (h) {
        SRJ_WS_CASE(1)
        SRJ_WS_CASE(2)
        SRJ_WS_CASE(3)
        SRJ_WS_CASE(4)
        SRJ_WS_CASE(5)
        SRJ_WS_CASE(6)
        default: break;
    }
#undef SRJ_WS_CASE
}

template <int S>
__global__ void __launch_bounds__(kWsThreads) k_ws2d_cycle(WsArgs a) {
    __shared__ double sh[32 * S];
    __shared__ double red[S];
    __shared__ double sh1[32];
    const int nb = gridDim.x;
    double* const buf[2] = {a.buf0, a.buf1};
    const int npasses = (a.M + a.s - 1) / a.s;
    int executed = a.M, status = kStatusRan, result = npasses & 1;
    double S2 = 0.0, res = 0.0;
    bool stopped = false;
    for (int p = 0; p < npasses && !stopped; ++p) {
        const int k0 = p * a.s;
        const int h = min(a.s, a.M - k0);
        double acc[S];
#pragma unroll
        for (int t = 0; t < S; ++t) acc[t] = 0.0;
        ws_pass<S>(a, buf[p & 1], buf[(p + 1) & 1], k0, h, acc, true);
        double* part = a.partials + (size_t)(p & 1) * kWsMaxS * nb;
        block_sums<S>(acc, h, sh, red);
        if (threadIdx.x < h) part[threadIdx.x * nb + blockIdx.x] = red[threadIdx.x];
        grid_barrier();
        reduce_partials_multi(part, nb, h, red);
        int stop_t = -1;
        for (int t = 0; t < h; ++t) {
            const int k = k0 + t;
            if (k == 0) continue;
            S2 = red[t];
            res = sqrt(S2) / a.baseline;
            if (blockIdx.x == 0 && threadIdx.x == 0) a.hist[k] = res;
            if (!isfinite(res)) { status = kStatusDiverged; stop_t = t; break; }
            if (res <= a.tol) { status = kStatusConverged; stop_t = t; break; }
        }
        __syncthreads();
        if (stop_t >= 0) {
            stopped = true;
            executed = k0 + stop_t;
            if (stop_t == 0) {
                result = p & 1;
            } else {
                ws_pass<S>(a, buf[p & 1], buf[(p + 1) & 1], k0, stop_t, acc, false);
                grid_barrier();
                result = (p + 1) & 1;
            }
        }
    }
    if (!stopped) {
        const int u0 = (int)((long long)a.g.units * blockIdx.x / nb);
        const int u1 = (int)((long long)a.g.units * (blockIdx.x + 1) / nb);
        double acc = walk_units<F2D, kResid>(a.g, buf[result], nullptr, a.b, 0.0, u0, u1);
        double* part = a.partials + (size_t)(npasses & 1) * kWsMaxS * nb;
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

template <int S>
static cudaError_t ws_setup(int& per_sm) {
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_ws2d_cycle<S>, kWsThreads, 0);
}

cudaError_t ws_plan_init(WsPlan& plan, const Geom& g, int num_sms) {
    plan = WsPlan();
    if (g.fam != F2D) return cudaSuccess;
    cudaError_t e;
    if ((e = ws_setup<2>(plan.per_sm[0])) != cudaSuccess) return e;
    if ((e = ws_setup<4>(plan.per_sm[1])) != cudaSuccess) return e;
    plan.num_sms = num_sms;
    plan.supported = plan.per_sm[0] >= 1 && plan.per_sm[1] >= 1;
    return cudaSuccess;
}

template <int S>
static cudaError_t ws_launch(const WsPlan& plan, int per_sm, WsArgs& a, cudaStream_t st) {
    const int vw = 64 - 2 * S;
    a.strips = (a.g.nx + vw - 1) / vw;
    const int blocks = std::max(1, per_sm * plan.num_sms);
    const long long warps = (long long)blocks * (kWsThreads / 32);
    // rows per item: about one item per warp, at least 8*S rows to amortise
    // the 2*S halo rows and the 2*S skew steps each item adds
    const long long chunks = std::max<long long>(1, warps / a.strips);
    a.rc = (int)std::max<long long>(8 * S, (a.g.ny + chunks - 1) / chunks);
    a.items = a.strips * ((a.g.ny + a.rc - 1) / a.rc);
    void* args[] = {&a};
    return cudaLaunchCooperativeKernel((const void*)k_ws2d_cycle<S>, dim3(blocks),
                                       dim3(kWsThreads), args, 0, st);
}

cudaError_t ws_launch_cycle(const WsPlan& plan, const Geom& g, double* x, double* x_alt,
                            const double* b, const double* omegas, int M, int s, double tol,
                            double baseline, double* partials, double* hist, int* out_i,
                            double* out_d, cudaStream_t st) {
    WsArgs a;
    a.g = g;
    a.buf0 = x;
    a.buf1 = x_alt;
    a.b = b;
    a.omegas = omegas;
    a.M = M;
    a.tol = tol;
    a.baseline = baseline;
    a.partials = partials;
    a.hist = hist;
    a.out_i = out_i;
    a.out_d = out_d;
    if (s <= 2) {
        a.s = std::max(1, s);
        return ws_launch<2>(plan, plan.per_sm[0], a, st);
    }
    // s > 4 is served by the S = 4 variant (4 sweeps per pass): the S = 6
    // variant is not parity-clean yet (negative results)
    a.s = std::min(s, 4);
    return ws_launch<4>(plan, plan.per_sm[1], a, st);
}

}  // namespace srj
