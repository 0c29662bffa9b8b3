// Temporally blocked SRJ cycle for the 2D 5-point constant-coefficient
// stencil (BASELINE config 2): up to S consecutive sweeps, each with its own
// omega, per HBM/L2 round trip of x and b.
//
// Tiling.  A CTA (one per SM, persistent, cooperative launch) owns 64 x 64
// output tiles.  For each tile the copy engine (TMA) brings the (64+2S)^2 region
// of x_{k0} and b into shared memory; boxes that stick out of the grid are
// zero-filled, which is the Dirichlet ghost.  The next tile's boxes are
// prefetched while the current tile computes.
//
// Register tiling.  Thread (c, seg) keeps rows [seg*V, seg*V+V) of region
// column c in registers; per sub-sweep it publishes them to a shared exchange
// buffer and reads only its west/east neighbours (plus one row above and below
// its segment) back: ~3 shared accesses per point instead of 6, and V
// independent fp64 dependency chains per thread.  Every point of the region is
// updated every sub-sweep (no divergence); values within t+1 rings of the
// region edge are garbage after sub-sweep t but never reach the owned tile,
// which after h <= S sub-sweeps holds x_{k0+h} exactly -- each value produced
// by the per-point arithmetic of the one-sweep kernel (bit-identical iterates).
// Grid-exterior points are held at 0.
//
// Residuals.  Sub-sweep t accumulates (b - A x_{k0+t})^2 over OWNED points only,
// so the per-CTA partials have the meaning of the one-sweep kernel's.  After a
// pass a grid barrier lets every CTA reduce them in a fixed order and apply the
// reference's per-sweep stopping rule (solver.py:216-222,235-239).  A stop at
// sweep k0+j, j >= 1, re-runs the pass with j sub-sweeps from its intact input
// buffer (rollback); j = 0 returns the input buffer itself.
#include <cooperative_groups.h>

#include <algorithm>

#include "srj_stencil.cuh"
#include "srj_tb.cuh"
#include "srj_tma.cuh"
#include "srj_walk.cuh"

namespace srj {
namespace tb2d {

template <int S>
struct Cfg {
    static constexpr int TX = 64, TY = 64;
    static constexpr int RX = TX + 2 * S, RY = TY + 2 * S;
    static constexpr int NSEG = 8;
    static constexpr int V = RY / NSEG;
    static_assert(RY % NSEG == 0, "segments must tile the region height");
    static constexpr int THREADS = RX * NSEG;
    static constexpr int EP = RX + 2;        // exchange buffer pitch (zero border)
    static constexpr int EROWS = RY + 2;
    static constexpr int STAGE = RX * RY;    // doubles per staged box
    static constexpr int EX = EP * EROWS;    // doubles per exchange buffer
    static constexpr size_t SMEM = (size_t)(2 * STAGE + 2 * EX) * sizeof(double) + 16;
    static constexpr uint32_t TX_BYTES = 2u * STAGE * sizeof(double);
};

}  // namespace tb2d

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
};

template <int S>
struct TbSmem {
    double* stx;
    double* stb;
    double* E0;
    double* E1;
    uint64_t* bar;
};

template <int S>
__device__ __forceinline__ void tb2d_issue(const TbArgs& a, const CUtensorMap* tm_in,
                                           const CUtensorMap* tm_b, const TbSmem<S>& sm, int q) {
    using C = tb2d::Cfg<S>;
    const int ox = (q % a.tiles_x) * C::TX, oy = (q / a.tiles_x) * C::TY;
    fence_proxy_async();
    mbar_expect_tx(sm.bar, C::TX_BYTES);
    tma_load_2d(sm.stx, tm_in, ox - S, oy - S, sm.bar);
    tma_load_2d(sm.stb, tm_b, ox - S, oy - S, sm.bar);
}

// One pass (h sub-sweeps, h <= S) over every tile this CTA owns.
template <int S>
__device__ __forceinline__ void tb2d_pass(const TbArgs& a, const CUtensorMap* tm_in,
                                          const CUtensorMap* tm_b, double* __restrict__ xout,
                                          int k0, int h, double (&acc)[S], bool accumulate,
                                          const TbSmem<S>& sm, uint32_t& phase) {
    using C = tb2d::Cfg<S>;
    constexpr int V = C::V, RX = C::RX, EP = C::EP;
    const int tid = threadIdx.x;
    const int c = tid % RX, seg = tid / RX, r0 = seg * V;
    const int nx = a.g.nx, ny = a.g.ny;
    const double coff = a.g.c_off, cdiag = a.g.c_diag, inv = a.g.inv_diag;
    if ((int)blockIdx.x >= a.ntiles) return;
    if (tid == 0) tb2d_issue<S>(a, tm_in, tm_b, sm, blockIdx.x);
    for (int q = blockIdx.x; q < a.ntiles; q += gridDim.x) {
        const int ox = (q % a.tiles_x) * C::TX, oy = (q / a.tiles_x) * C::TY;
        const int gx = ox - S + c;
        const int gy0 = oy - S + r0;
        const bool colin = gx >= 0 && gx < nx;
        const bool ocol = c >= S && c < S + C::TX;
        mbar_wait(sm.bar, phase);
        phase ^= 1u;
        double xr[V], br[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            xr[v] = sm.stx[(r0 + v) * RX + c];
            br[v] = sm.stb[(r0 + v) * RX + c];
            sm.E0[(r0 + v + 1) * EP + c + 1] = xr[v];
        }
        __syncthreads();  // staging consumed, E0 published
        if (tid == 0 && q + (int)gridDim.x < a.ntiles)
            tb2d_issue<S>(a, tm_in, tm_b, sm, q + gridDim.x);
#pragma unroll
        for (int t = 0; t < S; ++t) {
            if (t < h) {
                const double w = __ldg(a.omegas + k0 + t);
                const double* Ein = (t & 1) ? sm.E1 : sm.E0;
                double* Eout = (t & 1) ? sm.E0 : sm.E1;
                const double hs = Ein[r0 * EP + c + 1];
                const double hn = Ein[(r0 + V + 1) * EP + c + 1];
                double nr[V];
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    const double* e = Ein + (r0 + v + 1) * EP + c;
                    const double xs = v == 0 ? hs : xr[v - 1];
                    const double xn = v == V - 1 ? hn : xr[v + 1];
                    double y = DADD(0.0, DMUL(coff, xs));
                    y = DADD(y, DMUL(coff, e[0]));
                    y = DADD(y, DMUL(cdiag, xr[v]));
                    y = DADD(y, DMUL(coff, e[2]));
                    y = DADD(y, DMUL(coff, xn));
                    const double rr = DSUB(br[v], y);
                    const int gy = gy0 + v;
                    const bool in = colin && gy >= 0 && gy < ny;
                    nr[v] = in ? relax(xr[v], inv, rr, w) : 0.0;
                    const int r = r0 + v;
                    if (accumulate && in && ocol && r >= S && r < S + C::TY)
                        acc[t] = fma(rr, rr, acc[t]);
                }
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    Eout[(r0 + v + 1) * EP + c + 1] = nr[v];
                    xr[v] = nr[v];
                }
                __syncthreads();
            }
        }
        if (ocol && colin) {
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const int r = r0 + v, gy = gy0 + v;
                if (r >= S && r < S + C::TY && gy < ny) xout[(long long)gy * nx + gx] = xr[v];
            }
        }
    }
}

template <int S>
__global__ void __launch_bounds__(tb2d::Cfg<S>::THREADS, 1)
    k_tb2d_cycle(const __grid_constant__ CUtensorMap tm_x0,
                 const __grid_constant__ CUtensorMap tm_x1,
                 const __grid_constant__ CUtensorMap tm_b, TbArgs a) {
    using C = tb2d::Cfg<S>;
    extern __shared__ __align__(128) double smem[];
    __shared__ double sh[32];
    TbSmem<S> sm;
    sm.stx = smem;
    sm.stb = smem + C::STAGE;
    sm.E0 = smem + 2 * C::STAGE;
    sm.E1 = sm.E0 + C::EX;
    sm.bar = reinterpret_cast<uint64_t*>(sm.E1 + C::EX);
    for (int i = threadIdx.x; i < 2 * C::EX; i += blockDim.x) sm.E0[i] = 0.0;
    if (threadIdx.x == 0) {
        mbar_init(sm.bar, 1);
        prefetch_tensormap(&tm_x0);
        prefetch_tensormap(&tm_x1);
        prefetch_tensormap(&tm_b);
    }
    __syncthreads();
    uint32_t phase = 0;
    const int nb = gridDim.x;
    double* const buf[2] = {a.buf0, a.buf1};
    const CUtensorMap* const tmx[2] = {&tm_x0, &tm_x1};
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
        tb2d_pass<S>(a, tmx[p & 1], &tm_b, buf[(p + 1) & 1], k0, h, acc, true, sm, phase);
        double* part = a.partials + (size_t)(p & 1) * kTbMaxSub * nb;
#pragma unroll
        for (int t = 0; t < S; ++t) {
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
            S2 = reduce_partials(part + t * nb, nb, sh);
            res = sqrt(S2) / a.baseline;
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
                tb2d_pass<S>(a, tmx[p & 1], &tm_b, buf[(p + 1) & 1], k0, stop_t, acc, false, sm,
                             phase);
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
        double* part = a.partials + (size_t)(npasses & 1) * kTbMaxSub * nb;
        acc = block_allsum(acc, sh);
        if (threadIdx.x == 0) part[blockIdx.x] = acc;
        grid_barrier();
        S2 = reduce_partials(part, nb, sh);
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

// ----------------------------------------------------------------------------
// Host side
// ----------------------------------------------------------------------------

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    }
    return fn;
}

cudaError_t encode_field_map(CUtensorMap* map, const double* base, int nx, int ny, int box_x,
                             int box_y) {
    EncodeTiledFn fn = encode_fn();
    if (!fn) return cudaErrorNotSupported;
    const cuuint64_t dims[2] = {(cuuint64_t)nx, (cuuint64_t)ny};
    const cuuint64_t strides[1] = {(cuuint64_t)nx * sizeof(double)};
    const cuuint32_t box[2] = {(cuuint32_t)box_x, (cuuint32_t)box_y};
    const cuuint32_t es[2] = {1, 1};
    CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims,
                    strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorInvalidValue;
}

template <int S>
static cudaError_t setup_variant(int& per_sm) {
    using C = tb2d::Cfg<S>;
    cudaError_t e = cudaFuncSetAttribute(k_tb2d_cycle<S>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tb2d_cycle<S>, C::THREADS,
                                                         C::SMEM);
}

cudaError_t tb_plan_init(TbPlan& plan, const Geom& g, int num_sms) {
    plan = TbPlan();
    // TMA needs 16-byte row pitch: even nx.
    if (g.fam != F2D || (g.nx & 1) || !encode_fn()) return cudaSuccess;
    int per4 = 0, per8 = 0;
    cudaError_t e = setup_variant<4>(per4);
    if (e != cudaSuccess) return e;
    if ((e = setup_variant<8>(per8)) != cudaSuccess) return e;
    if (per4 < 1 || per8 < 1) return cudaSuccess;
    plan.tiles_x = (g.nx + 63) / 64;
    plan.ntiles = plan.tiles_x * ((g.ny + 63) / 64);
    plan.blocks = std::max(1, std::min(num_sms, plan.ntiles));
    plan.supported = true;
    return cudaSuccess;
}

template <int S>
static cudaError_t launch_variant(const TbPlan& plan, const CUtensorMap (&maps)[3], TbArgs& a,
                                  cudaStream_t st) {
    using C = tb2d::Cfg<S>;
    CUtensorMap m0 = maps[0], m1 = maps[1], mb = maps[2];
    void* args[] = {&m0, &m1, &mb, &a};
    return cudaLaunchCooperativeKernel((const void*)k_tb2d_cycle<S>, dim3(plan.blocks),
                                       dim3(C::THREADS), args, C::SMEM, st);
}

cudaError_t tb_launch_cycle(const TbPlan& plan, const Geom& g, double* x, double* x_alt,
                            const double* b, const double* omegas, int M, int s, double tol,
                            double baseline, double* partials, double* hist, int* out_i,
                            double* out_d, cudaStream_t st) {
    if ((((uintptr_t)x | (uintptr_t)x_alt | (uintptr_t)b) & 15) != 0)
        return cudaErrorMisalignedAddress;
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
    const int S = a.s <= 4 ? 4 : 8;
    const int box = 64 + 2 * S;
    CUtensorMap maps[3];
    cudaError_t e;
    if ((e = encode_field_map(&maps[0], x, g.nx, g.ny, box, box)) != cudaSuccess) return e;
    if ((e = encode_field_map(&maps[1], x_alt, g.nx, g.ny, box, box)) != cudaSuccess) return e;
    if ((e = encode_field_map(&maps[2], b, g.nx, g.ny, box, box)) != cudaSuccess) return e;
    return S == 4 ? launch_variant<4>(plan, maps, a, st) : launch_variant<8>(plan, maps, a, st);
}

}  // namespace srj
