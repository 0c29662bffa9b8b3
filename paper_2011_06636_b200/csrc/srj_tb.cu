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
#include <cstdlib>

#include "srj_stencil.cuh"
#include "srj_tb.cuh"
#include "srj_tma.cuh"
#include "srj_walk.cuh"

namespace srj {
namespace tb2d {

template <int S_, int TX_, int TY_, int NSEG_>
struct CfgBase {
    static constexpr int S = S_, TX = TX_, TY = TY_;
    static constexpr int RX = TX + 2 * S, RY = TY + 2 * S;
    static constexpr int NSEG = NSEG_;
    static constexpr int V = RY / NSEG;
    static_assert(RY % NSEG == 0, "segments must tile the region height");
    static constexpr int THREADS = RX * NSEG;
    // Registers are allocated per SM sub-partition (16K each, 4 per SM): with
    // W warps, ceil(W/4) warps share one.
    static constexpr int WARPS_PER_SMSP = ((THREADS + 31) / 32 + 3) / 4;
    static constexpr int MAXREG_RAW = (16384 / (WARPS_PER_SMSP * 32)) / 8 * 8;
    static constexpr int MAXREG = MAXREG_RAW > 255 ? 255 : MAXREG_RAW;
    static constexpr int EP = RX + 2;        // exchange buffer pitch (zero border)
    static constexpr int EROWS = RY + 2;
    static constexpr int STAGE = RX * RY;    // doubles per staged box
    static constexpr int EX = EP * EROWS;    // doubles per exchange buffer
    static constexpr size_t SMEM = (size_t)(2 * STAGE + 2 * EX) * sizeof(double) + 16;
    static constexpr uint32_t TX_BYTES = 2u * STAGE * sizeof(double);
};

// Kernel variants: K -> (sweeps per pass S, owned tile TX x TY, segments).
template <int K>
struct Cfg;
template <>
struct Cfg<0> : CfgBase<4, 64, 64, 8> {};  // 72x72 region, 576 threads
template <>
struct Cfg<1> : CfgBase<8, 64, 64, 8> {};  // 80x80 region, 640 threads
template <>
struct Cfg<2> : CfgBase<4, 56, 64, 8> {};  // 64x72 region, 512 threads (128 regs)
constexpr int kVariants = 3;

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

template <int K>
struct TbSmem {
    double* stx;
    double* stb;
    double* E0;
    double* E1;
    uint64_t* bar;
};

template <int K>
__device__ __forceinline__ void tb2d_issue(const TbArgs& a, const CUtensorMap* tm_in,
                                           const CUtensorMap* tm_b, const TbSmem<K>& sm, int q) {
    constexpr int S = tb2d::Cfg<K>::S;
    using C = tb2d::Cfg<K>;
    const int ox = (q % a.tiles_x) * C::TX, oy = (q / a.tiles_x) * C::TY;
    fence_proxy_async();
    mbar_expect_tx(sm.bar, C::TX_BYTES);
    tma_load_2d(sm.stx, tm_in, ox - S, oy - S, sm.bar);
    tma_load_2d(sm.stb, tm_b, ox - S, oy - S, sm.bar);
}

// H sub-sweeps (compile-time, H <= S) of the staged tile held in registers
// (xr) and in the exchange buffer E0.  MASKED tiles reach outside the grid:
// points there (bit clear in `inmask`) are held at 0.  Points with a bit set
// in `accmask` (owned, in the grid) add r^2 to acc[t].
template <int K, int H, bool MASKED>
__device__ __forceinline__ void tile_sweeps(double (&xr)[tb2d::Cfg<K>::V],
                                            const double (&br)[tb2d::Cfg<K>::V],
                                            const TbSmem<K>& sm, const double* omegas,
                                            const Geom& g, int r0, int c, unsigned inmask,
                                            unsigned accmask, double (&acc)[tb2d::Cfg<K>::S]) {
    using C = tb2d::Cfg<K>;
    constexpr int V = C::V, EP = C::EP;
    const double coff = g.c_off, cdiag = g.c_diag, inv = g.inv_diag;
#pragma unroll
    for (int t = 0; t < H; ++t) {
        const double w = __ldg(omegas + t);
        const double* Ein = (t & 1) ? sm.E1 : sm.E0;
        double* Eout = (t & 1) ? sm.E0 : sm.E1;
        const double* base = Ein + (r0 + 1) * EP + c;
        const double hs = base[1 - EP];
        const double hn = base[V * EP + 1];
        double nr[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const double xs = v == 0 ? hs : xr[v - 1];
            const double xn = v == V - 1 ? hn : xr[v + 1];
            double y = DADD(0.0, DMUL(coff, xs));
            y = DADD(y, DMUL(coff, base[v * EP]));
            y = DADD(y, DMUL(cdiag, xr[v]));
            y = DADD(y, DMUL(coff, base[v * EP + 2]));
            y = DADD(y, DMUL(coff, xn));
            const double rr = DSUB(br[v], y);
            const double nv = relax(xr[v], inv, rr, w);
            nr[v] = (!MASKED || ((inmask >> v) & 1u)) ? nv : 0.0;
            if ((accmask >> v) & 1u) acc[t] = fma(rr, rr, acc[t]);
        }
        double* obase = Eout + (r0 + 1) * EP + c + 1;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            obase[v * EP] = nr[v];
            xr[v] = nr[v];
        }
        __syncthreads();
    }
}

template <int K, bool MASKED>
__device__ __forceinline__ void tile_dispatch(int h, double (&xr)[tb2d::Cfg<K>::V],
                                              const double (&br)[tb2d::Cfg<K>::V],
                                              const TbSmem<K>& sm, const double* omegas,
                                              const Geom& g, int r0, int c, unsigned inmask,
                                              unsigned accmask, double (&acc)[tb2d::Cfg<K>::S]) {
    constexpr int S = tb2d::Cfg<K>::S;
#define SRJ_TB_CASE(H)                                                                     \
    case H:                                                                                \
        if constexpr (H <= S)                                                              \
            tile_sweeps<K, H, MASKED>(xr, br, sm, omegas, g, r0, c, inmask, accmask, acc); \
        break;
    switch (h) {
        SRJ_TB_CASE(1)
        SRJ_TB_CASE(2)
        SRJ_TB_CASE(3)
        SRJ_TB_CASE(4)
        SRJ_TB_CASE(5)
        SRJ_TB_CASE(6)
        SRJ_TB_CASE(7)
        SRJ_TB_CASE(8)
        default: break;
    }
#undef SRJ_TB_CASE
}

// One pass (h sub-sweeps, h <= S) over every tile this CTA owns.  If
// `first_issued`, the TMA for this CTA's first tile is already in flight.
template <int K>
__device__ __forceinline__ void tb2d_pass(const TbArgs& a, const CUtensorMap* tm_in,
                                          const CUtensorMap* tm_b, double* __restrict__ xout,
                                          int k0, int h, double (&acc)[tb2d::Cfg<K>::S], bool accumulate,
                                          unsigned ownmask, const TbSmem<K>& sm,
                                          uint32_t& phase, bool first_issued) {
    using C = tb2d::Cfg<K>;
    constexpr int S = C::S;
    constexpr int V = C::V, RX = C::RX, EP = C::EP;
    const int tid = threadIdx.x;
    const int c = tid % RX, seg = tid / RX, r0 = seg * V;
    const int nx = a.g.nx, ny = a.g.ny;
    if ((int)blockIdx.x >= a.ntiles) return;
    if (tid == 0 && !first_issued) tb2d_issue<K>(a, tm_in, tm_b, sm, blockIdx.x);
    for (int q = blockIdx.x; q < a.ntiles; q += gridDim.x) {
        const int ox = (q % a.tiles_x) * C::TX, oy = (q / a.tiles_x) * C::TY;
        const int gx = ox - S + c;
        const int gy0 = oy - S + r0;
        const bool masked = ox < S || oy < S || ox + C::TX + S > nx || oy + C::TY + S > ny;
        unsigned inmask = (1u << V) - 1u;
        if (masked) {
            inmask = 0u;
            if (gx >= 0 && gx < nx) {
#pragma unroll
                for (int v = 0; v < V; ++v)
                    if (gy0 + v >= 0 && gy0 + v < ny) inmask |= 1u << v;
            }
        }
        const unsigned storemask = ownmask & inmask;
        const unsigned accmask = accumulate ? storemask : 0u;
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
            tb2d_issue<K>(a, tm_in, tm_b, sm, q + gridDim.x);
        if (masked)
            tile_dispatch<K, true>(h, xr, br, sm, a.omegas + k0, a.g, r0, c, inmask, accmask, acc);
        else
            tile_dispatch<K, false>(h, xr, br, sm, a.omegas + k0, a.g, r0, c, inmask, accmask, acc);
        if (storemask) {
#pragma unroll
            for (int v = 0; v < V; ++v)
                if ((storemask >> v) & 1u) xout[(long long)(gy0 + v) * nx + gx] = xr[v];
        }
    }
}

template <int K>
__global__ void __maxnreg__(tb2d::Cfg<K>::MAXREG)
    k_tb2d_cycle(const __grid_constant__ CUtensorMap tm_x0,
                 const __grid_constant__ CUtensorMap tm_x1,
                 const __grid_constant__ CUtensorMap tm_b, TbArgs a) {
    using C = tb2d::Cfg<K>;
    constexpr int S = C::S;
    extern __shared__ __align__(128) double smem[];
    __shared__ double sh[32 * S];
    __shared__ double red[S];
    __shared__ double sh1[32];
    TbSmem<K> sm;
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
    // owned-point bits of this thread's column segment (tile-independent)
    unsigned ownmask = 0u;
    {
        const int c = threadIdx.x % C::RX, r0 = (threadIdx.x / C::RX) * C::V;
        if (c >= S && c < S + C::TX) {
#pragma unroll
            for (int v = 0; v < C::V; ++v)
                if (r0 + v >= S && r0 + v < S + C::TY) ownmask |= 1u << v;
        }
    }
    uint32_t phase = 0;
    const int nb = gridDim.x;
    double* const buf[2] = {a.buf0, a.buf1};
    const CUtensorMap* const tmx[2] = {&tm_x0, &tm_x1};
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
        tb2d_pass<K>(a, tmx[p & 1], &tm_b, buf[(p + 1) & 1], k0, h, acc, true, ownmask, sm,
                     phase, issued);
        issued = false;
        double* part = a.partials + (size_t)(p & 1) * kTbMaxSub * nb;
        block_sums<S>(acc, h, sh, red);
        if (threadIdx.x < h) part[threadIdx.x * nb + blockIdx.x] = red[threadIdx.x];
        grid_barrier();
        // Speculatively start the next pass's first tile while the stop test runs.
        if (p + 1 < npasses && (int)blockIdx.x < a.ntiles) {
            if (threadIdx.x == 0) tb2d_issue<K>(a, tmx[(p + 1) & 1], &tm_b, sm, blockIdx.x);
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
                mbar_wait(sm.bar, phase);
                phase ^= 1u;
                issued = false;
                __syncthreads();
            }
            if (stop_t == 0) {
                result = p & 1;
            } else {
                // rollback: x_{k0+stop_t} from the intact pass input
                tb2d_pass<K>(a, tmx[p & 1], &tm_b, buf[(p + 1) & 1], k0, stop_t, acc, false,
                             ownmask, sm, phase, false);
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

// ----------------------------------------------------------------------------
// Host side
// ----------------------------------------------------------------------------

template <int K>
static cudaError_t setup_variant(int& per_sm) {
    using C = tb2d::Cfg<K>;
    cudaError_t e = cudaFuncSetAttribute(k_tb2d_cycle<K>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tb2d_cycle<K>, C::THREADS,
                                                         C::SMEM);
}

template <int K>
static void plan_tiles(TbPlan& plan, const Geom& g, int num_sms) {
    using C = tb2d::Cfg<K>;
    plan.tiles_x[K] = (g.nx + C::TX - 1) / C::TX;
    plan.ntiles[K] = plan.tiles_x[K] * ((g.ny + C::TY - 1) / C::TY);
    plan.blocks[K] = std::max(1, std::min(num_sms, plan.ntiles[K]));
}

cudaError_t tb_plan_init(TbPlan& plan, const Geom& g, int num_sms) {
    plan = TbPlan();
    // TMA needs 16-byte row pitch: even nx.
    if (g.fam != F2D || (g.nx & 1) || !tma_available()) return cudaSuccess;
    int occ[tb2d::kVariants] = {0, 0, 0};
    cudaError_t e;
    if ((e = setup_variant<0>(occ[0])) != cudaSuccess) return e;
    if ((e = setup_variant<1>(occ[1])) != cudaSuccess) return e;
    if ((e = setup_variant<2>(occ[2])) != cudaSuccess) return e;
    plan.occupancy = std::min(occ[0], std::min(occ[1], occ[2]));
    if (plan.occupancy < 1) return cudaSuccess;
    plan_tiles<0>(plan, g, num_sms);
    plan_tiles<1>(plan, g, num_sms);
    plan_tiles<2>(plan, g, num_sms);
    // s <= 4 variant: SRJ_TB_VARIANT=0|2 overrides the default (tuning only)
    plan.small_variant = 2;
    if (const char* v = getenv("SRJ_TB_VARIANT")) plan.small_variant = atoi(v) == 0 ? 0 : 2;
    plan.supported = true;
    return cudaSuccess;
}

template <int K>
static cudaError_t launch_variant(const TbPlan& plan, const Geom& g, TbArgs& a, double* x,
                                  double* x_alt, const double* b, cudaStream_t st) {
    using C = tb2d::Cfg<K>;
    CUtensorMap m0, m1, mb;
    cudaError_t e;
    if ((e = encode_field_map(&m0, x, g.nx, g.ny, C::RX, C::RY)) != cudaSuccess) return e;
    if ((e = encode_field_map(&m1, x_alt, g.nx, g.ny, C::RX, C::RY)) != cudaSuccess) return e;
    if ((e = encode_field_map(&mb, b, g.nx, g.ny, C::RX, C::RY)) != cudaSuccess) return e;
    a.tiles_x = plan.tiles_x[K];
    a.ntiles = plan.ntiles[K];
    void* args[] = {&m0, &m1, &mb, &a};
    return cudaLaunchCooperativeKernel((const void*)k_tb2d_cycle<K>, dim3(plan.blocks[K]),
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
    if (a.s > 4) return launch_variant<1>(plan, g, a, x, x_alt, b, st);
    if (plan.small_variant == 0) return launch_variant<0>(plan, g, a, x, x_alt, b, st);
    return launch_variant<2>(plan, g, a, x, x_alt, b, st);
}

}  // namespace srj
