// Temporally blocked SRJ cycle for the 2D 5-point constant-coefficient
// stencil (BASELINE config 2): up to S = 4 consecutive sweeps, each with its
// own omega, per HBM/L2 round trip of x and b.
//
// Tiling.  A CTA (one per SM, persistent, cooperative launch) owns TX x 64
// output tiles.  For each tile the copy engine (TMA) brings the
// (TX+2S) x (64+2S) region of x_{k0} and b into shared memory; boxes that stick
// out of the grid are zero-filled, which is the Dirichlet ghost.  The next
// tile's boxes are prefetched (b double-buffered) while the current one
// computes.
//
// Shared products.  With constant coefficients the rounded product
// p_j = c_off * x_j is the same value for all four points that have x_j as a
// neighbour, so each point computes p once when its value is produced and
// publishes p (not x) to the exchange buffer:
//     y = ((((0 + p_s) + p_w) + c_diag*x) + p_e) + p_n
// is bit-identical to summing freshly rounded products (reference csr_matvec
// order), and costs 11 fp64 instructions per point-sweep instead of 15.
//
// Register tiling.  Thread (c, seg) keeps x and p of rows [seg*V, seg*V+V) of
// region column c in registers; per sub-sweep it reads its west/east
// neighbours' p and the p of one row above and below its segment from the
// exchange buffer, b from the staged tile, and publishes its new p.  Every
// region point is updated every sub-sweep; values within t+1 rings of the
// region edge are garbage after sub-sweep t but never reach the owned tile,
// which after h <= S sub-sweeps holds x_{k0+h} exactly (bit-identical
// iterates).  Grid-exterior points are held at 0.
//
// Residuals.  Sub-sweep t accumulates (b - A x_{k0+t})^2 over OWNED points
// only.  After a pass a grid barrier lets every CTA reduce the per-CTA partials
// in a fixed order and apply the reference's per-sweep stopping rule
// (solver.py:216-222,235-239).  A stop at sweep k0+j, j >= 1, re-runs the pass
// with j sub-sweeps from its intact input buffer (rollback); j = 0 returns the
// input buffer itself.
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
    static constexpr int EP = RX + 2;        // exchange buffer pitch (border columns)
    static constexpr int EROWS = RY + 2;
    static constexpr int STAGE = RX * RY;    // doubles per staged box
    static constexpr int EX = EP * EROWS;    // doubles per exchange buffer
    // x stage, two b stages, two exchange buffers, one mbarrier per b stage
    static constexpr size_t SMEM = (size_t)(3 * STAGE + 2 * EX) * sizeof(double) + 32;
    static constexpr uint32_t TX_BYTES = 2u * STAGE * sizeof(double);
};

// Kernel variants: K -> (sweeps per pass S, owned tile TX x TY, segments).
template <int K>
struct Cfg;
template <>
struct Cfg<0> : CfgBase<4, 64, 64, 8> {};  // 72x72 region, 576 threads
template <>
struct Cfg<1> : CfgBase<4, 56, 64, 8> {};  // 64x72 region, 512 threads
constexpr int kVariants = 2;

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

// Dynamic shared memory, indexed with compile-time offsets so every access
// compiles to LDS/STS (a pointer carried through a struct loses the address
// space and becomes a generic LD/ST).
extern __shared__ __align__(128) double tb_smem[];

template <int K>
struct TbLayout {
    using C = tb2d::Cfg<K>;
    static constexpr int STX = 0;                  // x stage
    static constexpr int STB = C::STAGE;           // b stages [2]
    static constexpr int E0 = 3 * C::STAGE;        // exchange buffers
    static constexpr int E1 = E0 + C::EX;
    static constexpr int BAR = E1 + C::EX;         // mbarriers [2] (one per b stage)
    __device__ static __forceinline__ double* stx() { return tb_smem + STX; }
    __device__ static __forceinline__ double* stb(int slot) { return tb_smem + STB + slot * C::STAGE; }
    __device__ static __forceinline__ double* e(int t) { return tb_smem + ((t & 1) ? E1 : E0); }
    __device__ static __forceinline__ uint64_t* bar(int slot) {
        return reinterpret_cast<uint64_t*>(tb_smem + BAR) + slot;
    }
};

template <int K>
__device__ __forceinline__ void tb2d_issue(const TbArgs& a, const CUtensorMap* tm_in,
                                           const CUtensorMap* tm_b, int q, int slot) {
    using C = tb2d::Cfg<K>;
    using L = TbLayout<K>;
    constexpr int S = C::S;
    const int ox = (q % a.tiles_x) * C::TX, oy = (q / a.tiles_x) * C::TY;
    fence_proxy_async();
    mbar_expect_tx(L::bar(slot), C::TX_BYTES);
    tma_load_2d(L::stx(), tm_in, ox - S, oy - S, L::bar(slot));
    tma_load_2d(L::stb(slot), tm_b, ox - S, oy - S, L::bar(slot));
}

// H sub-sweeps (compile-time, H <= S) of the staged tile: xr/pr hold this
// thread's x and p = c_off*x, the exchange buffer E0 holds everyone's p.
// MASKED tiles reach outside the grid: points there (bit clear in `inmask`)
// are held at 0.  Points with a bit set in `accmask` add r^2 to acc[t].
template <int K, int H, bool MASKED>
__device__ __forceinline__ void tile_sweeps(double (&xr)[tb2d::Cfg<K>::V],
                                            double (&pr)[tb2d::Cfg<K>::V], int slot,
                                            const double* omegas,
                                            const Geom& g, int r0, int c, unsigned inmask,
                                            unsigned accmask, double (&acc)[tb2d::Cfg<K>::S]) {
    using C = tb2d::Cfg<K>;
    constexpr int V = C::V, EP = C::EP, RX = C::RX;
    const double coff = g.c_off, cdiag = g.c_diag, inv = g.inv_diag;
    using L = TbLayout<K>;
    const double* bcol = L::stb(slot) + r0 * RX + c;
#pragma unroll
    for (int t = 0; t < H; ++t) {
        const double w = __ldg(omegas + t);
        const double* Ein = L::e(t);
        double* Eout = L::e(t + 1);
        const double* base = Ein + (r0 + 1) * EP + c;
        double south = base[1 - EP];            // p of the row above the segment
        const double north_end = base[V * EP + 1];  // p of the row below it
        double* obase = Eout + (r0 + 1) * EP + c + 1;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const double pn = v == V - 1 ? north_end : pr[v + 1];
            double y = DADD(0.0, south);
            y = DADD(y, base[v * EP]);
            y = DADD(y, DMUL(cdiag, xr[v]));
            y = DADD(y, base[v * EP + 2]);
            y = DADD(y, pn);
            const double rr = DSUB(bcol[v * RX], y);
            const double xn = relax(xr[v], inv, rr, w);
            if ((accmask >> v) & 1u) acc[t] = fma(rr, rr, acc[t]);
            south = pr[v];  // old p of row v: the south neighbour of row v+1
            xr[v] = (!MASKED || ((inmask >> v) & 1u)) ? xn : 0.0;
            pr[v] = DMUL(coff, xr[v]);
            obase[v * EP] = pr[v];
        }
        __syncthreads();
    }
}

template <int K, bool MASKED>
__device__ __forceinline__ void tile_dispatch(int h, double (&xr)[tb2d::Cfg<K>::V],
                                              double (&pr)[tb2d::Cfg<K>::V], int slot,
                                              const double* omegas,
                                              const Geom& g, int r0, int c, unsigned inmask,
                                              unsigned accmask, double (&acc)[tb2d::Cfg<K>::S]) {
    constexpr int S = tb2d::Cfg<K>::S;
#define SRJ_TB_CASE(H)                                                                      \
    case H:                                                                                 \
        if constexpr (H <= S)                                                               \
            tile_sweeps<K, H, MASKED>(xr, pr, slot, omegas, g, r0, c, inmask, accmask, acc); \
        break;
    switch (h) {
        SRJ_TB_CASE(1)
        SRJ_TB_CASE(2)
        SRJ_TB_CASE(3)
        SRJ_TB_CASE(4)
        default: break;
    }
#undef SRJ_TB_CASE
}

// One pass (h sub-sweeps, h <= S) over every tile this CTA owns.  If
// `first_issued`, the TMA for this CTA's first tile is already in flight in
// b slot `slot`.
template <int K>
__device__ __forceinline__ void tb2d_pass(const TbArgs& a, const CUtensorMap* tm_in,
                                          const CUtensorMap* tm_b, double* __restrict__ xout,
                                          int k0, int h, double (&acc)[tb2d::Cfg<K>::S],
                                          bool accumulate, unsigned ownmask, uint32_t& phase, int& slot, bool first_issued) {
    using C = tb2d::Cfg<K>;
    using L = TbLayout<K>;
    constexpr int S = C::S;
    constexpr int V = C::V, RX = C::RX, EP = C::EP;
    const int tid = threadIdx.x;
    const int c = tid % RX, seg = tid / RX, r0 = seg * V;
    const int nx = a.g.nx, ny = a.g.ny;
    const double coff = a.g.c_off;
    if ((int)blockIdx.x >= a.ntiles) return;
    if (tid == 0 && !first_issued) tb2d_issue<K>(a, tm_in, tm_b, blockIdx.x, slot);
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
        mbar_wait(L::bar(slot), (phase >> slot) & 1u);
        phase ^= 1u << slot;
        double xr[V], pr[V];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            xr[v] = L::stx()[(r0 + v) * RX + c];
            pr[v] = DMUL(coff, xr[v]);
            L::e(0)[(r0 + v + 1) * EP + c + 1] = pr[v];
        }
        __syncthreads();  // x staging consumed, E0 published
        if (tid == 0 && q + (int)gridDim.x < a.ntiles)
            tb2d_issue<K>(a, tm_in, tm_b, q + gridDim.x, slot ^ 1);
        if (masked)
            tile_dispatch<K, true>(h, xr, pr, slot, a.omegas + k0, a.g, r0, c, inmask, accmask,
                                   acc);
        else
            tile_dispatch<K, false>(h, xr, pr, slot, a.omegas + k0, a.g, r0, c, inmask, accmask,
                                    acc);
        if (storemask) {
#pragma unroll
            for (int v = 0; v < V; ++v)
                if ((storemask >> v) & 1u) xout[(long long)(gy0 + v) * nx + gx] = xr[v];
        }
        slot ^= 1;
    }
}

template <int K>
__global__ void __maxnreg__(tb2d::Cfg<K>::MAXREG)
    k_tb2d_cycle(const __grid_constant__ CUtensorMap tm_x0,
                 const __grid_constant__ CUtensorMap tm_x1,
                 const __grid_constant__ CUtensorMap tm_b, TbArgs a) {
    using C = tb2d::Cfg<K>;
    constexpr int S = C::S;
    using L = TbLayout<K>;
    __shared__ double sh[32 * S];
    __shared__ double red[S];
    __shared__ double sh1[32];
    for (int i = threadIdx.x; i < 2 * C::EX; i += blockDim.x) L::e(0)[i] = 0.0;
    if (threadIdx.x == 0) {
        mbar_init(L::bar(0), 1);
        mbar_init(L::bar(1), 1);
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
    int slot = 0;
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
        tb2d_pass<K>(a, tmx[p & 1], &tm_b, buf[(p + 1) & 1], k0, h, acc, true, ownmask, phase,
                     slot, issued);
        issued = false;
        double* part = a.partials + (size_t)(p & 1) * kTbMaxSub * nb;
        block_sums<S>(acc, h, sh, red);
        if (threadIdx.x < h) part[threadIdx.x * nb + blockIdx.x] = red[threadIdx.x];
        grid_barrier();
        // Speculatively start the next pass's first tile while the stop test runs.
        if (p + 1 < npasses && (int)blockIdx.x < a.ntiles) {
            if (threadIdx.x == 0)
                tb2d_issue<K>(a, tmx[(p + 1) & 1], &tm_b, blockIdx.x, slot);
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
                mbar_wait(L::bar(slot), (phase >> slot) & 1u);
                phase ^= 1u << slot;
                issued = false;
                __syncthreads();
            }
            if (stop_t == 0) {
                result = p & 1;
            } else {
                // rollback: x_{k0+stop_t} from the intact pass input
                tb2d_pass<K>(a, tmx[p & 1], &tm_b, buf[(p + 1) & 1], k0, stop_t, acc, false,
                             ownmask, phase, slot, false);
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
    int occ[tb2d::kVariants] = {0, 0};
    cudaError_t e;
    if ((e = setup_variant<0>(occ[0])) != cudaSuccess) return e;
    if ((e = setup_variant<1>(occ[1])) != cudaSuccess) return e;
    plan.occupancy = std::min(occ[0], occ[1]);
    if (plan.occupancy < 1) return cudaSuccess;
    plan_tiles<0>(plan, g, num_sms);
    plan_tiles<1>(plan, g, num_sms);
    // variant: SRJ_TB_VARIANT=0|1 overrides the default (tuning only)
    plan.small_variant = 1;
    if (const char* v = getenv("SRJ_TB_VARIANT")) plan.small_variant = atoi(v) == 0 ? 0 : 1;
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
    a.s = std::max(1, std::min(s, 4));  // the variants fuse at most 4 sweeps
    a.tol = tol;
    a.baseline = baseline;
    a.partials = partials;
    a.hist = hist;
    a.out_i = out_i;
    a.out_d = out_d;
    if (plan.small_variant == 0) return launch_variant<0>(plan, g, a, x, x_alt, b, st);
    return launch_variant<1>(plan, g, a, x, x_alt, b, st);
}

}  // namespace srj
