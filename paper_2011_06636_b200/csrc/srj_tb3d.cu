// Temporally blocked SRJ cycle for the 3D 7-point constant-coefficient
// stencil (BASELINE configs 3 and 5): S consecutive sweeps, each with its own
// omega, per HBM round trip of x and b.
//
// Tiling.  A CTA (one per SM, persistent, cooperative launch) owns TX x TY
// xy tiles and streams each through all z planes.  The copy engine (TMA)
// brings plane z of the RX x RY region (the tile plus an S-wide ring) of
// x_{k0} and b into a D-deep shared-memory ring; boxes that stick out of the
// grid are zero-filled (the Dirichlet ghost).
//
// Wavefront.  At plane step z, level t (t = 1..S) computes plane z-t of
// x_{k0+t} from planes z-t-1, z-t, z-t+1 of x_{k0+t-1}; the newest of those
// was produced by level t-1 in the same step (level 0 = the plane just loaded).
// (A 2-plane skew per level that makes the levels of a step independent was
// measured slower on B200: 699 vs 587 us per 512^3 sweep -- more live windows.)
// Each thread keeps, per level, a 3-plane register window of x and
// p = c_off*x for its CW x V points, so z-neighbours never touch shared
// memory; x-neighbours move by warp shuffle and y-neighbours come from the
// thread's own rows or from the edge rows the warps above/below published in
// the previous step.  Everything a step reads was published in the previous
// step (double-buffered by step parity), so one __syncthreads per plane step
// serves all S levels.
//
// Exactness.  y = 0 + p(z-1) + p(y-1) + p(x-1) + c_diag*x + p(x+1) + p(y+1)
// + p(z+1) in the reference csr_matvec column order with each product rounded
// once (shared between the six points that use it), r = b - y,
// x' = x + omega*(inv*r): bit-identical iterates.  Ghost terms (c_off*0) add
// signed zeros to a y that is never -0, so they are no-ops.  Region points
// outside the grid are held at 0; values within t rings of the region edge are
// garbage after level t but never reach the owned tile.
//
// Residuals and stopping: as the 2D kernel (srj_tb.cu) -- level t accumulates
// (b - A x_{k0+t-1})^2 over owned points, one grid barrier per pass, fixed-
// order reduction in every CTA, per-sweep stop test (solver.py:216-222,
// 235-239), rollback re-run of a pass that stops inside.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "srj_stencil.cuh"
#include "srj_tb.cuh"
#include "srj_tbdriver.cuh"
#include "srj_tma.cuh"
#include "srj_walk.cuh"

namespace srj {
namespace tb3d {

template <int S_, int NW_, int V_>
struct Cfg {
    static constexpr int S = S_;     // sweeps fused per pass (= ring width)
    static constexpr int CW = 2;     // columns per lane
    static constexpr int V = V_;     // rows per warp
    static constexpr int NW = NW_;   // warps
    static constexpr int RX = 32 * CW, RY = NW * V;
    static constexpr int TX = RX - 2 * S, TY = RY - 2 * S;
    static_assert(S % 2 == 0, "the box origin ox - S must stay 16-byte aligned");
    static constexpr int THREADS = 32 * NW;
    static constexpr int WARPS_PER_SMSP = (NW + 3) / 4;
    static constexpr int MAXREG_RAW = (16384 / (WARPS_PER_SMSP * 32)) / 8 * 8;
    static constexpr int MAXREG = MAXREG_RAW > 255 ? 255 : MAXREG_RAW;
    static constexpr int D = 4;                    // plane ring depth
    static constexpr int PLANE = RX * RY;          // doubles per staged plane box
    static constexpr int HROWS = NW + 2;           // edge rows incl. a zero row each side
    static constexpr int HB = 2 * HROWS * RX;      // top + bottom rows of one level, one parity
    // ring: D x-planes + D b-planes; edge rows [S levels][2 parities]; D mbarriers
    static constexpr size_t SMEM = (size_t)(2 * D * PLANE + 2 * S * HB) * sizeof(double) + 8 * D;
    static constexpr uint32_t TX_BYTES = 2u * PLANE * sizeof(double);
};

// Measured on B200, 512^3, us per sweep (plane-ring k_cycle3d: 557-574):
// C0 587, C1 598, C2 1109.
using C0 = Cfg<2, 10, 2>;  // 64x20 region, 60x16 tile, 320 threads
using C1 = Cfg<2, 20, 1>;  // 64x20 region, 60x16 tile, 640 threads
using C2 = Cfg<2, 16, 2>;  // 64x32 region, 60x28 tile, 512 threads

}  // namespace tb3d

using Tb3Args = TbArgs;


extern __shared__ __align__(128) double tb3_smem[];

template <class C>
struct Tb3Layout {
    static constexpr int XS = 0, BS = C::D * C::PLANE, H = 2 * C::D * C::PLANE;
    static constexpr int BAR = H + 2 * C::S * C::HB;
    __device__ static __forceinline__ double* xs(int slot) { return tb3_smem + XS + slot * C::PLANE; }
    __device__ static __forceinline__ double* bs(int slot) { return tb3_smem + BS + slot * C::PLANE; }
    // edge rows published by level-input u in a step of parity par
    __device__ static __forceinline__ double* top(int u, int par) {
        return tb3_smem + H + (u * 2 + par) * C::HB;
    }
    __device__ static __forceinline__ double* bot(int u, int par) {
        return tb3_smem + H + (u * 2 + par) * C::HB + C::HROWS * C::RX;
    }
    __device__ static __forceinline__ uint64_t* bar(int slot) {
        return reinterpret_cast<uint64_t*>(tb3_smem + BAR) + slot;
    }
};

template <int CW>
__device__ __forceinline__ void lds2(double (&d)[CW], const double* p) {
#pragma unroll
    for (int j = 0; j < CW; j += 2) {
        const double2 v = *reinterpret_cast<const double2*>(p + j);
        d[j] = v.x;
        d[j + 1] = v.y;
    }
}
template <int CW>
__device__ __forceinline__ void sts2(double* p, const double (&d)[CW]) {
#pragma unroll
    for (int j = 0; j < CW; j += 2) *reinterpret_cast<double2*>(p + j) = make_double2(d[j], d[j + 1]);
}

__device__ __forceinline__ void fma_sq_if3(double& acc, double r, unsigned cond) {
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p fma.rn.f64 %0, %1, %1, %0;\n\t}"
        : "+d"(acc)
        : "d"(r), "r"(cond));
}

// Load plane z of the region of tile (ox, oy) into ring slot z % D.
template <class C>
__device__ __forceinline__ void tb3_issue(const CUtensorMap* tm_x, const CUtensorMap* tm_b,
                                          int ox, int oy, int z) {
    using L = Tb3Layout<C>;
    const int slot = z % C::D;
    fence_proxy_async();
    mbar_expect_tx(L::bar(slot), C::TX_BYTES);
    tma_load_3d(L::xs(slot), tm_x, ox - C::S, oy - C::S, z, L::bar(slot));
    tma_load_3d(L::bs(slot), tm_b, ox - C::S, oy - C::S, z, L::bar(slot));
}

// Per-thread register windows of one level input u: x at the window centre
// plane c and at c+1, p = c_off*x at c-1, c, c+1.
template <class C>
struct Win {
    double xc[C::V][C::CW], xn[C::V][C::CW];
    double pm[C::V][C::CW], pc[C::V][C::CW], pn[C::V][C::CW];
};

// Stream one tile through all planes with H levels (H <= S sub-sweeps).
// `ph` holds one mbarrier parity bit per ring slot.  Returns with the ring
// idle (every issued load consumed).
template <class C, int H>
__device__ __forceinline__ void tb3_tile(const Tb3Args& a, const CUtensorMap* tm_in,
                                         const CUtensorMap* tm_b, double* __restrict__ xout,
                                         const double* omegas, int q, unsigned ownmask,
                                         bool accumulate, double (&acc)[C::S], uint32_t& ph) {
    using L = Tb3Layout<C>;
    constexpr int S = C::S, V = C::V, CW = C::CW, RX = C::RX, D = C::D;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c0 = lane * CW, r0 = warp * V;
    const int nx = a.g.nx, ny = a.g.ny, nz = a.g.nz;
    const long long pl = (long long)nx * ny;
    const double coff = a.g.c_off, cdiag = a.g.c_diag, inv = a.g.inv_diag;
    const int ox = (q % a.tiles_x) * C::TX, oy = (q / a.tiles_x) * C::TY;
    const int gx0 = ox - S + c0, gy0 = oy - S + r0;
    // in-grid (x, y) bits of this thread's points, bit v*CW + j
    unsigned inmask = 0u;
#pragma unroll
    for (int v = 0; v < V; ++v)
#pragma unroll
        for (int j = 0; j < CW; ++j)
            if (gy0 + v >= 0 && gy0 + v < ny && gx0 + j >= 0 && gx0 + j < nx)
                inmask |= 1u << (v * CW + j);
    const unsigned storemask = ownmask & inmask;
    const unsigned accmask = accumulate ? storemask : 0u;
    double w[H];
#pragma unroll
    for (int t = 0; t < H; ++t) w[t] = __ldg(omegas + t);

    // prologue: planes 0 .. D-1 in flight
    if (threadIdx.x == 0)
        for (int z = 0; z < D && z < nz; ++z) tb3_issue<C>(tm_in, tm_b, ox, oy, z);

    Win<C> W[H];
    double bw[H + 1][V][CW];  // b at planes z, z-1, ..., z-H
#pragma unroll
    for (int u = 0; u < H; ++u)
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
            for (int j = 0; j < CW; ++j) {
                W[u].xc[v][j] = W[u].xn[v][j] = 0.0;
                W[u].pm[v][j] = W[u].pc[v][j] = W[u].pn[v][j] = DMUL(coff, 0.0);
            }
#pragma unroll
    for (int k = 0; k <= H; ++k)
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
            for (int j = 0; j < CW; ++j) bw[k][v][j] = 0.0;

    for (int z = 0; z < nz + H; ++z) {
        const int par = z & 1;
        // ---- level-0 input: plane z of x_{k0} and b
        double xin[V][CW], bnew[V][CW];
        if (z < nz) {
            const int slot = z % D;
            mbar_wait(L::bar(slot), (ph >> slot) & 1u);
            ph ^= 1u << slot;
#pragma unroll
            for (int v = 0; v < V; ++v) {
                lds2<CW>(xin[v], L::xs(slot) + (r0 + v) * RX + c0);
                lds2<CW>(bnew[v], L::bs(slot) + (r0 + v) * RX + c0);
            }
        } else {
#pragma unroll
            for (int v = 0; v < V; ++v)
#pragma unroll
                for (int j = 0; j < CW; ++j) xin[v][j] = bnew[v][j] = 0.0;
        }
        // b window: bw[k] = b at plane z - k
#pragma unroll
        for (int k = H; k >= 1; --k)
#pragma unroll
            for (int v = 0; v < V; ++v)
#pragma unroll
                for (int j = 0; j < CW; ++j) bw[k][v][j] = bw[k - 1][v][j];
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
            for (int j = 0; j < CW; ++j) bw[0][v][j] = bnew[v][j];
#pragma unroll
        for (int t = 1; t <= H; ++t) {
            // ---- shift plane (z - t + 1) of level-input t-1 into its window
            Win<C>& Wu = W[t - 1];
#pragma unroll
            for (int v = 0; v < V; ++v)
#pragma unroll
                for (int j = 0; j < CW; ++j) {
                    Wu.pm[v][j] = Wu.pc[v][j];
                    Wu.pc[v][j] = Wu.pn[v][j];
                    Wu.xc[v][j] = Wu.xn[v][j];
                    Wu.xn[v][j] = xin[v][j];
                    Wu.pn[v][j] = DMUL(coff, xin[v][j]);
                }
            // publish the new plane's edge rows (read next step, when it is the centre)
            sts2<CW>(L::top(t - 1, par) + (warp + 1) * RX + c0, Wu.pn[0]);
            sts2<CW>(L::bot(t - 1, par) + (warp + 1) * RX + c0, Wu.pn[V - 1]);
            // ---- level t: plane c = z - t from the window centred at c
            const int c = z - t;
            const bool valid = c >= 0 && c < nz;
            double hs[CW], hn[CW];
            lds2<CW>(hs, L::bot(t - 1, par ^ 1) + warp * RX + c0);        // warp-1 bottom row
            lds2<CW>(hn, L::top(t - 1, par ^ 1) + (warp + 2) * RX + c0);  // warp+1 top row
            double pw[V], pe[V];
#pragma unroll
            for (int v = 0; v < V; ++v) {
                pw[v] = __shfl_up_sync(0xffffffffu, Wu.pc[v][CW - 1], 1);
                pe[v] = __shfl_down_sync(0xffffffffu, Wu.pc[v][0], 1);
            }
            const double* bt = &bw[t][0][0];  // b at plane z - t
            double sq0 = 0.0, sq1 = 0.0;
#pragma unroll
            for (int v = 0; v < V; ++v) {
                double y[CW];
#pragma unroll
                for (int j = 0; j < CW; ++j) y[j] = DADD(0.0, Wu.pm[v][j]);
#pragma unroll
                for (int j = 0; j < CW; ++j) y[j] = DADD(y[j], v == 0 ? hs[j] : Wu.pc[v - 1][j]);
#pragma unroll
                for (int j = 0; j < CW; ++j) y[j] = DADD(y[j], j == 0 ? pw[v] : Wu.pc[v][j - 1]);
#pragma unroll
                for (int j = 0; j < CW; ++j) y[j] = DADD(y[j], DMUL(cdiag, Wu.xc[v][j]));
#pragma unroll
                for (int j = 0; j < CW; ++j)
                    y[j] = DADD(y[j], j == CW - 1 ? pe[v] : Wu.pc[v][j + 1]);
#pragma unroll
                for (int j = 0; j < CW; ++j) y[j] = DADD(y[j], v == V - 1 ? hn[j] : Wu.pc[v + 1][j]);
#pragma unroll
                for (int j = 0; j < CW; ++j) y[j] = DADD(y[j], Wu.pn[v][j]);
#pragma unroll
                for (int j = 0; j < CW; ++j) {
                    const int bit = v * CW + j;
                    const double rr = DSUB(bt[v * CW + j], y[j]);
                    const double xn = relax(Wu.xc[v][j], inv, rr, w[t - 1]);
                    fma_sq_if3(j == 0 ? sq0 : sq1, rr, valid ? (accmask >> bit) & 1u : 0u);
                    xin[v][j] = (valid && ((inmask >> bit) & 1u)) ? xn : 0.0;
                }
            }
            acc[t - 1] = DADD(acc[t - 1], DADD(sq0, sq1));
            if (t == H && valid && storemask) {
                double* base = xout + (long long)c * pl;
#pragma unroll
                for (int v = 0; v < V; ++v) {
                    double* row = base + (long long)(gy0 + v) * nx + gx0;
                    const unsigned m2 = (storemask >> (v * CW)) & 3u;
                    if (m2 == 3u)
                        *reinterpret_cast<double2*>(row) = make_double2(xin[v][0], xin[v][1]);
                    else if (m2 == 1u)
                        row[0] = xin[v][0];
                    else if (m2 == 2u)
                        row[1] = xin[v][1];
                }
            }
        }
        __syncthreads();  // edge rows of this step published; ring slot z % D consumed
        if (threadIdx.x == 0 && z + D < nz) tb3_issue<C>(tm_in, tm_b, ox, oy, z + D);
    }
}

template <class C>
__device__ __forceinline__ void tb3_pass(const Tb3Args& a, const CUtensorMap* tm_in,
                                         const CUtensorMap* tm_b, double* xout, int k0, int h,
                                         double (&acc)[C::S], bool accumulate, unsigned ownmask,
                                         uint32_t& ph) {
    for (int q = blockIdx.x; q < a.ntiles; q += gridDim.x) {
        switch (h) {
            case 1: tb3_tile<C, 1>(a, tm_in, tm_b, xout, a.omegas + k0, q, ownmask, accumulate, acc, ph); break;
            case 2: tb3_tile<C, 2>(a, tm_in, tm_b, xout, a.omegas + k0, q, ownmask, accumulate, acc, ph); break;
            default: break;
        }
    }
}

template <class C>
__global__ void __launch_bounds__(C::THREADS, 1) __maxnreg__(C::MAXREG)
    k_tb3d_cycle(const __grid_constant__ CUtensorMap tm_x0, const __grid_constant__ CUtensorMap tm_x1,
                 const __grid_constant__ CUtensorMap tm_b, Tb3Args a) {
    using L = Tb3Layout<C>;
    constexpr int S = C::S;
    // zero edge rows (the rows beyond the first and last warp are never written)
    for (int i = threadIdx.x; i < 2 * S * C::HB; i += blockDim.x) L::top(0, 0)[i] = 0.0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < C::D; ++s) mbar_init(L::bar(s), 1);
        prefetch_tensormap(&tm_x0);
        prefetch_tensormap(&tm_x1);
        prefetch_tensormap(&tm_b);
    }
    __syncthreads();
    unsigned ownmask = 0u;
    {
        const int c0 = (threadIdx.x & 31) * C::CW, r0 = (threadIdx.x >> 5) * C::V;
#pragma unroll
        for (int v = 0; v < C::V; ++v)
#pragma unroll
            for (int j = 0; j < C::CW; ++j)
                if (c0 + j >= S && c0 + j < S + C::TX && r0 + v >= S && r0 + v < S + C::TY)
                    ownmask |= 1u << (v * C::CW + j);
    }
    uint32_t ph = 0;
    const CUtensorMap* const tmx[2] = {&tm_x0, &tm_x1};
    // tiles load their own planes (tile prologue): no speculative first-tile load
    tb_run_cycle<S, F3D, false>(
        a, (int)blockIdx.x < a.ntiles,
        [&](int in, double* xout, int k0, int h, double (&acc)[S], bool accumulate, bool) {
            tb3_pass<C>(a, tmx[in], &tm_b, xout, k0, h, acc, accumulate, ownmask, ph);
        },
        [](int) {}, []() {});
}

// ----------------------------------------------------------------------------
// Host side
// ----------------------------------------------------------------------------

template <class C>
static cudaError_t tb3_plan_variant(Tb3Plan& plan, const Geom& g, int num_sms) {
    cudaError_t e = cudaFuncSetAttribute(k_tb3d_cycle<C>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tb3d_cycle<C>, C::THREADS,
                                                           C::SMEM)) != cudaSuccess)
        return e;
    if (per_sm < 1) return cudaSuccess;
    plan.tiles_x = (g.nx + C::TX - 1) / C::TX;
    plan.ntiles = plan.tiles_x * ((g.ny + C::TY - 1) / C::TY);
    plan.blocks = std::max(1, std::min(num_sms, plan.ntiles));
    plan.sweeps = C::S;
    plan.supported = true;
    return cudaSuccess;
}

cudaError_t tb3_plan_init(Tb3Plan& plan, const Geom& g, int num_sms) {
    plan = Tb3Plan();
    // TMA needs a 16-byte row pitch (even nx).
    if (g.fam != F3D || (g.nx & 1) || !tma_available()) return cudaSuccess;
    plan.variant = 0;
    if (const char* v = getenv("SRJ_TB3_VARIANT")) plan.variant = std::max(0, std::min(2, atoi(v)));
    switch (plan.variant) {
        case 1: return tb3_plan_variant<tb3d::C1>(plan, g, num_sms);
        case 2: return tb3_plan_variant<tb3d::C2>(plan, g, num_sms);
        default: return tb3_plan_variant<tb3d::C0>(plan, g, num_sms);
    }
}

template <class C>
static cudaError_t tb3_launch(const Tb3Plan& plan, const Geom& g, double* x, double* x_alt,
                              const double* b, const double* omegas, int M, double tol,
                              double baseline, double* partials, double* hist, int* out_i,
                              double* out_d, cudaStream_t st) {
    CUtensorMap m0, m1, mb;
    cudaError_t e;
    if ((e = encode_volume_map(&m0, x, g.nx, g.ny, g.nz, C::RX, C::RY)) != cudaSuccess) return e;
    if ((e = encode_volume_map(&m1, x_alt, g.nx, g.ny, g.nz, C::RX, C::RY)) != cudaSuccess) return e;
    if ((e = encode_volume_map(&mb, b, g.nx, g.ny, g.nz, C::RX, C::RY)) != cudaSuccess) return e;
    Tb3Args a;
    a.g = g;
    a.buf0 = x;
    a.buf1 = x_alt;
    a.b = b;
    a.omegas = omegas;
    a.M = M;
    a.s = C::S;
    a.tol = tol;
    a.baseline = baseline;
    a.partials = partials;
    a.hist = hist;
    a.out_i = out_i;
    a.out_d = out_d;
    a.tiles_x = plan.tiles_x;
    a.ntiles = plan.ntiles;
    a.row_lo = 0;
    a.row_hi = g.ny;
    a.sums = nullptr;
    void* args[] = {&m0, &m1, &mb, &a};
    return cudaLaunchCooperativeKernel((const void*)k_tb3d_cycle<C>, dim3(plan.blocks),
                                       dim3(C::THREADS), args, C::SMEM, st);
}

cudaError_t tb3_launch_cycle(const Tb3Plan& plan, const Geom& g, double* x, double* x_alt,
                             const double* b, const double* omegas, int M, double tol,
                             double baseline, double* partials, double* hist, int* out_i,
                             double* out_d, cudaStream_t st) {
    if ((((uintptr_t)x | (uintptr_t)x_alt | (uintptr_t)b) & 15) != 0)
        return cudaErrorMisalignedAddress;
    switch (plan.variant) {
        case 1: return tb3_launch<tb3d::C1>(plan, g, x, x_alt, b, omegas, M, tol, baseline, partials, hist, out_i, out_d, st);
        case 2: return tb3_launch<tb3d::C2>(plan, g, x, x_alt, b, omegas, M, tol, baseline, partials, hist, out_i, out_d, st);
        default: return tb3_launch<tb3d::C0>(plan, g, x, x_alt, b, omegas, M, tol, baseline, partials, hist, out_i, out_d, st);
    }
}

}  // namespace srj
