// Temporally blocked SRJ cycle for the 2D 5-point VARIABLE-coefficient stencil
// (BASELINE config 4: -div(k grad u) = f with harmonic-mean faces): S = 6
// consecutive sweeps, each with its own omega, per HBM round trip.  Measured on
// B200 at 4096^2 (us per sweep): S = 4 55.2, S = 6 49.4, S = 8 57.0.
//
// Same frame as the constant-coefficient kernel (srj_tb.cu): persistent
// cooperative CTAs, 52x36 owned tiles in a 64x48 region (S-wide ring), TMA
// staging with the next tile's boxes loading while the current one computes,
// a split barrier for the halo rows, one grid barrier per pass with the
// fixed-order residual reduction, rollback of a pass that stops inside.
//
// Operator (reference problems.py assembly order; srj_stencil.cuh F2DV):
//   diag = ((c_w + c_e) + c_s) + c_n,   inv = 1 / diag
//   y = 0 + (-c_s) x_s + (-c_w) x_w + diag x + (-c_e) x_e + (-c_n) x_n
// (evaluated without the leading `0 +`: identical bits unless x0 holds -0.0
// entries, see srj_tb.cu)
// with c_w = fx[y][x], c_e = fx[y][x+1], c_s = fy[y][x], c_n = fy[y+1][x].
// A face product belongs to one point pair, so (unlike the constant case) x
// itself is exchanged: west/east by warp shuffle, north/south through the warp
// edge rows.  Per point the thread keeps x, b, c_w, c_s and diag in registers
// (loaded once per tile); c_e is the east point's c_w (own register or one
// shuffle per row per tile), c_n the south face of the row below (own register
// or the next warp's first row, published once per tile).  inv is precomputed
// once per operator (tbv_plan_init) with the reference's division, so it stays
// bit-identical; per tile each thread copies its inv values into a private
// shared-memory slot (the stage is refilled by the next tile's copy) and keeps
// diag in registers, computed once per tile (3 DADD per point per tile instead
// of per sub-sweep).
//
// Staged per tile: x, b, c_w (over the 16-byte-pitch copy of fx), c_s (fy) and
// inv boxes, all RX x RY at the region origin; zero fill outside the grid.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "srj_stencil.cuh"
#include "srj_tb.cuh"
#include "srj_tbdriver.cuh"
#include "srj_tma.cuh"
#include "srj_walk.cuh"

namespace srj {
namespace tbv {

struct Cfg {
    static constexpr int S = 6, CW = 2, V = 6, NSEG = 8;
    static constexpr int RX = 32 * CW, RY = NSEG * V;
    static constexpr int TX = RX - 2 * S, TY = RY - 2 * S;
    static constexpr int THREADS = 32 * NSEG;
    static constexpr int STAGE = RX * RY;          // doubles per staged box
    static constexpr int NST = 5;                  // x, b, c_w, c_s, inv
    static constexpr int HROWS = NSEG + 2;         // edge rows incl. a zero row each side
    static constexpr int HBUF = 2 * HROWS * RX;    // top + bottom rows, one parity
    static constexpr int CSE = HROWS * RX;         // first-row c_s of every warp
    static constexpr size_t SMEM =
        (size_t)(NST * STAGE + 2 * HBUF + 2 * CSE + STAGE) * sizeof(double) + 32;
    static constexpr uint32_t TX_BYTES = NST * STAGE * sizeof(double);
};

}  // namespace tbv

using TbvArgs = TbArgs;


struct TbvMaps {
    CUtensorMap x0, x1, b, fx, fy, inv;
};

extern __shared__ __align__(128) double tbv_smem[];

struct TbvLayout {
    using C = tbv::Cfg;
    static constexpr int ST = 0, H = C::NST * C::STAGE, CSE = H + 2 * C::HBUF, INV = CSE + 2 * C::CSE,
                         BAR = INV + C::STAGE;
    // stages: 0 x, 1 b, 2 c_w, 3 c_s, 4 inv
    __device__ static __forceinline__ double* st(int k) { return tbv_smem + ST + k * C::STAGE; }
    __device__ static __forceinline__ double* top(int t) { return tbv_smem + H + (t & 1) * C::HBUF; }
    __device__ static __forceinline__ double* bot(int t) {
        return tbv_smem + H + (t & 1) * C::HBUF + C::HROWS * C::RX;
    }
    // first-row c_s of every warp, double-buffered by tile parity
    __device__ static __forceinline__ double* cse(int t) { return tbv_smem + CSE + (t & 1) * C::CSE; }
    // the tile's 1/diag, copied out of the stage (thread-private positions)
    __device__ static __forceinline__ double* inv() { return tbv_smem + INV; }
    __device__ static __forceinline__ uint64_t* bar() {
        return reinterpret_cast<uint64_t*>(tbv_smem + BAR);
    }
    __device__ static __forceinline__ uint64_t* hbar(int i) {
        return reinterpret_cast<uint64_t*>(tbv_smem + BAR) + 1 + i;
    }
};

__device__ __forceinline__ void ld2(double (&d)[2], const double* p) {
    SRJ_ASSERT_SMEM(p, 16, tbv_smem);
    const double2 v = *reinterpret_cast<const double2*>(p);
    d[0] = v.x;
    d[1] = v.y;
}
__device__ __forceinline__ void st2(double* p, const double (&d)[2]) {
    SRJ_ASSERT_SMEM(p, 16, tbv_smem);
    *reinterpret_cast<double2*>(p) = make_double2(d[0], d[1]);
}

__device__ __forceinline__ void fma_sq_ifv(double& acc, double r, unsigned cond) {
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p fma.rn.f64 %0, %1, %1, %0;\n\t}"
        : "+d"(acc)
        : "d"(r), "r"(cond));
}

template <bool SLAB>
__device__ __forceinline__ void tbv_issue(const TbvArgs& a, const CUtensorMap* tm_in,
                                          const TbvMaps& m, int q) {
    using C = tbv::Cfg;
    using L = TbvLayout;
    const int ox = (q % a.tiles_x) * C::TX - C::S,
              oy = (SLAB ? a.row_lo : 0) + (q / a.tiles_x) * C::TY - C::S;
    fence_proxy_async();
    mbar_expect_tx(L::bar(), C::TX_BYTES);
    tma_load_2d(L::st(0), tm_in, ox, oy, L::bar());
    tma_load_2d(L::st(1), &m.b, ox, oy, L::bar());
    tma_load_2d(L::st(2), &m.fx, ox, oy, L::bar());
    tma_load_2d(L::st(3), &m.fy, ox, oy, L::bar());
    tma_load_2d(L::st(4), &m.inv, ox, oy, L::bar());
}

struct TbvRegs {
    using C = tbv::Cfg;
    double x[C::V][C::CW], b[C::V][C::CW];
    double cw[C::V][C::CW], cs[C::V][C::CW], dg[C::V][C::CW];  // dg: diagonal
    double ce[C::V];   // east face of column CW-1 (= next lane's c_w of column 0)
    double cn[C::CW];  // north face of row V-1 (= next warp's c_s of row 0)
};

template <int H, bool MASKED>
__device__ __forceinline__ void tbv_sweeps(TbvRegs& R, const double* omegas, int warp, int lane,
                                           unsigned inmask, unsigned accmask,
                                           double (&acc)[tbv::Cfg::S], uint32_t& na, uint32_t hb) {
    using C = tbv::Cfg;
    using L = TbvLayout;
    constexpr int V = C::V, CW = C::CW, RX = C::RX;
    // ring and tile aligned to warps and lanes: a thread owns all of its
    // points or none (see srj_tb.cu), so unmasked tiles select once per sub-sweep
    constexpr bool kAligned = C::S % V == 0 && C::TY % V == 0 && C::S % CW == 0 &&
                              C::TX % CW == 0;
    const int col = lane * CW;
#pragma unroll
    for (int t = 0; t < H; ++t) {
        const double w = __ldg(omegas + t);
        double sq[2] = {0.0, 0.0};
        // In-place row updates: a row's west/east neighbours are shuffled just
        // before the row is rewritten (the warp moves in lockstep, so they are
        // old values); old copies are kept only where a later row needs them.
        double old_up[CW];                 // old x of the row above the current one
        double old_r1[CW], old_rl[CW];     // old rows 1 and V-2 (for the edge rows)
        auto row = [&](int v, const double (&xs)[CW], const double (&xn)[CW]) {
            const double xw = shfl_up_d(R.x[v][CW - 1], 1);
            const double xe = shfl_down_d(R.x[v][0], 1);
            double iv[CW];
            ld2(iv, L::inv() + (warp * V + v) * RX + col);
            double xo[CW];
#pragma unroll
            for (int j = 0; j < CW; ++j) {
                const double c_w = R.cw[v][j];
                const double c_e = j == CW - 1 ? R.ce[v] : R.cw[v][j + 1];
                const double c_s = R.cs[v][j];
                const double c_n = v == V - 1 ? R.cn[j] : R.cs[v + 1][j];
                const double diag = R.dg[v][j];
                const double x_w = j == 0 ? xw : R.x[v][j - 1];
                const double x_e = j == CW - 1 ? xe : R.x[v][j + 1];
                double y = DMUL(-c_s, xs[j]);  // 0 + (-c_s) x_s (see header)
                y = DADD(y, DMUL(-c_w, x_w));
                y = DADD(y, DMUL(diag, R.x[v][j]));
                y = DADD(y, DMUL(-c_e, x_e));
                y = DADD(y, DMUL(-c_n, xn[j]));
                const double rr = DSUB(R.b[v][j], y);
                const double xnew = relax(R.x[v][j], iv[j], rr, w);
                const int bit = v * CW + j;
                if constexpr (!MASKED && kAligned)
                    sq[j] = fma(rr, rr, sq[j]);  // owned: decided per thread below
                else
                    fma_sq_ifv(sq[j], rr, (accmask >> bit) & 1u);
                xo[j] = (!MASKED || ((inmask >> bit) & 1u)) ? xnew : 0.0;
            }
#pragma unroll
            for (int j = 0; j < CW; ++j) R.x[v][j] = xo[j];
        };
        // interior rows 1 .. V-2, top to bottom (row 0 is still old)
#pragma unroll
        for (int j = 0; j < CW; ++j) old_up[j] = R.x[0][j];
#pragma unroll
        for (int v = 1; v < V - 1; ++v) {
            double cur[CW];
#pragma unroll
            for (int j = 0; j < CW; ++j) cur[j] = R.x[v][j];
            if (v == 1) {
#pragma unroll
                for (int j = 0; j < CW; ++j) old_r1[j] = cur[j];
            }
            if (v == V - 2) {
#pragma unroll
                for (int j = 0; j < CW; ++j) old_rl[j] = cur[j];
            }
            row(v, old_up, R.x[v + 1]);
#pragma unroll
            for (int j = 0; j < CW; ++j) old_up[j] = cur[j];
        }
        if (t > 0) {  // edge rows of sub-sweep t were published by every warp
            mbar_wait(L::hbar(na & 1), (na >> 1) & 1);
            ++na;
        }
        double hs[CW], hn[CW];  // x of the rows above / below this warp's rows
        ld2(hs, L::bot(hb + t) + warp * RX + col);        // bottom row of warp-1
        ld2(hn, L::top(hb + t) + (warp + 2) * RX + col);  // top row of warp+1
        row(0, hs, old_r1);
        row(V - 1, old_rl, hn);
        if constexpr (!MASKED && kAligned)
            acc[t] = accmask != 0u ? DADD(acc[t], DADD(sq[0], sq[1])) : acc[t];
        else
            acc[t] = DADD(acc[t], DADD(sq[0], sq[1]));
        if (t + 1 < H) {
            st2(L::top(hb + t + 1) + (warp + 1) * RX + col, R.x[0]);
            st2(L::bot(hb + t + 1) + (warp + 1) * RX + col, R.x[V - 1]);
            __syncwarp();
            if (lane == 0) mbar_arrive(L::hbar(na & 1));
        }
    }
}

template <bool MASKED>
__device__ __forceinline__ void tbv_dispatch(int h, TbvRegs& R, const double* omegas, int warp,
                                             int lane, unsigned inmask, unsigned accmask,
                                             double (&acc)[tbv::Cfg::S], uint32_t& na,
                                             uint32_t hb) {
    switch (h) {
        case 1: tbv_sweeps<1, MASKED>(R, omegas, warp, lane, inmask, accmask, acc, na, hb); break;
        case 2: tbv_sweeps<2, MASKED>(R, omegas, warp, lane, inmask, accmask, acc, na, hb); break;
        case 3: tbv_sweeps<3, MASKED>(R, omegas, warp, lane, inmask, accmask, acc, na, hb); break;
        case 4: tbv_sweeps<4, MASKED>(R, omegas, warp, lane, inmask, accmask, acc, na, hb); break;
        case 5: tbv_sweeps<5, MASKED>(R, omegas, warp, lane, inmask, accmask, acc, na, hb); break;
        case 6: tbv_sweeps<6, MASKED>(R, omegas, warp, lane, inmask, accmask, acc, na, hb); break;
        default: break;
    }
}

template <bool SLAB>
__device__ __forceinline__ void tbv_pass(const TbvArgs& a, const CUtensorMap* tm_in,
                                         const TbvMaps& m, double* __restrict__ xout, const double* om,
                                         int h, double (&acc)[tbv::Cfg::S], bool accumulate,
                                         unsigned ownmask, uint32_t& phase, bool first_issued,
                                         uint32_t& na, uint32_t& hb) {
    using C = tbv::Cfg;
    using L = TbvLayout;
    constexpr int S = C::S, V = C::V, CW = C::CW, RX = C::RX;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c0 = lane * CW, r0 = warp * V;
    const int nx = a.g.nx, ny = a.g.ny;
    if ((int)blockIdx.x >= a.ntiles) return;
    if (threadIdx.x == 0 && !first_issued) tbv_issue<SLAB>(a, tm_in, m, blockIdx.x);
    for (int q = blockIdx.x; q < a.ntiles; q += gridDim.x) {
        const int ox = (q % a.tiles_x) * C::TX, oy = (SLAB ? a.row_lo : 0) + (q / a.tiles_x) * C::TY;
        const int gx0 = ox - S + c0;
        const int gy0 = oy - S + r0;
        // slab: a tile crossing row_hi reaches into ghost rows (updated, not owned)
        const bool crosses = SLAB && oy + C::TY > a.row_hi;
        const bool masked = ox < S || oy < S || ox + C::TX + S > nx || oy + C::TY + S > ny ||
                            crosses;
        unsigned inmask = 0xffffffffu;
        unsigned storemask = ownmask;
        if (masked) {
            inmask = 0u;
#pragma unroll
            for (int v = 0; v < V; ++v)
#pragma unroll
                for (int j = 0; j < CW; ++j)
                    if (gy0 + v >= 0 && gy0 + v < ny && gx0 + j >= 0 && gx0 + j < nx)
                        inmask |= 1u << (v * CW + j);
            storemask &= inmask;
            if (crosses) {  // rows >= row_hi are ghost rows: updated, not owned
#pragma unroll
                for (int v = 0; v < V; ++v)
                    if (gy0 + v >= a.row_hi) storemask &= ~(((1u << CW) - 1u) << (v * CW));
            }
        }
        const unsigned accmask = accumulate ? storemask : 0u;
        mbar_wait(L::bar(), phase);
        phase ^= 1u;
        TbvRegs R;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            const int o = (r0 + v) * RX + c0;
            ld2(R.x[v], L::st(0) + o);
            ld2(R.b[v], L::st(1) + o);
            ld2(R.cw[v], L::st(2) + o);
            ld2(R.cs[v], L::st(3) + o);
            double iv[CW];
            ld2(iv, L::st(4) + o);
            st2(L::inv() + o, iv);
        }
        st2(L::top(hb) + (warp + 1) * RX + c0, R.x[0]);
        st2(L::bot(hb) + (warp + 1) * RX + c0, R.x[V - 1]);
        st2(L::cse(q / (int)gridDim.x) + (warp + 1) * RX + c0, R.cs[0]);
#pragma unroll
        for (int v = 0; v < V; ++v) R.ce[v] = __shfl_down_sync(0xffffffffu, R.cw[v][0], 1);
        __syncthreads();  // stages consumed, edge rows published
        ld2(R.cn, L::cse(q / (int)gridDim.x) + (warp + 2) * RX + c0);
        // diagonal once per tile (reference assembly order)
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
            for (int j = 0; j < CW; ++j) {
                const double c_e = j == CW - 1 ? R.ce[v] : R.cw[v][j + 1];
                const double c_n = v == V - 1 ? R.cn[j] : R.cs[v + 1][j];
                R.dg[v][j] = DADD(DADD(DADD(R.cw[v][j], c_e), R.cs[v][j]), c_n);
            }
        if (threadIdx.x == 0 && q + (int)gridDim.x < a.ntiles)
            tbv_issue<SLAB>(a, tm_in, m, q + gridDim.x);
        if (masked)
            tbv_dispatch<true>(h, R, om, warp, lane, inmask, accmask, acc, na, hb);
        else
            tbv_dispatch<false>(h, R, om, warp, lane, inmask, accmask, acc, na, hb);
        hb += h;  // the next tile publishes into the parity after this tile's last
        if (storemask) {
#pragma unroll
            for (int v = 0; v < V; ++v) {
                double* row = xout + (long long)(gy0 + v) * nx + gx0;
                // a lane's column pair is owned / inside the grid as a whole
                // (even nx, even ring and tile widths): one predicated store
                if ((storemask >> (v * CW)) & 1u) {
                    SRJ_ASSERT(gy0 + v >= (SLAB ? a.row_lo : 0) && gy0 + v < (SLAB ? a.row_hi : ny) &&
                               gx0 >= 0 && gx0 + 1 < nx);
                    *reinterpret_cast<double2*>(row) = make_double2(R.x[v][0], R.x[v][1]);
                }
            }
        }
        // No barrier here: the halo parity runs on across tiles (hb) and the
        // first-row faces alternate by tile (see srj_tb.cu tb2d_pass).
    }
}

template <bool SLAB, bool SOLVE>
__global__ void __launch_bounds__(tbv::Cfg::THREADS, 1)
    k_tbvar_cycle(const __grid_constant__ TbvMaps m, TbvArgs a) {
    using C = tbv::Cfg;
    using L = TbvLayout;
    constexpr int S = C::S;
    for (int i = threadIdx.x; i < 2 * C::HBUF + 2 * C::CSE; i += blockDim.x) L::top(0)[i] = 0.0;
    if (threadIdx.x == 0) {
        mbar_init(L::bar(), 1);
        mbar_init(L::hbar(0), C::NSEG);
        mbar_init(L::hbar(1), C::NSEG);
        prefetch_tensormap(&m.x0);
        prefetch_tensormap(&m.x1);
        prefetch_tensormap(&m.b);
        prefetch_tensormap(&m.fx);
        prefetch_tensormap(&m.fy);
        prefetch_tensormap(&m.inv);
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
    uint32_t phase = 0, na = 0, hb = 0;
    const CUtensorMap* const tmx[2] = {&m.x0, &m.x1};
    auto pass = [&](int in, double* xout, const double* om, int h, double (&acc)[S],
                    bool accumulate, bool first) __attribute__((always_inline)) {
        tbv_pass<SLAB>(a, tmx[in], m, xout, om, h, acc, accumulate, ownmask, phase, first, na, hb);
    };
    auto issue = [&](int in) {  // a lane of the last warp (it has no part in the pass sums)
        if (threadIdx.x == blockDim.x - 32) tbv_issue<SLAB>(a, tmx[in], m, blockIdx.x);
    };
    auto drain = [&]() __attribute__((always_inline)) {
        mbar_wait(L::bar(), phase);
        phase ^= 1u;
    };
    if constexpr (SOLVE)
        tb_run_solve<S, F2DV>(a, (int)blockIdx.x < a.ntiles, pass, issue, drain);
    else
        tb_run_cycle<S, F2DV, SLAB>(a, (int)blockIdx.x < a.ntiles, pass, issue, drain);
}

// inv[p] = 1 / (((c_w + c_e) + c_s) + c_n), the reference's diagonal and
// SparseMatrix's cached reciprocal (srj_stencil.cuh F2DV, sparse.py:44).
__global__ void k_tbv_inv(const double* __restrict__ fx, const double* __restrict__ fy,
                          double* __restrict__ inv, int nx, int ny) {
    const long long n = (long long)nx * ny;
    for (long long p = blockIdx.x * (long long)blockDim.x + threadIdx.x; p < n;
         p += (long long)gridDim.x * blockDim.x) {
        const long long y = p / nx, x = p % nx;
        const double cw = fx[y * (nx + 1) + x], ce = fx[y * (nx + 1) + x + 1];
        const double cs = fy[y * nx + x], cn = fy[(y + 1) * nx + x];
        inv[p] = __ddiv_rn(1.0, DADD(DADD(DADD(cw, ce), cs), cn));
    }
}

// ----------------------------------------------------------------------------
// Host side
// ----------------------------------------------------------------------------

cudaError_t tbv_plan_init(TbvPlan& plan, const Geom& g, int num_sms) {
    using C = tbv::Cfg;
    plan = TbvPlan();
    // TMA needs 16-byte row pitches: even nx (x, b, fy, inv; fx via a padded copy).
    if (g.fam != F2DV || (g.nx & 1) || !g.fx || !g.fy || !tma_available()) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(k_tbvar_cycle<false, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_tbvar_cycle<true, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_tbvar_cycle<false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tbvar_cycle<false, false>,
                                                           C::THREADS, C::SMEM)) != cudaSuccess)
        return e;
    if (per_sm < 1) return cudaSuccess;
    const size_t n = (size_t)g.nx * g.ny;
    plan.fx_pitch = g.nx + 2;
    if ((e = cudaMalloc(&plan.fx_pad, (size_t)plan.fx_pitch * g.ny * sizeof(double))) != cudaSuccess)
        return e;
    if ((e = cudaMemcpy2D(plan.fx_pad, plan.fx_pitch * sizeof(double), g.fx,
                          (size_t)(g.nx + 1) * sizeof(double), (size_t)(g.nx + 1) * sizeof(double),
                          g.ny, cudaMemcpyDeviceToDevice)) != cudaSuccess)
        return e;
    if ((e = cudaMalloc(&plan.inv, n * sizeof(double))) != cudaSuccess) return e;
    k_tbv_inv<<<4 * num_sms, 256>>>(g.fx, g.fy, plan.inv, g.nx, g.ny);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if ((e = cudaDeviceSynchronize()) != cudaSuccess) return e;
    plan.tiles_x = (g.nx + C::TX - 1) / C::TX;
    plan.ntiles = plan.tiles_x * ((g.ny + C::TY - 1) / C::TY);
    plan.blocks = std::max(1, std::min(num_sms, plan.ntiles));
    plan.supported = true;
    return cudaSuccess;
}

void tbv_plan_free(TbvPlan& plan) {
    if (plan.fx_pad) cudaFree(plan.fx_pad);
    if (plan.inv) cudaFree(plan.inv);
    plan.fx_pad = nullptr;
    plan.inv = nullptr;
}

cudaError_t tbv_launch_cycle(const TbvPlan& plan, const Geom& g, double* x, double* x_alt,
                             const double* b, const double* omegas, int M, int s, double tol,
                             double baseline, double* partials, double* hist, int* out_i,
                             double* out_d, cudaStream_t st, int row_lo, int row_hi,
                             double* sums, const SolveCtl* ctl) {
    using C = tbv::Cfg;
    if ((((uintptr_t)x | (uintptr_t)x_alt | (uintptr_t)b) & 15) != 0)
        return cudaErrorMisalignedAddress;
    TbvMaps m;
    cudaError_t e;
    if ((e = encode_field_map(&m.x0, x, g.nx, g.ny, C::RX, C::RY)) != cudaSuccess) return e;
    if ((e = encode_field_map(&m.x1, x_alt, g.nx, g.ny, C::RX, C::RY)) != cudaSuccess) return e;
    if ((e = encode_field_map(&m.b, b, g.nx, g.ny, C::RX, C::RY)) != cudaSuccess) return e;
    if ((e = encode_field_map_pitched(&m.fx, plan.fx_pad, g.nx + 1, g.ny, plan.fx_pitch, C::RX,
                                      C::RY)) != cudaSuccess)
        return e;
    if ((e = encode_field_map(&m.fy, g.fy, g.nx, g.ny + 1, C::RX, C::RY)) != cudaSuccess) return e;
    if ((e = encode_field_map(&m.inv, plan.inv, g.nx, g.ny, C::RX, C::RY)) != cudaSuccess) return e;
    TbvArgs a;
    a.ctl = ctl ? *ctl : SolveCtl{};
    a.g = g;
    a.buf0 = x;
    a.buf1 = x_alt;
    a.b = b;
    a.omegas = omegas;
    a.M = M;
    a.s = std::max(1, std::min(s, C::S));
    a.tol = tol;
    a.baseline = baseline;
    a.partials = partials;
    a.hist = hist;
    a.out_i = out_i;
    a.out_d = out_d;
    a.row_lo = row_lo;
    a.row_hi = row_hi;
    a.sums = sums;
    a.tiles_x = plan.tiles_x;
    a.ntiles = a.tiles_x * ((row_hi - row_lo + C::TY - 1) / C::TY);
    const int blocks = std::max(1, std::min(plan.blocks - plan.reserved, a.ntiles));
    void* args[] = {&m, &a};
    const void* kern = sums != nullptr ? (const void*)k_tbvar_cycle<true, false>
                       : ctl            ? (const void*)k_tbvar_cycle<false, true>
                                        : (const void*)k_tbvar_cycle<false, false>;
    return cudaLaunchCooperativeKernel(kern, dim3(blocks), dim3(C::THREADS), args, C::SMEM, st);
}

}  // namespace srj
