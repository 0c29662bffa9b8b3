// Temporally blocked SRJ cycle for the 2D 5-point constant-coefficient
// stencil (BASELINE config 2): up to S consecutive sweeps (S = 6 ring by
// default, S = 4 for <= 4 sweeps per pass), each with its own omega, per
// HBM/L2 round trip of x and b.
//
// Tiling.  A CTA (one per SM, persistent, cooperative launch) owns TX x TY
// output tiles.  For each tile the copy engine (TMA) brings the RX x RY region
// (the tile plus an S-wide ring) of x_{k0} and b into shared memory; boxes that
// stick out of the grid are zero-filled, which is the Dirichlet ghost.  Both
// are moved into registers at once, and the next tile's boxes are loaded
// into the same stage while the current tile computes.
//
// Register tiling.  Warp w owns rows [w*V, w*V+V) of the region; lane l owns
// columns [l*CW, l*CW+CW) of them.  x, b and p = c_off*x of those CW*V points
// live in registers for all S sub-sweeps.  Neighbours:
//   west/east  -- registers, or a warp shuffle across the lane boundary;
//   north/south -- registers, or the halo rows the warps above/below publish
//                  in shared memory (double-buffered by a halo parity that
//                  runs on across tiles; a split mbarrier per sub-sweep:
//                  interior rows are computed between a warp's arrival and
//                  its wait).
// No block-wide barrier inside a pass: a tile's first halo rows are one more
// hand-off round, and a "stage consumed" mbarrier (one arrival per warp) tells
// warp 0 when the next tile's copy may overwrite the stage.
// Measured on B200 (tools/probe/rates_probe.cu): a 64-bit warp shuffle costs
// ~1/3 of the shared-memory bandwidth an LDS.64 exchange needs, so the only
// shared traffic left is the staging load and the halo rows.
//
// Shared products.  With constant coefficients the rounded product
// p_j = c_off*x_j is the same value for all four points that have x_j as a
// neighbour, so it is computed once per point and sub-sweep:
//     y = ((((0 + p_s) + p_w) + c_diag*x) + p_e) + p_n
// is bit-identical to the reference csr_matvec order with freshly rounded
// products; 11 fp64 instructions per point-sweep.  The leading `0 +` is
// dropped (10 instructions): 0 + p_s and p_s differ only when p_s = -0, and
// that sign of zero can reach the result only through c_diag*x = -0, i.e.
// x = -0 at the point.  Iterates never create a -0 (x + t rounds an exact
// zero to +0; held and ghost points are +0), so the iterates are bit-identical
// unless x0 itself holds -0.0 entries -- then at most the sign of a zero can
// differ (equal values).
// The diagonal term reuses the shared product too: c_diag = -4*c_off exactly
// (tb_plan_init checks it), and scaling by 4 is exact, so
// rn(c_diag*x) = -4*rn(c_off*x) = -4*p and y + c_diag*x is one FMA,
// fma(p, -4, y) = rn(y - 4p), whose product is exact: 9 fp64 instructions
// per point-sweep.  (The identity needs rn(c_off*x) to be a normal number or
// zero, i.e. |x| >= 2^-1022/dx2 or x = 0; iterates of a solve are never that
// small without being exactly zero.)
//
// Every region point is updated every sub-sweep; values within t+1 rings of
// the region edge are garbage after sub-sweep t but never reach the owned tile,
// which after h <= S sub-sweeps holds x_{k0+h} exactly (bit-identical
// iterates).  Grid-exterior points are held at 0.
//
// Residuals.  Sub-sweep t accumulates (b - A x_{k0+t})^2 over OWNED points
// only; the per-cycle driver (srj_tbdriver.cuh) reduces them after each pass,
// applies the reference's per-sweep stopping rule (solver.py:216-222,235-239)
// and rolls back a pass that stops inside.  The SLAB instantiation serves
// srj_tb_pass: tiles cover the owned rows [row_lo, row_hi) of a row slab
// whose deep ghost rows are updated as ring points but never stored.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "srj_stencil.cuh"
#include "srj_tb.cuh"
#include "srj_tbdriver.cuh"
#include "srj_tma.cuh"
#include "srj_walk.cuh"

namespace srj {
namespace tb2d {

template <int S_, int CW_, int V_, int NSEG_>
struct CfgBase {
    static constexpr int S = S_;        // sweeps fused per pass (= ring width)
    static constexpr int CW = CW_;      // columns per lane
    static constexpr int V = V_;        // rows per warp
    static constexpr int NSEG = NSEG_;  // warps
    static constexpr int RX = 32 * CW, RY = NSEG * V;
    static constexpr int TX = RX - 2 * S, TY = RY - 2 * S;
    static_assert(CW * V <= 32, "point masks are 32-bit");
    static_assert(TX % 2 == 0, "tile origins must stay 16-byte aligned for TMA");
    static constexpr int THREADS = 32 * NSEG;
    // Registers are allocated per SM sub-partition (16K each, 4 per SM): with
    // W warps, ceil(W/4) warps share one.
    static constexpr int WARPS_PER_SMSP = (NSEG + 3) / 4;
    static constexpr int MAXREG_RAW = (16384 / (WARPS_PER_SMSP * 32)) / 8 * 8;
    static constexpr int MAXREG = MAXREG_RAW > 255 ? 255 : MAXREG_RAW;
    static constexpr int STAGE = RX * RY;          // doubles per staged box
    static constexpr int HROWS = NSEG + 2;         // halo rows incl. a zero row each side
    static constexpr int HBUF = 2 * HROWS * RX;    // top + bottom rows, one parity
    // x stage, b stage, halo rows [2 parities], TMA + 2 halo mbarriers
    static constexpr size_t SMEM = (size_t)(2 * STAGE + 2 * HBUF) * sizeof(double) + 32;
    static constexpr uint32_t TX_BYTES = 2u * STAGE * sizeof(double);
};

// Kernel variants: K -> (S, columns per lane, rows per warp, warps).
template <int K>
struct Cfg;
template <>
struct Cfg<0> : CfgBase<4, 2, 6, 12> {};  // 64x72 region, 56x64 tile, 384 threads
template <>
struct Cfg<1> : CfgBase<6, 2, 6, 12> {};  // 64x72 region, 52x60 tile, 384 threads (S = 6)
// The variant follows the requested sweeps per pass: s <= 4 -> K=0, s = 5, 6
// -> K=1.  Measured on B200 (2048^2 / 4096^2, us per sweep): K=0 at s=4 9.4 /
// 33.5, K=1 at s=6 9.2 / 30.7; an S=8 ring (48x56 tiles) 9.8 / 34.7 at s=8,
// 8 warps x 9 rows at S=4 9.7 / 35.0; 16-warp 64x96 and 18-warp 64x72 shapes
// spill (10.9 / 38.4), 64x128 spills heavily (15.7), 4 columns per lane
// (128x72) spills (15.0).
constexpr int kVariants = 2;

}  // namespace tb2d


// Dynamic shared memory, indexed with compile-time offsets so every access
// compiles to LDS/STS (a pointer carried through a struct loses the address
// space and becomes a generic LD/ST).
extern __shared__ __align__(128) double tb_smem[];

template <int K>
struct TbLayout {
    using C = tb2d::Cfg<K>;
    static constexpr int STX = 0, STB = C::STAGE, H = 2 * C::STAGE, BAR = H + 2 * C::HBUF;
    __device__ static __forceinline__ double* stx() { return tb_smem + STX; }
    __device__ static __forceinline__ double* stb() { return tb_smem + STB; }
    // halo rows of parity t: top rows then bottom rows, row index = warp + 1
    __device__ static __forceinline__ double* top(int t) { return tb_smem + H + (t & 1) * C::HBUF; }
    __device__ static __forceinline__ double* bot(int t) {
        return tb_smem + H + (t & 1) * C::HBUF + C::HROWS * C::RX;
    }
    __device__ static __forceinline__ uint64_t* bar() {
        return reinterpret_cast<uint64_t*>(tb_smem + BAR);
    }
    // halo hand-off barriers [2] (one arrival per warp)
    __device__ static __forceinline__ uint64_t* hbar(int i) {
        return reinterpret_cast<uint64_t*>(tb_smem + BAR) + 1 + i;
    }
    // stage consumed (one arrival per warp): the next tile's copy may start
    __device__ static __forceinline__ uint64_t* sempty() {
        return reinterpret_cast<uint64_t*>(tb_smem + BAR) + 3;
    }
};

// CW contiguous doubles at a 16-byte aligned shared address.
template <int CW>
__device__ __forceinline__ void lds_cols(double (&d)[CW], const double* p) {
    SRJ_ASSERT_SMEM(p, CW * sizeof(double), tb_smem);
#pragma unroll
    for (int j = 0; j < CW; j += 2) {
        const double2 v = *reinterpret_cast<const double2*>(p + j);
        d[j] = v.x;
        d[j + 1] = v.y;
    }
}
template <int CW>
__device__ __forceinline__ void sts_cols(double* p, const double (&d)[CW]) {
    SRJ_ASSERT_SMEM(p, CW * sizeof(double), tb_smem);
#pragma unroll
    for (int j = 0; j < CW; j += 2) *reinterpret_cast<double2*>(p + j) = make_double2(d[j], d[j + 1]);
}

template <int K, bool SLAB>
__device__ __forceinline__ void tb2d_issue(const TbArgs& a, const CUtensorMap* tm_in,
                                           const CUtensorMap* tm_b, int q) {
    using C = tb2d::Cfg<K>;
    using L = TbLayout<K>;
    constexpr int S = C::S;
    const int ox = (q % a.tiles_x) * C::TX, oy = (SLAB ? a.row_lo : 0) + (q / a.tiles_x) * C::TY;
    fence_proxy_async();
    mbar_expect_tx(L::bar(), C::TX_BYTES);
    tma_load_2d(L::stx(), tm_in, ox - S, oy - S, L::bar());
    tma_load_2d(L::stb(), tm_b, ox - S, oy - S, L::bar());
}

// acc += r*r when cond != 0, as one predicated DFMA (a C++ conditional
// becomes a DFMA plus two FSELs).
__device__ __forceinline__ void fma_sq_if(double& acc, double r, unsigned cond) {
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p fma.rn.f64 %0, %1, %1, %0;\n\t}"
        : "+d"(acc)
        : "d"(r), "r"(cond));
}

#ifdef SRJ_STRESS
// Negative control of the stress build: SRJ_STRESS_BREAK=1 in the environment
// skips the halo hand-off wait, a deliberate race the stress parity tests must
// catch (tests/test_gpu_stress.py).
__device__ int tb_stress_break = 0;
#endif

template <int K>
struct TileRegs {
    using C = tb2d::Cfg<K>;
    double x[C::V][C::CW], p[C::V][C::CW], b[C::V][C::CW];
};

// H sub-sweeps (compile-time, H <= S) of the tile held in registers.  MASKED
// tiles reach outside the grid: points there (bit clear in `inmask`, bit
// v*CW+j) are held at 0.  Points with a bit set in `accmask` add r^2 to acc[t].
//
// Halo hand-off between sub-sweeps is a split barrier: after publishing its
// edge rows a warp arrives on mbarrier `na & 1` (one elected lane per warp),
// computes its interior rows -- which need no halo -- and only then waits for
// the other warps' arrivals before its two edge rows.  `na` counts arrival
// rounds (identical in every thread).
template <int K, int H, bool MASKED>
__device__ __forceinline__ void tile_sweeps(TileRegs<K>& R, const double* omegas, const Geom& g,
                                            int warp, int lane, unsigned inmask, unsigned accmask,
                                            double (&acc)[tb2d::Cfg<K>::S], uint32_t& na,
                                            uint32_t hb) {
    using C = tb2d::Cfg<K>;
    using L = TbLayout<K>;
    constexpr int V = C::V, CW = C::CW, RX = C::RX;
    static_assert(V >= 3 && CW == 2, "row-pair groups of a 2-column lane");
    // Ring and tile aligned to warps (rows) and lanes (columns): a thread owns
    // all of its points or none, so unmasked tiles accumulate r^2
    // unconditionally and select once per sub-sweep (S = 6 ring with 6 rows
    // per warp: warps 0 and NSEG-1 own nothing, lanes 0-2 and 29-31 own nothing).
    constexpr bool kAligned = C::S % V == 0 && C::TY % V == 0 && C::S % CW == 0 &&
                              C::TX % CW == 0;
    const double coff = g.c_off, inv = g.inv_diag;
    const int col = lane * CW;
#pragma unroll
    for (int t = 0; t < H; ++t) {
        const double w = __ldg(omegas + t);
        double pw[V], pe[V];  // p across the lane boundary
#pragma unroll
        for (int v = 0; v < V; ++v) {
            pw[v] = shfl_up_d(R.p[v][CW - 1], 1);
            pe[v] = shfl_down_d(R.p[v][0], 1);
        }
        double hs[CW], hn[CW];  // p of the rows above / below this warp's rows
        double sq[4] = {0.0, 0.0, 0.0, 0.0};  // r^2 partial sums, one per group slot
        // Up to four rows (-1: unused), both columns, computed in lockstep so
        // the independent dependency chains interleave (fp64 latency ~9 clk on
        // B200): the four interior rows as one group of 8 chains (2048^2 sweep
        // 8.11 -> 7.96 us vs two groups of 4), then the two edge rows after the
        // halo hand-off.  Neighbours are the OLD p (updated after all rows).
        auto group = [&](int va, int vb, int vc, int vd) {
            constexpr int NP = 8;
            const int rows[4] = {va, vb, vc, vd};
            const int np = vd >= 0 ? 8 : vc >= 0 ? 6 : vb >= 0 ? 4 : 2;
            double y[NP], rr[NP];
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                if (k >= np) break;
                const int v = rows[k >> 1], j = k & 1;
                y[k] = v == 0 ? hs[j] : R.p[v - 1][j];  // 0 + p_s (see header)
            }
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                if (k >= np) break;
                const int v = rows[k >> 1], j = k & 1;
                y[k] = DADD(y[k], j == 0 ? pw[v] : R.p[v][j - 1]);
            }
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                if (k >= np) break;
                const int v = rows[k >> 1], j = k & 1;
                y[k] = __fma_rn(R.p[v][j], -4.0, y[k]);  // + c_diag*x = -4*p (see header)
            }
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                if (k >= np) break;
                const int v = rows[k >> 1], j = k & 1;
                y[k] = DADD(y[k], j == CW - 1 ? pe[v] : R.p[v][j + 1]);
            }
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                if (k >= np) break;
                const int v = rows[k >> 1], j = k & 1;
                y[k] = DADD(y[k], v == V - 1 ? hn[j] : R.p[v + 1][j]);
            }
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                if (k >= np) break;
                const int v = rows[k >> 1], j = k & 1;
                rr[k] = DSUB(R.b[v][j], y[k]);
            }
#pragma unroll
            for (int k = 0; k < NP; ++k) {
                if (k >= np) break;
                const int v = rows[k >> 1], j = k & 1;
                const int bit = v * CW + j;
                const double xn = relax(R.x[v][j], inv, rr[k], w);
                if constexpr (!MASKED && kAligned)
                    sq[k & 3] = fma(rr[k], rr[k], sq[k & 3]);  // owned: decided per thread below
                else
                    fma_sq_if(sq[k & 3], rr[k], (accmask >> bit) & 1u);
                R.x[v][j] = (!MASKED || ((inmask >> bit) & 1u)) ? xn : 0.0;
            }
        };
        static_assert(V == 6, "interior rows 1..4 form one group");
        group(1, 2, 3, 4);
        {  // halos of sub-sweep t were published by every warp (t = 0: at tile start)
#ifdef SRJ_STRESS
            if (!tb_stress_break)
#endif
                mbar_wait(L::hbar(na & 1), (na >> 1) & 1);
            ++na;
        }
        lds_cols<CW>(hs, L::bot(hb + t) + warp * RX + col);        // bottom row of warp-1
        lds_cols<CW>(hn, L::top(hb + t) + (warp + 2) * RX + col);  // top row of warp+1
        group(0, V - 1, -1, -1);
        if constexpr (!MASKED && kAligned)
            acc[t] = accmask != 0u ? DADD(acc[t], DADD(DADD(sq[0], sq[1]), DADD(sq[2], sq[3])))
                                   : acc[t];
        else
            acc[t] = DADD(acc[t], DADD(DADD(sq[0], sq[1]), DADD(sq[2], sq[3])));
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
            for (int j = 0; j < CW; ++j) R.p[v][j] = DMUL(coff, R.x[v][j]);
        if (t + 1 < H) {
            sts_cols<CW>(L::top(hb + t + 1) + (warp + 1) * RX + col, R.p[0]);
            sts_cols<CW>(L::bot(hb + t + 1) + (warp + 1) * RX + col, R.p[V - 1]);
            __syncwarp();
            if (lane == 0) mbar_arrive(L::hbar(na & 1));
        }
    }
}

template <int K, bool MASKED>
__device__ __forceinline__ void tile_dispatch(int h, TileRegs<K>& R, const double* omegas,
                                              const Geom& g, int warp, int lane, unsigned inmask,
                                              unsigned accmask, double (&acc)[tb2d::Cfg<K>::S],
                                              uint32_t& na, uint32_t hb) {
    constexpr int S = tb2d::Cfg<K>::S;
#define SRJ_TB_CASE(H)                                                                      \
    case H:                                                                                 \
        if constexpr (H <= S)                                                               \
            tile_sweeps<K, H, MASKED>(R, omegas, g, warp, lane, inmask, accmask, acc, na, hb); \
        break;
    switch (h) {
        SRJ_TB_CASE(1)
        SRJ_TB_CASE(2)
        SRJ_TB_CASE(3)
        SRJ_TB_CASE(4)
        SRJ_TB_CASE(5)
        SRJ_TB_CASE(6)
        default: break;
    }
#undef SRJ_TB_CASE
}

// One pass (h sub-sweeps, h <= S) over every tile this CTA owns.  If
// `first_issued`, the TMA for this CTA's first tile is already in flight.
template <int K, bool SLAB>
__device__ __forceinline__ void tb2d_pass(const TbArgs& a, const CUtensorMap* tm_in,
                                          const CUtensorMap* tm_b, double* __restrict__ xout,
                                          const double* om, int h, double (&acc)[tb2d::Cfg<K>::S],
                                          bool accumulate, unsigned ownmask, uint32_t& phase,
                                          bool first_issued, uint32_t& na, uint32_t& hb,
                                          uint32_t& ne) {
    using C = tb2d::Cfg<K>;
    using L = TbLayout<K>;
    constexpr int S = C::S, V = C::V, CW = C::CW, RX = C::RX;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c0 = lane * CW, r0 = warp * V;
    const int nx = a.g.nx, ny = a.g.ny;
    const double coff = a.g.c_off;
    if ((int)blockIdx.x >= a.ntiles) return;
    if (threadIdx.x == 0 && !first_issued) tb2d_issue<K, SLAB>(a, tm_in, tm_b, blockIdx.x);
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
        TileRegs<K> R;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            lds_cols<CW>(R.x[v], L::stx() + (r0 + v) * RX + c0);
            lds_cols<CW>(R.b[v], L::stb() + (r0 + v) * RX + c0);
#pragma unroll
            for (int j = 0; j < CW; ++j) R.p[v][j] = DMUL(coff, R.x[v][j]);
        }
        sts_cols<CW>(L::top(hb) + (warp + 1) * RX + c0, R.p[0]);
        sts_cols<CW>(L::bot(hb) + (warp + 1) * RX + c0, R.p[V - 1]);
        // No block barrier: each warp reports the stage consumed and its first
        // halo rows published (sub-sweep 0 waits for that round); warp 0
        // starts the next tile's copy once every warp has read the stage.
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(L::sempty());
            mbar_arrive(L::hbar(na & 1));
        }
        if (warp == 0 && q + (int)gridDim.x < a.ntiles) {
            mbar_wait(L::sempty(), ne & 1);  // the whole warp waits (no lone spinner)
            if (lane == 0) tb2d_issue<K, SLAB>(a, tm_in, tm_b, q + gridDim.x);
            __syncwarp();
        }
        ++ne;
        if (masked)
            tile_dispatch<K, true>(h, R, om, a.g, warp, lane, inmask, accmask, acc, na, hb);
        else
            tile_dispatch<K, false>(h, R, om, a.g, warp, lane, inmask, accmask, acc, na, hb);
        hb += h;  // the next tile publishes into the parity after this tile's last
        if (storemask) {
#pragma unroll
            for (int v = 0; v < V; ++v) {
                double* row = xout + (long long)(gy0 + v) * nx + gx0;
#pragma unroll
                for (int j = 0; j < CW; j += 2) {
                    // a lane's column pair is owned / inside the grid as a whole
                    // (even nx, even ring and tile widths): one predicated store
                    if ((storemask >> (v * CW + j)) & 1u) {
                        SRJ_ASSERT(gy0 + v >= (SLAB ? a.row_lo : 0) && gy0 + v < (SLAB ? a.row_hi : ny) &&
                                   gx0 + j >= 0 && gx0 + j + 1 < nx);
                        *reinterpret_cast<double2*>(row + j) = make_double2(R.x[v][j], R.x[v][j + 1]);
                    }
                }
            }
        }
        // No barrier here: the halo parity runs on across tiles (hb), so the
        // next tile's first halo rows go to the buffer last read in sub-sweep
        // h-2, which every warp had left before any warp passed the sub-sweep
        // h-1 hand-off (h = 1: two tiles back, behind the next tile-start
        // barrier).
    }
}

template <int K, bool SLAB, bool SOLVE>
__global__ void __launch_bounds__(tb2d::Cfg<K>::THREADS, 1) __maxnreg__(tb2d::Cfg<K>::MAXREG)
    k_tb2d_cycle(const __grid_constant__ CUtensorMap tm_x0,
                 const __grid_constant__ CUtensorMap tm_x1,
                 const __grid_constant__ CUtensorMap tm_b, TbArgs a) {
    using C = tb2d::Cfg<K>;
    using L = TbLayout<K>;
    constexpr int S = C::S;
    // zero halo rows (the rows beyond the first and last warp are never written)
    for (int i = threadIdx.x; i < 2 * C::HBUF; i += blockDim.x) L::top(0)[i] = 0.0;
    if (threadIdx.x == 0) {
        mbar_init(L::bar(), 1);
        mbar_init(L::hbar(0), C::NSEG);
        mbar_init(L::hbar(1), C::NSEG);
        mbar_init(L::sempty(), C::NSEG);
        prefetch_tensormap(&tm_x0);
        prefetch_tensormap(&tm_x1);
        prefetch_tensormap(&tm_b);
    }
    __syncthreads();
    // owned-point bits of this thread's CW x V block (tile-independent)
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
    uint32_t phase = 0, na = 0, hb = 0, ne = 0;
    const CUtensorMap* const tmx[2] = {&tm_x0, &tm_x1};
    auto pass = [&](int in, double* xout, const double* om, int h, double (&acc)[S],
                    bool accumulate, bool first) __attribute__((always_inline)) {
        tb2d_pass<K, SLAB>(a, tmx[in], &tm_b, xout, om, h, acc, accumulate, ownmask, phase, first,
                           na, hb, ne);
    };
    auto issue = [&](int in) {  // a lane of the last warp (it has no part in the pass sums)
        if (threadIdx.x == blockDim.x - 32) tb2d_issue<K, SLAB>(a, tmx[in], &tm_b, blockIdx.x);
    };
    auto drain = [&]() __attribute__((always_inline)) {
        mbar_wait(L::bar(), phase);
        phase ^= 1u;
    };
    if constexpr (SOLVE)
        tb_run_solve<S, F2D>(a, (int)blockIdx.x < a.ntiles, pass, issue, drain);
    else
        tb_run_cycle<S, F2D, SLAB>(a, (int)blockIdx.x < a.ntiles, pass, issue, drain);
}

// ----------------------------------------------------------------------------
// Host side
// ----------------------------------------------------------------------------

template <int K>
static cudaError_t setup_variant(int& per_sm) {
    using C = tb2d::Cfg<K>;
    cudaError_t e = cudaFuncSetAttribute(k_tb2d_cycle<K, false, false>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_tb2d_cycle<K, true, false>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_tb2d_cycle<K, false, true>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::SMEM);
    if (e != cudaSuccess) return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tb2d_cycle<K, false, false>,
                                                         C::THREADS, C::SMEM);
}

template <int K>
static void plan_tiles(TbPlan& plan, const Geom& g, int num_sms) {
    using C = tb2d::Cfg<K>;
    plan.tiles_x[K] = (g.nx + C::TX - 1) / C::TX;
    plan.ntiles[K] = plan.tiles_x[K] * ((g.ny + C::TY - 1) / C::TY);
    plan.blocks[K] = std::max(1, std::min(num_sms, plan.ntiles[K]));
}

int tb_variant_for(const TbPlan& plan, int s) {
    if (plan.small_variant >= 0) return plan.small_variant;
    return s > tb2d::Cfg<0>::S ? 1 : 0;
}

int tb_ring_for(const TbPlan& plan, int s) {
    return tb_variant_for(plan, s) == 1 ? tb2d::Cfg<1>::S : tb2d::Cfg<0>::S;
}

cudaError_t tb_plan_init(TbPlan& plan, const Geom& g, int num_sms) {
    plan = TbPlan();
    // TMA needs 16-byte row pitch: even nx.
    if (g.fam != F2D || (g.nx & 1) || !tma_available()) return cudaSuccess;
    if (g.c_diag != -4.0 * g.c_off) return cudaSuccess;  // the kernel's c_diag*x = -4*p
    int occ[tb2d::kVariants] = {};
    cudaError_t e;
    if ((e = setup_variant<0>(occ[0])) != cudaSuccess) return e;
    if ((e = setup_variant<1>(occ[1])) != cudaSuccess) return e;
    // variant: chosen per launch from the sweeps per pass; SRJ_TB_VARIANT=k
    // forces one (tuning only)
    plan.small_variant = -1;
    if (const char* v = getenv("SRJ_TB_VARIANT")) {
        const int k = atoi(v);
        if (k >= 0 && k < tb2d::kVariants) plan.small_variant = k;
    }
    plan.occupancy = std::min(occ[0], occ[1]);
    if (plan.occupancy < 1) return cudaSuccess;
#ifdef SRJ_STRESS
    {
        const char* br = getenv("SRJ_STRESS_BREAK");
        const int v = (br && atoi(br) == 1) ? 1 : 0;
        if ((e = cudaMemcpyToSymbol(tb_stress_break, &v, sizeof(int))) != cudaSuccess) return e;
    }
#endif
    plan_tiles<0>(plan, g, num_sms);
    plan_tiles<1>(plan, g, num_sms);
    plan.supported = true;
    // region rows per CTA and pass with the square S = 6 tiles (rounds x RY)
    plan.tile_rows = ((plan.ntiles[1] + plan.blocks[1] - 1) / plan.blocks[1]) * tb2d::Cfg<1>::RY;
    return tbs_plan_init(plan, g, num_sms);
}

// The skewed-tile kernel serves whole-grid cycles and solves at 5-6 sweeps per
// pass when it computes fewer region rows per CTA and pass than the square
// tiles (small grids: one 96-row tile per CTA loses to one 72-row tile).
// SRJ_TB_SKEW=0 / 1 forces the choice (tuning and tests).
bool tb_uses_skew(const TbPlan& plan, int s) {
    if (!plan.skew || s <= tb2d::Cfg<0>::S || plan.reserved > 0) return false;
    if (const char* v = getenv("SRJ_TB_SKEW"))
        if (atoi(v) == 1) return true;
    return plan.skew_rows < plan.tile_rows;
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
    a.ntiles = a.tiles_x * ((a.row_hi - a.row_lo + C::TY - 1) / C::TY);
    const int blocks = std::max(1, std::min(plan.blocks[K] - plan.reserved, a.ntiles));
    void* args[] = {&m0, &m1, &mb, &a};
    const void* kern = a.sums != nullptr        ? (const void*)k_tb2d_cycle<K, true, false>
                       : a.ctl.max_cycles > 0 ? (const void*)k_tb2d_cycle<K, false, true>
                                              : (const void*)k_tb2d_cycle<K, false, false>;
    return cudaLaunchCooperativeKernel(kern, dim3(blocks), dim3(C::THREADS), args, C::SMEM, st);
}

cudaError_t tb_launch_cycle(const TbPlan& plan, const Geom& g, double* x, double* x_alt,
                            const double* b, const double* omegas, int M, int s, double tol,
                            double baseline, double* partials, double* hist, int* out_i,
                            double* out_d, cudaStream_t st, int row_lo, int row_hi,
                            double* sums, const SolveCtl* ctl) {
    if ((((uintptr_t)x | (uintptr_t)x_alt | (uintptr_t)b) & 15) != 0)
        return cudaErrorMisalignedAddress;
    TbArgs a;
    a.ctl = ctl ? *ctl : SolveCtl{};
    a.g = g;
    a.buf0 = x;
    a.buf1 = x_alt;
    a.b = b;
    a.omegas = omegas;
    a.M = M;
    a.row_lo = row_lo;
    a.row_hi = row_hi;
    a.sums = sums;
    const int k = tb_variant_for(plan, s);
    a.s = std::max(1, std::min(s, k == 1 ? tb2d::Cfg<1>::S : tb2d::Cfg<0>::S));
    a.tol = tol;
    a.baseline = baseline;
    a.partials = partials;
    a.hist = hist;
    a.out_i = out_i;
    a.out_d = out_d;
    if (sums == nullptr && row_lo == 0 && row_hi == g.ny && tb_uses_skew(plan, s))
        return tbs_launch_cycle(plan, g, a, x, x_alt, b, st);
    switch (k) {
        case 1: return launch_variant<1>(plan, g, a, x, x_alt, b, st);
        default: return launch_variant<0>(plan, g, a, x, x_alt, b, st);
    }
}

}  // namespace srj
