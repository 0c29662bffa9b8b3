// Skewed (parallelogram) temporally blocked SRJ cycle for the 2D 5-point
// constant-coefficient stencil (BASELINE config 2): the same register tile,
// shuffle exchange, shared products and split hand-off barrier as the square
// tile kernel (srj_tb.cu), but without its redundant y-ring.
//
// Tiling.  The grid is cut into strips of TX = 52 owned columns (region RX = 64:
// the strip plus an S = 6 column ring each side, one column pair per lane).  A
// strip is walked top to bottom in tiles of RY = NW*V rows; the tile is skewed
// in time: after sub-sweep t a thread's slot v holds the row one above the row
// it held before, so level t of tile (oy) covers rows [oy - t, oy + RY - t).
// New slot v of warp w is computed from old slots v-2 (south), v-1 (centre) and
// v (north): every value a warp needs from below is its own, and the two rows
// it needs from above come from the warp above (x of its old slots V-2, V-1,
// published in shared memory; the products are recomputed by the reader) -- or, for
// warp 0, from the last warp of the PREVIOUS tile of the strip, which left
// them in a carry buffer, one entry per level.  Consecutive tiles of a strip
// therefore fit together without any redundant rows: per pass a strip computes
// its rows once per sub-sweep (the square tiles compute 72 region rows per 60
// owned).
//
// Segments.  148 CTAs need more parallelism than the strips offer, so a strip
// is cut into segments of rows [lo, hi); a segment inside the grid starts 2S rows
// early (tile oy = lo - 2S) with whatever the carry buffers hold: the values that
// depend on it (slots < 2t at level t) never reach slot 2S.  A cut moves up with
// the level -- the segment below it owns row >= cut - t at level t -- so ownership
// is a property of the slot (slot >= lo - oy, < hi - oy), cuts fall on multiples
// of V rows, and a warp owns all of its points at every level or none: only the
// grid's top and bottom rows need masks.  A segment costs 2S extra rows, once,
// instead of 2S rows per tile.  The host packs segments into equal budgets of T
// tiles per CTA (tbs_plan_init); at 2048^2 a CTA runs 6 tiles of 96 rows where
// the square tiles need 10 rounds of 72 region rows.
//
// b is read from the staged box every sub-sweep (the rows a thread needs move
// up with the skew), which takes it out of the registers; that makes room for
// 16 warps (4 per scheduler) at 128 registers.  The b stage is double-buffered
// across tiles, the x stage is consumed at tile start as in srj_tb.cu.
//
// Arithmetic, residual accumulation, per-pass stop test and rollback are those
// of srj_tb.cu / srj_tbdriver.cuh: iterates are bit-identical to the reference.
#include <cooperative_groups.h>

#include <algorithm>
#if defined(SRJ_TBS_TIMING) || defined(SRJ_TBS_PASSTIME)
#include <cstdio>
#endif
#include <cstdlib>
#include <vector>

#include "srj_stencil.cuh"
#include "srj_tb.cuh"
#include "srj_tbdriver.cuh"
#include "srj_tma.cuh"
#include "srj_walk.cuh"

#ifndef SRJ_TBS_ILP8
#define SRJ_TBS_ILP8 true
#endif
#ifndef SRJ_TBS_NW
#define SRJ_TBS_NW 16
#endif

namespace srj {
namespace tbs {

template <int NW_, int V_, bool ILP8_>
struct CfgT {
    static constexpr int S = 6;       // sweeps fused per pass (= column ring width)
    static constexpr int CW = 2;      // columns per lane
    static constexpr int V = V_;      // rows per warp
    static constexpr int NW = NW_;    // warps
    static constexpr int RX = 32 * CW, RY = NW * V;
    static constexpr int TX = RX - 2 * S;
    static constexpr int THREADS = 32 * NW;
    static constexpr int WARPS_PER_SMSP = (NW + 3) / 4;
    static constexpr int MAXREG_RAW = (16384 / (WARPS_PER_SMSP * 32)) / 8 * 8;
    static constexpr int MAXREG = MAXREG_RAW > 255 ? 255 : MAXREG_RAW;
    static constexpr int BROWS = RY + S;          // b rows staged per tile: [oy - S, oy + RY)
    static constexpr int XSTAGE = RX * RY, BSTAGE = RX * BROWS;
    static constexpr int HSLOT = 2 * RX;          // one publication: x[V-2], x[V-1]
    static constexpr int HBUF = NW * HSLOT;       // one parity of the warp-to-warp rows
    static constexpr int CARRY = S * HSLOT;       // one tile parity of the tile-to-tile rows
    // shared-memory layout (doubles)
    static constexpr int OFF_X = 0, OFF_B = XSTAGE, OFF_H = OFF_B + 2 * BSTAGE,
                         OFF_C = OFF_H + 2 * HBUF, OFF_BAR = OFF_C + 2 * CARRY;
    static constexpr int MAXT = 128;              // tile descriptors kept in shared memory
    // mbarriers: TMA full, 2 hand-off rounds, stage consumed
    static constexpr int OFF_OM = OFF_BAR + 4;             // the pass's omegas [S] (+ pad)
    static constexpr int OFF_DESC = OFF_OM + 8;            // int4[MAXT]
    static constexpr size_t SMEM = (size_t)(OFF_DESC + 2 * MAXT) * sizeof(double);
    static constexpr bool ILP8 = ILP8_;
    static constexpr uint32_t TX_BYTES = (uint32_t)((XSTAGE + BSTAGE) * sizeof(double));
    static_assert(V == 6, "row groups are written for 6 rows per warp");
    static_assert((XSTAGE * 8) % 128 == 0 && (BSTAGE * 8) % 128 == 0, "TMA destinations");
};

using Cfg = CfgT<SRJ_TBS_NW, 6, SRJ_TBS_ILP8>;  // 64 x 96 tiles, 512 threads, 128 registers

}  // namespace tbs

extern __shared__ __align__(128) double tbs_smem[];

template <class C>
struct TbsLayout {
    __device__ static __forceinline__ double* stx() { return tbs_smem + C::OFF_X; }
    __device__ static __forceinline__ double* stb(uint32_t par) {
        return tbs_smem + C::OFF_B + (par & 1u) * C::BSTAGE;
    }
    __device__ static __forceinline__ uint64_t* bar() {
        return reinterpret_cast<uint64_t*>(tbs_smem + C::OFF_BAR);
    }
    __device__ static __forceinline__ uint64_t* hbar(int i) {
        return reinterpret_cast<uint64_t*>(tbs_smem + C::OFF_BAR) + 1 + i;
    }
    // stage consumed (one arrival per warp): the next tile's copy may start
    __device__ static __forceinline__ uint64_t* sempty() {
        return reinterpret_cast<uint64_t*>(tbs_smem + C::OFF_BAR) + 3;
    }
    __device__ static __forceinline__ double* om() { return tbs_smem + C::OFF_OM; }
    __device__ static __forceinline__ int4* desc_ptr() {
        return reinterpret_cast<int4*>(tbs_smem + C::OFF_DESC);
    }
    __device__ static __forceinline__ int4 desc(int i) { return desc_ptr()[i]; }
    // Where warp `warp` publishes its level-`level` rows (read by the warp
    // below; the last warp's go to the carry of this tile for the next one).
    __device__ static __forceinline__ int wr_off(int warp, int level, uint32_t hb, uint32_t tc) {
        return warp == C::NW - 1 ? C::OFF_C + (int)(tc & 1u) * C::CARRY + level * C::HSLOT
                                 : C::OFF_H + (int)((hb + level) & 1u) * C::HBUF + warp * C::HSLOT;
    }
    // Where warp `warp` finds the level-`level` rows above its own.
    __device__ static __forceinline__ int rd_off(int warp, int level, uint32_t hb, uint32_t tc) {
        return warp == 0 ? C::OFF_C + (int)((tc + 1u) & 1u) * C::CARRY + level * C::HSLOT
                         : C::OFF_H + (int)((hb + level) & 1u) * C::HBUF + (warp - 1) * C::HSLOT;
    }
};

__device__ __forceinline__ void tbs_lds2(double (&d)[2], int off) {
    SRJ_ASSERT_SMEM(tbs_smem + off, 16, tbs_smem);
    const double2 v = *reinterpret_cast<const double2*>(tbs_smem + off);
    d[0] = v.x;
    d[1] = v.y;
}
__device__ __forceinline__ void tbs_sts2(int off, const double (&d)[2]) {
    SRJ_ASSERT_SMEM(tbs_smem + off, 16, tbs_smem);
    *reinterpret_cast<double2*>(tbs_smem + off) = make_double2(d[0], d[1]);
}

template <class C>
__device__ __forceinline__ void tbs_issue(const CUtensorMap* tm_in, const CUtensorMap* tm_b, int ox,
                                          int oy, uint32_t bpar) {
    using L = TbsLayout<C>;
    fence_proxy_async();
    mbar_expect_tx(L::bar(), C::TX_BYTES);
    tma_load_2d(L::stx(), tm_in, ox - C::S, oy, L::bar());
    tma_load_2d(L::stb(bpar), tm_b, ox - C::S, oy - C::S, L::bar());
}

__device__ __forceinline__ void tbs_fma_sq_if(double& acc, double r, unsigned cond) {
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p fma.rn.f64 %0, %1, %1, %0;\n\t}"
        : "+d"(acc)
        : "d"(r), "r"(cond));
}

// Loop state that runs on across tiles, passes and cycles of a launch.
struct TbsState {
    uint32_t phase;  // parity of the TMA-full barrier
    uint32_t hb;     // hand-off rounds so far (= parity base of the warp-to-warp row buffers)
    uint32_t tc;     // tiles started (b stage, carry and stage-consumed parity)
};

#ifdef SRJ_TBS_TIMING  // (tuning only) clock ticks of CTA 0, first / last warp, third tile
__shared__ long long tbs_tm[2][40];
#define TBS_TICK(k)                                                                        \
    do {                                                                                   \
        if (blockIdx.x == 0 && st.tc == 2u && (threadIdx.x & 31) == 0 &&                   \
            (threadIdx.x == 0 || threadIdx.x == 32 * (tbs::Cfg::NW - 1)))                  \
            tbs_tm[threadIdx.x != 0][k] = clock64();                                       \
    } while (0)
#else
#define TBS_TICK(k) ((void)0)
#endif

// Hand-off of the published rows: one mbarrier round per level (every warp
// arrives after publishing, waits before reading).  g = st.hb + level numbers
// the rounds across tiles, passes and cycles (barrier g & 1, use g >> 1).
template <class C>
struct TbsSync {
    using L = TbsLayout<C>;
    __device__ static __forceinline__ void wait_read(int level, const TbsState& st) {
        const uint32_t g = st.hb + level;
        mbar_wait(L::hbar(g & 1), (g >> 1) & 1);
    }
    __device__ static __forceinline__ void done_write(int lane, int level, const TbsState& st) {
        const uint32_t g = st.hb + level;
        __syncwarp();
        if (lane == 0) mbar_arrive(L::hbar(g & 1));
    }
};

// NR rows (2*NR chains) of new slots V0 .. V0+NR-1 from this thread's own old
// slots: south = old slot v-2, centre = old slot v-1, north = old slot v.
template <class C, int V0, int NR, bool MASKED>
__device__ __forceinline__ void tbs_rows(const double (&X)[C::V][2], const double (&P)[C::V][2],
                                         const double (&pw)[C::V], const double (&pe)[C::V],
                                         double (&Xn)[C::V][2], double (&sq)[4], double w,
                                         double inv, unsigned im, unsigned am, int boff) {
    constexpr int NP = 2 * NR, RX = C::RX;
    double y[NP], rr[NP];
#pragma unroll
    for (int k = 0; k < NP; ++k) y[k] = P[V0 + (k >> 1) - 2][k & 1];
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        const int c = V0 + (k >> 1) - 1, j = k & 1;
        y[k] = DADD(y[k], j == 0 ? pw[c] : P[c][0]);
    }
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        const int c = V0 + (k >> 1) - 1, j = k & 1;
        y[k] = __fma_rn(P[c][j], -4.0, y[k]);  // + c_diag*x = -4*p (srj_tb.cu header)
    }
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        const int c = V0 + (k >> 1) - 1, j = k & 1;
        y[k] = DADD(y[k], j == 1 ? pe[c] : P[c][1]);
    }
#pragma unroll
    for (int k = 0; k < NP; ++k) y[k] = DADD(y[k], P[V0 + (k >> 1)][k & 1]);
#pragma unroll
    for (int k = 0; k < NP; k += 2) {
        double bv[2];
        tbs_lds2(bv, boff + (V0 + (k >> 1)) * RX);
        rr[k] = DSUB(bv[0], y[k]);
        rr[k + 1] = DSUB(bv[1], y[k + 1]);
    }
#pragma unroll
    for (int k = 0; k < NP; ++k) {
        const int v = V0 + (k >> 1), j = k & 1;
        const double xn = relax(X[v - 1][j], inv, rr[k], w);
        if constexpr (!MASKED)
            sq[k & 3] = fma(rr[k], rr[k], sq[k & 3]);  // owned: decided per thread by the caller
        else
            tbs_fma_sq_if(sq[k & 3], rr[k], (am >> v) & 1u);
        Xn[v][j] = (!MASKED || ((im >> v) & 1u)) ? xn : 0.0;
    }
}

// H sub-sweeps (compile time) of the skewed tile held in registers: X, P are
// the thread's V x 2 values and products at level 0 on entry, level H on exit
// (slot v then holds row R0 + v - H).  MASKED warps (some row outside the grid
// at some level: the grid's top and bottom): inmask, bit i <-> row offset i - 6
// from R0 is inside the grid (the bit of new slot v at sub-sweep t is
// v - t + 5); a row outside is held at 0 and not counted.  accmask: the slots
// this thread owns (bit v; its column pair and `accumulate` folded in) -- all
// or none in the other warps (`accmask` != 0: all), which count and keep every
// point they compute.  boff: this thread's offset into the b stage,
// stb + (V*warp + 5)*RX + c0; the row of new slot v at sub-sweep t sits
// (v - t) rows further.
template <class C, int H, bool MASKED>
__device__ __forceinline__ void tbs_tile_sweeps(double (&X)[C::V][2], double (&P)[C::V][2],
                                                const double* omegas, double coff, double inv,
                                                int warp, int lane, unsigned inmask,
                                                unsigned accmask, double (&acc)[C::S],
                                                const TbsState& st, int boff) {
    using L = TbsLayout<C>;
    constexpr int V = C::V, RX = C::RX;
    const int c0 = lane * 2;
#pragma unroll
    for (int t = 0; t < H; ++t) {
        const double w = L::om()[t];
        const unsigned im = inmask >> (5 - t), am = im & accmask;
        double pw[V], pe[V];  // p across the lane boundary of the centre rows (old slots 0..V-2)
#pragma unroll
        for (int v = 1; v < V - 1; ++v) {
            pw[v] = shfl_up_d(P[v][1], 1);
            pe[v] = shfl_down_d(P[v][0], 1);
        }
        double Xn[V][2];
        double sq[4] = {0.0, 0.0, 0.0, 0.0};
        // new slots 2..5: everything they need is this thread's
        if constexpr (C::ILP8) {
            tbs_rows<C, 2, 4, MASKED>(X, P, pw, pe, Xn, sq, w, inv, im, am, boff - t * RX);
        } else {
            tbs_rows<C, 4, 2, MASKED>(X, P, pw, pe, Xn, sq, w, inv, im, am, boff - t * RX);
            tbs_rows<C, 2, 2, MASKED>(X, P, pw, pe, Xn, sq, w, inv, im, am, boff - t * RX);
        }
        // level-t rows of the warp above (t = 0: published at tile start)
        TBS_TICK(1 + 3 * t);
        TbsSync<C>::wait_read(t, st);
        TBS_TICK(2 + 3 * t);
        double p4[2], p5[2], x5[2];
        {
            const int ro = L::rd_off(warp, t, st.hb, st.tc) + c0;
            double x4[2];
            tbs_lds2(x4, ro);
            tbs_lds2(x5, ro + RX);
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                p4[j] = DMUL(coff, x4[j]);
                p5[j] = DMUL(coff, x5[j]);
            }
        }
        {  // new slots 0, 1 (4 chains)
            const double p5w = shfl_up_d(p5[1], 1), p5e = shfl_down_d(p5[0], 1);
            const double p0w = shfl_up_d(P[0][1], 1), p0e = shfl_down_d(P[0][0], 1);
            double y[4], rr[4];
            y[0] = p4[0];
            y[1] = p4[1];
            y[2] = p5[0];
            y[3] = p5[1];
            y[0] = DADD(y[0], p5w);
            y[1] = DADD(y[1], p5[0]);
            y[2] = DADD(y[2], p0w);
            y[3] = DADD(y[3], P[0][0]);
            y[0] = __fma_rn(p5[0], -4.0, y[0]);
            y[1] = __fma_rn(p5[1], -4.0, y[1]);
            y[2] = __fma_rn(P[0][0], -4.0, y[2]);
            y[3] = __fma_rn(P[0][1], -4.0, y[3]);
            y[0] = DADD(y[0], p5[1]);
            y[1] = DADD(y[1], p5e);
            y[2] = DADD(y[2], P[0][1]);
            y[3] = DADD(y[3], p0e);
            y[0] = DADD(y[0], P[0][0]);
            y[1] = DADD(y[1], P[0][1]);
            y[2] = DADD(y[2], P[1][0]);
            y[3] = DADD(y[3], P[1][1]);
            double b0[2], b1[2];
            tbs_lds2(b0, boff + (0 - t) * RX);
            tbs_lds2(b1, boff + (1 - t) * RX);
            rr[0] = DSUB(b0[0], y[0]);
            rr[1] = DSUB(b0[1], y[1]);
            rr[2] = DSUB(b1[0], y[2]);
            rr[3] = DSUB(b1[1], y[3]);
            const double xc[4] = {x5[0], x5[1], X[0][0], X[0][1]};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int v = k >> 1, j = k & 1;
                const double xn = relax(xc[k], inv, rr[k], w);
                if constexpr (!MASKED)
                    sq[k] = fma(rr[k], rr[k], sq[k]);
                else
                    tbs_fma_sq_if(sq[k], rr[k], (am >> v) & 1u);
                Xn[v][j] = (!MASKED || ((im >> v) & 1u)) ? xn : 0.0;
            }
        }
        if constexpr (!MASKED)
            acc[t] = accmask != 0u ? DADD(acc[t], DADD(DADD(sq[0], sq[1]), DADD(sq[2], sq[3])))
                                   : acc[t];
        else
            acc[t] = DADD(acc[t], DADD(DADD(sq[0], sq[1]), DADD(sq[2], sq[3])));
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
            for (int j = 0; j < 2; ++j) X[v][j] = Xn[v][j];
        if (t + 1 < H) {  // (the products of the pass's last level are never used)
#pragma unroll
            for (int v = 0; v < V; ++v)
#pragma unroll
                for (int j = 0; j < 2; ++j) P[v][j] = DMUL(coff, X[v][j]);
            const int wo = L::wr_off(warp, t + 1, st.hb, st.tc) + c0;
            tbs_sts2(wo, X[V - 2]);
            tbs_sts2(wo + RX, X[V - 1]);
            TbsSync<C>::done_write(lane, t + 1, st);
        }
        TBS_TICK(3 + 3 * t);
    }
}

template <class C, bool MASKED>
__device__ __forceinline__ void tbs_dispatch(int h, double (&X)[C::V][2], double (&P)[C::V][2],
                                             const double* omegas, double coff, double inv,
                                             int warp, int lane, unsigned inmask, unsigned accmask,
                                             double (&acc)[C::S], const TbsState& st, int boff) {
#define SRJ_TBS_CASE(H)                                                                        \
    case H:                                                                                    \
        tbs_tile_sweeps<C, H, MASKED>(X, P, omegas, coff, inv, warp, lane, inmask, accmask, acc, \
                                      st, boff);                                               \
        break;
    switch (h) {
        SRJ_TBS_CASE(1)
        SRJ_TBS_CASE(2)
        SRJ_TBS_CASE(3)
        SRJ_TBS_CASE(4)
        SRJ_TBS_CASE(5)
        SRJ_TBS_CASE(6)
        default: break;
    }
#undef SRJ_TBS_CASE
}

// Bits [a, b) of an 11-bit row mask, a and b clamped to [0, 11].
__device__ __forceinline__ unsigned tbs_range_mask(int a, int b) {
    a = min(max(a, 0), 11);
    b = min(max(b, 0), 11);
    return b > a ? ((1u << b) - 1u) & ~((1u << a) - 1u) : 0u;
}

// One pass (h sub-sweeps, 1 <= h <= S) over this CTA's tiles (descriptors in
// shared memory).  If `first_issued`, the TMA of the first tile is in flight.
template <class C>
__device__ __forceinline__ void tbs_pass(const TbArgs& a, const CUtensorMap* tm_in,
                                         const CUtensorMap* tm_b, double* __restrict__ xout,
                                         const double* om, int h, double (&acc)[C::S],
                                         bool accumulate, bool first_issued, int ntile,
                                         TbsState& st) {
    using L = TbsLayout<C>;
    constexpr int S = C::S, V = C::V, RX = C::RX;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c0 = lane * 2;
    const int nx = a.g.nx, ny = a.g.ny;
    const double coff = a.g.c_off;
    if (ntile == 0) return;
#ifdef SRJ_TBS_PASSTIME
    unsigned long long pt0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(pt0));
#endif
    // Pass start (every warp is past the previous pass's block barriers): the
    // pass's omegas into shared memory.
    if (threadIdx.x < h) L::om()[threadIdx.x] = __ldg(om + threadIdx.x);
    __syncthreads();
    if (threadIdx.x == 0 && !first_issued) {
        const int4 d = L::desc(0);
        tbs_issue<C>(tm_in, tm_b, d.x, d.y, st.tc);
    }
    const bool cown = lane >= S / 2 && lane < 32 - S / 2;  // region columns S .. RX-S-1
    for (int i = 0; i < ntile; ++i) {
        int R0, gx0, lo, hi;
        bool masked, cin;
        unsigned inmask = 0u, ownmask = 0u;
        {
            const int4 d = L::desc(i);
            lo = d.z;
            hi = d.w;
            R0 = d.y + warp * V;  // row of slot 0 at level 0
            gx0 = d.x - S + c0;
            // Ownership.  Inside the grid a segment boundary moves up with the level
            // (the pair (row, level t) belongs to the segment below the cut iff
            // row >= cut - t - 1 for residuals, cut - t for values), which makes it a
            // property of the SLOT: slot s = V*warp + v of the tile at oy is owned iff
            // lo - oy <= s < hi - oy; the packing cuts at multiples of V rows and
            // starts a segment 2S rows early, so a warp owns all of its slots or
            // none.  At the grid's top and bottom ownership is "inside the grid",
            // row by row and level by level (inmask).  Over all levels a warp's slots
            // hold rows R0-6 .. R0+4: a warp with all of them inside the grid runs
            // the unmasked code.  Columns outside the grid (first / last strip) need
            // no mask: a lane there relaxes with inv = 0, so its points stay at the
            // zero the copy engine filled in (x' = 0 + w*(0*r), r finite: such a
            // point has at most one non-zero neighbour product).
            const int s_lo = lo > 0 ? lo - d.y : 0, s_hi = hi < ny ? hi - d.y : C::RY;
            const int a0 = min(max(s_lo - warp * V, 0), V), a1 = min(max(s_hi - warp * V, 0), V);
            const unsigned slots = a1 > a0 ? ((1u << a1) - 1u) & ~((1u << a0) - 1u) : 0u;
            const bool allin = R0 - 6 >= 0 && R0 + 4 < ny;
            masked = !(allin && (slots == 0u || slots == (1u << V) - 1u));
            cin = gx0 >= 0 && gx0 < nx;  // a lane's column pair is inside as a whole (even nx)
            inmask = masked ? tbs_range_mask(6 - R0, ny + 6 - R0) : 0x7ffu;
            ownmask = (cin && cown) ? slots : 0u;
        }
        const unsigned accmask = accumulate ? ownmask : 0u;
        TBS_TICK(30);
        mbar_wait(L::bar(), st.phase);
        TBS_TICK(31);
        st.phase ^= 1u;
        double X[V][2], P[V][2];
#pragma unroll
        for (int v = 0; v < V; ++v) {
            tbs_lds2(X[v], C::OFF_X + (warp * V + v) * RX + c0);
#pragma unroll
            for (int j = 0; j < 2; ++j) P[v][j] = DMUL(coff, X[v][j]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(L::sempty());
        {
            const int wo = L::wr_off(warp, 0, st.hb, st.tc) + c0;
            tbs_sts2(wo, X[V - 2]);
            tbs_sts2(wo + RX, X[V - 1]);
            TbsSync<C>::done_write(lane, 0, st);
        }
        // warp 0 starts the next tile's copy once every warp has moved its rows of the
        // x stage into registers (issuing it later, after the first hand-off round, which
        // implies the same, measured 2% slower)
        if (warp == 0 && i + 1 < ntile) {
            mbar_wait(L::sempty(), st.tc & 1);  // the whole warp waits (no lone spinner)
            if (lane == 0) {
                const int4 dn = L::desc(i + 1);
                tbs_issue<C>(tm_in, tm_b, dn.x, dn.y, st.tc + 1u);
            }
            __syncwarp();
        }
        TBS_TICK(0);
        const int boff = C::OFF_B + (int)(st.tc & 1u) * C::BSTAGE + (warp * V + 5) * RX + c0;
        const double inv = cin ? a.g.inv_diag : 0.0;
        if (masked)
            tbs_dispatch<C, true>(h, X, P, om, coff, inv, warp, lane, inmask, accmask, acc, st, boff);
        else
            tbs_dispatch<C, false>(h, X, P, om, coff, inv, warp, lane, inmask, accmask, acc, st, boff);
        TBS_TICK(32);
        st.hb += h;
        ++st.tc;
        // slot v now holds row R0 + v - h (in-grid bit v - h + 6), owned by slot
        const unsigned sm = (inmask >> (6 - h)) & ownmask;
        if (sm) {
#pragma unroll
            for (int v = 0; v < V; ++v) {
                if ((sm >> v) & 1u) {
                    const int gy = R0 + v - h;
                    // the segment's rows at level h: cuts inside the grid have moved up by h
                    SRJ_ASSERT(gy >= (lo > 0 ? lo - h : 0) && gy < (hi < ny ? hi - h : ny) && gy >= 0 &&
                               gy < ny && gx0 >= 0 && gx0 + 1 < nx);
                    *reinterpret_cast<double2*>(xout + (long long)gy * nx + gx0) =
                        make_double2(X[v][0], X[v][1]);
                }
            }
        }
#ifdef SRJ_TBS_TIMING
        if (blockIdx.x == 0 && st.tc == 3u && lane == 0 && (warp == 0 || warp == C::NW - 1)) {
            const long long* tm = tbs_tm[warp != 0];
            const long long t1 = clock64();
            printf("warp %2d h %d: top->tma %lld  tma->pub0 %lld |", warp, h, tm[31] - tm[30], tm[0] - tm[31]);
            for (int t = 0; t < h; ++t)
                printf(" [int %lld wait %lld rest %lld]", tm[1 + 3 * t] - (t ? tm[3 * t] : tm[0]),
                       tm[2 + 3 * t] - tm[1 + 3 * t], tm[3 + 3 * t] - tm[2 + 3 * t]);
            printf(" | store %lld  tile %lld\n", t1 - tm[32], t1 - tm[30]);
        }
#endif
    }
#ifdef SRJ_TBS_PASSTIME
    if (st.tc == 4u * ntile && threadIdx.x == 0) {
        unsigned long long pt1;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(pt1));
        printf("PASS cta %d ntile %d start %llu dur %llu\n", (int)blockIdx.x, ntile, pt0, pt1 - pt0);
    }
#endif
}

template <class C, bool SOLVE>
__global__ void __launch_bounds__(C::THREADS, 1) __maxnreg__(C::MAXREG)
    k_tbs_cycle(const __grid_constant__ CUtensorMap tm_x0, const __grid_constant__ CUtensorMap tm_x1,
                const __grid_constant__ CUtensorMap tm_b, TbArgs a) {
    using L = TbsLayout<C>;
    constexpr int S = C::S;
    // the row buffers start as zeros (what a first tile reads before any
    // publication only reaches values that are never used, but keep them finite)
    for (int i = threadIdx.x; i < 2 * C::HBUF + 2 * C::CARRY; i += blockDim.x)
        tbs_smem[C::OFF_H + i] = 0.0;
    if (threadIdx.x == 0) {
        mbar_init(L::bar(), 1);
        mbar_init(L::hbar(0), C::NW);
        mbar_init(L::hbar(1), C::NW);
        mbar_init(L::sempty(), C::NW);
        prefetch_tensormap(&tm_x0);
        prefetch_tensormap(&tm_x1);
        prefetch_tensormap(&tm_b);
    }
    __syncthreads();
    TbsState st{0u, 0u, 0u};
    const CUtensorMap* const tmx[2] = {&tm_x0, &tm_x1};
    // this CTA's tile descriptors (until an entry with hi <= lo) into shared memory
    __shared__ int s_ntile;
    if (threadIdx.x == 0) s_ntile = a.tpc;
    __syncthreads();
    for (int i = threadIdx.x; i < a.tpc; i += blockDim.x) {
        const int4 d = __ldg(a.tab + (size_t)blockIdx.x * a.tpc + i);
        L::desc_ptr()[i] = d;
        if (d.w <= d.z) atomicMin(&s_ntile, i);
    }
    __syncthreads();
    const int ntile = s_ntile;
    auto pass = [&](int in, double* xout, const double* om, int h, double (&acc)[S],
                    bool accumulate, bool first_issued) __attribute__((always_inline)) {
        tbs_pass<C>(a, tmx[in], &tm_b, xout, om, h, acc, accumulate, first_issued, ntile, st);
    };
    auto issue = [&](int in) {  // a lane of the last warp (it has no part in the pass sums)
        if (threadIdx.x == blockDim.x - 32) {
            const int4 d = L::desc(0);
            tbs_issue<C>(tmx[in], &tm_b, d.x, d.y, st.tc);
        }
    };
    auto drain = [&]() __attribute__((always_inline)) {
        mbar_wait(L::bar(), st.phase);
        st.phase ^= 1u;
    };
    if constexpr (SOLVE)
        tb_run_solve<S, F2D>(a, ntile > 0, pass, issue, drain);
    else
        tb_run_cycle<S, F2D, false>(a, ntile > 0, pass, issue, drain);
}

// ----------------------------------------------------------------------------
// Host side
// ----------------------------------------------------------------------------

// Greedy packing of the strips' rows into `ncta` budgets of T tiles: a CTA
// takes rows of the current strip until its budget is used up (a segment of k
// tiles owns at most k*RY - 2S rows) and carries what is left of it into the
// next strip.  Returns false when T tiles per CTA are not enough.
static bool tbs_pack(int nx, int ny, int ncta, int T, std::vector<int4>& tab, int& used) {
    using C = tbs::Cfg;
    const int strips = (nx + C::TX - 1) / C::TX;
    tab.assign((size_t)ncta * T, make_int4(0, 0, 0, 0));
    int c = 0, left = T;
    for (int sx = 0; sx < strips; ++sx) {
        int pos = 0;
        while (pos < ny) {
            if (c >= ncta) return false;
            // lead: rows the first tile starts above the segment (a restart inside the
            // grid: two warps of slots that only feed the skew; at the grid top: the skew)
            const int lead = pos > 0 ? 2 * C::S : C::S;
            int rows, k;
            if (ny - pos + lead + C::S <= left * C::RY) {  // to the grid's bottom (skew: S rows)
                rows = ny - pos;
                k = (rows + lead + C::S + C::RY - 1) / C::RY;
            } else {  // cut inside the grid, at a multiple of V rows (whole warps own or not)
                rows = std::min((left * C::RY - lead) / C::V * C::V, (ny - pos - 1) / C::V * C::V);
                k = (rows + lead + C::RY - 1) / C::RY;
                if (rows <= 0) {  // (budget too small for a cut here: next CTA)
                    ++c;
                    left = T;
                    continue;
                }
            }
            for (int i = 0; i < k; ++i)
                tab[(size_t)c * T + (T - left) + i] =
                    make_int4(sx * C::TX, pos - lead + i * C::RY, pos, pos + rows);
            left -= k;
            pos += rows;
            if (left == 0) {
                ++c;
                left = T;
            }
        }
    }
    used = c + (left < T ? 1 : 0);
    return true;
}

// The smallest budget T of tiles per CTA that packs the grid into `ncta` CTAs,
// with its table (ncta * T entries {ox, oy, lo, hi}, hi <= lo: no tile) and
// the CTAs that own tiles.  Host only (no CUDA call): srj_skew_plan exposes it.
void tbs_plan_tiles(int nx, int ny, int ncta, std::vector<int4>& tab, int& T, int& used) {
    using C = tbs::Cfg;
    const int strips = (nx + C::TX - 1) / C::TX;
    const long long need = (long long)strips * (ny + 2 * C::S);  // one segment per strip
    T = (int)std::max<long long>(1, (need + (long long)C::RY * ncta - 1) / ((long long)C::RY * ncta));
    while (!tbs_pack(nx, ny, ncta, T, tab, used)) ++T;
}

int tbs_plan_table(int nx, int ny, int ncta, int* out, long long capacity, int* T, int* used) {
    std::vector<int4> tab;
    tbs_plan_tiles(nx, ny, ncta, tab, *T, *used);
    if (out == nullptr) return 0;
    if ((long long)tab.size() * 4 > capacity) return -1;
    for (size_t i = 0; i < tab.size(); ++i) {
        out[4 * i + 0] = tab[i].x;
        out[4 * i + 1] = tab[i].y;
        out[4 * i + 2] = tab[i].z;
        out[4 * i + 3] = tab[i].w;
    }
    return 0;
}

int tbs_tile_rows() { return tbs::Cfg::RY; }
int tbs_tile_cols() { return tbs::Cfg::TX; }
int tbs_sweeps() { return tbs::Cfg::S; }

cudaError_t tbs_plan_init(TbPlan& plan, const Geom& g, int num_sms) {
    using C = tbs::Cfg;
    plan.skew = false;
    if (const char* v = getenv("SRJ_TB_SKEW"))
        if (atoi(v) == 0) return cudaSuccess;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_tbs_cycle<C, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)C::SMEM)) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(k_tbs_cycle<C, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)C::SMEM)) != cudaSuccess)
        return e;
    int occ = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_tbs_cycle<C, true>, C::THREADS,
                                                           C::SMEM)) != cudaSuccess)
        return e;
    if (occ < 1) return cudaSuccess;
    std::vector<int4> tab;
    int T = 0, used = 0;
    tbs_plan_tiles(g.nx, g.ny, num_sms, tab, T, used);
    if (T > C::MAXT) return cudaSuccess;  // descriptors would not fit: square tiles serve the grid
    plan.skew_tpc = T;
    plan.skew_blocks = used;
    plan.skew_rows = T * C::RY;
    if ((e = cudaMalloc(&plan.skew_tab, tab.size() * sizeof(int4))) != cudaSuccess) return e;
    if ((e = cudaMemcpy(plan.skew_tab, tab.data(), tab.size() * sizeof(int4),
                        cudaMemcpyHostToDevice)) != cudaSuccess)
        return e;
    plan.skew = true;
    return cudaSuccess;
}

void tbs_plan_free(TbPlan& plan) {
    cudaFree(plan.skew_tab);
    plan.skew_tab = nullptr;
    plan.skew = false;
}

cudaError_t tbs_launch_cycle(const TbPlan& plan, const Geom& g, TbArgs& a, double* x, double* x_alt,
                             const double* b, cudaStream_t st) {
    using C = tbs::Cfg;
    CUtensorMap m0, m1, mb;
    cudaError_t e;
    if ((e = encode_field_map(&m0, x, g.nx, g.ny, C::RX, C::RY)) != cudaSuccess) return e;
    if ((e = encode_field_map(&m1, x_alt, g.nx, g.ny, C::RX, C::RY)) != cudaSuccess) return e;
    if ((e = encode_field_map(&mb, b, g.nx, g.ny, C::RX, C::BROWS)) != cudaSuccess) return e;
    a.tab = reinterpret_cast<const int4*>(plan.skew_tab);
    a.tpc = plan.skew_tpc;
    a.s = std::max(1, std::min(a.s, C::S));
    void* args[] = {&m0, &m1, &mb, &a};
    const void* kern = a.ctl.max_cycles > 0 ? (const void*)k_tbs_cycle<C, true>
                                            : (const void*)k_tbs_cycle<C, false>;
    return cudaLaunchCooperativeKernel(kern, dim3(plan.skew_blocks), dim3(C::THREADS), args, C::SMEM,
                                       st);
}

}  // namespace srj
