// Temporally blocked SRJ cycle for the 3D 7-point constant-coefficient
// stencil (BASELINE configs 3 and 5): two consecutive sweeps, each with its
// own omega, per HBM round trip of x and b.
//
// Work item = one TX x TY xy tile (60 x 32 owned points) over a run of planes
// [z0, z1).  The copy engine (TMA) streams plane z of x_{k0} (box 64 x 36: the
// tile plus a two-point ring) and of b (box 64 x 34) into a 6-stage
// shared-memory ring two planes ahead of the consuming step; full barriers
// carry the TMA byte count, empty barriers collect one arrival per warp, and
// thread 0 issues load n+2 at step n once its stage is free.  A stage lives
// for three steps: x of plane z is read at step z (new plane) and z+1
// (centre of level 1), b at z+1 (level 1) and z+2 (level 2).
//
// Compute warps are independent: warp w owns tile rows 4w .. 4w+3 and
// computes the first sweep on its rows plus one halo row above and below
// (6 rows), so the second sweep never needs another warp's values and no
// block-wide barrier is taken per plane.  Lane l owns box columns 2l, 2l+1;
// the first sweep reads its x-neighbours from the staged plane, the second
// gets them by warp shuffle; y-neighbours are the thread's own rows and
// z-neighbours stream through registers.
//
// Streaming form of the stencil.  Each level carries, per point of the
// previous plane c-1, the partial sum
//   ypart(c-1) = ((((p(z-1) + p(y-1)) + p(x-1)) + c_diag*x) + p(x+1)) + p(y+1)
// When plane c arrives, y(c-1) = ypart(c-1) + p(c) completes the reference's
// ascending-column sum (csr_matvec order, every product rounded once and shared
// by the six points that use it), r = b - y, x' = x + omega*(inv*r) -- the
// exactness recipe of SURVEY 8a.6, so iterates are bit-identical (the leading
// "0 +" is dropped as in the 2D kernels).  Level 1 at step z
// finishes plane z-1 of x_{k0+1}; level 2 takes that plane as its new plane and
// finishes plane z-2 of x_{k0+2}.  Points outside the grid and the ghost
// planes of x_{k0+1} are forced to zero (Dirichlet); ring values that go stale
// never reach an owned point.
//
// Residuals and stopping: the shared per-cycle driver (srj_tbdriver.cuh) --
// level t accumulates (b - A x_{k0+t-1})^2 over owned points, one grid barrier
// per pass, fixed-order reduction in every CTA, the reference's per-sweep stop
// test (solver.py:216-222, 235-239), rollback re-run of a pass that stops inside.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "srj_stencil.cuh"
#include "srj_tb.cuh"
#include "srj_tbdriver.cuh"
#include "srj_tma.cuh"
#include "srj_walk.cuh"

namespace srj {
namespace tb3d {

constexpr int S = 2;                    // sweeps fused per pass
constexpr int CW = 2;                   // columns per lane
constexpr int V = 4;                    // owned rows per warp
constexpr int NW = 8;                   // compute warps
constexpr int THREADS = 32 * NW;
constexpr int RX = 32 * CW;             // box columns (64)
constexpr int TX = RX - 2 * S;          // owned columns (60)
constexpr int TY = NW * V;              // owned rows (32)
constexpr int XROWS = TY + 2 * S;       // x box rows (36), origin oy - 2
constexpr int BROWS = TY + 2;           // b box rows (34), origin oy - 1
constexpr int D = 6;                    // ring stages (x box + b box each)
constexpr int XPLANE = RX * XROWS, BPLANE = RX * BROWS;
constexpr size_t SMEM = (size_t)(D * (XPLANE + BPLANE)) * sizeof(double) + sizeof(uint64_t) * 2 * D;
constexpr uint32_t TX_BYTES = (uint32_t)((XPLANE + BPLANE) * sizeof(double));

}  // namespace tb3d

extern __shared__ __align__(128) double tb3_smem[];

struct Tb3Ring {
    __device__ static __forceinline__ double* xs(int s) { return tb3_smem + s * tb3d::XPLANE; }
    __device__ static __forceinline__ double* bs(int s) {
        return tb3_smem + tb3d::D * tb3d::XPLANE + s * tb3d::BPLANE;
    }
    __device__ static __forceinline__ uint64_t* bars() {
        return reinterpret_cast<uint64_t*>(tb3_smem + tb3d::D * (tb3d::XPLANE + tb3d::BPLANE));
    }
    __device__ static __forceinline__ uint64_t* full(int s) { return bars() + s; }
    __device__ static __forceinline__ uint64_t* empty(int s) { return bars() + tb3d::D + s; }
};

// Work items: tiles x z-runs of zc planes over the owned planes [zlo, zhi)
// (the whole grid, or a slab's owned planes between its deep ghost planes).
struct Tb3Items {
    int tiles_x, ntiles, zc, items, zlo, zhi;
};

__device__ __forceinline__ void fma_sq_if(double& acc, double r, bool cond) {
    asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p fma.rn.f64 %0, %1, %1, %0;\n\t}"
        : "+d"(acc)
        : "d"(r), "r"((unsigned)cond));
}

__device__ __forceinline__ void lds_pair(double (&d)[2], const double* p) {
    SRJ_ASSERT_SMEM(p, 16, tb3_smem);
    const double2 v = *reinterpret_cast<const double2*>(p);
    d[0] = v.x;
    d[1] = v.y;
}

// Load cursor: the next (item, plane) to stage, in the order the warps
// consume them.  Thread 0 keeps it; `ld` numbers loads over the kernel's life.
// Plane steps of an item [z0, z1): the wavefront's two-plane lead-in and
// lead-out, rounded up to even (the step loop alternates two state sets).
__device__ __forceinline__ int tb3_steps(int z0, int z1) { return (z1 - z0 + 5) & ~1; }

struct Tb3Cursor {
    int item, z, zend, ox, oy;
};

__device__ __forceinline__ void tb3_cursor_at(Tb3Cursor& c, const Tb3Items& it, int nz, int item) {
    c.item = item;
    if (item < it.items) {
        const int tile = item % it.ntiles, zci = item / it.ntiles;
        c.ox = (tile % it.tiles_x) * tb3d::TX;
        c.oy = (tile / it.tiles_x) * tb3d::TY;
        const int z0 = it.zlo + zci * it.zc, z1 = min(z0 + it.zc, it.zhi);
        c.z = z0 - 2;
        c.zend = z0 - 2 + tb3_steps(z0, z1) - 1;
    }
}

// Stage load number `ld` (thread 0): wait until its stage is free (load ld-D
// released by every warp), then start the x and b boxes of the cursor's plane
// on the stage's full barrier.
__device__ __forceinline__ void tb3_issue(Tb3Cursor& c, const Tb3Items& it, int nz,
                                          const CUtensorMap* tm_x, const CUtensorMap* tm_b,
                                          uint32_t ld) {
    using namespace tb3d;
    using R = Tb3Ring;
    const int sx = ld % D;
    if (ld >= (uint32_t)D) mbar_wait(R::empty(sx), ((ld / D) - 1) & 1u);
    fence_proxy_async();
    mbar_expect_tx(R::full(sx), TX_BYTES);
    // x map spans the ghost planes (tensor plane p+1 = interior plane p);
    // planes beyond the ghosts only feed discarded ring values.
    const int zx = min(max(c.z, -1), nz) + 1;
    const int zb = min(max(c.z, 0), nz - 1);
    tma_load_3d(R::xs(sx), tm_x, c.ox - S, c.oy - S, zx, R::full(sx));
    tma_load_3d(R::bs(sx), tm_b, c.ox - S, c.oy - 1, zb, R::full(sx));
    if (++c.z > c.zend) tb3_cursor_at(c, it, nz, c.item + gridDim.x);
}

// Streaming state of level 2: per point of the previous plane, x and the
// partial sum ypart (p = c_off*x is recomputed).  Level 1 keeps only ypart:
// its previous plane is still staged in shared memory.
struct Tb3L1 {
    double y[tb3d::V + 2][tb3d::CW];
};
struct Tb3L2 {
    double x[tb3d::V][tb3d::CW], y[tb3d::V][tb3d::CW];
};

// Per-item constants of a thread.
struct Tb3Pt {
    int r0, c0, nx, ny;
    unsigned rowg;    // level-1 rows u on a Dirichlet ghost row (gy == -1 or ny): x_{k0+1} := 0
    unsigned rowacc;  // level-1 rows u = 1..V inside the grid (accumulated and stored)
    bool own0, own1;  // owned, in-grid columns
    bool gup, gdown;  // column 1 is the ghost column -1 / column 0 is the ghost column nx
    long long rowoff;  // flat offset of grid row oy + r0, column gx0
};

// A lane's column pair is owned / inside the grid as a whole (even nx, even
// box origin and ring), so own0 == own1: one predicated 16-byte store.
__device__ __forceinline__ void st_row(double* row, double v0, double v1, bool o0, bool) {
    if (o0) *reinterpret_cast<double2*>(row) = make_double2(v0, v1);
}

// One plane step.  Level 1 reads plane z of x_{k0} from stage n, finishes
// plane z-1 of x_{k0+1}; level 2 (H == 2) takes that plane and finishes plane
// z-2 of x_{k0+2}.  State moves from (i1, i2) to (o1, o2): the caller alternates
// two state sets, so no register copies are needed between steps.
// MAIN: a step inside the item (both finished planes owned and inside the grid,
// ny % V == 0), where residuals accumulate unconditionally into per-column
// sums (masked per item) and the only Dirichlet fix-ups are the ghost rows
// -1 / ny (halo rows u = 0 / V+1) and the ghost columns -1 / nx (shuffles);
// otherwise every ownership and ghost condition is tested.
template <int H, bool MAIN>
__device__ __forceinline__ void tb3_step(const Tb3Pt& t, int s, uint32_t n, int z, int z0, int z1,
                                         int nz, long long pl, double coff, double cdiag,
                                         double inv, double w0, double w1, bool accumulate,
                                         double* __restrict__ xout,
                                         const Tb3L1& i1, Tb3L1& o1, const Tb3L2& i2, Tb3L2& o2,
                                         double (&sq)[2][2]) {
    using namespace tb3d;
    using R = Tb3Ring;
    const int lane = threadIdx.x & 31;
    // ---- level-0 input: plane z of x (tile rows r0-2 .. r0+V+1) from stage n,
    // plane z-1 (tile rows r0-1 .. r0+V) still in stage n-1
    const int sn = n % D, sp = (n + D - 1) % D, spp = (n + D - 2) % D;
    double xn[V + 4][CW];
    {
        mbar_wait(R::full(sn), (n / D) & 1u);
        const double* xs = R::xs(sn) + t.r0 * RX + t.c0;
#pragma unroll
        for (int u = 0; u < V + 4; ++u) lds_pair(xn[u], xs + u * RX);
    }
    double pn[V + 4][CW];
#pragma unroll
    for (int u = 0; u < V + 4; ++u)
#pragma unroll
        for (int j = 0; j < CW; ++j) pn[u][j] = DMUL(coff, xn[u][j]);
    // ---- level 1
    const bool a1 = accumulate && z - 1 >= z0 && z - 1 < z1;
    double x1n[V + 2][CW];
    {
        double bb[V + 2][CW], xq[V + 2][CW], xw[V + 2], xe[V + 2];
        {
            const double* bs = R::bs(sp) + t.r0 * RX + t.c0;
            const double* xs = R::xs(sp) + (t.r0 + 1) * RX + t.c0;
            // x-neighbours of the new plane straight from the stage (the pairs
            // left and right of the lane's two columns; lanes 0 / 31 read ring
            // garbage from the adjacent row, never used for an owned point)
            const double* xc = R::xs(sn) + (t.r0 + 1) * RX + t.c0;
#pragma unroll
            for (int u = 0; u < V + 2; ++u) {
                lds_pair(bb[u], bs + u * RX);
                lds_pair(xq[u], xs + u * RX);
                double l[2], r[2];
                lds_pair(l, xc + u * RX - 2);
                lds_pair(r, xc + u * RX + 2);
                xw[u] = l[1];
                xe[u] = r[0];
            }
        }
#pragma unroll
        for (int u = 0; u < V + 2; ++u) {
            const double pw = DMUL(coff, xw[u]);
            const double pe = DMUL(coff, xe[u]);
#pragma unroll
            for (int j = 0; j < CW; ++j) {
                const double y = DADD(i1.y[u][j], pn[u + 1][j]);
                const double rr = DSUB(bb[u][j], y);
                x1n[u][j] = relax(xq[u][j], inv, rr, w0);
                if (u >= 1 && u <= V) {
                    if constexpr (MAIN)
                        sq[0][j] = fma(rr, rr, sq[0][j]);
                    else if (a1 && ((t.rowacc >> u) & 1u))
                        sq[0][j] = fma(rr, rr, sq[0][j]);
                }
                double yp = DADD(DMUL(coff, xq[u][j]), pn[u][j]);
                yp = DADD(yp, j == 0 ? pw : pn[u + 1][0]);
                yp = DADD(yp, DMUL(cdiag, xn[u + 1][j]));
                yp = DADD(yp, j == CW - 1 ? pe : pn[u + 1][1]);
                o1.y[u][j] = DADD(yp, pn[u + 2][j]);
            }
        }
        // Dirichlet: ghost planes and ghost rows of x_{k0+1} are zero
        if constexpr (!MAIN) {
            if (z - 1 < 0 || z - 1 >= nz) {
#pragma unroll
                for (int u = 0; u < V + 2; ++u) x1n[u][0] = x1n[u][1] = 0.0;
            } else if (t.rowg) {
#pragma unroll
                for (int u = 0; u < V + 2; ++u)
                    if ((t.rowg >> u) & 1u) x1n[u][0] = x1n[u][1] = 0.0;
            }
        }
    }
    if constexpr (H == 1) {
        if (xout && z - 1 >= z0 && z - 1 < z1) {
            double* base = xout + (long long)(z - 1) * pl + t.rowoff;
#pragma unroll
            for (int v = 0; v < V; ++v)
                if ((t.rowacc >> (v + 1)) & 1u)
                    st_row(base + (long long)v * t.nx, x1n[v + 1][0], x1n[v + 1][1], t.own0, t.own1);
        }
        __syncwarp();
        if (lane == 0 && s >= 2) mbar_arrive(R::empty(spp));
        return;
    }
    // ---- level 2
    const bool a2 = accumulate && z - 2 >= z0 && z - 2 < z1;
    double p1[V + 2][CW];
#pragma unroll
    for (int u = 0; u < V + 2; ++u)
#pragma unroll
        for (int j = 0; j < CW; ++j) p1[u][j] = DMUL(coff, x1n[u][j]);
    if constexpr (MAIN) {
        // ghost rows of x_{k0+1} enter level 2 only as y-neighbour products
#pragma unroll
        for (int j = 0; j < CW; ++j) {
            p1[0][j] = (t.rowg & 1u) ? -0.0 : p1[0][j];
            p1[V + 1][j] = (t.rowg >> (V + 1)) ? -0.0 : p1[V + 1][j];
        }
    }
    double bb[V][CW];
    {
        const double* bs = R::bs(spp) + (t.r0 + 1) * RX + t.c0;
#pragma unroll
        for (int v = 0; v < V; ++v) lds_pair(bb[v], bs + v * RX);
    }
    // stage n-2: its x plane was last read in step n-1, its b plane just now
    __syncwarp();
    if (lane == 0 && s >= 2) mbar_arrive(R::empty(spp));
    double xo[V][CW];
#pragma unroll
    for (int v = 0; v < V; ++v) {
        // ghost columns -1 / nx of x_{k0+1} enter only through the shuffles
        const double su = t.gup ? -0.0 : p1[v + 1][1];
        const double sd = t.gdown ? -0.0 : p1[v + 1][0];
        const double pw = shfl_up_d(su, 1);
        const double pe = shfl_down_d(sd, 1);
#pragma unroll
        for (int j = 0; j < CW; ++j) {
            const double y = DADD(i2.y[v][j], p1[v + 1][j]);
            const double rr = DSUB(bb[v][j], y);
            xo[v][j] = relax(i2.x[v][j], inv, rr, w1);
            if constexpr (MAIN)
                sq[1][j] = fma(rr, rr, sq[1][j]);
            else if (a2 && ((t.rowacc >> (v + 1)) & 1u))
                sq[1][j] = fma(rr, rr, sq[1][j]);
            double yp = DADD(DMUL(coff, i2.x[v][j]), p1[v][j]);
            yp = DADD(yp, j == 0 ? pw : p1[v + 1][0]);
            yp = DADD(yp, DMUL(cdiag, x1n[v + 1][j]));
            yp = DADD(yp, j == CW - 1 ? pe : p1[v + 1][1]);
            o2.y[v][j] = DADD(yp, p1[v + 2][j]);
            o2.x[v][j] = x1n[v + 1][j];
        }
    }
    if (MAIN ? t.rowacc != 0u : (z - 2 >= z0 && z - 2 < z1)) {
        double* base = xout + (long long)(z - 2) * pl + t.rowoff;
#pragma unroll
        for (int v = 0; v < V; ++v)
            if (MAIN || ((t.rowacc >> (v + 1)) & 1u))
                st_row(base + (long long)v * t.nx, xo[v][0], xo[v][1], t.own0, t.own1);
    }
}

// Compute warps: one pass of H (1 or 2) sub-sweeps over this CTA's items.
template <int H>
__device__ __forceinline__ void tb3_consume(const TbArgs& a, const Tb3Items& it,
                                            const CUtensorMap* tm_x, const CUtensorMap* tm_b,
                                            double* __restrict__ xout, const double* omegas,
                                            bool accumulate, double (&acc)[tb3d::S],
                                            uint32_t& ld) {
    using namespace tb3d;
    using R = Tb3Ring;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nx = a.g.nx, ny = a.g.ny, nz = a.g.nz;
    const long long pl = (long long)nx * ny;
    const double coff = a.g.c_off, cdiag = a.g.c_diag, inv = a.g.inv_diag;
    const double w0 = __ldg(omegas), w1 = H > 1 ? __ldg(omegas + 1) : 0.0;
    const bool issuer = threadIdx.x == 0;
    Tb3Cursor cur;
    uint32_t iss = ld;  // next load number to issue (thread 0)
    if (issuer) {
        tb3_cursor_at(cur, it, nz, blockIdx.x);
        // prologue: two planes ahead
        for (int q = 0; q < 2 && cur.item < it.items; ++q) tb3_issue(cur, it, nz, tm_x, tm_b, iss++);
    }
    Tb3Pt t;
    t.r0 = warp * V;
    t.c0 = lane * CW;
    t.nx = nx;
    t.ny = ny;
    for (int item = blockIdx.x; item < it.items; item += gridDim.x) {
        const int tile = item % it.ntiles, zci = item / it.ntiles;
        const int ox = (tile % it.tiles_x) * TX, oy = (tile / it.tiles_x) * TY;
        const int z0 = it.zlo + zci * it.zc, z1 = min(z0 + it.zc, it.zhi);
        const int gx0 = ox - S + t.c0;  // grid column of this lane's first point
        t.rowg = t.rowacc = 0u;
#pragma unroll
        for (int u = 0; u < V + 2; ++u) {
            const int gy = oy + t.r0 - 1 + u;  // level-1 row u
            if (gy == -1 || gy == ny) t.rowg |= 1u << u;
            if (u >= 1 && u <= V && gy < ny) t.rowacc |= 1u << u;
        }
        t.own0 = t.c0 >= S && t.c0 < S + TX && gx0 < nx;
        t.own1 = t.c0 + 1 >= S && t.c0 + 1 < S + TX && gx0 + 1 < nx;
        t.gup = gx0 + 1 == -1;
        t.gdown = gx0 == nx;
        t.rowoff = (long long)(oy + t.r0) * nx + gx0;
        Tb3L1 A1, B1;
        Tb3L2 A2, B2;
#pragma unroll
        for (int u = 0; u < V + 2; ++u)
#pragma unroll
            for (int j = 0; j < CW; ++j) A1.y[u][j] = 0.0;
#pragma unroll
        for (int v = 0; v < V; ++v)
#pragma unroll
            for (int j = 0; j < CW; ++j) A2.x[v][j] = A2.y[v][j] = 0.0;
        double sq[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
        const uint32_t base = ld;
        const int nsteps = tb3_steps(z0, z1);
        // steps s in [4, z1 - z0 + 2] finish owned planes at both levels
        const int main_end = (H == 2 && accumulate && ny % V == 0) ? z1 - z0 + 3 : 0;
        int s = 0;
        auto pair = [&](auto main_tag) {
            constexpr bool MAINP = decltype(main_tag)::value;
            const uint32_t n = base + s;
            const int z = z0 - 2 + s;
            if (issuer && cur.item < it.items) tb3_issue(cur, it, nz, tm_x, tm_b, iss++);
            tb3_step<H, MAINP>(t, s, n, z, z0, z1, nz, pl, coff, cdiag, inv, w0, w1, accumulate,
                               xout, A1, B1, A2, B2, sq);
            if (issuer && cur.item < it.items) tb3_issue(cur, it, nz, tm_x, tm_b, iss++);
            tb3_step<H, MAINP>(t, s + 1, n + 1, z + 1, z0, z1, nz, pl, coff, cdiag, inv, w0, w1,
                               accumulate, xout, B1, A1, B2, A2, sq);
            s += 2;
        };
        for (; s < 4 && s < nsteps; ) pair(std::false_type());
        for (; s + 2 <= main_end; ) pair(std::true_type());
        for (; s < nsteps; ) pair(std::false_type());
        // per-column sums of the item, masked once by ownership: main steps add
        // the warp's rows unconditionally, which are all inside the grid or
        // (rowacc == 0) all outside it
        const bool o0 = t.own0 && t.rowacc != 0u, o1 = t.own1 && t.rowacc != 0u;
        acc[0] = DADD(acc[0], DADD(o0 ? sq[0][0] : 0.0, o1 ? sq[0][1] : 0.0));
        if (H > 1) acc[1] = DADD(acc[1], DADD(o0 ? sq[1][0] : 0.0, o1 ? sq[1][1] : 0.0));
        // release the stages of the item's last two planes
        __syncwarp();
        if (lane == 0) {
            mbar_arrive(R::empty((base + nsteps - 2) % D));
            mbar_arrive(R::empty((base + nsteps - 1) % D));
        }
        ld = base + nsteps;
    }
}

template <bool SLAB, bool SOLVE>
__global__ void __launch_bounds__(tb3d::THREADS, 1)
    k_tb3d_cycle(const __grid_constant__ CUtensorMap tm_x0, const __grid_constant__ CUtensorMap tm_x1,
                 const __grid_constant__ CUtensorMap tm_b, TbArgs a, Tb3Items it) {
    using namespace tb3d;
    using R = Tb3Ring;
    if (threadIdx.x == 0) {
        for (int s = 0; s < D; ++s) {
            mbar_init(R::full(s), 1);
            mbar_init(R::empty(s), NW);
        }
        prefetch_tensormap(&tm_x0);
        prefetch_tensormap(&tm_x1);
        prefetch_tensormap(&tm_b);
    }
    __syncthreads();
    uint32_t ld = 0;
    const CUtensorMap* const tmx[2] = {&tm_x0, &tm_x1};
    auto pass = [&](int in, double* xout, const double* om, int h, double (&acc)[S],
                    bool accumulate, bool) __attribute__((always_inline)) {
        if (h == 2)
            tb3_consume<2>(a, it, tmx[in], &tm_b, xout, om, accumulate, acc, ld);
        else  // h = 1, or h = 0 (xout == nullptr): residual of the cycle's final iterate
            tb3_consume<1>(a, it, tmx[in], &tm_b, xout, om, accumulate, acc, ld);
    };
    if constexpr (SOLVE)
        tb_run_solve<S, F3D, true>(a, (int)blockIdx.x < it.items, pass, [](int) {}, []() {});
    else
        tb_run_cycle<S, F3D, SLAB, !SLAB>(a, (int)blockIdx.x < it.items, pass, [](int) {}, []() {});
}

// ----------------------------------------------------------------------------
// Host side
// ----------------------------------------------------------------------------

// Planes per work item: minimise rounds x (zc + 4), the 4 being the two-plane
// lead-in and lead-out of the wavefront.
static int tb3_choose_zc(int ntiles, int slots, int nz) {
    int best_zc = nz;
    double best = 1e300;
    for (int zc = 8; zc <= std::max(8, nz); zc += 8) {
        const int nzc = (nz + zc - 1) / zc;
        const long long items = (long long)ntiles * nzc;
        const long long rounds = (items + slots - 1) / slots;
        const double cost = (double)rounds * (std::min(zc, nz) + 4);
        if (cost < best) { best = cost; best_zc = zc; }
        if (zc >= nz) break;
    }
    return std::max(1, std::min(best_zc, nz));
}

template <bool SLAB, bool SOLVE>
static cudaError_t tb3_attr() {
    return cudaFuncSetAttribute(k_tb3d_cycle<SLAB, SOLVE>,
                                cudaFuncAttributeMaxDynamicSharedMemorySize, (int)tb3d::SMEM);
}

cudaError_t tb3_plan_init(Tb3Plan& plan, const Geom& g, int num_sms) {
    plan = Tb3Plan();
    // TMA needs a 16-byte row pitch (even nx).
    if (g.fam != F3D || (g.nx & 1) || !tma_available()) return cudaSuccess;
    cudaError_t e;
    if ((e = tb3_attr<false, false>()) != cudaSuccess || (e = tb3_attr<true, false>()) != cudaSuccess ||
        (e = tb3_attr<false, true>()) != cudaSuccess)
        return e;
    int per_sm = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tb3d_cycle<false, false>,
                                                           tb3d::THREADS, tb3d::SMEM)) != cudaSuccess)
        return e;
    if (per_sm < 1) return cudaSuccess;
    plan.num_sms = num_sms;
    plan.tiles_x = (g.nx + tb3d::TX - 1) / tb3d::TX;
    plan.ntiles = plan.tiles_x * ((g.ny + tb3d::TY - 1) / tb3d::TY);
    plan.zc = tb3_choose_zc(plan.ntiles, num_sms, g.nz);
    if (const char* v = getenv("SRJ_TB3_ZC")) plan.zc = std::max(1, std::min(atoi(v), g.nz));  // tuning
    plan.items = plan.ntiles * ((g.nz + plan.zc - 1) / plan.zc);
    plan.blocks = std::max(1, std::min(num_sms, plan.items));
    plan.sweeps = tb3d::S;
    plan.supported = true;
    return cudaSuccess;
}

cudaError_t tb3_launch_cycle(const Tb3Plan& plan, const Geom& g, double* x, double* x_alt,
                             const double* b, const double* omegas, int M, double tol,
                             double baseline, double* partials, double* hist, int* out_i,
                             double* out_d, cudaStream_t st, int z_lo, int z_hi, double* sums,
                             const SolveCtl* ctl) {
    if ((((uintptr_t)x | (uintptr_t)x_alt | (uintptr_t)b) & 15) != 0)
        return cudaErrorMisalignedAddress;
    const long long plane = (long long)g.nx * g.ny;
    CUtensorMap m0, m1, mb;
    cudaError_t e;
    // x maps span the ghost planes: base one plane before the interior
    if ((e = encode_volume_map(&m0, x - plane, g.nx, g.ny, g.nz + 2, tb3d::RX, tb3d::XROWS)) != cudaSuccess)
        return e;
    if ((e = encode_volume_map(&m1, x_alt - plane, g.nx, g.ny, g.nz + 2, tb3d::RX, tb3d::XROWS)) != cudaSuccess)
        return e;
    if ((e = encode_volume_map(&mb, b, g.nx, g.ny, g.nz, tb3d::RX, tb3d::BROWS)) != cudaSuccess)
        return e;
    TbArgs a;
    a.ctl = ctl ? *ctl : SolveCtl{};
    a.g = g;
    a.buf0 = x;
    a.buf1 = x_alt;
    a.b = b;
    a.omegas = omegas;
    a.M = M;
    a.s = tb3d::S;
    a.tol = tol;
    a.baseline = baseline;
    a.partials = partials;
    a.hist = hist;
    a.out_i = out_i;
    a.out_d = out_d;
    a.tiles_x = plan.tiles_x;
    a.ntiles = plan.ntiles;
    a.row_lo = z_lo;
    a.row_hi = z_hi;
    a.sums = sums;
    Tb3Items it;
    it.tiles_x = plan.tiles_x;
    it.ntiles = plan.ntiles;
    it.zlo = z_lo;
    it.zhi = z_hi;
    if (z_lo == 0 && z_hi == g.nz) {
        it.zc = plan.zc;
        it.items = plan.items;
    } else {
        const int nzr = z_hi - z_lo;
        it.zc = tb3_choose_zc(plan.ntiles, plan.num_sms, nzr);
        it.items = plan.ntiles * ((nzr + it.zc - 1) / it.zc);
    }
    const int blocks = std::max(1, std::min(plan.num_sms - plan.reserved, it.items));
    void* args[] = {&m0, &m1, &mb, &a, &it};
    const void* fn = sums  ? (const void*)k_tb3d_cycle<true, false>
                     : ctl ? (const void*)k_tb3d_cycle<false, true>
                           : (const void*)k_tb3d_cycle<false, false>;
    return cudaLaunchCooperativeKernel(fn, dim3(blocks), dim3(tb3d::THREADS), args, tb3d::SMEM, st);
}

}  // namespace srj
