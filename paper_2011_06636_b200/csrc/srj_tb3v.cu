// Temporally blocked SRJ cycle for the 3D 7-point VARIABLE-coefficient stencil:
// two consecutive sweeps, each with its own omega, per HBM round trip of x,
// b and the three face arrays (the one-sweep plane ring, srj_3dv.cu, streams
// at the HBM roofline; this halves its DRAM bytes per point-sweep).
//
// Operator and arithmetic exactly as srj_3dv.cu (reference csr_matvec order,
// diagonal = the six-face sum in the order west, east, south, north, bottom,
// top, 1/diag a correctly rounded reciprocal), so iterates are bit-identical.
//
// Work item = a 60 x 14 owned tile over a run of planes [z0, z1); level 1
// (sweep 1) runs on the 64 x 16 region around it (a one-point ring, two
// columns each side to keep the boxes 16-byte aligned), level 2 (sweep 2) on
// the owned points.  Thread (lane, warp) owns region columns 2*lane, 2*lane+1
// of row `warp` for the whole item and streams in z with its values in
// registers: x of planes p-1 and p (level 1 at step z = p+1 loads only the new
// plane p+1 and the in-plane neighbours), its faces, diagonal, 1/diagonal and
// b of plane p, and its level-1 results of planes p-1, p.  Level 2 is split
// like the constant-coefficient wavefront (srj_tb3d.cu): right after level 1
// of plane p has been published (one shared-memory plane, the only values
// another thread needs), every thread adds up the first six terms of its
// level-2 sum for plane p in the reference's column order; one step later the
// seventh (top) term, its own level-1 value of plane p+1, completes it.  One
// block barrier per plane step.  Copy-engine rings two planes ahead:
//   ring A (4 stages, plane p): x plane p (68 x 18 box with a two-point ring;
//          the x map spans the ghost planes) and face_z plane p (64 x 16);
//   ring B (3 stages, plane p): b, face_x (66 x 16 over the 16-byte-pitch
//          copy) and face_y (64 x 17).
// Level-1 values outside the grid and on ghost planes are zero (level 2's
// Dirichlet ghosts).  512 threads, one CTA per SM.
//
// Measured on B200 (level-14 cycle): 512^3 774 us per sweep (173 GLUP/s) vs
// 1,016 for the one-sweep ring; 256^3 112 vs 130 us.  Progression: level 1 and
// level 2 both from shared memory with two barriers per step (v2) 983 us --
// bound by shared-memory bandwidth (~500 B per point pair per step); this
// register-streaming form reads ~250 B and takes one barrier.  A 384-thread
// variant without the 128-register cap's small spills measured 851 us.
//
// Residuals, stopping and rollback: the shared driver (srj_tbdriver.cuh); the
// residual of a cycle's final iterate is a level-1-only pass (h = 0).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "srj_3d.cuh"
#include "srj_stencil.cuh"
#include "srj_tb.cuh"
#include "srj_tbdriver.cuh"
#include "srj_tma.cuh"
#include "srj_walk.cuh"

namespace srj {
namespace tb3v {
constexpr int S = 2;
constexpr int OX = 60, OY = 14;                 // owned tile
constexpr int RX = OX + 4, RY = OY + 2;         // level-1 region 64 x 16 (origin ox-2, oy-1)
constexpr int THREADS = 32 * RY;                // one warp per region row, 2 columns per lane
constexpr int XBX = RX + 4, XBY = RY + 2;       // x box 68 x 18 (origin ox-4, oy-2)
constexpr int XPL = ((XBX * XBY + 15) / 16) * 16;
constexpr int ZPL = RX * RY;                    // face_z box
constexpr int ASTRIDE = XPL + ZPL;              // ring A stage
constexpr int BPL = RX * RY;                    // b box
constexpr int FXW = RX + 2;                     // face_x box width (65 faces, 16-byte multiple)
constexpr int FXPL = ((FXW * RY + 15) / 16) * 16;
constexpr int FYPL = ((RX * (RY + 1) + 15) / 16) * 16;  // face_y box (RY + 1 rows)
constexpr int BSTRIDE = BPL + FXPL + FYPL;      // ring B stage
constexpr int L1PL = RX * RY;                   // published level-1 plane
constexpr int AST = 4, BST = 3, L1ST = 2;
constexpr int NDBL = AST * ASTRIDE + BST * BSTRIDE + L1ST * L1PL;
constexpr size_t SMEM = (size_t)NDBL * sizeof(double) + 8 * (AST + BST);
constexpr uint32_t ABYTES = (XBX * XBY + ZPL) * sizeof(double);
constexpr uint32_t BBYTES = (BPL + FXW * RY + RX * (RY + 1)) * sizeof(double);
static_assert((XPL * 8) % 128 == 0 && (ASTRIDE * 8) % 128 == 0 && (BSTRIDE * 8) % 128 == 0 &&
                  (FXPL * 8) % 128 == 0 && (BPL * 8) % 128 == 0 && (L1PL * 8) % 128 == 0,
              "TMA destinations stay 128-byte aligned");
}  // namespace tb3v

struct Tb3vMaps {
    CUtensorMap x0, x1, b, fx, fy, fz;
};

struct Tb3vItems {
    int tiles_x, ntiles, zc, items;
};

extern __shared__ __align__(128) double tb3v_smem[];

struct Tb3vRing {
    __device__ static __forceinline__ double* a(int s) { return tb3v_smem + s * tb3v::ASTRIDE; }
    __device__ static __forceinline__ double* b(int s) {
        return tb3v_smem + tb3v::AST * tb3v::ASTRIDE + s * tb3v::BSTRIDE;
    }
    __device__ static __forceinline__ double* l1(int s) {
        return tb3v_smem + tb3v::AST * tb3v::ASTRIDE + tb3v::BST * tb3v::BSTRIDE + s * tb3v::L1PL;
    }
    __device__ static __forceinline__ uint64_t* abar(int s) {
        return reinterpret_cast<uint64_t*>(tb3v_smem + tb3v::NDBL) + s;
    }
    __device__ static __forceinline__ uint64_t* bbar(int s) { return abar(tb3v::AST) + s; }
};

// ring A, plane p (x: tensor plane p+1 of the ghost-spanning map; face_z plane p)
__device__ __forceinline__ void tb3v_issue_a(const CUtensorMap* mx, const CUtensorMap* mz, int ox,
                                             int oy, int p) {
    using namespace tb3v;
    const int s = (p + 1) & (AST - 1);
    double* st = Tb3vRing::a(s);
    fence_proxy_async();
    mbar_expect_tx(Tb3vRing::abar(s), ABYTES);
    tma_load_3d(st, mx, ox - 4, oy - 2, p + 1, Tb3vRing::abar(s));
    tma_load_3d(st + XPL, mz, ox - 2, oy - 1, p, Tb3vRing::abar(s));
}

// ring B, plane p: b, face_x, face_y
__device__ __forceinline__ void tb3v_issue_b(const Tb3vMaps& m, int ox, int oy, int p) {
    using namespace tb3v;
    const int s = (p + 3) % BST;
    double* st = Tb3vRing::b(s);
    fence_proxy_async();
    mbar_expect_tx(Tb3vRing::bbar(s), BBYTES);
    tma_load_3d(st, &m.b, ox - 2, oy - 1, p, Tb3vRing::bbar(s));
    tma_load_3d(st + BPL, &m.fx, ox - 2, oy - 1, p, Tb3vRing::bbar(s));
    tma_load_3d(st + BPL + FXPL, &m.fy, ox - 2, oy - 1, p, Tb3vRing::bbar(s));
}

__device__ __forceinline__ double2 lds2(const double* p) {
    SRJ_ASSERT_SMEM(p, 16, tb3v_smem);
    return *reinterpret_cast<const double2*>(p);
}

// One pass over this CTA's items: H = 2 (two sweeps), 1 (one sweep into
// xout), 0 (residual of the input only, xout == nullptr).
template <int H>
__device__ __forceinline__ void tb3v_pass(const TbArgs& a, const Tb3vItems& it, const Tb3vMaps& m,
                                          const CUtensorMap* mx, double* __restrict__ xout,
                                          const double* om, bool accumulate,
                                          double (&acc)[tb3v::S], uint32_t& aph, uint32_t& bph) {
    using namespace tb3v;
    using R = Tb3vRing;
    const int lane = threadIdx.x & 31, r = threadIdx.x >> 5;  // region row
    const int c0 = 2 * lane;                                  // region columns c0, c0+1
    const int nx = a.g.nx, ny = a.g.ny, nz = a.g.nz;
    const long long plane = (long long)nx * ny;
    const double w0 = H >= 1 ? __ldg(om) : 0.0, w1 = H == 2 ? __ldg(om + 1) : 0.0;
    // owned columns / rows of the tile (region columns 2 .. 61, rows 1 .. 14)
    const bool lane_own = lane >= 1 && lane <= 30, row_own = r >= 1 && r <= OY;
    for (int item = blockIdx.x; item < it.items; item += gridDim.x) {
        const int tile = item % it.ntiles, zci = item / it.ntiles;
        const int ox = (tile % it.tiles_x) * OX, oy = (tile / it.tiles_x) * OY;
        const int z0 = zci * it.zc, z1 = min(z0 + it.zc, nz);
        const int L0 = H == 2 ? z0 - 1 : z0, L1 = H == 2 ? z1 + 1 : z1;  // level-1 planes
        if (threadIdx.x == 0) {
            for (int p = L0 - 1; p <= min(L0 + 2, L1); ++p) tb3v_issue_a(mx, &m.fz, ox, oy, p);
            for (int p = L0; p <= min(L0 + 2, L1 - 1); ++p) tb3v_issue_b(m, ox, oy, p);
        }
        auto wait_a = [&](int p) {
            const int s = (p + 1) & (AST - 1);
            mbar_wait(R::abar(s), (aph >> s) & 1u);
            aph ^= 1u << s;
        };
        auto wait_b = [&](int p) {
            const int s = (p + 3) % BST;
            mbar_wait(R::bbar(s), (bph >> s) & 1u);
            bph ^= 1u << s;
        };
        const int gx = ox - 2 + c0, gy = oy - 1 + r;  // grid point of column c0
        const bool in0 = gx >= 0 && gx < nx && gy >= 0 && gy < ny;
        const bool in1 = gx + 1 >= 0 && gx + 1 < nx && gy >= 0 && gy < ny;
        // owned column pair (even nx: both or neither inside the grid)
        const bool own = lane_own && row_own && gx < nx && gy < ny;
        const int xb_i = (r + 1) * XBX + c0 + 2;  // x box index of (c0, r)
        const int ri = r * RX + c0;               // region index of (c0, r)
        // streamed registers of the thread's two points
        double X0[2], X1[2], fzb[2];              // x(p-1), x(p), face_z(p)
        double Lp[2] = {0.0, 0.0};                // level-1 value of plane p-1
        double yp2[2], ct2[2], iv2[2], b2[2], lc2[2];  // level-2 partial of plane p-1
        wait_a(L0 - 1);
        wait_a(L0);
        {
            const double2 v0 = lds2(R::a(L0 & (AST - 1)) + xb_i);         // x(L0 - 1)
            const double2 v1 = lds2(R::a((L0 + 1) & (AST - 1)) + xb_i);   // x(L0)
            const double2 f1 = lds2(R::a((L0 + 1) & (AST - 1)) + XPL + ri);  // face_z(L0)
            X0[0] = v0.x; X0[1] = v0.y;
            X1[0] = v1.x; X1[1] = v1.y;
            fzb[0] = f1.x; fzb[1] = f1.y;
        }
        for (int z = L0 + 1; z <= L1; ++z) {
            const int p = z - 1;  // level-1 plane of this step
            wait_a(z);
            wait_b(p);
            const double* ac = R::a((p + 1) & (AST - 1));  // plane p: x neighbours
            const double* at = R::a((z + 1) & (AST - 1));  // plane p+1: x, face_z
            const double* sb = R::b((p + 3) % BST);
            // ---- level 1 of plane p at the thread's two points
            const double2 xt = lds2(at + xb_i);
            const double2 fzt = lds2(at + XPL + ri);
            const double2 xwp = lds2(ac + xb_i - 2), xep = lds2(ac + xb_i + 2);
            const double2 xs = lds2(ac + xb_i - XBX), xnn = lds2(ac + xb_i + XBX);
            const double2 bb = lds2(sb + ri);
            const double* sfx = sb + BPL + r * FXW + c0;
            const double2 fx01 = lds2(sfx);
            const double fx2 = sfx[2];
            const double2 fys = lds2(sb + BPL + FXPL + ri), fyn = lds2(sb + BPL + FXPL + ri + RX);
            const double cw[2] = {fx01.x, fx01.y}, ce[2] = {fx01.y, fx2};
            const double cs[2] = {fys.x, fys.y}, cn[2] = {fyn.x, fyn.y};
            const double ct[2] = {fzt.x, fzt.y};
            const double xw[2] = {xwp.y, X1[0]}, xe[2] = {X1[1], xep.x};
            const double xsv[2] = {xs.x, xs.y}, xnv[2] = {xnn.x, xnn.y}, xtv[2] = {xt.x, xt.y};
            const double bv[2] = {bb.x, bb.y};
            const bool plane_in = p >= 0 && p < nz;
            const bool plane_own = p >= z0 && p < z1;
            double d[2], iv[2], l1[2];
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                d[j] = DADD(DADD(DADD(DADD(DADD(cw[j], ce[j]), cs[j]), cn[j]), fzb[j]), ct[j]);
                double y = DADD(0.0, DMUL(-fzb[j], X0[j]));
                y = DADD(y, DMUL(-cs[j], xsv[j]));
                y = DADD(y, DMUL(-cw[j], xw[j]));
                y = DADD(y, DMUL(d[j], X1[j]));
                y = DADD(y, DMUL(-ce[j], xe[j]));
                y = DADD(y, DMUL(-cn[j], xnv[j]));
                y = DADD(y, DMUL(-ct[j], xtv[j]));
                const double rr = DSUB(bv[j], y);
                iv[j] = __drcp_rn(d[j]);
                const double xn = relax(X1[j], iv[j], rr, w0);
                const bool inj = plane_in && (j == 0 ? in0 : in1);
                l1[j] = inj ? xn : 0.0;
                if (accumulate && own && plane_own) acc[0] = fma(rr, rr, acc[0]);
            }
            if constexpr (H == 2) {
                *reinterpret_cast<double2*>(R::l1((p + 2) & 1) + ri) = make_double2(l1[0], l1[1]);
                // finish level 2 of plane p-1: the top term is this level-1 value
                if (own && p - 1 >= z0 && p - 1 < z1) {
                    double xo[2];
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        const double y = DADD(yp2[j], DMUL(-ct2[j], l1[j]));
                        const double rr = DSUB(b2[j], y);
                        xo[j] = relax(lc2[j], iv2[j], rr, w1);
                        if (accumulate) acc[1] = fma(rr, rr, acc[1]);
                    }
                    SRJ_ASSERT(gx + 1 < nx && gy < ny && p - 1 < nz);
                    *reinterpret_cast<double2*>(xout + (long long)(p - 1) * plane + (long long)gy * nx + gx) =
                        make_double2(xo[0], xo[1]);
                }
            } else if constexpr (H == 1) {
                if (own && plane_own) {
                    SRJ_ASSERT(gx + 1 < nx && gy < ny && p < nz);
                    *reinterpret_cast<double2*>(xout + (long long)p * plane + (long long)gy * nx + gx) =
                        make_double2(l1[0], l1[1]);
                }
            }
            __syncthreads();  // level-1 plane p published; stages of plane p-1 (A) / p (B) free
            if constexpr (H == 2) {
                // first six level-2 terms of plane p (bottom, south, west, diag, east, north)
                if (own && plane_own) {
                    const double* lp = R::l1((p + 2) & 1);
                    const double2 ls = lds2(lp + ri - RX), ln = lds2(lp + ri + RX);
                    const double2 lw = lds2(lp + ri - 2), le = lds2(lp + ri + 2);
                    const double lsv[2] = {ls.x, ls.y}, lnv[2] = {ln.x, ln.y};
                    const double lwv[2] = {lw.y, l1[0]}, lev[2] = {l1[1], le.x};
#pragma unroll
                    for (int j = 0; j < 2; ++j) {
                        double y = DADD(0.0, DMUL(-fzb[j], Lp[j]));
                        y = DADD(y, DMUL(-cs[j], lsv[j]));
                        y = DADD(y, DMUL(-cw[j], lwv[j]));
                        y = DADD(y, DMUL(d[j], l1[j]));
                        y = DADD(y, DMUL(-ce[j], lev[j]));
                        yp2[j] = DADD(y, DMUL(-cn[j], lnv[j]));
                        ct2[j] = ct[j];
                        iv2[j] = iv[j];
                        b2[j] = bv[j];
                        lc2[j] = l1[j];
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 2; ++j) {
                Lp[j] = l1[j];
                X0[j] = X1[j];
                X1[j] = xtv[j];
                fzb[j] = ct[j];
            }
            if (threadIdx.x == 0) {
                if (z + 2 <= L1) tb3v_issue_a(mx, &m.fz, ox, oy, z + 2);
                if (z + 2 <= L1 - 1) tb3v_issue_b(m, ox, oy, z + 2);
            }
        }
        __syncthreads();  // the next item's prologue reuses the rings
    }
}

template <bool SOLVE>
__global__ void __launch_bounds__(tb3v::THREADS, 1)
    k_tb3v_cycle(const __grid_constant__ Tb3vMaps m, TbArgs a, Tb3vItems it) {
    using namespace tb3v;
    using R = Tb3vRing;
    if (threadIdx.x == 0) {
        for (int s = 0; s < AST; ++s) mbar_init(R::abar(s), 1);
        for (int s = 0; s < BST; ++s) mbar_init(R::bbar(s), 1);
        prefetch_tensormap(&m.x0);
        prefetch_tensormap(&m.x1);
        prefetch_tensormap(&m.b);
        prefetch_tensormap(&m.fx);
        prefetch_tensormap(&m.fy);
        prefetch_tensormap(&m.fz);
    }
    __syncthreads();
    uint32_t aph = 0, bph = 0;
    const CUtensorMap* const tmx[2] = {&m.x0, &m.x1};
    auto pass = [&](int in, double* xout, const double* om, int h, double (&acc)[S],
                    bool accumulate, bool) __attribute__((always_inline)) {
        if (h == 2)
            tb3v_pass<2>(a, it, m, tmx[in], xout, om, accumulate, acc, aph, bph);
        else if (h == 1)
            tb3v_pass<1>(a, it, m, tmx[in], xout, om, accumulate, acc, aph, bph);
        else  // residual of the cycle's final iterate
            tb3v_pass<0>(a, it, m, tmx[in], nullptr, om, true, acc, aph, bph);
    };
    if constexpr (SOLVE)
        tb_run_solve<S, F3DV, true>(a, (int)blockIdx.x < it.items, pass, [](int) {}, []() {});
    else
        tb_run_cycle<S, F3DV, false, true>(a, (int)blockIdx.x < it.items, pass, [](int) {},
                                           []() {});
}

// ----------------------------------------------------------------------------
// Host side
// ----------------------------------------------------------------------------

cudaError_t tb3v_plan_init(Tb3vPlan& plan, const Geom& g, int num_sms, const double* fx_pad,
                           int fx_pitch) {
    plan = Tb3vPlan();
    if (g.fam != F3DV || (g.nx & 1) || !fx_pad || !tma_available()) return cudaSuccess;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_tb3v_cycle<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)tb3v::SMEM)) != cudaSuccess ||
        (e = cudaFuncSetAttribute(k_tb3v_cycle<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)tb3v::SMEM)) != cudaSuccess)
        return e;
    int per_sm = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_tb3v_cycle<false>,
                                                           tb3v::THREADS, tb3v::SMEM)) != cudaSuccess)
        return e;
    if (per_sm < 1) return cudaSuccess;
    plan.fx_pad = fx_pad;
    plan.fx_pitch = fx_pitch;
    plan.tiles_x = (g.nx + tb3v::OX - 1) / tb3v::OX;
    plan.ntiles = plan.tiles_x * ((g.ny + tb3v::OY - 1) / tb3v::OY);
    // planes per item: minimise rounds x (zc + 3) (two extra level-1 planes)
    double best = 1e300;
    plan.zc = g.nz;
    for (int zc = 8; zc <= std::max(8, g.nz); zc += 8) {
        const long long items = (long long)plan.ntiles * ((g.nz + zc - 1) / zc);
        const double cost = (double)((items + num_sms - 1) / num_sms) * (std::min(zc, g.nz) + 3);
        if (cost < best) { best = cost; plan.zc = zc; }
        if (zc >= g.nz) break;
    }
    plan.zc = std::max(1, std::min(plan.zc, g.nz));
    if (const char* v = getenv("SRJ_TB3V_ZC")) plan.zc = std::max(1, std::min(atoi(v), g.nz));
    plan.items = plan.ntiles * ((g.nz + plan.zc - 1) / plan.zc);
    plan.blocks = std::max(1, std::min(num_sms, plan.items));
    plan.supported = true;
    return cudaSuccess;
}

cudaError_t tb3v_launch_cycle(const Tb3vPlan& plan, const Geom& g, double* x, double* x_alt,
                              const double* b, const double* omegas, int M, double tol,
                              double baseline, double* partials, double* hist, int* out_i,
                              double* out_d, cudaStream_t st, const SolveCtl* ctl) {
    using namespace tb3v;
    if ((((uintptr_t)x | (uintptr_t)x_alt | (uintptr_t)b | (uintptr_t)g.fy | (uintptr_t)g.fz) &
         15) != 0)
        return cudaErrorMisalignedAddress;
    const long long plane = (long long)g.nx * g.ny;
    Tb3vMaps m;
    cudaError_t e;
    if ((e = encode_volume_map(&m.x0, x - plane, g.nx, g.ny, g.nz + 2, XBX, XBY)) != cudaSuccess) return e;
    if ((e = encode_volume_map(&m.x1, x_alt - plane, g.nx, g.ny, g.nz + 2, XBX, XBY)) != cudaSuccess)
        return e;
    if ((e = encode_volume_map(&m.b, b, g.nx, g.ny, g.nz, RX, RY)) != cudaSuccess) return e;
    if ((e = encode_volume_map_pitched(&m.fx, plan.fx_pad, g.nx + 1, g.ny, g.nz, plan.fx_pitch, FXW,
                                       RY)) != cudaSuccess)
        return e;
    if ((e = encode_volume_map(&m.fy, g.fy, g.nx, g.ny + 1, g.nz, RX, RY + 1)) != cudaSuccess) return e;
    if ((e = encode_volume_map(&m.fz, g.fz, g.nx, g.ny, g.nz + 1, RX, RY)) != cudaSuccess) return e;
    TbArgs a;
    a.ctl = ctl ? *ctl : SolveCtl{};
    a.g = g;
    a.buf0 = x;
    a.buf1 = x_alt;
    a.b = b;
    a.omegas = omegas;
    a.M = M;
    a.s = S;
    a.tol = tol;
    a.baseline = baseline;
    a.partials = partials;
    a.hist = hist;
    a.out_i = out_i;
    a.out_d = out_d;
    a.tiles_x = plan.tiles_x;
    a.ntiles = plan.ntiles;
    a.row_lo = 0;
    a.row_hi = g.nz;
    a.sums = nullptr;
    Tb3vItems it{plan.tiles_x, plan.ntiles, plan.zc, plan.items};
    void* args[] = {&m, &a, &it};
    const void* fn = ctl ? (const void*)k_tb3v_cycle<true> : (const void*)k_tb3v_cycle<false>;
    return cudaLaunchCooperativeKernel(fn, dim3(plan.blocks), dim3(THREADS), args, SMEM, st);
}

}  // namespace srj
