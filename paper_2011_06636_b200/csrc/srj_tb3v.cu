// Temporally blocked SRJ cycle for the 3D 7-point VARIABLE-coefficient stencil:
// two consecutive sweeps, each with its own omega, per HBM round trip of x,
// b and the three face arrays (the one-sweep plane ring, srj_3dv.cu, streams
// at the HBM roofline; this halves its DRAM bytes per point-sweep).
//
// Operator and arithmetic exactly as srj_3dv.cu (reference csr_matvec order,
// diagonal = the six-face sum in the order west, east, south, north, bottom,
// top, 1/diag a correctly rounded reciprocal), so iterates are bit-identical.
//
// Work item = a 60 x 16 owned tile over a run of planes [z0, z1).  Level 1
// (sweep 1) is computed on the 64 x 18 region around the tile (a one-point
// ring, two columns on each side to keep the boxes 16-byte aligned) and kept
// in a three-plane shared-memory ring; level 2 (sweep 2) reads its seven
// neighbours from that ring and writes the owned points.  Step z (plane z of
// x arrived): level 1 finishes plane z-1, level 2 finishes plane z-2.  Two
// copy-engine rings feed it two planes ahead:
//   ring A (4 stages, plane p): x plane p (68 x 20 box with a two-point ring;
//          the x map spans the ghost planes) and face_z plane p (64 x 18);
//   ring B (3 stages, plane p): b, face_x (66 x 18 over the 16-byte-pitch
//          copy) and face_y (64 x 19).
// 1/diag of the region (a correctly rounded reciprocal per point) is
// computed by level 1 and read back by level 2 of the same plane one step
// later (two-plane ring), so level 2 runs without the reciprocal.
// Level-1 values outside the grid and on ghost planes are forced to zero (they
// are level 2's Dirichlet ghosts).  Two block barriers per step (level 1 ->
// level 2, and before the next step overwrites the level-1 ring slot level 2
// read).  One CTA of 512 threads per SM (222 KB of shared memory).
//
// Residuals, stopping and rollback: the shared driver (srj_tbdriver.cuh); the
// residual of a cycle's final iterate is a level-1-only pass (h = 0).
//
// Measured on B200 (512^3, level 14): 983 us per sweep vs 1,021 for the
// one-sweep ring; solves 131 vs 127 GLUP/s, both at the board power cap -- the
// two-sweep kernel runs at 1.88 GHz (half the DRAM energy) against 1.33 GHz,
// so its fp64 and barrier latency, not DRAM, set its pace.  At 256^3 it is
// slower (114 vs 129: 288 items on 148 SMs).  Opt-in (sweeps_per_pass 2).
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
constexpr int OX = 60, OY = 16;                 // owned tile
constexpr int RX = OX + 4, RY = OY + 2;         // level-1 region 64 x 18 (origin ox-2, oy-1)
constexpr int THREADS = 512;
constexpr int TROWS = THREADS / RX;             // region rows one pass of the threads covers (8)
constexpr int XBX = RX + 4, XBY = RY + 2;       // x box 68 x 20 (origin ox-4, oy-2)
constexpr int XPL = ((XBX * XBY + 15) / 16) * 16;
constexpr int ZPL = RX * RY;                        // face_z box
constexpr int ASTRIDE = XPL + ZPL;                  // ring A stage
constexpr int BPL = RX * RY;                        // b box
constexpr int FXW = RX + 2;                         // 66: face_x box width (65 faces)
constexpr int FXPL = ((FXW * RY + 15) / 16) * 16;
constexpr int FYPL = ((RX * (RY + 1) + 15) / 16) * 16;  // face_y box (RY + 1 rows)
constexpr int BSTRIDE = BPL + FXPL + FYPL;          // ring B stage
constexpr int L1PL = RX * RY;                       // level-1 plane
constexpr int AST = 4, BST = 3, L1ST = 3, IVST = 2;
// + 1/diag of the level-1 region, computed by level 1 and reused by level 2
// one step later (two planes)
constexpr int NDBL = AST * ASTRIDE + BST * BSTRIDE + L1ST * L1PL + IVST * L1PL;
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
    __device__ static __forceinline__ double* iv(int s) {
        return tb3v_smem + tb3v::AST * tb3v::ASTRIDE + tb3v::BST * tb3v::BSTRIDE +
               tb3v::L1ST * tb3v::L1PL + s * tb3v::L1PL;
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
    const int s = (p + 4) & (AST - 1);
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

// Seven-point var-coef update of region point (c, r): centre and neighbours
// from a plane ring whose rows have pitch `pitch` (ctr / dn / up: the point's
// address in planes p, p-1, p+1); faces from the B stage of plane p and the
// face_z planes p (bottom) and p+1 (top).  Returns r, writes x'.
template <bool CACHED>
__device__ __forceinline__ double tb3v_point(const double* ctr, const double* dn, const double* up,
                                             int pitch, const double* sb, int c, int r,
                                             const double* fzb, const double* fzt, double w,
                                             double& xnew, double* ivp) {
    using namespace tb3v;
    const int pi = r * RX + c;
    const double* sfx = sb + BPL;
    const double* sfy = sb + BPL + FXPL;
    const double cw = sfx[r * FXW + c], ce = sfx[r * FXW + c + 1];
    const double cs = sfy[pi], cn = sfy[pi + RX];
    const double cb = fzb[pi], ct = fzt[pi];
    const double d = DADD(DADD(DADD(DADD(DADD(cw, ce), cs), cn), cb), ct);
    const double xc = ctr[0];
    double y = DADD(0.0, DMUL(-cb, dn[0]));
    y = DADD(y, DMUL(-cs, ctr[-pitch]));
    y = DADD(y, DMUL(-cw, ctr[-1]));
    y = DADD(y, DMUL(d, xc));
    y = DADD(y, DMUL(-ce, ctr[1]));
    y = DADD(y, DMUL(-cn, ctr[pitch]));
    y = DADD(y, DMUL(-ct, up[0]));
    const double rr = DSUB(sb[pi], y);
    // level 1 computes 1/diag and parks it; level 2 (same plane, next step)
    // reads it back
    double inv;
    if constexpr (CACHED) {
        inv = ivp[pi];
    } else {
        inv = __drcp_rn(d);
        if (ivp) ivp[pi] = inv;
    }
    xnew = relax(xc, inv, rr, w);
    return rr;
}

// One pass over this CTA's items: H = 2 (two sweeps), 1 (one sweep, xout),
// 0 (residual of the input only, xout == nullptr).
template <int H>
__device__ __forceinline__ void tb3v_pass(const TbArgs& a, const Tb3vItems& it, const Tb3vMaps& m,
                                          const CUtensorMap* mx, double* __restrict__ xout,
                                          const double* om, bool accumulate,
                                          double (&acc)[tb3v::S], uint32_t& aph, uint32_t& bph) {
    using namespace tb3v;
    using R = Tb3vRing;
    const int tid = threadIdx.x;
    const int c = tid & 63, rq = tid >> 6;  // column, first row (rows rq, rq+8, rq+16)
    const int nx = a.g.nx, ny = a.g.ny, nz = a.g.nz;
    const long long plane = (long long)nx * ny;
    const double w0 = H >= 1 ? __ldg(om) : 0.0, w1 = H == 2 ? __ldg(om + 1) : 0.0;
    for (int item = blockIdx.x; item < it.items; item += gridDim.x) {
        const int tile = item % it.ntiles, zci = item / it.ntiles;
        const int ox = (tile % it.tiles_x) * OX, oy = (tile / it.tiles_x) * OY;
        const int z0 = zci * it.zc, z1 = min(z0 + it.zc, nz);
        // level-1 planes [L0, L1)
        const int L0 = H == 2 ? z0 - 1 : z0, L1 = H == 2 ? z1 + 1 : z1;
        if (tid == 0) {
            for (int p = L0 - 1; p <= min(L0 + 2, L1); ++p) tb3v_issue_a(mx, &m.fz, ox, oy, p);
            for (int p = L0; p <= min(L0 + 1, L1 - 1); ++p) tb3v_issue_b(m, ox, oy, p);
        }
        auto wait_a = [&](int p) {
            const int s = (p + 4) & (AST - 1);
            mbar_wait(R::abar(s), (aph >> s) & 1u);
            aph ^= 1u << s;
        };
        auto wait_b = [&](int p) {
            const int s = (p + 3) % BST;
            mbar_wait(R::bbar(s), (bph >> s) & 1u);
            bph ^= 1u << s;
        };
        wait_a(L0 - 1);
        wait_a(L0);
        const int gx = ox - 2 + c;
        const bool colin = gx >= 0 && gx < nx;
        const bool colown = c >= 2 && c <= 61 && gx < nx;
        for (int z = L0 + 1; z <= L1; ++z) {
            const int p1 = z - 1;  // level-1 plane
            wait_a(z);
            wait_b(p1);
            // ---- level 1 over the 64 x 10 region of plane p1
            {
                const double* xm = R::a((p1 - 1 + 4) & (AST - 1));  // x planes p1-1, p1, p1+1
                const double* xc = R::a((p1 + 4) & (AST - 1));
                const double* xp = R::a((p1 + 1 + 4) & (AST - 1));
                const double* sb = R::b((p1 + 3) % BST);
                double* ivp = R::iv((p1 + 2) & 1);
                const bool plane_own = accumulate && p1 >= z0 && p1 < z1;
                const bool plane_in = p1 >= 0 && p1 < nz;
                double* l1 = R::l1((p1 + 3) % 3);
#pragma unroll
                for (int q = 0; q < (RY + TROWS - 1) / TROWS; ++q) {
                    const int r = rq + TROWS * q;
                    if (r < RY) {
                        const int bi = (r + 1) * XBX + c + 2;  // x box index of (c, r)
                        double xnew;
                        const double rr = tb3v_point<false>(xc + bi, xm + bi, xp + bi, XBX, sb, c,
                                                            r, xc + XPL, xp + XPL, w0, xnew,
                                                            H == 2 ? ivp : nullptr);
                        const int gy = oy - 1 + r;
                        const bool in = plane_in && colin && gy >= 0 && gy < ny;
                        const bool own = colown && r >= 1 && r <= OY && gy < ny;
                        if (plane_own && own) acc[0] = fma(rr, rr, acc[0]);
                        if constexpr (H == 2) {
                            l1[r * RX + c] = in ? xnew : 0.0;
                        } else if constexpr (H == 1) {
                            if (own && p1 >= z0 && p1 < z1) {
                                SRJ_ASSERT(gx < nx && gy < ny && p1 < nz);
                                xout[(long long)p1 * plane + (long long)gy * nx + gx] = xnew;
                            }
                        }
                    }
                }
            }
            __syncthreads();
            // ---- level 2 over the owned 60 x 8 tile of plane p2 = z - 2
            if constexpr (H == 2) {
                const int p2 = z - 2;
                if (p2 >= z0) {
                    const double* lm = R::l1((p2 - 1 + 3) % 3);
                    const double* lc = R::l1((p2 + 3) % 3);
                    const double* lp = R::l1((p2 + 1 + 3) % 3);
                    const double* sb = R::b((p2 + 3) % BST);
                    const double* ivp = R::iv((p2 + 2) & 1);
                    const double* fzb = R::a((p2 + 4) & (AST - 1)) + XPL;
                    const double* fzt = R::a((p2 + 1 + 4) & (AST - 1)) + XPL;
#pragma unroll
                    for (int q = 0; q < OY / TROWS; ++q) {
                        const int r = 1 + rq + TROWS * q;  // region rows 1 .. OY
                        const int li = r * RX + c;
                        if (colown) {
                            double xnew;
                            const double rr = tb3v_point<true>(lc + li, lm + li, lp + li, RX, sb,
                                                               c, r, fzb, fzt, w1, xnew,
                                                               const_cast<double*>(ivp));
                            const int gy = oy - 1 + r;
                            if (gy < ny) {
                                if (accumulate) acc[1] = fma(rr, rr, acc[1]);
                                SRJ_ASSERT(gx < nx && p2 < nz);
                                xout[(long long)p2 * plane + (long long)gy * nx + gx] = xnew;
                            }
                        }
                    }
                }
                __syncthreads();  // level-1 slot of plane p2-1 is rewritten next step
            }
            if (tid == 0) {
                // plane z-2's stages are free (ring A: x and face_z; ring B)
                if (z + 2 <= L1) tb3v_issue_a(mx, &m.fz, ox, oy, z + 2);
                if (z + 1 <= L1 - 1) tb3v_issue_b(m, ox, oy, z + 1);
            }
        }
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
