// Plane-streaming SRJ cycle kernel for the 3D 7-point VARIABLE-coefficient
// stencil (north_star: 3D variable-coefficient stencils; operator
// SRJ_STENCIL_3D7_VAR).
//
// Operator (srj.h): off-diagonals -face, diagonal
//     d = (((((c_w + c_e) + c_s) + c_n) + c_b) + c_t)
// (the CSR the golden scripts hand the reference, tests/golden/make_golden.py),
// so one point-sweep is the reference's csr_matvec over ascending columns
//     y = ((((((0 + (-c_b) x_b) + (-c_s) x_s) + (-c_w) x_w) + d x) + (-c_e) x_e)
//          + (-c_n) x_n) + (-c_t) x_t
// with every product and sum rounded on its own, r = b - y and
// x' = x + w (inv r), inv = 1/d correctly rounded (the reference's
// SparseMatrix.inv_diag = 1.0 / diag, sparse.py:42-44) -- recomputed from the
// faces every sweep instead of streamed (8 B per point-sweep less HBM traffic
// for ~10 fp64 instructions).  Absent boundary columns read a zero ghost
// (copy-engine zero fill in x/y, zero ghost planes in z): (-c)*0 = -0 leaves y
// unchanged, so iterates are bit-identical to the reference.
//
// Work item = one 64 x 8 xy tile over a run of zc planes.  Two copy-engine
// rings feed the compute, one plane ahead of it:
//   ring A (4 stages, plane p): x plane p with a one-point halo ring
//          (68 x 10 box; the x map spans the ghost planes) and the face_z
//          plane p (the bottom faces of plane p = the top faces of p-1);
//   ring B (2 stages, plane p): b, face_x (66 x 8 box over a 16-byte-pitch
//          copy of the (nx+1)-wide rows) and face_y (64 x 9 rows).
// HBM traffic per point-sweep: x, b, face_x, face_y, face_z read once, x
// written once = 48 B (halo rings and the two z re-reads come from L2).
// 64 KB of shared memory per CTA: three CTAs per SM.
//
// Cycle protocol as the other one-sweep cycle kernels (srj_3d.cu): residual
// of the INPUT iterate accumulated per CTA, grid barrier, fixed-order
// reduction in every CTA, the reference's per-sweep stop test
// (solver.py:216-222,235-239), a residual-only tail pass for res(x_M).
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "srj_3d.cuh"
#include "srj_stencil.cuh"
#include "srj_tma.cuh"
#include "srj_walk.cuh"

namespace srj {
namespace k3v {
constexpr int TX = 64, TY = 8;
constexpr int THREADS = 256;
constexpr int RSTEP = THREADS / TX;                 // 4 rows apart
constexpr int RPT = TY / RSTEP;                     // rows per thread (2)
constexpr int XOFF = 2;                             // box column of the tile's first point
constexpr int BX = TX + 2 * XOFF, BY = TY + 2;      // x box with the one-point halo ring
constexpr int FXW = TX + 2;                         // face_x box width (65 faces, 16-byte multiple)
constexpr int FYH = TY + 1;                         // face_y box rows
constexpr int XPL = ((BX * BY + 15) / 16) * 16;     // 688: x slot (128-byte aligned)
constexpr int ZPL = TX * TY;                        // face_z slot
constexpr int ASTRIDE = XPL + ZPL;                  // ring A stage (1200 doubles)
constexpr int BPL = TX * TY;                        // b slot
constexpr int FXPL = ((FXW * TY + 15) / 16) * 16;   // 528
constexpr int FYPL = ((TX * FYH + 15) / 16) * 16;   // 576
constexpr int BSTRIDE = BPL + FXPL + FYPL;          // ring B stage (1616 doubles)
constexpr int AST = 4, BST = 2;
constexpr size_t SMEM = (size_t)(AST * ASTRIDE + BST * BSTRIDE) * sizeof(double) + 8 * (AST + BST);
constexpr uint32_t ABYTES = (BX * BY + ZPL) * sizeof(double);
constexpr uint32_t BBYTES = (BPL + FXW * TY + TX * FYH) * sizeof(double);
static_assert((ASTRIDE * 8) % 128 == 0 && (BSTRIDE * 8) % 128 == 0 && (XPL * 8) % 128 == 0 &&
                  (BPL * 8) % 128 == 0 && (FXPL * 8) % 128 == 0,
              "TMA destinations stay 128-byte aligned");
}  // namespace k3v

struct Args3V {
    Geom g;
    double* buf0;
    double* buf1;
    const double* omegas;
    int M;
    double tol, baseline;
    double* partials;  // [2][gridDim.x]
    double* hist;
    int* out_i;
    double* out_d;
    int tiles_x, ntiles, zc, items;
};

struct Maps3V {
    CUtensorMap x0, x1, b, fx, fy, fz;
};

extern __shared__ __align__(128) double k3v_smem[];

struct Ring3V {
    uint32_t aphase, bphase;  // parity bit per stage
    __device__ static __forceinline__ double* a(int s) { return k3v_smem + s * k3v::ASTRIDE; }
    __device__ static __forceinline__ double* b(int s) {
        return k3v_smem + k3v::AST * k3v::ASTRIDE + s * k3v::BSTRIDE;
    }
    __device__ static __forceinline__ uint64_t* abar(int s) {
        return reinterpret_cast<uint64_t*>(k3v_smem + k3v::AST * k3v::ASTRIDE +
                                           k3v::BST * k3v::BSTRIDE) + s;
    }
    __device__ static __forceinline__ uint64_t* bbar(int s) { return abar(k3v::AST) + s; }
};

// Ring A, plane p (p = -1 .. nz): x (tensor plane p+1 of the ghost-spanning
// map) and face_z plane p (p = -1 is outside the map: zero fill, never read).
__device__ __forceinline__ void issue_a(const CUtensorMap* mx, const CUtensorMap* mz, int ox, int oy,
                                        int p) {
    using namespace k3v;
    const int s = (p + 1) & (AST - 1);
    double* st = Ring3V::a(s);
    fence_proxy_async();
    mbar_expect_tx(Ring3V::abar(s), ABYTES);
    tma_load_3d(st, mx, ox - XOFF, oy - 1, p + 1, Ring3V::abar(s));
    tma_load_3d(st + XPL, mz, ox, oy, p, Ring3V::abar(s));
}

// Ring B, plane p: b, face_x, face_y.
__device__ __forceinline__ void issue_b(const Maps3V& m, int ox, int oy, int p) {
    using namespace k3v;
    const int s = p & (BST - 1);
    double* st = Ring3V::b(s);
    fence_proxy_async();
    mbar_expect_tx(Ring3V::bbar(s), BBYTES);
    tma_load_3d(st, &m.b, ox, oy, p, Ring3V::bbar(s));
    tma_load_3d(st + BPL, &m.fx, ox, oy, p, Ring3V::bbar(s));
    tma_load_3d(st + BPL + FXPL, &m.fy, ox, oy, p, Ring3V::bbar(s));
}

__device__ __forceinline__ void wait_a(Ring3V& r, int p) {
    const int s = (p + 1) & (k3v::AST - 1);
    mbar_wait(Ring3V::abar(s), (r.aphase >> s) & 1u);
    r.aphase ^= 1u << s;
}

__device__ __forceinline__ void wait_b(Ring3V& r, int p) {
    const int s = p & (k3v::BST - 1);
    mbar_wait(Ring3V::bbar(s), (r.bphase >> s) & 1u);
    r.bphase ^= 1u << s;
}

// One sweep (WRITE) or residual evaluation (!WRITE) over this CTA's items.
template <bool WRITE>
__device__ __forceinline__ double sweep3v(const Args3V& a, const Maps3V& m, const CUtensorMap* mx,
                                          double* __restrict__ xout, double w, Ring3V& r) {
    using namespace k3v;
    const int tid = threadIdx.x;
    const int tx = tid % TX, ty0 = tid / TX;
    const int nx = a.g.nx, ny = a.g.ny, nz = a.g.nz;
    const long long plane = (long long)nx * ny;
    double acc = 0.0;
    for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
        const int tile = item % a.ntiles, zci = item / a.ntiles;
        const int ox = (tile % a.tiles_x) * TX, oy = (tile / a.tiles_x) * TY;
        const int z0 = zci * a.zc, z1 = min(z0 + a.zc, nz);
        if (tid == 0) {
            for (int p = z0 - 1; p <= min(z0 + 2, z1); ++p) issue_a(mx, &m.fz, ox, oy, p);
            for (int p = z0; p <= min(z0 + 1, z1 - 1); ++p) issue_b(m, ox, oy, p);
        }
        wait_a(r, z0 - 1);
        wait_a(r, z0);
        const int i = ox + tx;
        const bool colin = i < nx;
        for (int z = z0; z < z1; ++z) {
            wait_a(r, z + 1);
            wait_b(r, z);
            const double* am = Ring3V::a((z) & (AST - 1));      // plane z-1
            const double* ac = Ring3V::a((z + 1) & (AST - 1));  // plane z
            const double* ap = Ring3V::a((z + 2) & (AST - 1));  // plane z+1
            const double* sb = Ring3V::b(z & (BST - 1));
            const double* sfx = sb + BPL;
            const double* sfy = sb + BPL + FXPL;
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const int ty = ty0 + q * RSTEP;
                const int j = oy + ty;
                if (colin && j < ny) {
                    const int ci = (ty + 1) * BX + tx + XOFF;
                    const int pi = ty * TX + tx;
                    const double cw = sfx[ty * FXW + tx], ce = sfx[ty * FXW + tx + 1];
                    const double cs = sfy[pi], cn = sfy[pi + TX];
                    const double cb = ac[XPL + pi], ct = ap[XPL + pi];
                    const double d = DADD(DADD(DADD(DADD(DADD(cw, ce), cs), cn), cb), ct);
                    const double xc = ac[ci];
                    double y = DADD(0.0, DMUL(-cb, am[ci]));
                    y = DADD(y, DMUL(-cs, ac[ci - BX]));
                    y = DADD(y, DMUL(-cw, ac[ci - 1]));
                    y = DADD(y, DMUL(d, xc));
                    y = DADD(y, DMUL(-ce, ac[ci + 1]));
                    y = DADD(y, DMUL(-cn, ac[ci + BX]));
                    y = DADD(y, DMUL(-ct, ap[ci]));
                    const double rr = DSUB(sb[pi], y);
                    acc = fma(rr, rr, acc);
                    if constexpr (WRITE) {
                        SRJ_ASSERT(i < nx && j < ny && z < nz);
                        xout[(long long)z * plane + (long long)j * nx + i] =
                            relax(xc, __drcp_rn(d), rr, w);
                    }
                }
            }
            __syncthreads();  // ring A stage of plane z-1 and ring B stage of z are free
            if (tid == 0) {
                if (z + 3 <= z1) issue_a(mx, &m.fz, ox, oy, z + 3);
                if (z + 2 < z1) issue_b(m, ox, oy, z + 2);
            }
        }
    }
    return acc;
}

__global__ void __launch_bounds__(k3v::THREADS) k_cycle3dv(const __grid_constant__ Maps3V m,
                                                          Args3V a) {
    using namespace k3v;
    __shared__ double sh[32];
    Ring3V r;
    r.aphase = 0;
    r.bphase = 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < AST; ++s) mbar_init(Ring3V::abar(s), 1);
        for (int s = 0; s < BST; ++s) mbar_init(Ring3V::bbar(s), 1);
        prefetch_tensormap(&m.x0);
        prefetch_tensormap(&m.x1);
        prefetch_tensormap(&m.b);
        prefetch_tensormap(&m.fx);
        prefetch_tensormap(&m.fy);
        prefetch_tensormap(&m.fz);
    }
    __syncthreads();
    const int nb = gridDim.x;
    double* const buf[2] = {a.buf0, a.buf1};
    const CUtensorMap* const mx[2] = {&m.x0, &m.x1};
    int executed = a.M, status = kStatusRan;
    double S = 0.0, res = 0.0;
    for (int k = 0; k <= a.M; ++k) {
        const bool tail = (k == a.M);
        double acc = tail ? sweep3v<false>(a, m, mx[k & 1], nullptr, 0.0, r)
                          : sweep3v<true>(a, m, mx[k & 1], buf[(k + 1) & 1], a.omegas[k], r);
        double* part = a.partials + (k & 1) * nb;
        acc = block_allsum(acc, sh);
        if (threadIdx.x == 0) part[blockIdx.x] = acc;
        grid_barrier();
        if (k >= 1 || tail) {
            S = reduce_partials(part, nb, sh);
            res = sqrt(S) / a.baseline;
            if (k >= 1) {
                if (blockIdx.x == 0 && threadIdx.x == 0) a.hist[k] = res;
                if (!isfinite(res)) { executed = k; status = kStatusDiverged; break; }
                if (res <= a.tol) { executed = k; status = kStatusConverged; break; }
            }
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.out_i[0] = executed;
        a.out_i[1] = status;
        a.out_i[2] = executed & 1;
        a.out_d[0] = S;
        a.out_d[1] = res;
    }
}

cudaError_t plan3v_init(Plan3V& plan, const Geom& g, int num_sms) {
    plan = Plan3V();
    // TMA: 16-byte row pitch of x, b, face_y and face_z (even nx)
    if (g.fam != F3DV || (g.nx & 1) || !tma_available()) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(k_cycle3dv, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)k3v::SMEM);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cycle3dv, k3v::THREADS, k3v::SMEM);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaSuccess;
    plan.fx_pitch = g.nx + 2;
    const long long rows = (long long)g.ny * g.nz;
    if ((e = cudaMalloc(&plan.fx_pad, (size_t)plan.fx_pitch * rows * sizeof(double))) != cudaSuccess)
        return e;
    if ((e = cudaMemcpy2D(plan.fx_pad, plan.fx_pitch * sizeof(double), g.fx,
                          (size_t)(g.nx + 1) * sizeof(double), (size_t)(g.nx + 1) * sizeof(double),
                          rows, cudaMemcpyDeviceToDevice)) != cudaSuccess) {
        plan3v_free(plan);
        return e;
    }
    plan.per_sm = per_sm;
    plan.slots = per_sm * num_sms;
    plan.tiles_x = (g.nx + k3v::TX - 1) / k3v::TX;
    plan.tiles_y = (g.ny + k3v::TY - 1) / k3v::TY;
    // planes per item: minimise rounds * (zc + 2) (two-plane pipeline fill)
    const int ntiles = plan.tiles_x * plan.tiles_y;
    double best = 1e300;
    plan.zc = g.nz;
    for (int zc = 8; zc <= std::max(8, g.nz); zc += 8) {
        const long long items = (long long)ntiles * ((g.nz + zc - 1) / zc);
        const double cost = (double)((items + plan.slots - 1) / plan.slots) * (zc + 2);
        if (cost < best) { best = cost; plan.zc = zc; }
        if (zc >= g.nz) break;
    }
    plan.zc = std::max(1, std::min(plan.zc, g.nz));
    if (const char* v = getenv("SRJ_ZC")) plan.zc = std::max(1, std::min(atoi(v), g.nz));  // tuning
    plan.nzc = (g.nz + plan.zc - 1) / plan.zc;
    plan.items = ntiles * plan.nzc;
    plan.blocks = std::max(1, std::min(plan.slots, plan.items));
    plan.supported = true;
    return cudaSuccess;
}

void plan3v_free(Plan3V& plan) {
    if (plan.fx_pad) cudaFree(plan.fx_pad);
    plan.fx_pad = nullptr;
    plan.supported = false;
}

cudaError_t launch3v_cycle(const Plan3V& plan, const Geom& g, double* x, double* x_alt,
                           const double* b, const double* omegas, int M, double tol,
                           double baseline, double* partials, double* hist, int* out_i,
                           double* out_d, cudaStream_t st) {
    using namespace k3v;
    if ((((uintptr_t)x | (uintptr_t)b | (uintptr_t)g.fy | (uintptr_t)g.fz) & 15) != 0 ||
        (x_alt && ((uintptr_t)x_alt & 15) != 0))
        return cudaErrorMisalignedAddress;
    const long long plane = (long long)g.nx * g.ny;
    Maps3V m;
    cudaError_t e;
    // x maps span the ghost planes: base one plane before the interior
    if ((e = encode_volume_map(&m.x0, x - plane, g.nx, g.ny, g.nz + 2, BX, BY)) != cudaSuccess) return e;
    if ((e = encode_volume_map(&m.x1, (x_alt ? x_alt : x) - plane, g.nx, g.ny, g.nz + 2, BX, BY)) !=
        cudaSuccess)
        return e;
    if ((e = encode_volume_map(&m.b, b, g.nx, g.ny, g.nz, TX, TY)) != cudaSuccess) return e;
    if ((e = encode_volume_map_pitched(&m.fx, plan.fx_pad, g.nx + 1, g.ny, g.nz, plan.fx_pitch, FXW,
                                       TY)) != cudaSuccess)
        return e;
    if ((e = encode_volume_map(&m.fy, g.fy, g.nx, g.ny + 1, g.nz, TX, FYH)) != cudaSuccess) return e;
    if ((e = encode_volume_map(&m.fz, g.fz, g.nx, g.ny, g.nz + 1, TX, TY)) != cudaSuccess) return e;
    Args3V a;
    a.g = g;
    a.buf0 = x;
    a.buf1 = x_alt;
    a.omegas = omegas;
    a.M = M;
    a.tol = tol;
    a.baseline = baseline;
    a.partials = partials;
    a.hist = hist;
    a.out_i = out_i;
    a.out_d = out_d;
    a.tiles_x = plan.tiles_x;
    a.ntiles = plan.tiles_x * plan.tiles_y;
    a.zc = plan.zc;
    a.items = plan.items;
    void* args[] = {&m, &a};
    return cudaLaunchCooperativeKernel((const void*)k_cycle3dv, dim3(plan.blocks), dim3(THREADS),
                                       args, SMEM, st);
}

}  // namespace srj
