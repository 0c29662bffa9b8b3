// Plane-streaming SRJ cycle kernel for the 3D 7-point constant-coefficient
// stencil (BASELINE configs 3 and 5; also the per-GPU body of the z-slab
// decomposition).
//
// Work item = one 64 x 16 xy tile over a run of `zc` planes.  The copy engine
// streams x planes (with a one-point halo ring: box 68 x 18) and b planes
// (64 x 16) through a 4-stage / 2-stage shared-memory ring, three planes ahead
// of the compute; every point then reads its seven stencil values from shared
// memory.  The x tensor map spans the ghost planes of the buffer (nz + 2 planes),
// so the Dirichlet (zero) or slab-halo planes arrive like any other plane, and
// the x/y faces of the grid are the copy engine's zero fill.  DRAM traffic stays
// at 24 B per point-sweep: each plane is read once from HBM, the halo ring and the
// two z-neighbour re-reads of a run's ends come from L2.
//
// Sweeps use the same persistent/cooperative protocol as the other cycle
// kernels (see srj_capi.cu): residual of the INPUT iterate accumulated per CTA,
// grid barrier, fixed-order reduction in every CTA, per-sweep stop test.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdlib>

#include "srj_3d.cuh"
#include "srj_stencil.cuh"
#include "srj_tma.cuh"
#include "srj_walk.cuh"

namespace srj {
namespace k3 {
constexpr int TX = 64, TY = 16;
constexpr int THREADS = 256;
constexpr int RPT = TY / (THREADS / TX);    // rows per thread (4)
constexpr int XOFF = 2;                     // box column of the tile's first point
constexpr int BX = TX + 2 * XOFF, BY = TY + 2;  // x box covering the one-point halo ring
constexpr int XPL = ((BX * BY + 15) / 16) * 16;  // doubles per x stage (128-byte aligned)
constexpr int BPL = TX * TY;                // doubles per b stage
constexpr int XST = 4, BST = 2;             // ring depths
constexpr size_t SMEM = (size_t)(XST * XPL + BST * BPL) * sizeof(double) + 8 * (XST + BST);
constexpr uint32_t XBYTES = BX * BY * sizeof(double);
constexpr uint32_t BBYTES = BPL * sizeof(double);
}  // namespace k3

struct Args3D {
    Geom g;
    double* buf0;
    double* buf1;
    const double* b;
    const double* omegas;
    int M;
    double tol, baseline;
    double* partials;  // [2][gridDim.x]
    double* hist;
    int* out_i;
    double* out_d;
    int tiles_x, ntiles, zc, items;
    int zbase, zend;  // planes [zbase, zend) are swept (whole slab for a cycle)
};

struct Ring3D {
    double* xs;       // XST stages
    double* bs;       // BST stages
    uint64_t* xbar;   // XST barriers
    uint64_t* bbar;   // BST barriers
    uint32_t xphase;  // parity bit per stage
    uint32_t bphase;
};

// x planes: tensor plane z+1 holds interior plane z (the map spans the ghost
// planes).  The box starts two columns left of the tile: a box whose innermost
// start is not 16-byte aligned (x0 odd for fp64) raises an illegal-instruction
// fault on B200 (tools/probe/tma_probe.cu), so the halo column is read at x0-2.
__device__ __forceinline__ void issue_x(const CUtensorMap* map, Ring3D& r, int ox, int oy, int z) {
    const int s = (z + 1) & (k3::XST - 1);
    fence_proxy_async();
    mbar_expect_tx(r.xbar + s, k3::XBYTES);
    tma_load_3d(r.xs + s * k3::XPL, map, ox - k3::XOFF, oy - 1, z + 1, r.xbar + s);
}

__device__ __forceinline__ void issue_b(const CUtensorMap* map, Ring3D& r, int ox, int oy, int z) {
    const int s = z & (k3::BST - 1);
    fence_proxy_async();
    mbar_expect_tx(r.bbar + s, k3::BBYTES);
    tma_load_3d(r.bs + s * k3::BPL, map, ox, oy, z, r.bbar + s);
}

__device__ __forceinline__ void wait_x(Ring3D& r, int z) {
    const int s = (z + 1) & (k3::XST - 1);
    mbar_wait(r.xbar + s, (r.xphase >> s) & 1u);
    r.xphase ^= 1u << s;
}

__device__ __forceinline__ void wait_b(Ring3D& r, int z) {
    const int s = z & (k3::BST - 1);
    mbar_wait(r.bbar + s, (r.bphase >> s) & 1u);
    r.bphase ^= 1u << s;
}

// One sweep (WRITE) or residual evaluation (!WRITE) over this CTA's items.
template <bool WRITE>
__device__ __forceinline__ double sweep3d(const Args3D& a, const CUtensorMap* mx,
                                          const CUtensorMap* mb, double* __restrict__ xout,
                                          double w, Ring3D& r) {
    using namespace k3;
    const int tid = threadIdx.x;
    const int tx = tid % TX, ty0 = tid / TX;
    const int nx = a.g.nx, ny = a.g.ny;
    const long long plane = (long long)nx * ny;
    const double coff = a.g.c_off, cdiag = a.g.c_diag, inv = a.g.inv_diag;
    double acc = 0.0;
    for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
        const int tile = item % a.ntiles, zci = item / a.ntiles;
        const int ox = (tile % a.tiles_x) * TX, oy = (tile / a.tiles_x) * TY;
        const int z0 = a.zbase + zci * a.zc, z1 = min(z0 + a.zc, a.zend);
        if (tid == 0) {
            for (int z = z0 - 1; z <= min(z0 + 2, z1); ++z) issue_x(mx, r, ox, oy, z);
            for (int z = z0; z <= min(z0 + 1, z1 - 1); ++z) issue_b(mb, r, ox, oy, z);
        }
        wait_x(r, z0 - 1);
        wait_x(r, z0);
        const int i = ox + tx;
        const bool colin = i < nx;
        for (int z = z0; z < z1; ++z) {
            wait_x(r, z + 1);
            wait_b(r, z);
            const double* sm = r.xs + ((z) & (XST - 1)) * XPL;      // plane z-1 (ghosted z)
            const double* sc = r.xs + ((z + 1) & (XST - 1)) * XPL;  // plane z
            const double* sp = r.xs + ((z + 2) & (XST - 1)) * XPL;  // plane z+1
            const double* sb = r.bs + (z & (BST - 1)) * BPL;
#pragma unroll
            for (int q = 0; q < RPT; ++q) {
                const int ty = ty0 + q * (THREADS / TX);
                const int j = oy + ty;
                if (colin && j < ny) {
                    const int ci = (ty + 1) * BX + tx + XOFF;
                    const double xc = sc[ci];
                    double y = DADD(0.0, DMUL(coff, sm[ci]));
                    y = DADD(y, DMUL(coff, sc[ci - BX]));
                    y = DADD(y, DMUL(coff, sc[ci - 1]));
                    y = DADD(y, DMUL(cdiag, xc));
                    y = DADD(y, DMUL(coff, sc[ci + 1]));
                    y = DADD(y, DMUL(coff, sc[ci + BX]));
                    y = DADD(y, DMUL(coff, sp[ci]));
                    const double rr = DSUB(sb[ty * TX + tx], y);
                    acc = fma(rr, rr, acc);
                    if constexpr (WRITE)
                        xout[(long long)z * plane + (long long)j * nx + i] = relax(xc, inv, rr, w);
                }
            }
            __syncthreads();  // stages of plane z-1 (x) and z (b) are free
            if (tid == 0) {
                if (z + 3 <= z1) issue_x(mx, r, ox, oy, z + 3);
                if (z + 2 < z1) issue_b(mb, r, ox, oy, z + 2);
            }
        }
    }
    return acc;
}

__global__ void __launch_bounds__(k3::THREADS) k_cycle3d(const __grid_constant__ CUtensorMap mx0,
                                                         const __grid_constant__ CUtensorMap mx1,
                                                         const __grid_constant__ CUtensorMap mb,
                                                         Args3D a) {
    using namespace k3;
    extern __shared__ __align__(128) double smem[];
    __shared__ double sh[32];
    Ring3D r;
    r.xs = smem;
    r.bs = smem + XST * XPL;
    r.xbar = reinterpret_cast<uint64_t*>(r.bs + BST * BPL);
    r.bbar = r.xbar + XST;
    r.xphase = 0;
    r.bphase = 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < XST; ++s) mbar_init(r.xbar + s, 1);
        for (int s = 0; s < BST; ++s) mbar_init(r.bbar + s, 1);
        prefetch_tensormap(&mx0);
        prefetch_tensormap(&mx1);
        prefetch_tensormap(&mb);
    }
    __syncthreads();
    const int nb = gridDim.x;
    double* const buf[2] = {a.buf0, a.buf1};
    const CUtensorMap* const mx[2] = {&mx0, &mx1};
    int executed = a.M, status = kStatusRan;
    double S = 0.0, res = 0.0;
    for (int k = 0; k <= a.M; ++k) {
        const bool tail = (k == a.M);
        double acc = tail ? sweep3d<false>(a, mx[k & 1], &mb, nullptr, 0.0, r)
                          : sweep3d<true>(a, mx[k & 1], &mb, buf[(k + 1) & 1], a.omegas[k], r);
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

// One sweep (or residual, xout == nullptr) of planes [a.zbase, a.zend), the
// building block of the slab-decomposed solve: *result receives the planes'
// sum of r^2 (per-CTA partials reduced in a fixed order by the last CTA).
__global__ void __launch_bounds__(k3::THREADS) k_sweep3d(const __grid_constant__ CUtensorMap mx,
                                                         const __grid_constant__ CUtensorMap mb,
                                                         Args3D a, double* xout, double w,
                                                         double* block_part, unsigned* counter,
                                                         double* result) {
    using namespace k3;
    extern __shared__ __align__(128) double smem[];
    __shared__ double sh[32];
    Ring3D r;
    r.xs = smem;
    r.bs = smem + XST * XPL;
    r.xbar = reinterpret_cast<uint64_t*>(r.bs + BST * BPL);
    r.bbar = r.xbar + XST;
    r.xphase = 0;
    r.bphase = 0;
    if (threadIdx.x == 0) {
        for (int s = 0; s < XST; ++s) mbar_init(r.xbar + s, 1);
        for (int s = 0; s < BST; ++s) mbar_init(r.bbar + s, 1);
    }
    __syncthreads();
    double acc = xout ? sweep3d<true>(a, &mx, &mb, xout, w, r)
                      : sweep3d<false>(a, &mx, &mb, nullptr, 0.0, r);
    last_block_sum(acc, block_part, counter, result, sh);
}

cudaError_t plan3d_init(Plan3D& plan, const Geom& g, int num_sms) {
    plan = Plan3D();
    // TMA: 16-byte row pitch (even nx); tiles cover the grid in x/y
    if (g.fam != F3D || (g.nx & 1) || !tma_available()) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(k_cycle3d, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)k3::SMEM);
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_sweep3d, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)k3::SMEM);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cycle3d, k3::THREADS, k3::SMEM);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaSuccess;
    plan.per_sm = per_sm;
    plan.slots = per_sm * num_sms;
    plan.tiles_x = (g.nx + k3::TX - 1) / k3::TX;
    plan.tiles_y = (g.ny + k3::TY - 1) / k3::TY;
    plan.zc = choose_zc(plan, g.nz);
    if (const char* v = getenv("SRJ_ZC")) plan.zc = std::max(1, std::min(atoi(v), g.nz));  // tuning
    plan.nzc = (g.nz + plan.zc - 1) / plan.zc;
    plan.items = plan.tiles_x * plan.tiles_y * plan.nzc;
    plan.blocks = std::max(1, std::min(plan.slots, plan.items));
    plan.supported = true;
    return cudaSuccess;
}

// Planes per work item over a run of nzr planes: minimise the critical path
// ceil(items/slots)*zc plus a two-plane pipeline fill per item.
int choose_zc(const Plan3D& plan, int nzr) {
    const int ntiles = plan.tiles_x * plan.tiles_y;
    int best_zc = nzr;
    double best = 1e300;
    for (int zc = 8; zc <= std::max(8, nzr); zc += 8) {
        const int nzc = (nzr + zc - 1) / zc;
        const long long items = (long long)ntiles * nzc;
        const long long rounds = (items + plan.slots - 1) / plan.slots;
        const double cost = (double)rounds * (zc + 2);
        if (cost < best) { best = cost; best_zc = zc; }
        if (zc >= nzr) break;
    }
    return std::max(1, std::min(best_zc, nzr));
}

cudaError_t launch3d_sweep(const Plan3D& plan, const Geom& g, const double* x, double* x_out,
                           const double* b, double omega, int z_begin, int z_end,
                           double* block_part, unsigned* counter, double* result,
                           cudaStream_t st) {
    if ((((uintptr_t)x | (uintptr_t)b) & 15) != 0) return cudaErrorMisalignedAddress;
    const long long plane = (long long)g.nx * g.ny;
    CUtensorMap mx, mb;
    cudaError_t e;
    if ((e = encode_volume_map(&mx, x - plane, g.nx, g.ny, g.nz + 2, k3::BX, k3::BY)) != cudaSuccess)
        return e;
    if ((e = encode_volume_map(&mb, b, g.nx, g.ny, g.nz, k3::TX, k3::TY)) != cudaSuccess) return e;
    Args3D a = {};
    a.g = g;
    a.tiles_x = plan.tiles_x;
    a.ntiles = plan.tiles_x * plan.tiles_y;
    const int nzr = z_end - z_begin;
    a.zc = choose_zc(plan, nzr);
    a.items = a.ntiles * ((nzr + a.zc - 1) / a.zc);
    a.zbase = z_begin;
    a.zend = z_end;
    const int blocks = std::max(1, std::min(plan.slots, a.items));
    k_sweep3d<<<blocks, k3::THREADS, k3::SMEM, st>>>(mx, mb, a, x_out, omega, block_part, counter,
                                                     result);
    return cudaGetLastError();
}

cudaError_t launch3d_cycle(const Plan3D& plan, const Geom& g, double* x, double* x_alt,
                           const double* b, const double* omegas, int M, double tol,
                           double baseline, double* partials, double* hist, int* out_i,
                           double* out_d, cudaStream_t st) {
    if ((((uintptr_t)x | (uintptr_t)b) & 15) != 0 || (x_alt && ((uintptr_t)x_alt & 15) != 0))
        return cudaErrorMisalignedAddress;
    const long long plane = (long long)g.nx * g.ny;
    CUtensorMap m0, m1, mb;
    cudaError_t e;
    // x maps span the ghost planes: base one plane before the interior
    if ((e = encode_volume_map(&m0, x - plane, g.nx, g.ny, g.nz + 2, k3::BX, k3::BY)) != cudaSuccess)
        return e;
    if ((e = encode_volume_map(&m1, (x_alt ? x_alt : x) - plane, g.nx, g.ny, g.nz + 2, k3::BX,
                               k3::BY)) != cudaSuccess)
        return e;
    if ((e = encode_volume_map(&mb, b, g.nx, g.ny, g.nz, k3::TX, k3::TY)) != cudaSuccess) return e;
    Args3D a;
    a.g = g;
    a.buf0 = x;
    a.buf1 = x_alt;
    a.b = b;
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
    a.zbase = 0;
    a.zend = g.nz;
    void* args[] = {&m0, &m1, &mb, &a};
    return cudaLaunchCooperativeKernel((const void*)k_cycle3d, dim3(plan.blocks),
                                       dim3(k3::THREADS), args, k3::SMEM, st);
}

}  // namespace srj
