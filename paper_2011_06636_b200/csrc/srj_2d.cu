// Tile-streaming SRJ kernels for the 2D 5-point stencils: the cycle kernel for
// the variable-coefficient operator (BASELINE config 4) and for 2D grids the
// temporally blocked kernel does not serve, and the row-slab sweep of the
// multi-GPU decomposition.
//
// Work item = one 64-column strip over a run of rows, processed as 64 x TY
// tiles.  Per tile the copy engine stages, in one mbarrier transaction: the x
// box with its halo ring (68 x (TY+2); the x tensor map spans the ghost rows,
// so Dirichlet / slab-halo rows arrive like interior rows and the left/right
// faces are zero fill), b (64 x TY) and, for variable coefficients, the face
// boxes face_x (66 x TY) and face_y (64 x (TY+1)).  Two stages: tile t+1 lands
// while tile t computes.  Each point then reads its 5 x values, b and 4 faces
// from shared memory; every array is read from HBM once per sweep (halo rows
// and columns come from L2): 24 B (constant) / 40 B (variable) per point-sweep.
//
// Variable coefficients: faces are the dx2-scaled harmonic means; CSR stores
// -face off the diagonal and ((c_w + c_e) + c_s) + c_n on it, and the
// reference caches inv_diag = 1.0 / diag (sparse.py:44); both are recomputed
// here with the same rounding, so iterates stay bit-identical.
#include <cooperative_groups.h>

#include <algorithm>

#include "srj_2d.cuh"
#include "srj_stencil.cuh"
#include "srj_tma.cuh"
#include "srj_walk.cuh"

namespace srj {
namespace k2 {

constexpr int align16(int v) { return (v + 15) / 16 * 16; }  // doubles -> 128 B

template <bool VAR>
struct C {
    static constexpr int TX = 64;
    static constexpr int TY = VAR ? 16 : 32;
    static constexpr int THREADS = 256;
    static constexpr int RPT = TY / (THREADS / TX);
    static constexpr int XOFF = 2;  // 16-byte-aligned box start (see srj_3d.cu)
    static constexpr int BX = TX + 2 * XOFF, BY = TY + 2;
    static constexpr int FXW = TX + 2;
    static constexpr int XS = align16(BX * BY);
    static constexpr int BS = TX * TY;
    static constexpr int FXS = VAR ? align16(FXW * TY) : 0;
    static constexpr int FYS = VAR ? align16(TX * (TY + 1)) : 0;
    static constexpr int STAGE = XS + BS + FXS + FYS;  // doubles
    static constexpr int NST = 2;
    static constexpr size_t SMEM = (size_t)NST * STAGE * sizeof(double) + 8 * NST;
    static constexpr uint32_t BYTES =
        (uint32_t)((BX * BY + BS + (VAR ? FXW * TY + TX * (TY + 1) : 0)) * sizeof(double));
};

}  // namespace k2

struct Maps2D {
    CUtensorMap x0, x1, b, fx, fy;
};

struct Args2D {
    Geom g;
    double* buf0;
    double* buf1;
    const double* b;
    const double* omegas;
    int M;
    double tol, baseline;
    double* partials;
    double* hist;
    int* out_i;
    double* out_d;
    int tiles_x;
    int rbase, rend;  // rows [rbase, rend) are swept
    int rc;           // rows per work item (multiple of TY)
    int items;
};

template <bool VAR>
struct Ring2D {
    double* st;       // NST stages
    uint64_t* bar;    // NST barriers
    uint32_t phase;
};

template <bool VAR>
__device__ __forceinline__ void issue2d(const CUtensorMap* mx, const Maps2D& m, Ring2D<VAR>& r,
                                        int ox, int oy, int s) {
    using Cf = k2::C<VAR>;
    double* st = r.st + s * Cf::STAGE;
    fence_proxy_async();
    mbar_expect_tx(r.bar + s, Cf::BYTES);
    // ghosted row coordinate: tensor row oy holds interior row oy-1
    tma_load_2d(st, mx, ox - Cf::XOFF, oy, r.bar + s);
    tma_load_2d(st + Cf::XS, &m.b, ox, oy, r.bar + s);
    if constexpr (VAR) {
        tma_load_2d(st + Cf::XS + Cf::BS, &m.fx, ox, oy, r.bar + s);
        tma_load_2d(st + Cf::XS + Cf::BS + Cf::FXS, &m.fy, ox, oy, r.bar + s);
    }
}

template <bool VAR, bool WRITE>
__device__ __forceinline__ double sweep2d(const Args2D& a, const CUtensorMap* mx,
                                          const Maps2D& m, double* __restrict__ xout, double w,
                                          Ring2D<VAR>& r) {
    using Cf = k2::C<VAR>;
    constexpr int TX = Cf::TX, TY = Cf::TY, BX = Cf::BX;
    const int tid = threadIdx.x;
    const int tx = tid % TX, ty0 = tid / TX;
    const int nx = a.g.nx;
    const double coff = a.g.c_off, cdiag = a.g.c_diag, cinv = a.g.inv_diag;
    const int nchunks = (a.rend - a.rbase + a.rc - 1) / a.rc;
    double acc = 0.0;
    for (int item = blockIdx.x; item < a.items; item += gridDim.x) {
        const int strip = item % a.tiles_x, chunk = item / a.tiles_x;
        (void)nchunks;
        const int ox = strip * TX;
        const int r0 = a.rbase + chunk * a.rc, r1 = min(r0 + a.rc, a.rend);
        const int ntile = (r1 - r0 + TY - 1) / TY;
        if (tid == 0) {
            issue2d<VAR>(mx, m, r, ox, r0, 0);
            if (ntile > 1) issue2d<VAR>(mx, m, r, ox, r0 + TY, 1);
        }
        const int i = ox + tx;
        const bool colin = i < nx;
        for (int t = 0; t < ntile; ++t) {
            const int s = t & 1;
            const int oy = r0 + t * TY;
            mbar_wait(r.bar + s, (r.phase >> s) & 1u);
            r.phase ^= 1u << s;
            const double* xs = r.st + s * Cf::STAGE;
            const double* bs = xs + Cf::XS;
#pragma unroll
            for (int q = 0; q < Cf::RPT; ++q) {
                const int row = ty0 + q * (Cf::THREADS / TX);
                const int j = oy + row;
                if (colin && j < r1) {
                    const double* p = xs + (row + 1) * BX + tx + Cf::XOFF;
                    const double xc = p[0];
                    double y, inv;
                    if constexpr (VAR) {
                        const double* fxs = bs + Cf::BS;
                        const double* fys = fxs + Cf::FXS;
                        const double cw = fxs[row * Cf::FXW + tx], ce = fxs[row * Cf::FXW + tx + 1];
                        const double cs = fys[row * TX + tx], cn = fys[(row + 1) * TX + tx];
                        const double diag = DADD(DADD(DADD(cw, ce), cs), cn);
                        inv = __ddiv_rn(1.0, diag);
                        y = DADD(0.0, DMUL(-cs, p[-BX]));
                        y = DADD(y, DMUL(-cw, p[-1]));
                        y = DADD(y, DMUL(diag, xc));
                        y = DADD(y, DMUL(-ce, p[1]));
                        y = DADD(y, DMUL(-cn, p[BX]));
                    } else {
                        inv = cinv;
                        y = DADD(0.0, DMUL(coff, p[-BX]));
                        y = DADD(y, DMUL(coff, p[-1]));
                        y = DADD(y, DMUL(cdiag, xc));
                        y = DADD(y, DMUL(coff, p[1]));
                        y = DADD(y, DMUL(coff, p[BX]));
                    }
                    const double rr = DSUB(bs[row * TX + tx], y);
                    acc = fma(rr, rr, acc);
                    if constexpr (WRITE) xout[(long long)j * nx + i] = relax(xc, inv, rr, w);
                }
            }
            __syncthreads();  // stage s free
            if (tid == 0 && t + 2 < ntile) issue2d<VAR>(mx, m, r, ox, oy + 2 * TY, s);
        }
    }
    return acc;
}

template <bool VAR>
__device__ __forceinline__ void init_ring(Ring2D<VAR>& r, double* smem) {
    using Cf = k2::C<VAR>;
    r.st = smem;
    r.bar = reinterpret_cast<uint64_t*>(smem + Cf::NST * Cf::STAGE);
    r.phase = 0;
    if (threadIdx.x == 0)
        for (int s = 0; s < Cf::NST; ++s) mbar_init(r.bar + s, 1);
    __syncthreads();
}

template <bool VAR>
__global__ void __launch_bounds__(256) k_cycle2d(const __grid_constant__ Maps2D m, Args2D a) {
    extern __shared__ __align__(128) double smem[];
    __shared__ double sh[32];
    Ring2D<VAR> r;
    init_ring<VAR>(r, smem);
    const int nb = gridDim.x;
    double* const buf[2] = {a.buf0, a.buf1};
    const CUtensorMap* const mx[2] = {&m.x0, &m.x1};
    int executed = a.M, status = kStatusRan;
    double S = 0.0, res = 0.0;
    for (int k = 0; k <= a.M; ++k) {
        const bool tail = (k == a.M);
        double acc = tail ? sweep2d<VAR, false>(a, mx[k & 1], m, nullptr, 0.0, r)
                          : sweep2d<VAR, true>(a, mx[k & 1], m, buf[(k + 1) & 1], a.omegas[k], r);
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

template <bool VAR>
__global__ void __launch_bounds__(256) k_sweep2d(const __grid_constant__ Maps2D m, Args2D a,
                                                 double* xout, double w, double* block_part,
                                                 unsigned* counter, double* result) {
    extern __shared__ __align__(128) double smem[];
    __shared__ double sh[32];
    Ring2D<VAR> r;
    init_ring<VAR>(r, smem);
    const double acc = xout ? sweep2d<VAR, true>(a, &m.x0, m, xout, w, r)
                            : sweep2d<VAR, false>(a, &m.x0, m, nullptr, 0.0, r);
    last_block_sum(acc, block_part, counter, result, sh);
}

// ----------------------------------------------------------------------------
// Host side
// ----------------------------------------------------------------------------

template <bool VAR>
static cudaError_t setup(int& per_sm) {
    using Cf = k2::C<VAR>;
    cudaError_t e;
    if ((e = cudaFuncSetAttribute(k_cycle2d<VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)Cf::SMEM)) != cudaSuccess)
        return e;
    if ((e = cudaFuncSetAttribute(k_sweep2d<VAR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)Cf::SMEM)) != cudaSuccess)
        return e;
    return cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_cycle2d<VAR>, Cf::THREADS,
                                                         Cf::SMEM);
}

cudaError_t plan2d_init(Plan2D& plan, const Geom& g, int num_sms) {
    plan = Plan2D();
    if ((g.fam != F2D && g.fam != F2DV) || (g.nx & 1) || !tma_available()) return cudaSuccess;
    plan.var = g.fam == F2DV;
    int per_sm = 0;
    cudaError_t e = plan.var ? setup<true>(per_sm) : setup<false>(per_sm);
    if (e != cudaSuccess) return e;
    if (per_sm < 1) return cudaSuccess;
    plan.slots = per_sm * num_sms;
    plan.tiles_x = (g.nx + 63) / 64;
    if (plan.var) {
        // face_x rows hold nx+1 values; TMA needs a 16-byte row pitch
        plan.fx_pitch = g.nx + 2;
        if ((e = cudaMalloc(&plan.fx_pad, (size_t)plan.fx_pitch * g.ny * sizeof(double))) !=
            cudaSuccess)
            return e;
        if ((e = cudaMemcpy2D(plan.fx_pad, plan.fx_pitch * sizeof(double), g.fx,
                              (g.nx + 1) * sizeof(double), (g.nx + 1) * sizeof(double), g.ny,
                              cudaMemcpyDeviceToDevice)) != cudaSuccess)
            return e;
    }
    plan.supported = true;
    return cudaSuccess;
}

void plan2d_free(Plan2D& plan) {
    if (plan.fx_pad) cudaFree(plan.fx_pad);
    plan.fx_pad = nullptr;
}

template <bool VAR>
static cudaError_t make_maps(const Plan2D& plan, const Geom& g, const double* x,
                             const double* x_alt, const double* b, Maps2D& m) {
    using Cf = k2::C<VAR>;
    cudaError_t e;
    // x maps include the ghost rows: ny + 2 rows starting one row before the interior
    if ((e = encode_field_map(&m.x0, x - g.nx, g.nx, g.ny + 2, Cf::BX, Cf::BY)) != cudaSuccess)
        return e;
    if ((e = encode_field_map(&m.x1, (x_alt ? x_alt : x) - g.nx, g.nx, g.ny + 2, Cf::BX,
                              Cf::BY)) != cudaSuccess)
        return e;
    if ((e = encode_field_map(&m.b, b, g.nx, g.ny, Cf::TX, Cf::TY)) != cudaSuccess) return e;
    if constexpr (VAR) {
        if ((e = encode_field_map_pitched(&m.fx, plan.fx_pad, g.nx + 1, g.ny, plan.fx_pitch,
                                          Cf::FXW, Cf::TY)) != cudaSuccess)
            return e;
        if ((e = encode_field_map(&m.fy, g.fy, g.nx, g.ny + 1, Cf::TX, Cf::TY + 1)) !=
            cudaSuccess)
            return e;
    } else {
        m.fx = m.b;
        m.fy = m.b;
    }
    return cudaSuccess;
}

// rows per work item: multiple of TY balancing items over the resident CTAs
template <bool VAR>
static int choose_rc(const Plan2D& plan, int rows) {
    using Cf = k2::C<VAR>;
    int best = rows, best_cost = 1 << 30;
    for (int rc = Cf::TY; rc <= std::max(Cf::TY, rows); rc += Cf::TY) {
        const long long items = (long long)plan.tiles_x * ((rows + rc - 1) / rc);
        const long long rounds = (items + plan.slots - 1) / plan.slots;
        const int cost = (int)(rounds * (rc + Cf::TY));  // + one tile of pipeline fill
        if (cost < best_cost) { best_cost = cost; best = rc; }
        if (rc >= rows) break;
    }
    return best;
}

template <bool VAR>
static cudaError_t cycle_variant(const Plan2D& plan, const Geom& g, double* x, double* x_alt,
                                 const double* b, const double* omegas, int M, double tol,
                                 double baseline, double* partials, double* hist, int* out_i,
                                 double* out_d, cudaStream_t st) {
    using Cf = k2::C<VAR>;
    Maps2D m;
    cudaError_t e = make_maps<VAR>(plan, g, x, x_alt, b, m);
    if (e != cudaSuccess) return e;
    Args2D a = {};
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
    a.rbase = 0;
    a.rend = g.ny;
    a.rc = choose_rc<VAR>(plan, g.ny);
    a.items = plan.tiles_x * ((g.ny + a.rc - 1) / a.rc);
    const int blocks = std::max(1, std::min(plan.slots, a.items));
    void* args[] = {&m, &a};
    return cudaLaunchCooperativeKernel((const void*)k_cycle2d<VAR>, dim3(blocks),
                                       dim3(Cf::THREADS), args, Cf::SMEM, st);
}

cudaError_t launch2d_cycle(const Plan2D& plan, const Geom& g, double* x, double* x_alt,
                           const double* b, const double* omegas, int M, double tol,
                           double baseline, double* partials, double* hist, int* out_i,
                           double* out_d, cudaStream_t st) {
    if ((((uintptr_t)x | (uintptr_t)b) & 15) != 0 || (x_alt && ((uintptr_t)x_alt & 15) != 0))
        return cudaErrorMisalignedAddress;
    return plan.var ? cycle_variant<true>(plan, g, x, x_alt, b, omegas, M, tol, baseline, partials,
                                          hist, out_i, out_d, st)
                    : cycle_variant<false>(plan, g, x, x_alt, b, omegas, M, tol, baseline,
                                           partials, hist, out_i, out_d, st);
}

template <bool VAR>
static cudaError_t sweep_variant(const Plan2D& plan, const Geom& g, const double* x,
                                 double* x_out, const double* b, double omega, int r_begin,
                                 int r_end, double* block_part, unsigned* counter,
                                 double* result, cudaStream_t st) {
    using Cf = k2::C<VAR>;
    Maps2D m;
    cudaError_t e = make_maps<VAR>(plan, g, x, nullptr, b, m);
    if (e != cudaSuccess) return e;
    Args2D a = {};
    a.g = g;
    a.tiles_x = plan.tiles_x;
    a.rbase = r_begin;
    a.rend = r_end;
    a.rc = choose_rc<VAR>(plan, r_end - r_begin);
    a.items = plan.tiles_x * ((r_end - r_begin + a.rc - 1) / a.rc);
    const int blocks = std::max(1, std::min(plan.slots, a.items));
    k_sweep2d<VAR><<<blocks, Cf::THREADS, Cf::SMEM, st>>>(m, a, x_out, omega, block_part,
                                                          counter, result);
    return cudaGetLastError();
}

cudaError_t launch2d_sweep(const Plan2D& plan, const Geom& g, const double* x, double* x_out,
                           const double* b, double omega, int r_begin, int r_end,
                           double* block_part, unsigned* counter, double* result,
                           cudaStream_t st) {
    if ((((uintptr_t)x | (uintptr_t)b) & 15) != 0) return cudaErrorMisalignedAddress;
    return plan.var ? sweep_variant<true>(plan, g, x, x_out, b, omega, r_begin, r_end,
                                          block_part, counter, result, st)
                    : sweep_variant<false>(plan, g, x, x_out, b, omega, r_begin, r_end,
                                           block_part, counter, result, st);
}

}  // namespace srj
