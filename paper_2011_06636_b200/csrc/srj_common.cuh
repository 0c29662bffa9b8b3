// Shared device helpers for the SRJ sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "srj_stress.cuh"

// Separately rounded fp64 operations: the reference's scipy csr_matvec and
// numpy ufuncs round every multiply and add on their own, so the device must
// never contract them into FMAs (bit-identical iterates, SURVEY §8a parity
// recipe).
#define DMUL(a, b) __dmul_rn((a), (b))
#define DADD(a, b) __dadd_rn((a), (b))
#define DSUB(a, b) __dsub_rn((a), (b))

namespace srj {

enum Family { F1D = 1, F2D = 2, F3D = 3, F2DV = 4, FCSR = 5, F3DV = 6, F1DV = 7 };

// Cycle outcome codes (match enum srj_cycle_status in include/srj.h).
constexpr int kStatusRan = 0;
constexpr int kStatusConverged = 1;
constexpr int kStatusDiverged = 2;

// Device-resident solve (the host controller loop of solver.py:305-326 run on
// the device between cycles).  The scheme of level l is
// omegas_all[level_off[l] .. level_off[l+1]) (application order).
enum SolveMode { kSolveHeuristic = 0, kSolveIncreasing = 1, kSolveFixed = 2 };
// Why a device solve returned: paused (cycle cap or history buffer full; the
// host continues), converged, diverged, iteration budget exhausted.
enum SolveStop { kSolvePaused = 0, kSolveConverged = 1, kSolveDiverged = 2, kSolveBudget = 3 };

struct SolveRec {          // one cycle (matches srj_solve_rec in include/srj.h)
    int level, M, executed, status;
    double res_before, res_after;
};

struct SolveCtl {
    const double* omegas_all;  // device
    const int* level_off;      // device, n_levels + 1 entries
    int n_levels, mode, level0, max_cycles;
    double t_hi, t_lo;
    double res0;               // residual entering the first cycle
    double prev_ratio0;        // last finite residual ratio so far (NaN: none)
    long long budget;          // sweeps allowed (max_iterations - total so far)
    long long hist_cap;        // hist holds relative residuals of sweeps 1..hist_cap
    SolveRec* recs;            // device, max_cycles entries
};

// Operator geometry as the kernels see it.  The flat interior index is
// k = i + nx*j + nx*ny*z (x fastest, reference problems.py:119-120,158-161);
// buffers carry `plane` ghost elements before and after the interior.
struct Geom {
    int fam;
    int nx, ny, nz;
    long long n;        // interior points
    long long plane;    // ghost extent: 1 (1D), nx (2D), nx*ny (3D)
    int rows;           // number of x-rows: ny*nz (1 in 1D)
    int upr;            // 32-point units per row
    int units;          // rows * upr
    double c_off;       // off-diagonal value (-dx2)
    double c_diag;      // diagonal value (2d*dx2)
    double inv_diag;    // 1.0 / c_diag
    const double* fx;   // var-coef faces (see srj.h)
    const double* fy;
    const double* fz;
    // general CSR operator (canonical: sorted columns, no duplicates)
    const long long* rp;  // row pointers [n+1]
    const int* ci;        // column indices [nnz]
    const double* cv;     // values [nnz]
    const double* cinv;   // 1.0 / diagonal [n]
};

// 64-bit warp shuffles with the two 32-bit halves moved explicitly.  The
// built-in double overloads let ptxas land the halves in crossed registers and
// repair them with XOR swaps (3 LOP3 per shuffle; ~7% of the 2D TB kernel's
// instructions).
__device__ __forceinline__ double shfl_up_d(double v, unsigned d) {
    int lo = __double2loint(v), hi = __double2hiint(v);
    asm volatile("shfl.sync.up.b32 %0, %0, %2, 0, -1;\n\tshfl.sync.up.b32 %1, %1, %2, 0, -1;"
                 : "+r"(lo), "+r"(hi)
                 : "r"(d));
    return __hiloint2double(hi, lo);
}
__device__ __forceinline__ double shfl_down_d(double v, unsigned d) {
    int lo = __double2loint(v), hi = __double2hiint(v);
    asm volatile("shfl.sync.down.b32 %0, %0, %2, 31, -1;\n\tshfl.sync.down.b32 %1, %1, %2, 31, -1;"
                 : "+r"(lo), "+r"(hi)
                 : "r"(d));
    return __hiloint2double(hi, lo);
}

// max that propagates NaN (fmax would drop it): a NaN difference must read
// as non-finite in the solution-difference norm.
__device__ __forceinline__ double nanmax(double a, double b) {
    return (a != a || b != b) ? __longlong_as_double(0x7ff8000000000000ll) : fmax(a, b);
}

__device__ __forceinline__ double warp_allmax(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = nanmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

__device__ __forceinline__ double block_allmax(double v, double* sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    v = warp_allmax(v);
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double t = lane < nw ? sh[lane] : 0.0;
    return warp_allmax(t);
}

__device__ __forceinline__ double warp_allsum(double v) {
    // xor butterfly: partners add the same two operands (commutative), so
    // every lane ends with bit-identical sums.
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum, identical bits in every thread.  `sh` needs 32 doubles.
__device__ __forceinline__ double block_allsum(double v, double* sh) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int nw = (blockDim.x + 31) >> 5;
    v = warp_allsum(v);
    __syncthreads();
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double t = lane < nw ? sh[lane] : 0.0;
    return warp_allsum(t);
}

}  // namespace srj
