// Temporal blocking: several SRJ sweeps per HBM/L2 pass (declarations).
#pragma once

#include <cuda_runtime.h>
#include <stddef.h>

#include "srj_common.cuh"

namespace srj {

constexpr int kTbMaxSub = 8;  // most sweeps fused into one pass

struct TbPlan {
    bool supported = false;
    // per kernel variant (see srj_tb.cu, tb2d::Cfg<K>)
    int blocks[8] = {};   // cooperative grid (one CTA per SM)
    int tiles_x[8] = {};
    int ntiles[8] = {};
    int small_variant = -1;         // forced variant (SRJ_TB_VARIANT), -1: by sweeps per pass
    int occupancy = 0;              // min resident CTAs per SM over the variants
    int reserved = 0;               // SMs left free (srj_op_set_reserved_sms)
    // skewed-tile kernel (srj_tbs.cu): whole-grid cycles / solves at 5-6 sweeps per pass
    bool skew = false;
    int skew_tpc = 0;               // tile budget per CTA
    int skew_blocks = 0;            // CTAs that own tiles
    int skew_rows = 0, tile_rows = 0;  // region rows per CTA and pass: skewed / square tiles
    void* skew_tab = nullptr;       // device int4[blocks * tpc]: {ox, oy, lo, hi}
};

struct TbArgs;
// Skewed-tile kernel (srj_tbs.cu): plan (tile table on the device), launch.
cudaError_t tbs_plan_init(TbPlan& plan, const Geom& g, int num_sms);
void tbs_plan_free(TbPlan& plan);
cudaError_t tbs_launch_cycle(const TbPlan& plan, const Geom& g, TbArgs& a, double* x, double* x_alt,
                             const double* b, cudaStream_t st);
// Host-side packing of the skewed tiles (no CUDA call; srj_skew_plan).  `tab` gets
// ncta * T entries of 4 ints {ox, oy, lo, hi}.
int tbs_plan_table(int nx, int ny, int ncta, int* tab, long long capacity, int* T, int* used);
int tbs_tile_rows();
int tbs_tile_cols();
int tbs_sweeps();
// True when a whole-grid launch at s sweeps per pass runs the skewed-tile kernel.
bool tb_uses_skew(const TbPlan& plan, int s);

// Decide whether the operator has a temporal-blocking kernel and size its grid.
cudaError_t tb_plan_init(TbPlan& plan, const Geom& g, int num_sms);
// Kernel variant (tb2d::Cfg<K>) serving s sweeps per pass: K=0 (S=4 ring)
// for s <= 4, K=1 (S=6 ring) for s = 5, 6.
int tb_variant_for(const TbPlan& plan, int s);
// Sweeps one pass of the variant chosen for s can fuse (its ring width S).
int tb_ring_for(const TbPlan& plan, int s);

// ctl != nullptr (all three TB launchers): a device-resident solve from x
// (srj_tbdriver.cuh tb_run_solve) instead of one cycle; M and omegas are then
// unused, out_i = {cycles, stop, result buffer, next level}, out_d = {residual
// entering the next cycle, last finite ratio, sweeps}.
// Launch one cycle of M sweeps, s per pass (1 <= s <= kTbMaxSub; the 2D
// kernel fuses at most 4 and clamps larger requests).  Same
// outputs as the one-sweep cycle kernel: out_i = {executed, status, result
// buffer (0: x, 1: x_alt)}, out_d = {final sum of squares, res_after};
// hist[k] = relative residual of x_k for k = 1..executed.
// row_lo/row_hi: owned rows (slab with deep ghost rows; default the whole
// grid); sums != nullptr: pass mode (one pass of M <= s sweeps, raw owned
// sums of r^2 per sweep, no stop test, no residual tail; see srj_tbdriver.cuh).
cudaError_t tb_launch_cycle(const TbPlan& plan, const Geom& g, double* x, double* x_alt,
                            const double* b, const double* omegas, int M, int s, double tol,
                            double baseline, double* partials, double* hist, int* out_i,
                            double* out_d, cudaStream_t st, int row_lo, int row_hi,
                            double* sums, const SolveCtl* ctl = nullptr);

// 3D 7-point temporal blocking (srj_tb3d.cu): S = sweeps fused per pass.
struct Tb3Plan {
    bool supported = false;
    int blocks = 0, tiles_x = 0, ntiles = 0;
    int sweeps = 0;
    int zc = 0, items = 0;  // planes per work item, work items (tiles x z-runs)
    int num_sms = 0;
    int reserved = 0;       // SMs left free (srj_op_set_reserved_sms)
};

cudaError_t tb3_plan_init(Tb3Plan& plan, const Geom& g, int num_sms);

// One cycle of M sweeps, plan.sweeps per pass; outputs as tb_launch_cycle.
// The ghost planes of x and x_alt are the Dirichlet (zero) planes.
// z_lo/z_hi: owned planes (slab with deep ghost planes; default the whole
// grid); sums != nullptr: pass mode (one pass of M <= 2 sweeps, raw owned
// sums of r^2 per sweep, no stop test, no residual tail).
cudaError_t tb3_launch_cycle(const Tb3Plan& plan, const Geom& g, double* x, double* x_alt,
                             const double* b, const double* omegas, int M, double tol,
                             double baseline, double* partials, double* hist, int* out_i,
                             double* out_d, cudaStream_t st, int z_lo, int z_hi, double* sums,
                             const SolveCtl* ctl = nullptr);

// 3D variable-coefficient temporal blocking (srj_tb3v.cu): 2 sweeps per pass.
// Shares the 16-byte-pitch face_x copy of the one-sweep plan (Plan3V).
struct Tb3vPlan {
    bool supported = false;
    int blocks = 0, tiles_x = 0, ntiles = 0, zc = 0, items = 0;
    const double* fx_pad = nullptr;
    int fx_pitch = 0;
};

cudaError_t tb3v_plan_init(Tb3vPlan& plan, const Geom& g, int num_sms, const double* fx_pad,
                           int fx_pitch);
cudaError_t tb3v_launch_cycle(const Tb3vPlan& plan, const Geom& g, double* x, double* x_alt,
                              const double* b, const double* omegas, int M, double tol,
                              double baseline, double* partials, double* hist, int* out_i,
                              double* out_d, cudaStream_t st, const SolveCtl* ctl = nullptr);

// 2D variable-coefficient temporal blocking (srj_tbvar.cu), up to 6 sweeps per pass.
struct TbvPlan {
    bool supported = false;
    int blocks = 0, tiles_x = 0, ntiles = 0;
    double* fx_pad = nullptr;  // fx with a 16-byte row pitch (nx + 2)
    int fx_pitch = 0;
    double* inv = nullptr;     // 1 / diagonal, precomputed (reference order)
    int reserved = 0;          // SMs left free (srj_op_set_reserved_sms)
};

cudaError_t tbv_plan_init(TbvPlan& plan, const Geom& g, int num_sms);
void tbv_plan_free(TbvPlan& plan);
cudaError_t tbv_launch_cycle(const TbvPlan& plan, const Geom& g, double* x, double* x_alt,
                             const double* b, const double* omegas, int M, int s, double tol,
                             double baseline, double* partials, double* hist, int* out_i,
                             double* out_d, cudaStream_t st, int row_lo, int row_hi,
                             double* sums, const SolveCtl* ctl = nullptr);

}  // namespace srj
