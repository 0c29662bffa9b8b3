/*
 * srj.h -- C ABI of libsrj.so, the sm_100a device path of the Scheduled
 * Relaxation Jacobi (SRJ) solve (arXiv 2011.06636).
 *
 * The reference (pure Python, /root/reference/pkg/src/srj) has no FFI: its hot
 * path is the duck-typed operator surface `run_cycle` touches.  Each entry
 * point below names the reference code it replaces:
 *
 *   srj_run_cycle      solver.run_cycle's sweep loop            solver.py:216-243
 *   srj_solve          solver.solve's cycle loop on the device  solver.py:289-331
 *                      + the post-loop convergence test          solver.py:245-249
 *                      (x + w*(inv_diag*r), b - csr.dot(x), np.linalg.norm,
 *                       np.isfinite, per-sweep tol/budget tests, history)
 *   srj_residual_sq    b - A.scipy_csr().dot(x) and its squared norm, used for
 *                      the relative baseline and a cold cycle start
 *                                                                solver.py:209-210,300-304
 *   srj_sweep          sparse.weighted_jacobi_sweep              sparse.py:84-93
 *   srj_matvec         sparse.matvec / csr_matvec                sparse.py:78-81
 *   srj_fill_uniform_rhs  f_i = 2*SplitMix64(seed).uniform()-1 in index order
 *                      (rng.py:25-40; idiom of problems.py:382)
 *   srj_op_create      sparse.SparseMatrix construction for the structured
 *                      Dirichlet stencils (problems.py:50-69, 148-177)
 *
 * Conventions
 *   - Status codes: SRJ_OK, SRJ_DIVERGED, SRJ_BAD_ARGUMENT, SRJ_CUDA_ERROR;
 *     srj_last_error() returns a thread-local message for the last failure.
 *   - All vectors are caller-owned fp64 device buffers (torch tensors' data_ptr()).
 *     Every x / x_alt / b pointer addresses the FIRST INTERIOR point of a buffer
 *     that also holds `halo` ghost elements before and after the n interior points
 *     (halo = one plane: 1 in 1D, nx in 2D, nx*ny in 3D; see srj_op_layout).
 *     Ghost values are read, never written: zero for a Dirichlet side, the
 *     neighbour slab's boundary plane for an internal slab side.
 *   - Work is stream-ordered on `stream` (a cudaStream_t, NULL = legacy default).
 *     srj_run_cycle and srj_residual_sq synchronise the stream once before they
 *     return (the host reads one small result struct per cycle); the other
 *     calls are asynchronous.
 *   - No allocation inside a cycle: all scratch is owned by the srj_op handle.
 *     Handles are independent and may be used from different threads; one
 *     handle must not be used concurrently.
 *   - Iterates are bit-identical to the reference CSR path: every stencil sum is
 *     a left-to-right, separately rounded sum over ascending CSR columns and the
 *     update is t = inv_diag*r; t = w*t; x' = x + t (no FMA contraction).
 *     Residual norms are deterministic (fixed-order reductions) but are summed in
 *     a different order than OpenBLAS ddot, so they agree to ~1e-15 relative.
 */
#ifndef SRJ_H
#define SRJ_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SRJ_ABI_VERSION 2

enum srj_status {
    SRJ_OK = 0,
    SRJ_DIVERGED = 1,      /* a residual or iterate became non-finite */
    SRJ_BAD_ARGUMENT = 2,
    SRJ_CUDA_ERROR = 3
};

enum srj_family {
    SRJ_STENCIL_1D3 = 1,     /* 1D 3-point, (-1, 2, -1)*dx2                 */
    SRJ_STENCIL_2D5 = 2,     /* 2D 5-point, (-1,-1, 4,-1,-1)*dx2            */
    SRJ_STENCIL_3D7 = 3,     /* 3D 7-point, 6*dx2 diagonal, -dx2 neighbours  */
    SRJ_STENCIL_2D5_VAR = 4, /* 2D 5-point, harmonic-mean face coefficients  */
    SRJ_CSR = 5,             /* general canonical CSR matrix (sparse.SparseMatrix) */
    SRJ_STENCIL_3D7_VAR = 6, /* 3D 7-point, harmonic-mean face coefficients  */
    SRJ_STENCIL_1D3_VAR = 7  /* 1D 3-point, face coefficients                */
};

/* Outcome of one cycle; mirrors the reference's CycleStats plus the buffer
 * that holds the final iterate. */
enum srj_cycle_status {
    SRJ_CYCLE_RAN = 0,        /* all sweeps applied (or budget cut), tol not met */
    SRJ_CYCLE_CONVERGED = 1,  /* stopping rule met (mid-cycle or after last sweep) */
    SRJ_CYCLE_DIVERGED = 2    /* non-finite residual after sweep `executed`        */
};

typedef struct srj_op srj_op;

typedef struct srj_op_desc {
    int32_t family;        /* enum srj_family */
    int32_t device;        /* CUDA ordinal the buffers live on */
    int64_t nx, ny, nz;    /* interior extents of THIS operator's grid (slab); unused axes = 1 */
    double  dx2;           /* constant coefficient scale (N+1)^2 (ignored for *_VAR) */
    /* *_VAR only: face coefficients already scaled by dx2, device pointers.
     * Off-diagonals are -face; the diagonal is the sum of the point's faces in
     * the order west, east (, south, north (, bottom, top)).
     * face_x: ny*nz rows of nx+1 faces (face i sits between points i-1 and i);
     * face_y: nz planes of ny+1 rows of nx faces (row j sits between rows j-1
     *         and j); unused in 1D;
     * face_z (3D, at the end of the struct): nz+1 planes of ny x nx faces
     *         (plane z sits between planes z-1 and z). */
    const double* face_x;
    const double* face_y;
    /* SRJ_CSR only (nx = n, ny = nz = 1; vectors carry no ghosts): canonical
     * CSR -- ascending columns, duplicates summed, as sparse.SparseMatrix keeps
     * it (sparse.py:28-44) -- and 1.0/diagonal, all device pointers. */
    int64_t nnz;
    const int64_t* row_ptr;
    const int32_t* col_idx;
    const double* values;
    const double* inv_diag;
    /* SRJ_STENCIL_3D7_VAR only (ABI 2) */
    const double* face_z;
} srj_op_desc;

typedef struct srj_cycle_out {
    int32_t executed;       /* sweeps applied (CycleStats.executed) */
    int32_t status;         /* enum srj_cycle_status */
    int32_t result_in_alt;  /* 1: final iterate is in x_alt; 0: in x */
    int32_t launches;       /* kernel launches used by the cycle (diagnostic) */
    double  res_before;     /* CycleStats.residual_before */
    double  res_after;      /* CycleStats.residual_after  */
} srj_cycle_out;

int srj_abi_version(void);
const char* srj_last_error(void);

int srj_op_create(const srj_op_desc* desc, srj_op** out);
int srj_op_destroy(srj_op* op);
/* n interior points and the ghost elements required before/after them. */
int srj_op_layout(const srj_op* op, int64_t* n, int64_t* halo);
/* Diagonal value and its reciprocal for constant-coefficient families
 * (diag = 2d*dx2, inv = 1/diag as the reference's SparseMatrix caches it). */
int srj_op_diag(const srj_op* op, double* diag, double* inv_diag);
/* Temporal blocking: sweeps fused per HBM pass (1 = one sweep per pass).
 * Values > 1 take effect only where a temporally blocked kernel exists for the
 * operator (srj_op_info.tb_supported); elsewhere cycles run one sweep per pass. */
int srj_op_set_sweeps_per_pass(srj_op* op, int32_t s);

/* Launch configuration the handle chose (diagnostics and tests). */
typedef struct srj_op_info {
    int32_t num_sms;
    int32_t cycle_blocks;      /* one-sweep cycle kernel: cooperative grid */
    int32_t cycle_threads;
    int32_t sweeps_per_pass;   /* current setting */
    int32_t tb_supported;      /* 1 if a temporally blocked kernel serves this operator */
    int32_t tb_blocks;
    int32_t tb_occupancy;      /* resident CTAs per SM of the smallest TB variant */
    int32_t tb_tiles;
    int32_t cycle_kernel;      /* enum srj_cycle_kernel serving srj_run_cycle now */
} srj_op_info;

enum srj_cycle_kernel {
    SRJ_KERNEL_GENERIC = 0,    /* persistent row walker (any family)            */
    SRJ_KERNEL_TB2D = 1,       /* temporally blocked 2D (sweeps_per_pass > 1)   */
    SRJ_KERNEL_TILE2D = 2,     /* TMA tile streaming 2D (constant / variable)   */
    SRJ_KERNEL_PLANE3D = 3,    /* TMA plane streaming 3D                        */
    /* 4: retired (round-1 warp-streaming experiment, removed)                   */
    SRJ_KERNEL_TB3D = 5,       /* temporally blocked 3D z-wavefront (2 sweeps
                                  per pass when sweeps_per_pass > 1)            */
    SRJ_KERNEL_TBVAR = 6,      /* temporally blocked 2D variable coefficient    */
    SRJ_KERNEL_SMALL1D = 7,    /* single-CTA shared-memory 1D cycle (n <= 8192) */
    SRJ_KERNEL_REG1D = 8,      /* single-CTA register-resident 1D cycle (n <= 4096) */
    SRJ_KERNEL_PLANE3DV = 9,   /* TMA plane streaming 3D variable coefficient   */
    SRJ_KERNEL_TB3DV = 10,     /* temporally blocked 3D variable coefficient
                                  (2 sweeps per pass when sweeps_per_pass > 1)  */
    SRJ_KERNEL_TBS2D = 11      /* temporally blocked 2D, skewed tiles (whole-grid
                                  cycles and solves at 5-6 sweeps per pass)     */
};

/* Temporally blocked 2D kernel used when sweeps_per_pass > 1. */
enum srj_tb_kind {
    SRJ_TB_TILE = 0            /* TMA-staged overlapped tiles (srj_tb.cu), the only
                                  kind; other values return SRJ_BAD_ARGUMENT     */
};
int srj_op_set_temporal_kernel(srj_op* op, int32_t kind);

/* Work plan of the skewed-tile 2D kernel (SRJ_KERNEL_TBS2D) for an nx x ny grid
 * on num_ctas CTAs, computed on the host (no CUDA call; diagnostics and tests).
 * The grid is cut into strips of tile_cols owned columns; a strip's rows into
 * segments [lo, hi); a segment into tiles of tile_rows rows starting `sweeps`
 * rows above lo.  CTA c runs table[4*(c*tiles_per_cta + i)] = {ox, oy, lo, hi}
 * for i = 0.. until an entry with hi <= lo.  `table` may be NULL (sizes only);
 * `capacity` = ints it can hold (4 * num_ctas * tiles_per_cta needed, else
 * SRJ_BAD_ARGUMENT).  There is no reference counterpart: the reference sweeps
 * the whole vector at once (solver.py:225-233). */
int srj_skew_plan(int64_t nx, int64_t ny, int32_t num_ctas, int32_t* tiles_per_cta,
                  int32_t* ctas_used, int32_t* tile_rows, int32_t* tile_cols, int32_t* sweeps,
                  int32_t* table, int64_t capacity);
int srj_op_describe(const srj_op* op, srj_op_info* info);

/* sum_i (b - A x)_i^2 -> *sumsq_host.  Synchronises `stream`. */
int srj_residual_sq(srj_op* op, const double* x, const double* b,
                    double* sumsq_host, void* stream);

/* One SRJ cycle of up to min(M, budget) sweeps with omegas_dev[k] applied by
 * sweep k (device array, application order).  Before sweep k >= 1 the cycle
 * stops when ||b - A x_k|| / baseline <= tol or is non-finite; res_before is the
 * residual of the incoming x (the host already knows it).  x and x_alt are
 * ping-pong buffers (both with ghosts); x is overwritten, the final iterate is
 * in x (result_in_alt == 0) or x_alt.  history_host, if non-NULL, receives the
 * relative residual after each executed sweep (executed entries).
 * Returns SRJ_OK also for a diverged cycle (out->status says so). */
int srj_run_cycle(srj_op* op, double* x, double* x_alt, const double* b,
                  const double* omegas_dev, int32_t M, double tol, double baseline,
                  double res_before, int64_t budget, double* history_host,
                  srj_cycle_out* out, void* stream);

/* Device-resident solve: the controller loop of solver.solve (solver.py:305-326)
 * runs on the device between cycles, so a whole solve is one launch (or a few,
 * see SRJ_SOLVE_PAUSED).  Cycle j applies the scheme of its level
 * (omegas_all[level_off[l] .. level_off[l+1]), application order) with the
 * srj_run_cycle semantics, starting from x (the final iterate ends in x or
 * x_alt); between cycles the level moves as heuristic_next_level on the last
 * finite residual ratio (mode 0, thresholds t_hi / t_lo), by +1 (mode 1,
 * Increasing) or stays (mode 2, one fixed scheme).  The loop stops when a
 * cycle converges (or the incoming residual is already <= tol), diverges, the
 * sweep budget is spent, max_cycles records are written or the next cycle
 * would pass hist_cap sweeps (paused: continue with next_level, res_next,
 * prev_ratio and the result buffer).  recs_host receives one record per cycle
 * (out->cycles entries), history_host (nullable) the relative residual after
 * each sweep (out->sweeps entries).  Available where srj_op_solve_supported
 * says so (the temporally blocked kernels).  Synchronises `stream`. */
typedef struct srj_solve_args {
    const double* omegas_all;  /* device */
    const int32_t* level_off;  /* device, n_levels + 1 entries */
    int32_t n_levels;
    int32_t mode;              /* 0 heuristic, 1 increasing, 2 fixed */
    int32_t level0;
    int32_t max_cycles;
    double t_hi, t_lo;
    double res0;               /* residual entering the first cycle */
    double prev_ratio0;        /* last finite residual ratio so far, NaN if none */
    int64_t budget;            /* sweeps allowed: max_iterations - total so far */
    int64_t hist_cap;          /* >= 10000; sweeps one call may record */
} srj_solve_args;

typedef struct srj_solve_rec {
    int32_t level, M, executed, status;  /* status: enum srj_cycle_status */
    double res_before, res_after;
} srj_solve_rec;

enum srj_solve_stop {
    SRJ_SOLVE_PAUSED = 0, SRJ_SOLVE_CONVERGED = 1, SRJ_SOLVE_DIVERGED = 2, SRJ_SOLVE_BUDGET = 3
};

typedef struct srj_solve_out {
    int32_t cycles;            /* records written */
    int32_t stop;              /* enum srj_solve_stop */
    int32_t result_in_alt;     /* 1: the last iterate is in x_alt */
    int32_t next_level;        /* level of the next cycle (paused) */
    double res_next;           /* residual entering the next cycle (paused) */
    double prev_ratio;         /* last finite residual ratio (NaN if none) */
    int64_t sweeps;            /* sweeps applied by this call */
} srj_solve_out;

int srj_op_solve_supported(const srj_op* op);
/* Leave k SMs free in the temporally blocked kernels' persistent grids (default
 * 0), e.g. for the NCCL kernels of a halo exchange that overlaps a slab pass
 * (the persistent CTAs otherwise occupy every SM, so NCCL could not run
 * concurrently). */
int srj_op_set_reserved_sms(srj_op* op, int32_t k);
int srj_solve(srj_op* op, double* x, double* x_alt, const double* b, const srj_solve_args* args,
              double tol, double baseline, srj_solve_rec* recs_host, double* history_host,
              srj_solve_out* out, void* stream);

/* Same cycle under the solution-difference infinity norm (solver.py:200-203,
 * 224-228, 242-243): sweep k's norm is max|x_{k+1} - x_k| (bit-identical to
 * numpy), tested before the next sweep; res_before = the incoming norm or NaN
 * when unknown.  history_host receives the norm after each executed sweep. */
int srj_run_cycle_diffinf(srj_op* op, double* x, double* x_alt, const double* b,
                          const double* omegas_dev, int32_t M, double tol, double res_before,
                          int64_t budget, double* history_host, srj_cycle_out* out,
                          void* stream);

/* x_out = x + omega * inv_diag * (b - A x)  (one weighted Jacobi sweep). */
int srj_sweep(srj_op* op, const double* x, double* x_out, const double* b,
              double omega, void* stream);
/* Slab building blocks (multi-GPU decomposition).  The slab
 * axis is z in 3D and y (rows) in 2D; a 1D operator is one plane.
 * srj_op_planes: number of planes along the slab axis.
 * srj_sweep_planes: one weighted-Jacobi sweep of planes [z_begin, z_end) from x
 * into x_out (x_out == NULL: residual only) reading the ghost planes of x as
 * they are; *partial_dev (device) = sum over those planes of (b - A x)^2, reduced
 * in a fixed order.  Asynchronous; launches on the same `slot` (0 or 1) must
 * not overlap, launches on different slots may run concurrently (e.g. interior
 * planes while the halo exchange is in flight, then the boundary planes).
 * Replaces, per slab: sparse.weighted_jacobi_sweep + the norm of
 * solver.py:231-234. */
int64_t srj_op_planes(const srj_op* op);
int srj_sweep_planes(srj_op* op, const double* x, double* x_out, const double* b,
                     double omega, int64_t z_begin, int64_t z_end, double* partial_dev,
                     int32_t slot, void* stream);
/* Temporally blocked slab pass (2D constant or variable coefficient, or 3D
 * 7-point; even nx): h consecutive sweeps (h <= 6 in 2D, <= 2 in 3D) with
 * omegas_dev[0..h-1] over the operator's grid, storing only the owned rows
 * (3D: z planes) [row_lo, row_hi) of x_alt (the rows outside are the deep
 * ghost rows / planes of a slab: updated as ring points, never stored).
 * sums_dev[t] (device) = owned sum of (b - A x_t)^2 for t < h, reduced in a
 * fixed order.  No stop test and no residual tail: the caller (the slab
 * engine) decides per cycle.  Asynchronous.  Replaces, per slab, h iterations
 * of solver.py:216-243 between two deep halo exchanges. */
int srj_tb_pass(srj_op* op, double* x, double* x_alt, const double* b,
                const double* omegas_dev, int32_t h, int64_t row_lo, int64_t row_hi,
                double* sums_dev, void* stream);

/* Batched small 1D Poisson cycles (data collection, datacollect.py:79-117:
 * the candidate cycles of many independent trials in one launch).  Job j
 * applies M sweeps (no stopping) of the n-point Dirichlet system
 * (-1, 2, -1)*(n+1)^2 to x_pool[x_in_off .. +n) with b_pool[b_off .. +n) and
 * omega_pool[omega_off .. +M), writes the final iterate to x_pool[x_out_off ..)
 * and sum (b - A x)^2 of it to sumsq_dev[j].  jobs_dev is a device array;
 * max_n bounds every job's n (<= 12288).  Asynchronous. */
typedef struct srj_batch_job {
    int32_t n;
    int32_t M;
    int64_t omega_off;
    int64_t x_in_off;
    int64_t x_out_off;
    int64_t b_off;
} srj_batch_job;
int srj_batch_cycles_1d(const srj_batch_job* jobs_dev, int32_t njobs, int32_t max_n,
                        const double* omega_pool, double* x_pool, const double* b_pool,
                        double* sumsq_dev, int32_t device, void* stream);

/* y = A x (y needs no ghosts). */
int srj_matvec(srj_op* op, const double* x, double* y, void* stream);
/* out[i] = 2 * u_{start+i} - 1, u_j the j-th uniform of SplitMix64(seed). */
int srj_fill_uniform_rhs(double* out, int64_t n, uint64_t seed, int64_t start,
                         int32_t device, void* stream);

/* ---------------------------------------------------------------------------
 * Multi-GPU: one NCCL communicator per device.
 * The reference has no multi-process solve (its only concurrency is a process
 * pool of independent solves, cli.py:196-198); these entry points replace the
 * Python-side exchange of distributed.py (TorchTbExchanger) with native,
 * stream-ordered NCCL calls.  NCCL is loaded at run time (libnccl.so.2).
 * ------------------------------------------------------------------------- */
#define SRJ_NCCL_ID_BYTES 128
int srj_nccl_available(void);                       /* 1 if libnccl.so.2 resolved */
const char* srj_nccl_last_error(void);
int srj_nccl_unique_id(uint8_t id[SRJ_NCCL_ID_BYTES]);   /* on one rank, then broadcast */
int srj_nccl_comm_init(int32_t nranks, const uint8_t id[SRJ_NCCL_ID_BYTES], int32_t rank,
                       int32_t device, void** comm);
int srj_nccl_comm_destroy(void* comm);
/* Deep-halo exchange of a temporally blocked slab operator whose planes are
 * [0, g_lo) ghost, [g_lo, g_lo+count) owned, [g_lo+count, +g_hi) ghost: the
 * first / last `rows` owned planes go to rank-1 / rank+1 and their boundary
 * planes arrive in this slab's ghost planes, one NCCL group on `stream`. */
int srj_slab_exchange(const srj_op* op, void* comm, int32_t rank, int32_t nranks, double* x,
                      int64_t g_lo, int64_t count, int64_t g_hi, int32_t rows, void* stream);
/* The exchange's element offsets from x (first interior point) for planes of
 * `unit` points: plan[0] sent to rank-1, plan[1] received from rank-1,
 * plan[2] sent to rank+1, plan[3] received from rank+1, plan[4] values per
 * message.  No CUDA call.  The in-process virtual-rank exchanger copies by the
 * same plan, so every slab test exercises it. */
int srj_slab_exchange_plan(int64_t unit, int32_t rank, int32_t nranks, int64_t g_lo,
                           int64_t count, int64_t g_hi, int32_t rows, int64_t plan[5]);
/* gathered[r*K + k] = rank r's sums[k] (ncclAllGather; a copy when nranks == 1). */
int srj_allgather_sums(void* comm, int32_t nranks, const double* sums, double* gathered,
                       int64_t K, void* stream);
/* The forward part of one slab cycle (distributed.py TbSlabSolver.cycle):
 * snapshot x into x_snap (optional), M sweeps in passes of <= `ghost` sweeps
 * (each: exchange + srj_tb_pass over the owned planes), the exchange and
 * residual of x_M (sums_dev[M]), and the all-gather of the M+1 per-sweep owned
 * sums into gathered_dev[nranks*(M+1)].  No host synchronisation; x_M is in
 * x_alt when *result_in_alt.  The host applies the stopping rule to the rank-
 * ordered sums and rolls back from x_snap when a sweep inside stops. */
int srj_slab_cycle_forward(srj_op* op, void* comm, int32_t rank, int32_t nranks, double* x,
                           double* x_alt, double* x_snap, const double* b,
                           const double* omegas_dev, int32_t M, int32_t ghost, int64_t g_lo,
                           int64_t count, int64_t g_hi, double* sums_dev, double* gathered_dev,
                           int32_t* result_in_alt, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* SRJ_H */
