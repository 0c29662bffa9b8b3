/*
 * srj_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker and CPU baseline).
 *
 * Plain-C restatement of the reference SRJ sweep arithmetic on the structured
 * stencils, used by tests/, __graft_entry__.smoke() and bench.py's CPU
 * baseline.  It is never linked into or called by the product (libsrj.so).
 *
 * What it restates (reference = /root/reference/pkg/src/srj):
 *   y = A x          scipy csr_matvec over ascending CSR columns, sum starting
 *                    at 0.0, each product and sum rounded separately
 *                    (solver.py:233 -> sparse.py:81; CSR layout problems.py:58-63,
 *                    157-172)
 *   r = b - y        solver.py:233
 *   x' = x + w*(inv_diag*r)   solver.py:231 (three separately rounded ufuncs)
 *   sum r^2          np.linalg.norm(r)**2 -> ddot (solver.py:234); summation
 *                    order differs from OpenBLAS (norms agree to ~1e-15 rel.)
 * Build with -ffp-contract=off so no FMA is ever formed (see oracle/Makefile).
 *
 * Vectors are plain n-arrays (no ghosts).  Families: 1 = 1D 3-pt, 2 = 2D 5-pt,
 * 3 = 3D 7-pt (constant coefficient, off = -dx2, diag = 2d*dx2), 4 = 2D 5-pt
 * variable coefficient with faces fx (ny x (nx+1)) and fy ((ny+1) x nx),
 * 6 = 3D 7-pt variable coefficient with faces fx (nz*ny rows of nx+1), fy (nz
 * planes of (ny+1) x nx) and fz ((nz+1) planes of ny x nx), 7 = 1D 3-pt
 * variable coefficient with faces fx (nx+1).  Variable-coefficient operators
 * are symmetric with off-diagonals -face and the diagonal the sum of the
 * point's faces in the order west, east, south, north, bottom, top (the CSR
 * the golden scripts hand the reference via SparseMatrix.from_coo).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    int fam;
    int64_t nx, ny, nz;
    double dx2;
    const double* fx;
    const double* fy;
    const double* fz;
} oracle_op;

/* 3D variable coefficient: faces of point (i, j, z). */
static inline void faces3(const oracle_op* op, int64_t i, int64_t j, int64_t z, double* cw,
                          double* ce, double* cs, double* cn, double* cb, double* ct) {
    const int64_t nx = op->nx, ny = op->ny;
    const double* fxr = op->fx + (z * ny + j) * (nx + 1);
    *cw = fxr[i];
    *ce = fxr[i + 1];
    *cs = op->fy[(z * (ny + 1) + j) * nx + i];
    *cn = op->fy[(z * (ny + 1) + j + 1) * nx + i];
    *cb = op->fz[(z * ny + j) * nx + i];
    *ct = op->fz[((z + 1) * ny + j) * nx + i];
}

static inline double diag_var(const oracle_op* op, int64_t i, int64_t j) {
    const double* fxr = op->fx + j * (op->nx + 1);
    const double cw = fxr[i], ce = fxr[i + 1];
    const double cs = op->fy[j * op->nx + i], cn = op->fy[(j + 1) * op->nx + i];
    return ((cw + ce) + cs) + cn;
}

/* y_k = (A x)_k, ascending-column order, zero-started, no fusion. */
static inline double row_apply(const oracle_op* op, const double* x, int64_t k,
                               int64_t i, int64_t j, int64_t z) {
    const int64_t nx = op->nx, ny = op->ny, nz = op->nz, pl = nx * ny;
    double y = 0.0;
    if (op->fam == 1) {
        const double c = -1.0 * op->dx2, d = 2.0 * op->dx2;
        if (i > 0) y += c * x[k - 1];
        y += d * x[k];
        if (i < nx - 1) y += c * x[k + 1];
    } else if (op->fam == 2) {
        const double c = -1.0 * op->dx2, d = 4.0 * op->dx2;
        if (j > 0) y += c * x[k - nx];
        if (i > 0) y += c * x[k - 1];
        y += d * x[k];
        if (i < nx - 1) y += c * x[k + 1];
        if (j < ny - 1) y += c * x[k + nx];
    } else if (op->fam == 3) {
        const double c = -1.0 * op->dx2, d = 6.0 * op->dx2;
        if (z > 0) y += c * x[k - pl];
        if (j > 0) y += c * x[k - nx];
        if (i > 0) y += c * x[k - 1];
        y += d * x[k];
        if (i < nx - 1) y += c * x[k + 1];
        if (j < ny - 1) y += c * x[k + nx];
        if (z < nz - 1) y += c * x[k + pl];
    } else if (op->fam == 6) {
        double cw, ce, cs, cn, cb, ct;
        faces3(op, i, j, z, &cw, &ce, &cs, &cn, &cb, &ct);
        const double d = ((((cw + ce) + cs) + cn) + cb) + ct;
        if (z > 0) y += (-cb) * x[k - pl];
        if (j > 0) y += (-cs) * x[k - nx];
        if (i > 0) y += (-cw) * x[k - 1];
        y += d * x[k];
        if (i < nx - 1) y += (-ce) * x[k + 1];
        if (j < ny - 1) y += (-cn) * x[k + nx];
        if (z < nz - 1) y += (-ct) * x[k + pl];
    } else if (op->fam == 7) {
        const double cw = op->fx[i], ce = op->fx[i + 1];
        if (i > 0) y += (-cw) * x[k - 1];
        y += (cw + ce) * x[k];
        if (i < nx - 1) y += (-ce) * x[k + 1];
    } else {
        const double* fxr = op->fx + j * (nx + 1);
        if (j > 0) y += (-op->fy[j * nx + i]) * x[k - nx];
        if (i > 0) y += (-fxr[i]) * x[k - 1];
        y += diag_var(op, i, j) * x[k];
        if (i < nx - 1) y += (-fxr[i + 1]) * x[k + 1];
        if (j < ny - 1) y += (-op->fy[(j + 1) * nx + i]) * x[k + nx];
    }
    return y;
}

static inline double inv_diag_at(const oracle_op* op, int64_t i, int64_t j, int64_t z) {
    double d;
    if (op->fam == 4) {
        d = diag_var(op, i, j);
    } else if (op->fam == 6) {
        double cw, ce, cs, cn, cb, ct;
        faces3(op, i, j, z, &cw, &ce, &cs, &cn, &cb, &ct);
        d = ((((cw + ce) + cs) + cn) + cb) + ct;
    } else if (op->fam == 7) {
        d = op->fx[i] + op->fx[i + 1];
    } else {
        d = (op->fam == 1 ? 2.0 : op->fam == 2 ? 4.0 : 6.0) * op->dx2;
    }
    return 1.0 / d;
}

/* r = b - A x over all points; returns sum r^2 (sequential per thread chunk). */
double oracle_residual(int fam, int64_t nx, int64_t ny, int64_t nz, double dx2,
                       const double* fx, const double* fy, const double* fz, const double* x,
                       const double* b, double* r_out) {
    const oracle_op op = {fam, nx, ny, nz, dx2, fx, fy, fz};
    const int64_t rows = ny * nz;
    double total = 0.0;
#pragma omp parallel for schedule(static) reduction(+ : total)
    for (int64_t row = 0; row < rows; ++row) {
        const int64_t j = row % ny, z = row / ny;
        double s = 0.0;
        for (int64_t i = 0; i < nx; ++i) {
            const int64_t k = row * nx + i;
            const double r = b[k] - row_apply(&op, x, k, i, j, z);
            if (r_out) r_out[k] = r;
            s += r * r;
        }
        total += s;
    }
    return total;
}

/* x_out = x + w*(inv_diag*r)  (solver.py:231). */
void oracle_update(int fam, int64_t nx, int64_t ny, int64_t nz, double dx2,
                   const double* fx, const double* fy, const double* fz, const double* x,
                   const double* r, double w, double* x_out) {
    const oracle_op op = {fam, nx, ny, nz, dx2, fx, fy, fz};
    const int64_t rows = ny * nz;
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < rows; ++row) {
        const int64_t j = row % ny, z = row / ny;
        for (int64_t i = 0; i < nx; ++i) {
            const int64_t k = row * nx + i;
            const double t = inv_diag_at(&op, i, j, z) * r[k];
            x_out[k] = x[k] + w * t;
        }
    }
}

/* y = A x. */
void oracle_matvec(int fam, int64_t nx, int64_t ny, int64_t nz, double dx2,
                   const double* fx, const double* fy, const double* fz, const double* x,
                   double* y) {
    const oracle_op op = {fam, nx, ny, nz, dx2, fx, fy, fz};
    const int64_t rows = ny * nz;
#pragma omp parallel for schedule(static)
    for (int64_t row = 0; row < rows; ++row) {
        const int64_t j = row % ny, z = row / ny;
        for (int64_t i = 0; i < nx; ++i) {
            const int64_t k = row * nx + i;
            y[k] = row_apply(&op, x, k, i, j, z);
        }
    }
}

int oracle_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int t) {
#ifdef _OPENMP
    if (t > 0) omp_set_num_threads(t);
#else
    (void)t;
#endif
}
