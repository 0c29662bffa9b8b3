// Per-point stencil arithmetic shared by every SRJ kernel.
//
// Reference arithmetic being reproduced (bit for bit):
//   y = csr.dot(x): scipy sparsetools csr_matvec, sum starting at 0.0 over the
//       row's columns in ascending order, one rounding per multiply and add
//       (reference solver.py:233 -> sparse.py:81; SURVEY §8a parity recipe 6);
//   r = b - y                     (solver.py:233)
//   x' = x + w * (inv_diag * r)   (solver.py:231: three separately rounded ufuncs)
// Absent (boundary) columns are read as a zero ghost: c*0 = -0.0 for c < 0 and
// y + (-0.0) == y for every y, so adding them is identical to skipping them.
#pragma once

#include "srj_common.cuh"

namespace srj {

// (A x)_k at flat interior index k with in-plane coordinates (i, j) (j is
// the row within the plane; 2D/3D read y/z ghosts from the padded buffer).
// Also returns x_k and 1/diag_k (per point for variable coefficients).
template <int FAM>
__device__ __forceinline__ double apply_at(const Geom& g, const double* x,
                                           long long k, int i, int j,
                                           double& xc, double& inv) {
    double y;
    if constexpr (FAM == F1D) {
        const double c = g.c_off;
        xc = x[k];
        inv = g.inv_diag;
        y = DADD(0.0, DMUL(c, x[k - 1]));
        y = DADD(y, DMUL(g.c_diag, xc));
        y = DADD(y, DMUL(c, x[k + 1]));
    } else if constexpr (FAM == F2D) {
        const double c = g.c_off;
        const long long nx = g.nx;
        xc = x[k];
        inv = g.inv_diag;
        const double xw = i > 0 ? x[k - 1] : 0.0;
        const double xe = i < g.nx - 1 ? x[k + 1] : 0.0;
        y = DADD(0.0, DMUL(c, x[k - nx]));
        y = DADD(y, DMUL(c, xw));
        y = DADD(y, DMUL(g.c_diag, xc));
        y = DADD(y, DMUL(c, xe));
        y = DADD(y, DMUL(c, x[k + nx]));
    } else if constexpr (FAM == F3D) {
        const double c = g.c_off;
        const long long nx = g.nx, pl = g.plane;
        xc = x[k];
        inv = g.inv_diag;
        const double xs = j > 0 ? x[k - nx] : 0.0;
        const double xn = j < g.ny - 1 ? x[k + nx] : 0.0;
        const double xw = i > 0 ? x[k - 1] : 0.0;
        const double xe = i < g.nx - 1 ? x[k + 1] : 0.0;
        y = DADD(0.0, DMUL(c, x[k - pl]));
        y = DADD(y, DMUL(c, xs));
        y = DADD(y, DMUL(c, xw));
        y = DADD(y, DMUL(g.c_diag, xc));
        y = DADD(y, DMUL(c, xe));
        y = DADD(y, DMUL(c, xn));
        y = DADD(y, DMUL(c, x[k + pl]));
    } else if constexpr (FAM == FCSR) {
        // scipy csr_matvec (sparsetools): sum starts at 0, ascending columns
        const long long e = g.rp[k + 1];
        y = 0.0;
        for (long long jj = g.rp[k]; jj < e; ++jj) y = DADD(y, DMUL(__ldg(g.cv + jj), x[__ldg(g.ci + jj)]));
        xc = x[k];
        inv = __ldg(g.cinv + k);
    } else if constexpr (FAM == F3DV) {
        // faces pre-scaled by dx2; diagonal = sum of the point's faces in the
        // order west, east, south, north, bottom, top; j is the x-row index
        // z*ny + jy (the walker's row)
        const long long nx = g.nx, pl = g.plane;
        const int z = j / g.ny, jy = j - z * g.ny;
        const double* fxr = g.fx + (long long)j * (nx + 1);
        const double cw = __ldg(fxr + i), ce = __ldg(fxr + i + 1);
        const double* fyp = g.fy + (long long)(j + z) * nx + i;  // row z*(ny+1) + jy
        const double cs = __ldg(fyp), cn = __ldg(fyp + nx);
        const double cb = __ldg(g.fz + k), ct = __ldg(g.fz + k + pl);
        const double diag = DADD(DADD(DADD(DADD(DADD(cw, ce), cs), cn), cb), ct);
        inv = __ddiv_rn(1.0, diag);
        xc = x[k];
        const double xs = jy > 0 ? x[k - nx] : 0.0;
        const double xn = jy < g.ny - 1 ? x[k + nx] : 0.0;
        const double xw = i > 0 ? x[k - 1] : 0.0;
        const double xe = i < g.nx - 1 ? x[k + 1] : 0.0;
        y = DADD(0.0, DMUL(-cb, x[k - pl]));
        y = DADD(y, DMUL(-cs, xs));
        y = DADD(y, DMUL(-cw, xw));
        y = DADD(y, DMUL(diag, xc));
        y = DADD(y, DMUL(-ce, xe));
        y = DADD(y, DMUL(-cn, xn));
        y = DADD(y, DMUL(-ct, x[k + pl]));
    } else if constexpr (FAM == F1DV) {
        const double cw = __ldg(g.fx + k), ce = __ldg(g.fx + k + 1);
        const double diag = DADD(cw, ce);
        inv = __ddiv_rn(1.0, diag);
        xc = x[k];
        y = DADD(0.0, DMUL(-cw, x[k - 1]));
        y = DADD(y, DMUL(diag, xc));
        y = DADD(y, DMUL(-ce, x[k + 1]));
    } else {  // F2DV: faces pre-scaled by dx2; CSR stores -face off the diagonal
        const long long nx = g.nx;
        const long long row = j;
        const double* fxr = g.fx + row * (nx + 1);
        const double cw = __ldg(fxr + i), ce = __ldg(fxr + i + 1);
        const double cs = __ldg(g.fy + row * nx + i), cn = __ldg(g.fy + (row + 1) * nx + i);
        const double diag = DADD(DADD(DADD(cw, ce), cs), cn);
        inv = __ddiv_rn(1.0, diag);
        xc = x[k];
        const double xw = i > 0 ? x[k - 1] : 0.0;
        const double xe = i < g.nx - 1 ? x[k + 1] : 0.0;
        y = DADD(0.0, DMUL(-cs, x[k - nx]));
        y = DADD(y, DMUL(-cw, xw));
        y = DADD(y, DMUL(diag, xc));
        y = DADD(y, DMUL(-ce, xe));
        y = DADD(y, DMUL(-cn, x[k + nx]));
    }
    return y;
}

__device__ __forceinline__ double relax(double xc, double inv, double r, double w) {
    return DADD(xc, DMUL(w, DMUL(inv, r)));
}

}  // namespace srj
