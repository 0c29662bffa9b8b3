// Tile-streaming cycle/sweep kernels for the 2D 5-point stencils (constant
// and variable coefficient) -- declarations.
#pragma once

#include <cuda_runtime.h>

#include "srj_common.cuh"

namespace srj {

struct Plan2D {
    bool supported = false;
    bool var = false;
    int blocks = 0;        // cooperative grid of the cycle kernel
    int slots = 0;         // resident CTAs over the GPU
    int tiles_x = 0;       // 64-column strips
    double* fx_pad = nullptr;  // var-coef: face_x copy with an even row pitch
    int fx_pitch = 0;          // doubles per padded face_x row
};

// Setup (allocates fx_pad for variable coefficients; free with plan2d_free).
cudaError_t plan2d_init(Plan2D& plan, const Geom& g, int num_sms);
void plan2d_free(Plan2D& plan);

// One cycle of M sweeps (M = 0: residual only); outputs as the other cycle kernels.
cudaError_t launch2d_cycle(const Plan2D& plan, const Geom& g, double* x, double* x_alt,
                           const double* b, const double* omegas, int M, double tol,
                           double baseline, double* partials, double* hist, int* out_i,
                           double* out_d, cudaStream_t st);

// One sweep (x_out != nullptr) or residual of rows [r_begin, r_end); *result =
// sum of r^2 over them (device, fixed-order reduction).
cudaError_t launch2d_sweep(const Plan2D& plan, const Geom& g, const double* x, double* x_out,
                           const double* b, double omega, int r_begin, int r_end,
                           double* block_part, unsigned* counter, double* result,
                           cudaStream_t st);

}  // namespace srj
