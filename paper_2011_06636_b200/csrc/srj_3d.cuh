// Plane-streaming cycle kernel for the 3D 7-point stencil (declarations).
#pragma once

#include <cuda_runtime.h>

#include "srj_common.cuh"

namespace srj {

struct Plan3D {
    bool supported = false;
    int blocks = 0;     // cooperative grid
    int per_sm = 0;     // resident CTAs per SM
    int tiles_x = 0, tiles_y = 0;
    int zc = 0;         // planes per work item
    int nzc = 0;        // work items along z
    int items = 0;
    int slots = 0;      // resident CTAs over the whole GPU
};

cudaError_t plan3d_init(Plan3D& plan, const Geom& g, int num_sms);
int choose_zc(const Plan3D& plan, int nzr);

// One sweep (x_out != nullptr) or residual evaluation of planes
// [z_begin, z_end); *result (device) = sum of r^2 over them.  block_part needs
// plan.slots doubles, counter one zeroed unsigned (left zeroed on exit).
cudaError_t launch3d_sweep(const Plan3D& plan, const Geom& g, const double* x, double* x_out,
                           const double* b, double omega, int z_begin, int z_end,
                           double* block_part, unsigned* counter, double* result,
                           cudaStream_t st);

// One cycle of M sweeps (M = 0: residual of x only).  Outputs as the other
// cycle kernels: out_i = {executed, status, result buffer}, out_d = {sum r^2 of
// the last residual evaluated, res_after}; hist[k] for k = 1..executed.
cudaError_t launch3d_cycle(const Plan3D& plan, const Geom& g, double* x, double* x_alt,
                           const double* b, const double* omegas, int M, double tol,
                           double baseline, double* partials, double* hist, int* out_i,
                           double* out_d, cudaStream_t st);

// Plane-streaming cycle kernel for the 3D 7-point VARIABLE-coefficient
// stencil (srj_3dv.cu).  Owns a 16-byte-pitch copy of face_x.
struct Plan3V {
    bool supported = false;
    int blocks = 0, per_sm = 0, slots = 0;
    int tiles_x = 0, tiles_y = 0, zc = 0, nzc = 0, items = 0;
    double* fx_pad = nullptr;  // face_x with row pitch nx + 2
    int fx_pitch = 0;
};

cudaError_t plan3v_init(Plan3V& plan, const Geom& g, int num_sms);
void plan3v_free(Plan3V& plan);
cudaError_t launch3v_cycle(const Plan3V& plan, const Geom& g, double* x, double* x_alt,
                           const double* b, const double* omegas, int M, double tol,
                           double baseline, double* partials, double* hist, int* out_i,
                           double* out_d, cudaStream_t st);

}  // namespace srj
