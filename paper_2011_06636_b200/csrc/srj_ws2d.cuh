// Warp-streaming temporal blocking for the 2D 5-point constant-coefficient
// stencil (declarations; see srj_ws2d.cu).
#pragma once

#include <cuda_runtime.h>

#include "srj_common.cuh"

namespace srj {

struct WsPlan {
    bool supported = false;
    int per_sm[3] = {0, 0, 0};  // resident CTAs per SM of the S = 2 / 4 / 6 variants
    int num_sms = 0;
    cudaStream_t stream = nullptr;
};

cudaError_t ws_plan_init(WsPlan& plan, const Geom& g, int num_sms);

// One cycle of M sweeps, s per pass (1 <= s <= 6); outputs as tb_launch_cycle.
cudaError_t ws_launch_cycle(const WsPlan& plan, const Geom& g, double* x, double* x_alt,
                            const double* b, const double* omegas, int M, int s, double tol,
                            double baseline, double* partials, double* hist, int* out_i,
                            double* out_d, cudaStream_t st);

}  // namespace srj
