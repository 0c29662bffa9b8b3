// Temporal blocking: several SRJ sweeps per HBM pass (declarations).
#pragma once

#include <cuda_runtime.h>

#include "srj_common.cuh"

namespace srj {

constexpr int kTbMaxSub = 16;  // most sweeps fused into one pass

struct TbPlan {
    bool supported = false;
    int num_sms = 0;
};

void tb_plan_init(TbPlan& plan, const Geom& g, int num_sms);

int tb_run_cycle(TbPlan& plan, const Geom& g, double* x, double* x_alt, const double* b,
                 const double* omegas, int M, double tol, double baseline, int s,
                 double* partials, double* hist, int* out_i, double* out_d, cudaStream_t st,
                 int* launches);

const char* tb_last_error();

}  // namespace srj
