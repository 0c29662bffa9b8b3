// Temporal blocking: several SRJ sweeps per HBM pass.
#include <string>

#include "srj_tb.cuh"

namespace srj {

static thread_local std::string g_tb_error;

void tb_plan_init(TbPlan& plan, const Geom& g, int num_sms) {
    plan.supported = false;
    plan.num_sms = num_sms;
    (void)g;
}

int tb_run_cycle(TbPlan&, const Geom&, double*, double*, const double*, const double*, int,
                 double, double, int, double*, double*, int*, double*, cudaStream_t, int*) {
    g_tb_error = "temporal blocking not available for this operator";
    return 1;
}

const char* tb_last_error() { return g_tb_error.c_str(); }

}  // namespace srj
