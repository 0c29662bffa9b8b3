// Multi-GPU entry points of the C ABI (include/srj.h):
// an NCCL communicator per device, the deep-halo exchange of a temporally
// blocked slab, the per-cycle all-gather of per-sweep residual sums, and the
// whole forward part of a slab cycle (passes with their exchanges, residual
// of x_M, all-gather) as ONE stream-ordered call with no host synchronisation
// -- so a host loop issues one call per cycle, and the call can be captured
// in a CUDA graph.
//
// NCCL is resolved at run time (dlopen "libnccl.so.2": the copy torch already
// loaded when there is one), so libsrj has no link-time NCCL dependency and
// the single-GPU ABI works without it.  Built above the single-GPU ABI
// (srj_tb_pass, srj_sweep_planes, srj_op_layout), not inside it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <string>

#include "../../include/srj.h"

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    decltype(&ncclGetUniqueId) get_unique_id = nullptr;
    decltype(&ncclCommInitRank) comm_init_rank = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclSend) send = nullptr;
    decltype(&ncclRecv) recv = nullptr;
    decltype(&ncclAllGather) all_gather = nullptr;
    decltype(&ncclGroupStart) group_start = nullptr;
    decltype(&ncclGroupEnd) group_end = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static bool tried = false;
    if (tried) return api;
    tried = true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        api.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
        return api;
    }
#define SRJ_SYM(field, name)                                              \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));    \
    if (!api.field) {                                                     \
        api.why = std::string("NCCL symbol missing: ") + name;            \
        return api;                                                       \
    }
    SRJ_SYM(get_unique_id, "ncclGetUniqueId")
    SRJ_SYM(comm_init_rank, "ncclCommInitRank")
    SRJ_SYM(comm_destroy, "ncclCommDestroy")
    SRJ_SYM(send, "ncclSend")
    SRJ_SYM(recv, "ncclRecv")
    SRJ_SYM(all_gather, "ncclAllGather")
    SRJ_SYM(group_start, "ncclGroupStart")
    SRJ_SYM(group_end, "ncclGroupEnd")
    SRJ_SYM(error_string, "ncclGetErrorString")
#undef SRJ_SYM
    api.ok = true;
    return api;
}

thread_local std::string g_nccl_error;

int nfail(int code, const std::string& msg) {
    g_nccl_error = msg;
    return code;
}

#define NCCL_TRY(call)                                                                  \
    do {                                                                                \
        const ncclResult_t r_ = (call);                                                 \
        if (r_ != ncclSuccess)                                                          \
            return nfail(SRJ_CUDA_ERROR, std::string("NCCL: ") + nccl().error_string(r_)); \
    } while (0)

struct SlabGeom {
    int64_t n, halo, planes, unit;
};

int slab_geom(const srj_op* op, SlabGeom& s) {
    if (srj_op_layout(op, &s.n, &s.halo) != SRJ_OK) return SRJ_BAD_ARGUMENT;
    s.planes = srj_op_planes(op);
    if (s.planes < 1) return SRJ_BAD_ARGUMENT;
    s.unit = s.n / s.planes;
    return SRJ_OK;
}

}  // namespace

extern "C" {

const char* srj_nccl_last_error(void) { return g_nccl_error.c_str(); }

int srj_nccl_available(void) { return nccl().ok ? 1 : 0; }

int srj_nccl_unique_id(uint8_t id[SRJ_NCCL_ID_BYTES]) {
    if (!id) return nfail(SRJ_BAD_ARGUMENT, "null id");
    if (!nccl().ok) return nfail(SRJ_CUDA_ERROR, nccl().why);
    ncclUniqueId u;
    NCCL_TRY(nccl().get_unique_id(&u));
    std::memcpy(id, u.internal, SRJ_NCCL_ID_BYTES);
    return SRJ_OK;
}

int srj_nccl_comm_init(int32_t nranks, const uint8_t id[SRJ_NCCL_ID_BYTES], int32_t rank,
                       int32_t device, void** comm) {
    if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks)
        return nfail(SRJ_BAD_ARGUMENT, "bad communicator arguments");
    if (!nccl().ok) return nfail(SRJ_CUDA_ERROR, nccl().why);
    if (cudaSetDevice(device) != cudaSuccess) return nfail(SRJ_CUDA_ERROR, "cudaSetDevice failed");
    ncclUniqueId u;
    std::memcpy(u.internal, id, SRJ_NCCL_ID_BYTES);
    ncclComm_t c = nullptr;
    NCCL_TRY(nccl().comm_init_rank(&c, nranks, u, rank));
    *comm = c;
    return SRJ_OK;
}

int srj_nccl_comm_destroy(void* comm) {
    if (!comm) return SRJ_OK;
    if (!nccl().ok) return nfail(SRJ_CUDA_ERROR, nccl().why);
    NCCL_TRY(nccl().comm_destroy(static_cast<ncclComm_t>(comm)));
    return SRJ_OK;
}

int srj_slab_exchange_plan(int64_t unit, int32_t rank, int32_t nranks, int64_t g_lo,
                           int64_t count, int64_t g_hi, int32_t rows, int64_t plan[5]) {
    if (!plan || unit < 1 || rows < 1 || count < rows || g_lo < 0 || g_hi < 0 || nranks < 1 ||
        rank < 0 || rank >= nranks || (rank > 0 && g_lo < rows) ||
        (rank < nranks - 1 && g_hi < rows))
        return nfail(SRJ_BAD_ARGUMENT, "bad slab exchange arguments (ghost depth < rows?)");
    plan[0] = g_lo * unit;                   // first `rows` owned planes -> rank - 1
    plan[1] = (g_lo - rows) * unit;          // <- rank - 1's last owned planes
    plan[2] = (g_lo + count - rows) * unit;  // last `rows` owned planes -> rank + 1
    plan[3] = (g_lo + count) * unit;         // <- rank + 1's first owned planes
    plan[4] = (int64_t)rows * unit;          // values per message
    return SRJ_OK;
}

int srj_slab_exchange(const srj_op* op, void* comm, int32_t rank, int32_t nranks, double* x,
                      int64_t g_lo, int64_t count, int64_t g_hi, int32_t rows, void* stream) {
    if (!op || !x) return nfail(SRJ_BAD_ARGUMENT, "null argument");
    SlabGeom s;
    if (slab_geom(op, s) != SRJ_OK) return nfail(SRJ_BAD_ARGUMENT, "bad operator");
    if (g_lo + count + g_hi != s.planes)
        return nfail(SRJ_BAD_ARGUMENT, "slab planes do not match the operator");
    int64_t plan[5];
    const int rc = srj_slab_exchange_plan(s.unit, rank, nranks, g_lo, count, g_hi, rows, plan);
    if (rc != SRJ_OK) return rc;
    if (nranks == 1) return SRJ_OK;
    if (!comm) return nfail(SRJ_BAD_ARGUMENT, "null communicator");
    if (!nccl().ok) return nfail(SRJ_CUDA_ERROR, nccl().why);
    const NcclApi& api = nccl();
    ncclComm_t c = static_cast<ncclComm_t>(comm);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t cnt = (size_t)plan[4];
    NCCL_TRY(api.group_start());
    if (rank > 0) {
        NCCL_TRY(api.send(x + plan[0], cnt, ncclFloat64, rank - 1, c, st));
        NCCL_TRY(api.recv(x + plan[1], cnt, ncclFloat64, rank - 1, c, st));
    }
    if (rank < nranks - 1) {
        NCCL_TRY(api.send(x + plan[2], cnt, ncclFloat64, rank + 1, c, st));
        NCCL_TRY(api.recv(x + plan[3], cnt, ncclFloat64, rank + 1, c, st));
    }
    NCCL_TRY(api.group_end());
    return SRJ_OK;
}

int srj_allgather_sums(void* comm, int32_t nranks, const double* sums, double* gathered,
                       int64_t K, void* stream) {
    if (!sums || !gathered || K < 1 || nranks < 1)
        return nfail(SRJ_BAD_ARGUMENT, "bad all-gather arguments");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (nranks == 1) {
        if (cudaMemcpyAsync(gathered, sums, K * sizeof(double), cudaMemcpyDeviceToDevice, st) !=
            cudaSuccess)
            return nfail(SRJ_CUDA_ERROR, "copy failed");
        return SRJ_OK;
    }
    if (!comm) return nfail(SRJ_BAD_ARGUMENT, "null communicator");
    if (!nccl().ok) return nfail(SRJ_CUDA_ERROR, nccl().why);
    NCCL_TRY(nccl().all_gather(sums, gathered, (size_t)K, ncclFloat64,
                               static_cast<ncclComm_t>(comm), st));
    return SRJ_OK;
}

int srj_slab_cycle_forward(srj_op* op, void* comm, int32_t rank, int32_t nranks, double* x,
                           double* x_alt, double* x_snap, const double* b,
                           const double* omegas_dev, int32_t M, int32_t ghost, int64_t g_lo,
                           int64_t count, int64_t g_hi, double* sums_dev, double* gathered_dev,
                           int32_t* result_in_alt, void* stream) {
    if (!op || !x || !x_alt || !b || !omegas_dev || !sums_dev || !gathered_dev ||
        !result_in_alt || M < 1 || ghost < 1)
        return nfail(SRJ_BAD_ARGUMENT, "bad slab cycle arguments");
    SlabGeom s;
    if (slab_geom(op, s) != SRJ_OK) return nfail(SRJ_BAD_ARGUMENT, "bad operator");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t bytes = (size_t)(s.n + 2 * s.halo) * sizeof(double);
    if (x_snap &&
        cudaMemcpyAsync(x_snap - s.halo, x - s.halo, bytes, cudaMemcpyDeviceToDevice, st) != cudaSuccess)
        return nfail(SRJ_CUDA_ERROR, "snapshot copy failed");
    if (cudaMemsetAsync(sums_dev, 0, (size_t)(M + 1) * sizeof(double), st) != cudaSuccess)
        return nfail(SRJ_CUDA_ERROR, "memset failed");
    double* cur = x;
    double* alt = x_alt;
    int rc;
    for (int k = 0; k < M; k += ghost) {
        const int h = M - k < ghost ? M - k : ghost;
        if ((rc = srj_slab_exchange(op, comm, rank, nranks, cur, g_lo, count, g_hi, ghost,
                                    stream)) != SRJ_OK)
            return rc;
        if ((rc = srj_tb_pass(op, cur, alt, b, omegas_dev + k, h, g_lo, g_lo + count,
                              sums_dev + k, stream)) != SRJ_OK)
            return nfail(rc, std::string("srj_tb_pass: ") + srj_last_error());
        double* t = cur;
        cur = alt;
        alt = t;
    }
    if ((rc = srj_slab_exchange(op, comm, rank, nranks, cur, g_lo, count, g_hi, ghost, stream)) !=
        SRJ_OK)
        return rc;
    if ((rc = srj_sweep_planes(op, cur, nullptr, b, 0.0, g_lo, g_lo + count, sums_dev + M, 0,
                               stream)) != SRJ_OK)
        return nfail(rc, std::string("srj_sweep_planes: ") + srj_last_error());
    if ((rc = srj_allgather_sums(comm, nranks, sums_dev, gathered_dev, M + 1, stream)) != SRJ_OK)
        return rc;
    *result_in_alt = cur == x_alt ? 1 : 0;
    return SRJ_OK;
}

}  // extern "C"
