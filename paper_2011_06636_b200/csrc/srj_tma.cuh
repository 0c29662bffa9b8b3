// TMA (cp.async.bulk.tensor) and mbarrier helpers for the tiled SRJ kernels.
//
// A 2D tensor map describes the n-interior of a field (x fastest); boxes that
// stick out of the grid are zero-filled by the copy engine, which is exactly
// the Dirichlet ghost the stencil needs, so tile loads need no boundary code.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "srj_stress.cuh"

namespace srj {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

// Plain arrival (count 1), no transaction bytes.
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    SRJ_JITTER(1);
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#ifdef SRJ_STRESS
    // bounded wait: a lost arrival traps after ~2 s instead of hanging
    const uint64_t t0 = stress_clock();
    for (;;) {
        uint32_t ok;
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n}"
            : "=r"(ok)
            : "r"(smem_u32(bar)), "r"(parity)
            : "memory");
        if (ok) break;
        if (stress_clock() - t0 > 2000000000ull) __trap();
    }
    SRJ_JITTER(2);
#else
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
#endif
}

// 2D box load global -> shared, completion counted on `bar` in bytes.
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x0, int y0,
                                            uint64_t* bar) {
    SRJ_JITTER(3);
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(x0), "r"(y0), "r"(smem_u32(bar))
        : "memory");
}

// 3D box load (x fastest, then y, then z planes).
__device__ __forceinline__ void tma_load_3d(void* dst, const CUtensorMap* map, int x0, int y0,
                                            int z0, uint64_t* bar) {
    SRJ_JITTER(4);
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(smem_u32(dst)),
        "l"((uint64_t)map), "r"(x0), "r"(y0), "r"(z0), "r"(smem_u32(bar))
        : "memory");
}

// Order prior generic-proxy accesses (st.global by other CTAs, made visible by
// the grid barrier; ld.shared of the staging buffer by this CTA) before the
// async-proxy TMA traffic that follows.
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void prefetch_tensormap(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)map) : "memory");
}

// Host: true when the driver exposes cuTensorMapEncodeTiled.
bool tma_available();

// Host: encode a 2D fp64 tensor map over an nx x ny field (row pitch nx) with
// a box of box_x x box_y elements and zero fill out of bounds.
cudaError_t encode_field_map(CUtensorMap* map, const double* base, int nx, int ny, int box_x,
                             int box_y);

// Host: 2D map over rows of `width` valid values stored with row pitch `pitch`
// (doubles; pitch*8 must be a multiple of 16).
cudaError_t encode_field_map_pitched(CUtensorMap* map, const double* base, int width, int rows,
                                     int pitch, int box_x, int box_y);

// Host: 3D fp64 map over nz planes of nx x ny (plane pitch nx*ny), box of
// box_x x box_y x 1, zero fill out of bounds.
cudaError_t encode_volume_map(CUtensorMap* map, const double* base, int nx, int ny, int nz,
                              int box_x, int box_y);

// Host: 3D fp64 map over `planes` planes of `rows` rows of `width` valid
// values, row pitch `pitch` doubles (pitch*8 a multiple of 16), plane pitch
// pitch*rows; box of box_x x box_y x 1, zero fill out of bounds.
cudaError_t encode_volume_map_pitched(CUtensorMap* map, const double* base, int width, int rows,
                                      int planes, int pitch, int box_x, int box_y);

}  // namespace srj
