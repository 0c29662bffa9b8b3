// Race / bounds instrumentation of the barrier-free kernels (the stress build,
// libsrj_stress.so, compiled with -DSRJ_STRESS; the product build compiles all
// of this away).  compute-sanitizer is not available on the GPU pool, so the
// evidence that no ordering relies on timing comes from this build:
//   * SRJ_JITTER(site): at every synchronisation point (mbarrier arrive and
//     wait, TMA issue, grid barrier) a pseudo-random subset of warps sleeps for
//     up to ~4 us, so warps and CTAs drift far apart in every possible order;
//     a missing wait then shows up as a wrong (non bit-identical) iterate in
//     the parity tests run against this library;
//   * mbarrier waits are bounded (a lost arrival traps after ~2 s instead of
//     hanging the GPU);
//   * SRJ_ASSERT: shared-memory and global index bounds in the staged
//     kernels; a violation traps (cudaErrorLaunchFailure on the host).
#pragma once

#include <stdint.h>

namespace srj {

#ifdef SRJ_STRESS
__device__ __forceinline__ uint64_t stress_clock() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__device__ __forceinline__ uint32_t stress_hash(uint32_t h) {
    h ^= h >> 16;
    h *= 0x7feb352du;
    h ^= h >> 15;
    h *= 0x846ca68bu;
    h ^= h >> 16;
    return h;
}

__device__ __forceinline__ void stress_jitter(uint32_t site) {
    const uint64_t t = stress_clock();
    const uint32_t h = stress_hash((uint32_t)(t >> 5) ^ (blockIdx.x * 0x9E3779B9u) ^
                                   ((threadIdx.x >> 5) * 0x85EBCA6Bu) ^ (site * 0xC2B2AE35u));
    if ((h & 3u) == 0u) __nanosleep((h >> 8) & 4095u);
}

__device__ __forceinline__ uint32_t dyn_smem_bytes() {
    uint32_t v;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(v));
    return v;
}

#define SRJ_JITTER(site) ::srj::stress_jitter(site)
#define SRJ_ASSERT(cond)      \
    do {                      \
        if (!(cond)) __trap(); \
    } while (0)
// p .. p+bytes inside the CTA's dynamic shared memory (base `smem_base`)
#define SRJ_ASSERT_SMEM(p, bytes, smem_base)                                         \
    SRJ_ASSERT((const char*)(p) >= (const char*)(smem_base) &&                      \
               (const char*)(p) + (bytes) <= (const char*)(smem_base) + ::srj::dyn_smem_bytes())
#else
#define SRJ_JITTER(site) ((void)0)
#define SRJ_ASSERT(cond) ((void)0)
#define SRJ_ASSERT_SMEM(p, bytes, smem_base) ((void)0)
#endif

}  // namespace srj
