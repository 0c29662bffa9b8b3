// Probe: can a kernel with 2-CTA clusters run as a cooperative launch with
// cooperative_groups grid sync, and do DSMEM stores + barrier.cluster work?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ccp cluster_coop_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__global__ void __cluster_dims__(1, 2, 1) k_probe(int* out, int rounds) {
    __shared__ int box[2];
    cg::cluster_group cl = cg::this_cluster();
    cg::grid_group grid = cg::this_grid();
    const unsigned rank = cl.block_rank();
    for (int r = 0; r < rounds; ++r) {
        if (threadIdx.x == 0) {
            int* remote = cl.map_shared_rank(box, rank ^ 1);
            remote[r & 1] = (int)(blockIdx.y * 1000 + r);  // tell the partner who I am
        }
        cl.sync();
        if (threadIdx.x == 0) {
            const int got = box[r & 1];
            const int want = (int)((blockIdx.y ^ 1) * 1000 + r);
            if (got != want) atomicAdd(out, 1);
        }
        grid.sync();
    }
    if (threadIdx.x == 0 && blockIdx.y == 0 && blockIdx.x == 0) atomicAdd(out + 1, 1);
}

int main() {
    int* d;
    cudaMalloc(&d, 8);
    cudaMemset(d, 0, 8);
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_probe, 256, 0);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(sms / 2, 2, 1);
    cfg.blockDim = dim3(256);
    int nclusters = 0;
    cudaOccupancyMaxActiveClusters(&nclusters, (void*)k_probe, &cfg);
    printf("sms %d per_sm %d max active 2-CTA clusters %d\n", sms, per_sm, nclusters);
    int rounds = 100;
    void* args[] = {&d, &rounds};
    cudaError_t e = cudaLaunchCooperativeKernel((void*)k_probe, dim3(nclusters, 2, 1), dim3(256),
                                                args, 0, 0);
    printf("cooperative launch: %s\n", cudaGetErrorString(e));
    e = cudaDeviceSynchronize();
    printf("sync: %s\n", cudaGetErrorString(e));
    int h[2];
    cudaMemcpy(h, d, 8, cudaMemcpyDeviceToHost);
    printf("mismatches %d, done %d\n", h[0], h[1]);
    // timing of cl.sync(): 1000 rounds without the grid sync
    return 0;
}
