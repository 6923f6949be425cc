// barrier_bench.cu -- microbenchmark of the per-iteration synchronisation options
// for the single-instance kernels: cooperative grid.sync() over
// B CTAs, a hand-rolled global-memory barrier (atomic arrive + spin), and a
// thread-block-cluster barrier (barrier.cluster arrive/wait) with a DSMEM key
// exchange.  Not part of the library.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o barrier_bench tools/barrier_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

__global__ void k_gridsync(int iters, unsigned long long *out) {
    cg::grid_group g = cg::this_grid();
    unsigned long long acc = 0;
    for (int i = 0; i < iters; i++) {
        acc += threadIdx.x;
        g.sync();
    }
    if (acc == 12345) out[0] = acc;
}

// arrive counter + generation flag in global memory
__global__ void k_flagsync(int iters, unsigned int *count, volatile unsigned int *gen, unsigned long long *out) {
    unsigned long long acc = 0;
    for (int i = 0; i < iters; i++) {
        acc += threadIdx.x;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned int g0 = *gen;
            __threadfence();
            if (atomicAdd(count, 1u) == gridDim.x - 1) {
                *count = 0;
                __threadfence();
                *gen = g0 + 1;
            } else {
                while (*gen == g0) {
                }
            }
            __threadfence();
        }
        __syncthreads();
    }
    if (acc == 12345) out[0] = acc;
}

__global__ void __cluster_dims__(1, 1, 1) k_dummy() {}

// cluster barrier + each CTA publishes a 64-bit key into CTA 0's shared memory (DSMEM) and reads the min
__global__ void k_clustersync(int iters, unsigned long long *out) {
    cg::cluster_group cl = cg::this_cluster();
    __shared__ unsigned long long keys[16];
    unsigned long long acc = 0;
    const unsigned int r = cl.block_rank();
    for (int i = 0; i < iters; i++) {
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long *k0 = cl.map_shared_rank(keys, 0);
            k0[r] = (unsigned long long)(i * 7 + r);
        }
        cl.sync();
        if (threadIdx.x == 0) {
            unsigned long long *k0 = cl.map_shared_rank(keys, 0);
            unsigned long long m = ~0ull;
            for (unsigned int q = 0; q < cl.num_blocks(); q++) m = k0[q] < m ? k0[q] : m;
            acc += m;
        }
        cl.sync();
    }
    if (acc == 12345) out[0] = acc;
}

int main() {
    unsigned long long *out;
    unsigned int *cnt, *gen;
    cudaMalloc(&out, 8);
    cudaMalloc(&cnt, 4);
    cudaMalloc(&gen, 4);
    cudaMemset(cnt, 0, 4);
    cudaMemset(gen, 0, 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    int blocks_list[] = {1, 2, 8, 16, 37, 74, 148};
    for (int threads : {256, 768}) {
        for (int b : blocks_list) {
            int it = iters;
            void *args[] = {&it, &out};
            cudaLaunchCooperativeKernel((void *)k_gridsync, b, threads, args, 0, 0);
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel((void *)k_gridsync, b, threads, args, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            k_flagsync<<<b, threads>>>(it, cnt, gen, out);
            cudaEventRecord(e0);
            k_flagsync<<<b, threads>>>(it, cnt, gen, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms2;
            cudaEventElapsedTime(&ms2, e0, e1);
            printf("threads %4d blocks %3d: grid.sync %.3f us/iter, flag barrier %.3f us/iter (%s)\n", threads, b,
                   1e3 * ms / iters, 1e3 * ms2 / iters, cudaGetErrorString(cudaGetLastError()));
        }
        for (int cs : {2, 4, 8, 16}) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(cs, 1, 1);
            cfg.blockDim = dim3(threads, 1, 1);
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeClusterDimension;
            attr[0].val.clusterDim.x = cs;
            attr[0].val.clusterDim.y = 1;
            attr[0].val.clusterDim.z = 1;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            if (cs > 8) cudaFuncSetAttribute(k_clustersync, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
            cudaLaunchKernelEx(&cfg, k_clustersync, iters, out);
            cudaEventRecord(e0);
            cudaLaunchKernelEx(&cfg, k_clustersync, iters, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("threads %4d cluster %2d: 2 x cluster.sync + DSMEM key exchange %.3f us/iter (%s)\n", threads, cs,
                   1e3 * ms / iters, cudaGetErrorString(cudaGetLastError()));
        }
    }
    return 0;
}
