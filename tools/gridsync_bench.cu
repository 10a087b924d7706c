// Microbenchmark: cost of a grid-wide barrier for the small-grid persistent kernels.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gridsync_bench tools/gridsync_bench.cu
// (a) cooperative_groups grid.sync(); (b) a hierarchical barrier: cluster barrier, one atomic per
// cluster on a global counter + acquire poll by that cluster's rank-0 thread, cluster barrier.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>

namespace cg = cooperative_groups;

__global__ void k_grid(int iters) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}

__global__ void k_hier(int iters, unsigned *count) {
    cg::cluster_group cl = cg::this_cluster();
    const unsigned nclusters = gridDim.x / cl.num_blocks();
    for (int i = 0; i < iters; ++i) {
        cl.sync();
        if (cl.block_rank() == 0 && threadIdx.x == 0) {
            __threadfence();
            atomicAdd(count, 1u);
            const unsigned target = nclusters * (unsigned)(i + 1);
            while (ld_acquire(count) < target) {
            }
        }
        cl.sync();
    }
}

// (c) a flat barrier: CTA barrier, one release-add per CTA on a global counter, thread 0 polls with
// acquire loads until every CTA of this round arrived, CTA barrier.
__global__ void k_flat(int iters, unsigned *count) {
    for (int i = 0; i < iters; ++i) {
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(count) : "memory");
            const unsigned target = gridDim.x * (unsigned)(i + 1);
            while (ld_acquire(count) < target) {
            }
        }
        __syncthreads();
    }
}

int main() {
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 2000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int blocks : {64, 128, 148, 256}) {
        for (int threads : {256, 512, 1024}) {
            void *args[] = {(void *)&iters};
            cudaLaunchCooperativeKernel((void *)k_grid, blocks, threads, args, 0, 0);   // warm-up
            cudaEventRecord(e0);
            cudaLaunchCooperativeKernel((void *)k_grid, blocks, threads, args, 0, 0);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            cudaError_t e = cudaGetLastError();
            printf("{\"kind\": \"grid.sync\", \"blocks\": %d, \"threads\": %d, \"us_per_sync\": %.3f, \"err\": \"%s\"}\n",
                   blocks, threads, 1e3 * ms / iters, cudaGetErrorString(e));
        }
    }
    unsigned *count;
    cudaMalloc(&count, 4);
    for (int blocks : {128, 148}) {
        for (int threads : {512, 1024}) {
            for (int rep = 0; rep < 2; ++rep) {
                cudaMemset(count, 0, 4);
                void *args[] = {(void *)&iters, (void *)&count};
                cudaEventRecord(e0);
                cudaLaunchCooperativeKernel((void *)k_flat, blocks, threads, args, 0, 0);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                cudaError_t e = cudaGetLastError();
                if (rep)
                    printf("{\"kind\": \"flat\", \"blocks\": %d, \"threads\": %d, \"us_per_sync\": %.3f, \"err\": \"%s\"}\n",
                           blocks, threads, 1e3 * ms / iters, cudaGetErrorString(e));
            }
        }
    }
    for (int cs : {8, 16}) {
        cudaFuncSetAttribute(k_hier, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        for (int blocks : {128, 256}) {
            if (blocks % cs) continue;
            for (int rep = 0; rep < 2; ++rep) {
                cudaMemset(count, 0, 4);
                cudaLaunchConfig_t cfg = {};
                cudaLaunchAttribute at[2];
                at[0].id = cudaLaunchAttributeClusterDimension;
                at[0].val.clusterDim.x = cs;
                at[0].val.clusterDim.y = 1;
                at[0].val.clusterDim.z = 1;
                at[1].id = cudaLaunchAttributeCooperative;
                at[1].val.cooperative = 1;
                cfg.gridDim = dim3(blocks);
                cfg.blockDim = dim3(512);
                cfg.attrs = at;
                cfg.numAttrs = 2;
                cudaEventRecord(e0);
                cudaError_t le = cudaLaunchKernelEx(&cfg, k_hier, iters, count);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms = 0;
                cudaEventElapsedTime(&ms, e0, e1);
                cudaError_t e = cudaGetLastError();
                if (rep == 1)
                    printf("{\"kind\": \"cluster-hier\", \"cluster\": %d, \"blocks\": %d, \"us_per_sync\": %.3f, \"launch\": \"%s\", \"err\": \"%s\"}\n",
                           cs, blocks, 1e3 * ms / iters, cudaGetErrorString(le), cudaGetErrorString(e));
            }
        }
    }
    return 0;
}
