// tma_tensor_bench.cu -- throughput of 3D TMA tensor box loads (cp.async.bulk.tensor.3d) in a
// producer / consumer ring, as used by the streaming stage kernel; no arithmetic.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_tensor_bench tools/tma_tensor_bench.cu
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void wait(uint64_t *b, uint32_t par) {
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                     su32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void tma3(void *dst, const CUtensorMap *m, int x, int y, int z, uint64_t *b) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
                 ::"r"(su32(dst)), "l"((uint64_t)m), "r"(x), "r"(y), "r"(z), "r"(su32(b)) : "memory");
}

// grid of blocks; block b streams rows of strip (b % strips) of plane-group (b / strips) ...
__global__ void ring(const __grid_constant__ CUtensorMap map, int nx_strips, int bx, int R, int rows_total, int S, int NW,
                     unsigned long long *sink) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *full = (uint64_t *)sm, *empty = full + 32;
    char *slots = (char *)(empty + 32);
    const int t = threadIdx.x, w = t >> 5, l = t & 31;
    if (t == 0) {
        for (int q = 0; q < S; ++q) { mbar_init(&full[q], 1); mbar_init(&empty[q], NW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int strip = blockIdx.x % nx_strips, grp = blockIdx.x / nx_strips, ngrp = gridDim.x / nx_strips;
    const int rows = rows_total / ngrp, y0 = grp * rows;
    const uint32_t bytes = (uint32_t)(bx * R * 3 * 8);
    const int nsl = rows / R;
    if (w == NW) {
        if (l) return;
        for (int i = 0; i < nsl; ++i) {
            const int s = i % S;
            if (i >= S) wait(&empty[s], ((i / S) - 1) & 1);
            expect_tx(&full[s], bytes);
            tma3(slots + (size_t)s * bytes, &map, strip * (bx - 4), y0 + i * R, 0, &full[s]);
        }
        return;
    }
    unsigned long long acc = 0;
    for (int i = 0; i < nsl; ++i) {
        const int s = i % S;
        wait(&full[s], (i / S) & 1);
        acc += *(const unsigned long long *)(slots + (size_t)s * bytes + ((t * 8) % bytes));
        __syncwarp();
        if (l == 0) arrive(&empty[s]);
    }
    if (acc == 0x123456789ull) *sink = acc;
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int nx = 4096 + 4, ny = 8192;           // 3 planes of 4100 x 8192 doubles = 806 MB
    double *src;
    unsigned long long *sink;
    cudaMalloc(&src, (size_t)nx * ny * 3 * 8);
    cudaMalloc(&sink, 8);
    cudaMemset(src, 0, (size_t)nx * ny * 3 * 8);
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    printf("bx R S blocks/SM GBps\n");
    const int cfg[][4] = {{240, 1, 8, 2}, {240, 2, 6, 2}, {240, 4, 4, 2}, {240, 4, 3, 2}, {240, 8, 2, 2},
                          {240, 2, 8, 2}, {240, 4, 4, 1}, {240, 8, 4, 1}, {128, 4, 6, 3}, {256, 4, 4, 2},
                          {240, 2, 12, 1}, {64, 8, 6, 4}};
    for (auto &c : cfg) {
        const int bx = c[0], R = c[1], S = c[2], bps = c[3], NW = 8;
        CUtensorMap m;
        cuuint64_t dims[3] = {(cuuint64_t)nx, (cuuint64_t)ny, 3};
        cuuint64_t str[2] = {(cuuint64_t)nx * 8, (cuuint64_t)nx * ny * 8};
        cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)R, 3}, es[3] = {1, 1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
        const int strips = (nx - 4) / (bx - 4);
        int blocks = nsm * bps / strips * strips;
        const size_t smem = 512 + (size_t)S * bx * R * 3 * 8;
        const int ngrp = blocks / strips;
        const int rows_total = ny / ngrp / R * R * ngrp;
        ring<<<blocks, 32 * NW + 32, smem>>>(m, strips, bx, R, rows_total, S, NW, sink);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        ring<<<blocks, 32 * NW + 32, smem>>>(m, strips, bx, R, rows_total, S, NW, sink);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)strips * ngrp * (rows_total / ngrp / R) * bx * R * 3 * 8;
        cudaError_t e = cudaGetLastError();
        printf("%d %d %d %d %.0f %s\n", bx, R, S, bps, bytes / ms / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
