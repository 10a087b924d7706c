// ring_rw_bench.cu -- read+write streaming throughput of the stage kernels' memory skeleton, no
// arithmetic: TMA 3D box loads (bx x R rows x 3 fields) into a ring of S slots gated by
// full/empty mbarriers, NW consumer warps (60 columns each, lanes 1..30 with 128-bit accesses)
// copying each row of the 3 fields from shared memory to an output buffer with STG.
//   hold = 1: a slot is released one box late (as the stage kernels do: rows k-1, k-2 of the
//   previous box are still read); hold = 0: released as soon as it is consumed.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ring_rw_bench tools/ring_rw_bench.cu -lcuda
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

__global__ void ring(const __grid_constant__ CUtensorMap map, double *out, int pitch, long fstride, int strips, int Wo,
                     int R, int rows_total, int S, int NW, int hold) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *full = (uint64_t *)sm, *empty = full + 32;
    double *slots = (double *)(sm + 512);
    const int t = threadIdx.x, w = t >> 5, l = t & 31;
    const int bx = Wo + 8;
    if (t == 0) {
        for (int q = 0; q < S; ++q) { mbar_init(&full[q], 1); mbar_init(&empty[q], NW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int strip = blockIdx.x % strips, grp = blockIdx.x / strips, ngrp = gridDim.x / strips;
    const int rows = rows_total / ngrp, y0 = grp * rows;
    const int slot_el = (3 * R * bx * 8 + 127) / 128 * 128 / 8;
    const uint32_t bytes = (uint32_t)(3 * R * bx * 8);
    const int nsl = rows / R;
    if (w == NW) {
        if (l) return;
        for (int i = 0; i < nsl; ++i) {
            const int s = i % S;
            if (i >= S) wait(&empty[s], ((i / S) - 1) & 1);
            expect_tx(&full[s], bytes);
            tma3(slots + (size_t)s * slot_el, &map, strip * Wo, y0 + i * R, 0, &full[s]);
        }
        return;
    }
    const int cx = 60 * w + 2 * l - 2;
    const bool st = l >= 1 && l <= 30 && cx < Wo;
    for (int i = 0; i < nsl; ++i) {
        const int s = i % S;
        wait(&full[s], (i / S) & 1);
        const double *sl = slots + (size_t)s * slot_el + 4 + cx;
        for (int u = 0; u < R; ++u)
            if (st)
#pragma unroll
                for (int f = 0; f < 3; ++f) {
                    const double2 v = *(const double2 *)(sl + (f * R + u) * bx);
                    *(double2 *)(out + f * fstride + (long)(y0 + i * R + u) * pitch + strip * Wo + cx + 4) =
                        make_double2(v.x + 1.0, v.y);
                }
        __syncwarp();
        if (l == 0) {
            if (!hold) arrive(&empty[s]);
            else if (i >= 1) arrive(&empty[(i - 1) % S]);
        }
    }
    if (hold && l == 0) arrive(&empty[(nsl - 1) % S]);
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int nx = 4096, ny = 4096, pitch = nx + 8;
    const long fstride = (long)ny * pitch;
    double *src, *dst;
    cudaMalloc(&src, fstride * 3 * 8);
    cudaMalloc(&dst, fstride * 3 * 8);
    cudaMemset(src, 0, fstride * 3 * 8);
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    auto enc = (PFN_cuTensorMapEncodeTiled_v12000)p;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    const int strips = 18, Wo = 228, bx = Wo + 8, NW = 4;
    // {R, S, blocks/SM, hold}
    const int cfg[][4] = {{2, 6, 3, 1}, {2, 6, 3, 0}, {2, 4, 3, 1}, {2, 8, 2, 1}, {2, 8, 2, 0}, {4, 4, 2, 1},
                          {4, 4, 2, 0}, {2, 12, 1, 1}, {2, 3, 3, 1}, {2, 5, 4, 0}, {1, 8, 3, 0}, {1, 12, 2, 0}};
    for (auto &c : cfg) {
        const int R = c[0], S = c[1], bps = c[2], hold = c[3];
        if (R == 1 && hold) continue;
        CUtensorMap m;
        cuuint64_t dims[3] = {(cuuint64_t)pitch, (cuuint64_t)ny, 3};
        cuuint64_t str[2] = {(cuuint64_t)pitch * 8, (cuuint64_t)fstride * 8};
        cuuint32_t box[3] = {(cuuint32_t)bx, (cuuint32_t)R, 3}, es[3] = {1, 1, 1};
        CUresult r = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, src, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); continue; }
        const int blocks = nsm * bps / strips * strips;
        const size_t smem = 512 + (size_t)S * ((3 * R * bx * 8 + 127) / 128 * 128);
        const int ngrp = blocks / strips;
        const int rows_total = ny / ngrp / R * R * ngrp;
        ring<<<blocks, 32 * NW + 32, smem>>>(m, dst, pitch, fstride, strips, Wo, R, rows_total, S, NW, hold);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int k = 0; k < 3; ++k)
            ring<<<blocks, 32 * NW + 32, smem>>>(m, dst, pitch, fstride, strips, Wo, R, rows_total, S, NW, hold);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double by = 2.0 * 3 * (double)rows_total * nx * 8 * 3;
        cudaError_t e = cudaGetLastError();
        printf("R %d S %d blocks/SM %d hold %d smem %zu KB: %.0f GB/s read+write %s\n", R, S, bps, hold, smem / 1024,
               by / ms / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
