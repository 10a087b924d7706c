// store_bench.cu -- write-only streaming throughput of the stage kernels' store pattern:
// blocks of NW warps own strips of W columns (fp64, 60 per warp, 128-bit stores by lanes 1..30),
// grouped like the stage kernels, each block walking its row range and storing 3 field rows per
// row.  Compares against full 32-lane warps.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/store_bench tools/store_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void st(double *out, int nx, int pitch, long fstride, int rows, int strips, int Wo, int lanes30, int extra_warp) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x / 32 - extra_warp;
    if (warp >= nw) return;
    const int strip = blockIdx.x % strips, g = blockIdx.x / strips, G = gridDim.x / strips;
    const int r0 = (int)((long)rows * g / G), r1 = (int)((long)rows * (g + 1) / G);
    const int per = lanes30 ? 60 : 64;
    const int x = strip * Wo + per * warp + 2 * (lanes30 ? lane - 1 : lane);
    const bool ok = (!lanes30 || (lane >= 1 && lane <= 30)) && per * warp + 2 * (lanes30 ? lane - 1 : lane) < Wo && x < nx;
    for (int r = r0; r < r1; ++r) {
        if (ok) {
#pragma unroll
            for (int f = 0; f < 3; ++f)
                *reinterpret_cast<double2 *>(out + f * fstride + (long)(r + 2) * pitch + x + 4) = make_double2(r, f);
        }
    }
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int nx = 4096, ny = 4096, pitch = nx + 8;
    const long fstride = (long)(ny + 4) * pitch;
    double *o;
    cudaMalloc(&o, fstride * 3 * 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int strips = 18, Wo = 228;
    cudaFuncSetAttribute(st, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    for (int lanes30 = 1; lanes30 < 2; ++lanes30)
        for (int extra = 1; extra < 2; ++extra)
            for (int bps : {3, 4})
            for (int smkb : {0, 16, 32, 48, 54, 64}) {
                const int G = nsm * bps / strips;
                const int nw = lanes30 ? 4 : 4;
                const int threads = 32 * (nw + extra);
                const size_t sm = (size_t)smkb * 1024;
                st<<<G * strips, threads, sm>>>(o, nx, pitch, fstride, ny, strips, Wo, lanes30, extra);
                cudaEventRecord(e0);
                for (int k = 0; k < 5; ++k) st<<<G * strips, threads, sm>>>(o, nx, pitch, fstride, ny, strips, Wo, lanes30, extra);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("smem/block %d KB blocks/SM %d: %.0f GB/s write\n", smkb, bps,
                       3.0 * nx * ny * 8 * 5 / ms / 1e6);
            }
    return 0;
}
