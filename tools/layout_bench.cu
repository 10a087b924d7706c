// layout_bench.cu -- does the field layout change HBM efficiency for the streaming stage pattern?
// Blocks (grouped like the stage kernels: `strips` blocks per group, groups own disjoint row
// ranges) stream rows of a strip, reading 3 fields and writing 3 fields per row, with
//   planar      [field][row][x]  (3 read + 3 write streams per block), or
//   interleaved [row][field][x]  (1 read + 1 write stream per block).
// No arithmetic.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/layout_bench tools/layout_bench.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void stream(const double2 *__restrict__ in, double2 *__restrict__ out, int nx2, int rows, int strips,
                       int W2, int inter, long fstride2) {
    const int strip = blockIdx.x % strips, g = blockIdx.x / strips, G = gridDim.x / strips;
    const int r0 = (int)((long)rows * g / G), r1 = (int)((long)rows * (g + 1) / G);
    const int x = strip * W2 + threadIdx.x;
    if (threadIdx.x >= W2 || x >= nx2) return;
    for (int r = r0; r < r1; ++r) {
        double2 v[3];
#pragma unroll
        for (int f = 0; f < 3; ++f) {
            const long o = inter == 1 ? ((long)r * 3 + f) * nx2 + x : f * fstride2 + (long)r * nx2 + x;
            v[f] = inter == 2 ? make_double2(r, f) : in[o];
        }
#pragma unroll
        for (int f = 0; f < 3; ++f) {
            const long o = inter == 1 ? ((long)r * 3 + f) * nx2 + x : f * fstride2 + (long)r * nx2 + x;
            out[o] = make_double2(v[f].x + 1.0, v[f].y);
        }
    }
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const int nx = 512, members = 64, ny = 512;
    const long rows = (long)members * ny;        // members stacked in rows (same per-field size)
    const int nx2 = nx / 2;
    const long n2 = rows * nx2 * 3;
    double2 *a, *b;
    cudaMalloc(&a, n2 * 16);
    cudaMalloc(&b, n2 * 16);
    cudaMemset(a, 0, n2 * 16);
    cudaMemset(b, 0, n2 * 16);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int strips : {3}) {
        const int W2 = (nx2 + strips - 1) / strips;
        for (int bps : {1, 2, 4, 8}) {
            const int G = nsm * bps / strips;
            for (int inter = 0; inter < 3; inter += 2) {
                stream<<<G * strips, 256, 0>>>(a, b, nx2, (int)rows, strips, W2, inter, rows * nx2);
                cudaEventRecord(e0);
                for (int k = 0; k < 5; ++k) stream<<<G * strips, 256, 0>>>(a, b, nx2, (int)rows, strips, W2, inter, rows * nx2);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                float ms;
                cudaEventElapsedTime(&ms, e0, e1);
                printf("strips %d blocks/SM %d %-11s %.0f GB/s\n", strips, bps, inter == 2 ? "write-only" : "planar r+w",
                       (inter == 2 ? 1.0 : 2.0) * n2 * 16 * 5 / ms / 1e6);
            }
        }
    }
    // plain copy reference
    cudaEventRecord(e0);
    for (int k = 0; k < 5; ++k) cudaMemcpyAsync(b, a, n2 * 16, cudaMemcpyDeviceToDevice);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("cudaMemcpy D2D %.0f GB/s (read+write)\n", 2.0 * n2 * 16 * 5 / ms / 1e6);
    return 0;
}
