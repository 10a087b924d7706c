// fp64_peak.cu -- DFMA / FFMA throughput and dependent-chain latency on this GPU (ALU roofline
// of DESIGN.md 7).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/fp64_peak tools/fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <typename T, int CH>
__global__ void thr(T *out, int iters, T a, T b) {
    T x[CH];
#pragma unroll
    for (int c = 0; c < CH; ++c) x[c] = (T)(threadIdx.x + c);
    for (int i = 0; i < iters; ++i)
#pragma unroll
        for (int c = 0; c < CH; ++c) x[c] = x[c] * a + b;
    T s = 0;
#pragma unroll
    for (int c = 0; c < CH; ++c) s += x[c];
    if (s == (T)1.2345) out[0] = s;
}

__global__ void lat(double *out, long long *cyc, int iters, double a, double b) {
    double x = threadIdx.x;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) x = fma(x, a, b);
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[0] = x; }
}

int main() {
    int nsm, clk;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    double *o; long long *cy;
    cudaMalloc(&o, 64); cudaMalloc(&cy, 64);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    const int iters = 1 << 14;
    for (int bs : {256, 512, 1024}) {
        const int blocks = nsm * (2048 / bs);
        thr<double, 8><<<blocks, bs>>>(o, 16, 1.0000001, 1e-9);
        cudaEventRecord(e0);
        thr<double, 8><<<blocks, bs>>>(o, iters, 1.0000001, 1e-9);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double fl = 2.0 * 8 * iters * (double)blocks * bs;
        printf("DFMA block %d: %.2f TFLOP/s fp64\n", bs, fl / ms / 1e9);
    }
    {
        const int bs = 512, blocks = nsm * 4;
        thr<float, 8><<<blocks, bs>>>((float *)o, 16, 1.0000001f, 1e-9f);
        cudaEventRecord(e0);
        thr<float, 8><<<blocks, bs>>>((float *)o, iters, 1.0000001f, 1e-9f);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("FFMA: %.2f TFLOP/s fp32\n", 2.0 * 8 * iters * (double)blocks * bs / ms / 1e9);
    }
    lat<<<1, 32>>>(o, cy, 4096, 1.0000001, 1e-9);
    long long c; cudaMemcpy(&c, cy, 8, cudaMemcpyDeviceToHost);
    printf("DFMA dependent latency: %.2f cycles; SMs %d, clock attr %d kHz\n", c / 4096.0, nsm, clk);
    return 0;
}
