// tma_bench.cu -- microbenchmark of 1D TMA bulk copies (cp.async.bulk global->shared) in the
// producer / consumer ring structure of the streaming stage kernel, without any arithmetic.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tma_bench tools/tma_bench.cu
// Prints achieved read GB/s for combinations of copy size, copies per slot, ring depth, blocks/SM.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t su32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *b, uint32_t c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void expect_tx(uint64_t *b, uint32_t n) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(n) : "memory");
}
__device__ __forceinline__ void bulk(void *d, const void *s, uint32_t n, uint64_t *b) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     su32(d)),
                 "l"(s), "r"(n), "r"(su32(b))
                 : "memory");
}
__device__ __forceinline__ void wait(uint64_t *b, uint32_t par) {
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}" ::"r"(
                     su32(b)),
                 "r"(par)
                 : "memory");
}
__device__ __forceinline__ void arrive(uint64_t *b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}

// Each block streams `rows` loads; load i copies K chunks of B bytes (chunk f of row r at
// src + ((blk*rows + r) * K + f) * pitch).  One producer lane, NW consumer warps.
__global__ void ring(const char *src, size_t pitch, int rows, int K, int B, int S, int NW, unsigned long long *sink, int mode) {
    extern __shared__ __align__(128) unsigned char sm[];
    uint64_t *full = (uint64_t *)sm, *empty = full + 64;
    char *slots = (char *)(empty + 64);
    const int t = threadIdx.x, w = t >> 5, l = t & 31;
    if (t == 0) {
        for (int q = 0; q < S; ++q) { mbar_init(&full[q], 1); mbar_init(&empty[q], NW); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const size_t slot_bytes = (size_t)K * B;
    if (w == NW) {
        if (l) return;
        long long t0 = clock64(), tw = 0, ti = 0;
        for (int i = 0; i < rows; ++i) {
            const int s = i % S;
            long long a = clock64();
            if (i >= S && mode != 1) wait(&empty[s], ((i / S) - 1) & 1);
            long long b = clock64();
            tw += b - a;
            expect_tx(&full[s], (uint32_t)slot_bytes);
            for (int f = 0; f < K; ++f)
                bulk(slots + s * slot_bytes + (size_t)f * B,
                     src + (((size_t)blockIdx.x * rows + i) * K + f) * pitch, B, &full[s]);
            ti += clock64() - b;
        }
        if (blockIdx.x == 0) printf("    producer: total %lld cyc/slot, empty-wait %lld, issue %lld\n", (clock64() - t0) / rows, tw / rows, ti / rows);
        return;
    }
    unsigned long long acc = 0;
    for (int i = 0; i < rows; ++i) {
        const int s = i % S;
        if (mode != 2) wait(&full[s], (i / S) & 1);
        acc += *(const unsigned long long *)(slots + s * slot_bytes + ((t * 8) % slot_bytes));
        __syncwarp();
        if (l == 0) arrive(&empty[s]);
    }
    if (acc == 0x123456789ull) *sink = acc;
}

int main() {
    int nsm;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    const size_t total = (size_t)3 << 30;   // 3 GiB source
    char *src;
    unsigned long long *sink;
    cudaMalloc(&src, total);
    cudaMalloc(&sink, 8);
    cudaMemset(src, 1, total);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    printf("B K S blocks/SM mode GBps\n");
    const int cfgs[][5] = {{2048, 3, 8, 2, 0}, {2048, 3, 8, 2, 1}, {2048, 3, 8, 2, 2}, {2048, 1, 8, 2, 0},
                           {2048, 6, 8, 2, 0}, {2048, 12, 4, 2, 0}, {2048, 3, 8, 1, 0}, {2048, 3, 8, 1, 2}};
    for (auto &c : cfgs) {
        const int B = c[0], K = c[1], S = c[2], bps = c[3], mode = c[4], NW = 9;
        const size_t smem = 64 * 16 + (size_t)S * K * B;
        const int blocks = nsm * bps;
        const size_t pitch = B;
        const int rows = (int)(total / ((size_t)blocks * K * pitch)) - 1;
        ring<<<blocks, 32 * NW + 32, smem>>>(src, pitch, rows, K, B, S, NW, sink, mode);
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        ring<<<blocks, 32 * NW + 32, smem>>>(src, pitch, rows, K, B, S, NW, sink, mode);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double bytes = (double)blocks * rows * K * B;
        cudaError_t e = cudaGetLastError();
        printf("%d %d %d %d %d %.0f %s\n", B, K, S, bps, mode, bytes / ms / 1e6, e == cudaSuccess ? "" : cudaGetErrorString(e));
    }
    return 0;
}
