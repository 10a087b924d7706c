// Microbenchmark: issue cost of tcgen05.mma kind::f16 (bf16 x bf16 -> fp32, SS operands, K-major,
// no swizzle) per instruction for M in {64, 128} and N in {16 .. 256}, one CTA per SM, one issuing
// thread, back-to-back MMAs into one TMEM accumulator (commit + wait at the end).  Also the A
// operand laid out like the U-Net row kernel (LBO = 2080 B chunk planes, start shifted by 16 B).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mma_bench tools/mma_bench.cu
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)((lbo >> 4) & 0x3FFFu) << 16) |
           ((uint64_t)((sbo >> 4) & 0x3FFFu) << 32) | (1ull << 46);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int m, int n) {
    return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}

__global__ void mma_kernel(int M, int N, int iters, int layout, long long *cyc) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(&tslot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3f803f80u;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint32_t a = smem_u32(sm), b = a + 64 * 1024;
        // layout 0: compact canonical (A: 8-row groups 128 B apart, K chunks M*16 B apart)
        // layout 1: U-Net row kernel (K chunk planes 2080 B apart, start 16 B into the plane)
        const uint64_t ad = layout == 0 ? sdesc(a, (uint32_t)M * 16, 128) : sdesc(a + 16, 2080, 128);
        const uint64_t bd = sdesc(b, (uint32_t)N * 16, 128);
        const uint32_t id = idesc_bf16(M, N);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                "l"(ad), "l"(bd), "r"(id), "r"(i)
                : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar))
                     : "memory");
        asm volatile(
            "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
                smem_u32(&bar))
            : "memory");
        long long t1 = clock64();
        cyc[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem) : "memory");
}

int main() {
    long long *d;
    cudaMalloc(&d, 148 * sizeof(long long));
    cudaFuncSetAttribute(mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
    const int iters = 4096;
    for (int layout = 0; layout < 2; ++layout)
        for (int M : {64, 128})
            for (int N : {16, 32, 64, 128, 256}) {
                if (layout == 1 && M != 128) continue;
                mma_kernel<<<148, 128, 128 * 1024>>>(M, N, iters, layout, d);
                cudaError_t e = cudaDeviceSynchronize();
                long long h[148];
                cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
                double s = 0;
                for (int i = 0; i < 148; ++i) s += (double)h[i];
                const double cpm = s / 148 / iters;
                const double macs = (double)M * N * 16;
                printf("{\"layout\": %d, \"M\": %d, \"N\": %d, \"cycles_per_mma\": %.2f, \"macs_per_cycle\": %.1f, \"err\": \"%s\"}\n",
                       layout, M, N, cpm, macs / cpm, cudaGetErrorString(e));
            }
    return 0;
}
