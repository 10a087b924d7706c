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

__global__ void mma_kernel(int M, int N, int iters, int layout, int nwi, int walk, long long *cyc) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ uint32_t tslot;
    __shared__ __align__(8) uint64_t bars[4];
    uint64_t &bar = bars[threadIdx.x >> 5 & 3];
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(&tslot)) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::: "memory");
    }
    for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t *>(sm)[i] = 0x3f803f80u;
    if ((threadIdx.x & 31) == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    const uint32_t tmem = tslot;
    if ((threadIdx.x & 31) == 0 && warp < nwi) {
        const uint32_t a = smem_u32(sm), b = a + 64 * 1024;
        // layout 0: compact canonical (A: 8-row groups 128 B apart, K chunks M*16 B apart)
        // layout 1: U-Net row kernel (K chunk planes 2080 B apart, start 16 B into the plane)
        // layout 2: 128-byte swizzle, K-major (8-row atoms of 1024 B, SBO = 1024), layout type 2 at bits 61-63
        const uint64_t ad = layout == 0 ? sdesc(a, (uint32_t)M * 16, 128)
                          : layout == 1 ? sdesc(a + 16, 2080, 128)
                                        : (sdesc(a, 16, 1024) | (2ull << 61));
        const uint64_t bd = sdesc(b, (uint32_t)N * 16, 128);
        const uint32_t id = idesc_bf16(M, N);
        const uint32_t acc = tmem + (uint32_t)(warp * N);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(acc),
                "l"(ad + (walk ? (uint64_t)(((i * (layout == 2 ? 1024 : 2048)) & 32767) >> 4) + (layout == 1 ? (uint64_t)(i % 3) : 0) : 0)), "l"(bd), "r"(id), "r"(i)
                : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar))
                     : "memory");
        asm volatile(
            "{\n\t.reg .pred p;\nW:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W;\n}" ::"r"(
                smem_u32(&bar))
            : "memory");
        long long t1 = clock64();
        if (warp == 0) cyc[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem) : "memory");
}


// The whole warp runs the loop (descriptors warp-uniform, in uniform registers) and one elected
// lane issues each MMA: no per-MMA R2UR / election loop.
__device__ int g_stop;
__global__ void mma_uniform_kernel(int M, int N, int iters, int walk, long long *cyc, int ldw, int cpw,
                                   const uint4 *gsrc) {
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
    __shared__ int stop;
    if (threadIdx.x == 0) stop = 0;
    __syncthreads();
    if (warp >= 4 && warp < 4 + ldw) {   // epilogue-like TMEM readers on columns 128..255
        uint32_t r[16];
        const uint32_t ta = tmem + 128 + ((uint32_t)(32 * (warp & 3)) << 16);
        while (!*(volatile int *)&stop) {
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
                "%15}, [%16];\n"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
                  "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                : "r"(ta));
            asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
            if (r[3] == 0x12345) g_stop = 1;
        }
    }
    if (warp == 8 && cpw) {   // bulk copies of 2080 B into smem [96 KB, 128 KB), one mbarrier round per 8
        __shared__ __align__(8) uint64_t cb;
        if ((threadIdx.x & 31) == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&cb)) : "memory");
            uint32_t ph = 0;
            while (!*(volatile int *)&stop) {
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&cb)), "r"(8 * 2080) : "memory");
                for (int j = 0; j < 8; ++j)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                     smem_u32(sm) + 96 * 1024 + j * 2080 + 16),
                                 "l"(gsrc + j * 130), "r"(2080), "r"(smem_u32(&cb))
                                 : "memory");
                asm volatile("{\n\t.reg .pred p;\nW3:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W3;\n}" ::"r"(
                                 smem_u32(&cb)), "r"(ph)
                             : "memory");
                ph ^= 1;
            }
        }
    }
    if (warp == 0) {
        const uint32_t a = smem_u32(sm), b = a + 64 * 1024;
        const uint64_t ad = sdesc(a + 16, 2080, 128);
        const uint64_t bd = sdesc(b, (uint32_t)N * 16, 128);
        const uint32_t id = idesc_bf16(M, N);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint64_t adi = ad + (walk ? (uint64_t)(((i * 2080) & 32767) >> 4) : 0);
            asm volatile(
                "{\n\t.reg .pred p, e;\n\telect.sync _|e, 0xffffffff;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                "l"(adi), "l"(bd), "r"(id), "r"(i)
                : "memory");
        }
        asm volatile("{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
                     "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}\n" ::"r"(smem_u32(&bar))
                     : "memory");
        asm volatile(
            "{\n\t.reg .pred p;\nW2:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W2;\n}" ::"r"(
                smem_u32(&bar))
            : "memory");
        long long t1 = clock64();
        if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
        if (threadIdx.x == 0) *(volatile int *)&stop = 1;
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
    for (int walk = 0; walk < 2; ++walk)
    for (int nwi = 1; nwi <= 4; nwi *= 2)
    for (int layout = 0; layout < 3; ++layout)
        for (int M : {64, 128})
            for (int N : {16, 32, 64, 128, 256}) {
                if (layout >= 1 && M != 128) continue;
                if (nwi > 1 && (layout >= 1 || N > 64)) continue;
                if (walk && (nwi > 1 || M != 128 || N > 64)) continue;
                mma_kernel<<<148, 128, 128 * 1024>>>(M, N, iters, layout, nwi, walk, d);
                cudaError_t e = cudaDeviceSynchronize();
                long long h[148];
                cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
                double s = 0;
                for (int i = 0; i < 148; ++i) s += (double)h[i];
                const double cpm = s / 148 / iters / nwi;   // per MMA of the SM (nwi issuing warps)
                const double macs = (double)M * N * 16;
                printf("{\"walk\": %d, \"issuing_warps\": %d, \"layout\": %d, \"M\": %d, \"N\": %d, \"cycles_per_mma\": %.2f, \"macs_per_cycle\": %.1f, \"err\": \"%s\"}\n",
                       walk, nwi, layout, M, N, cpm, macs / cpm, cudaGetErrorString(e));
            }
    cudaFuncSetAttribute(mma_uniform_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
    uint4 *gsrc;
    cudaMalloc(&gsrc, 1 << 20);
    cudaMemset(gsrc, 0, 1 << 20);
    for (int ldw : {0, 4})
    for (int cpw : {0, 1})
    for (int walk = 0; walk < 2; ++walk)
        for (int N : {16, 32, 64, 128, 256}) {
            if ((ldw || cpw) && (N > 32 || !walk)) continue;
            mma_uniform_kernel<<<148, 320, 128 * 1024>>>(128, N, iters, walk, d, ldw, cpw, gsrc);
            cudaError_t e = cudaDeviceSynchronize();
            long long h[148];
            cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
            double s = 0;
            for (int i = 0; i < 148; ++i) s += (double)h[i];
            const double cpm = s / 148 / iters;
            printf("{\"tmem_readers\": %d, \"bulk_copier\": %d, \"uniform_issue\": 1, \"walk\": %d, \"layout\": 1, \"M\": 128, \"N\": %d, \"cycles_per_mma\": %.2f, \"macs_per_cycle\": %.1f, \"err\": \"%s\"}\n",
                   ldw, cpw, walk, N, cpm, 128.0 * N * 16 / cpm, cudaGetErrorString(e));
        }
    return 0;
}
