// mma_rate.cu -- microbenchmark: back-to-back tcgen05.mma (kind::f16, bf16 -> fp32) throughput
// per SM with operands already in shared memory (contents irrelevant), for K-major vs MN-major B
// (128-B swizzle descriptors as used by the BLR kernels) and several N.
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o mma_rate mma_rate.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= 1ull << 46;
    d |= 2ull << 61;  // SW128
    return d;
}

__global__ void __launch_bounds__(128, 1) k(int iters, int N, int b_mn, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint8_t* base = (uint8_t*)(((uintptr_t)sm + 1023) & ~(uintptr_t)1023);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t a = smem_u32(base), b = smem_u32(base + 65536);
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(b_mn & 1) << 16) | ((uint32_t)(N >> 3) << 17) |
                           ((128u >> 4) << 24);
    unsigned long long t0 = 0, t1 = 0;
    if (warp == 1 && lane == 0) {
        const uint64_t ad0 = desc(a, 16, 1024);
        const uint64_t bd0 = b_mn ? desc(b, 64 * 2 * 64, 1024) : desc(b, 16, 1024);
        const uint32_t bstep = b_mn ? 2048 : 32;
        t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const uint64_t ad = ad0 + ((kk * 32) >> 4);
                const uint64_t bd = bd0 + ((kk * bstep) >> 4);
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(slot),
                    "l"(ad), "l"(bd), "r"(idesc), "r"(1));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                         : "=r"(ok)
                         : "r"(smem_u32(&bar)));
        t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

int main() {
    unsigned long long* d;
    cudaMalloc(&d, 8 * 148);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    const int iters = 2000;
    for (int bmn = 0; bmn <= 1; ++bmn)
        for (int N : {64, 128, 192, 256}) {
            k<<<148, 128, 200 * 1024>>>(iters, N, bmn, d);
            k<<<148, 128, 200 * 1024>>>(iters, N, bmn, d);
            cudaDeviceSynchronize();
            unsigned long long h;
            cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
            const double macs = double(iters) * 4 * 128 * N * 16;
            printf("B %s N=%3d: %.0f MAC/clk/SM (%.2f of 4096), %.1f clk per MMA (%s)\n", bmn ? "MN-major" : "K-major ", N,
                   macs / h, macs / h / 4096, double(h) / (iters * 4), cudaGetErrorString(cudaGetLastError()));
        }
    return 0;
}
