// tma_ingress.cu -- microbenchmark: how fast can SMs pull tiles into shared memory with TMA?
//   mode 0: every CTA streams its own distinct slice of a buffer (L2-resident or HBM-sized)
//   mode 1: every CTA streams the SAME slice (all CTAs read identical addresses)
//   mode 2: clusters of C CTAs; the slice is split so each CTA loads 1/C and multicasts to all
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o tma_ingress tma_ingress.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e = (x);                                                                    \
        if (e != cudaSuccess) {                                                                 \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);     \
            exit(1);                                                                            \
        }                                                                                       \
    } while (0)

constexpr int STAGES = 12;
constexpr int BOX_ROWS = 128;  // 128 rows x 128 B = 16 KB per box

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(128, 1) ingress(const __grid_constant__ CUtensorMap tm, int iters, int mode,
                                                   int rows_per_cta, int total_rows, int csize,
                                                   unsigned long long* cycles, int nst, int bps) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t full[16], empty[16];
    uint32_t crank = 0;
    if (mode == 2) asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&empty[s])),
                         "r"(mode == 2 ? csize : 1));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (mode == 2) {
        asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;");
    } else {
        __syncthreads();
    }
    const uint32_t stage_bytes = BOX_ROWS * 128 * bps;
    unsigned long long t0 = clock64();
    if (threadIdx.x == 0) {
        // producer: loads; consumer (thread 32) releases
    }
    if (threadIdx.x == 0) {
        int stage = 0;
        uint32_t phase = 0;
        int cta = blockIdx.x;
        int base = (mode == 0) ? (cta * rows_per_cta) % total_rows : 0;
        if (mode == 2) base = ((cta / csize) * rows_per_cta) % total_rows;
        int roff = 0;  // incremental row offset within this CTA's slice (no division in the loop)
        const int step_rows = BOX_ROWS * bps;
        for (int it = 0; it < iters; ++it) {
            // wait empty
            uint32_t ok = 0;
            while (!ok) {
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                    : "=r"(ok)
                    : "r"(smem_u32(&empty[stage])), "r"(phase ^ 1));
            }
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[stage])),
                         "r"(stage_bytes));
            const int row = base + roff;
            roff += step_rows;
            if (roff + step_rows > rows_per_cta) roff = 0;
            const uint32_t dst = smem_u32(smem + stage * stage_bytes);
            if (mode == 2) {
                // this CTA loads its 1/csize share of the box rows and multicasts it to all CTAs
                const int part = BOX_ROWS / csize;
                const uint16_t mask = (uint16_t)((1u << csize) - 1);
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster"
                    " [%0], [%1, {%3, %4}], [%2], %5;" ::"r"(dst + crank * part * 128),
                    "l"((uint64_t)&tm), "r"(smem_u32(&full[stage])), "r"(0), "r"(row + (int)crank * part), "h"(mask)
                    : "memory");
            } else {
                for (int b = 0; b < bps; ++b)
                    asm volatile(
                        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
                        " [%0], [%1, {%3, %4}], [%2];" ::"r"(dst + b * BOX_ROWS * 128),
                        "l"((uint64_t)&tm), "r"(smem_u32(&full[stage])), "r"(0), "r"(row + b * BOX_ROWS)
                        : "memory");
            }
            if (++stage == nst) { stage = 0; phase ^= 1; }
        }
    } else if (threadIdx.x == 32) {
        int stage = 0;
        uint32_t phase = 0;
        for (int it = 0; it < iters; ++it) {
            uint32_t ok = 0;
            while (!ok) {
                asm volatile(
                    "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                    : "=r"(ok)
                    : "r"(smem_u32(&full[stage])), "r"(phase));
            }
            if (mode == 2) {
                // release the slot in every CTA of the cluster (each producer waits for all consumers)
                for (int c = 0; c < csize; ++c) {
                    uint32_t remote;
                    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"(smem_u32(&empty[stage])), "r"(c));
                    // default (CTA-scope release) semantics: the .release.cluster form compiles to a
                    // MEMBAR.ALL.GPU per arrive, which is what made this mode look 7x slower in round 1
                    asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(remote) : "memory");
                }
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[stage])) : "memory");
            }
            if (++stage == nst) { stage = 0; phase ^= 1; }
        }
    }
    __syncthreads();
    if (mode == 2) asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;");
    if (threadIdx.x == 0) cycles[blockIdx.x] = clock64() - t0;
}

int main() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q));
    auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    int clk_khz = 0;
    CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
    const size_t big = size_t(2) << 30;  // 2 GiB buffer, rows of 128 B
    void* buf;
    CK(cudaMalloc(&buf, big));
    CK(cudaMemset(buf, 1, big));
    unsigned long long* cyc;
    CK(cudaMalloc(&cyc, sizeof(unsigned long long) * 4096));
    const int smem = 226 * 1024;
    CK(cudaFuncSetAttribute(ingress, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    CK(cudaFuncSetAttribute(ingress, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));

    struct Case { const char* name; int mode; int grid; size_t footprint; int csize; int nst; int bps; int smem_kb; int wide = 1; };
    std::vector<Case> cases = {
        {"L2 32MiB 4x32KB, no cluster", 0, sms, size_t(32) << 20, 1, 4, 2, 0},
        {"L2 multicast cluster 2, 8x16KB", 2, 148, size_t(32) << 20, 2, 8, 1, 0},
        {"L2 multicast cluster 4, 8x16KB", 2, 148, size_t(32) << 20, 4, 8, 1, 0},
        {"HBM 2GiB 4x32KB, no cluster", 0, sms, size_t(2) << 30, 1, 4, 2, 0},
        {"HBM multicast cluster 2, 8x16KB", 2, 148, size_t(2) << 30, 2, 8, 1, 0},
    };
    for (auto& c : cases) {
        const uint64_t total_rows = c.footprint / 128;
        CUtensorMap tm;
        const uint64_t dims[2] = {64ull * c.wide, total_rows / c.wide};
        const uint64_t str[1] = {128ull * c.wide};
        const uint32_t box[2] = {64, (uint32_t)(c.mode == 2 ? BOX_ROWS / c.csize : BOX_ROWS)};
        const uint32_t es[2] = {1, 1};
        CUresult r = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) { printf("encode failed %d\n", (int)r); return 1; }
        int ctas_sharing = (c.mode == 2) ? c.grid / c.csize : c.grid;
        int rows_per_cta = (int)(total_rows / c.wide / (c.mode == 1 ? 1 : ctas_sharing)) / BOX_ROWS * BOX_ROWS;
        if (c.mode == 1) rows_per_cta = (int)total_rows / BOX_ROWS * BOX_ROWS;
        const int iters = 2000;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(c.grid);
        cfg.blockDim = dim3(128);
        cfg.dynamicSmemBytes = c.smem_kb ? c.smem_kb * 1024 : (c.nst * c.bps + 1) * BOX_ROWS * 128;
        cudaLaunchAttribute at[1];
        int na = 0;
        if (c.mode == 2) {
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = c.csize;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            na = 1;
        }
        cfg.attrs = at;
        cfg.numAttrs = na;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEvent_t e0, e1;
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            CK(cudaEventRecord(e0));
            CK(cudaLaunchKernelEx(&cfg, ingress, tm, iters, c.mode, rows_per_cta, (int)total_rows, c.csize, cyc, c.nst, c.bps));
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            std::vector<unsigned long long> h(c.grid);
            CK(cudaMemcpy(h.data(), cyc, sizeof(unsigned long long) * c.grid, cudaMemcpyDeviceToHost));
            double mean = 0;
            for (auto v : h) mean += v;
            mean /= c.grid;
            const double bytes_per_cta = double(iters) * BOX_ROWS * 128 * c.bps;  // bytes landing in each CTA's smem
            if (rep == 1)
                printf("%-36s grid %4d: %.1f B/clk/SM delivered, %.2f TB/s delivered chip-wide (%.3f ms)\n", c.name,
                       c.grid, bytes_per_cta / mean, bytes_per_cta * c.grid / (ms * 1e-3) / 1e12, ms);
        }
    }
    return 0;
}
