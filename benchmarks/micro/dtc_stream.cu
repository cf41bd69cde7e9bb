// dtc_stream.cu -- how should a small-token (decode) kernel tile a row-major [K][N] bf16 weight so
// that its TMA stream runs at HBM speed?  Every CTA streams a (rows x W columns) tile through a
// ring of stages (each stage = W/64 boxes of 64 columns x BR rows, 128-B swizzle); a consumer warp
// only waits and releases.  The whole matrix is covered once (non-persistent grid) and the kernel
// is timed with events after an L2 flush.
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o dtc_stream dtc_stream.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                               \
    do {                                                                                    \
        cudaError_t e = (x);                                                                \
        if (e != cudaSuccess) {                                                             \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                        \
        }                                                                                   \
    } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                     : "=r"(ok)
                     : "r"(bar), "r"(ph));
}

__global__ void __launch_bounds__(64) stream(const __grid_constant__ CUtensorMap tm, int rows, int W, int BR, int st,
                                             int ktiles, unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[16], empty[16];
    const int nt = blockIdx.x % (gridDim.x / ktiles), kt = blockIdx.x / (gridDim.x / ktiles);
    const int nbox = W / 64;
    const uint32_t stage_bytes = nbox * BR * 128;
    const int nst = rows / BR;
    if (threadIdx.x == 0) {
        for (int s = 0; s < st; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&empty[s])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < nst; ++i) {
            const int s = i % st, r = i / st;
            if (r) wait(su32(&empty[s]), (r - 1) & 1);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(stage_bytes));
            for (int b = 0; b < nbox; ++b)
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                        su32(sm + s * stage_bytes + b * BR * 128)),
                    "l"((uint64_t)&tm), "r"(su32(&full[s])), "r"(nt * W + b * 64), "r"(kt * rows + i * BR)
                    : "memory");
        }
    } else if (threadIdx.x == 32) {
        unsigned long long acc = 0;
        for (int i = 0; i < nst; ++i) {
            const int s = i % st;
            wait(su32(&full[s]), (i / st) & 1);
            acc += *(volatile uint32_t*)(sm + s * stage_bytes);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&empty[s])) : "memory");
        }
        if (acc == 0x123456789ull) sink[0] = acc;
    }
}

// read-only L2 flush: leaves the L2 full of CLEAN lines (a memset flush leaves ~126 MB of dirty
// lines whose write-back then competes with the timed kernel's reads)
__global__ void read_flush(const uint4* p, size_t n, unsigned long long* sink) {
    uint32_t acc = 0;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldcg(p + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == 0x9e3779b9u) sink[1] = acc;
}

int main(int argc, char** argv) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q));
    auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    const int K = argc > 1 ? atoi(argv[1]) : 1536, N = 11008;  // Llama-7B gate_up low-rank U (r = 1488 padded)
    void* buf;
    CK(cudaMalloc(&buf, size_t(K) * N * 2));
    CK(cudaMemset(buf, 1, size_t(K) * N * 2));
    void* flush;
    CK(cudaMalloc(&flush, size_t(512) << 20));
    unsigned long long* sink;
    CK(cudaMalloc(&sink, 64));
    CK(cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    struct C { int W, rows, BR, st, per_sm; };
    std::vector<C> cs = {{64, 768, 64, 8, 2},  {64, 768, 64, 4, 2},  {64, 192, 64, 3, 4},  {64, 1536, 64, 8, 2},
                         {128, 768, 64, 6, 2}, {256, 384, 32, 4, 2}, {256, 192, 32, 6, 2}, {256, 192, 64, 3, 2},
                         {512, 192, 32, 3, 2}, {512, 96, 32, 3, 2},  {1024, 96, 16, 3, 2}, {256, 96, 32, 3, 4},
                         {128, 384, 64, 4, 3}};
    for (auto c : cs) {
        CUtensorMap tm;
        const uint64_t dims[2] = {(uint64_t)N, (uint64_t)K};
        const uint64_t str[1] = {(uint64_t)N * 2};
        const uint32_t box[2] = {64, (uint32_t)c.BR};
        const uint32_t es[2] = {1, 1};
        if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS) {
            printf("encode failed\n");
            return 1;
        }
        const int ntiles = (N + c.W - 1) / c.W, ktiles = K / c.rows;
        const int grid = ntiles * ktiles;
        const size_t smem = std::max<size_t>((size_t)c.st * (c.W / 64) * c.BR * 128 + 1024, 200 * 1024 / c.per_sm);
        float best = 1e9, best_rf = 1e9;
        for (int rep = 0; rep < 10; ++rep) {
            const bool rf = rep & 1;
            CK(cudaMemset(flush, rep, size_t(512) << 20));
            if (rf) read_flush<<<148 * 4, 512>>>((const uint4*)flush, (size_t(512) << 20) / 16, sink);
            cudaEvent_t e0, e1;
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            CK(cudaEventRecord(e0));
            stream<<<grid, 64, smem>>>(tm, c.rows, c.W, c.BR, c.st, ktiles, sink);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (rf) best_rf = std::min(best_rf, ms);
            else best = std::min(best, ms);
        }
        const double bytes = double(ntiles) * c.W * K * 2;
        printf("W %4d rows %4d BR %3d stages %d (%2d KB in flight/CTA, %d CTA/SM): grid %5d  memset-flush %7.2f us %5.2f TB/s | read-flush %7.2f us %5.2f TB/s\n",
               c.W, c.rows, c.BR, c.st, c.st * (c.W / 64) * c.BR * 128 / 1024, c.per_sm, grid, best * 1e3,
               bytes / (best * 1e-3) / 1e12, best_rf * 1e3, bytes / (best_rf * 1e-3) / 1e12);
    }
    {  // calibration: an empty kernel and a device-to-device copy of the same bytes, event-timed
        float best_e = 1e9, best_c = 1e9;
        void* dst;
        CK(cudaMalloc(&dst, size_t(K) * N * 2));
        for (int rep = 0; rep < 10; ++rep) {
            CK(cudaMemset(flush, rep, size_t(512) << 20));
            read_flush<<<148 * 4, 512>>>((const uint4*)flush, (size_t(512) << 20) / 16, sink);
            cudaEvent_t e0, e1, e2;
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            CK(cudaEventCreate(&e2));
            CK(cudaEventRecord(e0));
            read_flush<<<1, 32>>>((const uint4*)flush, 0, sink);
            CK(cudaEventRecord(e1));
            CK(cudaMemcpyAsync(dst, buf, size_t(K) * N * 2, cudaMemcpyDeviceToDevice));
            CK(cudaEventRecord(e2));
            CK(cudaEventSynchronize(e2));
            float a, b;
            CK(cudaEventElapsedTime(&a, e0, e1));
            CK(cudaEventElapsedTime(&b, e1, e2));
            best_e = std::min(best_e, a);
            best_c = std::min(best_c, b);
        }
        printf("empty kernel %.2f us; D2D copy of %.1f MB %.2f us (%.2f TB/s read+write)\n", best_e * 1e3,
               K * (double)N * 2 / 1e6, best_c * 1e3, 2.0 * K * N * 2 / (best_c * 1e-3) / 1e12);
    }
    return 0;
}
