// launch_overhead.cu -- microbenchmark: event-timed cost of an (almost) empty 144-CTA kernel as a
// function of its dynamic shared memory, of what ran before it (a plain L1-using kernel forces an
// L1/shared carveout change), and of back-to-back repetition (stream order, no PDL).
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o launch_overhead launch_overhead.cu
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                               \
    do {                                                                                    \
        cudaError_t e = (x);                                                                \
        if (e != cudaSuccess) {                                                             \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                        \
        }                                                                                   \
    } while (0)

__global__ void empty_k(int* p) {
    extern __shared__ int sm[];
    if (p != nullptr && threadIdx.x == 0) sm[0] = *p;
}
__global__ void plain(float* p, int n) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = p[i] * 0.5f + 1.f;
}

int main() {
    CK(cudaFuncSetAttribute(empty_k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    float* buf;
    const int n = 1 << 24;
    CK(cudaMalloc(&buf, n * 4));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto timed = [&](const char* name, int smem, bool plain_before, int reps) {
        float best = 1e9;
        for (int t = 0; t < 7; ++t) {
            if (plain_before) plain<<<n / 256, 256>>>(buf, n);
            else empty_k<<<144, 128, smem>>>(nullptr);
            CK(cudaEventRecord(e0));
            for (int r = 0; r < reps; ++r) empty_k<<<144, 320, smem>>>(nullptr);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            best = ms < best ? ms : best;
        }
        printf("%-48s smem %6d x%2d: %.2f us per launch\n", name, smem, reps, best * 1e3 / reps);
    };
    for (int smem : {0, 64 * 1024, 200 * 1024, 227 * 1024}) {
        timed("empty after same kernel", smem, false, 1);
        timed("empty after plain L1 kernel", smem, true, 1);
        timed("empty back-to-back", smem, false, 10);
    }
    return 0;
}
