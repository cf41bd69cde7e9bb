// abi_trace.cu -- call libblr.so's blr_lowrank_matmul from plain CUDA (no torch allocator, no
// torch kernels in the stream) and print the intra-kernel trace of its two launches, to separate
// kernel behaviour from the environment the Python benchmarks create.
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o abi_trace abi_trace.cu \
//          -L../../paper_2512_20861_b200 -lblr -Xlinker -rpath=../../paper_2512_20861_b200
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../include/blr.h"
extern "C" void blr_debug_trace(unsigned long long* device_buf);

__global__ void fill(uint16_t* p, size_t n, uint32_t seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u ^ seed;
        h ^= h >> 13;
        h *= 0x5bd1e995u;
        h ^= h >> 15;
        const float f = ((h & 0xFFFF) / 65536.0f - 0.5f) * 0.1f;
        p[i] = (uint16_t)(__float_as_uint(f) >> 16);
    }
}

int main(int argc, char** argv) {
    const int64_t n = argc > 1 ? atoll(argv[1]) : 8192, di = 768, dout = 3072, r = 192;
    const bool flush_first = !(argc > 2 && argv[2][0] == '0');
    uint16_t *X, *V, *U, *Y;
    void* ws;
    cudaMalloc(&X, n * di * 2);
    cudaMalloc(&V, di * r * 2);
    cudaMalloc(&U, r * dout * 2);
    cudaMalloc(&Y, n * dout * 2);
    const size_t wsb = blr_lowrank_workspace_size(n, di, dout, r);
    cudaMalloc(&ws, wsb);
    fill<<<592, 256>>>(X, n * di, 1);
    fill<<<592, 256>>>(V, di * r, 2);
    fill<<<592, 256>>>(U, r * dout, 3);
    void* flush;
    cudaMalloc(&flush, size_t(512) << 20);
    unsigned long long* tr;
    const size_t trn = 4 * 256 * 128;
    cudaMalloc(&tr, trn * 8);
    cudaMemset(tr, 0, trn * 8);
    for (int i = 0; i < 3; ++i) blr_lowrank_matmul(X, n, di, dout, r, V, U, Y, ws, wsb, nullptr);
    {  // event-timed calls (no tracing): min over 10
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        float best = 1e9;
        for (int i = 0; i < 10; ++i) {
            if (flush_first) cudaMemset(flush, i, size_t(512) << 20);
            cudaEventRecord(a);
            blr_lowrank_matmul(X, n, di, dout, r, V, U, Y, ws, wsb, nullptr);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        printf("event-timed call (both kernels, eager): %.2f us\n", best * 1e3);
    }
    if (flush_first) cudaMemset(flush, 1, size_t(512) << 20);
    cudaDeviceSynchronize();
    blr_debug_trace(tr);
    const int st = blr_lowrank_matmul(X, n, di, dout, r, V, U, Y, ws, wsb, nullptr);
    blr_debug_trace(nullptr);
    cudaDeviceSynchronize();
    printf("status %d (%s), cuda %s, n=%lld flush=%d\n", st, blr_status_string((blr_status)st),
           cudaGetErrorString(cudaGetLastError()), (long long)n, (int)flush_first);
    std::vector<unsigned long long> h(trn);
    cudaMemcpy(h.data(), tr, trn * 8, cudaMemcpyDeviceToHost);
    // stamps other than [0] (globaltimer ns) and [8] (clock64 at entry) are clock64 values
    const double ghz = getenv("TRACE_GHZ") ? atof(getenv("TRACE_GHZ")) : 1.92;
    for (size_t c = 0; c < trn / 128; ++c) {
        unsigned long long* t = h.data() + c * 128;
        if (!t[0]) continue;
        for (int f = 1; f < 128; ++f)
            if (f != 8 && t[f]) t[f] = t[0] + (unsigned long long)((double)(long long)(t[f] - t[8]) / ghz);
    }
    for (int k = 0; k < 2; ++k) {
        if (!h[k * 256 * 128]) continue;
        const unsigned long long* t = h.data() + k * 256 * 128;
        unsigned long long t0 = ~0ull;
        int nc = 0;
        for (int c = 0; c < 256; ++c)
            if (t[c * 128]) { t0 = std::min(t0, t[c * 128]); ++nc; }
        const char* names[8] = {"entry", "setup", "gdwait", "1stfull", "lastmma", "epidone", "drained", "exit"};
        printf(" launch %d: %d CTAs\n", k, nc);
        for (int f = 0; f < 8; ++f) {
            std::vector<double> v;
            for (int c = 0; c < nc; ++c)
                if (t[c * 128 + f]) v.push_back((t[c * 128 + f] - t0) * 1e-3);
            if (v.empty()) continue;
            std::sort(v.begin(), v.end());
            printf("   %-8s %7.2f %7.2f %7.2f\n", names[f], v[0], v[v.size() / 2], v.back());
        }
        printf("   CTA0 producer issue:");
        for (int i = 0; i < 32; ++i)
            if (t[64 + i]) printf(" %.2f", (t[64 + i] - t0) * 1e-3);
        printf("\n   CTA0 MMA full-ready:");
        for (int i = 0; i < 32; ++i)
            if (t[96 + i]) printf(" %.2f", (t[96 + i] - t0) * 1e-3);
        printf("\n");
    }
    return 0;
}
