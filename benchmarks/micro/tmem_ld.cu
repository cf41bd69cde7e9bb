// tmem_ld.cu -- microbenchmark: tcgen05.ld (TMEM -> registers) throughput per SM, for the
// epilogue cost model.  W warps (multiple of 4) each read their lane quarter of a 128 x 512 fp32
// TMEM region repeatedly with 32x32b.x{8,32,64} loads.
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o tmem_ld tmem_ld.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int X>
__device__ __forceinline__ void ld(uint32_t taddr, uint32_t* r);
template <>
__device__ __forceinline__ void ld<8>(uint32_t t, uint32_t* r) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
                 : "r"(t));
}
template <>
__device__ __forceinline__ void ld<32>(uint32_t t, uint32_t* r) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
          "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
          "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(t));
}

template <int X>
__global__ void __launch_bounds__(512, 1) k(int iters, unsigned long long* out, uint32_t* sink) {
    __shared__ uint32_t slot;
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = slot + ((uint32_t)((warp & 3) * 32) << 16);
    const int nw = blockDim.x / 32;
    const int col0 = (warp >> 2) * 32;  // warps of the same quarter read different columns
    uint32_t acc = 0;
    __syncthreads();
    unsigned long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        uint32_t r[X];
        for (int c = col0; c + X <= 512; c += (nw / 4) * 32 > X ? (nw / 4) * 32 : X) {
            ld<X>(base + c, r);
            asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
            for (int j = 0; j < X; ++j) acc += r[j];
        }
    }
    unsigned long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}


// Emulates the BLAST fused epilogue's TMEM access: 8 warps (2 per lane quarter), each walks
// W=32 columns in 8-column steps; per step it loads b1=6 blocks (columns l*BN + col) in batches
// of 4 x8 loads per wait, and sums them (no smem).
__global__ void __launch_bounds__(320, 1) blast_like(int reps, int b1, int BN, unsigned long long* out, float* sink,
                                                     int mma_first, int mode) {
    const int b2 = b1;
    const int lane = threadIdx.x & 31;
    __shared__ uint32_t slot;
    __shared__ __align__(8) uint64_t bar;
    extern __shared__ __align__(1024) uint8_t dsm[];
    float* s_sm = reinterpret_cast<float*>(dsm + 49152);               // S tile [b1][b2][BN] fp32
    uint8_t* stg_sm = dsm + 49152 + 16384;                             // staging, 8 warps x b2 x 32 x W x 2
    for (int e = threadIdx.x; e < b1 * b2 * BN; e += blockDim.x) s_sm[e] = 0.5f + (e & 7);
    const int warp = threadIdx.x >> 5;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&slot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (threadIdx.x == 32) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (mma_first && threadIdx.x == 32) {  // write the accumulators with the tensor core first
        const uint32_t a = (smem_u32(dsm) + 1023) & ~1023u;
        auto desc = [](uint32_t addr) {
            uint64_t d = (uint64_t)((addr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | (1ull << 46) | (2ull << 61);
            return d;
        };
        const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((256u >> 3) << 17) | ((128u >> 4) << 24);
        for (int h = 0; h < 2; ++h)
            asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, 0, 0;\n\t"
                         "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(slot + 256 * h),
                         "l"(desc(a)), "l"(desc(a + 16384)), "r"(idesc));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        uint32_t ok = 0;
        while (!ok)
            asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0,1,0,p; }"
                         : "=r"(ok) : "r"(smem_u32(&bar)));
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    float acc = 0.f;
    unsigned long long t0 = clock64();
    if (warp >= 2) {
        const int ew = warp - 2, quarter = warp & 3, half = ew >> 2;
        (void)lane;
        const uint32_t tbase = slot + ((uint32_t)(quarter * 32) << 16);
        const int W = BN / 2;
        for (int r = 0; r < reps; ++r)
            for (int sc = 0; sc < W / 8; ++sc) {
                const int col = half * W + sc * 8;
                unsigned long long acc2[8][4];
#pragma unroll
                for (int k = 0; k < 8; ++k)
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc2[k][e] = 0ull;
                for (int lb = 0; lb < b1; lb += 4) {
                    uint32_t z[4][8];
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (lb + j < b1) ld<8>(tbase + (lb + j) * BN + col, z[j]);
                    asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        if (lb + j < b1) {
                            if (mode & 1) {  // the BLAST epilogue's S-weighted sums (S from smem)
                                unsigned long long z2[4];
#pragma unroll
                                for (int e = 0; e < 4; ++e)
                                    z2[e] = ((unsigned long long)z[j][2 * e + 1] << 32) | z[j][2 * e];
                                const float* srow = s_sm + ((lb + j) * b2) * BN + col;
#pragma unroll
                                for (int k = 0; k < 8; ++k) {
                                    if (k < b2) {
                                        ulonglong2 sa, sb;
                                        if (mode & 4) {  // S from registers (no shared loads)
                                            sa = make_ulonglong2(0x3f0000003f000000ull + k, 0x3f0000003f000000ull + lb + j);
                                            sb = make_ulonglong2(0x3f0000003f000000ull + 2 * k, 0x3f0000003f000000ull + j);
                                        } else {
                                            sa = *reinterpret_cast<const ulonglong2*>(srow + k * BN);
                                            sb = *reinterpret_cast<const ulonglong2*>(srow + k * BN + 4);
                                        }
                                        if (mode & 8) {  // plain FFMA on the low halves instead of FFMA2
                                            float a0 = __uint_as_float((uint32_t)acc2[k][0]);
                                            a0 = fmaf(__uint_as_float((uint32_t)sa.x), __uint_as_float((uint32_t)z2[0]), a0);
                                            float a1 = __uint_as_float((uint32_t)(acc2[k][0] >> 32));
                                            a1 = fmaf(__uint_as_float((uint32_t)(sa.x >> 32)), __uint_as_float((uint32_t)(z2[0] >> 32)), a1);
                                            acc2[k][0] = ((unsigned long long)__float_as_uint(a1) << 32) | __float_as_uint(a0);
                                            continue;
                                        }
                                        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc2[k][0]) : "l"(sa.x), "l"(z2[0]));
                                        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc2[k][1]) : "l"(sa.y), "l"(z2[1]));
                                        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc2[k][2]) : "l"(sb.x), "l"(z2[2]));
                                        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc2[k][3]) : "l"(sb.y), "l"(z2[3]));
                                    }
                                }
                            } else {
#pragma unroll
                                for (int e = 0; e < 8; ++e) acc += __uint_as_float(z[j][e]);
                            }
                        }
                    }
                }
                if (mode & 2) {  // stage b2 rows of 8 bf16 (16 B) per lane, 64-B swizzled rows
#pragma unroll
                    for (int k = 0; k < 8; ++k) {
                        if (k >= b2) break;
                        uint32_t off = lane * (W * 2) + sc * 16;
                        off ^= ((off >> 7) & 3u) << 4;
                        const uint32_t a = smem_u32(stg_sm) + (ew * b2 + k) * 32 * W * 2 + off;
                        const uint32_t w0 = (uint32_t)acc2[k][0], w1 = (uint32_t)acc2[k][1], w2 = (uint32_t)acc2[k][2],
                                       w3 = (uint32_t)acc2[k][3];
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(w0), "r"(w1), "r"(w2), "r"(w3)
                                     : "memory");
                    }
                }
#pragma unroll
                for (int k = 0; k < 8; ++k) acc += __uint_as_float((uint32_t)acc2[k][0]);
            }
    }
    unsigned long long t1 = clock64();
    __syncthreads();
    if (threadIdx.x == 64) out[blockIdx.x] = t1 - t0;
    sink[blockIdx.x * 320 + threadIdx.x] = acc;
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(slot));
}

template <int X>
void run(int warps) {
    unsigned long long* d;
    uint32_t* sink;
    cudaMalloc(&d, 8 * 148);
    cudaMalloc(&sink, 4 * 148 * 512);
    const int iters = 200;
    k<X><<<148, warps * 32>>>(iters, d, sink);
    cudaDeviceSynchronize();
    k<X><<<148, warps * 32>>>(iters, d, sink);
    cudaDeviceSynchronize();
    unsigned long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    // bytes read per CTA: each warp reads 32 lanes x (columns it visits) x 4 B
    const int step = (warps / 4) * 32 > X ? (warps / 4) * 32 : X;
    long long per_warp_cols = 0;
    for (int c = 0; c + X <= 512; c += step) per_warp_cols += X;
    const double bytes = double(iters) * warps * 32 * per_warp_cols * 4;
    printf("x%-3d warps %2d: %.1f B/clk/SM TMEM->RF (%s)\n", X, warps, bytes / h, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    {
        unsigned long long* d;
        float* sink;
        cudaMalloc(&d, 8 * 148);
        cudaMalloc(&sink, 4 * 148 * 320);
        cudaFuncSetAttribute(blast_like, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
        const char* names[16] = {"TMEM loads only", "+ S-weighted FFMA2 (S in smem)", "+ staging stores only",
                                 "+ FFMA2 + staging (full epilogue body)", "", "+ FFMA2 with S in registers", "", "",
                                 "", "+ FFMA (scalar) with S in smem", "", "", "", "+ FFMA (scalar) S in registers"};
        for (int mode : {0, 1, 5, 9, 13, 3})
            for (int mf = 1; mf <= 1; ++mf) {
                for (int rep = 0; rep < 2; ++rep) blast_like<<<148, 320, 180 * 1024>>>(100, 6, 64, d, sink, mf, mode);
                cudaDeviceSynchronize();
                unsigned long long h;
                cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
                printf("blast-like epilogue (b1=b2=6, BN=64, 8 warps, %s, %s): %.0f clk per 8-column step (%s)\n",
                       names[mode], mf ? "TMEM written by tcgen05.mma" : "TMEM never written", double(h) / (100 * 4),
                       cudaGetErrorString(cudaGetLastError()));
            }
    }
    for (int w : {4, 8, 16}) {
        run<8>(w);
        run<32>(w);
    }
    return 0;
}
