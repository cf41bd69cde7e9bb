// tile_reread.cu -- microbenchmark emulating the weight-stationary expand's operand stream:
// 144 CTAs = 12 slices x 12 token walkers; CTA (slice s, walker w) reads token tiles
// m = w, w + 12, ... of an [8192][192] bf16 matrix (each tile: 3 TMA boxes of 64 x 128 rows,
// 16 KB), through a 6-stage ring, consuming nothing.  With `shared`, the 12 slices read the
// same tiles in lockstep (as the kernel does); otherwise every CTA reads its own copy.
// The matrix is prepared by a preceding kernel that either WRITES it (fresh dirty lines, as
// when the previous GEMM produced it) or only READS it.
// Build: nvcc -std=c++17 -O3 -gencode arch=compute_100a,code=sm_100a -o tile_reread tile_reread.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>

#define CK(x)                                                                               \
    do {                                                                                    \
        cudaError_t e = (x);                                                                \
        if (e != cudaSuccess) {                                                             \
            printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__); \
            exit(1);                                                                        \
        }                                                                                   \
    } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void wait(uint32_t bar, uint32_t ph) {
    uint32_t ok = 0;
    while (!ok)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0,1,0,p; }"
                     : "=r"(ok)
                     : "r"(bar), "r"(ph));
}

// rows: token rows of one copy; copies: 1 (shared) or 12 (private per slice)
__global__ void __launch_bounds__(320, 1) reader(const __grid_constant__ CUtensorMap tm, const __grid_constant__ CUtensorMap tmb, int bres, int pdl, int adj, int extra, int tiles_m, int slices,
                                                  int walkers, int shared_copy, int nst, int boxes_per_stage, int kbl, int reps, int spin, int commit_rel,
                                                  unsigned long long* ns) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ __align__(8) uint64_t full[16], empty[16], done, bbar;
    __shared__ uint32_t tslot;
    // extra & 1: allocate 512 TMEM columns (as the GEMM kernel does); & 2: prefetch the tensor
    // maps; & 4: griddepcontrol.launch_dependents at the start
    if ((extra & 1) && threadIdx.x / 32 == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if ((extra & 2) && threadIdx.x == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tm) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"((uint64_t)&tmb) : "memory");
    }
    if (extra & 4) asm volatile("griddepcontrol.launch_dependents;");
    uint8_t* base = (uint8_t*)(((uintptr_t)smem + 1023) & ~(uintptr_t)1023);
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&full[s])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&empty[s])));
        }
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bbar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    // adj: the CTAs sharing a token tile are adjacent in blockIdx (same GPC), else strided
    const int slice = (adj & 1) ? blockIdx.x % slices : blockIdx.x / walkers;
    const int w = (adj & 1) ? blockIdx.x / slices : blockIdx.x % walkers;
    const int copy = shared_copy ? 0 : slice;
    const uint32_t box_bytes = 64 * 128 * 2;
    const int steps_per_tile = kbl / boxes_per_stage;
    if (threadIdx.x == 0) {
        int stage = 0;
        uint32_t ph = 0;
        if (bres) {  // resident weight slice: 12 boxes of 64 cols x 64 rows (8 KB) behind the ring
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bbar)), "r"(12 * 8192));
            for (int b = 0; b < 12; ++b) {
                const uint32_t dst = smem_u32(base + 6 * 16384 + b * 8192);
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                    " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
                    "l"((uint64_t)&tmb), "r"(smem_u32(&bbar)), "r"((slice * 4 + (b & 3)) * 64), "r"((b >> 2) * 64), "r"(0)
                    : "memory");
            }
        }
        if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
        for (int rp = 0; rp < reps; ++rp)
        for (int i = 0, m; (m = (adj & 2) ? w * tiles_m / walkers + i : w + i * walkers) < ((adj & 2) ? (w + 1) * tiles_m / walkers : tiles_m); ++i)
            for (int st = 0; st < steps_per_tile; ++st) {
                wait(smem_u32(&empty[stage]), ph ^ 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[stage])),
                             "r"(box_bytes * boxes_per_stage));
                for (int b = 0; b < boxes_per_stage; ++b) {
                    const uint32_t dst = smem_u32(base + (stage * boxes_per_stage + b) * box_bytes);
                    asm volatile(
                        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
                        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
                        "l"((uint64_t)&tm), "r"(smem_u32(&full[stage])), "r"((st * boxes_per_stage + b) * 64),
                        "r"(m * 128), "r"(copy)
                        : "memory");
                }
                if (++stage == nst) { stage = 0; ph ^= 1; }
            }
    } else if (threadIdx.x == 32) {
        int stage = 0;
        uint32_t ph = 0;
        for (int rp = 0; rp < reps; ++rp)
        for (int i = 0, m; (m = (adj & 2) ? w * tiles_m / walkers + i : w + i * walkers) < ((adj & 2) ? (w + 1) * tiles_m / walkers : tiles_m); ++i)
            for (int st = 0; st < steps_per_tile; ++st) {
                wait(smem_u32(&full[stage]), ph);
                if (commit_rel)
                    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                     smem_u32(&empty[stage])) : "memory");
                else
                    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[stage])) : "memory");
                if (++stage == nst) { stage = 0; ph ^= 1; }
            }
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&done)) : "memory");
    } else if (threadIdx.x >= 64 && threadIdx.x < 64 + 32 * spin) {
        wait(smem_u32(&done), 0);  // epilogue-like warps polling a barrier
    }
    __syncthreads();
    unsigned long long t1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
    if (threadIdx.x == 0) { ns[2 * blockIdx.x] = t0; ns[2 * blockIdx.x + 1] = t1; }
    if ((extra & 1) && threadIdx.x / 32 == 1) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tslot));
    }
}

__global__ void writer(uint4* p, size_t n16) {
    asm volatile("griddepcontrol.launch_dependents;");
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4((uint32_t)i, 1, 2, 3);
}
// writes the buffer with TMA bulk stores (smem -> global), as the GEMM epilogues do
__global__ void bulk_writer(uint8_t* p, size_t bytes) {
    extern __shared__ __align__(1024) uint8_t sm[];
    for (int i = threadIdx.x; i < 16384 / 16; i += blockDim.x)
        reinterpret_cast<uint4*>(sm)[i] = make_uint4(i, 1, 2, 3);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        for (size_t off = (size_t)blockIdx.x * 16384; off < bytes; off += (size_t)gridDim.x * 16384) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 16384;" ::"l"(p + off),
                         "r"(smem_u32(sm))
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}
__global__ void touch(const uint4* p, size_t n16, uint4* sink) {
    uint4 a = make_uint4(0, 0, 0, 0);
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
        uint4 v = p[i];
        a.x ^= v.x; a.y ^= v.y;
    }
    if (a.x == 0x12345) sink[0] = a;
}

int main() {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q));
    auto encode = (PFN_cuTensorMapEncodeTiled_v12000)fn;
    const int rows = 8192, K = 192, slices = 12, walkers = 12;
    const size_t copy_bytes = size_t(rows) * K * 2;
    void* buf;
    CK(cudaMalloc(&buf, copy_bytes * slices));
    void* flush;
    const size_t fl = size_t(512) << 20;
    CK(cudaMalloc(&flush, fl));
    uint4* sink;
    CK(cudaMalloc(&sink, 64));
    unsigned long long* ns;
    CK(cudaMalloc(&ns, 8 * 4096));
    CK(cudaFuncSetAttribute(reader, cudaFuncAttributeMaxDynamicSharedMemorySize, 226 * 1024));
    CUtensorMap tm;
    const uint64_t dims[3] = {(uint64_t)K, (uint64_t)rows, (uint64_t)slices};
    const uint64_t str[2] = {(uint64_t)K * 2, copy_bytes};
    const uint32_t box[3] = {64, 128, 1}, es[3] = {1, 1, 1};
    if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
        printf("encode failed\n");
        return 1;
    }
    void* ubuf;
    CK(cudaMalloc(&ubuf, size_t(192) * 3072 * 2));
    CUtensorMap tmb;
    {
        const uint64_t d2[3] = {3072, 192, 1};
        const uint64_t s2[2] = {3072 * 2, 3072ull * 192 * 2};
        const uint32_t b2[3] = {64, 64, 1};
        if (encode(&tmb, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, ubuf, d2, s2, b2, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
            CUDA_SUCCESS) {
            printf("encode b failed\n");
            return 1;
        }
    }
    struct Case { const char* name; int shared; int prep; int nst; int bps; int flushw; int reps = 1; int spin = 0; int commit = 0; int thr = 128; int bres = 0; int pdl = 0; int smem_kb = 200; int adj = 0; int extra = 0; };
    // prep: 0 = previous kernel wrote the operand, 1 = previous kernel read it, 2 = nothing
    std::vector<Case> cases = {
        {"plain                         6x16KB", 1, 0, 6, 1, 1},
        {"+tmem alloc 512               6x16KB", 1, 0, 6, 1, 1, 1, 0, 0, 128, 0, 0, 200, 0, 1},
        {"+prefetch tensormap           6x16KB", 1, 0, 6, 1, 1, 1, 0, 0, 128, 0, 0, 200, 0, 2},
        {"+launch_dependents            6x16KB", 1, 0, 6, 1, 1, 1, 0, 0, 128, 0, 0, 200, 0, 4},
        {"+all three, 320thr, res B, PDL 6x16KB", 1, 0, 6, 1, 1, 1, 8, 1, 320, 1, 1, 226, 3, 7},
    };
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (auto& c : cases) {
        double best = 1e9;
        char info[256] = "";
        for (int rep = 0; rep < 5; ++rep) {
            if (c.flushw) CK(cudaMemset(flush, rep, fl));
            const size_t n = (c.shared ? copy_bytes : copy_bytes * slices) / 16;
            if (c.pdl) CK(cudaEventRecord(e0));  // keep writer -> reader adjacent for PDL
            if (c.prep == 0) writer<<<148 * 4, 256>>>((uint4*)buf, n);
            if (c.prep == 1) touch<<<148 * 4, 256>>>((const uint4*)buf, n, sink);
            if (c.prep == 3) bulk_writer<<<148, 128, 17 * 1024>>>((uint8_t*)buf, n * 16);
            if (!c.pdl) CK(cudaEventRecord(e0));
            {
                cudaLaunchConfig_t cfg = {};
                cfg.gridDim = dim3(slices * walkers);
                cfg.blockDim = dim3(c.thr);
                cfg.dynamicSmemBytes = c.smem_kb * 1024;
                cudaLaunchAttribute at[1];
                at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
                at[0].val.programmaticStreamSerializationAllowed = c.pdl;
                cfg.attrs = at;
                cfg.numAttrs = 1;
                CK(cudaLaunchKernelEx(&cfg, reader, tm, tmb, c.bres, c.pdl, c.adj, c.extra, rows / 128, slices, walkers, c.shared, c.nst,
                                      c.bps, 3, c.reps, c.spin, c.commit, ns));
            }
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (ms < best) {
                best = ms;
                const int nc = slices * walkers;
                std::vector<unsigned long long> h(2 * nc);
                CK(cudaMemcpy(h.data(), ns, 8 * h.size(), cudaMemcpyDeviceToHost));
                unsigned long long s0 = ~0ull, s1 = 0, e0v = ~0ull, e1v = 0;
                std::vector<double> dur;
                for (int i = 0; i < nc; ++i) {
                    s0 = std::min(s0, h[2 * i]); s1 = std::max(s1, h[2 * i]);
                    e0v = std::min(e0v, h[2 * i + 1]); e1v = std::max(e1v, h[2 * i + 1]);
                    dur.push_back((h[2 * i + 1] - h[2 * i]) * 1e-3);
                }
                std::sort(dur.begin(), dur.end());
                snprintf(info, sizeof info, "start spread %.2f us, end %.2f..%.2f us, CTA dur min/med/max %.2f/%.2f/%.2f",
                         (s1 - s0) * 1e-3, (e0v - s0) * 1e-3, (e1v - s0) * 1e-3, dur[0], dur[nc / 2], dur[nc - 1]);
            }
        }
        const double delivered = double(copy_bytes) * slices * c.reps;  // every CTA slice reads all tiles once
        printf("%-42s kernel %.2f us: %.2f TB/s delivered; %s\n", c.name, best * 1e3,
               delivered / (best * 1e-3) / 1e12, info);
    }
    return 0;
}
