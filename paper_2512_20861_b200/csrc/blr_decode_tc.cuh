// Small-token (decode) path on the tensor cores: SURVEY §8 row f2.
//
// With n <= 16 tokens every stage of the three methods (PAPER.md L36 low rank, L53 Monarch, L74
// BLAST) is a weight stream: each factor byte is used n times, so the roofline is the factor bytes
// over the HBM bandwidth.  One kernel, decode_tc_kernel, runs every stage:
//
//   out[g][t][c] = sum_k A[g][t][k] * B[g][k][c]     (B "MN-major" [K][N], KMAJ = false), or
//                = sum_k A[g][t][k] * B[g][c][k]     (B "K-major"  [N][K], KMAJ = true)
//
//  * a producer warp streams the CTA's weight tile (W columns x its K range) through a ring of
//    16-KB stages of 128-B-swizzled TMA boxes, issued BEFORE griddepcontrol.wait when the launch is
//    not the first of a call, so the weight stream overlaps the previous stage.  W (64/128/256
//    columns, i.e. 128-512 contiguous bytes per weight row for MN-major weights) is chosen by the
//    host together with the K split (benchmarks/micro/dtc_stream.cu: 64-column strips stream
//    ~20% slower than 256-column ones);
//  * four MMA warps (W/4 columns each) run mma.sync m16n8k16 bf16 -> fp32 with the n <= 16 tokens
//    as the M dimension (ldmatrix from the A slice staged once in shared memory; .trans for
//    MN-major weights).  An fp32 A (a previous stage's intermediate) is staged as a bf16 pair
//    hi + lo with hi = bf16(a), lo = bf16(a - hi), both multiplied against the same weight
//    fragments: the intermediate keeps ~16 significant bits at no HBM cost;
//  * a K split (EPI 1) is reduced on chip: the S split CTAs of one output tile form a thread-block
//    cluster, park their fp32 partial tiles in shared memory and each sums a 1/S share of the tile
//    over the S peers through DSMEM in ascending split order (fixed order: bitwise deterministic,
//    SURVEY §8 c13), so there is neither a partial buffer in HBM nor a reduction launch;
//  * BLAST (EPI 2) fuses S2 into S1's epilogue: the cluster's CTAs hold all b1 tiles Z_l[t][rho-tile]
//    in shared memory and CTA q writes Z''_k[t][rho] = sum_l S[l,k,rho] Z_l[t][rho] (PAPER.md L74,
//    fixed l order, fp32) for k = q, q + cs, ..., so Z never leaves the chip.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

#include "ptx.cuh"

namespace blr {

constexpr int DTC_STAGE = 16384;                 // bytes per ring stage
constexpr int DTC_MMA_WARPS = 4;
constexpr int DTC_THREADS = 32 * (DTC_MMA_WARPS + 1);
constexpr int DTC_MAX_KC = 1024;                 // K rows per CTA (A slice <= 2 x 16 x 1032 bf16)
constexpr int DTC_MAX_UNITS = 4;                 // EPI 2: BLAST blocks l per CTA
constexpr int DTC_MAX_CLUSTER = 8;
constexpr int DTC_MAX_B1 = 16;
constexpr int DTC_MAX_N = 4096;                  // tokens the weight-streaming path may take (16-row chunks)

// K rows per stage and TMA boxes per stage of a (KMAJ, W) tile.  MN-major: W/64 boxes of 64
// columns x BK rows.  K-major (W = 64 output columns): 2 boxes of 64 k x 64 columns, BK = 128.
__host__ __device__ constexpr int dtc_bk(bool kmaj, int w) { return kmaj ? 128 : DTC_STAGE / (w * 2); }
__host__ __device__ constexpr int dtc_nbox(bool kmaj, int w) { return kmaj ? 2 : w / 64; }

struct DecodeTC {
    const void* A;          // bf16 (a_f32 = 0) or fp32 (a_f32 = 1: staged as hi + lo bf16)
    int a_f32;
    long long a_rs, a_gs;   // element strides: token rows, groups
    int n_tok, K, N, k_chunk, n_units, stages;
    int groups;             // G: grid.z = G x ceil(n_tok / 16) token chunks (EPI 2: the chunks alone)
    void* out;              // fp32 or bf16 (out_bf16, RNE)
    int out_bf16;
    long long o_rs, o_gs, o_cs;  // element strides: token rows, groups, output columns
    int col_map, mon_b2, mon_r;  // Monarch S1 (KMAJ): column c of group l -> Z'[k][t][l r' + rho]
    const __nv_bfloat16* s2;     // EPI 2: BLAST S [b1][b2][r] (r = N)
    int b1, b2;
    int pre;                // 1: not the first launch of a call (weights stream before the wait)
    unsigned long long* trace;  // debug (blr_debug_trace): per-CTA globaltimer stamps [2048][16]
};

namespace dtc {

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
                 : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t mapa(uint32_t addr, uint32_t rank) {
    uint32_t ra;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(addr), "r"(rank));
    return ra;
}
__device__ __forceinline__ float lds_bf16(uint32_t addr) {
    unsigned short h;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(h) : "r"(addr));
    return __uint_as_float(static_cast<uint32_t>(h) << 16);
}
__device__ __forceinline__ float4 ld_cluster_v4(uint32_t raddr) {
    float4 v;
    asm volatile("ld.shared::cluster.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                 : "r"(raddr)
                 : "memory");
    return v;
}
__device__ __forceinline__ float ld_cluster(uint32_t raddr) {
    float v;
    asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(raddr) : "memory");
    return v;
}

// shared-memory carve-up (host and device agree): [ring][A slices][partial tiles][S tile][barriers]
struct Layout {
    uint32_t a_off, a_ld, a_bytes, red_off, s_off, bar_off, total;
};
__host__ __device__ inline Layout layout(int k_chunk, int a_f32, int n_units, int stages, int epi, int w, int bk,
                                         int s_elems) {
    Layout L;
    const int kcp = (k_chunk + bk - 1) / bk * bk;
    L.a_ld = kcp + 8;  // +16 B per token row: the 8 rows of an ldmatrix hit distinct banks
    L.a_off = stages * DTC_STAGE;
    L.a_bytes = 16u * L.a_ld * 2u * (a_f32 ? 2u : 1u);  // per unit: [hi][lo] x 16 rows
    L.red_off = L.a_off + n_units * L.a_bytes;
    L.s_off = L.red_off + (epi == 2 ? n_units * 16u * w * 4u : 0u);  // EPI 1: the tile reuses the ring
    L.bar_off = L.s_off + ((s_elems * 2u + 15u) & ~15u);
    L.total = L.bar_off + 2u * stages * 8u + 1024u;  // + alignment slack for the 1-KB base
    return L;
}

}  // namespace dtc

// grid: EPI 0 (1, tiles, G); EPI 1 (S, tiles, G) with cluster (S, 1, 1); EPI 2 (cs, tiles, 1) with
// cluster (cs, 1, 1), CTA q owning the BLAST blocks l = q n_units + u.
template <bool KMAJ, int EPI, int W>
__global__ void __launch_bounds__(DTC_THREADS)
    decode_tc_kernel(const __grid_constant__ CUtensorMap tmB, const DecodeTC d) {
    constexpr int BK = dtc_bk(KMAJ, W), NBOX = dtc_nbox(KMAJ, W), BOXB = DTC_STAGE / NBOX;
    constexpr int NF = W / 32;  // n8 fragments per MMA warp (W / 4 columns)
    static_assert(!KMAJ || W == 64, "K-major tiles are 64 columns wide");
    extern __shared__ uint8_t dtc_raw[];
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(dtc_raw) + 1023) & ~uintptr_t(1023));
    const int nk_mine = EPI == 2 ? (d.b2 + gridDim.x - 1) / gridDim.x : 0;
    const dtc::Layout L = dtc::layout(d.k_chunk, d.a_f32, d.n_units, d.stages, EPI, W, BK, nk_mine * d.b1 * W);
    const uint32_t ring = ptx::smem_u32(base);
    const uint32_t sA = ptx::smem_u32(base + L.a_off);
    const uint32_t bar_full = ptx::smem_u32(base + L.bar_off);
    const uint32_t bar_empty = bar_full + 8u * d.stages;
    float* red = reinterpret_cast<float*>(base + (EPI == 1 ? 0u : L.red_off));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int split = EPI == 1 ? static_cast<int>(blockIdx.x) : 0;
    const int k0 = split * d.k_chunk;
    const int kc = min(d.k_chunk, d.K - k0);
    const int nkb = (kc + BK - 1) / BK;
    const int nt = blockIdx.y;
    // token chunk of 16 rows (n > 16: chunks are independent CTAs re-reading the weights from L2)
    const int chunk = EPI == 2 ? static_cast<int>(blockIdx.z) : static_cast<int>(blockIdx.z) / d.groups;
    const int gz = EPI == 2 ? 0 : static_cast<int>(blockIdx.z) - chunk * d.groups;
    const int n_here = min(16, d.n_tok - chunk * 16);
    const void* Ab = static_cast<const char*>(d.A) + static_cast<long long>(chunk) * 16 * d.a_rs * (d.a_f32 ? 4 : 2);
    void* Ob = static_cast<char*>(d.out) + static_cast<long long>(chunk) * 16 * d.o_rs * (d.out_bf16 ? 2 : 4);
    auto group_of = [&](int u) { return EPI == 2 ? static_cast<int>(blockIdx.x) * d.n_units + u : gz; };

    const int cta_lin = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z);
#ifdef BLR_DEBUG_KNOBS
    unsigned long long* tr = (d.trace && cta_lin < 2048) ? d.trace + cta_lin * 16 : nullptr;
#else
    unsigned long long* const tr = nullptr;  // timeline stamps: debug builds only (scripts/dtc_trace.py)
#endif
    if (tr && threadIdx.x == 0) tr[0] = ptx::globaltimer();
    if (threadIdx.x == 0) {
        for (int s = 0; s < d.stages; ++s) {
            ptx::mbar_init(bar_full + 8u * s, 1);
            ptx::mbar_init(bar_empty + 8u * s, DTC_MMA_WARPS);
        }
        ptx::fence_barrier_init();
    }
    __syncthreads();

    if (warp == DTC_MMA_WARPS) {  // ---------------------------------------------- producer ----
        if (lane == 0) {
            ptx::prefetch_tmap(&tmB);
            if (!d.pre) ptx::griddep_wait();  // first launch of a call: nothing before the wait
            if (tr) tr[1] = ptx::globaltimer();
            int s = 0, ph = 0, rnd = 0;
            for (int u = 0; u < d.n_units; ++u) {
                const int g = group_of(u);
                for (int kb = 0; kb < nkb; ++kb) {
                    if (rnd > 0) ptx::mbar_wait(bar_empty + 8u * s, ph ^ 1);
                    const uint32_t fb = bar_full + 8u * s;
                    ptx::mbar_arrive_expect_tx(fb, DTC_STAGE);
#pragma unroll
                    for (int b = 0; b < NBOX; ++b) {
                        const uint32_t dst = ring + s * DTC_STAGE + b * BOXB;
                        if (KMAJ)  // map (K, N, G): box 64 k x 64 columns
                            ptx::tma_load_3d(dst, &tmB, fb, k0 + kb * BK + b * 64, nt * W, g);
                        else       // map (N, K, G): box 64 columns x BK k
                            ptx::tma_load_3d(dst, &tmB, fb, nt * W + b * 64, k0 + kb * BK, g);
                    }
                    if (++s == d.stages) {
                        s = 0;
                        ph ^= 1;
                        rnd = 1;
                    }
                }
            }
        }
        return;
    }

    // ------------------------------------------------------------------------ MMA warps ----
    ptx::griddep_wait();  // A may be the previous stage's output
    ptx::griddep_launch_dependents();
    const int tid = threadIdx.x;
    if (tr && tid == 0) tr[2] = ptx::globaltimer();
    const int kcp = nkb * BK;
    {   // stage A[g][t][k0 : k0 + kc] (zero past kc and n); 4 chunks of 8 per thread in flight at once
        const int k8n = kcp / 8, total = 16 * k8n;
        const uint32_t lo_off = 16u * L.a_ld * 2u;
        for (int u = 0; u < d.n_units; ++u) {
            const int g = group_of(u);
            const uint32_t au = sA + u * L.a_bytes;
            for (int e0 = tid; e0 < total; e0 += 4 * DTC_MMA_WARPS * 32) {
                if (!d.a_f32) {
                    uint4 v[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int e = e0 + j * DTC_MMA_WARPS * 32;
                        const int t = e / k8n, k = (e - t * k8n) * 8;
                        v[j] = make_uint4(0, 0, 0, 0);
                        if (e < total && t < n_here && k < kc)
                            v[j] = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(Ab) +
                                                                   static_cast<long long>(g) * d.a_gs +
                                                                   static_cast<long long>(t) * d.a_rs + k0 + k);
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int e = e0 + j * DTC_MMA_WARPS * 32;
                        const int t = e / k8n, k = (e - t * k8n) * 8;
                        if (e < total) ptx::st_shared_v4(au + (t * L.a_ld + k) * 2, v[j]);
                    }
                } else {
                    float4 v[4][2];
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int e = e0 + j * DTC_MMA_WARPS * 32;
                        const int t = e / k8n, k = (e - t * k8n) * 8;
                        v[j][0] = v[j][1] = make_float4(0.f, 0.f, 0.f, 0.f);
                        if (e < total && t < n_here && k < kc) {
                            const float* p = static_cast<const float*>(Ab) + static_cast<long long>(g) * d.a_gs +
                                             static_cast<long long>(t) * d.a_rs + k0 + k;
                            v[j][0] = *reinterpret_cast<const float4*>(p);
                            v[j][1] = *reinterpret_cast<const float4*>(p + 4);
                        }
                    }
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int e = e0 + j * DTC_MMA_WARPS * 32;
                        if (e >= total) continue;
                        const int t = e / k8n, k = (e - t * k8n) * 8;
                        const float x[8] = {v[j][0].x, v[j][0].y, v[j][0].z, v[j][0].w,
                                            v[j][1].x, v[j][1].y, v[j][1].z, v[j][1].w};
                        uint32_t hi[4], lo[4];
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            const __nv_bfloat16 h0 = __float2bfloat16_rn(x[2 * q]), h1 = __float2bfloat16_rn(x[2 * q + 1]);
                            hi[q] = static_cast<uint32_t>(__bfloat16_as_ushort(h0)) |
                                    (static_cast<uint32_t>(__bfloat16_as_ushort(h1)) << 16);
                            lo[q] = ptx::pack_bf16x2(x[2 * q] - __bfloat162float(h0), x[2 * q + 1] - __bfloat162float(h1));
                        }
                        const uint32_t dst = au + (t * L.a_ld + k) * 2;
                        ptx::st_shared_v4(dst, make_uint4(hi[0], hi[1], hi[2], hi[3]));
                        ptx::st_shared_v4(dst + lo_off, make_uint4(lo[0], lo[1], lo[2], lo[3]));
                    }
                }
            }
        }
    }
    if (EPI == 2) {  // this CTA's S2 coefficients: sS[kk][l][col] = S[l][q + kk cs][nt W + col] (bf16)
        __nv_bfloat16* sS = reinterpret_cast<__nv_bfloat16*>(base + L.s_off);
        const int per = d.b1 * (W / 8);
        for (int e = tid; e < nk_mine * per; e += DTC_MMA_WARPS * 32) {
            const int kk = e / per, r = e - kk * per, l = r / (W / 8), c8 = (r - l * (W / 8)) * 8;
            const int k = blockIdx.x + kk * gridDim.x, rho = nt * W + c8;
            uint4 v = make_uint4(0, 0, 0, 0);
            if (k < d.b2 && rho < d.N)
                v = *reinterpret_cast<const uint4*>(d.s2 + (static_cast<long long>(l) * d.b2 + k) * d.N + rho);
            *reinterpret_cast<uint4*>(sS + (kk * d.b1 + l) * W + c8) = v;
        }
    }
    ptx::named_bar_sync(1, DTC_MMA_WARPS * 32);
    if (tr && tid == 0) tr[3] = ptx::globaltimer();

    // per-lane ldmatrix row addresses (matrix m = lane / 8, row lane % 8)
    const int m = lane >> 3, r8 = lane & 7;
    const uint32_t a_lane = ((m & 1) * 8 + r8) * L.a_ld * 2 + (m >> 1) * 16;  // + k * 2
    const int cw0 = warp * (W / 4);  // this warp's first tile column
    int s = 0, ph = 0, it = 0;
    for (int u = 0; u < d.n_units; ++u) {
        const uint32_t au = sA + u * L.a_bytes + a_lane;
        float acc[NF][4];
#pragma unroll
        for (int j = 0; j < NF; ++j)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[j][q] = 0.f;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
            ptx::mbar_wait(bar_full + 8u * s, ph);
            if (tr && tid == 0 && it < 8) tr[8 + it] = ptx::globaltimer();
            const uint32_t sb = ring + s * DTC_STAGE;
#pragma unroll
            for (int ks = 0; ks < BK / 16; ++ks) {
                uint32_t a[4], al[4];
                dtc::ldsm_x4(au + (kb * BK + ks * 16) * 2, a);
                if (d.a_f32) dtc::ldsm_x4(au + 16u * L.a_ld * 2u + (kb * BK + ks * 16) * 2, al);
#pragma unroll
                for (int jj = 0; jj < NF / 2; ++jj) {
                    uint32_t b[4];
                    if (KMAJ) {  // box (ks / 4): smem [column][64 k], rows = columns
                        const int row = cw0 + jj * 16 + (m >> 1) * 8 + r8;
                        const int ch = (ks & 3) * 2 + (m & 1);
                        dtc::ldsm_x4(sb + (ks >> 2) * BOXB + row * 128 + ((ch ^ (row & 7)) << 4), b);
                    } else {  // box (column / 64): smem [k][64 columns], transposed load
                        const int col = cw0 + jj * 16;
                        const int row = ks * 16 + (m & 1) * 8 + r8;
                        const int ch = ((col & 63) >> 3) + (m >> 1);
                        dtc::ldsm_x4_t(sb + (col >> 6) * BOXB + row * 128 + ((ch ^ (row & 7)) << 4), b);
                    }
                    dtc::mma16816(acc[2 * jj], a, b[0], b[1]);
                    dtc::mma16816(acc[2 * jj + 1], a, b[2], b[3]);
                    if (d.a_f32) {
                        dtc::mma16816(acc[2 * jj], al, b[0], b[1]);
                        dtc::mma16816(acc[2 * jj + 1], al, b[2], b[3]);
                    }
                }
            }
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(bar_empty + 8u * s);
            if (++s == d.stages) {
                s = 0;
                ph ^= 1;
            }
        }
        // fragment (j, q): token t = lane / 4 + 8 (q / 2), tile column cw0 + 8 j + 2 (lane % 4) + q % 2
        const int t0 = lane >> 2;
        if (EPI == 0) {
            const int g = group_of(u);
#pragma unroll
            for (int j = 0; j < NF; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int t = t0 + 8 * h;
                    const int c = nt * W + cw0 + j * 8 + 2 * (lane & 3);
                    if (t >= n_here || c >= d.N) continue;  // N % 8 == 0: c < N => c + 1 < N
                    const float v0 = acc[j][2 * h], v1 = acc[j][2 * h + 1];
                    if (d.col_map == 0 && d.o_cs == 1) {
                        const long long off = static_cast<long long>(g) * d.o_gs + static_cast<long long>(t) * d.o_rs + c;
                        if (d.out_bf16)
                            *reinterpret_cast<uint32_t*>(static_cast<__nv_bfloat16*>(Ob) + off) = ptx::pack_bf16x2(v0, v1);
                        else
                            *reinterpret_cast<float2*>(static_cast<float*>(Ob) + off) = make_float2(v0, v1);
                    } else {
#pragma unroll
                        for (int e = 0; e < 2; ++e) {
                            const int cc = c + e;
                            long long off;
                            if (d.col_map == 0) {
                                off = static_cast<long long>(g) * d.o_gs + static_cast<long long>(t) * d.o_rs + cc * d.o_cs;
                            } else {  // Monarch S1: column cc of block g = (k, rho) in either composite order
                                const int rho = d.col_map == 1 ? cc / d.mon_b2 : cc % d.mon_r;
                                const int k = d.col_map == 1 ? cc % d.mon_b2 : cc / d.mon_r;
                                off = static_cast<long long>(k) * d.o_gs + static_cast<long long>(t) * d.o_rs +
                                      static_cast<long long>(g) * d.mon_r + rho;
                            }
                            const float v = e ? v1 : v0;
                            if (d.out_bf16) static_cast<__nv_bfloat16*>(Ob)[off] = __float2bfloat16_rn(v);
                            else static_cast<float*>(Ob)[off] = v;
                        }
                    }
                }
        } else {  // park the fp32 tile for the cluster epilogue
            if (EPI == 1) ptx::named_bar_sync(1, DTC_MMA_WARPS * 32);  // the tile overwrites the ring
            float* ru = red + u * 16 * W;
#pragma unroll
            for (int j = 0; j < NF; ++j)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int col = cw0 + j * 8 + 2 * (lane & 3);
                    *reinterpret_cast<float2*>(ru + (t0 + 8 * h) * W + col) = make_float2(acc[j][2 * h], acc[j][2 * h + 1]);
                }
        }
    }
    if (tr && tid == 0) tr[4] = ptx::globaltimer();
    if (EPI == 0) {
        if (tr && tid == 0) tr[7] = ptx::globaltimer();
        return;
    }

    ptx::cluster_sync();  // every CTA's partial tiles are in place (release/acquire at cluster scope)
    if (tr && tid == 0) tr[5] = ptx::globaltimer();
    const uint32_t red_s = ptx::smem_u32(red);
    const int ncl = gridDim.x;  // cluster = the grid's x extent
    const int q = blockIdx.x;
    if (EPI == 1) {  // sum the S split partials of 1/S of the tile (4 columns per item), ascending split order
        const int g = gz;
        uint32_t rz[DTC_MAX_CLUSTER];
#pragma unroll
        for (int z = 0; z < DTC_MAX_CLUSTER; ++z) rz[z] = dtc::mapa(red_s, z < ncl ? z : 0);
        for (int e4 = q + ncl * tid; e4 < n_here * (W / 4); e4 += ncl * DTC_MMA_WARPS * 32) {
            const int t = e4 / (W / 4), col = (e4 - t * (W / 4)) * 4;
            const int c = nt * W + col;
            if (c >= d.N) continue;  // N % 8 == 0: c < N => c + 3 < N
            float4 pv[DTC_MAX_CLUSTER];
#pragma unroll
            for (int z = 0; z < DTC_MAX_CLUSTER; ++z)  // all loads in flight before the first add
                if (z < ncl) pv[z] = dtc::ld_cluster_v4(rz[z] + (t * W + col) * 4);
            float v[4] = {pv[0].x, pv[0].y, pv[0].z, pv[0].w};
#pragma unroll
            for (int z = 1; z < DTC_MAX_CLUSTER; ++z)
                if (z < ncl) {
                    v[0] += pv[z].x;
                    v[1] += pv[z].y;
                    v[2] += pv[z].z;
                    v[3] += pv[z].w;
                }
            if (d.col_map == 0 && d.o_cs == 1) {
                const long long off = static_cast<long long>(g) * d.o_gs + static_cast<long long>(t) * d.o_rs + c;
                if (d.out_bf16)
                    *reinterpret_cast<uint2*>(static_cast<__nv_bfloat16*>(Ob) + off) =
                        make_uint2(ptx::pack_bf16x2(v[0], v[1]), ptx::pack_bf16x2(v[2], v[3]));
                else
                    *reinterpret_cast<float4*>(static_cast<float*>(Ob) + off) = make_float4(v[0], v[1], v[2], v[3]);
                continue;
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int cc = c + j;
                long long off;
                if (d.col_map == 0) {
                    off = static_cast<long long>(g) * d.o_gs + static_cast<long long>(t) * d.o_rs + cc * d.o_cs;
                } else {
                    const int rho = d.col_map == 1 ? cc / d.mon_b2 : cc % d.mon_r;
                    const int k = d.col_map == 1 ? cc % d.mon_b2 : cc / d.mon_r;
                    off = static_cast<long long>(k) * d.o_gs + static_cast<long long>(t) * d.o_rs +
                          static_cast<long long>(g) * d.mon_r + rho;
                }
                if (d.out_bf16) static_cast<__nv_bfloat16*>(Ob)[off] = __float2bfloat16_rn(v[j]);
                else static_cast<float*>(Ob)[off] = v[j];
            }
        }
    } else {  // BLAST S2: Z''_k[t][rho] = sum_l S[l,k,rho] Z_l[t][rho], l ascending, k = q, q + cs, ...
        const uint32_t sS = ptx::smem_u32(base + L.s_off);
        uint32_t rz[DTC_MAX_B1];  // Z_l's tile in CTA l / n_units, slot l % n_units
#pragma unroll
        for (int l = 0; l < DTC_MAX_B1; ++l) {
            const int ll = l < d.b1 ? l : 0;
            rz[l] = dtc::mapa(red_s + (ll % d.n_units) * 16 * W * 4, ll / d.n_units);
        }
        for (int e4 = tid; e4 < n_here * (W / 4); e4 += DTC_MMA_WARPS * 32) {
            const int t = e4 / (W / 4), col = (e4 - t * (W / 4)) * 4;
            const int rho = nt * W + col;
            if (rho >= d.N) continue;
            float4 z[DTC_MAX_B1];
#pragma unroll
            for (int l = 0; l < DTC_MAX_B1; ++l)  // the b1 tiles' Z_l[t][rho : rho + 4], all loads in flight
                z[l] = l < d.b1 ? dtc::ld_cluster_v4(rz[l] + (t * W + col) * 4) : make_float4(0.f, 0.f, 0.f, 0.f);
            for (int kk = 0; kk < nk_mine; ++kk) {
                const int k = q + kk * ncl;
                if (k >= d.b2) break;
                float v[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                for (int l = 0; l < DTC_MAX_B1; ++l)
                    if (l < d.b1) {
                        const uint2 sv = ptx::ld_shared_v2u32(sS + ((kk * d.b1 + l) * W + col) * 2);
                        v[0] = fmaf(__uint_as_float(sv.x << 16), z[l].x, v[0]);
                        v[1] = fmaf(__uint_as_float(sv.x & 0xFFFF0000u), z[l].y, v[1]);
                        v[2] = fmaf(__uint_as_float(sv.y << 16), z[l].z, v[2]);
                        v[3] = fmaf(__uint_as_float(sv.y & 0xFFFF0000u), z[l].w, v[3]);
                    }
                *reinterpret_cast<float4*>(static_cast<float*>(Ob) + static_cast<long long>(k) * d.o_gs +
                                           static_cast<long long>(t) * d.o_rs + rho) = make_float4(v[0], v[1], v[2], v[3]);
            }
        }
    }
    if (tr && tid == 0) tr[6] = ptx::globaltimer();
    ptx::cluster_sync();  // no CTA leaves while a peer may still read its tiles
    if (tr && tid == 0) tr[7] = ptx::globaltimer();
}

}  // namespace blr
