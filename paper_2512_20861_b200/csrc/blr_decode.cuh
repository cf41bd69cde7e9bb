// blr_decode.cuh -- small-token (decode, n_tok <= DECODE_MAX_TOKENS) path of the three BLR
// products (§3.1: at small n the layer is bound by reading
// its factors, not by FLOPs).  Every stage streams its weight factor from HBM exactly once with
// 16-B/8-B vector loads on the CUDA cores; the (tiny) activations live in shared memory as fp32
// and the intermediates stay fp32 (no bf16 rounding between stages; only Y is rounded, RNE).
//
//   decode_mn_kernel : out[g][t][c] = sum_k A[g][t][k] * B[g][k][c]   (B "MN-major": [K][N])
//                      grid (N / 128 columns, groups, K splits); a split-K grid writes fp32
//                      partials [split][g][t][c] that decode_reduce sums in a fixed order (no
//                      atomics: results are bitwise run-to-run deterministic).
//   decode_k_kernel  : out[g][t][c]   = sum_k A[g][t][k] * B[g][c][k]   (B "K-major": [N][K])
//                      one warp per output column, lanes stride K with 16-B loads.
//   decode_s2_kernel : BLAST S2, Z''[k][t][rho] = sum_l S[l,k,rho] Z[l][t][rho]  (fp32)
//   decode_reduce    : out[g][t][c] = sum_z part[z][g][t][c] (warp-parallel over z, fixed order),
//                      fp32 or RNE bf16, strided dest.
#pragma once
#include <cuda_bf16.h>
#include <cstdint>

namespace blr {

constexpr int DECODE_MAX_TOKENS = 16;
constexpr int DECODE_THREADS = 256;
constexpr int DECODE_MN_COLS = 256;  // columns per decode_mn block (32 lanes x 8)

struct DecodeMN {
    const void* A;        // activations: bf16 (a_f32 = 0) or fp32
    int a_f32;
    long long a_rs, a_gs;  // element strides: token rows, groups
    const __nv_bfloat16* B;
    long long b_rs, b_gs;  // element strides: K rows (= N for dense [K][N]), groups
    void* out;            // k_split == 1: the destination (fp32 or bf16); else fp32 partials
    int out_bf16;         // 1: RNE bf16 store (only when k_split == 1)
    long long o_rs, o_gs, o_zs;  // element strides of out: token rows, groups, K splits
    int n_tok, K, N, k_chunk;
    int pre;  // 1 (not the first launch of a call): prefetch the block's weight slice into L2 before
              // griddepcontrol.wait, so it streams while the previous stage runs
};

__device__ __forceinline__ float4 bf16x4_to_f32(uint2 w) {
    return make_float4(__uint_as_float(w.x << 16), __uint_as_float(w.x & 0xFFFF0000u),
                       __uint_as_float(w.y << 16), __uint_as_float(w.y & 0xFFFF0000u));
}

template <int NT>
__global__ void __launch_bounds__(DECODE_THREADS) decode_mn_kernel(const DecodeMN d) {
    extern __shared__ float dsm[];  // A chunk [k_chunk][NT] (token fastest), then the reduction buffer
    const int g = blockIdx.y;
    const int k0 = blockIdx.z * d.k_chunk;
    const int k1 = min(d.K, k0 + d.k_chunk);
    const int kc = k1 - k0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int c0 = blockIdx.x * DECODE_MN_COLS + lane * 8;
    if (d.pre) {  // weights are never written by this library: stream the block's slice into L2 now
        const int cb0 = blockIdx.x * DECODE_MN_COLS;
        const int ncb = min(DECODE_MN_COLS, d.N - cb0);
        const __nv_bfloat16* bp0 = d.B + static_cast<long long>(g) * d.b_gs + cb0;
        for (int k = k0 + threadIdx.x; k < k1; k += DECODE_THREADS)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(bp0 + static_cast<long long>(k) * d.b_rs),
                         "r"(static_cast<uint32_t>(ncb * 2)) : "memory");
    }
    // stage A[g][t][k0:k1] as fp32, [k][t] so one k's NT values are contiguous (float4 reads)
    asm volatile("griddepcontrol.wait;" ::: "memory");  // A may be the previous kernel's output
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");  // (after the wait: first-launch rule)
    for (int e = threadIdx.x; e < NT * kc; e += DECODE_THREADS) {
        const int t = e / kc, k = e - t * kc;
        float v = 0.f;
        if (t < d.n_tok) {
            const long long off = static_cast<long long>(g) * d.a_gs + static_cast<long long>(t) * d.a_rs + k0 + k;
            v = d.a_f32 ? static_cast<const float*>(d.A)[off]
                        : __bfloat162float(static_cast<const __nv_bfloat16*>(d.A)[off]);
        }
        dsm[k * NT + t] = v;
    }
    __syncthreads();
    float acc[NT][8];
#pragma unroll
    for (int t = 0; t < NT; ++t)
#pragma unroll
        for (int j = 0; j < 8; ++j) acc[t][j] = 0.f;
    const bool col_ok = c0 < d.N;  // N is a multiple of 8 (ABI), so c0 < N => c0 + 8 <= N
    auto fma8 = [&](const uint4 w, const float* ak) {
        float b[8];
        b[0] = __uint_as_float(w.x << 16);
        b[1] = __uint_as_float(w.x & 0xFFFF0000u);
        b[2] = __uint_as_float(w.y << 16);
        b[3] = __uint_as_float(w.y & 0xFFFF0000u);
        b[4] = __uint_as_float(w.z << 16);
        b[5] = __uint_as_float(w.z & 0xFFFF0000u);
        b[6] = __uint_as_float(w.w << 16);
        b[7] = __uint_as_float(w.w & 0xFFFF0000u);
#pragma unroll
        for (int t4 = 0; t4 < NT; t4 += 4) {
            const float4 a = *reinterpret_cast<const float4*>(ak + t4);
            const float av[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
            for (int u = 0; u < 4; ++u)
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[t4 + u][j] = fmaf(av[u], b[j], acc[t4 + u][j]);
        }
    };
    if (col_ok) {
        const __nv_bfloat16* bp = d.B + static_cast<long long>(g) * d.b_gs + c0;
        // warp w takes k = k0 + w, w + 8, ...; UNR loads in flight per lane
        constexpr int UNR = NT <= 8 ? 8 : 4;
        int k = k0 + warp;
        for (; k + 8 * (UNR - 1) < k1; k += 8 * UNR) {
            uint4 w[UNR];
#pragma unroll
            for (int u = 0; u < UNR; ++u)
                w[u] = __ldg(reinterpret_cast<const uint4*>(bp + static_cast<long long>(k + 8 * u) * d.b_rs));
#pragma unroll
            for (int u = 0; u < UNR; ++u) fma8(w[u], dsm + (k + 8 * u - k0) * NT);
        }
        for (; k < k1; k += 8)
            fma8(__ldg(reinterpret_cast<const uint4*>(bp + static_cast<long long>(k) * d.b_rs)), dsm + (k - k0) * NT);
    }
    // tree-reduce the 8 warps' partial sums (fixed order: deterministic), 4 x NT x 256 floats
    float* red = dsm;
#pragma unroll
    for (int half = 4; half >= 1; half >>= 1) {
        __syncthreads();  // A chunk / previous round no longer needed
        if (warp >= half && warp < 2 * half) {
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                float4* dst = reinterpret_cast<float4*>(red + ((warp - half) * NT + t) * DECODE_MN_COLS + lane * 8);
                dst[0] = make_float4(acc[t][0], acc[t][1], acc[t][2], acc[t][3]);
                dst[1] = make_float4(acc[t][4], acc[t][5], acc[t][6], acc[t][7]);
            }
        }
        __syncthreads();
        if (warp < half) {
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const float4* src = reinterpret_cast<const float4*>(red + (warp * NT + t) * DECODE_MN_COLS + lane * 8);
                const float4 x = src[0], y = src[1];
                acc[t][0] += x.x; acc[t][1] += x.y; acc[t][2] += x.z; acc[t][3] += x.w;
                acc[t][4] += y.x; acc[t][5] += y.y; acc[t][6] += y.z; acc[t][7] += y.w;
            }
        }
    }
    if (warp == 0 && col_ok) {
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            if (t >= d.n_tok) break;
            const long long off = static_cast<long long>(blockIdx.z) * d.o_zs + static_cast<long long>(g) * d.o_gs +
                                  static_cast<long long>(t) * d.o_rs + c0;
            if (d.out_bf16) {
                uint4 w;
                w.x = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(acc[t][0])) |
                      ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(acc[t][1])) << 16);
                w.y = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(acc[t][2])) |
                      ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(acc[t][3])) << 16);
                w.z = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(acc[t][4])) |
                      ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(acc[t][5])) << 16);
                w.w = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(acc[t][6])) |
                      ((uint32_t)__bfloat16_as_ushort(__float2bfloat16_rn(acc[t][7])) << 16);
                *reinterpret_cast<uint4*>(static_cast<__nv_bfloat16*>(d.out) + off) = w;
            } else {
                float4* dst = reinterpret_cast<float4*>(static_cast<float*>(d.out) + off);
                dst[0] = make_float4(acc[t][0], acc[t][1], acc[t][2], acc[t][3]);
                dst[1] = make_float4(acc[t][4], acc[t][5], acc[t][6], acc[t][7]);
            }
        }
    }
}

// K-major B: out[g][t][c] = sum_k A[g][t][k] * B[g][c][k].  The output column c of group g may be
// remapped (Monarch S1 writes Z'[k][t][l r' + rho] for V row m = (rho, k)): col_map 0 = identity
// (out offset g*o_gs + t*o_rs + c); 1 = Monarch S1 with b2-fastest rows (m = rho*b2 + k);
// 2 = Monarch S1 with r'-fastest rows (m = k*r' + rho).  For maps 1/2: mon_b2, mon_r, and the
// output is Z'[k][t][g*r' + rho] with o_gs = n_tok * b1 * r' (stride of k), o_rs = b1 * r'.
struct DecodeK {
    const void* A;
    int a_f32;
    long long a_rs, a_gs;
    const __nv_bfloat16* B;
    long long b_rs, b_gs;  // element strides: output-column rows (= K), groups
    void* out;
    int out_bf16;
    long long o_rs, o_gs;
    int n_tok, K, N;
    int col_map, mon_b2, mon_r;
    int cols_per_block;
    long long o_cs;  // col_map 0: elements between output columns (1; b2 for Monarch's transposed order)
    int pre;         // 1: prefetch the block's weight rows into L2 before griddepcontrol.wait
};

template <int NT>
__global__ void __launch_bounds__(DECODE_THREADS) decode_k_kernel(const DecodeK d) {
    extern __shared__ float dsm[];  // A [NT][K] fp32
    const int g = blockIdx.y;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (d.pre) {
        const int cb = blockIdx.x * d.cols_per_block, ce = min(d.N, cb + d.cols_per_block);
        for (int c = cb + threadIdx.x; c < ce; c += DECODE_THREADS)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(d.B + static_cast<long long>(g) * d.b_gs +
                                                                               static_cast<long long>(c) * d.b_rs),
                         "r"(static_cast<uint32_t>(d.K * 2)) : "memory");
    }
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    for (int e = threadIdx.x; e < NT * d.K; e += DECODE_THREADS) {
        const int t = e / d.K, k = e - t * d.K;
        float v = 0.f;
        if (t < d.n_tok) {
            const long long off = static_cast<long long>(g) * d.a_gs + static_cast<long long>(t) * d.a_rs + k;
            v = d.a_f32 ? static_cast<const float*>(d.A)[off]
                        : __bfloat162float(static_cast<const __nv_bfloat16*>(d.A)[off]);
        }
        dsm[t * d.K + k] = v;
    }
    __syncthreads();
    const int cbeg = blockIdx.x * d.cols_per_block;
    const int cend = min(d.N, cbeg + d.cols_per_block);
    constexpr int CW = 4;  // columns per warp iteration: CW independent 16-B loads in flight per lane
    for (int cb = cbeg + warp * CW; cb < cend; cb += (DECODE_THREADS / 32) * CW) {
        float acc[CW][NT];
#pragma unroll
        for (int q = 0; q < CW; ++q)
#pragma unroll
            for (int t = 0; t < NT; ++t) acc[q][t] = 0.f;
        for (int k = lane * 8; k < d.K; k += 256) {  // K is a multiple of 8 (ABI)
            uint4 w[CW];
#pragma unroll
            for (int q = 0; q < CW; ++q) {
                const int c = min(cb + q, cend - 1);  // clamp: duplicate work, never stored
                w[q] = __ldg(reinterpret_cast<const uint4*>(d.B + static_cast<long long>(g) * d.b_gs +
                                                            static_cast<long long>(c) * d.b_rs + k));
            }
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const float* a = dsm + t * d.K + k;
                const float4 a0 = *reinterpret_cast<const float4*>(a);
                const float4 a1 = *reinterpret_cast<const float4*>(a + 4);
#pragma unroll
                for (int q = 0; q < CW; ++q) {
                    const float4 lo = bf16x4_to_f32(make_uint2(w[q].x, w[q].y));
                    const float4 hi = bf16x4_to_f32(make_uint2(w[q].z, w[q].w));
                    float s = acc[q][t];
                    s = fmaf(a0.x, lo.x, s);
                    s = fmaf(a0.y, lo.y, s);
                    s = fmaf(a0.z, lo.z, s);
                    s = fmaf(a0.w, lo.w, s);
                    s = fmaf(a1.x, hi.x, s);
                    s = fmaf(a1.y, hi.y, s);
                    s = fmaf(a1.z, hi.z, s);
                    s = fmaf(a1.w, hi.w, s);
                    acc[q][t] = s;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < CW; ++q)
#pragma unroll
            for (int t = 0; t < NT; ++t)
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc[q][t] += __shfl_xor_sync(0xffffffffu, acc[q][t], o);
#pragma unroll
        for (int q = 0; q < CW; ++q) {
            const int c = cb + q;
            if (c >= cend || lane >= NT || lane >= d.n_tok) continue;
            float v = 0.f;
#pragma unroll
            for (int t = 0; t < NT; ++t)
                if (t == lane) v = acc[q][t];
            long long off;
            if (d.col_map == 0) {
                off = static_cast<long long>(g) * d.o_gs + static_cast<long long>(lane) * d.o_rs + c * d.o_cs;
            } else {
                const int rho = d.col_map == 1 ? c / d.mon_b2 : c % d.mon_r;
                const int k = d.col_map == 1 ? c % d.mon_b2 : c / d.mon_r;
                off = static_cast<long long>(k) * d.o_gs + static_cast<long long>(lane) * d.o_rs +
                      static_cast<long long>(g) * d.mon_r + rho;
            }
            if (d.out_bf16) static_cast<__nv_bfloat16*>(d.out)[off] = __float2bfloat16_rn(v);
            else static_cast<float*>(d.out)[off] = v;
        }
    }
}

// BLAST S2 for the decode path: Z''[k][t][rho] = sum_l S[l,k,rho] * Z[l][t][rho], fp32 in/out.
__global__ void __launch_bounds__(DECODE_THREADS)
    decode_s2_kernel(const float* __restrict__ Z, const __nv_bfloat16* __restrict__ S, float* __restrict__ Zpp,
                     int n_tok, int b1, int b2, int r) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const long long total = static_cast<long long>(b2) * n_tok * r;
    for (long long e = blockIdx.x * static_cast<long long>(DECODE_THREADS) + threadIdx.x; e < total;
         e += static_cast<long long>(gridDim.x) * DECODE_THREADS) {
        const int rho = static_cast<int>(e % r);
        const long long kt = e / r;
        const int t = static_cast<int>(kt % n_tok);
        const int k = static_cast<int>(kt / n_tok);
        float s = 0.f;
        for (int l = 0; l < b1; ++l)
            s = fmaf(__bfloat162float(S[(static_cast<long long>(l) * b2 + k) * r + rho]),
                     Z[(static_cast<long long>(l) * n_tok + t) * r + rho], s);
        Zpp[e] = s;
    }
}

// Split-K reduction: part is [splits][groups][n_tok][N] fp32; out[g*gs + t*rs + c].  One warp
// per 32 consecutive outputs with the splits spread over 4 lane groups... -> here: one warp per
// 8 consecutive outputs; lane = (split residue s8 in 0..3, output j in 0..7): each lane sums the
// splits z = s8, s8 + 4, ... of its output in ascending order, then the 4 partial sums are combined
// by two fixed shuffle steps (a fixed tree: bitwise run-to-run deterministic).  A
// thread-per-output loop over 40-50 splits was latency-bound (~10 us for 1488 outputs).
__global__ void __launch_bounds__(DECODE_THREADS)
    decode_reduce(const float* __restrict__ part, int splits, int groups, int n_tok, int N, void* out, int out_bf16,
                  long long o_rs, long long o_gs) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    const long long count = static_cast<long long>(groups) * n_tok * N;
    const int lane = threadIdx.x & 31;
    const int j = lane & 7, s4 = lane >> 3;
    const long long warps = static_cast<long long>(gridDim.x) * (DECODE_THREADS / 32);
    for (long long wb = (static_cast<long long>(blockIdx.x) * (DECODE_THREADS / 32) + (threadIdx.x >> 5)) * 8;
         wb < count; wb += warps * 8) {
        const long long e = wb + j;
        float s = 0.f;
        if (e < count)
            for (int z = s4; z < splits; z += 4) s += __ldcg(part + static_cast<long long>(z) * count + e);
        s += __shfl_down_sync(0xffffffffu, s, 16);  // (s4, s4 + 2)
        s += __shfl_down_sync(0xffffffffu, s, 8);   // (0+2) + (1+3)
        if (s4 == 0 && e < count) {
            const int c = static_cast<int>(e % N);
            const long long gt = e / N;
            const int t = static_cast<int>(gt % n_tok);
            const int g = static_cast<int>(gt / n_tok);
            const long long off = static_cast<long long>(g) * o_gs + static_cast<long long>(t) * o_rs + c;
            if (out_bf16) static_cast<__nv_bfloat16*>(out)[off] = __float2bfloat16_rn(s);
            else static_cast<float*>(out)[off] = s;
        }
    }
}

}  // namespace blr
