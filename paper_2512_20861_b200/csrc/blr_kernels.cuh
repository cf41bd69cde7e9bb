// blr_kernels.cuh -- the sm_100a kernels of the BLR prefill forward (arXiv 2512.20861).
//
// One warp-specialized, persistent tcgen05 GEMM kernel template, instantiated for the two
// phases of every format:
//
//   PROJ  (stage S1, and S2 for BLAST):  per token tile T of 128 rows
//     lowrank : Z[t, rho]            = X[t,:] V[:, rho]
//     monarch : Z'[k][t][l r' + rho] = (X_l V_{l,k})[t, rho]
//               -- the r'<->b2 and b2<->b1 permutations are folded into a 4-D TMA box over V
//                  (rows delivered k-major) and into the epilogue's store address.
//     blast   : Z''[k][t][rho]       = sum_l S[l,k,rho] (X_l V_l)[t, rho]
//               -- b1 accumulators (one per l) live side by side in TMEM; the epilogue warps
//                  apply the S-weighted block sum on fp32 CUDA cores and round once to bf16.
//   EXPAND (stage S3):                    Y[t, k q + c] = sum_kk Z_k[t, kk] U_k[kk, c]
//
// Roles: warp 0 = TMA producer (1 thread), warp 1 = TMEM allocator + MMA issuer (1 thread),
// warps 2..9 = epilogue (two warps per TMEM lane quarter).  Operands stream through a
// STAGES-deep smem ring guarded by full/empty mbarriers; accumulators are double-buffered in
// TMEM when two fit in 512 columns, so the epilogue of tile j overlaps the MMAs of tile j+1.
#pragma once
#include "ptx.cuh"

namespace blr {

constexpr int BM = 128;            // token rows per tile == UMMA M
constexpr int BK = 64;             // K elements per pipeline stage (one 128-B swizzle row)
constexpr int UMMA_K = 16;         // K per tcgen05.mma for 16-bit inputs
constexpr int NUM_EPI_WARPS = 8;
constexpr int NUM_THREADS = 64 + 32 * NUM_EPI_WARPS;
constexpr int TMEM_COLS = 512;
constexpr int MAX_STAGES = 8;

enum Kind : int { KIND_GEMM = 0, KIND_MONARCH_PROJ = 1, KIND_BLAST_PROJ = 2 };

struct KParams {
    // ---- tiling
    int n_tok;        // M extent (tokens)
    int tiles_m;      // ceil(n_tok / BM)
    int tiles_n;      // N tiles per group
    int groups;       // number of independent GEMMs ("g")
    int total_tiles;  // tiles_m * groups * tiles_n
    int BN;           // N tile (MMA N), multiple of 16, <= 256
    int N;            // valid N extent per group
    int k_blocks;     // K blocks per sub-GEMM (2x when the A operand is compensated hi|lo)
    int kb_half;      // K blocks per part: blocks >= kb_half read the lo half of A
    int a_lo_off;     // column offset of the lo half inside A's rows (0: not compensated)
    int n_sub;        // sub-GEMMs accumulated into separate TMEM slots (BLAST proj: b1)
    int stages;       // smem ring depth
    int acc_bufs;     // TMEM accumulator buffers (1 or 2)
    // ---- B operand staging
    int b_mn_major;      // 1: B stored [K][N] (N contiguous), 0: B stored [N][K]
    int b_boxes;         // TMA boxes per stage for B (MN-major with BN > 64)
    int b_box_n;         // N elements per box (MN-major)
    uint32_t b_stage_bytes;
    uint32_t b_lbo, b_sbo, b_layout, b_kstep;  // UMMA descriptor parameters for B
    // ---- epilogue
    __nv_bfloat16* out;  // Y (GEMM), Z' (Monarch proj), Z'' (BLAST proj)
    long long out_ld;    // row pitch of out in elements
    long long out_lo_off;  // >0: also store lo = bf16(z - bf16(z)) at +out_lo_off (compensated)
    int r_blk;           // Monarch: r'
    int kb_per_tile;     // Monarch: output blocks k per N tile
    int b1, b2;          // Monarch / BLAST block counts
    int r;               // BLAST: rank
    const __nv_bfloat16* S;  // BLAST: S [b1][b2][r]
};

struct SmemLayout {
    uint32_t a_off, b_off, s_off, bar_off, total;
};

__host__ __device__ inline SmemLayout smem_layout(const KParams& p) {
    SmemLayout L;
    const uint32_t a_stage = BM * BK * 2;
    L.a_off = 0;
    L.b_off = L.a_off + a_stage * p.stages;
    L.s_off = L.b_off + p.b_stage_bytes * p.stages;
    uint32_t s_bytes = 0;
    if (p.b1 > 0 && p.b2 > 0 && p.S != nullptr) s_bytes = p.b1 * p.b2 * p.BN * 4;
    L.bar_off = (L.s_off + s_bytes + 15) & ~15u;
    L.total = L.bar_off + 8 * (2 * MAX_STAGES + 4) + 16;
    return L;
}

// Tile index -> (m block, group, n block); n block fastest so consecutive tiles share A.
struct TileCoord {
    int m_blk, g, n_blk;
};
__device__ __forceinline__ TileCoord tile_coord(const KParams& p, int tile) {
    TileCoord c;
    c.n_blk = tile % p.tiles_n;
    const int rest = tile / p.tiles_n;
    c.g = rest % p.groups;
    c.m_blk = rest / p.groups;
    return c;
}

// Store 8 fp32 values as bf16 (RNE); with lo_off > 0 also store the residual bf16(v - bf16(v))
// at dst + lo_off (compensated intermediate for short S3 contractions).
__device__ __forceinline__ void store8(__nv_bfloat16* dst, const float (&f)[8], long long lo_off) {
    uint4 w;
    w.x = ptx::pack_bf16x2(f[0], f[1]);
    w.y = ptx::pack_bf16x2(f[2], f[3]);
    w.z = ptx::pack_bf16x2(f[4], f[5]);
    w.w = ptx::pack_bf16x2(f[6], f[7]);
    *reinterpret_cast<uint4*>(dst) = w;
    if (lo_off > 0) {
        const uint32_t hw[4] = {w.x, w.y, w.z, w.w};
        float r[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            r[2 * e] = f[2 * e] - __uint_as_float(hw[e] << 16);
            r[2 * e + 1] = f[2 * e + 1] - __uint_as_float(hw[e] & 0xFFFF0000u);
        }
        uint4 l;
        l.x = ptx::pack_bf16x2(r[0], r[1]);
        l.y = ptx::pack_bf16x2(r[2], r[3]);
        l.z = ptx::pack_bf16x2(r[4], r[5]);
        l.w = ptx::pack_bf16x2(r[6], r[7]);
        *reinterpret_cast<uint4*>(dst + lo_off) = l;
    }
}

template <int KIND>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    blr_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const KParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B alignment for the 128-B swizzle atoms.
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const SmemLayout L = smem_layout(p);
    const uint32_t sbase = ptx::smem_u32(smem);
    const uint32_t a_base = sbase + L.a_off;
    const uint32_t b_base = sbase + L.b_off;
    float* s_tile = reinterpret_cast<float*>(smem + L.s_off);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    const uint32_t full_bar = ptx::smem_u32(bars);
    const uint32_t empty_bar = full_bar + 8 * MAX_STAGES;
    const uint32_t tfull_bar = empty_bar + 8 * MAX_STAGES;
    const uint32_t tempty_bar = tfull_bar + 16;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.bar_off + 8 * (2 * MAX_STAGES + 4));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;

    if (threadIdx.x == 0) {
        for (int s = 0; s < p.stages; ++s) {
            ptx::mbar_init(full_bar + 8 * s, 1);
            ptx::mbar_init(empty_bar + 8 * s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(tfull_bar + 8 * b, 1);
            ptx::mbar_init(tempty_bar + 8 * b, NUM_EPI_WARPS);
        }
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&tmA);
        ptx::prefetch_tmap(&tmB);
    }
    if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(ptx::smem_u32(tmem_slot));
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t acc_stride = static_cast<uint32_t>(p.n_sub * p.BN);  // columns per buffer

    if (warp == 0) {
        // ===================================================== TMA producer =================
        if (lane == 0) {
            const uint32_t a_bytes = BM * BK * 2;
            const uint32_t tx = a_bytes + (p.b_mn_major ? p.b_boxes * p.b_box_n * BK * 2
                                                        : static_cast<uint32_t>(p.BN) * BK * 2);
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < p.total_tiles; tile += gridDim.x) {
                const TileCoord tc = tile_coord(p, tile);
                const int m0 = tc.m_blk * BM;
                const int n0 = tc.n_blk * p.BN;
                for (int sub = 0; sub < p.n_sub; ++sub) {
                    for (int kb = 0; kb < p.k_blocks; ++kb) {
                        ptx::mbar_wait(empty_bar + 8 * stage, phase ^ 1);
                        const uint32_t fb = full_bar + 8 * stage;
                        ptx::mbar_arrive_expect_tx(fb, tx);
                        const uint32_t a_dst = a_base + stage * (BM * BK * 2);
                        const uint32_t b_dst = b_base + stage * p.b_stage_bytes;
                        const int k0 = kb * BK;
                        if constexpr (KIND == KIND_GEMM) {
                            // A = [groups][n_tok][K(|K)] ; B = [groups][K][N] (MN) or [groups][N][K]
                            // Compensated A: blocks >= kb_half read the lo half against the same B rows.
                            const int part = kb >= p.kb_half ? 1 : 0;
                            const int kk0 = (kb - part * p.kb_half) * BK;
                            ptx::tma_load_3d(a_dst, &tmA, fb, part * p.a_lo_off + kk0, m0, tc.g);
                            if (p.b_mn_major) {
                                for (int j = 0; j < p.b_boxes; ++j)
                                    ptx::tma_load_3d(b_dst + j * (p.b_box_n * BK * 2), &tmB, fb,
                                                     n0 + j * p.b_box_n, kk0, tc.g);
                            } else {
                                ptx::tma_load_3d(b_dst, &tmB, fb, kk0, n0, tc.g);
                            }
                        } else if constexpr (KIND == KIND_MONARCH_PROJ) {
                            // A = X viewed [n_tok][b1][p]; B = V viewed 4-D (a, rho', k, l):
                            // rows of the N tile arrive k-major whatever V's composite order.
                            ptx::tma_load_3d(a_dst, &tmA, fb, k0, tc.g, m0);
                            ptx::tma_load_4d(b_dst, &tmB, fb, k0, 0, tc.n_blk * p.kb_per_tile, tc.g);
                        } else {  // KIND_BLAST_PROJ: sub = l
                            ptx::tma_load_3d(a_dst, &tmA, fb, k0, sub, m0);
                            for (int j = 0; j < p.b_boxes; ++j)
                                ptx::tma_load_3d(b_dst + j * (p.b_box_n * BK * 2), &tmB, fb,
                                                 n0 + j * p.b_box_n, k0, sub);
                        }
                        if (++stage == p.stages) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================================================== MMA issuer ===================
        if (lane == 0) {
            const uint32_t idesc = ptx::idesc_bf16(BM, p.BN, p.b_mn_major);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int tile = blockIdx.x; tile < p.total_tiles; tile += gridDim.x) {
                ptx::mbar_wait(tempty_bar + 8 * acc, acc_phase ^ 1);
                ptx::tc_fence_after();
                for (int sub = 0; sub < p.n_sub; ++sub) {
                    const uint32_t d_tmem = tmem_base + acc * acc_stride + sub * p.BN;
                    for (int kb = 0; kb < p.k_blocks; ++kb) {
                        ptx::mbar_wait(full_bar + 8 * stage, phase);
                        ptx::tc_fence_after();
                        const uint32_t a_s = a_base + stage * (BM * BK * 2);
                        const uint32_t b_s = b_base + stage * p.b_stage_bytes;
#pragma unroll
                        for (int kk = 0; kk < BK / UMMA_K; ++kk) {
                            // A: K-major, 128-B swizzle, 8-row groups 1024 B apart; +32 B per K=16.
                            const uint64_t ad = ptx::smem_desc(a_s + kk * 32, 16, 1024, ptx::LAYOUT_SW128);
                            const uint64_t bd = ptx::smem_desc(b_s + kk * p.b_kstep, p.b_lbo, p.b_sbo, p.b_layout);
                            ptx::mma_bf16(d_tmem, ad, bd, idesc, (kb | kk) != 0);
                        }
                        ptx::mma_commit(empty_bar + 8 * stage);  // frees the smem slot
                        if (++stage == p.stages) { stage = 0; phase ^= 1; }
                    }
                }
                ptx::mma_commit(tfull_bar + 8 * acc);  // accumulator ready for the epilogue
                if (++acc == p.acc_bufs) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else {
        // ===================================================== epilogue =====================
        const int ew = warp - 2;              // 0..7
        const int quarter = warp & 3;         // TMEM lane quarter this warp may access
        const int half = ew >> 2;             // which half of the columns
        const int row_in_tile = quarter * 32 + lane;
        const uint32_t lane_addr = static_cast<uint32_t>(quarter * 32) << 16;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int tile = blockIdx.x; tile < p.total_tiles; tile += gridDim.x) {
            const TileCoord tc = tile_coord(p, tile);
            const int t = tc.m_blk * BM + row_in_tile;
            const int n0 = tc.n_blk * p.BN;
            if constexpr (KIND == KIND_BLAST_PROJ) {
                // stage S[l][k][n0 : n0+BN] (fp32) for the S-weighted block sum
                ptx::named_bar_sync(1, 32 * NUM_EPI_WARPS);
                const int cnt = p.b1 * p.b2 * p.BN;
                for (int e = ew * 32 + lane; e < cnt; e += 32 * NUM_EPI_WARPS) {
                    const int rho = e % p.BN;
                    const int lk = e / p.BN;
                    const int rr = n0 + rho;
                    s_tile[e] = rr < p.r ? __bfloat162float(p.S[static_cast<long long>(lk) * p.r + rr]) : 0.f;
                }
                ptx::named_bar_sync(1, 32 * NUM_EPI_WARPS);
            }
            ptx::mbar_wait(tfull_bar + 8 * acc, acc_phase);
            ptx::tc_fence_after();
            const uint32_t tbase = tmem_base + acc * acc_stride + lane_addr;

            if constexpr (KIND == KIND_BLAST_PROJ) {
                // Z''_k[t, rho] = sum_l S[l,k,rho] * Z_l[t, rho]   (Fig. 6 "s * z'")
                const int nsc = p.BN / 8;
                for (int sc = half; sc < nsc; sc += 2) {
                    float acc8[16][8];
#pragma unroll
                    for (int k = 0; k < 16; ++k)
#pragma unroll
                        for (int e = 0; e < 8; ++e) acc8[k][e] = 0.f;
                    for (int l = 0; l < p.b1; ++l) {
                        float z[8];
                        ptx::tmem_ld_x8(tbase + l * p.BN + sc * 8, z);
                        ptx::tmem_wait_ld();
                        const float* srow = s_tile + (l * p.b2) * p.BN + sc * 8;
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
                            if (k < p.b2) {
                                const float4 s0 = *reinterpret_cast<const float4*>(srow + k * p.BN);
                                const float4 s1 = *reinterpret_cast<const float4*>(srow + k * p.BN + 4);
                                acc8[k][0] = fmaf(s0.x, z[0], acc8[k][0]);
                                acc8[k][1] = fmaf(s0.y, z[1], acc8[k][1]);
                                acc8[k][2] = fmaf(s0.z, z[2], acc8[k][2]);
                                acc8[k][3] = fmaf(s0.w, z[3], acc8[k][3]);
                                acc8[k][4] = fmaf(s1.x, z[4], acc8[k][4]);
                                acc8[k][5] = fmaf(s1.y, z[5], acc8[k][5]);
                                acc8[k][6] = fmaf(s1.z, z[6], acc8[k][6]);
                                acc8[k][7] = fmaf(s1.w, z[7], acc8[k][7]);
                            }
                        }
                    }
                    const int rho0 = n0 + sc * 8;
                    if (t < p.n_tok && rho0 < p.r) {
#pragma unroll
                        for (int k = 0; k < 16; ++k) {
                            if (k < p.b2) {
                                __nv_bfloat16* dst = p.out + (static_cast<long long>(k) * p.n_tok + t) * p.out_ld + rho0;
                                store8(dst, acc8[k], p.out_lo_off);
                            }
                        }
                    }
                }
            } else {
                const int nvalid = min(p.BN, p.N - n0);
                for (int c0 = half * 32; c0 < nvalid; c0 += 64) {
                    uint32_t v[32];
                    ptx::tmem_ld_x32(tbase + c0, v);
                    ptx::tmem_wait_ld();
                    if (t < p.n_tok) {
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int c = c0 + j * 8;
                            if (c < nvalid) {
                                float f[8];
#pragma unroll
                                for (int e = 0; e < 8; ++e) f[e] = __uint_as_float(v[j * 8 + e]);
                                __nv_bfloat16* dst;
                                if constexpr (KIND == KIND_GEMM) {
                                    // Y[t, g*N + n0 + c]  (canonical k-major output)
                                    dst = p.out + static_cast<long long>(t) * p.out_ld +
                                          static_cast<long long>(tc.g) * p.N + n0 + c;
                                } else {
                                    // Monarch: column c of the tile is (k, rho') = (k0 + c / r', c % r');
                                    // Z'[k][t][l r' + rho']  (the b2 <-> b1 permutation)
                                    const int k = tc.n_blk * p.kb_per_tile + c / p.r_blk;
                                    const int rho = c % p.r_blk;
                                    dst = p.out + (static_cast<long long>(k) * p.n_tok + t) * p.out_ld +
                                          tc.g * p.r_blk + rho;
                                }
                                store8(dst, f, p.out_lo_off);
                            }
                        }
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(tempty_bar + 8 * acc);
            if (++acc == p.acc_bufs) { acc = 0; acc_phase ^= 1; }
        }
    }

    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<TMEM_COLS>(tmem_base);
    }
}

}  // namespace blr
