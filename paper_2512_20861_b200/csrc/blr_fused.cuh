// blr_fused.cuh -- one-launch low-rank / Monarch layer (SURVEY §8 rows a1-a2, m1-m3 in one kernel).
//
// For every 128-token tile the CTA computes the rank-r intermediate and consumes it on chip:
//   low rank  Z  = X V      then  Y   = Z U
//   Monarch   Z'_k = [X_l V_{l,k}]_l   then  Y_k = Z'_k U_k^T
// S1 accumulates Z in TMEM (sub-GEMM l of Monarch at columns l r': the b2<->b1 permutation of
// PAPER.md L194 is that column placement, the r'<->b2 one is the V tensor-map box as in the
// two-kernel path); the epilogue warps round Z once to bf16 (RNE, R11) straight into
// shared memory in the 128-B-swizzled K-major layout a TMA load would have produced, and S3 takes
// it from there as its A operand.  Z never reaches HBM and the layer is one launch instead of two
// (the intermediate round trip is what makes the unfused layer memory-bound).
//
// Work item = (128-token tile T, output block k (Monarch; 1 for low rank), part of the S3 N range).
// S1 is recomputed per part (the N split only exists to fill the SMs at small token counts).
// Roles as in blr_gemm_kernel: warp 0 TMA producer, warp 1 TMEM owner + MMA issuer, warps 2..9
// epilogue (two per TMEM lane quarter).  One operand ring carries S1 steps (X block + V block) and
// S3 steps (U block) in program order.  TMEM: two 256-column accumulator buffers used strictly
// alternately by the sequence  Z(item 0), Y chunks(item 0), Z(item 1), ...
#pragma once
#include "blr_kernels.cuh"

namespace blr {

struct FParams {
    int n_tok, tiles_m;
    int g2, n_parts, items;  // items = tiles_m * g2 * n_parts, item = (T * g2 + k) * n_parts + part
    int mon;                 // 1: Monarch operand addressing, 0: low rank
    uint32_t s1_bytes;       // bytes of one S1 step (X block + V block) in a ring slot
    // S1: g1 sub-GEMMs (Monarch l), each K1 = k1_blocks * 64, N = n1 columns at TMEM col s * n1
    int g1, k1_blocks, n1;
    int b1_mn, b1_boxes;
    uint32_t b1_bytes, b1_lbo, b1_sbo, b1_kstep;
    // Z: k2 = g1 * n1 columns (multiple of 64, <= 256), k2 / 64 swizzled 16-KB blocks in smem
    int k2;
    // S3: N range n2 per output block, chunks of bn2 columns, n2_part columns per item
    int n2, bn2, n2_part;
    int b2_mn, b2_boxes;
    uint32_t b2_bytes, b2_lbo, b2_sbo, b2_kstep;
    // ring / epilogue
    uint32_t slot_bytes;
    int stages;
    int c_box_w;
    uint32_t c_swz, stage_warp_bytes;  // stage_warp_bytes = stage_bufs x (32 rows x c_box_w bf16)
    int stage_bufs;
    // > 0: Monarch "transposed" output order, Y[t, c * y_cs + k] stored
    // directly (no TMA box exists for a 2-byte innermost extent)
    int y_cs;
    long long y_rs;
    __nv_bfloat16* y;
    int coop_store;  // 1: the four warps of a column half store a Y chunk's 128 rows as ONE tensor box
};

struct FLayout {
    uint32_t ring, zs, stg, bars, total;
};
__host__ __device__ inline FLayout fused_layout(const FParams& p) {
    FLayout L;
    L.ring = 0;
    L.zs = L.ring + p.slot_bytes * p.stages;
    L.stg = L.zs + (p.k2 / 64) * 16384u;
    L.bars = L.stg + p.stage_warp_bytes * NUM_EPI_WARPS;
    L.total = L.bars + 8 * (2 * MAX_STAGES + 6) + 16;
    return L;
}

__global__ void __launch_bounds__(NUM_THREADS, 1)
    blr_fused_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB1,
                     const __grid_constant__ CUtensorMap tmB2, const __grid_constant__ CUtensorMap tmC,
                     const FParams p) {
    extern __shared__ __align__(1024) uint8_t fsmem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(fsmem_raw) + 1023) & ~uintptr_t(1023));
    const FLayout L = fused_layout(p);
    const uint32_t sbase = ptx::smem_u32(smem);
    const uint32_t ring = sbase + L.ring, zs = sbase + L.zs;
    const uint32_t full_bar = sbase + L.bars;
    const uint32_t empty_bar = full_bar + 8 * MAX_STAGES;
    const uint32_t tfull_bar = empty_bar + 8 * MAX_STAGES;  // [2]
    const uint32_t tempty_bar = tfull_bar + 16;             // [2]
    const uint32_t zready_bar = tempty_bar + 16;            // epilogue -> MMA: Z staged in smem
    const uint32_t zsfree_bar = zready_bar + 8;             // MMA -> epilogue: S3 done reading Z
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.bars + 8 * (2 * MAX_STAGES + 6));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

    if (warp == 0) {
        for (int s = lane; s < p.stages; s += 32) {
            ptx::mbar_init(full_bar + 8 * s, 1);
            ptx::mbar_init(empty_bar + 8 * s, 1);
        }
        if (lane < 2) {
            ptx::mbar_init(tfull_bar + 8 * lane, 1);
            ptx::mbar_init(tempty_bar + 8 * lane, NUM_EPI_WARPS);
        }
        if (lane == 0) {
            ptx::mbar_init(zready_bar, NUM_EPI_WARPS);
            ptx::mbar_init(zsfree_bar, 1);
        }
        ptx::fence_barrier_init();
        if (lane == 0) {
            ptx::prefetch_tmap(&tmA);
            ptx::prefetch_tmap(&tmB1);
            ptx::prefetch_tmap(&tmB2);
            ptx::prefetch_tmap(&tmC);
        }
    }
    if (warp == 1) ptx::tmem_alloc<TMEM_COLS>(ptx::smem_u32(tmem_slot));
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    const int k2b = p.k2 / 64;
    // item -> (token tile, output block, part); the S3 column range of the item
    auto item_of = [&](int it, int& T, int& kq, int& c_lo, int& c_hi) {
        const int w = blockIdx.x + it * gridDim.x;
        const int part = w % p.n_parts;
        const int tk = w / p.n_parts;
        kq = tk % p.g2;
        T = tk / p.g2;
        c_lo = part * p.n2_part;
        c_hi = min(p.n2, c_lo + p.n2_part);
    };
    const int nitems = blockIdx.x < p.items ? (p.items - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

    if (warp == 0) {
        // ============================================================ TMA producer ==========
        int stage = 0;
        uint32_t phase = 0;
        // loop parameters pinned in registers (the compiler otherwise re-reads them from the
        // constant bank after every asm statement; DESIGN.md §5.1 "lean producer")
        const int stages = ptx::pin(p.stages), g1 = ptx::pin(p.g1), k1b = ptx::pin(p.k1_blocks);
        const int bn2 = ptx::pin(p.bn2), b1_boxes = ptx::pin(p.b1_boxes), b2_boxes = ptx::pin(p.b2_boxes);
        const uint32_t slot_bytes = ptx::pin(p.slot_bytes), s1_bytes = ptx::pin(p.s1_bytes);
        const uint32_t b2_bytes = ptx::pin(p.b2_bytes);
        const bool mon = p.mon != 0, b2_mn = p.b2_mn != 0;
        ptx::griddep_wait();  // X may be the previous kernel's output
        // the next kernel may start its prologue only once everything before this launch is
        // complete (it may read weights before its own griddepcontrol.wait)
        ptx::griddep_launch_dependents();
        for (int it = 0; it < nitems; ++it) {
            int T, kq, c_lo, c_hi;
            item_of(it, T, kq, c_lo, c_hi);
            const int m0 = T * BM;
            for (int s = 0; s < g1; ++s) {  // S1 steps: X block + V block
                for (int kb = 0; kb < k1b; ++kb) {
                    ptx::mbar_wait(empty_bar + 8 * stage, phase ^ 1);
                    const uint32_t slot = ring + stage * slot_bytes, fb = full_bar + 8 * stage;
                    if (ptx::elect_one()) {
                        ptx::mbar_arrive_expect_tx(fb, s1_bytes);
                        const int k0 = kb * BK;
                        if (mon) {
                            ptx::tma_load_3d(slot, &tmA, fb, k0, s, m0);              // X viewed (p, b1, n)
                            ptx::tma_load_4d(slot + BM * BK * 2, &tmB1, fb, k0, 0, kq, s);  // V_{l,k} rows
                        } else {
                            ptx::tma_load_3d(slot, &tmA, fb, k0, m0, 0);
                            for (int j = 0; j < b1_boxes; ++j)
                                ptx::tma_load_3d(slot + BM * BK * 2 + j * (64 * BK * 2), &tmB1, fb, j * 64, k0, 0);
                        }
                    }
                    __syncwarp();
                    if (++stage == stages) { stage = 0; phase ^= 1; }
                }
            }
            for (int c0 = c_lo; c0 < c_hi; c0 += bn2) {  // S3 steps: U blocks
                for (int kb = 0; kb < k2b; ++kb) {
                    ptx::mbar_wait(empty_bar + 8 * stage, phase ^ 1);
                    const uint32_t slot = ring + stage * slot_bytes, fb = full_bar + 8 * stage;
                    if (ptx::elect_one()) {
                        ptx::mbar_arrive_expect_tx(fb, b2_bytes);
                        if (b2_mn) {
                            for (int j = 0; j < b2_boxes; ++j)
                                ptx::tma_load_3d(slot + j * (64 * BK * 2), &tmB2, fb, c0 + j * 64, kb * BK, kq);
                        } else {
                            ptx::tma_load_3d(slot, &tmB2, fb, kb * BK, c0, kq);  // U_k [q][b1 r'] K-major
                        }
                    }
                    __syncwarp();
                    if (++stage == stages) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ============================================================ MMA issuer ============
        const uint32_t idesc1 = ptx::idesc_bf16(BM, p.n1, p.b1_mn);
        const uint32_t idesc2 = ptx::idesc_bf16(BM, p.bn2, p.b2_mn);
        const int stages = ptx::pin(p.stages), g1 = ptx::pin(p.g1), k1b = ptx::pin(p.k1_blocks), n1 = ptx::pin(p.n1);
        const int bn2 = ptx::pin(p.bn2);
        const uint32_t slot_bytes = ptx::pin(p.slot_bytes);
        const uint32_t b1_kstep = ptx::pin(p.b1_kstep), b1_lbo = ptx::pin(p.b1_lbo), b1_sbo = ptx::pin(p.b1_sbo);
        const uint32_t b2_kstep = ptx::pin(p.b2_kstep), b2_lbo = ptx::pin(p.b2_lbo), b2_sbo = ptx::pin(p.b2_sbo);
        int stage = 0;
        uint32_t phase = 0;
        uint32_t use = 0;  // accumulator uses so far (buffer = use & 1)
        for (int it = 0; it < nitems; ++it) {
            int T, kq, c_lo, c_hi;
            item_of(it, T, kq, c_lo, c_hi);
            {   // ---- S1: Z into buffer use & 1
                const uint32_t b = use & 1;
                ptx::mbar_wait(tempty_bar + 8 * b, ((use >> 1) & 1) ^ 1);
                ptx::tc_fence_after();
                for (int s = 0; s < g1; ++s) {
                    const uint32_t d = tmem_base + b * 256 + s * n1;
                    for (int kb = 0; kb < k1b; ++kb) {
                        ptx::mbar_wait(full_bar + 8 * stage, phase);
                        ptx::tc_fence_after();
                        if (ptx::elect_one()) {
                            const uint32_t slot = ring + stage * slot_bytes;
#pragma unroll
                            for (int kk = 0; kk < BK / UMMA_K; ++kk) {
                                const uint64_t ad = ptx::smem_desc(slot + kk * 32, 16, 1024, ptx::LAYOUT_SW128);
                                const uint64_t bd = ptx::smem_desc(slot + BM * BK * 2 + kk * b1_kstep, b1_lbo, b1_sbo,
                                                                   ptx::LAYOUT_SW128);
                                ptx::mma_bf16(d, ad, bd, idesc1, (kb | kk) != 0);
                            }
                            ptx::mma_commit(empty_bar + 8 * stage);
                        }
                        __syncwarp();
                        if (++stage == stages) { stage = 0; phase ^= 1; }
                    }
                }
                if (ptx::elect_one()) ptx::mma_commit(tfull_bar + 8 * b);
                __syncwarp();
                ++use;
            }
            ptx::mbar_wait(zready_bar, it & 1);  // Z (bf16) is in smem
            ptx::tc_fence_after();
            for (int c0 = c_lo; c0 < c_hi; c0 += bn2) {  // ---- S3 chunks
                const uint32_t b = use & 1;
                ptx::mbar_wait(tempty_bar + 8 * b, ((use >> 1) & 1) ^ 1);
                ptx::tc_fence_after();
                for (int kb = 0; kb < k2b; ++kb) {
                    ptx::mbar_wait(full_bar + 8 * stage, phase);
                    ptx::tc_fence_after();
                    if (ptx::elect_one()) {
                        const uint32_t slot = ring + stage * slot_bytes;
#pragma unroll
                        for (int kk = 0; kk < BK / UMMA_K; ++kk) {
                            const uint64_t ad = ptx::smem_desc(zs + kb * 16384 + kk * 32, 16, 1024, ptx::LAYOUT_SW128);
                            const uint64_t bd = ptx::smem_desc(slot + kk * b2_kstep, b2_lbo, b2_sbo, ptx::LAYOUT_SW128);
                            ptx::mma_bf16(tmem_base + b * 256, ad, bd, idesc2, (kb | kk) != 0);
                        }
                        ptx::mma_commit(empty_bar + 8 * stage);
                    }
                    __syncwarp();
                    if (++stage == stages) { stage = 0; phase ^= 1; }
                }
                if (ptx::elect_one()) ptx::mma_commit(tfull_bar + 8 * b);
                __syncwarp();
                ++use;
            }
            if (ptx::elect_one()) ptx::mma_commit(zsfree_bar);  // every S3 MMA of this item has read Z
            __syncwarp();
        }
    } else {
        // ============================================================ epilogue ==============
        const int ew = warp - 2, quarter = warp & 3, half = ew >> 2;
        const uint32_t lane_addr = static_cast<uint32_t>(quarter * 32) << 16;
        const uint32_t stg = sbase + L.stg + ew * p.stage_warp_bytes;
        const int row = quarter * 32 + lane;
        const int CW = p.c_box_w;
        const uint32_t row_bytes = CW * 2;
        uint32_t use = 0;
        uint32_t nstore = 0;  // staged Y chunks (staging buffer rotation)
        ptx::griddep_wait();  // our Y stores must not overtake the previous kernel's reads
        for (int it = 0; it < nitems; ++it) {
            int T, kq, c_lo, c_hi;
            item_of(it, T, kq, c_lo, c_hi);
            const int row0 = T * BM + quarter * 32;
            {   // ---- Z: TMEM -> bf16 (RNE) -> swizzled K-major smem, this warp's half of the columns
                const uint32_t b = use & 1;
                ptx::mbar_wait(tfull_bar + 8 * b, (use >> 1) & 1);
                ptx::tc_fence_after();
                if (it > 0) ptx::mbar_wait(zsfree_bar, (it - 1) & 1);  // previous item's S3 read Z
                const int cbeg = half * (p.k2 / 2), cend = cbeg + p.k2 / 2;
                for (int c = cbeg; c < cend; c += 32) {
                    float f[4][8];
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        if (c + j * 8 < cend) ptx::tmem_ld_x8(tmem_base + lane_addr + b * 256 + c + j * 8, f[j]);
                    ptx::tmem_wait_ld();
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const int cc = c + j * 8;
                        if (cc < cend) {
                            uint4 w;
                            w.x = ptx::pack_bf16x2(f[j][0], f[j][1]);
                            w.y = ptx::pack_bf16x2(f[j][2], f[j][3]);
                            w.z = ptx::pack_bf16x2(f[j][4], f[j][5]);
                            w.w = ptx::pack_bf16x2(f[j][6], f[j][7]);
                            const uint32_t chunk = (cc & 63) >> 3;
                            ptx::st_shared_v4(zs + (cc >> 6) * 16384u + row * 128u + ((chunk ^ (row & 7)) << 4), w);
                        }
                    }
                }
                ptx::fence_async_smem();  // generic-proxy writes -> visible to the tensor core
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    ptx::mbar_arrive(tempty_bar + 8 * b);
                    ptx::mbar_arrive(zready_bar);
                }
                ++use;
            }
            for (int n0 = c_lo; n0 < c_hi; n0 += p.bn2) {  // ---- Y chunks: TMEM -> bf16 -> TMA store
                const uint32_t b = use & 1;
                ptx::mbar_wait(tfull_bar + 8 * b, (use >> 1) & 1);
                ptx::tc_fence_after();
                const int nvalid = min(p.bn2, c_hi - n0);
                for (int c0 = half * CW; c0 < nvalid; c0 += 2 * CW) {
                    float fv[64];
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (j * 8 < CW) ptx::tmem_ld_x8(tmem_base + lane_addr + b * 256 + c0 + j * 8,
                                                        *reinterpret_cast<float(*)[8]>(&fv[j * 8]));
                    ptx::tmem_wait_ld();
                    if (p.y_cs > 0) {  // transposed order: Y[t, c * b2 + k], strided direct stores
                        const int t = T * BM + row;
                        if (t < p.n_tok) {
                            __nv_bfloat16* yb = p.y + static_cast<long long>(t) * p.y_rs + kq;
#pragma unroll
                            for (int j = 0; j < 64; ++j) {
                                const int c = n0 + c0 + j;
                                if (j < CW && c < p.n2) yb[static_cast<long long>(c) * p.y_cs] = __float2bfloat16_rn(fv[j]);
                            }
                        }
                        continue;
                    }
                    if (p.coop_store) {  // 128-row cooperative store (a quarter of the TMA store ops)
                        const uint32_t hbuf = sbase + L.stg + half * 4u * p.stage_warp_bytes +
                                              (nstore % p.stage_bufs) * (128u * row_bytes);
                        ++nstore;
                        const bool iss = (ew & 3) == 0 && lane == 0;
                        if (iss) {
                            if (p.stage_bufs == 2) ptx::bulk_wait_read<1>();
                            else ptx::bulk_wait_read<0>();
                        }
                        ptx::named_bar_sync(2 + half, 128);
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            if (j * 8 < CW)
                                stage_row8(hbuf, row, j, row_bytes, p.c_swz, *reinterpret_cast<const float(*)[8]>(&fv[j * 8]), 0);
                        ptx::fence_async_smem();
                        ptx::named_bar_sync(2 + half, 128);
                        if (iss) {
                            ptx::tma_store_4d(&tmC, hbuf, n0 + c0, 0, kq, T * BM);
                            ptx::bulk_commit();
                        }
                        continue;
                    }
                    const uint32_t buf = stg + (nstore % p.stage_bufs) * (32u * row_bytes);
                    ++nstore;
                    if (lane == 0) {  // the store that last read this staging buffer is done reading it
                        if (p.stage_bufs == 2) ptx::bulk_wait_read<1>();
                        else ptx::bulk_wait_read<0>();
                    }
                    __syncwarp();
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        if (j * 8 < CW)
                            stage_row8(buf, lane, j, row_bytes, p.c_swz, *reinterpret_cast<const float(*)[8]>(&fv[j * 8]), 0);
                    ptx::fence_async_smem();
                    __syncwarp();
                    if (lane == 0) {
                        ptx::tma_store_4d(&tmC, buf, n0 + c0, 0, kq, row0);  // Y (c, 0, k, t), rows >= n clipped
                        ptx::bulk_commit();
                    }
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(tempty_bar + 8 * b);
                ++use;
            }
        }
        if (lane == 0) ptx::bulk_wait_read<0>();
        __syncwarp();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<TMEM_COLS>(tmem_base);
    }
}

}  // namespace blr
