// blr_kernels.cuh -- the sm_100a kernels of the BLR prefill forward (arXiv 2512.20861).
//
// One warp-specialized, persistent tcgen05 GEMM kernel template, instantiated for the phases of
// every format:
//
//   KIND_GEMM          out[g](t, c) = sum_kk A[g](t, kk) B[g](kk, c)        grouped GEMM
//       lowrank S1: Z = X V, S3: Y = Z U
//       Monarch S3: Y_k = Z'_k U_k^T
//       BLAST   S1: Z_l = X_l V_l (grouped over l), S3: Y_k = Z''_k U_k
//   KIND_MONARCH_PROJ  Z'[k][t][l r' + rho] = (X_l V_{l,k})[t, rho]
//       the r'<->b2 and b2<->b1 permutations of PAPER.md L194 are folded into a 4-D TMA box
//       over V (N rows delivered k-major whatever V's layout) and into the store coordinates.
//   KIND_BLAST_PROJ    Z''[k][t][rho] = sum_l S[l,k,rho] (X_l V_l)[t, rho]
//       b1 accumulators side by side in TMEM; the epilogue applies the S-weighted block sum with
//       packed fp32x2 FMAs (used when b1 * r fits TMEM; else BLAST runs S1/S2/S3 separately).
//
// Roles: warp 0 = TMA producer (1 thread), warp 1 = TMEM allocator + MMA issuer (1 thread),
// warps 2..9 = epilogue (two warps per TMEM lane quarter, each half of the tile's columns).
// A streams through a STAGES-deep smem ring (full/empty mbarriers).  B either streams through
// the same ring, or -- "weight-stationary" mode -- is loaded once per (group, N-block) slice into
// a resident smem region while the CTA walks a contiguous run of token tiles, so per-SM ingress
// is only the activations (the per-SM TMA ingress is ~63 B/clk, benchmarks/micro).  TMEM
// accumulators are double-buffered when two fit in 512 columns.  Epilogue: tcgen05.ld ->
// bf16 (RNE) -> 128B-swizzled smem staging -> TMA bulk tensor store (full lines, OOB clipped).
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
constexpr int MAX_BRES = 48;       // max resident B k-blocks (one mbarrier each)

enum Kind : int { KIND_GEMM = 0, KIND_MONARCH_PROJ = 1, KIND_BLAST_PROJ = 2 };

// Debug switches that skip kernel stages (timing experiments only; the results are then wrong).
// Compiled in only with -DBLR_DEBUG_KNOBS; release builds ignore KParams::dbg entirely.
#ifdef BLR_DEBUG_KNOBS
constexpr bool kGenericProducer = true;
#define BLR_DBG_ON(p, bit) (((p).dbg & (bit)) != 0)
#else
// release builds carry only the lean producer loop: the smaller kernel measured faster on small
// problems, whose short launches start with a cold instruction cache (DiT-XL/2 one image 45 -> 42 us)
constexpr bool kGenericProducer = false;
#define BLR_DBG_ON(p, bit) false
#endif

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
    int a_gmid;       // A map coordinate order: 0 = (k, t, g), 1 = (k, g, t)
    int a_blocked;    // 1: A stored tile-blocked [g][T][K/8][128][8] (BLAST Z''): a 64-K block of a
                      //    tile is 8 adjacent 2-KB panels, one bulk copy into 8 no-swizzle K core-matrix columns
    const __nv_bfloat16* a_ptr;  // a_blocked: A base
    int a_nchunks;               // a_blocked: K / 8
    int a_tiles;                 // a_blocked: 128-row tiles per group in the layout
    int o_tiles;                 // OUTF 2: 128-row tiles per group of the tile-blocked output
    int kbox;         // 64-wide K blocks per pipeline stage (1 or 2; 2 halves the handshakes)
    int n_sub;        // sub-GEMMs accumulated into separate TMEM slots (BLAST proj: b1)
    int stages;       // smem ring depth
    int acc_bufs;     // TMEM accumulator buffers (1 or 2)
    int b_resident;   // 1: B slice resident in smem per (group, N-block) (weight-stationary)
    int nb_runs;      // streaming only: 1 = each CTA takes the tiles_n N blocks of one (token tile,
                      // group) back to back (its A tile re-read from L2 while hot), 0 = plain round robin
    int cps;          // >0 (resident only): each CTA owns slice blockIdx % slices and 1/cps of the
                      // token tiles; all CTAs walk their token range in lockstep (L2 reuse of A)
    // ---- B operand staging
    int b_mn_major;      // 1: B stored [K][N] (N contiguous), 0: B stored [N][K]
    int n_mma;           // 1, or 2 (wide tile, GEMM kind, streamed B): each K step issues two MMAs of
                         // N = BN/2 from the same A into adjacent TMEM columns; B is staged as two
                         // halves of b_half_bytes (half h covers tile columns [h BN/2, (h+1) BN/2))
    uint32_t b_half_bytes;
    int mc;              // PAIR 2, streamed B: CTA pairs per cluster sharing the tile's B (same group and
                         // N block, consecutive token tiles): each loads 1/mc of the K rows of every B
                         // box and TMA-multicasts it to the same-rank CTA of every pair (L2 -> SM bytes
                         // per MAC drop; the streamed GEMMs run at the chip's L2 read rate)
    int b_boxes;         // TMA boxes per k-block for B (MN-major; per half when n_mma = 2)
    int b_box_n;         // N elements per box (MN-major)
    uint32_t b_stage_bytes;  // bytes of one B k-block in smem
    uint32_t b_lbo, b_sbo, b_layout, b_kstep;  // UMMA descriptor parameters for B
    // ---- epilogue
    long long out_lo_off;  // >0: also store lo = bf16(z - bf16(z)) (compensated intermediate)
    int c_box_w;           // staged store chunk width (elements)
    uint32_t c_swz;        // staging swizzle mask (7: 128 B, 3: 64 B, 1: 32 B, 0: none) = TMA map's
    uint32_t stage_warp_bytes;  // staging bytes per epilogue warp
    int stage_bufs;        // staging buffers per warp (GEMM / Monarch kinds)
    void* out_ptr;         // OUTF 2 (tile-blocked [g][T][N/8][128][8] fp16, bulk stores) or out_cs: output base
    long long out_gstride; // OUTF 2 / out_cs: elements between groups
    long long out_rs;      // out_cs: elements between rows
    int out_cs;            // > 0: bf16 element (t, g, c) stored directly at t*out_rs + g*out_gstride + c*out_cs
                           //      (Monarch "transposed" output order: no TMA box exists
                           //      for a 2-byte innermost extent)
    int r_blk;             // Monarch: r'
    int kb_per_tile;       // Monarch: output blocks k per N tile
    int b1, b2;            // BLAST block counts
    int r;                 // BLAST: rank
    const __nv_bfloat16* S;  // BLAST: S [b1][b2][r]
    unsigned long long* trace;  // debug: per-CTA %globaltimer stamps [grid][64] (nullptr = off)
    int first;                  // 1: first launch of an API call (see the PDL note in the kernel)
    int mma_burst;              // 1: full K blocks issued as one unrolled MMA burst (MMA issuer)
    int dbg;                    // debug bits (BLR_DEBUG_KNOBS builds only): 1 skip bulk stores, 2 skip staging,
                                //   4 skip the whole GEMM epilogue, 8 skip MMAs, 16 plain-arrive slot release (PAIR 1),
                                //   32 no accumulator hand-off, 64 no resident weight loads
    int fast_prod;              // 1: the lean GEMM producer loop (BLR_FASTPROD=0 selects the generic one)
    int coop_store;             // 1: 128-row cooperative output stores (one box per chunk per column half)
    int l2_a, l2_b, l2_out;     // L2 cache-policy hints of the A / B loads and the output stores (lean
                                // producer and GEMM-kind epilogues): 0 none, 1 evict_first, 2 evict_last
    int b_slab2;                // 1: MN-major B with two 64-column boxes per K block: a slab view of B (tmB2,
    int b_nslab;                //    b_nslab whole 64-column slabs) loads both boxes with ONE TMA op when the
                                //    CTA's columns are two whole slabs (the per-SM TMA op rate)
    // ---- pipelined BLAST layer (blast_pipe_kernel): per-128-token-tile ready counters
    const unsigned int* pipe_wait;  // A's token tile t is ready once pipe_wait[t] >= pipe_target (nullptr: off)
    unsigned int pipe_target;
    unsigned int* pipe_sig;         // the epilogue adds 1 per (tile, store issuer) once the tile's stores landed
    const unsigned int* pipe_bp;    // back-pressure: token tile t starts once pipe_bp[t - pipe_bp_dist] >=
    unsigned int pipe_bp_target;    //   pipe_bp_target (the consumer stage is that far behind; nullptr: off)
    int pipe_bp_dist;
    int no_trigger;                 // 1: never trigger the dependent grid early (its CTAs could take the SMs
                                    //    this grid's later CTAs need while the earlier ones wait on them)
    int tab_n;                      // tile-table entries (0: TILE_TAB); wide plans take 128 so a fourth
                                    // 48-KB ring stage fits
    int last_nb;                    // > 0: the last N tile's MMA is only last_nb columns wide (its valid
                                    // columns rounded up to 16) and each CTA of a pair loads last_nb / 2
                                    // of them: no MMA work on padding columns (C4 gate S3: 688 = 256 +
                                    // 256 + 176)
    int last_half;                  // wide plan (split_rel): the last N tile holds <= BN/2 valid columns
                                    // and runs as column half 0 alone, last_nb wide (C4 gate S3: 688 =
                                    // 512 + 176): its B half 1 is neither loaded nor multiplied
    int split_rel;                  // wide tile, one accumulator: the epilogue frees the two MMA column
                                    // halves separately (tempty_bar[0] / [1]); the next tile's K steps
                                    // start on half 0 and hold their ring slots until half 1 is free,
                                    // then catch up
};

struct SmemLayout {
    uint32_t a_off, b_off, c_off, s_off, bar_off, tab_off, zero_off, total;
};
// Per-CTA tile table: the coordinates of the CTA's first TILE_TAB tiles, computed once by all
// threads in the prologue, so the single-thread producer / MMA loops and the epilogue do no
// integer division per tile (the per-tile index arithmetic of one thread measured ~0.5 us).
constexpr int TILE_TAB = 256;
__host__ __device__ inline int tile_tab_n(const KParams& p) { return p.tab_n > 0 ? p.tab_n : TILE_TAB; }

__host__ __device__ inline int kb_resident(const KParams& p) {  // resident B blocks (padded to kbox)
    return (p.kb_half + p.kbox - 1) / p.kbox * p.kbox;
}
__host__ __device__ inline uint32_t b_region_bytes(const KParams& p) {
    return p.b_resident ? p.b_stage_bytes * kb_resident(p) : p.b_stage_bytes * p.kbox * p.stages;
}

__host__ __device__ inline SmemLayout smem_layout(const KParams& p) {
    SmemLayout L;
    const uint32_t a_stage = BM * BK * 2 * p.kbox;
    L.a_off = 0;
    L.b_off = L.a_off + a_stage * p.stages;
    L.c_off = L.b_off + b_region_bytes(p);  // all multiples of 1024
    L.s_off = L.c_off + p.stage_warp_bytes * NUM_EPI_WARPS;
    uint32_t s_bytes = 0;
    if (p.S != nullptr) s_bytes = p.b1 * ((p.b2 + 7) / 8 * 8) * p.BN * 4;  // k rows zero-padded to 8
    L.bar_off = (L.s_off + s_bytes + 15) & ~15u;
    L.tab_off = L.bar_off + 8 * (2 * MAX_STAGES + 6 + MAX_BRES) + 16;
    // tile-blocked A whose K is an odd number of 8-wide panels: a 2-KB zero panel above everything
    // else stands in for the missing half of the last K = 16 step (see the MMA issuer)
    L.zero_off = (L.tab_off + tile_tab_n(p) * 8 + 127) & ~127u;
    L.total = L.zero_off + ((p.a_blocked && (p.a_nchunks & 1)) ? 2048u : 0u);
    return L;
}

// ---------------------------------------------------------------------------- tile schedule ----
// Streaming mode: round-robin tiles, n block fastest (consecutive tiles share the A tile in L2).
// Weight-stationary mode: tiles ordered slice-major (slice = (g, n block)), token tile fastest,
// and each CTA takes one contiguous run, so it reloads B only when its run crosses a slice.
struct TileCoord {
    int m_blk, g, n_blk, slice;
};
__device__ __forceinline__ TileCoord tile_coord(const KParams& p, int tile) {
    TileCoord c;
    if (p.b_resident) {
        c.m_blk = tile % p.tiles_m;
        c.slice = tile / p.tiles_m;
        c.g = c.slice / p.tiles_n;
        c.n_blk = c.slice % p.tiles_n;
    } else {
        c.n_blk = tile % p.tiles_n;
        const int rest = tile / p.tiles_n;
        c.g = rest % p.groups;
        c.m_blk = rest / p.groups;
        c.slice = -1;
    }
    return c;
}
// Tile sequence of this CTA (or CTA pair): tile_at(it) for it = 0, 1, ... until it returns -1.
//  * streaming: round-robin over all tiles (n block fastest).
//  * weight-stationary, #slices <= #units: unit u owns slice u % slices and 1/cps of its token tiles.
//  * weight-stationary, #slices >  #units: unit u takes slices u, u + units, ... each over all token
//    tiles.  Every unit walks token tiles in lockstep, so units sharing an activation tile read it
//    from L2 (the slices of one group are adjacent in the slice order).
struct TileIter {
    int unit, units, slices;
};
__device__ __forceinline__ TileIter tile_iter(const KParams& p, int pair, int vblock, int vgrid) {
    TileIter t;
    const int csz = pair * (p.mc > 1 ? p.mc : 1);  // CTAs per unit (cluster)
    t.unit = vblock / csz;
    t.units = vgrid / csz;
    t.slices = p.groups * p.tiles_n;
    return t;
}
__device__ __forceinline__ int tile_at(const KParams& p, const TileIter& t, int it) {
    if (!p.b_resident) {
        if (p.nb_runs) {  // (token tile, group) pairs round robin, their N blocks back to back
            const long long mg = t.unit + static_cast<long long>(it / p.tiles_n) * t.units;
            const long long tile = mg * p.tiles_n + it % p.tiles_n;
            return tile < p.total_tiles ? static_cast<int>(tile) : -1;
        }
        const long long tile = t.unit + static_cast<long long>(it) * t.units;
        return tile < p.total_tiles ? static_cast<int>(tile) : -1;
    }
    if (p.cps > 0) {  // slice ownership
        const int sl = t.unit % t.slices, part = t.unit / t.slices;
        const int mlo = (part * p.tiles_m) / p.cps, mhi = ((part + 1) * p.tiles_m) / p.cps;
        return mlo + it < mhi ? sl * p.tiles_m + mlo + it : -1;
    }
    const int sl = t.unit + (it / p.tiles_m) * t.units;  // slice round-robin in passes
    return sl < t.slices ? sl * p.tiles_m + it % p.tiles_m : -1;
}
// Number of tiles of this CTA's sequence (tile_at(it) >= 0 exactly for it < tile_count).
__device__ __forceinline__ int tile_count(const KParams& p, const TileIter& t) {
    if (!p.b_resident) {
        if (p.nb_runs) {
            const int mgs = p.total_tiles / p.tiles_n;
            return t.unit < mgs ? (mgs - t.unit + t.units - 1) / t.units * p.tiles_n : 0;
        }
        return t.unit < p.total_tiles ? (p.total_tiles - t.unit + t.units - 1) / t.units : 0;
    }
    if (p.cps > 0) {
        const int part = t.unit / t.slices;
        return ((part + 1) * p.tiles_m) / p.cps - (part * p.tiles_m) / p.cps;
    }
    return t.unit < t.slices ? (t.slices - t.unit + t.units - 1) / t.units * p.tiles_m : 0;
}
__device__ __forceinline__ uint2 tile_pack(const TileCoord& c) {
    return make_uint2(static_cast<uint32_t>(c.m_blk), (static_cast<uint32_t>(c.g) << 16) | static_cast<uint32_t>(c.n_blk));
}
// Coordinates of this CTA's tile `it` (< tile_count): from the table, else computed.
__device__ __forceinline__ TileCoord tile_get(const KParams& p, const TileIter& t, uint32_t tab, int it) {
    if (it < tile_tab_n(p)) {
        const uint2 e = ptx::ld_shared_v2u32(tab + 8u * it);
        TileCoord c;
        c.m_blk = static_cast<int>(e.x);
        c.g = static_cast<int>(e.y >> 16);
        c.n_blk = static_cast<int>(e.y & 0xFFFFu);
        c.slice = p.b_resident ? c.g * p.tiles_n + c.n_blk : -1;
        return c;
    }
    return tile_coord(p, tile_at(p, t, it));
}

// Stage 8 fp32 values (one 16-B chunk `chunk` of row `row`) as bf16 RNE into a row-major staging
// tile whose rows are `row_bytes` long, applying the TMA swizzle (16-B chunk index XOR address
// bits [7, 7+log2(mask+1)) ).  part 1 stages the compensation term lo = bf16(v - bf16(v)).
// OUTF != 0: store IEEE fp16 RNE instead (the BLAST split path's S1 output Z, R13).
template <int OUTF = 0>
__device__ __forceinline__ void stage_row8(uint32_t buf, int row, int chunk, uint32_t row_bytes, uint32_t swz,
                                           const float (&f)[8], int part) {
    uint4 w;
    if constexpr (OUTF != 0) {
        w.x = ptx::pack_f16x2(f[0], f[1]);
        w.y = ptx::pack_f16x2(f[2], f[3]);
        w.z = ptx::pack_f16x2(f[4], f[5]);
        w.w = ptx::pack_f16x2(f[6], f[7]);
    } else {
        w.x = ptx::pack_bf16x2(f[0], f[1]);
        w.y = ptx::pack_bf16x2(f[2], f[3]);
        w.z = ptx::pack_bf16x2(f[4], f[5]);
        w.w = ptx::pack_bf16x2(f[6], f[7]);
    }
    if (part) {
        const uint32_t hw[4] = {w.x, w.y, w.z, w.w};
        float r[8];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            r[2 * e] = f[2 * e] - __uint_as_float(hw[e] << 16);
            r[2 * e + 1] = f[2 * e + 1] - __uint_as_float(hw[e] & 0xFFFF0000u);
        }
        w.x = ptx::pack_bf16x2(r[0], r[1]);
        w.y = ptx::pack_bf16x2(r[2], r[3]);
        w.z = ptx::pack_bf16x2(r[4], r[5]);
        w.w = ptx::pack_bf16x2(r[6], r[7]);
    }
    uint32_t off = row * row_bytes + chunk * 16;
    off ^= ((off >> 7) & swz) << 4;
    ptx::st_shared_v4(buf + off, w);
}

// PAIR == 2: CTA pair (cluster of 2, tcgen05 cta_group::2): tile M = 256 tokens, each CTA loads
// its own 128 A rows and half of B's N columns (per-SM weight ingress halves); the leader CTA
// issues the MMAs; commits are multicast to both CTAs; each CTA drains its own TMEM rows.
// OUTF (GEMM kind only): output 0 = bf16, 1 = fp16, 2 = fp16 tile-blocked [g][T][N/8][128][8],
// 3 = e4m3 tile-blocked [g][T][N/8][128][8] (1-KB panels; the FP8 BLAST intermediate, row f4).
// The kernel body, callable from any kernel whose dynamic smem (1024-B aligned `smem`) holds
// smem_layout(p): blr_gemm_kernel below, and the S1 / S3 roles of the pipelined BLAST layer
// (blast_pipe_kernel), which run it with a virtual block index / grid size.
template <int KIND, int PAIR, int OUTF = 0>
__device__ __forceinline__ void gemm_body(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC,
                                          const CUtensorMap& tmB2, const KParams& p, uint8_t* smem, int vblock, int vgrid) {
    const SmemLayout L = smem_layout(p);
    const uint32_t sbase = ptx::smem_u32(smem);
    const uint32_t a_base = sbase + L.a_off;
    const uint32_t b_base = sbase + L.b_off;
    // S tile (BLAST fused epilogue), addressed through the shared window explicitly: a generic
    // pointer here compiled to generic LD.E loads with global-load latency (3 us per 8 columns)
    const uint32_t s_tile = sbase + L.s_off;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + L.bar_off);
    const uint32_t full_bar = ptx::smem_u32(bars);
    const uint32_t empty_bar = full_bar + 8 * MAX_STAGES;
    const uint32_t tfull_bar = empty_bar + 8 * MAX_STAGES;
    const uint32_t tempty_bar = tfull_bar + 16;
    const uint32_t bfree_bar = tempty_bar + 16;   // MMAs done reading the resident B
    const uint32_t bfull_bar = bfree_bar + 16;    // [MAX_BRES]: resident B k-block kb landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + L.bar_off + 8 * (2 * MAX_STAGES + 6 + MAX_BRES));

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    // rank within the pair (crank), pair index within a B-multicast cluster (pidx), its leader's rank
    const uint32_t cl_rank = PAIR == 2 ? ptx::cluster_ctarank() : 0u;
    const uint32_t crank = cl_rank & 1u;
    const uint32_t pidx = cl_rank >> 1;
    const int mcs = (PAIR == 2 && p.mc > 1) ? p.mc : 1;
    const uint32_t lead_rank = cl_rank & ~1u;
    const bool leader = crank == 0;
#ifdef BLR_DEBUG_KNOBS
    unsigned long long* trace = p.trace ? p.trace + vblock * 128 : nullptr;
#else
    unsigned long long* const trace = nullptr;  // per-CTA timeline stamps: debug builds only
#endif
    // trace stamps: [0] %globaltimer at entry, [8] %clock64 at entry; every other stamp is a
    // %clock64 value (cheap; converted on the host with the SM clock)
    if (trace && threadIdx.x == 0) {
        trace[0] = ptx::globaltimer();
        trace[8] = clock64();
    }

    if (warp == 0) {
        // the lanes of warp 0 initialise the barriers this plan uses in parallel (a single thread
        // initialising all of them sat on the critical path of every kernel boundary, ~1 us)
        const int nres = p.b_resident ? kb_resident(p) : 0;
        for (int s = lane; s < p.stages; s += 32) {
            ptx::mbar_init(full_bar + 8 * s, 1);
            ptx::mbar_init(empty_bar + 8 * s, mcs);  // multicast: every pair leader frees the slot
        }
        if (lane < 2) {
            ptx::mbar_init(tfull_bar + 8 * lane, 1);
            ptx::mbar_init(tempty_bar + 8 * lane, NUM_EPI_WARPS * PAIR);  // leader's: both CTAs drain
        }
        for (int kb = lane; kb < nres; kb += 32) ptx::mbar_init(bfull_bar + 8 * kb, 1);
        if (lane == 0) ptx::mbar_init(bfree_bar, 1);
        ptx::fence_barrier_init();
        if (lane == 0) {
            ptx::prefetch_tmap(&tmA);
            ptx::prefetch_tmap(&tmB);
            ptx::prefetch_tmap(&tmC);
            if (trace && KIND != KIND_BLAST_PROJ) trace[13] = clock64();
        }
    }
    if (warp == 1) {
        if constexpr (PAIR == 2) ptx::tmem_alloc_pair<TMEM_COLS>(ptx::smem_u32(tmem_slot));
        else ptx::tmem_alloc<TMEM_COLS>(ptx::smem_u32(tmem_slot));
        if (trace && lane == 0 && KIND != KIND_BLAST_PROJ) trace[14] = clock64();
    }
    const TileIter titer = tile_iter(p, PAIR, vblock, vgrid);
    const int ntiles = tile_count(p, titer);
    const uint32_t tile_tab = sbase + L.tab_off;  // explicit shared-window addressing (see s_tile)
    for (int e = threadIdx.x; e < ntiles && e < tile_tab_n(p); e += NUM_THREADS)
        ptx::st_shared_v2u32(tile_tab + 8u * e, tile_pack(tile_coord(p, tile_at(p, titer, e))));
    if (p.a_blocked && (p.a_nchunks & 1)) {  // the zero panel (generic stores -> async proxy)
        for (uint32_t o = threadIdx.x * 16u; o < 2048u; o += NUM_THREADS * 16u)
            ptx::st_shared_v4(sbase + L.zero_off + o, make_uint4(0, 0, 0, 0));
        ptx::fence_async_smem();
    }
    if (trace && threadIdx.x == 64 && KIND != KIND_BLAST_PROJ) trace[15] = clock64();
    ptx::tc_fence_before();
    __syncthreads();
    if constexpr (PAIR == 2) ptx::cluster_sync();  // peer barriers initialised before any remote use
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t acc_stride = static_cast<uint32_t>(p.n_sub * p.BN);  // columns per buffer
    if (trace && threadIdx.x == 0) trace[1] = clock64();
    // Programmatic dependent launch: everything above overlapped the previous kernel's tail.
    // Roles that read the previous kernel's output (producer: A) or write outputs it may still
    // read (epilogue) call griddep_wait() first.  Weights are never written by this library, so
    // a later launch of the same API call prefetches its resident weight slice before waiting.
    // The FIRST launch of a call (p.first) may follow a caller kernel that wrote the weights: it
    // waits before loading anything and lets the next grid start only after that wait, so by the
    // time any later launch of the call starts, all work enqueued before the call has completed.
    if (!p.first && !p.no_trigger) ptx::griddep_launch_dependents();

    if (warp == 0) {
        // ===================================================== TMA producer =================
        // The whole warp runs the (warp-uniform) schedule so that the compiler keeps coordinates
        // and addresses in uniform registers; one elected lane issues each TMA.  (A lone-lane
        // loop forces per-instruction ELECT/broadcast sequences and measured ~3x slower.)
        {
            const uint32_t a_blk = BM * BK * 2;  // one 64-wide K block of A (16 KB)
            // per-CTA bytes; a pair's leader expects both CTAs' bytes on its barrier
            const uint32_t b_bytes = p.b_mn_major ? p.n_mma * p.b_boxes * p.b_box_n * BK * 2
                                                  : static_cast<uint32_t>(p.BN / PAIR) * BK * 2;
            const uint32_t tx = p.kbox * (a_blk + (p.b_resident ? 0u : b_bytes)) * PAIR;
            const int a_nch = p.a_nchunks;  // a_blocked: K / 8 panels per group

            auto load3 = [&](uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1, int c2) {
                if constexpr (PAIR == 2) ptx::tma_load_3d_pair(dst, m, bar, c0, c1, c2);
                else ptx::tma_load_3d(dst, m, bar, c0, c1, c2);
            };
            auto load4 = [&](uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1, int c2, int c3) {
                if constexpr (PAIR == 2) ptx::tma_load_4d_pair(dst, m, bar, c0, c1, c2, c3);
                else ptx::tma_load_4d(dst, m, bar, c0, c1, c2, c3);
            };
            const int n_steps = (p.k_blocks + p.kbox - 1) / p.kbox;
            const int kbr = BLR_DBG_ON(p, 64) ? 0 : kb_resident(p);  // dbg 64: no weight loads
            if (p.first) {
                ptx::griddep_wait();
                if (!p.no_trigger) ptx::griddep_launch_dependents();
            }
            int stage = 0;
            uint32_t phase = 0;
            int cur_slice = -1;
            uint32_t nslices = 0;
            bool waited = p.first != 0;
            int nstep_tr = 0;
            int pipe_ok = -1;  // highest token tile of A known ready (pipelined layer)
            int bp_ok = -1;    // highest token tile cleared by back-pressure
            bool fast_done = false;
            {
                if (!kGenericProducer || (trace == nullptr && p.fast_prod)) {
                    // Lean producer for the GEMM kind: every parameter the K loop needs is hoisted
                    // into registers and every per-tile coordinate computed once per tile, so a K
                    // block costs a barrier wait, an expect_tx and its TMA issues.  (The generic loop
                    // below re-read kernel parameters after every asm statement and divided per K
                    // block: ~130 instructions at ~12 cycles each, 1.6k cycles per 480-cycle K block
                    // of MMA work -- the producer, not the tensor pipe, bounded C4 gate S3, ncu.)
                    fast_done = true;
                    const int kbox = ptx::pin(p.kbox), stages = ptx::pin(p.stages), kb_half = ptx::pin(p.kb_half);
                    const int a_lo_off = ptx::pin(p.a_lo_off);
                    const bool a_blk_mode = p.a_blocked != 0, a_gmid = p.a_gmid != 0;
                    const bool b_res = p.b_resident != 0, b_mn = p.b_mn_major != 0;
                    const int n_mma = ptx::pin(p.n_mma), b_boxes = ptx::pin(p.b_boxes), b_box_n = ptx::pin(p.b_box_n);
                    const int BNf = p.BN;
                    const int bn_h = ptx::pin(BNf / n_mma);     // columns per MMA half
                    const int bn_cta = bn_h / PAIR;             // this CTA's columns of a half
                    const uint32_t b_stage_b = ptx::pin(p.b_stage_bytes), b_half_b = ptx::pin(p.b_half_bytes);
                    const uint32_t box_b = static_cast<uint32_t>(b_box_n) * BK * 2;
                    const int a_tiles = p.a_tiles;
                    const bool slab2 = p.b_slab2 != 0;
                    const int nslab = p.b_nslab;
                    const int ns = ptx::pin(n_steps);
                    const uint32_t tx_f = ptx::pin(tx);
                    const uint32_t tx_lh = ptx::pin(p.kbox * (a_blk + b_bytes / 2) * PAIR);  // single-half last tile
                    const bool last_half = p.last_half != 0;
                    const int hint_a = p.l2_a, hint_b = p.l2_b;
                    const uint64_t pol_a = ptx::l2_policy(hint_a), pol_b = ptx::l2_policy(hint_b);
                    auto load3h = [&](uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1, int c2, int hint,
                                      uint64_t pol) {
                        if (hint == 0) {
                            load3(dst, m, bar, c0, c1, c2);
                        } else {
                            if constexpr (PAIR == 2) ptx::tma_load_3d_pair_hint(dst, m, bar, c0, c1, c2, pol);
                            else ptx::tma_load_3d_hint(dst, m, bar, c0, c1, c2, pol);
                        }
                    };
                    auto load4h = [&](uint32_t dst, const CUtensorMap* m, uint32_t bar, int c0, int c1, int c2, int c3,
                                      int hint, uint64_t pol) {
                        if (hint == 0) {
                            load4(dst, m, bar, c0, c1, c2, c3);
                        } else {
                            if constexpr (PAIR == 2) ptx::tma_load_4d_pair_hint(dst, m, bar, c0, c1, c2, c3, pol);
                            else ptx::tma_load_4d_hint(dst, m, bar, c0, c1, c2, c3, pol);
                        }
                    };
                    // B multicast across the mcs CTA pairs of a cluster (mcs > 1): this pair loads 1/mcs
                    // of every B box (K rows for MN-major, N rows for K-major) for all of them
                    uint16_t mc_mask = 0;
                    for (int j2 = 0; j2 < mcs; ++j2) mc_mask |= static_cast<uint16_t>(1u << (2 * j2 + crank));
                    const int mc_kr = BK / mcs;                              // MN-major: K rows per slice
                    const int mc_nr = ptx::pin(BNf / n_mma / PAIR / mcs);    // K-major: N rows per slice
                    const int last_nb = ptx::pin(p.last_nb), last_blk = ptx::pin(p.tiles_n - 1);
                    for (int it = 0; it < ntiles; ++it) {
                        const TileCoord tc = tile_get(p, titer, tile_tab, it);
                        const int t128 = (tc.m_blk * mcs + static_cast<int>(pidx)) * PAIR + static_cast<int>(crank);
                        const int m0 = t128 * BM;
                        // Monarch: first output block k of this CTA's share of the tile's k blocks
                        const int kblk0 = tc.n_blk * p.kb_per_tile + static_cast<int>(crank) * (p.kb_per_tile / PAIR);
                        if (b_res && tc.slice != cur_slice) {
                            if (nslices > 0) ptx::mbar_wait(bfree_bar, (nslices - 1) & 1);
                            if (ptx::elect_one()) {
                                const int n0 = tc.n_blk * BNf + static_cast<int>(crank) * (BNf / PAIR);
                                for (int kb = 0; kb < kbr; ++kb) {
                                    const uint32_t b_dst = b_base + kb * b_stage_b;
                                    const uint32_t bb = bfull_bar + 8 * kb;
                                    if (leader) ptx::mbar_arrive_expect_tx(bb, b_bytes * PAIR);
                                    if constexpr (KIND == KIND_MONARCH_PROJ) {
                                        load4(b_dst, &tmB, bb, kb * BK, 0, kblk0, tc.g);
                                    } else if (b_mn) {
                                        for (int j = 0; j < b_boxes; ++j)
                                            load3(b_dst + j * box_b, &tmB, bb, n0 + j * b_box_n, kb * BK, tc.g);
                                    } else {
                                        load3(b_dst, &tmB, bb, kb * BK, n0, tc.g);
                                    }
                                }
                            }
                            __syncwarp();
                            cur_slice = tc.slice;
                            ++nslices;
                        }
                        if (!waited) {
                            ptx::griddep_wait();
                            waited = true;
                        }
                        if (p.pipe_bp != nullptr && t128 >= p.pipe_bp_dist && t128 > bp_ok) {
                            // keep this stage at most pipe_bp_dist token tiles ahead of its consumer,
                            // so what it hands over is still in L2 when the consumer reads it
                            ptx::pipe_acquire(p.pipe_bp + (t128 - p.pipe_bp_dist), p.pipe_bp_target);
                            bp_ok = t128;
                        }
                        if (p.pipe_wait != nullptr && t128 > pipe_ok && t128 < a_tiles) {
                            ptx::pipe_acquire(p.pipe_wait + t128, p.pipe_target);  // A's token tile is ready
                            pipe_ok = t128;
                        }
                        const int a_row0 = (tc.g * a_tiles + t128) * a_nch * 16;  // tile-blocked A
                        const int a_c1 = a_gmid ? tc.g : m0, a_c2 = a_gmid ? m0 : tc.g;
                        const int nb0 = tc.n_blk * BNf + static_cast<int>(crank) *
                                        ((last_nb > 0 && tc.n_blk == last_blk) ? last_nb / PAIR : bn_cta);  // half 0, this CTA
                        const bool lh = last_half && tc.n_blk == last_blk;  // half 0 only
                        const int n_mma_t = lh ? 1 : n_mma;
                        const int n_sub = KIND == KIND_BLAST_PROJ ? p.n_sub : 1;  // BLAST proj: the b1 sub-GEMMs l
                        for (int sub = 0; sub < n_sub; ++sub)
                        for (int si = 0; si < ns; ++si) {
                            ptx::mbar_wait(empty_bar + 8 * stage, phase ^ 1);
                            const uint32_t fb = full_bar + 8 * stage;
                            const uint32_t a_st = a_base + stage * (a_blk * kbox);
                            const uint32_t b_st = b_base + stage * (b_stage_b * kbox);
                            if (ptx::elect_one()) {
                                if (leader) ptx::mbar_arrive_expect_tx(fb, lh ? tx_lh : tx_f);
                                for (int j = 0; j < kbox; ++j) {
                                    const int kb = si * kbox + j;
                                    const int part = (a_lo_off > 0 && kb >= kb_half) ? 1 : 0;
                                    const int k0 = (kb - part * kb_half) * BK;  // padded block: zero-filled
                                    const uint32_t a_dst = a_st + j * a_blk;
                                    if constexpr (KIND == KIND_MONARCH_PROJ) {
                                        // A = X viewed [n_tok][b1][p]; B = V viewed 4-D (a, rho', k, l): the
                                        // permutations of PAPER.md L194 are this box's coordinates (§5.2)
                                        load3(a_dst, &tmA, fb, k0, tc.g, m0);
                                        if (!b_res) load4(b_st + j * b_stage_b, &tmB, fb, k0, 0, kblk0, tc.g);
                                        continue;
                                    }
                                    if constexpr (KIND == KIND_BLAST_PROJ) {  // sub = l: X_l and V_l
                                        ptx::tma_load_3d(a_dst, &tmA, fb, k0, sub, m0);
                                        const uint32_t b_dst = b_st + j * b_stage_b;
                                        for (int q = 0; q < b_boxes; ++q)
                                            ptx::tma_load_3d(b_dst + q * box_b, &tmB, fb, nb0 + q * b_box_n, k0, sub);
                                        continue;
                                    }
                                    if (a_blk_mode) load3h(a_dst, &tmA, fb, 0, a_row0 + kb * 128, 0, hint_a, pol_a);
                                    else load3h(a_dst, &tmA, fb, part * a_lo_off + k0, a_c1, a_c2, hint_a, pol_a);
                                    if (!b_res) {
                                        const uint32_t b_dst = b_st + j * b_stage_b;
                                        for (int h = 0; h < n_mma_t; ++h) {
                                            const int nh = nb0 + h * bn_h;
                                            const uint32_t bh = b_dst + h * b_half_b;
                                            if constexpr (PAIR == 2) {
                                                if (mcs > 1) {
                                                    if (b_mn) {
                                                        for (int q = 0; q < b_boxes; ++q)
                                                            ptx::tma_load_3d_pair_mc(bh + q * box_b + pidx * mc_kr * (b_box_n * 2), &tmB, fb,
                                                                                     nh + q * b_box_n, k0 + static_cast<int>(pidx) * mc_kr,
                                                                                     tc.g, mc_mask);
                                                    } else {
                                                        ptx::tma_load_3d_pair_mc(bh + pidx * mc_nr * 128, &tmB, fb, k0,
                                                                                 nh + static_cast<int>(pidx) * mc_nr, tc.g, mc_mask);
                                                    }
                                                    continue;
                                                }
                                            }
                                            if (b_mn) {
                                                if (slab2 && (nh & 63) == 0 && (nh >> 6) + 2 <= nslab) {
                                                    // both 64-column boxes as one op: slab view (64, K, slab, g)
                                                    load4h(bh, &tmB2, fb, 0, k0, nh >> 6, tc.g, hint_b, pol_b);
                                                } else {
                                                    for (int q = 0; q < b_boxes; ++q)
                                                        load3h(bh + q * box_b, &tmB, fb, nh + q * b_box_n, k0, tc.g, hint_b, pol_b);
                                                }
                                            } else {
                                                load3h(bh, &tmB, fb, k0, nh, tc.g, hint_b, pol_b);
                                            }
                                        }
                                    }
                                }
                            }
                            __syncwarp();
                            if (++stage == stages) { stage = 0; phase ^= 1; }
                        }
                    }
                }
            }
#ifdef BLR_DEBUG_KNOBS  // the generic producer loop (BLR_FASTPROD=0, per-step trace stamps): debug builds only
            for (int it = 0; !fast_done && it < ntiles; ++it) {
                const TileCoord tc = tile_get(p, titer, tile_tab, it);
                const int m0 = ((tc.m_blk * mcs + static_cast<int>(pidx)) * PAIR + static_cast<int>(crank)) * BM;
                const int n0 = tc.n_blk * p.BN + static_cast<int>(crank) * (p.BN / PAIR);  // this CTA's B half
                // Monarch: first output block k of this CTA's share of the tile's k blocks
                const int kblk0 = tc.n_blk * p.kb_per_tile + static_cast<int>(crank) * (p.kb_per_tile / PAIR);
                if (p.b_resident && tc.slice != cur_slice) {
                    // (re)load the weight slice once for the contiguous run of token tiles
                    if (nslices > 0) ptx::mbar_wait(bfree_bar, (nslices - 1) & 1);
                    if (ptx::elect_one()) {
                        for (int kb = 0; kb < kbr; ++kb) {
                            const uint32_t b_dst = b_base + kb * p.b_stage_bytes;
                            const uint32_t bb = bfull_bar + 8 * kb;  // per-block barrier: MMA starts early
                            if (leader) ptx::mbar_arrive_expect_tx(bb, b_bytes * PAIR);
                            const int k0 = kb * BK;
                            if constexpr (KIND == KIND_MONARCH_PROJ) {
                                load4(b_dst, &tmB, bb, k0, 0, kblk0, tc.g);
                            } else if (p.b_mn_major) {
                                for (int j = 0; j < p.b_boxes; ++j)
                                    load3(b_dst + j * (p.b_box_n * BK * 2), &tmB, bb, n0 + j * p.b_box_n, k0, tc.g);
                            } else {
                                load3(b_dst, &tmB, bb, k0, n0, tc.g);
                            }
                        }
                    }
                    __syncwarp();
                    cur_slice = tc.slice;
                    ++nslices;
                }
                if (!waited) {
                    ptx::griddep_wait();  // A (activations / intermediate) comes from the previous kernel
                    waited = true;
                    if (trace && lane == 0) trace[2] = clock64();
                }
                for (int sub = 0; sub < p.n_sub; ++sub) {
                    for (int si = 0; si < n_steps; ++si) {
                        ptx::mbar_wait(empty_bar + 8 * stage, phase ^ 1);
                        const uint32_t fb = full_bar + 8 * stage;
                        const uint32_t a_st = a_base + stage * (a_blk * p.kbox);
                        const uint32_t b_st = b_base + stage * (p.b_stage_bytes * p.kbox);
                        if (ptx::elect_one()) {
                            const bool lh_g = p.last_half && tc.n_blk == p.tiles_n - 1;  // single-half last tile
                            if (leader)
                                ptx::mbar_arrive_expect_tx(fb, lh_g ? p.kbox * (a_blk + b_bytes / 2) * PAIR : tx);  // (tile-blocked A: always full tiles)
                            if (trace && nstep_tr < 32) trace[64 + nstep_tr] = clock64();
                            for (int j = 0; j < p.kbox; ++j) {
                                const int kb = si * p.kbox + j;
                                const uint32_t a_dst = a_st + j * a_blk;
                                const uint32_t b_dst = b_st + j * p.b_stage_bytes;
                                // compensated A: blocks >= kb_half read the lo half against the same B rows
                                const int part = (p.a_lo_off > 0 && kb >= p.kb_half) ? 1 : 0;
                                const int k0 = (kb - part * p.kb_half) * BK;  // padded block: k0 >= K, zero-filled
                                if constexpr (KIND == KIND_GEMM) {
                                    if (p.a_blocked) {
                                        // tile-blocked A [g][T][K/8][128][8]: the K block's 8 panels of
                                        // this CTA's 128-row tile are 128 consecutive 128-B rows of
                                        // the map (panels past K read the following panels or TMA's
                                        // zero fill: finite values against B's zero-filled rows)
                                        const int t128 = (tc.m_blk * mcs + static_cast<int>(pidx)) * PAIR + static_cast<int>(crank);
                                        const int row = ((tc.g * p.a_tiles + t128) * a_nch + (k0 >> 3)) * 16;
                                        load3(a_dst, &tmA, fb, 0, row, 0);
                                    } else if (p.a_gmid)
                                        load3(a_dst, &tmA, fb, part * p.a_lo_off + k0, tc.g, m0);
                                    else
                                        load3(a_dst, &tmA, fb, part * p.a_lo_off + k0, m0, tc.g);
                                    if (!p.b_resident) {
                                        for (int h = 0; h < (lh_g ? 1 : p.n_mma); ++h) {
                                            // this CTA's share of half h: columns n0h .. of the tile
                                            const int share = (p.last_nb > 0 && tc.n_blk == p.tiles_n - 1)
                                                                  ? p.last_nb / PAIR : p.BN / p.n_mma / PAIR;
                                            const int n0h = tc.n_blk * p.BN + h * (p.BN / p.n_mma) +
                                                            static_cast<int>(crank) * share;
                                            const uint32_t bh = b_dst + h * p.b_half_bytes;
                                            if constexpr (PAIR == 2) {
                                                if (mcs > 1) {
                                                    // this pair's slice of every B box, multicast to the
                                                    // same-rank CTA of every pair of the cluster
                                                    uint16_t mask = 0;
                                                    for (int j2 = 0; j2 < mcs; ++j2) mask |= static_cast<uint16_t>(1u << (2 * j2 + crank));
                                                    if (p.b_mn_major) {
                                                        const int kr = BK / mcs;  // K rows per slice
                                                        for (int q = 0; q < p.b_boxes; ++q)
                                                            ptx::tma_load_3d_pair_mc(bh + q * (p.b_box_n * BK * 2) + pidx * kr * (p.b_box_n * 2),
                                                                                     &tmB, fb, n0h + q * p.b_box_n, k0 + pidx * kr, tc.g, mask);
                                                    } else {
                                                        const int nr = p.BN / p.n_mma / PAIR / mcs;  // N rows per slice
                                                        ptx::tma_load_3d_pair_mc(bh + pidx * nr * 128, &tmB, fb, k0, n0h + pidx * nr, tc.g, mask);
                                                    }
                                                    continue;
                                                }
                                            }
                                            if (p.b_mn_major) {
                                                for (int q = 0; q < p.b_boxes; ++q)
                                                    load3(bh + q * (p.b_box_n * BK * 2), &tmB, fb, n0h + q * p.b_box_n, k0,
                                                          tc.g);
                                            } else {
                                                load3(bh, &tmB, fb, k0, n0h, tc.g);
                                            }
                                        }
                                    }
                                } else if constexpr (KIND == KIND_MONARCH_PROJ) {
                                    // A = X viewed [n_tok][b1][p]; B = V viewed 4-D (a, rho', k, l)
                                    load3(a_dst, &tmA, fb, k0, tc.g, m0);
                                    if (!p.b_resident) load4(b_dst, &tmB, fb, k0, 0, kblk0, tc.g);
                                } else {  // KIND_BLAST_PROJ: sub = l
                                    ptx::tma_load_3d(a_dst, &tmA, fb, k0, sub, m0);
                                    for (int q = 0; q < p.b_boxes; ++q)
                                        ptx::tma_load_3d(b_dst + q * (p.b_box_n * BK * 2), &tmB, fb,
                                                         n0 + q * p.b_box_n, k0, sub);
                                }
                            }
                        }
                        __syncwarp();
                        ++nstep_tr;
                        if (++stage == p.stages) { stage = 0; phase ^= 1; }
                    }
                }
            }
#endif
        }
    } else if (warp == 1) {
        // ===================================================== MMA issuer ===================
        // Warp-wide schedule (uniform registers); one elected lane issues the MMAs and commits.
        if (leader) {
            const uint32_t idesc = ptx::idesc_bf16(BM * PAIR, p.BN / p.n_mma, p.b_mn_major);
            const uint32_t idesc_last = p.last_nb > 0 ? ptx::idesc_bf16(BM * PAIR, p.last_nb, p.b_mn_major) : idesc;
            const uint16_t pair_mask = static_cast<uint16_t>(3u << (2 * pidx));
            const uint16_t all_mask = mcs > 1 ? static_cast<uint16_t>((1u << (2 * mcs)) - 1u) : pair_mask;
            auto commit = [&](uint32_t bar) {  // own pair (accumulator / resident-B hand-offs)
                if constexpr (PAIR == 2) ptx::mma_commit_pair_mask(bar, pair_mask);
                else ptx::mma_commit(bar);
            };
            auto commit_slot = [&](uint32_t bar) {  // a ring slot: every CTA whose loads land in it
                if constexpr (PAIR == 2) ptx::mma_commit_pair_mask(bar, all_mask);
                else ptx::mma_commit(bar);
            };
            // descriptors are built once; per-MMA only the 14-bit start-address field advances
            // (a 32-bit add on the low word: the field never carries out)
            // A: K-major 128-B swizzle (8-row groups 1024 B apart, +32 B per K=16), or for a
            // tile-blocked A the no-swizzle core-matrix layout [c][t][8] (LBO = BM*16 B between
            // K core matrices, SBO = 128 B between 8-row groups, +2 core matrices per K=16)
            const uint64_t a_desc0 = p.a_blocked ? ptx::smem_desc(a_base, BM * 16, 128, 0)
                                                 : ptx::smem_desc(a_base, 16, 1024, ptx::LAYOUT_SW128);
            const uint32_t a_kstep = p.a_blocked ? 2 * BM * 16 : 32;
            const uint64_t b_desc0 = ptx::smem_desc(b_base, p.b_lbo, p.b_sbo, p.b_layout);
            const uint32_t a_lo0 = static_cast<uint32_t>(a_desc0), a_hi = static_cast<uint32_t>(a_desc0 >> 32);
            const uint32_t b_lo0 = static_cast<uint32_t>(b_desc0), b_hi = static_cast<uint32_t>(b_desc0 >> 32);
            const uint32_t a_blk = BM * BK * 2;
            const int n_steps = (p.k_blocks + p.kbox - 1) / p.kbox;
            const int kbr = kb_resident(p);
            const bool wait_b = p.b_resident && !BLR_DBG_ON(p, 64);
            // loop-invariant parameters, hoisted (the asm memory clobbers would otherwise make the
            // compiler re-read them from the parameter bank every step)
            const int kbox_h = p.kbox, kb_half_h = p.kb_half, a_lo_off_h = p.a_lo_off;
            const bool b_res_h = p.b_resident != 0, two_h = p.n_mma == 2;
            const uint32_t b_stage_h = p.b_stage_bytes;
            const uint32_t a_ks = a_kstep >> 4, b_ks = p.b_kstep >> 4, b_hh = p.b_half_bytes >> 4;
            const uint32_t d_half = static_cast<uint32_t>(p.BN / 2);
            const bool split_h = KIND == KIND_GEMM && PAIR == 2 && p.split_rel != 0;  // (wide plans are pair plans)
            // K blocks issued as one unrolled burst of four K = 16 MMAs (all 8 panels valid).  Streamed
            // pair plans keep the per-step loop: the burst measured ~5% slower there at full size
            // (C4 gate S3 2.49 -> 2.62 ms, down S1 2.35 -> 2.49 ms, same box), while it speeds up
            // the weight-resident and Monarch-projection plans (C4 gate S1 1.6 -> 1.44 ms)
            const int full_kb = !p.mma_burst ? -1 : p.a_blocked ? (p.a_nchunks >> 3) : 0x7fffffff;
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            int cur_slice = -1;
            uint32_t nslices = 0;
            int mstep_tr = 0;
            for (int it = 0; it < ntiles; ++it) {
                const TileCoord tc = tile_get(p, titer, tile_tab, it);
                const uint32_t idesc_t = (p.last_nb > 0 && tc.n_blk == p.tiles_n - 1) ? idesc_last : idesc;
                bool fresh = false;  // first tile of a new resident slice: wait per B block
                if (p.b_resident && tc.slice != cur_slice) {
                    cur_slice = tc.slice;
                    ++nslices;
                    fresh = true;
                }
                if (!BLR_DBG_ON(p, 32)) ptx::mbar_wait(tempty_bar + 8 * acc, acc_phase ^ 1);
                ptx::tc_fence_after();
                if (split_h) {
                    // wide tile, one accumulator, per-half release (KParams::split_rel): column half 0
                    // is free (waited above).  Until the epilogue frees half 1, each K block issues
                    // only its half-0 MMAs and keeps its ring slot; once half 1 is free the held
                    // blocks' half-1 MMAs are issued in order and their slots released.  At most
                    // stages - 1 slots are held, so the producer always has one to fill.
                    // (a single-half last tile, KParams::last_half: half 0 alone, last_nb columns wide)
                    const bool lh = p.last_half && tc.n_blk == p.tiles_n - 1;
                    const uint32_t idesc_h = lh ? idesc_last : idesc;
                    bool h1 = lh;
                    int npend = 0, pst = 0, psi = 0;
                    auto issue = [&](int st, int si, int h) {  // elected lane: one 64-K block of half h
                        const uint32_t a_off = static_cast<uint32_t>(st) * a_blk;
                        const uint32_t a_lo = a_lo0 + (a_off >> 4);
                        const uint32_t b_lo = b_lo0 + ((static_cast<uint32_t>(st) * b_stage_h) >> 4) + (h ? b_hh : 0u);
                        const uint32_t d = tmem_base + (h ? d_half : 0u);
                        // tile-blocked A: only the K = 16 steps over valid panels, a half-valid last
                        // step takes its second core matrix from the zero panel (as in the loop below)
                        int n16 = BK / UMMA_K;
                        bool half_last = false;
                        if (p.a_blocked && si >= full_kb) {
                            const int vp = min(8, max(0, p.a_nchunks - si * 8));
                            n16 = (vp + 1) >> 1;
                            half_last = (vp & 1) != 0;
                        }
#pragma unroll
                        for (int kk = 0; kk < BK / UMMA_K; ++kk) {
                            if (kk >= n16) break;
                            uint64_t ad = ptx::desc_make(a_lo + kk * a_ks, a_hi);
                            if (half_last && kk == n16 - 1) {
                                const uint32_t pa = a_base + a_off + kk * a_kstep;
                                ad = ptx::smem_desc(pa, sbase + L.zero_off - pa, 128, 0);
                            }
                            const uint64_t bd = ptx::desc_make(b_lo + kk * b_ks, b_hi);
                            const uint32_t acc1 = (si | kk) != 0 ? 1u : 0u;
                            if constexpr (PAIR == 2) ptx::mma_bf16_pair(d, ad, bd, idesc_h, acc1);
                            else ptx::mma_bf16(d, ad, bd, idesc_h, acc1);
                        }
                    };
                    auto catch_up = [&]() {
                        ptx::tc_fence_after();
                        if (ptx::elect_one()) {
                            int st = pst;
                            for (int q = 0; q < npend; ++q) {
                                issue(st, psi + q, 1);
                                commit_slot(empty_bar + 8 * st);
                                if (++st == p.stages) st = 0;
                            }
                        }
                        __syncwarp();
                        npend = 0;
                        h1 = true;
                    };
                    const int max_pend = p.stages - 1;
                    for (int si = 0; si < n_steps; ++si) {
                        if (!h1 && npend >= max_pend) {
                            ptx::mbar_wait(tempty_bar + 8, acc_phase ^ 1);
                            catch_up();
                        }
                        ptx::mbar_wait(full_bar + 8 * stage, phase);
                        if (!h1) {
                            uint32_t ok = ptx::mbar_test_wait(tempty_bar + 8, acc_phase ^ 1) ? 1u : 0u;
                            ok = __shfl_sync(0xffffffffu, ok, 0);
                            if (ok) catch_up();
                        }
                        ptx::tc_fence_after();
                        if (ptx::elect_one()) {
                            issue(stage, si, 0);
                            if (h1) {
                                if (!lh) issue(stage, si, 1);
                                commit_slot(empty_bar + 8 * stage);
                            }
                        }
                        __syncwarp();
                        if (!h1) {
                            if (npend == 0) {
                                pst = stage;
                                psi = si;
                            }
                            ++npend;
                        }
                        ++mstep_tr;
                        if (++stage == p.stages) { stage = 0; phase ^= 1; }
                    }
                    if (!h1) {
                        ptx::mbar_wait(tempty_bar + 8, acc_phase ^ 1);
                        catch_up();
                    }
                } else
                for (int sub = 0; sub < p.n_sub; ++sub) {
                    const uint32_t d_tmem = tmem_base + acc * acc_stride + sub * p.BN;
                    for (int si = 0; si < n_steps; ++si) {
                        ptx::mbar_wait(full_bar + 8 * stage, phase);
                        if (fresh && wait_b) {  // this step's resident B blocks have landed
                            for (int j = 0; j < p.kbox; ++j) {
                                const int kb = si * p.kbox + j;
                                const int bkb = (p.a_lo_off > 0 && kb >= p.kb_half) ? kb - p.kb_half : kb;
                                if (kb < kbr) ptx::mbar_wait(bfull_bar + 8 * bkb, (nslices - 1) & 1);
                            }
                        }
                        ptx::tc_fence_after();
                        // Descriptors of this step are formed warp-wide (uniform registers, params
                        // hoisted out of the loop): the MMA issue is a short dependency-free burst
                        // (per-step issue overhead directly stalls the tensor pipe)
                        const uint32_t a_st = static_cast<uint32_t>(stage) * (a_blk * kbox_h);
                        const uint32_t b_st = static_cast<uint32_t>(stage) * (b_stage_h * kbox_h);
                        if (ptx::elect_one()) {
                            if (trace) {
                                if (mstep_tr == 0) trace[3] = clock64();
                                if (mstep_tr < 32) trace[96 + mstep_tr] = clock64();
                            }
                            for (int j = 0; j < kbox_h; ++j) {
                                const int kb = si * kbox_h + j;
                                const int bkb = (a_lo_off_h > 0 && kb >= kb_half_h) ? kb - kb_half_h : kb;
                                const uint32_t a_off = a_st + j * a_blk;
                                const uint32_t b_off = b_res_h ? bkb * b_stage_h : b_st + j * b_stage_h;
                                const uint32_t a_lo = a_lo0 + (a_off >> 4), b_lo = b_lo0 + (b_off >> 4);
                                const uint32_t accf = (si | j) != 0 ? 1u : 0u;
                                if (kb < full_kb) {  // fast path: all four K = 16 steps
#pragma unroll
                                    for (int kk = 0; kk < BK / UMMA_K; ++kk) {
                                        const uint64_t ad = ptx::desc_make(a_lo + kk * a_ks, a_hi);
                                        const uint64_t bd = ptx::desc_make(b_lo + kk * b_ks, b_hi);
                                        const uint32_t acc1 = accf | (kk != 0 ? 1u : 0u);
                                        if (BLR_DBG_ON(p, 8)) continue;  // debug: skip the MMA itself
                                        if constexpr (PAIR == 2) ptx::mma_bf16_pair(d_tmem, ad, bd, idesc_t, acc1);
                                        else ptx::mma_bf16(d_tmem, ad, bd, idesc_t, acc1);
                                        if (two_h) {  // second half: same A, B half 1, next TMEM columns
                                            const uint64_t bd2 = ptx::desc_make(b_lo + b_hh + kk * b_ks, b_hi);
                                            if constexpr (PAIR == 2) ptx::mma_bf16_pair(d_tmem + d_half, ad, bd2, idesc, acc1);
                                            else ptx::mma_bf16(d_tmem + d_half, ad, bd2, idesc, acc1);
                                        }
                                    }
                                    continue;
                                }
                                // tile-blocked A: the box of a K block that runs past K also holds the
                                // NEXT token tile's panels; only the K = 16 steps over valid panels
                                // are issued (a half-valid last step takes its second core matrix
                                // from the zero panel), so no other token's value -- NaN or Inf
                                // included -- enters this tile's sums (row independence)
                                int n16 = BK / UMMA_K;
                                bool half_last = false;
                                if (p.a_blocked) {
                                    const int vp = min(8, max(0, p.a_nchunks - kb * 8));  // valid panels
                                    n16 = (vp + 1) >> 1;
                                    half_last = (vp & 1) != 0;
                                }
#pragma unroll
                                for (int kk = 0; kk < BK / UMMA_K; ++kk) {
                                    if (kk >= n16) break;
                                    uint64_t ad = ptx::desc_make(a_lo0 + ((a_off + kk * a_kstep) >> 4), a_hi);
                                    if (half_last && kk == n16 - 1) {
                                        const uint32_t pa = a_base + a_off + kk * a_kstep;
                                        ad = ptx::smem_desc(pa, sbase + L.zero_off - pa, 128, 0);
                                    }
                                    const uint64_t bd = ptx::desc_make(b_lo0 + ((b_off + kk * p.b_kstep) >> 4), b_hi);
                                    if (BLR_DBG_ON(p, 8)) continue;  // debug: skip the MMA itself
                                    if constexpr (PAIR == 2) ptx::mma_bf16_pair(d_tmem, ad, bd, idesc_t, (si | j | kk) != 0);
                                    else ptx::mma_bf16(d_tmem, ad, bd, idesc_t, (si | j | kk) != 0);
                                    if (p.n_mma == 2) {  // second half: same A, B half 1, next TMEM columns
                                        const uint64_t bd2 = ptx::desc_make(
                                            b_lo0 + ((b_off + p.b_half_bytes + kk * p.b_kstep) >> 4), b_hi);
                                        const uint32_t d2 = d_tmem + static_cast<uint32_t>(p.BN / 2);
                                        if constexpr (PAIR == 2) ptx::mma_bf16_pair(d2, ad, bd2, idesc, (si | j | kk) != 0);
                                        else ptx::mma_bf16(d2, ad, bd2, idesc, (si | j | kk) != 0);
                                    }
                                }
                            }
                            if (BLR_DBG_ON(p, 16)) ptx::mbar_arrive(empty_bar + 8 * stage);  // debug: plain release
                            else commit_slot(empty_bar + 8 * stage);  // frees the smem slot (every CTA of the cluster)
                        }
                        __syncwarp();
                        ++mstep_tr;
                        if (++stage == p.stages) { stage = 0; phase ^= 1; }
                    }
                }
                const bool last_of_slice =
                    p.b_resident && (it + 1 >= ntiles || tile_get(p, titer, tile_tab, it + 1).slice != cur_slice);
                if (ptx::elect_one()) {
                    commit(tfull_bar + 8 * acc);  // accumulator ready for the epilogue(s)
                    if (last_of_slice) commit(bfree_bar);
                    if (trace) {
                        trace[4] = clock64();
                        if (it < 24) trace[16 + it] = trace[4];  // per-tile MMA issue-complete time
                    }
                }
                __syncwarp();
                if (++acc == p.acc_bufs) { acc = 0; acc_phase ^= 1; }
            }
        }
    } else {
        // ===================================================== epilogue =====================
        // Each warp owns TMEM lane quarter (warp % 4) = 32 token rows; the two warps of a quarter
        // split the tile's columns.  Results are rounded to bf16, staged in swizzled smem and
        // written with TMA bulk tensor stores (full 128-B lines, rows >= n_tok clipped by TMA).
        const int ew = warp - 2;              // 0..7
        const int quarter = warp & 3;         // TMEM lane quarter this warp may access
        const int half = ew >> 2;             // which half of the columns
        const uint32_t lane_addr = static_cast<uint32_t>(quarter * 32) << 16;
        const uint32_t stg = sbase + L.c_off + ew * p.stage_warp_bytes;  // this warp's staging
        int acc = 0;
        uint32_t acc_phase = 0;
        uint32_t nstore = 0;  // staged chunks written by this warp (buffer rotation)
        ptx::griddep_wait();  // our stores must not overtake the previous kernel's reads
        // pipelined layer (tile-blocked output): the chunk-store issuer of each column half signals
        // a token tile's ready counter once its stores have landed, two tiles later (bulk groups of
        // the newer tile may still be in flight; their count bounds the wait)
        const bool sig_iss = OUTF >= 2 && p.pipe_sig != nullptr && (ew & 3) == 0 && lane == 0;
        const uint64_t pol_out = ptx::l2_policy(p.l2_out);
        int sig_t[2] = {-1, -1};  // token tiles of the two previous tiles (oldest first)
        int sig_g = 0;            // bulk groups the previous tile committed
        auto sig_flush = [&](int keep_groups) {
            switch (keep_groups) {
                case 0: ptx::bulk_wait<0>(); break;
                case 1: ptx::bulk_wait<1>(); break;
                case 2: ptx::bulk_wait<2>(); break;
                case 3: ptx::bulk_wait<3>(); break;
                default: ptx::bulk_wait<0>(); break;
            }
        };
        for (int it = 0; !BLR_DBG_ON(p, 32) && it < ntiles; ++it) {
            const TileCoord tc = tile_get(p, titer, tile_tab, it);
            const int m0 = ((tc.m_blk * mcs + static_cast<int>(pidx)) * PAIR + static_cast<int>(crank)) * BM;
            const int row0 = m0 + quarter * 32;
            const int n0 = tc.n_blk * p.BN;
            if (sig_iss) {
                if (sig_t[0] >= 0) {  // the tile before last: all its groups are older than sig_g
                    sig_flush(sig_g);
                    ptx::pipe_release(p.pipe_sig + sig_t[0]);
                }
                sig_t[0] = sig_t[1];
                sig_t[1] = m0 / BM;
                sig_g = 0;
            }
            if constexpr (KIND == KIND_BLAST_PROJ) {
                // stage S[l][k][n0 : n0+BN] (fp32) for the S-weighted block sum
                ptx::named_bar_sync(1, 32 * NUM_EPI_WARPS);
                // k rows zero-padded to a multiple of 8: the accumulation loop below has no k bound
                const int b2p = (p.b2 + 7) / 8 * 8;
                const int cnt = p.b1 * b2p * p.BN;
                for (int e = ew * 32 + lane; e < cnt; e += 32 * NUM_EPI_WARPS) {
                    const int rho = e % p.BN;
                    const int lkp = e / p.BN;
                    const int l = lkp / b2p, k = lkp - l * b2p;
                    const int rr = n0 + rho;
                    ptx::st_shared_f32(s_tile + 4u * e,
                                       (k < p.b2 && rr < p.r)
                                           ? __bfloat162float(p.S[static_cast<long long>(l * p.b2 + k) * p.r + rr])
                                           : 0.f);
                }
                ptx::named_bar_sync(1, 32 * NUM_EPI_WARPS);
                if (trace && ew == 0 && lane == 0 && it == 0) trace[9] = clock64();
            }
            ptx::mbar_wait(tfull_bar + 8 * acc, acc_phase);
            ptx::tc_fence_after();
            if (trace && ew == 0 && lane == 0 && it == 0) trace[10] = clock64();
            const uint32_t tbase = tmem_base + acc * acc_stride + lane_addr;
            // per-half release (KParams::split_rel): column half 0 is freed as soon as this warp's
            // chunks below BN/2 are in registers
            const bool split_e = KIND == KIND_GEMM && PAIR == 2 && p.split_rel != 0;
            bool rel0 = false;
            auto release_h0 = [&]() {
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (PAIR == 2) ptx::mbar_arrive_remote(tempty_bar, lead_rank);
                    else ptx::mbar_arrive(tempty_bar);
                }
                rel0 = true;
            };

            if constexpr (KIND == KIND_BLAST_PROJ) {
                // Z''_k[t, rho] = sum_l S[l,k,rho] * Z_l[t, rho]   (Fig. 6 "s * z'")
                // This warp: rows of its quarter, rho in [n0 + half*BN/2, n0 + (half+1)*BN/2).
                const int W = p.BN / 2;               // staged row width (elements)
                const uint32_t row_bytes = W * 2;
                const uint32_t kstride = 32 * row_bytes;  // staging bytes per output block k
                const int parts = p.out_lo_off > 0 ? 2 : 1;
                // cooperative stores: the four warps of a column half stage [k][128 rows][W] together
                // and one thread stores each k as ONE box (instead of four 32-row boxes)
                const bool coop = p.coop_store != 0;
                const bool iss = (ew & 3) == 0 && lane == 0;
                const uint32_t kst = coop ? 4u * kstride : kstride;
                const uint32_t sbuf = coop ? sbase + L.c_off + half * 4u * p.stage_warp_bytes + quarter * kstride : stg;
                for (int part = 0; part < parts; ++part) {
                    if (coop) {
                        if (iss) ptx::bulk_wait_read<0>();
                        ptx::named_bar_sync(2 + half, 128);
                    } else {
                        if (lane == 0) ptx::bulk_wait_read<0>();
                        __syncwarp();
                    }
                    for (int sc = 0; sc < W / 8; ++sc) {
                        const int col = half * W + sc * 8;  // column within the tile
                        // output blocks k in groups of 8 (64 accumulator registers), inputs l in
                        // batches of 4 TMEM loads per wait (the loads' latency is paid once per
                        // batch, not once per l)
                        for (int kb0 = 0; kb0 < p.b2; kb0 += 8) {
                            unsigned long long acc2[8][4];
#pragma unroll
                            for (int k = 0; k < 8; ++k)
#pragma unroll
                                for (int e = 0; e < 4; ++e) acc2[k][e] = 0ull;
                            for (int lb = 0; lb < p.b1; lb += 4) {
                                float z[4][8];
#pragma unroll
                                for (int j = 0; j < 4; ++j)
                                    if (lb + j < p.b1) ptx::tmem_ld_x8(tbase + (lb + j) * p.BN + col, z[j]);
                                ptx::tmem_wait_ld();
                                if (trace && ew == 0 && lane == 0 && it == 0 && sc == 0 && lb == 0) trace[12] = clock64();
#pragma unroll
                                for (int j = 0; j < 4; ++j) {
                                    if (lb + j < p.b1) {
                                        unsigned long long z2[4];
#pragma unroll
                                        for (int e = 0; e < 4; ++e) z2[e] = ptx::pack_f32x2(z[j][2 * e], z[j][2 * e + 1]);
                                        const uint32_t srow =
                                            s_tile + 4u * (((lb + j) * ((p.b2 + 7) / 8 * 8) + kb0) * p.BN + col);
#pragma unroll
                                        for (int k = 0; k < 8; ++k) {  // rows k >= b2 of the S tile are zero
                                            const ulonglong2 sa = ptx::ld_shared_v2u64(srow + 4u * k * p.BN);
                                            const ulonglong2 sb = ptx::ld_shared_v2u64(srow + 4u * k * p.BN + 16u);
                                            ptx::ffma2(acc2[k][0], sa.x, z2[0]);
                                            ptx::ffma2(acc2[k][1], sa.y, z2[1]);
                                            ptx::ffma2(acc2[k][2], sb.x, z2[2]);
                                            ptx::ffma2(acc2[k][3], sb.y, z2[3]);
                                        }
                                    }
                                }
                            }
#pragma unroll
                            for (int k = 0; k < 8; ++k) {
                                if (kb0 + k < p.b2) {
                                    float f[8];
#pragma unroll
                                    for (int e = 0; e < 4; ++e) ptx::unpack_f32x2(acc2[k][e], f[2 * e], f[2 * e + 1]);
                                    stage_row8(sbuf + (kb0 + k) * kst, lane, sc, row_bytes, p.c_swz, f, part);
                                }
                            }
                        }
                        if (trace && ew == 0 && lane == 0 && it == 0 && sc < 2) trace[13 + sc] = clock64();
                    }
                    if (trace && ew == 0 && lane == 0 && it == 0) trace[11] = clock64();
                    ptx::fence_async_smem();
                    if (coop) {
                        ptx::named_bar_sync(2 + half, 128);
                        if (iss) {
                            const uint32_t hb = sbase + L.c_off + half * 4u * p.stage_warp_bytes;
                            for (int k = 0; k < p.b2; ++k)
                                ptx::tma_store_4d(&tmC, hb + k * kst, n0 + half * W, part, m0, k);
                            ptx::bulk_commit();
                        }
                    } else {
                        __syncwarp();
                        if (lane == 0) {
                            for (int k = 0; k < p.b2; ++k)
                                ptx::tma_store_4d(&tmC, stg + k * kstride, n0 + half * W, part, row0, k);
                            ptx::bulk_commit();
                        }
                    }
                }
            } else {
                const int nvalid = BLR_DBG_ON(p, 4) ? 0 : min(p.BN, p.N - n0);  // dbg 4: empty epilogue
                const int parts = p.out_lo_off > 0 ? 2 : 1;
                // column chunks of CW elements; chunk j of this warp starts at col = (half + 2 j) * CW
                const int CW = p.c_box_w;
                const uint32_t row_bytes = CW * 2;
                const uint32_t buf_bytes = 32 * row_bytes;
                for (int c0 = half * CW; c0 < nvalid; c0 += 2 * CW) {
                    if (split_e && !rel0 && c0 >= p.BN / 2) release_h0();
                    // TMEM -> registers: CW fp32 columns of this warp's 32 rows (mult. of 8; CW <= 64
                    // except for the unswizzled whole-r' Monarch chunks, staged 64 columns at a time)
                    float fv[64];
                    if (OUTF >= 2 || CW <= 64) {
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            if (j * 8 < CW) ptx::tmem_ld_x8(tbase + c0 + j * 8, *reinterpret_cast<float(*)[8]>(&fv[j * 8]));
                        ptx::tmem_wait_ld();
                    }
                    if constexpr (KIND == KIND_GEMM && OUTF == 0) {
                        if (p.out_cs > 0) {  // strided direct stores (transposed output order)
                            const int row = row0 + lane;
                            if (row < p.n_tok) {
                                __nv_bfloat16* yb = static_cast<__nv_bfloat16*>(p.out_ptr) +
                                                    static_cast<long long>(row) * p.out_rs + tc.g * p.out_gstride;
#pragma unroll
                                for (int j = 0; j < 64; ++j) {
                                    const int c = n0 + c0 + j;
                                    if (j < CW && c < p.N)
                                        yb[static_cast<long long>(c) * p.out_cs] = __float2bfloat16_rn(fv[j]);
                                }
                            }
                            continue;
                        }
                    }
                    if constexpr (OUTF == 3) {
                        // tile-blocked e4m3 output: as OUTF 2 below with 8-B panel rows (1-KB panels)
                        const uint32_t hbuf_bytes = 128u * CW;
                        const uint32_t hbuf = sbase + L.c_off + half * 4u * p.stage_warp_bytes +
                                              (nstore % p.stage_bufs) * hbuf_bytes;
                        ++nstore;
                        const bool iss = (ew & 3) == 0 && lane == 0;
                        if (iss) {
                            if (p.stage_bufs == 2) ptx::bulk_wait_read<1>();
                            else ptx::bulk_wait_read<0>();
                        }
                        ptx::named_bar_sync(2 + half, 128);
                        for (int h0 = 0; h0 < CW; h0 += 64) {  // chunks wider than 64: two passes
                            if (h0 > 0) {
#pragma unroll
                                for (int j = 0; j < 8; ++j)
                                    if (h0 + j * 8 < CW)
                                        ptx::tmem_ld_x8(tbase + c0 + h0 + j * 8, *reinterpret_cast<float(*)[8]>(&fv[j * 8]));
                                ptx::tmem_wait_ld();
                            }
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                if (h0 + j * 8 < CW) {
                                    uint2 w;
                                    w.x = ptx::pack_e4m3x2(fv[j * 8 + 0], fv[j * 8 + 1]) |
                                          (ptx::pack_e4m3x2(fv[j * 8 + 2], fv[j * 8 + 3]) << 16);
                                    w.y = ptx::pack_e4m3x2(fv[j * 8 + 4], fv[j * 8 + 5]) |
                                          (ptx::pack_e4m3x2(fv[j * 8 + 6], fv[j * 8 + 7]) << 16);
                                    ptx::st_shared_v2u32(hbuf + (h0 / 8 + j) * 1024u + (quarter * 32u + lane) * 8u, w);
                                }
                            }
                        }
                        ptx::fence_async_smem();
                        ptx::named_bar_sync(2 + half, 128);
                        // (a CTA pair's second tile past n_tok has no tile of its own in the
                        //  layout: its box would land on the next group's first tile)
                        if (iss && !BLR_DBG_ON(p, 1) && m0 < p.n_tok) {
                            const int cc = (n0 + c0) >> 3;
                            ptx::tma_store_4d(&tmC, hbuf, 0, 0, cc, tc.g * p.o_tiles + m0 / BM);
                            ptx::bulk_commit();
                            ++sig_g;
                        }
                        continue;
                    }
                    if constexpr (OUTF == 2) {
                        // tile-blocked fp16 output [g][T][N/8][128][8]: the four warps of this column
                        // half (one per TMEM lane quarter) stage the chunk's 128 rows together and one
                        // thread stores the chunk's panels as ONE bulk copy (per-quarter 512-B copies
                        // made the S1 epilogue TMA-op bound: 96 copies per tile)
                        const uint32_t hbuf_bytes = 128u * CW * 2u;
                        const uint32_t hbuf = sbase + L.c_off + half * 4u * p.stage_warp_bytes +
                                              (nstore % p.stage_bufs) * hbuf_bytes;
                        ++nstore;
                        const bool iss = (ew & 3) == 0 && lane == 0;
                        if (iss) {
                            if (p.stage_bufs == 2) ptx::bulk_wait_read<1>();
                            else ptx::bulk_wait_read<0>();
                        }
                        ptx::named_bar_sync(2 + half, 128);
                        for (int h0 = 0; h0 < CW; h0 += 64) {  // chunks wider than 64: two passes
                            if (h0 > 0) {
#pragma unroll
                                for (int j = 0; j < 8; ++j)
                                    if (h0 + j * 8 < CW)
                                        ptx::tmem_ld_x8(tbase + c0 + h0 + j * 8, *reinterpret_cast<float(*)[8]>(&fv[j * 8]));
                                ptx::tmem_wait_ld();
                            }
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                if (h0 + j * 8 < CW) {
                                    uint4 w;
                                    w.x = ptx::pack_f16x2(fv[j * 8 + 0], fv[j * 8 + 1]);
                                    w.y = ptx::pack_f16x2(fv[j * 8 + 2], fv[j * 8 + 3]);
                                    w.z = ptx::pack_f16x2(fv[j * 8 + 4], fv[j * 8 + 5]);
                                    w.w = ptx::pack_f16x2(fv[j * 8 + 6], fv[j * 8 + 7]);
                                    ptx::st_shared_v4(hbuf + (h0 / 8 + j) * 2048u + (quarter * 32u + lane) * 16u, w);
                                }
                            }
                        }
                        ptx::fence_async_smem();
                        ptx::named_bar_sync(2 + half, 128);
                        if (iss && !BLR_DBG_ON(p, 1) && m0 < p.n_tok) {
                            // tile-blocked [g][T][N/8][128][8]: this chunk's panels of tile T are
                            // contiguous -> one bulk copy (rows >= n_tok are zeros: A was OOB-filled;
                            // a pair's second tile past n_tok is skipped: it would alias the next
                            // group's first tile)
                            const int cc = (n0 + c0) >> 3;
                            if (p.l2_out) ptx::tma_store_4d_hint(&tmC, hbuf, 0, 0, cc, tc.g * p.o_tiles + m0 / BM, pol_out);
                            else ptx::tma_store_4d(&tmC, hbuf, 0, 0, cc, tc.g * p.o_tiles + m0 / BM);
                            ptx::bulk_commit();
                            ++sig_g;
                        }
                        continue;
                    }
                    if constexpr ((KIND == KIND_GEMM && OUTF <= 1) || KIND == KIND_MONARCH_PROJ) {
                        if (p.coop_store) {
                            // the four warps of this column half stage their 32 rows of the chunk into one
                            // 128-row buffer and one thread stores it as ONE tensor box: a quarter of the
                            // store ops (the per-SM TMA op rate bounds the streamed GEMMs)
                            const uint32_t hbuf_bytes = 4u * buf_bytes;
                            const bool iss = (ew & 3) == 0 && lane == 0;
                            for (int part = 0; part < parts; ++part) {
                                const uint32_t hbuf = sbase + L.c_off + half * 4u * p.stage_warp_bytes +
                                                      (nstore % p.stage_bufs) * hbuf_bytes;
                                ++nstore;
                                if (iss) {
                                    if (p.stage_bufs == 2) ptx::bulk_wait_read<1>();
                                    else ptx::bulk_wait_read<0>();
                                }
                                ptx::named_bar_sync(2 + half, 128);
#pragma unroll
                                for (int j = 0; j < 8; ++j)
                                    if (j * 8 < CW)
                                        stage_row8<OUTF>(hbuf, quarter * 32 + lane, j, row_bytes, p.c_swz,
                                                         *reinterpret_cast<const float(*)[8]>(&fv[j * 8]), part);
                                ptx::fence_async_smem();
                                ptx::named_bar_sync(2 + half, 128);
                                if (iss && !BLR_DBG_ON(p, 1)) {
                                    if constexpr (KIND == KIND_MONARCH_PROJ) {
                                        // Z'[k][t][l r' + rho] (the b2 <-> b1 permutation)
                                        const int k = tc.n_blk * p.kb_per_tile + c0 / p.r_blk;
                                        ptx::tma_store_5d(&tmC, hbuf, c0 % p.r_blk, tc.g, part, m0, k);
                                    } else {
                                        if (p.l2_out) ptx::tma_store_4d_hint(&tmC, hbuf, n0 + c0, part, tc.g, m0, pol_out);
                                        else ptx::tma_store_4d(&tmC, hbuf, n0 + c0, part, tc.g, m0);
                                    }
                                    ptx::bulk_commit();
                                }
                            }
                            continue;
                        }
                    }
                    for (int part = 0; part < parts; ++part) {
                        const uint32_t buf = stg + (nstore % p.stage_bufs) * buf_bytes;
                        ++nstore;
                        // the bulk store that last read `buf` must have finished reading it
                        if (lane == 0) {
                            if (p.stage_bufs == 2) ptx::bulk_wait_read<1>();
                            else ptx::bulk_wait_read<0>();
                        }
                        __syncwarp();
                        for (int h0 = 0; h0 < CW; h0 += 64) {
                            if (CW > 64) {  // wide chunk: the next <= 64 columns
#pragma unroll
                                for (int j = 0; j < 8; ++j)
                                    if (h0 + j * 8 < CW)
                                        ptx::tmem_ld_x8(tbase + c0 + h0 + j * 8, *reinterpret_cast<float(*)[8]>(&fv[j * 8]));
                                ptx::tmem_wait_ld();
                            }
#pragma unroll
                            for (int j = 0; j < 8; ++j) {
                                if (h0 + j * 8 < CW && !BLR_DBG_ON(p, 2)) {
                                    stage_row8<OUTF>(buf, lane, h0 / 8 + j, row_bytes, p.c_swz,
                                                     *reinterpret_cast<const float(*)[8]>(&fv[j * 8]), part);
                                }
                            }
                        }
                        ptx::fence_async_smem();
                        __syncwarp();
                        if (lane == 0 && !BLR_DBG_ON(p, 1)) {
                            if constexpr (KIND == KIND_GEMM) {
                                // out (N, comp, groups, rows): element (c, part, g, t); blocked
                                // out (8, rows, N/8, groups): element (c % 8, t, c / 8, g)
                                if constexpr (OUTF == 2) {  // CW/8 panels of 32 rows x 16 B, contiguous in global
                                    const int nch = p.N >> 3, rows = min(32, p.n_tok - row0);
                                    auto* ob = static_cast<uint16_t*>(p.out_ptr) + tc.g * p.out_gstride;
                                    for (int j = 0; j < CW / 8 && ((n0 + c0) >> 3) + j < nch; ++j)
                                        if (rows > 0)
                                            ptx::bulk_store(ob + ((static_cast<long long>((n0 + c0) >> 3) + j) * p.n_tok + row0) * 8,
                                                            buf + j * 512, rows * 16);
                                } else {
                                    ptx::tma_store_4d(&tmC, buf, n0 + c0, part, tc.g, row0);
                                }
                            } else {
                                // Monarch: chunk lies inside one output block k (CW divides r');
                                // Z'[k][t][l r' + rho]  (the b2 <-> b1 permutation)
                                const int k = tc.n_blk * p.kb_per_tile + c0 / p.r_blk;
                                ptx::tma_store_5d(&tmC, buf, c0 % p.r_blk, tc.g, part, row0, k);
                            }
                            ptx::bulk_commit();
                        }
                    }
                }
            }
            if (trace && ew == 0 && lane == 0 && it < 24) trace[40 + it] = clock64();  // epilogue done
            if (sig_iss) {
                // the CTA's last tile of this token-tile row: flush the deferred signals (the producer
                // may block on back-pressure before the next tile, which would otherwise hold them)
                const bool row_end = it + 1 >= ntiles || tile_get(p, titer, tile_tab, it + 1).m_blk != tc.m_blk;
                if (row_end) {
                    ptx::bulk_wait<0>();
                    for (int j = 0; j < 2; ++j)
                        if (sig_t[j] >= 0) ptx::pipe_release(p.pipe_sig + sig_t[j]);
                    sig_t[0] = -1;
                    sig_t[1] = -1;
                    sig_g = 0;
                }
            }
            if (split_e && !rel0) release_h0();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                const uint32_t tb = tempty_bar + 8 * (split_e ? 1 : acc);  // split: column half 1
                if constexpr (PAIR == 2) ptx::mbar_arrive_remote(tb, lead_rank);  // leader's barrier
                else ptx::mbar_arrive(tb);
            }
            if (++acc == p.acc_bufs) { acc = 0; acc_phase ^= 1; }
        }
        if (trace && ew == 0 && lane == 0) trace[5] = clock64();
        if (sig_iss) {  // the last two tiles
            ptx::bulk_wait<0>();
            for (int j = 0; j < 2; ++j)
                if (sig_t[j] >= 0) ptx::pipe_release(p.pipe_sig + sig_t[j]);
        }
        // only the staging smem must outlive the stores: wait for their smem reads, not for the
        // global writes (those complete with the grid, before any dependent grid proceeds)
        if (lane == 0) ptx::bulk_wait_read<0>();
        __syncwarp();
        if (trace && ew == 0 && lane == 0) trace[6] = clock64();
    }

    ptx::tc_fence_before();
    __syncthreads();
    if constexpr (PAIR == 2) ptx::cluster_sync();  // the peer's MMAs / remote arrivals are done
    if (trace && threadIdx.x == 0) trace[7] = clock64();
    if (warp == 1) {
        ptx::tc_fence_after();
        if constexpr (PAIR == 2) ptx::tmem_dealloc_pair<TMEM_COLS>(tmem_base);
        else ptx::tmem_dealloc<TMEM_COLS>(tmem_base);
    }
}

template <int KIND, int PAIR, int OUTF = 0>
__global__ void __launch_bounds__(NUM_THREADS, 1)
    blr_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmB2, const KParams p) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    // 1024-B alignment for the 128-B swizzle atoms.
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    gemm_body<KIND, PAIR, OUTF>(tmA, tmB, tmC, tmB2, p, smem, static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x));
}

// ------------------------------------------------------------------------- BLAST S2 kernel -----
// Z''[k][t][rho] = sum_l S[l,k,rho] * Z[l][t][rho]   (the S-weighted block sum)
// Used when b1 * r does not fit TMEM, between the S1 grouped GEMM and the S3 expand.
// Bandwidth-bound streaming kernel:
//  * work item = (64-wide rho chunk, S2_ROWS token rows); items are enumerated chunk-major and
//    each block walks a contiguous run of them, so it reloads its S slice at most twice;
//  * warp 0 is the TMA producer: one 3-D box (64 rho, S2_ROWS rows, b1 blocks) of Z per item into
//    an mbarrier ring of up to S2_MAX_STAGES -- all b1 blocks of the item in flight in one request;
//  * warps 1..NW each own KG output blocks k and keep their S[l, k, rho pair] for all l in
//    registers (packed fp32x2), so shared memory carries only Z: lane = 2 rho, a warp's read of
//    one (l, row) is one conflict-free 128/256-B line, and each Z value feeds KG packed FMAs;
//  * Z''_k rows are written straight from registers (bf16x2 per lane: one 128-B line per warp).
// Z is S1's output in fp16 (11-bit significand, R13).
// fp32 accumulation in ascending l, one RNE rounding to bf16 (plus the compensation term lo when
// comp == 2) -- the same single rounding of Z'' as the fused path; no atomics (deterministic).
constexpr int S2_ROWS = 8;
constexpr int S2_MAX_STAGES = 16;  // ring depth is chosen at launch (<= ~200 KB of smem)
constexpr int S2_MAXL = 16;
constexpr int S2_RU = 4;     // rows accumulated together per warp (independent FMA chains)
constexpr int S2_RSPLIT = 2; // warps sharing a k-group split the item's rows (S2_ROWS = RU x RSPLIT)

template <int KG, int NL>
__global__ void __launch_bounds__(32 * 16, 1)
    blast_s2_kernel(const __grid_constant__ CUtensorMap tmZ, const __nv_bfloat16* __restrict__ S,
                    __nv_bfloat16* __restrict__ Zpp, int n_tok, int b1, int b2, int r, int comp,
                    int slabs, int total_items, int items_per_block, int nchunks, int map_mode, int nst) {
    extern __shared__ __align__(1024) uint8_t s2_smem[];
    constexpr uint32_t ESZ = 2;  // fp16 Z
    constexpr uint32_t ROW_BYTES = 64 * ESZ;
    // a stage holds NL planes [l][row][64 rho]; planes b1..NL-1 are zeroed once (never loaded)
    constexpr uint32_t STAGE_BYTES = NL * S2_ROWS * ROW_BYTES;
    const uint32_t tx_bytes = static_cast<uint32_t>(b1) * S2_ROWS * ROW_BYTES;
    const uint32_t ring = ptx::smem_u32(s2_smem);
    const uint32_t bars = ring + nst * STAGE_BYTES;  // full[nst], empty[nst]
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = blockDim.x / 32;  // consumer warps: (k-group, row half) pairs
    // item j of this block -> (rho chunk, slab of S2_ROWS rows)
    //   map_mode 0: a contiguous run of the chunk-major item list
    //   map_mode 1: a fixed chunk (blockIdx % nchunks) and every (grid/nchunks)-th slab, so the
    //               blocks running at any moment read all chunks of the same rows (whole Z rows
    //               from DRAM rather than 128-B pieces of many)
    int it0, cnt, slab_step = 1;
    if (map_mode == 1) {
        const int gpc = gridDim.x / nchunks;
        it0 = (blockIdx.x % nchunks) * slabs + blockIdx.x / nchunks;
        cnt = (slabs - static_cast<int>(blockIdx.x / nchunks) + gpc - 1) / gpc;
        slab_step = gpc;
    } else {
        it0 = blockIdx.x * items_per_block;
        cnt = max(0, min(total_items, it0 + items_per_block) - it0);
    }
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            ptx::mbar_init(bars + 8 * s, 1);
            ptx::mbar_init(bars + 8 * (nst + s), nw);
        }
        ptx::fence_barrier_init();
    }
    if (b1 < NL) {
        const uint32_t pad = (NL - b1) * S2_ROWS * ROW_BYTES;
        for (int s = 0; s < nst; ++s)
            for (uint32_t o = threadIdx.x * 16; o < pad; o += blockDim.x * 16)
                ptx::st_shared_v4(ring + s * STAGE_BYTES + tx_bytes + o, make_uint4(0, 0, 0, 0));
    }
    __syncthreads();
    ptx::griddep_wait();  // Z is the previous kernel's output
    // producer: lane 0 of warp 0 (also a consumer) keeps nst - 1 items in flight; it
    // refills a slot once every consumer warp has released that slot's previous item
    auto produce = [&](int j) {
        const int it = it0 + j * slab_step;
        const int s = j % nst;
        if (j >= nst) ptx::mbar_wait(bars + 8 * (nst + s), ((j / nst) - 1) & 1);
        ptx::mbar_arrive_expect_tx(bars + 8 * s, tx_bytes);
        ptx::tma_load_3d(ring + s * STAGE_BYTES, &tmZ, bars + 8 * s, (it / slabs) * 64, (it % slabs) * S2_ROWS, 0);
    };
    if (threadIdx.x == 0) {
        ptx::prefetch_tmap(&tmZ);
        for (int j = 0; j < min(cnt, nst - 1); ++j) produce(j);
    }
    const int k0 = (warp % (nw / S2_RSPLIT)) * KG;
    const int rbase = (warp / (nw / S2_RSPLIT)) * S2_RU;
    const int row_stride = comp * r;  // elements between Z'' rows
    unsigned long long sreg[NL][KG];
    __nv_bfloat16* kbase[KG];         // Z''[k0 + kk][0][rho0]
    int cur_chunk = -1;
    for (int j = 0; j < cnt; ++j) {
        const int it = it0 + j * slab_step;
        const int chunk = it / slabs;
        const int rho0 = chunk * 64 + 2 * lane;
        const bool col_ok = rho0 < r;
        if (chunk != cur_chunk) {  // S[l, k0 + kk, rho0 .. rho0 + 1] for this warp's blocks
            cur_chunk = chunk;
#pragma unroll
            for (int kk = 0; kk < KG; ++kk)
                kbase[kk] = Zpp + static_cast<long long>(k0 + kk) * n_tok * row_stride + rho0;
#pragma unroll
            for (int l = 0; l < NL; ++l)
#pragma unroll
                for (int kk = 0; kk < KG; ++kk) {
                    uint32_t w = 0;
                    if (l < b1 && k0 + kk < b2 && col_ok)
                        w = __ldg(reinterpret_cast<const uint32_t*>(S + (static_cast<long long>(l) * b2 + k0 + kk) * r + rho0));
                    sreg[l][kk] = ptx::pack_f32x2(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
                }
        }
        if (threadIdx.x == 0 && j + nst - 1 < cnt) produce(j + nst - 1);
        const int s = j % nst;
        ptx::mbar_wait(bars + 8 * s, (j / nst) & 1);
        const uint8_t* buf = s2_smem + s * STAGE_BYTES + lane * 2 * ESZ;
        const int row0 = (it % slabs) * S2_ROWS;
        {
            const int rr = rbase;
            unsigned long long acc[S2_RU][KG];
#pragma unroll
            for (int u = 0; u < S2_RU; ++u)
#pragma unroll
                for (int kk = 0; kk < KG; ++kk) acc[u][kk] = 0ull;
#pragma unroll
            for (int l = 0; l < NL; ++l) {
#pragma unroll
                for (int u = 0; u < S2_RU; ++u) {
                    const uint8_t* a = buf + (l * S2_ROWS + rr + u) * ROW_BYTES;
                    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(a));
                    const unsigned long long z2 = ptx::pack_f32x2(f.x, f.y);
#pragma unroll
                    for (int kk = 0; kk < KG; ++kk) ptx::ffma2(acc[u][kk], sreg[l][kk], z2);
                }
            }
#pragma unroll
            for (int u = 0; u < S2_RU; ++u) {
                const int t = row0 + rr + u;
                if (col_ok && t < n_tok) {
                    const long long roff = static_cast<long long>(t) * row_stride;
#pragma unroll
                    for (int kk = 0; kk < KG; ++kk) {
                        if (k0 + kk < b2) {
                            float f0, f1;
                            ptx::unpack_f32x2(acc[u][kk], f0, f1);
                            const uint32_t hi = ptx::pack_bf16x2(f0, f1);
                            __nv_bfloat16* dst = kbase[kk] + roff;
                            *reinterpret_cast<uint32_t*>(dst) = hi;
                            if (comp == 2)
                                *reinterpret_cast<uint32_t*>(dst + r) = ptx::pack_bf16x2(
                                    f0 - __uint_as_float(hi << 16), f1 - __uint_as_float(hi & 0xFFFF0000u));
                        }
                    }
                }
            }
        }
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(bars + 8 * (nst + s));
    }
}

// ------------------------------------------------------------- BLAST S2 on the tensor cores ----
// Z''[k][t][rho] = sum_l S[l,k,rho] * Z[l][t][rho] as a tcgen05 contraction
// (DESIGN.md §5.3).  For an 8-wide rho chunk c the S-weighted block sum is one GEMM
//     Z''[t, (k, rho)] = sum_(l, rho') Z[t, (l, rho')] * B_c[(l, rho'), (k, rho)],
//     B_c[(l, rho'), (k, rho)] = S[l, k, 8c + rho] * delta(rho, rho'),
// M = 128 tokens, K = 8 b1, N = 8 b2 (<= 128).  In the canonical no-swizzle K-major UMMA layout
// an 8x8 core matrix of B_c is exactly diag(S[l, k, 8c .. 8c+7]), so B_c is a fixed zero
// pattern whose 8 b1 b2 diagonal entries are rewritten per item (S converted bf16 -> fp16), and
// the A operand is b1 panels of Z: core matrix (t/8, l) = 8 rows x 16 B, each panel moved by one
// 1-D bulk copy (a tensor box with 16-B rows moves one row per request: measured 2x slower).  The
// S1 epilogue writes that layout, S3 reads it.
// fp16 x fp16 products are exact, accumulation fp32; Z'' is rounded once to bf16 (RNE).
// Z and Z'' are tile-blocked, [l][T][r/8][128][8] and [k][T][r/8][128][8]: every
// (l, T, c) panel is 2 KB contiguous and the panels c = 0.. of one tile are adjacent.  Items
// (128-token tile T, chunk c) are enumerated tile-major and each CTA walks one contiguous run of
// them, so its b1 panel reads and b2 panel writes are sequential streams.
// Roles: warp 0 TMA producer, warp 1 TMEM owner + MMA issuer, warps 2-3 build B_c, warps 4-7
// epilogue (TMEM -> bf16 -> smem [k][t][8] -> b2 bulk stores of the (k, T, c) panels).
constexpr int S2M_ASTAGES = 4;  // barrier slots (fp16 Z uses 3 stages, e4m3 Z 4)
constexpr int S2M_THREADS = 256;
constexpr int S2M_THREADS_FP8 = 384;  // + warps 8-11 widening e4m3 Z with the builder warps 2-3
template <bool FP8>
__host__ __device__ constexpr int s2m_threads() { return FP8 ? S2M_THREADS_FP8 : S2M_THREADS; }
struct S2MLayout {  // byte offsets in dynamic smem (1024-aligned base)
    uint32_t a, a16, b, c, bars, tslot, total, a_bytes, b_bytes, c_bytes, stages;
};
// fp8: Z arrives as e4m3 panels (1 KB) in 4 raw slots (deeper than fp16's 3 x 2 KB: the bytes in
// flight per SM set the rate of this HBM-bound kernel) and is widened by the builder warps into two
// fp16 A buffers (2 KB panels) for the f16 MMA (no 8-bit kind: S stays 16-bit); B_c then has one
// buffer (it changes only when a CTA's run crosses a chunk)
__host__ __device__ inline S2MLayout s2m_layout(int b1, int b2, bool fp8 = false) {
    S2MLayout L;
    const int b1p = (b1 + 1) & ~1;  // K in pairs of 8-wide core matrices (UMMA K = 16)
    const int b2p = (b2 + 1) & ~1;  // UMMA N = 8 b2p, a multiple of 16
    L.stages = fp8 ? 4 : 3;
    L.a_bytes = static_cast<uint32_t>(b1p) * 128 * (fp8 ? 8 : 16);
    L.b_bytes = static_cast<uint32_t>(b2p) * b1p * 128;
    L.c_bytes = static_cast<uint32_t>(b2) * 128 * 16;
    L.a = 0;
    L.a16 = L.a + L.stages * L.a_bytes;
    L.b = L.a16 + (fp8 ? 2u * b1p * 2048u : 0u);
    L.c = L.b + (fp8 ? 1 : 2) * L.b_bytes;
    L.bars = L.c + 2 * L.c_bytes;
    L.tslot = L.bars + 8 * (2 * S2M_ASTAGES + 2 * 2 + 2 * 2 + 2 * 2);
    L.total = L.tslot + 16;
    return L;
}

// MAXB2: largest b2 of the instantiation (8: few output blocks -> half the epilogue registers and
// two CTAs per SM, which is what the short, latency-bound S2 of small layers needs; 16: b = 16).
// FP8: Z is e4m3; the widening to fp16 is exact, the MMA and everything after
// it are unchanged.
// Pipelined-layer hooks of the S2 body (blast_pipe_kernel): items are dealt round robin over the
// token-tile-major item list, each item waits for its token tile of Z and signals its token tile
// of Z'' once its stores have landed.
constexpr int S2_SIG_LAG = 8;
constexpr int S2_PIPE_WIN = 8;  // default token tiles per window of the pipelined S2 role
struct S2Pipe {
    const unsigned int* wait_ctr;  // Z token tile T ready once wait_ctr[T] >= wait_target
    unsigned int wait_target;
    unsigned int* sig_ctr;         // += 1 per item (T, c) once its Z'' panels are stored
    int win;                       // token tiles per window
    int dbg;                       // BLR_DEBUG_KNOBS builds: 1 no acquire waits, 2 no store-completion waits
    int l2_in, l2_out;             // L2 hints of the Z loads / Z'' stores (0 none, 1 evict_first, 2 evict_last)
};

template <int MAXB2, bool FP8 = false>
__device__ __forceinline__ void s2_body(const CUtensorMap& tmZ, const CUtensorMap& tmZpp, const void* __restrict__ Z,
                                        __nv_bfloat16* __restrict__ Zpp, const __nv_bfloat16* __restrict__ S,
                                        int n_tok, int b1, int b2, int r, int order, int t0, int t0o,
                                        uint8_t* s2m_smem, int vblock, int vgrid, const S2Pipe* pipe) {
    const S2MLayout L = s2m_layout(b1, b2, FP8);
    const int nst = static_cast<int>(L.stages);
    const int b1p = (b1 + 1) & ~1;
    const uint32_t base = ptx::smem_u32(s2m_smem);
    const uint32_t a_full = base + L.bars, a_empty = a_full + 8 * S2M_ASTAGES;
    const uint32_t b_full = a_empty + 8 * S2M_ASTAGES, b_empty = b_full + 16;
    const uint32_t d_full = b_empty + 16, d_empty = d_full + 16;
    const uint32_t w_full = d_empty + 16, w_empty = w_full + 16;  // FP8: widened fp16 A buffers
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr int NB = FP8 ? 1 : 2;  // B_c buffers
    constexpr int NT = s2m_threads<FP8>();
    constexpr int NCONV = FP8 ? 192 : 64;  // threads widening Z (FP8: warps 2-3 and 8-11)
    const int nchunks = r / 8;
    const int tiles = (n_tok + 127) / 128;
    const int total = tiles * nchunks;
    // each CTA walks one contiguous run of the chunk-major item list: its reads of every Z panel
    // (l, c) and writes of every Z'' panel (k, c) are sequential streams, and B_c changes only
    // when the run crosses a chunk (at most ~2 rebuilds per CTA)
    // Pipelined layer: the token tiles are walked in windows of S2_PIPE_WIN; this CTA owns the
    // chunks c = vblock, vblock + vgrid, ... and, per window, runs each of its chunks over the
    // window's token tiles (token tile fastest), so B_c is rebuilt once per window and chunk
    // (a per-item rebuild, with its global loads of S, bounded the role at ~20 GB/s per SM).
    const bool rr = pipe != nullptr;
    const int win = rr ? pipe->win : 1;
    const int nc_u = rr ? (vblock < nchunks ? (nchunks - vblock + vgrid - 1) / vgrid : 0) : 0;
    const int it0 = rr ? 0 : static_cast<int>(static_cast<long long>(vblock) * total / vgrid);
    const int cnt = rr ? nc_u * tiles : static_cast<int>(static_cast<long long>(vblock + 1) * total / vgrid) - it0;
    const bool tile_major = order != 0;
    auto item = [&](int j, int& T, int& c) {
        if (rr) {
            const int per_w = nc_u * win;
            const int w = j / per_w;
            const int rem = j - w * per_w;
            const int wc = min(win, tiles - w * win);  // the last window may be short
            const int ci = rem / wc;
            T = w * win + (rem - ci * wc);
            c = vblock + ci * vgrid;
            return;
        }
        const int i = it0 + j;
        if (tile_major) {  // panels (l, T, c), c = 0.. adjacent: sequential streams
            T = i / nchunks;
            c = i - T * nchunks;
        } else {  // chunk-major: B_c rebuilt only when the run changes chunk
            c = i / tiles;
            T = i - c * tiles;
        }
    };
    if (threadIdx.x == 0) {
        for (int s = 0; s < nst; ++s) {
            ptx::mbar_init(a_full + 8 * s, 1);
            ptx::mbar_init(a_empty + 8 * s, 1);
        }
        for (int s = 0; s < 2; ++s) {
            ptx::mbar_init(b_full + 8 * s, 64);
            ptx::mbar_init(b_empty + 8 * s, 1);
            ptx::mbar_init(d_full + 8 * s, 1);
            ptx::mbar_init(d_empty + 8 * s, 4);
            ptx::mbar_init(w_full + 8 * s, NCONV);
            ptx::mbar_init(w_empty + 8 * s, 1);
        }
        ptx::fence_barrier_init();
    }
    // zero both B_c buffers (the off-diagonal pattern never changes) and the A pad plane (b1 odd)
    for (uint32_t o = threadIdx.x * 16; o < NB * L.b_bytes; o += NT * 16)
        ptx::st_shared_v4(base + L.b + o, make_uint4(0, 0, 0, 0));
    if (b1p != b1) {
        if constexpr (FP8) {
            for (int s = 0; s < 2; ++s)
                for (uint32_t o = threadIdx.x * 16; o < 128 * 16; o += NT * 16)
                    ptx::st_shared_v4(base + L.a16 + s * b1p * 2048 + b1 * 2048 + o, make_uint4(0, 0, 0, 0));
        } else {
            // (the fp16 ring has L.stages = 3 slots, fewer than the S2M_ASTAGES barrier slots: zeroing
            //  a 4th pad plane wrote past the layout -- past the allocation for small b2 -- found by
            //  tests/test_gpu_fuzz.py with b1 = 11, b2 <= 2)
            for (int s = 0; s < nst; ++s)
                for (uint32_t o = threadIdx.x * 16; o < 128 * 16; o += NT * 16)
                    ptx::st_shared_v4(base + L.a + s * L.a_bytes + b1 * 2048 + o, make_uint4(0, 0, 0, 0));
        }
    }
    ptx::fence_async_smem();
    if (warp == 1) ptx::tmem_alloc<256>(base + L.tslot);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = *reinterpret_cast<volatile uint32_t*>(s2m_smem + L.tslot);
    if (!rr) ptx::griddep_launch_dependents();  // the S3 launch may start its prologue as SMs free up

    if (warp == 0) {  // ---------------------------------------------------------- TMA producer
        ptx::griddep_wait();  // Z is the previous kernel's output
        if (ptx::elect_one()) {
            int ok_t = -1;  // highest token tile of Z known ready (pipelined layer)
            for (int j = 0; j < cnt; ++j) {
                int T, c;
                item(j, T, c);
                const int s = j % nst;
                if (j >= nst) ptx::mbar_wait(a_empty + 8 * s, ((j / nst) - 1) & 1);
                if (rr && T > ok_t) {  // the whole window of token tiles this item opens
                    const int w_end = min(tiles, (T / win + 1) * win);
#ifdef BLR_DEBUG_KNOBS
                    if (!(pipe->dbg & 1))
#endif
                    for (int t = ok_t + 1; t < w_end; ++t) ptx::pipe_acquire(pipe->wait_ctr + t + t0, pipe->wait_target);
                    ok_t = w_end - 1;
                }
                ptx::mbar_arrive_expect_tx(a_full + 8 * s, static_cast<uint32_t>(b1 * (FP8 ? 1024 : 2048)));
                // the b1 panels (l, T, c) in ONE tensor copy: Z viewed (64, 16, tiles*r/8, b1),
                // box (64, 16, 1, b1) -> smem [l][2 KB] (fp8: 1-KB panels, 64-B rows)
                if (rr && pipe->l2_in)
                    ptx::tma_load_4d_hint(base + L.a + s * L.a_bytes, &tmZ, a_full + 8 * s, 0, 0, (T + t0) * nchunks + c, 0,
                                          ptx::l2_policy(pipe->l2_in));
                else
                    ptx::tma_load_4d(base + L.a + s * L.a_bytes, &tmZ, a_full + 8 * s, 0, 0, (T + t0) * nchunks + c, 0);
            }
        }
        __syncwarp();
    } else if (warp == 1) {  // ------------------------------------------------ MMA issuer
        const uint32_t idesc = ptx::idesc_f16(128, static_cast<uint32_t>((b2 + 1) & ~1) * 8);
        for (int j = 0; j < cnt; ++j) {
            const int s = j % nst, bb = j % NB, wb = j & 1, acc = j & 1;
            if (j >= 2) ptx::mbar_wait(d_empty + 8 * acc, ((j >> 1) - 1) & 1);
            if constexpr (FP8) ptx::mbar_wait(w_full + 8 * wb, (j >> 1) & 1);
            else ptx::mbar_wait(a_full + 8 * s, (j / nst) & 1);
            ptx::mbar_wait(b_full + 8 * bb, (j / NB) & 1);
            ptx::tc_fence_after();
            if (ptx::elect_one()) {
                const uint32_t a0 = FP8 ? base + L.a16 + wb * b1p * 2048 : base + L.a + s * L.a_bytes;
                const uint32_t b0 = base + L.b + bb * L.b_bytes;
                for (int kk = 0; kk < b1p / 2; ++kk) {
                    // A: core matrices (t/8, l) at l*2048 + (t/8)*128 -> LBO (K) 2048, SBO (M) 128
                    // B: core matrices (k, l) at k*(b1p*128) + l*128  -> LBO (K) 128, SBO (N) b1p*128
                    const uint64_t ad = ptx::smem_desc(a0 + kk * 4096, 2048, 128, 0);
                    const uint64_t bd = ptx::smem_desc(b0 + kk * 256, 128, b1p * 128, 0);
                    ptx::mma_bf16(tmem + acc * 128, ad, bd, idesc, kk > 0 ? 1u : 0u);
                }
                if constexpr (FP8) ptx::mma_commit(w_empty + 8 * wb);
                else ptx::mma_commit(a_empty + 8 * s);
                ptx::mma_commit(b_empty + 8 * bb);
                ptx::mma_commit(d_full + 8 * acc);
            }
            __syncwarp();
        }
    } else if (warp < 4 || (FP8 && warp >= 8)) {  // --- B_c builders (warps 2-3); FP8: Z widening (+ warps 8-11)
        const bool builder = warp < 4;
        const int tb = builder ? threadIdx.x - 64 : 64 + (threadIdx.x - 256);  // converter index
        const uint32_t sbo = static_cast<uint32_t>(b1p) * 128;
        for (int j = 0; j < cnt; ++j) {
            int T, c;
            item(j, T, c);
            const int bb = j % NB, wb = j & 1;
            if (builder) {
                if (j >= NB) ptx::mbar_wait(b_empty + 8 * bb, ((j / NB) - 1) & 1);
                const uint32_t b0 = base + L.b + bb * L.b_bytes;
                int Tp = 0, cp = -1;
                if (j >= NB) item(j - NB, Tp, cp);  // the item that last used this buffer
                for (int lk = tb; lk < b1 * b2 && c != cp; lk += 64) {
                    const int l = lk / b2, k = lk - l * b2;
                    const uint4 w = __ldg(reinterpret_cast<const uint4*>(S + static_cast<long long>(lk) * r + c * 8));
                    const uint32_t cm = b0 + k * sbo + l * 128;  // core matrix (k, l): diag at rho*18 B
                    // every core matrix starts on bank 0, so entry rho's bank depends on rho alone:
                    // lane-rotated rho order -> 8 distinct banks per store (4-way instead of 32-way)
#pragma unroll
                    for (int e8 = 0; e8 < 8; ++e8) {
                        const int rho = (e8 + lane) & 7;
                        const uint32_t wd = (rho & 4) ? ((rho & 2) ? w.w : w.z) : ((rho & 2) ? w.y : w.x);
                        const float f = __uint_as_float((rho & 1) ? (wd & 0xFFFF0000u) : (wd << 16));
                        ptx::st_shared_u16(cm + rho * 18, __half_as_ushort(__float2half_rn(f)));
                    }
                }
                ptx::fence_async_smem();  // generic-proxy writes -> visible to the tensor core
                ptx::mbar_arrive(b_full + 8 * bb);
            }
            if constexpr (FP8) {
                // widen the item's b1 e4m3 panels (1 KB) into fp16 panels (2 KB) of buffer wb
                const int s = j % nst;
                ptx::mbar_wait(a_full + 8 * s, (j / nst) & 1);
                if (j >= 2) ptx::mbar_wait(w_empty + 8 * wb, ((j >> 1) - 1) & 1);
                const uint32_t src = base + L.a + s * L.a_bytes, dst = base + L.a16 + wb * b1p * 2048;
                for (int e = tb; e < b1 * 128; e += NCONV) {  // one 8-value panel row per step
                    const uint2 v = ptx::ld_shared_v2u32(src + e * 8);
                    uint4 o;
                    o.x = ptx::e4m3x2_to_f16x2(static_cast<uint16_t>(v.x));
                    o.y = ptx::e4m3x2_to_f16x2(static_cast<uint16_t>(v.x >> 16));
                    o.z = ptx::e4m3x2_to_f16x2(static_cast<uint16_t>(v.y));
                    o.w = ptx::e4m3x2_to_f16x2(static_cast<uint16_t>(v.y >> 16));
                    ptx::st_shared_v4(dst + e * 16, o);
                }
                ptx::fence_async_smem();
                ptx::named_bar_sync(3, NCONV);  // every converter is done reading the raw slot
                if (tb == 0) ptx::mbar_arrive(a_empty + 8 * s);
                ptx::mbar_arrive(w_full + 8 * wb);
            }
        }
    } else if (warp < 8) {  // ------------------------------------------------ epilogue (warps 4-7)
        const int q = warp & 3;  // TMEM lane quarter
        const int row = q * 32 + lane;
        const bool issuer = (warp == 4 && lane == 0);
        // pipelined layer: token tiles of the last S2_SIG_LAG items (a store's completion is
        // awaited S2_SIG_LAG items later, so the issuer never waits out a store's full latency)
        int sig_t[S2_SIG_LAG];
#pragma unroll
        for (int e = 0; e < S2_SIG_LAG; ++e) sig_t[e] = -1;
        ptx::griddep_wait();  // Z'' may still be read by the previous kernel
        for (int j = 0; j < cnt; ++j) {
            int T, c;
            item(j, T, c);
            const int acc = j & 1, cb = j & 1;
            ptx::mbar_wait(d_full + 8 * acc, (j >> 1) & 1);
            ptx::tc_fence_after();
            uint32_t v[8 * MAXB2];
            const uint32_t taddr = tmem + (static_cast<uint32_t>(q * 32) << 16) + acc * 128;
#pragma unroll
            for (int g = 0; g < MAXB2 / 4; ++g)
                if (g * 4 < b2) ptx::tmem_ld_x32(taddr + g * 32, *reinterpret_cast<uint32_t(*)[32]>(&v[g * 32]));
            ptx::tmem_wait_ld();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(d_empty + 8 * acc);
            // staging buffer cb: the bulk store issued from it two items ago must have read it
            if (issuer) ptx::bulk_wait_read<1>();
            ptx::named_bar_sync(1, 128);
            const uint32_t c0 = base + L.c + cb * L.c_bytes + row * 16;
#pragma unroll
            for (int k = 0; k < MAXB2; ++k) {
                if (k < b2) {
                    uint4 o;
                    o.x = ptx::pack_bf16x2(__uint_as_float(v[8 * k + 0]), __uint_as_float(v[8 * k + 1]));
                    o.y = ptx::pack_bf16x2(__uint_as_float(v[8 * k + 2]), __uint_as_float(v[8 * k + 3]));
                    o.z = ptx::pack_bf16x2(__uint_as_float(v[8 * k + 4]), __uint_as_float(v[8 * k + 5]));
                    o.w = ptx::pack_bf16x2(__uint_as_float(v[8 * k + 6]), __uint_as_float(v[8 * k + 7]));
                    ptx::st_shared_v4(c0 + k * 2048, o);
                }
            }
            ptx::fence_async_smem();
            ptx::named_bar_sync(1, 128);
            if (issuer) {
                // panels (k, T, c) for all k in ONE tensor store (Z'' viewed like Z)
                if (rr && pipe->l2_out)
                    ptx::tma_store_4d_hint(&tmZpp, base + L.c + cb * L.c_bytes, 0, 0, (T + t0o) * nchunks + c, 0,
                                           ptx::l2_policy(pipe->l2_out));
                else
                    ptx::tma_store_4d(&tmZpp, base + L.c + cb * L.c_bytes, 0, 0, (T + t0o) * nchunks + c, 0);
                ptx::bulk_commit();
                if (rr) {  // item j - S2_SIG_LAG's stores have landed: signal its token tile
#ifdef BLR_DEBUG_KNOBS
                    if (!(pipe->dbg & 2))
#endif
                    ptx::bulk_wait<S2_SIG_LAG>();
                    if (sig_t[0] >= 0) ptx::pipe_release(pipe->sig_ctr + sig_t[0]);
#pragma unroll
                    for (int e = 0; e + 1 < S2_SIG_LAG; ++e) sig_t[e] = sig_t[e + 1];
                    sig_t[S2_SIG_LAG - 1] = T + t0o;
                    // last item of this CTA's share of a window: flush every pending signal (the
                    // producer may next block on the following window, and with S1 back-pressure an
                    // unreleased signal here would close a wait cycle)
                    int Tn = -1, cn = 0;
                    if (j + 1 < cnt) item(j + 1, Tn, cn);
                    if (j + 1 >= cnt || Tn / win != T / win) {
                        ptx::bulk_wait<0>();
#pragma unroll
                        for (int e = 0; e < S2_SIG_LAG; ++e) {
                            if (sig_t[e] >= 0) ptx::pipe_release(pipe->sig_ctr + sig_t[e]);
                            sig_t[e] = -1;
                        }
                    }
                }
            }
        }
        if (issuer) {
            ptx::bulk_wait<0>();
            if (rr)
#pragma unroll
                for (int e = 0; e < S2_SIG_LAG; ++e)
                    if (sig_t[e] >= 0) ptx::pipe_release(pipe->sig_ctr + sig_t[e]);
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc<256>(tmem);
    }
    (void)Z;
}

template <int MAXB2, bool FP8 = false>
__global__ void __launch_bounds__(s2m_threads<FP8>(), MAXB2 <= 8 ? 2 : 1)
    blast_s2_mma_kernel(const __grid_constant__ CUtensorMap tmZ, const __grid_constant__ CUtensorMap tmZpp,
                        const void* __restrict__ Z, __nv_bfloat16* __restrict__ Zpp,
                        const __nv_bfloat16* __restrict__ S, int n_tok, int b1, int b2, int r, int order,
                        int t0 = 0, int t0o = 0) {
    // t0 / t0o: first 128-token tile of Z this launch reads / of Z'' it writes (token-chunked
    // S1 -> S2); the items' tiles are numbered from 0
    extern __shared__ __align__(1024) uint8_t s2m_smem[];
    s2_body<MAXB2, FP8>(tmZ, tmZpp, Z, Zpp, S, n_tok, b1, b2, r, order, t0, t0o, s2m_smem,
                        static_cast<int>(blockIdx.x), static_cast<int>(gridDim.x), nullptr);
}

}  // namespace blr

namespace blr {

// ------------------------------------------------------------ pipelined BLAST layer (one launch) ----
// Y = BLAST(X) as ONE persistent launch whose CTA pairs take one of three roles:
//   S1  Z_l = X_l V_l            gemm_body<GEMM, 2, 2>  tile-blocked fp16 Z
//   S2  Z''_k = sum_l S_lk Z_l    s2_body<16>            tile-blocked bf16 Z''     (Fig. 6)
//   S3  Y_k = Z''_k U_k           gemm_body<GEMM, 2, 0>  Y
// All three walk the tokens in 128-row-tile order and hand each token tile to the next stage
// through per-tile ready counters in global memory (release/acquire, ptx::pipe_*), so a token
// tile's Z and Z'' are consumed while they are still in the 126-MB L2 -- the round trip through
// HBM the paper identifies (Table 2) becomes L2 traffic -- and S2's memory-bound
// work overlaps S1's and S3's tensor-core work instead of running between them.
// Roles are handed out by arrival order (an atomic ticket per cluster), S1 first, then S2, then
// S3: every wait is on work held by an earlier ticket, i.e. by a CTA that is already resident, so
// the launch cannot deadlock however many of its CTAs are co-resident.  The grid never triggers
// its dependent launch early (a dependent's CTAs could otherwise take the SMs later tickets need).
struct PipeArgs {
    unsigned int* ctr;   // [0] ticket, [1 .. tiles] Z ready, [1 + tiles .. 2 tiles] Z'' ready
    int n1, n2, n3;      // clusters (CTA pairs) per role
    const void* Z;       // S2 operands
    __nv_bfloat16* Zpp;
    const __nv_bfloat16* S;
    int n_tok, b1, b2, r;
    unsigned int z_target;  // S1 signals per token tile (b1 x N tiles x 2 column halves)
    int tiles_pad;          // counters per stage (128-token tiles of the pairs' 256-row tiles)
    uint32_t ticket_off;    // dynamic-smem byte offset of the role ticket
    int win;                // S2 role: token tiles per window
    int dbg;                // BLR_DEBUG_KNOBS builds: S2Pipe::dbg
    int l2_z, l2_zz;        // S2 role's L2 hints: Z loads, Z'' stores
};

constexpr uint32_t PIPE_SMEM_ALIGN = 1024;

__global__ void __launch_bounds__(NUM_THREADS, 1)
    blast_pipe_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmV,
                      const __grid_constant__ CUtensorMap tmZst, const __grid_constant__ CUtensorMap tmZ,
                      const __grid_constant__ CUtensorMap tmZpp, const __grid_constant__ CUtensorMap tmA3,
                      const __grid_constant__ CUtensorMap tmU, const __grid_constant__ CUtensorMap tmY,
                      const __grid_constant__ CUtensorMap tmV2, const __grid_constant__ CUtensorMap tmU2,
                      const KParams p1, const KParams p3, const PipeArgs pa) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + (PIPE_SMEM_ALIGN - 1)) &
                                               ~uintptr_t(PIPE_SMEM_ALIGN - 1));
    // the role ticket lives past every role's layout (no static smem: it would cost 1-2 KB)
    volatile uint32_t* s_ticket = reinterpret_cast<volatile uint32_t*>(smem_raw + pa.ticket_off);
    const uint32_t crank = ptx::cluster_ctarank();
    if (crank == 0 && threadIdx.x == 0) {
        const uint32_t t = atomicAdd(pa.ctr, 1u);
        *s_ticket = t;
        ptx::st_cluster_u32(ptx::smem_u32(smem_raw + pa.ticket_off), 1u, t);  // the peer CTA's copy
    }
    ptx::cluster_sync();
    const int ticket = static_cast<int>(*s_ticket);
    if (ticket < pa.n1) {
        gemm_body<KIND_GEMM, 2, 2>(tmX, tmV, tmZst, tmV2, p1, smem, 2 * ticket + static_cast<int>(crank), 2 * pa.n1);
    } else if (ticket < pa.n1 + pa.n2) {
        S2Pipe sp;
        sp.wait_ctr = pa.ctr + 1;
        sp.wait_target = pa.z_target;
        sp.sig_ctr = pa.ctr + 1 + pa.tiles_pad;
        sp.win = pa.win;
        sp.dbg = pa.dbg;
        sp.l2_in = pa.l2_z;
        sp.l2_out = pa.l2_zz;
        // (320 threads: warps 8-9 of the S2 role only join its barriers)
        s2_body<16, false>(tmZ, tmZpp, pa.Z, pa.Zpp, pa.S, pa.n_tok, pa.b1, pa.b2, pa.r, 1, 0, 0, smem,
                           2 * (ticket - pa.n1) + static_cast<int>(crank), 2 * pa.n2, &sp);
    } else {
        gemm_body<KIND_GEMM, 2, 0>(tmA3, tmU, tmY, tmU2, p3, smem, 2 * (ticket - pa.n1 - pa.n2) + static_cast<int>(crank),
                                   2 * pa.n3);
    }
}

}  // namespace blr
