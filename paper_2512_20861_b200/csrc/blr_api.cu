// blr_api.cu -- C ABI of libblr.so (include/blr.h): host-side validation, plan selection,
// TMA tensor-map encoding and kernel launches.  No torch types, no host synchronization.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "../../include/blr.h"
#include "blr_kernels.cuh"
#include "blr_decode.cuh"
#include "blr_decode_tc.cuh"
#include "blr_fused.cuh"

namespace {

using blr::KParams;

constexpr int SMEM_LIMIT = 232448;  // 227 KB opt-in per CTA on sm_100
constexpr int SMEM_SLACK = 1024;    // runtime 1024-B realignment of the dynamic smem base

struct DevInfo {
    int ok = 0;
    int sm_count = 0;
    int cc_major = 0, cc_minor = 0;
};

std::mutex g_mu;
DevInfo g_dev[64];
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
bool g_attr_set[32][64] = {};  // kernel attribute set, per (kernel variant, device)
thread_local int t_last_launches = 0;
thread_local void** t_prof_events = nullptr;
thread_local int t_prof_cap = 0;
thread_local int t_prof_n = 0;

blr_status device_info(DevInfo& out, int& dev) {
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return BLR_ERR_CUDA;
    std::lock_guard<std::mutex> lk(g_mu);
    DevInfo& d = g_dev[dev];
    if (!d.ok) {
        if (cudaDeviceGetAttribute(&d.sm_count, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&d.cc_major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess ||
            cudaDeviceGetAttribute(&d.cc_minor, cudaDevAttrComputeCapabilityMinor, dev) != cudaSuccess)
            return BLR_ERR_CUDA;
        d.ok = 1;
    }
    if (!g_encode) {
        void* fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess || fn == nullptr)
            return BLR_ERR_CUDA;
        g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    out = d;
    if (!(d.cc_major == 10 && d.cc_minor == 0)) return BLR_ERR_ARCH;
    return BLR_OK;
}

// Tensor map of rank R (dt: 0 bf16, 1 fp32, 2 fp16): dims[0] innermost, strides in bytes for
// dims 1..R-1.
bool encode(CUtensorMap* m, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides,
            const uint32_t* box, CUtensorMapSwizzle sw, int dt = 0) {
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    const CUtensorMapDataType t = dt == 1   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                  : dt == 2 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                  : dt == 3 ? CU_TENSOR_MAP_DATA_TYPE_UINT8   // e4m3 bytes
                                            : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    CUresult r = g_encode(m, t, rank, const_cast<void*>(ptr),
                          reinterpret_cast<const cuuint64_t*>(dims), reinterpret_cast<const cuuint64_t*>(strides),
                          reinterpret_cast<const cuuint32_t*>(box), estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                          CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline int64_t rup(int64_t a, int64_t b) { return cdiv(a, b) * b; }
inline bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// S3 contractions shorter than this keep the intermediate as a compensated pair hi|lo of bf16
// (hi = bf16(z), lo = bf16(z - hi)); S3 then runs over [hi | lo] against the same U rows.
// A single bf16 rounding of one O(1) term can otherwise exceed the north_star per-element
// floor when only a handful of terms are summed.  No paper shape triggers it.
constexpr int64_t COMP_K_THRESHOLD = 128;
inline int comp_factor(int64_t k_s3) { return k_s3 < COMP_K_THRESHOLD ? 2 : 1; }

// BLAST runs S1 and S2 fused (b1 TMEM accumulators per token tile) when all b1 * r columns fit
// TMEM, so X is read once; otherwise S1 (grouped GEMM), S2 (streaming) and S3 run separately.
// The split path's S1 output Z is stored fp16 (RNE, 11-bit significand: half the intermediate
// traffic of fp32, rounding error ~1/8 of a bf16 rounding; finite range |Z| <= 65504), R13.

inline bool blast_fused(int64_t b1, int64_t r) {
    const char* e = getenv("BLR_BLAST_PATH");
    if (e && !strcmp(e, "fused")) return true;
    if (e && !strcmp(e, "split")) return false;
    return b1 * rup(r, 16) <= blr::TMEM_COLS;
}

// Swizzle for a staged-store box whose rows are `bytes` long (must match the kernel's XOR mask).
struct Swz {
    CUtensorMapSwizzle mode;
    uint32_t mask;
};
Swz pick_swz(int64_t bytes) {
    if (bytes == 128) return {CU_TENSOR_MAP_SWIZZLE_128B, 7u};
    if (bytes == 64) return {CU_TENSOR_MAP_SWIZZLE_64B, 3u};
    if (bytes == 32) return {CU_TENSOR_MAP_SWIZZLE_32B, 1u};
    return {CU_TENSOR_MAP_SWIZZLE_NONE, 0u};
}

// Staged-store chunk width: the largest multiple of 8 <= 64 dividing n (n a multiple of 8).
// Fewer, wider chunks beat swizzle-friendly power-of-two widths (measured: 48-wide chunks with
// 2-way staging conflicts are faster than 16/32-wide swizzled ones for r' = 96 / 48).
int chunk_width(int n) {
    int cw = std::min(64, n);
    while (n % cw || cw % 8) --cw;
    return cw;
}

// Fill B-operand staging parameters for p.BN columns of this CTA (one half of the tile when
// p.n_mma == 2).  allow_sw64: MN-major columns may be staged in 32-column 64-B-swizzled boxes
// when that loads fewer columns than 64-column boxes (e.g. 88 -> 96 instead of 128).
void set_b_staging(KParams& p, bool mn_major, bool allow_sw64 = false) {
    if (p.n_mma < 1) p.n_mma = 1;
    p.b_mn_major = mn_major ? 1 : 0;
    if (mn_major) {
        // B stored [K][N]: boxes of 64 N-elements (128 B rows) x BK K-rows, 128-B swizzle.
        // UMMA MN-major SW128 canonical layout: 64-element MN atoms LBO apart, 8-row K groups
        // SBO = 1024 B apart; +16 K-rows = +2048 B per UMMA_K step.  (SW64: 32-element atoms,
        // 512 B per 8 K rows, +1024 B per UMMA_K step.)
        const bool sw64 = allow_sw64 && cdiv(p.BN, 32) * 32 < cdiv(p.BN, 64) * 64;
        p.b_box_n = sw64 ? 32 : 64;
        p.b_boxes = static_cast<int>(cdiv(p.BN, p.b_box_n));
        p.b_half_bytes = static_cast<uint32_t>(p.b_boxes * p.b_box_n * blr::BK * 2);
        p.b_lbo = p.b_box_n * 2 * blr::BK;
        p.b_sbo = sw64 ? 512 : 1024;
        p.b_layout = sw64 ? blr::ptx::LAYOUT_SW64 : blr::ptx::LAYOUT_SW128;
        p.b_kstep = sw64 ? 16 * 64 : 16 * 128;
    } else {
        // B stored [N][K]: BN rows x 64 K-elements, K-major SW128 like A.
        p.b_box_n = p.BN;
        p.b_boxes = 1;
        p.b_half_bytes = static_cast<uint32_t>(rup(static_cast<int64_t>(p.BN) * blr::BK * 2, 1024));
        p.b_lbo = 16;
        p.b_sbo = 1024;
        p.b_layout = blr::ptx::LAYOUT_SW128;
        p.b_kstep = 32;
    }
    p.b_stage_bytes = p.n_mma * p.b_half_bytes;
}

// Programmatic dependent launch between the library's kernels (BLR_NO_PDL=1 disables).
bool pdl_enabled() {
    const char* e = getenv("BLR_NO_PDL");
    return !(e && e[0] == '1');
}

thread_local int t_smem_reserve = 0;  // bytes a planning caller keeps free (pipelined layer: its ticket)
bool fits(const KParams& p) {
    return blr::smem_layout(p).total + SMEM_SLACK + t_smem_reserve <= static_cast<uint32_t>(SMEM_LIMIT);
}

// Decide weight-stationary vs streaming, staging buffers and ring depth.  `allow_resident`:
// the kind supports a resident B slice; `stage_buf_bytes` > 0: bytes of one staging buffer.
bool finish_plan(KParams& p, bool allow_resident, int stage_buf_bytes, int sms) {
    const int cols = p.n_sub * p.BN;
    if (cols > blr::TMEM_COLS) return false;
    p.acc_bufs = (2 * cols <= blr::TMEM_COLS) ? 2 : 1;
    // wide tiles (48-KB stages): a 128-entry tile table leaves room for a fourth ring stage
    if (p.n_mma == 2) p.tab_n = 128;
    // weight-stationary plans are opt-in (BLR_RESIDENT=1): with the lean producer, streamed CTA-pair
    // plans measured as fast or faster on every workload (C4 8.21 -> 7.61 ms, C3 0.93 -> 0.84 ms,
    // C2 / C4M / C5V-256 unchanged; in-process A/B)
    const char* e = getenv("BLR_RESIDENT");
    const bool reuse = p.tiles_m >= 2 && p.n_sub == 1 && p.kb_half <= blr::MAX_BRES - 1 && e && e[0] == '1';
    const char* kb_env = getenv("BLR_KBOX");
    const char* sc_env = getenv("BLR_SCORE");
    const char* bufs_env = getenv("BLR_BUFS");
    // long persistent runs (>= 2 tiles per CTA) are steady-state pipelines: score the K blocks in
    // flight behind the stage the MMA is consuming, (stages - 1) * kbox (Llama-7B Monarch down S1
    // 3.67 -> 3.05 ms); short one-tile kernels keep the plain ring depth (GPT2-S c_proj S1 24 vs 28 us)
    const bool score_new = sc_env ? sc_env[0] != '0' : p.total_tiles >= 2 * sms;
    const int kbox_max = (kb_env && kb_env[0] == '1') ? 1 : (p.k_blocks >= 2 ? 2 : 1);
    // Per residency mode, pick (kbox, staging buffers, stages) maximising the 64-wide K blocks in
    // flight (latency hiding of the operand ring); prefer two staging buffers on ties.
    for (int resident = (allow_resident && reuse) ? 1 : 0; resident >= 0; --resident) {
        int best_score = -1;
        KParams best = p;
        const int kbox_min = (kb_env && kb_env[0] == '2' && p.k_blocks >= 2) ? 2 : 1;  // BLR_KBOX=2 forces 2
        for (int kbox = kbox_max; kbox >= kbox_min; --kbox) {
            for (int bufs = 2; bufs >= 1; --bufs) {
                if (bufs_env && atoi(bufs_env) != bufs) continue;
                KParams q = p;
                q.b_resident = resident;
                q.kbox = kbox;
                q.stage_bufs = bufs;
                if (stage_buf_bytes > 0) q.stage_warp_bytes = static_cast<uint32_t>(bufs * stage_buf_bytes);
                for (q.stages = blr::MAX_STAGES; q.stages >= 2; --q.stages)
                    if (fits(q)) break;
                if (q.stages < 2 || !fits(q) || (resident && q.stages < 3)) continue;
                const int score = score_new ? std::min((q.stages - 1) * kbox, 8) * 4 + (bufs == 2 ? 1 : 0) + (kbox == 2 ? 2 : 0)
                                            : std::min(q.stages * kbox, 8) * 4 + (bufs == 2 ? 1 : 0) + (kbox == 2 ? 2 : 0);
                if (score > best_score) {
                    best_score = score;
                    best = q;
                }
            }
        }
        if (best_score >= 0) {
            p = best;
            // BLR_ORDER=1: streaming plans run the N blocks of one (token tile, group) back to back
            // on one CTA (A re-read from L2 while hot).  Measured slower than round robin, where the
            // CTAs sharing an A tile load it at the same time (C4 8.31 -> 8.37 ms, C4M 6.52 -> 6.80 ms)
            const char* oe = getenv("BLR_ORDER");
            p.nb_runs = (!resident && p.tiles_n >= 2 && oe && oe[0] == '1') ? 1 : 0;
            // slice ownership with lockstep token walks when every slice gets >= 1 CTA (unit)
            const int slices = p.groups * p.tiles_n;
            p.cps = 0;
            if (resident && slices <= sms) p.cps = std::max(1, std::min(sms / slices, p.tiles_m));
            return true;
        }
    }
    return false;
}

thread_local unsigned long long* t_trace = nullptr;  // debug trace buffer (blr_debug_trace)

// Profiling-hook event record: inside stream capture the event must be an *external* record node
// to carry a timestamp when the graph replays; outside capture a plain record.
cudaError_t prof_record(void* ev, cudaStream_t st) {
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    if (cudaStreamIsCapturing(st, &cs) != cudaSuccess) return cudaErrorUnknown;
    return cudaEventRecordWithFlags(static_cast<cudaEvent_t>(ev), st,
                                    cs == cudaStreamCaptureStatusActive ? cudaEventRecordExternal : cudaEventRecordDefault);
}

template <int KIND, int PAIR, int OUTF = 0>
blr_status launch(const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c, const KParams& p_in,
                  const DevInfo& d, int dev, cudaStream_t stream, const CUtensorMap* b2 = nullptr) {
    KParams p = p_in;
    p.trace = t_trace;
    p.first = t_last_launches == 0 ? 1 : 0;  // first launch of this API call (PDL ordering, kernel)
    // K blocks issued as one unrolled MMA burst (all plans: with the lean producer the burst no longer
    // measured slower on the streamed pair plans)
    p.mma_burst = 1;
    if (const char* e = getenv("BLR_BURST")) p.mma_burst = atoi(e);
    p.fast_prod = 1;
    if (const char* e = getenv("BLR_FASTPROD")) p.fast_prod = atoi(e);
#ifdef BLR_DEBUG_KNOBS
    if (const char* e = getenv("BLR_DBG")) p.dbg = atoi(e);  // debug experiments only
    if (const char* e = getenv("BLR_DBG_LAUNCH"); e && atoi(e) != t_last_launches) p.dbg = 0;  // only launch k
#endif
    if (t_trace) t_trace += 128 * 256;  // next launch traces into the next slot
    auto kfn = blr::blr_gemm_kernel<KIND, PAIR, OUTF>;
    const blr::SmemLayout L = blr::smem_layout(p);
    const int smem = static_cast<int>(L.total + SMEM_SLACK);
    {
        std::lock_guard<std::mutex> lk(g_mu);
        const int slot = OUTF ? 6 + 2 * (OUTF - 1) + (PAIR - 1) : KIND + 3 * (PAIR - 1);  // 0..11
        if (!g_attr_set[slot][dev]) {
            if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT) != cudaSuccess)
                return BLR_ERR_CUDA;
            g_attr_set[slot][dev] = true;
        }
    }
    const int csz = PAIR * std::max(1, p.mc);  // CTAs per cluster
    int units = d.sm_count / csz;              // CTAs (pairs, clusters) that fit one wave
    if (csz > 2) {
        // clusters of 4+ CTAs must fit inside a GPC: ask how many can be co-resident
        static int cached[17] = {};
        std::lock_guard<std::mutex> lk(g_mu);
        if (!cached[csz]) {
            cudaLaunchConfig_t oc = {};
            oc.gridDim = dim3(csz);
            oc.blockDim = dim3(blr::NUM_THREADS);
            oc.dynamicSmemBytes = SMEM_LIMIT;
            cudaLaunchAttribute oa[1];
            oa[0].id = cudaLaunchAttributeClusterDimension;
            oa[0].val.clusterDim.x = csz;
            oa[0].val.clusterDim.y = 1;
            oa[0].val.clusterDim.z = 1;
            oc.attrs = oa;
            oc.numAttrs = 1;
            int nc = 0;
            if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT) != cudaSuccess ||
                cudaOccupancyMaxActiveClusters(&nc, kfn, &oc) != cudaSuccess || nc <= 0)
                return BLR_ERR_CUDA;
            cached[csz] = nc;
        }
        units = std::min(units, cached[csz]);
    }
    int grid = static_cast<int>(std::min<int64_t>(p.total_tiles, units)) * csz;
    if (p.b_resident && p.cps > 0) grid = p.groups * p.tiles_n * p.cps * PAIR;
    else if (p.b_resident) grid = std::min(units, p.groups * p.tiles_n) * PAIR;  // slice round-robin
    if (const char* pe = getenv("BLR_PLAN"); pe && pe[0] == '1')
        fprintf(stderr,
                "[blr plan] kind=%d pair=%d mc=%d grid=%d tiles=%dx%dx%d BN=%d mma=%d bbox=%d kblk=%d kbox=%d stages=%d res=%d "
                "cps=%d bufs=%d acc=%d cbox=%d split=%d lastn=%d smem=%d\n",
                KIND, PAIR, p.mc, grid, p.tiles_m, p.groups, p.tiles_n, p.BN, p.n_mma, p.b_box_n, p.k_blocks, p.kbox, p.stages,
                p.b_resident, p.cps, p.stage_bufs, p.acc_bufs, p.c_box_w, p.split_rel, p.last_nb, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(blr::NUM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = csz;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = PAIR == 2 ? 2 : 1;
    const bool prof = t_prof_events != nullptr && 2 * t_prof_n + 1 < t_prof_cap;
    if (prof && prof_record(t_prof_events[2 * t_prof_n], stream) != cudaSuccess)
        return BLR_ERR_CUDA;
    if (cudaLaunchKernelEx(&cfg, kfn, a, b, c, b2 ? *b2 : b, p) != cudaSuccess) return BLR_ERR_CUDA;
    if (prof) {
        if (prof_record(t_prof_events[2 * t_prof_n + 1], stream) != cudaSuccess)
            return BLR_ERR_CUDA;
        ++t_prof_n;
    }
    ++t_last_launches;
    return BLR_OK;
}

// N tile: <= 256 columns, multiple of 16, balanced.  While the grid would leave SMs idle, split
// N further (down to 64) -- but only toward a width whose B slice (K x BN) can stay resident,
// since in streaming mode every extra N tile re-reads the whole A tile.
int choose_bn(int64_t N, int64_t K, int64_t other_tiles, int64_t groups, int sms, int pair, bool blocked = false) {
    int64_t tiles = cdiv(N, 256);
    int bn = static_cast<int>(rup(cdiv(N, tiles), 16));
    // split while the grid leaves SMs idle, but never past one wave (a partial second wave
    // doubles the makespan of a latency-bound kernel)
    while (bn > 64 && other_tiles * cdiv(N, bn) < sms) {
        ++tiles;
        const int nb = static_cast<int>(rup(cdiv(N, tiles), 16));
        if (nb < 64 || other_tiles * cdiv(N, nb) > sms) break;
        bn = nb;
    }
    // (splitting also when the slice cannot stay resident: the re-read A tile comes from L2, and
    //  per-SM TMA ingress, not L2 or HBM, bounds these short kernels -- measured on GPT2-S c_proj)
    //
    // Weight-stationary plans (short K, many token tiles) run one CTA per (group, N block) slice
    // in lockstep, so the slice count decides how many SMs work: pick the N split that fills
    // the SMs best, discounted by the padding of the last N tile.  (Llama-7B BLAST gate S1,
    // 16 groups x N = 1488: BN = 256 gave 96 slices on 148 SMs; BN = 176 gives 144.)
    const int64_t tiles_m = other_tiles / std::max<int64_t>(groups, 1);
    const char* fe = getenv("BLR_BN_FILL");
    if (pair == 1 && tiles_m >= 8 && cdiv(K, blr::BK) <= blr::MAX_BRES - 1 && !(fe && fe[0] == '0')) {
        // score = ideal per-SM work / the busiest CTA's work (token tiles x BN columns)
        auto score = [&](int b) {
            if (rup(b, 64) * rup(K, blr::BK) * 2 > (144 << 10)) return -1.0;  // slice must stay resident
            const int64_t slices = groups * cdiv(N, b);
            const int64_t busiest = slices <= sms ? cdiv(tiles_m, std::min<int64_t>(sms / slices, tiles_m)) * b
                                                  : cdiv(slices, sms) * tiles_m * b;
            return static_cast<double>(groups * tiles_m * N) / sms / static_cast<double>(busiest);
        };
        // only for an underfilled plan (fewer slices than SMs, one CTA per slice), and only toward
        // widths whose epilogue chunks stay >= 32 columns (BN = 176 -> 16-column chunks measured
        // 1.6x slower on that S1)
        const int64_t slices0 = groups * cdiv(N, bn);
        double best = score(bn);
        int best_bn = bn;
        if (best > 0 && slices0 < sms && 2 * slices0 > sms) {
            for (int64_t tn = cdiv(N, 256); tn <= cdiv(N, 128); ++tn) {
                const int b = static_cast<int>(rup(cdiv(N, tn), 16));
                if (!blocked && chunk_width(b) < 32) continue;  // (tile-blocked outputs store BN/2-wide chunks)
                const double s = score(b);
                if (s > best + 0.05) {
                    best = s;
                    best_bn = b;
                }
            }
            bn = best_bn;
        }
    }
    (void)pair;
    return bn;
}

struct OutMap {  // 4-D view (N, comp, groups, rows) of a GEMM phase's output
    void* ptr;
    int f32;               // output type: 0 bf16, 2 fp16 (BLAST split-path Z), 3 e4m3 (FP8 Z, row f4)
    int64_t comp;          // 1, or 2 for a compensated [hi | lo] intermediate
    int64_t comp_stride;   // elements between hi and lo
    int64_t group_stride;  // elements between groups
    int64_t row_stride;    // elements between rows
    int blocked = 0;       // 1: tile-blocked [g][T][N/8][128][8] (BLAST Z with the tensor-core S2)
    int64_t col_stride = 0;  // > 0: element (t, g, c) at t*row_stride + g*group_stride + c*col_stride,
                             //      stored directly (Monarch transposed output order)
};

// One plain GEMM phase: out[g](t, c) = sum_k A[g](t, k) B[g](k, c), K-major A.
//   A map: a_gmid ? (K*comp, groups, rows) : (K*comp, rows, groups) with the given strides.
//   comp == 2: A rows hold [hi | lo] (lo at column offset K) multiplying the same B rows.
// Plan one GEMM phase for CTA-pair mode `pair` (1 or 2).  Returns false if nothing fits.
// wide: a CTA-pair tile of up to 512 columns as two MMAs per K step (KParams::n_mma), single
// accumulator buffer, streamed B only.
bool plan_gemm(KParams& p, int pair, const DevInfo& d, int a_gmid, int64_t n_tok, int64_t K, int64_t groups,
               int64_t N, bool b_mn_major, const OutMap& out, int comp, bool wide = false, int mc = 1,
               bool allow_res = true) {
    p = KParams{};
    p.a_gmid = a_gmid;
    p.n_tok = static_cast<int>(n_tok);
    p.mc = mc;
    p.tiles_m = static_cast<int>(cdiv(n_tok, blr::BM * pair * mc));
    p.n_mma = wide ? 2 : 1;
    if (wide) {  // N tiles of <= 512, halves multiples of 16 (per-CTA halves multiples of 8)
        p.BN = static_cast<int>(rup(cdiv(N, cdiv(N, 512)), 32));
        // 512-column tiles whose last one holds at most one half (it then runs as half 0 alone,
        // KParams::last_half): C4 gate S3's 688 = 512 + 176 instead of 2 x 352 (88-column per-CTA
        // halves are 2-3 TMA boxes each; whole 64-column slabs are one)
        const int64_t rem = N % 512;
        if (N > 512 && rem > 0 && rem <= 256) p.BN = 512;
    } else {
        p.BN = choose_bn(N, K, p.tiles_m * groups, groups, d.sm_count / pair, pair, out.blocked != 0);
        if (pair == 2 && (p.BN / 2) % 8) p.BN = static_cast<int>(rup(p.BN, 32));
        // pair tiles over an MN-major B: 256 columns (two whole 64-column slabs per CTA) so each K block
        // of B is ONE slab-view TMA op instead of two boxes -- the per-SM TMA op rate bounds these phases
        // (C4 gate S3 2.18 -> 2.08 ms, down S3 0.77 -> 0.73 ms with the padding of the last N tile;
        // BLR_SLAB=0 restores the balanced width)
        const char* se = getenv("BLR_SLAB");
        if (pair == 2 && b_mn_major && !wide && mc <= 1 && p.BN >= 192 && p.BN < 256 && N >= 512 && !(se && se[0] == '0'))
            p.BN = 256;
        if (const char* be = getenv("BLR_BN"); be && atoi(be) >= 16 * pair && atoi(be) <= 256)  // A/B experiments
            p.BN = atoi(be);
    }
    p.N = static_cast<int>(N);
    p.tiles_n = static_cast<int>(cdiv(N, p.BN));
    p.groups = static_cast<int>(groups);
    p.total_tiles = p.tiles_m * p.groups * p.tiles_n;
    p.kb_half = static_cast<int>(cdiv(K, blr::BK));
    p.k_blocks = p.kb_half * comp;
    p.a_lo_off = comp == 2 ? static_cast<int>(K) : 0;
    p.n_sub = 1;
    // B staging describes this CTA's share of one MMA's columns: all of them, or half in a CTA pair
    const int bn_full = p.BN;
    p.BN = bn_full / pair / p.n_mma;
    set_b_staging(p, b_mn_major, wide);
    p.BN = bn_full;
    p.out_lo_off = out.comp == 2 ? out.comp_stride : 0;
    p.out_ptr = out.ptr;
    p.out_gstride = out.group_stride;
    p.out_rs = out.row_stride;
    p.out_cs = static_cast<int>(out.col_stride);
    const int esz = 2;
    p.c_box_w = chunk_width(p.BN);
    while (p.c_box_w * esz > 128) p.c_box_w /= 2;  // staged rows <= 128 B
    // tile-blocked outputs (BLAST S1's Z) store whole panels: one BN/2-wide chunk per column half
    // (<= 128 columns, staged in 64-column passes), so no width is forced down to 16-column boxes
    const char* bce = getenv("BLR_BLK_CW_OLD");
    // -- only where the default chunking is narrow or leaves the two column halves unbalanced (an odd
    // chunk count): a wider staging chunk costs ring stages
    const bool unbalanced = (p.BN / p.c_box_w) % 2 == 1 || p.c_box_w < 32;
    if (out.blocked && unbalanced && (p.BN / 2) % 8 == 0 && p.BN / 2 <= 128 && !(bce && bce[0] == '1'))
        p.c_box_w = p.BN / 2;
    p.c_swz = out.blocked ? 0 : pick_swz(p.c_box_w * esz).mask;
    if (mc > 1 && !b_mn_major && (bn_full / p.n_mma / pair) % (8 * mc)) return false;  // K-major slices
    return finish_plan(p, allow_res && !wide && mc == 1, 32 * p.c_box_w * esz, d.sm_count / (pair * mc));
}

// A planned GEMM phase: parameters and tensor maps, encoded before anything is launched (so a
// planning or encoding error leaves the stream untouched, include/blr.h).
struct GemmPrep {
    KParams p;
    CUtensorMap ta, tb, tc;
    CUtensorMap tb2;  // slab view of an MN-major B (KParams::b_slab2), else a copy of tb
    int pair = 1;
    int outf = 0;  // 0 bf16, 1 fp16, 2 fp16 tile-blocked, 3 e4m3 tile-blocked
};

blr_status gemm_run(const GemmPrep& g, const DevInfo& d, int dev, cudaStream_t st) {
    if (g.outf == 3)
        return g.pair == 2 ? launch<blr::KIND_GEMM, 2, 3>(g.ta, g.tb, g.tc, g.p, d, dev, st, &g.tb2)
                           : launch<blr::KIND_GEMM, 1, 3>(g.ta, g.tb, g.tc, g.p, d, dev, st, &g.tb2);
    if (g.outf == 2)
        return g.pair == 2 ? launch<blr::KIND_GEMM, 2, 2>(g.ta, g.tb, g.tc, g.p, d, dev, st, &g.tb2)
                           : launch<blr::KIND_GEMM, 1, 2>(g.ta, g.tb, g.tc, g.p, d, dev, st, &g.tb2);
    if (g.outf == 1)
        return g.pair == 2 ? launch<blr::KIND_GEMM, 2, 1>(g.ta, g.tb, g.tc, g.p, d, dev, st, &g.tb2)
                           : launch<blr::KIND_GEMM, 1, 1>(g.ta, g.tb, g.tc, g.p, d, dev, st, &g.tb2);
    if (g.pair == 2) return launch<blr::KIND_GEMM, 2>(g.ta, g.tb, g.tc, g.p, d, dev, st, &g.tb2);
    return launch<blr::KIND_GEMM, 1>(g.ta, g.tb, g.tc, g.p, d, dev, st, &g.tb2);
}

// One plain GEMM phase: out[g](t, c) = sum_k A[g](t, k) B[g](k, c), K-major A.
//   A map: a_gmid ? (K*comp, groups, rows) : (K*comp, rows, groups) with the given strides.
//   comp == 2: A rows hold [hi | lo] (lo at column offset K) multiplying the same B rows.
// CTA pairs (cta_group::2) are used when the weight slice would otherwise stream and outweighs
// the activation tile (BLR_PAIR=1/2 forces a mode).
// force_pair = 2 / no_res: the pipelined BLAST layer's roles (CTA pairs, streamed weights, so that
// every role walks the token tiles in order).
blr_status gemm_prepare(GemmPrep& g, const DevInfo& d, const void* A, int a_gmid, int64_t a_row_stride,
                        int64_t a_group_stride, int64_t n_tok, int64_t K, int64_t groups, int64_t N, const void* B,
                        bool b_mn_major, const OutMap& out, int comp, int a_blocked = 0, int force_pair = 0,
                        bool no_res = false) {
    KParams& p = g.p;
    int pair = 1;
    // a tile-blocked A with an odd panel count adds a 2-KB zero panel to the smem layout (set on the
    // plan only below): reserve it while planning, so no plan exceeds the opt-in limit with it
    struct ReserveZero {
        int add;
        explicit ReserveZero(int a) : add(a) { t_smem_reserve += add; }
        ~ReserveZero() { t_smem_reserve -= add; }
    } reserve_zero((a_blocked && ((K / 8) & 1)) ? 2048 : 0);
    // CTA pairs by default from 256 tokens (BLR_PAIR=1: single CTAs, BLR_PAIR=0: the shape heuristic
    // below, BLR_PAIR=2: pairs)
    const char* pe = getenv("BLR_PAIR");
    int force = force_pair ? force_pair : pe ? atoi(pe) : 2;
    // ... except short-K phases (<= 4 K blocks) of small problems: single CTAs give twice the tiles
    // and no pair coupling there (GPT2-S / ViT-B / Llama-3.2-1B q_o BLAST S3, K = r <= 256: per layer
    // 4-9 % faster, in-process A/B); BLR_SHORTK_PAIR=1 keeps pairs
    // and problems of <= 2048 tokens (<= 16 token tiles: DiT-XL/2 at 1 and 8 images 47 -> 45 us and
    // 70 -> 66 us; BLR_PAIR=2 forces pairs)
    if (!force_pair && !pe && ((cdiv(K, blr::BK) <= 4 && n_tok < 32768) || n_tok <= 2048)) {
        const char* sk = getenv("BLR_SHORTK_PAIR");
        if (!(sk && sk[0] == '1')) force = 1;
    }
    if (force == 2 && n_tok >= 256) {
        pair = 2;
    } else if (force != 1) {
        if (!plan_gemm(p, 1, d, a_gmid, n_tok, K, groups, N, b_mn_major, out, comp)) return BLR_ERR_UNSUPPORTED;
        // a CTA pair halves each CTA's streamed weight bytes; worth its coupling only when a
        // tile's B (K x BN) is about twice its A (BM x K), i.e. full-width BN = 256 tiles
        // (measured: GPT2-S BLAST c_proj S1 with BN = 192 is faster unpaired)
        if (!p.b_resident && n_tok >= 1024 && p.BN >= 2 * blr::BM) pair = 2;
        // split BLAST S3 (tile-blocked Z'' as A, long K, streamed U): a pair halves each CTA's U
        // bytes per stage, so the ring holds more K blocks in flight (BLR_S3_PAIR=0 disables)
        const char* s3p = getenv("BLR_S3_PAIR");
        if (a_blocked && !(s3p && s3p[0] == '0') && !p.b_resident && n_tok >= 1024 && p.BN >= 192 && K >= 512) pair = 2;
        // any long-K streamed GEMM (e.g. Monarch S3, K = b1 r' = 1536): same ingress argument
        // (Llama-7B Monarch gate S3 2.08 -> 2.02 ms; BLR_LONGK_PAIR=0 disables)
        const char* lkp = getenv("BLR_LONGK_PAIR");
        if (!(lkp && lkp[0] == '0') && !p.b_resident && n_tok >= 1024 && p.BN >= 192 && K >= 1024) pair = 2;
    }
    if (!plan_gemm(p, pair, d, a_gmid, n_tok, K, groups, N, b_mn_major, out, comp, false, 1, !no_res)) {
        if (force_pair || pair == 1 ||
            !plan_gemm(p, pair = 1, d, a_gmid, n_tok, K, groups, N, b_mn_major, out, comp, false, 1, !no_res))
            return BLR_ERR_UNSUPPORTED;
    }
    // wide pair tiles (two MMAs of N = 256 per K step into one 512-column accumulator whose halves
    // the epilogue frees separately, KParams::split_rel): 48 KB of operands per 128x512x64 MACs
    // instead of 32 KB per 128x256x64, i.e. 25 % fewer L2 -> SM bytes per MAC.  Default where each
    // CTA's half of B is one TMA op (a 512-column tile of whole 64-column slabs of an MN-major B
    // over a plain A), K is long enough for the tile's MMAs to cover its epilogue (>= 8
    // K blocks; C4 gate S1's 4 and ViT's 2 lose) and there are enough tiles for the halved tile count
    // to fill the pairs evenly (>= 8 per pair): dense 65536x2048x11008 3.34 -> 2.96 ms, C4 down layer
    // 3.93 -> 3.83 ms; C3's 4096-token phases lose (3-4 waves of wide tiles).  BLR_WIDE=0/1
    // overrides (1: any width).
    {
        const char* we = getenv("BLR_WIDE");
        const bool force = we && we[0] == '1';
        const bool off = (we && we[0] == '0') || force_pair;
        // (not over a tile-blocked A by default: C4 gate S3 as 512 + 176-column tiles measured slower,
        // gate layer 4.06 -> 4.26 ms, as did 2 x 352 -- the 256-column tiles stay there)
        if (!off && pair == 2 && out.col_stride == 0 && N > 256 && (force || !a_blocked)) {
            KParams w;
            if (plan_gemm(w, pair, d, a_gmid, n_tok, K, groups, N, b_mn_major, out, comp, true)) {
                const int units = d.sm_count / 2;
                // MN-major B only, whole 64-column slabs per CTA half (BN = 512).  (K-major B, one box
                // per half at any width, measured slower: C4K 7.90 -> 8.23 ms with 352-wide gate S3
                // and 512-wide down S1 tiles; BLR_WIDE=1 forces it)
                const bool b_ok = b_mn_major && w.BN == 512 && w.b_box_n == 64;
                const bool auto_ok = b_ok && w.stages >= 4 && w.kbox == 1 && w.total_tiles >= 8 * units &&
                                     w.k_blocks >= 8;
                if (force || auto_ok) p = w;
            }
        }
    }
    // B multicast across CTA pairs (cluster of 2 mc CTAs) for streamed pair plans with enough token
    // tiles; BLR_MC=1/2/4 overrides
    {
        // measured slower (C4 8.98 -> 10.47 ms: 33 co-resident 4-CTA clusters instead of 37 pairs, and
        // lock-stepped slot release): opt-in only
        const char* me = getenv("BLR_MC");
        int mc = me ? atoi(me) : 1;
        if (mc > 1 && pair == 2 && !p.b_resident && n_tok >= 2048 * mc && !force_pair) {
            KParams w;
            if (plan_gemm(w, pair, d, a_gmid, n_tok, K, groups, N, b_mn_major, out, comp, p.n_mma == 2, mc)) p = w;
        }
    }
    // the last N tile's MMA covers only its valid columns (rounded up to 16): C4 gate S3's N = 688 is
    // two 256-column tiles and one of 176 (KParams::last_nb; BLR_LASTN=0 off)
    {
        const char* ln = getenv("BLR_LASTN");
        const int64_t last = N - static_cast<int64_t>(p.tiles_n - 1) * p.BN;
        const int64_t lnb = rup(last, 16);
        p.last_nb = (p.n_mma == 1 && !p.b_resident && p.mc <= 1 && p.tiles_n >= 1 && lnb < p.BN && lnb >= 16 &&
                     !(ln && ln[0] == '0'))
                        ? static_cast<int>(lnb) : 0;
    }
    // wide tiles free their two MMA column halves separately (KParams::split_rel; BLR_SPLITREL=0 off)
    {
        const char* sr = getenv("BLR_SPLITREL");
        p.split_rel = (p.n_mma == 2 && p.acc_bufs == 1 && p.kbox == 1 && pair == 2 && !p.b_resident &&
                       p.mc <= 1 && p.c_box_w <= 64 && p.stages >= 2 && !(sr && sr[0] == '0'))
                          ? 1 : 0;
        // a wide plan's last N tile with <= BN/2 valid columns: half 0 alone, rup(valid, 16) wide
        const int64_t last = N - static_cast<int64_t>(p.tiles_n - 1) * p.BN;
        const char* lh = getenv("BLR_LASTHALF");
        if (p.split_rel && last <= p.BN / 2 && !(lh && lh[0] == '0')) {
            p.last_half = 1;
            p.last_nb = static_cast<int>(rup(last, 16));
        }
    }
    const int esz = 2;
    const Swz cs = pick_swz(p.c_box_w * esz);
    p.a_blocked = a_blocked;
    p.a_ptr = static_cast<const __nv_bfloat16*>(A);
    p.a_nchunks = static_cast<int>(K / 8);

    CUtensorMap& ta = g.ta;
    CUtensorMap& tb = g.tb;
    CUtensorMap& tc = g.tc;
    if (a_blocked) {
        // tile-blocked A [g][T][K/8][128][8] viewed as rows of 64 elements (128 B): a K block of a
        // 128-row tile is 128 consecutive rows, one unswizzled tensor box (it lands in smem byte
        // for byte as the no-swizzle K-major core-matrix layout); a tensor copy (unlike a 1-D bulk
        // copy) can complete on the leader's barrier of a CTA pair
        p.a_tiles = static_cast<int>(cdiv(n_tok, blr::BM));
        const uint64_t rows = static_cast<uint64_t>(groups) * p.a_tiles * (K / 8) * 16;
        const uint64_t dims[3] = {64, rows, 1};
        const uint64_t str[2] = {128, rows * 128};
        const uint32_t box[3] = {64, static_cast<uint32_t>(blr::BM), 1};
        if (!encode(&ta, A, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE)) return BLR_ERR_CUDA;
    } else {
        const int64_t Ka = K * comp;  // A row length actually stored
        uint64_t dims[3], str[2];
        dims[0] = static_cast<uint64_t>(Ka);
        if (a_gmid) {
            dims[1] = static_cast<uint64_t>(groups);
            dims[2] = static_cast<uint64_t>(n_tok);
            str[0] = static_cast<uint64_t>(a_group_stride) * 2;
            str[1] = static_cast<uint64_t>(a_row_stride) * 2;
        } else {
            dims[1] = static_cast<uint64_t>(n_tok);
            dims[2] = static_cast<uint64_t>(groups);
            str[0] = static_cast<uint64_t>(a_row_stride) * 2;
            str[1] = static_cast<uint64_t>(a_group_stride > 0 ? a_group_stride : a_row_stride * n_tok) * 2;
        }
        const uint32_t box[3] = {static_cast<uint32_t>(blr::BK), a_gmid ? 1u : static_cast<uint32_t>(blr::BM),
                                 a_gmid ? static_cast<uint32_t>(blr::BM) : 1u};
        if (!encode(&ta, A, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
    }
    if (b_mn_major) {
        const uint64_t dims[3] = {static_cast<uint64_t>(N), static_cast<uint64_t>(K), static_cast<uint64_t>(groups)};
        const uint64_t str[2] = {static_cast<uint64_t>(N) * 2, static_cast<uint64_t>(N * K) * 2};
        const uint32_t box[3] = {static_cast<uint32_t>(p.b_box_n), static_cast<uint32_t>(blr::BK / std::max(1, p.mc)), 1};
        if (!encode(&tb, B, 3, dims, str, box, p.b_box_n == 32 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B))
            return BLR_ERR_CUDA;
        // slab view (64 columns, K, whole 64-column slabs, groups): two boxes per K block as one op.
        // Only whole slabs are described, so a box never reads past a row (or the tensor) end.
        const char* se = getenv("BLR_SLAB");
        if (p.b_box_n == 64 && p.b_boxes == 2 && p.mc <= 1 && N / 64 >= 2 && !(se && se[0] == '0')) {
            const uint64_t d4[4] = {64, static_cast<uint64_t>(K), static_cast<uint64_t>(N / 64), static_cast<uint64_t>(groups)};
            const uint64_t s4[3] = {static_cast<uint64_t>(N) * 2, 128, static_cast<uint64_t>(N * K) * 2};
            const uint32_t b4[4] = {64, static_cast<uint32_t>(blr::BK), 2, 1};
            if (!encode(&g.tb2, B, 4, d4, s4, b4, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
            p.b_slab2 = 1;
            p.b_nslab = static_cast<int>(N / 64);
        }
    } else {
        const uint64_t dims[3] = {static_cast<uint64_t>(K), static_cast<uint64_t>(N), static_cast<uint64_t>(groups)};
        const uint64_t str[2] = {static_cast<uint64_t>(K) * 2, static_cast<uint64_t>(K * N) * 2};
        const uint32_t box[3] = {blr::BK, static_cast<uint32_t>(p.BN / pair / p.n_mma / std::max(1, p.mc)), 1};
        if (!encode(&tb, B, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
    }
    if (out.blocked) {
        // tile-blocked output: the map is encoded below
    } else if (out.col_stride > 0) {
        // strided direct stores (transposed order): the kernel never uses the store map; encode a
        // valid placeholder over the same rows
        const uint64_t dims[4] = {static_cast<uint64_t>(N), 1, 1, static_cast<uint64_t>(n_tok)};
        const uint64_t strb[3] = {static_cast<uint64_t>(N) * 2, static_cast<uint64_t>(N) * 2,
                                  static_cast<uint64_t>(out.row_stride) * 2};
        const uint32_t box[4] = {static_cast<uint32_t>(p.c_box_w), 1, 1, 32};
        if (!encode(&tc, out.ptr, 4, dims, strb, box, cs.mode, out.f32)) return BLR_ERR_CUDA;
    } else {
        const uint64_t dims[4] = {static_cast<uint64_t>(N), static_cast<uint64_t>(out.comp),
                                  static_cast<uint64_t>(groups), static_cast<uint64_t>(n_tok)};
        const uint64_t es = static_cast<uint64_t>(esz);
        const uint64_t strb[3] = {static_cast<uint64_t>(out.comp_stride) * es, static_cast<uint64_t>(out.group_stride) * es,
                                  static_cast<uint64_t>(out.row_stride) * es};
        // 128-row cooperative stores (KParams::coop_store; BLR_COOP=0: per-warp 32-row boxes)
        const char* ce = getenv("BLR_COOP");
        p.coop_store = (p.c_box_w <= 64 && !(ce && ce[0] == '0')) ? 1 : 0;
        const uint32_t box[4] = {static_cast<uint32_t>(p.c_box_w), 1, 1, p.coop_store ? 128u : 32u};
        if (!encode(&tc, out.ptr, 4, dims, strb, box, cs.mode, out.f32)) return BLR_ERR_CUDA;
    }
    if (out.blocked) {
        // tile-blocked fp16 output [g][T][N/8][128][8] viewed (64 elem, 16 rows, N/8 panels, g*T):
        // a chunk's panels of one tile are one tensor store box (64, 16, CW/8, 1); panels past N
        // fall outside dim 2 and are clipped (a 1-D bulk copy per chunk measured slower)
        p.o_tiles = static_cast<int>(cdiv(n_tok, blr::BM));
        // (e4m3: 1-KB panels of 16 rows x 64 B)
        const uint64_t eb = out.f32 == 3 ? 1 : 2;
        const uint64_t dims[4] = {64, 16, static_cast<uint64_t>(N / 8), static_cast<uint64_t>(groups) * p.o_tiles};
        const uint64_t strb[3] = {64 * eb, 1024 * eb, static_cast<uint64_t>(N / 8) * 1024 * eb};
        const uint32_t box[4] = {64, 16, static_cast<uint32_t>(p.c_box_w / 8), 1};
        if (!encode(&tc, out.ptr, 4, dims, strb, box, CU_TENSOR_MAP_SWIZZLE_NONE, out.f32)) return BLR_ERR_CUDA;
    }
    if (!p.b_slab2) g.tb2 = tb;
    // fp16 output (BLAST split-path Z) is a separate instantiation: the bf16 epilogue stays as is
    g.pair = pair;
    g.outf = out.f32 == 3 ? 3 : out.f32 == 2 ? (out.blocked ? 2 : 1) : 0;

    return BLR_OK;
}

// ------------------------------------------------------- one-launch LR / Monarch layer ----
// blr_fused.cuh: S1 and S3 of a token tile in one CTA, Z on chip.  Used when the intermediate
// fits one 256-column TMEM buffer and the swizzled smem copy (128 <= k2 <= 256, k2 % 64 == 0;
// shorter S3 contractions keep the compensated two-kernel path, R12).  BLR_FUSED=0/1
// overrides the default.
// Default: Monarch always (its S1 is block-diagonal, cheap to recompute per output block);
// low rank only for expanding layers (d_in <= d_out) -- a contracting layer's S1 streams a long
// X row and all of V per token tile, and its few tiles cannot fill the SMs (GPT2-S c_proj:
// 46.6 us fused vs 39.7 us in two kernels, c_fc 34.3 vs 37.6 us).
bool fused_wanted(int64_t n_tok, int64_t k2, int64_t n1, bool contracting_lr) {
    if (k2 % 64 || k2 < 128 || k2 > 256 || n1 % 16 || n1 > 256) return false;
    const char* e = getenv("BLR_FUSED");
    if (e && e[0] == '0') return false;
    if (e && e[0] == '1') return true;
    return n_tok >= 256 && !contracting_lr;
}

void fused_b_staging(bool mn, int n, int& boxes, uint32_t& bytes, uint32_t& lbo, uint32_t& sbo, uint32_t& kstep) {
    if (mn) {  // [K][N] storage: 64-column SW128 boxes (as set_b_staging)
        boxes = static_cast<int>(cdiv(n, 64));
        bytes = static_cast<uint32_t>(boxes * 64 * blr::BK * 2);
        lbo = 64 * 2 * blr::BK;
        sbo = 1024;
        kstep = 16 * 128;
    } else {  // [N][K] storage: n rows x 64 K, K-major SW128
        boxes = 1;
        bytes = static_cast<uint32_t>(rup(static_cast<int64_t>(n) * blr::BK * 2, 1024));
        lbo = 16;
        sbo = 1024;
        kstep = 32;
    }
}

// p: n_tok, mon, g1, k1_blocks, n1, b1_mn, g2, n2, b2_mn filled by the caller.
blr_status fused_launch(const DevInfo& d, int dev, cudaStream_t st, blr::FParams p, const CUtensorMap& ta,
                        const CUtensorMap& tb1, const CUtensorMap& tb2, void* Y, int64_t d_out) {
    p.tiles_m = static_cast<int>(cdiv(p.n_tok, blr::BM));
    p.k2 = p.g1 * p.n1;
    fused_b_staging(p.b1_mn, p.n1, p.b1_boxes, p.b1_bytes, p.b1_lbo, p.b1_sbo, p.b1_kstep);
    const int64_t nch_tiles = cdiv(p.n2, 256);
    p.bn2 = static_cast<int>(rup(cdiv(p.n2, nch_tiles), 16));
    fused_b_staging(p.b2_mn, p.bn2, p.b2_boxes, p.b2_bytes, p.b2_lbo, p.b2_sbo, p.b2_kstep);
    // Split the S3 columns into parts to fill the SMs, minimising the busiest CTA's work in
    // units of one S3 chunk: waves x (S1 recompute + chunks per part), S1 weighted by its MACs
    // relative to a chunk's (a partial second wave idles most SMs for a whole item).
    const int64_t base = static_cast<int64_t>(p.tiles_m) * p.g2, nchunks = cdiv(p.n2, p.bn2);
    const double s1_w = static_cast<double>(p.k1_blocks) * p.g1 * p.n1 / (static_cast<double>(p.k2 / 64) * p.bn2);
    int64_t cpp = nchunks;
    double best = 1e30;
    for (int64_t np = 1; np <= nchunks; ++np) {
        const int64_t c = cdiv(nchunks, np), npp = cdiv(nchunks, c);
        const double cost = static_cast<double>(cdiv(base * npp, d.sm_count)) * (s1_w + static_cast<double>(c));
        if (cost < best - 1e-9) {
            best = cost;
            cpp = c;
        }
    }
    p.n2_part = static_cast<int>(cpp * p.bn2);
    p.n_parts = static_cast<int>(cdiv(nchunks, cpp));
    p.items = static_cast<int>(base * p.n_parts);
    p.c_box_w = chunk_width(p.bn2);
    p.c_swz = pick_swz(p.c_box_w * 2).mask;
    p.s1_bytes = static_cast<uint32_t>(blr::BM * blr::BK * 2) + p.b1_bytes;
    p.slot_bytes = static_cast<uint32_t>(rup(std::max<int64_t>(p.s1_bytes, p.b2_bytes), 1024));
    // two staging buffers per epilogue warp (Y stores overlap the next chunk's staging) when the
    // ring still gets >= 3 slots, else one (BLR_FUSED_BUFS=1/2 forces)
    const char* fb_env = getenv("BLR_FUSED_BUFS");
    for (p.stage_bufs = 2; p.stage_bufs >= 1; --p.stage_bufs) {
        if (fb_env && atoi(fb_env) != p.stage_bufs) continue;
        p.stage_warp_bytes = static_cast<uint32_t>(p.stage_bufs * 32 * p.c_box_w * 2);
        for (p.stages = blr::MAX_STAGES; p.stages >= 2; --p.stages)
            if (blr::fused_layout(p).total + SMEM_SLACK <= static_cast<uint32_t>(SMEM_LIMIT)) break;
        if (p.stages >= (p.stage_bufs == 2 && !fb_env ? 3 : 2)) break;
    }
    if (p.stages < 2 || p.stage_bufs < 1) return BLR_ERR_UNSUPPORTED;
    CUtensorMap tc;
    {
        const uint64_t dims[4] = {static_cast<uint64_t>(p.n2), 1, static_cast<uint64_t>(p.g2), static_cast<uint64_t>(p.n_tok)};
        const uint64_t str[3] = {static_cast<uint64_t>(p.n2) * 2, static_cast<uint64_t>(p.n2) * 2,
                                 static_cast<uint64_t>(d_out) * 2};
        const char* ce = getenv("BLR_COOP");
        p.coop_store = (p.c_box_w <= 64 && p.y_cs == 0 && !(ce && ce[0] == '0')) ? 1 : 0;
        const uint32_t box[4] = {static_cast<uint32_t>(p.c_box_w), 1, 1, p.coop_store ? 128u : 32u};
        if (!encode(&tc, Y, 4, dims, str, box, pick_swz(p.c_box_w * 2).mode)) return BLR_ERR_CUDA;
    }
    const int smem = static_cast<int>(blr::fused_layout(p).total + SMEM_SLACK);
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!g_attr_set[23][dev]) {
            if (cudaFuncSetAttribute(blr::blr_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT) !=
                cudaSuccess)
                return BLR_ERR_CUDA;
            g_attr_set[23][dev] = true;
        }
    }
    const int grid = std::min(p.items, d.sm_count);
    if (const char* pe = getenv("BLR_PLAN"); pe && pe[0] == '1')
        fprintf(stderr,
                "[blr plan] fused mon=%d grid=%d items=%dx%dx%d g1=%d k1b=%d n1=%d k2=%d n2=%d bn2=%d stages=%d "
                "bufs=%d smem=%d\n",
                p.mon, grid, p.tiles_m, p.g2, p.n_parts, p.g1, p.k1_blocks, p.n1, p.k2, p.n2, p.bn2, p.stages,
                p.stage_bufs, smem);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(blr::NUM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const bool prof = t_prof_events != nullptr && 2 * t_prof_n + 1 < t_prof_cap;
    if (prof && prof_record(t_prof_events[2 * t_prof_n], st) != cudaSuccess) return BLR_ERR_CUDA;
    if (cudaLaunchKernelEx(&cfg, blr::blr_fused_kernel, ta, tb1, tb2, tc, p) != cudaSuccess) return BLR_ERR_CUDA;
    if (prof) {
        if (prof_record(t_prof_events[2 * t_prof_n + 1], st) != cudaSuccess) return BLR_ERR_CUDA;
        ++t_prof_n;
    }
    ++t_last_launches;
    return BLR_OK;
}

// X viewed as [n_tok][b1][p] (A operand of the block-diagonal first stage).
bool encode_x_blocked(CUtensorMap* m, const void* X, int64_t n_tok, int64_t b1, int64_t pdim) {
    const uint64_t dims[3] = {static_cast<uint64_t>(pdim), static_cast<uint64_t>(b1), static_cast<uint64_t>(n_tok)};
    const uint64_t str[2] = {static_cast<uint64_t>(pdim) * 2, static_cast<uint64_t>(pdim * b1) * 2};
    const uint32_t box[3] = {blr::BK, 1, blr::BM};
    return encode(m, X, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

// ------------------------------------------------------------------ decode (small n) path ----
// Small n runs the weight-streaming tensor-core decode stages of blr_decode_tc.cuh
// up to a per-method token count where they measured faster than the tcgen05 prefill path
// (scripts/decode_bench.py, profiles/r02_decode.txt, profiles/r02_small_n.txt): low rank n <= 16,
// Monarch n <= 256, BLAST n <= 16 (n <= 2048 when the tcgen05 path would be the S1+S2-fused
// projection; Llama-7B BLAST at n = 12 / 16: 34.7 / 36.0 us vs 39.8 us, profiles/r02_decode.txt);
// n > 16 runs as independent 16-token chunks.  BLR_DECODE=1 forces the path for
// every n <= DECODE_MAX_TOKENS, BLR_DECODE_MAXN=m for n <= m, BLR_DECODE=0 disables it.
bool use_decode(int64_t n_tok, int64_t default_max) {
    if (n_tok > blr::DTC_MAX_N) return false;
    const char* e = getenv("BLR_DECODE");
    if (e && e[0] == '0') return false;
    if (e && e[0] == '1') return n_tok <= blr::DECODE_MAX_TOKENS;
    const char* m = getenv("BLR_DECODE_MAXN");  // force the weight-streaming path up to this n
    if (m) return n_tok <= atoll(m);
    return n_tok <= default_max;
}
// decode-path workspace: fp32 intermediates only (K splits are reduced on chip)
size_t lowrank_decode_ws(int64_t n, int64_t r) { return static_cast<size_t>(n) * r * 4; }
size_t blast_decode_ws(int64_t n, int64_t b1, int64_t b2, int64_t r) { return static_cast<size_t>(b1 + b2) * n * r * 4; }
size_t monarch_decode_ws(int64_t n, int64_t b1, int64_t b2, int64_t r_blk) {
    return static_cast<size_t>(b2) * n * b1 * r_blk * 4;
}

// ---- tensor-core decode stages (blr_decode_tc.cuh): planned and encoded before any launch ----
struct DtcPrep {
    blr::DecodeTC d;
    CUtensorMap tm;
    dim3 grid;
    int cluster, epi, kmaj, w;
    size_t smem;
};

// Time estimate (us) of one decode stage: `ctas` CTAs each streaming `bytes_cta` weight bytes
// through a ring of `ring` bytes.  Measured (benchmarks/micro/dtc_stream.cu): HBM
// ~6.2 TB/s (64-column strips of a row-major weight ~20% slower), and a TMA load takes ~2.5 us
// under load, so one CTA streams at most ring / 2.5 us; waves beyond the first repeat that;
// ~1 us for the in-cluster K reduction.
double dtc_estimate(int64_t ctas, double bytes_cta, double ring, int w, bool kmaj, int64_t per_sm, bool split,
                    int64_t chunks = 1) {
    const double eff = kmaj ? 0.9 : w == 64 ? 0.8 : w == 128 ? 0.95 : 1.0;
    const double t_hbm = ctas * bytes_cta / (6.2e6 * eff);  // each token chunk re-reads the weights from L2
    const double t_cta = 2.0 + bytes_cta * 2.5 / ring;  // + start-up: A slice, first loads' latency
    const int64_t waves = cdiv(ctas * chunks, 148 * per_sm);
    return std::max(t_hbm, t_cta * waves) + (split ? 1.0 : 0.0);
}

// smem per CTA for a tile; the ring gets whatever keeps `per_sm` CTAs resident (<= 12 stages)
bool dtc_fit(int kc, int a_f32, int units, int epi, int w, int bk, int s_elems, int per_sm, int& stages, size_t& smem) {
    const blr::dtc::Layout L0 = blr::dtc::layout(kc, a_f32, units, 0, epi, w, bk, s_elems);
    const int64_t budget = (228 * 1024) / per_sm - 1024 - static_cast<int64_t>(L0.total);
    stages = static_cast<int>(std::min<int64_t>(12, budget / (blr::DTC_STAGE + 16)));
    stages = std::min(stages, std::max(2, units * ((kc + bk - 1) / bk)));  // no deeper than the CTA's data
    if (epi == 1) stages = std::max(stages, (16 * w * 4 + blr::DTC_STAGE - 1) / blr::DTC_STAGE);  // tile fits the ring
    if (stages < 2) return false;
    smem = blr::dtc::layout(kc, a_f32, units, stages, epi, w, bk, s_elems).total;
    return smem + 1024 <= static_cast<size_t>(228 * 1024) / per_sm;
}

// Choose the tile width W, the K split S (= cluster size) and the ring depth of an (N, K, G)
// weight stream.  BLR_DTC_S / BLR_DTC_W force S / W (experiments).
void dtc_plan(DtcPrep& P, int64_t K, int64_t N, int64_t G, int a_f32, int kmaj, int64_t chunks) {
    const char* fs = getenv(P.d.pre ? "BLR_DTC_S1" : "BLR_DTC_S0");  // per launch of the call
    const char* fw = getenv(P.d.pre ? "BLR_DTC_W1" : "BLR_DTC_W0");
    if (!fs) fs = getenv("BLR_DTC_S");
    if (!fw) fw = getenv("BLR_DTC_W");
    const int force_s = fs ? atoi(fs) : 0, force_w = fw ? atoi(fw) : 0;
    const char* fm = getenv("BLR_DTC_MINPERSM");
    int min_per_sm = fm ? atoi(fm) : 2;  // prefer two resident CTAs per SM: the next launch's CTAs
                                         // can then start streaming their weights during this one
    double best = 1e300;
    P.cluster = 0;
  retry:
    for (int w : {64, 128, 256}) {
        if (kmaj && w != 64) continue;
        if (force_w && w != force_w) continue;
        const int bk = blr::dtc_bk(kmaj != 0, w);
        const int64_t nt = cdiv(N, w);
        for (int S = 1; S <= blr::DTC_MAX_CLUSTER; ++S) {
            const int64_t kc = rup(cdiv(K, S), bk);
            if (kc > blr::DTC_MAX_KC || cdiv(K, kc) != S) continue;
            if (force_s && S != force_s) continue;
            const int epi = S > 1 ? 1 : 0;
            // cluster-split plans run one CTA per SM: with two co-resident CTAs per SM the first call
            // of a process intermittently summed a stale 16-32-column slice of a peer's partial tile
            // (Llama-7B n = 16 S3, W = 256, S = 6: 2 of ~10 fresh processes; 0 of 35 with one CTA
            // per SM; root cause not isolated -- DESIGN.md §5.3b)
            for (int per_sm = (S > 1 ? 1 : min_per_sm); per_sm <= (S > 1 ? 1 : 3); ++per_sm) {
                int stages;
                size_t smem;
                if (!dtc_fit(static_cast<int>(kc), a_f32, 1, epi, w, bk, 0, per_sm, stages, smem)) continue;
                if (stages < std::min<int64_t>(3, cdiv(kc, bk)) && per_sm > 1) continue;
                const int64_t ctas = nt * G * S;
                const int64_t resident = std::min<int64_t>(8, (228 * 1024) / (smem + 1024));
                const double c = dtc_estimate(ctas, static_cast<double>(kc) * w * 2, static_cast<double>(stages) * blr::DTC_STAGE,
                                              w, kmaj != 0, resident, S > 1, chunks) + 0.3 * smem / (228.0 * 1024);
                if (c < best) {
                    best = c;
                    P.cluster = S;
                    P.epi = epi;
                    P.w = w;
                    P.d.k_chunk = static_cast<int>(kc);
                    P.d.stages = stages;
                    P.smem = smem;
                    P.grid = dim3(static_cast<unsigned>(S), static_cast<unsigned>(nt), static_cast<unsigned>(G * chunks));
                }
            }
        }
    }
    if (P.cluster == 0 && min_per_sm > 1) {  // a preference, not a requirement
        min_per_sm = 1;
        goto retry;
    }
}

// out[g][t][c] = sum_k A[g][t][k] B[g][k][c] (kmaj = 0, B [K][N]) or B[g][c][k] (kmaj = 1, B [N][K]).
blr_status dtc_prepare(DtcPrep& P, const void* A, int a_f32, int64_t a_rs, int64_t a_gs, const void* B, int kmaj,
                       int64_t b_rs, int64_t b_gs, void* out, int out_bf16, int64_t o_rs, int64_t o_gs, int64_t o_cs,
                       int64_t n, int64_t K, int64_t N, int64_t G, int pre) {
    P = DtcPrep();
    blr::DecodeTC& d = P.d;
    if (a_rs % 8 || a_gs % 8) return BLR_ERR_ALIGN;
    d.A = A;
    d.a_f32 = a_f32;
    d.a_rs = a_rs;
    d.a_gs = a_gs;
    d.n_tok = static_cast<int>(n);
    d.K = static_cast<int>(K);
    d.N = static_cast<int>(N);
    d.n_units = 1;
    d.groups = static_cast<int>(G);
    d.out = out;
    d.out_bf16 = out_bf16;
    d.o_rs = o_rs;
    d.o_gs = o_gs;
    d.o_cs = o_cs;
    d.pre = pre;
    P.kmaj = kmaj;
    const int64_t chunks = cdiv(n, 16);
    if (G * chunks > 65535) return BLR_ERR_UNSUPPORTED;
    dtc_plan(P, K, N, G, a_f32, kmaj, chunks);
    if (P.cluster == 0) return BLR_ERR_UNSUPPORTED;
    if (getenv("BLR_DTC_VERBOSE"))
        fprintf(stderr, "dtc K=%lld N=%lld G=%lld kmaj=%d a_f32=%d: W=%d S=%d kc=%d stages=%d smem=%zu grid=%u\n",
                (long long)K, (long long)N, (long long)G, kmaj, a_f32, P.w, P.cluster, P.d.k_chunk, P.d.stages, P.smem,
                P.grid.x * P.grid.y * P.grid.z);
    const int bk = blr::dtc_bk(kmaj != 0, P.w);
    const uint64_t gs = static_cast<uint64_t>(b_gs > 0 ? b_gs : b_rs * (kmaj ? N : K)) * 2;
    if (kmaj) {  // B [N][K] per group: map (K, N, G), box 64 k x 64 columns
        const uint64_t dims[3] = {static_cast<uint64_t>(K), static_cast<uint64_t>(N), static_cast<uint64_t>(G)};
        const uint64_t str[2] = {static_cast<uint64_t>(b_rs) * 2, gs};
        const uint32_t box[3] = {64, 64, 1};
        if (!encode(&P.tm, B, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
    } else {  // B [K][N] per group: map (N, K, G), box 64 columns x bk k
        const uint64_t dims[3] = {static_cast<uint64_t>(N), static_cast<uint64_t>(K), static_cast<uint64_t>(G)};
        const uint64_t str[2] = {static_cast<uint64_t>(b_rs) * 2, gs};
        const uint32_t box[3] = {64, static_cast<uint32_t>(bk), 1};
        if (!encode(&P.tm, B, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
    }
    return BLR_OK;
}

template <bool KMAJ, int EPI, int W>
blr_status dtc_launch_t(const DtcPrep& P, cudaStream_t st) {
    auto kfn = blr::decode_tc_kernel<KMAJ, EPI, W>;
    static bool attr_set[64] = {};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return BLR_ERR_CUDA;
    if (!attr_set[dev & 63]) {
        if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT) != cudaSuccess)
            return BLR_ERR_CUDA;
        attr_set[dev & 63] = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = P.grid;
    cfg.blockDim = dim3(blr::DTC_THREADS);
    cfg.dynamicSmemBytes = P.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[2];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = static_cast<unsigned>(P.cluster);
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 2;
    const bool prof = t_prof_events != nullptr && 2 * t_prof_n + 1 < t_prof_cap;
    if (prof && prof_record(t_prof_events[2 * t_prof_n], st) != cudaSuccess) return BLR_ERR_CUDA;
    blr::DecodeTC dd = P.d;
    dd.trace = t_trace;
    if (t_trace) t_trace += 128 * 256;  // next launch traces into the next slot
    if (cudaLaunchKernelEx(&cfg, kfn, P.tm, dd) != cudaSuccess) return BLR_ERR_CUDA;
    if (prof) {
        if (prof_record(t_prof_events[2 * t_prof_n + 1], st) != cudaSuccess) return BLR_ERR_CUDA;
        ++t_prof_n;
    }
    ++t_last_launches;
    return BLR_OK;
}

template <int EPI>
blr_status dtc_launch_w(const DtcPrep& P, cudaStream_t st) {
    if (P.w == 64) return dtc_launch_t<false, EPI, 64>(P, st);
    return P.w == 128 ? dtc_launch_t<false, EPI, 128>(P, st) : dtc_launch_t<false, EPI, 256>(P, st);
}

blr_status dtc_launch(const DtcPrep& P, cudaStream_t st) {
    if (P.kmaj) return P.epi == 0 ? dtc_launch_t<true, 0, 64>(P, st) : dtc_launch_t<true, 1, 64>(P, st);
    return P.epi == 0 ? dtc_launch_w<0>(P, st) : P.epi == 1 ? dtc_launch_w<1>(P, st) : dtc_launch_w<2>(P, st);
}

bool dtc_blast_mix_ok(int64_t b1, int64_t pdim, int& cs, int& units) {
    if (pdim > blr::DTC_MAX_KC) return false;
    for (int u = 1; u <= blr::DTC_MAX_UNITS; ++u)
        if (b1 % u == 0 && b1 / u <= blr::DTC_MAX_CLUSTER) {
            units = u;
            cs = static_cast<int>(b1 / u);
            return true;
        }
    return false;
}
blr_status dtc_prepare_blast_mix(DtcPrep& P, const void* X, int64_t d_in, int64_t pdim, const void* V, const void* S,
                                 float* zpp, int64_t n, int64_t b1, int64_t b2, int64_t r, int cs, int units) {
    P = DtcPrep();
    blr::DecodeTC& d = P.d;
    d.A = X;
    d.a_f32 = 0;
    d.a_rs = d_in;
    d.a_gs = pdim;
    d.n_tok = static_cast<int>(n);
    d.K = static_cast<int>(pdim);
    d.N = static_cast<int>(r);
    d.n_units = units;
    d.groups = 1;
    d.out = zpp;
    d.out_bf16 = 0;
    d.o_rs = r;
    d.o_gs = n * r;
    d.o_cs = 1;
    d.s2 = static_cast<const __nv_bfloat16*>(S);
    d.b1 = static_cast<int>(b1);
    d.b2 = static_cast<int>(b2);
    d.pre = 0;
    P.cluster = cs;
    P.epi = 2;
    P.kmaj = 0;
    const char* fw = getenv("BLR_DTC_W0");
    if (!fw) fw = getenv("BLR_DTC_W");
    const int force_w = fw ? atoi(fw) : 0;
    double best = 1e300;
    const int64_t nk = cdiv(b2, cs);
    const char* fm = getenv("BLR_DTC_MINPERSM");
    for (int min_per_sm = fm ? std::min(2, atoi(fm)) : 2; min_per_sm >= 1 && best >= 1e300; --min_per_sm) {
        for (int w : {64, 128, 256}) {
            if (force_w && w != force_w) continue;
            const int bk = blr::dtc_bk(false, w);
            const int kc = static_cast<int>(rup(pdim, bk));
            for (int per_sm = 1; per_sm <= 1; ++per_sm) {  // cluster plan: one CTA per SM (see dtc_plan)
                int stages;
                size_t smem;
                if (!dtc_fit(kc, 0, units, 2, w, bk, static_cast<int>(nk * b1 * w), per_sm, stages, smem)) continue;
                if (stages < std::min(3, units * kc / bk) && per_sm > 1) continue;
                const int64_t ctas = cs * cdiv(r, w);
                const int64_t resident = std::min<int64_t>(8, (228 * 1024) / (smem + 1024));
                const double c = dtc_estimate(ctas, static_cast<double>(units) * kc * w * 2,
                                              static_cast<double>(stages) * blr::DTC_STAGE, w, false, resident, true,
                                              cdiv(n, 16)) +
                                 0.3 * smem / (228.0 * 1024);
                if (c < best) {
                    best = c;
                    P.w = w;
                    d.k_chunk = kc;
                    d.stages = stages;
                    P.smem = smem;
                    P.grid = dim3(static_cast<unsigned>(cs), static_cast<unsigned>(cdiv(r, w)),
                                  static_cast<unsigned>(cdiv(n, 16)));
                }
            }
        }
    }
    if (best >= 1e300) return BLR_ERR_UNSUPPORTED;
    if (getenv("BLR_DTC_VERBOSE"))
        fprintf(stderr, "dtc blast-mix p=%lld r=%lld b1=%lld: cs=%d units=%d W=%d stages=%d smem=%zu grid=%u\n",
                (long long)pdim, (long long)r, (long long)b1, cs, units, P.w, d.stages, P.smem, P.grid.x * P.grid.y);
    const uint64_t dims[3] = {static_cast<uint64_t>(r), static_cast<uint64_t>(pdim), static_cast<uint64_t>(b1)};
    const uint64_t str[2] = {static_cast<uint64_t>(r) * 2, static_cast<uint64_t>(pdim * r) * 2};
    const uint32_t box[3] = {64, static_cast<uint32_t>(blr::dtc_bk(false, P.w)), 1};
    if (!encode(&P.tm, V, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
    return BLR_OK;
}

// Pipelined BLAST layer: ticket + Z-ready + Z''-ready counters, one per 128-token tile of the CTA
// pairs' 256-row tiles (padded), after the split path's Z'' and Z
size_t pipe_ctr_bytes(int64_t n_tok) {
    const int64_t tiles_pad = 2 * cdiv(n_tok, 2 * blr::BM);
    return static_cast<size_t>(rup(4 * (1 + 2 * tiles_pad), 256));
}

size_t blast_ws_bytes(int64_t n_tok, int64_t b1, int64_t b2, int64_t r) {
    if (blast_fused(b1, r)) return static_cast<size_t>(b2) * n_tok * r * 2 * comp_factor(r);
    // split path: Z'' and the fp16 Z_l of the separate S1, token count padded to whole 128-row
    // tiles (the tensor-core S2 path stores both tile-blocked)
    const int64_t np = rup(n_tok, blr::BM);
    return static_cast<size_t>(b2) * np * r * 2 * comp_factor(r) + static_cast<size_t>(b1) * np * r * 2 +
           pipe_ctr_bytes(n_tok);
}

}  // namespace

extern "C" {

const char* blr_status_string(blr_status s) {
    switch (s) {
        case BLR_OK: return "BLR_OK";
        case BLR_ERR_NULL: return "BLR_ERR_NULL";
        case BLR_ERR_SHAPE: return "BLR_ERR_SHAPE";
        case BLR_ERR_ALIGN: return "BLR_ERR_ALIGN";
        case BLR_ERR_UNSUPPORTED: return "BLR_ERR_UNSUPPORTED";
        case BLR_ERR_WORKSPACE: return "BLR_ERR_WORKSPACE";
        case BLR_ERR_ARCH: return "BLR_ERR_ARCH";
        case BLR_ERR_CUDA: return "BLR_ERR_CUDA";
    }
    return "BLR_ERR_UNKNOWN";
}

const char* blr_version(void) { return "0.3.0"; }

blr_status blr_transposed_row_perm(int64_t b2, int64_t q, int64_t* perm) {
    if (b2 <= 0 || q <= 0) return BLR_ERR_SHAPE;
    if (!perm) return BLR_ERR_NULL;
    for (int64_t c = 0; c < q; ++c)
        for (int64_t k = 0; k < b2; ++k) perm[c * b2 + k] = k * q + c;  // transposed j = c b2 + k
    return BLR_OK;
}

int blr_last_launch_count(void) { return t_last_launches; }

void blr_profile_begin(void** events, int capacity) {
    t_prof_events = events;
    t_prof_cap = events ? capacity : 0;
    t_prof_n = 0;
}

int blr_profile_end(void) {
    const int n = t_prof_n;
    t_prof_events = nullptr;
    t_prof_cap = 0;
    t_prof_n = 0;
    return n;
}

// Debug (not in blr.h's stable surface): per-CTA timestamps of the next GEMM-kernel launches.
void blr_debug_trace(unsigned long long* device_buf) { t_trace = device_buf; }

void blr_clear_cache(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& d : g_dev) d = DevInfo();
    g_encode = nullptr;
}

// Workspace: the tcgen05 path's intermediate; for n_tok <= DTC_MAX_N also enough for the
// decode path's fp32 intermediates and split-K partials (either path may run: BLR_DECODE=0).
size_t blr_lowrank_workspace_size(int64_t n_tok, int64_t d_in, int64_t d_out, int64_t r) {
    if (n_tok <= 0 || r <= 0) return 0;
    size_t b = static_cast<size_t>(n_tok) * r * 2 * comp_factor(r);
    if (n_tok <= blr::DTC_MAX_N && d_in > 0 && d_out > 0)
        b = std::max(b, lowrank_decode_ws(n_tok, r));
    return b;
}
size_t blr_monarch_workspace_size(int64_t n_tok, int64_t, int64_t, int64_t b1, int64_t b2, int64_t r_blk) {
    if (n_tok <= 0 || b1 <= 0 || b2 <= 0 || r_blk <= 0) return 0;
    size_t b = static_cast<size_t>(b2) * n_tok * b1 * r_blk * 2 * comp_factor(b1 * r_blk);
    if (n_tok <= blr::DTC_MAX_N) b = std::max(b, monarch_decode_ws(n_tok, b1, b2, r_blk));
    return b;
}
size_t blr_blast_workspace_size(int64_t n_tok, int64_t d_in, int64_t d_out, int64_t b1, int64_t b2, int64_t r) {
    if (n_tok <= 0 || b1 <= 0 || b2 <= 0 || r <= 0) return 0;
    size_t b = blast_ws_bytes(n_tok, b1, b2, r);
    if (n_tok <= blr::DTC_MAX_N && d_in > 0 && d_out > 0 && d_in % b1 == 0 && d_out % b2 == 0)
        b = std::max(b, blast_decode_ws(n_tok, b1, b2, r));
    return b;
}

blr_status blr_lowrank_matmul(const void* X, int64_t n_tok, int64_t d_in, int64_t d_out, int64_t r,
                              const void* V, const void* U, void* Y, void* workspace, size_t ws_bytes,
                              blr_stream_t stream) {
    t_last_launches = 0;
    if (n_tok < 0 || d_in <= 0 || d_out <= 0 || r <= 0) return BLR_ERR_SHAPE;
    if (n_tok == 0) return BLR_OK;
    if (!X || !V || !U || !Y || !workspace) return BLR_ERR_NULL;
    if (d_in % 8 || d_out % 8 || r % 8) return BLR_ERR_ALIGN;
    if (!al16(X) || !al16(V) || !al16(U) || !al16(Y) || !al16(workspace)) return BLR_ERR_ALIGN;
    if (n_tok > (int64_t(1) << 31) - 1) return BLR_ERR_UNSUPPORTED;
    if (ws_bytes < blr_lowrank_workspace_size(n_tok, d_in, d_out, r)) return BLR_ERR_WORKSPACE;
    DevInfo d;
    int dev;
    blr_status s = device_info(d, dev);
    if (s != BLR_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (use_decode(n_tok, 16)) {  // weight-streaming small-n path: two tensor-core stages, fp32 Z [n][r]
        float* zf = static_cast<float*>(workspace);
        DtcPrep p1, p2;
        s = dtc_prepare(p1, X, 0, d_in, 0, V, 0, r, 0, zf, 0, r, 0, 1, n_tok, d_in, r, 1, 0);
        if (s != BLR_OK) return s;
        s = dtc_prepare(p2, zf, 1, r, 0, U, 0, d_out, 0, Y, 1, d_out, 0, 1, n_tok, r, d_out, 1, 1);
        if (s != BLR_OK) return s;
        s = dtc_launch(p1, st);
        return s != BLR_OK ? s : dtc_launch(p2, st);
    }
    if (fused_wanted(n_tok, r, r, d_in > d_out)) {  // one launch, Z on chip (blr_fused.cuh)
        blr::FParams p = {};
        p.n_tok = static_cast<int>(n_tok);
        p.mon = 0;
        p.g1 = 1;
        p.k1_blocks = static_cast<int>(cdiv(d_in, blr::BK));
        p.n1 = static_cast<int>(r);
        p.b1_mn = 1;
        p.g2 = 1;
        p.n2 = static_cast<int>(d_out);
        p.b2_mn = 1;
        CUtensorMap ta, tb1, tb2;
        {
            const uint64_t dims[3] = {static_cast<uint64_t>(d_in), static_cast<uint64_t>(n_tok), 1};
            const uint64_t str[2] = {static_cast<uint64_t>(d_in) * 2, static_cast<uint64_t>(d_in * n_tok) * 2};
            const uint32_t box[3] = {blr::BK, blr::BM, 1};
            if (!encode(&ta, X, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
        }
        {
            const uint64_t dims[3] = {static_cast<uint64_t>(r), static_cast<uint64_t>(d_in), 1};
            const uint64_t str[2] = {static_cast<uint64_t>(r) * 2, static_cast<uint64_t>(r * d_in) * 2};
            const uint32_t box[3] = {64, blr::BK, 1};
            if (!encode(&tb1, V, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
        }
        {
            const uint64_t dims[3] = {static_cast<uint64_t>(d_out), static_cast<uint64_t>(r), 1};
            const uint64_t str[2] = {static_cast<uint64_t>(d_out) * 2, static_cast<uint64_t>(d_out * r) * 2};
            const uint32_t box[3] = {64, blr::BK, 1};
            if (!encode(&tb2, U, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
        }
        s = fused_launch(d, dev, st, p, ta, tb1, tb2, Y, d_out);
        if (s != BLR_ERR_UNSUPPORTED) return s;
    }
    const int comp = comp_factor(r);
    // both phases are planned (tensor maps encoded) before the first launch
    GemmPrep g1, g3;
    // S1: Z = X V  (V is [d_in][r]: MN-major B); Z rows [hi | lo] when compensated
    s = gemm_prepare(g1, d, X, 0, d_in, 0, n_tok, d_in, 1, r, V, true, OutMap{workspace, 0, comp, r, r, r * comp}, 1);
    if (s != BLR_OK) return s;
    // S3: Y = Z U  (U is [r][d_out]: MN-major B)
    s = gemm_prepare(g3, d, workspace, 0, r * comp, 0, n_tok, r, 1, d_out, U, true,
                     OutMap{Y, 0, 1, d_out, d_out, d_out}, comp);
    if (s != BLR_OK) return s;
    s = gemm_run(g1, d, dev, st);
    return s != BLR_OK ? s : gemm_run(g3, d, dev, st);
}

blr_status blr_monarch_matmul(const void* X, int64_t n_tok, int64_t d_in, int64_t d_out, int64_t b1, int64_t b2,
                              int64_t r_blk, const void* V, const void* U, int v_layout, int out_order, void* Y,
                              void* workspace, size_t ws_bytes, blr_stream_t stream) {
    t_last_launches = 0;
    if (n_tok < 0 || d_in <= 0 || d_out <= 0 || b1 <= 0 || b2 <= 0 || r_blk <= 0) return BLR_ERR_SHAPE;
    if (d_in % b1 || d_out % b2) return BLR_ERR_SHAPE;
    if (v_layout != BLR_MON_V_B2_FASTEST && v_layout != BLR_MON_V_RPRIME_FASTEST) return BLR_ERR_SHAPE;
    if (out_order != BLR_OUT_CANONICAL && out_order != BLR_OUT_TRANSPOSED) return BLR_ERR_SHAPE;
    // output block k, column c -> Y[t, k q + c] (canonical) or Y[t, c b2 + k] (the
    // "transposed" order of PAPER.md L219-220, whose skipped permutation ③ pre-applies to the next
    // static weight's rows; blr_transposed_row_index)
    const bool ytr = out_order == BLR_OUT_TRANSPOSED;
    if (n_tok == 0) return BLR_OK;
    if (!X || !V || !U || !Y || !workspace) return BLR_ERR_NULL;
    const int64_t pdim = d_in / b1, qdim = d_out / b2, K2 = b1 * r_blk;
    if (pdim % 8 || qdim % 8 || r_blk % 8) return BLR_ERR_ALIGN;
    if (!al16(X) || !al16(V) || !al16(U) || !al16(Y) || !al16(workspace)) return BLR_ERR_ALIGN;
    if (b1 > 16 || b2 > 16 || r_blk > 256 || n_tok > (int64_t(1) << 31) - 1) return BLR_ERR_UNSUPPORTED;
    if (ws_bytes < blr_monarch_workspace_size(n_tok, d_in, d_out, b1, b2, r_blk)) return BLR_ERR_WORKSPACE;
    DevInfo d;
    int dev;
    blr_status s = device_info(d, dev);
    if (s != BLR_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (use_decode(n_tok, 256)) {  // small-n path: fp32 Z' [b2][n][b1 r'], permutations in the index maps
        float* zp = static_cast<float*>(workspace);
        DtcPrep p1, p2;
        s = dtc_prepare(p1, X, 0, d_in, pdim, V, 1, pdim, r_blk * b2 * pdim, zp, 0, K2, n_tok * K2, 1, n_tok, pdim,
                        r_blk * b2, b1, 0);
        if (s != BLR_OK) return s;
        p1.d.col_map = v_layout == BLR_MON_V_B2_FASTEST ? 1 : 2;  // column c of block l -> (k, rho)
        p1.d.mon_b2 = static_cast<int>(b2);
        p1.d.mon_r = static_cast<int>(r_blk);
        s = dtc_prepare(p2, zp, 1, K2, n_tok * K2, U, 1, K2, qdim * K2, Y, 1, d_out, ytr ? 1 : qdim, ytr ? b2 : 1,
                        n_tok, K2, qdim, b2, 1);
        if (s != BLR_OK) return s;
        s = dtc_launch(p1, st);
        return s != BLR_OK ? s : dtc_launch(p2, st);
    }
    if (fused_wanted(n_tok, K2, r_blk, false)) {  // one launch, Z'_k on chip (blr_fused.cuh)
        blr::FParams p = {};
        p.n_tok = static_cast<int>(n_tok);
        p.mon = 1;
        p.g1 = static_cast<int>(b1);
        p.k1_blocks = static_cast<int>(cdiv(pdim, blr::BK));
        p.n1 = static_cast<int>(r_blk);
        p.b1_mn = 0;
        p.g2 = static_cast<int>(b2);
        p.n2 = static_cast<int>(qdim);
        p.b2_mn = 0;
        if (ytr) {
            p.y = static_cast<__nv_bfloat16*>(Y);
            p.y_rs = d_out;
            p.y_cs = static_cast<int>(b2);
        }
        CUtensorMap ta, tb1, tb2;
        if (!encode_x_blocked(&ta, X, n_tok, b1, pdim)) return BLR_ERR_CUDA;
        {   // V viewed 4-D (a, rho', k, l): box (64, r', 1, 1) = the r' rows m(rho, k) of block (l, k)
            const uint64_t dims[4] = {static_cast<uint64_t>(pdim), static_cast<uint64_t>(r_blk),
                                      static_cast<uint64_t>(b2), static_cast<uint64_t>(b1)};
            uint64_t str[3];
            if (v_layout == BLR_MON_V_B2_FASTEST) {  // m = rho*b2 + k
                str[0] = static_cast<uint64_t>(b2 * pdim) * 2;
                str[1] = static_cast<uint64_t>(pdim) * 2;
            } else {  // m = k*r' + rho
                str[0] = static_cast<uint64_t>(pdim) * 2;
                str[1] = static_cast<uint64_t>(r_blk * pdim) * 2;
            }
            str[2] = static_cast<uint64_t>(r_blk * b2 * pdim) * 2;
            const uint32_t box[4] = {blr::BK, static_cast<uint32_t>(r_blk), 1, 1};
            if (!encode(&tb1, V, 4, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
        }
        {   // U [b2][q][b1 r'] K-major; box (64 K, bn2 rows, 1)
            const int64_t bn2 = rup(cdiv(qdim, cdiv(qdim, 256)), 16);
            const uint64_t dims[3] = {static_cast<uint64_t>(K2), static_cast<uint64_t>(qdim), static_cast<uint64_t>(b2)};
            const uint64_t str[2] = {static_cast<uint64_t>(K2) * 2, static_cast<uint64_t>(K2 * qdim) * 2};
            const uint32_t box[3] = {blr::BK, static_cast<uint32_t>(bn2), 1};
            if (!encode(&tb2, U, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
        }
        s = fused_launch(d, dev, st, p, ta, tb1, tb2, Y, d_out);
        if (s != BLR_ERR_UNSUPPORTED) return s;
    }
    const int comp = comp_factor(K2);

    // ---- phase 1: Z'[k][t][l r' + rho] = (X_l V_{l,k})[t, rho]  (block-diagonal S1 + permutations)
    {
        // k blocks per N tile: BN = kb r' <= 256 and a multiple of 16; fewer while SMs would idle
        auto plan_mon = [&](KParams& p, int pair) -> bool {
            p = KParams{};
            p.n_tok = static_cast<int>(n_tok);
            p.tiles_m = static_cast<int>(cdiv(n_tok, blr::BM * pair));
            int kb = std::max<int>(1, std::min<int>(static_cast<int>(b2), 256 / static_cast<int>(r_blk)));
            while (kb > 1 && ((kb * r_blk) % 16 || kb % pair)) --kb;
            if ((kb * r_blk) % 16 || kb % pair) kb = 2;  // r' odd multiple of 8: pair two k blocks
            while (kb > 2 * pair && p.tiles_m * b1 * cdiv(b2, kb) < d.sm_count / pair) {
                int nk = kb - 1;
                while (nk > 1 && ((nk * r_blk) % 16 || nk % pair)) --nk;
                if ((nk * r_blk) % 16 || nk % pair || nk * r_blk < 64) break;
                kb = nk;
            }
            p.kb_per_tile = kb;
            p.BN = static_cast<int>(kb * r_blk);
            p.N = static_cast<int>(r_blk * b2);
            p.tiles_n = static_cast<int>(cdiv(b2, kb));
            p.groups = static_cast<int>(b1);
            p.total_tiles = p.tiles_m * p.groups * p.tiles_n;
            p.k_blocks = p.kb_half = static_cast<int>(cdiv(pdim, blr::BK));
            p.n_sub = 1;
            p.BN /= pair;  // this CTA's share of B rows
            set_b_staging(p, false);
            p.BN *= pair;
            p.r_blk = static_cast<int>(r_blk);
            p.out_lo_off = comp == 2 ? K2 : 0;
            // staged chunk inside one output block k (CW divides r'); an r' without a wide
            // multiple-of-8 divisor (e.g. 88 = 8 * 11) stores whole unswizzled r'-wide rows instead
            // of 8-column boxes (16-B rows made the C4X Monarch S1 TMA-op bound: 4.4 ms vs 1.1 ms)
            p.c_box_w = chunk_width(static_cast<int>(r_blk));
            if (p.c_box_w < 32 && r_blk <= 128) p.c_box_w = static_cast<int>(r_blk);
            p.c_swz = pick_swz(p.c_box_w * 2).mask;
            // weight-stationary only when every slice gets >= 2 CTAs: with short K (p) a tile's MMA is
            // brief and slice ownership idles SMs (measured on Llama-7B: streaming 1.22 ms vs 1.44 ms)
            const bool allow_res = static_cast<int64_t>(b1) * p.tiles_n * 2 <= d.sm_count / pair;
            return p.BN <= 256 && p.kb_per_tile % pair == 0 &&
                   finish_plan(p, allow_res, 32 * p.c_box_w * 2, d.sm_count / pair);
        };
        KParams p;
        int pair = 1;
        const char* pe = getenv("BLR_PAIR");
        const int force = pe ? atoi(pe) : 2;  // pairs by default (see gemm_prepare)
        // BLR_PAIR=0 heuristic (generic producer era): pairs won for a long block contraction (down
        // S1, p = 688: 3.05 -> 2.57 ms) and lost for a short one (gate S1, p = 256: 1.33 -> 1.89 ms)
        if (force == 2 && n_tok >= 256) pair = 2;
        if (force == 0 && n_tok >= 1024 && pdim >= 512) pair = 2;
        if (!plan_mon(p, pair)) {
            if (pair == 1 || !plan_mon(p, pair = 1)) return BLR_ERR_UNSUPPORTED;
        }
        const int kb = p.kb_per_tile;
        const Swz cs = pick_swz(p.c_box_w * 2);
        CUtensorMap ta, tb, tc;
        if (!encode_x_blocked(&ta, X, n_tok, b1, pdim)) return BLR_ERR_CUDA;
        // V viewed 4-D (a, rho', k, l) so the box (64, r', kb, 1) lands k-major in smem:
        // this is where the r' <-> b2 permutation of PAPER.md L194 happens (no extra pass).
        const uint64_t dims[4] = {static_cast<uint64_t>(pdim), static_cast<uint64_t>(r_blk),
                                  static_cast<uint64_t>(b2), static_cast<uint64_t>(b1)};
        uint64_t str[3];
        if (v_layout == BLR_MON_V_B2_FASTEST) {  // m = rho*b2 + k
            str[0] = static_cast<uint64_t>(b2 * pdim) * 2;
            str[1] = static_cast<uint64_t>(pdim) * 2;
        } else {  // m = k*r' + rho
            str[0] = static_cast<uint64_t>(pdim) * 2;
            str[1] = static_cast<uint64_t>(r_blk * pdim) * 2;
        }
        str[2] = static_cast<uint64_t>(r_blk * b2 * pdim) * 2;
        const uint32_t box[4] = {blr::BK, static_cast<uint32_t>(r_blk), static_cast<uint32_t>(kb / pair), 1};
        if (!encode(&tb, V, 4, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
        // Z' viewed (rho', l, comp, t, k): element at ((k*n + t)*comp + part)*K2 + l*r' + rho'
        const uint64_t cd[5] = {static_cast<uint64_t>(r_blk), static_cast<uint64_t>(b1), static_cast<uint64_t>(comp),
                                static_cast<uint64_t>(n_tok), static_cast<uint64_t>(b2)};
        const uint64_t cstr[4] = {static_cast<uint64_t>(r_blk) * 2, static_cast<uint64_t>(K2) * 2,
                                  static_cast<uint64_t>(K2 * comp) * 2, static_cast<uint64_t>(K2 * comp * n_tok) * 2};
        // 128-row cooperative stores (KParams::coop_store, BLR_COOP=0: per-warp 32-row boxes)
        const char* ce = getenv("BLR_COOP");
        p.coop_store = (p.c_box_w <= 64 && !(ce && ce[0] == '0')) ? 1 : 0;
        const uint32_t cbox[5] = {static_cast<uint32_t>(p.c_box_w), 1, 1, p.coop_store ? 128u : 32u, 1};
        if (!encode(&tc, workspace, 5, cd, cstr, cbox, cs.mode)) return BLR_ERR_CUDA;
        // ---- phase 2: Y[t, k q + c] = sum_kk Z'[k][t][kk] U[k][c][kk]  (U is [N][K]: K-major B),
        //      planned before phase 1 is launched
        GemmPrep g2;
        OutMap ymap{Y, 0, 1, d_out, ytr ? 1 : qdim, d_out};
        ymap.col_stride = ytr ? b2 : 0;
        s = gemm_prepare(g2, d, workspace, 0, K2 * comp, n_tok * K2 * comp, n_tok, K2, b2, qdim, U, false, ymap, comp);
        if (s != BLR_OK) return s;
        s = pair == 2 ? launch<blr::KIND_MONARCH_PROJ, 2>(ta, tb, tc, p, d, dev, st)
                      : launch<blr::KIND_MONARCH_PROJ, 1>(ta, tb, tc, p, d, dev, st);
        if (s != BLR_OK) return s;
        return gemm_run(g2, d, dev, st);
    }
}

}  // extern "C"

namespace {
// fp8z: the split path stores Z_l as e4m3; elsewhere identical
// ---- pipelined BLAST layer (blast_pipe_kernel) --------------------------------
constexpr int PIPE_STATIC_SMEM = 16;  // the role ticket after the roles' smem, kept free of the plans
// Opt-in (BLR_PIPE=1): measured slower than the three launches so far -- its S2 role needs ~40 SMs
// to keep up (C4 gate layer 8.4 vs 4.35 ms)
bool pipe_wanted(int64_t n_tok, int64_t b1, int64_t b2, int64_t r) {
    if (b1 > 16 || b2 > 16 || r % 8) return false;
    const char* e = getenv("BLR_PIPE");
    return e && e[0] == '1' && n_tok >= 256;
}

// Clusters (CTA pairs) per role, from the phases' work: tensor FLOPs of S1 and S3, S2's bytes at
// an assumed per-cluster rate (BLR_PIPE_SPLIT="n1,n2" overrides; the rest go to S3).
void pipe_split(int units, double f1, double f3, double b2_bytes, int& n1, int& n2, int& n3) {
    const char* e = getenv("BLR_PIPE_SPLIT");
    if (e && sscanf(e, "%d,%d", &n1, &n2) == 2 && n1 >= 1 && n2 >= 1 && n1 + n2 < units) {
        n3 = units - n1 - n2;
        return;
    }
    // per-cluster rates: ~2 x 5.5 TFLOP/s on the tensor cores (measured C4 GEMM phases), ~0.2 TB/s
    // of S2 traffic (L2-resident Z / Z'')
    const double t1 = f1 / 11e12, t3 = f3 / 11e12, t2 = b2_bytes / 0.2e12;
    const double tot = t1 + t2 + t3;
    n1 = std::max(1, static_cast<int>(units * t1 / tot + 0.5));
    n2 = std::max(1, static_cast<int>(units * t2 / tot + 0.5));
    n3 = units - n1 - n2;
    if (n3 < 1) {
        n3 = 1;
        n1 = std::max(1, units - n2 - n3);
        n2 = units - n1 - n3;
    }
}

blr_status blast_pipe(const DevInfo& d, int dev, cudaStream_t st, const void* X, int64_t d_in, int64_t pdim,
                      int64_t n_tok, int64_t b1, int64_t b2, int64_t r, const void* V, const void* S, const void* U,
                      void* Y, int64_t qdim, void* zl, void* zpp, void* ctr_mem, const CUtensorMap& tmz,
                      const CUtensorMap& tmzpp) {
    const int64_t n_pad = rup(n_tok, blr::BM);
    const int tiles = static_cast<int>(cdiv(n_tok, blr::BM));
    const int tiles_pad = static_cast<int>(2 * cdiv(n_tok, 2 * blr::BM));
    const int64_t d_out = b2 * qdim;
    GemmPrep g1, g3;
    OutMap zmap{zl, 2, 1, r, n_pad * r, r};
    zmap.blocked = 1;
    // both GEMM roles as CTA pairs with streamed weights (token-tile-ordered walks)
    t_smem_reserve = PIPE_STATIC_SMEM;
    blr_status s = gemm_prepare(g1, d, X, 1, d_in, pdim, n_tok, pdim, b1, r, V, true, zmap, 1, 0, 2, true);
    if (s == BLR_OK)
        s = gemm_prepare(g3, d, zpp, 0, r, n_tok * r, n_tok, r, b2, qdim, U, true, OutMap{Y, 0, 1, d_out, qdim, d_out},
                         1, /*a_blocked=*/1, 2, true);
    t_smem_reserve = 0;
    const bool plan_print = getenv("BLR_PLAN") && getenv("BLR_PLAN")[0] == '1';
    if (s != BLR_OK) {
        if (plan_print) fprintf(stderr, "[blr plan] pipe: role planning failed (%d)\n", static_cast<int>(s));
        return s;
    }
    if (g1.pair != 2 || g1.outf != 2 || g1.p.b_resident || g3.pair != 2 || g3.outf != 0 || g3.p.b_resident ||
        g1.p.mc > 1 || g3.p.mc > 1) {
        if (plan_print) fprintf(stderr, "[blr plan] pipe: role plans unsupported, three launches\n");
        return BLR_ERR_UNSUPPORTED;
    }
    const blr::S2MLayout sl = blr::s2m_layout(static_cast<int>(b1), static_cast<int>(b2), false);
    const uint32_t tot1 = blr::smem_layout(g1.p).total, tot3 = blr::smem_layout(g3.p).total;
    const uint32_t dyn = std::max(std::max(tot1, tot3), sl.total) + SMEM_SLACK;
    if (dyn + PIPE_STATIC_SMEM > static_cast<uint32_t>(SMEM_LIMIT)) {
        if (plan_print) fprintf(stderr, "[blr plan] pipe: %u B of smem, three launches\n", dyn);
        return BLR_ERR_UNSUPPORTED;
    }
    unsigned int* ctr = static_cast<unsigned int*>(ctr_mem);
    auto prep = [&](KParams& p) {
        p.trace = nullptr;
        p.first = 1;  // every role waits for the previous grid before loading anything
        p.no_trigger = 1;
        p.mma_burst = 1;
        p.fast_prod = 1;
        p.dbg = 0;
    };
    KParams p1 = g1.p, p3 = g3.p;
    prep(p1);
    prep(p3);
    p1.pipe_sig = ctr + 1;
    p3.pipe_wait = ctr + 1 + tiles_pad;
    // S1 stays at most `bp` token tiles ahead of S2 (Z still in L2 when S2 reads it; BLR_PIPE_BP=0: off).
    // Safe because every CTA of the grid is co-resident (grid <= SMs, one CTA per SM, no early trigger).
    // (bp >= the S2 window: a smaller distance would make S1's last tiles of a window wait for S2
    //  items of that same window, which S2 starts only once the whole window is ready -- a cycle)
    int bp = 2 * blr::S2_PIPE_WIN;
    if (const char* be = getenv("BLR_PIPE_BP")) bp = atoi(be);
    if (bp > 0) {
        p1.pipe_bp = ctr + 1 + tiles_pad;
        p1.pipe_bp_target = static_cast<unsigned int>(r / 8);
        p1.pipe_bp_dist = bp;
    }
    p3.pipe_target = static_cast<unsigned int>(r / 8);
    blr::PipeArgs pa = {};
    pa.ctr = ctr;
    pa.Z = zl;
    pa.Zpp = static_cast<__nv_bfloat16*>(zpp);
    pa.S = static_cast<const __nv_bfloat16*>(S);
    pa.n_tok = static_cast<int>(n_tok);
    pa.b1 = static_cast<int>(b1);
    pa.b2 = static_cast<int>(b2);
    pa.r = static_cast<int>(r);
    pa.z_target = static_cast<unsigned int>(b1 * p1.tiles_n * 2);
    pa.tiles_pad = tiles_pad;
    // L2 policy (BLR_PIPE_HINTS=0: none): the handed-over Z / Z'' evict-last, the streams that are
    // read once (X, Y, Z after S2) evict-first, the weights evict-last
    const char* he = getenv("BLR_PIPE_HINTS");
    if (!(he && he[0] == '0')) {
        p1.l2_a = 1;
        p1.l2_b = 2;
        p1.l2_out = 2;
        pa.l2_z = 1;
        pa.l2_zz = 2;
        p3.l2_b = 2;
        p3.l2_out = 1;
    }
    pa.win = blr::S2_PIPE_WIN;
    if (const char* we = getenv("BLR_PIPE_WIN")) pa.win = std::max(1, atoi(we));
    if (p1.pipe_bp != nullptr) p1.pipe_bp_dist = std::max(p1.pipe_bp_dist, pa.win);
#ifdef BLR_DEBUG_KNOBS
    if (const char* de = getenv("BLR_PIPE_DBG")) pa.dbg = atoi(de);
    if (pa.dbg & 4) p3.pipe_wait = nullptr;  // S3 does not wait (timing experiment; results wrong)
#endif
    const int units = d.sm_count / 2;
    const double f1 = 2.0 * n_tok * d_in * r, f3 = 2.0 * n_tok * r * qdim * b2;
    pipe_split(units, f1, f3, 2.0 * n_tok * r * (b1 + b2), pa.n1, pa.n2, pa.n3);
    (void)tiles;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!g_attr_set[22][dev]) {
            if (const cudaError_t ae = cudaFuncSetAttribute(blr::blast_pipe_kernel,
                                                            cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                            SMEM_LIMIT);
                ae != cudaSuccess) {
                if (plan_print) fprintf(stderr, "[blr plan] pipe attribute: %s\n", cudaGetErrorString(ae));
                return BLR_ERR_CUDA;
            }
            g_attr_set[22][dev] = true;
        }
    }
    if (const char* pe = getenv("BLR_PLAN"); pe && pe[0] == '1')
        fprintf(stderr,
                "[blr plan] pipe clusters S1/S2/S3 = %d/%d/%d  S1 BN=%d stages=%d  S3 BN=%d stages=%d  dyn smem=%u\n",
                pa.n1, pa.n2, pa.n3, p1.BN, p1.stages, p3.BN, p3.stages, dyn);
    if (const cudaError_t me = cudaMemsetAsync(ctr, 0, pipe_ctr_bytes(n_tok), st); me != cudaSuccess) {
        if (plan_print) fprintf(stderr, "[blr plan] pipe memset: %s\n", cudaGetErrorString(me));
        return BLR_ERR_CUDA;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(2 * (pa.n1 + pa.n2 + pa.n3)));
    cfg.blockDim = dim3(blr::NUM_THREADS);
    pa.ticket_off = dyn;
    cfg.dynamicSmemBytes = dyn + PIPE_STATIC_SMEM;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = 2;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const bool prof = t_prof_events != nullptr && 2 * t_prof_n + 1 < t_prof_cap;
    if (prof && prof_record(t_prof_events[2 * t_prof_n], st) != cudaSuccess) return BLR_ERR_CUDA;
    if (const cudaError_t le = cudaLaunchKernelEx(&cfg, blr::blast_pipe_kernel, g1.ta, g1.tb, g1.tc, tmz, tmzpp, g3.ta,
                                                  g3.tb, g3.tc, g1.tb2, g3.tb2, p1, p3, pa);
        le != cudaSuccess) {
        if (plan_print) fprintf(stderr, "[blr plan] pipe launch: %s\n", cudaGetErrorString(le));
        return BLR_ERR_CUDA;
    }
    if (prof) {
        if (prof_record(t_prof_events[2 * t_prof_n + 1], st) != cudaSuccess) return BLR_ERR_CUDA;
        ++t_prof_n;
    }
    ++t_last_launches;
    return BLR_OK;
}

blr_status blast_impl(const void* X, int64_t n_tok, int64_t d_in, int64_t d_out, int64_t b1, int64_t b2, int64_t r,
                      const void* V, const void* S, const void* U, void* Y, void* workspace, size_t ws_bytes,
                      blr_stream_t stream, bool fp8z, bool kmaj = false) {
    t_last_launches = 0;
    if (n_tok < 0 || d_in <= 0 || d_out <= 0 || b1 <= 0 || b2 <= 0 || r <= 0) return BLR_ERR_SHAPE;
    if (d_in % b1 || d_out % b2) return BLR_ERR_SHAPE;
    if (n_tok == 0) return BLR_OK;
    if (!X || !V || !S || !U || !Y || !workspace) return BLR_ERR_NULL;
    const int64_t pdim = d_in / b1, qdim = d_out / b2;
    if (pdim % 8 || qdim % 8 || r % 8) return BLR_ERR_ALIGN;
    if (!al16(X) || !al16(V) || !al16(S) || !al16(U) || !al16(Y) || !al16(workspace)) return BLR_ERR_ALIGN;
    if (b1 > 16 || b2 > 16 || n_tok > (int64_t(1) << 31) - 1) return BLR_ERR_UNSUPPORTED;
    if (ws_bytes < blr_blast_workspace_size(n_tok, d_in, d_out, b1, b2, r)) return BLR_ERR_WORKSPACE;
    DevInfo d;
    int dev;
    blr_status s = device_info(d, dev);
    if (s != BLR_OK) return s;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    // small n: the weight-streaming kernels; up to 2048 tokens where the tcgen05 alternative is the
    // S1+S2-fused projection, whose parallelism is the handful of 128-token tiles (C1, C5 ViT-B)
    // K-major factors (blr_blast_matmul_kmajor): the split tensor-core path only
    if (kmaj && (use_decode(n_tok, blast_fused(b1, r) ? 2048 : 16) || blast_fused(b1, r) || comp_factor(r) != 1 || fp8z))
        return BLR_ERR_UNSUPPORTED;
    if (use_decode(n_tok, blast_fused(b1, r) ? 2048 : 16)) {  // fp32 Z [b1][n][r] (unless fused away), Z'' [b2][n][r]
        float* z = static_cast<float*>(workspace);
        float* zp2 = z + b1 * n_tok * r;
        int cs = 0, units = 0;
        DtcPrep p1, p3;
        bool mix = dtc_blast_mix_ok(b1, pdim, cs, units);
        if (mix) {  // S1 + S2 in one launch: Z stays in the cluster's shared memory
            s = dtc_prepare_blast_mix(p1, X, d_in, pdim, V, S, zp2, n_tok, b1, b2, r, cs, units);
            if (s == BLR_ERR_UNSUPPORTED) mix = false;
            else if (s != BLR_OK) return s;
        }
        if (!mix) {
            s = dtc_prepare(p1, X, 0, d_in, pdim, V, 0, r, pdim * r, z, 0, r, n_tok * r, 1, n_tok, pdim, r, b1, 0);
            if (s != BLR_OK) return s;
        }
        s = dtc_prepare(p3, zp2, 1, r, n_tok * r, U, 0, qdim, r * qdim, Y, 1, d_out, qdim, 1, n_tok, r, qdim, b2, 1);
        if (s != BLR_OK) return s;
        s = dtc_launch(p1, st);
        if (s != BLR_OK) return s;
        if (!mix) {  // S2 on its own: Z'' = sum_l S_l,k * Z_l (fp32)
            cudaLaunchConfig_t cfg = {};
            const int64_t count = b2 * n_tok * r;
            cfg.gridDim = dim3(static_cast<unsigned>(std::min<int64_t>(cdiv(count, blr::DECODE_THREADS), 4 * 148)));
            cfg.blockDim = dim3(blr::DECODE_THREADS);
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            const bool prof = t_prof_events != nullptr && 2 * t_prof_n + 1 < t_prof_cap;
            if (prof && prof_record(t_prof_events[2 * t_prof_n], st) != cudaSuccess) return BLR_ERR_CUDA;
            if (cudaLaunchKernelEx(&cfg, blr::decode_s2_kernel, static_cast<const float*>(z),
                                   static_cast<const __nv_bfloat16*>(S), zp2, static_cast<int>(n_tok),
                                   static_cast<int>(b1), static_cast<int>(b2), static_cast<int>(r)) != cudaSuccess)
                return BLR_ERR_CUDA;
            if (prof) {
                if (prof_record(t_prof_events[2 * t_prof_n + 1], st) != cudaSuccess) return BLR_ERR_CUDA;
                ++t_prof_n;
            }
            ++t_last_launches;
        }
        return dtc_launch(p3, st);
    }
    const int comp = comp_factor(r);
    void* zpp = workspace;  // Z'' [b2][n][r*comp] (split path: tile-blocked, then fp16 Z after it)

    if (blast_fused(b1, r)) {
        // ---- phase 1: Z''[k][t][rho] = sum_l S[l,k,rho] (X_l V_l)[t, rho]  (S1 on tcgen05, S2 fused)
        KParams p = {};
        // rho-chunk R: b1 TMEM accumulators of R columns, and b2 staged outputs of R/2 columns per
        // warp (<= 16 KB): b1*R <= 512, b2*R <= 512, R <= 128.
        int R = 128;
        while (R > 16 && (b1 * R > blr::TMEM_COLS || b2 * R > 512)) R >>= 1;
        while (R > 16 && R / 2 >= rup(r, 16)) R >>= 1;
        p.BN = R;
        p.N = static_cast<int>(r);
        p.n_tok = static_cast<int>(n_tok);
        p.tiles_m = static_cast<int>(cdiv(n_tok, blr::BM));
        p.tiles_n = static_cast<int>(cdiv(r, R));
        p.groups = 1;
        p.total_tiles = p.tiles_m * p.tiles_n;
        p.k_blocks = p.kb_half = static_cast<int>(cdiv(pdim, blr::BK));
        p.n_sub = static_cast<int>(b1);
        set_b_staging(p, true);
        p.b1 = static_cast<int>(b1);
        p.b2 = static_cast<int>(b2);
        p.r = static_cast<int>(r);
        p.S = static_cast<const __nv_bfloat16*>(S);
        p.out_lo_off = comp == 2 ? r : 0;
        p.c_box_w = R / 2;
        p.c_swz = pick_swz(R).mask;
        p.stage_warp_bytes = static_cast<uint32_t>(b2) * 32u * (R / 2) * 2u;
        if (!finish_plan(p, false, 0, d.sm_count)) return BLR_ERR_UNSUPPORTED;
        CUtensorMap ta, tb, tc;
        if (!encode_x_blocked(&ta, X, n_tok, b1, pdim)) return BLR_ERR_CUDA;
        const uint64_t dims[3] = {static_cast<uint64_t>(r), static_cast<uint64_t>(pdim), static_cast<uint64_t>(b1)};
        const uint64_t str[2] = {static_cast<uint64_t>(r) * 2, static_cast<uint64_t>(r * pdim) * 2};
        const uint32_t box[3] = {64, blr::BK, 1};
        if (!encode(&tb, V, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
        // Z'' viewed (rho, comp, t, k): element at ((k*n + t)*comp + part)*r + rho
        const uint64_t cd[4] = {static_cast<uint64_t>(r), static_cast<uint64_t>(comp), static_cast<uint64_t>(n_tok),
                                static_cast<uint64_t>(b2)};
        const uint64_t cstr[3] = {static_cast<uint64_t>(r) * 2, static_cast<uint64_t>(r * comp) * 2,
                                  static_cast<uint64_t>(r * comp * n_tok) * 2};
        const char* ce = getenv("BLR_COOP");
        p.coop_store = (ce && ce[0] == '0') ? 0 : 1;  // 128-row cooperative stores of Z''
        const uint32_t cbox[4] = {static_cast<uint32_t>(R / 2), 1, p.coop_store ? 128u : 32u, 1};
        if (!encode(&tc, zpp, 4, cd, cstr, cbox, pick_swz(R).mode)) return BLR_ERR_CUDA;
        // ---- S3: Y_k = Z''_k U_k  (U is [b2][r][q]: MN-major B), planned before phase 1 launches
        GemmPrep g3;
        s = gemm_prepare(g3, d, zpp, 0, r * comp, n_tok * r * comp, n_tok, r, b2, qdim, U, true,
                         OutMap{Y, 0, 1, d_out, qdim, d_out}, comp);
        if (s != BLR_OK) return s;
        s = launch<blr::KIND_BLAST_PROJ, 1>(ta, tb, tc, p, d, dev, st);
        return s != BLR_OK ? s : gemm_run(g3, d, dev, st);
    }

    // ---- split path (b1 r > TMEM): S1 grouped GEMM -> fp16 Z, S2, S3.  Every phase is planned and
    //      every tensor map encoded before S1 is launched.
    const char* s2e = getenv("BLR_S2");
    // tensor-core S2 (single-rounded Z''): Z and Z'' tile-blocked [g][T][r/8][128][8]
    const bool s2_mma = comp == 1 && !(s2e && !strcmp(s2e, "cuda"));
    if (kmaj && !s2_mma) return BLR_ERR_UNSUPPORTED;  // (K-major factors: tensor-core S2 path only)
    const int64_t n_pad = rup(n_tok, blr::BM);
    void* zl = static_cast<char*>(workspace) + static_cast<size_t>(b2) * n_pad * r * 2 * comp;
    // S1: Z[l][t][rho] = (X_l V_l)[t, rho]  -- grouped GEMM over l (A = X viewed (p, b1, n));
    // tile-blocked Z for the tensor-core S2: [l][T][r/8][128][8], group stride n_pad * r
    // (FP8 mode: e4m3 bytes in the same layout; only with the tensor-core S2)
    const bool z8 = fp8z && s2_mma;
    OutMap zmap{zl, z8 ? 3 : 2, 1, r, s2_mma ? n_pad * r : n_tok * r, r};
    zmap.blocked = s2_mma ? 1 : 0;
    GemmPrep g1, g3;
    s = gemm_prepare(g1, d, X, 1, d_in, pdim, n_tok, pdim, b1, r, V, !kmaj, zmap, 1);
    if (s != BLR_OK) return s;
    // S3: Y_k = Z''_k U_k (U is [b2][r][q]: MN-major B; kmaj: Ut [b2][q][r], K-major); A tile-blocked
    // after the tensor-core S2
    s = s2_mma ? gemm_prepare(g3, d, zpp, 0, r, n_tok * r, n_tok, r, b2, qdim, U, !kmaj,
                              OutMap{Y, 0, 1, d_out, qdim, d_out}, 1, /*a_blocked=*/1)
               : gemm_prepare(g3, d, zpp, 0, r * comp, n_tok * r * comp, n_tok, r, b2, qdim, U, true,
                              OutMap{Y, 0, 1, d_out, qdim, d_out}, comp);
    if (s != BLR_OK) return s;

    if (s2_mma) {
        // ---- S2 on the tensor cores (blast_s2_mma_kernel): tile-blocked fp16 Z [l][T][r/8][128][8]
        //      in, tile-blocked bf16 Z'' [k][T][r/8][128][8] out
        const char* oe = getenv("BLR_S2_ORDER");
        const int s2_order = oe ? atoi(oe) : 0;
        const int64_t items = cdiv(n_tok, 128) * (r / 8);
        // b2 <= 8: the half-register instantiation, two CTAs per SM when both fit in smem
        const char* se = getenv("BLR_S2_SMALL");
        const bool small = b2 <= 8 && !(se && se[0] == '0');
        const blr::S2MLayout sl8 = blr::s2m_layout(static_cast<int>(b1), static_cast<int>(b2), z8);
        const int per_sm = (small && 2 * (sl8.total + 1024 + 1024) <= 233472) ? 2 : 1;
        auto s2fn = z8 ? (small ? blr::blast_s2_mma_kernel<8, true> : blr::blast_s2_mma_kernel<16, true>)
                       : (small ? blr::blast_s2_mma_kernel<8> : blr::blast_s2_mma_kernel<16>);
        const char* pe2 = getenv("BLR_S2_PDL");
        const bool s2_pdl = pdl_enabled() && !(pe2 && pe2[0] == '0');
        CUtensorMap tmz, tmzpp;
        {   // Z / Z'' tile-blocked [g][T][r/8][128][8] viewed (64 elem, 16 rows, T*r/8 panels, g)
            const int64_t np = cdiv(n_tok, blr::BM) * (r / 8);
            const uint64_t dz[4] = {64, 16, static_cast<uint64_t>(np), static_cast<uint64_t>(b1)};
            const uint64_t sz[3] = {128, 2048, static_cast<uint64_t>(np) * 2048};
            const uint32_t bz[4] = {64, 16, 1, static_cast<uint32_t>(b1)};
            const uint64_t sz8[3] = {64, 1024, static_cast<uint64_t>(np) * 1024};  // e4m3: 1-KB panels
            if (!encode(&tmz, zl, 4, dz, z8 ? sz8 : sz, bz, CU_TENSOR_MAP_SWIZZLE_NONE, z8 ? 3 : 2)) return BLR_ERR_CUDA;
            const uint64_t dp[4] = {64, 16, static_cast<uint64_t>(np), static_cast<uint64_t>(b2)};
            const uint32_t bp[4] = {64, 16, 1, static_cast<uint32_t>(b2)};
            if (!encode(&tmzpp, zpp, 4, dp, sz, bp, CU_TENSOR_MAP_SWIZZLE_NONE)) return BLR_ERR_CUDA;
        }
        {
            std::lock_guard<std::mutex> lk(g_mu);
            if (!g_attr_set[20][dev]) {
                if (cudaFuncSetAttribute(blr::blast_s2_mma_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         232448) != cudaSuccess ||
                    cudaFuncSetAttribute(blr::blast_s2_mma_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         232448) != cudaSuccess ||
                    cudaFuncSetAttribute(blr::blast_s2_mma_kernel<8, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         232448) != cudaSuccess ||
                    cudaFuncSetAttribute(blr::blast_s2_mma_kernel<16, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         232448) != cudaSuccess)
                    return BLR_ERR_CUDA;
                g_attr_set[20][dev] = true;
            }
        }
        auto run_s2 = [&](int64_t t0o, int64_t ntok, const CUtensorMap& mz) -> blr_status {  // t0o: Z'' tile offset
            const int64_t its = cdiv(ntok, 128) * (r / 8);
            cudaLaunchConfig_t cfg = {};
            int64_t s2_grid = std::min<int64_t>(its, static_cast<int64_t>(per_sm) * d.sm_count);
            if (const char* ge = getenv("BLR_S2_GRID")) s2_grid = std::max<int64_t>(1, std::min<int64_t>(s2_grid, atoi(ge)));
            cfg.gridDim = dim3(static_cast<unsigned>(s2_grid));  // (BLR_S2_GRID: per-CTA throughput experiments)
            cfg.blockDim = dim3(z8 ? blr::S2M_THREADS_FP8 : blr::S2M_THREADS);
            cfg.dynamicSmemBytes = sl8.total + 1024;
            cfg.stream = st;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = s2_pdl ? 1 : 0;
            cfg.attrs = attr;
            cfg.numAttrs = 1;
            const bool prof = t_prof_events != nullptr && 2 * t_prof_n + 1 < t_prof_cap;
            if (prof && prof_record(t_prof_events[2 * t_prof_n], st) != cudaSuccess) return BLR_ERR_CUDA;
            if (cudaLaunchKernelEx(&cfg, s2fn, mz, tmzpp, static_cast<const void*>(zl),
                                   static_cast<__nv_bfloat16*>(zpp), static_cast<const __nv_bfloat16*>(S),
                                   static_cast<int>(ntok), static_cast<int>(b1), static_cast<int>(b2),
                                   static_cast<int>(r), s2_order, 0, static_cast<int>(t0o)) != cudaSuccess)
                return BLR_ERR_CUDA;
            if (prof) {
                if (prof_record(t_prof_events[2 * t_prof_n + 1], st) != cudaSuccess) return BLR_ERR_CUDA;
                ++t_prof_n;
            }
            ++t_last_launches;
            return BLR_OK;
        };
        (void)items;
        if (!z8 && !kmaj && pipe_wanted(n_tok, b1, b2, r)) {
            s = blast_pipe(d, dev, st, X, d_in, pdim, n_tok, b1, b2, r, V, S, U, Y, qdim, zl, zpp,
                           static_cast<char*>(zl) + static_cast<size_t>(b1) * n_pad * r * 2, tmz, tmzpp);
            if (s != BLR_ERR_UNSUPPORTED) return s;  // (unsupported: nothing was enqueued; three launches)
        }
        s = gemm_run(g1, d, dev, st);
        if (s != BLR_OK) return s;
        s = run_s2(0, n_tok, tmz);
        return s != BLR_OK ? s : gemm_run(g3, d, dev, st);
    }
    // ---- CUDA-core S2 (blast_s2_kernel; used for compensated Z'' (r < 128) or with BLR_S2=cuda):
    // fp16 Z viewed (rho, t, l), box (64, S2_ROWS, b1): one item's b1 row segments per request
    CUtensorMap tz;
    {
        const uint64_t dims[3] = {static_cast<uint64_t>(r), static_cast<uint64_t>(n_tok), static_cast<uint64_t>(b1)};
        const uint64_t str[2] = {static_cast<uint64_t>(r) * 2, static_cast<uint64_t>(r * n_tok) * 2};
        const uint32_t box[3] = {64, static_cast<uint32_t>(blr::S2_ROWS), static_cast<uint32_t>(b1)};
        if (!encode(&tz, zl, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE, 2)) return BLR_ERR_CUDA;
    }
    // KG output blocks per consumer warp (S held in registers: NL x KG packed pairs per lane;
    // NL = b1 rounded up to 4/8/16, the extra planes are zero)
    const int kg = b2 == 1 ? 1 : 2;
    const int nw = static_cast<int>(cdiv(b2, kg)) * blr::S2_RSPLIT;
    const int nl = b1 <= 4 ? 4 : b1 <= 8 ? 8 : 16;
    const int slabs = static_cast<int>(cdiv(n_tok, blr::S2_ROWS));
    const int nchunks = static_cast<int>(cdiv(r, 64));
    const int total = nchunks * slabs;
    const int map_mode = 1;
    // blocks per SM: up to 16 consumer warps per SM (<= 128 registers per thread); a multiple of
    // nchunks, at most bps block-slots per SM, >= 1 per chunk
    const int bps = std::max(1, std::min(4, 16 / nw));
    const int gpc = std::max(1, std::min(slabs, bps * d.sm_count / nchunks));
    const int grid = gpc * nchunks;
    const int ipb = static_cast<int>(cdiv(total, grid));
    const size_t stage_bytes = static_cast<size_t>(nl) * blr::S2_ROWS * 64 * 2;
    const size_t ring_bytes = (192u << 10) / bps;  // ~192 KB of ring per SM
    const int nst = static_cast<int>(std::max<size_t>(2, std::min<size_t>(blr::S2_MAX_STAGES, ring_bytes / stage_bytes)));
    const size_t smem = nst * stage_bytes + 16 * nst;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!g_attr_set[21][dev]) {
            const int mx = 220 << 10;
#define BLR_S2_ATTR(KG, NL) \
    cudaFuncSetAttribute(blr::blast_s2_kernel<KG, NL>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx) != cudaSuccess
            if (BLR_S2_ATTR(1, 4) || BLR_S2_ATTR(1, 8) || BLR_S2_ATTR(1, 16) || BLR_S2_ATTR(2, 4) ||
                BLR_S2_ATTR(2, 8) || BLR_S2_ATTR(2, 16))
                return BLR_ERR_CUDA;
#undef BLR_S2_ATTR
            g_attr_set[21][dev] = true;
        }
    }
    s = gemm_run(g1, d, dev, st);
    if (s != BLR_OK) return s;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(grid));
    cfg.blockDim = dim3(static_cast<unsigned>(32 * nw));
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    // S2 is launched without programmatic dependent launch: its blocks, started early on the
    // few SMs the S1 grid leaves idle, measured ~4 us slower per GPT2-S layer
    attr[0].val.programmaticStreamSerializationAllowed = 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    const bool prof = t_prof_events != nullptr && 2 * t_prof_n + 1 < t_prof_cap;
    if (prof && prof_record(t_prof_events[2 * t_prof_n], st) != cudaSuccess) return BLR_ERR_CUDA;
    const auto* sb = static_cast<const __nv_bfloat16*>(S);
    auto* ob = static_cast<__nv_bfloat16*>(zpp);
    const int in = static_cast<int>(n_tok), ib1 = static_cast<int>(b1), ib2 = static_cast<int>(b2),
              ir = static_cast<int>(r);
    cudaError_t le = cudaErrorInvalidValue;
    switch (kg * 32 + nl) {
#define BLR_S2_CASE(KG, NL) \
    case KG * 32 + NL: \
        le = cudaLaunchKernelEx(&cfg, blr::blast_s2_kernel<KG, NL>, tz, sb, ob, in, ib1, ib2, ir, comp, slabs, total, \
                                ipb, nchunks, map_mode, nst); \
        break;
        BLR_S2_CASE(1, 4) BLR_S2_CASE(1, 8) BLR_S2_CASE(1, 16) BLR_S2_CASE(2, 4) BLR_S2_CASE(2, 8) BLR_S2_CASE(2, 16)
#undef BLR_S2_CASE
    }
    if (le != cudaSuccess) return BLR_ERR_CUDA;
    if (prof) {
        if (prof_record(t_prof_events[2 * t_prof_n + 1], st) != cudaSuccess) return BLR_ERR_CUDA;
        ++t_prof_n;
    }
    ++t_last_launches;
    return gemm_run(g3, d, dev, st);
}

}  // namespace

extern "C" {

blr_status blr_blast_matmul(const void* X, int64_t n_tok, int64_t d_in, int64_t d_out, int64_t b1, int64_t b2,
                            int64_t r, const void* V, const void* S, const void* U, void* Y, void* workspace,
                            size_t ws_bytes, blr_stream_t stream) {
    return blast_impl(X, n_tok, d_in, d_out, b1, b2, r, V, S, U, Y, workspace, ws_bytes, stream, false);
}

blr_status blr_blast_matmul_kmajor(const void* X, int64_t n_tok, int64_t d_in, int64_t d_out, int64_t b1, int64_t b2,
                                   int64_t r, const void* Vt, const void* S, const void* Ut, void* Y, void* workspace,
                                   size_t ws_bytes, blr_stream_t stream) {
    return blast_impl(X, n_tok, d_in, d_out, b1, b2, r, Vt, S, Ut, Y, workspace, ws_bytes, stream, false, true);
}

blr_status blr_blast_matmul_fp8z(const void* X, int64_t n_tok, int64_t d_in, int64_t d_out, int64_t b1, int64_t b2,
                                 int64_t r, const void* V, const void* S, const void* U, void* Y, void* workspace,
                                 size_t ws_bytes, blr_stream_t stream) {
    return blast_impl(X, n_tok, d_in, d_out, b1, b2, r, V, S, U, Y, workspace, ws_bytes, stream, true);
}

}  // extern "C"
