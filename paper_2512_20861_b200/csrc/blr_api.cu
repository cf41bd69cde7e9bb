// blr_api.cu -- C ABI of libblr.so (include/blr.h): host-side validation, plan selection,
// TMA tensor-map encoding and kernel launches.  No torch types, no host synchronization.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "../../include/blr.h"
#include "blr_kernels.cuh"

namespace {

using blr::KParams;

constexpr int SMEM_LIMIT = 232448;  // 227 KB opt-in per CTA on sm_100

struct DevInfo {
    int ok = 0;
    int sm_count = 0;
    int cc_major = 0, cc_minor = 0;
};

std::mutex g_mu;
DevInfo g_dev[64];
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
bool g_attr_set[3][64] = {};
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

// bf16 tensor map of rank R: dims[0] innermost, strides in bytes for dims 1..R-1.
bool encode(CUtensorMap* m, const void* ptr, int rank, const uint64_t* dims, const uint64_t* strides,
            const uint32_t* box, CUtensorMapSwizzle sw) {
    cuuint32_t estr[5] = {1, 1, 1, 1, 1};
    CUresult r = g_encode(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, rank, const_cast<void*>(ptr),
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

// N tile for a plain GEMM phase: <= 256 columns, multiple of 16, balanced across tiles.
int choose_bn(int64_t N) {
    int64_t tiles = cdiv(N, 256);
    return static_cast<int>(rup(cdiv(N, tiles), 16));
}

// Fill B-operand staging parameters.
void set_b_staging(KParams& p, bool mn_major) {
    p.b_mn_major = mn_major ? 1 : 0;
    if (mn_major) {
        // B stored [K][N]: boxes of 64 N-elements (128 B rows) x BK K-rows, 128-B swizzle.
        // UMMA MN-major SW128 canonical layout: 64-element MN atoms LBO apart, 8-row K groups
        // SBO = 1024 B apart; +16 K-rows = +2048 B per UMMA_K step.
        p.b_box_n = 64;
        p.b_boxes = static_cast<int>(cdiv(p.BN, 64));
        p.b_stage_bytes = static_cast<uint32_t>(p.b_boxes * 64 * blr::BK * 2);
        p.b_lbo = 64 * 2 * blr::BK;
        p.b_sbo = 1024;
        p.b_layout = blr::ptx::LAYOUT_SW128;
        p.b_kstep = 16 * 128;
    } else {
        // B stored [N][K]: BN rows x 64 K-elements, K-major SW128 like A.
        p.b_box_n = p.BN;
        p.b_boxes = 1;
        p.b_stage_bytes = static_cast<uint32_t>(rup(static_cast<int64_t>(p.BN) * blr::BK * 2, 1024));
        p.b_lbo = 16;
        p.b_sbo = 1024;
        p.b_layout = blr::ptx::LAYOUT_SW128;
        p.b_kstep = 32;
    }
}

// Stages that fit next to the (optional) S tile.
bool finish_plan(KParams& p) {
    p.stages = blr::MAX_STAGES;
    while (p.stages > 1) {
        blr::SmemLayout L = blr::smem_layout(p);
        if (L.total + 1024 <= static_cast<uint32_t>(SMEM_LIMIT)) break;
        --p.stages;
    }
    blr::SmemLayout L = blr::smem_layout(p);
    if (L.total + 1024 > static_cast<uint32_t>(SMEM_LIMIT) || p.stages < 2) return false;
    const int cols = p.n_sub * p.BN;
    if (cols > blr::TMEM_COLS) return false;
    p.acc_bufs = (2 * cols <= blr::TMEM_COLS) ? 2 : 1;
    return true;
}

template <int KIND>
blr_status launch(const CUtensorMap& a, const CUtensorMap& b, const KParams& p, const DevInfo& d, int dev,
                  cudaStream_t stream) {
    auto kfn = blr::blr_gemm_kernel<KIND>;
    const blr::SmemLayout L = blr::smem_layout(p);
    const int smem = static_cast<int>(L.total + 1024);
    {
        std::lock_guard<std::mutex> lk(g_mu);
        if (!g_attr_set[KIND][dev]) {
            if (cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_LIMIT) != cudaSuccess)
                return BLR_ERR_CUDA;
            g_attr_set[KIND][dev] = true;
        }
    }
    const int grid = static_cast<int>(std::min<int64_t>(p.total_tiles, d.sm_count));
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(blr::NUM_THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cfg.numAttrs = 0;
    const bool prof = t_prof_events != nullptr && 2 * t_prof_n + 1 < t_prof_cap;
    if (prof && cudaEventRecord(static_cast<cudaEvent_t>(t_prof_events[2 * t_prof_n]), stream) != cudaSuccess)
        return BLR_ERR_CUDA;
    if (cudaLaunchKernelEx(&cfg, kfn, a, b, p) != cudaSuccess) return BLR_ERR_CUDA;
    if (prof) {
        if (cudaEventRecord(static_cast<cudaEvent_t>(t_prof_events[2 * t_prof_n + 1]), stream) != cudaSuccess)
            return BLR_ERR_CUDA;
        ++t_prof_n;
    }
    ++t_last_launches;
    return BLR_OK;
}

// One plain GEMM phase: out[t, g*N + c] = sum_k A[g][t][k] B[g](k, c), K-major A.
// comp == 2: A rows hold [hi | lo] (length 2K) and both halves multiply the same B rows.
// out_comp == 2: out rows hold [hi | lo] (length 2N), i.e. this phase produces an intermediate.
blr_status gemm_phase(const DevInfo& d, int dev, cudaStream_t st, const void* A, int64_t n_tok, int64_t K,
                      int64_t groups, int64_t N, const void* B, bool b_mn_major, void* out, int64_t out_ld,
                      int comp = 1, int out_comp = 1) {
    KParams p = {};
    p.n_tok = static_cast<int>(n_tok);
    p.tiles_m = static_cast<int>(cdiv(n_tok, blr::BM));
    p.BN = choose_bn(N);
    p.N = static_cast<int>(N);
    p.tiles_n = static_cast<int>(cdiv(N, p.BN));
    p.groups = static_cast<int>(groups);
    p.total_tiles = p.tiles_m * p.groups * p.tiles_n;
    p.kb_half = static_cast<int>(cdiv(K, blr::BK));
    p.k_blocks = p.kb_half * comp;
    p.a_lo_off = comp == 2 ? static_cast<int>(K) : 0;
    p.n_sub = 1;
    set_b_staging(p, b_mn_major);
    p.out = static_cast<__nv_bfloat16*>(out);
    p.out_ld = out_ld * out_comp;
    p.out_lo_off = out_comp == 2 ? out_ld : 0;
    if (!finish_plan(p)) return BLR_ERR_UNSUPPORTED;

    CUtensorMap ta, tb;
    {
        const int64_t Ka = K * comp;  // A row length
        const uint64_t dims[3] = {static_cast<uint64_t>(Ka), static_cast<uint64_t>(n_tok), static_cast<uint64_t>(groups)};
        const uint64_t str[2] = {static_cast<uint64_t>(Ka) * 2, static_cast<uint64_t>(Ka * n_tok) * 2};
        const uint32_t box[3] = {blr::BK, blr::BM, 1};
        if (!encode(&ta, A, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
    }
    if (b_mn_major) {
        const uint64_t dims[3] = {static_cast<uint64_t>(N), static_cast<uint64_t>(K), static_cast<uint64_t>(groups)};
        const uint64_t str[2] = {static_cast<uint64_t>(N) * 2, static_cast<uint64_t>(N * K) * 2};
        const uint32_t box[3] = {64, blr::BK, 1};
        if (!encode(&tb, B, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
    } else {
        const uint64_t dims[3] = {static_cast<uint64_t>(K), static_cast<uint64_t>(N), static_cast<uint64_t>(groups)};
        const uint64_t str[2] = {static_cast<uint64_t>(K) * 2, static_cast<uint64_t>(K * N) * 2};
        const uint32_t box[3] = {blr::BK, static_cast<uint32_t>(p.BN), 1};
        if (!encode(&tb, B, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
    }
    return launch<blr::KIND_GEMM>(ta, tb, p, d, dev, st);
}

// X viewed as [n_tok][b1][p] (A operand of the block-diagonal first stage).
bool encode_x_blocked(CUtensorMap* m, const void* X, int64_t n_tok, int64_t b1, int64_t pdim) {
    const uint64_t dims[3] = {static_cast<uint64_t>(pdim), static_cast<uint64_t>(b1), static_cast<uint64_t>(n_tok)};
    const uint64_t str[2] = {static_cast<uint64_t>(pdim) * 2, static_cast<uint64_t>(pdim * b1) * 2};
    const uint32_t box[3] = {blr::BK, 1, blr::BM};
    return encode(m, X, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
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

const char* blr_version(void) { return "0.1.0"; }

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

void blr_clear_cache(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    for (auto& d : g_dev) d = DevInfo();
    g_encode = nullptr;
}

size_t blr_lowrank_workspace_size(int64_t n_tok, int64_t, int64_t, int64_t r) {
    return (n_tok > 0 && r > 0) ? static_cast<size_t>(n_tok) * r * 2 * comp_factor(r) : 0;
}
size_t blr_monarch_workspace_size(int64_t n_tok, int64_t, int64_t, int64_t b1, int64_t b2, int64_t r_blk) {
    return (n_tok > 0 && b1 > 0 && b2 > 0 && r_blk > 0)
               ? static_cast<size_t>(b2) * n_tok * b1 * r_blk * 2 * comp_factor(b1 * r_blk)
               : 0;
}
size_t blr_blast_workspace_size(int64_t n_tok, int64_t, int64_t, int64_t, int64_t b2, int64_t r) {
    return (n_tok > 0 && b2 > 0 && r > 0) ? static_cast<size_t>(b2) * n_tok * r * 2 * comp_factor(r) : 0;
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
    const int comp = comp_factor(r);
    // S1: Z = X V (V is [d_in][r]: MN-major B)
    s = gemm_phase(d, dev, st, X, n_tok, d_in, 1, r, V, true, workspace, r, 1, comp);
    if (s != BLR_OK) return s;
    // S3: Y = Z U (U is [r][d_out]: MN-major B)
    return gemm_phase(d, dev, st, workspace, n_tok, r, 1, d_out, U, true, Y, d_out, comp, 1);
}

blr_status blr_monarch_matmul(const void* X, int64_t n_tok, int64_t d_in, int64_t d_out, int64_t b1, int64_t b2,
                              int64_t r_blk, const void* V, const void* U, int v_layout, int out_order, void* Y,
                              void* workspace, size_t ws_bytes, blr_stream_t stream) {
    t_last_launches = 0;
    if (n_tok < 0 || d_in <= 0 || d_out <= 0 || b1 <= 0 || b2 <= 0 || r_blk <= 0) return BLR_ERR_SHAPE;
    if (d_in % b1 || d_out % b2) return BLR_ERR_SHAPE;
    if (v_layout != BLR_MON_V_B2_FASTEST && v_layout != BLR_MON_V_RPRIME_FASTEST) return BLR_ERR_SHAPE;
    if (out_order != BLR_OUT_CANONICAL) return BLR_ERR_UNSUPPORTED;
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
    const int comp = comp_factor(K2);

    // ---- phase 1: Z'[k][t][l r' + rho] = (X_l V_{l,k})[t, rho]  (block-diagonal S1 + permutations)
    {
        KParams p = {};
        int kb = std::max<int>(1, std::min<int>(static_cast<int>(b2), 256 / static_cast<int>(r_blk)));
        while (kb > 1 && (kb * r_blk) % 16) --kb;
        if ((kb * r_blk) % 16) kb = 2;  // r' odd multiple of 8: pair two k blocks
        p.kb_per_tile = kb;
        p.BN = static_cast<int>(kb * r_blk);
        p.N = static_cast<int>(r_blk * b2);
        p.n_tok = static_cast<int>(n_tok);
        p.tiles_m = static_cast<int>(cdiv(n_tok, blr::BM));
        p.tiles_n = static_cast<int>(cdiv(b2, kb));
        p.groups = static_cast<int>(b1);
        p.total_tiles = p.tiles_m * p.groups * p.tiles_n;
        p.k_blocks = p.kb_half = static_cast<int>(cdiv(pdim, blr::BK));
        p.n_sub = 1;
        set_b_staging(p, false);
        p.out = static_cast<__nv_bfloat16*>(workspace);
        p.r_blk = static_cast<int>(r_blk);
        p.b1 = static_cast<int>(b1);
        p.b2 = static_cast<int>(b2);
        p.out_ld = K2 * comp;
        p.out_lo_off = comp == 2 ? K2 : 0;
        if (p.BN > 256 || !finish_plan(p)) return BLR_ERR_UNSUPPORTED;
        CUtensorMap ta, tb;
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
        const uint32_t box[4] = {blr::BK, static_cast<uint32_t>(r_blk), static_cast<uint32_t>(kb), 1};
        if (!encode(&tb, V, 4, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
        s = launch<blr::KIND_MONARCH_PROJ>(ta, tb, p, d, dev, st);
        if (s != BLR_OK) return s;
    }
    // ---- phase 2: Y[t, k q + c] = sum_kk Z'[k][t][kk] U[k][c][kk]  (U is [N][K]: K-major B)
    return gemm_phase(d, dev, st, workspace, n_tok, K2, b2, qdim, U, false, Y, d_out, comp, 1);
}

blr_status blr_blast_matmul(const void* X, int64_t n_tok, int64_t d_in, int64_t d_out, int64_t b1, int64_t b2,
                            int64_t r, const void* V, const void* S, const void* U, void* Y, void* workspace,
                            size_t ws_bytes, blr_stream_t stream) {
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
    const int comp = comp_factor(r);

    // ---- phase 1: Z''[k][t][rho] = sum_l S[l,k,rho] (X_l V_l)[t, rho]  (S1 on tcgen05, S2 fused)
    {
        KParams p = {};
        int R = 256;
        while (R > 16 && b1 * R > blr::TMEM_COLS) R >>= 1;
        R = static_cast<int>(std::min<int64_t>(R, rup(r, 16)));
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
        p.out = static_cast<__nv_bfloat16*>(workspace);
        p.out_ld = r * comp;
        p.out_lo_off = comp == 2 ? r : 0;
        p.b1 = static_cast<int>(b1);
        p.b2 = static_cast<int>(b2);
        p.r = static_cast<int>(r);
        p.S = static_cast<const __nv_bfloat16*>(S);
        if (!finish_plan(p)) return BLR_ERR_UNSUPPORTED;
        CUtensorMap ta, tb;
        if (!encode_x_blocked(&ta, X, n_tok, b1, pdim)) return BLR_ERR_CUDA;
        const uint64_t dims[3] = {static_cast<uint64_t>(r), static_cast<uint64_t>(pdim), static_cast<uint64_t>(b1)};
        const uint64_t str[2] = {static_cast<uint64_t>(r) * 2, static_cast<uint64_t>(r * pdim) * 2};
        const uint32_t box[3] = {64, blr::BK, 1};
        if (!encode(&tb, V, 3, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B)) return BLR_ERR_CUDA;
        s = launch<blr::KIND_BLAST_PROJ>(ta, tb, p, d, dev, st);
        if (s != BLR_OK) return s;
    }
    // ---- phase 2: Y_k = Z''_k U_k  (U is [b2][r][q]: MN-major B)
    return gemm_phase(d, dev, st, workspace, n_tok, r, b2, qdim, U, true, Y, d_out, comp, 1);
}

}  // extern "C"
