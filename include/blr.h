/*
 * blr.h -- C ABI of the B200-native block-low-rank (BLR) prefill library (arXiv 2512.20861).
 *
 * The library computes the multi-token forward product of one linear layer whose weight is
 * block-low-rank, Y = X W with W in R^{i x o} (§2.1), for three formats:
 *   - low-rank  W = V U
 *   - Monarch   W_{l,k} = V_{l,k} U_{l,k}
 *   - BLAST     W_{l,k} = V_l S_{l,k} U_k, S_{l,k} diag.
 * with X [n_tok, d_in] and Y [n_tok, d_out], blocks l in [b1] along the input, k in [b2] along
 * the output, p = d_in / b1, q = d_out / b2.
 *
 * Conventions shared by every entry point
 * ---------------------------------------
 *  - Every tensor argument is a CUDA DEVICE pointer to a dense, row-major, contiguous array of
 *    bf16 values (the 16-bit pattern of __nv_bfloat16), base address 16-byte aligned.
 *    Arithmetic: bf16 operands, fp32 accumulation, Y rounded RNE to bf16.  Intermediates
 *    (readings R11-R13):
 *      low rank, Monarch   Z (Z') rounded once to bf16 RNE; when the second-stage contraction
 *                          is shorter than 128 it is kept as a compensated bf16 pair hi|lo (R12)
 *      BLAST, b1*r <= 512  Z'' = sum_l S (.) Z_l formed in fp32 on chip, rounded once to bf16
 *      BLAST, b1*r >  512  Z_l = X_l V_l stored as IEEE fp16 (RNE, SATURATING: a value beyond
 *                          +-65504 is clamped, so results are within tolerance only while every
 *                          |(X_l V_l)[t, rho]| <= 65504; NaN stays NaN), then Z'' rounded to bf16
 *  - Row independence: Y[t, :] depends only on X[t, :] and the factors, bit for bit, whatever
 *    the other rows hold (NaN and Inf included).
 *  - Y must not alias X, a factor or the workspace.
 *  - Calls are asynchronous on `stream` (0 = legacy default stream) and stream-ordered: every
 *    kernel of a call starts reading X or a factor only after all work enqueued on `stream`
 *    before the call has completed.  The library never synchronizes, never allocates or frees
 *    caller memory and keeps no pointer after return.  The caller owns all memory;
 *    `workspace` must stay valid until the work on `stream` ends.
 *  - `workspace` holds the intermediates between the library's kernels; query its size with the
 *    matching *_workspace_size() function (its layout is private to the library).  ws_bytes
 *    smaller than that returns BLR_ERR_WORKSPACE.
 *  - Validation, planning and tensor-map encoding of every phase happen on the host before the
 *    first launch; on any of the errors below except a launch failure nothing is enqueued.
 *      BLR_ERR_NULL        a required pointer is NULL (with n_tok > 0)
 *      BLR_ERR_SHAPE       a non-positive dimension, n_tok < 0, b1 !| d_in, b2 !| d_out,
 *                          or (Monarch) r_blk inconsistent with the factor shapes
 *      BLR_ERR_ALIGN       a row pitch that is not a multiple of 16 bytes, i.e. d_in, d_out,
 *                          r, r', p or q not a multiple of 8, or a pointer not 16-B aligned
 *      BLR_ERR_UNSUPPORTED a shape outside the kernel envelope (b1 or b2 > 16, r' > 256,
 *                          n_tok >= 2^31) -- there is NO CPU fallback
 *      BLR_ERR_WORKSPACE   ws_bytes too small
 *      BLR_ERR_ARCH        the current device is not a compute-capability 10.0 (sm_100a) GPU
 *      BLR_ERR_CUDA        a CUDA runtime/driver error while encoding tensor maps (nothing
 *                          enqueued) or launching a kernel (earlier kernels of the same call
 *                          may already be enqueued; the stream then holds partial work)
 *  - n_tok == 0 is a successful no-op.
 *  - The library holds one process-wide, thread-safe cache (device properties and the
 *    tensor-map encoder); blr_clear_cache() drops it.
 */
#ifndef BLR_H_
#define BLR_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    BLR_OK = 0,
    BLR_ERR_NULL = 1,
    BLR_ERR_SHAPE = 2,
    BLR_ERR_ALIGN = 3,
    BLR_ERR_UNSUPPORTED = 4,
    BLR_ERR_WORKSPACE = 5,
    BLR_ERR_ARCH = 6,
    BLR_ERR_CUDA = 7
} blr_status;

/* Order of the composite (r' b2) middle dimension of the Monarch V tensor. */
typedef enum {
    BLR_MON_V_B2_FASTEST = 0,     /* original layout, "contiguous along b2 then r'":  m = rho*b2 + k */
    BLR_MON_V_RPRIME_FASTEST = 1  /* after re-layout (1), r' first:                  m = k*r' + rho */
} blr_monarch_vlayout;

/* Order of Monarch output columns (PAPER.md L45 footnote, L219-220). */
typedef enum {
    BLR_OUT_CANONICAL = 0,  /* Y[t, k*q + c]  (PAPER.md L53 Y_k blocks side by side)          */
    BLR_OUT_TRANSPOSED = 1  /* Y[t, c*b2 + k]: the order the paper's (3) leaves in place (PAPER.md
                               L219-220) -- the next static weight's rows are pre-permuted instead
                               (blr_transposed_row_perm) */
} blr_out_order;

typedef void* blr_stream_t; /* a cudaStream_t */

/*
 * Low-rank layer, Y = (X V) U.
 *   X [n_tok, d_in], V [d_in, r], U [r, d_out], Y [n_tok, d_out].
 *   Workspace: the intermediate Z [n_tok, r] (bf16; hi|lo pair when r < 128).
 */
blr_status blr_lowrank_matmul(const void* X, int64_t n_tok, int64_t d_in, int64_t d_out, int64_t r,
                              const void* V, const void* U, void* Y, void* workspace,
                              size_t ws_bytes, blr_stream_t stream);
size_t blr_lowrank_workspace_size(int64_t n_tok, int64_t d_in, int64_t d_out, int64_t r);

/*
 * Monarch layer, Y_k = sum_l X_l V_{l,k} U_{l,k}, factors in the paper's
 * storage:
 *   V [b1, r_blk*b2, p]   middle dimension ordered by v_layout (see blr_monarch_vlayout),
 *                         V_{l,k}[a, rho] = V[l, m(rho,k), a]
 *   U [b2, q, b1*r_blk]   inner dimension "contiguous along r' then b1",
 *                         U_{l,k}[rho, c] = U[k, c, l*r_blk + rho]
 *   Y [n_tok, d_out]      column k*q + c (BLR_OUT_CANONICAL) or c*b2 + k (BLR_OUT_TRANSPOSED)
 *                         holds output block k, column c.  The canonical order costs nothing here
 *                         (it is the store coordinate); the transposed order is written with
 *                         strided 2-byte stores (no TMA box has a 2-byte innermost extent).
 *   The r'<->b2 and b2<->b1 permutations are folded into the kernel's TMA
 *   addressing; V is read in place in either layout (no re-layout pass).
 *   Workspace: the intermediate Z' [b2][n_tok][b1*r_blk] (bf16; hi|lo pair when b1*r' < 128).
 */
blr_status blr_monarch_matmul(const void* X, int64_t n_tok, int64_t d_in, int64_t d_out, int64_t b1,
                              int64_t b2, int64_t r_blk, const void* V, const void* U,
                              int v_layout, int out_order, void* Y, void* workspace,
                              size_t ws_bytes, blr_stream_t stream);
size_t blr_monarch_workspace_size(int64_t n_tok, int64_t d_in, int64_t d_out, int64_t b1, int64_t b2,
                                  int64_t r_blk);

/*
 * BLAST layer, Y_k = ( sum_l (X_l V_l) S_{l,k} ) U_k, factors in the paper's
 * storage:
 *   V [b1, p, r], S [b1, b2, r] (the diagonals of S_{l,k}), U [b2, r, q], Y [n_tok, d_out].
 *   (north_star's s_ij is S[j, i, :]: index order (input block, output block); R5.)
 *   Workspace: the S-weighted block sums Z'' (bf16, b2 * n_tok * r values) and, when b1*r > 512,
 *   the fp16 first-stage outputs Z_l (b1 * n_tok * r values), token count padded to 128, then
 *   (b1*r > 512) 4-byte ready counters of the opt-in pipelined one-launch layer (1 + 2 per
 *   128-token tile of the padded 256-row tiles, rounded up to 256 B; the library zeroes them on
 *   `stream` itself before that launch).  The caller owns the memory; the library keeps nothing.
 */
blr_status blr_blast_matmul(const void* X, int64_t n_tok, int64_t d_in, int64_t d_out, int64_t b1,
                            int64_t b2, int64_t r, const void* V, const void* S, const void* U,
                            void* Y, void* workspace, size_t ws_bytes, blr_stream_t stream);
size_t blr_blast_workspace_size(int64_t n_tok, int64_t d_in, int64_t d_out, int64_t b1, int64_t b2,
                                int64_t r);

/*
 * BLAST layer with an FP8 first-stage intermediate (the paper's proposed
 * "intermediate activation quantization").  Same arguments, workspace and errors
 * as blr_blast_matmul.  On the split path (b1*r > 512 and r >= 128) Z_l = X_l V_l is stored as
 * OCP e4m3 (RNE, saturating at +-448, NaN stays NaN) instead of fp16 -- half the intermediate
 * bytes of the first round trip; it is widened exactly to fp16 for the tensor-core S2, and Z''
 * (bf16) and Y are as in blr_blast_matmul.  Every other path is identical to blr_blast_matmul.
 * ACCURACY CONTRACT: an e4m3 rounding (unit roundoff 2^-4) of every Z element
 * gives a relative error of ~0.027 rms (<= 0.036 for uniformly spread relative errors) -- outside
 * north_star's bound.  This entry point guarantees, on unit-variance inputs with |X_l V_l| <= 448,
 * relative Frobenius error <= 0.04 and per element |err| <= 0.2 (1 + |ref|).
 */
blr_status blr_blast_matmul_fp8z(const void* X, int64_t n_tok, int64_t d_in, int64_t d_out, int64_t b1,
                                 int64_t b2, int64_t r, const void* V, const void* S, const void* U,
                                 void* Y, void* workspace, size_t ws_bytes, blr_stream_t stream);

/*
 * BLAST factors in a statically re-laid-out, K-major storage (the paper's optimization (1) applied
 * to BLAST: a one-time re-layout of static weights so every operand is read contiguously along the
 * contraction):
 *   Vt [b1, r, p]  with Vt[l][rho][a] = V[l][a][rho]     (V of blr_blast_matmul, per block transposed)
 *   Ut [b2, q, r]  with Ut[k][c][rho] = U[k][rho][c]
 * S, X, Y, workspace and errors as blr_blast_matmul; the result is the same function of the same
 * factors (bitwise equal to blr_blast_matmul on this path).  Supported on the split tensor-core path
 * (b1*r > 512, r >= 128, n_tok above the small-n range); any other case returns
 * BLR_ERR_UNSUPPORTED before launching anything (use blr_blast_matmul with the paper layout).
 * Why: a K-major weight tile is one TMA box per K block whatever its width (an MN-major one needs a
 * box per 64 columns), and the per-SM TMA op rate bounds these GEMMs.
 */
blr_status blr_blast_matmul_kmajor(const void* X, int64_t n_tok, int64_t d_in, int64_t d_out, int64_t b1,
                                   int64_t b2, int64_t r, const void* Vt, const void* S, const void* Ut,
                                   void* Y, void* workspace, size_t ws_bytes, blr_stream_t stream);

/*
 * Row permutation for chaining a BLR_OUT_TRANSPOSED Monarch layer into the next layer without a
 * permutation pass (optimization (3)): fills the HOST array perm[b2*q] with
 * perm[c*b2 + k] = k*q + c.  If W is the next layer's weight (rows indexed by the canonical input
 * column), W'[j] = W[perm[j]] satisfies  Y_transposed W' = Y_canonical W.  A weight whose rows are
 * not block-structured (low rank V, dense, BLAST/Monarch with b1 = 1) keeps its format.  Pure index
 * arithmetic on the host (no device access).  BLR_ERR_SHAPE if b2 or q <= 0, BLR_ERR_NULL if perm
 * is NULL.
 */
blr_status blr_transposed_row_perm(int64_t b2, int64_t q, int64_t* perm);

/* Human-readable name of a status code (static storage, never NULL). */
const char* blr_status_string(blr_status s);

/* Library version "major.minor.patch" (static storage). */
const char* blr_version(void);

/* Number of CUDA kernel launches the most recent successful call on this thread enqueued. */
int blr_last_launch_count(void);

/*
 * Per-launch timing hook (measurement only).  While armed on the calling thread, every kernel
 * launch the library enqueues records events[2j] (cudaEvent_t) on the launch stream right before
 * launch j and events[2j+1] right after it, for j < capacity/2; no other effect.  Arm with a
 * caller-owned array of `capacity` created events; blr_profile_end() disarms and returns the
 * number of launches recorded.
 */
void blr_profile_begin(void** events, int capacity);
int blr_profile_end(void);

/* Drop the process-wide caches (device properties, tensor-map encoder entry point). */
void blr_clear_cache(void);

#ifdef __cplusplus
}
#endif
#endif /* BLR_H_ */
