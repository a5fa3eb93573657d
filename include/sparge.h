/*
 * sparge.h -- C ABI of the B200 (sm_100a) SpargeAttn hot path.
 *
 * SpargeAttn (arXiv 2502.18137) computes a two-stage block-sparse, INT8
 * quantised attention forward pass.  Citations are PAPER.md lines (P:Lnnn)
 * with the section / equation / Algorithm-1 line they sit in; readings of
 * silent passages are the R# items of DESIGN.md §3.
 *
 * Conventions for every call:
 *   - Pointers are DEVICE pointers unless the argument says "host".
 *   - The caller owns every buffer.  The library never allocates or frees
 *     device memory, never synchronises the stream (except
 *     sparge_attn_status, which says so) and never prints.
 *   - All work is enqueued asynchronously on `stream` (a cudaStream_t passed
 *     as an opaque pointer; NULL = the legacy default stream).  Stream order
 *     holds as for plain launches: the prediction, V-stage, launch-order and
 *     attention kernels are launched with programmatic dependent launch
 *     (CUDA PDL) and each waits (griddepcontrol.wait) for the work before it
 *     in the stream to complete before it reads or writes global memory;
 *     only their launch and on-chip set-up overlap the predecessor's tail.
 *     A caller kernel that itself uses PDL must not trigger its dependents
 *     before its outputs are written (the standard PDL contract).
 *   - Tensors of tokens are [B, H, N, d] with d contiguous; `sparge_strides`
 *     gives the element strides of the b, h and n axes.  Row starts must be
 *     16-byte aligned (d in {64, 128}, so stride_n*2 % 16 == 0).
 *   - Blocks: T_m = ceil(N / bq) query blocks, T_n = ceil(N / bk) key blocks
 *     (Definition 1; reading R6).  bq = 128, bk = 64, cw = 4
 *     are the only supported values (App. A.1).
 *   - GQA: query head h reads key/value head h / (Hq / Hkv)  (reading R18).
 *   - Return codes: SPARGE_OK, or SPARGE_EINVAL for argument validation
 *     failures (nothing is enqueued), SPARGE_ECUDA for a launch error
 *     (cudaGetLastError() holds the cause), SPARGE_ENOTIMPL for an option
 *     that is declared but not built.  Errors are returned, never thrown.
 */
#ifndef SPARGE_H_
#define SPARGE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum sparge_status {
  SPARGE_OK = 0,
  SPARGE_EINVAL = 2,     /* shape / stride / hyper-parameter validation      */
  SPARGE_EINTERNAL = 3,  /* a valid query row ended with l = 0 (R8)  */
  SPARGE_ECUDA = 4,      /* CUDA launch or driver error                      */
  SPARGE_ENOTIMPL = 5    /* declared option not implemented in this build    */
};

enum sparge_dtype { SPARGE_BF16 = 0, SPARGE_FP16 = 1 };
/* largest T_n = ceil(N / bk) sparge_predict_mask accepts (N <= 2^20) */
enum { SPARGE_MAX_TN = 16384 };
/* Operand type of the P~V product (Alg. 1 line 16):
 *   SPARGE_PV_SAME_AS_INPUT  P~ rounded to in_dtype, V in in_dtype (R12);
 *   SPARGE_PV_FP8_E4M3       scope row f4 (SageAttention2-style, footnote
 *                            P:L44; R27): V per-channel FP8 E4M3 with
 *                            s_c = amax_c / 448 over all N tokens of its kv-head,
 *                            P~ scaled by 2^7 and rounded to E4M3, fp32
 *                            accumulation, O = acc * s_c / l.  INT8 QK only. */
enum sparge_pv_dtype { SPARGE_PV_SAME_AS_INPUT = 0, SPARGE_PV_FP8_E4M3 = 1 };
/* Operand type of the QK^T product (stage 2, Alg. 1 line 12):
 *   SPARGE_QK_INT8   SageAttention per-block INT8 -- the
 *                    paper's default kernel ("SpargeAttn+SageAttn");
 *   SPARGE_QK_INPUT  no quantisation: QK^T of the in_dtype values with fp32
 *                    accumulation -- the paper's "SpargeAttn+FA2" kernel of
 *                    Fig. 7; scope row f1. */
enum sparge_qk_dtype { SPARGE_QK_INT8 = 0, SPARGE_QK_INPUT = 1 };
enum sparge_sim_mode {
  SPARGE_SIM_COSINE = 0,   /* R1-A: mean of the row-normalised Gram matrix  */
  SPARGE_SIM_LITERAL = 1   /* R1-B: mean(X X^T / |max(X X^T)|) on raw rows  */
};

typedef struct { int64_t b, h, n; } sparge_strides;

typedef struct {
  int B, Hq, Hkv, N, d;   /* d in {64, 128}; Hq % Hkv == 0; N >= 1          */
  int bq, bk, cw;         /* must be 128, 64, 4                            */
  int causal;             /* 0/1; block-causal handling per reading R8      */
  int in_dtype;           /* enum sparge_dtype of Q, K, V, O                 */
  int pv_dtype;           /* enum sparge_pv_dtype                            */
  int sim_mode;           /* enum sparge_sim_mode                           */
  int smooth_k;           /* 0/1: K smoothing (row f4, R28; INT8 QK only):   *
                           * K goes through sparge_smooth_k_mean +           *
                           * sparge_quantize_smooth_k                        */
  int qk_dtype;           /* enum sparge_qk_dtype                           */
} sparge_shape;

/* Human-readable name of a status code (static string, never NULL). */
const char* sparge_strerror(int status);

/*
 * hilbert_permute -- §3.7 "HilbertCurve Permutation" and
 * App. A.1.  HOST call, no CUDA.
 *
 * Builds the generalised 3-D Hilbert order (gilbert3d, reading R19) of a
 * T x H x W grid of visual tokens that follow `text_prefix` text tokens.
 * Source token layout: [text_prefix text tokens][(t, h, w) row-major].
 *   perm_host[r] = source index of position r of the permuted sequence
 *   inv_host[s]  = position of source token s         (inv[perm[r]] = r)
 * Both arrays have L = text_prefix + T*H*W int32 entries (host memory,
 * caller-allocated).  Text tokens map to themselves.
 * Errors: SPARGE_EINVAL if any extent < 1, text_prefix < 0, L > 2^31-1,
 * or a pointer is NULL.
 */
int hilbert_permute(int T, int H, int W, int text_prefix,
                    int32_t* perm_host, int32_t* inv_host);

/*
 * sparge_quantize -- Alg. 1 line 3 ("per-block quantization in
 * SageAttention"), line 4 (block mean) and line 5 (CosSim),
 * fused in one HBM pass.  Runs once for Q (is_key = 0, blocks of bq rows,
 * H = Hq) and once for K (is_key = 1, blocks of bk rows, H = Hkv).
 *
 *   x      [B, H, N, d] in_dtype, strided by x_str (read-only)
 *   perm   nullable int32 [N]: row r of the (permuted) sequence is x row
 *          perm[r] (the Hilbert gather of §3.7).  NULL = identity.
 *   xq     [B, H, N, d] contiguous, permuted order.  qk_dtype INT8: int8,
 *          per block i xq = clamp(rne(fl32(x * fl32(127/amax_i))), -127, 127)
 *          (R11).  qk_dtype INPUT: in_dtype, the rows of x copied bit for bit
 *          (the gathered operand of the unquantised f1 kernel).
 *   delta  fp32 [B, H, T]: fl32(amax_i / 127); 1 for an all-zero block; 1
 *          everywhere for qk_dtype INPUT
 *   pooled fp64 [B, H, T, d]: mean over the block's valid rows
 *   sim    fp64 [B, H, T]: CosSim of the block per sim_mode     (R1)
 * T = T_m (is_key = 0) or T_n (is_key = 1).
 * Errors: SPARGE_EINVAL (bad shape, NULL pointer, misaligned stride, K of a
 * smooth_k shape -- that one goes through sparge_quantize_smooth_k),
 * SPARGE_ECUDA.
 */
int sparge_quantize(const sparge_shape* shape, const void* x, sparge_strides x_str,
                    int is_key, const int32_t* perm,
                    void* xq, float* delta, double* pooled, double* sim,
                    void* stream);

/*
 * K smoothing -- scope row f4, the SageAttention "smooth K" step that the
 * paper's SageAttention2-based kernel inherits (footnote P:L44; reading R28).
 * K' = K - mu with mu the per-channel token mean of K: S' = S - q.mu is a
 * per-query-row constant, so softmax, the lambda gate (m_local - m_new) and O
 * are unchanged in exact arithmetic, and the INT8 blocks of K' lose the
 * channel offsets.  Stage 1 (pooled, CosSim, the mask) keeps the raw K (R14).
 *
 * sparge_smooth_k_workspace: bytes of fp64 chunk sums sparge_smooth_k_mean
 * needs (B*Hkv*ceil(N/128)*d doubles); 0 on invalid shape.
 * sparge_smooth_k_mean: mean fp32 [B, Hkv, d] (caller-allocated) =
 *   fl32( (sum over chunks of 128 tokens, in chunk order, of the sequential
 *   fp64 sum of the chunk's tokens in index order) / N ), tokens in their
 *   ORIGINAL order (before any Hilbert permutation).  k as in sparge_quantize
 *   (is_key = 1).  workspace: >= sparge_smooth_k_workspace, 8-B aligned.
 * sparge_quantize_smooth_k: sparge_quantize of K (is_key = 1) whose INT8
 *   path quantises fl32(k - mean[c]) per element (amax and delta of the
 *   smoothed block); pooled and sim are those of the raw k.
 * Errors: SPARGE_EINVAL, SPARGE_ENOTIMPL (qk_dtype INPUT: nothing to
 * smooth), SPARGE_ECUDA.  No synchronisation.
 */
size_t sparge_smooth_k_workspace(const sparge_shape* shape);
int sparge_smooth_k_mean(const sparge_shape* shape, const void* k, sparge_strides k_str,
                         void* workspace, size_t ws_bytes, float* mean, void* stream);
int sparge_quantize_smooth_k(const sparge_shape* shape, const void* k, sparge_strides k_str,
                             const int32_t* perm, const float* mean, void* kq, float* delta,
                             double* pooled, double* sim, void* stream);

/*
 * sparge_predict_mask -- stage 1 of Algorithm 1, lines 5-6,
 * §3.2 TopCdf and Eq. (5) fix-block forcing.
 * Inputs are the sparge_quantize statistics of Q (per q-head) and K (per
 * kv-head), so Q and K are read from HBM once.  fp64 (R15).
 *
 * For each (b, hq, i):
 *   S^[j] = q_i . k_j / sqrt(d)                                    (R2)
 *   S^[j] = -inf if k_sim[j] < theta, or if tile (i,j) is causally dead
 *   P^ = softmax(S^);  keep rank k of (P^ desc, j asc) iff
 *        cumsum_k <= tau * cumsum_last, and always rank 0          (R4)
 *   M[i,:] = 1 if q_sim[i] < theta; M[:,j] = 1 if k_sim[j] < theta;
 *   all -inf row -> all ones (R7); causal: M &= live, M[i, i*bq/bk] = 1 (R8)
 * Outputs (device):
 *   mask  nullable uint8 [B, Hq, T_m, T_n]  (M_g of Definition 1)
 *   lut   int32 [B, Hq, T_m, T_n]: kept j of row i in ascending order
 *   cnt   int32 [B, Hq, T_m]: number of kept j of row i (>= 1)
 *   workspace/ws_bytes  >= sparge_predict_workspace(shape), 256-byte aligned
 *         (scratch for S^; contents undefined on return)
 * tau in (0, 1], theta in [-1, 1] (float32, compared in fp64).
 * Errors: SPARGE_EINVAL (range / NULL / T_n > SPARGE_MAX_TN, i.e.
 * N > 1048576: one compressed-map row is held per warp in shared memory),
 * SPARGE_ECUDA.
 */
int sparge_predict_mask(const sparge_shape* shape,
                        const double* q_pooled, const double* q_sim,
                        const double* k_pooled, const double* k_sim,
                        float tau, float theta,
                        uint8_t* mask, int32_t* lut, int32_t* cnt,
                        void* workspace, size_t ws_bytes, void* stream);

/* Bytes of device workspace sparge_predict_mask needs (the fp64 compressed
 * map S^, B*Hq*T_m*T_n doubles).  0 on invalid shape. */
size_t sparge_predict_workspace(const sparge_shape* shape);

/* Bytes of device workspace sparge_attn_fwd needs for `shape`: the status
 * word (256 B), the V^T staging (16-bit tile-major [B, Hkv, N_pad/64, d, 64],
 * or E4M3 row-major [B, Hkv, d, N_pad] for pv_dtype FP8; N_pad = N rounded
 * up to 64; rounded to 256 B), for FP8 the per-channel amax and dequant scales, and the launch
 * order of the B*Hq*T_m attention work items (int32, longest first; rounded
 * to 256 B).  0 on invalid shape. */
size_t sparge_attn_workspace(const sparge_shape* shape);

/*
 * sparge_attn_fwd -- stage 2 of Algorithm 1, lines 7-21:
 * the sparse FlashAttention loop over the kept blocks with SageAttention
 * dequantisation (line 12) and the per-warp lambda gate (lines
 * 14-17; §3.4).
 *
 *   qq, dq   [B, Hq, N, d] + fp32 [B, Hq, T_m]  (sparge_quantize of Q)
 *   kq, dk   [B, Hkv, N, d] + fp32 [B, Hkv, T_n] (sparge_quantize of K)
 *            qq/kq are int8 (qk_dtype INT8: S = (Q^K^^T) dq dk / sqrt(d),
 *            integer-exact product) or in_dtype (qk_dtype INPUT: S =
 *            QK^T/sqrt(d) accumulated in fp32 on the tensor cores)
 *   v        [B, Hkv, N, d] in_dtype, strided by v_str, ORIGINAL token order
 *   lut, cnt from sparge_predict_mask
 *   lambda   natural-log units of S = QK^T/sqrt(d) (R3); -INFINITY disables
 *            the gate; must be < 0.  A warp of bq/cw rows computes its
 *            P~V slice iff max_rows(m_local - m_new) > lambda (R5).
 *   perm     nullable int32 [N]: the same permutation given to
 *            sparge_quantize; V rows are gathered through it and O rows are
 *            scattered back to original order.  Must be NULL when
 *            shape->causal is set (causality is defined on token positions,
 *            R8): SPARGE_EINVAL otherwise.
 *   o        [B, Hq, N, d] in_dtype, strided by o_str (written)
 *   counters nullable uint64 [B, Hq, 3], ACCUMULATED (caller zeroes):
 *            [0] executed QK tiles, [1] executed P~V warp slices,
 *            [2] issued P~V MMAs  (sparsity per R16)
 *   workspace/ws_bytes  >= sparge_attn_workspace(shape), 256-byte aligned;
 *            zero-initialised once by the caller (its first word is the
 *            status word, cleared again by sparge_attn_status)
 * Errors: SPARGE_EINVAL, SPARGE_ENOTIMPL (pv_dtype FP8 or smooth_k with
 * qk_dtype INPUT), SPARGE_ECUDA.  A
 * row finishing with l = 0 is recorded in the workspace status word and
 * reported by sparge_attn_status.
 */
int sparge_attn_fwd(const sparge_shape* shape,
                    const void* qq, const float* dq,
                    const void* kq, const float* dk,
                    const void* v, sparge_strides v_str,
                    const int32_t* lut, const int32_t* cnt,
                    float lambda, const int32_t* perm,
                    void* o, sparge_strides o_str,
                    uint64_t* counters,
                    void* workspace, size_t ws_bytes, void* stream);

/* sparge_attn_fwd split into its two launches, for per-kernel timing:
 *   flags = 0                          same as sparge_attn_fwd (the launch
 *                                      order kernels, then the V staging,
 *                                      which overlaps them, then attention)
 *   flags = SPARGE_ATTN_VPREP_ONLY     only stage V^T (+ Hilbert gather) into
 *                                      the workspace
 *   flags = SPARGE_ATTN_SKIP_VPREP     only the attention kernel; V^T must
 *                                      already be in the workspace from a
 *                                      VPREP_ONLY call with the same v/perm
 * Same arguments, validation and errors as sparge_attn_fwd. */
enum { SPARGE_ATTN_VPREP_ONLY = 1, SPARGE_ATTN_SKIP_VPREP = 2 };
int sparge_attn_fwd_ex(const sparge_shape* shape,
                       const void* qq, const float* dq,
                       const void* kq, const float* dk,
                       const void* v, sparge_strides v_str,
                       const int32_t* lut, const int32_t* cnt,
                       float lambda, const int32_t* perm,
                       void* o, sparge_strides o_str,
                       uint64_t* counters,
                       void* workspace, size_t ws_bytes, void* stream,
                       unsigned flags);

/*
 * sparge_attn_fwd_mpv -- sparge_attn_fwd plus a dump of every lambda-gate
 * decision (debug mode of SURVEY §8(c); Algorithm 1 lines 14-17):
 *   mpv  uint8 [B, Hq, T_m, T_n, c_w] device, caller-zeroed.  For every kept
 *        block (i, j) and warp group w (rows 32w..32w+31 of query block i):
 *        2 = the P~V slice was computed (max over the group's rows of
 *        m_local - m_new > lambda), 1 = skipped by the gate (also a group
 *        without valid rows, R6).  Entries of blocks that M_g drops stay 0.
 * Same arguments, validation and errors as sparge_attn_fwd (mpv NULL ->
 * SPARGE_EINVAL).  Writes one byte per (tile, warp): a test/debug entry
 * point, not the timed path.
 */
int sparge_attn_fwd_mpv(const sparge_shape* shape,
                        const void* qq, const float* dq,
                        const void* kq, const float* dk,
                        const void* v, sparge_strides v_str,
                        const int32_t* lut, const int32_t* cnt,
                        float lambda, const int32_t* perm,
                        void* o, sparge_strides o_str,
                        uint64_t* counters,
                        void* workspace, size_t ws_bytes, void* stream,
                        uint8_t* mpv);

/*
 * sparge_l1_sums -- the accuracy metric of §3.6, relative L1
 * = sum|O - O'| / sum|O'| (reference in the denominator, R17),
 * used by the hyper-parameter tuner (scope row f2) and the permutation study
 * (f3) to score an output against the dense reference on the device.
 *   o, o_ref  n contiguous 16-bit elements of `dtype` (enum sparge_dtype)
 *   out       device fp64 [SPARGE_L1_OUT_DOUBLES]: out[0] = sum|o - o_ref|,
 *             out[1] = sum|o_ref| (fp64 accumulation, deterministic); the
 *             rest is scratch
 * Errors: SPARGE_EINVAL (NULL, n < 1, bad dtype, misaligned), SPARGE_ECUDA.
 */
#define SPARGE_L1_OUT_DOUBLES 1186
int sparge_l1_sums(const void* o, const void* o_ref, int dtype, int64_t n, double* out,
                   void* stream);

/* SYNCHRONISES `stream`, reads and clears the workspace status word:
 * SPARGE_OK, or SPARGE_EINTERNAL if some valid row ended with l = 0. */
int sparge_attn_status(void* workspace, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPARGE_H_ */
