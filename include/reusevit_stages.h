/*
 * reusevit_stages.h — per-step entry points of libreusevit.so, one per row of the hot
 * path, exposed so the parity tests can drive each kernel on its
 * own with inputs taken from the oracle (teacher forcing).  rv_embed runs the same
 * kernels; nothing here is a separate implementation.
 *
 * Conventions: every pointer is a DEVICE pointer; work is enqueued on `stream` and is
 * complete in stream order (the caller synchronises).  Row indices are GLOBAL rows
 * slot*T + token into per-frame [slots][T][...] arrays.  A "wave descriptor" is int32
 * [n_w][4] = {slot, past_slot, future_slot, type} per frame of a level-wave, frames in
 * ascending computation-order position.  Errors as in reusevit.h.
 */
#ifndef REUSEVIT_STAGES_H
#define REUSEVIT_STAGES_H

#include "reusevit.h"

#ifdef __cplusplus
extern "C" {
#endif

/* a2+a3 — Eq. 1-4: for every patch token i of every non-I frame of the
 * wave, s_i = max cosine against the available references' rows of X [slots][T][D] fp32,
 * provider = argmax (ties -> past), v = [s, t, onehot(type), c], d = MLP_decision(v) with
 * the layer-`layer` gate weights loaded in ctx, M = d > 0 (or force[slot][layer][i] when
 * force != NULL).  t [slots][N] and codec [slots][N] fp32.  Writes
 *   masks [slots][L][N] u8 and scores [slots][L][N] fp32 (NaN for I frames) at `layer`,
 *   wmask [n_w][T] u8 (wave-local M, token 0 = 0), wprov [n_w][T] u8 (0 past, 1 future),
 *   cntR [n_w] int32 = |R| of each frame (reused patch tokens).                             */
rv_status rv_stage_score(rv_ctx* ctx, int32_t layer, const float* X, int32_t n_w,
                         const int32_t* wdesc, const float* t, const float* codec,
                         const uint8_t* force, uint8_t* masks, float* scores,
                         uint8_t* wmask, uint8_t* wprov, int32_t* cntR, void* stream);

/* a4 — Eq. 5-6 filtration as stream compaction (§5.3): from wmask,
 * wprov and cntR, writes idxC [<= n_w*T] (global rows of C, frames in wave order, tokens
 * ascending, CLS first), idxR / provrow [<= n_w*N] (global rows of R and of their
 * providers' same token), qoff [n_w+1] (exclusive prefix of |C|), counts[2] = {M_C, M_R}.
 * Bit-exact given the mask; all counts stay on the device. */
rv_status rv_stage_compact(rv_ctx* ctx, int32_t n_w, const int32_t* wdesc,
                           const uint8_t* wmask, const uint8_t* wprov, const int32_t* cntR,
                           int32_t* idxC, int32_t* idxR, int32_t* provrow, int32_t* qoff,
                           int32_t* counts, void* stream);

/* a6/a9-a12 building block — the tcgen05/TMEM tensor-core GEMM on its own:
 * out[m][n] = act(sum_k A[m][k] * B[n][k] + bias[n]) for m < M, n < N, with A bf16
 * [M][K] row-major, B bf16 [N][K] row-major (i.e. out = A * B^T), bias fp32 [N] or NULL,
 * act 0 = identity, 1 = QuickGELU; out fp32 (out_bf16 == 0) or bf16 [M][N].
 * K % 64 == 0, N % 64 == 0 (RV_ECONTRACT otherwise). */
rv_status rv_stage_gemm(rv_ctx* ctx, int32_t M, int32_t N, int32_t K, const void* A,
                        const void* B, const float* bias, int32_t act, void* out,
                        int32_t out_bf16, void* stream);

/* a9 / a11 / a12 building block — the same GEMM with the row-mapped epilogue of the embed:
 * out[out_rows[m]][n] = act(A[m] . B[n] + bias[n]) + resid[resid_rows[m]][n]  (fp32 resid,
 * NULL = none; resid_rows / out_rows NULL = identity; an out_rows entry < 0 skips row m).
 * K <= 128 with a residual selects the short-K residual-streaming variant (restoration R2,
 * Eq. 9-10).  Leading dimensions in elements.  RV_ECONTRACT on bad arguments. */
rv_status rv_stage_gemm_rows(rv_ctx* ctx, int32_t M, int32_t N, int32_t K, const void* A,
                             const void* B, const float* bias, int32_t act, const float* resid,
                             const int32_t* resid_rows, int64_t resid_ld, void* out,
                             const int32_t* out_rows, int64_t out_ld, int32_t out_bf16, void* stream);

/* a8 — attention of compacted queries over all T keys of their frame:
 * q [M_C][D] bf16 (rows qoff[w]..qoff[w+1]-1 belong to wave frame w, first row = CLS),
 * KV [slots][T][2D] bf16, per token row head-interleaved: head h's key in columns
 *    2h*dh..2h*dh+dh-1 and its value in the next dh columns (the layout the embed's QKV GEMM
 *    writes: one 2*dh segment per (token, head), 256 B at d_h = 64),
 * out [M_C][D] bf16 = softmax(q K^T / sqrt(dh)) V per head; pcls [slots][H][N] fp32 (or
 * NULL) = per-head CLS softmax row over the patch keys; its head mean is t for the next
 * layer.  q_rows = allocated rows of q (>= qoff[n_w]; the tcgen05 path
 * reads q with TMA in 64-row tiles).  kvsrc [slots][T] int32 (or NULL = identity) is the
 * reuse-cache row table of a7: key j of the frame in slot s is row kvsrc[s*T + j] of KV.
 * use_tc: 0 the mma.sync kernel (any supported shape); 1 the tcgen05/TMEM kernels (the
 * persistent one for T - 1 <= 256, else the general one); 2 the general tcgen05 kernel
 * (128-query tiles, online softmax over 128-key blocks, d_h = 64, T <= 1024).  RV_ECONTRACT
 * when the shape is outside the selected kernel's range. */
rv_status rv_stage_attention(rv_ctx* ctx, int32_t n_w, const int32_t* wdesc,
                             const int32_t* qoff, const void* q, int32_t q_rows, const void* KV,
                             const int32_t* kvsrc, void* out, float* pcls, int32_t use_tc,
                             void* stream);

#ifdef __cplusplus
}
#endif
#endif /* REUSEVIT_STAGES_H */
