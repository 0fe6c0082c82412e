/*
 * reusevit.h — C-ABI of libreusevit.so, the B200 (sm_100a) ReuseViT hot path of
 * Deja Vu (arxiv 2506.14107).
 *
 * The calls follow the paper's statement of the problem:
 *   - a ViT turns frames into embeddings                      (§2.3)
 *   - decision + restoration modules are trained offline per
 *     backbone and loaded next to the frozen ViT
 *   - frames are reordered inside the forward pass and results
 *     come back in display order; an I-frame every 20th frame
 *   - on a miss, embeddings are generated
 * Interface shapes follow SPEC.md (ViTConfig S:97-100, RVW1/RVG1 array orders S:160/S:280,
 * plan_gop S:308-316, reuse_forward S:253-256, execute_segment S:372-376).
 *
 * Conventions
 *   - All sizes are element counts.  Floating point is IEEE fp32 little-endian at the ABI;
 *     internally the path computes in bf16 (GEMM operands, K/V) with fp32 accumulation
 *     and an fp32 residual stream.
 *   - Ownership: the caller owns every buffer passed in.  Weights are copied to the device
 *     by rv_load_*; inputs must stay valid until rv_wait returns.
 *   - Errors: every call returns a negative rv_status on failure and records a message
 *     retrievable with rv_last_error(ctx).  Nothing throws across the ABI; the library
 *     never calls abort()/exit().
 *   - Threading: a context is bound to one device and has at most one embed in flight.
 *     It is thread-compatible, not thread-safe.
 *   - There is no CPU fallback: a context can only be created on a CUDA device of compute
 *     capability 10.0 (B200); anything else returns RV_ECUDA.
 */
#ifndef REUSEVIT_H
#define REUSEVIT_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  RV_OK = 0,
  RV_ECONFIG = -1,   /* invalid config (e.g. dim % heads != 0)                     */
  RV_ESHAPE = -2,    /* blob length / shape mismatch                       */
  RV_EPLAN = -3,     /* reference used before computed, cycle, bad type   */
  RV_ECACHE = -4,    /* provider missing from the reuse cache             */
  RV_ECONTRACT = -5, /* caller contract violated (null pointer, weights not loaded, ...)  */
  RV_ECUDA = -6,     /* CUDA error or no sm_100 device; message has cudaGetErrorString    */
  RV_ENOMEM = -7,    /* device allocation failed                                          */
  RV_EBUSY = -8      /* an embed is already in flight on this context                      */
} rv_status;

typedef struct rv_ctx rv_ctx;

/* Model dimensions (SPEC.md:97-100 ViTConfig; SURVEY §8 notation).
 *   N = (img/patch)^2 patch tokens, T = N + 1 with CLS, pp = 3*patch^2 pixels per patch.
 *   Requirements: dim % heads == 0, dim/heads in {16, 64}, dim % 64 == 0, ffn % 64 == 0,
 *   hidden_r % 64 == 0, 1 <= hidden_g <= 32, img % patch == 0, layers <= 64, T <= 768. */
typedef struct {
  int32_t layers, dim, heads, patch, img, ffn, hidden_r, hidden_g;
} rv_config;

/* Frame types = one-hot order of the reference-type feature r. */
enum { RV_I = 0, RV_P = 1, RV_B2 = 2, RV_B1 = 3 };

/* A frame plan (S:298-301 GopPlan).  Arrays are caller-allocated, length n, indexed by
 * DISPLAY frame index: type[f] in {RV_I..RV_B1}; past[f]/future[f] = reference display
 * index or -1 (none); order = the computation order (a permutation of 0..n-1 in which
 * every reference precedes its dependents). */
typedef struct {
  int32_t n;
  int8_t* type;
  int32_t* past;
  int32_t* future;
  int32_t* order;
} rv_plan;

/* Per-embed statistics (S:366-369 Metrics), filled by rv_wait. */
typedef struct {
  double reuse_nonI;          /* Eq. 14 mean of M over non-I frames, layers, patches   */
  double reuse_all;           /* reused token-layers / (n * L * T)                              */
  double flops_exec;          /* executed tensor FLOPs (SURVEY §8(d) F_exec formula)            */
  double flops_dense;         /* same frames with no reuse                                      */
  double bytes_alg;           /* algorithmic HBM bytes of the reuse path (DESIGN.md §6 model)  */
  uint64_t peak_cache_bytes;  /* allocated bytes of the activation cache: X ping-pong + one K/V
                                 layer, or every layer's X and K/V with RV_KEEP_ALL_CACHE         */
  uint64_t keepall_cache_bytes; /* bytes if every layer's X and K/V were kept (Fig. 12 analog) */
  float ms_total;             /* device time of the embed (CUDA events, H2D/D2H included)      */
  float ms_compute;           /* device time of the compute graph only                          */
  int32_t n_levels;           /* dependency levels (waves per layer)                            */
  int32_t n_launches;         /* kernels launched by the last embed (own kernels only)          */
  float reuse_by_layer[64];   /* per-layer Eq. 14 reuse rate over non-I frames                  */
  uint64_t device_bytes;      /* bytes of every per-embed device buffer the context allocated   */
  int32_t wave_ring;          /* wavefront schedule: ring size R of the layer buffers (X_l in
                                 slot l % R); 0 = serial level waves (see RV_SERIAL_WAVES)        */
} rv_stats;

/* rv_embed flags */
#define RV_DEVICE_PTRS 1u  /* patches/codec/emb/masks/scores are device pointers (stream order) */
#define RV_DENSE 2u        /* ignore the gates: every token recomputed (own-dense baseline)     */
#define RV_FORCE_MASKS 4u  /* masks is an INPUT [n][L][N]: forced reuse map (diagnostic, Q18)   */
#define RV_NO_GRAPH 8u     /* launch kernels directly instead of through a cached CUDA graph    */
#define RV_PROFILE 16u     /* time every kernel launch with CUDA events (see rv_profile)         */
#define RV_WAVE_FRAME 64u  /* ablation (SURVEY §8(d) ladder step 2): every frame is its own wave,
                              i.e. per-frame compaction instead of level-batched cross-frame
                              compaction (results identical, only the batching differs)         */
#define RV_CHAIN 128u      /* SPEC chain variant: the
                              decision on the FFN input x'_l gates FFN_l -> QKV_{l+1}; attention
                              and W_o dense for all tokens (general tcgen05 attention, q read
                              from the q|k|v cache through the source-row table)                */
#define RV_NO_COMPACTION 256u  /* ablation (SURVEY §8(d) ladder step 1, "masked dense"): every token
                              is recomputed (no stream compaction), then the reused tokens'
                              outputs are overwritten by the restoration; results equal the
                              compacted path bitwise (row-local kernels)                         */
#define RV_KEEP_ALL_CACHE 512u /* ablation of cached memory compaction (Fig. 12
                              analogue): keep every layer's X and K/V allocated; at the 7,200-frame
                              workload this needs ~371 GB and fails with RV_ENOMEM               */
#define RV_SERIAL_WAVES 1024u /* run the level waves strictly one after another (layer by layer).
                              Default: when every wave holds <= 512 frames, wave (l, k) starts as
                              soon as wave (l, k-1) and wave (l-1, k) are done (wavefront over
                              rings of R layer buffers, one stream per wave index);
                              results are bitwise identical, only the concurrency differs        */
#define RV_X_BF16 2048u    /* experimental: the residual stream X (every layer's input and
                              output token rows, the reuse cache's X part) is stored in bf16 instead
                              of fp32 — half the bytes of the score, LN1, residual and restoration
                              traffic; LN statistics, the decision, the GEMM accumulators and the
                              residual adds still compute in fp32 and round once on store.  D1 path
                              only (RV_ECONTRACT with RV_CHAIN)                                  */
#define RV_RESTORE_GEMMS 4096u /* diagnostic: restoration as the two GEMMs R1 (over all wave rows, hr to
                              HBM) and R2 instead of the fused k_restore kernel (results bitwise
                              equal; the fused kernel runs wherever Hr = 128 and D % 128 == 0)   */
#define RV_ATTN_SYNC 32u   /* diagnostic: attention on the mma.sync kernel (k_attn.cu) even where the
                              tcgen05/TMEM kernels (k_attn_tc.cu: d_h = 64) apply; without it the
                              mma.sync kernel runs only for d_h = 16 (the tiny config)            */

/* Per-kernel-class profile of the last RV_PROFILE embed (rv_profile). */
typedef struct {
  char name[24];       /* kernel class, e.g. "gemm_fc1", "score", "attention"               */
  int32_t launches;    /* launches of this class in the embed                               */
  double ms;           /* summed CUDA-event durations of those launches                     */
  double flops;        /* algorithmic tensor FLOPs (2*M*N*K with the actual compacted M)    */
  double bytes;        /* algorithmic HBM bytes (DESIGN.md §6 per-row byte model)            */
} rv_kernel_prof;

/* Create a context on CUDA device `device`.  Validates cfg (RV_ECONFIG) and requires a
 * compute-capability-10.x device (RV_ECUDA otherwise). */
rv_status rv_create(const rv_config* cfg, int device, rv_ctx** out);

/* Number of floats rv_load_vit / rv_load_gates expect for cfg (0 if cfg invalid). */
size_t rv_vit_blob_floats(const rv_config* cfg);
size_t rv_gate_blob_floats(const rv_config* cfg);

/* Load the frozen ViT weights: flat host fp32 array in RVW1 declaration order (
 * SURVEY §8(c)): W_pe[pp,D], cls[D], pos[T,D], lnpre_g[D], lnpre_b[D], then per layer
 * ln1_g, ln1_b, Wqkv[D,3D], bqkv[3D], Wo[D,D], bo[D], ln2_g, ln2_b, W1[D,F], b1[F],
 * W2[F,D], b2[D], then lnpost_g, lnpost_b.  Matrices are [in, out] row-major.  Copied
 * (and converted to bf16 [out, in]) to the device.  RV_ESHAPE if n_floats mismatches. */
rv_status rv_load_vit(rv_ctx* ctx, const float* blob, size_t n_floats);

/* Load the decision + restoration layers (P:345 decision MLP, P:377 restoration MLP),
 * RVG1 order, per layer: Wd1[7,Hg], bd1[Hg], Wd2[Hg], bd2[1],
 * Wr1[D,Hr], br1[Hr], Wr2[Hr,D], br2[D].  Decision-feature row order of Wd1:
 * [s, t, 1[I], 1[P], 1[B2], 1[B1], c] (Eq. 2). */
rv_status rv_load_gates(rv_ctx* ctx, const float* blob, size_t n_floats);

/* Build the frame plan for n frames: 5-frame units with
 * computation order 0,4,2,1,3, P-chain anchors every 4 frames, an I-frame at every
 * multiple of `refresh` (multiple of 4, >= 4), missing future references dropped at the
 * tail.  reorder == 0 gives the low-latency all-P chain.  `out`
 * arrays must hold n entries.  Host-only; needs no GPU. */
rv_status rv_plan_gop(int32_t n, int32_t refresh, int32_t reorder, rv_plan* out);

/* Validate a plan (RV_EPLAN on a bad type, an out-of-range reference, a reference that is
 * not computed before its dependent, or an order that is not a permutation).  Host-only. */
rv_status rv_plan_check(const rv_plan* plan);

/* Embed a frame batch ("generates them with ReuseViT"):
 *   patches [n][N][pp] fp32 — pre-patchified frames in display order (channel-major
 *                              (3,P,P) pixel vector per patch, row-major patch grid)
 *   codec   [n][N]     fp32 — codec-metadata feature c (synthetic stub)
 *   plan                    — reference schedule (rv_plan_gop or caller-built; validated)
 *   emb     [n][D]     fp32 — OUT: Z_f = LN_post(CLS) in display order
 *   masks   [n][L][N]  u8   — OUT reuse map M (Eq. 4), or IN with RV_FORCE_MASKS; may be NULL
 *   scores  [n][L][N]  fp32 — OUT decision logits d (Eq. 3; NaN where no decision ran); may be NULL
 * With RV_DEVICE_PTRS all five buffers are device pointers and results are complete in
 * `cuda_stream` order; otherwise they are host pointers (pinned for full overlap), copied
 * H2D/D2H on `cuda_stream` and complete when rv_wait returns.  `cuda_stream` may be NULL
 * (legacy default stream).  Asynchronous: call rv_wait before reading host outputs. */
rv_status rv_embed(rv_ctx* ctx, const float* patches, const float* codec, const rv_plan* plan,
                   uint32_t flags, void* cuda_stream, float* emb, uint8_t* masks, float* scores);

/* Wait for the in-flight embed; fill *stats if non-NULL.  RV_ECUDA on a kernel fault. */
rv_status rv_wait(rv_ctx* ctx, rv_stats* stats);

/* After rv_wait of an embed launched with RV_PROFILE: fill up to max_entries per-class
 * records (classes with at least one launch, pipeline order) and return how many were
 * written, or a negative rv_status.  Event durations are taken on the embed's stream. */
int32_t rv_profile(rv_ctx* ctx, rv_kernel_prof* out, int32_t max_entries);

/* After rv_wait: the level-wave structure of the last embed ("report the
 * level-size histogram and per-level M_C").  frames [max_waves] receives the frames of every
 * wave (waves in execution order: dependency levels, large levels split); counts
 * [L][n_waves][2] receives (M_C recomputed rows incl. CLS, M_R reused rows) per layer and wave.
 * Returns the number of waves (also when max_waves is too small or the buffers are NULL: a size
 * query), or a negative rv_status. */
int32_t rv_wave_counts(rv_ctx* ctx, int32_t* frames, int32_t* counts, int32_t max_waves);

/* Human-readable message for the last error on ctx (never NULL; "" when none).  With
 * ctx == NULL returns the last rv_create failure message. */
const char* rv_last_error(const rv_ctx* ctx);
const char* rv_status_string(rv_status s);

/* Free every device and host resource of ctx (NULL is a no-op). */
void rv_destroy(rv_ctx* ctx);

/* ---- Embedding store query (paper §6.1: embeddings are
 * cached per frame as fp16 (~2 KB each at D = 1024) and retrieved by similarity; on a miss the
 * frames are embedded).  No context: plain device buffers on `stream`.
 *
 * rv_f32_to_f16: dst[i] = fp16(src[i]) (round to nearest even), count elements, device
 *   pointers.  RV_ECONTRACT on a negative count or NULL buffers, RV_ECUDA on a launch error.
 * rv_topk_cosine: emb16 [n][D] fp16, q [nq][D] fp32, scores_tmp [nq][n] fp32 scratch (its
 *   contents are destroyed), out_idx [nq][k] int32, out_score [nq][k] fp32, all device.  Row t
 *   of query i is the stored record of t-th highest cosine similarity cos(q_i, e_r) =
 *   q.e / (|q| |e|) (0 when either norm is 0), descending; equal scores are ordered by
 *   the lower record index (SPEC embed-store: ties by (video_id, frame_index), i.e. the store's
 *   record order).  k > n: entries past n are -1 / -inf.  D % 8 == 0.  RV_ECONTRACT on bad
 *   arguments, RV_ECUDA on a launch error; results are complete in stream order. */
rv_status rv_f32_to_f16(const float* src, void* dst, int64_t count, void* stream);
rv_status rv_topk_cosine(const void* emb16, int32_t n, int32_t D, const float* q, int32_t nq, int32_t k,
                         float* scores_tmp, int32_t* out_idx, float* out_score, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* REUSEVIT_H */
