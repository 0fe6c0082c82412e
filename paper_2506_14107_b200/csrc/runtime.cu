// runtime.cu — host runtime of libreusevit: the C-ABI (include/reusevit.h, reusevit_stages.h),
// weight loading, the frame plan, the layer-wise / level-wave scheduler and the reuse cache.
//
// Scheduling (§5.1 P:492-501 layer-wise scheduling): for every layer l,
// the dependency levels of the plan run one after another; each level is ONE compacted wave
// over all resident frames of that level (SURVEY D8 generalises P:571-574's batching).  A
// wave is: score (Eq. 1-4) -> compact (Eq. 5-6) -> gather+LN1 -> QKV GEMM (K/V scattered to
// the cache) -> reused K/V copy + Delta (Eq. 8) -> attention -> CLS t -> W_o GEMM (+res) ->
// LN2 -> FC1 GEMM (+QuickGELU) -> FC2 GEMM (+res, scatter, Eq. 10 C side) -> restoration
// GEMMs (Eq. 9, scatter, Eq. 10 R side).  Counts stay on the device; the whole embed is
// captured once into a CUDA graph and replayed ("avoiding frequent CPU-GPU
// synchronization").
//
// Cached memory compaction (§5.2): the reuse cache holds only the current layer —
// X ping-pong [2][n][T][D] fp32 and K/V [n][T][2D] bf16 — never every layer's activations.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <string>
#include <vector>
#include <chrono>

#include "../../include/reusevit.h"
#include "../../include/reusevit_stages.h"
#include "rv_internal.h"

using namespace rv;

namespace {

struct LayerW {
  float *ln1_g, *ln1_b, *bqkv, *bo, *ln2_g, *ln2_b, *b1, *b2;
  bf16 *Wqkv, *Wo, *W1, *W2;      // [out][in] bf16 (K-major B operands)
  float* gate;                    // Wd1[7][Hg] | bd1[Hg] | Wd2[Hg] | bd2[1]  (fp32)
  bf16 *Wr1, *Wr2;                // [Hr][D], [D][Hr] bf16
  float *br1, *br2;
};

struct Wave {
  int off;   // offset (in frames) into the concatenated wave descriptor array
  int n_w;
  bool any_ref;  // at least one frame with a decision (non-I, not dense)
};

// Scratch of one level-wave (decision outputs, compaction maps, GEMM operands).  The serial
// schedule shares one set (the rv_ctx fields); the wavefront schedule gives every wave its own
// set, sized by its frames, with the A-operand tensor maps of its GEMMs (maps != false).
struct WaveBuf {
  uint8_t *wmask = nullptr, *wprov = nullptr;
  int *cntR = nullptr, *idxC = nullptr, *idxR = nullptr, *provrow = nullptr, *qoff = nullptr, *counts = nullptr,
      *rpos = nullptr, *rloc = nullptr;
  bf16 *A = nullptr, *q = nullptr, *att = nullptr, *h = nullptr, *hr = nullptr, *dfull = nullptr;
  float* x1 = nullptr;
  bool maps = false;
  CUtensorMap tmQ, tmA, tmAtt, tmH, tmD, tmHr;   // q {64 x 64}; GEMM A operands {64 x 128}
};

thread_local std::string g_create_err;

// Level waves of at most this many frames may use the wavefront schedule; larger waves fill the
// GPU on their own (the 7,200-frame workload's 360-1,440-frame waves run serially).
#ifndef RV_WF_MAX_WAVE   // experiment builds (build_variant) may raise it
#define RV_WF_MAX_WAVE 512
#endif
constexpr int kWavefrontMaxWave = RV_WF_MAX_WAVE;

}  // namespace

struct rv_ctx {
  rv_config cfg{};
  int L = 0, D = 0, H = 0, dh = 0, N = 0, T = 0, pp = 0, KP = 0, F = 0, Hr = 0, Hg = 0;
  int device = 0;
  std::string err;
  // ---- weights (device)
  std::vector<void*> wallocs;
  bf16* W_pe = nullptr;
  float *cls = nullptr, *pos = nullptr, *lnpre_g = nullptr, *lnpre_b = nullptr, *lnpost_g = nullptr,
        *lnpost_b = nullptr;
  std::vector<LayerW> lw;
  bool vit_loaded = false, gates_loaded = false;
  // ---- per-embed resources
  int n_cap = 0;
  long long capC = 0, capR = 0;   // row capacities of the wave buffers (multiples of 128)
  std::vector<void*> ballocs;
  float* X[2] = {nullptr, nullptr};
  bf16* KV = nullptr;
  // RV_KEEP_ALL_CACHE (cached memory compaction disabled, P:502-522 ablation): every layer's X
  // [L+1][n][T][D] and K/V [L][n][T][2D] stay allocated instead of the ping-pong / single layer
  bool keepall = false;
  float* Xall = nullptr;
  bf16* KVall = nullptr;
  std::vector<CUtensorMap> tmKVl;
  unsigned long long cache_bytes = 0, alloc_bytes = 0;   // allocated bytes: X + K/V cache, all per-embed buffers
  float* pclsh = nullptr;     // [n][H][N] per-head CLS attention of the previous layer (t)
  int* kvsrc = nullptr;       // [n][T] K/V source row of every token (reuse cache read in place)
  bf16* dfull = nullptr;      // [max_w][T][D] Delta of reused tokens (wave-local token rows, bf16)
  int* rpos = nullptr;        // [max_w][T] compact restoration row of token w*T+i (-1: recomputed)
  int* rloc = nullptr;        // [capR] wave-local Delta row w*T+i of compact reused row r (fused restoration)
  std::vector<CUtensorMap> tmR1, tmR2;   // per layer: W_r1 / W_r2 boxes {64, 128} (k_restore.cu)
  bool fused_restore = false;            // restore_supported(D, Hr): the fused kernel replaces R1 + R2
  bf16* patches_bf16 = nullptr;
  // host-pointer embeds only (no RV_DEVICE_PTRS): staging copies of the caller's host buffers
  int h_cap = 0, hs_cap = 0;
  std::vector<void*> hallocs, hsallocs;
  float *in_patches = nullptr, *in_codec = nullptr, *out_emb = nullptr, *out_scores = nullptr;
  uint8_t* out_masks = nullptr;
  int* wdesc = nullptr;
  int wdesc_cap = 0;
  uint8_t *wmask = nullptr, *wprov = nullptr;
  int *cntR = nullptr, *idxC = nullptr, *idxR = nullptr, *provrow = nullptr, *qoff = nullptr, *counts = nullptr;
  bf16 *A = nullptr, *q = nullptr, *att = nullptr, *h = nullptr, *hr = nullptr;
  float* x1 = nullptr;
  unsigned long long* reuse_ctr = nullptr;   // [L]
  // ---- SPEC chain variant (RV_CHAIN): per-layer q|k|v caches, chain inputs x'
  int chain_cap = 0;
  bf16* QKVc[2] = {nullptr, nullptr};  // [n][T][3D] rows [k | v | q] of layers l (even / odd)
  float* XP = nullptr;                 // [n][T][D] chain input x'_l = X_{l-1} + Attn.Wo + bo
  int* kvsrc2 = nullptr;               // second source-row table (layer l+1's, built by layer l)
  float* pcl2 = nullptr;               // second CLS-attention buffer (t of the next decision)
  int* wrows = nullptr;                // [n][T] global row f*T+i of every wave-local token, desc order
  int* qoffT = nullptr;                // [n+1] w*T (all T tokens of a frame are queries)
  std::vector<int> wrows_host, qoffT_host;
  // GEMM plans (tensor maps) bound to the buffers above
  GemmPlan pe;
  CUtensorMap tmQ;                 // q buffer [capC][D], box {64, 64} (tcgen05 attention)
  CUtensorMap tmKV;                // K/V cache [n T][2 D], box {64, 1}: row gathers (tcgen05 attention)
  std::vector<GemmPlan> g_qkv, g_wo, g_fc1, g_fc2, g_r1, g_r2;
  // ---- wavefront schedule (level waves too small to fill the GPU): wave (l, k)
  // runs as soon as wave (l, k-1) (its references) and wave (l-1, k) (its input) are done, on
  // one stream per wave index, so waves of different layers overlap along the diagonals.  X_l
  // lives in a ring of R layer buffers (Xr[l % R]), K/V_l and the source-row table in rings of
  // R - 1; wave (l, k) waits for wave (l-R+1, last) before overwriting a ring slot.
  int wf_R = 0;                        // ring size of the current embed (0: serial level waves)
  std::vector<long long> wf_key;       // (n_cap, R, wave sizes) the allocations below were made for
  std::vector<void*> wfallocs;
  std::vector<float*> Xr;              // [R]: Xr[0], Xr[1] alias X[0], X[1]
  std::vector<bf16*> KVr;              // [R-1]: KVr[0] aliases KV
  std::vector<int*> KSr;               // [R-1]: KSr[0] aliases kvsrc
  std::vector<CUtensorMap> tmKVr;
  std::vector<WaveBuf> wbuf;           // per wave; wbuf[0] points at the shared buffers
  std::vector<cudaStream_t> wstreams;  // one per wave index
  std::vector<cudaEvent_t> wevents;    // [L][waves] completion of wave (l, k)
  cudaEvent_t wf_fork = nullptr;
  unsigned long long wf_bytes = 0, wf_cache_bytes = 0;
  // ---- graph cache
  cudaGraphExec_t gexec = nullptr;
  std::vector<long long> gkey;
  cudaStream_t own_stream = nullptr;
  cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // ---- in-flight embed
  bool inflight = false;
  int cur_n = 0, cur_nonI = 0, cur_levels = 0, cur_launches = 0;
  uint32_t cur_flags = 0;
  std::vector<int> wdesc_dev_copy;  // what ctx->wdesc holds on the device (cleared on realloc)
  std::vector<int> chain_dev_copy;  // the plan the chain maps (wrows, qoffT) were uploaded for
  const int* chain_dev_ptr = nullptr;
  std::vector<long long> wf_sig;   // wave structure of the last wavefront decision, and its R
  int wf_R_last = 0;
  cudaStream_t cur_stream = nullptr;
  std::vector<Wave> waves;
  std::vector<int> wdesc_host;
  // ---- profiling (RV_PROFILE): event pairs around every launch + per-wave counts log
  struct ProfRec { int cls, l, w; cudaEvent_t a, b; };
  std::vector<cudaEvent_t> prof_pool;
  size_t prof_used = 0;
  std::vector<ProfRec> prof_recs;
  int* count_log = nullptr;          // [L][n_waves][2] = {M_C, M_R}
  int count_log_cap = 0;
  bool prof_valid = false;
  std::vector<rv_kernel_prof> prof_out;
};

enum { K_PATCH, K_PE, K_EMBED, K_SCORE, K_COMPACT, K_GATHER, K_QKV, K_ATTN, K_WO, K_LN2,
       K_FC1, K_FC2, K_R1, K_R2, K_LNPOST, K_RESTORE, K_NCLS };
static const char* kClsName[K_NCLS] = {"patch_to_bf16", "gemm_pe", "embed_finish", "score", "compact",
                                       "gather_ln1", "gemm_qkv", "attention", "gemm_wo", "ln2", "gemm_fc1",
                                       "gemm_fc2", "gemm_r1", "gemm_r2", "ln_post", "restore"};

namespace {

rv_status fail(rv_ctx* c, rv_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (c) c->err = buf;
  else g_create_err = buf;
  return s;
}

#define CK(call)                                                                              \
  do {                                                                                        \
    cudaError_t _e = (call);                                                                  \
    if (_e != cudaSuccess)                                                                    \
      return fail(ctx, RV_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(_e)); \
  } while (0)

bool cfg_valid(const rv_config* c, char* why, size_t n) {
  if (!c) { snprintf(why, n, "null config"); return false; }
  if (c->layers < 1 || c->layers > 64) { snprintf(why, n, "layers must be 1..64"); return false; }
  if (c->dim < 64 || c->dim > 1024 || c->dim % 64) { snprintf(why, n, "dim must be a multiple of 64 in [64,1024]"); return false; }
  if (c->heads < 1 || c->dim % c->heads) { snprintf(why, n, "dim %% heads != 0 (S:99)"); return false; }
  const int dh = c->dim / c->heads;
  if (dh != 16 && dh != 64) { snprintf(why, n, "dim/heads must be 16 or 64"); return false; }
  if (c->heads > 32) { snprintf(why, n, "heads must be <= 32"); return false; }
  if (c->patch < 1 || c->img < c->patch || c->img % c->patch) { snprintf(why, n, "img must be a positive multiple of patch"); return false; }
  const int N = (c->img / c->patch) * (c->img / c->patch);
  if (N + 1 > 768) { snprintf(why, n, "T = N+1 must be <= 768 (attention keeps a frame's K/V in smem)"); return false; }
  if (c->ffn < 64 || c->ffn % 64) { snprintf(why, n, "ffn must be a positive multiple of 64"); return false; }
  if (c->hidden_r < 64 || c->hidden_r % 64) { snprintf(why, n, "hidden_r must be a positive multiple of 64"); return false; }
  if (c->hidden_g < 1 || c->hidden_g > 32) { snprintf(why, n, "hidden_g must be 1..32"); return false; }
  return true;
}

size_t vit_floats(const rv_config* c) {
  const size_t D = c->dim, F = c->ffn, N = (size_t)(c->img / c->patch) * (c->img / c->patch), T = N + 1,
               pp = 3ull * c->patch * c->patch;
  size_t per = 2 * D + D * 3 * D + 3 * D + D * D + D + 2 * D + D * F + F + F * D + D;
  return pp * D + D + T * D + 2 * D + c->layers * per + 2 * D;
}
size_t gate_floats(const rv_config* c) {
  const size_t D = c->dim, Hr = c->hidden_r, Hg = c->hidden_g;
  return c->layers * (7 * Hg + Hg + Hg + 1 + D * Hr + Hr + Hr * D + D);
}

template <class T>
rv_status dalloc(rv_ctx* ctx, std::vector<void*>& list, T** p, size_t count) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return fail(ctx, RV_ENOMEM, "cudaMalloc(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
  }
  list.push_back(q);
  *p = reinterpret_cast<T*>(q);
  return RV_OK;
}

// Host conversion helpers for weight upload.
uint16_t f2bf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return 0x7fc0;
  const uint32_t r = 0x7fffu + ((u >> 16) & 1u);
  return (uint16_t)((u + r) >> 16);
}

// Upload an [in][out] fp32 matrix as bf16 [out][inP] (transposed, K zero-padded to inP).
rv_status upload_T(rv_ctx* ctx, std::vector<void*>& list, bf16** dst, const float* src, int in, int out, int inP) {
  std::vector<uint16_t> tmp((size_t)out * inP, 0);
  for (int i = 0; i < in; ++i)
    for (int o = 0; o < out; ++o) tmp[(size_t)o * inP + i] = f2bf(src[(size_t)i * out + o]);
  rv_status s = dalloc(ctx, list, dst, tmp.size());
  if (s) return s;
  CK(cudaMemcpy(*dst, tmp.data(), tmp.size() * 2, cudaMemcpyHostToDevice));
  return RV_OK;
}
rv_status upload_f(rv_ctx* ctx, std::vector<void*>& list, float** dst, const float* src, size_t n) {
  rv_status s = dalloc(ctx, list, dst, n);
  if (s) return s;
  CK(cudaMemcpy(*dst, src, n * 4, cudaMemcpyHostToDevice));
  return RV_OK;
}

void free_list(std::vector<void*>& l) {
  for (void* p : l) cudaFree(p);
  l.clear();
}

cudaEvent_t ctx_event(rv_ctx* ctx) {
  if (ctx->prof_used == ctx->prof_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ctx->prof_pool.push_back(e);
  }
  return ctx->prof_pool[ctx->prof_used++];
}

// ------------------------------------------------------------------ plan helpers
rv_status check_plan(rv_ctx* ctx, const rv_plan* p, std::vector<int>* level_out) {
  if (!p || p->n < 1 || !p->type || !p->past || !p->future || !p->order)
    return fail(ctx, RV_ECONTRACT, "plan: null array or n < 1");
  const int n = p->n;
  std::vector<int> pos(n, -1);
  for (int k = 0; k < n; ++k) {
    const int f = p->order[k];
    if (f < 0 || f >= n || pos[f] >= 0) return fail(ctx, RV_EPLAN, "plan: order is not a permutation (at %d)", k);
    pos[f] = k;
  }
  std::vector<int> lev(n, -1);
  for (int k = 0; k < n; ++k) {
    const int f = p->order[k];
    const int t = p->type[f];
    if (t < RV_I || t > RV_B1) return fail(ctx, RV_EPLAN, "plan: frame %d has bad type %d", f, t);
    const int r[2] = {p->past[f], p->future[f]};
    int lv = 0, nref = 0;
    for (int j = 0; j < 2; ++j) {
      if (r[j] == -1) continue;
      if (r[j] < 0 || r[j] >= n || r[j] == f) return fail(ctx, RV_EPLAN, "plan: frame %d has bad reference %d", f, r[j]);
      if (pos[r[j]] >= k) return fail(ctx, RV_EPLAN, "plan: frame %d references %d before it is computed (S:316)", f, r[j]);
      lv = std::max(lv, lev[r[j]] + 1);
      ++nref;
    }
    if (t == RV_I && nref) return fail(ctx, RV_EPLAN, "plan: I-frame %d has references", f);
    if (t != RV_I && !nref) return fail(ctx, RV_EPLAN, "plan: non-I frame %d has no reference", f);
    lev[f] = lv;
  }
  if (level_out) *level_out = lev;
  return RV_OK;
}

// ------------------------------------------------------------------ buffers
// Drop every per-embed buffer and the state encoded from their addresses (graph, tensor maps,
// GEMM plans): after a failed re-allocation the context holds no dangling pointer, and the
// next embed allocates again from scratch.
void release_wavefront(rv_ctx* ctx) {
  if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; ctx->gkey.clear(); }
  free_list(ctx->wfallocs);
  ctx->wf_key.clear();
  ctx->wf_sig.clear();
  ctx->Xr.clear(); ctx->KVr.clear(); ctx->KSr.clear(); ctx->tmKVr.clear(); ctx->wbuf.clear();
  ctx->wf_bytes = ctx->wf_cache_bytes = 0;
}

void release_buffers(rv_ctx* ctx) {
  release_wavefront(ctx);   // its rings alias X[0], X[1], KV and kvsrc
  if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; ctx->gkey.clear(); }
  free_list(ctx->ballocs);
  ctx->n_cap = 0; ctx->capC = 0; ctx->capR = 0; ctx->wdesc_cap = 0; ctx->chain_cap = 0;
  ctx->X[0] = ctx->X[1] = nullptr; ctx->KV = nullptr; ctx->pclsh = nullptr; ctx->kvsrc = nullptr;
  ctx->Xall = nullptr; ctx->KVall = nullptr; ctx->keepall = false; ctx->tmKVl.clear();
  ctx->cache_bytes = ctx->alloc_bytes = 0;
  ctx->dfull = nullptr; ctx->rpos = nullptr; ctx->rloc = nullptr; ctx->patches_bf16 = nullptr; ctx->wdesc = nullptr;
  ctx->wdesc_dev_copy.clear();
  ctx->wmask = ctx->wprov = nullptr;
  ctx->cntR = ctx->idxC = ctx->idxR = ctx->provrow = ctx->qoff = ctx->counts = nullptr;
  ctx->A = ctx->q = ctx->att = ctx->h = ctx->hr = nullptr; ctx->x1 = nullptr; ctx->reuse_ctr = nullptr;
  ctx->QKVc[0] = ctx->QKVc[1] = nullptr; ctx->XP = nullptr; ctx->kvsrc2 = nullptr; ctx->pcl2 = nullptr;
  ctx->wrows = nullptr; ctx->qoffT = nullptr;
}

rv_status ensure_buffers(rv_ctx* ctx, int n, long long capC, long long capR, int max_w, bool keepall) {
  capC = (capC + 127) / 128 * 128;
  capR = std::max<long long>(128, (capR + 127) / 128 * 128);
  if (n <= ctx->n_cap && capC <= ctx->capC && capR <= ctx->capR && max_w <= ctx->wdesc_cap && keepall == ctx->keepall)
    return RV_OK;
  if (keepall != ctx->keepall) release_buffers(ctx);   // switching modes: start from the request's sizes
  n = std::max(n, ctx->n_cap);
  capC = std::max(capC, ctx->capC);
  capR = std::max(capR, ctx->capR);
  max_w = std::max(max_w, ctx->wdesc_cap);
  release_buffers(ctx);
  const long long T = ctx->T, D = ctx->D, N = ctx->N;
  auto& B = ctx->ballocs;
  rv_status s;
  const long long L = ctx->L;
  unsigned long long bytes = 0;
#define AL(ptr, cnt)                                                                 \
  if ((s = dalloc(ctx, B, &ptr, (size_t)(cnt)))) { release_buffers(ctx); return s; } \
  bytes += (unsigned long long)(cnt) * sizeof(*ptr)
  if (keepall) {
    AL(ctx->Xall, (L + 1) * n * T * D);
    AL(ctx->KVall, L * n * T * 2 * D);
    ctx->X[0] = ctx->Xall;
    ctx->KV = ctx->KVall;
  } else {
    AL(ctx->X[0], n * T * D);
    AL(ctx->X[1], n * T * D);
    AL(ctx->KV, n * T * 2 * D);
  }
  const unsigned long long cache = bytes;
  AL(ctx->pclsh, n * ctx->H * N);
  AL(ctx->kvsrc, n * T);
  AL(ctx->dfull, (size_t)max_w * T * D);
  AL(ctx->rpos, max_w * T);
  AL(ctx->rloc, capR);
  AL(ctx->patches_bf16, (size_t)n * N * ctx->KP);
  AL(ctx->wdesc, (size_t)n * 4);
  AL(ctx->wmask, max_w * T);
  AL(ctx->wprov, max_w * T);
  AL(ctx->cntR, max_w);
  AL(ctx->qoff, max_w + 1);
  AL(ctx->counts, 2);
  AL(ctx->idxC, capC);
  AL(ctx->idxR, capR);
  AL(ctx->provrow, capR);
  AL(ctx->A, capC * D);
  AL(ctx->q, capC * D);
  AL(ctx->att, capC * D);
  AL(ctx->x1, capC * D);
  AL(ctx->h, capC * ctx->F);
  AL(ctx->hr, capR * ctx->Hr);
  AL(ctx->reuse_ctr, 64);
#undef AL
  // the restoration GEMM R1 also reads the never-written Delta rows of C tokens (results discarded)
  if (cudaMemset(ctx->dfull, 0, (size_t)max_w * T * D * sizeof(bf16)) != cudaSuccess) {
    release_buffers(ctx);
    return fail(ctx, RV_ECUDA, "cudaMemset failed");
  }
  char e[256];
  bool ok = make_tmap_bf16(&ctx->tmQ, ctx->q, capC, (int)D, 64, e, sizeof e) &&
            make_tmap_bf16(&ctx->tmKV, ctx->KV, (long long)n * T, 2 * (int)D, 1, e, sizeof e) &&
            gemm_make_plan(&ctx->pe, ctx->patches_bf16, (long long)n * N, ctx->W_pe, (int)D, ctx->KP, e, sizeof e);
  if (ok && keepall) {
    ctx->tmKVl.resize(L);
    for (int l = 0; ok && l < L; ++l)
      ok = make_tmap_bf16(&ctx->tmKVl[l], ctx->KVall + (size_t)l * n * T * 2 * D, (long long)n * T, 2 * (int)D, 1, e,
                          sizeof e);
  }
  ctx->g_qkv.resize(L); ctx->g_wo.resize(L); ctx->g_fc1.resize(L); ctx->g_fc2.resize(L);
  ctx->g_r1.resize(L); ctx->g_r2.resize(L);
  for (int l = 0; ok && l < L; ++l) {
    const LayerW& w = ctx->lw[l];
    ok = gemm_make_plan(&ctx->g_qkv[l], ctx->A, capC, w.Wqkv, 3 * (int)D, (int)D, e, sizeof e) &&
         gemm_make_plan(&ctx->g_wo[l], ctx->att, capC, w.Wo, (int)D, (int)D, e, sizeof e) &&
         gemm_make_plan(&ctx->g_fc1[l], ctx->A, capC, w.W1, ctx->F, (int)D, e, sizeof e) &&
         gemm_make_plan(&ctx->g_fc2[l], ctx->h, capC, w.W2, (int)D, ctx->F, e, sizeof e);
    if (ok && ctx->gates_loaded)
      ok = gemm_make_plan(&ctx->g_r1[l], ctx->dfull, max_w * T, w.Wr1, ctx->Hr, (int)D, e, sizeof e) &&
           gemm_make_plan(&ctx->g_r2[l], ctx->hr, capR, w.Wr2, (int)D, ctx->Hr, e, sizeof e);
  }
  ctx->fused_restore = ctx->gates_loaded && restore_supported((int)D, ctx->Hr);
  ctx->tmR1.resize(L); ctx->tmR2.resize(L);
  for (int l = 0; ok && ctx->fused_restore && l < L; ++l)
    ok = restore_make_maps(&ctx->tmR1[l], &ctx->tmR2[l], ctx->lw[l].Wr1, ctx->lw[l].Wr2, (int)D, ctx->Hr, e, sizeof e);
  if (!ok) {
    release_buffers(ctx);
    return fail(ctx, RV_ECUDA, "%s", e);
  }
  ctx->n_cap = n;
  ctx->capC = capC;
  ctx->capR = capR;
  ctx->wdesc_cap = max_w;
  ctx->keepall = keepall;
  ctx->cache_bytes = cache;
  ctx->alloc_bytes = bytes;
  return RV_OK;
}

// Bytes the wavefront schedule adds for ring size R on top of ensure_buffers' allocations.
unsigned long long wavefront_bytes(const rv_ctx* ctx, int n, int R, const std::vector<Wave>& waves) {
  const unsigned long long T = ctx->T, D = ctx->D, N = ctx->N, F = ctx->F, Hr = ctx->Hr;
  unsigned long long b = (unsigned long long)(R - 2) * n * T * D * 4 + (unsigned long long)(R - 2) * n * T * (2 * D * 2 + 4);
  for (size_t wi = 1; wi < waves.size(); ++wi) {
    const unsigned long long rows = waves[wi].n_w * T, capC = (rows + 127) / 128 * 128;
    const unsigned long long capR = std::max<unsigned long long>(128, (waves[wi].n_w * N + 127) / 128 * 128);
    b += rows * (2 + 4 + D * 2) + capC * (4 + D * 2 * 3 + D * 4 + F * 2) + capR * (8 + Hr * 2) + waves[wi].n_w * 8 + 64;
  }
  return b;
}

// Wavefront buffers for ring size R >= 3: the extra X / K/V / source-row ring slots and every
// wave's own scratch (wave 0 keeps the shared set).  Streams and events persist in the context.
rv_status ensure_wavefront(rv_ctx* ctx, int R) {
  const int nw = (int)ctx->waves.size(), L = ctx->L;
  std::vector<long long> key = {(long long)ctx->n_cap, (long long)R, ctx->capC, ctx->capR};
  for (const Wave& w : ctx->waves) key.push_back(w.n_w * 2 + (w.any_ref ? 1 : 0));
  if (key == ctx->wf_key) return RV_OK;
  release_wavefront(ctx);
  const long long n = ctx->n_cap, T = ctx->T, D = ctx->D, N = ctx->N;
  auto& B = ctx->wfallocs;
  rv_status s;
  unsigned long long bytes = 0, cache = 0;
#define AL(ptr, cnt)                                                                  \
  if ((s = dalloc(ctx, B, &ptr, (size_t)(cnt)))) { release_wavefront(ctx); return s; } \
  bytes += (unsigned long long)(cnt) * sizeof(*ptr)
  ctx->Xr.assign(R, nullptr);
  ctx->Xr[0] = ctx->X[0];
  ctx->Xr[1] = ctx->X[1];
  for (int r = 2; r < R; ++r) { AL(ctx->Xr[r], n * T * D); }
  ctx->KVr.assign(R - 1, nullptr);
  ctx->KSr.assign(R - 1, nullptr);
  ctx->KVr[0] = ctx->KV;
  ctx->KSr[0] = ctx->kvsrc;
  for (int r = 1; r < R - 1; ++r) {
    AL(ctx->KVr[r], n * T * 2 * D);
    AL(ctx->KSr[r], n * T);
  }
  cache = bytes;
  char e[256];
  bool ok = true;
  ctx->tmKVr.resize(R - 1);
  for (int r = 0; ok && r < R - 1; ++r) ok = make_tmap_bf16(&ctx->tmKVr[r], ctx->KVr[r], n * T, 2 * (int)D, 1, e, sizeof e);
  ctx->wbuf.assign(nw, WaveBuf());
  for (int wi = 0; ok && wi < nw; ++wi) {
    WaveBuf& b = ctx->wbuf[wi];
    const long long nwf = ctx->waves[wi].n_w;
    long long capC = ctx->capC, capR = ctx->capR, rowsD = (long long)ctx->wdesc_cap * T;
    if (wi == 0) {
      b.wmask = ctx->wmask; b.wprov = ctx->wprov; b.cntR = ctx->cntR; b.idxC = ctx->idxC; b.idxR = ctx->idxR;
      b.provrow = ctx->provrow; b.qoff = ctx->qoff; b.counts = ctx->counts; b.rpos = ctx->rpos; b.A = ctx->A;
      b.rloc = ctx->rloc;
      b.q = ctx->q; b.att = ctx->att; b.h = ctx->h; b.hr = ctx->hr; b.dfull = ctx->dfull; b.x1 = ctx->x1;
    } else {
      capC = (nwf * T + 127) / 128 * 128;
      capR = std::max<long long>(128, (nwf * N + 127) / 128 * 128);
      rowsD = nwf * T;
      AL(b.wmask, nwf * T);
      AL(b.wprov, nwf * T);
      AL(b.cntR, nwf);
      AL(b.qoff, nwf + 1);
      AL(b.counts, 2);
      AL(b.rpos, nwf * T);
      AL(b.rloc, capR);
      AL(b.idxC, capC);
      AL(b.idxR, capR);
      AL(b.provrow, capR);
      AL(b.A, capC * D);
      AL(b.q, capC * D);
      AL(b.att, capC * D);
      AL(b.x1, capC * D);
      AL(b.h, capC * ctx->F);
      AL(b.hr, capR * ctx->Hr);
      AL(b.dfull, rowsD * D);
      if (cudaMemset(b.dfull, 0, (size_t)rowsD * D * sizeof(bf16)) != cudaSuccess) {
        release_wavefront(ctx);
        return fail(ctx, RV_ECUDA, "cudaMemset failed");
      }
    }
    b.maps = true;
    ok = make_tmap_bf16(&b.tmQ, b.q, capC, (int)D, 64, e, sizeof e) &&
         make_tmap_bf16(&b.tmA, b.A, capC, (int)D, 128, e, sizeof e) &&
         make_tmap_bf16(&b.tmAtt, b.att, capC, (int)D, 128, e, sizeof e) &&
         make_tmap_bf16(&b.tmH, b.h, capC, ctx->F, 128, e, sizeof e) &&
         make_tmap_bf16(&b.tmD, b.dfull, rowsD, (int)D, 128, e, sizeof e) &&
         make_tmap_bf16(&b.tmHr, b.hr, capR, ctx->Hr, 128, e, sizeof e);
  }
#undef AL
  if (!ok) {
    release_wavefront(ctx);
    return fail(ctx, RV_ECUDA, "%s", e);
  }
  while ((int)ctx->wstreams.size() < nw) {
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    ctx->wstreams.push_back(st);
  }
  while ((int)ctx->wevents.size() < L * nw) {
    cudaEvent_t ev;
    CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    ctx->wevents.push_back(ev);
  }
  if (!ctx->wf_fork) CK(cudaEventCreateWithFlags(&ctx->wf_fork, cudaEventDisableTiming));
  ctx->wf_key = key;
  ctx->wf_bytes = bytes;
  ctx->wf_cache_bytes = cache;
  return RV_OK;
}

// Staging buffers of host-pointer embeds (never allocated on the RV_DEVICE_PTRS path).
rv_status ensure_host_buffers(rv_ctx* ctx, int n, bool scores) {
  rv_status s;
  if (n > ctx->h_cap) {
    if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; ctx->gkey.clear(); }
    free_list(ctx->hallocs);
    ctx->h_cap = 0;
    const long long N = ctx->N;
#define AL(ptr, cnt) if ((s = dalloc(ctx, ctx->hallocs, &ptr, (size_t)(cnt)))) { free_list(ctx->hallocs); return s; }
    AL(ctx->in_patches, (size_t)n * N * ctx->pp);
    AL(ctx->in_codec, n * N);
    AL(ctx->out_emb, (size_t)n * ctx->D);
    AL(ctx->out_masks, (size_t)n * ctx->L * N);
#undef AL
    ctx->h_cap = n;
  }
  if (scores && n > ctx->hs_cap) {
    if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; ctx->gkey.clear(); }
    free_list(ctx->hsallocs);
    ctx->hs_cap = 0;
    if ((s = dalloc(ctx, ctx->hsallocs, &ctx->out_scores, (size_t)n * ctx->L * ctx->N))) return s;
    ctx->hs_cap = n;
  }
  return RV_OK;
}

// ------------------------------------------------------------------ the embed sequence
struct Rec {
  rv_ctx* ctx;
  cudaStream_t s;
  int launches = 0;
  cudaError_t err = cudaSuccess;
  const char* where = "";
  bool prof = false;
  int cur_cls = -1, cur_l = -1, cur_w = -1;
  cudaEvent_t cur_ev = nullptr;
  // Start a timed launch of kernel class `cls` (profiling embeds only).
  void begin(int cls, int l, int wi) {
    if (!prof || err != cudaSuccess) return;
    cur_cls = cls; cur_l = l; cur_w = wi;
    cur_ev = ctx_event(ctx);
    cudaError_t e = cudaEventRecordWithFlags(cur_ev, s, cudaEventRecordExternal);
    if (e != cudaSuccess && err == cudaSuccess) { err = e; where = "event"; }
  }
  void chk(cudaError_t e, const char* w) {
    ++launches;
    if (e != cudaSuccess && err == cudaSuccess) { err = e; where = w; }
    if (prof && cur_cls >= 0 && err == cudaSuccess) {
      cudaEvent_t end = ctx_event(ctx);
      cudaError_t e2 = cudaEventRecordWithFlags(end, s, cudaEventRecordExternal);
      if (e2 != cudaSuccess && err == cudaSuccess) { err = e2; where = "event"; }
      ctx->prof_recs.push_back({cur_cls, cur_l, cur_w, cur_ev, end});
    }
    cur_cls = -1;
  }
};

void record_embed(rv_ctx* ctx, Rec& r, int n, uint32_t flags, const float* patches, const float* codec,
                  float* emb, uint8_t* masks, float* scores) {
  const int L = ctx->L, D = ctx->D, T = ctx->T, N = ctx->N, H = ctx->H, F = ctx->F, Hr = ctx->Hr;
  cudaStream_t s = r.s;
  const cudaStream_t s0 = s;   // the embed stream (wave streams fork from and join into it)
  const bool dense = flags & RV_DENSE;
  const bool force = flags & RV_FORCE_MASKS;
  // RV_X_BF16: the residual stream X (every layer's input/output rows) is stored in bf16; the X
  // buffers keep their fp32 size and hold the bf16 rows in their first half-rows
  const int xb = (flags & RV_X_BF16) ? 1 : 0;
  r.chk(launch_zero_words(ctx->reuse_ctr, 128, s), "zero reuse counters");
  // a1: patch embed (dense, all frames): bf16 operand, GEMM into X0 rows f*T+1+i, finish.
  r.begin(K_PATCH,-1,-1);
  r.chk(launch_patch_to_bf16(patches, ctx->patches_bf16, (long long)n * N, ctx->pp, ctx->KP, s), "patch_to_bf16");
  {
    Epi e;
    e.out = ctx->X[0];
    e.out_ld = D;
    e.out_bf16 = xb;
    e.row_div = N;
    e.row_add = 1;
    r.begin(K_PE,-1,-1);
    r.chk(gemm_launch(ctx->pe, nullptr, n * N, n * N, e, s), "gemm_pe");
  }
  r.begin(K_EMBED,-1,-1);
  r.chk(launch_embed_finish(ctx->X[0], xb, ctx->cls, ctx->pos, ctx->lnpre_g, ctx->lnpre_b, ctx->pclsh, n, T, D, N, H, s),
        "embed_finish");
  const bool keepall = ctx->keepall;
  const size_t nTD = (size_t)ctx->n_cap * T * D;
  const int R = ctx->wf_R;                 // >= 3: wavefront schedule over rings of layer buffers
  const int nwv = (int)ctx->waves.size();
  // X_l (input of layer l + 1), K/V_l and the source-row table of layer l
  auto Xbuf = [&](int l) -> float* {   // (bf16 rows with RV_X_BF16: same base, half the row stride)
    return keepall ? ctx->Xall + (size_t)l * nTD : (R ? ctx->Xr[l % R] : ctx->X[l & 1]);
  };
  auto KVbuf = [&](int l) -> bf16* {
    return keepall ? ctx->KVall + (size_t)l * 2 * nTD : (R ? ctx->KVr[l % (R - 1)] : ctx->KV);
  };
  auto tmKVbuf = [&](int l) -> const CUtensorMap& {
    return keepall ? ctx->tmKVl[l] : (R ? ctx->tmKVr[l % (R - 1)] : ctx->tmKV);
  };
  auto KSbuf = [&](int l) -> int* { return R ? ctx->KSr[l % (R - 1)] : ctx->kvsrc; };
  WaveBuf shared;   // the serial schedule's wave buffers (tensor maps: the GEMM plans' own)
  shared.wmask = ctx->wmask; shared.wprov = ctx->wprov; shared.cntR = ctx->cntR; shared.idxC = ctx->idxC;
  shared.idxR = ctx->idxR; shared.provrow = ctx->provrow; shared.qoff = ctx->qoff; shared.counts = ctx->counts;
  shared.rpos = ctx->rpos; shared.rloc = ctx->rloc; shared.A = ctx->A; shared.q = ctx->q; shared.att = ctx->att; shared.h = ctx->h;
  shared.hr = ctx->hr; shared.dfull = ctx->dfull; shared.x1 = ctx->x1;
  auto plan = [](const GemmPlan& p, const WaveBuf& b, const CUtensorMap& a) {
    GemmPlan q = p;
    if (b.maps) q.tmA = a;
    return q;
  };
  if (R) {   // fork: every wave stream starts after the patch embed
    r.chk(cudaEventRecord(ctx->wf_fork, s), "fork");
    --r.launches;
    for (int wi = 0; wi < nwv; ++wi) {
      r.chk(cudaStreamWaitEvent(ctx->wstreams[wi], ctx->wf_fork, 0), "fork");
      --r.launches;
    }
  }
  for (int l = 0; l < L; ++l) {
    const LayerW& w = ctx->lw[l];
    float* Xin = Xbuf(l);
    float* Xout = Xbuf(l + 1);
    bf16* KVl = KVbuf(l);
    const CUtensorMap& tmKVl = tmKVbuf(l);
    int* kvsrc = KSbuf(l);
    for (int wi = 0; wi < nwv; ++wi) {
      const Wave& wv = ctx->waves[wi];
      const int n_w = wv.n_w;
      const int* wd = ctx->wdesc + (size_t)wv.off * 4;
      const int maxC = n_w * T;
      const WaveBuf& b = R ? ctx->wbuf[wi] : shared;
      if (R) {
        // wave (l, wi) runs after wave (l, wi - 1) (the lower levels hold its references) and,
        // since it overwrites ring slots, after wave (l - R + 1, last): the last reader of
        // X_{l-R} (scores of layer l - R + 1) and of K/V_{l-R+1} and its source rows.  Wave
        // (l - 1, wi) precedes it on its own stream.
        s = ctx->wstreams[wi];
        r.s = s;
        if (wi > 0) {
          r.chk(cudaStreamWaitEvent(s, ctx->wevents[(size_t)l * nwv + wi - 1], 0), "wave dependency");
          --r.launches;
        }
        if (l - R + 1 >= 0) {
          r.chk(cudaStreamWaitEvent(s, ctx->wevents[(size_t)(l - R + 1) * nwv + nwv - 1], 0), "ring dependency");
          --r.launches;
        }
      }
      // a2-a3: Eq. 1-4
      r.begin(K_SCORE,l,wi);
      r.chk(launch_score(Xin, xb, T, D, N, L, l, n_w, wd, ctx->pclsh, H, codec, force ? masks : nullptr,
                         ctx->gates_loaded ? w.gate : nullptr, ctx->Hg, dense ? 1 : 0, masks, scores, b.wmask,
                         b.wprov, b.cntR, b.dfull, s),
            "score");
      // a4: Eq. 5-6 stream compaction
      r.begin(K_COMPACT,l,wi);
      r.chk(launch_compact(n_w, T, wd, b.wmask, b.wprov, b.cntR, b.idxC, b.idxR, b.provrow, b.qoff, b.counts, kvsrc,
                           ctx->reuse_ctr + l, ctx->count_log + ((size_t)l * nwv + wi) * 2, b.rpos,
                           (ctx->fused_restore && !(flags & RV_RESTORE_GEMMS)) ? b.rloc : nullptr, s,
                           (flags & RV_NO_COMPACTION) ? 1 : 0),
            "compact");
      const int* MC = b.counts;
      // a5: gather + LN1
      r.begin(K_GATHER,l,wi);
      r.chk(launch_gather_ln(Xin, xb, b.idxC, MC, 0, maxC, w.ln1_g, w.ln1_b, b.A, D, s), "gather_ln1");
      // a6: QKV; q compact, K/V scattered to the cache rows of C
      {
        Epi e;
        e.bias = w.bqkv;
        e.out = b.q;
        e.out_ld = D;
        e.out_bf16 = 1;
        e.split = D;
        e.out2 = KVl;
        e.out2_rows = b.idxC;
        e.out2_ld = 2LL * D;
        e.out2_bf16 = 1;
        r.begin(K_QKV,l,wi);
        r.chk(gemm_launch(plan(ctx->g_qkv[l], b, b.tmA), MC, 0, maxC, e, s), "gemm_qkv");
      }
      // a8: attention over all T keys; CLS row -> t for layer l+1
      r.begin(K_ATTN,l,wi);
      {
        float* pcl = (!dense && l + 1 < L) ? ctx->pclsh : nullptr;
        const CUtensorMap& tmQ = b.maps ? b.tmQ : ctx->tmQ;
        if (!(flags & RV_ATTN_SYNC) && attn_tc_supported(T, D, H))   // tcgen05/TMEM, T <= 257 (default)
          r.chk(launch_attention_tc(tmQ, tmKVl, KVl, kvsrc, b.att, wd, b.qoff, pcl, n_w, T, D, H, s), "attention");
        else if (!(flags & RV_ATTN_SYNC) && attn_tcg_supported(T, D, H))   // tcgen05/TMEM, any T (L/14@336)
          r.chk(launch_attention_tcg(&tmQ, b.q, D, 0, 0, KVl, 2LL * D, kvsrc, b.att, wd, b.qoff, pcl, n_w, T, D, H, s),
                "attention");
        else   // mma.sync kernel: d_h = 16 (tiny config) or RV_ATTN_SYNC
          r.chk(launch_attention(b.q, KVl, kvsrc, b.att, wd, b.qoff, pcl, n_w, T, D, H, s), "attention");
      }
      // a9: W_o + residual (gathered X_{l-1} rows)
      {
        Epi e;
        e.bias = w.bo;
        e.resid = Xin;
        e.resid_rows = b.idxC;
        e.resid_ld = D;
        e.resid_bf16 = xb;
        e.out = b.x1;
        e.out_ld = D;
        r.begin(K_WO,l,wi);
        r.chk(gemm_launch(plan(ctx->g_wo[l], b, b.tmAtt), MC, 0, maxC, e, s), "gemm_wo");
      }
      // a10: LN2 + FC1 + QuickGELU
      r.begin(K_LN2,l,wi);
      r.chk(launch_gather_ln(b.x1, 0, nullptr, MC, 0, maxC, w.ln2_g, w.ln2_b, b.A, D, s), "ln2");
      {
        Epi e;
        e.bias = w.b1;
        e.act = 1;
        e.out = b.h;
        e.out_ld = F;
        e.out_bf16 = 1;
        r.begin(K_FC1,l,wi);
        r.chk(gemm_launch(plan(ctx->g_fc1[l], b, b.tmA), MC, 0, maxC, e, s), "gemm_fc1");
      }
      // a11: FC2 + residual, scattered to X_l rows of C (Eq. 10, C side)
      {
        Epi e;
        e.bias = w.b2;
        e.resid = b.x1;
        e.resid_ld = D;
        e.out = Xout;
        e.out_rows = b.idxC;
        e.out_ld = D;
        e.out_bf16 = xb;
        r.begin(K_FC2,l,wi);
        r.chk(gemm_launch(plan(ctx->g_fc2[l], b, b.tmH), MC, 0, maxC, e, s), "gemm_fc2");
      }
      // a12: restoration (Eq. 9) + merge (Eq. 10, R side).  The score pass wrote Delta (Eq. 8)
      // into the wave-local token rows w*T+i; R1 reads them in place over all n_w*T rows and
      // stores only the reused rows, compacted (row map rpos; -1 for C rows): no Delta copy.
      // R2 runs over the M_R compact rows.  Where restore_supported (every CLIP shape) both are
      // one fused kernel over the M_R compact reused rows instead (k_restore.cu): Delta gathered
      // by rloc, hr kept on chip, provider rows of X_l streamed in, restored rows scattered.
      if (wv.any_ref && !dense && ctx->fused_restore && !(flags & RV_RESTORE_GEMMS)) {
        r.begin(K_RESTORE,l,wi);
        r.chk(launch_restore(ctx->tmR1[l], ctx->tmR2[l], b.dfull, b.rloc, b.provrow, b.idxR, b.counts + 1, n_w * N,
                             w.br1, w.br2, Xout, xb, D, s),
              "restore");
      } else if (wv.any_ref && !dense) {
        Epi e1;
        e1.bias = w.br1;
        e1.act = 1;
        e1.out = b.hr;
        e1.out_ld = Hr;
        e1.out_bf16 = 1;
        e1.out_rows = b.rpos;
        r.begin(K_R1,l,wi);
        r.chk(gemm_launch(plan(ctx->g_r1[l], b, b.tmD), nullptr, n_w * T, n_w * T, e1, s), "gemm_r1");
        Epi e2;
        e2.bias = w.br2;
        e2.resid = Xout;
        e2.resid_rows = b.provrow;
        e2.resid_ld = D;
        e2.resid_bf16 = xb;
        e2.out = Xout;
        e2.out_rows = b.idxR;
        e2.out_ld = D;
        e2.out_bf16 = xb;
        r.begin(K_R2,l,wi);
        r.chk(gemm_launch(plan(ctx->g_r2[l], b, b.tmHr), b.counts + 1, 0, n_w * N, e2, s), "gemm_r2");
      }
      if (R) {
        r.chk(cudaEventRecord(ctx->wevents[(size_t)l * nwv + wi], s), "wave event");
        --r.launches;
      }
    }
  }
  if (R) {   // join every wave stream back into the embed stream
    s = r.s = s0;
    for (int wi = 0; wi < nwv; ++wi) {
      r.chk(cudaStreamWaitEvent(s, ctx->wevents[(size_t)(L - 1) * nwv + wi], 0), "join");
      --r.launches;
    }
  }
  // a14: Z = LN_post(CLS), slots are display indices
  r.begin(K_LNPOST,-1,-1);
  r.chk(launch_ln_post(Xbuf(L), xb, ctx->lnpost_g, ctx->lnpost_b, emb, n, T, D, s), "ln_post");
}

// SPEC chain variant (RV_CHAIN; oracle/chain_ref.py):
// per layer l, attention and W_o run densely over all T tokens; the decision taken on the chain
// input x'_l gates FFN_l -> QKV_{l+1}; reused tokens take the provider's restored block output
// (X_l) and its q, k, v of layer l+1 (read in place through the source-row table).  Same kernels
// as the D1 path: the mma.sync attention in its cache-resident-q mode, the tcgen05 GEMMs with
// row-mapped epilogues, the score / compaction / restoration kernels unchanged.
void record_embed_chain(rv_ctx* ctx, Rec& r, int n, uint32_t flags, const float* patches, const float* codec,
                        float* emb, uint8_t* masks, float* scores) {
  const int L = ctx->L, D = ctx->D, T = ctx->T, N = ctx->N, H = ctx->H, F = ctx->F, Hr = ctx->Hr;
  cudaStream_t s = r.s;
  const bool dense = flags & RV_DENSE;
  const bool force = flags & RV_FORCE_MASKS;
  const long long ld3 = 3LL * D;
  r.chk(launch_zero_words(ctx->reuse_ctr, 128, s), "zero reuse counters");
  r.begin(K_PATCH,-1,-1);
  r.chk(launch_patch_to_bf16(patches, ctx->patches_bf16, (long long)n * N, ctx->pp, ctx->KP, s), "patch_to_bf16");
  {
    Epi e;
    e.out = ctx->X[0];
    e.out_ld = D;
    e.row_div = N;
    e.row_add = 1;
    r.begin(K_PE,-1,-1);
    r.chk(gemm_launch(ctx->pe, nullptr, n * N, n * N, e, s), "gemm_pe");
  }
  // embed_finish also writes the uniform t of the first decision into ctx->pclsh (= P[1])
  r.begin(K_EMBED,-1,-1);
  r.chk(launch_embed_finish(ctx->X[0], 0, ctx->cls, ctx->pos, ctx->lnpre_g, ctx->lnpre_b, ctx->pclsh, n, T, D, N, H, s),
        "embed_finish");
  float* P[2] = {ctx->pcl2, ctx->pclsh};       // attention of layer l writes P[l & 1]
  int* KS[2] = {ctx->kvsrc, ctx->kvsrc2};      // source rows of layer l's q|k|v: KS[l & 1]
  // layer-0 chain (not gated): QKV_1 of every token, per wave, into QKVc[0]
  for (int wi = 0; wi < (int)ctx->waves.size(); ++wi) {
    const Wave& wv = ctx->waves[wi];
    const int rows = wv.n_w * T;
    const int* wr = ctx->wrows + (size_t)wv.off * T;
    r.begin(K_GATHER,0,wi);
    r.chk(launch_gather_ln(ctx->X[0], 0, wr, nullptr, rows, rows, ctx->lw[0].ln1_g, ctx->lw[0].ln1_b, ctx->A, D, s),
          "gather_ln1");
    Epi e;
    e.bias = ctx->lw[0].bqkv;
    e.out = ctx->QKVc[0] + 2 * D;   // q columns -> cache columns [2D, 3D)
    e.out_rows = wr;
    e.out_ld = ld3;
    e.out_bf16 = 1;
    e.split = D;
    e.out2 = ctx->QKVc[0];          // k | v -> cache columns [0, 2D)
    e.out2_rows = wr;
    e.out2_ld = ld3;
    e.out2_bf16 = 1;
    r.begin(K_QKV,0,wi);
    r.chk(gemm_launch(ctx->g_qkv[0], nullptr, rows, rows, e, s), "gemm_qkv");
  }
  for (int l = 0; l < L; ++l) {
    const LayerW& w = ctx->lw[l];
    float* Xin = ctx->X[l & 1];
    float* Xout = ctx->X[(l + 1) & 1];
    bf16* Qc = ctx->QKVc[l & 1];
    bf16* Qn = ctx->QKVc[(l + 1) & 1];
    for (int wi = 0; wi < (int)ctx->waves.size(); ++wi) {
      const Wave& wv = ctx->waves[wi];
      const int n_w = wv.n_w;
      const int rows = n_w * T;
      const int* wd = ctx->wdesc + (size_t)wv.off * 4;
      const int* wr = ctx->wrows + (size_t)wv.off * T;
      const int maxC = rows;
      // dense attention of every token over all keys of its frame
      r.begin(K_ATTN,l,wi);
      float* pcl_chain = (!dense && l + 1 < L) ? P[l & 1] : nullptr;
      if (!(flags & RV_ATTN_SYNC) && attn_tcg_supported(T, D, H))   // tcgen05: q from the cache via the table
        r.chk(launch_attention_tcg(nullptr, Qc, ld3, 2 * D, 1, Qc, ld3, KS[l & 1], ctx->att, wd, ctx->qoffT, pcl_chain, n_w, T, D,
                                   H, s),
              "attention");
      else
        r.chk(launch_attention(nullptr, Qc, KS[l & 1], ctx->att, wd, ctx->qoffT, pcl_chain, n_w, T, D, H, s, ld3, 1),
              "attention");
      // W_o + residual for every token: x'_l (the chain input) into the XP cache
      {
        Epi e;
        e.bias = w.bo;
        e.resid = Xin;
        e.resid_rows = wr;
        e.resid_ld = D;
        e.out = ctx->XP;
        e.out_rows = wr;
        e.out_ld = D;
        r.begin(K_WO,l,wi);
        r.chk(gemm_launch(ctx->g_wo[l], nullptr, rows, rows, e, s), "gemm_wo");
      }
      // decision on x' (Eq. 1-4), t = the previous layer's CLS attention
      r.begin(K_SCORE,l,wi);
      r.chk(launch_score(ctx->XP, 0, T, D, N, L, l, n_w, wd, P[(l + 1) & 1], H, codec, force ? masks : nullptr,
                         ctx->gates_loaded ? w.gate : nullptr, ctx->Hg, dense ? 1 : 0, masks, scores, ctx->wmask,
                         ctx->wprov, ctx->cntR, ctx->dfull, s),
            "score");
      // filtration; the source-row table written here serves layer l+1's q|k|v
      r.begin(K_COMPACT,l,wi);
      r.chk(launch_compact(n_w, T, wd, ctx->wmask, ctx->wprov, ctx->cntR, ctx->idxC, ctx->idxR, ctx->provrow,
                           ctx->qoff, ctx->counts, KS[(l + 1) & 1], ctx->reuse_ctr + l,
                           ctx->count_log + ((size_t)l * ctx->waves.size() + wi) * 2, ctx->rpos,
                           (ctx->fused_restore && !(flags & RV_RESTORE_GEMMS)) ? ctx->rloc : nullptr, s),
            "compact");
      const int* MC = ctx->counts;
      // chain FFN_l on C: LN2(x') -> FC1 -> FC2 + x', scattered to X_l rows
      r.begin(K_LN2,l,wi);
      r.chk(launch_gather_ln(ctx->XP, 0, ctx->idxC, MC, 0, maxC, w.ln2_g, w.ln2_b, ctx->A, D, s), "ln2");
      {
        Epi e;
        e.bias = w.b1;
        e.act = 1;
        e.out = ctx->h;
        e.out_ld = F;
        e.out_bf16 = 1;
        r.begin(K_FC1,l,wi);
        r.chk(gemm_launch(ctx->g_fc1[l], MC, 0, maxC, e, s), "gemm_fc1");
      }
      {
        Epi e;
        e.bias = w.b2;
        e.resid = ctx->XP;
        e.resid_rows = ctx->idxC;
        e.resid_ld = D;
        e.out = Xout;
        e.out_rows = ctx->idxC;
        e.out_ld = D;
        r.begin(K_FC2,l,wi);
        r.chk(gemm_launch(ctx->g_fc2[l], MC, 0, maxC, e, s), "gemm_fc2");
      }
      // restoration of the block output (Delta of the chain inputs, written by the score pass):
      // the fused kernel where supported (as in the D1 path), else R1 + R2 GEMMs
      if (wv.any_ref && !dense && ctx->fused_restore && !(flags & RV_RESTORE_GEMMS)) {
        r.begin(K_RESTORE,l,wi);
        r.chk(launch_restore(ctx->tmR1[l], ctx->tmR2[l], ctx->dfull, ctx->rloc, ctx->provrow, ctx->idxR, ctx->counts + 1,
                             n_w * N, w.br1, w.br2, Xout, 0, D, s),
              "restore");
      } else if (wv.any_ref && !dense) {
        Epi e1;
        e1.bias = w.br1;
        e1.act = 1;
        e1.out = ctx->hr;
        e1.out_ld = Hr;
        e1.out_bf16 = 1;
        e1.out_rows = ctx->rpos;
        r.begin(K_R1,l,wi);
        r.chk(gemm_launch(ctx->g_r1[l], nullptr, rows, rows, e1, s), "gemm_r1");
        Epi e2;
        e2.bias = w.br2;
        e2.resid = Xout;
        e2.resid_rows = ctx->provrow;
        e2.resid_ld = D;
        e2.out = Xout;
        e2.out_rows = ctx->idxR;
        e2.out_ld = D;
        r.begin(K_R2,l,wi);
        r.chk(gemm_launch(ctx->g_r2[l], ctx->counts + 1, 0, n_w * N, e2, s), "gemm_r2");
      }
      // chain QKV_{l+1} on C (LN1 of layer l+1), scattered into the next q|k|v cache
      if (l + 1 < L) {
        const LayerW& wn = ctx->lw[l + 1];
        r.begin(K_GATHER,l + 1,wi);
        r.chk(launch_gather_ln(Xout, 0, ctx->idxC, MC, 0, maxC, wn.ln1_g, wn.ln1_b, ctx->A, D, s), "gather_ln1");
        Epi e;
        e.bias = wn.bqkv;
        e.out = Qn + 2 * D;
        e.out_rows = ctx->idxC;
        e.out_ld = ld3;
        e.out_bf16 = 1;
        e.split = D;
        e.out2 = Qn;
        e.out2_rows = ctx->idxC;
        e.out2_ld = ld3;
        e.out2_bf16 = 1;
        r.begin(K_QKV,l + 1,wi);
        r.chk(gemm_launch(ctx->g_qkv[l + 1], MC, 0, maxC, e, s), "gemm_qkv");
      }
    }
  }
  r.begin(K_LNPOST,-1,-1);
  r.chk(launch_ln_post(ctx->X[L & 1], 0, ctx->lnpost_g, ctx->lnpost_b, emb, n, T, D, s), "ln_post");
}

rv_status ensure_chain_buffers(rv_ctx* ctx, int n) {
  if (n <= ctx->chain_cap) return RV_OK;
  const long long T = ctx->T, D = ctx->D;
  auto& B = ctx->ballocs;
  rv_status s;
#define AL(ptr, cnt) if ((s = dalloc(ctx, B, &ptr, (size_t)(cnt)))) return s
  AL(ctx->QKVc[0], n * T * 3 * D);
  AL(ctx->QKVc[1], n * T * 3 * D);
  AL(ctx->XP, n * T * D);
  AL(ctx->kvsrc2, n * T);
  AL(ctx->pcl2, (long long)n * ctx->H * ctx->N);
  AL(ctx->wrows, n * T);
  AL(ctx->qoffT, n + 1);
#undef AL
  ctx->chain_cap = n;
  if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; ctx->gkey.clear(); }
  return RV_OK;
}

}  // namespace

// ====================================================================== C-ABI
extern "C" {

const char* rv_status_string(rv_status s) {
  switch (s) {
    case RV_OK: return "RV_OK";
    case RV_ECONFIG: return "RV_ECONFIG";
    case RV_ESHAPE: return "RV_ESHAPE";
    case RV_EPLAN: return "RV_EPLAN";
    case RV_ECACHE: return "RV_ECACHE";
    case RV_ECONTRACT: return "RV_ECONTRACT";
    case RV_ECUDA: return "RV_ECUDA";
    case RV_ENOMEM: return "RV_ENOMEM";
    case RV_EBUSY: return "RV_EBUSY";
  }
  return "RV_UNKNOWN";
}

const char* rv_last_error(const rv_ctx* ctx) { return ctx ? ctx->err.c_str() : g_create_err.c_str(); }

size_t rv_vit_blob_floats(const rv_config* cfg) {
  char why[128];
  return cfg_valid(cfg, why, sizeof why) ? vit_floats(cfg) : 0;
}
size_t rv_gate_blob_floats(const rv_config* cfg) {
  char why[128];
  return cfg_valid(cfg, why, sizeof why) ? gate_floats(cfg) : 0;
}

rv_status rv_plan_gop(int32_t n, int32_t refresh, int32_t reorder, rv_plan* out) {
  rv_ctx* ctx = nullptr;
  if (!out || !out->type || !out->past || !out->future || !out->order) return fail(ctx, RV_ECONTRACT, "rv_plan_gop: null output");
  if (n < 1) return fail(ctx, RV_ECONFIG, "rv_plan_gop: n must be >= 1");
  if (refresh < 4 || refresh % 4) return fail(ctx, RV_ECONFIG, "rv_plan_gop: refresh must be a multiple of 4 (S:310)");
  out->n = n;
  for (int i = 0; i < n; ++i) { out->type[i] = RV_I; out->past[i] = -1; out->future[i] = -1; }
  int k = 0;
  if (!reorder) {   // low-latency mode: each frame references its predecessor
    for (int i = 0; i < n; ++i) {
      if (i % refresh) { out->type[i] = RV_P; out->past[i] = i - 1; }
      out->order[k++] = i;
    }
    return RV_OK;
  }
  out->order[k++] = 0;   // I
  for (int a0 = 0; a0 + 1 < n; a0 += 4) {   // 5-frame unit [a0 .. a0+4]
    const int a1 = a0 + 4;
    if (a1 < n) {
      if (a1 % refresh) { out->type[a1] = RV_P; out->past[a1] = a0; }
      out->order[k++] = a1;
    }
    if (a0 + 2 < n) {
      out->type[a0 + 2] = RV_B2;
      out->past[a0 + 2] = a0;
      out->future[a0 + 2] = a1 < n ? a1 : -1;
      out->order[k++] = a0 + 2;
    }
    for (int b : {a0 + 1, a0 + 3}) {
      if (b < n) {
        out->type[b] = RV_B1;
        out->past[b] = b - 1;
        out->future[b] = b + 1 < n ? b + 1 : -1;
        out->order[k++] = b;
      }
    }
  }
  return RV_OK;
}

rv_status rv_plan_check(const rv_plan* plan) { return check_plan(nullptr, plan, nullptr); }

rv_status rv_create(const rv_config* cfg, int device, rv_ctx** out) {
  rv_ctx* ctx = nullptr;
  if (!out) return fail(ctx, RV_ECONTRACT, "rv_create: out is NULL");
  *out = nullptr;
  char why[160];
  if (!cfg_valid(cfg, why, sizeof why)) return fail(ctx, RV_ECONFIG, "rv_create: %s", why);
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return fail(ctx, RV_ECUDA, "rv_create: no CUDA device (%s); there is no CPU fallback",
                e != cudaSuccess ? cudaGetErrorString(e) : "0 devices");
  }
  if (device < 0 || device >= ndev) return fail(ctx, RV_ECUDA, "rv_create: device %d out of range (%d)", device, ndev);
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10)
    return fail(ctx, RV_ECUDA, "rv_create: device %d is sm_%d%d; this library is built for sm_100a only", device,
                prop.major, prop.minor);
  if (cudaSetDevice(device) != cudaSuccess) return fail(ctx, RV_ECUDA, "rv_create: cudaSetDevice failed");
  ctx = new rv_ctx();
  ctx->cfg = *cfg;
  ctx->device = device;
  ctx->L = cfg->layers;
  ctx->D = cfg->dim;
  ctx->H = cfg->heads;
  ctx->dh = cfg->dim / cfg->heads;
  ctx->N = (cfg->img / cfg->patch) * (cfg->img / cfg->patch);
  ctx->T = ctx->N + 1;
  ctx->pp = 3 * cfg->patch * cfg->patch;
  ctx->KP = (ctx->pp + 63) / 64 * 64;
  ctx->F = cfg->ffn;
  ctx->Hr = cfg->hidden_r;
  ctx->Hg = cfg->hidden_g;
  for (auto& ev : ctx->ev) cudaEventCreate(&ev);
  cudaStreamCreateWithFlags(&ctx->own_stream, cudaStreamNonBlocking);
  *out = ctx;
  return RV_OK;
}

rv_status rv_load_vit(rv_ctx* ctx, const float* blob, size_t n_floats) {
  if (!ctx) return RV_ECONTRACT;
  if (!blob) return fail(ctx, RV_ECONTRACT, "rv_load_vit: blob is NULL");
  if (ctx->inflight) return fail(ctx, RV_EBUSY, "rv_load_vit: embed in flight");
  const size_t want = vit_floats(&ctx->cfg);
  if (n_floats != want) return fail(ctx, RV_ESHAPE, "rv_load_vit: blob has %zu floats, config needs %zu", n_floats, want);
  CK(cudaSetDevice(ctx->device));
  const int D = ctx->D, T = ctx->T, F = ctx->F, pp = ctx->pp;
  // weights of a previous load stay allocated until destroy (gates share the list)
  std::vector<void*>& W = ctx->wallocs;
  const float* p = blob;
  rv_status s;
  if ((s = upload_T(ctx, W, &ctx->W_pe, p, pp, D, ctx->KP))) return s;
  p += (size_t)pp * D;
  if ((s = upload_f(ctx, W, &ctx->cls, p, D))) return s;
  p += D;
  if ((s = upload_f(ctx, W, &ctx->pos, p, (size_t)T * D))) return s;
  p += (size_t)T * D;
  if ((s = upload_f(ctx, W, &ctx->lnpre_g, p, D))) return s;
  p += D;
  if ((s = upload_f(ctx, W, &ctx->lnpre_b, p, D))) return s;
  p += D;
  ctx->lw.resize(ctx->L);
  for (int l = 0; l < ctx->L; ++l) {
    LayerW& w = ctx->lw[l];
    if ((s = upload_f(ctx, W, &w.ln1_g, p, D))) return s; p += D;
    if ((s = upload_f(ctx, W, &w.ln1_b, p, D))) return s; p += D;
    {
      // K/V cache layout (a7): the QKV output columns q | k | v (head h = columns h*dh..) are
      // reordered at load to q | (k_0 v_0) (k_1 v_1) ..., so one head's key and value of a token
      // are 2*dh contiguous bf16 (256 B at d_h = 64): the attention gathers one 256 B segment per
      // (token, head) instead of two 128 B rows 2 KB apart (tools/gather_rate.cu: 4.9 -> 6.1 TB/s)
      std::vector<float> wq((size_t)D * 3 * D), bq(3 * D);
      const int dh = ctx->dh;
      auto col = [&](int j) {
        if (j < D) return j;
        const int kv = (j - D) / D, h = ((j - D) % D) / dh, c = (j - D) % dh;
        return D + h * 2 * dh + kv * dh + c;
      };
      for (int j = 0; j < 3 * D; ++j) {
        const int nj = col(j);
        bq[nj] = p[(size_t)D * 3 * D + j];
        for (int i = 0; i < D; ++i) wq[(size_t)i * 3 * D + nj] = p[(size_t)i * 3 * D + j];
      }
      if ((s = upload_T(ctx, W, &w.Wqkv, wq.data(), D, 3 * D, D))) return s; p += (size_t)D * 3 * D;
      if ((s = upload_f(ctx, W, &w.bqkv, bq.data(), 3 * D))) return s; p += 3 * D;
    }
    if ((s = upload_T(ctx, W, &w.Wo, p, D, D, D))) return s; p += (size_t)D * D;
    if ((s = upload_f(ctx, W, &w.bo, p, D))) return s; p += D;
    if ((s = upload_f(ctx, W, &w.ln2_g, p, D))) return s; p += D;
    if ((s = upload_f(ctx, W, &w.ln2_b, p, D))) return s; p += D;
    if ((s = upload_T(ctx, W, &w.W1, p, D, F, D))) return s; p += (size_t)D * F;
    if ((s = upload_f(ctx, W, &w.b1, p, F))) return s; p += F;
    if ((s = upload_T(ctx, W, &w.W2, p, F, D, F))) return s; p += (size_t)F * D;
    if ((s = upload_f(ctx, W, &w.b2, p, D))) return s; p += D;
  }
  if ((s = upload_f(ctx, W, &ctx->lnpost_g, p, D))) return s;
  p += D;
  if ((s = upload_f(ctx, W, &ctx->lnpost_b, p, D))) return s;
  p += D;
  ctx->vit_loaded = true;
  release_buffers(ctx);   // the GEMM plans encode the weight addresses: rebuilt at the next embed
  return RV_OK;
}

rv_status rv_load_gates(rv_ctx* ctx, const float* blob, size_t n_floats) {
  if (!ctx) return RV_ECONTRACT;
  if (!blob) return fail(ctx, RV_ECONTRACT, "rv_load_gates: blob is NULL");
  if (!ctx->vit_loaded) return fail(ctx, RV_ECONTRACT, "rv_load_gates: load the ViT weights first");
  if (ctx->inflight) return fail(ctx, RV_EBUSY, "rv_load_gates: embed in flight");
  const size_t want = gate_floats(&ctx->cfg);
  if (n_floats != want) return fail(ctx, RV_ESHAPE, "rv_load_gates: blob has %zu floats, config needs %zu", n_floats, want);
  CK(cudaSetDevice(ctx->device));
  const int D = ctx->D, Hr = ctx->Hr, Hg = ctx->Hg;
  std::vector<void*>& W = ctx->wallocs;
  const float* p = blob;
  rv_status s;
  for (int l = 0; l < ctx->L; ++l) {
    LayerW& w = ctx->lw[l];
    const size_t ng = 7 * Hg + Hg + Hg + 1;
    if ((s = upload_f(ctx, W, &w.gate, p, ng))) return s; p += ng;
    if ((s = upload_T(ctx, W, &w.Wr1, p, D, Hr, D))) return s; p += (size_t)D * Hr;
    if ((s = upload_f(ctx, W, &w.br1, p, Hr))) return s; p += Hr;
    if ((s = upload_T(ctx, W, &w.Wr2, p, Hr, D, Hr))) return s; p += (size_t)Hr * D;
    if ((s = upload_f(ctx, W, &w.br2, p, D))) return s; p += D;
  }
  ctx->gates_loaded = true;
  release_buffers(ctx);
  return RV_OK;
}

rv_status rv_embed(rv_ctx* ctx, const float* patches, const float* codec, const rv_plan* plan, uint32_t flags,
                   void* cuda_stream, float* emb, uint8_t* masks, float* scores) {
  if (!ctx) return RV_ECONTRACT;
#ifdef RV_HOST_TIMING   // experiment builds only: host time of rv_embed's phases on stderr
  const auto ht0 = std::chrono::steady_clock::now();
  auto hms = [&]() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - ht0).count(); };
#endif
  if (ctx->inflight) return fail(ctx, RV_EBUSY, "rv_embed: an embed is already in flight");
  if (!ctx->vit_loaded) return fail(ctx, RV_ECONTRACT, "rv_embed: ViT weights not loaded");
  const bool dense = flags & RV_DENSE;
  if (!dense && !ctx->gates_loaded) return fail(ctx, RV_ECONTRACT, "rv_embed: gates not loaded (or pass RV_DENSE)");
  if (!patches || !codec || !emb) return fail(ctx, RV_ECONTRACT, "rv_embed: patches, codec and emb are required");
  if ((flags & RV_FORCE_MASKS) && !masks) return fail(ctx, RV_ECONTRACT, "rv_embed: RV_FORCE_MASKS needs masks");
  std::vector<int> lev;
  rv_status st = check_plan(ctx, plan, &lev);
  if (st) return st;
  CK(cudaSetDevice(ctx->device));
  const int n = plan->n, T = ctx->T, N = ctx->N, L = ctx->L, D = ctx->D;
  // ---- level-waves: frames of equal level in computation order; dense = one level.
  // Large levels are split into waves of at most kMaxWave frames (bounds the wave buffers).
  const int kMaxWave = (flags & RV_WAVE_FRAME) ? 1 : 1536;
  std::vector<std::vector<int>> levels;
  for (int k = 0; k < n; ++k) {
    const int f = plan->order[k];
    const int lv = dense ? 0 : lev[f];
    if ((int)levels.size() <= lv) levels.resize(lv + 1);
    levels[lv].push_back(f);
  }
  ctx->waves.clear();
  ctx->wdesc_host.clear();
  int max_w = 0, nonI = 0;
  bool any_ref_all = false;
  for (auto& lvf : levels) {
    for (size_t b = 0; b < lvf.size(); b += kMaxWave) {
      Wave wv;
      wv.off = (int)ctx->wdesc_host.size() / 4;
      wv.n_w = (int)std::min<size_t>(kMaxWave, lvf.size() - b);
      wv.any_ref = false;
      for (int j = 0; j < wv.n_w; ++j) {
        const int f = lvf[b + j];
        const int t = dense ? RV_I : plan->type[f];
        ctx->wdesc_host.push_back(f);
        ctx->wdesc_host.push_back(dense ? -1 : plan->past[f]);
        ctx->wdesc_host.push_back(dense ? -1 : plan->future[f]);
        ctx->wdesc_host.push_back(t);
        if (t != RV_I) { wv.any_ref = true; }
      }
      any_ref_all |= wv.any_ref;
      max_w = std::max(max_w, wv.n_w);
      ctx->waves.push_back(wv);
    }
  }
  for (int f = 0; f < n; ++f) nonI += (!dense && plan->type[f] != RV_I);
  const int total_desc = (int)ctx->wdesc_host.size() / 4;
  if (total_desc != n) return fail(ctx, RV_EPLAN, "rv_embed: internal wave bookkeeping mismatch");
  const bool keepall = flags & RV_KEEP_ALL_CACHE;
  if (keepall && (flags & RV_CHAIN)) return fail(ctx, RV_ECONTRACT, "rv_embed: RV_KEEP_ALL_CACHE is a D1-path ablation");
  if ((flags & RV_X_BF16) && (flags & RV_CHAIN))
    return fail(ctx, RV_ECONTRACT, "rv_embed: RV_X_BF16 is implemented for the D1 path only");
  if ((st = ensure_buffers(ctx, n, (long long)max_w * T, any_ref_all ? (long long)max_w * N : 0, max_w, keepall)))
    return st;
  // Wavefront schedule when the level waves are too small to fill the GPU and the
  // rings fit: the largest R <= min(L + 1, waves + 1) whose extra bytes stay within half of the
  // free device memory (the rest is left to the caller, e.g. a second pipelined context).
  // Profiled, ablation and chain embeds keep the serial level order.
  ctx->wf_R = 0;
  // the ring size is re-decided only when the wave structure or the buffers changed: the free
  // memory query behind it occasionally stalls the host for milliseconds (measured up to 7 ms on
  // a 2.5 ms clip), so repeated embeds of the same shape reuse the previous decision
  std::vector<long long> wf_sig = {(long long)ctx->n_cap, ctx->capC, ctx->capR};
  for (const Wave& w : ctx->waves) wf_sig.push_back(w.n_w * 2 + (w.any_ref ? 1 : 0));
  const bool wf_want = !(flags & (RV_SERIAL_WAVES | RV_PROFILE | RV_KEEP_ALL_CACHE | RV_CHAIN | RV_WAVE_FRAME)) &&
                       ctx->waves.size() >= 2 && max_w <= kWavefrontMaxWave;
  if (wf_want && wf_sig == ctx->wf_sig && ctx->wf_R_last >= 3 && ensure_wavefront(ctx, ctx->wf_R_last) == RV_OK) {
    ctx->wf_R = ctx->wf_R_last;
  } else if (wf_want) {
    size_t fr = 0, tot = 0;
#ifdef RV_HOST_TIMING
    const double ht_m0 = hms();
#endif
    CK(cudaMemGetInfo(&fr, &tot));
#ifdef RV_HOST_TIMING
    fprintf(stderr, "  memgetinfo %.3f ms (at %.3f)\n", hms() - ht_m0, ht_m0);
#endif
    const unsigned long long avail = fr + ctx->wf_bytes, reserve = 4ull << 30;
    const unsigned long long budget = avail > reserve ? (avail - reserve) / 2 : 0;
    int R = std::min(L + 1, (int)ctx->waves.size() + 1);
    while (R >= 3 && wavefront_bytes(ctx, ctx->n_cap, R, ctx->waves) > budget) --R;
    if (R >= 3) {
      if (ensure_wavefront(ctx, R) == RV_OK) {
        ctx->wf_R = R;
      } else {   // could not allocate the rings: the serial schedule needs nothing more
        release_wavefront(ctx);
        ctx->err.clear();
      }
    }
    ctx->wf_sig = wf_sig;
    ctx->wf_R_last = ctx->wf_R;
  }
  if (flags & RV_CHAIN) {
    if ((st = ensure_chain_buffers(ctx, n))) return st;
    const int nd = (int)ctx->wdesc_host.size() / 4;
    ctx->wrows_host.resize((size_t)nd * T);
    for (int k = 0; k < nd; ++k)
      for (int i = 0; i < T; ++i) ctx->wrows_host[(size_t)k * T + i] = ctx->wdesc_host[(size_t)k * 4] * T + i;
    ctx->qoffT_host.resize((size_t)n + 1);
    for (int w = 0; w <= n; ++w) ctx->qoffT_host[w] = w * T;
  }
  {
    const int need = L * (int)ctx->waves.size() * 2;
    if (need > ctx->count_log_cap) {
      if (ctx->count_log) cudaFree(ctx->count_log);
      ctx->count_log = nullptr;
      CK(cudaMalloc(&ctx->count_log, need * sizeof(int)));
      ctx->count_log_cap = need;
      if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; ctx->gkey.clear(); }
    }
  }
  ctx->prof_valid = false;
  cudaStream_t s = cuda_stream ? (cudaStream_t)cuda_stream : nullptr;
  const bool devp = flags & RV_DEVICE_PTRS;
  if (!devp && (st = ensure_host_buffers(ctx, n, scores != nullptr))) return st;
  const float* d_patches = devp ? patches : ctx->in_patches;
  const float* d_codec = devp ? codec : ctx->in_codec;
  float* d_emb = devp ? emb : ctx->out_emb;
  // masks / scores are written only when requested (the kernels skip null outputs)
  uint8_t* d_masks = devp ? masks : (masks ? ctx->out_masks : nullptr);
  float* d_scores = devp ? scores : (scores ? ctx->out_scores : nullptr);
  // Graph capture cannot run on the legacy NULL stream: work on the context's own stream,
  // ordered after / before the caller's stream with events.
  cudaStream_t ws = s ? s : ctx->own_stream;
  if (!s) {
    CK(cudaEventRecord(ctx->ev[3], 0));
    CK(cudaStreamWaitEvent(ws, ctx->ev[3], 0));
  }
  CK(cudaEventRecord(ctx->ev[0], ws));
#ifdef RV_HOST_TIMING
  const double ht_c0 = hms();
#endif
  // the wave descriptors change only with the plan: re-uploading them every call put a small
  // host-to-device copy into the copy-engine queue behind whatever the caller streams in
  // concurrently (the next step's inputs), stalling this embed until that copy finished
  if (ctx->wdesc_dev_copy != ctx->wdesc_host) {
    CK(cudaMemcpyAsync(ctx->wdesc, ctx->wdesc_host.data(), ctx->wdesc_host.size() * sizeof(int),
                       cudaMemcpyHostToDevice, ws));
    ctx->wdesc_dev_copy = ctx->wdesc_host;
  }
#ifdef RV_HOST_TIMING
  fprintf(stderr, "  wdesc copy %.3f ms (at %.3f)\n", hms() - ht_c0, ht_c0);
#endif
  if (flags & RV_CHAIN) {   // wave row map, query offsets, identity source rows of layer 1's q|k|v
    // (the maps follow the plan and are uploaded when it or the buffers change; the identity
    // rows are rewritten every call by a kernel, since the embed overwrites them)
    if (ctx->chain_dev_copy != ctx->wdesc_host || ctx->chain_dev_ptr != ctx->wrows) {
      CK(cudaMemcpyAsync(ctx->wrows, ctx->wrows_host.data(), ctx->wrows_host.size() * sizeof(int),
                         cudaMemcpyHostToDevice, ws));
      CK(cudaMemcpyAsync(ctx->qoffT, ctx->qoffT_host.data(), ctx->qoffT_host.size() * sizeof(int),
                         cudaMemcpyHostToDevice, ws));
      ctx->chain_dev_copy = ctx->wdesc_host;
      ctx->chain_dev_ptr = ctx->wrows;
    }
    CK(launch_iota(ctx->kvsrc, (long long)n * T, ws));
  }
  if (!devp) {
    CK(cudaMemcpyAsync(ctx->in_patches, patches, (size_t)n * N * ctx->pp * 4, cudaMemcpyHostToDevice, ws));
    CK(cudaMemcpyAsync(ctx->in_codec, codec, (size_t)n * N * 4, cudaMemcpyHostToDevice, ws));
    if (flags & RV_FORCE_MASKS)
      CK(cudaMemcpyAsync(ctx->out_masks, masks, (size_t)n * L * N, cudaMemcpyHostToDevice, ws));
  }
  CK(cudaEventRecord(ctx->ev[1], ws));
#ifdef RV_HOST_TIMING
  const double ht_pre = hms();
  bool ht_cap = false;
#endif
  // ---- compute: cached CUDA graph keyed on everything the recorded sequence depends on
  std::vector<long long> key = {(long long)n, (long long)(flags & ~RV_NO_GRAPH), (long long)(intptr_t)d_patches,
                                (long long)(intptr_t)d_codec, (long long)(intptr_t)d_emb,
                                (long long)(intptr_t)d_masks, (long long)(intptr_t)d_scores,
                                (long long)(intptr_t)ws, ctx->capC, ctx->capR, (long long)ctx->wf_R};
  for (int v : ctx->wdesc_host) key.push_back(v);
  Rec rec{ctx, ws};
  rec.prof = (flags & RV_PROFILE) != 0;
  if (flags & RV_NO_GRAPH) {
    ctx->prof_used = 0;
    ctx->prof_recs.clear();
    (flags & RV_CHAIN ? record_embed_chain : record_embed)(ctx, rec, n, flags, d_patches, d_codec, d_emb, d_masks,
                                                          d_scores);
    if (rec.err != cudaSuccess) return fail(ctx, RV_ECUDA, "launch %s: %s", rec.where, cudaGetErrorString(rec.err));
  } else {
    if (!ctx->gexec || key != ctx->gkey) {
#ifdef RV_HOST_TIMING
      ht_cap = true;
#endif
      if (ctx->gexec) { cudaGraphExecDestroy(ctx->gexec); ctx->gexec = nullptr; }
      cudaGraph_t g = nullptr;
      ctx->prof_used = 0;
      ctx->prof_recs.clear();
      CK(cudaStreamBeginCapture(ws, cudaStreamCaptureModeThreadLocal));
      (flags & RV_CHAIN ? record_embed_chain : record_embed)(ctx, rec, n, flags, d_patches, d_codec, d_emb, d_masks,
                                                          d_scores);
      cudaError_t ce = cudaStreamEndCapture(ws, &g);
      if (rec.err != cudaSuccess) {
        if (g) cudaGraphDestroy(g);
        return fail(ctx, RV_ECUDA, "capture %s: %s", rec.where, cudaGetErrorString(rec.err));
      }
      CK(ce);
      cudaError_t ie = cudaGraphInstantiate(&ctx->gexec, g, 0);
      cudaGraphDestroy(g);
      CK(ie);
      ctx->gkey = key;
      ctx->cur_launches = rec.launches;
    }
#ifdef RV_HOST_TIMING
    const double ht_l0 = hms();
#endif
    CK(cudaGraphLaunch(ctx->gexec, ws));
#ifdef RV_HOST_TIMING
    fprintf(stderr, "rv_embed host: pre %.3f ms, capture %d, to launch %.3f, launch %.3f ms\n", ht_pre, (int)ht_cap,
            ht_l0, hms() - ht_l0);
#endif
    rec.launches = ctx->cur_launches;
  }
  CK(cudaEventRecord(ctx->ev[2], ws));
  if (!devp) {
    CK(cudaMemcpyAsync(emb, ctx->out_emb, (size_t)n * D * 4, cudaMemcpyDeviceToHost, ws));
    if (masks && !(flags & RV_FORCE_MASKS))
      CK(cudaMemcpyAsync(masks, ctx->out_masks, (size_t)n * L * N, cudaMemcpyDeviceToHost, ws));
    if (scores) CK(cudaMemcpyAsync(scores, ctx->out_scores, (size_t)n * L * N * 4, cudaMemcpyDeviceToHost, ws));
  }
  CK(cudaEventRecord(ctx->ev[3], ws));
  if (!s) CK(cudaStreamWaitEvent(0, ctx->ev[3], 0));
  ctx->inflight = true;
  ctx->cur_n = n;
  ctx->cur_nonI = nonI;
  ctx->cur_flags = flags;
  ctx->cur_levels = (int)levels.size();
  ctx->cur_launches = rec.launches;
  ctx->cur_stream = ws;
  ctx->prof_valid = rec.prof;
  return RV_OK;
}

rv_status rv_wait(rv_ctx* ctx, rv_stats* stats) {
  if (!ctx) return RV_ECONTRACT;
  if (!ctx->inflight) return fail(ctx, RV_ECONTRACT, "rv_wait: no embed in flight");
  ctx->inflight = false;
  CK(cudaSetDevice(ctx->device));
  CK(cudaEventSynchronize(ctx->ev[3]));
  CK(cudaGetLastError());
  if (!stats) return RV_OK;
  memset(stats, 0, sizeof *stats);
  const int L = ctx->L, n = ctx->cur_n, T = ctx->T, N = ctx->N;
  unsigned long long ctr[64] = {0};
  CK(cudaMemcpy(ctr, ctx->reuse_ctr, L * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
  const double D = ctx->D, F = ctx->F, Hr = ctx->Hr, pp = ctx->pp;
  const double per_c = 2 * D * 3 * D + 2 * D * D + 4 * D * F + 4 * T * D;
  const double per_r = 4 * D * Hr;
  const bool chain = ctx->cur_flags & RV_CHAIN;
  double reused = 0, flops = 2.0 * n * N * pp * D, bytes = 0;
  if (chain) flops += (double)n * T * 2 * D * 3 * D;   // QKV_1 of every token (ungated layer-0 chain)
  for (int l = 0; l < L; ++l) {
    const double r = (double)ctr[l];
    const double c = (double)n * T - r;
    reused += r;
    if (chain)   // attention + W_o dense; FFN_l (+ QKV_{l+1}) on C; restoration on R
      flops += (double)n * T * (4 * T * D + 2 * D * D) + c * (4 * D * F + (l + 1 < L ? 6 * D * D : 0.0)) + r * per_r;
    else
      flops += c * per_c + r * per_r;
    // algorithmic bytes: 60 D per recomputed token-layer, 18 D per reused one;
    // RV_X_BF16 halves their X-row parts (16 D and 12 D): 52 D and 12 D
    if (ctx->cur_flags & RV_X_BF16) bytes += c * 52.0 * D + r * 12.0 * D;
    else bytes += c * 60.0 * D + r * 18.0 * D;
    stats->reuse_by_layer[l] = ctx->cur_nonI ? (float)(r / ((double)ctx->cur_nonI * N)) : 0.f;
  }
  stats->reuse_nonI = ctx->cur_nonI ? reused / ((double)ctx->cur_nonI * L * N) : 0.0;
  stats->reuse_all = reused / ((double)n * L * T);
  stats->flops_exec = flops;
  stats->flops_dense = 2.0 * n * N * pp * D + (double)n * L * T * per_c;
  stats->bytes_alg = bytes;
  const bool wf = ctx->wf_R >= 3;                  // wavefront rings and per-wave scratch in use
  stats->peak_cache_bytes = ctx->cache_bytes + (wf ? ctx->wf_cache_bytes : 0);   // X + K/V cache of the mode used
  stats->device_bytes = ctx->alloc_bytes + (wf ? ctx->wf_bytes : 0);            // every per-embed device buffer
  stats->wave_ring = ctx->wf_R;
  stats->keepall_cache_bytes = (uint64_t)((double)n * T * ((L + 1) * D * 4 + L * 2 * D * 2));
  float ms = 0, msc = 0;
  cudaEventElapsedTime(&ms, ctx->ev[0], ctx->ev[3]);
  cudaEventElapsedTime(&msc, ctx->ev[1], ctx->ev[2]);
  stats->ms_total = ms;
  stats->ms_compute = msc;
  stats->n_levels = ctx->cur_levels;
  stats->n_launches = ctx->cur_launches;
  return RV_OK;
}

void rv_destroy(rv_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  if (ctx->inflight) cudaEventSynchronize(ctx->ev[3]);
  if (ctx->gexec) cudaGraphExecDestroy(ctx->gexec);
  free_list(ctx->ballocs);
  free_list(ctx->hallocs);
  free_list(ctx->hsallocs);
  free_list(ctx->wallocs);
  if (ctx->count_log) cudaFree(ctx->count_log);
  free_list(ctx->wfallocs);
  for (auto st : ctx->wstreams) cudaStreamDestroy(st);
  for (auto e : ctx->wevents) cudaEventDestroy(e);
  if (ctx->wf_fork) cudaEventDestroy(ctx->wf_fork);
  for (auto e : ctx->prof_pool) cudaEventDestroy(e);
  for (auto& ev : ctx->ev) if (ev) cudaEventDestroy(ev);
  if (ctx->own_stream) cudaStreamDestroy(ctx->own_stream);
  delete ctx;
}

int32_t rv_wave_counts(rv_ctx* ctx, int32_t* frames, int32_t* counts, int32_t max_waves) {
  if (!ctx) return RV_ECONTRACT;
  if (ctx->inflight || ctx->waves.empty())
    return fail(ctx, RV_ECONTRACT, "rv_wave_counts: no completed embed (call rv_wait first)");
  const int nwv = (int)ctx->waves.size();
  if (!frames || !counts || max_waves < nwv) return nwv;   // size query
  CK(cudaSetDevice(ctx->device));
  for (int wi = 0; wi < nwv; ++wi) frames[wi] = ctx->waves[wi].n_w;
  CK(cudaMemcpy(counts, ctx->count_log, (size_t)ctx->L * nwv * 2 * sizeof(int), cudaMemcpyDeviceToHost));
  return nwv;
}

int32_t rv_profile(rv_ctx* ctx, rv_kernel_prof* out, int32_t max_entries) {
  if (!ctx || !out) return RV_ECONTRACT;
  if (!ctx->prof_valid || ctx->inflight)
    return fail(ctx, RV_ECONTRACT, "rv_profile: no completed RV_PROFILE embed (call rv_wait first)");
  CK(cudaSetDevice(ctx->device));
  const int nwv = (int)ctx->waves.size();
  std::vector<int> log((size_t)ctx->L * nwv * 2);
  CK(cudaMemcpy(log.data(), ctx->count_log, log.size() * sizeof(int), cudaMemcpyDeviceToHost));
  const double D = ctx->D, T = ctx->T, N = ctx->N, F = ctx->F, Hr = ctx->Hr, n = ctx->cur_n;
  // per-wave host facts: frames, decision frames and the DISTINCT reference frames they read
  // (compulsory traffic: a reference shared by several frames of the wave counts once)
  std::vector<double> wdec(nwv, 0), wrefs(nwv, 0);
  std::vector<int> ref_seen((size_t)std::max(ctx->n_cap, 1), -1);
  for (int wi = 0; wi < nwv; ++wi) {
    const Wave& wv = ctx->waves[wi];
    for (int j = 0; j < wv.n_w; ++j) {
      const int* d = &ctx->wdesc_host[(size_t)(wv.off + j) * 4];
      if (d[3] == RV_I) continue;
      wdec[wi] += 1;
      for (int k = 1; k <= 2; ++k)
        if (d[k] >= 0 && d[k] < (int)ref_seen.size() && ref_seen[d[k]] != wi) {
          ref_seen[d[k]] = wi;
          wrefs[wi] += 1;
        }
    }
  }
  std::vector<rv_kernel_prof> acc(K_NCLS);
  for (int c = 0; c < K_NCLS; ++c) {
    memset(&acc[c], 0, sizeof(rv_kernel_prof));
    snprintf(acc[c].name, sizeof acc[c].name, "%s", kClsName[c]);
  }
  for (const auto& r : ctx->prof_recs) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, r.a, r.b));
    rv_kernel_prof& a = acc[r.cls];
    a.launches += 1;
    a.ms += ms;
    double MC = 0, MR = 0, nw = 0;
    if (r.l >= 0) {
      MC = log[((size_t)r.l * nwv + r.w) * 2];
      MR = log[((size_t)r.l * nwv + r.w) * 2 + 1];
      nw = ctx->waves[r.w].n_w;
      if (ctx->cur_flags & RV_CHAIN) {
        // SPEC chain variant: attention and W_o run over every token; LN1 + QKV of layer l + 1
        // (tagged l + 1) are gated by layer l's decision, layer 1's run over every token
        if (r.cls == K_ATTN || r.cls == K_WO) MC = nw * T;
        if (r.cls == K_GATHER || r.cls == K_QKV)
          MC = r.l == 0 ? nw * T : log[((size_t)(r.l - 1) * nwv + r.w) * 2];
      }
    }
    // Algorithmic FLOPs (tensor work) and HBM bytes of this launch; xs = bytes
    // per element of the residual stream X (4, or 2 with RV_X_BF16)
    const double xs = (ctx->cur_flags & RV_X_BF16) ? 2.0 : 4.0;
    switch (r.cls) {
      case K_PATCH: a.bytes += n * N * (ctx->pp * 4.0 + ctx->KP * 2.0); break;
      case K_PE: a.flops += 2.0 * n * N * ctx->pp * D; a.bytes += n * N * (ctx->KP * 2.0 + D * xs); break;
      case K_EMBED: a.bytes += n * T * D * 2.0 * xs; break;
      case K_SCORE: a.bytes += (wdec[r.w] + wrefs[r.w]) * N * D * xs + wdec[r.w] * N * 10.0 + MR * D * 2.0; break;
      case K_COMPACT: a.bytes += nw * T * 2.0 + (MC + 2 * MR) * 4.0; break;
      case K_GATHER: a.bytes += MC * (D * xs + D * 2.0 + 4.0); break;
      case K_QKV: a.flops += 2.0 * MC * 3 * D * D; a.bytes += MC * (D * 2.0 + 3 * D * 2.0) + 3 * D * D * 2.0; break;
      case K_ATTN: a.flops += 4.0 * MC * T * D; a.bytes += MC * D * 4.0 + nw * T * 2 * D * 2.0; break;
      case K_WO: a.flops += 2.0 * MC * D * D; a.bytes += MC * (D * 2.0 + D * xs + D * 4.0) + D * D * 2.0; break;
      case K_LN2: a.bytes += MC * (D * 4.0 + D * 2.0); break;
      case K_FC1: a.flops += 2.0 * MC * F * D; a.bytes += MC * (D * 2.0 + F * 2.0) + F * D * 2.0; break;
      case K_FC2: a.flops += 2.0 * MC * D * F; a.bytes += MC * (F * 2.0 + D * 4.0 + D * xs) + F * D * 2.0; break;
      case K_R1: a.flops += 2.0 * MR * Hr * D; a.bytes += MR * (D * 2.0 + Hr * 2.0) + Hr * D * 2.0; break;
      case K_R2: a.flops += 2.0 * MR * D * Hr; a.bytes += MR * (Hr * 2.0 + D * xs * 2) + Hr * D * 2.0; break;
      case K_LNPOST: a.bytes += n * D * (xs + 4.0); break;
      case K_RESTORE:   // R1 + R2 tensor work; Delta row in, provider row in, restored row out
        a.flops += 4.0 * MR * D * Hr;
        a.bytes += MR * (D * 2.0 + D * xs * 2) + 2.0 * Hr * D * 2.0;
        break;
    }
  }
  int k = 0;
  for (int c = 0; c < K_NCLS && k < max_entries; ++c)
    if (acc[c].launches) out[k++] = acc[c];
  return k;
}

// ---------------------------------------------------------------------- stage entry points
rv_status rv_stage_score(rv_ctx* ctx, int32_t layer, const float* X, int32_t n_w, const int32_t* wdesc,
                         const float* t, const float* codec, const uint8_t* force, uint8_t* masks, float* scores,
                         uint8_t* wmask, uint8_t* wprov, int32_t* cntR, void* stream) {
  if (!ctx) return RV_ECONTRACT;
  if (!ctx->gates_loaded) return fail(ctx, RV_ECONTRACT, "rv_stage_score: gates not loaded");
  if (layer < 0 || layer >= ctx->L || n_w < 0) return fail(ctx, RV_ECONTRACT, "rv_stage_score: bad layer/n_w");
  CK(cudaSetDevice(ctx->device));
  CK(launch_score(X, 0, ctx->T, ctx->D, ctx->N, ctx->L, layer, n_w, wdesc, t, 1, codec, force, ctx->lw[layer].gate,
                  ctx->Hg, 0, masks, scores, wmask, wprov, cntR, nullptr, (cudaStream_t)stream));
  return RV_OK;
}

rv_status rv_stage_compact(rv_ctx* ctx, int32_t n_w, const int32_t* wdesc, const uint8_t* wmask,
                           const uint8_t* wprov, const int32_t* cntR, int32_t* idxC, int32_t* idxR,
                           int32_t* provrow, int32_t* qoff, int32_t* counts, void* stream) {
  if (!ctx) return RV_ECONTRACT;
  CK(cudaSetDevice(ctx->device));
  CK(launch_compact(n_w, ctx->T, wdesc, wmask, wprov, cntR, idxC, idxR, provrow, qoff, counts, nullptr, nullptr, nullptr,
                    nullptr, nullptr, (cudaStream_t)stream));
  return RV_OK;
}

rv_status rv_stage_gemm(rv_ctx* ctx, int32_t M, int32_t N, int32_t K, const void* A, const void* B, const float* bias,
                        int32_t act, void* out, int32_t out_bf16, void* stream) {
  if (!ctx) return RV_ECONTRACT;
  if (M < 0 || N % 64 || K % 64 || N <= 0 || K <= 0 || !A || !B || !out)
    return fail(ctx, RV_ECONTRACT, "rv_stage_gemm: need M >= 0, N and K positive multiples of 64");
  CK(cudaSetDevice(ctx->device));
  GemmPlan p;
  char e[256];
  if (!gemm_make_plan(&p, A, std::max(M, 1), B, N, K, e, sizeof e)) return fail(ctx, RV_ECUDA, "%s", e);
  Epi ep;
  ep.bias = bias;
  ep.act = act;
  ep.out = out;
  ep.out_ld = N;
  ep.out_bf16 = out_bf16;
  CK(gemm_launch(p, nullptr, M, M, ep, (cudaStream_t)stream));
  return RV_OK;
}

rv_status rv_stage_gemm_rows(rv_ctx* ctx, int32_t M, int32_t N, int32_t K, const void* A, const void* B,
                             const float* bias, int32_t act, const float* resid, const int32_t* resid_rows,
                             int64_t resid_ld, void* out, const int32_t* out_rows, int64_t out_ld, int32_t out_bf16,
                             void* stream) {
  if (!ctx) return RV_ECONTRACT;
  if (M < 0 || N % 64 || K % 64 || N <= 0 || K <= 0 || !A || !B || !out || out_ld < N || (resid && resid_ld < N))
    return fail(ctx, RV_ECONTRACT, "rv_stage_gemm_rows: bad arguments");
  CK(cudaSetDevice(ctx->device));
  GemmPlan p;
  char e[256];
  if (!gemm_make_plan(&p, A, std::max(M, 1), B, N, K, e, sizeof e)) return fail(ctx, RV_ECUDA, "%s", e);
  Epi ep;
  ep.bias = bias;
  ep.act = act;
  ep.resid = resid;
  ep.resid_rows = resid_rows;
  ep.resid_ld = resid_ld;
  ep.out = out;
  ep.out_rows = out_rows;
  ep.out_ld = out_ld;
  ep.out_bf16 = out_bf16;
  CK(gemm_launch(p, nullptr, M, M, ep, (cudaStream_t)stream));
  return RV_OK;
}

rv_status rv_stage_attention(rv_ctx* ctx, int32_t n_w, const int32_t* wdesc, const int32_t* qoff, const void* q,
                             int32_t q_rows, const void* KV, const int32_t* kvsrc, void* out, float* pcls,
                             int32_t use_tc, void* stream) {
  if (!ctx) return RV_ECONTRACT;
  if (q_rows < 1 || !q || !KV || !out) return fail(ctx, RV_ECONTRACT, "rv_stage_attention: bad arguments");
  CK(cudaSetDevice(ctx->device));
  if (use_tc == 2 || (use_tc == 1 && !attn_tc_supported(ctx->T, ctx->D, ctx->H))) {   // general tcgen05 kernel
    if (!attn_tcg_supported(ctx->T, ctx->D, ctx->H))
      return fail(ctx, RV_ECONTRACT, "rv_stage_attention: tcgen05 attention needs d_h = 64 and T <= 1025");
    CUtensorMap tm;
    char e[256];
    if (!make_tmap_bf16(&tm, q, q_rows, ctx->D, 64, e, sizeof e)) return fail(ctx, RV_ECUDA, "%s", e);
    CK(launch_attention_tcg(&tm, (const bf16*)q, ctx->D, 0, 0, (const bf16*)KV, 2LL * ctx->D, kvsrc, (bf16*)out, wdesc,
                            qoff, pcls, n_w, ctx->T, ctx->D, ctx->H, (cudaStream_t)stream));
    return RV_OK;
  }
  if (use_tc) {
    // K/V rows the wave can address: slots 0..max(slot); the tensor map needs the extent
    std::vector<int32_t> wd((size_t)n_w * 4);
    CK(cudaMemcpy(wd.data(), wdesc, wd.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
    long long slots = 0;
    for (int w = 0; w < n_w; ++w) slots = std::max<long long>(slots, wd[(size_t)w * 4] + 1LL);
    CUtensorMap tm, tkv;
    char e[256];
    if (!make_tmap_bf16(&tm, q, q_rows, ctx->D, 64, e, sizeof e) ||
        !make_tmap_bf16(&tkv, KV, slots * ctx->T, 2 * ctx->D, 1, e, sizeof e))
      return fail(ctx, RV_ECUDA, "%s", e);
    CK(launch_attention_tc(tm, tkv, (const bf16*)KV, kvsrc, (bf16*)out, wdesc, qoff, pcls, n_w, ctx->T, ctx->D, ctx->H,
                           (cudaStream_t)stream));
  } else {
    CK(launch_attention((const bf16*)q, (const bf16*)KV, kvsrc, (bf16*)out, wdesc, qoff, pcls, n_w, ctx->T,
                        ctx->D, ctx->H, (cudaStream_t)stream));
  }
  return RV_OK;
}

}  // extern "C"
