// rv_internal.h — launcher declarations shared by the kernel translation units and the
// host runtime (runtime.cu).  Not part of the ABI.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <cuda_bf16.h>

namespace rv {

// ---------------------------------------------------------------- GEMM epilogue (k_gemm.cu)
// out[orow(m)][n] = act(acc[m][n] + bias[n]) + resid[rrow(m)][n]   (fp32 residual, or bf16 with
// resid_bf16: the RV_X_BF16 residual stream)
// orow(m) = out_rows ? out_rows[m] : m + (row_div ? m / row_div : 0) + row_add; orow(m) < 0: row m
// is computed but not stored (restoration GEMM R1 over the wave's token rows)
// Columns n >= split go to out2 (column n - split) with rows out2_rows[m].
struct Epi {
  const float* bias = nullptr;
  int act = 0;                 // 0 identity, 1 QuickGELU
  const void* resid = nullptr;
  const int* resid_rows = nullptr;
  long long resid_ld = 0;
  int resid_bf16 = 0;
  void* out = nullptr;
  const int* out_rows = nullptr;
  long long out_ld = 0;
  int out_bf16 = 0;
  int row_div = 0, row_add = 0;
  int split = 1 << 30;
  void* out2 = nullptr;
  const int* out2_rows = nullptr;
  long long out2_ld = 0;
  int out2_bf16 = 1;
};

struct GemmPlan {
  CUtensorMap tmA;        // A bf16 [rows][K], box {64, 128}, SWIZZLE_128B
  CUtensorMap tmB;        // B bf16 [N][K],    box {64, BN},  SWIZZLE_128B
  CUtensorMap tmB2;       // B bf16 [N][K],    box {64, BN/2} (CTA-pair GEMM: half of B per CTA)
  int N = 0, K = 0, BN = 0;
};

// Encode the tensor maps for a GEMM with A = [a_rows][K] and B = [N][K] (bf16, row-major).
// bn_max caps the N tile (256 / 128 / 64): residual-streaming epilogues prefer 128 (all of a
// tile's residual rows in flight before its accumulator is ready).
bool gemm_make_plan(GemmPlan* p, const void* A, long long a_rows, const void* B, int N, int K,
                    char* err, size_t errlen, int bn_max = 256);
// Launch: M read from *M_dev when M_dev != nullptr, else M_host.  max_m = host upper bound of
// M (sizes the persistent grid).
cudaError_t gemm_launch(const GemmPlan& p, const int* M_dev, int M_host, int max_m, const Epi& e,
                        cudaStream_t s);

// ---------------------------------------------------------------- row kernels (k_elem.cu)
typedef __nv_bfloat16 bf16;
cudaError_t launch_patch_to_bf16(const float* src, bf16* dst, long long rows, int pp, int KP, cudaStream_t s);
// x_bf16 / src_bf16: the residual stream X is bf16 (RV_X_BF16) instead of fp32
cudaError_t launch_embed_finish(void* X, int x_bf16, const float* cls, const float* pos, const float* g,
                                const float* b, float* pclsh, int n, int T, int D, int N, int H, cudaStream_t s);
cudaError_t launch_gather_ln(const void* src, int src_bf16, const int* rows, const int* count, int M_host,
                             int max_rows, const float* g, const float* b, bf16* dst, int D, cudaStream_t s);
cudaError_t launch_ln_post(const void* X, int x_bf16, const float* g, const float* b, float* emb, int n, int T, int D,
                           cudaStream_t s);

// ---------------------------------------------------------------- decision + compaction (k_score.cu)
cudaError_t launch_score(const void* X, int x_bf16, int T, int D, int N, int L, int layer, int n_w, const int* wdesc,
                         const float* tsrc, int tH, const float* codec, const uint8_t* force, const float* gate,
                         int Hg, int dense, uint8_t* masks, float* scores, uint8_t* wmask, uint8_t* wprov,
                         int* cntR, bf16* dfull, cudaStream_t s);
cudaError_t launch_zero_words(void* p, long long n_words, cudaStream_t s);
cudaError_t launch_iota(int* p, long long n, cudaStream_t s);   // p[i] = i
cudaError_t launch_compact(int n_w, int T, const int* wdesc, const uint8_t* wmask, const uint8_t* wprov,
                           const int* cntR, int* idxC, int* idxR, int* provrow, int* qoff, int* counts, int* kvsrc,
                           unsigned long long* reuse_ctr, int* count_log, int* rpos, int* rloc, cudaStream_t s,
                           int all_c = 0);

// ---------------------------------------------------------------- fused restoration (k_restore.cu)
// Eq. 8-10 over the M_R = *M_dev compacted reused rows of a wave: X[idxR[r]] = X[provrow[r]] +
// QuickGELU(dfull[rloc[r]] W_r1^T + b_r1) W_r2^T + b_r2 (X fp32, or bf16 with x_bf16); Hr = 128.
bool restore_supported(int D, int Hr);
bool restore_make_maps(CUtensorMap* tmW1, CUtensorMap* tmW2, const bf16* Wr1, const bf16* Wr2, int D, int Hr,
                       char* err, size_t errlen);
cudaError_t launch_restore(const CUtensorMap& tmW1, const CUtensorMap& tmW2, const bf16* dfull, const int* rloc,
                           const int* provrow, const int* idxR, const int* M_dev, int max_rows, const float* br1,
                           const float* br2, void* X, int x_bf16, int D, cudaStream_t s);

// 2D bf16 tensor map, box {64 cols, box_rows}, SWIZZLE_128B (k_gemm.cu)
bool make_tmap_bf16(CUtensorMap* m, const void* ptr, long long rows, int cols, int box_rows, char* err,
                    size_t errlen);

// ---------------------------------------------------------------- attention (k_attn_tc.cu, k_attn.cu)
bool attn_tc_supported(int T, int D, int H);
cudaError_t launch_attention_tc(const CUtensorMap& tmQ, const CUtensorMap& tmKV, const bf16* KV, const int* kvsrc,
                                bf16* out,
                                const int* wdesc, const int* qoff, float* pclsh, int n_w, int T, int D, int H,
                                cudaStream_t s);
// general-shape tcgen05 attention (k_attn_tcg.cu): d_h = 64, T - 1 <= 1024.
// q_mode 0: compacted queries q[qoff[w] + r], loaded through tmQ (box {64, 64} over q, row stride
// q_ld = D); 1: every token of a frame is a query with its q row q[kvsrc[slot T + i]] at column
// q_col (chain variant's q|k|v cache, tmQ unused); K / V rows through kvsrc (identity if null)
// with stride kv_ld (head h: K at column 2 h d_h, V at 2 h d_h + d_h); output rows qoff[w] + r.
bool attn_tcg_supported(int T, int D, int H);
cudaError_t launch_attention_tcg(const CUtensorMap* tmQ, const bf16* q, long long q_ld, int q_col, int q_mode,
                                 const bf16* KV, long long kv_ld, const int* kvsrc, bf16* out, const int* wdesc,
                                 const int* qoff, float* pclsh, int n_w, int T, int D, int H, cudaStream_t s);
// kv_ld: K/V cache row stride (0 -> 2D); q_cache: queries are all T tokens of each frame with q read
// from the cache row at column 2D through kvsrc (SPEC chain variant), qoff[w] = w*T
cudaError_t launch_attention(const bf16* q, const bf16* KV, const int* kvsrc, bf16* out, const int* wdesc,
                             const int* qoff, float* pclsh, int n_w, int T, int D, int H, cudaStream_t s,
                             long long kv_ld = 0, int q_cache = 0);
}  // namespace rv
