// k_store.cu — embedding store query (paper §6.1: embeddings
// are cached per frame as fp16 and queried by cosine similarity; compute happens on a miss).
//   rv_f32_to_f16   : fp32 -> fp16 (RNE) conversion of embeddings entering the store
//   rv_topk_cosine  : for every query row, the k stored rows of highest cosine similarity,
//                     descending, ties broken by the lower record index; a zero-norm vector has
//                     cosine 0
// Pass 1 (cos_kernel): one warp per (query, stored row) pair stream, fp16 rows read with 16 B
// loads, fp32 dot products and norms -> scores [nq][n] (fp32).  Pass 2 (topk_kernel): one CTA
// per query selects k times the maximum of (score, -index) with a block reduction, marking the
// winner; k is small (retrieval), n may be large.
#include <cuda_fp16.h>

#include "common.cuh"
#include "rv_internal.h"
#include "reusevit.h"

namespace rv {
namespace {

__global__ void f32_to_f16_kernel(const float* __restrict__ src, __half* __restrict__ dst, long long count) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < count; i += (long long)gridDim.x * blockDim.x)
    dst[i] = __float2half_rn(src[i]);
}

// scores[qi][r] = cos(q[qi], emb[r]); grid (ceil(n / 8), nq), 8 warps, one row per warp
__global__ void cos_kernel(const __half* __restrict__ emb, int n, int D, const float* __restrict__ q, float* __restrict__ scores) {
  const int qi = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r = blockIdx.x * 8 + warp;
  if (r >= n) return;
  const float* qr = q + (long long)qi * D;
  const __half* er = emb + (long long)r * D;
  float dot = 0.f, ee = 0.f, qq = 0.f;
  for (int c = lane * 8; c < D; c += 256) {   // D % 8 == 0 (checked by the launcher)
    const uint4 u = *reinterpret_cast<const uint4*>(er + c);
    const __half2* h = reinterpret_cast<const __half2*>(&u);
    const float4 q0 = *reinterpret_cast<const float4*>(qr + c), q1 = *reinterpret_cast<const float4*>(qr + c + 4);
    const float qv[8] = {q0.x, q0.y, q0.z, q0.w, q1.x, q1.y, q1.z, q1.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __half22float2(h[e]);
      dot = fmaf(f.x, qv[2 * e], dot);
      dot = fmaf(f.y, qv[2 * e + 1], dot);
      ee = fmaf(f.x, f.x, ee);
      ee = fmaf(f.y, f.y, ee);
      qq = fmaf(qv[2 * e], qv[2 * e], qq);
      qq = fmaf(qv[2 * e + 1], qv[2 * e + 1], qq);
    }
  }
  dot = warp_sum(dot);
  ee = warp_sum(ee);
  qq = warp_sum(qq);
  if (lane == 0) {
    const float den = sqrtf(ee) * sqrtf(qq);
    scores[(long long)qi * n + r] = den > 0.f ? dot / den : 0.f;
  }
}

constexpr int TOPK_THREADS = 512;

// one CTA per query: k rounds of block-wide argmax over (score desc, index asc)
__global__ void __launch_bounds__(TOPK_THREADS) topk_kernel(float* __restrict__ scores, int n, int k,
                                                            int* __restrict__ out_idx, float* __restrict__ out_score) {
  const int qi = blockIdx.x;
  float* s = scores + (long long)qi * n;
  __shared__ float ws[TOPK_THREADS / 32];
  __shared__ int wi[TOPK_THREADS / 32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int t = 0; t < k; ++t) {
    float best = -INFINITY;
    int bi = 0x7fffffff;
    for (int r = threadIdx.x; r < n; r += TOPK_THREADS) {
      const float v = s[r];
      if (v > best || (v == best && r < bi)) { best = v; bi = r; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const float ov = __shfl_xor_sync(0xffffffffu, best, o);
      const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
    }
    if (lane == 0) { ws[warp] = best; wi[warp] = bi; }
    __syncthreads();
    if (warp == 0) {
      best = lane < TOPK_THREADS / 32 ? ws[lane] : -INFINITY;
      bi = lane < TOPK_THREADS / 32 ? wi[lane] : 0x7fffffff;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ov > best || (ov == best && oi < bi)) { best = ov; bi = oi; }
      }
      if (lane == 0) {
        const bool ok = bi < n && best != -INFINITY;
        out_idx[(long long)qi * k + t] = ok ? bi : -1;
        out_score[(long long)qi * k + t] = ok ? best : -INFINITY;
        if (ok) s[bi] = -INFINITY;   // selected: excluded from the next rounds
      }
    }
    __syncthreads();
  }
}

}  // namespace
}  // namespace rv

using namespace rv;

extern "C" {

rv_status rv_f32_to_f16(const float* src, void* dst, int64_t count, void* stream) {
  if (count < 0 || (count > 0 && (!src || !dst))) return RV_ECONTRACT;
  if (count == 0) return RV_OK;
  long long g = (count + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  f32_to_f16_kernel<<<(int)g, 256, 0, (cudaStream_t)stream>>>(src, reinterpret_cast<__half*>(dst), count);
  return cudaGetLastError() == cudaSuccess ? RV_OK : RV_ECUDA;
}

rv_status rv_topk_cosine(const void* emb16, int32_t n, int32_t D, const float* q, int32_t nq, int32_t k,
                         float* scores_tmp, int32_t* out_idx, float* out_score, void* stream) {
  if (n < 1 || D < 8 || D % 8 != 0 || nq < 1 || k < 1 || !emb16 || !q || !scores_tmp || !out_idx || !out_score)
    return RV_ECONTRACT;
  cudaStream_t s = (cudaStream_t)stream;
  cos_kernel<<<dim3((n + 7) / 8, nq), 256, 0, s>>>(reinterpret_cast<const __half*>(emb16), n, D, q, scores_tmp);
  if (cudaGetLastError() != cudaSuccess) return RV_ECUDA;
  topk_kernel<<<nq, TOPK_THREADS, 0, s>>>(scores_tmp, n, k, out_idx, out_score);
  return cudaGetLastError() == cudaSuccess ? RV_OK : RV_ECUDA;
}

}  // extern "C"
