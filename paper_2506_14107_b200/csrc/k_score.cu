// k_score.cu — reuse decision and stream compaction for one level-wave.
//
// score_kernel (SURVEY §8(a) a2+a3): one CTA per frame of the wave, one warp per patch token.
//   Eq. 1  s_i = max over the available references of cos(T_cur_i, T_ref_i), fp32,
//                  provider = argmax, ties -> past; cos = 0 on a zero norm (Q9)
//   Eq. 2  v_i = [s_i, t_i, 1[I], 1[P], 1[B2], 1[B1], c_i]
//   Eq. 3  d_i = MLP_decision(v_i): lane j < Hg computes hidden unit j (Hg <= 32 = warp)
//   Eq. 4  M_i = 1 iff d_i > 0; CLS (token 0) is never reused
//   HBM-bound: reads 2-3 fp32 rows of D per token.
// compact_kernel (a4): Eq. 5-6 filtration as stream compaction (§5.3).
//   One CTA per frame; the frame's output offset is the sum of |C| over earlier frames of the
//   wave (integer, exact); a block-wide ballot scan ranks tokens.  Emits global rows
//   slot*T + token, CLS first in each frame, tokens ascending: bit-exact, deterministic, and
//   the counts never leave the device.
#include "common.cuh"
#include "rv_internal.h"

namespace rv {
namespace {

constexpr int SCORE_THREADS = 256;
// tokens per CTA: grid = n_w x ceil(N / tok).  Large waves take 64 (8 warps x 8 tokens; bench at
// 7,200 frames, score ms per step, 3 CTAs per SM: 16 -> 83.8, 32 -> 79.1, 64 -> 77.1-77.4,
// 128 -> 79.3, 256 -> 84.7); small waves (a few frames: short clips, the wavefront schedule)
// take fewer tokens per CTA until the grid fills the GPU, so a warp's tokens are not a serial
// latency chain.  Per-token work is independent of the split: results do not change.
constexpr int SCORE_TOK = 64;

// VPL > 0: D == 128 * VPL, the token's 3 x VPL float4 per lane are loaded unconditionally
// (a missing reference re-reads the current row, an L1 hit) and without a loop-carried branch,
// so all of them are in flight together; VPL == 0: generic D.
// RV_SCORE_MINB: resident CTAs per SM for the register allocation.  Bench at 7,200 frames (score
// ms per step): no bound (ptxas: 64 registers) 83.8; 3 (80 registers) 78.8; 2 (128) 87.7;
// 1 (unbounded) 127
#ifndef RV_SCORE_MINB
#define RV_SCORE_MINB 3
#endif
// 4 consecutive elements 4 k4 .. 4 k4 + 3 of a residual-stream row (fp32, or bf16: RV_X_BF16)
RV_DEV float4 ld4(const float* __restrict__ row, int k4) { return __ldg(reinterpret_cast<const float4*>(row) + k4); }
RV_DEV float4 ld4(const bf16* __restrict__ row, int k4) {
  const uint2 u = __ldg(reinterpret_cast<const uint2*>(row) + k4);
  const float2 lo = unpack_bf16x2(u.x), hi = unpack_bf16x2(u.y);
  return make_float4(lo.x, lo.y, hi.x, hi.y);
}

template <int VPL, typename XT>
__global__ void __launch_bounds__(SCORE_THREADS, RV_SCORE_MINB)
    score_kernel(const XT* __restrict__ X, int T, int D, int N, int L, int layer,
                 const int4* __restrict__ wdesc, const float* __restrict__ tsrc, int tH,
                 const float* __restrict__ codec, const uint8_t* force,
                 const float* __restrict__ gate, int Hg, int dense, uint8_t* masks, float* scores,
                 uint8_t* __restrict__ wmask, uint8_t* __restrict__ wprov, int* __restrict__ cntR,
                 bf16* __restrict__ dfull, int tok) {
  __shared__ int s_reused;
  const int w = blockIdx.x;
  const int i_beg = 1 + blockIdx.y * tok;
  const int i_end = min(N, i_beg + tok - 1);
  const int4 d4 = wdesc[w];
  const int slot = d4.x, past = d4.y, fut = d4.z, type = d4.w;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long mrow = ((long long)slot * L + layer) * N;   // masks/scores row of (slot, layer)
  const bool no_decision = dense || type == 0 || (past < 0 && fut < 0);
  if (threadIdx.x == 0) {
    s_reused = 0;
    if (blockIdx.y == 0) {
      wmask[(long long)w * T] = 0;
      wprov[(long long)w * T] = 0;
    }
  }
  if (no_decision) {
    for (int i = i_beg + threadIdx.x; i <= i_end; i += SCORE_THREADS) {
      wmask[(long long)w * T + i] = 0;
      wprov[(long long)w * T + i] = 0;
      if (masks) masks[mrow + i - 1] = 0;
      if (scores) scores[mrow + i - 1] = __int_as_float(0x7fc00000);   // NaN: no decision ran
    }
    return;
  }
  __syncthreads();
  // Decision-MLP weights of this layer: Wd1[7][Hg], bd1[Hg], Wd2[Hg], bd2[1].
  float w1[7], b1 = 0.f, w2 = 0.f;
#pragma unroll
  for (int k = 0; k < 7; ++k) w1[k] = lane < Hg ? __ldg(gate + k * Hg + lane) : 0.f;
  if (lane < Hg) {
    b1 = __ldg(gate + 7 * Hg + lane);
    w2 = __ldg(gate + 8 * Hg + lane);
  }
  const float b2 = __ldg(gate + 9 * Hg);
  const float oh0 = type == 0, oh1 = type == 1, oh2 = type == 2, oh3 = type == 3;
  const int D4 = D >> 2;
  int my_reused = 0;
  for (int i = i_beg + warp; i <= i_end; i += SCORE_THREADS / 32) {
    const XT* cur = X + ((long long)slot * T + i) * D;
    const XT* rp = past >= 0 ? X + ((long long)past * T + i) * D : nullptr;
    const XT* rf = fut >= 0 ? X + ((long long)fut * T + i) * D : nullptr;
    float cc = 0.f, pp = 0.f, ff = 0.f, cp = 0.f, cf = 0.f;
    if constexpr (VPL > 0 && sizeof(XT) == 2) {
      // bf16 rows (RV_X_BF16): 16 B = 8 columns per load, VPL / 2 loads per row and lane
      constexpr int V8 = VPL / 2;
      const uint4* c16 = reinterpret_cast<const uint4*>(cur);
      const uint4* p16 = reinterpret_cast<const uint4*>(rp ? rp : cur);
      const uint4* f16 = reinterpret_cast<const uint4*>(rf ? rf : cur);
      uint4 cv[V8], pv[V8], fv[V8];
#pragma unroll
      for (int j = 0; j < V8; ++j) {
        cv[j] = __ldg(c16 + lane + 32 * j);
        pv[j] = __ldg(p16 + lane + 32 * j);
        fv[j] = __ldg(f16 + lane + 32 * j);
      }
#pragma unroll
      for (int j = 0; j < V8; ++j) {
        const uint32_t cu[4] = {cv[j].x, cv[j].y, cv[j].z, cv[j].w};
        const uint32_t pu[4] = {pv[j].x, pv[j].y, pv[j].z, pv[j].w};
        const uint32_t fu[4] = {fv[j].x, fv[j].y, fv[j].z, fv[j].w};
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 c = unpack_bf16x2(cu[e]), p = unpack_bf16x2(pu[e]), f = unpack_bf16x2(fu[e]);
          cc += c.x * c.x + c.y * c.y;
          pp += p.x * p.x + p.y * p.y;
          cp += c.x * p.x + c.y * p.y;
          ff += f.x * f.x + f.y * f.y;
          cf += c.x * f.x + c.y * f.y;
        }
      }
      if (!rp) pp = cp = 0.f;
      if (!rf) ff = cf = 0.f;
    } else if constexpr (VPL > 0) {
      const XT* rp2 = rp ? rp : cur;
      const XT* rf2 = rf ? rf : cur;
      float4 cv[VPL], pv[VPL], fv[VPL];
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        cv[j] = ld4(cur, lane + 32 * j);
        pv[j] = ld4(rp2, lane + 32 * j);
        fv[j] = ld4(rf2, lane + 32 * j);
      }
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const float4 c = cv[j], p = pv[j], f = fv[j];
        cc += c.x * c.x + c.y * c.y + c.z * c.z + c.w * c.w;
        pp += p.x * p.x + p.y * p.y + p.z * p.z + p.w * p.w;
        cp += c.x * p.x + c.y * p.y + c.z * p.z + c.w * p.w;
        ff += f.x * f.x + f.y * f.y + f.z * f.z + f.w * f.w;
        cf += c.x * f.x + c.y * f.y + c.z * f.z + c.w * f.w;
      }
      if (!rp) pp = cp = 0.f;
      if (!rf) ff = cf = 0.f;
    } else
#pragma unroll 4
    for (int k = lane; k < D4; k += 32) {
      const float4 c = ld4(cur, k);
      cc += c.x * c.x + c.y * c.y + c.z * c.z + c.w * c.w;
      if (rp) {
        const float4 p = ld4(rp, k);
        pp += p.x * p.x + p.y * p.y + p.z * p.z + p.w * p.w;
        cp += c.x * p.x + c.y * p.y + c.z * p.z + c.w * p.w;
      }
      if (rf) {
        const float4 f = ld4(rf, k);
        ff += f.x * f.x + f.y * f.y + f.z * f.z + f.w * f.w;
        cf += c.x * f.x + c.y * f.y + c.z * f.z + c.w * f.w;
      }
    }
    cc = warp_sum(cc);
    pp = warp_sum(pp);
    ff = warp_sum(ff);
    cp = warp_sum(cp);
    cf = warp_sum(cf);
    float s = -2.f;
    int prov = 0;
    if (rp) {
      const float den = sqrtf(cc * pp);
      s = den > 0.f ? cp / den : 0.f;
    }
    if (rf) {
      const float den = sqrtf(cc * ff);
      const float sf = den > 0.f ? cf / den : 0.f;
      if (sf > s) { s = sf; prov = 1; }   // strict: ties keep the past reference
    }
    // t_i = head-mean of the previous layer's CLS attention to token i (fixed order)
    float t = 0.f;
    for (int hh = 0; hh < tH; ++hh) t += __ldg(tsrc + ((long long)slot * tH + hh) * N + i - 1);
    t = t / (float)tH;
    const float c = __ldg(codec + (long long)slot * N + i - 1);
    float h = b1 + s * w1[0] + t * w1[1] + oh0 * w1[2] + oh1 * w1[3] + oh2 * w1[4] + oh3 * w1[5] + c * w1[6];
    h = lane < Hg ? quick_gelu(h) * w2 : 0.f;
    const float dlogit = warp_sum(h) + b2;
    int M = dlogit > 0.f ? 1 : 0;
    if (force) M = force[mrow + i - 1] ? 1 : 0;
    if (lane == 0) {
      if (masks) masks[mrow + i - 1] = (uint8_t)M;
      if (scores) scores[mrow + i - 1] = dlogit;
      wmask[(long long)w * T + i] = (uint8_t)M;
      wprov[(long long)w * T + i] = (uint8_t)prov;
      my_reused += M;
    }
    if (M && dfull) {
      // Eq. 8: Delta R_i = R_cur_i - R_ref_i, written now while both rows are cache-hot, to
      // the wave-local token row w*T + i: the restoration GEMM reads it there in place
      const XT* rr = prov ? rf : rp;
      if constexpr (sizeof(XT) == 2) {   // bf16 rows: 8 columns (16 B in, 16 B out) per lane step
        const uint4* a16 = reinterpret_cast<const uint4*>(cur);
        const uint4* b16 = reinterpret_cast<const uint4*>(rr);
        uint4* o16 = reinterpret_cast<uint4*>(dfull + ((long long)w * T + i) * D);
#pragma unroll 4
        for (int k = lane; k < (D >> 3); k += 32) {
          const uint4 a = __ldg(a16 + k), b = __ldg(b16 + k);
          const uint32_t au[4] = {a.x, a.y, a.z, a.w}, bu[4] = {b.x, b.y, b.z, b.w};
          uint32_t o[4];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 x = unpack_bf16x2(au[e]), y = unpack_bf16x2(bu[e]);
            o[e] = pack_bf16x2(x.x - y.x, x.y - y.y);
          }
          o16[k] = make_uint4(o[0], o[1], o[2], o[3]);
        }
        continue;
      }
      uint2* o = reinterpret_cast<uint2*>(dfull + ((long long)w * T + i) * D);
#pragma unroll 4
      for (int k = lane; k < D4; k += 32) {
        const float4 a = ld4(cur, k), b = ld4(rr, k);
        uint2 u;
        u.x = pack_bf16x2(a.x - b.x, a.y - b.y);
        u.y = pack_bf16x2(a.z - b.z, a.w - b.w);
        o[k] = u;
      }
    }
  }
  if (lane == 0 && my_reused) atomicAdd(&s_reused, my_reused);
  __syncthreads();
  if (threadIdx.x == 0 && s_reused) atomicAdd(cntR + w, s_reused);   // integer: order-independent
}

constexpr int COMPACT_THREADS = 256;

// all_c (RV_NO_COMPACTION, the ablation's "masked dense" step): every token of every frame is in
// the recompute list (idxC = all rows in order, qoff[w] = w*T) while idxR / provrow still list
// the reused tokens, whose outputs the restoration then overwrites.  Outputs are bitwise those
// of the compacted path (row-local GEMMs and attention rows are batch-invariant).
__global__ void __launch_bounds__(COMPACT_THREADS)
    compact_kernel(int n_w, int T, const int4* __restrict__ wdesc, const uint8_t* __restrict__ wmask,
                   const uint8_t* __restrict__ wprov, const int* __restrict__ cntR, int* __restrict__ idxC,
                   int* __restrict__ idxR, int* __restrict__ provrow, int* __restrict__ qoff,
                   int* __restrict__ counts, int* kvsrc, unsigned long long* reuse_ctr, int* count_log,
                   int* __restrict__ rpos, int* __restrict__ rloc, int all_c) {
  __shared__ int s_part[COMPACT_THREADS / 32];
  __shared__ int s_wc[COMPACT_THREADS / 32], s_wr[COMPACT_THREADS / 32];
  __shared__ int s_base[2];
  const int w = blockIdx.x;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // offR = sum_{v<w} |R_v| (exact integer reduction); offC = w*T - offR (or w*T: all_c)
  int part = 0;
  for (int v = threadIdx.x; v < w; v += COMPACT_THREADS) part += cntR[v];
  part = warp_sum_i(part);
  if (lane == 0) s_part[warp] = part;
  __syncthreads();
  if (threadIdx.x == 0) {
    int offR = 0;
    for (int k = 0; k < COMPACT_THREADS / 32; ++k) offR += s_part[k];
    const int offC = all_c ? w * T : w * T - offR;
    s_base[0] = offC;
    s_base[1] = offR;
    qoff[w] = offC;
    if (w == n_w - 1) {
      const int totR = offR + cntR[w];
      const int totC = all_c ? n_w * T : n_w * T - totR;
      qoff[n_w] = totC;
      counts[0] = totC;
      counts[1] = totR;
      if (reuse_ctr) atomicAdd(reuse_ctr, (unsigned long long)totR);
      if (count_log) { count_log[0] = totC; count_log[1] = totR; }
    }
  }
  __syncthreads();
  const int4 d4 = wdesc[w];
  const int slot = d4.x;
  int offC = s_base[0], offR = s_base[1];
  const uint8_t* mk = wmask + (long long)w * T;
  const uint8_t* pv = wprov + (long long)w * T;
  for (int base = 0; base < T; base += COMPACT_THREADS) {
    const int i = base + threadIdx.x;
    const bool valid = i < T;
    const bool isR = valid && i > 0 && mk[i] != 0;
    const bool isC = valid && (all_c || !isR);
    const unsigned bc = __ballot_sync(0xffffffffu, isC);
    const unsigned br = __ballot_sync(0xffffffffu, isR);
    if (lane == 0) { s_wc[warp] = __popc(bc); s_wr[warp] = __popc(br); }
    __syncthreads();
    int pc = 0, pr = 0, tc = 0, tr = 0;
    for (int k = 0; k < COMPACT_THREADS / 32; ++k) {
      if (k < warp) { pc += s_wc[k]; pr += s_wr[k]; }
      tc += s_wc[k];
      tr += s_wr[k];
    }
    const unsigned lt = (1u << lane) - 1u;
    if (isC) {
      idxC[offC + pc + __popc(bc & lt)] = slot * T + i;
      if (!isR) {
        if (rpos) rpos[(long long)w * T + i] = -1;   // restoration row map: not reused
        if (kvsrc) kvsrc[(long long)slot * T + i] = slot * T + i;
      }
    }
    if (isR) {
      const int r = offR + pr + __popc(br & lt);
      const int prow = (pv[i] ? d4.z : d4.y) * T + i;
      if (rpos) rpos[(long long)w * T + i] = r;
      if (rloc) rloc[r] = w * T + i;      // wave-local Delta row of reused token r (fused restoration)
      idxR[r] = slot * T + i;
      provrow[r] = prow;
      // reuse-cache read in place: K/V of a reused token = its provider's (already final,
      // the provider ran in an earlier level), chains resolved here (one hop at read time)
      if (kvsrc) kvsrc[(long long)slot * T + i] = kvsrc[prow];
    }
    offC += tc;
    offR += tr;
    __syncthreads();
  }
}

// zero n 32-bit words (a kernel, not a memset node: the embed graph then holds no copy-engine
// work that a concurrent host-to-device copy of the next inputs could delay)
__global__ void zero_words_kernel(uint32_t* __restrict__ p, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = 0u;
}

__global__ void iota_kernel(int* __restrict__ p, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = (int)i;
}

}  // namespace

cudaError_t launch_iota(int* p, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  long long g = (n + 255) / 256;
  if (g > 148 * 8) g = 148 * 8;
  iota_kernel<<<(int)g, 256, 0, s>>>(p, n);
  return cudaGetLastError();
}

cudaError_t launch_zero_words(void* p, long long n, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  long long g = (n + 255) / 256;
  if (g > 148) g = 148;
  zero_words_kernel<<<(int)g, 256, 0, s>>>(reinterpret_cast<uint32_t*>(p), n);
  return cudaGetLastError();
}

cudaError_t launch_score(const void* X, int x_bf16, int T, int D, int N, int L, int layer, int n_w, const int* wdesc,
                         const float* tsrc, int tH, const float* codec, const uint8_t* force, const float* gate,
                         int Hg, int dense, uint8_t* masks, float* scores, uint8_t* wmask, uint8_t* wprov,
                         int* cntR, bf16* dfull, cudaStream_t s) {
  if (n_w <= 0) return cudaSuccess;
  cudaError_t e = launch_zero_words(cntR, n_w, s);
  if (e != cudaSuccess) return e;
  int tok = SCORE_TOK;
  while (tok > SCORE_THREADS / 32 && (long long)n_w * ((N + tok - 1) / tok) < 3LL * dev_sms()) tok >>= 1;
  dim3 grid(n_w, (N + tok - 1) / tok);
  const int4* wd = reinterpret_cast<const int4*>(wdesc);
#define RV_SCORE(V, XT)                                                                                         \
  score_kernel<V, XT><<<grid, SCORE_THREADS, 0, s>>>(reinterpret_cast<const XT*>(X), T, D, N, L, layer, wd, tsrc, tH, \
                                                     codec, force, gate, Hg, dense, masks, scores, wmask, wprov, cntR, \
                                                     dfull, tok)
  if (x_bf16) {
    if (D == 1024) RV_SCORE(8, bf16);
    else if (D == 768) RV_SCORE(6, bf16);
    else RV_SCORE(0, bf16);
  } else {
    if (D == 1024) RV_SCORE(8, float);
    else if (D == 768) RV_SCORE(6, float);
    else RV_SCORE(0, float);
  }
#undef RV_SCORE
  return cudaGetLastError();
}

cudaError_t launch_compact(int n_w, int T, const int* wdesc, const uint8_t* wmask, const uint8_t* wprov,
                           const int* cntR, int* idxC, int* idxR, int* provrow, int* qoff, int* counts, int* kvsrc,
                           unsigned long long* reuse_ctr, int* count_log, int* rpos, int* rloc, cudaStream_t s,
                           int all_c) {
  if (n_w <= 0) return cudaSuccess;
  compact_kernel<<<n_w, COMPACT_THREADS, 0, s>>>(n_w, T, reinterpret_cast<const int4*>(wdesc), wmask, wprov,
                                                 cntR, idxC, idxR, provrow, qoff, counts, kvsrc, reuse_ctr, count_log,
                                                 rpos, rloc, all_c);
  return cudaGetLastError();
}

}  // namespace rv
