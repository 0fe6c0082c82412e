// trainer.cu — gate training of ReuseViT on the GPU (§4
// P:398-482; C-ABI include/reusevit_train.h).  The frozen ViT's forward is re-run soft-gated
// (Eq. 11-12, readings T1-T3 of DESIGN.md §3) for B groups of G frames, the grouped loss of
// Eq. 13-15 is formed on the device, and a hand-written reverse pass produces the gradient of
// every decision / restoration parameter (the ViT stays frozen); Adam updates
// them.  Toy-scale training: fp32 on the CUDA cores, plain tiled kernels, deterministic (no
// float atomics: cross-frame accumulations walk the group's computation order per token).
//
// Layouts (all fp32 unless noted): frame f = b*G + k (local frame k of group b, ascending
// display order); token rows r = f*T + i; per-layer saved activations [L][F][T][...].
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <string>
#include <vector>

#include "../../include/reusevit.h"
#include "../../include/reusevit_train.h"
#include "common.cuh"

namespace rv {
namespace trn {

// ------------------------------------------------------------------ generic fp32 GEMM
// C[m][n] = beta * C[m][n] + sum_k A(m, k) B(k, n) + bias[n], k ascending (deterministic).
// A(m, k) = TA ? A[k lda + m] : A[m lda + k];  B(k, n) = TB ? B[n ldb + k] : B[k ldb + n].
// beta == 0 never reads C.  64 x 64 tiles, 16-deep k slices, 4 x 4 outputs per thread.
template <int TA, int TB>
__global__ void __launch_bounds__(256) k_gemm(int M, int N, int K, const float* __restrict__ A, long long lda,
                                              const float* __restrict__ B, long long ldb, float* C, long long ldc,
                                              float beta, const float* __restrict__ bias) {
  __shared__ float As[16][65];
  __shared__ float Bs[16][65];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  float acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int e = threadIdx.x; e < 16 * 64; e += 256) {
      int kk, mm;
      if (TA) { mm = e % 64; kk = e / 64; } else { kk = e % 16; mm = e / 16; }
      int gm = m0 + mm, gk = k0 + kk;
      As[kk][mm] = (gm < M && gk < K) ? (TA ? A[(long long)gk * lda + gm] : A[(long long)gm * lda + gk]) : 0.f;
      int nn;
      if (TB) { kk = e % 16; nn = e / 16; } else { nn = e % 64; kk = e / 64; }
      const int gn = n0 + nn;
      gk = k0 + kk;
      Bs[kk][nn] = (gn < N && gk < K) ? (TB ? B[(long long)gn * ldb + gk] : B[(long long)gk * ldb + gn]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) { a[i] = As[kk][ty + 16 * i]; b[i] = Bs[kk][tx + 16 * i]; }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + ty + 16 * i, n = n0 + tx + 16 * j;
      if (m < M && n < N) {
        float v = acc[i][j] + (bias ? bias[n] : 0.f);
        float* c = C + (long long)m * ldc + n;
        *c = beta != 0.f ? beta * *c + v : v;
      }
    }
}

// out[n] = sum_m A[m lda + n] (rows ascending)
__global__ void k_colsum(int M, int N, const float* __restrict__ A, long long lda, float* out) {
  const int n = blockIdx.x * blockDim.x + threadIdx.x;
  if (n >= N) return;
  float s = 0.f;
  for (int m = 0; m < M; ++m) s += A[(long long)m * lda + n];
  out[n] = s;
}

RV_DEV float qg(float a) { return a / (1.f + expf(-1.702f * a)); }
RV_DEV float qg_grad(float a) {
  const float s = 1.f / (1.f + expf(-1.702f * a));
  return s + 1.702f * a * s * (1.f - s);
}

// y = qg(a)
__global__ void k_qg(long long n, const float* a, float* y) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = qg(a[i]);
}
// g = qg'(a) * g
__global__ void k_qg_bwd(long long n, const float* a, float* g) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    g[i] = qg_grad(a[i]) * g[i];
}
// y += x
__global__ void k_acc(long long n, const float* x, float* y) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] += x[i];
}

// LayerNorm over rows of D (biased variance, eps 1e-5), one warp per row.
__global__ void k_ln_fwd(int rows, int D, const float* X, long long ldx, const float* g, const float* b, float* Y,
                         long long ldy, float* mu, float* rs) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* x = X + (long long)row * ldx;
  float s = 0.f;
  for (int d = lane; d < D; d += 32) s += x[d];
  const float m = warp_sum(s) / D;
  float v = 0.f;
  for (int d = lane; d < D; d += 32) v += (x[d] - m) * (x[d] - m);
  const float r = 1.f / sqrtf(warp_sum(v) / D + 1e-5f);
  float* y = Y + (long long)row * ldy;
  for (int d = lane; d < D; d += 32) y[d] = (x[d] - m) * r * g[d] + b[d];
  if (lane == 0 && mu) { mu[row] = m; rs[row] = r; }
}
// dX += d LN(X) / dX . dY
__global__ void k_ln_bwd(int rows, int D, const float* dY, long long ldd, const float* X, long long ldx, const float* g,
                         const float* mu, const float* rs, float* dX, long long lddx) {
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float* x = X + (long long)row * ldx;
  const float* dy = dY + (long long)row * ldd;
  const float m = mu[row], r = rs[row];
  float s1 = 0.f, s2 = 0.f;
  for (int d = lane; d < D; d += 32) {
    const float gy = dy[d] * g[d], xh = (x[d] - m) * r;
    s1 += gy;
    s2 += gy * xh;
  }
  s1 = warp_sum(s1) / D;
  s2 = warp_sum(s2) / D;
  float* dx = dX + (long long)row * lddx;
  for (int d = lane; d < D; d += 32) {
    const float gy = dy[d] * g[d], xh = (x[d] - m) * r;
    dx[d] += r * (gy - s1 - xh * s2);
  }
}

// X0 rows before ln_pre: [cls; patches W_pe] + pos
__global__ void k_embed_pre(int F, int T, int N, int D, const float* E, const float* cls, const float* pos, float* X) {
  const long long n = (long long)F * T * D;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int d = (int)(e % D);
    const long long r = e / D;
    const int i = (int)(r % T);
    const long long f = r / T;
    X[e] = (i == 0 ? cls[d] : E[(f * N + i - 1) * D + d]) + pos[(long long)i * D + d];
  }
}

struct Plan {
  const int *type, *past, *fut, *order;   // [G] device
};

// Eq. 1-4 + Eq. 11 per token (one warp per token).  mode 0 soft, 1 dense (M = 0), 2 forced M.
// Writes M, provider frame (-1: no decision), features v[8] (7 used), decision hidden
// pre-activation hd[Hg], logit d (NaN without decision).
__global__ void __launch_bounds__(256) k_decision(int F, int G, int T, int D, int N, int H, int L, int l, Plan pl,
                                                  const float* X, const float* pcls, const float* codec,
                                                  const float* gumbel, const float* gate, int Hg, float tau, int mode,
                                                  const float* force, float* M, int* prov, float* v8, float* hd,
                                                  float* dlog) {
  const int f = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i = blockIdx.y * 8 + warp;
  if (i >= T) return;
  const int k = f % G, base = f - k;
  const int type = pl.type[k];
  const int pa = pl.past[k] >= 0 ? base + pl.past[k] : -1, fu = pl.fut[k] >= 0 ? base + pl.fut[k] : -1;
  const long long row = (long long)f * T + i;
  const bool decide = mode != 1 && type != RV_I && (pa >= 0 || fu >= 0) && i > 0;
  if (!decide) {
    if (lane == 0) { M[row] = 0.f; prov[row] = -1; dlog[row] = __int_as_float(0x7fc00000); }
    if (lane < 8) v8[row * 8 + lane] = 0.f;
    if (lane < Hg) hd[row * Hg + lane] = 0.f;
    return;
  }
  const float* cur = X + row * D;
  const float* rp = pa >= 0 ? X + ((long long)pa * T + i) * D : nullptr;
  const float* rf = fu >= 0 ? X + ((long long)fu * T + i) * D : nullptr;
  float cc = 0.f, pp = 0.f, cp = 0.f, ff = 0.f, cf = 0.f;
  for (int d = lane; d < D; d += 32) {
    const float c = cur[d];
    cc += c * c;
    if (rp) { pp += rp[d] * rp[d]; cp += c * rp[d]; }
    if (rf) { ff += rf[d] * rf[d]; cf += c * rf[d]; }
  }
  cc = warp_sum(cc); pp = warp_sum(pp); cp = warp_sum(cp); ff = warp_sum(ff); cf = warp_sum(cf);
  float s = -2.f;
  int pv = -1;
  if (rp) { const float den = sqrtf(cc * pp); s = den > 0.f ? cp / den : 0.f; pv = pa; }
  if (rf) {
    const float den = sqrtf(cc * ff);
    const float sf = den > 0.f ? cf / den : 0.f;
    if (sf > s) { s = sf; pv = fu; }   // ties keep the past reference (D3)
  }
  float t = 0.f;
  for (int h = 0; h < H; ++h) t += pcls[((long long)f * H + h) * N + i - 1];
  t /= (float)H;
  const float c = codec[(long long)f * N + i - 1];
  const float vv[7] = {s, t, type == RV_I ? 1.f : 0.f, type == RV_P ? 1.f : 0.f, type == RV_B2 ? 1.f : 0.f,
                       type == RV_B1 ? 1.f : 0.f, c};
  float contrib = 0.f;
  if (lane < Hg) {
    float h = gate[7 * Hg + lane];
#pragma unroll
    for (int q = 0; q < 7; ++q) h = fmaf(vv[q], gate[q * Hg + lane], h);
    hd[row * Hg + lane] = h;
    contrib = qg(h) * gate[8 * Hg + lane];
  }
  const float dl = warp_sum(contrib) + gate[9 * Hg];
  if (lane < 7) v8[row * 8 + lane] = vv[lane];
  if (lane == 7) v8[row * 8 + 7] = 0.f;
  if (lane == 0) {
    float m;
    if (mode == 2) {
      m = force[((long long)f * L + l) * N + i - 1];
    } else {   // Eq. 11, two logits (d + g_reuse, g_recompute) / tau: the reuse probability
      const float* g = gumbel + (((long long)f * L + l) * N + i - 1) * 2;
      m = 1.f / (1.f + expf(-(dl + g[0] - g[1]) / tau));
    }
    M[row] = m;
    prov[row] = pv;
    dlog[row] = dl;
  }
}

// K/V blend (reading T2) per (group, token), frames in computation order: a frame's blended
// row reads its provider's blended row of the same token (computed earlier in the loop by the
// same thread for the same column).
__global__ void k_kv_blend(int G, int T, int D, const int* order, const float* M, const int* prov, const float* qkv,
                           float* Ks, float* Vs) {
  const int b = blockIdx.x, i = blockIdx.y;
  for (int p = 0; p < G; ++p) {
    const long long row = (long long)(b * G + order[p]) * T + i;
    const int pf = prov[row];
    const float m = M[row];
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      const float kc = qkv[row * 3 * D + D + d], vc = qkv[row * 3 * D + 2 * D + d];
      if (pf >= 0) {
        const long long pr = ((long long)pf * T + i) * D + d;
        Ks[row * D + d] = m * Ks[pr] + (1.f - m) * kc;
        Vs[row * D + d] = m * Vs[pr] + (1.f - m) * vc;
      } else {
        Ks[row * D + d] = kc;
        Vs[row * D + d] = vc;
      }
    }
  }
}

// Attention of every token over all T (blended) keys of its frame; one CTA per (frame, head),
// one warp per query row.  Saves P [F][H][T][T]; CLS row's patch columns -> pcls (t of l+1).
__global__ void k_attn_fwd(int T, int D, int H, const float* qkv, const float* Ks, const float* Vs, float* P,
                           float* o, float* pcls, float scale) {
  extern __shared__ float sh[];
  const int f = blockIdx.x, h = blockIdx.y, dh = D / H;
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* sK = sh;                      // [T][dh]
  float* sV = sK + T * dh;             // [T][dh]
  float* sq = sV + T * dh + warp * (dh + T);   // per warp: q [dh], p [T]
  float* sp = sq + dh;
  for (int e = threadIdx.x; e < T * dh; e += blockDim.x) {
    const int j = e / dh, c = e % dh;
    const long long r = ((long long)f * T + j) * D + h * dh + c;
    sK[e] = Ks[r];
    sV[e] = Vs[r];
  }
  __syncthreads();
  for (int i = warp; i < T; i += nw) {
    const long long row = (long long)f * T + i;
    for (int c = lane; c < dh; c += 32) sq[c] = qkv[row * 3 * D + h * dh + c];
    __syncwarp();
    float mx = -INFINITY;
    for (int j = lane; j < T; j += 32) {
      float s = 0.f;
      for (int c = 0; c < dh; ++c) s = fmaf(sq[c], sK[j * dh + c], s);
      s *= scale;
      sp[j] = s;
      mx = fmaxf(mx, s);
    }
    mx = warp_max(mx);
    float sum = 0.f;
    for (int j = lane; j < T; j += 32) {
      const float e = expf(sp[j] - mx);
      sp[j] = e;
      sum += e;
    }
    const float inv = 1.f / warp_sum(sum);
    float* Prow = P + (((long long)f * H + h) * T + i) * T;
    for (int j = lane; j < T; j += 32) {
      sp[j] *= inv;
      Prow[j] = sp[j];
      if (i == 0 && j > 0) pcls[((long long)f * H + h) * (T - 1) + j - 1] = sp[j];
    }
    __syncwarp();
    for (int c = lane; c < dh; c += 32) {
      float acc = 0.f;
      for (int j = 0; j < T; ++j) acc = fmaf(sp[j], sV[j * dh + c], acc);
      o[row * D + h * dh + c] = acc;
    }
    __syncwarp();
  }
}

// Attention backward per (frame, head): phase 1 (warp per query row) dS = P (dP - rowsum(dP P)),
// dq = scale dS K; phase 2 (warp per key row) dK = scale dS^T q, dV = P^T dO.
__global__ void k_attn_bwd(int T, int D, int H, const float* qkv, const float* Ks, const float* Vs, const float* P,
                           const float* dO, float* dS, float* dqkv, float* dKs, float* dVs, float scale) {
  const int f = blockIdx.x, h = blockIdx.y, dh = D / H;
  const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long pb = ((long long)f * H + h) * T * T;
  for (int i = warp; i < T; i += nw) {
    const long long row = (long long)f * T + i;
    float rs = 0.f;
    for (int j = lane; j < T; j += 32) {
      float dp = 0.f;
      for (int c = 0; c < dh; ++c) dp = fmaf(dO[row * D + h * dh + c], Vs[((long long)f * T + j) * D + h * dh + c], dp);
      dS[pb + (long long)i * T + j] = dp;
      rs += dp * P[pb + (long long)i * T + j];
    }
    rs = warp_sum(rs);
    __syncwarp();
    for (int j = lane; j < T; j += 32) {
      const long long e = pb + (long long)i * T + j;
      dS[e] = P[e] * (dS[e] - rs);
    }
    __syncwarp();
    for (int c = lane; c < dh; c += 32) {
      float acc = 0.f;
      for (int j = 0; j < T; ++j) acc = fmaf(dS[pb + (long long)i * T + j], Ks[((long long)f * T + j) * D + h * dh + c], acc);
      dqkv[row * 3 * D + h * dh + c] = scale * acc;
    }
  }
  __syncthreads();
  for (int j = warp; j < T; j += nw) {
    const long long rj = (long long)f * T + j;
    for (int c = lane; c < dh; c += 32) {
      float ak = 0.f, av = 0.f;
      for (int i = 0; i < T; ++i) {
        const long long ri = (long long)f * T + i;
        ak = fmaf(dS[pb + (long long)i * T + j], qkv[ri * 3 * D + h * dh + c], ak);
        av = fmaf(P[pb + (long long)i * T + j], dO[ri * D + h * dh + c], av);
      }
      dKs[rj * D + h * dh + c] = scale * ak;
      dVs[rj * D + h * dh + c] = av;
    }
  }
}

// Delta = X_{l-1}[f][i] - X_{l-1}[prov][i] for decided tokens, else 0 (Eq. 8)
__global__ void k_delta(long long rows, int T, int D, const int* prov, const float* X, float* dl) {
  const long long n = rows * D;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const long long r = e / D;
    const int d = (int)(e % D);
    const int pf = prov[r];
    dl[e] = pf >= 0 ? X[e] - X[((long long)pf * T + (r % T)) * D + d] : 0.f;
  }
}

RV_DEV float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  __syncthreads();
  if (lane == 0) red[warp] = v;
  __syncthreads();
  float s = 0.f;
  for (int w = 0; w < nw; ++w) s += red[w];
  return s;
}

// Eq. 12 output blend per (group, token) in computation order: R_hat = X_l[prov] + r (r = the
// restoration MLP output, overwritten by R_hat), X_l = M R_hat + (1 - M) C_tilde.
__global__ void k_out_blend(int G, int T, int D, const int* order, const float* M, const int* prov, const float* Ct,
                            float* Rh, float* Xout) {
  const int b = blockIdx.x, i = blockIdx.y;
  for (int p = 0; p < G; ++p) {
    const long long row = (long long)(b * G + order[p]) * T + i;
    const int pf = prov[row];
    const float m = M[row];
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      const float ct = Ct[row * D + d];
      if (pf >= 0) {
        const float rh = Rh[row * D + d] + Xout[((long long)pf * T + i) * D + d];
        Rh[row * D + d] = rh;
        Xout[row * D + d] = m * rh + (1.f - m) * ct;
      } else {
        Xout[row * D + d] = ct;
      }
    }
  }
}

// Backward of k_out_blend, frames in reverse computation order (a frame's dX_l is complete
// once its dependents, later in the order, have added their dR_hat).  dMacc = (R_hat - C) . dX.
__global__ void k_out_blend_bwd(int G, int T, int D, const int* order, const float* M, const int* prov,
                                const float* Ct, const float* Rh, float* dXl, float* dRh, float* dCt, float* dMacc) {
  __shared__ float red[32];
  const int b = blockIdx.x, i = blockIdx.y;
  for (int p = G - 1; p >= 0; --p) {
    const long long row = (long long)(b * G + order[p]) * T + i;
    const int pf = prov[row];
    const float m = M[row];
    float dm = 0.f;
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      const float g = dXl[row * D + d];
      if (pf >= 0) {
        dRh[row * D + d] = m * g;
        dCt[row * D + d] = (1.f - m) * g;
        dm += (Rh[row * D + d] - Ct[row * D + d]) * g;
        dXl[((long long)pf * T + i) * D + d] += m * g;
      } else {
        dRh[row * D + d] = 0.f;
        dCt[row * D + d] = g;
      }
    }
    dm = block_sum(dm, red);
    if (threadIdx.x == 0) dMacc[row] = pf >= 0 ? dm : 0.f;
  }
}

// dX_{l-1}[f] += dDelta, dX_{l-1}[prov] -= dDelta per (group, token), computation order
__global__ void k_delta_bwd(int G, int T, int D, const int* order, const int* prov, const float* dDl, float* dXp) {
  const int b = blockIdx.x, i = blockIdx.y;
  for (int p = G - 1; p >= 0; --p) {
    const long long row = (long long)(b * G + order[p]) * T + i;
    const int pf = prov[row];
    if (pf < 0) continue;
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      const float g = dDl[row * D + d];
      dXp[row * D + d] += g;
      dXp[((long long)pf * T + i) * D + d] -= g;
    }
  }
}

// Backward of k_kv_blend, reverse computation order: own k/v gradient (1 - M) dK into dqkv,
// M dK added to the provider's blended-row gradient, dMacc += (K_prov - k_own) . dK + (V ...).
__global__ void k_kv_blend_bwd(int G, int T, int D, const int* order, const float* M, const int* prov,
                               const float* qkv, const float* Ks, const float* Vs, float* dKs, float* dVs,
                               float* dqkv, float* dMacc) {
  __shared__ float red[32];
  const int b = blockIdx.x, i = blockIdx.y;
  for (int p = G - 1; p >= 0; --p) {
    const long long row = (long long)(b * G + order[p]) * T + i;
    const int pf = prov[row];
    const float m = M[row];
    float dm = 0.f;
    for (int d = threadIdx.x; d < D; d += blockDim.x) {
      const float gk = dKs[row * D + d], gv = dVs[row * D + d];
      if (pf >= 0) {
        const long long pr = ((long long)pf * T + i) * D + d;
        dqkv[row * 3 * D + D + d] = (1.f - m) * gk;
        dqkv[row * 3 * D + 2 * D + d] = (1.f - m) * gv;
        dm += (Ks[pr] - qkv[row * 3 * D + D + d]) * gk + (Vs[pr] - qkv[row * 3 * D + 2 * D + d]) * gv;
        dKs[pr] += m * gk;
        dVs[pr] += m * gv;
      } else {
        dqkv[row * 3 * D + D + d] = gk;
        dqkv[row * 3 * D + 2 * D + d] = gv;
      }
    }
    dm = block_sum(dm, red);
    if (threadIdx.x == 0 && pf >= 0) dMacc[row] += dm;
  }
}

// Decision backward per token (warp): dd = (dMacc + dMcoef[b]) dM/dd, dM/dd = M (1 - M) / tau;
// dhpre = qg'(hd) dd Wd2; hact = qg(hd).  Undecided tokens: zeros.
__global__ void k_decision_bwd(long long rows, int G, int T, int Hg, const float* M, const int* prov, const float* hd,
                               const float* dMacc, const float* dMcoef, const float* gate, float tau, float* dd,
                               float* dhpre, float* hact) {
  const long long row = blockIdx.x * 8LL + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const int b = (int)(row / T) / G;
  if (prov[row] < 0) {
    if (lane == 0) dd[row] = 0.f;
    if (lane < Hg) { dhpre[row * Hg + lane] = 0.f; hact[row * Hg + lane] = 0.f; }
    return;
  }
  const float m = M[row];
  const float g = (dMacc[row] + dMcoef[b]) * m * (1.f - m) / tau;
  if (lane == 0) dd[row] = g;
  if (lane < Hg) {
    const float h = hd[row * Hg + lane];
    hact[row * Hg + lane] = qg(h);
    dhpre[row * Hg + lane] = qg_grad(h) * g * gate[8 * Hg + lane];
  }
}

// Eq. 13-15 per group (one CTA per group, warp per frame) and the loss gradients: dZ of the
// batch-mean loss, and the reuse term's dL/dM (the same for every decided token of a group).
__global__ void k_loss(int G, int L, int T, int D, int N, Plan pl, const float* Z, const float* Zref, const float* M,
                       long long Mstride, float alpha, float R, float invB, float* out, float* dZ, float* dMcoef) {
  __shared__ float red[32];
  __shared__ float cosk[32];
  const int b = blockIdx.x, warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int k = warp; k < G; k += nw) {
    const long long f = (long long)b * G + k;
    const float* z = Z + f * D;
    const float* zr = Zref + f * D;
    float zz = 0.f, rr = 0.f, zx = 0.f;
    for (int d = lane; d < D; d += 32) { zz += z[d] * z[d]; rr += zr[d] * zr[d]; zx += z[d] * zr[d]; }
    zz = warp_sum(zz); rr = warp_sum(rr); zx = warp_sum(zx);
    const float den = sqrtf(zz * rr);
    const float c = den > 0.f ? zx / den : 0.f;
    if (lane == 0) cosk[k] = c;
    // d(1 - cos)/dz = -(zr / den - cos z / |z|^2), times invB / G (batch mean of group means)
    const float sc = -invB / G;
    for (int d = lane; d < D; d += 32)
      dZ[f * D + d] = den > 0.f ? sc * (zr[d] / den - c * z[d] / zz) : 0.f;
  }
  // reuse: mean of M over non-I frames, layers, patch tokens (Eq. 14)
  float s = 0.f;
  int cnt = 0;
  for (int k = 0; k < G; ++k) {
    if (pl.type[k] == RV_I) continue;
    cnt += L * N;
    const long long f = (long long)b * G + k;
    for (int e = threadIdx.x; e < L * N; e += blockDim.x) {
      const int l = e / N, i = 1 + e % N;
      s += M[l * Mstride + f * T + i];
    }
  }
  s = block_sum(s, red);
  __syncthreads();
  if (threadIdx.x == 0) {
    float ls = 0.f, cs = 0.f;
    for (int k = 0; k < G; ++k) { ls += 1.f - cosk[k]; cs += cosk[k]; }
    ls /= G;
    const float lr = cnt ? s / cnt : 0.f;
    const float hinge = R - lr;
    out[b * 4 + 0] = ls;
    out[b * 4 + 1] = lr;
    out[b * 4 + 2] = ls + alpha * fmaxf(hinge, 0.f);
    out[b * 4 + 3] = cs;
    dMcoef[b] = (hinge > 0.f && cnt) ? -alpha * invB / cnt : 0.f;
  }
}

__global__ void k_adam(long long n, float* p, const float* g, float* m, float* v, float lr, float b1, float b2, float eps,
                       float c1, float c2) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float gi = g[i];
    m[i] = b1 * m[i] + (1.f - b1) * gi;
    v[i] = b2 * v[i] + (1.f - b2) * gi * gi;
    p[i] -= lr * (m[i] * c1) / (sqrtf(v[i] * c2) + eps);
  }
}

__global__ void k_fill(long long n, float* p, float v) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    p[i] = v;
}

}  // namespace trn
}  // namespace rv

using namespace rv::trn;

namespace {

struct VitOff {   // offsets (floats) of the RVW1 arrays
  size_t W_pe, cls, pos, lnpre_g, lnpre_b, lnpost_g, lnpost_b;
  struct Layer { size_t ln1_g, ln1_b, Wqkv, bqkv, Wo, bo, ln2_g, ln2_b, W1, b1, W2, b2; };
  std::vector<Layer> l;
};
struct GateOff {
  struct Layer { size_t Wd1, Wr1, br1, Wr2, br2; };   // decision block = [Wd1 | bd1 | Wd2 | bd2] from Wd1
  std::vector<Layer> l;
  size_t total = 0;
};

}  // namespace

struct rv_trainer {
  rv_config cfg{};
  int L = 0, D = 0, H = 0, N = 0, T = 0, pp = 0, Fh = 0, Hr = 0, Hg = 0, device = 0;
  int Bcap = 0, G = 0, F = 0;
  float alpha = 0, R = 0, lr = 0, b1 = 0.9f, b2 = 0.999f, eps = 1e-8f;
  int steps = 0;
  std::string err;
  std::vector<void*> allocs;
  VitOff vo;
  GateOff go;
  float* Wv = nullptr;                       // RVW1 fp32 on device
  float *P = nullptr, *dP = nullptr, *am = nullptr, *av = nullptr;   // RVG1 params, grads, Adam moments
  int *d_plan = nullptr;                     // type | past | future | order  [4][G]
  std::vector<int> order_h;
  // activations (per layer unless noted)
  float *X = nullptr;                        // [L+1][F][T][D]
  float *h1, *mu1, *rs1, *qkv, *Ks, *Vs, *Pa, *o, *x1, *h2, *mu2, *rs2, *a1, *g1, *Ct, *dl, *r1, *r1a, *Rh, *M, *v8,
      *hd, *dlog;
  int* prov = nullptr;
  float *pcls, *E, *Z, *Zref, *mup, *rsp;
  // backward scratch (one layer)
  float *dXl, *dXp, *dRh, *dCt, *dx1, *dg1, *dh, *dOa, *dS, *dqkv, *dKs, *dVs, *dMacc, *dr1, *dDl, *dhpre, *hact, *dd,
      *dZ, *dMcoef, *lossb;
};

namespace {

thread_local std::string g_terr;

rv_status tfail(rv_trainer* t, rv_status s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  if (t) t->err = buf;
  else g_terr = buf;
  return s;
}
#define TCK(call)                                                                                          \
  do {                                                                                                     \
    cudaError_t _e = (call);                                                                               \
    if (_e != cudaSuccess) return tfail(tr, RV_ECUDA, "%s:%d %s: %s", __FILE__, __LINE__, #call, cudaGetErrorString(_e)); \
  } while (0)

template <class T>
bool talloc(rv_trainer* t, T** p, size_t n) {
  void* q = nullptr;
  if (cudaMalloc(&q, std::max<size_t>(n, 1) * sizeof(T)) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  cudaMemset(q, 0, std::max<size_t>(n, 1) * sizeof(T));
  t->allocs.push_back(q);
  *p = reinterpret_cast<T*>(q);
  return true;
}

inline int nblk(long long n) { return (int)std::min<long long>((n + 255) / 256, 148LL * 16); }

void gemm(cudaStream_t s, int M, int N, int K, const float* A, long long lda, bool ta, const float* B, long long ldb,
          bool tb, float* C, long long ldc, float beta = 0.f, const float* bias = nullptr) {
  if (M <= 0 || N <= 0) return;
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  if (!ta && !tb) k_gemm<0, 0><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, beta, bias);
  else if (!ta && tb) k_gemm<0, 1><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, beta, bias);
  else if (ta && !tb) k_gemm<1, 0><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, beta, bias);
  else k_gemm<1, 1><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, beta, bias);
}
void colsum(cudaStream_t s, int M, int N, const float* A, long long lda, float* out) {
  k_colsum<<<(N + 127) / 128, 128, 0, s>>>(M, N, A, lda, out);
}

bool cfg_ok(const rv_config* c, char* why, size_t n) {
  if (!c || c->layers < 1 || c->dim < 16 || c->heads < 1 || c->dim % c->heads || c->patch < 1 || c->img % c->patch ||
      c->ffn < 1 || c->hidden_r < 1 || c->hidden_g < 1 || c->hidden_g > 32) {
    snprintf(why, n, "invalid config");
    return false;
  }
  const int N = (c->img / c->patch) * (c->img / c->patch);
  const int dh = c->dim / c->heads;
  if ((size_t)(2 * (N + 1) * dh + 4 * (dh + N + 1)) * 4 > 160 * 1024) {
    snprintf(why, n, "the trainer's attention keeps a frame-head's K/V in shared memory: T * d_h too large");
    return false;
  }
  return true;
}

}  // namespace

// ====================================================================== C-ABI
extern "C" {

const char* rv_trainer_last_error(const rv_trainer* t) { return t ? t->err.c_str() : g_terr.c_str(); }

void rv_trainer_destroy(rv_trainer* t) {
  if (!t) return;
  cudaSetDevice(t->device);
  for (void* p : t->allocs) cudaFree(p);
  delete t;
}

rv_status rv_trainer_create(const rv_config* cfg, int device, const float* vit_blob, size_t vit_floats,
                            const float* gate_blob, size_t gate_floats, const rv_train_config* tc, rv_trainer** out) {
  rv_trainer* tr = nullptr;
  if (!out) return tfail(tr, RV_ECONTRACT, "rv_trainer_create: out is NULL");
  *out = nullptr;
  char why[200];
  if (!cfg_ok(cfg, why, sizeof why)) return tfail(tr, RV_ECONFIG, "rv_trainer_create: %s", why);
  if (!vit_blob || !gate_blob || !tc || !tc->type || !tc->past || !tc->future || !tc->order)
    return tfail(tr, RV_ECONTRACT, "rv_trainer_create: null argument");
  if (tc->groups < 1 || tc->group_size < 1 || tc->group_size > 32)
    return tfail(tr, RV_ECONTRACT, "rv_trainer_create: groups >= 1 and 1 <= group_size <= 32");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev) {
    cudaGetLastError();
    return tfail(tr, RV_ECUDA, "rv_trainer_create: no CUDA device %d (there is no CPU fallback)", device);
  }
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess || prop.major != 10)
    return tfail(tr, RV_ECUDA, "rv_trainer_create: device %d is not sm_100", device);
  // plan check: types, references inside the group and computed before use
  const int G = tc->group_size;
  {
    std::vector<int> pos(G, -1);
    for (int p = 0; p < G; ++p) {
      const int k = tc->order[p];
      if (k < 0 || k >= G || pos[k] >= 0) return tfail(tr, RV_EPLAN, "group plan: order is not a permutation");
      pos[k] = p;
    }
    for (int k = 0; k < G; ++k) {
      const int t = tc->type[k];
      if (t < RV_I || t > RV_B1) return tfail(tr, RV_EPLAN, "group plan: bad type");
      const int r[2] = {tc->past[k], tc->future[k]};
      int nref = 0;
      for (int j = 0; j < 2; ++j) {
        if (r[j] == -1) continue;
        if (r[j] < 0 || r[j] >= G || r[j] == k || pos[r[j]] >= pos[k])
          return tfail(tr, RV_EPLAN, "group plan: frame %d reference %d invalid or not computed first", k, r[j]);
        ++nref;
      }
      if ((t == RV_I) != (nref == 0)) return tfail(tr, RV_EPLAN, "group plan: frame %d type/reference mismatch", k);
    }
  }
  cudaSetDevice(device);
  tr = new rv_trainer();
  tr->cfg = *cfg;
  tr->device = device;
  tr->L = cfg->layers; tr->D = cfg->dim; tr->H = cfg->heads;
  tr->N = (cfg->img / cfg->patch) * (cfg->img / cfg->patch); tr->T = tr->N + 1;
  tr->pp = 3 * cfg->patch * cfg->patch; tr->Fh = cfg->ffn; tr->Hr = cfg->hidden_r; tr->Hg = cfg->hidden_g;
  tr->Bcap = tc->groups; tr->G = G; tr->F = tc->groups * G;
  tr->alpha = tc->alpha; tr->R = tc->r_target; tr->lr = tc->lr;
  tr->b1 = tc->beta1; tr->b2 = tc->beta2; tr->eps = tc->eps;
  const int L = tr->L, D = tr->D, T = tr->T, Fh = tr->Fh, Hr = tr->Hr, Hg = tr->Hg, pp = tr->pp;
  // RVW1 / RVG1 offsets (SURVEY §8(c) declaration order)
  size_t o = 0;
  tr->vo.W_pe = o; o += (size_t)pp * D;
  tr->vo.cls = o; o += D;
  tr->vo.pos = o; o += (size_t)T * D;
  tr->vo.lnpre_g = o; o += D;
  tr->vo.lnpre_b = o; o += D;
  tr->vo.l.resize(L);
  for (int l = 0; l < L; ++l) {
    auto& w = tr->vo.l[l];
    w.ln1_g = o; o += D; w.ln1_b = o; o += D;
    w.Wqkv = o; o += (size_t)D * 3 * D; w.bqkv = o; o += 3 * D;
    w.Wo = o; o += (size_t)D * D; w.bo = o; o += D;
    w.ln2_g = o; o += D; w.ln2_b = o; o += D;
    w.W1 = o; o += (size_t)D * Fh; w.b1 = o; o += Fh;
    w.W2 = o; o += (size_t)Fh * D; w.b2 = o; o += D;
  }
  tr->vo.lnpost_g = o; o += D;
  tr->vo.lnpost_b = o; o += D;
  if (o != vit_floats) {
    rv_trainer_destroy(tr);
    return tfail(nullptr, RV_ESHAPE, "rv_trainer_create: ViT blob has %zu floats, config needs %zu", vit_floats, o);
  }
  size_t g = 0;
  tr->go.l.resize(L);
  for (int l = 0; l < L; ++l) {
    auto& w = tr->go.l[l];
    w.Wd1 = g; g += 7 * Hg + Hg + Hg + 1;
    w.Wr1 = g; g += (size_t)D * Hr; w.br1 = g; g += Hr;
    w.Wr2 = g; g += (size_t)Hr * D; w.br2 = g; g += D;
  }
  tr->go.total = g;
  if (g != gate_floats) {
    rv_trainer_destroy(tr);
    return tfail(nullptr, RV_ESHAPE, "rv_trainer_create: gate blob has %zu floats, config needs %zu", gate_floats, g);
  }
  const long long F = tr->F, FT = F * T, H = tr->H, N = tr->N;
  bool ok = talloc(tr, &tr->Wv, vit_floats) && talloc(tr, &tr->P, g) && talloc(tr, &tr->dP, g) &&
            talloc(tr, &tr->am, g) && talloc(tr, &tr->av, g) && talloc(tr, &tr->d_plan, 4 * G) &&
            talloc(tr, &tr->X, (size_t)(L + 1) * FT * D) && talloc(tr, &tr->h1, (size_t)L * FT * D) &&
            talloc(tr, &tr->mu1, (size_t)L * FT) && talloc(tr, &tr->rs1, (size_t)L * FT) &&
            talloc(tr, &tr->qkv, (size_t)L * FT * 3 * D) && talloc(tr, &tr->Ks, (size_t)L * FT * D) &&
            talloc(tr, &tr->Vs, (size_t)L * FT * D) && talloc(tr, &tr->Pa, (size_t)L * F * H * T * T) &&
            talloc(tr, &tr->o, (size_t)L * FT * D) && talloc(tr, &tr->x1, (size_t)L * FT * D) &&
            talloc(tr, &tr->h2, (size_t)L * FT * D) && talloc(tr, &tr->mu2, (size_t)L * FT) &&
            talloc(tr, &tr->rs2, (size_t)L * FT) && talloc(tr, &tr->a1, (size_t)L * FT * Fh) &&
            talloc(tr, &tr->g1, (size_t)L * FT * Fh) && talloc(tr, &tr->Ct, (size_t)L * FT * D) &&
            talloc(tr, &tr->dl, (size_t)L * FT * D) && talloc(tr, &tr->r1, (size_t)L * FT * Hr) &&
            talloc(tr, &tr->r1a, (size_t)L * FT * Hr) && talloc(tr, &tr->Rh, (size_t)L * FT * D) &&
            talloc(tr, &tr->M, (size_t)L * FT) && talloc(tr, &tr->prov, (size_t)L * FT) &&
            talloc(tr, &tr->v8, (size_t)L * FT * 8) && talloc(tr, &tr->hd, (size_t)L * FT * Hg) &&
            talloc(tr, &tr->dlog, (size_t)L * FT) && talloc(tr, &tr->pcls, (size_t)F * H * N) &&
            talloc(tr, &tr->E, (size_t)F * N * D) && talloc(tr, &tr->Z, (size_t)F * D) &&
            talloc(tr, &tr->Zref, (size_t)F * D) && talloc(tr, &tr->mup, (size_t)F) && talloc(tr, &tr->rsp, (size_t)F) &&
            talloc(tr, &tr->dXl, (size_t)FT * D) && talloc(tr, &tr->dXp, (size_t)FT * D) &&
            talloc(tr, &tr->dRh, (size_t)FT * D) && talloc(tr, &tr->dCt, (size_t)FT * D) &&
            talloc(tr, &tr->dx1, (size_t)FT * D) && talloc(tr, &tr->dg1, (size_t)FT * Fh) &&
            talloc(tr, &tr->dh, (size_t)FT * D) && talloc(tr, &tr->dOa, (size_t)FT * D) &&
            talloc(tr, &tr->dS, (size_t)F * H * T * T) && talloc(tr, &tr->dqkv, (size_t)FT * 3 * D) &&
            talloc(tr, &tr->dKs, (size_t)FT * D) && talloc(tr, &tr->dVs, (size_t)FT * D) &&
            talloc(tr, &tr->dMacc, (size_t)FT) && talloc(tr, &tr->dr1, (size_t)FT * Hr) &&
            talloc(tr, &tr->dDl, (size_t)FT * D) && talloc(tr, &tr->dhpre, (size_t)FT * Hg) &&
            talloc(tr, &tr->hact, (size_t)FT * Hg) && talloc(tr, &tr->dd, (size_t)FT) &&
            talloc(tr, &tr->dZ, (size_t)F * D) && talloc(tr, &tr->dMcoef, (size_t)tr->Bcap) &&
            talloc(tr, &tr->lossb, (size_t)tr->Bcap * 4);
  if (!ok) {
    rv_trainer_destroy(tr);
    return tfail(nullptr, RV_ENOMEM, "rv_trainer_create: cudaMalloc failed");
  }
  std::vector<int> ph(4 * G);
  for (int k = 0; k < G; ++k) {
    ph[k] = tc->type[k];
    ph[G + k] = tc->past[k];
    ph[2 * G + k] = tc->future[k];
    ph[3 * G + k] = tc->order[k];
  }
  tr->order_h.assign(tc->order, tc->order + G);
  if (cudaMemcpy(tr->d_plan, ph.data(), ph.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(tr->Wv, vit_blob, vit_floats * 4, cudaMemcpyHostToDevice) != cudaSuccess ||
      cudaMemcpy(tr->P, gate_blob, gate_floats * 4, cudaMemcpyHostToDevice) != cudaSuccess) {
    rv_trainer_destroy(tr);
    return tfail(nullptr, RV_ECUDA, "rv_trainer_create: upload failed");
  }
  *out = tr;
  return RV_OK;
}

}  // extern "C"

namespace {

Plan plan_of(rv_trainer* tr) {
  const int G = tr->G;
  return Plan{tr->d_plan, tr->d_plan + G, tr->d_plan + 2 * G, tr->d_plan + 3 * G};
}

// Soft-gated forward of B groups (mode 0 soft, 1 dense, 2 forced), activations saved.
cudaError_t forward(rv_trainer* tr, const float* patches, const float* codec, const float* gumbel, int B, float tau,
                    int mode, const float* force, float* Zout, cudaStream_t s) {
  const int L = tr->L, D = tr->D, H = tr->H, N = tr->N, T = tr->T, Fh = tr->Fh, Hr = tr->Hr, Hg = tr->Hg, G = tr->G;
  const long long F = (long long)B * G, FT = F * T, FTc = (long long)tr->F * T;
  const float* W = tr->Wv;
  const Plan pl = plan_of(tr);
  const int* order = pl.order;
  // a1: X0 = LN_pre([cls; patches W_pe] + pos)
  gemm(s, (int)(F * N), D, tr->pp, patches, tr->pp, false, W + tr->vo.W_pe, D, false, tr->E, D);
  k_embed_pre<<<nblk(FT * D), 256, 0, s>>>((int)F, T, N, D, tr->E, W + tr->vo.cls, W + tr->vo.pos, tr->dOa);
  k_ln_fwd<<<(int)((FT + 7) / 8), 256, 0, s>>>((int)FT, D, tr->dOa, D, W + tr->vo.lnpre_g, W + tr->vo.lnpre_b, tr->X,
                                               D, nullptr, nullptr);
  k_fill<<<nblk(F * H * N), 256, 0, s>>>(F * H * N, tr->pcls, 1.f / N);   // t of layer 1: uniform
  const float scale = 1.f / sqrtf((float)(D / H));
  const size_t attn_smem = (size_t)(2 * T * (D / H) + 4 * ((D / H) + T)) * 4;
  cudaError_t e = rv::ensure_smem<k_attn_fwd>(attn_smem);
  if (e != cudaSuccess) return e;
  for (int l = 0; l < L; ++l) {
    const auto& w = tr->vo.l[l];
    const auto& gw = tr->go.l[l];
    const float* Xin = tr->X + (size_t)l * FTc * D;
    float* Xout = tr->X + (size_t)(l + 1) * FTc * D;
    const size_t oD = (size_t)l * FTc * D, o1 = (size_t)l * FTc;
    float *h1 = tr->h1 + oD, *qkv = tr->qkv + oD * 3, *Ks = tr->Ks + oD, *Vs = tr->Vs + oD, *o = tr->o + oD,
          *x1 = tr->x1 + oD, *h2 = tr->h2 + oD, *a1 = tr->a1 + o1 * Fh, *g1 = tr->g1 + o1 * Fh, *Ct = tr->Ct + oD,
          *dl = tr->dl + oD, *r1 = tr->r1 + o1 * Hr, *r1a = tr->r1a + o1 * Hr, *Rh = tr->Rh + oD, *M = tr->M + o1;
    int* prov = tr->prov + o1;
    float* Pa = tr->Pa + (size_t)l * tr->F * H * T * T;
    // Eq. 1-4, 11
    k_decision<<<dim3((unsigned)F, (T + 7) / 8), 256, 0, s>>>((int)F, G, T, D, N, H, L, l, pl, Xin, tr->pcls, codec,
                                                              gumbel, tr->P + gw.Wd1, Hg, tau, mode, force, M, prov,
                                                              tr->v8 + o1 * 8, tr->hd + o1 * Hg, tr->dlog + o1);
    // recompute branch (Eq. 7) for every token; K/V blended (T2)
    k_ln_fwd<<<(int)((FT + 7) / 8), 256, 0, s>>>((int)FT, D, Xin, D, W + w.ln1_g, W + w.ln1_b, h1, D, tr->mu1 + o1,
                                                 tr->rs1 + o1);
    gemm(s, (int)FT, 3 * D, D, h1, D, false, W + w.Wqkv, 3 * D, false, qkv, 3 * D, 0.f, W + w.bqkv);
    k_kv_blend<<<dim3(B, T), 128, 0, s>>>(G, T, D, order, M, prov, qkv, Ks, Vs);
    k_attn_fwd<<<dim3((unsigned)F, H), 128, attn_smem, s>>>(T, D, H, qkv, Ks, Vs, Pa, o, tr->pcls, scale);
    cudaMemcpyAsync(x1, Xin, FT * D * 4, cudaMemcpyDeviceToDevice, s);
    gemm(s, (int)FT, D, D, o, D, false, W + w.Wo, D, false, x1, D, 1.f, W + w.bo);
    k_ln_fwd<<<(int)((FT + 7) / 8), 256, 0, s>>>((int)FT, D, x1, D, W + w.ln2_g, W + w.ln2_b, h2, D, tr->mu2 + o1,
                                                 tr->rs2 + o1);
    gemm(s, (int)FT, Fh, D, h2, D, false, W + w.W1, Fh, false, a1, Fh, 0.f, W + w.b1);
    k_qg<<<nblk(FT * Fh), 256, 0, s>>>(FT * Fh, a1, g1);
    cudaMemcpyAsync(Ct, x1, FT * D * 4, cudaMemcpyDeviceToDevice, s);
    gemm(s, (int)FT, D, Fh, g1, Fh, false, W + w.W2, D, false, Ct, D, 1.f, W + w.b2);
    // restoration branch (Eq. 8-9) and Eq. 12 blend
    k_delta<<<nblk(FT * D), 256, 0, s>>>(FT, T, D, prov, Xin, dl);
    gemm(s, (int)FT, Hr, D, dl, D, false, tr->P + gw.Wr1, Hr, false, r1, Hr, 0.f, tr->P + gw.br1);
    k_qg<<<nblk(FT * Hr), 256, 0, s>>>(FT * Hr, r1, r1a);
    gemm(s, (int)FT, D, Hr, r1a, Hr, false, tr->P + gw.Wr2, D, false, Rh, D, 0.f, tr->P + gw.br2);
    k_out_blend<<<dim3(B, T), 128, 0, s>>>(G, T, D, order, M, prov, Ct, Rh, Xout);
  }
  // Z = LN_post(X_L[CLS])
  k_ln_fwd<<<(int)((F + 7) / 8), 256, 0, s>>>((int)F, D, tr->X + (size_t)L * FTc * D, (long long)T * D,
                                              W + tr->vo.lnpost_g, W + tr->vo.lnpost_b, Zout, D, tr->mup, tr->rsp);
  return cudaGetLastError();
}

// Reverse pass of the last soft forward given dZ (batch-mean loss gradient) and dMcoef.
cudaError_t backward(rv_trainer* tr, int B, float tau, cudaStream_t s) {
  const int L = tr->L, D = tr->D, H = tr->H, T = tr->T, Fh = tr->Fh, Hr = tr->Hr, Hg = tr->Hg, G = tr->G;
  const long long F = (long long)B * G, FT = F * T, FTc = (long long)tr->F * T;
  const float* W = tr->Wv;
  const int* order = tr->d_plan + 3 * G;
  const float scale = 1.f / sqrtf((float)(D / H));
  cudaMemsetAsync(tr->dP, 0, tr->go.total * 4, s);
  cudaMemsetAsync(tr->dXl, 0, FT * D * 4, s);
  k_ln_bwd<<<(int)((F + 7) / 8), 256, 0, s>>>((int)F, D, tr->dZ, D, tr->X + (size_t)L * FTc * D, (long long)T * D,
                                              W + tr->vo.lnpost_g, tr->mup, tr->rsp, tr->dXl, (long long)T * D);
  for (int l = L - 1; l >= 0; --l) {
    const auto& w = tr->vo.l[l];
    const auto& gw = tr->go.l[l];
    const float* Xin = tr->X + (size_t)l * FTc * D;
    const size_t oD = (size_t)l * FTc * D, o1 = (size_t)l * FTc;
    const float *h1 = tr->h1 + oD, *qkv = tr->qkv + oD * 3, *Ks = tr->Ks + oD, *Vs = tr->Vs + oD, *x1 = tr->x1 + oD,
                *a1 = tr->a1 + o1 * Fh, *g1 = tr->g1 + o1 * Fh, *Ct = tr->Ct + oD, *dl = tr->dl + oD,
                *r1 = tr->r1 + o1 * Hr, *r1a = tr->r1a + o1 * Hr, *Rh = tr->Rh + oD, *M = tr->M + o1;
    (void)h1;
    (void)g1;
    const int* prov = tr->prov + o1;
    const float* Pa = tr->Pa + (size_t)l * tr->F * H * T * T;
    float* gP = tr->dP;
    cudaMemsetAsync(tr->dXp, 0, FT * D * 4, s);
    // Eq. 12 blend -> restored / recomputed branches, dL/dM, provider's X_l
    k_out_blend_bwd<<<dim3(B, T), 128, 0, s>>>(G, T, D, order, M, prov, Ct, Rh, tr->dXl, tr->dRh, tr->dCt, tr->dMacc);
    // restoration MLP (Eq. 9): r = qg(Delta Wr1 + br1) Wr2 + br2
    gemm(s, Hr, D, (int)FT, r1a, Hr, true, tr->dRh, D, false, gP + gw.Wr2, D);
    colsum(s, (int)FT, D, tr->dRh, D, gP + gw.br2);
    gemm(s, (int)FT, Hr, D, tr->dRh, D, false, tr->P + gw.Wr2, D, true, tr->dr1, Hr);
    k_qg_bwd<<<nblk(FT * Hr), 256, 0, s>>>(FT * Hr, r1, tr->dr1);
    gemm(s, D, Hr, (int)FT, dl, D, true, tr->dr1, Hr, false, gP + gw.Wr1, Hr);
    colsum(s, (int)FT, Hr, tr->dr1, Hr, gP + gw.br1);
    gemm(s, (int)FT, D, Hr, tr->dr1, Hr, false, tr->P + gw.Wr1, Hr, true, tr->dDl, D);
    k_delta_bwd<<<dim3(B, T), 128, 0, s>>>(G, T, D, order, prov, tr->dDl, tr->dXp);
    // recompute branch: C = x1 + qg(LN2(x1) W1 + b1) W2 + b2, x1 = X + o Wo + bo
    cudaMemcpyAsync(tr->dx1, tr->dCt, FT * D * 4, cudaMemcpyDeviceToDevice, s);
    gemm(s, (int)FT, Fh, D, tr->dCt, D, false, W + w.W2, D, true, tr->dg1, Fh);
    k_qg_bwd<<<nblk(FT * Fh), 256, 0, s>>>(FT * Fh, a1, tr->dg1);
    (void)g1;
    gemm(s, (int)FT, D, Fh, tr->dg1, Fh, false, W + w.W1, Fh, true, tr->dh, D);
    k_ln_bwd<<<(int)((FT + 7) / 8), 256, 0, s>>>((int)FT, D, tr->dh, D, x1, D, W + w.ln2_g, tr->mu2 + o1, tr->rs2 + o1,
                                                 tr->dx1, D);
    k_acc<<<nblk(FT * D), 256, 0, s>>>(FT * D, tr->dx1, tr->dXp);
    gemm(s, (int)FT, D, D, tr->dx1, D, false, W + w.Wo, D, true, tr->dOa, D);
    // attention, then the K/V blend (provider rows accumulate in reverse computation order)
    k_attn_bwd<<<dim3((unsigned)F, H), 128, 0, s>>>(T, D, H, qkv, Ks, Vs, Pa, tr->dOa, tr->dS, tr->dqkv, tr->dKs, tr->dVs,
                                                    scale);
    k_kv_blend_bwd<<<dim3(B, T), 128, 0, s>>>(G, T, D, order, M, prov, qkv, Ks, Vs, tr->dKs, tr->dVs, tr->dqkv,
                                              tr->dMacc);
    // QKV and LN1
    gemm(s, (int)FT, D, 3 * D, tr->dqkv, 3 * D, false, W + w.Wqkv, 3 * D, true, tr->dh, D);
    k_ln_bwd<<<(int)((FT + 7) / 8), 256, 0, s>>>((int)FT, D, tr->dh, D, Xin, D, W + w.ln1_g, tr->mu1 + o1, tr->rs1 + o1,
                                                 tr->dXp, D);
    // decision MLP (Eq. 3) through Eq. 11
    k_decision_bwd<<<(int)((FT + 7) / 8), 256, 0, s>>>(FT, G, T, Hg, M, prov, tr->hd + o1 * Hg, tr->dMacc, tr->dMcoef,
                                                       tr->P + gw.Wd1, tau, tr->dd, tr->dhpre, tr->hact);
    gemm(s, 7, Hg, (int)FT, tr->v8 + o1 * 8, 8, true, tr->dhpre, Hg, false, gP + gw.Wd1, Hg);   // dWd1 [7][Hg]
    colsum(s, (int)FT, Hg, tr->dhpre, Hg, gP + gw.Wd1 + 7 * Hg);                               // dbd1
    gemm(s, Hg, 1, (int)FT, tr->hact, Hg, true, tr->dd, 1, false, gP + gw.Wd1 + 8 * Hg, 1);     // dWd2
    colsum(s, (int)FT, 1, tr->dd, 1, gP + gw.Wd1 + 9 * Hg);                                    // dbd2
    std::swap(tr->dXl, tr->dXp);
  }
  return cudaGetLastError();
}

rv_status check_io(rv_trainer* tr, const float* patches, const float* codec, const float* gumbel, int B, float tau,
                   bool need_gumbel) {
  if (!tr) return RV_ECONTRACT;
  if (!patches || !codec || (need_gumbel && !gumbel)) return tfail(tr, RV_ECONTRACT, "null input");
  if (B < 1 || B > tr->Bcap) return tfail(tr, RV_ECONTRACT, "B = %d outside 1..%d (trainer capacity)", B, tr->Bcap);
  if (!(tau > 0.f)) return tfail(tr, RV_ECONTRACT, "temperature must be > 0 (S:203)");
  return RV_OK;
}

rv_status loss_grad(rv_trainer* tr, const float* patches, const float* codec, const float* gumbel, int B, float tau,
                    rv_train_log* log, cudaStream_t s) {
  const long long F = (long long)B * tr->G;
  cudaError_t e = forward(tr, patches, codec, gumbel, B, tau, 1, nullptr, tr->Zref, s);   // frozen ViT's Z
  if (e == cudaSuccess) e = forward(tr, patches, codec, gumbel, B, tau, 0, nullptr, tr->Z, s);
  if (e != cudaSuccess) return tfail(tr, RV_ECUDA, "forward: %s", cudaGetErrorString(e));
  k_loss<<<B, 256, 0, s>>>(tr->G, tr->L, tr->T, tr->D, tr->N, plan_of(tr), tr->Z, tr->Zref, tr->M,
                           (long long)tr->F * tr->T, tr->alpha, tr->R, 1.f / B, tr->lossb, tr->dZ, tr->dMcoef);
  e = backward(tr, B, tau, s);
  if (e != cudaSuccess) return tfail(tr, RV_ECUDA, "backward: %s", cudaGetErrorString(e));
  if (log) {
    std::vector<float> lb((size_t)B * 4);
    if (cudaMemcpyAsync(lb.data(), tr->lossb, lb.size() * 4, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
        cudaStreamSynchronize(s) != cudaSuccess)
      return tfail(tr, RV_ECUDA, "loss readback: %s", cudaGetErrorString(cudaGetLastError()));
    double a = 0, b = 0, c = 0, d = 0;
    for (int k = 0; k < B; ++k) { a += lb[k * 4]; b += lb[k * 4 + 1]; c += lb[k * 4 + 2]; d += lb[k * 4 + 3]; }
    log->l_sim = a / B;
    log->l_reuse = b / B;
    log->l_total = c / B;
    log->cos_mean = d / (double)F;
    log->step = tr->steps;
  }
  return RV_OK;
}

}  // namespace

extern "C" {

rv_status rv_trainer_forward(rv_trainer* tr, const float* patches, const float* codec, const float* gumbel, int32_t B,
                             float tau, uint32_t flags, const float* force, float* Z, float* M, float* d,
                             void* stream) {
  const int mode = (flags & RV_TRAIN_DENSE) ? 1 : ((flags & RV_TRAIN_FORCE) ? 2 : 0);
  rv_status st = check_io(tr, patches, codec, gumbel, B, tau, mode == 0);
  if (st) return st;
  if (mode == 2 && !force) return tfail(tr, RV_ECONTRACT, "RV_TRAIN_FORCE needs force");
  TCK(cudaSetDevice(tr->device));
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = forward(tr, patches, codec, gumbel, B, tau, mode, force, tr->Z, s);
  if (e != cudaSuccess) return tfail(tr, RV_ECUDA, "forward: %s", cudaGetErrorString(e));
  const int L = tr->L, N = tr->N, T = tr->T, D = tr->D, G = tr->G;
  const long long F = (long long)B * G;
  if (Z) TCK(cudaMemcpyAsync(Z, tr->Z, F * D * 4, cudaMemcpyDeviceToDevice, s));
  // M / d [B][G][L][N] from the per-layer [L][F][T] buffers (patch tokens)
  for (int l = 0; l < L && (M || d); ++l) {
    const size_t o1 = (size_t)l * tr->F * T;
    if (M) TCK(cudaMemcpy2DAsync(M + (size_t)l * N, (size_t)L * N * 4, tr->M + o1 + 1, (size_t)T * 4, N * 4, F,
                                 cudaMemcpyDeviceToDevice, s));
    if (d) TCK(cudaMemcpy2DAsync(d + (size_t)l * N, (size_t)L * N * 4, tr->dlog + o1 + 1, (size_t)T * 4, N * 4, F,
                                 cudaMemcpyDeviceToDevice, s));
  }
  return RV_OK;
}

rv_status rv_trainer_loss_grad(rv_trainer* tr, const float* patches, const float* codec, const float* gumbel,
                               int32_t B, float tau, float* grad_blob, rv_train_log* log, void* stream) {
  rv_status st = check_io(tr, patches, codec, gumbel, B, tau, true);
  if (st) return st;
  TCK(cudaSetDevice(tr->device));
  cudaStream_t s = (cudaStream_t)stream;
  if ((st = loss_grad(tr, patches, codec, gumbel, B, tau, log, s))) return st;
  if (grad_blob) TCK(cudaMemcpyAsync(grad_blob, tr->dP, tr->go.total * 4, cudaMemcpyDeviceToDevice, s));
  TCK(cudaStreamSynchronize(s));
  return RV_OK;
}

rv_status rv_trainer_step(rv_trainer* tr, const float* patches, const float* codec, const float* gumbel, int32_t B,
                          float tau, rv_train_log* log, void* stream) {
  rv_status st = check_io(tr, patches, codec, gumbel, B, tau, true);
  if (st) return st;
  TCK(cudaSetDevice(tr->device));
  cudaStream_t s = (cudaStream_t)stream;
  if ((st = loss_grad(tr, patches, codec, gumbel, B, tau, log, s))) return st;
  tr->steps += 1;
  const double c1 = 1.0 / (1.0 - pow((double)tr->b1, tr->steps)), c2 = 1.0 / (1.0 - pow((double)tr->b2, tr->steps));
  k_adam<<<nblk((long long)tr->go.total), 256, 0, s>>>((long long)tr->go.total, tr->P, tr->dP, tr->am, tr->av, tr->lr,
                                                       tr->b1, tr->b2, tr->eps, (float)c1, (float)c2);
  TCK(cudaGetLastError());
  TCK(cudaStreamSynchronize(s));
  if (log) log->step = tr->steps;
  return RV_OK;
}

rv_status rv_trainer_gates(rv_trainer* tr, float* gate_blob_host) {
  if (!tr || !gate_blob_host) return tfail(tr, RV_ECONTRACT, "rv_trainer_gates: null argument");
  TCK(cudaSetDevice(tr->device));
  TCK(cudaDeviceSynchronize());
  TCK(cudaMemcpy(gate_blob_host, tr->P, tr->go.total * 4, cudaMemcpyDeviceToHost));
  return RV_OK;
}

}  // extern "C"
