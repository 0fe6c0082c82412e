// k_attn.cu — attention of the compacted queries over all T keys of their frame
// (SURVEY §8(a) a8).  Every recomputed query attends to all tokens of its frame (P:313:
// attention "involves interactions among all tokens"); reused tokens contribute the K/V
// copied from their provider (a7).  One CTA = (64 compacted query rows of one frame, one
// head): K, V of that frame/head staged in shared memory, S = Q K^T and O = P V on the
// tensor cores (mma.sync m16n8k16 bf16, fp32 accumulate), online softmax in fp32 with
// exp2 and max subtraction.  Queries are variable per frame (qoff from the compaction
// kernel, read on the device); CTAs past a frame's query count exit at once.
//
// cls_prob_kernel: t for the next layer = head-mean of the CLS softmax row over the patch
// keys ("attention weights from the class token"), fp32, fixed summation
// order over heads (deterministic).
#include "common.cuh"
#include "rv_internal.h"

namespace rv {
namespace {

constexpr int QT = 64;   // query rows per CTA (4 warps x 16)
constexpr int KB = 64;   // keys per online-softmax block

RV_DEV void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <int DH>
__global__ void __launch_bounds__(128)
    attn_kernel(const bf16* __restrict__ q, const bf16* __restrict__ KV, bf16* __restrict__ out,
                const int4* __restrict__ wdesc, const int* __restrict__ qoff, int T, int D,
                float scale_log2) {
  constexpr int KS = DH + 8;  // padded row stride (bf16) of Ks / Qs: conflict-free fragments
  const int w = blockIdx.z, h = blockIdx.y, qt = blockIdx.x;
  const int q0 = qoff[w];
  const int nq = qoff[w + 1] - q0;
  if (qt * QT >= nq) return;
  const int slot = wdesc[w].x;
  const int Tp = (T + KB - 1) / KB * KB;
  extern __shared__ __align__(16) unsigned char attn_smem[];
  bf16* Ks = reinterpret_cast<bf16*>(attn_smem);  // [Tp][KS]
  bf16* Vs = Ks + Tp * KS;                        // [Tp][KS]
  bf16* Qs = Vs + Tp * KS;                        // [QT][KS]
  const long long ld = 2LL * D;
  const bf16* Kg = KV + (long long)slot * T * ld + h * DH;
  const bf16* Vg = Kg + D;
  constexpr int CH = DH / 8;  // 16-byte chunks per row
  const uint4 zero = make_uint4(0, 0, 0, 0);
  for (int idx = threadIdx.x; idx < Tp * CH; idx += blockDim.x) {
    const int j = idx / CH, c = idx % CH;
    const uint4 kv = j < T ? *reinterpret_cast<const uint4*>(Kg + j * ld + c * 8) : zero;
    *reinterpret_cast<uint4*>(Ks + j * KS + c * 8) = kv;
    const uint4 vv = j < T ? *reinterpret_cast<const uint4*>(Vg + j * ld + c * 8) : zero;
    *reinterpret_cast<uint4*>(Vs + j * KS + c * 8) = vv;
  }
  for (int idx = threadIdx.x; idx < QT * CH; idx += blockDim.x) {
    const int r = idx / CH, c = idx % CH;
    const int row = qt * QT + r;
    const uint4 qv = row < nq ? *reinterpret_cast<const uint4*>(q + (long long)(q0 + row) * D + h * DH + c * 8) : zero;
    *reinterpret_cast<uint4*>(Qs + r * KS + c * 8) = qv;
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int r0 = warp * 16;
  uint32_t qa[DH / 16][4];
#pragma unroll
  for (int kk = 0; kk < DH / 16; ++kk) {
    qa[kk][0] = *reinterpret_cast<const uint32_t*>(Qs + (r0 + g) * KS + kk * 16 + 2 * tq);
    qa[kk][1] = *reinterpret_cast<const uint32_t*>(Qs + (r0 + g + 8) * KS + kk * 16 + 2 * tq);
    qa[kk][2] = *reinterpret_cast<const uint32_t*>(Qs + (r0 + g) * KS + kk * 16 + 8 + 2 * tq);
    qa[kk][3] = *reinterpret_cast<const uint32_t*>(Qs + (r0 + g + 8) * KS + kk * 16 + 8 + 2 * tq);
  }
  float o[DH / 8][4];
#pragma unroll
  for (int i = 0; i < DH / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  for (int kb = 0; kb < Tp; kb += KB) {
    float s[KB / 8][4];
#pragma unroll
    for (int j = 0; j < KB / 8; ++j) {
      s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < DH / 16; ++kk) {
        const bf16* kr = Ks + (kb + j * 8 + g) * KS + kk * 16 + 2 * tq;
        mma16816(s[j], qa[kk], *reinterpret_cast<const uint32_t*>(kr), *reinterpret_cast<const uint32_t*>(kr + 8));
      }
      const int col = kb + j * 8 + 2 * tq;
      if (col >= T) { s[j][0] = -INFINITY; s[j][2] = -INFINITY; }
      if (col + 1 >= T) { s[j][1] = -INFINITY; s[j][3] = -INFINITY; }
    }
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int j = 0; j < KB / 8; ++j) {
      mx0 = fmaxf(mx0, fmaxf(s[j][0], s[j][1]));
      mx1 = fmaxf(mx1, fmaxf(s[j][2], s[j][3]));
    }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
    const float a0 = exp2f((m0 - mn0) * scale_log2), a1 = exp2f((m1 - mn1) * scale_log2);
    const float ms0 = mn0 * scale_log2, ms1 = mn1 * scale_log2;
    float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
    for (int j = 0; j < KB / 8; ++j) {
      s[j][0] = exp2f(fmaf(s[j][0], scale_log2, -ms0));
      s[j][1] = exp2f(fmaf(s[j][1], scale_log2, -ms0));
      s[j][2] = exp2f(fmaf(s[j][2], scale_log2, -ms1));
      s[j][3] = exp2f(fmaf(s[j][3], scale_log2, -ms1));
      rs0 += s[j][0] + s[j][1];
      rs1 += s[j][2] + s[j][3];
    }
    l0 = l0 * a0 + rs0;
    l1 = l1 * a1 + rs1;
    m0 = mn0;
    m1 = mn1;
#pragma unroll
    for (int i = 0; i < DH / 8; ++i) {
      o[i][0] *= a0; o[i][1] *= a0; o[i][2] *= a1; o[i][3] *= a1;
    }
#pragma unroll
    for (int kk = 0; kk < KB / 16; ++kk) {
      uint32_t pa[4];
      pa[0] = pack_bf16x2(s[2 * kk][0], s[2 * kk][1]);
      pa[1] = pack_bf16x2(s[2 * kk][2], s[2 * kk][3]);
      pa[2] = pack_bf16x2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
      pa[3] = pack_bf16x2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
      for (int dt = 0; dt < DH / 8; dt += 2) {
        // B fragments of V (row-major [key][dh]) via ldmatrix.trans: lanes 0-15 address keys
        // kb+16kk+0..15 at column block dt, lanes 16-31 the same keys at column block dt+1.
        const bf16* vr = Vs + (kb + kk * 16 + (lane & 15)) * KS + (dt + (lane >> 4)) * 8;
        uint32_t b0, b1, b2, b3;
        asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                     : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3)
                     : "r"((uint32_t)__cvta_generic_to_shared(vr)));
        mma16816(o[dt], pa, b0, b1);
        mma16816(o[dt + 1], pa, b2, b3);
      }
    }
  }
  l0 += __shfl_xor_sync(0xffffffffu, l0, 1);
  l0 += __shfl_xor_sync(0xffffffffu, l0, 2);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 1);
  l1 += __shfl_xor_sync(0xffffffffu, l1, 2);
  const float il0 = 1.f / l0, il1 = 1.f / l1;
  const int ra = qt * QT + r0 + g, rb = ra + 8;
#pragma unroll
  for (int dt = 0; dt < DH / 8; ++dt) {
    const int col = h * DH + dt * 8 + 2 * tq;
    if (ra < nq)
      *reinterpret_cast<uint32_t*>(out + (long long)(q0 + ra) * D + col) = pack_bf16x2(o[dt][0] * il0, o[dt][1] * il0);
    if (rb < nq)
      *reinterpret_cast<uint32_t*>(out + (long long)(q0 + rb) * D + col) = pack_bf16x2(o[dt][2] * il1, o[dt][3] * il1);
  }
}

__global__ void cls_prob_kernel(const bf16* __restrict__ q, const bf16* __restrict__ KV,
                                const int4* __restrict__ wdesc, const int* __restrict__ qoff,
                                float* __restrict__ pcls, int T, int D, int H, int DH, float scale) {
  extern __shared__ float cls_smem[];
  float* qs = cls_smem;            // [H][DH]
  float* ps = qs + H * DH;         // [H][T]
  const int w = blockIdx.x;
  const int slot = wdesc[w].x;
  const long long ld = 2LL * D;
  const bf16* qrow = q + (long long)qoff[w] * D;   // first compact row of the frame = CLS
  for (int k = threadIdx.x; k < D; k += blockDim.x) qs[k] = __bfloat162float(qrow[k]);
  __syncthreads();
  const int h = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (h < H) {
    const float* qh = qs + h * DH;
    const bf16* Kb = KV + (long long)slot * T * ld + h * DH;
    float mx = -INFINITY;
    for (int j = lane; j < T; j += 32) {
      const bf16* kr = Kb + j * ld;
      float acc = 0.f;
      for (int k = 0; k < DH; k += 8) {
        const uint4 u = *reinterpret_cast<const uint4*>(kr + k);
        const float2 a = unpack_bf16x2(u.x), b = unpack_bf16x2(u.y), c = unpack_bf16x2(u.z), d = unpack_bf16x2(u.w);
        acc += qh[k] * a.x + qh[k + 1] * a.y + qh[k + 2] * b.x + qh[k + 3] * b.y + qh[k + 4] * c.x +
               qh[k + 5] * c.y + qh[k + 6] * d.x + qh[k + 7] * d.y;
      }
      acc *= scale;
      ps[h * T + j] = acc;
      mx = fmaxf(mx, acc);
    }
    mx = warp_max(mx);
    float sum = 0.f;
    for (int j = lane; j < T; j += 32) {
      const float e = expf(ps[h * T + j] - mx);
      ps[h * T + j] = e;
      sum += e;
    }
    sum = warp_sum(sum);
    const float inv = 1.f / sum;
    for (int j = lane; j < T; j += 32) ps[h * T + j] *= inv;
  }
  __syncthreads();
  const int N = T - 1;
  for (int j = 1 + threadIdx.x; j < T; j += blockDim.x) {
    float acc = 0.f;
    for (int hh = 0; hh < H; ++hh) acc += ps[hh * T + j];
    pcls[(long long)slot * N + j - 1] = acc / (float)H;
  }
}

template <int DH>
cudaError_t launch_attn_dh(const bf16* q, const bf16* KV, bf16* out, const int* wdesc, const int* qoff, int n_w,
                           int T, int D, int H, cudaStream_t s) {
  const int Tp = (T + KB - 1) / KB * KB;
  const size_t smem = (size_t)(2 * Tp * (DH + 8) + QT * (DH + 8)) * sizeof(bf16);
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_kernel<DH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  dim3 grid((T + QT - 1) / QT, H, n_w);
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)DH);
  attn_kernel<DH><<<grid, 128, smem, s>>>(q, KV, out, reinterpret_cast<const int4*>(wdesc), qoff, T, D, scale_log2);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attention(const bf16* q, const bf16* KV, bf16* out, const int* wdesc, const int* qoff, int n_w,
                             int T, int D, int H, cudaStream_t s) {
  if (n_w <= 0) return cudaSuccess;
  const int dh = D / H;
  if (dh == 64) return launch_attn_dh<64>(q, KV, out, wdesc, qoff, n_w, T, D, H, s);
  if (dh == 16) return launch_attn_dh<16>(q, KV, out, wdesc, qoff, n_w, T, D, H, s);
  return cudaErrorInvalidValue;
}

cudaError_t launch_cls_prob(const bf16* q, const bf16* KV, const int* wdesc, const int* qoff, float* pcls, int n_w,
                            int T, int D, int H, cudaStream_t s) {
  if (n_w <= 0) return cudaSuccess;
  const int dh = D / H;
  const size_t smem = (size_t)(H * dh + H * T) * sizeof(float);
  static size_t attr = 0;
  if (smem > 48 * 1024 && smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(cls_prob_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  cls_prob_kernel<<<n_w, 32 * H, smem, s>>>(q, KV, reinterpret_cast<const int4*>(wdesc), qoff, pcls, T, D, H, dh,
                                            1.f / sqrtf((float)dh));
  return cudaGetLastError();
}

}  // namespace rv
