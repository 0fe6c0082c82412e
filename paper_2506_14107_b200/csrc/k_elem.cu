// k_elem.cu — HBM-bound row kernels of the hot path.
//
//   patch_to_bf16 : fp32 patches [rows][pp] -> bf16 GEMM operand [rows][KP] (zero K padding)
//   embed_finish  : X0 = LN_pre(concat(cls, patches W_pe) + pos) in place, t := 1/N
//   gather_ln     : A[m] = bf16(LN(src[rows[m]]))  — gather of recompute rows + LN1/LN2 (a5)
//   ln_post       : Z_f = LN_post(X_L[f][CLS])
// One warp per row; lane j owns elements j, j+32, ... (coalesced 128 B per warp access);
// LN statistics in fp32 with a fixed butterfly reduction order (deterministic).
#include "common.cuh"
#include "rv_internal.h"

namespace rv {
namespace {

constexpr int ROWS_PER_CTA = 8;  // 8 warps

RV_DEV float to_f(float v) { return v; }
RV_DEV float to_f(bf16 v) { return __bfloat162float(v); }
RV_DEV void from_f(float& d, float v) { d = v; }
RV_DEV void from_f(bf16& d, float v) { d = __float2bfloat16_rn(v); }

// XT = float (fp32 residual stream) or bf16 (RV_X_BF16)
template <int VPL, typename XT>
RV_DEV void load_row(const XT* __restrict__ src, int D, int lane, float (&x)[VPL]) {
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    const int k = lane + 32 * j;
    x[j] = k < D ? to_f(src[k]) : 0.f;
  }
}

template <int VPL>
RV_DEV void layer_norm_regs(float (&x)[VPL], int D, int lane, const float* __restrict__ g,
                            const float* __restrict__ b) {
  float s = 0.f;
#pragma unroll
  for (int j = 0; j < VPL; ++j) s += x[j];
  const float mean = warp_sum(s) / (float)D;
  float v = 0.f;
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    const int k = lane + 32 * j;
    const float d = k < D ? x[j] - mean : 0.f;
    v += d * d;
  }
  const float rstd = rsqrtf(warp_sum(v) / (float)D + 1e-5f);
#pragma unroll
  for (int j = 0; j < VPL; ++j) {
    const int k = lane + 32 * j;
    if (k < D) x[j] = (x[j] - mean) * rstd * __ldg(g + k) + __ldg(b + k);
  }
}

__global__ void patch_to_bf16_kernel(const float* __restrict__ src, bf16* __restrict__ dst,
                                     long long rows, int pp, int KP) {
  const long long total = rows * (long long)KP;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total;
       i += (long long)gridDim.x * blockDim.x) {
    const long long r = i / KP;
    const int c = (int)(i - r * KP);
    dst[i] = __float2bfloat16_rn(c < pp ? src[r * pp + c] : 0.f);
  }
}

template <int VPL, typename XT>
__global__ void embed_finish_kernel(XT* __restrict__ X, const float* __restrict__ cls,
                                    const float* __restrict__ pos, const float* __restrict__ g,
                                    const float* __restrict__ b, float* __restrict__ pclsh, int n,
                                    int T, int D, int N, int H) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long rows = (long long)n * T;
  for (long long r = blockIdx.x * (long long)ROWS_PER_CTA + warp; r < rows;
       r += (long long)gridDim.x * ROWS_PER_CTA) {
    const int tok = (int)(r % T);
    XT* row = X + r * D;
    float x[VPL];
    if (tok == 0) load_row<VPL>(cls, D, lane, x);
    else load_row<VPL>(row, D, lane, x);          // patches @ W_pe written by the PE GEMM
    float p[VPL];
    load_row<VPL>(pos + (long long)tok * D, D, lane, p);
#pragma unroll
    for (int j = 0; j < VPL; ++j) x[j] += p[j];
    layer_norm_regs<VPL>(x, D, lane, g, b);
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int k = lane + 32 * j;
      if (k < D) from_f(row[k], x[j]);
    }
    if (tok > 0 && lane < H) pclsh[((r / T) * H + lane) * N + (tok - 1)] = 1.0f / (float)N;  // layer-1 t
  }
}

// RV_LN_MINB: resident CTAs per SM the register allocation must allow (ptxas gave 125 registers
// without a bound: 2 CTAs = 16 warps per SM, 25% occupancy in ncu).  Bench at 7,200 frames
// (gather_ln1 / ln2 ms per step): no bound 15.2 / 14.1, 3 -> 14.2 / 13.7, 4 -> 16.9 / 16.7
// (64 registers spill the 32-value row), 1 -> 22.5 / 20.3
#ifndef RV_LN_MINB
#define RV_LN_MINB 3
#endif
template <int VPL, typename XT>
__global__ void __launch_bounds__(256, RV_LN_MINB) gather_ln_kernel(const XT* __restrict__ src, const int* __restrict__ rows,
                                 const int* __restrict__ count, int M_host, const float* __restrict__ g,
                                 const float* __restrict__ b, bf16* __restrict__ dst, int D) {
  const int M = count ? *count : M_host;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int m = blockIdx.x * ROWS_PER_CTA + warp; m < M; m += gridDim.x * ROWS_PER_CTA) {
    const long long r = rows ? rows[m] : m;
    float x[VPL];
    load_row<VPL>(src + r * D, D, lane, x);
    layer_norm_regs<VPL>(x, D, lane, g, b);
    bf16* o = dst + (long long)m * D;
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int k = lane + 32 * j;
      if (k < D) o[k] = __float2bfloat16_rn(x[j]);
    }
  }
}

// vectorised variant for D = 768 / 1024: lane holds float4 lane + 32 j (columns 4 (lane + 32 j)
// ..), 8 B bf16 stores.  Bench at 7,200 frames (LN1 + LN2 ms per step): 28.2 scalar -> 22.0
#ifndef RV_LN_VEC
#define RV_LN_VEC 1
#endif
template <int V4, typename XT>
__global__ void __launch_bounds__(256, RV_LN_MINB) gather_ln_vec_kernel(const XT* __restrict__ src, const int* __restrict__ rows,
                                     const int* __restrict__ count, int M_host, const float* __restrict__ g,
                                     const float* __restrict__ b, bf16* __restrict__ dst, int D) {
  const int M = count ? *count : M_host;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int m = blockIdx.x * ROWS_PER_CTA + warp; m < M; m += gridDim.x * ROWS_PER_CTA) {
    const long long r = rows ? rows[m] : m;
    float4 x[V4];
    if constexpr (sizeof(XT) == 4) {
      const float4* s4 = reinterpret_cast<const float4*>(src + r * D);
#pragma unroll
      for (int j = 0; j < V4; ++j) x[j] = s4[lane + 32 * j];
    } else {   // bf16 row: 8 B per 4 columns
      const uint2* s2 = reinterpret_cast<const uint2*>(src + r * D);
#pragma unroll
      for (int j = 0; j < V4; ++j) {
        const uint2 u = s2[lane + 32 * j];
        const float2 lo = unpack_bf16x2(u.x), hi = unpack_bf16x2(u.y);
        x[j] = make_float4(lo.x, lo.y, hi.x, hi.y);
      }
    }
    float sum = 0.f;
#pragma unroll
    for (int j = 0; j < V4; ++j) sum += (x[j].x + x[j].y) + (x[j].z + x[j].w);
    const float mean = warp_sum(sum) / (float)D;
    float v = 0.f;
#pragma unroll
    for (int j = 0; j < V4; ++j) {
      const float a = x[j].x - mean, bq = x[j].y - mean, c = x[j].z - mean, d = x[j].w - mean;
      v += (a * a + bq * bq) + (c * c + d * d);
    }
    const float rstd = rsqrtf(warp_sum(v) / (float)D + 1e-5f);
    uint2* o = reinterpret_cast<uint2*>(dst + (long long)m * D);
#pragma unroll
    for (int j = 0; j < V4; ++j) {
      const float4 gg = __ldg(reinterpret_cast<const float4*>(g) + lane + 32 * j);
      const float4 bb = __ldg(reinterpret_cast<const float4*>(b) + lane + 32 * j);
      o[lane + 32 * j] = make_uint2(pack_bf16x2((x[j].x - mean) * rstd * gg.x + bb.x, (x[j].y - mean) * rstd * gg.y + bb.y),
                                    pack_bf16x2((x[j].z - mean) * rstd * gg.z + bb.z, (x[j].w - mean) * rstd * gg.w + bb.w));
    }
  }
}

template <int VPL, typename XT>
__global__ void ln_post_kernel(const XT* __restrict__ X, const float* __restrict__ g,
                               const float* __restrict__ b, float* __restrict__ emb, int n, int T,
                               int D) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int f = blockIdx.x * ROWS_PER_CTA + warp; f < n; f += gridDim.x * ROWS_PER_CTA) {
    float x[VPL];
    load_row<VPL>(X + (long long)f * T * D, D, lane, x);
    layer_norm_regs<VPL>(x, D, lane, g, b);
#pragma unroll
    for (int j = 0; j < VPL; ++j) {
      const int k = lane + 32 * j;
      if (k < D) emb[(long long)f * D + k] = x[j];
    }
  }
}

int grid_rows(long long rows) {
  long long g = (rows + ROWS_PER_CTA - 1) / ROWS_PER_CTA;
  if (g > 148 * 16) g = 148 * 16;
  return g < 1 ? 1 : (int)g;
}

}  // namespace

// one warp per patch row, float4 loads and 8 B bf16 stores (pp % 4 == 0), zero padding to KP
__global__ void __launch_bounds__(256) patch_to_bf16_rows_kernel(const float* __restrict__ src, bf16* __restrict__ dst,
                                                                 long long rows, int pp, int KP) {
  const int lane = threadIdx.x & 31;
  for (long long r = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5; r < rows;
       r += ((long long)gridDim.x * blockDim.x) >> 5) {
    const float4* s4 = reinterpret_cast<const float4*>(src + r * pp);
    uint2* d2 = reinterpret_cast<uint2*>(dst + r * KP);
    for (int c = lane; c < KP / 4; c += 32) {
      const float4 v = c < pp / 4 ? __ldg(s4 + c) : make_float4(0.f, 0.f, 0.f, 0.f);
      d2[c] = make_uint2(pack_bf16x2(v.x, v.y), pack_bf16x2(v.z, v.w));
    }
  }
}

cudaError_t launch_patch_to_bf16(const float* src, bf16* dst, long long rows, int pp, int KP,
                                 cudaStream_t s) {
  // vectorised path (all CLIP shapes: pp = 3 p^2 with even p) needs 16 B aligned rows: a caller's
  // view with a storage offset that is not a multiple of 4 floats takes the scalar kernel
  if (pp % 4 == 0 && KP % 4 == 0 && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
    long long g = (rows + 7) / 8;
    if (g > 148 * 16) g = 148 * 16;
    patch_to_bf16_rows_kernel<<<(int)(g < 1 ? 1 : g), 256, 0, s>>>(src, dst, rows, pp, KP);
    return cudaGetLastError();
  }
  long long total = rows * KP;
  long long g = (total + 255) / 256;
  if (g > 148 * 32) g = 148 * 32;
  patch_to_bf16_kernel<<<(int)(g < 1 ? 1 : g), 256, 0, s>>>(src, dst, rows, pp, KP);
  return cudaGetLastError();
}

cudaError_t launch_embed_finish(void* X, int x_bf16, const float* cls, const float* pos, const float* g,
                                const float* b, float* pclsh, int n, int T, int D, int N, int H, cudaStream_t s) {
  const int grid = grid_rows((long long)n * T);
  const int v = (D + 31) / 32;
#define RV_EF(V, XT) embed_finish_kernel<V, XT><<<grid, 256, 0, s>>>(reinterpret_cast<XT*>(X), cls, pos, g, b, pclsh, n, T, D, N, H)
  if (x_bf16) {
    if (v <= 2) RV_EF(2, bf16); else if (v <= 24) RV_EF(24, bf16); else RV_EF(32, bf16);
  } else {
    if (v <= 2) RV_EF(2, float); else if (v <= 24) RV_EF(24, float); else RV_EF(32, float);
  }
#undef RV_EF
  return cudaGetLastError();
}

template <typename XT>
cudaError_t gather_ln_t(const XT* src, const int* rows, const int* count, int M_host, int max_rows,
                        const float* g, const float* b, bf16* dst, int D, cudaStream_t s) {
  const int grid = grid_rows(max_rows);
  const int v = (D + 31) / 32;
  if (RV_LN_VEC && D == 1024) {
    gather_ln_vec_kernel<8, XT><<<grid, 256, 0, s>>>(src, rows, count, M_host, g, b, dst, D);
    return cudaGetLastError();
  }
  if (RV_LN_VEC && D == 768) {
    gather_ln_vec_kernel<6, XT><<<grid, 256, 0, s>>>(src, rows, count, M_host, g, b, dst, D);
    return cudaGetLastError();
  }
  if (v <= 2) gather_ln_kernel<2, XT><<<grid, 256, 0, s>>>(src, rows, count, M_host, g, b, dst, D);
  else if (v <= 24) gather_ln_kernel<24, XT><<<grid, 256, 0, s>>>(src, rows, count, M_host, g, b, dst, D);
  else gather_ln_kernel<32, XT><<<grid, 256, 0, s>>>(src, rows, count, M_host, g, b, dst, D);
  return cudaGetLastError();
}

cudaError_t launch_gather_ln(const void* src, int src_bf16, const int* rows, const int* count, int M_host,
                             int max_rows, const float* g, const float* b, bf16* dst, int D, cudaStream_t s) {
  if (src_bf16) return gather_ln_t(reinterpret_cast<const bf16*>(src), rows, count, M_host, max_rows, g, b, dst, D, s);
  return gather_ln_t(reinterpret_cast<const float*>(src), rows, count, M_host, max_rows, g, b, dst, D, s);
}

cudaError_t launch_ln_post(const void* X, int x_bf16, const float* g, const float* b, float* emb, int n, int T, int D,
                           cudaStream_t s) {
  const int grid = grid_rows(n);
  const int v = (D + 31) / 32;
#define RV_LP(V, XT) ln_post_kernel<V, XT><<<grid, 256, 0, s>>>(reinterpret_cast<const XT*>(X), g, b, emb, n, T, D)
  if (x_bf16) {
    if (v <= 2) RV_LP(2, bf16); else if (v <= 24) RV_LP(24, bf16); else RV_LP(32, bf16);
  } else {
    if (v <= 2) RV_LP(2, float); else if (v <= 24) RV_LP(24, float); else RV_LP(32, float);
  }
#undef RV_LP
  return cudaGetLastError();
}

}  // namespace rv
