// common.cuh — small device helpers shared by the sm_100a kernels of libreusevit.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define RV_DEV __device__ __forceinline__

namespace rv {

typedef __nv_bfloat16 bf16;

RV_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
RV_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
RV_DEV int warp_sum_i(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// QuickGELU(x) = x * sigmoid(1.702 x) (OpenAI-CLIP activation).  expf, not
// __expf: the decision logit's sign is compared with the oracle's.
RV_DEV float quick_gelu(float x) { return x / (1.0f + expf(-1.702f * x)); }

// 2^x on the MUFU (ex2.approx.ftz): softmax terms, arguments <= 0.
RV_DEV float ex2f_fast(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

RV_DEV uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);  // RNE (cvt.rn.bf16x2.f32)
  return *reinterpret_cast<uint32_t*>(&h);
}
RV_DEV float2 unpack_bf16x2(uint32_t u) {
  __nv_bfloat162 h = *reinterpret_cast<__nv_bfloat162*>(&u);
  return __bfloat1622float2(h);
}

}  // namespace rv
