// common.cuh — small device helpers shared by the sm_100a kernels of libreusevit.
#pragma once
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

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

// ---- per-device host caches.  Function attributes and SM counts belong to a device, and one
// process may drive several GPUs through one library instance: cache per device, thread-safe.
inline int cur_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 ? 0 : (d & 63);
}
inline int dev_sms() {
  static std::atomic<int> cache[64];
  const int d = cur_device();
  int n = cache[d].load(std::memory_order_relaxed);
  if (!n) {
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, d);
    if (n <= 0) n = 148;
    cache[d].store(n, std::memory_order_relaxed);
  }
  return n;
}
// Raise kernel Kern's dynamic shared-memory limit to >= smem bytes on the current device.
template <auto Kern>
cudaError_t ensure_smem(size_t smem) {
  static std::atomic<size_t> done[64];
  const int d = cur_device();
  if (done[d].load() >= smem) return cudaSuccess;
  cudaError_t e = cudaFuncSetAttribute(Kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  size_t cur = done[d].load();
  while (cur < smem && !done[d].compare_exchange_weak(cur, smem)) {
  }
  return cudaSuccess;
}

}  // namespace rv
