// Legacy mma.sync (HMMA) throughput probe on sm_100a: independent m16n8k16 bf16 MMAs in
// registers, no memory traffic.  Reports TFLOP/s for 4..16 warps per SM.  Not part of the library.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__global__ void hmma_loop(float* out, int iters) {
  float c[8][4] = {};
  uint32_t a[4] = {threadIdx.x, threadIdx.x * 3u, threadIdx.x * 5u, threadIdx.x * 7u};
  uint32_t b0 = threadIdx.x * 11u, b1 = threadIdx.x * 13u;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
                   : "+f"(c[j][0]), "+f"(c[j][1]), "+f"(c[j][2]), "+f"(c[j][3])
                   : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
  }
  float s = 0;
  for (int j = 0; j < 8; ++j) s += c[j][0] + c[j][1] + c[j][2] + c[j][3];
  if (s == 12345.f) out[0] = s;
}
int main() {
  float* o;
  cudaMalloc(&o, 4);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int warps : {4, 8, 16, 32}) {
    const int iters = 4096;
    hmma_loop<<<sms, warps * 32>>>(o, 16);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    cudaEventRecord(a);
    hmma_loop<<<sms, warps * 32>>>(o, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double flops = 2.0 * 16 * 8 * 16 * 8.0 * iters * warps * sms;
    printf("warps/SM=%2d: %.1f TFLOP/s (mma.sync m16n8k16 bf16)\n", warps, flops / ms / 1e9);
  }
  return 0;
}
