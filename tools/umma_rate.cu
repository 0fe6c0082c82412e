// umma_rate.cu — issue/complete rate of single-CTA tcgen05.mma (kind::f16, bf16 in, fp32 acc)
// for the attention shapes: M in {64, 128}, N in {64, 128, 256}, A from SMEM (ss) or TMEM (ts).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/umma_rate tools/umma_rate.cu
// One CTA per SM (148), one thread issues `reps` MMAs back to back (accumulate), then commits;
// prints cycles per MMA for issue (loop) and for completion (commit observed), and the
// aggregate TFLOP/s across the grid (operands are zero: only timing matters).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t sdesc(uint32_t addr) {
  return ((uint64_t)((addr >> 4) & 0x3FFF)) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
__device__ __forceinline__ uint32_t idesc(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__global__ void bench(int M, int N, int ts, int reps, int nd, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar;
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  if (threadIdx.x == 0) {
    const uint32_t id = idesc(M, N);
    const uint64_t a = sdesc(su32(sm)), b = sdesc(su32(sm) + 32768);
    unsigned long long t0 = clock64();
    const uint32_t dstep = (N <= 64 ? 64 : 128);
    const uint32_t d0 = ts ? tmem + 256 : tmem;
    const uint32_t d1 = d0 + (nd > 1 ? dstep : 0), d2 = d0 + (nd > 2 ? 2 * dstep : 0), d3 = d0 + (nd > 3 ? 3 * dstep : 0);
    for (int r = 0; r < reps; r += 4) {
      if (ts) {
#define MMA_TS(D) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(D), "r"(tmem), "l"(b), "r"(id), "r"(1))
        MMA_TS(d0); MMA_TS(d1); MMA_TS(d2); MMA_TS(d3);
      } else {
#define MMA_SS(D) asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(D), "l"(a), "l"(b), "r"(id), "r"(1))
        MMA_SS(d0); MMA_SS(d1); MMA_SS(d2); MMA_SS(d3);
      }
    }
    unsigned long long t1 = clock64();
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar))
                 : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(su32(&bar))
          : "memory");
    unsigned long long t2 = clock64();
    if (blockIdx.x == 0) {
      out[0] = t1 - t0;
      out[1] = t2 - t0;
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const int reps = 4096;
  const int shapes[][4] = {{64, 64, 0, 1}, {64, 64, 0, 4}, {64, 64, 1, 1}, {64, 64, 1, 4}, {128, 64, 0, 1},
                           {128, 64, 0, 4}, {128, 128, 0, 1}, {128, 128, 0, 2}, {128, 256, 0, 1}, {64, 256, 0, 1},
                           {128, 128, 1, 1}, {128, 128, 1, 2}, {128, 256, 1, 1}};
  for (auto& s : shapes) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    bench<<<148, 128, 96 * 1024>>>(s[0], s[1], s[2], reps, s[3], d);
    cudaEventRecord(e0);
    bench<<<148, 128, 96 * 1024>>>(s[0], s[1], s[2], reps, s[3], d);
    cudaEventRecord(e1);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("M=%d N=%d %s: %s\n", s[0], s[1], s[2] ? "ts" : "ss", cudaGetErrorString(e));
      return 1;
    }
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * s[0] * s[1] * 16 * reps * 148;
    printf("nd=%d M=%3d N=%3d %s: issue %.1f cyc/mma, complete %.1f cyc/mma, %.0f TFLOP/s\n", s[3], s[0], s[1],
           s[2] ? "ts" : "ss", (double)h[0] / reps, (double)h[1] / reps, flops / ms / 1e9);
  }
  return 0;
}
