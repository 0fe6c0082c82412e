// umma_issuers.cu — does the tcgen05.mma issue cost (~93+ cycles per instruction from one
// thread, tools/umma_rate.cu) shrink when several warps issue concurrently into disjoint TMEM
// accumulators of the same CTA?  If yes, the attention kernels (issue-bound on their many
// small N = 64 / 96 MMAs) should give each softmax group its own MMA-issuing warp.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/umma_issuers tools/umma_issuers.cu
// One CTA per SM (148); W issuing warps (lane 0 of warps 0..W-1) each issue `reps` MMAs
// (accumulate) into their own TMEM column range, then commit to their own mbarrier; prints the
// aggregate cycles per MMA (slowest warp's cycles / (W * reps)) and the grid's TFLOP/s.
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

__global__ void bench(int M, int N, int ts, int reps, int W, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t tslot;
  __shared__ __align__(8) uint64_t bar[8];
  __shared__ unsigned long long t_end[8];
  for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    for (int i = 0; i < 8; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[i])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tslot;
  const unsigned long long t0 = clock64();
  if (warp < W && lane == 0) {
    const uint32_t id = idesc(M, N);
    const uint64_t a = sdesc(su32(sm)), b = sdesc(su32(sm) + 32768);
    // accumulators: columns [base + w * span, + N); ts mode keeps columns [0, 64) for A
    const uint32_t base = ts ? 64 : 0, span = (512 - base) / W;
    const uint32_t d = tmem + base + (uint32_t)warp * span;
    for (int r = 0; r < reps; ++r) {
      if (ts)
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}"
                     ::"r"(d), "r"(tmem), "l"(b), "r"(id), "r"(1));
      else
        asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\ttcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}"
                     ::"r"(d), "l"(a), "l"(b), "r"(id), "r"(1));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar[warp]))
                 : "memory");
    uint32_t ok = 0;
    while (!ok)
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(su32(&bar[warp]))
          : "memory");
    t_end[warp] = clock64() - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    unsigned long long mx = 0;
    for (int w = 0; w < W; ++w) mx = t_end[w] > mx ? t_end[w] : mx;
    out[0] = mx;
  }
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

int main() {
  unsigned long long* d;
  cudaMalloc(&d, 16);
  cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
  const int reps = 2048;
  // M, N, ts
  const int shapes[][3] = {{128, 64, 1}, {128, 96, 0}, {128, 64, 0}, {64, 64, 1}, {64, 256, 0}, {128, 128, 0},
                           {128, 256, 0}};
  for (auto& s : shapes) {
    for (int W = 1; W <= 4; W *= 2) {
      if (s[1] * W > (s[2] ? 448 : 512)) continue;
      bench<<<148, 128, 96 * 1024>>>(s[0], s[1], s[2], reps, W, d);
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      bench<<<148, 128, 96 * 1024>>>(s[0], s[1], s[2], reps, W, d);
      cudaEventRecord(e1);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("M=%d N=%d W=%d: %s\n", s[0], s[1], W, cudaGetErrorString(e));
        return 1;
      }
      unsigned long long h;
      cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double flops = 2.0 * s[0] * s[1] * 16 * reps * 148.0 * W;
      printf("M=%3d N=%3d %s issuers %d: %.1f cyc per MMA (aggregate), %.0f TFLOP/s\n", s[0], s[1],
             s[2] ? "ts" : "ss", W, (double)h / (reps * W), flops / ms / 1e9);
    }
  }
  return 0;
}
