// gather_rate.cu — how fast can one SM gather scattered 128 B K/V rows into shared memory?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o build/gather_rate tools/gather_rate.cu -lcuda
//   build/gather_rate
// A [R][2048] bf16 matrix (4 KB rows, like the [n][T][2D] K/V cache at D = 1024) of 4 GB (> L2).
// Persistent CTAs (one per SM) fill 32 KB tiles of 256 rows x 128 B (row indices drawn from a
// hash, column block = a head's 128 B) into a ring of NSLOT tiles and release them as soon as
// they complete (no compute), so the number is the pure gather rate.  Modes:
//   0: cp.async 16 B from LW loader warps (8 lanes per row), completion by arrive.noinc
//   1: cp.async.bulk 128 B per row (one row per lane), complete_tx on the slot's mbarrier
//   2: TMA 2D tile box {64, 1} per row (tensor map over the matrix, SWIZZLE_128B)
//   3: TMA tile::gather4 box {64, 1} (4 rows per instruction)
// Prints GB/s of delivered bytes for each mode and loader-warp count.
#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint32_t a, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                 : "=r"(ok) : "r"(a), "r"(parity) : "memory");
}
__device__ __forceinline__ uint32_t hrow(uint32_t x, uint32_t R) {
  return (x * 2654435761u) & (R - 1);   // R is a power of two: a cheap scatter
}

constexpr int NSLOT = 6;
constexpr uint32_t TILE = 256 * 128;

__global__ void __launch_bounds__(512, 1) gather(const __grid_constant__ CUtensorMap tm, const uint16_t* __restrict__ M,
                                                 uint32_t R, int tiles_per_cta, int mode, int lw, unsigned long long* sink, int seg) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ __align__(8) uint64_t full[NSLOT];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NSLOT; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[i])), "r"(mode == 0 ? lw * 32 : 1));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t base = su32(sm);
  if (warp < lw) {
    for (int t = 0; t < tiles_per_cta; ++t) {
      const int s = t % NSLOT;
      if (t >= NSLOT) mbar_wait(su32(&full[s]), ((t / NSLOT) - 1) & 1);   // slot free once it completed
      const uint32_t dst = base + s * TILE;
      const uint32_t seed = (blockIdx.x * 100003u + t) * 256u;
      const int head = (blockIdx.x + t) & 15;
      if (mode == 0) {
        // seg B contiguous per gathered row (seg / 16 lanes per row), TILE / seg rows per tile
        const int lpr = seg >> 4, rpw = 32 / lpr, nrow = TILE / seg;
        const int c = lane % lpr;
        const int hseg = head % (4096 / seg);
        for (int r = warp * rpw + lane / lpr; r < nrow; r += rpw * lw) {
          const uint32_t row = hrow(seed + r, R);
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + r * seg + (((c & 7) ^ (r & 7)) << 4) + ((c >> 3) << 7)),
                       "l"(M + (size_t)row * 2048 + hseg * (seg / 2) + c * 8) : "memory");
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&full[s])) : "memory");
      } else {
        if (warp == 0 && lane == 0)
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(TILE) : "memory");
        if (mode == 1) {
          for (int r = warp * 32 + lane; r < 256; r += 32 * lw) {
            const uint32_t row = hrow(seed + r, R);
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];" ::"r"(
                             dst + r * 128), "l"(M + (size_t)row * 2048 + head * 64), "r"(su32(&full[s])) : "memory");
          }
        } else if (mode == 2) {
          for (int r = warp * 32 + lane; r < 256; r += 32 * lw) {
            const uint32_t row = hrow(seed + r, R);
            asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                         ::"r"(dst + r * 128), "l"(&tm), "r"(head * 64), "r"(row), "r"(su32(&full[s])) : "memory");
          }
        } else {
          for (int g = warp * 32 + lane; g < 64; g += 32 * lw) {
            const uint32_t r0 = hrow(seed + 4 * g, R), r1 = hrow(seed + 4 * g + 1, R), r2 = hrow(seed + 4 * g + 2, R),
                           r3 = hrow(seed + 4 * g + 3, R);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
                "%5, %6}], [%7];" ::"r"(dst + g * 512), "l"(&tm), "r"(head * 64), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
                "r"(su32(&full[s])) : "memory");
          }
        }
      }
    }
    // drain
    for (int t = tiles_per_cta > NSLOT ? tiles_per_cta - NSLOT : 0; t < tiles_per_cta; ++t)
      mbar_wait(su32(&full[t % NSLOT]), (t / NSLOT) & 1);
  }
  __syncthreads();
  if (threadIdx.x == 0) sink[blockIdx.x] = *(volatile unsigned long long*)(sm + 8);
}

int main() {
  const uint32_t R = 1u << 20;   // 1 Mi rows x 4 KB = 4 GB
  uint16_t* d;
  if (cudaMalloc(&d, (size_t)R * 4096) != cudaSuccess) { printf("alloc failed\n"); return 1; }
  cudaMemset(d, 1, (size_t)R * 4096);
  unsigned long long* sink;
  cudaMalloc(&sink, 1024 * 8);
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  cuuint64_t dims[2] = {2048, R};
  cuuint64_t strides[1] = {4096};
  cuuint32_t box[2] = {64, 1};
  cuuint32_t es[2] = {1, 1};
  if (((EncodeFn)fn)(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    printf("encode failed\n");
    return 1;
  }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const size_t smem = NSLOT * TILE;
  cudaFuncSetAttribute(gather, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int tiles = 400;
  const char* names[4] = {"cp.async 16B", "cp.async.bulk 128B", "TMA 2D {64,1}", "TMA gather4"};
  for (int mode = 0; mode < 4; ++mode)
    for (int lw = 1; lw <= 16; lw *= 2) {
      gather<<<sms, 512, smem>>>(tm, d, R, 20, mode, lw, sink, 128);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      gather<<<sms, 512, smem>>>(tm, d, R, tiles, mode, lw, sink, 128);
      cudaEventRecord(b);
      cudaError_t e = cudaEventSynchronize(b);
      if (e != cudaSuccess || cudaGetLastError() != cudaSuccess) {
        printf("%s lw=%d: error %s\n", names[mode], lw, cudaGetErrorString(e));
        return 1;
      }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)sms * tiles * TILE;
      printf("%-20s loader warps %d: %.3f ms, %.0f GB/s (%.1f GB/s per SM)\n", names[mode], lw, ms, bytes / ms / 1e6,
             bytes / ms / 1e6 / sms);
    }
  // segment size: K and V of one head adjacent (256 B) or two heads (512 B) per gathered row
  for (int seg = 128; seg <= 512; seg *= 2)
    for (int lw = 2; lw <= 8; lw *= 2) {
      gather<<<sms, 512, smem>>>(tm, d, R, 20, 0, lw, sink, seg);
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a);
      gather<<<sms, 512, smem>>>(tm, d, R, tiles, 0, lw, sink, seg);
      cudaEventRecord(b);
      if (cudaEventSynchronize(b) != cudaSuccess) { printf("seg error\n"); return 1; }
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double bytes = (double)sms * tiles * TILE;
      printf("cp.async 16B seg %4d B  loader warps %d: %.3f ms, %.0f GB/s\n", seg, lw, ms, bytes / ms / 1e6);
    }
  return 0;
}
