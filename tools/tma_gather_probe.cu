// tma_gather_probe.cu — which TMA forms can gather K/V rows straight into a SWIZZLE_128B tile?
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o build/tma_gather_probe tools/tma_gather_probe.cu -lcuda
//   build/tma_gather_probe <mode>   (one mode per process: a faulting mode kills the context)
// A [R][128] bf16 matrix (value = row * 1000 + col) is read by three TMA variants into a
// 1024 B-aligned shared tile of 8 rows x 128 B; the tile is compared with the SWIZZLE_128B
// layout (16 B chunk c of row r at chunk c ^ (r & 7)) of rows {5, 17, 3, 40, 9, 22, 31, 0}.
//   mode 0: 2D tile box {64, 1}, one copy per row at dst + 128 r
//   mode 1: tile::gather4 box {64, 1}, two copies of 4 rows at dst + 512 g
//   mode 2: tile::gather4 box {64, 4}
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void probe(const __grid_constant__ CUtensorMap tm, int mode, uint16_t* out) {
  __shared__ __align__(1024) uint16_t tile[8 * 64];
  __shared__ __align__(8) uint64_t bar;
  const int rows[8] = {5, 17, 3, 40, 9, 22, 31, 0};
  for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) tile[i] = 0xFFFF;
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(1024) : "memory");
    if (mode == 0) {
      for (int r = 0; r < 8; ++r)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                su32(tile) + r * 128),
            "l"(&tm), "r"(0), "r"(rows[r]), "r"(su32(&bar))
            : "memory");
    } else {
      for (int g = 0; g < 2; ++g)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
            "%5, %6}], [%7];" ::"r"(su32(tile) + g * 512),
            "l"(&tm), "r"(0), "r"(rows[4 * g]), "r"(rows[4 * g + 1]), "r"(rows[4 * g + 2]), "r"(rows[4 * g + 3]),
            "r"(su32(&bar))
            : "memory");
    }
    uint32_t ok = 0;
    long spins = 0;
    while (!ok && spins < 100000000) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\tselp.u32 %0, 1, 0, p;\n\t}"
          : "=r"(ok)
          : "r"(su32(&bar))
          : "memory");
      ++spins;
    }
    out[8 * 64] = ok ? 1 : 0;
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 8 * 64; i += blockDim.x) out[i] = tile[i];
}

int main(int argc, char** argv) {
  const int only = argc > 1 ? atoi(argv[1]) : -1;
  const int R = 64, C = 128;   // bf16 elements per row: 128 (256 B); the box reads cols 0..63
  uint16_t* h = new uint16_t[R * C];
  for (int r = 0; r < R; ++r)
    for (int c = 0; c < C; ++c) h[r * C + c] = (uint16_t)(r * 256 + c);   // exact in uint16
  void* d;
  cudaMalloc(&d, R * C * 2);
  cudaMemcpy(d, h, R * C * 2, cudaMemcpyHostToDevice);
  uint16_t* dout;
  cudaMalloc(&dout, (8 * 64 + 1) * 2);
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  EncodeFn enc = (EncodeFn)fn;
  const int rows_expected[8] = {5, 17, 3, 40, 9, 22, 31, 0};
  for (int mode = 0; mode < 3; ++mode) {
    if (only >= 0 && mode != only) continue;
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)C, (cuuint64_t)R};
    cuuint64_t strides[1] = {(cuuint64_t)C * 2};
    cuuint32_t box[2] = {64, mode == 2 ? 4u : 1u};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, d, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("mode %d: encode failed %d\n", mode, (int)r);
      continue;
    }
    cudaMemset(dout, 0, (8 * 64 + 1) * 2);
    probe<<<1, 128>>>(tm, mode, dout);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("mode %d: kernel error %s\n", mode, cudaGetErrorString(e));
      return 1;   // context is dead after a fault
    }
    uint16_t o[8 * 64 + 1];
    cudaMemcpy(o, dout, sizeof o, cudaMemcpyDeviceToHost);
    int bad_sw = 0, bad_lin = 0;
    for (int rr = 0; rr < 8; ++rr)
      for (int c = 0; c < 64; ++c) {
        const uint16_t want = (uint16_t)(rows_expected[rr] * 256 + c);
        const int chunk = c / 8, within = c % 8;
        if (o[rr * 64 + ((chunk ^ (rr & 7)) * 8) + within] != want) ++bad_sw;
        if (o[rr * 64 + c] != want) ++bad_lin;
      }
    printf("mode %d: barrier %s, mismatches vs swizzled layout %d, vs linear layout %d\n", mode,
           o[8 * 64] ? "completed" : "TIMED OUT", bad_sw, bad_lin);
  }
  return 0;
}
