// Attention microbenchmark: times rv::launch_attention (k_attn.cu) on a synthetic wave.
// Built three times by tools/attn_bench.sh with -DRV_ATTN_NO_LOAD / -DRV_ATTN_NO_MMA to split
// load-bound from compute-bound time.  Not part of the library.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include "../paper_2506_14107_b200/csrc/k_attn.cu"

int main(int argc, char** argv) {
  const int T = 257, D = 1024, H = 16;
  const int n_w = argc > 1 ? atoi(argv[1]) : 1440;
  const int nq = argc > 2 ? atoi(argv[2]) : 57;
  std::vector<int> qoff(n_w + 1), wd(n_w * 4, 0);
  for (int i = 0; i <= n_w; ++i) qoff[i] = i * nq;
  for (int i = 0; i < n_w; ++i) wd[i * 4] = i;
  rv::bf16 *q, *KV, *out;
  int *dq, *dwd;
  float* pcl;
  cudaMalloc(&q, (size_t)n_w * nq * D * 2);
  cudaMalloc(&out, (size_t)n_w * nq * D * 2);
  cudaMalloc(&KV, (size_t)n_w * T * 2 * D * 2);
  cudaMemset(q, 0, (size_t)n_w * nq * D * 2);
  cudaMemset(KV, 0, (size_t)n_w * T * 2 * D * 2);
  cudaMalloc(&pcl, (size_t)n_w * H * (T - 1) * 4);
  cudaMalloc(&dq, (n_w + 1) * 4);
  cudaMalloc(&dwd, n_w * 16);
  cudaMemcpy(dq, qoff.data(), (n_w + 1) * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dwd, wd.data(), n_w * 16, cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int i = 0; i < 3; ++i) rv::launch_attention(q, KV, nullptr, out, dwd, dq, pcl, n_w, T, D, H, 0);
  cudaEventRecord(a);
  for (int i = 0; i < 10; ++i) rv::launch_attention(q, KV, nullptr, out, dwd, dq, pcl, n_w, T, D, H, 0);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  ms /= 10;
  const double flops = 4.0 * n_w * nq * T * D, bytes = (double)n_w * T * 2 * D * 2;
  printf("n_w=%d nq=%d: %.3f ms  %.1f TFLOP/s  %.0f GB/s (K/V)  err=%s\n", n_w, nq, ms, flops / ms / 1e9,
         bytes / ms / 1e6, cudaGetErrorString(cudaGetLastError()));
  return 0;
}
