// k_attn.cu — attention of the compacted queries over all T keys of their frame
// (SURVEY §8(a) a8).  Every recomputed query attends to all tokens of its frame (P:313:
// attention "involves interactions among all tokens").  Reused tokens contribute the K/V of
// their provider through the kvsrc row table written by the compaction kernel (a7: the reuse
// cache is read in place, chains resolved at write time, no copy).
//
// One CTA = (one frame of the wave, one head), 4 warps x 16 query rows per q-tile, looping
// over all q-tiles of the frame with K/V resident in shared memory:
//   * K/V rows gathered with cp.async (16 B, L2-only) in 64-key commit groups, so the first
//     key blocks are computed while later ones are still in flight;
//   * S = Q K^T and O = P V on the tensor cores (mma.sync m16n8k16 bf16, fp32 accumulate;
//     V fragments via ldmatrix.trans), online softmax in fp32 with exp2 and max subtraction;
//   * the CLS query (first compact row of every frame) additionally emits its normalised
//     softmax row over the patch keys for this head: pclsh[slot][h][j-1];
//     the score kernel of the next layer averages the H heads in a fixed order.
#include "common.cuh"
#include "rv_internal.h"

namespace rv {
namespace {

constexpr int QT = 64;   // query rows per q-tile (4 warps x 16)
constexpr int KB = 64;   // keys per online-softmax block / cp.async commit group

RV_DEV void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
RV_DEV void cp_async16(void* dst, const void* src, bool valid) {
  const uint32_t d = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
RV_DEV void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
RV_DEV void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
template <int DH>
RV_DEV void load_kv_block(bf16* Kb, bf16* Vb, const bf16* __restrict__ KV, const int* rows_s, int k0, int Tp, int T,
                          long long ld, int D, int h, int tid) {
  constexpr int KS = DH + 8, CH = DH / 8;
#ifdef RV_ATTN_NO_LOAD   // microbenchmark hook (tools/attn_bench.cu): compute without K/V traffic
  return;
#endif
  const int nrow = min(KB, Tp - k0);
  for (int idx = tid; idx < nrow * CH; idx += 128) {
    const int j = idx / CH, c = idx % CH;
    const bool ok = k0 + j < T;
    const bf16* kr = KV + (long long)rows_s[k0 + j] * ld + h * 2 * DH + c * 8;   // (k_h v_h) per token
    cp_async16(Kb + j * KS + c * 8, kr, ok);
    cp_async16(Vb + j * KS + c * 8, kr + DH, ok);
  }
}

// One CTA = (frame w of the wave, head h).  Q tile (64 rows) resident; K/V streamed in 64-key
// blocks through a 2-deep cp.async ring (the next block lands while this one is computed), so
// ~45 KB of shared memory per CTA and several CTAs per SM keep the memory system busy.
template <int DH>
__global__ void __launch_bounds__(128)
    attn_kernel(const bf16* __restrict__ q, const bf16* __restrict__ KV, const int* __restrict__ kvsrc,
                bf16* __restrict__ out, const int4* __restrict__ wdesc, const int* __restrict__ qoff,
                float* __restrict__ pclsh, int T, int D, int H, float scale_log2, long long kv_ld, int q_cache) {
  constexpr int KS = DH + 8;     // padded row stride (bf16): conflict-free fragments / ldmatrix
  constexpr int CH = DH / 8;     // 16-byte chunks per row
  const int h = blockIdx.x, w = blockIdx.y;
  const int q0 = qoff[w];
  const int nq = qoff[w + 1] - q0;
  const int slot = wdesc[w].x;
  const int Tp = (T + 15) / 16 * 16;        // keys padded to the mma k-step
  const int nkb = (Tp + KB - 1) / KB;
  extern __shared__ __align__(16) unsigned char attn_smem[];
  bf16* Kr = reinterpret_cast<bf16*>(attn_smem);    // ring [2][KB][KS]
  bf16* Vr = Kr + 2 * KB * KS;                       // ring [2][KB][KS]
  bf16* Qs = Vr + 2 * KB * KS;                       // [QT][KS]
  int* rows_s = reinterpret_cast<int*>(Qs + QT * KS);  // [Tp] K/V source row of every key
  float* scls = reinterpret_cast<float*>(rows_s + Tp); // [Tp] raw CLS logits (q_cls . k_j)
  __shared__ float s_cls[2];                          // CLS row max / sum
  const long long ld = kv_ld;       // K/V cache row stride: 2D ((k_h v_h) per head) or 3D (+ q, chain variant)
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  const int r0 = warp * 16;

  for (int j = tid; j < Tp; j += 128)
    rows_s[j] = j < T ? (kvsrc ? __ldg(kvsrc + (long long)slot * T + j) : slot * T + j) : 0;
  __syncthreads();

  const int ntiles = (nq + QT - 1) / QT;
  for (int qt = 0; qt < ntiles; ++qt) {
    // Q tile + first key block
    for (int idx = tid; idx < QT * CH; idx += 128) {
      const int r = idx / CH, c = idx % CH;
      const int row = qt * QT + r;
      const bool ok = row < nq;
      // q_cache (SPEC chain variant): every token of the frame is a query and its q row lives in
      // the cache next to k and v, read through the same source-row table as the keys
      const bf16* qsrc = q_cache ? KV + (long long)rows_s[ok ? row : 0] * ld + 2 * D + h * DH + c * 8
                                 : q + (long long)(q0 + (ok ? row : 0)) * D + h * DH + c * 8;
      cp_async16(Qs + r * KS + c * 8, qsrc, ok);
    }
    load_kv_block<DH>(Kr, Vr, KV, rows_s, 0, Tp, T, ld, D, h, tid);
    cp_commit();
    const bool active = qt * QT + r0 < nq;   // warp-uniform
    uint32_t qa[DH / 16][4];
    float o[DH / 8][4];
#pragma unroll
    for (int i = 0; i < DH / 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    for (int kb = 0; kb < nkb; ++kb) {
      const int buf = kb & 1;
      if (kb + 1 < nkb) {       // prefetch the next block into the other ring slot
        load_kv_block<DH>(Kr + (buf ^ 1) * KB * KS, Vr + (buf ^ 1) * KB * KS, KV, rows_s, (kb + 1) * KB, Tp, T, ld,
                          D, h, tid);
        cp_commit();
        cp_wait<1>();
      } else {
        cp_wait<0>();
      }
      __syncthreads();
      if (kb == 0 && active) {
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
          qa[kk][0] = *reinterpret_cast<const uint32_t*>(Qs + (r0 + g) * KS + kk * 16 + 2 * tq);
          qa[kk][1] = *reinterpret_cast<const uint32_t*>(Qs + (r0 + g + 8) * KS + kk * 16 + 2 * tq);
          qa[kk][2] = *reinterpret_cast<const uint32_t*>(Qs + (r0 + g) * KS + kk * 16 + 8 + 2 * tq);
          qa[kk][3] = *reinterpret_cast<const uint32_t*>(Qs + (r0 + g + 8) * KS + kk * 16 + 8 + 2 * tq);
        }
      }
#ifdef RV_ATTN_NO_MMA      // microbenchmark hook (tools/attn_bench.cu): K/V traffic only
      if (false) {
#else
      if (active) {
#endif
        const bf16* Ks = Kr + buf * KB * KS;
        const bf16* Vs = Vr + buf * KB * KS;
        const int k0 = kb * KB;
        const int nj = min(KB, Tp - k0) / 8;   // n-tiles of 8 keys in this block (even: Tp % 16 == 0)
        float s[KB / 8][4];
#pragma unroll
        for (int j = 0; j < KB / 8; ++j) s[j][0] = s[j][1] = s[j][2] = s[j][3] = 0.f;
        // S = Q K^T: kk outer so the 8 n-tile accumulators are independent; K fragments of two
        // n-tiles per ldmatrix.x4 (rows = keys, non-transposed)
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk) {
#pragma unroll
          for (int j = 0; j < KB / 8; j += 2) {
            if (j < nj) {
              const bf16* kr = Ks + (j * 8 + (lane & 7) + ((lane >> 4) << 3)) * KS + kk * 16 + ((lane >> 3) & 1) * 8;
              uint32_t b0, b1, b2, b3;
              asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
                           : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3)
                           : "r"((uint32_t)__cvta_generic_to_shared(kr)));
              mma16816(s[j], qa[kk], b0, b1);
              mma16816(s[j + 1], qa[kk], b2, b3);
            }
          }
        }
        if (k0 + KB > T) {      // last block: mask padded keys
#pragma unroll
          for (int j = 0; j < KB / 8; ++j) {
            const int col = k0 + j * 8 + 2 * tq;
            if (j >= nj || col >= T) { s[j][0] = -INFINITY; s[j][2] = -INFINITY; }
            if (j >= nj || col + 1 >= T) { s[j][1] = -INFINITY; s[j][3] = -INFINITY; }
          }
        }
        if (qt == 0 && warp == 0 && g == 0) {   // raw logits of the CLS row (row 0)
#pragma unroll
          for (int j = 0; j < KB / 8; ++j) {
            const int col = k0 + j * 8 + 2 * tq;
            if (j < nj) { scls[col] = s[j][0]; scls[col + 1] = s[j][1]; }
          }
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
        const float a0 = ex2f_fast((m0 - mn0) * scale_log2), a1 = ex2f_fast((m1 - mn1) * scale_log2);
        const float ms0 = mn0 * scale_log2, ms1 = mn1 * scale_log2;
        float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
        for (int j = 0; j < KB / 8; ++j) {
          s[j][0] = ex2f_fast(fmaf(s[j][0], scale_log2, -ms0));
          s[j][1] = ex2f_fast(fmaf(s[j][1], scale_log2, -ms0));
          s[j][2] = ex2f_fast(fmaf(s[j][2], scale_log2, -ms1));
          s[j][3] = ex2f_fast(fmaf(s[j][3], scale_log2, -ms1));
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
          if (2 * kk < nj) {
            uint32_t pa[4];
            pa[0] = pack_bf16x2(s[2 * kk][0], s[2 * kk][1]);
            pa[1] = pack_bf16x2(s[2 * kk][2], s[2 * kk][3]);
            pa[2] = pack_bf16x2(s[2 * kk + 1][0], s[2 * kk + 1][1]);
            pa[3] = pack_bf16x2(s[2 * kk + 1][2], s[2 * kk + 1][3]);
#pragma unroll
            for (int dt = 0; dt < DH / 8; dt += 2) {
              // V fragments (row-major [key][dh]) via ldmatrix.trans: lanes 0-15 address keys
              // 16kk+0..15 at column block dt, lanes 16-31 the same keys at block dt+1.
              const bf16* vr = Vs + (kk * 16 + (lane & 15)) * KS + (dt + (lane >> 4)) * 8;
              uint32_t b0, b1, b2, b3;
              asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
                           : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3)
                           : "r"((uint32_t)__cvta_generic_to_shared(vr)));
              mma16816(o[dt], pa, b0, b1);
              mma16816(o[dt + 1], pa, b2, b3);
            }
          }
        }
      }
      __syncthreads();   // ring slot `buf` is refilled by the next iteration's prefetch
    }
    if (active) {
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
      if (qt == 0 && warp == 0 && lane == 0) { s_cls[0] = m0; s_cls[1] = l0; }
    }
    if (qt == 0 && pclsh) {
      // CLS softmax row of this head over the patch keys: p_j = exp2((s_j - m) scale) / l
      __syncthreads();
      const float mcls = s_cls[0], linv = 1.f / s_cls[1];
      for (int j = 1 + tid; j < T; j += 128)
        pclsh[((long long)slot * H + h) * (T - 1) + (j - 1)] = ex2f_fast((scls[j] - mcls) * scale_log2) * linv;
    }
  }
}

template <int DH>
cudaError_t launch_attn_dh(const bf16* q, const bf16* KV, const int* kvsrc, bf16* out, const int* wdesc,
                           const int* qoff, float* pclsh, int n_w, int T, int D, int H, long long kv_ld, int q_cache,
                           cudaStream_t s) {
  const int Tp = (T + 15) / 16 * 16;
  const size_t smem = (size_t)(4 * KB * (DH + 8) + QT * (DH + 8)) * sizeof(bf16) + (size_t)Tp * 8;
  cudaError_t e = ensure_smem<attn_kernel<DH>>(smem);
  if (e != cudaSuccess) return e;
  dim3 grid(H, n_w);
  const float scale_log2 = 1.4426950408889634f / sqrtf((float)DH);
  attn_kernel<DH><<<grid, 128, smem, s>>>(q, KV, kvsrc, out, reinterpret_cast<const int4*>(wdesc), qoff, pclsh, T,
                                          D, H, scale_log2, kv_ld, q_cache);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attention(const bf16* q, const bf16* KV, const int* kvsrc, bf16* out, const int* wdesc,
                             const int* qoff, float* pclsh, int n_w, int T, int D, int H, cudaStream_t s,
                             long long kv_ld, int q_cache) {
  if (n_w <= 0) return cudaSuccess;
  const int dh = D / H;
  if (kv_ld <= 0) kv_ld = 2LL * D;
  if (dh == 64) return launch_attn_dh<64>(q, KV, kvsrc, out, wdesc, qoff, pclsh, n_w, T, D, H, kv_ld, q_cache, s);
  if (dh == 16) return launch_attn_dh<16>(q, KV, kvsrc, out, wdesc, qoff, pclsh, n_w, T, D, H, kv_ld, q_cache, s);
  return cudaErrorInvalidValue;
}

}  // namespace rv
