// k_attn_tc.cu — attention of the compacted queries over all T keys of their frame on the
// 5th-generation tensor cores (P:313 every recomputed query attends to all
// tokens; P:336 CLS attention row = feature t).  Used for d_h = 64 and T <= 288 (CLIP B/16,
// L/14 224 px); other shapes use the mma.sync kernel in k_attn.cu.
//
// Persistent CTAs (256 threads, two per SM so one CTA's softmax overlaps the other's MMAs and
// loads) walk (frame, head) items of the wave:
//   * K and V rows of the item are gathered through `kvsrc` (reuse cache read in place) with
//     cp.async into SWIZZLE_128B shared tiles;
//   * per 128-row query tile: Q by TMA; keys in chunks of 128: S_c = Q K_c^T with tcgen05.mma
//     (M=128, N<=128, K=64) into 128 TMEM columns.  Pass A: online row max / sum over the
//     chunks (fp32, ex2).  Pass B: S_c again, P_c = exp2((S_c - m) scale) written to TMEM as
//     packed bf16, O += P_c V_c with the TMEM-A form of tcgen05.mma (V as an MN-major shared
//     operand), the next S chunk overlapping the current P V; 8 warps (two per TMEM lane
//     quarter, each half of a chunk's columns; quarters without real query rows skip the
//     softmax); O read with tcgen05.ld, normalised by the row sum, stored as bf16;
//   * the CLS query of the frame (first compact row) also emits its normalised softmax row over
//     the patch keys for this head (pclsh).
#include <cuda.h>

#include "common.cuh"
#include "rv_internal.h"

namespace rv {
namespace {

constexpr int AT_THREADS = 256;            // 8 warps: 2 per TMEM lane quarter
constexpr int AT_QROWS = 128;
constexpr int AT_KC = 128;                 // keys per S chunk (tcgen05 N)
constexpr int AT_MAX_TP = 320;             // keys (padded to 16) held per item in smem
constexpr uint32_t AT_TMEM_COLS = 256;     // S chunk [0,128), P chunk [128,192), O [192,256): 2 CTAs/SM
constexpr uint32_t AT_P_COL = 128, AT_O_COL = 192;

RV_DEV uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
RV_DEV void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
RV_DEV void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
RV_DEV void mbar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = su32(b);
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
RV_DEV void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
RV_DEV void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
RV_DEV void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}
// SMEM-A x SMEM-B
RV_DEV void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// TMEM-A x SMEM-B
RV_DEV void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
// Shared-memory descriptor, SWIZZLE_128B, version 1.  K-major: SBO = 1024 B (8 rows x 128 B).
// MN-major (V): same 128 B x 8-row atoms, SBO = 1024 B between 8-row groups along K.
RV_DEV uint64_t sdesc(uint32_t addr) {
  return ((uint64_t)((addr >> 4) & 0x3FFF)) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// Instruction descriptor kind::f16: D fp32, A/B bf16, A K-major, B K-major (b_mn = 0) or
// MN-major (b_mn = 1), N >> 3 at bit 17, M >> 4 at bit 24.
RV_DEV uint32_t idesc(int N, int b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(AT_QROWS >> 4) << 24);
}
RV_DEV void tld16(uint32_t taddr, float (&v)[16]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
RV_DEV void tst8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(taddr), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
}
RV_DEV void cp16(uint32_t dst, const void* src, bool ok) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(ok ? 16 : 0) : "memory");
}

// Gather K and V rows of (frame slot, head h) into swizzled tiles: key j, 16-B chunk c at
// j*128 + ((c ^ (j & 7)) << 4).  Rows j >= T are zero-filled.
RV_DEV void load_kv(uint32_t kbuf, uint32_t vbuf, const bf16* __restrict__ KV, const int* __restrict__ kvsrc,
                    int slot, int h, int T, int Tp, int D, int tid) {
  const long long ld = 2LL * D;
  constexpr int RPT = (AT_MAX_TP + AT_THREADS / 8 - 1) / (AT_THREADS / 8);   // key rows per thread
  const int c = tid & 7;
  // all row indices first (independent loads in flight), then the copies
  int rows[RPT];
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int j = (tid >> 3) + k * (AT_THREADS / 8);
    rows[k] = j < T ? (kvsrc ? __ldg(kvsrc + (long long)slot * T + j) : slot * T + j) : 0;
  }
#pragma unroll
  for (int k = 0; k < RPT; ++k) {
    const int j = (tid >> 3) + k * (AT_THREADS / 8);
    if (j < Tp) {
      const bool ok = j < T;
      const bf16* src = KV + (long long)rows[k] * ld + h * 64 + c * 8;
      const uint32_t off = j * 128 + ((c ^ (j & 7)) << 4);
      cp16(kbuf + off, src, ok);
      cp16(vbuf + off, src + D, ok);
    }
  }
}

RV_DEV float ex2(float x) {   // MUFU.EX2, flush-to-zero (softmax terms are in [0, 1])
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__global__ void __launch_bounds__(AT_THREADS, 2)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const bf16* __restrict__ KV,
                   const int* __restrict__ kvsrc, bf16* __restrict__ out, const int4* __restrict__ wdesc,
                   const int* __restrict__ qoff, float* __restrict__ pclsh, int n_w, int T, int D, int H,
                   float scale_log2) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int Tp = (T + 15) / 16 * 16;
  const int kvbytes = Tp * 128;
  const uint32_t sQ = su32(sm);                       // [128][64] bf16, 16 KB (TMA, SWIZZLE_128B)
  const uint32_t sK = sQ + 16384;                     // [Tp][64] bf16, swizzled
  const uint32_t sV = sK + (uint32_t)kvbytes;         // [Tp][64] bf16, swizzled (MN-major B)
  float* red = reinterpret_cast<float*>(sm + 16384 + 2 * kvbytes);   // [2][2][128] part max / sum
  float* clsp = red + 4 * AT_QROWS;                                    // [Tp] CLS row exp values
  uint64_t* bars = reinterpret_cast<uint64_t*>(clsp + AT_MAX_TP);       // q, s, o
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bars + 3);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int quarter = warp & 3, part = warp >> 2;   // TMEM lane quarter, column half of a chunk
  const int row = quarter * 32 + lane;              // query row of this thread in the 128-row tile
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQ) : "memory");
    for (int i = 0; i < 3; ++i) mbar_init(&bars[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                 "r"(AT_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tslot;
  const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
  const int nchunks = (Tp + AT_KC - 1) / AT_KC;
  uint32_t ph_q = 0, ph_s = 0, ph_o = 0;
  const int n_items = n_w * H;

  // S chunk c (keys [c*128, c*128 + nc)) into TMEM columns [0, nc); thread 0 only
  auto issue_s = [&](int c) {
    const int nc = min(AT_KC, Tp - c * AT_KC);
    const uint32_t id = idesc(nc, 0);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      mma_ss(tmem, sdesc(sQ + k * 32), sdesc(sK + c * AT_KC * 128 + k * 32), id, k > 0);
    mma_commit(&bars[1]);
  };
  for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
    const int w = it / H, h = it % H;
    const int slot = wdesc[w].x;
    const int q0 = qoff[w], nq = qoff[w + 1] - q0;
    load_kv(sK, sV, KV, kvsrc, slot, h, T, Tp, D, tid);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic -> async proxy (UMMA reads)
    __syncthreads();
    const int ntiles = (nq + AT_QROWS - 1) / AT_QROWS;
    for (int qt = 0; qt < ntiles; ++qt) {
      const int nrows = min(AT_QROWS, nq - qt * AT_QROWS);
      const bool live = quarter * 32 < nrows;    // warp-uniform: this lane quarter holds real rows
      if (tid == 0) {
        mbar_expect_tx(&bars[0], AT_QROWS * 128);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                sQ),
            "l"(&tmQ), "r"(h * 64), "r"(q0 + qt * AT_QROWS), "r"(su32(&bars[0]))
            : "memory");
        mbar_wait(&bars[0], ph_q);
        tc_after();
        issue_s(0);
      }
      ph_q ^= 1;
      // ---- pass A: online row max / sum over the key chunks (this thread's column half)
      float m = -INFINITY, l = 0.f;
      for (int c = 0; c < nchunks; ++c) {
        mbar_wait(&bars[1], ph_s);
        ph_s ^= 1;
        tc_after();
        const int nc = min(AT_KC, Tp - c * AT_KC);
        const int hb = part * (nc / 2 / 16) * 16;               // this half: [hb, he)
        const int he = part ? nc : (nc / 2 / 16) * 16;
        if (live) {
          for (int c0 = hb; c0 < he; c0 += 16) {
            float v[16];
            tld16(tmem + lane_base + c0, v);
            const int key0 = c * AT_KC + c0;
            float cm = -INFINITY;
#pragma unroll
            for (int i = 0; i < 16; ++i) cm = fmaxf(cm, key0 + i < T ? v[i] : -INFINITY);
            const float mn = fmaxf(m, cm);
            float cs = 0.f;
#pragma unroll
            for (int i = 0; i < 16; ++i) cs += key0 + i < T ? ex2((v[i] - mn) * scale_log2) : 0.f;
            l = l * ex2((m - mn) * scale_log2) + cs;
            m = mn;
          }
        }
        tc_before();
        __syncthreads();                       // S chunk consumed
        if (tid == 0) {
          tc_after();
          issue_s(c + 1 < nchunks ? c + 1 : 0);  // next chunk, or chunk 0 again for pass B
        }
      }
      red[part * AT_QROWS + row] = m;
      red[2 * AT_QROWS + part * AT_QROWS + row] = l;
      __syncthreads();
      const float m0 = red[row], m1 = red[AT_QROWS + row];
      const float mrow = fmaxf(m0, m1);
      const float lrow = (m0 == -INFINITY ? 0.f : red[2 * AT_QROWS + row] * ex2((m0 - mrow) * scale_log2)) +
                         (m1 == -INFINITY ? 0.f : red[3 * AT_QROWS + row] * ex2((m1 - mrow) * scale_log2));
      const float ms = mrow * scale_log2;
      const bool cls_row = (qt == 0 && row == 0 && pclsh != nullptr);
      // ---- pass B: P = exp2((S - m) scale) chunk by chunk, O += P_c V_c on the tensor core
      for (int c = 0; c < nchunks; ++c) {
        mbar_wait(&bars[1], ph_s);
        ph_s ^= 1;
        tc_after();
        const int nc = min(AT_KC, Tp - c * AT_KC);
        const int hb = part * (nc / 2 / 16) * 16;
        const int he = part ? nc : (nc / 2 / 16) * 16;
        if (c > 0) {   // P chunk columns are free once the previous P*V retired
          mbar_wait(&bars[2], ph_o);
          ph_o ^= 1;
          tc_after();
        }
        if (live) {
          for (int c0 = hb; c0 < he; c0 += 16) {
            float v[16];
            tld16(tmem + lane_base + c0, v);
            const int key0 = c * AT_KC + c0;
            uint32_t pk[8];
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
              const float p0 = key0 + i < T ? ex2(fmaf(v[i], scale_log2, -ms)) : 0.f;
              const float p1 = key0 + i + 1 < T ? ex2(fmaf(v[i + 1], scale_log2, -ms)) : 0.f;
              pk[i / 2] = pack_bf16x2(p0, p1);
              if (cls_row) { clsp[key0 + i] = p0; clsp[key0 + i + 1] = p1; }
            }
            tst8(tmem + lane_base + AT_P_COL + (uint32_t)(c0 / 2), pk);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        tc_before();
        __syncthreads();                       // S chunk consumed, P chunk written
        if (tid == 0) {
          tc_after();
          const uint32_t id = idesc(64, 1);
          for (int k = 0; k < nc / 16; ++k)
            mma_ts(tmem + AT_O_COL, tmem + AT_P_COL + (uint32_t)(k * 8), sdesc(sV + (c * AT_KC + k * 16) * 128), id,
                   (c > 0 || k > 0) ? 1u : 0u);
          mma_commit(&bars[2]);
          if (c + 1 < nchunks) issue_s(c + 1);   // overlaps this chunk's P*V
        }
      }
      if (qt == 0 && pclsh) {   // normalised CLS row of this head over the patch keys 1..T-1
        const float lc = (red[0] == -INFINITY ? 0.f : red[2 * AT_QROWS] * ex2((red[0] - fmaxf(red[0], red[AT_QROWS])) * scale_log2)) +
                         (red[AT_QROWS] == -INFINITY ? 0.f : red[3 * AT_QROWS] * ex2((red[AT_QROWS] - fmaxf(red[0], red[AT_QROWS])) * scale_log2));
        const float linv = 1.f / lc;
        for (int j = 1 + tid; j < T; j += AT_THREADS)
          pclsh[((long long)slot * H + h) * (T - 1) + (j - 1)] = clsp[j] * linv;
      }
      mbar_wait(&bars[2], ph_o);
      ph_o ^= 1;
      tc_after();
      // ---- epilogue: 32 of the 64 O columns per warp, normalised, bf16
      if (live) {
        float v0[16], v1[16];
        tld16(tmem + lane_base + AT_O_COL + part * 32, v0);
        tld16(tmem + lane_base + AT_O_COL + part * 32 + 16, v1);
        if (row < nrows) {
          const float il = 1.f / lrow;
          uint4* o = reinterpret_cast<uint4*>(out + (long long)(q0 + qt * AT_QROWS + row) * D + h * 64 + part * 32);
          uint4 u;
          u.x = pack_bf16x2(v0[0] * il, v0[1] * il); u.y = pack_bf16x2(v0[2] * il, v0[3] * il);
          u.z = pack_bf16x2(v0[4] * il, v0[5] * il); u.w = pack_bf16x2(v0[6] * il, v0[7] * il);
          o[0] = u;
          u.x = pack_bf16x2(v0[8] * il, v0[9] * il); u.y = pack_bf16x2(v0[10] * il, v0[11] * il);
          u.z = pack_bf16x2(v0[12] * il, v0[13] * il); u.w = pack_bf16x2(v0[14] * il, v0[15] * il);
          o[1] = u;
          u.x = pack_bf16x2(v1[0] * il, v1[1] * il); u.y = pack_bf16x2(v1[2] * il, v1[3] * il);
          u.z = pack_bf16x2(v1[4] * il, v1[5] * il); u.w = pack_bf16x2(v1[6] * il, v1[7] * il);
          o[2] = u;
          u.x = pack_bf16x2(v1[8] * il, v1[9] * il); u.y = pack_bf16x2(v1[10] * il, v1[11] * il);
          u.z = pack_bf16x2(v1[12] * il, v1[13] * il); u.w = pack_bf16x2(v1[14] * il, v1[15] * il);
          o[3] = u;
        }
      }
      tc_before();
      __syncthreads();          // TMEM, Q tile, red[] and clsp are reused by the next q-tile / item
    }
  }
  tc_before();
  __syncthreads();
  if (warp == 0) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(AT_TMEM_COLS));
  }
}

}  // namespace

bool attn_tc_supported(int T, int D, int H) {
  return D / H == 64 && T >= AT_KC && (T + 15) / 16 * 16 <= AT_MAX_TP;
}

size_t attn_tc_smem(int T) {
  const int Tp = (T + 15) / 16 * 16;
  return 16384 + 2 * (size_t)Tp * 128 + 4 * AT_QROWS * 4 + AT_MAX_TP * 4 + 3 * 8 + 8;
}

cudaError_t launch_attention_tc(const CUtensorMap& tmQ, const bf16* KV, const int* kvsrc, bf16* out,
                                const int* wdesc, const int* qoff, float* pclsh, int n_w, int T, int D, int H,
                                cudaStream_t s) {
  if (n_w <= 0) return cudaSuccess;
  const size_t smem = attn_tc_smem(T);
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int items = n_w * H;
  const int grid = items < 2 * sms ? items : 2 * sms;   // two CTAs per SM overlap MMA and softmax
  const float scale_log2 = 1.4426950408889634f / 8.0f;   // 1/sqrt(64) * log2(e)
  attn_tc_kernel<<<grid, AT_THREADS, smem, s>>>(tmQ, KV, kvsrc, out, reinterpret_cast<const int4*>(wdesc), qoff,
                                                pclsh, n_w, T, D, H, scale_log2);
  return cudaGetLastError();
}

}  // namespace rv
