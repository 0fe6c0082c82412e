// k_attn_tc.cu — attention of the compacted queries over all T keys of their frame on the
// 5th-generation tensor cores (P:313 every recomputed query attends to all
// tokens; P:336 CLS attention row = feature t).  d_h = 64, 128 <= T <= 320 (CLIP B/16, L/14
// 224 px); selected with RV_ATTN_TC, otherwise the mma.sync kernel of k_attn.cu runs.
//
// Persistent, warp-specialised CTA (384 threads, one per SM) over work items
// (frame of the wave, head, 128-row query tile):
//   warps 0,2,3 loaders: gather the item's K and V rows through `kvsrc` (reuse cache read in
//               place) with cp.async into SWIZZLE_128B tiles and its Q tile by TMA, two items
//               in flight (K/V/Q double-buffered);
//   warp 1      TMEM allocator + single-thread MMA issuer: S_c = Q K_c^T per 128-key chunk
//               (tcgen05.mma M=128, N<=128, K=64) into a 2-slot TMEM ring, twice per item
//               (pass A: row statistics, pass B: probabilities), and O += P_c V_c with the
//               TMEM-A form (V as an MN-major shared operand) into a 2-item O ring;
//   warps 4-11  softmax + epilogue, two warps per TMEM lane quarter (each half of a chunk's
//               columns): pass A online max / sum (fp32, ex2), pass B P_c = exp2((S_c - m) s)
//               as packed bf16 into a 2-slot TMEM ring; O normalised and stored as bf16; the
//               CLS query's normalised row over the patch keys goes to pclsh (per head).
// TMEM (512 columns): S ring [0,256), P ring [256,384), O ring [384,512).  Every stage hands
// off through mbarriers, so loads, MMAs and softmax of consecutive chunks / items overlap.
#include <cuda.h>

#include "common.cuh"
#include "rv_internal.h"

namespace rv {
namespace {

constexpr int AT_THREADS = 384;
constexpr int AT_SM_THREADS = 256;         // softmax warps 4..11
constexpr int AT_QROWS = 128;
constexpr int AT_KC = 128;                 // keys per S chunk
constexpr int AT_MAX_TP = 320;
constexpr int AT_MAX_TILES = 3;            // q-tiles per frame (T <= 320 -> nq <= 320)
constexpr uint32_t AT_TMEM_COLS = 512;
constexpr uint32_t AT_S_COL = 0, AT_P_COL = 256, AT_O_COL = 384;

RV_DEV uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
RV_DEV void mbar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
RV_DEV void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
RV_DEV void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
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
RV_DEV void mma_ss(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
RV_DEV void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
// Shared-memory descriptor, SWIZZLE_128B, version 1, SBO = 1024 B (8 rows x 128 B).  The same
// 128 B x 8-row atoms serve K-major (Q, K) and MN-major (V) operands.
RV_DEV uint64_t sdesc(uint32_t addr) {
  return ((uint64_t)((addr >> 4) & 0x3FFF)) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// kind::f16 instruction descriptor: D fp32, A/B bf16, A K-major, B K-major (b_mn = 0) or
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
RV_DEV void named_bar_softmax() { asm volatile("bar.sync 1, %0;" ::"n"(AT_SM_THREADS) : "memory"); }

struct Item {   // a (frame, head, q-tile) work item
  int w, h, qt, q0, nrows, slot;
};
// Items are (w, h, qt) with qt < AT_MAX_TILES; tiles past a frame's query count are skipped
// by every role in the same way, so all roles see the same sequence of live items.
RV_DEV bool item_at(int it, int H, const int* __restrict__ qoff, const int4* __restrict__ wdesc, Item& o) {
  const int per_w = H * AT_MAX_TILES;
  o.w = it / per_w;
  const int r = it - o.w * per_w;
  o.h = r / AT_MAX_TILES;
  o.qt = r - o.h * AT_MAX_TILES;
  const int q0 = qoff[o.w], nq = qoff[o.w + 1] - q0;
  if (o.qt * AT_QROWS >= nq) return false;
  o.q0 = q0 + o.qt * AT_QROWS;
  o.nrows = min(AT_QROWS, nq - o.qt * AT_QROWS);
  o.slot = wdesc[o.w].x;
  return true;
}

__global__ void __launch_bounds__(AT_THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const bf16* __restrict__ KV,
                   const int* __restrict__ kvsrc, bf16* __restrict__ out, const int4* __restrict__ wdesc,
                   const int* __restrict__ qoff, float* __restrict__ pclsh, int n_w, int T, int D, int H,
                   float scale_log2) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int Tp = (T + 15) / 16 * 16;
  const int nchunks = (Tp + AT_KC - 1) / AT_KC;
  const uint32_t kvb = (uint32_t)Tp * 128;
  const uint32_t base = su32(sm);
  // [Q0 16K][Q1 16K][K0][V0][K1][V1] then stats / CLS row / barriers
  auto sQ = [&](int b) { return base + (uint32_t)b * 16384u; };
  auto sK = [&](int b) { return base + 32768u + (uint32_t)b * 2u * kvb; };
  auto sV = [&](int b) { return base + 32768u + (uint32_t)b * 2u * kvb + kvb; };
  float* red = reinterpret_cast<float*>(sm + 32768 + 4 * kvb);   // [2 stats][2 halves][128]
  float* clsp = red + 4 * AT_QROWS;                                // [AT_MAX_TP]
  uint64_t* bar = reinterpret_cast<uint64_t*>(clsp + AT_MAX_TP);
  uint64_t *kv_full = bar, *kv_empty = bar + 2, *s_full = bar + 4, *s_empty = bar + 6, *p_full = bar + 8,
           *p_empty = bar + 10, *o_full = bar + 12, *o_empty = bar + 14;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 16);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQ) : "memory");
    for (int i = 0; i < 2; ++i) {
      mbar_init(&kv_full[i], 97);           // 96 loader lanes + the Q TMA expect_tx arrival
      mbar_init(&kv_empty[i], 1);           // MMA commit
      mbar_init(&s_full[i], 1);             // MMA commit
      mbar_init(&s_empty[i], AT_SM_THREADS);
      mbar_init(&p_full[i], AT_SM_THREADS);
      mbar_init(&p_empty[i], 1);            // MMA commit
      mbar_init(&o_full[i], 1);             // MMA commit
      mbar_init(&o_empty[i], AT_SM_THREADS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                 "r"(AT_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tslot;
  const int n_items = n_w * H * AT_MAX_TILES;

  if (warp == 0 || warp == 2 || warp == 3) {
    // ===================================================== loaders (warps 0, 2, 3)
    constexpr int RPL = (AT_MAX_TP + 95) / 96;   // key rows per lane
    const int lrow = (warp == 0 ? 0 : warp - 1) * 32 + lane;   // 0..95
    int j = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      Item itm;
      if (!item_at(it, H, qoff, wdesc, itm)) continue;
      const int b = j & 1;
      mbar_wait(&kv_empty[b], ((j >> 1) & 1) ^ 1);
      if (warp == 0 && lane == 0) {
        mbar_expect_tx(&kv_full[b], AT_QROWS * 128);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                sQ(b)),
            "l"(&tmQ), "r"(itm.h * 64), "r"(itm.q0), "r"(su32(&kv_full[b]))
            : "memory");
      }
      int rows[RPL];
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        const int jr = lrow + 96 * k;
        rows[k] = jr < T ? (kvsrc ? __ldg(kvsrc + (long long)itm.slot * T + jr) : itm.slot * T + jr) : 0;
      }
      const long long ld = 2LL * D;
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        const int jr = lrow + 96 * k;
        if (jr < Tp) {
          const bool ok = jr < T;
          const bf16* src = KV + (long long)rows[k] * ld + itm.h * 64;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const uint32_t off = (uint32_t)jr * 128 + ((c ^ (jr & 7)) << 4);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sK(b) + off), "l"(src + c * 8),
                         "r"(ok ? 16 : 0)
                         : "memory");
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sV(b) + off), "l"(src + D + c * 8),
                         "r"(ok ? 16 : 0)
                         : "memory");
          }
        }
      }
      asm volatile("cp.async.wait_all;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic -> async proxy (UMMA)
      mbar_arrive(&kv_full[b]);
      ++j;
    }
  } else if (warp == 1) {
    // ===================================================== MMA issuer (one lane)
    if (lane == 0) {
      int j = 0;
      uint32_t sc = 0, pc = 0;
      for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
        Item itm;
        if (!item_at(it, H, qoff, wdesc, itm)) continue;
        const int b = j & 1;
        mbar_wait(&kv_full[b], (j >> 1) & 1);
        tc_after();
        auto issue_s = [&](int c) {
          const int s = sc & 1;
          mbar_wait(&s_empty[s], ((sc >> 1) & 1) ^ 1);
          tc_after();
          const int nc = min(AT_KC, Tp - c * AT_KC);
          const uint32_t id = idesc(nc, 0);
#pragma unroll
          for (int k = 0; k < 4; ++k)
            mma_ss(tmem + AT_S_COL + s * AT_KC, sdesc(sQ(b) + k * 32), sdesc(sK(b) + c * AT_KC * 128 + k * 32), id,
                   k > 0);
          mma_commit(&s_full[s]);
          ++sc;
        };
        for (int c = 0; c < nchunks; ++c) issue_s(c);          // pass A
        issue_s(0);                                              // pass B
        const int ob = j & 1;
        mbar_wait(&o_empty[ob], ((j >> 1) & 1) ^ 1);
        tc_after();
        for (int c = 0; c < nchunks; ++c) {
          if (c + 1 < nchunks) issue_s(c + 1);                  // keeps the softmax warps fed
          const int ps = pc & 1;
          mbar_wait(&p_full[ps], (pc >> 1) & 1);
          tc_after();
          const int nc = min(AT_KC, Tp - c * AT_KC);
          const uint32_t id = idesc(64, 1);
          for (int k = 0; k < nc / 16; ++k)
            mma_ts(tmem + AT_O_COL + ob * 64, tmem + AT_P_COL + ps * 64 + (uint32_t)(k * 8),
                   sdesc(sV(b) + (uint32_t)(c * AT_KC + k * 16) * 128), id, (c > 0 || k > 0) ? 1u : 0u);
          mma_commit(&p_empty[ps]);
          ++pc;
        }
        mma_commit(&o_full[ob]);
        mma_commit(&kv_empty[b]);     // K/V/Q buffers free once every MMA of the item retired
        ++j;
      }
    }
  } else if (warp >= 4) {
    // ===================================================== softmax + epilogue
    const int quarter = warp & 3, half = (warp - 4) >> 2;
    const int row = quarter * 32 + lane;
    const uint32_t lane_base = (uint32_t)(quarter * 32) << 16;
    const int stid = tid - 128;
    int j = 0;
    uint32_t sc = 0, pc = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      Item itm;
      if (!item_at(it, H, qoff, wdesc, itm)) continue;
      const bool live = quarter * 32 < itm.nrows;    // warp-uniform
      // ---- pass A: online row max / sum over this thread's half of every chunk
      float m = -INFINITY, l = 0.f;
      for (int c = 0; c < nchunks; ++c) {
        const int s = sc & 1;
        mbar_wait(&s_full[s], (sc >> 1) & 1);
        tc_after();
        const int nc = min(AT_KC, Tp - c * AT_KC);
        const int hb = half ? (nc / 32) * 16 : 0, he = half ? nc : (nc / 32) * 16;
        if (live) {
          for (int c0 = hb; c0 < he; c0 += 16) {
            float v[16];
            tld16(tmem + lane_base + AT_S_COL + s * AT_KC + c0, v);
            const int key0 = c * AT_KC + c0;
            float cm = -INFINITY;
#pragma unroll
            for (int i = 0; i < 16; ++i) cm = fmaxf(cm, key0 + i < T ? v[i] : -INFINITY);
            const float mn = fmaxf(m, cm);
            float cs = 0.f;
#pragma unroll
            for (int i = 0; i < 16; ++i) cs += key0 + i < T ? ex2f_fast((v[i] - mn) * scale_log2) : 0.f;
            l = (m == -INFINITY ? 0.f : l * ex2f_fast((m - mn) * scale_log2)) + cs;
            m = mn;
          }
        }
        tc_before();
        mbar_arrive(&s_empty[s]);
        ++sc;
      }
      red[half * AT_QROWS + row] = m;
      red[2 * AT_QROWS + half * AT_QROWS + row] = l;
      named_bar_softmax();
      const float m0 = red[row], m1 = red[AT_QROWS + row];
      const float mrow = fmaxf(m0, m1);
      const float lrow = (m0 == -INFINITY ? 0.f : red[2 * AT_QROWS + row] * ex2f_fast((m0 - mrow) * scale_log2)) +
                         (m1 == -INFINITY ? 0.f : red[3 * AT_QROWS + row] * ex2f_fast((m1 - mrow) * scale_log2));
      const float ms = mrow * scale_log2;
      const bool cls_row = (itm.qt == 0 && row == 0 && pclsh != nullptr);
      // ---- pass B: P_c = exp2((S_c - m) scale) as bf16 pairs into the P ring
      for (int c = 0; c < nchunks; ++c) {
        const int s = sc & 1, ps = pc & 1;
        mbar_wait(&s_full[s], (sc >> 1) & 1);
        mbar_wait(&p_empty[ps], ((pc >> 1) & 1) ^ 1);
        tc_after();
        const int nc = min(AT_KC, Tp - c * AT_KC);
        const int hb = half ? (nc / 32) * 16 : 0, he = half ? nc : (nc / 32) * 16;
        if (live) {
          for (int c0 = hb; c0 < he; c0 += 16) {
            float v[16];
            tld16(tmem + lane_base + AT_S_COL + s * AT_KC + c0, v);
            const int key0 = c * AT_KC + c0;
            uint32_t pk[8];
#pragma unroll
            for (int i = 0; i < 16; i += 2) {
              const float p0 = key0 + i < T ? ex2f_fast(fmaf(v[i], scale_log2, -ms)) : 0.f;
              const float p1 = key0 + i + 1 < T ? ex2f_fast(fmaf(v[i + 1], scale_log2, -ms)) : 0.f;
              pk[i / 2] = pack_bf16x2(p0, p1);
              if (cls_row) { clsp[key0 + i] = p0; clsp[key0 + i + 1] = p1; }
            }
            tst8(tmem + lane_base + AT_P_COL + ps * 64 + (uint32_t)(c0 / 2), pk);
          }
          asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
        tc_before();
        mbar_arrive(&s_empty[s]);
        mbar_arrive(&p_full[ps]);
        ++sc;
        ++pc;
      }
      if (itm.qt == 0 && pclsh) {   // normalised CLS row of this head over patch keys 1..T-1
        named_bar_softmax();         // clsp complete (written by the row-0 threads of both halves)
        const float r0 = fmaxf(red[0], red[AT_QROWS]);
        const float l0 = (red[0] == -INFINITY ? 0.f : red[2 * AT_QROWS] * ex2f_fast((red[0] - r0) * scale_log2)) +
                         (red[AT_QROWS] == -INFINITY ? 0.f
                                                     : red[3 * AT_QROWS] * ex2f_fast((red[AT_QROWS] - r0) * scale_log2));
        const float linv = 1.f / l0;
        for (int jj = 1 + stid; jj < T; jj += AT_SM_THREADS)
          pclsh[((long long)itm.slot * H + itm.h) * (T - 1) + (jj - 1)] = clsp[jj] * linv;
      }
      // ---- epilogue: O / l, this thread's 32 of the 64 head columns
      const int ob = j & 1;
      mbar_wait(&o_full[ob], (j >> 1) & 1);
      tc_after();
      if (live) {
        float v0[16], v1[16];
        tld16(tmem + lane_base + AT_O_COL + ob * 64 + half * 32, v0);
        tld16(tmem + lane_base + AT_O_COL + ob * 64 + half * 32 + 16, v1);
        if (row < itm.nrows) {
          const float il = 1.f / lrow;
          uint4* o = reinterpret_cast<uint4*>(out + (long long)(itm.q0 + row) * D + itm.h * 64 + half * 32);
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
      mbar_arrive(&o_empty[ob]);
      named_bar_softmax();           // red[] / clsp reused by the next item
      ++j;
    }
  }
  tc_before();
  __syncthreads();
  if (warp == 1) {
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
  return 32768 + 4 * (size_t)Tp * 128 + 4 * AT_QROWS * 4 + AT_MAX_TP * 4 + 16 * 8 + 16;
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
  const int items = n_w * H * AT_MAX_TILES;
  const int grid = items < sms ? items : sms;
  const float scale_log2 = 1.4426950408889634f / 8.0f;   // 1/sqrt(64) * log2(e)
  attn_tc_kernel<<<grid, AT_THREADS, smem, s>>>(tmQ, KV, kvsrc, out, reinterpret_cast<const int4*>(wdesc), qoff,
                                                pclsh, n_w, T, D, H, scale_log2);
  return cudaGetLastError();
}

}  // namespace rv
