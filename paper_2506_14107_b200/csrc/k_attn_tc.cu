// k_attn_tc.cu — attention of the compacted queries over all T keys of their frame on the
// 5th-generation tensor cores (P:313 every recomputed query attends to all
// tokens; P:336 CLS attention row = feature t).  d_h = 64 and T - 1 <= 256 patch keys (CLIP
// B/16, L/14 at 224 px); selected with RV_ATTN_TC, otherwise the mma.sync kernel of k_attn.cu.
//
// Work item = (frame of the wave, head, 64-row query tile).  Recomputed queries per frame are
// few (~57 of 257 at the paper's reuse rates), so the tile is M = 64: tcgen05 then puts the
// accumulator rows on lanes 0-15 of each of the four TMEM lane quarters, and with the
// 16x32bx2 TMEM access shape every thread of every SM sub-partition owns one (row, 32-column)
// piece: the softmax is spread over all four sub-partitions with full warps.
// Persistent, warp-specialised CTA (640 threads, one per SM):
//   warps 0,2,3   loaders: the Q tile by TMA; the K and V rows of the T-1 patch keys gathered
//                 through `kvsrc` (reuse cache read in place) with cp.async into SWIZZLE_128B
//                 tiles, completion tracked on mbarriers (no waiting in the loaders); the CLS
//                 key's K/V row.  Q, K and V are double-buffered and released separately (Q
//                 after the softmax read it, K when S retired, V when P V retired).
//   warp 1        TMEM allocator + single-thread MMA issuer, polling: S = Q K_patch^T (M=64,
//                 N<=256, K=64) into one of two TMEM regions, O = P V_patch (M=64, N=64, K<=256)
//                 with P read from TMEM (written over S) and V an MN-major shared operand.
//   warps 4..19   softmax + epilogue: one tcgen05.ld per item, row max / sum exchanged through
//                 shared memory (8 partials per row), P = exp2((S - m) s) packed to bf16 and
//                 stored over S; the epilogue of item j (O / l as bf16) runs after the softmax of
//                 item j+1, hiding the P V latency.
// The CLS key (key 0) is handled on the CUDA cores (s_cls = q . k_cls, O += p_cls v_cls), so
// the 256 patch keys of L/14 fill one N = 256 MMA.  TMEM: 2 regions x 256 columns, each S
// [0,256), P packed over [0,128), O [128,192).
#include <cuda.h>
#include <cstdio>

#include "common.cuh"
#include "rv_internal.h"

namespace rv {
namespace {

constexpr int AT_LOADER_WARPS = 3;                // warps 0, 2, 3 (20 warps: 96 registers per thread)
constexpr int AT_LOADERS = AT_LOADER_WARPS * 32;
constexpr int AT_WARPS = 2 + AT_LOADER_WARPS - 1 + 16;   // loaders, MMA (1), 16 softmax
constexpr int AT_THREADS = AT_WARPS * 32;
constexpr int AT_QROWS = 64;                       // M of both MMAs
constexpr int AT_MAXK = 256;                       // patch keys per item (N of the S MMA)
constexpr int AT_MAX_TILES = 5;                    // T <= 257 -> <= 257 compact queries per frame
constexpr uint32_t AT_TMEM_COLS = 512;
constexpr uint32_t AT_REGION = 256;                // S; P packed over its first half; O after P
constexpr uint32_t AT_O_OFF = 128;
constexpr uint32_t AT_Q_BYTES = AT_QROWS * 128;    // 8 KB
constexpr uint32_t AT_KV_BYTES = AT_MAXK * 128;    // 32 KB each for K and V
constexpr uint32_t AT_BUF = AT_Q_BYTES + 2 * AT_KV_BYTES;   // 72 KB (multiple of 1 KB)
constexpr int AT_SMX = 512;                        // softmax threads (the last 16 warps)

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
RV_DEV bool mbar_test(uint64_t* b, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(su32(b)), "r"(parity)
      : "memory");
  return ok != 0;
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
// 16x32bx2 shapes: lanes 0-15 of the warp access TMEM lanes base..base+15 at columns
// [c, c+n), lanes 16-31 the same TMEM lanes at columns [c+n, c+2n)  (n = x-count)
RV_DEV void tld32h(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32], 32;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
RV_DEV void tld8h(uint32_t taddr, float* v) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.16x32bx2.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], 8;"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr));
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __uint_as_float(r[i]);
}
RV_DEV void tst16h(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x32bx2.x16.b32 [%0], 16, {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}
RV_DEV void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(idesc), "r"(acc));
}
RV_DEV void tld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
RV_DEV void smx_bar() { asm volatile("bar.sync 1, %0;" ::"n"(AT_SMX) : "memory"); }

#ifdef RV_ATTN_TRACE   // experiment builds only (build.build_variant): event timeline of CTA 0
RV_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ unsigned long long g_at_trace[64 * 16];
#define AT_TRACE(j, k) do { if (blockIdx.x == 0 && (j) < 64) g_at_trace[(j) * 16 + (k)] = gtime(); } while (0)
#else
#define AT_TRACE(j, k) do { } while (0)
#endif

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
  const int NP = T - 1;                          // patch keys
  const int NK = (NP + 15) / 16 * 16;            // N of the S MMA (<= 256)
  const uint32_t base = su32(sm);
  auto sQ = [&](int b) { return base + (uint32_t)b * AT_BUF; };
  auto sK = [&](int b) { return base + (uint32_t)b * AT_BUF + AT_Q_BYTES; };
  auto sV = [&](int b) { return base + (uint32_t)b * AT_BUF + AT_Q_BYTES + AT_KV_BYTES; };
  // CLS key rows (k_cls, v_cls; 256 B) of item j in ring slot j & 3 (v_cls is read by the
  // epilogue of item j, while buffer j & 1 may already hold item j + 2)
  auto sC = [&](int jj) { return 2 * AT_BUF + (jj & 3) * 256; };
  // softmax exchange, double-buffered by item parity; 8 partials per row (warp, half)
  float* clsp = reinterpret_cast<float*>(sm + 2 * AT_BUF + 1024);    // [2][256] p of the CLS query row
  float* red_m = clsp + 2 * AT_MAXK;                                  // [2][8][64] partial row max
  float* red_l = red_m + 16 * AT_QROWS;                               // [2][8][64] partial row sums
  float* red_pc = red_l + 16 * AT_QROWS;                              // [2][64] p of the CLS key
  int* rows_s = reinterpret_cast<int*>(red_pc + 2 * AT_QROWS);        // [2][256] K/V source rows
  uint64_t* bar = reinterpret_cast<uint64_t*>(rows_s + 2 * AT_MAXK);
  // Q, K and V of an item are released separately (Q after the softmax read its rows, K when
  // S completed, V when P V completed), so the next item's K streams in during the softmax
  uint64_t *q_full = bar, *k_full = bar + 2, *v_full = bar + 4, *q_empty = bar + 6, *k_empty = bar + 8,
           *v_empty = bar + 10, *s_full = bar + 12, *p_full = bar + 14, *o_full = bar + 16, *r_free = bar + 18;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 20);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQ) : "memory");
    for (int i = 0; i < 2; ++i) {
      mbar_init(&q_full[i], 1);                 // expect_tx arrival + the Q TMA bytes
      mbar_init(&k_full[i], AT_LOADERS);        // loader lanes' cp.async completions (arrive.noinc)
      mbar_init(&v_full[i], AT_LOADERS);
      mbar_init(&q_empty[i], 16);               // softmax warps (Q rows read for s_cls)
      mbar_init(&k_empty[i], 1);                // MMA commit after S
      mbar_init(&v_empty[i], 1);                // MMA commit after P V
      mbar_init(&s_full[i], 1);                 // MMA commit after S
      mbar_init(&p_full[i], 16);                // one arrival per softmax warp
      mbar_init(&o_full[i], 1);                 // MMA commit after P V
      mbar_init(&r_free[i], 16);                // O read: TMEM region reusable
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

  if (warp == 0 || (warp >= 2 && warp < 2 + AT_LOADER_WARPS - 1)) {
    // ===================================================== loaders (warps 0, 2, 3)
    // K and V rows are gathered with cp.async, 8 consecutive lanes per 128 B row (coalesced),
    // into the SWIZZLE_128B tiles; k_full / v_full count each lane's copies as they land
    // (cp.async.mbarrier.arrive.noinc), so the loaders never wait for data and run ahead as far
    // as the buffers allow.  (TMA tile::gather4 works here too but moves 128 B rows no faster.)
    const int lrow = (warp == 0 ? 0 : warp - 1) * 32 + lane;   // 0 .. AT_LOADERS-1
    const long long ld = 2LL * D;
    constexpr int RPL = (AT_MAXK + AT_LOADERS - 1) / AT_LOADERS;
    constexpr int IT = (AT_MAXK * 8 + AT_LOADERS - 1) / AT_LOADERS;
    // K/V source rows of patch key kr (token 1 + kr) of an item, RPL per lane
    auto load_idx = [&](const Item& x, int (&r)[RPL]) {
#pragma unroll
      for (int k = 0; k < RPL; ++k) {
        const int kr = lrow + AT_LOADERS * k;
        r[k] = kr < NP ? (kvsrc ? __ldg(kvsrc + (long long)x.slot * T + 1 + kr) : x.slot * T + 1 + kr) : -1;
      }
    };
    auto next_item = [&](int from, Item& x) {
      while (from < n_items && !item_at(from, H, qoff, wdesc, x)) from += gridDim.x;
      return from;
    };
    // tile rows NP..NK-1 zero-filled
    auto copy_tile = [&](uint32_t dst, int col, const int* rows) {
      int rw[IT];
#pragma unroll
      for (int k = 0; k < IT; ++k) {
        const int idx = lrow + AT_LOADERS * k;
        rw[k] = idx < NK * 8 ? rows[idx >> 3] : -2;
      }
#pragma unroll
      for (int k = 0; k < IT; ++k) {
        const int idx = lrow + AT_LOADERS * k;
        if (rw[k] == -2) continue;
        const int kr = idx >> 3, c = idx & 7;
        const bool ok = rw[k] >= 0;
        const bf16* src = KV + (long long)(ok ? rw[k] : 0) * ld + col + c * 8;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + (uint32_t)kr * 128 +
                                                                            ((c ^ (kr & 7)) << 4)),
                     "l"(src), "r"(ok ? 16 : 0)
                     : "memory");
      }
    };
    Item itm;
    int it = next_item(blockIdx.x, itm);
    int rr[RPL];
    if (it < n_items) load_idx(itm, rr);
    int j = 0;
    while (it < n_items) {
      const int b = j & 1;
      const uint32_t ph = ((j >> 1) & 1) ^ 1;
      int* rows = rows_s + b * AT_MAXK;
      mbar_wait(&k_empty[b], ph);
#ifdef RV_ATTN_TRACE
      if (warp == 0 && lane == 0) AT_TRACE(j, 0);
#endif
#pragma unroll
      for (int k = 0; k < RPL; ++k)
        if (lrow + AT_LOADERS * k < NK) rows[lrow + AT_LOADERS * k] = rr[k];
      asm volatile("bar.sync 5, %0;" ::"n"(AT_LOADERS) : "memory");
      copy_tile(sK(b), itm.h * 64, rows);
      if (lrow < 8)   // CLS key (never reused: its own row), k_cls as a plain 128 B row
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(base + sC(j) + lrow * 16),
                     "l"(KV + (long long)itm.slot * T * ld + itm.h * 64 + lrow * 8)
                     : "memory");
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&k_full[b])) : "memory");
      if (warp == 0 && lane == 0) {
        mbar_wait(&q_empty[b], ph);
        mbar_expect_tx(&q_full[b], AT_Q_BYTES);
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                sQ(b)),
            "l"(&tmQ), "r"(itm.h * 64), "r"(itm.q0), "r"(su32(&q_full[b]))
            : "memory");
      }
#ifdef RV_ATTN_TRACE
      if (warp == 0 && lane == 0) AT_TRACE(j, 1);
#endif
      // next item's row indices now: their latency overlaps the wait for the V buffer
      Item nx;
      const int nit = next_item(it + gridDim.x, nx);
      if (nit < n_items) load_idx(nx, rr);
      mbar_wait(&v_empty[b], ph);
      copy_tile(sV(b), D + itm.h * 64, rows);
      if (lrow < 8)   // v_cls
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(base + sC(j) + 128 + lrow * 16),
                     "l"(KV + (long long)itm.slot * T * ld + D + itm.h * 64 + lrow * 8)
                     : "memory");
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&v_full[b])) : "memory");
#ifdef RV_ATTN_TRACE
      if (warp == 0 && lane == 0) AT_TRACE(j, 2);
#endif
      itm = nx;
      it = nit;
      ++j;
    }
  } else if (warp == 1) {
    // ===================================================== MMA issuer (one lane)
    if (lane == 0) {
      const uint32_t id_s = idesc(NK, 0), id_o = idesc(64, 1);
      int n_live = 0;
      {
        Item itm;
        for (int it = blockIdx.x; it < n_items; it += gridDim.x) n_live += item_at(it, H, qoff, wdesc, itm) ? 1 : 0;
      }
      // S(j) needs item j's operands (kv_full) and TMEM region j & 1 (r_free of item j-2);
      // P V(j) needs item j's probabilities (p_full).  Both are polled.
      int js = 0, jp = 0;
      while (jp < n_live) {
        if (js < n_live) {
          const int b = js & 1;
          const uint32_t ph = (js >> 1) & 1;
          if (mbar_test(&q_full[b], ph) && mbar_test(&k_full[b], ph) && mbar_test(&r_free[b], ph ^ 1)) {
            // K landed through cp.async (generic proxy): order it before the async-proxy reads
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tc_after();
#pragma unroll
            for (int k = 0; k < 4; ++k)
              mma_ss(tmem + b * AT_REGION, sdesc(sQ(b) + k * 32), sdesc(sK(b) + k * 32), id_s, k > 0);
            mma_commit(&s_full[b]);
            mma_commit(&k_empty[b]);   // K buffer b free once S retired
#ifdef RV_ATTN_TRACE
            AT_TRACE(js, 3);
#endif
            ++js;
            continue;
          }
        }
        if (jp < js) {
          const int b = jp & 1;
          if (mbar_test(&p_full[b], (jp >> 1) & 1) && mbar_test(&v_full[b], (jp >> 1) & 1)) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tc_after();
            for (int k = 0; k < NK / 16; ++k)   // P from TMEM: 16 keys = 8 packed columns per k-step
              mma_ts(tmem + b * AT_REGION + AT_O_OFF, tmem + b * AT_REGION + (uint32_t)(k * 8),
                     sdesc(sV(b) + (uint32_t)(k * 16) * 128), id_o, k > 0);
            mma_commit(&o_full[b]);
            mma_commit(&v_empty[b]);   // V buffer b free once P V retired
#ifdef RV_ATTN_TRACE
            AT_TRACE(jp, 4);
#endif
            ++jp;
          }
        }
      }
    }
  } else {
    // ===================================================== softmax + epilogue (last 16 warps)
    // M = 64 accumulator: tile row r on TMEM lane 32 (r / 16) + r % 16.  Warp (quarter q, sub)
    // covers rows 16 q .. 16 q + 15; with the 16x32bx2 shape lane t < 16 owns row 16 q + t,
    // columns [64 sub, 64 sub + 32), lane t >= 16 row 16 q + t - 16, columns [64 sub + 32, +32).
    const int q = warp & 3, sub = (warp - (AT_WARPS - 16)) >> 2;
    const int hl = lane >> 4;                       // which 32-column half of the warp's 64
    const int row = q * 16 + (lane & 15);           // query row of the tile
    const uint32_t lane_base = (uint32_t)(q * 32) << 16;
    const int pi = sub * 2 + hl;                    // partial index (0..7)
    const int key0 = sub * 64 + hl * 32;            // first S column (= patch key) of this thread
    const int nvalid = max(0, min(32, NP - key0));
    const bool cols = sub * 64 < NK;                // warp-uniform: this warp has S columns
    // Epilogue of item jj (after the softmax of item jj+1): O / l (+ p_cls v_cls) as bf16,
    // the CLS row's probabilities, and the TMEM region handed back to the MMA issuer.  O
    // (M=64, N=64) has the same lane layout; this thread: row, d_h [16 sub + 8 hl, +8).
    auto epilogue = [&](const Item& itm, int jj) {
      const int b = jj & 1;
      const uint32_t reg = tmem + lane_base + b * AT_REGION;
      mbar_wait(&o_full[b], (jj >> 1) & 1);
      tc_after();
      float o[8];
      tld8h(reg + AT_O_OFF + sub * 16, o);
      tld_wait();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&r_free[b]);
      const float* rl = red_l + b * 8 * AT_QROWS;
      float l = 0.f;
#pragma unroll
      for (int k = 0; k < 8; ++k) l += rl[k * AT_QROWS + row];
      const float il = 1.f / l;
      if (row < itm.nrows) {
        const float pc = red_pc[b * AT_QROWS + row];
        const int d0 = sub * 16 + hl * 8;
        const uint4 va = *reinterpret_cast<const uint4*>(sm + sC(jj) + 128 + d0 * 2);
        const uint32_t vw[4] = {va.x, va.y, va.z, va.w};
        uint32_t u[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 vf = unpack_bf16x2(vw[e]);
          u[e] = pack_bf16x2(fmaf(pc, vf.x, o[2 * e]) * il, fmaf(pc, vf.y, o[2 * e + 1]) * il);
        }
        *reinterpret_cast<uint4*>(out + (long long)(itm.q0 + row) * D + itm.h * 64 + d0) =
            make_uint4(u[0], u[1], u[2], u[3]);
      }
      if (pclsh && itm.qt == 0 && q == 0) {   // normalised CLS row (row 0) over the patch keys
        const float il0 = __shfl_sync(0xffffffffu, il, 0);
        const float* cp = clsp + b * AT_MAXK;
        float* dst = pclsh + ((long long)itm.slot * H + itm.h) * NP;
        for (int k = sub * 64 + lane; k < sub * 64 + 64 && k < NP; k += 32) dst[k] = cp[k] * il0;
      }
    };
    Item prev;
    int j = 0;
    for (int it = blockIdx.x; it < n_items; it += gridDim.x) {
      Item itm;
      if (!item_at(it, H, qoff, wdesc, itm)) continue;
      const int b = j & 1;
      const uint32_t reg = tmem + lane_base + b * AT_REGION;
      const bool vrow = row < itm.nrows;
      float* rm = red_m + b * 8 * AT_QROWS;
      mbar_wait(&q_full[b], (j >> 1) & 1);         // Q rows + k_cls visible to this thread
      mbar_wait(&k_full[b], (j >> 1) & 1);
      mbar_wait(&s_full[b], (j >> 1) & 1);
      tc_after();
#ifdef RV_ATTN_TRACE
      if (warp == AT_WARPS - 16 && lane == 0) AT_TRACE(j, 5);
#endif
      float m = -INFINITY, s_cls = -INFINITY;
      if (pi == 0 && vrow) {   // CLS key on the CUDA cores: s_cls = q_row . k_cls
        const uint8_t* qr = sm + (size_t)b * AT_BUF + (size_t)row * 128;
        const uint8_t* kc = sm + sC(j);
        float acc = 0.f;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 qa = *reinterpret_cast<const uint4*>(qr + ((c ^ (row & 7)) << 4));
          const uint4 ka = *reinterpret_cast<const uint4*>(kc + c * 16);
          const uint32_t qw[4] = {qa.x, qa.y, qa.z, qa.w}, kw[4] = {ka.x, ka.y, ka.z, ka.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 qf = unpack_bf16x2(qw[e]), kf = unpack_bf16x2(kw[e]);
            acc = fmaf(qf.x, kf.x, acc);
            acc = fmaf(qf.y, kf.y, acc);
          }
        }
        s_cls = acc;
        m = s_cls;
      }
      float v[32];
      if (cols) {
        tld32h(reg + sub * 64, v);
        tld_wait();
      }
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        if (i >= nvalid) v[i] = -INFINITY;
        m = fmaxf(m, v[i]);
      }
      rm[pi * AT_QROWS + row] = m;
      smx_bar();   // also: every S column of the region has been read before P is written over it
#ifdef RV_ATTN_TRACE
      if (warp == AT_WARPS - 16 && lane == 0) AT_TRACE(j, 9);
#endif
      m = rm[row];
#pragma unroll
      for (int k = 1; k < 8; ++k) m = fmaxf(m, rm[k * AT_QROWS + row]);
      const float ms = m * scale_log2;
      float psum = 0.f;
      uint32_t pk[16];
#pragma unroll
      for (int i = 0; i < 32; i += 2) {
        const float p0 = ex2f_fast(fmaf(v[i], scale_log2, -ms));
        const float p1 = ex2f_fast(fmaf(v[i + 1], scale_log2, -ms));
        psum += p0 + p1;
        pk[i / 2] = pack_bf16x2(p0, p1);
        v[i] = p0;
        v[i + 1] = p1;
      }
      // P over S: keys [64 sub + 32 hl, +32) -> packed columns [32 sub + 16 hl, +16)
      if (cols) {
        tst16h(reg + sub * 32, pk);
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
      }
      if (pclsh && itm.qt == 0 && q == 0 && (lane & 15) == 0) {   // CLS query row: keep p for pclsh
        float* cp = clsp + b * AT_MAXK + key0;
#pragma unroll
        for (int i = 0; i < 32; i += 4) *reinterpret_cast<float4*>(cp + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      }
      if (pi == 0) {
        const float pc = vrow ? ex2f_fast(fmaf(s_cls, scale_log2, -ms)) : 0.f;
        psum += pc;
        red_pc[b * AT_QROWS + row] = pc;
      }
      red_l[b * 8 * AT_QROWS + pi * AT_QROWS + row] = psum;
      tc_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&p_full[b]);
        mbar_arrive(&q_empty[b]);
      }
#ifdef RV_ATTN_TRACE
      if (warp == AT_WARPS - 16 && lane == 0) AT_TRACE(j, 6);
#endif
      if (j > 0) epilogue(prev, j - 1);
#ifdef RV_ATTN_TRACE
      if (warp == AT_WARPS - 16 && lane == 0) AT_TRACE(j, 7);
#endif
      prev = itm;
      ++j;
    }
    if (j > 0) epilogue(prev, j - 1);
  }
  tc_before();
  __syncthreads();
#ifdef RV_ATTN_TRACE
  if (blockIdx.x == 0 && tid == 0) {
    for (int j = 0; j < 64; ++j) {
      const unsigned long long* e = g_at_trace + j * 16;
      printf("T %d %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu\n", j, e[0], e[1], e[2], e[3], e[4], e[5], e[6],
             e[7], e[8], e[9]);
    }
  }
#endif
  if (warp == 1) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(AT_TMEM_COLS));
  }
}

}  // namespace

bool attn_tc_supported(int T, int D, int H) { return H > 0 && D / H == 64 && D % H == 0 && T >= 2 && T - 1 <= AT_MAXK; }

size_t attn_tc_smem() { return 2 * (size_t)AT_BUF + 1024 + 4 * AT_MAXK * 4 + 34 * AT_QROWS * 4 + 20 * 8 + 16; }

cudaError_t launch_attention_tc(const CUtensorMap& tmQ, const bf16* KV, const int* kvsrc, bf16* out,
                                const int* wdesc, const int* qoff, float* pclsh, int n_w, int T, int D, int H,
                                cudaStream_t s) {
  if (n_w <= 0) return cudaSuccess;
  if (!attn_tc_supported(T, D, H)) return cudaErrorInvalidValue;
  const size_t smem = attn_tc_smem();
  static size_t attr = 0;
  if (smem > attr) {
    cudaError_t e = cudaFuncSetAttribute(attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    attr = smem;
  }
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int items = n_w * H * AT_MAX_TILES;
  const int grid = items < sms ? items : sms;
  const float scale_log2 = 1.4426950408889634f / 8.0f;   // 1/sqrt(64) * log2(e)
  attn_tc_kernel<<<grid, AT_THREADS, smem, s>>>(tmQ, KV, kvsrc, out, reinterpret_cast<const int4*>(wdesc), qoff,
                                                pclsh, n_w, T, D, H, scale_log2);
  return cudaGetLastError();
}

}  // namespace rv
