// k_attn_tc.cu — attention of the compacted queries over all T keys of their frame on the
// 5th-generation tensor cores (P:313 every recomputed query attends to all
// tokens; P:336 CLS attention row = feature t).  d_h = 64 and T - 1 <= 256 patch keys (CLIP
// B/16, L/14 at 224 px); the mma.sync kernel of k_attn.cu covers the other shapes.
//
// Work item = (frame of the wave, head, 64-row query tile), a CTA taking whole frame-heads and
// running their tiles back to back on one K / V gather (A8_KV_SHARE); ~47-57 of a frame's 257 queries
// are recomputed at the paper's reuse rates, so the MMA M is 64 (accumulator rows on lanes
// 0-15 or 16-31 of each TMEM lane quarter).  Per item the kernel gathers 66 KB of K/V (rows
// scattered through `kvsrc`) for ~2 MFLOP, so it is built to keep bytes in flight and to
// spend few tcgen05.mma instructions (each costs >= ~93 cycles of issue on B200 whatever its
// N, tools/umma_rate.cu): S = Q K^T is 4 MMAs of N = 256 (all patch keys), P V 16 of N = 64.
//   warps 0-1  loaders.  Both scan the CTA's item slots 32 at a time (ballot) in the same
//              order; warp 0 also TMA-loads the Q tile and the CLS key's K / V rows and
//              publishes the item descriptor.  Each warp gathers half of the 256 patch keys'
//              K and V rows (128 B each per row and head, adjacent in the head-interleaved
//              cache row (k_h v_h); `kvsrc` indirection: the reuse cache is
//              read in place) with cp.async into SWIZZLE_128B tiles (a 2-slot K ring and a
//              3-slot V ring of 32 KB tiles); completion is counted on the
//              tile's mbarrier (cp.async.mbarrier.arrive.noinc), so loaders never wait for data.
//   warp 2     TMEM allocator + single-thread MMA issuer, polling: S(j) when its Q, K tile
//              and region are ready, P V(j) when its P and V tile are ready (neither waits
//              behind the other's inputs).  Item j uses TMEM region j % 4
//              (lane half (j & 1), column half (j >> 1) & 1: M = 64 fills half the lanes).
//   warps 4-11 two softmax groups of 4 warps (one per TMEM lane quarter); group g owns items
//              j = g (mod 2).  One row per lane pair (16x32bx2 shape: lane t < 16 keys
//              [0, 128), lane t + 16 keys [128, 256)), so the row max / sum need one shuffle
//              and no barrier; P (bf16) is stored over S; the CLS key (k_cls, v_cls) is done on
//              the CUDA cores; the epilogue writes O / l as bf16 and the normalised CLS row (t).
// Region: S [0, 256), P packed over [0, 128), O [128, 192).
#include <cuda.h>
#include <cstdio>

#include "common.cuh"
#include "rv_internal.h"

namespace rv {
namespace {

constexpr int A8_WARPS = 12;
constexpr int A8_THREADS = A8_WARPS * 32;
constexpr int A8_SMX0 = 4;                     // first softmax warp
constexpr int A8_LOADERS = 64;                 // cp.async lanes (warps 0-1)
constexpr int A8_QROWS = 64;                   // M of both MMAs
constexpr int A8_MAXK = 256;                   // patch keys per item
constexpr int A8_MAX_TILES = 5;                // T <= 257 -> <= 257 compact queries per frame
#ifndef A8_NKT_SLOTS
#define A8_NKT_SLOTS 2
#endif
#ifndef A8_NVT_SLOTS
#define A8_NVT_SLOTS 3
#endif
constexpr int A8_NKT = A8_NKT_SLOTS;           // K tile ring slots
constexpr int A8_NVT = A8_NVT_SLOTS;           // V tile ring slots
constexpr int A8_NT = A8_NKT + A8_NVT;
#ifndef A8_NQ_SLOTS
#define A8_NQ_SLOTS 4
#endif
// A8_PAIR_PV: items come in head pairs (h, h+1) of the same frame and query tile; their P V is
// one M = 128, N = 128 MMA per 16 keys (P of both items in the two TMEM lane halves, V of both
// heads as one MN-major operand over two adjacent V slots), 16 instead of 32 instructions
#ifndef A8_PAIR_PV
#define A8_PAIR_PV 0
#endif
static_assert(!A8_PAIR_PV || A8_NVT_SLOTS % 2 == 0, "pair P V needs an even V ring");
// A8_KV_SHARE: a CTA takes whole frame-heads and runs all of their query tiles back to back on
// one K / V gather (frames with > 64 recomputed queries, e.g. I frames with 257 = 5 tiles,
// otherwise re-gather the same 64 KB per tile); the tiles stay in their ring slots until the
// frame-head's last tile has used them
#ifndef A8_KV_SHARE
#define A8_KV_SHARE 1
#endif
static_assert(!(A8_KV_SHARE && A8_PAIR_PV), "A8_KV_SHARE and A8_PAIR_PV are exclusive");
constexpr int A8_NQ = A8_NQ_SLOTS;             // Q ring slots (items the loader may run ahead)
constexpr uint32_t A8_TILE = A8_MAXK * 128;    // 256 keys x 128 B
// Q tile, then the CLS key's K row at +8192 (row 0 of a 1 KB swizzle atom: unswizzled) and its
// V row at +8320 (row 1: 16 B chunk c stored at chunk c ^ 1)
constexpr uint32_t A8_QSLOT = 8192 + 1024;
constexpr uint32_t A8_QTX = 8192 + 256;        // bytes the Q slot's TMA deliver
constexpr uint32_t A8_RING = A8_NQ * A8_QSLOT; // tile ring offset (1 KB aligned)
constexpr uint32_t A8_ROWS = A8_RING + A8_NT * A8_TILE;   // int32 [A8_NQ][256] K/V source rows
constexpr uint32_t A8_META = A8_ROWS + A8_NQ * A8_MAXK * 4;
constexpr uint32_t A8_TMEM_COLS = 512;
constexpr uint32_t A8_O_OFF = 128;
#ifndef A8_POLL_SLEEP
#define A8_POLL_SLEEP 0
#endif
#ifndef A8_DEFER_EPI
#define A8_DEFER_EPI 0
#endif
#ifndef A8_POLY8
#define A8_POLY8 0   // of every 8 score pairs, this many take the FMA-pipe exp2 (rest: MUFU)
#endif

struct Meta {   // item descriptor written by loader warp 0, read by the MMA issuer and softmax
  int q0, nrows, slot, h, qt, done;
  int kv_first, kv_last;   // first / last query tile on this K / V gather (A8_KV_SHARE)
};

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
// MN-major (b_mn = 1), N >> 3 at bit 17, M >> 4 at bit 24 (M = 64).
RV_DEV uint32_t idesc64(int N, int b_mn, int M = A8_QROWS) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)b_mn << 16) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}
// MN-major operand spanning two 64-wide N blocks `lbo` bytes apart (leading byte offset)
[[maybe_unused]] RV_DEV uint64_t sdesc_lbo(uint32_t addr, uint32_t lbo) {
  return sdesc(addr) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16);
}
// 16x32bx2 shapes: lanes 0-15 access TMEM lanes base..base+15 at columns [c, c+n), lanes 16-31
// the same TMEM lanes at columns [c+OFF, c+OFF+n).
template <int OFF>
RV_DEV void tld32h(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.16x32bx2.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32], %33;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr), "n"(OFF));
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
template <int OFF>
RV_DEV void tst16h(uint32_t taddr, const uint32_t* r) {
  asm volatile(
      "tcgen05.st.sync.aligned.16x32bx2.x16.b32 [%0], %17, {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(
          taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "n"(OFF)
      : "memory");
}
RV_DEV void tld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
RV_DEV void tst_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

RV_DEV void tma_2d(uint32_t dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(tm), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}

#ifdef RV_A8_TRACE   // experiment builds: per-item event timeline of CTA 0 (printed at exit)
RV_DEV unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ unsigned long long g_a8_trace[64 * 12];
#define A8_TR(j, k) do { if (blockIdx.x == 0 && (j) < 64) g_a8_trace[(j) * 12 + (k)] = gtime(); } while (0)
#else
#define A8_TR(j, k) do { } while (0)
#endif

RV_DEV float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
RV_DEV unsigned long long f2pack(float a, float b) {
  unsigned long long r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
RV_DEV float2 f2unpack(unsigned long long r) {
  float2 v;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(v.x), "=f"(v.y) : "l"(r));
  return v;
}
RV_DEV unsigned long long ffma2(unsigned long long a, unsigned long long b, unsigned long long c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
RV_DEV unsigned long long fadd2(unsigned long long a, unsigned long long b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
// 2^x for a pair of x <= 0 on the FMA pipe: x = n + f, n = round(x) (1.5 * 2^23 shifter),
// 2^f on [-0.5, 0.5] by its degree-3 Taylor polynomial (relative error <= 6.2e-4, below the
// bf16 rounding of P), 2^n added to the exponent field.  x is clamped at -127 (2^-127 ~ 0).
RV_DEV float2 exp2_poly2(unsigned long long x2) {
  float2 x = f2unpack(x2);
  x.x = fmaxf(x.x, -127.f);
  x.y = fmaxf(x.y, -127.f);
  const unsigned long long sh = f2pack(12582912.f, 12582912.f);
  const unsigned long long t = fadd2(f2pack(x.x, x.y), sh);
  const unsigned long long nf = fadd2(t, f2pack(-12582912.f, -12582912.f));
  const unsigned long long f = ffma2(nf, f2pack(-1.f, -1.f), f2pack(x.x, x.y));
  unsigned long long p = ffma2(f2pack(0.0555041087f, 0.0555041087f), f, f2pack(0.240226507f, 0.240226507f));
  p = ffma2(p, f, f2pack(0.693147181f, 0.693147181f));
  p = ffma2(p, f, f2pack(1.f, 1.f));
  const float2 tv = f2unpack(t), pv = f2unpack(p);
  return make_float2(__int_as_float((__float_as_int(tv.x) << 23) + __float_as_int(pv.x)),
                     __int_as_float((__float_as_int(tv.y) << 23) + __float_as_int(pv.y)));
}
// A8_L2_PREFETCH (experiment knob): L2 fetch size hint of the K/V gathers.  Bench at 7,200
// frames: attention 83.5 ms (none), 82.4 (256 B), 82.6 (128 B): within run-to-run noise.
#ifndef A8_L2_PREFETCH
#define A8_L2_PREFETCH 0
#endif
RV_DEV void cp_async16(uint32_t dst, const void* src) {
#if A8_L2_PREFETCH == 256
  // L2 fetches the 256 B block: the row's K (or V) of the paired head h ^ 1, which a
  // neighbouring CTA gathers at about the same time (item slots walk the heads fastest)
  asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
#elif A8_L2_PREFETCH == 128
  asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
#else
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
#endif
}
// TMEM address of region j % 4: lane half (j & 1) -> lane offset 16, column half (j >> 1) & 1
RV_DEV uint32_t region(uint32_t tmem, int j) {
  return tmem + ((uint32_t)((j & 1) * 16) << 16) + (uint32_t)(((j >> 1) & 1) * 256);
}

__global__ void __launch_bounds__(A8_THREADS, 1)
    attn_tc_kernel(const __grid_constant__ CUtensorMap tmQ, const __grid_constant__ CUtensorMap tmKV,
                   const bf16* __restrict__ KV, const int* __restrict__ kvsrc, bf16* __restrict__ out,
                   const int4* __restrict__ wdesc, const int* __restrict__ qoff, float* __restrict__ pclsh,
                   int n_w, int T, int D, int H, float scale_log2) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const int NP = T - 1;                          // patch keys
  const uint32_t base = su32(sm);
  int* rowsbuf = reinterpret_cast<int*>(sm + A8_ROWS);                     // [A8_NQ][256]
  Meta* meta = reinterpret_cast<Meta*>(sm + A8_META);                       // [A8_NQ]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + A8_META + A8_NQ * sizeof(Meta));
  // t_full / t_empty: K ring slots 0 .. A8_NKT-1, then V ring slots
  uint64_t *q_full = bar, *q_empty = bar + A8_NQ, *t_full = bar + 2 * A8_NQ, *t_empty = t_full + A8_NT,
           *s_full = t_empty + A8_NT, *p_full = s_full + 4, *o_full = p_full + 4, *r_free = o_full + 4;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(r_free + 4);
  auto sQ = [&](int s) { return base + (uint32_t)s * A8_QSLOT; };
  auto sT = [&](uint32_t s) { return base + A8_RING + s * A8_TILE; };

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQ) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmKV) : "memory");
    for (int i = 0; i < A8_NQ; ++i) {
      mbar_init(&q_full[i], 1);    // loader's expect_tx arrival (+ TMA bytes), or the end marker
      mbar_init(&q_empty[i], 4);   // the owning softmax group's 4 warps, after the epilogue
    }
    for (int i = 0; i < A8_NT; ++i) {
      mbar_init(&t_full[i], A8_LOADERS);   // every loader lane's cp.async (arrive.noinc)
      mbar_init(&t_empty[i], 1);           // tcgen05.commit after the tile's MMAs
    }
    for (int i = 0; i < 4; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&o_full[i], 1);
      mbar_init(&r_free[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)),
                 "r"(A8_TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tslot;
  // Register split (whole warpgroups, each setmaxnreg inside its role's branch so that ptxas
  // sizes every role by its own limit): loaders / MMA / idle warp 3 give registers to the
  // softmax warps, whose row of 128 fp32 scores stays in registers without spilling.
#define A8_REG_DEC() asm volatile("setmaxnreg.dec.sync.aligned.u32 80;" ::: "memory")
#define A8_REG_INC() asm volatile("setmaxnreg.inc.sync.aligned.u32 208;" ::: "memory")
  if (warp < 2) {
    A8_REG_DEC();
    // ======================================================================== loaders
    // Item slots it = blockIdx.x + k * gridDim.x over (qt, w, h), qt slowest: the first n_w*H
    // slots (tile 0 of every frame-head) are all live; later tiles exist for large frames only.
    constexpr int HP = A8_PAIR_PV ? 2 : 1;        // heads per item slot
    const int Hs = H / HP;
    const long long n_items = (long long)n_w * Hs * (A8_KV_SHARE ? 1 : A8_MAX_TILES);
    const long long per_t = (long long)n_w * Hs;
    const long long ld = 2LL * D;
    const int half = warp;          // this warp gathers patch keys [128 half, 128 half + 128)
    uint32_t kseq = 0, vseq = 0;    // K / V tile sequence numbers
    int j = 0;                      // live item counter
    long long it0 = blockIdx.x;
    uint32_t ball = 0;
    int b_q0 = 0, b_nr = 0, b_sl = 0, b_h = 0, b_qt = 0;
    auto next_item = [&](int& iq0, int& inr, int& isl, int& ih, int& iqt) -> bool {
      while (ball == 0) {
        if (it0 >= n_items) return false;
        const long long my = it0 + (long long)lane * gridDim.x;
        int live = 0;
        if (my < n_items) {
          b_qt = (int)(my / per_t);
          const int rem = (int)(my - (long long)b_qt * per_t);
          const int w = rem / Hs;
          b_h = (rem - w * Hs) * HP;
          const int a = __ldg(qoff + w), nq = __ldg(qoff + w + 1) - a;
          live = b_qt * A8_QROWS < nq;
          b_q0 = a + b_qt * A8_QROWS;
          // A8_KV_SHARE: the whole frame-head (all nq queries); otherwise one 64-row tile
          b_nr = A8_KV_SHARE ? nq : min(A8_QROWS, nq - b_qt * A8_QROWS);
          b_sl = __ldg(&wdesc[w].x);
        }
        ball = __ballot_sync(0xffffffffu, live);
        it0 += 32LL * gridDim.x;
      }
      const int src = __ffs(ball) - 1;
      ball &= ball - 1;
      iq0 = __shfl_sync(0xffffffffu, b_q0, src);
      inr = __shfl_sync(0xffffffffu, b_nr, src);
      isl = __shfl_sync(0xffffffffu, b_sl, src);
      ih = __shfl_sync(0xffffffffu, b_h, src);
      iqt = __shfl_sync(0xffffffffu, b_qt, src);
      return true;
    };
    // K/V source rows of this lane's 4 patch keys 128 half + 4 lane + i (padding keys read the
    // frame's own CLS row: finite data, masked in the softmax)
    auto load_rows = [&](int isl, int (&rows)[4]) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int k = 128 * half + 4 * lane + i;
        rows[i] = k < NP ? (kvsrc ? __ldg(kvsrc + (long long)isl * T + 1 + k) : isl * T + 1 + k) : isl * T;
      }
    };
    // 128 rows x 128 B of column block `col` into the next K or V tile slot (rows 128 half ..):
    // per instruction 8 consecutive lanes copy one 128 B row, 4 rows per warp instruction;
    // the source rows come from the item's row table in shared memory, 8 at a time.
    auto issue_tile = [&](int col, const int* rb, bool is_v) {
      uint32_t& seq = is_v ? vseq : kseq;
      const uint32_t nslot = is_v ? A8_NVT : A8_NKT;
      const uint32_t s = (is_v ? A8_NKT : 0) + seq % nslot;
      mbar_wait(&t_empty[s], ((seq / nslot) & 1) ^ 1);
#ifndef RV_A8_NO_KV
      const uint32_t dst = sT(s);
      const int c = lane & 7;
      const bf16* src0 = KV + col + c * 8;
      const int* rl = rb + 128 * half + (lane >> 3);
#pragma unroll 1
      for (int b = 0; b < 32; b += 8) {
        int r8[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) r8[i] = rl[4 * (b + i)];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int kr = 128 * half + 4 * (b + i) + (lane >> 3);
          cp_async16(dst + (uint32_t)kr * 128 + ((c ^ (kr & 7)) << 4), src0 + (long long)r8[i] * ld);
        }
      }
#endif
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(su32(&t_full[s])) : "memory");
      ++seq;
    };
    int c_q0, c_nr, c_sl, c_h, c_qt, rows[4];
    bool have = next_item(c_q0, c_nr, c_sl, c_h, c_qt);
    if (have) load_rows(c_sl, rows);
    while (have) {
      // the next item's descriptor and row indices are fetched first: their latency overlaps
      // the waits and copies of the current item
      int n_q0 = 0, n_nr = 0, n_sl = 0, n_h = 0, n_qt = 0, nrows_[4];
      const bool nhave = next_item(n_q0, n_nr, n_sl, n_h, n_qt);
      if (nhave) load_rows(n_sl, nrows_);
#if A8_KV_SHARE
      const int ntile = (c_nr + A8_QROWS - 1) / A8_QROWS;
#pragma unroll 1
      for (int qt = 0; qt < ntile; ++qt) {   // the frame-head's query tiles on one K / V gather
        const int je = j + qt;
        const int qs = je % A8_NQ;
        mbar_wait(&q_empty[qs], ((je / A8_NQ) & 1) ^ 1);
        if (warp == 0 && lane == 0) {
          A8_TR(je, 0);
          Meta& m = meta[qs];
          m.q0 = c_q0 + qt * A8_QROWS; m.nrows = min(A8_QROWS, c_nr - qt * A8_QROWS); m.slot = c_sl; m.h = c_h;
          m.qt = qt; m.done = 0; m.kv_first = qt == 0; m.kv_last = qt == ntile - 1;
          mbar_expect_tx(&q_full[qs], A8_QTX);
          tma_2d(sQ(qs), &tmQ, c_h * 64, m.q0, &q_full[qs]);
          tma_2d(sQ(qs) + 8192, &tmKV, c_h * 128, c_sl * T, &q_full[qs]);       // k_cls
          tma_2d(sQ(qs) + 8320, &tmKV, c_h * 128 + 64, c_sl * T, &q_full[qs]);   // v_cls
        }
        if (qt == 0) {
          int* rb = rowsbuf + qs * A8_MAXK;
          *reinterpret_cast<int4*>(rb + 128 * half + 4 * lane) = make_int4(rows[0], rows[1], rows[2], rows[3]);
          __syncwarp();
          // K and V of head h are adjacent in the token's cache row (k_h v_h): issuing both
          // rows' 256 B in one instruction (joint K + V slots) measured neutral (r2t: 66.4 vs
          // 66.9 ms per step), as did an L2::256B fetch hint on these copies (66.1)
          issue_tile(c_h * 128, rb, false);                                   // K(frame-head)
          if (warp == 0 && lane == 0) A8_TR(je, 1);
          issue_tile(c_h * 128 + 64, rb, true);                                // V(frame-head)
          if (warp == 0 && lane == 0) A8_TR(je, 2);
        }
      }
#else
      int* rb = nullptr;
#pragma unroll 1
      for (int e = 0; e < HP; ++e) {        // items j, (j + 1): heads c_h, (c_h + 1)
        const int je = j + e, he = c_h + e;
        const int qs = je % A8_NQ;
        mbar_wait(&q_empty[qs], ((je / A8_NQ) & 1) ^ 1);
        if (warp == 0 && lane == 0) {
          A8_TR(je, 0);
          Meta& m = meta[qs];
          m.q0 = c_q0; m.nrows = c_nr; m.slot = c_sl; m.h = he; m.qt = c_qt; m.done = 0;
          mbar_expect_tx(&q_full[qs], A8_QTX);
          tma_2d(sQ(qs), &tmQ, he * 64, c_q0, &q_full[qs]);
          tma_2d(sQ(qs) + 8192, &tmKV, he * 128, c_sl * T, &q_full[qs]);       // k_cls
          tma_2d(sQ(qs) + 8320, &tmKV, he * 128 + 64, c_sl * T, &q_full[qs]);   // v_cls
        }
        if (e == 0) {   // the pair shares its frame's rows: the first item's table serves both
          rb = rowsbuf + qs * A8_MAXK;
          *reinterpret_cast<int4*>(rb + 128 * half + 4 * lane) = make_int4(rows[0], rows[1], rows[2], rows[3]);
          __syncwarp();
        }
        issue_tile(he * 128, rb, false);                                      // K(je)
        if (warp == 0 && lane == 0) A8_TR(je, 1);
        if (!A8_PAIR_PV) issue_tile(he * 128 + 64, rb, true);                  // V(je)
      }
      if (A8_PAIR_PV) {                       // V(j), V(j + 1) into adjacent slots
        issue_tile(c_h * 128 + 64, rb, true);
        issue_tile((c_h + 1) * 128 + 64, rb, true);
      }
      if (warp == 0 && lane == 0) A8_TR(j, 2);
#endif
#pragma unroll
      for (int i = 0; i < 4; ++i) rows[i] = nrows_[i];
      c_q0 = n_q0; c_nr = n_nr; c_sl = n_sl; c_h = n_h; c_qt = n_qt;
      have = nhave;
#if A8_KV_SHARE
      j += ntile;
#else
      j += HP;
#endif
    }
    // end markers in the next two Q slots: each softmax group waits only on its own items
    if (warp == 0)
      for (int e = 0; e < 2; ++e, ++j) {
        const int qs = j % A8_NQ;
        mbar_wait(&q_empty[qs], ((j / A8_NQ) & 1) ^ 1);
        if (lane == 0) {
          meta[qs].done = 1;
          mbar_arrive(&q_full[qs]);
        }
      }
  } else if (warp == 2) {
    A8_REG_DEC();
    // ======================================================================== MMA issuer
    if (lane == 0) {
      // Polling issuer: S(js) as soon as its Q, K tile and TMEM region are ready, P V(jp) as
      // soon as its P and V tile are ready, so neither waits behind the other's inputs.
      const uint32_t id_s = idesc64(256, 0), id_o = idesc64(64, 1);
      const uint32_t id_o2 = idesc64(128, 1, 128);   // pair P V: M = 128, N = 128 (A8_PAIR_PV)
      (void)id_o;
      (void)id_o2;
      uint32_t kseq = 0, vseq = 0;
      int js = 0, jp = 0, j_end = 0x7fffffff;
      while (jp < j_end) {
        const int js0 = js, jp0 = jp;
        (void)js0;
        (void)jp0;
        if (js < j_end) {
          const int qs = js % A8_NQ;
          if (mbar_test(&q_full[qs], (js / A8_NQ) & 1)) {
            if (meta[qs].done) {
              j_end = js;
              continue;
            }
            const uint32_t ks = kseq % A8_NKT;
            const bool kf = !A8_KV_SHARE || meta[qs].kv_first, kl = !A8_KV_SHARE || meta[qs].kv_last;
            if (mbar_test(&r_free[js & 3], ((js >> 2) & 1) ^ 1) && (!kf || mbar_test(&t_full[ks], (kseq / A8_NKT) & 1))) {
              A8_TR(js, 3);
              asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // cp.async data -> tensor core
              tc_after();
              const uint32_t reg = region(tmem, js);
#pragma unroll
              for (int k = 0; k < 4; ++k)   // S = Q K^T over all 256 patch keys, 16 d_h per step
                mma_ss(reg, sdesc(sQ(qs) + k * 32), sdesc(sT(ks) + k * 32), id_s, k != 0);
              if (kl) {                      // the K tile's last user: release the slot
                mma_commit(&t_empty[ks]);
                ++kseq;
              }
              mma_commit(&s_full[js & 3]);
              A8_TR(js, 4);
              ++js;
            }
          }
        }
#if A8_PAIR_PV
        if (jp + 1 < js) {
          const uint32_t vs = A8_NKT + vseq % A8_NVT;   // V(jp) at slot vs, V(jp + 1) at vs + 1
          if (mbar_test(&p_full[jp & 3], (jp >> 2) & 1) && mbar_test(&p_full[(jp + 1) & 3], ((jp + 1) >> 2) & 1) &&
              mbar_test(&t_full[vs], (vseq / A8_NVT) & 1) && mbar_test(&t_full[vs + 1], (vseq / A8_NVT) & 1)) {
            A8_TR(jp, 5);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tc_after();
            const uint32_t reg = region(tmem, jp);   // lane half 0: M = 128 spans both items' rows
#pragma unroll 4
            for (int k = 0; k < A8_MAXK / 16; ++k)
              mma_ts(reg + A8_O_OFF, reg + (uint32_t)(k * 8), sdesc_lbo(sT(vs) + (uint32_t)k * 2048, A8_TILE), id_o2,
                     k != 0);
            mma_commit(&t_empty[vs]);
            mma_commit(&t_empty[vs + 1]);
            mma_commit(&o_full[jp & 3]);
            mma_commit(&o_full[(jp + 1) & 3]);
            A8_TR(jp, 6);
            vseq += 2;
            jp += 2;
          }
        }
#else
        if (jp < js) {
          const uint32_t vs = A8_NKT + vseq % A8_NVT;
          const int qsp = jp % A8_NQ;   // the item's Q slot (and meta) live until its epilogue
          const bool vf = !A8_KV_SHARE || meta[qsp].kv_first, vl = !A8_KV_SHARE || meta[qsp].kv_last;
          if (mbar_test(&p_full[jp & 3], (jp >> 2) & 1) && (!vf || mbar_test(&t_full[vs], (vseq / A8_NVT) & 1))) {
            A8_TR(jp, 5);
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tc_after();
            const uint32_t reg = region(tmem, jp);
#pragma unroll 4
            for (int k = 0; k < A8_MAXK / 16; ++k)   // O = P V: 16 keys per MMA, P packed columns 8 k
              mma_ts(reg + A8_O_OFF, reg + (uint32_t)(k * 8), sdesc(sT(vs) + (uint32_t)k * 2048), id_o, k != 0);
            if (vl) {                        // the V tile's last user: release the slot
              mma_commit(&t_empty[vs]);
              ++vseq;
            }
            mma_commit(&o_full[jp & 3]);
            A8_TR(jp, 6);
            ++jp;
          }
        }
#endif
#if A8_POLL_SLEEP > 0
        // nothing issuable: back off so the polling does not steal issue slots from the softmax
        // warps sharing this SM sub-partition
        if (js == js0 && jp == jp0) __nanosleep(A8_POLL_SLEEP);
#endif
      }
    }
  } else if (warp < A8_SMX0) {
    A8_REG_DEC();   // idle warp of the first warpgroup
  } else {
    A8_REG_INC();
    // ======================================================================== softmax groups
    const int g = (warp - A8_SMX0) >> 2;           // items j = g (mod 2)
    const int q = warp & 3;                        // TMEM lane quarter this warp may access
    const int hl = lane >> 4;                      // key half: [0,128) or [128,256)
    const int row = q * 16 + (lane & 15);          // tile row
    // softmax of item j (S -> P in TMEM, row sum l and CLS-key weight pc returned)
    auto softmax = [&](int j, const Meta& m, int qs, float& l, float& pc) {
      const int r = j & 3;
      // region of item j: this warp's 16 lanes (quarter q, lane half j & 1)
      const uint32_t reg = region(tmem, j) + ((uint32_t)(q * 32) << 16);
      const bool act = q * 16 < m.nrows;          // warp-uniform: this quarter has live rows
      mbar_wait(&s_full[r], (j >> 2) & 1);
      if (q == 0 && lane == 0) A8_TR(j, 7);
      tc_after();
      l = 1.f;
      pc = 0.f;
      if (act) {
        float v[128];
#pragma unroll
        for (int i = 0; i < 4; ++i) tld32h<128>(reg + 32 * i, v + 32 * i);
        // CLS key on the CUDA cores while the TMEM loads are in flight:
        // s_cls = q_row . k_cls (this lane: d_h [32 hl, 32 hl + 32))
        const uint8_t* qr = sm + (size_t)qs * A8_QSLOT + (size_t)row * 128;
        const uint8_t* kc = sm + (size_t)qs * A8_QSLOT + 8192;
        float sc = 0.f;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const int ch = hl * 4 + c;
          const uint4 qa = *reinterpret_cast<const uint4*>(qr + ((ch ^ (row & 7)) << 4));
          const uint4 ka = *reinterpret_cast<const uint4*>(kc + ch * 16);
          const uint32_t qw[4] = {qa.x, qa.y, qa.z, qa.w}, kw[4] = {ka.x, ka.y, ka.z, ka.w};
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const float2 qf = unpack_bf16x2(qw[e]), kf = unpack_bf16x2(kw[e]);
            sc = fmaf(qf.x, kf.x, sc);
            sc = fmaf(qf.y, kf.y, sc);
          }
        }
        sc += __shfl_xor_sync(0xffffffffu, sc, 16);
        tld_wait();
        if (NP < A8_MAXK) {
#pragma unroll
          for (int i = 0; i < 128; ++i)
            if (hl * 128 + i >= NP) v[i] = -INFINITY;
        }
        // row max (3-input FMNMX), exponent argument (FFMA2) and row sum (FADD2) in
        // independent chains of paired fp32 values
        float mx4[4] = {sc, sc, sc, sc};
#pragma unroll
        for (int i = 0; i < 128; i += 8) {
          mx4[0] = fmax3(mx4[0], v[i], v[i + 1]);
          mx4[1] = fmax3(mx4[1], v[i + 2], v[i + 3]);
          mx4[2] = fmax3(mx4[2], v[i + 4], v[i + 5]);
          mx4[3] = fmax3(mx4[3], v[i + 6], v[i + 7]);
        }
        float mx = fmax3(mx4[0], mx4[1], fmaxf(mx4[2], mx4[3]));
        mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
        const float ms = mx * scale_log2;
        const unsigned long long sc2 = f2pack(scale_log2, scale_log2), nm2 = f2pack(-ms, -ms);
        unsigned long long acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
        for (int i = 0; i < 128; i += 2) {
          const unsigned long long x2 = ffma2(f2pack(v[i], v[i + 1]), sc2, nm2);
          float2 e;
          if (((i >> 1) & 7) < A8_POLY8) {
            e = exp2_poly2(x2);   // FMA-pipe exp2 for part of the row: the MUFU pipe is the limit
          } else {
            const float2 x = f2unpack(x2);
            e = make_float2(ex2f_fast(x.x), ex2f_fast(x.y));
          }
          v[i] = e.x;
          v[i + 1] = e.y;
          acc[(i >> 1) & 3] = fadd2(acc[(i >> 1) & 3], f2pack(e.x, e.y));
        }
        pc = ex2f_fast(fmaf(sc, scale_log2, -ms));
        const float2 s01 = f2unpack(fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3])));
        const float sum = s01.x + s01.y;
        l = sum + __shfl_xor_sync(0xffffffffu, sum, 16) + pc;
        if (pclsh && m.qt == 0 && q == 0 && (lane & 15) == 0) {   // CLS query row: normalised p
          const float il = 1.f / l;
          float* dst = pclsh + ((long long)m.slot * H + m.h) * NP + hl * 128;
          if (NP == A8_MAXK) {
#pragma unroll
            for (int i = 0; i < 128; i += 4)
              *reinterpret_cast<float4*>(dst + i) = make_float4(v[i] * il, v[i + 1] * il, v[i + 2] * il, v[i + 3] * il);
          } else {
#pragma unroll
            for (int i = 0; i < 128; ++i)
              if (hl * 128 + i < NP) dst[i] = v[i] * il;
          }
        }
        // P over S: keys [128 hl + 32 i, +32) -> packed columns 64 hl + 16 i
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          uint32_t pk[16];
#pragma unroll
          for (int e = 0; e < 16; ++e) pk[e] = pack_bf16x2(v[32 * i + 2 * e], v[32 * i + 2 * e + 1]);
          tst16h<64>(reg + 16 * i, pk);
        }
        tst_wait();
      }
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[r]);
      if (q == 0 && lane == 0) A8_TR(j, 8);
    };
    // epilogue of item j: O / l (+ p_cls v_cls) as bf16; this lane: row, d_h [32 hl, 32 hl + 32)
    auto epilogue = [&](int j, const Meta& m, int qs, float l, float pc) {
      const int r = j & 3;
      const uint32_t reg = region(tmem, j) + ((uint32_t)(q * 32) << 16);
      const bool act = q * 16 < m.nrows;
      mbar_wait(&o_full[r], (j >> 2) & 1);
      if (q == 0 && lane == 0) A8_TR(j, 9);
      tc_after();
      if (act) {
        float o[32];
        // pair P V: item j + 1 (odd) takes head h + 1's columns of the shared accumulator
        tld32h<32>(reg + A8_O_OFF + (A8_PAIR_PV ? (uint32_t)((j & 1) * 64) : 0u), o);
        tld_wait();
        if (row < m.nrows) {
          const float il = 1.f / l;
          const uint8_t* vc = sm + (size_t)qs * A8_QSLOT + 8320;
          bf16* dst = out + (long long)(m.q0 + row) * D + m.h * 64 + hl * 32;
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            const uint4 va = *reinterpret_cast<const uint4*>(vc + (((hl * 4 + c) ^ 1) << 4));
            const uint32_t vw[4] = {va.x, va.y, va.z, va.w};
            uint32_t u[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 vf = unpack_bf16x2(vw[e]);
              u[e] = pack_bf16x2(fmaf(pc, vf.x, o[8 * c + 2 * e]) * il, fmaf(pc, vf.y, o[8 * c + 2 * e + 1]) * il);
            }
            *reinterpret_cast<uint4*>(dst + 8 * c) = make_uint4(u[0], u[1], u[2], u[3]);
          }
        }
      }
      tc_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&r_free[r]);
        mbar_arrive(&q_empty[qs]);
      }
      if (q == 0 && lane == 0) A8_TR(j, 10);
    };
    // Items j = g, g + 2, ...  A8_DEFER_EPI: run an item's epilogue after the softmax of the
    // group's next item (hides P V latency, but holds the item's Q slot and TMEM region longer).
    int jp = -1, qsp = 0;
    Meta mp;
    float lp = 1.f, pcp = 0.f;
    for (int j = g;; j += 2) {
      const int qs = j % A8_NQ;
      mbar_wait(&q_full[qs], (j / A8_NQ) & 1);
      const Meta m = meta[qs];
      if (m.done) break;
      float l, pc;
      softmax(j, m, qs, l, pc);
      if (!A8_DEFER_EPI) {
        epilogue(j, m, qs, l, pc);
        continue;
      }
      if (jp >= 0) epilogue(jp, mp, qsp, lp, pcp);
      jp = j;
      qsp = qs;
      mp = m;
      lp = l;
      pcp = pc;
    }
    if (jp >= 0) epilogue(jp, mp, qsp, lp, pcp);
  }
  tc_before();
  __syncthreads();
#ifdef RV_A8_TRACE
  if (blockIdx.x == 0 && tid == 0)
    for (int j = 0; j < 64; ++j) {
      const unsigned long long* e = g_a8_trace + j * 12;
      printf("A8 %d %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu %llu\n", j, e[0], e[1], e[2], e[3], e[4], e[5],
             e[6], e[7], e[8], e[9], e[10]);
    }
#endif
  if (warp == 2) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(A8_TMEM_COLS));
  }
}


}  // namespace

bool attn_tc_supported(int T, int D, int H) { return H > 0 && D % H == 0 && D / H == 64 && T >= 2 && T - 1 <= A8_MAXK; }
size_t attn_tc_smem() { return A8_META + A8_NQ * sizeof(Meta) + (2 * A8_NQ + 2 * A8_NT + 16) * 8 + 16; }

cudaError_t launch_attention_tc(const CUtensorMap& tmQ, const CUtensorMap& tmKV, const bf16* KV, const int* kvsrc,
                                bf16* out,
                                const int* wdesc, const int* qoff, float* pclsh, int n_w, int T, int D, int H,
                                cudaStream_t s) {
  if (n_w <= 0) return cudaSuccess;
  if (!attn_tc_supported(T, D, H)) return cudaErrorInvalidValue;
  const size_t smem = attn_tc_smem();
  cudaError_t e = ensure_smem<attn_tc_kernel>(smem);
  if (e != cudaSuccess) return e;
  const int sms = dev_sms();
  const long long items = (long long)n_w * H;   // tile-0 items (all live)
  const int grid = items < sms ? (int)items : sms;
  const float scale_log2 = 1.4426950408889634f / 8.0f;   // 1/sqrt(64) * log2(e)
  attn_tc_kernel<<<grid, A8_THREADS, smem, s>>>(tmQ, tmKV, KV, kvsrc, out, reinterpret_cast<const int4*>(wdesc), qoff,
                                                pclsh, n_w, T, D, H, scale_log2);
  return cudaGetLastError();
}

}  // namespace rv
