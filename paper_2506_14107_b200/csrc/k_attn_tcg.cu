// k_attn_tcg.cu — general-shape attention on the 5th-generation tensor cores: the compacted
// queries of each frame against all T keys of the frame (P:313 every recomputed
// query attends to all tokens; P:336 the CLS query's attention row is the feature t), for any
// T <= 1025 with d_h = 64: CLIP L/14@336 (T = 577, BASELINE configs[4]) and the SPEC chain
// variant's dense attention (every token a query, q read from the q|k|v cache through the
// source-row table).
//
// Work: tile = (frame, head, 128 queries).  Tiles are taken two at a time ("pair": the next two
// tiles of the CTA's frame-head stream); when both belong to one frame-head (frames with > 128
// recomputed queries: I frames, the chain variant, low-reuse videos) they share every K / V
// load.  The patch keys are processed in chunks of 96 with an online softmax (running max moved
// lazily: only when a chunk's max exceeds it by 8 in log2 units, so P <= 2^8 and O in TMEM is
// rescaled rarely); the CLS key is done on the CUDA cores.  Each group double-buffers S in TMEM,
// so S of chunk c + 1 is computed while the softmax works on chunk c.
//   warp 3     producer: walks the CTA's frame-heads, forms the pairs, publishes each pair's
//              descriptor and loads its Q tiles (TMA in the compacted-query mode, cp.async rows
//              through the table in the chain mode) and CLS key K / V rows, and writes the row
//              table of every K / V chunk load into a ring of 8 shared-memory tables (`kvsrc`
//              read ahead: the reuse cache is read in place, a7).
//   warps 0-1  loaders (64 lanes): per chunk table, the 96 K rows then the 96 V rows (128 B
//              per row and head) with cp.async into SWIZZLE_128B tiles of 6-slot K and V rings;
//              completion on the slot's mbarrier (cp.async.mbarrier.arrive.noinc).  The gather
//              of scattered 128 B rows runs at <= ~4.9 TB/s on B200 (tools/gather_rate.cu).
//   warp 2     TMEM allocator (all 512 columns) + one MMA-issuing lane: per pair, both tiles in
//              lockstep: S(x, c + 1) = Q K^T (M = 128, N = 96, 4 K-steps) into the free S
//              buffer, then O_x (+)= P(x, c) V (6 MMAs, P read from TMEM) once group x stored P.
//   warps 4-7  softmax group 0 (tile a of each pair), warps 8-11 group 1 (tile b): one query
//              row per thread (32x32b TMEM accesses, warp w -> lanes 32 (w % 4) ..), 96 scores
//              in registers; epilogue O / l (+ the CLS key's p v_cls) -> bf16; the CLS query's
//              normalised probabilities over the patch keys (t) from a shared-memory stash.
#include <cuda.h>
#include <cstdio>
#include <cstring>

#include "rv_internal.h"
#include "tc_ptx.cuh"

namespace rv {
namespace {

// pairs of scores out of every 8 whose 2^x runs on the FMA pipe (ex2_poly2) instead of MUFU
#ifndef AG_POLY
#define AG_POLY 0
#endif
// 16 warps: K loaders 0 and 13, V loaders 1 and 14, issuer of group 0 (2), producer (3),
// softmax groups 4-7 and 8-11, issuer of group 1 (12), 15 idle.  Registers: warpgroups 0 and 3 drop to G_REG_LO, the two
// softmax warpgroups take G_REG_HI (2 x 128 x 80 + 256 x 176 = 65,536).
constexpr int G_THREADS = 16 * 32;
#define G_REG_LO 80
#define G_REG_HI 176
#define G_STR2(x) #x
#define G_STR(x) G_STR2(x)
constexpr int G_ROWS = 128;                             // query rows per tile = MMA M
constexpr int G_KC = 96;                                // keys per chunk = S MMA N
constexpr int G_MAXNC = 11;                             // chunks: T - 1 <= 1056
constexpr int G_NK = 6, G_NV = 6, G_NQ = 2;             // K ring, V ring, pair slots
constexpr int G_NI = 8;                                 // chunk row tables (producer -> loaders)
constexpr int G_ITAB = 4 + G_KC;                        // table: head, rows to load, pad, pad, 96 rows
constexpr uint32_t G_QTILE = G_ROWS * 128;              // Q tile: 128 rows x 128 B
constexpr uint32_t G_KVTILE = G_KC * 128;               // K or V chunk: 96 rows x 128 B
constexpr uint32_t G_PSLOT = 2 * G_QTILE + 1024;        // Q(a), Q(b), CLS K / V rows of a (+0, +128), b (+256, +384)
constexpr uint32_t G_KR = G_NQ * G_PSLOT;               // K ring (1 KB aligned)
constexpr uint32_t G_VR = G_KR + G_NK * G_KVTILE;       // V ring
constexpr uint32_t G_STASH = G_VR + G_NV * G_KVTILE;    // per group: CLS row p [G_MAXNC x G_KC] + chunk max [16]
constexpr uint32_t G_STASH_N = G_MAXNC * G_KC + 16;
constexpr uint32_t G_ITABS = G_STASH + 2 * G_STASH_N * 4;
constexpr uint32_t G_META = G_ITABS + G_NI * G_ITAB * 4;
// TMEM per group g (columns [256 g, 256 g + 256)): S / P double buffer at +0 and +96 (P packed
// bf16 over the first 48 columns of its buffer), O at +192.
constexpr uint32_t G_TO = 192;

struct GMeta {   // one pair, written by producer lane 0, read by the MMA issuer and both groups
  int q0[2], nr[2], slot[2], h[2], tile[2];   // per tile: first query / output row, rows, frame slot, head, tile index
  int seq0, stride, shared, has_b, done;      // ring sequence of chunk 0 of tile a; chunk stride; shared K / V
};
constexpr uint32_t G_BAR = (G_META + G_NQ * sizeof(GMeta) + 7) & ~7u;
constexpr uint32_t G_NBAR = 2 * G_NQ + 2 * G_NK + 2 * G_NV + 2 * G_NI + 10;
constexpr uint32_t G_SMEM = G_BAR + G_NBAR * 8 + 16;
static_assert(G_SMEM + 1024 <= 232448, "attn_tcg_kernel shared memory");

struct GTile {
  int fh, t, q0, nr, slot, h;
};

#ifdef RV_AG_TRACE   // experiment builds: event timeline of CTA 0 (printed at exit)
// each tracing thread appends to its own region (no atomics: the trace must not perturb timing)
constexpr int AG_REG = 2048;
__device__ unsigned long long g_ag_trace[7 * AG_REG][2];
__device__ int g_ag_cnt[7];
RV_DEV void ag_tr(int region, int& n, int code) {
  if (blockIdx.x != 0 || n >= AG_REG) return;
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  g_ag_trace[region * AG_REG + n][0] = (unsigned long long)code;
  g_ag_trace[region * AG_REG + n][1] = t;
  ++n;
  g_ag_cnt[region] = n;
}
// code: role (1 loader, 2 issuer, 3 softmax) << 24 | event << 16 | a << 8 | b
#define AG_TR(role, ev, a, b) ag_tr(ag_region, ag_n, ((role) << 24) | ((ev) << 16) | (((a) & 255) << 8) | ((b) & 255))
#else
#define AG_TR(role, ev, a, b) do { } while (0)
#endif

__global__ void __launch_bounds__(G_THREADS, 1)
    attn_tcg_kernel(const __grid_constant__ CUtensorMap tmQ, const bf16* __restrict__ qbuf, long long q_ld, int q_col,
                    int q_mode, const bf16* __restrict__ KV, long long kv_ld, const int* __restrict__ kvsrc,
                    bf16* __restrict__ out, const int4* __restrict__ wdesc, const int* __restrict__ qoff,
                    float* __restrict__ pclsh, int n_w, int T, int D, int H, float scale_log2) {
  extern __shared__ __align__(1024) uint8_t sm[];
  const uint32_t base = su32(sm);
  GMeta* meta = reinterpret_cast<GMeta*>(sm + G_META);
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + G_BAR);
  uint64_t *q_full = bar, *q_empty = q_full + G_NQ, *kf = q_empty + G_NQ, *ke = kf + G_NK, *vf = ke + G_NK,
           *ve = vf + G_NV, *s_full = ve + G_NV, *p_full = s_full + 2, *pv_full = p_full + 2, *r_free = pv_full + 2,
           *i_full = r_free + 2, *i_empty = i_full + G_NI, *s_taken = i_empty + G_NI;
  int* itab = reinterpret_cast<int*>(sm + G_ITABS);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + G_NBAR);
  const int NP = T - 1;                                 // patch keys
  const int nc = (NP + G_KC - 1) / G_KC;                // key chunks
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid == 0) {
    if (q_mode == 0) asm volatile("prefetch.tensormap [%0];" ::"l"(&tmQ) : "memory");
    for (int i = 0; i < G_NQ; ++i) {
      mbar_init(&q_full[i], 1 + 32);   // producer lane 0's (expect_tx) arrival + every producer lane's cp.async
      mbar_init(&q_empty[i], 8);       // both groups' 4 warps, after their epilogues
    }
    for (int i = 0; i < G_NK; ++i) {
      mbar_init(&kf[i], 64);
      mbar_init(&ke[i], 2);   // two commits per use (one per issuer, or both from the only reader)
    }
    for (int i = 0; i < G_NV; ++i) {
      mbar_init(&vf[i], 64);
      mbar_init(&ve[i], 2);
    }
    for (int i = 0; i < G_NI; ++i) {
      mbar_init(&i_full[i], 1);
      mbar_init(&i_empty[i], 4);   // the four loader warps
    }
    for (int g = 0; g < 2; ++g) {
      mbar_init(&s_full[g], 1);
      mbar_init(&p_full[g], 4);
      mbar_init(&pv_full[g], 1);
      mbar_init(&r_free[g], 4);
      mbar_init(&s_taken[g], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(tslot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tslot;

#ifdef RV_AG_TRACE
  int ag_n = 0;
  const int ag_region = warp < 4 ? (warp == 3 ? 2 : (warp == 2 ? 3 : warp)) : (warp == 12 ? 6 : (warp == 4 ? 4 : 5));
#endif
  if (warp < 2 || warp == 13 || warp == 14) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 " G_STR(G_REG_LO) ";" ::: "memory");
    // ======================================================================== K / V loaders
    // Consume the producer's chunk tables in sequence order.  Warps 0 and 13 load the K rows,
    // warps 1 and 14 the V rows (each warp half of the 96 rows, cp.async, 8 lanes per 128 B
    // row): a K load never queues behind a V slot, which frees only after P V, late in the
    // chunk's chain (ncu: with one loader stream per warp the loaders waited on V slots while
    // the softmax waited on S).
    const bool is_v = warp == 1 || warp == 14;
    const int part = warp < 2 ? 0 : 1;
    const int cc = lane & 7;                            // 16 B chunk of a 128 B row
    const int rsub = part * 4 + (lane >> 3);            // rows rsub + 8 i, i < 12
    const uint32_t nslot = is_v ? G_NV : G_NK;
    uint64_t* full = is_v ? vf : kf;
    uint64_t* empty = is_v ? ve : ke;
    const uint32_t ring = base + (is_v ? G_VR : G_KR);
    for (int seq = 0;; ++seq) {
      const int ti = seq % G_NI;
      mbar_wait(&i_full[ti], (uint32_t)(seq / G_NI) & 1);
      const int* tab = itab + ti * G_ITAB;
      if (lane == 0) AG_TR(1, 2, seq, warp);
      const int h = tab[0], nS = tab[1];
      if (nS == 0) break;                               // end of the stream
      int idx[G_KC / 8];
#pragma unroll
      for (int i = 0; i < G_KC / 8; ++i) idx[i] = tab[4 + rsub + 8 * i];
      __syncwarp();
      if (lane == 0) mbar_arrive(&i_empty[ti]);
      const uint32_t sl = (uint32_t)seq % nslot;
      const bf16* src = KV + h * 128 + (is_v ? 64 : 0) + cc * 8;   // (k_h v_h) per token
      mbar_wait(&empty[sl], ((uint32_t)(seq / nslot) & 1) ^ 1);
      const uint32_t dst = ring + sl * G_KVTILE;
#pragma unroll
      for (int i = 0; i < G_KC / 8; ++i) {
        const int r = rsub + 8 * i;
        if (8 * i < nS) cp_async16(dst + (uint32_t)r * 128 + ((cc ^ (r & 7)) << 4), src + (long long)idx[i] * kv_ld);
      }
      cp_async_arrive(&full[sl]);
      if (lane == 0) AG_TR(1, 3, seq, warp);
    }
  } else if (warp == 3) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 " G_STR(G_REG_LO) ";" ::: "memory");
    // ======================================================================== producer
    // Walks the CTA's frame-head stream (fh = blockIdx.x + k gridDim.x, head fastest), forms
    // pairs of tiles, publishes each pair's descriptor and Q / CLS loads, and writes the row
    // table of every K / V chunk load (kvsrc gathered ahead, so the loaders never wait on it).
    const long long n_fh = (long long)n_w * H;
    const int cc = lane & 7;
    long long f_fh = -1, nx_fh = blockIdx.x;
    int f_t = 0, f_nt = 0, f_q0 = 0, f_nq = 0, f_slot = 0, f_h = 0;
    auto next_tile = [&](GTile& x) -> bool {
      while (f_t >= f_nt) {
        if (nx_fh >= n_fh) return false;
        f_fh = nx_fh;
        const int w = (int)(f_fh / H);
        f_q0 = __ldg(qoff + w);
        f_nq = __ldg(qoff + w + 1) - f_q0;
        f_slot = __ldg(&wdesc[w].x);
        f_h = (int)(f_fh - (long long)w * H);
        f_t = 0;
        f_nt = (f_nq + G_ROWS - 1) / G_ROWS;
        nx_fh += gridDim.x;
      }
      x.fh = (int)f_fh;
      x.t = f_t;
      x.q0 = f_q0 + f_t * G_ROWS;
      x.nr = min(G_ROWS, f_nq - f_t * G_ROWS);
      x.slot = f_slot;
      x.h = f_h;
      ++f_t;
      return true;
    };
    int seq = 0, p = 0;
    auto put_table = [&](const GTile* x, int c) {   // row table of chunk c of tile x (null: end marker)
      const int ti = seq % G_NI;
      mbar_wait(&i_empty[ti], ((uint32_t)(seq / G_NI) & 1) ^ 1);
      int* tab = itab + ti * G_ITAB;
      if (x) {
        const long long fb = (long long)x->slot * T;
#pragma unroll
        for (int j = 0; j < G_KC / 32; ++j) {
          const int tok = 1 + min(c * G_KC + lane + 32 * j, NP - 1);   // padding keys: the last patch key's row
          tab[4 + lane + 32 * j] = kvsrc ? __ldg(kvsrc + fb + tok) : (int)(fb + tok);
        }
      }
      if (lane == 0) {
        tab[0] = x ? x->h : 0;
        tab[1] = x ? ((min(G_KC, NP - c * G_KC) + 15) & ~15) : 0;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&i_full[ti]);
      ++seq;
    };
    GTile A, B;
    while (next_tile(A)) {
      const bool has_b = next_tile(B);
      const bool shared = has_b && B.fh == A.fh, sep = has_b && !shared;
      const int ps = p % G_NQ;
      const uint32_t pslot = base + (uint32_t)ps * G_PSLOT;
      // the pair's K / V chunk tables first: the loaders start on them while this pair's Q slot
      // is still held by the pair before last (its epilogue), instead of after the Q loads
      const int seq_p = seq;
      for (int c = 0; c < nc; ++c) {   // chunk loads: chunk-major, tile a then (unless shared) tile b
        put_table(&A, c);
        if (sep) put_table(&B, c);
      }
      if (lane == 0) AG_TR(1, 0, p, 0);
      mbar_wait(&q_empty[ps], ((uint32_t)(p / G_NQ) & 1) ^ 1);
      if (lane == 0) AG_TR(1, 1, p, has_b * 2 + shared);
      if (lane == 0) {
        GMeta& m = meta[ps];
        const GTile* xs[2] = {&A, &B};
        for (int e = 0; e < 2; ++e) {
          m.q0[e] = xs[e]->q0; m.nr[e] = xs[e]->nr; m.slot[e] = xs[e]->slot; m.h[e] = xs[e]->h; m.tile[e] = xs[e]->t;
        }
        m.seq0 = seq_p; m.stride = sep ? 2 : 1; m.shared = shared; m.has_b = has_b; m.done = 0;
        if (q_mode == 0) {
          mbar_expect_tx(&q_full[ps], G_QTILE * (has_b ? 2 : 1));
          for (int e = 0; e < (has_b ? 2 : 1); ++e)
            for (int hh = 0; hh < 2; ++hh)
              tma_2d(pslot + e * G_QTILE + hh * 8192, &tmQ, xs[e]->h * 64, xs[e]->q0 + 64 * hh, &q_full[ps]);
        } else {
          mbar_arrive(&q_full[ps]);
        }
      }
      if (q_mode == 1) {   // chain: query rows = the frame's tokens, q through the source-row table
        for (int e = 0; e < (has_b ? 2 : 1); ++e) {
          const GTile& x = e ? B : A;
          const long long fb = (long long)x.slot * T + (long long)x.t * G_ROWS;
          const bf16* src = qbuf + q_col + x.h * 64 + cc * 8;
#pragma unroll 1
          for (int i0 = 0; i0 < 32; i0 += 16) {
            int qrow[16];   // 16 table reads in flight before the copies (two latencies per tile, not 8)
#pragma unroll
            for (int i = 0; i < 16; ++i) qrow[i] = __ldg(kvsrc + fb + min((lane >> 3) + 4 * (i0 + i), x.nr - 1));
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              const int r = (lane >> 3) + 4 * (i0 + i);
              cp_async16(pslot + e * G_QTILE + (uint32_t)r * 128 + ((cc ^ (r & 7)) << 4), src + (long long)qrow[i] * q_ld);
            }
          }
        }
      }
      {   // CLS key's K and V rows of tile a (lanes 0-15) and b (16-31)
        const int e = lane >> 4, kv = (lane >> 3) & 1;
        if (e == 0 || has_b) {
          const GTile& x = e ? B : A;
          const long long fb = (long long)x.slot * T;
          const long long row = kvsrc ? __ldg(kvsrc + fb) : fb;
          cp_async16(pslot + 2 * G_QTILE + e * 256 + kv * 128 + cc * 16, KV + row * kv_ld + x.h * 128 + kv * 64 + cc * 8);
        }
      }
      cp_async_arrive(&q_full[ps]);
      ++p;
    }
    // end markers: the loaders' table stream and the next pair slot
    put_table(nullptr, 0);
    {
      const int ps = p % G_NQ;
      mbar_wait(&q_empty[ps], ((uint32_t)(p / G_NQ) & 1) ^ 1);
      if (lane == 0) {
        meta[ps].done = 1;
        mbar_arrive(&q_full[ps]);
      }
      cp_async_arrive(&q_full[ps]);
    }
  } else if (warp == 2 || warp == 12 || warp == 15) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 " G_STR(G_REG_LO) ";" ::: "memory");
    // ======================================================================== MMA issuers
    // One issuing thread per softmax group (warp 2: group 0, warp 12: group 1): a thread issues
    // at most one tcgen05.mma every ~120 cycles whatever its size, and the attention's MMAs are
    // small (N = 96 / 64), so two issuers double the MMA rate (tools/umma_issuers.cu: 120 -> 60
    // cycles per M = 128, N = 64 MMA).  Per pair, group g: S(g, 0); per chunk c: S(g, c + 1) into
    // the other S buffer (its softmax starts chunk c + 1 as soon as chunk c is done), then
    // O_g (+)= P(g, c) V(c) once the group stored P.  MMAs of one thread execute in issue order,
    // so S(c + 2) overwrites P(c) only after P V(c) has read it.  K / V ring slots: their empty
    // barriers count 2 arrivals; each issuer commits once per slot it read, a slot read by one
    // group only (separate tiles, or a pair without a second tile) gets both commits from it.
    const int g = warp == 2 ? 0 : 1;
    if (lane == 0 && warp != 15) {
      const uint32_t id_o = idesc_f16(G_ROWS, 64, 1);
      int nch = 0, ntl = 0, ns = 0;
      for (int p = 0;; ++p) {
        const int ps = p % G_NQ;
        mbar_wait(&q_full[ps], (uint32_t)(p / G_NQ) & 1);
        const volatile GMeta& m = meta[ps];
        if (m.done) break;
        if (g == 1 && !m.has_b) continue;
        const int seq0 = m.seq0, stride = m.stride;
        const bool shared = m.shared;
        const int nrel = (shared && m.has_b) ? 1 : 2;   // commits this group owes each slot it reads
        const int seq_g = seq0 + ((g == 1 && !shared) ? 1 : 0);
        auto issue_s = [&](int c) {
          const int seq = seq_g + c * stride;
          const uint32_t ks = (uint32_t)seq % G_NK;
          mbar_wait(&kf[ks], (uint32_t)(seq / G_NK) & 1);
          // every mbarrier here may run at most one phase ahead of its waiter: S number k of the
          // group is issued only once its softmax has taken S number k - 1
          if (ns > 0) mbar_wait(&s_taken[g], (uint32_t)(ns - 1) & 1);
          ++ns;
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // cp.async data -> tensor core
          tc_after();
          const int nS = (min(G_KC, NP - c * G_KC) + 15) & ~15;
          const uint32_t tS = tmem + (uint32_t)g * 256 + (uint32_t)(c & 1) * G_KC;
          const uint32_t qa = base + (uint32_t)ps * G_PSLOT + (uint32_t)g * G_QTILE, ka = base + G_KR + ks * G_KVTILE;
          const uint32_t id_s = idesc_f16(G_ROWS, nS, 0);
#pragma unroll
          for (int k = 0; k < 4; ++k) mma_ss(tS, sdesc(qa + k * 32), sdesc(ka + k * 32), id_s, k != 0);
          mma_commit(&s_full[g]);
          for (int r = 0; r < nrel; ++r) mma_commit(&ke[ks]);
          AG_TR(2, 0, seq, g);
        };
        auto issue_pv = [&](int c) {
          const int seq = seq_g + c * stride;
          const uint32_t vs = (uint32_t)seq % G_NV;
          mbar_wait(&p_full[g], (uint32_t)nch & 1);
          mbar_wait(&vf[vs], (uint32_t)(seq / G_NV) & 1);
          if (c == 0) mbar_wait(&r_free[g], ((uint32_t)ntl & 1) ^ 1);   // previous tile's O read
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          tc_after();
          const int nS = (min(G_KC, NP - c * G_KC) + 15) & ~15;
          const uint32_t tS = tmem + (uint32_t)g * 256 + (uint32_t)(c & 1) * G_KC, tO = tmem + (uint32_t)g * 256 + G_TO;
          const uint32_t va = base + G_VR + vs * G_KVTILE;
          for (int k = 0; k < nS / 16; ++k)   // O (+)= P V: 16 keys per MMA, P packed at column 8 k
            mma_ts(tO, tS + (uint32_t)(k * 8), sdesc(va + (uint32_t)k * 2048), id_o, (c | k) != 0);
          mma_commit(&pv_full[g]);
          for (int r = 0; r < nrel; ++r) mma_commit(&ve[vs]);
          ++nch;
          AG_TR(2, 1, seq, g);
        };
        issue_s(0);
        for (int c = 0; c < nc; ++c) {
          if (c + 1 < nc) issue_s(c + 1);
          issue_pv(c);
        }
        ++ntl;
      }
    }
  } else {
    asm volatile("setmaxnreg.inc.sync.aligned.u32 " G_STR(G_REG_HI) ";" ::: "memory");
    // ======================================================================== softmax groups
    const int g = (warp - 4) >> 2;
    const int q = warp & 3;                            // TMEM lane quarter
    const int row = q * 32 + lane;                     // query row of the tile
    const uint32_t lrow = (uint32_t)(q * 32) << 16;
    const uint32_t tG = tmem + (uint32_t)g * 256 + lrow, tO = tG + G_TO;
    float* stash = reinterpret_cast<float*>(sm + G_STASH) + g * G_STASH_N;
    float* stash_m = stash + G_MAXNC * G_KC;
    const unsigned long long sc2 = f2pack(scale_log2, scale_log2);
    int nch = 0;          // S chunks consumed (s_full phases)
    int pv_seen = 0;      // P V completions consumed (pv_full phases)
    int pv_base = 0;      // P V index of the current tile's chunk 0
    auto wait_pv = [&](int target) {   // until P V number `target` (global count) has completed
      while (pv_seen <= target) {
        mbar_wait(&pv_full[g], (uint32_t)pv_seen & 1);
        ++pv_seen;
      }
    };
    for (int p = 0;; ++p) {
      const int ps = p % G_NQ;
      mbar_wait(&q_full[ps], (uint32_t)(p / G_NQ) & 1);
      const volatile GMeta& vm = meta[ps];
      if (vm.done) break;
      if (g == 1 && !vm.has_b) {
        __syncwarp();
        if (lane == 0) mbar_arrive(&q_empty[ps]);
        continue;
      }
      const int nr = vm.nr[g], q0 = vm.q0[g], slot = vm.slot[g], h = vm.h[g], tile = vm.tile[g];
      const bool act = q * 32 < nr;                    // warp-uniform: this quarter has live rows
      const bool cls = pclsh != nullptr && tile == 0 && q == 0;   // lane 0 holds the CLS query row
      const uint8_t* qrow = sm + (size_t)ps * G_PSLOT + (size_t)g * G_QTILE + (size_t)row * 128;
      const uint8_t* kcls = sm + (size_t)ps * G_PSLOT + 2 * G_QTILE + (size_t)g * 256;
      float mrun = -INFINITY, l = 0.f, pc = 0.f;
      for (int c = 0; c < nc; ++c) {
        mbar_wait(&s_full[g], (uint32_t)nch & 1);
        ++nch;
        __syncwarp();
        if (lane == 0) mbar_arrive(&s_taken[g]);
        if (q == 0 && lane == 0) AG_TR(3, 0, p, g * 16 + c);
        tc_after();
        const uint32_t tS = tG + (uint32_t)(c & 1) * G_KC;
        if (act) {
          float v[G_KC];
#pragma unroll
          for (int i = 0; i < G_KC / 32; ++i) tld32x32(tS + 32 * i, v + 32 * i);
          float sc = 0.f;
          if (c == 0) {   // CLS key on the CUDA cores while the TMEM loads are in flight
#pragma unroll
            for (int ch = 0; ch < 8; ++ch) {
              const uint4 qa = *reinterpret_cast<const uint4*>(qrow + ((ch ^ (row & 7)) << 4));
              const uint4 ka = *reinterpret_cast<const uint4*>(kcls + ch * 16);
              const uint32_t qw[4] = {qa.x, qa.y, qa.z, qa.w}, kw[4] = {ka.x, ka.y, ka.z, ka.w};
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 qf = unpack_bf16x2(qw[e]), kf2 = unpack_bf16x2(kw[e]);
                sc = fmaf(qf.x, kf2.x, sc);
                sc = fmaf(qf.y, kf2.y, sc);
              }
            }
          }
          tld_wait();
          const int kc = min(G_KC, NP - c * G_KC);
          if (kc < G_KC) {
#pragma unroll
            for (int i = 0; i < G_KC; ++i)
              if (i >= kc) v[i] = -INFINITY;
          }
          float mx4[4] = {v[0], v[1], v[2], v[3]};
#pragma unroll
          for (int i = 4; i < G_KC - 4; i += 8) {
            mx4[0] = fmax3(mx4[0], v[i], v[i + 1]);
            mx4[1] = fmax3(mx4[1], v[i + 2], v[i + 3]);
            mx4[2] = fmax3(mx4[2], v[i + 4], v[i + 5]);
            mx4[3] = fmax3(mx4[3], v[i + 6], v[i + 7]);
          }
          mx4[0] = fmax3(mx4[0], v[G_KC - 4], v[G_KC - 3]);
          mx4[1] = fmax3(mx4[1], v[G_KC - 2], v[G_KC - 1]);
          const float cm = fmax3(mx4[0], mx4[1], fmaxf(mx4[2], mx4[3])) * scale_log2;
          if (c == 0) {
            mrun = fmaxf(cm, sc * scale_log2);
            pc = ex2f_fast(fmaf(sc, scale_log2, -mrun));
            l = pc;
          } else {
            // lazy rescale: move the running max only when this chunk would push P above 2^8;
            // O must then hold chunks < c complete: wait for P V(c - 1) (rare)
            const bool need = cm > mrun + 8.f;
            if (__any_sync(0xffffffffu, need)) {
              wait_pv(pv_base + c - 1);
              tc_after();
              const float mnew = need ? cm : mrun;
              const float f = ex2f_fast(mrun - mnew);
#pragma unroll 1
              for (int hc = 0; hc < 2; ++hc) {
                float o[32];
                tld32x32(tO + 32 * hc, o);
                tld_wait();
                uint32_t u[32];
#pragma unroll
                for (int i = 0; i < 32; ++i) u[i] = __float_as_uint(o[i] * f);
                tst32x32(tO + 32 * hc, u);
              }
              l *= f;
              pc *= f;
              mrun = mnew;
            }
          }
          const unsigned long long nm2 = f2pack(-mrun, -mrun);
          unsigned long long acc[4] = {0ull, 0ull, 0ull, 0ull};
#pragma unroll
          for (int i = 0; i < G_KC; i += 2) {
            const unsigned long long x2 = ffma2(f2pack(v[i], v[i + 1]), sc2, nm2);
            if (((i >> 1) & 7) < AG_POLY) {   // this pair on the FMA pipe (MUFU relief)
              const float2 e = f2unpack(ex2_poly2(x2));
              v[i] = e.x;
              v[i + 1] = e.y;
            } else {
              const float2 x = f2unpack(x2);
              v[i] = ex2f_fast(x.x);
              v[i + 1] = ex2f_fast(x.y);
            }
            acc[(i >> 1) & 3] = fadd2(acc[(i >> 1) & 3], f2pack(v[i], v[i + 1]));
          }
          const float2 s01 = f2unpack(fadd2(fadd2(acc[0], acc[1]), fadd2(acc[2], acc[3])));
          l += s01.x + s01.y;
          if (cls && lane == 0) {   // the CLS query's p over this chunk's keys, relative to mrun
#pragma unroll
            for (int i = 0; i < G_KC; i += 4)
              *reinterpret_cast<float4*>(stash + c * G_KC + i) = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
            stash_m[c] = mrun;
          }
          uint32_t pk[G_KC / 2];
#pragma unroll
          for (int i = 0; i < G_KC / 2; ++i) pk[i] = pack_bf16x2(v[2 * i], v[2 * i + 1]);
          tst32x32(tS, pk);
          tst32x16(tS + 32, pk + 32);
          tst_wait();
        }
        // P(c) is announced only after P V(c - 1) completed, i.e. after the issuer took P(c - 1):
        // p_full and pv_full never run two phases ahead of their waiters
        if (c >= 1) wait_pv(pv_base + c - 1);
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[g]);
        if (q == 0 && lane == 0) AG_TR(3, 1, p, g * 16 + c);
      }
      // ---------------------------------------------------------------- epilogue
      wait_pv(pv_base + nc - 1);
      pv_base += nc;
      if (q == 0 && lane == 0) AG_TR(3, 2, p, g * 16);
      tc_after();
      if (act) {
        float o[64];
        tld32x32(tO, o);
        tld32x32(tO + 32, o + 32);
        tld_wait();
        if (row < nr) {
          const float il = 1.f / l;
          const uint8_t* vc = kcls + 128;
          bf16* dst = out + (long long)(q0 + row) * D + h * 64;
#pragma unroll
          for (int ch = 0; ch < 8; ++ch) {
            const uint4 va = *reinterpret_cast<const uint4*>(vc + ch * 16);
            const uint32_t vw[4] = {va.x, va.y, va.z, va.w};
            uint32_t u[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
              const float2 vf2 = unpack_bf16x2(vw[e]);
              u[e] = pack_bf16x2(fmaf(pc, vf2.x, o[8 * ch + 2 * e]) * il, fmaf(pc, vf2.y, o[8 * ch + 2 * e + 1]) * il);
            }
            *reinterpret_cast<uint4*>(dst + 8 * ch) = make_uint4(u[0], u[1], u[2], u[3]);
          }
        }
      }
      if (cls) {   // normalise the stashed CLS row: p_k 2^(m_chunk - m) / l
        const float mf = __shfl_sync(0xffffffffu, mrun, 0), il = 1.f / __shfl_sync(0xffffffffu, l, 0);
        __syncwarp();
        float* dst = pclsh + ((long long)slot * H + h) * NP;
        for (int k = lane; k < NP; k += 32) dst[k] = stash[k] * ex2f_fast(stash_m[k / G_KC] - mf) * il;
        __syncwarp();
      }
      tc_before();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&r_free[g]);
        mbar_arrive(&q_empty[ps]);
      }
      if (q == 0 && lane == 0) AG_TR(3, 3, p, g * 16);
    }
  }
  tc_before();
  __syncthreads();
#ifdef RV_AG_TRACE
  if (blockIdx.x == 0 && tid == 0) {
    for (int r = 0; r < 7; ++r) {
      for (int i = 0; i < g_ag_cnt[r]; ++i)
        printf("AG %llx %llu\n", g_ag_trace[r * AG_REG + i][0], g_ag_trace[r * AG_REG + i][1]);
      g_ag_cnt[r] = 0;
    }
  }
#endif
  if (warp == 2) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}

}  // namespace

bool attn_tcg_supported(int T, int D, int H) {
  return H > 0 && D % H == 0 && D / H == 64 && T >= 2 && T - 1 <= 1024;
}

cudaError_t launch_attention_tcg(const CUtensorMap* tmQ, const bf16* q, long long q_ld, int q_col, int q_mode,
                                 const bf16* KV, long long kv_ld, const int* kvsrc, bf16* out, const int* wdesc,
                                 const int* qoff, float* pclsh, int n_w, int T, int D, int H, cudaStream_t s) {
  if (n_w <= 0) return cudaSuccess;
  if (!attn_tcg_supported(T, D, H) || (q_mode == 0 && !tmQ) || (q_mode == 1 && !kvsrc)) return cudaErrorInvalidValue;
  cudaError_t e = ensure_smem<attn_tcg_kernel>(G_SMEM);
  if (e != cudaSuccess) return e;
  CUtensorMap none;
  memset(&none, 0, sizeof none);
  const long long fh = (long long)n_w * H;
  const int sms = dev_sms();
  const int grid = fh < sms ? (int)fh : sms;
  const float scale_log2 = 1.4426950408889634f / 8.0f;   // 1/sqrt(64) * log2(e)
  attn_tcg_kernel<<<grid, G_THREADS, G_SMEM, s>>>(q_mode == 0 ? *tmQ : none, q, q_ld, q_col, q_mode, KV, kv_ld, kvsrc,
                                                  out, reinterpret_cast<const int4*>(wdesc), qoff, pclsh, n_w, T, D, H,
                                                  scale_log2);
  return cudaGetLastError();
}

}  // namespace rv
