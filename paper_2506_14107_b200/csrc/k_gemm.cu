// k_gemm.cu — persistent, warp-specialised tcgen05/TMEM/TMA GEMM for sm_100a.
//
// Used for every dense contraction of the compacted batch:
// patch embed, QKV (Eq. 7 QKV part), W_o, FC1/FC2 (Eq. 7 FFN part) and the two
// restoration layers (Eq. 9).  out = epilogue(A[M,K] * B[N,K]^T), bf16 operands, fp32
// accumulation in TMEM.  M is read from device memory (the compaction kernel's count), so
// no host synchronisation is needed between compaction and the contractions
// and the whole layer loop is CUDA-graph capturable.
//
// CTA = 320 threads, one CTA per SM (persistent over 128 x BN output tiles; BN = 256 GEMMs run
// as CTA pairs over 256 x 256 tiles with tcgen05.mma.cta_group::2, see Cfg::PAIR):
//   warp 0 : TMA producer (one elected lane), STAGES-deep smem ring, SWIZZLE_128B tiles
//   warp 1 : MMA issuer (one lane): tcgen05.mma.cta_group::1.kind::f16, M=128, N=BN, K=16
//   warp 1 also allocates TMEM (2*BN fp32 columns: double-buffered accumulator)
//   warps 2.. : epilogue, 8 (16 in the SR variant) (warp%4 = TMEM lane quarter, (warp-2)/4 = column slice):
//               tcgen05.ld 32x32b.x32 -> smem transpose -> coalesced bias / QuickGELU /
//               residual / row-mapped (scatter) stores in fp32 or bf16
// Fixed tiles and no split-K: every output element is accumulated in the same K order
// regardless of M or of its row position, so results are batch-invariant.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <stdio.h>

#include "common.cuh"
#include "rv_internal.h"

namespace rv {

namespace {

constexpr int BM = 128;
constexpr int BK = 64;            // 64 bf16 = 128 B = one SWIZZLE_128B atom row
// TMA warp + MMA/TMEM warp + epilogue warps: 8, or 16 for the short-K residual-streaming (SR)
// variant, whose epilogue is a chain of dependent latencies per chunk and needs more warps
// (at least one 32-column chunk per warp: 16 warps need BN >= 128)
// MODE 0: plain; 1 (SR): short K with a streamed residual (restoration R2); 2 (RE): K <= 1024
// epilogue-heavy GEMMs (W_o, QKV, FC1): 16 epilogue warps and 3 mainloop stages
template <int BN, int MODE> constexpr int epi_warps() { return MODE != 0 && BN >= 128 ? 16 : 8; }
template <int BN, int MODE> constexpr int gemm_threads() { return (2 + epi_warps<BN, MODE>()) * 32; }

constexpr int RDEPTH = 2;         // residual chunks in flight per epilogue warp (SR variant)

// SR ("short K, streaming residual"): for K <= 256 the mainloop needs only 2 stages, and the
// freed shared memory holds a cp.async ring of residual rows RDEPTH chunks deep; the chunk's
// ring slot doubles as its transpose tile once the residual is in registers, so the HBM-bound
// epilogue keeps 128 KB of residual loads in flight per SM.
// PAIR: a CTA pair on one TPC (cluster of 2) computes a 256 x BN tile with
// tcgen05.mma.cta_group::2 (M = 256): each CTA stages its own 128 rows of A and half of the BN
// rows of B, the leader CTA issues the MMAs, each CTA's TMEM holds its 128 accumulator rows.
// Half the B bytes per CTA -> more mainloop stages in the same shared memory.
template <int BN, int MODE, bool PAIR = false>
struct Cfg {
  static constexpr bool SR = MODE == 1;
  static constexpr int A_BYTES = BM * BK * 2;
  static constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = PAIR ? (MODE == 2 ? 4 : (BN == 256 ? 6 : 8))
                                     : SR ? 2 : MODE == 2 ? 3 : (BN == 256 ? 4 : (BN == 128 ? 6 : 8));
  static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
  static constexpr int EPI = epi_warps<BN, MODE>();
  static constexpr int TILE_M = PAIR ? 2 * BM : BM;
  // per-warp 32x32 fp32 transpose tile + row maps (SR: output rows only; the ring slot is the
  // tile and the residual rows travel by shuffle)
  static constexpr int STAGE_OUT = SR ? EPI * 32 * 4 : EPI * (32 * 32 + 64) * 4;
  static constexpr int RESID = SR ? EPI * RDEPTH * 32 * 32 * 4 : 0;
  static constexpr int SMEM = STAGES * STAGE_BYTES + STAGE_OUT + RESID + 256 /*barriers*/;
  static_assert(SMEM <= 232448, "exceeds 227 KB of shared memory per CTA");
};

RV_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

RV_DEV void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
RV_DEV void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes)
               : "memory");
}
RV_DEV void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
RV_DEV uint32_t mbar_try_wait(uint32_t addr, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(ok)
      : "r"(addr), "r"(parity)
      : "memory");
  return ok;
}
RV_DEV void mbar_wait(uint64_t* b, uint32_t parity) {
  const uint32_t a = smem_u32(b);
  while (!mbar_try_wait(a, parity)) {
  }
}
RV_DEV void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}
RV_DEV void prefetch_tmap(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}
RV_DEV void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
RV_DEV float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}
// ---- CTA-pair (cluster of 2) helpers
RV_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
RV_DEV void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// shared::cluster address of the same shared variable in CTA `rank` of the cluster
RV_DEV uint32_t mapa_rank(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(smem_u32(p)), "r"(rank));
  return r;
}
// remote arrive with the default (.release.cta) semantics, as CUTLASS's ClusterBarrier::arrive:
// .release.cluster would add a MEMBAR + ERRBAR that waits for the warp's epilogue stores
RV_DEV void mbar_arrive_cl(uint32_t bar_cl) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(bar_cl) : "memory");
}
// TMA load into this CTA's shared memory, completion counted on the leader CTA's barrier
RV_DEV void tma_load_2d_pair(void* dst, const CUtensorMap* map, uint32_t bar_cl, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(x), "r"(y), "r"(bar_cl)
      : "memory");
}
RV_DEV void mma_bf16_pair(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
// arrive on the barrier at this offset in both CTAs of the pair once the MMAs retire
RV_DEV void mma_commit_pair(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                   smem_u32(bar)), "h"((uint16_t)3)
               : "memory");
}
RV_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
RV_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// SM100 shared-memory matrix descriptor, K-major, SWIZZLE_128B: start address >> 4 in
// [0,14), LBO unused for swizzled K-major, SBO = 1024 B (8 rows x 128 B) >> 4 in [32,46),
// version 1 in [46,48), layout type 2 (SWIZZLE_128B) in [61,64).
RV_DEV uint64_t smem_desc_sw128(const void* p) {
  const uint64_t addr = smem_u32(p);
  return ((addr >> 4) & 0x3FFFull) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// Instruction descriptor for kind::f16: D fp32 (bits 4-5 = 1), A bf16 (7-9 = 1), B bf16
// (10-12 = 1), both K-major, N >> 3 at bit 17, M >> 4 at bit 24.
template <int BN, int MM = BM>
__host__ __device__ constexpr uint32_t idesc_bf16() {
  return (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(BN >> 3) << 17) | (uint32_t(MM >> 4) << 24);
}
RV_DEV void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
RV_DEV void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}
RV_DEV void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// QuickGELU for the GEMM epilogue: x * sigmoid(1.702 x) = x * (0.5 + 0.5 tanh(0.851 x)), one
// MUFU.TANH per element (tanh.approx, rel. err ~2^-11; the result is rounded to bf16).
RV_DEV float quick_gelu_fast(float x) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.851f * x));
  return x * fmaf(0.5f, t, 0.5f);
}

// RB16: the residual rows are bf16 (RV_X_BF16), a separate instantiation so that the fp32
// residual path's register allocation is untouched
template <int BN, int MODE, bool PAIR, bool RB16 = false>
__global__ void __launch_bounds__(gemm_threads<BN, MODE>(), 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const int* __restrict__ M_dev, int M_host, int N, int K, const Epi e) {
  using C = Cfg<BN, MODE, PAIR>;
  constexpr bool SR = C::SR;
  extern __shared__ __align__(1024) uint8_t smem_raw[];   // SWIZZLE_128B needs 1024-B aligned stages
  uint8_t* smem = smem_raw;
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::STAGES * C::A_BYTES;
  float* sOut = reinterpret_cast<float*>(sB + C::STAGES * C::B_BYTES);
  float* sRes = reinterpret_cast<float*>(reinterpret_cast<uint8_t*>(sOut) + C::STAGE_OUT);   // SR ring
  uint64_t* full = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(sOut) + C::STAGE_OUT + C::RESID);
  uint64_t* empty = full + C::STAGES;
  uint64_t* tfull = empty + C::STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int M = M_dev ? *M_dev : M_host;
  const int tiles_n = N / BN;
  const int ntiles = ((M + C::TILE_M - 1) / C::TILE_M) * tiles_n;
  const int nk = K / BK;
  // PAIR: the pair (cluster) index walks the tiles; rank 1 holds rows 128..255 of each tile
  const uint32_t rank = PAIR ? cluster_rank() : 0u;
  const int tile0 = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int tstep = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;

  if (warp == 0 && lane == 0) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], PAIR ? 2 * C::EPI : C::EPI * 32);   // PAIR: one arrive per warp of both CTAs
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                   "r"(C::TMEM_COLS));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
  }
  tc_fence_before();
  __syncwarp();
  if constexpr (PAIR) cluster_sync_all(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = tile0; tile < ntiles; tile += tstep) {
        const int mb = tile / tiles_n, nb = tile % tiles_n;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if constexpr (PAIR) {
            const uint32_t fb = mapa_rank(&full[stage], 0);   // the leader's barrier counts both CTAs
            // leader: its own barrier, CTA-scope arrive (a .release.cluster arrive costs a
            // MEMBAR + ERRBAR per k-step and serialises the TMA ring: measured 2x slower)
            if (rank == 0) mbar_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
            tma_load_2d_pair(sA + stage * C::A_BYTES, &tmA, fb, kb * BK, mb * C::TILE_M + (int)rank * BM);
            tma_load_2d_pair(sB + stage * C::B_BYTES, &tmB, fb, kb * BK, nb * BN + (int)rank * (BN / 2));
          } else {
            mbar_expect_tx(&full[stage], C::STAGE_BYTES);
            tma_load_2d(sA + stage * C::A_BYTES, &tmA, &full[stage], kb * BK, mb * BM);
            tma_load_2d(sB + stage * C::B_BYTES, &tmB, &full[stage], kb * BK, nb * BN);
          }
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {
      constexpr uint32_t idesc = idesc_bf16<BN, C::TILE_M>();
      int stage = 0;
      uint32_t phase = 0;
      int it = 0;
      for (int tile = tile0; tile < ntiles; tile += tstep, ++it) {
        const int acc = it & 1;
        const uint32_t acc_phase = (it >> 1) & 1;
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = smem_desc_sw128(sA + stage * C::A_BYTES);
          const uint64_t bd = smem_desc_sw128(sB + stage * C::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {   // +32 B along K inside the 128 B swizzle atom
            if constexpr (PAIR) mma_bf16_pair(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
            else mma_bf16(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          }
          if constexpr (PAIR) mma_commit_pair(&empty[stage]);   // frees the slot in both CTAs
          else mma_commit(&empty[stage]);     // frees the smem slot once these MMAs retire
          if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
        }
        if constexpr (PAIR) mma_commit_pair(&tfull[acc]);
        else mma_commit(&tfull[acc]);         // accumulator ready for the epilogue
      }
    }
  } else if (warp >= 2) {
    // 8 epilogue warps: warp%4 selects the TMEM lane quarter (rows 32q..32q+31), (warp-4)/4
    // selects the column half.  Per 32-column chunk: tcgen05.ld (thread = row) -> rotated
    // st.shared (conflict-free) -> row-wise ld.shared (8 lanes per row, 4 rows per warp
    // access) -> bias / QuickGELU / residual / row-mapped store, all coalesced.  Row maps are
    // loaded once per tile and the 8 residual loads of a chunk are issued together (MLP).
    const int q = warp & 3;
    const int half = (warp - 2) >> 2;    // column slice of this warp (of C::EPI / 4)
    float* tile_s = SR ? nullptr : sOut + (warp - 2) * (32 * 32 + 64);
    int* orow_s = SR ? reinterpret_cast<int*>(sOut) + (warp - 2) * 32
                     : reinterpret_cast<int*>(tile_s + 32 * 32);   // [32] output row of each tile row
    int* rrow_s = orow_s + 32;                                       // [32] residual row (not SR)
    int rrow_reg = 0;                                                // SR: residual row of row `lane`
    uint32_t tile_u = SR ? 0u : smem_u32(tile_s);
    const int rsub = lane >> 3;          // row within a group of 4
    const int c4 = (lane & 7) * 4;       // first of this lane's 4 columns
    int it = 0;
    for (int tile = tile0; tile < ntiles; tile += tstep, ++it) {
      const int acc = it & 1;
      const uint32_t acc_phase = (it >> 1) & 1;
      const int mb = tile / tiles_n, nb = tile % tiles_n;
      const int row0 = mb * C::TILE_M + (int)rank * BM + q * 32;
      // per-tile row maps (lane = row within this warp's 32 rows), kept in shared memory
      {
        const int m = row0 + lane;
        const int mm = m < M ? m : 0;
        orow_s[lane] = e.out_rows ? __ldg(e.out_rows + mm) : mm + (e.row_div ? mm / e.row_div : 0) + e.row_add;
        const int rv = e.resid ? (e.resid_rows ? __ldg(e.resid_rows + mm) : mm) : 0;
        if constexpr (SR) rrow_reg = rv; else rrow_s[lane] = rv;
      }
      const int nvalid = min(32, M - row0);     // rows of this warp that exist (may be <= 0)
      __syncwarp();
      constexpr int CPW = (BN / 32) / (C::EPI / 4);   // 32-column chunks per warp and tile
      static_assert(CPW >= 1, "every epilogue warp needs a column chunk");
      const int c_beg = half * CPW, c_end = (half + 1) * CPW;
      // Residual rows are known before the accumulator is: load chunk c+1's residual while
      // chunk c is processed (8 x 16 B in flight per lane; the first batch overlaps the MMA).
      float4 xn[8];
      uint2 rn16[RB16 ? 8 : 1];   // RE + bf16 residual: the next chunk's rows, loaded with this chunk's
      auto load_resid16 = [&](int c, uint2* x) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = i * 4 + rsub;
          const long long off = (long long)rrow_s[rr] * e.resid_ld + nb * BN + c * 32 + c4;
          x[i] = (rr < nvalid && orow_s[rr] >= 0) ? *reinterpret_cast<const uint2*>(reinterpret_cast<const bf16*>(e.resid) + off)
                                                  : make_uint2(0u, 0u);
        }
      };
      auto load_resid = [&](int c, float4 (&x)[8]) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = i * 4 + rsub;
          const long long off = (long long)rrow_s[rr] * e.resid_ld + nb * BN + c * 32 + c4;
          if (!(rr < nvalid && orow_s[rr] >= 0)) {
            x[i] = make_float4(0.f, 0.f, 0.f, 0.f);
          } else if constexpr (RB16) {
            const uint2 u = *reinterpret_cast<const uint2*>(reinterpret_cast<const bf16*>(e.resid) + off);
            const float2 lo = unpack_bf16x2(u.x), hi = unpack_bf16x2(u.y);
            x[i] = make_float4(lo.x, lo.y, hi.x, hi.y);
          } else {
            x[i] = *reinterpret_cast<const float4*>(reinterpret_cast<const float*>(e.resid) + off);
          }
        }
      };
      // SR: this lane's 8 x 16 B of chunk c go to ring slot c % RDEPTH (read back by the same
      // lane, so a per-thread cp.async.wait_group is the only synchronisation needed)
      const uint32_t ring = smem_u32(sRes + (warp - 2) * RDEPTH * 1024);
      auto issue_resid = [&](int c) {
        if (c < c_end) {
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = i * 4 + rsub;
            const bool live = rr < nvalid && orow_s[rr] >= 0;
            const int rrow = __shfl_sync(0xffffffffu, rrow_reg, live ? rr : 0);
            const long long off = (long long)rrow * e.resid_ld + nb * BN + c * 32 + c4;
            const uint32_t dst = ring + (uint32_t)(((c % RDEPTH) * 32 + rr) * 128 + c4 * 4);
            if constexpr (RB16)   // 4 bf16 = 8 B into the first half of the lane's 16 B chunk
              asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst),
                           "l"(reinterpret_cast<const bf16*>(e.resid) + off), "r"(live ? 8 : 0)
                           : "memory");
            else
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst),
                           "l"(reinterpret_cast<const float*>(e.resid) + off), "r"(live ? 16 : 0)
                           : "memory");
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");   // one group per chunk slot (maybe empty)
      };
      if (e.resid) {
        if constexpr (SR) {
          for (int k = 0; k < RDEPTH; ++k) issue_resid(c_beg + k);
        } else if constexpr (MODE == 0) {
          load_resid(c_beg, xn);
        }
      }
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
#pragma unroll 1
      for (int c = c_beg; c < c_end; ++c) {
        float4 xc[8];
        if constexpr (SR) {
          if (e.resid) {
            asm volatile("cp.async.wait_group %0;" ::"n"(RDEPTH - 1) : "memory");
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const int rr = i * 4 + rsub;
              const uint32_t a = ring + (uint32_t)(((c % RDEPTH) * 32 + rr) * 128 + c4 * 4);
              if constexpr (RB16) {
                uint32_t u0, u1;
                asm volatile("ld.shared.v2.b32 {%0, %1}, [%2];" : "=r"(u0), "=r"(u1) : "r"(a) : "memory");
                const float2 lo = unpack_bf16x2(u0), hi = unpack_bf16x2(u1);
                xc[i] = make_float4(lo.x, lo.y, hi.x, hi.y);
              } else {
                xc[i] = lds128(a);
              }
            }
          }
          // the slot's residual is in registers: it now serves as this chunk's transpose tile
          tile_u = ring + (uint32_t)((c % RDEPTH) * 32 * 128);
          __syncwarp();
        } else if constexpr (MODE == 0) {
#pragma unroll
          for (int i = 0; i < 8; ++i) xc[i] = xn[i];
          if (e.resid && c + 1 < c_end) load_resid(c + 1, xn);
        } else {
          // RE: twice the warps hide the latency; this chunk's residual loads overlap the
          // TMEM load and the transpose below (no register prefetch: 96 registers per thread)
          if (RB16 && e.resid) {
            // bf16 rows: 32 columns are 64 B, half a line; the warp's next chunk holds the other
            // half, so both chunks' loads are issued together (one 128 B access per row instead
            // of two 64 B ones apart in time) and the next chunk's wait in registers (16)
            uint2 cur16[8];
            if (c == c_beg) {
              load_resid16(c, cur16);
              if (c + 1 < c_end) load_resid16(c + 1, rn16);
            } else {
#pragma unroll
              for (int i = 0; i < 8; ++i) cur16[i] = rn16[i];
              if (c + 1 < c_end) load_resid16(c + 1, rn16);
            }
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float2 lo = unpack_bf16x2(cur16[i].x), hi = unpack_bf16x2(cur16[i].y);
              xc[i] = make_float4(lo.x, lo.y, hi.x, hi.y);
            }
          } else if (e.resid) {
            load_resid(c, xc);
          }
        }
        uint32_t r[32];
        tmem_ld32(tmem_base + (uint32_t(q * 32) << 16) + acc * BN + c * 32, r);
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4)   // 16-B chunk j4 of row `lane` at chunk slot j4 ^ (lane & 7)
          sts128(tile_u + lane * 128 + ((j4 ^ (lane & 7)) << 4), r[4 * j4], r[4 * j4 + 1], r[4 * j4 + 2], r[4 * j4 + 3]);
        __syncwarp();
        const int n0 = nb * BN + c * 32 + c4;
        const bool second = n0 >= e.split;
        void* base = second ? e.out2 : e.out;
        const long long ld = second ? e.out2_ld : e.out_ld;
        const int col = second ? n0 - e.split : n0;
        const bool obf16 = second ? e.out2_bf16 : e.out_bf16;
        float4 b = make_float4(0.f, 0.f, 0.f, 0.f);
        if (e.bias) b = __ldg(reinterpret_cast<const float4*>(e.bias + n0));
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = i * 4 + rsub;
          const float4 t4 = lds128(tile_u + rr * 128 + (((lane & 7) ^ (rr & 7)) << 4));
          float4 v = make_float4(t4.x + b.x, t4.y + b.y, t4.z + b.z, t4.w + b.w);
          if (e.act == 1) {
            v.x = quick_gelu_fast(v.x); v.y = quick_gelu_fast(v.y);
            v.z = quick_gelu_fast(v.z); v.w = quick_gelu_fast(v.w);
          }
          if (e.resid) { v.x += xc[i].x; v.y += xc[i].y; v.z += xc[i].z; v.w += xc[i].w; }
          if (rr >= nvalid) continue;
          const int m = row0 + rr;
          const int orr = second ? (e.out2_rows ? __ldg(e.out2_rows + m) : m) : orow_s[rr];
          if (orr < 0) continue;   // row map -1: result not stored (restoration over C rows)
          const long long off = (long long)orr * ld + col;
          if (obf16) {
            uint2 u;
            u.x = pack_bf16x2(v.x, v.y);
            u.y = pack_bf16x2(v.z, v.w);
            *reinterpret_cast<uint2*>(reinterpret_cast<bf16*>(base) + off) = u;
          } else {
            *reinterpret_cast<float4*>(reinterpret_cast<float*>(base) + off) = v;
          }
        }
        __syncwarp();   // every lane has read the (transpose tile in the) slot
        if constexpr (SR) {
          if (e.resid) issue_resid(c + RDEPTH);   // refill the slot consumed above
        }
      }
      tc_fence_before();
      if constexpr (PAIR) {
        __syncwarp();
        if (lane == 0) mbar_arrive_cl(mapa_rank(&tempty[acc], 0));
      } else {
        mbar_arrive(&tempty[acc]);
      }
    }
  }
  tc_fence_before();
  __syncwarp();
  // PAIR: no CTA leaves while its partner may still signal its barriers or read its smem
  if constexpr (PAIR) cluster_sync_all(); else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS));
    else
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(C::TMEM_COLS));
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

bool encode_2d(CUtensorMap* m, const void* ptr, long long rows, int cols, int box_rows, char* err,
               size_t errlen) {
  auto fn = encode_fn();
  if (!fn) {
    snprintf(err, errlen, "cuTensorMapEncodeTiled unavailable");
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    snprintf(err, errlen, "cuTensorMapEncodeTiled failed (%d) rows=%lld cols=%d", (int)r, rows, cols);
    return false;
  }
  return true;
}

int num_sms() { return dev_sms(); }

template <int BN, int MODE, bool RB16 = false>
cudaError_t launch_mode(const GemmPlan& p, const int* M_dev, int M_host, int max_m, const Epi& e, cudaStream_t s) {
  using C = Cfg<BN, MODE>;
  cudaError_t err = ensure_smem<gemm_tc_kernel<BN, MODE, false, RB16>>(C::SMEM);
  if (err != cudaSuccess) return err;
  const int tiles = ((max_m + BM - 1) / BM) * (p.N / BN);
  int grid = tiles < num_sms() ? tiles : num_sms();
  if (grid < 1) grid = 1;
  gemm_tc_kernel<BN, MODE, false, RB16><<<grid, gemm_threads<BN, MODE>(), C::SMEM, s>>>(p.tmA, p.tmB, M_dev, M_host, p.N, p.K, e);
  return cudaGetLastError();
}

// CTA-pair launch: clusters of 2 (one TPC), grid = 2 x min(tiles, SMs / 2)
template <int BN, int MODE, bool RB16 = false>
cudaError_t launch_pair(const GemmPlan& p, const int* M_dev, int M_host, int max_m, const Epi& e, cudaStream_t s) {
  using C = Cfg<BN, MODE, true>;
  cudaError_t err = ensure_smem<gemm_tc_kernel<BN, MODE, true, RB16>>(C::SMEM);
  if (err != cudaSuccess) return err;
  cudaLaunchConfig_t cfg = {};
  cfg.blockDim = dim3(gemm_threads<BN, MODE>());
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  // persistent: only as many pairs as can be co-resident (TPC pairing can leave SMs unpaired;
  // a second wave of pairs would double the time of the tiles they own)
  static std::atomic<int> max_pairs_dev[64];   // per device (cudaOccupancyMaxActiveClusters)
  int max_pairs = max_pairs_dev[cur_device()].load();
  if (!max_pairs) {
    cfg.gridDim = dim3(num_sms() & ~1);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, gemm_tc_kernel<BN, MODE, true, RB16>, &cfg) != cudaSuccess || n < 1) {
      cudaGetLastError();
      n = num_sms() / 2;
    }
    max_pairs = n < num_sms() / 2 ? n : num_sms() / 2;
    max_pairs_dev[cur_device()].store(max_pairs);
  }
  const int tiles = ((max_m + C::TILE_M - 1) / C::TILE_M) * (p.N / BN);
  int pairs = max_pairs;
  if (tiles < pairs) pairs = tiles;
  if (pairs < 1) pairs = 1;
  cfg.gridDim = dim3(2 * pairs);
  return cudaLaunchKernelEx(&cfg, gemm_tc_kernel<BN, MODE, true, RB16>, p.tmA, p.tmB2, M_dev, M_host, p.N, p.K, e);
}

#ifndef RV_GEMM_RE
#define RV_GEMM_RE 1
#endif
#ifndef RV_GEMM_PAIR
#define RV_GEMM_PAIR 1
#endif
template <int BN>
cudaError_t launch_bn(const GemmPlan& p, const int* M_dev, int M_host, int max_m, const Epi& e,
                      cudaStream_t s) {
  // short K with a residual: 2-stage mainloop + cp.async residual ring (R2); a gathered residual
  // with K <= 1024 (W_o): 16 epilogue warps, 3 stages (tools/r2_bench.py: 57 -> 52 us on a
  // 16k-row W_o; FC2's K = 4096 mainloop needs its 4 stages).  Experiment builds only
  // (build.build_variant): -DRV_GEMM_RE=0 disables.
  constexpr bool re_on = RV_GEMM_RE != 0;
  // RV_GEMM_PAIR (compile-time): CTA pairs (256 x 256 tiles) for the MODE 0 / 2 GEMMs with
  // BN = 256 (tools/gemm_bench.py at M = 80k: QKV 432 -> 385 us, FC1 572 -> 521, FC2 508 -> 464,
  // W_o 193 -> 154; in the bench FC2 67 -> 60 ms per step); R1 (N = 128) stays single-CTA
  // (17 -> 20 ms as pairs: half as many 256-row tiles on small waves)
  constexpr bool pair_on = RV_GEMM_PAIR != 0;
  if (p.K <= 2 * BK && e.resid)
    return e.resid_bf16 ? launch_mode<BN, 1, true>(p, M_dev, M_host, max_m, e, s)
                        : launch_mode<BN, 1>(p, M_dev, M_host, max_m, e, s);
// RV_GEMM_RE_KMAX: largest K that takes the 16-warp epilogue (MODE 2).  FC2 (K = 4096) as MODE 2
// pairs: 70.1 vs 60.8 ms per step as MODE 0 pairs (fewer stages for its long mainloop)
#ifndef RV_GEMM_RE_KMAX
#define RV_GEMM_RE_KMAX 1024
#endif
  if constexpr (BN == 256) {
    if (pair_on) {
      if (re_on && p.K <= RV_GEMM_RE_KMAX && (e.resid ? BN >= 128 : BN == 256))
        return (e.resid && e.resid_bf16) ? launch_pair<BN, 2, true>(p, M_dev, M_host, max_m, e, s)
                                         : launch_pair<BN, 2>(p, M_dev, M_host, max_m, e, s);
      return launch_pair<BN, 0>(p, M_dev, M_host, max_m, e, s);
    }
  }
  // 16-warp epilogue: W_o (gathered residual, BN >= 128) and the wide bf16-output GEMMs with
  // K <= 1024 (QKV with its K/V scatter, FC1 with QuickGELU: 65 -> 57 and 82 -> 73 ms per step);
  // not R1 (N = 128: one N tile, slower)
  if (re_on && p.K <= 1024 && (e.resid ? BN >= 128 : BN == 256))
    return (e.resid && e.resid_bf16) ? launch_mode<BN, 2, true>(p, M_dev, M_host, max_m, e, s)
                                     : launch_mode<BN, 2>(p, M_dev, M_host, max_m, e, s);
  return (e.resid && e.resid_bf16) ? launch_mode<BN, 0, true>(p, M_dev, M_host, max_m, e, s)
                                   : launch_mode<BN, 0>(p, M_dev, M_host, max_m, e, s);
}

}  // namespace

bool make_tmap_bf16(CUtensorMap* m, const void* ptr, long long rows, int cols, int box_rows, char* err,
                    size_t errlen) {
  return encode_2d(m, ptr, rows, cols, box_rows, err, errlen);
}

bool gemm_make_plan(GemmPlan* p, const void* A, long long a_rows, const void* B, int N, int K, char* err,
                    size_t errlen, int bn_max) {
  if (K % BK != 0 || N % 64 != 0) {
    snprintf(err, errlen, "gemm: K=%d must be a multiple of 64 and N=%d a multiple of 64", K, N);
    return false;
  }
  p->N = N;
  p->K = K;
  p->BN = (N % 256 == 0 && bn_max >= 256) ? 256 : ((N % 128 == 0 && bn_max >= 128) ? 128 : 64);
  return encode_2d(&p->tmA, A, a_rows, K, BM, err, errlen) && encode_2d(&p->tmB, B, N, K, p->BN, err, errlen) &&
         encode_2d(&p->tmB2, B, N, K, p->BN >= 128 ? p->BN / 2 : p->BN, err, errlen);
}

cudaError_t gemm_launch(const GemmPlan& p, const int* M_dev, int M_host, int max_m, const Epi& e,
                        cudaStream_t s) {
  switch (p.BN) {
    case 256: return launch_bn<256>(p, M_dev, M_host, max_m, e, s);
    case 128: return launch_bn<128>(p, M_dev, M_host, max_m, e, s);
    default: return launch_bn<64>(p, M_dev, M_host, max_m, e, s);
  }
}

}  // namespace rv
