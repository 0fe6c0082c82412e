// k_restore.cu — fused restoration (Eq. 8-10) over the compacted
// reused rows of a level wave, one persistent warp-specialised tcgen05 kernel:
//
//   hr       = QuickGELU(Delta W_r1^T + b_r1)                 (Eq. 9 first layer, Hr = 128)
//   X_l[i]   = X_l[prov(i)] + hr W_r2^T + b_r2                 (Eq. 9 second layer + Eq. 10 merge)
//
// for the M_R reused tokens r of the wave (Delta rows written by score_kernel at the token's
// wave-local row rloc[r], Eq. 8; provider row provrow[r]; output row idxR[r]).  Compared with the
// two-GEMM path (R1 over all n_w T wave rows, hr through HBM, R2), it reads only the reused rows'
// Delta (gathered by cp.async), keeps hr on chip (TMEM -> bf16 SWIZZLE_128B tile in shared
// memory = the A operand of the second MMA) and streams the provider rows / output rows of X:
// 2 + 8 KB of HBM per reused row at D = 1024 (fp32 X; 2 + 4 KB with RV_X_BF16).
//
// Tile = 128 reused rows (MMA M).  CTA = 12 warps, one CTA per SM (persistent over tiles):
//   warps 0-1  Delta loaders: 128 rows x 64 columns (16 KB, SWIZZLE_128B K-major) per K chunk
//              into a 4-stage ring, completion by cp.async.mbarrier.arrive.noinc
//   warp 2     TMEM allocator (512 columns: acc1[2] at 0 / 128, acc2[2] at 256 / 384) and the
//              single-thread MMA issuer, software-pipelined R1(t+1) before R2(t) so the tensor
//              pipe has R1 work while the epilogue turns acc1(t) into the hr tile
//   warp 3     weight producer: TMA boxes {64, 128} of W_r1 (16 per tile) and W_r2 (2 per 128
//              output columns) into a 4-slot ring, in exactly the issuer's order
//   warps 4-11 epilogue (warp % 4 = TMEM lane quarter, (warp - 4) / 4 = column half):
//              (1) acc1 -> + b_r1 -> QuickGELU -> bf16 -> hr tile (A2), (2) per 32-column chunk
//              of acc2: provider rows prefetched by cp.async into a 2-deep ring whose slot then
//              serves as the transpose tile -> + b_r2 + residual -> coalesced row stores
// Arithmetic per element is the two-GEMM path's (same K order, same epilogue operations), so
// results are bitwise those of R1 + R2 as GEMMs.
#include <cuda.h>

#include "common.cuh"
#include "rv_internal.h"
#include "tc_ptx.cuh"

namespace rv {
namespace {

constexpr int RS_BM = 128;                 // reused rows per tile (MMA M)
constexpr int RS_HR = 128;                 // restoration hidden width (R1 N, R2 K)
constexpr int RS_NC = 128;                 // R2 output columns per accumulator chunk (MMA N)
#ifndef RS_AST_N
#define RS_AST_N 4
#endif
#ifndef RS_KPS_N
#define RS_KPS_N 1
#endif
#ifndef RS_WST_N
#define RS_WST_N 4
#endif
#ifndef RS_RDEPTH_N
#define RS_RDEPTH_N 2
#endif
constexpr int RS_AST = RS_AST_N;           // Delta ring stages
constexpr int RS_KPS = RS_KPS_N;           // 64-column K chunks per Delta stage (128 B x RS_KPS per row)
constexpr int RS_WST = RS_WST_N;           // weight chunk ring slots
constexpr int RS_EPI = 8;                  // epilogue warps
constexpr int RS_RDEPTH = RS_RDEPTH_N;     // residual chunks in flight per epilogue warp
constexpr int RS_THREADS = (4 + RS_EPI) * 32;
constexpr uint32_t RS_CHUNK = 128 * 128;   // 128 rows x 128 B (one SWIZZLE_128B K-major block)
constexpr uint32_t RS_OFF_W = RS_AST * RS_KPS * RS_CHUNK;
constexpr uint32_t RS_OFF_A2 = RS_OFF_W + RS_WST * RS_CHUNK;
constexpr uint32_t RS_OFF_EPI = RS_OFF_A2 + 2 * RS_CHUNK;
constexpr uint32_t RS_OFF_BAR = RS_OFF_EPI + RS_EPI * RS_RDEPTH * 4096;
constexpr uint32_t RS_SMEM = RS_OFF_BAR + 256 + 1024;   // + barriers + 1 KB alignment slack
static_assert(RS_SMEM <= 232448, "restore kernel exceeds 227 KB of shared memory");

RV_DEV void tma_2d_l(uint32_t dst, const CUtensorMap* tm, int c0, int c1, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          dst),
      "l"(tm), "r"(c0), "r"(c1), "r"(su32(bar))
      : "memory");
}
RV_DEV void sts128r(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}
RV_DEV float4 lds128r(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
  return v;
}
// tcgen05.ld 32x32b.x32 and its wait in one asm statement: the registers are defined only
// after the wait, so no use can be scheduled between the two
RV_DEV void tld32w(uint32_t taddr, float* v) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n\t"
      "tcgen05.wait::ld.sync.aligned;"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
        "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
        "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
        "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr)
      : "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}
// the GEMM epilogue's QuickGELU (k_gemm.cu), so hr is bitwise the R1 GEMM's
RV_DEV float quick_gelu_tanh(float x) {
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.851f * x));
  return x * fmaf(0.5f, t, 0.5f);
}

template <typename XT>
__global__ void __launch_bounds__(RS_THREADS, 1)
    restore_kernel(const __grid_constant__ CUtensorMap tmW1, const __grid_constant__ CUtensorMap tmW2,
                   const bf16* __restrict__ dfull, const int* __restrict__ rloc, const int* __restrict__ provrow,
                   const int* __restrict__ idxR, const int* __restrict__ M_dev, const float* __restrict__ br1,
                   const float* __restrict__ br2, XT* X, int D) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t base = (su32(smem_raw) + 1023u) & ~1023u;   // SWIZZLE_128B blocks: 1 KB aligned
  uint8_t* gbase = smem_raw + (base - su32(smem_raw));
  uint64_t* bars = reinterpret_cast<uint64_t*>(gbase + RS_OFF_BAR);
  uint64_t* a_full = bars;                  // [RS_AST]
  uint64_t* a_empty = a_full + RS_AST;      // [RS_AST]
  uint64_t* w_full = a_empty + RS_AST;      // [RS_WST]
  uint64_t* w_empty = w_full + RS_WST;      // [RS_WST]
  uint64_t* acc1_full = w_empty + RS_WST;   // [2]
  uint64_t* acc1_empty = acc1_full + 2;     // [2]
  uint64_t* acc2_full = acc1_empty + 2;     // [2]
  uint64_t* acc2_empty = acc2_full + 2;     // [2]
  uint64_t* a2_full = acc2_empty + 2;       // [1]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(a2_full + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int M = *M_dev;
  const int ntiles = (M + RS_BM - 1) / RS_BM;
  const int nk = D / 64;           // R1 K chunks
  const int nn = D / RS_NC;        // R2 output chunks
  if (threadIdx.x == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW1) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW2) : "memory");
    for (int i = 0; i < RS_AST; ++i) {
      mbar_init(&a_full[i], 64);    // every loader lane's cp.async (arrive.noinc)
      mbar_init(&a_empty[i], 1);    // MMA commit
    }
    for (int i = 0; i < RS_WST; ++i) {
      mbar_init(&w_full[i], 1);     // producer expect_tx + TMA bytes
      mbar_init(&w_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&acc1_full[i], 1);
      mbar_init(&acc1_empty[i], RS_EPI * 32);
      mbar_init(&acc2_full[i], 1);
      mbar_init(&acc2_empty[i], RS_EPI * 32);
    }
    mbar_init(a2_full, RS_EPI * 32);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)), "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tslot;

  if (warp < 2) {
    // ==================================================================== Delta loaders
    // lane L of the 64: 16 B column chunk L % 8 of rows L / 8 + 8 i (i < 16) of every K chunk
    const int l64 = warp * 32 + lane;
    // (RS_KPS chunks per stage: 8 RS_KPS lanes copy a row's 128 RS_KPS contiguous bytes)
    constexpr int LPR = 8 * RS_KPS, RPP = 64 / LPR, NIT = RS_BM / RPP;
    const int c16 = l64 % LPR, r0 = l64 / LPR, blk = c16 >> 3, c = c16 & 7;
    int s = 0;
    uint32_t ph = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      int src[NIT];
#pragma unroll
      for (int i = 0; i < NIT; ++i) {
        const int m = tile * RS_BM + r0 + RPP * i;
        src[i] = m < M ? __ldg(rloc + m) : -1;
      }
      for (int kc = 0; kc < nk; kc += RS_KPS) {
        mbar_wait(&a_empty[s], ph ^ 1);
        const uint32_t dst = base + (s * RS_KPS + blk) * RS_CHUNK;
#pragma unroll
        for (int i = 0; i < NIT; ++i) {
          const int r = r0 + RPP * i;
          const bf16* g = dfull + (long long)(src[i] < 0 ? 0 : src[i]) * D + kc * 64 + c16 * 8;
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + r * 128 + ((c ^ (r & 7)) << 4)),
                       "l"(g), "r"(src[i] < 0 ? 0 : 16)
                       : "memory");
        }
        cp_async_arrive(&a_full[s]);
        if (++s == RS_AST) { s = 0; ph ^= 1; }
      }
    }
  } else if (warp == 3) {
    // ==================================================================== weight producer
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      auto put = [&](const CUtensorMap* tm, int c0, int c1) {
        mbar_wait(&w_empty[s], ph ^ 1);
        mbar_expect_tx(&w_full[s], RS_CHUNK);
        tma_2d_l(base + RS_OFF_W + s * RS_CHUNK, tm, c0, c1, &w_full[s]);
        if (++s == RS_WST) { s = 0; ph ^= 1; }
      };
      int ntl = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) ++ntl;
      for (int it = 0; it <= ntl; ++it) {   // issuer order: R1(it), then R2(it - 1)
        if (it < ntl)
          for (int kc = 0; kc < nk; ++kc) put(&tmW1, kc * 64, 0);
        if (it >= 1)
          for (int nc = 0; nc < nn; ++nc) {
            put(&tmW2, 0, nc * RS_NC);
            put(&tmW2, 64, nc * RS_NC);
          }
      }
    }
  } else if (warp == 2) {
    // ==================================================================== MMA issuer
    if (lane == 0) {
      const uint32_t idesc = idesc_f16(RS_BM, 128, 0);
      int as = 0, ws = 0, n2 = 0;
      uint32_t aph = 0, wph = 0;
      int ntl = 0;
      for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) ++ntl;
      for (int it = 0; it <= ntl; ++it) {
        if (it < ntl) {   // R1(it): acc1[it & 1] = Delta W_r1^T
          const int b = it & 1;
          mbar_wait(&acc1_empty[b], ((it >> 1) & 1) ^ 1);
          tc_after();
          const uint32_t d = tmem + b * 128;
          for (int kc0 = 0; kc0 < nk; kc0 += RS_KPS) {
            mbar_wait(&a_full[as], aph);
            for (int bk = 0; bk < RS_KPS; ++bk) {
              const int kc = kc0 + bk;
              mbar_wait(&w_full[ws], wph);
              tc_after();
              const uint64_t ad = sdesc(base + (as * RS_KPS + bk) * RS_CHUNK), bd = sdesc(base + RS_OFF_W + ws * RS_CHUNK);
#pragma unroll
              for (int k = 0; k < 4; ++k) mma_ss(d, ad + 2 * k, bd + 2 * k, idesc, (kc | k) != 0);
              mma_commit(&w_empty[ws]);
              if (++ws == RS_WST) { ws = 0; wph ^= 1; }
            }
            mma_commit(&a_empty[as]);
            if (++as == RS_AST) { as = 0; aph ^= 1; }
          }
          mma_commit(&acc1_full[b]);
        }
        if (it >= 1) {    // R2(it - 1): acc2 chunks = hr W_r2^T, hr from the A2 tile
          mbar_wait(a2_full, (uint32_t)((it - 1) & 1));
          tc_after();
          for (int nc = 0; nc < nn; ++nc, ++n2) {
            const int b = n2 & 1;
            mbar_wait(&acc2_empty[b], ((n2 >> 1) & 1) ^ 1);
            tc_after();
            const uint32_t d = tmem + 256 + b * 128;
            for (int kh = 0; kh < 2; ++kh) {
              mbar_wait(&w_full[ws], wph);
              tc_after();
              const uint64_t ad = sdesc(base + RS_OFF_A2 + kh * RS_CHUNK), bd = sdesc(base + RS_OFF_W + ws * RS_CHUNK);
#pragma unroll
              for (int k = 0; k < 4; ++k) mma_ss(d, ad + 2 * k, bd + 2 * k, idesc, (kh | k) != 0);
              mma_commit(&w_empty[ws]);
              if (++ws == RS_WST) { ws = 0; wph ^= 1; }
            }
            mma_commit(&acc2_full[b]);
          }
        }
      }
    }
  } else {
    // ==================================================================== epilogue
    const int q = warp & 3;               // TMEM lane quarter: tile rows 32q .. 32q + 31
    const int half = (warp - 4) >> 2;     // hidden columns 64 half.. (1); output columns 64 half.. of a chunk (2)
    const int rsub = lane >> 3, c4 = (lane & 7) * 4;
    const uint32_t ring = base + RS_OFF_EPI + (uint32_t)(warp - 4) * RS_RDEPTH * 4096;
    const uint32_t tq = tmem + ((uint32_t)(q * 32) << 16);
    // column sub-chunks of a 128-column chunk per warp: fp32 X 2 x 32 columns (128 B of a row);
    // bf16 X one 64-column sub-chunk (also 128 B of a row), added in place in its ring slot
    constexpr bool XB = sizeof(XT) == 2;
    constexpr int NSUB = XB ? 1 : 2;
    int n2 = 0, it = 0;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x, ++it) {
      const int m = tile * RS_BM + q * 32 + lane;
      const bool valid = m < M;
      const int prow = valid ? __ldg(provrow + m) : 0;
      const int orow = valid ? __ldg(idxR + m) : -1;
      const int nsub = nn * NSUB;        // this warp's 32-column chunks of the tile
      auto col_of = [&](int cidx) { return (cidx / NSUB) * RS_NC + half * 64 + (cidx % NSUB) * 32; };
      auto issue_resid = [&](int cidx) {
        if (cidx < nsub) {
          const int col = col_of(cidx);
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = i * 4 + rsub;
            const int pr = __shfl_sync(0xffffffffu, prow, rr);
            const bool live = __shfl_sync(0xffffffffu, orow, rr) >= 0;
            if constexpr (!XB) {
              const uint32_t dst = ring + (uint32_t)(((cidx % RS_RDEPTH) * 32 + rr) * 128 + c4 * 4);
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst),
                           "l"(X + (long long)pr * D + col + c4), "r"(live ? 16 : 0)
                           : "memory");
            } else {   // 16 B = 8 bf16 columns c8 = lane & 7, XOR-swizzled by row
              const int c8 = lane & 7;
              const uint32_t dst = ring + (uint32_t)(((cidx % RS_RDEPTH) * 32 + rr) * 128 + ((c8 ^ (rr & 7)) << 4));
              asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst),
                           "l"(X + (long long)pr * D + col + c8 * 8), "r"(live ? 16 : 0)
                           : "memory");
            }
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
      };
      for (int k = 0; k < RS_RDEPTH; ++k) issue_resid(k);   // overlaps the R1 MMAs and (1)
      // ---- (1) hr = QuickGELU(acc1 + b_r1) -> bf16 A2 tile (row r = 32q + lane, columns 64 half ..)
      {
        const int b = it & 1;
        mbar_wait(&acc1_full[b], (uint32_t)((it >> 1) & 1));
        tc_after();
        const int r = q * 32 + lane;
        const uint32_t arow = base + RS_OFF_A2 + half * RS_CHUNK + r * 128;
#pragma unroll
        for (int h2 = 0; h2 < 2; ++h2) {
          float v[32];
          tld32w(tq + b * 128 + half * 64 + h2 * 32, v);
          uint32_t p[16];
#pragma unroll
          for (int j = 0; j < 16; ++j) {
            const int hc = half * 64 + h2 * 32 + 2 * j;
            p[j] = pack_bf16x2(quick_gelu_tanh(v[2 * j] + __ldg(br1 + hc)), quick_gelu_tanh(v[2 * j + 1] + __ldg(br1 + hc + 1)));
          }
#pragma unroll
          for (int j4 = 0; j4 < 4; ++j4) {
            const int ch = h2 * 4 + j4;   // 16 B chunk (8 bf16) of the 128 B row
            sts128r(arow + ((ch ^ (r & 7)) << 4), p[4 * j4], p[4 * j4 + 1], p[4 * j4 + 2], p[4 * j4 + 3]);
          }
        }
        tc_before();
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic stores -> tensor core
        mbar_arrive(&acc1_empty[b]);
        mbar_arrive(a2_full);
      }
      // ---- (2) X[idxR] = acc2 + b_r2 + X[provrow], 32 columns at a time
#pragma unroll 1
      for (int cidx = 0; cidx < nsub; ++cidx) {
        const int b = n2 & 1;
        if (cidx % NSUB == 0) {
          mbar_wait(&acc2_full[b], (uint32_t)((n2 >> 1) & 1));
          tc_after();
        }
        const int col = col_of(cidx);
        asm volatile("cp.async.wait_group %0;" ::"n"(RS_RDEPTH - 1) : "memory");
        if constexpr (XB) {
          // thread = row (TMEM lane 32q + lane): its 64 accumulators + b_r2 + its residual row
          // segment (from the slot), rounded once to bf16 and written back in place; then 8
          // lanes per row store the slot's rows coalesced
          const uint32_t slot = ring + (uint32_t)((cidx % RS_RDEPTH) * 32 * 128);
          __syncwarp();
#pragma unroll
          for (int h2 = 0; h2 < 2; ++h2) {
            float v[32];
            tld32w(tq + 256 + b * 128 + half * 64 + h2 * 32, v);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
              const int ch = h2 * 4 + j;   // 16 B chunk of the row segment = columns 8 ch ..
              const uint32_t a = slot + lane * 128 + ((ch ^ (lane & 7)) << 4);
              uint32_t u[4];
              asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]) : "r"(a) : "memory");
              const float4 b0 = __ldg(reinterpret_cast<const float4*>(br2 + col + 8 * ch));
              const float4 b1 = __ldg(reinterpret_cast<const float4*>(br2 + col + 8 * ch + 4));
              const float bb[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
              uint32_t o[4];
#pragma unroll
              for (int e = 0; e < 4; ++e) {
                const float2 x = unpack_bf16x2(u[e]);
                o[e] = pack_bf16x2((v[8 * j + 2 * e] + bb[2 * e]) + x.x, (v[8 * j + 2 * e + 1] + bb[2 * e + 1]) + x.y);
              }
              sts128r(a, o[0], o[1], o[2], o[3]);
            }
          }
          __syncwarp();
          const int c8 = lane & 7;
#pragma unroll
          for (int i = 0; i < 8; ++i) {
            const int rr = i * 4 + rsub;
            const int orr = __shfl_sync(0xffffffffu, orow, rr);
            uint32_t u[4];
            asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                         : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3])
                         : "r"(slot + rr * 128 + ((c8 ^ (rr & 7)) << 4))
                         : "memory");
            if (orr >= 0) *reinterpret_cast<uint4*>(X + (long long)orr * D + col + c8 * 8) = make_uint4(u[0], u[1], u[2], u[3]);
          }
          __syncwarp();
          issue_resid(cidx + RS_RDEPTH);
          if (cidx % NSUB == NSUB - 1) {
            tc_before();
            mbar_arrive(&acc2_empty[b]);
            ++n2;
          }
          continue;
        }
        float4 xc[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = i * 4 + rsub;
          const uint32_t a = ring + (uint32_t)(((cidx % RS_RDEPTH) * 32 + rr) * 128 + c4 * 4);
          xc[i] = lds128r(a);
        }
        const uint32_t tile_u = ring + (uint32_t)((cidx % RS_RDEPTH) * 32 * 128);
        __syncwarp();   // every lane has its residual: the slot becomes the transpose tile
        {
          float v[32];
          tld32w(tq + 256 + b * 128 + half * 64 + (cidx % NSUB) * 32, v);
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4)
            sts128r(tile_u + lane * 128 + ((j4 ^ (lane & 7)) << 4), __float_as_uint(v[4 * j4]),
                    __float_as_uint(v[4 * j4 + 1]), __float_as_uint(v[4 * j4 + 2]), __float_as_uint(v[4 * j4 + 3]));
        }
        __syncwarp();
        const float4 bb = __ldg(reinterpret_cast<const float4*>(br2 + col + c4));
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int rr = i * 4 + rsub;
          const int orr = __shfl_sync(0xffffffffu, orow, rr);
          const float4 t4 = lds128r(tile_u + rr * 128 + (((lane & 7) ^ (rr & 7)) << 4));
          float4 v = make_float4(t4.x + bb.x, t4.y + bb.y, t4.z + bb.z, t4.w + bb.w);
          v.x += xc[i].x; v.y += xc[i].y; v.z += xc[i].z; v.w += xc[i].w;
          if (orr < 0) continue;
          *reinterpret_cast<float4*>(reinterpret_cast<float*>(X) + (long long)orr * D + col + c4) = v;
        }
        __syncwarp();   // the slot's transpose reads are done before it is refilled
        issue_resid(cidx + RS_RDEPTH);
        if (cidx % NSUB == NSUB - 1) {
          tc_before();
          mbar_arrive(&acc2_empty[b]);
          ++n2;
        }
      }
    }
  }
  tc_before();
  __syncthreads();
  if (warp == 2) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

}  // namespace

bool restore_supported(int D, int Hr) { return Hr == RS_HR && D % RS_NC == 0 && D % (64 * RS_KPS) == 0 && D >= RS_NC; }

bool restore_make_maps(CUtensorMap* tmW1, CUtensorMap* tmW2, const bf16* Wr1, const bf16* Wr2, int D, int Hr,
                       char* err, size_t errlen) {
  // W_r1 [Hr][D] and W_r2 [D][Hr] (K-major B operands), boxes {64 columns, 128 rows}
  return make_tmap_bf16(tmW1, Wr1, Hr, D, 128, err, errlen) && make_tmap_bf16(tmW2, Wr2, D, Hr, 128, err, errlen);
}

cudaError_t launch_restore(const CUtensorMap& tmW1, const CUtensorMap& tmW2, const bf16* dfull, const int* rloc,
                           const int* provrow, const int* idxR, const int* M_dev, int max_rows, const float* br1,
                           const float* br2, void* X, int x_bf16, int D, cudaStream_t s) {
  if (max_rows <= 0) return cudaSuccess;
  const int sms = dev_sms();
  const int tiles = (max_rows + RS_BM - 1) / RS_BM;
  const int grid = tiles < sms ? tiles : sms;
  if (x_bf16) {
    cudaError_t e = ensure_smem<restore_kernel<bf16>>(RS_SMEM);
    if (e != cudaSuccess) return e;
    restore_kernel<bf16><<<grid, RS_THREADS, RS_SMEM, s>>>(tmW1, tmW2, dfull, rloc, provrow, idxR, M_dev, br1, br2,
                                                            reinterpret_cast<bf16*>(X), D);
  } else {
    cudaError_t e = ensure_smem<restore_kernel<float>>(RS_SMEM);
    if (e != cudaSuccess) return e;
    restore_kernel<float><<<grid, RS_THREADS, RS_SMEM, s>>>(tmW1, tmW2, dfull, rloc, provrow, idxR, M_dev, br1, br2,
                                                             reinterpret_cast<float*>(X), D);
  }
  return cudaGetLastError();
}

}  // namespace rv
