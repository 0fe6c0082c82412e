// ARCHIVED EXPERIMENT (not compiled into libreusevit; kept for the record of round 1):
// fused decision + R1 on the tensor cores.  Bitwise equal to score_kernel + the R1 GEMM but
// 201 ms per step vs 83 + 17 unfused.  Built only by hand against csrc/.
// k_score_r1.cu — reuse decision fused with the first restoration layer (SURVEY §8(a) a2+a3 and
// the R1 half of a12; Eq. 1-4, Eq. 8-9).
//
// The unfused path writes Delta = X_cur - X_prov (Eq. 8) as bf16 rows to HBM in the score
// kernel and reads them back in the R1 GEMM (2 x 2 KB per reused token at D = 1024).  Here a
// CTA scores 64 tokens of one frame, exactly as score_kernel does (same fp32 arithmetic, same
// decision, same outputs), and the warps that hold a reused token's rows in registers write
// its Delta (bf16) straight into a shared-memory A tile (SWIZZLE_128B, K-major: the layout TMA
// would produce).  One thread then runs hr = QuickGELU(Delta Wr1^T + br1) on the tensor cores
// (tcgen05.mma M = 64, N = Hr = 128, K = 16, fp32 accumulator in TMEM, Wr1 streamed from L2 by
// TMA in 64-column chunks, the same K order as the GEMM path), and 16 warps read the
// accumulator back and store hr to the token's wave-local row (bf16 [n_w * T][Hr]).  The R2 GEMM
// then runs over all n_w * T wave-local rows with per-row maps written here (output row of a
// reused token, -1 otherwise; its provider's row for the residual).
//
// CTA = 16 scoring / epilogue warps; warp 0 also allocates TMEM and issues the TMA and MMAs.
// Status: opt-in (RV_SCORE_R1=1), measured slower than the unfused pair (201 vs 83 + 17 ms per
// step at 7,200 frames): the A tile's shared memory allows one CTA (16 warps) per SM, so far
// fewer row loads are in flight than in score_kernel (up to 64 warps per SM), and the tile's
// MMA phase (Wr1 streamed from L2) does not overlap the next tile's loads.
// Shared memory: A tile 64 x D bf16 (128 KB at D = 1024) + a 3-stage Wr1 ring (3 x 16 KB).
#include <cuda.h>

#include "common.cuh"
#include "rv_internal.h"

namespace rv {
namespace {

constexpr int SR1_TOK = 64;          // tokens (A rows) per CTA: the MMA M
constexpr int SR1_WARPS = 16;        // scoring warps (also the epilogue: 4 per TMEM lane quarter)
constexpr int SR1_THREADS = SR1_WARPS * 32;   // warp 0 also allocates TMEM and issues TMA / MMAs
                                              // (a 17th warp would cap registers at 96: spills)
constexpr int SR1_HR = 128;          // restoration hidden width (the MMA N)
constexpr int SR1_STG = 3;           // Wr1 ring stages
constexpr int SR1_CHUNK = SR1_HR * 128;   // one 64-column chunk of Wr1: 128 rows x 128 B

RV_DEV uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
RV_DEV void bar_init(uint64_t* b, uint32_t c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
RV_DEV void bar_expect(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
RV_DEV void bar_wait(uint64_t* b, uint32_t parity) {
  uint32_t ok = 0;
  while (!ok) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(su32(b)), "r"(parity)
        : "memory");
  }
}
RV_DEV void tma2d(void* dst, const CUtensorMap* m, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          su32(dst)),
      "l"(m), "r"(x), "r"(y), "r"(su32(bar))
      : "memory");
}
RV_DEV uint64_t desc_sw128(const void* p) {
  const uint64_t a = su32(p);
  return ((a >> 4) & 0x3FFFull) | (uint64_t(1024 >> 4) << 32) | (1ull << 46) | (2ull << 61);
}
// kind::f16, D fp32, A/B bf16 K-major, N = 128, M = 64
constexpr uint32_t SR1_IDESC = (1u << 4) | (1u << 7) | (1u << 10) | (uint32_t(SR1_HR >> 3) << 17) |
                               (uint32_t(SR1_TOK >> 4) << 24);
RV_DEV void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(SR1_IDESC), "r"(acc));
}
RV_DEV void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}
RV_DEV float gelu_tanh(float x) {   // identical to the GEMM epilogue's QuickGELU (k_gemm.cu)
  float t;
  asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(0.851f * x));
  return x * fmaf(0.5f, t, 0.5f);
}

template <int VPL>
__global__ void __launch_bounds__(SR1_THREADS, 1)
    score_r1_kernel(const float* __restrict__ X, int T, int D, int N, int L, int layer,
                    const int4* __restrict__ wdesc, const float* __restrict__ tsrc, int tH,
                    const float* __restrict__ codec, const uint8_t* force, const float* __restrict__ gate, int Hg,
                    uint8_t* masks, float* scores, uint8_t* __restrict__ wmask, uint8_t* __restrict__ wprov,
                    int* __restrict__ cntR, const __grid_constant__ CUtensorMap tmW1, const float* __restrict__ br1,
                    bf16* __restrict__ hr_full, int* __restrict__ r2_out, int* __restrict__ r2_res) {
  extern __shared__ __align__(1024) uint8_t smem[];
  uint8_t* sA = smem;                                  // D / 64 chunks of [64 rows x 128 B]
  uint8_t* sW = smem + SR1_TOK * D * 2;                // SR1_STG x [128 rows x 128 B]
  uint64_t* full = reinterpret_cast<uint64_t*>(sW + SR1_STG * SR1_CHUNK);
  uint64_t* empty = full + SR1_STG;
  uint64_t* tfull = empty + SR1_STG;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tfull + 1);
  int* s_reused = reinterpret_cast<int*>(tslot + 1);
  uint8_t* s_M = reinterpret_cast<uint8_t*>(s_reused + 1);   // [64] decision of each A row

  const int w = blockIdx.x;
  const int i0 = 1 + blockIdx.y * SR1_TOK;             // token of A row 0
  const int i_end = min(N, i0 + SR1_TOK - 1);
  const int4 d4 = wdesc[w];
  const int slot = d4.x, past = d4.y, fut = d4.z, type = d4.w;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long mrow = ((long long)slot * L + layer) * N;
  const long long wrow = (long long)w * T;
  if (blockIdx.y == 0 && threadIdx.x == 0) {
    wmask[wrow] = 0;
    wprov[wrow] = 0;
    r2_out[wrow] = -1;                                 // CLS: never reused
  }
  if (type == 0 || (past < 0 && fut < 0)) {            // no decision in this frame (uniform per CTA)
    for (int i = i0 + threadIdx.x; i <= i_end; i += SR1_THREADS) {
      wmask[wrow + i] = 0;
      wprov[wrow + i] = 0;
      r2_out[wrow + i] = -1;
      if (masks) masks[mrow + i - 1] = 0;
      if (scores) scores[mrow + i - 1] = __int_as_float(0x7fc00000);
    }
    return;
  }
  const int nk = D / 64;
  if (warp == 0) {
    if (lane == 0) {
      for (int s = 0; s < SR1_STG; ++s) {
        bar_init(&full[s], 1);
        bar_init(&empty[s], 1);
      }
      bar_init(tfull, 1);
      *s_reused = 0;
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(tslot)), "r"(SR1_HR));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x < SR1_TOK) s_M[threadIdx.x] = 0;
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tslot;

  if (warp == 0 && lane == 0) {
    // Wr1 chunks 0 .. STG-1 load while the tokens are scored
    for (int c = 0; c < SR1_STG && c < nk; ++c) {
      bar_expect(&full[c], SR1_CHUNK);
      tma2d(sW + c * SR1_CHUNK, &tmW1, &full[c], c * 64, 0);
    }
  }
  {
    // ---- Eq. 1-4 for tokens i0 + warp + 16 k (score_kernel's arithmetic, D = 128 VPL)
    float w1[7], b1 = 0.f, w2 = 0.f;
#pragma unroll
    for (int k = 0; k < 7; ++k) w1[k] = lane < Hg ? __ldg(gate + k * Hg + lane) : 0.f;
    if (lane < Hg) {
      b1 = __ldg(gate + 7 * Hg + lane);
      w2 = __ldg(gate + 8 * Hg + lane);
    }
    const float b2 = __ldg(gate + 9 * Hg);
    const float oh0 = type == 0, oh1 = type == 1, oh2 = type == 2, oh3 = type == 3;
    int my_reused = 0;
    for (int i = i0 + warp; i <= i_end; i += SR1_WARPS) {
      const float4* cur = reinterpret_cast<const float4*>(X + ((long long)slot * T + i) * D);
      const float4* rp = past >= 0 ? reinterpret_cast<const float4*>(X + ((long long)past * T + i) * D) : nullptr;
      const float4* rf = fut >= 0 ? reinterpret_cast<const float4*>(X + ((long long)fut * T + i) * D) : nullptr;
      const float4* rp2 = rp ? rp : cur;
      const float4* rf2 = rf ? rf : cur;
      float4 cv[VPL], pv[VPL], fv[VPL];
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        cv[j] = __ldg(cur + lane + 32 * j);
        pv[j] = __ldg(rp2 + lane + 32 * j);
        fv[j] = __ldg(rf2 + lane + 32 * j);
      }
      float cc = 0.f, pp = 0.f, ff = 0.f, cp = 0.f, cf = 0.f;
#pragma unroll
      for (int j = 0; j < VPL; ++j) {
        const float4 c = cv[j], p = pv[j], f = fv[j];
        cc += c.x * c.x + c.y * c.y + c.z * c.z + c.w * c.w;
        pp += p.x * p.x + p.y * p.y + p.z * p.z + p.w * p.w;
        cp += c.x * p.x + c.y * p.y + c.z * p.z + c.w * p.w;
        ff += f.x * f.x + f.y * f.y + f.z * f.z + f.w * f.w;
        cf += c.x * f.x + c.y * f.y + c.z * f.z + c.w * f.w;
      }
      if (!rp) pp = cp = 0.f;
      if (!rf) ff = cf = 0.f;
      cc = warp_sum(cc);
      pp = warp_sum(pp);
      ff = warp_sum(ff);
      cp = warp_sum(cp);
      cf = warp_sum(cf);
      float s = -2.f;
      int prov = 0;
      if (rp) {
        const float den = sqrtf(cc * pp);
        s = den > 0.f ? cp / den : 0.f;
      }
      if (rf) {
        const float den = sqrtf(cc * ff);
        const float sf = den > 0.f ? cf / den : 0.f;
        if (sf > s) { s = sf; prov = 1; }   // strict: ties keep the past reference
      }
      float t = 0.f;
      for (int hh = 0; hh < tH; ++hh) t += __ldg(tsrc + ((long long)slot * tH + hh) * N + i - 1);
      t = t / (float)tH;
      const float c = __ldg(codec + (long long)slot * N + i - 1);
      float h = b1 + s * w1[0] + t * w1[1] + oh0 * w1[2] + oh1 * w1[3] + oh2 * w1[4] + oh3 * w1[5] + c * w1[6];
      h = lane < Hg ? quick_gelu(h) * w2 : 0.f;
      const float dlogit = warp_sum(h) + b2;
      int M = dlogit > 0.f ? 1 : 0;
      if (force) M = force[mrow + i - 1] ? 1 : 0;
      const int r = i - i0;
      if (lane == 0) {
        if (masks) masks[mrow + i - 1] = (uint8_t)M;
        if (scores) scores[mrow + i - 1] = dlogit;
        wmask[wrow + i] = (uint8_t)M;
        wprov[wrow + i] = (uint8_t)prov;
        r2_out[wrow + i] = M ? slot * T + i : -1;
        r2_res[wrow + i] = ((prov ? fut : past) < 0 ? slot : (prov ? fut : past)) * T + i;
        s_M[r] = (uint8_t)M;
        my_reused += M;
      }
      if (M) {
        // Eq. 8 into A row r: lane's float4 j covers columns 128 j + 4 lane .. +3, i.e. chunk
        // 2 j + (lane >= 16), 16-B granule (lane & 15) / 2 (XOR-swizzled by r & 7), half lane & 1
        const uint32_t rowb = su32(sA) + r * 128 + (lane & 1) * 8;
        const uint32_t gsw = (uint32_t)((((lane & 15) >> 1) ^ (r & 7)) << 4);
#pragma unroll
        for (int j = 0; j < VPL; ++j) {
          const float4 a = cv[j], b = prov ? fv[j] : pv[j];
          const uint32_t kc = 2 * j + (lane >> 4);
          asm volatile("st.shared.v2.b32 [%0], {%1, %2};" ::"r"(rowb + kc * (SR1_TOK * 128) + gsw),
                       "r"(pack_bf16x2(a.x - b.x, a.y - b.y)), "r"(pack_bf16x2(a.z - b.z, a.w - b.w))
                       : "memory");
        }
      }
    }
    if (lane == 0 && my_reused) atomicAdd(s_reused, my_reused);
    // generic-proxy shared stores -> visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  const int nreused = *s_reused;
  if (threadIdx.x == 0 && nreused) atomicAdd(cntR + w, nreused);   // integer: order-independent

  if (warp == 0) {
    if (lane == 0) {
      if (nreused) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        for (int c = 0; c < nk; ++c) {
          const int st = c % SR1_STG;
          bar_wait(&full[st], (c / SR1_STG) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint64_t ad = desc_sw128(sA + c * (SR1_TOK * 128));
          const uint64_t bd = desc_sw128(sW + st * SR1_CHUNK);
#pragma unroll
          for (int k = 0; k < 4; ++k) mma(tmem, ad + 2 * k, bd + 2 * k, (c | k) != 0);
          commit(&empty[st]);
          // refill the previous chunk's stage (its MMAs were issued one chunk ago)
          if (c >= 1 && c - 1 + SR1_STG < nk) {
            const int ps = (c - 1) % SR1_STG;
            bar_wait(&empty[ps], ((c - 1) / SR1_STG) & 1);
            bar_expect(&full[ps], SR1_CHUNK);
            tma2d(sW + ps * SR1_CHUNK, &tmW1, &full[ps], (c - 1 + SR1_STG) * 64, 0);
          }
        }
        commit(tfull);
      } else {
        // nothing to restore: drain the prefetched chunks before the CTA exits
        for (int c = 0; c < SR1_STG && c < nk; ++c) bar_wait(&full[c], 0);
      }
    }
    __syncwarp();
  }
  if (nreused) {
    // ---- epilogue: warp (q = warp & 3) reads TMEM lane quarter q (A rows 16 q .. 16 q + 15 on
    // lanes 0-15, M = 64 layout) columns 32 (warp >> 2) .. +31: hr = QuickGELU(acc + br1)
    const int q = warp & 3, cchunk = warp >> 2;
    bar_wait(tfull, 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    uint32_t v[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
          "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
          "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
          "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
        : "r"(tmem + (uint32_t(q * 32) << 16) + cchunk * 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    const int r = q * 16 + lane;
    const int i = i0 + r;
    if (lane < 16 && i <= i_end && s_M[r]) {
      uint4* o = reinterpret_cast<uint4*>(hr_full + (wrow + i) * SR1_HR + cchunk * 32);
      const float* bb = br1 + cchunk * 32;
#pragma unroll
      for (int g = 0; g < 4; ++g) {
        uint32_t u[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int k = 8 * g + 2 * e;
          u[e] = pack_bf16x2(gelu_tanh(__uint_as_float(v[k]) + __ldg(bb + k)),
                             gelu_tanh(__uint_as_float(v[k + 1]) + __ldg(bb + k + 1)));
        }
        o[g] = make_uint4(u[0], u[1], u[2], u[3]);
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(SR1_HR));
  }
}

}  // namespace

int score_r1_smem(int D) { return SR1_TOK * D * 2 + SR1_STG * SR1_CHUNK + 256; }

bool score_r1_supported(int D, int Hr) { return Hr == SR1_HR && (D == 1024 || D == 768); }

cudaError_t launch_score_r1(const float* X, int T, int D, int N, int L, int layer, int n_w, const int* wdesc,
                            const float* tsrc, int tH, const float* codec, const uint8_t* force, const float* gate,
                            int Hg, uint8_t* masks, float* scores, uint8_t* wmask, uint8_t* wprov, int* cntR,
                            const CUtensorMap* tmW1, const float* br1, bf16* hr_full, int* r2_out, int* r2_res,
                            cudaStream_t s) {
  if (n_w <= 0) return cudaSuccess;
  if (!score_r1_supported(D, SR1_HR)) return cudaErrorInvalidValue;
  cudaError_t e = cudaMemsetAsync(cntR, 0, (size_t)n_w * sizeof(int), s);
  if (e != cudaSuccess) return e;
  const int smem = score_r1_smem(D);
  dim3 grid(n_w, (N + SR1_TOK - 1) / SR1_TOK);
  const int4* wd = reinterpret_cast<const int4*>(wdesc);
#define RV_SR1(V)                                                                                                \
  do {                                                                                                           \
    static bool attr = false;                                                                                    \
    if (!attr) {                                                                                                 \
      e = cudaFuncSetAttribute(score_r1_kernel<V>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);           \
      if (e != cudaSuccess) return e;                                                                            \
      attr = true;                                                                                               \
    }                                                                                                            \
    score_r1_kernel<V><<<grid, SR1_THREADS, smem, s>>>(X, T, D, N, L, layer, wd, tsrc, tH, codec, force, gate,  \
                                                       Hg, masks, scores, wmask, wprov, cntR, *tmW1, br1,      \
                                                       hr_full, r2_out, r2_res);                                 \
  } while (0)
  if (D == 1024) RV_SR1(8);
  else RV_SR1(6);
#undef RV_SR1
  return cudaGetLastError();
}

}  // namespace rv
