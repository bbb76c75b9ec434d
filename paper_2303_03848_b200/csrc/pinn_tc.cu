// pinn_tc.cu — K4: the PINN coarse chain on the 5th-generation tensor cores (tcgen05), for wide
// networks (W ∈ {64, 128, 256}: 8×256 is 920 kflop per point-eval).
//
// Same chain as K3 (pinn_chain.cuh; Eq. 7): every point walks the local
// slices, g = G_n(U_n), Ĝ_n = g, U_{n+1} = g + D_n, δ partials.  A CTA of 128 threads owns a tile
// of 128 grid points (thread t ↔ point t ↔ TMEM lane t).  Per slice:
//   layer 0 (IN → W, K = 2 or 4: far too thin for an MMA) in fp32 on the FMA pipe; its fp16 (or
//     bf16) activations are stored to shared memory as the A operand [128 × W], K-major, in
//     8×8 core matrices (SWIZZLE_NONE: LBO = 128 B along K, SBO = 16·W B along M);
//   hidden layers W → W: one elected thread issues W/16 `tcgen05.mma.cta_group::1.kind::f16`
//     (M = 128, N = W, K = 16) with the layer's weights [W × W] (K-major, same core-matrix
//     layout, bulk-copied from L2 or resident) as B; accumulators in TMEM (W fp32 columns);
//     `tcgen05.commit` → mbarrier;
//   epilogue: each thread `tcgen05.ld`s its own TMEM lane 32 columns at a time, adds the bias,
//     applies the activation, and either writes the next A operand (fp16) or, after the last
//     hidden layer, accumulates the output layer W → 1 in fp32.
// fp16 operands, fp32 accumulation: the north_star tolerance for a tensor-core PINN is 1e-3.
#include <type_traits>
#include <stdlib.h>
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include "launch.h"
#include "pinn_chain.cuh"

namespace pr {

__device__ __forceinline__ uint32_t tc_smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
// PR_DEBUG_BOUNDS builds (test-only variant): index checks that trap on violation
#ifdef PR_DEBUG_BOUNDS
#define PR_CHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define PR_CHECK(cond) do { } while (0)
#endif

// UMMA shared-memory matrix descriptor (SWIZZLE_NONE, K-major): start >> 4 [0,14), LBO >> 4
// [16,30), SBO >> 4 [32,46), version 1 [46,48) (sm_100), base offset 0, layout type 0.
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)((sbo >> 4) & 0x3FFF) << 32) | (1ull << 46);
}
// instruction descriptor, kind::f16: D f32 [4,6) = 1; A, B format [7,10) [10,13) (0 f16, 1 bf16);
// K-major A and B; N >> 3 at [17,23); M >> 4 at [24,29)
template <bool BF16>
__host__ __device__ constexpr uint32_t umma_idesc(int M, int N) {
  return (1u << 4) | ((BF16 ? 1u : 0u) << 7) | ((BF16 ? 1u : 0u) << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void tc_mbar_init(uint64_t *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tc_mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "PR_TC_WAIT%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra PR_TC_WAIT%=;\n}\n" ::"r"(tc_smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(tc_smem_u32(bar)), "r"(bytes)
               : "memory");
  // bulk copies are limited to 2^20 bytes each and must be 16-B multiples (host guarantees)
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   tc_smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(tc_smem_u32(bar))
               : "memory");
}

template <class T>
__device__ __forceinline__ uint32_t pack2(float a, float b);  // two values, round to nearest
template <>
__device__ __forceinline__ uint32_t pack2<__half>(float a, float b) {
  const __half2 h = __floats2half2_rn(a, b);
  return *reinterpret_cast<const uint32_t *>(&h);
}
template <>
__device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float a, float b) {
  const __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<const uint32_t *>(&h);
}

// element offset of (row r, column c) in the K-major core-matrix layout of a [rows × K] operand
__host__ __device__ constexpr size_t cm_offset(int r, int c, int K) {
  return (size_t)(r / 8) * (K / 8) * 64 + (size_t)(c / 8) * 64 + (r % 8) * 8 + (c % 8);
}

// 32 TMEM columns of this thread's lane → registers
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
      "%15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

struct PinnTcArgs {
  PinnArgs g;              // chain; wts: fp32 W0[W][IN], b0[W], hidden biases [(LH−1)][W], Wo[W], bo
  const void *wh;          // hidden matrices in K-chunks (see pinn_tc_pack), pre-scaled
  int resident;            // 1: every chunk fits in shared memory (loaded once)
};

constexpr int kTcKC = 32;  // K columns per weight chunk

// Activation of the tensor-core epilogue.  Exact mode: the K3 tanh (ex2 + rcp, 2 MUFU ops, ~2e-7).
// FAST (bf16 mode, itself ~1e-2): tanh.approx.f32 (1 MUFU op, ~5e-4) on the un-prescaled argument.
template <int ACT, bool FAST>
__device__ __forceinline__ float act_tc(float zs) {
  if (ACT == 1 || !FAST) return act<ACT>(zs);
  float r;
  asm("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(zs * 0.34657359027997264f));  // zs / (2 log2 e)
  return r;
}

// SPLIT (PR_PREC_FP16_TC): operands split hi + lo in fp16, D = A_hi·B_hi + A_hi·B_lo + A_lo·B_hi —
// fp32-level accuracy (~2e-6 on 8×256 nets) at 3× the MMAs.  !SPLIT (PR_PREC_BF16_TC): one bf16 pass.
// H16 (with !SPLIT, PR_PREC_FP16X1_TC): one fp16 pass — fp16's 2^-11 unit roundoff is 8x finer than
// bf16's for the [-1,1] activations and O(1) weights, at bf16's speed (exact tanh in the epilogue).
// NT = 256: two threads per row of the tile (thread t: row t & 127, columns of half t >> 7), so
// the epilogue (TMEM loads, bias, tanh, operand stores) has two warps per sub-partition instead of
// one; the per-point chain state and outputs stay with the first half, the output layer's two
// column halves are added in a fixed order.
template <int IN, int W, int ACT, bool SPLIT, bool H16, int NT = 128>
__global__ void __launch_bounds__(NT) k_pinn_chain_tc(PinnTcArgs ta) {
  using T = typename std::conditional<SPLIT || H16, __half, __nv_bfloat16>::type;
  constexpr int TILE = 128;
  constexpr int NP = SPLIT ? 2 : 1;                         // hi (+ lo) planes
  constexpr uint32_t kIdesc = umma_idesc<!(SPLIT || H16)>(TILE, W);
  constexpr uint32_t kPlaneA = (uint32_t)TILE * W * 2;       // bytes of one A plane
  constexpr uint32_t kPlaneB = (uint32_t)W * kTcKC * 2;      // bytes of one chunk plane
  constexpr uint32_t kChunk = NP * kPlaneB;
  constexpr int NCH = W / kTcKC;                             // chunks per layer
  constexpr int HALVES = NT / 128, WH = W / HALVES;           // column halves per row
  static_assert(WH >= 32 && WH % 32 == 0, "a half holds whole 32-column TMEM loads");
  const PinnArgs &a = ta.g;
  extern __shared__ __align__(128) unsigned char tc_smem[];
  T *sA = reinterpret_cast<T *>(tc_smem);                    // NP planes [128 × W]
  unsigned char *sB = tc_smem + NP * kPlaneA;                // 1 chunk, or all (LH−1)·NCH chunks
  const int nchunks = ta.resident ? (a.LH - 1) * NCH : 2;  // resident, or two streaming buffers
  float *sP = reinterpret_cast<float *>(sB + (size_t)nchunks * kChunk);
  __shared__ __align__(8) uint64_t bar_mma, bar_w, bar_full[2], bar_free[2];
  __shared__ uint32_t s_tmem;
  __shared__ double red[64];
  __shared__ float s_y[HALVES > 1 ? 128 : 1], s_u[HALVES > 1 ? 128 : 1];
  const int t = threadIdx.x, w = t >> 5, r = t & 127, hh = t >> 7, col0 = hh * WH;
  for (int i = t; i < a.nfloats; i += blockDim.x) sP[i] = a.wts[i];
  if (t == 0) {
    tc_mbar_init(&bar_mma);
    tc_mbar_init(&bar_w);
    tc_mbar_init(&bar_full[0]);
    tc_mbar_init(&bar_full[1]);
    tc_mbar_init(&bar_free[0]);
    tc_mbar_init(&bar_free[1]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem_u32(&s_tmem)),
                 "r"((uint32_t)W));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  const uint32_t tlane = tmem + ((uint32_t)(32 * (w & 3)) << 16);  // this warp's TMEM lane quarter
  uint32_t ph_mma = 0, ph_w = 0;
  if (ta.resident && a.LH > 1) {  // every chunk loaded once (≤ 200 KB, one bulk copy)
    if (t == 0) tc_bulk_g2s(sB, ta.wh, (uint32_t)((a.LH - 1) * NCH) * kChunk, &bar_w);
    tc_mbar_wait(&bar_w, ph_w);
    ph_w ^= 1;
  }
  // Streaming: chunk g of the repeating sequence (layer-major, all slices) goes to buffer g & 1;
  // thread 0 loads chunk g+1 while the MMAs of chunk g run (after those of chunk g−1, which used
  // that buffer, have completed).
  const int nseq = (a.LH - 1) * NCH;
  unsigned g_next = 0;  // next chunk of the sequence to be consumed
  auto load_chunk = [&](unsigned g) {
    tc_bulk_g2s(sB + (size_t)(g & 1) * kChunk, (const unsigned char *)ta.wh + (size_t)(g % nseq) * kChunk, kChunk,
                &bar_full[g & 1]);
  };
  if (!ta.resident && a.LH > 1 && t == 0) load_chunk(0);
  const float *W0 = sP, *b0 = sP + W * IN;
  const float *Wo = sP + W * IN + W + (size_t)(a.LH - 1) * W;
  const float bo = Wo[W];
  // store 8 consecutive activations (fp32) of column block c0 as the A operand (hi, lo)
  auto store_a = [&](int c0, const float (&h)[8]) {
    const size_t off = cm_offset(r, c0, W);
    float lo[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float hi = SPLIT ? __half2float(__float2half_rn(h[q])) : 0.f;
      lo[q] = h[q] - hi;
    }
    *reinterpret_cast<uint4 *>(sA + off) =
        make_uint4(pack2<T>(h[0], h[1]), pack2<T>(h[2], h[3]), pack2<T>(h[4], h[5]), pack2<T>(h[6], h[7]));
    if (SPLIT)
      *reinterpret_cast<uint4 *>(sA + (size_t)TILE * W + off) = make_uint4(
          pack2<T>(lo[0], lo[1]), pack2<T>(lo[2], lo[3]), pack2<T>(lo[4], lo[5]), pack2<T>(lo[6], lo[7]));
  };

  const int b = blockIdx.y;
  const double Lb = a.Lb[b];
  const float gscale = (float)(Lb * (double)a.out_scale);
  const float invL = (float)(1.0 / Lb);
  const size_t sstride = (size_t)a.B * a.Mp;
  const int j = (blockIdx.x + a.cta0) * TILE + r;
  const bool ok = j < a.M;
  const double dS = Lb / (a.M + 1);
  const float s_over_L = (float)(((j + 1) * dS) / Lb);
  float *u0 = a.U + (size_t)a.ln0 * sstride + (size_t)b * a.Mp;
  float u = 0.f;
  if (a.Fcopy) {
    const float *f = a.Fcopy + (size_t)b * a.Mp;
    double num = 0.0, den = 0.0;
    if (ok) {
      u = f[j];
      if (hh == 0) {
        const double dd = (double)u - (double)u0[j];
        num = dd * dd;
        den = (double)u * u;
      }
    }
    __syncthreads();
    if (ok && hh == 0) u0[j] = u;
    if (a.partials) {
      cta_reduce2(num, den, red);
      if (t == 0) {
        double *pp = a.partials + (((size_t)a.ln0 * a.B + b) * a.nch + blockIdx.x + a.cta0) * 2;
        pp[0] = num;
        pp[1] = den;
      }
    }
  } else if (ok) {
    u = u0[j];
  }
  const uint32_t aHi = tc_smem_u32(sA), aLo = aHi + kPlaneA, bBase = tc_smem_u32(sB);
  const int ln_end = a.Gout ? a.ln0 + 1 : a.ln1;
#pragma unroll 1
  for (int ln = a.ln0; ln < ln_end; ++ln) {
    const int n = a.n_base + ln;
    const float tf = (float)((a.T - n * a.dT) / a.T), tt = (float)((a.T - (n + 1) * a.dT) / a.T);
    float x[IN];
    if (IN == 4) {
      x[0] = tf * a.cs0;
      x[1] = tt * a.cs1;
      x[2] = (u * invL) * a.cs2;
      x[3] = s_over_L * a.cs3;
    } else {
      x[0] = tt * a.cs0;
      x[IN - 1] = s_over_L * a.cs1;
    }
    // ---- layer 0 (fp32) → A operand
#pragma unroll 1
    for (int c0 = col0; c0 < col0 + WH; c0 += 8) {
      float h[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float z = b0[c0 + q];
#pragma unroll
        for (int i = 0; i < IN; ++i) z = fmaf(W0[(c0 + q) * IN + i], x[i], z);
        h[q] = act<ACT>(z);
      }
      store_a(c0, h);
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    float y = 0.f;
#pragma unroll 1
    for (int l = 1; l < a.LH; ++l) {
      // ---- D[128 × W] = A · W_l^T, chunk by chunk along K (one thread issues)
      if (t == 0) {
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
        for (int c = 0; c < NCH; ++c) {
          uint32_t bc;
          unsigned g = 0;
          if (ta.resident) {
            bc = bBase + (uint32_t)((l - 1) * NCH + c) * kChunk;
          } else {
            g = g_next++;
            tc_mbar_wait(&bar_full[g & 1], (g >> 1) & 1);
            bc = bBase + (g & 1) * kChunk;
          }
#pragma unroll
          for (int ks = 0; ks < kTcKC / 16; ++ks) {
            // A: K offset c·KC + 16·ks = core matrix (c·KC/8 + 2ks) along K; B chunk: core matrix 2ks
            const uint32_t ao = (uint32_t)(c * (kTcKC / 8) + 2 * ks) * 128, bo2 = (uint32_t)(2 * ks) * 128;
            const uint64_t dah = umma_desc(aHi + ao, 128, 16 * W), dbh = umma_desc(bc + bo2, 128, 16 * kTcKC);
            const uint32_t acc = (c > 0 || ks > 0) ? 1u : 0u;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                "l"(dah), "l"(dbh), "r"(kIdesc), "r"(acc));
            if (SPLIT) {
              const uint64_t dal = umma_desc(aLo + ao, 128, 16 * W);
              const uint64_t dbl = umma_desc(bc + kPlaneB + bo2, 128, 16 * kTcKC);
              asm volatile(
                  "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                  "l"(dah), "l"(dbl), "r"(kIdesc), "r"(1u));
              asm volatile(
                  "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                  "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
                  "l"(dal), "l"(dbh), "r"(kIdesc), "r"(1u));
            }
          }
          if (!ta.resident) {
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             tc_smem_u32(&bar_free[g & 1]))
                         : "memory");
            // buffer (g+1)&1 held chunk g−1: reload it with chunk g+1 once chunk g−1's MMAs completed
            if (g >= 1) tc_mbar_wait(&bar_free[(g - 1) & 1], ((g - 1) >> 1) & 1);
            load_chunk(g + 1);
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         tc_smem_u32(&bar_mma))
                     : "memory");
      }
      tc_mbar_wait(&bar_mma, ph_mma);
      ph_mma ^= 1;
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const float *bl = sP + W * IN + W + (size_t)(l - 1) * W;
      const bool last = l == a.LH - 1;
#pragma unroll 1
      for (int c0 = col0; c0 < col0 + WH; c0 += 32) {
        float v[32];
        tmem_ld32(tlane + (uint32_t)c0, v);
#pragma unroll
        for (int q = 0; q < 32; ++q) v[q] = act_tc<ACT, !SPLIT && !H16>(v[q] + bl[c0 + q]);
        if (last) {
#pragma unroll
          for (int q = 0; q < 32; ++q) y = fmaf(Wo[c0 + q], v[q], y);
        } else {
#pragma unroll
          for (int q = 0; q < 32; q += 8) {
            const float h[8] = {v[q], v[q + 1], v[q + 2], v[q + 3], v[q + 4], v[q + 5], v[q + 6], v[q + 7]};
            store_a(c0 + q, h);
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncthreads();
    }
    if (HALVES > 1) {  // the output layer's column halves, added in a fixed order
      if (hh == 1) s_y[r] = y;
      __syncthreads();
      if (hh == 0) y += s_y[r];
    }
    y += bo;
    const float g = gscale * y;
    if (a.Gout) {
      if (ok && hh == 0) a.Gout[(size_t)b * a.Mp + j] = g;
      break;
    }
    const size_t row = (size_t)ln * sstride + (size_t)b * a.Mp;
    float nv = 0.f;
    double num = 0.0, den = 0.0;
    if (ok && hh == 0) {
      nv = a.D ? g + a.D[row + j] : g;
      if (a.Gh) a.Gh[row + j] = g;
      if (a.partials) {
        const double dd = (double)nv - (double)a.U[row + sstride + j];
        num = dd * dd;
        den = (double)nv * nv;
      }
      a.U[row + sstride + j] = nv;
    }
    if (HALVES > 1) {  // the next slice's feature U_{n+1} for the second half
      if (hh == 0) s_u[r] = nv;
      __syncthreads();
      nv = s_u[r];
    }
    u = nv;
    if (a.partials) {
      cta_reduce2(num, den, red);
      if (t == 0) {
        double *pp = a.partials + (((size_t)(ln + 1) * a.B + b) * a.nch + blockIdx.x + a.cta0) * 2;
        pp[0] = num;
        pp[1] = den;
      }
    }
  }
  if (!ta.resident && a.LH > 1 && t == 0) tc_mbar_wait(&bar_full[g_next & 1], (g_next >> 1) & 1);  // last prefetch
  __syncthreads();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)W));
}

// ---------------------------------------------------------------- K4 ping-pong (bf16)
constexpr int kTc2Ring = 4;  // weight-chunk ring of the ping-pong kernel (one CTA per SM: a deeper ring)
// Two 128-point tiles per CTA and a warp-specialised schedule, so one tile's epilogue overlaps
// the other tile's MMAs: warpgroups 0 and 1 (threads 0-255) each own a tile (thread ↔ point ↔
// TMEM lane of its tile's W accumulator columns), warp 8 allocates TMEM (2W columns) and its lane 0
// issues every MMA and weight load.  Per hidden layer and tile: the issuer waits for the tile's A
// operand (bar_a[w], 128 arrivals after the tile's previous epilogue, which also means its TMEM
// columns have been read), issues the K-chunked MMAs and commits to bar_mma[w]; the warpgroup
// waits on bar_mma[w], runs the epilogue and arrives on bar_a[w].  With tile 0's epilogue running
// while tile 1's MMAs do (and vice versa) the tensor pipe no longer idles through every epilogue
// (k_pinn_chain_tc: 20-25 % tensor-pipe activity).  Weights stream through the same 2-chunk ring,
// in the order (slice, layer, tile, chunk) — each tile re-reads its layer's chunks — or stay
// resident when they fit.  Same arithmetic per point as k_pinn_chain_tc<…, SPLIT = false>.
__device__ __forceinline__ void tc_mbar_init_n(uint64_t *bar, uint32_t n) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc_smem_u32(bar)), "r"(n) : "memory");
}
__device__ __forceinline__ void tc_mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tc_smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 256;" ::: "memory"); }

// SPLIT (PR_PREC_FP16_TC, W ≤ 128): hi + lo fp16 planes for every A tile and weight chunk and the
// three MMAs of k_pinn_chain_tc<…, SPLIT> per K step — the accurate mode with the ping-pong overlap.
template <int IN, int W, int ACT, bool H16, bool SPLIT>
__global__ void __launch_bounds__(288, 1) k_pinn_chain_tc2(PinnTcArgs ta) {
  using T = typename std::conditional<H16 || SPLIT, __half, __nv_bfloat16>::type;
  constexpr int TILE = 128;
  constexpr int NP = SPLIT ? 2 : 1;  // operand planes (hi, lo)
  constexpr uint32_t kIdesc = umma_idesc<!(H16 || SPLIT)>(TILE, W);
  constexpr uint32_t kPlaneA = (uint32_t)TILE * W * 2;
  constexpr uint32_t kPlaneB = (uint32_t)W * kTcKC * 2;
  constexpr uint32_t kChunk = NP * kPlaneB;
  constexpr int NCH = W / kTcKC;
  const PinnArgs &a = ta.g;
  extern __shared__ __align__(128) unsigned char tc_smem[];
  T *sA = reinterpret_cast<T *>(tc_smem);  // [2 tiles][NP planes][128 × W]
  unsigned char *sB = tc_smem + 2 * NP * kPlaneA;
  constexpr int NB = kTc2Ring;  // streaming ring depth (NB − 1 chunks in flight)
  const int nchunks = ta.resident ? (a.LH - 1) * NCH : NB;
  float *sP = reinterpret_cast<float *>(sB + (size_t)nchunks * kChunk);
  __shared__ __align__(8) uint64_t bar_mma[2], bar_a[2], bar_w, bar_full[NB], bar_free[NB];
  __shared__ uint32_t s_tmem;
  __shared__ double red[16];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const int wg = t >> 7;  // 0, 1: epilogue warpgroups; 2: the issuer warp
  for (int i = t; i < a.nfloats; i += blockDim.x) sP[i] = a.wts[i];
  if (t == 0) {
    for (int i = 0; i < 2; ++i) {
      tc_mbar_init_n(&bar_mma[i], 1);
      tc_mbar_init_n(&bar_a[i], TILE);
    }
    for (int i = 0; i < NB; ++i) {
      tc_mbar_init_n(&bar_full[i], 1);
      tc_mbar_init_n(&bar_free[i], 1);
    }
    tc_mbar_init_n(&bar_w, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem_u32(&s_tmem)),
                 "r"((uint32_t)(2 * W)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  const int ln_end = a.Gout ? a.ln0 + 1 : a.ln1;
  const int nslices = ln_end - a.ln0;

  if (wg == 2) {  // ---------------- the issuer (lane 0 of warp 8)
    if (lane == 0 && a.LH > 1) {
      const uint32_t aBase = tc_smem_u32(sA), bBase = tc_smem_u32(sB);
      const int nseq = (a.LH - 1) * NCH;  // chunks of one tile's pass over the hidden layers
      auto wchunk = [&](unsigned g) {      // sequence g → weight chunk (order: slice, layer, tile, chunk)
        const unsigned q = g % (unsigned)(2 * nseq);
        return (q / (2 * NCH)) * NCH + q % NCH;
      };
      auto load_chunk = [&](unsigned g) {
        tc_bulk_g2s(sB + (size_t)(g % NB) * kChunk, (const unsigned char *)ta.wh + (size_t)wchunk(g) * kChunk, kChunk,
                    &bar_full[g % NB]);
      };
      if (ta.resident) {
        tc_bulk_g2s(sB, ta.wh, (uint32_t)((a.LH - 1) * NCH) * kChunk, &bar_w);
        tc_mbar_wait(&bar_w, 0);
      } else {
        for (unsigned d = 0; d + 1 < (unsigned)NB; ++d) load_chunk(d);
      }
      unsigned g = 0;
      uint32_t ph_a[2] = {0, 0};
#pragma unroll 1
      for (int sl = 0; sl < nslices; ++sl) {
#pragma unroll 1
        for (int l = 1; l < a.LH; ++l) {
#pragma unroll 1
          for (int w = 0; w < 2; ++w) {
            tc_mbar_wait(&bar_a[w], ph_a[w]);
            ph_a[w] ^= 1;
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t aw = aBase + (uint32_t)(w * NP) * kPlaneA, dw = tmem + (uint32_t)(w * W);
#pragma unroll 1
            for (int c = 0; c < NCH; ++c) {
              uint32_t bc;
              if (ta.resident) {
                bc = bBase + (uint32_t)((l - 1) * NCH + c) * kChunk;
              } else {
                tc_mbar_wait(&bar_full[g % NB], (g / NB) & 1);
                bc = bBase + (g % NB) * kChunk;
              }
#pragma unroll
              for (int ks = 0; ks < kTcKC / 16; ++ks) {
                const uint32_t ao = (uint32_t)(c * (kTcKC / 8) + 2 * ks) * 128, bo2 = (uint32_t)(2 * ks) * 128;
                const uint64_t da = umma_desc(aw + ao, 128, 16 * W), db = umma_desc(bc + bo2, 128, 16 * kTcKC);
                const uint32_t acc = (c > 0 || ks > 0) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dw),
                    "l"(da), "l"(db), "r"(kIdesc), "r"(acc));
                if (SPLIT) {  // + A_hi·B_lo + A_lo·B_hi
                  const uint64_t dbl = umma_desc(bc + kPlaneB + bo2, 128, 16 * kTcKC);
                  const uint64_t dal = umma_desc(aw + kPlaneA + ao, 128, 16 * W);
                  asm volatile(
                      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dw),
                      "l"(da), "l"(dbl), "r"(kIdesc), "r"(1u));
                  asm volatile(
                      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dw),
                      "l"(dal), "l"(db), "r"(kIdesc), "r"(1u));
                }
              }
              if (!ta.resident) {
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 tc_smem_u32(&bar_free[g % NB]))
                             : "memory");
                // the buffer of chunk g−1 takes chunk g + NB − 1 once chunk g−1's MMAs completed
                if (g >= 1) tc_mbar_wait(&bar_free[(g - 1) % NB], ((g - 1) / NB) & 1);
                load_chunk(g + NB - 1);
                ++g;
              }
            }
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             tc_smem_u32(&bar_mma[w]))
                         : "memory");
          }
        }
      }
      if (!ta.resident)  // the prefetches still in flight
        for (unsigned q = g; q + 1 < g + (unsigned)NB; ++q) tc_mbar_wait(&bar_full[q % NB], (q / NB) & 1);
    }
    __syncwarp();
  } else {  // ---------------- epilogue warpgroup wg: tile wg of this CTA
    const int tw = t & 127;
    T *sAw = sA + (size_t)(wg * NP) * TILE * W;
    const uint32_t tlane = tmem + (uint32_t)(wg * W) + ((uint32_t)(32 * (warp & 3)) << 16);
    const float *W0 = sP, *b0 = sP + W * IN;
    const float *Wo = sP + W * IN + W + (size_t)(a.LH - 1) * W;
    const float bo = Wo[W];
    auto store_a = [&](int c0, const float (&h)[8]) {
      const size_t off = cm_offset(tw, c0, W);
      *reinterpret_cast<uint4 *>(sAw + off) =
          make_uint4(pack2<T>(h[0], h[1]), pack2<T>(h[2], h[3]), pack2<T>(h[4], h[5]), pack2<T>(h[6], h[7]));
      if (SPLIT) {
        float lo[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) lo[q] = h[q] - __half2float(__float2half_rn(h[q]));
        *reinterpret_cast<uint4 *>(sAw + (size_t)TILE * W + off) = make_uint4(
            pack2<T>(lo[0], lo[1]), pack2<T>(lo[2], lo[3]), pack2<T>(lo[4], lo[5]), pack2<T>(lo[6], lo[7]));
      }
    };
    // fixed-order sum of (num, den) over the 256 epilogue threads; valid in thread 0
    auto reduce256 = [&](double &num, double &den) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, o);
        den += __shfl_xor_sync(0xffffffffu, den, o);
      }
      epi_sync();
      if (lane == 0) { red[2 * warp] = num; red[2 * warp + 1] = den; }
      epi_sync();
      if (t == 0) {
        num = 0.0; den = 0.0;
        for (int q = 0; q < 8; ++q) { num += red[2 * q]; den += red[2 * q + 1]; }
      }
    };
    const int b = blockIdx.y;
    const double Lb = a.Lb[b];
    const float gscale = (float)(Lb * (double)a.out_scale);
    const float invL = (float)(1.0 / Lb);
    const size_t sstride = (size_t)a.B * a.Mp;
    const int j = (blockIdx.x + a.cta0) * (2 * TILE) + wg * TILE + tw;
    const bool ok = j < a.M;
    const double dS = Lb / (a.M + 1);
    const float s_over_L = (float)(((j + 1) * dS) / Lb);
    float *u0 = a.U + (size_t)a.ln0 * sstride + (size_t)b * a.Mp;
    float u = 0.f;
    if (a.Fcopy) {
      const float *f = a.Fcopy + (size_t)b * a.Mp;
      double num = 0.0, den = 0.0;
      if (ok) {
        u = f[j];
        const double dd = (double)u - (double)u0[j];
        num = dd * dd;
        den = (double)u * u;
      }
      epi_sync();
      if (ok) u0[j] = u;
      if (a.partials) {
        reduce256(num, den);
        if (t == 0) {
          double *pp = a.partials + (((size_t)a.ln0 * a.B + b) * a.nch + blockIdx.x + a.cta0) * 2;
          pp[0] = num;
          pp[1] = den;
        }
      }
    } else if (ok) {
      u = u0[j];
    }
    uint32_t ph_m = 0;
#pragma unroll 1
    for (int ln = a.ln0; ln < ln_end; ++ln) {
      const int n = a.n_base + ln;
      const float tf = (float)((a.T - n * a.dT) / a.T), tt = (float)((a.T - (n + 1) * a.dT) / a.T);
      float x[IN];
      if (IN == 4) {
        x[0] = tf * a.cs0;
        x[1] = tt * a.cs1;
        x[2] = (u * invL) * a.cs2;
        x[3] = s_over_L * a.cs3;
      } else {
        x[0] = tt * a.cs0;
        x[IN - 1] = s_over_L * a.cs1;
      }
#pragma unroll 1
      for (int c0 = 0; c0 < W; c0 += 8) {
        float h[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float z = b0[c0 + q];
#pragma unroll
          for (int i = 0; i < IN; ++i) z = fmaf(W0[(c0 + q) * IN + i], x[i], z);
          h[q] = act<ACT>(z);
        }
        store_a(c0, h);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      tc_mbar_arrive(&bar_a[wg]);
      float y = 0.f;
#pragma unroll 1
      for (int l = 1; l < a.LH; ++l) {
        tc_mbar_wait(&bar_mma[wg], ph_m);
        ph_m ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const float *bl = sP + W * IN + W + (size_t)(l - 1) * W;
        const bool last = l == a.LH - 1;
#pragma unroll 1
        for (int c0 = 0; c0 < W; c0 += 32) {
          float v[32];
          tmem_ld32(tlane + (uint32_t)c0, v);
#pragma unroll
          for (int q = 0; q < 32; ++q) v[q] = act_tc<ACT, !H16 && !SPLIT>(v[q] + bl[c0 + q]);
          if (last) {
#pragma unroll
            for (int q = 0; q < 32; ++q) y = fmaf(Wo[c0 + q], v[q], y);
          } else {
#pragma unroll
            for (int q = 0; q < 32; q += 8) {
              const float h[8] = {v[q], v[q + 1], v[q + 2], v[q + 3], v[q + 4], v[q + 5], v[q + 6], v[q + 7]};
              store_a(c0 + q, h);
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
        if (!last) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          tc_mbar_arrive(&bar_a[wg]);
        }
      }
      y += bo;
      const float g = gscale * y;
      if (a.Gout) {
        if (ok) a.Gout[(size_t)b * a.Mp + j] = g;
        continue;  // (ln_end = ln0 + 1)
      }
      const size_t row = (size_t)ln * sstride + (size_t)b * a.Mp;
      float nv = 0.f;
      double num = 0.0, den = 0.0;
      if (ok) {
        nv = a.D ? g + a.D[row + j] : g;
        if (a.Gh) a.Gh[row + j] = g;
        if (a.partials) {
          const double dd = (double)nv - (double)a.U[row + sstride + j];
          num = dd * dd;
          den = (double)nv * nv;
        }
        a.U[row + sstride + j] = nv;
      }
      u = nv;
      if (a.partials) {
        reduce256(num, den);
        if (t == 0) {
          double *pp = a.partials + (((size_t)(ln + 1) * a.B + b) * a.nch + blockIdx.x + a.cta0) * 2;
          pp[0] = num;
          pp[1] = den;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 8) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)(2 * W)));
  }
}

// ---------------------------------------------------------------- K4 layer-pipelined one-tile kernel
// One 128-point tile per CTA and 288 threads: warpgroups 0 and 1 (threads 0-255) share the tile's
// epilogue — thread t owns row t & 127 and the 32-column blocks c ≡ t >> 7 (mod 2) of every layer —
// and warp 8's lane 0 issues every MMA and weight load.  The accumulators are double-buffered in
// TMEM (2W columns: layer l in half l & 1), so the MMAs of layer l+1 start as soon as the epilogue of
// layer l has written the first 64 columns of their A operand: per 64-column step st the epilogue
// threads arrive on bar_a[st] and the issuer runs that step's two K-chunks.  The tensor pipe and the
// epilogue's MUFU/FMA work overlap within one tile, where k_pinn_chain_tc serialises them (ncu: 56 %
// of its stall samples wait for the layer's MMAs).  One bar_a per step: a thread arrives on each
// once per layer, and its next arrival on the same barrier comes after bar_mma of the next layer,
// i.e. after the issuer consumed the phase (no run-ahead across phases).  Same per-point arithmetic
// as k_pinn_chain_tc except the K-chunk accumulation order, which is unchanged (chunks 0 … NCH−1).
template <int IN, int W, int ACT, bool SPLIT, bool H16, int NB>
__global__ void __launch_bounds__(288, W <= 128 ? 2 : 1) k_pinn_chain_tc3(PinnTcArgs ta) {
  using T = typename std::conditional<H16 || SPLIT, __half, __nv_bfloat16>::type;
  constexpr int TILE = 128;
  constexpr int NP = SPLIT ? 2 : 1;
  constexpr uint32_t kIdesc = umma_idesc<!(H16 || SPLIT)>(TILE, W);
  constexpr uint32_t kPlaneA = (uint32_t)TILE * W * 2;
  constexpr uint32_t kPlaneB = (uint32_t)W * kTcKC * 2;
  constexpr uint32_t kChunk = NP * kPlaneB;
  constexpr int NCH = W / kTcKC;   // K-chunks per layer
  constexpr int NSTEP = W / 64;    // 64-column steps per layer (two K-chunks each)
  static_assert(kTcKC == 32 && W % 64 == 0, "two 32-column K-chunks per step");
  const PinnArgs &a = ta.g;
  extern __shared__ __align__(128) unsigned char tc_smem[];
  T *sA = reinterpret_cast<T *>(tc_smem);  // NP planes [128 × W]
  unsigned char *sB = tc_smem + NP * kPlaneA;
  const int nchunks = ta.resident ? (a.LH - 1) * NCH : NB;
  float *sP = reinterpret_cast<float *>(sB + (size_t)nchunks * kChunk);
  __shared__ __align__(8) uint64_t bar_mma, bar_a[NSTEP], bar_w, bar_full[NB], bar_free[NB];
  __shared__ uint32_t s_tmem;
  __shared__ double red[16];
  __shared__ float s_y[128], s_u[128];
  const int t = threadIdx.x, warp = t >> 5, lane = t & 31;
  for (int i = t; i < a.nfloats; i += blockDim.x) sP[i] = a.wts[i];
  if (t == 0) {
    tc_mbar_init_n(&bar_mma, 1);
    for (int i = 0; i < NSTEP; ++i) tc_mbar_init_n(&bar_a[i], 256);
    for (int i = 0; i < NB; ++i) {
      tc_mbar_init_n(&bar_full[i], 1);
      tc_mbar_init_n(&bar_free[i], 1);
    }
    tc_mbar_init_n(&bar_w, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 8) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc_smem_u32(&s_tmem)),
                 "r"((uint32_t)(2 * W)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = s_tmem;
  const int ln_end = a.Gout ? a.ln0 + 1 : a.ln1;
  const int nslices = ln_end - a.ln0;

  if (warp == 8) {  // ---------------- the issuer (lane 0 of warp 8)
    if (lane == 0 && a.LH > 1) {
      const uint32_t aHi = tc_smem_u32(sA), aLo = aHi + kPlaneA, bBase = tc_smem_u32(sB);
      const int nseq = (a.LH - 1) * NCH;  // chunks of one pass over the hidden layers
      auto load_chunk = [&](unsigned g) {
        tc_bulk_g2s(sB + (size_t)(g % NB) * kChunk, (const unsigned char *)ta.wh + (size_t)(g % nseq) * kChunk,
                    kChunk, &bar_full[g % NB]);
      };
      if (ta.resident) {
        tc_bulk_g2s(sB, ta.wh, (uint32_t)((a.LH - 1) * NCH) * kChunk, &bar_w);
        tc_mbar_wait(&bar_w, 0);
      } else {
        for (unsigned d = 0; d + 1 < (unsigned)NB; ++d) load_chunk(d);
      }
      unsigned g = 0;
      uint32_t ph_a = 0;  // every bar_a[st] completes once per layer: one shared phase bit per layer
#pragma unroll 1
      for (int sl = 0; sl < nslices; ++sl) {
#pragma unroll 1
        for (int l = 1; l < a.LH; ++l) {
          const uint32_t dl = tmem + (uint32_t)((l & 1) * W);  // layer l's accumulator half
#pragma unroll 1
          for (int st = 0; st < NSTEP; ++st) {
            tc_mbar_wait(&bar_a[st], ph_a);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
            for (int cc = 0; cc < 2; ++cc) {
              const int c = 2 * st + cc;
              uint32_t bc;
              if (ta.resident) {
                PR_CHECK((l - 1) * NCH + c < nchunks);
                bc = bBase + (uint32_t)((l - 1) * NCH + c) * kChunk;
              } else {
                tc_mbar_wait(&bar_full[g % NB], (g / NB) & 1);
                bc = bBase + (g % NB) * kChunk;
              }
              PR_CHECK(c < NCH);
#pragma unroll
              for (int ks = 0; ks < kTcKC / 16; ++ks) {
                const uint32_t ao = (uint32_t)(c * (kTcKC / 8) + 2 * ks) * 128, bo2 = (uint32_t)(2 * ks) * 128;
                const uint64_t dah = umma_desc(aHi + ao, 128, 16 * W), dbh = umma_desc(bc + bo2, 128, 16 * kTcKC);
                const uint32_t acc = (c > 0 || ks > 0) ? 1u : 0u;
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dl),
                    "l"(dah), "l"(dbh), "r"(kIdesc), "r"(acc));
                if (SPLIT) {  // + A_hi·B_lo + A_lo·B_hi
                  const uint64_t dbl = umma_desc(bc + kPlaneB + bo2, 128, 16 * kTcKC);
                  const uint64_t dal = umma_desc(aLo + ao, 128, 16 * W);
                  asm volatile(
                      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dl),
                      "l"(dah), "l"(dbl), "r"(kIdesc), "r"(1u));
                  asm volatile(
                      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(dl),
                      "l"(dal), "l"(dbh), "r"(kIdesc), "r"(1u));
                }
              }
              if (!ta.resident) {
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                                 tc_smem_u32(&bar_free[g % NB]))
                             : "memory");
                // the buffer of chunk g−1 takes chunk g + NB − 1 once chunk g−1's MMAs completed
                if (g >= 1) tc_mbar_wait(&bar_free[(g - 1) % NB], ((g - 1) / NB) & 1);
                load_chunk(g + NB - 1);
                ++g;
              }
            }
          }
          ph_a ^= 1;
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                           tc_smem_u32(&bar_mma))
                       : "memory");
        }
      }
      if (!ta.resident)  // the prefetches still in flight
        for (unsigned q = g; q + 1 < g + (unsigned)NB; ++q) tc_mbar_wait(&bar_full[q % NB], (q / NB) & 1);
    }
    __syncwarp();
  } else {  // ---------------- the epilogue: row r, column blocks of parity hh
    const int r = t & 127, hh = t >> 7;
    const uint32_t tlane = tmem + ((uint32_t)(32 * (warp & 3)) << 16);
    const float *W0 = sP, *b0 = sP + W * IN;
    const float *Wo = sP + W * IN + W + (size_t)(a.LH - 1) * W;
    const float bo = Wo[W];
    auto store_a = [&](int c0, const float (&h)[8]) {
      const size_t off = cm_offset(r, c0, W);
      PR_CHECK(c0 + 8 <= W && off + 8 <= (size_t)TILE * W);
      *reinterpret_cast<uint4 *>(sA + off) =
          make_uint4(pack2<T>(h[0], h[1]), pack2<T>(h[2], h[3]), pack2<T>(h[4], h[5]), pack2<T>(h[6], h[7]));
      if (SPLIT) {
        float lo[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) lo[q] = h[q] - __half2float(__float2half_rn(h[q]));
        *reinterpret_cast<uint4 *>(sA + (size_t)TILE * W + off) = make_uint4(
            pack2<T>(lo[0], lo[1]), pack2<T>(lo[2], lo[3]), pack2<T>(lo[4], lo[5]), pack2<T>(lo[6], lo[7]));
      }
    };
    // fixed-order sum of (num, den) over the 256 epilogue threads; valid in thread 0
    auto reduce256 = [&](double &num, double &den) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, o);
        den += __shfl_xor_sync(0xffffffffu, den, o);
      }
      epi_sync();
      if (lane == 0) { red[2 * warp] = num; red[2 * warp + 1] = den; }
      epi_sync();
      if (t == 0) {
        num = 0.0; den = 0.0;
        for (int q = 0; q < 8; ++q) { num += red[2 * q]; den += red[2 * q + 1]; }
      }
    };
    const int b = blockIdx.y;
    const double Lb = a.Lb[b];
    const float gscale = (float)(Lb * (double)a.out_scale);
    const float invL = (float)(1.0 / Lb);
    const size_t sstride = (size_t)a.B * a.Mp;
    const int j = (blockIdx.x + a.cta0) * TILE + r;
    const bool ok = j < a.M;
    const double dS = Lb / (a.M + 1);
    const float s_over_L = (float)(((j + 1) * dS) / Lb);
    float *u0 = a.U + (size_t)a.ln0 * sstride + (size_t)b * a.Mp;
    float u = 0.f;
    if (a.Fcopy) {
      const float *f = a.Fcopy + (size_t)b * a.Mp;
      double num = 0.0, den = 0.0;
      if (ok) {
        u = f[j];
        if (hh == 0) {
          const double dd = (double)u - (double)u0[j];
          num = dd * dd;
          den = (double)u * u;
        }
      }
      epi_sync();
      if (ok && hh == 0) u0[j] = u;
      if (a.partials) {
        reduce256(num, den);
        if (t == 0) {
          double *pp = a.partials + (((size_t)a.ln0 * a.B + b) * a.nch + blockIdx.x + a.cta0) * 2;
          pp[0] = num;
          pp[1] = den;
        }
      }
    } else if (ok) {
      u = u0[j];
    }
    uint32_t ph_m = 0;
#pragma unroll 1
    for (int ln = a.ln0; ln < ln_end; ++ln) {
      const int n = a.n_base + ln;
      const float tf = (float)((a.T - n * a.dT) / a.T), tt = (float)((a.T - (n + 1) * a.dT) / a.T);
      float x[IN];
      if (IN == 4) {
        x[0] = tf * a.cs0;
        x[1] = tt * a.cs1;
        x[2] = (u * invL) * a.cs2;
        x[3] = s_over_L * a.cs3;
      } else {
        x[0] = tt * a.cs0;
        x[IN - 1] = s_over_L * a.cs1;
      }
      // layer 0 (fp32) → A, one 32-column block per step, then the step's arrival
#pragma unroll 1
      for (int st = 0; st < NSTEP; ++st) {
        const int cb = (2 * st + hh) * 32;
#pragma unroll 1
        for (int c0 = cb; c0 < cb + 32; c0 += 8) {
          float h[8];
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            float z = b0[c0 + q];
#pragma unroll
            for (int i = 0; i < IN; ++i) z = fmaf(W0[(c0 + q) * IN + i], x[i], z);
            h[q] = act<ACT>(z);
          }
          store_a(c0, h);
        }
        if (a.LH > 1) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          tc_mbar_arrive(&bar_a[st]);
        }
      }
      float y = 0.f;
#pragma unroll 1
      for (int l = 1; l < a.LH; ++l) {
        tc_mbar_wait(&bar_mma, ph_m);
        ph_m ^= 1;
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        const float *bl = sP + W * IN + W + (size_t)(l - 1) * W;
        const bool last = l == a.LH - 1;
        const uint32_t tl = tlane + (uint32_t)((l & 1) * W);
#pragma unroll 1
        for (int st = 0; st < NSTEP; ++st) {
          const int c0 = (2 * st + hh) * 32;
          float v[32];
          tmem_ld32(tl + (uint32_t)c0, v);
#pragma unroll
          for (int q = 0; q < 32; ++q) v[q] = act_tc<ACT, !H16 && !SPLIT>(v[q] + bl[c0 + q]);
          if (last) {
#pragma unroll
            for (int q = 0; q < 32; ++q) y = fmaf(Wo[c0 + q], v[q], y);
          } else {
#pragma unroll
            for (int q = 0; q < 32; q += 8) {
              const float h[8] = {v[q], v[q + 1], v[q + 2], v[q + 3], v[q + 4], v[q + 5], v[q + 6], v[q + 7]};
              store_a(c0 + q, h);
            }
            asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            tc_mbar_arrive(&bar_a[st]);
          }
        }
        if (last) asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      }
      // the output layer's column halves, added in a fixed order
      if (hh == 1) s_y[r] = y;
      epi_sync();
      if (hh == 0) y += s_y[r];
      y += bo;
      const float g = gscale * y;
      if (a.Gout) {
        if (ok && hh == 0) a.Gout[(size_t)b * a.Mp + j] = g;
        continue;  // (ln_end = ln0 + 1)
      }
      const size_t row = (size_t)ln * sstride + (size_t)b * a.Mp;
      float nv = 0.f;
      double num = 0.0, den = 0.0;
      if (ok && hh == 0) {
        nv = a.D ? g + a.D[row + j] : g;
        if (a.Gh) a.Gh[row + j] = g;
        if (a.partials) {
          const double dd = (double)nv - (double)a.U[row + sstride + j];
          num = dd * dd;
          den = (double)nv * nv;
        }
        a.U[row + sstride + j] = nv;
      }
      if (hh == 0) s_u[r] = nv;
      epi_sync();
      u = s_u[r];
      if (a.partials) {
        reduce256(num, den);
        if (t == 0) {
          double *pp = a.partials + (((size_t)(ln + 1) * a.B + b) * a.nch + blockIdx.x + a.cta0) * 2;
          pp[0] = num;
          pp[1] = den;
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 8) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"((uint32_t)(2 * W)));
  }
}

typedef void (*TcKernel)(PinnTcArgs);
template <bool SPLIT, bool H16>
static TcKernel tc_kernel_t(int IN, int W, int act, bool wide) {
  if (act != 0 && act != 1) return nullptr;
#define PR_TC_CASE(IN_, W_)                                                                        \
  if (IN == IN_ && W == W_)                                                                        \
    return wide ? (act ? k_pinn_chain_tc<IN_, W_, 1, SPLIT, H16, 256> : k_pinn_chain_tc<IN_, W_, 0, SPLIT, H16, 256>) \
                : (act ? k_pinn_chain_tc<IN_, W_, 1, SPLIT, H16> : k_pinn_chain_tc<IN_, W_, 0, SPLIT, H16>);
  PR_TC_CASE(4, 64) PR_TC_CASE(4, 128) PR_TC_CASE(4, 256) PR_TC_CASE(2, 64) PR_TC_CASE(2, 128) PR_TC_CASE(2, 256)
#undef PR_TC_CASE
  return nullptr;
}
// mode: kTcSplit16 (hi + lo fp16, 3 MMAs), kTcBF16 (one bf16 pass), kTcF16 (one fp16 pass)
// one-tile kernel width: 256 threads (two per tile row) unless PR_TC_WIDE=0 (A/B)
static bool tc_wide() {
  static const int v = getenv("PR_TC_WIDE") ? atoi(getenv("PR_TC_WIDE")) : 1;
  return v != 0;
}
static TcKernel tc_kernel(int IN, int W, int act, int mode) {
  const bool wide = tc_wide();
  return mode == kTcSplit16 ? tc_kernel_t<true, true>(IN, W, act, wide)
         : mode == kTcBF16  ? tc_kernel_t<false, false>(IN, W, act, wide)
                            : tc_kernel_t<false, true>(IN, W, act, wide);
}

bool pinn_tc_supported(int IN, int W, int act, int mode) { return tc_kernel(IN, W, act, mode) != nullptr; }

// shared memory: A planes [128 × W] + weight chunks (all if they fit, else one) + fp32 parameters
size_t pinn_tc_smem(int W, int LH, int nfloats, int mode, bool *resident) {
  const size_t np = mode == kTcSplit16 ? 2 : 1;
  const size_t a = np * 128 * W * 2, chunk = np * (size_t)W * kTcKC * 2, p = (size_t)nfloats * 4;
  const size_t all = (size_t)(LH - 1) * (W / kTcKC) * chunk;
  const size_t limit = 200 * 1024;
  if (a + all + p <= limit) {
    *resident = true;
    return a + all + p;
  }
  *resident = false;
  return a + 2 * chunk + p;
}

// host: hidden layer l's [W][W] (fp32, pre-scaled) → its W/64 K-chunks, each [hi plane][lo plane],
// a plane [W rows × 64 K] in the core-matrix K-major layout (SBO = 1024 B)
size_t pinn_tc_layer_elems(int W, int mode) { return (size_t)(mode == kTcSplit16 ? 2 : 1) * W * W; }
void pinn_tc_pack(const float *Wl, int W, int mode, uint16_t *out) {
  const int np = mode == kTcSplit16 ? 2 : 1;
  for (int c = 0; c < W / kTcKC; ++c) {
    uint16_t *hi = out + (size_t)c * np * W * kTcKC, *lo = hi + (size_t)W * kTcKC;
    for (int o = 0; o < W; ++o)
      for (int i = 0; i < kTcKC; ++i) {
        const float v = Wl[(size_t)o * W + c * kTcKC + i];
        const size_t off = cm_offset(o, i, kTcKC);
        if (mode == kTcBF16) {
          const __nv_bfloat16 h = __float2bfloat16_rn(v);
          hi[off] = *reinterpret_cast<const uint16_t *>(&h);
        } else if (mode == kTcF16) {
          const __half h = __float2half_rn(v);
          hi[off] = *reinterpret_cast<const uint16_t *>(&h);
        } else {
          const __half h = __float2half_rn(v);
          const __half l2 = __float2half_rn(v - __half2float(h));
          hi[off] = *reinterpret_cast<const uint16_t *>(&h);
          lo[off] = *reinterpret_cast<const uint16_t *>(&l2);
        }
      }
  }
}

// ping-pong kernel (bf16): two A planes; weights resident when they fit, else the 2-chunk ring
template <bool H16, bool SPLIT>
static TcKernel tc2_kernel_t(int IN, int W, int act) {
#define PR_TC2_CASE(IN_, W_) \
  if (IN == IN_ && W == W_) return act ? k_pinn_chain_tc2<IN_, W_, 1, H16, SPLIT> : k_pinn_chain_tc2<IN_, W_, 0, H16, SPLIT>;
  PR_TC2_CASE(4, 64) PR_TC2_CASE(4, 128) PR_TC2_CASE(4, 256) PR_TC2_CASE(2, 64) PR_TC2_CASE(2, 128) PR_TC2_CASE(2, 256)
#undef PR_TC2_CASE
  return nullptr;
}
static TcKernel tc2_kernel(int IN, int W, int act, int mode) {
  if (mode == kTcSplit16) return W <= 128 ? tc2_kernel_t<true, true>(IN, W, act) : nullptr;
  return mode == kTcF16 ? tc2_kernel_t<true, false>(IN, W, act) : tc2_kernel_t<false, false>(IN, W, act);
}
// the layer-pipelined split kernel (k_pinn_chain_tc3): ring depth NB ∈ {2, 4} by shared memory
template <int NB, bool SPLIT = true, bool H16 = true>
static TcKernel tc3_kernel_nb(int IN, int W, int act) {
#define PR_TC3_CASE(IN_, W_) \
  if (IN == IN_ && W == W_) return act ? k_pinn_chain_tc3<IN_, W_, 1, SPLIT, H16, NB> : k_pinn_chain_tc3<IN_, W_, 0, SPLIT, H16, NB>;
  PR_TC3_CASE(4, 64) PR_TC3_CASE(4, 128) PR_TC3_CASE(4, 256) PR_TC3_CASE(2, 64) PR_TC3_CASE(2, 128) PR_TC3_CASE(2, 256)
#undef PR_TC3_CASE
  return nullptr;
}
static size_t pinn_tc3_smem(int W, int LH, int nfloats, bool *resident, int *nb, int np = 2) {
  const size_t a = (size_t)np * 128 * W * 2, chunk = (size_t)np * W * kTcKC * 2, p = (size_t)nfloats * 4;
  const size_t all = (size_t)(LH - 1) * (W / kTcKC) * chunk;
  *resident = a + all + p <= 200 * 1024;
  *nb = (W > 128 && a + 4 * chunk + p <= 215 * 1024) ? 4 : 2;  // W ≤ 128: two CTAs per SM
  return *resident ? a + all + p : a + (size_t)*nb * chunk + p;
}
// PR_TC_PIPE (tuning): 1 (default) the layer-pipelined kernel for the split mode at W ≥ 128, 0 the
// one-tile kernel, 2 the layer-pipelined kernel for every mode at W ≥ 128 (the single-pass modes are
// slower with it: 8×256 fp16x1 55.5 → 65.5 ms, bf16 47.3 → 59.0 — their one-tile CTAs run two per SM)
static int tc3_env() {
  static const int on = getenv("PR_TC_PIPE") ? atoi(getenv("PR_TC_PIPE")) : 1;
  return on;
}
static size_t pinn_tc2_smem(int W, int LH, int nfloats, int np, bool *resident) {
  const size_t a = 2 * (size_t)np * 128 * W * 2, chunk = (size_t)np * W * kTcKC * 2, p = (size_t)nfloats * 4;
  const size_t all = (size_t)(LH - 1) * (W / kTcKC) * chunk;
  *resident = a + all + p <= 200 * 1024;
  return *resident ? a + all + p : a + kTc2Ring * chunk + p;
}
// PR_TC_PINGPONG (tuning): 1 (default) every mode, 0 none, 2 the single-pass modes only
static int pingpong_env() {
  static const int on = getenv("PR_TC_PINGPONG") ? atoi(getenv("PR_TC_PINGPONG")) : 1;
  return on;
}

// The ping-pong kernel for nets with enough MMA work per slice to hide the other tile's epilogue
// ((LH−1)·W² ≥ 24576: 4×64 measured 8.3 vs 9.3 G evals/s, 8×64 4.9 vs 3.5).  Single-pass modes:
// with resident weights only (with streamed weights — 8×256: 128 KB per layer and tile — both
// kernels are bound by the weight traffic from L2 and the one-tile kernel, two CTAs per SM, is as
// fast: 631 vs 610 M evals/s).  Split mode: W ≤ 128 (four A planes).
static bool tc_uses_pingpong(int W, int LH, int nfloats, int mode, bool *resident2, size_t *smem2) {
  const int on = pingpong_env();
  const bool split = mode == kTcSplit16;
  *smem2 = pinn_tc2_smem(W, LH, nfloats, split ? 2 : 1, resident2);
  if (on == 0 || (split && on == 2) || (long)(LH - 1) * W * W < 24576) return false;
  // split: measured at C5 (scripts/tc_split_ab.py) 8×64 resident 24.9 → 14.8 ms, 3×128 streamed
  // 17.6 → 13.8, but 4×128 / 8×128 streamed 17.8 → 18.6 / 36.6 → 38.0: resident, or ≤ 2 hidden MMA layers
  if (split) return W <= 128 && *smem2 <= 220 * 1024 && (*resident2 || LH <= 3);
  return *resident2;
}
int pinn_tc_points_per_cta(int W, int LH, int nfloats, int mode) {
  bool r2 = false;
  size_t sm2 = 0;
  return tc_uses_pingpong(W, LH, nfloats, mode, &r2, &sm2) ? 256 : 128;
}

// grid.x: CTAs along j in units of pinn_tc_points_per_cta points (from CTA a.cta0 on)
cudaError_t launch_pinn_tc(int IN, int W, int act, int mode, const PinnArgs &a, const void *wh, dim3 grid,
                           cudaStream_t s) {
  bool resident2 = false;
  size_t smem2 = 0;
  const bool pingpong = tc_uses_pingpong(W, a.LH, a.nfloats, mode, &resident2, &smem2);
  // The ping-pong kernel when the weights stay resident (its two A planes leave room for a short
  // ring only): with streamed weights (8×256: 128 KB per layer and tile) both kernels are bound by
  // the weight traffic from L2 and the one-tile kernel, two CTAs per SM, is as fast (measured
  // 631 vs 610 M evals/s); with resident weights the ping-pong kernel is 1.86× faster (4×128)
  // (and only for nets with enough MMA work per slice to hide the second tile's epilogue: 4×64
  // measured 8.3 vs 9.3 G evals/s, 8×64 4.9 vs 3.5)
  if (pingpong) {
    TcKernel k2 = tc2_kernel(IN, W, act, mode);
    if (!k2) return cudaErrorInvalidValue;
    const bool resident = resident2;
    const size_t smem = smem2;
    cudaError_t e = cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    PinnTcArgs ta;
    ta.g = a;
    ta.wh = wh;
    ta.resident = resident ? 1 : 0;
    k2<<<grid, 288, smem, s>>>(ta);  // two 128-point tiles per CTA
    return cudaGetLastError();
  }
  // the layer-pipelined split kernel for W ≥ 128 where the ping-pong kernel is not used
  // (scripts/tc_wide_ab.py, ms per C5 chain pair: 8×256 122.8 → 95.7, 4×256 56.8 → 44.2 with one
  // CTA per SM and a 4-deep weight ring; 4×128 16.8 → 15.1, 8×128 34.5 → 30.7 with two CTAs per SM
  // and a 2-deep ring — with one CTA per SM it was slower there: 21.8 / 45.1); W = 64: no gain
  // (6×64 16.7 → 16.6, one 64-column step per layer).  PR_TC_PIPE = 3 forces it for every width.
  if ((W >= 128 || tc3_env() == 3) && (mode == kTcSplit16 ? tc3_env() != 0 : tc3_env() == 2)) {
    bool resident3 = false;
    int nb = 2;
    const size_t smem3 = pinn_tc3_smem(W, a.LH, a.nfloats, &resident3, &nb, mode == kTcSplit16 ? 2 : 1);
    TcKernel k3 = mode == kTcSplit16 ? (nb == 4 ? tc3_kernel_nb<4>(IN, W, act) : tc3_kernel_nb<2>(IN, W, act))
                  : mode == kTcF16 ? (nb == 4 ? tc3_kernel_nb<4, false, true>(IN, W, act) : tc3_kernel_nb<2, false, true>(IN, W, act))
                                   : (nb == 4 ? tc3_kernel_nb<4, false, false>(IN, W, act) : tc3_kernel_nb<2, false, false>(IN, W, act));
    if (!k3) return cudaErrorInvalidValue;
    cudaError_t e = cudaFuncSetAttribute(k3, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem3);
    if (e != cudaSuccess) return e;
    PinnTcArgs ta;
    ta.g = a;
    ta.wh = wh;
    ta.resident = resident3 ? 1 : 0;
    k3<<<grid, 288, smem3, s>>>(ta);
    return cudaGetLastError();
  }
  TcKernel k = tc_kernel(IN, W, act, mode);
  if (!k) return cudaErrorInvalidValue;
  bool resident = false;
  const size_t smem = pinn_tc_smem(W, a.LH, a.nfloats, mode, &resident);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  PinnTcArgs ta;
  ta.g = a;
  ta.wh = wh;
  ta.resident = resident ? 1 : 0;
  k<<<grid, tc_wide() ? 256 : 128, smem, s>>>(ta);
  return cudaGetLastError();
}

}  // namespace pr
