// pinn_chain.cuh — K3: the PINN coarse propagator chained over slices, fp32 SIMT.
//
// G is pointwise in S (Fig. 2 caption P:217; reading Q6): each
// thread owns PTS grid points of one instance and walks them through the
// local slices n = ln0..ln1−1 with no inter-CTA synchronisation:
//     g = G_n(U_n);  Ĝ_n = g;  U_{n+1} = g + D_n      (Eq. 7)
// fusing the Parareal correction and the δ partial sums (reading Q13) into
// the epilogue.  The network (tanh per north_star) is evaluated
// with its weights in shared memory (uniform addresses → broadcast reads),
// activations in registers, hidden width W a template parameter so every
// layer is a fully unrolled W×W FMA block.
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef PR_PINN_CHAIN_ARGS
#define PR_PINN_CHAIN_ARGS
namespace pr {

struct PinnArgs {
  int M, Mp, B;
  const float *wts;        // packed: W0[W][IN], b0[W], {Wl[W][W], bl[W]} x (LH−1), Wo[W], bo
  int nfloats;             // packed length
  int LH;                  // hidden layers
  float cs0, cs1, cs2, cs3;  // in_scale
  float out_scale;
  double T, dT;
  int n_base;              // global slice index of local slice 0
  int ln0, ln1;            // chain over local slices [ln0, ln1)
  float *U;                // [Nloc+1][B][Mp]: reads U[ln0], writes U[ln+1]
  float *Gh;               // nullable [Nloc][B][Mp]
  const float *D;          // nullable [Nloc][B][Mp]
  const float *Fcopy;      // nullable [B][Mp]: first U[ln0] := Fcopy (+ δ partial)
  const double *Lb;        // [B]
  double *partials;        // nullable [(ln·B + b)·nch + chunk]·2
  int nch;
  float *Gout;             // test hook: non-null → write G_{ln0}(U[ln0]) only, no chain
  int cta0;                // first CTA (along j) of this launch: a j-chunk of the chain (NEXT-2 wavefront)
};

}  // namespace pr
#endif  // PR_PINN_CHAIN_ARGS

#if !defined(PR_ARGS_ONLY) && !defined(PR_PINN_CHAIN_IMPL)
#define PR_PINN_CHAIN_IMPL
namespace pr {
// tanh with the argument pre-scaled: the host multiplies the weights and biases of every
// tanh layer by 2·log2(e), so the layer produces z' = 2·log2(e)·z and
//     tanh(z) = 1 − 2 / (2^{z'} + 1)          (MUFU.EX2, FADD, MUFU.RCP, FFMA: 4 instructions)
// ex2.approx and rcp.approx are accurate to ~2^-22 relative, so |error| ≲ 2e-7 absolute; the
// limits are exact (2^{z'} → ∞ gives 1, → 0 gives −1).  This is NOT tanh.approx.f32 (2^-11).
__device__ __forceinline__ float tanh_prescaled(float zs) {
  float e, r;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(zs));
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(e + 1.0f));
  return fmaf(-2.0f, r, 1.0f);
}

template <int ACT>
__device__ __forceinline__ float act(float z) {
  if (ACT == 1) return fmaxf(z, 0.0f);
  return tanh_prescaled(z);
}

// fixed-order CTA reduction of (a, b); result valid in thread 0
__device__ __forceinline__ void cta_reduce2(double &a, double &b, double *red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  __syncthreads();
  if ((threadIdx.x & 31) == 0) { red[2 * w] = a; red[2 * w + 1] = b; }
  __syncthreads();
  if (threadIdx.x == 0) {
    a = 0.0; b = 0.0;
    for (int q = 0; q < nw; ++q) { a += red[2 * q]; b += red[2 * q + 1]; }
  }
}

template <int IN, int W, int ACT, int PTS>
__device__ __forceinline__ void mlp_eval(const float *__restrict__ sw, int LH, const float (&x)[PTS][IN],
                                         float (&y)[PTS]) {
  float h[PTS][W];
  // layer 0: IN → W
#pragma unroll
  for (int o = 0; o < W; ++o) {
    const float bo = sw[W * IN + o];
#pragma unroll
    for (int p = 0; p < PTS; ++p) {
      float z = bo;
#pragma unroll
      for (int i = 0; i < IN; ++i) z = fmaf(sw[o * IN + i], x[p][i], z);
      h[p][o] = act<ACT>(z);
    }
  }
  const float *lw = sw + W * IN + W;
#pragma unroll 1
  for (int l = 1; l < LH; ++l) {
    float z[PTS][W];
#pragma unroll
    for (int o = 0; o < W; ++o) {
      const float bo = lw[W * W + o];
#pragma unroll
      for (int p = 0; p < PTS; ++p) z[p][o] = bo;
#pragma unroll
      for (int i = 0; i < W; ++i) {
        const float wv = lw[o * W + i];
#pragma unroll
        for (int p = 0; p < PTS; ++p) z[p][o] = fmaf(wv, h[p][i], z[p][o]);
      }
    }
#pragma unroll
    for (int o = 0; o < W; ++o)
#pragma unroll
      for (int p = 0; p < PTS; ++p) h[p][o] = act<ACT>(z[p][o]);
    lw += W * W + W;
  }
  // output layer W → 1
  const float bout = lw[W];
#pragma unroll
  for (int p = 0; p < PTS; ++p) {
    float z = bout;
#pragma unroll
    for (int i = 0; i < W; ++i) z = fmaf(lw[i], h[p][i], z);
    y[p] = z;
  }
}

// The chain over slices shared by all network evaluators (`ev(x, y)` evaluates the MLP).
// G threads cooperate on one point when G > 1 (PTS = 1): all of them evaluate (the evaluator
// exchanges activations by shuffles), only the group's first thread stores and counts δ.
template <int IN, int PTS, class Eval, int G = 1>
__device__ __forceinline__ void pinn_chain_body(const PinnArgs &a, Eval ev) {
  static_assert(G == 1 || PTS == 1, "grouped evaluation handles one point per group");
  __shared__ double red[2 * 32];
  const int b = blockIdx.y;
  const double Lb = a.Lb[b];
  const float gscale = (float)(Lb * (double)a.out_scale);
  const float invL = (float)(1.0 / Lb);
  const size_t sstride = (size_t)a.B * a.Mp;
  // G > 1: 32/G groups per warp (lanes beyond them idle when G does not divide 32)
  constexpr int GPW = 32 / G;
  const int lane_ = threadIdx.x & 31;
  const bool active = (G == 1) || lane_ < GPW * G;
  const bool leader = (G == 1) || (active && lane_ % G == 0);
  const int cta = blockIdx.x + a.cta0;  // CTA index along j (δ partial slot)
  int j[PTS];
  bool ok[PTS];
  float s_over_L[PTS], u[PTS];
#pragma unroll
  for (int p = 0; p < PTS; ++p) {
    j[p] = (G == 1) ? cta * (blockDim.x * PTS) + p * blockDim.x + threadIdx.x
                    : cta * ((blockDim.x >> 5) * GPW) + (threadIdx.x >> 5) * GPW + lane_ / G;
    ok[p] = active && j[p] < a.M;
    // S_j / L_b = j dS / L_b with dS = L_b / (M+1)  (reading Q4, Q8)
    const double dS = Lb / (a.M + 1);
    s_over_L[p] = (float)(((j[p] + 1) * dS) / Lb);
  }
  float *u0 = a.U + (size_t)a.ln0 * sstride + (size_t)b * a.Mp;
  if (a.Fcopy) {
    const float *f = a.Fcopy + (size_t)b * a.Mp;
    double num = 0.0, den = 0.0;
#pragma unroll
    for (int p = 0; p < PTS; ++p) {
      u[p] = 0.f;
      if (ok[p]) {
        u[p] = f[j[p]];
        if (leader) {
          const double dd = (double)u[p] - (double)u0[j[p]];
          num += dd * dd;
          den += (double)u[p] * u[p];
        }
      }
    }
    __syncthreads();  // every thread of the CTA has read U[ln0] before it is overwritten
#pragma unroll
    for (int p = 0; p < PTS; ++p) {
      if (ok[p] && leader) u0[j[p]] = u[p];
    }
    if (a.partials) {
      cta_reduce2(num, den, red);
      if (threadIdx.x == 0) {
        double *pp = a.partials + (((size_t)a.ln0 * a.B + b) * a.nch + cta) * 2;
        pp[0] = num;
        pp[1] = den;
      }
    }
  } else {
#pragma unroll
    for (int p = 0; p < PTS; ++p) u[p] = ok[p] ? u0[j[p]] : 0.f;
  }
  const int ln_end = a.Gout ? a.ln0 + 1 : a.ln1;
  // δ partials: per-warp sums buffered per slice in shared memory and flushed (fixed order:
  // warps in index order) every kPartBuf slices, instead of a CTA barrier per slice
  constexpr int kPartBuf = 32;
  __shared__ double wpart[kPartBuf][4][2];
  const int wid = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
  auto flush = [&](int ln_first, int count) {
    __syncthreads();
    if (threadIdx.x < count) {
      double num = 0.0, den = 0.0;
      for (int q = 0; q < nwarp; ++q) { num += wpart[threadIdx.x][q][0]; den += wpart[threadIdx.x][q][1]; }
      double *pp = a.partials + (((size_t)(ln_first + threadIdx.x + 1) * a.B + b) * a.nch + cta) * 2;
      pp[0] = num;
      pp[1] = den;
    }
    __syncthreads();
  };
  // D_n and the old U_{n+1} are loaded one slice ahead (their latency hides behind the
  // previous slice's network); loads precede this kernel's stores to the same rows.
  float dn[PTS], uo[PTS];
  auto prefetch = [&](int ln, float (&d)[PTS], float (&o)[PTS]) {
    const size_t row = (size_t)ln * sstride + (size_t)b * a.Mp;
#pragma unroll
    for (int p = 0; p < PTS; ++p) {
      d[p] = (a.D && ok[p] && ln < ln_end) ? __ldcg(a.D + row + j[p]) : 0.f;
      o[p] = (a.partials && ok[p] && ln < ln_end) ? __ldcg(a.U + row + sstride + j[p]) : 0.f;
    }
  };
  prefetch(a.ln0, dn, uo);
#pragma unroll 1
  for (int ln = a.ln0; ln < ln_end; ++ln) {
    const int n = a.n_base + ln;
    // t_from/T, t_to/T (reading Q7): uniform per slice
    const float tf = (float)((a.T - n * a.dT) / a.T), tt = (float)((a.T - (n + 1) * a.dT) / a.T);
    const size_t row = (size_t)ln * sstride + (size_t)b * a.Mp;
    float dnx[PTS], uox[PTS];
    prefetch(ln + 1, dnx, uox);
    float x[PTS][IN], y[PTS];
#pragma unroll
    for (int p = 0; p < PTS; ++p) {
      if (IN == 4) {
        x[p][0] = tf * a.cs0;
        x[p][1] = tt * a.cs1;
        x[p][2] = (u[p] * invL) * a.cs2;  // V/L_b (reading Q8); fp32, ≤ 1.5 ulp
        x[p][3] = s_over_L[p] * a.cs3;
      } else {
        x[p][0] = tt * a.cs0;
        x[p][IN - 1] = s_over_L[p] * a.cs1;
      }
    }
    ev(x, y);
    if (a.Gout) {
#pragma unroll
      for (int p = 0; p < PTS; ++p)
        if (ok[p] && leader) a.Gout[(size_t)b * a.Mp + j[p]] = gscale * y[p];
      return;
    }
    float *un = a.U + row + sstride;
    double num = 0.0, den = 0.0;
#pragma unroll
    for (int p = 0; p < PTS; ++p) {
      const float g = gscale * y[p];
      float nv = 0.f;
      if (ok[p]) {
        nv = a.D ? g + dn[p] : g;
        if (leader) {
          if (a.Gh) a.Gh[row + j[p]] = g;
          if (a.partials) {
            const double dd = (double)nv - (double)uo[p];
            num += dd * dd;
            den += (double)nv * nv;
          }
          un[j[p]] = nv;
        }
      }
      u[p] = nv;
      dn[p] = dnx[p];
      uo[p] = uox[p];
    }
    if (a.partials) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, o);
        den += __shfl_xor_sync(0xffffffffu, den, o);
      }
      const int slot = (ln - a.ln0) % kPartBuf;
      if ((threadIdx.x & 31) == 0) { wpart[slot][wid][0] = num; wpart[slot][wid][1] = den; }
      if (slot == kPartBuf - 1 || ln == ln_end - 1) flush(ln - slot, slot + 1);
    }
  }
}


// Latency mode for few grid points: G threads share one point, thread q owning neurons
// [q·W/G, (q+1)·W/G) of every layer; after each layer the W activations are gathered with
// warp shuffles.  Per-thread work per slice drops ~G× (the coarse chain is serial in n, so at
// small M its length is what the GPU can hide least).  Weights in shared memory.
template <int IN, int W, int G, int ACT>
__device__ __forceinline__ float mlp_split(const float *__restrict__ sw, int LH, const float (&x)[IN]) {
  constexpr int NPT = W / G;
  const int lane = threadIdx.x & 31, q = lane % G, gbase = lane - q;
  float own[NPT], h[W];
#pragma unroll
  for (int k = 0; k < NPT; ++k) {
    const int o = q * NPT + k;
    float z = sw[W * IN + o];
#pragma unroll
    for (int i = 0; i < IN; ++i) z = fmaf(sw[o * IN + i], x[i], z);
    own[k] = act<ACT>(z);
  }
  const float *lw = sw + W * IN + W;
#pragma unroll 1
  for (int l = 1; l < LH; ++l) {
#pragma unroll
    for (int i = 0; i < W; ++i) h[i] = __shfl_sync(0xffffffffu, own[i % NPT], gbase + i / NPT);
    // the NPT neurons' sums advance together input by input (NPT independent FMA chains in flight;
    // each neuron's summation order is unchanged: bias, then inputs 0 … W−1)
    float z[NPT];
#pragma unroll
    for (int k = 0; k < NPT; ++k) z[k] = lw[W * W + q * NPT + k];
#pragma unroll
    for (int i = 0; i < W; ++i)
#pragma unroll
      for (int k = 0; k < NPT; ++k) z[k] = fmaf(lw[(q * NPT + k) * W + i], h[i], z[k]);
#pragma unroll
    for (int k = 0; k < NPT; ++k) own[k] = act<ACT>(z[k]);
    lw += W * W + W;
  }
  float y = 0.f;
#pragma unroll
  for (int k = 0; k < NPT; ++k) y = fmaf(lw[q * NPT + k], own[k], y);
  // butterfly sum, then every thread takes the group leader's value: a butterfly alone leaves
  // each lane its own rounding, so a thread's next-slice feature U/L_b could differ from the
  // stored U that another rank or schedule reads back
#pragma unroll
  for (int d = 1; d < G; d <<= 1) y += __shfl_xor_sync(0xffffffffu, y, d);
  y = __shfl_sync(0xffffffffu, y, gbase);
  return y + lw[W];
}

template <int IN, int W, int G, int ACT>
__global__ void __launch_bounds__(128) k_pinn_chain_split(PinnArgs a) {
  extern __shared__ float sw[];
  for (int i = threadIdx.x; i < a.nfloats; i += blockDim.x) sw[i] = a.wts[i];
  __syncthreads();
  static_assert(W % G == 0 && (G & (G - 1)) == 0, "G must be a power of two dividing W");
  auto ev = [&](const float (&x)[1][IN], float (&y)[1]) { y[0] = mlp_split<IN, W, G, ACT>(sw, a.LH, x[0]); };
  pinn_chain_body<IN, 1, decltype(ev), G>(a, ev);
}

// Latency mode for wider nets (the paper's 10×50): G threads per point (GPW = 32/G groups
// per warp; W % G == 0), thread q owning the NPT = W/G consecutive neurons q·NPT … of every
// layer.  After each layer the group's activations are exchanged through a per-group row of
// shared memory (one store per owned neuron, W/4 broadcast float4 loads) instead of W shuffles;
// weights are read from global memory through L1, the hidden matrices host-permuted to
// [i][q][k] so a group's loads for input i are one coalesced segment (row-major rows would put
// each lane on its own cache line: G lines per load), so the kernel needs no dynamic shared
// memory and many chain CTAs can be co-resident (pipe.cu).
// Two accumulators per neuron halve the FMA dependency chain.  The output layer's G partial
// sums are added in lane order (deterministic).
template <int W>
struct GroupRow {
  static constexpr int kPad = (W + 3) / 4 * 4;  // floats per group row (16-B aligned)
};
template <int IN, int W, int G, int ACT>
__device__ __forceinline__ float mlp_group(const float *__restrict__ gw, int LH, const float (&x)[IN],
                                           float *__restrict__ row, bool active) {
  static_assert(W % G == 0 && G <= 32, "G must divide W");
  constexpr int NPT = W / G;
  constexpr int KP = GroupRow<W>::kPad;
  const int q = (threadIdx.x & 31) % G;
  float own[NPT];
#pragma unroll
  for (int k = 0; k < NPT; ++k) {
    const int o = q * NPT + k;
    float z = __ldg(gw + W * IN + o);
#pragma unroll
    for (int i = 0; i < IN; ++i) z = fmaf(__ldg(gw + o * IN + i), x[i], z);
    own[k] = act<ACT>(z);
  }
  const float *lw = gw + W * IN + W;
#pragma unroll 1
  for (int l = 1; l < LH; ++l) {
    __syncwarp();
    if (active) {
#pragma unroll
      for (int k = 0; k < NPT; ++k) row[q * NPT + k] = own[k];
    }
    __syncwarp();
    float h[KP];
#pragma unroll
    for (int i = 0; i < KP; i += 4) {
      const float4 v = *reinterpret_cast<const float4 *>(row + i);
      h[i] = v.x; h[i + 1] = v.y; h[i + 2] = v.z; h[i + 3] = v.w;
    }
    // hidden matrix in the group order [i][q][k] (host-packed): for each input i the group's
    // lanes read consecutive addresses (coalesced), NPT weights per lane
    float z0[NPT], z1[NPT];
#pragma unroll
    for (int k = 0; k < NPT; ++k) {
      z0[k] = __ldg(lw + W * W + q * NPT + k);
      z1[k] = 0.f;
    }
    const float *wq = lw + q * NPT;
#pragma unroll
    for (int i = 0; i < W; ++i) {
      float wv[NPT];
      if constexpr (NPT % 4 == 0) {
#pragma unroll
        for (int k = 0; k < NPT; k += 4) {
          const float4 t = __ldg(reinterpret_cast<const float4 *>(wq + i * W + k));
          wv[k] = t.x; wv[k + 1] = t.y; wv[k + 2] = t.z; wv[k + 3] = t.w;
        }
      } else if constexpr (NPT % 2 == 0) {
#pragma unroll
        for (int k = 0; k < NPT; k += 2) {
          const float2 t = __ldg(reinterpret_cast<const float2 *>(wq + i * W + k));
          wv[k] = t.x; wv[k + 1] = t.y;
        }
      } else {
#pragma unroll
        for (int k = 0; k < NPT; ++k) wv[k] = __ldg(wq + i * W + k);
      }
#pragma unroll
      for (int k = 0; k < NPT; ++k) {
        if (i & 1) z1[k] = fmaf(wv[k], h[i], z1[k]);
        else z0[k] = fmaf(wv[k], h[i], z0[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < NPT; ++k) own[k] = act<ACT>(z0[k] + z1[k]);
    lw += W * W + W;
  }
  float y = 0.f;
#pragma unroll
  for (int k = 0; k < NPT; ++k) y = fmaf(__ldg(lw + q * NPT + k), own[k], y);
  __syncwarp();
  if (active) row[q] = y;
  __syncwarp();
  float s = __ldg(lw + W);
#pragma unroll
  for (int r = 0; r < G; ++r) s += row[r];
  return s;
}

template <int IN, int W, int G, int ACT>
__global__ void __launch_bounds__(128) k_pinn_chain_group(PinnArgs a) {
  constexpr int GPW = 32 / G, KP = GroupRow<W>::kPad;
  __shared__ __align__(16) float xrow[4][GPW][KP];
  const int lane = threadIdx.x & 31;
  const int grp = lane / G < GPW ? lane / G : GPW - 1;  // idle lanes read (never write) the last row
  const bool active = lane < GPW * G;
  float *row = &xrow[threadIdx.x >> 5][grp][0];
  auto ev = [&](const float (&x)[1][IN], float (&y)[1]) { y[0] = mlp_group<IN, W, G, ACT>(a.wts, a.LH, x[0], row, active); };
  pinn_chain_body<IN, 1, decltype(ev), G>(a, ev);
}

template <int IN, int W, int ACT, int PTS>
__global__ void __launch_bounds__(128) k_pinn_chain(PinnArgs a) {
  extern __shared__ float sw[];
  for (int i = threadIdx.x; i < a.nfloats; i += blockDim.x) sw[i] = a.wts[i];
  __syncthreads();
  pinn_chain_body<IN, PTS>(a, [&](const float (&x)[PTS][IN], float (&y)[PTS]) {
    mlp_eval<IN, W, ACT, PTS>(sw, a.LH, x, y);
  });
}

// Small networks: every weight is a kernel parameter (constant bank), so each FFMA takes its
// weight as a c[0x0][imm] operand -- no shared-memory loads and only two register reads per
// FMA.  Layers fully unrolled (LH is a template parameter).
template <int IN, int W, int LH>
struct ParamNet {
  static constexpr int kFloats = W * IN + W + (LH - 1) * (W * W + W) + W + 1;
  float w[kFloats];
};

template <int IN, int W, int LH, int ACT>
__device__ __forceinline__ float mlp_param(const ParamNet<IN, W, LH> &P, const float (&x)[IN]) {
  float h[W];
#pragma unroll
  for (int o = 0; o < W; ++o) {
    float z = P.w[W * IN + o];
#pragma unroll
    for (int i = 0; i < IN; ++i) z = fmaf(P.w[o * IN + i], x[i], z);
    h[o] = act<ACT>(z);
  }
#pragma unroll
  for (int l = 1; l < LH; ++l) {
    constexpr int base0 = W * IN + W;
    const int base = base0 + (l - 1) * (W * W + W);
    float z[W];
#pragma unroll
    for (int o = 0; o < W; ++o) {
      z[o] = P.w[base + W * W + o];
#pragma unroll
      for (int i = 0; i < W; ++i) z[o] = fmaf(P.w[base + o * W + i], h[i], z[o]);
    }
#pragma unroll
    for (int o = 0; o < W; ++o) h[o] = act<ACT>(z[o]);
  }
  constexpr int ob = W * IN + W + (LH - 1) * (W * W + W);
  float y = P.w[ob + W];
#pragma unroll
  for (int i = 0; i < W; ++i) y = fmaf(P.w[ob + i], h[i], y);
  return y;
}

template <int IN, int W, int LH, int ACT>
__global__ void __launch_bounds__(128) k_pinn_chain_param(PinnArgs a, const __grid_constant__ ParamNet<IN, W, LH> P) {
  pinn_chain_body<IN, 1>(a, [&](const float (&x)[1][IN], float (&y)[1]) { y[0] = mlp_param<IN, W, LH, ACT>(P, x[0]); });
}

}  // namespace pr
#endif  // PR_PINN_CHAIN_IMPL
