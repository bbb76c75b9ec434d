// pinn_train.cu — GPU training of the PINN coarse propagator (
// PAPER.md §3.3; C ABI in include/pinn_train.h).
//
// One Adam step is two kernels:
//  k_train_grad  G threads per collocation point of the step's batch (its epoch's shuffle of
//                each set), each owning W/G neurons of every layer: forward jets (Ṽ, Ṽ_t,
//                Ṽ_S, Ṽ_SS) through the net with the weights in shared memory and the layer
//                activations exchanged through a shared row per point, the point's loss term
//                (Eqs. 12-14) and its adjoint, then reverse accumulation layer by layer.
//                Each layer's weight gradient Σ_points Σ_jet z̄_c ⊗ h_c is contracted per CTA from
//                the points' shared rows and written as the CTA's partial (no atomics: fixed
//                summation order, run-to-run bitwise).  The forward pre-activation jets are
//                stashed in shared memory for the reverse pass.
//  k_adam        32 parameters per CTA: the fp64 sum of the CTA partials (fixed tree), Adam
//                (P:210); the last CTA (completion ticket) writes the batch's loss terms into the
//                history and advances the step counter.
// One epoch (batches × the two kernels) is captured as a CUDA graph and replayed; both kernels
// read the step counter from device memory, so the same graph serves every epoch.
#include "../../include/pinn_train.h"

#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace {

constexpr int kTPB = 128;          // threads per CTA of the gradient kernel
constexpr int kAdamThreads = 1024;
constexpr int kActTanh = PR_ACT_TANH;

struct Market {
  float K, sig, r, T, L;
  int asym;  // 1: V(t, L) = L − K e^{−r(T−t)} (reading Q3), 0: V(t, L) = 0
};

struct GradArgs {
  const float *theta;
  int np, LH;
  float *gpart;     // [nblk][np] CTA partial gradients
  double *lpart;    // [nblk][3] CTA partial loss terms
  const float *t_f, *S_f, *t_b, *S_b, *S_e;
  int n_f, n_b, n_e, batches;
  const long long *d_step;  // the global step counter (device)
  long long step_override;  // ≥ 0: train on this step's batch instead of *d_step's
  int full;                 // 1: every point of every set, unshuffled (the full-set loss)
  unsigned long long seed;
  Market mk;
};

// ---------------------------------------------------------------- the shuffle
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// position i of the epoch's order of a set of n points → the point's index
__device__ long long perm_at(unsigned long long seed, long long epoch, int which, long long n, long long i) {
  if (n <= 1) return 0;
  int b = 64 - __clzll((long long)(n - 1));
  if (b < 1) b = 1;
  const unsigned long long mask = b >= 64 ? ~0ull : ((1ull << b) - 1ull);
  const int s = b / 2 > 1 ? b / 2 : 1;
  const unsigned long long base = splitmix64(seed ^ splitmix64((unsigned long long)(4 * epoch + which)));
  unsigned long long k[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) k[r] = splitmix64(base + (unsigned long long)r);
  unsigned long long x = (unsigned long long)i;
  do {
#pragma unroll
    for (int r = 0; r < 4; ++r) {
      x = (x * (k[r] | 1ull)) & mask;
      x = (x + (k[r] >> 40)) & mask;
      x ^= x >> s;
    }
  } while (x >= (unsigned long long)n);
  return (long long)x;
}

// σ, σ', σ'', σ''' from the activation's output h (tanh: σ' = 1 − h², σ'' = −2hσ',
// σ''' = σ'(6h² − 2); ReLU: σ' = [h > 0], σ'' = σ''' = 0)
template <int ACT>
__device__ __forceinline__ void act_derivs(float h, float &s1, float &s2, float &s3) {
  if (ACT == kActTanh) {
    s1 = fmaf(-h, h, 1.0f);
    s2 = -2.0f * h * s1;
    s3 = s1 * fmaf(6.0f * h, h, -2.0f);
  } else {
    s1 = h > 0.0f ? 1.0f : 0.0f;
    s2 = 0.0f;
    s3 = 0.0f;
  }
}
template <int ACT>
__device__ __forceinline__ float act(float z) {
  return ACT == kActTanh ? tanhf(z) : fmaxf(z, 0.0f);
}

__device__ __forceinline__ double block_sum3(double v, int c, double *sl) {
  // fixed-order CTA sum of one fp64 value per thread (for component c of 3); result on thread 0
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) sl[w * 3 + c] = v;
  return v;
}

// Geometry of the gradient kernel: G threads per collocation point, each owning NPT = W/G neurons
// of every layer (groups of G consecutive lanes; 32/G groups per warp, lanes beyond them idle).
template <int W> struct TrainGeom;
template <> struct TrainGeom<8> { static constexpr int G = 2; };
template <> struct TrainGeom<16> { static constexpr int G = 4; };
template <> struct TrainGeom<20> { static constexpr int G = 4; };
template <> struct TrainGeom<32> { static constexpr int G = 4; };
template <> struct TrainGeom<50> { static constexpr int G = 10; };
template <> struct TrainGeom<64> { static constexpr int G = 8; };
template <int W>
struct TG {
  static constexpr int G = TrainGeom<W>::G, NPT = W / G, GPW = 32 / G;
  static constexpr int PP = (kTPB / 32) * GPW;  // collocation points per CTA
  static constexpr int RS = 4 * W + 1;          // shared row stride of one point's 4 jet rows (odd: no conflicts)
};
// shared memory of the gradient kernel (floats after the 128-B loss scratch): weights, the
// forward stash [LH][PP][4W], two exchange rows [PP][RS] (z̄ / activations, and h_prev jets), ȳ [PP][4]
template <int W>
size_t train_smem_floats(int np, int LH) {
  using T = TG<W>;
  return (size_t)np + (size_t)LH * T::PP * 4 * W + 2 * (size_t)T::PP * T::RS + 4 * T::PP + 4;
}

// Gradient of the batch loss (GRAD) or the loss terms only (!GRAD) over this CTA's PP points.
//  forward   lane q of point p computes the jets (z, z_t, z_S, z_SS) of its NPT neurons of each
//            layer from the whole previous layer (read from the point's shared row), stashes
//            (h, z_t, z_S, z_SS) in shared memory and writes its activation jets back to the row;
//  loss      the group's output-layer partials are summed by the leader in lane order; it forms the
//            loss term and the output adjoints (Eqs. 12-14, Eq. 11) and shares them;
//  backward  per layer, top down: z-bar of its own neurons from h-bar (jet chain rules, up to the
//            third derivative of the activation), written to the shared row; the CTA contracts the
//            layer's weight gradient sum_p sum_c zbar_c (x) h_c over its points (fixed order); h-bar
//            of the layer below for its own neurons = sum_i W_ij zbar_i.
template <int W, int ACT, bool GRAD>
__global__ void __launch_bounds__(kTPB) k_train_grad(GradArgs a) {
  using T = TG<W>;
  constexpr int G = T::G, NPT = T::NPT, GPW = T::GPW, PP = T::PP, RS = T::RS;
  extern __shared__ __align__(16) unsigned char smraw[];
  double *sl = reinterpret_cast<double *>(smraw);  // [kTPB/32][3]
  float *sw = reinterpret_cast<float *>(smraw + 128);
  const int LH = a.LH;
  float *sst = sw + a.np;                           // [LH][PP][4W]
  float *sZ = sst + (size_t)LH * PP * 4 * W;        // [PP][RS]
  float *sH = sZ + PP * RS;                         // [PP][RS]
  float *sY = sH + PP * RS;                         // [PP][4]
  const int tid = threadIdx.x, blk = blockIdx.x, lane = tid & 31;
  for (int i = tid; i < a.np; i += kTPB) sw[i] = a.theta[i];
  const int grp = lane / G, q = lane - (lane / G) * G;
  const bool act_lane = grp < GPW;
  const int pidx = (tid >> 5) * GPW + (act_lane ? grp : 0);  // (idle lanes shadow group 0)
  const int i0 = q * NPT;                                     // this lane's first neuron

  // ---- the point (batch part ib of each set's shuffle)
  const long long step = a.step_override >= 0 ? a.step_override : *a.d_step;
  const long long epoch = step / a.batches;
  const int ib = (int)(step - epoch * a.batches);
  long long lo0, lo1, lo2, c0, c1, c2;
  {
    const long long n0 = a.n_f, n1 = a.n_b, n2 = a.n_e;
    lo0 = a.full ? 0 : ib * n0 / a.batches, c0 = a.full ? n0 : (ib + 1) * n0 / a.batches - lo0;
    lo1 = a.full ? 0 : ib * n1 / a.batches, c1 = a.full ? n1 : (ib + 1) * n1 / a.batches - lo1;
    lo2 = a.full ? 0 : ib * n2 / a.batches, c2 = a.full ? n2 : (ib + 1) * n2 / a.batches - lo2;
  }
  const long long gpt = (long long)blk * PP + pidx;
  int kind = -1;
  if (act_lane) {
    if (gpt < c0) kind = 0;
    else if (gpt < c0 + c1) kind = 1;
    else if (gpt < c0 + c1 + c2) kind = 2;
  }
  const Market mk = a.mk;
  float t = 0.0f, S = 0.0f;
  if (kind == 0) {
    const long long idx = a.full ? gpt : perm_at(a.seed, epoch, 0, a.n_f, lo0 + gpt);
    t = a.t_f[idx], S = a.S_f[idx];
  } else if (kind == 1) {
    const long long pos = gpt - c0, idx = a.full ? pos : perm_at(a.seed, epoch, 1, a.n_b, lo1 + pos);
    t = a.t_b[idx], S = a.S_b[idx];
  } else if (kind == 2) {
    const long long pos = gpt - c0 - c1, idx = a.full ? pos : perm_at(a.seed, epoch, 2, a.n_e, lo2 + pos);
    t = mk.T, S = a.S_e[idx];
  }
  __syncthreads();

  // ---- forward jets; features x = (t/T, S/L): x_t = (1/T, 0), x_S = (0, 1/L)
  const float iT = 1.0f / mk.T, iL = 1.0f / mk.L;
  const float x0 = t * iT, x1 = S * iL;
  float *rowZ = sZ + pidx * RS, *rowH = sH + pidx * RS;
  {
    const float *W0 = sw, *b0 = sw + 2 * W;
    float *st = sst + (size_t)pidx * 4 * W;
#pragma unroll
    for (int ii = 0; ii < NPT; ++ii) {
      const int i = i0 + ii;
      const float z = fmaf(W0[2 * i], x0, fmaf(W0[2 * i + 1], x1, b0[i]));
      const float zt = W0[2 * i] * iT, zS = W0[2 * i + 1] * iL;
      const float hv = act<ACT>(z);
      float s1, s2, s3;
      act_derivs<ACT>(hv, s1, s2, s3);
      if (act_lane) {
        if (GRAD) st[i] = hv, st[W + i] = zt, st[2 * W + i] = zS, st[3 * W + i] = 0.0f;
        rowZ[i] = hv, rowZ[W + i] = s1 * zt, rowZ[2 * W + i] = s1 * zS, rowZ[3 * W + i] = s2 * zS * zS;
      }
    }
  }
  __syncthreads();
  int off = 3 * W;
  for (int l = 1; l < LH; ++l) {
    const float *Wl = sw + off, *bl = sw + off + W * W;
    float z[NPT], zt[NPT], zS[NPT], zSS[NPT];
#pragma unroll
    for (int ii = 0; ii < NPT; ++ii) z[ii] = bl[i0 + ii], zt[ii] = 0.0f, zS[ii] = 0.0f, zSS[ii] = 0.0f;
#pragma unroll 4
    for (int j = 0; j < W; ++j) {
      const float h0 = rowZ[j], h1 = rowZ[W + j], h2 = rowZ[2 * W + j], h3 = rowZ[3 * W + j];
#pragma unroll
      for (int ii = 0; ii < NPT; ++ii) {
        const float w = Wl[(i0 + ii) * W + j];
        z[ii] = fmaf(w, h0, z[ii]), zt[ii] = fmaf(w, h1, zt[ii]), zS[ii] = fmaf(w, h2, zS[ii]),
        zSS[ii] = fmaf(w, h3, zSS[ii]);
      }
    }
    __syncthreads();  // every lane has read the previous layer's row
    float *st = sst + ((size_t)l * PP + pidx) * 4 * W;
#pragma unroll
    for (int ii = 0; ii < NPT; ++ii) {
      const int i = i0 + ii;
      const float hv = act<ACT>(z[ii]);
      float s1, s2, s3;
      act_derivs<ACT>(hv, s1, s2, s3);
      if (act_lane) {
        if (GRAD) st[i] = hv, st[W + i] = zt[ii], st[2 * W + i] = zS[ii], st[3 * W + i] = zSS[ii];
        rowZ[i] = hv, rowZ[W + i] = s1 * zt[ii], rowZ[2 * W + i] = s1 * zS[ii],
        rowZ[3 * W + i] = fmaf(s2 * zS[ii], zS[ii], s1 * zSS[ii]);
      }
    }
    __syncthreads();
    off += W * W + W;
  }
  const int off_o = off;  // output layer: wo [W], bo
  const float *wo = sw + off_o;
  {  // group partials of y_c over this lane's neurons -> the leader (lane order, fixed)
    float y[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
    for (int ii = 0; ii < NPT; ++ii) {
      const int i = i0 + ii;
#pragma unroll
      for (int c = 0; c < 4; ++c) y[c] = fmaf(wo[i], rowZ[c * W + i], y[c]);
    }
    if (act_lane)
#pragma unroll
      for (int c = 0; c < 4; ++c) rowH[c * G + q] = y[c];
  }
  __syncthreads();
  double ell[3] = {0.0, 0.0, 0.0};
  if (act_lane && q == 0) {
    float y[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float acc = c == 0 ? sw[off_o + W] : 0.0f;
      for (int r = 0; r < G; ++r) acc += rowH[c * G + r];
      y[c] = acc;
    }
    const float V = mk.L * y[0], Vt = mk.L * y[1], VS = mk.L * y[2], VSS = mk.L * y[3];
    float Vb = 0.0f, Vtb = 0.0f, VSb = 0.0f, VSSb = 0.0f;
    if (kind == 0) {
      const float hs2 = 0.5f * mk.sig * mk.sig * S * S;
      const float f = Vt + hs2 * VSS + mk.r * S * VS - mk.r * V;  // Eq. (1) applied to the network
      ell[0] = (double)f * (double)f / (double)c0;
      const float fb = 2.0f * f / (float)c0;
      Vb = -mk.r * fb, Vtb = fb, VSb = mk.r * S * fb, VSSb = hs2 * fb;
    } else if (kind == 1) {
      const float tgt = S > 0.5f * mk.L ? (mk.asym ? mk.L - mk.K * expf(-mk.r * (mk.T - t)) : 0.0f) : 0.0f;
      const float e = V - tgt;
      ell[1] = (double)e * (double)e / (double)c1;
      Vb = 2.0f * e / (float)c1;
    } else if (kind == 2) {
      const float e = V - fmaxf(S - mk.K, 0.0f);
      ell[2] = (double)e * (double)e / (double)c2;
      Vb = 2.0f * e / (float)c2;
    }
    float *yb = sY + pidx * 4;
    yb[0] = mk.L * Vb, yb[1] = mk.L * Vtb, yb[2] = mk.L * VSb, yb[3] = mk.L * VSSb;
  }
  for (int c = 0; c < 3; ++c) block_sum3(ell[c], c, sl);
  __syncthreads();
  if (tid < 3) {
    double s = 0.0;
    for (int w = 0; w < kTPB / 32; ++w) s += sl[w * 3 + tid];
    a.lpart[(size_t)blk * 3 + tid] = s;
  }
  if (!GRAD) return;

  // ---- reverse accumulation
  float *gout = a.gpart + (size_t)blk * a.np;
  // output layer: grad wo_i = sum_p sum_c ybar_c h_c,i (h rows still in sZ), grad bo = sum_p ybar_0
  for (int e = tid; e <= W; e += kTPB) {
    float acc = 0.0f;
    if (e < W) {
      for (int p = 0; p < PP; ++p)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc = fmaf(sY[p * 4 + c], sZ[p * RS + c * W + e], acc);
    } else {
      for (int p = 0; p < PP; ++p) acc += sY[p * 4];
    }
    gout[off_o + e] = acc;
  }
  float hb[4][NPT];
  {
    const float *yb = sY + pidx * 4;
#pragma unroll
    for (int ii = 0; ii < NPT; ++ii)
#pragma unroll
      for (int c = 0; c < 4; ++c) hb[c][ii] = wo[i0 + ii] * yb[c];
  }
  __syncthreads();  // sZ is rewritten below
  for (int l = LH - 1; l >= 0; --l) {
    const float *st = sst + ((size_t)l * PP + pidx) * 4 * W;
    // z-bar of this lane's neurons through the activation's jet rules -> the point's row
#pragma unroll
    for (int ii = 0; ii < NPT; ++ii) {
      const int i = i0 + ii;
      const float hv = st[i], zt = st[W + i], zS = st[2 * W + i], zSS = st[3 * W + i];
      float s1, s2, s3;
      act_derivs<ACT>(hv, s1, s2, s3);
      const float zb = hb[0][ii] * s1 + hb[1][ii] * s2 * zt + hb[2][ii] * s2 * zS + hb[3][ii] * fmaf(s3 * zS, zS, s2 * zSS);
      const float zbS = fmaf(hb[3][ii] * 2.0f * s2, zS, hb[2][ii] * s1);
      hb[0][ii] = zb, hb[1][ii] = hb[1][ii] * s1, hb[2][ii] = zbS, hb[3][ii] = hb[3][ii] * s1;
      if (act_lane)
#pragma unroll
        for (int c = 0; c < 4; ++c) rowZ[c * W + i] = hb[c][ii];
    }
    // activation jets of the layer below (this layer's input): from the stash, or the features
    int Wi, offl;
    if (l > 0) {
      Wi = W;
      offl = 3 * W + (l - 1) * (W * W + W);
      const float *sp = sst + ((size_t)(l - 1) * PP + pidx) * 4 * W;
#pragma unroll
      for (int ii = 0; ii < NPT; ++ii) {
        const int j = i0 + ii;
        const float hv = sp[j], zt = sp[W + j], zS = sp[2 * W + j], zSS = sp[3 * W + j];
        float s1, s2, s3;
        act_derivs<ACT>(hv, s1, s2, s3);
        if (act_lane)
          rowH[j] = hv, rowH[W + j] = s1 * zt, rowH[2 * W + j] = s1 * zS, rowH[3 * W + j] = fmaf(s2 * zS, zS, s1 * zSS);
      }
    } else {
      Wi = 2;
      offl = 0;
      if (act_lane && q == 0) {
        rowH[0] = x0, rowH[1] = x1, rowH[W] = iT, rowH[W + 1] = 0.0f;
        rowH[2 * W] = 0.0f, rowH[2 * W + 1] = iL, rowH[3 * W] = 0.0f, rowH[3 * W + 1] = 0.0f;
      }
    }
    __syncthreads();
    // the layer's weight block [W][Wi] and bias over the CTA's points, fixed order
    const int nW = W * Wi;
    for (int e = tid; e < nW + W; e += kTPB) {
      float acc = 0.0f;
      if (e < nW) {
        const int i = e / Wi, j = e - (e / Wi) * Wi;
        for (int p = 0; p < PP; ++p) {
          const float *zr = sZ + p * RS, *hr = sH + p * RS;
#pragma unroll
          for (int c = 0; c < 4; ++c) acc = fmaf(zr[c * W + i], hr[c * W + j], acc);
        }
      } else {
        const int i = e - nW;
        for (int p = 0; p < PP; ++p) acc += sZ[p * RS + i];
      }
      gout[offl + e] = acc;
    }
    if (l > 0) {  // h-bar of the layer below, this lane's neurons: sum_i W_l[i][j] zbar_c,i
      const float *Wl = sw + offl;
      float nb[4][NPT];
#pragma unroll
      for (int ii = 0; ii < NPT; ++ii)
#pragma unroll
        for (int c = 0; c < 4; ++c) nb[c][ii] = 0.0f;
#pragma unroll 4
      for (int i = 0; i < W; ++i) {
        const float z0 = rowZ[i], z1 = rowZ[W + i], z2 = rowZ[2 * W + i], z3 = rowZ[3 * W + i];
#pragma unroll
        for (int ii = 0; ii < NPT; ++ii) {
          const float w = Wl[i * W + i0 + ii];
          nb[0][ii] = fmaf(w, z0, nb[0][ii]), nb[1][ii] = fmaf(w, z1, nb[1][ii]), nb[2][ii] = fmaf(w, z2, nb[2][ii]),
          nb[3][ii] = fmaf(w, z3, nb[3][ii]);
        }
      }
#pragma unroll
      for (int ii = 0; ii < NPT; ++ii)
#pragma unroll
        for (int c = 0; c < 4; ++c) hb[c][ii] = nb[c][ii];
    }
    __syncthreads();
  }
}

// Adam over the CTA partials.  A CTA owns 32 parameters (lanes) and sums their partials with its
// 32 warps (warp w: partials w, w+32, …), then the 32 warp sums in warp order (a fixed tree: the
// result is run-to-run bitwise); Adam (Kingma & Ba, Alg. 1) unless update == 0.  d_ctr[0] is the
// step counter, d_ctr[1] a completion ticket: the CTA that finishes last (every CTA has read the
// step by then) sums the loss partials, writes them into hist[step − step0] and advances the step.
constexpr int kAdamWarps = kAdamThreads / 32;
__global__ void __launch_bounds__(kAdamThreads)
    k_adam(float *theta, float *m, float *v, const float *gpart, const double *lpart, int nblk, int np,
           long long *d_ctr, long long step0, double *hist, double lr, double b1, double b2, double eps,
           int update, float *gout, double *lout) {
  __shared__ double red[kAdamWarps][33];
  __shared__ bool last;
  const long long step = d_ctr[0];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int p = blockIdx.x * 32 + lane;
  if (update || gout) {
    double g = 0.0;
    if (p < np)
      for (int k = w; k < nblk; k += kAdamWarps) g += (double)gpart[(size_t)k * np + p];
    red[w][lane] = g;
    __syncthreads();
    if (w == 0 && p < np) {
      double s = 0.0;
      for (int q = 0; q < kAdamWarps; ++q) s += red[q][lane];
      if (gout) gout[p] = (float)s;
      if (update) {
        const double t = (double)(step + 1);
        const double bc1 = 1.0 - pow(b1, t), bc2 = 1.0 - pow(b2, t);
        const double mm = b1 * (double)m[p] + (1.0 - b1) * s;
        const double vv = b2 * (double)v[p] + (1.0 - b2) * s * s;
        m[p] = (float)mm;
        v[p] = (float)vv;
        theta[p] = (float)((double)theta[p] - lr * (mm / bc1) / (sqrt(vv / bc2) + eps));
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(reinterpret_cast<unsigned long long *>(d_ctr + 1), 1ull) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  for (int c = 0; c < 3; ++c) {  // loss terms: the same fixed tree over the CTA partials
    double s = 0.0;
    for (int k = threadIdx.x; k < nblk; k += kAdamThreads) s += lpart[(size_t)k * 3 + c];
    red[w][lane] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double tot = 0.0;
      for (int q = 0; q < kAdamWarps; ++q)
        for (int l = 0; l < 32; ++l) tot += red[q][l];
      if (hist) hist[(step - step0) * 3 + c] = tot;
      if (lout) lout[c] = tot;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    d_ctr[1] = 0;
    if (update) d_ctr[0] = step + 1;
  }
}

// ---------------------------------------------------------------- dispatch on (W, ACT)
using GradFn = void (*)(GradArgs);
template <bool GRAD>
GradFn grad_kernel(int W, int act) {
#define PT_CASE(w)                                                                        \
  if (W == w) return act == kActTanh ? k_train_grad<w, PR_ACT_TANH, GRAD> : k_train_grad<w, PR_ACT_RELU, GRAD>;
  PT_CASE(8)
  PT_CASE(16)
  PT_CASE(20)
  PT_CASE(32)
  PT_CASE(50)
  PT_CASE(64)
#undef PT_CASE
  return nullptr;
}
// collocation points per CTA and shared memory of the gradient kernel
void grad_geometry(int W, int np, int LH, int *pp, size_t *smem) {
#define PT_G(w)                                                        \
  if (W == w) {                                                        \
    *pp = TG<w>::PP;                                                   \
    *smem = 128 + train_smem_floats<w>(np, LH) * sizeof(float);        \
    return;                                                            \
  }
  PT_G(8) PT_G(16) PT_G(20) PT_G(32) PT_G(50) PT_G(64)
#undef PT_G
  *pp = 0;
  *smem = 0;
}

std::string g_init_err = "no error";

std::string fmt(const char *f, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, f);
  vsnprintf(buf, sizeof buf, f, ap);
  va_end(ap);
  return buf;
}
}  // namespace

struct pt_trainer {
  std::string err = "no error";
  bool poisoned = false;
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  std::vector<int> dims;
  int W = 0, LH = 0, act = 0, np = 0, batches = 1;
  int n_f = 0, n_b = 0, n_e = 0, nblk = 0, nblk_full = 0;
  Market mk{};
  unsigned long long seed = 0;
  double b1 = 0.9, b2 = 0.999, eps = 1e-8;
  float *theta = nullptr, *m = nullptr, *v = nullptr, *gpart = nullptr, *gout = nullptr;
  int pp = 0;       // collocation points per CTA of the gradient kernel
  size_t smem = 0;  // its dynamic shared memory
  float *pts = nullptr;  // t_f, S_f, t_b, S_b, S_e
  double *lpart = nullptr, *lout = nullptr, *hist = nullptr;
  size_t hist_cap = 0;
  long long *d_step = nullptr;
  long long steps = 0;
};

namespace {
pr_status tfail(pt_trainer *tr, pr_status s, const std::string &msg) {
  if (tr) {
    tr->err = msg;
    if (s == PR_ERR_CUDA) tr->poisoned = true;
  } else {
    g_init_err = msg;
  }
  return s;
}
#define TCU(call)                                                                                      \
  do {                                                                                                 \
    cudaError_t e_ = (call);                                                                           \
    if (e_ != cudaSuccess)                                                                             \
      return tfail(tr, e_ == cudaErrorMemoryAllocation ? PR_ERR_OUT_OF_MEMORY : PR_ERR_CUDA,           \
                   fmt("%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__));   \
  } while (0)

pr_status check(pt_trainer *tr) {
  if (!tr) return tfail(nullptr, PR_ERR_INVALID_ARGUMENT, "trainer is NULL");
  if (tr->poisoned) return PR_ERR_STATE;
  TCU(cudaSetDevice(tr->device));
  return PR_OK;
}

GradArgs grad_args(pt_trainer *tr, bool full, long long step_override) {
  GradArgs a{};
  a.theta = tr->theta;
  a.np = tr->np;
  a.LH = tr->LH;
  a.gpart = tr->gpart;
  a.lpart = tr->lpart;
  a.t_f = tr->pts;
  a.S_f = tr->pts + tr->n_f;
  a.t_b = tr->pts + 2 * (size_t)tr->n_f;
  a.S_b = a.t_b + tr->n_b;
  a.S_e = a.S_b + tr->n_b;
  a.n_f = tr->n_f, a.n_b = tr->n_b, a.n_e = tr->n_e;
  a.batches = tr->batches;
  a.d_step = tr->d_step;
  a.step_override = step_override;
  a.full = full ? 1 : 0;
  a.seed = tr->seed;
  a.mk = tr->mk;
  return a;
}

pr_status launch_grad(pt_trainer *tr, bool grad, bool full, long long step_override) {
  const GradArgs a = grad_args(tr, full, step_override);
  GradFn fn = grad ? grad_kernel<true>(tr->W, tr->act) : grad_kernel<false>(tr->W, tr->act);
  const int nblk = full ? tr->nblk_full : tr->nblk;
  void *args[] = {(void *)&a};
  TCU(cudaLaunchKernel((const void *)fn, dim3(nblk), dim3(kTPB), args, tr->smem, tr->stream));
  return PR_OK;
}

pr_status launch_adam(pt_trainer *tr, int nblk, long long step0, double *hist, double lr, int update, float *gout,
                      double *lout) {
  k_adam<<<(tr->np + 31) / 32, kAdamThreads, 0, tr->stream>>>(tr->theta, tr->m, tr->v, tr->gpart, tr->lpart, nblk, tr->np, tr->d_step,
                                             step0, hist, lr, tr->b1, tr->b2, tr->eps, update, gout, lout);
  TCU(cudaPeekAtLastError());
  return PR_OK;
}
}  // namespace

extern "C" {

const char *pinn_train_last_error(const pt_trainer *tr) { return tr ? tr->err.c_str() : g_init_err.c_str(); }

pr_status pinn_train_init(const pt_config *cfg, pt_trainer **out) {
  pt_trainer *tr = nullptr;
  if (!out) return tfail(nullptr, PR_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (!cfg) return tfail(nullptr, PR_ERR_INVALID_ARGUMENT, "cfg is NULL");
  if (cfg->struct_size != sizeof(pt_config))
    return tfail(nullptr, PR_ERR_INVALID_ARGUMENT, fmt("cfg.struct_size = %u, expected %zu", cfg->struct_size, sizeof(pt_config)));
  const pt_config &c = *cfg;
  if (!(c.sigma > 0)) return tfail(nullptr, PR_ERR_INVALID_ARGUMENT, "cfg.sigma must be > 0");
  if (!(c.rate >= 0)) return tfail(nullptr, PR_ERR_INVALID_ARGUMENT, "cfg.rate must be >= 0");
  if (!(c.strike >= 0)) return tfail(nullptr, PR_ERR_INVALID_ARGUMENT, "cfg.strike must be >= 0");
  if (!(c.L > 0)) return tfail(nullptr, PR_ERR_INVALID_ARGUMENT, "cfg.L must be > 0");
  if (!(c.T > 0)) return tfail(nullptr, PR_ERR_INVALID_ARGUMENT, "cfg.T must be > 0");
  if (c.upper_bc != PR_BC_CALL_ASYMPTOTIC && c.upper_bc != PR_BC_ZERO)
    return tfail(nullptr, PR_ERR_INVALID_ARGUMENT, "cfg.upper_bc must be PR_BC_*");
  if (c.activation != PR_ACT_TANH && c.activation != PR_ACT_RELU)
    return tfail(nullptr, PR_ERR_INVALID_ARGUMENT, "cfg.activation must be PR_ACT_TANH or PR_ACT_RELU");
  if (c.n_linear < 2 || !c.dims || !c.W || !c.b)
    return tfail(nullptr, PR_ERR_INVALID_ARGUMENT, "cfg.n_linear must be >= 2 with dims, W, b given");
  if (c.dims[0] != 2 || c.dims[c.n_linear] != 1)
    return tfail(nullptr, PR_ERR_INVALID_ARGUMENT, "cfg.dims must start with 2 (t, S) and end with 1");
  const int W = c.dims[1];
  for (int l = 1; l < c.n_linear; ++l)
    if (c.dims[l] != W) return tfail(nullptr, PR_ERR_UNSUPPORTED, "cfg.dims: hidden widths must be equal");
  if (!grad_kernel<true>(W, c.activation))
    return tfail(nullptr, PR_ERR_UNSUPPORTED, fmt("cfg.dims: hidden width %d not in {8, 16, 20, 32, 50, 64}", W));
  if (c.n_f < 1 || c.n_b < 1 || c.n_exp < 1 || !c.t_f || !c.S_f || !c.t_b || !c.S_b || !c.S_exp)
    return tfail(nullptr, PR_ERR_INVALID_ARGUMENT, "cfg: every collocation set needs >= 1 point (n_f, n_b, n_exp)");
  if (c.batches < 1 || c.batches > c.n_f || c.batches > c.n_b || c.batches > c.n_exp)
    return tfail(nullptr, PR_ERR_INVALID_ARGUMENT, "cfg.batches must be in [1, min(n_f, n_b, n_exp)]");
  if (!(c.beta1 >= 0 && c.beta1 < 1 && c.beta2 >= 0 && c.beta2 < 1 && c.eps > 0))
    return tfail(nullptr, PR_ERR_INVALID_ARGUMENT, "cfg.beta1/beta2 must be in [0,1) and eps > 0");
  for (int l = 0; l < c.n_linear; ++l)
    if (!c.W[l] || !c.b[l]) return tfail(nullptr, PR_ERR_INVALID_ARGUMENT, fmt("cfg.W[%d] / cfg.b[%d] is NULL", l, l));

  tr = new pt_trainer;
  tr->device = c.device;
  tr->dims.assign(c.dims, c.dims + c.n_linear + 1);
  tr->W = W;
  tr->LH = c.n_linear - 1;
  tr->act = c.activation;
  tr->batches = c.batches;
  tr->n_f = c.n_f, tr->n_b = c.n_b, tr->n_e = c.n_exp;
  tr->mk = Market{(float)c.strike, (float)c.sigma, (float)c.rate, (float)c.T, (float)c.L,
                  c.upper_bc == PR_BC_CALL_ASYMPTOTIC ? 1 : 0};
  tr->seed = c.shuffle_seed;
  tr->b1 = c.beta1, tr->b2 = c.beta2, tr->eps = c.eps;
  std::vector<float> packed;
  for (int l = 0; l < c.n_linear; ++l) {
    packed.insert(packed.end(), c.W[l], c.W[l] + (size_t)c.dims[l + 1] * c.dims[l]);
    packed.insert(packed.end(), c.b[l], c.b[l] + c.dims[l + 1]);
  }
  tr->np = (int)packed.size();
  long long maxb = 0;
  for (int ib = 0; ib < c.batches; ++ib) {
    long long s = 0;
    for (long long n : {(long long)c.n_f, (long long)c.n_b, (long long)c.n_exp})
      s += (ib + 1) * n / c.batches - ib * n / c.batches;
    maxb = s > maxb ? s : maxb;
  }
  grad_geometry(W, tr->np, tr->LH, &tr->pp, &tr->smem);
  tr->nblk = (int)((maxb + tr->pp - 1) / tr->pp);
  tr->nblk_full = (int)(((long long)c.n_f + c.n_b + c.n_exp + tr->pp - 1) / tr->pp);
  auto bail = [&](pr_status s) {
    g_init_err = tr->err;
    pinn_train_free(tr);
    return s;
  };
#define ICU(call)                                                         \
  do {                                                                    \
    cudaError_t e_ = (call);                                              \
    if (e_ != cudaSuccess) {                                              \
      tr->err = fmt("%s failed: %s", #call, cudaGetErrorString(e_));      \
      return bail(e_ == cudaErrorMemoryAllocation ? PR_ERR_OUT_OF_MEMORY : PR_ERR_CUDA); \
    }                                                                     \
  } while (0)
  ICU(cudaSetDevice(tr->device));
  if (c.stream) {
    tr->stream = (cudaStream_t)c.stream;
  } else {
    ICU(cudaStreamCreateWithFlags(&tr->stream, cudaStreamNonBlocking));
    tr->own_stream = true;
  }
  const size_t smem = tr->smem;
  int max_optin = 0;
  ICU(cudaDeviceGetAttribute(&max_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, tr->device));
  if (smem > (size_t)max_optin) {
    tr->err = fmt("network needs %zu B of shared memory (> %d)", smem, max_optin);
    return bail(PR_ERR_UNSUPPORTED);
  }
  ICU(cudaFuncSetAttribute((const void *)grad_kernel<true>(W, tr->act), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  ICU(cudaFuncSetAttribute((const void *)grad_kernel<false>(W, tr->act), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const size_t np = tr->np, npts = 2 * (size_t)c.n_f + 2 * (size_t)c.n_b + c.n_exp;
  const int nb_max = tr->nblk > tr->nblk_full ? tr->nblk : tr->nblk_full;
  ICU(cudaMalloc(&tr->theta, np * sizeof(float)));
  ICU(cudaMalloc(&tr->m, np * sizeof(float)));
  ICU(cudaMalloc(&tr->v, np * sizeof(float)));
  ICU(cudaMalloc(&tr->gout, np * sizeof(float)));
  ICU(cudaMalloc(&tr->gpart, (size_t)tr->nblk * np * sizeof(float)));
  ICU(cudaMalloc(&tr->lpart, (size_t)nb_max * 3 * sizeof(double)));
  ICU(cudaMalloc(&tr->lout, 3 * sizeof(double)));
  ICU(cudaMalloc(&tr->pts, npts * sizeof(float)));
  ICU(cudaMalloc(&tr->d_step, 2 * sizeof(long long)));  // step counter, k_adam's completion ticket
  ICU(cudaMemcpyAsync(tr->theta, packed.data(), np * sizeof(float), cudaMemcpyHostToDevice, tr->stream));
  ICU(cudaMemsetAsync(tr->m, 0, np * sizeof(float), tr->stream));
  ICU(cudaMemsetAsync(tr->v, 0, np * sizeof(float), tr->stream));
  ICU(cudaMemsetAsync(tr->d_step, 0, 2 * sizeof(long long), tr->stream));
  float *p = tr->pts;
  const std::pair<const float *, int> parts[] = {{c.t_f, c.n_f}, {c.S_f, c.n_f}, {c.t_b, c.n_b}, {c.S_b, c.n_b},
                                                 {c.S_exp, c.n_exp}};
  for (auto &pr : parts) {
    ICU(cudaMemcpyAsync(p, pr.first, (size_t)pr.second * sizeof(float), cudaMemcpyHostToDevice, tr->stream));
    p += pr.second;
  }
  ICU(cudaStreamSynchronize(tr->stream));
#undef ICU
  *out = tr;
  return PR_OK;
}

static pr_status pinn_train_epochs_(pt_trainer *tr, int32_t epochs, double lr, double *loss_hist);
pr_status pinn_train_epochs(pt_trainer *tr, int32_t epochs, double lr, double *loss_hist) {
  const nvtxRangeId_t r = nvtxRangeStartA("pinn_train_epochs");
  const pr_status st = pinn_train_epochs_(tr, epochs, lr, loss_hist);
  nvtxRangeEnd(r);
  return st;
}
static pr_status pinn_train_epochs_(pt_trainer *tr, int32_t epochs, double lr, double *loss_hist) {
  pr_status st = check(tr);
  if (st) return st;
  if (epochs < 1) return tfail(tr, PR_ERR_INVALID_ARGUMENT, "epochs must be >= 1");
  if (!(lr > 0)) return tfail(tr, PR_ERR_INVALID_ARGUMENT, "lr must be > 0");
  const size_t nsteps = (size_t)epochs * tr->batches;
  double *hist = nullptr;
  if (loss_hist) {
    if (tr->hist_cap < nsteps) {
      cudaFree(tr->hist);
      tr->hist = nullptr;
      tr->hist_cap = 0;
      TCU(cudaMalloc(&tr->hist, nsteps * 3 * sizeof(double)));
      tr->hist_cap = nsteps;
    }
    hist = tr->hist;
  }
  const long long step0 = tr->steps;
  // one epoch as a graph (the kernels read the step counter, so the graph serves every epoch)
  cudaGraphExec_t exec = nullptr;
  if (tr->stream != nullptr && tr->stream != cudaStreamLegacy && tr->stream != cudaStreamPerThread) {
    cudaGraph_t graph = nullptr;
    TCU(cudaStreamBeginCapture(tr->stream, cudaStreamCaptureModeThreadLocal));
    pr_status s = PR_OK;
    for (int ib = 0; ib < tr->batches && s == PR_OK; ++ib) {
      s = launch_grad(tr, true, false, -1);
      if (s == PR_OK) s = launch_adam(tr, tr->nblk, step0, hist, lr, 1, nullptr, nullptr);
    }
    const cudaError_t ec = cudaStreamEndCapture(tr->stream, &graph);
    if (s) {
      if (graph) cudaGraphDestroy(graph);
      return s;
    }
    TCU(ec);
    const cudaError_t ei = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    TCU(ei);
  }
  for (int e = 0; e < epochs; ++e) {
    if (exec) {
      const cudaError_t el = cudaGraphLaunch(exec, tr->stream);
      if (el != cudaSuccess) {
        cudaGraphExecDestroy(exec);
        TCU(el);
      }
    } else {
      for (int ib = 0; ib < tr->batches; ++ib) {
        st = launch_grad(tr, true, false, -1);
        if (!st) st = launch_adam(tr, tr->nblk, step0, hist, lr, 1, nullptr, nullptr);
        if (st) return st;
      }
    }
  }
  const cudaError_t es = cudaStreamSynchronize(tr->stream);
  if (exec) cudaGraphExecDestroy(exec);
  TCU(es);
  tr->steps += (long long)nsteps;
  if (loss_hist) TCU(cudaMemcpy(loss_hist, hist, nsteps * 3 * sizeof(double), cudaMemcpyDeviceToHost));
  return PR_OK;
}

pr_status pinn_train_loss(pt_trainer *tr, double out[3]) {
  pr_status st = check(tr);
  if (st) return st;
  if (!out) return tfail(tr, PR_ERR_INVALID_ARGUMENT, "out is NULL");
  st = launch_grad(tr, false, true, 0);
  if (st) return st;
  st = launch_adam(tr, tr->nblk_full, 0, nullptr, 0.0, 0, nullptr, tr->lout);
  if (st) return st;
  TCU(cudaMemcpyAsync(out, tr->lout, 3 * sizeof(double), cudaMemcpyDeviceToHost, tr->stream));
  TCU(cudaStreamSynchronize(tr->stream));
  return PR_OK;
}

pr_status pinn_train_batch_gradient(pt_trainer *tr, int64_t step, float *grad, double loss[3]) {
  pr_status st = check(tr);
  if (st) return st;
  if (step < 0 || !grad) return tfail(tr, PR_ERR_INVALID_ARGUMENT, "step must be >= 0 and grad non-NULL");
  st = launch_grad(tr, true, false, step);
  if (st) return st;
  st = launch_adam(tr, tr->nblk, 0, nullptr, 0.0, 0, tr->gout, tr->lout);
  if (st) return st;
  TCU(cudaMemcpyAsync(grad, tr->gout, (size_t)tr->np * sizeof(float), cudaMemcpyDeviceToHost, tr->stream));
  double l[3];
  TCU(cudaMemcpyAsync(l, tr->lout, sizeof l, cudaMemcpyDeviceToHost, tr->stream));
  TCU(cudaStreamSynchronize(tr->stream));
  if (loss) std::memcpy(loss, l, sizeof l);
  return PR_OK;
}

int64_t pinn_train_param_count(const pt_trainer *tr) { return tr ? tr->np : 0; }
int64_t pinn_train_step_count(const pt_trainer *tr) { return tr ? tr->steps : 0; }

pr_status pinn_train_get_params(pt_trainer *tr, float *packed) {
  pr_status st = check(tr);
  if (st) return st;
  if (!packed) return tfail(tr, PR_ERR_INVALID_ARGUMENT, "packed is NULL");
  TCU(cudaMemcpyAsync(packed, tr->theta, (size_t)tr->np * sizeof(float), cudaMemcpyDeviceToHost, tr->stream));
  TCU(cudaStreamSynchronize(tr->stream));
  return PR_OK;
}

pr_status pinn_train_get_weights(pt_trainer *tr, float *const *W, float *const *b) {
  if (!W || !b) return tfail(tr, PR_ERR_INVALID_ARGUMENT, "W / b is NULL");
  std::vector<float> packed(tr ? tr->np : 0);
  pr_status st = pinn_train_get_params(tr, packed.data());
  if (st) return st;
  size_t o = 0;
  for (size_t l = 0; l + 1 < tr->dims.size(); ++l) {
    const size_t nW = (size_t)tr->dims[l + 1] * tr->dims[l];
    if (!W[l] || !b[l]) return tfail(tr, PR_ERR_INVALID_ARGUMENT, fmt("W[%zu] / b[%zu] is NULL", l, l));
    std::memcpy(W[l], packed.data() + o, nW * sizeof(float));
    std::memcpy(b[l], packed.data() + o + nW, tr->dims[l + 1] * sizeof(float));
    o += nW + tr->dims[l + 1];
  }
  return PR_OK;
}

void pinn_train_free(pt_trainer *tr) {
  if (!tr) return;
  cudaSetDevice(tr->device);
  if (tr->stream) cudaStreamSynchronize(tr->stream);
  cudaFree(tr->theta);
  cudaFree(tr->m);
  cudaFree(tr->v);
  cudaFree(tr->gout);
  cudaFree(tr->gpart);
  cudaFree(tr->lpart);
  cudaFree(tr->lout);
  cudaFree(tr->pts);
  cudaFree(tr->d_step);
  cudaFree(tr->hist);
  if (tr->own_stream) cudaStreamDestroy(tr->stream);
  delete tr;
}

}  // extern "C"
