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
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

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
};

template <int ACT>
__device__ __forceinline__ float act(float z) {
  if (ACT == 1) return fmaxf(z, 0.0f);
  return tanhf(z);
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

template <int IN, int W, int ACT, int PTS>
__global__ void __launch_bounds__(128) k_pinn_chain(PinnArgs a) {
  extern __shared__ float sw[];
  __shared__ double red[2 * 32];
  for (int i = threadIdx.x; i < a.nfloats; i += blockDim.x) sw[i] = a.wts[i];
  __syncthreads();
  const int b = blockIdx.y;
  const double Lb = a.Lb[b];
  const float gscale = (float)(Lb * (double)a.out_scale);
  const size_t sstride = (size_t)a.B * a.Mp;
  int j[PTS];
  bool ok[PTS];
  float s_over_L[PTS], u[PTS];
#pragma unroll
  for (int p = 0; p < PTS; ++p) {
    j[p] = blockIdx.x * (blockDim.x * PTS) + p * blockDim.x + threadIdx.x;
    ok[p] = j[p] < a.M;
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
        const double dd = (double)u[p] - (double)u0[j[p]];
        num += dd * dd;
        den += (double)u[p] * u[p];
        u0[j[p]] = u[p];
      }
    }
    if (a.partials) {
      cta_reduce2(num, den, red);
      if (threadIdx.x == 0) {
        double *pp = a.partials + (((size_t)a.ln0 * a.B + b) * a.nch + blockIdx.x) * 2;
        pp[0] = num;
        pp[1] = den;
      }
    }
  } else {
#pragma unroll
    for (int p = 0; p < PTS; ++p) u[p] = ok[p] ? u0[j[p]] : 0.f;
  }
  const int ln_end = a.Gout ? a.ln0 + 1 : a.ln1;
#pragma unroll 1
  for (int ln = a.ln0; ln < ln_end; ++ln) {
    const int n = a.n_base + ln;
    const double t_from = a.T - n * a.dT, t_to = a.T - (n + 1) * a.dT;
    float x[PTS][IN], y[PTS];
#pragma unroll
    for (int p = 0; p < PTS; ++p) {
      if (IN == 4) {
        x[p][0] = (float)(t_from / a.T) * a.cs0;
        x[p][1] = (float)(t_to / a.T) * a.cs1;
        x[p][2] = (float)((double)u[p] / Lb) * a.cs2;
        x[p][3] = s_over_L[p] * a.cs3;
      } else {
        x[p][0] = (float)(t_to / a.T) * a.cs0;
        x[p][IN - 1] = s_over_L[p] * a.cs1;
      }
    }
    mlp_eval<IN, W, ACT, PTS>(sw, a.LH, x, y);
    const size_t row = (size_t)ln * sstride + (size_t)b * a.Mp;
    if (a.Gout) {
#pragma unroll
      for (int p = 0; p < PTS; ++p)
        if (ok[p]) a.Gout[(size_t)b * a.Mp + j[p]] = gscale * y[p];
      return;
    }
    float *un = a.U + row + sstride;
    double num = 0.0, den = 0.0;
#pragma unroll
    for (int p = 0; p < PTS; ++p) {
      const float g = gscale * y[p];
      float nv = 0.f;
      if (ok[p]) {
        if (a.Gh) a.Gh[row + j[p]] = g;
        nv = a.D ? g + a.D[row + j[p]] : g;
        if (a.partials) {
          const double dd = (double)nv - (double)un[j[p]];
          num += dd * dd;
          den += (double)nv * nv;
        }
        un[j[p]] = nv;
      }
      u[p] = nv;
    }
    if (a.partials) {
      cta_reduce2(num, den, red);
      if (threadIdx.x == 0) {
        double *pp = a.partials + (((size_t)(ln + 1) * a.B + b) * a.nch + blockIdx.x) * 2;
        pp[0] = num;
        pp[1] = den;
      }
    }
  }
}

}  // namespace pr
