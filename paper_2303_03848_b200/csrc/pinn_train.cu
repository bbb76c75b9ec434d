// pinn_train.cu — GPU training of the PINN coarse propagator (
// PAPER.md §3.3; C ABI in include/pinn_train.h).
//
// One Adam step is two kernels:
//  k_train_grad  one thread per collocation point of the step's batch (its epoch's shuffle of
//                each set): forward jets (Ṽ, Ṽ_t, Ṽ_S, Ṽ_SS) through the net with the
//                weights in shared memory, the point's loss term (Eqs. 12-14) and its adjoint,
//                then reverse accumulation layer by layer.  Each layer's weight
//                gradient Σ_points Σ_jet z̄_c ⊗ h_c is contracted per CTA from shared-memory
//                tiles of the 128 points' adjoints and inputs and written as the CTA's partial
//                (no atomics: fixed summation order, run-to-run bitwise).  The forward
//                pre-activation jets are stashed per thread (coalesced, L2-resident) for the
//                reverse pass.
//  k_adam        one CTA: the fp64 sum of the CTA partials in CTA order, Adam, the
//                batch's loss terms into the history, the step counter.
// One epoch (batches × the two kernels) is captured as a CUDA graph and replayed; both kernels
// read the step counter from device memory, so the same graph serves every epoch.
#include "../../include/pinn_train.h"

#include <cuda_runtime.h>

#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

namespace {

constexpr int kTPB = 128;          // points per CTA of the gradient kernel (one per thread)
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
  float *stash;     // [nblk][LH][4][W][kTPB] forward pre-activation jets (h, z_t, z_S, z_SS)
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

// Contracts one layer's gradient over the CTA's points: entry (i, j) of the [Wo][Wi] weight block
// = Σ_p Σ_c A[c][p][i]·B[c][p][j]; bias i = Σ_p A[0][p][i].  A, B in shared memory, p-major rows.
template <int W>
__device__ __forceinline__ void contract(const float *sA, int Wo, const float *sB, int Wi, float *gout) {
  const int nW = Wo * Wi;
  for (int e = threadIdx.x; e < nW + Wo; e += kTPB) {
    float acc = 0.0f;
    if (e < nW) {
      const int i = e / Wi, j = e - (e / Wi) * Wi;
#pragma unroll 4
      for (int p = 0; p < kTPB; ++p) {
#pragma unroll
        for (int c = 0; c < 4; ++c) acc = fmaf(sA[(c * kTPB + p) * W + i], sB[(c * kTPB + p) * W + j], acc);
      }
    } else {
      const int i = e - nW;
#pragma unroll 8
      for (int p = 0; p < kTPB; ++p) acc += sA[p * W + i];
    }
    gout[e] = acc;
  }
}

template <int W, int ACT, bool GRAD>
__global__ void __launch_bounds__(kTPB) k_train_grad(GradArgs a) {
  extern __shared__ __align__(16) unsigned char smraw[];
  double *sl = reinterpret_cast<double *>(smraw);                  // [kTPB/32][3]
  float *sA = reinterpret_cast<float *>(smraw + 128);              // [4][kTPB][W]
  float *sB = sA + 4 * kTPB * W;                                   // [4][kTPB][W]
  float *sw = sB + 4 * kTPB * W;                                   // [np]
  const int tid = threadIdx.x, blk = blockIdx.x, LH = a.LH;
  for (int i = tid; i < a.np; i += kTPB) sw[i] = a.theta[i];

  // ---- the point this thread owns (batch part ib of each set's shuffle)
  const long long step = a.step_override >= 0 ? a.step_override : *a.d_step;
  const long long epoch = step / a.batches;
  const int ib = (int)(step - epoch * a.batches);
  long long lo[3], cnt[3];
  const long long n[3] = {a.n_f, a.n_b, a.n_e};
  for (int c = 0; c < 3; ++c) {
    lo[c] = a.full ? 0 : ib * n[c] / a.batches;
    cnt[c] = a.full ? n[c] : (ib + 1) * n[c] / a.batches - lo[c];
  }
  const long long g = (long long)blk * kTPB + tid;
  int kind = -1;
  long long pos = 0;
  if (g < cnt[0]) kind = 0, pos = g;
  else if (g < cnt[0] + cnt[1]) kind = 1, pos = g - cnt[0];
  else if (g < cnt[0] + cnt[1] + cnt[2]) kind = 2, pos = g - cnt[0] - cnt[1];
  const Market mk = a.mk;
  float t = 0.0f, S = 0.0f;
  if (kind >= 0) {
    const long long idx = a.full ? pos : perm_at(a.seed, epoch, kind, n[kind], lo[kind] + pos);
    if (kind == 0) t = a.t_f[idx], S = a.S_f[idx];
    else if (kind == 1) t = a.t_b[idx], S = a.S_b[idx];
    else t = mk.T, S = a.S_e[idx];
  }
  __syncthreads();

  // ---- forward jets (value, ∂t, ∂S, ∂SS) through the hidden layers; features (t/T, S/L)
  const float iT = 1.0f / mk.T, iL = 1.0f / mk.L;
  const float x0 = t * iT, x1 = S * iL;
  float h[W], ht[W], hS[W], hSS[W];
  float *st = a.stash + (size_t)blk * LH * 4 * W * kTPB + tid;
  {
    const float *W0 = sw, *b0 = sw + 2 * W;
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const float z = fmaf(W0[2 * i], x0, fmaf(W0[2 * i + 1], x1, b0[i]));
      const float zt = W0[2 * i] * iT, zS = W0[2 * i + 1] * iL;
      const float hv = act<ACT>(z);
      float s1, s2, s3;
      act_derivs<ACT>(hv, s1, s2, s3);
      if (GRAD) {
        st[(0 * W + i) * kTPB] = hv;
        st[(1 * W + i) * kTPB] = zt;
        st[(2 * W + i) * kTPB] = zS;
        st[(3 * W + i) * kTPB] = 0.0f;
      }
      h[i] = hv, ht[i] = s1 * zt, hS[i] = s1 * zS, hSS[i] = s2 * zS * zS;
    }
  }
  int off = 3 * W;  // start of layer 1's parameters
  for (int l = 1; l < LH; ++l) {
    const float *Wl = sw + off, *bl = sw + off + W * W;
    float z[W], zt[W], zS[W], zSS[W];
#pragma unroll
    for (int i = 0; i < W; ++i) {
      float a0 = bl[i], a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
#pragma unroll
      for (int j = 0; j < W; ++j) {
        const float w = Wl[i * W + j];
        a0 = fmaf(w, h[j], a0), a1 = fmaf(w, ht[j], a1), a2 = fmaf(w, hS[j], a2), a3 = fmaf(w, hSS[j], a3);
      }
      z[i] = a0, zt[i] = a1, zS[i] = a2, zSS[i] = a3;
    }
    float *sl_ = st + (size_t)l * 4 * W * kTPB;
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const float hv = act<ACT>(z[i]);
      float s1, s2, s3;
      act_derivs<ACT>(hv, s1, s2, s3);
      if (GRAD) {
        sl_[(0 * W + i) * kTPB] = hv;
        sl_[(1 * W + i) * kTPB] = zt[i];
        sl_[(2 * W + i) * kTPB] = zS[i];
        sl_[(3 * W + i) * kTPB] = zSS[i];
      }
      h[i] = hv, ht[i] = s1 * zt[i], hS[i] = s1 * zS[i], hSS[i] = fmaf(s2 * zS[i], zS[i], s1 * zSS[i]);
    }
    off += W * W + W;
  }
  const int off_o = off;  // output layer: wo [W], bo
  const float *wo = sw + off_o;
  float y = sw[off_o + W], yt = 0.0f, yS = 0.0f, ySS = 0.0f;
#pragma unroll
  for (int j = 0; j < W; ++j) y = fmaf(wo[j], h[j], y), yt = fmaf(wo[j], ht[j], yt), yS = fmaf(wo[j], hS[j], yS),
                              ySS = fmaf(wo[j], hSS[j], ySS);
  const float V = mk.L * y, Vt = mk.L * yt, VS = mk.L * yS, VSS = mk.L * ySS;

  // ---- loss term and output adjoints (Eqs. 12-14; MSE_total Eq. 11)
  float Vb = 0.0f, Vtb = 0.0f, VSb = 0.0f, VSSb = 0.0f;
  double ell[3] = {0.0, 0.0, 0.0};
  if (kind == 0) {
    const float hs2 = 0.5f * mk.sig * mk.sig * S * S;
    const float f = Vt + hs2 * VSS + mk.r * S * VS - mk.r * V;  // Eq. (1) applied to Ṽ
    ell[0] = (double)f * (double)f / (double)cnt[0];
    const float fb = 2.0f * f / (float)cnt[0];
    Vb = -mk.r * fb, Vtb = fb, VSb = mk.r * S * fb, VSSb = hs2 * fb;
  } else if (kind == 1) {
    const float tgt = S > 0.5f * mk.L ? (mk.asym ? mk.L - mk.K * expf(-mk.r * (mk.T - t)) : 0.0f) : 0.0f;
    const float e = V - tgt;
    ell[1] = (double)e * (double)e / (double)cnt[1];
    Vb = 2.0f * e / (float)cnt[1];
  } else if (kind == 2) {
    const float e = V - fmaxf(S - mk.K, 0.0f);
    ell[2] = (double)e * (double)e / (double)cnt[2];
    Vb = 2.0f * e / (float)cnt[2];
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
  const float yb[4] = {mk.L * Vb, mk.L * Vtb, mk.L * VSb, mk.L * VSSb};
  // output layer: A = ȳ (one "neuron"), B = last hidden jets
#pragma unroll
  for (int c = 0; c < 4; ++c) sA[(c * kTPB + tid) * W] = yb[c];
#pragma unroll
  for (int j = 0; j < W; ++j) {
    sB[(0 * kTPB + tid) * W + j] = h[j];
    sB[(1 * kTPB + tid) * W + j] = ht[j];
    sB[(2 * kTPB + tid) * W + j] = hS[j];
    sB[(3 * kTPB + tid) * W + j] = hSS[j];
  }
  __syncthreads();
  contract<W>(sA, 1, sB, W, gout + off_o);
  float hb[W], hbt[W], hbS[W], hbSS[W];
#pragma unroll
  for (int j = 0; j < W; ++j) hb[j] = wo[j] * yb[0], hbt[j] = wo[j] * yb[1], hbS[j] = wo[j] * yb[2], hbSS[j] = wo[j] * yb[3];
  __syncthreads();

  for (int l = LH - 1; l >= 0; --l) {
    const float *sl_ = st + (size_t)l * 4 * W * kTPB;
    // z̄ from h̄ through the activation's jet rules (in place)
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const float hv = sl_[(0 * W + i) * kTPB], zt = sl_[(1 * W + i) * kTPB], zS = sl_[(2 * W + i) * kTPB],
                  zSS = sl_[(3 * W + i) * kTPB];
      float s1, s2, s3;
      act_derivs<ACT>(hv, s1, s2, s3);
      const float zb = hb[i] * s1 + hbt[i] * s2 * zt + hbS[i] * s2 * zS + hbSS[i] * fmaf(s3 * zS, zS, s2 * zSS);
      const float zbS = fmaf(hbSS[i] * 2.0f * s2, zS, hbS[i] * s1);
      hb[i] = zb, hbt[i] = hbt[i] * s1, hbS[i] = zbS, hbSS[i] = hbSS[i] * s1;
      sA[(0 * kTPB + tid) * W + i] = hb[i];
      sA[(1 * kTPB + tid) * W + i] = hbt[i];
      sA[(2 * kTPB + tid) * W + i] = hbS[i];
      sA[(3 * kTPB + tid) * W + i] = hbSS[i];
    }
    int Wi, offl;
    if (l > 0) {
      Wi = W;
      offl = 3 * W + (l - 1) * (W * W + W);
      const float *sp = st + (size_t)(l - 1) * 4 * W * kTPB;
#pragma unroll
      for (int j = 0; j < W; ++j) {
        const float hv = sp[(0 * W + j) * kTPB], zt = sp[(1 * W + j) * kTPB], zS = sp[(2 * W + j) * kTPB],
                    zSS = sp[(3 * W + j) * kTPB];
        float s1, s2, s3;
        act_derivs<ACT>(hv, s1, s2, s3);
        sB[(0 * kTPB + tid) * W + j] = hv;
        sB[(1 * kTPB + tid) * W + j] = s1 * zt;
        sB[(2 * kTPB + tid) * W + j] = s1 * zS;
        sB[(3 * kTPB + tid) * W + j] = fmaf(s2 * zS, zS, s1 * zSS);
      }
    } else {
      Wi = 2;
      offl = 0;
      sB[(0 * kTPB + tid) * W + 0] = x0, sB[(0 * kTPB + tid) * W + 1] = x1;
      sB[(1 * kTPB + tid) * W + 0] = iT, sB[(1 * kTPB + tid) * W + 1] = 0.0f;
      sB[(2 * kTPB + tid) * W + 0] = 0.0f, sB[(2 * kTPB + tid) * W + 1] = iL;
      sB[(3 * kTPB + tid) * W + 0] = 0.0f, sB[(3 * kTPB + tid) * W + 1] = 0.0f;
    }
    __syncthreads();
    contract<W>(sA, W, sB, Wi, gout + offl);
    if (l > 0) {  // h̄_prev = W_lᵀ z̄ for every jet component
      const float *Wl = sw + offl;
      float nb[W], nbt[W], nbS[W], nbSS[W];
#pragma unroll
      for (int j = 0; j < W; ++j) nb[j] = nbt[j] = nbS[j] = nbSS[j] = 0.0f;
#pragma unroll
      for (int i = 0; i < W; ++i) {
#pragma unroll
        for (int j = 0; j < W; ++j) {
          const float w = Wl[i * W + j];
          nb[j] = fmaf(w, hb[i], nb[j]), nbt[j] = fmaf(w, hbt[i], nbt[j]), nbS[j] = fmaf(w, hbS[i], nbS[j]),
          nbSS[j] = fmaf(w, hbSS[i], nbSS[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < W; ++j) hb[j] = nb[j], hbt[j] = nbt[j], hbS[j] = nbS[j], hbSS[j] = nbSS[j];
    }
    __syncthreads();
  }
}

// One CTA: g = Σ_blk partial (fp64, CTA order); Adam (Kingma & Ba, Alg. 1) unless update == 0;
// the batch's loss terms into hist[step − step0]; the step counter.
__global__ void __launch_bounds__(kAdamThreads)
    k_adam(float *theta, float *m, float *v, const float *gpart, const double *lpart, int nblk, int np,
           long long *d_step, long long step0, double *hist, double lr, double b1, double b2, double eps,
           int update, float *gout, double *lout) {
  const long long step = *d_step;
  const double t = (double)(step + 1);
  const double bc1 = 1.0 - pow(b1, t), bc2 = 1.0 - pow(b2, t);
  for (int p = threadIdx.x; p < np && (update || gout); p += kAdamThreads) {
    double g = 0.0;
    for (int k = 0; k < nblk; ++k) g += (double)gpart[(size_t)k * np + p];
    if (gout) gout[p] = (float)g;
    if (update) {
      const double mm = b1 * (double)m[p] + (1.0 - b1) * g;
      const double vv = b2 * (double)v[p] + (1.0 - b2) * g * g;
      m[p] = (float)mm;
      v[p] = (float)vv;
      theta[p] = (float)((double)theta[p] - lr * (mm / bc1) / (sqrt(vv / bc2) + eps));
    }
  }
  if (threadIdx.x < 3) {
    double s = 0.0;
    for (int k = 0; k < nblk; ++k) s += lpart[(size_t)k * 3 + threadIdx.x];
    if (hist) hist[(step - step0) * 3 + threadIdx.x] = s;
    if (lout) lout[threadIdx.x] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0 && update) *d_step = step + 1;
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
#undef PT_CASE
  return nullptr;
}
size_t grad_smem(int W, int np) { return 128 + 2 * (size_t)4 * kTPB * W * sizeof(float) + (size_t)np * sizeof(float); }

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
  float *theta = nullptr, *m = nullptr, *v = nullptr, *gpart = nullptr, *stash = nullptr, *gout = nullptr;
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
  a.stash = tr->stash;
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
  TCU(cudaLaunchKernel((const void *)fn, dim3(nblk), dim3(kTPB), args, grad_smem(tr->W, tr->np), tr->stream));
  return PR_OK;
}

pr_status launch_adam(pt_trainer *tr, int nblk, long long step0, double *hist, double lr, int update, float *gout,
                      double *lout) {
  k_adam<<<1, kAdamThreads, 0, tr->stream>>>(tr->theta, tr->m, tr->v, tr->gpart, tr->lpart, nblk, tr->np, tr->d_step,
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
    return tfail(nullptr, PR_ERR_UNSUPPORTED, fmt("cfg.dims: hidden width %d not in {8, 16, 20, 32}", W));
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
  tr->nblk = (int)((maxb + kTPB - 1) / kTPB);
  tr->nblk_full = (int)(((long long)c.n_f + c.n_b + c.n_exp + kTPB - 1) / kTPB);
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
  const size_t smem = grad_smem(W, tr->np);
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
  ICU(cudaMalloc(&tr->stash, (size_t)tr->nblk * tr->LH * 4 * W * kTPB * sizeof(float)));
  ICU(cudaMalloc(&tr->pts, npts * sizeof(float)));
  ICU(cudaMalloc(&tr->d_step, sizeof(long long)));
  ICU(cudaMemcpyAsync(tr->theta, packed.data(), np * sizeof(float), cudaMemcpyHostToDevice, tr->stream));
  ICU(cudaMemsetAsync(tr->m, 0, np * sizeof(float), tr->stream));
  ICU(cudaMemsetAsync(tr->v, 0, np * sizeof(float), tr->stream));
  ICU(cudaMemsetAsync(tr->d_step, 0, sizeof(long long), tr->stream));
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

pr_status pinn_train_epochs(pt_trainer *tr, int32_t epochs, double lr, double *loss_hist) {
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
  cudaFree(tr->stash);
  cudaFree(tr->pts);
  cudaFree(tr->d_step);
  cudaFree(tr->hist);
  if (tr->own_stream) cudaStreamDestroy(tr->stream);
  delete tr;
}

}  // extern "C"
