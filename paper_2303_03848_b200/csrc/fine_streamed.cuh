// fine_streamed.cuh — K2: HBM-streamed implicit-Euler propagator for large M.
//
// Same mathematics as K1 (fine_resident.cuh): every implicit step solves
// (I − dτA) x⁺ = x + dτ(a_M+b_M) g(τ⁺) e_M.  With the LU
// factors of the tridiagonal matrix (pivots p_j, off-diagonals l_j, u_j) it is
// a forward pass and a backward pass, each a first-order linear recurrence:
//   forward   w_j = r_j/p_j − m̃_j w_{j−1},   m̃_j = l_j/p_j      (w = y/p)
//   backward  x_j = w_j − c_j x_{j+1},        c_j = u_j/p_j
// (the usual elimination y_j = r_j − (l_j/p_{j−1}) y_{j−1}, x_j = y_j/p_j − c_j x_{j+1},
// with the division by p_j moved into the forward pass).  A system (one instance ×
// one slice, up to 2^20 points and more) is cut into tiles of kSTile points (one
// CTA) and threads of kSPS points; one pass is one kernel launch.
//
// Pre-aggregated passes.  Over a thread's kSPS points a recurrence is an
// affine map v ↦ A + B·v of the value entering the thread.  B is a product of
// constant factors (host table), and A is linear in the pass's *input* — the
// previous pass's *output*.  So every pass, as it produces its outputs, also
// accumulates the next pass's per-thread A (and, reduced over the CTA, the
// per-tile A) and publishes them.  A pass therefore starts with every
// aggregate it needs already in memory: the value entering its tile is the
// composition of its predecessors' tile aggregates (look-back), the value
// entering each thread a CTA scan of its tile's thread aggregates, and each
// thread then runs its recurrence once, sequentially, from the exact entering
// value — no waiting on other CTAs, no second pass over registers.  The first
// pass of a slice takes its aggregates from k_agg0.
//
// S systems per CTA.  A CTA runs the same tile of S systems that share one
// factor set (S consecutive slices of one instance): the factor loads, their
// derivation and the multiplier scan are done once for the S systems.
//
// Look-back truncation.  Tile i composes the aggregates of predecessors
// i−1 … i−W_i only, W_i (host-computed) being the first window whose
// multiplier product falls below kLookbackEps: tiles further back change the
// entering value by < kLookbackEps·|y| (eight orders below fp64 rounding).
// Fixed composition orders → bitwise reproducible results.
//
// Factors.  Only 1/p_j is stored (fp64, interleaved); m̃_j and c_j are formed
// in registers from the closed-form off-diagonals l_j = −dτ(a_j−b_j),
// u_j = −dτ(a_j+b_j) (a_j = σ²j²/2, b_j = rj/2, j = 1..M).
// Per point and pass: 4 B state read + 4 B written (HBM); 8/S B of 1/p (L2).
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>
#include <stdlib.h>
#include <type_traits>

#ifndef PR_FINE_STREAMED_ARGS
#define PR_FINE_STREAMED_ARGS
namespace pr {

constexpr int kSPS = 16;                 // points per thread
constexpr int kSNT = 128;                // threads per tile
constexpr int kSTile = kSPS * kSNT;      // 2048 points per tile
constexpr double kLookbackEps = 1e-24;   // look-back truncation (see above)

// Interleaved ("thread-major") layout: point j of a row sits at
// tile·kSTile + i·kSNT + t  (tile = j / kSTile, t = (j % kSTile) / kSPS, i = j % kSPS),
// so the i-th point of every thread of a warp is one contiguous segment.
__host__ __device__ inline size_t il_index(size_t j) {
  return (j / kSTile) * kSTile + (j % kSPS) * kSNT + (j % kSTile) / kSPS;
}
inline int streamed_Mt(int M) { return (M + kSTile - 1) / kSTile * kSTile; }
inline int streamed_ntiles(int M) { return (M + kSTile - 1) / kSTile; }

// Constant data of one implicit scheme (I − dτA) for K2, per factor set.
struct StreamedFactors {
  const double *ip;              // interleaved [nsets][Mt] 1/p_j, 1 beyond M
  const double *coef;            // [nsets][2]: dτ·r/2, dτ·σ²/2  (l_j = j(c0 − c1 j), u_j = −j(c0 + c1 j))
  const double *thrB;            // [2][nsets][Mt/kSPS] thread multiplier Π(−m̃_j) / Π(−c_j)
  const double *tileB;           // [2][nsets][ntiles] tile multiplier, indexed by scan position
  const int *tileW;              // [2][nsets][ntiles] look-back window (predecessors)
};

struct StreamedState {
  float *X = nullptr, *Y = nullptr;   // [nsys][Mt] ping-pong state (interleaved)
  double *aggT[2] = {nullptr, nullptr};  // [nsys][Mt/kSPS] thread aggregates: [0] read by forward passes, [1] by backward
  double *aggL[2] = {nullptr, nullptr};  // [nsys][ntiles] tile aggregates (tile index)
  int ntiles = 0;
  size_t nsys_max = 0;
};

inline size_t streamed_state_bytes(int M, int Mp, int B, int Nloc) {
  (void)Mp;
  const size_t nsys = (size_t)B * (size_t)(Nloc > 0 ? Nloc : 1);
  const size_t Mt = (size_t)streamed_Mt(M);
  return 2 * nsys * Mt * sizeof(float) + 2 * nsys * (Mt / kSPS) * sizeof(double) +
         2 * nsys * streamed_ntiles(M) * sizeof(double) + 2048;
}
inline void streamed_state_bind(StreamedState &s, char *base, int M, int Mp, int B, int Nloc) {
  (void)Mp;
  const size_t nsys = (size_t)B * (size_t)(Nloc > 0 ? Nloc : 1);
  const size_t Mt = (size_t)streamed_Mt(M);
  s.ntiles = streamed_ntiles(M);
  s.nsys_max = nsys;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char *p = base + off;
    off = (off + bytes + 255) / 256 * 256;
    return p;
  };
  s.X = (float *)take(nsys * Mt * sizeof(float));
  s.Y = (float *)take(nsys * Mt * sizeof(float));
  for (int k = 0; k < 2; ++k) s.aggT[k] = (double *)take(nsys * (Mt / kSPS) * sizeof(double));
  for (int k = 0; k < 2; ++k) s.aggL[k] = (double *)take(nsys * s.ntiles * sizeof(double));
}

// Epilogue of a backward pass
enum { EPI_X = 0, EPI_SWEEP = 1, EPI_CHAIN = 2 };

struct PassArgs {
  int M, Mp, Mt, B, ntiles, nsys, nsets;
  int nsl, ngroups;          // systems s = ls·B + b, ls < nsl; CTA group g ↔ (b = g % B, slices (g/B)·S …)
  StreamedFactors f;
  const int *fset;
  const float *in;           // [nsys][Mp] natural rows (first pass of a slice) or [nsys][Mt] interleaved
  float *out;                // [nsys][Mt] interleaved (forward passes, EPI_X)
  const double *aggT_cur, *aggL_cur;  // aggregates of this pass (complete at launch)
  double *aggT_next, *aggL_next;      // aggregates of the next pass (written here)
  // forward boundary term
  const double *bcoef, *Lb, *Kb, *rb;
  int upper_bc;
  double dT, dtau;           // τ_{m+1} = (n·dT + m·dτ) + dτ  (same association as the oracle)
  int step_m;
  int n_base, ln0;           // system s ↔ local slice ln0 + s / B, instance s % B
  // epilogue (backward pass of the last step of a slice)
  int epi;
  const float *Gh;           // EPI_SWEEP: D = x − Gh   (per system rows)
  float *D;
  float *Fk; int fk_sys_lo, fk_sys_hi;  // EPI_SWEEP: systems in [lo,hi) write F̂ to Fk[b]
  float *Fout;               // EPI_SWEEP: non-null → every system writes F̂ to Fout[s]
  // EPI_CHAIN (systems = instances, one slice):
  float *Unext;              // [B][Mp]: U_{n+1} (old value read for δ, then overwritten)
  float *GhW;                // nullable
  const float *Dc;           // nullable
  double *partials;          // nullable: [(b)·nch + tile]·2 (caller offsets by slice)
  int nch;
};

struct StreamedJob {       // fine sweep over local slices [ln0, ln0+nsl)
  const float *U, *Gh;
  float *D, *Fk, *Fout;
  int fk_ln, ln0, nsl, n_base;
};
struct StreamedChainJob {  // chain over local slices [ln0, ln1), one system per instance
  float *U, *Gh;
  const float *D, *Fcopy;
  double *partials;
  int nch, ln0, ln1, n_base;
  size_t ustride;          // 0 → in place
};

struct StreamedProblem {   // what every pass of one scheme shares
  StreamedFactors f;
  int nsets;
  const int *fset;
  const double *bcoef, *L, *K, *r;
  int upper_bc;
  double dT, dtau;
  int steps, M, Mp, B;
};

cudaError_t streamed_sweep(StreamedState &st, const StreamedProblem &p, const StreamedJob &j, cudaStream_t s,
                           int *nl);
cudaError_t streamed_chain(StreamedState &st, const StreamedProblem &p, const StreamedChainJob &j,
                           cudaStream_t s, int *nl);

}  // namespace pr
#endif  // PR_FINE_STREAMED_ARGS

#if !defined(PR_ARGS_ONLY) && !defined(PR_FINE_STREAMED_IMPL)
#define PR_FINE_STREAMED_IMPL
namespace pr {

template <int DIR>
__device__ __forceinline__ double shfl_prev(double v, int d) {
  return DIR == 0 ? __shfl_up_sync(0xffffffffu, v, d) : __shfl_down_sync(0xffffffffu, v, d);
}

// dτ(a_M+b_M)·g(τ_{m+1}) of step m of slice n, g the upper boundary value (reading Q3)
__device__ __forceinline__ double bc_term(const PassArgs &a, int b, int n, int m) {
  const double tau = (n * a.dT + m * a.dtau) + a.dtau;
  const double g = a.upper_bc ? 0.0 : a.Lb[b] - a.Kb[b] * exp(-a.rb[b] * tau);
  return a.bcoef[b] * g;
}

// m̃_j = l_j/p_j and c_j = u_j/p_j at 0-based point j (J = j+1) from 1/p.  EDGE: apply the
// boundary rows (no l at j = 0, no u at j = M−1) and the identity padding beyond M.
template <bool EDGE>
__device__ __forceinline__ void factors(double c0, double c1, double J, double ip, int j, int M, double &mt,
                                        double &cj) {
  const double l = J * fma(-c1, J, c0);
  const double u = -J * fma(c1, J, c0);
  mt = l * ip;
  cj = u * ip;
  if (EDGE) {
    if (!(j >= 1 && j < M)) mt = 0.0;
    if (!(j < M - 1)) cj = 0.0;
  }
}

__device__ __forceinline__ void load_natural(const float *in, int j0, int M, float x[kSPS]) {
  if (j0 + kSPS <= M) {
#pragma unroll
    for (int i = 0; i < kSPS; i += 4) {
      const float4 v = *reinterpret_cast<const float4 *>(in + j0 + i);
      x[i] = v.x; x[i + 1] = v.y; x[i + 2] = v.z; x[i + 3] = v.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < kSPS; ++i) x[i] = (j0 + i < M) ? in[j0 + i] : 0.0f;
  }
}

// Ordered composition of S per-thread maps (A_q, B) (common multiplier B) over the CTA in the
// scan order of direction D (0: threads ascending, 1: descending), fixed tree.  Thread 0 gets T.
template <int D, int NW, int S>
__device__ __forceinline__ void cta_compose(double (&A)[S], double B, double *red, int t, double (&T)[S]) {
  const int lane = t & 31, w = t >> 5;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double oB = __shfl_down_sync(0xffffffffu, B, d);
#pragma unroll
    for (int q = 0; q < S; ++q) {
      const double oA = __shfl_down_sync(0xffffffffu, A[q], d);
      if ((lane & (2 * d - 1)) == 0) A[q] = D == 0 ? fma(oB, A[q], oA) : fma(B, oA, A[q]);
    }
    if ((lane & (2 * d - 1)) == 0) B *= oB;
  }
  __syncthreads();  // red[] may still be read by an earlier phase
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < S; ++q) red[(S + 1) * w + q] = A[q];
    red[(S + 1) * w + S] = B;
  }
  __syncthreads();
  if (t == 0) {
#pragma unroll
    for (int q = 0; q < S; ++q) {
      double v = 0.0;
      if (D == 0) {
        for (int k = 0; k < NW; ++k) v = fma(red[(S + 1) * k + S], v, red[(S + 1) * k + q]);
      } else {
        for (int k = NW - 1; k >= 0; --k) v = fma(red[(S + 1) * k + S], v, red[(S + 1) * k + q]);
      }
      T[q] = v;
    }
  }
}

// The value entering the tile at scan position `pos` of system s: composition of the tile
// aggregates of its W_pos predecessors (published by the previous launch).  Warp-level; lane 0.
template <int DIR>
__device__ __forceinline__ double look_back(const PassArgs &a, int s, int pos, int set, int lane) {
  if (pos == 0) return 0.0;
  const size_t tb = ((size_t)DIR * a.nsets + set) * a.ntiles;
  const double *agg = a.aggL_cur + (size_t)s * a.ntiles;
  const int W = __ldg(a.f.tileW + tb + pos);
  double accA = 0.0, accB = 1.0;
  for (int base = 0; base < W; base += 32) {
    const int k = base + lane;          // predecessor at distance k+1 in scan order
    double mA = 0.0, mB = 1.0;          // identity beyond the window
    if (k < W) {
      const int p = pos - 1 - k;
      mA = agg[DIR == 0 ? p : a.ntiles - 1 - p];
      mB = __ldg(a.f.tileB + tb + p);
    }
    // ordered composition lane 0 ∘ lane 1 ∘ … ∘ lane 31 (fixed tree: deterministic)
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double oA = __shfl_down_sync(0xffffffffu, mA, d);
      const double oB = __shfl_down_sync(0xffffffffu, mB, d);
      if ((lane & (2 * d - 1)) == 0) {
        mA = fma(mB, oA, mA);
        mB *= oB;
      }
    }
    accA = fma(accB, mA, accA);  // lane 0 holds the window's composition
    accB *= mB;
  }
  return accA;
}

// Aggregates of the first (forward) pass of a slice, from its natural-layout input rows
// (one system per CTA): w_last = Σ_i r_i/p_i Π_{k>i}(−m̃_k) + Π(−m̃)·w_in.
__global__ void __launch_bounds__(kSNT) k_agg0(PassArgs a) {
  constexpr int NW = kSNT / 32;
  __shared__ double red[2 * NW];
  const int s = blockIdx.x % a.nsys, tile = blockIdx.x / a.nsys;
  const int b = s % a.B, ln = a.ln0 + s / a.B, set = a.fset[b];
  const int t = threadIdx.x;
  const int j0 = tile * kSTile + t * kSPS;
  float x[kSPS];
  double ipv[kSPS];
  load_natural(a.in + (size_t)s * a.Mp, j0, a.M, x);
  const double *ip = a.f.ip + (size_t)set * a.Mt + (size_t)tile * kSTile + t;
#pragma unroll
  for (int i = 0; i < kSPS; ++i) ipv[i] = __ldg(ip + i * kSNT);
  const double c0 = __ldg(a.f.coef + 2 * set), c1 = __ldg(a.f.coef + 2 * set + 1);
  const bool has_bc = j0 <= a.M - 1 && a.M - 1 < j0 + kSPS;
  const double bcv = has_bc ? bc_term(a, b, a.n_base + ln, 0) : 0.0;
  const double J0 = (double)(j0 + 1);
  double A[1] = {0.0}, P = 1.0;
#pragma unroll
  for (int i = kSPS - 1; i >= 0; --i) {
    const int j = j0 + i;
    double mt, cj;
    factors<true>(c0, c1, J0 + i, ipv[i], j, a.M, mt, cj);
    const double r = (j == a.M - 1) ? (double)x[i] + bcv : (double)x[i];
    A[0] = fma(r * ipv[i], P, A[0]);
    P *= -mt;
  }
  const size_t nthr = (size_t)a.Mt / kSPS;
  a.aggT_next[(size_t)s * nthr + (size_t)tile * kSNT + t] = A[0];
  double T[1];
  cta_compose<0, NW, 1>(A, P, red, t, T);
  if (t == 0) a.aggL_next[(size_t)s * a.ntiles + tile] = T[0];
}

// One pass over one tile of S systems (kSNT threads × kSPS points each).  NEXT: also publish
// the next pass's thread and tile aggregates.
template <int DIR, bool IN_IL, bool OUT_IL, bool NEXT, int S>
__global__ void __launch_bounds__(kSNT) k_streamed_pass(PassArgs a) {
  constexpr int NW = kSNT / 32;
  constexpr int ND = 1 - DIR;  // direction of the next pass
  static_assert(S <= NW, "one look-back warp per system");
  __shared__ double sA[S][NW], sB[NW];
  __shared__ double s_yin[S];
  __shared__ double red[(S + 1) * NW];
  const int g = (int)(blockIdx.x % a.ngroups);
  const int pos = (int)(blockIdx.x / a.ngroups);       // position in scan order
  const int tile = DIR == 0 ? pos : a.ntiles - 1 - pos;
  const int b = g % a.B;
  const int ls0 = (g / a.B) * S;                       // first launch-local slice of the group
  const int set = a.fset[b];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int j0 = tile * kSTile + t * kSPS;
  const size_t til = (size_t)tile * kSTile + t;   // interleaved offset of this thread's point 0
  const size_t nthr = (size_t)a.Mt / kSPS;
  const size_t thr = (size_t)tile * kSNT + t;     // thread index within the system
  int sys[S];
  bool ok[S];
#pragma unroll
  for (int q = 0; q < S; ++q) {
    ok[q] = ls0 + q < a.nsl;
    sys[q] = ok[q] ? (ls0 + q) * a.B + b : (ls0 * a.B + b);  // invalid → duplicate of the first (no stores)
  }

  // ---- issue every load: thread aggregates and multiplier, the state, 1/p
  double tA[S];
#pragma unroll
  for (int q = 0; q < S; ++q) tA[q] = a.aggT_cur[(size_t)sys[q] * nthr + thr];
  const double tB = __ldg(a.f.thrB + ((size_t)DIR * a.nsets + set) * nthr + thr);
  float x[S][kSPS];
#pragma unroll
  for (int q = 0; q < S; ++q) {
    if (IN_IL) {
      const float *in = a.in + (size_t)sys[q] * a.Mt + til;
#pragma unroll
      for (int i = 0; i < kSPS; ++i) x[q][i] = __ldcs(in + i * kSNT);
    } else {
      load_natural(a.in + (size_t)sys[q] * a.Mp, j0, a.M, x[q]);
    }
  }
  double ipv[kSPS];
  {
    const double *ip = a.f.ip + (size_t)set * a.Mt + til;
#pragma unroll
    for (int i = 0; i < kSPS; ++i) ipv[i] = __ldg(ip + i * kSNT);
  }
  const double c0 = __ldg(a.f.coef + 2 * set), c1 = __ldg(a.f.coef + 2 * set + 1);
  // ---- the value entering the tile (one warp per system), and the CTA scan of the thread maps
  if (w >= NW - S) {
    const int q = NW - 1 - w;
    const double y = look_back<DIR>(a, sys[q], pos, set, lane);
    if (lane == 0) s_yin[q] = y;
  }
  const int sl = DIR == 0 ? lane : 31 - lane;  // scan-order lane
  double iA[S], iB = tB;
#pragma unroll
  for (int q = 0; q < S; ++q) iA[q] = tA[q];
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double pB = shfl_prev<DIR>(iB, d);
#pragma unroll
    for (int q = 0; q < S; ++q) {
      const double pA = shfl_prev<DIR>(iA[q], d);
      if (sl >= d) iA[q] = fma(iB, pA, iA[q]);
    }
    if (sl >= d) iB *= pB;
  }
  const int sw = DIR == 0 ? w : NW - 1 - w;    // scan-order warp
  if (sl == 31) {
#pragma unroll
    for (int q = 0; q < S; ++q) sA[q][sw] = iA[q];
    sB[sw] = iB;
  }
  __syncthreads();  // sA/sB and s_yin ready
  double eB = shfl_prev<DIR>(iB, 1);
  if (sl == 0) eB = 1.0;
  double wB = 1.0;
  for (int k = 0; k < sw; ++k) wB *= sB[k];
  double v[S];  // value entering this thread, per system
#pragma unroll
  for (int q = 0; q < S; ++q) {
    double wA = 0.0;  // prefix of preceding warps (in scan order)
    for (int k = 0; k < sw; ++k) wA = fma(sB[k], wA, sA[q][k]);
    double eA = shfl_prev<DIR>(iA[q], 1);
    if (sl == 0) eA = 0.0;
    v[q] = fma(eB * wB, s_yin[q], fma(eB, wA, eA));
  }
  // ---- the recurrence, once, from the exact entering value; next pass's aggregate on the fly
  double An[S], Pn = 1.0;
#pragma unroll
  for (int q = 0; q < S; ++q) An[q] = 0.0;
  const double J0 = (double)(j0 + 1);
  auto run = [&](auto edge_tag) {
    constexpr bool EDGE = decltype(edge_tag)::value;
    double bcv[S];
#pragma unroll
    for (int q = 0; q < S; ++q) {
      bcv[q] = 0.0;
      if (EDGE && j0 <= a.M - 1 && a.M - 1 < j0 + kSPS && (DIR == 0 || NEXT))
        bcv[q] = bc_term(a, b, a.n_base + a.ln0 + ls0 + q, a.step_m + DIR);
    }
    if (DIR == 0) {
#pragma unroll
      for (int i = 0; i < kSPS; ++i) {
        const int j = j0 + i;
        double mt, cj;
        factors<EDGE>(c0, c1, J0 + i, ipv[i], j, a.M, mt, cj);
#pragma unroll
        for (int q = 0; q < S; ++q) {
          const double r = (EDGE && j == a.M - 1) ? (double)x[q][i] + bcv[q] : (double)x[q][i];
          v[q] = fma(-mt, v[q], r * ipv[i]);
          x[q][i] = (float)v[q];
          // backward map of the thread: x_{j0} = Σ_i w_i Π_{k<i}(−c_k) + Pn·x_{j0+kSPS}
          if (NEXT) An[q] = fma(v[q], Pn, An[q]);
        }
        if (NEXT) Pn *= -cj;
      }
    } else {
#pragma unroll
      for (int i = kSPS - 1; i >= 0; --i) {
        const int j = j0 + i;
        double mt, cj;
        factors<EDGE>(c0, c1, J0 + i, ipv[i], j, a.M, mt, cj);
#pragma unroll
        for (int q = 0; q < S; ++q) {
          v[q] = fma(-cj, v[q], (double)x[q][i]);
          x[q][i] = (float)v[q];
          // forward map of step m+1: w_last = Σ_i r_i/p_i Π_{k>i}(−m̃_k) + Pn·w_{j0−1}
          if (NEXT) {
            const double r = (EDGE && j == a.M - 1) ? v[q] + bcv[q] : v[q];
            An[q] = fma(r * ipv[i], Pn, An[q]);
          }
        }
        if (NEXT) Pn *= -mt;
      }
    }
  };
  // Aggregates use the unrounded outputs: the next pass then sees the recurrence applied to
  // inputs within fp32 rounding of the stored ones — the same perturbation storage makes.
  const bool edge = j0 == 0 || j0 + kSPS > a.M - 1;
  if (edge) run(std::true_type{});
  else run(std::false_type{});
  // ---- stores / epilogues
  if (OUT_IL) {
#pragma unroll
    for (int q = 0; q < S; ++q) {
      if (!ok[q]) continue;
      float *op = a.out + (size_t)sys[q] * a.Mt + til;
#pragma unroll
      for (int i = 0; i < kSPS; ++i) __stcs(op + i * kSNT, x[q][i]);
    }
  } else if (a.epi == EPI_SWEEP) {
#pragma unroll
    for (int q = 0; q < S; ++q) {
      if (!ok[q]) continue;
      const int s = sys[q];
      float *op;
      bool diff = false;
      if (a.Fout) op = a.Fout + (size_t)s * a.Mp;
      else if (s >= a.fk_sys_lo && s < a.fk_sys_hi) op = a.Fk + (size_t)b * a.Mp;
      else { op = a.D + (size_t)s * a.Mp; diff = true; }
      if (diff) {
        float gh[kSPS];
        load_natural(a.Gh + (size_t)s * a.Mp, j0, a.M, gh);
#pragma unroll
        for (int i = 0; i < kSPS; ++i) x[q][i] = (float)((double)x[q][i] - (double)gh[i]);
      }
      if (j0 + kSPS <= a.M) {
#pragma unroll
        for (int i = 0; i < kSPS; i += 4)
          *reinterpret_cast<float4 *>(op + j0 + i) = make_float4(x[q][i], x[q][i + 1], x[q][i + 2], x[q][i + 3]);
      } else {
#pragma unroll
        for (int i = 0; i < kSPS; ++i)
          if (j0 + i < a.M) op[j0 + i] = x[q][i];
      }
    }
  } else {  // EPI_CHAIN (S = 1): g = x; Ĝ_n = g; U_{n+1} = g + D_n; δ partial against the old U_{n+1}
    const size_t row = (size_t)b * a.Mp;
    float old[kSPS], dc[kSPS];
    if (a.partials) load_natural(a.Unext + row, j0, a.M, old);
    if (a.Dc) load_natural(a.Dc + row, j0, a.M, dc);
    double num = 0.0, den = 0.0;
#pragma unroll
    for (int i = 0; i < kSPS; ++i) {
      const int j = j0 + i;
      if (j < a.M) {
        if (a.GhW) a.GhW[row + j] = x[0][i];
        const float nv = a.Dc ? (float)((double)x[0][i] + (double)dc[i]) : x[0][i];
        if (a.partials) {
          const double dd = (double)nv - (double)old[i];
          num += dd * dd;
          den += (double)nv * nv;
        }
        a.Unext[row + j] = nv;
      }
    }
    if (a.partials) {
#pragma unroll
      for (int q2 = 16; q2 > 0; q2 >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, q2);
        den += __shfl_xor_sync(0xffffffffu, den, q2);
      }
      __syncthreads();
      if (lane == 0) { red[2 * w] = num; red[2 * w + 1] = den; }
      __syncthreads();
      if (t == 0) {
        num = 0.0; den = 0.0;
        for (int q2 = 0; q2 < NW; ++q2) { num += red[2 * q2]; den += red[2 * q2 + 1]; }
        double *pp = a.partials + ((size_t)b * a.nch + tile) * 2;
        pp[0] = num;
        pp[1] = den;
      }
    }
  }
  if (NEXT) {
#pragma unroll
    for (int q = 0; q < S; ++q)
      if (ok[q]) a.aggT_next[(size_t)sys[q] * nthr + thr] = An[q];
    double T[S];
    cta_compose<ND, NW, S>(An, Pn, red, t, T);
    if (t == 0) {
#pragma unroll
      for (int q = 0; q < S; ++q)
        if (ok[q]) a.aggL_next[(size_t)sys[q] * a.ntiles + tile] = T[q];
    }
  }
}

// U_k := F̂_{k−1} with the δ partial of slice k (reading Q12), elementwise.
__global__ void k_copy_delta(float *Uk, const float *F, int M, int Mp, double *partials, int B, int nch) {
  __shared__ double red[64];
  const int b = blockIdx.y;
  double num = 0.0, den = 0.0;
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < M) {
    const float nv = F[(size_t)b * Mp + j];
    const double dd = (double)nv - (double)Uk[(size_t)b * Mp + j];
    num = dd * dd;
    den = (double)nv * nv;
    Uk[(size_t)b * Mp + j] = nv;
  }
  if (!partials) return;
  for (int o = 16; o > 0; o >>= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, o);
    den += __shfl_xor_sync(0xffffffffu, den, o);
  }
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) { red[2 * w] = num; red[2 * w + 1] = den; }
  __syncthreads();
  if (threadIdx.x == 0) {
    num = 0.0; den = 0.0;
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) { num += red[2 * q]; den += red[2 * q + 1]; }
    double *pp = partials + ((size_t)b * nch + blockIdx.x) * 2;
    pp[0] = num;
    pp[1] = den;
  }
}

// Systems per CTA for a launch over nsl slices (S consecutive slices share a factor set).
static int pick_S(int nsl, int epi) {
  if (epi == EPI_CHAIN) return 1;
  if (const char *e = getenv("PR_K2_S")) {  // tuning override (1, 2 or 4)
    const int v = atoi(e);
    if (v == 1 || v == 2 || v == 4) return nsl >= v ? v : 1;
  }
  if (nsl >= 2) return 2;  // S = 4 measured slower at C3 (170 registers: 3 CTAs/SM)
  return 1;
}

template <int S>
static void launch_S(int dir, bool in_il, bool next, const PassArgs &a, unsigned grid, cudaStream_t s) {
  if (dir == 0) {
    if (in_il) k_streamed_pass<0, true, true, true, S><<<grid, kSNT, 0, s>>>(a);
    else k_streamed_pass<0, false, true, true, S><<<grid, kSNT, 0, s>>>(a);
  } else if (a.epi == EPI_X) {
    if (next) k_streamed_pass<1, true, true, true, S><<<grid, kSNT, 0, s>>>(a);
    else k_streamed_pass<1, true, true, false, S><<<grid, kSNT, 0, s>>>(a);
  } else {
    k_streamed_pass<1, true, false, false, S><<<grid, kSNT, 0, s>>>(a);
  }
}

// Forward passes read aggregates [0] and write [1]; backward passes read [1] and write [0].
static cudaError_t launch_pass(StreamedState &st, int dir, bool in_il, bool next, PassArgs a, int S,
                               cudaStream_t s) {
  a.ntiles = st.ntiles;
  a.aggT_cur = st.aggT[dir];
  a.aggL_cur = st.aggL[dir];
  a.aggT_next = st.aggT[1 - dir];
  a.aggL_next = st.aggL[1 - dir];
  a.ngroups = a.B * ((a.nsl + S - 1) / S);
  const unsigned grid = (unsigned)((unsigned long long)a.ngroups * st.ntiles);
  if (S == 4) launch_S<4>(dir, in_il, next, a, grid, s);
  else if (S == 2) launch_S<2>(dir, in_il, next, a, grid, s);
  else launch_S<1>(dir, in_il, next, a, grid, s);
  return cudaGetLastError();
}

static PassArgs pass_base(const StreamedProblem &p) {
  PassArgs a;
  memset(&a, 0, sizeof a);
  a.M = p.M; a.Mp = p.Mp; a.B = p.B; a.Mt = streamed_Mt(p.M); a.nsets = p.nsets;
  a.f = p.f; a.fset = p.fset;
  a.bcoef = p.bcoef; a.Lb = p.L; a.Kb = p.K; a.rb = p.r; a.upper_bc = p.upper_bc;
  a.dT = p.dT; a.dtau = p.dtau;
  return a;
}

// `steps` implicit steps on a.nsys = a.nsl·B systems: in0 → ... → the epilogue set in `a`.
static cudaError_t streamed_steps(StreamedState &st, const PassArgs &a, const float *in0, int steps,
                                  cudaStream_t s, int *nl) {
  {  // aggregates of the first forward pass
    PassArgs g = a;
    g.ntiles = st.ntiles;
    g.in = in0;
    g.aggT_next = st.aggT[0];
    g.aggL_next = st.aggL[0];
    k_agg0<<<(unsigned)((unsigned long long)a.nsys * st.ntiles), kSNT, 0, s>>>(g);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    *nl += 1;
  }
  const int S = pick_S(a.nsl, a.epi);
  for (int m = 0; m < steps; ++m) {
    PassArgs f = a;
    f.step_m = m;
    f.in = (m == 0) ? in0 : st.X;
    f.out = st.Y;
    f.epi = EPI_X;
    cudaError_t e = launch_pass(st, 0, m > 0, true, f, S, s);
    if (e != cudaSuccess) return e;
    PassArgs g = a;
    g.step_m = m;
    g.in = st.Y;
    g.out = st.X;
    if (m < steps - 1) g.epi = EPI_X;
    e = launch_pass(st, 1, true, m < steps - 1, g, S, s);
    if (e != cudaSuccess) return e;
    *nl += 2;
  }
  return cudaSuccess;
}

cudaError_t streamed_sweep(StreamedState &st, const StreamedProblem &p, const StreamedJob &j, cudaStream_t s,
                           int *nl) {
  PassArgs a = pass_base(p);
  const size_t off = (size_t)j.ln0 * p.B * p.Mp;
  a.nsl = j.nsl;
  a.nsys = j.nsl * p.B;
  a.n_base = j.n_base;
  a.ln0 = j.ln0;
  a.epi = EPI_SWEEP;
  a.Gh = j.Gh ? j.Gh + off : nullptr;
  a.D = j.D ? j.D + off : nullptr;
  a.Fk = j.Fk;
  a.Fout = j.Fout;
  a.fk_sys_lo = a.fk_sys_hi = 0;
  if (j.fk_ln >= j.ln0) {
    a.fk_sys_lo = (j.fk_ln - j.ln0) * p.B;
    a.fk_sys_hi = a.fk_sys_lo + p.B;
  }
  return streamed_steps(st, a, j.U + off, p.steps, s, nl);
}

cudaError_t streamed_chain(StreamedState &st, const StreamedProblem &p, const StreamedChainJob &j,
                           cudaStream_t s, int *nl) {
  if (j.Fcopy) {
    dim3 grid((p.M + 255) / 256, p.B);
    k_copy_delta<<<grid, 256, 0, s>>>(j.U + (size_t)j.ln0 * j.ustride, j.Fcopy, p.M, p.Mp,
                                      j.partials ? j.partials + (size_t)j.ln0 * p.B * j.nch * 2 : nullptr, p.B,
                                      j.nch);
    *nl += 1;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  PassArgs a = pass_base(p);
  a.nsl = 1;
  a.nsys = p.B;
  a.epi = EPI_CHAIN;
  a.nch = j.nch;
  for (int ln = j.ln0; ln < j.ln1; ++ln) {
    a.n_base = j.n_base + ln;  // one slice per launch: system s = instance b, ln0 = 0
    a.ln0 = 0;
    a.Unext = j.U + (size_t)(ln + 1) * j.ustride;
    a.GhW = j.Gh ? j.Gh + (size_t)ln * p.B * p.Mp : nullptr;
    a.Dc = j.D ? j.D + (size_t)ln * p.B * p.Mp : nullptr;
    a.partials = j.partials ? j.partials + (size_t)(ln + 1) * p.B * j.nch * 2 : nullptr;
    cudaError_t e = streamed_steps(st, a, j.U + (size_t)ln * j.ustride, p.steps, s, nl);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace pr
#endif  // PR_FINE_STREAMED_IMPL
