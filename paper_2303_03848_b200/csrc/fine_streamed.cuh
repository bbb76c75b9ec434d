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
// one slice, up to 2^20 points and more) is cut into tiles of kSTile points and
// threads of kSPS points; one pass is one kernel launch.
//
// Pre-aggregated, pre-scanned passes.  Over a thread's kSPS points a recurrence
// is an affine map v ↦ A_t + B_t·v of the value entering the thread.  B_t is a
// product of constant factors; A_t is linear in the pass's *input* — the
// previous pass's *output*.  So every pass, as it produces its outputs, also
// accumulates the next pass's A_t, scans them over its tile (in the next pass's
// direction) and publishes, per thread, the exclusive in-tile prefix E_t and,
// per tile, the tile total.  A pass therefore starts with everything it needs
// in memory: the value entering thread t is  v_t = E_t + P_t·y_tile  (P_t, the
// product of the preceding threads' multipliers, is a host table), where
// y_tile, the value entering the tile, is the composition of its
// predecessors' tile totals (look-back).  Each thread then runs its recurrence
// once, from the exact entering value: no waiting on other CTAs, no second pass.
// The first pass of a slice takes its aggregates from k_agg0.
//
// Look-back truncation.  Tile i composes the totals of predecessors
// i−1 … i−W_i only, W_i (host-computed) being the first window whose
// multiplier product falls below kLookbackEps: tiles further back change the
// entering value by < kLookbackEps·|y| (eight orders below fp64 rounding).
// Fixed composition orders → bitwise reproducible results.
//
// Factors.  Only 1/p_j is stored (fp64, interleaved); m̃_j and c_j are formed
// from the closed-form off-diagonals l_j = −dτ(a_j−b_j), u_j = −dτ(a_j+b_j)
// (a_j = σ²j²/2, b_j = rj/2, j = 1..M).
//
// Two kernels.  k_pass_res (the middle passes of a sweep, interleaved in and
// out) is persistent: each CTA takes a contiguous tile-major range of items
// (one tile of SP·H systems sharing a factor set), keeps the tile's factors in
// shared memory across its items, and streams the items' state in with bulk
// async copies (cp.async.bulk + mbarrier) NST items ahead.  k_streamed_pass
// (first pass of a slice from natural-layout rows, last pass with the
// epilogues, and chain mode) is one CTA per tile with register-resident data.
// Per point and pass: 4 B state read + 4 B written (HBM).
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
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
  const double *thrP;            // [2][nsets][Mt/kSPS] P_t: product of the multipliers of the threads
                                 //   preceding t in its tile, in the pass direction (dir 0: Π(−m̃), 1: Π(−c))
  const double *tileB;           // [2][nsets][ntiles] tile multiplier, indexed by scan position
  const int *tileW;              // [2][nsets][ntiles] look-back window (predecessors)
  // θ < 1 (Crank–Nicolson, NEXT-1): explicit part and the tile-edge corrections of forward passes
  const double *ecoef;           // [nsets][3] (1−θ)dτσ²/2, (1−θ)dτr/2, (1−θ)dτr
  const double *PL;              // [nsets][Mt/kSPS] Π(−m̃_k), k = tile start+1 … thread start−1
  const double *tileL;           // [nsets][ntiles] Π(−m̃_k), k = tile start+1 … tile end
};

struct StreamedState {
  float *X = nullptr, *Y = nullptr;   // [nsys][Mt] ping-pong state (interleaved)
  double *aggT[2] = {nullptr, nullptr};  // [nsys][Mt/kSPS] E_t: [0] read by forward passes, [1] by backward
  double *aggL[2] = {nullptr, nullptr};  // [nsys][ntiles] tile totals (tile index)
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
  int nsl, ngroups;          // systems s = ls·B + b (ls < nsl); group g ↔ (b = g % B, slices (g/B)·SG …)
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
  double theta;              // θ-step (1: implicit Euler)
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
  double dT, dtau, theta;
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

constexpr int kNW = kSNT / 32;  // warps per tile

template <int DIR>
__device__ __forceinline__ double shfl_prev(double v, int d) {
  return DIR == 0 ? __shfl_up_sync(0xffffffffu, v, d) : __shfl_down_sync(0xffffffffu, v, d);
}

// dτ(a_M+b_M)·[θ g(τ_{m+1}) + (1−θ) g(τ_m)] of step m of slice n, g the upper boundary value
// (reading Q3); θ = 1: dτ(a_M+b_M)·g(τ_{m+1}).
__device__ __forceinline__ double g_up(const PassArgs &a, int b, double tau) {
  return a.upper_bc ? 0.0 : a.Lb[b] - a.Kb[b] * exp(-a.rb[b] * tau);
}
__device__ __forceinline__ double bc_term(const PassArgs &a, int b, int n, int m) {
  const double tau0 = n * a.dT + m * a.dtau;
  const double g1 = g_up(a, b, tau0 + a.dtau);
  if (a.theta == 1.0) return a.bcoef[b] * g1;
  return a.bcoef[b] * (a.theta * g1 + (1.0 - a.theta) * g_up(a, b, tau0));
}

// Explicit part of a θ-step (θ < 1) at 0-based point j (J = j+1): x_j + (1−θ)dτ(A x)_j with
// (1−θ)dτ(a_j−b_j, −(2a_j+r), a_j+b_j) = (q−p, −(2q+er), q+p), q = e0 J², p = e1 J.
struct Expl {
  double e0, e1, er;
  __device__ __forceinline__ double rhs(double J, double xm, double x0, double xp) const {
    const double q = e0 * J * J, pp = e1 * J;
    return fma(q, (xm - 2.0 * x0) + xp, fma(pp, xp - xm, fma(-er, x0, x0)));
  }
  __device__ __forceinline__ double lower(double J) const { return J * fma(e0, J, -e1); }  // q − p
  __device__ __forceinline__ double upper(double J) const { return J * fma(e0, J, e1); }   // q + p
};
__device__ __forceinline__ Expl load_expl(const PassArgs &a, int set) {
  return Expl{__ldg(a.f.ecoef + 3 * set), __ldg(a.f.ecoef + 3 * set + 1), __ldg(a.f.ecoef + 3 * set + 2)};
}
// The pass input at 0-based point j of system s (interleaved or natural rows).
template <bool IN_IL>
__device__ __forceinline__ float in_at(const PassArgs &a, int s, int j) {
  return IN_IL ? a.in[(size_t)s * a.Mt + il_index((size_t)j)] : a.in[(size_t)s * a.Mp + j];
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

// Inclusive warp scan, in the order of direction D, of SP maps (A_q, B) with a common B.
// Returns the exclusive values (eA_q, eB) of the lane; lane 31 (scan order) holds the totals.
template <int D, int SP>
__device__ __forceinline__ void warp_scan(double (&A)[SP], double &B, double (&eA)[SP], double &eB, int lane) {
  const int sl = D == 0 ? lane : 31 - lane;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    // lanes without a predecessor at distance d keep their map: coefficient 0 / factor 1 instead
    // of a select per value (fma(0, finite, A) = A exactly)
    const bool has = sl >= d;
    const double pB = shfl_prev<D>(B, d);
    const double Bm = has ? B : 0.0;
#pragma unroll
    for (int q = 0; q < SP; ++q) A[q] = fma(Bm, shfl_prev<D>(A[q], d), A[q]);
    B *= has ? pB : 1.0;
  }
  eB = shfl_prev<D>(B, 1);
#pragma unroll
  for (int q = 0; q < SP; ++q) eA[q] = shfl_prev<D>(A[q], 1);
  if (sl == 0) {
    eB = 1.0;
#pragma unroll
    for (int q = 0; q < SP; ++q) eA[q] = 0.0;
  }
}

// Composition of the nearest predecessors' tile totals (lane l: distance base+l+1),
// fixed tree (deterministic).  Warp-level; result in lane 0.
__device__ __forceinline__ void compose_window(double &mA, double &mB, int lane) {
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double oA = __shfl_down_sync(0xffffffffu, mA, d);
    const double oB = __shfl_down_sync(0xffffffffu, mB, d);
    const bool take = (lane & (2 * d - 1)) == 0;  // masked as in warp_scan (bitwise the same)
    mA = fma(take ? mB : 0.0, oA, mA);
    mB *= take ? oB : 1.0;
  }
}

// The value entering the tile at scan position `pos` of system s, composing the window from
// predecessor distance base0+1 on onto (accA, accB).  Warp-level; result in lane 0.
template <int DIR, bool CN = false, bool IN_IL = true>
__device__ __forceinline__ double look_back(const PassArgs &a, int s, int pos, int set, int lane, int base0,
                                            double accA, double accB) {
  const size_t tb = ((size_t)DIR * a.nsets + set) * a.ntiles;
  const double *agg = a.aggL_cur + (size_t)s * a.ntiles;
  const int W = pos > 0 ? __ldg(a.f.tileW + tb + pos) : 0;
  for (int base = base0; base < W; base += 32) {
    const int k = base + lane;
    double mA = 0.0, mB = 1.0;
    if (k < W) {
      const int p = pos - 1 - k;
      mA = agg[DIR == 0 ? p : a.ntiles - 1 - p];
      mB = __ldg(a.f.tileB + tb + p);
      if (CN && DIR == 0) {
        // the producer built tile p's total without the stencil terms that reach across its
        // edges (x_{j0−1}, x_{j1+1}: other tiles' outputs); add them from this pass's input
        const Expl ex = load_expl(a, set);
        const double *ip = a.f.ip + (size_t)set * a.Mt;
        const int j0 = p * kSTile, j1 = j0 + kSTile - 1;  // a predecessor tile is full (j1+1 < M)
        double dl = 0.0;
        if (j0 > 0) dl = __ldg(ip + il_index(j0)) * ex.lower((double)(j0 + 1)) * (double)in_at<IN_IL>(a, s, j0 - 1);
        const double dr = __ldg(ip + il_index(j1)) * ex.upper((double)(j1 + 1)) * (double)in_at<IN_IL>(a, s, j1 + 1);
        mA = fma(dl, __ldg(a.f.tileL + (size_t)set * a.ntiles + p), mA) + dr;
      }
    }
    compose_window(mA, mB, lane);
    accA = fma(accB, mA, accA);
    accB *= mB;
  }
  return accA;
}

// ---------------------------------------------------------------- k_agg0
// Aggregates of the first (forward) pass of a slice, from its natural-layout input rows:
// A_t = Σ_i r_i/p_i Π_{k>i}(−m̃_k) (w-form forward map of the thread), scanned over the tile.
// θ < 1: r = the explicit part of step 0; its stencil terms across the tile's edges are left out
// (the consumer adds them, see look_back), exactly as a backward pass producing these aggregates.
template <bool CN>
__global__ void __launch_bounds__(kSNT) k_agg0(PassArgs a) {
  __shared__ double tot[kNW][2];
  const int s = blockIdx.x % a.nsys, tile = blockIdx.x / a.nsys;
  const int b = s % a.B, ln = a.ln0 + s / a.B, set = a.fset[b];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
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
  double xr = 0.0, xl = 0.0;  // neighbours across the thread's chunk (0 across the tile's edges)
  Expl ex{0.0, 0.0, 0.0};
  if (CN) {
    ex = load_expl(a, set);
    const float *row = a.in + (size_t)s * a.Mp;
    if (t > 0 && j0 > 0) xl = row[j0 - 1];
    if (t < kSNT - 1 && j0 + kSPS < a.M) xr = row[j0 + kSPS];
  }
  double A[1] = {0.0}, P = 1.0;
#pragma unroll
  for (int i = kSPS - 1; i >= 0; --i) {
    const int j = j0 + i;
    double mt, cj;
    factors<true>(c0, c1, J0 + i, ipv[i], j, a.M, mt, cj);
    double r = (double)x[i];
    if (CN) {
      r = ex.rhs(J0 + i, i > 0 ? (double)x[i - 1] : xl, (double)x[i], i < kSPS - 1 ? (double)x[i + 1] : xr);
      if (j >= a.M) r = 0.0;
    }
    if (j == a.M - 1) r += bcv;
    A[0] = fma(r * ipv[i], P, A[0]);
    P *= -mt;
  }
  double eA[1], eB;
  warp_scan<0, 1>(A, P, eA, eB, lane);
  if (lane == 31) { tot[w][0] = A[0]; tot[w][1] = P; }
  __syncthreads();
  double wA = 0.0;
  for (int k = 0; k < w; ++k) wA = fma(tot[k][1], wA, tot[k][0]);
  const size_t nthr = (size_t)a.Mt / kSPS;
  a.aggT_next[(size_t)s * nthr + (size_t)tile * kSNT + t] = fma(eB, wA, eA[0]);
  if (t == 0) {
    double T = 0.0;
    for (int k = 0; k < kNW; ++k) T = fma(tot[k][1], T, tot[k][0]);
    a.aggL_next[(size_t)s * a.ntiles + tile] = T;
  }
}

// ---------------------------------------------------------------- k_streamed_pass
// One CTA per tile of SP systems (the same tile of SP consecutive slices of one instance), data
// in registers.  Used for the first pass of a slice (natural input), the last pass (epilogues)
// and chain mode.  NEXT: also publish the next pass's aggregates.
// CN (θ < 1): a forward pass first forms the explicit part r = (I + (1−θ)dτA)x of its input
// (neighbours across threads by shuffle / shared memory, across the tile's edges from memory),
// and adds the stencil terms its producer could not see (tile-edge neighbours) to the entering
// values; a backward pass with NEXT builds the next forward map from r of its rounded outputs,
// leaving out the terms across the tile's edges.
template <int DIR, bool IN_IL, bool OUT_IL, bool NEXT, int SP, bool CN>
__global__ void __launch_bounds__(kSNT) k_streamed_pass(PassArgs a) {
  constexpr int ND = 1 - DIR;  // direction of the next pass
  static_assert(SP <= kNW, "one look-back warp per system");
  __shared__ double s_yin[SP];
  __shared__ float s_edge[2][kNW][SP];
  __shared__ double s_dl[SP];
  __shared__ double tot[kNW][SP + 1];
  __shared__ double red[2 * kNW];
  const int g = (int)(blockIdx.x % a.ngroups);
  const int pos = (int)(blockIdx.x / a.ngroups);       // position in scan order
  const int tile = DIR == 0 ? pos : a.ntiles - 1 - pos;
  const int b = g % a.B;
  const int ls0 = (g / a.B) * SP;                      // first launch-local slice of the group
  const int set = a.fset[b];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int j0 = tile * kSTile + t * kSPS;
  const size_t til = (size_t)tile * kSTile + t;   // interleaved offset of this thread's point 0
  const size_t nthr = (size_t)a.Mt / kSPS;
  const size_t thr = (size_t)tile * kSNT + t;     // thread index within the system
  int sys[SP];
  bool ok[SP];
#pragma unroll
  for (int q = 0; q < SP; ++q) {
    ok[q] = ls0 + q < a.nsl;
    sys[q] = ok[q] ? (ls0 + q) * a.B + b : (ls0 * a.B + b);  // invalid → duplicate of the first (no stores)
  }

  // ---- issue every load
  double E[SP];
#pragma unroll
  for (int q = 0; q < SP; ++q) E[q] = a.aggT_cur[(size_t)sys[q] * nthr + thr];
  const double P = __ldg(a.f.thrP + ((size_t)DIR * a.nsets + set) * nthr + thr);
  float x[SP][kSPS];
#pragma unroll
  for (int q = 0; q < SP; ++q) {
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
  const double J0 = (double)(j0 + 1);
  // ---- CN forward pass: neighbours of the thread's chunk in the input
  Expl ex{0.0, 0.0, 0.0};
  float xl[SP], xr[SP];
  double PLt = 0.0;
  if (CN) ex = load_expl(a, set);
  if (CN && DIR == 0) {
    PLt = __ldg(a.f.PL + (size_t)set * nthr + thr);
#pragma unroll
    for (int q = 0; q < SP; ++q) {
      xl[q] = __shfl_up_sync(0xffffffffu, x[q][kSPS - 1], 1);
      xr[q] = __shfl_down_sync(0xffffffffu, x[q][0], 1);
      if (lane == 31) s_edge[0][w][q] = x[q][kSPS - 1];
      if (lane == 0) s_edge[1][w][q] = x[q][0];
      if (t == 0) {
        xl[q] = j0 > 0 ? in_at<IN_IL>(a, sys[q], j0 - 1) : 0.0f;
        s_dl[q] = j0 > 0 ? ipv[0] * ex.lower(J0) * (double)xl[q] : 0.0;
      }
      if (t == kSNT - 1) xr[q] = j0 + kSPS < a.M ? in_at<IN_IL>(a, sys[q], j0 + kSPS) : 0.0f;
    }
  }
  // ---- the value entering the tile (one warp per system)
  if (w >= kNW - SP) {
    const int q = kNW - 1 - w;
    const double y = pos > 0 ? look_back<DIR, CN, IN_IL>(a, sys[q], pos, set, lane, 0, 0.0, 1.0) : 0.0;
    if (lane == 0) s_yin[q] = y;
  }
  __syncthreads();
  if (CN && DIR == 0) {
#pragma unroll
    for (int q = 0; q < SP; ++q) {
      if (lane == 0 && w > 0) xl[q] = s_edge[0][w - 1][q];
      if (lane == 31 && w < kNW - 1) xr[q] = s_edge[1][w + 1][q];
    }
  }
  double v[SP];
#pragma unroll
  for (int q = 0; q < SP; ++q) {
    v[q] = fma(P, s_yin[q], E[q]);
    // the tile's left-edge stencil term, missing from its producer's prefixes
    if (CN && DIR == 0 && t > 0) v[q] = fma(s_dl[q], PLt, v[q]);
  }
  // ---- the recurrence, once, from the exact entering value; next pass's map on the fly
  double An[SP], Pn = 1.0;
#pragma unroll
  for (int q = 0; q < SP; ++q) An[q] = 0.0;
  double pv[SP];  // CN: the previous point's input value
#pragma unroll
  for (int q = 0; q < SP; ++q) pv[q] = CN && DIR == 0 ? (double)xl[q] : 0.0;
  auto run = [&](auto edge_tag) {
    constexpr bool EDGE = decltype(edge_tag)::value;
    double bcv[SP];
#pragma unroll
    for (int q = 0; q < SP; ++q) {
      bcv[q] = 0.0;
      if (EDGE && j0 <= a.M - 1 && a.M - 1 < j0 + kSPS && (DIR == 0 || NEXT))
        bcv[q] = bc_term(a, b, a.n_base + a.ln0 + ls0 + q, a.step_m + DIR);
    }
#pragma unroll
    for (int ii = 0; ii < kSPS; ++ii) {
      const int i = DIR == 0 ? ii : kSPS - 1 - ii;
      const int j = j0 + i;
      double mt, cj;
      factors<EDGE>(c0, c1, J0 + i, ipv[i], j, a.M, mt, cj);
#pragma unroll
      for (int q = 0; q < SP; ++q) {
        if (DIR == 0) {
          double r = (double)x[q][i];
          if (CN) {
            const double cur = r;
            r = ex.rhs(J0 + i, pv[q], cur, i < kSPS - 1 ? (double)x[q][i + 1] : (double)xr[q]);
            if (EDGE && j >= a.M) r = 0.0;
            pv[q] = cur;
          }
          if (EDGE && j == a.M - 1) r += bcv[q];
          v[q] = fma(-mt, v[q], r * ipv[i]);
          // backward map of the thread: x_{j0} = Σ_i w_i Π_{k<i}(−c_k) + Pn·x_{j0+kSPS}
          if (NEXT) An[q] = fma(v[q], Pn, An[q]);
        } else {
          v[q] = fma(-cj, v[q], (double)x[q][i]);
          // forward map of step m+1: w_last = Σ_i r_i/p_i Π_{k>i}(−m̃_k) + Pn·w_{j0−1}
          if (NEXT && !CN) {
            const double r = (EDGE && j == a.M - 1) ? v[q] + bcv[q] : v[q];
            An[q] = fma(r * ipv[i], Pn, An[q]);
          }
        }
        x[q][i] = (float)v[q];
      }
      if (NEXT && !(CN && DIR == 1)) Pn *= DIR == 0 ? -cj : -mt;
    }
  };
  // Aggregates use the unrounded outputs: the next pass then sees the recurrence applied to
  // inputs within fp32 rounding of the stored ones — the same perturbation storage makes.
  if (j0 == 0 || j0 + kSPS > a.M - 1) run(std::true_type{});
  else run(std::false_type{});
  if (CN && DIR == 1 && NEXT) {
    // next forward map from r = (I + (1−θ)dτA)x of the rounded outputs (tile-edge terms left out)
    float ol[SP], orr[SP];
#pragma unroll
    for (int q = 0; q < SP; ++q) {
      ol[q] = __shfl_up_sync(0xffffffffu, x[q][kSPS - 1], 1);
      orr[q] = __shfl_down_sync(0xffffffffu, x[q][0], 1);
      if (lane == 31) s_edge[0][w][q] = x[q][kSPS - 1];
      if (lane == 0) s_edge[1][w][q] = x[q][0];
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < SP; ++q) {
      if (lane == 0) ol[q] = w > 0 ? s_edge[0][w - 1][q] : 0.0f;
      if (lane == 31) orr[q] = w < kNW - 1 ? s_edge[1][w + 1][q] : 0.0f;
    }
    const bool has_bc = j0 <= a.M - 1 && a.M - 1 < j0 + kSPS;
    double bcn[SP];
#pragma unroll
    for (int q = 0; q < SP; ++q) bcn[q] = has_bc ? bc_term(a, b, a.n_base + a.ln0 + ls0 + q, a.step_m + 1) : 0.0;
#pragma unroll
    for (int i = kSPS - 1; i >= 0; --i) {
      const int j = j0 + i;
      double mt, cj;
      factors<true>(c0, c1, J0 + i, ipv[i], j, a.M, mt, cj);
#pragma unroll
      for (int q = 0; q < SP; ++q) {
        double r = ex.rhs(J0 + i, i > 0 ? (double)x[q][i - 1] : (double)ol[q], (double)x[q][i],
                          i < kSPS - 1 ? (double)x[q][i + 1] : (double)orr[q]);
        if (j >= a.M) r = 0.0;
        if (j == a.M - 1) r += bcn[q];
        An[q] = fma(r * ipv[i], Pn, An[q]);
      }
      Pn *= -mt;
    }
  }
  // ---- stores / epilogues
  if (OUT_IL) {
#pragma unroll
    for (int q = 0; q < SP; ++q) {
      if (!ok[q]) continue;
      float *op = a.out + (size_t)sys[q] * a.Mt + til;
#pragma unroll
      for (int i = 0; i < kSPS; ++i) __stcs(op + i * kSNT, x[q][i]);
    }
  } else if (a.epi == EPI_SWEEP) {
#pragma unroll
    for (int q = 0; q < SP; ++q) {
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
  } else {  // EPI_CHAIN (SP = 1): g = x; Ĝ_n = g; U_{n+1} = g + D_n; δ partial against the old U_{n+1}
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
      if (lane == 0) { red[2 * w] = num; red[2 * w + 1] = den; }
      __syncthreads();
      if (t == 0) {
        num = 0.0; den = 0.0;
        for (int q2 = 0; q2 < kNW; ++q2) { num += red[2 * q2]; den += red[2 * q2 + 1]; }
        double *pp = a.partials + ((size_t)b * a.nch + tile) * 2;
        pp[0] = num;
        pp[1] = den;
      }
    }
  }
  // ---- the next pass's aggregates: exclusive in-tile prefixes E_t and tile totals
  if (NEXT) {
    double eA[SP], eB;
    warp_scan<ND, SP>(An, Pn, eA, eB, lane);
    const int sl = ND == 0 ? lane : 31 - lane;
    const int sw = ND == 0 ? w : kNW - 1 - w;
    if (sl == 31) {
#pragma unroll
      for (int q = 0; q < SP; ++q) tot[sw][q] = An[q];
      tot[sw][SP] = Pn;
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < SP; ++q) {
      double wA = 0.0;
      for (int k = 0; k < sw; ++k) wA = fma(tot[k][SP], wA, tot[k][q]);
      if (ok[q]) a.aggT_next[(size_t)sys[q] * nthr + thr] = fma(eB, wA, eA[q]);
    }
    if (t == 0) {
#pragma unroll
      for (int q = 0; q < SP; ++q) {
        double T = 0.0;
        for (int k = 0; k < kNW; ++k) T = fma(tot[k][SP], T, tot[k][q]);
        if (ok[q]) a.aggL_next[(size_t)sys[q] * a.ntiles + tile] = T;
      }
    }
  }
}

// ---------------------------------------------------------------- k_pass_res (persistent)
// Items in tile-major order (item = pos·ngroups + g); a group is SP·H systems sharing a factor
// set: half h (kSNT threads) runs systems h·SP … h·SP+SP−1 of the group, SP per thread.
// One __syncthreads per item: the look-back broadcast and scan scratch are double-buffered by
// item parity, and an item's next-pass prefixes/totals and its stage refill are finished after
// the next item's barrier (which every warp reaches only once done with the item).
template <int SP, int H, int NST>
struct ResSmem {
  double ip[kSTile], mt[kSTile], cj[kSTile];  // interleaved, this CTA's current tile
  float x[NST][H][SP][kSTile];
};
template <int SP, int H, int NST>
constexpr size_t res_smem_bytes() { return sizeof(ResSmem<SP, H, NST>); }

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "PR_MBAR_WAIT%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra PR_MBAR_WAIT%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Item cursor in tile-major order: item = pos·ngroups + g, g = lg·B + b.
template <int SG>
struct ResCursor {
  int pos, g, b, lg;
  __device__ __forceinline__ void init(const PassArgs &a, unsigned k) {
    const unsigned ng = (unsigned)a.ngroups;
    pos = (int)(k / ng);
    g = (int)(k - (unsigned)pos * ng);
    lg = g / a.B;
    b = g - lg * a.B;
  }
  __device__ __forceinline__ void step(const PassArgs &a) {
    if (++g == a.ngroups) { g = 0; b = 0; lg = 0; ++pos; return; }
    if (++b == a.B) { b = 0; ++lg; }
  }
  template <int DIR>
  __device__ __forceinline__ int tile(const PassArgs &a) const { return DIR == 0 ? pos : a.ntiles - 1 - pos; }
  __device__ __forceinline__ bool ok(const PassArgs &a, int slot) const { return lg * SG + slot < a.nsl; }
  __device__ __forceinline__ int sys(const PassArgs &a, int slot) const {
    return (ok(a, slot) ? lg * SG + slot : lg * SG) * a.B + b;
  }
};

template <int DIR, int SP, int H, int NST>
__global__ void __launch_bounds__(H *kSNT) k_pass_res(PassArgs a) {
  constexpr int ND = 1 - DIR;
  constexpr int SG = SP * H;  // systems per item
  static_assert(SP <= kNW, "one look-back warp per system");
  extern __shared__ __align__(128) unsigned char res_smem_raw[];
  ResSmem<SP, H, NST> &sm = *reinterpret_cast<ResSmem<SP, H, NST> *>(res_smem_raw);
  __shared__ __align__(8) uint64_t full[NST];
  __shared__ double s_yin[2][H][SP];
  __shared__ double tot[2][H][kNW][SP + 1];
  const int t = threadIdx.x, h = t / kSNT, tt = t % kSNT, lane = t & 31, wl = tt >> 5;
  const unsigned nitems = (unsigned)a.ngroups * (unsigned)a.ntiles;
  const unsigned lo = (unsigned)(((unsigned long long)blockIdx.x * nitems) / gridDim.x);
  const unsigned hi = (unsigned)(((unsigned long long)(blockIdx.x + 1) * nitems) / gridDim.x);
  const size_t nthr = (size_t)a.Mt / kSPS;
  const int swN = ND == 0 ? wl : kNW - 1 - wl;  // this warp's position in the next pass's order
  const int slN = ND == 0 ? lane : 31 - lane;
  const uint64_t pol_stream = policy_evict_first();
  using Cur = ResCursor<SG>;

  Cur cur, nxt, iss, prev;
  auto issue = [&](int stage) {  // one thread: stream item `iss` into `stage`
    mbar_expect_tx(&full[stage], (uint32_t)(SG * kSTile * sizeof(float)));
    const int tile = iss.template tile<DIR>(a);
#pragma unroll
    for (int hh = 0; hh < H; ++hh)
#pragma unroll
      for (int q = 0; q < SP; ++q)
        bulk_g2s(sm.x[stage][hh][q], a.in + (size_t)iss.sys(a, hh * SP + q) * a.Mt + (size_t)tile * kSTile,
                 kSTile * sizeof(float), &full[stage], pol_stream);
    iss.step(a);
  };
  if (t == 0) {
    for (int i = 0; i < NST; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cur.init(a, lo);
  nxt = cur;
  iss = cur;
  prev = cur;
  if (t == 0)
    for (int i = 0; i < NST && lo + i < hi; ++i) issue(i);
  // register prefetch of an item's entering prefixes and look-back operands (own systems),
  // two items ahead (slot i & 1); the factor set of the last instance seen is cached
  struct Pre {
    double E[SP], P, LA, LB;
    int W, set;
  };
  Pre pre[2];
  int cb = -1, cset = 0;
  auto prefetch = [&](const Cur &c, Pre &r) {
    const int tile = c.template tile<DIR>(a);
    if (c.b != cb) {
      cb = c.b;
      cset = a.fset[cb];
    }
    const int set = cset;
    r.set = set;
    const size_t thr = (size_t)tile * kSNT + tt;
#pragma unroll
    for (int q = 0; q < SP; ++q) r.E[q] = a.aggT_cur[(size_t)c.sys(a, h * SP + q) * nthr + thr];
    r.P = __ldg(a.f.thrP + ((size_t)DIR * a.nsets + set) * nthr + thr);
    r.LA = 0.0;
    r.LB = 1.0;
    r.W = 0;
    if (wl >= kNW - SP && c.pos > 0) {
      const int q = kNW - 1 - wl;
      const size_t tb = ((size_t)DIR * a.nsets + set) * a.ntiles;
      r.W = __ldg(a.f.tileW + tb + c.pos);
      const int p = c.pos - 1 - lane;
      if (p >= 0) {
        r.LA = a.aggL_cur[(size_t)c.sys(a, h * SP + q) * a.ntiles + (DIR == 0 ? p : a.ntiles - 1 - p)];
        r.LB = __ldg(a.f.tileB + tb + p);
      }
    }
  };
  // the previous item's next-pass aggregates (its warp totals are in tot[pb]), after a barrier
  double qA[SP], qB = 1.0;  // the previous item's exclusive in-warp prefixes (next-pass order)
  auto finish = [&](int pb) {
    const int tile = prev.template tile<DIR>(a);
#pragma unroll
    for (int q = 0; q < SP; ++q) {
      double wA = 0.0;
      for (int k = 0; k < swN; ++k) wA = fma(tot[pb][h][k][SP], wA, tot[pb][h][k][q]);
      const int slot = h * SP + q;
      if (prev.ok(a, slot))
        a.aggT_next[(size_t)prev.sys(a, slot) * nthr + (size_t)tile * kSNT + tt] = fma(qB, wA, qA[q]);
    }
    if (tt < SP) {  // thread q of each half: tile total of system q
      const int q = tt;
      double T = 0.0;
      for (int k = 0; k < kNW; ++k) T = fma(tot[pb][h][k][SP], T, tot[pb][h][k][q]);
      const int slot = h * SP + q;
      if (prev.ok(a, slot)) a.aggL_next[(size_t)prev.sys(a, slot) * a.ntiles + tile] = T;
    }
  };
  if (lo < hi) prefetch(nxt, pre[0]);
  nxt.step(a);
  if (lo + 1 < hi) prefetch(nxt, pre[1]);
  nxt.step(a);
  int fac_tile = -1, fac_set = -1;
  int n = 0;
  for (unsigned k = lo; k < hi; ++k, ++n) {
    const int stage = n % NST;
    const int pb = n & 1;
    const uint32_t parity = (uint32_t)(n / NST) & 1u;
    double E[SP], P, LA, LB;
    int W, set;
    if (n & 1) {  // (static register indexing)
#pragma unroll
      for (int q = 0; q < SP; ++q) E[q] = pre[1].E[q];
      P = pre[1].P; LA = pre[1].LA; LB = pre[1].LB; W = pre[1].W; set = pre[1].set;
      if (k + 2 < hi) prefetch(nxt, pre[1]);
    } else {
#pragma unroll
      for (int q = 0; q < SP; ++q) E[q] = pre[0].E[q];
      P = pre[0].P; LA = pre[0].LA; LB = pre[0].LB; W = pre[0].W; set = pre[0].set;
      if (k + 2 < hi) prefetch(nxt, pre[0]);
    }
    if (k + 2 < hi) nxt.step(a);
    const int tile = cur.template tile<DIR>(a);
    // ---- the value entering the tile (warps kNW−SP … kNW−1 of each half)
    if (wl >= kNW - SP) {
      const int q = kNW - 1 - wl;
      double mA = lane < W ? LA : 0.0, mB = lane < W ? LB : 1.0;
      compose_window(mA, mB, lane);
      double y = mA;
      if (W > 32) y = look_back<DIR>(a, cur.sys(a, h * SP + q), cur.pos, set, lane, 32, mA, mB);  // rare
      if (lane == 0) s_yin[pb][h][q] = y;
    }
    __syncthreads();  // the barrier of the item
    if (n > 0) {
      finish(pb ^ 1);
      if (t == 0 && k - 1 + NST < hi) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue((n - 1) % NST);
      }
    }
    // ---- factors of a new tile: 1/p from global, m̃ and c derived once
    if (tile != fac_tile || set != fac_set) {
      const double *ipg = a.f.ip + (size_t)set * a.Mt + (size_t)tile * kSTile;
      const double c0 = __ldg(a.f.coef + 2 * set), c1 = __ldg(a.f.coef + 2 * set + 1);
      constexpr int kPer = kSTile / (H * kSNT);
      double ipl[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) ipl[u] = __ldg(ipg + t + u * H * kSNT);  // all loads in flight
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int e = t + u * H * kSNT;
        const int j = tile * kSTile + (e % kSNT) * kSPS + e / kSNT;
        double mtj, cjj;
        factors<true>(c0, c1, (double)(j + 1), ipl[u], j, a.M, mtj, cjj);
        sm.ip[e] = ipl[u];
        sm.mt[e] = mtj;
        sm.cj[e] = cjj;
      }
      fac_tile = tile;
      fac_set = set;
      __syncthreads();
    }
    double v[SP];
#pragma unroll
    for (int q = 0; q < SP; ++q) v[q] = fma(P, s_yin[pb][h][q], E[q]);
    // ---- the recurrence over the staged tile
    mbar_wait(&full[stage], parity);
    const int j0 = tile * kSTile + tt * kSPS;
    const double *ips = sm.ip + tt, *mts = sm.mt + tt, *cjs = sm.cj + tt;
    double An[SP], Pn = 1.0;
    float *op[SP];
    const float *xs[SP];
    bool okq[SP];
#pragma unroll
    for (int q = 0; q < SP; ++q) {
      An[q] = 0.0;
      okq[q] = cur.ok(a, h * SP + q);
      op[q] = a.out + (size_t)cur.sys(a, h * SP + q) * a.Mt + (size_t)tile * kSTile + tt;
      xs[q] = sm.x[stage][h][q] + tt;
    }
    auto run = [&](auto bc_tag) {
      constexpr bool BC = decltype(bc_tag)::value;
      double bcv[SP];
      const int ibc = a.M - 1 - j0;
#pragma unroll
      for (int q = 0; q < SP; ++q)
        bcv[q] = BC ? bc_term(a, cur.b, a.n_base + a.ln0 + cur.lg * SG + h * SP + q, a.step_m + DIR) : 0.0;
#pragma unroll
      for (int ii = 0; ii < kSPS; ++ii) {
        const int i = DIR == 0 ? ii : kSPS - 1 - ii;
        const double ipj = ips[i * kSNT];
        const double f1 = DIR == 0 ? mts[i * kSNT] : cjs[i * kSNT];  // this pass's multiplier
        const double f2 = DIR == 0 ? cjs[i * kSNT] : mts[i * kSNT];  // the next pass's
#pragma unroll
        for (int q = 0; q < SP; ++q) {
          const double xin = (double)xs[q][i * kSNT];
          if (DIR == 0) {
            const double r = (BC && i == ibc) ? xin + bcv[q] : xin;
            v[q] = fma(-f1, v[q], r * ipj);
            An[q] = fma(v[q], Pn, An[q]);
          } else {
            v[q] = fma(-f1, v[q], xin);
            const double r = (BC && i == ibc) ? v[q] + bcv[q] : v[q];
            An[q] = fma(r * ipj, Pn, An[q]);
          }
          if (okq[q]) __stcs(op[q] + i * kSNT, (float)v[q]);
        }
        Pn *= -f2;
      }
    };
    if (j0 <= a.M - 1 && a.M - 1 < j0 + kSPS) run(std::true_type{});
    else run(std::false_type{});
    // ---- next-pass aggregates: in-warp scan now, cross-warp after the next barrier
    warp_scan<ND, SP>(An, Pn, qA, qB, lane);
    if (slN == 31) {
#pragma unroll
      for (int q = 0; q < SP; ++q) tot[pb][h][swN][q] = An[q];
      tot[pb][h][swN][SP] = Pn;
    }
    prev = cur;
    cur.step(a);
  }
  __syncthreads();
  if (n > 0) finish((n - 1) & 1);
}

// ---------------------------------------------------------------- k_pass_res2 (persistent, paired)
// As k_pass_res, but each thread runs two adjacent 16-point chunks ("virtual threads" v0 = 2t',
// v1 = 2t'+1 of the tile's kSNT) of each of its systems.  Both chunks' entering values are known
// up front (E_v + P_v·y_tile), so they are two independent recurrences (twice the ILP per
// thread); their inputs, outputs and factors are adjacent in the interleaved layout (float2 /
// double2 accesses: half the load/store instructions); and the per-item work (prefetch, scans,
// folds, cursors) is paid once per 32 points instead of 16.  The next pass's maps of the two
// chunks are composed in-thread (in the next pass's order) before the warp scan, and expanded
// back to per-chunk prefixes after it, so the aggregates keep the per-16-point format every
// other K2 kernel reads.
constexpr int kHT = kSNT / 2;   // threads per half (one tile of SP systems)
constexpr int kNW2 = kHT / 32;  // warps per half

template <int DIR, int SP, int H, int NST>
__global__ void __launch_bounds__(H *kHT) k_pass_res2(PassArgs a) {
  constexpr int ND = 1 - DIR;
  constexpr int SG = SP * H;  // systems per item
  constexpr int CF = ND == 0 ? 0 : 1;  // the chunk the next pass visits first
  static_assert(SP <= kNW2, "one look-back warp per system");
  extern __shared__ __align__(128) unsigned char res_smem_raw[];
  ResSmem<SP, H, NST> &sm = *reinterpret_cast<ResSmem<SP, H, NST> *>(res_smem_raw);
  __shared__ __align__(8) uint64_t full[NST];
  __shared__ double s_yin[2][H][SP];
  __shared__ double tot[2][H][kNW2][SP + 1];
  const int t = threadIdx.x, h = t / kHT, tt = t % kHT, lane = t & 31, wl = tt >> 5;
  const int v0 = 2 * tt;  // this thread's first chunk (index among the tile's kSNT chunks)
  const unsigned nitems = (unsigned)a.ngroups * (unsigned)a.ntiles;
  const unsigned lo = (unsigned)(((unsigned long long)blockIdx.x * nitems) / gridDim.x);
  const unsigned hi = (unsigned)(((unsigned long long)(blockIdx.x + 1) * nitems) / gridDim.x);
  const size_t nthr = (size_t)a.Mt / kSPS;
  const int swN = ND == 0 ? wl : kNW2 - 1 - wl;
  const int slN = ND == 0 ? lane : 31 - lane;
  const uint64_t pol_stream = policy_evict_first();
  using Cur = ResCursor<SG>;

  Cur cur, nxt, iss, prev;
  auto issue = [&](int stage) {
    mbar_expect_tx(&full[stage], (uint32_t)(SG * kSTile * sizeof(float)));
    const int tile = iss.template tile<DIR>(a);
#pragma unroll
    for (int hh = 0; hh < H; ++hh)
#pragma unroll
      for (int q = 0; q < SP; ++q)
        bulk_g2s(sm.x[stage][hh][q], a.in + (size_t)iss.sys(a, hh * SP + q) * a.Mt + (size_t)tile * kSTile,
                 kSTile * sizeof(float), &full[stage], pol_stream);
    iss.step(a);
  };
  if (t == 0) {
    for (int i = 0; i < NST; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cur.init(a, lo);
  nxt = cur;
  iss = cur;
  prev = cur;
  if (t == 0)
    for (int i = 0; i < NST && lo + i < hi; ++i) issue(i);
  struct Pre {
    double E[2][SP], P[2], LA, LB, LA2, LB2;  // look-back operands: predecessors 1-32 and 33-64
    int W, set;
  };
  Pre pre[2];
  int cb = -1, cset = 0;
  auto prefetch = [&](const Cur &c, Pre &r) {
    const int tile = c.template tile<DIR>(a);
    if (c.b != cb) {
      cb = c.b;
      cset = a.fset[cb];
    }
    const int set = cset;
    r.set = set;
    const size_t thr = (size_t)tile * kSNT + v0;
#pragma unroll
    for (int q = 0; q < SP; ++q) {
      const double2 e = *reinterpret_cast<const double2 *>(a.aggT_cur + (size_t)c.sys(a, h * SP + q) * nthr + thr);
      r.E[0][q] = e.x;
      r.E[1][q] = e.y;
    }
    const double2 pp = __ldg(reinterpret_cast<const double2 *>(a.f.thrP + ((size_t)DIR * a.nsets + set) * nthr + thr));
    r.P[0] = pp.x;
    r.P[1] = pp.y;
    r.LA = 0.0;
    r.LB = 1.0;
    r.LA2 = 0.0;
    r.LB2 = 1.0;
    r.W = 0;
    if (wl >= kNW2 - SP && c.pos > 0) {
      const int q = kNW2 - 1 - wl;
      const size_t tb = ((size_t)DIR * a.nsets + set) * a.ntiles;
      r.W = __ldg(a.f.tileW + tb + c.pos);
      const double *aggl = a.aggL_cur + (size_t)c.sys(a, h * SP + q) * a.ntiles;
      const int p = c.pos - 1 - lane;
      if (p >= 0) {
        r.LA = aggl[DIR == 0 ? p : a.ntiles - 1 - p];
        r.LB = __ldg(a.f.tileB + tb + p);
      }
      // the second window too: a third of the C3 tiles look back 33-48 tiles (multipliers
      // within 5e-4 of 1 at the top of the grid), which otherwise costs a synchronous load
      // round trip in front of the item's barrier
      const int p2 = p - 32;
      if (p2 >= 0) {
        r.LA2 = aggl[DIR == 0 ? p2 : a.ntiles - 1 - p2];
        r.LB2 = __ldg(a.f.tileB + tb + p2);
      }
    }
  };
  // the previous item's exclusive pair prefixes (next-pass order) and its first chunks' maps
  double qA[SP], qB = 1.0, fA[SP], fB = 1.0;
  auto finish = [&](int pb) {
    const int tile = prev.template tile<DIR>(a);
#pragma unroll
    for (int q = 0; q < SP; ++q) {
      double wA = 0.0;
      for (int k = 0; k < swN; ++k) wA = fma(tot[pb][h][k][SP], wA, tot[pb][h][k][q]);
      const double eF = fma(qB, wA, qA[q]);  // entering the pair = entering its first chunk
      const double eS = fma(fB, eF, fA[q]);  // entering the second chunk
      const int slot = h * SP + q;
      if (prev.ok(a, slot))
        *reinterpret_cast<double2 *>(a.aggT_next + (size_t)prev.sys(a, slot) * nthr + (size_t)tile * kSNT + v0) =
            CF == 0 ? make_double2(eF, eS) : make_double2(eS, eF);
    }
    if (tt < SP) {
      const int q = tt;
      double T = 0.0;
      for (int k = 0; k < kNW2; ++k) T = fma(tot[pb][h][k][SP], T, tot[pb][h][k][q]);
      const int slot = h * SP + q;
      if (prev.ok(a, slot)) a.aggL_next[(size_t)prev.sys(a, slot) * a.ntiles + tile] = T;
    }
  };
  if (lo < hi) prefetch(nxt, pre[0]);
  nxt.step(a);
  if (lo + 1 < hi) prefetch(nxt, pre[1]);
  nxt.step(a);
  int fac_tile = -1, fac_set = -1;
  int n = 0;
  for (unsigned k = lo; k < hi; ++k, ++n) {
    const int stage = n % NST;
    const int pb = n & 1;
    const uint32_t parity = (uint32_t)(n / NST) & 1u;
    double E[2][SP], P[2], LA, LB, LA2, LB2;
    int W, set;
    if (n & 1) {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        P[c] = pre[1].P[c];
#pragma unroll
        for (int q = 0; q < SP; ++q) E[c][q] = pre[1].E[c][q];
      }
      LA = pre[1].LA; LB = pre[1].LB; LA2 = pre[1].LA2; LB2 = pre[1].LB2; W = pre[1].W; set = pre[1].set;
      if (k + 2 < hi) prefetch(nxt, pre[1]);
    } else {
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        P[c] = pre[0].P[c];
#pragma unroll
        for (int q = 0; q < SP; ++q) E[c][q] = pre[0].E[c][q];
      }
      LA = pre[0].LA; LB = pre[0].LB; LA2 = pre[0].LA2; LB2 = pre[0].LB2; W = pre[0].W; set = pre[0].set;
      if (k + 2 < hi) prefetch(nxt, pre[0]);
    }
    if (k + 2 < hi) nxt.step(a);
    const int tile = cur.template tile<DIR>(a);
    if (wl >= kNW2 - SP) {
      const int q = kNW2 - 1 - wl;
      double mA = lane < W ? LA : 0.0, mB = lane < W ? LB : 1.0;
      compose_window(mA, mB, lane);
      double y = mA;
      if (W > 32) {  // (warp-uniform) predecessors 33-64 from the prefetched second window
        double mA2 = lane + 32 < W ? LA2 : 0.0, mB2 = lane + 32 < W ? LB2 : 1.0;
        compose_window(mA2, mB2, lane);
        y = fma(mB, mA2, mA);
        if (W > 64) y = look_back<DIR>(a, cur.sys(a, h * SP + q), cur.pos, set, lane, 64, y, mB * mB2);  // rare
      }
      if (lane == 0) s_yin[pb][h][q] = y;
    }
    __syncthreads();  // the barrier of the item
    if (n > 0) {
      finish(pb ^ 1);
      if (t == 0 && k - 1 + NST < hi) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue((n - 1) % NST);
      }
    }
    if (tile != fac_tile || set != fac_set) {
      const double *ipg = a.f.ip + (size_t)set * a.Mt + (size_t)tile * kSTile;
      const double c0 = __ldg(a.f.coef + 2 * set), c1 = __ldg(a.f.coef + 2 * set + 1);
      constexpr int kPer = kSTile / (H * kHT);
      double ipl[kPer];
#pragma unroll
      for (int u = 0; u < kPer; ++u) ipl[u] = __ldg(ipg + t + u * H * kHT);
#pragma unroll
      for (int u = 0; u < kPer; ++u) {
        const int e = t + u * H * kHT;
        const int j = tile * kSTile + (e % kSNT) * kSPS + e / kSNT;
        double mtj, cjj;
        factors<true>(c0, c1, (double)(j + 1), ipl[u], j, a.M, mtj, cjj);
        sm.ip[e] = ipl[u];
        sm.mt[e] = mtj;
        sm.cj[e] = cjj;
      }
      fac_tile = tile;
      fac_set = set;
      __syncthreads();
    }
    double v[2][SP];
#pragma unroll
    for (int c = 0; c < 2; ++c)
#pragma unroll
      for (int q = 0; q < SP; ++q) v[c][q] = fma(P[c], s_yin[pb][h][q], E[c][q]);
    mbar_wait(&full[stage], parity);
    const int j0 = tile * kSTile + v0 * kSPS;  // chunk 1 starts at j0 + kSPS
    const double *ips = sm.ip + v0, *mts = sm.mt + v0, *cjs = sm.cj + v0;
    double An[2][SP], Pn[2] = {1.0, 1.0};
    float *op[SP];
    const float *xs[SP];
    bool okq[SP];
#pragma unroll
    for (int q = 0; q < SP; ++q) {
      An[0][q] = 0.0;
      An[1][q] = 0.0;
      okq[q] = cur.ok(a, h * SP + q);
      op[q] = a.out + (size_t)cur.sys(a, h * SP + q) * a.Mt + (size_t)tile * kSTile + v0;
      xs[q] = sm.x[stage][h][q] + v0;
    }
    auto run = [&](auto bc_tag) {
      constexpr bool BC = decltype(bc_tag)::value;
      double bcv[SP];
      const int ibc0 = a.M - 1 - j0, ibc1 = ibc0 - kSPS;
#pragma unroll
      for (int q = 0; q < SP; ++q)
        bcv[q] = BC ? bc_term(a, cur.b, a.n_base + a.ln0 + cur.lg * SG + h * SP + q, a.step_m + DIR) : 0.0;
#pragma unroll
      for (int ii = 0; ii < kSPS; ++ii) {
        const int i = DIR == 0 ? ii : kSPS - 1 - ii;
        const double2 ipj = *reinterpret_cast<const double2 *>(ips + i * kSNT);
        const double2 mtj = *reinterpret_cast<const double2 *>(mts + i * kSNT);
        const double2 cjj = *reinterpret_cast<const double2 *>(cjs + i * kSNT);
        const double ipc[2] = {ipj.x, ipj.y};
        const double f1[2] = {DIR == 0 ? mtj.x : cjj.x, DIR == 0 ? mtj.y : cjj.y};  // this pass's multiplier
        const double f2[2] = {DIR == 0 ? cjj.x : mtj.x, DIR == 0 ? cjj.y : mtj.y};  // the next pass's
#pragma unroll
        for (int q = 0; q < SP; ++q) {
          const float2 xin2 = *reinterpret_cast<const float2 *>(xs[q] + i * kSNT);
          const double xin[2] = {(double)xin2.x, (double)xin2.y};
          float o[2];
#pragma unroll
          for (int c = 0; c < 2; ++c) {
            const bool isbc = BC && i == (c == 0 ? ibc0 : ibc1);
            if (DIR == 0) {
              const double r = isbc ? xin[c] + bcv[q] : xin[c];
              v[c][q] = fma(-f1[c], v[c][q], r * ipc[c]);
              An[c][q] = fma(v[c][q], Pn[c], An[c][q]);
            } else {
              v[c][q] = fma(-f1[c], v[c][q], xin[c]);
              const double r = isbc ? v[c][q] + bcv[q] : v[c][q];
              An[c][q] = fma(r * ipc[c], Pn[c], An[c][q]);
            }
            o[c] = (float)v[c][q];
          }
          if (okq[q]) __stcs(reinterpret_cast<float2 *>(op[q] + i * kSNT), make_float2(o[0], o[1]));
        }
        Pn[0] *= -f2[0];
        Pn[1] *= -f2[1];
      }
    };
    if (j0 <= a.M - 1 && a.M - 1 < j0 + 2 * kSPS) run(std::true_type{});
    else run(std::false_type{});
    // next-pass map of the pair (first chunk CF, then the other), in-warp scan now
    constexpr int CS = 1 - CF;
    double pA[SP];
#pragma unroll
    for (int q = 0; q < SP; ++q) {
      pA[q] = fma(Pn[CS], An[CF][q], An[CS][q]);
      fA[q] = An[CF][q];
    }
    double pB = Pn[CS] * Pn[CF];
    fB = Pn[CF];
    warp_scan<ND, SP>(pA, pB, qA, qB, lane);
    if (slN == 31) {
#pragma unroll
      for (int q = 0; q < SP; ++q) tot[pb][h][swN][q] = pA[q];
      tot[pb][h][swN][SP] = pB;
    }
    prev = cur;
    cur.step(a);
  }
  __syncthreads();
  if (n > 0) finish((n - 1) & 1);
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

// ---------------------------------------------------------------- host drivers
static int env_int(const char *name, int dflt) {
  const char *e = getenv(name);
  return e ? atoi(e) : dflt;
}
// tuning overrides: PR_K2_PIPE=0 (no persistent kernel), PR_K2_SP (1|2), PR_K2_H (1|2), PR_K2_STAGES (2|3|4)
struct ResConfig {
  int enabled, sp, h, nst, pair;
};
static ResConfig res_config() {
  static const ResConfig c = [] {
    ResConfig r;
    r.enabled = env_int("PR_K2_PIPE", 1);
    r.sp = env_int("PR_K2_SP", 2) == 1 ? 1 : 2;
    r.h = env_int("PR_K2_H", 2);
    r.h = r.h == 1 ? 1 : r.h == 4 ? 4 : 2;
    const int n = env_int("PR_K2_STAGES", 2);  // (SP, H, NST) = (2, 2, 2): best measured at C3
    r.nst = n == 3 || n == 4 ? n : 2;
    r.pair = env_int("PR_K2_PAIR", 1);  // k_pass_res2 (two chunks per thread); 0: k_pass_res
    if (r.pair && r.sp == 2 && r.h == 4) r.h = 2;
    return r;
  }();
  return c;
}

template <int DIR, int SP, int H, int NST, bool PAIR>
static cudaError_t launch_res_dir(PassArgs a, cudaStream_t s) {
  static int grid_cap = 0;
  constexpr size_t smem = res_smem_bytes<SP, H, NST>();
  constexpr int nthreads = PAIR ? H * kHT : H * kSNT;
  auto kern = PAIR ? k_pass_res2<DIR, SP, H, NST> : k_pass_res<DIR, SP, H, NST>;
  if (grid_cap == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int dev = 0, nsm = 0, occ = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, nthreads, smem);
    if (e != cudaSuccess) return e;
    grid_cap = nsm * (occ > 0 ? occ : 1);
  }
  a.ngroups = a.B * ((a.nsl + SP * H - 1) / (SP * H));
  const long long nitems = (long long)a.ngroups * a.ntiles;
  const unsigned grid = (unsigned)(nitems < grid_cap ? nitems : grid_cap);
  kern<<<grid, nthreads, smem, s>>>(a);
  return cudaGetLastError();
}
template <int SP, int H, bool PAIR>
static cudaError_t launch_res_hp(int dir, const PassArgs &a, int nst, cudaStream_t s) {
  switch (nst) {
    case 2: return dir == 0 ? launch_res_dir<0, SP, H, 2, PAIR>(a, s) : launch_res_dir<1, SP, H, 2, PAIR>(a, s);
    case 4: return dir == 0 ? launch_res_dir<0, SP, H, 4, PAIR>(a, s) : launch_res_dir<1, SP, H, 4, PAIR>(a, s);
    default: return dir == 0 ? launch_res_dir<0, SP, H, 3, PAIR>(a, s) : launch_res_dir<1, SP, H, 3, PAIR>(a, s);
  }
}
template <int SP, int H>
static cudaError_t launch_res_h(int dir, const PassArgs &a, int nst, cudaStream_t s) {
  return res_config().pair ? launch_res_hp<SP, H, true>(dir, a, nst, s) : launch_res_hp<SP, H, false>(dir, a, nst, s);
}
static cudaError_t launch_res(int dir, const PassArgs &a, cudaStream_t s) {
  const ResConfig c = res_config();
  // no more systems per item than the launch has slices (an empty slot would stream a duplicate)
  int sp = c.sp, h = c.h;
  while (sp * h > a.nsl) {
    if (sp > 1) sp = 1;
    else h = 1;
  }
  if (sp == 2) return h == 2 ? launch_res_h<2, 2>(dir, a, c.nst, s) : launch_res_h<2, 1>(dir, a, c.nst, s);
  if (h == 4 && c.pair) return launch_res_hp<1, 4, true>(dir, a, c.nst, s);
  return h >= 2 ? launch_res_h<1, 2>(dir, a, c.nst, s) : launch_res_h<1, 1>(dir, a, c.nst, s);
}

template <int SP, bool CN>
static void launch_tile_cn(int dir, bool in_il, bool next, const PassArgs &a, cudaStream_t s) {
  const unsigned grid = (unsigned)((unsigned long long)a.ngroups * a.ntiles);
  if (dir == 0) {
    if (in_il) k_streamed_pass<0, true, true, true, SP, CN><<<grid, kSNT, 0, s>>>(a);
    else k_streamed_pass<0, false, true, true, SP, CN><<<grid, kSNT, 0, s>>>(a);
  } else if (a.epi == EPI_X) {
    if (next) k_streamed_pass<1, true, true, true, SP, CN><<<grid, kSNT, 0, s>>>(a);
    else k_streamed_pass<1, true, true, false, SP, CN><<<grid, kSNT, 0, s>>>(a);
  } else {
    k_streamed_pass<1, true, false, false, SP, CN><<<grid, kSNT, 0, s>>>(a);
  }
}
template <int SP>
static void launch_tile(int dir, bool in_il, bool next, const PassArgs &a, cudaStream_t s) {
  if (a.theta != 1.0) launch_tile_cn<SP, true>(dir, in_il, next, a, s);
  else launch_tile_cn<SP, false>(dir, in_il, next, a, s);
}

// Forward passes read aggregates [0] and write [1]; backward passes read [1] and write [0].
static cudaError_t launch_pass(StreamedState &st, int dir, bool in_il, bool next, PassArgs a, cudaStream_t s) {
  a.ntiles = st.ntiles;
  a.aggT_cur = st.aggT[dir];
  a.aggL_cur = st.aggL[dir];
  a.aggT_next = st.aggT[1 - dir];
  a.aggL_next = st.aggL[1 - dir];
  // The persistent kernel pays off when several items share each tile's factors (C3: 16 groups
  // of 4 slices); a lone system (the serial fine solve) runs one CTA per tile.
  if (in_il && next && a.epi == EPI_X && res_config().enabled && a.B * a.nsl >= 16 && a.theta == 1.0)
    return launch_res(dir, a, s);
  const int sp = (a.epi != EPI_CHAIN && a.nsl >= 2) ? 2 : 1;
  a.ngroups = a.B * ((a.nsl + sp - 1) / sp);
  if (sp == 2) launch_tile<2>(dir, in_il, next, a, s);
  else launch_tile<1>(dir, in_il, next, a, s);
  return cudaGetLastError();
}

static PassArgs pass_base(const StreamedProblem &p) {
  PassArgs a;
  memset(&a, 0, sizeof a);
  a.M = p.M; a.Mp = p.Mp; a.B = p.B; a.Mt = streamed_Mt(p.M); a.nsets = p.nsets;
  a.f = p.f; a.fset = p.fset;
  a.bcoef = p.bcoef; a.Lb = p.L; a.Kb = p.K; a.rb = p.r; a.upper_bc = p.upper_bc;
  a.dT = p.dT; a.dtau = p.dtau; a.theta = p.theta;
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
    const unsigned grid = (unsigned)((unsigned long long)a.nsys * st.ntiles);
    if (a.theta != 1.0) k_agg0<true><<<grid, kSNT, 0, s>>>(g);
    else k_agg0<false><<<grid, kSNT, 0, s>>>(g);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    *nl += 1;
  }
  for (int m = 0; m < steps; ++m) {
    PassArgs f = a;
    f.step_m = m;
    f.in = (m == 0) ? in0 : st.X;
    f.out = st.Y;
    f.epi = EPI_X;
    cudaError_t e = launch_pass(st, 0, m > 0, true, f, s);
    if (e != cudaSuccess) return e;
    PassArgs g = a;
    g.step_m = m;
    g.in = st.Y;
    g.out = st.X;
    if (m < steps - 1) g.epi = EPI_X;
    e = launch_pass(st, 1, true, m < steps - 1, g, s);
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
