// fine_resident.cuh — K1: on-chip implicit-Euler propagator for M ≤ 2048 (kResidentMaxM).
//
// One "system" = one (instance, slice) state vector of M interior points
// (§3.2), owned by NT threads with P consecutive points each.
// The state, the fp64 LU factors of M_f = I − dτA and every scan coefficient
// live in registers for all implicit steps of the slice; HBM is touched once
// per slice (load U_n, store F̂_n or D_n = F̂_n − Ĝ_n).
//
// Per θ-step (implicit Euler θ=1 by reading Q1, Crank–Nicolson θ=1/2 = NEXT-1) the
// constant-matrix solve (I − θdτA) x⁺ = (I + (1−θ)dτA) x + dτ(a_M+b_M)[θg(τ⁺) + (1−θ)g(τ)] e_M
// first forms the explicit right-hand side (θ < 1: a 3-point stencil, neighbours across threads
// by shuffle and across warps through shared memory) and then splits into two first-order
// linear recurrences (forward elimination y_j = r_j − m_j y_{j−1}, back
// substitution x_j = y_j/p_j − (u_j/p_j) x_{j+1}).  Each is evaluated as a
// chunked scan of affine maps v ↦ A + B·v: a sequential pass over the
// thread's P points, a Hillis–Steele warp scan of the A parts (the B parts
// are products of constant factors, so every level coefficient is
// precomputed once per kernel), a fold over the ≤16 warp totals in shared
// memory, and a fix-up with precomputed prefix products.
#include <cuda_runtime.h>
#include <stdint.h>

#ifndef PR_FINE_RESIDENT_ARGS
#define PR_FINE_RESIDENT_ARGS
namespace pr {

constexpr unsigned kFull = 0xffffffffu;

struct ResidentArgs {
  int M, Mp, B;
  // factors of the scheme used by this launch: [nsets][Mp] each (fp64)
  const double *fm, *fip, *fcu;
  const double *zz;         // θ = 1: zig-zag factors [6][nsets][Mp] (ip, nml, ncu, iq, ncl, nmu)
  int nsets;
  int use_zz;               // 1: the kernels run the zig-zag form (host choice, pipe.cu consistent)
  const int *fset;          // [B] factor-set index per instance
  const double *bcoef;      // [B] dτ (a_M + b_M) of this scheme (boundary term of row M)
  double theta;             // θ of the θ-step (1: implicit Euler; 1/2: Crank–Nicolson)
  const double *ecoef;      // θ < 1: [nsets][3] (1−θ)dτσ²/2, (1−θ)dτr/2, (1−θ)dτr (explicit part)
  const double *Lb, *Kb, *rb;
  int upper_bc;             // 0 asymptotic call value, 1 zero
  double dT, dtau;          // slice length, implicit step
  int steps;                // implicit steps per slice
  int n_base;               // global index of local slice 0
  // ---- sweep mode (independent slices; blockIdx → (slice, instance))
  int ln0, nsl;             // local slices [ln0, ln0+nsl)
  const float *U;           // [Nloc+1][B][Mp]   inputs U_n
  const float *Gh;          // [Nloc][B][Mp]     Ĝ_n (D mode)
  float *D;                 // [Nloc][B][Mp]     D_n = F̂_n − Ĝ_n
  float *Fk;                // [B][Mp]           F̂ of local slice fk_ln
  int fk_ln;                // -1: none
  float *Fout;              // non-null: F̂ of every job → Fout[(ln-ln0)][B][Mp] (test hook)
  // ---- chain mode (serial in n, one system per instance)
  float *Uw;                // writable rows Uw + ln·ustride: reads row c_ln0, writes row ln+1
  size_t ustride;           // elements between slice rows of Uw (0 → one row updated in place)
  float *GhW;               // nullable: Ĝ_n = g
  const float *Dc;          // nullable: U_{n+1} = g + D_n
  const float *Fcopy;       // nullable: first U[c_ln0] := Fcopy (+ δ partial)
  int c_ln0, c_ln1;
  double *partials;         // nullable: [(ln)·B + b]·nch + 0 → (num, den)
  int nch;
};

}  // namespace pr
#endif  // PR_FINE_RESIDENT_ARGS

#if !defined(PR_ARGS_ONLY) && !defined(PR_FINE_RESIDENT_IMPL)
#define PR_FINE_RESIDENT_IMPL
// The barrier of one system's threads: the whole CTA by default; a translation unit whose CTAs
// hold other work besides the system (pipe.cu) defines it as a named barrier first.
#ifndef PR_TRI_SYNC
#define PR_TRI_SYNC() __syncthreads()
#endif
namespace pr {
__device__ __forceinline__ double g_upper(const ResidentArgs &a, int b, double tau) {
  // Reading Q3: V(L, τ) = L − K e^{−rτ} (default) or 0 (paper-literal P:161)
  return a.upper_bc ? 0.0 : a.Lb[b] - a.Kb[b] * exp(-a.rb[b] * tau);
}

template <int P, int NT, bool CN = false, bool ZZ = false>
struct Tri {
  static constexpr int NW = NT / 32;
  static constexpr int kShm = 6 * NW + 2;  // doubles of shared scratch per system
  double nm[P], ip[P], ncu[P], qf[P], qb[P];
  double cfL[5], cbL[5];
  double cf_exc, cb_exc;
  // cross-warp fold, NW ≥ 4: warp totals are combined as one weighted sum (the weights — products
  // of the constant warp multipliers between warp q and this warp — precomputed by fold_setup)
  static constexpr bool kParFold = NW >= 4;
  double cfw[kParFold ? NW : 1], cbw[kParFold ? NW : 1];
  double e0, e1, er, J0;  // CN: explicit-part coefficients, J of the thread's first point
  int lane, w, M, j0;

  // shared layout per system: ctf[NW], ctb[NW], sy[2][NW], (CN) edge values [2][NW]
  __device__ void setup(const ResidentArgs &a, int set, int t, double *sh) {
    lane = t & 31;
    w = t >> 5;
    M = a.M;
    j0 = t * P;
    J0 = (double)(j0 + 1);
    if (CN) {
      e0 = a.ecoef[3 * set];
      e1 = a.ecoef[3 * set + 1];
      er = a.ecoef[3 * set + 2];
    }
    const double *fm = a.fm + (size_t)set * a.Mp;
    const double *fip = a.fip + (size_t)set * a.Mp;
    const double *fcu = a.fcu + (size_t)set * a.Mp;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int j = t * P + i;
      if (j < a.M) {
        nm[i] = -fm[j];
        ip[i] = fip[j];
        ncu[i] = -fcu[j];
      } else {  // identity padding rows
        nm[i] = 0.0;
        ip[i] = 1.0;
        ncu[i] = 0.0;
      }
    }
    double c = 1.0;
#pragma unroll
    for (int i = 0; i < P; ++i) { c *= nm[i]; qf[i] = c; }
    c = 1.0;
#pragma unroll
    for (int i = P - 1; i >= 0; --i) { c *= ncu[i]; qb[i] = c; }
    // warp-scan level coefficients (products of constant maps)
    double cf = qf[P - 1], cb = qb[0];
#pragma unroll
    for (int l = 0; l < 5; ++l) {
      const int d = 1 << l;
      const double pf = __shfl_up_sync(kFull, cf, d);
      const double pb = __shfl_down_sync(kFull, cb, d);
      cfL[l] = (lane >= d) ? cf : 0.0;
      cbL[l] = (lane + d <= 31) ? cb : 0.0;
      if (lane >= d) cf *= pf;
      if (lane + d <= 31) cb *= pb;
    }
    const double ef = __shfl_up_sync(kFull, cf, 1);
    const double eb = __shfl_down_sync(kFull, cb, 1);
    cf_exc = (lane == 0) ? 1.0 : ef;
    cb_exc = (lane == 31) ? 1.0 : eb;
    if (NW > 1) {
      if (lane == 31) sh[w] = cf;       // total forward product of warp w
      if (lane == 0) sh[NW + w] = cb;   // total backward product of warp w
    }
  }
  // after the barrier that follows setup: fold weights Π_{q<r<w} B_r (forward), Π_{w<r<q} B_r (backward)
  __device__ void fold_setup(const double *sh) {
    if (!kParFold) return;
#pragma unroll
    for (int q = 0; q < NW; ++q) {
      double pf = 1.0, pb = 1.0;
      for (int r = q + 1; r < w; ++r) pf *= sh[r];
      for (int r = w + 1; r < q; ++r) pb *= sh[NW + r];
      cfw[q] = (q < w) ? pf : 0.0;
      cbw[q] = (q > w) ? pb : 0.0;
    }
  }
  // fixed-order pairwise sum of the weighted warp totals
  __device__ __forceinline__ double fold(const double (&c)[kParFold ? NW : 1], const double *sy) const {
    double t[NW];
#pragma unroll
    for (int q = 0; q < NW; ++q) t[q] = c[q] * sy[q];
#pragma unroll
    for (int d = 1; d < NW; d <<= 1)
#pragma unroll
      for (int q = 0; q + d < NW; q += 2 * d) t[q] += t[q + d];
    return t[0];
  }

  // One implicit step in place on x[P] (fp64).  bc_i: point index inside this thread that
  // receives the boundary term (−1 if none); bcg = dτ(a_M+b_M) g(τ⁺).
  // Explicit part (CN): x ← (I + (1−θ)dτA) x, with V_0 = 0 below row 1; the upper boundary value
  // is in the tabulated boundary term.  (a_j−b_j, −(2a_j+r), a_j+b_j)(1−θ)dτ = (q−p, −(2q+er), q+p)
  // with q = e0 J², p = e1 J.  Rows beyond M (padding) stay 0.
  __device__ __forceinline__ void explicit_part(double (&x)[P], double *sh) {
    double xl = __shfl_up_sync(kFull, x[P - 1], 1), xr = __shfl_down_sync(kFull, x[0], 1);
    if (NW > 1) {
      double *xb = sh + 4 * NW + 2;
      if (lane == 31) xb[w] = x[P - 1];
      if (lane == 0) xb[NW + w] = x[0];
      PR_TRI_SYNC();
      if (lane == 0) xl = (w > 0) ? xb[w - 1] : 0.0;
      if (lane == 31) xr = (w < NW - 1) ? xb[NW + w + 1] : 0.0;
    } else {
      if (lane == 0) xl = 0.0;
      if (lane == 31) xr = 0.0;
    }
    double prev = xl, cur = x[0];
    const bool pad = j0 + P > M;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const double nxt = (i < P - 1) ? x[i + 1] : xr;
      const double J = J0 + i;
      const double q = e0 * J * J, pp = e1 * J;
      double r = fma(q, (prev - 2.0 * cur) + nxt, fma(pp, nxt - prev, fma(-er, cur, cur)));
      if (pad && j0 + i >= M) r = 0.0;
      x[i] = r;
      prev = cur;
      cur = nxt;
    }
  }

  // BCL: row M is the thread's last point and bcg is 0 on every other thread (run_steps)
  template <bool BCL = false>
  __device__ __forceinline__ void step(double (&x)[P], int bc_i, double bcg, double *sh) {
    if (CN) explicit_part(x, sh);
    if (BCL) {
      x[P - 1] += bcg;
    } else {
#pragma unroll
      for (int i = 0; i < P; ++i)
        if (i == bc_i) x[i] += bcg;
    }
    // ---- forward elimination y_j = r_j − m_j y_{j−1}
#pragma unroll
    for (int i = 1; i < P; ++i) x[i] = fma(nm[i], x[i - 1], x[i]);
    double v = x[P - 1];
#pragma unroll
    for (int l = 0; l < 5; ++l) v = fma(cfL[l], __shfl_up_sync(kFull, v, 1 << l), v);
    double ve = __shfl_up_sync(kFull, v, 1);
    if (lane == 0) ve = 0.0;
    double in = 0.0;
    if (NW > 1) {
      double *sy = sh + 2 * NW;
      if (lane == 31) sy[w] = v;
      PR_TRI_SYNC();
      if constexpr (kParFold) {
        in = fold(cfw, sy);
      } else {
#pragma unroll 1
        for (int q = 0; q < w; ++q) in = fma(sh[q], in, sy[q]);
      }
    }
    const double yin = fma(cf_exc, in, ve);
#pragma unroll
    for (int i = 0; i < P; ++i) x[i] = fma(qf[i], yin, x[i]);
    // ---- back substitution x_j = y_j/p_j − (u_j/p_j) x_{j+1}
    x[P - 1] *= ip[P - 1];
#pragma unroll
    for (int i = P - 2; i >= 0; --i) x[i] = fma(ncu[i], x[i + 1], x[i] * ip[i]);
    v = x[0];
#pragma unroll
    for (int l = 0; l < 5; ++l) v = fma(cbL[l], __shfl_down_sync(kFull, v, 1 << l), v);
    ve = __shfl_down_sync(kFull, v, 1);
    if (lane == 31) ve = 0.0;
    in = 0.0;
    if (NW > 1) {
      double *sy = sh + 3 * NW;
      if (lane == 0) sy[w] = v;
      PR_TRI_SYNC();
      if constexpr (kParFold) {
        in = fold(cbw, sy);
      } else {
#pragma unroll 1
        for (int q = NW - 1; q > w; --q) in = fma(sh[NW + q], in, sy[q]);
      }
    }
    const double xin = fma(cb_exc, in, ve);
#pragma unroll
    for (int i = 0; i < P; ++i) x[i] = fma(qb[i], xin, x[i]);
  }
};

// ---------------------------------------------------------------- zig-zag implicit Euler (θ = 1)
// Implicit steps alternate between the LU and the UL factorisation of the same constant matrix
// M_f = I − dτA (both exact in fp64; constant coefficients).  Step m (LU when m is even)
// is an elimination sweep and a substitution sweep in opposite directions; the UL step runs them
// reversed.  So the substitution of step m and the elimination of step m+1 run in the SAME
// direction and are evaluated as one pass of a 2-state recurrence s_j = A_j s_{j∓1} + a_j (A_j
// lower triangular: the elimination consumes the substituted value of the same point):
//   ↓↓ (after an LU step):  x_j = w_j + ncu_j x_{j+1},   w̃_j = iq_j (x_j + bc_j) + nmu_j w̃_{j+1}
//   ↑↑ (after a UL step):   x_j = w̃_j + ncl_j x_{j−1},   w_j = ip_j (x_j + bc_j) + nml_j w_{j−1}
// (w = y/p, w̃ = ỹ/q: eliminations in divided form).  An n-step slice is n+1 passes: a lone
// elimination ↑, n−1 merged passes, a lone substitution — one chunked scan per implicit step
// instead of two (one barrier instead of two).  Each pass: the thread's P points from a zero
// entering state (chunk total), a Hillis–Steele warp scan of the 2-vector affine parts whose
// level coefficients (the lane's composite chunk maps, constant) are precomputed once per kernel,
// a serial fold over the ≤ NW preceding warp totals (warp maps constant, in shared memory), then
// the P points again from the exact entering state.  The lone passes use the same scan with one
// component zero (lower-triangular maps compose their diagonal entries independently).
template <int P, int NT>
struct Tri<P, NT, false, true> {
  static constexpr int NW = NT / 32;
  // shared per system: per direction [NW][2] pass totals + [NW][3] constant warp maps
  static constexpr int kShm = 10 * NW + 2;
  double ip[P], nml[P], ncu[P], iq[P], ncl[P], nmu[P];
  double uC[5][3], dC[5][3];  // level coefficients (lane's composite at the level, 0 without predecessor)
  double uX[3], dX[3];        // exclusive maps (identity for the first lane in pass order)
  double uA11, uA21, uA22, dA11, dA21, dA22;  // the thread's chunk maps
  int lane, w;

  __device__ void setup(const ResidentArgs &a, int set, int t, double *sh) {
    lane = t & 31;
    w = t >> 5;
    const size_t ks = (size_t)a.nsets * a.Mp;
    const double *z = a.zz + (size_t)set * a.Mp;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int j = t * P + i;
      const bool in = j < a.Mp;  // rows M..Mp−1 are identity in the table; beyond Mp too
      ip[i] = in ? z[j] : 1.0;
      nml[i] = in ? z[ks + j] : 0.0;
      ncu[i] = in ? z[2 * ks + j] : 0.0;
      iq[i] = in ? z[3 * ks + j] : 1.0;
      ncl[i] = in ? z[4 * ks + j] : 0.0;
      nmu[i] = in ? z[5 * ks + j] : 0.0;
    }
    // chunk maps, composed in pass order: M ← A_i · M
    double m11 = 1.0, m21 = 0.0, m22 = 1.0;
#pragma unroll
    for (int i = P - 1; i >= 0; --i) {  // ↓↓: A = [[ncu, 0], [iq·ncu, nmu]]
      const double a21 = iq[i] * ncu[i];
      m21 = a21 * m11 + nmu[i] * m21;
      m11 *= ncu[i];
      m22 *= nmu[i];
    }
    dA11 = m11, dA21 = m21, dA22 = m22;
    m11 = 1.0, m21 = 0.0, m22 = 1.0;
#pragma unroll
    for (int i = 0; i < P; ++i) {  // ↑↑: A = [[ncl, 0], [ip·ncl, nml]]
      const double a21 = ip[i] * ncl[i];
      m21 = a21 * m11 + nml[i] * m21;
      m11 *= ncl[i];
      m22 *= nml[i];
    }
    uA11 = m11, uA21 = m21, uA22 = m22;
    levels<true>(uA11, uA21, uA22, uC, uX, sh);
    levels<false>(dA11, dA21, dA22, dC, dX, sh);
  }
  // the warp scan of the (constant) chunk maps: per level the lane's composite before combining
  // (0 if it has no predecessor at that distance), the exclusive map, and the warp total
  template <bool UP>
  __device__ __forceinline__ void levels(double m11, double m21, double m22, double (&C)[5][3], double (&X)[3],
                                         double *sh) {
#pragma unroll
    for (int l = 0; l < 5; ++l) {
      const int d = 1 << l;
      const double p11 = UP ? __shfl_up_sync(kFull, m11, d) : __shfl_down_sync(kFull, m11, d);
      const double p21 = UP ? __shfl_up_sync(kFull, m21, d) : __shfl_down_sync(kFull, m21, d);
      const double p22 = UP ? __shfl_up_sync(kFull, m22, d) : __shfl_down_sync(kFull, m22, d);
      const bool has = UP ? lane >= d : lane + d <= 31;
      C[l][0] = has ? m11 : 0.0;
      C[l][1] = has ? m21 : 0.0;
      C[l][2] = has ? m22 : 0.0;
      if (has) {
        m21 = fma(m21, p11, m22 * p21);
        m11 *= p11;
        m22 *= p22;
      }
    }
    X[0] = UP ? __shfl_up_sync(kFull, m11, 1) : __shfl_down_sync(kFull, m11, 1);
    X[1] = UP ? __shfl_up_sync(kFull, m21, 1) : __shfl_down_sync(kFull, m21, 1);
    X[2] = UP ? __shfl_up_sync(kFull, m22, 1) : __shfl_down_sync(kFull, m22, 1);
    if (lane == (UP ? 0 : 31)) X[0] = 1.0, X[1] = 0.0, X[2] = 1.0;
    if (NW > 1 && lane == (UP ? 31 : 0)) {
      double *o = sh + (UP ? 0 : 5 * NW) + 2 * NW + 3 * w;  // constant warp map of this direction
      o[0] = m11, o[1] = m21, o[2] = m22;
    }
  }
  __device__ void fold_setup(const double *) {}

  // entering state of this thread's chunk for a pass in direction UP from the chunk totals (s1, s2)
  template <bool UP>
  __device__ __forceinline__ void enter(double s1, double s2, double *sh, double &e1, double &e2) const {
    const double(&C)[5][3] = UP ? uC : dC;
    const double(&X)[3] = UP ? uX : dX;
#pragma unroll
    for (int l = 0; l < 5; ++l) {
      const int d = 1 << l;
      const double q1 = UP ? __shfl_up_sync(kFull, s1, d) : __shfl_down_sync(kFull, s1, d);
      const double q2 = UP ? __shfl_up_sync(kFull, s2, d) : __shfl_down_sync(kFull, s2, d);
      s2 = fma(C[l][1], q1, fma(C[l][2], q2, s2));  // coefficient 0 without predecessor: s unchanged
      s1 = fma(C[l][0], q1, s1);
    }
    double xs1 = UP ? __shfl_up_sync(kFull, s1, 1) : __shfl_down_sync(kFull, s1, 1);
    double xs2 = UP ? __shfl_up_sync(kFull, s2, 1) : __shfl_down_sync(kFull, s2, 1);
    if (lane == (UP ? 0 : 31)) xs1 = 0.0, xs2 = 0.0;
    double i1 = 0.0, i2 = 0.0;
    if (NW > 1) {
      double *tot = sh + (UP ? 0 : 5 * NW);  // [NW][2] pass totals, then [NW][3] warp maps
      if (lane == (UP ? 31 : 0)) tot[2 * w] = s1, tot[2 * w + 1] = s2;
      PR_TRI_SYNC();
      const double *mp = tot + 2 * NW;
      // every warp's total and map loaded at once, then the serial composition over the
      // predecessors in pass order (predicated: the same fixed order for every warp)
      double t1[NW], t2[NW], a11[NW], a21[NW], a22[NW];
#pragma unroll
      for (int q = 0; q < NW; ++q) {
        t1[q] = tot[2 * q], t2[q] = tot[2 * q + 1];
        a11[q] = mp[3 * q], a21[q] = mp[3 * q + 1], a22[q] = mp[3 * q + 2];
      }
#pragma unroll
      for (int k = 0; k < NW; ++k) {
        const int q = UP ? k : NW - 1 - k;
        if (UP ? q < w : q > w) {
          i2 = fma(a21[q], i1, fma(a22[q], i2, t2[q]));
          i1 = fma(a11[q], i1, t1[q]);
        }
      }
    }
    e2 = fma(X[1], i1, fma(X[2], i2, xs2));
    e1 = fma(X[0], i1, xs1);
  }

  // the boundary term dτ(a_M+b_M)g of row M enters the elimination at one point of one thread.
  // BCL (M a multiple of P): row M is the last point of its thread, and bcg is passed as 0 to every
  // other thread, so the term is one add at point P−1 (no per-point compare and select); else
  // the general point test.
  template <bool BCL>
  __device__ __forceinline__ static double bc_add(int i, double x, int bc_i, double bcg) {
    if (BCL) return i == P - 1 ? x + bcg : x;
    return i == bc_i ? x + bcg : x;
  }
  // ↓↓: x (LU substitution of the previous step) and w̃ (UL elimination of this step, bc at bc_i)
  template <bool BCL>
  __device__ __forceinline__ void pass_down2(double (&v)[P], int bc_i, double bcg, double *sh) const {
    double x = 0.0, z = 0.0;
#pragma unroll
    for (int i = P - 1; i >= 0; --i) {
      x = fma(ncu[i], x, v[i]);
      z = fma(nmu[i], z, iq[i] * bc_add<BCL>(i, x, bc_i, bcg));
    }
    double e1, e2;
    enter<false>(x, z, sh, e1, e2);
    x = e1, z = e2;
#pragma unroll
    for (int i = P - 1; i >= 0; --i) {
      x = fma(ncu[i], x, v[i]);
      z = fma(nmu[i], z, iq[i] * bc_add<BCL>(i, x, bc_i, bcg));
      v[i] = z;
    }
  }
  // ↑↑: x (UL substitution of the previous step) and w (LU elimination of this step)
  template <bool BCL>
  __device__ __forceinline__ void pass_up2(double (&v)[P], int bc_i, double bcg, double *sh) const {
    double x = 0.0, z = 0.0;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      x = fma(ncl[i], x, v[i]);
      z = fma(nml[i], z, ip[i] * bc_add<BCL>(i, x, bc_i, bcg));
    }
    double e1, e2;
    enter<true>(x, z, sh, e1, e2);
    x = e1, z = e2;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      x = fma(ncl[i], x, v[i]);
      z = fma(nml[i], z, ip[i] * bc_add<BCL>(i, x, bc_i, bcg));
      v[i] = z;
    }
  }
  // lone LU elimination ↑ (first step of a slice): w_j = ip_j (x_j + bc_j) + nml_j w_{j−1}
  template <bool BCL>
  __device__ __forceinline__ void pass_up_elim(double (&v)[P], int bc_i, double bcg, double *sh) const {
    double z = 0.0;
#pragma unroll
    for (int i = 0; i < P; ++i) z = fma(nml[i], z, ip[i] * bc_add<BCL>(i, v[i], bc_i, bcg));
    double e1, e2;
    enter<true>(0.0, z, sh, e1, e2);  // first component 0: the (2,2) entries carry the scan
    z = e2;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      z = fma(nml[i], z, ip[i] * bc_add<BCL>(i, v[i], bc_i, bcg));
      v[i] = z;
    }
  }
  // lone substitution of the last step: LU (↓, x_j = w_j + ncu_j x_{j+1}) or UL (↑)
  template <bool UP>
  __device__ __forceinline__ void pass_sub(double (&v)[P], double *sh) const {
    double x = 0.0;
    if (UP) {
#pragma unroll
      for (int i = 0; i < P; ++i) x = fma(ncl[i], x, v[i]);
    } else {
#pragma unroll
      for (int i = P - 1; i >= 0; --i) x = fma(ncu[i], x, v[i]);
    }
    double e1, e2;
    enter<UP>(x, 0.0, sh, e1, e2);  // the (1,1) entries carry the scan; component 2 is ignored
    x = e1;
    if (UP) {
#pragma unroll
      for (int i = 0; i < P; ++i) v[i] = x = fma(ncl[i], x, v[i]);
    } else {
#pragma unroll
      for (int i = P - 1; i >= 0; --i) v[i] = x = fma(ncu[i], x, v[i]);
    }
  }
  // implicit step m of the slice (its elimination merged with the substitution of step m−1)
  template <bool BCL = false>
  __device__ __forceinline__ void zz_step(int m, double (&v)[P], int bc_i, double bcg, double *sh) const {
    if (m == 0) pass_up_elim<BCL>(v, bc_i, bcg, sh);
    else if (m & 1) pass_down2<BCL>(v, bc_i, bcg, sh);
    else pass_up2<BCL>(v, bc_i, bcg, sh);
  }
  // after the last step n−1: its substitution (LU ↓ when n−1 is even, UL ↑ when odd)
  __device__ __forceinline__ void zz_finish(int n, double (&v)[P], double *sh) const {
    if ((n - 1) & 1) pass_sub<true>(v, sh);
    else pass_sub<false>(v, sh);
  }
};

// Fixed-order block reduction of two doubles over the threads of one system (NT threads).
template <int NT>
__device__ __forceinline__ void sys_reduce2(double &a, double &b, int t, double *red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(kFull, a, o);
    b += __shfl_xor_sync(kFull, b, o);
  }
  if (NT > 32) {
    constexpr int NW = NT / 32;
    PR_TRI_SYNC();
    if ((t & 31) == 0) { red[2 * (t >> 5)] = a; red[2 * (t >> 5) + 1] = b; }
    PR_TRI_SYNC();
    a = 0.0; b = 0.0;
#pragma unroll 1
    for (int q = 0; q < NW; ++q) { a += red[2 * q]; b += red[2 * q + 1]; }
  }
}

constexpr int kBcChunk = 128;  // boundary terms tabulated per chunk of implicit steps

// All implicit steps of slice n.  The boundary term dτ(a_M+b_M)·g(τ_{m+1}) of each step needs an
// fp64 exp; it is tabulated in shared memory for kBcChunk steps at a time (one exp per thread)
// so no exp sits on the per-step critical path.
template <int P, int NT, bool CN, bool ZZ = false>
__device__ __forceinline__ void run_steps(Tri<P, NT, CN, ZZ> &tri, const ResidentArgs &a, int b, int n,
                                          int t, double (&x)[P], double *sh, double *bct) {
  const int bc_t = (a.M - 1) / P, bc_ip = (a.M - 1) % P;
  const int bc_i = (t == bc_t) ? bc_ip : -1;
  const bool bcl = bc_ip == P - 1;  // M a multiple of P (C1, C2, C4)
  const double coef = a.bcoef[b];
  const double tau0 = n * a.dT;
#pragma unroll 1
  for (int m0 = 0; m0 < a.steps; m0 += kBcChunk) {
    PR_TRI_SYNC();  // readers of the previous chunk are done
    for (int i = t; i < kBcChunk; i += NT) {
      const int m = m0 + i;
      if (m < a.steps) {
        const double gp = g_upper(a, b, (tau0 + m * a.dtau) + a.dtau);
        // dτ(a_M+b_M)[θ g(τ_{m+1}) + (1−θ) g(τ_m)]
        bct[i] = CN ? coef * (a.theta * gp + (1.0 - a.theta) * g_upper(a, b, tau0 + m * a.dtau)) : coef * gp;
      }
    }
    PR_TRI_SYNC();
    const int mend = min(a.steps - m0, kBcChunk);
#pragma unroll 1
    if constexpr (ZZ) {
      if (bcl) {  // row M is the last point of thread bc_t: bcg is 0 for every other thread
        for (int mm = 0; mm < mend; ++mm) tri.template zz_step<true>(m0 + mm, x, bc_i, bc_i >= 0 ? bct[mm] : 0.0, sh);
      } else {
        for (int mm = 0; mm < mend; ++mm) tri.zz_step(m0 + mm, x, bc_i, bc_i >= 0 ? bct[mm] : 0.0, sh);
      }
    } else {
      if (bcl) {
        for (int mm = 0; mm < mend; ++mm) tri.template step<true>(x, bc_i, bc_i >= 0 ? bct[mm] : 0.0, sh);
      } else {
        for (int mm = 0; mm < mend; ++mm) tri.step(x, bc_i, bc_i >= 0 ? bct[mm] : 0.0, sh);
      }
    }
  }
  if constexpr (ZZ) tri.zz_finish(a.steps, x, sh);
}

// SWEEP: every (slice, instance) system independently; blockIdx.x = system group.
template <int P, int NT, int SPB, bool CN, bool ZZ = false>
__global__ void __launch_bounds__(NT * SPB) k_fine_sweep(ResidentArgs a) {
  constexpr int NW = NT / 32;
  __shared__ double shm[SPB][Tri<P, NT, CN, ZZ>::kShm];
  __shared__ double bctab[SPB][kBcChunk];
  const int sys = blockIdx.x * SPB + threadIdx.x / NT;
  const int t = threadIdx.x % NT;
  const int nsys = a.nsl * a.B;
  const bool live = sys < nsys;
  const int s = live ? sys : nsys - 1;  // dead systems shadow a live one (barriers stay uniform)
  const int ln = a.ln0 + s / a.B, b = s % a.B;
  double *sh = shm[threadIdx.x / NT];
  Tri<P, NT, CN, ZZ> tri;
  tri.setup(a, a.fset[b], t, sh);
  if (NW > 1) PR_TRI_SYNC();
  tri.fold_setup(sh);
  const float *u = a.U + ((size_t)ln * a.B + b) * a.Mp;
  double x[P];
#pragma unroll
  for (int i = 0; i < P; ++i) {
    const int j = t * P + i;
    x[i] = (j < a.M) ? (double)u[j] : 0.0;
  }
  run_steps<P, NT, CN, ZZ>(tri, a, b, a.n_base + ln, t, x, sh, bctab[threadIdx.x / NT]);
  if (!live) return;
  const size_t row = ((size_t)ln * a.B + b) * a.Mp;
  if (a.Fout) {
    float *o = a.Fout + ((size_t)(ln - a.ln0) * a.B + b) * a.Mp;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int j = t * P + i;
      if (j < a.M) o[j] = (float)x[i];
    }
  } else if (ln == a.fk_ln) {
    float *o = a.Fk + (size_t)b * a.Mp;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int j = t * P + i;
      if (j < a.M) o[j] = (float)x[i];
    }
  } else {
    const float *gh = a.Gh + row;
    float *d = a.D + row;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int j = t * P + i;
      if (j < a.M) d[j] = (float)(x[i] - (double)gh[j]);
    }
  }
}

// CHAIN: one system per instance walks slices c_ln0..c_ln1-1 serially (numerical coarse
// G with the Parareal correction; or the serial fine solve, Eq. 6).
template <int P, int NT, int SPB, bool CN, bool ZZ = false>
__global__ void __launch_bounds__(NT * SPB) k_resident_chain(ResidentArgs a) {
  constexpr int NW = NT / 32;
  __shared__ double shm[SPB][Tri<P, NT, CN, ZZ>::kShm];
  __shared__ double red[SPB][2 * NW + 2];
  __shared__ double bctab[SPB][kBcChunk];
  const int sys = blockIdx.x * SPB + threadIdx.x / NT;
  const int t = threadIdx.x % NT;
  const bool live = sys < a.B;
  const int b = live ? sys : a.B - 1;
  double *sh = shm[threadIdx.x / NT];
  double *rd = red[threadIdx.x / NT];
  Tri<P, NT, CN, ZZ> tri;
  tri.setup(a, a.fset[b], t, sh);
  if (NW > 1) PR_TRI_SYNC();
  tri.fold_setup(sh);
  const size_t sstride = (size_t)a.B * a.Mp;
  double x[P];
  float *u0 = a.Uw + (size_t)a.c_ln0 * a.ustride + (size_t)b * a.Mp;
  if (a.Fcopy) {
    // U^k_k := F̂_{k−1} (reading Q12: copied, not recomputed) + δ partial of slice k
    const float *f = a.Fcopy + (size_t)b * a.Mp;
    double num = 0.0, den = 0.0;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int j = t * P + i;
      float nv = 0.f;
      if (j < a.M) {
        nv = f[j];
        const double dd = (double)nv - (double)u0[j];
        num += dd * dd;
        den += (double)nv * nv;
      }
      x[i] = (double)nv;
    }
    sys_reduce2<NT>(num, den, t, rd);
    if (live) {
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const int j = t * P + i;
        if (j < a.M) u0[j] = (float)x[i];
      }
      if (a.partials && t == 0) {
        double *pp = a.partials + (((size_t)a.c_ln0 * a.B + b) * a.nch) * 2;
        pp[0] = num;
        pp[1] = den;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int j = t * P + i;
      x[i] = (j < a.M) ? (double)u0[j] : 0.0;
    }
  }
#pragma unroll 1
  for (int ln = a.c_ln0; ln < a.c_ln1; ++ln) {
    run_steps<P, NT, CN, ZZ>(tri, a, b, a.n_base + ln, t, x, sh, bctab[threadIdx.x / NT]);
    const size_t row = (size_t)ln * sstride + (size_t)b * a.Mp;
    float *un = a.Uw + (size_t)(ln + 1) * a.ustride + (size_t)b * a.Mp;
    double num = 0.0, den = 0.0;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int j = t * P + i;
      float nv = 0.f;
      if (j < a.M) {
        if (a.GhW && live) a.GhW[row + j] = (float)x[i];
        nv = a.Dc ? (float)(x[i] + (double)a.Dc[row + j]) : (float)x[i];
        if (a.partials) {
          const double dd = (double)nv - (double)un[j];
          num += dd * dd;
          den += (double)nv * nv;
        }
      }
      x[i] = (double)nv;  // continue from the stored fp32 value (same input the fine sweep sees)
    }
    if (a.partials) sys_reduce2<NT>(num, den, t, rd);
    if (live) {
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const int j = t * P + i;
        if (j < a.M) un[j] = (float)x[i];
      }
      if (a.partials && t == 0) {
        double *pp = a.partials + (((size_t)(ln + 1) * a.B + b) * a.nch) * 2;
        pp[0] = num;
        pp[1] = den;
      }
    }
  }
}

}  // namespace pr
#endif  // PR_FINE_RESIDENT_IMPL
