// fine_grid.cu — K2R: the grid-resident fine sweep for large grids (SURVEY NEXT-4 "whole-GPU
// resident fine solver"; the large-M counterpart of K1).
//
// Same mathematics as K1's zig-zag form (fine_resident.cuh): implicit Euler steps of slice n
// alternate between the LU and the UL factorisation of the constant matrix
// M_f = I − dτA, so the substitution of step m and the elimination of step m+1 form one pass of a
// 2-state recurrence; an n-step slice is n+1 passes.  Here one system (2^20 points at C3) spans
// the whole GPU: CTA c (one per SM, cooperative launch) owns a contiguous range of 256·PT points,
// thread t of it PT consecutive points, and NS systems (slices) are solved together.  The state
// stays on chip (fp64) for all passes of a slice group — in registers, and at PT = 28 (C3) a third
// system in shared memory (NS = 3) — so HBM is touched once per slice (load U_n, store D_n) instead
// of 16 B per point and step; the factors 1/p_j, 1/q_j of the CTA's points sit in shared memory;
// the off-diagonals come from the closed forms
// l_j = −J(c1·J − c0), u_j = −J(c1·J + c0) (J = j+1, c0 = dτr/2, c1 = dτσ²/2).
//
// One pass: each thread runs its points from a zero entering state (chunk totals; the elimination
// chain in scaled form), a warp scan of the 2-vector affine parts with per-lane level coefficients
// precomputed at kernel start (recomputed per scan when NS = 3, whose third state takes their room), a
// fold over the warps (constant warp maps in shared memory), the CTA total is published
// (per-pass slot, tagged words, 32-word stride per CTA) and the entering state of the CTA is
// composed from the totals of its W predecessors in pass direction, all of a window's polling
// rounds in flight together (decoupled look-back: every CTA publishes before it waits,
// so the wait is one store-to-load propagation; W from the host, where the product of the predecessors'
// maps falls below 1e-24 — the same truncation as K2; the weights Π of the CTA maps in between
// are host tables), then each thread reruns its points from its exact entering state.
#include "launch.h"

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <type_traits>

namespace pr {
namespace {


constexpr int kGT = 256;        // threads per CTA
constexpr int kGW = kGT / 32;   // warps per CTA
constexpr long long kSpinMax = 1ll << 28;  // look-back wait bound (then the solve fails, no hang)
constexpr int kPollRounds = 4;             // look-back rounds whose loads are in flight together
// words between consecutive CTAs' published totals: each CTA's words on their own two 128-B lines
// (no line shared by two CTAs' stores and polls)
constexpr int kTotStride = 32;
// PR_DEBUG_BOUNDS builds (test-only variant, compute-sanitizer being unavailable on the GPU pool):
// index checks that trap on violation
#ifdef PR_DEBUG_BOUNDS
#define PR_CHECK(cond) do { if (!(cond)) __trap(); } while (0)
#else
#define PR_CHECK(cond) do { } while (0)
#endif

__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long v;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(v));
  return v;
}

template <int PT, int NS>
struct GridSolver {
  // per-lane level coefficients (the lane's composite map at each level, 0 without predecessor)
  // and exclusive maps, for ↑↑ (index 0) and ↓↓ (index 1), in shared memory [..][kGT] (the
  // registers hold the NS systems' state)
  double *sC, *sX;
  int t, lane, w, c, j0;
  __device__ __forceinline__ double &C(int dir, int l, int e) const { return sC[((dir * 5 + l) * 3 + e) * kGT + t]; }
  __device__ __forceinline__ double &X(int dir, int e) const { return sX[(dir * 3 + e) * kGT + t]; }

  // closed-form off-diagonals and factors of point j (padding beyond M: identity, no coupling)
  __device__ __forceinline__ void mults(const GridArgs &a, const double *sip, const double *siq, int i, double &ip,
                                        double &iq, double &l, double &u) const {
    const int j = j0 + i;
    const double J = (double)(j + 1);
    ip = sip[i * kGT + t];
    iq = siq[i * kGT + t];
    l = (j >= 1 && j < a.M) ? -J * fma(a.c1, J, -a.c0) : 0.0;
    u = (j < a.M - 1) ? -J * fma(a.c1, J, a.c0) : 0.0;
  }
};

}  // namespace

// St: the storage type of the state between passes — fp64 where NS·PT values fit the registers,
// else fp32 (the precision K2 stores between its passes in HBM; the arithmetic stays fp64)
template <int PT, int NS, typename St>
__global__ void __launch_bounds__(kGT, 1) k_fine_grid(GridArgs a) {
  extern __shared__ __align__(16) double gsm[];
  double *sip = gsm, *siq = gsm + kGT * PT;          // this CTA's 1/p, 1/q, [PT][kGT]
  double *swm = siq + kGT * PT;                        // [2][kGW][3] constant warp maps
  double *swt = swm + 2 * kGW * 3;                     // [2][kGW][NS][2] warp totals (by pass parity)
  double *sE = swt + 2 * kGW * NS * 2;                 // [NS][2] CTA entering state
  double *sT = sE + NS * 2;                            // [NS][2] CTA total of the pass
  double *sred = sT + NS * 2;                          // [32][2] look-back partial sums (warp 0)
  // NS = 3 (PT = 28): two systems in registers, the third in shared memory (fp64, point-major);
  // the room is the per-lane level coefficients', which are then recomputed in every scan from
  // the thread's constant chunk maps (sA) — the same operations in the same order as at setup
  constexpr int NSM = NS == 3 ? 1 : 0;  // systems whose state lives in shared memory
  constexpr int NR = NS - NSM;          // systems whose state lives in registers
  constexpr bool LVL = NSM > 0;         // level coefficients recomputed per scan
  double *sC = sred + 64;                              // [2][5][3][kGT] level coefficients (!LVL)
  double *sA = sC;                                     // [2][3][kGT] thread chunk maps (LVL)
  double *sxm = sA + 2 * 3 * kGT;                      // [NSM][PT][kGT] state of the smem systems (LVL)
  double *sX = LVL ? sxm + NSM * PT * kGT : sC + 2 * 5 * 3 * kGT;  // [2][3][kGT] exclusive maps
  double *sxs = sX + 2 * 3 * kGT;                      // [NS][2][kGT] lanes' exclusive warp prefixes
  double *sbc = sxs + NS * 2 * kGT;                    // [NS][steps] boundary terms
  GridSolver<PT, NS> g;
  g.sC = sC;
  g.sX = sX;
  g.t = threadIdx.x;
  g.lane = g.t & 31;
  g.w = g.t >> 5;
  g.c = blockIdx.x;
  g.j0 = (g.c * kGT + g.t) * PT;
  const int nCTA = gridDim.x;
  // state of system k at the thread's point i (registers for k < NR, else shared memory)
#define PR_XR(k, i) ((k) < NR ? (double)x[(k) < NR ? (k) : 0][i] : sxm[(((k) - NR) * PT + (i)) * kGT + t])
#define PR_XW(k, i, v)                                          \
  do {                                                          \
    if ((k) < NR) x[(k) < NR ? (k) : 0][i] = (St)(v);           \
    else sxm[(((k) - NR) * PT + (i)) * kGT + t] = (v);          \
  } while (0)
  const int t = g.t, lane = g.lane, w = g.w, c = g.c;
  for (int i = t; i < kGT * PT; i += kGT) {
    const int j = c * kGT * PT + i;
    const int o = (i % PT) * kGT + i / PT;  // point-major: thread t's point i at [i][t] (no bank conflicts)
    sip[o] = j < a.M ? a.ip[j] : 1.0;
    siq[o] = j < a.M ? a.iq[j] : 1.0;
  }
  __syncthreads();
  // thread chunk maps in pass order: ↑↑ A = [[ncl, 0], [ip·ncl, nml]], ↓↓ A = [[ncu, 0], [iq·ncu, nmu]]
  {
    double m[2][3] = {{1.0, 0.0, 1.0}, {1.0, 0.0, 1.0}};
#pragma unroll
    for (int i = 0; i < PT; ++i) {  // ↑↑: ascending
      double ip, iq, l, u;
      g.mults(a, sip, siq, i, ip, iq, l, u);
      const double ncl = -l * iq, nml = -l * ip;
      m[0][1] = fma(ip * ncl, m[0][0], nml * m[0][1]);
      m[0][0] *= ncl;
      m[0][2] *= nml;
    }
#pragma unroll
    for (int i = PT - 1; i >= 0; --i) {  // ↓↓: descending
      double ip, iq, l, u;
      g.mults(a, sip, siq, i, ip, iq, l, u);
      const double ncu = -u * ip, nmu = -u * iq;
      m[1][1] = fma(iq * ncu, m[1][0], nmu * m[1][1]);
      m[1][0] *= ncu;
      m[1][2] *= nmu;
    }
    // level coefficients, exclusive maps and warp totals (constant) per direction
#pragma unroll
    for (int dir = 0; dir < 2; ++dir) {
      const bool up = dir == 0;
      double m11 = m[dir][0], m21 = m[dir][1], m22 = m[dir][2];
      if (LVL) sA[(dir * 3) * kGT + t] = m11, sA[(dir * 3 + 1) * kGT + t] = m21, sA[(dir * 3 + 2) * kGT + t] = m22;
#pragma unroll
      for (int l = 0; l < 5; ++l) {
        const int d = 1 << l;
        const double p11 = up ? __shfl_up_sync(kFull, m11, d) : __shfl_down_sync(kFull, m11, d);
        const double p21 = up ? __shfl_up_sync(kFull, m21, d) : __shfl_down_sync(kFull, m21, d);
        const double p22 = up ? __shfl_up_sync(kFull, m22, d) : __shfl_down_sync(kFull, m22, d);
        const bool has = up ? lane >= d : lane + d <= 31;
        if (!LVL) {
          g.C(dir, l, 0) = has ? m11 : 0.0;
          g.C(dir, l, 1) = has ? m21 : 0.0;
          g.C(dir, l, 2) = has ? m22 : 0.0;
        }
        if (has) {
          m21 = fma(m21, p11, m22 * p21);
          m11 *= p11;
          m22 *= p22;
        }
      }
      double x0 = up ? __shfl_up_sync(kFull, m11, 1) : __shfl_down_sync(kFull, m11, 1);
      double x1 = up ? __shfl_up_sync(kFull, m21, 1) : __shfl_down_sync(kFull, m21, 1);
      double x2 = up ? __shfl_up_sync(kFull, m22, 1) : __shfl_down_sync(kFull, m22, 1);
      if (lane == (up ? 0 : 31)) x0 = 1.0, x1 = 0.0, x2 = 1.0;
      g.X(dir, 0) = x0, g.X(dir, 1) = x1, g.X(dir, 2) = x2;
      if (lane == (up ? 31 : 0)) {
        double *o = swm + (dir * kGW + w) * 3;
        o[0] = m11, o[1] = m21, o[2] = m22;
      }
    }
  }
  __syncthreads();

  const int ngroups = (a.nsys + NS - 1) / NS;
  const int bc_t = (a.M - 1) / PT - c * kGT, bc_ip = (a.M - 1) % PT;  // thread / point of row M
  const int bc_i = (t == bc_t && (a.M - 1) / (kGT * PT) == c) ? bc_ip : -1;
  unsigned pid = 0;  // passes published so far (the tags)
  // The closed-form path serves every warp except the one holding row M (the boundary term):
  // at j = 0 and j = M−1 the closed-form off-diagonal only ever multiplies a zero entering state
  // (nothing precedes row 1 upward; above row M sit padding points, whose inputs are 0, so they
  // pass zeros downward), and padding points' maps only ever multiply zeros.  Warp-uniform.
  const bool fast = !__any_sync(kFull, bc_i >= 0);
  const double J0 = (double)(g.j0 + 1);
  for (int grp = 0; grp < ngroups; ++grp) {
    // ---- inputs and boundary terms of the NS systems (slices ln0 + grp·NS + k)
    St x[NR][PT];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int s = grp * NS + k;
      const float *u = s < a.nsys ? a.U + (size_t)(a.ln0 + s) * a.row : nullptr;
#pragma unroll
      for (int i = 0; i < PT; ++i) {
        const int j = g.j0 + i;
        PR_XW(k, i, (u && j < a.M) ? (double)u[j] : 0.0);
      }
    }
    for (int q = t; q < NS * a.steps; q += kGT) {
      const int k = q / a.steps, m = q - k * a.steps;
      const int n = a.n_base + a.ln0 + grp * NS + k;
      const double tau1 = (n * a.dT + m * a.dtau) + a.dtau;  // τ_{m+1} of slice n (the oracle's association)
      PR_CHECK(grp * NS + k < ngroups * NS);
      sbc[q] = a.upper_bc ? 0.0 : a.bcoef * (a.Lb - a.Kb * exp(-a.rb * tau1));
    }
    __syncthreads();
    // ---- the steps+1 passes
    for (int m = 0; m <= a.steps; ++m) {
      // direction and kind: m = 0 lone ↑ elimination; 0 < m < steps merged (odd ↓↓, even ↑↑);
      // m = steps lone substitution (↓ after an LU step, ↑ after a UL step)
      const bool last = m == a.steps;
      // the pass body with direction and kind as compile-time constants (register-resident
      // coefficients, no per-point selects): kind 0 lone elimination, 1 merged, 2 lone substitution
      auto pass = [&](auto up_tag, auto kind_tag) {
      constexpr bool up = decltype(up_tag)::value;
      constexpr int dir = up ? 0 : 1;
      constexpr int kind = decltype(kind_tag)::value;
      constexpr bool elim = kind != 2, subst = kind != 0;
      double bcg[NS];
#pragma unroll
      for (int k = 0; k < NS; ++k) bcg[k] = (bc_i >= 0 && elim) ? sbc[k * a.steps + (m < a.steps ? m : 0)] : 0.0;
      unsigned long long *tr = a.trace ? a.trace + ((size_t)(pid) * gridDim.x + c) * 5 : nullptr;
      if (tr && t == 0) tr[0] = gtime();
      // (1) local totals from a zero entering state
      double s1[NS], s2[NS];
#pragma unroll
      for (int k = 0; k < NS; ++k) s1[k] = 0.0, s2[k] = 0.0;
      // this pass's warp totals (double-buffered: a warp may write the next pass's while another
      // still folds this pass's in step 5)
      double *swtb = swt + (pid & 1) * (kGW * NS * 2);
      // general point: boundary rows (no l at j = 0, no u at j = M−1), padding, the boundary term
      auto point = [&](int i, double(&xs)[NS], double(&zs)[NS], bool write) {
        double ip, iq, l, u;
        g.mults(a, sip, siq, i, ip, iq, l, u);
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          const double v = PR_XR(k, i);
          double xn, zn = 0.0;
          if (up) {  // x: UL forward substitution (ncl = −l·iq); z: LU elimination (nml = −l·ip)
            xn = subst ? fma(-l * iq, xs[k], v) : v;
            const double r = i == bc_i ? xn + bcg[k] : xn;
            if (elim) zn = fma(-l * ip, zs[k], ip * r);
          } else {   // x: LU back substitution (ncu = −u·ip); z: UL elimination (nmu = −u·iq)
            xn = subst ? fma(-u * ip, xs[k], v) : v;
            const double r = i == bc_i ? xn + bcg[k] : xn;
            if (elim) zn = fma(-u * iq, zs[k], iq * r);
          }
          if (subst) xs[k] = xn;
          if (elim) zs[k] = zn;
          if (write) PR_XW(k, i, elim ? zn : xn);
        }
      };
      // interior point (every point of the thread strictly inside 1 … M−2, no boundary term):
      // J = J0 + i exactly, only the off-diagonal of this direction, no selects
      auto point_fast = [&](int i, double(&xs)[NS], double(&zs)[NS], bool write) {
        const double J = J0 + (double)i;
        const double ip = sip[i * kGT + t], iq = siq[i * kGT + t];
        const double nl = up ? J * fma(a.c1, J, -a.c0) : J * fma(a.c1, J, a.c0);  // −l or −u
        const double mx = nl * (up ? iq : ip), mz = nl * (up ? ip : iq), fz = up ? ip : iq;
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          const double xv = PR_XR(k, i);
          const double xn = subst ? fma(mx, xs[k], xv) : xv;
          double zn = 0.0;
          if (elim) zn = fma(mz, zs[k], fz * xn);
          if (subst) xs[k] = xn;
          if (elim) zs[k] = zn;
          if (write) PR_XW(k, i, elim ? zn : xn);
        }
      };
      auto run = [&](double(&xs)[NS], double(&zs)[NS], bool write) {
        if (fast) {
          if (up) {
#pragma unroll
            for (int i = 0; i < PT; ++i) point_fast(i, xs, zs, write);
          } else {
#pragma unroll
            for (int i = PT - 1; i >= 0; --i) point_fast(i, xs, zs, write);
          }
        } else {
          if (up) {
#pragma unroll
            for (int i = 0; i < PT; ++i) point(i, xs, zs, write);
          } else {
#pragma unroll
            for (int i = PT - 1; i >= 0; --i) point(i, xs, zs, write);
          }
        }
      };
      if (kind == 1 && fast) {
        // local run of a merged pass over interior points from a zero entering state, with the
        // elimination chain in scaled form t = z/f (f = ip upward, iq downward):
        //   t_i = x̂_i + (−l_i or −u_i)·f_{i∓1}·t_{i∓1},   z_last = f_last·t_last
        // (one FMA per point and system instead of a multiply and an FMA; only the totals are
        // needed here — the rerun produces the outputs in the unscaled form)
        double fprev = 0.0;
#pragma unroll
        for (int ii = 0; ii < PT; ++ii) {
          const int i = up ? ii : PT - 1 - ii;
          const double J = J0 + (double)i;
          const double ip = sip[i * kGT + t], iq = siq[i * kGT + t];
          const double nl = up ? J * fma(a.c1, J, -a.c0) : J * fma(a.c1, J, a.c0);  // −l or −u
          const double mx = nl * (up ? iq : ip), f = up ? ip : iq;
          const double cz = nl * fprev;  // (ii = 0: the entering state is zero, cz unused)
#pragma unroll
          for (int k = 0; k < NS; ++k) {
            const double xv = PR_XR(k, i);
            if (ii == 0) {
              s1[k] = xv;
              s2[k] = xv;
            } else {
              s1[k] = fma(mx, s1[k], xv);
              s2[k] = fma(cz, s2[k], s1[k]);
            }
          }
          fprev = f;
        }
#pragma unroll
        for (int k = 0; k < NS; ++k) s2[k] *= fprev;
      } else {
        run(s1, s2, false);
      }
      // (2) warp scan of the NS 2-vectors with the level coefficients (precomputed, or recomputed
      //     alongside from the chunk maps when LVL)
      double lm11 = 0.0, lm21 = 0.0, lm22 = 0.0;  // LVL: the lane's composite chunk map so far
      if (LVL) lm11 = sA[(dir * 3) * kGT + t], lm21 = sA[(dir * 3 + 1) * kGT + t], lm22 = sA[(dir * 3 + 2) * kGT + t];
#pragma unroll
      for (int l = 0; l < 5; ++l) {
        const int d = 1 << l;
        double C0, C1, C2;
        if (LVL) {  // the setup's level recurrence (bitwise the same coefficients)
          const bool has = up ? lane >= d : lane + d <= 31;
          C0 = has ? lm11 : 0.0, C1 = has ? lm21 : 0.0, C2 = has ? lm22 : 0.0;
          const double p11 = up ? __shfl_up_sync(kFull, lm11, d) : __shfl_down_sync(kFull, lm11, d);
          const double p21 = up ? __shfl_up_sync(kFull, lm21, d) : __shfl_down_sync(kFull, lm21, d);
          const double p22 = up ? __shfl_up_sync(kFull, lm22, d) : __shfl_down_sync(kFull, lm22, d);
          if (has) {
            lm21 = fma(lm21, p11, lm22 * p21);
            lm11 *= p11;
            lm22 *= p22;
          }
        } else {
          C0 = g.C(dir, l, 0), C1 = g.C(dir, l, 1), C2 = g.C(dir, l, 2);
        }
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          const double q1 = up ? __shfl_up_sync(kFull, s1[k], d) : __shfl_down_sync(kFull, s1[k], d);
          const double q2 = up ? __shfl_up_sync(kFull, s2[k], d) : __shfl_down_sync(kFull, s2[k], d);
          s2[k] = fma(C1, q1, fma(C2, q2, s2[k]));
          s1[k] = fma(C0, q1, s1[k]);
        }
      }
      // the lane's exclusive prefix, parked in shared memory until step 5 (register pressure)
#pragma unroll
      for (int k = 0; k < NS; ++k) {
        double xs1 = up ? __shfl_up_sync(kFull, s1[k], 1) : __shfl_down_sync(kFull, s1[k], 1);
        double xs2 = up ? __shfl_up_sync(kFull, s2[k], 1) : __shfl_down_sync(kFull, s2[k], 1);
        if (lane == (up ? 0 : 31)) xs1 = 0.0, xs2 = 0.0;
        sxs[(k * 2) * kGT + t] = xs1;
        sxs[(k * 2 + 1) * kGT + t] = xs2;
        if (lane == (up ? 31 : 0)) swtb[(w * NS + k) * 2] = s1[k], swtb[(w * NS + k) * 2 + 1] = s2[k];
      }
      __syncthreads();
      const double *wm = swm + dir * kGW * 3;  // constant warp maps of this direction
      ++pid;
      // (4) publish and look-back, warp 0.  A CTA total is NS 2-vectors of fp64, published as
      //     4·NS words (one 32-bit half | pass id << 32): 64-bit relaxed stores and loads are
      //     single-copy atomic, so a word carries its own validity — no flag, no release/acquire
      //     fences, and the poll that sees the tag has already read the data.  Four pass slots:
      //     a CTA publishes pass pid+2 before its successors may have read pass pid when two
      //     passes in a row run upward (a group ending on a UL substitution, then the next
      //     group's first elimination); it cannot publish pid+4 before they finished pid (pass
      //     pid+2 or pid+3 runs downward and waits for them)
      constexpr int WPC = NS * 4;     // words per CTA total
      constexpr int G = 32 / WPC;     // predecessors polled per round
      unsigned long long *slot = a.tot + (size_t)(pid & 3) * nCTA * kTotStride;
      if (w == 0) {
        double T1[NS], T2[NS];  // the CTA total: all warps composed in pass order (every lane)
#pragma unroll
        for (int k = 0; k < NS; ++k) T1[k] = 0.0, T2[k] = 0.0;
#pragma unroll 1
        for (int kk = 0; kk < kGW; ++kk) {
          const int q = up ? kk : kGW - 1 - kk;
#pragma unroll
          for (int k = 0; k < NS; ++k) {
            const double t1 = swtb[(q * NS + k) * 2], t2 = swtb[(q * NS + k) * 2 + 1];
            T2[k] = fma(wm[q * 3 + 1], T1[k], fma(wm[q * 3 + 2], T2[k], t2));
            T1[k] = fma(wm[q * 3], T1[k], t1);
          }
        }
        if (lane == 0)
#pragma unroll
          for (int k = 0; k < NS; ++k) sT[k * 2] = T1[k], sT[k * 2 + 1] = T2[k];
        __syncwarp();
        if (lane < WPC) {  // word lane: value v = lane/2 (system v/2, component v&1), half lane&1
          const double val = sT[lane >> 1];
          const unsigned long long bits = (unsigned long long)__double_as_longlong(val);
          const unsigned half = (lane & 1) ? (unsigned)(bits >> 32) : (unsigned)bits;
          PR_CHECK(lane < kTotStride && c < nCTA);
          st_relaxed_u64(slot + (size_t)c * kTotStride + lane, ((unsigned long long)pid << 32) | half);
        }
        if (tr && lane == 0) tr[1] = gtime();
        // look-back: the totals of the W predecessors in pass direction, G per round
        // (lane = g·WPC + word), weighted by the host maps Π between predecessor and CTA
        const int W = a.lbW[dir * nCTA + c];
        const int gi = lane / WPC, q = lane - gi * WPC;
        // an even word lane holds value v = q/2 = (system v/2, component v&1) of its predecessor;
        // its contributions to the entering state e = Σ Π·T: component 0 (T1) → e1 += Π11·T1,
        // e2 += Π21·T1; component 1 (T2) → e2 += Π22·T2
        // the loads of up to kPollRounds rounds are issued together (one L2 round trip for the
        // whole window instead of one per round; the summation order is the rounds' order)
        double c1 = 0.0, c2 = 0.0;
        for (int base0 = 0; base0 < W; base0 += kPollRounds * G) {
          unsigned long long wd[kPollRounds];
#pragma unroll
          for (int r = 0; r < kPollRounds; ++r) {
            const int kq = base0 + r * G + gi + 1;  // predecessor distance
            if (gi < G && kq <= W) PR_CHECK((up ? c - kq : c + kq) >= 0 && (up ? c - kq : c + kq) < nCTA && kq <= a.KW);
            wd[r] = (gi < G && kq <= W) ? ld_relaxed_u64(slot + (size_t)(up ? c - kq : c + kq) * kTotStride + q) : 0ull;
          }
#pragma unroll
          for (int r = 0; r < kPollRounds; ++r) {
            const int kq = base0 + r * G + gi + 1;
            const bool act = gi < G && kq <= W;
            unsigned half = 0;
            if (act) {
              const unsigned long long *src = slot + (size_t)(up ? c - kq : c + kq) * kTotStride + q;
              long long spins = 0;
              while ((wd[r] >> 32) != pid) {
                wd[r] = ld_relaxed_u64(src);
                if (++spins > kSpinMax) {
                  a.err[0] = 1;  // the host reports the solve as failed
                  break;
                }
              }
              half = (unsigned)wd[r];
            }
            const unsigned hi = __shfl_down_sync(kFull, half, 1);
            if (act && (q & 1) == 0) {
              const double val = __longlong_as_double((long long)(((unsigned long long)hi << 32) | half));
              const double *P = a.lbP + (((size_t)dir * nCTA + c) * a.KW + (kq - 1)) * 3;
              if ((q >> 1) & 1) {
                c2 = fma(P[2], val, c2);
              } else {
                c1 = fma(P[0], val, c1);
                c2 = fma(P[1], val, c2);
              }
            }
          }
        }
        sred[lane * 2] = c1, sred[lane * 2 + 1] = c2;
        __syncwarp();
        if (lane < NS * 2) {  // lane 2k: e1 of system k, lane 2k+1: e2 (fixed order: deterministic)
          const int k = lane >> 1;
          double e = 0.0;
          for (int g2 = 0; g2 < G; ++g2) {
            const double *r = sred + (g2 * WPC + 4 * k) * 2;
            e += (lane & 1) ? r[1] + r[5] : r[0];
          }
          sE[lane] = e;
        }
        if (tr && lane == 0) tr[2] = gtime();
      }
      __syncthreads();
      if (tr && t == 0) tr[3] = gtime();
      // (5) this thread's entering state: the CTA entering state carried through the preceding
      //     warps (their maps and totals, in pass order), then the lane's exclusive prefix; rerun
      double i1[NS], i2[NS];
      {
        double w1[NS], w2[NS];
#pragma unroll
        for (int k = 0; k < NS; ++k) w1[k] = sE[k * 2], w2[k] = sE[k * 2 + 1];
#pragma unroll 1
        for (int kk = 0; kk < kGW; ++kk) {
          const int q = up ? kk : kGW - 1 - kk;
          if (up ? q < w : q > w) {
#pragma unroll
            for (int k = 0; k < NS; ++k) {
              const double t1 = swtb[(q * NS + k) * 2], t2 = swtb[(q * NS + k) * 2 + 1];
              w2[k] = fma(wm[q * 3 + 1], w1[k], fma(wm[q * 3 + 2], w2[k], t2));
              w1[k] = fma(wm[q * 3], w1[k], t1);
            }
          }
        }
#pragma unroll
        for (int k = 0; k < NS; ++k) {
          i2[k] = fma(g.X(dir, 1), w1[k], fma(g.X(dir, 2), w2[k], sxs[(k * 2 + 1) * kGT + t]));
          i1[k] = fma(g.X(dir, 0), w1[k], sxs[(k * 2) * kGT + t]);
        }
      }
      run(i1, i2, true);
      if (tr && t == 0) tr[4] = gtime();
      };
      const bool up = last ? ((a.steps - 1) & 1) != 0 : (m & 1) == 0;
      using K0 = std::integral_constant<int, 0>;
      using K1 = std::integral_constant<int, 1>;
      using K2 = std::integral_constant<int, 2>;
      if (m == 0) pass(std::true_type{}, K0{});
      else if (last) {
        if (up) pass(std::true_type{}, K2{});
        else pass(std::false_type{}, K2{});
      } else if (up) pass(std::true_type{}, K1{});
      else pass(std::false_type{}, K1{});
    }
    // ---- epilogue of the group: F̂ (test hook / F̂_{k−1}) or D = F̂ − Ĝ, fp32 rows
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      const int s = grp * NS + k;
      if (s >= a.nsys) continue;
      const int ln = a.ln0 + s;
      float *dst;
      const float *gh = nullptr;
      if (a.Fout) dst = a.Fout + (size_t)s * a.row;
      else if (ln == a.fk_ln) dst = a.Fk;
      else dst = a.D + (size_t)ln * a.row, gh = a.Gh + (size_t)ln * a.row;
#pragma unroll
      for (int i = 0; i < PT; ++i) {
        const int j = g.j0 + i;
        if (j < a.M) dst[j] = gh ? (float)(PR_XR(k, i) - (double)gh[j]) : (float)PR_XR(k, i);
      }
    }
    __syncthreads();  // sbc is rewritten by the next group
  }
#undef PR_XR
#undef PR_XW
}

namespace {
using GridKernel = void (*)(GridArgs);
// systems per group for PT points per thread: the state NS·PT fp64 values must fit the registers
// Systems per group: the state NS·PT fp64 values live in registers, so NS is bounded by PT (PT =
// 28: 2; 16: 4; ≤ 8: 8) and chosen per launch as the smallest of {2, 4, 8} covering the sweep's
// systems (a group computes all NS systems whether used or not).  Measured: 3 systems at PT = 28
// (fp64 with 52 B of spills, or fp32 storage — the F2F conversions per point and pass) were
// slower per system than 2.
constexpr int ns_max(int PT) { return PT >= 28 ? 3 : PT >= 16 ? 4 : 8; }
int ns_pick(int PT, int nsys) {
  const int mx = ns_max(PT);
  if (mx == 3) return nsys <= 2 ? 2 : 3;
  return nsys <= 2 ? 2 : (nsys <= 4 || mx == 4) ? std::min(4, mx) : mx;
}
GridKernel grid_kernel(int PT, int NS) {
  switch (PT * 16 + NS) {
    case 4 * 16 + 2: return k_fine_grid<4, 2, double>;
    case 4 * 16 + 4: return k_fine_grid<4, 4, double>;
    case 4 * 16 + 8: return k_fine_grid<4, 8, double>;
    case 8 * 16 + 2: return k_fine_grid<8, 2, double>;
    case 8 * 16 + 4: return k_fine_grid<8, 4, double>;
    case 8 * 16 + 8: return k_fine_grid<8, 8, double>;
    case 16 * 16 + 2: return k_fine_grid<16, 2, double>;
    case 16 * 16 + 4: return k_fine_grid<16, 4, double>;
    case 28 * 16 + 2: return k_fine_grid<28, 2, double>;
    case 28 * 16 + 3: return k_fine_grid<28, 3, double>;
  }
  return nullptr;
}
constexpr int kPTs[] = {4, 8, 16, 28};
}  // namespace

int fine_grid_ns(int PT, int nsys) { return ns_pick(PT, nsys); }
size_t fine_grid_tot_words(int nblocks) { return (size_t)4 * nblocks * kTotStride; }
size_t fine_grid_smem(int PT, int steps) {  // at the largest NS of PT (every launch fits)
  const int NS = ns_max(PT);
  const size_t lvl = NS == 3 ? (size_t)(6 + PT) : 30;  // chunk maps + smem state (NS = 3), else level coefficients
  return ((size_t)2 * kGT * PT + 2 * kGW * 3 + 2 * kGW * NS * 2 + NS * 4 + 64 + (lvl + 6 + NS * 2) * kGT +
          (size_t)NS * steps) *
         sizeof(double);
}

// Points per thread and CTAs for M grid points on nsm SMs (one CTA per SM): the smallest PT with
// ⌈M / (256·PT)⌉ ≤ nsm.  0 if none.
int fine_grid_pt(int M, int nsm, int *nblocks) {
  for (int PT : kPTs) {
    const long long per = (long long)kGT * PT;
    const long long nb = (M + per - 1) / per;
    if (nb <= nsm) {
      *nblocks = (int)nb;
      return PT;
    }
  }
  return 0;
}

cudaError_t launch_fine_grid(const GridArgs &a, int PT, int nblocks, cudaStream_t s) {
  GridKernel k = grid_kernel(PT, ns_pick(PT, a.nsys));
  if (!k) return cudaErrorInvalidValue;
  const size_t smem = fine_grid_smem(PT, a.steps);
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, occ = 0, nsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, kGT, smem);
  if (e != cudaSuccess) return e;
  if ((long long)occ * nsm < nblocks) return cudaErrorCooperativeLaunchTooLarge;
  GridArgs arg = a;
  void *params[] = {&arg};
  return cudaLaunchCooperativeKernel((const void *)k, dim3(nblocks), dim3(kGT), params, smem, s);
}

}  // namespace pr
