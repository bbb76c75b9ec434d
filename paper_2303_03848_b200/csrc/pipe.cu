// pipe.cu — pipelined Parareal on one GPU (Eq. 8).
//
// The blocking schedule runs, per iteration k, the fine sweep F̂^k_n = F(U^{k−1}_n) over all
// slices and then the coarse chain U^k_{n+1} = G(U^k_n) + F̂^k_n − Ĝ^{k−1}_n (Eq. 7).
// At small grids both are latency-bound and neither fills the GPU, so here they run at the
// same time in one cooperative kernel and each waits only for the data it needs:
//
//   fine(k, n)   needs U^{k−1}_n                  (chain k−1 past slice n−1, or its copy step)
//                and, for D_n = F̂ − Ĝ^{k−1}_n, Ĝ^{k−1}_n (chain k−1 past slice n)
//   chain(k, n)  needs D_n                        (fine(k, n) done)
//                and may overwrite U_{n+1} only once fine(k, n+1) has read U^{k−1}_{n+1}
//
// so iteration k's fine solves start slice by slice behind chain k−1 and chain k trails them,
// approaching Eq. (8)'s pipelined cost instead of the blocking sum.  Results are bitwise those of
// the blocking schedule (same kernels' arithmetic, same orders).  The δ partial sums of each
// iteration go to their own buffer and are reduced by the kernel's tail after a grid barrier.
//
// Roles: CTAs [0, (K+1)·B·C) run the PINN chain of iteration k = CTA / (B·C) in latency mode
// (kPinnSplitG threads per point, 128/kPinnSplitG points per CTA, C chunks per instance), the
// next B·N CTAs one K1 system (slice n, instance b) each for all its iterations.  At each slice
// the chains pass in iteration order (chain k+1 needs fine(k+1, n), which needs chain k past n).  Counters (per instance and slice):
//   cnt[b][n]      += 1 by every chain warp of b after it wrote U_{n+1} (or, at its copy step, U_k)
//   floaded[b][n]  = k after fine(k, n) loaded its input,   fdone[b][n] = k after it stored D_n / F̂
// Waits are by one thread (ld.acquire) followed by a CTA barrier; data written by other CTAs is
// read through L2 (ld.global.cg).  All CTAs are co-resident (cooperative launch), and the wait
// graph is acyclic, so the kernel cannot deadlock.
#include "launch.h"
// fine-role CTAs run one K1 system on their first 128 threads (the rest exit at once when the
// chain CTAs are wider): every K1 barrier is the named barrier 1 over those 128 threads
#define PR_TRI_SYNC() asm volatile("bar.sync 1, 128;" ::: "memory")
#include "fine_resident.cuh"
#include "pinn_chain.cuh"

namespace pr {

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
// Flags are polled with relaxed gpu-scope loads: an ld.acquire.gpu compiles to LDG.STRONG.GPU +
// CCTL.IVALL, i.e. every poll would invalidate the SM's L1 -- and with it the weights the group
// chains read through L1 (measured: chain 5.6x slower per slice).  Every datum guarded by a flag
// is read through L2 (ld.global.cg) after the polling loop has observed the flag (the loads are
// issued only once the flag value has returned), and the producers publish with a release
// (fence + st.release / red.release), so L1 never has to be invalidated.
__device__ __forceinline__ int ld_flag(const int *p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// The relaxed polls are followed by one acquire fence once the flag is observed: with the
// producer's release (fence + st.release / red.release) this is the PTX memory model's
// release/acquire pattern through a relaxed read (morally strong: same scope, same address), so
// the data reads after it are ordered after the producer's writes.  One fence per wait, not per
// poll: the L1 is invalidated at most once per wait.
__device__ __forceinline__ void wait_geq(const int *p, int target) {
  while (ld_flag(p) < target) __nanosleep(20);
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
// after a CTA (or warp) barrier: publish the stores of the threads that reached it
__device__ __forceinline__ void publish_add(int *p) {
  __threadfence();
  atomicAdd(p, 1);
}
__device__ __forceinline__ void publish_add_release(int *p) {
  asm volatile("red.release.gpu.global.add.s32 [%0], 1;" ::"l"(p) : "memory");
}
__device__ __forceinline__ void publish_set(int *p, int v) {
  __threadfence();
  asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Coarse chain, warp-granular: each warp (128/(32·…) — 32/kPinnSplitG = 8 points) waits for
// its inputs and publishes its outputs by itself (no CTA barrier per slice).  δ partial sums are
// staged per warp and folded per CTA, warps in index order, at the end of each iteration — the
// blocking kernel's summation order, so δ is bitwise the same.
// The network evaluator: G = kPinnSplitG threads per point (latency mode, W = 20) or one thread
// per point (shared-memory weights, any instantiated width: the paper's 10×50 net).
template <int IN, int W, int G, int ACT>
__device__ __forceinline__ float chain_eval(const float *sw, int LH, const float (&x)[IN], float *row, bool active) {
  if constexpr (G > 1 && !(W == 20 && G == kPinnSplitG)) {
    return mlp_group<IN, W, G, ACT>(sw, LH, x, row, active);  // sw = the global weights here
  } else if constexpr (G > 1) {
    return mlp_split<IN, W, G, ACT>(sw, LH, x);
  } else {
    float xx[1][IN], y[1];
#pragma unroll
    for (int i = 0; i < IN; ++i) xx[0][i] = x[i];
    mlp_eval<IN, W, ACT, 1>(sw, LH, xx, y);
    return y[0];
  }
}

constexpr int kChunkWarps = 4;  // warps per δ chunk: the blocking chain kernel's CTA (128 threads)

// One row's δ chunks summed by one warp in k_delta's fixed order (misc.cu row_rel: lane l adds
// chunks l, l+32, … in index order, then the xor-shuffle tree; lane 0's value is used).  The row
// is left zero: a later launch whose chain covers fewer chunks (another net loaded into the
// context: other chain-CTA widths) must not sum this launch's partials.
__device__ __forceinline__ double tail_row_rel(double *p, int nch, int lane) {
  double num = 0.0, den = 0.0;
  for (int c = lane; c < nch; c += 32) {
    num += p[2 * c];
    den += p[2 * c + 1];
    p[2 * c] = 0.0;
    p[2 * c + 1] = 0.0;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, o);
    den += __shfl_xor_sync(0xffffffffu, den, o);
  }
  return (den > 0.0) ? sqrt(num) / sqrt(den) : sqrt(num);
}

// Kernel start: δ^1..δ^K zeroed (CTA 0) before the tail's barrier orders them before its maxima;
// returns the barrier's generation (it changes only when this launch's barrier opens, so it is
// read here, off the tail's critical path).
__device__ __forceinline__ unsigned long long pipe_head(const PipeArgs &pa) {
  if (blockIdx.x == 0)
    for (int k = threadIdx.x; k < pa.K; k += blockDim.x) pa.dmax[k] = 0ull;
  unsigned long long gen = 0;
  if (threadIdx.x == 0) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(gen) : "l"(pa.gbar + 1) : "memory");
  return gen;
}
// Kernel tail, in place of the flag memset, the δ memset and the δ launch that each solve needed:
// a grid barrier (arrival count + generation word; the last arrival resets the count and bumps the
// generation, so the barrier holds for any grid size a later launch on the same buffers uses), then δ^1..δ^K from the per-iteration partials with
// k_delta's per-row sums and max (rows left zero), and the flags zeroed for the next launch.  NT threads of
// the CTA take part (the fine CTAs' first 128: their barrier is the named barrier 1).
template <int NT, bool FINE>
__device__ void pipe_tail(const PipeArgs &pa, unsigned long long gen) {
  __threadfence();
  if (FINE) PR_TRI_SYNC(); else __syncthreads();
  if (threadIdx.x == 0) {  // gbar[0]: arrivals (back to 0 after every barrier), gbar[1]: generation
    unsigned long long old;
    asm volatile("atom.acq_rel.gpu.global.add.u64 %0, [%1], 1;" : "=l"(old) : "l"(pa.gbar) : "memory");
    if (old == (unsigned long long)gridDim.x - 1) {  // last arrival: reset the count, open the barrier
      asm volatile("st.relaxed.gpu.global.u64 [%0], 0;" ::"l"(pa.gbar) : "memory");
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(pa.gbar + 1), "l"(gen + 1) : "memory");
    } else {
      for (;;) {
        unsigned long long v;
        asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(pa.gbar + 1) : "memory");
        if (v != gen) break;
        __nanosleep(32);
      }
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
  }
  if (FINE) PR_TRI_SYNC(); else __syncthreads();
  const int B = pa.g.B, lane = threadIdx.x & 31;
  constexpr int NW = NT / 32;
  const int gw = blockIdx.x * NW + (threadIdx.x >> 5), nwarps = gridDim.x * NW;
  for (int k = 1; k <= pa.K; ++k) {
    const int total = (pa.N - k + 1) * B;
    for (int row = gw; row < total; row += nwarps) {
      const int ln = k + row / B, b = row % B;
      double *p = pa.partials + (size_t)k * pa.pstride + (((size_t)ln * B + b) * pa.nch) * 2;
      const double rel = tail_row_rel(p, pa.nch, lane);
      if (lane == 0) atomicMax(pa.dmax + (k - 1), (unsigned long long)__double_as_longlong(rel));
    }
  }
  for (int i = blockIdx.x * NT + threadIdx.x; i < 3 * B * pa.N; i += gridDim.x * NT) pa.cnt[i] = 0;
}

template <int IN, int W, int G, int ACT, int NWC>
__device__ void chain_role(const PipeArgs &pa, int k, int b, int chunk, const float *sw) {
  static_assert(NWC % kChunkWarps == 0, "a chain CTA holds whole δ chunks");
  const PinnArgs &a = pa.g;
  const double Lb = a.Lb[b];
  const float gscale = (float)(Lb * (double)a.out_scale);
  const float invL = (float)(1.0 / Lb);
  const size_t sstride = (size_t)a.B * a.Mp;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int GPW = 32 / G;  // point groups per warp (lanes beyond them idle)
  const bool active = lane < GPW * G;
  const bool leader = active && lane % G == 0;
  const int j = chunk * (NWC * GPW) + wid * GPW + lane / G;
  const bool ok = active && j < a.M;
  constexpr bool kGroup = G > 1 && !(W == 20 && G == kPinnSplitG);
  __shared__ __align__(16) float xrow[NWC][kGroup ? GPW : 1][kGroup ? GroupRow<W>::kPad : 4];  // group exchange rows
  float *xr = &xrow[wid][kGroup && lane / G < GPW ? lane / G : (kGroup ? GPW - 1 : 0)][0];
  const double dS = Lb / (a.M + 1);
  const float s_over_L = (float)(((j + 1) * dS) / Lb);
  int *cnt = pa.cnt + (size_t)b * pa.N;
  const int *floaded = pa.floaded + (size_t)b * pa.N, *fdone = pa.fdone + (size_t)b * pa.N;
  const int cta = b * pa.C + chunk;
  // per-warp partial of (row ln) in this iteration's staging block:
  // stage[k][((ln·B·C) + cta)·NWC + wid]·2
  double *wst = pa.wstage + (size_t)k * (pa.N + 1) * a.B * pa.C * NWC * 2;
  // (non-zero partials sit on the group leaders only — lanes ≡ 0 mod G — so for a power-of-two G the
  // butterfly stops at distance G: the lower levels would add exact zeros to lane 0's sum)
  constexpr int kLowLevel = (G & (G - 1)) == 0 ? G : 1;
  auto stage_partial = [&](int ln, double num, double den) {
#pragma unroll
    for (int o = 16; o >= kLowLevel; o >>= 1) {
      num += __shfl_xor_sync(0xffffffffu, num, o);
      den += __shfl_xor_sync(0xffffffffu, den, o);
    }
    if (lane == 0) {
      double *ps = wst + ((((size_t)ln * a.B * pa.C) + cta) * NWC + wid) * 2;
      ps[0] = num;
      ps[1] = den;
    }
  };
  float u = 0.f;
  if (k == 0 && ok) u = __ldcg(a.U + (size_t)b * a.Mp + j);  // U_0 (written before the kernel)
  {
    int n0 = 0;
    if (k > 0) {
      // U^k_k := F̂^k_{k−1} (copied, reading Q12), with the δ partial of slice k
      if (lane == 0) {
        wait_geq(fdone + (k - 1), k);
        if (k <= pa.N - 1) wait_geq(floaded + k, k);
      }
      __syncwarp();
      float *uk = a.U + (size_t)k * sstride + (size_t)b * a.Mp;
      double num = 0.0, den = 0.0;
      if (ok) {
        const float f = __ldcg(a.Fcopy + (size_t)(k & 1) * sstride + (size_t)b * a.Mp + j);
        if (leader) {
          const double dd = (double)f - (double)__ldcg(uk + j);
          num = dd * dd;
          den = (double)f * f;
        }
        u = f;
      }
      stage_partial(k, num, den);
      __syncwarp();
      if (ok && leader) uk[j] = u;
      __syncwarp();
      if (lane == 0) publish_add(cnt + (k - 1));
      n0 = k;
    }
    // slice n's inputs (D_n and the old U_{n+1}) are fetched as soon as their flags are seen set:
    // for the next slice, speculatively right after this one's stores (a non-blocking check of the
    // flags lane 0 loaded at the top of this slice, so their L2 latency hides behind the network),
    // else at the top of the next slice (blocking wait)
    float dn = 0.f, uo = 0.f;
    bool have = false;
    int fd_next = 0, fl_next = 0;  // lane 0: fdone[n+1], floaded[n+2] as loaded at the top of slice n
    auto flags_ready = [&](int n) -> bool {  // lane 0's view, broadcast: the early loads, else a fresh
      bool r = true;                          // check (a long evaluation — the paper's net — may have
      if (lane == 0) {                        // outlived the early values)
        r = fd_next >= k && (n + 1 > pa.N - 1 || fl_next >= k);
        if (!r) {
          r = ld_flag(fdone + n) >= k;
          if (r && n + 1 <= pa.N - 1) r = ld_flag(floaded + n + 1) >= k;
        }
      }
      return __shfl_sync(0xffffffffu, r ? 1 : 0, 0) != 0;
    };
    auto fetch = [&](int n) {
      const size_t row = (size_t)n * sstride + (size_t)b * a.Mp;
      if (ok) {
        dn = __ldcg(a.D + row + j);
        uo = __ldcg(a.U + row + sstride + j);
      }
    };
    for (int n = n0; n < pa.N; ++n) {
      if (k > 0 && !have) {
        if (lane == 0) {
          wait_geq(fdone + n, k);                               // D_n of this iteration
          if (n + 1 <= pa.N - 1) wait_geq(floaded + n + 1, k);  // U^{k−1}_{n+1} has been read
        }
        __syncwarp();
        fetch(n);
      }
      if (k > 0 && lane == 0 && n + 1 < pa.N) {  // issued now, read after the evaluation
        fd_next = ld_flag(fdone + n + 1);
        fl_next = n + 2 <= pa.N - 1 ? ld_flag(floaded + n + 2) : k;
      }
      const size_t row = (size_t)n * sstride + (size_t)b * a.Mp;
      const int ng = a.n_base + n;
      const float tf = (float)((a.T - ng * a.dT) / a.T), tt = (float)((a.T - (ng + 1) * a.dT) / a.T);
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
      const float y = chain_eval<IN, W, G, ACT>(sw, a.LH, x, xr, active);
      const float g = gscale * y;
      float nv = 0.f;
      double num = 0.0, den = 0.0;
      if (ok) {
        nv = k > 0 ? g + dn : g;
        if (leader) {
          a.Gh[row + j] = g;
          if (k > 0) {
            const double dd = (double)nv - (double)uo;
            num = dd * dd;
            den = (double)nv * nv;
          }
          a.U[row + sstride + j] = nv;
        }
      }
      u = nv;
      if (k > 0) stage_partial(n + 1, num, den);
      have = false;
      if (k > 0 && n + 1 < pa.N && flags_ready(n + 1)) {
        fetch(n + 1);
        have = true;
      }
      __syncwarp();
      if (lane == 0) publish_add_release(cnt + n);
      if (pa.trace && cta == 0 && threadIdx.x == 0) pa.trace[((size_t)k * pa.N + n) * 3] = gtimer();
    }
    if (k > 0) {  // fold this iteration's per-warp partials, warps in order (the blocking order):
      // every kChunkWarps warps form the δ chunk the blocking kernel's CTA over the same points writes
      __syncthreads();
      double *part = pa.partials + (size_t)k * pa.pstride;
      constexpr int SUBS = NWC / kChunkWarps;
      for (int it = (int)threadIdx.x; it < (pa.N + 1 - k) * SUBS; it += blockDim.x) {
        const int ln = k + it / SUBS, sub = it % SUBS;
        const double *ps = wst + ((((size_t)ln * a.B * pa.C) + cta) * NWC + sub * kChunkWarps) * 2;
        double num = 0.0, den = 0.0;
        for (int q = 0; q < kChunkWarps; ++q) { num += ps[2 * q]; den += ps[2 * q + 1]; }
        double *pp = part + (((size_t)ln * a.B + b) * a.nch + chunk * SUBS + sub) * 2;
        pp[0] = num;
        pp[1] = den;
      }
      __syncthreads();
    }
  }
}

template <int P, bool CN, int NWC>
__device__ void fine_role(const PipeArgs &pa, int n, int b) {
  constexpr int NT = 128;
  const ResidentArgs &a = pa.r;
  // the zig-zag form where the 128-thread chain CTAs leave the registers for it (NWC = 4); the
  // host sets ResidentArgs::use_zz for the blocking kernels of the same problem identically
  constexpr bool ZZ = !CN && NWC == 4;
  __shared__ double sh[Tri<P, NT, CN, ZZ>::kShm];
  __shared__ double bct[kBcChunk];
  const int t = threadIdx.x;
  Tri<P, NT, CN, ZZ> tri;
  tri.setup(a, a.fset[b], t, sh);
  PR_TRI_SYNC();
  tri.fold_setup(sh);
  const int C = pa.cpub;  // chain publications per (instance, slice)
  const int *cnt = pa.cnt + (size_t)b * pa.N;
  int *floaded = pa.floaded + (size_t)b * pa.N, *fdone = pa.fdone + (size_t)b * pa.N;
  const size_t row = ((size_t)n * a.B + b) * a.Mp;
  const int kmax = min(pa.K, n + 1);
  const size_t fstride = (size_t)a.B * a.Mp;  // Fk holds two rows: F̂ of iteration k in row k & 1
  for (int k = 1; k <= kmax; ++k) {
    // U^{k−1}_n.  For n = k−1 ≥ 1 it is F̂^{k−1}_{k−2} (Q12), which chain k−1 copies into U_n: read
    // it where fine(k−1, k−2) left it instead, as soon as that solve is done — the same floats,
    // without waiting for the chain's copy (one hand-off less on the critical path).  fine(k+1, k)
    // overwrites that row only after chain k−1 has passed slice k−1 (this CTA's iteration k waits
    // on that), so the copy has read it first.
    const bool from_f = n >= 1 && n == k - 1;
    if (n >= 1 && t == 0) {
      if (from_f) wait_geq(fdone + (n - 1), k - 1);  // F̂^{k−1}_{k−2} written
      else wait_geq(cnt + (n - 1), k * C);           // U^{k−1}_n written
    }
    PR_TRI_SYNC();
    const float *src = from_f ? a.Fk + (size_t)((k - 1) & 1) * fstride + (size_t)b * a.Mp : a.U + row;
    double x[P];
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int j = t * P + i;
      x[i] = (j < a.M) ? (double)__ldcg(src + j) : 0.0;
    }
    PR_TRI_SYNC();
    if (t == 0) publish_set(floaded + n, k);
    if (pa.trace && b == 0 && t == 0) pa.trace[((size_t)k * pa.N + n) * 3 + 1] = gtimer();
    run_steps<P, NT, CN, ZZ>(tri, a, b, a.n_base + n, t, x, sh, bct);
    if (n == k - 1) {  // F̂_{k−1}: copied into U^k_k by chain k
      float *o = a.Fk + (size_t)(k & 1) * fstride + (size_t)b * a.Mp;
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const int j = t * P + i;
        if (j < a.M) o[j] = (float)x[i];
      }
    } else {  // D_n = F̂_n − Ĝ^{k−1}_n once chain k−1 has passed slice n
      if (t == 0) wait_geq(cnt + n, k * C);
      PR_TRI_SYNC();
#pragma unroll
      for (int i = 0; i < P; ++i) {
        const int j = t * P + i;
        if (j < a.M) a.D[row + j] = (float)(x[i] - (double)__ldcg(a.Gh + row + j));
      }
    }
    PR_TRI_SYNC();
    if (t == 0) publish_set(fdone + n, k);
    if (pa.trace && b == 0 && t == 0) pa.trace[((size_t)k * pa.N + n) * 3 + 2] = gtimer();
  }
}

// Numerical coarse G (implicit Euler, n_c steps per slice) as the chain of iteration k
// for instance b: one K1 system (128 threads, the coarse scheme's factors) walking the slices —
// k_resident_chain's arithmetic and δ partials (chunk 0, sys_reduce2) with the flag protocol of
// the PINN chain: it reads D_n once fine(k, n) is done and overwrites U_{n+1} once fine(k, n+1)
// has read it; one publication per slice.
template <int P>
__device__ void chain_role_num(const PipeArgs &pa, int k, int b) {
  constexpr int NT = 128, NW = NT / 32;
  const ResidentArgs &a = pa.rc;
  __shared__ double shc[Tri<P, NT, false, true>::kShm];
  __shared__ double bcc[kBcChunk];
  __shared__ double rdc[2 * NW + 2];
  const int t = threadIdx.x;
  Tri<P, NT, false, true> tri;  // the coarse scheme is implicit Euler: zig-zag (use_zz on the host too)
  tri.setup(a, a.fset[b], t, shc);
  PR_TRI_SYNC();
  tri.fold_setup(shc);
  const size_t sstride = (size_t)a.B * a.Mp;
  int *cnt = pa.cnt + (size_t)b * pa.N;
  const int *floaded = pa.floaded + (size_t)b * pa.N, *fdone = pa.fdone + (size_t)b * pa.N;
  double *part = pa.partials + (size_t)k * pa.pstride;
  float *U = pa.g.U;  // the writable view of the boundary rows
  double x[P];
  int n0 = 0;
  if (k == 0) {
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int j = t * P + i;
      x[i] = (j < a.M) ? (double)__ldcg(U + (size_t)b * a.Mp + j) : 0.0;
    }
  } else {
    // U^k_k := F̂^k_{k−1} (copied, reading Q12) with the δ partial of slice k
    if (t == 0) {
      wait_geq(fdone + (k - 1), k);
      if (k <= pa.N - 1) wait_geq(floaded + k, k);
    }
    PR_TRI_SYNC();
    float *uk = U + (size_t)k * sstride + (size_t)b * a.Mp;
    const float *f = pa.r.Fk + (size_t)(k & 1) * sstride + (size_t)b * a.Mp;
    double num = 0.0, den = 0.0;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int j = t * P + i;
      float nv = 0.f;
      if (j < a.M) {
        nv = __ldcg(f + j);
        const double dd = (double)nv - (double)__ldcg(uk + j);
        num += dd * dd;
        den += (double)nv * nv;
      }
      x[i] = (double)nv;
    }
    sys_reduce2<NT>(num, den, t, rdc);
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int j = t * P + i;
      if (j < a.M) uk[j] = (float)x[i];
    }
    if (t == 0) {
      double *pp = part + (((size_t)k * a.B + b) * a.nch) * 2;
      pp[0] = num;
      pp[1] = den;
    }
    PR_TRI_SYNC();
    if (t == 0) publish_add(cnt + (k - 1));
    n0 = k;
  }
#pragma unroll 1
  for (int n = n0; n < pa.N; ++n) {
    run_steps<P, NT, false, true>(tri, a, b, a.n_base + n, t, x, shc, bcc);  // g = G(U_n)
    if (k > 0) {
      if (t == 0) {
        wait_geq(fdone + n, k);                               // D_n of this iteration
        if (n + 1 <= pa.N - 1) wait_geq(floaded + n + 1, k);  // U^{k−1}_{n+1} has been read
      }
      PR_TRI_SYNC();
    }
    const size_t row = (size_t)n * sstride + (size_t)b * a.Mp;
    float *un = U + row + sstride;
    double num = 0.0, den = 0.0;
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int j = t * P + i;
      float nv = 0.f;
      if (j < a.M) {
        pa.g.Gh[row + j] = (float)x[i];
        nv = k > 0 ? (float)(x[i] + (double)__ldcg(pa.r.D + row + j)) : (float)x[i];
        if (k > 0) {
          const double dd = (double)nv - (double)__ldcg(un + j);
          num += dd * dd;
          den += (double)nv * nv;
        }
      }
      x[i] = (double)nv;  // continue from the stored fp32 value (as k_resident_chain)
    }
    if (k > 0) sys_reduce2<NT>(num, den, t, rdc);
#pragma unroll
    for (int i = 0; i < P; ++i) {
      const int j = t * P + i;
      if (j < a.M) un[j] = (float)x[i];
    }
    if (k > 0 && t == 0) {
      double *pp = part + (((size_t)(n + 1) * a.B + b) * a.nch) * 2;
      pp[0] = num;
      pp[1] = den;
    }
    PR_TRI_SYNC();
    if (t == 0) publish_add(cnt + n);
    if (pa.trace && b == 0 && t == 0) pa.trace[((size_t)k * pa.N + n) * 3] = gtimer();
  }
}

template <int P, bool CN>
__global__ void __launch_bounds__(128) k_parareal_pipe_num(PipeArgs pa) {
  const unsigned long long gen = pipe_head(pa);
  const int nchain = (pa.K + 1) * pa.g.B;
  if ((int)blockIdx.x < nchain) {
    chain_role_num<P>(pa, blockIdx.x / pa.g.B, blockIdx.x % pa.g.B);
  } else {
    const int f = blockIdx.x - nchain;
    fine_role<P, CN, 4>(pa, f / pa.g.B, f % pa.g.B);
  }
  pipe_tail<128, true>(pa, gen);  // (128-thread CTAs: named barrier 1 is the whole CTA)
}

// CTAs [0, S·B·C): chain CTA set s = blockIdx / (B·C) runs the chains of iterations k ≡ s (mod S),
// one after the other; then one CTA per fine system.  S = K+1 (every chain its own CTAs) when that
// grid fits one CTA per SM, else S = 2 (pa.S, host): chain k+1 still runs behind chain k on its own
// CTAs while chain k+2 — which at C2 starts only after chain k has finished — reuses chain k's
// CTAs; no chain waits on a later one, so the reuse cannot deadlock.  At C2 with the 3×20 net one
// set per iteration is 160 CTAs > 148 SMs, and the chain CTAs that shared an SM paced every later
// iteration (1.7 vs 1.2 µs per slice); with the paper's 10×50 net (12-warp chain CTAs, 148 CTAs)
// the chains overlap in time, and reusing CTAs would serialise them (0.84 → 0.97 ms).
template <int P, bool CN, int IN, int W, int G, int ACT, int NWC>
__global__ void __launch_bounds__(NWC * 32) k_parareal_pipe(PipeArgs pa) {
  extern __shared__ float sw[];
  const unsigned long long gen = pipe_head(pa);
  const int per = pa.g.B * pa.C;
  const int S = pa.S;
  const int nchain = S * per;
  if ((int)blockIdx.x < nchain) {
    const float *w = pa.g.wts;  // group kernels read the weights through L1
    if (G == 1 || (W == 20 && G == kPinnSplitG)) {  // smem weights (group chains read them through L1)
      for (int i = threadIdx.x; i < pa.g.nfloats; i += blockDim.x) sw[i] = pa.g.wts[i];
      __syncthreads();
      w = sw;
    }
    const int s0 = blockIdx.x / per, r = blockIdx.x % per;
#pragma unroll 1
    for (int k = s0; k <= pa.K; k += S) {
      chain_role<IN, W, G, ACT, NWC>(pa, k, r / pa.C, r % pa.C, w);
      __syncthreads();  // (chain k's CTA-wide δ fold is done before chain k+S starts)
    }
    pipe_tail<NWC * 32, false>(pa, gen);
  } else {
    if (threadIdx.x >= 128) return;  // one K1 system per fine CTA (128 threads)
    const int f = blockIdx.x - nchain;
    fine_role<P, CN, NWC>(pa, f / pa.g.B, f % pa.g.B);
    pipe_tail<128, true>(pa, gen);
  }
}

typedef void (*PipeKernel)(PipeArgs);
// Chain CTAs of the group chains (the paper's 10×50 net) are 12 warps wide: with one K1 system
// per 128 threads of a fine CTA and ~168 registers per thread, a 384-thread CTA fills an SM, so
// (K+1)·C chain CTAs + N fine CTAs ≤ 148 run one per SM and the chains do not share SMs with the
// fine solves (measured: 3× slower chain slices when they did).
template <int IN, int W, int G>
constexpr int pipe_nwc() { return (G > 1 && !(W == 20 && G == kPinnSplitG)) ? 12 : 4; }
int pipe_chain_warps(int W, int G) { return pinn_split_is_group(W, G) ? 12 : 4; }

template <bool CN, int IN, int W, int G, int ACT>
static PipeKernel pipe_kernel_p(int M) {
  constexpr int NWC = pipe_nwc<IN, W, G>();
  if (M <= 256) return k_parareal_pipe<2, CN, IN, W, G, ACT, NWC>;
  if (M <= 512) return k_parareal_pipe<4, CN, IN, W, G, ACT, NWC>;
  if (M <= 1024) return k_parareal_pipe<8, CN, IN, W, G, ACT, NWC>;
  return nullptr;
}
template <int IN, int W, int G, int ACT>
static PipeKernel pipe_kernel_c(int M, bool cn) {
  return cn ? pipe_kernel_p<true, IN, W, G, ACT>(M) : pipe_kernel_p<false, IN, W, G, ACT>(M);
}
// instantiated: latency-mode 20-wide nets (G = 4), and one thread per point for the paper's
// 10×50 architecture (tanh or ReLU) and 32-wide tanh nets
static PipeKernel pipe_kernel(int M, bool cn, int IN, int W, int act, int G) {
  if (G == 10) {  // group chains (12-warp CTAs)
    if (IN == 4 && W == 50) return act ? pipe_kernel_c<4, 50, 10, 1>(M, cn) : pipe_kernel_c<4, 50, 10, 0>(M, cn);
    return nullptr;
  }
  if (G == kPinnSplitG) {  // shuffle chain
    if (W != 20 || act != 0) return nullptr;
    if (IN == 4) return pipe_kernel_c<4, 20, kPinnSplitG, 0>(M, cn);
    if (IN == 2) return pipe_kernel_c<2, 20, kPinnSplitG, 0>(M, cn);
    return nullptr;
  }
  if (G != 1) return nullptr;
  if (IN == 4 && W == 50) return act ? pipe_kernel_c<4, 50, 1, 1>(M, cn) : pipe_kernel_c<4, 50, 1, 0>(M, cn);
  if (IN == 4 && W == 32 && act == 0) return pipe_kernel_c<4, 32, 1, 0>(M, cn);
  return nullptr;
}

typedef void (*PipeNumKernel)(PipeArgs);
static PipeNumKernel pipe_num_kernel(int M, bool cn) {
  if (M <= 256) return cn ? k_parareal_pipe_num<2, true> : k_parareal_pipe_num<2, false>;
  if (M <= 512) return cn ? k_parareal_pipe_num<4, true> : k_parareal_pipe_num<4, false>;
  if (M <= 1024) return cn ? k_parareal_pipe_num<8, true> : k_parareal_pipe_num<8, false>;
  return nullptr;
}
bool pipe_num_supported(int M, bool cn) { return pipe_num_kernel(M, cn) != nullptr; }
cudaError_t launch_parareal_pipe_num(const PipeArgs &pa, int M, bool cn, cudaStream_t s) {
  PipeNumKernel k = pipe_num_kernel(M, cn);
  if (!k) return cudaErrorInvalidValue;
  int dev = 0, nsm = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 128, 0);
  if (e != cudaSuccess) return e;
  const int grid = (pa.K + 1) * pa.g.B + pa.g.B * pa.N;
  if (grid > occ * nsm) return cudaErrorCooperativeLaunchTooLarge;
  PipeArgs arg = pa;
  void *params[] = {&arg};
  return cudaLaunchCooperativeKernel((const void *)k, dim3(grid), dim3(128), params, 0, s);
}

bool pipe_supported(int M, bool cn, int IN, int W, int act, int G) {
  return pipe_kernel(M, cn, IN, W, act, G) != nullptr;
}

// Launches the cooperative kernel; cudaErrorCooperativeLaunchTooLarge (or not supported) tells
// the caller to use the blocking schedule.
cudaError_t launch_parareal_pipe(const PipeArgs &pa, int M, bool cn, int IN, int W, int act, int G,
                                 size_t smem, cudaStream_t s) {
  PipeKernel k = pipe_kernel(M, cn, IN, W, act, G);
  if (!k) return cudaErrorInvalidValue;
  if (pinn_split_is_group(W, G)) smem = 0;  // group chains read the weights through L1
  cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  int dev = 0, nsm = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const int nthreads = 32 * pipe_chain_warps(W, G);
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, nthreads, smem);
  if (e != cudaSuccess) return e;
  int S = pa.K + 1;
  if ((long)S * pa.g.B * pa.C + (long)pa.g.B * pa.N > nsm) S = S < 2 ? S : 2;  // one CTA per SM, else two sets
  const int grid = S * pa.g.B * pa.C + pa.g.B * pa.N;
  if (grid > occ * nsm) return cudaErrorCooperativeLaunchTooLarge;
  PipeArgs arg = pa;
  arg.S = S;
  void *params[] = {&arg};
  return cudaLaunchCooperativeKernel((const void *)k, dim3(grid), dim3(nthreads), params, smem, s);
}

}  // namespace pr
