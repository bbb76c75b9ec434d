// fine_streamed.cuh — K2: HBM-streamed implicit-Euler propagator for large M.
//
// Same mathematics as K1 (fine_resident.cuh): every implicit step of
// (I − dτA) x⁺ = x + dτ(a_M+b_M) g(τ⁺) e_M is a forward
// elimination  y_j = r_j − m_j y_{j−1}  and a back substitution
// x_j = y_j/p_j − (u_j/p_j) x_{j+1}, each a linear recurrence evaluated as a
// scan of affine maps v ↦ A + B·v.  A system (one instance × one slice, up to
// 2^20 points and more) is cut into tiles of kSTile points, one CTA per tile;
// a pass is one kernel: a sequential pass over 16 points per thread, a CTA
// scan, and a look-back across tiles.
//
// Look-back.  The tile multipliers B (products of the constant factors) are
// precomputed on the host, so a CTA publishes only its offset A, in one
// 16-byte {A, epoch} word (single 128-bit store/load: no fences).  The value
// entering tile i is the composition of the aggregates of its predecessors
// i−1, …, i−W_i, where W_i (host-computed) is the first window whose
// multiplier product falls below kLookbackEps: the tiles further back change
// it by < kLookbackEps·|y| (eight orders below fp64 rounding).  No CTA waits
// on an inclusive prefix, so there is no dependency chain across the wave,
// and the composition order is fixed: results are bitwise reproducible.
// A dedicated look-back warp requests the window, multipliers and status words
// of the 64 nearest predecessors in one round trip while the data warps load.
// Tiles map to CTA indices interleaved across the launch's independent systems
// (CTAs are dispatched in index order), so a tile's predecessor started nsys
// CTAs earlier.
//
// Layout.  The fp64 factors and the sweep-private fp32 ping-pong buffers are
// stored thread-interleaved (see il_index) so every warp access is coalesced.
// Traffic: 16 B per point-step of fp32 state from HBM; factors 8 B (forward)
// and 16 B (backward) per point per pass from L2.
#include <cuda_runtime.h>
#include <stdint.h>
#include <string.h>

#ifndef PR_FINE_STREAMED_ARGS
#define PR_FINE_STREAMED_ARGS
namespace pr {

constexpr int kSPS = 16;                 // points per thread
constexpr int kSNT = 128;                // data threads per tile (+1 look-back warp)
constexpr int kSTile = kSPS * kSNT;      // 2048 points per tile
constexpr double kLookbackEps = 1e-24;   // look-back truncation (see above)

// Interleaved ("thread-major") layout: point j of a row sits at
// tile·kSTile + i·kSNT + t  (tile = j / kSTile, t = (j % kSTile) / kSPS, i = j % kSPS),
// so the i-th point of every thread of a warp is one contiguous segment.
inline size_t il_index(size_t j) {
  return (j / kSTile) * kSTile + (j % kSPS) * kSNT + (j % kSTile) / kSPS;
}
inline int streamed_Mt(int M) { return (M + kSTile - 1) / kSTile * kSTile; }
inline int streamed_ntiles(int M) { return (M + kSTile - 1) / kSTile; }

// Constant data of one implicit scheme (I − dτA) for K2, per factor set.
struct StreamedFactors {
  const double *m, *ip, *cu;     // interleaved [nsets][Mt], identity-padded beyond M
  const double *tileB;           // [2][nsets][ntiles] tile multiplier, indexed by scan position
  const int *tileW;              // [2][nsets][ntiles] look-back window (predecessors)
};

struct StreamedState {
  float *X = nullptr, *Y = nullptr;      // [nsys][Mt] ping-pong state (interleaved)
  double *status = nullptr;              // [nsys][ntiles] × {A, epoch} (16 B)
  unsigned long long *ticket = nullptr;  // global ticket counter
  unsigned long long epoch = 0;          // host: last epoch used
  unsigned long long ticket_base = 0;    // host: tickets consumed so far
  int ntiles = 0;
  size_t nsys_max = 0;
};

inline size_t streamed_state_bytes(int M, int Mp, int B, int Nloc) {
  (void)Mp;
  const size_t nsys = (size_t)B * (size_t)(Nloc > 0 ? Nloc : 1);
  return 2 * nsys * (size_t)streamed_Mt(M) * sizeof(float) + nsys * streamed_ntiles(M) * 16 + 512;
}
inline void streamed_state_bind(StreamedState &s, char *base, int M, int Mp, int B, int Nloc) {
  (void)Mp;
  const size_t nsys = (size_t)B * (size_t)(Nloc > 0 ? Nloc : 1);
  const size_t Mt = (size_t)streamed_Mt(M);
  s.ntiles = streamed_ntiles(M);
  s.nsys_max = nsys;
  size_t off = 0;
  s.X = (float *)(base + off); off += nsys * Mt * sizeof(float);
  s.Y = (float *)(base + off); off += nsys * Mt * sizeof(float);
  off = (off + 255) / 256 * 256;
  s.status = (double *)(base + off); off += nsys * s.ntiles * 16;
  off = (off + 255) / 256 * 256;
  s.ticket = (unsigned long long *)(base + off);
  s.epoch = 0;
  s.ticket_base = 0;
}

// Epilogue of a backward pass
enum { EPI_X = 0, EPI_SWEEP = 1, EPI_CHAIN = 2 };

struct PassArgs {
  int M, Mp, Mt, B, ntiles, nsys, nsets;
  StreamedFactors f;
  const int *fset;
  const float *in;           // [nsys][Mp] natural rows (first pass of a slice) or [nsys][Mt] interleaved
  float *out;                // [nsys][Mt] interleaved (forward passes, EPI_X)
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
  // look-back
  double *status;
  unsigned long long *ticket;
  unsigned long long ticket_base, epoch;
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

// {A, epoch} status word: one 128-bit relaxed store / load (single-copy atomic for an aligned
// 16-byte access), so a reader that sees this pass's epoch also sees its value -- no fence.
// The load must be .relaxed (not a weak ld): ptxas may hoist a weak load out of the spin loop.
__device__ __forceinline__ void st_status(double *p, double v, unsigned long long e) {
  asm volatile("st.relaxed.gpu.global.v2.u64 [%0], {%1, %2};" ::"l"(p), "l"(__double_as_longlong(v)), "l"(e)
               : "memory");
}
__device__ __forceinline__ void ld_status(const double *p, double &v, unsigned long long &e) {
  unsigned long long a;
  asm volatile("ld.relaxed.gpu.global.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(e) : "l"(p) : "memory");
  v = __longlong_as_double(a);
}

template <int DIR>
__device__ __forceinline__ double shfl_prev(double v, int d) {
  return DIR == 0 ? __shfl_up_sync(0xffffffffu, v, d) : __shfl_down_sync(0xffffffffu, v, d);
}

__device__ __forceinline__ void bar_data() {  // named barrier over the kSNT data threads only
  asm volatile("bar.sync 1, %0;" ::"n"(kSNT) : "memory");
}

// Look-back warp: the value entering tile `pos` = composition of the aggregates of its W_pos
// predecessors (scan order), written to *yin by lane 0.
template <int DIR>
__device__ __forceinline__ void look_back(const PassArgs &a, int s, int pos, int set, int lane, double *yin) {
  if (pos == 0) {
    if (lane == 0) *yin = 0.0;
    return;
  }
  const size_t tb = ((size_t)DIR * a.nsets + set) * a.ntiles;
  const double *sts = a.status + 2 * (size_t)s * a.ntiles;
  // Speculative first round: the window size, the multipliers and the status words of the 64
  // nearest predecessors are requested together (one L2 round trip); the window then masks them
  // and only the in-window ones are waited for.
  const int W = a.f.tileW[tb + pos];
  double sv[2], bv[2];
  unsigned long long se[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int k = lane + 32 * h, p = pos - 1 - k;
    bv[h] = (p >= 0) ? a.f.tileB[tb + p] : 1.0;
    sv[h] = 0.0;
    se[h] = a.epoch;
    if (p >= 0) ld_status(sts + 2 * p, sv[h], se[h]);
  }
  double accA = 0.0, accB = 1.0;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int k = lane + 32 * h;
    double mA = 0.0, mB = 1.0;          // identity beyond the window
    if (k < W) {
      while (se[h] != a.epoch) ld_status(sts + 2 * (pos - 1 - k), sv[h], se[h]);
      mA = sv[h];
      mB = bv[h];
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double oA = __shfl_down_sync(0xffffffffu, mA, d);
      const double oB = __shfl_down_sync(0xffffffffu, mB, d);
      if ((lane & (2 * d - 1)) == 0) {
        mA = fma(mB, oA, mA);
        mB *= oB;
      }
    }
    mA = __shfl_sync(0xffffffffu, mA, 0);
    mB = __shfl_sync(0xffffffffu, mB, 0);
    accA = fma(accB, mA, accA);
    accB *= mB;
  }
  for (int base = 64; base < W; base += 32) {  // rare: windows beyond 64 tiles
    const int k = base + lane;          // predecessor at distance k+1 in scan order
    double mA = 0.0, mB = 1.0;          // identity beyond the window
    if (k < W) {
      const int p = pos - 1 - k;
      mB = a.f.tileB[tb + p];
      double v;
      unsigned long long e;
      do { ld_status(a.status + 2 * ((size_t)s * a.ntiles + p), v, e); } while (e != a.epoch);
      mA = v;
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
    mA = __shfl_sync(0xffffffffu, mA, 0);
    mB = __shfl_sync(0xffffffffu, mB, 0);
    accA = fma(accB, mA, accA);
    accB *= mB;
  }
  if (lane == 0) *yin = accA;
}

// One pass over one tile.  kSNT data threads (kSPS points each) plus one look-back warp that
// composes the predecessors' aggregates while the data warps load and scan their tile, so the
// look-back latency overlaps the tile's own memory traffic instead of following it.
template <int DIR, bool IN_IL, bool OUT_IL>
__global__ void __launch_bounds__(kSNT + 32) k_streamed_pass(PassArgs a) {
  constexpr int NW = kSNT / 32;
  __shared__ double sA[NW], sB[NW];
  __shared__ double s_yin;
  __shared__ double red[2 * NW];
  // Tile order: CTAs are dispatched in increasing index order (the assumption CUB's single-pass
  // scan makes), so every predecessor a CTA waits for is resident or finished.  Indices are
  // interleaved across the independent systems of the launch (slices × instances): the
  // predecessor of (s, pos) is CTA tk − nsys, which with many systems published long before.
  const unsigned long long tk = blockIdx.x;
  const int s = (int)(tk % a.nsys);
  const int pos = (int)(tk / a.nsys);                 // position in scan order
  const int tile = DIR == 0 ? pos : a.ntiles - 1 - pos;
  const int b = s % a.B;
  const int ln = a.ln0 + s / a.B;
  const int set = a.fset[b];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  if (w == NW) {  // ---- look-back warp
    look_back<DIR>(a, s, pos, set, lane, &s_yin);
    __syncthreads();  // s_yin published to the data warps
    return;
  }
  const int j0 = tile * kSTile + t * kSPS;
  const size_t til = (size_t)tile * kSTile + t;   // interleaved offset of this thread's point 0
  const double *fa = (DIR == 0 ? a.f.m : a.f.ip) + (size_t)set * a.Mt + til;
  const double *fb = DIR ? a.f.cu + (size_t)set * a.Mt + til : nullptr;

  double x[kSPS], ca[kSPS], cb[kSPS];
  // factors: interleaved, identity-padded (m=0, 1/p=1, u/p=0 beyond M) → no guards
#pragma unroll
  for (int i = 0; i < kSPS; ++i) {
    ca[i] = __ldg(fa + i * kSNT);
    if (DIR) cb[i] = __ldg(fb + i * kSNT);
  }
  if (IN_IL) {
    const float *in = a.in + (size_t)s * a.Mt + til;
#pragma unroll
    for (int i = 0; i < kSPS; ++i) x[i] = __ldcs(in + i * kSNT);
  } else {
    const float *in = a.in + (size_t)s * a.Mp;
    if (j0 + kSPS <= a.M) {
#pragma unroll
      for (int i = 0; i < kSPS; i += 4) {
        const float4 v = *reinterpret_cast<const float4 *>(in + j0 + i);
        x[i] = v.x; x[i + 1] = v.y; x[i + 2] = v.z; x[i + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < kSPS; ++i) x[i] = (j0 + i < a.M) ? (double)in[j0 + i] : 0.0;
    }
  }
  // local sequential pass with zero input, and the thread's map (A, B)
  double Bt = 1.0;
  if (DIR == 0) {
    if (j0 <= a.M - 1 && a.M - 1 < j0 + kSPS) {
      const int n = a.n_base + ln;
      const double tau = (n * a.dT + a.step_m * a.dtau) + a.dtau;
      const double g = a.upper_bc ? 0.0 : a.Lb[b] - a.Kb[b] * exp(-a.rb[b] * tau);
#pragma unroll
      for (int i = 0; i < kSPS; ++i)
        if (j0 + i == a.M - 1) x[i] += a.bcoef[b] * g;
    }
#pragma unroll
    for (int i = 0; i < kSPS; ++i) {
      ca[i] = -ca[i];  // −m_j
      if (i > 0) x[i] = fma(ca[i], x[i - 1], x[i]);
      Bt *= ca[i];
    }
  } else {
#pragma unroll
    for (int i = kSPS - 1; i >= 0; --i) {
      cb[i] = -cb[i];  // −u_j/p_j
      x[i] = (i < kSPS - 1) ? fma(cb[i], x[i + 1], x[i] * ca[i]) : x[i] * ca[i];
      Bt *= cb[i];
    }
  }
  const double At = DIR == 0 ? x[kSPS - 1] : x[0];
  // CTA inclusive scan in scan order (DIR 0: ascending threads; DIR 1: descending)
  const int sl = DIR == 0 ? lane : 31 - lane;  // scan-order lane
  double iA = At, iB = Bt;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double pA = shfl_prev<DIR>(iA, d), pB = shfl_prev<DIR>(iB, d);
    if (sl >= d) {
      iA = fma(iB, pA, iA);
      iB *= pB;
    }
  }
  const int sw = DIR == 0 ? w : NW - 1 - w;    // scan-order warp
  if (sl == 31) { sA[sw] = iA; sB[sw] = iB; }
  bar_data();
  // ---- publish this tile's offset at once (successors' look-back warps are waiting on it)
  if (t == 0) {
    double TA = 0.0;
    for (int q = 0; q < NW; ++q) TA = fma(sB[q], TA, sA[q]);
    st_status(a.status + 2 * ((size_t)s * a.ntiles + pos), TA, a.epoch);
  }
  // exclusive prefix of this thread within the tile (independent of the look-back)
  double wA = 0.0, wB = 1.0;  // prefix of preceding warps (in scan order)
  for (int q = 0; q < sw; ++q) { wA = fma(sB[q], wA, sA[q]); wB *= sB[q]; }
  double eA = shfl_prev<DIR>(iA, 1), eB = shfl_prev<DIR>(iB, 1);
  if (sl == 0) { eA = 0.0; eB = 1.0; }
  const double xA = fma(eB, wA, eA), xB = eB * wB;
  __syncthreads();  // the look-back warp has written s_yin
  const double yin = fma(xB, s_yin, xA);
  // fix-up with running prefix products
  double q = 1.0;
  if (DIR == 0) {
#pragma unroll
    for (int i = 0; i < kSPS; ++i) { q *= ca[i]; x[i] = fma(q, yin, x[i]); }
  } else {
#pragma unroll
    for (int i = kSPS - 1; i >= 0; --i) { q *= cb[i]; x[i] = fma(q, yin, x[i]); }
  }
  // ---- stores / epilogues
  if (OUT_IL) {
    float *o = a.out + (size_t)s * a.Mt + til;
#pragma unroll
    for (int i = 0; i < kSPS; ++i) __stcs(o + i * kSNT, (float)x[i]);
    return;
  }
  if (a.epi == EPI_SWEEP) {
    float *o;
    bool diff = false;
    if (a.Fout) o = a.Fout + (size_t)s * a.Mp;
    else if (s >= a.fk_sys_lo && s < a.fk_sys_hi) o = a.Fk + (size_t)b * a.Mp;
    else { o = a.D + (size_t)s * a.Mp; diff = true; }
    const float *gh = a.Gh + (size_t)s * a.Mp;
#pragma unroll
    for (int i = 0; i < kSPS; ++i) {
      const int j = j0 + i;
      if (j < a.M) o[j] = diff ? (float)(x[i] - (double)gh[j]) : (float)x[i];
    }
    return;
  }
  // EPI_CHAIN: g = x; Ĝ_n = g; U_{n+1} = g + D_n; δ partial against the old U_{n+1}
  {
    const size_t row = (size_t)b * a.Mp;
    double num = 0.0, den = 0.0;
#pragma unroll
    for (int i = 0; i < kSPS; ++i) {
      const int j = j0 + i;
      if (j < a.M) {
        if (a.GhW) a.GhW[row + j] = (float)x[i];
        const float nv = a.Dc ? (float)(x[i] + (double)a.Dc[row + j]) : (float)x[i];
        if (a.partials) {
          const double dd = (double)nv - (double)a.Unext[row + j];
          num += dd * dd;
          den += (double)nv * nv;
        }
        a.Unext[row + j] = nv;
      }
    }
    if (a.partials) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        num += __shfl_xor_sync(0xffffffffu, num, o);
        den += __shfl_xor_sync(0xffffffffu, den, o);
      }
      if (lane == 0) { red[2 * w] = num; red[2 * w + 1] = den; }
      bar_data();
      if (t == 0) {
        num = 0.0; den = 0.0;
        for (int q2 = 0; q2 < NW; ++q2) { num += red[2 * q2]; den += red[2 * q2 + 1]; }
        double *pp = a.partials + ((size_t)b * a.nch + tile) * 2;
        pp[0] = num;
        pp[1] = den;
      }
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

static cudaError_t launch_pass(StreamedState &st, int dir, bool in_il, PassArgs a, cudaStream_t s) {
  a.ntiles = st.ntiles;
  a.status = st.status;
  a.ticket = st.ticket;
  a.ticket_base = st.ticket_base;
  a.epoch = ++st.epoch;
  const unsigned long long grid = (unsigned long long)a.nsys * st.ntiles;
  st.ticket_base += grid;
  if (dir == 0) {
    if (in_il) k_streamed_pass<0, true, true><<<(unsigned)grid, kSNT + 32, 0, s>>>(a);
    else k_streamed_pass<0, false, true><<<(unsigned)grid, kSNT + 32, 0, s>>>(a);
  } else {
    if (a.epi == EPI_X) k_streamed_pass<1, true, true><<<(unsigned)grid, kSNT + 32, 0, s>>>(a);
    else k_streamed_pass<1, true, false><<<(unsigned)grid, kSNT + 32, 0, s>>>(a);
  }
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

// `steps` implicit steps on a.nsys systems: in0 → ... → the epilogue set in `a` (last step).
static cudaError_t streamed_steps(StreamedState &st, const PassArgs &a, const float *in0, int steps,
                                  cudaStream_t s, int *nl) {
  for (int m = 0; m < steps; ++m) {
    PassArgs f = a;
    f.step_m = m;
    f.in = (m == 0) ? in0 : st.X;
    f.out = st.Y;
    cudaError_t e = launch_pass(st, 0, m > 0, f, s);
    if (e != cudaSuccess) return e;
    PassArgs g = a;
    g.step_m = m;
    g.in = st.Y;
    g.out = st.X;
    if (m < steps - 1) g.epi = EPI_X;
    e = launch_pass(st, 1, true, g, s);
    if (e != cudaSuccess) return e;
    *nl += 2;
  }
  return cudaSuccess;
}

cudaError_t streamed_sweep(StreamedState &st, const StreamedProblem &p, const StreamedJob &j, cudaStream_t s,
                           int *nl) {
  PassArgs a = pass_base(p);
  const size_t off = (size_t)j.ln0 * p.B * p.Mp;
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
