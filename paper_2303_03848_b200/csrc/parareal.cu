// parareal.cu — host side of the C ABI (include/parareal.h): validation,
// fp64 factorisation, workspace, the Parareal iteration (Eq. 7,
// schedule reading Q12), NCCL hand-off of slice-boundary states between
// ranks, reporting.  All device work is issued on one stream.
#include "../../include/parareal.h"

#include <cuda_runtime.h>
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <thread>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "launch.h"
#include <nvtx3/nvToolsExt.h>  // header-only NVTX: phase ranges for nsys/ncu --nvtx (no-ops untraced)

// ============================================================================ NCCL (dlopen)
// NCCL is resolved at run time so the library loads without it (world == 1 never touches
// it).  Under torch the wheel's libnccl.so.2 is already mapped and dlopen returns it.
namespace {
typedef struct ncclComm *ncclComm_t;
typedef struct { char internal[128]; } ncclUniqueId;
typedef int ncclResult_t;
enum { kNcclFloat32 = 7, kNcclFloat64 = 8, kNcclSum = 0, kNcclMax = 2, kNcclInProgress = 7 /* ncclResult_t */ };

struct Nccl {
  bool tried = false, ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(ncclResult_t) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
};
std::mutex g_nccl_mu;
Nccl g_nccl;

Nccl &nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.tried) return g_nccl;
  g_nccl.tried = true;
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) {
    g_nccl.why = std::string("dlopen(libnccl.so.2) failed: ") + dlerror();
    return g_nccl;
  }
#define PR_SYM(field, name)                                          \
  g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name)); \
  if (!g_nccl.field) { g_nccl.why = "missing NCCL symbol " name; return g_nccl; }
  PR_SYM(GetUniqueId, "ncclGetUniqueId");
  PR_SYM(CommInitRank, "ncclCommInitRank");
  PR_SYM(CommDestroy, "ncclCommDestroy");
  PR_SYM(CommAbort, "ncclCommAbort");
  PR_SYM(Send, "ncclSend");
  PR_SYM(Recv, "ncclRecv");
  PR_SYM(AllReduce, "ncclAllReduce");
  PR_SYM(GroupStart, "ncclGroupStart");
  PR_SYM(GroupEnd, "ncclGroupEnd");
  PR_SYM(GetErrorString, "ncclGetErrorString");
  PR_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
#undef PR_SYM
  g_nccl.ok = true;
  return g_nccl;
}

thread_local std::string g_init_error = "no error";

std::string fmt(const char *f, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, f);
  vsnprintf(buf, sizeof buf, f, ap);
  va_end(ap);
  return buf;
}

// fp64 LU factors of one implicit-Euler matrix  I − dτ A, per factor set.
struct Scheme {
  double dtau = 0;
  int steps = 0;
  double *m = nullptr, *ip = nullptr, *cu = nullptr;  // device [nsets][Mp] (K1)
  double *zz = nullptr;  // device [6][nsets][Mp] K1 zig-zag factors (θ = 1): ip, nml, ncu (LU), iq, ncl, nmu (UL)
  double *iip = nullptr;                            // device [nsets][Mt] 1/p, interleaved (K2)
  double *coef = nullptr;                           // device [nsets][2] dτr/2, dτσ²/2 (K2)
  double *thrP = nullptr;                           // device [2][nsets][Mt/kSPS] (K2 in-tile prefix multipliers)
  double *tileB = nullptr;                          // device [2][nsets][ntiles] (K2 look-back)
  int *tileW = nullptr;
  double *bcoef = nullptr;                          // device [B]
  double theta = 1.0;                               // θ-step (1: implicit Euler, 1/2: Crank–Nicolson)
  double *ecoef = nullptr;                          // device [nsets][3] explicit part (θ < 1)
  double *PL = nullptr, *tileL = nullptr;           // device K2 θ < 1 tile-edge correction tables
  // K2R grid-resident solver (fine_grid.cu; θ = 1, one factor set, M > kResidentMaxM)
  double *giq = nullptr;                            // device [M] 1/q_j (UL pivots)
  double *lbP = nullptr;                            // device [2][nb][KW][3] look-back weights
  int *lbW = nullptr;                               // device [2][nb] windows
  int g_pt = 0, g_nb = 0, g_kw = 0;                 // points per thread, CTAs, table stride (0: no grid solver)
  double g_c0 = 0, g_c1 = 0, g_bcoef = 0;         // closed-form coefficients; dτ(a_M+b_M) of instance 0
};

constexpr int kResidentMaxM = 2048;
constexpr int kPinnTPB = 128;
constexpr int kPinnSmemBudget = 200 * 1024;  // dynamic shared memory for the fp32 PINN weights
struct LoopGroup;  // in-process loopback transport (defined with the transport calls below)
}  // namespace

// ============================================================================ context
struct pr_ctx {
  std::string err = "no error";
  bool poisoned = false;
  // problem
  int M = 0, Mp = 0, B = 0, N = 0, nf = 0, nc = 0, coarse = 0, max_iter = 0, upper_bc = 0;
  double fine_theta = 1.0;
  double T = 0, dT = 0, tol = 0;
  std::vector<double> K, sig, r, L;
  // placement
  int rank = 0, world = 1, device = 0, n0 = 0, n1 = 0, Nloc = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  ncclComm_t comm = nullptr;
  LoopGroup *loop = nullptr;  // in-process loopback transport (test only), else NCCL
  // constants on device
  int nsets = 0;
  int *d_fset = nullptr;
  double *d_L = nullptr, *d_K = nullptr, *d_r = nullptr;
  std::vector<int> fset;
  std::vector<std::pair<double, double>> sets;  // (sigma, r)
  Scheme fine, crs;
  // workspace
  void *ws = nullptr;
  size_t ws_bytes = 0;
  bool own_ws = false, ws_ready = false;
  float *U = nullptr, *Gh = nullptr, *D = nullptr, *Fk = nullptr, *tmp = nullptr;
  double *partials = nullptr;
  unsigned long long *d_delta = nullptr;
  int nch = 1;
  double *h_delta = nullptr;  // pinned [max_iter]
  // streamed-kernel state
  pr::StreamedState sst;
  // PINN
  bool have_pinn = false;
  int IN = 4, W = 0, LH = 0, act = 0, nfloats = 0;
  float cs[4] = {1, 1, 1, 1}, out_scale = 1;
  float *d_wts = nullptr;
  float *d_wgrp = nullptr;   // the packed weights with the hidden matrices in the group-kernel order
  std::vector<float> h_wts;  // packed copy for the parameter-space kernels
  int tc = 0;                // PR_PREC_FP16_TC / PR_PREC_BF16_TC: K4 (tensor cores), else 0
  float *d_tcp = nullptr;    // K4 compact fp32 parameters
  void *d_wh = nullptr;      // K4 hidden matrices (fp16/bf16, core-matrix layout)
  int tc_nfloats = 0;
  // options
  int opt_pinn_kernel = 0;
  int opt_fine_kernel = 0;
  int opt_graphs = 0;
  int opt_pipeline = 0;  // 0 auto, 1 off (PR_OPT_PIPELINE)
  int64_t comm_timeout_ms = 600000;  // PR_OPT_COMM_TIMEOUT_MS (0: wait forever)
  int opt_wavefront = 0;             // PR_OPT_WAVEFRONT: 0 auto, 1 blocking chain, n ≥ 2 chunks
  int opt_spatial = 0;               // PR_OPT_SPATIAL_CHAIN: 0 auto, 1 off, 2 on
  // K2R grid-resident fine solver: published totals, flags, timeout flag (mapped host memory)
  unsigned long long *g_tot = nullptr;  // K2R published totals (tagged 32-bit halves)
  size_t g_tot_words = 0;
  int *g_err_h = nullptr, *g_err_d = nullptr;
  // spatially sharded chain (NEXT-4): every slice's rows, this rank's j-range meaningful
  float *sp_U = nullptr, *sp_Gh = nullptr, *sp_D = nullptr, *sp_F = nullptr;
  double *sp_part = nullptr;
  bool capturing = false;
  // pipelined schedule (pipe.cu): per-iteration δ partials and the slice counters
  double *pipe_partials = nullptr;
  int *pipe_flags = nullptr;
  double *pipe_wstage = nullptr;
  size_t pipe_pstride = 0;
  int pipe_ok = -1;  // -1 unknown, 0 no, 1 yes
  // captured solve (PR_OPT_USE_GRAPHS)
  cudaGraphExec_t g_exec = nullptr;
  const float *g_vt = nullptr;
  float *g_v0 = nullptr;
  bool g_dev = false;  // the captured solve took device pointers
  int g_K = 0;
  int64_t g_launches = 0;
  cudaEvent_t g_e0 = nullptr, g_e1 = nullptr;
  std::vector<cudaEvent_t> g_events;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> g_spans;
  int64_t launches = 0;
  bool solved = false;
  // timing
  std::vector<cudaEvent_t> ev;
  int ev_used = 0;
};

namespace {

pr_status fail(pr_ctx *c, pr_status s, const std::string &msg) {
  if (c) {
    c->err = msg;
    if (s == PR_ERR_CUDA || s == PR_ERR_NCCL) c->poisoned = true;
  } else {
    g_init_error = msg;
  }
  return s;
}

#define CU(call)                                                                              \
  do {                                                                                        \
    cudaError_t e_ = (call);                                                                  \
    if (e_ != cudaSuccess)                                                                    \
      return fail(c, e_ == cudaErrorMemoryAllocation ? PR_ERR_OUT_OF_MEMORY : PR_ERR_CUDA,    \
                  fmt("%s failed: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__)); \
  } while (0)

#define NC(call)                                                                              \
  do {                                                                                        \
    ncclResult_t e_ = (call);                                                                 \
    if (e_ != 0)                                                                              \
      return fail(c, PR_ERR_NCCL, fmt("%s failed: %s", #call, nccl().GetErrorString(e_)));    \
  } while (0)

// Every launcher returns the launch's cudaError_t (and leaves the sticky error state alone);
// a failed launch poisons the context like any other CUDA failure (include/parareal.h).
#define LAUNCH(call)                                                                          \
  do {                                                                                        \
    c->launches++;                                                                            \
    cudaError_t e_ = (call);                                                                  \
    if (e_ == cudaSuccess) e_ = cudaPeekAtLastError();                                        \
    if (e_ != cudaSuccess)                                                                    \
      return fail(c, PR_ERR_CUDA, fmt("kernel launch failed: %s (%s:%d)", cudaGetErrorString(e_), \
                                      __FILE__, __LINE__));                                   \
  } while (0)

// Waits for the context stream.  With an NCCL communicator the wait polls instead of blocking:
// ncclCommGetAsyncError reports a failed collective (a peer that died, a network error), and a
// wait longer than PR_OPT_COMM_TIMEOUT_MS (a hung peer that reports nothing) aborts the
// communicator; both poison the context with PR_ERR_NCCL instead of hanging every rank
// (failures are reported, per slice and iteration, not waited on forever).
pr_status sync_stream(pr_ctx *c) {
  if (!c->comm) {
    CU(cudaStreamSynchronize(c->stream));
    return PR_OK;
  }
  const auto t0 = std::chrono::steady_clock::now();
  for (unsigned spin = 0;; ++spin) {
    const cudaError_t q = cudaStreamQuery(c->stream);
    if (q == cudaSuccess) return PR_OK;
    if (q != cudaErrorNotReady) CU(q);
    ncclResult_t ae = 0;
    NC(nccl().CommGetAsyncError(c->comm, &ae));
    if (ae != 0 && ae != kNcclInProgress) {
      nccl().CommAbort(c->comm);
      c->comm = nullptr;
      return fail(c, PR_ERR_NCCL, fmt("NCCL asynchronous error on rank %d: %s", c->rank, nccl().GetErrorString(ae)));
    }
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (c->comm_timeout_ms > 0 && ms > (double)c->comm_timeout_ms) {
      nccl().CommAbort(c->comm);
      c->comm = nullptr;
      return fail(c, PR_ERR_NCCL, fmt("rank %d: stream wait exceeded PR_OPT_COMM_TIMEOUT_MS = %lld ms (a peer rank "
                                      "stalled or died); communicator aborted", c->rank, (long long)c->comm_timeout_ms));
    }
    if (spin > 64) std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
}
#define SYNC()                          \
  do {                                  \
    pr_status s_ = sync_stream(c);      \
    if (s_ != PR_OK) return s_;         \
  } while (0)

pr_status check_ctx(pr_ctx *c) {
  if (!c) return fail(nullptr, PR_ERR_INVALID_ARGUMENT, "ctx is NULL");
  if (c->poisoned) return PR_ERR_STATE;
  // every entry point works on the context's device, whatever the calling thread has current
  const cudaError_t e = cudaSetDevice(c->device);
  if (e != cudaSuccess) return fail(c, PR_ERR_CUDA, fmt("cudaSetDevice(%d): %s", c->device, cudaGetErrorString(e)));
  return PR_OK;
}

// Host fp64 factorisation of I − dτA for (σ, r): m_j, 1/p_j, u_j/p_j (Mp-padded).
pr_status factorise(pr_ctx *c, double dtau, std::vector<double> &m, std::vector<double> &ip,
                    std::vector<double> &cu) {
  const int M = c->M, Mp = c->Mp;
  m.assign((size_t)c->nsets * Mp, 0.0);
  ip.assign((size_t)c->nsets * Mp, 1.0);
  cu.assign((size_t)c->nsets * Mp, 0.0);
  for (int s = 0; s < c->nsets; ++s) {
    const double sg = c->sets[s].first, rr = c->sets[s].second;
    double p_prev = 0, u_prev = 0;
    for (int i = 0; i < M; ++i) {
      const double j = i + 1;
      const double a = 0.5 * sg * sg * j * j, b = 0.5 * rr * j;
      const double d = 1.0 + dtau * (2.0 * a + rr);   // diagonal of I − dτA
      const double l = -dtau * (a - b);               // sub-diagonal (coefficient of V_{j−1})
      const double u = -dtau * (a + b);               // super-diagonal (coefficient of V_{j+1})
      double mm = 0.0, p = d;
      if (i > 0) {
        mm = l / p_prev;
        p = d - mm * u_prev;
      }
      if (!(p > 0.0))
        return fail(c, PR_ERR_NUMERICAL, fmt("non-positive pivot %g at j=%d (sigma=%g r=%g dtau=%g)", p,
                                             i + 1, sg, rr, dtau));
      m[(size_t)s * Mp + i] = mm;
      ip[(size_t)s * Mp + i] = 1.0 / p;
      cu[(size_t)s * Mp + i] = (i < M - 1) ? u / p : 0.0;
      p_prev = p;
      u_prev = u;
    }
  }
  return PR_OK;
}

// K1 zig-zag factors of I − dτA (θ = 1; fine_resident.cuh "zig-zag"): the LU factorisation in
// w = y/p form (w_j = ip_j r_j + nml_j w_{j−1}; back substitution x_j = w_j + ncu_j x_{j+1}) and the
// UL factorisation (pivots q_j from the bottom row up) in w̃ = ỹ/q form (w̃_j = iq_j r_j + nmu_j w̃_{j+1};
// forward substitution x_j = w̃_j + ncl_j x_{j−1}).  Layout [6][nsets][Mp], padding rows identity.
pr_status factorise_zz(pr_ctx *c, double dtau, std::vector<double> &zz) {
  const int M = c->M, Mp = c->Mp, ns = c->nsets;
  zz.assign((size_t)6 * ns * Mp, 0.0);
  auto at = [&](int k, int s, int i) -> double & { return zz[((size_t)k * ns + s) * Mp + i]; };
  std::vector<double> d(M), l(M), u(M), q(M);
  for (int s = 0; s < ns; ++s) {
    const double sg = c->sets[s].first, rr = c->sets[s].second;
    for (int i = 0; i < M; ++i) {
      const double j = i + 1, a = 0.5 * sg * sg * j * j, b = 0.5 * rr * j;
      d[i] = 1.0 + dtau * (2.0 * a + rr);
      l[i] = i > 0 ? -dtau * (a - b) : 0.0;       // coupling to V_{j−1} (none in row 1: V_0 = 0)
      u[i] = i < M - 1 ? -dtau * (a + b) : 0.0;   // coupling to V_{j+1} (row M: the boundary term)
    }
    double p = 0.0;
    for (int i = 0; i < M; ++i) {
      p = i > 0 ? d[i] - l[i] / p * u[i - 1] : d[i];
      if (!(p > 0.0)) return fail(c, PR_ERR_NUMERICAL, fmt("non-positive LU pivot %g at j=%d", p, i + 1));
      at(0, s, i) = 1.0 / p;
      at(1, s, i) = -l[i] / p;
      at(2, s, i) = -u[i] / p;
    }
    q[M - 1] = d[M - 1];
    for (int i = M - 2; i >= 0; --i) q[i] = d[i] - u[i] / q[i + 1] * l[i + 1];
    for (int i = 0; i < M; ++i) {
      if (!(q[i] > 0.0)) return fail(c, PR_ERR_NUMERICAL, fmt("non-positive UL pivot %g at j=%d", q[i], i + 1));
      at(3, s, i) = 1.0 / q[i];
      at(4, s, i) = -l[i] / q[i];
      at(5, s, i) = -u[i] / q[i];
    }
    for (int i = M; i < Mp; ++i) at(0, s, i) = at(3, s, i) = 1.0;
  }
  return PR_OK;
}

// K2R tables (fine_grid.cu): the UL inverse pivots 1/q_j, and per CTA of the grid partition its
// composite maps (↑↑ and ↓↓, from the same closed-form multipliers the kernel uses) and the
// look-back weights P_k = M_{c∓1}·…·M_{c∓(k−1)} up to the window W where max|P| < 1e-24 (K2's
// truncation).  ip: the LU inverse pivots of factorise (row 0 of [nsets][Mp]).
pr_status grid_tables(pr_ctx *c, Scheme &sc, double dtau, const std::vector<double> &ip) {
  int dev = 0, nsm = 0;
  CU(cudaGetDevice(&dev));
  CU(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  int nb = 0;
  const int PT = pr::fine_grid_pt(c->M, nsm, &nb);
  if (!PT) return PR_OK;  // too large for one pass over the GPU: K2 only
  int smem_max = 0;
  CU(cudaDeviceGetAttribute(&smem_max, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
  if (pr::fine_grid_smem(PT, sc.steps) > (size_t)smem_max) return PR_OK;  // boundary terms of very long slices: K2
  const int M = c->M;
  const double sg = c->sets[0].first, rr = c->sets[0].second;
  const double c0 = dtau * (0.5 * rr), c1 = dtau * (0.5 * sg * sg);
  std::vector<double> iq(M), q(M), d(M), l(M), u(M);
  for (int i = 0; i < M; ++i) {
    const double J = i + 1, a = 0.5 * sg * sg * J * J, b = 0.5 * rr * J;
    d[i] = 1.0 + dtau * (2.0 * a + rr);
    l[i] = i > 0 ? -dtau * (a - b) : 0.0;
    u[i] = i < M - 1 ? -dtau * (a + b) : 0.0;
  }
  q[M - 1] = d[M - 1];
  for (int i = M - 2; i >= 0; --i) q[i] = d[i] - u[i] / q[i + 1] * l[i + 1];
  for (int i = 0; i < M; ++i) {
    if (!(q[i] > 0.0)) return fail(c, PR_ERR_NUMERICAL, fmt("non-positive UL pivot %g at j=%d", q[i], i + 1));
    iq[i] = 1.0 / q[i];
  }
  // per-CTA maps in pass order (the kernel's multipliers: closed forms, identity padding)
  const int per = 256 * PT;
  std::vector<double> cm((size_t)2 * nb * 3);
  for (int cb = 0; cb < nb; ++cb) {
    for (int dir = 0; dir < 2; ++dir) {
      double m11 = 1.0, m21 = 0.0, m22 = 1.0;
      for (int k = 0; k < per; ++k) {
        const int j = dir == 0 ? cb * per + k : cb * per + per - 1 - k;
        double a11 = 0.0, a21 = 0.0, a22 = 0.0;
        if (j < M) {
          const double J = j + 1;
          const double lj = (j >= 1) ? -J * std::fma(c1, J, -c0) : 0.0;
          const double uj = (j < M - 1) ? -J * std::fma(c1, J, c0) : 0.0;
          const double pj = ip[j], qj = iq[j];
          if (dir == 0) a11 = -lj * qj, a21 = pj * a11, a22 = -lj * pj;   // ↑↑
          else a11 = -uj * pj, a21 = qj * a11, a22 = -uj * qj;            // ↓↓
        }
        m21 = a21 * m11 + a22 * m21;
        m11 *= a11;
        m22 *= a22;
      }
      double *o = &cm[((size_t)dir * nb + cb) * 3];
      o[0] = m11, o[1] = m21, o[2] = m22;
    }
  }
  // look-back weights
  std::vector<std::vector<double>> P((size_t)2 * nb);
  std::vector<int> W((size_t)2 * nb, 0);
  int KW = 1;
  for (int dir = 0; dir < 2; ++dir)
    for (int cb = 0; cb < nb; ++cb) {
      std::vector<double> &pv = P[(size_t)dir * nb + cb];
      double p11 = 1.0, p21 = 0.0, p22 = 1.0;
      const int maxk = dir == 0 ? cb : nb - 1 - cb;
      int k = 1;
      for (; k <= maxk; ++k) {
        if (std::max(std::fabs(p11), std::max(std::fabs(p21), std::fabs(p22))) < pr::kLookbackEps) break;
        pv.push_back(p11), pv.push_back(p21), pv.push_back(p22);
        const int pc = dir == 0 ? cb - k : cb + k;  // the k-th predecessor: its map joins the product
        const double *mm = &cm[((size_t)dir * nb + pc) * 3];
        p21 = p21 * mm[0] + p22 * mm[1];  // P ← P · M_pc
        p11 *= mm[0];
        p22 *= mm[2];
      }
      W[(size_t)dir * nb + cb] = k - 1;
      KW = std::max(KW, k - 1);
    }
  std::vector<double> lb((size_t)2 * nb * KW * 3, 0.0);
  for (int i = 0; i < 2 * nb; ++i)
    for (size_t e = 0; e < P[i].size(); ++e) lb[(size_t)i * KW * 3 + e] = P[i][e];
  CU(cudaMalloc(&sc.giq, (size_t)M * sizeof(double)));
  CU(cudaMalloc(&sc.lbP, lb.size() * sizeof(double)));
  CU(cudaMalloc(&sc.lbW, W.size() * sizeof(int)));
  CU(cudaMemcpy(sc.giq, iq.data(), (size_t)M * sizeof(double), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(sc.lbP, lb.data(), lb.size() * sizeof(double), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(sc.lbW, W.data(), W.size() * sizeof(int), cudaMemcpyHostToDevice));
  sc.g_pt = PT, sc.g_nb = nb, sc.g_kw = KW, sc.g_c0 = c0, sc.g_c1 = c1;
  return PR_OK;
}

pr_status upload_scheme(pr_ctx *c, Scheme &sc, int steps, double theta) {
  sc.steps = steps;
  sc.dtau = c->dT / steps;
  std::vector<double> m, ip, cu;
  sc.theta = theta;
  const double dti = theta * sc.dtau;  // implicit side I − θdτA
  pr_status st = factorise(c, dti, m, ip, cu);
  if (st) return st;
  const size_t n = m.size();
  CU(cudaMalloc(&sc.m, n * sizeof(double)));
  CU(cudaMalloc(&sc.ip, n * sizeof(double)));
  CU(cudaMalloc(&sc.cu, n * sizeof(double)));
  CU(cudaMemcpy(sc.m, m.data(), n * sizeof(double), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(sc.ip, ip.data(), n * sizeof(double), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(sc.cu, cu.data(), n * sizeof(double), cudaMemcpyHostToDevice));
  if (theta == 1.0 && c->M <= kResidentMaxM) {
    std::vector<double> zz;
    st = factorise_zz(c, dti, zz);
    if (st) return st;
    CU(cudaMalloc(&sc.zz, zz.size() * sizeof(double)));
    CU(cudaMemcpy(sc.zz, zz.data(), zz.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  if (theta == 1.0 && c->M > kResidentMaxM && c->nsets == 1 && c->B == 1 && (st = grid_tables(c, sc, dti, ip)))
    return st;
  // K2: 1/p in the thread-interleaved layout (1 beyond M), the closed-form off-diagonal
  // coefficients, and the per-thread multipliers Π(−l_j/p_j) (dir 0) / Π(−u_j/p_j) (dir 1)
  const int Mt = pr::streamed_Mt(c->M);
  const size_t nthr = (size_t)Mt / pr::kSPS;
  // K2's forward pass runs on w = y/p: multiplier m̃_j = l_j/p_j (none in row 0)
  std::vector<double> mt((size_t)c->nsets * c->Mp, 0.0);
  for (int s = 0; s < c->nsets; ++s)
    for (int i = 1; i < c->M; ++i) {
      const double sg = c->sets[s].first, rr = c->sets[s].second, j = i + 1;
      const double a = 0.5 * sg * sg * j * j, b = 0.5 * rr * j;
      mt[(size_t)s * c->Mp + i] = -dti * (a - b) * ip[(size_t)s * c->Mp + i];
    }
  std::vector<double> iip((size_t)c->nsets * Mt, 1.0), coef((size_t)c->nsets * 2), thB((size_t)2 * c->nsets * nthr);
  for (int s = 0; s < c->nsets; ++s) {
    for (int j = 0; j < c->M; ++j) iip[(size_t)s * Mt + pr::il_index(j)] = ip[(size_t)s * c->Mp + j];
    coef[2 * s] = dti * (0.5 * c->sets[s].second);
    coef[2 * s + 1] = dti * (0.5 * c->sets[s].first * c->sets[s].first);
    for (int dir = 0; dir < 2; ++dir)
      for (size_t q = 0; q < nthr; ++q) {
        double prod = 1.0;
        for (int i = 0; i < pr::kSPS; ++i) {
          const size_t j = q * pr::kSPS + i;
          const double f = j < (size_t)c->M ? (dir == 0 ? mt[(size_t)s * c->Mp + j] : cu[(size_t)s * c->Mp + j]) : 0.0;
          prod *= -f;
        }
        thB[((size_t)dir * c->nsets + s) * nthr + q] = prod;
      }
  }
  // → P_t: product of the multipliers of the threads preceding t in its tile, in pass order
  std::vector<double> thP(thB.size());
  for (int dir = 0; dir < 2; ++dir)
    for (int s = 0; s < c->nsets; ++s)
      for (size_t tile = 0; tile < nthr / pr::kSNT; ++tile) {
        const size_t base = ((size_t)dir * c->nsets + s) * nthr + tile * pr::kSNT;
        double prod = 1.0;
        for (int k = 0; k < pr::kSNT; ++k) {
          const int t = dir == 0 ? k : pr::kSNT - 1 - k;
          thP[base + t] = prod;
          prod *= thB[base + t];
        }
      }
  if (theta != 1.0) {
    // K2 tile-edge corrections (forward passes): PL_t = Π(−m̃_k), k = tile start+1 … thread start−1;
    // tileL = Π(−m̃_k), k = tile start+1 … tile end (m̃ = 0 beyond M)
    const int ntl = pr::streamed_ntiles(c->M);
    std::vector<double> PL((size_t)c->nsets * nthr, 1.0), TL((size_t)c->nsets * ntl);
    for (int s = 0; s < c->nsets; ++s)
      for (int tile = 0; tile < ntl; ++tile) {
        double prod = 1.0;
        const size_t j0 = (size_t)tile * pr::kSTile;
        for (int k = 1; k < pr::kSTile; ++k) {
          if (k % pr::kSPS == 0) PL[(size_t)s * nthr + (size_t)tile * pr::kSNT + k / pr::kSPS] = prod;
          const size_t j = j0 + k;
          prod *= j < (size_t)c->M ? -mt[(size_t)s * c->Mp + j] : -0.0;
        }
        TL[(size_t)s * ntl + tile] = prod;
      }
    CU(cudaMalloc(&sc.PL, PL.size() * sizeof(double)));
    CU(cudaMalloc(&sc.tileL, TL.size() * sizeof(double)));
    CU(cudaMemcpy(sc.PL, PL.data(), PL.size() * sizeof(double), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(sc.tileL, TL.data(), TL.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  CU(cudaMalloc(&sc.iip, iip.size() * sizeof(double)));
  CU(cudaMalloc(&sc.coef, coef.size() * sizeof(double)));
  CU(cudaMalloc(&sc.thrP, thP.size() * sizeof(double)));
  CU(cudaMemcpy(sc.iip, iip.data(), iip.size() * sizeof(double), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(sc.coef, coef.data(), coef.size() * sizeof(double), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(sc.thrP, thP.data(), thP.size() * sizeof(double), cudaMemcpyHostToDevice));
  // K2 look-back data, indexed by scan position (dir 0: tiles ascending, dir 1: descending):
  // tile multiplier B = Π(−l_j/p_j) resp. Π(−u_j/p_j) over the tile, and the window W = number of
  // predecessors whose aggregates are composed: the first W with |Π_{k≤W} B_{pos−k}| below
  // kLookbackEps (all predecessors if never).
  const int nt = pr::streamed_ntiles(c->M);
  std::vector<double> tB((size_t)2 * c->nsets * nt);
  std::vector<int> tW((size_t)2 * c->nsets * nt);
  for (int dir = 0; dir < 2; ++dir)
    for (int s = 0; s < c->nsets; ++s) {
      const size_t base = ((size_t)dir * c->nsets + s) * nt;
      for (int pos = 0; pos < nt; ++pos) {
        const int tile = dir == 0 ? pos : nt - 1 - pos;
        double prod = 1.0;
        for (int j = tile * pr::kSTile; j < std::min((tile + 1) * pr::kSTile, c->M); ++j)
          prod *= dir == 0 ? -mt[(size_t)s * c->Mp + j] : -cu[(size_t)s * c->Mp + j];
        if ((tile + 1) * pr::kSTile > c->M && dir == 0) prod = 0.0;  // identity padding: m = 0
        tB[base + pos] = prod;
      }
      for (int pos = 0; pos < nt; ++pos) {
        double P = 1.0;
        int W = pos;
        for (int k = 1; k <= pos; ++k) {
          P *= tB[base + pos - k];
          if (std::fabs(P) < pr::kLookbackEps) {
            W = k;
            break;
          }
        }
        tW[base + pos] = W;
      }
    }
  CU(cudaMalloc(&sc.tileB, tB.size() * sizeof(double)));
  CU(cudaMalloc(&sc.tileW, tW.size() * sizeof(int)));
  CU(cudaMemcpy(sc.tileB, tB.data(), tB.size() * sizeof(double), cudaMemcpyHostToDevice));
  CU(cudaMemcpy(sc.tileW, tW.data(), tW.size() * sizeof(int), cudaMemcpyHostToDevice));
  std::vector<double> bc(c->B);
  for (int b = 0; b < c->B; ++b) {
    const double sg = c->sig[b], rr = c->r[b], j = c->M;
    bc[b] = sc.dtau * (0.5 * sg * sg * j * j + 0.5 * rr * j);  // dτ (a_M + b_M)
  }
  CU(cudaMalloc(&sc.bcoef, c->B * sizeof(double)));
  CU(cudaMemcpy(sc.bcoef, bc.data(), c->B * sizeof(double), cudaMemcpyHostToDevice));
  sc.g_bcoef = bc[0];
  if (theta != 1.0) {  // explicit part (1−θ)dτ·(σ²/2, r/2, r) per factor set
    std::vector<double> ec((size_t)c->nsets * 3);
    const double dte = (1.0 - theta) * sc.dtau;
    for (int s = 0; s < c->nsets; ++s) {
      const double sg = c->sets[s].first, rr = c->sets[s].second;
      ec[3 * s] = dte * (0.5 * sg * sg);
      ec[3 * s + 1] = dte * (0.5 * rr);
      ec[3 * s + 2] = dte * rr;
    }
    CU(cudaMalloc(&sc.ecoef, ec.size() * sizeof(double)));
    CU(cudaMemcpy(sc.ecoef, ec.data(), ec.size() * sizeof(double), cudaMemcpyHostToDevice));
  }
  return PR_OK;
}

void free_scheme(Scheme &s) {
  cudaFree(s.tileB);
  cudaFree(s.tileW);
  cudaFree(s.iip);
  cudaFree(s.coef);
  cudaFree(s.thrP);
  cudaFree(s.m);
  cudaFree(s.ip);
  cudaFree(s.cu);
  cudaFree(s.zz);
  cudaFree(s.giq);
  cudaFree(s.lbP);
  cudaFree(s.lbW);
  cudaFree(s.bcoef);
  cudaFree(s.ecoef);
  cudaFree(s.PL);
  cudaFree(s.tileL);
  s = Scheme();
}

pr::StreamedProblem sprob(const pr_ctx *c, const Scheme &sc) {
  pr::StreamedProblem p;
  p.f.ip = sc.iip;
  p.f.coef = sc.coef;
  p.f.thrP = sc.thrP;
  p.f.tileB = sc.tileB;
  p.f.tileW = sc.tileW;
  p.nsets = c->nsets;
  p.fset = c->d_fset;
  p.bcoef = sc.bcoef;
  p.L = c->d_L;
  p.K = c->d_K;
  p.r = c->d_r;
  p.upper_bc = c->upper_bc;
  p.dT = c->dT;
  p.dtau = sc.dtau;
  p.theta = sc.theta;
  p.f.ecoef = sc.ecoef;
  p.f.PL = sc.PL;
  p.f.tileL = sc.tileL;
  p.steps = sc.steps;
  p.M = c->M;
  p.Mp = c->Mp;
  p.B = c->B;
  return p;
}

bool use_resident(const pr_ctx *c) {
  if (c->opt_fine_kernel == 1) return true;
  if (c->opt_fine_kernel == 2) return false;
  return c->M <= kResidentMaxM;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

size_t layout(pr_ctx *c, char *base) {
  // carve the workspace; returns total bytes.  base == nullptr → size only.
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char *p = base ? base + off : nullptr;
    off = align_up(off + bytes, 256);
    return p;
  };
  const size_t row = (size_t)c->B * c->Mp;
  c->U = (float *)take((size_t)(c->Nloc + 1) * row * sizeof(float));
  c->Gh = (float *)take((size_t)std::max(c->Nloc, 1) * row * sizeof(float));
  c->D = (float *)take((size_t)std::max(c->Nloc, 1) * row * sizeof(float));
  c->Fk = (float *)take(2 * row * sizeof(float));  // (two rows for the pipelined schedule)
  c->tmp = (float *)take(2 * row * sizeof(float));
  c->partials = (double *)take((size_t)(c->Nloc + 1) * c->B * c->nch * 2 * sizeof(double));
  c->d_delta = (unsigned long long *)take((size_t)c->max_iter * sizeof(unsigned long long));
  char *sb = take(pr::streamed_state_bytes(c->M, c->Mp, c->B, std::max(c->Nloc, 1)));
  if (base) pr::streamed_state_bind(c->sst, sb, c->M, c->Mp, c->B, std::max(c->Nloc, 1));
  return off;
}

pr_status ensure_ws(pr_ctx *c) {
  if (c->ws_ready) return PR_OK;
  const size_t need = layout(c, nullptr);
  if (!c->ws) {
    CU(cudaMalloc(&c->ws, need));
    c->own_ws = true;
    c->ws_bytes = need;
  }
  layout(c, (char *)c->ws);
  CU(cudaMemsetAsync(c->ws, 0, need, c->stream));
  c->ws_ready = true;
  return PR_OK;
}

cudaEvent_t next_event(pr_ctx *c) {
  if (c->ev_used >= (int)c->ev.size()) {
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
    c->ev.push_back(e);
  }
  return c->ev[c->ev_used++];
}

// ---------------------------------------------------------------- resident launches
bool use_split_pinn(const pr_ctx *c);
int split_G(const pr_ctx *c);
// The K1 kernels run the zig-zag form (fine_resident.cuh) for implicit Euler schemes, except in
// problems whose PINN chain is a group kernel: the pipelined kernel of those has 384-thread CTAs
// (168 registers per thread), too few for the zig-zag solver, and the blocking kernels of a
// problem must do the pipelined kernel's arithmetic (bitwise-equal schedules).
bool use_zz(const pr_ctx *c, const Scheme &sc) {
  if (sc.theta != 1.0 || !sc.zz) return false;
  if (c->coarse == PR_COARSE_PINN && c->have_pinn && !c->tc && use_split_pinn(c) &&
      pr::pinn_split_is_group(c->W, split_G(c)))
    return false;
  return true;
}
pr::ResidentArgs base_args(pr_ctx *c, const Scheme &sc) {
  pr::ResidentArgs a;
  std::memset(&a, 0, sizeof a);
  a.M = c->M;
  a.Mp = c->Mp;
  a.B = c->B;
  a.fm = sc.m;
  a.fip = sc.ip;
  a.fcu = sc.cu;
  a.zz = sc.zz;
  a.nsets = c->nsets;
  a.use_zz = use_zz(c, sc) ? 1 : 0;
  a.fset = c->d_fset;
  a.bcoef = sc.bcoef;
  a.theta = sc.theta;
  a.ecoef = sc.ecoef;
  a.Lb = c->d_L;
  a.Kb = c->d_K;
  a.rb = c->d_r;
  a.upper_bc = c->upper_bc;
  a.dT = c->dT;
  a.dtau = sc.dtau;
  a.steps = sc.steps;
  a.n_base = c->n0;
  a.fk_ln = -1;
  a.nch = c->nch;
  a.ustride = (size_t)c->B * c->Mp;
  return a;
}

cudaError_t dispatch_res(bool chain, int M, const pr::ResidentArgs &a, int nsys, cudaStream_t s) {
  return pr::launch_resident(chain, M, a, nsys, s);
}

// ---------------------------------------------------------------- PINN launches
// Few grid points (B·M ≤ kSplitMaxPoints): the coarse chain is latency-bound, so a latency mode
// runs it with G threads per point (split_G): the group kernels (pinn_group_G(W) threads, shared-
// memory exchange, group-ordered weights) while B·M ≤ kGroupMaxPoints, where one thread per
// point leaves most SMs idle; 20-wide nets beyond that use the 4-thread shuffle kernel.  Otherwise
// constant-bank weights when instantiated, else shared-memory weights.
// PR_OPT_PINN_KERNEL: 0 auto, 1 shared memory, 2 latency mode.
constexpr long kSplitMaxPoints = 65536;
constexpr long kGroupMaxPoints = 16384;
// PR_PREC_*_TC → the K4 operand mode (pinn_tc.cu)
int tc_mode(int precision) {
  return precision == PR_PREC_FP16_TC ? pr::kTcSplit16 : precision == PR_PREC_BF16_TC ? pr::kTcBF16 : pr::kTcF16;
}
bool split_allowed(const pr_ctx *c) { return (long)c->B * c->M <= kSplitMaxPoints; }
// 20-wide nets: in a problem the pipelined schedule can run (one GPU, fixed K, resident fine
// kernel, M ≤ 1024) the 4-thread shuffle chain, whose 4-warp chain CTAs pack several per SM
// beside the fine CTAs (measured 0.281 vs 0.287 ms per C2 solve with the group chain); elsewhere
// the group kernel (blocking C2: 0.38 vs 0.43 ms).  The choice depends on the problem only, not on
// PR_OPT_PIPELINE, so both schedules of one context use the same evaluator (bitwise-equal results).
// (independent of the rank count, so a problem's evaluator — and its results — are the same on any R)
bool pipe_shape(const pr_ctx *c) {
  return c->tol == 0.0 && c->max_iter >= 1 && !c->tc && c->coarse == PR_COARSE_PINN && use_resident(c) &&
         c->M <= 1024;
}
int split_G(const pr_ctx *c) {
  const bool small = (long)c->B * c->M <= kGroupMaxPoints;
  if (c->W == 20) return small && !pipe_shape(c) ? pr::pinn_group_G(20) : pr::kPinnSplitG;
  if (pr::pinn_group_G(c->W) > 0 && (small || c->opt_pinn_kernel == 2)) return pr::pinn_group_G(c->W);
  return 0;
}
bool use_split_pinn(const pr_ctx *c) {
  if (c->tc || c->opt_pinn_kernel == 1) return false;
  if (c->opt_pinn_kernel == 0 && !split_allowed(c)) return false;
  const int G = split_G(c);
  return G > 0 && pr::pinn_split_supported(c->IN, c->W, c->act, G);
}
bool use_param_pinn(const pr_ctx *c) {
  if (c->tc || c->opt_pinn_kernel != 0 || use_split_pinn(c)) return false;
  return pr::pinn_param_supported(c->IN, c->W, c->LH, c->act);
}

pr::PinnArgs pinn_args(pr_ctx *c) {
  pr::PinnArgs a;
  std::memset(&a, 0, sizeof a);
  a.M = c->M;
  a.Mp = c->Mp;
  a.B = c->B;
  a.wts = c->d_wts;
  a.nfloats = c->nfloats;
  a.LH = c->LH;
  a.cs0 = c->cs[0];
  a.cs1 = c->cs[1];
  a.cs2 = c->cs[2];
  a.cs3 = c->cs[3];
  a.out_scale = c->out_scale;
  a.T = c->T;
  a.dT = c->dT;
  a.n_base = c->n0;
  a.Lb = c->d_L;
  a.nch = c->nch;
  return a;
}

// CTA geometry of the PINN chain along j: points per CTA and CTAs per instance row of the
// evaluator launch_pinn picks (a j-chunk of the chain is a CTA range, so a chunked chain does the
// arithmetic of the whole one, δ partial slots included).
void pinn_geometry(const pr_ctx *c, int *ppc, int *gx) {
  int p;
  if (c->tc) p = pr::pinn_tc_points_per_cta(c->W, c->LH, c->tc_nfloats, tc_mode(c->tc));
  else if (use_split_pinn(c)) p = pr::pinn_split_ppc(split_G(c));
  else if (use_param_pinn(c)) p = kPinnTPB;
  else p = kPinnTPB * pr::pinn_smem_pts(c->W);
  *ppc = p;
  *gx = (c->M + p - 1) / p;
}

// The PINN chain over the CTAs [cta_lo, cta_hi) along j (cta_hi < 0: all of them).
pr_status launch_pinn(pr_ctx *c, const pr::PinnArgs &a0, int cta_lo = 0, int cta_hi = -1) {
  int ppc, gx;
  pinn_geometry(c, &ppc, &gx);
  if (cta_hi < 0) cta_hi = gx;
  if (cta_hi <= cta_lo) return PR_OK;
  pr::PinnArgs a = a0;
  a.cta0 = cta_lo;
  const dim3 grid(cta_hi - cta_lo, c->B);
  if (c->tc) {  // K4: tensor cores (wide nets)
    pr::PinnArgs t = a;
    t.wts = c->d_tcp;
    t.nfloats = c->tc_nfloats;
    LAUNCH(pr::launch_pinn_tc(c->IN, c->W, c->act, tc_mode(c->tc), t, c->d_wh, grid, c->stream));
    return PR_OK;
  }
  if (use_split_pinn(c)) {
    const int G = split_G(c);
    pr::PinnArgs t = a;
    if (pr::pinn_split_is_group(c->W, G)) t.wts = c->d_wgrp;  // group kernels: hidden matrices in the group order
    LAUNCH(pr::launch_pinn_split(c->IN, c->W, c->act, G, t, grid, (size_t)c->nfloats * sizeof(float), c->stream));
    return PR_OK;
  }
  if (use_param_pinn(c)) {
    LAUNCH(pr::launch_pinn_param(c->IN, c->W, c->LH, c->act, c->h_wts.data(), a, grid, c->stream));
    return PR_OK;
  }
  if (!pr::pinn_smem_supported(c->IN, c->W, c->act)) return fail(c, PR_ERR_UNSUPPORTED, "no PINN kernel for this width");
  LAUNCH(pr::launch_pinn_smem(c->IN, c->W, c->act, a, grid, (size_t)c->nfloats * sizeof(float), c->stream));
  return PR_OK;
}

// ---------------------------------------------------------------- K2R grid-resident fine sweep
// Used for θ = 1, one instance, M > kResidentMaxM when the partition fits the GPU and the cost
// model below predicts it ahead of K2 (auto), or forced with PR_OPT_FINE_KERNEL = 3.  The model
// (µs per fine step of the sweep; constants fitted to scripts/grid_vs_k2.py on B200,
// profiles/r02/grid_vs_k2.txt, M = 2^12 … 2^20, 4 … 64 systems, within ~15 %):
//   K2    12 + 16 B · M · nsys / 4.4 TB/s             (launch/look-back floor + HBM streaming)
//   grid  ⌈nsys / NS⌉ · (0.4 + 3.5 · nCTA/148 + 0.5 · NS)  (one latency-bound pass per group)
// e.g. 2^18 … 2^20 points: grid ahead at every count (1.7× at 64 systems of 2^20); 2^12 … 2^16
// points: grid up to ~16 systems, K2 beyond (its cost stays near the floor, the grid's grows
// per group).
bool use_grid(const pr_ctx *c, int nsys) {
  // (not with the in-process loopback transport: its ranks share one GPU, and the cooperative
  // grid of one rank cannot be co-resident with another's)
  if (!c->fine.g_pt || c->loop || c->opt_fine_kernel == 1 || c->opt_fine_kernel == 2) return false;
  if (c->opt_fine_kernel == 3) return true;
  if (c->M <= kResidentMaxM) return false;
  const double k2 = 12.0 + 16.0 * (double)c->M * nsys / 4.4e6;
  const int ns = pr::fine_grid_ns(c->fine.g_pt, nsys);
  const double grid = (double)((nsys + ns - 1) / ns) * (0.4 + 3.5 * c->fine.g_nb / 148.0 + 0.5 * ns);
  return grid < k2;
}
pr_status ensure_grid(pr_ctx *c) {
  if (c->g_tot) return PR_OK;
  const int nb = c->fine.g_nb;
  c->g_tot_words = pr::fine_grid_tot_words(nb);
  CU(cudaMalloc(&c->g_tot, c->g_tot_words * sizeof(unsigned long long)));
  CU(cudaHostAlloc((void **)&c->g_err_h, sizeof(int), cudaHostAllocMapped));
  *c->g_err_h = 0;
  CU(cudaHostGetDevicePointer((void **)&c->g_err_d, c->g_err_h, 0));
  return PR_OK;
}
// One grid sweep over the local slices [ln0, ln0+nsl): D (or F̂ into Fk / Fout)
pr_status grid_sweep(pr_ctx *c, int ln0, int nsl, int n_base, const float *U, float *Fout, int fk_ln) {
  pr_status st = ensure_grid(c);
  if (st) return st;
  const Scheme &sc = c->fine;
  pr::GridArgs g;
  std::memset(&g, 0, sizeof g);
  g.M = c->M;
  g.nsys = nsl;
  g.ln0 = ln0;
  g.n_base = n_base;
  g.steps = sc.steps;
  g.row = (size_t)c->B * c->Mp;
  g.dT = c->dT;
  g.dtau = sc.dtau;
  g.c0 = sc.g_c0;
  g.c1 = sc.g_c1;
  g.ip = sc.ip;
  g.iq = sc.giq;
  g.bcoef = sc.g_bcoef;
  g.Lb = c->L[0];
  g.Kb = c->K[0];
  g.rb = c->r[0];
  g.upper_bc = c->upper_bc;
  g.lbP = sc.lbP;
  g.lbW = sc.lbW;
  g.KW = sc.g_kw;
  g.tot = c->g_tot;
  g.err = c->g_err_d;
  g.U = U;
  g.Gh = c->Gh;
  g.D = c->D;
  g.Fk = c->Fk;
  g.Fout = Fout;
  g.fk_ln = fk_ln;
  CU(cudaMemsetAsync(c->g_tot, 0, c->g_tot_words * sizeof(unsigned long long), c->stream));  // tags 0
  // PR_GRID_TRACE=file (tuning): %globaltimer stamps per pass and CTA, written after the launch
  static const char *trace_path = getenv("PR_GRID_TRACE");
  const int ns = pr::fine_grid_ns(sc.g_pt, nsl);
  const size_t npass = (size_t)((nsl + ns - 1) / ns) * (sc.steps + 1);
  unsigned long long *trace = nullptr;
  if (trace_path && !c->capturing) {
    CU(cudaMalloc(&trace, npass * sc.g_nb * 5 * sizeof(unsigned long long)));
    CU(cudaMemsetAsync(trace, 0, npass * sc.g_nb * 5 * sizeof(unsigned long long), c->stream));
    g.trace = trace;
  }
  LAUNCH(pr::launch_fine_grid(g, sc.g_pt, sc.g_nb, c->stream));
  if (trace) {
    std::vector<unsigned long long> h(npass * sc.g_nb * 5);
    CU(cudaMemcpyAsync(h.data(), trace, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    SYNC();
    cudaFree(trace);
    if (FILE *f = fopen(trace_path, "w")) {
      for (size_t ps = 0; ps < npass; ++ps)
        for (int cb = 0; cb < sc.g_nb; ++cb) {
          const unsigned long long *r = &h[(ps * sc.g_nb + cb) * 5];
          fprintf(f, "%zu %d %llu %llu %llu %llu %llu\n", ps, cb, r[0], r[1], r[2], r[3], r[4]);
        }
      fclose(f);
    }
  }
  return PR_OK;
}
// after a sync: a look-back wait that timed out (a failed launch or a lost CTA) fails the solve
pr_status grid_check(pr_ctx *c) {
  if (c->g_err_h && *c->g_err_h) {
    *c->g_err_h = 0;
    return fail(c, PR_ERR_CUDA, "grid-resident fine sweep: look-back wait timed out");
  }
  return PR_OK;
}

// ---------------------------------------------------------------- phases of one iteration
// Fine sweep over local slices [ln_lo, Nloc) reading U^{k−1}: D_n = F̂_n − Ĝ_n, and
// F̂ of local slice fk_ln (= k−1 when owned here) into Fk.
pr_status fine_sweep(pr_ctx *c, int ln_lo, int fk_ln) {
  const int nsl = c->Nloc - ln_lo;
  if (nsl <= 0) return PR_OK;
  if (use_grid(c, nsl)) return grid_sweep(c, ln_lo, nsl, c->n0, c->U, nullptr, fk_ln);
  if (use_resident(c)) {
    pr::ResidentArgs a = base_args(c, c->fine);
    a.ln0 = ln_lo;
    a.nsl = nsl;
    a.U = c->U;
    a.Gh = c->Gh;
    a.D = c->D;
    a.Fk = c->Fk;
    a.fk_ln = fk_ln;
    LAUNCH(dispatch_res(false, c->M, a, nsl * c->B, c->stream));
    return PR_OK;
  }
  pr::StreamedJob j;
  j.U = c->U; j.Gh = c->Gh; j.D = c->D; j.Fk = c->Fk; j.fk_ln = fk_ln; j.Fout = nullptr;
  j.ln0 = ln_lo; j.nsl = nsl; j.n_base = c->n0;
  int nl = 0;
  cudaError_t e = pr::streamed_sweep(c->sst, sprob(c, c->fine), j, c->stream, &nl);
  c->launches += nl;
  if (e != cudaSuccess) return fail(c, PR_ERR_CUDA, fmt("streamed sweep: %s", cudaGetErrorString(e)));
  return PR_OK;
}

// Coarse chain with correction over local slices [ln0, Nloc).  k == 0: no correction, no δ.
// PINN G: only the CTAs [cta_lo, cta_hi) along j (a wavefront chunk; cta_hi < 0: all).
pr_status coarse_chain(pr_ctx *c, int k, int ln0, bool copy, int cta_lo = 0, int cta_hi = -1) {
  const bool corr = k > 0;
  if (c->coarse == PR_COARSE_PINN) {
    pr::PinnArgs a = pinn_args(c);
    a.ln0 = ln0;
    a.ln1 = c->Nloc;
    a.U = c->U;
    a.Gh = c->Gh;
    a.D = corr ? c->D : nullptr;
    a.Fcopy = copy ? c->Fk : nullptr;
    a.partials = corr ? c->partials : nullptr;
    if (ln0 >= c->Nloc && !copy) return PR_OK;
    if (ln0 >= c->Nloc) {  // copy only (chain empty): still need U_k := F̂_{k−1} and its δ
      a.ln1 = ln0;
    }
    return launch_pinn(c, a, cta_lo, cta_hi);
  }
  if (!use_resident(c)) {
    pr::StreamedChainJob j;
    j.U = c->U; j.Gh = c->Gh; j.D = corr ? c->D : nullptr; j.Fcopy = copy ? c->Fk : nullptr;
    j.partials = corr ? c->partials : nullptr; j.nch = c->nch;
    j.ln0 = ln0; j.ln1 = c->Nloc; j.n_base = c->n0; j.ustride = (size_t)c->B * c->Mp;
    int nl = 0;
    cudaError_t e = pr::streamed_chain(c->sst, sprob(c, c->crs), j, c->stream, &nl);
    c->launches += nl;
    if (e != cudaSuccess) return fail(c, PR_ERR_CUDA, fmt("streamed chain: %s", cudaGetErrorString(e)));
    return PR_OK;
  }
  pr::ResidentArgs a = base_args(c, c->crs);
  a.Uw = c->U;
  a.GhW = c->Gh;
  a.Dc = corr ? c->D : nullptr;
  a.Fcopy = copy ? c->Fk : nullptr;
  a.c_ln0 = ln0;
  a.c_ln1 = c->Nloc;
  a.partials = corr ? c->partials : nullptr;
  if (ln0 >= c->Nloc && !copy) return PR_OK;
  LAUNCH(dispatch_res(true, c->M, a, c->B, c->stream));
  return PR_OK;
}

// ---------------------------------------------------------------- rank transport
// NCCL between processes (one per GPU), or — for tests on a single GPU — an in-process loopback:
// contexts whose 128-byte id starts with "PRLOOPBK" and shares the rest form a group whose ranks
// (each driven by its own host thread) hand the same rows through device mailboxes, fully
// synchronously.  The schedule, kernels and buffers are those of the NCCL path; only the three
// transport calls below differ.
struct LoopGroup {
  int world = 0, refs = 0;
  std::mutex mu;
  std::condition_variable cv;
  // [src·world + dst] FIFO of device messages: a send never blocks (like NCCL's grouped p2p, any
  // number of messages may be in flight per pair), a receive takes the oldest
  std::vector<std::deque<std::pair<void *, size_t>>> box;
  std::vector<unsigned long long> vals;  // all-reduce contributions (bit patterns of doubles ≥ 0)
  unsigned long long result = 0;
  std::vector<std::vector<double>> sums;  // SUM all-reduce contributions
  std::vector<double> sum_result;
  int arrived = 0, gen = 0;
};
std::mutex g_loop_mu;
std::map<std::string, LoopGroup *> g_loops;
const char kLoopMagic[8] = {'P', 'R', 'L', 'O', 'O', 'P', 'B', 'K'};

bool loop_id(const uint8_t *id) { return id && std::memcmp(id, kLoopMagic, 8) == 0; }
LoopGroup *loop_join(const uint8_t *id, int world) {
  std::lock_guard<std::mutex> lk(g_loop_mu);
  const std::string key((const char *)id + 8, 120);
  LoopGroup *&g = g_loops[key];
  if (!g) {
    g = new LoopGroup;
    g->world = world;
    g->box.assign((size_t)world * world, {});
    g->vals.assign(world, 0);
    g->sums.assign(world, {});
  }
  if (g->world != world) return nullptr;
  g->refs++;
  return g;
}
void loop_leave(LoopGroup *g) {
  std::lock_guard<std::mutex> lk(g_loop_mu);
  if (--g->refs > 0) return;
  for (auto &q : g->box)
    for (auto &m : q) cudaFree(m.first);
  for (auto it = g_loops.begin(); it != g_loops.end(); ++it)
    if (it->second == g) {
      g_loops.erase(it);
      break;
    }
  delete g;
}

pr_status comm_send(pr_ctx *c, const float *buf, size_t count, int peer) {
  if (!c->loop) {
    NC(nccl().Send(buf, count, kNcclFloat32, peer, c->comm, c->stream));
    return PR_OK;
  }
  LoopGroup *g = c->loop;
  const size_t bytes = count * sizeof(float), idx = (size_t)c->rank * g->world + peer;
  SYNC();  // the row is complete
  void *m = nullptr;
  CU(cudaMalloc(&m, bytes ? bytes : 4));
  CU(cudaMemcpy(m, buf, bytes, cudaMemcpyDeviceToDevice));
  std::lock_guard<std::mutex> lk(g->mu);
  g->box[idx].push_back({m, bytes});
  g->cv.notify_all();
  return PR_OK;
}
pr_status comm_recv(pr_ctx *c, float *buf, size_t count, int peer) {
  if (!c->loop) {
    NC(nccl().Recv(buf, count, kNcclFloat32, peer, c->comm, c->stream));
    return PR_OK;
  }
  LoopGroup *g = c->loop;
  const size_t bytes = count * sizeof(float), idx = (size_t)peer * g->world + c->rank;
  SYNC();  // earlier work reading buf is done
  std::pair<void *, size_t> m;
  {
    std::unique_lock<std::mutex> lk(g->mu);
    g->cv.wait(lk, [&] { return !g->box[idx].empty(); });
    m = g->box[idx].front();
    g->box[idx].pop_front();
  }
  if (m.second != bytes) {
    cudaFree(m.first);
    return fail(c, PR_ERR_STATE, fmt("loopback message from rank %d has %zu bytes, expected %zu", peer, m.second, bytes));
  }
  CU(cudaMemcpy(buf, m.first, bytes, cudaMemcpyDeviceToDevice));
  CU(cudaFree(m.first));
  return PR_OK;
}
// SUM over ranks of `count` doubles in place (loopback: summed in rank order on the host)
pr_status comm_allreduce_sum(pr_ctx *c, double *buf, size_t count) {
  if (!c->loop) {
    NC(nccl().AllReduce(buf, buf, count, kNcclFloat64, kNcclSum, c->comm, c->stream));
    return PR_OK;
  }
  LoopGroup *g = c->loop;
  std::vector<double> mine(count);
  SYNC();
  CU(cudaMemcpy(mine.data(), buf, count * sizeof(double), cudaMemcpyDeviceToHost));
  std::vector<double> res;
  {
    std::unique_lock<std::mutex> lk(g->mu);
    const int my_gen = g->gen;
    g->sums[c->rank] = std::move(mine);
    if (++g->arrived == g->world) {
      g->sum_result.assign(count, 0.0);
      for (int q = 0; q < g->world; ++q)
        for (size_t i = 0; i < count; ++i) g->sum_result[i] += g->sums[q][i];
      g->arrived = 0;
      g->gen++;
      g->cv.notify_all();
    } else {
      g->cv.wait(lk, [&] { return g->gen != my_gen; });
    }
    res = g->sum_result;
  }
  CU(cudaMemcpy(buf, res.data(), count * sizeof(double), cudaMemcpyHostToDevice));
  return PR_OK;
}
// MAX over ranks of one non-negative double held as its bit pattern (δ, reading Q13)
pr_status comm_allreduce_max(pr_ctx *c, unsigned long long *slot) {
  if (!c->loop) {
    NC(nccl().AllReduce(slot, slot, 1, kNcclFloat64, kNcclMax, c->comm, c->stream));
    return PR_OK;
  }
  LoopGroup *g = c->loop;
  unsigned long long v = 0;
  SYNC();
  CU(cudaMemcpy(&v, slot, sizeof v, cudaMemcpyDeviceToHost));
  unsigned long long res;
  {
    std::unique_lock<std::mutex> lk(g->mu);
    const int my_gen = g->gen;
    g->vals[c->rank] = v;
    if (++g->arrived == g->world) {
      unsigned long long m = 0;
      for (unsigned long long x : g->vals) m = x > m ? x : m;
      g->result = m;
      g->arrived = 0;
      g->gen++;
      g->cv.notify_all();
    } else {
      g->cv.wait(lk, [&] { return g->gen != my_gen; });
    }
    res = g->result;  // (the next generation needs this rank's arrival first)
  }
  CU(cudaMemcpy(slot, &res, sizeof res, cudaMemcpyHostToDevice));
  return PR_OK;
}

// One wavefront hand-off: send `scount` values to `speer` and receive `rcount` from `rpeer` (either
// may be absent: count 0).  NCCL: one group, so the send of chunk c−1 and the receive of chunk c
// progress together; loopback: the send, then the receive.
pr_status comm_sendrecv(pr_ctx *c, const float *sbuf, size_t scount, int speer, float *rbuf, size_t rcount, int rpeer) {
  if (!c->loop) {
    NC(nccl().GroupStart());
    if (scount) NC(nccl().Send(sbuf, scount, kNcclFloat32, speer, c->comm, c->stream));
    if (rcount) NC(nccl().Recv(rbuf, rcount, kNcclFloat32, rpeer, c->comm, c->stream));
    NC(nccl().GroupEnd());
    return PR_OK;
  }
  pr_status st;
  if (scount && (st = comm_send(c, sbuf, scount, speer))) return st;
  if (rcount && (st = comm_recv(c, rbuf, rcount, rpeer))) return st;
  return PR_OK;
}

// Chunks of the PINN chain's wavefront across ranks: G is pointwise in S, so the
// chain of grid-point chunk q needs only chunk q of U_{n0} from the previous rank; a rank hands on
// each chunk of U_{n1} as soon as its chain has finished it and the next rank starts on it while
// this one chains the next chunk.  Coarse time per iteration ≈ (1 + (R−1)/C)·t_rank instead of
// R·t_rank.  Pointwise G and one instance row (contiguous chunks) only; 1 = the blocking chain.
int wavefront_chunks(const pr_ctx *c) {
  if (c->world == 1 || c->coarse != PR_COARSE_PINN || c->B != 1 || c->opt_wavefront == 1) return 1;
  int ppc, gx;
  pinn_geometry(c, &ppc, &gx);
  const int want = c->opt_wavefront >= 2 ? c->opt_wavefront : (c->M >= (1 << 16) ? 8 : 1);
  return std::max(1, std::min(want, gx));
}

// The chain of iteration k on this rank with the receive of U_{n0} before it and the send of
// U_{n1} after it (plan P), as one blocking exchange or as a chunk wavefront.
pr_status chain_exchange(pr_ctx *c, int k, const pr_plan &P, bool run_chain, double *ms_comm_unused) {
  (void)ms_comm_unused;
  const size_t row = (size_t)c->B * c->Mp;
  float *u_in = c->U, *u_out = c->U + (size_t)c->Nloc * row;
  const int r = c->rank, C = wavefront_chunks(c);
  pr_status st;
  if (C <= 1) {
    if (P.recv_first && (st = comm_recv(c, u_in, row, r - 1))) return st;
    if (run_chain && (st = coarse_chain(c, k, P.chain_lo, P.copy != 0))) return st;
    if (P.send_last && (st = comm_send(c, u_out, row, r + 1))) return st;
    return PR_OK;
  }
  int ppc, gx;
  pinn_geometry(c, &ppc, &gx);
  auto jr = [&](int q, int *lo, int *hi) {  // grid points of chunk q (CTA-aligned)
    const int c0 = (int)((long)q * gx / C), c1 = (int)((long)(q + 1) * gx / C);
    *lo = std::min(c0 * ppc, c->M);
    *hi = std::min(c1 * ppc, c->M);
    return std::make_pair(c0, c1);
  };
  int plo = 0, phi = 0;  // previous chunk (to send)
  for (int q = 0; q < C; ++q) {
    int lo, hi;
    const auto ctas = jr(q, &lo, &hi);
    const size_t sc = (q > 0 && P.send_last) ? (size_t)(phi - plo) : 0, rc = P.recv_first ? (size_t)(hi - lo) : 0;
    if ((sc || rc) && (st = comm_sendrecv(c, u_out + plo, sc, r + 1, u_in + lo, rc, r - 1))) return st;
    if (run_chain && (st = coarse_chain(c, k, P.chain_lo, P.copy != 0, ctas.first, ctas.second))) return st;
    plo = lo, phi = hi;
  }
  if (P.send_last && (st = comm_send(c, u_out + plo, (size_t)(phi - plo), r + 1))) return st;
  return PR_OK;
}

pr_status delta_reduce(pr_ctx *c, int k, int ln_lo, int ln_hi, int nch) {
  unsigned long long *slot = c->d_delta + (k - 1);
  CU(cudaMemsetAsync(slot, 0, sizeof(unsigned long long), c->stream));
  if (ln_hi >= ln_lo) {
    const int total = (ln_hi - ln_lo + 1) * c->B;
    (void)total;
    LAUNCH(pr::launch_delta(c->partials, c->B, nch, ln_lo, ln_hi, slot, c->stream));
  }
  if (c->world > 1) return comm_allreduce_max(c, slot);
  return PR_OK;
}

pr_status load_initial(pr_ctx *c, const float *V_T, bool device_ptr) {
  const size_t row = (size_t)c->B * c->Mp;
  if (V_T) {
    if (c->Mp == c->M) {
      CU(cudaMemcpyAsync(c->U, V_T, row * sizeof(float),
                         device_ptr ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream));
    } else {
      CU(cudaMemcpy2DAsync(c->U, c->Mp * sizeof(float), V_T, c->M * sizeof(float), c->M * sizeof(float), c->B,
                           device_ptr ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, c->stream));
    }
  } else {
    LAUNCH(pr::launch_payoff(c->U, c->M, c->Mp, c->B, c->d_L, c->d_K, c->stream));
  }
  return PR_OK;
}

pr_status store_rows(pr_ctx *c, float *dst, const float *src, bool device_ptr) {
  if (c->Mp == c->M) {
    CU(cudaMemcpyAsync(dst, src, (size_t)c->B * c->M * sizeof(float),
                       device_ptr ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
  } else {
    CU(cudaMemcpy2DAsync(dst, c->M * sizeof(float), src, c->Mp * sizeof(float), c->M * sizeof(float), c->B,
                         device_ptr ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, c->stream));
  }
  return PR_OK;
}

// Timing events; under stream capture they must be captured as timestamp (external) nodes.
void record(pr_ctx *c, cudaEvent_t e) {
  if (c->capturing && c->opt_graphs == 2) return;  // lean graph: no timing nodes
  if (c->capturing) cudaEventRecordWithFlags(e, c->stream, cudaEventRecordExternal);
  else cudaEventRecord(e, c->stream);
}

struct PhaseTimer {
  pr_ctx *c;
  std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>> spans;
  cudaEvent_t a = nullptr;
  int cur = -1;
  nvtxRangeId_t rid = 0;
  void begin(int phase) {
    static const char *const names[] = {"pr: coarse chain", "pr: fine sweep", "pr: exchange", "pr: setup"};
    rid = nvtxRangeStartA(names[phase & 3]);  // host-side phase range (nsys / ncu --nvtx)
    a = next_event(c);
    cur = phase;
    if (a) record(c, a);
  }
  void end() {
    cudaEvent_t b = next_event(c);
    if (a && b) {
      record(c, b);
      spans.push_back({cur, {a, b}});
    }
    nvtxRangeEnd(rid);
  }
};
enum { PH_COARSE = 0, PH_FINE = 1, PH_COMM = 2, PH_SETUP = 3 };

// The per-rank schedule of iteration k (include/parareal.h pr_plan).
pr_plan make_plan(int N, int world, int rank, int k) {
  const int per = N / world, n0 = rank * per, n1 = n0 + per;
  pr_plan P;
  std::memset(&P, 0, sizeof P);
  P.fk_local = -1;
  P.delta_lo = 1;
  P.delta_hi = 0;
  if (k == 0) {  // initial coarse sweep U_{n+1} = G(U_n)
    P.recv_first = rank > 0;
    P.chain_lo = 0;
    P.chain_hi = per;
    P.send_last = rank < world - 1;
    return P;
  }
  // (i) fine sweep over active slices n = k−1..N−1 (frozen prefix n < k−1)
  if (k - 1 < n1) {
    P.fine_lo = std::max(0, k - 1 - n0);
    P.fine_hi = per;
    P.fk_local = (k - 1 >= n0) ? k - 1 - n0 : -1;
  }
  // (ii) coarse chain with correction starting at slice k
  if (k - 1 >= n0 && k - 1 < n1) {         // this rank computed F̂_{k−1}: U_k := F̂_{k−1}
    P.copy = 1;
    P.chain_lo = k - n0;
    P.chain_hi = per;
    P.delta_lo = k - n0;
    P.delta_hi = per;
  } else if (n0 >= k && rank > 0) {         // U_{n0} arrives from rank−1's chain
    P.recv_first = 1;
    P.chain_lo = 0;
    P.chain_hi = per;
    P.delta_lo = 1;                         // U_{n0}'s δ is reduced by rank−1 (its U_{n1})
    P.delta_hi = per;
  }                                         // else: frozen rank, no chain
  P.send_last = (n1 >= k) && rank < world - 1;
  return P;
}

// ---------------------------------------------------------------- pipelined schedule (NEXT-2)
// Eligible: one GPU, fixed K (tol = 0: no host decision between iterations), PINN G in latency
// mode, resident fine kernel with M ≤ 1024, and every CTA co-resident (checked at first launch).
bool pipe_eligible(const pr_ctx *c) {
  if (c->opt_pipeline == 1 || c->pipe_ok == 0) return false;
  if (c->world != 1 || c->tol != 0.0 || c->max_iter < 1 || c->tc) return false;
  if (!use_resident(c) || c->M > 1024) return false;
  if (c->coarse == PR_COARSE_IMPLICIT_EULER) return pr::pipe_num_supported(c->M, c->fine_theta != 1.0);
  // the chain evaluates as the blocking kernel would: latency mode if it is the one chosen
  return pr::pipe_supported(c->M, c->fine_theta != 1.0, c->IN, c->W, c->act, use_split_pinn(c) ? split_G(c) : 1);
}

pr_status ensure_pipe(pr_ctx *c) {
  if (c->pipe_partials) return PR_OK;
  c->pipe_pstride = (size_t)(c->Nloc + 1) * c->B * c->nch * 2;
  CU(cudaMalloc(&c->pipe_partials, (size_t)(c->max_iter + 1) * c->pipe_pstride * sizeof(double)));
  CU(cudaMalloc(&c->pipe_flags, (size_t)3 * c->B * c->N * sizeof(int) + 2 * sizeof(unsigned long long)));
  // flags and the tail's grid-barrier counter zeroed once: every launch leaves the flags zero
  CU(cudaMemset(c->pipe_flags, 0, (size_t)3 * c->B * c->N * sizeof(int) + 2 * sizeof(unsigned long long)));
  CU(cudaMalloc(&c->pipe_wstage, (size_t)(c->max_iter + 1) * (c->N + 1) * c->B * c->nch * 4 * 2 * sizeof(double)));
  CU(cudaMemset(c->pipe_partials, 0, (size_t)(c->max_iter + 1) * c->pipe_pstride * sizeof(double)));
  return PR_OK;
}

// All K iterations (and the k = 0 coarse sweep) in one cooperative launch, then the K δ's.
// Returns PR_ERR_UNSUPPORTED (nothing enqueued) if the grid cannot be co-resident.
pr_status solve_pipelined(pr_ctx *c) {
  pr::PipeArgs pa;
  std::memset(&pa, 0, sizeof pa);
  pa.r = base_args(c, c->fine);
  pa.r.U = c->U;
  pa.r.Gh = c->Gh;
  pa.r.D = c->D;
  pa.r.Fk = c->Fk;
  pa.g = pinn_args(c);
  const int G = use_split_pinn(c) ? split_G(c) : 1;  // chain threads per point
  if (pr::pinn_split_is_group(c->W, G)) pa.g.wts = c->d_wgrp;  // group chain: group-order weights
  pa.g.U = c->U;
  pa.g.Gh = c->Gh;
  pa.g.D = c->D;
  pa.g.Fcopy = c->Fk;
  pa.N = c->N;
  pa.K = c->max_iter;
  const bool num = c->coarse == PR_COARSE_IMPLICIT_EULER;
  if (num) {  // one K1 chain system per (iteration, instance), one publication per slice
    pa.rc = base_args(c, c->crs);
    pa.g.B = c->B;
    pa.C = 1;
    pa.cpub = 1;
  } else {
    // chain points per CTA: the blocking chain's CTA (4 warps) times the chain-CTA width in warps / 4
    const int nwc = pr::pipe_chain_warps(c->W, G);
    const int ppc = (G > 1 ? pr::pinn_split_ppc(G) : 128) * (nwc / 4);
    pa.C = (c->M + ppc - 1) / ppc;  // chain CTAs per instance
    pa.cpub = pa.C * nwc;           // every chain warp publishes
    if ((size_t)pa.C * (nwc / 4) > (size_t)c->nch || (size_t)pa.C * nwc > (size_t)c->nch * 4) {
      c->pipe_ok = 0;
      return PR_ERR_UNSUPPORTED;  // δ chunks / warp staging would not fit: blocking schedule
    }
  }
  pa.partials = c->pipe_partials;
  pa.pstride = c->pipe_pstride;
  pa.wstage = c->pipe_wstage;
  static const char *trace_path = getenv("PR_PIPE_TRACE");  // debugging: dump the kernel's timeline
  unsigned long long *d_trace = nullptr;
  const size_t ntr = (size_t)(c->max_iter + 1) * c->N * 3;
  if (trace_path && !c->capturing) {
    CU(cudaMalloc(&d_trace, ntr * sizeof(unsigned long long)));
    CU(cudaMemsetAsync(d_trace, 0, ntr * sizeof(unsigned long long), c->stream));
    pa.trace = d_trace;
  }
  pa.cnt = c->pipe_flags;
  pa.floaded = c->pipe_flags + (size_t)c->B * c->N;
  pa.fdone = c->pipe_flags + (size_t)2 * c->B * c->N;
  pa.gbar = (unsigned long long *)(c->pipe_flags + align_up((size_t)3 * c->B * c->N, 2));
  pa.dmax = c->d_delta;
  pa.nch = c->nch;
  const cudaError_t e =
      num ? pr::launch_parareal_pipe_num(pa, c->M, c->fine_theta != 1.0, c->stream)
          : pr::launch_parareal_pipe(pa, c->M, c->fine_theta != 1.0, c->IN, c->W, c->act, G,
                                     (size_t)c->nfloats * sizeof(float), c->stream);
  if (e == cudaErrorCooperativeLaunchTooLarge) {
    cudaGetLastError();
    c->pipe_ok = 0;
    return PR_ERR_UNSUPPORTED;
  }
  if (e != cudaSuccess) return fail(c, PR_ERR_CUDA, fmt("pipelined Parareal launch: %s", cudaGetErrorString(e)));
  c->pipe_ok = 1;
  c->launches++;
  if (d_trace) {
    std::vector<unsigned long long> h(ntr);
    CU(cudaMemcpyAsync(h.data(), d_trace, ntr * sizeof(unsigned long long), cudaMemcpyDeviceToHost, c->stream));
    SYNC();
    cudaFree(d_trace);
    if (FILE *f = fopen(trace_path, "w")) {
      for (int k = 0; k <= c->max_iter; ++k)
        for (int n = 0; n < c->N; ++n)
          fprintf(f, "%d %d %llu %llu %llu\n", k, n, h[((size_t)k * c->N + n) * 3], h[((size_t)k * c->N + n) * 3 + 1],
                  h[((size_t)k * c->N + n) * 3 + 2]);
      fclose(f);
    }
  }
  // δ^1..δ^K: computed by the kernel's tail (k_delta's fixed-order sums per row)
  return PR_OK;
}

using Spans = std::vector<std::pair<int, std::pair<cudaEvent_t, cudaEvent_t>>>;

// lean: this solve ran a lean (PR_OPT_USE_GRAPHS = 2) graph, which records no timing events
pr_status solve_report(pr_ctx *c, int K, int conv, cudaEvent_t e0, cudaEvent_t e1, const Spans &spans,
                       int64_t launches, pr_report *rep, bool lean) {
  c->solved = true;
  if (!rep) return PR_OK;
  rep->iterations = K;
  rep->converged = (c->tol > 0.0 && K > 0 && c->h_delta[K - 1] < c->tol) ? 1 : conv;
  if (rep->delta)
    for (int i = 0; i < K; ++i) rep->delta[i] = c->h_delta[i];
  rep->kernel_launches = launches;
  if (lean) {  // lean graph: no timing events were captured
    rep->ms_total = rep->ms_coarse = rep->ms_fine = rep->ms_comm = rep->ms_setup = 0.0;
    return PR_OK;
  }
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  rep->ms_total = ms;
  double ph[4] = {0, 0, 0, 0};
  for (auto &sp : spans) {
    float m = 0;
    cudaEventElapsedTime(&m, sp.second.first, sp.second.second);
    ph[sp.first] += m;
  }
  rep->ms_coarse = ph[PH_COARSE];
  rep->ms_fine = ph[PH_FINE];
  rep->ms_comm = ph[PH_COMM];
  rep->ms_setup = ph[PH_SETUP];
  rep->kernel_launches = launches;
  return PR_OK;
}

void drop_graph(pr_ctx *c) {
  if (c->g_exec) cudaGraphExecDestroy(c->g_exec);
  c->g_exec = nullptr;
  for (cudaEvent_t e : c->g_events) cudaEventDestroy(e);
  c->g_events.clear();
  c->g_vt = nullptr;
  c->g_v0 = nullptr;
}

// ---------------------------------------------------------------- NEXT-4: spatially sharded chain
// PINN G is pointwise in S, so the coarse chain of iteration k can run on every rank at once, each
// over ALL slices but only its own range of grid points (a CTA range of the same kernel), while the
// fine sweep stays sharded by slices (it couples every point of a slice).  Per iteration two
// exchanges convert between the layouts: the boundary states U^{k−1}_n and Ĝ_n of the active
// slices go from the point owners to the slice owners (the fine epilogue forms D_n = F̂_n − Ĝ_n in
// fp64, as on one rank), and D_n and F̂_{k−1} go back.  The δ partial slots (one per chain CTA)
// are summed over ranks (each slot has one non-zero contributor: exact) and reduced as on one
// rank.  Every rank's chain then takes t_chain/R instead of the wavefront's ≈ (1 + (R−1)/C)·t_chain/R
// and the exchanges cost ≈ 2·N·M·4 B·(R−1)/R² per rank; results are bitwise the one-rank solve's.
bool spatial_chain(const pr_ctx *c) {
  if (c->world == 1 || c->coarse != PR_COARSE_PINN || c->B != 1 || c->opt_spatial == 1) return false;
  return c->opt_spatial == 2 || c->tc != 0;  // auto: the tensor-core (wide) nets, whose chain dominates
}

struct SpGeom {
  int ppc, gx;
  std::vector<int> jlo, jhi, clo, chi;  // per rank: grid points and chain CTAs
};
SpGeom sp_geom(const pr_ctx *c) {
  SpGeom g;
  pinn_geometry(c, &g.ppc, &g.gx);
  const int R = c->world;
  for (int q = 0; q < R; ++q) {
    const int a = (int)((long)q * g.gx / R), b = (int)((long)(q + 1) * g.gx / R);
    g.clo.push_back(a);
    g.chi.push_back(b);
    g.jlo.push_back(std::min(a * g.ppc, c->M));
    g.jhi.push_back(std::min(b * g.ppc, c->M));
  }
  return g;
}

// Rows [a, b] of the sharded buffers (sp_U / sp_Gh, this rank's point range) → the slice owners'
// local rows (U / Gh), every owner receiving every rank's piece.  The owner of slices [n0, n1) holds
// U rows n0..n1 and Gh rows n0..n1−1.  NCCL: one group; messages between a pair in ascending n.
pr_status sp_to_owners(pr_ctx *c, const SpGeom &g, int a, int b, bool with_gh) {
  const int R = c->world, r = c->rank, per = c->Nloc;
  const size_t row = (size_t)c->Mp;
  std::vector<std::function<pr_status()>> ops;  // sends first (loopback: non-blocking), then receives
  std::vector<std::function<pr_status()>> rcv;
  for (int n = a; n <= b; ++n) {
    for (int o = 0; o < R; ++o) {  // owners holding row n of U: o = n / per (row n − n0) and o = n/per − 1 (row per)
      const int n0 = o * per;
      if (n < n0 || n > n0 + per) continue;
      const int ln = n - n0;
      for (int part = 0; part < (with_gh && n < n0 + per ? 2 : 1); ++part) {
        const float *src = (part == 0 ? c->sp_U : c->sp_Gh) + (size_t)n * row;
        float *dst = (part == 0 ? c->U : c->Gh) + (size_t)ln * row;
        if (o == r) {
          for (int q = 0; q < R; ++q) {
            const size_t cnt = (size_t)(g.jhi[q] - g.jlo[q]);
            if (!cnt) continue;
            if (q == r)
              ops.push_back([=]() -> pr_status {
                CU(cudaMemcpyAsync(dst + g.jlo[q], src + g.jlo[q], cnt * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
                return PR_OK;
              });
            else
              rcv.push_back([=]() { return comm_recv(c, dst + g.jlo[q], cnt, q); });
          }
        } else {
          const size_t cnt = (size_t)(g.jhi[r] - g.jlo[r]);
          if (cnt) ops.push_back([=]() { return comm_send(c, src + g.jlo[r], cnt, o); });
        }
      }
    }
  }
  if (!c->loop) NC(nccl().GroupStart());
  pr_status st = PR_OK;
  for (auto &f : ops)
    if ((st = f())) break;
  if (!st)
    for (auto &f : rcv)
      if ((st = f())) break;
  if (!c->loop) NC(nccl().GroupEnd());
  return st;
}

// This rank's fine outputs → the point owners: D_n (local rows of slices [lo, n1)) into sp_D, and
// F̂_{k−1} (if this rank owns slice k−1) into sp_F on every rank.
pr_status sp_from_owners(pr_ctx *c, const SpGeom &g, int k) {
  const int R = c->world, r = c->rank, per = c->Nloc;
  const size_t row = (size_t)c->Mp;
  std::vector<std::function<pr_status()>> ops, rcv;
  auto piece = [&](const float *src_row, float *dst_row, int owner) {  // every rank's range of one row
    if (owner == r) {
      for (int q = 0; q < R; ++q) {
        const size_t cnt = (size_t)(g.jhi[q] - g.jlo[q]);
        if (!cnt) continue;
        if (q == r)
          ops.push_back([=]() -> pr_status {
            CU(cudaMemcpyAsync(dst_row + g.jlo[q], src_row + g.jlo[q], cnt * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
            return PR_OK;
          });
        else
          ops.push_back([=]() { return comm_send(c, src_row + g.jlo[q], cnt, q); });
      }
    } else {
      const size_t cnt = (size_t)(g.jhi[r] - g.jlo[r]);
      if (cnt) rcv.push_back([=]() { return comm_recv(c, dst_row + g.jlo[r], cnt, owner); });
    }
  };
  for (int n = k - 1; n < c->N; ++n) {
    const int o = n / per;
    if (n == k - 1) piece(c->Fk, c->sp_F, o);
    else piece(c->D + (size_t)(n - o * per) * row, c->sp_D + (size_t)n * row, o);
  }
  if (!c->loop) NC(nccl().GroupStart());
  pr_status st = PR_OK;
  for (auto &f : ops)
    if ((st = f())) break;
  if (!st)
    for (auto &f : rcv)
      if ((st = f())) break;
  if (!c->loop) NC(nccl().GroupEnd());
  return st;
}

pr_status sp_chain(pr_ctx *c, const SpGeom &g, int k) {
  pr::PinnArgs a = pinn_args(c);
  a.n_base = 0;  // global slice indices
  a.ln0 = k;
  a.ln1 = c->N;
  a.U = c->sp_U;
  a.Gh = c->sp_Gh;
  a.D = k > 0 ? c->sp_D : nullptr;
  a.Fcopy = k > 0 ? c->sp_F : nullptr;
  a.partials = k > 0 ? c->sp_part : nullptr;
  return launch_pinn(c, a, g.clo[c->rank], g.chi[c->rank]);
}

// Parareal with the spatially sharded chain (R > 1, B == 1).  Leaves U (local rows) and δ exactly
// as the slice-sharded schedule does, so the gather of U_N and copy_iterates work unchanged.
pr_status solve_spatial(pr_ctx *c, const float *V_T, bool device_ptr, PhaseTimer &pt, int &K, int &conv) {
  const int N = c->N, r = c->rank;
  const size_t row = (size_t)c->Mp, rows = (size_t)(N + 1) * row;
  pr_status st;
  if (!c->sp_U) {
    CU(cudaMalloc(&c->sp_U, rows * sizeof(float)));
    CU(cudaMalloc(&c->sp_Gh, rows * sizeof(float)));
    CU(cudaMalloc(&c->sp_D, rows * sizeof(float)));
    CU(cudaMalloc(&c->sp_F, row * sizeof(float)));
    CU(cudaMalloc(&c->sp_part, (size_t)(N + 1) * c->nch * 2 * sizeof(double)));
    CU(cudaMemsetAsync(c->sp_U, 0, rows * sizeof(float), c->stream));
    CU(cudaMemsetAsync(c->sp_Gh, 0, rows * sizeof(float), c->stream));
    CU(cudaMemsetAsync(c->sp_D, 0, rows * sizeof(float), c->stream));
  }
  const size_t npart = (size_t)(N + 1) * c->nch * 2;
  const SpGeom g = sp_geom(c);
  // U_0 from rank 0 (V_T or the payoff) to every rank's point range
  pt.begin(PH_SETUP);
  if (r == 0 && (st = load_initial(c, V_T, device_ptr))) return st;
  {
    std::vector<std::function<pr_status()>> ops, rcv;
    for (int q = 0; q < c->world; ++q) {
      const size_t cnt = (size_t)(g.jhi[q] - g.jlo[q]);
      if (!cnt) continue;
      if (r == 0 && q == 0) {
        CU(cudaMemcpyAsync(c->sp_U + g.jlo[0], c->U + g.jlo[0], cnt * sizeof(float), cudaMemcpyDeviceToDevice, c->stream));
      } else if (r == 0) {
        if ((st = comm_send(c, c->U + g.jlo[q], cnt, q))) return st;
      } else if (q == r) {
        if ((st = comm_recv(c, c->sp_U + g.jlo[r], cnt, 0))) return st;
      }
    }
  }
  pt.end();
  pt.begin(PH_COARSE);
  if ((st = sp_chain(c, g, 0))) return st;  // k = 0: U_{n+1} = G(U_n), all slices, own points
  pt.end();
  for (int k = 1; k <= c->max_iter; ++k) {
    const pr_plan P = make_plan(N, c->world, r, k);
    pt.begin(PH_COMM);
    if ((st = sp_to_owners(c, g, k - 1, N, true))) return st;  // U^{k−1}_n, Ĝ_n of the active slices
    pt.end();
    pt.begin(PH_FINE);
    if (P.fine_hi > P.fine_lo && (st = fine_sweep(c, P.fine_lo, P.fk_local))) return st;
    pt.end();
    pt.begin(PH_COMM);
    if ((st = sp_from_owners(c, g, k))) return st;  // D_n, F̂_{k−1} → point owners
    pt.end();
    pt.begin(PH_COARSE);
    CU(cudaMemsetAsync(c->sp_part, 0, npart * sizeof(double), c->stream));
    if ((st = sp_chain(c, g, k))) return st;
    pt.end();
    pt.begin(PH_COMM);
    if ((st = comm_allreduce_sum(c, c->sp_part + (size_t)k * c->nch * 2, (size_t)(N + 1 - k) * c->nch * 2))) return st;
    pt.end();
    unsigned long long *slot = c->d_delta + (k - 1);
    CU(cudaMemsetAsync(slot, 0, sizeof(unsigned long long), c->stream));
    LAUNCH(pr::launch_delta(c->sp_part, c->B, c->nch, k, N, slot, c->stream));
    K = k;
    if (c->tol > 0.0) {
      CU(cudaMemcpyAsync(c->h_delta + (k - 1), slot, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
      SYNC();
      if (c->h_delta[k - 1] < c->tol) {
        conv = 1;
        break;
      }
    }
  }
  // the final iterate back into the slice owners' rows (U_N then reaches rank 0 as usual)
  pt.begin(PH_COMM);
  st = sp_to_owners(c, g, 0, N, false);
  pt.end();
  return st;
}

pr_status solve_impl_(pr_ctx *c, const float *V_T, float *V_0, bool device_ptr, pr_report *rep);
pr_status solve_impl(pr_ctx *c, const float *V_T, float *V_0, bool device_ptr, pr_report *rep) {
  const nvtxRangeId_t r = nvtxRangeStartA("parareal_solve");
  const pr_status st = solve_impl_(c, V_T, V_0, device_ptr, rep);
  nvtxRangeEnd(r);
  return st;
}
pr_status solve_impl_(pr_ctx *c, const float *V_T, float *V_0, bool device_ptr, pr_report *rep) {
  pr_status st = check_ctx(c);
  if (st) return st;
  if (c->coarse == PR_COARSE_PINN && !c->have_pinn)
    return fail(c, PR_ERR_STATE, "coarse == PR_COARSE_PINN but no weights loaded (parareal_load_pinn_weights)");
  if ((st = ensure_ws(c))) return st;
  // CUDA-graph replay of a fixed-K single-GPU device-pointer solve (PR_OPT_USE_GRAPHS): the whole
  // solve (≈ 4K+4 kernels) is captured once per (V_T, V_0) pair and relaunched as one graph.
  // (host buffers qualify when they are pinned: the graph's copy nodes then stay valid; a replay
  // with host buffers always returns with V_0 written)
  auto pinned = [](const void *h) {
    if (!h) return true;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, h) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  };
  // (a replay of the captured (V_T, V_0) pair was checked when it was captured: no attribute queries)
  const bool replay = c->opt_graphs && c->tol == 0.0 && c->world == 1 && c->g_exec && c->g_vt == V_T &&
                      c->g_v0 == V_0 && c->g_dev == device_ptr;
  const bool use_graph = replay || (c->opt_graphs && c->tol == 0.0 && c->world == 1 &&
                                    (device_ptr || (pinned(V_T) && pinned(V_0))));
  if (replay) {
    CU(cudaGraphLaunch(c->g_exec, c->stream));
    c->launches += c->g_launches;
    if (c->opt_graphs == 2 && device_ptr) {  // stream-ordered replay: return once enqueued (no δ, no times)
      c->solved = true;
      if (rep) {
        rep->iterations = c->g_K;
        rep->converged = 0;
        rep->kernel_launches = c->g_launches;
        rep->ms_total = rep->ms_coarse = rep->ms_fine = rep->ms_comm = rep->ms_setup = 0.0;
      }
      return PR_OK;
    }
    SYNC();
    return solve_report(c, c->g_K, 0, c->g_e0, c->g_e1, c->g_spans, c->g_launches, rep, c->opt_graphs == 2);
  }
  if (pipe_eligible(c) && (st = ensure_pipe(c))) return st;  // (allocation cannot be captured)
  if (c->fine.g_pt && (st = ensure_grid(c))) return st;
  if (use_graph) {
    drop_graph(c);
    CU(cudaStreamBeginCapture(c->stream, cudaStreamCaptureModeThreadLocal));
    c->capturing = true;
  }
  c->ev_used = 0;
  const int64_t launches0 = c->launches;
  PhaseTimer pt{c};
  cudaEvent_t e0 = next_event(c), e1 = nullptr;
  int K = 0, conv = 0;
  st = [&]() -> pr_status {
  pr_status st = PR_OK;
  record(c, e0);
  const int R = c->world, r = c->rank;
  const size_t row = (size_t)c->B * c->Mp;
  // δ partials are rewritten slice by slice; clear stale chunks of earlier solves
  if (!pipe_eligible(c))
    CU(cudaMemsetAsync(c->partials, 0, (size_t)(c->Nloc + 1) * c->B * c->nch * 2 * sizeof(double), c->stream));
  // ---- k = 0: U_0 and the initial coarse sweep U_{n+1} = G(U_n)
  pt.begin(PH_SETUP);
  if (r == 0 && (st = load_initial(c, V_T, device_ptr))) return st;
  pt.end();
  bool piped = false;
  if (pipe_eligible(c)) {  // NEXT-2: fine solves and coarse chain overlapped in one kernel
    pt.begin(PH_FINE);
    st = solve_pipelined(c);
    pt.end();
    if (st == PR_OK) {
      piped = true;
      K = c->max_iter;
      pt.spans.push_back({PH_COARSE, pt.spans.back().second});  // overlapped: same span for both
    } else if (st != PR_ERR_UNSUPPORTED) {
      return st;
    } else {  // cannot be co-resident: blocking schedule (its partials were not cleared above)
      CU(cudaMemsetAsync(c->partials, 0, (size_t)(c->Nloc + 1) * c->B * c->nch * 2 * sizeof(double), c->stream));
    }
  }
  if (!piped && spatial_chain(c)) {
    if ((st = solve_spatial(c, V_T, device_ptr, pt, K, conv))) return st;
  } else if (!piped) {
  {
    const pr_plan P0 = make_plan(c->N, R, r, 0);
    pt.begin(PH_COARSE);  // (with R > 1 this span includes the hand-offs of U_{n0} / U_{n1})
    if ((st = chain_exchange(c, 0, P0, true, nullptr))) return st;
    pt.end();
  }
  for (int k = 1; k <= c->max_iter; ++k) {
    const pr_plan P = make_plan(c->N, R, r, k);
    // (i) fine sweep F̂_n = F(U^{k−1}_n), n = k−1..N−1 (parallel across slices)
    pt.begin(PH_FINE);
    if (P.fine_hi > P.fine_lo && (st = fine_sweep(c, P.fine_lo, P.fk_local))) return st;
    pt.end();
    // (ii) coarse chain with correction, serial in n across ranks (blocking or chunk wavefront)
    pt.begin(PH_COARSE);
    if ((st = chain_exchange(c, k, P, P.copy || P.recv_first, nullptr))) return st;
    pt.end();
    const int dlo = P.delta_lo, dhi = P.delta_hi;
    // (iii) δ^k and the stop rule (Q13)
    if ((st = delta_reduce(c, k, dlo, dhi, c->nch))) return st;
    K = k;
    if (c->tol > 0.0) {
      CU(cudaMemcpyAsync(c->h_delta + (k - 1), c->d_delta + (k - 1), sizeof(double), cudaMemcpyDeviceToHost,
                         c->stream));
      SYNC();
      if (c->h_delta[k - 1] < c->tol) {
        conv = 1;
        break;
      }
    }
  }
  }  // !piped
  // final state U^K_N: last rank → rank 0 (→ V_0)
  if (R > 1) {
    pt.begin(PH_COMM);
    if (r == R - 1 && (st = comm_send(c, c->U + (size_t)c->Nloc * row, row, 0))) return st;
    if (r == 0 && (st = comm_recv(c, c->tmp, row, R - 1))) return st;
    pt.end();
  }
  if (r == 0 && V_0) {
    const float *src = (R > 1) ? c->tmp : c->U + (size_t)c->Nloc * row;
    if ((st = store_rows(c, V_0, src, device_ptr))) return st;
  }
  e1 = next_event(c);
  record(c, e1);
  CU(cudaMemcpyAsync(c->h_delta, c->d_delta, K * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  return PR_OK;
  }();
  if (use_graph) {
    cudaGraph_t g = nullptr;
    c->capturing = false;
    const cudaError_t ce = cudaStreamEndCapture(c->stream, &g);
    if (st) {
      if (g) cudaGraphDestroy(g);
      return st;
    }
    if (ce != cudaSuccess) return fail(c, PR_ERR_CUDA, fmt("graph capture: %s", cudaGetErrorString(ce)));
    const cudaError_t ie = cudaGraphInstantiate(&c->g_exec, g, 0);
    cudaGraphDestroy(g);
    if (ie != cudaSuccess) return fail(c, PR_ERR_CUDA, fmt("graph instantiate: %s", cudaGetErrorString(ie)));
    // the graph owns the events it records: move them out of the reusable pool
    c->g_events.assign(c->ev.begin(), c->ev.begin() + c->ev_used);
    c->ev.erase(c->ev.begin(), c->ev.begin() + c->ev_used);
    c->ev_used = 0;
    c->g_vt = V_T;
    c->g_v0 = V_0;
    c->g_dev = device_ptr;
    c->g_K = K;
    c->g_e0 = e0;
    c->g_e1 = e1;
    c->g_spans = pt.spans;
    c->g_launches = c->launches - launches0;
    CU(cudaGraphLaunch(c->g_exec, c->stream));
  } else if (st) {
    return st;
  }
  SYNC();
  if ((st = grid_check(c))) return st;
  return solve_report(c, K, conv, e0, e1, pt.spans, c->launches - launches0, rep, use_graph && c->opt_graphs == 2);
}

pr_status serial_fine_impl(pr_ctx *c, const float *V_T, float *V_0, bool device_ptr, double *ms) {
  pr_status st = check_ctx(c);
  if (st) return st;
  if ((st = ensure_ws(c))) return st;
  c->ev_used = 0;
  cudaEvent_t e0 = next_event(c), e1 = next_event(c);
  cudaEventRecord(e0, c->stream);
  // initial state into tmp row 0
  float *save = c->U;
  c->U = c->tmp;
  st = load_initial(c, V_T, device_ptr);
  c->U = save;
  if (st) return st;
  if (use_resident(c)) {
    pr::ResidentArgs a = base_args(c, c->fine);
    a.n_base = 0;
    a.Uw = c->tmp;
    a.ustride = 0;  // one row, updated in place slice after slice
    a.c_ln0 = 0;
    a.c_ln1 = c->N;
    LAUNCH(dispatch_res(true, c->M, a, c->B, c->stream));
  } else if (use_grid(c, 1)) {  // one grid-resident slice solve per slice, in place (each CTA owns its points)
    for (int n = 0; n < c->N; ++n)
      if ((st = grid_sweep(c, 0, 1, n, c->tmp, c->tmp, -1))) return st;
  } else {
    pr::StreamedChainJob j;
    j.U = c->tmp; j.Gh = nullptr; j.D = nullptr; j.Fcopy = nullptr; j.partials = nullptr; j.nch = 1;
    j.ln0 = 0; j.ln1 = c->N; j.n_base = 0; j.ustride = 0;
    int nl = 0;
    cudaError_t e = pr::streamed_chain(c->sst, sprob(c, c->fine), j, c->stream, &nl);
    c->launches += nl;
    if (e != cudaSuccess) return fail(c, PR_ERR_CUDA, fmt("streamed serial fine: %s", cudaGetErrorString(e)));
  }
  cudaEventRecord(e1, c->stream);
  if (V_0 && (st = store_rows(c, V_0, c->tmp, device_ptr))) return st;
  SYNC();
  if ((st = grid_check(c))) return st;
  if (ms) {
    float m = 0;
    cudaEventElapsedTime(&m, e0, e1);
    *ms = m;
  }
  return PR_OK;
}

}  // namespace

// ============================================================================ ABI
extern "C" {

const char *parareal_status_string(pr_status s) {
  switch (s) {
    case PR_OK: return "PR_OK";
    case PR_ERR_INVALID_ARGUMENT: return "PR_ERR_INVALID_ARGUMENT";
    case PR_ERR_OUT_OF_MEMORY: return "PR_ERR_OUT_OF_MEMORY";
    case PR_ERR_CUDA: return "PR_ERR_CUDA";
    case PR_ERR_NCCL: return "PR_ERR_NCCL";
    case PR_ERR_STATE: return "PR_ERR_STATE";
    case PR_ERR_NUMERICAL: return "PR_ERR_NUMERICAL";
    case PR_ERR_UNSUPPORTED: return "PR_ERR_UNSUPPORTED";
  }
  return "unknown pr_status";
}

const char *parareal_last_error(const pr_ctx *ctx) { return ctx ? ctx->err.c_str() : g_init_error.c_str(); }

pr_status parareal_get_nccl_id(uint8_t out[128]) {
  pr_ctx *c = nullptr;
  if (!out) return fail(c, PR_ERR_INVALID_ARGUMENT, "out is NULL");
  Nccl &n = nccl();
  if (!n.ok) return fail(c, PR_ERR_NCCL, n.why);
  ncclUniqueId id;
  NC(n.GetUniqueId(&id));
  std::memcpy(out, id.internal, 128);
  return PR_OK;
}

pr_status parareal_init(const pr_problem *p, const pr_dist *dist, pr_ctx **out) {
  pr_ctx *c = nullptr;
  if (!out) return fail(c, PR_ERR_INVALID_ARGUMENT, "out is NULL");
  *out = nullptr;
  if (!p) return fail(c, PR_ERR_INVALID_ARGUMENT, "problem is NULL");
  if (p->struct_size != sizeof(pr_problem))
    return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("problem.struct_size=%u, expected %zu (ABI mismatch)", p->struct_size,
                                                sizeof(pr_problem)));
  if (p->M < 1) return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("problem.M=%d must be >= 1", p->M));
  if (p->B < 1) return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("problem.B=%d must be >= 1", p->B));
  if (!p->strike || !p->sigma || !p->rate || !p->L)
    return fail(c, PR_ERR_INVALID_ARGUMENT, "problem.strike/sigma/rate/L must be non-NULL [B] arrays");
  for (int b = 0; b < p->B; ++b) {
    if (!(p->sigma[b] > 0)) return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("problem.sigma[%d]=%g must be > 0", b, p->sigma[b]));
    if (!(p->rate[b] >= 0)) return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("problem.rate[%d]=%g must be >= 0", b, p->rate[b]));
    if (!(p->strike[b] >= 0)) return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("problem.strike[%d]=%g must be >= 0", b, p->strike[b]));
    if (!(p->L[b] > p->strike[b]))
      return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("problem.L[%d]=%g must exceed strike %g", b, p->L[b], p->strike[b]));
  }
  if (!(p->T > 0)) return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("problem.T=%g must be > 0", p->T));
  if (p->upper_bc != PR_BC_CALL_ASYMPTOTIC && p->upper_bc != PR_BC_ZERO)
    return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("problem.upper_bc=%d unknown", p->upper_bc));
  if (p->N < 1) return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("problem.N=%d must be >= 1", p->N));
  if (p->fine_steps < 1) return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("problem.fine_steps=%d must be >= 1", p->fine_steps));
  if (p->coarse != PR_COARSE_PINN && p->coarse != PR_COARSE_IMPLICIT_EULER)
    return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("problem.coarse=%d unknown", p->coarse));
  if (p->coarse == PR_COARSE_IMPLICIT_EULER && p->coarse_steps < 1)
    return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("problem.coarse_steps=%d must be >= 1", p->coarse_steps));
  if (p->max_iter < 1 || p->max_iter > p->N)
    return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("problem.max_iter=%d must be in [1, N=%d]", p->max_iter, p->N));
  if (!(p->tol >= 0)) return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("problem.tol=%g must be >= 0", p->tol));
  if (!(p->fine_theta >= 0.5 && p->fine_theta <= 1.0))
    return fail(c, PR_ERR_INVALID_ARGUMENT,
                fmt("problem.fine_theta=%g: must be in [0.5, 1] (1 implicit Euler, 0.5 Crank-Nicolson)", p->fine_theta));
  pr_dist dd = {0, 1, 0, nullptr, nullptr};
  if (dist) dd = *dist;
  if (dd.world < 1 || dd.rank < 0 || dd.rank >= dd.world)
    return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("dist.rank=%d/world=%d invalid", dd.rank, dd.world));
  if (p->N % dd.world)
    return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("problem.N=%d must be divisible by dist.world=%d", p->N, dd.world));
  if (dd.world > 1 && !dd.nccl_id) return fail(c, PR_ERR_INVALID_ARGUMENT, "dist.nccl_id is NULL with world > 1");
  if ((size_t)p->M * p->B > (size_t)1 << 31)
    return fail(c, PR_ERR_UNSUPPORTED, "M*B above 2^31 points per slice");
  if (p->B > 65535)  // the instance index is a grid y coordinate in the payoff, PINN and K2 kernels
    return fail(c, PR_ERR_UNSUPPORTED, fmt("problem.B=%d above 65535 instances per context", p->B));

  c = new pr_ctx();
  pr_status st = PR_OK;
  auto bail = [&](pr_status s) {
    g_init_error = c->err;
    parareal_free(c);
    return s;
  };
  c->M = p->M;
  c->Mp = (p->M + 31) / 32 * 32;
  c->B = p->B;
  c->N = p->N;
  c->nf = p->fine_steps;
  c->fine_theta = p->fine_theta;
  c->nc = p->coarse_steps;
  c->coarse = p->coarse;
  c->max_iter = p->max_iter;
  c->upper_bc = p->upper_bc;
  c->T = p->T;
  c->dT = p->T / p->N;
  c->tol = p->tol;
  c->K.assign(p->strike, p->strike + p->B);
  c->sig.assign(p->sigma, p->sigma + p->B);
  c->r.assign(p->rate, p->rate + p->B);
  c->L.assign(p->L, p->L + p->B);
  c->rank = dd.rank;
  c->world = dd.world;
  c->device = dd.device;
  const int per = p->N / dd.world;
  c->n0 = dd.rank * per;
  c->n1 = c->n0 + per;
  c->Nloc = per;
  {
    cudaError_t e = cudaSetDevice(dd.device);
    if (e != cudaSuccess) {
      c->err = fmt("cudaSetDevice(%d): %s", dd.device, cudaGetErrorString(e));
      return bail(PR_ERR_CUDA);
    }
  }
  if (dd.stream) {
    c->stream = (cudaStream_t)dd.stream;
  } else {
    if (cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess) {
      c->err = "cudaStreamCreate failed";
      return bail(PR_ERR_CUDA);
    }
    c->own_stream = true;
  }
  // distinct (σ, r) factor sets: the operator does not depend on K or L (a_j, b_j of P:156)
  std::map<std::pair<double, double>, int> idx;
  for (int b = 0; b < c->B; ++b) {
    auto key = std::make_pair(c->sig[b], c->r[b]);
    auto it = idx.find(key);
    if (it == idx.end()) {
      it = idx.emplace(key, (int)c->sets.size()).first;
      c->sets.push_back(key);
    }
    c->fset.push_back(it->second);
  }
  c->nsets = (int)c->sets.size();
  {
    auto up = [&](void **d, const void *h, size_t n) { return cudaMalloc(d, n) == cudaSuccess && cudaMemcpy(*d, h, n, cudaMemcpyHostToDevice) == cudaSuccess; };
    if (!up((void **)&c->d_fset, c->fset.data(), c->B * sizeof(int)) ||
        !up((void **)&c->d_L, c->L.data(), c->B * sizeof(double)) ||
        !up((void **)&c->d_K, c->K.data(), c->B * sizeof(double)) ||
        !up((void **)&c->d_r, c->r.data(), c->B * sizeof(double))) {
      c->err = "allocating/uploading instance parameters failed";
      return bail(PR_ERR_OUT_OF_MEMORY);
    }
  }
  if ((st = upload_scheme(c, c->fine, c->nf, c->fine_theta))) return bail(st);
  if (c->coarse == PR_COARSE_IMPLICIT_EULER && (st = upload_scheme(c, c->crs, c->nc, 1.0))) return bail(st);
  if (cudaMallocHost(&c->h_delta, std::max(c->max_iter, 1) * sizeof(double)) != cudaSuccess) {
    c->err = "cudaMallocHost(delta) failed";
    return bail(PR_ERR_OUT_OF_MEMORY);
  }
  // δ partial chunks per (slice, instance): upper bound over every producer (PINN CTAs with one
  // point per thread, 256-wide copy blocks, streamed tiles, one resident system)
  c->nch = std::max(1, (c->M + kPinnTPB - 1) / kPinnTPB);
  if (split_allowed(c)) c->nch = std::max(1, (c->M + pr::kPinnSplitMinPPC - 1) / pr::kPinnSplitMinPPC);
  if (dd.world > 1 && loop_id(dd.nccl_id)) {  // test transport (one process, one GPU)
    c->loop = loop_join(dd.nccl_id, dd.world);
    if (!c->loop) {
      c->err = "loopback group joined with a different world size";
      return bail(PR_ERR_INVALID_ARGUMENT);
    }
  } else if (dd.world > 1) {
    Nccl &n = nccl();
    if (!n.ok) {
      c->err = n.why;
      return bail(PR_ERR_NCCL);
    }
    ncclUniqueId id;
    std::memcpy(id.internal, dd.nccl_id, 128);
    ncclResult_t e = n.CommInitRank(&c->comm, dd.world, id, dd.rank);
    if (e != 0) {
      c->err = fmt("ncclCommInitRank: %s", n.GetErrorString(e));
      c->comm = nullptr;
      return bail(PR_ERR_NCCL);
    }
  }
  *out = c;
  return PR_OK;
}

pr_status parareal_workspace_bytes(const pr_ctx *ctx, size_t *bytes) {
  pr_ctx *c = const_cast<pr_ctx *>(ctx);
  pr_status st = check_ctx(c);
  if (st) return st;
  if (!bytes) return fail(c, PR_ERR_INVALID_ARGUMENT, "bytes is NULL");
  pr_ctx tmp_view = *c;  // layout() only writes pointer fields of the copy
  *bytes = layout(&tmp_view, nullptr);
  return PR_OK;
}

pr_status parareal_bind_workspace(pr_ctx *c, void *ptr, size_t bytes) {
  pr_status st = check_ctx(c);
  if (st) return st;
  if (c->ws_ready) return fail(c, PR_ERR_STATE, "workspace already in use (bind before the first solve)");
  if (!ptr || ((uintptr_t)ptr % 256)) return fail(c, PR_ERR_INVALID_ARGUMENT, "device_ptr is NULL or not 256-B aligned");
  pr_ctx tmp_view = *c;
  const size_t need = layout(&tmp_view, nullptr);
  if (bytes < need) return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("workspace of %zu bytes < required %zu", bytes, need));
  c->ws = ptr;
  c->ws_bytes = bytes;
  c->own_ws = false;
  return PR_OK;
}

pr_status parareal_load_pinn_weights(pr_ctx *c, int32_t n_linear, const int32_t *dims, const float *const *W,
                                     const float *const *b, int32_t activation, const float *in_scale,
                                     float out_scale, int32_t precision) {
  pr_status st = check_ctx(c);
  if (st) return st;
  drop_graph(c);  // the parameter-space PINN kernels capture the weights by value
  if (n_linear < 2) return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("n_linear=%d must be >= 2 (at least one hidden layer)", n_linear));
  if (!dims || !W || !b) return fail(c, PR_ERR_INVALID_ARGUMENT, "dims/W/b must be non-NULL");
  if (dims[0] != 2 && dims[0] != 4) return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("dims[0]=%d must be 2 or 4", dims[0]));
  if (dims[n_linear] != 1) return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("dims[%d]=%d must be 1", n_linear, dims[n_linear]));
  const int Wd = dims[1];
  for (int l = 1; l < n_linear; ++l)
    if (dims[l] != Wd) return fail(c, PR_ERR_UNSUPPORTED, fmt("dims[%d]=%d: hidden widths must all equal dims[1]=%d", l, dims[l], Wd));
  if (activation != PR_ACT_TANH && activation != PR_ACT_RELU)
    return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("activation=%d unknown", activation));
  if (precision < 0 || precision > PR_PREC_FP16X1_TC) return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("precision=%d unknown", precision));
  const bool tc = precision != PR_PREC_FP32;
  if (precision == PR_PREC_TF32_TC)
    return fail(c, PR_ERR_UNSUPPORTED, "PR_PREC_TF32_TC is not in this build (PR_PREC_FP16X1_TC is the 1e-3 mode)");
  if (tc && (n_linear < 3 || !pr::pinn_tc_supported(dims[0], Wd, activation, tc_mode(precision))))
    return fail(c, PR_ERR_UNSUPPORTED, fmt("tensor-core PINN needs >= 2 hidden layers of width 64, 128 or 256 (got %d x %d)",
                                           n_linear - 1, Wd));
  if (!tc && !pr::pinn_smem_supported(dims[0], Wd, activation))
    return fail(c, PR_ERR_UNSUPPORTED, fmt("hidden width %d not instantiated (8,16,20,32,50,64; tensor cores: 64,128,256)", Wd));
  for (int l = 0; l < n_linear; ++l)
    if (!W[l] || !b[l]) return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("W[%d]/b[%d] is NULL", l, l));
  const int IN = dims[0], LH = n_linear - 1;
  // packed W_l then b_l per layer; the layers feeding a tanh are pre-scaled by 2·log2(e) so the
  // kernels evaluate tanh(z) = 1 − 2/(2^{z'} + 1) on z' = 2·log2(e)·z (pinn_chain.cuh)
  const double kTanhScale = 2.0 * 1.4426950408889634;  // 2·log2(e)
  std::vector<float> pk;
  for (int l = 0; l < n_linear; ++l) {
    const bool pre = activation == PR_ACT_TANH && l < n_linear - 1;
    const size_t nw = (size_t)dims[l + 1] * dims[l];
    for (size_t i = 0; i < nw; ++i) pk.push_back(pre ? (float)(kTanhScale * W[l][i]) : W[l][i]);
    for (int i = 0; i < dims[l + 1]; ++i) pk.push_back(pre ? (float)(kTanhScale * b[l][i]) : b[l][i]);
  }
  if (tc) {
    // K4: compact fp32 params (W0, b0, hidden biases, Wo, bo) + the hidden matrices in fp16/bf16,
    // core-matrix K-major (pinn_tc.cu)
    const int bf = tc_mode(precision);
    // packed fp32 layout (pk): W0[W][IN], b0[W], {W_l[W][W], b_l[W]} x (LH−1), Wo[W], bo
    const size_t n0 = (size_t)Wd * IN, nh = (size_t)Wd * Wd + Wd;
    const size_t le = pr::pinn_tc_layer_elems(Wd, bf);
    std::vector<uint16_t> wh((size_t)(LH - 1) * le);
    std::vector<float> tq(pk.begin(), pk.begin() + n0 + Wd);  // W0, b0
    for (int l = 1; l < LH; ++l) {
      const size_t o = n0 + Wd + (size_t)(l - 1) * nh;
      pr::pinn_tc_pack(pk.data() + o, Wd, bf, wh.data() + (size_t)(l - 1) * le);
      tq.insert(tq.end(), pk.begin() + o + (size_t)Wd * Wd, pk.begin() + o + nh);  // b_l
    }
    const size_t oo = n0 + Wd + (size_t)(LH - 1) * nh;
    tq.insert(tq.end(), pk.begin() + oo, pk.begin() + oo + Wd + 1);  // Wo, bo
    if (c->d_tcp) cudaFree(c->d_tcp);
    if (c->d_wh) cudaFree(c->d_wh);
    c->d_tcp = nullptr;
    c->d_wh = nullptr;
    CU(cudaMalloc(&c->d_tcp, tq.size() * sizeof(float)));
    CU(cudaMemcpy(c->d_tcp, tq.data(), tq.size() * sizeof(float), cudaMemcpyHostToDevice));
    CU(cudaMalloc(&c->d_wh, wh.size() * sizeof(uint16_t)));
    CU(cudaMemcpy(c->d_wh, wh.data(), wh.size() * sizeof(uint16_t), cudaMemcpyHostToDevice));
    c->tc_nfloats = (int)tq.size();
  }
  c->tc = tc ? precision : 0;
  const size_t bytes = pk.size() * sizeof(float);
  if (!tc && bytes > (size_t)kPinnSmemBudget)
    return fail(c, PR_ERR_UNSUPPORTED, fmt("network of %zu bytes exceeds the shared-memory budget", bytes));
  if (!tc) {
    // the attribute is per kernel and process-wide: set it to the whole budget (never lowered by
    // a smaller net loaded into another context that shares the kernel)
    CU(pr::pinn_smem_prepare(IN, Wd, activation, kPinnSmemBudget));
    if (pr::pinn_split_supported(IN, Wd, activation, pr::kPinnSplitG))
      CU(pr::pinn_split_prepare(IN, Wd, activation, pr::kPinnSplitG, kPinnSmemBudget));
  }
  if (c->d_wts) cudaFree(c->d_wts);
  c->d_wts = nullptr;
  CU(cudaMalloc(&c->d_wts, bytes));
  CU(cudaMemcpy(c->d_wts, pk.data(), bytes, cudaMemcpyHostToDevice));
  if (c->d_wgrp) cudaFree(c->d_wgrp);
  c->d_wgrp = nullptr;
  if (!tc && pr::pinn_group_G(Wd) > 0 && pr::pinn_split_supported(IN, Wd, activation, pr::pinn_group_G(Wd))) {
    // group kernels (pinn_chain.cuh, mlp_group): hidden matrix l stored as [i][q][k] =
    // W_l[q·NPT + k][i], so the G threads of a group read consecutive addresses for input i
    const int G = pr::pinn_group_G(Wd), NPT = Wd / G;
    std::vector<float> pg(pk);
    for (int l = 1; l < LH; ++l) {
      const size_t o = (size_t)Wd * IN + Wd + (size_t)(l - 1) * ((size_t)Wd * Wd + Wd);
      for (int i = 0; i < Wd; ++i)
        for (int q = 0; q < G; ++q)
          for (int k = 0; k < NPT; ++k)
            pg[o + ((size_t)i * G + q) * NPT + k] = pk[o + (size_t)(q * NPT + k) * Wd + i];
    }
    CU(cudaMalloc(&c->d_wgrp, bytes));
    CU(cudaMemcpy(c->d_wgrp, pg.data(), bytes, cudaMemcpyHostToDevice));
  }
  c->h_wts = pk;
  c->IN = IN;
  c->W = Wd;
  c->LH = LH;
  c->act = activation;
  c->nfloats = (int)pk.size();
  for (int i = 0; i < 4; ++i) c->cs[i] = 1.f;
  if (in_scale)
    for (int i = 0; i < IN; ++i) c->cs[i] = in_scale[i];
  c->out_scale = out_scale;
  c->have_pinn = true;
  return PR_OK;
}

pr_status parareal_solve(pr_ctx *c, const float *V_T, float *V_0, pr_report *rep) {
  pr_status st = check_ctx(c);
  if (st) return st;
  if (c->rank == 0 && !V_0) return fail(c, PR_ERR_INVALID_ARGUMENT, "V_0 is NULL on rank 0");
  return solve_impl(c, V_T, V_0, false, rep);
}

pr_status parareal_solve_device(pr_ctx *c, const float *d_V_T, float *d_V_0, pr_report *rep) {
  pr_status st = check_ctx(c);
  if (st) return st;
  return solve_impl(c, d_V_T, d_V_0, true, rep);
}

pr_status parareal_serial_fine(pr_ctx *c, const float *V_T, float *V_0, double *ms) {
  pr_status st = check_ctx(c);
  if (st) return st;
  return serial_fine_impl(c, V_T, V_0, false, ms);
}

pr_status parareal_serial_fine_device(pr_ctx *c, const float *d_V_T, float *d_V_0, double *ms) {
  pr_status st = check_ctx(c);
  if (st) return st;
  return serial_fine_impl(c, d_V_T, d_V_0, true, ms);
}

pr_status parareal_initial_state(pr_ctx *c, float *V_T) {
  pr_status st = check_ctx(c);
  if (st) return st;
  if (!V_T) return fail(c, PR_ERR_INVALID_ARGUMENT, "V_T is NULL");
  if ((st = ensure_ws(c))) return st;
  float *save = c->U;
  c->U = c->tmp;
  st = load_initial(c, nullptr, false);
  c->U = save;
  if (st) return st;
  if ((st = store_rows(c, V_T, c->tmp, false))) return st;
  SYNC();
  return PR_OK;
}

pr_status parareal_apply_fine(pr_ctx *c, int32_t n, const float *U_in, float *U_out) {
  pr_status st = check_ctx(c);
  if (st) return st;
  if (n < 0 || n >= c->N) return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("n=%d outside [0, N=%d)", n, c->N));
  if (!U_in || !U_out) return fail(c, PR_ERR_INVALID_ARGUMENT, "U_in/U_out is NULL");
  if ((st = ensure_ws(c))) return st;
  float *save = c->U;
  c->U = c->tmp;
  st = load_initial(c, U_in, false);
  c->U = save;
  if (st) return st;
  const size_t row = (size_t)c->B * c->Mp;
  if (use_grid(c, 1)) {
    if ((st = grid_sweep(c, 0, 1, n, c->tmp, c->tmp + row, -1))) return st;
  } else if (use_resident(c)) {
    pr::ResidentArgs a = base_args(c, c->fine);
    a.n_base = n;
    a.ln0 = 0;
    a.nsl = 1;
    a.U = c->tmp;
    a.Fout = c->tmp + row;
    LAUNCH(dispatch_res(false, c->M, a, c->B, c->stream));
  } else {
    pr::StreamedJob j;
    j.U = c->tmp; j.Gh = nullptr; j.D = nullptr; j.Fk = nullptr; j.fk_ln = -1; j.Fout = c->tmp + row;
    j.ln0 = 0; j.nsl = 1; j.n_base = n;
    int nl = 0;
    cudaError_t e = pr::streamed_sweep(c->sst, sprob(c, c->fine), j, c->stream, &nl);
    c->launches += nl;
    if (e != cudaSuccess) return fail(c, PR_ERR_CUDA, fmt("streamed apply: %s", cudaGetErrorString(e)));
  }
  if ((st = store_rows(c, U_out, c->tmp + row, false))) return st;
  SYNC();
  return grid_check(c);
}

pr_status parareal_apply_coarse(pr_ctx *c, int32_t n, const float *U_in, float *U_out) {
  pr_status st = check_ctx(c);
  if (st) return st;
  if (n < 0 || n >= c->N) return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("n=%d outside [0, N=%d)", n, c->N));
  if (!U_in || !U_out) return fail(c, PR_ERR_INVALID_ARGUMENT, "U_in/U_out is NULL");
  if (c->coarse == PR_COARSE_PINN && !c->have_pinn) return fail(c, PR_ERR_STATE, "no PINN weights loaded");
  if ((st = ensure_ws(c))) return st;
  float *save = c->U;
  c->U = c->tmp;
  st = load_initial(c, U_in, false);
  c->U = save;
  if (st) return st;
  const size_t row = (size_t)c->B * c->Mp;
  if (c->coarse == PR_COARSE_PINN) {
    pr::PinnArgs a = pinn_args(c);
    a.n_base = n;
    a.ln0 = 0;
    a.ln1 = 1;
    a.U = c->tmp;
    a.Gout = c->tmp + row;
    if ((st = launch_pinn(c, a))) return st;
    if ((st = store_rows(c, U_out, c->tmp + row, false))) return st;
  } else if (use_resident(c)) {
    pr::ResidentArgs a = base_args(c, c->crs);
    a.n_base = n;
    a.Uw = c->tmp;
    a.ustride = 0;
    a.c_ln0 = 0;
    a.c_ln1 = 1;
    LAUNCH(dispatch_res(true, c->M, a, c->B, c->stream));
    if ((st = store_rows(c, U_out, c->tmp, false))) return st;
  } else {
    pr::StreamedChainJob j;
    j.U = c->tmp; j.Gh = nullptr; j.D = nullptr; j.Fcopy = nullptr; j.partials = nullptr; j.nch = 1;
    j.ln0 = 0; j.ln1 = 1; j.n_base = n; j.ustride = 0;
    int nl = 0;
    cudaError_t e = pr::streamed_chain(c->sst, sprob(c, c->crs), j, c->stream, &nl);
    c->launches += nl;
    if (e != cudaSuccess) return fail(c, PR_ERR_CUDA, fmt("streamed coarse apply: %s", cudaGetErrorString(e)));
    if ((st = store_rows(c, U_out, c->tmp, false))) return st;
  }
  SYNC();
  return PR_OK;
}

pr_status parareal_copy_iterates(pr_ctx *c, int32_t n_first, int32_t n_count, float *host) {
  pr_status st = check_ctx(c);
  if (st) return st;
  if (!c->solved) return fail(c, PR_ERR_STATE, "no solve has run on this context");
  if (!host || n_count < 0 || n_first < c->n0 || n_first + n_count > c->n1 + 1)
    return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("[n_first=%d, +%d) not within this rank's [%d, %d]", n_first, n_count,
                                                c->n0, c->n1));
  const size_t row = (size_t)c->B * c->Mp;
  for (int i = 0; i < n_count; ++i) {
    if ((st = store_rows(c, host + (size_t)i * c->B * c->M, c->U + (size_t)(n_first - c->n0 + i) * row, false)))
      return st;
  }
  SYNC();
  return PR_OK;
}

pr_status parareal_plan_iteration(int32_t N, int32_t world, int32_t rank, int32_t k, pr_plan *out) {
  pr_ctx *c = nullptr;
  if (!out) return fail(c, PR_ERR_INVALID_ARGUMENT, "out is NULL");
  if (N < 1 || world < 1 || N % world || rank < 0 || rank >= world || k < 0)
    return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("plan(N=%d, world=%d, rank=%d, k=%d) invalid", N, world, rank, k));
  *out = make_plan(N, world, rank, k);
  return PR_OK;
}

pr_status parareal_set_option(pr_ctx *c, int32_t key, int64_t value) {
  pr_status st = check_ctx(c);
  if (st) return st;
  drop_graph(c);  // a captured solve bakes in kernel choices
  switch (key) {
    case PR_OPT_FINE_KERNEL:
      if (value < 0 || value > 3) return fail(c, PR_ERR_INVALID_ARGUMENT, "PR_OPT_FINE_KERNEL must be 0, 1, 2 or 3");
      if (value == 3 && !c->fine.g_pt)
        return fail(c, PR_ERR_UNSUPPORTED, "grid-resident fine kernel needs theta = 1, B = 1, M > 2048 and a grid that fits the GPU");
      if (value == 1 && c->M > kResidentMaxM)
        return fail(c, PR_ERR_UNSUPPORTED, fmt("resident fine kernel needs M <= %d", kResidentMaxM));
      c->opt_fine_kernel = (int)value;
      return PR_OK;
    case PR_OPT_PINN_KERNEL:
      if (value < 0 || value > 2) return fail(c, PR_ERR_INVALID_ARGUMENT, "PR_OPT_PINN_KERNEL must be 0, 1 or 2");
      if (value == 2 && !split_allowed(c))
        return fail(c, PR_ERR_UNSUPPORTED, fmt("latency-mode PINN kernel needs B*M <= %ld", kSplitMaxPoints));
      c->opt_pinn_kernel = (int)value;
      return PR_OK;
    case PR_OPT_USE_GRAPHS:
      if (value < 0 || value > 2) return fail(c, PR_ERR_INVALID_ARGUMENT, "PR_OPT_USE_GRAPHS must be 0, 1 or 2");
      if (value != c->opt_graphs) drop_graph(c);
      c->opt_graphs = (int)value;
      return PR_OK;
    case PR_OPT_PIPELINE:
      if (value < 0 || value > 1) return fail(c, PR_ERR_INVALID_ARGUMENT, "PR_OPT_PIPELINE must be 0 or 1");
      c->opt_pipeline = (int)value;
      return PR_OK;
    case PR_OPT_WAVEFRONT:
      if (value < 0 || value > 4096) return fail(c, PR_ERR_INVALID_ARGUMENT, "PR_OPT_WAVEFRONT must be in [0, 4096]");
      c->opt_wavefront = (int)value;
      return PR_OK;
    case PR_OPT_SPATIAL_CHAIN:
      if (value < 0 || value > 2) return fail(c, PR_ERR_INVALID_ARGUMENT, "PR_OPT_SPATIAL_CHAIN must be 0, 1 or 2");
      c->opt_spatial = (int)value;
      return PR_OK;
    case PR_OPT_COMM_TIMEOUT_MS:
      if (value < 0) return fail(c, PR_ERR_INVALID_ARGUMENT, "PR_OPT_COMM_TIMEOUT_MS must be >= 0");
      c->comm_timeout_ms = value;
      return PR_OK;
  }
  return fail(c, PR_ERR_INVALID_ARGUMENT, fmt("unknown option key %d", key));
}

void parareal_free(pr_ctx *c) {
  if (!c) return;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  drop_graph(c);
  if (c->loop) loop_leave(c->loop);
  if (c->comm) {
    Nccl &n = nccl();
    if (n.ok) (c->poisoned ? n.CommAbort(c->comm) : n.CommDestroy(c->comm));
  }
  free_scheme(c->fine);
  free_scheme(c->crs);
  cudaFree(c->d_fset);
  cudaFree(c->d_L);
  cudaFree(c->d_K);
  cudaFree(c->d_r);
  cudaFree(c->d_wts);
  cudaFree(c->d_wgrp);
  cudaFree(c->d_tcp);
  cudaFree(c->d_wh);
  if (c->own_ws) cudaFree(c->ws);
  if (c->h_delta) cudaFreeHost(c->h_delta);
  cudaFree(c->pipe_partials);
  cudaFree(c->g_tot);
  if (c->g_err_h) cudaFreeHost(c->g_err_h);
  cudaFree(c->sp_U);
  cudaFree(c->sp_Gh);
  cudaFree(c->sp_D);
  cudaFree(c->sp_F);
  cudaFree(c->sp_part);
  cudaFree(c->pipe_flags);
  cudaFree(c->pipe_wstage);
  for (auto e : c->ev) cudaEventDestroy(e);
  if (c->own_stream) cudaStreamDestroy(c->stream);
  delete c;
}

}  // extern "C"
