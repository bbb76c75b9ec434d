/* parareal.h — C ABI of the B200-native Parareal + PINN solver (ABI version 1).
 *
 * Implements the data-parallel hot path of arXiv 2303.03848 (Ibrahim,
 * Götschel, Ruprecht, "Parareal with a physics-informed neural network as
 * coarse propagator") for the Black–Scholes European call:
 *
 *   problem    PAPER.md:86-111 (§3, Eqs. 1-4): V_t + ½σ²S²V_SS + rSV_S − rV = 0,
 *              V(T,S) = max(S−K,0), V(t,0) = 0, upper bound S = L.
 *   slices     PAPER.md:121 (§3.1): N time slices [T^n, T^{n+1}].
 *   F          PAPER.md:122-127 Eq. (6) + §3.2: centred finite
 *              differences in S, implicit Euler in τ = T − t (reading Q1).
 *   G          PAPER.md:167 (§3.3) + Fig. 2 caption: a PINN mapping
 *              (t_start, t_end, V(t_start), S) → V(t_end), or implicit Euler.
 *   iteration  PAPER.md:129-135 Eq. (7): V^{k+1}_{n+1} = G(V^{k+1}_n) + F(V^k_n) − G(V^k_n),
 *              with the schedule and stop rule of DESIGN.md readings Q12-Q14.
 *
 * Conventions
 *  - Ownership: every pointer argument is borrowed for the duration of the
 *    call only; nothing is retained.  The context owns the device memory it
 *    allocates, unless the caller binds a workspace with
 *    parareal_bind_workspace (the caller then keeps it alive until
 *    parareal_free).
 *  - Errors: every call returns pr_status; parareal_last_error(ctx) returns
 *    a message naming the offending field or failing call.  No exception
 *    crosses the ABI and nothing aborts or exits.  After a CUDA or NCCL
 *    failure the context is poisoned: every later call except
 *    parareal_free / parareal_last_error returns PR_ERR_STATE.
 *  - Threading: a context is used by one host thread at a time.  With
 *    world > 1, parareal_init, parareal_solve[_device] and parareal_free are
 *    collective over all ranks (same arguments on every rank).
 *  - Not converging within max_iter is NOT an error (rep->converged = 0).
 *  - Device work is issued on the stream given in pr_dist (or a stream the
 *    context creates); every call that returns host data synchronises it.
 *  - Precision: states are stored as fp32 [B][M] rows; the implicit solves
 *    run in fp64 arithmetic with fp64 factors.
 */
#ifndef PARAREAL_H
#define PARAREAL_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define PARAREAL_ABI_VERSION 1

typedef struct pr_ctx pr_ctx;

typedef enum {
  PR_OK = 0,
  PR_ERR_INVALID_ARGUMENT = 1, /* a field fails validation (message names it)        */
  PR_ERR_OUT_OF_MEMORY = 2,    /* device or pinned-host allocation failed             */
  PR_ERR_CUDA = 3,             /* a CUDA runtime call failed (context poisoned)       */
  PR_ERR_NCCL = 4,             /* NCCL missing or failed (context poisoned)           */
  PR_ERR_STATE = 5,            /* call not valid in this state (e.g. no PINN weights) */
  PR_ERR_NUMERICAL = 6,        /* non-positive pivot while factorising        */
  PR_ERR_UNSUPPORTED = 7       /* valid request this build does not implement        */
} pr_status;

/* coarse propagator kind (P:162 numerical G; P:167 PINN G) */
enum { PR_COARSE_PINN = 0, PR_COARSE_IMPLICIT_EULER = 1 };
/* upper boundary value V(L, τ) (reading Q3): asymptotic L − K e^{−rτ} (default) or 0 */
enum { PR_BC_CALL_ASYMPTOTIC = 0, PR_BC_ZERO = 1 };
/* hidden-layer activation: tanh (north_star) or ReLU */
enum { PR_ACT_TANH = 0, PR_ACT_RELU = 1 };
/* PINN arithmetic.  FP32: fp32 SIMT kernels (any width instantiated: 8,16,20,32,50,64), parity 1e-5.
 * The tensor-core modes (K4: tcgen05, hidden widths 64/128/256 with >= 2 hidden layers, fp32
 * accumulation in TMEM; north_star's tensor-core tolerance is 1e-3):
 * FP16_TC:   operands split hi + lo in fp16, three MMAs per product: fp32-level accuracy (1e-4 tests).
 * FP16X1_TC: one fp16 pass (unit roundoff 2^-11 on [-1,1] activations), exact tanh: one MMA per
 *            product; measured 3e-4 .. 4e-3 of the row maximum on random Kaiming nets,
 *            8x finer than BF16_TC, but not within 1e-3 for every net: only FP16_TC is.
 * BF16_TC:   one bf16 pass, tanh.approx: fastest, ~1e-2 (outside north_star's 1e-3; not credited).
 * TF32_TC:   not in this build (PR_ERR_UNSUPPORTED). */
enum { PR_PREC_FP32 = 0, PR_PREC_FP16_TC = 1, PR_PREC_BF16_TC = 2, PR_PREC_TF32_TC = 3, PR_PREC_FP16X1_TC = 4 };

/* Problem statement.  Host pointers, copied by init. */
typedef struct {
  uint32_t struct_size;         /* = sizeof(pr_problem) (ABI check)                          */
  int32_t M;                    /* interior grid points; S_j = j·L_b/(M+1), j = 1..M (Q4)   */
  int32_t B;                    /* independent instances (portfolio, config C4)              */
  const double *strike;         /* [B] K_b ≥ 0                                               */
  const double *sigma;          /* [B] σ_b > 0                                               */
  const double *rate;           /* [B] r_b ≥ 0                                               */
  const double *L;              /* [B] artificial bound L_b > K_b                    */
  double T;                     /* expiry > 0                                                */
  int32_t upper_bc;             /* PR_BC_*                                                   */
  int32_t N;                    /* time slices ≥ 1; N % world == 0                   */
  int32_t fine_steps;           /* implicit steps per slice of F ≥ 1 (Q2)                    */
  double fine_theta;            /* θ of the fine θ-step, in [0.5, 1]: 1 implicit Euler (Q1), 0.5 Crank–Nicolson (NEXT-1) */
  int32_t coarse;               /* PR_COARSE_*                                               */
  int32_t coarse_steps;         /* implicit Euler steps per slice for numerical G ≥ 1        */
  int32_t max_iter;             /* 1 ≤ max_iter ≤ N                                          */
  double tol;                   /* stop at the first k with δ^k < tol; 0 → run max_iter     */
} pr_problem;

/* Process placement.  world == 1: single GPU, nccl_id must be NULL.
 * Test transport: an id whose first 8 bytes are "PRLOOPBK" makes the world contexts created
 * with the same id in ONE process (one host thread per rank, any device) exchange through
 * device mailboxes instead of NCCL (send / receive / MAX all-reduce, fully synchronous); every
 * other step is the multi-process path.  For tests on a single GPU only. */
typedef struct {
  int32_t rank, world;          /* this process / all processes (one GPU each)               */
  int32_t device;               /* CUDA device ordinal                                       */
  const uint8_t *nccl_id;       /* 128 bytes from parareal_get_nccl_id on rank 0, broadcast   */
  void *stream;                 /* cudaStream_t to issue on, or NULL → context-owned stream  */
} pr_dist;

/* Result report (S:356-359 ParRealReport analogue). */
typedef struct {
  int32_t iterations;           /* K: fine sweeps executed after the k=0 coarse sweep (Q14)  */
  int32_t converged;            /* 1 iff δ^K < tol                                           */
  double *delta;                /* caller buffer [max_iter] or NULL: δ^k, k = 1..K            */
  double ms_total;              /* device time of the solve on this rank                      */
  double ms_coarse, ms_fine, ms_comm, ms_setup;  /* per-phase device time on this rank; with world > 1
                                   ms_coarse includes the chain's hand-offs of U_{n0}/U_{n1} (they
                                   overlap the chain in the wavefront) and ms_comm is the gather of U_N */
  int64_t kernel_launches;      /* this library's kernels launched during the solve          */
} pr_report;

const char *parareal_status_string(pr_status s);
/* Last error message of ctx (or of the last failed init when ctx == NULL).  Never NULL. */
const char *parareal_last_error(const pr_ctx *ctx);

/* Writes a fresh NCCL unique id (128 bytes) for a world > 1 init.  PR_ERR_NCCL if NCCL
 * cannot be loaded. */
pr_status parareal_get_nccl_id(uint8_t out[128]);

/* Validates *prob (PR_ERR_INVALID_ARGUMENT naming the field: σ>0, T>0, r≥0, L>K≥0, M≥1,
 * N≥1, steps≥1, 1≤max_iter≤N, tol≥0, N % world == 0, 0.5 ≤ fine_theta ≤ 1), selects the device,
 * factorises M_f = I − dτ_f A (and M_c for numerical G) in fp64 on the host
 * (PR_ERR_NUMERICAL on a non-positive pivot), uploads factors and, for world > 1, creates
 * the NCCL communicator (collective).  Rank r owns slices [rN/world, (r+1)N/world). */
pr_status parareal_init(const pr_problem *prob, const pr_dist *dist, pr_ctx **out);

/* Device bytes the context needs for its iterate storage. */
pr_status parareal_workspace_bytes(const pr_ctx *ctx, size_t *bytes);
/* Optional: use caller device memory (≥ workspace_bytes, 256-B aligned) instead of cudaMalloc. */
pr_status parareal_bind_workspace(pr_ctx *ctx, void *device_ptr, size_t bytes);

/* PINN coarse propagator weights (reading Q6-Q11).
 *   n_linear affine layers; dims[n_linear+1] with dims[0] ∈ {2,4}, dims[n_linear] = 1 and
 *   all hidden widths equal (one of 8, 16, 20, 32, 50, 64);  W[l] row-major [dims[l+1]][dims[l]],
 *   b[l] [dims[l+1]] (host fp32, copied);  activation PR_ACT_*;  in_scale [dims[0]] extra input
 *   multipliers (NULL → 1);  out_scale extra output multiplier;  precision PR_PREC_*.
 * G_n(U)_j = L_b·out_scale·MLP(c0·t_from/T, c1·t_to/T, c2·U_j/L_b, c3·S_j/L_b)
 *   with t_from = T − nΔT, t_to = T − (n+1)ΔT  (2-input form: (c0·t_to/T, c1·S_j/L_b)). */
pr_status parareal_load_pinn_weights(pr_ctx *ctx, int32_t n_linear, const int32_t *dims,
                                     const float *const *W, const float *const *b, int32_t activation,
                                     const float *in_scale, float out_scale, int32_t precision);

/* Runs Parareal (collective).  V_T: host [B][M] initial state at τ = 0 (t = T), or NULL →
 * payoff max(S_j − K_b, 0) (Eq. 2).  V_0: host [B][M], receives U^K_N (prices at t = 0) on
 * rank 0 (ignored on other ranks; may be NULL there).  rep may be NULL.
 * PR_ERR_STATE if coarse == PINN and no weights are loaded. */
pr_status parareal_solve(pr_ctx *ctx, const float *V_T, float *V_0, pr_report *rep);
/* Same with device pointers (d_V_T may be NULL; d_V_0 on rank 0), stream-ordered on the
 * context stream; returns after the result is complete on the device. */
pr_status parareal_solve_device(pr_ctx *ctx, const float *d_V_T, float *d_V_0, pr_report *rep);

/* Serial fine propagation V_{n+1} = F(V_n), n = 0..N−1 (Eq. 6) of all N slices on THIS
 * rank's GPU (not collective): the speedup baseline.  Host arrays as in parareal_solve;
 * *ms (nullable) receives the device time. */
pr_status parareal_serial_fine(pr_ctx *ctx, const float *V_T, float *V_0, double *ms);
pr_status parareal_serial_fine_device(pr_ctx *ctx, const float *d_V_T, float *d_V_0, double *ms);

/* Writes the initial state U_0 = max(S_j − K_b, 0) (Eq. 2) of every instance into
 * host [B][M] (computed by the same device kernel parareal_solve uses when V_T == NULL). */
pr_status parareal_initial_state(pr_ctx *ctx, float *V_T);

/* Test hooks (single-propagator parity).  U_in/U_out host [B][M]; n is a
 * global slice index 0..N−1.  apply_coarse uses the configured coarse propagator. */
pr_status parareal_apply_fine(pr_ctx *ctx, int32_t n, const float *U_in, float *U_out);
pr_status parareal_apply_coarse(pr_ctx *ctx, int32_t n, const float *U_in, float *U_out);
/* Copies boundary states U_n, n ∈ [n_first, n_first+n_count) (global indices owned by this
 * rank, i.e. within [n0, n1]) of the last solve into host [n_count][B][M]. */
pr_status parareal_copy_iterates(pr_ctx *ctx, int32_t n_first, int32_t n_count, float *host);

/* Per-rank work of Parareal iteration k (reading Q12 schedule; P:130-136 with the N slices
 * sharded contiguously, rank r owning global slices [n0, n1) = [rN/world, (r+1)N/world)).
 * All indices are LOCAL (global = n0 + local).  parareal_solve executes exactly this plan;
 * it is exported so the host-side distributed logic is testable without a GPU.
 *   k = 0: no fine sweep; recv U_{n0} from rank−1 (r > 0); G-chain over [0, Nloc); send U_{n1}.
 *   k ≥ 1: fine sweep over [fine_lo, fine_hi) reading U^{k−1} (D_n = F̂_n − Ĝ_n, and F̂ of
 *          fk_local → U_k);  then either copy (U_k := F̂_{k−1} at chain_lo) or recv, the
 *          G-chain with correction over [chain_lo, chain_hi), and send; δ partials of the
 *          boundary states [delta_lo, delta_hi] (inclusive; empty when lo > hi). */
typedef struct {
  int32_t fine_lo, fine_hi;     /* local slices swept by F (empty when lo ≥ hi)             */
  int32_t fk_local;             /* local slice whose F̂ becomes U_k, or −1                   */
  int32_t recv_first;           /* 1: receive U_{n0} from rank−1 before the chain           */
  int32_t copy;                 /* 1: the chain starts with U_k := F̂_{k−1} at chain_lo      */
  int32_t chain_lo, chain_hi;   /* local slices chained by G (may be empty with copy = 1)   */
  int32_t send_last;            /* 1: send U_{n1} (local index Nloc) to rank+1 afterwards  */
  int32_t delta_lo, delta_hi;   /* local boundary indices this rank reduces into δ^k        */
} pr_plan;
/* PR_ERR_INVALID_ARGUMENT unless N ≥ 1, 1 ≤ world, N % world == 0, 0 ≤ rank < world, k ≥ 0. */
pr_status parareal_plan_iteration(int32_t N, int32_t world, int32_t rank, int32_t k, pr_plan *out);

/* Tuning/test options (values are validated; unknown keys → PR_ERR_INVALID_ARGUMENT). */
enum {
  PR_OPT_FINE_KERNEL = 1,   /* 0 auto, 1 resident K1 (M ≤ 2048), 2 streamed K2, 3 grid-resident K2R
                               (θ = 1, B = 1, M > 2048, partition fits the GPU; else PR_ERR_UNSUPPORTED).
                               Auto: K1 for M ≤ 2048, else K2R or K2 by a fitted cost model (K2R for
                               every sweep at 2^18 … 2^20 points, K2 for many small systems).  */
  PR_OPT_USE_GRAPHS = 2,    /* 0/1: a fixed-K (tol == 0), single-GPU solve with device pointers (or pinned
                               host buffers, whose copies become graph nodes) is captured
                               into a CUDA graph on its first call per (V_T, V_0) pair and replayed on
                               later calls (same kernels, same results); any other solve runs eagerly.
                               set_option / load_pinn_weights / free discard the captured graph.
                               2: the same, but the graph is captured without the phase-timing events
                               and a device-pointer replay returns as soon as it is enqueued on the context stream
                               (stream-ordered, like a library call: the caller synchronises; rep, if
                               given, receives iterations and kernel_launches, zero times, no δ).  */
  PR_OPT_PINN_KERNEL = 3,   /* 0 auto, 1 shared-memory weights, 2 latency mode (4 threads/point; B·M ≤ 65536) */
  PR_OPT_PIPELINE = 4,      /* 0 auto: a single-GPU fixed-K (tol == 0) solve with PINN G in latency mode (or
                               the numerical G) and the resident fine kernel at M ≤ 1024 runs pipelined
                               (SURVEY NEXT-2): fine
                               solves and the coarse chain overlapped in one cooperative kernel, bitwise the
                               blocking results; its report gives the overlapped time as both ms_fine and
                               ms_coarse.  1: always the blocking schedule. */
  PR_OPT_COMM_TIMEOUT_MS = 5, /* world > 1 with NCCL: every host wait on the context stream polls
                               ncclCommGetAsyncError; an asynchronous NCCL error, or a wait longer than
                               this many milliseconds (a peer rank that died or hangs), aborts the
                               communicator and poisons the context (PR_ERR_NCCL) instead of hanging.
                               Default 600000; 0 waits forever.  No effect with world == 1. */
  PR_OPT_WAVEFRONT = 6,      /* world > 1, PINN G, B == 1: the coarse chain runs as a wavefront of j-chunks
                               across ranks (G is pointwise in S): each chunk of U_{n1} goes
                               to the next rank as soon as it is chained, so the ranks chain concurrently.
                               Results are bitwise those of the blocking chain (the chunks are CTA ranges
                               of the same kernel).  0 auto (8 chunks when M ≥ 65536, else blocking),
                               1 blocking, n ≥ 2: n chunks (at most one per CTA).  Numerical G (coupled in
                               S) and B > 1 always chain blocking. */
  PR_OPT_SPATIAL_CHAIN = 7   /* world > 1, PINN G, B == 1: every rank chains ALL slices over
                               its own range of grid points (G is pointwise in S) while the fine sweep
                               stays sharded by slices; per iteration U/Ĝ rows go to the slice owners and
                               D rows (+ F̂_{k−1}) back, δ's partial slots are summed over ranks.  Bitwise
                               the one-rank results.  0 auto (on for tensor-core nets, whose chain
                               dominates), 1 off (slice-sharded chain / wavefront), 2 on. */
};
pr_status parareal_set_option(pr_ctx *ctx, int32_t key, int64_t value);

/* Releases everything the context owns (collective for world > 1).  NULL-safe. */
void parareal_free(pr_ctx *ctx);

#ifdef __cplusplus
}
#endif
#endif /* PARAREAL_H */
