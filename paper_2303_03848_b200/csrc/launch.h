// launch.h — argument structs and the launchers each kernel translation unit exports to
// the host code (parareal.cu).  Kernel bodies are compiled only in their own .cu file.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#define PR_ARGS_ONLY
#include "fine_resident.cuh"
#include "fine_streamed.cuh"
#include "pinn_chain.cuh"
#undef PR_ARGS_ONLY

namespace pr {
// K1 (res.cu): sweep (chain=false) or serial chain (chain=true) over nsys systems
cudaError_t launch_resident(bool chain, int M, const ResidentArgs &a, int nsys, cudaStream_t s);
// K3, shared-memory weights (pinn_smem.cu)
bool pinn_smem_supported(int IN, int W, int act);
int pinn_smem_pts(int W);
cudaError_t pinn_smem_prepare(int IN, int W, int act, int smem_bytes);
cudaError_t launch_pinn_smem(int IN, int W, int act, const PinnArgs &a, dim3 grid, size_t smem, cudaStream_t s);
// K3 latency mode (pinn_smem.cu): G threads per point; G = kPinnSplitG with 20-wide nets is the
// shuffle kernel, any other G a group kernel (shared-memory exchange, group-ordered weights:
// pinn_group_G(W) = 10 for 20/50-wide, 8 for 32-wide, 16 for 64-wide nets); pinn_split_ppc(G)
// points per 128-thread CTA
constexpr int kPinnSplitG = 4;
constexpr int kPinnSplitMinPPC = 8;  // the fewest points per CTA of any latency-mode kernel
int pinn_group_G(int W);
bool pinn_split_is_group(int W, int G);
int pinn_split_ppc(int G);
bool pinn_split_supported(int IN, int W, int act, int G);
cudaError_t pinn_split_prepare(int IN, int W, int act, int G, int smem_bytes);
cudaError_t launch_pinn_split(int IN, int W, int act, int G, const PinnArgs &a, dim3 grid, size_t smem,
                              cudaStream_t s);
// K3, constant-bank weights (pinn_param.cu)
bool pinn_param_supported(int IN, int W, int LH, int act);
cudaError_t launch_pinn_param(int IN, int W, int LH, int act, const float *pk, const PinnArgs &a, dim3 grid,
                              cudaStream_t s);
// K4: PINN chain on tcgen05 tensor cores for wide nets (pinn_tc.cu); wts = compact fp32 params
// K4 operand modes: hi + lo fp16 (3 MMAs, fp32-level), one bf16 pass, one fp16 pass
enum { kTcSplit16 = 0, kTcBF16 = 1, kTcF16 = 2 };
bool pinn_tc_supported(int IN, int W, int act, int mode);
size_t pinn_tc_smem(int W, int LH, int nfloats, int mode, bool *resident);
size_t pinn_tc_layer_elems(int W, int mode);
void pinn_tc_pack(const float *Wl, int W, int mode, uint16_t *out);
int pinn_tc_points_per_cta(int W, int LH, int nfloats, int mode);  // 256 (ping-pong kernel) or 128
cudaError_t launch_pinn_tc(int IN, int W, int act, int mode, const PinnArgs &a, const void *wh, dim3 grid,
                           cudaStream_t s);
// K2R grid-resident fine sweep (fine_grid.cu): one system per GPU, NS systems at a time, state in
// registers for all passes; θ = 1, one instance (B = 1).
struct GridArgs {
  int M, nsys, ln0, n_base, steps;  // systems = local slices ln0 … ln0 + nsys − 1 of instance 0
  size_t row;                        // floats between slice rows (B·Mp)
  double dT, dtau, c0, c1;           // c0 = dτr/2, c1 = dτσ²/2 (closed-form off-diagonals)
  const double *ip, *iq;             // [M] 1/p_j (LU), 1/q_j (UL), natural layout
  double bcoef, Lb, Kb, rb;          // boundary term dτ(a_M+b_M)·g(τ) of instance 0
  int upper_bc;
  const double *lbP;                 // [2][nCTA][KW][3] look-back weights (maps between predecessor and CTA)
  const int *lbW;                    // [2][nCTA] look-back windows
  int KW;
  unsigned long long *tot;           // [4][nCTA][32] published CTA totals per pass slot (NS·4 words used): each
                                     // fp64 total as two words (32-bit half | pass id << 32), zeroed
                                     // before the launch
  int *err;                          // set when a look-back wait times out
  const float *U, *Gh;               // [.][row] inputs U_n, Ĝ_n
  float *D, *Fk, *Fout;              // outputs: D_n = F̂_n − Ĝ_n, F̂ of local slice fk_ln, or F̂ rows (test hook)
  int fk_ln;
  unsigned long long *trace;         // nullable: per (pass, CTA) %globaltimer stamps (PR_GRID_TRACE)
};
size_t fine_grid_smem(int PT, int steps);
int fine_grid_pt(int M, int nsm, int *nblocks);  // points per thread for M points (0: too large)
int fine_grid_ns(int PT, int nsys);               // systems per group of a launch over nsys systems
size_t fine_grid_tot_words(int nblocks);          // words of the look-back slots (GridArgs::tot)
cudaError_t launch_fine_grid(const GridArgs &a, int PT, int nblocks, cudaStream_t s);
// Pipelined Parareal on one GPU (pipe.cu, NEXT-2): PINN chain (latency mode) and K1 fine solves
// in one cooperative kernel, synchronised per slice.
struct PipeArgs {
  ResidentArgs r;          // fine scheme and the U / Gh / D / Fk rows
  PinnArgs g;              // coarse chain (same rows)
  ResidentArgs rc;         // numerical coarse G (PR_COARSE_IMPLICIT_EULER): its scheme (n_c steps)
  int N, K, C;             // slices, iterations, chain CTAs per instance
  int S;                   // chain CTA sets (set s runs the chains k ≡ s mod S; set by the launcher)
  int cpub;                // chain publications per (instance, slice): chain warps (PINN) or 1 (numerical)
  double *partials;        // [K+1][pstride] δ partials per iteration
  size_t pstride;
  double *wstage;          // [N+1][B·C][4 warps][2] per-warp δ partials of the current iteration
  int *cnt, *floaded, *fdone;  // [B][N] counters (contiguous), zero at launch; the kernel's tail
                               // zeroes them again for the next launch
  unsigned long long *gbar;    // [2] the tail's grid barrier: arrival count (0 between launches), generation
  unsigned long long *dmax;    // [K] δ^k (ordered double bits): zeroed at the start, set by the tail
  int nch;                     // δ chunks per (slice, instance) row
  unsigned long long *trace;   // nullable: [K+1][N][3] %globaltimer (chain warp 0 of CTA 0 at each
                               // slice; fine (n, b=0) start and end), for PR_PIPE_TRACE
};
bool pipe_supported(int M, bool cn, int IN, int W, int act, int G);  // G: chain threads per point (1: one)
bool pipe_num_supported(int M, bool cn);  // numerical coarse G (one K1 chain CTA per iteration and instance)
cudaError_t launch_parareal_pipe_num(const PipeArgs &pa, int M, bool cn, cudaStream_t s);
int pipe_chain_warps(int W, int G);  // warps per chain CTA (the chain's points per CTA = warps · 32/G)
cudaError_t launch_parareal_pipe(const PipeArgs &pa, int M, bool cn, int IN, int W, int act, int G,
                                 size_t smem, cudaStream_t s);
// K6/K7 (misc.cu)
cudaError_t launch_payoff(float *U0, int M, int Mp, int B, const double *Lb, const double *Kb, cudaStream_t s);
cudaError_t launch_delta(const double *partials, int B, int nch, int ln_lo, int ln_hi, unsigned long long *dmax,
                         cudaStream_t s);
}  // namespace pr
