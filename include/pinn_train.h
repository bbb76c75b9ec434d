/* pinn_train.h — C ABI of the GPU PINN trainer (same library as parareal.h).
 *
 * Trains the network the PINN coarse propagator evaluates, as PAPER.md §3.3 describes:
 *
 *   network     Ṽ(t, S) = L · y(t/T, S/L): a fully connected net, 2 inputs (t, S) — the
 *               function the losses are written over (reading Q28) — hidden layers
 *               of equal width W ∈ {8,16,20,32,50,64} with tanh (north_star) or ReLU,
 *               linear output (the paper's 10×50 ReLU net included; shared memory bounds the depth).
 *               The trained weights plug into parareal_load_pinn_weights unchanged as a 2-input
 *               G (dims[0] = 2, features (t_to/T, S/L_b), output × L_b; reading Q8).
 *   loss        MSE_total = MSE_f + MSE_exp + MSE_b (Eq. 11) over three collocation
 *               sets: the PDE residual f = Ṽ_t + ½σ²S²Ṽ_SS + rSṼ_S − rṼ on
 *               interior points (Eq. 12, Eq. 1), Ṽ − V on the boundary S ∈ {0, L} (Eq. 13; target
 *               0 at S = 0 (Eq. 3) and, at S = L, L − K e^{−r(T−t)} or 0 per upper_bc (reading Q3)),
 *               Ṽ(T, S) − max(S − K, 0) at expiry (Eq. 14, Eq. 2).
 *   derivatives Ṽ_t, Ṽ_S, Ṽ_SS by forward jets through every layer; the parameter gradient by
 *               reverse accumulation through the same chain rules ("automatic differentiation",
 *               P:191).  fp32 arithmetic, fp64 loss sums and block-gradient reductions.
 *   optimiser   Adam (β1, β2, ε from the config), learning rate per call, so the paper's
 *               schedule is two calls: (5000 epochs, 1e-2) then (800 epochs, 1e-3).
 *   batches     every epoch shuffles each set ("shuffled during every epoch") with a
 *               counter-based bijection of (seed, epoch, set) and splits each into `batches`
 *               consecutive parts; step s trains on part s mod batches of epoch s / batches.
 *               The shuffle is defined in DESIGN.md "PINN training" (SplitMix64 keys, four
 *               multiply/add/xor-shift rounds on ⌈log2 n⌉-bit integers, cycle-walking).
 *
 * Conventions: those of parareal.h (status codes, borrowed pointers copied by the call, no
 * exceptions, a CUDA failure poisons the trainer: later calls return PR_ERR_STATE).
 * One epoch is captured as a CUDA graph (batches × (gradient kernel, Adam kernel)) and replayed.
 */
#ifndef PINN_TRAIN_H
#define PINN_TRAIN_H

#include <stddef.h>
#include <stdint.h>

#include "parareal.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct pt_trainer pt_trainer;

typedef struct {
  uint32_t struct_size;          /* = sizeof(pt_config)                                          */
  double strike, sigma, rate;    /* K, σ > 0, r ≥ 0 of Eq. (1)-(2) the net is trained for         */
  double L, T;                   /* domain [0, L] × [0, T], L > 0, T > 0 ([0,5000]×[0,1])  */
  int32_t upper_bc;              /* PR_BC_*: the boundary target at S = L (reading Q3)            */
  int32_t n_linear;              /* linear layers ≥ 2                                             */
  const int32_t *dims;           /* [n_linear+1]: dims[0] = 2, hidden widths equal and in
                                    {8, 16, 20, 32, 50, 64}, dims[n_linear] = 1                   */
  int32_t activation;            /* PR_ACT_TANH / PR_ACT_RELU                                     */
  const float *const *W;         /* [n_linear] initial weights, row-major [out][in] (copied)      */
  const float *const *b;         /* [n_linear] initial biases (copied)                            */
  int32_t n_f, n_b, n_exp;       /* collocation counts ≥ 1 each (100000, 10000, 10000)     */
  const float *t_f, *S_f;        /* [n_f] interior points (t, S) (copied)                         */
  const float *t_b, *S_b;        /* [n_b] boundary points; S_b[i] ∈ {0, L} (copied)               */
  const float *S_exp;            /* [n_exp] expiry points, t = T (copied)                         */
  int32_t batches;               /* mini-batches per epoch, 1 ≤ batches ≤ min(n_f, n_b, n_exp)    */
  uint64_t shuffle_seed;
  double beta1, beta2, eps;      /* Adam: 0 ≤ β < 1, ε > 0 (the paper's defaults: .9, .999, 1e-8) */
  int32_t device;                /* CUDA device ordinal                                           */
  void *stream;                  /* cudaStream_t to issue on, or NULL → a trainer-owned stream    */
} pt_config;

/* Validates the config (PR_ERR_INVALID_ARGUMENT naming the field; PR_ERR_UNSUPPORTED for a
 * hidden width outside {8,16,20,32,50,64}, unequal widths, or a net whose weights and forward
 * stash exceed the shared memory of one CTA), copies weights and points to the
 * device, zeroes Adam's moments and the step counter. */
pr_status pinn_train_init(const pt_config *cfg, pt_trainer **out);

/* Runs `epochs` ≥ 1 epochs of Adam with learning rate lr > 0 (epochs × batches steps).
 * loss_hist (nullable, host): [epochs·batches][3] receives each step's batch (MSE_f, MSE_b,
 * MSE_exp) at the parameters before its update.  Returns when the work is done. */
pr_status pinn_train_epochs(pt_trainer *tr, int32_t epochs, double lr, double *loss_hist);

/* (MSE_f, MSE_b, MSE_exp) over the complete sets at the current parameters (Eqs. 12-14). */
pr_status pinn_train_loss(pt_trainer *tr, double out[3]);

/* Test hook: the gradient of MSE_total over the batch of step `step` ≥ 0 (its epoch's shuffle)
 * at the current parameters, without updating anything.  grad: host [param_count] in the packed
 * order (per layer W row-major, then b); loss (nullable): the batch's three terms. */
pr_status pinn_train_batch_gradient(pt_trainer *tr, int64_t step, float *grad, double loss[3]);

/* Number of trainable parameters Σ_l dims[l+1]·(dims[l] + 1). */
int64_t pinn_train_param_count(const pt_trainer *tr);
/* Steps taken so far (epochs × batches over all pinn_train_epochs calls). */
int64_t pinn_train_step_count(const pt_trainer *tr);

/* Current parameters: packed (host [param_count]) or per layer (W[l] [dims[l+1]·dims[l]],
 * b[l] [dims[l+1]], host). */
pr_status pinn_train_get_params(pt_trainer *tr, float *packed);
pr_status pinn_train_get_weights(pt_trainer *tr, float *const *W, float *const *b);

const char *pinn_train_last_error(const pt_trainer *tr);  /* never NULL (tr == NULL: last failed init) */
void pinn_train_free(pt_trainer *tr);                      /* NULL-safe */

#ifdef __cplusplus
}
#endif
#endif /* PINN_TRAIN_H */
