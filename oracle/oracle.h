/* oracle.h — TEST INFRASTRUCTURE ONLY (not product code).
 *
 * Plain, slow, serial CPU oracle of the Parareal + PINN method of
 * arXiv 2303.03848 ("Parareal with a physics-informed neural network as
 * coarse propagator", Ibrahim, Götschel, Ruprecht).  Every function follows
 * one passage of /root/reference/PAPER.md (cited as P:<line>) in the paper's
 * order and notation; where the paper is silent the reading is SURVEY.md §8(c)
 * Q<n>, listed in DESIGN.md "Readings".
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load this library.  It shares no code, header or constant with the CUDA
 * path (paper_2303_03848_b200/csrc); the CUDA path never loads it.
 *
 * All functions are instantiated in FP64 (prefix or64_) and, for the
 * stability gate of SURVEY.md §8(c), in FP32 (prefix or32_); the FP32 build
 * rounds every intermediate to float but takes and returns double arrays.
 * Return codes: 0 ok, 1 invalid argument, 3 non-positive pivot.
 */
#ifndef PARAREAL_ORACLE_H
#define PARAREAL_ORACLE_H
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int M, B;                 /* interior points, instances                   */
  const double *strike, *sigma, *rate, *L;  /* [B]                          */
  double T;                 /* expiry                                       */
  int upper_bc;             /* 0: V(L,tau)=L-K e^{-r tau}; 1: V(L,tau)=0    */
  int N, fine_steps;        /* slices; steps per slice                      */
  double fine_theta;        /* 1 implicit Euler, 0.5 Crank-Nicolson         */
  int coarse, coarse_steps; /* 0 PINN, 1 implicit Euler                     */
  int max_iter;
  double tol;
} or_problem;

typedef struct {
  int n_linear;              /* number of affine layers                      */
  const int *dims;           /* [n_linear+1]; dims[0] in {2,4}; dims[n]=1    */
  const double *const *W;    /* W[l] row-major [dims[l+1]][dims[l]]          */
  const double *const *b;    /* b[l] [dims[l+1]]                             */
  int activation;            /* 0 tanh, 1 relu                               */
  const double *in_scale;    /* [dims[0]] or NULL                            */
  double out_scale;
} or_net;

/* closed-form European call (standard Black-Scholes formula) */
double or_bs_call(double S, double K, double r, double sigma, double tau);

/* tau-form semi-discrete operator rows j=1..M (P:155-158 reversed in time) */
void or64_operator(int M, double sigma, double r, double *lower, double *diag, double *upper);

/* plain Thomas algorithm: sub[i] (i>=1) x[i-1] + diag[i] x[i] + sup[i] x[i+1] (i<=n-2) = rhs[i] */
int or64_thomas(int n, const double *sub, const double *diag, const double *sup,
                const double *rhs, double *x);
int or32_thomas(int n, const double *sub, const double *diag, const double *sup,
                const double *rhs, double *x);

/* one theta-step of instance b from tau0 to tau0+dtau, in place on w[M] */
int or64_theta_step(const or_problem *p, int b, double theta, double tau0, double dtau, double *w);

/* `steps` theta-steps across slice n (tau in [n dT, (n+1) dT]) of all instances, U[B][M] in place */
int or64_propagate(const or_problem *p, int n, double theta, int steps, double *U);
int or32_propagate(const or_problem *p, int n, double theta, int steps, double *U);

/* scalar MLP: y = W_L act(... act(W_1 x + b_1) ...) + b_L */
void or64_mlp(const or_net *net, const double *x, double *y);
void or32_mlp(const or_net *net, const double *x, double *y);

/* PINN coarse propagator over slice n for all instances: out[B][M] = G(U[B][M]) */
int or64_pinn_G(const or_problem *p, const or_net *net, int n, const double *U, double *out);
int or32_pinn_G(const or_problem *p, const or_net *net, int n, const double *U, double *out);

/* U_0 = payoff (Eq. 2) for all instances -> U0[B][M] */
void or64_payoff(const or_problem *p, double *U0);

/* serial fine (Eq. 6): U[N+1][B][M], U[0] = V_T (or payoff if V_T==NULL) */
int or64_serial_fine(const or_problem *p, const double *V_T, double *U);
int or32_serial_fine(const or_problem *p, const double *V_T, double *U);

/* Parareal (Eq. 7, schedule Q12, stop rule Q13).
 *   U     [N+1][B][M]  final iterate U^K
 *   delta [max_iter]   delta^k, k=1..K (entries beyond K untouched)
 *   hist  NULL or [max_iter+1][N+1][B][M]: U^k for k=0..K
 *   iterations -> K */
int or64_parareal(const or_problem *p, const or_net *net, const double *V_T,
                  double *U, double *delta, int *iterations, double *hist);
int or32_parareal(const or_problem *p, const or_net *net, const double *V_T,
                  double *U, double *delta, int *iterations, double *hist);
/* or64_parareal with the fine sweep's slices on nthreads std::threads (bitwise the serial result) */
int or64_parareal_mt(const or_problem *p, const or_net *net, const double *V_T, double *U,
                     double *delta, int *iterations, double *hist, int nthreads);

#ifdef __cplusplus
}
#endif
#endif
