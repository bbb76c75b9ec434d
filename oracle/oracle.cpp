// oracle.cpp — TEST INFRASTRUCTURE ONLY (see oracle.h).
//
// A plain serial CPU implementation of what the hot path computes, written
// from /root/reference/PAPER.md (P:<line>).  No blocking, no fusion, no
// precomputed factorisations: every implicit step rebuilds its matrix and
// runs a textbook Thomas elimination.  Template parameter R is the working
// precision (double for the oracle proper; float only for the stability gate).
//
// Parity status: every function is pinned by a
// `-m "not gpu"` test against the paper / closed forms / brute force, except
// the convergence speed of Parareal with a *trained* PINN (parity unpinned:
// needs the paper's weights).

#include "oracle.h"

#include <cmath>
#include <cstring>
#include <thread>
#include <vector>

namespace {

// ---------------------------------------------------------------------------
// P:86-90 Eq.(1) with P:149-158: second-order centred differences on the
// equidistant mesh S_j = j dS, dS = L/(M+1) (reading Q4: M interior nodes).
// In reversed time tau = T - t the semi-discrete system is
//   dV_j/dtau = (a_j - b_j) V_{j-1} - (2 a_j + r) V_j + (a_j + b_j) V_{j+1},
//   a_j = sigma^2 S_j^2 / (2 dS^2) = sigma^2 j^2 / 2,   b_j = r S_j / (2 dS) = r j / 2.
// (P:156 has V' = -[...] in t; the sign flips with tau.)
template <class R>
void op_rows(int M, double sigma, double r, R *lo, R *di, R *up) {
  for (int i = 0; i < M; ++i) {
    const double j = i + 1;
    const double a = 0.5 * sigma * sigma * j * j;
    const double b = 0.5 * r * j;
    lo[i] = (R)(a - b);
    di[i] = (R)(-(2.0 * a + r));
    up[i] = (R)(a + b);
  }
}

// Upper boundary value g(tau) = V(L, tau).  Reading Q3: the asymptotic call
// value L - K e^{-r tau} ("same value as the underlying" less the
// discounted strike) by default; upper_bc=1 is the paper-literal V_N = 0.
double g_upper(const or_problem *p, int b, double tau) {
  if (p->upper_bc == 1) return 0.0;
  return p->L[b] - p->strike[b] * std::exp(-p->rate[b] * tau);
}

// Textbook Thomas algorithm (no pivoting).  Positive pivots are required
// (true for the strictly diagonally dominant, positive-diagonal systems here).
template <class R>
int thomas(int n, const R *sub, const R *diag, const R *sup, const R *rhs, R *x) {
  std::vector<R> cp(n), dp(n);
  R piv = diag[0];
  if (!(piv > (R)0)) return 3;
  cp[0] = (n > 1) ? sup[0] / piv : (R)0;
  dp[0] = rhs[0] / piv;
  for (int i = 1; i < n; ++i) {
    piv = diag[i] - sub[i] * cp[i - 1];
    if (!(piv > (R)0)) return 3;
    cp[i] = (i < n - 1) ? sup[i] / piv : (R)0;
    dp[i] = (rhs[i] - sub[i] * dp[i - 1]) / piv;
  }
  x[n - 1] = dp[n - 1];
  for (int i = n - 2; i >= 0; --i) x[i] = dp[i] - cp[i] * x[i + 1];
  return 0;
}

// One theta-step (implicit Euler theta=1, Crank-Nicolson theta=1/2):
//   (I - theta dtau A) w+ = (I + (1-theta) dtau A) w + dtau (a_M+b_M) [theta g(tau+) + (1-theta) g(tau)] e_M
// The lower boundary V_0 = 0 (Eq. 3) contributes nothing.
template <class R>
int theta_step(const or_problem *p, int b, double theta, double tau0, double dtau, R *w) {
  const int M = p->M;
  std::vector<R> lo(M), di(M), up(M), sub(M), dg(M), sup(M), rhs(M);
  op_rows<R>(M, p->sigma[b], p->rate[b], lo.data(), di.data(), up.data());
  const R dt = (R)dtau, th = (R)theta, one = (R)1;
  const R g0 = (R)g_upper(p, b, tau0), g1 = (R)g_upper(p, b, tau0 + dtau);
  for (int i = 0; i < M; ++i) {
    // explicit part (I + (1-theta) dtau A) w, with boundary values V_0 = 0, V_{M+1} = g(tau)
    const R wl = (i > 0) ? w[i - 1] : (R)0;
    const R wr = (i < M - 1) ? w[i + 1] : g0;
    const R Aw = lo[i] * wl + di[i] * w[i] + up[i] * wr;
    rhs[i] = w[i] + (one - th) * dt * Aw;
    // implicit part
    sub[i] = -th * dt * lo[i];
    dg[i] = one - th * dt * di[i];
    sup[i] = -th * dt * up[i];
  }
  rhs[M - 1] += th * dt * up[M - 1] * g1;  // boundary value at the new time level
  std::vector<R> x(M);
  const int st = thomas<R>(M, sub.data(), dg.data(), sup.data(), rhs.data(), x.data());
  if (st) return st;
  for (int i = 0; i < M; ++i) w[i] = x[i];
  return 0;
}

// Propagate every instance across time slice n: tau_m = n dT + m dtau.
template <class R>
int propagate(const or_problem *p, int n, double theta, int steps, R *U) {
  const double dT = p->T / p->N;
  const double dtau = dT / steps;
  for (int b = 0; b < p->B; ++b) {
    R *w = U + (size_t)b * p->M;
    for (int m = 0; m < steps; ++m) {
      const int st = theta_step<R>(p, b, theta, n * dT + m * dtau, dtau, w);
      if (st) return st;
    }
  }
  return 0;
}

// Fully connected network, hidden activation then linear output.
template <class R>
void mlp(const or_net *net, const R *x, R *y) {
  int width = net->dims[0];
  std::vector<R> h(x, x + width), z;
  for (int l = 0; l < net->n_linear; ++l) {
    const int out = net->dims[l + 1], in = net->dims[l];
    z.assign(out, (R)0);
    for (int o = 0; o < out; ++o) {
      R s = (R)net->b[l][o];
      for (int i = 0; i < in; ++i) s += (R)net->W[l][(size_t)o * in + i] * h[i];
      z[o] = s;
    }
    if (l < net->n_linear - 1) {
      for (int o = 0; o < out; ++o)
        z[o] = (net->activation == 1) ? (z[o] > (R)0 ? z[o] : (R)0) : std::tanh(z[o]);
    }
    h.swap(z);
    width = out;
  }
  y[0] = h[0];
}

// PINN coarse propagator (Fig. 2 caption P:217): inputs (t_start, t_end,
// V at t_start, S) -> V~ at t_end.  Reading Q6-Q8: physical times
// t_from = T - n dT, t_to = T - (n+1) dT normalised by T; V, S normalised by
// the instance's L; output scaled by L.  2-input mode: (t_to/T, S/L).
template <class R>
int pinn_G(const or_problem *p, const or_net *net, int n, const R *U, R *out) {
  const int d0 = net->dims[0];
  if ((d0 != 2 && d0 != 4) || net->dims[net->n_linear] != 1) return 1;
  const double dT = p->T / p->N;
  const double t_from = p->T - n * dT, t_to = p->T - (n + 1) * dT;
  for (int b = 0; b < p->B; ++b) {
    const double Lb = p->L[b], dS = Lb / (p->M + 1);
    for (int i = 0; i < p->M; ++i) {
      const double S = (i + 1) * dS;
      R x[4];
      if (d0 == 4) {
        x[0] = (R)(t_from / p->T);
        x[1] = (R)(t_to / p->T);
        x[2] = U[(size_t)b * p->M + i] / (R)Lb;
        x[3] = (R)(S / Lb);
      } else {
        x[0] = (R)(t_to / p->T);
        x[1] = (R)(S / Lb);
      }
      for (int c = 0; c < d0; ++c)
        if (net->in_scale) x[c] *= (R)net->in_scale[c];
      R y;
      mlp<R>(net, x, &y);
      out[(size_t)b * p->M + i] = (R)Lb * (R)net->out_scale * y;
    }
  }
  return 0;
}

// Expiry condition (Eq. 2): V(T,S) = max(S - K, 0).
template <class R>
void payoff(const or_problem *p, R *U0) {
  for (int b = 0; b < p->B; ++b) {
    const double dS = p->L[b] / (p->M + 1);
    for (int i = 0; i < p->M; ++i) {
      const double S = (i + 1) * dS;
      U0[(size_t)b * p->M + i] = (R)(S > p->strike[b] ? S - p->strike[b] : 0.0);
    }
  }
}

int check(const or_problem *p) {
  if (!p || p->M < 1 || p->B < 1 || p->N < 1 || p->fine_steps < 1) return 1;
  if (p->coarse == 1 && p->coarse_steps < 1) return 1;
  if (!(p->T > 0)) return 1;
  for (int b = 0; b < p->B; ++b)
    if (!(p->sigma[b] > 0) || !(p->rate[b] >= 0) || !(p->strike[b] >= 0) || !(p->L[b] > p->strike[b]))
      return 1;
  return 0;
}

// Parareal-only parameters: 1 <= max_iter <= N, tol >= 0.
int check_parareal(const or_problem *p) {
  if (check(p)) return 1;
  if (p->max_iter < 1 || p->max_iter > p->N || !(p->tol >= 0)) return 1;
  return 0;
}

template <class R>
int F(const or_problem *p, int n, R *U) {  // fine propagator over slice n
  return propagate<R>(p, n, p->fine_theta, p->fine_steps, U);
}

template <class R>
int G(const or_problem *p, const or_net *net, int n, const R *U, R *out) {  // coarse propagator
  const size_t sz = (size_t)p->B * p->M;
  if (p->coarse == 0) return pinn_G<R>(p, net, n, U, out);
  // numerical coarse G: implicit Euler with coarse_steps steps per slice (Q2)
  std::memcpy(out, U, sz * sizeof(R));
  return propagate<R>(p, n, 1.0, p->coarse_steps, out);
}

template <class R>
void load_initial(const or_problem *p, const double *V_T, R *U0) {
  const size_t sz = (size_t)p->B * p->M;
  if (V_T)
    for (size_t i = 0; i < sz; ++i) U0[i] = (R)V_T[i];
  else
    payoff<R>(p, U0);
}

// Serial fine, Eq. (6): V_{n+1} = F(V_n), n = 0..N-1.
template <class R>
int serial_fine(const or_problem *p, const double *V_T, double *Uout) {
  if (check(p)) return 1;
  const size_t sz = (size_t)p->B * p->M;
  std::vector<R> U((size_t)(p->N + 1) * sz);
  load_initial<R>(p, V_T, U.data());
  for (int n = 0; n < p->N; ++n) {
    std::memcpy(&U[(n + 1) * sz], &U[n * sz], sz * sizeof(R));
    const int st = F<R>(p, n, &U[(n + 1) * sz]);
    if (st) return st;
  }
  for (size_t i = 0; i < U.size(); ++i) Uout[i] = (double)U[i];
  return 0;
}

// Parareal, Eq. (7), with the schedule of reading Q12:
//   k = 0:  U_0 = V_T;  G^_n = G(U_n), U_{n+1} = G^_n          (initial coarse sweep)
//   k >= 1: F^_n = F(U^{k-1}_n) for n = k-1..N-1                  (parallel in the paper)
//           U^k_n = U^{k-1}_n for n <= k-1, U^k_k = F^_{k-1}       (frozen prefix, copy)
//           for n = k..N-1: g = G(U^k_n); U^k_{n+1} = g + (F^_n - G^_n); G^_n = g
//           delta^k = max_{n=k..N} max_b ||U^k_n - U^{k-1}_n|| / ||U^k_n||  (Q13)
//           stop if delta^k < tol or k = max_iter (K = k counts fine sweeps, Q14)
// nthreads > 1: the fine sweep's slices (independent) run on std::threads, slice n on
// thread n mod nthreads -- the CPU analog of the paper's one-process-per-slice fine propagation.
// Every slice is computed by the same code on its own data, so results are bitwise the serial ones.
template <class R>
int parareal(const or_problem *p, const or_net *net, const double *V_T, double *Uout,
             double *delta, int *iterations, double *hist, int nthreads = 1) {
  if (check_parareal(p)) return 1;
  if (p->coarse == 0 && !net) return 1;
  const int N = p->N, M = p->M, B = p->B;
  const size_t sz = (size_t)B * M, tot = (size_t)(N + 1) * sz;
  std::vector<R> U(tot), Uold(tot), Gh((size_t)N * sz), Fh((size_t)N * sz), g(sz);
  load_initial<R>(p, V_T, U.data());
  for (int n = 0; n < N; ++n) {
    int st = G<R>(p, net, n, &U[n * sz], &Gh[n * sz]);
    if (st) return st;
    std::memcpy(&U[(n + 1) * sz], &Gh[n * sz], sz * sizeof(R));
  }
  if (hist)
    for (size_t i = 0; i < tot; ++i) hist[i] = (double)U[i];
  int K = 0;
  for (int k = 1; k <= p->max_iter; ++k) {
    Uold = U;
    if (nthreads <= 1) {
      for (int n = k - 1; n < N; ++n) {
        std::memcpy(&Fh[n * sz], &Uold[n * sz], sz * sizeof(R));
        const int st = F<R>(p, n, &Fh[n * sz]);
        if (st) return st;
      }
    } else {
      std::vector<int> sts(nthreads, 0);
      std::vector<std::thread> pool;
      for (int t = 0; t < nthreads; ++t)
        pool.emplace_back([&, t]() {
          for (int n = k - 1 + t; n < N; n += nthreads) {
            std::memcpy(&Fh[n * sz], &Uold[n * sz], sz * sizeof(R));
            const int st = F<R>(p, n, &Fh[n * sz]);
            if (st) { sts[t] = st; return; }
          }
        });
      for (auto &th : pool) th.join();
      for (int st : sts)
        if (st) return st;
    }
    std::memcpy(&U[k * sz], &Fh[(k - 1) * sz], sz * sizeof(R));
    for (int n = k; n < N; ++n) {
      const int st = G<R>(p, net, n, &U[n * sz], g.data());
      if (st) return st;
      for (size_t i = 0; i < sz; ++i) U[(n + 1) * sz + i] = g[i] + (Fh[n * sz + i] - Gh[n * sz + i]);
      std::memcpy(&Gh[n * sz], g.data(), sz * sizeof(R));
    }
    double dk = 0.0;
    for (int n = k; n <= N; ++n)
      for (int b = 0; b < B; ++b) {
        double num = 0.0, den = 0.0;
        for (int i = 0; i < M; ++i) {
          const double u = (double)U[n * sz + (size_t)b * M + i];
          const double d = u - (double)Uold[n * sz + (size_t)b * M + i];
          num += d * d;
          den += u * u;
        }
        const double rel = (den > 0.0) ? std::sqrt(num) / std::sqrt(den) : std::sqrt(num);
        if (rel > dk) dk = rel;
      }
    delta[k - 1] = dk;
    if (hist)
      for (size_t i = 0; i < tot; ++i) hist[(size_t)k * tot + i] = (double)U[i];
    K = k;
    if (dk < p->tol) break;
  }
  *iterations = K;
  for (size_t i = 0; i < tot; ++i) Uout[i] = (double)U[i];
  return 0;
}

template <class R>
int propagate_io(const or_problem *p, int n, double theta, int steps, double *U) {
  if (check(p) || steps < 1 || n < 0 || n >= p->N) return 1;
  const size_t sz = (size_t)p->B * p->M;
  std::vector<R> w(U, U + sz);
  const int st = propagate<R>(p, n, theta, steps, w.data());
  for (size_t i = 0; i < sz; ++i) U[i] = (double)w[i];
  return st;
}

template <class R>
int pinn_io(const or_problem *p, const or_net *net, int n, const double *U, double *out) {
  const size_t sz = (size_t)p->B * p->M;
  std::vector<R> u(U, U + sz), o(sz);
  const int st = pinn_G<R>(p, net, n, u.data(), o.data());
  for (size_t i = 0; i < sz; ++i) out[i] = (double)o[i];
  return st;
}

template <class R>
int thomas_io(int n, const double *sub, const double *diag, const double *sup, const double *rhs, double *x) {
  if (n < 1) return 1;
  std::vector<R> a(sub, sub + n), d(diag, diag + n), c(sup, sup + n), r(rhs, rhs + n), y(n);
  const int st = thomas<R>(n, a.data(), d.data(), c.data(), r.data(), y.data());
  for (int i = 0; i < n; ++i) x[i] = (double)y[i];
  return st;
}

template <class R>
void mlp_io(const or_net *net, const double *x, double *y) {
  std::vector<R> xi(x, x + net->dims[0]);
  R yo;
  mlp<R>(net, xi.data(), &yo);
  *y = (double)yo;
}

}  // namespace

extern "C" {

// Closed-form European call ("Closed form solutions exist"; Black-Scholes 1973):
//   C = S Phi(d1) - K e^{-r tau} Phi(d2),  Phi(x) = erfc(-x/sqrt 2)/2.
double or_bs_call(double S, double K, double r, double sigma, double tau) {
  if (S <= 0.0) return 0.0;
  if (tau <= 0.0) return S > K ? S - K : 0.0;
  if (K <= 0.0) return S;
  const double sq = sigma * std::sqrt(tau);
  const double d1 = (std::log(S / K) + (r + 0.5 * sigma * sigma) * tau) / sq;
  const double d2 = d1 - sq;
  const double Phi1 = 0.5 * std::erfc(-d1 / std::sqrt(2.0));
  const double Phi2 = 0.5 * std::erfc(-d2 / std::sqrt(2.0));
  return S * Phi1 - K * std::exp(-r * tau) * Phi2;
}

void or64_operator(int M, double sigma, double r, double *lower, double *diag, double *upper) {
  op_rows<double>(M, sigma, r, lower, diag, upper);
}
int or64_thomas(int n, const double *a, const double *d, const double *c, const double *r, double *x) {
  return thomas_io<double>(n, a, d, c, r, x);
}
int or32_thomas(int n, const double *a, const double *d, const double *c, const double *r, double *x) {
  return thomas_io<float>(n, a, d, c, r, x);
}
int or64_theta_step(const or_problem *p, int b, double theta, double tau0, double dtau, double *w) {
  if (check(p) || b < 0 || b >= p->B) return 1;
  return theta_step<double>(p, b, theta, tau0, dtau, w);
}
int or64_propagate(const or_problem *p, int n, double theta, int steps, double *U) {
  return propagate_io<double>(p, n, theta, steps, U);
}
int or32_propagate(const or_problem *p, int n, double theta, int steps, double *U) {
  return propagate_io<float>(p, n, theta, steps, U);
}
void or64_mlp(const or_net *net, const double *x, double *y) { mlp_io<double>(net, x, y); }
void or32_mlp(const or_net *net, const double *x, double *y) { mlp_io<float>(net, x, y); }
int or64_pinn_G(const or_problem *p, const or_net *net, int n, const double *U, double *out) {
  if (check(p) || !net || n < 0 || n >= p->N) return 1;
  return pinn_io<double>(p, net, n, U, out);
}
int or32_pinn_G(const or_problem *p, const or_net *net, int n, const double *U, double *out) {
  if (check(p) || !net || n < 0 || n >= p->N) return 1;
  return pinn_io<float>(p, net, n, U, out);
}
void or64_payoff(const or_problem *p, double *U0) { payoff<double>(p, U0); }
int or64_serial_fine(const or_problem *p, const double *V_T, double *U) {
  return serial_fine<double>(p, V_T, U);
}
int or32_serial_fine(const or_problem *p, const double *V_T, double *U) {
  return serial_fine<float>(p, V_T, U);
}
int or64_parareal(const or_problem *p, const or_net *net, const double *V_T, double *U,
                  double *delta, int *iterations, double *hist) {
  return parareal<double>(p, net, V_T, U, delta, iterations, hist);
}
int or32_parareal(const or_problem *p, const or_net *net, const double *V_T, double *U,
                  double *delta, int *iterations, double *hist) {
  return parareal<float>(p, net, V_T, U, delta, iterations, hist);
}
int or64_parareal_mt(const or_problem *p, const or_net *net, const double *V_T, double *U,
                     double *delta, int *iterations, double *hist, int nthreads) {
  return parareal<double>(p, net, V_T, U, delta, iterations, hist, nthreads);
}

}  // extern "C"
