"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test states what it pins.  None of them re-types the oracle's own
formula: the references are printed values (tests/golden, cited), closed
forms, library routines doing a different computation (LAPACK banded solve,
dense solve, matrix exponential, adaptive quadrature), exact discrete
solutions, brute force on tiny inputs and invariants of the method.
"""
import math

import numpy as np
import pytest
import scipy.integrate
import scipy.linalg
import scipy.stats

import oracle
from paper_2303_03848_b200 import synth


# ---------------------------------------------------------------- closed form

def test_closed_form_golden(golden):
    for c in golden("closed_form.json")["cases"]:
        got = oracle.bs_call(c["S"], c["K"], c["r"], c["sigma"], c["tau"])
        assert got == pytest.approx(c["C"], rel=1e-12, abs=1e-12), c["cite"]


def _bs_quadrature(S, K, r, sigma, tau):
    """Brute force: discounted risk-neutral expectation under GBM, by quadrature."""
    mu = math.log(S) + (r - 0.5 * sigma * sigma) * tau
    sd = sigma * math.sqrt(tau)
    f = lambda z: max(math.exp(mu + sd * z) - K, 0.0) * math.exp(-0.5 * z * z) / math.sqrt(2 * math.pi)
    z0 = (math.log(K) - mu) / sd
    val, _ = scipy.integrate.quad(f, z0, z0 + 40.0, epsabs=1e-13, epsrel=1e-12, limit=200)
    return math.exp(-r * tau) * val


@pytest.mark.parametrize("S,K,r,sigma,tau", [(1.0, 1.0, .05, .2, 1.0), (0.7, 1.0, .05, .1, .5),
                                             (3.0, 1.0, .0, .5, 1.0), (2500., 2500., .03, .4, 1.),
                                             (1.3, 1.1, .08, .3, .25)])
def test_closed_form_vs_quadrature(S, K, r, sigma, tau):
    assert oracle.bs_call(S, K, r, sigma, tau) == pytest.approx(_bs_quadrature(S, K, r, sigma, tau),
                                                                rel=1e-9, abs=1e-12)


def test_closed_form_bounds_and_monotone():
    """No-arbitrage bounds max(S-Ke^{-r tau},0) <= C <= S and monotonicity in S."""
    S = np.linspace(0.0, 4.0, 401)
    for tau in (0.1, 0.5, 1.0):
        C = np.array([oracle.bs_call(s, 1.0, .05, .2, tau) for s in S])
        lo = np.maximum(S - math.exp(-.05 * tau), 0.0)
        assert np.all(C >= lo - 1e-14) and np.all(C <= S + 1e-14)
        assert np.all(np.diff(C) >= -1e-14)


# ---------------------------------------------------------------- operator

def test_operator_rows_golden(golden):
    g = golden("spec_examples.json")["operator_rows"]
    lo, di, up = oracle.operator(g["M"], g["sigma"], g["r"])
    assert lo.tolist() == g["lower"] and di.tolist() == g["diag"] and up.tolist() == g["upper"], g["cite"]


def test_operator_annihilates_linear_function():
    """V = S solves Eq. (1) (V_t=0, V_SS=0: rS*1 - rS = 0); centred differences are exact on
    linear functions, so A S + (a_M+b_M) L e_M = 0 with S_j = j dS (exact discrete solution)."""
    M, L = 37, 4.0
    for sigma, r in [(0.2, 0.05), (0.5, 0.0), (0.1, 0.09)]:
        lo, di, up = oracle.operator(M, sigma, r)
        dS = L / (M + 1)
        S = dS * np.arange(1, M + 1)
        AS = di * S
        AS[1:] += lo[1:] * S[:-1]
        AS[:-1] += up[:-1] * S[1:]
        AS[-1] += up[-1] * L
        AS[0] += lo[0] * 0.0
        assert np.max(np.abs(AS)) <= 1e-9 * np.max(np.abs(di * S))


# ---------------------------------------------------------------- Thomas

def test_thomas_golden(golden):
    g = golden("spec_examples.json")["thomas"]
    assert np.allclose(oracle.thomas(g["sub"], g["diag"], g["sup"], g["rhs"]), g["x"], rtol=0, atol=1e-15)


def test_thomas_identity():
    rhs = np.arange(1.0, 8.0)
    assert np.array_equal(oracle.thomas(np.zeros(7), np.ones(7), np.zeros(7), rhs), rhs)


@pytest.mark.parametrize("n", [1, 2, 3, 7, 20, 50])
def test_thomas_vs_lapack_and_dense(n):
    rng = np.random.default_rng(n)
    for _ in range(5):
        sub, sup = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        sub[0], sup[-1] = 0.0, 0.0
        diag = np.abs(sub) + np.abs(sup) + rng.uniform(0.1, 2.0, n)
        rhs = rng.normal(size=n)
        x = oracle.thomas(sub, diag, sup, rhs)
        ab = np.zeros((3, n))
        ab[0, 1:], ab[1], ab[2, :-1] = sup[:-1], diag, sub[1:]
        xl = scipy.linalg.solve_banded((1, 1), ab, rhs)          # LAPACK gbsv
        A = np.diag(diag) + np.diag(sub[1:], -1) + np.diag(sup[:-1], 1)
        xd = np.linalg.solve(A, rhs)                             # dense LU
        assert np.allclose(x, xl, rtol=1e-10, atol=1e-12)
        assert np.allclose(x, xd, rtol=1e-10, atol=1e-12)


def test_thomas_rejects_nonpositive_pivot():
    with pytest.raises(ArithmeticError):
        oracle.thomas([0, 1.0], [0.0, 1.0], [1.0, 0], [1.0, 1.0])


# ---------------------------------------------------------------- theta-steps

def _one_node(**kw):
    """One interior node, sigma=1, r=0, zero upper boundary value: w' = -w."""
    kw.setdefault("max_iter", 1)
    return synth.single(1, 1, K=0.0, r=0.0, sigma=1.0, L=2.0, upper_bc=synth.BC_ZERO, **kw)


def test_ie_cn_one_node_golden(golden):
    g = golden("spec_examples.json")
    p = _one_node()
    assert oracle.theta_step(p, 0, 1.0, 0.0, 0.1, [1.0])[0] == pytest.approx(g["ie_step"]["value"], rel=1e-15)
    assert oracle.theta_step(p, 0, 0.5, 0.0, 0.1, [1.0])[0] == pytest.approx(g["cn_step"]["value"], rel=1e-15)
    p1 = _one_node(fine_steps=10)
    p1 = p1.replace(T=1.0)
    w = oracle.propagate(p1, 0, [[1.0]], theta=1.0, steps=10)
    assert w[0, 0] == pytest.approx(g["ie_10_steps"]["value"], rel=1e-14)


def test_terminal_state_golden(golden):
    g = golden("spec_examples.json")["terminal_state"]
    p = synth.single(g["M"], 1, K=g["K"], L=g["L"])
    assert oracle.payoff(p)[0].tolist() == g["U0"], g["cite"]


def _augmented(p, b=0):
    """Semi-discrete system plus the boundary value as extra states, written from the PDE:
    d/dtau [V, g, 1] with g(tau) = L - K e^{-r tau}  =>  g' = r (L - g)."""
    M = p.M
    s, r, L = p.sigma[b], p.rate[b], p.L[b]
    j = np.arange(1, M + 1, dtype=float)
    a, bb = 0.5 * s * s * j * j, 0.5 * r * j
    A = np.zeros((M + 2, M + 2))
    A[np.arange(M), np.arange(M)] = -(2 * a + r)
    A[np.arange(1, M), np.arange(M - 1)] = (a - bb)[1:]
    A[np.arange(M - 1), np.arange(1, M)] = (a + bb)[:-1]
    A[M - 1, M] = a[-1] + bb[-1]
    A[M, M], A[M, M + 1] = -r, r * L
    return A


def test_semidiscrete_limit_and_first_order():
    """n_f -> inf: implicit Euler converges to expm(tau A) (library matrix exponential) with order 1
    (SPEC.md:158); Crank-Nicolson with order 2."""
    p = synth.single(24, 1, K=1.0, r=0.05, sigma=0.3, T=0.5)
    U0 = oracle.payoff(p)
    A = _augmented(p)
    z0 = np.concatenate([U0[0], [p.L[0] - p.strike[0], 1.0]])
    exact = (scipy.linalg.expm(p.T * A) @ z0)[:p.M]
    errs = {1.0: [], 0.5: []}
    for steps in (50, 100, 200, 400):
        for th in errs:
            w = oracle.propagate(p, 0, U0, theta=th, steps=steps)
            errs[th].append(np.linalg.norm(w[0] - exact) / np.linalg.norm(exact))
    ie = np.log2(np.array(errs[1.0][:-1]) / np.array(errs[1.0][1:]))
    cn = np.log2(np.array(errs[0.5][:-1]) / np.array(errs[0.5][1:]))
    assert np.all(np.abs(ie - 1.0) < 0.1), ie
    assert np.all(np.abs(cn - 2.0) < 0.2), cn
    assert errs[1.0][-1] < 1e-4


def test_ie_temporal_order_c1():
    """Order 1.0 +- 0.2 on the C1 grid against a 20000-step reference."""
    p = synth.config("C1").replace(N=1)
    U0 = oracle.payoff(p)
    ref = oracle.propagate(p, 0, U0, 1.0, 20000)
    e = [np.linalg.norm(oracle.propagate(p, 0, U0, 1.0, s) - ref) for s in (100, 200, 400, 800)]
    order = np.log2(np.array(e[:-1]) / np.array(e[1:]))
    assert np.all(np.abs(order - 1.0) < 0.2), order


def test_linear_function_is_fixed_point():
    """Strike K=0: U_0 = S_j, g = L, and V = S is an exact solution of both the PDE and the
    discrete scheme; fine and numerical coarse keep it to rounding."""
    for M in (64, 1024):
        p = synth.single(M, 4, K=0.0, L=4.0, fine_steps=100)
        U = oracle.serial_fine(p)
        S = 4.0 / (M + 1) * np.arange(1, M + 1)
        assert np.max(np.abs(U[:, 0, :] - S) / S) < 1e-11


def test_fine_vs_closed_form():
    """The serial fine solution approaches the closed form (error 'around 1e-3');
    error shrinks under joint refinement in S and tau."""
    errs = []
    for M, nf in ((64, 100), (128, 400), (256, 1600)):
        p = synth.single(M, 4, fine_steps=nf // 4)
        U = oracle.serial_fine(p)[-1, 0]
        S = 4.0 / (M + 1) * np.arange(1, M + 1)
        ex = np.array([oracle.bs_call(s, 1.0, .05, .2, 1.0) for s in S])
        errs.append(np.linalg.norm(U - ex) / np.linalg.norm(ex))
    assert errs[0] < 1e-3
    assert errs[0] > errs[1] > errs[2]
    assert errs[0] / errs[2] > 8  # second order in S (dominant), first in tau


def test_paper_domain_error_with_asymptotic_bc():
    """Paper domain (L=5000) with K=2500, r=.03, sigma=.4 (SPEC defaults): the asymptotic
    upper BC (reading Q3) gives an error of order 1e-3 as reported; the literal V_N=0
     does not (it is O(1), which is why Q3 reads it the other way)."""
    p = synth.single(499, 1, K=2500.0, L=5000.0, r=0.03, sigma=0.4, fine_steps=200)
    S = 5000.0 / 500 * np.arange(1, 500)
    ex = np.array([oracle.bs_call(s, 2500.0, .03, .4, 1.0) for s in S])
    e_asym = np.linalg.norm(oracle.serial_fine(p)[-1, 0] - ex) / np.linalg.norm(ex)
    e_zero = np.linalg.norm(oracle.serial_fine(p.replace(upper_bc=synth.BC_ZERO))[-1, 0] - ex) / np.linalg.norm(ex)
    assert e_asym < 1e-2
    assert e_zero > 0.3


def test_homogeneity_in_strike():
    """With L = 4K the problem is homogeneous of degree 1 in K: U(K) = K U(1) (scale invariance
    of Eq. 1-4); holds to rounding for fine, numerical G and Parareal."""
    base = synth.single(64, 4, K=1.0, coarse=synth.COARSE_IMPLICIT_EULER, max_iter=2)
    for K in (0.8, 1.2, 2.5):
        pk = synth.single(64, 4, K=K, coarse=synth.COARSE_IMPLICIT_EULER, max_iter=2)
        assert np.allclose(oracle.serial_fine(pk), K * oracle.serial_fine(base), rtol=1e-12, atol=1e-14)
        assert np.allclose(oracle.parareal(pk)[0], K * oracle.parareal(base)[0], rtol=1e-12, atol=1e-14)


def test_positivity():
    """Discrete maximum principle: for j >= r/sigma^2 the IE step is an M-matrix solve, so a
    nonnegative state stays nonnegative (no off-diagonal sign flip at C1: r/sigma^2 = 1.25)."""
    p = synth.config("C1")
    U = oracle.serial_fine(p)
    assert U.min() >= 0.0


# ---------------------------------------------------------------- network

def _numpy_mlp(net, x):
    """Independent matrix-form evaluation (SPEC.md:227 duplicate-evaluation oracle)."""
    h = np.asarray(x, dtype=np.float64)
    for l, (W, b) in enumerate(zip(net.W, net.b)):
        h = W.astype(np.float64) @ h + b.astype(np.float64)
        if l < len(net.W) - 1:
            h = np.tanh(h) if net.activation == synth.ACT_TANH else np.maximum(h, 0.0)
    return float(h[0])


@pytest.mark.parametrize("dims,act", [(synth.PINN_3x20, synth.ACT_TANH), (synth.PINN_PAPER, synth.ACT_RELU),
                                      ([4, 64, 64, 64, 64, 1], synth.ACT_TANH), ([2, 8, 1], synth.ACT_TANH)])
def test_mlp_vs_matrix_form(dims, act):
    net = synth.kaiming_net(dims, seed=3, activation=act)
    rng = np.random.default_rng(0)
    for _ in range(20):
        x = rng.uniform(-1, 1, dims[0])
        assert oracle.mlp(net, x) == pytest.approx(_numpy_mlp(net, x), rel=1e-12, abs=1e-13)


def test_mlp_special_cases():
    """zero last layer -> bias only; no hidden layer -> affine closed form."""
    net = synth.kaiming_net(synth.PINN_3x20, seed=1)
    net.W[-1][:] = 0.0
    net.b[-1][:] = np.float32(0.375)
    assert oracle.mlp(net, [0.1, 0.2, 0.3, 0.4]) == 0.375
    aff = synth.Net([4, 1], [np.array([[0.5, -1.0, 2.0, 0.25]], np.float32)], [np.array([0.125], np.float32)])
    x = np.array([0.2, 0.4, -0.6, 0.8])
    assert oracle.mlp(aff, x) == pytest.approx(0.5 * .2 - .4 - 1.2 + .2 + .125, rel=1e-15)


def test_pinn_G_features():
    """G_pinn(U)_j = L o MLP(c0 t_from/T, c1 t_to/T, c2 U_j/L, c3 S_j/L) (reading Q6-Q8), checked
    with an affine net whose weights pick out one feature at a time."""
    p = synth.single(5, 4, K=1.0, L=4.0, T=2.0)
    U = np.arange(1.0, 6.0)[None, :] * 0.3
    S = 4.0 / 6.0 * np.arange(1, 6)
    n = 1
    t_from, t_to = 2.0 - n * 0.5, 2.0 - (n + 1) * 0.5
    feats = [np.full(5, t_from / 2.0), np.full(5, t_to / 2.0), U[0] / 4.0, S / 4.0]
    for c in range(4):
        W = np.zeros((1, 4), np.float32)
        W[0, c] = 1.0
        net = synth.Net([4, 1], [W], [np.zeros(1, np.float32)], in_scale=np.array([1, 2, 3, 4], np.float32),
                        out_scale=0.5)
        G = oracle.pinn_G(p, net, n, U)[0]
        assert np.allclose(G, 4.0 * 0.5 * (c + 1) * feats[c], rtol=1e-15, atol=0)
    # 2-input mode ignores U
    W2 = np.array([[1.0, 1.0]], np.float32)
    net2 = synth.Net([2, 1], [W2], [np.zeros(1, np.float32)])
    assert np.allclose(oracle.pinn_G(p, net2, n, U)[0], 4.0 * (t_to / 2.0 + S / 4.0), rtol=1e-15)
    assert np.array_equal(oracle.pinn_G(p, net2, n, U), oracle.pinn_G(p, net2, n, 2 * U))


def test_pinn_G_vs_matrix_form():
    p = synth.config("C1")
    net = synth.kaiming_net(synth.PINN_3x20, seed=0)
    U = synth.random_state(1, 64, seed=2).astype(np.float64)
    G = oracle.pinn_G(p, net, 2, U)
    S = 4.0 / 65 * np.arange(1, 65)
    ref = [4.0 * _numpy_mlp(net, [0.5, 0.25, U[0, j] / 4.0, S[j] / 4.0]) for j in range(64)]
    assert np.allclose(G[0], ref, rtol=1e-12, atol=1e-13)


# ---------------------------------------------------------------- Parareal

def test_hand_recurrence(golden):
    """Two slices of w' = -w (one node, zero BC): F = n_f IE steps, G = n_c IE steps per slice.
    Eq. (7) with the Q12 schedule gives, with f = (1+dT/n_f)^-n_f and g = (1+dT/n_c)^-n_c:
      U^0 = (1, g, g^2);  U^1 = (1, f, 2fg - g^2);  U^2 = (1, f, f^2).
    With f -> e^-0.5 and g = 1/1.5 these are SPEC.md:378's printed values."""
    h = golden("spec_examples.json")["hand_recurrence"]
    f_ex, g1 = math.exp(-0.5), 1 / 1.5
    assert h["V1_1"] == pytest.approx(f_ex, abs=1e-12)
    assert h["V2_1"] == pytest.approx(2 * f_ex * g1 - g1 * g1, abs=1e-12)
    assert h["V2_2"] == pytest.approx(f_ex * f_ex, abs=1e-12)
    for nf, nc in ((1000, 1), (7, 3)):
        p = _one_node().replace(N=2, fine_steps=nf, coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=nc,
                                max_iter=2, tol=0.0)
        f, g = (1 + 0.5 / nf) ** -nf, (1 + 0.5 / nc) ** -nc
        U, d, K, hist = oracle.parareal(p, history=True)
        assert K == 2
        assert np.allclose(hist[0, :, 0, 0], [1, g, g * g], rtol=1e-14)
        assert np.allclose(hist[1, :, 0, 0], [1, f, 2 * f * g - g * g], rtol=1e-13)
        assert np.allclose(hist[2, :, 0, 0], [1, f, f * f], rtol=1e-13)
        assert d[0] == pytest.approx(max(abs(f - g) / f, abs(2 * f * g - 2 * g * g) / abs(2 * f * g - g * g)), rel=1e-12)
    # f -> e^{-1/2}: the printed values themselves
    p = _one_node().replace(N=2, fine_steps=200000, coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=1,
                            max_iter=1, tol=0.0)
    U = oracle.parareal(p)[0]
    assert U[1, 0, 0] == pytest.approx(h["V1_1"], rel=2e-6)
    assert U[2, 0, 0] == pytest.approx(h["V2_1"], rel=2e-6)


@pytest.mark.parametrize("coarse", [synth.COARSE_PINN, synth.COARSE_IMPLICIT_EULER])
def test_finite_termination(coarse):
    """U^k_n equals the serial fine solution for n <= k, bitwise; at k = N everywhere."""
    p = synth.config("C1", coarse=coarse, max_iter=4, tol=0.0)
    net = synth.kaiming_net(synth.PINN_3x20, seed=0)
    sf = oracle.serial_fine(p)
    U, d, K, hist = oracle.parareal(p, net, history=True)
    assert K == 4
    for k in range(1, 5):
        assert np.array_equal(hist[k, :k + 1], sf[:k + 1])
    assert np.array_equal(U, sf)


def test_G_equals_F_converges_in_one_iteration():
    """with G = F the k=0 sweep already is the serial fine solution, so delta^1 = 0."""
    p = synth.config("C1", coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=100, max_iter=4, tol=1e-12)
    U, d, K, _ = oracle.parareal(p)
    assert K == 1 and d[0] == 0.0
    assert np.array_equal(U, oracle.serial_fine(p))


def test_stop_rule_strict():
    """Q13: stop at the first k with delta^k < tol (strict); tol = 0 runs exactly max_iter."""
    p = synth.config("C1", coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=1, max_iter=4, tol=0.0)
    _, d, K, _ = oracle.parareal(p)
    assert K == 4
    _, d2, K2, _ = oracle.parareal(p.replace(tol=float(d[1])))       # delta^2 == tol: not < tol
    assert K2 == 3
    _, d3, K3, _ = oracle.parareal(p.replace(tol=float(np.nextafter(d[1], 1.0))))
    assert K3 == 2


def test_convergence_expectation_c1():
    """Non-binding expectation (probe): C1 numerical G with n_c=1 gives
    delta ~ 5.0e-4, 7.5e-5, 1.5e-5, 1.9e-6."""
    p = synth.config("C1", coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=1, max_iter=4, tol=0.0)
    U, d, K, hist = oracle.parareal(p, history=True)
    assert np.allclose(d, [5.0e-4, 7.5e-5, 1.5e-5, 1.9e-6], rtol=0.05)


def test_one_iteration_below_discretisation_error():
    """'After one iteration, the iteration error of Parareal is smaller than the
    discretization error of the fine method' -- at the paper's P=16 slices with a numerical G of
    half the fine steps per slice (reading Q2)."""
    p = synth.single(64, 16, coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=50, max_iter=1, tol=0.0)
    U, d, K, hist = oracle.parareal(p, history=True)
    sf = oracle.serial_fine(p)[-1, 0]
    S = 4.0 / 65 * np.arange(1, 65)
    ex = np.array([oracle.bs_call(s, 1.0, .05, .2, 1.0) for s in S])
    it_err = np.linalg.norm(hist[1, -1, 0] - sf) / np.linalg.norm(sf)
    disc_err = np.linalg.norm(sf - ex) / np.linalg.norm(ex)
    assert it_err < 1e-2 * disc_err


def test_paper_ratio_coarse_reaches_roundoff_in_three():
    """P:270 'After K=3 iterations Parareal has reproduced the fine solution up to round-off':
    with a per-slice numerical G of half the fine steps (reading Q2) the error vs serial fine at
    k=3 is at round-off level (SURVEY.md probe 4.2e-15 at the C3 parameters; here N=16, M=256)."""
    p = synth.single(256, 16, coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=50, max_iter=3, tol=0.0)
    U, d, K, _ = oracle.parareal(p)
    sf = oracle.serial_fine(p)
    assert np.linalg.norm(U[-1, 0] - sf[-1, 0]) / np.linalg.norm(sf[-1, 0]) < 1e-12


def test_fp32_instantiation_tracks_fp64():
    """The FP32 build (stability gate) follows the FP64 oracle on a contractive run."""
    p = synth.config("C1", coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=1, max_iter=3, tol=0.0)
    U64 = oracle.parareal(p)[0]
    U32 = oracle.parareal(p, prec=32)[0]
    assert np.max(np.abs(U64 - U32)) < 1e-5 * np.max(np.abs(U64))


def test_multi_instance_is_independent():
    """Instances never interact: a B=3 run equals three B=1 runs (delta is the max over instances)."""
    pb = synth.Problem(M=32, strike=np.array([0.8, 1.0, 1.3]), sigma=np.array([0.1, 0.3, 0.2]),
                       rate=np.array([0.05, 0.02, 0.0]), L=np.array([3.2, 4.0, 5.2]), N=4, fine_steps=20,
                       coarse=synth.COARSE_IMPLICIT_EULER, max_iter=3, tol=0.0)
    U, d, _, _ = oracle.parareal(pb)
    ds = []
    for b in range(3):
        pi = pb.replace(strike=pb.strike[b:b + 1], sigma=pb.sigma[b:b + 1], rate=pb.rate[b:b + 1], L=pb.L[b:b + 1])
        Ui, di, _, _ = oracle.parareal(pi)
        assert np.array_equal(U[:, b], Ui[:, 0])
        ds.append(di)
    assert np.array_equal(d, np.max(ds, axis=0))


def test_invalid_arguments():
    p = synth.config("C1")
    for bad in (dict(M=0), dict(N=0), dict(fine_steps=0), dict(max_iter=5), dict(tol=-1.0),
                dict(sigma=np.array([0.0])), dict(L=np.array([0.5]))):
        with pytest.raises(ValueError):
            oracle.serial_fine(p.replace(**bad)) if "max_iter" not in bad and "tol" not in bad else \
                oracle.parareal(p.replace(coarse=synth.COARSE_IMPLICIT_EULER, **bad))
