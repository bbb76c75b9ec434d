"""Pins of the PINN-training oracle (oracle/pinn_train.py).

The references are independent of the oracle's own code: the C++ oracle's scalar MLP (another
implementation of the network), central finite differences (the definition of a derivative),
hand-differentiated special nets, exact solutions of Eq. (1) (V = S,
SPEC S:214), PyTorch autograd and torch.optim.Adam (independent AD and optimiser
implementations, CPU, float64), and invariants (the shuffle is a bijection).
"""
import numpy as np
import pytest
import torch

import oracle
from oracle import pinn_train as pt
from paper_2303_03848_b200 import synth

MK = dict(K=1.0, sigma=0.2, r=0.05, T=1.0, L=4.0, upper_bc=0)


def _params(net):
    return [(np.asarray(W, np.float64), np.asarray(b, np.float64)) for W, b in zip(net.W, net.b)]


def _points(n, seed=0):
    rng = np.random.default_rng(seed)
    return rng.uniform(0, MK["T"], n), rng.uniform(0.05, MK["L"], n)


# ---------------------------------------------------------------- the shuffle

@pytest.mark.parametrize("n", [1, 2, 3, 7, 64, 1000, 10000, 65537])
def test_perm_is_a_bijection_and_deterministic(n):
    p = pt.perm(11, 5, 0, n)
    assert np.array_equal(np.sort(p), np.arange(n))
    assert np.array_equal(p, pt.perm(11, 5, 0, n))


def test_perm_differs_between_epochs_sets_and_seeds():
    a = pt.perm(1, 0, 0, 5000)
    for other in (pt.perm(1, 1, 0, 5000), pt.perm(1, 0, 1, 5000), pt.perm(2, 0, 0, 5000)):
        assert np.mean(a != other) > 0.99
    # a shuffle, not a near-identity: positions move, and the order is far from monotone
    assert np.mean(a == np.arange(5000)) < 0.01
    assert abs(np.corrcoef(a, np.arange(5000))[0, 1]) < 0.1


def test_batches_partition_each_set():
    n_f, n_b, n_e, nb = 1003, 101, 99, 7
    got = [pt.batch_indices(3, 2, nb, i, n_f, n_b, n_e) for i in range(nb)]
    for which, n in enumerate((n_f, n_b, n_e)):
        allidx = np.concatenate([g[which] for g in got])
        assert np.array_equal(np.sort(allidx), np.arange(n))


def test_splitmix64_reference_values():
    # SplitMix64 sequence from state 0 (Vigna's reference implementation: first outputs)
    s, outs = 0, []
    for _ in range(3):
        outs.append(pt.splitmix64(s))
        s = (s + 0x9E3779B97F4A7C15) & ((1 << 64) - 1)
    assert outs == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


# ---------------------------------------------------------------- network and jets

@pytest.mark.parametrize("dims,act", [([2, 20, 20, 20, 1], pt.TANH), ([2, 8, 1], pt.TANH), ([2, 16, 16, 1], pt.RELU)])
def test_value_matches_the_cpp_mlp(dims, act):
    net = synth.kaiming_net(dims, seed=3, activation=act)
    t, S = _points(50)
    V = pt.forward_jet(_params(net), act, MK["T"], MK["L"], t, S)[0]
    ref = [MK["L"] * oracle.mlp(net, np.array([ti / MK["T"], Si / MK["L"]])) for ti, Si in zip(t, S)]
    np.testing.assert_allclose(V, ref, rtol=1e-12, atol=1e-12)


def test_jets_match_central_differences():
    net = synth.kaiming_net([2, 20, 20, 20, 1], seed=1)
    P = _params(net)
    t, S = _points(40, seed=2)
    V, V_t, V_S, V_SS = pt.forward_jet(P, pt.TANH, MK["T"], MK["L"], t, S)
    f = lambda tt, SS: pt.forward_jet(P, pt.TANH, MK["T"], MK["L"], tt, SS)[0]
    h = 1e-5
    np.testing.assert_allclose(V_t, (f(t + h, S) - f(t - h, S)) / (2 * h), rtol=1e-6, atol=1e-8)
    np.testing.assert_allclose(V_S, (f(t, S + h) - f(t, S - h)) / (2 * h), rtol=1e-6, atol=1e-8)
    h2 = 1e-3
    np.testing.assert_allclose(V_SS, (f(t, S + h2) - 2 * V + f(t, S - h2)) / (h2 * h2), rtol=1e-4, atol=1e-6)


def test_single_tanh_neuron_by_hand():
    # u = tanh(w_t t/T + w_s S/L + b), Ṽ = L (w_o u + b_o):
    # Ṽ_S = w_o w_s (1 − u²),  Ṽ_SS = −2 u (1 − u²) w_o w_s² / L,  Ṽ_t = L w_o w_t (1 − u²) / T
    wt, ws, b, wo, bo = 0.7, -1.3, 0.2, 1.9, -0.4
    P = [(np.array([[wt, ws]]), np.array([b])), (np.array([[wo]]), np.array([bo]))]
    t, S = np.array([0.3, 0.9]), np.array([1.1, 3.7])
    T, L = 1.5, 4.0
    u = np.tanh(wt * t / T + ws * S / L + b)
    V, V_t, V_S, V_SS = pt.forward_jet(P, pt.TANH, T, L, t, S)
    np.testing.assert_allclose(V, L * (wo * u + bo), rtol=1e-14)
    np.testing.assert_allclose(V_t, L * wo * wt * (1 - u * u) / T, rtol=1e-14)
    np.testing.assert_allclose(V_S, wo * ws * (1 - u * u), rtol=1e-14)
    np.testing.assert_allclose(V_SS, -2 * u * (1 - u * u) * wo * ws * ws / L, rtol=1e-13)


def test_residual_exact_solution_and_hand_substitution():
    # V = S solves Eq. (1): affine net y = S/L, Ṽ = L·y = S → f = rS − rS = 0
    P = [(np.array([[0.0, 1.0]]), np.array([0.0]))]
    t, S = _points(30)
    jet = pt.forward_jet(P, pt.TANH, MK["T"], MK["L"], t, S)
    np.testing.assert_allclose(jet[0], S, rtol=1e-15)
    assert np.max(np.abs(pt.residual(jet, S, 0.4, 0.03))) < 1e-14
    # hand substitution (SPEC S:216 analogue): jet (V, V_t, V_S, V_SS) = (S², 0, 2S, 2) at S = 100,
    # σ = 0.4, r = 0.03 → ½σ²S²·2 + rS·2S − rS² = (σ² + r) S² = 1900
    S1 = np.array([100.0])
    f = pt.residual((S1 ** 2, np.zeros(1), 2 * S1, np.full(1, 2.0)), S1, 0.4, 0.03)
    assert f[0] == pytest.approx(1900.0, rel=1e-14)


def test_zero_network_losses():
    # the identically zero network gives MSE_f = 0, MSE_b = mean target², MSE_exp = mean payoff²
    net = synth.kaiming_net([2, 20, 20, 1], seed=0)
    P = _params(net)
    P[-1] = (np.zeros_like(P[-1][0]), np.zeros_like(P[-1][1]))
    sets = synth.collocation(MK, 500, 60, 70, seed=4)
    mf, mb, me = pt.loss_terms(P, pt.TANH, MK, *sets)
    t_b, S_b, S_e = np.asarray(sets[2], float), np.asarray(sets[3], float), np.asarray(sets[4], float)
    up = MK["L"] - MK["K"] * np.exp(-MK["r"] * (MK["T"] - t_b))
    assert mf == 0.0
    assert mb == pytest.approx(np.mean(np.where(S_b > 0, up, 0.0) ** 2), rel=1e-14)
    assert me == pytest.approx(np.mean(np.maximum(S_e - MK["K"], 0) ** 2), rel=1e-14)


# ---------------------------------------------------------------- gradient and optimiser

def _torch_loss(params, act, mk, sets):
    """The same losses, written with torch autograd (double backward for V_SS)."""
    Ps = [(torch.tensor(W, requires_grad=True), torch.tensor(b, requires_grad=True)) for W, b in params]
    T, L, K, sig, r = mk["T"], mk["L"], mk["K"], mk["sigma"], mk["r"]
    phi = torch.tanh if act == pt.TANH else torch.relu

    def V(t, S):
        h = torch.stack([t / T, S / L], 1)
        for W, b in Ps[:-1]:
            h = phi(h @ W.T + b)
        return L * (h @ Ps[-1][0].T + Ps[-1][1])[:, 0]

    t_f, S_f, t_b, S_b, S_e = [torch.tensor(np.asarray(a, np.float64)) for a in sets]
    t_f.requires_grad_(True)
    S_f.requires_grad_(True)
    v = V(t_f, S_f)
    vt, vs = torch.autograd.grad(v.sum(), (t_f, S_f), create_graph=True)
    vss, = torch.autograd.grad(vs.sum(), S_f, create_graph=True)
    f = vt + 0.5 * sig * sig * S_f * S_f * vss + r * S_f * vs - r * v
    tgt = torch.where(S_b > 0.5 * L, L - K * torch.exp(-r * (T - t_b)), torch.zeros_like(t_b))
    loss = (f ** 2).mean() + ((V(t_b, S_b) - tgt) ** 2).mean() + \
        ((V(torch.full_like(S_e, T), S_e) - torch.clamp(S_e - K, min=0)) ** 2).mean()
    loss.backward()
    return float(loss.detach()), [(W.grad.numpy(), b.grad.numpy()) for W, b in Ps]


@pytest.mark.parametrize("dims,act", [([2, 20, 20, 20, 1], pt.TANH), ([2, 12, 12, 1], pt.RELU)])
def test_gradient_matches_torch_autograd(dims, act):
    net = synth.kaiming_net(dims, seed=5, activation=act)
    sets = synth.collocation(MK, 300, 40, 50, seed=6)
    (mf, mb, me), g = pt.loss_and_grad(_params(net), act, MK, *sets)
    loss, gt = _torch_loss(_params(net), act, MK, sets)
    assert mf + mb + me == pytest.approx(loss, rel=1e-12)
    np.testing.assert_allclose(pt.flatten(g), pt.flatten(gt), rtol=1e-9, atol=1e-12 * np.max(np.abs(pt.flatten(gt))))


def test_gradient_matches_finite_differences():
    # ≤ 200 parameters, tanh, relative 1e-5
    net = synth.kaiming_net([2, 8, 8, 1], seed=9)
    sets = synth.collocation(MK, 120, 20, 20, seed=1)
    P = _params(net)
    _, g = pt.loss_and_grad(P, pt.TANH, MK, *sets)
    theta = pt.flatten(P)
    assert theta.size <= 200
    fd = np.empty_like(theta)
    h = 1e-6
    for i in range(theta.size):
        tp, tm = theta.copy(), theta.copy()
        tp[i] += h
        tm[i] -= h
        fp = sum(pt.loss_terms(pt.unflatten(tp, net.dims), pt.TANH, MK, *sets))
        fm = sum(pt.loss_terms(pt.unflatten(tm, net.dims), pt.TANH, MK, *sets))
        fd[i] = (fp - fm) / (2 * h)
    np.testing.assert_allclose(pt.flatten(g), fd, rtol=1e-5, atol=1e-7 * np.max(np.abs(fd)))


def test_adam_matches_torch_optim():
    rng = np.random.default_rng(0)
    theta0 = rng.standard_normal(37)
    th = theta0.copy()
    m, v = np.zeros(37), np.zeros(37)
    tt = torch.tensor(theta0.copy(), requires_grad=True)
    opt = torch.optim.Adam([tt], lr=1e-2, betas=(0.9, 0.999), eps=1e-8)
    for step in range(1, 8):
        g = rng.standard_normal(37) * (1 + step)
        pt.adam_step(th, m, v, g, step, 1e-2)
        opt.zero_grad()
        tt.grad = torch.tensor(g)
        opt.step()
    np.testing.assert_allclose(th, tt.detach().numpy(), rtol=1e-13, atol=1e-15)


def test_training_reduces_the_loss_and_approaches_the_closed_form():
    # P:210-211 / Table 1: Adam drives all three terms down; the trained Ṽ(0, S) approaches the
    # closed-form price (the PINN is a usable coarse propagator)
    net = synth.kaiming_net([2, 16, 16, 1], seed=2)
    sets = synth.collocation(MK, 2000, 200, 200, seed=3)
    tr = pt.Trainer(net, MK, sets, batches=1, seed=1)
    before = sum(tr.full_loss())
    tr.epochs(600, 1e-2)
    after = sum(tr.full_loss())
    assert after < before / 100
    S = np.linspace(0.2, 3.8, 50)
    V0 = pt.forward_jet(tr.params(), pt.TANH, MK["T"], MK["L"], np.zeros(50), S)[0]
    ref = np.array([oracle.bs_call(s, MK["K"], MK["r"], MK["sigma"], MK["T"]) for s in S])
    assert np.linalg.norm(V0 - ref) / np.linalg.norm(ref) < 0.1
