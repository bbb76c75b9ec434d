"""GPU PINN training (include/pinn_train.h) against the training oracle
(oracle/pinn_train.py, pinned in tests/test_pinn_train_pins.py), through the C ABI.

fp32 kernels vs the fp64 oracle.  Tolerances: loss terms 1e-4 relative (fp32 residual sums over
10^4-10^5 points); gradients |g − ref| ≤ 1e-3·|ref| + 1e-4·‖ref‖∞ (fp32 contraction of 10^4
points' jets); trajectories through the loss history (Adam's sign-like steps amplify fp32
differences in near-zero gradient components, so parameters are compared in norm)."""
import numpy as np
import pytest

import oracle
from oracle import pinn_train as opt
from paper_2303_03848_b200 import parareal, pinn_train, synth

pytestmark = pytest.mark.gpu

MK = dict(K=1.0, sigma=0.2, r=0.05, T=1.0, L=4.0, upper_bc=0)


def _grad_close(g, ref, what):
    g, ref = np.asarray(g, np.float64), np.asarray(ref, np.float64)
    tol = 1e-3 * np.abs(ref) + 1e-4 * np.max(np.abs(ref))
    bad = np.abs(g - ref) > tol
    assert not bad.any(), "%s: %d of %d gradient entries off (max rel %.3g)" % (
        what, bad.sum(), bad.size, np.max(np.abs(g - ref) / np.max(np.abs(ref))))


@pytest.mark.parametrize("dims,act", [([2, 20, 20, 20, 1], synth.ACT_TANH), ([2, 8, 8, 1], synth.ACT_TANH),
                                      ([2, 16, 16, 16, 16, 1], synth.ACT_TANH), ([2, 32, 32, 1], synth.ACT_TANH),
                                      ([2, 20, 20, 1], synth.ACT_RELU), ([2, 64, 64, 64, 1], synth.ACT_TANH),
                                      ([2] + [50] * 10 + [1], synth.ACT_RELU),   # the paper's net
                                      ([2] + [50] * 4 + [1], synth.ACT_TANH)])
def test_full_loss_and_batch_gradient_match_oracle(dims, act):
    net = synth.pinn2_net(dims, seed=1, activation=act)
    sets = synth.collocation(MK, 3000, 300, 300, seed=2)   # 3600 points: 28 CTAs, ragged tail
    tr_o = opt.Trainer(net, MK, sets, batches=3, seed=7)
    with pinn_train.Trainer(net, MK, sets, batches=3, seed=7) as tr:
        np.testing.assert_allclose(tr.loss(), tr_o.full_loss(), rtol=1e-4)
        for step in (0, 4, 8):                            # epochs 0, 1, 2: three different shuffles
            l, g = tr.batch_gradient(step)
            (lo, go) = tr_o.gradient(step)
            np.testing.assert_allclose(l, lo, rtol=1e-4, err_msg="batch loss of step %d" % step)
            _grad_close(g, go, "step %d %s" % (step, dims))


def test_batch_selection_follows_the_shuffle():
    """The batch loss equals the oracle's on the oracle's shuffled batch (to fp32 rounding) and
    differs clearly from the loss of the unshuffled split, so the device perm is the oracle's."""
    net = synth.pinn2_net([2, 20, 20, 1], seed=3)
    sets = synth.collocation(MK, 4000, 400, 400, seed=5)
    tr_o = opt.Trainer(net, MK, sets, batches=8, seed=123)
    with pinn_train.Trainer(net, MK, sets, batches=8, seed=123) as tr:
        for step in (0, 5, 9, 31):
            l, _ = tr.batch_gradient(step)
            lo, _ = tr_o.gradient(step)
            np.testing.assert_allclose(l, lo, rtol=2e-5, err_msg="step %d" % step)
    t_f, S_f, t_b, S_b, S_e = sets
    plain = opt.loss_terms(tr_o.params(), opt.TANH, MK, t_f[:500], S_f[:500], t_b[:50], S_b[:50], S_e[:50])
    assert abs(plain[0] - lo[0]) > 1e-3 * abs(lo[0]) or abs(plain[2] - lo[2]) > 1e-3 * abs(lo[2])


def test_adam_trajectory_matches_oracle():
    net = synth.pinn2_net([2, 20, 20, 20, 1], seed=0)
    sets = synth.collocation(MK, 2000, 200, 200, seed=1)
    tr_o = opt.Trainer(net, MK, sets, batches=4, seed=3)
    h_o = tr_o.epochs(5, 1e-2)
    with pinn_train.Trainer(net, MK, sets, batches=4, seed=3) as tr:
        h = tr.epochs(3, 1e-2)
        h = np.concatenate([h, tr.epochs(2, 1e-2)])        # two calls continue the same run
        assert tr.steps == 20
        theta = tr.params()
    np.testing.assert_allclose(h, h_o, rtol=2e-3)
    theta0 = opt.flatten([(np.asarray(W, np.float64), np.asarray(b, np.float64)) for W, b in zip(net.W, net.b)])
    assert np.linalg.norm(theta - tr_o.theta) < 1e-2 * np.linalg.norm(tr_o.theta - theta0)


def test_training_is_deterministic():
    net = synth.pinn2_net([2, 20, 20, 20, 1], seed=0)
    sets = synth.collocation(MK, 5000, 500, 500, seed=1)
    out = []
    for _ in range(2):
        with pinn_train.Trainer(net, MK, sets, batches=5, seed=9) as tr:
            h = tr.epochs(10, 1e-2)
            out.append((h, tr.params()))
    assert np.array_equal(out[0][0], out[1][0]) and np.array_equal(out[0][1], out[1][1])


def test_paper_schedule_trains_a_usable_coarse_propagator():
    """P:190 collocation counts, P:210-211 schedule (5000 epochs at 1e-2, 800 at 1e-3), shuffled
    batches of 10 per epoch, 3x20 tanh net for the C2 market.  The trained Ṽ(0, S)
    approaches the closed form and, as a 2-input coarse propagator in Parareal at
    C2, the GPU solve matches the oracle's on every iterate with the same K."""
    net0 = synth.pinn2_net([2, 20, 20, 20, 1], seed=0)
    n_f, n_b, n_e = synth.PAPER_COLLOCATION
    sets = synth.collocation(MK, n_f, n_b, n_e, seed=0)
    with pinn_train.Trainer(net0, MK, sets, batches=10, seed=0) as tr:
        l0 = tr.loss()
        tr.epochs(5000, 1e-2, history=False)
        tr.epochs(800, 1e-3, history=False)
        l1 = tr.loss()
        net = tr.net()
    assert np.all(np.isfinite(l1)) and l1.sum() < 1e-3 * l0.sum()
    np.testing.assert_allclose(l1, opt.loss_terms(
        [(np.asarray(W, np.float64), np.asarray(b, np.float64)) for W, b in zip(net.W, net.b)], opt.TANH, MK, *sets), rtol=1e-3)
    p = synth.config("C2", coarse=synth.COARSE_PINN, max_iter=4, tol=0.0)
    S = np.arange(1, p.M + 1) * 4.0 / (p.M + 1)
    with parareal.Context(p) as c:
        c.load_weights(net)
        G0 = c.apply_coarse(p.N - 1, np.zeros((1, p.M), np.float32))[0]   # Ṽ(t = 0, S)
        U, rep = c.solve()
        it = c.copy_iterates(0, p.N + 1)
    ref = np.array([oracle.bs_call(s, 1.0, 0.05, 0.2, 1.0) for s in S])
    assert np.linalg.norm(G0 - ref) / np.linalg.norm(ref) < 3e-2
    ref_U, ref_d, K, _ = oracle.parareal(p, net)
    assert rep["iterations"] == K
    rel = np.max(np.abs(it - ref_U)) / np.max(np.abs(ref_U))
    assert rel < 1e-5, rel
