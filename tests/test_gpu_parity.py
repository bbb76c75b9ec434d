"""CUDA path vs the CPU oracle, element by element on the same seeded inputs.

Every call goes through the C ABI (libparareal.so) via the ctypes binding."""
import numpy as np
import pytest

import oracle
from gpu_helpers import TOL_FP32, assert_close, assert_delta, rel_err
from paper_2303_03848_b200 import parareal, synth

pytestmark = pytest.mark.gpu

FINE_KERNELS = [1, 2]   # resident, streamed (PR_OPT_FINE_KERNEL); the grid-resident kernel (3) has its own tests


def ctx_for(p, net=None, fine_kernel=0):
    c = parareal.Context(p)
    if fine_kernel:
        c.set_option(parareal.OPT_FINE_KERNEL, fine_kernel)
    if net is not None:
        c.load_weights(net)
    return c


# ------------------------------------------------------------------ single propagators (T1)

@pytest.mark.parametrize("kernel", FINE_KERNELS)
@pytest.mark.parametrize("M,N,n", [(1, 2, 1), (5, 4, 0), (64, 4, 3), (100, 8, 5), (1024, 32, 17), (2000, 4, 2)])
def test_fine_single_slice(kernel, M, N, n):
    p = synth.single(M, N)
    U = synth.random_state(1, M, seed=M)
    with ctx_for(p, fine_kernel=kernel) as c:
        got = c.apply_fine(n, U)
    ref = oracle.fine(p, n, U.astype(np.float64))
    assert_close(got, ref, what="F M=%d n=%d kernel=%d" % (M, n, kernel))


@pytest.mark.parametrize("M", [4097, 12345, 1 << 16])
def test_fine_streamed_multi_tile(M):
    """Several 2048-point tiles with a ragged tail: look-back across tiles."""
    p = synth.single(M, 64, fine_steps=20)
    U = synth.random_state(1, M, seed=3)
    with ctx_for(p, fine_kernel=2) as c:
        got = c.apply_fine(7, U)
    assert_close(got, oracle.fine(p, 7, U.astype(np.float64)), what="F streamed M=%d" % M)


def test_fine_c3_size_single_slice():
    """C3 grid (2^20 points, dtau = 1/6400), one slice of 100 steps, default (streamed) kernel."""
    p = synth.config("C3")
    U0 = oracle.payoff(p)
    with ctx_for(p) as c:
        got = c.apply_fine(0, U0.astype(np.float32))
    ref = oracle.fine(p, 0, U0)
    assert_close(got, ref, what="F C3")


def test_fine_portfolio_instances():
    """C4-style instances (distinct sigma and strike, L_b = 4K_b) share one launch."""
    p = synth.portfolio(n_k=4, n_s=8, M=256, N=16)
    U = oracle.payoff(p).astype(np.float32)
    for kernel in FINE_KERNELS:
        with ctx_for(p, fine_kernel=kernel) as c:
            got = c.apply_fine(3, U)
        assert_close(got, oracle.fine(p, 3, U.astype(np.float64)), what="F portfolio kernel=%d" % kernel)


# ------------------------------------------------------------------ θ-step fine propagator (NEXT-1)
# Crank–Nicolson (θ = 1/2, the paper's F) and a θ = 3/4 scheme: explicit 3-point stencil
# plus the implicit solve, against the oracle's θ-step (pinned in test_oracle_pins).

@pytest.mark.parametrize("kernel", FINE_KERNELS)
@pytest.mark.parametrize("M,N,n,theta", [(1, 2, 1, 0.5), (64, 4, 3, 0.5), (1000, 8, 5, 0.5), (2000, 4, 1, 0.75),
                                         (2048, 4, 0, 0.5), (5000, 8, 2, 0.5), (12345, 16, 9, 0.5)])
def test_fine_theta_single_slice(kernel, M, N, n, theta):
    if kernel == 1 and M > 2048:
        pytest.skip("resident kernel holds M <= 2048")
    p = synth.single(M, N, fine_theta=theta, fine_steps=40)
    U = synth.random_state(1, M, seed=M + 1)
    with ctx_for(p, fine_kernel=kernel) as c:
        got = c.apply_fine(n, U)
    ref = oracle.fine(p, n, U.astype(np.float64))
    assert_close(got, ref, what="F theta=%g M=%d n=%d kernel=%d" % (theta, M, n, kernel))


def test_fine_cn_portfolio_and_payoff():
    """CN on C4-style instances (several factor sets and strikes) from the payoff kink, both kernels."""
    p = synth.portfolio(n_k=3, n_s=4, M=256, N=16, fine_theta=0.5)
    U = oracle.payoff(p).astype(np.float32)
    for kernel in FINE_KERNELS:
        with ctx_for(p, fine_kernel=kernel) as c:
            got = c.apply_fine(5, U)
        assert_close(got, oracle.fine(p, 5, U.astype(np.float64)), what="F CN portfolio kernel=%d" % kernel)


def test_fine_cn_c3_size_single_slice():
    """CN at the C3 grid (2^20 points, 100 steps): dτ·a_j reaches 3e6, far outside the M-matrix
    range of the explicit part; fp32 state between streamed passes stays within tolerance."""
    p = synth.config("C3", fine_theta=0.5)
    U0 = oracle.payoff(p)
    with ctx_for(p) as c:
        got = c.apply_fine(0, U0.astype(np.float32))
    assert_close(got, oracle.fine(p, 0, U0), what="F CN C3")


@pytest.mark.parametrize("kernel,M", [(1, 300), (2, 300), (2, 6000)])
def test_serial_fine_cn(kernel, M):
    p = synth.single(M, 8, fine_theta=0.5, fine_steps=20)
    with ctx_for(p, fine_kernel=kernel) as c:
        got, _ = c.serial_fine()
    ref = oracle.serial_fine(p)[-1]
    assert_close(got, ref, what="serial fine CN kernel=%d M=%d" % (kernel, M))


@pytest.mark.parametrize("kernel,M,N", [(1, 64, 4), (2, 5000, 6), (2, 3000, 17)])
def test_parareal_cn_fine_ie_coarse(kernel, M, N):
    """Parareal with the CN fine propagator and the implicit-Euler coarse one (the paper's
    numerical pairing): every iterate against the oracle, fixed K."""
    p = synth.single(M, N, fine_theta=0.5, fine_steps=20, coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=2,
                     max_iter=3, tol=0.0)
    with ctx_for(p, fine_kernel=kernel) as c:
        _, rep = c.solve()
        it = c.copy_iterates(0, p.N + 1)
    ref_U, ref_d, K, _ = oracle.parareal(p)
    assert rep["iterations"] == K == 3
    assert_close(it, ref_U, what="CN Parareal iterates kernel=%d M=%d" % (kernel, M))
    assert_delta(rep["delta"], ref_d)


@pytest.mark.parametrize("dims,act", [(synth.PINN_3x20, synth.ACT_TANH), (synth.PINN_PAPER, synth.ACT_RELU),
                                      (synth.PINN_PAPER, synth.ACT_TANH), ([4, 64, 64, 64, 64, 1], synth.ACT_TANH),
                                      ([4, 8, 8, 1], synth.ACT_TANH), ([2, 16, 16, 1], synth.ACT_TANH),
                                      ([4, 32, 32, 1], synth.ACT_RELU)])
def test_pinn_G_single_slice(dims, act):
    p = synth.single(1000, 8)
    net = synth.kaiming_net(dims, seed=5, activation=act, in_scale=[1.0, 0.5, 2.0, 1.5][:dims[0]],
                            out_scale=0.75)
    U = synth.random_state(1, 1000, seed=9) * 2.0
    with ctx_for(p, net) as c:
        got = c.apply_coarse(3, U)
    ref = oracle.pinn_G(p, net, 3, U.astype(np.float64))
    assert_close(got, ref, what="G %s" % dims)


@pytest.mark.parametrize("pinn_kernel", [0, 1, 2])
@pytest.mark.parametrize("dims,act", [(synth.PINN_3x20, synth.ACT_TANH), (synth.PINN_3x20, synth.ACT_RELU),
                                      ([2, 20, 20, 20, 1], synth.ACT_TANH), (synth.PINN_PAPER, synth.ACT_TANH),
                                      (synth.PINN_PAPER, synth.ACT_RELU), ([4, 64, 64, 64, 1], synth.ACT_TANH),
                                      ([4, 32, 32, 32, 1], synth.ACT_TANH)])
def test_pinn_G_both_weight_paths(pinn_kernel, dims, act):
    """Every evaluator agrees with the oracle: constant-bank weights (auto for small nets at this
    size), shared-memory weights (one thread per point), and the latency modes (4 threads per
    point with shuffles for 20-wide nets; groups of W/NPT threads with a shared-memory exchange
    for 32/50/64-wide nets, including the paper's 10x50 architecture).  M = 3000 gives a
    ragged last CTA in every mode."""
    p = synth.single(3000, 8)
    net = synth.kaiming_net(dims, seed=11, activation=act)
    U = synth.random_state(1, 3000, seed=12) * 3.0
    with ctx_for(p, net) as c:
        c.set_option(parareal.OPT_PINN_KERNEL, pinn_kernel)
        got = c.apply_coarse(6, U)
    assert_close(got, oracle.pinn_G(p, net, 6, U.astype(np.float64)), what="G %s path %d" % (dims, pinn_kernel))


# ------------------------------------------------------------------ K4: tensor-core PINN (wide nets)
# PR_PREC_FP16_TC: operands split hi + lo in fp16, three MMAs per product (fp32-level accuracy:
# ~2e-6 emulated on 8x256 nets) -- held to 1e-4.  PR_PREC_BF16_TC: one bf16 pass (8-bit
# mantissa), the fast approximate mode -- its error grows with depth (~1e-2 at 3 layers).

TOL_TC = 1e-4


@pytest.mark.parametrize("W,LH,act", [(64, 2, synth.ACT_TANH), (64, 8, synth.ACT_TANH), (128, 4, synth.ACT_TANH),
                                      (256, 3, synth.ACT_TANH), (256, 8, synth.ACT_TANH), (128, 4, synth.ACT_RELU)])
def test_pinn_G_tensor_cores(W, LH, act):
    """C5 widths: 128-point tiles, tcgen05 MMAs with TMEM accumulators, weights
    resident (small nets) or streamed in 64-column chunks (8x256); a ragged last tile (M = 1000)
    and two instances."""
    p = synth.portfolio(n_k=2, n_s=1, M=1000, N=8)
    net = synth.kaiming_net([4] + [W] * LH + [1], seed=W + LH, activation=act)
    U = oracle.payoff(p) * (1.0 + 0.05 * np.sin(np.arange(1000) / 37.0))
    with ctx_for(p) as c:
        c.load_weights(net, precision=parareal.PREC_FP16_TC)
        got = c.apply_coarse(5, U.astype(np.float32))
    assert_close(got, oracle.pinn_G(p, net, 5, U), tol=TOL_TC, what="G TC W=%d LH=%d" % (W, LH))


@pytest.mark.parametrize("W,LH", [(64, 2), (256, 3), (128, 4), (64, 8)])
def test_pinn_G_tensor_cores_bf16(W, LH):
    p = synth.portfolio(n_k=2, n_s=1, M=700, N=8)
    net = synth.kaiming_net([4] + [W] * LH + [1], seed=3 * W + LH)
    U = oracle.payoff(p)
    with ctx_for(p) as c:
        c.load_weights(net, precision=parareal.PREC_BF16_TC)
        got = c.apply_coarse(2, U.astype(np.float32))
    assert_close(got, oracle.pinn_G(p, net, 2, U), tol=3e-2, what="G TC bf16 W=%d LH=%d" % (W, LH))


@pytest.mark.parametrize("W,LH,act", [(64, 2, synth.ACT_TANH), (256, 3, synth.ACT_TANH), (128, 4, synth.ACT_TANH),
                                      (64, 8, synth.ACT_TANH), (256, 8, synth.ACT_TANH), (128, 3, synth.ACT_RELU)])
def test_pinn_G_tensor_cores_fp16_single_pass(W, LH, act):
    """PR_PREC_FP16X1_TC: one fp16 MMA pass (fp32 accumulation).  Its error on random Kaiming nets
    is 3e-4 .. 4e-3 of the row maximum (scripts/tc_accuracy.py; a numpy emulation with fp16-rounded
    weights and activations gives the same spread), so it is held to 8e-3 here and NOT credited
    with north_star's 1e-3 tensor-core tolerance -- only the split mode (FP16_TC, 1e-4) is.  4x128
    and deeper nets with resident weights run the ping-pong kernel."""
    p = synth.portfolio(n_k=2, n_s=1, M=700, N=8)
    net = synth.kaiming_net([4] + [W] * LH + [1], seed=5 * W + LH, activation=act)
    U = oracle.payoff(p) * (1.0 + 0.05 * np.sin(np.arange(700) / 29.0))
    with ctx_for(p) as c:
        c.load_weights(net, precision=parareal.PREC_FP16X1_TC)
        got = c.apply_coarse(3, U.astype(np.float32))
    assert_close(got, oracle.pinn_G(p, net, 3, U), tol=8e-3, what="G TC fp16x1 W=%d LH=%d" % (W, LH))


@pytest.mark.parametrize("prec,dims,tol", [(1, [4, 128, 128, 128, 1], TOL_TC), (2, [4, 128, 128, 128, 1], 5e-2),
                                           (4, [4, 128, 128, 128, 1], 8e-3), (4, [4, 64, 64, 64, 1], 8e-3)])
def test_pinn_tensor_core_parareal_chain(prec, dims, tol):
    """Full Parareal with the K4 coarse chain (correction fused, δ partials, the copy step) at a
    C5-like width: iterates within the TC tolerance of the oracle with the same fp32-exact fine
    propagator.  prec 1: split fp16 (one-tile kernel); prec 2: bf16 with resident weights, i.e.
    the ping-pong kernel (two tiles per CTA, 256-point δ chunks); M = 3000 leaves a ragged CTA."""
    p = synth.single(3000, 6, coarse=synth.COARSE_PINN, max_iter=2, tol=0.0)
    net = synth.kaiming_net(dims, seed=9)
    with ctx_for(p) as c:
        c.load_weights(net, precision=prec)
        _, rep = c.solve()
        it = c.copy_iterates(0, p.N + 1)
    ref_U, ref_d, K, _ = oracle.parareal(p, net)
    assert rep["iterations"] == K == 2
    assert_close(it, ref_U, tol=tol, what="TC Parareal iterates (precision %d)" % prec)


@pytest.mark.parametrize("W,LH", [(64, 4), (128, 3), (256, 2)])
def test_pinn_tensor_core_two_input_nets(W, LH):
    """2-input (t_to, S) networks -- the form the GPU trainer produces (reading Q28) and the C5
    study runs on the split-fp16 tensor-core chain (profiles/r02/c5_study.md): one G application
    (ragged last tile) and a K = 2 Parareal solve against the oracle at the TC tolerance."""
    net = synth.kaiming_net([2] + [W] * LH + [1], seed=7 * W + LH)
    p = synth.single(1000, 6, coarse=synth.COARSE_PINN, max_iter=2, tol=0.0)
    U = oracle.payoff(p) * (1.0 + 0.05 * np.sin(np.arange(1000) / 23.0))
    with ctx_for(p) as c:
        c.load_weights(net, precision=parareal.PREC_FP16_TC)
        got = c.apply_coarse(4, U.astype(np.float32))
        _, rep = c.solve()
        it = c.copy_iterates(0, p.N + 1)
    assert_close(got, oracle.pinn_G(p, net, 4, U), tol=TOL_TC, what="2-input G TC W=%d LH=%d" % (W, LH))
    ref_U, ref_d, K, _ = oracle.parareal(p, net)
    assert rep["iterations"] == K == 2
    assert_close(it, ref_U, tol=TOL_TC, what="2-input TC Parareal W=%d LH=%d" % (W, LH))
    assert_delta(rep["delta"], ref_d)


def test_pinn_tensor_core_errors():
    p = synth.single(256, 4)
    with ctx_for(p) as c:
        with pytest.raises(parareal.PararealError) as ei:
            c.load_weights(synth.kaiming_net([4, 20, 20, 1]), precision=parareal.PREC_FP16_TC)   # too narrow
        assert ei.value.status == 7
        with pytest.raises(parareal.PararealError) as ei:
            c.load_weights(synth.kaiming_net([4, 64, 64, 1]), precision=parareal.PREC_TF32_TC)
        assert ei.value.status == 7


def test_pinn_G_portfolio():
    p = synth.portfolio(n_k=3, n_s=5, M=300, N=16)
    net = synth.kaiming_net(synth.PINN_3x20, seed=1)
    U = oracle.payoff(p)
    with ctx_for(p, net) as c:
        got = c.apply_coarse(15, U.astype(np.float32))
    assert_close(got, oracle.pinn_G(p, net, 15, U), what="G portfolio")


@pytest.mark.parametrize("kernel", FINE_KERNELS)
def test_numerical_G_single_slice(kernel):
    p = synth.single(777, 8, coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=3)
    U = synth.random_state(1, 777, seed=4)
    with ctx_for(p, fine_kernel=kernel) as c:
        got = c.apply_coarse(2, U)
    assert_close(got, oracle.coarse_ie(p, 2, U.astype(np.float64)), what="G_num")


# ------------------------------------------------------------------ serial fine and Parareal (T2/T3)

@pytest.mark.parametrize("kernel", FINE_KERNELS)
def test_serial_fine_c1(kernel):
    p = synth.config("C1")
    with ctx_for(p, fine_kernel=kernel) as c:
        got, ms = c.serial_fine()
    assert ms > 0
    assert_close(got, oracle.serial_fine(p)[-1], what="serial fine")


@pytest.mark.parametrize("kernel", FINE_KERNELS)
@pytest.mark.parametrize("cfg,tol,K_expected", [("C1", 3e-5, 3), ("C2", 1e-5, 3)])
def test_parareal_numerical_G_converges_like_oracle(kernel, cfg, tol, K_expected):
    """Numerical coarse G (n_c = 1): identical iteration count, delta history and iterates.
    The tol values satisfy the near-tie guard of reading Q18 (checked on the oracle side)."""
    p = synth.config(cfg, coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=1, tol=tol)
    p = p.replace(max_iter=min(p.N, 6))
    ref_U, ref_d, ref_K, _ = oracle.parareal(p)
    assert ref_K == K_expected
    assert ref_d[ref_K - 2] >= 1.5 * tol and ref_d[ref_K - 1] <= tol / 1.5   # Q18 guard
    with ctx_for(p, fine_kernel=kernel) as c:
        U, rep = c.solve()
        it = c.copy_iterates(0, p.N + 1)
    assert rep["iterations"] == ref_K and rep["converged"]
    assert_delta(rep["delta"], ref_d)
    assert_close(U, ref_U[-1], what="U_N")
    assert_close(it, ref_U, what="all U_n")


def _gate_or_amplification(gpu, ref64, ref32, what):
    """Stability gate of SURVEY.md §8(c): if the fp32 oracle stays within the parity tolerance of
    the fp64 oracle, the GPU must too; otherwise the trajectory amplifies rounding and the GPU's
    deviation must stay at the fp32 oracle's own level (factor 10)."""
    try:
        assert_close(ref32, ref64, what="gate")
        gate = True
    except AssertionError:
        gate = False
    if gate:
        assert_close(gpu, ref64, what=what)
    else:
        assert rel_err(gpu, ref64) <= 10 * max(rel_err(ref32, ref64), 1e-6), (what, rel_err(gpu, ref64),
                                                                             rel_err(ref32, ref64))
    return gate


@pytest.mark.parametrize("kernel", FINE_KERNELS)
def test_parareal_pinn_fixed_K(kernel):
    """PINN coarse (random 3x20 weights), fixed K=3: iterates and delta vs the oracle."""
    p = synth.config("C1", coarse=synth.COARSE_PINN, max_iter=3, tol=0.0)
    net = synth.kaiming_net(synth.PINN_3x20, seed=0)
    ref_U, ref_d, ref_K, hist = oracle.parareal(p, net, history=True)
    U32, d32, _, _ = oracle.parareal(p, net, prec=32)
    with ctx_for(p, net, fine_kernel=kernel) as c:
        U, rep = c.solve()
        it = c.copy_iterates(0, p.N + 1)
    assert rep["iterations"] == 3
    _gate_or_amplification(it, ref_U, U32, "PINN iterates C1")
    assert_delta(rep["delta"], ref_d)


def test_parareal_pinn_k1_c2():
    """C2 (32 slices), PINN coarse, one iteration: all boundary states U^1_n vs the oracle."""
    p = synth.config("C2", coarse=synth.COARSE_PINN, max_iter=1, tol=0.0)
    net = synth.kaiming_net(synth.PINN_3x20, seed=2)
    _, _, _, hist = oracle.parareal(p, net, history=True)
    h32 = oracle.parareal(p, net, prec=32, history=True)[3]
    with ctx_for(p, net) as c:
        c.solve()
        it = c.copy_iterates(0, p.N + 1)
    _gate_or_amplification(it, hist[1], h32[1], "C2 PINN k=1")
    # the exact part of the iterate: U^1_0 = U_0 and U^1_1 = F(U_0)
    assert_close(it[:2], hist[1][:2], what="C2 PINN exact prefix")


@pytest.mark.parametrize("coarse", [synth.COARSE_PINN, synth.COARSE_IMPLICIT_EULER])
@pytest.mark.parametrize("kernel", FINE_KERNELS)
def test_finite_termination_bitwise(coarse, kernel):
    """at k = N Parareal reproduces the serial fine solution -- bitwise against the GPU's
    own serial fine with the same kernel configuration (T3), and within tolerance of the oracle."""
    p = synth.config("C1", coarse=coarse, max_iter=4, tol=0.0)
    net = synth.kaiming_net(synth.PINN_3x20, seed=0)
    with ctx_for(p, net if coarse == synth.COARSE_PINN else None, fine_kernel=kernel) as c:
        U, rep = c.solve()
        sf, _ = c.serial_fine()
    assert rep["iterations"] == p.N
    assert np.array_equal(U, sf)
    assert_close(U, oracle.serial_fine(p)[-1], what="k=N vs oracle")


def test_strike_zero_exact_solution():
    """K = 0: V = S is a fixed point of F and numerical G (exact discrete solution)."""
    p = synth.single(1000, 8, K=0.0, L=4.0, coarse=synth.COARSE_IMPLICIT_EULER, max_iter=2, tol=0.0)
    S = 4.0 / 1001 * np.arange(1, 1001)
    with ctx_for(p) as c:
        U, rep = c.solve()
    assert np.max(np.abs(U[0] - S) / S) < 1e-6


def test_determinism():
    p = synth.config("C2", coarse=synth.COARSE_PINN, max_iter=3, tol=0.0)
    net = synth.kaiming_net(synth.PINN_3x20, seed=1)
    with ctx_for(p, net) as c:
        a, ra = c.solve()
        b, rb = c.solve()
    assert np.array_equal(a, b) and np.array_equal(ra["delta"], rb["delta"])


def test_streamed_determinism_and_parity():
    """K2 (streamed, multi-tile, windowed look-back): bitwise run-to-run reproducible and within
    tolerance of the oracle over a short Parareal run with numerical G."""
    p = synth.single(20000, 8, fine_steps=10, coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=2, max_iter=2,
                     tol=0.0)
    with ctx_for(p, fine_kernel=2) as c:
        a, ra = c.solve()
        b, rb = c.solve()
        it = c.copy_iterates(0, p.N + 1)
    assert np.array_equal(a, b) and np.array_equal(ra["delta"], rb["delta"])
    ref_U, ref_d, _, _ = oracle.parareal(p)
    assert_close(it, ref_U, what="streamed Parareal iterates")
    assert_delta(ra["delta"], ref_d)


@pytest.mark.parametrize("M,N,B,theta", [(10000, 20, 1, 1.0), (6000, 18, 1, 1.0), (5000, 9, 2, 1.0),
                                         (10000, 20, 1, 0.5), (5000, 9, 2, 0.5), (4500, 17, 1, 0.75)])
def test_streamed_persistent_kernel_parity(M, N, B, theta):
    """K2's persistent factor-resident kernel (sweeps with >= 16 systems): every iterate against
    the oracle, including ragged item groups (18 slices in groups of 4) and two instances with
    different factor sets sharing a launch; theta-steps run these sweeps on the tile kernel
    (explicit stencil, tile-edge terms) and are checked the same way."""
    if B == 1:
        p = synth.single(M, N, fine_steps=6, coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=1, max_iter=2, tol=0.0,
                         fine_theta=theta)
    else:
        p = synth.portfolio(n_k=1, n_s=2, M=M, N=N, fine_steps=6, coarse=synth.COARSE_IMPLICIT_EULER,
                            coarse_steps=1, max_iter=2, tol=0.0, fine_theta=theta)
    with ctx_for(p, fine_kernel=2) as c:
        _, rep = c.solve()
        it = c.copy_iterates(0, p.N + 1)
    ref_U, ref_d, K, _ = oracle.parareal(p)
    assert rep["iterations"] == K == 2
    assert_close(it, ref_U, what="persistent K2 M=%d N=%d B=%d" % (M, N, B))
    assert_delta(rep["delta"], ref_d)


def test_portfolio_parareal_sampled():
    """C4 layout (many instances, 64 factor sets) at reduced instance count; fixed K."""
    p = synth.portfolio(n_k=4, n_s=16, M=256, N=16, coarse=synth.COARSE_IMPLICIT_EULER, max_iter=3, tol=0.0)
    ref_U, ref_d, _, _ = oracle.parareal(p)
    with ctx_for(p) as c:
        U, rep = c.solve()
    assert_close(U, ref_U[-1], what="portfolio U_N")
    assert_delta(rep["delta"], ref_d)


def test_homogeneity_c4_full_sampled():
    """Full C4 size (4096 instances): sampled instances against single-instance oracle runs."""
    p = synth.config("C4", coarse=synth.COARSE_IMPLICIT_EULER, max_iter=2, tol=0.0)
    with ctx_for(p) as c:
        U, rep = c.solve()
    assert rep["iterations"] == 2
    for b in (0, 777, 2048, 4095):
        pb = p.replace(strike=p.strike[b:b + 1], sigma=p.sigma[b:b + 1], rate=p.rate[b:b + 1], L=p.L[b:b + 1])
        ref = oracle.parareal(pb)[0][-1, 0]
        assert_close(U[b:b + 1], ref[None], what="C4 instance %d" % b)


def test_device_entry_points():
    """Device-pointer variants and a caller-bound workspace give the host-path results bitwise."""
    import torch
    p = synth.config("C2", coarse=synth.COARSE_IMPLICIT_EULER, max_iter=2, tol=0.0)
    with ctx_for(p) as c:
        ws = torch.empty(c.workspace_bytes(), dtype=torch.uint8, device="cuda")
        c.bind_workspace(ws)
        out = torch.empty((1, p.M), dtype=torch.float32, device="cuda")
        rep = c.solve_device(out)
        dev = out.cpu().numpy()
        host, rep2 = c.solve()
        ms = c.serial_fine_device(out)
        sf_dev = out.cpu().numpy()
        sf_host, _ = c.serial_fine()
        v0 = c.initial_state()
    assert rep["iterations"] == 2 and ms > 0
    assert np.array_equal(dev, host) and np.array_equal(sf_dev, sf_host)
    assert np.array_equal(v0, oracle.payoff(p).astype(np.float32))


@pytest.mark.parametrize("name,M,N,B,theta,dims,act,K", [
    ("C1", 64, 4, 1, 1.0, synth.PINN_3x20, synth.ACT_TANH, 3), ("C2", 1024, 32, 1, 1.0, synth.PINN_3x20, synth.ACT_TANH, 3),
    ("C2", 1024, 32, 1, 0.5, synth.PINN_3x20, synth.ACT_TANH, 3), ("portfolio", 256, 8, 6, 1.0, synth.PINN_3x20, synth.ACT_TANH, 3),
    ("odd", 700, 12, 1, 1.0, synth.PINN_3x20, synth.ACT_TANH, 3),
    ("C2 paper net", 1024, 32, 1, 1.0, synth.PINN_PAPER, synth.ACT_RELU, 3),
    ("paper net tanh", 300, 8, 2, 1.0, synth.PINN_PAPER, synth.ACT_TANH, 3),
    ("C2 K=8: chain CTAs reused (k, k+2, ...)", 1024, 32, 1, 1.0, synth.PINN_3x20, synth.ACT_TANH, 8),
    ("C2 paper net K=8", 1024, 32, 1, 1.0, synth.PINN_PAPER, synth.ACT_RELU, 8)])
def test_pipelined_matches_blocking(name, M, N, B, theta, dims, act, K):
    """PR_OPT_PIPELINE (NEXT-2): the overlapped single-kernel schedule gives the blocking
    schedule's iterates, output and δ bitwise (and is the one auto mode takes here), with the
    latency-mode chain (3x20) and the one-thread-per-point chain (the paper's 10x50 net); K = 8
    runs several chains on each chain CTA (sets of iterations k ≡ s mod 2)."""
    if B > 1:
        p = synth.portfolio(n_k=B // 2 if B > 2 else 1, n_s=3 if B > 2 else 2, M=M, N=N, coarse=synth.COARSE_PINN,
                            max_iter=K, tol=0.0)
    else:
        p = synth.single(M, N, coarse=synth.COARSE_PINN, max_iter=K, tol=0.0, fine_theta=theta)
    net = synth.kaiming_net(dims, seed=2, activation=act)
    with ctx_for(p, net) as c:
        a, ra = c.solve()
        it_a = c.copy_iterates(0, p.N + 1)
        c.set_option(parareal.OPT_PIPELINE, 1)
        b, rb = c.solve()
        it_b = c.copy_iterates(0, p.N + 1)
    assert ra["kernel_launches"] < rb["kernel_launches"], "auto mode did not pipeline"
    assert ra["iterations"] == rb["iterations"] == K
    assert np.array_equal(a, b) and np.array_equal(it_a, it_b)
    assert np.array_equal(ra["delta"], rb["delta"])


def test_pipelined_grid_changes_within_one_context():
    """The pipelined kernel's tail (grid barrier, δ reduction, flag reset) leaves its buffers clean
    for the next launch even when that launch has another grid: one context alternates the
    latency-mode 3x20 chain (4-warp chain CTAs) and the paper's 10x50 net (12-warp chain CTAs,
    another CTA count); every pipelined solve equals the blocking solve of the same net bitwise."""
    p = synth.single(1024, 32, coarse=synth.COARSE_PINN, max_iter=3, tol=0.0)
    nets = [synth.kaiming_net(synth.PINN_3x20, seed=2), synth.kaiming_net(synth.PINN_PAPER, seed=2, activation=synth.ACT_RELU)]
    with ctx_for(p, nets[0]) as c:
        for i in (0, 1, 0, 1, 1, 0):
            c.load_weights(nets[i])
            c.set_option(parareal.OPT_PIPELINE, 0)
            a, ra = c.solve()
            c.set_option(parareal.OPT_PIPELINE, 1)
            b, rb = c.solve()
            assert ra["kernel_launches"] < rb["kernel_launches"], "auto mode did not pipeline"
            assert np.array_equal(a, b) and np.array_equal(ra["delta"], rb["delta"])


def test_graph_replay_matches_eager():
    """PR_OPT_USE_GRAPHS: captured + replayed solves give the eager results bitwise, replays
    are repeatable, and new weights are picked up (the graph is re-captured)."""
    import torch
    p = synth.config("C2", coarse=synth.COARSE_PINN, max_iter=3, tol=0.0)
    net0, net1 = synth.kaiming_net(synth.PINN_3x20, seed=0), synth.kaiming_net(synth.PINN_3x20, seed=3)
    out = None
    with ctx_for(p, net0) as c:
        out = torch.empty((1, p.M), dtype=torch.float32, device="cuda")
        c.solve_device(out)
        eager = out.cpu().numpy()
        c.set_option(parareal.OPT_USE_GRAPHS, 1)
        reps = []
        for _ in range(3):
            out.zero_()
            reps.append(c.solve_device(out))
            assert np.array_equal(out.cpu().numpy(), eager)
        assert all(r["iterations"] == 3 and r["ms_total"] > 0 for r in reps)
        c.load_weights(net1)
        out.zero_()
        c.solve_device(out)
        g1 = out.cpu().numpy()
        c.set_option(parareal.OPT_USE_GRAPHS, 0)
        c.solve_device(out)
        assert np.array_equal(out.cpu().numpy(), g1) and not np.array_equal(g1, eager)
        # lean stream-ordered replays (no timing nodes; the call returns once enqueued)
        c.set_option(parareal.OPT_USE_GRAPHS, 2)
        for _ in range(3):
            out.zero_()
            r = c.solve_device(out)
            torch.cuda.synchronize()
            assert r["iterations"] == 3 and r["kernel_launches"] > 0
            assert np.array_equal(out.cpu().numpy(), g1)


def test_errors_on_gpu():
    p = synth.config("C1", coarse=synth.COARSE_PINN)
    with parareal.Context(p) as c:
        with pytest.raises(parareal.PararealError) as ei:
            c.solve()
        assert ei.value.status == 5   # no weights loaded
        with pytest.raises(parareal.PararealError):
            c.load_weights(synth.kaiming_net([4, 20, 30, 1]))   # unequal hidden widths
        with pytest.raises(parareal.PararealError) as ei:
            c.load_weights(synth.kaiming_net([4, 24, 24, 1]))   # width not instantiated
        assert ei.value.status == 7
        with pytest.raises(parareal.PararealError):
            c.apply_fine(99, np.zeros((1, 64), np.float32))


def test_pipeline_falls_back_when_not_co_resident():
    """The pipelined kernel needs every CTA co-resident: the paper's 10x50 net on two C2 instances
    needs 2 chain sets x 2 instances x 29 twelve-warp CTAs + 2 x 32 fine CTAs = 180 > 148 SMs, so
    auto mode must run the blocking schedule (same launches as PR_OPT_PIPELINE=1) and give its
    results bitwise."""
    p = synth.portfolio(n_k=1, n_s=2, M=1024, N=32, coarse=synth.COARSE_PINN, max_iter=8, tol=0.0)
    net = synth.kaiming_net(synth.PINN_PAPER, seed=4)
    with ctx_for(p, net) as c:
        a, ra = c.solve()
        c.set_option(parareal.OPT_PIPELINE, 1)
        b, rb = c.solve()
    assert ra["kernel_launches"] == rb["kernel_launches"], "auto mode should have fallen back"
    assert ra["iterations"] == rb["iterations"] == 8
    assert np.array_equal(a, b) and np.array_equal(ra["delta"], rb["delta"])


@pytest.mark.parametrize("M,N,B,theta,nc", [(1024, 32, 1, 1.0, 1), (1024, 32, 1, 1.0, 50), (1024, 32, 1, 0.5, 1),
                                           (700, 12, 1, 1.0, 3), (256, 8, 6, 1.0, 1), (64, 4, 1, 1.0, 1)])
def test_pipelined_numerical_G_matches_blocking(M, N, B, theta, nc):
    """NEXT-2 with the numerical coarse propagator (implicit Euler, n_c steps): one K1
    chain system per iteration runs beside the fine solves in the cooperative kernel; iterates,
    output and δ are bitwise the blocking schedule's, which the oracle check of the blocking
    path (test_parareal_*) covers; here also the final state against the oracle."""
    if B > 1:
        p = synth.portfolio(n_k=B // 2, n_s=2, M=M, N=N, coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=nc,
                            max_iter=3, tol=0.0)
    else:
        p = synth.single(M, N, coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=nc, max_iter=min(3, N), tol=0.0,
                         fine_theta=theta)
    with ctx_for(p) as c:
        a, ra = c.solve()
        it_a = c.copy_iterates(0, p.N + 1)
        c.set_option(parareal.OPT_PIPELINE, 1)
        b, rb = c.solve()
        it_b = c.copy_iterates(0, p.N + 1)
    assert ra["kernel_launches"] < rb["kernel_launches"], "auto mode did not pipeline"
    assert ra["iterations"] == rb["iterations"] == p.max_iter
    assert np.array_equal(a, b) and np.array_equal(it_a, it_b)
    assert np.array_equal(ra["delta"], rb["delta"])
    U_ref = oracle.parareal(p)[0]
    assert_close(a, U_ref[-1], what="pipelined numerical-G Parareal M=%d" % M)


def test_graph_replay_with_pinned_host_buffers():
    """PR_OPT_USE_GRAPHS with host buffers: pinned ones are captured as graph copy nodes (the
    bench's e2e path), pageable ones run eagerly; every result is the eager solve's, bitwise."""
    import torch
    p = synth.config("C2", coarse=synth.COARSE_PINN, max_iter=3, tol=0.0)
    net = synth.kaiming_net(synth.PINN_3x20, seed=5)
    with ctx_for(p, net) as c:
        eager, _ = c.solve()
        vt = torch.from_numpy(c.initial_state()).pin_memory()
        v0 = torch.zeros((p.B, p.M), dtype=torch.float32).pin_memory()
        for mode in (1, 2):
            c.set_option(parareal.OPT_USE_GRAPHS, mode)
            launches = []
            for _ in range(3):
                v0.zero_()
                r = c.solve_host_ptrs(vt.data_ptr(), v0.data_ptr())   # returns with V_0 written
                launches.append(r["kernel_launches"])
                assert np.array_equal(v0.numpy(), eager)
            assert r["iterations"] == 3 and launches[0] == launches[-1] > 0
        c.set_option(parareal.OPT_USE_GRAPHS, 1)
        again, _ = c.solve()   # pageable buffers: eager
        assert np.array_equal(again, eager)


# ------------------------------------------------------------------ the configurations the bench reports
# (VERDICT r01 "What's weak" 1-2: the exact headline configuration and the C3-scale K2 kernel)

def _k2_lookback_windows(M, sigma, r, dtau):
    """Largest look-back window (in predecessor tiles) of the K2 passes for this grid, computed
    here from a plain fp64 factorisation of I - dτA: the number of predecessor tiles
    whose multiplier product stays above 1e-24 (fine_streamed.cuh kLookbackEps), per direction."""
    j = np.arange(1, M + 1, dtype=np.float64)
    a, b = 0.5 * sigma ** 2 * j ** 2, 0.5 * r * j
    d, lo, up = 1.0 + dtau * (2 * a + r), -dtau * (a - b), -dtau * (a + b)
    p = np.empty(M)
    p[0] = d[0]
    for i in range(1, M):
        p[i] = d[i] - lo[i] / p[i - 1] * up[i - 1]
    mt = np.concatenate([[0.0], lo[1:] / p[1:]])
    cu = np.concatenate([up[:-1] / p[:-1], [0.0]])
    T = 2048
    nt = (M + T - 1) // T
    best = 0
    for f in (mt, cu):
        lt = np.array([np.sum(np.log(np.abs(f[t * T:(t + 1) * T]) + 1e-300)) for t in range(nt)])
        for pos in range(nt):
            acc, w = 0.0, pos
            for k in range(1, pos + 1):
                acc += lt[pos - k] if f is mt else lt[nt - 1 - (pos - k)]
                if acc < np.log(1e-24):
                    w = k
                    break
            best = max(best, w)
    return best


def test_headline_bench_config_matches_oracle():
    """The exact bench.py default step: C2 (1024 x 32 slices, 100 IE steps), PINN 3x20 tanh seed 0,
    fixed K = 3, auto schedule (the pipelined cooperative kernel), workspace bound by the caller,
    lean graph capture + stream-ordered replays (PR_OPT_USE_GRAPHS = 2) on a caller stream -- every
    iterate U^3_n against the oracle (Eq. 7) under the stability gate of SURVEY §8(c),
    and K, δ from an instrumented solve of the same context."""
    import torch
    p = synth.config("C2", coarse=synth.COARSE_PINN, coarse_steps=1, tol=0.0, fine_theta=1.0).replace(max_iter=3)
    net = synth.kaiming_net(synth.PINN_3x20, seed=0)
    ref_U, ref_d, ref_K, _ = oracle.parareal(p, net)
    U32, _, _, _ = oracle.parareal(p, net, prec=32)
    stream = torch.cuda.Stream()
    with parareal.Context(p, stream=stream.cuda_stream) as c:
        c.load_weights(net)
        ws = torch.empty(c.workspace_bytes(), dtype=torch.uint8, device="cuda")
        c.bind_workspace(ws)
        c.set_option(parareal.OPT_USE_GRAPHS, 2)
        out = torch.empty((p.B, p.M), dtype=torch.float32, device="cuda")
        with torch.cuda.stream(stream):
            for _ in range(4):                     # capture, then replays (as the timed loop)
                out.zero_()
                rep = c.solve_device(out)
            stream.synchronize()
        U = out.cpu().numpy()
        it = c.copy_iterates(0, p.N + 1)
        assert rep["iterations"] == ref_K == 3
        c.set_option(parareal.OPT_PIPELINE, 1)
        _, rb = c.solve()                          # the blocking schedule's launch count
        c.set_option(parareal.OPT_PIPELINE, 0)
        c.set_option(parareal.OPT_USE_GRAPHS, 0)
        _, ra = c.solve()                          # instrumented: δ history
    assert rep["kernel_launches"] < rb["kernel_launches"], "the bench step did not run the pipelined kernel"
    assert np.array_equal(U, it[-1])
    _gate_or_amplification(it, ref_U, U32, "headline C2 iterates")
    assert ra["iterations"] == 3
    assert_delta(ra["delta"], ref_d)


def test_k2_persistent_pass_long_lookback():
    """k_pass_res2 (>= 16 systems) on a grid whose look-back windows exceed 32 and 64 predecessor
    tiles (the prefetched second window and the > 64 fallback of fine_streamed.cuh): 2^18 points,
    dτ = 1/96, 16 slices of 6 IE steps, one Parareal iteration with numerical G -- every iterate
    against the oracle."""
    M, N, nf = 1 << 18, 16, 6
    p = synth.single(M, N, fine_steps=nf, coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=1, max_iter=1, tol=0.0)
    W = _k2_lookback_windows(M, 0.2, 0.05, 1.0 / (N * nf))
    assert W > 64, W
    with ctx_for(p, fine_kernel=2) as c:
        _, rep = c.solve()
        it = c.copy_iterates(0, p.N + 1)
    ref_U, ref_d, K, _ = oracle.parareal(p)
    assert rep["iterations"] == K == 1
    assert_close(it, ref_U, what="K2 long look-back M=2^18")
    assert_delta(rep["delta"], ref_d)


@pytest.mark.parametrize("kernel", [2, 3])
def test_c3_grid_fine_sweep_persistent(kernel):
    """The C3 grid (2^20 points, the C3 step dτ = 1/6400) on the persistent K2 kernel (2) and on
    the grid-resident kernel (3): 16 slices of 2 steps, one Parareal iteration with numerical G --
    all 17 boundary states (about 17 M values) against the oracle."""
    M, N, nf = 1 << 20, 16, 2
    p = synth.single(M, N, fine_steps=nf, coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=1, max_iter=1, tol=0.0,
                     T=N * nf / 6400.0)
    with ctx_for(p, fine_kernel=kernel) as c:
        _, rep = c.solve()
        it = c.copy_iterates(0, p.N + 1)
    ref_U, ref_d, K, _ = oracle.parareal(p)
    assert rep["iterations"] == K == 1
    assert_close(it, ref_U, what="C3-grid Parareal iterate")
    assert_delta(rep["delta"], ref_d)



# ------------------------------------------------------------------ K2R grid-resident fine solver
# (fine_grid.cu: one system spans the GPU, state in registers for all passes, LU/UL zig-zag)

@pytest.mark.parametrize("M,N,n,nf", [(2049, 4, 0, 3), (3000, 4, 1, 10), (5000, 8, 3, 7), (70000, 4, 2, 5),
                                      (1 << 18, 4, 1, 6)])
def test_grid_fine_single_slice(M, N, n, nf):
    """One F application (n_f IE steps) on the grid-resident kernel against the oracle: ragged last
    CTA (2049, 3000, 70000), several CTAs and look-back windows, the 2^18 C5 grid."""
    p = synth.single(M, N, fine_steps=nf)
    U = synth.random_state(1, M, seed=M + n)
    with ctx_for(p, fine_kernel=3) as c:
        got = c.apply_fine(n, U)
    assert_close(got, oracle.fine(p, n, U.astype(np.float64)), what="grid F M=%d" % M)


@pytest.mark.parametrize("M,N,K", [(3000, 6, 3), (5000, 9, 2), (40000, 4, 4)])
def test_grid_parareal_iterates(M, N, K):
    """Parareal with numerical G on the grid-resident fine kernel: every iterate against the
    oracle; odd slice counts leave a group with one live system; K = N (finite termination)."""
    p = synth.single(M, N, fine_steps=8, coarse=synth.COARSE_IMPLICIT_EULER, max_iter=K, tol=0.0)
    with ctx_for(p, fine_kernel=3) as c:
        _, rep = c.solve()
        it = c.copy_iterates(0, p.N + 1)
        again, _ = c.solve()
        it2 = c.copy_iterates(0, p.N + 1)
    ref_U, ref_d, Kr, _ = oracle.parareal(p)
    assert rep["iterations"] == Kr == K
    assert_close(it, ref_U, what="grid Parareal M=%d" % M)
    assert_delta(rep["delta"], ref_d)
    assert np.array_equal(it, it2)  # run-to-run bitwise (fixed composition orders)


def test_grid_serial_fine_matches_oracle():
    """The serial fine solve (the speedup baseline) runs one grid-resident solve per slice for
    M > 2048: against the oracle's serial fine solution."""
    p = synth.single(6000, 8, fine_steps=12)
    with ctx_for(p) as c:
        got, _ = c.serial_fine()
    assert_close(got, oracle.serial_fine(p)[-1], what="grid serial fine")
