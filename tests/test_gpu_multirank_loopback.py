"""The multi-rank schedule on one GPU: R contexts in one process, one host
thread each, exchanging through the library's in-process loopback transport (a 128-byte id
starting "PRLOOPBK") instead of NCCL.  Everything else is the multi-GPU path — per-rank plan,
kernels, the U_{n0} receive / U_{n1} send around each coarse chain, the MAX all-reduce of δ that
decides the stop, the gather of U_N to rank 0 — so this executes it on real kernels.  The results
must be bitwise the one-rank solve's: every slice's arithmetic is independent of R and MAX is
order-free."""
import threading

import numpy as np
import pytest

from paper_2303_03848_b200 import parareal, synth

pytestmark = pytest.mark.gpu


def solve_ranks(p, net, world, key, opts=None, precision=parareal.PREC_FP32):
    nid = b"PRLOOPBK" + key.ljust(120, b"\0")
    ctxs = [parareal.Context(p, rank=r, world=world, device=0, nccl_id=nid) for r in range(world)]
    try:
        for c in ctxs:
            if net is not None:
                c.load_weights(net, precision=precision)
            for k, v in (opts or {}).items():
                c.set_option(k, v)
        outs, reps, its, errs = [None] * world, [None] * world, [None] * world, []

        def work(r):
            try:
                outs[r], reps[r] = ctxs[r].solve()
                n0 = r * (p.N // world)
                its[r] = ctxs[r].copy_iterates(n0, p.N // world + 1)
            except Exception as e:  # pragma: no cover - reported below
                errs.append((r, e))

        th = [threading.Thread(target=work, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join(timeout=120)
        assert not any(t.is_alive() for t in th), "loopback ranks deadlocked"
        assert not errs, errs
        return outs[0], reps, its
    finally:
        for c in ctxs:
            c.close()


@pytest.mark.parametrize("name,world", [("pinn", 2), ("pinn", 4), ("ie", 2), ("ie_tol", 2), ("ie_tol", 4),
                                        ("streamed", 2), ("portfolio", 2)])
def test_multirank_matches_one_rank(name, world):
    # (the loopback ranks share one GPU and never run the cooperative grid-resident fine kernel:
    # problems that would use it pin K2 on every side)
    net, opts = None, {}
    if name == "pinn":
        p = synth.single(1024, 32, coarse=synth.COARSE_PINN, max_iter=3, tol=0.0)
        net = synth.kaiming_net(synth.PINN_3x20, seed=1)
    elif name == "ie":
        p = synth.single(700, 8, coarse=synth.COARSE_IMPLICIT_EULER, max_iter=3, tol=0.0)
    elif name == "ie_tol":  # C1 with numerical G: K = 3 at tol = 3e-5, decided by the all-reduced δ
        p = synth.config("C1", coarse=synth.COARSE_IMPLICIT_EULER, max_iter=4, tol=3e-5)
    elif name == "streamed":  # K2 fine sweeps and the streamed numerical chain
        p = synth.single(5000, 4, coarse=synth.COARSE_IMPLICIT_EULER, max_iter=2, tol=0.0, fine_steps=20)
        opts = {parareal.OPT_FINE_KERNEL: 2}
    else:
        p = synth.portfolio(n_k=2, n_s=2, M=256, N=8, coarse=synth.COARSE_PINN, max_iter=3, tol=0.0)
        net = synth.kaiming_net(synth.PINN_3x20, seed=2)
    with parareal.Context(p) as c:
        if net is not None:
            c.load_weights(net)
        c.set_option(parareal.OPT_PIPELINE, 1)  # the blocking schedule (multi-rank runs blocking)
        for k, v in opts.items():
            c.set_option(k, v)
        ref, rref = c.solve()
        it_ref = c.copy_iterates(0, p.N + 1)
    out, reps, its = solve_ranks(p, net, world, ("%s-%d" % (name, world)).encode(), opts)
    assert all(r["iterations"] == rref["iterations"] for r in reps)
    assert np.array_equal(reps[0]["delta"], rref["delta"])
    assert np.array_equal(out, ref)
    per = p.N // world
    for r in range(world):
        assert np.array_equal(its[r], it_ref[r * per:(r + 1) * per + 1]), "rank %d iterates" % r


@pytest.mark.parametrize("case,world,chunks", [("c2", 2, 3), ("c2", 4, 5), ("c2", 4, 64), ("big", 2, 0), ("big", 4, 0),
                                               ("tc", 2, 3)])
def test_chain_wavefront_matches_one_rank(case, world, chunks):
    """NEXT-2 across ranks: the PINN chain as a wavefront of j-chunks (PR_OPT_WAVEFRONT; 0 = auto,
    8 chunks at M >= 65536).  Every chunk is a CTA range of the same kernel, so output, every
    rank's iterates and δ are bitwise the one-rank (and the blocking multi-rank) solve's."""
    prec = parareal.PREC_FP32
    if case == "c2":
        p = synth.single(1024, 32, coarse=synth.COARSE_PINN, max_iter=3, tol=0.0)
        net = synth.kaiming_net(synth.PINN_3x20, seed=1)
    elif case == "big":
        p = synth.single(1 << 16, 8, coarse=synth.COARSE_PINN, max_iter=2, tol=0.0, fine_steps=4)
        net = synth.kaiming_net(synth.PINN_3x20, seed=3)
    else:  # tensor-core chain (K4, split fp16)
        p = synth.single(3000, 8, coarse=synth.COARSE_PINN, max_iter=2, tol=0.0, fine_steps=10)
        net, prec = synth.kaiming_net([4, 64, 64, 64, 1], seed=4), parareal.PREC_FP16_TC
    fk = {parareal.OPT_FINE_KERNEL: 2} if p.M > 2048 else {}  # (no grid-resident kernel in loopback)
    with parareal.Context(p) as c:
        c.load_weights(net, precision=prec)
        c.set_option(parareal.OPT_PIPELINE, 1)
        for k, v in fk.items():
            c.set_option(k, v)
        ref, rref = c.solve()
        it_ref = c.copy_iterates(0, p.N + 1)
    key = ("wave-%s-%d-%d" % (case, world, chunks)).encode()
    off = {parareal.OPT_SPATIAL_CHAIN: 1, **fk}  # (auto would shard the TC chain spatially instead)
    out, reps, its = solve_ranks(p, net, world, key, {**off, parareal.OPT_WAVEFRONT: chunks}, prec)
    _, breps, _ = solve_ranks(p, net, world, key + b"b", {**off, parareal.OPT_WAVEFRONT: 1}, prec)
    assert np.array_equal(out, ref)
    assert np.array_equal(reps[0]["delta"], rref["delta"])
    per = p.N // world
    for r in range(world):
        assert np.array_equal(its[r], it_ref[r * per:(r + 1) * per + 1]), "rank %d iterates" % r
    # the wavefront really ran: more (chunked) chain launches than the blocking schedule
    assert reps[-1]["kernel_launches"] > breps[-1]["kernel_launches"]


@pytest.mark.parametrize("case,world", [("c2", 2), ("c2", 4), ("tc", 2), ("tc", 4), ("tol", 2), ("kN", 4)])
def test_spatial_chain_matches_one_rank(case, world):
    """NEXT-4: the spatially sharded coarse chain (PR_OPT_SPATIAL_CHAIN; every rank chains all
    slices over its own point range, the fine sweep stays slice-sharded, rows change owner twice
    per iteration, δ slots summed over ranks).  Output, every rank's iterates, δ and K are bitwise
    the one-rank solve's; "tc" runs the auto choice (on for tensor-core nets)."""
    prec, opts = parareal.PREC_FP32, {parareal.OPT_SPATIAL_CHAIN: 2}
    if case == "c2":
        p = synth.single(1024, 32, coarse=synth.COARSE_PINN, max_iter=3, tol=0.0)
        net = synth.kaiming_net(synth.PINN_3x20, seed=1)
    elif case == "tc":
        p = synth.single(3000, 8, coarse=synth.COARSE_PINN, max_iter=3, tol=0.0, fine_steps=10)
        net, prec, opts = synth.kaiming_net([4, 128, 128, 128, 1], seed=4), parareal.PREC_FP16_TC, {}
    elif case == "tol":  # a tolerance: the stop is decided from the δ every rank reduces from the summed slots
        p = synth.single(256, 8, coarse=synth.COARSE_PINN, max_iter=8, tol=1e-3, fine_steps=10)
        net = synth.kaiming_net([4, 16, 16, 1], seed=7)
    else:  # K = N: the last iteration's chain is the copy step alone (finite termination)
        p = synth.single(200, 4, coarse=synth.COARSE_PINN, max_iter=4, tol=0.0, fine_steps=7)
        net = synth.kaiming_net([4, 8, 8, 1], seed=8)
    if p.M > 2048:
        opts = {**opts, parareal.OPT_FINE_KERNEL: 2}  # (no grid-resident kernel in loopback)
    with parareal.Context(p) as c:
        c.load_weights(net, precision=prec)
        c.set_option(parareal.OPT_PIPELINE, 1)
        for k, v in opts.items():
            if k == parareal.OPT_FINE_KERNEL:
                c.set_option(k, v)
        ref, rref = c.solve()
        it_ref = c.copy_iterates(0, p.N + 1)
    out, reps, its = solve_ranks(p, net, world, ("spatial-%s-%d" % (case, world)).encode(), opts, prec)
    assert all(r["iterations"] == rref["iterations"] for r in reps)
    assert np.array_equal(out, ref)
    for r in reps:
        assert np.array_equal(r["delta"], rref["delta"])
    per = p.N // world
    for r in range(world):
        assert np.array_equal(its[r], it_ref[r * per:(r + 1) * per + 1]), "rank %d iterates" % r
