"""Multi-rank host logic on CPU (gloo, world_size 2 and 4).

The CUDA path shards the N slices across ranks; the per-rank schedule it runs
(parareal_plan_iteration, the product's own host code) is checked here:
  * pure invariants over many (N, world, k);
  * executed by real processes exchanging slice-boundary states with gloo
    send/recv and a MAX all-reduce of delta, using the CPU oracle's propagators
    for F and G -- the result must be bitwise identical to the single-process
    oracle (the R-invariance claim of SURVEY.md §8(e));
  * the NCCL unique-id broadcast used by bench.py.
"""
import os
import socket

import numpy as np
import pytest

from paper_2303_03848_b200 import parareal, synth


@pytest.mark.parametrize("N,world", [(1, 1), (4, 1), (4, 2), (4, 4), (32, 8), (64, 8), (12, 3), (16, 16)])
def test_plan_invariants(N, world):
    per = N // world
    for k in range(0, N + 1):
        plans = [parareal.plan_iteration(N, world, r, k) for r in range(world)]
        fine, chain, delta, copies = set(), [], set(), 0
        for r, P in enumerate(plans):
            n0 = r * per
            fine |= {n0 + l for l in range(P["fine_lo"], P["fine_hi"])}
            chain += [n0 + l for l in range(P["chain_lo"], P["chain_hi"]) if (P["copy"] or P["recv_first"] or k == 0)]
            delta |= {n0 + l for l in range(P["delta_lo"], P["delta_hi"] + 1)}
            copies += P["copy"]
            if P["fk_local"] >= 0:
                assert n0 + P["fk_local"] == k - 1
            # hand-off symmetry: r sends iff r+1 receives
            if r < world - 1:
                assert P["send_last"] == plans[r + 1]["recv_first"], (N, world, k, r)
            else:
                assert P["send_last"] == 0
        if k == 0:
            assert chain == list(range(N)) and not fine and not delta
            continue
        assert fine == set(range(k - 1, N))                         # active window
        assert sorted(chain) == list(range(k, N))                    # each G slice once
        assert delta == set(range(k, N + 1))                         # delta over n = k..N (Q13)
        assert copies == (1 if k <= N else 0)


def test_plan_rejects_bad_arguments():
    for args in [(0, 1, 0, 0), (4, 3, 0, 1), (4, 2, 2, 1), (4, 2, 0, -1)]:
        with pytest.raises(parareal.PararealError):
            parareal.plan_iteration(*args)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, cfg, coarse, K, out_q, chunks=1):
    import torch
    import torch.distributed as dist

    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = synth.config(cfg, coarse=coarse, coarse_steps=1, max_iter=K, tol=0.0)
        net = synth.kaiming_net(synth.PINN_3x20, seed=0)
        N, B, M = p.N, p.B, p.M
        per = N // world
        n0 = rank * per

        def G(n, u):
            return oracle.pinn_G(p, net, n, u) if coarse == synth.COARSE_PINN else oracle.coarse_ie(p, n, u)

        U = np.zeros((per + 1, B, M))
        Gh = np.zeros((per, B, M))
        D = np.zeros((per, B, M))
        if rank == 0:
            U[0] = oracle.payoff(p)

        def recv0():
            t = torch.zeros(B * M, dtype=torch.float64)
            dist.recv(t, src=rank - 1)
            U[0] = t.numpy().reshape(B, M)

        def send_last():
            dist.send(torch.from_numpy(U[per].reshape(-1).copy()), dst=rank + 1)

        def chain(P, k, lo=0, hi=None):
            """G chain over local slices, grid points [lo, hi) only (G is pointwise in S)."""
            hi = M if hi is None else hi
            if k > 0 and P["copy"]:
                U[P["chain_lo"], :, lo:hi] = Fk[:, lo:hi]
            for l in range(P["chain_lo"], P["chain_hi"]):
                g = G(n0 + l, U[l])[:, lo:hi]
                U[l + 1, :, lo:hi] = g + D[l, :, lo:hi] if k > 0 else g
                Gh[l, :, lo:hi] = g

        def exchange(P, k, run):
            """The chain with its hand-offs: blocking, or the NEXT-2 wavefront of j-chunks (the
            product's PR_OPT_WAVEFRONT schedule: per chunk q, send chunk q-1 of U_{n1} and receive
            chunk q of U_{n0} as one group, chain chunk q; finally send the last chunk)."""
            if chunks <= 1:
                if P["recv_first"]:
                    recv0()
                if run:
                    chain(P, k)
                if P["send_last"]:
                    send_last()
                return
            bnd = [q * M // chunks for q in range(chunks + 1)]
            for q in range(chunks):
                reqs = []
                if q > 0 and P["send_last"]:
                    reqs.append(dist.isend(torch.from_numpy(U[per, :, bnd[q - 1]:bnd[q]].copy().reshape(-1)),
                                           dst=rank + 1))
                if P["recv_first"]:
                    t = torch.zeros(B * (bnd[q + 1] - bnd[q]), dtype=torch.float64)
                    reqs.append(dist.irecv(t, src=rank - 1))
                for rq in reqs:
                    rq.wait()
                if P["recv_first"]:
                    U[0, :, bnd[q]:bnd[q + 1]] = t.numpy().reshape(B, -1)
                if run:
                    chain(P, k, bnd[q], bnd[q + 1])
            if P["send_last"]:
                dist.send(torch.from_numpy(U[per, :, bnd[-2]:bnd[-1]].copy().reshape(-1)), dst=rank + 1)

        Fk = None
        P0 = parareal.plan_iteration(N, world, rank, 0)
        exchange(P0, 0, True)
        deltas = []
        for k in range(1, K + 1):
            P = parareal.plan_iteration(N, world, rank, k)
            Uold = U.copy()
            Fk = None
            for l in range(P["fine_lo"], P["fine_hi"]):
                Fh = oracle.fine(p, n0 + l, Uold[l])
                if l == P["fk_local"]:
                    Fk = Fh
                else:
                    D[l] = Fh - Gh[l]
            exchange(P, k, P["copy"] or P["recv_first"])
            dk = 0.0
            for l in range(P["delta_lo"], P["delta_hi"] + 1):
                for b in range(B):
                    num = np.sqrt(np.sum((U[l, b] - Uold[l, b]) ** 2))
                    den = np.sqrt(np.sum(U[l, b] ** 2))
                    dk = max(dk, num / den if den > 0 else num)
            t = torch.tensor([dk], dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            deltas.append(float(t.item()))
        # final state to rank 0
        if world > 1:
            if rank == world - 1:
                dist.send(torch.from_numpy(U[per].reshape(-1).copy()), dst=0)
            if rank == 0:
                t = torch.zeros(B * M, dtype=torch.float64)
                dist.recv(t, src=world - 1)
                final = t.numpy().reshape(B, M)
        else:
            final = U[per]
        if rank == 0:
            out_q.put((final, deltas))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,coarse,chunks", [(2, synth.COARSE_IMPLICIT_EULER, 1), (2, synth.COARSE_PINN, 1),
                                                 (4, synth.COARSE_IMPLICIT_EULER, 1), (2, synth.COARSE_PINN, 3),
                                                 (4, synth.COARSE_PINN, 5)])
def test_sharded_schedule_matches_serial_oracle(world, coarse, chunks):
    import torch.multiprocessing as mp

    import oracle
    cfg, K = "C1", 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, cfg, coarse, K, q, chunks)) for r in range(world)]
    for pr in procs:
        pr.start()
    final, deltas = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = synth.config(cfg, coarse=coarse, coarse_steps=1, max_iter=K, tol=0.0)
    net = synth.kaiming_net(synth.PINN_3x20, seed=0)
    U, d, Kr, _ = oracle.parareal(p, net)
    assert np.array_equal(final, U[-1])                 # bitwise: sharding does not change arithmetic
    assert np.allclose(deltas, d, rtol=1e-12, atol=0)


def _id_main(rank, world, port, out_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        obj = [parareal.get_nccl_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        out_q.put((rank, obj[0]))
    finally:
        dist.destroy_process_group()


def test_nccl_id_broadcast():
    """bench.py's rendezvous: rank 0 creates the NCCL id, every rank receives the same bytes."""
    import torch  # noqa: F401  (maps torch's libnccl.so.2 so dlopen finds it)
    try:
        parareal.get_nccl_id()
    except parareal.PararealError as e:
        pytest.skip("NCCL not loadable here: %s" % e)
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_id_main, args=(r, 2, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    got = dict(q.get(timeout=120) for _ in range(2))
    for pr in procs:
        pr.join(timeout=60)
    assert len(got[0]) == 128 and got[0] == got[1]


def _spatial_main(rank, world, port, K, out_q):
    """The NEXT-4 schedule (PR_OPT_SPATIAL_CHAIN) with the oracle's propagators: fine sweep sharded
    by slices, the PINN chain of every slice sharded by grid points, rows changing owner twice per
    iteration (gloo point-to-point), δ's per-slice sums added over ranks."""
    import torch
    import torch.distributed as dist

    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        p = synth.config("C1", coarse=synth.COARSE_PINN, max_iter=K, tol=0.0)
        net = synth.kaiming_net(synth.PINN_3x20, seed=0)
        N, M = p.N, p.M
        per = N // world
        jb = [q * M // world for q in range(world + 1)]
        lo, hi = jb[rank], jb[rank + 1]
        owner = lambda n: n // per
        Us = np.zeros((N + 1, M)); Ghs = np.zeros((N, M)); Ds = np.zeros((N, M)); Fs = np.zeros(M)
        U = np.zeros((N + 1, M)); Gh = np.zeros((N, M)); D = np.zeros((N, M)); Fk = None
        Us[0, lo:hi] = oracle.payoff(p)[0, lo:hi]

        def move(rows, src, dst, frm_owner):
            """rows: list of n.  frm_owner False: point owners → slice owner(n) (src sharded by
            points); True: slice owner(n) → point owners."""
            reqs, pend = [], []
            for n in rows:
                o = owner(min(n, N - 1))
                for q in range(world):
                    a, b = jb[q], jb[q + 1]
                    s_, d_ = (o, q) if frm_owner else (q, o)
                    if s_ == d_ == rank:
                        dst[n, a:b] = src[n, a:b]
                    elif s_ == rank:
                        reqs.append(dist.isend(torch.from_numpy(src[n, a:b].copy()), dst=d_))
                    elif d_ == rank:
                        t = torch.zeros(b - a, dtype=torch.float64)
                        reqs.append(dist.irecv(t, src=s_))
                        pend.append((n, a, b, t))
            for rq in reqs:
                rq.wait()
            for n, a, b, t in pend:
                dst[n, a:b] = t.numpy()

        def chain(k):
            if k > 0:
                Us[k, lo:hi] = Fs[lo:hi]
            for n in range(k, N):
                g = oracle.pinn_G(p, net, n, Us[n][None])[0, lo:hi]
                Us[n + 1, lo:hi] = g + Ds[n, lo:hi] if k > 0 else g
                Ghs[n, lo:hi] = g

        chain(0)
        deltas = []
        for k in range(1, K + 1):
            Uold = Us.copy()
            move(range(k - 1, N), Us, U, False)
            move(range(k - 1, N), Ghs, Gh, False)
            for n in range(max(k - 1, rank * per), (rank + 1) * per):
                Fh = oracle.fine(p, n, U[n][None])[0]
                if n == k - 1:
                    Fk = Fh
                else:
                    D[n] = Fh - Gh[n]
            if Fk is not None and owner(k - 1) == rank:
                Ftmp = np.zeros((N + 1, M)); Ftmp[k - 1] = Fk
            else:
                Ftmp = np.zeros((N + 1, M))
            move([k - 1], Ftmp, Ftmp, True)
            Fs[:] = Ftmp[k - 1]
            move(range(k, N), D, Ds, True)
            chain(k)
            num = np.array([np.sum((Us[n, lo:hi] - Uold[n, lo:hi]) ** 2) for n in range(k, N + 1)])
            den = np.array([np.sum(Us[n, lo:hi] ** 2) for n in range(k, N + 1)])
            t = torch.from_numpy(np.concatenate([num, den]))
            dist.all_reduce(t, op=dist.ReduceOp.SUM)
            nn, dd = t.numpy()[:N + 1 - k], t.numpy()[N + 1 - k:]
            deltas.append(float(np.max(np.sqrt(nn) / np.sqrt(dd))))
        # U_N: every rank's point range (zeros elsewhere), summed = gathered
        t = torch.from_numpy(np.where((np.arange(M) >= lo) & (np.arange(M) < hi), Us[N], 0.0))
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        final = t.numpy()
        if rank == 0:
            out_q.put((final, deltas))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_spatial_chain_schedule_matches_serial_oracle(world):
    import torch.multiprocessing as mp

    import oracle
    K = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_spatial_main, args=(r, world, port, K, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    final, deltas = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    p = synth.config("C1", coarse=synth.COARSE_PINN, max_iter=K, tol=0.0)
    U, d, _, _ = oracle.parareal(p, synth.kaiming_net(synth.PINN_3x20, seed=0))
    assert np.array_equal(final, U[-1][0])               # G pointwise: sharding points changes no arithmetic
    assert np.allclose(deltas, d, rtol=1e-12, atol=0)    # (δ's sums are split over ranks: rounding only)
