"""Host-side pieces: synthetic inputs, weight blob, speedup bounds (no GPU)."""
import os

import numpy as np
import pytest

from paper_2303_03848_b200 import report, synth


def test_speedup_bound_golden(golden):
    g = golden("spec_examples.json")["speedup_bound"]
    for c in g["cases"]:
        assert report.speedup_bound(c["K"], c["P"], c["ratio"]) == pytest.approx(c["s"], rel=1e-6), g["cite"]


def test_speedup_bound_is_pipelined_cost_model():
    """Eq. (8) equals P c_f / ((P+K) c_c + K c_f) (Q19) and dominates the blocking bound."""
    for K, P, cc, cf in [(3, 16, 1.0, 40.0), (2, 8, 0.3, 1.0), (5, 64, 2.0, 3.0)]:
        assert report.speedup_bound(K, P, cc / cf) == pytest.approx(P * cf / ((P + K) * cc + K * cf), rel=1e-12)
        assert report.speedup_bound_blocking(K, P, cc / cf) <= report.speedup_bound(K, P, cc / cf)


def test_kaiming_statistics():
    """empirical weight variance within 10% of 2/fan_in; deterministic per seed."""
    net = synth.kaiming_net([50] * 12, seed=4)
    w = np.concatenate([W.ravel() for W in net.W])
    assert abs(w.var() / (2.0 / 50) - 1.0) < 0.1
    net2 = synth.kaiming_net([50] * 12, seed=4)
    assert all(np.array_equal(a, b) for a, b in zip(net.W, net2.W))
    assert all(np.all(np.abs(b) <= 1 / np.sqrt(50)) for b in net.b)


def test_blob_roundtrip(tmp_path):
    net = synth.kaiming_net(synth.PINN_3x20, seed=2, in_scale=[1, 2, 3, 4], out_scale=0.5)
    path = os.path.join(tmp_path, "w.bin")
    synth.save_blob(net, path)
    back = synth.load_blob(path)
    assert back.dims == net.dims and back.activation == net.activation and back.out_scale == 0.5
    assert np.array_equal(back.scales(), net.scales())
    for a, b in zip(net.W + net.b, back.W + back.b):
        assert np.array_equal(a, b)


def test_configs_match_baseline():
    c = {k: synth.config(k) for k in ("C1", "C2", "C3", "C4", "C5")}
    assert (c["C1"].M, c["C1"].N) == (64, 4)
    assert (c["C2"].M, c["C2"].N) == (1024, 32)
    assert (c["C3"].M, c["C3"].N) == (1 << 20, 64)
    assert (c["C4"].M, c["C4"].N, c["C4"].B) == (256, 16, 4096)
    assert np.allclose(c["C4"].L, 4 * c["C4"].strike)
    assert (c["C5"].M, c["C5"].N) == (1 << 18, 64)
    for p in c.values():
        assert p.fine_steps == 100 and p.fine_theta == 1.0 and p.T == 1.0


def test_oracle_threaded_fine_is_bitwise_serial():
    """The threaded-fine CPU baseline: slices of each fine sweep on std::threads give
    exactly the serial oracle's iterates and deltas (each slice is the same code on its own data)."""
    import oracle
    for cfg in (dict(coarse=synth.COARSE_PINN), dict(coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=2)):
        p = synth.single(64, 7, max_iter=3, tol=0.0, **cfg)
        net = synth.kaiming_net(synth.PINN_3x20, seed=4) if cfg["coarse"] == synth.COARSE_PINN else None
        a = oracle.parareal(p, net, history=True)
        b = oracle.parareal(p, net, history=True, threads=3)
        assert a[2] == b[2] and np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1]) and np.array_equal(a[3], b[3])


def test_instance_sharding_covers_and_matches_the_oracle():
    """C4's multi-GPU layout: every rank solves B/R instances as its own
    problem; the shards cover the instances in order, and (instances being independent, K fixed)
    the oracle's output per shard is bitwise the full problem's rows."""
    import numpy as np
    import oracle
    from paper_2303_03848_b200 import synth
    p = synth.portfolio(n_k=2, n_s=2, M=32, N=4, coarse=synth.COARSE_IMPLICIT_EULER, max_iter=2, tol=0.0)
    full = oracle.parareal(p)[0][-1]
    for world in (1, 2, 4):
        shards = [synth.shard_instances(p, r, world) for r in range(world)]
        assert [s.B for s in shards] == [p.B // world] * world
        assert np.array_equal(np.concatenate([s.strike for s in shards]), p.strike)
        assert np.array_equal(np.concatenate([s.sigma for s in shards]), p.sigma)
        got = np.concatenate([oracle.parareal(s)[0][-1] for s in shards])
        assert np.array_equal(got, full)
    with pytest.raises(ValueError):
        synth.shard_instances(p, 0, 3)
