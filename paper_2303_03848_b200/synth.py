"""Seeded synthetic inputs shared by the CUDA path and the CPU oracle.

This module holds NO arithmetic of the method (no payoff, no operator, no
propagator, no network evaluation): only problem parameters, random network
weights and random test states.  Both `oracle/` and the CUDA binding consume
what it produces; neither side imports the other.

Workload recipe (BASELINE.json `configs`):
  C1  K=1, r=.05, sigma=.2, T=1, L=4K, M=64,   N=4,  100 IE steps/slice, PINN [4,20,20,20,1]
  C2  as C1 with M=1024, N=32                    (configs[1]: the 1-GPU bench workload)
  C3  as C1 with M=2^20, N=64                    (configs[2]: sharded over 1/2/4/8 GPUs)
  C4  B=4096 instances, K_b in {0.8+0.4i/63} x sigma_b in {0.1+0.4j/63}, r=.05, L_b=4K_b,
      M=256, N=16                              (configs[3])
  C5  as C1 with M=2^18, N=64, PINN widths 20/64/256 x 4-8 hidden layers (configs[4])
Readings used: L = 4K (Q5), M = interior unknowns (Q4),
step counts per slice (Q2), IE fine propagator (Q1), 4-input PINN (Q6),
Kaiming-normal weights with U(+-1/sqrt(fan_in)) biases (Q11; §3.3).
"""
from __future__ import annotations

import dataclasses
import struct
from typing import List, Optional, Sequence

import numpy as np

# enum values mirrored from include/parareal.h (plain constants, no arithmetic)
COARSE_PINN = 0
COARSE_IMPLICIT_EULER = 1
BC_CALL_ASYMPTOTIC = 0
BC_ZERO = 1
ACT_TANH = 0
ACT_RELU = 1


@dataclasses.dataclass
class Problem:
    """Problem statement of PAPER.md §3 (Eqs. 1-4) + §3.1 decomposition + §3.2 steps."""
    M: int                      # interior grid points per instance
    strike: np.ndarray          # [B] K_b
    sigma: np.ndarray           # [B]
    rate: np.ndarray            # [B]
    L: np.ndarray               # [B] artificial upper bound S = L
    T: float = 1.0
    N: int = 4                  # time slices
    fine_steps: int = 100       # implicit steps per slice (Q2)
    fine_theta: float = 1.0     # 1 = implicit Euler (Q1); 0.5 = Crank-Nicolson (NEXT-1)
    coarse: int = COARSE_PINN
    coarse_steps: int = 1
    max_iter: int = 4
    tol: float = 0.0
    upper_bc: int = BC_CALL_ASYMPTOTIC

    @property
    def B(self) -> int:
        return int(len(self.strike))

    def replace(self, **kw) -> "Problem":
        return dataclasses.replace(self, **kw)


@dataclasses.dataclass
class Net:
    """Fully connected network: W[l] row-major [out][in] fp32."""
    dims: List[int]
    W: List[np.ndarray]
    b: List[np.ndarray]
    activation: int = ACT_TANH
    in_scale: Optional[np.ndarray] = None   # [dims[0]] extra input multipliers (Q8), default 1
    out_scale: float = 1.0

    @property
    def n_linear(self) -> int:
        return len(self.W)

    def scales(self) -> np.ndarray:
        if self.in_scale is None:
            return np.ones(self.dims[0], dtype=np.float32)
        return np.asarray(self.in_scale, dtype=np.float32)


def single(M: int, N: int, *, K: float = 1.0, r: float = 0.05, sigma: float = 0.2,
           L: Optional[float] = None, **kw) -> Problem:
    """One European call instance; L defaults to 4K (reading Q5)."""
    if L is None:
        L = 4.0 * K
    kw.setdefault("max_iter", min(4, N))
    return Problem(M=M, strike=np.array([K]), sigma=np.array([sigma]), rate=np.array([r]),
                   L=np.array([L]), N=N, **kw)


def portfolio(n_k: int = 64, n_s: int = 64, M: int = 256, N: int = 16, r: float = 0.05, **kw) -> Problem:
    """C4: strike x volatility sweep, L_b = 4 K_b (instance index = i*n_s + j)."""
    Ks = 0.8 + 0.4 * np.arange(n_k) / max(n_k - 1, 1)
    Ss = 0.1 + 0.4 * np.arange(n_s) / max(n_s - 1, 1)
    strike = np.repeat(Ks, n_s)
    sigma = np.tile(Ss, n_k)
    kw.setdefault("max_iter", min(4, N))
    return Problem(M=M, strike=strike, sigma=sigma, rate=np.full(strike.shape, r),
                   L=4.0 * strike, N=N, **kw)


def config(name: str, **kw) -> Problem:
    """BASELINE.json configs C1..C5."""
    name = name.upper()
    if name == "C1":
        return single(64, 4, **kw)
    if name == "C2":
        return single(1024, 32, **kw)
    if name == "C3":
        return single(1 << 20, 64, **kw)
    if name == "C4":
        return portfolio(**kw)
    if name == "C5":
        return single(1 << 18, 64, **kw)
    raise KeyError(name)


def shard_instances(p: Problem, rank: int, world: int) -> Problem:
    """Instances [rank·B/world, (rank+1)·B/world) of p: the C4 multi-GPU layout (SURVEY.md §8(e):
    independent problems, no data-path exchange; with a fixed K there is no collective at all)."""
    if world < 1 or not 0 <= rank < world or p.B % world:
        raise ValueError("B=%d instances cannot be split over %d ranks" % (p.B, world))
    n = p.B // world
    sl = slice(rank * n, (rank + 1) * n)
    return p.replace(strike=p.strike[sl].copy(), sigma=p.sigma[sl].copy(), rate=p.rate[sl].copy(),
                     L=p.L[sl].copy())


PINN_3x20 = [4, 20, 20, 20, 1]          # BASELINE configs "PINN 3x20 tanh"
PINN_PAPER = [4] + [50] * 10 + [1]      # PAPER.md:203 "10 fully connected layers with 50 neurons"


def kaiming_net(dims: Sequence[int], seed: int = 0, activation: int = ACT_TANH,
                in_scale=None, out_scale: float = 1.0) -> Net:
    """Kaiming-He normal weights, std sqrt(2/fan_in), biases
    U(-1/sqrt(fan_in), 1/sqrt(fan_in)) so the bias path is exercised (Q11).
    numpy PCG64 with the given seed; fp32."""
    rng = np.random.Generator(np.random.PCG64(seed))
    W, b = [], []
    for l in range(len(dims) - 1):
        fan_in, fan_out = dims[l], dims[l + 1]
        W.append((rng.standard_normal((fan_out, fan_in)) * np.sqrt(2.0 / fan_in)).astype(np.float32))
        lim = 1.0 / np.sqrt(fan_in)
        b.append(rng.uniform(-lim, lim, size=fan_out).astype(np.float32))
    return Net(list(dims), W, b, activation,
               None if in_scale is None else np.asarray(in_scale, np.float32), float(out_scale))


def random_state(B: int, M: int, seed: int = 0, scale: float = 1.0) -> np.ndarray:
    """A smooth-plus-noise nonnegative random state [B][M] (fp32) for single-propagator tests."""
    rng = np.random.Generator(np.random.PCG64(seed + 7919))
    x = np.linspace(0.0, 1.0, M, dtype=np.float64)[None, :]
    base = scale * np.maximum(0.0, x * rng.uniform(1.0, 4.0, size=(B, 1)) - rng.uniform(0.0, 1.0, size=(B, 1)))
    noise = 0.05 * scale * rng.random((B, M))
    return (base + noise).astype(np.float32)


# ---- weight blob (SURVEY.md §8(b) "Weight blob"; replaces SPEC's text checkpoint S:300-307)
MAGIC = b"PRPINN01"


def save_blob(net: Net, path: str) -> None:
    with open(path, "wb") as f:
        f.write(MAGIC)
        f.write(struct.pack("<I", net.n_linear))
        f.write(struct.pack("<%dI" % len(net.dims), *net.dims))
        f.write(struct.pack("<I", net.activation))
        f.write(net.scales().astype("<f4").tobytes())
        f.write(struct.pack("<f", net.out_scale))
        for W, b in zip(net.W, net.b):
            f.write(np.ascontiguousarray(W, "<f4").tobytes())
            f.write(np.ascontiguousarray(b, "<f4").tobytes())


def load_blob(path: str) -> Net:
    with open(path, "rb") as f:
        data = f.read()
    if data[:8] != MAGIC:
        raise ValueError("bad magic")
    off = 8
    (n,) = struct.unpack_from("<I", data, off); off += 4
    dims = list(struct.unpack_from("<%dI" % (n + 1), data, off)); off += 4 * (n + 1)
    (act,) = struct.unpack_from("<I", data, off); off += 4
    ins = np.frombuffer(data, "<f4", dims[0], off).copy(); off += 4 * dims[0]
    (outs,) = struct.unpack_from("<f", data, off); off += 4
    W, b = [], []
    for l in range(n):
        W.append(np.frombuffer(data, "<f4", dims[l + 1] * dims[l], off).reshape(dims[l + 1], dims[l]).copy())
        off += 4 * dims[l + 1] * dims[l]
        b.append(np.frombuffer(data, "<f4", dims[l + 1], off).copy())
        off += 4 * dims[l + 1]
    if off != len(data):
        raise ValueError("trailing bytes in blob")
    return Net(dims, W, b, act, ins, float(outs))


# ---- PINN training inputs ("randomly generate N_f=100,000 collocation
# points within the domain ..., N_b=10,000 at the boundary and N_exp=10,000 ... over [0,5000]")
PAPER_COLLOCATION = (100000, 10000, 10000)   # N_f, N_b, N_exp


def collocation(market: dict, n_f: int, n_b: int, n_exp: int, seed: int = 0):
    """Seeded collocation sets (float32) for the market dict(K, sigma, r, T, L): interior (t, S)
    uniform over [0,T]x[0,L]; boundary (t, S) with t uniform and S alternating 0, L (SPEC S:236:
    both ends in equal proportion); expiry S uniform over [0,L].  Returns (t_f, S_f, t_b, S_b, S_e)."""
    rng = np.random.Generator(np.random.PCG64(seed + 104729))
    T, L = float(market["T"]), float(market["L"])
    t_f = rng.uniform(0.0, T, n_f).astype(np.float32)
    S_f = rng.uniform(0.0, L, n_f).astype(np.float32)
    t_b = rng.uniform(0.0, T, n_b).astype(np.float32)
    S_b = np.where(np.arange(n_b) % 2 == 0, 0.0, L).astype(np.float32)
    S_e = rng.uniform(0.0, L, n_exp).astype(np.float32)
    return t_f, S_f, t_b, S_b, S_e


def pinn2_net(dims: Sequence[int], seed: int = 0, activation: int = ACT_TANH) -> Net:
    """A 2-input (t, S) network for training (dims[0] = 2): Kaiming-normal weights, zero biases
    (SPEC S:197)."""
    net = kaiming_net(dims, seed=seed, activation=activation)
    net.b = [np.zeros_like(b) for b in net.b]
    return net
