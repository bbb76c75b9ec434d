"""CPU oracle of PINN training — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this
module; the product path (paper_2303_03848_b200) never imports it and never
falls back to it.  Plain numpy in float64, one formula per step, in the
paper's order and notation:

  network     Ṽ(t, S) = L · y(t/T, S/L), y a fully connected net whose hidden
              layers apply tanh or ReLU and whose output layer is linear
              (§3.3; inputs (t, S) as the losses use them,
              P:177-189, reading Q28 in DESIGN.md; normalisation reading Q8).
  derivatives the residual needs Ṽ_t, Ṽ_S, Ṽ_SS, "calculated by automatic
              differentiation": forward jets (value, ∂t, ∂S, ∂SS)
              through every layer, and reverse accumulation of the loss through
              the same chain rules for the parameter gradient.
  losses      MSE_total = MSE_f + MSE_exp + MSE_b (Eq. 11):
                MSE_f   = mean f(Ṽ)², f = Ṽ_t + ½σ²S²Ṽ_SS + rSṼ_S − rṼ  (Eq. 12, Eq. 1)
                MSE_b   = mean (Ṽ(t_i,S_i) − V(t_i,S_i))², S_i ∈ {0, L}      (Eq. 13; targets Eq. 3
                          V(t,0)=0 and, at S=L, reading Q3: L − K e^{−r(T−t)}, or 0 with BC_ZERO)
                MSE_exp = mean (Ṽ(T,S_i) − max(S_i − K, 0))²                 (Eq. 14, Eq. 2)
  optimiser   Adam (Kingma & Ba) with β = (0.9, 0.999), ε = 1e-8.
  batches     each epoch shuffles each collocation set ("shuffled during every
              epoch") and splits it into `batches` consecutive parts;
              batch i of an epoch holds part i of every set.  The shuffle is a
              counter-based bijection (`perm`) that the CUDA side implements
              independently from the same definition.

Parameters are kept as a list of (W, b) float64 arrays, W row-major [out][in].
"""
from __future__ import annotations

from typing import List, Sequence, Tuple

import numpy as np

TANH, RELU = 0, 1
BC_CALL_ASYMPTOTIC, BC_ZERO = 0, 1
_MASK64 = (1 << 64) - 1


# ---------------------------------------------------------------- the shuffle (counter-based)

def splitmix64(z: int) -> int:
    """SplitMix64 finaliser (Steele, Lea, Flood 2014) on an unsigned 64-bit integer."""
    z = (z + 0x9E3779B97F4A7C15) & _MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
    return z ^ (z >> 31)


def perm_keys(seed: int, epoch: int, which: int) -> List[int]:
    """Four round keys of the permutation of set `which` (0 interior, 1 boundary, 2 expiry) in
    epoch `epoch`: base = splitmix64(seed XOR splitmix64(4·epoch + which)), k_r = splitmix64(base + r)."""
    base = splitmix64((seed & _MASK64) ^ splitmix64((4 * epoch + which) & _MASK64))
    return [splitmix64((base + r) & _MASK64) for r in range(4)]


def perm(seed: int, epoch: int, which: int, n: int) -> np.ndarray:
    """The shuffle of a set of n points: position i of the epoch's order holds point perm[i].
    On b = max(1, ⌈log2 n⌉)-bit integers x, four rounds of
        x ← (x · (k_r | 1)) mod 2^b;  x ← (x + (k_r >> 40)) mod 2^b;  x ← x XOR (x >> s),  s = max(1, b//2)
    (each step a bijection of [0, 2^b)), then cycle-walking (re-apply until x < n), which makes it
    a bijection of [0, n)."""
    if n <= 0:
        return np.zeros(0, dtype=np.int64)
    b = max(1, int(n - 1).bit_length())
    mask = (1 << b) - 1
    s = max(1, b // 2)
    keys = perm_keys(seed, epoch, which)

    def F(x: int) -> int:
        for k in keys:
            x = (x * (k | 1)) & mask
            x = (x + (k >> 40)) & mask
            x ^= x >> s
        return x

    out = np.empty(n, dtype=np.int64)
    for i in range(n):
        x = F(i)
        while x >= n:
            x = F(x)
        out[i] = x
    return out


_perm_cache: dict = {}


def batch_indices(seed: int, epoch: int, batches: int, ib: int, n_f: int, n_b: int, n_e: int):
    """Indices (interior, boundary, expiry) of batch ib of an epoch: part ib of each shuffled set,
    part i = positions [i·n//batches, (i+1)·n//batches)."""
    out = []
    for which, n in enumerate((n_f, n_b, n_e)):
        key = (seed, epoch, which, n)
        if key not in _perm_cache:
            if len(_perm_cache) > 64:
                _perm_cache.clear()
            _perm_cache[key] = perm(seed, epoch, which, n)
        p = _perm_cache[key]
        out.append(p[ib * n // batches:(ib + 1) * n // batches])
    return tuple(out)


# ---------------------------------------------------------------- network with forward jets

def _act(z, act):
    """σ(z) and its first three derivatives σ', σ'', σ''' (tanh or ReLU)."""
    if act == TANH:
        h = np.tanh(z)
        d1 = 1.0 - h * h
        return h, d1, -2.0 * h * d1, d1 * (6.0 * h * h - 2.0)
    h = np.maximum(z, 0.0)
    d1 = (z > 0).astype(np.float64)
    zero = np.zeros_like(z)
    return h, d1, zero, zero


def forward_jet(params, act: int, T: float, L: float, t, S, keep: bool = False):
    """Ṽ and its partials (Ṽ_t, Ṽ_S, Ṽ_SS) at the points (t, S) (arrays of equal length).

    Input features x = (t/T, S/L), so x_t = (1/T, 0), x_S = (0, 1/L), x_SS = 0.  Affine layer
    z = W h + b maps each jet component linearly (the bias only enters the value); an activation
    maps (h, h_t, h_S, h_SS) ↦ (σ(z), σ'z_t, σ'z_S, σ''z_S² + σ'z_SS) (chain rule).
    keep=True also returns each hidden layer's (z, z_t, z_S, z_SS) for the reverse pass."""
    t = np.asarray(t, np.float64)
    S = np.asarray(S, np.float64)
    n = t.shape[0]
    h = np.stack([t / T, S / L], axis=1)
    h_t = np.tile([1.0 / T, 0.0], (n, 1))
    h_S = np.tile([0.0, 1.0 / L], (n, 1))
    h_SS = np.zeros((n, 2))
    saved = []
    for W, b in params[:-1]:
        z, z_t, z_S, z_SS = h @ W.T + b, h_t @ W.T, h_S @ W.T, h_SS @ W.T
        s0, s1, s2, _ = _act(z, act)
        saved.append((z, z_t, z_S, z_SS))
        h, h_t, h_S, h_SS = s0, s1 * z_t, s1 * z_S, s2 * z_S * z_S + s1 * z_SS
    Wo, bo = params[-1]
    jet = (L * (h @ Wo.T + bo)[:, 0], L * (h_t @ Wo.T)[:, 0], L * (h_S @ Wo.T)[:, 0], L * (h_SS @ Wo.T)[:, 0])
    return (jet, saved) if keep else jet


def residual(jet, S, sigma: float, r: float):
    """f(Ṽ) = Ṽ_t + ½σ²S²Ṽ_SS + rSṼ_S − rṼ: Eq. (1) applied to the network (Eq. 12)."""
    V, V_t, V_S, V_SS = jet
    S = np.asarray(S, np.float64)
    return V_t + 0.5 * sigma * sigma * S * S * V_SS + r * S * V_S - r * V


def boundary_target(t, S, K: float, r: float, T: float, L: float, upper_bc: int = BC_CALL_ASYMPTOTIC):
    """V(t, 0) = 0 (Eq. 3); V(t, L) = L − K e^{−r(T−t)} (reading Q3) or 0 (BC_ZERO)."""
    t = np.asarray(t, np.float64)
    S = np.asarray(S, np.float64)
    upper = (L - K * np.exp(-r * (T - t))) if upper_bc == BC_CALL_ASYMPTOTIC else np.zeros_like(t)
    return np.where(S > 0.5 * L, upper, 0.0)


def loss_terms(params, act, mk, t_f, S_f, t_b, S_b, S_e) -> Tuple[float, float, float]:
    """(MSE_f, MSE_b, MSE_exp) of Eqs. (12)-(14) over the given points; mk = dict(K, sigma, r, T, L, upper_bc)."""
    T, L = mk["T"], mk["L"]
    jf = forward_jet(params, act, T, L, t_f, S_f)
    mse_f = float(np.mean(residual(jf, S_f, mk["sigma"], mk["r"]) ** 2)) if len(t_f) else 0.0
    Vb = forward_jet(params, act, T, L, t_b, S_b)[0]
    tgt = boundary_target(t_b, S_b, mk["K"], mk["r"], T, L, mk.get("upper_bc", 0))
    mse_b = float(np.mean((Vb - tgt) ** 2)) if len(t_b) else 0.0
    S_e = np.asarray(S_e, np.float64)
    Ve = forward_jet(params, act, T, L, np.full(S_e.shape, T), S_e)[0]
    mse_e = float(np.mean((Ve - np.maximum(S_e - mk["K"], 0.0)) ** 2)) if len(S_e) else 0.0
    return mse_f, mse_b, mse_e


# ---------------------------------------------------------------- reverse accumulation

def _backward(params, act, T, L, t, S, V_bar):
    """Parameter gradient of Σ_i (V̄_i · jet_i) for output adjoints V_bar = (V̄, V̄_t, V̄_S, V̄_SS)
    per point: reverse accumulation through the forward-jet chain rules of `forward_jet`."""
    (_, saved) = forward_jet(params, act, T, L, t, S, keep=True)
    n = len(t)
    grads = [None] * len(params)
    # hidden-layer outputs (jets) recomputed from the saved pre-activations
    hs = []
    for z, z_t, z_S, z_SS in saved:
        s0, s1, s2, _ = _act(z, act)
        hs.append((s0, s1 * z_t, s1 * z_S, s2 * z_S * z_S + s1 * z_SS))
    x = (np.stack([np.asarray(t) / T, np.asarray(S) / L], 1), np.tile([1.0 / T, 0.0], (n, 1)),
         np.tile([0.0, 1.0 / L], (n, 1)), np.zeros((n, 2)))
    # output layer: V_c = L · (Wo h_c (+ bo for the value))
    Wo, _ = params[-1]
    y_bar = [L * np.asarray(v, np.float64)[:, None] for v in V_bar]          # [n,1] per component
    h_last = hs[-1] if hs else x
    gW = sum(y_bar[c].T @ h_last[c] for c in range(4))
    grads[-1] = (gW, y_bar[0].sum(axis=0))
    h_bar = [y_bar[c] @ Wo for c in range(4)]
    for l in range(len(params) - 2, -1, -1):
        W, _ = params[l]
        z, z_t, z_S, z_SS = saved[l]
        _, s1, s2, s3 = _act(z, act)
        hb, hb_t, hb_S, hb_SS = h_bar
        zb_t = hb_t * s1
        zb_S = hb_S * s1 + hb_SS * 2.0 * s2 * z_S
        zb_SS = hb_SS * s1
        zb = hb * s1 + hb_t * s2 * z_t + hb_S * s2 * z_S + hb_SS * (s3 * z_S * z_S + s2 * z_SS)
        z_bar = (zb, zb_t, zb_S, zb_SS)
        h_prev = hs[l - 1] if l > 0 else x
        grads[l] = (sum(z_bar[c].T @ h_prev[c] for c in range(4)), zb.sum(axis=0))
        h_bar = [z_bar[c] @ W for c in range(4)]
    return grads


def loss_and_grad(params, act, mk, t_f, S_f, t_b, S_b, S_e):
    """(MSE_f, MSE_b, MSE_exp) and ∇_θ MSE_total (Eq. 11) over the given points."""
    T, L, K, sig, r = mk["T"], mk["L"], mk["K"], mk["sigma"], mk["r"]
    S_f = np.asarray(S_f, np.float64)
    S_e = np.asarray(S_e, np.float64)
    terms = loss_terms(params, act, mk, t_f, S_f, t_b, S_b, S_e)
    total = [(np.zeros_like(W), np.zeros_like(b)) for W, b in params]
    # interior: d/dθ mean f² = mean 2f ∂f/∂jet · ∂jet/∂θ, ∂f/∂(V, V_t, V_S, V_SS) = (−r, 1, rS, ½σ²S²)
    if len(t_f):
        f = residual(forward_jet(params, act, T, L, t_f, S_f), S_f, sig, r)
        fb = 2.0 * f / len(t_f)
        g = _backward(params, act, T, L, t_f, S_f, (-r * fb, fb, r * S_f * fb, 0.5 * sig * sig * S_f * S_f * fb))
        total = [(a[0] + c[0], a[1] + c[1]) for a, c in zip(total, g)]
    if len(t_b):
        Vb = forward_jet(params, act, T, L, t_b, S_b)[0]
        e = 2.0 * (Vb - boundary_target(t_b, S_b, K, r, T, L, mk.get("upper_bc", 0))) / len(t_b)
        z0 = np.zeros_like(e)
        g = _backward(params, act, T, L, t_b, S_b, (e, z0, z0, z0))
        total = [(a[0] + c[0], a[1] + c[1]) for a, c in zip(total, g)]
    if len(S_e):
        tT = np.full(S_e.shape, T)
        Ve = forward_jet(params, act, T, L, tT, S_e)[0]
        e = 2.0 * (Ve - np.maximum(S_e - K, 0.0)) / len(S_e)
        z0 = np.zeros_like(e)
        g = _backward(params, act, T, L, tT, S_e, (e, z0, z0, z0))
        total = [(a[0] + c[0], a[1] + c[1]) for a, c in zip(total, g)]
    return terms, total


# ---------------------------------------------------------------- Adam and the training loop

def flatten(params) -> np.ndarray:
    """Parameters in the library's packed order: per layer W (row-major) then b."""
    return np.concatenate([np.concatenate([W.ravel(), b.ravel()]) for W, b in params])


def unflatten(vec, dims: Sequence[int]):
    out, o = [], 0
    for l in range(len(dims) - 1):
        nW = dims[l + 1] * dims[l]
        out.append((vec[o:o + nW].reshape(dims[l + 1], dims[l]).copy(), vec[o + nW:o + nW + dims[l + 1]].copy()))
        o += nW + dims[l + 1]
    return out


def adam_step(theta, m, v, g, step: int, lr: float, beta1=0.9, beta2=0.999, eps=1e-8):
    """One Adam update (Kingma & Ba, Algorithm 1) at step number `step` ≥ 1 (arrays updated in place)."""
    m *= beta1
    m += (1.0 - beta1) * g
    v *= beta2
    v += (1.0 - beta2) * g * g
    mhat = m / (1.0 - beta1 ** step)
    vhat = v / (1.0 - beta2 ** step)
    theta -= lr * mhat / (np.sqrt(vhat) + eps)


class Trainer:
    """The training procedure of P:207-211: Adam over shuffled mini-batches, learning rate per call."""

    def __init__(self, net, mk, sets, batches: int, seed: int, beta1=0.9, beta2=0.999, eps=1e-8):
        self.dims = list(net.dims)
        self.act = int(net.activation)
        self.mk = dict(mk)
        self.theta = flatten([(np.asarray(W, np.float64), np.asarray(b, np.float64)) for W, b in zip(net.W, net.b)])
        self.m = np.zeros_like(self.theta)
        self.v = np.zeros_like(self.theta)
        self.sets = [np.asarray(a, np.float64) for a in sets]   # t_f, S_f, t_b, S_b, S_e
        self.batches, self.seed, self.step = int(batches), int(seed), 0
        self.beta1, self.beta2, self.eps = beta1, beta2, eps

    def params(self):
        return unflatten(self.theta, self.dims)

    def batch(self, step: int):
        t_f, S_f, t_b, S_b, S_e = self.sets
        e, ib = divmod(step, self.batches)
        i_f, i_b, i_e = batch_indices(self.seed, e, self.batches, ib, len(t_f), len(t_b), len(S_e))
        return t_f[i_f], S_f[i_f], t_b[i_b], S_b[i_b], S_e[i_e]

    def gradient(self, step: int):
        terms, g = loss_and_grad(self.params(), self.act, self.mk, *self.batch(step))
        return terms, flatten(g)

    def epochs(self, n: int, lr: float):
        hist = []
        for _ in range(n * self.batches):
            terms, g = self.gradient(self.step)
            self.step += 1
            adam_step(self.theta, self.m, self.v, g, self.step, lr, self.beta1, self.beta2, self.eps)
            hist.append(terms)
        return np.array(hist)

    def full_loss(self):
        return loss_terms(self.params(), self.act, self.mk, *self.sets)
