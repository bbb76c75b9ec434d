"""ctypes wrapper of the CPU oracle (oracle/oracle.cpp) — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
leg may import this package.  The product path (paper_2303_03848_b200) never
imports it and never falls back to it.

All arrays are float64 numpy.  `prec=64` runs the FP64 oracle proper;
`prec=32` runs the same algorithm with every intermediate in float (used only
for the stability gate of SURVEY.md §8(c)).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from typing import Optional, Tuple

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_HDR = os.path.join(_HERE, "oracle.h")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with g++ (-O2, no FP contraction: Q27)."""
    stale = (not os.path.exists(_LIB)) or any(
        os.path.getmtime(s) > os.path.getmtime(_LIB) for s in (_SRC, _HDR))
    if force or stale:
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["g++", "-O2", "-std=c++17", "-ffp-contract=off", "-fPIC", "-shared", "-pthread",
                               "-Wall", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


class _Problem(C.Structure):
    _fields_ = [("M", C.c_int), ("B", C.c_int),
                ("strike", C.POINTER(C.c_double)), ("sigma", C.POINTER(C.c_double)),
                ("rate", C.POINTER(C.c_double)), ("L", C.POINTER(C.c_double)),
                ("T", C.c_double), ("upper_bc", C.c_int), ("N", C.c_int), ("fine_steps", C.c_int),
                ("fine_theta", C.c_double), ("coarse", C.c_int), ("coarse_steps", C.c_int),
                ("max_iter", C.c_int), ("tol", C.c_double)]


class _Net(C.Structure):
    _fields_ = [("n_linear", C.c_int), ("dims", C.POINTER(C.c_int)),
                ("W", C.POINTER(C.POINTER(C.c_double))), ("b", C.POINTER(C.POINTER(C.c_double))),
                ("activation", C.c_int), ("in_scale", C.POINTER(C.c_double)), ("out_scale", C.c_double)]


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            dp = C.POINTER(C.c_double)
            L.or_bs_call.restype = C.c_double
            L.or_bs_call.argtypes = [C.c_double] * 5
            L.or64_operator.argtypes = [C.c_int, C.c_double, C.c_double, dp, dp, dp]
            L.or64_operator.restype = None
            for pre in ("or64_", "or32_"):
                getattr(L, pre + "thomas").argtypes = [C.c_int, dp, dp, dp, dp, dp]
                getattr(L, pre + "propagate").argtypes = [C.POINTER(_Problem), C.c_int, C.c_double, C.c_int, dp]
                getattr(L, pre + "mlp").argtypes = [C.POINTER(_Net), dp, dp]
                getattr(L, pre + "mlp").restype = None
                getattr(L, pre + "pinn_G").argtypes = [C.POINTER(_Problem), C.POINTER(_Net), C.c_int, dp, dp]
                getattr(L, pre + "serial_fine").argtypes = [C.POINTER(_Problem), dp, dp]
                getattr(L, pre + "parareal").argtypes = [C.POINTER(_Problem), C.POINTER(_Net), dp, dp, dp,
                                                         C.POINTER(C.c_int), dp]
            L.or64_parareal_mt.argtypes = [C.POINTER(_Problem), C.POINTER(_Net), dp, dp, dp, C.POINTER(C.c_int), dp,
                                           C.c_int]
            L.or64_theta_step.argtypes = [C.POINTER(_Problem), C.c_int, C.c_double, C.c_double, C.c_double, dp]
            L.or64_payoff.argtypes = [C.POINTER(_Problem), dp]
            L.or64_payoff.restype = None
            _lib = L
    return _lib


def _dp(a: Optional[np.ndarray]):
    if a is None:
        return None
    return a.ctypes.data_as(C.POINTER(C.c_double))


class _Keep:
    """Holds numpy buffers alive while a ctypes struct points into them."""

    def __init__(self):
        self.refs = []

    def f64(self, a) -> np.ndarray:
        a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
        self.refs.append(a)
        return a


def _problem(p, keep: _Keep) -> _Problem:
    s = _Problem()
    s.M, s.B = int(p.M), int(p.B)
    s.strike = _dp(keep.f64(p.strike))
    s.sigma = _dp(keep.f64(p.sigma))
    s.rate = _dp(keep.f64(p.rate))
    s.L = _dp(keep.f64(p.L))
    s.T, s.upper_bc, s.N, s.fine_steps = float(p.T), int(p.upper_bc), int(p.N), int(p.fine_steps)
    s.fine_theta, s.coarse, s.coarse_steps = float(p.fine_theta), int(p.coarse), int(p.coarse_steps)
    s.max_iter, s.tol = int(p.max_iter), float(p.tol)
    return s


def _net(net, keep: _Keep) -> Optional[_Net]:
    if net is None:
        return None
    s = _Net()
    s.n_linear = len(net.W)
    dims = (C.c_int * len(net.dims))(*net.dims)
    keep.refs.append(dims)
    s.dims = dims
    Ws = [keep.f64(W) for W in net.W]
    bs = [keep.f64(b) for b in net.b]
    Wp = (C.POINTER(C.c_double) * len(Ws))(*[_dp(w) for w in Ws])
    bp = (C.POINTER(C.c_double) * len(bs))(*[_dp(b) for b in bs])
    keep.refs += [Wp, bp]
    s.W, s.b = Wp, bp
    s.activation = int(net.activation)
    s.in_scale = _dp(keep.f64(net.in_scale)) if net.in_scale is not None else None
    s.out_scale = float(net.out_scale)
    return s


def _ok(st: int, what: str):
    if st == 1:
        raise ValueError("oracle %s: invalid argument" % what)
    if st == 3:
        raise ArithmeticError("oracle %s: non-positive pivot" % what)
    if st:
        raise RuntimeError("oracle %s: status %d" % (what, st))


def bs_call(S, K, r, sigma, tau) -> float:
    return lib().or_bs_call(float(S), float(K), float(r), float(sigma), float(tau))


def operator(M: int, sigma: float, r: float) -> Tuple[np.ndarray, np.ndarray, np.ndarray]:
    lo, di, up = (np.zeros(M) for _ in range(3))
    lib().or64_operator(M, sigma, r, _dp(lo), _dp(di), _dp(up))
    return lo, di, up


def thomas(sub, diag, sup, rhs, prec: int = 64) -> np.ndarray:
    keep = _Keep()
    a, d, c, r = (keep.f64(v) for v in (sub, diag, sup, rhs))
    x = np.zeros(len(d))
    _ok(getattr(lib(), "or%d_thomas" % prec)(len(d), _dp(a), _dp(d), _dp(c), _dp(r), _dp(x)), "thomas")
    return x


def theta_step(p, b: int, theta: float, tau0: float, dtau: float, w) -> np.ndarray:
    keep = _Keep()
    s = _problem(p, keep)
    w = keep.f64(w).copy()
    _ok(lib().or64_theta_step(C.byref(s), b, theta, tau0, dtau, _dp(w)), "theta_step")
    return w


def propagate(p, n: int, U, theta: Optional[float] = None, steps: Optional[int] = None,
              prec: int = 64) -> np.ndarray:
    """`steps` theta-steps across slice n for all instances; U [B][M] -> new array."""
    keep = _Keep()
    s = _problem(p, keep)
    U = keep.f64(U).reshape(p.B, p.M).copy()
    theta = p.fine_theta if theta is None else theta
    steps = p.fine_steps if steps is None else steps
    _ok(getattr(lib(), "or%d_propagate" % prec)(C.byref(s), n, float(theta), int(steps), _dp(U)), "propagate")
    return U


def fine(p, n: int, U, prec: int = 64) -> np.ndarray:
    return propagate(p, n, U, p.fine_theta, p.fine_steps, prec)


def coarse_ie(p, n: int, U, prec: int = 64) -> np.ndarray:
    return propagate(p, n, U, 1.0, p.coarse_steps, prec)


def mlp(net, x, prec: int = 64) -> float:
    keep = _Keep()
    s = _net(net, keep)
    x = keep.f64(x)
    y = np.zeros(1)
    getattr(lib(), "or%d_mlp" % prec)(C.byref(s), _dp(x), _dp(y))
    return float(y[0])


def pinn_G(p, net, n: int, U, prec: int = 64) -> np.ndarray:
    keep = _Keep()
    s, sn = _problem(p, keep), _net(net, keep)
    U = keep.f64(U).reshape(p.B, p.M)
    out = np.zeros_like(U)
    _ok(getattr(lib(), "or%d_pinn_G" % prec)(C.byref(s), C.byref(sn), n, _dp(U), _dp(out)), "pinn_G")
    return out


def payoff(p) -> np.ndarray:
    keep = _Keep()
    s = _problem(p, keep)
    out = np.zeros((p.B, p.M))
    lib().or64_payoff(C.byref(s), _dp(out))
    return out


def serial_fine(p, V_T=None, prec: int = 64) -> np.ndarray:
    """Eq. (6): all slice boundaries U[N+1][B][M]."""
    keep = _Keep()
    s = _problem(p, keep)
    vt = None if V_T is None else keep.f64(V_T).reshape(p.B, p.M)
    U = np.zeros((p.N + 1, p.B, p.M))
    _ok(getattr(lib(), "or%d_serial_fine" % prec)(C.byref(s), _dp(vt), _dp(U)), "serial_fine")
    return U


def parareal(p, net=None, V_T=None, prec: int = 64, history: bool = False, threads: int = 1):
    """Eq. (7) with schedule Q12.  Returns (U[N+1][B][M], delta[K], K, hist or None).
    threads > 1 (fp64 only): the fine sweep's slices on that many std::threads, bitwise the same."""
    keep = _Keep()
    s = _problem(p, keep)
    sn = _net(net, keep)
    vt = None if V_T is None else keep.f64(V_T).reshape(p.B, p.M)
    U = np.zeros((p.N + 1, p.B, p.M))
    delta = np.zeros(p.max_iter)
    K = C.c_int(0)
    hist = np.zeros((p.max_iter + 1, p.N + 1, p.B, p.M)) if history else None
    args = (C.byref(s), C.byref(sn) if sn is not None else None, _dp(vt), _dp(U), _dp(delta), C.byref(K), _dp(hist))
    if threads > 1 and prec == 64:
        _ok(lib().or64_parareal_mt(*args, int(threads)), "parareal")
    else:
        _ok(getattr(lib(), "or%d_parareal" % prec)(*args), "parareal")
    k = K.value
    return U, delta[:k].copy(), k, (hist[:k + 1] if history else None)
