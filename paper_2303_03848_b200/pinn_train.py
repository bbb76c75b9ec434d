"""Thin ctypes binding of include/pinn_train.h (argument marshalling only).

Every step of training runs in libparareal.so's CUDA kernels (k_train_grad, k_adam); there is no
CPU fallback.  Names follow the C ABI: pinn_train_init → Trainer(...), pinn_train_epochs →
Trainer.epochs, pinn_train_loss → Trainer.loss, pinn_train_batch_gradient →
Trainer.batch_gradient, pinn_train_get_weights → Trainer.net().
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Sequence

import numpy as np

from . import parareal, synth

# every symbol include/pinn_train.h declares (checked by tests/test_abi.py)
EXPORTS = ["pinn_train_init", "pinn_train_epochs", "pinn_train_loss", "pinn_train_batch_gradient",
           "pinn_train_param_count", "pinn_train_step_count", "pinn_train_get_params", "pinn_train_get_weights",
           "pinn_train_last_error", "pinn_train_free"]


class Config(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("strike", C.c_double), ("sigma", C.c_double), ("rate", C.c_double),
                ("L", C.c_double), ("T", C.c_double), ("upper_bc", C.c_int32), ("n_linear", C.c_int32),
                ("dims", C.POINTER(C.c_int32)), ("activation", C.c_int32),
                ("W", C.POINTER(C.POINTER(C.c_float))), ("b", C.POINTER(C.POINTER(C.c_float))),
                ("n_f", C.c_int32), ("n_b", C.c_int32), ("n_exp", C.c_int32),
                ("t_f", C.POINTER(C.c_float)), ("S_f", C.POINTER(C.c_float)),
                ("t_b", C.POINTER(C.c_float)), ("S_b", C.POINTER(C.c_float)), ("S_exp", C.POINTER(C.c_float)),
                ("batches", C.c_int32), ("shuffle_seed", C.c_uint64),
                ("beta1", C.c_double), ("beta2", C.c_double), ("eps", C.c_double),
                ("device", C.c_int32), ("stream", C.c_void_p)]


_declared = False


def lib() -> C.CDLL:
    global _declared
    L = parareal.lib()
    if not _declared:
        vp, fp, dp = C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_double)
        L.pinn_train_init.argtypes = [C.POINTER(Config), C.POINTER(vp)]
        L.pinn_train_epochs.argtypes = [vp, C.c_int32, C.c_double, dp]
        L.pinn_train_loss.argtypes = [vp, dp]
        L.pinn_train_batch_gradient.argtypes = [vp, C.c_int64, fp, dp]
        L.pinn_train_param_count.argtypes = [vp]
        L.pinn_train_param_count.restype = C.c_int64
        L.pinn_train_step_count.argtypes = [vp]
        L.pinn_train_step_count.restype = C.c_int64
        L.pinn_train_get_params.argtypes = [vp, fp]
        L.pinn_train_get_weights.argtypes = [vp, C.POINTER(fp), C.POINTER(fp)]
        L.pinn_train_last_error.argtypes = [vp]
        L.pinn_train_last_error.restype = C.c_char_p
        L.pinn_train_free.argtypes = [vp]
        L.pinn_train_free.restype = None
        for n in ("pinn_train_init", "pinn_train_epochs", "pinn_train_loss", "pinn_train_batch_gradient",
                  "pinn_train_get_params", "pinn_train_get_weights"):
            getattr(L, n).restype = C.c_int
        _declared = True
    return L


def _fp(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_float))


class Trainer:
    """pinn_train_init … pinn_train_free.  `market` = dict(K, sigma, r, T, L[, upper_bc]);
    `sets` = (t_f, S_f, t_b, S_b, S_e) (float32, e.g. synth.collocation)."""

    def __init__(self, net: synth.Net, market: dict, sets: Sequence[np.ndarray], batches: int = 1, seed: int = 0,
                 beta1: float = 0.9, beta2: float = 0.999, eps: float = 1e-8, device: int = 0,
                 stream: Optional[int] = None):
        self._L = lib()
        self.dims = list(net.dims)
        self.activation = int(net.activation)
        self._keep = []
        c = Config()
        c.struct_size = C.sizeof(Config)
        c.strike, c.sigma, c.rate = float(market["K"]), float(market["sigma"]), float(market["r"])
        c.L, c.T = float(market["L"]), float(market["T"])
        c.upper_bc = int(market.get("upper_bc", synth.BC_CALL_ASYMPTOTIC))
        c.n_linear = len(net.W)
        dims = (C.c_int32 * len(net.dims))(*net.dims)
        Ws = [np.ascontiguousarray(W, np.float32) for W in net.W]
        bs = [np.ascontiguousarray(b, np.float32) for b in net.b]
        Wp = (C.POINTER(C.c_float) * len(Ws))(*[_fp(w) for w in Ws])
        bp = (C.POINTER(C.c_float) * len(bs))(*[_fp(b) for b in bs])
        pts = [np.ascontiguousarray(a, np.float32) for a in sets]
        self._keep += [dims, Ws, bs, Wp, bp, pts]
        c.dims, c.activation, c.W, c.b = dims, self.activation, Wp, bp
        c.n_f, c.n_b, c.n_exp = len(pts[0]), len(pts[2]), len(pts[4])
        c.t_f, c.S_f, c.t_b, c.S_b, c.S_exp = [_fp(a) for a in pts]
        c.batches, c.shuffle_seed = int(batches), int(seed)
        c.beta1, c.beta2, c.eps = float(beta1), float(beta2), float(eps)
        c.device = int(device)
        c.stream = stream
        self.batches = int(batches)
        h = C.c_void_p()
        st = self._L.pinn_train_init(C.byref(c), C.byref(h))
        if st:
            raise parareal.PararealError(st, self._L.pinn_train_last_error(None).decode())
        self._h = h

    def _check(self, st: int):
        if st:
            raise parareal.PararealError(st, self._L.pinn_train_last_error(self._h).decode())

    @property
    def param_count(self) -> int:
        return int(self._L.pinn_train_param_count(self._h))

    @property
    def steps(self) -> int:
        return int(self._L.pinn_train_step_count(self._h))

    def epochs(self, n: int, lr: float, history: bool = True) -> Optional[np.ndarray]:
        """pinn_train_epochs: n epochs at learning rate lr; returns [n·batches, 3] loss terms."""
        hist = np.zeros((n * self.batches, 3)) if history else None
        self._check(self._L.pinn_train_epochs(self._h, int(n), float(lr),
                                              hist.ctypes.data_as(C.POINTER(C.c_double)) if history else None))
        return hist

    def loss(self) -> np.ndarray:
        out = np.zeros(3)
        self._check(self._L.pinn_train_loss(self._h, out.ctypes.data_as(C.POINTER(C.c_double))))
        return out

    def batch_gradient(self, step: int):
        g = np.zeros(self.param_count, np.float32)
        l = np.zeros(3)
        self._check(self._L.pinn_train_batch_gradient(self._h, int(step), _fp(g), l.ctypes.data_as(C.POINTER(C.c_double))))
        return l, g

    def params(self) -> np.ndarray:
        out = np.zeros(self.param_count, np.float32)
        self._check(self._L.pinn_train_get_params(self._h, _fp(out)))
        return out

    def net(self) -> synth.Net:
        """pinn_train_get_weights → a 2-input net for parareal_load_pinn_weights (dims[0] = 2)."""
        Ws = [np.zeros((self.dims[l + 1], self.dims[l]), np.float32) for l in range(len(self.dims) - 1)]
        bs = [np.zeros(self.dims[l + 1], np.float32) for l in range(len(self.dims) - 1)]
        Wp = (C.POINTER(C.c_float) * len(Ws))(*[_fp(w) for w in Ws])
        bp = (C.POINTER(C.c_float) * len(bs))(*[_fp(b) for b in bs])
        self._check(self._L.pinn_train_get_weights(self._h, Wp, bp))
        return synth.Net(list(self.dims), Ws, bs, self.activation)

    def close(self):
        if getattr(self, "_h", None):
            self._L.pinn_train_free(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
