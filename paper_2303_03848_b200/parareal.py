"""Thin ctypes binding of the C ABI in include/parareal.h (argument marshalling only).

Every step of the hot path runs in libparareal.so's CUDA kernels.  There is no
CPU fallback: if the library or a GPU is missing the calls raise.
Names follow the C ABI: parareal_init → Context(...), parareal_solve →
Context.solve, parareal_solve_device → Context.solve_device, etc.
"""
from __future__ import annotations

import ctypes as C
import os
import threading
from typing import Optional, Tuple

import numpy as np

from . import synth

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PR_LIB_VARIANT") or os.path.join(_HERE, "libparareal.so")  # variant: A/B experiments only

PR_OK = 0
STATUS = {0: "PR_OK", 1: "PR_ERR_INVALID_ARGUMENT", 2: "PR_ERR_OUT_OF_MEMORY", 3: "PR_ERR_CUDA",
          4: "PR_ERR_NCCL", 5: "PR_ERR_STATE", 6: "PR_ERR_NUMERICAL", 7: "PR_ERR_UNSUPPORTED"}
PREC_FP32, PREC_FP16_TC, PREC_BF16_TC, PREC_TF32_TC, PREC_FP16X1_TC = 0, 1, 2, 3, 4
OPT_FINE_KERNEL, OPT_USE_GRAPHS, OPT_PINN_KERNEL, OPT_PIPELINE, OPT_COMM_TIMEOUT_MS, OPT_WAVEFRONT, OPT_SPATIAL_CHAIN = 1, 2, 3, 4, 5, 6, 7

# every symbol include/parareal.h declares (checked by tests/test_abi.py)
EXPORTS = ["parareal_status_string", "parareal_last_error", "parareal_get_nccl_id", "parareal_init",
           "parareal_workspace_bytes", "parareal_bind_workspace", "parareal_load_pinn_weights",
           "parareal_solve", "parareal_solve_device", "parareal_serial_fine", "parareal_serial_fine_device",
           "parareal_initial_state", "parareal_apply_fine", "parareal_apply_coarse", "parareal_copy_iterates", "parareal_set_option",
           "parareal_plan_iteration", "parareal_free"]


class PararealError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("%s: %s" % (STATUS.get(status, status), msg))
        self.status = status


class Problem(C.Structure):
    _fields_ = [("struct_size", C.c_uint32), ("M", C.c_int32), ("B", C.c_int32),
                ("strike", C.POINTER(C.c_double)), ("sigma", C.POINTER(C.c_double)),
                ("rate", C.POINTER(C.c_double)), ("L", C.POINTER(C.c_double)),
                ("T", C.c_double), ("upper_bc", C.c_int32), ("N", C.c_int32), ("fine_steps", C.c_int32),
                ("fine_theta", C.c_double), ("coarse", C.c_int32), ("coarse_steps", C.c_int32),
                ("max_iter", C.c_int32), ("tol", C.c_double)]


class Dist(C.Structure):
    _fields_ = [("rank", C.c_int32), ("world", C.c_int32), ("device", C.c_int32),
                ("nccl_id", C.POINTER(C.c_uint8)), ("stream", C.c_void_p)]


class Plan(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("fine_lo", "fine_hi", "fk_local", "recv_first", "copy", "chain_lo",
                                        "chain_hi", "send_last", "delta_lo", "delta_hi")]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("delta", C.POINTER(C.c_double)),
                ("ms_total", C.c_double), ("ms_coarse", C.c_double), ("ms_fine", C.c_double),
                ("ms_comm", C.c_double), ("ms_setup", C.c_double), ("kernel_launches", C.c_int64)]


_lock = threading.Lock()
_lib = None


def lib() -> C.CDLL:
    """Load the in-tree CUDA library.  Raises if it has not been built (no fallback)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise FileNotFoundError("%s not built: run `python -c 'import __graft_entry__ as g; g.build()'`"
                                        % LIB_PATH)
            L = C.CDLL(LIB_PATH)
            vp, fp, dp = C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_double)
            L.parareal_status_string.restype = C.c_char_p
            L.parareal_status_string.argtypes = [C.c_int]
            L.parareal_last_error.restype = C.c_char_p
            L.parareal_last_error.argtypes = [vp]
            L.parareal_get_nccl_id.argtypes = [C.POINTER(C.c_uint8)]
            L.parareal_init.argtypes = [C.POINTER(Problem), C.POINTER(Dist), C.POINTER(vp)]
            L.parareal_workspace_bytes.argtypes = [vp, C.POINTER(C.c_size_t)]
            L.parareal_bind_workspace.argtypes = [vp, vp, C.c_size_t]
            L.parareal_load_pinn_weights.argtypes = [vp, C.c_int32, C.POINTER(C.c_int32), C.POINTER(fp),
                                                     C.POINTER(fp), C.c_int32, fp, C.c_float, C.c_int32]
            L.parareal_solve.argtypes = [vp, fp, fp, C.POINTER(Report)]
            L.parareal_solve_device.argtypes = [vp, vp, vp, C.POINTER(Report)]
            L.parareal_serial_fine.argtypes = [vp, fp, fp, dp]
            L.parareal_serial_fine_device.argtypes = [vp, vp, vp, dp]
            L.parareal_initial_state.argtypes = [vp, fp]
            L.parareal_apply_fine.argtypes = [vp, C.c_int32, fp, fp]
            L.parareal_apply_coarse.argtypes = [vp, C.c_int32, fp, fp]
            L.parareal_copy_iterates.argtypes = [vp, C.c_int32, C.c_int32, fp]
            L.parareal_set_option.argtypes = [vp, C.c_int32, C.c_int64]
            L.parareal_plan_iteration.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.POINTER(Plan)]
            L.parareal_free.argtypes = [vp]
            L.parareal_free.restype = None
            for name in ("parareal_get_nccl_id", "parareal_init", "parareal_workspace_bytes",
                         "parareal_bind_workspace", "parareal_load_pinn_weights", "parareal_solve",
                         "parareal_solve_device", "parareal_serial_fine", "parareal_serial_fine_device",
                         "parareal_initial_state", "parareal_apply_fine", "parareal_apply_coarse", "parareal_copy_iterates",
                         "parareal_set_option", "parareal_plan_iteration"):
                getattr(L, name).restype = C.c_int
            _lib = L
    return _lib


def _fp(a: Optional[np.ndarray]):
    return None if a is None else a.ctypes.data_as(C.POINTER(C.c_float))


def _f32(a, shape) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float32).reshape(shape))


def get_nccl_id() -> bytes:
    buf = (C.c_uint8 * 128)()
    st = lib().parareal_get_nccl_id(buf)
    if st:
        raise PararealError(st, lib().parareal_last_error(None).decode())
    return bytes(buf)


def plan_iteration(N: int, world: int, rank: int, k: int) -> dict:
    """parareal_plan_iteration: this rank's share of Parareal iteration k (local indices)."""
    P = Plan()
    st = lib().parareal_plan_iteration(int(N), int(world), int(rank), int(k), C.byref(P))
    if st:
        raise PararealError(st, lib().parareal_last_error(None).decode())
    return {n: getattr(P, n) for n, _ in Plan._fields_}


def _ptr(t) -> Optional[int]:
    """Device pointer of a torch tensor (or an int), None for None."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


class Context:
    """parareal_init … parareal_free.  `problem` is a synth.Problem."""

    def __init__(self, problem: "synth.Problem", rank: int = 0, world: int = 1, device: int = 0,
                 nccl_id: Optional[bytes] = None, stream: Optional[int] = None):
        self.p = problem
        self._keep = [np.ascontiguousarray(problem.strike, np.float64), np.ascontiguousarray(problem.sigma, np.float64),
                      np.ascontiguousarray(problem.rate, np.float64), np.ascontiguousarray(problem.L, np.float64)]
        dp = lambda a: a.ctypes.data_as(C.POINTER(C.c_double))
        s = Problem()
        s.struct_size = C.sizeof(Problem)
        s.M, s.B = int(problem.M), int(problem.B)
        s.strike, s.sigma, s.rate, s.L = (dp(a) for a in self._keep)
        s.T, s.upper_bc, s.N, s.fine_steps = float(problem.T), int(problem.upper_bc), int(problem.N), int(problem.fine_steps)
        s.fine_theta, s.coarse, s.coarse_steps = float(problem.fine_theta), int(problem.coarse), int(problem.coarse_steps)
        s.max_iter, s.tol = int(problem.max_iter), float(problem.tol)
        d = Dist()
        d.rank, d.world, d.device = int(rank), int(world), int(device)
        self._id = None
        if nccl_id is not None:
            self._id = (C.c_uint8 * 128)(*nccl_id)
            d.nccl_id = C.cast(self._id, C.POINTER(C.c_uint8))
        d.stream = stream
        self.rank, self.world = rank, world
        h = C.c_void_p()
        st = lib().parareal_init(C.byref(s), C.byref(d), C.byref(h))
        if st:
            raise PararealError(st, lib().parareal_last_error(None).decode())
        self.h = h
        self._ws = None

    # ------------------------------------------------------------------ helpers
    def _check(self, st: int):
        if st:
            raise PararealError(st, lib().parareal_last_error(self.h).decode())

    @property
    def last_error(self) -> str:
        return lib().parareal_last_error(self.h).decode()

    def close(self):
        if getattr(self, "h", None):
            lib().parareal_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # ------------------------------------------------------------------ ABI calls
    def workspace_bytes(self) -> int:
        n = C.c_size_t()
        self._check(lib().parareal_workspace_bytes(self.h, C.byref(n)))
        return n.value

    def bind_workspace(self, tensor) -> None:
        """Use a caller tensor (e.g. torch.empty(bytes, dtype=torch.uint8, device='cuda')) as workspace."""
        self._check(lib().parareal_bind_workspace(self.h, _ptr(tensor), tensor.numel() * tensor.element_size()))
        self._ws = tensor

    def load_weights(self, net: "synth.Net", precision: int = PREC_FP32) -> None:
        n = net.n_linear
        dims = (C.c_int32 * (n + 1))(*net.dims)
        Ws = [_f32(W, (net.dims[l + 1], net.dims[l])) for l, W in enumerate(net.W)]
        bs = [_f32(b, (net.dims[l + 1],)) for l, b in enumerate(net.b)]
        Wp = (C.POINTER(C.c_float) * n)(*[_fp(w) for w in Ws])
        bp = (C.POINTER(C.c_float) * n)(*[_fp(b) for b in bs])
        ins = _f32(net.scales(), (net.dims[0],))
        self._check(lib().parareal_load_pinn_weights(self.h, n, dims, Wp, bp, int(net.activation), _fp(ins),
                                                     float(net.out_scale), int(precision)))

    def _report(self):
        rep = Report()
        buf = np.zeros(max(self.p.max_iter, 1), np.float64)
        rep.delta = buf.ctypes.data_as(C.POINTER(C.c_double))
        return rep, buf

    @staticmethod
    def _rep_dict(rep: Report, buf: np.ndarray) -> dict:
        k = rep.iterations
        return dict(iterations=k, converged=bool(rep.converged), delta=buf[:k].copy(), ms_total=rep.ms_total,
                    ms_coarse=rep.ms_coarse, ms_fine=rep.ms_fine, ms_comm=rep.ms_comm, ms_setup=rep.ms_setup,
                    kernel_launches=rep.kernel_launches)

    def solve(self, V_T: Optional[np.ndarray] = None) -> Tuple[Optional[np.ndarray], dict]:
        """parareal_solve with host buffers: returns (U^K_N [B][M] on rank 0 else None, report)."""
        B, M = self.p.B, self.p.M
        vt = None if V_T is None else _f32(V_T, (B, M))
        out = np.zeros((B, M), np.float32) if self.rank == 0 else None
        rep, buf = self._report()
        self._check(lib().parareal_solve(self.h, _fp(vt), _fp(out), C.byref(rep)))
        return out, self._rep_dict(rep, buf)

    def solve_device(self, d_V0, d_VT=None) -> dict:
        """parareal_solve_device: d_V0 / d_VT are device tensors (or raw pointers) of [B][M] fp32."""
        rep, buf = self._report()
        self._check(lib().parareal_solve_device(self.h, _ptr(d_VT), _ptr(d_V0), C.byref(rep)))
        return self._rep_dict(rep, buf)

    def solve_host_ptrs(self, V_T_ptr: Optional[int], V_0_ptr: Optional[int], report: bool = True) -> Optional[dict]:
        """parareal_solve with raw host pointers (e.g. pinned torch CPU tensors' data_ptr()); report=False
        passes no report (the ABI's nullable rep) and returns None."""
        fp = C.POINTER(C.c_float)
        vt = C.cast(V_T_ptr, fp) if V_T_ptr else None
        v0 = C.cast(V_0_ptr, fp) if V_0_ptr else None
        if not report:
            self._check(lib().parareal_solve(self.h, vt, v0, None))
            return None
        rep, buf = self._report()
        self._check(lib().parareal_solve(self.h, vt, v0, C.byref(rep)))
        return self._rep_dict(rep, buf)

    def initial_state(self) -> np.ndarray:
        out = np.zeros((self.p.B, self.p.M), np.float32)
        self._check(lib().parareal_initial_state(self.h, _fp(out)))
        return out

    def serial_fine(self, V_T: Optional[np.ndarray] = None) -> Tuple[np.ndarray, float]:
        B, M = self.p.B, self.p.M
        vt = None if V_T is None else _f32(V_T, (B, M))
        out = np.zeros((B, M), np.float32)
        ms = C.c_double()
        self._check(lib().parareal_serial_fine(self.h, _fp(vt), _fp(out), C.byref(ms)))
        return out, ms.value

    def serial_fine_device(self, d_V0, d_VT=None) -> float:
        ms = C.c_double()
        self._check(lib().parareal_serial_fine_device(self.h, _ptr(d_VT), _ptr(d_V0), C.byref(ms)))
        return ms.value

    def apply_fine(self, n: int, U: np.ndarray) -> np.ndarray:
        B, M = self.p.B, self.p.M
        u = _f32(U, (B, M))
        out = np.zeros((B, M), np.float32)
        self._check(lib().parareal_apply_fine(self.h, int(n), _fp(u), _fp(out)))
        return out

    def apply_coarse(self, n: int, U: np.ndarray) -> np.ndarray:
        B, M = self.p.B, self.p.M
        u = _f32(U, (B, M))
        out = np.zeros((B, M), np.float32)
        self._check(lib().parareal_apply_coarse(self.h, int(n), _fp(u), _fp(out)))
        return out

    def copy_iterates(self, n_first: int, n_count: int) -> np.ndarray:
        out = np.zeros((n_count, self.p.B, self.p.M), np.float32)
        self._check(lib().parareal_copy_iterates(self.h, int(n_first), int(n_count), _fp(out)))
        return out

    def set_option(self, key: int, value: int) -> None:
        self._check(lib().parareal_set_option(self.h, int(key), int(value)))
