"""B200-native Parareal with a PINN coarse propagator (arXiv 2303.03848).

The hot path lives in libparareal.so (CUDA, sm_100a) behind the C ABI of
include/parareal.h; `parareal` is its ctypes binding, `synth` the seeded
input generators, `report` the Eq. (8) speedup bounds.
"""
from . import report, synth  # noqa: F401
from .parareal import Context, PararealError, get_nccl_id  # noqa: F401

__all__ = ["Context", "PararealError", "get_nccl_id", "synth", "report"]
