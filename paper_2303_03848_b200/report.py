"""Reporting helpers: the speedup bounds of PAPER.md Eq. (8).

s_bound(P) = 1 / ((1 + K/P) c_c/c_f + K/P)   -- the pipelined Parareal cost model
                                               (P c_f) / ((P+K) c_c + K c_f)  (reading Q19)
s_block(P) = 1 / ((K+1) c_c/c_f + K/P)       -- a blocking schedule: (K+1) full coarse sweeps
                                               of P c_c each plus K fine sweeps of c_f.
"""


def speedup_bound(K: float, P: float, ratio: float) -> float:
    """Eq. (8): K iterations, P processes (= slices), ratio = c_c / c_f."""
    return 1.0 / ((1.0 + K / P) * ratio + K / P)


def speedup_bound_blocking(K: float, P: float, ratio: float) -> float:
    """Bound for the non-pipelined schedule this build runs (Q19)."""
    return 1.0 / ((K + 1.0) * ratio + K / P)
