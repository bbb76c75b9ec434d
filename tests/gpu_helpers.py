"""Shared helpers for the GPU parity tests (tolerance of reading Q17)."""
import numpy as np

TOL_FP32 = 1e-5   # north_star: "within 1e-5 relative (FP32) per grid value"


def assert_close(gpu, ref, tol=TOL_FP32, what=""):
    """|gpu_j - ref_j| <= tol |ref_j| + tol ||ref_row||_inf, row = one instance state (Q17)."""
    g = np.asarray(gpu, np.float64)
    r = np.asarray(ref, np.float64)
    assert g.shape == r.shape, (g.shape, r.shape)
    r2 = r.reshape(-1, r.shape[-1])
    g2 = g.reshape(-1, g.shape[-1])
    scale = np.max(np.abs(r2), axis=1, keepdims=True)
    bound = tol * np.abs(r2) + tol * scale
    err = np.abs(g2 - r2)
    bad = err > bound
    if bad.any():
        i = np.unravel_index(np.argmax(err / np.maximum(bound, 1e-300)), err.shape)
        raise AssertionError("%s: %d/%d values outside tolerance; worst row %d col %d gpu=%r ref=%r bound=%g"
                             % (what, bad.sum(), bad.size, i[0], i[1], g2[i], r2[i], bound[i]))


def rel_err(gpu, ref):
    g = np.asarray(gpu, np.float64)
    r = np.asarray(ref, np.float64)
    return float(np.max(np.abs(g - r)) / max(np.max(np.abs(r)), 1e-300))


def assert_delta(got, ref, what="delta"):
    """δ^k (reading Q13) is a ratio of l2 norms of fp32-stored states: GPU and oracle agree to
    rtol 1e-3 (north_star's TC tolerance) plus an absolute 5e-7, a few fp32 roundings of the
    states it is formed from (2^-24 ~ 6e-8 per value; Q15 fp32 storage) -- the absolute part
    matters only when δ itself is near the fp32 floor."""
    g = np.asarray(got, np.float64)
    r = np.asarray(ref, np.float64)
    assert g.shape == r.shape, (what, g.shape, r.shape)
    assert np.allclose(g, r, rtol=1e-3, atol=5e-7), (what, g, r)
