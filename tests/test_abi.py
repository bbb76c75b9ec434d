"""The C-ABI library loads and exports what include/parareal.h declares; host-side
validation runs before any device call, so it is testable without a GPU."""
import os
import re

import numpy as np
import pytest

from paper_2303_03848_b200 import parareal, pinn_train, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions(header="parareal.h", prefix="parareal_"):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(%s\w+)\s*\(" % prefix, src)))


def _all_declared():
    return _header_functions() + _header_functions("pinn_train.h", "pinn_train_")


def test_header_matches_binding_list():
    assert _header_functions() == sorted(parareal.EXPORTS)
    assert _header_functions("pinn_train.h", "pinn_train_") == sorted(pinn_train.EXPORTS)


def test_library_exports_every_declared_symbol():
    L = parareal.lib()
    for name in _all_declared():
        assert hasattr(L, name), name


def test_exports_are_c_symbols():
    """nm -D: every declared entry point is an unmangled global text symbol."""
    import subprocess
    out = subprocess.check_output(["nm", "-D", "--defined-only", parareal.LIB_PATH]).decode()
    syms = {l.split()[-1] for l in out.splitlines() if " T " in l}
    for name in _all_declared():
        assert name in syms, name


def test_status_strings():
    L = parareal.lib()
    for code, name in parareal.STATUS.items():
        assert L.parareal_status_string(code).decode() == name


def test_library_has_sm100a_code():
    """The fatbin carries sm_100a SASS (cuobjdump lists the ELF for that arch)."""
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.check_output([exe, "--list-elf", parareal.LIB_PATH]).decode()
    assert "sm_100a" in out


@pytest.mark.parametrize("field,kw,frag", [
    ("M", dict(M=0), "problem.M"),
    ("N", dict(N=0), "problem.N"),
    ("fine_steps", dict(fine_steps=0), "problem.fine_steps"),
    ("sigma", dict(sigma=np.array([0.0])), "problem.sigma[0]"),
    ("rate", dict(rate=np.array([-0.1])), "problem.rate[0]"),
    ("L", dict(L=np.array([0.5])), "problem.L[0]"),
    ("strike", dict(strike=np.array([-1.0]), L=np.array([4.0])), "problem.strike[0]"),
    ("T", dict(T=0.0), "problem.T"),
    ("max_iter", dict(max_iter=5), "problem.max_iter"),
    ("tol", dict(tol=-1.0), "problem.tol"),
    ("coarse_steps", dict(coarse=synth.COARSE_IMPLICIT_EULER, coarse_steps=0), "problem.coarse_steps"),
    ("upper_bc", dict(upper_bc=7), "problem.upper_bc"),
])
def test_init_validation_names_the_field(field, kw, frag):
    p = synth.config("C1").replace(**kw)
    with pytest.raises(parareal.PararealError) as ei:
        parareal.Context(p)
    assert ei.value.status == 1 and frag in str(ei.value), str(ei.value)


@pytest.mark.parametrize("theta", [0.3, 0.0, 1.5, float("nan")])
def test_init_rejects_theta_outside_stable_range(theta):
    """θ-step fine propagator: θ in [1/2, 1] (CN .. implicit Euler); others are rejected by name."""
    with pytest.raises(parareal.PararealError) as ei:
        parareal.Context(synth.config("C1").replace(fine_theta=theta))
    assert ei.value.status == 1 and "fine_theta" in str(ei.value), str(ei.value)


def test_init_rejects_bad_partition():
    with pytest.raises(parareal.PararealError) as ei:
        parareal.Context(synth.config("C1"), rank=0, world=3, nccl_id=bytes(128))
    assert ei.value.status == 1 and "divisible" in str(ei.value)


def test_no_cpu_fallback_without_gpu():
    """A valid problem on a box without a GPU fails loudly with PR_ERR_CUDA (never a CPU path)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(parareal.PararealError) as ei:
        parareal.Context(synth.config("C1"))
    assert ei.value.status == 3


# ---------------------------------------------------------------- pinn_train.h validation (no device call)

_MK = dict(K=1.0, sigma=0.2, r=0.05, T=1.0, L=4.0)


@pytest.mark.parametrize("change,frag", [
    (dict(market=dict(_MK, sigma=0.0)), "cfg.sigma"),
    (dict(market=dict(_MK, L=-1.0)), "cfg.L"),
    (dict(dims=[3, 20, 1]), "cfg.dims"),
    (dict(dims=[2, 20, 16, 1]), "hidden widths"),
    (dict(dims=[2, 24, 24, 1]), "hidden width 24"),
    (dict(batches=0), "cfg.batches"),
    (dict(batches=1000), "cfg.batches"),
    (dict(beta1=1.0), "cfg.beta1"),
])
def test_pinn_train_init_validates_before_touching_the_device(change, frag):
    dims = change.get("dims", [2, 20, 20, 1])
    net = synth.pinn2_net([2 if i == 0 and dims[0] == 2 else d for i, d in enumerate(dims)], seed=0) \
        if dims[0] == 2 else synth.kaiming_net(dims, seed=0)
    sets = synth.collocation(_MK, 500, 50, 50, seed=0)
    with pytest.raises(parareal.PararealError) as ei:
        pinn_train.Trainer(net, change.get("market", _MK), sets, batches=change.get("batches", 5),
                           beta1=change.get("beta1", 0.9))
    assert frag in str(ei.value)
