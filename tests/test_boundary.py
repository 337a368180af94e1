"""The C-ABI boundary: libvxq.so loads, exports every symbol include/vxq.h declares,
host-only entry points are bit-exact with the reference, and the product path fails
loudly (no CPU fallback) without a GPU.  CPU only."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2501_19221_b200 as vxq
from paper_2501_19221_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "vxq.h")).read()
    return sorted(set(re.findall(r"VXQ_API\s+[\w\s\*]+?\b(vxq_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    L = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)
    assert L.vxq_abi_version() == 5


def header_constants(prefix):
    text = open(os.path.join(ROOT, "include", "vxq.h")).read()
    return {int(v): k for k, v in re.findall(r"#define\s+(" + prefix + r"\w+)\s+(\d+)", text)}


def test_kernel_and_kind_codes_match_header():
    """The names the Python layer reports (info["kernel"], info["dense_kind"]) are the
    header's VXQ_KERNEL_* / VXQ_DENSE_KIND_* codes."""
    kernels = header_constants("VXQ_KERNEL_")
    assert set(kernels) == set(_lib.STEP_KERNELS)
    for code, macro in kernels.items():
        name = _lib.STEP_KERNELS[code]
        if code == 0:
            assert name is None and macro == "VXQ_KERNEL_NONE"
        else:  # VXQ_KERNEL_PA_STEP_COOP <-> k_pa_step_coop
            assert name == "k_" + macro[len("VXQ_KERNEL_"):].lower(), (macro, name)
    kinds = header_constants("VXQ_DENSE_KIND_")
    assert set(kinds) == set(_lib.DENSE_KINDS)
    for code, macro in kinds.items():
        if code:
            assert _lib.DENSE_KINDS[code] == macro[len("VXQ_DENSE_KIND_"):].lower()


def test_struct_layouts_match_header():
    # field order / sizes of the ctypes mirrors (x86-64 SysV)
    assert ctypes.sizeof(_lib.PaParamsC) == 48
    assert ctypes.sizeof(_lib.SbmParamsC) == 64
    assert ctypes.sizeof(_lib.SaParamsC) == 48
    assert ctypes.sizeof(_lib.RunOptsC) == 32
    assert ctypes.sizeof(_lib.OutputsC) == 96
    assert _lib.OutputsC.step_kernel.offset == 88  # ABI 5


@pytest.mark.parametrize("T", [1, 2, 3, 10, 999, 1000, 10_000])
@pytest.mark.parametrize("a0", [1.0, 0.3, 7.77, 1e-300])
def test_sbm_schedule_is_numpy_linspace(T, a0):
    assert np.array_equal(vxq.sbm_schedule(a0, T), np.linspace(0.0, a0, T))


@pytest.mark.parametrize("sweeps", [1, 2, 1000])
def test_sa_schedule_is_reference_expression(sweeps):
    ratio = (0.002 / 2.0) ** (1.0 / (sweeps - 1)) if sweeps > 1 else 1.0
    ref = 2.0 * ratio ** np.arange(sweeps) if sweeps > 1 else np.array([2.0])
    assert np.array_equal(vxq.sa_schedule(2.0, 0.002, sweeps), ref)
    out = np.empty(sweeps)
    assert _lib.load().vxq_sa_schedule(2.0, 0.002, sweeps, _lib.ptr(out)) == 0
    np.testing.assert_allclose(out, ref, rtol=4e-16, atol=0)  # C pow: within an ulp


@pytest.mark.parametrize("T", [1, 7, 1000, 4096])
@pytest.mark.parametrize("lam0", [7.0, 0.3635822054430425, 1e-12, 123.456])
def test_pa_schedule_is_reference_expression(T, lam0):
    ref = np.array([lam0 * (1.0 - t / T) for t in range(T)])
    assert np.array_equal(vxq.pa_schedule(lam0, T), ref)


def test_no_cpu_fallback_without_gpu():
    if _lib.device_count() > 0:
        pytest.skip("GPU present")
    m = vxq.IsingModel.from_terms(2, couplings=[(0, 1, -1.0)])
    with pytest.raises(vxq.QubokitError):
        vxq.solve_pa(m, vxq.PaParams(steps=10, replicas=2))
    with pytest.raises(vxq.QubokitError):
        vxq.solve_sbm(m, vxq.SbmParams(steps=10, replicas=2))
    with pytest.raises(vxq.QubokitError):
        m.energies(np.ones((1, 2), dtype=np.int8))


def test_c_layer_reports_errors_without_gpu():
    if _lib.device_count() > 0:
        pytest.skip("GPU present")
    L = _lib.load()
    h = ctypes.c_void_p()
    rows = np.array([0], dtype=np.int64)
    cols = np.array([1], dtype=np.int64)
    vals = np.array([1.0])
    hv = np.zeros(2)
    rc = L.vxq_problem_create(2, 1, _lib.ptr(rows), _lib.ptr(cols), _lib.ptr(vals),
                              _lib.ptr(hv), 0.0, 0, ctypes.byref(h))
    assert rc != 0 and L.vxq_last_error()


def test_params_validation_before_the_call():
    with pytest.raises(vxq.ValidationError):
        vxq.PaParams(momentum=1.0).validate()
    with pytest.raises(vxq.ValidationError):
        vxq.SbmParams(dt=-0.1).validate()
    with pytest.raises(vxq.ValidationError):
        vxq.PaParams(steps=0).validate()
    with pytest.raises(vxq.ValidationError):
        vxq.params_from_dict("pa", {"stepz": 3})
    p = vxq.PaParams(steps=123, learning_rate=0.07, seed=5)
    assert vxq.params_from_dict("pa", vxq.params_to_dict(p)) == p
    q = vxq.SbmParams(steps=10, dt=0.2, c0=0.5)
    assert vxq.params_from_dict("sbm", vxq.params_to_dict(q)) == q
    # SaParams.validate (common.py:84-91)
    for bad in (dict(sweeps=0), dict(replicas=0), dict(schedule="linear"),
                dict(T_init=1.0, T_final=2.0), dict(T_init=1.0, T_final=0.0)):
        with pytest.raises(vxq.ValidationError):
            vxq.SaParams(**bad).validate()
    a = vxq.SaParams(sweeps=77, T_init=3.0, T_final=0.5, replicas=8, seed=2)
    assert vxq.params_from_dict("sa", vxq.params_to_dict(a)) == a
    with pytest.raises(vxq.ValidationError):
        vxq.params_from_dict("sa", {"swups": 10})
    # model validation (model.py:81-104)
    with pytest.raises(vxq.ValidationError):
        vxq.IsingModel.from_terms(3, couplings=[(1, 1, 2.0)])
    with pytest.raises(vxq.ValidationError):
        vxq.IsingModel.from_terms(3, couplings=[(0, 5, 2.0)])
    with pytest.raises(vxq.ValidationError):
        vxq.IsingModel.from_terms(0)
