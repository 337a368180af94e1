"""ctypes binding of libvxq.so (include/vxq.h).

The product path has no CPU fallback: if the shared library is missing or the
GPU is absent, every compute entry point raises ``QubokitError``.
"""

from __future__ import annotations

import ctypes
import math
import os
import threading

import numpy as np

from .errors import QubokitError, ValidationError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_lib", "libvxq.so")
if os.environ.get("VXQ_LIB"):  # A/B experiments: a variant build (build.py --variant)
    LIB_PATH = os.environ["VXQ_LIB"]

VXQ_OK, VXQ_ERR_INVALID, VXQ_ERR_OOM, VXQ_ERR_CUDA, VXQ_ERR_UNSUPPORTED = 0, 1, 2, 3, 4
FP32, FP64 = 0, 1
PATHS = {"auto": 0, "resident": 1, "sparse": 2, "dense": 3}
PATH_NAMES = {v: k for k, v in PATHS.items()}
STEP_KERNELS = {0: None, 1: "k_pa_step", 2: "k_pa_step_coop", 3: "k_pa_cluster",
                4: "k_pa_resident", 5: "k_sbm_step", 6: "k_sbm_block", 7: "k_sbm_resident",
                8: "k_dense_run", 9: "k_sa_run"}
DENSE_KINDS = {0: None, 1: "mxf4", 2: "f8f6f4", 3: "i8x3", 4: "f16x2", 5: "bf16x3", 6: "j16x2",
               7: "jq16"}

i64, u64, f64, i32 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_int32
P = ctypes.c_void_p

# exported symbols, as declared in include/vxq.h (checked by tests/test_boundary.py)
EXPORTS = (
    "vxq_problem_create", "vxq_problem_destroy", "vxq_problem_info", "vxq_problem_lambda0",
    "vxq_problem_c0", "vxq_pa_solve", "vxq_sbm_solve", "vxq_sbm_integrate", "vxq_energies",
    "vxq_pa_schedule", "vxq_sbm_schedule", "vxq_last_error", "vxq_abi_version",
    "vxq_device_count", "vxq_exchange_row_bytes", "vxq_session_create", "vxq_session_step",
    "vxq_session_finish", "vxq_session_destroy", "vxq_problem_generate", "vxq_problem_export",
    "vxq_sa_solve", "vxq_sa_schedule", "vxq_session_set_peers", "vxq_exchange_alloc",
    "vxq_exchange_free", "vxq_ipc_handle", "vxq_ipc_open", "vxq_ipc_close",
    "vxq_dense_eligible", "vxq_problem_eig_info",
)
IPC_HANDLE_BYTES = 64


class PaParamsC(ctypes.Structure):
    _fields_ = [("steps", i64), ("learning_rate", f64), ("momentum", f64), ("lambda0", f64),
                ("replicas", i64), ("seed", u64)]


class SbmParamsC(ctypes.Structure):
    _fields_ = [("steps", i64), ("dt", f64), ("a0", f64), ("c0", f64), ("q_cap", f64),
                ("init_noise", f64), ("replicas", i64), ("seed", u64)]


class SaParamsC(ctypes.Structure):
    _fields_ = [("sweeps", i64), ("T_init", f64), ("T_final", f64), ("replicas", i64),
                ("seed", u64), ("temps", P)]


class RunOptsC(ctypes.Structure):
    _fields_ = [("precision", i32), ("path", i32), ("outputs_on_device", i32),
                ("track_best", i32), ("replica_begin", i64), ("stream", P)]


class OutputsC(ctypes.Structure):
    _fields_ = [("states", P), ("energies", P), ("x", P), ("m", P), ("order", P),
                ("energy_trace", P), ("lambda0_used", f64), ("c0_used", f64), ("loop_ms", f64),
                ("launches", i64), ("path_used", i32), ("dense_kind", i32),
                ("step_kernel", i32), ("reserved", i32)]


_lib = None
_lock = threading.Lock()


def load():
    """Load libvxq.so (building it first if the sources are newer)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            try:
                from . import build as _build
                _build.build()
            except Exception as e:  # pragma: no cover - fails loudly by design
                raise QubokitError(f"libvxq.so is missing and could not be built: {e}") from e
        L = ctypes.CDLL(LIB_PATH)
        L.vxq_problem_create.argtypes = [i64, i64, P, P, P, P, f64, ctypes.c_int,
                                         ctypes.POINTER(P)]
        L.vxq_problem_destroy.argtypes = [P]
        L.vxq_problem_generate.argtypes = [i32, i64, u64, ctypes.c_int, ctypes.POINTER(P)]
        L.vxq_problem_export.argtypes = [P, P, P, P, P, ctypes.POINTER(f64)]
        L.vxq_problem_info.argtypes = [P, P]
        L.vxq_dense_eligible.argtypes = [P, i32, i64, f64, f64, ctypes.POINTER(i32)]
        L.vxq_problem_lambda0.argtypes = [P, ctypes.POINTER(f64)]
        L.vxq_problem_c0.argtypes = [P, ctypes.POINTER(f64)]
        L.vxq_problem_eig_info.argtypes = [P, P]
        L.vxq_pa_solve.argtypes = [P, ctypes.POINTER(PaParamsC), ctypes.POINTER(RunOptsC),
                                   ctypes.POINTER(OutputsC)]
        L.vxq_sbm_solve.argtypes = [P, ctypes.POINTER(SbmParamsC), ctypes.POINTER(RunOptsC),
                                    ctypes.POINTER(OutputsC)]
        L.vxq_sbm_integrate.argtypes = [i64, P, P, P, P, i64, P, P, P, i64, f64, f64, f64, f64,
                                        ctypes.POINTER(RunOptsC)]
        L.vxq_sa_solve.argtypes = [P, ctypes.POINTER(SaParamsC), ctypes.POINTER(RunOptsC),
                                   ctypes.POINTER(OutputsC)]
        L.vxq_sa_schedule.argtypes = [f64, f64, i64, P]
        L.vxq_energies.argtypes = [P, P, i64, P, ctypes.POINTER(RunOptsC)]
        L.vxq_pa_schedule.argtypes = [f64, i64, P]
        L.vxq_sbm_schedule.argtypes = [f64, i64, P]
        L.vxq_exchange_row_bytes.argtypes = [i32, i64, i32, ctypes.POINTER(i64)]
        L.vxq_session_create.argtypes = [P, i32, ctypes.POINTER(PaParamsC),
                                         ctypes.POINTER(SbmParamsC), i64, i64, i64, P, P,
                                         ctypes.POINTER(RunOptsC), ctypes.POINTER(P)]
        L.vxq_session_step.argtypes = [P, i64]
        L.vxq_session_finish.argtypes = [P, ctypes.POINTER(OutputsC)]
        L.vxq_session_destroy.argtypes = [P]
        L.vxq_session_set_peers.argtypes = [P, i32, i32, ctypes.c_uint32, P, P, P]
        L.vxq_exchange_alloc.argtypes = [ctypes.c_int, i64, ctypes.POINTER(P)]
        L.vxq_exchange_free.argtypes = [P]
        L.vxq_ipc_handle.argtypes = [P, P]
        L.vxq_ipc_open.argtypes = [P, ctypes.c_int, ctypes.POINTER(P)]
        L.vxq_ipc_close.argtypes = [P]
        L.vxq_last_error.restype = ctypes.c_char_p
        L.vxq_abi_version.restype = ctypes.c_int
        L.vxq_device_count.restype = ctypes.c_int
        for name in EXPORTS:
            if not hasattr(L, name):
                raise QubokitError(f"libvxq.so does not export {name}")
        _lib = L
    return _lib


def check(rc: int):
    if rc == VXQ_OK:
        return
    msg = load().vxq_last_error().decode(errors="replace")
    if rc == VXQ_ERR_INVALID:
        raise ValidationError(msg)
    raise QubokitError(f"vxq error {rc}: {msg}")


def ptr(a: np.ndarray | None):
    if a is None:
        return None
    if not a.flags["C_CONTIGUOUS"]:
        raise ValueError("array must be C-contiguous")
    return ctypes.c_void_p(a.ctypes.data)


def nan_if_none(v):
    return math.nan if v is None else float(v)


def device_count() -> int:
    return int(load().vxq_device_count())


def require_gpu():
    if device_count() < 1:
        raise QubokitError("no CUDA device visible: the vxq path runs on B200 (sm_100a) only "
                           "and has no CPU fallback")
