"""ctypes binding of the sm_100a C ABI (``include/blreg_b200.h``).

The shared library is built in-tree by ``paper_1807_05117_b200.build``.  There
is no CPU fallback: if the library or a CUDA device is missing, every entry
point raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# BLR_LIB_PATH: an in-tree variant library built by build.py with BLR_OUT_DIR (A/B experiments)
LIB_PATH = os.environ.get("BLR_LIB_PATH") or os.path.join(_HERE, "_lib", "libblreg_b200.so")
if not os.path.isabs(LIB_PATH):  # relative variant paths are relative to the repository root
    LIB_PATH = os.path.join(os.path.dirname(_HERE), LIB_PATH)

_vp, _i, _i64, _d = C.c_void_p, C.c_int, C.c_int64, C.c_double
_ip, _dp = C.POINTER(C.c_int), C.POINTER(C.c_double)

# name -> argtypes (restype is always c_int unless listed in _RESTYPES)
SIGNATURES = {
    "blr_ctx_create": [C.POINTER(_vp), _i, _ip, _ip, _ip, _d, _i, _dp, _i, _i],
    "blr_ctx_destroy": [_vp],
    "blr_set_stream": [_vp, _vp],
    "blr_last_error": [],
    "blr_launch_count": [],
    "blr_version": [],
    "blr_profile_enable": [_i],
    "blr_set_fused_forward": [_i],
    "blr_profile_report": [C.c_char_p, _i64],
    "blr_include": [_vp, _i, _vp, _i, _ip, _vp],
    "blr_project": [_vp, _i, _vp, _i, _vp],
    "blr_helmholtz": [_vp, _vp, _i, _i, _vp],
    "blr_leray": [_vp, _vp, _i, _vp],
    "blr_divergence": [_vp, _vp, _i, _vp],
    "blr_symmetrize": [_vp, _vp, _i, _vp],
    "blr_inner": [_vp, _vp, _vp, _i64, _dp],
    "blr_inner_nodes": [_vp, _vp, _vp, _i, _i64, _dp, _dp],
    "blr_axpby": [_vp, _d, _vp, _d, _vp, _i64],
    "blr_pcg_update": [_vp, _d, _vp, _vp, _vp, _vp, _i64],
    "blr_max_abs": [_vp, _vp, _i64, _dp],
    "blr_sq_dist": [_vp, _vp, _vp, _i64, _dp],
    "blr_all_finite": [_vp, _vp, _i64, _ip],
    "blr_forward_map": [_vp, _vp, _i, _i, _i, _vp, _vp],
    "blr_inverse_map_and_volume": [_vp, _vp, _i, _i, _i, _vp, _vp],
    "blr_state_tangents": [_vp, _vp, _vp, _i, _i, _i, _i, _vp, _vp, _vp, _vp],
    "blr_momentum": [_vp, _vp, _i, _i, _i, _vp, _vp],
    "blr_momentum_tangent": [_vp, _vp, _vp, _i, _i, _i, _vp, _vp, _i, _vp, _vp],
    "blr_contract": [_vp, _vp, _vp, _i, _dp, _i, _vp, _i, _vp],
    "blr_momentum_contract": [_vp, _vp, _i, _i, _i, _vp, _vp, _dp, _i, _vp, _i, _vp],
    "blr_conv_matvec": [_vp, _vp, _vp, _i, _vp],
    "blr_warp": [_vp, _vp, _i, _vp, _i, _i, _vp],
    "blr_grid_gradient": [_vp, _vp, _i, _i, _vp],
    "blr_jacobian_det": [_vp, _vp, _vp],
    "blr_state_gn_accumulate": [_vp, _vp, _vp, _vp, _vp, _i, _dp, _i, _vp],
    "blr_dot_fields": [_vp, _vp, _vp, _d, _vp],
    "blr_scale_fields": [_vp, _vp, _vp, _vp],
    "blr_scaled_diff": [_vp, _vp, _vp, _d, _vp],
    "blr_mul": [_vp, _vp, _vp, _i64, _vp],
    "blr_state_data": [_vp, _vp, _vp, _vp, _i, _dp, _vp],
    "blr_state_newton": [_vp, _vp, _vp, _i, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i, _dp, _i, _vp],
    "blr_lam_matvec_add": [_vp, _vp, _vp, _vp, _vp],
}
_RESTYPES = {"blr_last_error": C.c_char_p, "blr_launch_count": C.c_int64}

_lock = threading.Lock()
_lib = None


class CudaExtensionMissing(RuntimeError):
    """The sm_100a library is not built or cannot be loaded; there is no fallback."""


def load(path: str = LIB_PATH):
    """Load (once) and return the ctypes library handle."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise CudaExtensionMissing(
                f"{path} is missing; build it with `python -m paper_1807_05117_b200.build`")
        lib = C.CDLL(path)
        for name, args in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.argtypes = args
            fn.restype = _RESTYPES.get(name, C.c_int)
        _lib = lib
        return lib


def last_error() -> str:
    return load().blr_last_error().decode(errors="replace")


def launch_count() -> int:
    return int(load().blr_launch_count())


def check(rc: int, name: str):
    if rc == 0:
        return
    msg = f"{name}: {last_error()}"
    if rc == 1:
        raise ValueError(msg)
    raise RuntimeError(msg)


def call(name: str, *args):
    check(getattr(load(), name)(*args), name)


def profile_enable(on: bool = True):
    call("blr_profile_enable", int(bool(on)))


def profile_report() -> dict:
    """Per-category {name: (launches, total_ms, algorithmic_bytes)} since the last report."""
    import json

    buf = C.create_string_buffer(1 << 16)
    call("blr_profile_report", buf, len(buf))
    return {k: tuple(v) for k, v in json.loads(buf.value.decode()).items()}


def int_array(values):
    arr = (C.c_int * len(values))(*[int(v) for v in values])
    return arr


def double_array(values):
    vals = np.ascontiguousarray(values, dtype=np.float64)
    return vals.ctypes.data_as(_dp), vals  # keep vals alive


def out_double():
    return C.c_double(0.0)
