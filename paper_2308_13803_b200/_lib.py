"""ctypes binding of libdnnscaler_b200.so (the C ABI in include/dnnscaler_b200.h).

The shared library is built in-tree (``make -C paper_2308_13803_b200``) and is
the only compute path: there is no Python or CPU fallback. Loading fails
loudly when the library is missing.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libdnnscaler_b200.so")

DS_OK, DS_EINVAL, DS_ERUNTIME, DS_ECUDA = 0, 1, 2, 3


class DsError(RuntimeError):
    """Non-EINVAL failure of a ds_* call (runtime or CUDA)."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status


class DsConfig(ctypes.Structure):
    _fields_ = [("abs_max_bs", ctypes.c_int), ("max_mtl", ctypes.c_int)]


class DsModelInfo(ctypes.Structure):
    _fields_ = [
        ("in_h", ctypes.c_int),
        ("in_w", ctypes.c_int),
        ("classes", ctypes.c_int),
        ("n_ops", ctypes.c_int),
        ("n_params", ctypes.c_int),
        ("macs_per_image", ctypes.c_double),
        ("weight_count", ctypes.c_double),
        ("act_bytes_per_image", ctypes.c_double),
        ("feature_buffer", ctypes.c_int),
        ("feature_channels", ctypes.c_int),
        ("head_k", ctypes.c_int),
    ]


class DsBackendStats(ctypes.Structure):
    _fields_ = [
        ("kernel_launches", ctypes.c_int64),
        ("h2d_bytes", ctypes.c_int64),
        ("d2h_bytes", ctypes.c_int64),
        ("instances_created", ctypes.c_int),
        ("kernels_per_forward", ctypes.c_int),
        ("device_bytes", ctypes.c_double),
    ]


class DsKernelCost(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int), ("flops_per_image", ctypes.c_double),
                ("bytes_per_image", ctypes.c_double), ("fixed_bytes", ctypes.c_double)]


_c_double_p = ctypes.POINTER(ctypes.c_double)
_vp = ctypes.c_void_p

# name -> (restype, argtypes)
SIGNATURES = {
    "ds_last_error": (ctypes.c_char_p, []),
    "ds_backend_create": (
        ctypes.c_int,
        [ctypes.c_char_p, DsConfig, ctypes.c_uint64, ctypes.c_int, ctypes.POINTER(_vp)],
    ),
    "ds_backend_destroy": (None, [_vp]),
    "ds_run_batch": (ctypes.c_int, [_vp, ctypes.c_int, _c_double_p]),
    "ds_run_mt_request": (ctypes.c_int, [_vp, _c_double_p]),
    "ds_apply_instance_change": (ctypes.c_int, [_vp, ctypes.c_int, _c_double_p]),
    "ds_set_mtl": (ctypes.c_int, [_vp, ctypes.c_int, _c_double_p]),
    "ds_mtl": (ctypes.c_int, [_vp]),
    "ds_clock_ms": (ctypes.c_double, [_vp]),
    "ds_get_config": (DsConfig, [_vp]),
    "ds_run_batches": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp]),
    "ds_run_mt_requests": (ctypes.c_int, [_vp, ctypes.c_int, _vp]),
    "ds_run_combo_requests": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, _vp]),
    "ds_forward": (ctypes.c_int, [_vp, _vp, ctypes.c_int, _vp, _vp]),
    "ds_set_host_io": (ctypes.c_int, [_vp, ctypes.c_int]),
    "ds_drain": (ctypes.c_int, [_vp]),
    "ds_nvtx_push": (None, [ctypes.c_char_p]),
    "ds_nvtx_pop": (None, []),
    "ds_timer_start": (ctypes.c_int, [_vp]),
    "ds_timer_stop": (ctypes.c_int, [_vp, _c_double_p]),
    "ds_set_mt_mode": (ctypes.c_int, [_vp, ctypes.c_int]),
    "ds_get_mt_mode": (ctypes.c_int, [_vp]),
    "ds_kernel_spans": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_int64)]),
    "ds_last_output": (ctypes.c_int, [_vp, ctypes.c_int, _vp, ctypes.c_size_t,
                                       ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)]),
    "ds_model_info_get": (ctypes.c_int, [ctypes.c_char_p, ctypes.POINTER(DsModelInfo)]),
    "ds_backend_stats_get": (ctypes.c_int, [_vp, ctypes.POINTER(DsBackendStats)]),
    "ds_model_kernels": (
        ctypes.c_int,
        [ctypes.c_char_p, ctypes.POINTER(DsKernelCost), ctypes.c_int, ctypes.POINTER(ctypes.c_int)],
    ),
    "ds_profile_kernels": (ctypes.c_int, [_vp, ctypes.c_int, ctypes.c_int, _vp, ctypes.c_int]),
    "ds_generate_images": (
        ctypes.c_int,
        [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, _vp],
    ),
    "ds_model_param": (
        ctypes.c_int,
        [
            ctypes.c_char_p,
            ctypes.c_int,
            _vp,
            ctypes.c_size_t,
            ctypes.POINTER(ctypes.c_size_t),
            _vp,
            ctypes.c_size_t,
            ctypes.POINTER(ctypes.c_size_t),
            ctypes.POINTER(ctypes.c_int),
        ],
    ),
}

_lib = None


def load() -> ctypes.CDLL:
    """Loads the in-tree library once; raises if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `make -C paper_2308_13803_b200` "
            "(there is no fallback implementation)"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().ds_last_error()
    return msg.decode() if msg else ""


def check(status: int) -> None:
    """Maps a ds_status to the reference's exception types."""
    if status == DS_OK:
        return
    msg = last_error()
    if status == DS_EINVAL:
        raise ValueError(msg)  # std::invalid_argument in the reference
    raise DsError(status, msg)
