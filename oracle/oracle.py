"""ctypes access to the CPU oracles — TEST INFRASTRUCTURE ONLY.

Importable only from tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference leg, as the checker or the CPU baseline.
The product package never imports this module.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
FWD_LIB = os.path.join(HERE, "_build", "liboracle_fwd.so")
REF_LIB = os.path.join(HERE, "_ref", "libref_replay.so")
HEAD_DIR = os.environ.get("DS_HEAD_DIR") or os.path.join(os.path.dirname(HERE),
                                                         "paper_2308_13803_b200", "data", "heads")

_fwd = None


def fwd() -> ctypes.CDLL:
    global _fwd
    if _fwd is None:
        if not os.path.exists(FWD_LIB):
            raise ImportError(f"{FWD_LIB} missing: run `make -C oracle`")
        lib = ctypes.CDLL(FWD_LIB)
        lib.oracle_forward.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_void_p]
        lib.oracle_generate_images.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64,
                                               ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
        lib.oracle_model_info.argtypes = [ctypes.c_char_p] + [ctypes.c_void_p] * 5
        lib.oracle_param_device_layout.argtypes = [
            ctypes.c_char_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t,
            ctypes.POINTER(ctypes.c_size_t), ctypes.c_void_p, ctypes.POINTER(ctypes.c_int)]
        lib.oracle_set_threads.argtypes = [ctypes.c_int]
        lib.oracle_get_threads.restype = ctypes.c_int
        lib.oracle_debug_features.argtypes = [ctypes.c_void_p]
        lib.oracle_set_head_dir.argtypes = [ctypes.c_char_p]
        # The calibrated classifier heads are model data shared with the
        # product (same directory the product library reads).
        lib.oracle_set_head_dir(HEAD_DIR.encode())
        _fwd = lib
    return _fwd


def model_info(model: str) -> dict:
    h, w, c, n = ctypes.c_int(), ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    macs = ctypes.c_double()
    if fwd().oracle_model_info(model.encode(), ctypes.byref(h), ctypes.byref(w), ctypes.byref(c),
                               ctypes.byref(n), ctypes.byref(macs)):
        raise ValueError(model)
    return {"in_h": h.value, "in_w": w.value, "classes": c.value, "n_params": n.value,
            "macs": macs.value}


def images(model: str, first: int, count: int, seed: int = 42) -> np.ndarray:
    info = model_info(model)
    out = np.empty((count, info["in_h"], info["in_w"], 3), dtype=np.uint8)
    fwd().oracle_generate_images(info["in_h"], info["in_w"], seed, first, count, out.ctypes.data)
    return out


def forward(model: str, imgs: np.ndarray, bf16_storage: bool = True,
            threads: int = 0) -> np.ndarray:
    info = model_info(model)
    imgs = np.ascontiguousarray(imgs, dtype=np.uint8)
    out = np.empty((imgs.shape[0], info["classes"]), dtype=np.float32)
    fwd().oracle_set_threads(threads)
    if fwd().oracle_forward(model.encode(), imgs.ctypes.data, imgs.shape[0],
                            1 if bf16_storage else 0, out.ctypes.data):
        raise ValueError(model)
    return out


def param_device_layout(model: str, layer: int):
    n = ctypes.c_size_t()
    kp = ctypes.c_int()
    lib = fwd()
    if lib.oracle_param_device_layout(model.encode(), layer, None, 0, ctypes.byref(n), None,
                                      ctypes.byref(kp)):
        raise ValueError((model, layer))
    w = np.zeros(n.value, dtype=np.uint16)
    b = np.zeros(4096, dtype=np.float32)
    lib.oracle_param_device_layout(model.encode(), layer, w.ctypes.data, n.value, ctypes.byref(n),
                                   b.ctypes.data, ctypes.byref(kp))
    return w, b, kp.value
