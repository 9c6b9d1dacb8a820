"""Layer-by-layer device vs FP32-oracle diff for one image (debug tool).

    python tools/debug_layers.py inception_v3 [image_index]
"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402
from paper_2308_13803_b200 import Config, GpuBackend, _lib  # noqa: E402

model = sys.argv[1]
idx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
img = oracle.images(model, idx, 1)
lib = oracle.fwd()
lib.oracle_debug_buffer.restype = ctypes.c_long
lib.oracle_debug_buffer.argtypes = [ctypes.c_char_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_void_p]
L = _lib.load()
L.ds_debug_read_buffer.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_void_p,
                                   ctypes.c_size_t, ctypes.POINTER(ctypes.c_size_t)]
be = GpuBackend(model, Config(abs_max_bs=1, max_mtl=1))
be.forward(img)
b = 1
worst = []
while True:
    n = lib.oracle_debug_buffer(model.encode(), img.ctypes.data, 1, b, None)
    if n < 0:
        break
    ref = np.empty(n, np.float32)
    lib.oracle_debug_buffer(model.encode(), img.ctypes.data, 1, b, ref.ctypes.data)
    ln = ctypes.c_size_t()
    if L.ds_debug_read_buffer(be._h, b, 1, None, 0, ctypes.byref(ln)) != 0:
        break
    raw = np.empty(ln.value, np.uint8)
    L.ds_debug_read_buffer(be._h, b, 1, raw.ctypes.data, raw.size, ctypes.byref(ln))
    if ln.value == 4 * n:
        dev = raw.view(np.float32)
    else:
        dev = (raw.view(np.uint16).astype(np.uint32) << 16).view(np.float32)
    err = np.abs(dev - ref).max() / max(1e-6, np.abs(ref).max())
    nbad = int((np.abs(dev - ref) > 0.05 * np.abs(ref).max()).sum())
    print(f"buffer {b:3d} n={n:8d} max|ref|={np.abs(ref).max():9.3f} rel_err={err:.2e} bad={nbad}")
    b += 1
