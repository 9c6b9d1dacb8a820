"""The C ABI library (CPU only): it loads, exports every function
include/dnnscaler_b200.h declares, and its device-free entry points work;
device entry points fail loudly (no CPU fallback) when there is no GPU.
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2308_13803_b200 import _lib
from paper_2308_13803_b200.backend import kernel_costs, model_info

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dnnscaler_b200.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ds_[a-z0-9_]+)\s*\(", text)))


def test_every_declared_symbol_is_exported():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) > 40
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (ds_[a-z0-9_]+)", out))
    assert set(names) <= exported


def test_library_is_native_sm100a():
    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_device_free_entry_points():
    mi = model_info("mobilenet_v1")
    assert (mi.in_h, mi.in_w, mi.classes) == (224, 224, 1000)
    ks = kernel_costs("resnet50_v1")
    # the 7x7/2 stem runs over a space-to-depth input: a staging launch
    # (u8 image in, [115][115][16] bf16 out) then the stem conv
    assert ks[0]["kind"] == "stage" and ks[1]["kind"] == "conv_gemm" and ks[-1]["kind"] == "softmax"
    assert ks[0]["bytes_per_image"] == 224 * 224 * 3 + 115 * 115 * 16 * 2
    # the stride-1 synthetic stem reads the u8 images itself (staging fused)
    ks_syn = kernel_costs("synthetic_cnn")
    assert ks_syn[0]["kind"] == "conv_gemm"
    assert ks_syn[0]["bytes_per_image"] < 32 * 32 * 3 + 32 * 32 * 32 * 2 + 1
    assert abs(sum(k["flops_per_image"] for k in ks) - 2 * model_info("resnet50_v1").macs_per_image) < 1
    with pytest.raises(ValueError, match="unknown model"):
        model_info("vgg16")


def test_launch_plan_one_kernel_per_layer():
    """Host-side launch plan: the space-to-depth staging kernel (stride-2
    stems; the stride-1 synthetic stem reads the u8 images itself), one kernel
    per layer, softmax; the kernel count and algorithmic FLOPs match the model."""
    from paper_2308_13803_b200 import model_info
    for model, staging in (("synthetic_cnn", 0), ("mobilenet_v1", 1), ("resnet50_v1", 1),
                           ("inception_v3", 1)):
        ks = kernel_costs(model)
        assert [k["kind"] for k in ks].count("stage") == staging, model
        assert ks[-1]["kind"] == "softmax"
        assert abs(sum(k["flops_per_image"] for k in ks) - 2 * model_info(model).macs_per_image) < 1
    kinds = [k["kind"] for k in kernel_costs("mobilenet_v1")]
    assert kinds.count("dwconv") == 13 and kinds.count("conv_gemm") == 15


def test_device_calls_fail_loudly_without_gpu():
    import torch

    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    lib = _lib.load()
    h = ctypes.c_void_p()
    st = lib.ds_backend_create(b"synthetic_cnn", _lib.DsConfig(8, 2), 42, 0, ctypes.byref(h))
    assert st == _lib.DS_ECUDA and not h
    assert "cuda" in _lib.last_error().lower() or "CUDA" in _lib.last_error()


def test_null_handles_are_errors():
    lib = _lib.load()
    lat = ctypes.c_double()
    assert lib.ds_run_batch(None, 1, ctypes.byref(lat)) == _lib.DS_EINVAL
    assert lib.ds_mtl(None) == 0


def test_graph_rewrites_keep_the_algorithm(monkeypatch):
    """Build-time rewrites (model.hpp fuse_sibling_1x1, swap_avgpool_1x1):
    fewer launches, the same algorithmic FLOPs, no more algorithmic bytes
    (a fused launch reads its shared input once; the swapped pool runs over
    the conv's channels instead of its input's)."""
    from paper_2308_13803_b200 import model_info

    def plan(model, fuse, swap):
        monkeypatch.setenv("DS_FUSE_1X1", "1" if fuse else "0")
        monkeypatch.setenv("DS_POOL_SWAP", "1" if swap else "0")
        ks = kernel_costs(model)
        return (len(ks), sum(k["flops_per_image"] for k in ks),
                sum(k["bytes_per_image"] for k in ks), [k["kind"] for k in ks])

    for model in ("resnet50_v1", "inception_v3", "mobilenet_v1"):
        n0, f0, b0, _ = plan(model, False, False)
        n1, f1, b1, kinds1 = plan(model, True, True)
        macs2 = 2 * model_info(model).macs_per_image
        assert abs(f0 - macs2) < 1 and abs(f1 - macs2) < 1, model
        assert b1 <= b0 + 1, model
        if model == "mobilenet_v1":
            assert n1 == n0  # no siblings, no average pools
    n_plain = plan("inception_v3", False, False)[0]
    n_fused = plan("inception_v3", True, False)[0]
    n_both, _, _, kinds = plan("inception_v3", True, True)
    # 3 Inception-A blocks: 3 sibling heads -> 1 (2 launches each); B: none;
    # 4 C blocks: 3 -> 1; D: 2 -> 1; 2 E blocks: 3 -> 1
    assert n_plain - n_fused == 3 * 2 + 4 * 2 + 1 + 2 * 2
    # the 9 branch avgpool -> 1x1 pairs: the 1x1 joins its block's fused heads
    assert n_fused - n_both == 9
    assert kinds.count("pool") == plan("inception_v3", False, False)[3].count("pool")
    # ResNet: the first block of each stage fuses conv1 with the projection
    assert plan("resnet50_v1", False, False)[0] - plan("resnet50_v1", True, True)[0] == 4
