"""Pinning the oracles (CPU only).

The logits oracle (oracle/fwd_oracle.c) cannot be pinned to the reference
(it has no forward pass); it is pinned to
  * an independent torch.nn.functional execution of the same layers
    (tests/golden/xcheck_*.npz, made by tests/golden/torch_xcheck.py),
  * the reference's generator (tests/golden/ref_random.json, dumped from the
    compiled reference's RandomStream / mix_seed),
  * published architecture sizes and torchvision's Inception-v3 layout.
The product's host-side weight/image generation must equal the oracle's.
"""
import ctypes
import json
import os

import numpy as np
import pytest

import oracle
import ref as refo
from paper_2308_13803_b200 import _lib, generate_images
from paper_2308_13803_b200.backend import model_info

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
MODELS = ["synthetic_cnn", "mobilenet_v1", "resnet50_v1", "inception_v3"]


def _random(lib_fn, seed, n=1000):
    u, g, m = np.zeros(n, np.uint64), np.zeros(n), np.zeros(n, np.uint64)
    lib_fn(ctypes.c_uint64(seed), n, u.ctypes.data_as(ctypes.c_void_p),
           g.ctypes.data_as(ctypes.c_void_p), m.ctypes.data_as(ctypes.c_void_p))
    return u, g, m


def test_oracle_rng_matches_reference_fixture():
    fix = json.load(open(os.path.join(GOLDEN, "ref_random.json")))
    for seed, exp in fix.items():
        u, g, m = _random(oracle.fwd().oracle_random, int(seed))
        assert [int(v) for v in u[:16]] == exp["u64"]
        assert int(u[999]) == exp["u64_999"]
        assert [float(v).hex() for v in g[:16]] == exp["gauss"]
        assert float(g[999]).hex() == exp["gauss_999"]
        assert [int(v) for v in m[:8]] == exp["mix"]


@pytest.mark.skipif(not refo.available(), reason="oracle/_ref not built")
def test_oracle_rng_matches_live_reference():
    for seed in (1, 99, 2 ** 40 + 3):
        a = _random(refo.lib().ref_random, seed)
        b = _random(oracle.fwd().oracle_random, seed)
        for x, y in zip(a, b):
            assert np.array_equal(x.view(np.uint64), y.view(np.uint64))


@pytest.mark.parametrize("model", MODELS)
def test_oracle_matches_torch_crosscheck(model):
    fix = np.load(os.path.join(GOLDEN, f"xcheck_{model}.npz"))
    ref = fix["logits"]
    ours = oracle.forward(model, oracle.images(model, int(fix["image_first"]), ref.shape[0]),
                          bf16_storage=False)
    rel = np.abs(ours - ref).max(1) / np.abs(ref).max(1)
    assert rel.max() < 1e-4, rel


@pytest.mark.parametrize("model", MODELS)
def test_product_weights_and_images_equal_oracle(model):
    lib = _lib.load()
    info = oracle.model_info(model)
    assert info["n_params"] == model_info(model).n_params
    for layer in range(info["n_params"]):
        w_or, b_or, kp_or = oracle.param_device_layout(model, layer)
        n = ctypes.c_size_t()
        bl = ctypes.c_size_t()
        kp = ctypes.c_int()
        w = np.zeros(w_or.size, np.uint16)
        b = np.zeros(4096, np.float32)
        _lib.check(lib.ds_model_param(model.encode(), layer, w.ctypes.data, w.size, ctypes.byref(n),
                                      b.ctypes.data, b.size, ctypes.byref(bl), ctypes.byref(kp)))
        assert kp.value == kp_or and n.value == w_or.size
        assert np.array_equal(w, w_or), (model, layer)
        assert np.array_equal(b[:bl.value], b_or[:bl.value]), (model, layer)
    assert np.array_equal(generate_images(model, 5, 3), oracle.images(model, 5, 3))


def test_architecture_sizes():
    # multiply-accumulates per image (real channels) and parameter counts:
    # MobileNet-v1 1.0/224: 569 M MACs, 4.2 M params (Howard et al. Table 1);
    # ResNet-50 v1 (stride on 1x1): 3.86 G MACs; Inception-v3/299: 5.71 G MACs
    # (SURVEY §6 layer-hook probe); synthetic CNN of config 1.
    expect = {"mobilenet_v1": (568.74e6, 4.23e6), "resnet50_v1": (3857.97e6, 25.53e6),
              "inception_v3": (5713.2e6, 23.82e6), "synthetic_cnn": (10.3232e6, 0.0945e6)}
    for model, (macs, params) in expect.items():
        mi = model_info(model)
        assert abs(mi.macs_per_image - macs) / macs < 1e-4, (model, mi.macs_per_image)
        assert abs(mi.weight_count - params) / params < 5e-3, (model, mi.weight_count)
        assert abs(oracle.model_info(model)["macs"] - mi.macs_per_image) < 1.0


def test_inception_layout_matches_torchvision():
    tv = pytest.importorskip("torchvision")
    import torch.nn as nn

    net = tv.models.inception_v3(weights=None, aux_logits=False, init_weights=False)
    tv_convs = [(m.out_channels, m.kernel_size, m.stride, m.padding)
                for m in net.modules() if isinstance(m, nn.Conv2d)]
    L = oracle.fwd()
    L.oracle_num_ops.argtypes = [ctypes.c_char_p]
    L.oracle_op.argtypes = [ctypes.c_char_p, ctypes.c_int, ctypes.c_void_p]
    ours = []
    for i in range(L.oracle_num_ops(b"inception_v3")):
        f = np.zeros(14, np.int32)
        L.oracle_op(b"inception_v3", i, f.ctypes.data)
        if f[0] == 0:  # conv
            ours.append((int(f[13]), (int(f[5]), int(f[6])), (int(f[7]), int(f[8])),
                         (int(f[9]), int(f[10]))))
    # torchvision defines branch modules in the same order the oracle emits them
    assert sorted(ours) == sorted(tv_convs)
    assert len(ours) == len(tv_convs) == 94


def test_stem_normalisation_exact():
    """The fused stem producer (conv_gemm kStemU8) normalises a pixel byte as
    bf16_rn((p - 127.5f) * (1/63.75f)); the staging kernel and the oracle use
    bf16_rn((p - 127.5f) / 63.75f). The fp32 intermediates differ for some p,
    but the bf16 results agree for every byte value (exhaustive)."""
    def bf16_rn(x):
        u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
        return (((u + 0x7FFF + ((u >> 16) & 1)) >> 16) & 0xFFFF).astype(np.uint16)

    p = np.arange(256, dtype=np.float32)
    t = (p - np.float32(127.5)).astype(np.float32)
    div = bf16_rn((t / np.float32(63.75)).astype(np.float32))
    mul = bf16_rn((t * (np.float32(1) / np.float32(63.75))).astype(np.float32))
    assert np.array_equal(div, mul)


@pytest.mark.parametrize("model", MODELS)
def test_top1_fixture_reproduces(model):
    """The 4,096-image top-1 fixture (tests/golden/make_top1.py) is the
    current oracle's verdict: its first images re-run here."""
    g = np.load(os.path.join(GOLDEN, f"top1_{model}.npz"))
    n = 8
    ref = oracle.forward(model, oracle.images(model, 0, n), bf16_storage=False)
    assert np.array_equal(ref.argmax(1), g["top1_32"][:n])
    s = np.sort(ref, 1)
    np.testing.assert_allclose(s[:, -1] - s[:, -2], g["margin_32"][:n], rtol=1e-5, atol=1e-6)


def test_heads_shared_with_product():
    """Product and oracle build the FC from the same calibrated head files."""
    for model in MODELS:
        assert model_info(model).head_k > 0, model
        assert os.path.exists(os.path.join(oracle.HEAD_DIR, model + ".head"))
