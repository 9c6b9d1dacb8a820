"""Kernel-mode A/B tests: every non-default conv / depthwise / pool / stem
variant against the path it replaces, on the same seeded inputs (bit-identical
where the K order is the same). Regression tests of the product against
itself; the oracle parity tests are in test_forward_parity_gpu.py.
"""
import numpy as np
import pytest

from paper_2308_13803_b200 import Config, GpuBackend, generate_images

pytestmark = pytest.mark.gpu

REL_TOL = 4e-2


def row_rel_err(dev, ref):
    """max|dev - ref| per row over the row's input-dependent logit range."""
    return np.abs(dev - ref).max(axis=1) / np.abs(ref).max(axis=1)


def test_forward_deterministic_and_batch_invariant():
    imgs = generate_images("mobilenet_v1", 100, 6)
    with GpuBackend("mobilenet_v1", Config(abs_max_bs=8, max_mtl=1)) as be:
        a = be.forward(imgs)
        b = be.forward(imgs)
        one = np.concatenate([be.forward(imgs[i:i + 1]) for i in range(6)])
    assert np.array_equal(a, b)
    # Row results do not depend on batch composition (no cross-row reduction).
    assert np.array_equal(a, one)


@pytest.mark.parametrize("model,bs", [("resnet50_v1", 3), ("inception_v3", 2)])
def test_window_conv_matches_im2col_gather(monkeypatch, model, bs, oracle_mod):
    """kWindow on every eligible conv (stride-1 R x S convs as shifted-window
    MMAs over halo boxes, 16 x 8 pixel-block tiles) against the im2col gather
    on all of them: the same products summed in a different K order (channel
    block outer, tap inner); over ~50 layers of bf16 storage the logits move
    by ~2e-3 relative, and both stay inside the oracle bound."""
    imgs = generate_images(model, 5, bs)
    monkeypatch.setenv("DS_CONV_WINDOW", "1")
    with GpuBackend(model, Config(abs_max_bs=4, max_mtl=1)) as be:
        win = be.forward(imgs)
    monkeypatch.setenv("DS_CONV_WINDOW", "0")
    with GpuBackend(model, Config(abs_max_bs=4, max_mtl=1)) as be:
        gather = be.forward(imgs)
    assert np.isfinite(win).all()
    assert row_rel_err(win, gather).max() <= REL_TOL
    ref = oracle_mod.forward(model, imgs, bf16_storage=True)
    assert row_rel_err(win, ref).max() <= REL_TOL
    assert row_rel_err(gather, ref).max() <= REL_TOL


def test_softmax_probs():
    imgs = generate_images("synthetic_cnn", 0, 5)
    with GpuBackend("synthetic_cnn", Config(abs_max_bs=8, max_mtl=1)) as be:
        logits, probs = be.forward(imgs, probs=True)
    ref = np.exp(logits - logits.max(1, keepdims=True))
    ref /= ref.sum(1, keepdims=True)
    np.testing.assert_allclose(probs, ref, rtol=1e-5, atol=1e-7)


@pytest.mark.parametrize("model,bs", [("mobilenet_v1", 5), ("resnet50_v1", 3), ("inception_v3", 2)])
def test_pair_mma_matches_single_cta(monkeypatch, model, bs):
    """1x1 convs on CTA pairs (kPairTmaA: one M = 256 cta_group::2 MMA per K
    step, each CTA holding its 128 A rows and half of the B block; two
    epilogue teams per tile when the gather warps idle) against single-CTA
    M = 128 MMAs: the same products summed in the same K order, so
    bit-identical logits."""
    imgs = generate_images(model, 17, bs)
    monkeypatch.setenv("DS_CONV_PAIR", "1")
    with GpuBackend(model, Config(abs_max_bs=8, max_mtl=1)) as be:
        pair = be.forward(imgs)
    monkeypatch.setenv("DS_CONV_PAIR", "0")
    monkeypatch.setenv("DS_CONV_TPA", "0")
    with GpuBackend(model, Config(abs_max_bs=8, max_mtl=1)) as be:
        single = be.forward(imgs)
    assert np.isfinite(pair).all()
    assert np.array_equal(pair, single)


def test_narrow_window_convs_match_gather(monkeypatch):
    """Inception's 16/32-channel stride-1 3x3 convs as kS2D window MMAs (one
    32 B-swizzled halo box per 16-channel block, padding as negative box
    coordinates) against the im2col gather: the same K order (tap, channel),
    so bit-identical logits."""
    imgs = generate_images("inception_v3", 31, 2)
    monkeypatch.setenv("DS_CONV_NARROW", "1")
    with GpuBackend("inception_v3", Config(abs_max_bs=4, max_mtl=1)) as be:
        win = be.forward(imgs)
    monkeypatch.setenv("DS_CONV_NARROW", "0")
    with GpuBackend("inception_v3", Config(abs_max_bs=4, max_mtl=1)) as be:
        gather = be.forward(imgs)
    assert np.array_equal(win, gather)


def test_residual_tma_staging_matches_register_loads(monkeypatch):
    """ResNet residual 1x1s with each 32-column residual slice TMA-loaded into
    the epilogue's staging buffer (one slice ahead) against per-lane global
    loads: the same bf16 residual added to the same fp32 sum, so
    bit-identical logits."""
    imgs = generate_images("resnet50_v1", 41, 3)
    monkeypatch.setenv("DS_RES_TMA", "1")
    with GpuBackend("resnet50_v1", Config(abs_max_bs=4, max_mtl=1)) as be:
        staged = be.forward(imgs)
    monkeypatch.setenv("DS_RES_TMA", "0")
    with GpuBackend("resnet50_v1", Config(abs_max_bs=4, max_mtl=1)) as be:
        loads = be.forward(imgs)
    assert np.array_equal(staged, loads)


@pytest.mark.parametrize("model,bs", [("resnet50_v1", 3), ("inception_v3", 2)])
def test_tma_im2col_matches_gather(monkeypatch, model, bs):
    """Convs with C % 64 == 0 whose A blocks are TMA im2col loads (the tensor
    map walks 128 output pixels' windows for one tap and 64 channels, padding
    and stride in the map) against the cp.async gather: the same K order, so
    bit-identical logits."""
    imgs = generate_images(model, 43, bs)
    monkeypatch.setenv("DS_CONV_IM2COL", "1")
    with GpuBackend(model, Config(abs_max_bs=4, max_mtl=1)) as be:
        tma = be.forward(imgs)
    monkeypatch.setenv("DS_CONV_IM2COL", "0")
    with GpuBackend(model, Config(abs_max_bs=4, max_mtl=1)) as be:
        gather = be.forward(imgs)
    assert np.isfinite(tma).all()
    assert np.array_equal(tma, gather)


@pytest.mark.parametrize("model,bs", [("resnet50_v1", 3), ("inception_v3", 2), ("inception_v3", 37)])
def test_tma_pools_match_register_pools(monkeypatch, model, bs):
    """3x3 max / average pools over TMA halo boxes (pool_tma.cu: ragged last
    tiles, channel blocks of 32/64, concat-slice outputs) against the
    register-blocked pool kernel: the same taps in the same order, so
    bit-identical logits."""
    imgs = generate_images(model, 47, bs)
    monkeypatch.setenv("DS_POOL_SWAP", "0")  # (the register pools have no post-bias epilogue)
    monkeypatch.setenv("DS_POOL_TMA", "1")
    with GpuBackend(model, Config(abs_max_bs=max(8, bs), max_mtl=1)) as be:
        tma = be.forward(imgs)
    monkeypatch.setenv("DS_POOL_TMA", "0")
    with GpuBackend(model, Config(abs_max_bs=max(8, bs), max_mtl=1)) as be:
        regs = be.forward(imgs)
    assert np.isfinite(tma).all()
    assert np.array_equal(tma, regs)


@pytest.mark.parametrize("model,bs", [("inception_v3", 3), ("resnet50_v1", 5)])
def test_fused_sibling_1x1_matches_separate_launches(monkeypatch, model, bs):
    """Sibling 1x1 convs fused into one launch (model.hpp fuse_sibling_1x1:
    Inception's branch heads, ResNet's first conv + projection shortcut;
    concatenated weights, per-segment output maps and ReLU) against the
    separate launches: the same products in the same K order, so
    bit-identical logits, and fewer kernels per forward."""
    imgs = generate_images(model, 53, bs)
    monkeypatch.setenv("DS_FUSE_1X1", "1")
    with GpuBackend(model, Config(abs_max_bs=8, max_mtl=1)) as be:
        fused = be.forward(imgs)
        k_fused = be.stats()["kernels_per_forward"]
    monkeypatch.setenv("DS_FUSE_1X1", "0")
    with GpuBackend(model, Config(abs_max_bs=8, max_mtl=1)) as be:
        separate = be.forward(imgs)
        k_sep = be.stats()["kernels_per_forward"]
    assert np.isfinite(fused).all()
    assert np.array_equal(fused, separate)
    assert k_fused < k_sep


def test_avgpool_1x1_swap_within_oracle_bound(monkeypatch, oracle_mod):
    """Inception's avgpool3x3 -> 1x1 branches computed as a bias-free 1x1 (fused
    with its siblings) followed by a pool over its 32-192 channels that adds
    the bias and applies the ReLU (model.hpp swap_avgpool_1x1; linear, so equal
    up to where the bf16 rounding happens): both orders stay within the oracle
    bound and close to each other, with fewer pooled channels."""
    imgs = generate_images("inception_v3", 61, 4)
    monkeypatch.setenv("DS_POOL_SWAP", "1")
    with GpuBackend("inception_v3", Config(abs_max_bs=8, max_mtl=1)) as be:
        swapped = be.forward(imgs)
    monkeypatch.setenv("DS_POOL_SWAP", "0")
    with GpuBackend("inception_v3", Config(abs_max_bs=8, max_mtl=1)) as be:
        plain = be.forward(imgs)
    ref = oracle_mod.forward("inception_v3", imgs, bf16_storage=True)
    mean = np.load(__import__("os").path.join(__import__("os").path.dirname(__file__), "golden",
                                              "top1_inception_v3.npz"))["mean_32"]
    dep = np.abs(ref - mean).max(1)
    assert np.isfinite(swapped).all()
    assert (np.abs(swapped - ref).max(1) / dep).max() <= 4e-2
    assert (np.abs(plain - ref).max(1) / dep).max() <= 4e-2
    assert (np.abs(swapped - plain).max(1) / dep).max() <= 4e-2
