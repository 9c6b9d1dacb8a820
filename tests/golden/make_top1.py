"""Regenerates tests/golden/top1_<model>.npz: the FP32 CPU oracle's verdict on
TOP1_N synthetic images per model (image indices 0..TOP1_N-1, seed 42), for
the 4,096-image top-1 statistic of SURVEY §8(d) / north_star (the GPU test
tests/test_forward_parity_gpu.py::test_top1_4096 compares the device's
argmax with these). Run in the build container (oracle is CPU-only; ~15 min
on 8 cores): python tests/golden/make_top1.py [model ...]

Per image and oracle mode (32 = pure fp32 activations, 16 = bf16 activation
storage): top-1 class, runner-up class, top-2 margin; plus the fp32 logits'
mean over the set and each image's input-dependent range
dep_i = max_j |ref_ij - mean_j| (the error normaliser).
"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402

TOP1_N = 4096
MODELS = ("synthetic_cnn", "mobilenet_v1", "resnet50_v1", "inception_v3")


def verdict(logits):
    order = np.argsort(logits, axis=1)
    top1, top2 = order[:, -1], order[:, -2]
    rows = np.arange(len(logits))
    return top1.astype(np.int16), top2.astype(np.int16), \
        (logits[rows, top1] - logits[rows, top2]).astype(np.float32)


def make(model, n=TOP1_N, chunk=256):
    t = time.time()
    l32, l16 = [], []
    for i in range(0, n, chunk):
        imgs = oracle.images(model, i, min(chunk, n - i))
        l32.append(oracle.forward(model, imgs, bf16_storage=False))
        l16.append(oracle.forward(model, imgs, bf16_storage=True))
    l32, l16 = np.concatenate(l32), np.concatenate(l16)
    mean = l32.mean(0)
    dep = np.abs(l32 - mean).max(1).astype(np.float32)
    t32, r32, m32 = verdict(l32)
    t16, r16, m16 = verdict(l16)
    out = os.path.join(HERE, f"top1_{model}.npz")
    np.savez_compressed(out, first=0, n=n, top1_32=t32, top2_32=r32, margin_32=m32,
                        top1_16=t16, top2_16=r16, margin_16=m16, mean_32=mean.astype(np.float32),
                        dep_32=dep, head_k=oracle.model_info(model).get("head_k", -1))
    print(f"{model}: {n} images in {time.time() - t:.0f}s, distinct top-1 {len(set(t32))}, "
          f"fp32/bf16 top-1 agreement {np.mean(t32 == t16):.4f}, median margin {np.median(m32):.3f}, "
          f"median dep {np.median(dep):.3f} -> {out}")


if __name__ == "__main__":
    for m in (sys.argv[1:] or MODELS):
        make(m)
