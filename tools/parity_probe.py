"""Device-vs-oracle logit statistics for one model (bring-up aid, GPU box).

    python tools/parity_probe.py <model> [n_images] [bs]

Prints, against both oracle modes (bf16 activation storage, pure fp32):
max|dev-ref| / max|ref|, the same normalised by the input-dependent part
max|ref - mean_ref| (mean over the image set), top-1 agreement, distinct
top-1 classes and the top-2 margin distribution.
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
import oracle  # noqa: E402  (checker)
from paper_2308_13803_b200 import Config, GpuBackend, generate_images, model_info  # noqa: E402

model = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
bs = int(sys.argv[3]) if len(sys.argv) > 3 else min(n, 128)
imgs = generate_images(model, 0, n)
with GpuBackend(model, Config(abs_max_bs=bs, max_mtl=1)) as be:
    dev = np.concatenate([be.forward(imgs[i:i + bs]) for i in range(0, n, bs)])
t = time.time()
r16 = oracle.forward(model, imgs, bf16_storage=True)
r32 = oracle.forward(model, imgs, bf16_storage=False)
print(f"{model}: head_k={model_info(model).head_k} oracle {time.time() - t:.1f}s")
for name, ref in (("bf16", r16), ("fp32", r32)):
    dep = np.abs(ref - ref.mean(0)).max(1)
    err = np.abs(dev - ref).max(1)
    s = np.sort(ref, 1)
    marg = s[:, -1] - s[:, -2]
    print(f"  vs {name}: err/max {np.max(err / np.abs(ref).max(1)):.3e} "
          f"err/dep {np.max(err / dep):.3e} top1 {np.mean(dev.argmax(1) == ref.argmax(1)):.4f} "
          f"distinct {len(set(ref.argmax(1)))}/{n} margin min/med {marg.min():.4f}/{np.median(marg):.4f} "
          f"max err {err.max():.4f} dep/max {dep.max() / np.abs(ref).max():.3f}")
