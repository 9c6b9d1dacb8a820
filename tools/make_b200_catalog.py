"""Measures the B200 catalog (paper_2308_13803_b200/data/b200_catalog.json) on
a B200: per architecture a batching sweep and a multi-tenancy sweep through
the device seam, written in the reference's catalog format (catalog.cpp:51-94)
— SURVEY §8(f) row 4. These rows are mt_init's matrix-completion donors
(derive_mt_rows, harness.cpp:315-327) and the L(BS=1) basis of config 5's
per-job SLOs.

    python tools/make_b200_catalog.py [out.json]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2308_13803_b200 import Config, GpuBackend  # noqa: E402
from paper_2308_13803_b200 import serving as S  # noqa: E402

BS = (1, 2, 4, 8, 16, 32, 64, 128, 256)
MT = (1, 2, 4, 6, 8, 10, 12, 16)


def main(out):
    rows = []
    for model in ("synthetic_cnn", "mobilenet_v1", "resnet50_v1", "inception_v3"):
        max_bs, max_mtl = S.MODEL_LIMITS[model]
        with GpuBackend(model, Config(max_bs, max_mtl)) as be:
            bsw = S.batch_sweep(be, [b for b in BS if b <= max_bs], calls=40)
            msw = S.mt_sweep(be, [k for k in MT if k <= max_mtl], calls_per_instance=25)
        row = S.catalog_row(model, bsw, msw)
        rows.append(row)
        print(model, "bs:", [(c["bs"], round(c["measured_throughput"])) for c in bsw])
        print(model, "mt:", [(c["mtl"], round(c["measured_throughput"])) for c in msw], flush=True)
    S.write_catalog(rows, out)
    print("->", out)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else S.B200_CATALOG)
