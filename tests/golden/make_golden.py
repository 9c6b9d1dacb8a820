"""Regenerates the committed fixtures under tests/golden/ (run in the build
container, where /root/reference exists; the GPU box only reads the output).

1. ref_data/: the reference's data fixtures (P40 calibration catalog and the
   scenarios), copied verbatim — data, not source: the paper's Table 4
   measurements as shipped in /root/reference/proj/data.
2. torch_xcheck_*.npz: the FP32 CPU oracle cross-checked against an
   independent torch.nn.functional implementation of the same network on a
   few images (see test_oracle.py). The reference has no forward pass, so
   this (not the reference) is what pins the logits oracle.
"""
import os
import shutil
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_DATA = "/root/reference/proj/data"


def copy_ref_data():
    out = os.path.join(HERE, "ref_data")
    os.makedirs(out, exist_ok=True)
    for name in sorted(os.listdir(REF_DATA)):
        if name.endswith(".json"):
            shutil.copyfile(os.path.join(REF_DATA, name), os.path.join(out, name))
            print("copied", name)


if __name__ == "__main__":
    copy_ref_data()
    if "--xcheck" in sys.argv:
        sys.path.insert(0, HERE)
        import torch_xcheck
        torch_xcheck.main()
