"""R forwards of one model at batch bs inside an NVTX range "timed" (for ncu
launch lists: ncu --nvtx --nvtx-include "timed/" ... python tools/fwd_loop.py
model bs R). Prints the per-kernel algorithmic costs of one forward (launch
order) as JSON on stdout so launch lists can be joined to layers."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2308_13803_b200 import Config, GpuBackend, _lib  # noqa: E402
from paper_2308_13803_b200.backend import kernel_costs  # noqa: E402

model, bs, reps = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 3
with GpuBackend(model, Config(abs_max_bs=bs, max_mtl=1)) as be:
    be.run_batches(bs, 3)
    L = _lib.load()
    L.ds_nvtx_push(b"timed")
    be.run_batches(bs, reps)
    L.ds_nvtx_pop()
    print(json.dumps({"model": model, "bs": bs, "reps": reps,
                      "kernels_per_forward": be.stats()["kernels_per_forward"],
                      "costs": kernel_costs(model)}))
