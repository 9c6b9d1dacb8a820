"""Drop-in proof: the reference's own scenario loader, harness, Profiler,
Scaler and report writers — compiled unmodified against the B200 GpuSim
header (include/dnnscaler_b200/drop_in) into oracle/_ref/ref_on_b200 —
serve a MobileNet-v1 job on the B200 backend.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from paper_2308_13803_b200 import Config, GpuBackend

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "ref_on_b200")
DONORS = os.path.join(ROOT, "paper_2308_13803_b200", "data", "p40_donors.json")


@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/ref_on_b200 not built")
def test_reference_harness_serves_on_b200(tmp_path):
    with GpuBackend("mobilenet_v1", Config(128, 10)) as be:
        be.run_batches(1, 5)
        l1 = float(np.median(be.run_batches(1, 20)))
        l32 = float(np.median(be.run_batches(32, 10)))
    t1 = 1000.0 / l1
    row = {"id": "mobilenet_v1", "params_millions": 4.23, "mflops": 1137.5,
           "batching_points": [[1, t1], [32, 32000.0 / min(max(l32, l1 * 1.001), 32 * l1 * 0.999)]],
           "mt_points": [[1, t1], [8, 4 * t1]]}
    with open(DONORS) as f:
        catalog = [row] + json.load(f)
    (tmp_path / "catalog.json").write_text(json.dumps(catalog))
    scen = {"catalog_path": "catalog.json", "controller": "dnnscaler", "seed": 42,
            "jobs": [{"job_id": 1, "dnn_id": "mobilenet_v1", "slo_ms": 13.44 * l1,
                      "duration_s": 1.0}]}
    (tmp_path / "scenario.json").write_text(json.dumps(scen))
    env = dict(os.environ, DNNSCALER_B200_MODEL="mobilenet_v1")
    out = subprocess.run([BIN, str(tmp_path / "scenario.json"), str(tmp_path / "metrics.csv")],
                         capture_output=True, text=True, env=env, timeout=300)
    assert out.returncode == 0, out.stderr
    summary = json.loads(out.stdout)
    job = summary["jobs"][0] if "jobs" in summary else summary[0]
    assert "error" not in job, job
    assert job["profiled"] and job["periods"] >= 3
    assert job["slo_compliance"] > 0.9
    assert (tmp_path / "metrics.csv").read_text().count("\n") >= 3
