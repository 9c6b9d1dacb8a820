"""The CLI (paper_2308_13803_b200/cli.py) on the B200: a scenario served on
the device seam writes the reference-format reports, the profile and sweep
subcommands run on the device."""
import json
import os

import pytest

from paper_2308_13803_b200 import cli
from paper_2308_13803_b200 import serving as S

pytestmark = pytest.mark.gpu


def test_cli_run_on_device(tmp_path, capsys):
    doc = {"catalog_path": os.path.abspath(S.B200_CATALOG), "controller": "dnnscaler", "seed": 42,
           "alpha": 0.85, "m": 32, "n": 8, "abs_max_bs": 64, "max_mtl": 8, "window": 20, "sigma": 0.05,
           "jobs": [{"job_id": 1, "dnn_id": "synthetic_cnn", "slo_ms": 0.2, "duration_s": 0.05},
                    {"job_id": 2, "dnn_id": "mobilenet_v1", "slo_ms": 2.0, "duration_s": 0.2}]}
    spath = tmp_path / "scenario.json"
    spath.write_text(json.dumps(doc))
    out = tmp_path / "out"
    assert cli.main(["run", "--config", str(spath), "--out", str(out), "--seam", "device"]) == 0
    summary = json.loads((out / "summary.json").read_text())
    assert [j["job_id"] for j in summary["jobs"]] == [1, 2]
    assert all("error" not in j and j["total_items"] > 0 for j in summary["jobs"])
    rows = (out / "metrics.csv").read_text().splitlines()
    assert rows[0].startswith("time_s,job_id,knob_kind") and len(rows) > 2
    assert "synthetic_cnn" in capsys.readouterr().out


def test_cli_profile_and_sweep_on_device(tmp_path, capsys):
    assert cli.main(["profile", "--dnn", "synthetic_cnn", "--m", "16", "--n", "4", "--seam", "device"]) == 0
    out = capsys.readouterr().out
    assert "approach:" in out and '"tput_base"' in out
    assert cli.main(["sweep", "--dnn", "synthetic_cnn", "--bs", "1,8", "--mtl", "1,2", "--out",
                     str(tmp_path), "--samples", "10", "--seam", "device"]) == 0
    lines = (tmp_path / "sweep.csv").read_text().splitlines()
    assert lines[0] == "bs,mtl,mean_ms,p95_ms,throughput" and len(lines) == 5
