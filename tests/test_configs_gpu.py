"""BASELINE.json configs 3 and 4 as device tests.

Config 3: ResNet-50 v1, batching sweep 1..256 under the p95 SLO, plus the
DNNScaler job with abs_max_bs = 256 (its Profiler decision recorded).
Config 4: Inception-v3, multi-tenancy sweep 1..16 co-located instances
(forced MT, static controller), plus a DNNScaler job with max_mtl = 16.
Every job's tape replays bit-exactly through the reference control plane.
"""
import os

import numpy as np
import pytest

import ref as refo
from paper_2308_13803_b200 import Config, GpuBackend
from paper_2308_13803_b200 import control as C

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DONORS = os.path.join(ROOT, "paper_2308_13803_b200", "data", "p40_donors.json")


def _row(be, model, m=32, n=8):
    be.run_batches(1, 5)
    l1 = float(np.median(be.run_batches(1, 20)))
    lm = float(np.median(be.run_batches(m, 10)))
    lm = min(max(lm, l1 * 1.001), m * l1 * 0.999)
    be.set_mtl(n)
    mt = be.run_mt_requests(8 * n)
    be.set_mtl(1)
    t1 = 1000.0 / l1
    tmt = max(mt.size * 1000.0 / (mt.sum() / n), t1 * 1.0001)
    return l1, [C.DnnProfile(model, [(1, t1), (m, m * 1000.0 / lm)], [(1, t1), (n, tmt)])] + \
        C.load_catalog(DONORS)


def _replay_matches_reference(sc, job, catalog, dev, tmp_path):
    ours = C.run_job(sc, job, catalog, "replay", tape=dev.tape, energy_tape=dev.energy_tape)
    assert np.array_equal(ours.records.view(np.uint64), dev.records.view(np.uint64))
    if not refo.available():
        return
    doc = sc.to_json([job], "catalog.json")
    spath = refo.write_scenario(doc, [p.to_json() for p in catalog], str(tmp_path))
    theirs = refo.run_job(spath, 0, "replay", tape=dev.tape)
    cols = [c for c in range(dev.records.shape[1]) if c != 7]  # power_w: measured vs PowerModel
    assert np.array_equal(theirs["records"][:, cols].view(np.uint64),
                          dev.records[:, cols].view(np.uint64))
    assert theirs["consumed"] == dev.tape.size


def test_config3_resnet50_batching_sweep_and_dnnscaler(tmp_path):
    with GpuBackend("resnet50_v1", Config(256, 10)) as be:
        lat = {}
        for bs in (1, 2, 4, 8, 16, 32, 64, 128, 256):
            be.run_batches(bs, 3)
            lat[bs] = float(np.median(be.run_batches(bs, 10)))
        tput = {bs: bs * 1000.0 / v for bs, v in lat.items()}
        print({bs: (round(lat[bs], 3), round(tput[bs])) for bs in lat})
        # latency grows with the batch (bs 1-4 sit on the fixed per-forward cost,
        # so neighbours there may tie to the microsecond)
        assert all(lat[b2] >= 0.98 * lat[b1] for b1, b2 in zip(list(lat)[:-1], list(lat)[1:]))
        assert lat[256] > 2 * lat[16]
        assert lat[128] > 2 * lat[1]
        assert tput[256] > 8 * tput[1]  # batching pays on B200
        l1, catalog = _row(be, "resnet50_v1")
        slo = 4.66 * l1
        # brute-force best static batch under the SLO (reference acceptance
        # best_batch: largest bs whose latency <= SLO)
        best = max([bs for bs in lat if lat[bs] <= slo], default=1)
        sc = C.Scenario(abs_max_bs=256, max_mtl=10)
        job = C.JobSpec(10, "resnet50_v1", slo, 1.5)
        dev = C.run_job(sc, job, catalog, "device", backend=be)
    assert dev.error == ""
    kind, value = dev.summary["steady_knob"]
    print("profiler ti_b %.1f ti_mt %.1f -> %s %d (static best %d)" % (
        dev.summary["ti_batching"], dev.summary["ti_mt"], "MT" if kind else "B", value, best))
    # the Scaler settles on batching within the SLO band near the brute-force
    # best static batch (its pseudo-binary search stops inside the alpha band,
    # reference scaler.cpp:28-63, so it may sit below the best)
    assert kind == C.BATCHING
    assert 0.5 * best <= value <= 256
    _replay_matches_reference(sc, job, catalog, dev, tmp_path)


def test_config4_inception_mt_sweep_and_dnnscaler(tmp_path):
    with GpuBackend("inception_v3", Config(128, 16)) as be:
        res = {}
        for k in (1, 2, 4, 8, 12, 16):
            be.set_mtl(k)
            be.run_mt_requests(4 * k)
            lat = be.run_mt_requests(16 * k)
            res[k] = (float(np.percentile(lat, 95)), k * 1000.0 / float(np.mean(lat)))
        be.set_mtl(1)
        print({k: (round(p, 3), round(t)) for k, (p, t) in res.items()})
        assert res[8][1] > 2.0 * res[1][1]  # co-location raises throughput at bs=1
        assert be.stats()["instances_created"] == 16
        l1, catalog = _row(be, "inception_v3")
        # forced MT: static knob at 12 co-located instances
        sc = C.Scenario(controller="static", static_knob=(C.MULTI_TENANCY, 12), abs_max_bs=128,
                        max_mtl=16)
        job = C.JobSpec(16, "inception_v3", 22.54 * l1, 0.4)
        dev = C.run_job(sc, job, catalog, "device", backend=be)
        assert dev.error == "" and dev.summary["steady_knob"] == (C.MULTI_TENANCY, 12)
        _replay_matches_reference(sc, job, catalog, dev, tmp_path / "static")
        # DNNScaler with max_mtl = 16 (a fresh reference GpuSim starts at one
        # instance; the shared backend is brought back there first)
        be.set_mtl(1)
        sc2 = C.Scenario(abs_max_bs=128, max_mtl=16, n=8)
        job2 = C.JobSpec(17, "inception_v3", 22.54 * l1, 1.0)
        dev2 = C.run_job(sc2, job2, catalog, "device", backend=be)
    assert dev2.error == ""
    os.makedirs(tmp_path / "dnn", exist_ok=True)
    _replay_matches_reference(sc2, job2, catalog, dev2, tmp_path / "dnn")
