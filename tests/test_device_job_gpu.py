"""The B200 backend behind the GpuSim seam, and the control plane on it.

1. Seam contract (reference test_perf_model.cpp:149-207 restated for the
   device): clock += latency per batch, += latency/mtl per MT request,
   += delay per instance change; reference error messages.
2. Bit-exact replay (north_star): a DNNScaler job runs on the device and
   records its latency tape; the same tape replayed through (a) the
   product's ReplaySeam and (b) the UNMODIFIED reference control plane
   (oracle/_ref: reference profiler.cpp/scaler.cpp/harness.cpp/
   matrix_completion.cpp over the tape seam) must reproduce the Profiler
   decision and every period's knob, p95, mean, throughput and verdict to
   the bit.
"""
import json
import math
import os

import numpy as np
import pytest

import ref as refo
from paper_2308_13803_b200 import Config, GpuBackend
from paper_2308_13803_b200 import control as C

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DONORS = os.path.join(ROOT, "paper_2308_13803_b200", "data", "p40_donors.json")


def test_seam_clock_and_errors():
    with GpuBackend("synthetic_cnn", Config(abs_max_bs=8, max_mtl=3)) as be:
        assert be.mtl() == 1 and be.clock_ms() == 0.0
        lat = be.run_batch(4)
        assert lat > 0 and be.clock_ms() == lat
        c0 = be.clock_ms()
        d = be.apply_instance_change(1)
        assert be.mtl() == 2 and be.clock_ms() == c0 + d
        c1 = be.clock_ms()
        m = be.run_mt_request()
        assert be.clock_ms() == c1 + m / 2.0
        with pytest.raises(ValueError, match="invalid batch size"):
            be.run_batch(9)
        with pytest.raises(ValueError, match="invalid batch size"):
            be.run_batch(0)
        with pytest.raises(ValueError, match="instance changes are single steps"):
            be.apply_instance_change(2)
        with pytest.raises(ValueError, match="instance limit exceeded"):
            be.set_mtl(4)
        with pytest.raises(ValueError, match="cannot terminate last instance"):
            be.set_mtl(0)
        be.set_mtl(1)
        with pytest.raises(ValueError, match="cannot terminate last instance"):
            be.apply_instance_change(-1)
        assert be.apply_instance_change(0) == 0.0
    with pytest.raises(ValueError, match="invalid device limits"):
        GpuBackend("synthetic_cnn", Config(abs_max_bs=0, max_mtl=1))


def test_windows_equal_single_calls_semantics():
    with GpuBackend("mobilenet_v1", Config(abs_max_bs=16, max_mtl=4)) as be:
        lat = be.run_batches(16, 20)
        assert lat.shape == (20,) and (lat > 0).all()
        clock = be.clock_ms()
        assert math.isclose(clock, float(np.sum(lat)), rel_tol=0, abs_tol=1e-9)
        be.set_mtl(4)
        c0 = be.clock_ms()
        mt = be.run_mt_requests(40)
        assert abs(be.clock_ms() - (c0 + float(np.sum(mt / 4.0)))) < 1e-9
        # co-located requests each take longer than alone, but 4 in flight
        # serve faster than one at a time
        be.set_mtl(1)
        solo = np.median(be.run_mt_requests(20))
        assert np.median(mt) > 0 and np.median(mt) / 4 < solo * 1.01


def test_host_io_mode_counts_copies():
    with GpuBackend("synthetic_cnn", Config(abs_max_bs=8, max_mtl=2)) as be:
        be.set_host_io(True)
        be.run_batches(8, 5)
        s = be.stats()
        img = 32 * 32 * 3
        assert s["h2d_bytes"] >= 5 * 8 * img and s["d2h_bytes"] >= 5 * 8 * 10 * 4
        be.set_host_io(False)


def _device_catalog(be, model, m, n):
    be.run_batches(1, 5)
    l1 = float(np.median(be.run_batches(1, 20)))
    lm = float(np.median(be.run_batches(m, 10)))
    lm = min(max(lm, l1 * 1.001), m * l1 * 0.999)
    be.set_mtl(n)
    mt = be.run_mt_requests(10 * n)
    be.set_mtl(1)
    t1 = 1000.0 / l1
    tmt = max(mt.size * 1000.0 / (mt.sum() / n), t1 * 1.0001)
    row = C.DnnProfile(model, [(1, t1), (m, m * 1000.0 / lm)], [(1, t1), (n, tmt)])
    return l1, [row] + C.load_catalog(DONORS)


@pytest.mark.parametrize("model,m,n,max_bs,max_mtl,c,steps,controller", [
    ("synthetic_cnn", 32, 4, 32, 4, 4.15, [], "dnnscaler"),
    ("mobilenet_v1", 32, 8, 128, 10, 13.44, [], "dnnscaler"),
    ("mobilenet_v1", 32, 8, 128, 10, 13.44, [(0.4, 0.5)], "dnnscaler"),  # SLO step-down
    # the Clipper baseline (clipper.cpp:17-35, AIMD on the
    # batch size) driving the same B200 backend, replayed through the reference
    ("mobilenet_v1", 32, 8, 128, 10, 13.44, [], "clipper"),
])
def test_device_job_replays_bit_exact(model, m, n, max_bs, max_mtl, c, steps, controller,
                                      tmp_path):
    with GpuBackend(model, Config(max_bs, max_mtl)) as be:
        l1, catalog = _device_catalog(be, model, m, n)
        slo = c * l1
        sc = C.Scenario(controller=controller, m=m, n=n, abs_max_bs=max_bs, max_mtl=max_mtl,
                        window=100)
        sched = [(t, slo * f) for t, f in steps]
        job = C.JobSpec(7, model, slo, 0.8, slo_schedule=sched)
        dev = C.run_job(sc, job, catalog, "device", backend=be)
    assert dev.error == "", dev.error
    assert dev.records.shape[0] >= 3 and dev.tape.size > 0
    # measured board power: NVML energy per period
    assert dev.summary["power_measured"] == 1
    assert dev.energy_tape.size == 3 * (dev.records.shape[0] + 2)
    assert np.all((dev.records[:, 7] > 50) & (dev.records[:, 7] < 2000)), dev.records[:, 7]
    assert 50 < dev.summary["avg_power_w"] < 2000 and dev.summary["power_efficiency"] > 0
    # (a) product replay of its own device tape (latencies + energy readings)
    ours = C.run_job(sc, job, catalog, "replay", tape=dev.tape, energy_tape=dev.energy_tape)
    assert np.array_equal(ours.records.view(np.uint64), dev.records.view(np.uint64))
    assert ours.report == dev.report
    assert ours.summary == dev.summary
    # (b) the reference control plane on the same tape
    if not refo.available():
        pytest.skip("oracle/_ref not built")
    doc = sc.to_json([job], "catalog.json")
    spath = refo.write_scenario(doc, [p.to_json() for p in catalog], str(tmp_path))
    theirs = refo.run_job(spath, 0, "replay", tape=dev.tape)
    assert theirs["consumed"] == dev.tape.size
    # every column but power_w (the reference prices power with its P40
    # PowerModel; the device run measured it)
    cols = [c for c in range(dev.records.shape[1]) if c != 7]
    assert np.array_equal(theirs["records"][:, cols].view(np.uint64),
                          dev.records[:, cols].view(np.uint64))
    for k in ("approach_kind", "ti_batching", "ti_mt", "profiling_cost_ms", "knob_changes",
              "settle_period", "periods", "steady_throughput", "p95_overall_ms", "slo_compliance",
              "total_items"):
        assert float(dev.summary[k]) == theirs["summary"][k], k
    assert dev.summary["steady_knob"] == (int(theirs["summary"]["steady_kind"]),
                                          int(theirs["summary"]["steady_value"]))
    if controller != "dnnscaler":
        return  # (no Profiler probe in Clipper's tape)
    # and the reference's profile() on the probe prefix of the tape
    rep, appr = refo.profile_tape(dev.tape, m, n, 10, max_bs, max_mtl)
    for k, v in rep.items():
        assert float(dev.report[k]) == v, k
    assert appr == dev.summary["approach_kind"]


def test_model_power_mode_replays_fully(monkeypatch, tmp_path):
    """DS_MODEL_POWER=1 keeps the reference PowerModel on the device seam: the
    whole record (power column included) then replays bit-exactly through the
    reference."""
    monkeypatch.setenv("DS_MODEL_POWER", "1")
    model, m, n = "mobilenet_v1", 32, 8
    with GpuBackend(model, Config(128, 10)) as be:
        l1, catalog = _device_catalog(be, model, m, n)
        sc = C.Scenario(m=m, n=n, abs_max_bs=128, max_mtl=10, window=100)
        job = C.JobSpec(8, model, 13.44 * l1, 0.5)
        dev = C.run_job(sc, job, catalog, "device", backend=be)
    assert dev.summary["power_measured"] == 0 and dev.energy_tape.size == 0
    if not refo.available():
        pytest.skip("oracle/_ref not built")
    doc = sc.to_json([job], "catalog.json")
    spath = refo.write_scenario(doc, [p.to_json() for p in catalog], str(tmp_path))
    theirs = refo.run_job(spath, 0, "replay", tape=dev.tape)
    assert np.array_equal(theirs["records"].view(np.uint64), dev.records.view(np.uint64))
    assert float(dev.summary["avg_power_w"]) == theirs["summary"]["avg_power_w"]


def test_combination_sweep_on_device():
    """the B x MT combination on the device (several
    full-size instances, each serving batches concurrently), reported per
    cell like the reference's combination_sweep (harness.cpp:356-386): mean,
    nearest-rank p95, throughput = bs * mtl * 1000 / mean."""
    with GpuBackend("mobilenet_v1", Config(abs_max_bs=32, max_mtl=3)) as be:
        c0 = be.clock_ms()
        lat = be.run_combo_requests(8, 2, 6)
        assert lat.shape == (6,) and (lat > 0).all()
        assert be.clock_ms() == pytest.approx(c0 + lat.sum() / 2, rel=1e-12)
        with pytest.raises(ValueError, match="invalid instance count"):
            be.run_combo_requests(8, 4, 1)
        with pytest.raises(ValueError, match="invalid batch size"):
            be.run_combo_requests(33, 1, 1)
        cells = be.combination_sweep([8, 32], [1, 2], samples_per_cell=20)
        # the batching path is unaffected afterwards
        assert be.run_batch(32) > 0
    assert [(c["bs"], c["mtl"]) for c in cells] == [(8, 1), (8, 2), (32, 1), (32, 2)]
    for c in cells:
        assert c["p95_ms"] >= c["mean_ms"] * 0.5 and c["throughput"] > 0
        assert c["throughput"] == pytest.approx(c["bs"] * c["mtl"] * 1000.0 / c["mean_ms"])
        assert c["measured_throughput"] > 0
    by = {(c["bs"], c["mtl"]): c for c in cells}
    # two concurrent instances deliver more than one (or at worst about the same)
    assert by[(8, 2)]["measured_throughput"] > 0.8 * by[(8, 1)]["measured_throughput"]


@pytest.mark.parametrize("model,bs", [("mobilenet_v1", 64), ("resnet50_v1", 32)])
def test_live_kernel_spans(model, bs):
    """Live per-kernel timing inside the real graph launches (ds_kernel_spans):
    every kernel of the forward has a positive in-situ span, and the spans of
    one forward add up to the forward's device time (back-to-back batches)."""
    with GpuBackend(model, Config(abs_max_bs=bs, max_mtl=1)) as be:
        be.run_batches(bs, 5)
        be.timer_start()
        be.reset_kernel_spans(0)
        be.run_batches(bs, 40)
        ms = be.timer_stop()
        spans, n = be.kernel_spans(0)
    assert n == 40 + 1  # (the run keeps kDepth requests in flight: one more forward ran)
    assert np.all(spans > 0), spans
    per_fwd = ms / n
    print(f"{model} bs {bs}: sum of spans {spans.sum():.4f} ms vs timer {per_fwd:.4f} ms per forward")
    assert 0.7 * per_fwd < spans.sum() < 1.1 * per_fwd
