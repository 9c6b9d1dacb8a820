"""Host control plane (product C++ via the C ABI) against the reference.

1. Known-answer tests transcribed from the reference's own suites
   (test_domain.cpp, test_profiler.cpp, test_scaler.cpp, test_harness.cpp).
2. Whole-scenario parity: every job of the reference's 30-job scenario and
   the SLO-sensitivity scenarios, run by the product on the analytic seam
   and by the compiled, unmodified reference (oracle/_ref) — per-period
   records, summaries and profiler decisions must be bit-identical.
3. Tape replay: a tape recorded from the reference replays through the
   product's ReplaySeam to the same bits (the mechanism the GPU tests use
   for device tapes).
"""
import json
import os

import numpy as np
import pytest

import ref as refo
from paper_2308_13803_b200 import control as C

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "ref_data")
CATALOG = C.load_catalog(os.path.join(GOLDEN, "catalog.json"))
CATALOG_JSON = json.load(open(os.path.join(GOLDEN, "catalog.json")))


# ------------------------------------------------------------ known answers
def test_percentile_nearest_rank():  # test_domain.cpp:14-35
    assert C.percentile(np.arange(1, 101, dtype=float), 0.95) == 95.0
    assert C.percentile([7.0], 0.95) == 7.0
    assert C.percentile([5, 5, 5, 5], 0.95) == 5.0
    with pytest.raises(ValueError, match="no samples"):
        C.percentile([], 0.95)
    with pytest.raises(ValueError, match="quantile out of range"):
        C.percentile([1.0], 1.5)


def test_band_verdict_edges():  # test_scaler.cpp:13-20
    assert C.band_verdict(100.0, 419.0) == 0
    assert C.band_verdict(356.15, 419.0) == 1
    assert C.band_verdict(419.0, 419.0) == 1
    assert C.band_verdict(419.01, 419.0) == 2
    assert C.band_verdict(356.0, 419.0) == 0
    with pytest.raises(ValueError, match="invalid slo"):
        C.band_verdict(10.0, 0.0)


def _drive(alpha):  # test_scaler.cpp:32-42
    st = C.BatchScaler(128)
    visited = []
    for _ in range(64):
        p95 = 19.18 + 7.99 * st.s.current_bs
        if not st.step(p95, 419.0, alpha):
            break
        visited.append(st.s.current_bs)
    return visited


def test_batch_search_trajectories():  # test_scaler.cpp:54-69
    assert _drive(0.85) == [65, 33, 81, 57, 45]
    assert _drive(0.95) == [65, 33, 81, 57, 45, 87, 66, 55, 50]


def test_batch_step_restart_and_infeasible():  # test_scaler.cpp:83-105
    st = C.BatchScaler(128)
    st.s.min_bs, st.s.max_bs, st.s.current_bs = 33, 57, 33
    st.step(500.0, 419.0)
    assert (st.s.current_bs, st.s.min_bs, st.s.max_bs) == (17, 1, 33)
    st = C.BatchScaler(128)
    assert not st.step(500.0, 419.0) and st.s.infeasible == 1
    assert st.step(10.0, 838.0) and st.s.current_bs == 65 and st.s.infeasible == 0


def test_mt_step_damper():  # test_scaler.cpp:171-220
    st = C.MtScaler(3, 10)
    assert st.step(10.0, 100.0) == (1, False) and st.s.mtl == 4      # add
    assert st.step(120.0, 100.0) == (2, False) and st.s.mtl == 3     # remove, damper armed
    assert st.s.damped == 1
    assert st.step(10.0, 100.0) == (0, False) and st.s.mtl == 3      # held by damper
    assert st.step(90.0, 100.0) == (0, False) and st.s.damped == 0   # in band disarms
    st = C.MtScaler(1, 10)
    assert st.step(200.0, 100.0) == (0, True)


def test_profiler_gains_and_decisions():  # test_profiler.cpp:20-57
    def prof(b1, b32, m8):
        job = C.JobSpec(1, "x", 1e9, 20.0)
        cat = [C.DnnProfile("x", [(1, b1), (32, b32)], [(1, b1), (8, m8)], sigma=0.0)]
        r = C.run_job(C.Scenario(sigma=0.0), job, cat, "analytic")
        return r.report, r.summary
    rep, s = prof(118.66, 125.67, 237.28)
    assert abs(rep["tput_base"] - 118.66) < 1e-6 and abs(rep["tput_mt"] - 237.28) < 1e-6
    assert abs(rep["ti_mt"] - 99.96) < 0.01 and abs(rep["ti_batching"] - 5.91) < 0.01
    assert s["approach_kind"] == C.MULTI_TENANCY
    assert rep["items_served"] == 10.0 * (1 + 32) + 10.0 * 8
    assert rep["transition_ms"] == 7 * 500.0 + 7 * 100.0
    rep, s = prof(492.00, 7145.89, 2163.80)
    assert abs(rep["ti_batching"] - 1352.42) < 0.01 and s["approach_kind"] == C.BATCHING
    assert C.decide(100.0, 100.3, 10.0, 12.0) == C.BATCHING          # tie -> latency
    assert C.decide(100.0, 100.3, 12.0, 10.0) == C.MULTI_TENANCY
    assert C.decide(50.0, 50.0, 10.0, 10.0) == C.BATCHING
    with pytest.raises(ValueError, match="eps must be non-negative"):
        C.decide(1, 2, eps=-0.1)


def test_calibration_goldens():  # test_perf_model.cpp:14-59
    a, b = C.calibrate_batching([(1, 36.81), (32, 116.41)])
    assert abs(a - 19.175439) < 1e-4 and abs(b - 7.991093) < 1e-4
    assert abs((a + b) - 1000.0 / 36.81) < 1e-9 and abs((a + 32 * b) - 32000.0 / 116.41) < 1e-9
    l1, cap = C.calibrate_mt([(1, 118.66), (8, 237.28)])
    assert abs(l1 - 8.4274) < 1e-4 and abs(cap - 1.9996629) < 1e-6


def test_harness_inc_v1_settles_at_mtl8():  # test_harness.cpp:65-92
    job = C.JobSpec(1, "inc-v1-imagenet", 35.0, 60.0)
    r = C.run_job(C.Scenario(sigma=0.0), job, CATALOG, "analytic")
    assert r.summary["steady_knob"] == (C.MULTI_TENANCY, 8)
    assert abs(r.summary["steady_throughput"] - 237.28) < 1e-6
    assert r.error == ""


def test_harness_slo_step_down_trace():  # test_harness.cpp:167-187
    cat = [C.DnnProfile("flat", [(1, 100.0), (32, 110.0)], [(1, 100.0), (10, 1000.0)], sigma=0.0)]
    job = C.JobSpec(1, "flat", 12.0, 30.0, slo_schedule=[(10.0, 6.0)])
    r = C.run_job(C.Scenario(sigma=0.0), job, cat + CATALOG, "analytic")
    assert r.error == ""
    assert len(r.readaptations) == 1


def test_unknown_dnn_is_a_job_error():  # harness.cpp:341-351
    r = C.run_job(C.Scenario(), C.JobSpec(1, "nope", 10.0, 1.0), CATALOG, "analytic")
    assert r.error == "unknown dnn: nope" and r.summary["failed"] == 1


# ------------------------------------------------------------ whole scenarios vs _ref
def _scenario_from_json(doc):
    sc = C.Scenario(controller=doc.get("controller", "dnnscaler"), seed=doc.get("seed", 42),
                    alpha=doc.get("alpha", 0.85), m=doc.get("m", 32), n=doc.get("n", 8),
                    abs_max_bs=doc.get("abs_max_bs", 128), max_mtl=doc.get("max_mtl", 10),
                    window=doc.get("window", 100), sigma=doc.get("sigma", 0.05))
    jobs = [C.JobSpec(j["job_id"], j["dnn_id"], float(j["slo_ms"]), float(j["duration_s"]),
                      [tuple(s) for s in j.get("slo_schedule", [])]) for j in doc["jobs"]]
    return sc, jobs


def _compare(ours, theirs):
    assert ours.records.shape == theirs["records"].shape
    # bit-exact: every per-period field
    assert np.array_equal(ours.records.view(np.uint64), theirs["records"].view(np.uint64))
    s = ours.summary
    t = theirs["summary"]
    for k in ("approach_kind", "profiled", "ti_batching", "ti_mt", "profiling_cost_ms",
              "converged", "knob_changes", "settle_period", "periods", "duration_s",
              "total_items", "avg_throughput", "steady_throughput", "p95_overall_ms",
              "slo_compliance", "avg_power_w", "power_efficiency", "final_slo_ms"):
        assert float(s[k]) == t[k], k
    assert s["steady_knob"] == (int(t["steady_kind"]), int(t["steady_value"]))
    assert ours.readaptations == theirs["readaptations"]


SCENARIOS = ["scenario_30jobs.json", "sensitivity_bs_down.json", "sensitivity_bs_up.json",
             "sensitivity_mt_down.json", "sensitivity_mt_up.json"]


@pytest.mark.skipif(not refo.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", SCENARIOS)
@pytest.mark.parametrize("controller", ["dnnscaler", "clipper"])
def test_scenario_bit_exact_vs_reference(name, controller, tmp_path):
    doc = json.load(open(os.path.join(GOLDEN, name)))
    doc["controller"] = controller
    spath = refo.write_scenario(doc, CATALOG_JSON, str(tmp_path))
    sc, jobs = _scenario_from_json(doc)
    for i, job in enumerate(jobs):
        ours = C.run_job(sc, job, CATALOG, "analytic")
        theirs = refo.run_job(spath, i, "record")
        _compare(ours, theirs)
        assert np.array_equal(ours.tape, theirs["tape"])


@pytest.mark.skipif(not refo.available(), reason="oracle/_ref not built")
def test_static_knob_controller_vs_reference(tmp_path):
    doc = json.load(open(os.path.join(GOLDEN, "scenario_30jobs.json")))
    doc["jobs"] = doc["jobs"][:6]
    for kind, value in (("batching", 17), ("multi-tenancy", 5)):
        doc["controller"] = "static"
        doc["static_knob"] = {"kind": kind, "value": value}
        spath = refo.write_scenario(doc, CATALOG_JSON, str(tmp_path))
        sc, jobs = _scenario_from_json(doc)
        sc.static_knob = (0 if kind == "batching" else 1, value)
        for i, job in enumerate(jobs):
            _compare(C.run_job(sc, job, CATALOG, "analytic"), refo.run_job(spath, i, "stock"))


@pytest.mark.skipif(not refo.available(), reason="oracle/_ref not built")
def test_reference_tape_replays_through_product(tmp_path):
    doc = json.load(open(os.path.join(GOLDEN, "scenario_30jobs.json")))
    spath = refo.write_scenario(doc, CATALOG_JSON, str(tmp_path))
    sc, jobs = _scenario_from_json(doc)
    for i in (0, 2, 9, 17):  # MT and batching jobs
        theirs = refo.run_job(spath, i, "record")
        ours = C.run_job(sc, jobs[i], CATALOG, "replay", tape=theirs["tape"])
        _compare(ours, theirs)
        # and the reference replaying its own tape reproduces itself
        again = refo.run_job(spath, i, "replay", tape=theirs["tape"])
        assert np.array_equal(again["records"], theirs["records"])
        assert again["consumed"] == theirs["tape"].size


@pytest.mark.skipif(not refo.available(), reason="oracle/_ref not built")
def test_profile_on_tape_matches_reference():
    rng = np.random.default_rng(3)
    for m, n in ((32, 8), (16, 4)):
        tape = np.concatenate([rng.uniform(1, 2, 10), rng.uniform(5, 9, 10), rng.uniform(0.1, 0.2, n - 1),
                               rng.uniform(2, 4, 10 * n), rng.uniform(0.1, 0.2, n - 1)])
        ref_report, ref_appr = refo.profile_tape(tape, m, n, 10)
        cat = [C.DnnProfile("x", [(1, 100.0), (32, 110.0)], [(1, 100.0), (8, 150.0)])]
        # one DNNScaler job whose tape starts with exactly these probe values
        job = C.JobSpec(1, "x", 1e6, 0.5)
        sc = C.Scenario(m=m, n=n, window=1)
        full = np.concatenate([tape, np.full(100_000, 1.0)])
        ours = C.run_job(sc, job, cat, "replay", tape=full)
        for k, v in ref_report.items():
            assert float(ours.report[k]) == v, k


@pytest.mark.skipif(not refo.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", ["scenario_30jobs.json", "sensitivity_bs_down.json",
                                  "sensitivity_mt_up.json"])
@pytest.mark.parametrize("controller", ["dnnscaler", "clipper"])
def test_report_writers_byte_identical_to_reference(name, controller, tmp_path):
    """metrics.csv / summary.json from the product's writers (report.py) over
    the product's own job results equal, byte for byte, what the reference's
    renderers (report.cpp) write for the reference's run of the same scenario."""
    from paper_2308_13803_b200 import report as R
    doc = json.load(open(os.path.join(GOLDEN, name)))
    doc["controller"] = controller
    spath = refo.write_scenario(doc, CATALOG_JSON, str(tmp_path))
    sc, jobs, cat_path = R.load_scenario(spath)
    catalog = C.load_catalog(cat_path)
    results = [C.run_job(sc, j, catalog, "analytic") for j in jobs]
    ref_csv, ref_json = refo.render_scenario(spath)
    assert R.render_metrics_csv(results) == ref_csv
    assert R.render_summary_json(sc, jobs, results) == ref_json


def test_report_writer_formats():
    from paper_2308_13803_b200 import report as R
    cells = [{"bs": 4, "mtl": 2, "mean_ms": 1.25, "p95_ms": 1.5, "throughput": 6400.0}]
    assert R.render_sweep_csv(cells) == "bs,mtl,mean_ms,p95_ms,throughput\n4,2,1.250000,1.500000,6400.000000\n"


@pytest.mark.skipif(not refo.available(), reason="oracle/_ref not built")
def test_cli_run_and_compare_write_reference_reports(tmp_path):
    """The CLI (cli.py, the reference CLI's subcommands) on the analytic seam:
    run writes the reference's metrics.csv / summary.json bytes; compare writes
    both controllers' reports and the comparison table; a missing config is an
    error exit."""
    from paper_2308_13803_b200 import cli
    doc = json.load(open(os.path.join(GOLDEN, "scenario_30jobs.json")))
    doc["jobs"] = doc["jobs"][:5]
    spath = refo.write_scenario(doc, CATALOG_JSON, str(tmp_path))
    out = tmp_path / "out"
    assert cli.main(["run", "--config", spath, "--out", str(out)]) == 0
    ref_csv, ref_json = refo.render_scenario(spath)
    assert (out / "metrics.csv").read_text() == ref_csv
    assert (out / "summary.json").read_text() == ref_json
    assert cli.main(["compare", "--config", spath, "--out", str(out)]) == 0
    comp = (out / "comparison.csv").read_text().splitlines()
    assert comp[0].startswith("job_id,dnn_id,approach") and len(comp) == 6
    assert cli.main(["run", "--config", str(tmp_path / "missing.json"), "--out", str(out)]) != 0


@pytest.mark.skipif(not refo.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("dnn,m,n,seed,sigma", [(0, 32, 8, 42, None), (1, 16, 4, 7, 0.1),
                                                (2, 64, 10, 3, 0.0)])
def test_cli_profile_byte_identical_to_reference(dnn, m, n, seed, sigma, tmp_path, capsys):
    """`profile` (cli.py over ds_profile_dnn) prints the reference CLI's
    render_profile_json bytes for the same catalog, probe sizes, seed and
    sigma override on the analytic seam."""
    from paper_2308_13803_b200 import cli
    cat_path = tmp_path / "catalog.json"
    cat_path.write_text(json.dumps(CATALOG_JSON))
    dnn_id = CATALOG_JSON[dnn]["id"]
    argv = ["profile", "--catalog", str(cat_path), "--dnn", dnn_id, "--m", str(m), "--n", str(n),
            "--seed", str(seed)]
    if sigma is not None:
        argv += ["--sigma", str(sigma)]
    assert cli.main(argv) == 0
    out = capsys.readouterr().out
    ref = refo.render_profile(str(cat_path), dnn_id, m, n, 10, seed, -1.0 if sigma is None else sigma)
    assert out.endswith(ref) and ("approach: " + json.loads(ref)["approach"]) in out
    assert cli.main(["profile", "--catalog", str(cat_path), "--dnn", "no_such_net"]) != 0


@pytest.mark.skipif(not refo.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("dnn,seed,sigma", [(0, 42, None), (3, 7, 0.08), (5, 1, 0.0)])
def test_cli_sweep_byte_identical_to_reference(dnn, seed, sigma, tmp_path, capsys):
    """`sweep` on the analytic seam (ds_combination_sweep) writes the
    reference CLI's sweep.csv bytes: same grid, noise draws and percentiles."""
    from paper_2308_13803_b200 import cli
    cat_path = tmp_path / "catalog.json"
    cat_path.write_text(json.dumps(CATALOG_JSON))
    dnn_id = CATALOG_JSON[dnn]["id"]
    bs, mtl = [1, 4, 16, 64], [1, 2, 3, 8]
    argv = ["sweep", "--catalog", str(cat_path), "--dnn", dnn_id, "--bs", ",".join(map(str, bs)),
            "--mtl", ",".join(map(str, mtl)), "--out", str(tmp_path), "--samples", "50",
            "--seed", str(seed)]
    if sigma is not None:
        argv += ["--sigma", str(sigma)]
    assert cli.main(argv) == 0
    ref = refo.render_sweep(str(cat_path), dnn_id, bs, mtl, 50, seed, -1.0 if sigma is None else sigma)
    assert (tmp_path / "sweep.csv").read_text() == ref
    assert capsys.readouterr().out == ref
    assert cli.main(argv + ["--samples", "0"]) == 2  # std::invalid_argument -> exit 2, as the reference


@pytest.mark.skipif(not refo.available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("name", ["sensitivity_bs_up.json", "sensitivity_mt_down.json"])
def test_cli_sensitivity_writes_reference_reports(name, tmp_path, capsys):
    """`sensitivity` (the reference CLI's cmd_sensitivity): the reference's
    report bytes, one readaptation line per SLO step; a scenario without an
    slo_schedule is refused with the reference's exit code 2."""
    from paper_2308_13803_b200 import cli
    doc = json.load(open(os.path.join(GOLDEN, name)))
    spath = refo.write_scenario(doc, CATALOG_JSON, str(tmp_path))
    out = tmp_path / "out"
    assert cli.main(["sensitivity", "--config", spath, "--out", str(out)]) == 0
    ref_csv, ref_json = refo.render_scenario(spath)
    assert (out / "metrics.csv").read_text() == ref_csv
    assert (out / "summary.json").read_text() == ref_json
    steps = sum(len(j.get("slo_schedule", [])) for j in doc["jobs"])
    assert capsys.readouterr().out.count(": slo step at ") == steps
    plain = dict(doc, jobs=[{k: v for k, v in j.items() if k != "slo_schedule"} for j in doc["jobs"]])
    ppath = refo.write_scenario(plain, CATALOG_JSON, str(tmp_path / "plain"))
    assert cli.main(["sensitivity", "--config", ppath, "--out", str(out)]) == 2
