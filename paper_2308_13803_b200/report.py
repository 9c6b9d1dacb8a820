"""Scenario files in, reports out — the reference's byte-stable writers.

* ``load_scenario(path)``: a reference scenario JSON (scenario.cpp schema:
  catalog_path relative to the file, controller, seed, alpha, m, n,
  abs_max_bs, max_mtl, window, sigma, static_knob, jobs[] with optional
  slo_schedule) -> (Scenario, [JobSpec], catalog path).
* ``render_metrics_csv`` / ``render_summary_json`` / ``render_sweep_csv`` /
  ``render_comparison_csv`` / ``render_profile_json``: the same bytes as the
  reference renderers (report.cpp:60-190; nlohmann ordered_json dump(2), C
  "%.6f" fields) for the same job results — checked byte for byte against
  the compiled reference on its own scenarios (tests/test_control_plane.py).

The job results come from ``control.run_job`` on any seam (the B200 device,
the reference's analytic GPU, or a recorded tape).
"""
from __future__ import annotations

import json
import math
import os
from typing import List, Sequence, Tuple

from . import control as C

_KNOB = {0: "batching", 1: "multi-tenancy"}


def _fixed6(v: float) -> str:
    return "%.6f" % v


def load_scenario(path: str) -> Tuple[C.Scenario, List[C.JobSpec], str]:
    """Reference scenario JSON -> (Scenario, jobs, catalog path); the catalog
    path is resolved against the scenario file's directory, as the reference
    loader does."""
    doc = json.load(open(path))
    sc = C.Scenario(controller=doc.get("controller", "dnnscaler"), seed=int(doc.get("seed", 42)),
                    alpha=float(doc.get("alpha", 0.85)), m=int(doc.get("m", 32)), n=int(doc.get("n", 8)),
                    abs_max_bs=int(doc.get("abs_max_bs", 128)), max_mtl=int(doc.get("max_mtl", 10)),
                    window=int(doc.get("window", 100)), sigma=float(doc.get("sigma", 0.05)))
    if "static_knob" in doc:
        k = doc["static_knob"]
        sc.static_knob = (0 if k.get("kind", "batching") == "batching" else 1, int(k["value"]))
    jobs = [C.JobSpec(int(j["job_id"]), j["dnn_id"], float(j["slo_ms"]), float(j["duration_s"]),
                      [tuple(s) for s in j.get("slo_schedule", [])]) for j in doc["jobs"]]
    cat = doc.get("catalog_path", "")
    if cat and not os.path.isabs(cat):
        cat = os.path.join(os.path.dirname(os.path.abspath(path)), cat)
    return sc, jobs, cat


def render_metrics_csv(results: Sequence[C.JobResult]) -> str:
    """== render_metrics_csv (report.cpp:60-88): one row per control period."""
    out = ["time_s,job_id,knob_kind,knob_value,p95_ms,mean_ms,throughput,power_w,slo_ms,violated\n"]
    for r in results:
        for rec in r.records:
            out.append(",".join([_fixed6(rec[0]), str(int(rec[1])), _KNOB[int(rec[2])], str(int(rec[3])),
                                 _fixed6(rec[4]), _fixed6(rec[5]), _fixed6(rec[6]), _fixed6(rec[7]),
                                 _fixed6(rec[8]), "1" if rec[9] else "0"]) + "\n")
    return "".join(out)


def _jnum(v: float):
    # nlohmann dumps a double as its shortest round-trip form (integral values
    # keep ".0"), as Python's repr does; non-finite values become null
    return v if math.isfinite(v) else None


def _summary(job: C.JobSpec, r: C.JobResult, controller: str) -> dict:
    s = r.summary
    j = {"job_id": int(s["job_id"]) if not r.error else job.job_id, "dnn_id": job.dnn_id,
         "controller": controller}
    if r.error:
        j["error"] = r.error
        return j
    j["approach"] = _KNOB[int(s["approach_kind"])]
    j["profiled"] = bool(s["profiled"])
    if s["profiled"]:
        j["ti_batching"] = _jnum(s["ti_batching"])
        j["ti_mt"] = _jnum(s["ti_mt"])
        j["profiling_cost_ms"] = _jnum(s["profiling_cost_ms"])
    kind, value = s["steady_knob"]
    j["steady_knob"] = {"kind": _KNOB[int(kind)], "value": int(value)}
    j["converged"] = bool(s["converged"])
    j["knob_changes"] = int(s["knob_changes"])
    j["settle_period"] = int(s["settle_period"])
    j["periods"] = int(s["periods"])
    for k in ("duration_s", "total_items", "avg_throughput", "steady_throughput", "p95_overall_ms",
              "slo_compliance", "avg_power_w", "power_efficiency", "final_slo_ms"):
        j[k] = _jnum(float(s[k]))
    if r.readaptations:
        j["readaptations"] = [{"at_s": _jnum(a), "periods": int(p)} for a, p in r.readaptations]
    return j


def render_summary_json(scenario: C.Scenario, jobs: Sequence[C.JobSpec],
                        results: Sequence[C.JobResult]) -> str:
    """== render_summary_json (report.cpp:90-101): scenario header + one
    summary object per job (errors carry only id, dnn, controller, error)."""
    doc = {"seed": int(scenario.seed), "controller": scenario.controller,
           "sigma": _jnum(scenario.sigma), "alpha": _jnum(scenario.alpha),
           "jobs": [_summary(j, r, scenario.controller) for j, r in zip(jobs, results)]}
    return json.dumps(doc, indent=2, ensure_ascii=False) + "\n"


def render_sweep_csv(cells: Sequence[dict]) -> str:
    """== render_sweep_csv (report.cpp:103-118) over combination_sweep cells."""
    out = ["bs,mtl,mean_ms,p95_ms,throughput\n"]
    for c in cells:
        out.append(",".join([str(int(c["bs"])), str(int(c["mtl"])), _fixed6(c["mean_ms"]),
                             _fixed6(c["p95_ms"]), _fixed6(c["throughput"])]) + "\n")
    return "".join(out)


def render_profile_json(report: dict, dnn_id: str, approach: str) -> str:
    """== render_profile_json (report.cpp:120-138)."""
    j = {"dnn_id": dnn_id, "m": int(report["m"]), "n": int(report["n"]),
         "batches_per_point": int(report["batches_per_point"])}
    for k in ("tput_base", "tput_batching", "tput_mt", "ti_batching", "ti_mt", "base_latency_ms",
              "probe_latency_batching_ms", "probe_latency_mt_ms", "profiling_cost_ms"):
        j[k] = _jnum(float(report[k]))
    j["approach"] = approach
    return json.dumps(j, indent=2) + "\n"


def _improvement(a: float, b: float) -> float:
    # throughput_improvement (domain.cpp): (a - b) / b * 100
    return (a - b) / b * 100.0


def render_comparison_csv(jobs: Sequence[C.JobSpec], scaler: Sequence[C.JobResult],
                          clipper: Sequence[C.JobResult]) -> str:
    """== build_comparison + render_comparison_csv (report.cpp:140-190)."""
    out = ["job_id,dnn_id,approach,scaler_throughput,clipper_throughput,improvement_pct,"
           "scaler_steady,clipper_steady,steady_improvement_pct\n"]
    for job, a, b in zip(jobs, scaler, clipper):
        if a.error or b.error:
            continue
        sa, sb = a.summary, b.summary
        steady = (_improvement(sa["steady_throughput"], sb["steady_throughput"])
                  if sb["steady_throughput"] > 0.0 else 0.0)
        out.append(",".join([str(job.job_id), job.dnn_id, _KNOB[int(sa["approach_kind"])],
                             _fixed6(sa["avg_throughput"]), _fixed6(sb["avg_throughput"]),
                             _fixed6(_improvement(sa["avg_throughput"], sb["avg_throughput"])),
                             _fixed6(sa["steady_throughput"]), _fixed6(sb["steady_throughput"]),
                             _fixed6(steady)]) + "\n")
    return "".join(out)


def summary_table(jobs: Sequence[C.JobSpec], results: Sequence[C.JobResult]) -> str:
    """The reference CLI's console table (dnnscaler_main.cpp:72-86)."""
    lines = ["%5s  %-26s %-13s %6s  %12s  %10s  %10s  %8s" % (
        "job", "dnn", "knob", "value", "throughput", "p95_ms", "compliance", "power_w")]
    for job, r in zip(jobs, results):
        if r.error:
            lines.append("%5d  %-26s failed: %s" % (job.job_id, job.dnn_id, r.error))
            continue
        s = r.summary
        kind, value = s["steady_knob"]
        lines.append("%5d  %-26s %-13s %6d  %12.2f  %10.2f  %10.3f  %8.1f" % (
            job.job_id, job.dnn_id, _KNOB[int(kind)], int(value), s["avg_throughput"],
            s["p95_overall_ms"], s["slo_compliance"], s["avg_power_w"]))
    return "\n".join(lines) + "\n"
