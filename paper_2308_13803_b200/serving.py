"""Serving runs on the B200 backend: knob sweeps, measured catalog rows and
closed-loop jobs under a p95 SLO — the pieces bench.py assembles into
BASELINE.json's five configs.

  batch_sweep / mt_sweep   static-knob sweeps (the reference's kStaticKnob
                           controller, harness.cpp:122-131, run as raw seam
                           windows): per knob the mean / nearest-rank p95
                           latency and throughput, timed on the device
  catalog_row              a reference-format catalog row (catalog.cpp:51-94)
                           from the sweeps: B200 curves for derive_mt_rows'
                           matrix-completion donors (harness.cpp:315-327)
  serve                    one job through the C++ JobRunner on the device
                           seam (Profiler + Scaler, or Clipper, or a static
                           knob), converged, then K control periods timed
                           device-resident and K more with host I/O (e2e)
  roofline_img_s           SURVEY §8(d) whole-network roofline
"""
from __future__ import annotations

import json
import os
from typing import Optional, Sequence

import numpy as np

from . import control as C
from .backend import Config, GpuBackend, kernel_costs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data")
B200_CATALOG = os.path.join(DATA, "b200_catalog.json")
P40_DONORS = os.path.join(DATA, "p40_donors.json")

# SLO = c x L(BS=1); c per model from the paper's jobs
# (job 18 MobV1-1, job 10 ResV2-50, job 16 Inc-V3, bench-net)
SLO_FACTOR = {"mobilenet_v1": 13.44, "resnet50_v1": 4.66, "inception_v3": 22.54,
              "synthetic_cnn": 4.15}
# (abs_max_bs, max_mtl) per config
MODEL_LIMITS = {"mobilenet_v1": (128, 10), "resnet50_v1": (256, 10), "inception_v3": (128, 16),
                "synthetic_cnn": (32, 4)}
PROBE = {"synthetic_cnn": (32, 4)}  # Profiler (m, n); default (32, 8)


def nearest_rank_p95(x) -> float:
    """reference percentile(), domain.cpp:14-24 (nearest rank)."""
    x = np.sort(np.asarray(x, dtype=np.float64))
    rank = int(np.ceil(0.95 * len(x) - 1e-9))
    return float(x[max(1, min(rank, len(x))) - 1])


def load_peaks():
    """(HBM GB/s, bf16 TFLOP/s burst, sustained, source) from MEASURED_PEAKS.json,
    else the B200_PROFILING.md fallback."""
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained"), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


def roofline_fwd_ms(model: str, bs: int) -> float:
    """Sum over the forward's kernels of max(flops / tensor peak, bytes / HBM)."""
    hbm, tflops, _, _ = load_peaks()
    t = 0.0
    for k in kernel_costs(model):
        t += max(bs * k["flops_per_image"] / (tflops * 1e12),
                 (bs * k["bytes_per_image"] + k["fixed_bytes"]) / (hbm * 1e9))
    return t * 1e3


def roofline_img_s(model: str, bs: int) -> float:
    """Whole-network roofline throughput at batch bs (MT with k instances
    each holding its own weights: the bs = 1 figure)."""
    return bs * 1e3 / roofline_fwd_ms(model, bs)


def batch_sweep(be: GpuBackend, bs_list: Sequence[int], calls: int = 30) -> list:
    out = []
    for bs in bs_list:
        be.run_batches(bs, 3)  # graph capture + warm-up
        be.timer_start()
        lat = be.run_batches(bs, calls)
        ms = be.timer_stop()
        mean = float(lat.mean())
        out.append({"bs": bs, "mean_ms": round(mean, 5), "p95_ms": round(nearest_rank_p95(lat), 5),
                    "throughput": round(bs * 1000.0 / mean, 2),
                    "measured_throughput": round(bs * calls * 1000.0 / ms, 2)})
    return out


def mt_sweep(be: GpuBackend, k_list: Sequence[int], calls_per_instance: int = 20) -> list:
    out = []
    for k in k_list:
        be.set_mtl(k)
        be.run_mt_requests(4 * k)  # warm-up
        be.timer_start()
        lat = be.run_mt_requests(calls_per_instance * k)
        ms = be.timer_stop()
        mean = float(lat.mean())
        out.append({"mtl": k, "mean_ms": round(mean, 5), "p95_ms": round(nearest_rank_p95(lat), 5),
                    "throughput": round(k * 1000.0 / mean, 2),
                    "measured_throughput": round(len(lat) * 1000.0 / ms, 2)})
    be.set_mtl(1)
    return out


def best_under_slo(sweep: list, key: str, slo_ms: float) -> Optional[dict]:
    """Brute-force operating point: max measured throughput with p95 <= SLO."""
    ok = [c for c in sweep if c["p95_ms"] <= slo_ms]
    return max(ok, key=lambda c: c["measured_throughput"]) if ok else None


def catalog_row(model: str, bsweep: list, msweep: list) -> C.DnnProfile:
    """Reference catalog row (domain.hpp:26-34) from device sweeps. The
    reference fits a + b*bs to the batching points and needs throughput to
    rise with bs (perf_model.cpp:37-44), and l1/capacity to the MT points;
    points are kept in sweep order."""
    from .backend import model_info
    mi = model_info(model)
    bp = [(c["bs"], c["measured_throughput"]) for c in bsweep]
    mp = [(c["mtl"], c["measured_throughput"]) for c in msweep]
    return C.DnnProfile(model, bp, mp, params_millions=round(mi.weight_count / 1e6, 3),
                        mflops=round(2 * mi.macs_per_image / 1e6, 1))


def write_catalog(rows: Sequence[C.DnnProfile], path: str) -> None:
    with open(path, "w") as f:
        json.dump([r.to_json() for r in rows], f, indent=1)
        f.write("\n")


def load_donors() -> list:
    """Matrix-completion donors for mt_init: the committed B200 catalog
    (measured sweeps, tools/make_b200_catalog.py), else the paper's P40 rows."""
    return C.load_catalog(B200_CATALOG if os.path.exists(B200_CATALOG) else P40_DONORS)


def probe_row(be: GpuBackend, model: str, m: int, n: int):
    """L(BS=1) and a minimal measured row (BS=1, BS=m, MT=n) of the served model."""
    be.run_batches(1, 10)
    l1 = float(np.median(be.run_batches(1, 50)))
    lat_m = float(np.median(be.run_batches(m, 20)))
    be.set_mtl(n)
    be.run_mt_requests(4 * n)
    mt = be.run_mt_requests(20 * n)
    be.set_mtl(1)
    # keep the row inside the reference catalog schema (increasing batch cost
    # with a non-negative intercept, perf_model.cpp:37-44)
    lat_m = min(max(lat_m, l1 * 1.001), m * l1 * 0.999)
    t1 = 1000.0 / l1
    t_mt = max(mt.size * 1000.0 / (mt.sum() / n), t1 * 1.0001)
    return l1, C.DnnProfile(model, [(1, t1), (m, m * 1000.0 / lat_m)], [(1, t1), (n, t_mt)])


def serve(be: GpuBackend, model: str, *, controller: str = "dnnscaler", slo_factor: float = None,
          limits=None, probe=None, steps: int = 10, warmup: int = 3, max_converge: int = 40,
          knob=None, e2e: bool = True, job_id: int = 1, nvtx=None, between=None) -> dict:
    """One closed-loop job on `be` (the C++ JobRunner over the device seam):
    run until the knob holds for 4 periods, W warm-up periods, then K timed
    periods device-resident (cudaEvent timer over every instance stream), and
    (e2e) W/2 + K more with host I/O inside every request. `knob` = (kind,
    value) runs the reference's static-knob controller instead of the search.
    `between(timed_fn)` lets the caller wrap the timed region (clocks, energy)."""
    max_bs, max_mtl = limits or MODEL_LIMITS[model]
    m, n = probe or PROBE.get(model, (32, 8))
    window = 100
    l1, row = probe_row(be, model, m, n)
    catalog = [row] + [d for d in load_donors() if d.id != model]
    slo = (slo_factor or SLO_FACTOR[model]) * l1
    sc = C.Scenario(controller=controller, seed=42, alpha=0.85, m=m, n=n, abs_max_bs=max_bs,
                    max_mtl=max_mtl, window=window)
    if knob is not None:
        sc.controller = "static"
        sc.static_knob = (0 if knob[0] in (0, "batching") else 1, int(knob[1]))
    sess = C.JobSession(sc, C.JobSpec(job_id, model, slo, 1e9), catalog, seam="device", backend=be)
    knobs = []
    for _ in range(max_converge):
        rec, _ = sess.step()
        knobs.append(rec["knob"])
        if len(knobs) >= 4 and knobs[-1] == knobs[-2] == knobs[-3] == knobs[-4]:
            break
    for _ in range(warmup):
        sess.step()

    def timed(k, tag):
        items = 0.0
        st0 = be.stats()
        if nvtx:
            nvtx(tag, True)
        be.timer_start()
        be.reset_kernel_spans(0)
        recs = []
        for _ in range(k):
            rec, _ = sess.step()
            recs.append(rec)
            kk = rec["knob"]
            items += window * (kk[1] if kk[0] == 0 else 1)
        ms = be.timer_stop()
        if nvtx:
            nvtx(tag, False)
        spans[tag] = be.kernel_spans(0)
        return items, ms, recs, st0, be.stats()

    spans = {}

    if between is not None:
        items, ms, recs, st0, st1 = between(lambda: timed(steps, "timed"))
    else:
        items, ms, recs, st0, st1 = timed(steps, "timed")
    out = {"items": items, "ms": ms, "launches": int(st1["kernel_launches"] - st0["kernel_launches"]),
           "kernel_spans_ms": spans["timed"][0].tolist(), "span_forwards": spans["timed"][1]}
    e_warm = 0
    if e2e:
        be.set_host_io(True)
        e_warm = max(1, warmup // 2)
        for _ in range(e_warm):
            sess.step()
        e_items, e_ms, e_recs, e0, e1 = timed(steps, "timed_e2e")
        be.set_host_io(False)
        out.update(e_items=e_items, e_ms=e_ms, e_knob=list(e_recs[-1]["knob"]),
                   h2d=int((e1["h2d_bytes"] - e0["h2d_bytes"]) / steps),
                   d2h=int((e1["d2h_bytes"] - e0["d2h_bytes"]) / steps))
    res = sess.finish()
    tail = ((e_warm + steps) * window) if e2e else 0  # latencies served after the timed region
    end = res.latencies.size - tail
    timed_lat = res.latencies[end - steps * window:end]
    rep = res.report
    k = recs[-1]["knob"]
    p95 = nearest_rank_p95(timed_lat)
    bs_op = k[1] if k[0] == 0 else 1
    out.update({
        "value": items / (ms * 1e-3),
        "knob": {"kind": "batching" if k[0] == 0 else "multi-tenancy", "value": k[1]},
        "knob_trajectory": [list(x) for x in knobs],
        "slo_ms": slo, "l1_ms": l1, "p95_ms_timed": p95, "p95_within_slo": bool(p95 <= slo),
        "controller": sc.controller,
        "profiler": ({"ti_batching": rep.get("ti_batching", 0.0), "ti_mt": rep.get("ti_mt", 0.0),
                      "approach": "multi-tenancy" if res.summary["approach_kind"] else "batching",
                      "tput_base": rep.get("tput_base", 0.0),
                      "tput_batching": rep.get("tput_batching", 0.0),
                      "tput_mt": rep.get("tput_mt", 0.0)}
                     if sc.controller == "dnnscaler" else None),
        "static_knob": list(sc.static_knob) if sc.controller == "static" else None,
        "scenario": {"m": m, "n": n, "abs_max_bs": max_bs, "max_mtl": max_mtl, "window": window,
                     "alpha": 0.85},
        "roofline_img_s": roofline_img_s(model, bs_op),
        "summary": res.summary,
    })
    out["roofline_achieved_frac"] = out["value"] / out["roofline_img_s"]
    return out
