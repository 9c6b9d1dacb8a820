"""bench.py --impl reference: the reference's serving path on this host's CPU
cores — TEST/BASELINE INFRASTRUCTURE ONLY.

The reference has no forward pass (its GpuSim returns a + b*bs ms,
reference perf_model.cpp:70-86), so its "CPU implementation of the path" is
assembled from:
  * the UNMODIFIED reference control plane — profile()/decide(), the Scaler,
    matrix completion, run_job() — compiled from /root/reference sources into
    oracle/_ref/libref_replay.so, with GpuSim replaced by a callback seam;
  * the FP32 C oracle forward pass (oracle/fwd_oracle.c) as the device: each
    run_batch(bs) is a timed CPU forward of bs synthetic images on all host
    threads; each run_mt_request() at mtl k is one of k concurrent
    single-image forwards (k instances co-located on the CPU).
Same metric, workload and SLO rule as the B200 arm (SLO = c x L(BS=1)
measured on this platform) and the same --steps K / --warmup W; each step
is a bounded sample of the workload (a control window of 10 requests
instead of 100: one bs-128 window costs ~6 s of CPU forward), so the run
stays within minutes.
"""
from __future__ import annotations

import ctypes
import json
import os
import time

import numpy as np

import oracle
import ref

HERE = os.path.dirname(os.path.abspath(__file__))
DONORS = os.path.join(os.path.dirname(HERE), "paper_2308_13803_b200", "data", "p40_donors.json")
WINDOW = 10

_BATCH = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.c_int)
_MT = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.c_int)
_CHANGE = ctypes.CFUNCTYPE(ctypes.c_double, ctypes.c_int)


class CpuDevice:
    """The CPU 'device' behind the reference seam."""

    def __init__(self, model: str, max_images: int):
        self.model = model
        self.imgs = oracle.images(model, 0, max_images)
        self.threads = oracle.fwd().oracle_get_threads()
        self.mt_queue = []
        self.calls = 0

    def forward_ms(self, count: int, threads: int) -> float:
        t0 = time.perf_counter()
        oracle.forward(self.model, self.imgs[:count], bf16_storage=False, threads=threads)
        return (time.perf_counter() - t0) * 1000.0

    def batch(self, bs: int) -> float:
        self.calls += 1
        return self.forward_ms(bs, self.threads)

    def mt(self, k: int) -> float:
        # k co-located single-image instances run together; each of the next k
        # requests reports that co-located latency.
        self.calls += 1
        if not self.mt_queue:
            lat = self.forward_ms(k, min(k, self.threads))
            self.mt_queue = [lat] * k
        return self.mt_queue.pop()

    def change(self, delta: int) -> float:
        self.mt_queue = []
        return 0.001  # instances share the process: launching one is free on the CPU


def run(model: str, steps: int, warmup: int, slo_factor: float, limits, probe) -> dict:
    max_bs, max_mtl = limits
    m, n = probe
    dev = CpuDevice(model, max_bs)
    # L(BS=1) and the served model's catalog row, measured on this CPU
    l1 = float(np.median([dev.forward_ms(1, dev.threads) for _ in range(3)]))
    lm = dev.forward_ms(m, dev.threads)
    lmt = dev.forward_ms(n, min(n, dev.threads))
    lm = min(max(lm, l1 * 1.001), m * l1 * 0.999)
    t1 = 1000.0 / l1
    catalog = [{"id": model, "params_millions": 1.0, "mflops": 1.0,
                "batching_points": [[1, t1], [m, m * 1000.0 / lm]],
                "mt_points": [[1, t1], [n, max(n * 1000.0 / lmt, t1 * 1.0001)]]}]
    with open(DONORS) as f:
        catalog += json.load(f)
    slo = slo_factor * l1
    # duration: profiling plus enough control periods to converge + W + K
    period_guess_ms = WINDOW * lm
    # (enough periods for the search to converge, then W warm-up + K timed)
    duration_s = (30 * l1 + 10 * lm + 10 * lmt + (16 + warmup + steps) * period_guess_ms) / 1000.0
    sc = {"controller": "dnnscaler", "seed": 42, "alpha": 0.85, "m": m, "n": n,
          "abs_max_bs": max_bs, "max_mtl": max_mtl, "window": WINDOW, "sigma": 0.05,
          "jobs": [{"job_id": 1, "dnn_id": model, "slo_ms": slo, "duration_s": duration_s}]}
    d = ref.tempdir()
    spath = ref.write_scenario(sc, catalog, d)
    lib = ref.lib()
    cbs = (_BATCH(dev.batch), _MT(dev.mt), _CHANGE(dev.change))
    lib.ref_set_callbacks.argtypes = [_BATCH, _MT, _CHANGE]
    lib.ref_set_callbacks(*cbs)
    t0 = time.perf_counter()
    res = ref.run_job(spath, 0, "callback")
    wall = time.perf_counter() - t0
    recs = res["records"]  # [time_s, job, kind, value, p95, mean, tput, power, slo, violated]
    if len(recs) < steps:
        raise RuntimeError(f"reference job served {len(recs)} periods < {steps} timed steps")
    k = steps
    tail = recs[-k:]
    # per-period elapsed = items / throughput; value over the last K periods
    items = np.where(tail[:, 2] == 0, WINDOW * tail[:, 3], WINDOW)
    elapsed_ms = items * 1000.0 / tail[:, 6]
    value = float(items.sum() * 1000.0 / elapsed_ms.sum())
    summ = res["summary"]
    knob = ("batching" if tail[-1, 2] == 0 else "multi-tenancy", int(tail[-1, 3]))
    return {
        "metric": "inferences/sec at p95 latency SLO (Batching vs Multi-Tenancy), 1/2/4/8 B200",
        "value": round(value, 3),
        "unit": "inferences/s",
        "n_gpus": 1,
        "steps": k,
        "warmup": warmup,
        "ms_per_step": round(float(elapsed_ms.mean()), 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "fp32",
        "data": "synthetic (same seeded images and weights as the B200 arm)",
        "config": {"workload": f"{model} {dev.imgs.shape[1]}x{dev.imgs.shape[2]}, DNNScaler "
                               f"Profiler+Scaler, SLO = {slo_factor} x L(BS=1)",
                   "model": model, "global_batch": knob[1] if knob[0] == "batching" else 1,
                   "device": f"host CPU, {dev.threads} threads (reference control plane + "
                             f"FP32 C oracle forward)",
                   "slo_ms": round(slo, 3), "l1_ms": round(l1, 3),
                   "knob": {"kind": knob[0], "value": knob[1]},
                   "profiler": {"ti_batching": round(summ["ti_batching"], 2),
                                "ti_mt": round(summ["ti_mt"], 2),
                                "approach": "multi-tenancy" if summ["approach_kind"] else "batching"},
                   "window": WINDOW, "periods": len(recs), "p95_ms_last": round(float(tail[-1, 4]), 3),
                   "wall_s": round(wall, 1)},
        "cpu_baseline": {"value": round(value, 3), "unit": "inferences/s", "cores": dev.threads,
                         "kind": "reference",
                         "sample": f"reference control plane (oracle/_ref, compiled from "
                                   f"/root/reference sources) driving the FP32 C oracle forward "
                                   f"on {dev.threads} threads; last {k} of {len(recs)} periods of "
                                   f"{WINDOW} requests"},
        "e2e": {"value": round(value, 3), "unit": "inferences/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
