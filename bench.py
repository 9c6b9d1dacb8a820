#!/usr/bin/env python
"""DNNScaler on B200 — headline benchmark.

Metric (BASELINE.json): inferences/sec at p95 latency SLO (Batching vs
Multi-Tenancy). N=1 workload = configs[1]: MobileNet-v1 224x224 synthetic
images, Profiler + Scaler on one B200 (m=32, n=8, abs_max_bs=128,
max_mtl=10, window=100, alpha=0.85), SLO = 13.44 x L(BS=1) measured on the
device at start (paper's job-18 ratio).

A "step" is one control period: 100 seam calls at the Scaler's current knob
(100 batches of bs images, or 100 co-located bs=1 requests) plus the Scaler
decision. After the job has converged and W warm-up periods, K periods are
timed with cudaEvents (drain + event at both ends, max over ranks).

  value        items/s over the K timed periods, inputs resident in HBM
  e2e          the same through the C ABI with host I/O: every request copies
               its u8 images from pinned host memory and its fp32 logits back
               inside its timed event pair
  roofline     dominant kernel = the tcgen05 implicit-GEMM conv (all its
               launches in one forward at the steady knob), timed live with
               event nodes between kernels
  cpu_baseline FP32 C oracle forward (port) on this host, bounded sample

--impl reference: the reference's CPU path on this host — the compiled,
unmodified reference control plane (oracle/_ref) driving the FP32 C oracle
forward pass (the reference has no forward pass of its own).
Multi-GPU (torchrun): one independent replica per GPU (weak scaling, no
collective on the data path); value = sum of items / max elapsed.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SLO_FACTOR = {"mobilenet_v1": 13.44, "resnet50_v1": 4.66, "inception_v3": 22.54,
              "synthetic_cnn": 4.15}
MODEL_LIMITS = {"mobilenet_v1": (128, 10), "resnet50_v1": (256, 10), "inception_v3": (128, 16),
                "synthetic_cnn": (32, 4)}
PROBE = {"synthetic_cnn": (32, 4)}  # (m, n); default (32, 8)


def dist_setup(gpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        return rank, world, local, dist
    return rank, world, local, None


def reduce_max_sum(dist, local, values_max, values_sum):
    if dist is None:
        return values_max, values_sum
    import torch
    t = torch.tensor(values_max, dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    s = torch.tensor(values_sum, dtype=torch.float64, device=f"cuda:{local}")
    dist.all_reduce(s, op=dist.ReduceOp.SUM)
    return t.tolist(), s.tolist()


def barrier(dist):
    if dist is not None:
        dist.barrier()


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms (B200_PROFILING.md)."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.lines = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.device}", f"--query-gpu={self.QUERY}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        sm, mx, reasons, power = [], [], set(), []
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm),
                "power_w_median": float(np.median(power)) if power else None}


class EnergyMeter:
    """NVML board energy counter across the timed region (SURVEY §8(f) row 1:
    measured power for the paper's throughput-per-watt comparison, Table 5)."""

    def __init__(self, device):
        self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device)
        except Exception:  # noqa: BLE001 - no NVML: report null
            self.h = None

    def read_mj(self):
        if self.h is None:
            return None
        try:
            return self.nvml.nvmlDeviceGetTotalEnergyConsumption(self.h)  # millijoules
        except Exception:  # noqa: BLE001
            return None


def nearest_rank_p95(x):
    x = np.sort(np.asarray(x))
    rank = int(np.ceil(0.95 * len(x) - 1e-9))
    return float(x[max(1, min(rank, len(x))) - 1])


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], p.get("bf16_tflops_sustained"), "measured"
    return 6650.0, 1590.0, 1400.0, "fallback"


def roofline(be, model, knob, kernel_costs):
    """Dominant kernel (implicit-GEMM conv) at the steady knob, timed live."""
    bs = knob[1] if knob[0] == 0 else 1
    ms = be.profile_kernels(bs, reps=20)
    conv = [i for i, k in enumerate(kernel_costs) if k["kind"] == "conv_gemm"]
    conv_ms = float(sum(ms[i] for i in conv))
    conv_bytes = sum(bs * kernel_costs[i]["bytes_per_image"] + kernel_costs[i]["fixed_bytes"]
                     for i in conv)
    conv_flops = sum(bs * kernel_costs[i]["flops_per_image"] for i in conv)
    fwd_ms = float(ms.sum())
    hbm, tflops, tflops_sus, src = load_peaks()
    ai = conv_flops / conv_bytes
    ridge = tflops * 1e12 / (hbm * 1e9)
    per_launch = [dict(kernel=i, kind=kernel_costs[i]["kind"], ms=float(ms[i]),
                       gbs=(bs * kernel_costs[i]["bytes_per_image"] + kernel_costs[i]["fixed_bytes"])
                       / (ms[i] * 1e-3) / 1e9,
                       tflops=bs * kernel_costs[i]["flops_per_image"] / (ms[i] * 1e-3) / 1e12)
                  for i in range(len(ms))]
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        with open(tpath) as f:
            t = json.load(f)
        key = f"{model}:bs{bs}"
        if key in t:
            traffic = t[key].get("conv_gemm_dram_bytes_per_forward")
    if ai < ridge:
        achieved = conv_bytes / (conv_ms * 1e-3) / 1e9
        r = {"bound": "hbm", "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
             "frac": round(achieved / hbm, 4), "traffic": traffic}
    else:
        achieved = conv_flops / (conv_ms * 1e-3) / 1e12
        r = {"bound": "tensor", "achieved": round(achieved, 1), "peak": tflops, "unit": "TFLOP/s",
             "frac": round(achieved / tflops, 4), "traffic": traffic}
    r.update({"kernel": "conv_gemm (tcgen05 implicit GEMM), all launches of one forward",
              "peak_source": src, "batch": bs, "launches": len(conv),
              "algorithmic_bytes": conv_bytes, "algorithmic_flops": conv_flops,
              "arith_intensity": round(ai, 1), "ridge": round(ridge, 1),
              "kernel_ms": round(conv_ms, 4), "forward_ms": round(fwd_ms, 4),
              "share_of_forward": round(conv_ms / fwd_ms, 4),
              "forward_hbm_frac": round(
                  (sum(bs * k["bytes_per_image"] + k["fixed_bytes"] for k in kernel_costs)
                   / (fwd_ms * 1e-3) / 1e9) / hbm, 4)})
    return r, per_launch


def cpu_baseline(model, seconds=12.0):
    """FP32 C oracle forward (the reference has no forward pass: port) on all host cores."""
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import oracle
    threads = oracle.fwd().oracle_get_threads()
    imgs = oracle.images(model, 0, 1)
    t0 = time.perf_counter()
    oracle.forward(model, imgs, bf16_storage=False, threads=threads)
    one = time.perf_counter() - t0
    n = int(max(threads, min(8192, seconds / max(one, 1e-6) * threads)))
    n = max(threads, (n // threads) * threads)
    imgs = oracle.images(model, 0, n)
    t0 = time.perf_counter()
    oracle.forward(model, imgs, bf16_storage=False, threads=threads)
    dt = time.perf_counter() - t0
    return {"value": round(n / dt, 3), "unit": "inferences/s", "cores": threads, "kind": "port",
            "sample": f"{n} synthetic {model} images through the FP32 C oracle "
                      f"(oracle/fwd_oracle.c), {threads} threads, {dt:.1f} s"}


def build_catalog(be, model, m, n):
    """The served model's catalog row, measured on the device (B200 curves),
    plus the paper's P40 rows as matrix-completion donors."""
    from paper_2308_13803_b200 import control as C
    be.run_batches(1, 10)
    l1 = float(np.median(be.run_batches(1, 50)))
    lat_m = float(np.median(be.run_batches(m, 20)))
    be.set_mtl(n)
    be.run_mt_requests(4 * n)
    mt = be.run_mt_requests(20 * n)
    be.set_mtl(1)
    # The reference catalog schema needs an increasing, non-negative-intercept
    # batch cost (perf_model.cpp:37-44); keep the measured row inside it even
    # when a profiler distorts the timings.
    lat_m = min(max(lat_m, l1 * 1.001), m * l1 * 0.999)
    t1 = 1000.0 / l1
    t_mt = max(mt.size * 1000.0 / (mt.sum() / n), t1 * 1.0001)
    row = C.DnnProfile(model, [(1, t1), (m, m * 1000.0 / lat_m)], [(1, t1), (n, t_mt)])
    donors = C.load_catalog(os.path.join(ROOT, "paper_2308_13803_b200", "data", "p40_donors.json"))
    return l1, [row] + donors


def run_ours(args, rank, world, local, dist):
    from paper_2308_13803_b200 import Config, GpuBackend
    from paper_2308_13803_b200 import control as C
    from paper_2308_13803_b200.backend import kernel_costs

    model = args.model
    max_bs, max_mtl = MODEL_LIMITS[model]
    m, n = PROBE.get(model, (32, 8))
    window = 100
    be = GpuBackend(model, Config(max_bs, max_mtl), seed=42 + rank, device=local)
    l1, catalog = build_catalog(be, model, m, n)
    slo = SLO_FACTOR[model] * l1
    sc = C.Scenario(controller=args.controller, seed=42, alpha=0.85, m=m, n=n,
                    abs_max_bs=max_bs, max_mtl=max_mtl, window=window)
    if args.knob:  # static knob (profiling runs): skips the Profiler/Scaler search
        kind, value = args.knob.split(":")
        sc.controller = "static"
        sc.static_knob = (0 if kind == "batching" else 1, int(value))
    job = C.JobSpec(1 + rank, model, slo, 1e9)
    sess = C.JobSession(sc, job, catalog, seam="device", backend=be)
    # converge: until the knob holds for 3 periods
    knobs = []
    for _ in range(args.max_converge):
        rec, _ = sess.step()
        knobs.append(rec["knob"])
        if len(knobs) >= 4 and knobs[-1] == knobs[-2] == knobs[-3] == knobs[-4]:
            break
    for _ in range(args.warmup):
        sess.step()

    from paper_2308_13803_b200 import _lib as L

    def timed(steps, tag):
        items = 0.0
        st0 = be.stats()
        barrier(dist)
        be.timer_start()
        L.load().ds_nvtx_push(tag.encode())
        recs = []
        for _ in range(steps):
            rec, _ = sess.step()
            recs.append(rec)
            k = rec["knob"]
            items += window * (k[1] if k[0] == 0 else 1)
        ms = be.timer_stop()
        L.load().ds_nvtx_pop()
        st1 = be.stats()
        return items, ms, recs, st0, st1

    sampler = ClockSampler(local)
    meter = EnergyMeter(local)
    sampler.start()
    e_start = meter.read_mj()
    items, ms, recs, st0, st1 = timed(args.steps, "timed")
    e_end = meter.read_mj()
    clocks = sampler.stop()
    energy = None
    if e_start is not None and e_end is not None and e_end > e_start:
        joules = (e_end - e_start) / 1000.0
        energy = {"joules": round(joules, 3), "avg_power_w": round(joules / (ms * 1e-3), 1),
                  "inferences_per_joule": round(items / joules, 1),
                  "source": "NVML total energy counter over the timed periods (board power)"}
    # e2e through host buffers, same session (the Scaler keeps control)
    be.set_host_io(True)
    e_warm = max(1, args.warmup // 2)
    for _ in range(e_warm):
        sess.step()
    e_items, e_ms, e_recs, e0, e1 = timed(args.steps, "timed_e2e")
    be.set_host_io(False)
    res = sess.finish()
    tail = (e_warm + args.steps) * window  # latencies served after the timed region
    end = res.latencies.size - tail
    timed_lat = res.latencies[end - args.steps * window:end]
    knob = recs[-1]["knob"]
    costs = kernel_costs(model)
    rl, per_launch = roofline(be, model, knob, costs) if rank == 0 else (None, None)
    (max_ms, max_ems), (sum_items, sum_eitems) = reduce_max_sum(dist, local, [ms, e_ms],
                                                                [items, e_items])
    value = sum_items / (max_ms * 1e-3)
    e2e = sum_eitems / (max_ems * 1e-3)
    if rank != 0:
        return None
    rep = res.report
    info = be.info
    fwd_flops = 2 * info.macs_per_image
    out = {
        "metric": "inferences/sec at p95 latency SLO (Batching vs Multi-Tenancy), 1/2/4/8 B200",
        "value": round(value, 2),
        "unit": "inferences/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(max_ms / args.steps, 4),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (seeded u8 images, seeded He-init weights with folded BN; DESIGN.md)",
        "config": {
            "workload": f"{model} {info.in_h}x{info.in_w}, "
                        f"{'DNNScaler Profiler+Scaler' if args.controller == 'dnnscaler' else 'Clipper AIMD'}, "
                        f"SLO = {SLO_FACTOR[model]} x L(BS=1)",
            "model": model,
            "global_batch": knob[1] if knob[0] == 0 else knob[1] * world,
            "knob": {"kind": "batching" if knob[0] == 0 else "multi-tenancy", "value": knob[1]},
            "slo_ms": round(slo, 4),
            "l1_ms": round(l1, 4),
            "p95_ms_timed": round(nearest_rank_p95(timed_lat), 4),
            "p95_within_slo": bool(nearest_rank_p95(timed_lat) <= slo),
            "profiler": {"ti_batching": round(rep.get("ti_batching", 0.0), 2),
                         "ti_mt": round(rep.get("ti_mt", 0.0), 2),
                         "approach": res.summary["approach_kind"] and "multi-tenancy" or "batching",
                         "tput_base": round(rep.get("tput_base", 0.0), 1),
                         "tput_batching": round(rep.get("tput_batching", 0.0), 1),
                         "tput_mt": round(rep.get("tput_mt", 0.0), 1)}
            if args.controller == "dnnscaler" else None,
            "controller": args.controller,
            "knob_trajectory": [list(k) for k in knobs],
            "scenario": {"m": m, "n": n, "abs_max_bs": max_bs, "max_mtl": max_mtl,
                         "window": window, "alpha": 0.85},
            "parallelism": f"replicas x{world} (no collective on the data path)",
            "l2": "working set per step > 126 MB L2 (bs x 21 MB activations per MobileNet image)"
                  if knob[0] == 0 and knob[1] >= 8 else "bs=1 requests; weights L2-resident",
            "fwd_gflop_per_image": round(fwd_flops / 1e9, 4),
            "achieved_tflops_whole_forward": round(value * fwd_flops / 1e12, 2),
        },
        "e2e": {"value": round(e2e, 2), "unit": "inferences/s",
                "h2d_bytes_per_step": int((e1["h2d_bytes"] - e0["h2d_bytes"]) / args.steps),
                "d2h_bytes_per_step": int((e1["d2h_bytes"] - e0["d2h_bytes"]) / args.steps),
                "knob": list(e_recs[-1]["knob"])},
        "gpu_launches": int(st1["kernel_launches"] - st0["kernel_launches"]),
        "roofline": rl,
        "clocks": clocks,
        "energy": energy,
    }
    if world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(model, args.cpu_seconds)
    if args.kernel_table:
        out["kernel_table"] = per_launch
    be.close()
    return out


def run_reference(args, rank, world, local, dist):
    """The reference's CPU serving path on this host (rank 0 only)."""
    if rank != 0:
        return None
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    import ref_cpu_serving
    return ref_cpu_serving.run(args.model, args.steps, args.warmup, SLO_FACTOR[args.model],
                               MODEL_LIMITS[args.model], PROBE.get(args.model, (32, 8)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--model", default="mobilenet_v1", choices=sorted(SLO_FACTOR))
    ap.add_argument("--max-converge", type=int, default=40)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--kernel-table", action="store_true")
    ap.add_argument("--knob", default="", help="static knob, e.g. batching:128 (profiling only)")
    ap.add_argument("--controller", default="dnnscaler", choices=["dnnscaler", "clipper"],
                    help="clipper: the paper's baseline controller on the same backend "
                         "(Table 5 comparison; the headline is dnnscaler)")
    args = ap.parse_args()
    if args.warmup < 3:
        ap.error("--warmup must be >= 3")
    rank, world, local, dist = dist_setup(args.gpus)
    out = (run_reference if args.impl == "reference" else run_ours)(args, rank, world, local, dist)
    if out is not None:
        if args.impl == "reference":
            out["impl"] = "reference"
        print(json.dumps(out), flush=True)
    if dist is not None:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
