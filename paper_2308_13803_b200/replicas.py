"""Multi-GPU serving of a job trace: replicas only.

Jobs are independent — per-job seeds mix_seed(seed, job_id) (reference
harness.cpp:40-41), no cross-job state — so each rank (one
process per GPU) runs its share of the trace sequentially on its own
backend, Profiler and Scaler, exactly as the reference's run_scenario does
on one device (harness.cpp:340-352). Nothing crosses NVLink on the data
path; torch.distributed is only used to gather per-job summaries.

Shards are assigned by LPT (longest expected job first onto the least
loaded rank) on the jobs' durations.
"""
from __future__ import annotations

import json
import os
from dataclasses import dataclass
from typing import Callable, List, Optional, Sequence

from . import control as C


def shard_jobs(jobs: Sequence[C.JobSpec], world: int) -> List[List[C.JobSpec]]:
    """LPT on duration; deterministic (ties broken by job_id)."""
    if world < 1:
        raise ValueError("world must be positive")
    load = [0.0] * world
    shards: List[List[C.JobSpec]] = [[] for _ in range(world)]
    for job in sorted(jobs, key=lambda j: (-j.duration_s, j.job_id)):
        r = min(range(world), key=lambda i: (load[i], i))
        shards[r].append(job)
        load[r] += job.duration_s
    for s in shards:
        s.sort(key=lambda j: j.job_id)  # run in trace order on each rank
    return shards


@dataclass
class JobOutcome:
    job_id: int
    dnn_id: str
    rank: int
    steady_knob: tuple
    steady_throughput: float
    total_items: float
    duration_s: float
    slo_compliance: float
    records_digest: int
    error: str


def _digest(records) -> int:
    import hashlib

    return int.from_bytes(hashlib.sha256(records.tobytes()).digest()[:8], "little")


def run_shard(rank: int, jobs: Sequence[C.JobSpec], scenario: C.Scenario,
              catalog: Sequence[C.DnnProfile], seam: str = "device", device: int = 0,
              run: Optional[Callable] = None) -> List[JobOutcome]:
    """Runs this rank's jobs in order (each on a fresh seam, seeded by job id)."""
    run = run or C.run_job
    out = []
    for job in jobs:
        res = run(scenario, job, catalog, seam=seam, device=device)
        s = res.summary
        out.append(JobOutcome(job.job_id, job.dnn_id, rank, tuple(s["steady_knob"]),
                              s["steady_throughput"], s["total_items"], s["duration_s"],
                              s["slo_compliance"], _digest(res.records), res.error))
    return out


def aggregate(outcomes: Sequence[JobOutcome], world: int) -> dict:
    """Whole-trace inferences/s = total items / makespan (slowest rank)."""
    busy = [0.0] * world
    items = 0.0
    for o in outcomes:
        busy[o.rank] += o.duration_s
        items += o.total_items
    makespan = max(busy) if busy else 0.0
    return {"items": items, "makespan_s": makespan,
            "inferences_per_s": items / makespan if makespan > 0 else 0.0,
            "jobs": len(outcomes), "failed": sum(1 for o in outcomes if o.error)}


def run_distributed(jobs: Sequence[C.JobSpec], scenario: C.Scenario,
                    catalog: Sequence[C.DnnProfile], seam: str = "device") -> Optional[dict]:
    """Under torchrun: shard, serve this rank's share, gather on rank 0."""
    import torch.distributed as dist

    rank, world = dist.get_rank(), dist.get_world_size()
    mine = shard_jobs(jobs, world)[rank]
    import os

    import torch

    device = int(os.environ.get("LOCAL_RANK", rank % max(1, torch.cuda.device_count())))
    local = run_shard(rank, mine, scenario, catalog, seam=seam, device=device)
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(local, gathered, dst=0)
    if rank != 0:
        return None
    flat = [o for part in gathered for o in part]
    flat.sort(key=lambda o: o.job_id)
    res = aggregate(flat, world)
    res["outcomes"] = flat
    return res


# ------------------------------------------------------------------ config 5

TRACE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "scenario_30jobs.json")
# the reference trace's DNN families -> the architectures built here
FAMILY = (("mobv1-", "mobilenet_v1"), ("resv2-", "resnet50_v1"), ("inc-", "inception_v3"))


def _l1_ms(row: C.DnnProfile) -> float:
    """L(BS=1) of a catalog row: 1000 / throughput at bs = 1."""
    for x, t in row.batching_points:
        if int(x) == 1:
            return 1000.0 / float(t)
    raise ValueError(f"catalog row {row.id} has no bs=1 point")


def mixed_trace(b200_catalog: Sequence[C.DnnProfile], p40_catalog: Sequence[C.DnnProfile],
                duration_scale: float = 1.0 / 200.0, trace_path: str = TRACE):
    """the reference's 30-job trace
    (data/scenario_30jobs.json) restricted to the implemented families. Each
    job keeps its SLO tightness c = slo_ms / L_P40(BS=1) of its own P40 DNN
    (PAPER.md:384 rule), re-based on the B200 L(BS=1) of the architecture that
    serves it; durations scaled by duration_scale (virtual = device time).
    Returns (scenario, jobs)."""
    with open(trace_path) as f:
        doc = json.load(f)
    p40 = {r.id: r for r in p40_catalog}
    b200 = {r.id: r for r in b200_catalog}
    jobs = []
    for j in doc["jobs"]:
        model = next((m for pre, m in FAMILY if j["dnn_id"].startswith(pre)), None)
        if model is None or j["dnn_id"] not in p40 or model not in b200:
            continue
        c = float(j["slo_ms"]) / _l1_ms(p40[j["dnn_id"]])
        jobs.append(C.JobSpec(int(j["job_id"]), model, c * _l1_ms(b200[model]),
                              float(j["duration_s"]) * duration_scale))
    sc = C.Scenario(controller=doc.get("controller", "dnnscaler"), seed=int(doc.get("seed", 42)),
                    alpha=float(doc.get("alpha", 0.85)), m=int(doc.get("m", 32)),
                    n=int(doc.get("n", 8)), abs_max_bs=int(doc.get("abs_max_bs", 128)),
                    max_mtl=int(doc.get("max_mtl", 10)), window=int(doc.get("window", 100)))
    return sc, jobs
