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
    local = run_shard(rank, mine, scenario, catalog, seam=seam, device=rank % 8)
    gathered = [None] * world if rank == 0 else None
    dist.gather_object(local, gathered, dst=0)
    if rank != 0:
        return None
    flat = [o for part in gathered for o in part]
    flat.sort(key=lambda o: o.job_id)
    res = aggregate(flat, world)
    res["outcomes"] = flat
    return res
