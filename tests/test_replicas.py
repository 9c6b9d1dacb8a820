"""Config 5 host logic on CPU: a mixed trace sharded over world_size 2 with
the gloo backend (the analytic seam stands in for the devices). Per-job
traces must not depend on placement (SURVEY §8(e) invariant), and the
aggregate is total items / makespan.
"""
import json
import os

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_13803_b200 import control as C
from paper_2308_13803_b200 import replicas as R

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "ref_data")


def _trace():
    doc = json.load(open(os.path.join(GOLDEN, "scenario_30jobs.json")))
    jobs = [C.JobSpec(j["job_id"], j["dnn_id"], float(j["slo_ms"]), float(j["duration_s"]) / 20.0)
            for j in doc["jobs"][:12]]
    return jobs, C.load_catalog(os.path.join(GOLDEN, "catalog.json"))


def test_lpt_sharding_balances_and_covers():
    jobs, _ = _trace()
    for world in (1, 2, 4, 8):
        shards = R.shard_jobs(jobs, world)
        ids = sorted(j.job_id for s in shards for j in s)
        assert ids == sorted(j.job_id for j in jobs)
        loads = [sum(j.duration_s for j in s) for s in shards]
        assert max(loads) - min(loads) <= max(j.duration_s for j in jobs) + 1e-9
    with pytest.raises(ValueError):
        R.shard_jobs(jobs, 0)


def _worker(rank, world, port, out_path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    jobs, catalog = _trace()
    res = R.run_distributed(jobs, C.Scenario(), catalog, seam="analytic")
    if rank == 0:
        json.dump({"agg": {k: v for k, v in res.items() if k != "outcomes"},
                   "digests": {o.job_id: o.records_digest for o in res["outcomes"]},
                   "ranks": {o.job_id: o.rank for o in res["outcomes"]}}, open(out_path, "w"))
    dist.barrier()
    dist.destroy_process_group()


def test_two_ranks_gloo_match_single_process(tmp_path):
    jobs, catalog = _trace()
    single = R.run_shard(0, jobs, C.Scenario(), catalog, seam="analytic")
    out = tmp_path / "agg.json"
    port = 29500 + os.getpid() % 1000
    mp.spawn(_worker, args=(2, port, str(out)), nprocs=2, join=True)
    got = json.load(open(out))
    # placement-independent per-job traces
    for o in single:
        assert got["digests"][str(o.job_id)] == o.records_digest
    assert set(got["ranks"].values()) == {0, 1}
    items = sum(o.total_items for o in single)
    assert abs(got["agg"]["items"] - items) < 1e-6 * items
    assert got["agg"]["failed"] == 0
    one = R.aggregate(single, 1)
    assert got["agg"]["makespan_s"] < one["makespan_s"]  # two replicas finish sooner
