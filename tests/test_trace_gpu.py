"""Config 5 on the device: the reference's mixed
30-job trace restricted to the built families, per-job SLO tightness kept
(replicas.mixed_trace), served job by job on the B200 with per-job seeds;
then the recorded tapes are replayed with the jobs LPT-sharded over a
world-size-2 gloo group: every job's records are identical wherever it runs
(per-job seeds make traces placement-independent)."""
import json
import os

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2308_13803_b200 import control as C
from paper_2308_13803_b200 import replicas as R
from paper_2308_13803_b200 import serving as S

pytestmark = pytest.mark.gpu


def _trace():
    b200 = C.load_catalog(S.B200_CATALOG)
    sc, jobs = R.mixed_trace(b200, C.load_catalog(S.P40_DONORS), duration_scale=1.0 / 1500.0)
    picked = [j for j in jobs if j.dnn_id == "mobilenet_v1"][:2] + \
             [j for j in jobs if j.dnn_id == "resnet50_v1"][:2] + \
             [j for j in jobs if j.dnn_id == "inception_v3"][:2]
    return sc, picked, b200


def _replay_worker(rank, world, port, path):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    doc = json.load(open(path))
    sc, jobs, b200 = _trace()
    tapes = {int(k): np.array(v) for k, v in doc["tapes"].items()}
    etapes = {int(k): np.array(v) for k, v in doc["energy"].items()}

    def run(scenario, job, catalog, seam, device):
        return C.run_job(scenario, job, catalog, "replay", tape=tapes[job.job_id],
                         energy_tape=etapes[job.job_id])

    mine = R.shard_jobs(jobs, world)[rank]
    out = R.run_shard(rank, mine, sc, b200, seam="replay", run=run)
    gathered = [None] * world
    dist.all_gather_object(gathered, out)
    if rank == 0:
        flat = [o for part in gathered for o in part]
        json.dump({"digests": {o.job_id: o.records_digest for o in flat},
                   "ranks": {o.job_id: o.rank for o in flat},
                   "agg": R.aggregate(flat, world)}, open(path + ".out", "w"))
    dist.barrier()
    dist.destroy_process_group()


def test_mixed_trace_on_device_replays_placement_independent(tmp_path):
    sc, jobs, b200 = _trace()
    assert {j.dnn_id for j in jobs} == {"mobilenet_v1", "resnet50_v1", "inception_v3"}
    results = {}
    for job in jobs:
        res = C.run_job(sc, job, b200, "device")
        assert res.error == "", (job.job_id, res.error)
        assert res.summary["power_measured"] == 1
        results[job.job_id] = res
    outcomes = R.run_shard(0, jobs, sc, b200, seam="replay",
                           run=lambda s, j, c, seam, device: C.run_job(
                               s, j, c, "replay", tape=results[j.job_id].tape,
                               energy_tape=results[j.job_id].energy_tape))
    for o in outcomes:
        dev = results[o.job_id]
        assert o.records_digest == R._digest(dev.records), o.job_id
        assert o.total_items == dev.summary["total_items"]
    agg = R.aggregate(outcomes, 1)
    print("trace: %d jobs, %.0f items, makespan %.3f s -> %.0f inferences/s" % (
        agg["jobs"], agg["items"], agg["makespan_s"], agg["inferences_per_s"]))
    assert agg["failed"] == 0 and agg["inferences_per_s"] > 0
    path = str(tmp_path / "tapes.json")
    json.dump({"tapes": {j: r.tape.tolist() for j, r in results.items()},
               "energy": {j: r.energy_tape.tolist() for j, r in results.items()}}, open(path, "w"))
    port = 29600 + os.getpid() % 1000
    mp.spawn(_replay_worker, args=(2, port, path), nprocs=2, join=True)
    got = json.load(open(path + ".out"))
    for o in outcomes:
        assert got["digests"][str(o.job_id)] == o.records_digest
    assert set(got["ranks"].values()) == {0, 1}
    assert abs(got["agg"]["items"] - agg["items"]) <= 1e-6 * agg["items"]
    assert got["agg"]["makespan_s"] < agg["makespan_s"]
