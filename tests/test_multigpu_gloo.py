"""World-size-2 gloo test of the multi-GPU host path:
mod-G partition of the trace, one independent instance per rank, all_gather
of per-job completion records.  The per-rank schedule is computed by the
CPU oracle (no GPU here); the GPU path uses the same host functions."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import scheduler as OS
from paper_1902_04610_b200 import multigpu as MG
from workloads import c4_trace


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        jobs, cap = c4_trace(n_jobs=60, seed=9, burst=True)
        mine = MG.partition_jobs(jobs, world, rank)
        res = OS.simulate(mine, cap, OS.PACK)
        stats = {jid: {"job_id": s.job_id, "first_lane": s.first_lane, "admit_tick": s.admit_tick,
                       "first_start_tick": s.first_start_tick, "completion_tick": s.completion_tick,
                       "completion_seq": s.completion_seq} for jid, s in res.stats.items()}
        merged = MG.gather_stats(stats, rank, world)
        out[rank] = merged
    finally:
        dist.destroy_process_group()


def test_partition_is_exact_cover():
    jobs, cap = c4_trace(n_jobs=61, seed=9)
    parts = [MG.partition_jobs(jobs, 4, r) for r in range(4)]
    ids = sorted(j.job_id for p in parts for j in p)
    assert ids == sorted(j.job_id for j in jobs)
    assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


def test_gloo_world2_allgather_matches_per_partition_oracle():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
        got = [dict(out[r]) for r in range(world)]
    assert got[0] == got[1]                         # every rank holds the same merged view
    jobs, cap = c4_trace(n_jobs=60, seed=9, burst=True)
    assert sorted(got[0]) == sorted(j.job_id for j in jobs)
    for r in range(world):
        res = OS.simulate(MG.partition_jobs(jobs, world, r), cap, OS.PACK)
        for jid, s in res.stats.items():
            g = got[0][jid]
            assert g["rank"] == r
            assert (g["completion_tick"], g["completion_seq"], g["first_lane"]) == \
                (s.completion_tick, s.completion_seq, s.first_lane)
