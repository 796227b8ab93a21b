"""Multi-GPU plumbing: one independent Salus instance per GPU.

Jobs are independent units, so the path shards with no data-path
collective: the k-th job in (arrival, id) order goes to GPU k mod G
(`partition_jobs`; tests hold it to oracle/placement.py).  The only collective is one all_gather of fixed-size
per-GPU completion records after the run (NCCL over NVLink on the GPU box,
gloo in the CPU tests).  Host logic only — marshalling, no method arithmetic.
"""
from __future__ import annotations

import heapq
from typing import Dict, Iterable

import numpy as np

# one int64 record per job: job_id, first_lane, admit, first_start, completion,
# completion_seq, rank, and the physical end of its last iteration relative to
# its rank's kernel start (ns; -1 if the caller gave no start stamp)
REC_FIELDS = ("job_id", "first_lane", "admit_tick", "first_start_tick", "completion_tick",
              "completion_seq", "rank", "wall_end_rel_ns")


def pack_stats(stats: Dict[int, dict], rank: int, n_pad: int, t0_ns=None):
    """{job_id: stat dict} -> int64 array [n_pad, 8], padded with job_id -1."""
    out = np.full((n_pad, len(REC_FIELDS)), -1, dtype=np.int64)
    for i, jid in enumerate(sorted(stats)):
        s = stats[jid]
        rel = int(s["wall_end_ns"]) - int(t0_ns) if t0_ns is not None and "wall_end_ns" in s else -1
        out[i] = (s["job_id"], s["first_lane"], s["admit_tick"], s["first_start_tick"],
                  s["completion_tick"], np.int64(np.uint64(s["completion_seq"]).astype(np.int64)), rank, rel)
    return out


def gather_stats(stats: Dict[int, dict], rank: int, world: int, device=None, t0_ns=None) -> Dict[int, dict]:
    """All-gather every rank's per-job records; returns the merged dict.
    `t0_ns` (this rank's kernel start, globaltimer) turns each job's
    wall_end_ns into a rank-relative physical completion time."""
    import torch
    import torch.distributed as dist
    n = torch.tensor([len(stats)], dtype=torch.int64, device=device)
    if world > 1:
        dist.all_reduce(n, op=dist.ReduceOp.MAX)
    rec = torch.from_numpy(pack_stats(stats, rank, int(n.item()), t0_ns)).to(device)
    parts = [torch.empty_like(rec) for _ in range(world)]
    if world > 1:
        dist.all_gather(parts, rec)
    else:
        parts = [rec]
    merged = {}
    for row in torch.cat(parts).cpu().numpy():
        if row[0] < 0:
            continue
        merged[int(row[0])] = dict(zip(REC_FIELDS, (int(x) for x in row)))
    return merged


def partition_jobs(jobs: Iterable, world: int, rank: int, placement: str = "mod"):
    """This rank's jobs.  placement "mod": the k-th job in (arrival, id)
    order goes to GPU k mod G.  "lpt" (NEXT-4, reading A36):
    longest logical work n*c first, each to the least-loaded GPU so far
    (ties: lowest rank) -- balances heterogeneous traces such as C5, where
    mod-G leaves one GPU with far more work than the others.  Either way the
    rank's jobs are returned in (arrival, id) order."""
    jobs = list(jobs)
    if placement == "mod":
        order = sorted(jobs, key=lambda j: (j.arrival_tick, j.job_id))
        return [j for k, j in enumerate(order) if k % world == rank]
    if placement != "lpt":
        raise ValueError(f"unknown placement {placement!r}")
    heap = [(0, r) for r in range(world)]       # (work so far, rank)
    mine = []
    for j in sorted(jobs, key=lambda j: (-(j.n_iters * j.iter_ticks), j.arrival_tick, j.job_id)):
        w, r = heapq.heappop(heap)
        if r == rank:
            mine.append(j)
        heapq.heappush(heap, (w + j.n_iters * j.iter_ticks, r))
    return sorted(mine, key=lambda j: (j.arrival_tick, j.job_id))


def progress(ctx, world: int, device=None):
    """Streaming stats across GPUs (NEXT-4): jobs physically finished on all
    ranks so far, while every rank's salus_run_async is in flight -- each
    rank polls its own instance (salus_poll_stats) and one all_reduce sums
    the counts.  Collective: every rank must call it the same number of times."""
    import torch
    import torch.distributed as dist
    _, done = ctx.poll_stats()
    t = torch.tensor([done], dtype=torch.int64, device=device)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return int(t.item())
