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


# --------------------------------------------------------------------------
# Automatic migration at drain time (NEXT-4, reading A39 of DESIGN.md)
# --------------------------------------------------------------------------

def device_schedule(jobs, cap, policy, device=0, **kw):
    """The logical schedule of one instance as this package's own device
    scheduler computes it (a schedule-only run, SALUS_FLAG_NULL_WORK):
    ({job_id: sorted dispatch ticks}, makespan in ticks)."""
    from . import salus as S
    ctx = S.Context(jobs, cap, policy, device=device, null_work=True, log=True, **kw)
    try:
        stats = ctx.run()
        log = np.frombuffer(ctx.log_bytes(), dtype=S.LOG_DTYPE)
    finally:
        ctx.close()
    disp = log[log["kind"] == 1]                          # DISPATCH records
    ticks: Dict[int, list] = {}
    for jid, t in zip(disp["job"].tolist(), disp["tick"].tolist()):
        ticks.setdefault(int(jid), []).append(int(t))
    makespan = max((int(s["completion_tick"]) for s in stats.values()), default=0)
    return ticks, makespan


def plan_rebalance(parts, schedule, max_moves: int = 4, tol: float = 0.05):
    """Drain-time migration planner over G independent instances.

    parts: per rank, its jobs (workloads.Job-like: job_id, n_iters,
    iter_ticks, arrival_tick).  schedule(rank, jobs) -> ({job_id: dispatch
    ticks}, makespan): the rank's logical schedule.  Repeatedly, while the
    busiest rank m's makespan exceeds the first-draining rank d's by more
    than tol x makespan[m]: at T = makespan[d], the job on m with the most
    remaining logical work (n - k) * c, k = its iterations completed by T
    (dispatch + c <= T), leaves m at that iteration boundary -- m keeps its
    first k iterations, d runs the other n - k, arriving at T, resumed from
    m's state image (A37).  A rank is never both a source and a target.
    Returns (moves [(job_id, src, dst, k, T)], new parts, makespans)."""
    import dataclasses
    parts = [list(p) for p in parts]
    scheds = [schedule(r, p) for r, p in enumerate(parts)]
    moves, srcs, dsts = [], set(), set()
    for _ in range(max_moves):
        ms = [s[1] for s in scheds]
        d = min(range(len(ms)), key=lambda r: (ms[r], r))
        m = max(range(len(ms)), key=lambda r: (ms[r], -r))
        if d == m or d in srcs or m in dsts or ms[m] - ms[d] <= tol * ms[m]:
            break
        T = ms[d]
        best = None
        for j in parts[m]:
            ticks = scheds[m][0].get(j.job_id, [])
            k = sum(1 for t in ticks if t + j.iter_ticks <= T)
            rem = (j.n_iters - k) * j.iter_ticks
            if k < j.n_iters and (best is None or (rem, -j.job_id) > (best[0], -best[1].job_id)):
                best = (rem, j, k)
        if best is None:
            break
        rem, j, k = best
        keep = [x for x in parts[m] if x.job_id != j.job_id]
        if k > 0:
            keep.append(dataclasses.replace(j, n_iters=k))
        new_m = sorted(keep, key=lambda x: (x.arrival_tick, x.job_id))
        new_d = sorted(parts[d] + [dataclasses.replace(j, n_iters=j.n_iters - k, arrival_tick=max(T, j.arrival_tick))],
                       key=lambda x: (x.arrival_tick, x.job_id))
        sm, sd = schedule(m, new_m), schedule(d, new_d)
        if max(sm[1], sd[1]) >= ms[m]:                 # a job's iterations are sequential: moving the
            break                                      # tail only pays if m has other work behind it
        parts[m], parts[d], scheds[m], scheds[d] = new_m, new_d, sm, sd
        moves.append((j.job_id, m, d, k, T))
        srcs.add(m)
        dsts.add(d)
    return moves, parts, [s[1] for s in scheds]


def plan_rebalance_dist(my_jobs, rank: int, world: int, schedule, max_moves: int = 4, tol: float = 0.05):
    """plan_rebalance run by every rank on its own partition, with
    collectives instead of a central planner: per step one all_gather of
    the makespans (all ranks then agree on m, d and T), the source m alone
    computes its candidate and broadcasts it, every rank applies the move to
    its own partition and m and d re-schedule.  schedule(jobs) -> (ticks,
    makespan) of this rank.  Returns (moves, my new jobs, makespans)."""
    import dataclasses
    import torch.distributed as dist
    mine = sorted(my_jobs, key=lambda x: (x.arrival_tick, x.job_id))
    sched = schedule(mine)
    moves, srcs, dsts = [], set(), set()
    while True:
        ms = [None] * world
        if world > 1:
            dist.all_gather_object(ms, sched[1])
        else:
            ms = [sched[1]]
        if len(moves) >= max_moves:
            break
        d = min(range(world), key=lambda r: (ms[r], r))
        m = max(range(world), key=lambda r: (ms[r], -r))
        if d == m or d in srcs or m in dsts or ms[m] - ms[d] <= tol * ms[m]:
            break
        T = ms[d]
        cand = [None]
        if rank == m:
            best = None
            for j in mine:
                k = sum(1 for t in sched[0].get(j.job_id, []) if t + j.iter_ticks <= T)
                rem = (j.n_iters - k) * j.iter_ticks
                if k < j.n_iters and (best is None or (rem, -j.job_id) > (best[0], -best[1].job_id)):
                    best = (rem, j, k)
            cand = [None if best is None else (best[1], best[2])]
        if world > 1:
            dist.broadcast_object_list(cand, src=m)
        if cand[0] is None:
            break
        j, k = cand[0]
        trial = mine
        if rank == m:
            trial = [x for x in mine if x.job_id != j.job_id] + ([dataclasses.replace(j, n_iters=k)] if k else [])
        if rank == d:
            trial = mine + [dataclasses.replace(j, n_iters=j.n_iters - k, arrival_tick=max(T, j.arrival_tick))]
        trial = sorted(trial, key=lambda x: (x.arrival_tick, x.job_id))
        tsched = schedule(trial) if rank in (m, d) else sched
        # accepted only if it lowers the busier of the two (all ranks agree)
        tm = [None] * world
        if world > 1:
            dist.all_gather_object(tm, tsched[1])
        else:
            tm = [tsched[1]]
        if max(tm[m], tm[d]) >= ms[m]:
            break
        mine, sched = trial, tsched
        moves.append((j.job_id, m, d, k, T))
        srcs.add(m)
        dsts.add(d)
    return moves, mine, ms


# --------------------------------------------------------------------------
# Request-rate autoscaling of inference models (NEXT-4; reading A40)
# --------------------------------------------------------------------------

def request_rates(arrivals, t_end: float, window: float):
    """{model: requests per second} over the window (t_end - window, t_end]
    of each model's arrival times (seconds)."""
    return {m: sum(1 for t in ts if t_end - window < t <= t_end) / window for m, ts in arrivals.items()}


def autoscale(rates, service_s, util_target: float = 0.5, max_gpus: int = 8):
    """How many GPUs the inference models need and where each runs.

    A model's load is rate x per-request service time (GPU-seconds per
    second); the fleet gets G = ceil(total load / util_target) GPUs
    (1..max_gpus) -- consolidation when requests are slow, scale-out when
    they are not -- and a model whose own load exceeds util_target gets
    ceil(load / util_target) replicas (<= G) sharing its requests equally.
    Replicas are placed longest first on the least-loaded GPU that does not
    yet hold the model (ties: lowest GPU).  Returns (G, {model: [gpus]},
    per-GPU load)."""
    import math
    load = {m: rates[m] * service_s[m] for m in rates}
    total = sum(load.values())
    G = min(max_gpus, max(1, math.ceil(total / util_target - 1e-12)))
    items = []
    for m in sorted(load):
        rep = min(G, max(1, math.ceil(load[m] / util_target - 1e-12)))
        items += [(load[m] / rep, m, i) for i in range(rep)]
    items.sort(key=lambda x: (-x[0], x[1], x[2]))
    gpu_load = [0.0] * G
    place = {m: [] for m in load}
    for w, m, _ in items:
        free = [g for g in range(G) if g not in place[m]] or list(range(G))
        g = min(free, key=lambda x: (gpu_load[x], x))
        place[m].append(g)
        gpu_load[g] += w
    return G, place, gpu_load
