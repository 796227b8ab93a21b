"""ORACLE — test infrastructure only.  Placement of a trace's jobs on G
independent Salus instances (one per GPU), SURVEY §8(e) and §8(f) NEXT-4.

The paper leaves multi-GPU placement as future work ("...extend
Salus to multiple GPUs..."); the north star fixes one independent instance
per GPU with jobs partitioned across them.  Two rules, written out plainly:

* mod:  the k-th job in (arrival, id) order goes to GPU k mod G (§8(e)).
* lpt:  Graham's longest-processing-time-first list scheduling over each
        job's logical work w_j = n_j * c_j (A17's iteration cost, the same
        quantity SRTF ranks by): visit jobs by (-w, arrival, id) and
        give each to the GPU with the least work so far (ties: lowest rank).
        Reading A36 of DESIGN.md.

Both return, per GPU, its jobs in (arrival, id) order.
"""
from __future__ import annotations

from typing import List, Sequence


def place_mod(jobs: Sequence, G: int) -> List[list]:
    order = sorted(jobs, key=lambda j: (j.arrival_tick, j.job_id))
    parts = [[] for _ in range(G)]
    for k, j in enumerate(order):
        parts[k % G].append(j)
    return parts


def place_lpt(jobs: Sequence, G: int) -> List[list]:
    order = sorted(jobs, key=lambda j: (-j.n_iters * j.iter_ticks, j.arrival_tick, j.job_id))
    load = [0] * G
    parts = [[] for _ in range(G)]
    for j in order:
        g = min(range(G), key=lambda r: (load[r], r))
        parts[g].append(j)
        load[g] += j.n_iters * j.iter_ticks
    return [sorted(p, key=lambda j: (j.arrival_tick, j.job_id)) for p in parts]


def loads(parts) -> List[int]:
    return [sum(j.n_iters * j.iter_ticks for j in p) for p in parts]


def rebalance(parts, cap, policy, max_moves=4, tol=0.05):
    """Drain-time migration (reading A39), written out with the
    oracle's own schedule simulation: while the busiest GPU m finishes more
    than tol x its makespan after the first GPU d to drain, at T = d's
    makespan move the rest of m's job with the most remaining logical work
    (n - k) * c -- k = its iterations finished by T -- to d, arriving at T;
    m keeps the first k.  The move is made only if afterwards both m and d
    finish before m did; no GPU is both a source and a target.
    Returns (moves [(job_id, src, dst, k, T)], makespans)."""
    import dataclasses
    from . import scheduler as OS
    parts = [list(p) for p in parts]

    def run(p):
        r = OS.simulate(p, cap, policy)
        ticks = {}
        for rec in r.dispatch:                      # (seq, tick, lane, job, iter, busy_until)
            ticks.setdefault(rec[3], []).append(rec[1])
        return ticks, max([s.completion_tick for s in r.stats.values()] + [0])

    res = [run(p) for p in parts]
    moves, srcs, dsts = [], [], []
    while len(moves) < max_moves:
        ms = [x[1] for x in res]
        d = ms.index(min(ms))                       # first (lowest) rank with the least
        m = ms.index(max(ms))                       # first (lowest) rank with the most
        if d == m or d in srcs or m in dsts or ms[m] - ms[d] <= tol * ms[m]:
            break
        T = ms[d]
        pick = None
        for j in sorted(parts[m], key=lambda x: x.job_id):
            k = 0
            for t in res[m][0].get(j.job_id, []):
                if t + j.iter_ticks <= T:
                    k += 1
            if k == j.n_iters:
                continue
            rem = (j.n_iters - k) * j.iter_ticks
            if pick is None or rem > pick[0]:
                pick = (rem, j, k)
        if pick is None:
            break
        _, j, k = pick
        rest = [x for x in parts[m] if x.job_id != j.job_id]
        if k > 0:
            rest.append(dataclasses.replace(j, n_iters=k))
        rest = sorted(rest, key=lambda x: (x.arrival_tick, x.job_id))
        moved = dataclasses.replace(j, n_iters=j.n_iters - k, arrival_tick=max(T, j.arrival_tick))
        more = sorted(parts[d] + [moved], key=lambda x: (x.arrival_tick, x.job_id))
        rm, rd = run(rest), run(more)
        if max(rm[1], rd[1]) >= ms[m]:              # no gain for the busier of the two: stop
            break
        parts[m], parts[d], res[m], res[d] = rest, more, rm, rd
        moves.append((j.job_id, m, d, k, T))
        srcs.append(m)
        dsts.append(d)
    return moves, [x[1] for x in res]


def autoscale(rates, service_s, util_target=0.5, max_gpus=8):
    """Request-rate autoscaling (reading A40), written out:
    load_m = rate_m * service_m; G = ceil(sum load / util_target) clamped to
    [1, max_gpus]; model m gets ceil(load_m / util_target) replicas (at
    least 1, at most G) of load load_m / replicas each; replicas visited by
    (-load, model, replica index), each to the GPU with the least load among
    those not holding the model yet (all GPUs if every one does), ties to
    the lowest GPU.  Returns (G, {model: [gpu per replica]}, per-GPU load)."""
    import math
    load = {}
    for m in rates:
        load[m] = rates[m] * service_s[m]
    total = 0.0
    for m in load:
        total += load[m]
    G = math.ceil(total / util_target - 1e-12)
    G = max(1, min(max_gpus, G))
    reps = []
    for m in sorted(load):
        r = math.ceil(load[m] / util_target - 1e-12)
        r = max(1, min(G, r))
        for i in range(r):
            reps.append((-(load[m] / r), m, i))
    reps.sort()
    per_gpu = [0.0] * G
    where = {}
    for m in load:
        where[m] = []
    for neg, m, i in reps:
        best = None
        for g in range(G):
            if g in where[m] and len(where[m]) < G:
                continue
            if best is None or per_gpu[g] < per_gpu[best]:
                best = g
        where[m].append(best)
        per_gpu[best] += -neg
    return G, where, per_gpu
