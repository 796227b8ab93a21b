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
