"""ORACLE — test infrastructure only.  The progressive-allocation deadlock of
PAPER.md §3.3 (`fig:deadlock`) and why lanes avoid it
(optional oracle-only demo).

"A job can start its iteration as long as its model memory is available,
and then the ephemeral memory is allocated gradually by a series of GPU
kernels ... 12 GB GPU memory capacity ... P_A = P_B = 1 GB and E_A = E_B =
7 GB ... if both jobs attempt to allocate their remaining requirements as
follows: (E_A += 3 GB) and (E_B += 3 GB), neither will be able to proceed,
causing a deadlock!".

`progressive(C, steps)` replays allocation requests in the given
interleaving; a request that does not fit blocks its job (its later steps
wait), and the replay reports a deadlock when every unfinished job is
blocked.  `with_lanes(C, jobs)` is Salus's answer: a job's iteration starts
only inside a lane whose size already covers its whole E (Algorithm 1 +
the safety condition), so its ephemeral allocations never wait
on another job; iterations sharing a lane are serialised.  Sizes are
integers (GB in the paper's example).
"""
from __future__ import annotations

from typing import Dict, List, Sequence, Tuple


def progressive(C: int, steps: Sequence[Tuple[str, str, int]]):
    """steps: (job, 'P'|'E', amount) in issue order.  A job's steps run in
    order; a blocked step is retried whenever memory is freed (never, here:
    memory is only freed when an iteration completes, i.e. after its last
    step).  Returns ('done', used) or ('deadlock', {job: pending step})."""
    used = 0
    per_job: Dict[str, List[Tuple[str, int]]] = {}
    for job, kind, amt in steps:
        per_job.setdefault(job, []).append((kind, amt))
    order = [job for job, _, _ in steps]
    pos = {j: 0 for j in per_job}
    held = {j: 0 for j in per_job}
    pending = list(order)
    blocked = set()
    while pending:
        progressed = False
        for i, job in enumerate(pending):
            if job in blocked:
                continue
            kind, amt = per_job[job][pos[job]]
            if used + amt <= C:
                used += amt
                held[job] += amt
                pos[job] += 1
                pending.pop(i)
                if pos[job] == len(per_job[job]):     # iteration complete: ephemeral freed
                    used -= held[job]
                    held[job] = 0
                    blocked.clear()
                progressed = True
                break
            blocked.add(job)
        if not progressed:
            return "deadlock", {j: per_job[j][pos[j]] for j in per_job if pos[j] < len(per_job[j])}
    return "done", used


def with_lanes(C: int, jobs: Sequence[Tuple[str, int, int]]):
    """jobs: (name, P, E).  Admit in order with FindLane under the safety
    condition sum P + sum L <= C (one lane of size max E if every job fits
    beside the others, else a job waits for admission), then run each lane's
    iterations one at a time: an iteration's ephemeral allocations are inside
    its lane and always succeed.  Returns ('done', admitted order, lanes)."""
    sumP, lanes, admitted, waiting = 0, [], [], []
    for name, P, E in jobs:
        S = sumP + sum(L for L, _ in lanes)
        if S + P + E <= C:
            lanes.append([E, [name]])
        else:
            fit = [ln for ln in lanes if ln[0] >= E and S + P <= C]
            if fit:
                min(fit, key=lambda ln: ln[0])[1].append(name)
            else:
                waiting.append(name)
                continue
        sumP += P
        admitted.append(name)
    assert sumP + sum(L for L, _ in lanes) <= C
    return "done", admitted, [list(r) for _, r in lanes], waiting
