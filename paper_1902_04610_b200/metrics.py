"""Job-level statistics of a run, computed from the device's per-job records
(salus_job_stat), for the bench and callers -- the quantities of the paper's
`tab:exp11`: makespan, average queuing, average JCT,
95% JCT, plus physical JCT from the device's globaltimer stamps.

  JCT_i     = completion_i - arrival_i           (logical ticks, A17)
  queuing_i = first_start_i - arrival_i
  makespan  = max completion - min arrival
  p95       = nearest rank: the ceil(0.95 n)-th smallest (A23)

Host bookkeeping over the product's own outputs; independent of oracle/.
"""
from __future__ import annotations

import math
from typing import Dict, Iterable


def nearest_rank(values, pct: float):
    v = sorted(values)
    if not v:
        raise ValueError("empty")
    return v[max(1, math.ceil(pct / 100.0 * len(v))) - 1]


def summarize(jobs: Iterable, stats: Dict[int, dict]) -> dict:
    """Logical-tick summary of a finished run; `stats` = {job_id: record}."""
    arr = {j.job_id: j.arrival_tick for j in jobs}
    jct = [stats[i]["completion_tick"] - a for i, a in arr.items()]
    que = [stats[i]["first_start_tick"] - a for i, a in arr.items()]
    return {"n_jobs": len(jct),
            "avg_jct_ticks": sum(jct) / len(jct),
            "p95_jct_ticks": nearest_rank(jct, 95),
            "avg_queuing_ticks": sum(que) / len(que),
            "makespan_ticks": max(stats[i]["completion_tick"] for i in arr) - min(arr.values())}


def physical(stats: Dict[int, dict], t0_ns: int) -> dict:
    """Physical JCT from the device stamps of jobs that all arrived at the
    kernel start t0_ns (burst traces): last tile end - t0."""
    jct = [(s["wall_end_ns"] - t0_ns) / 1e6 for s in stats.values()]
    return {"avg_jct_ms": sum(jct) / len(jct), "p95_jct_ms": nearest_rank(jct, 95),
            "makespan_ms": max(jct)}
