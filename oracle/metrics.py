"""ORACLE — test infrastructure only.  Aggregate statistics of `tab:exp11`
(PAPER.md P:545-563): makespan, average queuing, average JCT, 95% JCT.

  JCT_i     = completion_i - arrival_i
  queuing_i = first_start_i - arrival_i
  makespan  = max completion - min arrival
  p-th percentile: nearest rank on the sorted values (A23):
                   the ceil(p/100 * n)-th smallest.
"""
import math


def nearest_rank(values, pct: float):
    v = sorted(values)
    if not v:
        raise ValueError("empty")
    r = max(1, math.ceil(pct / 100.0 * len(v)))
    return v[r - 1]


def summarize(jobs, stats):
    """stats: {job_id: JobStat-like with first_start_tick, completion_tick}."""
    arr = {j.job_id: j.arrival_tick for j in jobs}
    jct = [stats[i].completion_tick - arr[i] for i in arr]
    que = [stats[i].first_start_tick - arr[i] for i in arr]
    return {
        "makespan": max(stats[i].completion_tick for i in arr) - min(arr.values()),
        "avg_queuing": sum(que) / len(que),
        "avg_jct": sum(jct) / len(jct),
        "p95_jct": nearest_rank(jct, 95),
        "n_jobs": len(jct),
    }


def jct_cdf(jcts):
    """Right-continuous step CDF [(x, F(x))] at the distinct values."""
    v = sorted(jcts)
    n = len(v)
    out = []
    for i, x in enumerate(v):
        if i + 1 == n or v[i + 1] != x:
            out.append((x, (i + 1) / n))
    return out
