"""SM occupancy across packed jobs (north star: "SM occupancy across packed
jobs"; from the device tile log, %smid + globaltimer, bucketed
over time).  Runs C2a (300-job sweep, PACK, 20 iterations per job) and C3
(42 inference models, FAIR over 8 lanes) with SALUS_FLAG_TRACE and reports,
over the middle 80% of each run in 50 us windows: the fraction of SMs with a
tile in flight (claim .. end), the number of distinct jobs with a tile in
flight, and how evenly the SM-time is spread over the co-resident jobs.
Prints one JSON line.

usage: python tools/occupancy.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def summarize(tr, n_sm, win_ns=50_000):
    t0, t1 = int(tr["t_claim"].min()), int(tr["t_end"].max())
    lo, hi = t0 + (t1 - t0) // 10, t1 - (t1 - t0) // 10
    edges = np.arange(lo, hi, win_ns)
    busy_frac, jobs_live, top_share = [], [], []
    s, e, sm, job = tr["t_claim"].astype(np.int64), tr["t_end"].astype(np.int64), tr["smid"], tr["job"]
    for w0 in edges:
        w1 = w0 + win_ns
        m = (s < w1) & (e > w0)
        if not m.any():
            busy_frac.append(0.0)
            jobs_live.append(0)
            continue
        ov = np.minimum(e[m], w1) - np.maximum(s[m], w0)          # ns of this tile inside the window
        sm_time = np.zeros(n_sm)
        np.add.at(sm_time, sm[m], ov)
        busy_frac.append(float(np.minimum(sm_time, win_ns).sum() / (n_sm * win_ns)))
        jt = {}
        for j, o in zip(job[m].tolist(), ov.tolist()):
            jt[j] = jt.get(j, 0) + o
        jobs_live.append(len(jt))
        top_share.append(max(jt.values()) / sum(jt.values()))
    q = lambda a, p: float(np.percentile(a, p)) if len(a) else None
    return {"windows": len(edges), "window_us": win_ns / 1e3,
            "sm_busy_frac": {"mean": float(np.mean(busy_frac)), "p10": q(busy_frac, 10), "p50": q(busy_frac, 50)},
            "jobs_with_tiles_in_flight": {"mean": float(np.mean(jobs_live)), "p10": q(jobs_live, 10),
                                          "p50": q(jobs_live, 50), "p90": q(jobs_live, 90)},
            "largest_job_share_of_sm_time": {"mean": float(np.mean(top_share)) if top_share else None},
            "sms_used": int(len(np.unique(sm)))}


def main():
    from paper_1902_04610_b200 import build, salus as S
    from workloads import c2_trace, c3_trace
    build.build()
    import torch
    n_sm = torch.cuda.get_device_properties(0).multi_processor_count
    out = {}
    for name, (jobs, cap), pol, ml in (("c2a_pack", c2_trace("a", n_iters=20), S.PACK, 0),
                                       ("c3_fair8", c3_trace(), S.FAIR, 8)):
        ctx = S.Context(jobs, cap, pol, max_lanes=ml, trace=True, trace_capacity=3_000_000, log=False)
        try:
            ctx.run()
            tr = ctx.trace()
            rs = ctx.run_stats()
        finally:
            ctx.close()
        r = summarize(tr, n_sm)
        r.update({"jobs": len(jobs), "iterations": int(rs["n_dispatch"]), "tiles": int(len(tr)),
                  "kernel_ms": rs["kernel_ns"] / 1e6})
        out[name] = r
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
