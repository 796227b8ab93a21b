"""NEXT-4 request-rate autoscaling (A40) on C3, one B200.

1. Calibration: the 42 models under FAIR/8 with live Poisson requests at 20
   per model per second; per-request service time of each model = median
   device time of its requests (first tile start -> last tile end).
2. A day profile of per-model rates; for each phase the controller measures
   the rates of the phase's requests (multigpu.request_rates) and
   multigpu.autoscale picks the number of GPUs and places the models.
3. Measured: the busiest GPU's share of that phase (its models; a replicated
   model's requests split round-robin) served live on this B200, against
   all 42 models on the one GPU without autoscaling.

usage: python tools/c3_autoscale.py [util_target]"""
import dataclasses
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

from paper_1902_04610_b200 import build, multigpu as MG, salus as S  # noqa: E402
from workloads import c3_trace  # noqa: E402


def poisson(rng, rate, dur):
    t = np.cumsum(rng.exponential(1.0 / rate, size=int(rate * dur * 3) + 8)) if rate > 0 else np.array([])
    return t[t < dur]


def serve(models, cap, arrivals, dur):
    """Live run of `models` with arrivals {job_id: times}; request latency stats."""
    jobs = [dataclasses.replace(j, n_iters=max(1, len(arrivals[j.job_id])), request_ticks=()) for j in models]
    due = sorted((float(t), j.job_id) for j in jobs for t in (arrivals[j.job_id] if len(arrivals[j.job_id])
                                                                else [dur / 2]))
    ctx = S.Context(jobs, cap, S.FAIR, max_lanes=8, log=True, online=True)
    try:
        ctx.run_async()
        ctx.serve(due)
        ctx.end_submissions()
        ctx.wait()
        w = ctx.wall()
        seen = {j.job_id: ctx.requests(j.job_id)[1].astype(np.int64) for j in jobs}
    finally:
        ctx.close()
    w = w[np.argsort(w["seq"])]
    k, lat, svc = {}, [], {}
    for r in w:
        jid = int(r["job"])
        i = k.get(jid, 0)
        k[jid] = i + 1
        lat.append((int(r["end_ns"]) - int(seen[jid][i])) / 1e3)
        svc.setdefault(jid, []).append((int(r["end_ns"]) - int(r["start_ns"])) / 1e9)
    return {"requests": len(due), "offered_rps": len(due) / dur,
            "latency_us_p50": float(np.percentile(lat, 50)), "latency_us_p99": float(np.percentile(lat, 99))}, svc


def main():
    build.build()
    util = float(sys.argv[1]) if len(sys.argv) > 1 else 0.5
    models, cap = c3_trace()
    rng = np.random.default_rng(3)
    dur = 0.4
    cal = {j.job_id: poisson(rng, 20, 1.0) for j in models}
    _, svc = serve(models, cap, cal, 1.0)
    service = {jid: float(np.median(v)) for jid, v in svc.items()}
    out = {"util_target": util, "service_us": {k: v * 1e6 for k, v in service.items()}, "phases": []}
    for lam in (20, 200, 2000, 5000):
        arr = {j.job_id: poisson(rng, lam, dur) for j in models}
        rates = MG.request_rates(arr, dur, dur)
        G, place, load = MG.autoscale(rates, service, util, 8)
        g0 = max(range(G), key=lambda g: load[g])
        share, share_arr = [], {}
        for j in models:
            if g0 in place[j.job_id]:
                reps = place[j.job_id]
                i = reps.index(g0)
                share.append(j)
                share_arr[j.job_id] = arr[j.job_id][i::len(reps)]
        one, _ = serve(models, cap, arr, dur)
        busiest, _ = serve(share, cap, share_arr, dur)
        ph = {"lambda_per_model": lam, "gpus": G, "gpu_load": load, "busiest_gpu_models": len(share),
              "all_on_one_gpu": one, "busiest_gpu_after_autoscale": busiest}
        out["phases"].append(ph)
        print(json.dumps(ph), flush=True)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
