"""Where C4's time goes (SRTF, real work): per job, measured iteration time
(device wall stamps) against its roofline time max(F/peak, B/BW), grouped by
width.  usage: python tools/c4_breakdown.py [c4|c5] [srtf|pack|fifo]"""
import json
import os
import sys
from collections import defaultdict

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from paper_1902_04610_b200 import build, salus as S
    from workloads import algorithmic_bytes, algorithmic_flops, c4_trace, c5_trace
    build.build()
    cfg = sys.argv[1] if len(sys.argv) > 1 else "c4"
    pol = {"srtf": S.SRTF, "pack": S.PACK, "fifo": S.FIFO}[sys.argv[2] if len(sys.argv) > 2 else "srtf"]
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    bw, tf = pk["hbm_gbs"] * 1e9, pk["bf16_tflops_sustained"] * 1e12
    jobs, cap = c4_trace() if cfg == "c4" else c5_trace()
    ctx = S.Context(jobs, cap, pol, log=True)
    try:
        ctx.run()
        w = ctx.wall()
        rs = ctx.run_stats()
        log = np.frombuffer(ctx.log_bytes(), dtype=S.LOG_DTYPE)
    finally:
        ctx.close()
    J = {j.job_id: j for j in jobs}
    meas = defaultdict(float)
    for r in w:
        meas[int(r["job"])] += (int(r["end_ns"]) - int(r["start_ns"])) / 1e9
    groups = defaultdict(lambda: [0.0, 0.0, 0])
    gb = defaultdict(lambda: [0.0, 0.0, 0])
    for jid, j in J.items():
        ideal = j.n_iters * max(algorithmic_flops(j.kind, j.dims, j.batch) / tf,
                                algorithmic_bytes(j.kind, j.dims, j.batch) / bw)
        for g in (groups[(j.dims[0], len(j.dims) - 1)], gb[(j.dims[0], j.batch)]):
            g[0] += meas[jid]
            g[1] += ideal
            g[2] += j.n_iters
    kern = rs["kernel_ns"] / 1e9
    busy = sum(meas.values())
    out = {"config": cfg, "policy": int(pol), "kernel_s": kern, "sum_iteration_s": busy, "gap_s": kern - busy,
           "mean_concurrent_iterations": busy / kern,
           "groups": {f"w{k[0]}_L{k[1]}": {"measured_s": v[0], "ideal_s": v[1], "frac": v[1] / v[0] if v[0] else None,
                                          "iters": v[2], "us_per_iter": 1e6 * v[0] / v[2]}
                      for k, v in sorted(groups.items())},
           "by_batch": {f"w{k[0]}_B{k[1]}": {"measured_s": round(v[0], 4), "frac": round(v[1] / v[0], 3) if v[0] else None,
                                             "us_per_iter": round(1e6 * v[0] / v[2], 1)}
                        for k, v in sorted(gb.items())}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
