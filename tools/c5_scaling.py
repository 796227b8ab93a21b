"""C5 scaling (BASELINE configs[4]) measured on ONE
B200: the 2000-job burst trace is partitioned across G = 1, 2, 4, 8
independent Salus instances (mod-G and LPT placement, A36) and every
partition is executed, one after another, on this GPU under PACK with a
16 GiB arena.  The instances share nothing during a run (no data-path
collective), so the G-GPU makespan is the slowest partition's kernel time and
the aggregate throughput is total iterations / that time -- what a G-GPU run
measures minus the stats all_gather (tens of us).  Prints one JSON line.

usage: python tools/c5_scaling.py [--n-jobs 2000] [--gpus 1,2,4,8] [--placements mod,lpt]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-jobs", type=int, default=2000)
    ap.add_argument("--gpus", default="1,2,4,8")
    ap.add_argument("--placements", default="mod,lpt")
    args = ap.parse_args()
    from paper_1902_04610_b200 import build, multigpu as MG, salus as S
    from workloads import c5_trace
    build.build()
    jobs, cap = c5_trace(n_jobs=args.n_jobs)
    total = sum(j.n_iters for j in jobs)
    out = {"config": f"C5 burst: {len(jobs)} jobs, {total} iterations, PACK, 16 GiB per instance",
           "runs": []}
    one = None
    for G in [int(x) for x in args.gpus.split(",")]:
        for pl in args.placements.split(","):
            if G == 1 and pl != args.placements.split(",")[0]:
                continue
            ms = []
            for r in range(G):
                part = MG.partition_jobs(jobs, G, r, pl)
                ctx = S.Context(part, cap, S.PACK, device=0, log=False)
                try:
                    ctx.run()
                    rs = ctx.run_stats()
                finally:
                    ctx.close()
                assert rs["n_dispatch"] == sum(j.n_iters for j in part)
                ms.append(rs["kernel_ns"] / 1e6)
            agg = total / (max(ms) / 1e3)
            if G == 1:
                one = agg
            out["runs"].append({"gpus": G, "placement": pl, "partition_ms": ms, "makespan_ms": max(ms),
                                "aggregate_iters_per_s": agg,
                                "efficiency_vs_1": agg / (G * one) if one else None})
            print(json.dumps(out["runs"][-1]), file=sys.stderr, flush=True)
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
