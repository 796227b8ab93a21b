"""NEXT-4 drain-time migration (A39) on C5, measured on one B200
with G instances run one after another: logical makespans per instance
before and after the plan (from the device's own schedule-only runs), and
the physical kernel time of every instance's real-work run (migrated jobs:
the source runs the first k iterations with SALUS_DUMP_STATE, the target
resumes the image).  Aggregate iters/s = all iterations / the slowest
instance, as if the G instances ran side by side on G GPUs.

usage: python tools/c5_rebalance.py [G ...]   (default 4 8)"""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

from paper_1902_04610_b200 import build, multigpu as MG, salus as S  # noqa: E402
from workloads import c5_trace  # noqa: E402


def run_parts(parts, cap, moves):
    """Real-work runs of every instance; sources first (their images feed the targets)."""
    srcs = {m[1] for m in moves}
    order = sorted(range(len(parts)), key=lambda r: (r not in srcs, r))
    imgs, times = {}, [0.0] * len(parts)
    moved = {m[0]: m for m in moves}
    for r in order:
        dump, resume = {}, {}
        for j in parts[r]:
            if j.job_id in moved:
                jid, src, dst, k, T = moved[j.job_id]
                if r == src:
                    dump[jid] = S.DUMP_STATE
                elif r == dst and k:
                    resume[jid] = (imgs[jid], k)
        ctx = S.Context(parts[r], cap, S.PACK, dump=dump, resume=resume, log=False)
        try:
            ctx.run()
            times[r] = ctx.run_stats()["kernel_ns"] / 1e9
            for jid in dump:
                imgs[jid] = ctx.read_state(jid)
        finally:
            ctx.close()
    return times


def main():
    build.build()
    jobs, cap = c5_trace()
    total = sum(j.n_iters for j in jobs)
    out = {}
    for G in [int(x) for x in sys.argv[1:]] or [4, 8]:
        parts = [MG.partition_jobs(jobs, G, r) for r in range(G)]
        before = [MG.device_schedule(p, cap, S.PACK)[1] for p in parts]
        moves, new, after = MG.plan_rebalance(parts, lambda r, p: MG.device_schedule(p, cap, S.PACK))
        t0 = run_parts(parts, cap, [])
        t1 = run_parts(new, cap, moves)
        out[G] = {"moves": moves, "logical_makespan_before": before, "logical_makespan_after": after,
                  "kernel_s_before": t0, "kernel_s_after": t1,
                  "iters_per_s_before": total / max(t0), "iters_per_s_after": total / max(t1)}
        print(json.dumps({G: out[G]}), flush=True)


if __name__ == "__main__":
    main()
