"""Run one config once through the C ABI (used under ncu / for quick timing).

usage: python tools/run_cfg.py c1|c2|c2s|c3|c4 [policy] [reps]
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))

import numpy as np  # noqa: E402

from paper_1902_04610_b200 import build, salus as S  # noqa: E402
from workloads import c1_trace, c2_trace, c3_trace, c4_trace  # noqa: E402

POL = {"fifo": S.FIFO, "srtf": S.SRTF, "pack": S.PACK, "fair": S.FAIR}


def main():
    name = sys.argv[1]
    pol = POL[sys.argv[2]] if len(sys.argv) > 2 else S.PACK
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    build.build()
    if name == "c1":
        jobs, cap = c1_trace()
    elif name == "c2":
        jobs, cap = c2_trace("a")
    elif name == "c2s":
        jobs, cap = c2_trace("a", n_jobs=37, n_iters=10)
    elif name == "c3":
        jobs, cap = c3_trace()
    else:
        jobs, cap = c4_trace()
    ctx = S.Context(jobs, cap, pol, max_lanes=8 if (name == "c3" and pol == S.FAIR) else 0)
    for r in range(reps):
        ctx.run()
        rs = ctx.run_stats()
        w = ctx.wall()
        dur = (w["end_ns"] - w["start_ns"]) / 1e3
        print(f"{name} rep {r}: kernel {rs['kernel_ns'] / 1e6:.3f} ms, {rs['n_dispatch']} iters, "
              f"{rs['n_dispatch'] / (rs['kernel_ns'] / 1e9):.0f} iters/s, iter us p50 {np.median(dur):.1f}, "
              f"tasks {rs['n_tasks']}, sched_wait {rs['sched_wait_ns'] / 1e6:.3f} ms", flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
