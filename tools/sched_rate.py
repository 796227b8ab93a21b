"""Scheduler-only rate: NULL_WORK runs (no tiles execute) of C2a and C3.
usage: python tools/sched_rate.py"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1902_04610_b200 import salus as S
from workloads import c2_trace, c3_trace
for name, (jobs, cap), pol, ml in (("c2a pack", c2_trace("a"), S.PACK, 0), ("c3 fair8", c3_trace(), S.FAIR, 8),
                                   ("c3 pack", c3_trace(), S.PACK, 0)):
    for log in (False, True):
        ctx = S.Context(jobs, cap, pol, max_lanes=ml, null_work=True, log=log)
        ctx.run(); ctx.run()
        rs = ctx.run_stats()
        ctx.close()
        print(f"{name} log={log}: {rs['n_dispatch']} dispatches, {rs['n_ticks']} ticks, kernel {rs['kernel_ns'] / 1e6:.2f} ms, "
              f"{rs['kernel_ns'] / 1e3 / rs['n_dispatch']:.2f} us/dispatch, {rs['kernel_ns'] / 1e3 / rs['n_ticks']:.2f} us/tick")
