"""Scheduler time per phase (SALUS_DBG_SCHED build): next_event,
completions, arrivals, admission, dispatch (incl. append), append.
usage: SALUS_LIB=build/libsalus_dbgs.so python tools/sched_phases.py c3|c2 [policy] [null]"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from paper_1902_04610_b200 import salus as S
from workloads import c2_trace, c3_trace
name = sys.argv[1] if len(sys.argv) > 1 else "c3"
pol = {"fair": S.FAIR, "pack": S.PACK}[sys.argv[2] if len(sys.argv) > 2 else "fair"]
null = len(sys.argv) > 3 and sys.argv[3] == "null"
jobs, cap = c3_trace() if name == "c3" else c2_trace("a")
ctx = S.Context(jobs, cap, pol, max_lanes=8 if (name == "c3" and pol == S.FAIR) else 0, trace=True,
                trace_capacity=64, null_work=null)
ctx.run()
rs = ctx.run_stats()
tr = ctx.trace()
ctx.close()
d = np.frombuffer(tr.tobytes(), dtype=np.uint64)[-8:].astype(np.float64) / 1e6
names = ["next_event", "completions", "arrivals", "admission", "dispatch", "  of which append"]
print(f"{name} {sys.argv[2] if len(sys.argv) > 2 else 'fair'} null={null}: kernel {rs['kernel_ns'] / 1e6:.1f} ms, "
      f"{rs['n_dispatch']} dispatches, {rs['n_ticks']} ticks, sched wait {rs['sched_wait_ns'] / 1e6:.1f} ms")
for n, v in zip(names, list(d[:5]) + [d[6]]):
    print(f"  {n:18s} {v:8.2f} ms  {v * 1e3 / max(1, rs['n_dispatch']):6.2f} us/dispatch")
