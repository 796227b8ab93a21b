"""Iteration-boundary gaps on the lanes of C3 (FAIR, 8 lanes): percentiles
and the largest gaps with context (time into the run, first iteration of a
model or not).  usage: python tools/c3_gaps.py [policy] [max_lanes]"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from paper_1902_04610_b200 import salus as S
from workloads import c3_trace
pol = {"fair": S.FAIR, "pack": S.PACK}[sys.argv[1] if len(sys.argv) > 1 else "fair"]
ml = int(sys.argv[2]) if len(sys.argv) > 2 else 8
jobs, cap = c3_trace()
ctx = S.Context(jobs, cap, pol, max_lanes=ml, log=True)
ctx.run()
ctx.run()
w = ctx.wall()
rs = ctx.run_stats()
ctx.close()
w = w[np.argsort(w["seq"])]
t0 = w["start_ns"].min()
seen, last, rows = set(), {}, []
for r in w:
    ln, jb = int(r["lane"]), int(r["job"])
    first = jb not in seen
    seen.add(jb)
    if ln in last:
        p = last[ln]
        late = (int(r["append_ns"]) - int(p["end_ns"])) / 1e3          # > 0: record came after the lane idled
        qd = (int(r["start_ns"]) - max(int(r["append_ns"]), int(p["end_ns"]))) / 1e3   # publish -> first tile
        rows.append(((int(r["start_ns"]) - int(p["end_ns"])) / 1e3, (int(p["end_ns"]) - t0) / 1e3, ln,
                     int(p["job"]), jb, first, (int(r["end_ns"]) - int(r["start_ns"])) / 1e3, late, qd))
    last[ln] = r
g = np.array([x[0] for x in rows])
sw = np.array([x[0] for x in rows if x[3] != x[4]])
print(f"kernel {rs['kernel_ns'] / 1e6:.2f} ms, {rs['n_dispatch']} iterations, lanes {len(last)}, sched wait {rs['sched_wait_ns'] / 1e6:.1f} ms (fences {rs['sched_fence_ns'] / 1e6:.1f}, ring {rs['sched_ring_ns'] / 1e6:.1f})")
for name, a in (("all gaps", g), ("switches", sw)):
    print(name, len(a), "p50 %.1f p90 %.1f p95 %.1f p99 %.1f max %.1f us" % tuple(np.percentile(a, [50, 90, 95, 99, 100])))
print("largest gaps: gap_us  t_us  lane prev_job next_job first_iter next_iter_us append_after_idle_us start_after_ready_us")
for x in sorted(rows, key=lambda x: -x[0])[:25]:
    print("  %8.1f %9.1f %3d %4d %4d %5s %8.1f %8.1f %8.1f" % x)
late = np.array([x[7] for x in rows]); qd = np.array([x[8] for x in rows])
print("append after idle (us) p50 %.1f p90 %.1f p99 %.1f; start after ready p50 %.1f p90 %.1f p99 %.1f" %
      tuple(list(np.percentile(late, [50, 90, 99])) + list(np.percentile(qd, [50, 90, 99]))))
dur = np.array([x[6] for x in rows])
print("iteration duration p50 %.1f p99 %.1f us" % tuple(np.percentile(dur, [50, 99])))
