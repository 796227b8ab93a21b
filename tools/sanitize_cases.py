"""Small real-work cases for compute-sanitizer runs (SALUS_COOP=0):
C1 under FIFO and SRTF, a ragged tiny training + inference pair, and a
12-model slice of C3 under FAIR, and (NEXT-3) the eviction hand trace HW-EV
with real work, whose swap records copy pages to pinned host memory and back.
usage: python tools/sanitize_cases.py"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_1902_04610_b200 import salus as S
from workloads import c1_trace, c3_trace, make_job, TRAIN, INFER
cases = [("c1 fifo", c1_trace(), S.FIFO, 0), ("c1 srtf", c1_trace(), S.SRTF, 0)]
jobs = [make_job(0, TRAIN, 0, (200, 256, 72), 300, 2, lr=1e-2, seed=3),
        make_job(1, INFER, 0, (384, 128, 256, 128), 7, 2, seed=4, request_ticks=(0, 5))]
cases.append(("ragged", (jobs, 1 << 30), S.PACK, 0))
c3, cap = c3_trace()
cases.append(("c3 slice fair", ([j for j in c3 if j.job_id % 4 == 0][:12], cap), S.FAIR, 4))
G = 1 << 16
ev = [make_job(0, TRAIN, 0, (128, 256, 128), 128, 4, iter_ticks=100, persistent_bytes=8 * G,
               ephemeral_bytes=6 * G, lr=1e-2, seed=11),
      make_job(1, TRAIN, 150, (128, 256, 128), 128, 1, iter_ticks=100, persistent_bytes=8 * G,
               ephemeral_bytes=6 * G, lr=1e-2, seed=12)]
cases.append(("evict hw-ev", (ev, 20 * G), S.SRTF, 0))
for name, (jobs, cap), pol, ml in cases:
    ctx = S.Context(jobs, cap, pol, max_lanes=ml, evict=name.startswith("evict"))
    ctx.run()
    rs = ctx.run_stats()
    ctx.close()
    print(f"{name}: status {rs['status']}, {rs['n_dispatch']} iterations, {rs['n_tasks']} tiles, "
          f"swaps {rs['n_swap_out']}/{rs['n_swap_in']}")
