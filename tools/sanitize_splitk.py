"""Small split-K runs for compute-sanitizer (memcheck / racecheck) on the
opt-in build: one lone wide job (narrow records, split F / dX stages) and a
6-job C4 slice under PACK (two narrow lanes).
usage: SALUS_LIB=<split build> SALUS_SPLITK=1 compute-sanitizer ... python tools/sanitize_splitk.py"""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_04610_b200 import salus as S  # noqa: E402
from workloads import TRAIN, c4_trace, footprint_bytes, make_job  # noqa: E402

dims, b = (2048, 2048, 2048, 512), 128
e = footprint_bytes(TRAIN, dims, b)[1] + (64 << 20)
runs = [([make_job(0, TRAIN, 0, dims, b, 2, ephemeral_bytes=e, seed=3)], 1 << 34, S.FIFO)]
jobs, cap = c4_trace(n_jobs=24)
sub = [dataclasses.replace(j, n_iters=min(j.n_iters, 3)) for j in jobs if j.job_id in (0, 11, 12, 13)]
runs.append((sub, cap, S.PACK))
for jobs_, cap_, pol in runs:
    ctx = S.Context(jobs_, cap_, pol, timeout_ms=600000)
    try:
        ctx.run()
        print("ok", len(jobs_), "jobs", ctx.run_stats()["n_tasks"], "tasks", flush=True)
    finally:
        ctx.close()
