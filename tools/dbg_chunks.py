"""Per-K-chunk timing of GEMM tiles (variant build with SALUS_DBG_CHUNKS):
t_ready = loader issued chunk 0, t_mma = loader issued the last chunk,
t_end = MMA thread saw the last chunk land in both CTAs.
usage: SALUS_LIB=build/libsalus_dbg.so python tools/dbg_chunks.py c2one|c2s"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from paper_1902_04610_b200 import salus as S
from workloads import c2_trace
name = sys.argv[1]
jobs, cap = c2_trace("a", n_jobs=1, n_iters=20) if name == "c2one" else c2_trace("a", n_jobs=37, n_iters=10)
ctx = S.Context(jobs, cap, S.PACK, trace=True)
for rep in range(2):
    ctx.run()
tr = ctx.trace()
stage = (tr["task"] >> 21) & 31
for s in sorted(set(stage.tolist())):
    m = (stage == s) & (tr["t_ready"] > 0) & (tr["t_end"] > tr["t_ready"])
    if not m.any():
        continue
    issue = (tr["t_mma"][m] - tr["t_ready"][m]) / 1e3
    land = (tr["t_end"][m] - tr["t_mma"][m]) / 1e3
    first = (tr["t_ready"][m] - tr["t_claim"][m]) / 1e3
    print(f"stage {s}: n={m.sum()} claim->chunk0 issue {np.median(first):6.2f}  issue span {np.median(issue):6.2f}  last issue->landed {np.median(land):6.2f} us")
