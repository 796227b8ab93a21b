"""Per-K-chunk stamps of one F1 tile (job 0, iteration 10, task 0) from a
SALUS_DBG_CHUNKS2 build: loader issue (leader / peer), own chunk landed,
peer chunk landed (forwarder), MMA issued.  usage:
SALUS_LIB=build/libsalus_dbg2.so python tools/dbg_chunks2.py c2one|c2s"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from paper_1902_04610_b200 import salus as S
from workloads import c2_trace
name = sys.argv[1] if len(sys.argv) > 1 else "c2one"
jobs, cap = c2_trace("a", n_jobs=1, n_iters=20) if name == "c2one" else c2_trace("a", n_jobs=37, n_iters=20)
ctx = S.Context(jobs, cap, S.PACK, trace=True, trace_capacity=64)
ctx.run()
tr = ctx.trace()
ctx.close()
d = np.frombuffer(tr.tobytes(), dtype=np.uint64)[-256:].astype(np.int64)
li, pi, own, mma, peer = d[0:16], d[64:80], d[160:176], d[192:208], d[224:240]
t0 = min(li[0], pi[0])
print("chunk  lead_issue peer_issue own_land peer_land mma_issue   (us from first issue)")
for k in range(16):
    print("%5d %10.2f %10.2f %8.2f %9.2f %9.2f" % (k, (li[k] - t0) / 1e3, (pi[k] - t0) / 1e3, (own[k] - t0) / 1e3,
                                                 (peer[k] - t0) / 1e3, (mma[k] - t0) / 1e3))
