"""Per-stage timeline of one config from the device tile trace.
usage: python tools/trace_stages.py c1|c2s|c2one|job:W:L:B [policy]
(job:W:L:B = one training job of width W, depth L, batch B, 10 iterations;
its iteration timeline is printed as per-stage spans)"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from paper_1902_04610_b200 import build, salus as S
from workloads import TRAIN, c1_trace, c2_trace, make_job
build.build()
name = sys.argv[1]
pol = {"fifo": S.FIFO, "srtf": S.SRTF, "pack": S.PACK}[sys.argv[2] if len(sys.argv) > 2 else "fifo"]
if name.startswith("job:"):
    _, W, L, B = name.split(":")
    # declared E with 256 MiB of slack (as C4 / C5 jobs have): split-K workspace
    from workloads import footprint_bytes
    dims = (int(W),) * (int(L) + 1)
    e = footprint_bytes(TRAIN, dims, int(B))[1] + (256 << 20)
    jobs, cap = [make_job(0, TRAIN, 0, dims, int(B), 10, ephemeral_bytes=e, seed=0)], 16 << 30
else:
    jobs, cap = (c1_trace() if name == "c1" else c2_trace("a", n_jobs=1, n_iters=20) if name == "c2one"
                 else c2_trace("a", n_jobs=37, n_iters=10))
ctx = S.Context(jobs, cap, pol, trace=True)
for rep in range(2):
    ctx.run()
tr = ctx.trace()
rs = ctx.run_stats()
print("kernel ms", rs["kernel_ns"] / 1e6, "tasks", len(tr))
t0 = tr["t_claim"].min()
stage = (tr["task"] >> 21) & 31
ready = (tr["t_ready"] - tr["t_claim"]) / 1e3
mma = (tr["t_mma"] - tr["t_ready"]) / 1e3
epi = (tr["t_end"] - tr["t_mma"]) / 1e3
print("per-tile us (median): decode+xlate %.2f  mma %.2f  epilogue %.2f" % (np.median(ready), np.median(mma), np.median(epi)))
for s in sorted(set(stage.tolist())):
    m = stage == s
    print(f"stage {s:2d}: n={m.sum():5d} ready {np.median(ready[m]):6.2f} mma {np.median(mma[m]):6.2f} epi {np.median(epi[m]):6.2f}")
# one iteration timeline
key = (tr["job"].astype(np.int64) << 20) | tr["iter"]
k0 = key[np.argsort(tr["t_claim"])][len(tr) // 2]
m = key == k0
order = np.argsort(tr["t_claim"][m])
sub = tr[m][order]
base = sub["t_claim"].min()
print("stage spans of that iteration (us from first claim): stage tiles first_claim last_claim first_ready max_mma max_end  median(mma-ready) median(end-mma)")
for s_ in sorted(set(((sub["task"] >> 21) & 31).tolist())):
    q = sub[((sub["task"] >> 21) & 31) == s_]
    print(f"  s{s_:2d} n={len(q):4d} {(q['t_claim'].min() - base) / 1e3:8.2f} {(q['t_claim'].max() - base) / 1e3:8.2f} "
          f"{(q['t_ready'].min() - base) / 1e3:8.2f} {(q['t_mma'].max() - base) / 1e3:8.2f} {(q['t_end'].max() - base) / 1e3:8.2f}"
          f"  {np.median(q['t_mma'] - q['t_ready']) / 1e3:7.2f} {np.median(q['t_end'] - q['t_mma']) / 1e3:7.2f}")
if os.environ.get("SALUS_DBG_SK"):   # t_claim = split partial written + counted
    for s_ in sorted(set(((sub["task"] >> 21) & 31).tolist())):
        q = sub[((sub["task"] >> 21) & 31) == s_]
        print(f"  dbg s{s_:2d}: mma->counted {np.median(q['t_claim'] - q['t_mma']) / 1e3:7.2f}  counted->end "
              f"{np.median(q['t_end'] - q['t_claim']) / 1e3:7.2f}  max {(q['t_end'] - q['t_claim']).max() / 1e3:7.2f}")
print("timeline of one iteration (us from first claim): stage tile claim ready mma end sm")
for r in (sub if len(sub) <= 80 else []):
    print(f"  s{(r['task'] >> 21) & 31:2d} t{r['task'] & 0x1FFFFF:4d} {(r['t_claim'] - base) / 1e3:8.2f} {(r['t_ready'] - base) / 1e3:8.2f} {(r['t_mma'] - base) / 1e3:8.2f} {(r['t_end'] - base) / 1e3:8.2f} sm{r['smid']}")
# SM busy fraction: per SM, union of [t_ready, t_end] intervals / kernel span
span = (tr["t_end"].max() - tr["t_claim"].min())
busy = 0
for sm in np.unique(tr["smid"]):
    m = tr["smid"] == sm
    iv = sorted(zip(tr["t_ready"][m].tolist(), tr["t_end"][m].tolist()))
    cur_s, cur_e, tot = None, None, 0
    for s_, e_ in iv:
        if cur_e is None or s_ > cur_e:
            if cur_e is not None: tot += cur_e - cur_s
            cur_s, cur_e = s_, e_
        else:
            cur_e = max(cur_e, e_)
    tot += cur_e - cur_s
    busy += tot
print(f"SM busy fraction (epilogue-side, union of tile intervals): {busy / (span * len(np.unique(tr['smid']))):.3f} over {span / 1e6:.2f} ms")
