"""Per-SM tile timeline from the device trace (C2 small).  Prints, for one SM,
consecutive tiles: stage, phases (claim, epilogue-ready, acc-ready, end) in us
relative to the first, plus aggregate phase sums."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
import numpy as np
from paper_1902_04610_b200 import build, salus as S
from workloads import c2_trace
build.build()
jobs, cap = c2_trace("a", n_jobs=int(sys.argv[1]) if len(sys.argv) > 1 else 37, n_iters=10)
ctx = S.Context(jobs, cap, S.PACK, trace=True)
ctx.run(); ctx.run()
tr = ctx.trace()
rs = ctx.run_stats()
print("kernel ms", rs["kernel_ns"] / 1e6, "iters", rs["n_dispatch"], "tasks", len(tr))
stage = (tr["task"] >> 21) & 31
sm = np.bincount(tr["smid"]).argmax()
m = tr["smid"] == sm
sub = tr[m][np.argsort(tr["t_ready"][m])]
base = sub["t_claim"].min()
mid = len(sub) // 2
print(f"SM {sm}: {len(sub)} tiles; middle 30:")
for r in sub[mid:mid + 30]:
    st = (r["task"] >> 21) & 31
    print(f"  s{st:2d} claim {(r['t_claim'] - base) / 1e3:9.2f} ready {(r['t_ready'] - base) / 1e3:9.2f} "
          f"acc {(r['t_mma'] - base) / 1e3:9.2f} end {(r['t_end'] - base) / 1e3:9.2f}  "
          f"wait_acc {(r['t_mma'] - r['t_ready']) / 1e3:6.2f} epi {(r['t_end'] - r['t_mma']) / 1e3:6.2f}")
# per-SM: fraction of time the epilogue side is (a) waiting acc, (b) in epilogue, (c) idle (no desc)
span = tr["t_end"].max() - tr["t_claim"].min()
wa = np.sum(tr["t_mma"] - tr["t_ready"]) / 1e3
ep = np.sum(tr["t_end"] - tr["t_mma"]) / 1e3
n_sm = len(np.unique(tr["smid"]))
print(f"epilogue side over {n_sm} SMs x {span / 1e6:.3f} ms: waiting-acc {wa / (n_sm * span / 1e3):.3f}, "
      f"epilogue {ep / (n_sm * span / 1e3):.3f}")
for s in sorted(set(stage.tolist())):
    k = stage == s
    print(f"stage {s:2d}: n={k.sum():6d} wait_acc med {np.median((tr['t_mma'] - tr['t_ready'])[k]) / 1e3:6.2f} "
          f"epi med {np.median((tr['t_end'] - tr['t_mma'])[k]) / 1e3:6.2f}  epi sum share "
          f"{np.sum((tr['t_end'] - tr['t_mma'])[k]) / 1e3 / ep:.3f}")
