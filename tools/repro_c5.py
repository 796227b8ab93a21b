"""Run C5-generator traces of growing size with a device watchdog and report
which complete (debugging aid).  usage: python tools/repro_c5.py [n ...]"""
import os
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

CHILD = r'''
import sys, time
sys.path.insert(0, %r)
from paper_1902_04610_b200 import salus as S
from workloads import c5_trace
n, pol = int(sys.argv[1]), sys.argv[2]
jobs, cap = c5_trace(n_jobs=n)
ctx = S.Context(jobs, cap, {"pack": S.PACK, "srtf": S.SRTF}[pol], timeout_ms=%d)
t = time.time()
try:
    ctx.run()
    print("OK", n, pol, round(time.time() - t, 2), ctx.run_stats()["n_dispatch"], flush=True)
finally:
    ctx.close()
'''


def main():
    ns = [int(x) for x in sys.argv[1:]] or [50, 200, 600, 2000]
    for pol in ("pack",):
        for n in ns:
            code = CHILD % (ROOT, 150000)
            t = time.time()
            r = subprocess.run([sys.executable, "-c", code, str(n), pol], capture_output=True, text=True,
                               timeout=400)
            print(f"n={n} {pol} rc={r.returncode} {time.time() - t:.1f}s", (r.stdout + r.stderr).strip()[-300:],
                  flush=True)


if __name__ == "__main__":
    main()
