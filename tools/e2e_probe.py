import sys, time
sys.path.insert(0, '.')
import torch
from paper_1902_04610_b200 import build, salus as S
from workloads import c2_trace
build.build()
jobs, cap = c2_trace("a")
for i in range(8):
    t0 = time.perf_counter()
    c = S.Context(jobs, cap, S.PACK, log=False)
    t1 = time.perf_counter()
    c.run()
    t2 = time.perf_counter()
    rs = c.run_stats()
    c.close()
    t3 = time.perf_counter()
    print(f"open+submit+prepare {1e3*(t1-t0):.1f} ms, run {1e3*(t2-t1):.1f} ms (kernel {rs['kernel_ns']/1e6:.1f}), close {1e3*(t3-t2):.1f} ms", flush=True)
