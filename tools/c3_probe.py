"""What bounds C3 (42 inference models): per policy, kernel time, scheduler
wait (and its fence / ring parts), and the physical busy time of each lane
from the wall stamps -- the busiest lane bounds a run whose scheduler waits.
usage: python tools/c3_probe.py"""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), '..'))
from paper_1902_04610_b200 import build, salus as S
from workloads import c3_trace
import numpy as np
build.build()
jobs,cap=c3_trace()
for pol,ml in ((S.FAIR,8),(S.PACK,0)):
    ctx=S.Context(jobs,cap,pol,max_lanes=ml,log=True)
    ctx.run(); ctx.run(); rs=ctx.run_stats(); w=ctx.wall()
    ctx.close()
    busy=np.zeros(64)
    for ln in np.unique(w['lane']):
        m=w[w['lane']==ln]; busy[ln]=np.sum(m['end_ns']-m['start_ns'])/1e6
    print(pol, 'kernel ms', rs['kernel_ns']/1e6, 'wait', rs['sched_wait_ns']/1e6, 'fence', rs['sched_fence_ns']/1e6, 'ring', rs['sched_ring_ns']/1e6,
          'lanes', len(np.unique(w['lane'])), 'lane busy ms (mean,max)', busy[busy>0].mean(), busy.max())
