"""Stress: C4 under FIFO/SRTF/PACK/FAIR repeatedly in ONE process (the bench's
c4 section pattern), each run with a 30 s device watchdog.  Debugging aid for
the opt-in split-K build.  usage: SALUS_LIB=... SALUS_SPLITK=1 python tools/stress_c4.py [rounds]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1902_04610_b200 import salus as S  # noqa: E402
from workloads import c4_trace, c5_trace  # noqa: E402

rounds = int(sys.argv[1]) if len(sys.argv) > 1 else 3
jobs, cap = c4_trace()
print("lib", S.LIB_PATH, "splitk", os.environ.get("SALUS_SPLITK"), flush=True)
for r in range(rounds):
    for name, pol in (("fifo", S.FIFO), ("srtf", S.SRTF), ("pack", S.PACK), ("fair", S.FAIR)):
        t = time.time()
        ctx = S.Context(jobs, cap, pol, timeout_ms=30000)
        try:
            ctx.run()
            print(f"round {r} {name}: ok {time.time() - t:.1f} s kernel {ctx.run_stats()['kernel_ns'] / 1e6:.0f} ms",
                  flush=True)
        except Exception as exc:  # noqa: BLE001
            print(f"round {r} {name}: FAIL after {time.time() - t:.1f} s: {exc}", flush=True)
            sys.exit(1)
        finally:
            ctx.close()
