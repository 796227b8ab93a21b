"""Helpers for the -m gpu parity tests: run a trace through the C ABI and
through the oracle, and compare."""
import numpy as np

from oracle import logfmt as LG
from oracle import scheduler as OS


def run_gpu(jobs, cap, policy, **kw):
    from paper_1902_04610_b200 import build, salus as S
    build.build()
    ctx = S.Context(jobs, cap, policy, **kw)
    try:
        stats = ctx.run()
        return ctx, stats
    except Exception:
        ctx.close()
        raise


def first_diff(a: bytes, b: bytes, context=3):
    ra, rb = LG.decode(a), LG.decode(b)
    for i, (x, y) in enumerate(zip(ra, rb)):
        if x != y:
            lo = max(0, i - context)
            lines = [f"record {i}:"]
            for k in range(lo, min(i + context + 1, len(ra), len(rb))):
                mark = ">>" if k == i else "  "
                lines.append(f"{mark} gpu    {LG.fmt(ra[k])}")
                lines.append(f"{mark} oracle {LG.fmt(rb[k])}")
            return "\n".join(lines)
    return f"length differs: gpu {len(ra)} oracle {len(rb)} records"


def assert_schedule_parity(jobs, cap, policy, max_lanes=0, switch_ticks=0, null_work=True, evict=False,
                           **kw):
    """Byte-identical canonical log and identical per-job stats (north star:
    'run order, lane ids, per-job completion iteration ... bit-exactly')."""
    ref = OS.simulate(jobs, cap, policy, max_lanes=max_lanes, switch_ticks=switch_ticks, evict=evict)
    ctx, stats = run_gpu(jobs, cap, policy, max_lanes=max_lanes, switch_ticks=switch_ticks,
                         null_work=null_work, log=True, evict=evict, **kw)
    try:
        got = ctx.log_bytes()
        want = ref.log_bytes()
        assert got == want, first_diff(got, want)
        for jid, s in ref.stats.items():
            g = stats[jid]
            assert (g["first_lane"], g["admit_tick"], g["first_start_tick"], g["completion_tick"],
                    g["completion_seq"]) == (s.first_lane, s.admit_tick, s.first_start_tick,
                                             s.completion_tick, s.completion_seq), jid
        rs = ctx.run_stats()
        assert rs["status"] == 0 and rs["n_dispatch"] == len(ref.dispatch)
        return ctx, ref, stats
    except Exception:
        ctx.close()
        raise


def normwise_rel(g, r):
    """A24: max|g - r| / max|r| per tensor."""
    g = np.asarray(g, dtype=np.float64)
    r = np.asarray(r, dtype=np.float64)
    den = np.max(np.abs(r))
    return float(np.max(np.abs(g - r)) / (den if den > 0 else 1.0))
