"""A/B of eager stage publication (REC_FLAG_EAGER): the same
configs with SALUS_EAGER_LANES = 0 (never eager) and = 64 (always), two
interleaved rounds on one GPU.  Kernel times from CUDA events (run_stats),
iteration times from the device wall stamps.

usage: python tools/ab_eager.py [--c5] [--rounds 2] [--values 0,64]
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1902_04610_b200 import build, salus as S  # noqa: E402
from workloads import c1_trace, c2_trace, c3_trace, c4_trace, c5_trace  # noqa: E402


def run(jobs, cap, pol, max_lanes=0, log=False, reps=1):
    ctx = S.Context(jobs, cap, pol, device=0, max_lanes=max_lanes, log=log)
    try:
        ks = []
        for _ in range(reps):
            ctx.run()
            ks.append(ctx.run_stats()["kernel_ns"] / 1e6)
        w = ctx.wall() if log else None
    finally:
        ctx.close()
    return float(np.median(ks)), w


def iter_us(w):
    return float(np.median((w["end_ns"] - w["start_ns"]) / 1e3))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--c5", action="store_true")
    ap.add_argument("--rounds", type=int, default=2)
    ap.add_argument("--values", default="0,64")
    args = ap.parse_args()
    build.build()
    vals = [int(v) for v in args.values.split(",")]
    out = {v: {} for v in vals}
    for r in range(args.rounds):
        for v in vals:
            os.environ["SALUS_EAGER_LANES"] = str(v)
            res = out[v]
            for pol, name in ((S.FIFO, "c1_fifo"), (S.SRTF, "c1_srtf")):
                ms, w = run(*c1_trace(), pol, log=True, reps=3)
                res.setdefault(name + "_iter_us", []).append(iter_us(w))
            ms, w = run(*c2_trace("a"), S.PACK, reps=3)
            res.setdefault("c2a_ms", []).append(ms)
            ms, w = run(*c3_trace(), S.FAIR, max_lanes=8, log=True)
            res.setdefault("c3_fair8_ms", []).append(ms)
            res.setdefault("c3_iter_us", []).append(iter_us(w))
            ms, w = run(*c3_trace(), S.PACK)
            res.setdefault("c3_pack_ms", []).append(ms)
            for pol, name in ((S.SRTF, "c4_srtf_ms"), (S.PACK, "c4_pack_ms")):
                ms, _ = run(*c4_trace(), pol)
                res.setdefault(name, []).append(ms)
            if args.c5:
                ms, _ = run(*c5_trace(), S.PACK)
                res.setdefault("c5_pack_ms", []).append(ms)
            print(json.dumps({"round": r, "eager_lanes": v, **{k: x[-1] for k, x in res.items()}}), flush=True)
    print(json.dumps({str(v): {k: float(np.mean(x)) for k, x in out[v].items()} for v in vals}), flush=True)


if __name__ == "__main__":
    main()
