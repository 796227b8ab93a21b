"""Bring-up probe: run small pieces of the GPU path step by step and print
what happens (used during development under gpurun)."""
import os
import sys
import time
import traceback

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import scheduler as OS, layers as OL  # noqa: E402
from paper_1902_04610_b200 import build, salus as S  # noqa: E402
from workloads import TRAIN, INFER, c1_trace, tiny_math_trace, c2_trace  # noqa: E402
from gpu_helpers import first_diff, normwise_rel  # noqa: E402


def step(name, fn):
    t = time.time()
    try:
        r = fn()
        print(f"[ok ] {name} ({time.time() - t:.2f}s) {r if r is not None else ''}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"[ERR] {name} ({time.time() - t:.2f}s): {e}", flush=True)
        traceback.print_exc()


def sched(jobs, cap, pol, **kw):
    ref = OS.simulate(jobs, cap, pol, max_lanes=kw.get("max_lanes", 0))
    ctx = S.Context(jobs, cap, pol, timeout_ms=30000, **kw)
    st = ctx.run()
    got = ctx.log_bytes()
    rs = ctx.run_stats()
    ok = got == ref.log_bytes()
    msg = f"parity={ok} n_dispatch={rs['n_dispatch']} ticks={rs['n_ticks']} kernel_ms={rs['kernel_ns'] / 1e6:.3f}"
    if not ok:
        msg += "\n" + first_diff(got, ref.log_bytes())
    return ctx, msg


def main():
    print(torch.cuda.get_device_name(0), flush=True)
    build.build(verbose=True)
    jobs, cap = c1_trace()
    for pol in (OS.FIFO, OS.SRTF):
        step(f"c1 null-work pol={pol}", lambda: sched(jobs, cap, pol, null_work=True)[1])

    def tiny(kind):
        js, c = tiny_math_trace(kind, n_jobs=1, dims=(128, 128), batch=128, n_iters=1)
        dump = {js[0].job_id: S.DUMP_OUTPUTS | (S.DUMP_WEIGHTS if kind == TRAIN else 0)}
        ctx, msg = sched(js, c, OS.PACK, dump=dump)
        outs, W = OL.run_job(js[0])
        g = ctx.layers(js[0].job_id, 0).reshape(128, 128)
        r = outs[0]
        msg += f" out_rel={normwise_rel(g, r):.3e} g[0,:4]={g[0, :4]} r[0,:4]={r[0, :4]}"
        if kind == TRAIN:
            W0 = OL.init_weights(js[0])
            wg = ctx.layers(js[0].job_id, S.WEIGHTS).reshape(128, 128)
            msg += f" dW_rel={normwise_rel(wg - W0[0], W[0] - W0[0]):.3e}"
        return msg

    step("tiny infer 1 layer", lambda: tiny(INFER))
    step("tiny train 1 layer", lambda: tiny(TRAIN))

    def c1real(pol):
        dump = {j.job_id: S.DUMP_OUTPUTS | S.DUMP_WEIGHTS for j in jobs}
        ctx, msg = sched(jobs, cap, pol, dump=dump)
        worst = 0
        for j in jobs:
            outs, W = OL.run_job(j)
            for k in range(j.n_iters):
                worst = max(worst, normwise_rel(ctx.layers(j.job_id, k).reshape(j.batch, -1), outs[k]))
        w = ctx.wall()
        gaps = (w["start_ns"][1:].astype(np.int64) - w["end_ns"][:-1].astype(np.int64)) / 1e3
        return msg + f" worst_out_rel={worst:.3e} iter_us={np.median((w['end_ns'] - w['start_ns']) / 1e3):.1f} gap_us_med={np.median(gaps):.2f}"

    step("c1 real FIFO", lambda: c1real(OS.FIFO))
    step("c1 real SRTF", lambda: c1real(OS.SRTF))

    def c2(n_jobs, n_iters):
        js, c = c2_trace("a", n_jobs=n_jobs, n_iters=n_iters)
        ctx, msg = sched(js, c, OS.PACK)
        rs = ctx.run_stats()
        return msg + f" iters/s={rs['n_dispatch'] / (rs['kernel_ns'] / 1e9):.0f}"

    step("c2 small (10 jobs x 5 it)", lambda: c2(10, 5))
    step("c2 full", lambda: c2(300, 100))


if __name__ == "__main__":
    main()
