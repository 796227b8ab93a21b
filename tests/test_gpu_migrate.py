"""Migration primitive: a job run for k iterations in
one Salus context, its persistent state exported (SALUS_DUMP_STATE -> a
swap record at JobFinish -> salus_read_state) and resumed in another
context (resume_state, resume_iter) for the remaining n - k iterations must
reproduce the uninterrupted run bit for bit -- the kernel's math is
deterministic per job, the data generator is keyed by the job's own
iteration index (A29), and the bf16 weight copy parity follows it -- and
stay within the north-star tolerance of the oracle's n-iteration
trajectory.  On a multi-GPU box the image moves between GPUs through host
memory; here both contexts share the one GPU (one after the other)."""
import dataclasses

import numpy as np
import pytest

from oracle import layers as OL
from oracle import scheduler as OS
from workloads import TRAIN, make_job

from gpu_helpers import normwise_rel

pytestmark = pytest.mark.gpu


def _run(jobs, dump, policy=OS.PACK, resume=None, cap=1 << 30):
    from paper_1902_04610_b200 import build, salus as S
    build.build()
    ctx = S.Context(jobs, cap, policy, dump=dump, resume=resume, log=True)
    try:
        ctx.run()
        assert ctx.run_stats()["status"] == 0
        return ctx
    except Exception:
        ctx.close()
        raise


@pytest.mark.parametrize("k,slack", [(1, 0), (2, 0), (5, 0), (2, 8 << 20)])
def test_split_run_equals_straight_run(k, slack):
    """slack > 0: the declared P leaves room for the GEN-prefetch X buffers,
    which then travel inside the state image."""
    from paper_1902_04610_b200 import salus as S
    from workloads import footprint_bytes
    n = 6
    full = make_job(7, TRAIN, 0, (256, 512, 256), 200, n, lr=1e-2, seed=41,
                    persistent_bytes=footprint_bytes(TRAIN, (256, 512, 256), 200)[0] + slack)
    ctx = _run([full], {7: S.DUMP_WEIGHTS | S.DUMP_OUTPUTS})
    W_straight = ctx.layers(7, S.WEIGHTS).copy()
    out_straight = [ctx.layers(7, i).copy() for i in range(n)]
    ctx.close()

    first = dataclasses.replace(full, n_iters=k)
    ctx = _run([first], {7: S.DUMP_STATE | S.DUMP_OUTPUTS})
    img = ctx.read_state(7)
    out_first = [ctx.layers(7, i).copy() for i in range(k)]
    ctx.close()

    # the rest, resumed beside an unrelated job (different pages, other lane)
    rest = dataclasses.replace(full, n_iters=n - k)
    other = make_job(8, TRAIN, 0, (384, 128, 256), 100, 3, lr=1e-2, seed=5)
    ctx = _run([other, rest], {7: S.DUMP_WEIGHTS | S.DUMP_OUTPUTS}, resume={7: (img, k)})
    W_split = ctx.layers(7, S.WEIGHTS).copy()
    out_rest = [ctx.layers(7, i).copy() for i in range(n - k)]
    ctx.close()

    assert np.array_equal(W_split, W_straight)
    for i, o in enumerate(out_first + out_rest):
        assert np.array_equal(o, out_straight[i]), i
    # and the oracle's uninterrupted trajectory (north-star tolerance, A32)
    outs, W = OL.run_job(full, store=OL.bf16)
    off = 0
    for l in range(len(full.dims) - 1):
        m = full.dims[l] * full.dims[l + 1]
        assert normwise_rel(W_split[off:off + m].reshape(full.dims[l], full.dims[l + 1]), W[l]) <= 2e-2
        off += m
    assert normwise_rel(out_rest[-1].reshape(full.batch, -1), outs[n - 1]) <= 2e-2


def test_resumed_job_under_eviction():
    """The resumed job is also a candidate victim: SRTF with eviction swaps it
    out and back; its weights still equal the straight run's."""
    from paper_1902_04610_b200 import salus as S
    G = 1 << 16
    n, k = 8, 3
    full = make_job(0, TRAIN, 0, (128, 256, 128), 128, n, iter_ticks=100, persistent_bytes=10 * G,
                    ephemeral_bytes=6 * G, lr=1e-2, seed=11)      # 8 + 2 X-buffer pages: GEN prefetch
    ctx = _run([full], {0: S.DUMP_WEIGHTS})
    W_straight = ctx.layers(0, S.WEIGHTS).copy()
    ctx.close()
    ctx = _run([dataclasses.replace(full, n_iters=k)], {0: S.DUMP_STATE})
    img = ctx.read_state(0)
    ctx.close()
    rest = dataclasses.replace(full, n_iters=n - k)
    short = make_job(1, TRAIN, 150, (128, 256, 128), 128, 1, iter_ticks=100, persistent_bytes=10 * G,
                     ephemeral_bytes=6 * G, lr=1e-2, seed=12)
    from paper_1902_04610_b200 import build
    build.build()
    ref = OS.simulate([rest, short], 24 * G, OS.SRTF, evict=True)
    assert sum(1 for r in ref.log if r[1] == 10) == 1
    ctx = S.Context([rest, short], 24 * G, S.SRTF, evict=True, dump={0: S.DUMP_WEIGHTS},
                    resume={0: (img, k)}, log=True)
    try:
        ctx.run()
        assert ctx.log_bytes() == ref.log_bytes()
        assert ctx.run_stats()["n_swap_out"] == 1
        assert np.array_equal(ctx.layers(0, S.WEIGHTS), W_straight)
    finally:
        ctx.close()


def test_rebalance_plan_from_device_schedules_equals_oracle():
    """NEXT-4 (A39): the drain-time migration plan computed from this
    package's own device schedules (schedule-only runs) equals the oracle
    rule's, and the migrated job's two parts give the uninterrupted job's
    weights bit for bit."""
    from oracle import placement as OP
    from paper_1902_04610_b200 import multigpu as MG, salus as S
    from workloads import c4_trace
    jobs, cap = c4_trace(n_jobs=40, seed=11, burst=True)
    parts = OP.place_mod(jobs, 3)
    moves, new, ms = MG.plan_rebalance(parts, lambda r, p: MG.device_schedule(p, cap, OS.PACK))
    assert (moves, ms) == OP.rebalance(parts, cap, OS.PACK) and moves
    jid, src, dst, k, T = moves[0]
    full = [j for j in jobs if j.job_id == jid][0]
    small = dataclasses.replace(full, n_iters=min(full.n_iters, k + 3))   # a short run of the same job
    ctx = _run([small], {jid: S.DUMP_WEIGHTS}, cap=cap)
    W_straight = ctx.layers(jid, S.WEIGHTS).copy()
    ctx.close()
    if k:
        ctx = _run([dataclasses.replace(small, n_iters=k)], {jid: S.DUMP_STATE}, cap=cap)
        img = ctx.read_state(jid)
        ctx.close()
        rest = dataclasses.replace(small, n_iters=small.n_iters - k, arrival_tick=T)
        ctx = _run([rest], {jid: S.DUMP_WEIGHTS}, resume={jid: (img, k)}, cap=cap)
    else:
        ctx = _run([dataclasses.replace(small, arrival_tick=T)], {jid: S.DUMP_WEIGHTS}, cap=cap)
    try:
        assert np.array_equal(ctx.layers(jid, S.WEIGHTS), W_straight)
    finally:
        ctx.close()
