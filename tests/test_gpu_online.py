"""Online submission (the paper's "a session is created
when a job is submitted"): jobs handed to the RUNNING
persistent kernel with salus_submit_live.  The device stamps each live job's
arrival tick (logged as JOB_QUEUED); parity = replaying those logged ticks
through the oracle reproduces the whole canonical log byte for byte, and
the math of a live job still matches the oracle."""
import dataclasses
import time

import numpy as np
import pytest

from oracle import layers as OL
from oracle import scheduler as OS
from workloads import TRAIN, make_job

from gpu_helpers import first_diff, normwise_rel

pytestmark = pytest.mark.gpu

JOB_QUEUED = 7


def _queued_ticks(log_bytes, S):
    recs = np.frombuffer(log_bytes, dtype=S.LOG_DTYPE)
    m = recs["kind"] == JOB_QUEUED
    return {int(j): int(t) for j, t in zip(recs["job"][m], recs["tick"][m])}


def _small(job_id, seed, n_iters=6):
    rng = np.random.default_rng(seed)
    w = int(rng.choice([128, 256, 384]))
    depth = int(rng.integers(1, 4))
    batch = int(rng.choice([64, 128, 200]))
    # odd seeds declare 4 MiB of persistent slack: those jobs take the GEN /
    # target prefetch path (their X, T live in per-job buffers)
    from workloads import footprint_bytes
    dims = (w,) * (depth + 1)
    slack = (4 << 20) if seed % 2 else 0
    return make_job(job_id, TRAIN, 0, dims, batch, n_iters, lr=1e-2, seed=seed,
                    persistent_bytes=footprint_bytes(TRAIN, dims, batch)[0] + slack)


def _run_online(policy, pre, live, cap, delays_s, null_work, max_lanes=0):
    from paper_1902_04610_b200 import salus as S
    ctx = S.Context(pre, cap, policy, online=True, max_jobs=len(pre) + len(live), null_work=null_work,
                    max_lanes=max_lanes)
    ctx.run_async()
    for j, dt in zip(live, delays_s):
        time.sleep(dt)
        ctx.submit_live(j)
    ctx.end_submissions()
    stats = ctx.wait()
    return ctx, stats


def _check_replay(ctx, jobs, cap, policy, stats, max_lanes=0):
    from paper_1902_04610_b200 import salus as S
    got = ctx.log_bytes()
    arr = _queued_ticks(got, S)
    assert sorted(arr) == sorted(j.job_id for j in jobs)
    replay = [dataclasses.replace(j, arrival_tick=arr[j.job_id]) for j in jobs]
    ref = OS.simulate(replay, cap, policy, max_lanes=max_lanes)
    want = ref.log_bytes()
    assert got == want, first_diff(got, want)
    for jid, s in ref.stats.items():
        assert stats[jid]["completion_tick"] == s.completion_tick
        assert stats[jid]["completion_seq"] == s.completion_seq
    return arr


@pytest.mark.parametrize("policy", [OS.PACK, OS.SRTF, OS.FAIR])
def test_live_jobs_replay_to_the_oracle_log(policy):
    pre = [_small(i, 100 + i) for i in range(3)]
    live = [_small(10 + i, 200 + i) for i in range(12)]
    delays = [0.0005 * (i % 4) for i in range(12)]
    cap = 1 << 30
    ctx, stats = _run_online(policy, pre, live, cap, delays, null_work=False)
    try:
        arr = _check_replay(ctx, pre + live, cap, policy, stats)
        # live arrivals are stamped after every pre-submitted arrival, in order
        ticks = [arr[j.job_id] for j in live]
        assert ticks == sorted(ticks) and min(ticks) >= 1
        assert all(stats[j.job_id]["completion_tick"] > 0 for j in pre + live)
    finally:
        ctx.close()


def test_idle_kernel_waits_for_live_jobs_and_their_math_matches():
    """No job at launch: the kernel idles until the host submits, then runs
    them; a live job's outputs and weight updates match the oracle."""
    from paper_1902_04610_b200 import salus as S
    live = [_small(1 + i, 300 + i, n_iters=4) for i in range(6)]
    cap = 1 << 30
    ctx = S.Context([], cap, S.PACK, online=True, max_jobs=len(live), dump_bytes=64 << 20)
    try:
        ctx.run_async()
        time.sleep(0.05)                       # the kernel is up and idle
        for j in live:
            ctx.submit_live(j, dump=S.DUMP_OUTPUTS | S.DUMP_WEIGHTS)
            time.sleep(0.002)
        ctx.end_submissions()
        stats = ctx.wait()
        _check_replay(ctx, live, cap, OS.PACK, stats)
        wall = ctx.wall()
        assert len(wall) == sum(j.n_iters for j in live)
        assert np.all(wall["end_ns"] > wall["start_ns"])
        for j in live[-2:]:
            outs64, _ = OL.run_job(j)
            _, W = OL.run_job(j, store=OL.bf16)   # A31/A32: weight updates vs the bf16-storage oracle
            g = ctx.layers(j.job_id, j.n_iters - 1).reshape(j.batch, j.dims[-1])
            assert normwise_rel(g, outs64[j.n_iters - 1]) <= 2e-2
            flat = ctx.layers(j.job_id, S.WEIGHTS)
            W0 = OL.init_weights(j)
            Wg = flat[:j.dims[0] * j.dims[1]].reshape(j.dims[0], j.dims[1])
            dg, dr = Wg - W0[0], W[0] - W0[0]
            assert np.linalg.norm(dg - dr) / np.linalg.norm(dr) <= 2e-2
    finally:
        ctx.close()


def test_live_submission_errors():
    from paper_1902_04610_b200 import salus as S
    cap = 1 << 30
    plain = S.Context([_small(1, 1)], cap, S.PACK)
    try:
        with pytest.raises(S.SalusError):
            plain.submit_live(_small(2, 2))          # not an online context
    finally:
        plain.close()
    ctx = S.Context([_small(5, 5)], cap, S.PACK, online=True, max_jobs=4, null_work=True)
    try:
        with pytest.raises(S.SalusError):
            ctx.submit_live(_small(6, 6))            # not running yet
        ctx.run_async()
        with pytest.raises(S.SalusError):
            ctx.submit_live(_small(4, 4))            # ids must increase
        ctx.submit_live(_small(7, 7))
        ctx.end_submissions()
        with pytest.raises(S.SalusError):
            ctx.submit_live(_small(8, 8))            # submissions ended
        stats = ctx.wait()
        assert sorted(stats) == [5, 7]
    finally:
        ctx.close()


def test_poll_stats_streams_completions():
    """NEXT-4 streaming stats: while the kernel runs, salus_poll_stats sees
    jobs finish one by one (monotone done count, partial progress observed),
    and every record it reports as done equals salus_wait's final record."""
    import time
    from paper_1902_04610_b200 import build, salus as S
    from workloads import TRAIN, make_job
    build.build()
    jobs = [make_job(k, TRAIN, 0, (1024, 1024, 1024), 256, 30 + 10 * k, lr=1e-3, seed=k) for k in range(24)]
    ctx = S.Context(jobs, 1 << 28, S.SRTF, log=False)      # one lane: jobs finish one after another
    try:
        ctx.run_async()
        seen, last, snaps = [], -1, []
        t0 = time.time()
        while time.time() - t0 < 60:
            st, done = ctx.poll_stats()
            assert done >= last
            last = done
            seen.append(done)
            snaps.append(st)
            if done == len(jobs):
                break
            time.sleep(0.0005)
        final = ctx.wait()
    finally:
        ctx.close()
    assert last == len(jobs)
    assert any(0 < d < len(jobs) for d in seen), seen[:20]
    for st in snaps:
        for jid, s in st.items():
            if s["wall_end_ns"]:
                assert s == final[jid], jid


# --------------------------------------------------------------------------
# Live inference requests (salus_submit_requests): the paper's low-rate
# inference requests arriving in wall-clock time (A27).  Each
# request the scheduler sees at tick t gets arrival tick t + 1; parity =
# replaying the read-back request ticks through the oracle gives the log.
# --------------------------------------------------------------------------

def _infer(job_id, seed, n, dims=(256, 512, 128), b=8):
    from workloads import INFER
    from workloads.traces import footprint_bytes
    p, e = footprint_bytes(INFER, dims, b)
    return make_job(job_id, INFER, 0, dims, b, n, seed=seed, request_ticks=tuple([0] * n),
                    persistent_bytes=p, ephemeral_bytes=e)


def _live_request_run(policy, jobs, cap, schedule, max_lanes=0, dump=None, null_work=False):
    """jobs: INFER jobs (their request_ticks are ignored: live); schedule:
    list of (delay_s, [job ids]) batches."""
    from paper_1902_04610_b200 import salus as S
    live = [dataclasses.replace(j, request_ticks=()) for j in jobs]
    ctx = S.Context(live, cap, policy, online=True, max_lanes=max_lanes, dump=dump, null_work=null_work)
    ctx.run_async()
    for dt, ids in schedule:
        if dt:
            time.sleep(dt)
        ctx.submit_requests(ids)
    ctx.end_submissions()
    stats = ctx.wait()
    return ctx, stats


def _replay_requests(ctx, jobs, cap, policy, stats, max_lanes=0):
    got = ctx.log_bytes()
    replay, seen = [], {}
    for j in jobs:
        ticks, s = ctx.requests(j.job_id)
        assert np.all(np.diff(ticks) >= 0) and np.all(s > 0)
        seen[j.job_id] = s
        replay.append(dataclasses.replace(j, request_ticks=tuple(int(x) for x in ticks)))
    ref = OS.simulate(replay, cap, policy, max_lanes=max_lanes)
    want = ref.log_bytes()
    assert got == want, first_diff(got, want)
    for jid, s in ref.stats.items():
        assert stats[jid]["completion_tick"] == s.completion_tick
    return replay, seen


@pytest.mark.parametrize("policy,max_lanes", [(OS.PACK, 0), (OS.FAIR, 2), (OS.FAIR, 1)])
def test_live_requests_replay_to_the_oracle_log(policy, max_lanes):
    jobs = [_infer(i, 300 + i, 12) for i in range(5)]
    rng = np.random.default_rng(7)
    order = [j.job_id for j in jobs for _ in range(j.n_iters)]
    rng.shuffle(order)
    # batches of 1-3 requests, 0-300 us apart (some arrive while lanes are busy)
    schedule, k = [], 0
    while k < len(order):
        n = int(rng.integers(1, 4))
        schedule.append((float(rng.choice([0.0, 1e-4, 3e-4])), order[k:k + n]))
        k += n
    ctx, stats = _live_request_run(policy, jobs, 1 << 30, schedule, max_lanes=max_lanes)
    try:
        _replay_requests(ctx, jobs, 1 << 30, policy, stats, max_lanes=max_lanes)
    finally:
        ctx.close()


def test_live_requests_math_and_latency_stamps():
    """Outputs of live requests equal the oracle's (data keyed by the request
    index, A29), and every request's first tile starts after it was seen."""
    from paper_1902_04610_b200 import salus as S
    jobs = [_infer(0, 401, 6, dims=(512, 1024, 256), b=16), _infer(1, 402, 6, dims=(128, 384, 64), b=1)]
    schedule = [(2e-4, [0, 1]) for _ in range(6)]
    ctx, stats = _live_request_run(OS.PACK, jobs, 1 << 30, schedule,
                                   dump={0: S.DUMP_OUTPUTS, 1: S.DUMP_OUTPUTS})
    try:
        replay, seen = _replay_requests(ctx, jobs, 1 << 30, OS.PACK, stats)
        for j in replay:
            outs, _ = OL.run_job(j)
            for k in range(j.n_iters):
                g = ctx.layers(j.job_id, k).reshape(j.batch, j.dims[-1])
                assert normwise_rel(g, outs[k]) <= 2e-2, (j.job_id, k)
        w = ctx.wall()
        for j in jobs:
            starts = np.sort(w["start_ns"][w["job"] == j.job_id].astype(np.int64))
            assert len(starts) == j.n_iters
            assert np.all(starts >= seen[j.job_id].astype(np.int64))
    finally:
        ctx.close()


def test_live_request_errors():
    from paper_1902_04610_b200 import salus as S
    jobs = [_infer(0, 501, 2)]
    ctx = S.Context([dataclasses.replace(jobs[0], request_ticks=())], 1 << 30, OS.PACK, online=True,
                    null_work=True)
    try:
        with pytest.raises(S.SalusError):
            ctx.submit_requests([0])                      # not running
        ctx.run_async()
        with pytest.raises(S.SalusError):
            ctx.submit_requests([7])                      # unknown job
        with pytest.raises(S.SalusError):
            ctx.submit_requests([0, 0, 0])                # more than n_iters: nothing published
        ctx.submit_requests([0, 0])
        ctx.end_submissions()
        stats = ctx.wait()
        assert stats[0]["completion_tick"] > 0
    finally:
        ctx.close()
    # an offline context needs request ticks
    with pytest.raises(S.SalusError):
        S.Context([dataclasses.replace(jobs[0], request_ticks=())], 1 << 30, OS.PACK)
