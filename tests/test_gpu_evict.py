"""GPU parity for SRTF admission with persistent eviction (SURVEY §8(f)
NEXT-3, reading A35).  The device scheduler must reproduce
the oracle's log byte for byte (JOB_EVICT / JOB_RESTORE records included),
and the kernel's swap records -- persistent pages copied to pinned host
memory and back into fresh arena pages -- must leave every evicted job's
math exactly on its own trajectory: outputs of every iteration and final
weights within the north-star tolerance of the oracle's (which never
swaps)."""
import numpy as np
import pytest

from oracle import logfmt as LG
from oracle import scheduler as OS
from workloads import PAGE_BYTES, TRAIN, INFER, make_job, random_sched_trace

from gpu_helpers import assert_schedule_parity
from test_gpu_math import _check_math

pytestmark = pytest.mark.gpu
G = PAGE_BYTES


def _n_evicts(ref):
    return sum(1 for r in ref.log if r[1] == LG.JOB_EVICT)


@pytest.mark.parametrize("null_work", [True, False])
def test_hand_trace_evict(null_work):
    """HW-EV of tests/test_oracle_evict.py on the device, with real work the
    evicted job's outputs and weights survive the swap round trip."""
    from paper_1902_04610_b200 import salus as S
    jobs = [make_job(0, TRAIN, 0, (128, 256, 128), 128, 10, iter_ticks=100, persistent_bytes=8 * G,
                     ephemeral_bytes=6 * G, lr=1e-2, seed=11),
            make_job(1, TRAIN, 150, (128, 256, 128), 128, 1, iter_ticks=100, persistent_bytes=8 * G,
                     ephemeral_bytes=6 * G, lr=1e-2, seed=12)]
    cap = 20 * G
    dump = None if null_work else {j.job_id: S.DUMP_OUTPUTS | S.DUMP_WEIGHTS for j in jobs}
    ctx, ref, stats = assert_schedule_parity(jobs, cap, OS.SRTF, evict=True, null_work=null_work, dump=dump)
    try:
        assert _n_evicts(ref) == 1
        rs = ctx.run_stats()
        if not null_work:
            assert rs["n_swap_out"] == 1 and rs["n_swap_in"] == 1
            _check_math(ctx, jobs)
    finally:
        ctx.close()


@pytest.mark.parametrize("max_lanes", [1, 2, 4])
def test_random_traces_schedule(max_lanes):
    rng = np.random.default_rng(900 + max_lanes)
    total = 0
    for trial in range(25):
        jobs, C = random_sched_trace(rng, int(rng.integers(2, 14)), cap_pages=int(rng.integers(8, 40)),
                                     infer_frac=0.2, max_iters=8)
        ctx, ref, stats = assert_schedule_parity(jobs, C, OS.SRTF, max_lanes=max_lanes, evict=True)
        total += _n_evicts(ref)
        ctx.close()
    assert total > 0


def _pressure_trace(seed, n_jobs=8, cap_pages=96):
    """Real MLPs under memory pressure: a long job first, shorter ones
    arriving while it runs (each alone fits; two do not share the GPU)."""
    rng = np.random.default_rng(seed)
    jobs = []
    shapes = [((256, 256, 256), 128), ((128, 384, 128), 200), ((256, 128, 256, 128), 96)]
    for j in range(n_jobs):
        dims, b = shapes[j % len(shapes)]
        n = 12 if j == 0 else int(rng.integers(2, 6))
        p = int(rng.integers(20, 40))
        e = int(rng.integers(30, cap_pages - p - 5))
        jobs.append(make_job(j, TRAIN if j % 4 != 3 else INFER, 0 if j == 0 else int(rng.integers(50, 4000)),
                             dims, b, n, iter_ticks=int(rng.integers(100, 400)), persistent_bytes=p * G,
                             ephemeral_bytes=e * G, lr=5e-3, seed=100 + j,
                             request_ticks=tuple(sorted(int(x) for x in rng.integers(4000, 6000, size=n)))
                             if j % 4 == 3 else ()))
    return jobs, cap_pages * G


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_real_work_swap_round_trip(seed):
    from paper_1902_04610_b200 import salus as S
    jobs, cap = _pressure_trace(seed)
    ref = OS.simulate(jobs, cap, OS.SRTF, evict=True)
    assert _n_evicts(ref) >= 1, "trace must exercise eviction"
    dump = {j.job_id: S.DUMP_OUTPUTS | (S.DUMP_WEIGHTS if j.kind == TRAIN else 0) for j in jobs}
    ctx, ref, stats = assert_schedule_parity(jobs, cap, OS.SRTF, evict=True, null_work=False, dump=dump)
    try:
        rs = ctx.run_stats()
        n_ev = _n_evicts(ref)
        n_re = sum(1 for r in ref.log if r[1] == LG.JOB_RESTORE)
        assert (rs["n_swap_out"], rs["n_swap_in"]) == (n_ev, n_re)
        _check_math(ctx, jobs)
    finally:
        ctx.close()


def test_evict_flag_validation():
    from paper_1902_04610_b200 import salus as S
    jobs = [make_job(0, TRAIN, 0, (128, 128), 128, 1, iter_ticks=10)]
    for pol in (S.FIFO, S.PACK, S.FAIR):
        with pytest.raises(S.SalusError):
            S.Context(jobs, 1 << 26, pol, evict=True)


def test_c4e_schedule_parity():
    """C4e (the bench's eviction config, 13 evictions) with the allocator and
    dispatch only: byte-identical log."""
    from workloads import c4_trace
    jobs, cap = c4_trace(p_scale=8.0)
    ctx, ref, stats = assert_schedule_parity(jobs, cap, OS.SRTF, evict=True)
    assert _n_evicts(ref) >= 10
    ctx.close()


def test_c4e_real_work_swaps_do_not_change_math():
    """Full size: C4e executed with eviction (the [4096]^5 B=1024 job 49 is
    swapped out and back 11 times, 0.5 GB each way) and without it must give
    bit-identical final weights for every evicted job -- the kernel's math is
    deterministic per job, so any byte lost or misplaced by a swap round trip
    would show (the oracle cannot follow 1583 iterations of this job)."""
    from paper_1902_04610_b200 import salus as S
    from workloads import c4_trace
    jobs, cap = c4_trace(p_scale=8.0)
    ref = OS.simulate(jobs, cap, OS.SRTF, evict=True)
    victims = sorted({r[3] for r in ref.log if r[1] == LG.JOB_EVICT})
    assert victims
    dump = {v: S.DUMP_WEIGHTS for v in victims}
    out = {}
    for ev in (True, False):
        ctx, r2, stats = assert_schedule_parity(jobs, cap, OS.SRTF, evict=ev, null_work=False, dump=dump,
                                                timeout_ms=300000)
        try:
            out[ev] = {v: ctx.layers(v, S.WEIGHTS).copy() for v in victims}
            if ev:
                rs = ctx.run_stats()
                assert rs["n_swap_out"] == _n_evicts(ref) == rs["n_swap_in"]
        finally:
            ctx.close()
    for v in victims:
        assert np.isfinite(out[True][v]).all()
        assert np.array_equal(out[True][v], out[False][v]), v
