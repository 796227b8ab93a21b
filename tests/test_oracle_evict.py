"""Pins for SRTF admission with persistent eviction (SURVEY §8(f) NEXT-3,
reading A35 of DESIGN.md) in the oracle, against what the paper fixes:

* P:530 "The higher priority job is admitted as long as its own safety
  condition is met -- i.e., at least, it can run alone on the GPU --
  regardless of other already-running jobs": a hand-worked trace (the
  expected log written out record by record), and invariant I8 (the
  top-priority queued job is never left waiting behind idle lower-priority
  jobs) on random traces;
* P:479-486 the safety condition, recomputed from the log alone with the
  EVICT / RESTORE records;
* P:353-354 / 645 preemption only at iteration boundaries: a victim is never
  mid-iteration, and its iterations continue where they stopped.
"""
import numpy as np
import pytest

from oracle import logfmt as LG
from oracle import scheduler as S
from workloads import PAGE_BYTES, TRAIN, INFER, make_job, random_sched_trace

G = PAGE_BYTES
N = LG.NONE32


def _job(jid, arr, p, e, n, c):
    return make_job(jid, TRAIN, arr, (128, 128), 128, n, iter_ticks=c,
                    persistent_bytes=p * G, ephemeral_bytes=e * G)


def test_hand_trace_eviction():
    """HW-EV: C = 10 pages, one lane.  J0 (p 3, e 6, 10 x 100 ticks, arr 0)
    runs; J1 (p 3, e 6, 1 x 100 ticks, arr 150) cannot join (3 + 6 + 3 > 10)
    nor open a second lane.  At 150 J0 is mid-iteration (not evictable); at
    its iteration boundary 200 J0 (remaining 800) is swapped out for J1
    (remaining 100), J1 runs alone, finishes at 300, and J0 is restored and
    resumes at iteration 2."""
    jobs = [_job(0, 0, 3, 6, 10, 100), _job(1, 150, 3, 6, 1, 100)]
    res = S.simulate(jobs, 10 * G, S.SRTF, evict=True, check_invariants=True)
    exp = [
        (0, LG.JOB_QUEUED, N, 0, 0, 0),
        (0, LG.LANE_OPEN, 0, 0, 6, 0),
        (0, LG.JOB_ADMIT, 0, 0, 3, 6),
        (0, LG.DISPATCH, 0, 0, 0, 0),
        (100, LG.DISPATCH, 0, 0, 1, 1),
        (150, LG.JOB_QUEUED, N, 1, 0, 0),
        (200, LG.JOB_EVICT, 0, 0, 3, 2),
        (200, LG.LANE_CLOSE, 0, 0, 0, 0),
        (200, LG.LANE_OPEN, 1, 1, 6, 0),
        (200, LG.JOB_ADMIT, 1, 1, 3, 6),
        (200, LG.DISPATCH, 1, 1, 0, 2),
        (300, LG.JOB_FINISH, 1, 1, 1, 2),
        (300, LG.LANE_CLOSE, 1, 1, 0, 0),
        (300, LG.LANE_OPEN, 2, 0, 6, 0),
        (300, LG.JOB_RESTORE, 2, 0, 3, 6),
    ] + [(300 + 100 * (k - 2), LG.DISPATCH, 2, 0, k, k + 1) for k in range(2, 10)] + [
        (1100, LG.JOB_FINISH, 2, 0, 10, 10),
        (1100, LG.LANE_CLOSE, 2, 0, 0, 0),
    ]
    assert res.log == exp
    st = res.stats
    assert (st[0].first_lane, st[0].admit_tick, st[0].first_start_tick, st[0].completion_tick,
            st[0].completion_seq) == (0, 0, 0, 1100, 10)
    assert (st[1].first_lane, st[1].admit_tick, st[1].completion_tick) == (1, 200, 300)
    # without eviction J1 waits for J0: JCTs {1000, 950} -> {1100, 150}
    plain = S.simulate(jobs, 10 * G, S.SRTF)
    assert [plain.stats[j].completion_tick - a for j, a in ((0, 0), (1, 150))] == [1000, 950]
    assert [res.stats[j].completion_tick - a for j, a in ((0, 0), (1, 150))] == [1100, 150]


def test_no_eviction_of_higher_or_equal_priority():
    """A newcomer with MORE remaining work than the resident never evicts it."""
    jobs = [_job(0, 0, 3, 6, 2, 100), _job(1, 50, 3, 6, 5, 100)]
    res = S.simulate(jobs, 10 * G, S.SRTF, evict=True, check_invariants=True)
    assert not any(r[1] == LG.JOB_EVICT for r in res.log)
    assert res.log_bytes() == S.simulate(jobs, 10 * G, S.SRTF).log_bytes()


def test_all_or_nothing():
    """Evicting every lower-priority idle job must make the newcomer fit,
    else nobody is evicted: J2 (p 6) cannot fit while J0 (higher priority
    than J2) holds 3 + 4 pages of a 12-page GPU, so J1 stays resident."""
    jobs = [_job(0, 0, 3, 4, 3, 10), _job(1, 0, 2, 3, 50, 10), _job(2, 5, 6, 4, 20, 10)]
    res = S.simulate(jobs, 12 * G, S.SRTF, max_lanes=2, evict=True, check_invariants=True)
    ev = [r for r in res.log if r[1] == LG.JOB_EVICT]
    # J0 (remaining 30) outranks J2 (200): J2 may only evict J1 (remaining 500),
    # and J1 alone does not free enough (3 + 4 + 6 + 4 > 12) until J0 finishes
    assert all(r[0] >= res.stats[0].completion_tick for r in ev)


def test_evict_requires_srtf():
    jobs = [_job(0, 0, 1, 1, 1, 1)]
    for pol in (S.FIFO, S.PACK, S.FAIR):
        with pytest.raises(ValueError):
            S.simulate(jobs, 10 * G, pol, evict=True)


def test_no_pressure_same_as_plain_srtf():
    rng = np.random.default_rng(31)
    for _ in range(30):
        jobs, _ = random_sched_trace(rng, 8, cap_pages=40, infer_frac=0.3)
        C = 100000 * G                       # every job fits beside every other
        a = S.simulate(jobs, C, S.SRTF, evict=True).log_bytes()
        assert a == S.simulate(jobs, C, S.SRTF).log_bytes()


@pytest.mark.parametrize("max_lanes", [1, 2, 4])
def test_random_eviction_properties(max_lanes):
    rng = np.random.default_rng(700 + max_lanes)
    n_evicts = 0
    for trial in range(120):
        jobs, C = random_sched_trace(rng, int(rng.integers(2, 12)), cap_pages=int(rng.integers(8, 40)),
                                     infer_frac=0.2, max_iters=8)
        J = {j.job_id: j for j in jobs}
        res = S.simulate(jobs, C, S.SRTF, max_lanes=max_lanes, evict=True, check_invariants=True)
        Cp = C // G
        # the safety condition from the log alone (I1) with EVICT / RESTORE
        lanes, Pj, sumP = {}, {}, 0
        n_disp = {j: 0 for j in J}
        busy_until = {}                              # job -> end of its latest dispatch
        admitted_once = set()
        evicted_at = {}
        evicted_now = set()                          # victims since the last admission
        for (t, kind, lane, job, a, b) in res.log:
            if kind == LG.LANE_OPEN:
                lanes[lane] = a
            elif kind in (LG.LANE_RESIZE, LG.LANE_SHRINK):
                assert lanes[lane] == b
                lanes[lane] = a
            elif kind == LG.LANE_CLOSE:
                del lanes[lane]
            elif kind in (LG.JOB_ADMIT, LG.JOB_RESTORE):
                assert (kind == LG.JOB_RESTORE) == (job in admitted_once)
                assert evicted_at.get(job) != t          # not restored in its eviction pass
                admitted_once.add(job)
                Pj[job] = a
                sumP += a
                assert b <= lanes[lane]
                # every job evicted at this tick has lower priority than the admitted one
                for v, tv in evicted_at.items():
                    if tv == t and v in evicted_now:
                        rv = ((J[v].n_iters - n_disp[v]) * J[v].iter_ticks, J[v].arrival_tick, v)
                        rj = ((J[job].n_iters - n_disp[job]) * J[job].iter_ticks, J[job].arrival_tick, job)
                        assert rv > rj, (t, v, job)
                evicted_now.clear()
            elif kind == LG.JOB_EVICT:
                assert busy_until.get(job, -1) <= t      # only at an iteration boundary
                assert b == n_disp[job]                  # progress kept
                sumP -= Pj.pop(job)
                evicted_at[job] = t
                evicted_now.add(job)
                n_evicts += 1
            elif kind == LG.JOB_FINISH:
                sumP -= Pj.pop(job)
            elif kind == LG.DISPATCH:
                assert a == n_disp[job]                  # iterations continue in order
                n_disp[job] += 1
                busy_until[job] = t + J[job].iter_ticks
            assert sumP + sum(lanes.values()) <= Cp
        assert not lanes and sumP == 0
        assert all(n_disp[j] == J[j].n_iters for j in J)
    assert n_evicts > 20, n_evicts          # the traces do exercise eviction
