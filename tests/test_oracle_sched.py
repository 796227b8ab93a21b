"""Pins for the oracle scheduler (oracle/scheduler.py) against what the paper
and mathematics fix: hand-worked traces, FIFO's closed form, brute-force
optimality of SRTF on its optimality classes, FAIR's service bound, the
safety condition recomputed from the log alone, and exhaustive FindLane.
"""
import functools
import itertools
import json
import os

import numpy as np
import pytest

from oracle import logfmt as LG
from oracle import metrics as M
from oracle import scheduler as S
from workloads import PAGE_BYTES, TRAIN, INFER, make_job, c1_trace, random_sched_trace

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def single_lane_jobs(spec):
    """[(arrival, n, c)] -> tiny jobs that all fit in one lane."""
    G = PAGE_BYTES
    return [make_job(j, TRAIN, a, (128, 128), 128, n, iter_ticks=c,
                     persistent_bytes=G, ephemeral_bytes=G) for j, (a, n, c) in enumerate(spec)]


def jcts(jobs, res):
    return [res.stats[j.job_id].completion_tick - j.arrival_tick for j in jobs]


def runs(res):
    """Collapse consecutive dispatches of a job into [job, start, end] runs."""
    out = []
    for seq, t, lane, job, it, end in res.dispatch:
        if out and out[-1][0] == job and out[-1][2] == t:
            out[-1][2] = end
        else:
            out.append([job, t, end])
    return out


# ---------------------------------------------------------------- FindLane

def test_algorithm1_examples():
    for case in _gold("algorithm1_examples.json")["cases"]:
        got = S.find_lane(case["sumP"], [tuple(x) for x in case["lanes"]], case["p"], case["e"],
                          case["Cp"], case["max_lanes"])
        exp = case["expect"]
        assert (got is None if exp is None else list(got) == exp), case["_cite"]


def _brute_find_lane(sumP, lanes, p, e, Cp, max_lanes):
    """Independent evaluator: enumerate every candidate post-state, keep the
    ones that satisfy the safety condition sum P + sum L <= C with
    L_j >= E_i for the lane the job joins, then apply the
    paper's preference order new > existing (best match) > replace."""
    def safe(P, Ls):
        return P + sum(Ls) <= Cp
    Ls = [L for _, L in lanes]
    if len(lanes) < max_lanes and safe(sumP + p, Ls + [e]):
        return ("new", None, e)
    reuse = [(L, lid) for lid, L in lanes if L >= e and safe(sumP + p, Ls)]
    if reuse:
        L, lid = min(reuse)
        return ("reuse", lid, L)
    repl = []
    for i, (lid, L) in enumerate(lanes):
        if L < e:
            post = Ls[:i] + [e] + Ls[i + 1:]
            if safe(sumP + p, post):
                repl.append((L, lid))
    if repl:
        L, lid = min(repl)
        return ("resize", lid, e)
    return None


def test_find_lane_exhaustive():
    """every state with <= 3 lanes on a quantised grid."""
    n = 0
    for Cp in range(0, 9):
        for nl in range(0, 4):
            for sizes in itertools.product(range(0, 5), repeat=nl):
                lanes = list(enumerate(sizes))
                for sumP in range(0, 5):
                    if sumP + sum(sizes) > Cp:
                        continue            # only reachable (safe) states
                    for p in range(1, 4):
                        for e in range(0, 6):
                            for ml in (1, 2, 64):
                                a = S.find_lane(sumP, lanes, p, e, Cp, ml)
                                b = _brute_find_lane(sumP, lanes, p, e, Cp, ml)
                                assert a == b, (Cp, lanes, sumP, p, e, ml, a, b)
                                n += 1
    assert n > 10000


# ----------------------------------------------------------- hand traces

def test_hw_c1():
    g = _gold("hand_traces.json")["HW_C1"]
    jobs, C = c1_trace()
    fifo = S.simulate(jobs, C, S.FIFO, check_invariants=True)
    srtf = S.simulate(jobs, C, S.SRTF, check_invariants=True)
    assert jcts(jobs, fifo) == g["fifo_jct"]
    assert [fifo.stats[i].completion_seq for i in (0, 1)] == g["fifo_completion_seq"]
    assert [fifo.stats[i].first_lane for i in (0, 1)] == g["fifo_lanes"]
    assert jcts(jobs, srtf) == g["srtf_jct"]
    assert [srtf.stats[i].completion_seq for i in (0, 1)] == g["srtf_completion_seq"]
    assert [srtf.stats[i].first_lane for i in (0, 1)] == g["srtf_lanes"]
    assert [d[3] for d in srtf.dispatch] == g["srtf_dispatch_jobs"]
    # J1 joins J0's lane via branch 2 (reuse), never opening a second lane
    assert any(r[1] == LG.LANE_REUSE and r[3] == 1 for r in srtf.log)
    # 1.60x avg-JCT ratio of the hand trace
    assert M.summarize(jobs, fifo.stats)["avg_jct"] == 82500
    assert M.summarize(jobs, srtf.stats)["avg_jct"] == 51500


@pytest.mark.parametrize("name", ["HW2", "HW3b"])
def test_hw_fifo_srtf(name):
    g = _gold("hand_traces.json")[name]
    jobs = single_lane_jobs(g["jobs"])
    C = 64 * PAGE_BYTES
    assert jcts(jobs, S.simulate(jobs, C, S.FIFO)) == g["fifo_jct"]
    assert jcts(jobs, S.simulate(jobs, C, S.SRTF)) == g["srtf_jct"]
    assert sum(g["srtf_jct"]) >= g["optimum_sum_jct"]
    assert _brute_opt(tuple(tuple(x) for x in g["jobs"])) == g["optimum_sum_jct"]


def test_hw3a_srtf_not_optimal():
    g = _gold("hand_traces.json")["HW3a"]
    jobs = single_lane_jobs(g["jobs"])
    assert sum(jcts(jobs, S.simulate(jobs, 64 * PAGE_BYTES, S.SRTF))) == g["srtf_sum_jct"]
    assert _brute_opt(tuple(tuple(x) for x in g["jobs"])) == g["optimum_sum_jct"]


def test_srtf_episode_fig_srtf_compute():
    """#1 preempts #0; #3 before the earlier #2; #5 preempts #4;
    #0 runs only when alone."""
    g = _gold("hand_traces.json")["HW_EP"]
    jobs = single_lane_jobs(g["jobs"])
    res = S.simulate(jobs, 64 * PAGE_BYTES, S.SRTF, check_invariants=True)
    assert runs(res) == g["srtf_runs"]
    assert {str(k): v.completion_tick for k, v in res.stats.items()} == g["srtf_completion"]


# ---------------------------------------------------- FIFO closed form (T4)

@pytest.mark.parametrize("seed", range(20))
def test_fifo_closed_form(seed):
    rng = np.random.default_rng(seed)
    jobs, C = random_sched_trace(rng, int(rng.integers(1, 12)), cap_pages=40)
    res = S.simulate(jobs, C, S.FIFO, check_invariants=True)
    order = sorted(jobs, key=lambda j: (j.arrival_tick, j.job_id))
    prev = None
    for j in order:                       # C_k = max(a_k, C_{k-1}) + n_k c_k
        start = j.arrival_tick if prev is None else max(j.arrival_tick, prev)
        prev = start + j.n_iters * j.iter_ticks
        assert res.stats[j.job_id].completion_tick == prev
        assert res.stats[j.job_id].first_start_tick == start
    comp = [res.stats[j.job_id].completion_seq for j in order]
    assert comp == sorted(comp)           # completion order == arrival order


# --------------------------------------------- SRTF vs brute force (T5)

@functools.lru_cache(maxsize=None)
def _brute_opt(spec):
    """Min sum of completion-minus-arrival over every iteration-granular
    single-lane schedule (including idling until an arrival)."""
    arr = [a for a, n, c in spec]

    @functools.lru_cache(maxsize=None)
    def go(t, rem):
        if all(r == 0 for r in rem):
            return 0
        best = None
        for j, (a, n, c) in enumerate(spec):
            if rem[j] > 0 and a <= t:
                r2 = list(rem)
                r2[j] -= 1
                cost = (t + c - a) if r2[j] == 0 else 0
                v = cost + go(t + c, tuple(r2))
                best = v if best is None else min(best, v)
        future = [a for j, a in enumerate(arr) if rem[j] > 0 and a > t]
        if future:
            v = go(min(future), rem)
            best = v if best is None else min(best, v)
        return best

    return go(0, tuple(n for a, n, c in spec))


@pytest.mark.parametrize("cls", ["i", "ii"])
def test_srtf_optimal_in_its_class(cls):
    """SRTF = SPT is optimal when all jobs arrive at 0 (class i); with equal
    iteration costs and arrivals on the c-grid it is SRPT for 1|r_j,pmtn|sum C_j
    (class ii).  Brute force over all schedules must agree."""
    rng = np.random.default_rng(11 if cls == "i" else 12)
    for trial in range(150):
        nj = int(rng.integers(1, 5))
        if cls == "i":
            spec = tuple((0, int(rng.integers(1, 4)), int(rng.integers(1, 5))) for _ in range(nj))
        else:
            c = int(rng.integers(1, 4))
            spec = tuple((c * int(rng.integers(0, 5)), int(rng.integers(1, 4)), c) for _ in range(nj))
        jobs = single_lane_jobs(spec)
        res = S.simulate(jobs, 64 * PAGE_BYTES, S.SRTF)
        assert sum(jcts(jobs, res)) == _brute_opt(spec), spec


# --------------------------------------------------------------- FAIR (T6)

def test_fair_equal_service():
    """three identical jobs starting at 0/15/30 -- each job's
    share is halved, then reduces to about a third; service gap between
    co-resident jobs never exceeds one iteration."""
    jobs = single_lane_jobs([(0, 40, 1), (15, 40, 1), (30, 40, 1)])
    res = S.simulate(jobs, 64 * PAGE_BYTES, S.FAIR, check_invariants=True)
    # for every pair, service received from the later arrival onwards stays
    # within one iteration while both are unfinished
    for a, b in ((0, 1), (0, 2), (1, 2)):
        t0 = max(jobs[a].arrival_tick, jobs[b].arrival_tick)
        t1 = min(res.stats[a].completion_tick, res.stats[b].completion_tick)
        got = {a: 0, b: 0}
        for seq, t, lane, job, it, end in res.dispatch:
            if t0 <= t < t1 and job in got:
                got[job] += 1
                assert abs(got[a] - got[b]) <= 1, (a, b, t, got)
    # window [15, 30): two jobs -> 1/2 each; [30, ...) three jobs -> 1/3 each
    w2 = [d[3] for d in res.dispatch if 16 <= d[1] < 30]
    assert abs(w2.count(0) - w2.count(1)) <= 1
    w3 = [d[3] for d in res.dispatch if 31 <= d[1] < 61]
    for j in (0, 1, 2):
        assert abs(w3.count(j) - 10) <= 1


def test_fair_newcomer_virtual_time():
    """A12: a newcomer starts at the lane's min service, so it does not
    monopolise the lane on arrival ('each job's share is halved')."""
    jobs = single_lane_jobs([(0, 50, 1), (20, 50, 1)])
    res = S.simulate(jobs, 64 * PAGE_BYTES, S.FAIR)
    after = [d[3] for d in res.dispatch if 20 <= d[1] < 30]
    assert 4 <= after.count(1) <= 6


# ------------------------------------------ invariants on random traces

def _replay_safety(log, Cp):
    """Recompute sum P + sum L from the log alone (independent of the
    oracle's internal state) and check the safety condition after every
    record (I1), plus lane id monotonicity (I5)."""
    lanes, Pj, sumP, max_id = {}, {}, 0, -1
    for t, kind, lane, job, a, b in log:
        if kind == LG.LANE_OPEN:
            assert lane > max_id
            max_id = lane
            lanes[lane] = a
        elif kind in (LG.LANE_RESIZE, LG.LANE_SHRINK):
            assert lanes[lane] == b
            lanes[lane] = a
        elif kind == LG.LANE_CLOSE:
            del lanes[lane]
        elif kind == LG.JOB_ADMIT:
            Pj[job] = a
            sumP += a
            assert b <= lanes[lane]           # E_i <= L_j of its lane
        elif kind == LG.JOB_FINISH:
            sumP -= Pj.pop(job)
        assert sumP + sum(lanes.values()) <= Cp, (t, kind)
    assert not lanes and sumP == 0


@pytest.mark.parametrize("policy", [S.FIFO, S.SRTF, S.PACK, S.FAIR])
def test_random_traces_invariants(policy):
    rng = np.random.default_rng(100 + policy)
    for trial in range(60):
        jobs, C = random_sched_trace(rng, int(rng.integers(1, 14)), cap_pages=int(rng.integers(8, 80)),
                                     infer_frac=0.3)
        ml = int(rng.integers(1, 6)) if policy != S.FIFO else 0
        res = S.simulate(jobs, C, policy, max_lanes=ml, check_invariants=True,
                         switch_ticks=int(rng.integers(0, 3)))
        _replay_safety(res.log, C // PAGE_BYTES)
        # I6: exactly n dispatches per job, all in one lane; I3: no overlap
        per_job, busy = {}, {}
        for seq, t, lane, job, it, end in res.dispatch:
            per_job.setdefault(job, []).append((lane, it))
            assert busy.get(lane, -1) <= t
            busy[lane] = end
        for j in jobs:
            its = per_job[j.job_id]
            assert [i for _, i in its] == list(range(j.n_iters))
            assert len({ln for ln, _ in its}) == 1
        # inference: the k-th iteration never starts before the k-th request
        for j in jobs:
            if j.kind == INFER:
                starts = [t for seq, t, lane, job, it, end in res.dispatch if job == j.job_id]
                assert all(s >= r for s, r in zip(starts, j.request_ticks))
        # literal A5 (admission pass every tick) gives the identical log
        lit = S.simulate(jobs, C, policy, max_lanes=ml, literal=True,
                         switch_ticks=0)
        fast = S.simulate(jobs, C, policy, max_lanes=ml, switch_ticks=0)
        assert lit.log_bytes() == fast.log_bytes()


def test_determinism():
    rng = np.random.default_rng(5)
    jobs, C = random_sched_trace(rng, 12, infer_frac=0.3)
    a = S.simulate(jobs, C, S.PACK, max_lanes=4).log_bytes()
    b = S.simulate(list(reversed(jobs)), C, S.PACK, max_lanes=4).log_bytes()
    assert a == b


def test_switch_ticks_charged_once_per_change():
    jobs = single_lane_jobs([(0, 3, 2), (0, 3, 2)])
    res = S.simulate(jobs, 64 * PAGE_BYTES, S.FAIR, switch_ticks=5)
    prev = None
    for seq, t, lane, job, it, end in res.dispatch:
        pen = 5 if (prev is not None and prev != job) else 0
        assert end - t == 2 + pen
        prev = job


def test_unschedulable_and_duplicates():
    G = PAGE_BYTES
    j = make_job(0, TRAIN, 0, (128, 128), 128, 1, iter_ticks=1, persistent_bytes=5 * G,
                 ephemeral_bytes=6 * G)
    with pytest.raises(S.Unschedulable):
        S.simulate([j], 10 * G, S.PACK)
    with pytest.raises(ValueError):
        S.simulate([j, j], 100 * G, S.PACK)


def test_zero_ephemeral_job():
    """A21: E = 0 is allowed and still serialises in its lane."""
    G = PAGE_BYTES
    jobs = [make_job(i, TRAIN, 0, (128, 128), 128, 2, iter_ticks=3, persistent_bytes=G,
                     ephemeral_bytes=0) for i in range(3)]
    res = S.simulate(jobs, 4 * G, S.PACK, check_invariants=True)
    assert len({s.first_lane for s in res.stats.values()}) == 3
    assert max(s.completion_tick for s in res.stats.values()) == 6


def test_pack_beats_fifo_makespan_when_memory_allows():
    """packing all-ready jobs shortens the makespan."""
    G = PAGE_BYTES
    jobs = [make_job(i, TRAIN, 0, (128, 128), 128, 5, iter_ticks=10, persistent_bytes=G,
                     ephemeral_bytes=2 * G) for i in range(8)]
    fifo = M.summarize(jobs, S.simulate(jobs, 64 * G, S.FIFO).stats)["makespan"]
    pack = M.summarize(jobs, S.simulate(jobs, 64 * G, S.PACK).stats)["makespan"]
    assert fifo == 400 and pack == 50


def fair_a28_jobs(real_work=False):
    """The hand trace HW_FAIR_A28 (tests/golden/hand_traces.json).  With
    real_work the declared sizes are the device footprints (all still fit
    one lane, so the dispatches are the same)."""
    G = PAGE_BYTES
    spec = _gold("hand_traces.json")["HW_FAIR_A28"]["jobs"]
    sz = {} if real_work else {"persistent_bytes": G, "ephemeral_bytes": G}
    return [make_job(j, TRAIN if kind == "train" else INFER, a, (128, 128), 128, n, iter_ticks=c,
                     request_ticks=tuple(req), **sz)
            for j, (kind, a, n, c, req) in enumerate(spec)]


def test_fair_idle_inference_reentry_a28():
    """A28 pinned by a hand-worked FAIR trace: an inference job that
    went idle re-enters at the min service of its lane's runnable
    co-residents; the golden file lists which mutation of the rule changes
    which dispatch."""
    g = _gold("hand_traces.json")["HW_FAIR_A28"]
    jobs = fair_a28_jobs()
    res = S.simulate(jobs, 64 * PAGE_BYTES, S.FAIR, check_invariants=True)
    assert [[t, job, it] for seq, t, lane, job, it, end in res.dispatch] == g["dispatch"]
    assert {str(k): v.completion_tick for k, v in res.stats.items()} == g["completion"]
    assert {d[2] for d in res.dispatch} == {0}          # one lane for life (A9, I6)
