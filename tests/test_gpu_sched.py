"""GPU schedule parity: the device-resident scheduler (CTA 0 of the
persistent kernel) must reproduce the oracle's canonical log byte for byte
on every config and policy (north star: bit-exact schedules)."""
import numpy as np
import pytest

from oracle import scheduler as OS
from workloads import (c1_trace, c1_tie_trace, c2_trace, c3_trace, c4_trace, c5_trace,
                       random_sched_trace)

from gpu_helpers import assert_schedule_parity

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("policy", [OS.FIFO, OS.SRTF, OS.PACK, OS.FAIR])
def test_c1(policy):
    jobs, cap = c1_trace()
    ctx, ref, stats = assert_schedule_parity(jobs, cap, policy)
    ctx.close()
    jobs, cap = c1_tie_trace()
    assert_schedule_parity(jobs, cap, policy)[0].close()


@pytest.mark.parametrize("policy", [OS.FIFO, OS.PACK])
def test_c2_sweep(policy):
    jobs, cap = c2_trace("a")
    assert_schedule_parity(jobs, cap, policy)[0].close()


@pytest.mark.parametrize("policy,max_lanes", [(OS.PACK, 0), (OS.FAIR, 8), (OS.FAIR, 1), (OS.SRTF, 4)])
def test_c3_inference(policy, max_lanes):
    jobs, cap = c3_trace()
    assert_schedule_parity(jobs, cap, policy, max_lanes=max_lanes)[0].close()


@pytest.mark.parametrize("policy,max_lanes", [(OS.FAIR, 8), (OS.PACK, 0)])
def test_c3_real_work_wall_stamps(policy, max_lanes):
    """C3 with every request executing (the bench's switch-latency config):
    schedule parity, and physically consistent wall stamps -- a lane starts
    an iteration only after the scheduler appended its record and after the
    lane's previous iteration ended (run-ahead, A30)."""
    jobs, cap = c3_trace()
    ctx, ref, stats = assert_schedule_parity(jobs, cap, policy, max_lanes=max_lanes, null_work=False)
    try:
        w = ctx.wall()
        rs = ctx.run_stats()
        assert len(w) == rs["n_dispatch"] == 8400
        assert np.all(w["end_ns"] > w["start_ns"])
        assert np.all(w["append_ns"] <= w["start_ns"])
        w = w[np.argsort(w["seq"])]
        for ln in np.unique(w["lane"]):
            m = w[w["lane"] == ln]
            assert np.all(m["start_ns"][1:] >= m["end_ns"][:-1])
        assert rs["sched_fence_ns"] + rs["sched_ring_ns"] <= rs["sched_wait_ns"]
    finally:
        ctx.close()


@pytest.mark.parametrize("policy", [OS.FIFO, OS.SRTF, OS.PACK, OS.FAIR])
def test_c4_mixed(policy):
    jobs, cap = c4_trace()
    assert_schedule_parity(jobs, cap, policy, switch_ticks=1000)[0].close()


def test_c5_2000_jobs_pack():
    jobs, cap = c5_trace()
    assert_schedule_parity(jobs, cap, OS.PACK)[0].close()


@pytest.mark.parametrize("policy", [OS.FIFO, OS.SRTF, OS.PACK, OS.FAIR])
def test_random_traces(policy):
    rng = np.random.default_rng(1000 + policy)
    for trial in range(12):
        jobs, cap = random_sched_trace(rng, int(rng.integers(1, 40)), cap_pages=int(rng.integers(8, 120)),
                                       infer_frac=0.3)
        ml = int(rng.integers(1, 9)) if policy != OS.FIFO else 0
        assert_schedule_parity(jobs, cap, policy, max_lanes=ml,
                               switch_ticks=int(rng.integers(0, 3)), check=True)[0].close()


def test_fair_a28_hand_trace():
    """The hand-worked FAIR trace pinning A28 (tests/golden/hand_traces.json
    HW_FAIR_A28): the device scheduler's log equals the oracle's, whose
    dispatches tests/test_oracle_sched.py holds to the hand-worked ones."""
    import os
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from test_oracle_sched import _gold, fair_a28_jobs
    from workloads import PAGE_BYTES
    want = _gold("hand_traces.json")["HW_FAIR_A28"]["dispatch"]
    for real in (False, True):
        ctx, ref, stats = assert_schedule_parity(fair_a28_jobs(real), 64 * PAGE_BYTES, OS.FAIR,
                                                 null_work=not real, check=True)
        ctx.close()
        assert [[t, job, it] for seq, t, lane, job, it, end in ref.dispatch] == want


@pytest.mark.parametrize("policy", [OS.PACK, OS.SRTF])
def test_i4_page_reuse_waits_for_the_previous_owner(policy):
    """SURVEY §8(c) I4 from the GPU's own stamps: every page the pool hands to
    a lane while the page's previous user (another lane slot) still had a
    record queued is used only by records that start after that record
    ended.  C4 with real work (run-ahead: the scheduler is far ahead of the
    workers, so hand-offs with pending fences occur), SALUS_FLAG_CHECK."""
    import numpy as np
    jobs, cap = c4_trace()
    ctx, ref, stats = assert_schedule_parity(jobs, cap, policy, null_work=False, check=True, timeout_ms=300000)
    try:
        h = ctx.handoffs()
        w = ctx.wall()
    finally:
        ctx.close()
    assert len(h) > 0                                   # the trace does exercise fenced reuse
    end = {int(s): int(e) for s, e in zip(w["seq"], w["end_ns"])}
    order = np.argsort(w["seq"])
    seqs, lanes, starts = w["seq"][order].astype(np.int64), w["lane"][order], w["start_ns"][order].astype(np.int64)
    pairs = {(int(a), int(b), int(c)) for a, b, c in zip(h["to_lane"], h["from_seq"], h["to_seq"])}
    checked = 0
    for to_lane, from_seq, to_seq in pairs:
        later = (lanes == to_lane) & (seqs >= to_seq)
        if later.any():
            first = starts[later].min()
            assert first >= end[from_seq], (to_lane, from_seq, to_seq, first - end[from_seq])
            checked += 1
    assert checked > 0
