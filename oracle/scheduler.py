"""ORACLE — test infrastructure only.  Salus lane assignment + iteration
scheduling as a plain discrete-event loop in integer logical ticks.

Follows PAPER.md (LaTeX source of arXiv 1902.04610):
  * Algorithm 1 "GPU Lane Assignment"  P:415-477 (JobArrive, JobFinish,
    LaneMoved, ProcessRequests, FindLane)
  * the safety condition
      sum_jobs P_i + sum_lanes L_j <= C,   L_j = max_{i in j} E_i
  * "event-driven and reacts when there are jobs arriving or finishing, or at
    iteration boundaries"
  * iteration-granularity switching    P:353-354 (§3.2.2)
  * lanes: execution serialised within a lane, parallel across lanes P:371-373
  * policies FIFO, PACK, SRTF,
    FAIR
with the readings A1..A30 of SURVEY.md §8(c), restated in DESIGN.md
("Readings of the paper").  The ones this file implements are cited inline.

Units: sizes in pages (A18: p = ceil(P/G), e = ceil(E/G), Cp = floor(C/G));
time in int64 logical ticks (A17).  Nothing here touches floating point.
"""
from __future__ import annotations

import dataclasses
from typing import Dict, List, Optional, Sequence, Tuple

from . import logfmt as LG

FIFO, SRTF, PACK, FAIR = 0, 1, 2, 3
POLICY_NAMES = {FIFO: "fifo", SRTF: "srtf", PACK: "pack", FAIR: "fair"}
# A9: lanes per policy.  FIFO holds one job at a time; SRTF and FAIR use a
# single lane ("we consider a single GPU lane"); PACK up to the table.
DEFAULT_MAX_LANES = {FIFO: 1, SRTF: 1, PACK: 64, FAIR: 1}
MAX_LANES = 64

NOT_ARRIVED, QUEUED, ADMITTED, DONE, SWAPPED = 0, 1, 2, 3, 4
TRAIN, INFER = 0, 1


class Unschedulable(ValueError):
    """P_i + E_i > C after page rounding: rejected at submit (A22)."""


class Stuck(RuntimeError):
    """No event remains while jobs are unfinished."""


def pages_ceil(nbytes: int, G: int) -> int:
    return -(-int(nbytes) // G)


# --------------------------------------------------------------------------
# Algorithm 1, FindLane
# --------------------------------------------------------------------------

def find_lane(sumP: int, lanes: Sequence[Tuple[int, int]], p: int, e: int, Cp: int,
              max_lanes: int):
    """FindLane(P, E) of Algorithm 1.

    `lanes` = [(lane_id, L_j)] of existing lanes.  Returns None ("return not
    found") or (branch, lane_id, new_L) with branch in
    {"new", "reuse", "resize"}; lane_id is None for "new".

      S = sum_i P_i + sum_j L_j
      1. "Try to create a new lane": S + P + E <= C, and fewer
         than max_lanes lanes exist (A9).
      2. "Try to put into an existing lane": L_j >= E "and is the
         best match".  A1: the safety condition is checked here too
         (S + P <= C), because P:479 says it "is always kept".  A2: best
         match = smallest L_j >= E, ties to the lowest lane id.
      3. "Try to replace an existing lane": for r in ascending
         L_r, if S + P - L_r + E <= C then L_r <- E.  A3: only lanes with
         L_r < E qualify (L_r <- E must not shrink an occupied lane below its
         residents' E); ties in L_r go to the lowest id.
    """
    S = sumP + sum(L for _, L in lanes)
    if len(lanes) < max_lanes and S + p + e <= Cp:                 # branch 1
        return ("new", None, e)
    if S + p <= Cp:                                                 # branch 2
        best = None
        for lid, L in lanes:
            if L >= e and (best is None or (L, lid) < best):
                best = (L, lid)
        if best is not None:
            return ("reuse", best[1], best[0])
    for L, lid in sorted((L, lid) for lid, L in lanes if L < e):    # branch 3
        if S - L + p + e <= Cp:
            return ("resize", lid, e)
    return None


def safety_ok(sumP: int, lane_sizes: Sequence[int], Cp: int) -> bool:
    """The safety condition: sum P_i + sum L_j <= C."""
    return sumP + sum(lane_sizes) <= Cp


# --------------------------------------------------------------------------
# The event loop
# --------------------------------------------------------------------------

@dataclasses.dataclass
class _Lane:
    id: int
    L: int
    residents: List[int]
    busy_until: Optional[int] = None     # None == idle
    cur: Optional[int] = None
    last: Optional[int] = None


@dataclasses.dataclass
class JobStat:
    job_id: int
    first_lane: int
    admit_tick: int
    first_start_tick: int
    completion_tick: int
    completion_seq: int


@dataclasses.dataclass
class SimResult:
    log: List[tuple]                 # canonical records (logfmt.REC fields)
    stats: Dict[int, JobStat]
    dispatch: List[tuple]            # (seq, tick, lane, job, iter, end_tick)
    n_ticks: int

    def log_bytes(self) -> bytes:
        return LG.encode(self.log)


def _admission_key(policy, job, c, done=0):
    # A10: SRTF orders the pending queue by remaining time (n - done)*c (n*c
    # for a job that has not run yet; A35: a swapped-out job keeps its
    # progress); A13/A14: the others by arrival.  Ties: (arrival, id).
    if policy == SRTF:
        return ((job.n_iters - done) * c, job.arrival_tick, job.job_id)
    return (job.arrival_tick, job.job_id)


def simulate(jobs, capacity_bytes: int, policy: int, *, page_bytes: int = 65536,
             max_lanes: int = 0, switch_ticks: int = 0, literal: bool = False,
             check_invariants: bool = False, evict: bool = False) -> SimResult:
    """Run the whole trace.  Tick phases (A15):

      t  = min(busy_until of busy lanes, next arrival, next pending request)
      P1 completions (lane id asc): iteration ends; JobFinish
      P2 arrivals ((arrival, id) asc): JobArrive appends to Q;
         inference requests arriving at t become pending (A27)
      P3 ProcessRequests over Q, one in-order pass (A5, A7, A8)
      P4 dispatch: every idle lane picks its next iteration

    `literal=True` runs P3 at every tick with a non-empty Q (A5 as written).
    The default runs it only on ticks where a job arrived or finished: the
    only events that change what FindLane can return (one pass is a fixpoint,
    A8); tests check the two modes produce identical logs.

    `evict=True` (SRTF only, reading A35 of DESIGN.md):
    "the higher priority job is admitted as long as its own safety condition
    is met -- i.e., at least, it can run alone on the GPU -- regardless of
    other already-running jobs".  When FindLane fails for a queued
    job j, admitted jobs of strictly lower priority (larger
    ((n-done)*c, arrival, id)) that are not mid-iteration are swapped out,
    lowest priority first, until FindLane succeeds; if it cannot succeed,
    nobody is evicted.  A victim leaves its lane (JobFinish's lane update,
    A4), its P pages are freed, and it joins Q after the pass (SWAPPED) with
    its progress kept; re-admission logs JOB_RESTORE.  Admission runs at
    every tick with a non-empty Q (an iteration end makes its job
    evictable).  Swap time is not modelled in logical ticks (like A16).
    """
    if evict and policy != SRTF:
        raise ValueError("evict applies to SRTF only")
    G = int(page_bytes)
    Cp = int(capacity_bytes) // G
    if max_lanes <= 0:
        max_lanes = DEFAULT_MAX_LANES[policy]
    max_lanes = min(max_lanes, MAX_LANES)

    J: Dict[int, object] = {}
    for j in jobs:
        if j.job_id in J:
            raise ValueError(f"duplicate job id {j.job_id}")
        if j.n_iters < 1 or j.iter_ticks < 1:
            raise ValueError(f"job {j.job_id}: n_iters and iter_ticks must be >= 1")
        if j.kind == INFER:
            rt = list(j.request_ticks)
            if len(rt) != j.n_iters or rt != sorted(rt) or (rt and rt[0] < j.arrival_tick):
                raise ValueError(f"job {j.job_id}: bad request ticks")
        J[j.job_id] = j
    p = {jid: pages_ceil(j.persistent_bytes, G) for jid, j in J.items()}
    e = {jid: pages_ceil(j.ephemeral_bytes, G) for jid, j in J.items()}
    c = {jid: j.iter_ticks for jid, j in J.items()}
    for jid in J:
        if p[jid] + e[jid] > Cp:                     # A22 / S:138
            raise Unschedulable(f"job {jid}: p+e={p[jid] + e[jid]} > C={Cp} pages")

    st = {jid: NOT_ARRIVED for jid in J}
    done = {jid: 0 for jid in J}
    svc = {jid: 0 for jid in J}
    pending = {jid: 0 for jid in J}
    next_req = {jid: 0 for jid in J}
    lane_of: Dict[int, int] = {}
    first_lane: Dict[int, int] = {}
    first_start: Dict[int, int] = {}
    admit_tick: Dict[int, int] = {}
    last_seq: Dict[int, int] = {}
    stats: Dict[int, JobStat] = {}

    by_arrival = sorted(J.values(), key=lambda j: (j.arrival_tick, j.job_id))
    # inference jobs are visited in (arrival, id) order, like every other tie (A15)
    infer_ids = [j.job_id for j in by_arrival if j.kind == INFER]
    arr_ptr = 0
    lanes: List[_Lane] = []          # kept in lane-id order
    lane_by_id: Dict[int, _Lane] = {}
    Q: List[int] = []
    sumP = 0
    seq = 0
    next_lane = 0
    n_done = 0
    n_ticks = 0
    log: List[tuple] = []
    dispatch: List[tuple] = []
    dirty = False

    def runnable(jid):
        return J[jid].kind == TRAIN or pending[jid] > 0

    def invariants(where):
        # I1 safety, I2 L_j = max E_i over residents, I5 monotone ids.
        assert safety_ok(sumP, [ln.L for ln in lanes], Cp), (where, sumP, [ln.L for ln in lanes])
        for ln in lanes:
            assert ln.residents, where
            assert ln.L == max(e[r] for r in ln.residents), (where, ln)
        ids = [ln.id for ln in lanes]
        assert ids == sorted(ids) and len(set(ids)) == len(ids)
        assert sumP == sum(p[r] for ln in lanes for r in ln.residents)

    def prio(jid):
        return _admission_key(policy, J[jid], c[jid], done[jid])

    def lane_left(t, ln, jid):
        """`jid` left lane `ln` (JobFinish or eviction): delete the lane if
        ref(lane) == 0, else L = max E of the residents (A4)."""
        if not ln.residents:
            lanes.remove(ln)
            del lane_by_id[ln.id]
            log.append((t, LG.LANE_CLOSE, ln.id, jid, 0, 0))
        else:
            newL = max(e[r] for r in ln.residents)
            if newL < ln.L:
                log.append((t, LG.LANE_SHRINK, ln.id, jid, newL, ln.L))
                ln.L = newL

    def evict_for(t, jid, evicted):
        """A35: swap out lower-priority idle residents, lowest priority
        first, until FindLane(p_j, e_j) succeeds; all or nothing."""
        nonlocal sumP
        kj = prio(jid)
        cands = [v for ln in lanes for v in ln.residents
                 if prio(v) > kj and not (ln.busy_until is not None and ln.cur == v)]
        cands.sort(key=prio, reverse=True)
        hres = {ln.id: list(ln.residents) for ln in lanes}
        hP = sumP
        chosen = []
        for v in cands:
            chosen.append(v)
            hP -= p[v]
            hres[lane_of[v]].remove(v)
            hl = [(ln.id, max(e[r] for r in hres[ln.id])) for ln in lanes if hres[ln.id]]
            if find_lane(hP, hl, p[jid], e[jid], Cp, max_lanes) is not None:
                break
        else:
            return None
        for v in chosen:
            ln = lane_by_id[lane_of[v]]
            st[v] = SWAPPED
            sumP -= p[v]
            ln.residents.remove(v)
            log.append((t, LG.JOB_EVICT, ln.id, v, p[v], done[v]))
            lane_left(t, ln, v)
            evicted.append(v)
        return find_lane(sumP, [(ln.id, ln.L) for ln in lanes], p[jid], e[jid], Cp, max_lanes)

    def admission_pass(t, dry=False):
        nonlocal sumP, next_lane
        admitted = 0
        order = sorted(Q, key=prio)
        busy_job = any(st[x] == ADMITTED for x in J) if policy == FIFO else False
        evicted: List[int] = []
        for jid in order:
            if policy == FIFO and busy_job:          # A14: exclusive GPU, strict HOL
                break
            d = find_lane(sumP, [(ln.id, ln.L) for ln in lanes], p[jid], e[jid], Cp, max_lanes)
            if d is None and evict and not dry:
                d = evict_for(t, jid, evicted)
            if d is None:
                if policy == FIFO:
                    break
                continue                              # A7: no HOL inside the pass
            if dry:
                admitted += 1
                break
            branch, lid, newL = d
            if branch == "new":
                ln = _Lane(next_lane, e[jid], [])
                next_lane += 1
                lanes.append(ln)
                lane_by_id[ln.id] = ln
                log.append((t, LG.LANE_OPEN, ln.id, jid, ln.L, 0))
            elif branch == "reuse":
                ln = lane_by_id[lid]
                log.append((t, LG.LANE_REUSE, ln.id, jid, ln.L, 0))
            else:
                ln = lane_by_id[lid]
                old = ln.L
                ln.L = newL
                log.append((t, LG.LANE_RESIZE, ln.id, jid, newL, old))
            # A12: FAIR newcomer starts at the min service of the lane's other
            # unfinished residents (virtual time), else 0.
            if policy == FAIR:
                svc[jid] = min((svc[r] for r in ln.residents), default=0)
            ln.residents.append(jid)
            sumP += p[jid]
            restored = st[jid] == SWAPPED
            st[jid] = ADMITTED
            admit_tick.setdefault(jid, t)
            first_lane.setdefault(jid, ln.id)
            lane_of[jid] = ln.id
            log.append((t, LG.JOB_RESTORE if restored else LG.JOB_ADMIT, ln.id, jid, p[jid], e[jid]))
            Q.remove(jid)
            admitted += 1
            busy_job = True
        Q.extend(evicted)                             # A35: victims queue after the pass
        return admitted

    while n_done < len(J):
        # ---- next event time (A4 of §8(a)) --------------------------------
        cand = [ln.busy_until for ln in lanes if ln.busy_until is not None]
        if arr_ptr < len(by_arrival):
            cand.append(by_arrival[arr_ptr].arrival_tick)
        for jid in infer_ids:
            if st[jid] in (QUEUED, ADMITTED, SWAPPED) and next_req[jid] < J[jid].n_iters:
                cand.append(J[jid].request_ticks[next_req[jid]])
        if not cand:
            raise Stuck(f"no event left with {len(J) - n_done} jobs unfinished")
        t = min(cand)
        n_ticks += 1
        dirty = False

        # ---- P1: iteration completions, JobFinish -------------
        for ln in list(lanes):
            if ln.busy_until != t:
                continue
            jid = ln.cur
            done[jid] += 1
            svc[jid] += c[jid]
            ln.busy_until = None
            if done[jid] == J[jid].n_iters:
                st[jid] = DONE
                n_done += 1
                dirty = True
                sumP -= p[jid]
                ln.residents.remove(jid)
                stats[jid] = JobStat(jid, first_lane[jid], admit_tick[jid], first_start[jid], t,
                                     last_seq[jid])
                log.append((t, LG.JOB_FINISH, ln.id, jid, done[jid], last_seq[jid]))
                lane_left(t, ln, jid)
        if check_invariants:
            invariants("P1")

        # ---- P2: arrivals (JobArrive) and inference requests ---
        while arr_ptr < len(by_arrival) and by_arrival[arr_ptr].arrival_tick == t:
            jid = by_arrival[arr_ptr].job_id
            arr_ptr += 1
            st[jid] = QUEUED
            Q.append(jid)
            log.append((t, LG.JOB_QUEUED, LG.NONE32, jid, 0, 0))
            dirty = True
        for jid in infer_ids:
            if st[jid] not in (QUEUED, ADMITTED, SWAPPED):
                continue
            rt = J[jid].request_ticks
            k = 0
            while next_req[jid] < len(rt) and rt[next_req[jid]] == t:
                next_req[jid] += 1
                k += 1
            if k == 0:
                continue
            was_idle = pending[jid] == 0
            pending[jid] += k
            if policy == FAIR and st[jid] == ADMITTED and was_idle:
                ln = lane_by_id[lane_of[jid]]
                running = ln.busy_until is not None and ln.cur == jid
                if not running:
                    # A28: an idle inference job re-enters at the min service
                    # of its lane's runnable co-residents.
                    co = [svc[r] for r in ln.residents if r != jid and runnable(r)]
                    if co:
                        svc[jid] = max(svc[jid], min(co))

        # ---- P3: ProcessRequests ------------------------------
        if Q and (dirty or literal or evict):
            admission_pass(t)
        if check_invariants:
            invariants("P3")
            if Q and not evict:
                assert admission_pass(t, dry=True) == 0, "I7: second pass admitted a job"
            if Q and evict:
                # I8: the highest-priority queued job is admitted
                # "regardless of other already-running jobs" once every
                # admitted job has lower priority and none is mid-iteration.
                top = min(Q, key=prio)
                adm = [r for ln in lanes for r in ln.residents]
                busy = any(ln.busy_until is not None for ln in lanes)
                assert not (all(prio(r) > prio(top) for r in adm) and not busy), ("I8", t, top)

        # ---- P4: dispatch at iteration boundaries ----
        for ln in lanes:
            if ln.busy_until is not None:
                continue
            R = [r for r in ln.residents if runnable(r)]
            if not R:
                continue
            if policy == SRTF:       # A11: remaining = (n - done) * c
                key = lambda r: ((J[r].n_iters - done[r]) * c[r], J[r].arrival_tick, r)
            elif policy == FAIR:     # P:537 equalise total service
                key = lambda r: (svc[r], J[r].arrival_tick, r)
            else:                    # FIFO / PACK (A13): earliest arrival
                key = lambda r: (J[r].arrival_tick, r)
            jid = min(R, key=key)
            pen = switch_ticks if (ln.last is not None and ln.last != jid) else 0   # A16
            ln.busy_until = t + pen + c[jid]
            ln.cur = jid
            ln.last = jid
            if J[jid].kind == INFER:
                pending[jid] -= 1
            first_start.setdefault(jid, t)
            last_seq[jid] = seq
            log.append((t, LG.DISPATCH, ln.id, jid, done[jid], seq))
            dispatch.append((seq, t, ln.id, jid, done[jid], ln.busy_until))
            seq += 1

    return SimResult(log=log, stats=stats, dispatch=dispatch, n_ticks=n_ticks)
