"""World-size-2 gloo test of the multi-GPU host path:
mod-G partition of the trace, one independent instance per rank, all_gather
of per-job completion records.  The per-rank schedule is computed by the
CPU oracle (no GPU here); the GPU path uses the same host functions."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import scheduler as OS
from paper_1902_04610_b200 import multigpu as MG
from workloads import c4_trace


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        jobs, cap = c4_trace(n_jobs=60, seed=9, burst=True)
        mine = MG.partition_jobs(jobs, world, rank)
        res = OS.simulate(mine, cap, OS.PACK)
        stats = {jid: {"job_id": s.job_id, "first_lane": s.first_lane, "admit_tick": s.admit_tick,
                       "first_start_tick": s.first_start_tick, "completion_tick": s.completion_tick,
                       "completion_seq": s.completion_seq} for jid, s in res.stats.items()}
        merged = MG.gather_stats(stats, rank, world)
        out[rank] = merged
    finally:
        dist.destroy_process_group()


class _FakeCtx:
    def __init__(self, done):
        self.done = done

    def poll_stats(self):
        return {}, self.done


def _progress_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        out[rank] = [MG.progress(_FakeCtx(3 * k + rank), world) for k in range(3)]
    finally:
        dist.destroy_process_group()


def test_gloo_world2_streaming_progress():
    """NEXT-4 streaming stats: per-rank done counts summed across ranks."""
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        procs = [ctx.Process(target=_progress_worker, args=(r, world, port, out)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
        got = [list(out[r]) for r in range(world)]
    assert got[0] == got[1] == [1, 7, 13]


def test_partition_is_exact_cover():
    jobs, cap = c4_trace(n_jobs=61, seed=9)
    parts = [MG.partition_jobs(jobs, 4, r) for r in range(4)]
    ids = sorted(j.job_id for p in parts for j in p)
    assert ids == sorted(j.job_id for j in jobs)
    assert max(len(p) for p in parts) - min(len(p) for p in parts) <= 1


def test_gloo_world2_allgather_matches_per_partition_oracle():
    world = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        procs = [ctx.Process(target=_worker, args=(r, world, port, out)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(120)
            assert p.exitcode == 0
        got = [dict(out[r]) for r in range(world)]
    assert got[0] == got[1]                         # every rank holds the same merged view
    jobs, cap = c4_trace(n_jobs=60, seed=9, burst=True)
    assert sorted(got[0]) == sorted(j.job_id for j in jobs)
    for r in range(world):
        res = OS.simulate(MG.partition_jobs(jobs, world, r), cap, OS.PACK)
        for jid, s in res.stats.items():
            g = got[0][jid]
            assert g["rank"] == r
            assert (g["completion_tick"], g["completion_seq"], g["first_lane"]) == \
                (s.completion_tick, s.completion_seq, s.first_lane)


# ---------------------------------------------------------------- NEXT-4 placement

def _tiny_jobs(ws, arr=None):
    from workloads import make_job, TRAIN
    return [make_job(i, TRAIN, 0 if arr is None else arr[i], (128, 128), 128, n, iter_ticks=c)
            for i, (n, c) in enumerate(ws)]


def test_lpt_placement_equals_oracle_rule():
    """The product's heap-based LPT gives the oracle's plain-loop placement."""
    import numpy as np
    from oracle import placement as OP
    rng = np.random.default_rng(3)
    for trial in range(60):
        n = int(rng.integers(1, 40))
        G = int(rng.integers(1, 9))
        ws = [(int(rng.integers(1, 20)), int(rng.integers(1, 5)) * 10) for _ in range(n)]
        jobs = _tiny_jobs(ws, arr=[int(x) for x in rng.integers(0, 5, size=n)])
        ref = OP.place_lpt(jobs, G)
        for r in range(G):
            assert [j.job_id for j in MG.partition_jobs(jobs, G, r, "lpt")] == [j.job_id for j in ref[r]]
        refm = OP.place_mod(jobs, G)
        for r in range(G):
            assert [j.job_id for j in MG.partition_jobs(jobs, G, r, "mod")] == [j.job_id for j in refm[r]]


def test_lpt_graham_bound_against_brute_force():
    """Pin of the oracle rule: LPT's max load <= (4/3 - 1/(3G)) OPT (Graham
    1969), OPT by enumerating every assignment of <= 8 jobs to <= 3 GPUs;
    and with identical works LPT is a balanced round robin."""
    import itertools
    import numpy as np
    from oracle import placement as OP
    rng = np.random.default_rng(11)
    for trial in range(150):
        n = int(rng.integers(1, 9))
        G = int(rng.integers(1, 4))
        ws = [(int(rng.integers(1, 12)), 1) for _ in range(n)]
        jobs = _tiny_jobs(ws)
        w = [a * b for a, b in ws]
        opt = min(max(sum(w[i] for i in range(n) if a[i] == g) for g in range(G))
                  for a in itertools.product(range(G), repeat=n))
        got = max(OP.loads(OP.place_lpt(jobs, G)))
        assert got * 3 * G <= (4 * G - 1) * opt, (ws, G, got, opt)
        assert sum(OP.loads(OP.place_lpt(jobs, G))) == sum(w)
    same = _tiny_jobs([(5, 10)] * 13)
    sizes = [len(p) for p in OP.place_lpt(same, 4)]
    assert max(sizes) - min(sizes) <= 1


def test_lpt_balances_c5_better_than_mod():
    from oracle import placement as OP
    from workloads import c5_trace
    jobs, cap = c5_trace()
    for G in (2, 4, 8):
        lm = OP.loads(OP.place_mod(jobs, G))
        ll = OP.loads(OP.place_lpt(jobs, G))
        assert sum(lm) == sum(ll)
        assert max(ll) <= max(lm)
        assert max(ll) <= 1.01 * sum(ll) / G      # near-perfect balance on 2000 jobs


# ---------------------------------------------------------------- NEXT-4 migration (A39)

def _oracle_schedule(cap, policy):
    def sched(jobs):
        r = OS.simulate(jobs, cap, policy)
        ticks = {}
        for rec in r.dispatch:
            ticks.setdefault(rec[3], []).append(rec[1])
        return ticks, max([s.completion_tick for s in r.stats.values()] + [0])
    return sched


def test_rebalance_hand_worked():
    """Two GPUs under FIFO.  (a) GPU0 = one job of 10 x 100 ticks, GPU1 = 2 x 100:
    moving the long job's last 8 iterations at T = 200 would only shift the
    finish (200 + 800 = 1000 = before): no move.  (b) GPU0 also holds a job
    of 5 x 100 queued behind it (FIFO: done at 1500): at T = 200 the long
    job has finished k = 2 iterations (dispatched at 0 and 100), its 800
    remaining ticks beat the queued job's 500, so it moves: GPU1 ends at
    200 + 800 = 1000, GPU0 at 200 + 500 = 700."""
    from oracle import placement as OP
    from workloads import make_job, TRAIN
    a = make_job(0, TRAIN, 0, (128, 128), 128, 10, iter_ticks=100)
    b = make_job(1, TRAIN, 0, (128, 128), 128, 2, iter_ticks=100)
    q = make_job(2, TRAIN, 0, (128, 128), 128, 5, iter_ticks=100)
    assert OP.rebalance([[a], [b]], 1 << 30, OS.FIFO) == ([], [1000, 200])
    assert OP.rebalance([[a, q], [b]], 1 << 30, OS.FIFO) == ([(0, 0, 1, 2, 200)], [700, 1000])
    sched = _oracle_schedule(1 << 30, OS.FIFO)
    moves, parts, ms = MG.plan_rebalance([[a, q], [b]], lambda r, p: sched(p))
    assert (moves, ms) == ([(0, 0, 1, 2, 200)], [700, 1000])
    assert [(j.job_id, j.n_iters, j.arrival_tick) for j in parts[1]] == [(1, 2, 0), (0, 8, 200)]


@pytest.mark.parametrize("G,seed", [(2, 9), (3, 9), (3, 11), (4, 12)])
def test_rebalance_planner_equals_oracle_rule(G, seed):
    from oracle import placement as OP
    jobs, cap = c4_trace(n_jobs=40, seed=seed, burst=True)
    parts = OP.place_mod(jobs, G)
    sched = _oracle_schedule(cap, OS.PACK)
    moves, _, ms = MG.plan_rebalance(parts, lambda r, p: sched(p))
    assert (moves, ms) == OP.rebalance(parts, cap, OS.PACK)
    before = [sched(p)[1] for p in parts]
    assert max(ms) <= max(before)


def _rebalance_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        jobs, cap = c4_trace(n_jobs=40, seed=11, burst=True)
        mine = MG.partition_jobs(jobs, world, rank)
        moves, new, ms = MG.plan_rebalance_dist(mine, rank, world, _oracle_schedule(cap, OS.PACK))
        out[rank] = (moves, [(j.job_id, j.n_iters, j.arrival_tick) for j in new], ms)
    finally:
        dist.destroy_process_group()


def test_gloo_world3_rebalance_matches_oracle():
    """The collective planner (every rank on its own partition: all_gather of
    makespans, the source broadcasts its candidate) against the oracle rule."""
    from oracle import placement as OP
    world, port = 3, _free_port()
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        procs = [ctx.Process(target=_rebalance_worker, args=(r, world, port, out)) for r in range(world)]
        for p in procs:
            p.start()
        for p in procs:
            p.join(300)
            assert p.exitcode == 0
        got = [out[r] for r in range(world)]
    jobs, cap = c4_trace(n_jobs=40, seed=11, burst=True)
    parts = OP.place_mod(jobs, world)
    want_moves, want_ms = OP.rebalance(parts, cap, OS.PACK)
    assert want_moves                                   # this trace does migrate
    for r in range(world):
        assert got[r][0] == want_moves and got[r][2] == want_ms
    for jid, src, dst, k, T in want_moves:
        assert (jid, [j for j in jobs if j.job_id == jid][0].n_iters - k, T) in \
            [(a, n, t) for a, n, t in got[dst][1]]


# ---------------------------------------------------------------- NEXT-4 autoscaling (A40)

def test_autoscale_hand_worked():
    """Loads 0.1, 0.1, 0.8 GPU-s/s at a 0.5 target: G = ceil(1.0 / 0.5) = 2;
    model 2 gets ceil(0.8 / 0.5) = 2 replicas of 0.4 (one per GPU), models 0
    and 1 fill to 0.5 each.  At a tenth of the rates one GPU takes all."""
    from oracle import placement as OP
    rates, svc = {0: 1000, 1: 500, 2: 4000}, {0: 1e-4, 1: 2e-4, 2: 2e-4}
    want = (2, {0: [0], 1: [1], 2: [0, 1]}, [0.5, 0.5])
    assert OP.autoscale(rates, svc) == want
    assert MG.autoscale(rates, svc) == want
    low = {m: r / 10 for m, r in rates.items()}
    G, place, load = MG.autoscale(low, svc)
    assert G == 1 and all(p == [0] for p in place.values())


def test_autoscale_equals_oracle_rule_random():
    import numpy as np
    from oracle import placement as OP
    rng = np.random.default_rng(0)
    for _ in range(200):
        n = int(rng.integers(1, 43))
        rates = {m: float(rng.choice([0.0, rng.uniform(1, 5000)])) for m in range(n)}
        svc = {m: float(rng.uniform(2e-5, 5e-4)) for m in range(n)}
        u = float(rng.choice([0.3, 0.5, 0.8]))
        got, want = MG.autoscale(rates, svc, u, 8), OP.autoscale(rates, svc, u, 8)
        assert got[0] == want[0] and got[1] == want[1]
        assert np.allclose(got[2], want[2])


def test_request_rates_window():
    arr = {0: [0.1, 0.5, 0.9, 1.2], 1: [1.05]}
    assert MG.request_rates(arr, 1.0, 1.0) == {0: 3.0, 1: 0.0}
    assert MG.request_rates(arr, 1.5, 0.5) == {0: 2.0, 1: 2.0}
