"""Randomised real-work traces on the GPU: small MLP jobs (training and
inference, ragged widths and batches, with and without persistent slack --
i.e. with and without the GEN/target prefetch path) under memory pressure,
every policy, SRTF also with eviction.  Byte-identical schedule log and
every job's outputs / weights against the oracle."""
import numpy as np
import pytest

from oracle import logfmt as LG
from oracle import scheduler as OS
from workloads import INFER, PAGE_BYTES, TRAIN, footprint_bytes, make_job

from gpu_helpers import assert_schedule_parity
from test_gpu_math import _check_math

pytestmark = pytest.mark.gpu
G = PAGE_BYTES


def _trace(seed, n_jobs=7):
    rng = np.random.default_rng(seed)
    jobs = []
    for j in range(n_jobs):
        kind = INFER if rng.random() < 0.3 else TRAIN
        depth = int(rng.integers(1, 4))
        dims = tuple(int(rng.choice([72, 128, 200, 256, 384])) for _ in range(depth + 1))
        batch = int(rng.choice([16, 64, 128, 200]))
        n = int(rng.integers(1, 5))
        p, e = footprint_bytes(kind, dims, batch)
        slack = int(rng.choice([0, 0, 1 << 20, 4 << 20]))
        arr = int(rng.integers(0, 400))
        req = tuple(sorted(int(arr + x) for x in rng.integers(0, 600, size=n))) if kind == INFER else ()
        jobs.append(make_job(j, kind, arr, dims, batch, n, iter_ticks=int(rng.integers(20, 120)),
                             persistent_bytes=p + slack, ephemeral_bytes=e + int(rng.integers(0, 4)) * G,
                             lr=1e-2, seed=500 + seed * 16 + j, request_ticks=req))
    # capacity: the largest job alone fits, roughly two to three side by side
    need = max(-(-j.persistent_bytes // G) + -(-j.ephemeral_bytes // G) for j in jobs)
    return jobs, int(need * 2.2) * G


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("policy,max_lanes,evict", [(OS.PACK, 0, False), (OS.FAIR, 3, False),
                                                    (OS.SRTF, 1, True), (OS.FIFO, 0, False)])
def test_random_real_work(seed, policy, max_lanes, evict):
    from paper_1902_04610_b200 import salus as S
    jobs, cap = _trace(seed)
    dump = {j.job_id: S.DUMP_OUTPUTS | (S.DUMP_WEIGHTS if j.kind == TRAIN else 0) for j in jobs}
    ctx, ref, stats = assert_schedule_parity(jobs, cap, policy, max_lanes=max_lanes, evict=evict,
                                             null_work=False, dump=dump)
    try:
        if evict:
            rs = ctx.run_stats()
            n_ev = sum(1 for r in ref.log if r[1] == LG.JOB_EVICT)
            assert rs["n_swap_out"] <= n_ev          # jobs without persistent pages copy nothing
        _check_math(ctx, jobs)
    finally:
        ctx.close()
