"""Split-K tiles (DevJob.splitk): in narrow latency-mode
records a stage whose F / dX part has few pair tasks and a long K runs as S
K-slices; the last slice of a tile sums the fp32 partials in slice order
and runs the epilogue.  The math is the same GEMM (P:98-104 forward /
backward of a dense layer), so parity is the oracle's at the north-star
tolerance; the fixed summation order makes repeated runs bit-identical."""
import os

import numpy as np
import pytest

from oracle import scheduler as OS
from workloads import INFER, TRAIN, make_job, footprint_bytes

MIB = 1 << 20

from gpu_helpers import assert_schedule_parity
from test_gpu_math import _check_math

pytestmark = pytest.mark.gpu


def _job(jid, kind, dims, batch, n, slack=64 * MIB, **kw):
    _, e = footprint_bytes(kind, dims, batch)
    req = tuple(range(0, 10 * n, 10)) if kind == INFER else ()
    return make_job(jid, kind, 0, dims, batch, n, ephemeral_bytes=e + slack, request_ticks=req, **kw)


CASES = [
    # (kind, dims, batch): F / dX stages of 16-32 N=128 pair tasks, K 1024-4096
    (TRAIN, (2048, 2048, 2048, 512), 128),
    (TRAIN, (1024, 2048, 1024), 200),          # bp = 256: both CTA halves hold rows, ragged batch
    (TRAIN, (4096, 4096, 256), 64),
    (INFER, (4096, 4096, 256), 8),
]


def _run(jobs, env=None):
    from paper_1902_04610_b200 import salus as S
    env = {"SALUS_SPLITK": "1", **(env or {})}     # split-K is opt-in
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        dump = {j.job_id: S.DUMP_OUTPUTS | (S.DUMP_WEIGHTS if j.kind == TRAIN else 0) for j in jobs}
        return assert_schedule_parity(jobs, 1 << 34, OS.FIFO, null_work=False, dump=dump)
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


@pytest.mark.parametrize("kind,dims,batch", CASES)
def test_splitk_parity(kind, dims, batch):
    """One job alone (FIFO: one lane, narrow records): outputs of every
    iteration and the final weights / weight updates within 2e-2 of the
    oracle; split-K actually ran (more tiles than with SALUS_SPLITK=0)."""
    jobs = [_job(5, kind, dims, batch, 3, lr=5e-3, seed=11)]
    ctx, _, _ = _run(jobs)
    try:
        worst_split = _check_math(ctx, jobs)
        n_split = ctx.run_stats()["n_tasks"]
    finally:
        ctx.close()
    ctx, _, _ = _run(jobs, {"SALUS_SPLITK": "0"})
    try:
        worst_plain = _check_math(ctx, jobs)
        n_plain = ctx.run_stats()["n_tasks"]
    finally:
        ctx.close()
    print(f"worst rel: split {worst_split:.3e} plain {worst_plain:.3e}")
    assert n_split > n_plain, (n_split, n_plain)


def test_splitk_deterministic():
    """The last slice sums the partials in slice order whichever slice
    arrives last: two runs give bit-identical outputs and weights."""
    from paper_1902_04610_b200 import salus as S
    jobs = [_job(7, TRAIN, (2048, 2048, 2048, 512), 128, 3, lr=1e-2, seed=12)]
    got = []
    for _ in range(2):
        ctx, _, _ = _run(jobs)
        try:
            got.append((np.concatenate([ctx.layers(7, k).ravel() for k in range(3)]), ctx.layers(7, S.WEIGHTS).copy()))
        finally:
            ctx.close()
    assert np.array_equal(got[0][0], got[1][0]) and np.array_equal(got[0][1], got[1][1])


def test_splitk_needs_slack():
    """A job that declares exactly its footprint has no workspace: no split."""
    dims, batch = (2048, 2048, 2048, 512), 128
    jobs = [_job(9, TRAIN, dims, batch, 2, slack=0, lr=1e-2, seed=13)]
    ctx, _, _ = _run(jobs)
    try:
        _check_math(ctx, jobs)
        a = ctx.run_stats()["n_tasks"]
    finally:
        ctx.close()
    ctx, _, _ = _run(jobs, {"SALUS_SPLITK": "0"})
    try:
        assert ctx.run_stats()["n_tasks"] == a
    finally:
        ctx.close()
