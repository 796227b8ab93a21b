"""K9 skinny-batch tiles (opt-in with SALUS_SWAP=1): an
inference job whose batch pads to 128 rows runs its F_l GEMMs transposed
(M = output features, N = batch) except in narrow records, which keep the
non-transposed N = 128 tiles.  Skinny training and inference jobs against
the oracle (inference requests of b = 1..16; SURVEY §2c
K9) in every execution mode, with and without K9 tiles, plus run-to-run
bit-reproducibility."""
import numpy as np
import pytest

from oracle import layers as OL
from oracle import scheduler as OS
from workloads import TRAIN, INFER, make_job

from gpu_helpers import assert_schedule_parity, normwise_rel

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _jobs(b):
    # training: K = 1024, an odd number of 128-feature blocks (384: the last
    # pair's peer half is empty), a ragged width (1000 -> 1024), dX with K = 640;
    # inference: a 4096-wide layer (16 output pairs) and K = 4096
    return [make_job(0, TRAIN, 0, (1024, 1000, 640, 40), b, 3, lr=1e-2, seed=11),
            make_job(1, TRAIN, 0, (256, 384, 200), b, 2, lr=1e-2, seed=13),
            make_job(2, INFER, 0, (4096, 4096, 1024), b, 3, seed=12, request_ticks=(0, 1, 2))]


def _check(ctx, jobs):
    from paper_1902_04610_b200 import salus as S
    for j in jobs:
        outs64, _ = OL.run_job(j)
        outs16, W16 = OL.run_job(j, store=OL.bf16)
        for k in range(j.n_iters):
            g = ctx.layers(j.job_id, k).reshape(j.batch, j.dims[-1])
            rel = max(normwise_rel(g, outs64[k]), normwise_rel(g, outs16[k]))
            assert rel <= TOL, (j.job_id, k, rel)
        if j.kind == TRAIN:
            W0 = OL.init_weights(j)
            flat = ctx.layers(j.job_id, S.WEIGHTS)
            off = 0
            for l in range(len(j.dims) - 1):
                n = j.dims[l] * j.dims[l + 1]
                Wg = flat[off:off + n].reshape(j.dims[l], j.dims[l + 1])
                off += n
                assert normwise_rel(Wg, W16[l]) <= TOL, (j.job_id, l)
                dg, dr = Wg - W0[l], W16[l] - W0[l]
                assert np.linalg.norm(dg - dr) / np.linalg.norm(dr) <= TOL, (j.job_id, "dW", l)


@pytest.mark.parametrize("b", [1, 4, 8, 16, 100, 128])
@pytest.mark.parametrize("eager,narrow,swap", [(None, None, "1"), (None, "0", "1"), ("0", None, "1"),
                                               (None, None, "0")])
def test_skinny_batches(b, eager, narrow, swap, monkeypatch):
    """Latency mode with narrow tiles (3 lanes open here: narrow lanes = 2
    covers the tail), latency mode with wide / K9 tiles (narrow lanes 0),
    throughput mode (eager lanes 0), and without K9 tiles."""
    from paper_1902_04610_b200 import salus as S
    monkeypatch.setenv("SALUS_SWAP", swap)
    if eager is not None:
        monkeypatch.setenv("SALUS_EAGER_LANES", eager)
    if narrow is not None:
        monkeypatch.setenv("SALUS_NARROW_LANES", narrow)
    jobs = _jobs(b)
    dump = {j.job_id: S.DUMP_OUTPUTS | (S.DUMP_WEIGHTS if j.kind == TRAIN else 0) for j in jobs}
    ctx, ref, stats = assert_schedule_parity(jobs, 1 << 30, OS.PACK, null_work=False, dump=dump)
    try:
        _check(ctx, jobs)
    finally:
        ctx.close()


@pytest.mark.parametrize("eager", [None, "0"])
def test_runs_are_bit_identical(eager, monkeypatch):
    """Two runs of the same context give bit-identical outputs and weights
    (every reduction has a fixed order)."""
    from paper_1902_04610_b200 import salus as S
    monkeypatch.setenv("SALUS_SWAP", "1")
    if eager is not None:
        monkeypatch.setenv("SALUS_EAGER_LANES", eager)
    jobs = _jobs(16)
    dump = {j.job_id: S.DUMP_OUTPUTS | (S.DUMP_WEIGHTS if j.kind == TRAIN else 0) for j in jobs}
    ctx = S.Context(jobs, 1 << 30, OS.PACK, dump=dump)
    try:
        ctx.run()
        first = {(j.job_id, k): ctx.layers(j.job_id, k).copy() for j in jobs for k in range(j.n_iters)}
        w0 = ctx.layers(0, S.WEIGHTS).copy()
        ctx.run()
        for key, v in first.items():
            assert np.array_equal(v, ctx.layers(*key)), key
        assert np.array_equal(w0, ctx.layers(0, S.WEIGHTS))
    finally:
        ctx.close()
