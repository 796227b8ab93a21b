"""GPU layer parity on the BENCHMARKED configurations:
the exact runs bench.py times -- the C2a sweep (300 jobs packed over ~37
lanes, 100 iterations, lr up to 1e-2), a C2b job ([4096]^4, B = 2048) and
the C5 2000-job trace -- executed with real work in one persistent kernel,
schedule log byte-compared with the oracle, and the outputs of every
iteration plus the final weights of sampled jobs compared element by element
with the oracle's layer math (oracle/layers.py, §2.1 P:88-104 as
restated in SURVEY §8(c)).

Tolerances (readings A24, A31, A32, A38):
* outputs vs the bf16-storage oracle (the kernel's storage precision, A31):
  max|g - r| / max|r| <= 2e-2 at every iteration (north star);
* outputs vs the fp64 definition: <= 2e-2 at iteration 0 (identical
  weights: a per-layer check), <= 3e-2 along the trajectory (A38: once the
  weights leave the bf16 grid the bf16 weight copy carries up to 2^-9
  relative rounding per element that the fp64 definition does not; the two
  oracles alone differ by up to 1.99e-2 on C2a);
* weight updates, Frobenius-relative: <= 2e-2 vs the bf16-storage oracle
  (A32), <= 0.15 vs the fp64 definition (A38: ReLU-mask decisions flip where
  |Z| is within bf16 rounding of 0; derived bound ~0.09 for three layers,
  measured 0.067-0.078) -- per step from the kernel's own weights on the
  100-iteration C2a jobs (check_job_steps), W_final - W_0 on the short
  C2b / C5 jobs (check_job_trajectory).
"""
import numpy as np
import pytest

from oracle import layers as OL
from oracle import scheduler as OS
from workloads import TRAIN, c2_trace, c5_trace

from gpu_helpers import assert_schedule_parity, normwise_rel

pytestmark = pytest.mark.gpu

TOL = 2e-2
TOL_TRAJ_FP64 = 3e-2
TOL_DW_FP64 = 0.15


def check_job_trajectory(ctx, job, S, report):
    """Every iteration's output and the final weights of one dumped job
    against both oracle precisions; returns the worst errors seen."""
    outs64, W64 = OL.run_job(job)
    outs16, W16 = OL.run_job(job, store=OL.bf16)
    worst = {"out_bf16": 0.0, "out_fp64": 0.0, "dw_bf16": 0.0, "dw_fp64": 0.0}
    for k in range(job.n_iters):
        g = ctx.layers(job.job_id, k).reshape(job.batch, job.dims[-1])
        e16, e64 = normwise_rel(g, outs16[k]), normwise_rel(g, outs64[k])
        worst["out_bf16"] = max(worst["out_bf16"], e16)
        worst["out_fp64"] = max(worst["out_fp64"], e64)
        assert e16 <= TOL, (job.job_id, k, "vs bf16-storage oracle", e16)
        assert e64 <= (TOL if k == 0 else TOL_TRAJ_FP64), (job.job_id, k, "vs fp64", e64)
    if job.kind == TRAIN:
        W0 = OL.init_weights(job)
        flat = ctx.layers(job.job_id, S.WEIGHTS)
        off = 0
        for l in range(len(job.dims) - 1):
            n = job.dims[l] * job.dims[l + 1]
            Wg = flat[off:off + n].reshape(job.dims[l], job.dims[l + 1])
            off += n
            assert normwise_rel(Wg, W16[l]) <= TOL and normwise_rel(Wg, W64[l]) <= TOL, (job.job_id, l)
            dg = Wg - W0[l]
            r16 = float(np.linalg.norm(dg - (W16[l] - W0[l])) / np.linalg.norm(W16[l] - W0[l]))
            r64 = float(np.linalg.norm(dg - (W64[l] - W0[l])) / np.linalg.norm(W64[l] - W0[l]))
            worst["dw_bf16"] = max(worst["dw_bf16"], r16)
            worst["dw_fp64"] = max(worst["dw_fp64"], r64)
            assert r16 <= TOL, (job.job_id, l, "dW vs bf16-storage oracle", r16)
            assert r64 <= TOL_DW_FP64, (job.job_id, l, "dW vs fp64", r64)
    report[job.job_id] = worst
    return worst


def split_weights(flat, dims):
    out, off = [], 0
    for l in range(len(dims) - 1):
        n = dims[l] * dims[l + 1]
        out.append(flat[off:off + n].reshape(dims[l], dims[l + 1]).astype(np.float64))
        off += n
    return out


def check_job_steps(ctx, job, S, report):
    """Teacher-forced parity of EVERY iteration (SALUS_DUMP_WEIGHT_STEPS):
    the kernel's own weights before iteration k (W_0 = the A29 init, then its
    dump after iteration k - 1) drive the oracle's iteration k, whose output
    and update W_{k+1} - W_k = -lr dW_k must match the kernel's -- a per-step
    check that long-trajectory amplification (A32) cannot blur.  Plus the
    final weights against the oracle's own bf16-storage trajectory."""
    lr = float(np.float32(job.lr))
    Wk = OL.init_weights(job)
    worst = {"out_bf16": 0.0, "out_fp64": 0.0, "step_bf16": 0.0, "step_fp64": 0.0}
    for k in range(job.n_iters):
        X, T = OL.inputs(job, k)
        A16, dW16 = OL.gradients(Wk, X, T, OL.bf16)
        A64, dW64 = OL.gradients(Wk, X, T)
        g = ctx.layers(job.job_id, k).reshape(job.batch, job.dims[-1])
        e16, e64 = normwise_rel(g, A16[-1]), normwise_rel(g, A64[-1])
        worst["out_bf16"] = max(worst["out_bf16"], e16)
        worst["out_fp64"] = max(worst["out_fp64"], e64)
        assert e16 <= TOL, (job.job_id, k, "output vs bf16-storage oracle", e16)
        assert e64 <= (TOL if k == 0 else TOL_TRAJ_FP64), (job.job_id, k, "output vs fp64", e64)
        Wn = split_weights(ctx.layers(job.job_id, S.weights_after(k)), job.dims)
        for l in range(len(Wk)):
            dg = Wn[l] - Wk[l]
            r16 = float(np.linalg.norm(dg + lr * dW16[l]) / np.linalg.norm(lr * dW16[l]))
            r64 = float(np.linalg.norm(dg + lr * dW64[l]) / np.linalg.norm(lr * dW64[l]))
            worst["step_bf16"] = max(worst["step_bf16"], r16)
            worst["step_fp64"] = max(worst["step_fp64"], r64)
            assert r16 <= TOL, (job.job_id, k, l, "step vs bf16-storage oracle", r16)
            assert r64 <= TOL_DW_FP64, (job.job_id, k, l, "step vs fp64", r64)
        Wk = Wn
    _, W16 = OL.run_job(job, store=OL.bf16)
    for l, (a, b) in enumerate(zip(Wk, W16)):
        assert normwise_rel(a, b) <= TOL, (job.job_id, l, "final weights vs oracle trajectory")
    report[job.job_id] = worst
    return worst


def test_c2a_sweep_full_run_sampled_jobs():
    """The bench's headline run (BASELINE configs[1]): 300 jobs x 100
    iterations under PACK in a 1 GiB arena, every iteration executed; jobs
    with id = 0 (mod 50) dump every output and the weights after every
    iteration (teacher-forced per-step parity, check_job_steps)."""
    from paper_1902_04610_b200 import salus as S
    jobs, cap = c2_trace("a")
    pick = [j for j in jobs if j.job_id % 50 == 0]
    dump = {j.job_id: S.DUMP_OUTPUTS | S.DUMP_WEIGHT_STEPS for j in pick}
    ctx, ref, stats = assert_schedule_parity(jobs, cap, OS.PACK, null_work=False, dump=dump)
    report = {}
    try:
        for j in pick:
            check_job_steps(ctx, j, S, report)
    finally:
        ctx.close()
    print("c2a sweep parity:", report)


def test_c2b_job_full_size():
    """One C2b job ([4096]^4, B = 2048: 16 x 32 K-chunks per tile, the
    tensor-bound sweep member) for 2 iterations."""
    from paper_1902_04610_b200 import salus as S
    jobs, cap = c2_trace("b", n_jobs=1, n_iters=2)
    ctx, ref, stats = assert_schedule_parity(jobs, cap, OS.PACK, null_work=False,
                                             dump={jobs[0].job_id: S.DUMP_OUTPUTS | S.DUMP_WEIGHTS})
    report = {}
    try:
        check_job_trajectory(ctx, jobs[0], S, report)
    finally:
        ctx.close()
    print("c2b parity:", report)


def c5_sample(jobs, k_small=4):
    """Sampled C5 jobs the oracle replays in seconds: the k_small cheapest
    (n * flops) jobs, the cheapest job at each width >= 1024, the cheapest
    4-layer job and the cheapest job with batch >= 512."""
    from workloads import algorithmic_flops
    cost = lambda j: j.n_iters * algorithmic_flops(j.kind, j.dims, j.batch)
    pick = sorted(jobs, key=cost)[:k_small]
    for w in (1024, 2048, 4096):
        cands = [j for j in jobs if j.dims[0] == w]
        if cands:
            pick.append(min(cands, key=cost))
    for sel in (lambda j: len(j.dims) == 5, lambda j: j.batch >= 512):
        cands = [j for j in jobs if sel(j)]
        if cands:
            pick.append(min(cands, key=cost))
    seen, out = set(), []
    for j in pick:
        if j.job_id not in seen:
            seen.add(j.job_id)
            out.append(j)
    return out


def test_c5_full_trace_sampled_jobs():
    """BASELINE configs[4] at one GPU: the 2000-job burst trace under PACK in
    a 16 GiB arena (the bench's C5 run), every iteration executed; a sample
    of jobs (cheapest, and one per wide width; most take the GEN/target
    prefetch path) dump every output and their final weights."""
    from paper_1902_04610_b200 import salus as S
    jobs, cap = c5_trace()
    pick = c5_sample(jobs)
    assert sum(j.n_iters * j.batch * j.dims[-1] for j in pick) < 4e8    # dump area stays small
    dump = {j.job_id: S.DUMP_OUTPUTS | S.DUMP_WEIGHTS for j in pick}
    ctx, ref, stats = assert_schedule_parity(jobs, cap, OS.PACK, null_work=False, dump=dump,
                                             timeout_ms=600000)
    report = {}
    try:
        for j in pick:
            check_job_trajectory(ctx, j, S, report)
    finally:
        ctx.close()
    print("c5 parity:", report)
