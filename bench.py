"""Benchmark of the Salus hot path on B200 (BASELINE.json metric:
"aggregate iters/s at 1-8 B200; job-switch µs; avg JCT vs FIFO baseline").

One step = one salus_run of the whole workload: every job's admission, lane
assignment, page allocation, iteration dispatch and every iteration's
tcgen05 GEMM work, inside the persistent kernel (§8(a) rows a1..a9).

Workload at N=1: BASELINE configs[1] = C2a, the 300-job hyper-parameter sweep
([1024]^4 MLP, batch 256, 100 iterations each, PACK, 1 GiB arena).  Under
torchrun with N ranks each GPU runs an independent Salus instance on its
mod-N partition of a 300*N-job sweep (weak scaling); the only
collective is one NCCL all_gather of per-GPU completion statistics.

usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl salus|reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from workloads import (TRAIN, algorithmic_bytes, algorithmic_flops, c2_trace,  # noqa: E402
                       c3_trace)

METRIC = "aggregate iters/s at 1-8 B200; job-switch µs; avg JCT vs FIFO baseline"
S_PACK = 2          # salus.h SALUS_PACK (the oracle uses the same numbering)
UNIT = "iters/s"
N_JOBS, N_ITERS = 300, 100


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload(world, rank):
    from paper_1902_04610_b200 import multigpu as MG
    jobs, cap = c2_trace("a", n_jobs=N_JOBS * world, n_iters=N_ITERS)
    return MG.partition_jobs(jobs, world, rank), cap


def work_per_iter(job):
    return (algorithmic_flops(job.kind, job.dims, job.batch),
            algorithmic_bytes(job.kind, job.dims, job.batch))


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p["hbm_gbs"], p["bf16_tflops"], "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, 1590.0, "fallback"


def roofline_frac(jobs, seconds, gpus=1):
    """SURVEY §8(d) reported fraction: the ideal perfectly-packed time,
    sum over iterations of max(flops / tensor peak, bytes / HBM peak), over
    the measured device time (peaks x G for G GPUs).  Peaks: the measured
    burst figures of MEASURED_PEAKS.json."""
    hbm, bf16, _ = peaks()
    ideal = sum(j.n_iters * max(algorithmic_flops(j.kind, j.dims, j.batch) / (bf16 * 1e12),
                                algorithmic_bytes(j.kind, j.dims, j.batch) / (hbm * 1e9)) for j in jobs)
    return ideal / (seconds * gpus)


def c5_section(S, local, rank, world, with_cpu_baseline):
    """BASELINE configs[4] (C5): the 2000-job trace (burst, PACK, 16 GiB per
    GPU) partitioned k mod N over the N ranks -- STRONG scaling, one
    independent Salus instance per GPU, no data-path collective -- then one
    NCCL all_gather of every job's completion record.  One
    timed run: barrier + CUDA events on each rank, max over ranks.
    Collective: every rank calls it."""
    import torch
    import torch.distributed as dist
    from paper_1902_04610_b200 import metrics as PM, multigpu as MG
    from workloads import c5_trace
    jobs_all, cap = c5_trace()
    mine = MG.partition_jobs(jobs_all, world, rank)
    dev = f"cuda:{local}"
    ctx = S.Context(mine, cap, S.PACK, device=local, log=False)
    try:
        stream = torch.cuda.current_stream(local)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        stats = ctx.run()
        e1.record(stream)
        torch.cuda.synchronize()
        rs = ctx.run_stats()
    finally:
        ctx.close()
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    per_rank = [torch.zeros_like(t) for _ in range(world)]
    if world > 1:
        dist.all_gather(per_rank, t)
    else:
        per_rank = [t]
    per_rank = [float(x.item()) for x in per_rank]
    ms_max = max(per_rank)
    torch.cuda.synchronize()
    ta = time.perf_counter()
    merged = MG.gather_stats(stats, rank, world, device=dev, t0_ns=rs["wall_first_ns"])
    torch.cuda.synchronize()
    allgather_us = (time.perf_counter() - ta) * 1e6
    # the FIFO baseline of the same partition: schedule only (logical ticks
    # do not depend on the work executed), records gathered the same way
    cf = S.Context(mine, cap, S.FIFO, device=local, log=False, null_work=True)
    try:
        fifo_merged = MG.gather_stats(cf.run(), rank, world, device=dev)
    finally:
        cf.close()
    if rank != 0:
        return None
    iters = sum(j.n_iters for j in jobs_all)
    logical = PM.summarize(jobs_all, merged)
    fifo = PM.summarize(jobs_all, fifo_merged)
    phys = [merged[j.job_id]["wall_end_rel_ns"] / 1e6 for j in jobs_all]
    out = {"config": f"C5: {len(jobs_all)} jobs (C4 generator, seed 5, burst), PACK, 16 GiB per GPU, "
                     f"partitioned k mod {world} (strong scaling)",
           "gpus": world, "jobs": len(jobs_all), "iterations": iters,
           "makespan_ms": ms_max, "per_rank_ms": per_rank,
           "iters_per_s": iters / (ms_max / 1e3),
           "roofline_frac": roofline_frac(jobs_all, ms_max / 1e3, world),
           "avg_jct_ms": float(np.mean(phys)), "p95_jct_ms": float(np.percentile(phys, 95)),
           **logical, "fifo_avg_jct_ticks": fifo["avg_jct_ticks"],
           "avg_jct_fifo_over_pack": fifo["avg_jct_ticks"] / logical["avg_jct_ticks"],
           "stats_allgathered": len(merged), "allgather_us": allgather_us,
           "kernel_launches": world}
    if with_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(jobs_all, cap, S_PACK, budget_s=10.0, iters_per_job=1)
    return out


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for n, v in zip(names, f[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def switch_latency(S, device):
    """North-star secondary metric: iteration-boundary switch latency with
    42 packed inference models (C3: 14 architectures x 3 instances, FAIR over
    8 time-shared lanes).  From the device wall stamps of one run: for
    consecutive iterations of a lane, start(next) - end(prev), split into job
    switches and same-job continuations."""
    jobs, cap = c3_trace()
    ctx = S.Context(jobs, cap, S.FAIR, device=device, max_lanes=8, log=True)
    ctx.run()
    rs = ctx.run_stats()
    w = ctx.wall()
    log = np.frombuffer(ctx.log_bytes(), dtype=S.LOG_DTYPE)
    ctx.close()
    # request latency in logical ticks (ns nominal, A17): the k-th request of a
    # model is served by its k-th iteration (A27): end of that iteration - request tick
    J = {j.job_id: j for j in jobs}
    d = log[log["kind"] == 1]                       # DISPATCH records: a = iteration index
    req_lat = [int(r["tick"]) + J[int(r["job"])].iter_ticks - J[int(r["job"])].request_ticks[int(r["a"])]
               for r in d]
    w = w[np.argsort(w["seq"])]
    sw, rdy, gap, last = [], [], [], {}
    for r in w:
        ln = int(r["lane"])
        if ln in last:
            prev = last[ln]
            d = (int(r["start_ns"]) - int(prev["end_ns"])) / 1e3
            if prev["job"] == r["job"]:
                gap.append(d)
            else:
                sw.append(d)
                # from the moment the switch could happen (previous iteration
                # done AND the scheduler's dispatch appended) to the first tile
                rdy.append((int(r["start_ns"]) - max(int(prev["end_ns"]), int(r["append_ns"]))) / 1e3)
        last[ln] = r

    def pct(a):
        return {"n": len(a), "p50": float(np.median(a)) if a else None,
                "p99": float(np.percentile(a, 99)) if a else None}
    byts = sum(j.n_iters * algorithmic_bytes(j.kind, j.dims, j.batch) for j in jobs)
    flops = sum(j.n_iters * algorithmic_flops(j.kind, j.dims, j.batch) for j in jobs)
    return {"config": "C3: 42 inference models (14 archs x 3), FAIR, 8 lanes, 16 GiB",
            "models_coresident": len(jobs), "requests": int(rs["n_dispatch"]),
            "requests_per_s": rs["n_dispatch"] / (rs["kernel_ns"] / 1e9),
            "algorithmic_gbs": byts / rs["kernel_ns"], "algorithmic_tflops": flops / rs["kernel_ns"] / 1e3,
            "switch_us": pct(sw), "switch_from_ready_us": pct(rdy),
            "same_job_gap_us": pct(gap),
            "request_latency_logical_us": {"avg": float(np.mean(req_lat)) / 1e3,
                                           "p99": float(np.percentile(req_lat, 99)) / 1e3},
            "paper_context": "inference latency overhead < 5 ms average on P100 (P:737)"}


def c3_live(S, device, rates=((20, 1.0), (100, 0.5), (1000, 0.2)), seed=3):
    """C3 in wall-clock time (SURVEY §8(d) C3, NEXT-2 live requests): the 42
    models stay resident under FAIR over 8 lanes while a host thread submits
    each model's Poisson requests (rate lambda per model, for `duration` s of
    wall time) through salus_submit_requests as they fall due.  Per request,
    from the device's own stamps: queueing = first tile start - the moment the
    scheduler saw it, latency = last tile end - seen; per lane, the physical
    switch gap = start - max(previous end, seen).  Sustained = every request
    served and the run ending within the offered window plus the tail."""
    import dataclasses
    base, cap = c3_trace()
    out = {}
    for lam, dur in rates:
        rng = np.random.default_rng(seed)
        due, jobs = [], []
        for j in base:
            t = np.cumsum(rng.exponential(1.0 / lam, size=int(lam * dur * 3) + 8))
            t = t[t < dur]
            if len(t) == 0:
                t = np.array([dur * rng.random()])
            jobs.append(dataclasses.replace(j, n_iters=len(t), request_ticks=()))
            due += [(float(x), j.job_id) for x in t]
        due.sort()
        ctx = S.Context(jobs, cap, S.FAIR, device=device, max_lanes=8, log=True, online=True)
        try:
            ctx.run_async()
            t0 = time.perf_counter()
            lag = ctx.serve(due)
            ctx.end_submissions()
            ctx.wait()
            span = time.perf_counter() - t0
            w = ctx.wall()
            seen = {j.job_id: ctx.requests(j.job_id)[1].astype(np.int64) for j in jobs}
        finally:
            ctx.close()
        w = w[np.argsort(w["seq"])]
        kreq, q, lat, sw, last, s2a, a2s = {}, [], [], [], {}, [], []
        for r in w:
            jid = int(r["job"])
            kk = kreq.get(jid, 0)
            kreq[jid] = kk + 1
            s0 = int(seen[jid][kk])
            q.append((int(r["start_ns"]) - s0) / 1e3)
            if int(r["append_ns"]) >= s0:              # queueing split: scheduler / publication + decode
                s2a.append((int(r["append_ns"]) - s0) / 1e3)
                a2s.append((int(r["start_ns"]) - int(r["append_ns"])) / 1e3)
            lat.append((int(r["end_ns"]) - s0) / 1e3)
            ln = int(r["lane"])
            if ln in last and int(last[ln]["job"]) != jid:
                sw.append((int(r["start_ns"]) - max(int(last[ln]["end_ns"]), s0)) / 1e3)
            last[ln] = r

        def pct(a):
            return {"n": len(a), "p50": float(np.percentile(a, 50)) if a else None,
                    "p99": float(np.percentile(a, 99)) if a else None,
                    "max": float(np.max(a)) if a else None}
        out[f"lambda{lam}"] = {
            "models": len(jobs), "requests": len(due), "offered_rps": len(due) / dur, "window_s": dur,
            "served": int(len(w)), "run_s": span,
            "queueing_us": pct(q), "latency_us": pct(lat), "switch_gap_us": pct(sw),
            "seen_to_append_us": pct(s2a), "append_to_first_tile_us": pct(a2s),
            "host_submit_lag_us": pct([x * 1e6 for x in lag])}
    return {"config": "C3 live: 42 inference models (14 archs x 3), FAIR over 8 lanes, 16 GiB; "
                      "Poisson requests per model in wall time via salus_submit_requests",
            "paper_context": "inference latency overhead < 5 ms average on P100 (P:737)", **out}


def c1_config(S, device):
    """BASELINE configs[0] (C1: 2 jobs, FIFO vs SRTF): the device schedule's
    average JCT in logical ticks (bit-identical to the oracle's) and the
    physical per-iteration time and job-switch gap on the lane."""
    from workloads import c1_trace
    jobs, cap = c1_trace()
    arr = {j.job_id: j.arrival_tick for j in jobs}
    out = {}
    for name, pol in (("fifo", S.FIFO), ("srtf", S.SRTF)):
        ctx = S.Context(jobs, cap, pol, device=device, log=True)
        try:
            st = ctx.run()
            w = ctx.wall()
        finally:
            ctx.close()
        w = w[np.argsort(w["seq"])]
        sw = [(int(b["start_ns"]) - int(a["end_ns"])) / 1e3 for a, b in zip(w[:-1], w[1:]) if a["job"] != b["job"]]
        out[name] = {"avg_jct_ticks": float(np.mean([v["completion_tick"] - arr[k] for k, v in st.items()])),
                     "iter_us_p50": float(np.median((w["end_ns"] - w["start_ns"]) / 1e3)),
                     "switch_gap_us": sw}
    out["fifo_over_srtf_avg_jct"] = out["fifo"]["avg_jct_ticks"] / out["srtf"]["avg_jct_ticks"]
    return out


def jct_physical(S, device, jobs, cap):
    """The sweep executed (not simulated) under PACK and under FIFO (the
    baseline): average JCT and makespan from the device stamps (every job
    arrives at tick 0, so a job's JCT = its last tile end - kernel start)."""
    out = {}
    for name, pol in (("pack", S.PACK), ("fifo", S.FIFO)):
        ctx = S.Context(jobs, cap, pol, device=device, log=False)
        try:
            st = ctx.run()
            rs = ctx.run_stats()
        finally:
            ctx.close()
        t0 = rs["wall_first_ns"]
        jct = [(v["wall_end_ns"] - t0) / 1e6 for v in st.values()]
        out[name] = {"avg_jct_ms": float(np.mean(jct)), "makespan_ms": float(max(jct))}
    out["fifo_over_pack_avg_jct"] = out["fifo"]["avg_jct_ms"] / out["pack"]["avg_jct_ms"]
    out["fifo_over_pack_makespan"] = out["fifo"]["makespan_ms"] / out["pack"]["makespan_ms"]
    return out


def c4_jct(S, device):
    """BASELINE configs[3] (C4: 100-job mixed training trace, Poisson
    arrivals, varied footprints, 16 GiB): the paper's headline "avg JCT vs
    FIFO" (PAPER.md tab:exp11; 3.19x on its private trace) as the
    device scheduler computes it, every iteration's GEMM work executed.  The
    JCTs are logical (A17's iteration-cost model; the GPU tests hold the same
    log byte-identical to the oracle's); the physical columns are the measured
    kernel time of the whole trace under each policy."""
    from paper_1902_04610_b200 import metrics as PM
    from workloads import c4_trace
    jobs, cap = c4_trace()
    flops = sum(j.n_iters * algorithmic_flops(j.kind, j.dims, j.batch) for j in jobs)
    byts = sum(j.n_iters * algorithmic_bytes(j.kind, j.dims, j.batch) for j in jobs)
    out = {"config": "C4: 100 jobs, widths 256-4096, depth 2-4, B 64-1024, n 10-2000, Poisson rho~1.2, 16 GiB",
           "iterations": sum(j.n_iters for j in jobs)}
    for name, pol in (("fifo", S.FIFO), ("srtf", S.SRTF), ("pack", S.PACK), ("fair", S.FAIR)):
        ctx = S.Context(jobs, cap, pol, device=device, log=False)
        try:
            st = ctx.run()
            rs = ctx.run_stats()
        finally:
            ctx.close()
        m = PM.summarize(jobs, st)
        ks = rs["kernel_ns"] / 1e9
        out[name] = {**m, "kernel_ms": ks * 1e3, "iters_per_s": rs["n_dispatch"] / ks,
                     "roofline_frac": roofline_frac(jobs, ks)}
    out["fifo_over_srtf_avg_jct"] = out["fifo"]["avg_jct_ticks"] / out["srtf"]["avg_jct_ticks"]
    out["paper_context"] = "3.19x avg JCT FIFO/SRTF on the paper's 100-job trace, 2x P100 (P:612-629)"
    return out


def c4e_evict(S, device):
    """SURVEY §8(f) NEXT-3 (reading A35): the C4 trace with 8x the
    declared persistent memory (C4e), so SRTF admission runs into the safety
    condition.  SRTF without and with eviction, every iteration executed:
    logical average JCT from the device's records, and the swap records the
    kernel executed -- persistent pages copied to pinned host memory and
    back -- with their measured bandwidth."""
    from paper_1902_04610_b200 import metrics as PM
    from workloads import c4_trace
    jobs, cap = c4_trace(p_scale=8.0)
    out = {"config": "C4e: C4 with declared P x8 (0.89-6.6 GB), SRTF, 1 lane, 16 GiB"}
    for name, ev in (("srtf", False), ("srtf_evict", True)):
        ctx = S.Context(jobs, cap, S.SRTF, device=device, log=False, evict=ev)
        try:
            st = ctx.run()
            rs = ctx.run_stats()
        finally:
            ctx.close()
        m = PM.summarize(jobs, st)
        r = {"avg_jct_ticks": m["avg_jct_ticks"], "makespan_ticks": m["makespan_ticks"],
             "kernel_ms": rs["kernel_ns"] / 1e6}
        if ev:
            r.update({"n_swap_out": rs["n_swap_out"], "n_swap_in": rs["n_swap_in"],
                      "swap_gib": rs["swap_bytes"] / 2**30,
                      "swap_gbs": rs["swap_bytes"] / max(1, rs["swap_ns"]),
                      "swap_ms_total": rs["swap_ns"] / 1e6})
        out[name] = r
    out["srtf_over_evict_avg_jct"] = out["srtf"]["avg_jct_ticks"] / out["srtf_evict"]["avg_jct_ticks"]
    return out


def c3_rate_sweep(S, device):
    """the request-rate sweep {20, 100, 1k, 10k} req/s
    per model (42 models, PACK: one lane each; FAIR over 8 lanes), every
    request executed.  Logical request latency (A17 cost model; end of the
    serving iteration - request tick, from the oracle-identical log) shows
    where the lanes saturate; requests/s is the device's physical rate."""
    out = {}
    for lam in (20, 100, 1000, 10000):
        jobs, cap = c3_trace(rate_per_s=float(lam))
        J = {j.job_id: j for j in jobs}
        for name, pol, ml in (("pack", S.PACK, 0), ("fair8", S.FAIR, 8)):
            ctx = S.Context(jobs, cap, pol, device=device, max_lanes=ml, log=True)
            try:
                ctx.run()
                rs = ctx.run_stats()
                log = np.frombuffer(ctx.log_bytes(), dtype=S.LOG_DTYPE)
            finally:
                ctx.close()
            d = log[log["kind"] == 1]
            lat = np.array([int(r["tick"]) + J[int(r["job"])].iter_ticks - J[int(r["job"])].request_ticks[int(r["a"])]
                            for r in d], dtype=np.float64) / 1e3
            out[f"{name}_lambda{lam}"] = {"latency_logical_us": {"avg": float(lat.mean()),
                                                                 "p99": float(np.percentile(lat, 99))},
                                          "requests_per_s_device": rs["n_dispatch"] / (rs["kernel_ns"] / 1e9)}
    return out


def sched_rate(S, device):
    """SURVEY §8(d) C1 row "scheduler ns/event": the device scheduler alone
    (SALUS_FLAG_NULL_WORK: admission, lanes, pages, dispatch, no tiles) on
    C2a, C3 and C4 (the oracle's simulation speed is in cpu_baseline)."""
    from workloads import c4_trace
    out = {}
    for name, (jobs, cap), pol, ml in (("c2a_pack", c2_trace("a"), S.PACK, 0),
                                       ("c3_fair8", c3_trace(), S.FAIR, 8),
                                       ("c4_srtf", c4_trace(), S.SRTF, 0)):
        ctx = S.Context(jobs, cap, pol, device=device, max_lanes=ml, null_work=True, log=False)
        try:
            ctx.run()
            ctx.run()
            rs = ctx.run_stats()
        finally:
            ctx.close()
        out[name] = {"ticks": int(rs["n_ticks"]), "dispatches": int(rs["n_dispatch"]),
                     "device_ns_per_tick": rs["kernel_ns"] / rs["n_ticks"],
                     "device_ns_per_dispatch": rs["kernel_ns"] / rs["n_dispatch"]}
    return out


def c2b_tensor(S, device, n_jobs=8, n_iters=20):
    """C2b: the compute-heavy sweep member, MLP [4096]^4
    B=2048 training (AI 683 flop/B, tensor-bound), n_jobs packed into one
    16 GiB arena: achieved dense bf16 TFLOP/s of the persistent kernel
    (algorithmic flops / device kernel time) against the measured peak."""
    jobs, cap = c2_trace("b", n_jobs=n_jobs, n_iters=n_iters)
    flops = sum(j.n_iters * algorithmic_flops(j.kind, j.dims, j.batch) for j in jobs)
    _, bf16, src = peaks()
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            sus = json.load(f).get("bf16_tflops_sustained", bf16)
    except Exception:  # noqa: BLE001
        sus = bf16
    ctx = S.Context(jobs, cap, S.PACK, device=device, log=False)
    try:
        ctx.run()
        ks = []
        for _ in range(3):
            ctx.run()
            ks.append(ctx.run_stats()["kernel_ns"] / 1e9)
    finally:
        ctx.close()
    k = float(np.median(ks))
    tf = flops / k / 1e12
    return {"config": f"C2b: {n_jobs} x MLP [4096]^4 B=2048 x {n_iters} iters, PACK, 16 GiB",
            "kernel_ms": k * 1e3, "iters_per_s": n_jobs * n_iters / k, "achieved_tflops": tf,
            "peak_tflops_sustained": sus, "frac_sustained": tf / sus, "peak_tflops_burst": bf16,
            "frac_burst": tf / bf16, "peak_source": src}


def online_submission(S, device, n_jobs=64, period_s=0.002, n_iters=20):
    """C2a-shaped training jobs (MLP [1024]^4, B=256)
    handed to the RUNNING kernel one every `period_s` (PACK, 1 GiB).  Host
    cost of salus_submit_live, and device time from the scheduler taking a
    job's arrival to its first tile (both clocks: globaltimer)."""
    import time
    from workloads import make_job
    jobs = [make_job(1 + k, TRAIN, 0, (1024, 1024, 1024, 1024), 256, n_iters, lr=1e-3, seed=1000 + k)
            for k in range(n_jobs)]
    ctx = S.Context([], 1 << 30, S.PACK, device=device, online=True, max_jobs=n_jobs, log=True)
    host_us = []
    try:
        ctx.run_async()
        time.sleep(0.02)
        for j in jobs:
            t0 = time.perf_counter()
            ctx.submit_live(j)
            host_us.append((time.perf_counter() - t0) * 1e6)
            time.sleep(period_s)
        ctx.end_submissions()
        stats = ctx.wait()
        rs = ctx.run_stats()
    finally:
        ctx.close()
    lat = [(s["wall_start_ns"] - s["wall_arrive_ns"]) / 1e3 for s in stats.values()]
    span = (max(s["wall_end_ns"] for s in stats.values()) - min(s["wall_arrive_ns"] for s in stats.values())) / 1e9
    return {"config": f"{n_jobs} x MLP[1024]^4 B=256 x {n_iters} iters, one live submission per "
                      f"{period_s * 1e3:.1f} ms into a running kernel, PACK, 1 GiB",
            "jobs": len(stats), "iterations": int(rs["n_dispatch"]),
            "submit_call_us": {"p50": float(np.median(host_us)), "p99": float(np.percentile(host_us, 99))},
            "arrival_to_first_tile_us": {"p50": float(np.median(lat)), "p99": float(np.percentile(lat, 99))},
            "iters_per_s_over_span": rs["n_dispatch"] / span}


def overhead_vs_standalone(S, device, dims=(1024, 1024, 1024, 1024), batch=256, iters=100):
    """SURVEY NEXT-1 (the analogue of PAPER.md fig:exp5-17): the
    per-iteration time of ONE job running alone inside Salus (device wall
    stamps) vs the same training step issued standalone through PyTorch /
    cuBLAS (bf16 GEMMs, fp32 master SGD) and replayed from a CUDA graph.
    A comparison baseline only -- never the product path."""
    import torch
    from workloads import make_job
    job = make_job(0, TRAIN, 0, dims, batch, iters, lr=1e-3, seed=1)
    ctx = S.Context([job], 1 << 30, S.PACK, device=device, log=True)
    ctx.run()
    w = ctx.wall()
    ctx.close()
    salus_us = float(np.median((w["end_ns"][1:] - w["start_ns"][1:]) / 1e3))
    dev = f"cuda:{device}"
    L = len(dims) - 1
    W32 = [torch.randn(dims[l], dims[l + 1], device=dev) * dims[l] ** -0.5 for l in range(L)]
    Wb = [w_.to(torch.bfloat16) for w_ in W32]
    X = torch.randn(batch, dims[0], device=dev).to(torch.bfloat16)
    T = torch.randn(batch, dims[-1], device=dev)

    def step():
        A = [X]
        for l in range(L):
            Z = A[-1] @ Wb[l]
            A.append(torch.relu(Z) if l < L - 1 else Z)
        G = ((A[-1].float() - T) / batch).to(torch.bfloat16)
        for l in range(L - 1, -1, -1):
            dW = (A[l].t() @ G).float()
            if l > 0:
                G = (G @ Wb[l].t()) * (A[l] > 0)
            W32[l].sub_(1e-3 * dW)
            Wb[l].copy_(W32[l])

    s = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(s):
        for _ in range(3):
            step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        for _ in range(5):
            g.replay()
        e0.record(s)
        for _ in range(iters):
            g.replay()
        e1.record(s)
    torch.cuda.synchronize()
    torch_us = e0.elapsed_time(e1) * 1e3 / iters
    return {"shape": f"MLP {list(dims)} B={batch}, one job alone", "salus_iter_us": salus_us,
            "standalone_torch_graph_iter_us": torch_us, "ratio": salus_us / torch_us}


def _oracle_sample_worker(args):
    """One process of the CPU baseline: fp64 oracle iterations (the oracle
    as it stands) of its share of the sampled jobs, one BLAS thread, until
    the deadline.  Returns (iterations, algorithmic flops, busy seconds)."""
    job_list, iters_per_job, deadline = args
    from threadpoolctl import threadpool_limits
    from oracle import layers as OL
    done, flops, busy = 0, 0, 0.0
    with threadpool_limits(1):
        for j in job_list:
            if time.time() >= deadline:
                break
            W = OL.init_weights(j)
            for k in range(min(iters_per_job, j.n_iters)):
                if time.time() >= deadline:
                    break
                t0 = time.perf_counter()
                if j.kind == TRAIN:
                    OL.train_step(W, j, k)
                else:
                    OL.infer_step(W, j, k)
                busy += time.perf_counter() - t0
                done += 1
                flops += algorithmic_flops(j.kind, j.dims, j.batch)
    return done, flops, busy


def cpu_baseline(jobs, cap, policy, budget_s=12.0, iters_per_job=2, seed=0):
    """The oracle as it stands, timed on this host's cores (the cpu_baseline
    leg: the only place bench.py runs oracle/): the full schedule simulation
    of the workload (one core, Python) plus fp64 layer math of a bounded
    sample -- a seeded shuffle of the jobs, `iters_per_job` iterations each,
    spread over one process per core (one BLAS thread each) for ~budget_s --
    extrapolated to every iteration of the workload by algorithmic flops."""
    import multiprocessing as mp
    from oracle import scheduler as OS
    t0 = time.perf_counter()
    ref = OS.simulate(jobs, cap, policy)
    t_sched = time.perf_counter() - t0
    cores = os.cpu_count() or 1
    order = [jobs[i] for i in np.random.default_rng(seed).permutation(len(jobs))]
    deadline = time.time() + budget_s
    with mp.get_context("spawn").Pool(cores) as pool:
        res = pool.map(_oracle_sample_worker, [(order[w::cores], iters_per_job, deadline) for w in range(cores)])
    done = sum(r[0] for r in res)
    rate = sum(r[1] / r[2] for r in res if r[2] > 0)            # flop/s over all cores
    total_iters = sum(j.n_iters for j in jobs)
    total_flops = sum(j.n_iters * algorithmic_flops(j.kind, j.dims, j.batch) for j in jobs)
    t_math = total_flops / rate if rate > 0 else float("inf")
    value = total_iters / (t_sched + t_math)
    return {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"full schedule simulation of {len(jobs)} jobs / {ref.n_ticks} ticks ({t_sched:.2f} s, "
                      f"1 core) + {done} fp64 iterations of a seeded job sample on {cores} processes x 1 BLAS "
                      f"thread ({rate / 1e9:.1f} GFLOP/s aggregate), extrapolated by flops to {total_iters} "
                      f"iterations ({t_math:.1f} s)",
            "oracle_sched_ns_per_tick": t_sched * 1e9 / max(1, ref.n_ticks),
            "extrapolated": True}


def run_reference(args, rank, world):
    """--impl reference: the oracle (CPU) is this tier's reference arm, timed
    on the host's cores on the headline workload (C2a): W untimed warm-up
    samples, then K timed steps, each a bounded sample of the workload."""
    if rank != 0:
        return
    jobs, cap = workload(1, 0)
    for _ in range(args.warmup):
        cpu_baseline(jobs, cap, S_PACK, budget_s=1.0, iters_per_job=1, seed=99)
    vals, cbs = [], []
    t_all = time.perf_counter()
    for k in range(args.steps):
        cb = cpu_baseline(jobs, cap, S_PACK, budget_s=max(3.0, 60.0 / max(1, args.steps)), seed=k)
        vals.append(cb["value"])
        cbs.append(cb)
    value = float(np.mean(vals))
    elapsed = time.perf_counter() - t_all
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": 1000.0 * sum(j.n_iters for j in jobs) / value,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": "C2a hyper-parameter sweep (BASELINE configs[1]), "
                                                        "oracle on CPU", "jobs": len(jobs),
                                            "iters_per_job": N_ITERS, "policy": "pack"},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cbs[-1]["cores"], "kind": "oracle",
                             "sample": cbs[-1]["sample"]},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "wall_s": elapsed}
    print(json.dumps(line), flush=True)


SIDE_SECTIONS = {
    "overhead": ("overhead_vs_standalone", lambda S, d, jobs, cap: overhead_vs_standalone(S, d)),
    "c3": ("c3_switch", lambda S, d, jobs, cap: switch_latency(S, d)),
    "c3live": ("c3_live", lambda S, d, jobs, cap: c3_live(S, d)),
    "c1": ("c1", lambda S, d, jobs, cap: c1_config(S, d)),
    "jct": ("jct_physical", lambda S, d, jobs, cap: jct_physical(S, d, jobs, cap)),
    "c4": ("c4_jct", lambda S, d, jobs, cap: c4_jct(S, d)),
    "c2b": ("c2b_tensor", lambda S, d, jobs, cap: c2b_tensor(S, d)),
    "evict": ("c4e_evict", lambda S, d, jobs, cap: c4e_evict(S, d)),
    "sched": ("scheduler_only", lambda S, d, jobs, cap: sched_rate(S, d)),
    "c3rate": ("c3_rate_sweep", lambda S, d, jobs, cap: c3_rate_sweep(S, d)),
    "online": ("online_submission", lambda S, d, jobs, cap: online_submission(S, d)),
}


def side_section(key, S, device, jobs=None, cap=None):
    """One secondary measurement of the bench line; errors are recorded, not raised."""
    if jobs is None:
        jobs, cap = workload(1, 0)
    t0 = time.time()
    try:
        out = SIDE_SECTIONS[key][1](S, device, jobs, cap)
        print(f"[bench] section {key}: ok ({time.time() - t0:.1f} s)", file=sys.stderr, flush=True)
        return out
    except Exception as exc:  # noqa: BLE001
        print(f"[bench] section {key}: ERROR {exc}", file=sys.stderr, flush=True)
        return {"error": str(exc)[:200]}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="salus", choices=["salus", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 (2000-job) strong-scaling section")
    ap.add_argument("--no-side", action="store_true", help="skip the single-GPU side sections (headline only)")
    ap.add_argument("--only", default="",
                    help="comma list of side sections to run alone and print (c1,c2b,c3,c3rate,c4,evict,jct,online,overhead,sched)")
    args = ap.parse_args()
    rank, world, local = dist_env()

    import torch
    import torch.distributed as dist
    if world > 1:
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    if args.impl == "reference":
        run_reference(args, rank, world)
        if world > 1:
            dist.barrier()
            dist.destroy_process_group()
        return

    from paper_1902_04610_b200 import build, salus as S
    torch.cuda.set_device(local)
    if rank == 0 or world == 1:
        build.build()
    if args.only:
        print(json.dumps({k: side_section(k, S, local) for k in args.only.split(",")}), flush=True)
        return
    if world > 1:
        dist.barrier()
    jobs, cap = workload(world, rank)
    n_iters_rank = sum(j.n_iters for j in jobs)
    ctx = S.Context(jobs, cap, S.PACK, device=local, log=True)
    for _ in range(max(3, args.warmup)):
        ctx.run()
    # one logged run for switch latency / JCT statistics (outside the timed region)
    stats = ctx.run()
    wall = ctx.wall()
    rs0 = ctx.run_stats()

    stream = torch.cuda.current_stream(local)
    kernel_ns = []
    with ClockSampler(local) as clk:
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            ctx.run()
            kernel_ns.append(ctx.run_stats()["kernel_ns"])
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    total_iters = n_iters_rank * world
    value = total_iters / (ms_max / 1000.0)

    # NCCL all_gather of per-GPU completion statistics
    from paper_1902_04610_b200 import multigpu as MG
    torch.cuda.synchronize()
    ta = time.perf_counter()
    all_stats = MG.gather_stats(stats, rank, world, device=f"cuda:{local}")
    allgather_us = (time.perf_counter() - ta) * 1e6

    # e2e: the same metric through the C ABI from host buffers (open + submit
    # + prepare [H2D job tables] + run + stats readback [D2H]) every step
    torch.cuda.synchronize()
    e2e_t = []
    h2d = d2h = 0
    for _ in range(max(1, min(args.steps, 3))):
        t0 = time.perf_counter()
        c2 = S.Context(jobs, cap, S.PACK, device=local, log=False)
        c2.run()
        r2 = c2.run_stats()
        h2d, d2h = r2["h2d_bytes"], r2["d2h_bytes"]
        c2.close()
        e2e_t.append(time.perf_counter() - t0)
    e2e_s = torch.tensor([float(np.median(e2e_t))], dtype=torch.float64, device=f"cuda:{local}")
    if world > 1:
        dist.all_reduce(e2e_s, op=dist.ReduceOp.MAX)
    e2e_value = total_iters / float(e2e_s.item())

    if rank == 0:
        flops, byts = work_per_iter(jobs[0])
        hbm, bf16, src = peaks()
        # one launch of the persistent kernel per step: its average duration is
        # the CUDA-event time of the step on the launching stream (the device
        # globaltimer span of the kernel is reported beside it)
        kms = ms
        kms_gt = float(np.mean(kernel_ns)) / 1e6
        achieved = n_iters_rank * byts / (kms / 1e3) / 1e9       # GB/s of the persistent kernel
        traffic = None
        tp = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                traffic = json.load(f).get("c2a_dram_bytes_per_launch")
        # switch latency: consecutive iterations of different jobs in a lane;
        # iteration gap: same job continuing (wall stamps of the logged run)
        sw, gap = [], []
        order = np.argsort(wall["seq"])
        w = wall[order]
        last = {}
        for r in w:
            ln = int(r["lane"])
            if ln in last:
                prev = last[ln]
                d = (int(r["start_ns"]) - int(prev["end_ns"])) / 1e3
                (gap if prev["job"] == r["job"] else sw).append(d)
            last[ln] = r
        # JCT vs the FIFO baseline (logical ticks), both from the device's
        # records: the timed PACK run and the same sweep under FIFO
        # (schedule only, SALUS_FLAG_NULL_WORK: logical ticks do not depend
        # on the work executed)
        from paper_1902_04610_b200 import metrics as PM
        cf = S.Context(jobs, cap, S.FIFO, device=local, log=False, null_work=True)
        try:
            fifo = PM.summarize(jobs, cf.run())
        finally:
            cf.close()
        pack = PM.summarize(jobs, stats)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": "C2a hyper-parameter sweep (BASELINE configs[1])",
                       "jobs": len(jobs) * world, "jobs_per_gpu": len(jobs), "iters_per_job": N_ITERS,
                       "model": "MLP [1024,1024,1024,1024]", "global_batch": 256, "policy": "pack",
                       "arena_gib_per_gpu": cap / 2**30, "parallelism": f"independent instance per GPU x{world}",
                       "l2": "no flush: the per-step working set (~37 packed jobs x 24 MiB persistent "
                             "+ lanes, ~1 GiB) exceeds the 126 MB L2"},
            "gpu_launches": args.steps,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": traffic,
                         "peak_source": f"{src} (MEASURED_PEAKS.json hbm_gbs)",
                         "algorithmic_bytes_per_iter": byts, "flops_per_iter": flops,
                         "tensor_frac": n_iters_rank * flops / (kms / 1e3) / 1e12 / bf16,
                         "launch_ms_events": kms, "launch_ms_globaltimer": kms_gt},
            "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "clocks": clk.summary(),
            "switch_us": {"n": len(sw), "p50": float(np.median(sw)) if sw else None,
                          "p99": float(np.percentile(sw, 99)) if sw else None},
            "iter_gap_us": {"n": len(gap), "p50": float(np.median(gap)) if gap else None,
                            "p99": float(np.percentile(gap, 99)) if gap else None},
            "jct": {"source": "device per-job records (FIFO: schedule-only run; PACK: the logged run)",
                    "avg_fifo_ticks": fifo["avg_jct_ticks"], "avg_pack_ticks": pack["avg_jct_ticks"],
                    "fifo_over_pack": fifo["avg_jct_ticks"] / pack["avg_jct_ticks"],
                    "makespan_fifo_over_pack": fifo["makespan_ticks"] / pack["makespan_ticks"]},
            "stats_allgathered": len(all_stats), "allgather_us": allgather_us,
            "sched_wait_frac": rs0["sched_wait_ns"] / max(1, rs0["kernel_ns"]),
        }
        # single-GPU side measurements: at N = 1 only (the other ranks would
        # otherwise wait minutes at the C5 barrier)
        for k in (SIDE_SECTIONS if world == 1 and not args.no_side else ()):
            line[SIDE_SECTIONS[k][0]] = side_section(k, S, local, jobs, cap)
        # the paper's figures (2x P100, TF 1.5, private traces) beside ours: context only
        try:
            if args.no_side:
                raise KeyError("side sections skipped (--no-side)")
            line["paper_context"] = {
                "avg_jct_fifo_over_srtf": {"ours_c4": line["c4_jct"]["fifo_over_srtf_avg_jct"], "paper": 3.19},
                "sweep_fifo_over_salus": {"ours_c2a_physical_makespan":
                                          line["jct_physical"]["fifo_over_pack_makespan"],
                                          "paper_makespan": "2.38 (superres_128) / 1.07 (resnet50_50)"},
                "inference_models_on_one_gpu": {"ours_c3": line["c3_switch"]["models_coresident"],
                                                "ours_switch_from_ready_p99_us":
                                                    line["c3_switch"]["switch_from_ready_us"]["p99"],
                                                "paper": "42 (42x consolidation)"},
                "paper_hardware": "2x Tesla P100 16 GB, TensorFlow 1.5, fp32 (P:594-597)"}
        except Exception as exc:  # noqa: BLE001
            line["paper_context"] = {"error": str(exc)[:200]}
        if not args.no_cpu_baseline and world == 1:
            line["cpu_baseline"] = cpu_baseline(jobs, cap, S_PACK)
    ctx.close()
    # C5 (configs[4], the metric's multi-GPU config): every rank takes part
    if not args.no_c5:
        try:
            c5 = c5_section(S, local, rank, world, with_cpu_baseline=(not args.no_cpu_baseline and world == 1))
        except Exception as exc:  # noqa: BLE001  (recorded; the headline line still prints)
            print(f"[bench] section c5: ERROR {exc}", file=sys.stderr, flush=True)
            c5 = {"error": str(exc)[:200]}
        if rank == 0:
            line["c5"] = c5
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
