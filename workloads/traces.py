"""Seeded synthetic job traces shaped like the paper's workloads.

Salus (arXiv 1902.04610) evaluates on private TensorFlow traces (PAPER.md
§5.1, "a job trace of 100 workloads ... followed one found in a
production cluster"), a 300-job hyper-parameter sweep (§5.2) and
42 low-rate inference models (§5.3).  None of those traces or
models is available, so this module generates seeded stand-ins with the
shapes SURVEY.md §8(d) fixes (configs C1..C5 of BASELINE.json).

Every job is a small dense MLP (the "small-model forward/backward dense
layers" of the north star).  A job carries the quantities the paper's
problem statement gives the scheduler: persistent bytes P_i and ephemeral
bytes E_i, a known duration n_iters * iter_ticks (P:532,
"we assume the job execution time is known"), and an arrival time.

Nothing here decides anything the method decides; it only produces inputs.
"""
from __future__ import annotations

import dataclasses
import hashlib
import json
import math
from typing import List, Optional, Sequence, Tuple

import numpy as np

TRAIN = 0
INFER = 1
PAGE_BYTES = 65536          # G in SURVEY §8(c)-A18
GIB = 1 << 30
MIB = 1 << 20


def pad128(x: int) -> int:
    """Every GEMM dimension is padded to a multiple of 128 in the device
    layout."""
    return (int(x) + 127) // 128 * 128


@dataclasses.dataclass(frozen=True)
class Job:
    job_id: int
    kind: int                  # TRAIN | INFER
    arrival_tick: int          # logical ns
    persistent_bytes: int      # declared P_i
    ephemeral_bytes: int       # declared E_i
    n_iters: int               # INFER: number of requests
    iter_ticks: int            # known per-iteration duration
    dims: Tuple[int, ...]      # d_0 .. d_L, L <= 8
    batch: int
    lr: float                  # fp32-representable
    seed: int                  # u64
    request_ticks: Tuple[int, ...] = ()   # INFER only, len == n_iters

    @property
    def n_layers(self) -> int:
        return len(self.dims) - 1


# --------------------------------------------------------------------------
# Footprint of the device layout (what the library checks declared >= actual)
# and the algorithmic work per iteration.
# --------------------------------------------------------------------------

def footprint_bytes(kind: int, dims: Sequence[int], batch: int) -> Tuple[int, int]:
    """(P_actual, E_actual) of the device layout described in DESIGN.md.

    Training persistent: fp32 master + two bf16 copies per weight (8 B/param).
    Inference persistent: one bf16 copy (2 B/param).
    Training ephemeral: X, A_1..A_{L-1} (bf16) + two ping-pong gradient
    buffers of B x max(d).  Inference ephemeral: X, A_1..A_L (bf16).
    """
    dp = [pad128(d) for d in dims]
    bp = pad128(batch)
    L = len(dims) - 1
    wparams = sum(dp[l - 1] * dp[l] for l in range(1, L + 1))
    if kind == TRAIN:
        p = 8 * wparams
        e = 2 * bp * (dp[0] + sum(dp[1:L])) + 2 * (2 * bp * max(dp))
    else:
        p = 2 * wparams
        e = 2 * bp * sum(dp)
    return p, e


def algorithmic_flops(kind: int, dims: Sequence[int], batch: int) -> int:
    """training 4B*W + 2B*sum_{l>=2} d_{l-1}d_l; inference 2B*W."""
    L = len(dims) - 1
    W = sum(dims[l - 1] * dims[l] for l in range(1, L + 1))
    if kind == TRAIN:
        return 4 * batch * W + 2 * batch * sum(dims[l - 1] * dims[l] for l in range(2, L + 1))
    return 2 * batch * W


def algorithmic_bytes(kind: int, dims: Sequence[int], batch: int) -> int:
    """SURVEY §8(d) compulsory HBM bytes per iteration (unpadded)."""
    L = len(dims) - 1
    B = batch
    W = sum(dims[l - 1] * dims[l] for l in range(1, L + 1))
    inner = sum(dims[1:L])
    if kind == TRAIN:
        return 2 * B * dims[0] + 2 * B * dims[L] + 4 * B * sum(dims[1:]) + 4 * B * inner + 12 * W
    return 2 * B * dims[0] + 2 * B * dims[L] + 4 * B * inner + 2 * W


def iter_ticks_for(kind: int, dims: Sequence[int], batch: int) -> int:
    """ceil(max(flops/1e5, bytes/1e3)) + 2000 (trace spec)."""
    f = algorithmic_flops(kind, dims, batch)
    b = algorithmic_bytes(kind, dims, batch)
    return max(-(-f // 100000), -(-b // 1000)) + 2000


def _f32(x: float) -> float:
    return float(np.float32(x))


def _round_up(x: int, g: int) -> int:
    return (int(x) + g - 1) // g * g


def make_job(job_id, kind, arrival_tick, dims, batch, n_iters, *, iter_ticks=None,
             persistent_bytes=None, ephemeral_bytes=None, lr=1e-3, seed=None,
             request_ticks=()) -> Job:
    """Build a job whose declared P/E default to the device footprint."""
    dims = tuple(int(d) for d in dims)
    p_act, e_act = footprint_bytes(kind, dims, batch)
    if persistent_bytes is None:
        persistent_bytes = p_act
    if ephemeral_bytes is None:
        ephemeral_bytes = e_act
    if iter_ticks is None:
        iter_ticks = iter_ticks_for(kind, dims, batch)
    return Job(job_id=int(job_id), kind=int(kind), arrival_tick=int(arrival_tick),
               persistent_bytes=int(persistent_bytes), ephemeral_bytes=int(ephemeral_bytes),
               n_iters=int(n_iters), iter_ticks=int(iter_ticks), dims=dims, batch=int(batch),
               lr=_f32(lr), seed=int(seed if seed is not None else job_id) & (2**64 - 1),
               request_ticks=tuple(int(t) for t in request_ticks))


# --------------------------------------------------------------------------
# Configs of BASELINE.json
# --------------------------------------------------------------------------

def c1_trace() -> Tuple[List[Job], int]:
    """C1 = hand trace HW-C1: two 2-layer width-256 MLPs.

    J0: arrival 0, n=10, c=8000, B=1024; J1: arrival 5000, n=10, c=1000,
    B=128.  p=16 pages, e={48,6} pages.  C = 1 GiB.
    """
    G = PAGE_BYTES
    jobs = [
        make_job(0, TRAIN, 0, (256, 256, 256), 1024, 10, iter_ticks=8000,
                 persistent_bytes=16 * G, ephemeral_bytes=48 * G, lr=1e-3, seed=0),
        make_job(1, TRAIN, 5000, (256, 256, 256), 128, 10, iter_ticks=1000,
                 persistent_bytes=16 * G, ephemeral_bytes=6 * G, lr=1e-3, seed=1),
    ]
    return jobs, GIB


def c1_tie_trace() -> Tuple[List[Job], int]:
    """C1 identical-job tie variant: both B=256, arrival 0."""
    G = PAGE_BYTES
    jobs = [make_job(j, TRAIN, 0, (256, 256, 256), 256, 10, iter_ticks=3000,
                     persistent_bytes=16 * G, ephemeral_bytes=12 * G, lr=1e-3, seed=j)
            for j in range(2)]
    return jobs, GIB


def c2_trace(variant: str = "a", n_jobs: int = 300, n_iters: int = 100,
             job_id_base: int = 0) -> Tuple[List[Job], int]:
    """C2 hyper-parameter sweep (§5.2): 300 jobs ready at 0.

    lr_j = 10^(-4 + 2j/299), seed j.
    (a) [1024]^4 B=256, P=24 MiB, E=3.5 MiB, C=1 GiB -> ~37 lanes.
    (b) [4096]^4 B=2048, compute-heavy (the resnet50_50 regime), C=16 GiB.
    """
    jobs = []
    for j in range(n_jobs):
        lr = 10.0 ** (-4.0 + 2.0 * j / max(1, (n_jobs - 1)))
        jid = job_id_base + j
        if variant == "a":
            jobs.append(make_job(jid, TRAIN, 0, (1024,) * 4, 256, n_iters,
                                 persistent_bytes=24 * MIB, ephemeral_bytes=7 * MIB // 2,
                                 lr=lr, seed=jid))
        elif variant == "b":
            jobs.append(make_job(jid, TRAIN, 0, (4096,) * 4, 2048, n_iters,
                                 ephemeral_bytes=96 * MIB, lr=lr * 0.1, seed=jid))
        else:
            raise ValueError(variant)
    return jobs, (GIB if variant == "a" else 16 * GIB)


# 14 architectures for C3: 7 MLPs + 7 conv-as-GEMM chains.
C3_ARCHS = [
    # (dims, batch)   MLPs, b in {1,4,8,16}
    ((256, 256, 256), 1),
    ((512, 512, 512, 512), 4),
    ((1024, 1024, 1024), 8),
    ((1024, 1024, 1024, 1024, 1024), 16),
    ((2048, 2048, 2048), 4),
    ((4096, 4096, 4096), 1),
    ((768, 3072, 768, 768), 8),
    # conv-as-GEMM: im2col 3x3 first layer (K = 9*C_in), then 1x1 convs;
    # batch = spatial positions H*W in {1024, 3136}
    ((9 * 64, 256, 256, 256), 1024),
    ((9 * 32, 128, 128, 256, 256), 3136),
    ((9 * 128, 256, 512), 1024),
    ((9 * 16, 64, 64, 128), 3136),
    ((9 * 256, 512, 512, 512), 1024),
    ((9 * 64, 128, 256), 3136),
    ((9 * 32, 64, 128, 128, 256), 1024),
]


def c3_trace(rate_per_s: float = 20.0, n_requests: int = 200, seed: int = 3,
             instances: int = 3) -> Tuple[List[Job], int]:
    """C3: 42 inference models = 14 architectures x 3 instances, all arrive
    at 0 (§5.3); Poisson requests at `rate_per_s` per model
    (ticks are ns), 200 requests each.  C = 16 GiB (the P100's 16 GB)."""
    rng = np.random.default_rng(seed)
    jobs = []
    jid = 0
    mean_gap = 1e9 / rate_per_s
    for inst in range(instances):
        for dims, b in C3_ARCHS:
            gaps = rng.exponential(mean_gap, size=n_requests)
            ticks = np.floor(np.cumsum(gaps)).astype(np.int64)
            jobs.append(make_job(jid, INFER, 0, dims, b, n_requests, lr=0.0, seed=1000 + jid,
                                 request_ticks=tuple(int(t) for t in ticks)))
            jid += 1
    return jobs, 16 * GIB


def _loguniform(rng, lo, hi):
    return float(math.exp(rng.uniform(math.log(lo), math.log(hi))))


def c4_trace(n_jobs: int = 100, seed: int = 4, load: float = 1.2, burst: bool = False,
             rate_scale: float = 1.0, job_id_base: int = 0, p_scale: float = 1.0) -> Tuple[List[Job], int]:
    """C4: mixed training trace (stand-in for the unpublished Gandiva
    distribution).  n log-uniform [10, 2000]; width {256..4096} x
    depth {2,3,4} x B {64..1024}; declared P log-uniform [110.9 MB, 822.2 MB]
    (P:159), E log-uniform up to 13.8 GB - P; Poisson arrivals at
    offered load `load` of one lane.  C = 16 GiB.

    `p_scale` multiplies the declared P (C4e, the eviction config of
    SURVEY §8(f) NEXT-3: p_scale 8 -> P in [0.89, 6.6] GB, so admitted jobs'
    persistent memory fills the GPU and SRTF admission has to evict)."""
    rng = np.random.default_rng(seed)
    widths = [256, 512, 1024, 2048, 4096]
    batches = [64, 128, 256, 512, 1024]
    proto = []
    for j in range(n_jobs):
        w = widths[int(rng.integers(0, len(widths)))]
        depth = int(rng.integers(2, 5))
        b = batches[int(rng.integers(0, len(batches)))]
        n = int(round(_loguniform(rng, 10, 2000)))
        dims = (w,) * (depth + 1)
        p_act, e_act = footprint_bytes(TRAIN, dims, b)
        P = max(p_act, int(p_scale * _loguniform(rng, 110.9e6, 822.2e6)))
        e_lo = max(e_act, 64 * MIB)
        e_hi = max(e_lo + 1, int(13.8e9) - P)
        E = max(e_act, int(_loguniform(rng, e_lo, e_hi)))
        lr = _loguniform(rng, 1e-4, 1e-2)
        proto.append((dims, b, n, P, E, lr))
    c = [iter_ticks_for(TRAIN, d, b) for (d, b, *_r) in proto]
    mean_dur = float(np.mean([n * ci for (_, _, n, *_r), ci in zip(proto, c)]))
    rate = load / mean_dur * rate_scale
    gaps = rng.exponential(1.0 / rate, size=n_jobs)
    arr = np.floor(np.cumsum(gaps)).astype(np.int64) - int(math.floor(gaps[0]))
    jobs = []
    for j, ((dims, b, n, P, E, lr), ci) in enumerate(zip(proto, c)):
        jid = job_id_base + j
        jobs.append(make_job(jid, TRAIN, 0 if burst else int(arr[j]), dims, b, n, iter_ticks=ci,
                             persistent_bytes=P, ephemeral_bytes=E, lr=lr, seed=jid))
    return jobs, 16 * GIB


def c5_trace(n_jobs: int = 2000, seed: int = 5, burst: bool = True,
             gpus: int = 1) -> Tuple[List[Job], int]:
    """C5: 2000 jobs from the C4 generator.  burst: all arrive at 0 (PACK
    throughput scaling); otherwise Poisson at rate x G (constant per-GPU load)."""
    return c4_trace(n_jobs=n_jobs, seed=seed, burst=burst, rate_scale=float(gpus))


# --------------------------------------------------------------------------
# Small generators for property / parity tests
# --------------------------------------------------------------------------

def random_sched_trace(rng: np.random.Generator, n_jobs: int, *, cap_pages: int = 64,
                       max_iters: int = 6, max_ticks: int = 20, arrival_span: int = 60,
                       infer_frac: float = 0.0, max_requests_span: int = 80,
                       same_ticks: bool = False) -> Tuple[List[Job], int]:
    """Random tiny traces (sizes in pages) for scheduler property tests.
    Layer dims are tiny and irrelevant to the schedule."""
    G = PAGE_BYTES
    jobs = []
    for j in range(n_jobs):
        p = int(rng.integers(1, max(2, cap_pages // 4)))
        e = int(rng.integers(0, max(1, cap_pages - p)))
        if rng.random() < 0.1:
            e = 0
        kind = INFER if rng.random() < infer_frac else TRAIN
        n = int(rng.integers(1, max_iters + 1))
        c = 1 if same_ticks else int(rng.integers(1, max_ticks + 1))
        a = int(rng.integers(0, arrival_span + 1))
        req = ()
        if kind == INFER:
            req = tuple(sorted(int(a + x) for x in rng.integers(0, max_requests_span + 1, size=n)))
        jobs.append(make_job(j, kind, a, (128, 128), 128, n, iter_ticks=c,
                             persistent_bytes=p * G - int(rng.integers(0, G)),
                             ephemeral_bytes=max(0, e * G - int(rng.integers(0, G))) if e else 0,
                             lr=1e-3, seed=j, request_ticks=req))
    return jobs, cap_pages * G + int(rng.integers(0, G))


def tiny_math_trace(kind: int = TRAIN, n_jobs: int = 2, dims=(128, 256, 128), batch: int = 128,
                    n_iters: int = 3, lr: float = 1e-2) -> Tuple[List[Job], int]:
    """Small jobs for GEMM parity: several tiles and a ragged batch tail."""
    jobs = []
    for j in range(n_jobs):
        req = tuple(range(100 * j, 100 * j + 10 * n_iters, 10)) if kind == INFER else ()
        jobs.append(make_job(j, kind, 100 * j, dims, batch, n_iters, lr=lr, seed=77 + j,
                             request_ticks=req))
    return jobs, GIB


# --------------------------------------------------------------------------
# Trace file format (JSONL, one job per line) + hash
# --------------------------------------------------------------------------

def to_jsonl(jobs: Sequence[Job]) -> str:
    lines = []
    for j in jobs:
        d = dataclasses.asdict(j)
        d["dims"] = list(j.dims)
        d["request_ticks"] = list(j.request_ticks)
        lines.append(json.dumps(d, sort_keys=True))
    return "\n".join(lines) + ("\n" if lines else "")


def from_jsonl(text: str) -> List[Job]:
    jobs = []
    seen = set()
    for n, line in enumerate(text.splitlines(), 1):
        if not line.strip():
            continue
        try:
            d = json.loads(line)
            d["dims"] = tuple(d["dims"])
            d["request_ticks"] = tuple(d.get("request_ticks", ()))
            job = Job(**d)
        except Exception as exc:  # noqa: BLE001
            raise ValueError(f"trace line {n}: {exc}") from exc
        if job.job_id in seen:
            raise ValueError(f"trace line {n}: duplicate job id {job.job_id}")
        seen.add(job.job_id)
        jobs.append(job)
    return jobs


def trace_sha256(jobs: Sequence[Job]) -> str:
    return hashlib.sha256(to_jsonl(jobs).encode()).hexdigest()
