"""Thin ctypes binding of libsalus.so (include/salus.h).

Argument marshalling only: every step of the hot path (admission, lane
assignment, page allocation, dispatch, iteration execution) runs inside the
persistent CUDA kernel.  PyTorch is used for device memory (arena, meta) and
the stream.  If the library is missing this module raises — there is no CPU
fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, Iterable, List, Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SALUS_LIB", os.path.join(HERE, "libsalus.so"))

FIFO, SRTF, PACK, FAIR = 0, 1, 2, 3
TRAIN, INFER = 0, 1
FLAG_LOG, FLAG_NULL_WORK, FLAG_CHECK, FLAG_TRACE, FLAG_ONLINE, FLAG_EVICT = 1, 2, 4, 8, 16, 32
DUMP_OUTPUTS, DUMP_WEIGHTS, DUMP_STATE, DUMP_WEIGHT_STEPS = 1, 2, 4, 8
WEIGHTS = 0xFFFFFFFF


def weights_after(k: int) -> int:
    """salus_read_layers index of the weights after iteration k (DUMP_WEIGHT_STEPS)."""
    return 0x80000000 | int(k)

ERRORS = {-1: "E_INVAL", -2: "E_DUPLICATE", -3: "E_UNSCHEDULABLE", -4: "E_STATE",
          -5: "E_CAPACITY", -6: "E_CUDA", -7: "E_STUCK", -8: "E_TIMEOUT"}


class SalusError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{ERRORS.get(code, code)}: {msg}")
        self.code = code


class Config(C.Structure):
    _fields_ = [("device", C.c_int32), ("policy", C.c_uint32), ("arena", C.c_void_p),
                ("arena_bytes", C.c_uint64), ("stream", C.c_void_p), ("capacity_bytes", C.c_uint64),
                ("page_bytes", C.c_uint32), ("max_lanes", C.c_uint32), ("max_jobs", C.c_uint32),
                ("flags", C.c_uint32), ("switch_ticks", C.c_uint64), ("log_capacity", C.c_uint64),
                ("dump_bytes", C.c_uint64), ("n_workers", C.c_uint32), ("timeout_ms", C.c_uint32),
                ("trace_capacity", C.c_uint64)]


class JobDesc(C.Structure):
    _fields_ = [("job_id", C.c_uint32), ("kind", C.c_uint32), ("arrival_tick", C.c_int64),
                ("persistent_bytes", C.c_uint64), ("ephemeral_bytes", C.c_uint64),
                ("n_iters", C.c_uint32), ("n_layers", C.c_uint32), ("iter_ticks", C.c_uint64),
                ("dims", C.c_uint32 * 9), ("batch", C.c_uint32), ("lr", C.c_float),
                ("dump", C.c_uint32), ("seed", C.c_uint64), ("request_ticks", C.POINTER(C.c_int64)),
                ("resume_state", C.c_void_p), ("resume_bytes", C.c_uint64), ("resume_iter", C.c_uint32),
                ("_reserved", C.c_uint32)]


class JobStat(C.Structure):
    _fields_ = [("job_id", C.c_uint32), ("first_lane", C.c_uint32), ("admit_tick", C.c_int64),
                ("first_start_tick", C.c_int64), ("completion_tick", C.c_int64),
                ("completion_seq", C.c_uint64), ("wall_start_ns", C.c_uint64), ("wall_end_ns", C.c_uint64),
                ("wall_arrive_ns", C.c_uint64)]


class RunStats(C.Structure):
    _fields_ = [("n_dispatch", C.c_uint64), ("n_ticks", C.c_uint64), ("n_log", C.c_uint64),
                ("n_tasks", C.c_uint64), ("kernel_ns", C.c_uint64), ("wall_first_ns", C.c_uint64),
                ("wall_last_ns", C.c_uint64), ("sched_wait_ns", C.c_uint64), ("status", C.c_int32),
                ("n_workers", C.c_uint32), ("h2d_bytes", C.c_uint64), ("d2h_bytes", C.c_uint64),
                ("sched_fence_ns", C.c_uint64), ("sched_ring_ns", C.c_uint64),
                ("n_swap_out", C.c_uint64), ("n_swap_in", C.c_uint64), ("swap_bytes", C.c_uint64),
                ("swap_ns", C.c_uint64)]


WALL_DTYPE = np.dtype([("seq", "<u8"), ("lane", "<u4"), ("job", "<u4"), ("start_ns", "<u8"),
                       ("end_ns", "<u8"), ("append_ns", "<u8")])
TRACE_DTYPE = np.dtype([("task", "<u4"), ("smid", "<u4"), ("job", "<u4"), ("iter", "<u4"),
                        ("t_claim", "<u8"), ("t_ready", "<u8"), ("t_mma", "<u8"), ("t_end", "<u8")])
HANDOFF_DTYPE = np.dtype([("page", "<u4"), ("to", "<u4"), ("from", "<u4"), ("to_lane", "<u4"),
                          ("from_seq", "<u8"), ("to_seq", "<u8")])
LOG_DTYPE = np.dtype([("tick", "<i8"), ("kind", "<u4"), ("lane", "<u4"), ("job", "<u4"),
                      ("a", "<u4"), ("b", "<u8")])

EXPORTS = ["salus_open", "salus_job_footprint", "salus_submit_job", "salus_meta_bytes",
           "salus_prepare", "salus_run", "salus_read_run_stats", "salus_read_log",
           "salus_read_wall", "salus_read_trace", "salus_read_layers", "salus_last_error", "salus_close",
           "salus_run_async", "salus_submit_live", "salus_end_submissions", "salus_wait",
           "salus_swap_bytes", "salus_set_swap", "salus_poll_stats", "salus_read_state",
           "salus_submit_requests", "salus_read_requests", "salus_read_handoffs", "salus_debug_layout",
           "salus_debug_read"]

_lib = None
_POISONED: List[tuple] = []   # buffers of poisoned contexts, kept alive for the process


def lib():
    """Load libsalus.so (fails loudly if it was not built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_1902_04610_b200.build` "
                               "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        P = C.c_void_p
        L.salus_open.argtypes = [C.POINTER(Config), C.POINTER(P)]
        L.salus_job_footprint.argtypes = [C.POINTER(JobDesc), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.salus_submit_job.argtypes = [P, C.POINTER(JobDesc)]
        L.salus_meta_bytes.argtypes = [P, C.POINTER(C.c_uint64)]
        L.salus_prepare.argtypes = [P, P, C.c_uint64]
        L.salus_run.argtypes = [P, C.POINTER(JobStat), C.c_uint64, C.POINTER(C.c_uint64)]
        L.salus_read_run_stats.argtypes = [P, C.POINTER(RunStats)]
        L.salus_read_log.argtypes = [P, P, C.c_uint64, C.POINTER(C.c_uint64)]
        L.salus_read_wall.argtypes = [P, P, C.c_uint64, C.POINTER(C.c_uint64)]
        L.salus_read_trace.argtypes = [P, P, C.c_uint64, C.POINTER(C.c_uint64)]
        L.salus_read_layers.argtypes = [P, C.c_uint32, C.c_uint32, C.POINTER(C.c_float), C.c_uint64,
                                        C.POINTER(C.c_uint64)]
        L.salus_last_error.argtypes = [P]
        L.salus_last_error.restype = C.c_char_p
        L.salus_close.argtypes = [P]
        L.salus_run_async.argtypes = [P]
        L.salus_submit_live.argtypes = [P, C.POINTER(JobDesc)]
        L.salus_end_submissions.argtypes = [P]
        L.salus_read_handoffs.argtypes = [P, P, C.c_uint64, C.POINTER(C.c_uint64)]
        L.salus_submit_requests.argtypes = [P, C.POINTER(C.c_uint32), C.c_uint32]
        L.salus_read_requests.argtypes = [P, C.c_uint32, C.POINTER(C.c_int64), C.POINTER(C.c_uint64),
                                          C.c_uint64, C.POINTER(C.c_uint64)]
        L.salus_wait.argtypes = [P, C.POINTER(JobStat), C.c_uint64, C.POINTER(C.c_uint64)]
        L.salus_swap_bytes.argtypes = [P, C.POINTER(C.c_uint64)]
        L.salus_set_swap.argtypes = [P, P, C.c_uint64]
        L.salus_read_state.argtypes = [P, C.c_uint32, P, C.c_uint64, C.POINTER(C.c_uint64)]
        L.salus_poll_stats.argtypes = [P, C.POINTER(JobStat), C.c_uint64, C.POINTER(C.c_uint64),
                                       C.POINTER(C.c_uint64)]
        for name in EXPORTS:
            if name != "salus_last_error":
                getattr(L, name).restype = C.c_int
        _lib = L
    return _lib


def job_desc(job, dump: int = 0, resume=None):
    """Marshal a workloads.Job-like object into a salus_job; returns (desc, keepalive)."""
    d = JobDesc()
    d.job_id = job.job_id
    d.kind = job.kind
    d.arrival_tick = job.arrival_tick
    d.persistent_bytes = job.persistent_bytes
    d.ephemeral_bytes = job.ephemeral_bytes
    d.n_iters = job.n_iters
    d.n_layers = len(job.dims) - 1
    d.iter_ticks = job.iter_ticks
    for i, v in enumerate(job.dims):
        d.dims[i] = v
    d.batch = job.batch
    d.lr = job.lr
    d.dump = dump
    d.seed = job.seed & (2**64 - 1)
    keep = None
    if job.kind == INFER and len(job.request_ticks):   # empty: live requests (online contexts)
        keep = (C.c_int64 * len(job.request_ticks))(*job.request_ticks)
        d.request_ticks = C.cast(keep, C.POINTER(C.c_int64))
    if resume is not None:                       # migration (NEXT-4): (state image, iterations done)
        img, it = resume
        img = np.ascontiguousarray(img, dtype=np.uint8)
        d.resume_state = C.c_void_p(img.ctypes.data)
        d.resume_bytes = img.nbytes
        d.resume_iter = int(it)
        keep = (keep, img)
    return d, keep


def footprint(job):
    d, _ = job_desc(job)
    p, e = C.c_uint64(), C.c_uint64()
    rc = lib().salus_job_footprint(C.byref(d), C.byref(p), C.byref(e))
    if rc:
        raise SalusError(rc, "footprint")
    return p.value, e.value


class Context:
    """One Salus instance on one GPU: open + submit + prepare (salus.h)."""

    def __init__(self, jobs: Iterable, capacity_bytes: int, policy: int, *, device: int = 0,
                 max_lanes: int = 0, switch_ticks: int = 0, log: bool = True, null_work: bool = False,
                 check: bool = False, dump: Optional[Dict[int, int]] = None, n_workers: int = 0,
                 timeout_ms: int = 0, page_bytes: int = 65536, trace: bool = False,
                 trace_capacity: int = 0, online: bool = False, max_jobs: int = 0, dump_bytes: int = 0,
                 evict: bool = False, resume: Optional[Dict[int, tuple]] = None,
                 poison: Optional[bool] = None):
        import torch
        self._torch = torch
        self.L = lib()
        self.jobs = list(jobs)
        self.device = device
        G = page_bytes
        Cp = capacity_bytes // G
        self.arena = torch.empty(Cp * G, dtype=torch.uint8, device=f"cuda:{device}")
        # debug: fill the arena with 0xFF (NaN in bf16 and fp32) before every
        # run, so a read of a page this run has not written yet shows up as NaN
        # instead of whatever an earlier run left there (SALUS_POISON=1)
        self.poison = (os.environ.get("SALUS_POISON") == "1") if poison is None else poison
        self.stream = torch.cuda.current_stream(device)
        cfg = Config()
        cfg.device = device
        cfg.policy = policy
        cfg.arena = self.arena.data_ptr()
        cfg.arena_bytes = Cp * G
        cfg.stream = self.stream.cuda_stream
        cfg.capacity_bytes = capacity_bytes
        cfg.page_bytes = page_bytes
        cfg.max_lanes = max_lanes
        cfg.max_jobs = max(1, len(self.jobs), max_jobs)
        cfg.flags = ((FLAG_LOG if log else 0) | (FLAG_NULL_WORK if null_work else 0) |
                     (FLAG_CHECK if check else 0) | (FLAG_TRACE if trace else 0) |
                     (FLAG_ONLINE if online else 0) | (FLAG_EVICT if evict else 0))
        cfg.switch_ticks = switch_ticks
        cfg.n_workers = n_workers
        cfg.timeout_ms = timeout_ms
        cfg.trace_capacity = trace_capacity
        cfg.dump_bytes = dump_bytes          # 0: exactly what the submitted jobs dump
        self.flags = cfg.flags
        self.ctx = C.c_void_p()
        self._check(self.L.salus_open(C.byref(cfg), C.byref(self.ctx)), "open")
        dump = dump or {}
        resume = resume or {}
        for j in self.jobs:
            d, keep = job_desc(j, dump.get(j.job_id, 0), resume.get(j.job_id))
            self._check(self.L.salus_submit_job(self.ctx, C.byref(d)), f"submit {j.job_id}")
        self.swap = None
        # caller-owned pinned host swap area: eviction (A35) and migration state (NEXT-4)
        sb = C.c_uint64()
        self._check(self.L.salus_swap_bytes(self.ctx, C.byref(sb)), "swap_bytes")
        if sb.value:
            self.swap = torch.empty(sb.value + 256, dtype=torch.uint8, pin_memory=True)
            base = self.swap.data_ptr()
            self._check(self.L.salus_set_swap(self.ctx, C.c_void_p((base + 255) // 256 * 256), sb.value),
                        "set_swap")
        mb = C.c_uint64()
        self._check(self.L.salus_meta_bytes(self.ctx, C.byref(mb)), "meta_bytes")
        self.meta = torch.empty(max(256, mb.value), dtype=torch.uint8, device=f"cuda:{device}")
        if self.poison:
            # ... and the meta buffer all ones: a read of a table entry the
            # library never wrote (a lane page not backed) faults at once
            self.meta.fill_(0xFF)
        self._check(self.L.salus_prepare(self.ctx, C.c_void_p(self.meta.data_ptr()), mb.value), "prepare")

    def _poison(self):
        if self.poison:
            with self._torch.cuda.stream(self.stream):
                self.arena.fill_(0xFF)

    def _check(self, rc, what):
        if rc != 0:
            msg = self.L.salus_last_error(self.ctx) if getattr(self, "ctx", None) else b""
            raise SalusError(rc, f"{what}: {(msg or b'').decode()}")

    def _stats(self, fn, what) -> Dict[int, dict]:
        n = max(1, len(self.jobs))
        arr = (JobStat * n)()
        cnt = C.c_uint64()
        self._check(fn(self.ctx, arr, n, C.byref(cnt)), what)
        out = {}
        for s in arr[:cnt.value]:
            out[s.job_id] = {k: getattr(s, k) for k, _ in JobStat._fields_}
        return out

    def run(self) -> Dict[int, dict]:
        """One salus_run; returns {job_id: stat dict}."""
        self._poison()
        return self._stats(self.L.salus_run, "run")

    # ---- online submission (online=True)
    def run_async(self):
        """Launch the persistent kernel and return while it runs."""
        self._poison()
        self._check(self.L.salus_run_async(self.ctx), "run_async")

    def submit_live(self, job, dump: int = 0):
        """Hand a TRAIN job to the running kernel (arrival stamped on device)."""
        d, keep = job_desc(job, dump)
        self._check(self.L.salus_submit_live(self.ctx, C.byref(d)), f"submit_live {job.job_id}")
        self.jobs.append(job)

    def end_submissions(self):
        self._check(self.L.salus_end_submissions(self.ctx), "end_submissions")

    def submit_requests(self, job_ids):
        """Live inference requests: one request per entry, for INFER jobs
        submitted with no request ticks (arrival stamped on device)."""
        ids = np.ascontiguousarray(job_ids, dtype=np.uint32)
        self._check(self.L.salus_submit_requests(self.ctx, ids.ctypes.data_as(C.POINTER(C.c_uint32)), len(ids)),
                    "submit_requests")

    def handoffs(self) -> np.ndarray:
        """SALUS_FLAG_CHECK: fenced page hand-offs of the last run (I4)."""
        n = C.c_uint64()
        self._check(self.L.salus_read_handoffs(self.ctx, None, 0, C.byref(n)), "handoffs size")
        out = np.zeros(n.value, dtype=HANDOFF_DTYPE)
        self._check(self.L.salus_read_handoffs(self.ctx, C.c_void_p(out.ctypes.data), n.value, C.byref(n)),
                    "handoffs")
        return out

    def serve(self, due):
        """Submit live requests at their wall-clock times: `due` = sorted
        (seconds from now, job_id) pairs; requests that fall due together go
        in one salus_submit_requests call.  Returns each request's submit lag
        (seconds after its due time)."""
        import time
        t0 = time.perf_counter()
        lag, k = [], 0
        while k < len(due):
            now = time.perf_counter() - t0
            if due[k][0] > now:
                if due[k][0] - now > 5e-4:
                    time.sleep(due[k][0] - now - 3e-4)
                continue
            m = k
            while m < len(due) and due[m][0] <= now:
                m += 1
            self.submit_requests([jid for _, jid in due[k:m]])
            lag += [now - due[i][0] for i in range(k, m)]
            k = m
        return lag

    def requests(self, job_id: int):
        """(request ticks, globaltimer at which each live request was seen)."""
        n = C.c_uint64()
        self._check(self.L.salus_read_requests(self.ctx, job_id, None, None, 0, C.byref(n)), "requests size")
        ticks = np.zeros(n.value, dtype=np.int64)
        seen = np.zeros(n.value, dtype=np.uint64)
        self._check(self.L.salus_read_requests(self.ctx, job_id, ticks.ctypes.data_as(C.POINTER(C.c_int64)),
                                               seen.ctypes.data_as(C.POINTER(C.c_uint64)), n.value,
                                               C.byref(n)), "requests")
        return ticks, seen

    def wait(self) -> Dict[int, dict]:
        """Wait for the run to finish; returns {job_id: stat dict}."""
        return self._stats(self.L.salus_wait, "wait")

    def read_state(self, job_id: int) -> np.ndarray:
        """Migration (NEXT-4): the persistent state image of a DUMP_STATE job
        after the run -- resume it elsewhere with Context(resume={id: (img, iters)})."""
        n = C.c_uint64()
        self._check(self.L.salus_read_state(self.ctx, job_id, None, 0, C.byref(n)), "state size")
        out = np.empty(n.value, dtype=np.uint8)
        self._check(self.L.salus_read_state(self.ctx, job_id, C.c_void_p(out.ctypes.data), n.value, C.byref(n)),
                    "state")
        return out

    def poll_stats(self):
        """Streaming stats (NEXT-4) while run_async is in flight:
        ({job_id: stat dict as it stands}, number of jobs physically done)."""
        n = max(1, len(self.jobs))
        arr = (JobStat * n)()
        cnt, done = C.c_uint64(), C.c_uint64()
        self._check(self.L.salus_poll_stats(self.ctx, arr, n, C.byref(cnt), C.byref(done)), "poll_stats")
        return ({s.job_id: {k: getattr(s, k) for k, _ in JobStat._fields_} for s in arr[:cnt.value]},
                int(done.value))

    def run_stats(self) -> dict:
        rs = RunStats()
        self._check(self.L.salus_read_run_stats(self.ctx, C.byref(rs)), "run_stats")
        return {k: getattr(rs, k) for k, _ in RunStats._fields_}

    def log_bytes(self) -> bytes:
        n = C.c_uint64()
        self._check(self.L.salus_read_log(self.ctx, None, 0, C.byref(n)), "log size")
        buf = C.create_string_buffer(max(1, n.value))
        self._check(self.L.salus_read_log(self.ctx, buf, n.value, C.byref(n)), "log")
        return buf.raw[:n.value]

    def wall(self) -> np.ndarray:
        n = C.c_uint64()
        self._check(self.L.salus_read_wall(self.ctx, None, 0, C.byref(n)), "wall size")
        out = np.zeros(n.value, dtype=WALL_DTYPE)
        self._check(self.L.salus_read_wall(self.ctx, C.c_void_p(out.ctypes.data), n.value, C.byref(n)), "wall")
        return out

    def trace(self) -> np.ndarray:
        n = C.c_uint64()
        self._check(self.L.salus_read_trace(self.ctx, None, 0, C.byref(n)), "trace size")
        out = np.zeros(n.value, dtype=TRACE_DTYPE)
        self._check(self.L.salus_read_trace(self.ctx, C.c_void_p(out.ctypes.data), n.value, C.byref(n)), "trace")
        return out

    def layers(self, job_id: int, iteration: int) -> np.ndarray:
        n = C.c_uint64()
        self._check(self.L.salus_read_layers(self.ctx, job_id, iteration, None, 0, C.byref(n)), "layers size")
        out = np.zeros(n.value, dtype=np.float32)
        self._check(self.L.salus_read_layers(self.ctx, job_id, iteration,
                                             out.ctypes.data_as(C.POINTER(C.c_float)), n.value, C.byref(n)),
                    "layers")
        return out

    def close(self):
        if getattr(self, "ctx", None):
            if self.L.salus_close(self.ctx) != 0:
                # poisoned context (salus.h): a kernel that ignored the abort may
                # still touch the arena / meta / swap -- never free them
                _POISONED.append(tuple(getattr(self, k, None) for k in ("arena", "meta", "swap")))
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass
