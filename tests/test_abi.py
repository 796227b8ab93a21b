"""CPU-only checks of the C-ABI library: it loads, exports every symbol
include/salus.h declares, and its host-side validation (page rounding,
footprints, error codes) behaves as documented.  No compute calls."""
import ctypes as C
import os
import re

import pytest

from paper_1902_04610_b200 import build, salus as S
from workloads import PAGE_BYTES, TRAIN, INFER, footprint_bytes, make_job, c1_trace, c3_trace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    build.build()
    return S.lib()


def declared_functions():
    src = open(os.path.join(ROOT, "include", "salus.h")).read()
    return set(re.findall(r"^\s*(?:int|uint64_t|const char \*)\s*\*?\s*(salus_\w+)\s*\(", src, re.M))


def test_exports_every_declared_symbol(L):
    names = declared_functions()
    assert len(names) >= 12, names
    for n in names:
        assert hasattr(L, n), n
    assert names == set(S.EXPORTS)


def test_struct_sizes_match_header_layout():
    assert C.sizeof(S.JobStat) == 64
    assert C.sizeof(S.RunStats) == 136
    assert S.LOG_DTYPE.itemsize == 32 and S.WALL_DTYPE.itemsize == 40


def test_footprint_matches_documented_layout(L):
    for kind in (TRAIN, INFER):
        for dims, b in [((256, 256, 256), 1024), ((1024,) * 4, 256), ((576, 256, 256), 1), ((27, 100), 3)]:
            j = make_job(0, kind, 0, dims, b, 1, iter_ticks=1, request_ticks=(0,) if kind else ())
            assert S.footprint(j) == footprint_bytes(kind, dims, b)


def _open(L, cap=64 * PAGE_BYTES, policy=S.PACK, max_jobs=16):
    cfg = S.Config()
    cfg.policy = policy
    cfg.arena = 1 << 20            # never dereferenced by open/submit
    cfg.arena_bytes = cap
    cfg.capacity_bytes = cap
    cfg.max_jobs = max_jobs
    ctx = C.c_void_p()
    rc = L.salus_open(C.byref(cfg), C.byref(ctx))
    return rc, ctx


def test_open_validation(L):
    rc, ctx = _open(L)
    assert rc == 0
    L.salus_close(ctx)
    cfg = S.Config()
    cfg.arena = 1 << 20
    cfg.capacity_bytes = cfg.arena_bytes = 64 * PAGE_BYTES
    cfg.max_jobs = 1
    cfg.policy = 7
    ctx = C.c_void_p()
    assert L.salus_open(C.byref(cfg), C.byref(ctx)) == -1          # bad policy
    cfg.policy = 0
    cfg.page_bytes = 4096
    assert L.salus_open(C.byref(cfg), C.byref(ctx)) == -1          # v1: 64 KiB pages only
    cfg.page_bytes = 0
    cfg.arena_bytes = 10
    assert L.salus_open(C.byref(cfg), C.byref(ctx)) == -1          # arena < C
    assert L.salus_close(None) == 0


def test_submit_errors(L):
    rc, ctx = _open(L, cap=40 * PAGE_BYTES)
    assert rc == 0
    G = PAGE_BYTES
    ok = make_job(1, TRAIN, 0, (128, 128), 128, 2, iter_ticks=5)
    d, _ = S.job_desc(ok)
    assert L.salus_submit_job(ctx, C.byref(d)) == 0
    assert L.salus_submit_job(ctx, C.byref(d)) == -2                 # duplicate id
    big = make_job(2, TRAIN, 0, (128, 128), 128, 2, iter_ticks=5, persistent_bytes=20 * G,
                   ephemeral_bytes=20 * G + 1)                       # 20 + 21 pages > 40
    d, _ = S.job_desc(big)
    assert L.salus_submit_job(ctx, C.byref(d)) == -3                 # unschedulable (A22)
    small = make_job(3, TRAIN, 0, (128, 128), 128, 2, iter_ticks=5, persistent_bytes=10)
    d, _ = S.job_desc(small)
    assert L.salus_submit_job(ctx, C.byref(d)) == -1                 # below footprint
    zero = make_job(4, TRAIN, 0, (128, 128), 128, 2, iter_ticks=0)
    d, _ = S.job_desc(zero)
    assert L.salus_submit_job(ctx, C.byref(d)) == -1
    inf = make_job(5, INFER, 10, (128, 128), 1, 2, iter_ticks=5, request_ticks=(12, 11))
    d, keep = S.job_desc(inf)
    assert L.salus_submit_job(ctx, C.byref(d)) == -1                 # unsorted requests
    inf = make_job(6, INFER, 10, (128, 128), 1, 2, iter_ticks=5, request_ticks=(11, 12))
    d, keep = S.job_desc(inf, dump=S.DUMP_WEIGHT_STEPS)
    assert L.salus_submit_job(ctx, C.byref(d)) == -1                 # weight steps: TRAIN only
    n = C.c_uint64()
    assert L.salus_meta_bytes(ctx, C.byref(n)) == 0 and n.value > 0
    assert L.salus_run(ctx, None, 0, None) == -4                     # not prepared
    L.salus_close(ctx)


def test_whole_configs_validate(L):
    for jobs, cap in (c1_trace(), c3_trace()):
        rc, ctx = _open(L, cap=cap, max_jobs=len(jobs))
        assert rc == 0
        keep = []
        for j in jobs:
            d, k = S.job_desc(j)
            keep.append(k)
            assert L.salus_submit_job(ctx, C.byref(d)) == 0, j.job_id
        L.salus_close(ctx)


def test_evict_swap_and_migration_validation(L):
    """NEXT-3 / NEXT-4 entry points, host-side checks only (no GPU):
    SALUS_FLAG_EVICT is SRTF-only; the swap area is needed exactly when
    EVICT, DUMP_STATE or a resume image is present; a resume image must have
    the job's persistent-backing size; poll / read_state need a run."""
    import numpy as np
    G = PAGE_BYTES
    cfg = S.Config()
    cfg.arena = 1 << 20
    cfg.capacity_bytes = cfg.arena_bytes = 64 * G
    cfg.max_jobs = 4
    ctx = C.c_void_p()
    for pol in (S.FIFO, S.PACK, S.FAIR):
        cfg.policy, cfg.flags = pol, S.FLAG_EVICT
        assert L.salus_open(C.byref(cfg), C.byref(ctx)) == -1
    cfg.policy, cfg.flags = S.SRTF, S.FLAG_EVICT | S.FLAG_ONLINE
    assert L.salus_open(C.byref(cfg), C.byref(ctx)) == -1

    # no swap needed: 0 bytes, salus_set_swap refuses
    rc, ctx = _open(L, cap=64 * G)
    j = make_job(1, TRAIN, 0, (128, 256, 128), 128, 2, iter_ticks=5)
    d, _ = S.job_desc(j)
    assert L.salus_submit_job(ctx, C.byref(d)) == 0
    n = C.c_uint64(7)
    assert L.salus_swap_bytes(ctx, C.byref(n)) == 0 and n.value == 0
    buf = np.zeros(1 << 20, dtype=np.uint8)
    assert L.salus_set_swap(ctx, C.c_void_p(buf.ctypes.data), buf.nbytes) == -4
    assert L.salus_poll_stats(ctx, None, 0, None, None) == -4          # nothing running
    assert L.salus_read_state(ctx, 1, None, 0, C.byref(n)) == -4        # no run yet
    L.salus_close(ctx)

    # DUMP_STATE: one region = the job's persistent backing (8 pages here)
    rc, ctx = _open(L, cap=64 * G)
    d, _ = S.job_desc(j, S.DUMP_STATE)
    assert L.salus_submit_job(ctx, C.byref(d)) == 0
    assert L.salus_swap_bytes(ctx, C.byref(n)) == 0 and n.value == 8 * G
    L.salus_close(ctx)

    # resume: the image must have exactly that size; resume_iter needs an image
    rc, ctx = _open(L, cap=64 * G)
    d, keep = S.job_desc(j, 0, (np.zeros(8 * G - 1, dtype=np.uint8), 3))
    assert L.salus_submit_job(ctx, C.byref(d)) == -1
    d, keep = S.job_desc(j, 0, (np.zeros(8 * G, dtype=np.uint8), 3))
    assert L.salus_submit_job(ctx, C.byref(d)) == 0
    assert L.salus_swap_bytes(ctx, C.byref(n)) == 0 and n.value == 8 * G
    j2 = make_job(2, TRAIN, 0, (128, 256, 128), 128, 2, iter_ticks=5)
    d, _ = S.job_desc(j2)
    d.resume_iter = 4
    assert L.salus_submit_job(ctx, C.byref(d)) == -1
    L.salus_close(ctx)
