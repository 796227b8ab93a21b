"""Canonical schedule log (ORACLE — test infrastructure only).

Fixed-width little-endian 32-byte records, SURVEY §8(c) "Canonical log":

    int64 tick; uint32 kind; uint32 lane; uint32 job; uint32 a; uint64 b

The byte-compare of this log between the CUDA path and the oracle is the
schedule-parity test.  The record kinds and field meanings are part of the
C ABI contract (include/salus.h, SALUS_REC_*); they are restated here, not
imported, so the oracle shares no code with the product.
"""
import struct

import numpy as np

REC = struct.Struct("<qIIIIQ")
assert REC.size == 32

DISPATCH = 1      # lane, job, a = iteration index (done_j), b = dispatch seq
LANE_OPEN = 2     # lane, job, a = L pages
LANE_REUSE = 3    # lane, job, a = L pages
LANE_RESIZE = 4   # lane, job, a = new L, b = old L
LANE_SHRINK = 5   # lane, job (the finishing job), a = new L, b = old L
LANE_CLOSE = 6    # lane, job (the finishing job)
JOB_QUEUED = 7    # lane = NONE, job
JOB_ADMIT = 8     # lane, job, a = p pages, b = e pages
JOB_FINISH = 9    # lane, job, a = n iterations, b = completion_seq
JOB_EVICT = 10    # lane (left), job (the victim), a = p pages, b = iterations done (A35)
JOB_RESTORE = 11  # lane, job, a = p pages, b = e pages: a swapped job re-admitted (A35)

NONE32 = 0xFFFFFFFF

NAMES = {DISPATCH: "DISPATCH", LANE_OPEN: "LANE_OPEN", LANE_REUSE: "LANE_REUSE",
         LANE_RESIZE: "LANE_RESIZE", LANE_SHRINK: "LANE_SHRINK", LANE_CLOSE: "LANE_CLOSE",
         JOB_QUEUED: "JOB_QUEUED", JOB_ADMIT: "JOB_ADMIT", JOB_FINISH: "JOB_FINISH",
         JOB_EVICT: "JOB_EVICT", JOB_RESTORE: "JOB_RESTORE"}

DTYPE = np.dtype([("tick", "<i8"), ("kind", "<u4"), ("lane", "<u4"), ("job", "<u4"),
                  ("a", "<u4"), ("b", "<u8")])


def encode(records) -> bytes:
    return b"".join(REC.pack(*r) for r in records)


def decode(buf: bytes):
    n = len(buf) // REC.size
    return [REC.unpack_from(buf, i * REC.size) for i in range(n)]


def as_array(buf: bytes) -> np.ndarray:
    return np.frombuffer(buf, dtype=DTYPE)


def fmt(rec) -> str:
    t, k, lane, job, a, b = rec
    ln = "-" if lane == NONE32 else str(lane)
    return f"t={t} {NAMES.get(k, k)} lane={ln} job={job} a={a} b={b}"
