"""Seeded synthetic inputs shared by the CUDA path and the oracle.

This package holds only input *generators* (job traces shaped like the
paper's workloads) and the trace-file format.  It contains
none of the method's arithmetic: no lane assignment, no scheduling policy,
no layer math.  Both `oracle/` and the product binding may import it.
"""
from .traces import (  # noqa: F401
    Job, TRAIN, INFER, PAGE_BYTES,
    pad128, footprint_bytes, algorithmic_flops, algorithmic_bytes, iter_ticks_for,
    make_job, c1_trace, c1_tie_trace, c2_trace, c3_trace, c4_trace, c5_trace,
    random_sched_trace, tiny_math_trace,
    to_jsonl, from_jsonl, trace_sha256,
)
