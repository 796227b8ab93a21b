"""ORACLE — test infrastructure only.

A plain, slow, obviously-correct CPU implementation of what the Salus hot
path computes (arXiv 1902.04610), written from PAPER.md and the readings in
DESIGN.md ("Readings of the paper").  Only `tests/`, `__graft_entry__.smoke()`
and `bench.py` (its `cpu_baseline` leg and `--impl reference`) may import it.
The product path (`paper_1902_04610_b200`) never imports, links or executes
anything under `oracle/`, and shares no code with it: the only shared module
is `workloads/` (seeded input generators, none of the method's arithmetic).

Modules
  scheduler.py — Algorithm 1 (GPU Lane Assignment), the safety
                 condition, the FIFO/SRTF/PACK/FAIR policies
                 (§4) and the iteration-granular event loop.
  layers.py    — fp64 dense MLP forward/backward/SGD per dispatched iteration.
  datagen.py   — the counter-based data generator.
  metrics.py   — JCT / makespan / queuing / nearest-rank percentile (tab:exp11).
  logfmt.py    — the canonical 32-byte log record encoding.

Parity pins: every function is pinned by `tests/test_oracle_*.py` against
values the paper prints, closed forms, brute force and finite differences.
"""
