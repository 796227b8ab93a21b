#!/bin/bash
# A/B of the GEN/target prefetch: C4 under SRTF and PACK with
# SALUS_XPRE=1 (default) and =0, two interleaved rounds, plus C2a / C1 sanity
# (their jobs declare no persistent slack, so they never take the path).
# usage (on the GPU box): bash tools/ab_xpre.sh
for r in 1 2; do
for x in 1 0; do
  echo "== SALUS_XPRE=$x round $r"
  SALUS_XPRE=$x timeout 200 python tools/run_cfg.py c4 srtf 2 2>&1 | tail -1
  SALUS_XPRE=$x timeout 200 python tools/run_cfg.py c4 pack 2 2>&1 | tail -1
done; done
timeout 120 python tools/run_cfg.py c2 pack 3 2>&1 | tail -1
timeout 120 python tools/run_cfg.py c1 fifo 3 2>&1 | tail -1
