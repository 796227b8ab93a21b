#!/bin/bash
# A/B of the latency-mode knobs: narrow tiles and the relaxed
# backward barrier, on the latency-bound configs (C1, C4) and C2a as a check.
for r in 1 2; do
for cfg in "0 0" "32 0" "0 1" "32 1"; do
  set -- $cfg
  echo "== SALUS_NARROW_BELOW=$1 SALUS_RELAX=$2 round $r"
  export SALUS_NARROW_BELOW=$1 SALUS_RELAX=$2
  timeout 100 python tools/run_cfg.py c1 fifo 3 2>&1 | tail -1
  timeout 200 python tools/run_cfg.py c4 srtf 1 2>&1 | tail -1
  timeout 200 python tools/run_cfg.py c4 pack 1 2>&1 | tail -1
  [ $r = 1 ] && timeout 200 python tools/run_cfg.py c2 pack 2 2>&1 | tail -1
done; done
