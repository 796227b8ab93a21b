#!/bin/bash
# sweep of SALUS_NARROW_BELOW (latency mode's narrow-tile threshold) on C4 (C5's generator)
for r in 1 2; do
for nb in 16 32 64 128; do
  echo "== SALUS_NARROW_BELOW=$nb round $r"
  SALUS_NARROW_BELOW=$nb timeout 200 python tools/run_cfg.py c4 srtf 1 2>&1 | tail -1
  SALUS_NARROW_BELOW=$nb timeout 200 python tools/run_cfg.py c4 pack 1 2>&1 | tail -1
done; done
