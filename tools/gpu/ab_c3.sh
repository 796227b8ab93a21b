#!/bin/bash
# A/B on C3 (inference): K9 tiles (SALUS_SWAP) x narrow lanes x eager lanes, same box
for r in 1 2; do
for cfg in "1 2 8" "0 2 8" "1 0 8" "0 0 8" "0 0 0"; do
  set -- $cfg
  export SALUS_SWAP=$1 SALUS_NARROW_LANES=$2 SALUS_EAGER_LANES=$3
  echo "== SWAP=$1 NARROW_LANES=$2 EAGER_LANES=$3 round $r"
  timeout 200 python tools/run_cfg.py c3 fair 2 2>&1 | tail -1
  timeout 200 python tools/run_cfg.py c3 pack 2 2>&1 | tail -1
done; done
unset SALUS_SWAP SALUS_NARROW_LANES SALUS_EAGER_LANES
timeout 200 python tools/run_cfg.py c2 pack 3 2>&1 | tail -1
