#!/bin/bash
# A/B of the K9 skinny-batch tiles (SALUS_SWAP) and their split-K (SALUS_SPLIT_MAX=1: none)
for r in 1 2; do
for cfg in "0 1" "1 1"; do
  set -- $cfg
  echo "== SALUS_SWAP=$1 SALUS_SPLIT_MAX=$2 round $r"
  export SALUS_SWAP=$1 SALUS_SPLIT_MAX=$2
  timeout 200 python tools/run_cfg.py c4 srtf 1 2>&1 | tail -1
  timeout 200 python tools/run_cfg.py c4 pack 1 2>&1 | tail -1
  timeout 200 python tools/run_cfg.py c3 fair 2 2>&1 | tail -1
  timeout 200 python tools/run_cfg.py c3 pack 2 2>&1 | tail -1
  [ $r = 1 ] && timeout 200 python tools/run_cfg.py c2 pack 2 2>&1 | tail -1
done; done
