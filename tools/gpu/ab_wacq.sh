#!/bin/bash
# A/B: eager stage wait polling with acquire loads (SALUS_WAIT_ACQ=1) vs relaxed polls + one acquire re-load
for r in 1 2; do for lib in paper_1902_04610_b200/libsalus.so build/ab/libsalus_wacq.so; do
  echo "== $lib round $r"
  SALUS_LIB=$lib timeout 100 python tools/run_cfg.py c1 fifo 3 2>&1 | tail -1
  SALUS_LIB=$lib timeout 100 python tools/run_cfg.py c1 srtf 3 2>&1 | tail -1
  SALUS_LIB=$lib timeout 200 python tools/run_cfg.py c4 srtf 1 2>&1 | tail -1
  SALUS_LIB=$lib timeout 200 python tools/run_cfg.py c4 pack 1 2>&1 | tail -1
  SALUS_LIB=$lib timeout 200 python tools/run_cfg.py c3 fair 2 2>&1 | tail -1
done; done
